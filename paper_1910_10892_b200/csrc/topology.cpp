#include "topology.hpp"

#include <algorithm>
#include <cstdlib>
#include <stdexcept>

namespace mrf {

namespace {

// Lines of the canonical (non-negative) step (a, b) on an H x W grid, as
// (head h, head w, length) in canonical coordinates, ordered by the line
// invariant. Rows (a = 0) are keyed by h, every other family by
// kappa = a*w - b*h; a line's head is its in-bounds node of smallest h.
struct CanonLine {
  int h, w, len;
};

std::vector<CanonLine> canonical_lines(int H, int W, int a, int b) {
  std::vector<CanonLine> out;
  auto walk = [&](int h, int w) {
    int n = 0;
    for (int y = h, x = w; y < H && x >= 0 && x < W; y += a, x += b) ++n;
    return n;
  };
  if (a == 0) {  // horizontal: one line per row
    for (int h = 0; h < H; ++h) out.push_back({h, 0, W});
    return out;
  }
  const int kmin = -b * (H - 1), kmax = a * (W - 1);
  for (int kappa = kmin; kappa <= kmax; ++kappa) {
    // smallest h in [0, H) with w = (kappa + b*h)/a integral and in [0, W)
    for (int h = 0; h < H; ++h) {
      const int num = kappa + b * h;
      if (num < 0 || num % a != 0) continue;
      const int w = num / a;
      if (w >= W) break;  // w grows with h (b >= 0): nothing further
      out.push_back({h, w, walk(h, w)});
      break;
    }
  }
  return out;
}

}  // namespace

Topology::Topology(int height, int width, int connectivity) : H_(height), W_(width), R_(connectivity) {
  if (height < 1 || width < 1) throw std::invalid_argument("topology: H and W must be >= 1");
  if (connectivity != 4 && connectivity != 8 && connectivity != 16)
    throw std::invalid_argument("topology: connectivity must be 4, 8 or 16");
  if (int64_t(height) * width > (int64_t(1) << 30)) throw std::invalid_argument("topology: grid too large");
  lines_.resize(R_);
  count_.assign(R_, 0);
  offset_.assign(R_, 0);
  maxlen_.assign(R_, 0);
  for (int r = 0; r < R_; ++r) {
    const Step s = direction_step(r);
    int32_t edges = 0;
    for (const CanonLine& c : canonical_lines(H_, W_, std::abs(s.dh), std::abs(s.dw))) {
      const int h = s.dh < 0 ? H_ - 1 - c.h : c.h;
      const int w = s.dw < 0 ? W_ - 1 - c.w : c.w;
      lines_[r].push_back({h * W_ + w, c.len, edges});
      edges += c.len - 1;
      maxlen_[r] = std::max(maxlen_[r], c.len);
    }
    count_[r] = edges;
    offset_[r] = total_;
    total_ += edges;
  }
}

std::vector<int32_t> Topology::edge_index() const {
  const int N = nodes();
  std::vector<int32_t> out(size_t(R_) * N, -1);
  for (int r = 0; r < R_; ++r) {
    const int st = node_step(r);
    for (const Line& l : lines_[r])
      for (int j = 1; j < l.length; ++j) out[size_t(r) * N + l.first + size_t(j) * st] = l.edge_base + j - 1;
  }
  return out;
}

}  // namespace mrf
