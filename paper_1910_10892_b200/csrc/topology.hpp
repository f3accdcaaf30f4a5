// Grid geometry for the scanline engines (host side, setup only).
//
// Reproduces the reference's GridTopology exactly (grid.hpp:73-96,
// src/grid.cpp:13-114): direction order, scanline order and the dense
// per-direction edge numbering fix the p/q byte layout, so they are part of
// the drop-in contract. The formulation here is our own: a scanline of the
// canonical step (a,b) = (|dh|,|dw|) is the set of nodes sharing the
// invariant kappa = a*w - b*h (rows: kappa = h); scanlines are ordered by
// kappa ascending, start at their smallest-h node, and are mirrored for
// negative step components. Every scanline is straight, so on the device it
// is just {first node, length, edge base}: node j = first + j*(dh*W + dw).
#pragma once

#include <cstdint>
#include <vector>

namespace mrf {

struct Step {
  int dh, dw;
};

// Direction r and its opposite r^1 (src/grid.cpp:17-26).
inline Step direction_step(int r) {
  static const Step k[16] = {{0, 1},  {0, -1},  {1, 0},  {-1, 0}, {1, 1},  {-1, -1}, {1, -1}, {-1, 1},
                             {1, 2},  {-1, -2}, {1, -2}, {-1, 2}, {2, 1},  {-2, -1}, {2, -1}, {-2, 1}};
  return k[r];
}

struct Line {
  int32_t first;      // head node id
  int32_t length;     // nodes on the line (>= 1)
  int32_t edge_base;  // edge id of node 1 within its direction
};

class Topology {
 public:
  Topology(int height, int width, int connectivity);

  int height() const { return H_; }
  int width() const { return W_; }
  int nodes() const { return H_ * W_; }
  int num_dirs() const { return R_; }
  int64_t total_edges() const { return total_; }
  int64_t edge_count(int r) const { return count_[r]; }
  int64_t dir_offset(int r) const { return offset_[r]; }
  int node_step(int r) const { return direction_step(r).dh * W_ + direction_step(r).dw; }
  const std::vector<Line>& lines(int r) const { return lines_[r]; }
  int max_length(int r) const { return maxlen_[r]; }
  std::vector<int32_t> edge_index() const;  // [R][N], -1 at heads

 private:
  int H_, W_, R_;
  std::vector<std::vector<Line>> lines_;
  std::vector<int64_t> count_, offset_;
  std::vector<int> maxlen_;
  int64_t total_ = 0;
};

}  // namespace mrf
