// mrf/mp_cuda.hpp -- C++ drop-in for the reference library's hot path.
//
// A user of the reference (/root/reference/proj, namespace mp) who includes
// <mp/isgmr.hpp>, <mp/trwp.hpp>, <mp/autodiff.hpp> and calls
//   mp::isgmr_forward<float>(topo, pots, K, threads)        isgmr.hpp:145-152
//   mp::trwp_forward<float>(topo, pots, rho, K, threads)    trwp.hpp:148-156
//   mp::isgmr_backward<float>(topo, pots, indices, dc, t)   autodiff.hpp:63-126
//   mp::trwp_backward<float>(topo, pots, rho, indices, dc, t) autodiff.hpp:133-197
// includes this header instead and links libmrf_cuda.so. Types, names,
// layouts and exceptions follow the reference (grid.hpp, potentials.hpp,
// index_store.hpp, inference.hpp, autodiff.hpp); `threads` is accepted and
// ignored; every computation runs on the current CUDA device through the
// C-ABI (include/mrf_cuda.h), with host<->device copies of the std::vector
// arguments and results. Only Real = float exists here: the double
// instantiation of the reference stays a CPU tool (gradient checking).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <cuda_runtime_api.h>

#include "../mrf_cuda.h"

namespace mp {

inline constexpr int kMaxLabels = 256;

namespace cuda_detail {

inline void check(int rc) {
  if (rc == MRF_OK) return;
  if (rc == MRF_EINVAL) throw std::invalid_argument(mrf_last_error());
  throw std::runtime_error(std::string("mrf_cuda: ") + mrf_last_error());
}
inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device allocation (stream-ordered on the legacy default stream).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) : bytes_(bytes) {
    if (bytes) check_cuda(cudaMalloc(&ptr_, bytes), "cudaMalloc");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(std::exchange(o.ptr_, nullptr)), bytes_(o.bytes_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      if (ptr_) cudaFree(ptr_);
      ptr_ = std::exchange(o.ptr_, nullptr);
      bytes_ = o.bytes_;
    }
    return *this;
  }
  ~DeviceBuffer() {
    if (ptr_) cudaFree(ptr_);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(ptr_);
  }
  size_t bytes() const { return bytes_; }

  // `slack` extra bytes after the copied elements, zero-filled (p/q index
  // buffers: the kernels read them as aligned 32-bit words)
  template <class T>
  static DeviceBuffer upload(const T* src, size_t count, size_t slack = 0) {
    DeviceBuffer b(sizeof(T) * count + slack);
    if (count) check_cuda(cudaMemcpy(b.ptr_, src, sizeof(T) * count, cudaMemcpyHostToDevice), "H2D");
    if (slack) check_cuda(cudaMemset(static_cast<char*>(b.ptr_) + sizeof(T) * count, 0, slack), "memset");
    return b;
  }
  template <class T>
  void download(T* dst, size_t count) const {
    if (count) check_cuda(cudaMemcpy(dst, ptr_, sizeof(T) * count, cudaMemcpyDeviceToHost), "D2H");
  }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace cuda_detail

// ------------------------------------------------------------------ geometry

/// grid.hpp:11-25
struct GridGraph {
  int height = 0;
  int width = 0;
  GridGraph() = default;
  GridGraph(int h, int w) : height(h), width(w) {
    if (h < 1 || w < 1) throw std::invalid_argument("GridGraph: H and W must be >= 1");
  }
  int nodes() const { return height * width; }
  int id(int h, int w) const { return h * width + w; }
  std::pair<int, int> coords(int node) const { return {node / width, node % width}; }
  bool contains(int h, int w) const { return h >= 0 && h < height && w >= 0 && w < width; }
};

/// grid.hpp:29-33
struct Direction {
  int dh = 0;
  int dw = 0;
  int opposite = -1;
};

/// grid.hpp:38-50; order E,W,S,N,SE,NW,SW,NE,... with opposite = r^1.
class DirectionSet {
 public:
  static DirectionSet build(int connectivity) {
    if (connectivity != 4 && connectivity != 8 && connectivity != 16)
      throw std::invalid_argument("DirectionSet: connectivity must be 4, 8 or 16");
    static const int k[16][2] = {{0, 1},  {0, -1},  {1, 0},  {-1, 0}, {1, 1},  {-1, -1}, {1, -1}, {-1, 1},
                                 {1, 2},  {-1, -2}, {1, -2}, {-1, 2}, {2, 1},  {-2, -1}, {2, -1}, {-2, 1}};
    DirectionSet s;
    for (int r = 0; r < connectivity; ++r) s.dirs_.push_back(Direction{k[r][0], k[r][1], r ^ 1});
    return s;
  }
  int size() const { return static_cast<int>(dirs_.size()); }
  int connectivity() const { return size(); }
  int families() const { return size() / 2; }
  const Direction& operator[](int r) const { return dirs_[r]; }
  const std::vector<Direction>& all() const { return dirs_; }

 private:
  std::vector<Direction> dirs_;
};

/// grid.hpp:53-57
struct Scanline {
  int direction = -1;
  std::pair<int, int> first_node{};
  std::vector<int32_t> nodes;
};

/// grid.hpp:73-96. Geometry is computed by libmrf_cuda (identical scanline
/// order and edge numbering); the handle also carries the device line tables.
class GridTopology {
 public:
  GridTopology(const GridGraph& g, DirectionSet dirs) : grid_(g), dirs_(std::move(dirs)) {
    mrf_topology_t h = nullptr;
    cuda_detail::check(mrf_topology_create(g.height, g.width, dirs_.size(), &h));
    handle_ = std::shared_ptr<mrf_topology_s>(h, [](mrf_topology_t t) { mrf_topology_destroy(t); });
    const int R = dirs_.size();
    edge_count_.resize(R);
    dir_offset_.resize(R);
    int nd = 0;
    cuda_detail::check(mrf_topology_info(h, &nd, &total_edges_, edge_count_.data(), dir_offset_.data()));
    edge_index_.assign(size_t(R) * g.nodes(), -1);
    cuda_detail::check(mrf_topology_edge_index(h, edge_index_.data()));
    scanlines_.resize(R);
    for (int r = 0; r < R; ++r) {
      int32_t cnt = 0;
      cuda_detail::check(mrf_topology_scanlines(h, r, nullptr, nullptr, &cnt, 0));
      std::vector<int32_t> first(cnt), len(cnt);
      cuda_detail::check(mrf_topology_scanlines(h, r, first.data(), len.data(), &cnt, cnt));
      const int step = dirs_[r].dh * g.width + dirs_[r].dw;
      for (int t = 0; t < cnt; ++t) {
        Scanline sl;
        sl.direction = r;
        for (int j = 0; j < len[t]; ++j) sl.nodes.push_back(first[t] + j * step);
        sl.first_node = g.coords(sl.nodes.front());
        scanlines_[r].push_back(std::move(sl));
      }
    }
  }

  const GridGraph& grid() const { return grid_; }
  const DirectionSet& dirs() const { return dirs_; }
  int num_dirs() const { return dirs_.size(); }
  const std::vector<Scanline>& scanlines(int r) const { return scanlines_[r]; }
  int32_t edge_index(int r, int node) const { return edge_index_[size_t(r) * grid_.nodes() + node]; }
  std::int64_t edge_count(int r) const { return edge_count_[r]; }
  std::int64_t total_edges() const { return total_edges_; }
  std::int64_t dir_offset(int r) const { return dir_offset_[r]; }
  mrf_topology_t handle() const { return handle_.get(); }

 private:
  GridGraph grid_;
  DirectionSet dirs_;
  std::shared_ptr<mrf_topology_s> handle_;
  std::vector<std::vector<Scanline>> scanlines_;
  std::vector<int32_t> edge_index_;
  std::vector<std::int64_t> edge_count_, dir_offset_;
  std::int64_t total_edges_ = 0;
};

// --------------------------------------------------------------- potentials

enum class PairwiseKind { potts, truncated_linear, truncated_quadratic, sgm_p1p2, explicit_matrix };

struct PairwiseParams {
  double trunc = -1.0;
  double p1 = 1.0;
  double p2 = 1.0;
};

/// potentials.hpp:27-35
template <class Real>
struct PairwiseFunction {
  PairwiseKind kind = PairwiseKind::potts;
  int labels = 0;
  std::vector<Real> table;
  Real operator()(int a, int b) const { return table[a * labels + b]; }
  Real& at(int a, int b) { return table[a * labels + b]; }
};

/// potentials.hpp:38-72: built-ins computed in double from |a-b|, cast.
template <class Real>
PairwiseFunction<Real> build_pairwise(PairwiseKind kind, const PairwiseParams& params, int labels) {
  if (labels < 1 || labels > kMaxLabels) throw std::invalid_argument("build_pairwise: label count must be in [1, 256]");
  PairwiseFunction<Real> v;
  v.kind = kind;
  v.labels = labels;
  v.table.assign(size_t(labels) * labels, Real(0));
  for (int a = 0; a < labels; ++a)
    for (int b = 0; b < labels; ++b) {
      const double d = std::abs(a - b);
      double val = 0.0;
      switch (kind) {
        case PairwiseKind::potts: val = a == b ? 0.0 : 1.0; break;
        case PairwiseKind::truncated_linear:
          if (params.trunc <= 0) throw std::invalid_argument("truncated_linear: trunc must be > 0");
          val = d < params.trunc ? d : params.trunc;
          break;
        case PairwiseKind::truncated_quadratic:
          if (params.trunc <= 0) throw std::invalid_argument("truncated_quadratic: trunc must be > 0");
          val = d * d < params.trunc ? d * d : params.trunc;
          break;
        case PairwiseKind::sgm_p1p2:
          if (!(0 < params.p1 && params.p1 <= params.p2)) throw std::invalid_argument("sgm_p1p2: need 0 < P1 <= P2");
          val = a == b ? 0.0 : (d == 1.0 ? params.p1 : params.p2);
          break;
        case PairwiseKind::explicit_matrix:
          throw std::invalid_argument("build_pairwise: explicit_matrix takes a user table");
      }
      v.at(a, b) = static_cast<Real>(val);
    }
  return v;
}

template <class Real>
PairwiseFunction<Real> explicit_pairwise(std::vector<Real> table, int labels) {
  if (table.size() != size_t(labels) * labels) throw std::invalid_argument("explicit_pairwise: table size mismatch");
  PairwiseFunction<Real> v;
  v.kind = PairwiseKind::explicit_matrix;
  v.labels = labels;
  v.table = std::move(table);
  return v;
}

/// potentials.hpp:88-105
template <class Real>
struct UnaryVolume {
  int height = 0, width = 0, labels = 0;
  std::vector<Real> values;
  UnaryVolume() = default;
  UnaryVolume(int h, int w, int l, Real fill = Real(0)) : height(h), width(w), labels(l), values(size_t(h) * w * l, fill) {
    if (l < 1 || l > kMaxLabels) throw std::invalid_argument("UnaryVolume: label count must be in [1, 256]");
  }
  Real at(int node, int label) const { return values[size_t(node) * labels + label]; }
  Real& at(int node, int label) { return values[size_t(node) * labels + label]; }
  const Real* row(int node) const { return values.data() + size_t(node) * labels; }
  int nodes() const { return height * width; }
};

/// potentials.hpp:113-139
template <class Real>
class EdgeWeights {
 public:
  static EdgeWeights constant(Real w) {
    if (!(w >= 0)) throw std::invalid_argument("EdgeWeights: weights must be nonnegative");
    EdgeWeights e;
    e.constant_ = w;
    return e;
  }
  static EdgeWeights planes(std::vector<std::vector<Real>> planes) {
    EdgeWeights e;
    e.planes_ = std::move(planes);
    return e;
  }
  bool is_constant() const { return planes_.empty(); }
  const std::vector<std::vector<Real>>& plane_data() const { return planes_; }
  std::vector<std::vector<Real>>& plane_data() { return planes_; }
  Real weight(int r, int prev, int cur) const {
    if (planes_.empty()) return constant_;
    return planes_[r >> 1][(r & 1) ? cur : prev];
  }
  static int plane_node(int r, int prev, int cur) { return (r & 1) ? cur : prev; }

 private:
  Real constant_ = Real(1);
  std::vector<std::vector<Real>> planes_;
};

/// potentials.hpp:143-163
template <class Real>
struct TreeCoefficients {
  Real uniform = Real(0.5);
  std::vector<std::vector<Real>> planes;
  Real at(int r, int prev, int cur) const {
    if (planes.empty()) return uniform;
    return planes[r >> 1][(r & 1) ? cur : prev];
  }
};

template <class Real>
TreeCoefficients<Real> default_rho(int connectivity, Real value = Real(0.5)) {
  DirectionSet::build(connectivity);
  if (!(value > 0 && value <= 1)) throw std::invalid_argument("rho must be in (0, 1]");
  return TreeCoefficients<Real>{value, {}};
}

template <class Real>
struct PotentialSet {
  UnaryVolume<Real> unary;
  PairwiseFunction<Real> pairwise;
  EdgeWeights<Real> weights = EdgeWeights<Real>::constant(Real(1));
};

// --------------------------------------------------------------- outputs

/// index_store.hpp:16-58 (same byte layout; filled from the device)
class IndexStore {
 public:
  IndexStore(const GridTopology& topo, int labels) : labels_(labels), edges_(topo.total_edges()) {}
  void append_iteration() { set_iterations(iterations_ + 1); }
  // not in the reference: size the store for k iterations at once (the
  // device path fills every iteration in one copy)
  void set_iterations(int k) {
    iterations_ = k;
    p_.resize(size_t(iterations_) * edges_ * labels_, 0);
    q_.resize(size_t(iterations_) * edges_, 0);
  }
  int iterations() const { return iterations_; }
  const std::vector<std::uint8_t>& p_data() const { return p_; }
  const std::vector<std::uint8_t>& q_data() const { return q_; }
  std::vector<std::uint8_t>& p_data() { return p_; }
  std::vector<std::uint8_t>& q_data() { return q_; }
  int labels() const { return labels_; }
  std::int64_t edges() const { return edges_; }
  size_t bytes() const { return p_.size() + q_.size(); }
  std::uint8_t* p_row(const GridTopology& topo, int k, int r, int32_t e) { return p_.data() + flat(topo, k, r, e) * labels_; }
  const std::uint8_t* p_row(const GridTopology& topo, int k, int r, int32_t e) const {
    return p_.data() + flat(topo, k, r, e) * labels_;
  }
  std::uint8_t& q_at(const GridTopology& topo, int k, int r, int32_t e) { return q_[flat(topo, k, r, e)]; }
  std::uint8_t q_at(const GridTopology& topo, int k, int r, int32_t e) const { return q_[flat(topo, k, r, e)]; }

 private:
  size_t flat(const GridTopology& topo, int k, int r, int32_t e) const {
    return size_t(k) * edges_ + topo.dir_offset(r) + e;
  }
  int labels_ = 0;
  int iterations_ = 0;
  std::int64_t edges_ = 0;
  std::vector<std::uint8_t> p_, q_;
};

/// inference.hpp:16-23
template <class Real>
struct CostOutput {
  int height = 0, width = 0, labels = 0;
  std::vector<Real> cost;
  std::vector<std::uint16_t> labels_map;
  const Real* row(int node) const { return cost.data() + size_t(node) * labels; }
};

/// inference.hpp:62-68. min_argmin_gap is a diagnostic the GPU path does not
/// track; it is +inf.
template <class Real>
struct ForwardResult {
  CostOutput<Real> output;
  std::vector<Real> messages;
  IndexStore indices;
  Real min_argmin_gap;
};

/// autodiff.hpp:17-29
template <class Real>
struct GradientSet {
  std::vector<Real> unary;
  std::vector<Real> pairwise;
  std::vector<std::vector<Real>> edge_weights;
  Real edge_weight_total() const {
    Real s = Real(0);
    for (const auto& p : edge_weights)
      for (Real v : p) s += v;
    return s;
  }
};

// ------------------------------------------------------------ entry points

namespace cuda_detail {

template <class Real>
constexpr void require_float() {
  static_assert(std::is_same_v<Real, float>, "mrf_cuda computes in FP32; use the CPU reference for Real=double");
}

struct DeviceProblem {
  DeviceBuffer unary, V, wplanes, rplanes;
  mrf_problem_f32 prob{};
};

inline std::vector<float> flatten(const std::vector<std::vector<float>>& planes, size_t n, int fam) {
  std::vector<float> out(size_t(fam) * n);
  if (planes.size() != size_t(fam)) throw std::invalid_argument("plane count mismatch");
  for (int f = 0; f < fam; ++f) {
    if (planes[f].size() != n) throw std::invalid_argument("plane size mismatch");
    std::memcpy(out.data() + f * n, planes[f].data(), sizeof(float) * n);
  }
  return out;
}

inline DeviceProblem upload(const GridTopology& topo, const PotentialSet<float>& pots, const TreeCoefficients<float>* rho,
                            bool check_finite) {
  const auto& u = pots.unary;
  const int L = u.labels;
  if (L > kMaxLabels) throw std::invalid_argument("engine: more than 256 labels");
  if (u.height != topo.grid().height || u.width != topo.grid().width)
    throw std::invalid_argument("unary volume does not match the topology");
  if (check_finite)
    for (float v : u.values)
      if (!std::isfinite(static_cast<double>(v))) throw std::invalid_argument("engine: non-finite unary potential");
  if (pots.pairwise.labels != L || pots.pairwise.table.size() != size_t(L) * L)
    throw std::invalid_argument("pairwise table does not match the label count");
  DeviceProblem d;
  const size_t n = size_t(topo.grid().nodes());
  const int fam = topo.num_dirs() / 2;
  d.unary = DeviceBuffer::upload(u.values.data(), u.values.size());
  d.V = DeviceBuffer::upload(pots.pairwise.table.data(), pots.pairwise.table.size());
  d.prob.batch = 1;
  d.prob.height = u.height;
  d.prob.width = u.width;
  d.prob.labels = L;
  d.prob.unary = d.unary.as<float>();
  d.prob.pairwise = d.V.as<float>();
  if (pots.weights.is_constant()) {
    d.prob.weight = pots.weights.weight(0, 0, 0);
  } else {
    const auto flat = flatten(pots.weights.plane_data(), n, fam);
    d.wplanes = DeviceBuffer::upload(flat.data(), flat.size());
    d.prob.weight_planes = d.wplanes.as<float>();
  }
  d.prob.rho = 0.5f;
  if (rho) {
    if (rho->planes.empty()) {
      d.prob.rho = rho->uniform;
    } else {
      const auto flat = flatten(rho->planes, n, fam);
      d.rplanes = DeviceBuffer::upload(flat.data(), flat.size());
      d.prob.rho_planes = d.rplanes.as<float>();
    }
  }
  return d;
}

inline ForwardResult<float> forward(int engine, const GridTopology& topo, const PotentialSet<float>& pots,
                                    const TreeCoefficients<float>* rho, int K) {
  if (K < 1)
    throw std::invalid_argument(engine == MRF_ENGINE_ISGMR ? "isgmr_forward: iterations must be >= 1"
                                                           : "trwp_forward: iterations must be >= 1");
  DeviceProblem d = upload(topo, pots, rho, true);
  d.prob.assume_finite = 1;  // checked on the host above
  const int L = d.prob.labels, R = topo.num_dirs();
  const size_t n = size_t(topo.grid().nodes()), E = size_t(topo.total_edges());
  DeviceBuffer cost(sizeof(float) * n * L), labels(2 * n), msg(sizeof(float) * R * n * L), p(size_t(K) * E * L + 4),
      q(size_t(K) * E + 4);
  const size_t wsb = mrf_forward_workspace_bytes(topo.handle(), &d.prob, engine, K);
  DeviceBuffer ws(wsb);
  mrf_forward_out out{cost.as<float>(), labels.as<uint16_t>(), msg.as<float>(), p.as<uint8_t>(), q.as<uint8_t>()};
  if (engine == MRF_ENGINE_ISGMR)
    check(mrf_isgmr_forward_f32(topo.handle(), &d.prob, K, &out, ws.as<void>(), wsb, nullptr));
  else
    check(mrf_trwp_forward_f32(topo.handle(), &d.prob, K, &out, ws.as<void>(), wsb, nullptr));
  ForwardResult<float> res{CostOutput<float>{}, {}, IndexStore(topo, L), std::numeric_limits<float>::infinity()};
  res.output.height = topo.grid().height;
  res.output.width = topo.grid().width;
  res.output.labels = L;
  res.output.cost.resize(n * L);
  res.output.labels_map.resize(n);
  res.messages.resize(size_t(R) * n * L);
  res.indices.set_iterations(K);
  cost.download(res.output.cost.data(), n * L);
  labels.download(res.output.labels_map.data(), n);
  msg.download(res.messages.data(), res.messages.size());
  p.download(res.indices.p_data().data(), res.indices.p_data().size());
  q.download(res.indices.q_data().data(), res.indices.q_data().size());
  return res;
}

inline GradientSet<float> backward(int engine, const GridTopology& topo, const PotentialSet<float>& pots,
                                   const TreeCoefficients<float>* rho, const IndexStore& indices,
                                   const std::vector<float>& grad_cost) {
  const size_t n = size_t(topo.grid().nodes());
  const int L = pots.unary.labels, R = topo.num_dirs();
  if (grad_cost.size() != n * L) throw std::invalid_argument("backward: cost gradient size mismatch");
  if (indices.labels() != L || indices.edges() != topo.total_edges())
    throw std::invalid_argument("backward: index store does not match the problem");
  const int K = indices.iterations();
  DeviceProblem d = upload(topo, pots, rho, false);
  DeviceBuffer p = DeviceBuffer::upload(indices.p_data().data(), indices.p_data().size(), 4);
  DeviceBuffer q = DeviceBuffer::upload(indices.q_data().data(), indices.q_data().size(), 4);
  DeviceBuffer gc = DeviceBuffer::upload(grad_cost.data(), grad_cost.size());
  DeviceBuffer gu(sizeof(float) * n * L), gv(sizeof(float) * L * L), gw(sizeof(float) * (R / 2) * n);
  const size_t wsb = mrf_backward_workspace_bytes(topo.handle(), &d.prob, engine, K);
  DeviceBuffer ws(wsb);
  mrf_grads_f32 g{gu.as<float>(), gv.as<float>(), gw.as<float>()};
  if (engine == MRF_ENGINE_ISGMR)
    check(mrf_isgmr_backward_f32(topo.handle(), &d.prob, K, p.as<uint8_t>(), q.as<uint8_t>(), gc.as<float>(), &g,
                                 ws.as<void>(), wsb, nullptr));
  else
    check(mrf_trwp_backward_f32(topo.handle(), &d.prob, K, p.as<uint8_t>(), q.as<uint8_t>(), gc.as<float>(), &g,
                                ws.as<void>(), wsb, nullptr));
  GradientSet<float> out;
  out.unary.resize(n * L);
  out.pairwise.resize(size_t(L) * L);
  out.edge_weights.assign(R / 2, std::vector<float>(n));
  gu.download(out.unary.data(), out.unary.size());
  gv.download(out.pairwise.data(), out.pairwise.size());
  std::vector<float> flat((R / 2) * n);
  gw.download(flat.data(), flat.size());
  for (int f = 0; f < R / 2; ++f) std::memcpy(out.edge_weights[f].data(), flat.data() + f * n, sizeof(float) * n);
  return out;
}

}  // namespace cuda_detail

/// isgmr.hpp:145-152
template <class Real>
ForwardResult<Real> isgmr_forward(const GridTopology& topo, const PotentialSet<Real>& pots, int iterations,
                                  int threads = 1) {
  cuda_detail::require_float<Real>();
  (void)threads;
  return cuda_detail::forward(MRF_ENGINE_ISGMR, topo, pots, nullptr, iterations);
}

/// trwp.hpp:148-156
template <class Real>
ForwardResult<Real> trwp_forward(const GridTopology& topo, const PotentialSet<Real>& pots,
                                 const TreeCoefficients<Real>& rho, int iterations, int threads = 1) {
  cuda_detail::require_float<Real>();
  (void)threads;
  if (rho.planes.empty() && !(rho.uniform > 0 && rho.uniform <= 1)) throw std::invalid_argument("rho must be in (0, 1]");
  return cuda_detail::forward(MRF_ENGINE_TRWP, topo, pots, &rho, iterations);
}

/// autodiff.hpp:63-126
template <class Real>
GradientSet<Real> isgmr_backward(const GridTopology& topo, const PotentialSet<Real>& pots, const IndexStore& indices,
                                 const std::vector<Real>& grad_cost, int threads = 1) {
  cuda_detail::require_float<Real>();
  (void)threads;
  return cuda_detail::backward(MRF_ENGINE_ISGMR, topo, pots, nullptr, indices, grad_cost);
}

/// autodiff.hpp:133-197
template <class Real>
GradientSet<Real> trwp_backward(const GridTopology& topo, const PotentialSet<Real>& pots,
                                const TreeCoefficients<Real>& rho, const IndexStore& indices,
                                const std::vector<Real>& grad_cost, int threads = 1) {
  cuda_detail::require_float<Real>();
  (void)threads;
  return cuda_detail::backward(MRF_ENGINE_TRWP, topo, pots, &rho, indices, grad_cost);
}

namespace cuda_detail {

// Device state of one IsgmrEngine / TrwpEngine: the potentials uploaded once,
// messages (ISGMR: published m and swept mhat), and the index store on the
// device, grown by doubling when step() runs past its capacity (the
// reference's append_iteration regrows the host vectors every iteration,
// index_store.hpp:21-25). Host copies are made on demand.
class EngineState {
 public:
  EngineState(int engine, const GridTopology& topo, const PotentialSet<float>& pots, const TreeCoefficients<float>* rho,
              bool diagnostic)
      : engine_(engine), topo_(topo), d_(upload(topo, pots, rho, true)) {
    d_.prob.assume_finite = 1;  // checked on the host by upload()
    L_ = d_.prob.labels;
    R_ = topo.num_dirs();
    n_ = size_t(topo.grid().nodes());
    E_ = size_t(topo.total_edges());
    const size_t mb = sizeof(float) * R_ * n_ * L_;
    m_ = DeviceBuffer(mb);
    check_cuda(cudaMemset(m_.as<void>(), 0, mb), "memset");
    if (engine == MRF_ENGINE_ISGMR) {
      mhat_ = DeviceBuffer(mb);
      check_cuda(cudaMemset(mhat_.as<void>(), 0, mb), "memset");
    }
    reserve(1);
    if (diagnostic) {
      const float inf = std::numeric_limits<float>::infinity();
      gap_ = DeviceBuffer::upload(&inf, 1);
      d_.prob.diag_gap = gap_.as<float>();
    }
  }

  void step() {
    if (k_ == cap_) reserve(2 * cap_);
    if (engine_ == MRF_ENGINE_ISGMR) {
      check(mrf_isgmr_step_f32(topo_.handle(), &d_.prob, k_, cap_, m_.as<float>(), mhat_.as<float>(),
                               p_.as<std::uint8_t>(), q_.as<std::uint8_t>(), nullptr));
      std::swap(m_, mhat_);  // publish m <- mhat (isgmr.hpp:55)
    } else {
      check(mrf_trwp_step_f32(topo_.handle(), &d_.prob, k_, cap_, m_.as<float>(), p_.as<std::uint8_t>(),
                              q_.as<std::uint8_t>(), nullptr));
    }
    ++k_;
  }

  int iterations() const { return k_; }

  CostOutput<float> aggregate() const {
    DeviceBuffer cost(sizeof(float) * n_ * L_), labels(2 * n_);
    check(mrf_aggregate_f32(topo_.handle(), &d_.prob, m_.as<float>(), cost.as<float>(), labels.as<std::uint16_t>(),
                            nullptr));
    CostOutput<float> out;
    out.height = topo_.grid().height;
    out.width = topo_.grid().width;
    out.labels = L_;
    out.cost.resize(n_ * L_);
    out.labels_map.resize(n_);
    cost.download(out.cost.data(), out.cost.size());
    labels.download(out.labels_map.data(), n_);
    return out;
  }

  void messages(std::vector<float>& out) const {
    out.resize(size_t(R_) * n_ * L_);
    m_.download(out.data(), out.size());
  }

  IndexStore indices() const {
    IndexStore st(topo_, L_);
    st.set_iterations(k_);
    p_.download(st.p_data().data(), st.p_data().size());
    q_.download(st.q_data().data(), st.q_data().size());
    return st;
  }

  float gap() const {
    float g = std::numeric_limits<float>::infinity();
    if (gap_.bytes()) gap_.download(&g, 1);
    return g;
  }

 private:
  void reserve(int cap) {
    // +4 bytes: the kernels read p/q as aligned 32-bit words
    DeviceBuffer p(size_t(cap) * E_ * L_ + 4), q(size_t(cap) * E_ + 4);
    if (k_) {
      check_cuda(cudaMemcpy(p.as<void>(), p_.as<void>(), size_t(k_) * E_ * L_, cudaMemcpyDeviceToDevice), "D2D");
      check_cuda(cudaMemcpy(q.as<void>(), q_.as<void>(), size_t(k_) * E_, cudaMemcpyDeviceToDevice), "D2D");
    }
    p_ = std::move(p);
    q_ = std::move(q);
    cap_ = cap;
  }

  int engine_;
  const GridTopology& topo_;
  DeviceProblem d_;
  int L_ = 0, R_ = 0;
  size_t n_ = 0, E_ = 0;
  int k_ = 0, cap_ = 0;
  DeviceBuffer m_, mhat_, p_, q_, gap_;
};

}  // namespace cuda_detail

/// isgmr.hpp:26-143. Same interface; the potentials are uploaded at
/// construction (the reference keeps references to them), every step() runs
/// on the device and host copies are made by messages() / indices() /
/// aggregate(). `diagnostic` (not in the reference) turns on min_argmin_gap
/// tracking (dense min-plus kernel: same results, slower); without it
/// min_argmin_gap() is +inf.
template <class Real>
class IsgmrEngine {
 public:
  IsgmrEngine(const GridTopology& topo, const PotentialSet<Real>& pots, int threads = 1, bool diagnostic = false)
      : st_((cuda_detail::require_float<Real>(), MRF_ENGINE_ISGMR), topo, pots, nullptr, diagnostic) {
    (void)threads;
  }
  void step() { st_.step(); }
  int iterations() const { return st_.iterations(); }
  CostOutput<Real> aggregate() const { return st_.aggregate(); }
  const std::vector<Real>& messages() const {
    st_.messages(m_);
    return m_;
  }
  const IndexStore& indices() const {
    idx_.emplace(st_.indices());
    return *idx_;
  }
  IndexStore&& take_indices() {
    idx_.emplace(st_.indices());
    return std::move(*idx_);
  }
  Real min_argmin_gap() const { return st_.gap(); }

 private:
  cuda_detail::EngineState st_;
  mutable std::vector<Real> m_;
  mutable std::optional<IndexStore> idx_;
};

/// trwp.hpp:25-146 (see IsgmrEngine).
template <class Real>
class TrwpEngine {
 public:
  TrwpEngine(const GridTopology& topo, const PotentialSet<Real>& pots, TreeCoefficients<Real> rho, int threads = 1,
             bool diagnostic = false)
      : rho_(check_rho(std::move(rho))), st_(MRF_ENGINE_TRWP, topo, pots, &rho_, diagnostic) {
    (void)threads;
  }
  void step() { st_.step(); }
  int iterations() const { return st_.iterations(); }
  CostOutput<Real> aggregate() const { return st_.aggregate(); }
  const std::vector<Real>& messages() const {
    st_.messages(m_);
    return m_;
  }
  const IndexStore& indices() const {
    idx_.emplace(st_.indices());
    return *idx_;
  }
  IndexStore&& take_indices() {
    idx_.emplace(st_.indices());
    return std::move(*idx_);
  }
  Real min_argmin_gap() const { return st_.gap(); }

 private:
  static TreeCoefficients<Real> check_rho(TreeCoefficients<Real> rho) {
    cuda_detail::require_float<Real>();
    if (rho.planes.empty() && !(rho.uniform > 0 && rho.uniform <= 1)) throw std::invalid_argument("rho must be in (0, 1]");
    return rho;
  }
  TreeCoefficients<Real> rho_;
  cuda_detail::EngineState st_;
  mutable std::vector<Real> m_;
  mutable std::optional<IndexStore> idx_;
};

/// softhead.hpp:15-20
template <class Real>
struct SoftHeadResult {
  std::vector<Real> confidence;  // N*L, softmax(-c) per node
  std::vector<Real> disparity;   // N, expected label under confidence
  Real loss;                     // mean absolute error against ground truth
};

namespace cuda_detail {

// One fused pass (mrf_soft_head_f32): confidence, disparity, loss and, when
// grad != nullptr, the loss gradient with respect to the cost volume.
inline SoftHeadResult<float> soft_head(const CostOutput<float>& cost, const std::vector<float>& target,
                                       std::vector<float>* grad, const char* who) {
  const int L = cost.labels;
  const size_t n = L ? cost.cost.size() / size_t(L) : 0;
  if (target.size() != n) throw std::invalid_argument(std::string(who) + ": target size mismatch");
  SoftHeadResult<float> res;
  res.confidence.resize(cost.cost.size());
  res.disparity.resize(n);
  res.loss = 0.0f;
  if (n == 0) return res;
  auto c = DeviceBuffer::upload(cost.cost.data(), cost.cost.size());
  auto t = DeviceBuffer::upload(target.data(), target.size());
  DeviceBuffer f(sizeof(float) * cost.cost.size()), d(sizeof(float) * n), g(grad ? sizeof(float) * cost.cost.size() : 0),
      loss(sizeof(float));
  check(mrf_soft_head_f32(1, int(n), L, c.as<float>(), t.as<float>(), f.as<float>(), d.as<float>(),
                          grad ? g.as<float>() : nullptr, loss.as<float>(), nullptr));
  f.download(res.confidence.data(), res.confidence.size());
  d.download(res.disparity.data(), n);
  loss.download(&res.loss, 1);
  if (grad) {
    grad->resize(cost.cost.size());
    g.download(grad->data(), grad->size());
  }
  return res;
}

}  // namespace cuda_detail

/// softhead.hpp:22-56
template <class Real>
SoftHeadResult<Real> soft_head_forward(const CostOutput<Real>& cost, const std::vector<Real>& target) {
  cuda_detail::require_float<Real>();
  return cuda_detail::soft_head(cost, target, nullptr, "soft_head_forward");
}

/// softhead.hpp:58-74 (the gradient is recomputed from the cost volume in the
/// same fused pass; `head` is the forward's result for the same inputs)
template <class Real>
std::vector<Real> soft_head_backward(const CostOutput<Real>& cost, const SoftHeadResult<Real>& head,
                                     const std::vector<Real>& target) {
  cuda_detail::require_float<Real>();
  (void)head;
  std::vector<float> grad;
  cuda_detail::soft_head(cost, target, &grad, "soft_head_backward");
  return grad;
}

/// potentials.hpp:175-199
template <class Real, class Label>
double energy(const GridTopology& topo, const PotentialSet<Real>& pots, const std::vector<Label>& labels) {
  cuda_detail::require_float<Real>();
  const GridGraph& g = topo.grid();
  if (static_cast<int>(labels.size()) != g.nodes()) throw std::invalid_argument("energy: labelling size mismatch");
  std::vector<std::uint16_t> lab(labels.size());
  for (size_t i = 0; i < labels.size(); ++i) {
    const long long x = static_cast<long long>(labels[i]);
    if (x < 0 || x >= pots.unary.labels) throw std::out_of_range("energy: label out of range");
    lab[i] = static_cast<std::uint16_t>(x);
  }
  auto d = cuda_detail::upload(topo, pots, nullptr, false);
  auto dl = cuda_detail::DeviceBuffer::upload(lab.data(), lab.size());
  double e = 0.0;
  cuda_detail::check(mrf_energy_f32(topo.handle(), &d.prob, dl.as<std::uint16_t>(), &e, nullptr));
  return e;
}

/// baselines.hpp:16-24
enum class SgmVariant { standard, revised };

template <class Real>
struct SgmResult {
  CostOutput<Real> output;
  std::vector<Real> messages;  // R*N*L
};

namespace cuda_detail {

// One SGM round on uploaded potentials (mrf_sgm_f32), results left on the device.
struct SgmRound {
  DeviceBuffer msg, cost, labels;
};

inline SgmRound sgm_round(const GridTopology& topo, const mrf_problem_f32& prob, SgmVariant variant) {
  const size_t n = size_t(topo.grid().nodes()), L = size_t(prob.labels), R = size_t(topo.num_dirs());
  SgmRound rd{DeviceBuffer(sizeof(float) * R * n * L), DeviceBuffer(sizeof(float) * n * L), DeviceBuffer(2 * n)};
  check(mrf_sgm_f32(topo.handle(), &prob, variant == SgmVariant::revised ? 1 : 0, rd.msg.as<float>(),
                    rd.cost.as<float>(), rd.labels.as<std::uint16_t>(), nullptr));
  return rd;
}

inline CostOutput<float> download_cost(const GridTopology& topo, int L, const SgmRound& rd) {
  const size_t n = size_t(topo.grid().nodes());
  CostOutput<float> out;
  out.height = topo.grid().height;
  out.width = topo.grid().width;
  out.labels = L;
  out.cost.resize(n * L);
  out.labels_map.resize(n);
  rd.cost.download(out.cost.data(), out.cost.size());
  rd.labels.download(out.labels_map.data(), n);
  return out;
}

}  // namespace cuda_detail

/// baselines.hpp:31-98
template <class Real>
SgmResult<Real> sgm_forward(const GridTopology& topo, const PotentialSet<Real>& pots, SgmVariant variant,
                            int threads = 1) {
  cuda_detail::require_float<Real>();
  (void)threads;
  auto d = cuda_detail::upload(topo, pots, nullptr, false);
  const auto rd = cuda_detail::sgm_round(topo, d.prob, variant);
  SgmResult<float> res;
  res.output = cuda_detail::download_cost(topo, d.prob.labels, rd);
  res.messages.resize(size_t(topo.num_dirs()) * topo.grid().nodes() * d.prob.labels);
  rd.msg.download(res.messages.data(), res.messages.size());
  return res;
}

/// baselines.hpp:108-145: each round's unary volume is the previous round's
/// message sum, per-node minimum subtracted (mrf_sgm_next_unary_f32); the
/// volume stays on the device between rounds.
template <class Real>
class SgmIterative {
 public:
  SgmIterative(const GridTopology& topo, const PotentialSet<Real>& pots, SgmVariant variant = SgmVariant::standard,
               int threads = 1)
      : topo_(topo), d_((cuda_detail::require_float<Real>(), cuda_detail::upload(topo, pots, nullptr, false))),
        variant_(variant) {
    (void)threads;
  }

  const CostOutput<Real>& step() {
    const auto rd = cuda_detail::sgm_round(topo_, d_.prob, variant_);
    last_ = cuda_detail::download_cost(topo_, d_.prob.labels, rd);
    cuda_detail::DeviceBuffer next(sizeof(float) * size_t(topo_.grid().nodes()) * d_.prob.labels);
    cuda_detail::check(mrf_sgm_next_unary_f32(topo_.handle(), &d_.prob, rd.msg.as<float>(), next.as<float>(), nullptr));
    d_.unary = std::move(next);
    d_.prob.unary = d_.unary.as<float>();
    return last_;
  }

  const CostOutput<Real>& last() const { return last_; }

 private:
  const GridTopology& topo_;
  cuda_detail::DeviceProblem d_;
  SgmVariant variant_;
  CostOutput<Real> last_;
};

/// baselines.hpp:147-161
template <class Real>
std::vector<CostOutput<Real>> sgm_iterative(const GridTopology& topo, const PotentialSet<Real>& pots, int iterations,
                                            SgmVariant variant = SgmVariant::standard, int threads = 1) {
  if (iterations < 1) throw std::invalid_argument("sgm_iterative: iterations must be >= 1");
  SgmIterative<Real> it(topo, pots, variant, threads);
  std::vector<CostOutput<Real>> out;
  out.reserve(iterations);
  for (int k = 0; k < iterations; ++k) out.push_back(it.step());
  return out;
}

/// isgmr.hpp:156-169: energy of the aggregated labelling after each
/// iteration, optionally on a separate evaluation topology (the 4-connected
/// protocol).
template <class Real>
std::vector<double> isgmr_iterate_energy(const GridTopology& topo, const PotentialSet<Real>& pots, int iterations,
                                         int threads = 1, const GridTopology* eval_topo = nullptr) {
  const GridTopology& et = eval_topo ? *eval_topo : topo;
  IsgmrEngine<Real> engine(topo, pots, threads);
  std::vector<double> energies;
  energies.reserve(iterations > 0 ? iterations : 0);
  for (int k = 0; k < iterations; ++k) {
    engine.step();
    energies.push_back(energy(et, pots, engine.aggregate().labels_map));
  }
  return energies;
}

/// trwp.hpp:158-171
template <class Real>
std::vector<double> trwp_iterate_energy(const GridTopology& topo, const PotentialSet<Real>& pots,
                                        const TreeCoefficients<Real>& rho, int iterations, int threads = 1,
                                        const GridTopology* eval_topo = nullptr) {
  const GridTopology& et = eval_topo ? *eval_topo : topo;
  TrwpEngine<Real> engine(topo, pots, rho, threads);
  std::vector<double> energies;
  energies.reserve(iterations > 0 ? iterations : 0);
  for (int k = 0; k < iterations; ++k) {
    engine.step();
    energies.push_back(energy(et, pots, engine.aggregate().labels_map));
  }
  return energies;
}

}  // namespace mp
