// libmrf_cuda.so: C-ABI entry points (include/mrf_cuda.h) over the sm_100a
// message-passing kernels. Host code here only validates, plans launches and
// owns the per-device topology upload; all arithmetic runs on the GPU.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mrf_cuda.h"
#include "common.cuh"
#include "launch.hpp"
#include "aggregate.cuh"
#include "topology.hpp"

using namespace mrf;

namespace {

thread_local std::string g_last_error;

struct MrfError : std::runtime_error {
  int code;
  MrfError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw MrfError(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(e == cudaErrorMemoryAllocation ? MRF_ENOMEM : MRF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MRF_OK;
  } catch (const MrfError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MRF_EINVAL;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return MRF_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MRF_ECUDA;
  }
}

constexpr int kBwdSlots = 592;  // 4 x 148 SMs: persistent backward CTAs per image

// Optional launch instrumentation: when enabled, every kernel launch is
// bracketed by CUDA events recorded on its own stream, so callers can read
// per-kernel-class device time for a region (bench.py's roofline).
struct Profiler {
  struct Rec {
    int cls;
    cudaEvent_t a, b;
  };
  std::mutex mu;
  bool on = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;

  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void recycle() {
    for (auto& r : recs) {
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    recs.clear();
  }
};
Profiler g_prof;

class ProfScope {
 public:
  ProfScope(cudaStream_t s, int cls) : s_(s), cls_(cls) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (!g_prof.on) return;
    a_ = g_prof.take();
    b_ = g_prof.take();
    cudaEventRecord(a_, s_);
  }
  ~ProfScope() {
    if (!a_) return;
    cudaEventRecord(b_, s_);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.recs.push_back({cls_, a_, b_});
  }

 private:
  cudaStream_t s_;
  int cls_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

}  // namespace

// Topology handle: host geometry plus lazily uploaded per-device line tables.
struct mrf_topology_s {
  Topology host;
  std::vector<LineDesc> all_lines;                 // ISGMR: every direction, longest first
  std::vector<std::vector<LineDesc>> dir_lines;    // per direction, longest first
  std::vector<size_t> dir_start;                   // offset of dir r's block in the upload
  std::vector<std::vector<LineDesc>> dir_lines_all;  // per direction incl. single-node lines (backward)
  std::vector<size_t> dir_all_start;
  std::vector<LineDesc> every_line;                // ISGMR backward: every direction incl. single nodes, longest first
  size_t every_start = 0;
  struct Dev {
    LineDesc* lines = nullptr;  // [all_lines | dir 0 | ... | dir R-1 | all-lines dir 0 | ... | every_line]
  };
  std::map<int, Dev> dev;
  std::mutex mu;

  mrf_topology_s(int H, int W, int conn) : host(H, W, conn) {
    dir_lines.resize(host.num_dirs());
    dir_lines_all.resize(host.num_dirs());
    for (int r = 0; r < host.num_dirs(); ++r) {
      for (const Line& l : host.lines(r)) {
        if (l.length >= 2) dir_lines[r].push_back({l.first, l.length, l.edge_base, r});
        dir_lines_all[r].push_back({l.first, l.length, l.edge_base, r});
      }
      std::stable_sort(dir_lines_all[r].begin(), dir_lines_all[r].end(),
                       [](const LineDesc& a, const LineDesc& b) { return a.length > b.length; });
      std::stable_sort(dir_lines[r].begin(), dir_lines[r].end(),
                       [](const LineDesc& a, const LineDesc& b) { return a.length > b.length; });
      all_lines.insert(all_lines.end(), dir_lines[r].begin(), dir_lines[r].end());
    }
    std::stable_sort(all_lines.begin(), all_lines.end(),
                     [](const LineDesc& a, const LineDesc& b) { return a.length > b.length; });
    size_t off = all_lines.size();
    for (int r = 0; r < host.num_dirs(); ++r) {
      dir_start.push_back(off);
      off += dir_lines[r].size();
    }
    for (int r = 0; r < host.num_dirs(); ++r) {
      dir_all_start.push_back(off);
      off += dir_lines_all[r].size();
      every_line.insert(every_line.end(), dir_lines_all[r].begin(), dir_lines_all[r].end());
    }
    std::stable_sort(every_line.begin(), every_line.end(),
                     [](const LineDesc& a, const LineDesc& b) { return a.length > b.length; });
    every_start = off;
  }

  ~mrf_topology_s() {
    for (auto& kv : dev) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(kv.first);
      cudaFree(kv.second.lines);
      cudaSetDevice(cur);
    }
  }

  const LineDesc* device_lines() {
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second.lines;
    std::vector<LineDesc> all(all_lines);
    for (auto& v : dir_lines) all.insert(all.end(), v.begin(), v.end());
    for (auto& v : dir_lines_all) all.insert(all.end(), v.begin(), v.end());
    all.insert(all.end(), every_line.begin(), every_line.end());
    Dev dv;
    cuda_check(cudaMalloc(&dv.lines, sizeof(LineDesc) * std::max<size_t>(1, all.size())), "cudaMalloc(lines)");
    cuda_check(cudaMemcpy(dv.lines, all.data(), sizeof(LineDesc) * all.size(), cudaMemcpyHostToDevice),
               "upload lines");
    dev[d] = dv;
    return dv.lines;
  }
};

namespace {

void validate_problem(mrf_topology_t topo, const mrf_problem_f32* pr) {
  if (!topo) fail(MRF_EINVAL, "null topology");
  if (!pr) fail(MRF_EINVAL, "null problem");
  if (pr->batch < 1) fail(MRF_EINVAL, "batch must be >= 1");
  if (pr->height != topo->host.height() || pr->width != topo->host.width())
    fail(MRF_EINVAL, "problem grid does not match topology");
  if (pr->labels < 1 || pr->labels > 256) fail(MRF_EINVAL, "label count must be in [1, 256]");
  if (!pr->unary || !pr->pairwise) fail(MRF_EINVAL, "null unary or pairwise");
  if (!pr->weight_planes && !(pr->weight >= 0.0f)) fail(MRF_EINVAL, "edge weight must be nonnegative");
}

// The reference engines reject non-finite unaries (isgmr.hpp:32-35,
// trwp.hpp:33-36). The scan is enqueued ahead of the sweeps and writes its
// verdict straight into mapped pinned host memory (no copy-engine operation:
// a 4-byte copy would queue behind the caller's bulk H2D / D2H copies on the
// copy engines and stall the compute stream); the host waits for it only
// after it has enqueued the whole forward, so the GPU never idles on the
// check. On MRF_EINVAL the outputs are unspecified (the reference produces
// none).
class FiniteCheck {
 public:
  FiniteCheck(const mrf_problem_f32* pr, int N, cudaStream_t s) {
    if (pr->assume_finite) return;
    State& st = state();
    *st.host = 1;  // no scan of this thread is in flight (every call waits for its own)
    cuda_check(launch_finite_scan(pr->unary, size_t(pr->batch) * N * pr->labels, st.dev, s), "finite scan");
    cuda_check(cudaEventRecord(st.done, s), "finite event");
    armed_ = true;
  }
  ~FiniteCheck() {  // an error path left the scan in flight: let it land before the flag is reused
    if (armed_) cudaEventSynchronize(state().done);
  }
  FiniteCheck(const FiniteCheck&) = delete;
  FiniteCheck& operator=(const FiniteCheck&) = delete;
  void finish(const char* who) {
    if (!armed_) return;
    armed_ = false;
    State& st = state();
    cuda_check(cudaEventSynchronize(st.done), "finite event");
    if (!*reinterpret_cast<volatile int*>(st.host)) fail(MRF_EINVAL, std::string(who) + ": non-finite unary potential");
  }

 private:
  struct State {  // per host thread and device: mapped pinned verdict and an event
    int* host = nullptr;
    int* dev = nullptr;  // device alias of host
    cudaEvent_t done = nullptr;
    State() = default;
    State(const State&) = delete;
    State& operator=(const State&) = delete;
    ~State() {  // thread exit (errors ignored: the context may already be gone)
      if (done) cudaEventDestroy(done);
      if (host) cudaFreeHost(host);
    }
  };
  static State& state() {
    thread_local std::map<int, State> states;
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    State& st = states[d];
    if (!st.host) {
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&st.host), sizeof(int), cudaHostAllocMapped), "cudaHostAlloc");
      cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&st.dev), st.host, 0), "cudaHostGetDevicePointer");
      cuda_check(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming), "cudaEventCreate");
    }
    return st;
  }
  bool armed_ = false;
};

void validate_rho(const mrf_problem_f32* pr) {
  if (!pr->rho_planes && !(pr->rho > 0.0f && pr->rho <= 1.0f)) fail(MRF_EINVAL, "rho must be in (0, 1]");
}

Geometry make_geometry(mrf_topology_t topo, const mrf_problem_f32* pr, int K_cap) {
  Geometry g{};
  g.N = topo->host.nodes();
  g.L = pr->labels;
  g.R = topo->host.num_dirs();
  g.W = topo->host.width();
  g.K_cap = K_cap;
  g.E = topo->host.total_edges();
  for (int r = 0; r < g.R; ++r) {
    g.dir_offset[r] = topo->host.dir_offset(r);
    g.node_step[r] = topo->host.node_step(r);
  }
  return g;
}

Potentials make_potentials(const mrf_problem_f32* pr) {
  return Potentials{pr->unary, pr->pairwise, pr->weight, pr->weight_planes, pr->rho, pr->rho_planes};
}

size_t messages_bytes(mrf_topology_t topo, const mrf_problem_f32* pr) {
  return sizeof(float) * size_t(pr->batch) * topo->host.num_dirs() * topo->host.nodes() * pr->labels;
}

int threads_for(int L) { return std::min(256, (L + 31) / 32 * 32); }

// Per-call device description of V (banded vs dense strategy), stream-ordered.
class PairDescHolder {
 public:
  PairDescHolder(const mrf_problem_f32* pr, int R, cudaStream_t s) : s_(s) {
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&d_), sizeof(PairDesc), s), "cudaMallocAsync(desc)");
    const int64_t planes = int64_t(pr->batch) * (R / 2) * pr->height * pr->width;
    ProfScope ps(s, MRF_KCLASS_AUX);
    analyze_pairwise_kernel<<<1, 1024, 0, s>>>(pr->pairwise, pr->labels, pr->weight, pr->weight_planes != nullptr, d_); note_launch();
    cuda_check(cudaGetLastError(), "analyze_pairwise launch");
    for (const float* pl : {pr->weight_planes, pr->rho_planes}) {
      if (!pl) continue;
      const int blocks = int(std::min<int64_t>(148 * 4, (planes + 255) / 256));
      scan_neg_zero_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(pl), planes, d_); note_launch();
      cuda_check(cudaGetLastError(), "scan_neg_zero launch");
    }
  }
  ~PairDescHolder() { cudaFreeAsync(d_, s_); }
  const PairDesc* get() const { return d_; }

 private:
  cudaStream_t s_;
  PairDesc* d_ = nullptr;
};

template <bool TRWP>
void launch_forward_sweep(const mrf_problem_f32* pr, const Geometry& g, const LineDesc* lines, int nlines,
                          const float* m_in, float* m_out, uint8_t* p, uint8_t* q, int k, const PairDesc* desc,
                          cudaStream_t stream, float* agg_cost = nullptr, uint16_t* agg_labels = nullptr,
                          int dir = -1) {
  if (nlines == 0) return;
  // The pairwise strategy is only known on the device (desc), so the banded
  // D == 2 specialisation and the generic kernel are both launched; each
  // returns at once when the other one owns the sweep.
  // Diagnostic mode (pr->diag_gap): only the generic kernel, dense, tracking gaps.
  const bool diag = pr->diag_gap != nullptr;
  const bool band2 = !diag && (g.R == 4 || g.R == 8);
  const bool small = !diag && fwd_small_applies(g.L, g.R);
  FwdArgs a{g, make_potentials(pr), lines, nlines, m_in, m_out, p, q, k, desc, band2 ? 1 : 0, band2 ? fwd_bandw_max() : 0,
            small ? 1 : 0, agg_cost, agg_labels, dir, pr->diag_gap};
  ProfScope ps(stream, MRF_KCLASS_FWD_SWEEP);
  if (band2) {
    cuda_check(TRWP ? launch_fwd_band2_trwp(a, pr->batch, stream) : launch_fwd_band2_isgmr(a, pr->batch, stream),
               "fwd_band2_kernel launch");
    cuda_check(launch_fwd_bandw(a, pr->batch, TRWP, stream), "fwd_bandw_kernel launch");
  }
  if (small) cuda_check(launch_fwd_small(a, pr->batch, TRWP, stream), "fwd_small_kernel launch");
  cuda_check(launch_fwd_generic(a, pr->batch, TRWP, stream), "fwd_warp_kernel launch");
}

// fused: bit 0 -- the banded D == 2 forward aggregated in its last sweep;
// bit 1 -- the dense small-L forward did (each only when it owned the call)
void launch_aggregate(const mrf_problem_f32* pr, int R, int N, const float* messages, float* cost, uint16_t* labels,
                      cudaStream_t stream, const PairDesc* desc = nullptr, int fused = 0) {
  if (!cost && !labels) return;
  const int64_t warps = int64_t(pr->batch) * N;
  const int per_block = 8;
  const int64_t blocks = std::min<int64_t>((warps + per_block - 1) / per_block, 148 * 16);
  ProfScope ps(stream, MRF_KCLASS_AGGREGATE);
  aggregate_kernel<<<unsigned(blocks), per_block * 32, 0, stream>>>(pr->batch, N, pr->labels, R, pr->unary, messages,
                                                                    cost, labels, desc, fused);
  note_launch();
  cuda_check(cudaGetLastError(), "aggregate_kernel launch");
}

void isgmr_step(mrf_topology_t topo, const mrf_problem_f32* pr, int k, int K_cap, const float* m_in, float* m_out,
                uint8_t* p, uint8_t* q, const PairDesc* desc, cudaStream_t stream) {
  const Geometry g = make_geometry(topo, pr, K_cap);
  const LineDesc* lines = topo->device_lines();
  launch_forward_sweep<false>(pr, g, lines, int(topo->all_lines.size()), m_in, m_out, p, q, k, desc, stream);
}

void trwp_step(mrf_topology_t topo, const mrf_problem_f32* pr, int k, int K_cap, float* m, uint8_t* p, uint8_t* q,
               const PairDesc* desc, cudaStream_t stream, float* agg_cost = nullptr, uint16_t* agg_labels = nullptr) {
  const Geometry g = make_geometry(topo, pr, K_cap);
  const LineDesc* lines = topo->device_lines();
  for (int r = 0; r < g.R; ++r)  // directions strictly sequential (trwp.hpp:50)
    launch_forward_sweep<true>(pr, g, lines + topo->dir_start[r], int(topo->dir_lines[r].size()), m, m, p, q, k, desc,
                               stream, r == g.R - 1 ? agg_cost : nullptr, r == g.R - 1 ? agg_labels : nullptr, r);
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

template <bool TRWP>
void launch_dtheta_acc(dim3 grid, cudaStream_t s, int R, int N, int L, const float* A, float rho, const float* rho_planes,
                       const Geometry& g, float* dtheta, const float* src) {
  if (R <= 4)
    dtheta_acc_kernel<TRWP, 4><<<grid, 256, 0, s>>>(R, N, L, A, rho, rho_planes, g, dtheta, src);
  else if (R <= 8)
    dtheta_acc_kernel<TRWP, 8><<<grid, 256, 0, s>>>(R, N, L, A, rho, rho_planes, g, dtheta, src);
  else
    dtheta_acc_kernel<TRWP, 16><<<grid, 256, 0, s>>>(R, N, L, A, rho, rho_planes, g, dtheta, src);
  note_launch();
}

// the most lines one backward launch sweeps: TRWP one direction, ISGMR all
int bwd_max_lines(mrf_topology_t topo, bool trwp) {
  size_t m = topo->every_line.size();
  if (trwp) {
    m = 0;
    for (const auto& v : topo->dir_lines_all) m = std::max(m, v.size());
  }
  return int(m);
}

int dv_slots(mrf_topology_t topo, const mrf_problem_f32* pr, bool trwp) {
  return dv_slots_for(pr->labels, bwd_max_lines(topo, trwp));
}

size_t gvacc_bytes(mrf_topology_t topo, const mrf_problem_f32* pr, bool trwp) {
  return sizeof(float) * size_t(pr->batch) * dv_slots(topo, pr, trwp) * pr->labels * pr->labels;
}

size_t dwr_bytes(const mrf_problem_f32* pr, int R, int N) { return sizeof(float) * size_t(pr->batch) * R * N; }

// Backward (autodiff.hpp:63-197) over per-direction scatter planes A
// (bwd_common.cuh, bwd_split.cuh): TRWP replays directions R-1..0 per iteration, one launch
// each (directions are sequential, :147); ISGMR's directions only read the
// previous iteration's planes, so one launch covers all of them. After each
// iteration the unary gradient collects every sweep's contribution.
template <bool TRWP>
void run_backward(mrf_topology_t topo, const mrf_problem_f32* pr, int K, const uint8_t* p, const uint8_t* q,
                  const float* grad_cost, const mrf_grads_f32* grads, void* ws, size_t ws_bytes,
                  cudaStream_t stream) {
  const int R = topo->host.num_dirs(), N = topo->host.nodes(), L = pr->labels, B = pr->batch;
  const size_t mb = messages_bytes(topo, pr), vb = gvacc_bytes(topo, pr, TRWP);
  const int nslots = dv_slots(topo, pr, TRWP);
  const bool isgmr_dw = !TRWP && grads->weight_planes;
  const size_t need = align_up(mb) * (TRWP ? 1 : 2) + align_up(vb) + (TRWP ? 0 : align_up(dwr_bytes(pr, R, N)));
  if (ws_bytes < need || (!ws && need)) fail(MRF_EINVAL, "backward workspace too small");
  if (int64_t(R) * N * L >= (int64_t(1) << 31) || int64_t(K) * topo->host.total_edges() * L >= (int64_t(1) << 32))
    fail(MRF_EINVAL, "backward: image too large (R*N*L must be < 2^31 and K*E*L < 2^32)");
  // edge indices over the whole batch are 32-bit in the backward kernels
  if (int64_t(B) * K * topo->host.total_edges() >= (int64_t(1) << 32))
    fail(MRF_EINVAL, "backward: batch too large for one call (B*K*E must be < 2^32)");
  char* w = static_cast<char*>(ws);
  float* A[2] = {reinterpret_cast<float*>(w), TRWP ? nullptr : reinterpret_cast<float*>(w + align_up(mb))};
  float* gvacc = reinterpret_cast<float*>(w + align_up(mb) * (TRWP ? 1 : 2));
  float* dwr = TRWP ? nullptr : reinterpret_cast<float*>(w + align_up(mb) * 2 + align_up(vb));
  const size_t NL = size_t(N) * L;

  // make_gradients (autodiff.hpp:33-44): dtheta <- dc, dV <- 0, dw <- 0
  if (grads->weight_planes)
    cuda_check(cudaMemsetAsync(grads->weight_planes, 0, sizeof(float) * B * (R / 2) * N, stream), "zero dw");
  if (isgmr_dw) cuda_check(cudaMemsetAsync(dwr, 0, dwr_bytes(pr, R, N), stream), "zero dw partials");
  cuda_check(cudaMemsetAsync(gvacc, 0, vb, stream), "zero dV accumulators");
  // dtheta <- dc is not copied: the first unary-gradient update reads dc
  // directly (a device-to-device copy would also queue on a copy engine
  // behind the caller's host transfers)
  const float* dt_src = grad_cost;

  const Geometry g = make_geometry(topo, pr, K);
  const Potentials pot = make_potentials(pr);
  const LineDesc* lines = topo->device_lines();
  PairDescHolder desc(pr, R, stream);
  const dim3 dt_grid(unsigned(std::min<int64_t>(148 * 8 / B + 1, (int64_t(NL) / 4 + 255) / 256)), unsigned(B));
  for (int k = K - 1; k >= 0; --k) {
    float* ain = TRWP ? A[0] : A[(k + 1) & 1];
    float* aout = TRWP ? A[0] : A[k & 1];
    if (TRWP) {
      // the warp-specialised kernel's last sweep of the iteration also collects
      // the iteration's unary gradient; the one-warp-per-line kernel leaves it
      // to dtheta_acc_kernel
      const int lines0 = int(topo->dir_lines_all[0].size());
      const bool fuse = !bwd_uses_small(L, lines0, B) || bwd_small_fuse() ||
                        (bwd_uses_grp(L, R, pr->rho_planes != nullptr, lines0, B) && bwd_grp_fuse());
      for (int r = R - 1; r >= 0; --r) {  // directions in reverse (autodiff.hpp:147)
        AccArgs a{g, pot, lines + topo->dir_all_start[r], int(topo->dir_lines_all[r].size()), p, q, k, grad_cost,
                  ain, aout, grads->weight_planes, gvacc, nslots, desc.get(),
                  (r == 0 && fuse) ? grads->unary : nullptr, dt_src};
        ProfScope ps(stream, MRF_KCLASS_BWD_SWEEP);
        cuda_check(launch_bwd_trwp(a, B, stream), "bwd_split_kernel launch");
        if (r == 0 && fuse) dt_src = grads->unary;
      }
      if (!fuse) {
        ProfScope ps(stream, MRF_KCLASS_AUX);
        launch_dtheta_acc<TRWP>(dt_grid, stream, R, N, L, aout, pr->rho, pr->rho_planes, g, grads->unary, dt_src);
        dt_src = grads->unary;
        cuda_check(cudaGetLastError(), "dtheta_acc launch");
      }
    } else {
      {
        AccArgs a{g, pot, lines + topo->every_start, int(topo->every_line.size()), p, q, k, grad_cost,
                  ain, aout, isgmr_dw ? dwr : nullptr, gvacc, nslots, desc.get(), nullptr, nullptr};
        ProfScope ps(stream, MRF_KCLASS_BWD_SWEEP);
        cuda_check(launch_bwd_isgmr(a, B, stream), "bwd_split_kernel launch");
      }
      // ISGMR's directions run concurrently: the unary gradient is collected after the launch
      ProfScope ps(stream, MRF_KCLASS_AUX);
      launch_dtheta_acc<TRWP>(dt_grid, stream, R, N, L, aout, pr->rho, nullptr, g, grads->unary, dt_src);
      dt_src = grads->unary;
      cuda_check(cudaGetLastError(), "dtheta_acc launch");
    }
  }
  if (isgmr_dw) {
    ProfScope ps(stream, MRF_KCLASS_AUX);
    combine_dw_kernel<<<int(std::min<int64_t>(148 * 4, (int64_t(B) * (R / 2) * N + 255) / 256)), 256, 0, stream>>>(
        B, R, N, dwr, grads->weight_planes); note_launch();
    cuda_check(cudaGetLastError(), "combine_dw launch");
  }
  if (grads->pairwise) {
    const int64_t total = int64_t(B) * L * L;
    ProfScope ps(stream, MRF_KCLASS_AUX);
    reduce_gvacc_kernel<<<unsigned((total + 255) / 256), 256, 0, stream>>>(B, L, nslots, nslots, gvacc,
                                                                           grads->pairwise); note_launch();
    cuda_check(cudaGetLastError(), "reduce_gvacc launch");
  }
}

}  // namespace

extern "C" {

const char* mrf_last_error(void) { return g_last_error.c_str(); }
// 2.0.0: mrf_problem_f32 gained assume_finite and diag_gap (round 2)
int mrf_version(void) { return 20000; }

int mrf_topology_create(int height, int width, int connectivity, mrf_topology_t* out) {
  return guarded([&] {
    if (!out) fail(MRF_EINVAL, "null out");
    *out = new mrf_topology_s(height, width, connectivity);
  });
}

int mrf_topology_destroy(mrf_topology_t topo) {
  return guarded([&] { delete topo; });
}

int mrf_topology_info(mrf_topology_t topo, int* num_dirs, int64_t* total_edges, int64_t* edge_count,
                      int64_t* dir_offset) {
  return guarded([&] {
    if (!topo) fail(MRF_EINVAL, "null topology");
    if (num_dirs) *num_dirs = topo->host.num_dirs();
    if (total_edges) *total_edges = topo->host.total_edges();
    for (int r = 0; r < topo->host.num_dirs(); ++r) {
      if (edge_count) edge_count[r] = topo->host.edge_count(r);
      if (dir_offset) dir_offset[r] = topo->host.dir_offset(r);
    }
  });
}

int mrf_topology_edge_index(mrf_topology_t topo, int32_t* out) {
  return guarded([&] {
    if (!topo || !out) fail(MRF_EINVAL, "null argument");
    const auto v = topo->host.edge_index();
    std::memcpy(out, v.data(), sizeof(int32_t) * v.size());
  });
}

int mrf_topology_scanlines(mrf_topology_t topo, int r, int32_t* first, int32_t* length, int32_t* count, int cap) {
  return guarded([&] {
    if (!topo || r < 0 || r >= topo->host.num_dirs()) fail(MRF_EINVAL, "bad topology or direction");
    const auto& ls = topo->host.lines(r);
    if (count) *count = int32_t(ls.size());
    for (int t = 0; t < int(ls.size()) && t < cap; ++t) {
      if (first) first[t] = ls[t].first;
      if (length) length[t] = ls[t].length;
    }
  });
}

int mrf_check_finite_f32(const float* data, size_t count, int* all_finite, cudaStream_t stream);

size_t mrf_forward_workspace_bytes(mrf_topology_t topo, const mrf_problem_f32* prob, int engine, int iterations) {
  (void)iterations;
  if (!topo || !prob) return 0;
  return engine == MRF_ENGINE_ISGMR ? align_up(messages_bytes(topo, prob)) : 0;
}

int mrf_isgmr_forward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const mrf_forward_out* out,
                          void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (iterations < 1) fail(MRF_EINVAL, "isgmr_forward: iterations must be >= 1");
    if (!out || !out->messages || !out->p || !out->q) fail(MRF_EINVAL, "null forward output");
    FiniteCheck finite(prob, topo->host.nodes(), stream);
    const size_t mb = messages_bytes(topo, prob);
    if (!workspace || workspace_bytes < mb) fail(MRF_EINVAL, "forward workspace too small");
    float* bufs[2] = {out->messages, static_cast<float*>(workspace)};
    cuda_check(cudaMemsetAsync(bufs[0], 0, mb, stream), "zero m");
    cuda_check(cudaMemsetAsync(bufs[1], 0, mb, stream), "zero mhat");
    // Iteration k writes bufs[(K-1-k)&1] so the last one lands in out->messages;
    // the publish m <- mhat (isgmr.hpp:55) is the buffer swap.
    PairDescHolder desc(prob, topo->host.num_dirs(), stream);
    for (int k = 0; k < iterations; ++k) {
      float* dst = bufs[(iterations - 1 - k) & 1];
      const float* src = bufs[(iterations - k) & 1];
      isgmr_step(topo, prob, k, iterations, src, dst, out->p, out->q, desc.get(), stream);
    }
    launch_aggregate(prob, topo->host.num_dirs(), topo->host.nodes(), out->messages, out->cost, out->labels, stream);
    finite.finish("isgmr_forward");
  });
}

int mrf_trwp_forward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const mrf_forward_out* out,
                         void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  (void)workspace;
  (void)workspace_bytes;
  return guarded([&] {
    validate_problem(topo, prob);
    validate_rho(prob);
    if (iterations < 1) fail(MRF_EINVAL, "trwp_forward: iterations must be >= 1");
    if (!out || !out->messages || !out->p || !out->q) fail(MRF_EINVAL, "null forward output");
    FiniteCheck finite(prob, topo->host.nodes(), stream);
    cuda_check(cudaMemsetAsync(out->messages, 0, messages_bytes(topo, prob), stream), "zero m");
    PairDescHolder desc(prob, topo->host.num_dirs(), stream);
    // 4 directions: the last sweep's banded D == 2 kernel aggregates on the
    // fly (every node is a prev or the tail of one of its lines). Direction 3
    // runs along columns, so this needs H >= 2: with H == 1 it has no line of
    // two nodes and never launches.
    const bool fuse = topo->host.num_dirs() == 4 && topo->host.height() >= 2 && !prob->diag_gap &&
                      (out->cost || out->labels);
    for (int k = 0; k < iterations; ++k) {
      const bool last = fuse && k == iterations - 1;
      trwp_step(topo, prob, k, iterations, out->messages, out->p, out->q, desc.get(), stream,
                last ? out->cost : nullptr, last ? out->labels : nullptr);
    }
    const int fused = fuse ? (1 | (fwd_small_applies(prob->labels, topo->host.num_dirs()) ? 2 : 0)) : 0;
    launch_aggregate(prob, topo->host.num_dirs(), topo->host.nodes(), out->messages, out->cost, out->labels, stream,
                     desc.get(), fused);
    finite.finish("trwp_forward");
  });
}

int mrf_isgmr_step_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int k, int K_cap, const float* m_in,
                       float* m_out, uint8_t* p, uint8_t* q, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (k < 0 || k >= K_cap) fail(MRF_EINVAL, "iteration index out of range");
    if (!m_in || !m_out || !p || !q || m_in == m_out) fail(MRF_EINVAL, "bad step buffers");
    PairDescHolder desc(prob, topo->host.num_dirs(), stream);
    isgmr_step(topo, prob, k, K_cap, m_in, m_out, p, q, desc.get(), stream);
  });
}

int mrf_trwp_step_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int k, int K_cap, float* messages, uint8_t* p,
                      uint8_t* q, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    validate_rho(prob);
    if (k < 0 || k >= K_cap) fail(MRF_EINVAL, "iteration index out of range");
    if (!messages || !p || !q) fail(MRF_EINVAL, "bad step buffers");
    PairDescHolder desc(prob, topo->host.num_dirs(), stream);
    trwp_step(topo, prob, k, K_cap, messages, p, q, desc.get(), stream);
  });
}

int mrf_aggregate_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const float* messages, float* cost,
                      uint16_t* labels, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (!messages) fail(MRF_EINVAL, "null messages");
    launch_aggregate(prob, topo->host.num_dirs(), topo->host.nodes(), messages, cost, labels, stream);
  });
}

size_t mrf_backward_workspace_bytes(mrf_topology_t topo, const mrf_problem_f32* prob, int engine, int iterations) {
  (void)iterations;
  if (!topo || !prob) return 0;
  const size_t mb = align_up(messages_bytes(topo, prob));
  if (engine == MRF_ENGINE_ISGMR)
    return mb * 2 + align_up(gvacc_bytes(topo, prob, false)) +
           align_up(dwr_bytes(prob, topo->host.num_dirs(), topo->host.nodes()));
  return mb + align_up(gvacc_bytes(topo, prob, true));
}

int mrf_isgmr_backward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const uint8_t* p,
                           const uint8_t* q, const float* grad_cost, const mrf_grads_f32* grads, void* workspace,
                           size_t workspace_bytes, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (iterations < 1) fail(MRF_EINVAL, "backward: iterations must be >= 1");
    if (!p || !q || !grad_cost || !grads || !grads->unary) fail(MRF_EINVAL, "null backward argument");
    run_backward<false>(topo, prob, iterations, p, q, grad_cost, grads, workspace, workspace_bytes, stream);
  });
}

int mrf_trwp_backward_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int iterations, const uint8_t* p,
                          const uint8_t* q, const float* grad_cost, const mrf_grads_f32* grads, void* workspace,
                          size_t workspace_bytes, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    validate_rho(prob);
    if (iterations < 1) fail(MRF_EINVAL, "backward: iterations must be >= 1");
    if (!p || !q || !grad_cost || !grads || !grads->unary) fail(MRF_EINVAL, "null backward argument");
    run_backward<true>(topo, prob, iterations, p, q, grad_cost, grads, workspace, workspace_bytes, stream);
  });
}

int mrf_soft_head_f32(int batch, int nodes, int labels, const float* cost, const float* target, float* confidence,
                      float* disparity, float* grad_cost, float* loss, cudaStream_t stream) {
  return guarded([&] {
    if (batch < 1 || nodes < 1 || labels < 1) fail(MRF_EINVAL, "soft_head: empty volume");
    if (!cost || !target || !loss) fail(MRF_EINVAL, "soft_head: null cost, target or loss");
    const int nblk = soft_head_blocks(nodes);
    double* partial = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&partial), sizeof(double) * batch * nblk, stream),
               "cudaMallocAsync(soft head partials)");
    ProfScope ps(stream, MRF_KCLASS_AUX);
    cuda_check(launch_soft_head(batch, nodes, labels, cost, target, confidence, disparity, grad_cost, loss, partial,
                                nblk, stream),
               "soft_head launch");
    cuda_check(cudaFreeAsync(partial, stream), "cudaFreeAsync");
  });
}

int mrf_energy_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const uint16_t* labels, double* energy,
                   cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (!labels || !energy) fail(MRF_EINVAL, "energy: null labels or output");
    const int B = prob->batch, H = topo->host.height(), W = topo->host.width(), R = topo->host.num_dirs();
    EvenSteps st{};
    for (int r = 0; r < R; r += 2) st.dh[r >> 1] = direction_step(r).dh, st.dw[r >> 1] = direction_step(r).dw;
    const int nblk = energy_blocks(H * W);
    double* partial = nullptr;
    double* out = nullptr;
    int* bad = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&partial), sizeof(double) * (size_t(B) * nblk + B) + 16, stream),
               "cudaMallocAsync(energy)");
    out = partial + size_t(B) * nblk;
    bad = reinterpret_cast<int*>(out + B);
    cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), stream), "zero flag");
    {
      ProfScope ps(stream, MRF_KCLASS_AUX);
      cuda_check(launch_energy(B, H, W, prob->labels, R, st, prob->unary, prob->pairwise, prob->weight,
                               prob->weight_planes, labels, out, partial, nblk, bad, stream),
                 "energy launch");
    }
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(energy, out, sizeof(double) * B, cudaMemcpyDeviceToHost, stream), "energy D2H");
    cuda_check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream), "flag D2H");
    cuda_check(cudaFreeAsync(partial, stream), "cudaFreeAsync");
    cuda_check(cudaStreamSynchronize(stream), "energy sync");
    if (hbad) fail(MRF_EINVAL, "energy: label out of range");
  });
}

int mrf_sgm_f32(mrf_topology_t topo, const mrf_problem_f32* prob, int variant, float* messages, float* cost,
                uint16_t* labels, cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (!messages) fail(MRF_EINVAL, "sgm_forward: null messages");
    const int R = topo->host.num_dirs(), N = topo->host.nodes();
    if (variant == 1) {  // revised == one ISGMR iteration
      const size_t E = size_t(prob->batch) * topo->host.total_edges();
      uint8_t* pq = nullptr;
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&pq), E * (prob->labels + 1), stream), "cudaMallocAsync(p, q)");
      float* other = nullptr;
      const size_t mb = messages_bytes(topo, prob);
      cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&other), mb, stream), "cudaMallocAsync(mhat)");
      cuda_check(cudaMemsetAsync(other, 0, mb, stream), "zero m");
      cuda_check(cudaMemsetAsync(messages, 0, mb, stream), "zero mhat");
      PairDescHolder desc(prob, R, stream);
      isgmr_step(topo, prob, 0, 1, other, messages, pq, pq + E * prob->labels, desc.get(), stream);
      launch_aggregate(prob, R, N, messages, cost, labels, stream);
      cuda_check(cudaFreeAsync(other, stream), "cudaFreeAsync");
      cuda_check(cudaFreeAsync(pq, stream), "cudaFreeAsync");
    } else if (variant == 0) {
      const Geometry g = make_geometry(topo, prob, 1);
      {
        ProfScope ps(stream, MRF_KCLASS_FWD_SWEEP);
        cuda_check(launch_sgm_standard(g, make_potentials(prob), topo->device_lines() + topo->every_start,
                                       int(topo->every_line.size()), messages, prob->batch, stream),
                   "sgm_standard launch");
      }
      if (cost || labels) {
        mrf_problem_f32 p2 = *prob;
        p2.unary = nullptr;  // cost = sum_r m^r (baselines.hpp:84-93)
        launch_aggregate(&p2, R, N, messages, cost, labels, stream);
      }
    } else {
      fail(MRF_EINVAL, "sgm_forward: unknown variant");
    }
  });
}

int mrf_sgm_next_unary_f32(mrf_topology_t topo, const mrf_problem_f32* prob, const float* messages, float* next_unary,
                           cudaStream_t stream) {
  return guarded([&] {
    validate_problem(topo, prob);
    if (!messages || !next_unary) fail(MRF_EINVAL, "sgm_next_unary: null messages or output");
    ProfScope ps(stream, MRF_KCLASS_AUX);
    cuda_check(launch_sgm_next_unary(prob->batch, topo->host.nodes(), prob->labels, topo->host.num_dirs(), messages,
                                     next_unary, stream),
               "sgm_next_unary launch");
  });
}

int mrf_profiler_enable(int on) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.recycle();
    g_prof.on = on != 0;
  });
}

int mrf_profiler_read(int kernel_class, double* total_ms, int64_t* launches) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    double t = 0.0;
    int64_t n = 0;
    for (const auto& r : g_prof.recs) {
      if (r.cls != kernel_class) continue;
      cuda_check(cudaEventSynchronize(r.b), "profiler sync");
      float ms = 0.0f;
      cuda_check(cudaEventElapsedTime(&ms, r.a, r.b), "profiler elapsed");
      t += ms;
      ++n;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = n;
  });
}

}  // extern "C"
