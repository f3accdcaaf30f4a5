// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (mrfmp, namespace mp)
// compiled from its own sources under /root/reference/proj by oracle/Makefile.
// The shim only marshals plain pointers into the reference's own types and
// calls the reference's public entry points:
//   mp::isgmr_forward   proj/include/mp/isgmr.hpp:145-152
//   mp::trwp_forward    proj/include/mp/trwp.hpp:148-156
//   mp::isgmr_backward  proj/include/mp/autodiff.hpp:63-126
//   mp::trwp_backward   proj/include/mp/autodiff.hpp:133-197
//   mp::soft_head_*     proj/include/mp/softhead.hpp:22-74
//   mp::GridTopology    proj/src/grid.cpp:96-114
// Everything mp:: stays hidden (-fvisibility=hidden); only ref_* is exported,
// so this .so can share a process with the product library.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "mp/autodiff.hpp"
#include "mp/grid.hpp"
#include "mp/isgmr.hpp"
#include "mp/potentials.hpp"
#include "mp/softhead.hpp"
#include "mp/trwp.hpp"
#include "mp/baselines.hpp"
#include "mp/gradcheck.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

mp::GridTopology make_topo(int H, int W, int conn) {
  return mp::GridTopology(mp::GridGraph(H, W), mp::DirectionSet::build(conn));
}

template <class Real>
mp::PotentialSet<Real> make_pots(int H, int W, int L, int R, const Real* unary, const Real* table,
                                 Real w_const, const Real* w_planes) {
  mp::PotentialSet<Real> pots;
  pots.unary = mp::UnaryVolume<Real>(H, W, L);
  std::memcpy(pots.unary.values.data(), unary, sizeof(Real) * size_t(H) * W * L);
  pots.pairwise = mp::explicit_pairwise(std::vector<Real>(table, table + size_t(L) * L), L);
  if (w_planes) {
    const size_t n = size_t(H) * W;
    std::vector<std::vector<Real>> planes(R / 2, std::vector<Real>(n));
    for (int f = 0; f < R / 2; ++f) std::memcpy(planes[f].data(), w_planes + f * n, sizeof(Real) * n);
    pots.weights = mp::EdgeWeights<Real>::planes(std::move(planes));
  } else {
    pots.weights = mp::EdgeWeights<Real>::constant(w_const);
  }
  return pots;
}

template <class Real>
mp::TreeCoefficients<Real> make_rho(int R, int n, Real uniform, const Real* planes) {
  mp::TreeCoefficients<Real> rho;
  rho.uniform = uniform;
  if (planes) {
    rho.planes.assign(R / 2, std::vector<Real>(n));
    for (int f = 0; f < R / 2; ++f) std::memcpy(rho.planes[f].data(), planes + size_t(f) * n, sizeof(Real) * n);
  }
  return rho;
}

template <class Real>
void export_forward(const mp::ForwardResult<Real>& res, Real* cost, uint16_t* labels, Real* messages,
                    uint8_t* p, uint8_t* q, Real* min_gap) {
  if (cost) std::memcpy(cost, res.output.cost.data(), sizeof(Real) * res.output.cost.size());
  if (labels) std::memcpy(labels, res.output.labels_map.data(), 2 * res.output.labels_map.size());
  if (messages) std::memcpy(messages, res.messages.data(), sizeof(Real) * res.messages.size());
  if (p) std::memcpy(p, res.indices.p_data().data(), res.indices.p_data().size());
  if (q) std::memcpy(q, res.indices.q_data().data(), res.indices.q_data().size());
  if (min_gap) *min_gap = res.min_argmin_gap;
}

// Rebuilds an IndexStore from flat p/q arrays in the reference layout
// (proj/include/mp/index_store.hpp:35-46).
mp::IndexStore make_store(const mp::GridTopology& topo, int L, int K, const uint8_t* p, const uint8_t* q) {
  mp::IndexStore st(topo, L);
  for (int k = 0; k < K; ++k) st.append_iteration();
  for (int k = 0; k < K; ++k)
    for (int r = 0; r < topo.num_dirs(); ++r)
      for (int64_t e = 0; e < topo.edge_count(r); ++e) {
        const size_t flat = size_t(k) * topo.total_edges() + topo.dir_offset(r) + e;
        std::memcpy(st.p_row(topo, k, r, int32_t(e)), p + flat * L, L);
        st.q_at(topo, k, r, int32_t(e)) = q[flat];
      }
  return st;
}

template <class Real>
void export_grads(const mp::GradientSet<Real>& g, Real* gu, Real* gv, Real* gw) {
  if (gu) std::memcpy(gu, g.unary.data(), sizeof(Real) * g.unary.size());
  if (gv) std::memcpy(gv, g.pairwise.data(), sizeof(Real) * g.pairwise.size());
  if (gw)
    for (size_t f = 0; f < g.edge_weights.size(); ++f)
      std::memcpy(gw + f * g.edge_weights[f].size(), g.edge_weights[f].data(),
                  sizeof(Real) * g.edge_weights[f].size());
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

/// Topology dump: total edges, per-direction edge counts / offsets, the dense
/// edge_index [R][N], and per-direction scanline (first node, length) lists
/// written into caller arrays of capacity `cap` per direction.
REF_API int ref_topology(int H, int W, int conn, int64_t* total_edges, int64_t* edge_count,
                         int64_t* dir_offset, int32_t* edge_index, int32_t* nlines,
                         int32_t* line_first, int32_t* line_len, int cap) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const int R = topo.num_dirs();
    const int n = H * W;
    *total_edges = topo.total_edges();
    for (int r = 0; r < R; ++r) {
      edge_count[r] = topo.edge_count(r);
      dir_offset[r] = topo.dir_offset(r);
      for (int i = 0; i < n; ++i) edge_index[size_t(r) * n + i] = topo.edge_index(r, i);
      const auto& lines = topo.scanlines(r);
      nlines[r] = int32_t(lines.size());
      for (size_t t = 0; t < lines.size() && int(t) < cap; ++t) {
        line_first[size_t(r) * cap + t] = lines[t].nodes.front();
        line_len[size_t(r) * cap + t] = int32_t(lines[t].nodes.size());
      }
    }
  });
}

/// Full node list of every scanline of direction r, concatenated.
REF_API int ref_scanline_nodes(int H, int W, int conn, int r, int32_t* nodes_out) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    size_t o = 0;
    for (const auto& sl : topo.scanlines(r))
      for (int32_t v : sl.nodes) nodes_out[o++] = v;
  });
}

REF_API int ref_isgmr_forward_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                  float w_const, const float* w_planes, int K, int threads, float* cost,
                                  uint16_t* labels, float* messages, uint8_t* p, uint8_t* q, float* min_gap) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    export_forward(mp::isgmr_forward(topo, pots, K, threads), cost, labels, messages, p, q, min_gap);
  });
}

REF_API int ref_trwp_forward_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                 float w_const, const float* w_planes, float rho_uniform,
                                 const float* rho_planes, int K, int threads, float* cost, uint16_t* labels,
                                 float* messages, uint8_t* p, uint8_t* q, float* min_gap) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto rho = make_rho<float>(conn, H * W, rho_uniform, rho_planes);
    export_forward(mp::trwp_forward(topo, pots, rho, K, threads), cost, labels, messages, p, q, min_gap);
  });
}

REF_API int ref_isgmr_backward_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                   float w_const, const float* w_planes, int K, const uint8_t* p,
                                   const uint8_t* q, const float* grad_cost, int threads, float* g_unary,
                                   float* g_pairwise, float* g_wplanes) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto st = make_store(topo, L, K, p, q);
    std::vector<float> gc(grad_cost, grad_cost + size_t(H) * W * L);
    export_grads(mp::isgmr_backward(topo, pots, st, gc, threads), g_unary, g_pairwise, g_wplanes);
  });
}

REF_API int ref_trwp_backward_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                  float w_const, const float* w_planes, float rho_uniform,
                                  const float* rho_planes, int K, const uint8_t* p, const uint8_t* q,
                                  const float* grad_cost, int threads, float* g_unary, float* g_pairwise,
                                  float* g_wplanes) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto rho = make_rho<float>(conn, H * W, rho_uniform, rho_planes);
    const auto st = make_store(topo, L, K, p, q);
    std::vector<float> gc(grad_cost, grad_cost + size_t(H) * W * L);
    export_grads(mp::trwp_backward(topo, pots, rho, st, gc, threads), g_unary, g_pairwise, g_wplanes);
  });
}

/// Reference soft readout head (softhead.hpp:22-74) on a float cost volume:
/// returns the loss and writes d loss / d cost.
REF_API int ref_soft_head_f32(int H, int W, int L, const float* cost, const float* target, float* loss,
                              float* disparity, float* grad_cost) {
  return guarded([&] {
    mp::CostOutput<float> c;
    c.height = H;
    c.width = W;
    c.labels = L;
    c.cost.assign(cost, cost + size_t(H) * W * L);
    std::vector<float> t(target, target + size_t(H) * W);
    const auto head = mp::soft_head_forward(c, t);
    if (loss) *loss = head.loss;
    if (disparity) std::memcpy(disparity, head.disparity.data(), sizeof(float) * head.disparity.size());
    if (grad_cost) {
      const auto g = mp::soft_head_backward(c, head, t);
      std::memcpy(grad_cost, g.data(), sizeof(float) * g.size());
    }
  });
}

/// Revised SGM (baselines.hpp:31-161), which the reference pins bit-for-bit to
/// one ISGMR iteration (tests/test_baselines.cpp:58-68).
REF_API int ref_sgm_revised_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                float w_const, const float* w_planes, float* cost, float* messages) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto res = mp::sgm_forward(topo, pots, mp::SgmVariant::revised, 1);
    if (cost) std::memcpy(cost, res.output.cost.data(), sizeof(float) * res.output.cost.size());
    if (messages) std::memcpy(messages, res.messages.data(), sizeof(float) * res.messages.size());
  });
}

/// Standard SGM (baselines.hpp:31-98, SgmVariant::standard): cost, labels, messages.
REF_API int ref_sgm_standard_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                 float w_const, const float* w_planes, float* cost, uint16_t* labels, float* messages) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto res = mp::sgm_forward(topo, pots, mp::SgmVariant::standard, 1);
    if (cost) std::memcpy(cost, res.output.cost.data(), sizeof(float) * res.output.cost.size());
    if (labels) std::memcpy(labels, res.output.labels_map.data(), sizeof(uint16_t) * res.output.labels_map.size());
    if (messages) std::memcpy(messages, res.messages.data(), sizeof(float) * res.messages.size());
  });
}

/// Iterated SGM (baselines.hpp:108-161): per round cost [K][N][L] and labels [K][N].
REF_API int ref_sgm_iterative_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                                  float w_const, const float* w_planes, int iterations, int variant, float* costs,
                                  uint16_t* labels) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    const auto out = mp::sgm_iterative(topo, pots, iterations,
                                       variant ? mp::SgmVariant::revised : mp::SgmVariant::standard, 1);
    const size_t nl = size_t(H) * W * L, n = size_t(H) * W;
    for (size_t k = 0; k < out.size(); ++k) {
      std::memcpy(costs + k * nl, out[k].cost.data(), sizeof(float) * nl);
      std::memcpy(labels + k * n, out[k].labels_map.data(), sizeof(uint16_t) * n);
    }
  });
}

/// Energy of a labelling (potentials.hpp:175-199), double accumulation.
REF_API int ref_energy_f32(int H, int W, int L, int conn, const float* unary, const float* table,
                           float w_const, const float* w_planes, const uint16_t* labels, double* out) {
  return guarded([&] {
    const auto topo = make_topo(H, W, conn);
    const auto pots = make_pots<float>(H, W, L, conn, unary, table, w_const, w_planes);
    std::vector<uint16_t> lab(labels, labels + size_t(H) * W);
    *out = mp::energy(topo, pots, lab);
  });
}

/// Double-precision finite-difference gradient check of the reference
/// (gradcheck.hpp:111-171); pins the backward semantics the oracle restates.
REF_API int ref_gradient_check(int H, int W, int L, int conn, int K, int trwp, int per_edge, uint64_t seed,
                               double* max_rel_err, uint64_t* components, uint64_t* skipped) {
  return guarded([&] {
    mp::GradCheckConfig cfg;
    cfg.height = H;
    cfg.width = W;
    cfg.labels = L;
    cfg.connectivity = conn;
    cfg.iterations = K;
    cfg.engine = trwp ? mp::Engine::trwp : mp::Engine::isgmr;
    cfg.per_edge_weights = per_edge != 0;
    cfg.seed = seed;
    const auto rep = mp::gradient_check(cfg);
    *max_rel_err = rep.max_rel_err;
    *components = rep.components;
    *skipped = rep.skipped_ties;
  });
}
