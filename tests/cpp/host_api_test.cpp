// Drop-in C++ API test (include/mrf/mp_cuda.hpp): reference-style calls on
// the GPU compared bit-for-bit (forward) / within 1e-5 normwise (backward)
// with the C restatement (oracle/mrf_oracle.c, test infrastructure only).
// Mirrors test_isgmr.cpp / test_trwp.cpp / test_autodiff.cpp call shapes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <random>

#include "mrf/mp_cuda.hpp"
#include "mrf_oracle.h"

using namespace mp;

static int failures = 0;
#define CHECK(c)                                                     \
  do {                                                               \
    if (!(c)) {                                                      \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
      ++failures;                                                    \
    }                                                                \
  } while (0)

static double normwise(const std::vector<float>& a, const std::vector<float>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += double(a[i] - b[i]) * (a[i] - b[i]);
    den += double(b[i]) * b[i];
  }
  return den == 0 ? std::sqrt(num) : std::sqrt(num / den);
}

static void run_case(bool trwp, int H, int W, int L, int conn, int K, bool planes, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uu(0.0, 10.0), uv(0.0, 3.0), uw(0.1, 2.0);
  const GridTopology topo(GridGraph(H, W), DirectionSet::build(conn));
  PotentialSet<float> pots;
  pots.unary = UnaryVolume<float>(H, W, L);
  for (auto& v : pots.unary.values) v = float(uu(rng));
  std::vector<float> table(size_t(L) * L);
  for (auto& v : table) v = float(uv(rng));
  for (int l = 0; l < L; ++l) table[size_t(l) * L + l] = 0.f;
  pots.pairwise = explicit_pairwise(table, L);
  std::vector<std::vector<float>> pl(conn / 2, std::vector<float>(size_t(H) * W));
  if (planes) {
    for (auto& p : pl)
      for (auto& v : p) v = float(uw(rng));
    pots.weights = EdgeWeights<float>::planes(pl);
  } else {
    pots.weights = EdgeWeights<float>::constant(0.75f);
  }
  const auto rho = default_rho<float>(conn, 0.5f);
  const auto fwd = trwp ? trwp_forward(topo, pots, rho, K) : isgmr_forward(topo, pots, K);

  // oracle
  std::vector<float> flat;
  for (auto& p : pl) flat.insert(flat.end(), p.begin(), p.end());
  orc_problem pr{H, W, L, pots.unary.values.data(), table.data(), 0.75f, planes ? flat.data() : nullptr, 0.5f, nullptr};
  orc_topo* ot = orc_topo_create(H, W, conn);
  const size_t n = size_t(H) * W, E = size_t(orc_total_edges(ot));
  std::vector<float> cost(n * L), msg(size_t(conn) * n * L);
  std::vector<uint16_t> lab(n);
  std::vector<uint8_t> p(K * E * L), q(K * E);
  (trwp ? orc_trwp_forward : orc_isgmr_forward)(ot, &pr, K, cost.data(), lab.data(), msg.data(), p.data(), q.data());
  CHECK(std::memcmp(fwd.output.cost.data(), cost.data(), 4 * cost.size()) == 0);
  CHECK(fwd.output.labels_map == lab);
  CHECK(std::memcmp(fwd.messages.data(), msg.data(), 4 * msg.size()) == 0);
  CHECK(fwd.indices.p_data() == p);
  CHECK(fwd.indices.q_data() == q);
  CHECK(fwd.indices.bytes() == K * E * (L + 1));

  std::vector<float> gc(n * L);
  std::normal_distribution<double> nd;
  for (auto& v : gc) v = float(nd(rng));
  const auto g = trwp ? trwp_backward(topo, pots, rho, fwd.indices, gc) : isgmr_backward(topo, pots, fwd.indices, gc);
  std::vector<float> gu(n * L), gv(size_t(L) * L), gw((conn / 2) * n);
  (trwp ? orc_trwp_backward : orc_isgmr_backward)(ot, &pr, K, p.data(), q.data(), gc.data(), gu.data(), gv.data(),
                                                  gw.data());
  std::vector<float> gwd;
  for (auto& v : g.edge_weights) gwd.insert(gwd.end(), v.begin(), v.end());
  CHECK(normwise(g.unary, gu) < 1e-5);
  CHECK(normwise(g.pairwise, gv) < 1e-5);
  CHECK(normwise(gwd, gw) < 1e-5);
  orc_topo_free(ot);
}

// Engine classes (isgmr.hpp:26-68, trwp.hpp:25-68): step() K times; after
// every step the messages, the aggregated cost/labels and the indices so far
// equal the oracle's K=k+1 forward; take_indices() feeds the backward;
// *_iterate_energy (isgmr.hpp:156-169, trwp.hpp:158-171) equals the energy
// of the oracle's labelling after each iteration.
static void engine_case(bool trwp, int H, int W, int L, int conn, int K, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> uu(0.0, 10.0);
  const GridTopology topo(GridGraph(H, W), DirectionSet::build(conn));
  PotentialSet<float> pots;
  pots.unary = UnaryVolume<float>(H, W, L);
  for (auto& v : pots.unary.values) v = float(uu(rng));
  pots.pairwise = build_pairwise<float>(PairwiseKind::truncated_linear, {2.0, 1.0, 1.0}, L);
  pots.weights = EdgeWeights<float>::constant(1.25f);
  const auto rho = default_rho<float>(conn, 0.5f);
  orc_problem pr{H, W, L, pots.unary.values.data(), pots.pairwise.table.data(), 1.25f, nullptr, 0.5f, nullptr};
  orc_topo* ot = orc_topo_create(H, W, conn);
  const size_t n = size_t(H) * W, E = size_t(orc_total_edges(ot));
  std::optional<IsgmrEngine<float>> ie;
  std::optional<TrwpEngine<float>> te;
  if (trwp)
    te.emplace(topo, pots, rho, 4);
  else
    ie.emplace(topo, pots, 4);
  std::vector<double> energies;
  for (int k = 0; k < K; ++k) {
    if (trwp)
      te->step();
    else
      ie->step();
    const int kk = k + 1;
    std::vector<float> cost(n * L), msg(size_t(conn) * n * L);
    std::vector<uint16_t> lab(n);
    std::vector<uint8_t> p(kk * E * L), q(kk * E);
    (trwp ? orc_trwp_forward : orc_isgmr_forward)(ot, &pr, kk, cost.data(), lab.data(), msg.data(), p.data(), q.data());
    const auto agg = trwp ? te->aggregate() : ie->aggregate();
    const auto& m = trwp ? te->messages() : ie->messages();
    const auto& idx = trwp ? te->indices() : ie->indices();
    CHECK((trwp ? te->iterations() : ie->iterations()) == kk);
    CHECK(std::memcmp(m.data(), msg.data(), 4 * msg.size()) == 0);
    CHECK(std::memcmp(agg.cost.data(), cost.data(), 4 * cost.size()) == 0);
    CHECK(agg.labels_map == lab);
    CHECK(idx.iterations() == kk && idx.p_data() == p && idx.q_data() == q);
    CHECK(std::isinf(trwp ? te->min_argmin_gap() : ie->min_argmin_gap()));  // not tracked outside diagnostic mode
    energies.push_back(energy(topo, pots, lab));
  }
  IndexStore st = trwp ? te->take_indices() : ie->take_indices();
  CHECK(st.iterations() == K && st.bytes() == K * E * (L + 1));
  std::vector<float> gc(n * L, 1.0f / float(n * L));
  const auto g = trwp ? trwp_backward(topo, pots, rho, st, gc) : isgmr_backward(topo, pots, st, gc);
  std::vector<float> gu(n * L), gv(size_t(L) * L), gw((conn / 2) * n);
  (trwp ? orc_trwp_backward : orc_isgmr_backward)(ot, &pr, K, st.p_data().data(), st.q_data().data(), gc.data(),
                                                  gu.data(), gv.data(), gw.data());
  CHECK(normwise(g.unary, gu) < 1e-5);
  CHECK(normwise(g.pairwise, gv) < 1e-5);
  const auto it = trwp ? trwp_iterate_energy(topo, pots, rho, K) : isgmr_iterate_energy(topo, pots, K);
  CHECK(it.size() == energies.size());
  for (size_t k = 0; k < it.size() && k < energies.size(); ++k)
    CHECK(std::fabs(it[k] - energies[k]) <= 1e-9 * std::fabs(energies[k]));
  // diagnostic mode: same messages, a finite gap
  if (trwp) {
    TrwpEngine<float> d(topo, pots, rho, 1, true);
    for (int k = 0; k < K; ++k) d.step();
    CHECK(d.messages() == te->messages());
    CHECK(std::isfinite(d.min_argmin_gap()) && d.min_argmin_gap() >= 0.f);
  } else {
    IsgmrEngine<float> d(topo, pots, 1, true);
    for (int k = 0; k < K; ++k) d.step();
    CHECK(d.messages() == ie->messages());
    CHECK(std::isfinite(d.min_argmin_gap()) && d.min_argmin_gap() >= 0.f);
  }
  orc_topo_free(ot);
}

int main() {
  engine_case(false, 8, 11, 24, 4, 5, 11);  // 5 steps: the device index store regrows past capacity
  engine_case(true, 9, 7, 40, 4, 3, 12);
  engine_case(true, 6, 10, 7, 8, 4, 13);
  {
    // the engines reject non-finite unaries like the reference constructors
    PotentialSet<float> bad;
    bad.unary = UnaryVolume<float>(3, 3, 2);
    bad.unary.values[5] = std::nanf("");
    bad.pairwise = build_pairwise<float>(PairwiseKind::potts, {}, 2);
    const GridTopology t3(GridGraph(3, 3), DirectionSet::build(4));
    bool threw = false;
    try {
      TrwpEngine<float> e(t3, bad, default_rho<float>(4, 0.5f));
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  run_case(false, 7, 9, 5, 4, 3, true, 1);
  run_case(true, 7, 9, 5, 8, 3, true, 2);
  run_case(false, 9, 6, 16, 8, 2, false, 3);
  run_case(true, 5, 11, 33, 4, 2, false, 4);
  // topology parity with the reference accessors
  const GridTopology t(GridGraph(5, 7), DirectionSet::build(16));
  int64_t total = 0;
  for (int r = 0; r < 16; ++r) total += t.edge_count(r);
  CHECK(total == t.total_edges());
  // invalid inputs are rejected like the reference (test_isgmr.cpp:111-120)
  PotentialSet<float> bad;
  bad.unary = UnaryVolume<float>(2, 2, 2);
  bad.unary.values[0] = std::numeric_limits<float>::infinity();
  bad.pairwise = build_pairwise<float>(PairwiseKind::potts, {}, 2);
  const GridTopology t2(GridGraph(2, 2), DirectionSet::build(4));
  bool threw = false;
  try {
    isgmr_forward(t2, bad, 1);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  bad.unary.values[0] = 0.f;
  threw = false;
  try {
    isgmr_forward(t2, bad, 0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  // SGM baselines (baselines.hpp:31-161): revised == one ISGMR iteration
  // (test_baselines.cpp:58-68); iterated SGM's first round is sgm_forward's
  // and later rounds change the labelling's input (exact parity with the
  // reference library: tests/test_gpu_head.py)
  {
    const int H = 7, W = 8, L = 6;
    std::mt19937 rng(5);
    std::uniform_real_distribution<float> U(0.f, 6.f);
    PotentialSet<float> pots;
    pots.unary = UnaryVolume<float>(H, W, L);
    for (auto& v : pots.unary.values) v = U(rng);
    pots.pairwise = build_pairwise<float>(PairwiseKind::truncated_linear, {2.0, 1.0, 1.0}, L);
    const GridTopology t4(GridGraph(H, W), DirectionSet::build(4));
    const auto rev = sgm_forward(t4, pots, SgmVariant::revised);
    const auto one = isgmr_forward(t4, pots, 1);
    CHECK(rev.output.cost == one.output.cost && rev.messages == one.messages);
    const auto std1 = sgm_forward(t4, pots, SgmVariant::standard);
    const auto it = sgm_iterative(t4, pots, 3);
    CHECK(it.size() == 3 && it[0].cost == std1.output.cost && it[0].labels_map == std1.output.labels_map);
    CHECK(it[1].cost != it[0].cost);
    bool threw = false;
    try {
      sgm_iterative(t4, pots, 0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  // readout and evaluation (softhead.hpp:22-74, potentials.hpp:175-199)
  {
    const int H = 6, W = 7, L = 9;
    std::mt19937 rng(7);
    std::uniform_real_distribution<float> U(0.f, 8.f);
    CostOutput<float> c;
    c.height = H, c.width = W, c.labels = L;
    c.cost.resize(size_t(H) * W * L);
    for (auto& v : c.cost) v = U(rng);
    std::vector<float> target(size_t(H) * W);
    for (auto& v : target) v = U(rng);
    const auto head = soft_head_forward(c, target);
    const auto grad = soft_head_backward(c, head, target);
    std::vector<float> d_ref(target.size()), g_ref(c.cost.size());
    const float loss_ref = orc_soft_head(H * W, L, c.cost.data(), target.data(), d_ref.data(), g_ref.data());
    CHECK(std::fabs(head.loss - loss_ref) <= 1e-5f * std::fabs(loss_ref));
    CHECK(normwise(head.disparity, d_ref) <= 1e-5);
    CHECK(normwise(grad, g_ref) <= 1e-5);
    PotentialSet<float> pots;
    pots.unary = UnaryVolume<float>(H, W, L);
    for (auto& v : pots.unary.values) v = U(rng);
    pots.pairwise = build_pairwise<float>(PairwiseKind::potts, {}, L);
    const GridTopology t4(GridGraph(H, W), DirectionSet::build(4));
    std::vector<std::uint16_t> lab(size_t(H) * W);
    for (auto& x : lab) x = std::uint16_t(rng() % L);
    double want = 0.0;
    for (int i = 0; i < H * W; ++i) want += double(pots.unary.values[size_t(i) * L + lab[i]]);
    for (int h = 0; h < H; ++h)
      for (int w = 0; w < W; ++w) {
        if (w + 1 < W) want += (lab[h * W + w] != lab[h * W + w + 1]) ? 1.0 : 0.0;
        if (h + 1 < H) want += (lab[h * W + w] != lab[(h + 1) * W + w]) ? 1.0 : 0.0;
      }
    CHECK(std::fabs(energy(t4, pots, lab) - want) <= 1e-9 * std::fabs(want));
    lab[3] = std::uint16_t(L);
    bool oor = false;
    try {
      energy(t4, pots, lab);
    } catch (const std::out_of_range&) {
      oor = true;
    }
    CHECK(oor);
  }
  std::printf(failures ? "host_api_test: %d FAILURES\n" : "host_api_test: OK%.0d\n", failures);
  return failures ? 1 : 0;
}
