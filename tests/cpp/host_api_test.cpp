// Drop-in C++ API test (include/mrf/mp_cuda.hpp): reference-style calls on
// the GPU compared bit-for-bit (forward) / within 1e-5 normwise (backward)
// with the C restatement (oracle/mrf_oracle.c, test infrastructure only).
// Mirrors test_isgmr.cpp / test_trwp.cpp / test_autodiff.cpp call shapes.
#include <cmath>
#include <cstdio>
#include <cstring>
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

int main() {
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
  std::printf(failures ? "host_api_test: %d FAILURES\n" : "host_api_test: OK%.0d\n", failures);
  return failures ? 1 : 0;
}
