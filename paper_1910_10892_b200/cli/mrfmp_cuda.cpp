// mrfmp_cuda: the reference CLI's `run` driver (proj/tools/mrfmp.cpp:77-166)
// on the B200 path. Same options, inputs, outputs and stdout line:
//
//   mrfmp_cuda run [--method sgm|sgm-std|isgmr|trwp] [--dirs 4|8|16] [--iters K]
//                  [--pairwise potts|tl|tq|p1p2] [--trunc T] [--p1 P] [--p2 P]
//                  [--rho R] [--max-disp L] [--unary-file F.mpcv | --left L.pgm
//                  --right R.pgm | --image I.pgm] [--seed S] [--height H]
//                  [--width W] [--weight w] [--out-csv run.csv]
//                  [--out-labels labels.pgm] [--timing-repeats N]
//                  [--threads T] [--precision f32]
//
// Unaries: an MPCV1 cost volume, stereo |left - right| from two PGMs, the
// denoising data term of a noisy PGM, or a seeded U[0, 8) synthetic volume.
// Each iteration is an engine step on the GPU; the energy of its labelling
// on the 4-connected edge set and the step's wall time go to the CSV
// (mrfmp.cpp:91-101). Not carried over: `--method mf` (the mean-field
// baseline is not on the path) and `--precision f64` (the GPU path is FP32;
// the reference's double build stays a CPU tool).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "mrf/io.hpp"
#include "mrf/mp_cuda.hpp"

namespace {

struct RunOpts {
  std::string method = "isgmr";
  int dirs = 4;
  int iters = 5;
  std::string pairwise = "potts";
  double trunc = -1.0;
  double p1 = 1.0, p2 = 1.0;
  double rho = 0.5;
  int max_disp = 8;
  std::string unary_file, left_file, right_file, image_file;
  std::uint64_t seed = 0;
  int threads = 1;
  std::string precision = "f32";
  int height = 32, width = 32;
  double weight = 1.0;
  std::string out_csv = "run.csv";
  std::string out_labels = "labels.pgm";
  int timing_repeats = 0;
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

mp::PairwiseKind parse_pairwise(const std::string& name) {
  static const std::map<std::string, mp::PairwiseKind> kinds = {{"potts", mp::PairwiseKind::potts},
                                                                {"tl", mp::PairwiseKind::truncated_linear},
                                                                {"tq", mp::PairwiseKind::truncated_quadratic},
                                                                {"p1p2", mp::PairwiseKind::sgm_p1p2}};
  const auto it = kinds.find(name);
  if (it == kinds.end()) throw UsageError("--pairwise: unknown pairwise '" + name + "'");
  return it->second;
}

RunOpts parse(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) != "run") throw UsageError("usage: mrfmp_cuda run [options]");
  RunOpts o;
  std::map<std::string, std::string*> strs = {{"--method", &o.method},         {"--pairwise", &o.pairwise},
                                              {"--unary-file", &o.unary_file}, {"--left", &o.left_file},
                                              {"--right", &o.right_file},      {"--image", &o.image_file},
                                              {"--precision", &o.precision},   {"--out-csv", &o.out_csv},
                                              {"--out-labels", &o.out_labels}};
  std::map<std::string, int*> ints = {{"--dirs", &o.dirs},       {"--iters", &o.iters},   {"--max-disp", &o.max_disp},
                                      {"--threads", &o.threads}, {"--height", &o.height}, {"--width", &o.width},
                                      {"--timing-repeats", &o.timing_repeats}};
  std::map<std::string, double*> dbls = {{"--trunc", &o.trunc}, {"--p1", &o.p1},   {"--p2", &o.p2},
                                         {"--rho", &o.rho},     {"--weight", &o.weight}};
  for (int i = 2; i < argc; ++i) {
    const std::string key = argv[i];
    if (i + 1 >= argc) throw UsageError(key + ": missing value");
    const std::string val = argv[++i];
    try {
      if (strs.count(key)) {
        *strs[key] = val;
      } else if (ints.count(key)) {
        std::size_t used = 0;
        *ints[key] = std::stoi(val, &used);
        if (used != val.size()) throw std::invalid_argument(val);
      } else if (dbls.count(key)) {
        std::size_t used = 0;
        *dbls[key] = std::stod(val, &used);
        if (used != val.size()) throw std::invalid_argument(val);
      } else if (key == "--seed") {
        o.seed = std::stoull(val);
      } else {
        throw UsageError("unknown option " + key);
      }
    } catch (const UsageError&) {
      throw;
    } catch (const std::exception&) {
      throw UsageError(key + ": bad value '" + val + "'");
    }
  }
  if (o.iters < 1) throw UsageError("--iters: must be positive");
  if (o.precision != "f32") throw UsageError("--precision: the GPU path computes in f32");
  return o;
}

mp::UnaryVolume<float> make_unaries(const RunOpts& o) {
  if (!o.unary_file.empty()) return mp::load_cost_volume<float>(o.unary_file);
  if (!o.left_file.empty() || !o.right_file.empty()) {
    if (o.left_file.empty() || o.right_file.empty()) throw UsageError("--left/--right: both stereo images are required");
    return mp::stereo_unaries<float>(mp::load_pgm(o.left_file), mp::load_pgm(o.right_file), o.max_disp);
  }
  if (!o.image_file.empty()) {
    const double tau = o.trunc > 0 ? o.trunc : std::numeric_limits<double>::infinity();
    const auto kind = parse_pairwise(o.pairwise) == mp::PairwiseKind::truncated_quadratic
                          ? mp::PairwiseKind::truncated_quadratic
                          : mp::PairwiseKind::truncated_linear;
    return mp::denoise_unaries<float>(mp::load_pgm(o.image_file), o.max_disp, kind, tau);
  }
  // seeded synthetic volume (the reference's smoke-run fallback): U[0, 8)
  mp::UnaryVolume<float> vol(o.height, o.width, o.max_disp);
  std::mt19937_64 rng(o.seed);
  std::uniform_real_distribution<double> u(0.0, 8.0);
  for (auto& v : vol.values) v = static_cast<float>(u(rng));
  return vol;
}

int run(const RunOpts& o) {
  mp::PotentialSet<float> pots;
  pots.unary = make_unaries(o);
  mp::PairwiseParams params;
  params.trunc = o.trunc;
  params.p1 = o.p1;
  params.p2 = o.p2;
  pots.pairwise = mp::build_pairwise<float>(parse_pairwise(o.pairwise), params, pots.unary.labels);
  pots.weights = mp::EdgeWeights<float>::constant(static_cast<float>(o.weight));
  const mp::GridGraph g(pots.unary.height, pots.unary.width);
  const mp::GridTopology topo(g, mp::DirectionSet::build(o.dirs));
  const mp::GridTopology eval4(g, mp::DirectionSet::build(4));  // energies on the 4-connected edge set
  const auto rho = mp::default_rho<float>(o.dirs, static_cast<float>(o.rho));

  std::vector<mp::EnergyRow> rows;
  std::vector<std::uint16_t> final_labels;
  auto record = [&](int k, double ms, const std::vector<std::uint16_t>& labels) {
    rows.push_back({k + 1, mp::energy(eval4, pots, labels), ms});
    final_labels = labels;
  };
  // a step's wall time includes its device work (the aggregation's copy back
  // synchronises), as the reference times the CPU step
  if (o.method == "isgmr" || o.method == "trwp") {
    std::optional<mp::IsgmrEngine<float>> ie;
    std::optional<mp::TrwpEngine<float>> te;
    if (o.method == "isgmr")
      ie.emplace(topo, pots, o.threads);
    else
      te.emplace(topo, pots, rho, o.threads);
    for (int k = 0; k < o.iters; ++k) {
      const double t0 = now_ms();
      if (ie) ie->step(); else te->step();
      cudaDeviceSynchronize();
      const double t1 = now_ms();
      record(k, t1 - t0, (ie ? ie->aggregate() : te->aggregate()).labels_map);
    }
  } else if (o.method == "sgm" || o.method == "sgm-std") {
    mp::SgmIterative<float> eng(topo, pots, o.method == "sgm" ? mp::SgmVariant::revised : mp::SgmVariant::standard,
                                o.threads);
    for (int k = 0; k < o.iters; ++k) {
      const double t0 = now_ms();
      const auto& out = eng.step();
      const double t1 = now_ms();
      record(k, t1 - t0, out.labels_map);
    }
  } else if (o.method == "mf") {
    throw UsageError("--method mf: the mean-field baseline is not on the GPU path (use the reference CLI)");
  } else {
    throw UsageError("--method: unknown method '" + o.method + "'");
  }

  mp::write_energy_csv(o.out_csv, rows);
  mp::save_label_map(o.out_labels, pots.unary.height, pots.unary.width, final_labels);
  std::printf("method=%s dirs=%d iters=%d final_energy=%.10g\n", o.method.c_str(), o.dirs, o.iters, rows.back().energy);

  if (o.timing_repeats > 0) {
    double total = 0.0;
    for (int rep = 0; rep < o.timing_repeats; ++rep) {
      const double t0 = now_ms();
      if (o.method == "trwp")
        mp::trwp_forward(topo, pots, rho, o.iters, o.threads);
      else if (o.method == "isgmr")
        mp::isgmr_forward(topo, pots, o.iters, o.threads);
      else
        mp::sgm_iterative(topo, pots, o.iters,
                          o.method == "sgm-std" ? mp::SgmVariant::standard : mp::SgmVariant::revised, o.threads);
      total += now_ms() - t0;
    }
    std::printf("mean_forward_ms=%.3f over %d repeats\n", total / o.timing_repeats, o.timing_repeats);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(parse(argc, argv));
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
