// Instantiations of the small-L dense forward (L <= 32; 4 / 8 directions).
#include "fwd_grp.cuh"
#include "fwd_small.cuh"
#include "launch.hpp"

#include <cstdlib>

namespace mrf {

template <bool TRWP, int R, int LMAX, bool WPL, bool AGG>
static cudaError_t run1a(const FwdArgs& a, int batch, cudaStream_t s) {
  constexpr int rows = 1 + (TRWP ? R - 1 : R - 2);
  const int wpc = 4;
  const int smem = fwd_small_warp_floats(rows, kStages, WPL ? LMAX : 0) * int(sizeof(float)) * wpc;
  auto kern = fwd_small_kernel<TRWP, R, LMAX, WPL, AGG>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <bool TRWP, int R, int LMAX, bool WPL>
static cudaError_t run1(const FwdArgs& a, int batch, cudaStream_t s) {
  // the aggregation rides on TRWP's last 4-direction sweep (host sets agg_*)
  if (TRWP && R == 4 && (a.agg_cost || a.agg_labels)) return run1a<TRWP, R, LMAX, WPL, TRWP && R == 4>(a, batch, s);
  return run1a<TRWP, R, LMAX, WPL, false>(a, batch, s);
}

template <bool TRWP, int R, int LMAX>
static cudaError_t run(const FwdArgs& a, int batch, cudaStream_t s) {
  return a.pot.w_planes ? run1<TRWP, R, LMAX, true>(a, batch, s) : run1<TRWP, R, LMAX, false>(a, batch, s);
}

template <bool TRWP, int R>
static cudaError_t run_l(const FwdArgs& a, int batch, cudaStream_t s) {
  if (a.g.L <= 8) return run<TRWP, R, 8>(a, batch, s);
  if (a.g.L <= 16) return run<TRWP, R, 16>(a, batch, s);
  if (a.g.L <= 24) return run<TRWP, R, 24>(a, batch, s);
  return run<TRWP, R, 32>(a, batch, s);
}

// TRWP-4, 16 < L <= 24: 8 lanes x 3 labels per line, 4 lines per warp (fwd_grp.cuh)
template <int MU, bool WPL, bool AGG>
static cudaError_t run_grp(const FwdArgs& a, int batch, cudaStream_t s) {
  const int wpc = kGrpWarps;
  const int smem = fwd_grp_cta_floats(4, 3, wpc) * int(sizeof(float));
  auto kern = fwd_grp_kernel<3, MU, WPL, AGG>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int per_cta = wpc * kGrpLines;
  const int blocks = (a.nlines + per_cta - 1) / per_cta < 65535 ? (a.nlines + per_cta - 1) / per_cta : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <int MU>
static cudaError_t run_grp_mu(const FwdArgs& a, int batch, cudaStream_t s) {
  const bool agg = a.agg_cost || a.agg_labels;
  if (a.pot.w_planes) return agg ? run_grp<MU, true, true>(a, batch, s) : run_grp<MU, true, false>(a, batch, s);
  return agg ? run_grp<MU, false, true>(a, batch, s) : run_grp<MU, false, false>(a, batch, s);
}

static bool grp_enabled() {
  const char* env = getenv("MRF_FWD_GRP");  // A/B: 0 = lane-per-label kernel only
  return !(env && env[0] == '0');
}

bool fwd_small_applies(int L, int R) { return L <= 32 && (R == 4 || R == 8); }
cudaError_t launch_fwd_small(const FwdArgs& a, int batch, bool trwp, cudaStream_t s) {
  if (trwp && a.g.R == 4 && a.dir >= 0 && a.g.L > 16 && a.g.L <= 24 && grp_enabled()) {
    if (a.g.L <= 20) return run_grp_mu<20>(a, batch, s);
    if (a.g.L <= 22) return run_grp_mu<22>(a, batch, s);
    return run_grp_mu<24>(a, batch, s);
  }
  if (a.g.R == 4) return trwp ? run_l<true, 4>(a, batch, s) : run_l<false, 4>(a, batch, s);
  return trwp ? run_l<true, 8>(a, batch, s) : run_l<false, 8>(a, batch, s);
}

}  // namespace mrf
