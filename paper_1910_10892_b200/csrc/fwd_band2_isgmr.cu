// Instantiations of the banded D == 2 forward for ISGMR (4 / 8 directions).
#include "fwd_band2.cuh"
#include "launch.hpp"

namespace mrf {

template <int EPL, int R, bool FULL, int ST>
static cudaError_t run_(const FwdArgs& a, int batch, cudaStream_t s) {
  constexpr int rows = 1 + (false ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = band2_smem_floats(EPL, rows, ST) * int(sizeof(float)) * wpc;
  auto kern = fwd_band2_kernel<EPL, false, R, FULL, false, -1, ST>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <int EPL, int R, bool FULL>
static cudaError_t run(const FwdArgs& a, int batch, cudaStream_t s) {
  return band2_stages(a.nlines, batch, a.g.L) == 3 ? run_<EPL, R, FULL, 3>(a, batch, s) : run_<EPL, R, FULL, 4>(a, batch, s);
}

template <int EPL>
static cudaError_t run_epl(const FwdArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) return full ? run<EPL, 4, true>(a, batch, s) : run<EPL, 4, false>(a, batch, s);
  return full ? run<EPL, 8, true>(a, batch, s) : run<EPL, 8, false>(a, batch, s);
}

cudaError_t launch_fwd_band2_isgmr(const FwdArgs& a, int batch, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return run_epl<1>(a, batch, s);
    case 2: return run_epl<2>(a, batch, s);
    case 4: return run_epl<4>(a, batch, s);
    case 6: return run_epl<6>(a, batch, s);
    default: return run_epl<8>(a, batch, s);
  }
}

}  // namespace mrf
