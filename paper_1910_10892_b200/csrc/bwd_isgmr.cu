// Instantiations of the warp-per-scanline backward for ISGMR (4 / 8
// directions compile-time, any other count at run time).
#include "launch.hpp"

namespace mrf {

template <int EPL, int RT, bool FULL>
static cudaError_t run(const BwdArgs& a, int batch, cudaStream_t s) {
  const int R = a.g.R;
  const int rowsF = 2 + (false ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = bwd_warp_smem_floats(EPL, rowsF) * int(sizeof(float)) * wpc;
  auto kern = bwd_warp_kernel<EPL, false, RT, FULL>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a);
  return cudaGetLastError();
}

template <int EPL>
static cudaError_t run_r(const BwdArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) return full ? run<EPL, 4, true>(a, batch, s) : run<EPL, 4, false>(a, batch, s);
  if (a.g.R == 8) return full ? run<EPL, 8, true>(a, batch, s) : run<EPL, 8, false>(a, batch, s);
  return run<EPL, 0, false>(a, batch, s);
}

cudaError_t launch_bwd_isgmr(const BwdArgs& a, int batch, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return run_r<1>(a, batch, s);
    case 2: return run_r<2>(a, batch, s);
    case 4: return run_r<4>(a, batch, s);
    case 6: return run_r<6>(a, batch, s);
    default: return run_r<8>(a, batch, s);
  }
}

}  // namespace mrf
