// Instantiations of the warp-per-scanline backward (4 / 8 directions
// compile-time, any other count at run time).
#include "launch.hpp"

namespace mrf {

template <int EPL, bool TRWP, int RT>
static cudaError_t run(const BwdArgs& a, int batch, cudaStream_t s) {
  const int R = a.g.R;
  const int rowsF = 2 + (TRWP ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = bwd_warp_smem_floats(EPL, rowsF) * int(sizeof(float)) * wpc;
  auto kern = bwd_warp_kernel<EPL, TRWP, RT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a);
  return cudaGetLastError();
}

template <int EPL, bool TRWP>
static cudaError_t run_r(const BwdArgs& a, int batch, cudaStream_t s) {
  if (a.g.R == 4) return run<EPL, TRWP, 4>(a, batch, s);
  if (a.g.R == 8) return run<EPL, TRWP, 8>(a, batch, s);
  return run<EPL, TRWP, 0>(a, batch, s);
}

cudaError_t launch_bwd(const BwdArgs& a, int batch, bool trwp, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return trwp ? run_r<1, true>(a, batch, s) : run_r<1, false>(a, batch, s);
    case 2: return trwp ? run_r<2, true>(a, batch, s) : run_r<2, false>(a, batch, s);
    case 4: return trwp ? run_r<4, true>(a, batch, s) : run_r<4, false>(a, batch, s);
    case 6: return trwp ? run_r<6, true>(a, batch, s) : run_r<6, false>(a, batch, s);
    default: return trwp ? run_r<8, true>(a, batch, s) : run_r<8, false>(a, batch, s);
  }
}

}  // namespace mrf
