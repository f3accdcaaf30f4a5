// Instantiations of the generic warp-per-scanline forward (dense and banded
// with any D; banded D == 2 for 16 directions).
#include "launch.hpp"

namespace mrf {

template <int EPL, bool TRWP>
static cudaError_t run(const FwdArgs& a, int batch, cudaStream_t s) {
  const int R = a.g.R;
  const int rows = 1 + (TRWP ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = fwd_warp_smem_floats(EPL, rows) * int(sizeof(float)) * wpc;
  auto kern = fwd_warp_kernel<EPL, TRWP>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

cudaError_t launch_fwd_generic(const FwdArgs& a, int batch, bool trwp, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return trwp ? run<1, true>(a, batch, s) : run<1, false>(a, batch, s);
    case 2: return trwp ? run<2, true>(a, batch, s) : run<2, false>(a, batch, s);
    case 4: return trwp ? run<4, true>(a, batch, s) : run<4, false>(a, batch, s);
    case 6: return trwp ? run<6, true>(a, batch, s) : run<6, false>(a, batch, s);
    default: return trwp ? run<8, true>(a, batch, s) : run<8, false>(a, batch, s);
  }
}

}  // namespace mrf
