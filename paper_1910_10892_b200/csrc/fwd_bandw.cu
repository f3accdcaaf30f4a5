// Instantiations of the wide-band forward (2 < D <= 16; 4 / 8 directions).
#include "fwd_bandw.cuh"
#include "launch.hpp"

namespace mrf {

constexpr int kBandW = 16;

template <int EPL, bool TRWP, int R, bool FULL>
static cudaError_t run(const FwdArgs& a, int batch, cudaStream_t s) {
  constexpr int rows = 1 + (TRWP ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = bandw_smem_floats(EPL, kBandW, rows) * int(sizeof(float)) * wpc;
  auto kern = fwd_bandw_kernel<EPL, TRWP, R, FULL, kBandW>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <int EPL, bool TRWP>
static cudaError_t run_epl(const FwdArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) return full ? run<EPL, TRWP, 4, true>(a, batch, s) : run<EPL, TRWP, 4, false>(a, batch, s);
  return full ? run<EPL, TRWP, 8, true>(a, batch, s) : run<EPL, TRWP, 8, false>(a, batch, s);
}

template <bool TRWP>
static cudaError_t launch(const FwdArgs& a, int batch, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return run_epl<1, TRWP>(a, batch, s);
    case 2: return run_epl<2, TRWP>(a, batch, s);
    case 4: return run_epl<4, TRWP>(a, batch, s);
    case 6: return run_epl<6, TRWP>(a, batch, s);
    default: return run_epl<8, TRWP>(a, batch, s);
  }
}

int fwd_bandw_max() { return kBandW; }
cudaError_t launch_fwd_bandw(const FwdArgs& a, int batch, bool trwp, cudaStream_t s) {
  return trwp ? launch<true>(a, batch, s) : launch<false>(a, batch, s);
}

}  // namespace mrf
