// Instantiations of the banded D == 2 forward for TRWP (4 / 8 directions).
#include "fwd_band2.cuh"
#include "launch.hpp"

namespace mrf {

template <int EPL, int R, bool FULL, bool AGG, int RD, int ST>
static cudaError_t run_(const FwdArgs& a, int batch, cudaStream_t s) {
  constexpr int rows = 1 + (true ? R - 1 : R - 2);
  // one warp per CTA: the scheduler placement of these lone-warp chains is
  // then the hardware's to spread (measured on C2 against 2 / 4 warps per
  // CTA: horizontal sweeps 710 -> 690 us, vertical 531 -> 485 us; forward
  // 12.15 -> 11.60 ms per step). The ISGMR launches (all directions at once,
  // C1 / C3) measured better with warps_per_cta().
  const int wpc = 1;
  const int smem = band2_smem_floats(EPL, rows, ST) * int(sizeof(float)) * wpc;
  auto kern = fwd_band2_kernel<EPL, true, R, FULL, AGG, RD, ST>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <int EPL, int R, bool FULL, bool AGG = false, int RD = -1>
static cudaError_t run(const FwdArgs& a, int batch, cudaStream_t s) {
  return band2_stages(a.nlines, batch, a.g.L) == 3 ? run_<EPL, R, FULL, AGG, RD, 3>(a, batch, s)
                                            : run_<EPL, R, FULL, AGG, RD, 4>(a, batch, s);
}

template <int EPL>
static cudaError_t run_epl(const FwdArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) {
    switch (a.dir) {  // one direction per launch: compile-time row selection
      case 0: return full ? run<EPL, 4, true, false, 0>(a, batch, s) : run<EPL, 4, false, false, 0>(a, batch, s);
      case 1: return full ? run<EPL, 4, true, false, 1>(a, batch, s) : run<EPL, 4, false, false, 1>(a, batch, s);
      case 2: return full ? run<EPL, 4, true, false, 2>(a, batch, s) : run<EPL, 4, false, false, 2>(a, batch, s);
      case 3:
        if (a.agg_cost || a.agg_labels)  // last sweep of the call: aggregation fused
          return full ? run<EPL, 4, true, true, 3>(a, batch, s) : run<EPL, 4, false, true, 3>(a, batch, s);
        return full ? run<EPL, 4, true, false, 3>(a, batch, s) : run<EPL, 4, false, false, 3>(a, batch, s);
      default: return full ? run<EPL, 4, true>(a, batch, s) : run<EPL, 4, false>(a, batch, s);
    }
  }
  return full ? run<EPL, 8, true>(a, batch, s) : run<EPL, 8, false>(a, batch, s);
}

cudaError_t launch_fwd_band2_trwp(const FwdArgs& a, int batch, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return run_epl<1>(a, batch, s);
    case 2: return run_epl<2>(a, batch, s);
    case 4: return run_epl<4>(a, batch, s);
    case 6: return run_epl<6>(a, batch, s);
    default: return run_epl<8>(a, batch, s);
  }
}

}  // namespace mrf
