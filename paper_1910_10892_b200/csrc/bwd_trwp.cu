// Instantiations of the backward for TRWP (4 / 8 directions compile-time,
// any other count at run time). Few long scanlines (a KITTI row direction:
// 375 lines on 148 SMs) are latency-bound: each line gets a warp pair (chain
// warp + leaf warp, bwd_ws.cuh). Many lines are issue-bound: one warp per
// line (bwd_warp.cuh), which executes fewer instructions in total.
#include "bwd_warp.cuh"
#include "bwd_ws.cuh"
#include "launch.hpp"

namespace mrf {

template <int EPL, int RT, bool FULL>
static cudaError_t run_ws(const BwdArgs& a, int batch, cudaStream_t s) {
  const int R = a.g.R;
  const int nrowB = 1 + (true ? R - 1 : R - 2);
  const int per_pair = bws_pair_floats(EPL, nrowB) * int(sizeof(float));
  int pairs = warps_per_cta(a.nlines);
  while (pairs > 1 && per_pair * pairs > 220 * 1024) pairs >>= 1;
  const int smem = per_pair * pairs;
  auto kern = bwd_ws_kernel<EPL, true, RT, FULL>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + pairs - 1) / pairs < 65535 ? (a.nlines + pairs - 1) / pairs : 65535;
  kern<<<dim3(blocks, batch), 64 * pairs, smem, s>>>(a);
  return cudaGetLastError();
}

template <int EPL, int RT, bool FULL>
static cudaError_t run_warp(const BwdArgs& a, int batch, cudaStream_t s) {
  const int R = a.g.R;
  const int rowsF = 2 + (true ? R - 1 : R - 2);
  const int wpc = warps_per_cta(a.nlines);
  const int smem = bwd_warp_smem_floats(EPL, rowsF) * int(sizeof(float)) * wpc;
  auto kern = bwd_warp_kernel<EPL, true, RT, FULL>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = (a.nlines + wpc - 1) / wpc < 65535 ? (a.nlines + wpc - 1) / wpc : 65535;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a);
  return cudaGetLastError();
}

template <int EPL, int RT, bool FULL>
static cudaError_t run(const BwdArgs& a, int batch, cudaStream_t s) {
  // fewer than ~4 warps per SM of lines: pair them up
  return int64_t(a.nlines) * batch <= 148 * 3 ? run_ws<EPL, RT, FULL>(a, batch, s) : run_warp<EPL, RT, FULL>(a, batch, s);
}

template <int EPL>
static cudaError_t run_r(const BwdArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) return full ? run<EPL, 4, true>(a, batch, s) : run<EPL, 4, false>(a, batch, s);
  if (a.g.R == 8) return full ? run<EPL, 8, true>(a, batch, s) : run<EPL, 8, false>(a, batch, s);
  return run<EPL, 0, false>(a, batch, s);
}

cudaError_t launch_bwd_trwp(const BwdArgs& a, int batch, cudaStream_t s) {
  switch (epl_for(a.g.L)) {
    case 1: return run_r<1>(a, batch, s);
    case 2: return run_r<2>(a, batch, s);
    case 4: return run_r<4>(a, batch, s);
    case 6: return run_r<6>(a, batch, s);
    default: return run_r<8>(a, batch, s);
  }
}

}  // namespace mrf
