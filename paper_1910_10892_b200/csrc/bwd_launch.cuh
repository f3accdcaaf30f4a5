// Launcher for the warp-specialised backward (bwd_split.cuh): one CTA per
// scanline (CHAIN + POST + kSplitPre producer warps).
#pragma once

#include "bwd_common.cuh"
#include "bwd_grp.cuh"
#include "bwd_small.cuh"
#include "bwd_split.cuh"
#include "bwd_warp.cuh"
#include "launch.hpp"

namespace mrf {

// Persistent grid: at most one wave of resident CTAs (and at most
// kDvSlotsSplit, the private dV slots per image); CTA c sweeps lines c, c + G,
// ... (lines sorted longest first), the same lines in every call.
static int split_grid(const void* kern, int threads, int smem, int nlines) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  const int g = occ * sms < kDvSlotsSplit ? occ * sms : kDvSlotsSplit;
  return nlines < g ? nlines : g;
}

template <int EPL, bool TRWP, int RT, bool FULL, int MODE>
static cudaError_t run_split1(const AccArgs& a, int batch, cudaStream_t s) {
  constexpr int NPRE = kSplitPre;
  const int smem = split_smem_floats(EPL, acc_rows(TRWP, a.g.R), NPRE, MODE == 2) * int(sizeof(float));
  auto kern = bwd_split_kernel<EPL, TRWP, RT, FULL, NPRE, MODE>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int blocks = split_grid(reinterpret_cast<const void*>(kern), 32 * (2 + NPRE), smem, a.nlines);
  kern<<<dim3(blocks, batch), 32 * (2 + NPRE), smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

// banded D <= 2: one warp per line (bwd_warp.cuh)
template <int EPL, bool TRWP, int RT, bool FULL>
static cudaError_t run_warp(const AccArgs& a, int batch, cudaStream_t s) {
  const int wpc = 4;
  const int smem = bwarp_warp_floats(EPL, acc_rows(TRWP, a.g.R)) * wpc * int(sizeof(float));
  auto kern = bwd_warp_kernel<EPL, TRWP, RT, FULL>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int warps = a.nlines < kDvSlotsWarp ? a.nlines : kDvSlotsWarp;
  kern<<<dim3((warps + wpc - 1) / wpc, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

// Banded D <= 2 launches with many lines take one warp per line; few lines
// (C2's 375-row horizontal TRWP sweeps: 2.5 lines per SM) keep the
// warp-specialised split kernel, whose roles pipeline a lone line's node
// steps (measured per launch, C2: 375 lines 2.05 ms one-warp vs 0.85 ms
// split; 1242 lines 0.77 vs 0.77; C3's 7496-line ISGMR launch 3.16 vs
// 3.61 ms per iteration; C1 0.31 vs 0.32). A/B: MRF_BWD_BAND=split|warp.
inline bool bwd_band_split(int nlines, int batch) {
  const char* env = getenv("MRF_BWD_BAND");
  if (env && (env[0] == 's' || env[0] == 'w')) return env[0] == 's';
  return int64_t(nlines) * batch < 148 * 9;
}

// The pairwise strategy is known on the device only: every mode is launched
// and the instantiations that do not own the sweep exit at once.
template <int EPL, bool TRWP, int RT, bool FULL>
static cudaError_t run_split(const AccArgs& a, int batch, cudaStream_t s) {
  cudaError_t e = bwd_band_split(a.nlines, batch) ? run_split1<EPL, TRWP, RT, FULL, 1>(a, batch, s)
                                                  : run_warp<EPL, TRWP, RT, FULL>(a, batch, s);
  if (e == cudaSuccess) e = run_split1<EPL, TRWP, RT, FULL, 2>(a, batch, s);
  if (e == cudaSuccess) e = run_split1<EPL, TRWP, RT, FULL, 0>(a, batch, s);
  return e;
}

template <int EPL, bool TRWP>
static cudaError_t run_split_r(const AccArgs& a, int batch, cudaStream_t s) {
  const bool full = a.g.L == 32 * EPL;
  if (a.g.R == 4) return full ? run_split<EPL, TRWP, 4, true>(a, batch, s) : run_split<EPL, TRWP, 4, false>(a, batch, s);
  if (a.g.R == 8) return full ? run_split<EPL, TRWP, 8, true>(a, batch, s) : run_split<EPL, TRWP, 8, false>(a, batch, s);
  return run_split<EPL, TRWP, 0, false>(a, batch, s);
}

// L <= 32: one warp per scanline, lane = label (bwd_small.cuh)
template <bool TRWP, int RT>
static cudaError_t run_small(const AccArgs& a, int batch, cudaStream_t s) {
  const int wpc = 4;
  const int smem = small_cta_floats(acc_rows(TRWP, a.g.R), a.g.L, wpc) * int(sizeof(float));
  auto kern = bwd_small_kernel<TRWP, RT>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  // at most kDvSlotsSmall warps per image (one private dV slot each)
  const int want = (a.nlines + wpc - 1) / wpc;
  const int blocks = want < kDvSlotsSmall / wpc ? want : kDvSlotsSmall / wpc;
  kern<<<dim3(blocks, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

// TRWP-4, 16 < L <= 24, constant rho, unary gradient not fused: 8 lanes x 3
// labels per line, 4 lines per warp (bwd_grp.cuh); one private dV slot per
// line group, at most kDvSlotsSmall per image
static cudaError_t run_grp(const AccArgs& a, int batch, cudaStream_t s) {
  const int wpc = kBgWarps;
  const int smem = bwd_grp_cta_floats(wpc, a.dtheta != nullptr) * int(sizeof(float));
  // a.dtheta is set only on the direction-0 launches of a fused call
  auto kern = a.dtheta ? bwd_grp_kernel<true> : bwd_grp_kernel<false>;
  cudaError_t e = ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int per_cta = wpc * kGrpLines;
  const int want = (a.nlines + per_cta - 1) / per_cta;
  const int cap = kDvSlotsSmall / per_cta;
  kern<<<dim3(want < cap ? want : cap, batch), 32 * wpc, smem, s>>>(a); note_launch();
  return cudaGetLastError();
}

template <bool TRWP>
static cudaError_t launch_bwd_sweep(const AccArgs& a, int batch, cudaStream_t s) {
  if (a.nlines == 0) return cudaSuccess;
  if (TRWP && bwd_uses_grp(a.g.L, a.g.R, a.pot.rho_planes != nullptr, a.nlines, batch)) return run_grp(a, batch, s);
  // L <= 32 with many lines: one warp per line; few lines: warp-specialised
  if (bwd_uses_small(a.g.L, a.nlines, batch)) {
    if (a.g.R == 4) return run_small<TRWP, 4>(a, batch, s);
    if (a.g.R == 8) return run_small<TRWP, 8>(a, batch, s);
    return run_small<TRWP, 0>(a, batch, s);
  }
  switch (epl_for(a.g.L)) {
    case 1: return run_split_r<1, TRWP>(a, batch, s);
    case 2: return run_split_r<2, TRWP>(a, batch, s);
    case 4: return run_split_r<4, TRWP>(a, batch, s);
    case 6: return run_split_r<6, TRWP>(a, batch, s);
    default: return run_split_r<8, TRWP>(a, batch, s);
  }
}

}  // namespace mrf
