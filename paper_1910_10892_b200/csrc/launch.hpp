// Kernel launchers, one translation unit per kernel family (compiled in
// parallel). Each returns the CUDA error of its launch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "bwd_common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

// every kernel launch of the library is counted (mrf_launch_count)
void note_launch();
// clears *flag when data[0:count) holds Inf / NaN (misc.cu)
cudaError_t launch_finite_scan(const float* data, size_t count, int* flag, cudaStream_t stream);

// labels per lane for the warp-per-scanline kernels
inline int epl_for(int L) {
  if (L <= 32) return 1;
  if (L <= 64) return 2;
  if (L <= 128) return 4;
  if (L <= 192) return 6;
  return 8;
}

// cp.async ring depth of the banded D == 2 forward for a launch of nlines
// lines x batch with L labels: 3 when warps share schedulers and rows are
// long, else 4 (measured, real-run fwd time per step: C2 13.35 -> 12.70 ms
// with 3 on the vertical sweeps only; the horizontal ones (lone warps) lose at
// 3; C1 (L = 16) loses 6 % at 3, C3 (L = 128) is neutral).
// MRF_BAND2_STAGES=3|4 forces one (A/B measurements).
inline int band2_stages(int nlines, int batch, int L) {
  const char* env = getenv("MRF_BAND2_STAGES");
  if (env && (env[0] == '3' || env[0] == '4')) return env[0] - '0';
  return int64_t(nlines) * batch > 4 * 148 && L > 128 ? 3 : 4;
}

// Readout and evaluation (head.cu)
struct EvenSteps {
  int dh[8], dw[8];  // step of direction 2f (the even direction of family f)
};
cudaError_t launch_soft_head(int B, int N, int L, const float* cost, const float* target, float* conf, float* disp,
                             float* grad, float* loss, double* partial, int nblk, cudaStream_t s);
int soft_head_blocks(int N);
cudaError_t launch_energy(int B, int H, int W, int L, int R, const EvenSteps& st, const float* unary, const float* V,
                          float w, const float* wplanes, const uint16_t* labels, double* out, double* partial, int nblk,
                          int* bad, cudaStream_t s);
int energy_blocks(int N);
cudaError_t launch_sgm_next_unary(int B, int N, int L, int R, const float* messages, float* next, cudaStream_t s);
cudaError_t launch_sgm_standard(const Geometry& g, const Potentials& pot, const LineDesc* lines, int nlines, float* m,
                                int batch, cudaStream_t s);

// backward kernel choice: one warp per line (L <= 32, many lines) or warp-specialised
inline bool bwd_uses_small(int L, int nlines, int batch) {
  const char* env = getenv("MRF_BWD_SMALL");  // A/B and tests: 0 = never, 1 = whenever L <= 32
  if (env && (env[0] == '0' || env[0] == '1')) return L <= 32 && env[0] == '1';
  return L <= 32 && int64_t(nlines) * batch >= 148 * 16;
}
// TRWP with the one-warp-per-line small-L kernel: fuse the unary-gradient
// collection into its direction-0 sweep (else dtheta_acc_kernel per iteration)
inline bool bwd_small_fuse() {
  const char* env = getenv("MRF_SMALL_FUSE");
  return env && env[0] == '1';
}

// TRWP-4, 16 < L <= 24, constant rho: the grouped small-L backward
// (bwd_grp.cuh) takes the launches bwd_uses_small gives the small-L kernels
inline bool bwd_grp_enabled(int L, int R, bool rho_planes) {
  const char* env = getenv("MRF_BWD_GRP");  // A/B: 0 = lane-per-label kernel only
  if (env && env[0] == '0') return false;
  return R == 4 && L > 16 && L <= 24 && !rho_planes;
}
// The grouped kernel takes launches of >= 592 lines (4 per SM) -- C4 on 8
// GPUs (4 images per rank, 2048 lines): 12.9 ms per backward against 34.6
// on the warp-specialised kernel; MRF_BWD_SMALL=0 / 1 forces it off / on
inline bool bwd_uses_grp(int L, int R, bool rho_planes, int nlines, int batch) {
  if (!bwd_grp_enabled(L, R, rho_planes)) return false;
  const char* env = getenv("MRF_BWD_SMALL");
  if (env && (env[0] == '0' || env[0] == '1')) return env[0] == '1';
  return int64_t(nlines) * batch >= 148 * 4;
}
// ... and collects the unary gradient in its direction-0 sweep (A/B:
// MRF_GRP_FUSE=0 leaves it to dtheta_acc_kernel)
inline bool bwd_grp_fuse() {
  const char* env = getenv("MRF_GRP_FUSE");
  return !(env && env[0] == '0');
}

// warps per CTA: few long chains -> spread them over every SM
inline int warps_per_cta(int nlines) {
  const char* env = getenv("MRF_FWD_WPC");  // A/B: force 1, 2 or 4 warps per CTA
  if (env && (env[0] == '1' || env[0] == '2' || env[0] == '4')) return env[0] - '0';
  return nlines >= 148 * 8 ? 4 : (nlines >= 148 * 2 ? 2 : 1);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size) instead of on every launch (it costs host time on the launch path).
cudaError_t ensure_dynamic_smem(const void* kern, int bytes);

cudaError_t launch_fwd_generic(const FwdArgs& a, int batch, bool trwp, cudaStream_t s);
cudaError_t launch_fwd_bandw(const FwdArgs& a, int batch, bool trwp, cudaStream_t s);
int fwd_bandw_max();  // widest band D the wide-band forward covers
bool fwd_small_applies(int L, int R);  // dense small-L forward (fwd_small.cuh) covers the sweep
cudaError_t launch_fwd_small(const FwdArgs& a, int batch, bool trwp, cudaStream_t s);
cudaError_t launch_fwd_band2_isgmr(const FwdArgs& a, int batch, cudaStream_t s);
cudaError_t launch_fwd_band2_trwp(const FwdArgs& a, int batch, cudaStream_t s);
cudaError_t launch_bwd_isgmr(const AccArgs& a, int batch, cudaStream_t s);
cudaError_t launch_bwd_trwp(const AccArgs& a, int batch, cudaStream_t s);


}  // namespace mrf
