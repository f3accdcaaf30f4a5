// Backward over per-direction scatter planes (sm_100a): the algebra shared by
// the backward kernels (bwd_split.cuh), isgmr_backward / trwp_backward
// (autodiff.hpp:63-126, :133-197) restated so that a node step reads the
// gradient it consumes and writes ONE row.
//
// The reference keeps message-gradient planes gm[d] and, for every label l of
// every edge (prev -> cur) of direction r, adds the reparametrised row g_l to
// dtheta[prev][p_l], gm[r][prev][p_l] (the sweep's own chain) and to the
// other planes at prev (TRWP: rho*g to every d, -g extra to r^1; ISGMR: g to
// gm_next[d] for d not in {r, r^1}). All those additions are the same
// per-node vector acc_r[prev][mu] = sum_{l : p_l = mu} g_l (times rho). So
// the sweep stores acc_r once, into plane A[r], and the planes the reference
// accumulates are recovered when they are consumed:
//
//   TRWP  gm[r](cur) at sweep (k, r) =
//           [k == K-1] dc(cur)                           (initial broadcast, :142-144)
//         + sum_{d != r, in sweep order since plane r was last cleared}
//               rho_d(cur) A[d](cur) - [d == r^1] A[d](cur)
//         (A[d] holds direction d's most recent sweep: iteration k+1 for d < r,
//          k for d > r; at k == K-1 only d > r have run; the clear of :190-193
//          is the window boundary)
//   ISGMR gm[r](cur) at iteration k = [k == K-1] dc(cur)
//         + [k < K-1] sum_{d not in {r, r^1}} A_{k+1}[d](cur)   (gm_next, swap :122-123)
//   dtheta = dc + sum_{k, d} rho_d A_k[d]  (accumulated once per iteration by
//                                           dtheta_acc_kernel)
//
// plus, as in the reference, the sweep's own chain ("carry": rho_r acc_r at
// prev is exactly what node prev reads next from gm[r]). Per node and sweep
// that is R-1 (TRWP) / R-2 (ISGMR) row reads and one row write instead of
// R+1 read-modify-writes, and ISGMR's directions become independent within an
// iteration (one launch per iteration, all R directions' scanlines).
// Per-mu aggregation and the regrouped row sums reorder the reference's
// per-label additions, so gradients match within the 1e-5 tolerance rather
// than bitwise. The tail row of every line is written as zeros (no edge has it as prev),
// so planes never need clearing.
#pragma once

#include "common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

// dV accumulation: every CTA (bwd_split) / warp (bwd_small) owns a private
// [L][L] slot per image, accumulated over all sweeps of the backward (lines
// are assigned to CTAs statically) and reduced over the slots in a fixed order
// at the end, so dV is bit-identical run to run (the reference's per-scanline
// partials reduced in order, autodiff.hpp:119-120, test_autodiff.cpp:86-110).
// Within a slot every addition is ordered: one warp writes it, lanes of one
// instruction hit distinct entries and successive instructions are separated
// by __syncwarp().
constexpr int kDvSlotsSplit = 592;      // persistent CTAs per image of bwd_split (<= 4 per SM)
constexpr int kDvSlotsSmall = 592 * 4;  // warps per image of bwd_small
constexpr int kDvSlotsWarp = 2048;      // warps per image of bwd_warp (one line each up to this many)
// slots one backward call needs for the largest launch of `maxlines` lines
__host__ __device__ inline int dv_slots_for(int L, int maxlines) {
  const int m = maxlines > 1 ? maxlines : 1;
  if (L <= 32) return kDvSlotsSmall;
  const int w = m < kDvSlotsWarp ? m : kDvSlotsWarp;
  return w > kDvSlotsSplit ? w : (m < kDvSlotsSplit ? m : kDvSlotsSplit);
}

struct AccArgs {
  Geometry g;
  Potentials pot;
  const LineDesc* lines;  // TRWP: direction r's lines; ISGMR: every direction's lines
  int nlines;
  const uint8_t* p;
  const uint8_t* q;
  int k;
  const float* dc;   // [B][N][L] cost gradient (read at k == K-1)
  const float* ain;  // [B][R][N][L] planes read (TRWP: == aout; ISGMR: iteration k+1)
  float* aout;       // [B][R][N][L] planes written (plane r of each line)
  float* gw;         // TRWP: [B][R/2][N] (family planes); ISGMR: [B][R][N] per direction; or null
  float* gvacc;      // [B][dv_slots][L][L] private dV slots, V orientation (x = first label)
  int dv_slots;
  const PairDesc* desc;
  float* dtheta;     // TRWP direction 0: dtheta += rho_d A[d] of the iteration, fused (else null)
  const float* dtheta_src;  // the running dtheta read by that update: dc on the first one (no dc -> dtheta copy)
};

// row slots: TRWP R-1 planes (+ dc at k == K-1: at most R), ISGMR R-2 planes or dc
__host__ __device__ constexpr int acc_rows(bool trwp, int R) { return trwp ? R : (R - 2 > 1 ? R - 2 : 1); }

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// dtheta[n] += sum_d rho_d(n) A[d](n) (TRWP; rho_d(n) is the tree coefficient
// of direction d's edge with n as prev) or sum_d A[d](n) (ISGMR), d
// ascending: the iteration's contribution of every sweep to the unary
// gradient (autodiff.hpp:101 / :173). Image b = blockIdx.y; float4 when L % 4
// == 0 (a vector never straddles two nodes).
// RT: the direction count as a compile-time bound (4, 8 or 16): the row
// loads of one vector stay in registers without capping occupancy.
template <bool TRWP, int RT = 16>
__global__ void __launch_bounds__(256) dtheta_acc_kernel(int R, int N, int L, const float* __restrict__ A, float rho,
                                  const float* __restrict__ rho_planes, Geometry g, float* __restrict__ dtheta,
                                  const float* dtheta_src) {
  // dtheta = dtheta_src + sum_d rho_d A[d]; dtheta_src is dc on the first update
  const int NL = N * L;
  const int b = blockIdx.y;
  const float* Ab = A + size_t(b) * R * NL;
  float* dt = dtheta + size_t(b) * NL;
  const float* ds = dtheta_src + size_t(b) * NL;
  auto rho_of = [&](int d, int n) {
    if (!TRWP) return 1.0f;
    if (!rho_planes) return rho;
    const int wn = (d & 1) ? n + g.node_step[d] : n;
    return __ldg(rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + min(max(wn, 0), N - 1));
  };
  // rho per element only with rho planes (a 4-vector may straddle nodes when L % 4 != 0)
  const bool per_elem = TRWP && rho_planes != nullptr;
  if ((NL & 3) == 0) {  // every image's block is 16-byte aligned
    const int n4 = NL >> 2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
      float4 v[RT];  // every row load in flight before the sums
#pragma unroll
      for (int d = 0; d < RT; ++d)
        if (d < R) v[d] = __ldcs(reinterpret_cast<const float4*>(Ab + size_t(d) * NL) + i);
      float4 o = reinterpret_cast<const float4*>(ds)[i];
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int d = 0; d < RT; ++d) {
        if (d >= R) continue;
        float4 t = v[d];
        if (TRWP) {
          if (per_elem) {
            const int e0 = i << 2;
            t.x = fmul(rho_of(d, e0 / L), t.x), t.y = fmul(rho_of(d, (e0 + 1) / L), t.y);
            t.z = fmul(rho_of(d, (e0 + 2) / L), t.z), t.w = fmul(rho_of(d, (e0 + 3) / L), t.w);
          } else {
            t.x = fmul(rho, t.x), t.y = fmul(rho, t.y), t.z = fmul(rho, t.z), t.w = fmul(rho, t.w);
          }
        }
        s.x = fadd(s.x, t.x), s.y = fadd(s.y, t.y), s.z = fadd(s.z, t.z), s.w = fadd(s.w, t.w);
      }
      o.x = fadd(o.x, s.x), o.y = fadd(o.y, s.y), o.z = fadd(o.z, s.z), o.w = fadd(o.w, s.w);
      reinterpret_cast<float4*>(dt)[i] = o;
    }
  } else {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < NL; i += gridDim.x * blockDim.x) {
      float s = 0.0f;
      for (int d = 0; d < R; ++d) {
        const float v = __ldcs(Ab + size_t(d) * NL + i);
        s = fadd(s, TRWP ? fmul(per_elem ? rho_of(d, i / L) : rho, v) : v);
      }
      dt[i] = fadd(ds[i], s);
    }
  }
}

// ISGMR per-direction dw partials -> family planes: gw[b][f][n] = dwr[b][2f][n] + dwr[b][2f+1][n]
static __global__ void combine_dw_kernel(int B, int R, int N, const float* __restrict__ dwr, float* __restrict__ gw) {
  const int64_t total = int64_t(B) * (R / 2) * N;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t n = i % N, bf = i / N;
    gw[i] = fadd(dwr[(2 * bf) * N + n], dwr[(2 * bf + 1) * N + n]);
  }
}

// dV[b][xy] = sum over slots s = 0, 1, ... of acc[b][s][xy], in slot order
// (deterministic). Slots are summed in chunks of 8 loads in flight.
static __global__ void reduce_gvacc_kernel(int B, int L, int slots, int used, const float* __restrict__ acc,
                                           float* __restrict__ gv) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t LL = int64_t(L) * L;
  if (i >= B * LL) return;
  const int64_t b = i / LL, xy = i - b * LL;
  const float* base = acc + size_t(b) * slots * LL + xy;
  float s = 0.0f;
  int t = 0;
  for (; t + 8 <= used; t += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(base + size_t(t + u) * LL);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = fadd(s, v[u]);
  }
  for (; t < used; ++t) s = fadd(s, __ldcs(base + size_t(t) * LL));
  gv[i] = s;
}

}  // namespace mrf
