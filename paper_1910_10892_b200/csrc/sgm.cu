// Standard SGM pass (baselines.hpp:31-98, SgmVariant::standard), the scanline
// baseline the paper compares against, on the message-passing skeleton:
// one warp per scanline, every direction's lines in one launch (a direction's
// messages depend only on its own chain). The message keeps the unary:
//   m^r(head) = theta(head);
//   m^r(cur, l) = theta(cur, l) + min_mu (m^r(prev, mu) + w V'(mu, l)) - min_mu m^r(prev, mu)
// with the reference's operation order and std::min semantics (ascending mu,
// the first of equal values kept: only the sign of a zero can differ, and it
// is carried). Dense candidates from a shared copy of the predecessor row.
// The revised variant is one ISGMR iteration (test_baselines.cpp:58-68) and
// is served by mrf_isgmr_forward_f32 with K = 1.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "fwd_warp.cuh"
#include "launch.hpp"

namespace mrf {
namespace {

template <int EPL>
__global__ void __launch_bounds__(128) sgm_standard_kernel(Geometry g, Potentials pot, const LineDesc* __restrict__ lines,
                                                           int nlines, float* __restrict__ m) {
  extern __shared__ float smem[];
  const int L = g.L, N = g.N, R = g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  float* s_m = smem + wid * 32 * EPL;
  const int b = blockIdx.y;
  const float* un = pot.unary + size_t(b) * N * L;
  const int l0 = lane * EPL;
  for (int li = blockIdx.x * wpc + wid; li < nlines; li += gridDim.x * wpc) {
    const LineDesc ld = lines[li];
    const int r = ld.dir, st = g.node_step[r];
    float* mr = m + (size_t(b) * R + r) * N * L;
    // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r): the reference's vrow[mu]
    const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int l = l0 + i;
      carry[i] = l < L ? __ldg(un + size_t(ld.first) * L + l) : kInf;
      if (l < L) mr[size_t(ld.first) * L + l] = carry[i];
    }
    for (int j = 1; j < ld.length; ++j) {
      const int prev = ld.first + (j - 1) * st, cur = prev + st;
      const float w = plane_value(pot.w_planes, pot.w, N, R, b, r, prev, cur);
      // prev_min = min_mu m(prev, mu), first of equal values (the -0 sign kept)
      uint32_t kk = 0xffffffffu, kt = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (l0 + i < L) {
          const uint32_t k = order_key(fadd(carry[i], 0.0f));
          if (k < kk) kk = k, kt = (uint32_t(l0 + i) << 1) | (__float_as_uint(carry[i]) == 0x80000000u ? 1u : 0u);
        }
      }
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, kk);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, kk == kmin ? kt : 0xffffffffu);
      float prev_min = key_value(kmin);
      if (tmin & 1u) prev_min = -0.0f;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < EPL; ++i) s_m[l0 + i] = carry[i];
      __syncwarp();
      float best[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) best[i] = kInf;
      for (int mu = 0; mu < L; ++mu) {
        const float mm = s_m[mu];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int l = l0 + i < L ? l0 + i : 0;
          const float v = fadd(mm, fmul(w, __ldg(pot.V + mu * vs_mu + l * vs_l)));
          if (v < best[i]) best[i] = v;
        }
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int l = l0 + i;
        if (l < L) {
          carry[i] = fsub(fadd(__ldg(un + size_t(cur) * L + l), best[i]), prev_min);
          mr[size_t(cur) * L + l] = carry[i];
        } else {
          carry[i] = kInf;
        }
      }
    }
  }
}

template <int EPL>
cudaError_t run(const Geometry& g, const Potentials& pot, const LineDesc* lines, int nlines, float* m, int batch,
                cudaStream_t s) {
  const int wpc = 4;
  const int blocks = (nlines + wpc - 1) / wpc < 65535 ? (nlines + wpc - 1) / wpc : 65535;
  sgm_standard_kernel<EPL><<<dim3(blocks, batch), 32 * wpc, sizeof(float) * 32 * EPL * wpc, s>>>(g, pot, lines, nlines, m); note_launch();
  return cudaGetLastError();
}

// Iterated SGM's unary update (baselines.hpp:120-134): s(l) = sum_r m^r(l)
// (r ascending from +0), lo = min_l s(l) (std::min from +inf: first of equal
// values), next(l) = s(l) - lo. One warp per node.
__global__ void __launch_bounds__(256) sgm_next_unary_kernel(int N, int L, int R, const float* __restrict__ m,
                                                              float* __restrict__ next) {
  const int lane = threadIdx.x & 31;
  const int64_t node = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b = blockIdx.y;
  if (node >= N) return;
  const float* mb = m + size_t(b) * R * N * L + size_t(node) * L;
  float* nb = next + (size_t(b) * N + node) * L;
  float s[8];
  float lo = kInf;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int l = lane + 32 * i;
    s[i] = 0.0f;
    if (l < L) {
      for (int r = 0; r < R; ++r) s[i] = fadd(s[i], __ldcs(mb + size_t(r) * N * L + l));
      lo = s[i] < lo ? s[i] : lo;  // s is never -0 (+0 + x), so fminf order does not matter
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int l = lane + 32 * i;
    if (l < L) nb[l] = fsub(s[i], lo);
  }
}

}  // namespace

cudaError_t launch_sgm_next_unary(int B, int N, int L, int R, const float* messages, float* next, cudaStream_t s) {
  const int wpb = 8;
  sgm_next_unary_kernel<<<dim3(unsigned((int64_t(N) + wpb - 1) / wpb), unsigned(B)), 32 * wpb, 0, s>>>(N, L, R, messages,
                                                                                                      next);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_sgm_standard(const Geometry& g, const Potentials& pot, const LineDesc* lines, int nlines, float* m,
                                int batch, cudaStream_t s) {
  if (nlines == 0) return cudaSuccess;
  switch (epl_for(g.L)) {
    case 1: return run<1>(g, pot, lines, nlines, m, batch, s);
    case 2: return run<2>(g, pot, lines, nlines, m, batch, s);
    case 4: return run<4>(g, pot, lines, nlines, m, batch, s);
    case 6: return run<6>(g, pot, lines, nlines, m, batch, s);
    default: return run<8>(g, pot, lines, nlines, m, batch, s);
  }
}

}  // namespace mrf
