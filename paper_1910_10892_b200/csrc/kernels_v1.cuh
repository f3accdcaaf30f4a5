// Generic dense sweep kernels: one CTA walks one scanline, one thread per
// label. These cover every V (explicit tables, any L <= 256) and are the
// parity baseline for the specialised kernels.
#pragma once

#include "common.cuh"

namespace mrf {

// Table modes for the L x L pairwise term.
enum TableMode : int {
  kTabWV = 0,     // smem holds fl(w * V'(mu,l)) (constant w)
  kTabV = 1,      // smem holds V'(mu,l); w per edge, fl(w * V') per candidate
  kTabGlobal = 2  // V read from global (L too large for smem)
};

__device__ __forceinline__ float vprime_global(const float* V, int L, int r, int mu, int l) {
  return __ldg(V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l));
}

// Forward sweep (ISGMR Alg. 1 / TRWP Alg. 2 inner loop; isgmr.hpp:71-133,
// trwp.hpp:71-135). Thread t owns label l = t for the min-plus and mu = t for
// the base assembly, so the carried message m^r_prev stays in a register.
template <bool TRWP>
__global__ void __launch_bounds__(256) fwd_dense_kernel(Geometry g, Potentials pot, const LineDesc* __restrict__ lines,
                                                        int nlines, const float* m_in, float* m_out,
                                                        uint8_t* __restrict__ p, uint8_t* __restrict__ q, int k,
                                                        int table_mode) {
  extern __shared__ float smem[];
  const int L = g.L, N = g.N, R = g.R;
  float* s_base = smem;
  uint32_t* s_key = reinterpret_cast<uint32_t*>(smem + 256);
  uint32_t* s_idx = s_key + 8;
  float* s_tab = smem + 256 + 16;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int b = blockIdx.y;
  const bool own = tid < L;
  const float* un = pot.unary + size_t(b) * N * L;
  const size_t img = size_t(b) * R * N * L;
  int tab_parity = -1;

  for (int li = blockIdx.x; li < nlines; li += gridDim.x) {
    const LineDesc ld = lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r];
    if (table_mode != kTabGlobal && tab_parity != (r & 1)) {
      __syncthreads();
      for (int i = tid; i < L * L; i += blockDim.x) {
        const int mu = i / L, l = i - mu * L;
        const float v = vprime_global(pot.V, L, r, mu, l);
        s_tab[i] = table_mode == kTabWV ? fmul(pot.w, v) : v;
      }
      tab_parity = r & 1;
      __syncthreads();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + k) * g.E + g.dir_offset[r] + ld.edge_base;
    float carry = 0.0f;  // m^r (TRWP) / mhat^r (ISGMR) of the previous node, label tid
    for (int j = 1; j < ld.length; ++j) {
      const int prev = ld.first + (j - 1) * st, cur = prev + st;
      if (own) {
        const int mu = tid;
        float bse;
        if (!TRWP) {
          // ((theta + mhat^r) + m^d1) + m^d2 ..., d ascending, d not in {r, r-} (isgmr.hpp:82-88)
          bse = fadd(__ldg(un + size_t(prev) * L + mu), carry);
          for (int d = 0; d < R; ++d) {
            if (d == r || d == opp) continue;
            bse = fadd(bse, m_in[img + (size_t(d) * N + prev) * L + mu]);
          }
        } else {
          // s = theta + sum_d m^d (fresh m^r carried); base = rho*s - m^{r-} (trwp.hpp:84-90)
          float s = __ldg(un + size_t(prev) * L + mu), mo = 0.0f;
          for (int d = 0; d < R; ++d) {
            const float md = d == r ? carry : m_in[img + (size_t(d) * N + prev) * L + mu];
            if (d == opp) mo = md;
            s = fadd(s, md);
          }
          const float rho = plane_value(pot.rho_planes, pot.rho, N, R, b, r, prev, cur);
          bse = fsub(fmul(rho, s), mo);
        }
        s_base[mu] = bse;
      }
      __syncthreads();

      uint32_t key = 0xffffffffu, tag = 0xffffffffu;
      float out = 0.0f;
      if (own) {
        const int l = tid;
        const float w = plane_value(pot.w_planes, pot.w, N, R, b, r, prev, cur);
        float best = __int_as_float(0x7f800000);
        int arg = 0;
        for (int mu = 0; mu < L; ++mu) {
          float wv;
          if (table_mode == kTabWV) wv = s_tab[mu * L + l];
          else if (table_mode == kTabV) wv = fmul(w, s_tab[mu * L + l]);
          else wv = fmul(w, vprime_global(pot.V, L, r, mu, l));
          const float v = fadd(s_base[mu], wv);
          if (v < best) {
            best = v;
            arg = mu;
          }
        }
        out = best;
        p[(pq_base + j - 1) * L + l] = uint8_t(arg);
        key = order_key(fadd(best, 0.0f));
        tag = (uint32_t(l) << 1) | (__float_as_uint(best) == 0x80000000u ? 1u : 0u);
      }
      // reparametrisation argmin (isgmr.hpp:118-131): lowest label wins ties
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, key);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, key == kmin ? tag : 0xffffffffu);
      if (lane == 0) {
        s_key[wid] = kmin;
        s_idx[wid] = tmin;
      }
      __syncthreads();
      uint32_t bk = s_key[0], bt = s_idx[0];
      for (int w = 1; w < nw; ++w) {
        const uint32_t kw = s_key[w], tw = s_idx[w];
        if (kw < bk || (kw == bk && tw < bt)) {
          bk = kw;
          bt = tw;
        }
      }
      float lo = key_value(bk);
      if (bt & 1u) lo = -0.0f;
      if (own) {
        out = fsub(out, lo);
        m_out[img + (size_t(r) * N + cur) * L + tid] = out;
        carry = out;
      }
      if (tid == 0) q[pq_base + j - 1] = uint8_t(bt >> 1);
    }
  }
}

// c = theta + sum_r m^r (r ascending) and labels = first argmin
// (inference.hpp:25-57). One warp per node.
__global__ void aggregate_kernel(int B, int N, int L, int R, const float* __restrict__ unary,
                                 const float* __restrict__ m, float* __restrict__ cost, uint16_t* __restrict__ labels) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gw >= int64_t(B) * N) return;
  const int b = int(gw / N), i = int(gw - int64_t(b) * N);
  const size_t row = (size_t(b) * N + i) * L;
  uint32_t best_k = 0xffffffffu, best_t = 0xffffffffu;
  for (int l = lane; l < L; l += 32) {
    float c = __ldg(unary + row + l);
    for (int r = 0; r < R; ++r) c = fadd(c, __ldg(m + ((size_t(b) * R + r) * N + i) * L + l));
    if (cost) cost[row + l] = c;
    const uint32_t kk = order_key(fadd(c, 0.0f));
    if (kk < best_k) {
      best_k = kk;
      best_t = uint32_t(l);
    }
  }
  const uint32_t kmin = __reduce_min_sync(0xffffffffu, best_k);
  const uint32_t tmin = __reduce_min_sync(0xffffffffu, best_k == kmin ? best_t : 0xffffffffu);
  if (lane == 0 && labels) labels[size_t(b) * N + i] = uint16_t(tmin);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Backward sweep for one direction r (isgmr_backward autodiff.hpp:83-118,
// trwp_backward :152-186): nodes in reverse, reparam backward, then the
// index-driven scatter. Thread t owns label l = t of the current row and
// mu = t of the predecessor row, so the in-flight chain gradient gm^r_prev
// stays in a register. Scatter targets are aggregated per mu in shared
// memory before one read-modify-write per row element.
// vslots: [B][G][2][L][L] private dV partials (even / odd orientation),
// G >= gridDim.x slot columns per image, column blockIdx.x written only by
// CTA (blockIdx.x, b): no atomics.
template <bool TRWP>
__global__ void __launch_bounds__(256) bwd_dense_kernel(Geometry g, Potentials pot, const LineDesc* __restrict__ lines,
                                                        int nlines, int r, const uint8_t* __restrict__ p,
                                                        const uint8_t* __restrict__ q, int k, float* gm, float* gnext,
                                                        float* gu, float* gw, float* vslots, int G) {
  __shared__ float s_acc[256];
  __shared__ float s_sum[8];
  __shared__ float s_wp[8];
  const int L = g.L, N = g.N, R = g.R;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int b = blockIdx.y;
  const bool own = tid < L;
  const int opp = r ^ 1, st = g.node_step[r];
  const size_t img = size_t(b) * R * N * L;
  float* gr = gm + img + size_t(r) * N * L;
  float* slot = vslots + ((size_t(b) * G + blockIdx.x) * 2 + (r & 1)) * L * L;
  if (own) s_acc[tid] = 0.0f;
  __syncthreads();

  for (int li = blockIdx.x; li < nlines; li += gridDim.x) {
    const LineDesc ld = lines[li];
    const size_t pq_base = (size_t(b) * g.K_cap + k) * g.E + g.dir_offset[r] + ld.edge_base;
    float carry = 0.0f;
    for (int j = ld.length - 1; j >= 1; --j) {
      const int cur = ld.first + j * st, prev = cur - st;
      const size_t e = pq_base + j - 1;
      float row = 0.0f;
      if (own) row = fadd(gr[size_t(cur) * L + tid], carry);
      const float ws = warp_sum(row);
      if (lane == 0) s_sum[wid] = ws;
      __syncthreads();
      float S = s_sum[0];
      for (int w = 1; w < nw; ++w) S = fadd(S, s_sum[w]);
      const float w = plane_value(pot.w_planes, pot.w, N, R, b, r, prev, cur);
      float wpart = 0.0f;
      if (own) {
        const int l = tid;
        if (l == int(q[e])) row = fsub(row, S);  // reparam backward (autodiff.hpp:48-53)
        if (row != 0.0f) {
          const int mu = p[e * L + l];
          atomicAdd(&s_acc[mu], row);
          const float vv = (r & 1) ? __ldg(pot.V + size_t(l) * L + mu) : __ldg(pot.V + size_t(mu) * L + l);
          wpart = fmul(row, vv);
          float* sp = slot + size_t(mu) * L + l;
          *sp = fadd(*sp, fmul(row, w));
        }
      }
      wpart = warp_sum(wpart);
      if (lane == 0) s_wp[wid] = wpart;
      __syncthreads();
      if (own) {
        const int mu = tid;
        const float a = s_acc[mu];
        s_acc[mu] = 0.0f;
        const size_t pm = size_t(prev) * L + mu;
        float* gub = gu + size_t(b) * N * L;
        if (!TRWP) {
          gub[pm] = fadd(gub[pm], a);
          for (int d = 0; d < R; ++d) {
            if (d == r || d == opp) continue;
            float* t = gnext + img + size_t(d) * N * L + pm;
            *t = fadd(*t, a);
          }
          carry = a;
        } else {
          const float rho = plane_value(pot.rho_planes, pot.rho, N, R, b, r, prev, cur);
          const float ra = fmul(rho, a);
          gub[pm] = fadd(gub[pm], ra);
          for (int d = 0; d < R; ++d) {
            if (d == r) continue;
            float* t = gm + img + size_t(d) * N * L + pm;
            float v = fadd(*t, ra);
            if (d == opp) v = fsub(v, a);
            *t = v;
          }
          carry = ra;
        }
      }
      if (tid == 0 && gw) {
        float wsum = s_wp[0];
        for (int w2 = 1; w2 < nw; ++w2) wsum = fadd(wsum, s_wp[w2]);
        const int wnode = (r & 1) ? cur : prev;
        float* t = gw + (size_t(b) * (R / 2) + (r >> 1)) * N + wnode;
        *t = fadd(*t, wsum);
      }
    }
  }
}

// dV[b][a][c] = sum_s even[b][s][a][c] + odd[b][s][c][a], slots in fixed order.
__global__ void reduce_vslots_kernel(int B, int G, int L, const float* __restrict__ vslots, float* __restrict__ gv) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t LL = int64_t(L) * L;
  if (i >= B * LL) return;
  const int b = int(i / LL);
  const int ac = int(i - b * LL), a = ac / L, c = ac - a * L;
  float s = 0.0f;
  for (int sl = 0; sl < G; ++sl) {
    const float* base = vslots + (size_t(b) * G + sl) * 2 * LL;
    s = fadd(s, base[ac]);
    s = fadd(s, base[LL + size_t(c) * L + a]);
  }
  gv[i] = s;
}

// dst[b][r][:] = src[b][:] for r in [0, R): the gm <- dc initialisation.
__global__ void broadcast_planes_kernel(int B, int R, int64_t NL, const float* __restrict__ src, float* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(B) * R * NL) return;
  const int64_t b = i / (R * NL);
  const int64_t rem = i - b * R * NL;
  dst[i] = src[b * NL + rem % NL];
}

// make_gradients + gm init (autodiff.hpp:33-44, :72-74) in one pass:
// gu[b] = dc[b] and gm[b][r] = dc[b] for every r. float4 body (NL % 4 == 0),
// grid-stride over (image, chunk); one read of dc, R+1 writes.
__global__ void init_grads_kernel(int B, int R, int64_t NL4, const float4* __restrict__ gc, float4* __restrict__ gu,
                                  float4* __restrict__ gm) {
  const int64_t total = int64_t(B) * NL4;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = i / NL4, x = i - b * NL4;
    const float4 v = __ldcs(gc + i);
    __stcs(gu + i, v);
    float4* dst = gm + b * R * NL4 + x;
    for (int r = 0; r < R; ++r) __stcs(dst + r * NL4, v);
  }
}

}  // namespace mrf
