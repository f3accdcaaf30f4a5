// Forward sweep for small label sets with a dense (explicit) V, L <= 32
// (the segmentation config: 21 labels, learned 21x21 V, per-edge weights,
// batch 32), one warp per scanline, lane = label (sm_100a). The reference's
// min-plus (isgmr.hpp:98-131 / trwp.hpp:100-133) as written: for every
// label l the candidates mu = 0..L-1 in ascending order with strict '<',
// cost fl(base(mu) + fl(w V'(mu, l))) -- base(mu) comes from lane mu by a
// shuffle, V'(., l) is the lane's column of V (orientation r & 1) held in
// registers for the line, pre-multiplied by w once per line when w is
// constant. Then the reparametrisation's first argmin (-0 carried as in the
// reference) and m = out - min.
#pragma once

#include "fwd_warp.cuh"

namespace mrf {

// per-warp ring stage: ROWS rows of 32 floats + {w, rho}, padded to 16 B
__host__ __device__ constexpr int fwd_small_stage(int rows) { return rows * 32 + 4; }
// per-warp floats: the ring + base(mu) of the current node (32, 16 B aligned)
__host__ __device__ constexpr int fwd_small_warp_floats(int rows, int stages) { return stages * fwd_small_stage(rows) + 32; }

__device__ __forceinline__ uint64_t pack2f(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void unpack2f(uint64_t v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
// two IEEE round-to-nearest adds in one FADD2 (products stay scalar: ptxas
// would contract mul.rn.f32x2 + add.rn.f32x2 into FFMA2)
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// AGG (TRWP, last sweep only, every node on a line of that direction): the
// base sum s = theta + sum_d m^d at prev is that node's aggregated cost in
// the reference's order (inference.hpp:40-57), so the sweep also writes the
// cost row and the first-argmin label (the tail of each line at its end).
template <bool TRWP, int R, int LMAX, bool WPL, bool AGG = false>
__global__ void __launch_bounds__(128) fwd_small_kernel(FwdArgs a) {
  if (a.desc->banded || WPL != (a.pot.w_planes != nullptr)) return;  // another kernel owns the sweep
  extern __shared__ float smem[];
  constexpr int NP = TRWP ? R - 1 : R - 2;
  constexpr int ROWS = NP + 1;
  constexpr int STG = fwd_small_stage(ROWS);
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  float* ring = smem + size_t(wid) * fwd_small_warp_floats(ROWS, kStages);
  float* s_base = ring + kStages * STG;  // base(mu) of the current node, broadcast to every label
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int b = blockIdx.y;
  const bool valid = lane < L;
  const float* un = a.pot.unary + size_t(b) * N * L + lane;
  const size_t img = size_t(b) * R * N * L;
  constexpr bool wpl = WPL;
  const bool rpl = TRWP && a.pot.rho_planes != nullptr;
  const int l = valid ? lane : 0;
  int v_orient = -1;
  float vcol[LMAX], wv[LMAX];

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    if (v_orient != (r & 1)) {  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
      v_orient = r & 1;
#pragma unroll
      for (int mu = 0; mu < LMAX; ++mu)
        vcol[mu] = mu < L ? __ldg(a.pot.V + (v_orient ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
#pragma unroll
      for (int mu = 0; mu < LMAX; ++mu) wv[mu] = wpl ? 0.0f : fmul(a.pot.w, vcol[mu]);
    }
    float w_last = __uint_as_float(0xffffffffu);  // per-edge w of the cached products: none yet
    const float* rowp[ROWS];
    rowp[0] = un;
#pragma unroll
    for (int rr = 1; rr < ROWS; ++rr) {
      const int idx = rr - 1;
      const int d = TRWP ? (idx < r ? idx : idx + 1) : (idx < (r & ~1) ? idx : idx + 2);
      rowp[rr] = a.m_in + img + size_t(d) * N * L + lane;
    }
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    // incremental issue state (row pointers, ring slot, edge node) advanced
    // one node step per issue: no 64-bit index arithmetic per step
    const ptrdiff_t row_step = ptrdiff_t(st) * L;
#pragma unroll
    for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += ptrdiff_t(ld.first) * L;
    int islot = 0, wnode_i = (r & 1) ? ld.first + st : ld.first;
    auto issue = [&](int /*j*/) {
      const uint32_t base_s = ring_s + 4u * uint32_t(islot * STG);
      if (valid) {
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) cp_async_u32(base_s + 4u * (rr * 32 + lane), rowp[rr], 4);
      }
      if (wpl && lane == 0) cp_async_u32(base_s + 4u * (ROWS * 32), wrow + wnode_i, 4);
      if (rpl && lane == 1) cp_async_u32(base_s + 4u * (ROWS * 32 + 1), rrow + wnode_i, 4);
#pragma unroll
      for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += row_step;
      wnode_i += st;
      islot = islot == kStages - 1 ? 0 : islot + 1;
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (1 + s <= nsteps) issue(1 + s);
      cp_commit();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
    // output pointers at node step 1, advanced one step per node
    uint8_t* pout = a.p + pq_base * L + lane;
    uint8_t* qout = a.q + pq_base;
    float* mout = a.m_out + img + size_t(r) * N * L + lane + ptrdiff_t(ld.first + st) * L;
    float carry = 0.0f;
    int cslot = 0;
    // cost row + first argmin label of node n from its summed row c
    auto agg_row = [&](int n, float c) {
      const size_t nb = size_t(b) * N + n;
      if (a.agg_cost && valid) a.agg_cost[nb * L + lane] = c;
      const uint32_t kk = valid ? order_key(fadd(c, 0.0f)) : 0xffffffffu;
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, kk);
      const uint32_t lmin = __reduce_min_sync(0xffffffffu, kk == kmin ? uint32_t(lane) : 0xffffffffu);
      if (lane == 0 && a.agg_labels) a.agg_labels[nb] = uint16_t(lmin);
    };

    for (int j = 1; j <= nsteps; ++j) {
      if (j + kStages - 1 <= nsteps) issue(j + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      __syncwarp();  // the edge scalars were copied by lanes 0 / 1
      const float* srow = ring + cslot * STG + lane;
      cslot = cslot == kStages - 1 ? 0 : cslot + 1;
      // ---- base (isgmr.hpp:82-88 / trwp.hpp:84-90 addition order)
      float base;
      if (!TRWP) {
        base = fadd(srow[0], carry);
#pragma unroll
        for (int rr = 1; rr < ROWS; ++rr) base = fadd(base, srow[rr * 32]);
      } else {
        const float rho = rpl ? srow[ROWS * 32 + 1 - lane] : a.pot.rho;
        float s = srow[0], mo = 0.0f;
#pragma unroll
        for (int d = 0; d < R; ++d) {
          const float t = srow[(d < r ? d + 1 : (d > r ? d : 1)) * 32];
          mo = d == opp ? t : mo;
          s = fadd(s, d == r ? carry : t);
        }
        base = fsub(fmul(rho, s), mo);
        if (AGG) agg_row(ld.first + (j - 1) * st, s);
      }
      const float w = wpl ? srow[ROWS * 32 - lane] : 0.0f;
      if (wpl && __float_as_uint(w) != __float_as_uint(w_last)) {
        // per-edge weight: the products fl(w V'(mu, l)) of this lane's column,
        // recomputed only when w changes along the line (weight maps are
        // piecewise constant; bitwise compare, so -0 / NaN never alias)
        w_last = w;
#pragma unroll
        for (int mu = 0; mu < LMAX; ++mu) wv[mu] = fmul(w, vcol[mu]);
      }
      if (!valid) base = kInf;  // labels >= L never win (their V' column is 0)
      // ---- dense min-plus, ascending mu, strict '<': independent chains over
      // mu blocks of 8 (shorter dependency chains), merged in index order with
      // the earlier block winning ties. base(mu) comes from a 16-byte
      // broadcast load of the staged row (4 mu per load), two candidates
      // share one packed add.
      constexpr int NB = LMAX / 8;
      float bb[NB];
      int ba[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) bb[c] = kInf, ba[c] = 0;
      s_base[lane] = base;
      __syncwarp();
#pragma unroll
      for (int m4 = 0; m4 < LMAX; m4 += 4) {
        const ulonglong2 b4 = *reinterpret_cast<const ulonglong2*>(s_base + m4);
        float v[4];
        if (wpl) {
          unpack2f(fadd2(b4.x, pack2f(wv[m4], wv[m4 + 1])), v[0], v[1]);
          unpack2f(fadd2(b4.y, pack2f(wv[m4 + 2], wv[m4 + 3])), v[2], v[3]);
        } else {
          unpack2f(fadd2(b4.x, pack2f(wv[m4], wv[m4 + 1])), v[0], v[1]);
          unpack2f(fadd2(b4.y, pack2f(wv[m4 + 2], wv[m4 + 3])), v[2], v[3]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int mu = m4 + u, c = mu / 8;
          const bool p = v[u] < bb[c];
          bb[c] = p ? v[u] : bb[c];
          ba[c] = p ? mu : ba[c];
        }
      }
      float best = bb[0];
      int arg = ba[0];
#pragma unroll
      for (int c = 1; c < NB; ++c) {
        const bool p = bb[c] < best;
        best = p ? bb[c] : best;
        arg = p ? ba[c] : arg;
      }
      // ---- p, reparametrisation first argmin (lowest label, -0 as the reference)
      if (valid) *pout = uint8_t(arg);
      pout += L;
      const uint32_t lk = valid ? order_key(fadd(best, 0.0f)) : 0xffffffffu;
      const uint32_t lt = valid ? (uint32_t(lane) << 1) | (__float_as_uint(best) == 0x80000000u ? 1u : 0u) : 0xffffffffu;
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, lk);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, lk == kmin ? lt : 0xffffffffu);
      float lo = key_value(kmin);
      if (tmin & 1u) lo = -0.0f;
      carry = fsub(best, lo);
      if (valid) *mout = carry;
      mout += row_step;
      if (lane == 0) *qout = uint8_t(tmin >> 1);
      ++qout;
    }
    if (TRWP && AGG) {
      // the tail is no edge's prev: its cost from its rows and the final message
      const int tail = ld.first + nsteps * st;
      float c = valid ? __ldcg(a.pot.unary + (size_t(b) * N + tail) * L + lane) : 0.0f;
#pragma unroll
      for (int d = 0; d < R; ++d)
        c = fadd(c, d == r ? carry : (valid ? __ldcg(a.m_in + img + (size_t(d) * N + tail) * L + lane) : 0.0f));
      agg_row(tail, c);
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
