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

#include <type_traits>

#include "fwd_warp.cuh"

namespace mrf {

// per-warp ring stage: ROWS rows of 32 floats + {w, rho}, padded to 16 B
__host__ __device__ constexpr int fwd_small_stage(int rows) { return rows * 32 + 4; }
// per-warp floats: the ring + base(mu) of the current node (32, 16 B aligned)
// + with per-edge weights the lane's V' column [LMAX][32] (read only when w
// changes: 24 registers fewer in the node loop)
__host__ __device__ constexpr int fwd_small_warp_floats(int rows, int stages, int vcols = 0) {
  return stages * fwd_small_stage(rows) + 32 + vcols * 32;
}

// mu 2^-90 for mu = 0..31 as float pairs: the first-winner key offsets
// (constant bank, not const: loaded once into uniform registers, which FADD2
// reads as operands; a const array is folded into per-use UMOVs)
__constant__ uint64_t kMuKey2[16] = {
#define MRF_MK(mu) (uint64_t(__builtin_bit_cast(uint32_t, float(mu) * 0x1p-90f)) | \
                    (uint64_t(__builtin_bit_cast(uint32_t, float(mu + 1) * 0x1p-90f)) << 32))
    MRF_MK(0),  MRF_MK(2),  MRF_MK(4),  MRF_MK(6),  MRF_MK(8),  MRF_MK(10), MRF_MK(12), MRF_MK(14),
    MRF_MK(16), MRF_MK(18), MRF_MK(20), MRF_MK(22), MRF_MK(24), MRF_MK(26), MRF_MK(28), MRF_MK(30)};
#undef MRF_MK

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
  float* ring = smem + size_t(wid) * fwd_small_warp_floats(ROWS, kStages, WPL ? LMAX : 0);
  float* s_base = ring + kStages * STG;  // base(mu) of the current node, broadcast to every label
  float* s_vcol = s_base + 32;           // WPL: V'(mu, lane) at [mu][lane]
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const int b = blockIdx.y;
  const bool valid = lane < L;
  const float* un = a.pot.unary + size_t(b) * N * L + lane;
  const size_t img = size_t(b) * R * N * L;
  constexpr bool wpl = WPL;
  const bool rpl = TRWP && a.pot.rho_planes != nullptr;
  const int l = valid ? lane : 0;
  int v_orient = -1;
  float wv[LMAX];

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    if (v_orient != (ld.dir & 1)) {  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
      v_orient = ld.dir & 1;
#pragma unroll
      for (int mu = 0; mu < LMAX; ++mu) {
        const float vc = mu < L ? __ldg(a.pot.V + (v_orient ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
        if (wpl) s_vcol[mu * 32 + lane] = vc;
        wv[mu] = wpl ? 0.0f : fmul(a.pot.w, vc);
      }
    }
    // the line body with the direction a compile-time constant where TRWP's
    // addition order depends on it (R == 4: every row offset and select of
    // the base sum static), else the runtime direction
    auto sweep = [&](auto rd_tag) {
    constexpr int RD = decltype(rd_tag)::value;
    const int r = RD >= 0 ? RD : ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
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
      const float cn = valid ? fadd(c, 0.0f) : kInf;
      const float cmin = warp_min_f32(cn);
      const uint32_t lmin = __reduce_min_sync(0xffffffffu, cn == cmin ? uint32_t(lane) : 0xffffffffu);
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
        for (int mu = 0; mu < LMAX; ++mu) wv[mu] = fmul(w, s_vcol[mu * 32 + lane]);
      }
      if (!valid) base = kInf;  // labels >= L never win (their V' column is 0)
      // ---- dense min-plus candidates fl(base(mu) + fl(w V'(mu, l))): base(mu)
      // from a 16-byte broadcast load of the staged row (4 mu per load), two
      // candidates per packed add
      s_base[lane] = base;
      __syncwarp();
      float v[LMAX];
#pragma unroll
      for (int m4 = 0; m4 < LMAX; m4 += 4) {
        const ulonglong2 b4 = *reinterpret_cast<const ulonglong2*>(s_base + m4);
        unpack2f(fadd2(b4.x, pack2f(wv[m4], wv[m4 + 1])), v[m4], v[m4 + 1]);
        unpack2f(fadd2(b4.y, pack2f(wv[m4 + 2], wv[m4 + 3])), v[m4 + 2], v[m4 + 3]);
      }
      // ---- the reference's ascending strict-'<' scan, restated: its winner is
      // the FIRST mu whose candidate equals the minimum m (FMNMX3 tree: m is
      // one of the candidates, bit for bit). For finite |m| >= 2^-60 every
      // other candidate differs from m by >= 2^-84, so the key fl(fl(v - m) +
      // mu 2^-90) is exactly mu 2^-90 where v == m and >= 2^-84 elsewhere:
      // min(key) names the first winner with no per-candidate compare/select
      // (two packed adds and half an FMNMX3 per candidate, FMA pipe heavy).
      // m == +-0 (sign of the first winner), +inf / NaN (no winner: label 0,
      // value +inf) and tiny m take the scan as written.
      float m0 = v[0], m1 = v[1];
#pragma unroll
      for (int mu = 2; mu < LMAX; mu += 2) m0 = fminf(m0, v[mu]), m1 = fminf(m1, v[mu + 1]);
      const float m = fminf(m0, m1);
      float best;
      int arg;
      if (fabsf(m) >= 0x1p-60f && fabsf(m) < kInf) {
        const uint64_t mneg = pack2f(-m, -m);
        float k0 = kInf, k1 = kInf;
#pragma unroll
        for (int mu = 0; mu < LMAX; mu += 2) {
          float x, y;
          unpack2f(fadd2(fadd2(pack2f(v[mu], v[mu + 1]), mneg), kMuKey2[mu / 2]), x, y);
          k0 = fminf(k0, x), k1 = fminf(k1, y);
        }
        arg = int(fmul(fminf(k0, k1), 0x1p90f));
        best = m;
      } else {
        best = kInf, arg = 0;
#pragma unroll
        for (int mu = 0; mu < LMAX; ++mu) {
          const bool p = v[mu] < best;
          best = p ? v[mu] : best;
          arg = p ? mu : arg;
        }
      }
      // ---- p, reparametrisation first argmin (lowest label, -0 as the reference)
      if (valid) *pout = uint8_t(arg);
      pout += L;
      const float bn = valid ? fadd(best, 0.0f) : kInf;  // -0 -> +0: no -0 reaches the float minimum
      const uint32_t lt = valid ? (uint32_t(lane) << 1) | (__float_as_uint(best) == 0x80000000u ? 1u : 0u) : 0xffffffffu;
      const float bmin = warp_min_f32(bn);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, bn == bmin ? lt : 0xffffffffu);
      const float lo = (tmin & 1u) ? -0.0f : bmin;
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
    };
    if constexpr (TRWP && R == 4) {
      switch (ld.dir) {
        case 0: sweep(std::integral_constant<int, 0>()); break;
        case 1: sweep(std::integral_constant<int, 1>()); break;
        case 2: sweep(std::integral_constant<int, 2>()); break;
        default: sweep(std::integral_constant<int, 3>()); break;
      }
    } else {
      sweep(std::integral_constant<int, -1>());
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
