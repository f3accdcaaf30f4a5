// TRWP-4 forward sweep for small dense label sets, 16 < L <= 24 (the
// segmentation config C4: 21 labels, learned 21x21 V, per-edge weights,
// batch 32): 8 lanes per scanline, 3 labels per lane, 4 scanlines per warp
// (sm_100a).
//
// fwd_small.cuh maps lane = label, so at L = 21 eleven of 32 lanes idle
// through every per-label instruction and each warp carries one line's
// fixed per-step overhead. Here a lane owns labels l0 = 3 gl .. l0 + 2 of
// the line of its lane group (gi = lane / 8): 84 of 96 slots busy, and the
// per-step overhead (ring issue, waits, loop) is shared by four lines.
//
// Per node step the arithmetic is exactly fwd_small's (trwp.hpp:84-133 as
// written): base(mu) = fl(rho s - m_opp) with s summed in the reference's
// direction order, candidates fl(base(mu) + fl(w V'(mu, l))) for mu = 0..L-1
// ascending with strict '<' (the FMNMX3 minimum and the keyed first winner of
// fwd_small.cuh, the scan as written for zero, tiny and non-finite minima),
// the reparametrisation's first argmin with -0 carried, m = out - min, and
// with AGG the node's aggregated cost row and first-argmin label
// (inference.hpp:40-57). The minima over a line's labels are 8-lane xor
// shuffles instead of warp-wide CREDUX.
#pragma once

#include <type_traits>

#include "fwd_small.cuh"

namespace mrf {

constexpr int kGrpLanes = 8;                  // lanes per scanline
constexpr int kGrpLines = 32 / kGrpLanes;     // scanlines per warp
constexpr int kGrpStages = 4;                 // cp.async ring depth
#ifndef MRF_GRP_WARPS
#define MRF_GRP_WARPS 4
#endif
constexpr int kGrpWarps = MRF_GRP_WARPS;  // warps per CTA
// register budget: 3 CTAs of 4 warps per SM (168); -DMRF_GRP_MAXREG=n caps it instead (A/B)
#ifdef MRF_GRP_MAXREG
#define MRF_GRP_BOUNDS __maxnreg__(MRF_GRP_MAXREG)
#else
#define MRF_GRP_BOUNDS __launch_bounds__(128, 3)
#endif

// per warp floats: ring [stages][lines][R rows][8 EPL] + edge scalars
// [stages][lines][w, rho] + base(mu) [lines][8 EPL]
__host__ __device__ constexpr int fwd_grp_warp_floats(int rows, int EPL) {
  return kGrpStages * kGrpLines * rows * 8 * EPL + kGrpStages * kGrpLines * 2 + kGrpLines * 8 * EPL;
}
// V' block of one lane-in-group: [EPL targets][8 EPL mu], padded so that the
// 8 lanes' 16-byte reads hit disjoint banks (EPL = 3: stride 76)
__host__ __device__ constexpr int fwd_grp_vstride(int EPL) { return EPL * 8 * EPL + 4; }
__host__ __device__ constexpr int fwd_grp_cta_floats(int rows, int EPL, int wpc) {
  return 8 * fwd_grp_vstride(EPL) + wpc * fwd_grp_warp_floats(rows, EPL);
}

__device__ __forceinline__ float grp_min_f32(float v) {
  v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  v = fminf(v, __shfl_xor_sync(0xffffffffu, v, 2));
  return fminf(v, __shfl_xor_sync(0xffffffffu, v, 4));
}
__device__ __forceinline__ uint32_t grp_min_u32(uint32_t v) {
  v = min(v, __shfl_xor_sync(0xffffffffu, v, 1));
  v = min(v, __shfl_xor_sync(0xffffffffu, v, 2));
  return min(v, __shfl_xor_sync(0xffffffffu, v, 4));
}

// MU: candidates evaluated per label (L rounded up to even; labels in [MU, 8 EPL) are padding)
template <int EPL, int MU, bool WPL, bool AGG>
__global__ void MRF_GRP_BOUNDS fwd_grp_kernel(FwdArgs a) {
  if (a.desc->banded || WPL != (a.pot.w_planes != nullptr)) return;  // another kernel owns the sweep
  extern __shared__ __align__(16) float smem[];
  constexpr int R = 4, ROWS = R;  // theta + the three other directions' messages
  constexpr int LP = 8 * EPL;     // padded labels per line
  constexpr int STG = kGrpLines * ROWS * LP;
  constexpr int VS = fwd_grp_vstride(EPL);
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int gi = lane >> 3, gl = lane & 7, l0 = gl * EPL;
  const int nv = min(EPL, max(0, L - l0));  // this lane's valid labels
  float* s_v = smem;                        // [8][VS]: V'(mu, l0 + t) at [gl][t][mu]
  float* ring = smem + 8 * VS + size_t(wid) * fwd_grp_warp_floats(ROWS, EPL);
  float* s_sc = ring + kGrpStages * STG;             // [stages][lines][2]
  float* s_base = s_sc + kGrpStages * kGrpLines * 2;  // [lines][LP]
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t sc_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_sc));
  const int b = blockIdx.y;
  const size_t img = size_t(b) * R * N * L;
  const bool rpl = a.pot.rho_planes != nullptr;

  // every line of a TRWP launch sweeps a.dir: one V orientation
  const int orient = a.dir & 1;  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
  for (int t = threadIdx.x; t < 8 * EPL * LP; t += blockDim.x) {
    const int gg = t / (EPL * LP), rem = t - gg * (EPL * LP), tt = rem / LP, mu = rem - tt * LP;
    const int l = gg * EPL + tt;
    s_v[gg * VS + tt * LP + mu] =
        (l < L && mu < L) ? __ldg(a.pot.V + (orient ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
  }
  __syncthreads();
  // fl(w V'(mu, l0 + t)) as packed pairs (mu, mu + 1), in registers (they
  // outweigh occupancy: 7 CTAs per SM with V' re-read and multiplied per step
  // measured 38.5 ms per C4 forward against 34.5 here at 3)
  static_assert(MU % 2 == 0 && MU <= 8 * EPL, "MU: even, at most the padded label count");
  uint64_t wv2[EPL][MU / 2];
  auto products = [&](float w) {
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
#pragma unroll
      for (int m2 = 0; m2 < MU / 2; ++m2) {
        const float2 c = *reinterpret_cast<const float2*>(s_v + gl * VS + t * LP + 2 * m2);
        wv2[t][m2] = pack2f(fmul(w, c.x), fmul(w, c.y));
      }
    }
  };
  if (!WPL) products(a.pot.w);

  for (int wl = blockIdx.x * wpc + wid; wl * kGrpLines < a.nlines; wl += gridDim.x * wpc) {
    const int li = wl * kGrpLines + gi;
    const bool has = li < a.nlines;
    const LineDesc ld = a.lines[has ? li : wl * kGrpLines];
    const int nsteps = has ? ld.length - 1 : 0;
    int maxs = nsteps;
    maxs = max(maxs, __shfl_xor_sync(0xffffffffu, maxs, 8));
    maxs = max(maxs, __shfl_xor_sync(0xffffffffu, maxs, 16));

    auto sweep = [&](auto rd_tag) {
      constexpr int r = decltype(rd_tag)::value, opp = r ^ 1, fam = r >> 1;
      const int st = g.node_step[r];
      const float* rowp[ROWS];
      rowp[0] = a.pot.unary + size_t(b) * N * L + l0;
#pragma unroll
      for (int rr = 1; rr < ROWS; ++rr) {
        const int idx = rr - 1, d = idx < r ? idx : idx + 1;
        rowp[rr] = a.m_in + img + size_t(d) * N * L + l0;
      }
      const ptrdiff_t row_step = ptrdiff_t(st) * L;
#pragma unroll
      for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += ptrdiff_t(ld.first) * L;
      const float* wrow = WPL ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
      const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
      int islot = 0, wnode = (r & 1) ? ld.first + st : ld.first, issued = 0;
      auto issue = [&]() {
        ++issued;
        if (issued <= nsteps) {
          const uint32_t sb = ring_s + 4u * uint32_t(islot * STG + gi * ROWS * LP + l0);
#pragma unroll
          for (int rr = 0; rr < ROWS; ++rr) {
#pragma unroll
            for (int i = 0; i < EPL; ++i)
              if (i < nv) cp_async_u32(sb + 4u * uint32_t(rr * LP + i), rowp[rr] + i, 4);
          }
          const uint32_t xs = sc_s + 4u * uint32_t((islot * kGrpLines + gi) * 2);
          if (WPL && gl == 0) cp_async_u32(xs, wrow + wnode, 4);
          if (rpl && gl == 1) cp_async_u32(xs + 4u, rrow + wnode, 4);
        }
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += row_step;
        wnode += st;
        islot = islot == kGrpStages - 1 ? 0 : islot + 1;
      };
#pragma unroll
      for (int s = 0; s < kGrpStages - 1; ++s) {
        issue();
        cp_commit();
      }
      const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
      uint8_t* pout = a.p + pq_base * L + l0;
      uint8_t* qout = a.q + pq_base;
      float* mout = a.m_out + img + size_t(r) * N * L + l0 + ptrdiff_t(ld.first + st) * L;
      float carry[EPL];
#pragma unroll
      for (int t = 0; t < EPL; ++t) carry[t] = 0.0f;
      float w_last = __uint_as_float(0xffffffffu);  // per-edge w of the cached products: none yet
      int cslot = 0;
      // cost row + first argmin label of node n from its summed row c (all lanes call)
      auto agg_row = [&](bool act, int n, const float (&c)[EPL]) {
        const size_t nb = size_t(b) * N + n;
        float cn[EPL];
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          if (act && a.agg_cost && t < nv) a.agg_cost[nb * L + l0 + t] = c[t];
          cn[t] = t < nv ? fadd(c[t], 0.0f) : kInf;
        }
        float cm = cn[0];
#pragma unroll
        for (int t = 1; t < EPL; ++t) cm = fminf(cm, cn[t]);
        cm = grp_min_f32(cm);
        uint32_t lm = 0xffffffffu;
#pragma unroll
        for (int t = EPL - 1; t >= 0; --t) lm = cn[t] == cm ? uint32_t(l0 + t) : lm;
        lm = grp_min_u32(lm);
        if (act && gl == 0 && a.agg_labels) a.agg_labels[nb] = uint16_t(lm);
      };

      for (int j = 1; j <= maxs; ++j) {
        issue();
        cp_commit();
        cp_wait<kGrpStages - 1>();
        __syncwarp();  // the edge scalars were copied by lanes 0 / 1 of each group
        const bool act = j <= nsteps;
        const float* srow = ring + cslot * STG + gi * ROWS * LP + l0;
        const float* ssc = s_sc + (cslot * kGrpLines + gi) * 2;
        cslot = cslot == kGrpStages - 1 ? 0 : cslot + 1;
        // ---- base (trwp.hpp:84-90 addition order)
        const float rho = rpl ? ssc[1] : a.pot.rho;
        float s[EPL], base[EPL];
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          float sv = srow[t], mo = 0.0f;
#pragma unroll
          for (int d = 0; d < R; ++d) {
            const float x = d == r ? carry[t] : srow[(d < r ? d + 1 : d) * LP + t];
            if (d == opp) mo = x;
            sv = fadd(sv, x);
          }
          s[t] = sv;
          base[t] = t < nv ? fsub(fmul(rho, sv), mo) : kInf;  // labels >= L never win
        }
        if (AGG) agg_row(act, ld.first + (j - 1) * st, s);
        if (WPL) {
          const float w = ssc[0];
          // per-edge weight: products recomputed only when w changes along the
          // line (bitwise compare: -0 / NaN never alias)
          if (__float_as_uint(w) != __float_as_uint(w_last)) {
            w_last = w;
            products(w);
          }
        }
        // ---- base(mu) of the line to all its lanes: 16-byte broadcast reads
#pragma unroll
        for (int t = 0; t < EPL; ++t) s_base[gi * LP + l0 + t] = base[t];
        __syncwarp();
        // ---- per label: dense min-plus, first winner (fwd_small.cuh rules)
        uint64_t bp[MU / 2];
#pragma unroll
        for (int m4 = 0; m4 + 4 <= MU; m4 += 4) {
          const ulonglong2 b4 = *reinterpret_cast<const ulonglong2*>(s_base + gi * LP + m4);
          bp[m4 / 2] = b4.x, bp[m4 / 2 + 1] = b4.y;
        }
        if (MU % 4 == 2) bp[MU / 2 - 1] = *reinterpret_cast<const uint64_t*>(s_base + gi * LP + MU - 2);
        float best[EPL];
#pragma unroll
        for (int u = 0; u < EPL; ++u) best[u] = 0.0f;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          float v[MU], bt;
          int at;
#pragma unroll
          for (int m2 = 0; m2 < MU / 2; ++m2) unpack2f(fadd2(bp[m2], wv2[t][m2]), v[2 * m2], v[2 * m2 + 1]);
          float m0 = v[0], m1 = v[1];
#pragma unroll
          for (int mu = 2; mu < MU; mu += 2) m0 = fminf(m0, v[mu]), m1 = fminf(m1, v[mu + 1]);
          const float m = fminf(m0, m1);
          if (fabsf(m) >= 0x1p-60f && fabsf(m) < kInf) {
            const uint64_t mneg = pack2f(-m, -m);
            float k0 = kInf, k1 = kInf;
#pragma unroll
            for (int mu = 0; mu < MU; mu += 2) {
              float x, y;
              unpack2f(fadd2(fadd2(pack2f(v[mu], v[mu + 1]), mneg), kMuKey2[mu / 2]), x, y);
              k0 = fminf(k0, x), k1 = fminf(k1, y);
            }
            at = int(fmul(fminf(k0, k1), 0x1p90f));
            bt = m;
          } else {
            float bb = kInf;
            int aa = 0;
#pragma unroll
            for (int mu = 0; mu < MU; ++mu) {
              const bool p = v[mu] < bb;
              bb = p ? v[mu] : bb;
              aa = p ? mu : aa;
            }
            bt = bb, at = aa;
          }
          if (act && t < nv) pout[t] = uint8_t(at);
#pragma unroll
          for (int u = 0; u < EPL; ++u) best[u] = t == u ? bt : best[u];
        }
        // ---- p, reparametrisation first argmin (lowest label, -0 as the reference)
        float bn[EPL];
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          bn[t] = t < nv ? fadd(best[t], 0.0f) : kInf;  // -0 -> +0: no -0 reaches the float minimum
        }
        float bm = bn[0];
#pragma unroll
        for (int t = 1; t < EPL; ++t) bm = fminf(bm, bn[t]);
        bm = grp_min_f32(bm);
        uint32_t tk = 0xffffffffu;
#pragma unroll
        for (int t = EPL - 1; t >= 0; --t)
          tk = (t < nv && bn[t] == bm)
                   ? (uint32_t(l0 + t) << 1) | (__float_as_uint(best[t]) == 0x80000000u ? 1u : 0u)
                   : tk;
        tk = grp_min_u32(tk);
        const float lo = (tk & 1u) ? -0.0f : bm;
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          const float c = fsub(best[t], lo);
          carry[t] = act ? c : carry[t];
          if (act && t < nv) mout[t] = c;
        }
        if (act && gl == 0) *qout = uint8_t(tk >> 1);
        pout += L;
        mout += row_step;
        ++qout;
      }
      if (AGG) {
        // the tail is no edge's prev: its cost from its rows and the final message
        const int tail = ld.first + nsteps * st;
        float c[EPL];
#pragma unroll
        for (int t = 0; t < EPL; ++t) {
          const bool ok = has && t < nv;
          c[t] = ok ? __ldcg(a.pot.unary + (size_t(b) * N + tail) * L + l0 + t) : 0.0f;
#pragma unroll
          for (int d = 0; d < R; ++d)
            c[t] = fadd(c[t], d == r ? carry[t] : (ok ? __ldcg(a.m_in + img + (size_t(d) * N + tail) * L + l0 + t) : 0.0f));
        }
        agg_row(has, tail, c);
      }
    };
    switch (a.dir) {
      case 0: sweep(std::integral_constant<int, 0>()); break;
      case 1: sweep(std::integral_constant<int, 1>()); break;
      case 2: sweep(std::integral_constant<int, 2>()); break;
      default: sweep(std::integral_constant<int, 3>()); break;
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
