// Forward sweep specialised for banded pairwise terms with D == 2 (V(a,b) =
// g(|a-b|), g(d) = g(2) for d >= 2: truncated linear tau <= 2, Potts-like
// P1/P2, ... -- the stereo configurations C1-C3) and 4 / 8 directions.
//
// Same exact algorithm as the banded path of fwd_warp.cuh (see there), with
// everything the per-node chain touches kept in registers and shuffles:
// compile-time R unrolls the plane loops, FULL (L == 32*EPL) drops all
// per-label validity handling, invalid labels are carried as +inf instead of
// branches, and p bytes are packed into one store per lane.
#pragma once

#include "fwd_warp.cuh"

#ifndef MRF_BAND2_COOP
#define MRF_BAND2_COOP 1
#endif

namespace mrf {

__host__ __device__ constexpr int band2_smem_floats(int EPL, int rows, int stages = kStages) {
  return ((stages * rows + 1) * 32 * EPL + stages * 64 + 31) / 32 * 32;
}

// EPL bytes (one per label) -> one (or a few) packed stores at row + l0.
template <int EPL, bool FULL>
__device__ __forceinline__ void store_p(uint8_t* row, int l0, const int (&am)[EPL], int nvalid) {
  if (FULL && EPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 4) {
      const uint32_t w = uint32_t(am[i]) | (uint32_t(am[i + 1]) << 8) | (uint32_t(am[i + 2]) << 16) |
                         (uint32_t(am[i + 3]) << 24);
      *reinterpret_cast<uint32_t*>(row + l0 + i) = w;
    }
  } else if (FULL && EPL % 2 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2)
      *reinterpret_cast<uint16_t*>(row + l0 + i) = uint16_t(am[i] | (am[i + 1] << 8));
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i)
      if (FULL || i < nvalid) row[l0 + i] = uint8_t(am[i]);
  }
}

// aggregate_costs + argmin_labels (inference.hpp:25-57) of one node from its
// already summed cost row c = theta + sum_r m^r (r ascending).
template <int EPL, bool FULL>
__device__ __forceinline__ void agg_node(const FwdArgs& a, size_t node_row, size_t label_idx, const float (&c)[EPL],
                                         int l0, int nvalid, int L, int lane) {
  if (a.agg_cost) stg_slice<EPL>(a.agg_cost + node_row, l0, c, FULL ? EPL : nvalid, L);
  uint32_t bk = 0xffffffffu, bt = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const uint32_t kk = (FULL || i < nvalid) ? order_key(fadd(c[i], 0.0f)) : 0xffffffffu;
    const bool t = kk < bk;
    bk = t ? kk : bk;
    bt = t ? uint32_t(l0 + i) : bt;
  }
  const uint32_t kmin = __reduce_min_sync(0xffffffffu, bk);
  const uint32_t tmin = __reduce_min_sync(0xffffffffu, bk == kmin ? bt : 0xffffffffu);
  if (lane == 0 && a.agg_labels) a.agg_labels[label_idx] = uint16_t(tmin);
}

// AGG (TRWP, last sweep only): also aggregate cost / labels on the fly.
// RD >= 0: every line of the launch sweeps direction RD (TRWP launches one
// direction at a time), so the row selection below folds at compile time.
// ST: cp.async ring depth (ST - 1 node steps in flight).
template <int EPL, bool TRWP, int R, bool FULL, bool AGG = false, int RD = -1, int ST = kStages>
__global__ void __launch_bounds__(128) fwd_band2_kernel(FwdArgs a) {
  if (!(a.desc->banded && a.desc->D == 2)) return;  // fwd_warp_kernel handles it
  extern __shared__ float smem[];
  constexpr int NP = TRWP ? R - 1 : R - 2;
  constexpr int ROWS = NP + 1;
  constexpr int LS = 32 * EPL;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  float* ring = smem + size_t(wid) * band2_smem_floats(EPL, ROWS, ST);
  float* s_x = ring + ST * ROWS * LS;
  float* s_u = s_x + ST * 64;  // far-candidate costs of the current node
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t x_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_x));

  const int b = blockIdx.y;
  const float* un = a.pot.unary + size_t(b) * N * L;
  const size_t img = size_t(b) * R * N * L;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const float g0 = a.desc->g[0], g1 = a.desc->g[1], g2 = a.desc->g[2];
  float wg0 = fmul(a.pot.w, g0), wg1 = fmul(a.pot.w, g1), c = fmul(a.pot.w, g2);

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = RD >= 0 ? RD : ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    const float* rowp[ROWS];
    rowp[0] = un + l0;
#pragma unroll
    for (int rr = 1; rr < ROWS; ++rr) {
      const int idx = rr - 1;
      const int d = TRWP ? (idx < r ? idx : idx + 1) : (idx < (r & ~1) ? idx : idx + 2);
      rowp[rr] = a.m_in + img + size_t(d) * N * L + l0;
    }
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    // Issue of node step j's rows into ring slot (j-1) % ST. Short rows
    // (EPL <= 2) keep incremental state -- row pointers advanced one node
    // step per issue, slot counters -- which cuts the per-step index
    // arithmetic (C1 forward -9 %); at EPL >= 4 that form measured slower
    // (C2 +2 %: the lone-warp horizontal sweeps are scheduling-sensitive), so
    // those recompute the addresses.
    constexpr bool kIncIssue = EPL <= 2;
    // FULL rows at 6 labels per lane: whole-row 16-byte chunks (MRF_BAND2_COOP=0: per-lane slices)
    constexpr bool kCoopIssue = FULL && EPL == 6 && MRF_BAND2_COOP;
    const ptrdiff_t row_step = ptrdiff_t(st) * L;
    if (kIncIssue) {
#pragma unroll
      for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += ptrdiff_t(ld.first) * L;
    }
    int islot = 0, wnode_i = (r & 1) ? ld.first + st : ld.first;
    auto issue = [&](int j) {
      if constexpr (kIncIssue) {
        const uint32_t sbase = ring_s + 4u * uint32_t(islot * ROWS * LS + l0);
        if (FULL || nvalid > 0) {
#pragma unroll
          for (int rr = 0; rr < ROWS; ++rr) cp_slice_t<EPL, FULL>(sbase + 4u * uint32_t(rr * LS), rowp[rr], nvalid);
        }
        if (wpl) cp_async_u32(x_s + 4u * uint32_t(islot * 64 + lane), wrow + wnode_i, 4);
        if (rpl) cp_async_u32(x_s + 4u * uint32_t(islot * 64 + 32 + lane), rrow + wnode_i, 4);
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) rowp[rr] += row_step;
        wnode_i += st;
        islot = islot == ST - 1 ? 0 : islot + 1;
      } else {
        const int slot = (j - 1) % ST;
        const int prev = ld.first + (j - 1) * st;
        const size_t off = size_t(prev) * L;
        if (kCoopIssue) {
          // 16-byte chunks of the whole row, lanes = chunks (a lane's own 24-byte
          // slice would take three 8-byte copies); readers sync the warp
#pragma unroll
          for (int rr = 0; rr < ROWS; ++rr) {
            const float* src = rowp[rr] - l0 + off;
#pragma unroll
            for (int u = lane; u < 8 * EPL; u += 32)
              cp_async_u32(ring_s + 4u * uint32_t((slot * ROWS + rr) * LS + 4 * u), src + 4 * u, 16);
          }
        } else if (FULL || nvalid > 0) {
#pragma unroll
          for (int rr = 0; rr < ROWS; ++rr)
            cp_slice_t<EPL, FULL>(ring_s + 4u * uint32_t((slot * ROWS + rr) * LS + l0), rowp[rr] + off, nvalid);
        }
        const int wnode = (r & 1) ? prev + st : prev;
        if (wpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + lane), wrow + wnode, 4);
        if (rpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + 32 + lane), rrow + wnode, 4);
      }
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
      if (1 + s <= nsteps) issue(1 + s);
      cp_commit();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
    float* mout = a.m_out + img + size_t(r) * N * L;
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;

    int slot_c = 0;
    for (int j = 1; j <= nsteps; ++j) {
      if (j + ST - 1 <= nsteps) issue(j + ST - 1);
      cp_commit();
      cp_wait<ST - 1>();
      if (kCoopIssue) __syncwarp();  // rows were copied by other lanes
      const int slot = kIncIssue ? slot_c : (j - 1) % ST;  // ring slot of node step j
      slot_c = slot_c == ST - 1 ? 0 : slot_c + 1;
      const float* srow = ring + slot * ROWS * LS + l0;
      if (wpl) {
        const float w = s_x[slot * 64 + lane];
        wg0 = fmul(w, g0), wg1 = fmul(w, g1), c = fmul(w, g2);
      }

      // ---- base (isgmr.hpp:82-88 / trwp.hpp:84-90 addition order)
      float base[EPL];
      {
        float t[EPL];
        lds_slice<EPL>(t, srow);
        if (!TRWP) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) base[i] = fadd(t[i], carry[i]);
#pragma unroll
          for (int rr = 1; rr < ROWS; ++rr) {
            lds_slice<EPL>(t, srow + rr * LS);
#pragma unroll
            for (int i = 0; i < EPL; ++i) base[i] = fadd(base[i], t[i]);
          }
        } else {
          const float rho = rpl ? s_x[slot * 64 + 32 + lane] : a.pot.rho;
          float s[EPL], mo[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) s[i] = t[i], mo[i] = 0.0f;
#pragma unroll
          for (int d = 0; d < R; ++d) {
            lds_slice<EPL>(t, srow + (d < r ? d + 1 : d) * LS);  // d == r: unused read
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const float x = d == r ? carry[i] : t[i];
              mo[i] = d == opp ? t[i] : mo[i];
              s[i] = fadd(s[i], x);
            }
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) base[i] = fsub(fmul(rho, s[i]), mo[i]);
          // last sweep (r == R-1, carry = the new m^r): s is node prev's
          // aggregated cost in the reference's order
          if (AGG) {
            const int prev = ld.first + (j - 1) * st;
            agg_node<EPL, FULL>(a, (size_t(b) * N + prev) * L, size_t(b) * N + prev, s, l0, nvalid, L, lane);
          }
        }
      }
      if (!FULL) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) base[i] = i < nvalid ? base[i] : kInf;
      }

      // left / right far winners per label, two exact strategies:
      //  * EPL >= 4: warp prefix / suffix (value, first index) scans of u
      //    (few shuffle rounds per label, best when a lane owns many labels);
      //  * EPL <= 2: reductions around the global first argmin (below).
      float LV[EPL], RV[EPL], bl, br;
      int LI[EPL], RI[EPL];
      if constexpr (EPL >= 4) {
      // ---- far-candidate cost, prefix / suffix (value, first index) scans
      float u[EPL], pv[EPL], sv[EPL];
      int pi[EPL], si[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) u[i] = fadd(base[i], c);
      pv[0] = u[0];
      pi[0] = l0;
#pragma unroll
      for (int i = 1; i < EPL; ++i) {
        const bool t = u[i] < pv[i - 1];
        pv[i] = t ? u[i] : pv[i - 1];
        pi[i] = t ? l0 + i : pi[i - 1];
      }
      sv[EPL - 1] = u[EPL - 1];
      si[EPL - 1] = l0 + EPL - 1;
#pragma unroll
      for (int i = EPL - 2; i >= 0; --i) {
        const bool t = sv[i + 1] < u[i];
        sv[i] = t ? sv[i + 1] : u[i];
        si[i] = t ? si[i + 1] : l0 + i;
      }
      {
        float tpv = pv[EPL - 1], tsv = sv[0];
        int tpi = pi[EPL - 1], tsi = si[0];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float opv = __shfl_up_sync(0xffffffffu, tpv, off);
          const int opi = __shfl_up_sync(0xffffffffu, tpi, off);
          const float osv = __shfl_down_sync(0xffffffffu, tsv, off);
          const int osi = __shfl_down_sync(0xffffffffu, tsi, off);
          const bool tp = lane >= off && !(tpv < opv);
          const bool ts = lane + off < 32 && osv < tsv;
          tpv = tp ? opv : tpv;
          tpi = tp ? opi : tpi;
          tsv = ts ? osv : tsv;
          tsi = ts ? osi : tsi;
        }
        float epv = __shfl_up_sync(0xffffffffu, tpv, 1);
        const int epi = __shfl_up_sync(0xffffffffu, tpi, 1);
        float esv = __shfl_down_sync(0xffffffffu, tsv, 1);
        const int esi = __shfl_down_sync(0xffffffffu, tsi, 1);
        epv = lane > 0 ? epv : kInf;
        esv = lane < 31 ? esv : kInf;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const bool tp = !(pv[i] < epv);
          pv[i] = tp ? epv : pv[i];
          pi[i] = tp ? epi : pi[i];
          const bool ts = esv < sv[i];
          sv[i] = ts ? esv : sv[i];
          si[i] = ts ? esi : si[i];
        }
      }

      // ---- neighbours across lanes: base(l0-1), base(l0+EPL), far segment
      // summaries at l-2 / l+2 for the lane's first / last two labels
      bl = __shfl_up_sync(0xffffffffu, base[EPL - 1], 1);
      br = __shfl_down_sync(0xffffffffu, base[0], 1);
      bl = lane > 0 ? bl : kInf;
      br = lane < 31 ? br : kInf;
      constexpr int E2 = EPL >= 2 ? 2 : 1;  // labels per lane needing the neighbour's far summary
      constexpr int SH = EPL >= 2 ? 1 : 2;  // lane distance of l-2 / l+2
      float pvm[E2], svp[E2];
      int pim[E2], sip[E2];
#pragma unroll
      for (int e = 0; e < E2; ++e) {
        const int src_lo = EPL >= 2 ? EPL - 2 + e : 0;  // element l0 - 2 + e of lane - SH
        const int src_hi = EPL >= 2 ? e : 0;            // element l0 + EPL + e of lane + SH
        pvm[e] = __shfl_up_sync(0xffffffffu, pv[src_lo], SH);
        pim[e] = __shfl_up_sync(0xffffffffu, pi[src_lo], SH);
        svp[e] = __shfl_down_sync(0xffffffffu, sv[src_hi], SH);
        sip[e] = __shfl_down_sync(0xffffffffu, si[src_hi], SH);
        pvm[e] = lane >= SH ? pvm[e] : kInf;
        svp[e] = lane + SH < 32 ? svp[e] : kInf;
      }

#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        LV[i] = i >= 2 ? pv[i >= 2 ? i - 2 : 0] : pvm[i < E2 ? i : 0];
        LI[i] = i >= 2 ? pi[i >= 2 ? i - 2 : 0] : pim[i < E2 ? i : 0];
        const int hi = i + 2 - EPL;  // >= 0: right far summary lives in lane + SH
        RV[i] = hi < 0 ? sv[hi < 0 ? i + 2 : 0] : svp[hi >= 0 && hi < E2 ? hi : 0];
        RI[i] = hi < 0 ? si[hi < 0 ? i + 2 : 0] : sip[hi >= 0 && hi < E2 ? hi : 0];
      }
      } else {
      // ---- far candidates: u(mu) = fl(base(mu) + fl(w g(2))). With mu* the
      // global first argmin of u, every label l with |l - mu*| >= 2 has mu* in
      // its far set and no earlier index reaches u(mu*), so its far winner is
      // (u*, mu*) -- in the left segment when mu* < l (first in index order,
      // wins ties; the right segment can then never hold the first argmin)
      // or in the right one when mu* > l (the left can then never reach u*).
      // Only l in {mu*-1, mu*, mu*+1} need the prefix winners over [0, mu*-3],
      // [0, mu*-2], [0, mu*-1] and the suffix winners over [mu*+1, L),
      // [mu*+2, L), [mu*+3, L): two masked warp reductions plus four values.
      float u[EPL];
      uint32_t ku[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        u[i] = fadd(base[i], c);  // +inf on invalid labels (base +inf)
        ku[i] = order_key(u[i]);
        s_u[l0 + i] = u[i];
      }
      uint32_t mk = ku[0];
      int mi = l0;
#pragma unroll
      for (int i = 1; i < EPL; ++i) {
        const bool t = ku[i] < mk;
        mk = t ? ku[i] : mk;
        mi = t ? l0 + i : mi;
      }
      const uint32_t gk = __reduce_min_sync(0xffffffffu, mk);
      const int mstar = __reduce_min_sync(0xffffffffu, mk == gk ? mi : 0x7fffffff);
      const float ustar = key_value(gk);
      uint32_t pk = 0xffffffffu, sk = 0xffffffffu;
      int pix = 0x7fffffff, six = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int l = l0 + i;
        const bool tp = l <= mstar - 3 && ku[i] < pk;
        pk = tp ? ku[i] : pk;
        pix = tp ? l : pix;
        const bool ts = l >= mstar + 3 && ku[i] < sk;
        sk = ts ? ku[i] : sk;
        six = ts ? l : six;
      }
      const uint32_t pkm = __reduce_min_sync(0xffffffffu, pk);
      const uint32_t skm = __reduce_min_sync(0xffffffffu, sk);
      const int pim = __reduce_min_sync(0xffffffffu, pk == pkm ? pix : 0x7fffffff);
      const int sim = __reduce_min_sync(0xffffffffu, sk == skm ? six : 0x7fffffff);
      __syncwarp();
      const float um2 = mstar >= 2 ? s_u[mstar - 2] : kInf, um1 = mstar >= 1 ? s_u[mstar - 1] : kInf;
      const float up1 = mstar + 1 < L ? s_u[mstar + 1] : kInf, up2 = mstar + 2 < L ? s_u[mstar + 2] : kInf;
      // prefix winners P3, P2, P1 and suffix winners S3, S2, S1 (empty = +inf)
      const float P3v = pkm == 0xffffffffu ? kInf : key_value(pkm);
      const int P3i = pim;
      const bool t2 = um2 < P3v;
      const float P2v = t2 ? um2 : P3v;
      const int P2i = t2 ? mstar - 2 : P3i;
      const bool t1 = um1 < P2v;
      const float P1v = t1 ? um1 : P2v;
      const int P1i = t1 ? mstar - 1 : P2i;
      const float S3v = skm == 0xffffffffu ? kInf : key_value(skm);
      const int S3i = sim;
      const bool s2 = S3v < up2;  // earlier element wins ties
      const float S2v = s2 ? S3v : up2;
      const int S2i = s2 ? S3i : mstar + 2;
      const bool s1 = S2v < up1;
      const float S1v = s1 ? S2v : up1;
      const int S1i = s1 ? S2i : mstar + 1;
      __syncwarp();  // s_u reads done before the next node overwrites it

      // ---- neighbours across lanes for the near band: base(l0-1), base(l0+EPL)
      bl = __shfl_up_sync(0xffffffffu, base[EPL - 1], 1);
      br = __shfl_down_sync(0xffffffffu, base[0], 1);
      bl = lane > 0 ? bl : kInf;
      br = lane < 31 ? br : kInf;

#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int dl = l0 + i - mstar;
        float lv = dl >= 2 ? ustar : kInf, rv = dl <= -2 ? ustar : kInf;
        int lix = mstar, rix = mstar;
        lv = dl == -1 ? P3v : lv, lix = dl == -1 ? P3i : lix;
        lv = dl == 0 ? P2v : lv, lix = dl == 0 ? P2i : lix;
        lv = dl == 1 ? P1v : lv, lix = dl == 1 ? P1i : lix;
        rv = dl == -1 ? S1v : rv, rix = dl == -1 ? S1i : rix;
        rv = dl == 0 ? S2v : rv, rix = dl == 0 ? S2i : rix;
        rv = dl == 1 ? S3v : rv, rix = dl == 1 ? S3i : rix;
        LV[i] = lv, LI[i] = lix, RV[i] = rv, RI[i] = rix;
      }
      }

      // ---- combine in index order: [0,l-2] | l-1 | l | l+1 | [l+2,L)
      // (an infinite left summary -- l < 2 -- always loses to the finite
      // near candidates, so its index needs no masking)
      float out[EPL];
      int am[EPL];
      float nb[EPL];  // base + w g(1): the near candidate of both neighbouring labels
#pragma unroll
      for (int i = 0; i < EPL; ++i) nb[i] = fadd(base[i], wg1);
      const float nbl = fadd(bl, wg1), nbr = fadd(br, wg1);
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int l = l0 + i;
        const float lv = LV[i], rv = RV[i];
        const int lix = LI[i], rix = RI[i];
        float best = lv;
        int arg = lix;
        float v = i >= 1 ? nb[i >= 1 ? i - 1 : 0] : nbl;
        bool t = v < best;
        best = t ? v : best;
        arg = t ? l - 1 : arg;
        v = fadd(base[i], wg0);
        t = v < best;
        best = t ? v : best;
        arg = t ? l : arg;
        v = i + 1 < EPL ? nb[i + 1 < EPL ? i + 1 : 0] : nbr;
        t = v < best;
        best = t ? v : best;
        arg = t ? l + 1 : arg;
        t = rv < best;
        best = t ? rv : best;
        arg = t ? rix : arg;
        out[i] = (FULL || i < nvalid) ? best : kInf;
        am[i] = arg;
      }

      // ---- p row, reparametrisation (first argmin; banded values are never -0)
      store_p<EPL, FULL>(a.p + (pq_base + j - 1) * L, l0, am, nvalid);
      // lane minimum by fminf (exact: no candidate is NaN or -0, PairDesc),
      // its first position by equality, scanning down
      float lm = out[0];
#pragma unroll
      for (int i = 1; i < EPL; ++i) lm = fminf(lm, out[i]);
      int lidx = l0 + EPL - 1;
#pragma unroll
      for (int i = EPL - 2; i >= 0; --i) lidx = out[i] == lm ? l0 + i : lidx;
      const float lo = warp_min_f32(lm);
      const uint32_t qmin = __reduce_min_sync(0xffffffffu, lm == lo ? uint32_t(lidx) : 0xffffffffu);
#pragma unroll
      for (int i = 0; i < EPL; ++i) carry[i] = fsub(out[i], lo);
      const int cur = ld.first + j * st;
      stg_slice<EPL>(mout + size_t(cur) * L, l0, carry, FULL ? EPL : nvalid, L);
      if (lane == 0) a.q[pq_base + j - 1] = uint8_t(qmin);
    }
    if (TRWP && AGG) {
      // the tail is no edge's prev: its cost from its rows and the final message
      const int tail = ld.first + nsteps * st;
      float c[EPL], t[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) c[i] = (FULL || i < nvalid) ? __ldcg(un + size_t(tail) * L + l0 + i) : 0.0f;
#pragma unroll
      for (int d = 0; d < R; ++d) {
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          t[i] = d == r ? carry[i] : ((FULL || i < nvalid) ? __ldcg(a.m_in + img + (size_t(d) * N + tail) * L + l0 + i) : 0.0f);
#pragma unroll
        for (int i = 0; i < EPL; ++i) c[i] = fadd(c[i], t[i]);
      }
      agg_node<EPL, FULL>(a, (size_t(b) * N + tail) * L, size_t(b) * N + tail, c, l0, nvalid, L, lane);
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
