// Forward sweep for banded pairwise terms with 2 < D <= DW (sm_100a): the
// truncated quadratic of the denoising config (V = min(d^2, 200): D = 15),
// truncated linear with tau > 2, ... Same exact restatement of the
// reference's ascending strict-'<' scan (isgmr.hpp:98-131, trwp.hpp:100-133)
// as fwd_band2.cuh -- left far segment [0, l-D] (first argmin of u = base +
// w g(D), warp prefix scan), the band mu in (l-D, l+D) explicitly, right far
// segment [l+D, L) (suffix scan), combined in index order -- but the band is
// evaluated from a register window instead of per-candidate shared-memory
// loads: per node step the warp stores its base row once into a padded
// per-warp row (lane stride EPL+1 words: conflict-free), each lane loads
// base(l0-DW+1 .. l0+EPL+DW-2) into registers, and every label runs its
// 2DW-1 taps (t = mu - l) out of registers with the scaled band table
// wg[|t|] = w g(|t|) for |t| < D and +inf beyond (those candidates belong to
// the far segments, which already hold them in the same index order).
#pragma once

#include "fwd_band2.cuh"

namespace mrf {

// per-warp shared memory (floats): ring [kStages][rows][32*EPL], edge scalars
// [kStages][64], padded base row, far summaries pv / sv, their indices (u8)
template <int EPL, int DW>
struct BandwSmem {
  static constexpr int M = (DW + EPL - 1) / EPL * EPL;       // left margin (labels), multiple of EPL
  static constexpr int NB = (32 * EPL + 2 * M) / EPL * (EPL + 1);  // padded base row
  static __host__ __device__ constexpr int idx(int l) { return (l + M) + (l + M) / EPL; }
};
__host__ __device__ constexpr int bandw_smem_floats(int EPL, int DW, int rows) {
  return ((kStages * rows + 2) * 32 * EPL + kStages * 64 + ((32 * EPL + 2 * ((DW + EPL - 1) / EPL * EPL)) / EPL) * (EPL + 1) +
          (2 * 32 * EPL + 3) / 4 + 31) / 32 * 32;
}

template <int EPL, bool TRWP, int R, bool FULL, int DW>
__global__ void __launch_bounds__(128) fwd_bandw_kernel(FwdArgs a) {
  const int D = a.desc->D;
  if (!(a.desc->banded && D > 2 && D <= DW)) return;  // another kernel owns the sweep
  extern __shared__ float smem[];
  using SM = BandwSmem<EPL, DW>;
  constexpr int NP = TRWP ? R - 1 : R - 2;
  constexpr int ROWS = NP + 1;
  constexpr int LS = 32 * EPL;
  constexpr int NWIN = EPL + 2 * DW - 2;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  float* ring = smem + size_t(wid) * bandw_smem_floats(EPL, DW, ROWS);
  float* s_x = ring + kStages * ROWS * LS;
  float* s_base = s_x + kStages * 64;  // padded, SM::NB
  float* s_pv = s_base + SM::NB;
  float* s_sv = s_pv + LS;
  uint8_t* s_pi = reinterpret_cast<uint8_t*>(s_sv + LS);
  uint8_t* s_si = s_pi + LS;
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t x_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_x));

  const int b = blockIdx.y;
  const float* un = a.pot.unary + size_t(b) * N * L;
  const size_t img = size_t(b) * R * N * L;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const float* gt = a.desc->g;
  // labels outside [0, L) read +inf from the padded row: fill it once
  for (int t = lane; t < SM::NB; t += 32) s_base[t] = kInf;
  __syncwarp();
  // scaled band table: wg[t] = w g(t) for t < D, +inf for D <= t < DW; c = w g(D)
  float wgt[DW];
  float c;
  auto scale = [&](float w) {
#pragma unroll
    for (int t = 0; t < DW; ++t) wgt[t] = t < D ? fmul(w, gt[t]) : kInf;
    c = fmul(w, gt[D]);
  };
  scale(a.pot.w);

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
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
    auto issue = [&](int j) {
      const int slot = (j - 1) % kStages;
      const int prev = ld.first + (j - 1) * st;
      const size_t off = size_t(prev) * L;
      if (FULL || nvalid > 0) {
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr)
          cp_slice_t<EPL, FULL>(ring_s + 4u * uint32_t((slot * ROWS + rr) * LS + l0), rowp[rr] + off, nvalid);
      }
      const int wnode = (r & 1) ? prev + st : prev;
      if (wpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + lane), wrow + wnode, 4);
      if (rpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + 32 + lane), rrow + wnode, 4);
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (1 + s <= nsteps) issue(1 + s);
      cp_commit();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
    float* mout = a.m_out + img + size_t(r) * N * L;
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;

    for (int j = 1; j <= nsteps; ++j) {
      if (j + kStages - 1 <= nsteps) issue(j + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      const int slot = (j - 1) % kStages;
      const float* srow = ring + slot * ROWS * LS + l0;
      if (wpl) scale(s_x[slot * 64 + lane]);

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
        }
      }
      if (!FULL) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) base[i] = i < nvalid ? base[i] : kInf;
      }

      // ---- far segments: warp prefix / suffix (value, first index) scans of u
      float pv[EPL], sv[EPL];
      int pi[EPL], si[EPL];
      {
        float u[EPL];
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

      // ---- publish base (padded) and the far summaries; gather the window
      __syncwarp();  // the previous step's reads are done
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        s_base[SM::idx(l0 + i)] = base[i];
        s_pv[l0 + i] = pv[i];
        s_sv[l0 + i] = sv[i];
        s_pi[l0 + i] = uint8_t(pi[i]);
        s_si[l0 + i] = uint8_t(si[i]);
      }
      __syncwarp();
      float win[NWIN];
#pragma unroll
      for (int k = 0; k < NWIN; ++k) win[k] = s_base[SM::idx(l0 - (DW - 1) + k)];

      // ---- per label: [0, l-D] | band mu = l-DW+1 .. l+DW-1 | [l+D, L)
      float out[EPL];
      int am[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int l = l0 + i;
        float best = kInf;
        int arg = 0;
        if (l - D >= 0) best = s_pv[l - D], arg = s_pi[l - D];
#pragma unroll
        for (int t = -(DW - 1); t <= DW - 1; ++t) {
          const float v = fadd(win[i + t + DW - 1], wgt[t < 0 ? -t : t]);
          const bool p = v < best;
          best = p ? v : best;
          arg = p ? l + t : arg;
        }
        if (l + D <= L - 1) {
          const float v = s_sv[l + D];
          const bool p = v < best;
          best = p ? v : best;
          arg = p ? int(s_si[l + D]) : arg;
        }
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
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
