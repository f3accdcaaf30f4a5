// Backward sweep, warp-per-scanline (sm_100a): isgmr_backward /
// trwp_backward inner loop (autodiff.hpp:83-118, :152-186) for one direction.
//
// Lane a owns labels l = a*EPL + i of the current row and the same mu slice
// of the predecessor row. Per node (reverse order):
//   row  = gm^r[cur] + carry                (carry: this sweep's own scatter into
//                                             gm^r[cur], kept in registers)
//   row[q] -= sum(row)                       (reparam backward, :48-53)
//   acc[mu] = sum_{l : p[l] = mu, g_l != 0} g_l   (index-driven scatter)
//   dtheta[prev] += acc (ISGMR) / rho*acc (TRWP); gm_next / gm planes likewise
//   dw[edge] += sum_l g_l V'(p_l, l);  dV[p_l, l] += g_l * w
// The scatter is resolved inside the warp without shared-memory atomics:
// targets within one label of the source (the common case) go to the owner's
// registers (neighbour lanes via one shuffle); the others are summed per
// distinct target with warp reductions, the smallest and largest pending
// target per round; L <= 32 gathers instead. Every read-modify-write row is
// owned by exactly one warp within a launch (scanlines of one direction are
// node-disjoint), so dtheta / gm / dw need no atomics and are deterministic;
// dV partials use fire-and-forget reductions (RED) into a few replicas
// (near-diagonal ones accumulate in registers over the whole sweep). The
// per-edge dw sums are deferred: lane partials of 32 consecutive edges are
// parked in shared memory and reduced together. The rows a step touches do
// not depend on the chain and are prefetched with cp.async kStages-1 steps
// ahead, as in the forward. All in-image addressing is 32-bit (the host
// rejects images with R*N*L >= 2^31 floats or K*E*L >= 2^32 index bytes).
#pragma once

#include "common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

constexpr int kVRep = 4;  // dV accumulation replicas per image

struct BwdArgs {
  Geometry g;
  Potentials pot;
  const LineDesc* lines;  // direction r, every line (length >= 1)
  int nlines;
  int r;
  const uint8_t* p;
  const uint8_t* q;
  int k;
  float* gm;     // [B][R][N][L]
  float* gnext;  // [B][R][N][L] (ISGMR) or null
  float* gu;     // [B][N][L]
  float* gw;     // [B][R/2][N] or null
  float* gvacc;  // [B][kVRep][2][L][L]
  const PairDesc* desc;  // banded V: V'(mu, l) = g(min(|mu - l|, D)) without a table load
};

// per-warp ring stage: rowsF float rows + p words + {q, w, rho} words per lane
__host__ __device__ constexpr int bwd_stage_floats(int EPL, int rowsF) { return rowsF * 32 * EPL + 8 * EPL + 4 + 96; }
// ring + dw parking [32][33]
__host__ __device__ constexpr int bwd_warp_smem_floats(int EPL, int rowsF) {
  return (kStages * bwd_stage_floats(EPL, rowsF) + 32 * 33 + 31) / 32 * 32;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// RT: compile-time direction count (4 or 8), or 0 for runtime R.
// FULL: L == 32*EPL (every lane owns EPL valid labels).
template <int EPL, bool TRWP, int RT, bool FULL>
__global__ void __launch_bounds__(128) bwd_warp_kernel(BwdArgs a) {
  extern __shared__ float smem[];
  constexpr int NPMAX = RT ? (TRWP ? RT - 1 : RT - 2) : 15;
  constexpr int LS = 32 * EPL;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int r = a.r, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
  const int NP = TRWP ? R - 1 : R - 2;
  const int rowsF = 2 + NP;  // gm^r[cur], dtheta[prev], NP gradient planes at prev
  const int stage_f = bwd_stage_floats(EPL, rowsF);
  float* ring = smem + size_t(wid) * bwd_warp_smem_floats(EPL, rowsF);
  float* s_wp = ring + kStages * stage_f;  // [32][33] parked dw lane partials
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));

  const int b = blockIdx.y;
  const int NL = N * L;
  const int stL = st * L;
  float* img_gm = a.gm + size_t(b) * R * NL;
  float* gmr = img_gm + r * NL + lane * EPL;  // lane slice of plane r, node 0
  float* gub = a.gu + size_t(b) * NL + lane * EPL;
  float* planes = (TRWP ? img_gm : a.gnext + size_t(b) * R * NL) + lane * EPL;
  const uint8_t* pimg = a.p + size_t(b) * g.K_cap * g.E * L;
  const uint8_t* qimg = a.q + size_t(b) * g.K_cap * g.E;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const int warp_global = blockIdx.x * wpc + wid;
  float* gvacc = a.gvacc + ((size_t(b) * kVRep + warp_global % kVRep) * 2 + (r & 1)) * L * L;
  const bool do_w = a.gw != nullptr;
  float* gwrow = do_w ? a.gw + (size_t(b) * (R / 2) + fam) * N : nullptr;
  // V'(mu, l) = V[mu*vs_mu + l*vs_l]: V(mu,l) on even directions, V(l,mu) on odd
  const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
  const float* Vl = a.pot.V + lane * EPL * vs_l;  // lane's first label
  float* gvl = gvacc + lane * EPL;
  const bool band = a.desc->banded != 0;
  const int Dband = a.desc->D;
  const float* gband = a.desc->g;
  const bool band2 = band && Dband <= 2;
  const float gD = gband[Dband];
  // far dV contributions: per label, a one-entry cache of the last far target
  // (targets move slowly along a scanline), flushed with RED on change
  int fkey[EPL];
  float fval[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) fkey[i] = -1, fval[i] = 0.0f;
  // plane offsets (elements) at node 0, ascending d: TRWP skips r, ISGMR skips {r, r^1}
  int poff[NPMAX];
#pragma unroll
  for (int rr = 0; rr < NPMAX; ++rr) {
    const int d = TRWP ? (rr < r ? rr : rr + 1) : (rr < (r & ~1) ? rr : rr + 2);
    poff[rr] = d * NL;
  }
  // near-diagonal V'(l + delta, l), delta = -1, 0, 1 (for dw)
  float vloc[EPL][3];
#pragma unroll
  for (int i = 0; i < EPL; ++i)
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int l = l0 + i, mu = l + t - 1;
      const bool ok = do_w && l < L && mu >= 0 && mu < L;
      vloc[i][t] = ok ? __ldg(a.pot.V + mu * vs_mu + l * vs_l) : 0.0f;
    }

  float vacc[EPL][3];  // near-diagonal dV partials, (mu = l + delta, l)
#pragma unroll
  for (int i = 0; i < EPL; ++i) vacc[i][0] = vacc[i][1] = vacc[i][2] = 0.0f;
  float zero[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) zero[i] = 0.0f;

  for (int li = warp_global; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int nsteps = ld.length - 1;
    // in-image index of edge (k, r, e) for node position j: ebase + j - 1
    const uint32_t ebase = uint32_t(a.k) * uint32_t(g.E) + uint32_t(g.dir_offset[r]) + uint32_t(ld.edge_base);
    const int o_first = ld.first * L;

    // step s (0-based) handles node position j = nsteps - s (reverse order)
    auto issue = [&](int s) {
      const int slot = s % kStages;
      const uint32_t base_s = ring_s + 4u * uint32_t(slot * stage_f);
      const int j = nsteps - s;
      const int ocur = o_first + j * stL, oprev = ocur - stL;
      if (FULL || nvalid > 0) {
        cp_slice_t<EPL, FULL>(base_s + 4u * l0, gmr + ocur, nvalid);
        cp_slice_t<EPL, FULL>(base_s + 4u * (LS + l0), gub + oprev, nvalid);
#pragma unroll
        for (int rr = 0; rr < NPMAX; ++rr)
          if (RT || rr < NP) cp_slice_t<EPL, FULL>(base_s + 4u * ((2 + rr) * LS + l0), planes + poff[rr] + oprev, nvalid);
      }
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint32_t pdst = base_s + 4u * (rowsF * LS);
      if (FULL) {
        // row start e*L is 4-byte aligned; L/4 = 8*EPL words, at most 2 per lane
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg + size_t(e) * L);
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (lane + 32 * t < 8 * EPL) cp_async_u32(pdst + 4u * (lane + 32 * t), pw + lane + 32 * t, 4);
      } else {
        // the aligned words covering bytes [e*L, e*L + L)
        const size_t pb = size_t(e) * L;
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg) + (pb >> 2);
        const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
        for (int t = lane; t < nwords; t += 32) cp_async_u32(pdst + 4u * t, pw + t, 4);
      }
      // per-lane copies of the q word, w and rho (no cross-lane dependency)
      const uint32_t xdst = pdst + 4u * (8 * EPL + 4);
      cp_async_u32(xdst + 4u * lane, reinterpret_cast<const uint32_t*>(qimg) + (e >> 2), 4);
      if (wpl || rpl) {
        const int node = ld.first + j * st;
        const int wnode = (r & 1) ? node : node - st;
        if (wpl) cp_async_u32(xdst + 4u * (32 + lane), wrow + wnode, 4);
        if (rpl) cp_async_u32(xdst + 4u * (64 + lane), rrow + wnode, 4);
      }
    };
    // deferred per-edge dw: reduce parked lane partials of steps [s0, s0+cnt)
    auto flush_w = [&](int s0, int cnt) {
      __syncwarp();
      if (lane < cnt) {
        float t = 0.0f;
#pragma unroll 8
        for (int c = 0; c < 32; ++c) t = fadd(t, s_wp[lane * 33 + c]);
        const int node = ld.first + (nsteps - (s0 + lane)) * st;
        float* dst = gwrow + ((r & 1) ? node : node - st);
        *dst = fadd(*dst, t);
      }
      __syncwarp();
    };

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nsteps) issue(s);
      cp_commit();
    }
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;

    for (int s = 0; s < nsteps; ++s) {
      if (s + kStages - 1 < nsteps) issue(s + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      __syncwarp();  // p words were copied by other lanes
      const float* slot = ring + (s % kStages) * stage_f;
      const int j = nsteps - s;
      const int ocur = o_first + j * stL, oprev = ocur - stL;
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint8_t* prow = reinterpret_cast<const uint8_t*>(slot + rowsF * LS) + (FULL ? 0 : ((size_t(e) * L) & 3)) + l0;
      const float* xs = slot + rowsF * LS + 8 * EPL + 4;
      const int qv = (__float_as_uint(xs[lane]) >> (8 * (e & 3))) & 0xff;
      const float w = wpl ? xs[32 + lane] : a.pot.w;
      const float rho = TRWP ? (rpl ? xs[64 + lane] : a.pot.rho) : 1.0f;

      // ---- row = gm^r[cur] + carry; consume (zero) gm^r[cur]
      // The reparametrisation backward row[q] -= sum(row) (:48-53) only moves
      // one entry, and the scatter is linear, so the scatter runs on the raw
      // row while the warp sum is in flight; -sum is then added to the target
      // of q (and g_q is corrected for dw / dV).
      float row[EPL];
      int d[EPL], mu[EPL];
      float S;
      {
        float t[EPL];
        lds_slice<EPL>(t, slot + l0);
        float lsum = 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          row[i] = (FULL || i < nvalid) ? fadd(t[i], carry[i]) : 0.0f;
          lsum = fadd(lsum, row[i]);
          mu[i] = (FULL || i < nvalid) ? int(prow[i]) : l0 + i;
          d[i] = mu[i] - (l0 + i);
        }
        stg_slice<EPL>(gmr - l0 + ocur, l0, zero, nvalid, L);
        S = warp_sum_f(lsum);
      }
      // split by target offset d = p[l] - l (masked copies are exact zeros
      // elsewhere, so adding them unconditionally leaves every sum unchanged)
      float gm1[EPL], g00[EPL], gp1[EPL];
      bool far[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        gm1[i] = d[i] == -1 ? row[i] : 0.0f;
        g00[i] = d[i] == 0 ? row[i] : 0.0f;
        gp1[i] = d[i] == 1 ? row[i] : 0.0f;
        far[i] = uint32_t(d[i] + 1) > 2u;
      }
      // far targets' V' values, issued early so their latency overlaps the scatter
      float vfar[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (band2) {
          vfar[i] = gD;  // banded with D <= 2: every far candidate costs g(D)
        } else {
          const float* src = band ? gband + min(abs(d[i]), Dband) : Vl + mu[i] * vs_mu + i * vs_l;
          vfar[i] = (do_w && far[i]) ? __ldg(src) : 0.0f;
        }
      }

      // ---- scatter: acc[mu] = sum over l with p[l] = mu of g_l
      float acc[EPL];
      if (EPL == 1) {
        acc[0] = 0.0f;
        const float g0 = row[0];
#pragma unroll 8
        for (int lam = 0; lam < L; ++lam) {
          const int pl = __shfl_sync(0xffffffffu, mu[0], lam);
          const float gl = __shfl_sync(0xffffffffu, g0, lam);
          acc[0] = (pl == lane && gl != 0.0f) ? fadd(acc[0], gl) : acc[0];
        }
      } else {
        // acc[mu] gets g(mu) [d=0], g(mu+1) [d=-1], g(mu-1) [d=+1]; the labels
        // just outside the lane's slice come from the neighbour lanes
        float m1n = __shfl_down_sync(0xffffffffu, gm1[0], 1);
        float p1n = __shfl_up_sync(0xffffffffu, gp1[EPL - 1], 1);
        m1n = lane < 31 ? m1n : 0.0f;
        p1n = lane > 0 ? p1n : 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const float m1 = i + 1 < EPL ? gm1[i + 1 < EPL ? i + 1 : 0] : m1n;
          const float p1 = i > 0 ? gp1[i > 0 ? i - 1 : 0] : p1n;
          acc[i] = fadd(fadd(g00[i], m1), p1);
        }
        // far targets: per round, the smallest and the largest pending target
        // are summed with two independent warp reductions (usually one round)
        int klo[EPL], khi[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          klo[i] = far[i] ? mu[i] : 0x7fffffff;
          khi[i] = far[i] ? mu[i] : -1;
        }
        while (true) {
          int mn = klo[0], mx = khi[0];
#pragma unroll
          for (int i = 1; i < EPL; ++i) mn = min(mn, klo[i]), mx = max(mx, khi[i]);
          const int kmin = __reduce_min_sync(0xffffffffu, mn);
          if (kmin == 0x7fffffff) break;
          const int kmax = __reduce_max_sync(0xffffffffu, mx);
          float pa = 0.0f, pb2 = 0.0f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            pa = fadd(pa, klo[i] == kmin ? row[i] : 0.0f);
            pb2 = fadd(pb2, khi[i] == kmax ? row[i] : 0.0f);
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const bool done = klo[i] == kmin || khi[i] == kmax;
            klo[i] = done ? 0x7fffffff : klo[i];
            khi[i] = done ? -1 : khi[i];
          }
          if (kmax == kmin) pb2 = 0.0f;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            pa = fadd(pa, __shfl_xor_sync(0xffffffffu, pa, o));
            pb2 = fadd(pb2, __shfl_xor_sync(0xffffffffu, pb2, o));
          }
          const int ia = kmin - l0, ib = kmax - l0;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            if (ia == i) acc[i] = fadd(acc[i], pa);
            if (ib == i) acc[i] = fadd(acc[i], pb2);
          }
        }
      }
      // reparametrisation backward: g_q = row_q - S lands on target p[q]
      {
        const int iq = qv - l0;
        int muq = 0;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          if (iq == i) {
            muq = mu[i];
            row[i] = fsub(row[i], S);
          }
        }
        muq = __shfl_sync(0xffffffffu, muq, qv / EPL);
        const int im = muq - l0;
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          if (im == i) acc[i] = fsub(acc[i], S);
        // masks for dV / dw see the corrected g_q (only element iq changes)
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          if (iq != i) continue;
          gm1[i] = d[i] == -1 ? row[i] : 0.0f;
          g00[i] = d[i] == 0 ? row[i] : 0.0f;
          gp1[i] = d[i] == 1 ? row[i] : 0.0f;
        }
      }

      // ---- apply to the predecessor rows; carry the own-plane share
      {
        float outv[EPL], t[EPL], add[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          add[i] = TRWP ? fmul(rho, acc[i]) : acc[i];
          carry[i] = add[i];
        }
        lds_slice<EPL>(t, slot + LS + l0);
#pragma unroll
        for (int i = 0; i < EPL; ++i) outv[i] = fadd(t[i], add[i]);
        stg_slice<EPL>(gub - l0 + oprev, l0, outv, nvalid, L);
#pragma unroll
        for (int rr = 0; rr < NPMAX; ++rr) {
          if (RT || rr < NP) {
            const bool is_opp = TRWP && (rr < r ? rr : rr + 1) == opp;
            lds_slice<EPL>(t, slot + (2 + rr) * LS + l0);
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const float v = fadd(t[i], add[i]);
              outv[i] = is_opp ? fsub(v, acc[i]) : v;
            }
            stg_slice<EPL>(planes - l0 + poff[rr] + oprev, l0, outv, nvalid, L);
          }
        }
      }

      // ---- dw (parked) and dV contributions of this edge
      float wpart = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (do_w) {
          const float vv = d[i] == -1 ? vloc[i][0] : d[i] == 0 ? vloc[i][1] : d[i] == 1 ? vloc[i][2] : vfar[i];
          const float c = fmul(row[i], vv);
          wpart = row[i] != 0.0f ? fadd(wpart, c) : wpart;
        }
        vacc[i][0] = fadd(vacc[i][0], fmul(gm1[i], w));
        vacc[i][1] = fadd(vacc[i][1], fmul(g00[i], w));
        vacc[i][2] = fadd(vacc[i][2], fmul(gp1[i], w));
        if (far[i] && row[i] != 0.0f) {
          const float gwv = fmul(row[i], w);
          if (mu[i] == fkey[i]) {
            fval[i] = fadd(fval[i], gwv);
          } else {
            if (fkey[i] >= 0) red_add_global(gvl + fkey[i] * L + i, fval[i]);
            fkey[i] = mu[i];
            fval[i] = gwv;
          }
        }
      }
      if (do_w) {
        s_wp[(s & 31) * 33 + lane] = wpart;
        if ((s & 31) == 31 || s == nsteps - 1) flush_w(s & ~31, (s & 31) + 1);
      }
      __syncwarp();
    }
    // head row of plane r: its incoming scatter (carry) is dropped and the row
    // cleared, like the reference's plane clear / buffer swap (:122-123, :190-193)
    stg_slice<EPL>(gmr - l0 + o_first, l0, zero, nvalid, L);
    cp_wait<0>();
    __syncwarp();
  }
  // flush the far-target caches and the near-diagonal dV partials
#pragma unroll
  for (int i = 0; i < EPL; ++i)
    if (fkey[i] >= 0) red_add_global(gvl + fkey[i] * L + i, fval[i]);
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int l = l0 + i;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int mu = l + t - 1;
      if (l < L && mu >= 0 && mu < L && vacc[i][t] != 0.0f) red_add_global(gvacc + mu * L + l, vacc[i][t]);
    }
  }
}

// dV[b][x][y] = sum_rep acc[b][rep][0][x][y] + acc[b][rep][1][y][x]
static __global__ void reduce_gvacc_kernel(int B, int L, const float* __restrict__ acc, float* __restrict__ gv) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t LL = int64_t(L) * L;
  if (i >= B * LL) return;
  const int b = int(i / LL);
  const int xy = int(i - b * LL), x = xy / L, y = xy - x * L;
  float s = 0.0f;
  for (int rep = 0; rep < kVRep; ++rep) {
    const float* base = acc + (size_t(b) * kVRep + rep) * 2 * LL;
    s = fadd(s, base[xy]);
    s = fadd(s, base[LL + size_t(y) * L + x]);
  }
  gv[i] = s;
}

}  // namespace mrf
