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
// ahead, as in the forward.
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
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int r = a.r, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
  const int NP = TRWP ? R - 1 : R - 2;
  const int rowsF = 2 + NP;  // gm^r[cur], dtheta[prev], NP gradient planes at prev
  constexpr int LS = 32 * EPL;
  const int stage_f = bwd_stage_floats(EPL, rowsF);
  float* ring = smem + size_t(wid) * bwd_warp_smem_floats(EPL, rowsF);
  float* s_wp = ring + kStages * stage_f;  // [32][33] parked dw lane partials
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));

  const int b = blockIdx.y;
  const size_t img = size_t(b) * R * N * L;
  const size_t NL = size_t(N) * L;
  float* gmr = a.gm + img + size_t(r) * NL;
  float* gub = a.gu + size_t(b) * NL;
  float* planes_base = TRWP ? a.gm + img : a.gnext + img;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const int warp_global = blockIdx.x * wpc + wid;
  float* gvacc = a.gvacc + ((size_t(b) * kVRep + warp_global % kVRep) * 2 + (r & 1)) * L * L;
  const bool do_w = a.gw != nullptr;
  float* gwrow = do_w ? a.gw + (size_t(b) * (R / 2) + fam) * N : nullptr;
  // plane offsets at a node, ascending d: TRWP skips r, ISGMR skips {r, r^1}
  size_t poff[RT ? (TRWP ? RT - 1 : RT - 2) : 15];
#pragma unroll
  for (int rr = 0; rr < (RT ? (TRWP ? RT - 1 : RT - 2) : 15); ++rr) {
    const int d = TRWP ? (rr < r ? rr : rr + 1) : (rr < (r & ~1) ? rr : rr + 2);
    poff[rr] = size_t(d) * NL + l0;
  }
  // near-diagonal V'(l + delta, l), delta = -1, 0, 1 (for dw), per direction parity
  float vloc[EPL][3];
#pragma unroll
  for (int i = 0; i < EPL; ++i)
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int l = l0 + i, mu = l + t - 1;
      const bool ok = do_w && l < L && mu >= 0 && mu < L;
      vloc[i][t] = ok ? __ldg(a.pot.V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
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
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;

    // step s (0-based) handles node position j = nsteps - s (reverse order)
    auto issue = [&](int s) {
      const int slot = s % kStages;
      const uint32_t base_s = ring_s + 4u * uint32_t(slot * stage_f);
      const int j = nsteps - s;
      const int cur = ld.first + j * st, prev = cur - st;
      if (FULL || nvalid > 0) {
        const size_t pn = size_t(prev) * L;
        cp_slice_t<EPL, FULL>(base_s + 4u * l0, gmr + size_t(cur) * L + l0, nvalid);
        cp_slice_t<EPL, FULL>(base_s + 4u * (LS + l0), gub + pn + l0, nvalid);
#pragma unroll
        for (int rr = 0; rr < (RT ? (TRWP ? RT - 1 : RT - 2) : 15); ++rr)
          if (RT || rr < NP) cp_slice_t<EPL, FULL>(base_s + 4u * ((2 + rr) * LS + l0), planes_base + poff[rr] + pn, nvalid);
      }
      // p row: the aligned words covering bytes [flat*L, flat*L + L)
      const size_t flat = pq_base + j - 1;
      const size_t pb = flat * L;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(a.p) + (pb >> 2);
      const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
      const uint32_t pdst = base_s + 4u * (rowsF * LS);
      for (int t = lane; t < nwords; t += 32) cp_async_u32(pdst + 4u * t, pw + t, 4);
      // per-lane copies of the q word, w and rho (no cross-lane dependency)
      const uint32_t xdst = pdst + 4u * (8 * EPL + 4);
      cp_async_u32(xdst + 4u * lane, reinterpret_cast<const uint32_t*>(a.q) + (flat >> 2), 4);
      const int wnode = (r & 1) ? cur : prev;
      if (wpl) cp_async_u32(xdst + 4u * (32 + lane), wrow + wnode, 4);
      if (rpl) cp_async_u32(xdst + 4u * (64 + lane), rrow + wnode, 4);
    };
    // deferred per-edge dw: reduce parked lane partials of steps [s0, s0+cnt)
    auto flush_w = [&](int s0, int cnt) {
      __syncwarp();
      if (lane < cnt) {
        float t = 0.0f;
#pragma unroll 8
        for (int c = 0; c < 32; ++c) t = fadd(t, s_wp[lane * 33 + c]);
        const int j = nsteps - (s0 + lane);
        const int cur = ld.first + j * st;
        float* dst = gwrow + ((r & 1) ? cur : cur - st);
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
      const int cur = ld.first + j * st, prev = cur - st;
      const size_t flat = pq_base + j - 1;
      const uint8_t* prow = reinterpret_cast<const uint8_t*>(slot + rowsF * LS) + ((flat * L) & 3) + l0;
      const float* xs = slot + rowsF * LS + 8 * EPL + 4;
      const int qv = (__float_as_uint(xs[lane]) >> (8 * (flat & 3))) & 0xff;
      const float w = wpl ? xs[32 + lane] : a.pot.w;
      const float rho = TRWP ? (rpl ? xs[64 + lane] : a.pot.rho) : 1.0f;

      // ---- row = gm^r[cur] + carry; consume (zero) gm^r[cur]; reparam backward
      float row[EPL];
      int pm[EPL];
      {
        float t[EPL];
        lds_slice<EPL>(t, slot + l0);
        float lsum = 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          row[i] = (FULL || i < nvalid) ? fadd(t[i], carry[i]) : 0.0f;
          lsum = fadd(lsum, row[i]);
          pm[i] = (FULL || i < nvalid) ? int(prow[i]) : 0;
        }
        stg_slice<EPL>(gmr + size_t(cur) * L, l0, zero, nvalid, L);
        const float S = warp_sum_f(lsum);
#pragma unroll
        for (int i = 0; i < EPL; ++i) row[i] = l0 + i == qv ? fsub(row[i], S) : row[i];
      }
      bool live[EPL];
      int dl[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        live[i] = (FULL || i < nvalid) && row[i] != 0.0f;
        dl[i] = pm[i] - (l0 + i);
      }
      // far targets' V' values, issued early so their latency overlaps the scatter
      float vfar[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const int l = l0 + i, mu = pm[i];
        const bool far = do_w && live[i] && (dl[i] < -1 || dl[i] > 1);
        vfar[i] = far ? __ldg(a.pot.V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
      }

      // ---- scatter: acc[mu] = sum over l with p[l] = mu of g_l
      float acc[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = 0.0f;
      if (EPL == 1) {
        const float g0 = live[0] ? row[0] : 0.0f;
#pragma unroll 8
        for (int lam = 0; lam < L; ++lam) {
          const int pl = __shfl_sync(0xffffffffu, pm[0], lam);
          const float gl = __shfl_sync(0xffffffffu, g0, lam);
          acc[0] = (pl == lane && gl != 0.0f) ? fadd(acc[0], gl) : acc[0];
        }
      } else {
        bool rem[EPL];
        float accL = 0.0f, accR = 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const float gi = row[i];
          acc[i] = live[i] && dl[i] == 0 ? fadd(acc[i], gi) : acc[i];
          if (i > 0) {
            acc[i > 0 ? i - 1 : 0] = live[i] && dl[i] == -1 ? fadd(acc[i > 0 ? i - 1 : 0], gi) : acc[i > 0 ? i - 1 : 0];
          } else {
            accL = live[i] && dl[i] == -1 ? fadd(accL, gi) : accL;
          }
          if (i + 1 < EPL) {
            acc[i + 1 < EPL ? i + 1 : 0] =
                live[i] && dl[i] == 1 ? fadd(acc[i + 1 < EPL ? i + 1 : 0], gi) : acc[i + 1 < EPL ? i + 1 : 0];
          } else {
            accR = live[i] && dl[i] == 1 ? fadd(accR, gi) : accR;
          }
          rem[i] = live[i] && (dl[i] < -1 || dl[i] > 1);
        }
        const float fromR = __shfl_down_sync(0xffffffffu, accL, 1);
        const float fromL = __shfl_up_sync(0xffffffffu, accR, 1);
        acc[EPL - 1] = lane < 31 ? fadd(acc[EPL - 1], fromR) : acc[EPL - 1];
        acc[0] = lane > 0 ? fadd(acc[0], fromL) : acc[0];
        // remaining targets: per round, the smallest and the largest pending
        // target are summed with two independent warp reductions
        while (true) {
          uint32_t mn = 0xffffffffu, mx = 0u;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            mn = rem[i] ? min(mn, uint32_t(pm[i])) : mn;
            mx = rem[i] ? max(mx, uint32_t(pm[i]) + 1u) : mx;
          }
          const uint32_t kmin = __reduce_min_sync(0xffffffffu, mn);
          if (kmin == 0xffffffffu) break;
          const uint32_t kmax = __reduce_max_sync(0xffffffffu, mx) - 1u;
          float pa = 0.0f, pb2 = 0.0f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const bool ia = rem[i] && uint32_t(pm[i]) == kmin;
            const bool ib = rem[i] && uint32_t(pm[i]) == kmax && kmax != kmin;
            pa = ia ? fadd(pa, row[i]) : pa;
            pb2 = ib ? fadd(pb2, row[i]) : pb2;
            rem[i] = rem[i] && !ia && !ib;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            pa = fadd(pa, __shfl_xor_sync(0xffffffffu, pa, o));
            pb2 = fadd(pb2, __shfl_xor_sync(0xffffffffu, pb2, o));
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            acc[i] = int(kmin) == l0 + i ? fadd(acc[i], pa) : acc[i];
            acc[i] = (kmax != kmin && int(kmax) == l0 + i) ? fadd(acc[i], pb2) : acc[i];
          }
        }
      }

      // ---- apply to the predecessor rows; carry the own-plane share
      {
        float outv[EPL], t[EPL], add[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) add[i] = TRWP ? fmul(rho, acc[i]) : acc[i];
#pragma unroll
        for (int i = 0; i < EPL; ++i) carry[i] = add[i];
        const size_t pn = size_t(prev) * L;
        lds_slice<EPL>(t, slot + LS + l0);
#pragma unroll
        for (int i = 0; i < EPL; ++i) outv[i] = fadd(t[i], add[i]);
        stg_slice<EPL>(gub + pn, l0, outv, nvalid, L);
#pragma unroll
        for (int rr = 0; rr < (RT ? (TRWP ? RT - 1 : RT - 2) : 15); ++rr) {
          if (RT || rr < NP) {
            const bool is_opp = TRWP && (rr < r ? rr : rr + 1) == opp;
            lds_slice<EPL>(t, slot + (2 + rr) * LS + l0);
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const float v = fadd(t[i], add[i]);
              outv[i] = is_opp ? fsub(v, acc[i]) : v;
            }
            stg_slice<EPL>(planes_base + poff[rr] - l0 + pn, l0, outv, nvalid, L);
          }
        }
      }

      // ---- dw (parked) and dV contributions of this edge
      float wpart = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const float gi = row[i];
        const int d = dl[i];
        const float vv = d == -1 ? vloc[i][0] : d == 0 ? vloc[i][1] : d == 1 ? vloc[i][2] : vfar[i];
        wpart = live[i] ? fadd(wpart, fmul(gi, vv)) : wpart;
        const float gwv = fmul(gi, w);
        vacc[i][0] = live[i] && d == -1 ? fadd(vacc[i][0], gwv) : vacc[i][0];
        vacc[i][1] = live[i] && d == 0 ? fadd(vacc[i][1], gwv) : vacc[i][1];
        vacc[i][2] = live[i] && d == 1 ? fadd(vacc[i][2], gwv) : vacc[i][2];
        if (live[i] && (d < -1 || d > 1)) atomicAdd(gvacc + size_t(pm[i]) * L + l0 + i, gwv);
      }
      if (do_w) {
        s_wp[(s & 31) * 33 + lane] = wpart;
        if ((s & 31) == 31 || s == nsteps - 1) flush_w(s & ~31, (s & 31) + 1);
      }
      __syncwarp();
    }
    // head row of plane r: its incoming scatter (carry) is dropped and the row
    // cleared, like the reference's plane clear / buffer swap (:122-123, :190-193)
    stg_slice<EPL>(gmr + size_t(ld.first) * L, l0, zero, nvalid, L);
    cp_wait<0>();
    __syncwarp();
  }
  // flush near-diagonal dV partials
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int l = l0 + i;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int mu = l + t - 1;
      if (l < L && mu >= 0 && mu < L && vacc[i][t] != 0.0f) atomicAdd(gvacc + size_t(mu) * L + l, vacc[i][t]);
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
