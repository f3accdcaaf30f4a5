// Backward sweep with warp specialisation (sm_100a): isgmr_backward /
// trwp_backward inner loop (autodiff.hpp:83-118, :152-186) for one direction.
//
// A scanline is walked by a PAIR of warps. The chain warp (A) does only what
// the next node depends on:
//   row  = gm^r[cur] + carry, consume (zero) gm^r[cur]
//   acc[mu] = sum_{l : p[l] = mu} g_l        (index-driven scatter)
//   row[q] -= sum(row)  -> applied to acc[p[q]] (reparam backward, :48-53;
//                          linear, so the warp sum is off the chain)
//   carry = rho*acc (TRWP) / acc (ISGMR)     (own plane at prev)
// and hands {g, acc, carry, p} of the node to the leaf warp (B) through a
// double-buffered shared-memory slot, one named barrier per node. B, one node
// behind, does everything nothing downstream waits for: the read-modify-write
// of dtheta[prev] and the other gradient planes at prev, the dw partial and
// the dV partials. Both warps prefetch their own rows kStages-1 nodes ahead
// with cp.async. Lane a owns labels a*EPL + i in both warps.
//
// The scatter is resolved inside A without shared-memory atomics: targets
// within one label of the source go to the owner's registers (neighbour lanes
// via one shuffle); the others are summed per distinct target with warp
// reductions (smallest and largest pending target per round); L <= 32
// gathers instead. Rows of one direction are node-disjoint, so dtheta / gm /
// dw need no atomics and are deterministic; dV partials accumulate in
// registers (near-diagonal, for the whole sweep; far targets, while the
// target repeats) and are flushed with RED into a few replicas.
#pragma once

#include "bwd_warp.cuh"
#include "common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

// per-pair shared memory (floats)
__host__ __device__ constexpr int bws_stageA(int EPL) { return 32 * EPL + 8 * EPL + 4 + 64; }
__host__ __device__ constexpr int bws_stageB(int EPL, int nrow) { return nrow * 32 * EPL + 32; }
__host__ __device__ constexpr int bws_hand(int EPL) { return 3 * 32 * EPL + 8 * EPL; }
__host__ __device__ constexpr int bws_pair_floats(int EPL, int nrowB) {
  return (kStages * bws_stageA(EPL) + kStages * bws_stageB(EPL, nrowB) + 2 * bws_hand(EPL) + 32 * 33 + 31) / 32 * 32;
}

__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }

template <int EPL, bool TRWP, int RT, bool FULL>
__global__ void __launch_bounds__(256) bwd_ws_kernel(BwdArgs a) {
  extern __shared__ float smem[];
  constexpr int NPMAX = RT ? (TRWP ? RT - 1 : RT - 2) : 15;
  constexpr int LS = 32 * EPL;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp >> 1, role = warp & 1, npairs = blockDim.x >> 6;
  const int r = a.r, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
  const int NP = TRWP ? R - 1 : R - 2;
  const int nrowB = 1 + NP;  // dtheta[prev] + NP gradient planes at prev
  float* base = smem + size_t(pair) * bws_pair_floats(EPL, nrowB);
  float* ringA = base;
  float* ringB = ringA + kStages * bws_stageA(EPL);
  float* hand = ringB + kStages * bws_stageB(EPL, nrowB);
  float* s_wp = hand + 2 * bws_hand(EPL);
  const int bar_id = 1 + pair;

  const int b = blockIdx.y;
  const int NL = N * L;
  const int stL = st * L;
  float* img_gm = a.gm + size_t(b) * R * NL;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const int gpair = blockIdx.x * npairs + pair;
  float zero[EPL];
#pragma unroll
  for (int i = 0; i < EPL; ++i) zero[i] = 0.0f;

  if (role == 0) {
    // ======================= chain warp =======================
    float* gmr = img_gm + r * NL + l0;  // lane slice of plane r, node 0
    const uint8_t* pimg = a.p + size_t(b) * g.K_cap * g.E * L;
    const uint8_t* qimg = a.q + size_t(b) * g.K_cap * g.E;
    const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ringA));
    for (int li = gpair; li < a.nlines; li += gridDim.x * npairs) {
      const LineDesc ld = a.lines[li];
      const int nsteps = ld.length - 1;
      const uint32_t ebase = uint32_t(a.k) * uint32_t(g.E) + uint32_t(g.dir_offset[r]) + uint32_t(ld.edge_base);
      const int o_first = ld.first * L;
      auto issue = [&](int s) {
        const uint32_t bs = ring_s + 4u * uint32_t((s % kStages) * bws_stageA(EPL));
        const int j = nsteps - s;
        if (FULL || nvalid > 0) cp_slice_t<EPL, FULL>(bs + 4u * l0, gmr + o_first + j * stL, nvalid);
        const uint32_t e = ebase + uint32_t(j - 1);
        const uint32_t pdst = bs + 4u * LS;
        if (FULL) {
          const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg + size_t(e) * L);
#pragma unroll
          for (int t = 0; t < 2; ++t)
            if (lane + 32 * t < 8 * EPL) cp_async_u32(pdst + 4u * (lane + 32 * t), pw + lane + 32 * t, 4);
        } else {
          const size_t pb = size_t(e) * L;
          const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg) + (pb >> 2);
          const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
          for (int t = lane; t < nwords; t += 32) cp_async_u32(pdst + 4u * t, pw + t, 4);
        }
        const uint32_t xdst = pdst + 4u * (8 * EPL + 4);
        cp_async_u32(xdst + 4u * lane, reinterpret_cast<const uint32_t*>(qimg) + (e >> 2), 4);
        if (rpl) {
          const int node = ld.first + j * st;
          cp_async_u32(xdst + 4u * (32 + lane), rrow + ((r & 1) ? node : node - st), 4);
        }
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
        const float* slot = ringA + (s % kStages) * bws_stageA(EPL);
        const int j = nsteps - s;
        const uint32_t e = ebase + uint32_t(j - 1);
        const uint8_t* prow = reinterpret_cast<const uint8_t*>(slot + LS) + (FULL ? 0 : ((size_t(e) * L) & 3)) + l0;
        const float* xs = slot + LS + 8 * EPL + 4;
        const int qv = (__float_as_uint(xs[lane]) >> (8 * (e & 3))) & 0xff;
        const float rho = TRWP ? (rpl ? xs[32 + lane] : a.pot.rho) : 1.0f;

        float row[EPL];
        int mu[EPL], d[EPL];
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
          stg_slice<EPL>(gmr - l0 + o_first + j * stL, l0, zero, nvalid, L);
          S = warp_sum_f(lsum);
        }
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
          float gm1[EPL], g00[EPL], gp1[EPL];
          int klo[EPL], khi[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            gm1[i] = d[i] == -1 ? row[i] : 0.0f;
            g00[i] = d[i] == 0 ? row[i] : 0.0f;
            gp1[i] = d[i] == 1 ? row[i] : 0.0f;
            const bool far = uint32_t(d[i] + 1) > 2u;
            klo[i] = far ? mu[i] : 0x7fffffff;
            khi[i] = far ? mu[i] : -1;
          }
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
          for (int i = 0; i < EPL; ++i)
            if (iq == i) {
              muq = mu[i];
              row[i] = fsub(row[i], S);
            }
          muq = __shfl_sync(0xffffffffu, muq, qv / EPL);
          const int im = muq - l0;
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (im == i) acc[i] = fsub(acc[i], S);
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) carry[i] = TRWP ? fmul(rho, acc[i]) : acc[i];
        // hand the node to the leaf warp: g, acc, carry, targets
        float* h = hand + (s & 1) * bws_hand(EPL);
        if (FULL || nvalid > 0) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            h[l0 + i] = row[i];
            h[LS + l0 + i] = acc[i];
            h[2 * LS + l0 + i] = carry[i];
            reinterpret_cast<uint8_t*>(h + 3 * LS)[l0 + i] = uint8_t(mu[i]);
          }
        }
        pair_sync(bar_id);
      }
      // head row of plane r: its incoming scatter (carry) is dropped and the
      // row cleared (the reference's plane clear / swap-and-clear, :122-123, :190-193)
      stg_slice<EPL>(gmr - l0 + o_first, l0, zero, nvalid, L);
      cp_wait<0>();
      pair_sync(bar_id);  // leaf warp done with this line's handoff slots
    }
  } else {
    // ======================= leaf warp =======================
    float* gub = a.gu + size_t(b) * NL + l0;
    float* planes = (TRWP ? img_gm : a.gnext + size_t(b) * R * NL) + l0;
    const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ringB));
    float* gvacc = a.gvacc + ((size_t(b) * kVRep + gpair % kVRep) * 2 + (r & 1)) * L * L;
    float* gvl = gvacc + l0;
    const bool do_w = a.gw != nullptr;
    float* gwrow = do_w ? a.gw + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
    const float* Vl = a.pot.V + l0 * vs_l;
    const bool band = a.desc->banded != 0;
    const int Dband = a.desc->D;
    const float* gband = a.desc->g;
    const bool band2 = band && Dband <= 2;
    const float gD = gband[Dband];
    int poff[NPMAX];
#pragma unroll
    for (int rr = 0; rr < NPMAX; ++rr) {
      const int d = TRWP ? (rr < r ? rr : rr + 1) : (rr < (r & ~1) ? rr : rr + 2);
      poff[rr] = d * NL;
    }
    float vloc[EPL][3];
#pragma unroll
    for (int i = 0; i < EPL; ++i)
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int l = l0 + i, m = l + t - 1;
        const bool ok = do_w && l < L && m >= 0 && m < L;
        vloc[i][t] = ok ? __ldg(a.pot.V + m * vs_mu + l * vs_l) : 0.0f;
      }
    float vacc[EPL][3];
    int fkey[EPL];
    float fval[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) vacc[i][0] = vacc[i][1] = vacc[i][2] = 0.0f, fkey[i] = -1, fval[i] = 0.0f;

    for (int li = gpair; li < a.nlines; li += gridDim.x * npairs) {
      const LineDesc ld = a.lines[li];
      const int nsteps = ld.length - 1;
      const int o_first = ld.first * L;
      auto issue = [&](int s) {
        const uint32_t bs = ring_s + 4u * uint32_t((s % kStages) * bws_stageB(EPL, nrowB));
        const int j = nsteps - s;
        const int oprev = o_first + (j - 1) * stL;
        if (FULL || nvalid > 0) {
          cp_slice_t<EPL, FULL>(bs + 4u * l0, gub + oprev, nvalid);
#pragma unroll
          for (int rr = 0; rr < NPMAX; ++rr)
            if (RT || rr < NP) cp_slice_t<EPL, FULL>(bs + 4u * ((1 + rr) * LS + l0), planes + poff[rr] + oprev, nvalid);
        }
        if (wpl) {
          const int node = ld.first + j * st;
          cp_async_u32(bs + 4u * (nrowB * LS + lane), wrow + ((r & 1) ? node : node - st), 4);
        }
      };
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
      for (int s = 0; s < nsteps; ++s) {
        if (s + kStages - 1 < nsteps) issue(s + kStages - 1);
        cp_commit();
        pair_sync(bar_id);  // node s handed over
        cp_wait<kStages - 1>();
        const float* slot = ringB + (s % kStages) * bws_stageB(EPL, nrowB);
        const float* h = hand + (s & 1) * bws_hand(EPL);
        const int j = nsteps - s;
        const int oprev = o_first + (j - 1) * stL;
        float row[EPL], acc[EPL], add[EPL];
        int mu[EPL];
        lds_slice<EPL>(row, h + l0);
        lds_slice<EPL>(acc, h + LS + l0);
        lds_slice<EPL>(add, h + 2 * LS + l0);
#pragma unroll
        for (int i = 0; i < EPL; ++i) mu[i] = reinterpret_cast<const uint8_t*>(h + 3 * LS)[l0 + i];
        const float w = wpl ? slot[nrowB * LS + lane] : a.pot.w;

        // dtheta[prev] and the gradient planes at prev (one writer per row)
        {
          float t[EPL], outv[EPL];
          lds_slice<EPL>(t, slot + l0);
#pragma unroll
          for (int i = 0; i < EPL; ++i) outv[i] = fadd(t[i], add[i]);
          stg_slice<EPL>(gub - l0 + oprev, l0, outv, nvalid, L);
#pragma unroll
          for (int rr = 0; rr < NPMAX; ++rr) {
            if (RT || rr < NP) {
              const bool is_opp = TRWP && (rr < r ? rr : rr + 1) == opp;
              lds_slice<EPL>(t, slot + (1 + rr) * LS + l0);
#pragma unroll
              for (int i = 0; i < EPL; ++i) {
                const float v = fadd(t[i], add[i]);
                outv[i] = is_opp ? fsub(v, acc[i]) : v;
              }
              stg_slice<EPL>(planes - l0 + poff[rr] + oprev, l0, outv, nvalid, L);
            }
          }
        }
        // dw (parked) and dV partials
        float wpart = 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const bool live = (FULL || i < nvalid) && row[i] != 0.0f;
          const int d = mu[i] - (l0 + i);
          const bool far = uint32_t(d + 1) > 2u;
          if (do_w) {
            float vv;
            if (!far) vv = d == -1 ? vloc[i][0] : d == 0 ? vloc[i][1] : vloc[i][2];
            else if (band2) vv = gD;
            else vv = __ldg(band ? gband + min(abs(d), Dband) : Vl + mu[i] * vs_mu + i * vs_l);
            wpart = live ? fadd(wpart, fmul(row[i], vv)) : wpart;
          }
          const float gwv = live ? fmul(row[i], w) : 0.0f;
          vacc[i][0] = d == -1 ? fadd(vacc[i][0], gwv) : vacc[i][0];
          vacc[i][1] = d == 0 ? fadd(vacc[i][1], gwv) : vacc[i][1];
          vacc[i][2] = d == 1 ? fadd(vacc[i][2], gwv) : vacc[i][2];
          if (far && live) {
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
      }
      cp_wait<0>();
      pair_sync(bar_id);  // line done
    }
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      if (fkey[i] >= 0) red_add_global(gvl + fkey[i] * L + i, fval[i]);
      const int l = l0 + i;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int m = l + t - 1;
        if (l < L && m >= 0 && m < L && vacc[i][t] != 0.0f) red_add_global(gvacc + m * L + l, vacc[i][t]);
      }
    }
  }
}

}  // namespace mrf
