// Backward sweep for banded V with D <= 2 (the stereo configurations C1-C3),
// ONE WARP PER SCANLINE (sm_100a): isgmr_backward / trwp_backward
// (autodiff.hpp:63-126, :133-197) over the scatter planes of bwd_common.cuh.
//
// Same algebra and decode as bwd_split.cuh's banded mode (see there), with the
// three roles folded into one warp: per node step (tail to head) the warp
// assembles x = gm^r(cur) without the carry and its sum S from rows staged
// kStages-1 steps ahead by cp.async, decodes the p row into the near-target
// mask word (l-1 / l / l+1) and the far target(s), and then does
//   acc  = scatter(x + carry) - S e_{p_q}     (near targets by neighbour
//          shuffles, the main far group by one warp reduction)
//   A[r](prev) = acc,   carry' = rho acc,
//   g = x + carry - S e_q  ->  dV partials (w folded at flush when constant),
//          dw (g(0)-g(D)) s0 + (g(1)-g(D)) s1, and on the TRWP direction-0
//          sweep dtheta(cur) = dtheta + sum_d rho_d A[d](cur) + carry.
// No mbarriers, no slot round trips through shared memory: ~1/2.5 of the
// split kernel's instructions per node. Lines are assigned to warps
// statically (warp w sweeps lines w, w + G, ..., longest first); every warp
// owns a private dV slot (deterministic, bwd_common.cuh).
#pragma once

#include "bwd_common.cuh"
#include "bwd_split.cuh"

namespace mrf {

constexpr int kWarpStages = 3;  // cp.async ring depth (node steps in flight + 1): 12 warps per SM fit

// per-warp ring stage: NR rows + the fused dtheta row + p bytes (8*EPL words)
// + scalars {q word, w, rho, pad} + rho_d[NR] per lane
__host__ __device__ constexpr int bwarp_stage_floats(int EPL, int NR) {
  return (NR + 1) * 32 * EPL + 8 * EPL + 4 + 32 * NR;
}
// ring + other-pairs list (16*EPL words) + dw parking [32][33]
__host__ __device__ constexpr int bwarp_warp_floats(int EPL, int NR) {
  return (kWarpStages * bwarp_stage_floats(EPL, NR) + 16 * EPL + 32 * 33 + 3) / 4 * 4;
}

template <int EPL, bool TRWP, int RT, bool FULL>
__global__ void __launch_bounds__(128) bwd_warp_kernel(AccArgs a) {
  if (split_mode(a.desc->banded, a.desc->D, a.g.L) != 1) return;  // the split kernel owns other modes
  extern __shared__ __align__(16) float smem[];
  constexpr int NRMAX = RT ? acc_rows(TRWP, RT) : 16;
  constexpr int LS = 32 * EPL;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int NR = acc_rows(TRWP, R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int stage_f = bwarp_stage_floats(EPL, NR);
  float* ring = smem + size_t(wid) * bwarp_warp_floats(EPL, NR);
  uint16_t* olist = reinterpret_cast<uint16_t*>(ring + kWarpStages * stage_f);
  float* s_wp = ring + kWarpStages * stage_f + 16 * EPL;
  const uint32_t ring_s = smem_u32(ring);

  const int b = blockIdx.y;
  const int NL = N * L;
  const bool first = a.k == g.K_cap - 1;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const bool do_w = a.gw != nullptr;
  const bool fuse = TRWP && a.dtheta != nullptr;
  const int warp_g = blockIdx.x * wpc + wid, nwarps = gridDim.x * wpc;
  // this warp's private dV slot; entry (mu, l) of V' is V[mu][l] (even r) / V[l][mu] (odd r)
  float* gvacc = a.gvacc + (size_t(b) * a.dv_slots + warp_g) * L * L;
  const float* dcb = a.dc + size_t(b) * NL;
  const float* ainb = a.ain + size_t(b) * R * NL;
  const float* dtsb = fuse ? a.dtheta_src + size_t(b) * NL : nullptr;
  float* dthb = fuse ? a.dtheta + size_t(b) * NL : nullptr;
  const float* gband = a.desc->g;
  const int Dband = a.desc->D;
  const float gb0 = gband[0], gb1 = gband[L > 1 ? 1 : 0], gbD = gband[Dband];
  const float wfold = wpl ? 1.0f : a.pot.w;

  for (int li = warp_g; li < a.nlines; li += nwarps) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    const int stL = st * L;
    const int o_first = ld.first * L;
    // edge index over the whole batch (p / q words aligned for any b, K, E)
    const uint32_t ebase = (uint32_t(b) * uint32_t(g.K_cap) + uint32_t(a.k)) * uint32_t(g.E) +
                           uint32_t(g.dir_offset[r]) + uint32_t(ld.edge_base);
    const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
    float* aout_r = a.aout + size_t(b) * R * NL + size_t(r) * NL;
    float* gwrow = do_w ? a.gw + (TRWP ? (size_t(b) * (R / 2) + fam) * N : (size_t(b) * R + r) * N) : nullptr;
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    // rows gm^r(cur) is assembled from, in accumulation order (-1 = dc): as bwd_split.cuh
    int nrows = 0, opp_slot = -1;
    int sd[NRMAX];
#pragma unroll
    for (int rr = 0; rr < NRMAX; ++rr) sd[rr] = 0;
    auto push = [&](int d) {
#pragma unroll
      for (int rr = 0; rr < NRMAX; ++rr)
        if (rr == nrows) sd[rr] = d;
      if (d == opp) opp_slot = nrows;
      ++nrows;
    };
    if (first) push(-1);
    if (TRWP) {
      if (!first)
        for (int d = r - 1; d >= 0; --d) push(d);
      for (int d = R - 1; d > r; --d) push(d);
    } else if (!first) {
      for (int d = 0; d < R; ++d)
        if (d != r && d != opp) push(d);
    }
    const int a0 = first ? 1 : 0;
    const int npl = nrows;
    const bool fz = fuse;  // this sweep also carries dtheta (TRWP direction 0)
    const float* rowb[NRMAX];
#pragma unroll
    for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] = sd[rr] < 0 ? dcb : ainb + size_t(sd[rr] > 0 ? sd[rr] : 0) * NL;

    // FULL rows: this lane's 16-byte chunk of every staged row and of the p
    // row at the line's last node step, stepped back one node per issue
    const float* rsrc[NRMAX + 1];
#pragma unroll
    for (int rr = 0; rr <= NRMAX; ++rr)
      rsrc[rr] = (rr == nrows ? dtsb : rowb[rr < NRMAX ? rr : 0]) + (o_first + nsteps * stL + 4 * lane);
    const uint8_t* psrc = a.p + size_t(ebase + uint32_t(nsteps - 1)) * L + 16 * lane;
    int islot = 0;
    // node step s (cur = node nsteps - s) into ring slot s % stages (issued in order)
    auto issue = [&](int s) {
      const uint32_t base_s = ring_s + 4u * uint32_t(islot * stage_f);
      islot = islot == kWarpStages - 1 ? 0 : islot + 1;
      const int j = nsteps - s;
      const int ocur = o_first + j * stL;
#pragma unroll
      for (int rr = 0; rr <= NRMAX; ++rr) {
        const bool is_dt = rr == nrows;  // the running dtheta row after the plane rows
        if (rr < nrows || (is_dt && fz)) {
          if (FULL) {
            const uint32_t d = base_s + 4u * (rr * LS) + 16u * lane;
            if (lane < 8 * EPL) cp_async_u32(d, rsrc[rr], 16);
            if (lane + 32 < 8 * EPL) cp_async_u32(d + 512u, rsrc[rr] + 128, 16);
          } else if (nvalid > 0) {
            const float* src = (is_dt ? dtsb : rowb[rr < NRMAX ? rr : 0]) + ocur;
            cp_slice_t<EPL, false>(base_s + 4u * (rr * LS + l0), src + l0, nvalid);
          }
        }
        if (FULL) rsrc[rr] -= stL;
      }
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint32_t pdst = base_s + 4u * ((NR + 1) * LS);
      if (FULL) {
        if (lane < 2 * EPL) cp_async_u32(pdst + 16u * lane, psrc, 16);
        psrc -= L;
      } else {
        const size_t pb = size_t(e) * L;
        const uint32_t* pwd = reinterpret_cast<const uint32_t*>(a.p) + (pb >> 2);
        const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
        for (int u = lane; u < nwords; u += 32) cp_async_u32(pdst + 4u * u, pwd + u, 4);
      }
      const uint32_t xdst = pdst + 4u * (8 * EPL);
      const int cur = ld.first + j * st;
      const int wnode = (r & 1) ? cur : cur - st;
      if (lane == 0) cp_async_u32(xdst, reinterpret_cast<const uint32_t*>(a.q) + (e >> 2), 4);
      if (wpl && lane == 1) cp_async_u32(xdst + 4u, wrow + wnode, 4);
      if (rpl && lane == 2) cp_async_u32(xdst + 8u, rrow + wnode, 4);
      if (rpl) {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr) {
          if (rr < nrows && sd[rr] >= 0) {
            const int d = sd[rr];
            const int wn = (d & 1) ? cur + g.node_step[d] : cur;
            cp_async_u32(xdst + 4u * (4 + 32 * rr + lane),
                         a.pot.rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + min(max(wn, 0), N - 1), 4);
          }
        }
      }
    };
#pragma unroll
    for (int t = 0; t < kWarpStages - 1; ++t) {
      if (t < nsteps) issue(t);
      cp_commit();
    }
    // the tail is no edge's prev: its plane-r row is zero
    {
      float zero[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) zero[i] = 0.0f;
      stg_slice<EPL>(aout_r + o_first + nsteps * stL, l0, zero, nvalid, L);
    }
    float carry[EPL], accl[EPL], rhol = 0.0f;
    float vacc[EPL][3], fval[EPL];
    int fkey = -1;
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = accl[i] = fval[i] = vacc[i][0] = vacc[i][1] = vacc[i][2] = 0.0f;
    auto flush_far = [&]() {
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (fval[i] != 0.0f) red_add_global(gvacc + fkey * vs_mu + (l0 + i) * vs_l, fmul(fval[i], wfold));
        fval[i] = 0.0f;
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

    for (int s = 0; s < nsteps; ++s) {
      if (s + kWarpStages - 1 < nsteps) issue(s + kWarpStages - 1);
      cp_commit();
      cp_wait<kWarpStages - 1>();
      __syncwarp();  // rows and words were copied by other lanes
      const float* stg = ring + (s % kWarpStages) * stage_f;
      const int j = nsteps - s;
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint8_t* prow0 = reinterpret_cast<const uint8_t*>(stg + (NR + 1) * LS) + (FULL ? 0 : ((size_t(e) * L) & 3));
      const uint8_t* prow = prow0 + l0;
      const float* xs = stg + (NR + 1) * LS + 8 * EPL;
      const int qv = (__float_as_uint(xs[0]) >> (8 * (e & 3))) & 0xff;
      const float w = wpl ? xs[1] : a.pot.w;
      const float rho = TRWP ? (rpl ? xs[2] : a.pot.rho) : 1.0f;

      // ---- x = gm^r(cur) without the carry, rsum = sum_d rho_d A[d](cur)
      float x[EPL], tv[EPL], rsum[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) x[i] = rsum[i] = 0.0f;
      if (!rpl) {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr) {
          if (rr >= a0 && rr < npl) {
            lds_slice<EPL>(tv, stg + rr * LS + l0);
#pragma unroll
            for (int i = 0; i < EPL; ++i) x[i] = fadd(x[i], tv[i]);
          }
        }
        if (TRWP && npl > a0) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) rsum[i] = x[i] = fmul(a.pot.rho, x[i]);
          if (opp_slot >= 0) {
            lds_slice<EPL>(tv, stg + opp_slot * LS + l0);
#pragma unroll
            for (int i = 0; i < EPL; ++i) x[i] = fsub(x[i], tv[i]);
          }
        }
        if (first) {
          lds_slice<EPL>(tv, stg + l0);
#pragma unroll
          for (int i = 0; i < EPL; ++i) x[i] = fadd(tv[i], x[i]);
        }
      } else {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr) {
          if (rr < npl) {
            lds_slice<EPL>(tv, stg + rr * LS + l0);
            const int dd = sd[rr];
            const float rd = xs[4 + 32 * rr + lane];
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              float c = tv[i];
              if (dd >= 0) {
                c = fmul(rd, tv[i]);
                rsum[i] = fadd(rsum[i], c);
                if (dd == opp) c = fsub(c, tv[i]);
              }
              x[i] = fadd(x[i], c);
            }
          }
        }
      }

      // ---- decode p: near codes (l-1 / l / l+1) and far targets
      int mu[EPL];
      bool far[EPL];
      float lsum = 0.0f;
      uint32_t mword = 0;
      int kmn = 0x7fffffff, kmx = -1;
      if (FULL && EPL % 2 == 0) {
#pragma unroll
        for (int i = 0; i < EPL; i += 2) {
          const uint32_t v = *reinterpret_cast<const uint16_t*>(prow + i);
          mu[i] = int(v & 0xffu), mu[i + 1] = int(v >> 8);
        }
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const bool valid = FULL || i < nvalid;
        if (!valid) x[i] = 0.0f;
        lsum = fadd(lsum, x[i]);
        if (!(FULL && EPL % 2 == 0)) mu[i] = valid ? int(prow[i]) : l0 + i;
        const uint32_t c = uint32_t(mu[i] - (l0 + i) + 1);  // 0, 1, 2: target l-1, l, l+1
        const bool nr = valid && c <= 2u;
        mword |= nr ? (1u << (8 * c + i)) : 0u;
        far[i] = valid && !nr;
        kmn = min(kmn, far[i] ? mu[i] : 0x7fffffff);
        kmx = max(kmx, far[i] ? mu[i] : -1);
      }
      const float S = warp_sum_f(lsum);
      kmn = __reduce_min_sync(0xffffffffu, kmn);
      kmx = __reduce_max_sync(0xffffffffu, kmx);
      int main_t = kmx;  // -1: no far label
      const bool split = kmx >= 0 && kmn != kmx;
      if (split) {
        // several far targets: the main one is the most frequent among
        // {target of label 0, of label L-1, smallest, largest}
        const int c0 = __shfl_sync(0xffffffffu, far[0] ? mu[0] : kmn, 0);
        int lastv = kmx;
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          if (l0 + i == L - 1 && far[i]) lastv = mu[i];
        const int c1 = __shfl_sync(0xffffffffu, lastv, (L - 1) / EPL);
        const int cand[4] = {c0, c1, kmn, kmx};
        int bestn = 0;
#pragma unroll
        for (int cI = 0; cI < 4; ++cI) {
          int cnt = 0;
#pragma unroll
          for (int i = 0; i < EPL; ++i) cnt += (far[i] && mu[i] == cand[cI]) ? 1 : 0;
          cnt = int(__reduce_add_sync(0xffffffffu, uint32_t(cnt)));
          if (cnt > bestn) bestn = cnt, main_t = cand[cI];
        }
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) mword |= (far[i] && mu[i] == main_t ? 1u : 0u) << (24 + i);
      int noth = 0;
      if (split) {
        // remaining far pairs, compacted in (element, lane) order
        uint32_t lanemask_lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lanemask_lt));
        __syncwarp();  // the previous step's list reads are done
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const bool o = far[i] && mu[i] != main_t;
          const uint32_t ball = __ballot_sync(0xffffffffu, o);
          if (o) olist[noth + __popc(ball & lanemask_lt)] = uint16_t((l0 + i) | (mu[i] << 8));
          noth += __popc(ball);
        }
        __syncwarp();
      }

      // ---- acc = scatter(x + carry) - S e_{p_q}
      float row[EPL], acc[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) row[i] = fadd(x[i], carry[i]), acc[i] = 0.0f;
      scatter_row<EPL, true, false>(acc, row, mword, main_t, noth, olist, nullptr, lane);
      {
        const int im = int(prow0[qv]) - l0;
#pragma unroll
        for (int i = 0; i < EPL; ++i)
          if (im == i) acc[i] = fsub(acc[i], S);
      }
      stg_slice<EPL>(aout_r + o_first + (j - 1) * stL, l0, acc, nvalid, L);
      if (fz) {  // dtheta(cur) = dtheta + sum_d rho_d A[d](cur) + this sweep's share (the carry)
        float dto[EPL], dt[EPL];
        lds_slice<EPL>(dto, stg + nrows * LS + l0);
#pragma unroll
        for (int i = 0; i < EPL; ++i) dt[i] = fadd(fadd(dto[i], rsum[i]), carry[i]);
        stg_slice<EPL>(dthb + o_first + j * stL, l0, dt, nvalid, L);
      }

      // ---- reparametrised row g = x + carry - S e_q: dV and dw of this edge
      float gg[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) gg[i] = qv == l0 + i ? fsub(row[i], S) : row[i];
      if (main_t != fkey) {  // warp-uniform
        if (fkey >= 0) flush_far();
        fkey = main_t;
      }
      float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const float ga = wpl ? fmul(gg[i], w) : gg[i];  // dV addend (w folded at flush when constant)
        const bool cm = bit(mword, i), c0 = bit(mword, 8 + i), cp = bit(mword, 16 + i), cf = bit(mword, 24 + i);
        if (cm) vacc[i][0] = fadd(vacc[i][0], ga);
        if (c0) vacc[i][1] = fadd(vacc[i][1], ga);
        if (cp) vacc[i][2] = fadd(vacc[i][2], ga);
        if (cf) fval[i] = fadd(fval[i], ga);
        if (c0) s0 = fadd(s0, gg[i]);
        if (cm || cp) s1 = fadd(s1, gg[i]);
      }
      for (int t = 0; t < noth; ++t) {  // the other far pairs (rare): dV (tgt, src) += g_src w
        const int src = olist[t] & 0xff, tgt = olist[t] >> 8;
        const float gv = __shfl_sync(0xffffffffu, sel_elem<EPL>(gg, src % EPL), src / EPL);
        if (lane == 0 && gv != 0.0f) red_add_global(gvacc + tgt * vs_mu + src * vs_l, fmul(gv, w));
      }
      if (do_w) {
        // dw = g(0) s0 + g(1) s1 + g(D) (sum_l g_l - s0 - s1), sum_l g_l = 0
        // (the reparametrised row sums to zero), far pairs included in g(D)
        s_wp[(s & 31) * 33 + lane] = fadd(fmul(fsub(gb0, gbD), s0), fmul(fsub(gb1, gbD), s1));
        if ((s & 31) == 31 || s == nsteps - 1) flush_w(s & ~31, (s & 31) + 1);
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        accl[i] = acc[i];
        carry[i] = TRWP ? fmul(rho, acc[i]) : acc[i];
      }
      rhol = rho;
    }
    if (fz) {
      // the head is no edge's cur: dtheta(head) = dtheta + sum_{d != 0} rho_d A[d](head) + rho acc_last
      const int head = ld.first;
      float hs[EPL], t[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) hs[i] = 0.0f;
      for (int d = 1; d < R; ++d) {
        float rd = a.pot.rho;
        if (rpl) {
          const int wn = (d & 1) ? head + g.node_step[d] : head;
          rd = __ldg(a.pot.rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + min(max(wn, 0), N - 1));
        }
        const float* src = ainb + size_t(d) * NL + size_t(head) * L;
#pragma unroll
        for (int i = 0; i < EPL; ++i) t[i] = (FULL || i < nvalid) ? __ldcg(src + l0 + i) : 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) hs[i] = fadd(hs[i], fmul(rd, t[i]));
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (FULL || i < nvalid) {
          const size_t o = size_t(head) * L + l0 + i;
          dthb[o] = fadd(fadd(dtsb[o], hs[i]), nsteps > 0 ? fmul(rhol, accl[i]) : 0.0f);
        }
      }
    }
    if (fkey >= 0) flush_far();
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int l = l0 + i;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        const int m = l + t - 1;
        if (l < L && m >= 0 && m < L && vacc[i][t] != 0.0f)
          red_add_global(gvacc + m * vs_mu + l * vs_l, fmul(vacc[i][t], wfold));
      }
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
