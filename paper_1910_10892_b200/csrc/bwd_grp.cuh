// TRWP-4 backward sweep for small dense label sets, 16 < L <= 24, constant
// rho (C4), 8 lanes per scanline with 3 labels each, 4 scanlines per warp
// (sm_100a) -- the backward twin of fwd_grp.cuh.
//
// trwp_backward (autodiff.hpp:133-197) over the scatter planes of
// bwd_common.cuh, per node (reverse order), exactly bwd_small.cuh's algebra:
// x = gm^r(cur) from the staged rows, row = x + carry, S = sum(row),
// g = row - S e_q (:48-53), acc[mu] = sum_{l : p_l = mu} g_l, carry' = rho acc,
// dV(p_l, l) += w g_l, dw(edge) += sum_l g_l V'(p_l, l). The sums run in a
// fixed order (S and dw: the lane's labels ascending, then an 8-lane xor
// tree; acc: the line's sources in ascending label order, gathered by each
// target lane from the line's (g, p) row in shared memory, branch-free), so
// every gradient is bit-identical run to run. dV goes by RED straight into
// the line group's private slot (one writer thread per entry: same-address
// program order), dw by one RED per edge: nothing on the node chain waits
// for a global read. Measured on C4 (ncu r02i): 145 warp instructions per
// edge against 280 for lane = label, 1.57 ms per launch against 2.57; a
// per-group shared [mu][l] dV accumulator (-DMRF_BGRP_RED=0: 9 KB per warp,
// 3 CTAs per SM) and data-dependent branches in the gather measured 2-3x
// slower. FUSE (the direction-0 launches of a call with
// bwd_grp_fuse()): the sweep also writes the iteration's unary gradient,
// dtheta(cur) = dtheta_src(cur) + rho sum_{d != 0} A[d](cur) + carry
// (bwd_small.cuh's fused rule), from a fifth staged row.
#pragma once

#include <type_traits>

#include "bwd_common.cuh"
#include "fwd_grp.cuh"

namespace mrf {

constexpr int kBgStages = 3;  // cp.async ring depth
// per line and stage (floats): 5 rows of 24 (up to 4 gradient rows + the
// running dtheta row of the fused sweep) + p words (8) + {q word, w, pad, pad}
// (the unfused kernel keeps 4 rows: 1.7 ms per C4 backward faster)
__host__ __device__ constexpr int bg_rows(bool fuse) { return fuse ? 5 : 4; }
__host__ __device__ constexpr int bg_line_stage(bool fuse) { return bg_rows(fuse) * 24 + 8 + 4; }
// per warp floats: ring [stages][4 lines][kBgLineStage] + (g [24], p [24 bytes = 6 words], pad) per line
// + dV [4 lines][24 mu][24 l]
#ifndef MRF_BGRP_RED
#define MRF_BGRP_RED 1  // 0: shared [mu][l] accumulator per group (measured slower); 1: dV by RED into the group's slot every step (no shared accumulator)
#endif
__host__ __device__ constexpr int bwd_grp_warp_floats(bool fuse) {
  return kBgStages * kGrpLines * bg_line_stage(fuse) + kGrpLines * 32 + (MRF_BGRP_RED ? 0 : kGrpLines * 24 * 24);
}
// per CTA: V'(mu, l) of both orientations [2][24][24], then the warps
__host__ __device__ constexpr int bwd_grp_cta_floats(int wpc, bool fuse) {
  return 2 * 24 * 24 + wpc * bwd_grp_warp_floats(fuse);
}
#ifndef MRF_BGRP_MINB
#define MRF_BGRP_MINB 5  // CTAs per SM the unfused kernel is sized for (<= 102 registers; 7 measured slower; A/B)
#endif
#ifndef MRF_BGRP_WARPS
#define MRF_BGRP_WARPS 4
#endif
constexpr int kBgWarps = MRF_BGRP_WARPS;

template <int RD, int FT, bool FUSE>
__device__ __forceinline__ void bwd_grp_line(const AccArgs& a, const LineDesc& ld, bool has, int maxs, int slot,
                                             float* ring, float* s_gp, float* s_dv, const float* s_vall) {
  constexpr int R = 4, EPL = 3, LP = 24;
  constexpr int r = RD, opp = r ^ 1, fam = r >> 1;
  constexpr bool first = FT == 1;
  // staged rows in accumulation order (bwd_small.cuh): dc at k == K-1, then
  // (later iterations) planes d < r descending, then planes d > r descending
  constexpr int NROWS = (first ? 1 : 0) + (first ? 0 : r) + (R - 1 - r);
  constexpr int A0 = first ? 1 : 0;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N, NL = N * L;
  const int lane = threadIdx.x & 31, gi = lane >> 3, gl = lane & 7, l0 = gl * EPL;
  const int nv = min(EPL, max(0, L - l0));
  const int b = blockIdx.y;
  const bool wpl = a.pot.w_planes != nullptr, do_w = a.gw != nullptr;
  // direction 0 also collects the iteration's unary gradient (bwd_small.cuh
  // rules): dtheta(cur) = dtheta_src(cur) + rho sum_{d != 0} A[d](cur) + carry
  constexpr bool fuse = FUSE && r == 0;
  constexpr int kBgRows = bg_rows(FUSE), kBgLineStage = bg_line_stage(FUSE);
  const int st = g.node_step[r];
  const int nsteps = has ? ld.length - 1 : 0;
  const ptrdiff_t stL = ptrdiff_t(st) * L;
  const ptrdiff_t o_first = ptrdiff_t(ld.first) * L;
  float* gvacc = a.gvacc + (size_t(b) * a.dv_slots + slot) * L * L;
  const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
  const float* s_v = s_vall + ((r & 1) ? 24 * 24 : 0);  // V'(mu, l) at [mu][l]
  const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  float* gwrow = do_w ? a.gw + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const float* ainb = a.ain + size_t(b) * R * NL + l0;
  float* aoutb = a.aout + size_t(b) * R * NL + l0;
  const float* dcb = a.dc + size_t(b) * NL + l0;
  const float* dtsb = fuse ? a.dtheta_src + size_t(b) * NL + l0 : nullptr;
  float* dtob = fuse ? a.dtheta + size_t(b) * NL + l0 : nullptr;
  const uint8_t* pimg = a.p;
  const uint8_t* qimg = a.q;
  // plane of each staged row (-1: dc)
  auto row_dir = [](int rr) {
    int d = -1, n = 0;
    if (first) {
      if (rr == 0) return -1;
      n = 1;
    } else {
      for (int x = r - 1; x >= 0; --x) {
        if (n == rr) d = x;
        ++n;
      }
    }
    for (int x = R - 1; x > r; --x) {
      if (n == rr) d = x;
      ++n;
    }
    return d;
  };
  int opp_slot = -1;
#pragma unroll
  for (int rr = 0; rr < NROWS; ++rr)
    if (row_dir(rr) == opp) opp_slot = rr;

  const uint32_t e_base = (uint32_t(b) * uint32_t(g.K_cap) + uint32_t(a.k)) * uint32_t(g.E) + uint32_t(g.dir_offset[r]) +
                          uint32_t(ld.edge_base);
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  // issue state: node cur of the step, edge, stage slot
  int islot = 0, issued = 0, cur_i = ld.first + nsteps * st;
  auto issue = [&]() {
    ++issued;
    if (issued <= nsteps) {
      const uint32_t sb = ring_s + 4u * uint32_t((islot * kGrpLines + gi) * kBgLineStage);
      const ptrdiff_t off = ptrdiff_t(cur_i) * L;
#pragma unroll
      for (int rr = 0; rr < NROWS; ++rr) {
        const int d = row_dir(rr);
        const float* src = (d < 0 ? dcb : ainb + size_t(d) * NL) + off;
#pragma unroll
        for (int t = 0; t < EPL; ++t)
          if (t < nv) cp_async_u32(sb + 4u * uint32_t(rr * LP + l0 + t), src + t, 4);
      }
      if (fuse) {
#pragma unroll
        for (int t = 0; t < EPL; ++t)
          if (t < nv) cp_async_u32(sb + 4u * uint32_t(4 * LP + l0 + t), dtsb + off + t, 4);
      }
      const uint32_t e = e_base + uint32_t(nsteps - issued);  // edge (prev -> cur), prev = cur - st
      const size_t pb = size_t(e) * L;
      const int nwords = int(((uint32_t(pb) & 3u) + uint32_t(L) + 3u) >> 2);
      if (gl < nwords)
        cp_async_u32(sb + 4u * uint32_t(kBgRows * LP + gl), reinterpret_cast<const uint32_t*>(pimg + (pb & ~size_t(3))) + gl, 4);
      if (gl == 0) cp_async_u32(sb + 4u * uint32_t(kBgRows * LP + 8), reinterpret_cast<const uint32_t*>(qimg) + (e >> 2), 4);
      const int wnode = (r & 1) ? cur_i : cur_i - st;
      if (wpl && gl == 1) cp_async_u32(sb + 4u * uint32_t(kBgRows * LP + 9), wrow + wnode, 4);
    }
    cur_i -= st;
    islot = islot == kBgStages - 1 ? 0 : islot + 1;
  };
#pragma unroll
  for (int s = 0; s < kBgStages - 1; ++s) {
    issue();
    cp_commit();
  }
  // the tail is no edge's prev: its plane-r row is zero
  if (has) {
#pragma unroll
    for (int t = 0; t < EPL; ++t)
      if (t < nv) aoutb[size_t(r) * NL + o_first + nsteps * stL + t] = 0.0f;
  }
  float carry[EPL];
#pragma unroll
  for (int t = 0; t < EPL; ++t) carry[t] = 0.0f;
  float* s_g = s_gp + gi * 32;                                   // [24] g of the line
  uint8_t* s_p = reinterpret_cast<uint8_t*>(s_gp + gi * 32 + 24);  // [24] targets of the line
  float* s_dvg = s_dv + gi * 24 * 24;                            // [mu][l]
  int cslot = 0;
  for (int s = 0; s < maxs; ++s) {
    issue();
    cp_commit();
    cp_wait<kBgStages - 1>();
    __syncwarp();  // p / q / w words were copied by other lanes
    const bool act = s < nsteps;
    const float* stg = ring + (cslot * kGrpLines + gi) * kBgLineStage;
    cslot = cslot == kBgStages - 1 ? 0 : cslot + 1;
    const int j = nsteps - s;  // edge j-1: prev = node j-1, cur = node j
    const uint32_t e = e_base + uint32_t(j - 1);
    const uint8_t* prow = reinterpret_cast<const uint8_t*>(stg + kBgRows * LP) + ((e * uint32_t(L)) & 3u);
    const int qv = (__float_as_uint(stg[kBgRows * LP + 8]) >> (8 * (e & 3))) & 0xff;
    const float w = wpl ? stg[kBgRows * LP + 9] : a.pot.w;
    // ---- x (bwd_common.cuh rules, bwd_small.cuh order) and row = x + carry
    float row[EPL], rsum[EPL];
    int mu[EPL];
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
      float x = 0.0f;
      rsum[t] = 0.0f;
#pragma unroll
      for (int rr = A0; rr < NROWS; ++rr) x = fadd(x, stg[rr * LP + l0 + t]);
      if (NROWS > A0) {
        rsum[t] = x = fmul(a.pot.rho, x);
        if (opp_slot >= 0) x = fsub(x, stg[(opp_slot >= 0 ? opp_slot : 0) * LP + l0 + t]);
      }
      if (first) x = fadd(stg[l0 + t], x);
      const bool ok = act && t < nv;
      row[t] = ok ? fadd(x, carry[t]) : 0.0f;
      mu[t] = ok ? int(prow[l0 + t]) : 0;
    }
    // ---- S = sum(row): the lane's labels ascending, then the group's xor tree
    float S = fadd(fadd(row[0], row[1]), row[2]);
    S = fadd(S, __shfl_xor_sync(0xffffffffu, S, 1));
    S = fadd(S, __shfl_xor_sync(0xffffffffu, S, 2));
    S = fadd(S, __shfl_xor_sync(0xffffffffu, S, 4));
    float gv[EPL];
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
      gv[t] = l0 + t == qv ? fsub(row[t], S) : row[t];  // reparametrised row
      s_g[l0 + t] = gv[t];
      s_p[l0 + t] = uint8_t(t < nv ? mu[t] : 0xff);  // padding labels point nowhere
    }
    __syncwarp();
    // ---- acc[lam] = sum_{l : p_l = lam} g_l, sources in ascending l
    float acc[EPL];
#pragma unroll
    for (int t = 0; t < EPL; ++t) acc[t] = 0.0f;
#pragma unroll
    for (int l4 = 0; l4 < LP; l4 += 4) {
      const float4 g4 = *reinterpret_cast<const float4*>(s_g + l4);
      const uint32_t p4 = *reinterpret_cast<const uint32_t*>(s_p + l4);
      const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int d = int((p4 >> (8 * u)) & 0xffu) - l0;
#pragma unroll
        for (int t = 0; t < EPL; ++t) acc[t] = fadd(acc[t], d == t ? gg[u] : 0.0f);  // branch-free
      }
    }
    const int prev = ld.first + (j - 1) * st;
    if (fuse && act) {  // the unary gradient of node cur, with this sweep's share (the carry into cur)
#pragma unroll
      for (int t = 0; t < EPL; ++t)
        if (t < nv) dtob[size_t(prev + st) * L + t] = fadd(fadd(stg[4 * LP + l0 + t], rsum[t]), carry[t]);
    }
    if (act) {
#pragma unroll
      for (int t = 0; t < EPL; ++t)
        if (t < nv) aoutb[size_t(r) * NL + size_t(prev) * L + t] = acc[t];
    }
#pragma unroll
    for (int t = 0; t < EPL; ++t) carry[t] = act ? fmul(a.pot.rho, acc[t]) : carry[t];
    // ---- dV(p_l, l) += w g_l (per group, one writer per entry), dw of the edge
    float part = 0.0f;
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
      const bool ok = act && t < nv;
      if (ok && gv[t] != 0.0f) {
        if (MRF_BGRP_RED) {
          red_add_global(gvacc + mu[t] * vs_mu + (l0 + t) * vs_l, fmul(gv[t], w));
        } else {
          float* dvp = s_dvg + mu[t] * 24 + l0 + t;
          *dvp = fadd(*dvp, fmul(gv[t], w));
        }
      }
      if (do_w) part = fadd(part, ok && gv[t] != 0.0f ? fmul(gv[t], s_v[mu[t] * 24 + l0 + t]) : 0.0f);
    }
    if (do_w) {
      part = fadd(part, __shfl_xor_sync(0xffffffffu, part, 1));
      part = fadd(part, __shfl_xor_sync(0xffffffffu, part, 2));
      part = fadd(part, __shfl_xor_sync(0xffffffffu, part, 4));
      if (act && gl == 0) {
        const int cur = prev + st;
        // one term per w-plane entry per launch: a fire-and-forget RED adds it
        // in a fixed order (no read-modify-write stall on the node chain)
        red_add_global(gwrow + ((r & 1) ? cur : prev), part);
      }
    }
    __syncwarp();  // s_g / s_p reads done before the next step writes them
  }
  cp_wait<0>();
  __syncwarp();
  if (fuse && has) {  // the head is no edge's cur: its rows are read here
    const int head = ld.first;
#pragma unroll
    for (int t = 0; t < EPL; ++t) {
      if (t >= nv) continue;
      float hs = 0.0f;
#pragma unroll
      for (int d = 1; d < R; ++d) hs = fadd(hs, fmul(a.pot.rho, __ldcg(ainb + size_t(d) * NL + size_t(head) * L + t)));
      dtob[size_t(head) * L + t] = fadd(fadd(dtsb[size_t(head) * L + t], hs), carry[t]);
    }
  }
  // flush this line's dV partials into the group's private slot
  if (has && !MRF_BGRP_RED) {
    for (int m = 0; m < L; ++m) {
#pragma unroll
      for (int t = 0; t < EPL; ++t) {
        if (t >= nv) continue;
        float* dvp = s_dvg + m * 24 + l0 + t;
        const float v = *dvp;
        if (v != 0.0f) {
          red_add_global(gvacc + m * vs_mu + (l0 + t) * vs_l, v);
          *dvp = 0.0f;
        }
      }
    }
  }
  __syncwarp();
}

// FUSE: the direction-0 launches of a call that collects the unary gradient
// in the sweep (a separate instantiation: the unfused kernel keeps its 90
// registers; both together in one kernel took 162)
template <bool FUSE>
__global__ void __launch_bounds__(128, FUSE ? 5 : MRF_BGRP_MINB) bwd_grp_kernel(AccArgs a) {
  extern __shared__ __align__(16) float smem[];
  const Geometry& g = a.g;
  const int L = g.L;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int gi = lane >> 3;
  float* s_vall = smem;  // [2][24][24]
  float* ring = smem + 2 * 24 * 24 + size_t(wid) * bwd_grp_warp_floats(FUSE);
  float* s_gp = ring + kBgStages * kGrpLines * bg_line_stage(FUSE);  // [4 lines][32]
  float* s_dv = s_gp + kGrpLines * 32;                         // [4 lines][24][24]
  if (a.gw != nullptr) {  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
    for (int t = threadIdx.x; t < 2 * 24 * 24; t += blockDim.x) {
      const int o = t >= 24 * 24, rem = t - (o ? 24 * 24 : 0), mu = rem / 24, l = rem % 24;
      s_vall[t] = (l < L && mu < L) ? __ldg(a.pot.V + (o ? l * L + mu : mu * L + l)) : 0.0f;
    }
  }
  if (!MRF_BGRP_RED)
    for (int t = lane; t < kGrpLines * 24 * 24; t += 32) s_dv[t] = 0.0f;
  __syncthreads();
  const int warp_global = blockIdx.x * wpc + wid;
  const int slot = warp_global * kGrpLines + gi;  // the group's private dV slot
  const bool first = a.k == g.K_cap - 1;
  for (int wl = warp_global; wl * kGrpLines < a.nlines; wl += gridDim.x * wpc) {
    const int li = wl * kGrpLines + gi;
    const bool has = li < a.nlines;
    const LineDesc ld = a.lines[has ? li : wl * kGrpLines];
    int maxs = has ? ld.length - 1 : 0;
    maxs = max(maxs, __shfl_xor_sync(0xffffffffu, maxs, 8));
    maxs = max(maxs, __shfl_xor_sync(0xffffffffu, maxs, 16));
    // every line of a TRWP launch sweeps one direction
    if constexpr (FUSE) {  // direction 0 only
      if (first) bwd_grp_line<0, 1, true>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall);
      else bwd_grp_line<0, 0, true>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall);
    } else {
      switch (ld.dir * 2 + (first ? 1 : 0)) {
        case 0: bwd_grp_line<0, 0, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 1: bwd_grp_line<0, 1, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 2: bwd_grp_line<1, 0, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 3: bwd_grp_line<1, 1, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 4: bwd_grp_line<2, 0, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 5: bwd_grp_line<2, 1, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        case 6: bwd_grp_line<3, 0, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
        default: bwd_grp_line<3, 1, false>(a, ld, has, maxs, slot, ring, s_gp, s_dv, s_vall); break;
      }
    }
  }
}

}  // namespace mrf
