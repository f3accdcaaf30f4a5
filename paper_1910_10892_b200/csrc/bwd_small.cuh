// Backward sweep for small label sets (L <= 32), one warp per scanline, lane
// = label (sm_100a). isgmr_backward / trwp_backward (autodiff.hpp:63-126,
// :133-197) over the per-direction scatter planes of bwd_common.cuh, for the
// many-short-lines regime (the segmentation config: 21 labels, batch 32,
// 16384 scanlines per sweep) where per-line latency is hidden by occupancy
// and the warp-specialised kernel's per-node hand-offs would dominate.
//
// Per node (reverse order): x = gm^r(cur) from the scatter planes, row = x +
// carry, S = sum(row) (exact, the reference's :48-53), and the scatter
// acc[mu] = sum_{l : p_l = mu} g_l is a gather: the warp publishes (g_l, p_l)
// in shared memory and lane mu sums the rows that point at it in ascending l
// -- the reference's own accumulation order, deterministic, for any V.
// dV partials go to a per-warp shared [L][32] accumulator (one writer per
// entry and step: lane l owns column l), flushed with RED at the end of a
// line; the per-edge dw terms g_l V'(p_l, l) are parked [32 edges][L] and
// summed in ascending l by one lane per edge, 32 edges at a time. V' of both
// orientations is shared by the CTA. For TRWP-4 with a constant rho (C4) the
// direction and the first-iteration flag are compile-time constants of the
// node loop (every staged row and select static).
#pragma once

#include <type_traits>

#include "bwd_common.cuh"
#include "fwd_warp.cuh"

#ifndef MRF_BSMALL_STAGES
#define MRF_BSMALL_STAGES 3  // cp.async ring depth of the small-L backward (3 vs 4: 7 CTAs per SM at L = 21)
#endif
#ifndef MRF_BSMALL_MINB
#define MRF_BSMALL_MINB 7  // CTAs per SM the register budget is sized for (7 x 4 warps: 73 registers)
#endif

namespace mrf {

// per-warp ring stage (floats, 16 B multiple): NR rows + the running-dtheta
// row of 32 floats, p (12 words: L bytes from any offset), {q, w, rho, pad},
// rho_d[NR]
__host__ __device__ constexpr int small_stage_floats(int NR) { return ((NR + 1) * 32 + 16 + NR + 3) / 4 * 4; }
constexpr int kSmallStages = MRF_BSMALL_STAGES;
// per-edge dw terms parked [kPark edges][L labels] with an odd row stride
// (conflict-free both ways) and summed kPark edges at a time
constexpr int kPark = 16;
__host__ __device__ constexpr int small_part_stride(int L) { return L | 1; }
// per warp: ring + (g, source mask) exchange [64] + dV [L][32] + dw parking
// (C4, L = 21: 31.2 KB per 4-warp CTA with 3 ring stages and 16 parked
// edges: 7 CTAs per SM; 38.5 KB with 4 stages and 32 edges: 5. The kernel is
// latency-bound, 5 -> 6 -> 7 CTAs took its sweeps 59.2 -> 55.0 -> 53.4 ms per step)
__host__ __device__ constexpr int small_warp_floats(int NR, int L) {
  return (kSmallStages * small_stage_floats(NR) + 64 + L * 32 + kPark * small_part_stride(L) + 3) / 4 * 4;
}
// per CTA: V'(mu, l) of both orientations [2][L][32] (lane l reads column l:
// conflict-free for any mu), then the warps
__host__ __device__ constexpr int small_cta_floats(int NR, int L, int wpc) {
  return 2 * L * 32 + wpc * small_warp_floats(NR, L);
}

template <bool TRWP, int RT>
__global__ void __launch_bounds__(128, MRF_BSMALL_MINB) bwd_small_kernel(AccArgs a) {
  extern __shared__ __align__(16) float smem[];
  constexpr int NRMAX = RT ? acc_rows(TRWP, RT) : 16;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int NR = acc_rows(TRWP, R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int stage_f = small_stage_floats(NR);
  const int PS = small_part_stride(L);
  float* s_vall = smem;  // [2][L][32]
  float* ring = smem + 2 * L * 32 + size_t(wid) * small_warp_floats(NR, L);
  float* s_g = ring + kSmallStages * stage_f;                      // [32] g
  uint32_t* s_m = reinterpret_cast<uint32_t*>(s_g + 32);      // [32] source masks per target
  float* s_dv = s_g + 64;                                     // [L][32]: (mu, l)
  float* s_part = s_dv + L * 32;                              // [kPark][PS] per-edge dw terms
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));

  const int b = blockIdx.y;
  const int NL = N * L;
  const bool valid = lane < L;
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const bool do_w = a.gw != nullptr;
  const bool fuse = TRWP && a.dtheta != nullptr;
  const float* dcb = a.dc + size_t(b) * NL + lane;
  const float* ainb = a.ain + size_t(b) * R * NL + lane;
  float* aoutb = a.aout + size_t(b) * R * NL + lane;
  float* dthb = fuse ? a.dtheta + size_t(b) * NL : nullptr;
  const float* dths = fuse ? a.dtheta_src + size_t(b) * NL : nullptr;  // running dtheta (dc on the first update)
  const uint8_t* pimg = a.p;
  const uint8_t* qimg = a.q;
  const int warp_global = blockIdx.x * wpc + wid;
  if (do_w) {  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
    for (int t = threadIdx.x; t < 2 * L * 32; t += blockDim.x) {
      const int o = t >= L * 32, rem = t - (o ? L * 32 : 0), mu = rem >> 5, l = rem & 31;
      s_vall[t] = l < L ? __ldg(a.pot.V + (o ? l * L + mu : mu * L + l)) : 0.0f;
    }
    __syncthreads();
  }
  for (int t = lane; t < L * 32; t += 32) s_dv[t] = 0.0f;

  for (int li = warp_global; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    // the line body; RD / FT >= 0: direction / first-iteration flag as
    // compile-time constants, -1: runtime
    auto sweep = [&](auto rd_tag, auto ft_tag) {
    constexpr int RD = decltype(rd_tag)::value;
    constexpr int FT = decltype(ft_tag)::value;
    const int r = RD >= 0 ? RD : ld.dir;
    const bool first = FT >= 0 ? FT == 1 : a.k == g.K_cap - 1;
    const int opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    const int stL = st * L;
    const int o_first = ld.first * L;
    // this warp's private dV slot, V orientation (bwd_common.cuh)
    float* gvacc = a.gvacc + (size_t(b) * a.dv_slots + warp_global) * L * L;
    const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
    const float* s_v = s_vall + ((r & 1) ? L * 32 : 0);
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    float* gwrow = do_w ? a.gw + (TRWP ? (size_t(b) * (R / 2) + fam) * N : (size_t(b) * R + r) * N) : nullptr;

    // rows gm^r(cur) is assembled from, in accumulation order (-1 = dc)
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
      if (!first) {
#pragma unroll
        for (int d = NRMAX - 1; d >= 0; --d)
          if (d < r) push(d);
      }
#pragma unroll
      for (int d = NRMAX - 1; d >= 0; --d)
        if (d < R && d > r) push(d);
    } else if (!first) {
      for (int d = 0; d < R; ++d)
        if (d != r && d != opp) push(d);
    }
    const int a0 = first ? 1 : 0;
    const int npl = nrows;  // plane rows end here
    // edge index over the whole batch: p/q words are addressed from a.p/a.q so
    // that byte offsets stay word-aligned for any b, K_cap and E (K*E odd)
    const uint32_t ebase = (uint32_t(b) * uint32_t(g.K_cap) + uint32_t(a.k)) * uint32_t(g.E) + uint32_t(g.dir_offset[r]) + uint32_t(ld.edge_base);
    const float* rowb[NRMAX];  // this lane's element of each staged row, at node 0
#pragma unroll
    for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] = sd[rr] < 0 ? dcb : ainb + size_t(sd[rr] > 0 ? sd[rr] : 0) * NL;

    // incremental issue state: row pointers at node cur, ring slot, edge
    // (index and p byte offset), all stepped back one node per issue
#pragma unroll
    for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] += o_first + nsteps * stL;
    const float* dtp = fuse ? dths + o_first + nsteps * stL + lane : nullptr;
    int islot = 0, cur_i = ld.first + nsteps * st;
    uint32_t e_i = ebase + uint32_t(nsteps - 1);
    size_t pb_i = size_t(e_i) * L;
    auto issue = [&](int /*s*/) {
      const uint32_t base_s = ring_s + 4u * uint32_t(islot * stage_f);
      if (valid) {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr)
          if (rr < nrows)
            cp_async_u32(base_s + 4u * (rr * 32 + lane), rowb[rr], 4);
        if (fuse) cp_async_u32(base_s + 4u * (NR * 32 + lane), dtp, 4);
      }
#pragma unroll
      for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] -= stL;
      if (fuse) dtp -= stL;
      const uint32_t e = e_i;
      const size_t pb = pb_i;
      const int cur = cur_i;
      --e_i, pb_i -= L, cur_i -= st;
      islot = islot == kSmallStages - 1 ? 0 : islot + 1;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg + (pb & ~size_t(3)));
      const int nwords = int(((uint32_t(pb) & 3u) + uint32_t(L) + 3u) >> 2);
      const uint32_t pdst = base_s + 4u * ((NR + 1) * 32);
      if (lane < nwords) cp_async_u32(pdst + 4u * lane, pw + lane, 4);
      const uint32_t xdst = pdst + 4u * 12;
      const int wnode = (r & 1) ? cur : cur - st;
      if (lane == 0) cp_async_u32(xdst, reinterpret_cast<const uint32_t*>(qimg) + (e >> 2), 4);
      if (wpl && lane == 1) cp_async_u32(xdst + 4u, wrow + wnode, 4);
      if (rpl && lane == 2) cp_async_u32(xdst + 8u, rrow + wnode, 4);
      if (rpl && lane < NRMAX) {
        const int rr = lane;
        if (rr < nrows && sd[rr] >= 0) {
          const int d = sd[rr];
          const int wn = (d & 1) ? cur + g.node_step[d] : cur;
          cp_async_u32(xdst + 4u * (4 + rr), a.pot.rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + min(max(wn, 0), N - 1),
                       4);
        }
      }
    };
#pragma unroll
    for (int s = 0; s < kSmallStages - 1; ++s) {
      if (s < nsteps) issue(s);
      cp_commit();
    }
    // the tail is no edge's prev: its plane-r row is zero
    if (valid) aoutb[size_t(r) * NL + o_first + nsteps * stL] = 0.0f;
    float carry = 0.0f;

    int cslot = 0;
    float* aout_p = aoutb + size_t(r) * NL + o_first + (nsteps - 1) * stL;  // A row of step 0's prev
    float* dto_p = fuse ? dthb + o_first + nsteps * stL + lane : nullptr;     // dtheta(cur) of step 0
    for (int s = 0; s < nsteps; ++s) {
      if (s + kSmallStages - 1 < nsteps) issue(s + kSmallStages - 1);
      cp_commit();
      cp_wait<kSmallStages - 1>();
      __syncwarp();  // p / q words were copied by other lanes
      const float* stg = ring + cslot * stage_f;
      cslot = cslot == kSmallStages - 1 ? 0 : cslot + 1;
      const int j = nsteps - s;
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint8_t* prow = reinterpret_cast<const uint8_t*>(stg + (NR + 1) * 32) + ((e * uint32_t(L)) & 3u);
      const float* xs = stg + (NR + 1) * 32 + 12;
      const int qv = (__float_as_uint(xs[0]) >> (8 * (e & 3))) & 0xff;
      const float w = wpl ? xs[1] : a.pot.w;
      const float rho = TRWP ? (rpl ? xs[2] : a.pot.rho) : 1.0f;

      // ---- x (bwd_common.cuh rules) and row = x + carry
      float x = 0.0f, rsum = 0.0f;
      if (!rpl) {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr)
          if (rr >= a0 && rr < npl) x = fadd(x, stg[rr * 32 + lane]);
        if (TRWP && npl > a0) {
          rsum = x = fmul(a.pot.rho, x);
          if (opp_slot >= 0) x = fsub(x, stg[opp_slot * 32 + lane]);
        }
        if (first) x = fadd(stg[lane], x);
      } else {
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr) {
          if (rr >= npl) continue;
          const float t = stg[rr * 32 + lane];
          float c = t;
          if (sd[rr] >= 0) {
            c = fmul(xs[4 + rr], t);
            rsum = fadd(rsum, c);
            if (sd[rr] == opp) c = fsub(c, t);
          }
          x = fadd(x, c);
        }
      }
      const float row = valid ? fadd(x, carry) : 0.0f;
      const int mu = valid ? int(prow[lane]) : 0;

      // ---- scatter acc[mu] = sum_{l : p_l = mu} g_l with g = row - S e_q
      // (:48-53): the largest group of equal targets by one warp reduction
      // (its row sum F' runs beside S's; F = F' - S when q is in the group),
      // every other group gathered by its target lane from the group's lane
      // mask (ascending l)
      const uint32_t grp = __match_any_sync(0xffffffffu, valid ? mu : -1 - lane);
      const uint32_t key = valid ? (uint32_t(__popc(grp)) << 8) | uint32_t(255 - mu) : 0u;
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
      const int main_mu = 255 - int(kmax & 0xffu);
      const bool in_main = valid && mu == main_mu;
      float S = row, Fp = in_main ? row : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float s2 = __shfl_xor_sync(0xffffffffu, S, o), f2 = __shfl_xor_sync(0xffffffffu, Fp, o);
        S = fadd(S, s2), Fp = fadd(Fp, f2);
      }
      const float gl = lane == qv ? fsub(row, S) : row;  // reparametrised row
      const bool q_main = __shfl_sync(0xffffffffu, in_main ? 1 : 0, qv & 31) != 0;
      const float F = q_main ? fsub(Fp, S) : Fp;
      s_m[lane] = 0u;
      s_g[lane] = gl;
      __syncwarp();
      if (valid && !in_main) s_m[mu] = grp;  // every member writes the same mask
      __syncwarp();
      uint32_t m = s_m[lane];
      const int nit = int(__reduce_max_sync(0xffffffffu, uint32_t(__popc(m))));
      float acc = lane == main_mu ? F : 0.0f;
      // two sources per trip (ascending): both loads in flight
      for (int it = 0; it < nit; it += 2) {
        const int k1 = __ffs(m) - 1;
        m &= m - 1;
        const int k2 = __ffs(m) - 1;
        m &= m - 1;
        const float v1 = s_g[k1 >= 0 ? k1 : 0], v2 = s_g[k2 >= 0 ? k2 : 0];
        if (k1 >= 0) acc = fadd(acc, v1);
        if (k2 >= 0) acc = fadd(acc, v2);
      }
      if (valid) *aout_p = acc;
      aout_p -= stL;
      // fused unary gradient: dtheta(cur) += sum_d rho_d A[d](cur) + this sweep's share
      if (fuse && valid) *dto_p = fadd(fadd(stg[NR * 32 + lane], rsum), carry);
      if (fuse) dto_p -= stL;
      carry = TRWP ? fmul(rho, acc) : acc;

      // ---- dV (shared accumulator, w folded per edge) and dw of this edge
      if (valid && gl != 0.0f) s_dv[mu * 32 + lane] = fadd(s_dv[mu * 32 + lane], fmul(gl, w));
      if (do_w) {
        if (valid) s_part[(s & (kPark - 1)) * PS + lane] = gl != 0.0f ? fmul(gl, s_v[mu * 32 + lane]) : 0.0f;
        // parked per-edge terms, summed in ascending l by lane e and written
        // kPark edges at a time (one writer per edge)
        if ((s & (kPark - 1)) == kPark - 1 || s == nsteps - 1) {
          __syncwarp();
          const int cnt = (s & (kPark - 1)) + 1, s0 = s & ~(kPark - 1);
          if (lane < cnt) {
            const float* pr = s_part + lane * PS;
            float part = 0.0f;
            for (int l = 0; l < L; ++l) part = fadd(part, pr[l]);
            const int node = ld.first + (nsteps - (s0 + lane)) * st;
            float* dst = gwrow + ((r & 1) ? node : node - st);
            *dst = fadd(*dst, part);
          }
        }
      }
      __syncwarp();  // s_g / s_m / s_part reads done before the next step writes
    }
    cp_wait<0>();
    __syncwarp();
    if (fuse && valid) {  // the head is no edge's cur: its rows are read here
      const int head = ld.first;
      float hs = 0.0f;
      for (int d = 1; d < R; ++d) {
        float rd = a.pot.rho;
        if (rpl) {
          const int wn = (d & 1) ? head + g.node_step[d] : head;
          rd = __ldg(a.pot.rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + min(max(wn, 0), N - 1));
        }
        hs = fadd(hs, fmul(rd, __ldcg(ainb + size_t(d) * NL + size_t(head) * L)));
      }
      dthb[size_t(head) * L + lane] = fadd(fadd(dths[size_t(head) * L + lane], hs), carry);
    }
    // flush this line's dV partials (lane l owns column l)
    if (valid) {
      for (int m = 0; m < L; ++m) {
        const float v = s_dv[m * 32 + lane];
        if (v != 0.0f) {
          red_add_global(gvacc + m * vs_mu + lane * vs_l, v);
          s_dv[m * 32 + lane] = 0.0f;
        }
      }
    }
    __syncwarp();
    };
    using M1 = std::integral_constant<int, -1>;
    if constexpr (TRWP && RT == 4) {
      if (!rpl) {
        const int fl = a.k == g.K_cap - 1 ? 1 : 0;
        switch (ld.dir * 2 + fl) {
          case 0: sweep(std::integral_constant<int, 0>(), std::integral_constant<int, 0>()); break;
          case 1: sweep(std::integral_constant<int, 0>(), std::integral_constant<int, 1>()); break;
          case 2: sweep(std::integral_constant<int, 1>(), std::integral_constant<int, 0>()); break;
          case 3: sweep(std::integral_constant<int, 1>(), std::integral_constant<int, 1>()); break;
          case 4: sweep(std::integral_constant<int, 2>(), std::integral_constant<int, 0>()); break;
          case 5: sweep(std::integral_constant<int, 2>(), std::integral_constant<int, 1>()); break;
          case 6: sweep(std::integral_constant<int, 3>(), std::integral_constant<int, 0>()); break;
          default: sweep(std::integral_constant<int, 3>(), std::integral_constant<int, 1>()); break;
        }
      } else {
        sweep(M1(), M1());
      }
    } else {
      sweep(M1(), M1());
    }
  }
}

}  // namespace mrf
