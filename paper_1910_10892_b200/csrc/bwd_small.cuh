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
// dV partials go to a per-warp shared [L][L] accumulator (one writer per
// entry and step: lane l owns column l), flushed with RED at the end of a
// line; dw per edge is a warp sum parked 32 edges at a time.
#pragma once

#include "bwd_common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

// per-warp ring stage: NR rows of 32 floats + p (12 words: L bytes from any
// offset) + {q, w, rho, pad} + rho_d[NR]
__host__ __device__ constexpr int small_stage_floats(int NR) { return NR * 32 + 12 + 4 + NR; }
// ring + (g, p) exchange [32] float2 + dV [32][32] + dw parking [32] + V' [32][33]
__host__ __device__ constexpr int small_warp_floats(int NR) {
  return (kStages * small_stage_floats(NR) + 64 + 32 * 32 + 32 + 32 * 33 + 31) / 32 * 32;
}

template <bool TRWP, int RT>
__global__ void __launch_bounds__(128) bwd_small_kernel(AccArgs a) {
  extern __shared__ __align__(16) float smem[];
  constexpr int NRMAX = RT ? acc_rows(TRWP, RT) : 16;
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int NR = acc_rows(TRWP, R);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int stage_f = small_stage_floats(NR);
  float* ring = smem + size_t(wid) * small_warp_floats(NR);
  float2* s_gp = reinterpret_cast<float2*>(ring + kStages * stage_f);  // [32] (g, p)
  float* s_dv = ring + kStages * stage_f + 64;                         // [32][32]: (mu, l)
  float* s_wp = s_dv + 32 * 32;                                         // [32] parked per-edge dw
  float* s_v = s_wp + 32;                                               // [32][33]: V'(mu, l) of orientation r&1
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));

  const int b = blockIdx.y;
  const int NL = N * L;
  const bool first = a.k == g.K_cap - 1;
  const bool valid = lane < L;
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const bool do_w = a.gw != nullptr;
  const float* dcb = a.dc + size_t(b) * NL + lane;
  const float* ainb = a.ain + size_t(b) * R * NL + lane;
  float* aoutb = a.aout + size_t(b) * R * NL + lane;
  const uint8_t* pimg = a.p;
  const uint8_t* qimg = a.q;
  const int warp_global = blockIdx.x * wpc + wid;
  for (int t = lane; t < 32 * 32; t += 32) s_dv[t] = 0.0f;
  int v_orient = -1;

  for (int li = warp_global; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    const int stL = st * L;
    const int o_first = ld.first * L;
    // this warp's private dV slot, V orientation (bwd_common.cuh)
    float* gvacc = a.gvacc + (size_t(b) * a.dv_slots + warp_global) * L * L;
    const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    float* gwrow = do_w ? a.gw + (TRWP ? (size_t(b) * (R / 2) + fam) * N : (size_t(b) * R + r) * N) : nullptr;
    if (do_w && v_orient != (r & 1)) {  // V'(mu, l) = V(mu, l) (even r) / V(l, mu) (odd r)
      v_orient = r & 1;
      __syncwarp();
      for (int t = lane; t < L * L; t += 32) {
        const int mu = t / L, l = t - mu * L;
        s_v[mu * 33 + l] = __ldg(a.pot.V + (v_orient ? l * L + mu : t));
      }
      __syncwarp();
    }

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
      if (!first)
        for (int d = r - 1; d >= 0; --d) push(d);
      for (int d = R - 1; d > r; --d) push(d);
    } else if (!first) {
      for (int d = 0; d < R; ++d)
        if (d != r && d != opp) push(d);
    }
    const int a0 = first ? 1 : 0;
    const int npl = nrows;  // plane rows end here
    const bool fuse = TRWP && a.dtheta != nullptr;
    float* dthb = fuse ? a.dtheta + size_t(b) * NL : nullptr;
    const float* dths = fuse ? a.dtheta_src + size_t(b) * NL : nullptr;  // running dtheta (dc on the first update)
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
      }
#pragma unroll
      for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] -= stL;
      const uint32_t e = e_i;
      const size_t pb = pb_i;
      const int cur = cur_i;
      --e_i, pb_i -= L, cur_i -= st;
      islot = islot == kStages - 1 ? 0 : islot + 1;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(pimg) + (pb >> 2);
      const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
      const uint32_t pdst = base_s + 4u * (NR * 32);
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
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nsteps) issue(s);
      cp_commit();
    }
    // the tail is no edge's prev: its plane-r row is zero
    if (valid) aoutb[size_t(r) * NL + o_first + nsteps * stL] = 0.0f;
    float carry = 0.0f;
    // fused unary gradient: dtheta(cur) loaded one step ahead
    float dtn = (fuse && valid && nsteps > 0) ? __ldcg(dths + o_first + nsteps * stL + lane) : 0.0f;

    int cslot = 0;
    float* aout_p = aoutb + size_t(r) * NL + o_first + (nsteps - 1) * stL;  // A row of step 0's prev
    for (int s = 0; s < nsteps; ++s) {
      if (s + kStages - 1 < nsteps) issue(s + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      __syncwarp();  // p / q words were copied by other lanes
      const float* stg = ring + cslot * stage_f;
      cslot = cslot == kStages - 1 ? 0 : cslot + 1;
      const int j = nsteps - s;
      const uint32_t e = ebase + uint32_t(j - 1);
      const uint8_t* prow = reinterpret_cast<const uint8_t*>(stg + NR * 32) + ((size_t(e) * L) & 3);
      const float* xs = stg + NR * 32 + 12;
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
      const float S = warp_sum_f(row);
      const float gl = lane == qv ? fsub(row, S) : row;  // reparametrised row (:48-53)

      // ---- scatter acc[mu] = sum_{l : p_l = mu} g_l: the largest group of
      // equal targets by one warp reduction, every other group gathered by
      // its target lane from the group's lane mask (ascending l)
      const uint32_t grp = __match_any_sync(0xffffffffu, valid ? mu : -1 - lane);
      const uint32_t key = valid ? (uint32_t(__popc(grp)) << 8) | uint32_t(255 - mu) : 0u;
      const uint32_t kmax = __reduce_max_sync(0xffffffffu, key);
      const int main_mu = 255 - int(kmax & 0xffu);
      const bool in_main = valid && mu == main_mu;
      const float F = warp_sum_f(in_main ? gl : 0.0f);
      float* s_g = reinterpret_cast<float*>(s_gp);        // [32] g
      uint32_t* s_m = reinterpret_cast<uint32_t*>(s_gp) + 32;  // [32] source masks per target
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
      if (fuse && valid) {
        const float dnew = fadd(fadd(dtn, rsum), carry);
        if (s + 1 < nsteps) dtn = __ldcg(dths + o_first + (j - 1) * stL + lane);
        dthb[o_first + j * stL + lane] = dnew;
      }
      carry = TRWP ? fmul(rho, acc) : acc;

      // ---- dV (shared accumulator, w folded per edge) and dw of this edge
      if (valid && gl != 0.0f) s_dv[mu * 32 + lane] = fadd(s_dv[mu * 32 + lane], fmul(gl, w));
      if (do_w) {
        float part = (valid && gl != 0.0f) ? fmul(gl, s_v[mu * 33 + lane]) : 0.0f;
        part = warp_sum_f(part);
        if (lane == 0) s_wp[s & 31] = part;
        // parked per-edge sums, written 32 edges at a time (one writer per edge)
        if ((s & 31) == 31 || s == nsteps - 1) {
          __syncwarp();
          const int cnt = (s & 31) + 1, s0 = s & ~31;
          if (lane < cnt) {
            const int node = ld.first + (nsteps - (s0 + lane)) * st;
            float* dst = gwrow + ((r & 1) ? node : node - st);
            *dst = fadd(*dst, s_wp[lane]);
          }
        }
      }
      __syncwarp();  // s_gp / s_wp reads done before the next step writes
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
  }
}

}  // namespace mrf
