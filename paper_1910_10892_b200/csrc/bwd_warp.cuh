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
// registers (neighbour lanes via one shuffle), the rest are summed per
// distinct target with a warp reduction; L <= 32 gathers instead. Every
// read-modify-write row is owned by exactly one warp within a launch
// (scanlines of one direction are node-disjoint), so no atomics are needed
// for dtheta / gm / dw; dV partials use fire-and-forget reductions (RED)
// into a few replicas (near-diagonal ones accumulate in registers first).
// The rows a step touches do not depend on the chain and are prefetched with
// cp.async kStages-1 steps ahead, as in the forward.
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

__host__ __device__ constexpr int bwd_warp_smem_floats(int EPL, int rowsF) {
  return (kStages * (rowsF * 32 * EPL + (32 * EPL) / 4 + 8) + 31) / 32 * 32;
}

template <int EPL>
__device__ __forceinline__ void store_slice(float* row, int l0, const float (&v)[EPL], int nvalid, int L) {
  if (nvalid == EPL && EPL % 4 == 0 && (L & 3) == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 4)
      *reinterpret_cast<float4*>(row + l0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else if (nvalid == EPL && EPL % 2 == 0 && (L & 1) == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2) *reinterpret_cast<float2*>(row + l0 + i) = make_float2(v[i], v[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i)
      if (i < nvalid) row[l0 + i] = v[i];
  }
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int EPL, bool TRWP>
__global__ void __launch_bounds__(128) bwd_warp_kernel(BwdArgs a) {
  extern __shared__ float smem[];
  const Geometry& g = a.g;
  const int L = g.L, N = g.N, R = g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int r = a.r, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
  const int NP = TRWP ? R - 1 : R - 2;
  const int rowsF = 2 + NP;  // gm^r[cur], dtheta[prev], NP gradient planes at prev
  const int LS = 32 * EPL;
  const int stage_f = rowsF * LS + LS / 4 + 8;
  float* ring = smem + size_t(wid) * bwd_warp_smem_floats(EPL, rowsF);

  const int b = blockIdx.y;
  const size_t img = size_t(b) * R * N * L;
  float* gmr = a.gm + img + size_t(r) * N * L;
  float* gub = a.gu + size_t(b) * N * L;
  float* planes_base = TRWP ? a.gm + img : a.gnext + img;
  const int l0 = lane * EPL;
  const int nvalid = min(EPL, max(0, L - l0));
  const int chunk = nvalid == EPL ? Chunk<EPL>::bytes(L) : 4;
  const bool wplanes = a.pot.w_planes != nullptr, rplanes = TRWP && a.pot.rho_planes != nullptr;
  const float* wpl = wplanes ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const float* rpl = rplanes ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
  const int warp_global = blockIdx.x * wpc + wid;
  float* gvacc = a.gvacc + ((size_t(b) * kVRep + warp_global % kVRep) * 2 + (r & 1)) * L * L;
  auto plane_of = [&](int idx) { return TRWP ? (idx < r ? idx : idx + 1) : (idx < (r & ~1) ? idx : idx + 2); };

  float vacc[EPL][3];  // near-diagonal dV partials, (mu = l + delta, l), delta = -1, 0, 1
#pragma unroll
  for (int i = 0; i < EPL; ++i) vacc[i][0] = vacc[i][1] = vacc[i][2] = 0.0f;

  for (int li = warp_global; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int nsteps = ld.length - 1;
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;

    // step s (0-based) handles node position j = nsteps - s (reverse order)
    auto issue = [&](int s) {
      float* slot = ring + (s % kStages) * stage_f;
      const int j = nsteps - s;
      const int cur = ld.first + j * st, prev = cur - st;
      if (nvalid > 0) {
        for (int rr = 0; rr < rowsF; ++rr) {
          const float* src = rr == 0 ? gmr + size_t(cur) * L
                             : rr == 1 ? gub + size_t(prev) * L
                                       : planes_base + (size_t(plane_of(rr - 2)) * N + prev) * L;
          float* dst = slot + rr * LS;
          for (int off = 0; off < nvalid * 4; off += chunk)
            cp_async(reinterpret_cast<char*>(dst + l0) + off, reinterpret_cast<const char*>(src + l0) + off, chunk);
        }
      }
      // p row: the aligned words covering bytes [flat*L, flat*L + L)
      const size_t flat = pq_base + j - 1;
      const size_t pb = flat * L;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(a.p) + (pb >> 2);
      const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
      float* pdst = slot + rowsF * LS;
      for (int t = lane; t < nwords; t += 32) cp_async(pdst + t, pw + t, 4);
      if (lane == 0) {
        float* xs = pdst + LS / 4 + 2;
        cp_async(xs, reinterpret_cast<const uint32_t*>(a.q) + (flat >> 2), 4);
        const int wnode = (r & 1) ? cur : prev;
        if (wplanes) cp_async(xs + 1, wpl + wnode, 4);
        if (rplanes) cp_async(xs + 2, rpl + wnode, 4);
      }
    };

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
      __syncwarp();
      const float* slot = ring + (s % kStages) * stage_f;
      const int j = nsteps - s;
      const int cur = ld.first + j * st, prev = cur - st;
      const size_t flat = pq_base + j - 1;
      const uint8_t* prow = reinterpret_cast<const uint8_t*>(slot + rowsF * LS) + ((flat * L) & 3);
      const float* xs = slot + rowsF * LS + LS / 4 + 2;
      const int qv = (__float_as_uint(xs[0]) >> (8 * (flat & 3))) & 0xff;
      const float w = wplanes ? xs[1] : a.pot.w;
      const float rho = TRWP ? (rplanes ? xs[2] : a.pot.rho) : 1.0f;

      // ---- row = gm^r[cur] + carry; consume (zero) gm^r[cur]; reparam backward
      float row[EPL];
      float lsum = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        row[i] = i < nvalid ? fadd(slot[l0 + i], carry[i]) : 0.0f;
        lsum = fadd(lsum, row[i]);
      }
      {
        float z[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) z[i] = 0.0f;
        store_slice<EPL>(gmr + size_t(cur) * L, l0, z, nvalid, L);
      }
      const float S = warp_sum_f(lsum);
      int pm[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (l0 + i == qv) row[i] = fsub(row[i], S);
        pm[i] = i < nvalid ? int(prow[l0 + i]) : 0;
      }

      // ---- scatter: acc[mu] = sum over l with p[l] = mu of g_l
      float acc[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) acc[i] = 0.0f;
      if (EPL == 1) {
        const float g0 = nvalid ? row[0] : 0.0f;
        for (int lam = 0; lam < L; ++lam) {
          const int pl = __shfl_sync(0xffffffffu, pm[0], lam);
          const float gl = __shfl_sync(0xffffffffu, g0, lam);
          if (pl == lane && gl != 0.0f) acc[0] = fadd(acc[0], gl);
        }
      } else {
        bool rem[EPL];
        float accL = 0.0f, accR = 0.0f;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          rem[i] = false;
          const float gi = row[i];
          if (i >= nvalid || gi == 0.0f) continue;
          const int d = pm[i] - (l0 + i);
          if (d == 0) {
            acc[i] = fadd(acc[i], gi);
          } else if (d == -1) {
            if (i > 0) acc[i - 1 > 0 ? i - 1 : 0] = fadd(acc[i - 1 > 0 ? i - 1 : 0], gi);
            else accL = fadd(accL, gi);
          } else if (d == 1) {
            if (i < EPL - 1) acc[i + 1 < EPL ? i + 1 : EPL - 1] = fadd(acc[i + 1 < EPL ? i + 1 : EPL - 1], gi);
            else accR = fadd(accR, gi);
          } else {
            rem[i] = true;
          }
        }
        const float fromR = __shfl_down_sync(0xffffffffu, accL, 1);
        const float fromL = __shfl_up_sync(0xffffffffu, accR, 1);
        if (lane < 31) acc[EPL - 1] = fadd(acc[EPL - 1], fromR);
        if (lane > 0) acc[0] = fadd(acc[0], fromL);
        // remaining targets: one warp reduction per distinct target, ascending
        while (true) {
          uint32_t mk = 0xffffffffu;
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (rem[i]) mk = min(mk, uint32_t(pm[i]));
          const uint32_t key = __reduce_min_sync(0xffffffffu, mk);
          if (key == 0xffffffffu) break;
          float part = 0.0f;
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (rem[i] && uint32_t(pm[i]) == key) {
              part = fadd(part, row[i]);
              rem[i] = false;
            }
          const float tot = warp_sum_f(part);
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (int(key) == l0 + i) acc[i] = fadd(acc[i], tot);
        }
      }

      // ---- dw and dV contributions of this edge
      float wpart = 0.0f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const float gi = row[i];
        if (i >= nvalid || gi == 0.0f) continue;
        const int l = l0 + i, mu = pm[i];
        if (a.gw) {
          const float vv = __ldg(a.pot.V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l));
          wpart = fadd(wpart, fmul(gi, vv));
        }
        const float gwv = fmul(gi, w);
        const int d = mu - l;
        if (d == -1) vacc[i][0] = fadd(vacc[i][0], gwv);
        else if (d == 0) vacc[i][1] = fadd(vacc[i][1], gwv);
        else if (d == 1) vacc[i][2] = fadd(vacc[i][2], gwv);
        else atomicAdd(gvacc + size_t(mu) * L + l, gwv);
      }
      if (a.gw) {
        const float wsum = warp_sum_f(wpart);
        if (lane == 0) {
          float* t = a.gw + (size_t(b) * (R / 2) + fam) * N + ((r & 1) ? cur : prev);
          *t = fadd(*t, wsum);
        }
      }

      // ---- apply to the predecessor rows
      float outv[EPL];
      if (!TRWP) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) outv[i] = fadd(slot[LS + l0 + i], acc[i]);
        store_slice<EPL>(gub + size_t(prev) * L, l0, outv, nvalid, L);
        for (int rr = 0; rr < NP; ++rr) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) outv[i] = fadd(slot[(2 + rr) * LS + l0 + i], acc[i]);
          store_slice<EPL>(planes_base + (size_t(plane_of(rr)) * N + prev) * L, l0, outv, nvalid, L);
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) carry[i] = acc[i];
      } else {
        float ra[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          ra[i] = fmul(rho, acc[i]);
          outv[i] = fadd(slot[LS + l0 + i], ra[i]);
        }
        store_slice<EPL>(gub + size_t(prev) * L, l0, outv, nvalid, L);
        for (int rr = 0; rr < NP; ++rr) {
          const int d = plane_of(rr);
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            float v = fadd(slot[(2 + rr) * LS + l0 + i], ra[i]);
            if (d == opp) v = fsub(v, acc[i]);
            outv[i] = v;
          }
          store_slice<EPL>(planes_base + (size_t(d) * N + prev) * L, l0, outv, nvalid, L);
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) carry[i] = ra[i];
      }
      __syncwarp();
    }
    // head row of plane r: its incoming scatter (carry) is dropped and the row
    // cleared, like the reference's plane clear / buffer swap (:122-123, :190-193)
    {
      float z[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) z[i] = 0.0f;
      store_slice<EPL>(gmr + size_t(ld.first) * L, l0, z, nvalid, L);
    }
    cp_wait<0>();
    __syncwarp();
  }
  // flush near-diagonal dV partials
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const int l = l0 + i;
    if (i >= nvalid) continue;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int mu = l + t - 1;
      if (mu >= 0 && mu < L && vacc[i][t] != 0.0f) atomicAdd(gvacc + size_t(mu) * L + l, vacc[i][t]);
    }
  }
}

// dV[b][x][y] = sum_rep acc[b][rep][0][x][y] + acc[b][rep][1][y][x]
__global__ void reduce_gvacc_kernel(int B, int L, const float* __restrict__ acc, float* __restrict__ gv) {
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
