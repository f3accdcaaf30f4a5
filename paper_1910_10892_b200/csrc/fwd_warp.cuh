// Forward sweep, warp-per-scanline (sm_100a).
//
// One warp walks one scanline; lane a owns the EPL contiguous labels
// l = a*EPL + i (and the same mu range for the base assembly), so the carried
// message m^r_prev stays in registers and a node step needs no CTA barrier.
// The rows a step reads (theta and the other directions' messages at prev)
// do not depend on the chain; each lane streams its own slice of them
// kStages-1 steps ahead with cp.async into a per-warp shared-memory ring.
//
// Min-plus (isgmr.hpp:98-116 / trwp.hpp:100-118), exact strategies chosen on
// the device per call by analyze_pairwise_kernel:
//  * banded: V symmetric Toeplitz, V(a,b) = g(|a-b|), with a constant tail
//    g(d) = g(D) for d >= D (Potts, truncated linear / quadratic, P1P2 all
//    have one). Candidates with |l-mu| >= D all cost u(mu) = fl(base(mu) +
//    fl(w*g(D))); the first argmin of u over the left part [0, l-D] and the
//    right part [l+D, L) come from warp prefix / suffix (value, first index)
//    scans, the 2D-1 near candidates are evaluated explicitly, and the three
//    segment winners are combined in index order with strict '<'. That is the
//    reference's ascending strict-'<' scan restated over segments, so values
//    and indices are bit-identical (fl(x + c) is monotone in x, and no
//    candidate can be -0: see analyze_pairwise_kernel). D == 2 (truncated
//    linear with tau = 2, the stereo configs) exchanges its neighbours with
//    shuffles only; other D go through per-warp shared memory.
//  * dense: every (mu, l) candidate, ascending mu, strict '<'.
#pragma once

#include "common.cuh"

namespace mrf {

// Device-side description of V for one forward call.
struct PairDesc {
  int banded;   // 1: banded strategy valid and profitable
  int D;        // band half-width: g(d) == g(D) for all d >= D
  float g[256]; // g(d) = V(0, d)
};

// One block. Bit-level checks: symmetric Toeplitz, constant tail, and no -0
// in the constant weight (planes are checked by scan_neg_zero_kernel), so no
// candidate value can be -0, which makes the scanned minimum value equal to
// the first argmin's raw value. D = 1 + the last index d < L-1 whose g(d)
// differs from the tail g(L-1) (at least 1), found by a block max-reduction.
static __global__ void __launch_bounds__(1024) analyze_pairwise_kernel(const float* __restrict__ V, int L, float wconst,
                                                                       int has_wplanes, PairDesc* __restrict__ out) {
  int ok = 1;
  for (int i = threadIdx.x; i < L * L; i += blockDim.x) {
    const int a = i / L, b = i - a * L;
    const int d = a > b ? a - b : b - a;
    if (__float_as_uint(__ldg(V + i)) != __float_as_uint(__ldg(V + d))) ok = 0;
  }
  if (!has_wplanes && __float_as_uint(wconst) == 0x80000000u) ok = 0;
  ok = __syncthreads_and(ok);
  const uint32_t tail = __float_as_uint(V[L - 1]);
  int last = 0;  // 1 + the last d < L-1 with g(d) != g(L-1)
  for (int d = threadIdx.x; d < 256; d += blockDim.x) {
    const float gd = d < L ? V[d] : 0.0f;
    out->g[d] = gd;
    if (d < L - 1 && __float_as_uint(gd) != tail) last = d + 1;
  }
  __shared__ int s_last[32];
  for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  if ((threadIdx.x & 31) == 0) s_last[threadIdx.x >> 5] = last;
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) m = max(m, s_last[w]);
    const int D = L > 1 ? max(m, 1) : 1;
    out->D = D;
    out->banded = ok && (2 * D - 1) * 2 <= L;
  }
}

// Runs after analyze_pairwise_kernel: any -0 in the weight / rho planes
// disables the banded strategy (grid-wide scan; every writer writes 0).
static __global__ void scan_neg_zero_kernel(const uint32_t* __restrict__ x, int64_t n, PairDesc* __restrict__ out) {
  int found = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    found |= __ldg(x + i) == 0x80000000u;
  if (__syncthreads_or(found) && threadIdx.x == 0) out->banded = 0;
}

struct FwdArgs {
  Geometry g;
  Potentials pot;
  const LineDesc* lines;
  int nlines;
  const float* m_in;   // published messages (ISGMR) / in-place buffer (TRWP)
  float* m_out;        // swept buffer (ISGMR) / same as m_in (TRWP)
  uint8_t* p;
  uint8_t* q;
  int k;
  const PairDesc* desc;
  int band2_launched;  // fwd_band2_kernel covers banded D == 2 in this sweep
  int bandw_max;       // fwd_bandw_kernel covers banded 2 < D <= bandw_max (0: not launched)
  int dense_small;     // fwd_small_kernel covers dense V with L <= 32
  // TRWP, last sweep of the last iteration (4 directions): the banded D == 2
  // kernel also writes the aggregated cost / labels (else null)
  float* agg_cost;
  uint16_t* agg_labels;
  int dir;  // the one direction every line of the launch sweeps (TRWP), -1: mixed (ISGMR)
  // diagnostic mode (mrf_problem_f32::diag_gap): [B] floats min-accumulating
  // the (second best - best) argmin gaps; only fwd_warp_kernel is launched
  float* diag_gap;
};

__device__ __forceinline__ void cp_async_u32(uint32_t saddr, const void* gmem, int bytes) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  cp_async_u32(static_cast<uint32_t>(__cvta_generic_to_shared(smem)), gmem, bytes);
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int EPL>
struct Chunk {
  // bytes per cp.async for a lane's full EPL slice given L's alignment
  static __device__ __forceinline__ int bytes(int L) {
    if (EPL % 4 == 0 && (L & 3) == 0) return 16;
    if (EPL % 2 == 0 && (L & 1) == 0) return 8;
    return 4;
  }
};

// Copy a lane's slice (nvalid floats at src) to shared memory at saddr.
template <int EPL>
__device__ __forceinline__ void cp_slice(uint32_t saddr, const float* src, int nvalid, int chunk) {
  if (nvalid == EPL) {
    if (chunk == 16) {
#pragma unroll
      for (int c = 0; c < EPL / 4; ++c) cp_async_u32(saddr + 16 * c, src + 4 * c, 16);
    } else if (chunk == 8) {
#pragma unroll
      for (int c = 0; c < EPL / 2; ++c) cp_async_u32(saddr + 8 * c, src + 2 * c, 8);
    } else {
#pragma unroll
      for (int c = 0; c < EPL; ++c) cp_async_u32(saddr + 4 * c, src + c, 4);
    }
  } else {
    for (int c = 0; c < nvalid; ++c) cp_async_u32(saddr + 4 * c, src + c, 4);
  }
}

// Compile-time variant: FULL slices (L == 32*EPL, so rows are 16 B aligned)
// use the widest chunk the slice allows; otherwise 4 B copies of the valid
// elements. No runtime chunk selection (which would be predicated into both
// instruction sequences).
template <int EPL, bool FULL>
__device__ __forceinline__ void cp_slice_t(uint32_t saddr, const float* src, int nvalid) {
  if (FULL) {
    constexpr int CH = EPL % 4 == 0 ? 16 : (EPL % 2 == 0 ? 8 : 4);
#pragma unroll
    for (int c = 0; c < EPL * 4 / CH; ++c) cp_async_u32(saddr + CH * c, src + (CH / 4) * c, CH);
  } else {
#pragma unroll
    for (int c = 0; c < EPL; ++c)
      if (c < nvalid) cp_async_u32(saddr + 4 * c, src + c, 4);
  }
}

// Read a lane's EPL floats from shared memory (vectorised when aligned).
template <int EPL>
__device__ __forceinline__ void lds_slice(float (&v)[EPL], const float* s) {
  if (EPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(s + i);
      v[i] = t.x, v[i + 1] = t.y, v[i + 2] = t.z, v[i + 3] = t.w;
    }
  } else if (EPL % 2 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2) {
      const float2 t = *reinterpret_cast<const float2*>(s + i);
      v[i] = t.x, v[i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) v[i] = s[i];
  }
}

template <int EPL>
__device__ __forceinline__ void stg_slice(float* row, int l0, const float (&v)[EPL], int nvalid, int L) {
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

#ifndef MRF_FWD_STAGES
#define MRF_FWD_STAGES 4
#endif
constexpr int kStages = MRF_FWD_STAGES;  // cp.async ring depth (steps in flight + 1)
constexpr float kInf = __builtin_huge_valf();

// Per-warp shared memory (floats): ring [kStages][rows][32*EPL], per-lane
// edge scalars [kStages][2][32], base / scan values [3][32*EPL], scan index
// bytes [2][32*EPL], scaled band [256].
__host__ __device__ constexpr int fwd_warp_smem_floats(int EPL, int rows) {
  return ((kStages * rows + 3) * 32 * EPL + kStages * 64 + (2 * 32 * EPL + 3) / 4 + 256 + 31) / 32 * 32;
}

// min over gaps with the reference's `if (g < gap) gap = g` (NaN never wins)
__device__ __forceinline__ void gap_min(float& gap, float g) {
  if (g < gap) gap = g;
}

// MODE 0 dense, 1 banded (shared memory), 2 banded D == 2 (shuffles). GAP
// (MODE 0 only): also track min_argmin_gap the way the reference's sweep
// does (isgmr.hpp:100-116,119-129: second best per label and for the
// reparametrisation argmin) and atomically min it into a.diag_gap[b].
template <int EPL, bool TRWP, int MODE, bool GAP = false>
__device__ __forceinline__ void fwd_sweep_lines(const FwdArgs& a, float* ws) {
  const Geometry& g = a.g;
  const int L = g.L, N = g.N, R = g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int NP = TRWP ? R - 1 : R - 2;  // message planes read per step
  const int rows = 1 + NP;
  constexpr int LS = 32 * EPL;
  float* ring = ws;
  float* s_x = ring + kStages * rows * LS;  // [kStages][2][32]: w, rho per lane
  float* s_base = s_x + kStages * 64;
  float* s_pv = s_base + LS;
  float* s_sv = s_pv + LS;
  uint8_t* s_pi = reinterpret_cast<uint8_t*>(s_sv + LS);
  uint8_t* s_si = s_pi + LS;
  float* s_wg = s_sv + LS + (2 * LS + 3) / 4;
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  const uint32_t x_s = static_cast<uint32_t>(__cvta_generic_to_shared(s_x));

  const int b = blockIdx.y;
  const float* un = a.pot.unary + size_t(b) * N * L;
  const size_t img = size_t(b) * R * N * L;
  const int l0 = lane * EPL;
  const int nvalid = min(EPL, max(0, L - l0));
  const int chunk = nvalid == EPL ? Chunk<EPL>::bytes(L) : 4;
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const int D = a.desc->D;
  const float* gt = a.desc->g;
  // constant-w band scaled once; per-edge weights rescale per step
  float g0 = 0.f, g1 = 0.f, g2 = 0.f, wg0 = 0.f, wg1 = 0.f, wgD = 0.f;
  if (MODE == 2) {
    g0 = gt[0], g1 = gt[1], g2 = gt[2];
    wg0 = fmul(a.pot.w, g0), wg1 = fmul(a.pot.w, g1), wgD = fmul(a.pot.w, g2);
  }
  if (MODE == 1) {
    for (int d = lane; d <= D && d < 256; d += 32) s_wg[d] = fmul(a.pot.w, gt[d]);
    __syncwarp();
  }
  float gap = kInf;  // GAP: this lane's running minimum

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    // idx-th plane read per step, ascending d (base order, isgmr.hpp:84-88 /
    // trwp.hpp:85-88): TRWP skips r, ISGMR skips the pair {r, r^1}.
    auto plane_of = [&](int idx) { return TRWP ? (idx < r ? idx : idx + 1) : (idx < (r & ~1) ? idx : idx + 2); };
    const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
    auto issue = [&](int j) {  // rows of step j (prev = node j-1) into slot (j-1) % kStages
      const int slot = (j - 1) % kStages;
      const int prev = ld.first + (j - 1) * st;
      if (nvalid > 0) {
        cp_slice<EPL>(ring_s + 4u * uint32_t((slot * rows) * LS + l0), un + size_t(prev) * L + l0, nvalid, chunk);
        for (int rr = 1; rr < rows; ++rr)
          cp_slice<EPL>(ring_s + 4u * uint32_t((slot * rows + rr) * LS + l0),
                        a.m_in + img + (size_t(plane_of(rr - 1)) * N + prev) * L + l0, nvalid, chunk);
      }
      const int wnode = (r & 1) ? prev + st : prev;
      if (wpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + lane), wrow + wnode, 4);
      if (rpl) cp_async_u32(x_s + 4u * uint32_t(slot * 64 + 32 + lane), rrow + wnode, 4);
    };
    for (int s = 0; s < kStages - 1; ++s) {
      if (1 + s <= nsteps) issue(1 + s);
      cp_commit();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;
    // dense small-L: this lane's column of V' (orientation fixed per line)
    float vcol[EPL == 1 ? 32 : 1];
    if (MODE == 0 && EPL == 1) {
      const int l = l0 < L ? l0 : 0;
#pragma unroll
      for (int mu = 0; mu < 32; ++mu)
        vcol[mu] = mu < L ? __ldg(a.pot.V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l)) : 0.0f;
    }

    for (int j = 1; j <= nsteps; ++j) {
      if (j + kStages - 1 <= nsteps) issue(j + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      const int slot = (j - 1) % kStages;
      const float* srow = ring + slot * rows * LS + l0;
      const float w = wpl ? s_x[slot * 64 + lane] : a.pot.w;

      // ---- base assembly (registers; own mu slice)
      float base[EPL];
      {
        float t[EPL];
        lds_slice<EPL>(t, srow);
        if (!TRWP) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) base[i] = fadd(t[i], carry[i]);
          for (int rr = 1; rr < rows; ++rr) {
            lds_slice<EPL>(t, srow + rr * LS);
#pragma unroll
            for (int i = 0; i < EPL; ++i) base[i] = fadd(base[i], t[i]);
          }
        } else {
          const float rho = rpl ? s_x[slot * 64 + 32 + lane] : a.pot.rho;
          float s[EPL], mo[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) s[i] = t[i], mo[i] = 0.0f;
          int rr = 1;
          for (int d = 0; d < R; ++d) {
            if (d == r) {
#pragma unroll
              for (int i = 0; i < EPL; ++i) s[i] = fadd(s[i], carry[i]);
            } else {
              lds_slice<EPL>(t, srow + rr * LS);
              ++rr;
              if (d == opp) {
#pragma unroll
                for (int i = 0; i < EPL; ++i) mo[i] = t[i];
              }
#pragma unroll
              for (int i = 0; i < EPL; ++i) s[i] = fadd(s[i], t[i]);
            }
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) base[i] = fsub(fmul(rho, s[i]), mo[i]);
        }
      }

      float out[EPL];
      int arg[EPL];
      float sec[EPL];  // GAP: second best candidate per label
#pragma unroll
      for (int i = 0; i < EPL; ++i) sec[i] = kInf;
      if (MODE != 0) {
        float c;
        if (MODE == 2) {
          if (wpl) wg0 = fmul(w, g0), wg1 = fmul(w, g1), wgD = fmul(w, g2);
          c = wgD;
        } else {
          if (wpl) {
            for (int d = lane; d <= D && d < 256; d += 32) s_wg[d] = fmul(w, gt[d]);
          }
          c = wpl ? fmul(w, gt[D]) : s_wg[D];
        }
        // u(mu) = fl(base(mu) + fl(w*g(D))): every far candidate's cost
        float u[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) u[i] = i < nvalid ? fadd(base[i], c) : kInf;
        // prefix (value, first index) with op(earlier e, later x) = x.v < e.v ? x : e
        float pv[EPL];
        int pi[EPL];
        pv[0] = u[0];
        pi[0] = l0;
#pragma unroll
        for (int i = 1; i < EPL; ++i) {
          const bool t = u[i] < pv[i - 1];
          pv[i] = t ? u[i] : pv[i - 1];
          pi[i] = t ? l0 + i : pi[i - 1];
        }
        // suffix (value, first index): S(s) = op(u(s), S(s+1))
        float sv[EPL];
        int si[EPL];
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
          if (lane >= off && !(tpv < opv)) tpv = opv, tpi = opi;
          if (lane + off < 32 && osv < tsv) tsv = osv, tsi = osi;
        }
        {
          const float epv = __shfl_up_sync(0xffffffffu, tpv, 1);
          const int epi = __shfl_up_sync(0xffffffffu, tpi, 1);
          const float esv = __shfl_down_sync(0xffffffffu, tsv, 1);
          const int esi = __shfl_down_sync(0xffffffffu, tsi, 1);
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            if (lane > 0 && !(pv[i] < epv)) pv[i] = epv, pi[i] = epi;
            if (lane < 31 && esv < sv[i]) sv[i] = esv, si[i] = esi;
          }
        }
        if (MODE == 2) {
          // D == 2: near band {l-1, l, l+1}; far segments end/start at l-2 / l+2
          const float bl = __shfl_up_sync(0xffffffffu, base[EPL - 1], 1);   // base(l0 - 1)
          const float br = __shfl_down_sync(0xffffffffu, base[0], 1);       // base(l0 + EPL)
          float pvm[2], svp[2];
          int pim[2], sip[2];
          if (EPL >= 2) {
            pvm[0] = __shfl_up_sync(0xffffffffu, pv[EPL - 2 >= 0 ? EPL - 2 : 0], 1);
            pvm[1] = __shfl_up_sync(0xffffffffu, pv[EPL - 1], 1);
            pim[0] = __shfl_up_sync(0xffffffffu, pi[EPL - 2 >= 0 ? EPL - 2 : 0], 1);
            pim[1] = __shfl_up_sync(0xffffffffu, pi[EPL - 1], 1);
            svp[0] = __shfl_down_sync(0xffffffffu, sv[0], 1);
            svp[1] = __shfl_down_sync(0xffffffffu, sv[EPL >= 2 ? 1 : 0], 1);
            sip[0] = __shfl_down_sync(0xffffffffu, si[0], 1);
            sip[1] = __shfl_down_sync(0xffffffffu, si[EPL >= 2 ? 1 : 0], 1);
          } else {
            pvm[0] = __shfl_up_sync(0xffffffffu, pv[0], 2);
            pim[0] = __shfl_up_sync(0xffffffffu, pi[0], 2);
            svp[1] = __shfl_down_sync(0xffffffffu, sv[0], 2);
            sip[1] = __shfl_down_sync(0xffffffffu, si[0], 2);
            pvm[1] = 0.f, pim[1] = 0, svp[0] = 0.f, sip[0] = 0;
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const int l = l0 + i;
            float best = kInf;
            int am = 0;
            // left far: first argmin of u over [0, l-2]
            const float lv = i >= 2 ? pv[i >= 2 ? i - 2 : 0] : (EPL >= 2 ? pvm[i] : pvm[0]);
            const int lix = i >= 2 ? pi[i >= 2 ? i - 2 : 0] : (EPL >= 2 ? pim[i] : pim[0]);
            if (l >= 2 && lv < best) best = lv, am = lix;
            // near band, ascending mu
            const float bm1 = i >= 1 ? base[i >= 1 ? i - 1 : 0] : bl;
            const float bp1 = i + 1 < EPL ? base[i + 1 < EPL ? i + 1 : 0] : br;
            if (l >= 1) {
              const float v = fadd(bm1, wg1);
              if (v < best) best = v, am = l - 1;
            }
            {
              const float v = fadd(base[i], wg0);
              if (v < best) best = v, am = l;
            }
            if (l + 1 < L) {
              const float v = fadd(bp1, wg1);
              if (v < best) best = v, am = l + 1;
            }
            // right far: first argmin of u over [l+2, L)
            const float rv = i + 2 < EPL ? sv[i + 2 < EPL ? i + 2 : 0] : (EPL >= 2 ? svp[i + 2 - EPL >= 0 ? i + 2 - EPL : 0] : svp[1]);
            const int rix = i + 2 < EPL ? si[i + 2 < EPL ? i + 2 : 0] : (EPL >= 2 ? sip[i + 2 - EPL >= 0 ? i + 2 - EPL : 0] : sip[1]);
            if (l + 2 < L && rv < best) best = rv, am = rix;
            out[i] = best;
            arg[i] = am;
          }
        } else {
          // generic D: neighbours through per-warp shared memory
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            s_base[l0 + i] = base[i];
            s_pv[l0 + i] = pv[i];
            s_sv[l0 + i] = sv[i];
            s_pi[l0 + i] = uint8_t(pi[i]);
            s_si[l0 + i] = uint8_t(si[i]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const int l = l0 + i;
            float best = kInf;
            int am = 0;
            if (l - D >= 0 && l < L) {
              const float v = s_pv[l - D];
              if (v < best) best = v, am = s_pi[l - D];
            }
            for (int t = 0; t < 2 * D - 1; ++t) {
              const int mu = l - D + 1 + t;
              const bool ok = mu >= 0 && mu < L && l < L;
              const float v = fadd(s_base[ok ? mu : 0], s_wg[t < D ? D - 1 - t : t - D + 1]);
              if (ok && v < best) best = v, am = mu;
            }
            if (l + D <= L - 1) {
              const float v = s_sv[l + D];
              if (v < best) best = v, am = s_si[l + D];
            }
            out[i] = best;
            arg[i] = am;
          }
        }
      } else {
        // dense: every mu ascending, strict '<' (isgmr.hpp:103-112)
#pragma unroll
        for (int i = 0; i < EPL; ++i) s_base[l0 + i] = base[i], out[i] = kInf, arg[i] = 0;
        __syncwarp();
        if (EPL == 1) {
#pragma unroll
          for (int mu = 0; mu < 32; ++mu) {
            if (mu < L) {
              const float v = fadd(s_base[mu], fmul(w, vcol[mu < 32 ? mu : 0]));
              if (GAP) {
                if (v < out[0]) sec[0] = out[0], out[0] = v, arg[0] = mu;
                else if (v < sec[0]) sec[0] = v;
              } else if (v < out[0]) {
                out[0] = v, arg[0] = mu;
              }
            }
          }
        } else {
          for (int mu = 0; mu < L; ++mu) {
            const float bm = s_base[mu];
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const int l = l0 + i < L ? l0 + i : 0;
              const float vv = __ldg(a.pot.V + ((r & 1) ? size_t(l) * L + mu : size_t(mu) * L + l));
              const float v = fadd(bm, fmul(w, vv));
              if (GAP) {
                if (v < out[i]) sec[i] = out[i], out[i] = v, arg[i] = mu;
                else if (v < sec[i]) sec[i] = v;
              } else if (v < out[i]) {
                out[i] = v, arg[i] = mu;
              }
            }
          }
        }
      }

      // ---- p row and the reparametrisation argmin (lowest label on ties)
      const int cur = ld.first + j * st;
      uint8_t* prow = a.p + (pq_base + j - 1) * L;
      uint32_t lk = 0xffffffffu, lt = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (i < nvalid) {
          prow[l0 + i] = uint8_t(arg[i]);
          const uint32_t kk = order_key(fadd(out[i], 0.0f));
          if (kk < lk) lk = kk, lt = (uint32_t(l0 + i) << 1) | (__float_as_uint(out[i]) == 0x80000000u ? 1u : 0u);
        }
      }
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, lk);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, lk == kmin ? lt : 0xffffffffu);
      float lo = key_value(kmin);
      if (tmin & 1u) lo = -0.0f;
      if (GAP) {
        // second smallest message entry = min over l != lstar (ties included)
        const int lstar = int(tmin >> 1);
        uint32_t sk = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          if (i < nvalid) {
            gap_min(gap, fsub(sec[i], out[i]));
            if (l0 + i != lstar) sk = min(sk, order_key(fadd(out[i], 0.0f)));
          }
        }
        const uint32_t skm = __reduce_min_sync(0xffffffffu, sk);
        const float second = skm == 0xffffffffu ? kInf : key_value(skm);
        gap_min(gap, fsub(second, lo));
      }
#pragma unroll
      for (int i = 0; i < EPL; ++i) carry[i] = fsub(out[i], lo);
      stg_slice<EPL>(a.m_out + img + (size_t(r) * N + cur) * L, l0, carry, nvalid, L);
      if (lane == 0) a.q[pq_base + j - 1] = uint8_t(tmin >> 1);
      if (MODE != 2 || wpl) __syncwarp();
    }
    cp_wait<0>();
    __syncwarp();
  }
  if (GAP) {
    // gaps are >= 0 (or -0, or +inf): their int bits order like the values
    int gi = __float_as_int(gap);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) gi = min(gi, __shfl_xor_sync(0xffffffffu, gi, off));
    if (lane == 0 && gi != __float_as_int(kInf)) atomicMin(reinterpret_cast<int*>(a.diag_gap) + b, gi);
  }
}

template <int EPL, bool TRWP>
__global__ void __launch_bounds__(128) fwd_warp_kernel(FwdArgs a) {
  extern __shared__ float smem[];
  const int R = a.g.R;
  const int rows = 1 + (TRWP ? R - 1 : R - 2);
  float* ws = smem + size_t(threadIdx.x >> 5) * fwd_warp_smem_floats(EPL, rows);
  if (a.diag_gap) {  // diagnostic mode: the only kernel launched for the sweep
    fwd_sweep_lines<EPL, TRWP, 0, true>(a, ws);
    return;
  }
  if (a.desc->banded) {
    if (a.desc->D == 2) {
      if (!a.band2_launched) fwd_sweep_lines<EPL, TRWP, 2>(a, ws);
    } else if (!(a.desc->D > 2 && a.desc->D <= a.bandw_max)) {
      fwd_sweep_lines<EPL, TRWP, 1>(a, ws);
    }
  } else if (!a.dense_small) {
    fwd_sweep_lines<EPL, TRWP, 0>(a, ws);
  }
}

}  // namespace mrf
