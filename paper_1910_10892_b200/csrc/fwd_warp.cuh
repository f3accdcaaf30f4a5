// Forward sweep, warp-per-scanline (sm_100a).
//
// One warp walks one scanline; lane a owns the EPL contiguous labels
// l = a*EPL + i (and the same mu range for the base assembly), so the carried
// message m^r_prev stays in registers and a node step needs no CTA barrier.
// The rows a step reads (theta and the other directions' messages at prev)
// do not depend on the chain; each lane streams its own slice of them S-1
// steps ahead with cp.async into a per-warp shared-memory ring.
//
// Min-plus (isgmr.hpp:98-116 / trwp.hpp:100-118), two exact strategies chosen
// on the device per call by analyze_pairwise_kernel:
//  * banded: V symmetric Toeplitz, V(a,b) = g(|a-b|), with a constant tail
//    g(d) = g(D) for d >= D (Potts, truncated linear / quadratic, P1P2 all
//    have one). Candidates with |l-mu| >= D all cost u(mu) = fl(base(mu) +
//    fl(w*g(D))); the first argmin of u over the left part [0, l-D] and the
//    right part [l+D, L) come from warp prefix / suffix (value, first index)
//    scans, the 2D-1 near candidates are evaluated explicitly, and the three
//    segment winners are combined in index order with strict '<'. That is the
//    reference's ascending strict-'<' scan restated over segments, so values
//    and indices are bit-identical (fl(x + c) is monotone in x, and no
//    candidate can be -0: see analyze_pairwise_kernel).
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
// in the weight / rho planes (so no candidate value can be -0, which makes the
// scanned minimum value equal to the first argmin's raw value).
__global__ void analyze_pairwise_kernel(const float* __restrict__ V, int L, const float* __restrict__ wplanes,
                                        int64_t nw, float wconst, const float* __restrict__ rplanes, int64_t nr,
                                        PairDesc* __restrict__ out) {
  int ok = 1;
  for (int i = threadIdx.x; i < L * L; i += blockDim.x) {
    const int a = i / L, b = i - a * L;
    const int d = a > b ? a - b : b - a;
    if (__float_as_uint(V[i]) != __float_as_uint(V[d])) ok = 0;
  }
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x)
    if (__float_as_uint(wplanes[i]) == 0x80000000u) ok = 0;
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x)
    if (__float_as_uint(rplanes[i]) == 0x80000000u) ok = 0;
  if (wplanes == nullptr && __float_as_uint(wconst) == 0x80000000u) ok = 0;
  ok = __syncthreads_and(ok);
  for (int d = threadIdx.x; d < L; d += blockDim.x) out->g[d] = V[d];
  if (threadIdx.x == 0) {
    int D = L > 1 ? L - 1 : 1;
    const uint32_t tail = __float_as_uint(V[L - 1]);
    while (D > 1 && __float_as_uint(V[D - 1]) == tail) --D;
    out->D = D;
    out->banded = ok && (2 * D - 1) * 2 <= L;
  }
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
};

template <int EPL>
struct Chunk {
  // bytes per cp.async for a lane's full EPL slice given L's alignment
  static __device__ __forceinline__ int bytes(int L) {
    if (EPL % 4 == 0 && (L & 3) == 0) return 16;
    if (EPL % 2 == 0 && (L & 1) == 0) return 8;
    return 4;
  }
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
  else if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kStages = 4;

// Shared memory per warp (floats): ring [kStages][rows][32*EPL] + base, scan
// values and the index bytes of the two scans.
__host__ __device__ constexpr int fwd_warp_smem_floats(int EPL, int rows) {
  return ((kStages * rows + 3) * 32 * EPL + (2 * 32 * EPL + 3) / 4 + 31) / 32 * 32;
}

template <int EPL, bool TRWP>
__global__ void __launch_bounds__(128) fwd_warp_kernel(FwdArgs a) {
  extern __shared__ float smem[];
  const Geometry& g = a.g;
  const int L = g.L, N = g.N, R = g.R;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int NP = TRWP ? R - 1 : R - 2;  // message planes read per step
  const int rows = 1 + NP;
  const int LS = 32 * EPL;
  float* ws = smem + size_t(wid) * fwd_warp_smem_floats(EPL, rows);
  float* ring = ws;
  float* s_base = ring + kStages * rows * LS;
  float* s_pv = s_base + LS;
  float* s_sv = s_pv + LS;
  uint8_t* s_pi = reinterpret_cast<uint8_t*>(s_sv + LS);
  uint8_t* s_si = s_pi + LS;

  const int b = blockIdx.y;
  const float* un = a.pot.unary + size_t(b) * N * L;
  const size_t img = size_t(b) * R * N * L;
  const int l0 = lane * EPL;
  const int nvalid = min(EPL, max(0, L - l0));
  const int chunk = nvalid == EPL ? Chunk<EPL>::bytes(L) : 4;
  const bool banded = a.desc->banded != 0;
  const int D = a.desc->D;
  const float* gtab = a.desc->g;

  for (int li = blockIdx.x * wpc + wid; li < a.nlines; li += gridDim.x * wpc) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r];
    const int nsteps = ld.length - 1;
    // idx-th plane read per step, ascending d (base order, isgmr.hpp:84-88 /
    // trwp.hpp:85-88): TRWP skips r, ISGMR skips the pair {r, r^1}.
    auto plane_of = [&](int idx) { return TRWP ? (idx < r ? idx : idx + 1) : (idx < (r & ~1) ? idx : idx + 2); };
    auto issue = [&](int j) {  // rows of step j (prev = node j-1) into slot (j-1) % kStages
      float* slot = ring + ((j - 1) % kStages) * rows * LS;
      const int prev = ld.first + (j - 1) * st;
      if (nvalid > 0) {
        for (int rr = 0; rr < rows; ++rr) {
          const float* src = rr == 0 ? un + size_t(prev) * L
                                     : a.m_in + img + (size_t(plane_of(rr - 1)) * N + prev) * L;
          float* dst = slot + rr * LS;
          for (int off = 0; off < nvalid * 4; off += chunk)
            cp_async(reinterpret_cast<char*>(dst + l0) + off, reinterpret_cast<const char*>(src + l0) + off, chunk);
        }
      }
    };
    for (int s = 0; s < kStages - 1; ++s) {
      if (1 + s <= nsteps) issue(1 + s);
      cp_commit();
    }
    const size_t pq_base = (size_t(b) * g.K_cap + a.k) * g.E + g.dir_offset[r] + ld.edge_base;
    float carry[EPL];
#pragma unroll
    for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;

    for (int j = 1; j <= nsteps; ++j) {
      if (j + kStages - 1 <= nsteps) issue(j + kStages - 1);
      cp_commit();
      cp_wait<kStages - 1>();
      const float* slot = ring + ((j - 1) % kStages) * rows * LS;
      const int prev = ld.first + (j - 1) * st, cur = prev + st;

      // ---- base assembly (registers; own mu slice)
      float base[EPL];
      if (!TRWP) {
#pragma unroll
        for (int i = 0; i < EPL; ++i) base[i] = fadd(slot[l0 + i], carry[i]);
        for (int rr = 1; rr < rows; ++rr) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) base[i] = fadd(base[i], slot[rr * LS + l0 + i]);
        }
      } else {
        const float rho = plane_value(a.pot.rho_planes, a.pot.rho, N, R, b, r, prev, cur);
        float s[EPL], mo[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) s[i] = slot[l0 + i];
        int rr = 1;
        for (int d = 0; d < R; ++d) {
          if (d == r) {
#pragma unroll
            for (int i = 0; i < EPL; ++i) s[i] = fadd(s[i], carry[i]);
          } else {
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const float md = slot[rr * LS + l0 + i];
              if (d == opp) mo[i] = md;
              s[i] = fadd(s[i], md);
            }
            ++rr;
          }
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) base[i] = fsub(fmul(rho, s[i]), mo[i]);
      }
      const float w = plane_value(a.pot.w_planes, a.pot.w, N, R, b, r, prev, cur);

      float out[EPL];
      int arg[EPL];
      if (banded) {
        // u(mu) = fl(base(mu) + fl(w*g(D))): the far-candidate cost
        const float c = fmul(w, gtab[D]);
        float u[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          u[i] = i < nvalid ? fadd(base[i], c) : __int_as_float(0x7f800000);
          s_base[l0 + i] = base[i];
        }
        // prefix (value, first index): op(earlier e, later x) = x.v < e.v ? x : e
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
        float tv = pv[EPL - 1];
        int ti = pi[EPL - 1];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float ov = __shfl_up_sync(0xffffffffu, tv, off);
          const int oi = __shfl_up_sync(0xffffffffu, ti, off);
          if (lane >= off && !(tv < ov)) {
            tv = ov;
            ti = oi;
          }
        }
        {
          const float ev = __shfl_up_sync(0xffffffffu, tv, 1);
          const int ei = __shfl_up_sync(0xffffffffu, ti, 1);
          if (lane > 0) {
#pragma unroll
            for (int i = 0; i < EPL; ++i)
              if (!(pv[i] < ev)) {
                pv[i] = ev;
                pi[i] = ei;
              }
          }
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
        tv = sv[0];
        ti = si[0];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float ov = __shfl_down_sync(0xffffffffu, tv, off);
          const int oi = __shfl_down_sync(0xffffffffu, ti, off);
          if (lane + off < 32 && ov < tv) {
            tv = ov;
            ti = oi;
          }
        }
        {
          const float ev = __shfl_down_sync(0xffffffffu, tv, 1);
          const int ei = __shfl_down_sync(0xffffffffu, ti, 1);
          if (lane < 31) {
#pragma unroll
            for (int i = 0; i < EPL; ++i)
              if (ev < sv[i]) {
                sv[i] = ev;
                si[i] = ei;
              }
          }
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          s_pv[l0 + i] = pv[i];
          s_sv[l0 + i] = sv[i];
          s_pi[l0 + i] = uint8_t(pi[i]);
          s_si[l0 + i] = uint8_t(si[i]);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int l = l0 + i;
          float best = __int_as_float(0x7f800000);
          int am = 0;
          if (l < L) {
            if (l - D >= 0) {  // left far segment [0, l-D]
              const float v = s_pv[l - D];
              if (v < best) {
                best = v;
                am = s_pi[l - D];
              }
            }
            const int lo_mu = max(0, l - D + 1), hi_mu = min(L - 1, l + D - 1);
            for (int mu = lo_mu; mu <= hi_mu; ++mu) {  // near band, ascending
              const int d = mu > l ? mu - l : l - mu;
              const float v = fadd(s_base[mu], fmul(w, gtab[d]));
              if (v < best) {
                best = v;
                am = mu;
              }
            }
            if (l + D <= L - 1) {  // right far segment [l+D, L)
              const float v = s_sv[l + D];
              if (v < best) {
                best = v;
                am = s_si[l + D];
              }
            }
          }
          out[i] = best;
          arg[i] = am;
        }
      } else {
        // dense: every mu ascending, strict '<' (isgmr.hpp:103-112)
#pragma unroll
        for (int i = 0; i < EPL; ++i) s_base[l0 + i] = base[i];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          out[i] = __int_as_float(0x7f800000);
          arg[i] = 0;
        }
        if (nvalid > 0) {
          for (int mu = 0; mu < L; ++mu) {
            const float bm = s_base[mu];
#pragma unroll
            for (int i = 0; i < EPL; ++i) {
              const int l = l0 + i;
              const float vv = __ldg(a.pot.V + ((r & 1) ? size_t(l < L ? l : 0) * L + mu : size_t(mu) * L + (l < L ? l : 0)));
              const float v = fadd(bm, fmul(w, vv));
              if (v < out[i]) {
                out[i] = v;
                arg[i] = mu;
              }
            }
          }
        }
      }

      // ---- p row and the reparametrisation argmin (lowest label on ties)
      uint8_t* prow = a.p + (pq_base + j - 1) * L;
      uint32_t lk = 0xffffffffu, lt = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        if (i < nvalid) {
          prow[l0 + i] = uint8_t(arg[i]);
          const uint32_t kk = order_key(fadd(out[i], 0.0f));
          if (kk < lk) {
            lk = kk;
            lt = (uint32_t(l0 + i) << 1) | (__float_as_uint(out[i]) == 0x80000000u ? 1u : 0u);
          }
        }
      }
      const uint32_t kmin = __reduce_min_sync(0xffffffffu, lk);
      const uint32_t tmin = __reduce_min_sync(0xffffffffu, lk == kmin ? lt : 0xffffffffu);
      float lo = key_value(kmin);
      if (tmin & 1u) lo = -0.0f;
      float* mrow = a.m_out + img + (size_t(r) * N + cur) * L;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        carry[i] = fsub(out[i], lo);
        if (i < nvalid) mrow[l0 + i] = carry[i];
      }
      if (lane == 0) a.q[pq_base + j - 1] = uint8_t(tmin >> 1);
      __syncwarp();
    }
    cp_wait<0>();
    __syncwarp();
  }
}

}  // namespace mrf
