// Backward sweep, one CTA per scanline with warp-specialised roles (sm_100a):
// isgmr_backward / trwp_backward (autodiff.hpp:63-126, :133-197) over the
// per-direction scatter planes A of bwd_common.cuh (same algebra, restated here
// so that the sequential part of a node step is a handful of instructions).
//
// Per node step (edge prev -> cur, walked tail to head) the reference does
//   row  = gm^r(cur) + carry           (carry: the sweep's own scatter into cur)
//   g    = row - S e_q, S = sum(row)   (reparametrisation backward, :48-53)
//   acc[mu] = sum_{l : p_l = mu} g_l   (index-driven scatter into prev)
//   carry' = rho acc (TRWP) / acc (ISGMR)
// Everything is linear in row, and with x = gm^r(cur) without the carry:
//   acc = [scatter(x) - S_x e_{p_q}] + scatter(carry)
// because sum(carry) = rho * sum(acc_prev) = rho * sum(g_prev) = 0 (the
// reparametrised row sums to zero), i.e. S = S_x up to rounding of the same
// order as the reference's own summation. So only scatter(carry) is
// sequential. Roles (warps of the CTA):
//   PRE  (NPRE warps, node-parallel): stream the rows of node cur with
//        cp.async, assemble x (bwd_common.cuh rules), S_x, decode p into a
//        per-lane mask word (near targets l-1 / l / l+1 and the "main" far
//        target) plus a list of any other far (label, target) pairs, and
//        B = scatter(x) - S_x e_{p_q};
//   CHAIN (1 warp): acc = B + scatter(carry): near targets through registers
//        and one shuffle each way, the main far group by one shared-memory
//        warp reduction, other pairs one shuffle each; carry' = rho acc;
//   POST (1 warp, node-parallel): store A[r](prev) = acc, rebuild the
//        reparametrised row g = x + carry - S_x e_q and accumulate dw (per
//        edge, parked and reduced 32 edges at a time) and dV (near-diagonal
//        and main-far partials in registers, other pairs with RED into a few
//        replicas).
// The roles hand nodes over through a ring of kSplitSlots shared-memory slots
// guarded by mbarriers (PRE -> full, CHAIN -> done, POST -> empty).
//
// BAND (banded V with D <= 2, decided on the device by analyze_pairwise):
// every candidate at distance >= 2 costs g(D), so a node's far labels all
// pick the unique first argmin of u in practice; the PRE fast path checks
// that (one min / max reduction) and POST folds dw into three masked sums
// (V' = g(0), g(1), g(D)). Anything else takes the general path.
#pragma once

#include <cstdio>

#include "bwd_common.cuh"
#include "common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

#ifndef MRF_SPLIT_SLOTS
#define MRF_SPLIT_SLOTS 4
#endif
#ifndef MRF_PRE_STAGES
#define MRF_PRE_STAGES 3
#endif
constexpr int kSplitSlots = MRF_SPLIT_SLOTS;  // node slots between the roles (A/B: -DMRF_SPLIT_SLOTS=n)
constexpr int kPreStages = MRF_PRE_STAGES;    // cp.async stages per PRE warp (A/B: -DMRF_PRE_STAGES=n)
#ifndef MRF_SPLIT_PRE
#define MRF_SPLIT_PRE 3
#endif
constexpr int kSplitPre = MRF_SPLIT_PRE;  // PRE warps per CTA (A/B: -DMRF_SPLIT_PRE=n)

// ---- mbarrier helpers (CTA scope; arrive = release, try_wait = acquire)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// shared-window addresses of the barriers, computed once per kernel
__device__ __forceinline__ void mbar_arrive(uint32_t bar_s) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_s) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar_s, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar_s),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Slot layout (floats), LS = 32*EPL:
//   X[LS] B[LS] ACC[LS] CIN[LS] P[8*EPL words] MASK[32] OTH[16*EPL words] WM[LS words] DT[LS] SC[8]
// DT (fused dtheta sweep): dtheta(cur) + sum_d rho_d A[d](cur), the carry is added by POST.
// WM (window mode): per target label mu, bit s + kWin set when source
// mu + s (|s| <= kWin) has p == mu.
template <int EPL>
struct SlotLayout {
  static constexpr int LS = 32 * EPL;
  static constexpr int X = 0, B = LS, ACC = 2 * LS, CIN = 3 * LS, P = 4 * LS, MASK = P + 8 * EPL,
                       OTH = MASK + 32, WM = OTH + 16 * EPL, DT = WM + LS, SC = DT + LS, SIZE = (SC + 8 + 3) / 4 * 4;
};
constexpr int kWin = 15;  // window mode: targets within +-kWin labels of the source are gathered
// scalar words of a slot
enum { SC_Q = 0, SC_S = 1, SC_MAIN = 2, SC_NOTH = 3, SC_W = 4, SC_RHO = 5 };

__host__ __device__ constexpr int split_slot_floats(int EPL) { return (216 * EPL + 40 + 3) / 4 * 4; }
// PRE ring stage: NR rows + p bytes (8*EPL words) + scalars {q word, w, rho, pad} + rho_d[NR] per lane
__host__ __device__ constexpr int split_stage_floats(int EPL, int NR) { return NR * 32 * EPL + 8 * EPL + 4 + 32 * NR; }
// slots + PRE rings + dw parking [32][33] + chain reduction [32] + 3*NS
// mbarriers (+ window mode: the chain's padded carry row and POST's
// near-band dV accumulators [32*EPL][2*kWin+1])
__host__ __device__ constexpr int split_smem_floats(int EPL, int NR, int npre, bool win) {
  return kSplitSlots * split_slot_floats(EPL) + npre * kPreStages * split_stage_floats(EPL, NR) + 32 * 33 + 32 +
         3 * kSplitSlots * 2 + 8 + (win ? 32 * (EPL + 1) + 32 * EPL * (2 * kWin + 1) : 0);
}
// padded row index (lane stride EPL+1 words: conflict-free neighbour gathers)
template <int EPL>
__device__ __forceinline__ int pidx(int l) { return l + l / EPL; }

// acc[i] += sum over the sources of target l0+i recorded in wm[i] of val(source)
template <int EPL, class F>
__device__ __forceinline__ void window_gather(float (&acc)[EPL], const uint32_t (&wm)[EPL], int l0, F val) {
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    uint32_t m = wm[i];
    // two sources per trip: both loads in flight, added in ascending order
    while (m) {
      const int k1 = __ffs(m) - 1;
      m &= m - 1;
      const int k2 = m ? __ffs(m) - 1 : k1;
      const bool two = m != 0u;
      m &= m - 1;
      const float v1 = val(l0 + i + k1 - kWin), v2 = val(l0 + i + k2 - kWin);
      acc[i] = fadd(acc[i], v1);
      if (two) acc[i] = fadd(acc[i], v2);
    }
  }
}

// Store a lane's EPL floats to shared memory (vectorised).
template <int EPL>
__device__ __forceinline__ void sts_slice(float* s, const float (&v)[EPL]) {
  if (EPL % 4 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 4) *reinterpret_cast<float4*>(s + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else if (EPL % 2 == 0) {
#pragma unroll
    for (int i = 0; i < EPL; i += 2) *reinterpret_cast<float2*>(s + i) = make_float2(v[i], v[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < EPL; ++i) s[i] = v[i];
  }
}

template <int EPL>
__device__ __forceinline__ float sel_elem(const float (&v)[EPL], int i) {
  float r = v[0];
#pragma unroll
  for (int t = 1; t < EPL; ++t) r = i == t ? v[t] : r;
  return r;
}

__device__ __forceinline__ bool bit(uint32_t w, int k) { return (w >> k) & 1u; }

// acc += scatter of row v given the decoded mask word: near targets through
// registers and neighbour shuffles; the main far group through a warp
// reduction (shared memory `red`, 32 floats, 16 B aligned); other far pairs
// one shuffle each.
template <int EPL, bool NEAR = true, bool SMEM_RED = true>
__device__ __forceinline__ void scatter_row(float (&acc)[EPL], const float (&v)[EPL], uint32_t mword, int main_t,
                                            int noth, const uint16_t* oth, float* red, int lane) {
  float nm[EPL], np[EPL], part = 0.0f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    nm[i] = bit(mword, i) ? v[i] : 0.0f;
    np[i] = bit(mword, 16 + i) ? v[i] : 0.0f;
    part = fadd(part, bit(mword, 24 + i) ? v[i] : 0.0f);
  }
  // label l's target l-1 is owned by l-1: element i-1, or the previous lane's last
  float mn = __shfl_down_sync(0xffffffffu, nm[0], 1);
  float pn = __shfl_up_sync(0xffffffffu, np[EPL - 1], 1);
  mn = lane < 31 ? mn : 0.0f;
  pn = lane > 0 ? pn : 0.0f;
  if (SMEM_RED && main_t >= 0) {
    __syncwarp();
    red[lane] = part;
    __syncwarp();
  }
  if (NEAR) {
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const float m1 = i + 1 < EPL ? nm[i + 1 < EPL ? i + 1 : 0] : mn;
      const float p1 = i > 0 ? np[i > 0 ? i - 1 : 0] : pn;
      acc[i] = fadd(fadd(fadd(acc[i], bit(mword, 8 + i) ? v[i] : 0.0f), m1), p1);
    }
  }
  if (main_t >= 0) {
    float F;
    if (SMEM_RED) {
      float s[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float4 q4 = reinterpret_cast<const float4*>(red)[t];
        s[t] = fadd(fadd(q4.x, q4.y), fadd(q4.z, q4.w));
      }
      F = fadd(fadd(fadd(s[0], s[1]), fadd(s[2], s[3])), fadd(fadd(s[4], s[5]), fadd(s[6], s[7])));
    } else {
      F = warp_sum_f(part);  // throughput role: fewer instructions than the shared-memory tree
    }
    const int im = main_t - lane * EPL;
#pragma unroll
    for (int i = 0; i < EPL; ++i)
      if (im == i) acc[i] = fadd(acc[i], F);
  }
  for (int t = 0; t < noth; ++t) {
    const uint32_t e = oth[t];
    const int src = int(e & 0xffu), tgt = int(e >> 8);
    const float val = __shfl_sync(0xffffffffu, sel_elem<EPL>(v, src % EPL), src / EPL);
    const int it = tgt - lane * EPL;
#pragma unroll
    for (int i = 0; i < EPL; ++i)
      if (it == i) acc[i] = fadd(acc[i], val);
  }
}

// MODE 1: banded D <= 2 (near targets l-1 / l / l+1 through shuffles);
// MODE 2: window (banded D <= 16, or any V with L <= 32): targets within
// +-kWin gathered through per-target source masks; MODE 0: everything else.
__host__ __device__ inline int split_mode(int banded, int D, int L) {
  return (banded && D <= 2) ? 1 : (((banded && D <= 16) || (!banded && L <= 32)) ? 2 : 0);
}

template <int EPL, bool TRWP, int RT, bool FULL, int NPRE, int MODE>
// 3 CTAs per SM: few long scanlines (KITTI rows: 375 lines) run in one wave,
// many lines get 15 warps per SM to hide latency (measured on C2 and C3)
#ifndef MRF_SPLIT_MINB
#define MRF_SPLIT_MINB 3
#endif
__global__ void __launch_bounds__(32 * (2 + NPRE), MRF_SPLIT_MINB) bwd_split_kernel(AccArgs a) {
  const bool band = a.desc->banded != 0;
  const int Dband = a.desc->D;
  if (split_mode(band, Dband, a.g.L) != MODE) return;  // another instantiation owns this sweep
  constexpr bool BAND = MODE == 1, WIN = MODE == 2;
  extern __shared__ __align__(16) float smem[];
  using SL = SlotLayout<EPL>;
  constexpr int NRMAX = RT ? acc_rows(TRWP, RT) : 16;
  constexpr int LS = 32 * EPL;
  constexpr int SLOT = split_slot_floats(EPL);
  static_assert(SL::SIZE <= SLOT, "slot layout");
  const Geometry& g = a.g;
  const int L = g.L, N = g.N;
  const int R = RT ? RT : g.R;
  const int NR = acc_rows(TRWP, R);
#ifndef MRF_ROLE_ROT
#define MRF_ROLE_ROT 3
#endif
  // role index: 0 = CHAIN, 1 = POST, 2.. = PRE, from the hardware warp rotated
  // by MRF_ROLE_ROT: 3 puts CHAIN and POST on hardware warps 2 and 3 (PRE on
  // 0, 1, 4), measured best of the five rotations (C2 backward 16.78 ->
  // 16.12 ms, C3 17.14 -> 16.93; the rotations change which roles share a
  // warp scheduler)
  const int lane = threadIdx.x & 31, warp = ((threadIdx.x >> 5) + MRF_ROLE_ROT) % (2 + NPRE);
  const int stage_f = split_stage_floats(EPL, NR);

  float* slots = smem;                                       // [NS][SLOT]
  float* pre_ring = slots + kSplitSlots * SLOT;              // [NPRE][kPreStages][stage_f]
  float* s_wp = pre_ring + NPRE * kPreStages * stage_f;      // [32][33] POST dw parking
  float* s_red = s_wp + 32 * 33;                             // [32] CHAIN reduction
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_red + 32);  // full[NS], done[NS], empty[NS]
  float* s_c = reinterpret_cast<float*>(bars + 3 * kSplitSlots + 4);  // WIN: chain carry row (padded)
  float* s_dv = s_c + 32 * (EPL + 1);                                    // WIN: [32*EPL][2*kWin+1]
  const uint32_t bar_full = smem_u32(bars);  // [slot] at + 8 * slot
  const uint32_t bar_done = bar_full + 8u * kSplitSlots;
  const uint32_t bar_empty = bar_full + 16u * kSplitSlots;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3 * kSplitSlots; ++i) mbar_init(bars + i, 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int b = blockIdx.y;
  const int NL = N * L;
  const bool first = a.k == g.K_cap - 1;
  const int l0 = lane * EPL;
  const int nvalid = FULL ? EPL : min(EPL, max(0, L - l0));
  const bool wpl = a.pot.w_planes != nullptr, rpl = TRWP && a.pot.rho_planes != nullptr;
  const bool do_w = a.gw != nullptr;

#ifdef MRF_SPLIT_PROF
  long long t_begin = clock64(), t_wait = 0, n_split = 0, n_oth = 0, t_c0 = 0, t_c1 = 0;
  long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tmark = clock64();
#define PMARK(k) { const long long t_ = clock64(); tt[k] += t_ - tmark; tmark = t_; }
#define SPLIT_WAIT(bar, par)         \
  {                                  \
    const long long t0_ = clock64(); \
    mbar_wait(bar, par);             \
    t_wait += clock64() - t0_;       \
  }
#else
#define SPLIT_WAIT(bar, par) mbar_wait(bar, par)
#define PMARK(k)
#endif
  // global step counter across this CTA's lines (slot / phase bookkeeping)
  uint32_t gs0 = 0;
  for (int li = blockIdx.x; li < a.nlines; li += gridDim.x) {
    const LineDesc ld = a.lines[li];
    const int r = ld.dir, opp = r ^ 1, st = g.node_step[r], fam = r >> 1;
    const int nsteps = ld.length - 1;
    const int stL = st * L;
    const int o_first = ld.first * L;
    // edge index over the whole batch: p/q words are addressed from a.p/a.q so
    // that byte offsets stay word-aligned for any b, K_cap and E (K*E odd)
    const uint32_t ebase = (uint32_t(b) * uint32_t(g.K_cap) + uint32_t(a.k)) * uint32_t(g.E) + uint32_t(g.dir_offset[r]) + uint32_t(ld.edge_base);

    if (warp >= 2) {
      // =============================== PRE ===============================
      const int pw = warp - 2;
      float* ring = pre_ring + pw * kPreStages * stage_f;
      const uint32_t ring_s = smem_u32(ring);
      const float* dcb = a.dc + size_t(b) * NL;
      const float* ainb = a.ain + size_t(b) * R * NL;
      const uint8_t* pimg = a.p;
      const uint8_t* qimg = a.q;
      const float* wrow = wpl ? a.pot.w_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
      const float* rrow = rpl ? a.pot.rho_planes + (size_t(b) * (R / 2) + fam) * N : nullptr;
      // the rows gm^r(cur) is assembled from, in accumulation order (-1 = dc)
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
      const int a0 = first ? 1 : 0;  // first plane slot
      const int npl = nrows;         // plane rows end here
      const bool fuse = TRWP && a.dtheta != nullptr;
      const float* rowb[NRMAX];  // each staged row at node 0
#pragma unroll
      for (int rr = 0; rr < NRMAX; ++rr) rowb[rr] = sd[rr] < 0 ? dcb : ainb + size_t(sd[rr] > 0 ? sd[rr] : 0) * NL;

      // this warp's steps: s = pw, pw + NPRE, ...; local index t = s / NPRE
      const int nmine = nsteps > pw ? (nsteps - pw + NPRE - 1) / NPRE : 0;
      // FULL rows: this lane's 16-byte chunks of the staged rows and of the p
      // row at this warp's first node step, stepped back NPRE nodes per issue
      const float* rsrc[NRMAX];
#pragma unroll
      for (int rr = 0; rr < NRMAX; ++rr) rsrc[rr] = rowb[rr] + (o_first + (nsteps - pw) * stL + 4 * lane);
      const uint8_t* psrc = pimg + size_t(ebase + uint32_t(nsteps - pw - 1)) * L + 16 * lane;
      int islot = 0;
      auto issue = [&](int t) {  // t = 0, 1, ... in order
        const int s = pw + t * NPRE;
        const uint32_t base_s = ring_s + 4u * uint32_t(islot * stage_f);
        islot = islot == kPreStages - 1 ? 0 : islot + 1;
        const int j = nsteps - s;
        const int ocur = o_first + j * stL;
#pragma unroll
        for (int rr = 0; rr < NRMAX; ++rr) {
          if (rr < nrows) {
            if (FULL) {  // the row is 8*EPL 16-byte chunks
              const uint32_t d = base_s + 4u * (rr * LS) + 16u * lane;
              if (lane < 8 * EPL) cp_async_u32(d, rsrc[rr], 16);
              if (lane + 32 < 8 * EPL) cp_async_u32(d + 512u, rsrc[rr] + 128, 16);
            } else if (nvalid > 0) {
              cp_slice_t<EPL, false>(base_s + 4u * (rr * LS + l0), rowb[rr] + ocur + l0, nvalid);
            }
          }
          if (FULL) rsrc[rr] -= NPRE * stL;
        }
        const uint32_t e = ebase + uint32_t(j - 1);
        const uint32_t pdst = base_s + 4u * (NR * LS);
        if (FULL) {  // p row: 32*EPL bytes at e*L (16 B aligned)
          if (lane < 2 * EPL) cp_async_u32(pdst + 16u * lane, psrc, 16);
          psrc -= NPRE * L;
        } else {
          const size_t pb = size_t(e) * L;
          const uint32_t* pwd = reinterpret_cast<const uint32_t*>(pimg) + (pb >> 2);
          const int nwords = int(((pb + L - 1) >> 2) - (pb >> 2)) + 1;
          for (int u = lane; u < nwords; u += 32) cp_async_u32(pdst + 4u * u, pwd + u, 4);
        }
        const uint32_t xdst = pdst + 4u * (8 * EPL);
        const int cur = ld.first + j * st;
        const int wnode = (r & 1) ? cur : cur - st;
        if (lane == 0) cp_async_u32(xdst, reinterpret_cast<const uint32_t*>(qimg) + (e >> 2), 4);
        if (wpl && lane == 1) cp_async_u32(xdst + 4u, wrow + wnode, 4);
        if (rpl && lane == 2) cp_async_u32(xdst + 8u, rrow + wnode, 4);
        if (rpl) {
#pragma unroll
          for (int rr = 0; rr < NRMAX; ++rr) {
            if (rr < nrows && sd[rr] >= 0) {
              // rho of direction d's edge with cur as its prev (a tail row is
              // zero, so the clamped entry is then irrelevant)
              const int d = sd[rr];
              const int wn = (d & 1) ? cur + g.node_step[d] : cur;
              const int wc = min(max(wn, 0), N - 1);
              cp_async_u32(xdst + 4u * (4 + 32 * rr + lane),
                           a.pot.rho_planes + (size_t(b) * (R / 2) + (d >> 1)) * N + wc, 4);
            }
          }
        }
      };
#pragma unroll
      for (int t = 0; t < kPreStages - 1; ++t) {
        if (t < nmine) issue(t);
        cp_commit();
      }
      for (int t = 0; t < nmine; ++t) {
        PMARK(7);
        if (t + kPreStages - 1 < nmine) issue(t + kPreStages - 1);
        cp_commit();
        PMARK(0);
        cp_wait<kPreStages - 1>();
        __syncwarp();  // rows and words were copied by other lanes
        PMARK(1);
        const int s = pw + t * NPRE;
        const float* stg = ring + (t % kPreStages) * stage_f;
        const int j = nsteps - s;
        const uint32_t e = ebase + uint32_t(j - 1);
        const uint8_t* prow = reinterpret_cast<const uint8_t*>(stg + NR * LS) + (FULL ? 0 : ((size_t(e) * L) & 3)) + l0;
        const float* xs = stg + NR * LS + 8 * EPL;
        const int qv = (__float_as_uint(xs[0]) >> (8 * (e & 3))) & 0xff;
        // fused dtheta: the running dtheta(cur) row, loaded here so the load
        // overlaps the decode (POST then only adds the carry)
        float dto[EPL];
        if (fuse) {
          const float* src = a.dtheta_src + size_t(b) * NL + o_first + j * stL + l0;
          if (FULL && EPL % 2 == 0) {
#pragma unroll
            for (int i = 0; i < EPL; i += 2) {
              const float2 t2 = __ldcg(reinterpret_cast<const float2*>(src + i));
              dto[i] = t2.x, dto[i + 1] = t2.y;
            }
          } else {
#pragma unroll
            for (int i = 0; i < EPL; ++i) dto[i] = (FULL || i < nvalid) ? __ldcg(src + i) : 0.0f;
          }
        }
#ifdef MRF_SPLIT_PROF
        const long long tc0 = clock64();
#endif

        // ---- x = gm^r(cur) without the carry
        float x[EPL], tv[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) x[i] = 0.0f;
        float rsum[EPL];  // fused dtheta: sum_d rho_d A[d](cur)
        if (!rpl) {
          // uniform rho: x = dc + rho * sum_d A_d - A_opp (TRWP) / dc or sum_d A_d (ISGMR)
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
          for (int i = 0; i < EPL; ++i) rsum[i] = 0.0f;
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
        if (fuse && !(npl > a0)) {
#pragma unroll
          for (int i = 0; i < EPL; ++i) rsum[i] = 0.0f;
        }

        // ---- decode p: near codes, far targets
        int mu[EPL];
        bool far[EPL], near[EPL];
        float lsum = 0.0f;
        uint32_t mword = 0;
        int kmn = 0x7fffffff, kmx = -1;
        if (FULL && EPL % 2 == 0) {  // the lane's p bytes, two per 16-bit load (l0 even: aligned)
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
          const int d = mu[i] - (l0 + i);
          near[i] = valid && uint32_t(d + (WIN ? kWin : 1)) <= uint32_t(WIN ? 2 * kWin : 2);
          far[i] = valid && !near[i];
          // targets l-1 / l / l+1 go through registers in every mode (the
          // window masks carry only 2 <= |d| <= kWin): code c = d + 1 in
          // {0, 1, 2} sets bit 8c + i
          const uint32_t c = uint32_t(d + 1);
          mword |= (valid && c <= 2u) ? (1u << (8 * c + i)) : 0u;
          kmn = min(kmn, far[i] ? mu[i] : 0x7fffffff);
          kmx = max(kmx, far[i] ? mu[i] : -1);
        }
        const float S = warp_sum_f(lsum);
        kmn = __reduce_min_sync(0xffffffffu, kmn);
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        int main_t = kmx;  // -1: no far label
        const bool split = kmx >= 0 && kmn != kmx;
#ifdef MRF_SPLIT_PROF
        n_split += split;
#endif
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

#ifdef MRF_SPLIT_PROF
        t_c0 += clock64() - tc0;
#endif
        // B = scatter(x) - S_x e_{p_q}: needs no slot unless the window masks
        // or the other-pairs list live in it
        const uint8_t* prow0 = prow - l0;  // staged p row, label 0
        float B[EPL];
#pragma unroll
        for (int i = 0; i < EPL; ++i) B[i] = 0.0f;
        auto qfix = [&]() {
          const int im = int(prow0[qv]) - l0;
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (im == i) B[i] = fsub(B[i], S);
        };
        const bool early = !WIN && !split;
        if (early) {
          scatter_row<EPL, true, false>(B, x, mword, main_t, 0, nullptr, nullptr, lane);
          qfix();
        }
        // ---- wait for the slot, then publish
        const uint32_t gs = gs0 + uint32_t(s);
        const int slot = int(gs % kSplitSlots);
        const uint32_t use = gs / kSplitSlots;
        PMARK(2);
        if (use > 0) SPLIT_WAIT(bar_empty + 8u * slot, (use - 1) & 1u);
        PMARK(3);
        float* sl = slots + slot * SLOT;
        uint16_t* olist = reinterpret_cast<uint16_t*>(sl + SL::OTH);
        int noth = 0;
        if (split) {
          // remaining far pairs, compacted in (element, lane) order
          uint32_t lanemask_lt;
          asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lanemask_lt));
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const bool o = far[i] && mu[i] != main_t;
            const uint32_t ball = __ballot_sync(0xffffffffu, o);
            if (o) olist[noth + __popc(ball & lanemask_lt)] = uint16_t((l0 + i) | (mu[i] << 8));
            noth += __popc(ball);
          }
          __syncwarp();
        }
#ifdef MRF_SPLIT_PROF
        n_oth += noth;
#endif
        if (WIN) {
          uint32_t* wmk = reinterpret_cast<uint32_t*>(sl + SL::WM);
#pragma unroll
          for (int i = 0; i < EPL; ++i) wmk[l0 + i] = 0u;
          sts_slice<EPL>(sl + SL::X + l0, x);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < EPL; ++i)
            if (near[i] && uint32_t(mu[i] - (l0 + i) + 1) > 2u) atomicOr(wmk + mu[i], 1u << (kWin - (mu[i] - (l0 + i))));
          __syncwarp();
          uint32_t wm[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) wm[i] = wmk[l0 + i];
          const float* xr = sl + SL::X;
          window_gather<EPL>(B, wm, l0, [&](int l) { return xr[l]; });
        }
        if (!early) {
          scatter_row<EPL>(B, x, mword, main_t, noth, olist, sl + SL::CIN, lane);  // CIN: reduction scratch
          qfix();
        }
        __syncwarp();
        PMARK(4);
        if (!WIN) sts_slice<EPL>(sl + SL::X + l0, x);
        sts_slice<EPL>(sl + SL::B + l0, B);
        if (fuse) {  // dtheta_old + sum_d rho_d A[d](cur), the reference's first add
#pragma unroll
          for (int i = 0; i < EPL; ++i) rsum[i] = fadd(dto[i], rsum[i]);
          sts_slice<EPL>(sl + SL::DT + l0, rsum);
        }
        if (!BAND) {
          uint8_t* pb = reinterpret_cast<uint8_t*>(sl + SL::P);
#pragma unroll
          for (int i = 0; i < EPL; ++i) pb[l0 + i] = uint8_t(mu[i]);
        }
        reinterpret_cast<uint32_t*>(sl + SL::MASK)[lane] = mword;
        if (lane == 0) {
          uint32_t* sc = reinterpret_cast<uint32_t*>(sl + SL::SC);
          sc[SC_Q] = uint32_t(qv);
          sc[SC_S] = __float_as_uint(S);
          sc[SC_MAIN] = uint32_t(main_t);
          sc[SC_NOTH] = uint32_t(noth);
          sc[SC_W] = __float_as_uint(wpl ? xs[1] : a.pot.w);
          sc[SC_RHO] = __float_as_uint(TRWP ? (rpl ? xs[2] : a.pot.rho) : 1.0f);
        }
        mbar_arrive(bar_full + 8u * slot);
        PMARK(5);
      }
      cp_wait<0>();
      __syncwarp();
    } else if (warp == 0) {
      // ============================== CHAIN ==============================
      float carry[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) carry[i] = 0.0f;
      for (int s = 0; s < nsteps; ++s) {
        const uint32_t gs = gs0 + uint32_t(s);
        const int slot = int(gs % kSplitSlots);
        SPLIT_WAIT(bar_full + 8u * slot, (gs / kSplitSlots) & 1u);
        float* sl = slots + slot * SLOT;
        const uint32_t* sc = reinterpret_cast<const uint32_t*>(sl + SL::SC);
        const int main_t = int(sc[SC_MAIN]);
        const int noth = int(sc[SC_NOTH]);
        const float rho = __uint_as_float(sc[SC_RHO]);
        const uint32_t mword = reinterpret_cast<const uint32_t*>(sl + SL::MASK)[lane];
        float acc[EPL];
        lds_slice<EPL>(acc, sl + SL::B + l0);
        if (WIN) {
          __syncwarp();  // the previous step's gathers are done
#pragma unroll
          for (int i = 0; i < EPL; ++i) s_c[pidx<EPL>(l0 + i)] = carry[i];
          uint32_t wm[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) wm[i] = reinterpret_cast<const uint32_t*>(sl + SL::WM)[l0 + i];
          __syncwarp();
          window_gather<EPL>(acc, wm, l0, [&](int l) { return s_c[pidx<EPL>(l)]; });
        }
        scatter_row<EPL>(acc, carry, mword, main_t, noth, reinterpret_cast<const uint16_t*>(sl + SL::OTH), s_red,
                               lane);
        sts_slice<EPL>(sl + SL::CIN + l0, carry);
        sts_slice<EPL>(sl + SL::ACC + l0, acc);
        mbar_arrive(bar_done + 8u * slot);
#pragma unroll
        for (int i = 0; i < EPL; ++i) carry[i] = TRWP ? fmul(rho, acc[i]) : acc[i];
      }
    } else {
      // =============================== POST ==============================
      float* aout_r = a.aout + size_t(b) * R * NL + size_t(r) * NL;
      // this CTA's private dV slot; entry (mu, l) of V' is V[mu][l] (even r) / V[l][mu] (odd r)
      float* gvacc = a.gvacc + (size_t(b) * a.dv_slots + blockIdx.x) * L * L;
      const int vs_mu = (r & 1) ? 1 : L, vs_l = (r & 1) ? L : 1;
      float* gwrow = do_w ? a.gw + (TRWP ? (size_t(b) * (R / 2) + fam) * N : (size_t(b) * R + r) * N) : nullptr;
      const float* gband = a.desc->g;
      const float gb0 = gband[0], gb1 = gband[L > 1 ? 1 : 0], gbD = gband[Dband];
      float zero[EPL];
#pragma unroll
      for (int i = 0; i < EPL; ++i) zero[i] = 0.0f;
      // the tail is no edge's prev: its plane-r row is zero
      stg_slice<EPL>(aout_r + o_first + nsteps * stL, l0, zero, nvalid, L);
      if (WIN && gs0 == 0) {
        for (int t = lane; t < 32 * EPL * (2 * kWin + 1); t += 32) s_dv[t] = 0.0f;
        __syncwarp();
      }
      // dV partials (w folded in at flush when w is constant): near diagonal
      // (mu = l-1, l, l+1) and the main far target while it repeats
      float vacc[EPL][3], fval[EPL];
      int fkey = -1;
#pragma unroll
      for (int i = 0; i < EPL; ++i) fval[i] = vacc[i][0] = vacc[i][1] = vacc[i][2] = 0.0f;
      const float wfold = wpl ? 1.0f : a.pot.w;
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
      const bool fuse = TRWP && a.dtheta != nullptr;
      float* dthb = fuse ? a.dtheta + size_t(b) * NL : nullptr;
      float accl[EPL], rhol = 0.0f;  // last step's acc / rho (the head's own contribution)
#pragma unroll
      for (int i = 0; i < EPL; ++i) accl[i] = 0.0f;
      for (int s = 0; s < nsteps; ++s) {
        const uint32_t gs = gs0 + uint32_t(s);
        const int slot = int(gs % kSplitSlots);
        SPLIT_WAIT(bar_done + 8u * slot, (gs / kSplitSlots) & 1u);
        const float* sl = slots + slot * SLOT;
        const uint32_t* sc = reinterpret_cast<const uint32_t*>(sl + SL::SC);
        const int qv = int(sc[SC_Q]);
        const float S = __uint_as_float(sc[SC_S]);
        const int main_t = int(sc[SC_MAIN]);
        const int noth = int(sc[SC_NOTH]);
        const float w = __uint_as_float(sc[SC_W]);
        const uint32_t mword = reinterpret_cast<const uint32_t*>(sl + SL::MASK)[lane];
        const int j = nsteps - s;
        float acc[EPL], gg[EPL], cin[EPL];
        lds_slice<EPL>(acc, sl + SL::ACC + l0);
        lds_slice<EPL>(gg, sl + SL::X + l0);
        lds_slice<EPL>(cin, sl + SL::CIN + l0);
        stg_slice<EPL>(aout_r + o_first + (j - 1) * stL, l0, acc, nvalid, L);
        if (fuse) {  // dtheta(cur) += sum_d rho_d A[d](cur) + this sweep's own share (the carry)
          float dt[EPL], rs[EPL];
          lds_slice<EPL>(rs, sl + SL::DT + l0);
#pragma unroll
          for (int i = 0; i < EPL; ++i) dt[i] = fadd(rs[i], cin[i]), accl[i] = acc[i];
          stg_slice<EPL>(dthb + o_first + j * stL, l0, dt, nvalid, L);
          rhol = __uint_as_float(sc[SC_RHO]);
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          gg[i] = fadd(gg[i], cin[i]);
          if (qv == l0 + i) gg[i] = fsub(gg[i], S);
        }
        if (main_t != fkey) {  // warp-uniform
          if (fkey >= 0) flush_far();
          fkey = main_t;
        }
        float wpart = 0.0f;
        if (BAND) {
          // dw = g(0) s0 + g(1) s1 + g(D) (sum_l g_l - s0 - s1) with s0 / s1 the
          // sums over p_l == l / |p_l - l| == 1, and sum_l g_l = 0 (the
          // reparametrised row sums to zero: dropping it changes dw only at the
          // rounding level of the reference's own sum)
          // (predicated adds: a label feeds exactly one of the accumulators)
          float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const float ga = wpl ? fmul(gg[i], w) : gg[i];  // dV addend (w folded later if constant)
            const bool cm = bit(mword, i), c0 = bit(mword, 8 + i), cp = bit(mword, 16 + i), cf = bit(mword, 24 + i);
            if (cm) vacc[i][0] = fadd(vacc[i][0], ga);
            if (c0) vacc[i][1] = fadd(vacc[i][1], ga);
            if (cp) vacc[i][2] = fadd(vacc[i][2], ga);
            if (cf) fval[i] = fadd(fval[i], ga);
            if (c0) s0 = fadd(s0, gg[i]);
            if (cm || cp) s1 = fadd(s1, gg[i]);
          }
          if (do_w) wpart = fadd(fmul(fsub(gb0, gbD), s0), fmul(fsub(gb1, gbD), s1));
        } else {
          const uint8_t* pb = reinterpret_cast<const uint8_t*>(sl + SL::P);
          // V'(p_l, l) of every label first: independent loads in flight
          // together instead of one L1 round trip per label in the dw chain
          float vvs[EPL];
          int ms[EPL];
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const int l = l0 + i;
            const bool valid = FULL || i < nvalid;
            ms[i] = valid ? int(pb[l]) : l;
            const int d = ms[i] - l;
            vvs[i] = !do_w ? 0.0f : band ? __ldg(gband + min(abs(d), Dband)) : __ldg(a.pot.V + ms[i] * vs_mu + l * vs_l);
          }
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const float ga = wpl ? fmul(gg[i], w) : gg[i];
            const bool cf = bit(mword, 24 + i);
            const int l = l0 + i;
            const bool valid = FULL || i < nvalid;
            const int m = ms[i];
            const int d = m - l;
            if (WIN) {
              // near-band dV partial of (m, l): this lane owns row l of the
              // shared accumulator, so a plain read-modify-write suffices
              if (valid && d >= -kWin && d <= kWin && ga != 0.0f) {
                float* dv = s_dv + l * (2 * kWin + 1) + d + kWin;
                *dv = fadd(*dv, ga);
              }
            } else {
              const bool cm = bit(mword, i), c0 = bit(mword, 8 + i), cp = bit(mword, 16 + i);
              vacc[i][0] = fadd(vacc[i][0], cm ? ga : 0.0f);
              vacc[i][1] = fadd(vacc[i][1], c0 ? ga : 0.0f);
              vacc[i][2] = fadd(vacc[i][2], cp ? ga : 0.0f);
            }
            fval[i] = fadd(fval[i], cf ? ga : 0.0f);
            if (do_w && valid && gg[i] != 0.0f) {
              wpart = fadd(wpart, fmul(gg[i], vvs[i]));
            }
          }
        }
        if (do_w) {
          s_wp[(s & 31) * 33 + lane] = wpart;
          if ((s & 31) == 31 || s == nsteps - 1) flush_w(s & ~31, (s & 31) + 1);
        }
        if (noth > 0) {
          const uint16_t* ol = reinterpret_cast<const uint16_t*>(sl + SL::OTH);
          for (int t = lane; t < noth; t += 32) {
            const int src = ol[t] & 0xff, tgt = ol[t] >> 8;
            float gv = fadd(sl[SL::X + src], sl[SL::CIN + src]);
            if (src == qv) gv = fsub(gv, S);
            const float gwv = fmul(gv, w);
            if (gwv != 0.0f) red_add_global(gvacc + tgt * vs_mu + src * vs_l, gwv);
          }
        }
        __syncwarp();
        mbar_arrive(bar_empty + 8u * slot);
      }
      if (fuse) {
        // the head is no edge's cur: dtheta(head) += sum_{d != 0} rho_d A[d](head) + rho acc_last
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
          const float* src = a.ain + size_t(b) * R * NL + size_t(d) * NL + size_t(head) * L;
#pragma unroll
          for (int i = 0; i < EPL; ++i) t[i] = (FULL || i < nvalid) ? __ldcg(src + l0 + i) : 0.0f;
#pragma unroll
          for (int i = 0; i < EPL; ++i) hs[i] = fadd(hs[i], fmul(rd, t[i]));
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          if (FULL || i < nvalid) {
            const size_t o = size_t(b) * NL + size_t(head) * L + l0 + i;
            a.dtheta[o] = fadd(fadd(a.dtheta_src[o], hs[i]), nsteps > 0 ? fmul(rhol, accl[i]) : 0.0f);
          }
        }
      }
      if (fkey >= 0) flush_far();
      if (WIN) {
        __syncwarp();
        for (int t = lane; t < L * (2 * kWin + 1); t += 32) {
          const float v = s_dv[t];
          if (v != 0.0f) {
            const int l = t / (2 * kWin + 1), m = l + t % (2 * kWin + 1) - kWin;
            red_add_global(gvacc + m * vs_mu + l * vs_l, fmul(v, wfold));
            s_dv[t] = 0.0f;
          }
        }
        __syncwarp();
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int l = l0 + i;
#pragma unroll
          for (int t = 0; t < 3; ++t) {
            const int m = l + t - 1;
            if (l < L && m >= 0 && m < L && vacc[i][t] != 0.0f) red_add_global(gvacc + m * vs_mu + l * vs_l, fmul(vacc[i][t], wfold));
          }
        }
      }
    }
    gs0 += uint32_t(nsteps);
  }
#ifdef MRF_SPLIT_PROF
  if (lane == 0 && blockIdx.y == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x / 2))
    printf("split cta %d warp %d steps %u total %lld wait %lld split %lld noth %lld | issue %lld cpwait %lld decode %lld empty %lld scatter %lld publish %lld loop %lld\n", blockIdx.x, warp, gs0,
           clock64() - t_begin, t_wait, n_split, n_oth, tt[0], tt[1], tt[2], tt[3], tt[4], tt[5], tt[7]);
#endif
#undef SPLIT_WAIT
}

}  // namespace mrf
