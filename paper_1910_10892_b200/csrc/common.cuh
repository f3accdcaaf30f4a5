// Shared device helpers for the message-passing kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mrf {

constexpr int kMaxDirs = 16;

// Everything a sweep kernel needs to address one image's tensors. Strides are
// per image (batch index = blockIdx.y).
struct Geometry {
  int N, L, R, W;
  int K_cap;                       // iterations the index store holds
  int64_t E;                       // total edges per iteration
  int64_t dir_offset[kMaxDirs];    // IndexStore::dir_offset(r)
  int node_step[kMaxDirs];         // dh*W + dw
};

struct Potentials {
  const float* unary;      // [B][N][L]
  const float* V;          // [L][L]
  float w;                 // constant weight (w_planes == nullptr)
  const float* w_planes;   // [B][R/2][N]
  float rho;               // constant rho (rho_planes == nullptr)
  const float* rho_planes; // [B][R/2][N]
};

// A scanline with at least one edge: head node, node count, edge base, direction.
struct __align__(16) LineDesc {
  int32_t first, length, edge_base, dir;
};

__device__ __forceinline__ float plane_value(const float* planes, float c, int N, int R, int b, int r, int prev,
                                             int cur) {
  if (planes == nullptr) return c;
  return __ldg(planes + (size_t(b) * (R / 2) + (r >> 1)) * N + ((r & 1) ? cur : prev));
}

// Monotone float -> uint32 map (non-NaN inputs). -0 is folded onto +0 by the
// caller (v + 0.0f) so that equal values compare equal, as the reference's
// strict '<' scans treat them.
// packed f32x2 helpers (FADD2)
__device__ __forceinline__ uint64_t pack2f(float x, float y) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void unpack2f(uint64_t v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}
// two IEEE round-to-nearest adds in one FADD2 (products stay scalar: ptxas
// would contract mul.rn.f32x2 + add.rn.f32x2 into FFMA2)
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// warp-wide minimum of a float in one CREDUX.MIN.F32 (sm_100a); callers pass
// no NaN and no -0 (values normalised by +0 where a -0 can occur), so the
// result equals the order-key minimum bit for bit
__device__ __forceinline__ float warp_min_f32(float v) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ uint32_t order_key(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_value(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// No FMA contraction anywhere on the path: one rounding per operation, in the
// reference's order (SURVEY.md §7 hard part 1).
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }

// Fire-and-forget global float reduction (RED.E.ADD.F32), without the
// generic-address space test atomicAdd() emits.
__device__ __forceinline__ void red_add_global(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;\n" ::"l"(p), "f"(v) : "memory");
}

}  // namespace mrf
