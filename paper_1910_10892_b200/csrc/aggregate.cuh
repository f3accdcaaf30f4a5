// Aggregation (inference.hpp:25-57): c = theta + sum_r m^r in direction
// order and the first argmin label per node (strict '<', lowest label on
// ties). A null unary gives the plain message sum of standard SGM
// (baselines.hpp:84-93). One warp per node row.
#pragma once

#include "common.cuh"
#include "fwd_warp.cuh"

namespace mrf {

// c = theta + sum_r m^r (r ascending) and labels = first argmin
// (inference.hpp:25-57). One warp per node.
// fused: the last TRWP sweep already wrote cost / labels when its owner was
// the banded D == 2 kernel (bit 0) or the dense small-L kernel (bit 1; PairDesc).
__global__ void aggregate_kernel(int B, int N, int L, int R, const float* __restrict__ unary,
                                 const float* __restrict__ m, float* __restrict__ cost, uint16_t* __restrict__ labels,
                                 const PairDesc* __restrict__ desc, int fused) {
  if ((fused & 1) && desc->banded && desc->D == 2) return;
  if ((fused & 2) && !desc->banded) return;
  const int lane = threadIdx.x & 31;
  // persistent grid (capped on the host): a fused call exits in microseconds
  const int64_t nwarp = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); gw < int64_t(B) * N; gw += nwarp) {
    const int b = int(gw / N), i = int(gw - int64_t(b) * N);
    const size_t row = (size_t(b) * N + i) * L;
    uint32_t best_k = 0xffffffffu, best_t = 0xffffffffu;
    for (int l = lane; l < L; l += 32) {
      float c = unary ? __ldg(unary + row + l) : 0.0f;  // null: plain message sum (standard SGM)
      for (int r = 0; r < R; ++r) c = fadd(c, __ldg(m + ((size_t(b) * R + r) * N + i) * L + l));
      if (cost) cost[row + l] = c;
      const uint32_t kk = order_key(fadd(c, 0.0f));
      if (kk < best_k) {
        best_k = kk;
        best_t = uint32_t(l);
      }
    }
    const uint32_t kmin = __reduce_min_sync(0xffffffffu, best_k);
    const uint32_t tmin = __reduce_min_sync(0xffffffffu, best_k == kmin ? best_t : 0xffffffffu);
    if (lane == 0 && labels) labels[size_t(b) * N + i] = uint16_t(tmin);
  }
}

}  // namespace mrf
