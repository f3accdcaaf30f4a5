// Small C-ABI utilities: finiteness scan, shared-gradient packing and the one
// data-parallel collective (NCCL all-reduce, resolved at run time).
#include <dlfcn.h>

#include <algorithm>
#include <atomic>

#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "launch.hpp"

namespace mrf {

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_total() { return g_launches.load(std::memory_order_relaxed); }

cudaError_t ensure_dynamic_smem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& cur = done[{kern, dev}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

}  // namespace mrf

#include "../../include/mrf_cuda.h"
#include "common.cuh"

namespace {

// Clears *flag when any of x[0:n] is Inf or NaN (exponent all ones). 16-byte
// loads for the aligned bulk; every thread folds its words, one vote per warp.
__global__ void finite_kernel(const float* __restrict__ x, size_t n, int* flag) {
  const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = size_t(gridDim.x) * blockDim.x;
  const size_t head = (reinterpret_cast<uintptr_t>(x) & 15u) ? n : 0;  // unaligned: scalar only
  const size_t nv = (n - head) / 4;
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  uint32_t bad = 0;
  for (size_t i = tid; i < nv; i += nth) {
    const uint4 v = __ldcs(xv + i);
    bad |= ((v.x & 0x7f800000u) == 0x7f800000u) | ((v.y & 0x7f800000u) == 0x7f800000u) |
           ((v.z & 0x7f800000u) == 0x7f800000u) | ((v.w & 0x7f800000u) == 0x7f800000u);
  }
  for (size_t i = 4 * nv + tid; i < n; i += nth) bad |= (__float_as_uint(x[i]) & 0x7f800000u) == 0x7f800000u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 0;
}

// out[0:L*L] = sum_b pairwise[b] (b ascending); out[L*L] = sum of all weight
// planes (GradientSet::edge_weight_total, autodiff.hpp:24-28), one block.
__global__ void pack_kernel(int B, int L, int64_t plane_elems, const float* __restrict__ gv, const float* __restrict__ gw,
                            float* __restrict__ out) {
  const int LL = L * L;
  for (int i = threadIdx.x; i < LL; i += blockDim.x) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s = mrf::fadd(s, gv[size_t(b) * LL + i]);
    out[i] = s;
  }
  __shared__ float part[1024];
  float s = 0.0f;
  if (gw)
    for (int64_t i = threadIdx.x; i < int64_t(B) * plane_elems; i += blockDim.x) s = mrf::fadd(s, gw[i]);
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int i = 0; i < int(blockDim.x); ++i) t = mrf::fadd(t, part[i]);
    out[LL] = t;
  }
}

}  // namespace

extern "C" {

int mrf_check_finite_f32(const float* data, size_t count, int* all_finite, cudaStream_t stream) {
  if (!data || !all_finite) return MRF_EINVAL;
  int* dflag = nullptr;
  cudaError_t e = cudaMallocAsync(&dflag, sizeof(int), stream);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? MRF_ENOMEM : MRF_ECUDA;
  const int one = 1;
  cudaMemcpyAsync(dflag, &one, sizeof(int), cudaMemcpyHostToDevice, stream);
  if (count) {
    const size_t blocks = std::min<size_t>(148 * 8, (count / 4 + 255) / 256 + 1);
    finite_kernel<<<unsigned(blocks), 256, 0, stream>>>(data, count, dflag);
    mrf::note_launch();
  }
  int h = 0;
  cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, stream);
  cudaFreeAsync(dflag, stream);
  e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return MRF_ECUDA;
  *all_finite = h;
  return MRF_OK;
}

int mrf_pack_shared_grads_f32(const mrf_problem_f32* prob, int num_dirs, const mrf_grads_f32* grads, float* out,
                              cudaStream_t stream) {
  if (!prob || !grads || !grads->pairwise || !out || prob->batch < 1 || prob->labels < 1) return MRF_EINVAL;
  const int64_t plane_elems = int64_t(num_dirs / 2) * prob->height * prob->width;
  pack_kernel<<<1, 1024, 0, stream>>>(prob->batch, prob->labels, plane_elems, grads->pairwise, grads->weight_planes,
                                      out);
  mrf::note_launch();
  return cudaGetLastError() == cudaSuccess ? MRF_OK : MRF_ECUDA;
}

int mrf_allreduce_grads_f32(void* nccl_comm, float* buffer, size_t count, cudaStream_t stream) {
  // ncclAllReduce(sendbuff, recvbuff, count, ncclFloat=7, ncclSum=0, comm, stream)
  using AllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  static AllReduceFn fn = nullptr;
  if (!nccl_comm || !buffer) return MRF_EINVAL;
  if (!fn) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return MRF_ECUDA;
    fn = reinterpret_cast<AllReduceFn>(dlsym(h, "ncclAllReduce"));
    if (!fn) return MRF_ECUDA;
  }
  return fn(buffer, buffer, count, /*ncclFloat32*/ 7, /*ncclSum*/ 0, nccl_comm, stream) == 0 ? MRF_OK : MRF_ECUDA;
}

}  // extern "C"

extern "C" int mrf_launch_count(int64_t* total) {
  if (!total) return MRF_EINVAL;
  *total = mrf::launch_total();
  return MRF_OK;
}
