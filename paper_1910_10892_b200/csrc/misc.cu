// Small C-ABI utilities: finiteness scan, shared-gradient packing and the one
// data-parallel collective (NCCL all-reduce, resolved at run time).
#include <dlfcn.h>

#include <algorithm>
#include <atomic>

#include <cstdio>
#include <cstring>
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

// Shared-gradient pack, deterministic (fixed partition, fixed-order sums):
// pack_dw_kernel: block j sums the contiguous chunk j of all weight-plane
// gradients (grid-size independent of the device) into part[j];
// pack_kernel: out[0:L*L] = sum_b pairwise[b] (b ascending) and out[L*L] =
// sum_j part[j] (GradientSet::edge_weight_total, autodiff.hpp:24-28).
constexpr int kPackChunks = 1024;

__global__ void __launch_bounds__(256) pack_dw_kernel(int64_t n, const float* __restrict__ gw, float* __restrict__ part) {
  const int64_t per = (n + kPackChunks - 1) / kPackChunks;
  const int64_t lo = int64_t(blockIdx.x) * per, hi = lo + per < n ? lo + per : n;
  float s = 0.0f;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) s = mrf::fadd(s, gw[i]);
  __shared__ float red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (int(threadIdx.x) < o) red[threadIdx.x] = mrf::fadd(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void pack_kernel(int B, int L, const float* __restrict__ gv, const float* __restrict__ part,
                            float* __restrict__ out) {
  const int LL = L * L;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < LL; i += gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s = mrf::fadd(s, gv[size_t(b) * LL + i]);
    out[i] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float t = 0.0f;
    if (part)
      for (int j = 0; j < kPackChunks; ++j) t = mrf::fadd(t, part[j]);
    out[LL] = t;
  }
}

}  // namespace

namespace mrf {
cudaError_t launch_finite_scan(const float* data, size_t count, int* flag, cudaStream_t stream) {
  if (!count) return cudaSuccess;
  const size_t blocks = std::min<size_t>(148 * 8, (count / 4 + 255) / 256 + 1);
  finite_kernel<<<unsigned(blocks), 256, 0, stream>>>(data, count, flag);
  note_launch();
  return cudaGetLastError();
}
}  // namespace mrf

extern "C" {

int mrf_check_finite_f32(const float* data, size_t count, int* all_finite, cudaStream_t stream) {
  if (!data || !all_finite) return MRF_EINVAL;
  int* dflag = nullptr;
  cudaError_t e = cudaMallocAsync(&dflag, sizeof(int), stream);
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? MRF_ENOMEM : MRF_ECUDA;
  const int one = 1;
  cudaMemcpyAsync(dflag, &one, sizeof(int), cudaMemcpyHostToDevice, stream);
  mrf::launch_finite_scan(data, count, dflag, stream);
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
  const int64_t n = int64_t(prob->batch) * (num_dirs / 2) * prob->height * prob->width;
  float* part = nullptr;
  if (grads->weight_planes) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(float) * kPackChunks, stream) != cudaSuccess)
      return MRF_ENOMEM;
    pack_dw_kernel<<<kPackChunks, 256, 0, stream>>>(n, grads->weight_planes, part);
    mrf::note_launch();
  }
  const int LL = prob->labels * prob->labels;
  pack_kernel<<<(LL + 255) / 256, 256, 0, stream>>>(prob->batch, prob->labels, grads->pairwise, part, out);
  mrf::note_launch();
  if (part) cudaFreeAsync(part, stream);
  return cudaGetLastError() == cudaSuccess ? MRF_OK : MRF_ECUDA;
}

}  // extern "C"

namespace {

// NCCL is resolved at run time (no link dependency): the library torch
// already loaded when present, else the system libnccl.so.2.
struct NcclUniqueId {
  char internal[128];
};
struct Nccl {
  int (*get_unique_id)(NcclUniqueId*) = nullptr;
  int (*comm_init_rank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*get_error_string)(int) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl t;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return t;
    t.get_unique_id = reinterpret_cast<decltype(t.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    t.comm_init_rank = reinterpret_cast<decltype(t.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    t.comm_destroy = reinterpret_cast<decltype(t.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    t.all_reduce = reinterpret_cast<decltype(t.all_reduce)>(dlsym(h, "ncclAllReduce"));
    t.get_error_string = reinterpret_cast<decltype(t.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    t.ok = t.get_unique_id && t.comm_init_rank && t.comm_destroy && t.all_reduce;
    return t;
  }();
  return n;
}

}  // namespace

extern "C" {

int mrf_nccl_unique_id(void* out, size_t bytes) {
  const Nccl& n = nccl();
  if (!out || bytes < sizeof(NcclUniqueId)) return MRF_EINVAL;
  if (!n.ok) return MRF_ECUDA;
  return n.get_unique_id(static_cast<NcclUniqueId*>(out)) == 0 ? MRF_OK : MRF_ECUDA;
}

int mrf_nccl_comm_init(void** comm, int nranks, const void* unique_id, int rank) {
  const Nccl& n = nccl();
  if (!comm || !unique_id || nranks < 1 || rank < 0 || rank >= nranks) return MRF_EINVAL;
  if (!n.ok) return MRF_ECUDA;
  NcclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  return n.comm_init_rank(comm, nranks, id, rank) == 0 ? MRF_OK : MRF_ECUDA;
}

int mrf_nccl_comm_destroy(void* comm) {
  const Nccl& n = nccl();
  if (!comm) return MRF_EINVAL;
  if (!n.ok) return MRF_ECUDA;
  return n.comm_destroy(comm) == 0 ? MRF_OK : MRF_ECUDA;
}

int mrf_allreduce_grads_f32(void* nccl_comm, float* buffer, size_t count, cudaStream_t stream) {
  const Nccl& n = nccl();
  if (!nccl_comm || !buffer) return MRF_EINVAL;
  if (!n.ok) return MRF_ECUDA;
  // ncclAllReduce(sendbuff, recvbuff, count, ncclFloat32 = 7, ncclSum = 0, comm, stream), in place
  return n.all_reduce(buffer, buffer, count, 7, 0, nccl_comm, stream) == 0 ? MRF_OK : MRF_ECUDA;
}

}  // extern "C"

extern "C" int mrf_launch_count(int64_t* total) {
  if (!total) return MRF_EINVAL;
  *total = mrf::launch_total();
  return MRF_OK;
}
