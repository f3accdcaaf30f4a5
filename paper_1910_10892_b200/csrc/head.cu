// Readout and evaluation around the message-passing path (sm_100a), the
// callers SURVEY.md §8f ranks first and second:
//  * soft head (softhead.hpp:22-74): per node softmax(-c), expected label d,
//    mean |d - target| loss, and the loss gradient w.r.t. the cost volume --
//    the backward's input in training -- in ONE pass over the cost volume
//    (forward and backward fused: both only need the node's own row);
//  * energy of a labelling (potentials.hpp:175-199): unaries plus every
//    undirected edge once (the even direction of each family), in double.
// One warp per node row, lanes strided over labels; per-image totals come
// from fixed-order block partials (deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"

namespace mrf {
namespace {

constexpr int kHeadWarps = 8;  // warps (nodes in flight) per block

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fadd(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// grid (blocks_x, B): block partials of sum_i |d_i - t_i| in double
__global__ void __launch_bounds__(32 * kHeadWarps)
    soft_head_kernel(int N, int L, const float* __restrict__ cost, const float* __restrict__ target,
                     float* __restrict__ conf, float* __restrict__ disp, float* __restrict__ grad,
                     double* __restrict__ partial) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int b = blockIdx.y;
  const size_t NL = size_t(N) * L;
  double acc = 0.0;
  for (int i = blockIdx.x * kHeadWarps + wid; i < N; i += gridDim.x * kHeadWarps) {
    const float* c = cost + b * NL + size_t(i) * L;
    // softhead.hpp:36-45: f = exp(-c - max(-c)) / sum
    float hi = -kInf;
    for (int l = lane; l < L; l += 32) hi = fmaxf(hi, -c[l]);
    hi = warp_max_f(hi);
    float sum = 0.0f;
    for (int l = lane; l < L; l += 32) sum = fadd(sum, expf(fsub(-c[l], hi)));
    sum = warp_sum(sum);
    float d = 0.0f;
    for (int l = lane; l < L; l += 32) {
      const float f = __fdiv_rn(expf(fsub(-c[l], hi)), sum);
      if (conf) conf[b * NL + size_t(i) * L + l] = f;
      d = fadd(d, fmul(float(l), f));
    }
    d = warp_sum(d);
    const float t = target[size_t(b) * N + i];
    const float diff = fsub(d, t);
    if (lane == 0) {
      if (disp) disp[size_t(b) * N + i] = d;
      acc += fabs(double(diff));
    }
    if (grad) {
      // softhead.hpp:62-73: sign(d - t)/N * (-f (l - d)); exact ties give zero
      const float s = diff == 0.0f ? 0.0f : __fdiv_rn(diff > 0.0f ? 1.0f : -1.0f, float(N));
      for (int l = lane; l < L; l += 32) {
        const float f = __fdiv_rn(expf(fsub(-c[l], hi)), sum);
        grad[b * NL + size_t(i) * L + l] = diff == 0.0f ? 0.0f : fmul(s, -fmul(f, fsub(float(l), d)));
      }
    }
  }
  __shared__ double s_acc[kHeadWarps];
  if (lane == 0) s_acc[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kHeadWarps; ++w) t += s_acc[w];
    partial[size_t(b) * gridDim.x + blockIdx.x] = t;
  }
}

// loss[b] = (sum of the image's partials in block order) / N, as float
__global__ void finish_mean_kernel(int B, int nblk, int N, const double* __restrict__ partial, float* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double t = 0.0;
  for (int k = 0; k < nblk; ++k) t += partial[size_t(b) * nblk + k];
  out[b] = float(t / double(N));
}

// grid (blocks_x, B): partials of the unary and pairwise terms in double
__global__ void __launch_bounds__(256)
    energy_kernel(int H, int W, int L, int R, EvenSteps st, const float* __restrict__ unary,
                  const float* __restrict__ V, float w, const float* __restrict__ wplanes,
                  const uint16_t* __restrict__ labels, double* __restrict__ partial, int* __restrict__ bad) {
  const int b = blockIdx.y;
  const int N = H * W;
  const uint16_t* lab = labels + size_t(b) * N;
  double e = 0.0;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const int x = lab[n];
    if (x >= L) {
      *bad = 1;
      continue;
    }
    e += double(unary[(size_t(b) * N + n) * L + x]);
    const int h = n / W, c = n - h * W;
    for (int r = 0; r < R; r += 2) {  // every undirected edge once: the family's even direction
      const int h2 = h + st.dh[r >> 1], c2 = c + st.dw[r >> 1];
      if (h2 < 0 || h2 >= H || c2 < 0 || c2 >= W) continue;
      const int m = h2 * W + c2;
      const int y = lab[m];
      if (y >= L) continue;  // reported by its own node
      const float we = wplanes ? wplanes[(size_t(b) * (R / 2) + (r >> 1)) * N + n] : w;  // plane at prev (even r)
      e += double(we) * double(V[size_t(x) * L + y]);
    }
  }
  __shared__ double s[256];
  s[threadIdx.x] = e;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[size_t(b) * gridDim.x + blockIdx.x] = s[0];
}

__global__ void finish_sum_kernel(int B, int nblk, const double* __restrict__ partial, double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double t = 0.0;
  for (int k = 0; k < nblk; ++k) t += partial[size_t(b) * nblk + k];
  out[b] = t;
}

}  // namespace

cudaError_t launch_soft_head(int B, int N, int L, const float* cost, const float* target, float* conf, float* disp,
                             float* grad, float* loss, double* partial, int nblk, cudaStream_t s) {
  soft_head_kernel<<<dim3(nblk, B), 32 * kHeadWarps, 0, s>>>(N, L, cost, target, conf, disp, grad, partial); note_launch();
  finish_mean_kernel<<<(B + 127) / 128, 128, 0, s>>>(B, nblk, N, partial, loss); note_launch();
  return cudaGetLastError();
}

int soft_head_blocks(int N) { return std::max(1, std::min(148 * 8, (N + kHeadWarps - 1) / kHeadWarps)); }

cudaError_t launch_energy(int B, int H, int W, int L, int R, const EvenSteps& st, const float* unary, const float* V,
                          float w, const float* wplanes, const uint16_t* labels, double* out, double* partial, int nblk,
                          int* bad, cudaStream_t s) {
  energy_kernel<<<dim3(nblk, B), 256, 0, s>>>(H, W, L, R, st, unary, V, w, wplanes, labels, partial, bad); note_launch();
  finish_sum_kernel<<<(B + 127) / 128, 128, 0, s>>>(B, nblk, partial, out); note_launch();
  return cudaGetLastError();
}

int energy_blocks(int N) { return std::max(1, std::min(148 * 4, (N + 255) / 256)); }

}  // namespace mrf
