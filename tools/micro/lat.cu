// Dependent-chain latency of warp primitives on this GPU (cycles per op).
#include <cstdio>
#include <cstdint>
__global__ void k(int* out, float* fo, int n) {
  int lane = threadIdx.x;
  __shared__ float sm[64];
  sm[lane] = lane; sm[lane+32] = lane;
  __syncwarp();
  long long t0, t1;
  // shfl chain
  float v = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffff, v, 1) + 1.0f;
  t1 = clock64();
  if (lane == 0) out[0] = int((t1 - t0) / n);
  // redux chain
  unsigned u = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_min_sync(0xffffffff, u + lane) ;
  t1 = clock64();
  if (lane == 0) out[1] = int((t1 - t0) / n);
  // fadd chain
  float f = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  t1 = clock64();
  if (lane == 0) out[2] = int((t1 - t0) / n);
  // lds chain
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = int(sm[idx & 63]) ;
  t1 = clock64();
  if (lane == 0) out[3] = int((t1 - t0) / n);
  // sts -> syncwarp -> lds round trip
  float w = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { sm[lane] = w; __syncwarp(); w = sm[(lane + 1) & 31] + 1.0f; __syncwarp(); }
  t1 = clock64();
  if (lane == 0) out[4] = int((t1 - t0) / n);
  // fmin + fsetp/select chain (argmin step)
  float b = 1e30f; int bi = 0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { float c = f + i; bool p = c < b; b = p ? c : b; bi = p ? i : bi; f = b; }
  t1 = clock64();
  if (lane == 0) out[5] = int((t1 - t0) / n);
  // bar.sync 64 between 2 warps measured separately
  fo[lane] = v + f + u + idx + w + b + bi;
}
__global__ void kb(int* out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 64;");
  long long t1 = clock64();
  if (threadIdx.x == 0) out[6] = int((t1 - t0) / n);
}
int main() {
  int* d; float* fo; cudaMalloc(&d, 64); cudaMalloc(&fo, 256);
  k<<<1, 32>>>(d, fo, 1000); kb<<<1, 64>>>(d, 1000);
  int h[8]; cudaMemcpy(h, d, 28, cudaMemcpyDeviceToHost);
  printf("cycles/op: shfl+fadd %d, redux %d, fadd %d, lds %d, sts-sync-lds %d, argmin-step %d, bar.sync(2 warps) %d\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
}
