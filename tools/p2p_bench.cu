// P2P access-pattern microbenchmark (2 GPUs): which load/store flavour and
// how much memory-level parallelism reaches the NVLink roofline.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float4 ld_nc(const float4* p) { float4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p)); return v; }
__device__ __forceinline__ float4 ld_cg(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ float4 ld_pl(const float4* p) { return *p; }
template <int MODE, int U>
__global__ void rd(const float4* __restrict__ src, float4* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x * U;
  for (long long b = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; b < n; b += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = b + (long long)u * blockDim.x; if (j < n) v[u] = MODE == 0 ? ld_pl(src + j) : MODE == 1 ? ld_nc(src + j) : ld_cg(src + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long j = b + (long long)u * blockDim.x; if (j < n) dst[j] = v[u]; }
  }
}
template <int MODE, int U>
float run(const float4* src, float4* dst, long long n, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) rd<MODE, U><<<blocks, threads>>>(src, dst, n);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) rd<MODE, U><<<blocks, threads>>>(src, dst, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 5;
}
int main() {
  long long bytes = 256ll << 20, n = bytes / 16;
  float4 *remote, *local, *local2;
  cudaSetDevice(1); cudaMalloc(&remote, bytes); cudaMemset(remote, 0, bytes);
  cudaSetDevice(0); cudaDeviceEnablePeerAccess(1, 0); cudaMalloc(&local, bytes); cudaMalloc(&local2, bytes); cudaMemset(local, 0, bytes);
  int cfgs[][2] = {{148 * 4, 256}, {148 * 8, 256}, {148 * 2, 1024}, {148 * 16, 256}};
  for (auto& c : cfgs) {
    printf("grid %d x %d\n", c[0], c[1]);
    printf("  read remote plain U1 %.1f U4 %.1f | nc U1 %.1f U4 %.1f | cg U1 %.1f U4 %.1f GB/s\n",
      bytes / run<0,1>(remote, local, n, c[0], c[1]) / 1e6, bytes / run<0,4>(remote, local, n, c[0], c[1]) / 1e6,
      bytes / run<1,1>(remote, local, n, c[0], c[1]) / 1e6, bytes / run<1,4>(remote, local, n, c[0], c[1]) / 1e6,
      bytes / run<2,1>(remote, local, n, c[0], c[1]) / 1e6, bytes / run<2,4>(remote, local, n, c[0], c[1]) / 1e6);
    printf("  write remote plain U1 %.1f U4 %.1f GB/s ; local copy U4 %.1f GB/s (r+w)\n",
      bytes / run<0,1>(local, remote, n, c[0], c[1]) / 1e6, bytes / run<0,4>(local, remote, n, c[0], c[1]) / 1e6,
      2 * bytes / run<0,4>(local, local2, n, c[0], c[1]) / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
