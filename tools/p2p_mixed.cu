// Both GPUs at once: each reads N bytes from its peer and writes N bytes into
// its peer (the sharded step's traffic pattern). Reports per-direction GB/s.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void mixed(const float4* __restrict__ peer_src, float4* __restrict__ peer_dst,
                      const float4* __restrict__ lsrc, float4* __restrict__ ldst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    if (MODE & 1) { float4 v = peer_src[j]; ldst[j] = v; }        // pull-style
    if (MODE & 2) { float4 v = lsrc[j]; peer_dst[j] = v; }        // push-style
  }
}
int main() {
  long long bytes = 256ll << 20, n = bytes / 16;
  float4 *a[2], *b[2], *c[2], *dd[2]; cudaStream_t s[2]; cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaDeviceEnablePeerAccess(1 - g, 0);
    cudaMalloc(&a[g], bytes); cudaMalloc(&b[g], bytes); cudaMalloc(&c[g], bytes); cudaMalloc(&dd[g], bytes);
    cudaMemset(a[g], 0, bytes); cudaStreamCreate(&s[g]); cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]); }
  for (int mode = 1; mode <= 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventRecord(e0[g], s[g]);
        if (mode == 1) mixed<1><<<148 * 8, 256, 0, s[g]>>>(a[1 - g], b[1 - g], c[g], dd[g], n);
        if (mode == 2) mixed<2><<<148 * 8, 256, 0, s[g]>>>(a[1 - g], b[1 - g], c[g], dd[g], n);
        if (mode == 3) mixed<3><<<148 * 8, 256, 0, s[g]>>>(a[1 - g], b[1 - g], c[g], dd[g], n);
        cudaEventRecord(e1[g], s[g]); }
      float ms[2];
      for (int g = 0; g < 2; ++g) { cudaSetDevice(g); cudaEventSynchronize(e1[g]); cudaEventElapsedTime(&ms[g], e0[g], e1[g]); }
      float m = ms[0] > ms[1] ? ms[0] : ms[1];
      double per_dir = (mode == 3 ? 2.0 : 1.0) * bytes / (m * 1e6);
      printf("mode %s: %.3f ms -> %.1f GB/s per direction\n", mode == 1 ? "both-read" : mode == 2 ? "both-write" : "read+write", m, per_dir);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
