// The sharded step's NVLink traffic with nothing else: every GPU reads slice
// g of every peer's update buffer and writes slice g into every peer's
// replica, all GPUs at once. Kernels start together on a host-mapped flag
// and time themselves with %globaltimer (per GPU; the max span over GPUs),
// so launch skew between GPUs is not counted. Reports GB/s received per GPU: (G-1)*S*16 per direction for
// "read" or "write", twice that for "read+write" (the sharded step).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/p2p_alltoall tools/p2p_alltoall.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kMax = 8;
struct Ptrs { const float4* src[kMax]; float4* dst[kMax]; float4* mine; };

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int MODE, int G>
__global__ void __launch_bounds__(256) step(Ptrs p, long long nv, long long lo, const volatile int* go,
                                            unsigned long long* t_out) {
  if (threadIdx.x == 0) while (*go == 0) {}
  __syncthreads();
  const unsigned long long t0 = gtime();
  const long long stride = (long long)gridDim.x * blockDim.x * 2;
  for (long long base = (long long)blockIdx.x * blockDim.x * 2 + threadIdx.x; base < nv; base += stride) {
    float4 x[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
    if (MODE & 1) {
      float4 g[2][G];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (base + u * blockDim.x < nv)
#pragma unroll
          for (int i = 0; i < G; ++i) g[u][i] = __ldcs(p.src[i] + lo + base + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int i = 0; i < G; ++i) { x[u].x += g[u][i].x; x[u].y += g[u][i].y; x[u].z += g[u][i].z; x[u].w += g[u][i].w; }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long j = base + u * blockDim.x;
      if (j < nv) {
        if (MODE & 2) {
#pragma unroll
          for (int q = 0; q < G; ++q) p.dst[q][lo + j] = x[u];
        } else {
          p.mine[lo + j] = x[u];  // keep the loads live: one local store
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(&t_out[0], t0);
    atomicMax(&t_out[1], gtime());
  }
}

template <int G>
void launch(int mode, int g, Ptrs P, long long nv_shard, const int* go, unsigned long long* t, cudaStream_t s) {
  const long long lo = g * nv_shard;
  const int ctas = 148 * 2;
  if (mode == 1) step<1, G><<<ctas, 256, 0, s>>>(P, nv_shard, lo, go, t);
  if (mode == 2) step<2, G><<<ctas, 256, 0, s>>>(P, nv_shard, lo, go, t);
  if (mode == 3) step<3, G><<<ctas, 256, 0, s>>>(P, nv_shard, lo, go, t);
}

int main(int argc, char** argv) {
  int G = 0;
  cudaGetDeviceCount(&G);
  if (G > kMax) G = kMax;
  if (G < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const long long d = argc > 1 ? atoll(argv[1]) : 23528522ll;
  const long long nv = (d / 4 + G - 1) / G * G, nv_shard = nv / G;
  float4 *src[kMax], *dst[kMax];
  cudaStream_t s[kMax];
  unsigned long long* tdev[kMax];
  int* go = nullptr;
  cudaHostAlloc((void**)&go, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable);
  for (int g = 0; g < G; ++g) {
    cudaSetDevice(g);
    for (int q = 0; q < G; ++q) if (q != g) cudaDeviceEnablePeerAccess(q, 0);
    cudaMalloc(&src[g], nv * 16); cudaMalloc(&dst[g], nv * 16);
    cudaMemset(src[g], 0, nv * 16);
    cudaMalloc(&tdev[g], 16);
    cudaStreamCreate(&s[g]);
  }
  Ptrs P[kMax];
  for (int g = 0; g < G; ++g) {
    for (int q = 0; q < G; ++q) { P[g].src[q] = src[q]; P[g].dst[q] = dst[q]; }
    P[g].mine = dst[g];
  }
  for (int mode = 1; mode <= 3; ++mode) {
    double best = 1e30;
    for (int rep = 0; rep < 6; ++rep) {
      *(volatile int*)go = 0;
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        unsigned long long init[2] = {~0ull, 0ull};
        cudaMemcpy(tdev[g], init, 16, cudaMemcpyHostToDevice);
        int* gdev = nullptr;
        cudaHostGetDevicePointer((void**)&gdev, go, 0);
        if (G == 2) launch<2>(mode, g, P[g], nv_shard, gdev, tdev[g], s[g]);
        else if (G <= 4) launch<4>(mode, g, P[g], nv_shard, gdev, tdev[g], s[g]);
        else launch<8>(mode, g, P[g], nv_shard, gdev, tdev[g], s[g]);
      }
      *(volatile int*)go = 1;
      // %globaltimer is per GPU: each GPU's own span, the max over GPUs
      unsigned long long span = 0;
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        cudaStreamSynchronize(s[g]);
        unsigned long long t[2];
        cudaMemcpy(t, tdev[g], 16, cudaMemcpyDeviceToHost);
        if (t[1] - t[0] > span) span = t[1] - t[0];
      }
      const double ms = span * 1e-6;
      if (rep > 0 && ms < best) best = ms;
    }
    const double per_dir = (double)(G - 1) * nv_shard * 16 * (mode == 3 ? 2 : 1) / (best * 1e6);
    printf("G=%d d=%lld mode=%-10s %.3f ms -> %.1f GB/s received per GPU\n", G, d,
           mode == 1 ? "read" : mode == 2 ? "write" : "read+write", best, per_dir);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
