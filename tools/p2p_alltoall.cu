// All G GPUs at once, the sharded step's traffic without any flags: GPU g
// reads slice g of every peer's update buffer and writes slice g into every
// peer's replica. Reports per-GPU received GB/s ((G-1)*S*4 per direction per
// mode, 2x for read+write). Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kMax = 8;
struct Ptrs { const float4* src[kMax]; float4* dst[kMax]; };

template <int MODE, int G, int U>
__global__ void __launch_bounds__(256) step(Ptrs p, int me, long long nv, long long lo) {
  const long long stride = (long long)gridDim.x * blockDim.x * U;
  for (long long base = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; base < nv; base += stride) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (MODE & 1) {
      float4 g[U][G];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = base + (long long)u * blockDim.x;
        if (j < nv)
#pragma unroll
          for (int i = 0; i < G; ++i) g[u][i] = __ldcs(p.src[i] + lo + j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < G; ++i) { x[u].x += g[u][i].x; x[u].y += g[u][i].y; x[u].z += g[u][i].z; x[u].w += g[u][i].w; }
    }
    if (MODE & 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long j = base + (long long)u * blockDim.x;
        if (j < nv)
#pragma unroll
          for (int q = 0; q < G; ++q) p.dst[q][lo + j] = x[u];
      }
    }
  }
}

template <int G, int U>
void run(int mode, Ptrs* P, cudaStream_t* s, cudaEvent_t* e0, cudaEvent_t* e1, long long nv_shard, int ctas) {
  for (int g = 0; g < G; ++g) {
    cudaSetDevice(g);
    cudaEventRecord(e0[g], s[g]);
    const long long lo = g * nv_shard;
    if (mode == 1) step<1, G, U><<<ctas, 256, 0, s[g]>>>(P[g], g, nv_shard, lo);
    if (mode == 2) step<2, G, U><<<ctas, 256, 0, s[g]>>>(P[g], g, nv_shard, lo);
    if (mode == 3) step<3, G, U><<<ctas, 256, 0, s[g]>>>(P[g], g, nv_shard, lo);
    cudaEventRecord(e1[g], s[g]);
  }
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
  cudaEvent_t e0[kMax], e1[kMax];
  for (int g = 0; g < G; ++g) {
    cudaSetDevice(g);
    for (int q = 0; q < G; ++q) if (q != g) cudaDeviceEnablePeerAccess(q, 0);
    cudaMalloc(&src[g], nv * 16); cudaMalloc(&dst[g], nv * 16);
    cudaMemset(src[g], 0, nv * 16);
    cudaStreamCreate(&s[g]); cudaEventCreate(&e0[g]); cudaEventCreate(&e1[g]);
  }
  Ptrs P[kMax];
  for (int g = 0; g < G; ++g) for (int q = 0; q < G; ++q) { P[g].src[q] = src[q]; P[g].dst[q] = dst[q]; }
  const int ctas_list[] = {148, 296, 592};
  for (int mode = 1; mode <= 3; ++mode)
    for (int ci = 0; ci < 3; ++ci)
      for (int ui = 0; ui < 2; ++ui) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
          const int ctas = ctas_list[ci];
#define RUN(GG) if (G == GG) { if (ui == 0) run<GG, 1>(mode, P, s, e0, e1, nv_shard, ctas); else run<GG, 2>(mode, P, s, e0, e1, nv_shard, ctas); }
          RUN(2) RUN(4) RUN(8)
          float m = 0.f;
          for (int g = 0; g < G; ++g) {
            cudaSetDevice(g); cudaEventSynchronize(e1[g]);
            float ms; cudaEventElapsedTime(&ms, e0[g], e1[g]);
            if (ms > m) m = ms;
          }
          if (rep > 0 && m < best) best = m;
        }
        const double per_dir = (double)(G - 1) * nv_shard * 16 * (mode == 3 ? 2 : 1) / (best * 1e6);
        printf("G=%d d=%lld mode=%s ctas=%d U=%d: %.3f ms -> %.1f GB/s received per GPU\n", G, d,
               mode == 1 ? "read" : mode == 2 ? "write" : "read+write", ctas_list[ci], ui + 1, best, per_dir);
      }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
