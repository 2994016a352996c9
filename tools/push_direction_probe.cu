// Which NVLink direction should carry the sharded step's push? (VERDICT r1,
// "test the other sharded push direction".) One process drives G GPUs; every
// kernel starts together on a host-mapped flag and times itself with
// %globaltimer (per GPU span, max over GPUs; host launch skew not counted).
//
//  A  owner loads (the engine's k_shard_run): owner g streams its shard once,
//     loading every worker's update slice (G-1 of them over NVLink), applying
//     them in order and storing the new slice into every replica (G-1 over
//     NVLink). One pass: NVLink reads + writes at once.
//  B  worker stores (the north star's sketch): phase 1, every worker stores
//     its update slices into the owners' inboxes (NVLink writes only); phase
//     2, every owner applies from its local inbox and stores the new slice
//     into every replica (NVLink writes only). Two passes; the barrier
//     between them is NOT counted (an upper bound on B's benefit).
// Same arithmetic (w - lr*g, rounded, no FMA) and the same bytes per GPU.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/push_direction_probe tools/push_direction_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kMax = 8;
struct Bufs {
  const float4* upd[kMax];  // each worker's update (full d)
  float4* rep[kMax];        // each worker's replica (full d)
  float4* inbox[kMax];      // each owner's inbox: [G][S]
  float4* w;                // this owner's shard
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ float4 ap(float4 x, float lr, float4 g) {
  x.x = __fsub_rn(x.x, __fmul_rn(lr, g.x)); x.y = __fsub_rn(x.y, __fmul_rn(lr, g.y));
  x.z = __fsub_rn(x.z, __fmul_rn(lr, g.z)); x.w = __fsub_rn(x.w, __fmul_rn(lr, g.w));
  return x;
}
__device__ __forceinline__ void start(const volatile int* go) {
  if (threadIdx.x == 0) while (*go == 0) {}
  __syncthreads();
}
__device__ __forceinline__ void stop(unsigned long long t0, unsigned long long* t) {
  __syncthreads();
  if (threadIdx.x == 0) { atomicMin(&t[0], t0); atomicMax(&t[1], gtime()); }
}

template <int G>
__global__ void __launch_bounds__(256) owner_loads(Bufs b, int me, long long S, float lr, const volatile int* go,
                                                   unsigned long long* t) {
  start(go);
  const unsigned long long t0 = gtime();
  const long long lo = me * S, stride = (long long)gridDim.x * blockDim.x * 2;
  for (long long base = (long long)blockIdx.x * blockDim.x * 2 + threadIdx.x; base < S; base += stride) {
    float4 g[2][G], x[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long j = base + u * blockDim.x;
      if (j < S) {
#pragma unroll
        for (int i = 0; i < G; ++i) g[u][i] = __ldcs(b.upd[i] + lo + j);
        x[u] = b.w[j];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long j = base + u * blockDim.x;
      if (j < S) {
#pragma unroll
        for (int i = 0; i < G; ++i) x[u] = ap(x[u], lr, g[u][i]);
        b.w[j] = x[u];
#pragma unroll
        for (int q = 0; q < G; ++q) b.rep[q][lo + j] = x[u];
      }
    }
  }
  stop(t0, t);
}

template <int G>
__global__ void __launch_bounds__(256) worker_stores(Bufs b, int me, long long S, const volatile int* go,
                                                     unsigned long long* t) {
  start(go);
  const unsigned long long t0 = gtime();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < S; j += stride) {
    float4 v[G];
#pragma unroll
    for (int o = 0; o < G; ++o) v[o] = __ldcs(b.upd[me] + o * S + j);
#pragma unroll
    for (int o = 0; o < G; ++o)
      if (o != me) b.inbox[o][(long long)me * S + j] = v[o];
  }
  stop(t0, t);
}

template <int G>
__global__ void __launch_bounds__(256) owner_inbox_apply(Bufs b, int me, long long S, float lr,
                                                         const volatile int* go, unsigned long long* t) {
  start(go);
  const unsigned long long t0 = gtime();
  const long long lo = me * S, stride = (long long)gridDim.x * blockDim.x * 2;
  const float4* in = b.inbox[me];
  for (long long base = (long long)blockIdx.x * blockDim.x * 2 + threadIdx.x; base < S; base += stride) {
    float4 g[2][G], x[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long j = base + u * blockDim.x;
      if (j < S) {
#pragma unroll
        for (int i = 0; i < G; ++i) g[u][i] = __ldcs(i == me ? b.upd[me] + lo + j : in + (long long)i * S + j);
        x[u] = b.w[j];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const long long j = base + u * blockDim.x;
      if (j < S) {
#pragma unroll
        for (int i = 0; i < G; ++i) x[u] = ap(x[u], lr, g[u][i]);
        b.w[j] = x[u];
#pragma unroll
        for (int q = 0; q < G; ++q) b.rep[q][lo + j] = x[u];
      }
    }
  }
  stop(t0, t);
}

template <int G>
double run(int which, Bufs* B, long long S, int* go, int* gdev[], unsigned long long* tdev[], cudaStream_t* s) {
  double best = 1e30;
  for (int rep = 0; rep < 7; ++rep) {
    *(volatile int*)go = 0;
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      unsigned long long init[2] = {~0ull, 0ull};
      cudaMemcpy(tdev[g], init, 16, cudaMemcpyHostToDevice);
      if (which == 0) owner_loads<G><<<296, 256, 0, s[g]>>>(B[g], g, S, 0.05f, gdev[g], tdev[g]);
      if (which == 1) worker_stores<G><<<296, 256, 0, s[g]>>>(B[g], g, S, gdev[g], tdev[g]);
      if (which == 2) owner_inbox_apply<G><<<296, 256, 0, s[g]>>>(B[g], g, S, 0.05f, gdev[g], tdev[g]);
    }
    *(volatile int*)go = 1;
    unsigned long long span = 0;
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      cudaStreamSynchronize(s[g]);
      unsigned long long t[2];
      cudaMemcpy(t, tdev[g], 16, cudaMemcpyDeviceToHost);
      if (t[1] - t[0] > span) span = t[1] - t[0];
    }
    if (rep > 0 && span * 1e-3 < best) best = span * 1e-3;
  }
  return best;  // us
}

int main(int argc, char** argv) {
  int G = 0;
  cudaGetDeviceCount(&G);
  if (argc > 2) G = atoi(argv[2]) < G ? atoi(argv[2]) : G;
  if (G > kMax) G = kMax;
  if (G < 2) { printf("need >= 2 GPUs\n"); return 0; }
  const long long d = argc > 1 ? atoll(argv[1]) : 23528522ll;
  const long long S = (d / 4 + G - 1) / G;  // float4 per shard
  const long long dv = S * G;
  float4 *upd[kMax], *rep[kMax], *inbox[kMax], *w[kMax];
  cudaStream_t s[kMax];
  unsigned long long* tdev[kMax];
  int* gdev[kMax];
  int* go = nullptr;
  cudaHostAlloc((void**)&go, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable);
  for (int g = 0; g < G; ++g) {
    cudaSetDevice(g);
    for (int q = 0; q < G; ++q) if (q != g) cudaDeviceEnablePeerAccess(q, 0);
    cudaMalloc(&upd[g], dv * 16); cudaMalloc(&rep[g], dv * 16);
    cudaMalloc(&inbox[g], dv * 16); cudaMalloc(&w[g], S * 16);
    cudaMemset(upd[g], 0, dv * 16); cudaMemset(w[g], 0, S * 16);
    cudaMalloc(&tdev[g], 16);
    cudaStreamCreateWithFlags(&s[g], cudaStreamNonBlocking);
    cudaHostGetDevicePointer((void**)&gdev[g], go, 0);
    cudaDeviceSynchronize();
  }
  Bufs B[kMax];
  for (int g = 0; g < G; ++g) {
    for (int q = 0; q < G; ++q) { B[g].upd[q] = upd[q]; B[g].rep[q] = rep[q]; B[g].inbox[q] = inbox[q]; }
    B[g].w = w[g];
  }
  double a, b1, b2;
  if (G == 2) { a = run<2>(0, B, S, go, gdev, tdev, s); b1 = run<2>(1, B, S, go, gdev, tdev, s); b2 = run<2>(2, B, S, go, gdev, tdev, s); }
  else if (G <= 4) { a = run<4>(0, B, S, go, gdev, tdev, s); b1 = run<4>(1, B, S, go, gdev, tdev, s); b2 = run<4>(2, B, S, go, gdev, tdev, s); }
  else { a = run<8>(0, B, S, go, gdev, tdev, s); b1 = run<8>(1, B, S, go, gdev, tdev, s); b2 = run<8>(2, B, S, go, gdev, tdev, s); }
  const double bytes = 2.0 * (G - 1) * S * 16;  // received per GPU per step
  printf("G=%d d=%lld  A owner-loads %.1f us (%.0f GB/s received per GPU) | B worker-stores %.1f + inbox-apply %.1f = %.1f us (%.0f GB/s)\n",
         G, d, a, bytes / (a * 1e3), b1, b2, b1 + b2, bytes / ((b1 + b2) * 1e3));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
