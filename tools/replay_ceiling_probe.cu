// The data side of the C2 replay with no control at all: every warp owns a
// register-resident slice of the weights (V float4 per lane, the replay's
// layout) and runs a fixed stream of calls over it -- pulls (store the slice
// into one of 8 replica buffers) and applies (load one of 8 resident update
// slices, w = w - lr*g) -- with no numbering, no gate, no verdicts. It is the
// ceiling the replay's data warps (csrc/ps_sim.cu data_warp_replay_spec) are
// measured against: the same stores and loads on the same L2-resident working
// set, issued as fast as the SM can.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/replay_ceiling_probe tools/replay_ceiling_probe.cu
//   tools/replay_ceiling_probe [d=272474] [pulls=1004] [applies=1000]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int V>
__global__ void __launch_bounds__(256) k_stream(float4* W, float4* rep, const float4* upd, long long nv,
                                                long long dv4, int pulls, int applies, float lr, float4* sink) {
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long dw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long per = (nv + nw - 1) / nw;
  const long long lo = dw * per < nv ? dw * per : nv, hi = lo + per < nv ? lo + per : nv;
  float4 w[V];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    w[u] = j < hi ? W[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // interleave like the recorded stream: an apply, then a pull, while both last
  const int n = pulls > applies ? pulls : applies;
  for (int c = 0; c < n; ++c) {
    if (c < applies) {
      const float4* g = upd + (long long)(c & 7) * dv4;
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const long long j = lo + lane + 32ll * u;
        if (j < hi) {
          float4 x;
          asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(g + j));
          w[u].x = __fsub_rn(w[u].x, __fmul_rn(lr, x.x));
          w[u].y = __fsub_rn(w[u].y, __fmul_rn(lr, x.y));
          w[u].z = __fsub_rn(w[u].z, __fmul_rn(lr, x.z));
          w[u].w = __fsub_rn(w[u].w, __fmul_rn(lr, x.w));
        }
      }
    }
    if (c < pulls) {
      float4* dst = rep + (long long)(c & 7) * dv4;
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const long long j = lo + lane + 32ll * u;
        if (j < hi) dst[j] = w[u];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    if (j < hi) sink[j] = w[u];
  }
}

int main(int argc, char** argv) {
  const long long d = argc > 1 ? atoll(argv[1]) : 272474;
  const int pulls = argc > 2 ? atoi(argv[2]) : 1004;
  const int applies = argc > 3 ? atoi(argv[3]) : 1000;
  const long long nv = (d + 3) / 4, dv4 = nv;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float4 *W, *rep, *upd, *sink;
  CK(cudaMalloc(&W, nv * 16));
  CK(cudaMalloc(&rep, 8 * nv * 16));
  CK(cudaMalloc(&upd, 8 * nv * 16));
  CK(cudaMalloc(&sink, nv * 16));
  CK(cudaMemset(W, 0, nv * 16));
  CK(cudaMemset(upd, 0, 8 * nv * 16));
  const long long warps = (long long)sms * 8;
  const long long need_v = ((nv + warps - 1) / warps + 31) / 32;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 7; ++it) {
    CK(cudaEventRecord(e0));
    if (need_v <= 1) k_stream<1><<<sms, 256>>>(W, rep, upd, nv, dv4, pulls, applies, 0.05f, sink);
    else if (need_v <= 2) k_stream<2><<<sms, 256>>>(W, rep, upd, nv, dv4, pulls, applies, 0.05f, sink);
    else k_stream<4><<<sms, 256>>>(W, rep, upd, nv, dv4, pulls, applies, 0.05f, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best) best = ms;
  }
  const double bytes = 16.0 * nv * (pulls + applies);
  printf("d=%lld V=%lld pulls=%d applies=%d best_ms=%.4f us_per_call=%.4f l2_TBps=%.2f\n", d, need_v, pulls,
         applies, best, 1e3 * best / (pulls > applies ? pulls : applies) / ((pulls && applies) ? 2 : 1),
         bytes / (best * 1e-3) / 1e12);
  return 0;
}
