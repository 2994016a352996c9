/*
 * c_abi_client.c -- the engine driven through its C-ABI alone (no Python):
 * the calls a non-Python host (the reference's FFI, any language) makes.
 *
 *   create (ParameterServer.__init__, server.py:45-52)
 *   push   (handle_push = apply_gradient + decide_push, server.py:58-82)
 *   pull   (handle_pull, server.py:84-91)
 *
 * It checks one push + pull bit for bit against the fp32 rule
 * w - lr*g (server.py:37, rounded multiply then rounded subtract), then
 * times the per-call path at C2 size (d = 272,474) with host and device
 * buffers. Build: make -C examples (links libdssp_ps.so and cudart).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/dssp_ps.h"

static double now_us(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

#define CHECK(call)                                                                 \
  do {                                                                              \
    int rc_ = (call);                                                               \
    if (rc_ < 0) {                                                                  \
      fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, ps_last_error(h));       \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main(int argc, char** argv) {
  const int64_t d = argc > 1 ? atoll(argv[1]) : 272474;
  const int reps = argc > 2 ? atoi(argv[2]) : 400;
  ps_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.paradigm = PS_ASP;
  cfg.worker_count = 4;
  cfg.learning_rate = 0.05;
  cfg.dimension = d;
  cfg.device = 0;
  float* w0 = (float*)malloc(d * sizeof(float));
  float* g = NULL;
  float* out = NULL;
  cudaMallocHost((void**)&g, d * sizeof(float));
  cudaMallocHost((void**)&out, d * sizeof(float));
  for (int64_t i = 0; i < d; ++i) {
    w0[i] = (float)((i % 1000) * 1e-3 - 0.5);
    g[i] = (float)(((i * 7919) % 2001) * 1e-3 - 1.0);
  }
  ps_server* h = NULL;
  if (ps_create(&cfg, w0, PS_F32, &h) != PS_OK) {
    fprintf(stderr, "ps_create: %s\n", ps_last_error(NULL));
    return 1;
  }
  int32_t applied = 0, granted = 0;
  uint64_t released = 0;
  int64_t version = 0;
  CHECK(ps_push(h, 0, g, PS_F32, 0, 1.0, &applied, &granted, &released));
  CHECK(ps_pull(h, 0, out, PS_F32, 0, &version));
  const float lr = (float)cfg.learning_rate;
  int64_t bad = 0;
  for (int64_t i = 0; i < d; ++i) {
    volatile float prod = lr * g[i];  /* rounded multiply ... */
    const float want = w0[i] - prod;  /* ... then rounded subtract */
    if (memcmp(&want, &out[i], 4) != 0) ++bad;
  }
  printf("c_abi_client: d=%lld push+pull %s (applied=%d granted=%d version=%lld)\n", (long long)d,
         bad ? "MISMATCH" : "bit-exact", applied, granted, (long long)version);
  if (bad) return 1;
  float *gd = NULL, *outd = NULL;
  cudaMalloc((void**)&gd, d * sizeof(float));
  cudaMalloc((void**)&outd, d * sizeof(float));
  cudaMemcpy(gd, g, d * sizeof(float), cudaMemcpyHostToDevice);
  double* t = (double*)malloc(reps * sizeof(double));
  const char* names[4] = {"push (device g)", "pull (device dst)", "push (pinned host g)", "pull (pinned host dst)"};
  for (int kind = 0; kind < 4; ++kind) {
    for (int r = 0; r < reps + 20; ++r) {
      const double t0 = now_us();
      if (kind == 0) CHECK(ps_push(h, r % 4, gd, PS_F32, 1, 2.0 + r, &applied, &granted, &released));
      if (kind == 1) CHECK(ps_pull(h, r % 4, outd, PS_F32, 1, &version));
      if (kind == 2) CHECK(ps_push(h, r % 4, g, PS_F32, 0, 2.0 + r, &applied, &granted, &released));
      if (kind == 3) CHECK(ps_pull(h, r % 4, out, PS_F32, 0, &version));
      if (r >= 20) t[r - 20] = now_us() - t0;
    }
    qsort(t, reps, sizeof(double), cmp_double);
    printf("  %-24s median %7.2f us  p90 %7.2f us\n", names[kind], t[reps / 2], t[reps * 9 / 10]);
  }
  ps_destroy(h);
  return 0;
}
