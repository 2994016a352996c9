// ps_server.cu -- single-GPU parameter server: push-apply, pull and the device
// gate behind the C-ABI of include/dssp_ps.h.
//
// Push-apply (server.py:29-69). The weights are double buffered: one pass
// reads w[cur] and the update, writes w[cur^1] (12 B/parameter: read w, read g,
// write w) and ORs two flags per CTA -- non-finite gradient, non-finite result.
// The last CTA to finish (threadfence-reduction election) publishes the
// outcome: a clean pass flips `cur` and bumps the version; a non-finite
// gradient is rejected and counted (server.py:65-67) and a non-finite result
// is a DivergenceError (server.py:38-41) -- in both cases w[cur] was never
// touched, so the reference's "weights unchanged" semantics hold exactly with
// a single streaming pass and no grid barrier. In the fused push
// (handle_push, server.py:80-82) the same last CTA then runs the gate
// decision, so apply + clock increment + decision is one launch.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>

#include "common.cuh"
#include "gate.cuh"
#include "server.h"

using namespace dssp;

static thread_local std::string g_create_error;

int ps_fail(ps_server* h, int code, const std::string& msg) {
  if (h) h->err = msg; else g_create_error = msg;
  return code;
}

int ps_cuda_fail(ps_server* h, cudaError_t e, const char* what) {
  std::string m = std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what;
  return ps_fail(h, PS_E_CUDA, m);
}

namespace {

constexpr int kApplyThreads = 256;
constexpr int kApplyUnroll = 4;

template <typename G>
struct Vec4Load;
template <>
struct Vec4Load<float> {
  static __device__ __forceinline__ float4 load(const float* g, long long j) {
    return ld_stream(reinterpret_cast<const float4*>(g) + j);
  }
  static __device__ __forceinline__ float one(const float* g, long long i) { return g[i]; }
};
template <>
struct Vec4Load<double> {
  static __device__ __forceinline__ float4 load(const double* g, long long j) {
    const double2* p = reinterpret_cast<const double2*>(g) + 2 * j;
    double2 a = p[0], b = p[1];
    return make_float4((float)a.x, (float)a.y, (float)b.x, (float)b.y);
  }
  static __device__ __forceinline__ float one(const double* g, long long i) { return (float)g[i]; }
};

// Warp-collective copy of the control block into the host-mapped mirror, so
// the host reads every op's result and the gate tables without a D2H copy.
// Only the live part crosses PCIe: the header, the first P entries of each
// 64-slot gate table, the gate counters and the op result (3 + 5P + 8 words).
// An apply alone changes none of the tables: then only the counters and the
// result cross PCIe (8 words).
__device__ __forceinline__ void publish_ctrl(const Ctrl* ctrl, Ctrl* mirror, bool tables = true) {
  static_assert(sizeof(ps_gate_state) == 8 * (3 + 5 * PS_MAX_WORKERS + 4), "gate layout");
  static_assert(sizeof(Ctrl) == sizeof(ps_gate_state) + 32, "ctrl layout");
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(ctrl);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(mirror);
  const int P = tables ? ctrl->gate.worker_count : 0;
  const int n = 3 + 5 * P + 8;
  for (int i = (threadIdx.x & 31) + (tables ? 0 : 3); i < n; i += 32) {
    int word;
    if (i < 3) word = i;                                              // header
    else if (i < 3 + 5 * P) word = 3 + ((i - 3) / P) * PS_MAX_WORKERS + (i - 3) % P;  // tables
    else word = 3 + 5 * PS_MAX_WORKERS + (i - 3 - 5 * P);             // counters + result
    d[word] = s[word];
  }
}

// One streaming pass w[cur^1] = w[cur] - lr*g with flag reduction; the last CTA
// publishes the result and (fuse=1) runs the gate decision. g may live in
// device memory or in pinned host memory (read over PCIe, zero-copy).
template <typename G, int kApplyUnroll>
__global__ void __launch_bounds__(kApplyThreads)
k_apply(float* __restrict__ w0, float* __restrict__ w1, const G* __restrict__ g, long long n,
        float lr, Ctrl* ctrl, int cur, int fuse, int worker, double now, Ctrl* mirror) {
  // cur comes from the host (h->cur, refreshed after every op's sync -- the
  // same value pulls read from): no dependent load ahead of the data loads
  const float4* src = reinterpret_cast<const float4*>(cur ? w1 : w0);
  float4* dst = reinterpret_cast<float4*>(cur ? w0 : w1);
  const long long nv = n >> 2;
  unsigned bad = 0;
  const long long step = (long long)gridDim.x * kApplyThreads * kApplyUnroll;
  for (long long base = (long long)blockIdx.x * kApplyThreads * kApplyUnroll + threadIdx.x; base < nv;
       base += step) {
    float4 a[kApplyUnroll], b[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      const long long j = base + (long long)u * kApplyThreads;
      if (j < nv) {
        a[u] = src[j];
        b[u] = Vec4Load<G>::load(g, j);
      }
    }
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      const long long j = base + (long long)u * kApplyThreads;
      if (j < nv) {
        const float4 r = apply4(a[u], lr, b[u]);
        bad |= nonfinite4(b[u]) ? 1u : 0u;
        bad |= nonfinite4(r) ? 2u : 0u;
        dst[j] = r;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {  // ragged tail
    const long long i = (nv << 2) + threadIdx.x;
    const float* s = cur ? w1 : w0;
    float* o = cur ? w0 : w1;
    const float gi = Vec4Load<G>::one(g, i);
    const float r = apply1(s[i], lr, gi);
    bad |= nonfinite(gi) ? 1u : 0u;
    bad |= nonfinite(r) ? 2u : 0u;
    o[i] = r;
  }
  bad = __reduce_or_sync(kFull, bad);
  __shared__ unsigned s_bad;
  __shared__ int s_last;
  __shared__ unsigned s_flags;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(&s_bad, bad);
  __syncthreads();
  if (threadIdx.x == 0) {
    // one 64-bit GPU-scope acq_rel arrival on the (arrive, bad) pair: the low
    // word counts CTAs, the high word counts CTAs that saw a non-finite
    // update (bits 0-15) or result (bits 16-31), so the last arriver holds
    // every CTA's verdict without a second atomic
    static_assert(offsetof(Ctrl, bad) == offsetof(Ctrl, arrive) + 4 && offsetof(Ctrl, arrive) % 8 == 0,
                  "arrive/bad pair");
    const unsigned long long add =
        1ull | ((unsigned long long)((s_bad & 1u) | ((s_bad & 2u) << 15)) << 32);
    const unsigned long long prev =
        atom_add_acq_rel_gpu_u64(reinterpret_cast<unsigned long long*>(&ctrl->arrive), add);
    s_last = ((unsigned)prev == gridDim.x - 1);
    s_flags = (unsigned)((prev + add) >> 32);
  }
  __syncthreads();
  if (!s_last || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int status = PS_OK;
  if (lane == 0) {
    const unsigned b = s_flags;
    int applied = 0;
    if (b & 0xffffu) {
      status = PS_REJECTED;
      ctrl->gate.rejected += 1;
    } else if (b >> 16) {
      status = PS_E_DIVERGED;
    } else {
      ctrl->cur = cur ^ 1;
      ctrl->gate.version += 1;
      applied = 1;
    }
    ctrl->arrive = 0;
    ctrl->bad = 0;
    ctrl->status = status;
    ctrl->applied = applied;
    ctrl->granted = 0;
    ctrl->released = 0;
  }
  status = __shfl_sync(kFull, status, 0);
  if (fuse && status != PS_E_DIVERGED) {
    const GateResult r = gate_on_push(&ctrl->gate, worker, now);
    if (lane == 0) {
      if (r.status != PS_OK) ctrl->status = r.status;
      ctrl->granted = (r.status == PS_OK && r.outcome == 0) ? 1 : 0;
      ctrl->released = r.released;
    }
  }
  __syncwarp();
  publish_ctrl(ctrl, mirror, fuse != 0);
}

__global__ void k_decide(Ctrl* ctrl, int worker, double now, Ctrl* mirror) {
  const GateResult r = gate_on_push(&ctrl->gate, worker, now);
  if (threadIdx.x == 0) {
    ctrl->status = r.status;
    ctrl->granted = (r.status == PS_OK && r.outcome == 0) ? 1 : 0;
    ctrl->released = r.released;
  }
  __syncwarp();
  publish_ctrl(ctrl, mirror);
}

template <typename T>
__global__ void __launch_bounds__(256) k_copy_out(const float* __restrict__ src, T* __restrict__ dst,
                                                  long long n) {
  // kApplyUnroll float4 per thread per trip, all loads issued before the
  // stores: enough bytes in flight per SM to cover HBM latency
  constexpr int U = kApplyUnroll;
  const long long nv = n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x * U;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  for (long long base = (long long)blockIdx.x * blockDim.x * U + threadIdx.x; base < nv; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * blockDim.x;
      if (j < nv) v[u] = ld_stream(s4 + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * blockDim.x;
      if (j < nv) {
        if constexpr (sizeof(T) == 4) {
          reinterpret_cast<float4*>(dst)[j] = v[u];
        } else {
          double2* o = reinterpret_cast<double2*>(dst) + 2 * j;
          o[0] = make_double2(v[u].x, v[u].y);
          o[1] = make_double2(v[u].z, v[u].w);
        }
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const long long i = (nv << 2) + threadIdx.x;
    dst[i] = (T)src[i];
  }
}

template <typename T>
__global__ void k_load_in(const T* __restrict__ src, float* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (float)src[i];
}

// apply_update on plain vectors (ps_apply_vectors): out = w - lr*g, any
// non-finite result raises the flag word.
__global__ void k_apply_vec(const float* __restrict__ w, const float* __restrict__ g,
                            float* __restrict__ out, long long n, float lr, unsigned* flag) {
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float r = apply1(w[i], lr, g[i]);
    bad |= nonfinite(r);
    out[i] = r;
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void k_controller_batch(const double* tables, const int* r_max, int n, int* out) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (row >= n) return;  // warp-uniform
  const double* t = tables + 4 * (long long)row;
  const int rm = r_max[row];
  const int r = rm <= 0 ? 0 : controller_grid(t[0], t[1], t[2], t[3], rm);
  if ((threadIdx.x & 31) == 0) out[row] = r;
}

constexpr unsigned long long kProfileSpinNs = 50000;

__global__ void k_spin(unsigned long long ns) {
  const unsigned long long t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) {
  }
}

int grid_for(const ps_server* h, long long nv, int unroll = kApplyUnroll) {
  long long per_block = (long long)kApplyThreads * unroll;
  long long blocks = (nv + per_block - 1) / per_block;
  long long cap = (long long)h->sm_count * 8;
  if (blocks < 1) blocks = 1;
  if (blocks > cap) blocks = cap;
  return (int)blocks;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

int ensure_stage(ps_server* h, size_t bytes) {
  if (h->stage_bytes >= bytes) return PS_OK;
  if (h->stage) cudaFree(h->stage);
  if (h->hstage) cudaFreeHost(h->hstage);
  h->stage = nullptr;
  h->hstage = nullptr;
  h->stage_bytes = 0;
  PS_CK(h, cudaMalloc(&h->stage, bytes));
  PS_CK(h, cudaMallocHost(&h->hstage, bytes));
  h->stage_bytes = bytes;
  return PS_OK;
}

// Full D2H refresh of the mirror (after launches that do not publish it).
int sync_ctrl(ps_server* h) {
  PS_CK(h, cudaMemcpyAsync(h->hctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  h->cur = h->hctrl->cur;
  return PS_OK;
}

// Wait for an op whose kernel published the mirror itself.
int finish_op(ps_server* h) {
  PS_CK(h, cudaStreamSynchronize(h->stream));
  h->cur = h->hctrl->cur;
  if (h->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    h->last_ms = ms;
  }
  return PS_OK;
}

int mark(ps_server* h, cudaEvent_t e) {
  if (!h->profile) return PS_OK;
  // the start event goes in behind a short device spin: the op's launches
  // are then queued before the GPU reaches it, so ev0..ev1 is device time
  // only, not the host's submit gap on an idle stream
  if (e == h->ev0) {
    k_spin<<<1, 32, 0, h->stream>>>(kProfileSpinNs);
    PS_CK(h, cudaGetLastError());
  }
  PS_CK(h, cudaEventRecord(e, h->stream));
  return PS_OK;
}

// Stream-order the server after the caller's producer stream (e.g. the
// PyTorch stream whose backward wrote the update, or that will read a pull):
// an event edge, no host synchronization.
int after_producer(ps_server* h) {
  if (!h->producer) return PS_OK;
  if (!h->ev_in) PS_CK(h, cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming));
  PS_CK(h, cudaEventRecord(h->ev_in, h->producer));
  PS_CK(h, cudaStreamWaitEvent(h->stream, h->ev_in, 0));
  return PS_OK;
}

// Host transfers through the copy engines instead of zero-copy kernel access
// (PS_HOST_DMA=1; an A/B switch for the e2e path).
bool host_dma() {
  static const bool on = [] {
    const char* v = getenv("PS_HOST_DMA");
    return v && v[0] == '1';
  }();
  return on;
}

// float4 per thread per trip of the apply on small vectors (PS_APPLY_SMALL_U,
// an A/B knob; the large-vector path keeps kApplyUnroll)
int apply_small_unroll() {
  static const int u = [] {
    const char* v = getenv("PS_APPLY_SMALL_U");
    const int x = v ? atoi(v) : 2;
    return (x == 1 || x == 2 || x == 4) ? x : 2;
  }();
  return u;
}

// Pinned (page-locked, UVA-mapped) host memory can be read and written by
// kernels directly over PCIe; pageable memory has to be staged.
bool pinned_host(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
  ~DevGuard() { cudaSetDevice(prev); }
};

// Launch the apply (optionally fused with the decision) on a device- or host-
// resident update: device or pinned host memory is read in place (the kernel
// streams a pinned host update over PCIe, no separate copy); pageable host
// memory and misaligned device views go through staging.
int res_push(ps_server* h, int worker, const void* g, int g_dtype, int g_on_device, int fuse, double now);
bool res_active(const ps_server* h);

int launch_apply(ps_server* h, int worker, const void* g, int g_dtype, int g_on_device, int fuse,
                 double now) {
  if (res_active(h)) return res_push(h, worker, g, g_dtype, g_on_device, fuse, now);
  if (g_dtype != PS_F32 && g_dtype != PS_F64) return ps_fail(h, PS_E_VALUE, "bad gradient dtype");
  if (!g) return ps_fail(h, PS_E_VALUE, "null gradient");
  const size_t esz = g_dtype == PS_F64 ? 8 : 4;
  const size_t bytes = (size_t)h->d * esz;
  const void* dg = g;
  int rc = after_producer(h);
  if (rc) return rc;
  const bool direct = aligned16(g) && (g_on_device || (!host_dma() && pinned_host(g)));
  if (!direct) {
    if ((rc = ensure_stage(h, bytes))) return rc;
    PS_CK(h, cudaMemcpyAsync(h->stage, g, bytes, g_on_device ? cudaMemcpyDeviceToDevice
                                                               : cudaMemcpyHostToDevice, h->stream));
    dg = h->stage;
  }
  const float lr = (float)h->cfg.learning_rate;
  const int grid = grid_for(h, h->nv);
  if ((rc = mark(h, h->ev0))) return rc;
  // small vectors: one float4 per thread per trip over more CTAs (the op is
  // latency-bound there: spread it over every SM); large ones: four in flight
  const int small_u = apply_small_unroll();
  const bool small = h->nv <= (long long)h->sm_count * kApplyThreads * 8;
  const int U = small ? small_u : kApplyUnroll;
  const int grid2 = grid_for(h, h->nv, U);
  (void)grid;
#define PS_LAUNCH_APPLY(T, UU)                                                                      \
  k_apply<T, UU><<<grid2, kApplyThreads, 0, h->stream>>>(h->w[0], h->w[1], (const T*)dg, h->d, lr, \
                                                        h->ctrl, h->cur, fuse, worker, now, h->hctrl_dev)
  if (g_dtype == PS_F32) {
    if (U == 1) PS_LAUNCH_APPLY(float, 1); else if (U == 2) PS_LAUNCH_APPLY(float, 2); else PS_LAUNCH_APPLY(float, 4);
  } else {
    if (U == 1) PS_LAUNCH_APPLY(double, 1); else if (U == 2) PS_LAUNCH_APPLY(double, 2); else PS_LAUNCH_APPLY(double, 4);
  }
#undef PS_LAUNCH_APPLY
  PS_CK(h, cudaGetLastError());
  if ((rc = mark(h, h->ev1))) return rc;
  return finish_op(h);
}

// ---------------------------------------------------------------------------
// Resident mode (ps_set_resident): the per-call API without a launch or a
// stream synchronization per call. A persistent kernel of a few CTAs stays on
// the GPU; the host posts each reference call (apply_gradient, decide_push,
// handle_push, handle_pull -- server.py:58-91) into a pinned, mapped mailbox
// and spins on the response the kernel writes back into host memory. CTA 0
// polls the mailbox over PCIe and forwards the request to the other CTAs
// through device memory; the last CTA to finish an op commits it (verdict,
// buffer flip, version, gate decision) exactly like k_apply's last CTA and
// answers. Weights, gate tables and the cur index are read at L2 (ld.cg):
// across requests another SM may have written them, and no kernel boundary
// invalidates L1. An idle kernel retires itself after ~2 s (mbox.alive = 0)
// and the next call relaunches it, so nothing spins on a GPU forever.
// ---------------------------------------------------------------------------
enum { RES_STOP = 0, RES_APPLY = 1, RES_PUSH = 2, RES_DECIDE = 3, RES_PULL = 4 };

struct ResReq {
  int32_t op, worker;
  double now;
  const void* src;       // APPLY / PUSH: the update
  void* dst;             // PULL: the destination
  int32_t dtype;         // of src (APPLY / PUSH) or dst (PULL)
  int32_t host_mem;      // 1: src / dst is pinned host memory
};

struct ResResp {
  int32_t status, applied, granted, cur;
  uint64_t released;
  int64_t version;
};

struct ResMbox {                       // pinned host memory, mapped for the device
  volatile unsigned long long req_seq;
  unsigned long long _p0[7];
  ResReq req;
  unsigned long long _p1[4];
  volatile unsigned long long resp_seq;
  volatile int32_t alive;              // the kernel is serving (0: retired / retiring)
  int32_t _p2;
  unsigned long long _p3[6];
  ResResp resp;
};

struct ResDev {                        // device memory
  unsigned long long dseq;             // the request CTA 0 forwarded last
  unsigned long long _p0[7];
  ResReq req;
  unsigned long long arrive;           // low: CTAs done, high: non-finite flag counts
};

struct ResArgs {
  float* w0;
  float* w1;
  long long n, nv;
  float lr;
  Ctrl* ctrl;
  Ctrl* mirror;
  ResMbox* mbox;                       // device alias of the host mailbox
  ResDev* rd;
  unsigned long long seq0;             // first request sequence number to serve
  unsigned long long idle_ns;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys_u64_v(const volatile unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <typename G>
__device__ __forceinline__ float4 res_load_g(const G* g, long long j, bool host);
template <>
__device__ __forceinline__ float4 res_load_g<float>(const float* g, long long j, bool host) {
  const float4* p = reinterpret_cast<const float4*>(g) + j;
  return host ? __ldcv(p) : __ldcg(p);
}
template <>
__device__ __forceinline__ float4 res_load_g<double>(const double* g, long long j, bool host) {
  const double2* p = reinterpret_cast<const double2*>(g) + 2 * j;
  const double2 a = host ? __ldcv(p) : __ldcg(p), b = host ? __ldcv(p + 1) : __ldcg(p + 1);
  return make_float4((float)a.x, (float)a.y, (float)b.x, (float)b.y);
}

template <typename G>
__device__ unsigned res_apply(const ResArgs& a, int cur, const G* g, bool host) {
  const float4* src = reinterpret_cast<const float4*>(cur ? a.w1 : a.w0);
  float4* dst = reinterpret_cast<float4*>(cur ? a.w0 : a.w1);
  unsigned bad = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < a.nv; j += stride) {
    const float4 gv = res_load_g<G>(g, j, host);
    const float4 r = apply4(__ldcg(src + j), a.lr, gv);
    bad |= nonfinite4(gv) ? 1u : 0u;
    bad |= nonfinite4(r) ? 2u : 0u;
    __stcg(dst + j, r);
  }
  if (blockIdx.x == 0 && threadIdx.x < (a.n & 3)) {
    const long long i = (a.nv << 2) + threadIdx.x;
    const float* sw = cur ? a.w1 : a.w0;
    float* dw = cur ? a.w0 : a.w1;
    const float gi = host ? (float)*(const volatile G*)(g + i) : (float)__ldcg(g + i);
    const float r = apply1(__ldcg(sw + i), a.lr, gi);
    bad |= nonfinite(gi) ? 1u : 0u;
    bad |= nonfinite(r) ? 2u : 0u;
    __stcg(dw + i, r);
  }
  return bad;
}

template <typename T>
__device__ void res_pull(const ResArgs& a, int cur, T* dst) {
  const float4* src = reinterpret_cast<const float4*>(cur ? a.w1 : a.w0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < a.nv; j += stride) {
    const float4 v = __ldcg(src + j);
    if constexpr (sizeof(T) == 4) {
      reinterpret_cast<float4*>(dst)[j] = v;
    } else {
      double2* o = reinterpret_cast<double2*>(dst) + 2 * j;
      o[0] = make_double2(v.x, v.y);
      o[1] = make_double2(v.z, v.w);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (a.n & 3)) {
    const long long i = (a.nv << 2) + threadIdx.x;
    dst[i] = (T)__ldcg((cur ? a.w1 : a.w0) + i);
  }
}

// Warp 0 of the committing CTA: the gate decision on an L2-fresh copy of the
// tables in shared memory, written back at L2.
// Only the live words move: the header, the first P entries of each table and
// the counters (as publish_ctrl).
__device__ __forceinline__ int live_word(int i, int P) {
  if (i < 3) return i;
  if (i < 3 + 5 * P) return 3 + ((i - 3) / P) * PS_MAX_WORKERS + (i - 3) % P;
  return 3 + 5 * PS_MAX_WORKERS + (i - 3 - 5 * P);
}

__device__ GateResult res_gate(const ResArgs& a, int worker, double now, ps_gate_state* sg) {
  const int lane = threadIdx.x & 31;
  unsigned long long* s8 = reinterpret_cast<unsigned long long*>(sg);
  unsigned long long* g8 = reinterpret_cast<unsigned long long*>(&a.ctrl->gate);
  const int P = __ldcg(&a.ctrl->gate.worker_count);
  const int n = 3 + 5 * P + 4;  // header, tables, deferred / version / rejected / decisions
  for (int i = lane; i < n; i += 32) { const int w = live_word(i, P); s8[w] = __ldcg(g8 + w); }
  __syncwarp();
  const GateResult r = gate_on_push(sg, worker, now);
  __syncwarp();
  for (int i = lane; i < n; i += 32) { const int w = live_word(i, P); __stcg(g8 + w, s8[w]); }
  __syncwarp();
  return r;
}

// Warp-collective: the live part of the control block into the host mirror
// (as publish_ctrl, reading at L2).
__device__ void res_publish(const ResArgs& a) {
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(a.ctrl);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(a.mirror);
  const int P = __ldcg(&a.ctrl->gate.worker_count);
  const int n = 3 + 5 * P + 8;
  for (int i = threadIdx.x & 31; i < n; i += 32) {
    int word;
    if (i < 3) word = i;
    else if (i < 3 + 5 * P) word = 3 + ((i - 3) / P) * PS_MAX_WORKERS + (i - 3) % P;
    else word = 3 + 5 * PS_MAX_WORKERS + (i - 3 - 5 * P);
    d[word] = __ldcg(s + word);
  }
}

__device__ void res_respond(const ResArgs& a, unsigned long long seq, int status, int applied, int granted,
                            unsigned long long released) {
  // lane 0 of the committing warp
  ResMbox* m = a.mbox;
  m->resp.status = status;
  m->resp.applied = applied;
  m->resp.granted = granted;
  m->resp.cur = __ldcg(&a.ctrl->cur);
  m->resp.released = released;
  m->resp.version = __ldcg(&a.ctrl->gate.version);
  __threadfence_system();
  m->resp_seq = seq;
}

__global__ void __launch_bounds__(256) k_resident(ResArgs a) {
  __shared__ ResReq s_req;
  __shared__ int s_last;
  __shared__ unsigned s_flags, s_bad;
  __shared__ ps_gate_state sg;
  unsigned long long seq = a.seq0;
  const int lane = threadIdx.x & 31;
  for (;; ++seq) {
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        unsigned long long t0 = globaltimer_ns();
        unsigned backoff = 32;
        bool got = false;
        for (;;) {
          if (ld_acquire_sys_u64_v(&a.mbox->req_seq) == seq) { got = true; break; }
          if (globaltimer_ns() - t0 > a.idle_ns) {
            // retire: announce it, then look once more (a request posted
            // before the host saw alive = 0 is still served)
            a.mbox->alive = 0;
            __threadfence_system();
            if (ld_acquire_sys_u64_v(&a.mbox->req_seq) == seq) { a.mbox->alive = 1; got = true; }
            break;
          }
          __nanosleep(backoff);
          backoff = backoff < 256 ? backoff * 2 : 256;
        }
        ResReq r{};
        r.op = RES_STOP;
        if (got) {
          r.op = *(volatile int32_t*)&a.mbox->req.op;
          r.worker = *(volatile int32_t*)&a.mbox->req.worker;
          r.now = *(volatile double*)&a.mbox->req.now;
          r.src = *(const void* volatile*)&a.mbox->req.src;
          r.dst = *(void* volatile*)&a.mbox->req.dst;
          r.dtype = *(volatile int32_t*)&a.mbox->req.dtype;
          r.host_mem = *(volatile int32_t*)&a.mbox->req.host_mem;
        }
        a.rd->req = r;
        __threadfence();
        st_release_u64(&a.rd->dseq, seq);
      } else {
        unsigned backoff = 32;
        while (ld_acquire_u64(&a.rd->dseq) != seq) {
          __nanosleep(backoff);
          backoff = backoff < 512 ? backoff * 2 : 512;
        }
      }
      ResReq r;
      r.op = __ldcg(&a.rd->req.op);
      r.worker = __ldcg(&a.rd->req.worker);
      r.now = __ldcg(&a.rd->req.now);
      r.src = (const void*)__ldcg((const unsigned long long*)&a.rd->req.src);
      r.dst = (void*)__ldcg((const unsigned long long*)&a.rd->req.dst);
      r.dtype = __ldcg(&a.rd->req.dtype);
      r.host_mem = __ldcg(&a.rd->req.host_mem);
      s_req = r;
      s_bad = 0;
    }
    __syncthreads();
    const ResReq r = s_req;
    if (r.op == RES_STOP) return;
    if (r.op == RES_DECIDE) {
      if (blockIdx.x == 0 && threadIdx.x < 32) {
        const GateResult g = res_gate(a, r.worker, r.now, &sg);
        if (lane == 0) {
          __stcg(&a.ctrl->status, g.status);
          __stcg(&a.ctrl->granted, (g.status == PS_OK && g.outcome == 0) ? 1 : 0);
          __stcg((unsigned long long*)&a.ctrl->released, g.released);
        }
        __syncwarp();
        res_publish(a);
        __syncwarp();
        if (lane == 0) res_respond(a, seq, g.status, 0, (g.status == PS_OK && g.outcome == 0) ? 1 : 0, g.released);
      }
      continue;
    }
    const int cur = __ldcg(&a.ctrl->cur);
    unsigned bad = 0;
    if (r.op == RES_APPLY || r.op == RES_PUSH) {
      bad = r.dtype == PS_F64 ? res_apply<double>(a, cur, (const double*)r.src, r.host_mem != 0)
                              : res_apply<float>(a, cur, (const float*)r.src, r.host_mem != 0);
    } else {  // RES_PULL
      if (r.dtype == PS_F64) res_pull<double>(a, cur, (double*)r.dst);
      else res_pull<float>(a, cur, (float*)r.dst);
    }
    bad = __reduce_or_sync(kFull, bad);
    if (lane == 0 && bad) atomicOr(&s_bad, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (r.host_mem && r.op == RES_PULL) __threadfence_system();  // host stores before the answer
      const unsigned long long add =
          1ull | ((unsigned long long)((s_bad & 1u) | ((s_bad & 2u) << 15)) << 32);
      const unsigned long long prev = atom_add_acq_rel_gpu_u64(&a.rd->arrive, add);
      s_last = ((unsigned)prev == gridDim.x - 1);
      s_flags = (unsigned)((prev + add) >> 32);
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) continue;
    // the committing CTA (every CTA's writes acquired through the arrival)
    int status = PS_OK, applied = 0, granted = 0;
    unsigned long long released = 0;
    if (lane == 0) a.rd->arrive = 0;  // nobody arrives again before the answer
    if (r.op == RES_PULL) {
      if (lane == 0) {
        __threadfence_system();
        res_respond(a, seq, PS_OK, 0, 0, 0);
      }
      continue;
    }
    if (lane == 0) {
      const unsigned f = s_flags;
      if (f & 0xffffu) {
        status = PS_REJECTED;
        __stcg(&a.ctrl->gate.rejected, __ldcg(&a.ctrl->gate.rejected) + 1);
      } else if (f >> 16) {
        status = PS_E_DIVERGED;
      } else {
        __stcg(&a.ctrl->cur, cur ^ 1);
        __stcg(&a.ctrl->gate.version, __ldcg(&a.ctrl->gate.version) + 1);
        applied = 1;
      }
    }
    status = __shfl_sync(kFull, status, 0);
    applied = __shfl_sync(kFull, applied, 0);
    if (r.op == RES_PUSH && status != PS_E_DIVERGED) {
      __threadfence();
      const GateResult g = res_gate(a, r.worker, r.now, &sg);
      if (g.status != PS_OK) status = g.status;
      granted = (g.status == PS_OK && g.outcome == 0) ? 1 : 0;
      released = g.released;
    }
    if (lane == 0) {
      __stcg(&a.ctrl->status, status);
      __stcg(&a.ctrl->applied, applied);
      __stcg(&a.ctrl->granted, granted);
      __stcg((unsigned long long*)&a.ctrl->released, released);
    }
    __syncwarp();
    res_publish(a);
    __syncwarp();
    if (lane == 0) res_respond(a, seq, status, applied, granted, released);
  }
}

}  // namespace

int ps_order_after_producer(ps_server* h) { return after_producer(h); }

struct ps_resident {
  int ctas = 0;                 // 0: resident mode off
  bool running = false;
  cudaStream_t stream = nullptr;
  ResMbox* mbox = nullptr;      // pinned host mailbox
  ResMbox* mbox_dev = nullptr;  // its device alias
  ResDev* rd = nullptr;
  unsigned long long seq = 1;   // the next request's sequence number
  cudaEvent_t ev = nullptr;
};

namespace {

constexpr unsigned long long kResidentIdleNs = 2ull * 1000 * 1000 * 1000;

int res_launch(ps_server* h) {
  ps_resident* r = h->res;
  r->mbox->alive = 1;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  ResArgs a{};
  a.w0 = h->w[0];
  a.w1 = h->w[1];
  a.n = h->d;
  a.nv = h->d >> 2;  // whole float4s; the n & 3 tail is element-wise
  a.lr = (float)h->cfg.learning_rate;
  a.ctrl = h->ctrl;
  a.mirror = h->hctrl_dev;
  a.mbox = r->mbox_dev;
  a.rd = r->rd;
  a.seq0 = r->seq;
  a.idle_ns = kResidentIdleNs;
  // every earlier use of the server's state (on its own stream) is complete
  PS_CK(h, cudaStreamSynchronize(h->stream));
  k_resident<<<r->ctas, 256, 0, r->stream>>>(a);
  PS_CK(h, cudaGetLastError());
  r->running = true;
  return PS_OK;
}

bool res_retired(ps_resident* r) {
  return r->mbox->alive == 0 && cudaStreamQuery(r->stream) == cudaSuccess;
}

// Post one request and spin on the answer in host memory.
int res_call(ps_server* h, const ResReq& q, ResResp* out) {
  ps_resident* r = h->res;
  int rc;
  if (!r->running || res_retired(r)) {
    if (r->running) PS_CK(h, cudaStreamSynchronize(r->stream));
    if ((rc = res_launch(h))) return rc;
  }
  const unsigned long long seq = r->seq;
  std::memcpy((void*)&r->mbox->req, &q, sizeof(q));
  std::atomic_thread_fence(std::memory_order_seq_cst);
  r->mbox->req_seq = seq;
  const auto t0 = std::chrono::steady_clock::now();
  unsigned long long spins = 0;
  while (r->mbox->resp_seq != seq) {
    if ((++spins & 4095) == 0) {
      const cudaError_t e = cudaStreamQuery(r->stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return ps_cuda_fail(h, e, "resident server");
      if (e == cudaSuccess && r->mbox->resp_seq != seq) {
        // retired before it saw the request: relaunch, it picks it up
        if ((rc = res_launch(h))) return rc;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
        return ps_fail(h, PS_E_TIMEOUT, "resident server did not answer within 30 s");
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  std::memcpy(out, (const void*)&r->mbox->resp, sizeof(*out));
  r->seq = seq + 1;
  h->cur = out->cur;
  return PS_OK;
}

// Device tensors come from the caller's producer stream: with no kernel
// launch to carry an event edge, the host waits for that stream's work.
int res_after_producer(ps_server* h) {
  if (!h->producer) return PS_OK;
  ps_resident* r = h->res;
  if (!r->ev) PS_CK(h, cudaEventCreateWithFlags(&r->ev, cudaEventDisableTiming));
  PS_CK(h, cudaEventRecord(r->ev, h->producer));
  PS_CK(h, cudaEventSynchronize(r->ev));
  return PS_OK;
}

// Update operand for a resident push: device or pinned host memory in place,
// anything else staged on the server stream first.
int res_operand(ps_server* h, const void* g, int g_dtype, int g_on_device, ResReq* q) {
  if (g_dtype != PS_F32 && g_dtype != PS_F64) return ps_fail(h, PS_E_VALUE, "bad gradient dtype");
  if (!g) return ps_fail(h, PS_E_VALUE, "null gradient");
  const size_t bytes = (size_t)h->d * (g_dtype == PS_F64 ? 8 : 4);
  int rc;
  q->dtype = g_dtype;
  if (aligned16(g) && g_on_device) {
    if ((rc = res_after_producer(h))) return rc;
    q->src = g;
    q->host_mem = 0;
  } else {
    // host memory (pinned or not): the copy engine into the stage -- a few
    // resident CTAs reading pinned memory over PCIe are slower than the DMA
    if (g_on_device && (rc = res_after_producer(h))) return rc;
    if ((rc = ensure_stage(h, bytes))) return rc;
    PS_CK(h, cudaMemcpyAsync(h->stage, g, bytes, g_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             h->stream));
    PS_CK(h, cudaStreamSynchronize(h->stream));
    q->src = h->stage;
    q->host_mem = 0;
  }
  return PS_OK;
}

bool res_active(const ps_server* h) { return h->res && h->res->ctas > 0; }

// The kernel published the op's result and the gate tables into the host
// mirror before answering: the callers read h->hctrl exactly as after a launch.
int res_push(ps_server* h, int worker, const void* g, int g_dtype, int g_on_device, int fuse, double now) {
  ResReq q{};
  q.op = fuse ? RES_PUSH : RES_APPLY;
  q.worker = worker;
  q.now = now;
  int rc = res_operand(h, g, g_dtype, g_on_device, &q);
  if (rc) return rc;
  ResResp resp;
  return res_call(h, q, &resp);
}

}  // namespace

int ps_resident_pause(ps_server* h) {
  ps_resident* r = h->res;
  if (!r || !r->running) return PS_OK;
  if (r->mbox->alive || cudaStreamQuery(r->stream) != cudaSuccess) {
    const unsigned long long seq = r->seq;
    ResReq q{};
    q.op = RES_STOP;
    std::memcpy((void*)&r->mbox->req, &q, sizeof(q));
    std::atomic_thread_fence(std::memory_order_seq_cst);
    r->mbox->req_seq = seq;
    PS_CK(h, cudaStreamSynchronize(r->stream));
    // the STOP was consumed unless the kernel retired first: then un-post it
    r->mbox->req_seq = seq - 1;
  }
  PS_CK(h, cudaStreamSynchronize(r->stream));
  r->running = false;
  return PS_OK;
}


extern "C" {

int ps_device_count(int32_t* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  *n = (e == cudaSuccess) ? c : 0;
  return e == cudaSuccess ? PS_OK : ps_cuda_fail(nullptr, e, "cudaGetDeviceCount");
}

const char* ps_last_error(const ps_server* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

int ps_create(const ps_config* cfg, const void* w0_host, int32_t w0_dtype, ps_server** out) {
  *out = nullptr;
  if (!cfg) return ps_fail(nullptr, PS_E_VALUE, "null config");
  if (cfg->paradigm < PS_BSP || cfg->paradigm > PS_DSSP)
    return ps_fail(nullptr, PS_E_VALUE, "paradigm: must be one of bsp, asp, ssp, dssp");
  if (cfg->worker_count < 1 || cfg->worker_count > PS_MAX_WORKERS)
    return ps_fail(nullptr, PS_E_VALUE, "worker_count: must be in [1, 64]");
  if (cfg->s_lower < 0 || cfg->r_max < 0)
    return ps_fail(nullptr, PS_E_VALUE, "staleness: s_lower and r_max must be >= 0");
  if (!(cfg->learning_rate > 0)) return ps_fail(nullptr, PS_E_VALUE, "learning_rate must be > 0");
  if (cfg->dimension < 1) return ps_fail(nullptr, PS_E_VALUE, "dimension: must be >= 1");
  ps_server* h = new ps_server();
  h->cfg = *cfg;
  h->dev = cfg->device;
  DevGuard guard(h->dev);
  cudaError_t e = cudaSetDevice(h->dev);
  if (e != cudaSuccess) {
    delete h;
    return ps_cuda_fail(nullptr, e, "cudaSetDevice");
  }
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->dev);
  h->d = cfg->dimension;
  h->nv = (h->d + 3) / 4;
  h->dpad = h->nv * 4;
  auto bail = [&](cudaError_t err, const char* what) {
    int rc = ps_cuda_fail(nullptr, err, what);
    ps_destroy(h);
    return rc;
  };
  if ((e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking))) return bail(e, "stream");
  if ((e = cudaEventCreate(&h->ev0)) || (e = cudaEventCreate(&h->ev1))) return bail(e, "event");
  for (int b = 0; b < 2; ++b) {
    if ((e = cudaMalloc(&h->w[b], h->dpad * sizeof(float)))) return bail(e, "cudaMalloc weights");
    if ((e = cudaMemsetAsync(h->w[b], 0, h->dpad * sizeof(float), h->stream))) return bail(e, "memset");
  }
  if ((e = cudaMalloc(&h->ctrl, sizeof(Ctrl)))) return bail(e, "cudaMalloc ctrl");
  if ((e = cudaHostAlloc((void**)&h->hctrl, sizeof(Ctrl), cudaHostAllocMapped)))
    return bail(e, "cudaHostAlloc ctrl mirror");
  if ((e = cudaHostGetDevicePointer((void**)&h->hctrl_dev, h->hctrl, 0)))
    return bail(e, "cudaHostGetDevicePointer");
  std::memset(h->hctrl, 0, sizeof(Ctrl));
  ps_gate_state& gs = h->hctrl->gate;
  gs.paradigm = cfg->paradigm;
  gs.worker_count = cfg->worker_count;
  gs.s_lower = cfg->s_lower;
  gs.r_max = cfg->r_max;
  gs.threshold = cfg->paradigm == PS_BSP ? 0 : cfg->s_lower;  // policy.py:143-146
  if ((e = cudaMemcpyAsync(h->ctrl, h->hctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream)))
    return bail(e, "ctrl upload");
  if (w0_host) {
    const size_t esz = w0_dtype == PS_F64 ? 8 : 4;
    void* tmp = nullptr;
    if ((e = cudaMalloc(&tmp, h->d * esz))) return bail(e, "cudaMalloc w0");
    if ((e = cudaMemcpyAsync(tmp, w0_host, h->d * esz, cudaMemcpyHostToDevice, h->stream)))
      return bail(e, "w0 upload");
    if (w0_dtype == PS_F64)
      k_load_in<double><<<h->sm_count * 4, 256, 0, h->stream>>>((const double*)tmp, h->w[0], h->d);
    else
      k_load_in<float><<<h->sm_count * 4, 256, 0, h->stream>>>((const float*)tmp, h->w[0], h->d);
    if ((e = cudaStreamSynchronize(h->stream))) return bail(e, "w0 convert");
    cudaFree(tmp);
  }
  if ((e = cudaStreamSynchronize(h->stream))) return bail(e, "create sync");
  *out = h;
  return PS_OK;
}

void ps_destroy(ps_server* h) {
  if (!h) return;
  DevGuard guard(h->dev);
  if (h->res) {
    ps_resident_pause(h);
    if (h->res->stream) cudaStreamDestroy(h->res->stream);
    if (h->res->mbox) cudaFreeHost(h->res->mbox);
    cudaFree(h->res->rd);
    if (h->res->ev) cudaEventDestroy(h->res->ev);
    delete h->res;
    h->res = nullptr;
  }
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->w[0]);
  cudaFree(h->w[1]);
  cudaFree(h->ctrl);
  cudaFreeHost(h->hctrl);
  cudaFree(h->stage);
  cudaFreeHost(h->hstage);
  ps_sim_buffers& s = h->sim;
  cudaFree(s.ops); cudaFree(s.gcount);
  cudaFree(s.rep); cudaFree(s.gbuf); cudaFree(s.center); cudaFree(s.ctime);
  cudaFree(s.trace); cudaFree(s.losses); cudaFree(s.out);
  cudaFree(s.calls); cudaFree(s.decisions); cudaFree(s.dstream); cudaFree(s.pred);
  ps_workers_free(h);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->habort) cudaFreeHost(h->habort);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

int ps_apply(ps_server* h, int32_t worker, const void* g, int32_t g_dtype, int32_t g_on_device,
             int32_t* applied) {
  DevGuard guard(h->dev);
  int rc = launch_apply(h, worker, g, g_dtype, g_on_device, 0, 0.0);
  if (rc) return rc;
  *applied = h->hctrl->applied;
  const int st = h->hctrl->status;
  if (st == PS_E_DIVERGED)
    return ps_fail(h, PS_E_DIVERGED, "non-finite weights after update " +
                                         std::to_string(h->hctrl->gate.version + 1) + " from worker " +
                                         std::to_string(worker));
  return st;
}

int ps_decide(ps_server* h, int32_t worker, double now, int32_t* granted, uint64_t* released) {
  DevGuard guard(h->dev);
  int rc;
  if (h->res && h->res->ctas > 0) {
    ResReq q{};
    q.op = RES_DECIDE;
    q.worker = worker;
    q.now = now;
    ResResp resp;
    if ((rc = res_call(h, q, &resp))) return rc;
  } else {
    if ((rc = mark(h, h->ev0))) return rc;
    k_decide<<<1, 32, 0, h->stream>>>(h->ctrl, worker, now, h->hctrl_dev);
    PS_CK(h, cudaGetLastError());
    if ((rc = mark(h, h->ev1)) || (rc = finish_op(h))) return rc;
  }
  *granted = h->hctrl->granted;
  *released = h->hctrl->released;
  if (h->hctrl->status == PS_E_PROTOCOL)
    return ps_fail(h, PS_E_PROTOCOL, "worker " + std::to_string(worker) +
                                         " is unknown or pushed while deferred");
  return PS_OK;
}

int ps_push(ps_server* h, int32_t worker, const void* g, int32_t g_dtype, int32_t g_on_device,
            double now, int32_t* applied, int32_t* granted, uint64_t* released) {
  DevGuard guard(h->dev);
  int rc = launch_apply(h, worker, g, g_dtype, g_on_device, 1, now);
  if (rc) return rc;
  *applied = h->hctrl->applied;
  *granted = h->hctrl->granted;
  *released = h->hctrl->released;
  const int st = h->hctrl->status;
  if (st == PS_E_DIVERGED)
    return ps_fail(h, PS_E_DIVERGED, "non-finite weights after update " +
                                         std::to_string(h->hctrl->gate.version + 1));
  if (st == PS_E_PROTOCOL)
    return ps_fail(h, PS_E_PROTOCOL, "worker " + std::to_string(worker) +
                                         " is unknown or pushed while deferred");
  return st;
}

int ps_pull(ps_server* h, int32_t worker, void* dst, int32_t dst_dtype, int32_t dst_on_device,
            int64_t* version) {
  if (worker < 0 || worker >= h->cfg.worker_count)
    return ps_fail(h, PS_E_PROTOCOL, "unknown worker " + std::to_string(worker));
  if ((h->hctrl->gate.deferred >> worker) & 1ull)
    return ps_fail(h, PS_E_PROTOCOL, "worker " + std::to_string(worker) + " pulled while deferred");
  return ps_read_weights(h, dst, dst_dtype, dst_on_device, version);
}

int ps_read_weights(ps_server* h, void* dst, int32_t dst_dtype, int32_t dst_on_device,
                    int64_t* version) {
  DevGuard guard(h->dev);
  if (dst_dtype != PS_F32 && dst_dtype != PS_F64) return ps_fail(h, PS_E_VALUE, "bad dtype");
  const float* src = h->w[h->cur];
  const size_t esz = dst_dtype == PS_F64 ? 8 : 4;
  if (version) *version = h->hctrl->gate.version;
  int rc = mark(h, h->ev0);
  if (rc) return rc;
  // device or pinned host destinations are written by the copy kernel itself
  // (over PCIe for pinned host memory); pageable ones take a staged copy
  if ((rc = after_producer(h))) return rc;  // the destination may still be in use there
  // f32 to host: the copy engine (measured faster than kernel stores over
  // PCIe); f64 to pinned host: the conversion kernel writes it in place
  const bool kernel_dst = dst_on_device || (dst_dtype == PS_F64 && !host_dma() && pinned_host(dst));
  if (h->res && h->res->ctas > 0 && aligned16(dst) && kernel_dst) {
    // resident: the persistent kernel copies; the host waits on its answer
    if (dst_on_device && (rc = res_after_producer(h))) return rc;
    ResReq q{};
    q.op = RES_PULL;
    q.dst = dst;
    q.dtype = dst_dtype;
    q.host_mem = dst_on_device ? 0 : 1;
    ResResp resp;
    if ((rc = res_call(h, q, &resp))) return rc;
    if (version) *version = resp.version;
    return PS_OK;
  }
  if (aligned16(dst) && kernel_dst) {
    const int grid = grid_for(h, h->nv);
    if (dst_dtype == PS_F32)
      k_copy_out<float><<<grid, 256, 0, h->stream>>>(src, (float*)dst, h->d);
    else
      k_copy_out<double><<<grid, 256, 0, h->stream>>>(src, (double*)dst, h->d);
    PS_CK(h, cudaGetLastError());
  } else if (dst_dtype == PS_F32) {
    PS_CK(h, cudaMemcpyAsync(dst, src, h->d * 4, cudaMemcpyDefault, h->stream));
  } else {
    if ((rc = ensure_stage(h, h->d * esz))) return rc;
    k_copy_out<double><<<grid_for(h, h->nv), 256, 0, h->stream>>>(src, (double*)h->stage, h->d);
    PS_CK(h, cudaGetLastError());
    PS_CK(h, cudaMemcpyAsync(dst, h->stage, h->d * esz, cudaMemcpyDefault, h->stream));
  }
  if ((rc = mark(h, h->ev1))) return rc;
  PS_CK(h, cudaStreamSynchronize(h->stream));
  if (h->profile) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    h->last_ms = ms;
  }
  return PS_OK;
}

int ps_get_state(ps_server* h, ps_gate_state* out) {
  DevGuard guard(h->dev);
  if (int prc = ps_resident_pause(h)) return prc;
  int rc = sync_ctrl(h);
  if (rc) return rc;
  *out = h->hctrl->gate;
  return PS_OK;
}

int ps_peek_state(const ps_server* h, ps_gate_state* out) {
  *out = h->hctrl->gate;
  return PS_OK;
}

int ps_set_state(ps_server* h, const ps_gate_state* in) {
  DevGuard guard(h->dev);
  if (int prc = ps_resident_pause(h)) return prc;
  if (in->worker_count != h->cfg.worker_count || in->paradigm != h->cfg.paradigm)
    return ps_fail(h, PS_E_VALUE, "state does not match the server configuration");
  for (int q = 0; q < in->worker_count; ++q)
    if (in->credits[q] < 0) return ps_fail(h, PS_E_VALUE, "credits cannot go negative");
  h->hctrl->gate = *in;
  PS_CK(h, cudaMemcpyAsync(&h->ctrl->gate, &h->hctrl->gate, sizeof(ps_gate_state),
                           cudaMemcpyHostToDevice, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  return PS_OK;
}

int ps_set_resident(ps_server* h, int32_t ctas) {
  DevGuard guard(h->dev);
  if (ctas < 0 || ctas > h->sm_count) return ps_fail(h, PS_E_VALUE, "resident CTAs must be in [0, SM count]");
  if (int rc = ps_resident_pause(h)) return rc;
  if (ctas == 0) {
    if (h->res) h->res->ctas = 0;
    return PS_OK;
  }
  if (!h->res) {
    h->res = new ps_resident();
    ps_resident* r = h->res;
    PS_CK(h, cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    PS_CK(h, cudaHostAlloc((void**)&r->mbox, sizeof(ResMbox), cudaHostAllocMapped));
    std::memset((void*)r->mbox, 0, sizeof(ResMbox));
    PS_CK(h, cudaHostGetDevicePointer((void**)&r->mbox_dev, r->mbox, 0));
    PS_CK(h, cudaMalloc(&r->rd, sizeof(ResDev)));
    PS_CK(h, cudaMemset(r->rd, 0, sizeof(ResDev)));
    PS_CK(h, cudaDeviceSynchronize());
  }
  h->res->ctas = ctas;
  return PS_OK;
}

int ps_last_kernel_ms(ps_server* h, double* ms) {
  *ms = h->last_ms;
  return PS_OK;
}

int ps_profile_floor(ps_server* h, double* ms) {
  // the profiling bracket around an empty kernel: what every per-op
  // last_kernel_ms figure contains besides the op itself (the launch as the
  // GPU sees it and the two timestamps)
  DevGuard guard(h->dev);
  k_spin<<<1, 32, 0, h->stream>>>(kProfileSpinNs);
  PS_CK(h, cudaEventRecord(h->ev0, h->stream));
  k_spin<<<1, 32, 0, h->stream>>>(0);
  PS_CK(h, cudaEventRecord(h->ev1, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  float e = 0.f;
  PS_CK(h, cudaEventElapsedTime(&e, h->ev0, h->ev1));
  *ms = e;
  return PS_OK;
}

int ps_set_profiling(ps_server* h, int32_t on) {
  h->profile = on ? 1 : 0;
  return PS_OK;
}

int ps_abort(ps_server* h) {
  if (h->habort) *reinterpret_cast<volatile int*>(h->habort) = 1;
  return PS_OK;
}

int ps_set_producer_stream(ps_server* h, void* cuda_stream) {
  h->producer = (cudaStream_t)cuda_stream;
  return PS_OK;
}

int ps_controller_batch(int32_t device, const double* tables, const int32_t* r_max, int32_t n,
                        int32_t* out) {
  if (n <= 0) return PS_OK;
  if (!tables || !r_max || !out) return ps_fail(nullptr, PS_E_VALUE, "null controller batch buffer");
  DevGuard guard(device);
  double* dt = nullptr;
  int* dr = nullptr;
  int* dout = nullptr;
  cudaStream_t st = nullptr;
  const char* what = "controller batch";
  // every step checked; every allocation freed on every path; a server-style
  // non-blocking stream, not the legacy one
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (!e) { what = "controller alloc"; e = cudaMalloc(&dt, sizeof(double) * 4 * n); }
  if (!e) e = cudaMalloc(&dr, sizeof(int) * n);
  if (!e) e = cudaMalloc(&dout, sizeof(int) * n);
  if (!e) { what = "controller input copy"; e = cudaMemcpyAsync(dt, tables, sizeof(double) * 4 * n, cudaMemcpyHostToDevice, st); }
  if (!e) e = cudaMemcpyAsync(dr, r_max, sizeof(int) * n, cudaMemcpyHostToDevice, st);
  if (!e) {
    what = "controller launch";
    const int warps_per_block = 4;
    k_controller_batch<<<(n + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
        dt, dr, n, dout);
    e = cudaGetLastError();
  }
  if (!e) { what = "controller result copy"; e = cudaMemcpyAsync(out, dout, sizeof(int) * n, cudaMemcpyDeviceToHost, st); }
  if (!e) e = cudaStreamSynchronize(st);
  cudaFree(dt);
  cudaFree(dr);
  cudaFree(dout);
  if (st) cudaStreamDestroy(st);
  return e == cudaSuccess ? PS_OK : ps_cuda_fail(nullptr, e, what);
}

int ps_apply_vectors(int32_t device, const void* w, const void* g, int32_t dtype, int64_t n,
                     double lr, void* out, int32_t* status) {
  if (!(lr > 0)) return ps_fail(nullptr, PS_E_VALUE, "learning_rate must be > 0");
  if (n < 1) return ps_fail(nullptr, PS_E_VALUE, "dimension must be >= 1");
  if (dtype != PS_F32 && dtype != PS_F64) return ps_fail(nullptr, PS_E_VALUE, "bad dtype");
  if (!w || !g || !out || !status) return ps_fail(nullptr, PS_E_VALUE, "null buffer");
  // Stateless: no server, control block or mapped mirror -- one stream, three
  // stream-ordered scratch buffers, the rounding loads, one apply pass whose
  // non-finite result flag comes back with the weights.
  DevGuard guard(device);
  const size_t esz = dtype == PS_F64 ? 8 : 4;
  const long long dpad = (n + 3) / 4 * 4;
  cudaStream_t st = nullptr;
  void* raw = nullptr;   // host-dtype staging of w and g
  float* f = nullptr;    // [w | g | out] fp32, each dpad long, + 1 flag word
  const char* what = "apply_vectors";
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (!e) e = cudaMallocAsync(&raw, 2 * n * esz, st);
  if (!e) e = cudaMallocAsync((void**)&f, (3 * dpad + 4) * sizeof(float), st);
  if (!e) e = cudaMemsetAsync(f, 0, (3 * dpad + 4) * sizeof(float), st);
  if (!e) { what = "apply_vectors upload"; e = cudaMemcpyAsync(raw, w, n * esz, cudaMemcpyHostToDevice, st); }
  if (!e) e = cudaMemcpyAsync((char*)raw + n * esz, g, n * esz, cudaMemcpyHostToDevice, st);
  unsigned flag = 0;
  if (!e) {
    what = "apply_vectors launch";
    const int blocks = (int)std::min<long long>((n + 255) / 256, 4096);
    if (dtype == PS_F64) {
      k_load_in<double><<<blocks, 256, 0, st>>>((const double*)raw, f, n);
      k_load_in<double><<<blocks, 256, 0, st>>>((const double*)raw + n, f + dpad, n);
    } else {
      k_load_in<float><<<blocks, 256, 0, st>>>((const float*)raw, f, n);
      k_load_in<float><<<blocks, 256, 0, st>>>((const float*)raw + n, f + dpad, n);
    }
    k_apply_vec<<<blocks, 256, 0, st>>>(f, f + dpad, f + 2 * dpad, n, (float)lr,
                                        reinterpret_cast<unsigned*>(f + 3 * dpad));
    e = cudaGetLastError();
  }
  if (!e) {
    what = "apply_vectors result copy";
    e = cudaMemcpyAsync(&flag, f + 3 * dpad, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  }
  if (!e && dtype == PS_F32) e = cudaMemcpyAsync(out, f + 2 * dpad, n * 4, cudaMemcpyDeviceToHost, st);
  if (!e && dtype == PS_F64) {
    k_copy_out<double><<<(int)std::min<long long>((n / 4 + 255) / 256 + 1, 4096), 256, 0, st>>>(
        f + 2 * dpad, (double*)raw, n);
    e = cudaGetLastError();
    if (!e) e = cudaMemcpyAsync(out, raw, n * 8, cudaMemcpyDeviceToHost, st);
  }
  if (!e) e = cudaStreamSynchronize(st);
  if (raw) cudaFreeAsync(raw, st);
  if (f) cudaFreeAsync(f, st);
  if (st) { cudaStreamSynchronize(st); cudaStreamDestroy(st); }
  if (e) return ps_cuda_fail(nullptr, e, what);
  // apply_update (server.py:29-42) has no gradient check of its own: a
  // non-finite gradient surfaces as a non-finite result (DivergenceError)
  *status = flag ? PS_E_DIVERGED : PS_OK;
  return PS_OK;
}

}  // extern "C"
