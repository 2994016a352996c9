// ps_shard.cu -- the parameter server sharded across G GPUs (one process per
// GPU), contiguous-range shards, all data movement over NVLink P2P.
//
// Layout: shard s owns parameters [s*S, min(d,(s+1)*S))
// with S = ceil(d/G) rounded up to a multiple of 4 (so no float4 straddles two
// shards). Rank r hosts shard r, worker r's update buffer (full d) and a small
// flag array that its peers write into through CUDA-IPC mappings.
//
// One step = one same-instant push group of all G workers (the homogeneous
// schedule of simnet.py:167-201: apply every update in seq order, then decide
// each), three kernels in stream order on every rank, with no host in the loop
// and no collective:
//
//   K1 k_shard_ready  worker r scans its update for non-finite values
//                     (server.py:65-67 needs the whole vector's verdict before
//                     any shard applies it) and release-stores
//                     ready = (t<<1)|bad into every owner's flag array.
//   K2 k_shard_apply  owner r waits for all G ready flags, then streams its
//                     shard once: w = w - lr*g_p for p = 0..G-1 in ticket
//                     order (skipping rejected updates), reading each g_p slice
//                     straight from worker p's HBM over NVLink (P2P loads,
//                     payload crosses once). Per-element order == global push
//                     order, no atomics on weights. The last CTA publishes
//                     applied = t to every worker and runs the replicated gate
//                     (gate.cuh) for the G pushes -- every rank computes the same
//                     decisions from the same inputs, so no gate traffic crosses
//                     NVLink.
//   K3 k_shard_pull   worker r waits for all G applied flags and gathers the
//                     full weights (handle_pull, server.py:84-91) from the G
//                     shards into its replica with P2P loads.
//
// Waits are only ever on flags written by OTHER GPUs' kernels that never wait
// on the waiter's later work, so the protocol cannot deadlock; every spin has a
// watchdog that aborts the kernel instead of hanging the GPU.
#include <cuda_runtime.h>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gate.cuh"

using namespace dssp;

namespace {

constexpr int kMaxRanks = 16;
constexpr int kThreads = 256;
constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct ShardPtrs {
  const float* w[kMaxRanks];            // each shard's weights (peer mappings)
  const float* upd[kMaxRanks];          // each worker's update buffer
  unsigned long long* flags[kMaxRanks]; // each rank's flag array: ready[G] then applied[G]
  long long lo[kMaxRanks];
};

struct ShardCtl {
  ps_gate_state gate;
  uint32_t arrive[3];
  uint32_t bad;
  int32_t status;
  int32_t _pad;
  unsigned long long trace_n;
  // Ticket order of the current push group: the seq order in which the
  // previous group's decisions scheduled the workers' GRANT_DELIVER events
  // (grant -> pusher first, then released ids ascending; simnet.py:192-201),
  // which every later event of the homogeneous chain inherits.
  int32_t order[kMaxRanks];
};

struct IpcBlob {
  cudaIpcMemHandle_t w, upd, flags;
  long long lo, hi;
  int rank, world;
};

__device__ bool wait_flags(const unsigned long long* f, int n, unsigned long long want,
                           unsigned long long* acc_bad, ShardCtl* ctl) {
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long bad = 0;
  for (int q = 0; q < n; ++q) {
    unsigned long long v;
    while ((v = ld_acquire_sys_u64(f + q)) < want) {
      if (globaltimer_ns() - t0 > kTimeoutNs) {
        atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT);
        return false;
      }
      __nanosleep(100);
    }
    if (acc_bad && (v & 1ull)) bad |= 1ull << q;
  }
  if (acc_bad) *acc_bad = bad;
  return true;
}

// Last-CTA election; returns true in exactly one CTA (counter k is reset).
__device__ bool last_cta(ShardCtl* ctl, int k) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(&ctl->arrive[k], 1u);
    s_last = (prev == gridDim.x - 1);
    if (s_last) ctl->arrive[k] = 0;
  }
  __syncthreads();
  return s_last;
}

__global__ void __launch_bounds__(kThreads)
k_shard_ready(const float* __restrict__ upd, long long d, ShardPtrs P, int G, int me,
              unsigned long long t, ShardCtl* ctl) {
  const long long nv = d >> 2;
  unsigned bad = 0;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long j = (long long)blockIdx.x * kThreads + threadIdx.x; j < nv; j += stride)
    bad |= nonfinite4(ld_stream(reinterpret_cast<const float4*>(upd) + j)) ? 1u : 0u;
  if (blockIdx.x == 0 && threadIdx.x < (d & 3)) bad |= nonfinite(upd[(nv << 2) + threadIdx.x]) ? 1u : 0u;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && bad) atomicOr(&ctl->bad, 1u);
  if (!last_cta(ctl, 0)) return;
  if (threadIdx.x == 0) {
    const unsigned b = atomicExch(&ctl->bad, 0u);
    __threadfence_system();
    for (int s = 0; s < G; ++s) st_release_sys_u64(P.flags[s] + me, (t << 1) | (b ? 1ull : 0ull));
  }
}

template <int G_MAX>
__global__ void __launch_bounds__(kThreads)
k_shard_apply(float* __restrict__ w, long long n_local, ShardPtrs P, int G, int me,
              unsigned long long t, float lr, ShardCtl* ctl, double now, ps_trace_row* trace,
              long long trace_cap) {
  __shared__ unsigned long long s_bad;
  if (threadIdx.x == 0) {
    unsigned long long bad = 0;
    if (!wait_flags(P.flags[me], G, t << 1, &bad, ctl)) bad = ~0ull;
    s_bad = bad;
  }
  __syncthreads();
  const unsigned long long badmask = s_bad;
  if (badmask == ~0ull) return;  // watchdog fired
  const long long nv = (n_local + 3) >> 2;
  const long long lo = P.lo[me];
  const float4* src[G_MAX];
  bool skip[G_MAX];
#pragma unroll
  for (int i = 0; i < G_MAX; ++i) {
    const int p = i < G ? ctl->order[i] : 0;
    src[i] = reinterpret_cast<const float4*>(P.upd[p] + lo);
    skip[i] = (badmask >> p) & 1ull;
  }
  unsigned dbad = 0;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long j = (long long)blockIdx.x * kThreads + threadIdx.x; j < nv; j += stride) {
    float4 g[G_MAX];
#pragma unroll
    for (int i = 0; i < G_MAX; ++i)
      if (i < G) g[i] = ld_stream(src[i] + j);
    float4 x = reinterpret_cast<float4*>(w)[j];
#pragma unroll
    for (int i = 0; i < G_MAX; ++i)
      if (i < G && !skip[i]) x = apply4(x, lr, g[i]);
    dbad |= nonfinite4(x) ? 1u : 0u;
    reinterpret_cast<float4*>(w)[j] = x;
  }
  dbad = __syncthreads_or(dbad);
  if (threadIdx.x == 0 && dbad) atomicCAS(&ctl->status, PS_OK, PS_E_DIVERGED);
  if (!last_cta(ctl, 1)) return;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int s = 0; s < G; ++s) st_release_sys_u64(P.flags[s] + G + me, t);
      ctl->gate.version += G - __popcll(badmask);
      ctl->gate.rejected += __popcll(badmask);
    }
    __syncwarp();
    // the replicated gate: every rank decides the same group in ticket order
    int next[kMaxRanks];
    int n_next = 0;
    for (int i = 0; i < G; ++i) {
      const int p = ctl->order[i];
      const GateResult r = gate_on_push(&ctl->gate, p, now);
      if (threadIdx.x == 0) {
        if (r.status != PS_OK) atomicCAS(&ctl->status, PS_OK, r.status);
        if (r.status == PS_OK && r.outcome == 0) {
          next[n_next++] = p;
          for (int q = 0; q < G; ++q)
            if ((r.released >> q) & 1ull) next[n_next++] = q;
        }
        const unsigned long long n = ctl->trace_n++;
        if ((long long)n < trace_cap) {
          ps_trace_row row;
          row.time = now;
          row.worker = p;
          row.kind = PS_EV_PUSH_ARRIVE;
          row.count = ctl->gate.clocks[p];
          row.decision = r.outcome;
          row._pad = 0;
          row.released = r.released;
          trace[n] = row;
        }
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) {
      // every worker must be back for the next group (homogeneous schedule)
      if (n_next != G) atomicCAS(&ctl->status, PS_OK, PS_E_PROTOCOL);
      for (int i = 0; i < n_next && i < G; ++i) ctl->order[i] = next[i];
    }
  }
}

__global__ void __launch_bounds__(kThreads)
k_shard_pull(float* __restrict__ dst, long long d, long long S, ShardPtrs P, int G, int me,
             unsigned long long t, ShardCtl* ctl) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = wait_flags(P.flags[me] + G, G, t, nullptr, ctl) ? 1 : 0;
  __syncthreads();
  if (!s_ok) return;
  const long long nv = (d + 3) >> 2;
  const long long S4 = S >> 2;
  const long long stride = (long long)gridDim.x * kThreads;
  constexpr int U = 4;
  for (long long base = (long long)blockIdx.x * kThreads * U + threadIdx.x; base < nv; base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * kThreads;
      if (j < nv) {
        const int s = (int)(j / S4);
        v[u] = ld_stream(reinterpret_cast<const float4*>(P.w[s]) + (j - (long long)s * S4));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * kThreads;
      if (j < nv) reinterpret_cast<float4*>(dst)[j] = v[u];
    }
  }
}

template <typename T>
__global__ void k_shard_load(const T* src, float* dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = (float)src[i];
}

}  // namespace

struct ps_shard_server {
  ps_config cfg{};
  int world = 1, rank = 0, dev = 0, sm_count = 148;
  cudaStream_t stream = nullptr;
  long long d = 0, S = 0, lo = 0, hi = 0, n_local = 0, dpad = 0;
  float* w = nullptr;                 // local shard (padded to a multiple of 4)
  float* upd = nullptr;               // worker update buffer [dpad]
  float* rep = nullptr;               // worker replica [dpad]
  unsigned long long* flags = nullptr;
  ShardCtl* ctl = nullptr;
  ShardCtl* hctl = nullptr;
  ps_trace_row* trace = nullptr;
  long long trace_cap = 0;
  ShardPtrs ptrs{};
  std::vector<void*> opened;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
};

namespace {

thread_local std::string g_shard_error;

int sfail(ps_shard_server* h, int code, const std::string& m) {
  if (h) h->err = m; else g_shard_error = m;
  return code;
}

#define SCK(h, call)                                                                     \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      return sfail((h), PS_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(_e) + \
                                       " in " #call);                                    \
  } while (0)

struct Dev {
  int prev = 0;
  explicit Dev(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
  ~Dev() { cudaSetDevice(prev); }
};

void shard_range(long long d, int G, int r, long long* S, long long* lo, long long* hi) {
  long long s = (d + G - 1) / G;
  s = (s + 3) / 4 * 4;
  *S = s;
  *lo = s * r < d ? s * r : d;
  *hi = s * (r + 1) < d ? s * (r + 1) : d;
}

}  // namespace

extern "C" {

int ps_shard_range(int64_t d, int32_t world, int32_t rank, int64_t* lo, int64_t* hi) {
  long long S, l, h;
  shard_range(d, world, rank, &S, &l, &h);
  *lo = l;
  *hi = h;
  return PS_OK;
}

const char* ps_shard_last_error(const ps_shard_server* h) {
  return h ? h->err.c_str() : g_shard_error.c_str();
}

int ps_shard_create(const ps_config* cfg, int32_t world, int32_t rank, const void* w0,
                    int64_t w0_flags, ps_shard_server** out) {
  *out = nullptr;
  if (world < 1 || world > kMaxRanks) return sfail(nullptr, PS_E_VALUE, "world size must be 1..16");
  if (cfg->worker_count != world)
    return sfail(nullptr, PS_E_VALUE, "sharded server: one worker per rank (worker_count == world)");
  if (!(cfg->learning_rate > 0)) return sfail(nullptr, PS_E_VALUE, "learning_rate must be > 0");
  auto* h = new ps_shard_server();
  h->cfg = *cfg;
  h->world = world;
  h->rank = rank;
  h->dev = cfg->device;
  Dev guard(h->dev);
  cudaSetDevice(h->dev);
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->dev);
  h->d = cfg->dimension;
  shard_range(h->d, world, rank, &h->S, &h->lo, &h->hi);
  h->n_local = h->hi - h->lo;
  h->dpad = (h->d + 3) / 4 * 4;
  const size_t shard_bytes = (size_t)((h->n_local + 3) / 4 * 4 + 4) * sizeof(float);
  cudaError_t e;
  auto bail = [&](const char* what) {
    int rc = sfail(nullptr, PS_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e) + " in " + what);
    ps_shard_destroy(h);
    return rc;
  };
  if ((e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking))) return bail("stream");
  if ((e = cudaEventCreate(&h->ev0)) || (e = cudaEventCreate(&h->ev1))) return bail("events");
  if ((e = cudaMalloc(&h->w, shard_bytes))) return bail("shard");
  if ((e = cudaMemset(h->w, 0, shard_bytes))) return bail("shard memset");
  if ((e = cudaMalloc(&h->upd, h->dpad * sizeof(float)))) return bail("update buffer");
  if ((e = cudaMemset(h->upd, 0, h->dpad * sizeof(float)))) return bail("update memset");
  if ((e = cudaMalloc(&h->rep, h->dpad * sizeof(float)))) return bail("replica");
  if ((e = cudaMalloc(&h->flags, 2 * kMaxRanks * sizeof(unsigned long long)))) return bail("flags");
  if ((e = cudaMemset(h->flags, 0, 2 * kMaxRanks * sizeof(unsigned long long)))) return bail("flags memset");
  if ((e = cudaMalloc(&h->ctl, sizeof(ShardCtl)))) return bail("ctl");
  if ((e = cudaMallocHost(&h->hctl, sizeof(ShardCtl)))) return bail("hctl");
  std::memset(h->hctl, 0, sizeof(ShardCtl));
  ps_gate_state& gs = h->hctl->gate;
  gs.paradigm = cfg->paradigm;
  gs.worker_count = cfg->worker_count;
  gs.s_lower = cfg->s_lower;
  gs.r_max = cfg->r_max;
  gs.threshold = cfg->paradigm == PS_BSP ? 0 : cfg->s_lower;
  for (int r = 0; r < kMaxRanks; ++r) h->hctl->order[r] = r;  // initial pulls arrive in worker order
  if ((e = cudaMemcpy(h->ctl, h->hctl, sizeof(ShardCtl), cudaMemcpyHostToDevice))) return bail("ctl upload");
  // w0: full-length initial weights; bit 0 of w0_flags = on device, bit 1 = fp64
  if (w0) {
    const bool on_dev = w0_flags & 1, f64 = w0_flags & 2;
    const size_t esz = f64 ? 8 : 4;
    const char* src = (const char*)w0 + (size_t)h->lo * esz;
    void* tmp = nullptr;
    if (!on_dev) {
      if ((e = cudaMalloc(&tmp, h->n_local * esz + 16))) return bail("w0 staging");
      if ((e = cudaMemcpy(tmp, src, h->n_local * esz, cudaMemcpyHostToDevice))) return bail("w0 upload");
      src = (const char*)tmp;
    }
    if (h->n_local > 0) {
      if (f64) k_shard_load<double><<<h->sm_count * 2, 256, 0, h->stream>>>((const double*)src, h->w, h->n_local);
      else k_shard_load<float><<<h->sm_count * 2, 256, 0, h->stream>>>((const float*)src, h->w, h->n_local);
    }
    if ((e = cudaStreamSynchronize(h->stream))) return bail("w0 convert");
    if (tmp) cudaFree(tmp);
  }
  *out = h;
  return PS_OK;
}

void ps_shard_destroy(ps_shard_server* h) {
  if (!h) return;
  Dev guard(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->opened) cudaIpcCloseMemHandle(p);
  cudaFree(h->w); cudaFree(h->upd); cudaFree(h->rep); cudaFree(h->flags); cudaFree(h->ctl);
  cudaFree(h->trace);
  if (h->hctl) cudaFreeHost(h->hctl);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

// Opaque per-rank blob for the host to all-gather (torch.distributed plumbing).
int ps_shard_ipc_handles(ps_shard_server* h, void* out, int64_t cap) {
  if (cap < (int64_t)sizeof(IpcBlob)) return sfail(h, PS_E_VALUE, "blob buffer too small");
  Dev guard(h->dev);
  IpcBlob b{};
  SCK(h, cudaIpcGetMemHandle(&b.w, h->w));
  SCK(h, cudaIpcGetMemHandle(&b.upd, h->upd));
  SCK(h, cudaIpcGetMemHandle(&b.flags, h->flags));
  b.lo = h->lo;
  b.hi = h->hi;
  b.rank = h->rank;
  b.world = h->world;
  std::memcpy(out, &b, sizeof(b));
  return (int)sizeof(IpcBlob);
}

int ps_shard_connect(ps_shard_server* h, const void* blobs, int64_t len) {
  if (len < (int64_t)sizeof(IpcBlob) * h->world) return sfail(h, PS_E_VALUE, "need one blob per rank");
  Dev guard(h->dev);
  const IpcBlob* b = (const IpcBlob*)blobs;
  for (int r = 0; r < h->world; ++r) {
    if (b[r].rank != r || b[r].world != h->world) return sfail(h, PS_E_VALUE, "blobs out of order");
    h->ptrs.lo[r] = b[r].lo;
    if (r == h->rank) {
      h->ptrs.w[r] = h->w;
      h->ptrs.upd[r] = h->upd;
      h->ptrs.flags[r] = h->flags;
      continue;
    }
    void *pw = nullptr, *pu = nullptr, *pf = nullptr;
    SCK(h, cudaIpcOpenMemHandle(&pw, b[r].w, cudaIpcMemLazyEnablePeerAccess));
    SCK(h, cudaIpcOpenMemHandle(&pu, b[r].upd, cudaIpcMemLazyEnablePeerAccess));
    SCK(h, cudaIpcOpenMemHandle(&pf, b[r].flags, cudaIpcMemLazyEnablePeerAccess));
    h->opened.push_back(pw);
    h->opened.push_back(pu);
    h->opened.push_back(pf);
    h->ptrs.w[r] = (const float*)pw;
    h->ptrs.upd[r] = (const float*)pu;
    h->ptrs.flags[r] = (unsigned long long*)pf;
  }
  return PS_OK;
}

// Device pointer of this rank's update buffer (the worker writes its update here).
int ps_shard_update_buffer(ps_shard_server* h, void** ptr, int64_t* padded_len) {
  *ptr = h->upd;
  *padded_len = h->dpad;
  return PS_OK;
}

// Enqueue `steps` push groups starting at step index t0 (1-based tickets) and
// wait for them. now[i] is the virtual push time of step i; dst (device, fp32,
// may be NULL) receives the pulled weights, else the internal replica does.
int ps_shard_run(ps_shard_server* h, int64_t t0, int32_t steps, const double* now, void* dst,
                 double* ms) {
  Dev guard(h->dev);
  if (steps < 1) return PS_OK;
  const long long need = (long long)(t0 + steps) * h->world + 8;
  if (need > h->trace_cap) {
    cudaFree(h->trace);
    h->trace = nullptr;
    const long long cap = need * 2;
    SCK(h, cudaMalloc(&h->trace, cap * sizeof(ps_trace_row)));
    h->trace_cap = cap;
  }
  float* out = dst ? (float*)dst : h->rep;
  const int G = h->world, me = h->rank;
  const float lr = (float)h->cfg.learning_rate;
  const int grid = h->sm_count * 4;
  SCK(h, cudaEventRecord(h->ev0, h->stream));
  for (int i = 0; i < steps; ++i) {
    const unsigned long long t = (unsigned long long)(t0 + i);
    k_shard_ready<<<grid, kThreads, 0, h->stream>>>(h->upd, h->d, h->ptrs, G, me, t, h->ctl);
    if (G <= 2)
      k_shard_apply<2><<<grid, kThreads, 0, h->stream>>>(h->w, h->n_local, h->ptrs, G, me, t, lr, h->ctl,
                                                         now[i], h->trace, h->trace_cap);
    else if (G <= 4)
      k_shard_apply<4><<<grid, kThreads, 0, h->stream>>>(h->w, h->n_local, h->ptrs, G, me, t, lr, h->ctl,
                                                         now[i], h->trace, h->trace_cap);
    else if (G <= 8)
      k_shard_apply<8><<<grid, kThreads, 0, h->stream>>>(h->w, h->n_local, h->ptrs, G, me, t, lr, h->ctl,
                                                         now[i], h->trace, h->trace_cap);
    else
      k_shard_apply<16><<<grid, kThreads, 0, h->stream>>>(h->w, h->n_local, h->ptrs, G, me, t, lr, h->ctl,
                                                          now[i], h->trace, h->trace_cap);
    k_shard_pull<<<grid, kThreads, 0, h->stream>>>(out, h->d, h->S, h->ptrs, G, me, t, h->ctl);
  }
  SCK(h, cudaGetLastError());
  SCK(h, cudaEventRecord(h->ev1, h->stream));
  SCK(h, cudaMemcpyAsync(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  float e = 0.f;
  cudaEventElapsedTime(&e, h->ev0, h->ev1);
  if (ms) *ms = e;
  const int st = h->hctl->status;
  if (st == PS_E_TIMEOUT) return sfail(h, PS_E_TIMEOUT, "device watchdog fired waiting for a peer");
  if (st == PS_E_DIVERGED) return sfail(h, PS_E_DIVERGED, "non-finite weights in the sharded server");
  if (st == PS_E_PROTOCOL) return sfail(h, PS_E_PROTOCOL, "protocol violation in the replicated gate");
  return PS_OK;
}

int ps_shard_read_shard(ps_shard_server* h, void* dst_host, int64_t* n) {
  Dev guard(h->dev);
  *n = h->n_local;
  if (h->n_local > 0) SCK(h, cudaMemcpy(dst_host, h->w, h->n_local * sizeof(float), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_shard_read_replica(ps_shard_server* h, void* dst_host) {
  Dev guard(h->dev);
  SCK(h, cudaMemcpy(dst_host, h->rep, h->d * sizeof(float), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_shard_get_state(ps_shard_server* h, ps_gate_state* out) {
  Dev guard(h->dev);
  SCK(h, cudaMemcpy(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost));
  *out = h->hctl->gate;
  return PS_OK;
}

int ps_shard_trace(ps_shard_server* h, ps_trace_row* rows, int64_t cap, int64_t* n) {
  Dev guard(h->dev);
  SCK(h, cudaMemcpy(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost));
  const long long have = (long long)h->hctl->trace_n < h->trace_cap ? (long long)h->hctl->trace_n : h->trace_cap;
  *n = have;
  const long long m = have < cap ? have : cap;
  if (m > 0) SCK(h, cudaMemcpy(rows, h->trace, m * sizeof(ps_trace_row), cudaMemcpyDeviceToHost));
  return PS_OK;
}

}  // extern "C"
