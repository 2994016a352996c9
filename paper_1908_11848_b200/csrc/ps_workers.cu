// ps_workers.cu -- free-running workers gated by device flags (north star (4)).
//
// The reference's threaded runner (runner.py:168-291) runs one OS thread per
// worker around ONE lock: apply_gradient -> decide_push(w, now) under the lock
// (runner.py:226-249), a deferred worker parks on its release Event until a
// granting push sets it (runner.py:243-263), and the pull happens under the
// lock again (runner.py:273-284). Here every worker is a CUDA stream and the
// host is out of the per-iteration loop:
//
//   worker stream p:  ... backward (writes the bound gradient buffer)
//                     k_wpush(p)   take a ticket, wait for the turn, apply,
//                                  decide at the device clock, write go flags
//                     wait go[p]   cuStreamWaitValue32(go[p] == 1): the stream
//                                  blocks WITHOUT occupying an SM or the host
//                     k_wpull(p)   take a ticket, wait for the turn, copy the
//                                  weights into the bound parameter buffer,
//                                  clear go[p]
//                     ... next forward
//
// The ticket order is the lock: every push and pull takes the next ticket when
// its first CTA starts and waits until `served` reaches it, so applies, gate
// decisions and pulls are serialized exactly like the runner's critical
// sections, in device arrival order. A grant sets go[p]; _release's released
// workers get go[q] (policy.py:197-206). All state is device-resident and
// indexed by worker, so an iteration can be captured in a CUDA graph once and
// replayed with no host work at all.
//
// Workers may sit on other GPUs of the box (one process, peer access over
// NVLink): the server's weights, gate tables, ticket counters and logs stay in
// the server GPU's HBM; a worker's push / pull kernels run on the worker's
// own GPU and reach them with P2P loads, stores and system-scope atomics; its
// go flag lives in its own GPU's memory (the stream waits on local memory) and
// is raised remotely by whichever GPU runs the granting push. Ticket hand-off
// then uses fence.sc.sys + system-scope release / acquire instead of the
// GPU-scope pair.
//
// Weights are double buffered as in k_apply: a non-finite update is rejected
// and counted (server.py:65-67), a non-finite result aborts the run with the
// weights unchanged (server.py:38-41): every go flag is raised so no stream
// stays blocked, and later kernels only advance the ticket.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstring>
#include <string>

#include "common.cuh"
#include "gate.cuh"
#include "server.h"

using namespace dssp;

namespace {

constexpr int kWThreads = 256;
constexpr int kWUnroll = 4;

struct WSlot {                    // per worker; reset by the last CTA of each kernel
  unsigned start;                 // CTAs that have started (first one takes the ticket)
  unsigned _pad;
  unsigned long long ticket;      // ticket + 1 once taken (0 = not yet)
  unsigned long long arrive;      // low: CTAs done, high: non-finite flag counts
  long long pushes;               // pushes of this worker so far (record ring index)
  long long pulls;
};

struct WCtl {
  unsigned long long next_ticket;
  unsigned long long served;      // tickets completed (the turn)
  unsigned* go[PS_MAX_WORKERS];   // worker q's go flag (on q's GPU): 1 = may pull
  int aborted;                    // a non-finite result: the run is over
  int status;                     // first error (PS_E_DIVERGED / PS_E_PROTOCOL)
  int diverged_worker;
  int _pad;
  unsigned long long t0;          // %globaltimer at ps_workers_start
  double time_scale;              // gate seconds per wall-clock second
  long long n_dec, n_pull;        // log lengths
  WSlot slot[PS_MAX_WORKERS];
};

struct WDec {                     // one decided push, in ticket order
  unsigned long long ticket;
  double now;
  int worker;
  int outcome;                    // 0 grant, 1 defer
  unsigned long long released;
  long long version;              // after this push's apply
  int applied;                    // 0: rejected (non-finite update)
  int _pad;
};

struct WPull {
  unsigned long long ticket;
  double now;
  int worker;
  int _pad;
  long long version;              // the snapshot's version
};

struct WArgs {
  WCtl* c;
  Ctrl* ctrl;                     // the server's control block (gate tables, cur, version)
  float* w0;
  float* w1;
  long long n, nv;
  float lr;
  int worker;
  const float* grad;              // bound gradient (push source)
  float* params;                  // bound parameters (pull destination)
  float* record;                  // optional [cap][dpad] ring of pushed updates
  long long record_cap, dpad;
  WDec* dec;
  WPull* pull;
  long long dec_cap, pull_cap;
  unsigned long long timeout_ns;
  unsigned* my_go;                // this worker's go flag (local to the launching GPU)
  int sys;                        // 1: the cluster spans GPUs (system-scope hand-off)
  long long clk_off;              // server GPU %globaltimer - this GPU's (ns), calibrated at bind
};

// The gate's clock: seconds since ps_workers_start on the SERVER GPU's
// %globaltimer. A worker on a peer GPU reads its own timer, shifted by the
// offset calibrated when it was bound (the GPUs' timers are not one clock:
// controller intervals mix every worker's timestamps, runner.py:234).
__device__ __forceinline__ double gate_now(const WCtl* c, long long clk_off) {
  const long long t = (long long)globaltimer_ns() + clk_off - (long long)c->t0;
  return (double)t * 1e-9 * c->time_scale;
}

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p, int sys) {
  return sys ? ld_acquire_sys_u64(p) : ld_acquire_u64(p);
}

// First CTA to start takes the next global ticket; every CTA then waits for
// the turn. Returns the ticket (thread 0 of every CTA; broadcast via smem).
__device__ __forceinline__ unsigned long long take_turn(const WArgs& a, WSlot* s) {
  __shared__ unsigned long long s_t;
  if (threadIdx.x == 0) {
    unsigned long long t;
    if (atomicAdd_system(&s->start, 1u) == 0u) {
      t = atomicAdd_system(&a.c->next_ticket, 1ull);
      if (a.sys) st_release_sys_u64(&s->ticket, t + 1);
      else st_release_u64(&s->ticket, t + 1);
    } else {
      unsigned long long v;
      while ((v = ld_acq(&s->ticket, a.sys)) == 0ull) __nanosleep(64);
      t = v - 1;
    }
    const unsigned long long start = globaltimer_ns();
    unsigned backoff = 32;
    while (ld_acq(&a.c->served, a.sys) != t) {
      __nanosleep(backoff);
      backoff = backoff < 1024 ? backoff * 2 : 1024;
      if (globaltimer_ns() - start > a.timeout_ns) {  // watchdog: never hang the box
        atomicCAS(&a.c->status, PS_OK, PS_E_TIMEOUT);
        a.c->aborted = 1;
        break;
      }
    }
    s_t = t;
  }
  __syncthreads();
  return s_t;
}

// Arrival at the end of a kernel: returns true in the last CTA (all CTAs'
// writes acquired), with the accumulated flag counts in *flags.
__device__ __forceinline__ bool arrive_last(WSlot* s, unsigned bad, unsigned* flags) {
  __shared__ unsigned s_bad;
  __shared__ int s_last;
  __shared__ unsigned s_flags;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  bad = __reduce_or_sync(kFull, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(&s_bad, bad);
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long add = 1ull | ((unsigned long long)((s_bad & 1u) | ((s_bad & 2u) << 15)) << 32);
    const unsigned long long prev = atom_add_acq_rel_gpu_u64(&s->arrive, add);
    s_last = ((unsigned)prev == gridDim.x - 1);
    s_flags = (unsigned)((prev + add) >> 32);
  }
  __syncthreads();
  *flags = s_flags;
  return s_last;
}

// The last CTA holds (acquired) every CTA's writes: the next ticket holder,
// possibly on another GPU, acquires them through `served`.
__device__ __forceinline__ void finish_turn(const WArgs& a, WSlot* s, unsigned long long t) {
  s->start = 0;
  s->ticket = 0;
  s->arrive = 0;
  if (a.sys) {
    __threadfence_system();
    st_release_sys_u64(&a.c->served, t + 1);
  } else {
    __threadfence();
    st_release_u64(&a.c->served, t + 1);
  }
}

__device__ __forceinline__ void raise_go(WCtl* c, int q) {
  unsigned* g = c->go[q];
  if (g) st_release_u32_sys(g, 1u);
}

__device__ __forceinline__ void raise_all(WCtl* c, int P) {
  for (int q = 0; q < P; ++q) raise_go(c, q);
}

// handle_push on the device (runner.py:226-252): apply in ticket order, then
// the gate decision at the device clock, then release flags.
__global__ void __launch_bounds__(kWThreads) k_wpush(WArgs a) {
  WSlot* s = &a.c->slot[a.worker];
  const unsigned long long t = take_turn(a, s);
  const bool skip = ld_volatile_s32_(&a.c->aborted) != 0;
  const int cur = ld_volatile_s32_(&a.ctrl->cur);
  const float4* src = reinterpret_cast<const float4*>(cur ? a.w1 : a.w0);
  float4* dst = reinterpret_cast<float4*>(cur ? a.w0 : a.w1);
  const float4* g4 = reinterpret_cast<const float4*>(a.grad);
  float4* rec = nullptr;
  if (a.record && a.record_cap > 0)
    rec = reinterpret_cast<float4*>(a.record + (s->pushes % a.record_cap) * a.dpad);
  unsigned bad = 0;
  if (!skip) {
    // kWUnroll float4 per thread per trip, every load issued before the
    // first use: the weights may sit across NVLink, where one load in flight
    // per thread would leave the link idle
    const long long stride = (long long)gridDim.x * kWThreads * kWUnroll;
    for (long long base = (long long)blockIdx.x * kWThreads * kWUnroll + threadIdx.x; base < a.nv;
         base += stride) {
      float4 g[kWUnroll], w[kWUnroll];
#pragma unroll
      for (int u = 0; u < kWUnroll; ++u) {
        const long long j = base + (long long)u * kWThreads;
        if (j < a.nv) {
          g[u] = ld_stream(g4 + j);
          w[u] = src[j];
        }
      }
#pragma unroll
      for (int u = 0; u < kWUnroll; ++u) {
        const long long j = base + (long long)u * kWThreads;
        if (j < a.nv) {
          const float4 r = apply4(w[u], a.lr, g[u]);
          bad |= nonfinite4(g[u]) ? 1u : 0u;
          bad |= nonfinite4(r) ? 2u : 0u;
          dst[j] = r;
          if (rec) rec[j] = g[u];
        }
      }
    }
    if (blockIdx.x == 0 && threadIdx.x < (a.n & 3)) {
      const long long i = (a.nv << 2) + threadIdx.x;
      const float* sw = cur ? a.w1 : a.w0;
      float* dw = cur ? a.w0 : a.w1;
      const float gi = a.grad[i];
      const float r = apply1(sw[i], a.lr, gi);
      bad |= nonfinite(gi) ? 1u : 0u;
      bad |= nonfinite(r) ? 2u : 0u;
      dw[i] = r;
      if (rec) reinterpret_cast<float*>(rec)[i] = gi;
    }
  }
  unsigned flags = 0;
  if (!arrive_last(s, bad, &flags) || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  WCtl* c = a.c;
  ps_gate_state* gs = &a.ctrl->gate;
  const int P = gs->worker_count;
  if (skip) {
    if (lane == 0) { s->pushes += 1; raise_all(c, P); finish_turn(a, s, t); }
    return;
  }
  int applied = 0, diverged = 0;
  if (lane == 0) {
    if (flags & 0xffffu) {
      gs->rejected += 1;                       // server.py:65-67
    } else if (flags >> 16) {
      diverged = 1;                            // server.py:38-41: weights unchanged
    } else {
      a.ctrl->cur = cur ^ 1;
      gs->version += 1;
      applied = 1;
    }
  }
  diverged = __shfl_sync(kFull, diverged, 0);
  if (diverged) {
    if (lane == 0) {
      if (atomicCAS(&c->status, PS_OK, PS_E_DIVERGED) == PS_OK) c->diverged_worker = a.worker;
      c->aborted = 1;
      s->pushes += 1;
      raise_all(c, P);
      finish_turn(a, s, t);
    }
    return;
  }
  // the gate tables, possibly in a peer GPU's memory, run from shared memory:
  // one coalesced copy in, the decision, the live entries back
  __shared__ ps_gate_state sg;
  {
    const unsigned long long* src8 = reinterpret_cast<const unsigned long long*>(gs);
    unsigned long long* dst8 = reinterpret_cast<unsigned long long*>(&sg);
    for (int i = lane; i < (int)(sizeof(ps_gate_state) / 8); i += 32) dst8[i] = src8[i];
  }
  __syncwarp();
  // runner.py:234: the decision's timestamp is taken at decision time
  double now = 0.0;
  if (lane == 0) now = gate_now(c, a.clk_off);
  now = __shfl_sync(kFull, now, 0);
  const GateResult r = gate_on_push(&sg, a.worker, now);
  __syncwarp();
  for (int q = lane; q < P; q += 32) {
    gs->clocks[q] = sg.clocks[q];
    gs->latest[q] = sg.latest[q];
    gs->previous[q] = sg.previous[q];
    gs->populated[q] = sg.populated[q];
    gs->credits[q] = sg.credits[q];
  }
  if (lane == 0) {
    gs->deferred = sg.deferred;
    gs->decisions = sg.decisions;
    if (r.status != PS_OK) {
      atomicCAS(&c->status, PS_OK, r.status);
      c->aborted = 1;
      raise_all(c, P);
    } else {
      if (r.outcome == 0) raise_go(c, a.worker);
      for (unsigned long long m = r.released; m; m &= m - 1) raise_go(c, __ffsll((long long)m) - 1);
    }
    const long long k = c->n_dec;
    if (k < a.dec_cap) {
      WDec e;
      e.ticket = t; e.now = now; e.worker = a.worker; e.outcome = r.outcome;
      e.released = r.released; e.version = gs->version; e.applied = applied; e._pad = 0;
      a.dec[k] = e;
    }
    c->n_dec = k + 1;
    s->pushes += 1;
    finish_turn(a, s, t);
  }
}

// handle_pull on the device (runner.py:273-284): the weights at this ticket
// into the worker's parameters; clears the worker's go flag.
__global__ void __launch_bounds__(kWThreads) k_wpull(WArgs a) {
  WSlot* s = &a.c->slot[a.worker];
  const unsigned long long t = take_turn(a, s);
  const bool skip = ld_volatile_s32_(&a.c->aborted) != 0;
  if (!skip) {
    const int cur = ld_volatile_s32_(&a.ctrl->cur);
    const float4* src = reinterpret_cast<const float4*>(cur ? a.w1 : a.w0);
    float4* dst = reinterpret_cast<float4*>(a.params);
    const long long stride = (long long)gridDim.x * kWThreads * kWUnroll;
    for (long long base = (long long)blockIdx.x * kWThreads * kWUnroll + threadIdx.x; base < a.nv;
         base += stride) {
      float4 v[kWUnroll];
#pragma unroll
      for (int u = 0; u < kWUnroll; ++u) {
        const long long j = base + (long long)u * kWThreads;
        if (j < a.nv) v[u] = src[j];
      }
#pragma unroll
      for (int u = 0; u < kWUnroll; ++u) {
        const long long j = base + (long long)u * kWThreads;
        if (j < a.nv) dst[j] = v[u];
      }
    }
    if (blockIdx.x == 0 && threadIdx.x < (a.n & 3)) {
      const long long i = (a.nv << 2) + threadIdx.x;
      a.params[i] = (cur ? a.w1 : a.w0)[i];
    }
  }
  unsigned flags = 0;
  if (!arrive_last(s, 0u, &flags) || threadIdx.x != 0) return;
  WCtl* c = a.c;
  if (!skip) {
    const long long k = c->n_pull;
    if (k < a.pull_cap) {
      WPull e;
      e.ticket = t;
      e.now = gate_now(c, a.clk_off);
      e.worker = a.worker; e._pad = 0;
      e.version = a.ctrl->gate.version;
      a.pull[k] = e;
    }
    c->n_pull = k + 1;
    *a.my_go = 0u;          // consumed: the next wait blocks until the next grant
  }
  s->pulls += 1;
  finish_turn(a, s, t);
}

// Fallback blocking (PS_WORKERS_SPIN=1, or where stream memory operations are
// unavailable): one warp polls go[p]. Occupies one warp slot while deferred.
__global__ void k_wwait(const unsigned* go, const int* aborted) {
  if (threadIdx.x != 0) return;
  unsigned backoff = 64;
  while (ld_acquire_u32(go) == 0u && ld_volatile_s32_(aborted) == 0) {
    __nanosleep(backoff);
    backoff = backoff < 4096 ? backoff * 2 : 4096;
  }
}

// Device busy-wait of `ns` on the worker's stream (the runner's spin_compute,
// runner.py:185-189): the 1x/2x/4x throttle of BASELINE configs[3].
__global__ void k_wspin(unsigned long long ns) {
  const unsigned long long t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}

__global__ void k_wstart(WCtl* c, double time_scale) {
  c->t0 = globaltimer_ns();
  c->time_scale = time_scale;
}

}  // namespace

struct ps_worker_rt {
  WCtl* c = nullptr;
  WDec* dec = nullptr;
  WPull* pull = nullptr;
  long long dec_cap = 0, pull_cap = 0;
  int ctas = 0;
  int spin_wait = 0;
  int sys = 0;                    // some worker sits on another GPU
  double time_scale = 1.0;
  struct Bind {
    cudaStream_t stream = nullptr;
    int dev = -1;
    const float* grad = nullptr;
    float* params = nullptr;
    float* record = nullptr;
    long long record_cap = 0;
    unsigned* go = nullptr;       // the worker's go flag, in its own GPU's memory
    int ctas = 0;
    long long clk_off = 0;        // server GPU clock - worker GPU clock (ns)
  } bind[PS_MAX_WORKERS];
};

void ps_workers_free(ps_server* h) {
  if (!h->wrt) return;
  for (auto& b : h->wrt->bind)
    if (b.go) { cudaSetDevice(b.dev); cudaFree(b.go); }
  cudaSetDevice(h->dev);
  cudaFree(h->wrt->c);
  cudaFree(h->wrt->dec);
  cudaFree(h->wrt->pull);
  delete h->wrt;
  h->wrt = nullptr;
}

namespace {

struct DevGuardW {
  int prev = 0;
  explicit DevGuardW(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
  ~DevGuardW() { cudaSetDevice(prev); }
};

WArgs make_args(ps_server* h, int worker) {
  ps_worker_rt* rt = h->wrt;
  WArgs a{};
  a.c = rt->c;
  a.ctrl = h->ctrl;
  a.w0 = h->w[0];
  a.w1 = h->w[1];
  a.n = h->d;
  a.nv = h->d >> 2;
  a.lr = (float)h->cfg.learning_rate;
  a.worker = worker;
  a.grad = rt->bind[worker].grad;
  a.params = rt->bind[worker].params;
  a.record = rt->bind[worker].record;
  a.record_cap = rt->bind[worker].record_cap;
  a.dpad = h->dpad;
  a.dec = rt->dec;
  a.pull = rt->pull;
  a.dec_cap = rt->dec_cap;
  a.pull_cap = rt->pull_cap;
  a.timeout_ns = 60ull * 1000 * 1000 * 1000;
  a.my_go = rt->bind[worker].go;
  a.sys = rt->sys;
  a.clk_off = rt->bind[worker].clk_off;
  return a;
}

// Reset the run state: counters, slots and logs zeroed, every bound worker's
// go flag cleared, the go-pointer table rewritten, the gate clock started.
int reset_run(ps_server* h) {
  ps_worker_rt* rt = h->wrt;
  WCtl hc;
  std::memset(&hc, 0, sizeof(hc));
  hc.time_scale = rt->time_scale;
  for (int q = 0; q < PS_MAX_WORKERS; ++q) hc.go[q] = rt->bind[q].go;
  PS_CK(h, cudaMemcpyAsync(rt->c, &hc, sizeof(WCtl), cudaMemcpyHostToDevice, h->stream));
  k_wstart<<<1, 1, 0, h->stream>>>(rt->c, rt->time_scale);
  PS_CK(h, cudaGetLastError());
  PS_CK(h, cudaStreamSynchronize(h->stream));
  for (int q = 0; q < PS_MAX_WORKERS; ++q) {
    auto& b = rt->bind[q];
    if (!b.go) continue;
    DevGuardW g(b.dev);
    // fully complete before any worker stream (non-blocking: no implicit
    // order with the legacy stream) can raise the flag
    PS_CK(h, cudaMemsetAsync(b.go, 0, sizeof(unsigned), 0));
    PS_CK(h, cudaDeviceSynchronize());
  }
  return PS_OK;
}

}  // namespace

extern "C" {

int ps_workers_start(ps_server* h, int64_t log_cap, double time_scale) {
  DevGuardW guard(h->dev);
  if (log_cap < 1) return ps_fail(h, PS_E_VALUE, "log capacity must be >= 1");
  if (!(time_scale > 0)) return ps_fail(h, PS_E_VALUE, "time_scale must be > 0");
  if (int prc = ps_resident_pause(h)) return prc;
  PS_CK(h, cudaStreamSynchronize(h->stream));
  if (!h->wrt) {
    h->wrt = new ps_worker_rt();
    ps_worker_rt* rt = h->wrt;
    PS_CK(h, cudaMalloc(&rt->c, sizeof(WCtl)));
    const char* v = getenv("PS_WORKERS_SPIN");
    rt->spin_wait = v && v[0] == '1';
  }
  ps_worker_rt* rt = h->wrt;
  if (rt->dec_cap < log_cap) {
    cudaFree(rt->dec);
    cudaFree(rt->pull);
    rt->dec = nullptr;
    rt->pull = nullptr;
    PS_CK(h, cudaMalloc(&rt->dec, log_cap * sizeof(WDec)));
    PS_CK(h, cudaMalloc(&rt->pull, log_cap * sizeof(WPull)));
    rt->dec_cap = rt->pull_cap = log_cap;
  }
  rt->time_scale = time_scale;
  return reset_run(h);
}

__global__ void k_read_timer(unsigned long long* out) { *out = globaltimer_ns(); }

// (this GPU's %globaltimer - the host's steady clock) in ns, from the sample
// with the shortest host round trip: the GPU read lies within it, so the
// error is at most half of it (a few us).
static int gpu_minus_host_ns(ps_server* h, int dev, long long* out) {
  DevGuardW g(dev);
  unsigned long long* d = nullptr;
  PS_CK(h, cudaMalloc(&d, sizeof(unsigned long long)));
  long long best_rtt = -1, best = 0;
  int rc = PS_OK;
  for (int i = 0; i < 9 && rc == PS_OK; ++i) {
    unsigned long long v = 0;
    const auto t0 = std::chrono::steady_clock::now();
    k_read_timer<<<1, 1>>>(d);
    if (cudaMemcpy(&v, d, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) { rc = PS_E_CUDA; break; }
    const auto t1 = std::chrono::steady_clock::now();
    const long long a = std::chrono::duration_cast<std::chrono::nanoseconds>(t0.time_since_epoch()).count();
    const long long b = std::chrono::duration_cast<std::chrono::nanoseconds>(t1.time_since_epoch()).count();
    if (i > 0 && (best_rtt < 0 || b - a < best_rtt)) {  // sample 0 warms the launch path
      best_rtt = b - a;
      best = (long long)v - (a + (b - a) / 2);
    }
  }
  cudaFree(d);
  if (rc) return ps_fail(h, rc, "clock calibration failed");
  *out = best;
  return PS_OK;
}

int ps_bind_worker_stream(ps_server* h, int32_t worker, void* cuda_stream, const float* grad,
                          float* params) {
  if (!h->wrt) return ps_fail(h, PS_E_VALUE, "call ps_workers_start first");
  if (worker < 0 || worker >= h->cfg.worker_count)
    return ps_fail(h, PS_E_PROTOCOL, "unknown worker " + std::to_string(worker));
  if (!grad || !params || ((uintptr_t)grad & 15u) || ((uintptr_t)params & 15u))
    return ps_fail(h, PS_E_VALUE, "gradient / parameter buffers must be 16-byte aligned device memory");
  // the worker's GPU is where its buffers live; a peer GPU reaches the
  // server's memory over NVLink (and the server GPU the worker's go flag)
  cudaPointerAttributes pa;
  PS_CK(h, cudaPointerGetAttributes(&pa, grad));
  if (pa.type != cudaMemoryTypeDevice) return ps_fail(h, PS_E_VALUE, "gradient buffer is not device memory");
  const int wdev = pa.device;
  ps_worker_rt* rt = h->wrt;
  auto& b = rt->bind[worker];
  // every GPU of the cluster must reach every other one: the server's memory
  // from each worker GPU, and each worker's go flag from whichever GPU runs a
  // granting push
  for (int other = -1; other < PS_MAX_WORKERS; ++other) {
    const int odev = other < 0 ? h->dev : rt->bind[other].dev;
    if (odev < 0 || odev == wdev || (other >= 0 && !rt->bind[other].grad)) continue;
    int ok = 0;
    PS_CK(h, cudaDeviceCanAccessPeer(&ok, wdev, odev));
    if (!ok) return ps_fail(h, PS_E_VALUE, "worker GPU cannot reach GPU " + std::to_string(odev) + " (no peer access)");
    for (int pass = 0; pass < 2; ++pass) {
      DevGuardW g(pass ? odev : wdev);
      cudaError_t e = cudaDeviceEnablePeerAccess(pass ? wdev : odev, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e) return ps_cuda_fail(h, e, "cudaDeviceEnablePeerAccess");
    }
    rt->sys = 1;
  }
  if (b.go && b.dev != wdev) {
    DevGuardW g(b.dev);
    cudaFree(b.go);
    b.go = nullptr;
  }
  if (!b.go) {
    DevGuardW g(wdev);
    PS_CK(h, cudaMalloc(&b.go, 256));
    PS_CK(h, cudaMemsetAsync(b.go, 0, 256, 0));
    PS_CK(h, cudaDeviceSynchronize());
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, wdev);
  // a small footprint for small models (the workers keep their GPU); more
  // CTAs as the vector grows -- each CTA keeps a bounded number of loads in
  // flight, and a remote (NVLink) apply is latency-bound per CTA -- up to
  // half the SMs (PS_WORKERS_CTAS overrides)
  {
    const long long per_cta = 256LL * kWUnroll * 4;  // float4 per CTA: about four trips
    long long want = ((h->d >> 2) + per_cta - 1) / per_cta;
    const long long lo_c = sms / 8 > 4 ? sms / 8 : 4, hi_c = sms / 2 > lo_c ? sms / 2 : lo_c;
    want = want < lo_c ? lo_c : want > hi_c ? hi_c : want;
    const char* v = getenv("PS_WORKERS_CTAS");
    b.ctas = v && atoi(v) > 0 ? atoi(v) : (int)want;
  }
  // a worker on a peer GPU stamps its decisions with the server GPU's clock
  b.clk_off = 0;
  if (wdev != h->dev) {
    long long ws = 0, ss = 0;
    int rc = gpu_minus_host_ns(h, h->dev, &ss);
    if (!rc) rc = gpu_minus_host_ns(h, wdev, &ws);
    if (rc) return rc;
    b.clk_off = ss - ws;
  }
  b.dev = wdev;
  b.stream = (cudaStream_t)cuda_stream;
  b.grad = grad;
  b.params = params;
  DevGuardW guard(h->dev);
  // (on the server stream and waited for: a pageable cudaMemcpy may return
  // before its DMA lands, and the worker streams do not order against it)
  PS_CK(h, cudaMemcpyAsync(&rt->c->go[worker], &b.go, sizeof(unsigned*), cudaMemcpyHostToDevice, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  return PS_OK;
}

int ps_worker_record(ps_server* h, int32_t worker, float* ring, int64_t capacity) {
  if (!h->wrt) return ps_fail(h, PS_E_VALUE, "call ps_workers_start first");
  if (worker < 0 || worker >= h->cfg.worker_count) return ps_fail(h, PS_E_PROTOCOL, "unknown worker");
  if (ring && ((uintptr_t)ring & 15u)) return ps_fail(h, PS_E_VALUE, "record ring must be 16-byte aligned");
  h->wrt->bind[worker].record = ring;
  h->wrt->bind[worker].record_cap = ring ? capacity : 0;
  return PS_OK;
}

// cuStreamWaitValue32 through the runtime's driver entry point: the library
// then has no link-time dependency on libcuda (it loads on a GPU-less host).
typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValue32Fn wait_value32() {
  static WaitValue32Fn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<WaitValue32Fn>(p);
  }();
  return fn;
}

int ps_enqueue_iteration(ps_server* h, int32_t worker, void* cuda_stream, uint64_t throttle_ns) {
  ps_worker_rt* rt = h->wrt;
  if (!rt) return ps_fail(h, PS_E_VALUE, "call ps_workers_start first");
  if (worker < 0 || worker >= h->cfg.worker_count)
    return ps_fail(h, PS_E_PROTOCOL, "unknown worker " + std::to_string(worker));
  auto& b = rt->bind[worker];
  if (!b.grad) return ps_fail(h, PS_E_VALUE, "worker " + std::to_string(worker) + " is not bound");
  DevGuardW guard(b.dev);   // the worker's kernels run on the worker's GPU
  cudaStream_t st = cuda_stream ? (cudaStream_t)cuda_stream : b.stream;
  WArgs a = make_args(h, worker);
  if (throttle_ns) {
    k_wspin<<<1, 32, 0, st>>>(throttle_ns);
    PS_CK(h, cudaGetLastError());
  }
  k_wpush<<<b.ctas, kWThreads, 0, st>>>(a);
  PS_CK(h, cudaGetLastError());
  if (rt->spin_wait) {
    k_wwait<<<1, 32, 0, st>>>(b.go, &rt->c->aborted);
    PS_CK(h, cudaGetLastError());
  } else {
    WaitValue32Fn wait = wait_value32();
    if (!wait) return ps_fail(h, PS_E_CUDA, "cuStreamWaitValue32 unavailable (set PS_WORKERS_SPIN=1)");
    CUresult r = wait((CUstream)st, (CUdeviceptr)b.go, 1u, CU_STREAM_WAIT_VALUE_EQ);
    if (r != CUDA_SUCCESS)
      return ps_fail(h, PS_E_CUDA, "cuStreamWaitValue32 failed with CUresult " + std::to_string((int)r));
  }
  k_wpull<<<b.ctas, kWThreads, 0, st>>>(a);
  PS_CK(h, cudaGetLastError());
  return PS_OK;
}

int ps_workers_status(ps_server* h, ps_workers_report* out) {
  DevGuardW guard(h->dev);
  ps_worker_rt* rt = h->wrt;
  if (!rt) return ps_fail(h, PS_E_VALUE, "call ps_workers_start first");
  WCtl c;
  PS_CK(h, cudaMemcpyAsync(&c, rt->c, sizeof(WCtl), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  std::memset(out, 0, sizeof(*out));
  out->tickets = (int64_t)c.served;
  out->decisions = c.n_dec;
  out->pulls = c.n_pull;
  out->status = c.status;
  out->diverged_worker = c.status == PS_E_DIVERGED ? c.diverged_worker : -1;
  out->aborted = c.aborted;
  for (int q = 0; q < PS_MAX_WORKERS; ++q) {
    const auto& b = rt->bind[q];
    if (!b.go) continue;
    unsigned v = 0;
    DevGuardW g(b.dev);
    PS_CK(h, cudaMemcpy(&v, b.go, sizeof(unsigned), cudaMemcpyDeviceToHost));
    out->go_mask |= (uint64_t)(v ? 1u : 0u) << q;
  }
  PS_CK(h, cudaMemcpyAsync(h->hctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  h->cur = h->hctrl->cur;
  return PS_OK;
}

int ps_workers_log(ps_server* h, ps_worker_decision* dec, int64_t dec_cap, ps_worker_pull* pulls,
                   int64_t pull_cap, int64_t* n_dec, int64_t* n_pull) {
  DevGuardW guard(h->dev);
  ps_worker_rt* rt = h->wrt;
  if (!rt) return ps_fail(h, PS_E_VALUE, "call ps_workers_start first");
  static_assert(sizeof(WDec) == sizeof(ps_worker_decision), "decision row layout");
  static_assert(sizeof(WPull) == sizeof(ps_worker_pull), "pull row layout");
  WCtl c;
  PS_CK(h, cudaMemcpyAsync(&c, rt->c, sizeof(WCtl), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  const long long nd = c.n_dec < rt->dec_cap ? c.n_dec : rt->dec_cap;
  const long long np = c.n_pull < rt->pull_cap ? c.n_pull : rt->pull_cap;
  *n_dec = c.n_dec;
  *n_pull = c.n_pull;
  if (dec && dec_cap > 0 && nd > 0)
    PS_CK(h, cudaMemcpy(dec, rt->dec, (nd < dec_cap ? nd : dec_cap) * sizeof(WDec), cudaMemcpyDeviceToHost));
  if (pulls && pull_cap > 0 && np > 0)
    PS_CK(h, cudaMemcpy(pulls, rt->pull, (np < pull_cap ? np : pull_cap) * sizeof(WPull), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_workers_abort(ps_server* h) {
  ps_worker_rt* rt = h->wrt;
  if (!rt) return PS_OK;
  // separate streams: the worker streams may be blocked; raise every flag
  int one = 1;
  unsigned ones = 1u;
  {
    DevGuardW g(h->dev);
    cudaStream_t st;
    PS_CK(h, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaError_t e = cudaMemcpyAsync(&rt->c->aborted, &one, sizeof(int), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e) return ps_cuda_fail(h, e, "ps_workers_abort");
  }
  for (auto& b : rt->bind) {
    if (!b.go) continue;
    DevGuardW g(b.dev);
    cudaStream_t st;
    PS_CK(h, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaError_t e = cudaMemcpyAsync(b.go, &ones, sizeof(unsigned), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (e) return ps_cuda_fail(h, e, "ps_workers_abort");
  }
  return PS_OK;
}

}  // extern "C"
