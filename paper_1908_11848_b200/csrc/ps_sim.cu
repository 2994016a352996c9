// ps_sim.cu -- the device-resident parameter-server run loop.
//
// One cooperative persistent kernel executes a whole simulated cluster run
// (simnet.py:127-201) with the host out of the loop:
//
//   * CTA 0 is a single CONTROL warp. It runs the reference's event loop --
//     (time, seq) ordered events, one in flight per worker, same-instant push
//     aggregation (simnet.py:167-201: apply every gradient of the group in seq
//     order, then decide each) -- and every gate decision, with all tables in
//     registers: replicated scalars for P <= 8 (ctl_regs.cuh), one worker per
//     lane for P <= 32 (ctl_lanes.cuh), shared memory beyond (CtlState). It
//     appends TraceEntry rows (trace.py:28-37) and emits data operations into
//     an HBM op log as self-tagged 64-bit words. It never waits for the data
//     side; it is the run's critical path (~3 us per worker iteration).
//   * every other warp is a DATA warp that owns a fixed contiguous slice of
//     the parameter vector and replays the op log in order over its slice:
//       PULL  (handle_pull, server.py:84-91)  copy the weights into the
//             worker's staging replica -- the snapshot is materialized at
//             PULL_ARRIVE, adopted at PULL_RETURN (simnet.py:135-138, :156-159);
//       GRAD  (WorkerState.begin_iteration, engine.py:263-272) produce the
//             worker's update (quadratic bowl g = w_local - c, engine.py:46-60,
//             or a resident synthetic N(0,1) buffer) and contribute to its
//             whole-vector finiteness flag;
//       APPLY (apply_gradient, server.py:58-69) wait until every data warp
//             has flagged that update, then w = w - lr*g on the slice, or skip
//             it when any element was non-finite (rejected, counted).
//     Every element is touched by exactly one thread in op order, so per-element
//     update order equals the global push order with no atomics on weights and
//     no grid barrier; the only cross-warp dependency is the per-update
//     finiteness count.
#include <cuda_runtime.h>
#include <type_traits>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gate.cuh"
#include "ctl_lanes.cuh"
#include "ctl_regs.cuh"
#include "server.h"

using namespace dssp;

namespace {

enum OpType : int32_t { OP_PULL = 1, OP_GRAD = 2, OP_APPLY = 3, OP_END = 4 };

// One op is a single 64-bit word, written once per run with one relaxed store
// and self-validating through its run tag, so the control warp never fences
// and the data warps never read a separate "produced" counter:
//   [0,16) run tag   [16,19) type   [19,26) worker   [26,34) buf   [34,64) slot
// buf -- PULL: staging replica; GRAD: active replica (bowl) or synthetic index;
//        APPLY: synthetic index.  slot -- update id (GRAD/APPLY).
typedef unsigned long long Op;
__host__ __device__ __forceinline__ Op op_pack(unsigned tag, int type, int w, int buf, long long slot) {
  return (unsigned long long)(tag & 0xffffu) | ((unsigned long long)(type & 7) << 16) |
         ((unsigned long long)(w & 127) << 19) | ((unsigned long long)(buf & 255) << 26) |
         ((unsigned long long)slot << 34);
}
__device__ __forceinline__ int op_type(Op o) { return (int)((o >> 16) & 7); }
__device__ __forceinline__ int op_worker(Op o) { return (int)((o >> 19) & 127); }
__device__ __forceinline__ int op_buf(Op o) { return (int)((o >> 26) & 255); }
__device__ __forceinline__ long long op_slot(Op o) { return (long long)(o >> 34); }
__device__ __forceinline__ unsigned op_tag(Op o) { return (unsigned)(o & 0xffffu); }

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_s32(const int* p) {
  return p ? *reinterpret_cast<const volatile int*>(p) : 0;
}

struct ReplayCall {  // ps_replay_call
  double now;
  int kind;    // kCallPull / kCallApply / kCallDecide
  int worker;
};
constexpr int kCallPull = 0, kCallApply = 1, kCallDecide = 2;

struct SimOut {
  long long events, pushes, trace_rows, applied, rejected;
  unsigned long long unfinished;
  int status, diverged_worker;
  unsigned long long t_start, t_control_done, t_data_done;  // %globaltimer ns
  unsigned long long validated;  // replay: (calls validated by the gate << 1) | done
  unsigned long long dvalid;     // replay: (data-call descriptors published << 1) | done
};

struct SimArgs {
  int P, budget, grad_kind, n_synth, loss_every, record_trace, reset_gate;
  long long nv, dpad, max_events, trace_cap, loss_cap, ops_cap;
  double comm_delay;
  float lr;
  float* W;
  float* rep;
  float* gbuf;
  const float* center;
  const float* synth;
  const double* ctime;
  Op* ops;
  unsigned* gword;   // per update: data CTAs done (low 16 bits) | non-finite CTAs << 16
  ps_trace_row* trace;
  double* losses;
  Ctrl* ctrl;
  SimOut* out;
  unsigned n_data_warps;
  unsigned long long timeout_ns;
  long long base_version;
  int mode;                   // 0: simulated run, 1: replay of a recorded call stream,
                              // 2: free-running (events fire on the wall clock)
  double time_scale;          // mode 2: wall-clock seconds per schedule second
  unsigned long long deadline_ns;  // mode 2: watchdog (deadline_guard, runner.py:294-298)
  const int* abort_flag;      // mode 2: host-set abort (ThreadedRun.abort, runner.py:110-111)
  const struct ReplayCall* calls;
  long long n_calls;
  long long* decisions;       // replay: (released << 8) | outcome per decide
  unsigned tag;
  unsigned n_ctas;
  int gate_scan;              // replay: the scan gate when eligible (PS_REPLAY_GATE_SCAN, default on)
  unsigned long long* dstream;  // replay: the gate's data-call descriptors (DataEmit)
  long long n_data;           // replay: pulls + applies in the stream (upper bound of dstream)
  unsigned long long* pred;    // replay: controller results by call (predict_warp_replay)
  int pred_ahead;             // replay: the gate reads them (PS_REPLAY_CTL_AHEAD, default on)
};

// The replay's data calls as a descriptor stream. A second warp of CTA 0 --
// the emitter, beside the gate warp -- numbers the pulls and applies (apply:
// resident update k % n_synthetic of the worker's k-th apply; pull: replica
// (k + 1) % 2 of its k-th pull) and compacts them into one 64-bit word per
// data call: run tag << 32 | pull << 16 | worker << 8 | buffer. It runs ahead
// of the gate, and follows the gate's validated-calls watermark with a
// data-call watermark (count << 1 | done), so the data never passes a
// protocol error. The register-slice data warps read that stream instead of
// every call and numbering it themselves: decides never reach them and the
// per-call bookkeeping is done once, not once per data warp, and off the
// gate's critical path. The tag makes every word self-validating (a reader
// re-polls a word from an older run), so nobody needs an acquire -- which
// would invalidate the L1 where the data warps keep the resident updates.
__device__ void emit_warp_replay(const SimArgs& a) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const long long n = a.n_calls;
  const long long nchunks = (n + 31) / 32;
  const unsigned long long t0 = globaltimer_ns();
  int sidx_lo = 0, sidx_hi = 0, stg_lo = 0, stg_hi = 0;  // lane q: workers q and q + 32
  long long count = 0, published = -1;
  // per call chunk k: data calls before the end of k (dprefix) and its mask
  // (dmask); written and read by this warp only
  long long* dprefix = reinterpret_cast<long long*>(a.dstream + a.n_data + 32);
  unsigned* dmask = reinterpret_cast<unsigned*>(dprefix + nchunks + 2);
  bool done = false;
  auto try_publish = [&](long long emitted) {
    unsigned long long v = 0;
    if (lane == 0) v = ld_relaxed_u64(&a.out->validated);
    v = __shfl_sync(kFull, v, 0);
    const long long vc = (long long)(v >> 1);
    const bool gdone = v & 1ull;
    long long dc;
    bool final_ = false;
    if (gdone && vc <= emitted * 32) {  // the gate is done and we have emitted past its end
      const long long kk = vc / 32, r = vc % 32;
      dc = (kk > 0 ? dprefix[kk - 1] : 0) + (r ? __popc(dmask[kk] & ((1u << r) - 1u)) : 0);
      final_ = true;
    } else {
      const long long kk = (vc / 32 < emitted ? vc / 32 : emitted);  // whole chunks validated and emitted
      dc = kk > 0 ? dprefix[kk - 1] : 0;
    }
    if (final_ || dc > published) {
      if (lane == 0) st_relaxed_u64(&a.out->dvalid, ((unsigned long long)dc << 1) | (final_ ? 1ull : 0ull));
      published = dc;
    }
    done = final_;
  };
  int2 nxt = make_int2(-1, 0);
  if (lane < n) nxt = *reinterpret_cast<const int2*>(&a.calls[lane].kind);
  for (long long k = 0; k < nchunks && !done; ++k) {
    const int kind = nxt.x, worker = nxt.y;
    const long long i1 = (k + 1) * 32 + lane;
    nxt = i1 < n ? *reinterpret_cast<const int2*>(&a.calls[i1].kind) : make_int2(-1, 0);
    const bool okw = worker >= 0 && worker < a.P;
    const bool isa = okw && kind == kCallApply, isp = okw && kind == kCallPull;
    const unsigned md = __ballot_sync(kFull, isa || isp);
    if (md) {
      const unsigned ma = __ballot_sync(kFull, isa);
      const unsigned peers = __match_any_sync(kFull, isa ? worker : isp ? 64 + worker : 128 + lane);
      const int rank = __popc(peers & lt);
      const int wq = worker & 31;
      const int s_lo = __shfl_sync(kFull, sidx_lo, wq), s_hi = __shfl_sync(kFull, sidx_hi, wq);
      const int g_lo = __shfl_sync(kFull, stg_lo, wq), g_hi = __shfl_sync(kFull, stg_hi, wq);
      int buf = 0;
      if (isa) buf = ((worker < 32 ? s_lo : s_hi) + rank) % a.n_synth;
      if (isp) buf = (worker < 32 ? g_lo : g_hi) ^ ((rank + 1) & 1);
      if (isa || isp)
        st_relaxed_u64(a.dstream + count + __popc(md & lt),
                       ((unsigned long long)a.tag << 32) | (isp ? 1u << 16 : 0u) | ((unsigned)worker << 8) | (unsigned)buf);
      // per-worker counters forward: the last lane of each (worker, kind) group
      // tells the worker's home lane through a shuffle round per group leader
      for (unsigned lead = __ballot_sync(kFull, (isa || isp) && rank == __popc(peers) - 1); lead; lead &= lead - 1) {
        const int l = __ffs(lead) - 1;
        const int wl = __shfl_sync(kFull, worker, l);
        const int cnt = __shfl_sync(kFull, __popc(peers), l);
        const bool app = (ma >> l) & 1u;
        if (lane == (wl & 31)) {
          if (app) { if (wl < 32) sidx_lo += cnt; else sidx_hi += cnt; }
          else { if (wl < 32) stg_lo ^= cnt & 1; else stg_hi ^= cnt & 1; }
        }
      }
    }
    count += __popc(md);
    if (lane == 0) { dmask[k] = md; dprefix[k] = count; }
    __syncwarp();
    try_publish(k + 1);
  }
  while (!done) {
    if (globaltimer_ns() - t0 > a.timeout_ns) break;
    __nanosleep(64);
    try_publish(nchunks);
  }
}

// Cycle accounting of the control warp, compiled in with -DPS_SIM_PROFILE.
#ifdef PS_SIM_PROFILE
#define PROF_DECL() long long c_pop = 0, c_push = 0, c_other = 0, c_gate = 0
#define PROF_MARK(t) const long long t = clock64()
#define PROF_ADD(acc, t) acc += clock64() - (t)
#define PROF_PRINT()                                                                         \
  if ((threadIdx.x & 31) == 0)                                                               \
  printf("PROF P=%d events=%lld pop=%lld push=%lld (gate=%lld) other=%lld\n", a.P, processed, \
         c_pop, c_push, c_gate, c_other)
#else
#define PROF_DECL() do {} while (0)
#define PROF_MARK(t) do {} while (0)
#define PROF_ADD(acc, t) do {} while (0)
#define PROF_PRINT() do {} while (0)
#endif

constexpr int kSimThreads = 256;
constexpr int kMaxP = PS_MAX_WORKERS;
constexpr int kLaneP = 32;  // one worker per control-warp lane up to this many workers

struct CtlState {
  ps_gate_state gate;
  double ev_time[kMaxP];
  long long ev_seq[kMaxP];
  int ev_kind[kMaxP];         // -1: no event in flight for this worker
  int iterations[kMaxP];
  int active[kMaxP];          // replica the worker computes on
  int staged[kMaxP];          // replica the last pull wrote
  int grad_slot[kMaxP];
  int synth_idx[kMaxP];
  int finished[kMaxP];
  int group[kMaxP];           // current push group, in seq order
  int group_len, group_pos;
  double group_at;
  long long seq, processed, n_ops, n_trace, pushes, next_slot;
  int status;
};

__device__ __forceinline__ void ctl_trace(const SimArgs& a, CtlState& s, double t, int w, int kind,
                                          int decision, unsigned long long released) {
  if (a.record_trace && s.n_trace < a.trace_cap) {
    ps_trace_row r;
    r.time = t;
    r.worker = w;
    r.kind = kind;
    r.count = s.gate.clocks[w];
    r.decision = decision;
    r._pad = 0;
    r.released = released;
    a.trace[s.n_trace] = r;
  }
  s.n_trace += 1;
}

__device__ __forceinline__ void ctl_schedule(CtlState& s, double at, int kind, int w) {
  s.ev_time[w] = at;
  s.ev_seq[w] = s.seq++;
  s.ev_kind[w] = kind;
}

__device__ __forceinline__ void ctl_emit(const SimArgs& a, CtlState& s, int type, int w, int buf,
                                         long long slot) {
  st_relaxed_u64(a.ops + s.n_ops, op_pack(a.tag, type, w, buf, slot));
  s.n_ops += 1;
}

// Lane 0 only. Advances the event loop until a decision is needed (returns 1,
// *p/*now set) or the run is over (returns 2).
__device__ int ctl_advance(const SimArgs& a, CtlState& s, int* p, double* now) {
  for (;;) {
    if (s.group_pos < s.group_len) {
      *p = s.group[s.group_pos];
      *now = s.group_at;
      return 1;
    }
    if (s.status != PS_OK) return 2;
    // pop the (time, seq)-minimum event
    int w = -1;
    for (int q = 0; q < a.P; ++q) {
      if (s.ev_kind[q] < 0) continue;
      if (w < 0 || s.ev_time[q] < s.ev_time[w] ||
          (s.ev_time[q] == s.ev_time[w] && s.ev_seq[q] < s.ev_seq[w]))
        w = q;
    }
    if (w < 0) return 2;
    if (a.max_events > 0 && s.processed >= a.max_events) {
      s.status = PS_E_BUDGET;
      return 2;
    }
    const double at = s.ev_time[w];
    const int kind = s.ev_kind[w];
    s.ev_kind[w] = -1;
    s.processed += 1;
    if (kind == PS_EV_PULL_ARRIVE) {
      const int st = 1 - s.active[w];
      ctl_emit(a, s, OP_PULL, w, st, 0);
      s.staged[w] = st;
      ctl_trace(a, s, at, w, kind, -1, 0);
      ctl_schedule(s, at + a.comm_delay, PS_EV_PULL_RETURN, w);
    } else if (kind == PS_EV_PULL_RETURN) {
      s.active[w] = s.staged[w];  // adopt (simnet.py:156-165)
      ctl_trace(a, s, at, w, kind, -1, 0);
      if (s.iterations[w] < a.budget) {
        ctl_schedule(s, at + a.ctime[(long long)w * a.budget + s.iterations[w]], PS_EV_COMPUTE_DONE, w);
      } else {
        s.finished[w] = 1;
      }
    } else if (kind == PS_EV_COMPUTE_DONE) {
      s.iterations[w] += 1;
      const int slot = (int)s.next_slot++;
      s.grad_slot[w] = slot;
      const int buf = a.grad_kind == PS_GRAD_BOWL ? s.active[w] : (s.synth_idx[w] % a.n_synth);
      ctl_emit(a, s, OP_GRAD, w, buf, slot);
      ctl_trace(a, s, at, w, kind, -1, 0);
      ctl_schedule(s, at + a.comm_delay, PS_EV_PUSH_ARRIVE, w);
    } else if (kind == PS_EV_GRANT_DELIVER) {
      ctl_trace(a, s, at, w, kind, -1, 0);
      ctl_schedule(s, at + a.comm_delay, PS_EV_PULL_ARRIVE, w);
    } else {
      // PUSH_ARRIVE: aggregate every push queued at the same instant
      // (simnet.py:167-182), ordered by seq, the popped one first.
      int n = 0;
      s.group[n++] = w;
      for (int q = 0; q < a.P; ++q) {
        if (s.ev_kind[q] == PS_EV_PUSH_ARRIVE && s.ev_time[q] == at) {
          int i = n++;
          while (i > 1 && s.ev_seq[s.group[i - 1]] > s.ev_seq[q]) {
            s.group[i] = s.group[i - 1];
            --i;
          }
          s.group[i] = q;
          s.ev_kind[q] = -1;
        }
      }
      for (int i = 0; i < n; ++i) {
        const int m = s.group[i];
        const int buf = a.grad_kind == PS_GRAD_BOWL ? 0 : (s.synth_idx[m] % a.n_synth);
        ctl_emit(a, s, OP_APPLY, m, buf, s.grad_slot[m]);
        s.synth_idx[m] += 1;
      }
      s.group_len = n;
      s.group_pos = 0;
      s.group_at = at;
    }
  }
}

__device__ void ctl_after_decision(const SimArgs& a, CtlState& s, const GateResult& r) {
  const int m = s.group[s.group_pos++];
  const double at = s.group_at;
  s.pushes += 1;
  if (r.status != PS_OK) {
    s.status = r.status;
    s.group_len = s.group_pos;
    return;
  }
  ctl_trace(a, s, at, m, PS_EV_PUSH_ARRIVE, r.outcome, r.released);
  if (r.outcome == 0) {
    ctl_schedule(s, at + a.comm_delay, PS_EV_GRANT_DELIVER, m);
    for (int q = 0; q < a.P; ++q)
      if ((r.released >> q) & 1ull) ctl_schedule(s, at + a.comm_delay, PS_EV_GRANT_DELIVER, q);
  }
}

__device__ void control_warp(const SimArgs& a, CtlState& s) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    s.gate = a.ctrl->gate;
    if (a.reset_gate) {
      for (int q = 0; q < kMaxP; ++q) {
        s.gate.clocks[q] = 0; s.gate.latest[q] = 0.0; s.gate.previous[q] = 0.0;
        s.gate.populated[q] = 0; s.gate.credits[q] = 0;
      }
      s.gate.deferred = 0ull;
    }
    for (int q = 0; q < kMaxP; ++q) {
      s.ev_kind[q] = -1;
      s.iterations[q] = 0;
      s.active[q] = 0;
      s.staged[q] = 0;
      s.grad_slot[q] = 0;
      s.synth_idx[q] = 0;
      s.finished[q] = 0;
    }
    s.group_len = s.group_pos = 0;
    s.seq = s.processed = s.n_ops = s.n_trace = s.pushes = s.next_slot = 0;
    s.status = PS_OK;
    for (int q = 0; q < a.P; ++q) ctl_schedule(s, a.comm_delay, PS_EV_PULL_ARRIVE, q);
  }
  if (lane == 0) a.out->t_start = globaltimer_ns();
  __syncwarp();
  for (;;) {
    int cmd = 0, p = 0;
    double now = 0.0;
    if (lane == 0) cmd = ctl_advance(a, s, &p, &now);
    cmd = __shfl_sync(kFull, cmd, 0);
    if (cmd == 2) break;
    p = __shfl_sync(kFull, p, 0);
    now = __shfl_sync(kFull, now, 0);
    const GateResult r = gate_on_push(&s.gate, p, now);
    if (lane == 0) ctl_after_decision(a, s, r);
    __syncwarp();
  }
  if (lane == 0) {
    ctl_emit(a, s, OP_END, 0, 0, 0);
    a.out->t_control_done = globaltimer_ns();
    unsigned long long unfinished = 0;
    for (int q = 0; q < a.P; ++q)
      if (!s.finished[q]) unfinished |= 1ull << q;
    // gate tables back to the control block; version/rejected belong to the data side
    const long long v = a.ctrl->gate.version, rj = a.ctrl->gate.rejected;
    a.ctrl->gate = s.gate;
    a.ctrl->gate.version = v;
    a.ctrl->gate.rejected = rj;
    a.out->events = s.processed;
    a.out->pushes = s.pushes;
    a.out->trace_rows = s.n_trace;
    a.out->unfinished = s.status == PS_OK ? unfinished : 0ull;
    if (s.status != PS_OK) atomicCAS(&a.out->status, PS_OK, s.status);
  }
}

// Register-resident control warp for P <= PM (see ctl_regs.cuh): all lanes run
// the identical event loop; lane 0 alone writes trace rows and op words.
template <int PM>
__device__ void control_warp_regs(const SimArgs& a) {
  const int lane = threadIdx.x & 31;
  const bool w0 = lane == 0;
  const int P = a.P, budget = a.budget, nsyn = a.n_synth;
  const bool bowl = a.grad_kind == PS_GRAD_BOWL;
  const double comm = a.comm_delay;
  const unsigned tag = a.tag;
  Op* const ops = a.ops;
  ps_trace_row* const trace = a.trace;
  const long long trace_cap = a.record_trace ? a.trace_cap : 0;
  RegGate<PM> g;
  g.load(a.ctrl->gate, a.reset_gate != 0);
  double ev_time[PM], nct[PM];
  int ev_seq[PM], ev_kind[PM], iters[PM], active[PM], staged[PM], gslot[PM], sidx[PM];
#pragma unroll
  for (int q = 0; q < PM; ++q) {
    ev_kind[q] = -1; iters[q] = 0; active[q] = 0; staged[q] = 0; gslot[q] = 0; sidx[q] = 0;
    ev_time[q] = 0.0; ev_seq[q] = 0;
    nct[q] = (q < P && budget > 0) ? a.ctime[(long long)q * budget] : 0.0;  // next compute draw
  }
  unsigned finished = 0;
  int seq = 0, status = PS_OK;
  long long processed = 0, n_ops = 0, n_trace = 0, pushes = 0, next_slot = 0;
  double pend_v = 0.0;  // a compute draw in flight to nct[pend_w]
  int pend_w = -1;
  auto emit = [&](int type, int w, int buf, long long slot) {
    if (w0) st_relaxed_u64(ops + n_ops, op_pack(tag, type, w, buf, slot));
    n_ops += 1;
  };
  auto trace_row = [&](double t, int w, int kind, int decision, unsigned long long released) {
    if (w0 && n_trace < trace_cap) {
      ps_trace_row r;
      r.time = t; r.worker = w; r.kind = kind; r.count = rget<PM>(g.clocks, w);
      r.decision = decision; r._pad = 0; r.released = released;
      trace[n_trace] = r;
    }
    n_trace += 1;
  };
  auto schedule = [&](double at, int kind, int w) {
#pragma unroll
    for (int q = 0; q < PM; ++q)
      if (q == w) { ev_time[q] = at; ev_seq[q] = seq; ev_kind[q] = kind; }
    seq += 1;
  };
#pragma unroll
  for (int q = 0; q < PM; ++q)
    if (q < P) schedule(comm, PS_EV_PULL_ARRIVE, q);
  if (w0) a.out->t_start = globaltimer_ns();
  const bool realtime = a.mode == 2;
  const double ns_per_s = 1e9 * a.time_scale;  // config seconds -> wall-clock ns
  // lanes run the loop redundantly, so every clock/flag read is lane 0's
  const unsigned long long t_real0 = __shfl_sync(0xffffffffu, globaltimer_ns(), 0);
  const unsigned long long deadline = t_real0 + a.deadline_ns;
  bool aborted = false;
  PROF_DECL();
  for (;;) {
    PROF_MARK(t_a);
    // pop the (time, seq)-minimum event
    int w = -1;
    double bt = 0.0;
    int bs = 0;
#pragma unroll
    for (int q = 0; q < PM; ++q) {
      if (q < P && ev_kind[q] >= 0 &&
          (w < 0 || ev_time[q] < bt || (ev_time[q] == bt && ev_seq[q] < bs))) {
        w = q; bt = ev_time[q]; bs = ev_seq[q];
      }
    }
    if (w < 0) break;
    PROF_MARK(t_b);
    PROF_ADD(c_pop, t_a);
    if (a.max_events > 0 && processed >= a.max_events) { status = PS_E_BUDGET; break; }
    double at = bt;
    if (realtime) {
      // free-running (runner.py:168-291): the event fires when the wall clock
      // reaches it and carries the time it actually fired at
      // (the abort flag lives in host memory: poll it while idle and every
      // 64 events, not on every event)
      const unsigned long long due = t_real0 + (unsigned long long)(bt * ns_per_s);
      unsigned long long nw;
      bool stop = (processed & 63) == 0 && ld_volatile_s32(a.abort_flag);
      while (!stop && (nw = globaltimer_ns()) < due) stop = nw > deadline || ld_volatile_s32(a.abort_flag);
      nw = __shfl_sync(0xffffffffu, globaltimer_ns(), 0);
      stop = __shfl_sync(0xffffffffu, stop, 0);
      if (stop || nw > deadline) { aborted = true; break; }
      at = (double)(nw - t_real0) / ns_per_s;
    }
    const int kind = rget<PM>(ev_kind, w);
    rset<PM>(ev_kind, w, -1);
    processed += 1;
    if (kind == PS_EV_PULL_ARRIVE) {
      const int st = 1 - rget<PM>(active, w);
      emit(OP_PULL, w, st, 0);
      rset<PM>(staged, w, st);
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PULL_RETURN, w);
    } else if (kind == PS_EV_PULL_RETURN) {
      rset<PM>(active, w, rget<PM>(staged, w));  // adopt (simnet.py:156-165)
      trace_row(at, w, kind, -1, 0);
      if (pend_w >= 0) { rset<PM>(nct, pend_w, pend_v); pend_w = -1; }
      if (rget<PM>(iters, w) < budget) schedule(at + rget<PM>(nct, w), PS_EV_COMPUTE_DONE, w);
      else finished |= 1u << w;
    } else if (kind == PS_EV_COMPUTE_DONE) {
      const int it = rget<PM>(iters, w) + 1;
      rset<PM>(iters, w, it);
      // the next draw: loaded now, written into the table only when a later
      // event needs it, so the load's latency hides behind those events
      if (pend_w >= 0) rset<PM>(nct, pend_w, pend_v);
      pend_w = -1;
      if (it < budget) { pend_v = a.ctime[(long long)w * budget + it]; pend_w = w; }
      const long long slot = next_slot++;
      rset<PM>(gslot, w, (int)slot);
      emit(OP_GRAD, w, bowl ? rget<PM>(active, w) : rget<PM>(sidx, w) % nsyn, slot);
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PUSH_ARRIVE, w);
    } else if (kind == PS_EV_GRANT_DELIVER) {
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PULL_ARRIVE, w);
    } else {
      // PUSH_ARRIVE: every push queued at the same instant joins the group
      // (simnet.py:167-182); the popped one first, the rest by seq. Free-
      // running, each push is its own apply -> decide under the server lock
      // (runner.py:226-249).
      unsigned rest = 0;
      if (!realtime) {
#pragma unroll
        for (int q = 0; q < PM; ++q)
          if (q < P && ev_kind[q] == PS_EV_PUSH_ARRIVE && ev_time[q] == at) {
            rest |= 1u << q;
            ev_kind[q] = -1;
          }
      }
      // the group's order as a packed list of 4-bit worker ids: the loops
      // below run n times (usually once) instead of being unrolled PM times
      // around an inlined gate
      unsigned long long order = (unsigned long long)w;
      int n = 1;
      while (rest) {
        int m = -1, ms = 0;
#pragma unroll
        for (int q = 0; q < PM; ++q)
          if (((rest >> q) & 1u) && (m < 0 || ev_seq[q] < ms)) { m = q; ms = ev_seq[q]; }
        rest &= ~(1u << m);
        order |= (unsigned long long)m << (4 * n);
        n += 1;
      }
#pragma unroll 1
      for (int i = 0; i < n; ++i) {
        const int m = (int)((order >> (4 * i)) & 15ull);
        const int si = rget<PM>(sidx, m);
        emit(OP_APPLY, m, bowl ? 0 : si % nsyn, rget<PM>(gslot, m));
        rset<PM>(sidx, m, si + 1);
      }
#pragma unroll 1
      for (int i = 0; i < n && status == PS_OK; ++i) {
        const int m = (int)((order >> (4 * i)) & 15ull);
        PROF_MARK(t_g);
        const GateResult r = g.on_push(m, at);
        PROF_ADD(c_gate, t_g);
        pushes += 1;
        if (r.status != PS_OK) {
          status = r.status;
        } else {
          trace_row(at, m, PS_EV_PUSH_ARRIVE, r.outcome, r.released);
          if (r.outcome == 0) {
            schedule(at + comm, PS_EV_GRANT_DELIVER, m);
            for (unsigned long long rel = r.released; rel; rel &= rel - 1)
              schedule(at + comm, PS_EV_GRANT_DELIVER, __ffsll((long long)rel) - 1);
          }
        }
      }
      if (status != PS_OK) break;
    }
    PROF_ADD(kind == PS_EV_PUSH_ARRIVE ? c_push : c_other, t_b);
  }
  PROF_PRINT();
  emit(OP_END, 0, 0, 0);
  if (w0) {
    a.out->t_control_done = globaltimer_ns();
    unsigned long long unfinished = 0;
    for (int q = 0; q < P; ++q)
      if (!((finished >> q) & 1u)) unfinished |= 1ull << q;
    ps_gate_state& dst = a.ctrl->gate;
    if (a.reset_gate) {
      for (int q = 0; q < kMaxP; ++q) {
        dst.clocks[q] = 0; dst.latest[q] = 0.0; dst.previous[q] = 0.0;
        dst.populated[q] = 0; dst.credits[q] = 0;
      }
    }
    g.store(dst);
    a.out->events = processed;
    a.out->pushes = pushes;
    a.out->trace_rows = n_trace;
    // an aborted free-running run reports its stuck workers (runner.py:120-164)
    a.out->unfinished = (status == PS_OK || aborted) ? unfinished : 0ull;
    if (aborted) status = PS_E_TIMEOUT;
    if (status != PS_OK) atomicCAS(&a.out->status, PS_OK, status);
  }
}

// Control warp for P <= 32 (ctl_lanes.cuh): lane q owns worker q; the event
// loop is warp-uniform; lane 0 stores op words, lanes 0-4 one trace row each.
__device__ void control_warp_lanes(const SimArgs& a) {
  const int lane = threadIdx.x & 31;
  const int P = a.P, budget = a.budget, nsyn = a.n_synth;
  const bool bowl = a.grad_kind == PS_GRAD_BOWL;
  const bool mine = lane < P;
  const double comm = a.comm_delay;
  const unsigned tag = a.tag;
  Op* const ops = a.ops;
  unsigned long long* const trace = reinterpret_cast<unsigned long long*>(a.trace);
  const long long trace_cap = a.record_trace ? a.trace_cap : 0;
  LaneGate g;
  {
    const ps_gate_state& s = a.ctrl->gate;
    const bool z = a.reset_gate || !mine;
    g.paradigm = s.paradigm; g.P = P; g.s_lower = s.s_lower; g.r_max = s.r_max;
    g.threshold = s.threshold;
    g.deferred = a.reset_gate ? 0u : (unsigned)s.deferred;
    g.decisions = s.decisions;
    g.clock = z ? 0 : (int)s.clocks[lane];
    g.latest = z ? 0.0 : s.latest[lane];
    g.previous = z ? 0.0 : s.previous[lane];
    g.populated = z ? 0 : (int)s.populated[lane];
    g.credits = z ? 0 : (int)s.credits[lane];
  }
  // this lane's worker
  double ev_time = 0.0;
  int ev_seq = 0x7fffffff, ev_kind = -1;
  int iters = 0, active = 0, staged = 0, gslot = 0, sidx = 0, order_i = 0;
  bool finished = false;
  double nct = (mine && budget > 0) ? a.ctime[(long long)lane * budget] : 0.0;  // next compute draw
  int seq = 0, status = PS_OK;
  long long processed = 0, n_ops = 0, n_trace = 0, pushes = 0, next_slot = 0;

  auto emit = [&](int type, int w, int buf, long long slot) {
    if (lane == 0) st_relaxed_u64(ops + n_ops, op_pack(tag, type, w, buf, slot));
    n_ops += 1;
  };
  // ps_trace_row as five 8-byte words, one per lane 0..4, one store
  auto trace_row = [&](double t, int w, int kind, int decision, unsigned long long released) {
    if (n_trace < trace_cap) {
      const long long count = from_lane(g.clock, w);
      unsigned long long v = 0;
      if (lane == 0) v = dbits(t);
      else if (lane == 1) v = ((unsigned long long)(unsigned)kind << 32) | (unsigned)w;
      else if (lane == 2) v = (unsigned long long)count;
      else if (lane == 3) v = (unsigned)decision;
      else if (lane == 4) v = released;
      if (lane < 5) trace[n_trace * 5 + lane] = v;
    }
    n_trace += 1;
  };
  auto schedule = [&](double at, int kind, int w) {
    if (lane == w) { ev_time = at; ev_seq = seq; ev_kind = kind; }
    seq += 1;
  };
  for (int q = 0; q < P; ++q) schedule(comm, PS_EV_PULL_ARRIVE, q);
  if (lane == 0) a.out->t_start = globaltimer_ns();
  // free-running (mode 2): see control_warp_regs
  const bool realtime = a.mode == 2;
  const double ns_per_s = 1e9 * a.time_scale;
  const unsigned long long t_real0 = __shfl_sync(kFull, globaltimer_ns(), 0);
  const unsigned long long deadline = t_real0 + a.deadline_ns;
  bool aborted = false;
  for (;;) {
    // pop the (time, seq)-minimum event: time bits, then seq
    const bool cand = mine && ev_kind >= 0;
    const unsigned long long tb = dbits(ev_time);
    const unsigned hi = __reduce_min_sync(kFull, cand ? (unsigned)(tb >> 32) : 0xffffffffu);
    const bool c1 = cand && (unsigned)(tb >> 32) == hi;
    const unsigned lo = __reduce_min_sync(kFull, c1 ? (unsigned)tb : 0xffffffffu);
    const bool c2 = c1 && (unsigned)tb == lo;
    const int ms = __reduce_min_sync(kFull, c2 ? ev_seq : 0x7fffffff);
    const unsigned who = __ballot_sync(kFull, c2 && ev_seq == ms);
    if (!who) break;
    const int w = __ffs(who) - 1;
    if (a.max_events > 0 && processed >= a.max_events) { status = PS_E_BUDGET; break; }
    double at = from_lane(ev_time, w);
    if (realtime) {
      const unsigned long long due = t_real0 + (unsigned long long)(at * ns_per_s);
      unsigned long long nw;
      bool stop = (processed & 63) == 0 && ld_volatile_s32(a.abort_flag);
      while (!stop && (nw = globaltimer_ns()) < due) stop = nw > deadline || ld_volatile_s32(a.abort_flag);
      nw = __shfl_sync(kFull, globaltimer_ns(), 0);
      stop = __shfl_sync(kFull, stop, 0);
      if (stop || nw > deadline) { aborted = true; break; }
      at = (double)(nw - t_real0) / ns_per_s;
    }
    const int kind = from_lane(ev_kind, w);
    if (lane == w) ev_kind = -1;
    processed += 1;
    if (kind == PS_EV_PULL_ARRIVE) {
      const int st = 1 - from_lane(active, w);
      emit(OP_PULL, w, st, 0);
      if (lane == w) staged = st;
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PULL_RETURN, w);
    } else if (kind == PS_EV_PULL_RETURN) {
      if (lane == w) active = staged;  // adopt (simnet.py:156-165)
      trace_row(at, w, kind, -1, 0);
      if (from_lane(iters, w) < budget) schedule(at + from_lane(nct, w), PS_EV_COMPUTE_DONE, w);
      else if (lane == w) finished = true;
    } else if (kind == PS_EV_COMPUTE_DONE) {
      if (lane == w) {
        iters += 1;
        if (iters < budget) nct = a.ctime[(long long)w * budget + iters];  // prefetch the next draw
        gslot = (int)next_slot;
      }
      const long long slot = next_slot++;
      emit(OP_GRAD, w, bowl ? from_lane(active, w) : from_lane(sidx, w) % nsyn, slot);
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PUSH_ARRIVE, w);
    } else if (kind == PS_EV_GRANT_DELIVER) {
      trace_row(at, w, kind, -1, 0);
      schedule(at + comm, PS_EV_PULL_ARRIVE, w);
    } else {
      // PUSH_ARRIVE: every push queued at the same instant joins the group
      // (simnet.py:167-182); the popped one first, the rest by seq.
      const bool join = !realtime && mine && ev_kind == PS_EV_PUSH_ARRIVE && dbits(ev_time) == dbits(at);
      unsigned rest = __ballot_sync(kFull, join);
      if (join) ev_kind = -1;
      int n = 1;
      if (lane == 0) order_i = w;
      while (rest) {
        const int sm = __reduce_min_sync(kFull, ((rest >> lane) & 1u) ? ev_seq : 0x7fffffff);
        const int m = __ffs(__ballot_sync(kFull, ((rest >> lane) & 1u) && ev_seq == sm)) - 1;
        if (lane == n) order_i = m;
        rest &= ~(1u << m);
        n += 1;
      }
      for (int i = 0; i < n; ++i) {
        const int m = from_lane(order_i, i);
        emit(OP_APPLY, m, bowl ? 0 : from_lane(sidx, m) % nsyn, from_lane(gslot, m));
        if (lane == m) sidx += 1;
      }
      for (int i = 0; i < n && status == PS_OK; ++i) {
        const int m = from_lane(order_i, i);
        const GateResult r = g.on_push(lane, m, at);
        pushes += 1;
        if (r.status != PS_OK) { status = r.status; break; }
        trace_row(at, m, PS_EV_PUSH_ARRIVE, r.outcome, r.released);
        if (r.outcome == 0) {
          schedule(at + comm, PS_EV_GRANT_DELIVER, m);
          for (unsigned rel = (unsigned)r.released; rel; rel &= rel - 1)
            schedule(at + comm, PS_EV_GRANT_DELIVER, __ffs(rel) - 1);
        }
      }
      if (status != PS_OK) break;
    }
  }
  emit(OP_END, 0, 0, 0);
  const unsigned done = __ballot_sync(kFull, mine && finished);
  ps_gate_state& dst = a.ctrl->gate;
  if (mine) {
    dst.clocks[lane] = g.clock; dst.latest[lane] = g.latest; dst.previous[lane] = g.previous;
    dst.populated[lane] = g.populated; dst.credits[lane] = g.credits;
  }
  if (lane == 0) {
    a.out->t_control_done = globaltimer_ns();
    const unsigned all = P == 32 ? 0xffffffffu : ((1u << P) - 1u);
    dst.deferred = g.deferred;
    dst.decisions = g.decisions;
    a.out->events = processed;
    a.out->pushes = pushes;
    a.out->trace_rows = n_trace;
    a.out->unfinished = (status == PS_OK || aborted) ? (unsigned long long)(all & ~done) : 0ull;
    if (aborted) status = PS_E_TIMEOUT;
    if (status != PS_OK) atomicCAS(&a.out->status, PS_OK, status);
  }
}

// ---------------------------------------------------------------------------
// Replay mode: the server serving a recorded request stream.
//
// The kernel reads the reference's boundary call sequence (pull / apply /
// decide, in the order simnet.py:127-201 issues them) from HBM and executes
// it: every decide runs the gate on the device (gate warp), every pull and
// apply runs on the data warps' parameter slices in call order. It is what a
// parameter server does with the requests its workers send, without
// simulating the workers -- the same work the reference arm times on the CPU
// (ParameterServer.apply_gradient / decide_push / handle_pull). Decisions
// never feed the data (they only validate the protocol), so the two sides
// run concurrently, coupled by the gate's validated-calls watermark.
// ---------------------------------------------------------------------------

template <int PM>
struct ReplayGate {  // scalar register tables (ctl_regs.cuh), P <= PM
  RegGate<PM> g;
  __device__ __forceinline__ void load(const ps_gate_state& s, bool reset, ps_gate_state*) { g.load(s, reset); }
  __device__ __forceinline__ void store(ps_gate_state& d) { g.store(d); }
  __device__ __forceinline__ unsigned long long deferred_mask() const { return g.deferred; }
  __device__ __forceinline__ GateResult on_push(int p, double now) { return g.on_push(p, now); }
};

template <>
struct ReplayGate<0> {  // shared-memory tables (gate.cuh), any P <= 64
  ps_gate_state* s;
  __device__ __forceinline__ void load(const ps_gate_state& src, bool reset, ps_gate_state* smem) {
    s = smem;
    if ((threadIdx.x & 31) == 0) {
      *s = src;
      if (reset) {
        for (int q = 0; q < kMaxP; ++q) {
          s->clocks[q] = 0; s->latest[q] = 0.0; s->previous[q] = 0.0;
          s->populated[q] = 0; s->credits[q] = 0;
        }
        s->deferred = 0ull;
      }
    }
    __syncwarp();
  }
  __device__ __forceinline__ void store(ps_gate_state& d) {
    if ((threadIdx.x & 31) == 0) {
      const long long v = d.version, r = d.rejected;
      d = *s;
      d.version = v;
      d.rejected = r;
    }
  }
  __device__ __forceinline__ unsigned long long deferred_mask() const {
    return *reinterpret_cast<const volatile unsigned long long*>(&s->deferred);
  }
  __device__ __forceinline__ GateResult on_push(int p, double now) {
    const GateResult r = gate_on_push(s, p, now);
    __syncwarp();
    return r;
  }
};

// The replay gate as a scan (P <= PM <= 8, credits < 256).
//
// Of the gate's state only the credits and the deferred set depend on earlier
// OUTCOMES. Clocks, the two-deep push history and the populated counts follow
// from the sequence of pushes alone (every push counts and is recorded,
// policy.py:152-170), and so do min / max / slowest, the gap, the controller's
// inputs and the release-ready set of every decision (policy.py:60-73,
// 108-132, 197-206). Per 32-call chunk the warp therefore evaluates all of
// that for every DECIDE at once, one decision per lane (prefix counts over
// per-worker ballots, the controller per lane), and packs each into one word
// -- worker | class | minted credits | ready set. The serial part that is
// left is the credit / deferred recurrence of policy.py:172-206, ~20 scalar
// instructions per decision on packed registers. Decisions and final state are
// those of gate_on_push in call order; tests/test_gpu_replay.py and the
// golden decide streams hold both paths to the reference.
template <int PM>
__device__ bool gate_scan_eligible(const RegGate<PM>& g) {
  if (g.P > PM || PM > 8) return false;
  if (g.paradigm == PS_DSSP && g.s_lower + g.r_max > 255) return false;  // credits are 8-bit fields
#pragma unroll
  for (int q = 0; q < PM; ++q)
    if (g.credits[q] < 0 || g.credits[q] > 255) return false;
  return true;
}

template <int PM, bool PREDICT = false>
__device__ void gate_warp_replay_scan(const SimArgs& a, RegGate<PM>& g) {
  // credits, 8 bits per worker: one 32-bit word up to 4 workers
  using CW = typename std::conditional<(PM <= 4), unsigned, unsigned long long>::type;
  __shared__ unsigned sw[32];  // the chunk's packed decisions by slot
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
  const int P = g.P;
  const bool dssp = g.paradigm == PS_DSSP, asp = g.paradigm == PS_ASP;
  long long n_dec = 0, pushes = 0, valid = 0;
  int status = PS_OK;
  const long long n = a.n_calls;
  if (!PREDICT && lane == 0) a.out->t_start = globaltimer_ns();
  // PREDICT: this warp is the controller-ahead helper (see predict_warp_replay)
  const bool ahead = !PREDICT && a.pred_ahead && dssp;
  const unsigned long long t_pred = globaltimer_ns();
  CW cw = 0;
#pragma unroll
  for (int q = 0; q < PM; ++q) cw |= (CW)(q < P ? g.credits[q] : 0) << (8 * q);
  unsigned defm = (unsigned)g.deferred;
  auto load = [&](long long base, ReplayCall& c) {
    const long long i = base + lane;
    if (i < n) c = a.calls[i];
    else { c.now = 0.0; c.kind = -1; c.worker = 0; }
  };
  ReplayCall c, nx;
  load(0, c);
#ifdef PS_SIM_PROFILE
  long long pc_pre = 0, pc_dssp = 0, pc_ctl = 0, pc_scan = 0, pc_tail = 0, pc_t = clock64();
#define SCAN_STAMP(acc) do { const long long t_ = clock64(); acc += t_ - pc_t; pc_t = t_; } while (0)
#else
#define SCAN_STAMP(acc) do {} while (0)
#endif
  for (long long base = 0; base < n; base += 32) {
    load(base + 32, nx);
    // the helper's controller results for this chunk, in flight meanwhile
    unsigned long long pv = 0;
    if (ahead) pv = base + lane < n ? ld_relaxed_u64(a.pred + base + lane) : 0ull;
    const int m = n - base < 32 ? (int)(n - base) : 32;
    const unsigned live = m >= 32 ? kFull : ((1u << m) - 1u);
    const unsigned badw = __ballot_sync(kFull, lane < m && (c.worker < 0 || c.worker >= P));
    const int limit = badw ? __ffs(badw) - 1 : m;
    const unsigned below_limit = limit >= 32 ? kFull : ((1u << limit) - 1u);
    const unsigned md = __ballot_sync(kFull, c.kind == kCallDecide) & live & below_limit;
    const unsigned mp = __ballot_sync(kFull, c.kind == kCallPull) & live & below_limit;
    const bool is_dec = (md >> lane) & 1u;
    const int w = is_dec ? c.worker : 0;
    // ---- every decision of the chunk at once (one per lane) ----
    unsigned mq[PM];
#pragma unroll
    for (int q = 0; q < PM; ++q) mq[q] = __ballot_sync(kFull, is_dec && w == q);
    int cnt[PM];
    int low = 0x7fffffff, high = -0x7fffffff;
#pragma unroll
    for (int q = 0; q < PM; ++q) {
      cnt[q] = g.clocks[q] + __popc(mq[q] & le);
      if (q < P) { low = cnt[q] < low ? cnt[q] : low; high = cnt[q] > high ? cnt[q] : high; }
    }
    int sl = 0;
#pragma unroll
    for (int q = PM - 1; q >= 0; --q)
      if (q < P && cnt[q] == low) sl = q;
    const int count = rget<PM>(cnt, w);
    const int gap = count - low;
    unsigned ready = 0;
    if (!asp) {
#pragma unroll
      for (int q = 0; q < PM; ++q)
        if (q < P && cnt[q] - low <= g.threshold) ready |= 1u << q;
    }
    SCAN_STAMP(pc_pre);
    int cls = gap <= g.threshold ? 0 : 1;  // SSP / BSP: grant or defer
    int mint = 0;
    if (asp) cls = 0;
    if (dssp) {
      cls = gap <= g.s_lower ? 0 : (count < high ? 1 : 2);
      // the controller's inputs after this push is recorded
      const unsigned mine = rget<PM>(mq, w) & le;     // this worker's pushes up to here
      const unsigned prior = mine & lt;
      const double pp_in = __shfl_sync(kFull, c.now, prior ? 31 - __clz(prior) : lane);
      const double pp = prior ? pp_in : rget<PM>(g.latest, w);
      const unsigned msl = rget<PM>(mq, sl) & le;
      const int l1 = msl ? 31 - __clz(msl) : lane;
      const unsigned rest = msl & ~(1u << (l1 & 31));
      const double ls_in = __shfl_sync(kFull, c.now, l1);
      const double ps_in = __shfl_sync(kFull, c.now, rest ? 31 - __clz(rest) : lane);
      const double ls = msl ? ls_in : rget<PM>(g.latest, sl);
      const double ps = rest ? ps_in : (msl ? rget<PM>(g.latest, sl) : rget<PM>(g.previous, sl));
      const int pop_p = rget<PM>(g.populated, w) + __popc(mine);
      const int pop_sl = rget<PM>(g.populated, sl) + __popc(msl);
      const bool need = is_dec && cls == 2 && g.r_max > 0 && pop_p >= 2 && pop_sl >= 2;
      int pred = 0;
      const unsigned needm = __ballot_sync(kFull, need);
      SCAN_STAMP(pc_dssp);
      if (needm && ahead) {  // computed by the helper warp, tagged with this run
        while (__any_sync(kFull, need && (unsigned)(pv >> 32) != a.tag)) {
          if (need && (unsigned)(pv >> 32) != a.tag) pv = ld_relaxed_u64(a.pred + base + lane);
          if (globaltimer_ns() - t_pred > a.timeout_ns) break;
        }
        pred = need ? (int)(unsigned)pv : 0;
      } else if (needm) {  // one lane per decision, one forward sweep of its grid
        bool ok = true;
        pred = controller_lane(c.now, pp, ls, ps, g.r_max, ok);
        if (!need) pred = 0;
        if constexpr (PREDICT) {
          if (need) st_relaxed_u64(a.pred + base + lane, ((unsigned long long)a.tag << 32) | (unsigned)pred);
        }
      }
      SCAN_STAMP(pc_ctl);
      int headroom = g.s_lower + g.r_max - gap;
      headroom = headroom < 0 ? 0 : headroom;
      mint = pred < headroom ? pred : headroom;
    }
    if constexpr (PREDICT) {
      // the helper only moves the tables on (every decide of the valid
      // prefix counts: the gate stops at the first protocol error anyway)
#pragma unroll
      for (int q = 0; q < PM; ++q) {
        const unsigned mqa = mq[q];
        const int k = __popc(mqa);
        const int l1 = mqa ? 31 - __clz(mqa) : 0;
        const unsigned rest = mqa & ~(1u << l1);
        const double t1 = __shfl_sync(kFull, c.now, l1);
        const double t2 = __shfl_sync(kFull, c.now, rest ? 31 - __clz(rest) : 0);
        if (k) {
          g.previous[q] = k >= 2 ? t2 : g.latest[q];
          g.latest[q] = t1;
          g.clocks[q] += k;
          g.populated[q] += k;
        }
      }
      if (limit < m) break;
      c = nx;
      continue;
    }
    // the outcome and the credits a decision leaves when the worker holds no
    // credit are fixed by now: pack worker | outcome | credits | ready set
    const unsigned out0 = cls == 2 ? (mint ? 0u : 1u) : (unsigned)cls;
    const unsigned word = (unsigned)w | (out0 << 3) | ((unsigned)(cls == 2 ? mint : 0) << 4) | (ready << 12);
    // decisions compacted into slots 0..nd-1, slot j in lane j
    const int nd = __popc(md);
    const int myslot = __popc(md & lt);
    if (is_dec) sw[myslot] = word;
    __syncwarp();
    const unsigned wslot = sw[lane];
    __syncwarp();
    // ---- the credit / deferred recurrence, in call order: branch-free,
    // each slot's result left in its lane ----
    const unsigned def0 = defm;
    const CW cw0 = cw;
    unsigned myres = 0, mydef = 0;
    CW mycw = 0;
    int failslot = 32;
    auto scan = [&](int nlim) {
      for (int g0 = 0; g0 < nlim; g0 += 8) {
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int j = g0 + t;
          const bool act = j < nlim;
          const unsigned cur = __shfl_sync(kFull, wslot, j & 31);
          const int p = (int)(cur & 7u), sh = p << 3;
          const bool bad = act && ((defm >> p) & 1u);  // pushed while deferred
          failslot = (bad && failslot == 32) ? j : failslot;
          const unsigned cred = (unsigned)(cw >> sh) & 0xffu;
          const bool has = cred != 0u;
          const unsigned nf = has ? cred - 1u : ((cur >> 4) & 0xffu);
          const unsigned out = has ? 0u : ((cur >> 3) & 1u);
          const CW ncw = cw ^ ((CW)(cred ^ nf) << sh);
          const unsigned rel = out ? 0u : (defm & (cur >> 12));
          const unsigned ndef = (defm | (out << p)) & ~rel;
          cw = act ? ncw : cw;
          defm = act ? ndef : defm;
          const bool mine = lane == j;
          myres = mine ? ((rel << 8) | out) : myres;
          mydef = mine ? defm : mydef;
          mycw = mine ? cw : mycw;
        }
      }
    };
    scan(nd);
    int ndone = nd;
    if (failslot < 32) {  // rare: redo up to the failing decision from the chunk's start
      ndone = failslot;
      cw = cw0;
      defm = def0;
      scan(ndone);
    }
    SCAN_STAMP(pc_scan);
    const unsigned fdl = __ballot_sync(kFull, is_dec && myslot == failslot);
    const unsigned fail_dec = fdl ? (unsigned)(__ffs(fdl) - 1) : 32u;
    // ---- pulls: none from a deferred worker (the set after the last decision before it) ----
    const unsigned done = fail_dec < 32 ? (md & ((1u << fail_dec) - 1u)) : md;
    const unsigned pl_mask = mp & (fail_dec < 32 ? ((1u << fail_dec) - 1u) : kFull);
    const int slot_before = __popc(done & lt) - 1;
    const unsigned dm_sh = __shfl_sync(kFull, mydef, slot_before < 0 ? 0 : slot_before);
    const unsigned dm_here = slot_before < 0 ? def0 : dm_sh;
    const unsigned hit = __ballot_sync(kFull, ((pl_mask >> lane) & 1u) && ((dm_here >> (c.worker & 31)) & 1u));
    int fail = -1;
    unsigned applied = done;
    int napplied = ndone;
    if (hit) {
      fail = __ffs(hit) - 1;
      applied = done & ((1u << fail) - 1u);
      napplied = __popc(applied);
      // the recurrence rolls back to the last decision before the failing pull
      const unsigned long long back_cw = (unsigned long long)mycw;
      const unsigned rd = __shfl_sync(kFull, mydef, napplied > 0 ? napplied - 1 : 0);
      const unsigned long long rc = __shfl_sync(kFull, back_cw, napplied > 0 ? napplied - 1 : 0);
      defm = napplied > 0 ? rd : def0;
      cw = napplied > 0 ? (CW)rc : cw0;
    } else if (fail_dec < 32) {
      fail = (int)fail_dec;
      pushes += 1;
    } else if (limit < m) {
      fail = limit;
    }
    // ---- the chunk's decisions out, tables forward ----
    const int nap = napplied;
    if (lane < nap && n_dec + lane < a.trace_cap) a.decisions[n_dec + lane] = (long long)myres;
    n_dec += nap;
    pushes += nap;
    g.decisions += nap;
#pragma unroll
    for (int q = 0; q < PM; ++q) {
      const unsigned mqa = mq[q] & applied;
      const int k = __popc(mqa);
      const int l1 = mqa ? 31 - __clz(mqa) : 0;
      const unsigned rest = mqa & ~(1u << l1);
      const double t1 = __shfl_sync(kFull, c.now, l1);
      const double t2 = __shfl_sync(kFull, c.now, rest ? 31 - __clz(rest) : 0);
      if (k) {
        g.previous[q] = k >= 2 ? t2 : g.latest[q];
        g.latest[q] = t1;
        g.clocks[q] += k;
        g.populated[q] += k;
      }
    }
    __syncwarp();
    if (fail >= 0) {
      status = PS_E_PROTOCOL;
      valid = base + fail;
      break;
    }
    valid = base + m;
    if (lane == 0 && valid < n) st_relaxed_u64(&a.out->validated, (unsigned long long)valid << 1);
    c = nx;
    SCAN_STAMP(pc_tail);
  }
#ifdef PS_SIM_PROFILE
  if (lane == 0)
    printf("[scan-gate] calls %lld: pre %lld dssp %lld controller %lld recurrence %lld tail %lld cycles\n", n, pc_pre,
           pc_dssp, pc_ctl, pc_scan, pc_tail);
#endif
#undef SCAN_STAMP
  if constexpr (PREDICT) return;
  if (lane == 0) st_relaxed_u64(&a.out->validated, ((unsigned long long)valid << 1) | 1ull);
#pragma unroll
  for (int q = 0; q < PM; ++q) g.credits[q] = (int)((cw >> (8 * q)) & (CW)0xffu);
  g.deferred = defm;
  if (lane == 0) g.store(a.ctrl->gate);
  if (lane == 0) {
    a.out->t_control_done = globaltimer_ns();
    a.out->events = valid;
    a.out->pushes = pushes;
    a.out->trace_rows = n_dec;
    a.out->unfinished = 0ull;
    if (status != PS_OK) atomicCAS(&a.out->status, PS_OK, status);
  }
}

// The controller-ahead helper (CTA 0, warp 2): the DSSP controller grids of a
// replay depend only on the push sequence (policy.py:108-132 reads the
// push history, never an outcome), so this warp runs the scan gate's
// per-chunk evaluation ahead of the gate warp and publishes every grid's
// result, tagged with the run, for the gate to read instead of computing it.
template <int PM>
__device__ void predict_warp_replay(const SimArgs& a) {
  if (!a.pred_ahead || !a.gate_scan) return;
  RegGate<PM> rg;
  rg.load(a.ctrl->gate, a.reset_gate != 0);
  if (rg.paradigm != PS_DSSP || !gate_scan_eligible<PM>(rg)) return;
  gate_warp_replay_scan<PM, true>(a, rg);
}

// The gate warp of a replay: decides every DECIDE in order and validates the
// protocol (unknown worker, pull or push while deferred). It publishes a
// watermark -- (calls validated << 1) | done -- once per 32 calls; the data
// warps number and execute the pulls / applies themselves (data_warp_replay)
// and never run past it, so a protocol error stops the data exactly where
// the reference would have raised.
template <int PM>
__device__ void gate_warp_replay(const SimArgs& a, ps_gate_state* sgate) {
  __shared__ double2 dq[32];  // this chunk's decides: (now, call index << 32 | worker)
  const int lane = threadIdx.x & 31;
  const int P = a.P;
  if constexpr (PM > 0) {
    if (a.gate_scan) {
      RegGate<PM> rg;
      rg.load(a.ctrl->gate, a.reset_gate != 0);
      if (gate_scan_eligible<PM>(rg)) {
        gate_warp_replay_scan<PM>(a, rg);
        return;
      }
    }
  }
  ReplayGate<PM> g;
  g.load(a.ctrl->gate, a.reset_gate != 0, sgate);
  long long n_dec = 0, pushes = 0, valid = 0;
  int status = PS_OK;
  const long long n = a.n_calls;
  if (lane == 0) a.out->t_start = globaltimer_ns();
#ifdef PS_SIM_PROFILE
  long long c_gate = 0;
  const long long c_start = clock64();
#endif
  auto load = [&](long long base, ReplayCall& c) {
    const long long i = base + lane;
    if (i < n) c = a.calls[i];
    else { c.now = 0.0; c.kind = -1; c.worker = 0; }
  };
  ReplayCall c, nx;
  load(0, c);
  for (long long base = 0; base < n && status == PS_OK; base += 32) {
    load(base + 32, nx);  // in flight while this chunk is decided
    const int m = n - base < 32 ? (int)(n - base) : 32;
    const unsigned live = m >= 32 ? kFull : ((1u << m) - 1u);
    const bool inr = lane < m;
    // an unknown worker ends the valid prefix of the chunk
    const unsigned badw = __ballot_sync(kFull, inr && (c.worker < 0 || c.worker >= P));
    const int limit = badw ? __ffs(badw) - 1 : m;
    const unsigned below_limit = limit >= 32 ? kFull : ((1u << limit) - 1u);
    unsigned md = __ballot_sync(kFull, c.kind == kCallDecide) & live & below_limit;
    const unsigned mp = __ballot_sync(kFull, c.kind == kCallPull) & live & below_limit;
    int prev = 0;
    int fail = -1;
    // pulls in [from, to) must not come from a deferred worker (one vote per
    // run of pulls: the deferred set only changes at decides)
    auto check_pulls = [&](int from, int to) {
      const unsigned long long dm = g.deferred_mask();
      if (!dm) return;  // nobody is deferred: no pull can violate
      const unsigned rng = mp & (to >= 32 ? kFull : ((1u << to) - 1u)) & ~((1u << from) - 1u);
      if (!rng) return;
      const unsigned hit = __ballot_sync(kFull, ((rng >> lane) & 1u) && ((dm >> (c.worker & 63)) & 1ull));
      if (hit) fail = __ffs(hit) - 1;
    };
    // the chunk's decision words stay in registers (lane j holds the j-th)
    // and leave in one coalesced store at the end of the chunk
    unsigned long long dword = 0;
    int nd = 0;
    auto flush_decisions = [&]() {
      if (lane < nd && n_dec + lane < a.trace_cap) a.decisions[n_dec + lane] = (long long)dword;
      n_dec += nd;
      pushes += nd;
      nd = 0;
    };
    // the chunk's decides, compacted once into shared memory in call order
    // (one scatter per chunk): the serial loop then reads its next (call,
    // worker, now) with one broadcast load issued a decision ahead, instead
    // of a find-first-set -> shuffle chain per decide on its critical path
    const int n_dec_chunk = __popc(md);
    if ((md >> lane) & 1u) {
      const int slot = __popc(md & ((1u << lane) - 1u));
      dq[slot] = make_double2(c.now, __longlong_as_double(((long long)lane << 32) | (unsigned)c.worker));
    }
    __syncwarp();
    double2 q = n_dec_chunk ? dq[0] : make_double2(0.0, 0.0);
    for (int j = 0; j < n_dec_chunk && fail < 0; ++j) {
      const double2 nq = dq[(j + 1) & 31];  // the next decide's, in flight during this one
      const long long packed = __double_as_longlong(q.y);
      const int i = (int)(packed >> 32);
      const int w = (int)(unsigned)packed;
      const double now = q.x;
      check_pulls(prev, i);
      if (fail >= 0) break;
#ifdef PS_SIM_PROFILE
      const long long tg = clock64();
#endif
      const GateResult r = g.on_push(w, now);
#ifdef PS_SIM_PROFILE
      c_gate += clock64() - tg;
#endif
      if (r.status != PS_OK) { pushes += 1; status = r.status; fail = i; break; }
      if (lane == nd) dword = (r.released << 8) | (unsigned)r.outcome;
      nd += 1;
      prev = i + 1;
      q = nq;
    }
    __syncwarp();
    flush_decisions();
    if (fail < 0) check_pulls(prev, limit);
    if (fail < 0 && limit < m) fail = limit;
    if (fail >= 0) {
      if (status == PS_OK) status = PS_E_PROTOCOL;
      valid = base + fail;
      break;
    }
    valid = base + m;
    // relaxed: the call watermark publishes no data, only how far the data may go
    if (lane == 0 && valid < n) st_relaxed_u64(&a.out->validated, (unsigned long long)valid << 1);
    c = nx;
  }
  if (lane == 0) st_relaxed_u64(&a.out->validated, ((unsigned long long)valid << 1) | 1ull);
#ifdef PS_SIM_PROFILE
  if (lane == 0)
    printf("[replay-gate] calls %lld decides %lld: total %lld cycles, on_push %lld, controller %lld calls %lld cycles\n",
           n, pushes, clock64() - c_start, c_gate, g_ctl_calls, g_ctl_cycles);
#endif
  g.store(a.ctrl->gate);
  if (lane == 0) {
    a.out->t_control_done = globaltimer_ns();
    a.out->events = valid;
    a.out->pushes = pushes;
    a.out->trace_rows = n_dec;
    a.out->unfinished = 0ull;
    if (status != PS_OK) atomicCAS(&a.out->status, PS_OK, status);
  }
}

constexpr int kRing = 256;  // per-CTA finiteness aggregation ring (> max warp skew in updates)

// Loads of one worker's update slice; V float4 per lane, element u at lo + lane + 32u.
// KEEP: the source is read-only for the whole kernel and re-read by this warp
// (the replay's resident updates) -- cache it in L1. Never for buffers the
// kernel itself writes (the simulated run's gradient slots): .nc loads are not
// coherent with this kernel's own stores.
template <int V, bool KEEP = false>
__device__ __forceinline__ void load_slice(float4 (&r)[V], const float4* src, long long lo, long long hi,
                                           int lane) {
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    if constexpr (KEEP) r[u] = j < hi ? ld_keep(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    else r[u] = j < hi ? ld_stream(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Data warp with its weight slice held in registers for the whole run (V
// float4 per lane); V == 0 is the general path that keeps it in HBM.
template <int V>
__device__ void data_warp(const SimArgs& a, unsigned dw, unsigned* s_ring, int warps_here) {
  const int lane = threadIdx.x & 31;
  const long long per = (a.nv + a.n_data_warps - 1) / a.n_data_warps;
  const long long lo = (long long)dw * per < a.nv ? (long long)dw * per : a.nv;
  const long long hi = lo + per < a.nv ? lo + per : a.nv;
  float4* W = reinterpret_cast<float4*>(a.W);
  const float4* C = reinterpret_cast<const float4*>(a.center);
  float4 wr[V > 0 ? V : 1];
  if constexpr (V > 0) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long j = lo + lane + 32ll * u;
      wr[u] = j < hi ? W[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  long long applied = 0, rejected = 0;
  const unsigned long long t0 = globaltimer_ns();
  long long base = 0;
  int have = 0;
  Op batch = 0;
  for (long long i = 0;; ++i) {
    if (i >= base + have) {
      // fetch up to 32 published ops at once (one coalesced 256 B load)
      base = i;
      unsigned backoff = 32;  // ns; doubles while the log is dry (the control
                              // warp emits ~1 op/us: hot polling only steals
                              // L2 bandwidth from the op stores it waits for)
      for (;;) {
        const long long k = base + lane;
        batch = k < a.ops_cap ? ld_relaxed_u64(a.ops + k) : 0ull;
        const unsigned valid = __ballot_sync(kFull, op_tag(batch) == (a.tag & 0xffffu));
        have = valid == kFull ? 32 : __ffs(~valid) - 1;
        if (have > 0) break;
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          if (lane == 0) atomicCAS(&a.out->status, PS_OK, PS_E_TIMEOUT);
          return;
        }
        __nanosleep(backoff);
        backoff = backoff < 512 ? backoff * 2 : 512;
      }
    }
    const Op op = __shfl_sync(kFull, batch, (int)(i - base));
    const int type = op_type(op), w = op_worker(op), buf = op_buf(op);
    const long long slot = op_slot(op);
    if (type == OP_END) break;
    if (type == OP_PULL) {
      float4* dst = reinterpret_cast<float4*>(a.rep + ((long long)w * 2 + buf) * a.dpad);
      if constexpr (V > 0) {
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const long long j = lo + lane + 32ll * u;
          if (j < hi) dst[j] = wr[u];
        }
      } else {
        for (long long j = lo + lane; j < hi; j += 32) dst[j] = W[j];
      }
    } else if (type == OP_GRAD) {
      bool bad = false;
      if (a.grad_kind == PS_GRAD_BOWL) {
        const float4* src = reinterpret_cast<const float4*>(a.rep + ((long long)w * 2 + buf) * a.dpad);
        float4* g = reinterpret_cast<float4*>(a.gbuf + (long long)w * a.dpad);
        for (long long j = lo + lane; j < hi; j += 32) {
          const float4 x = src[j], c = C[j];
          const float4 r = make_float4(__fsub_rn(x.x, c.x), __fsub_rn(x.y, c.y),
                                       __fsub_rn(x.z, c.z), __fsub_rn(x.w, c.w));
          bad |= nonfinite4(r);
          g[j] = r;
        }
      } else {
        const float4* src =
            reinterpret_cast<const float4*>(a.synth + ((long long)w * a.n_synth + buf) * a.dpad);
        if constexpr (V > 0) {
          float4 r[V];
          load_slice<V>(r, src, lo, hi, lane);
#pragma unroll
          for (int u = 0; u < V; ++u) bad |= nonfinite4(r[u]);
        } else {
          for (long long j = lo + lane; j < hi; j += 32) bad |= nonfinite4(ld_stream(src + j));
        }
      }
      const bool any_bad = __any_sync(kFull, bad);
      if (lane == 0) {
        // CTA-level aggregation: the last warp of this CTA to flag the update
        // adds one count (and a non-finite mark) to its global word
        const unsigned inc = 1u + (any_bad ? 0x10000u : 0u);
        const unsigned old = atomicAdd(&s_ring[slot & (kRing - 1)], inc);
        if ((old & 0xffffu) == (unsigned)warps_here - 1) {
          atomicExch(&s_ring[slot & (kRing - 1)], 0u);
          const unsigned badc = (old >> 16) + (any_bad ? 1u : 0u);
          atomicAdd(&a.gword[slot], 1u + (badc ? 0x10000u : 0u));
        }
      }
    } else if (type == OP_APPLY) {
      const float4* g = a.grad_kind == PS_GRAD_BOWL
                            ? reinterpret_cast<const float4*>(a.gbuf + (long long)w * a.dpad)
                            : reinterpret_cast<const float4*>(a.synth + ((long long)w * a.n_synth + buf) * a.dpad);
      float4 gr[V > 0 ? V : 1];
      if constexpr (V > 0) {
        if (a.grad_kind == PS_GRAD_BOWL) {
#pragma unroll
          for (int u = 0; u < V; ++u) {
            const long long j = lo + lane + 32ll * u;
            gr[u] = j < hi ? g[j] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        } else {
          load_slice<V>(gr, g, lo, hi, lane);  // in flight while we wait for the verdict
        }
      }
      unsigned v = 0;
      if (lane == 0) {
        while (((v = ld_relaxed_u32(&a.gword[slot])) & 0xffffu) < a.n_ctas) {
          if (globaltimer_ns() - t0 > a.timeout_ns) { v = 0xffffffffu; break; }
          __nanosleep(20);
        }
      }
      v = __shfl_sync(kFull, v, 0);
      if (v == 0xffffffffu) {
        if (lane == 0) atomicCAS(&a.out->status, PS_OK, PS_E_TIMEOUT);
        return;
      }
      if (v >> 16) {
        rejected += 1;
        continue;
      }
      bool dbad = false;
      if constexpr (V > 0) {
#pragma unroll
        for (int u = 0; u < V; ++u) {
          wr[u] = apply4(wr[u], a.lr, gr[u]);
          dbad |= nonfinite4(wr[u]);
        }
      } else {
        for (long long j = lo + lane; j < hi; j += 32) {
          const float4 r = apply4(W[j], a.lr, g[j]);
          dbad |= nonfinite4(r);
          W[j] = r;
        }
      }
      applied += 1;
      if (__any_sync(kFull, dbad) && lane == 0) {
        if (atomicCAS(&a.out->status, PS_OK, PS_E_DIVERGED) == PS_OK) a.out->diverged_worker = w;
      }
      if (a.loss_every > 0 && (a.base_version + applied) % a.loss_every == 0) {
        double acc = 0.0;
        if constexpr (V > 0) {
#pragma unroll
          for (int u = 0; u < V; ++u) {
            const long long j = lo + lane + 32ll * u;
            if (j < hi) {
              const float4 x = wr[u], c = C[j];
              const double d0 = (double)x.x - (double)c.x, d1 = (double)x.y - (double)c.y;
              const double d2 = (double)x.z - (double)c.z, d3 = (double)x.w - (double)c.w;
              acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
            }
          }
        } else {
          for (long long j = lo + lane; j < hi; j += 32) {
            const float4 x = W[j], c = C[j];
            const double d0 = (double)x.x - (double)c.x, d1 = (double)x.y - (double)c.y;
            const double d2 = (double)x.z - (double)c.z, d3 = (double)x.w - (double)c.w;
            acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off);
        const long long sample = (a.base_version + applied) / a.loss_every - 1 -
                                 a.base_version / a.loss_every;
        if (lane == 0 && sample >= 0 && sample < a.loss_cap) atomicAdd(&a.losses[sample], 0.5 * acc);
      }
    }
  }
  if constexpr (V > 0) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long j = lo + lane + 32ll * u;
      if (j < hi) W[j] = wr[u];
    }
  }
  if (lane == 0) atomicMax(&a.out->t_data_done, globaltimer_ns());
  if (dw == 0 && lane == 0) {
    a.out->applied = applied;
    a.out->rejected = rejected;
  }
}

// Replay data warp. The op stream of a replay is a function of the call list
// alone: an apply's update index is the number of earlier applies by the
// same worker, a pull's replica buffer the parity of that worker's earlier
// pulls. Every data warp derives these per 32-call chunk with ballots /
// match_any (prefix counts, no serial producer) and keeps two chunks of
// lookahead: while it executes chunk c it numbers and scans chunk c+2.
//
// Finiteness verdicts are per chunk (server.py:65-67 rejects an update if ANY
// element is non-finite, and every warp sees only its slice): each warp ORs
// the calls whose slice holds a non-finite value into a 32-bit mask, the CTA
// aggregates its warps in a shared 64-bit word {warps done << 32 | bits},
// and the last warp adds the CTA to the chunk's global word {CTAs done << 32
// | bits} -- an OR then an ADD on the same address, so a reader that sees the
// full count sees every CTA's bits without a fence. Executing a chunk takes
// ONE poll of that word.
template <int V>
__device__ void data_warp_replay(const SimArgs& a, unsigned dw, unsigned* s_ring32, int warps_here) {
  constexpr int K = V == 1 ? 8 : V == 2 ? 4 : V == 4 ? 2 : 1;     // scan: update slices in flight
  constexpr int KG = V == 1 ? 16 : V == 2 ? 8 : V == 4 ? 4 : V == 8 ? 2 : 1;  // execute: calls per group
  constexpr int VV = V > 0 ? V : 1;
  constexpr int kRingChunks = kRing / 2;
  unsigned long long* s_ring = reinterpret_cast<unsigned long long*>(s_ring32);
  unsigned long long* gchunk = reinterpret_cast<unsigned long long*>(a.gword);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int P = a.P, nsyn = a.n_synth;
  const long long n = a.n_calls;
  const long long per = (a.nv + a.n_data_warps - 1) / a.n_data_warps;
  const long long lo = (long long)dw * per < a.nv ? (long long)dw * per : a.nv;
  const long long hi = lo + per < a.nv ? lo + per : a.nv;
  float4* W = reinterpret_cast<float4*>(a.W);
  float4 wr[VV];
  if constexpr (V > 0) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long j = lo + lane + 32ll * u;
      wr[u] = j < hi ? W[j] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  const unsigned long long t0 = globaltimer_ns();
  // per-worker counters, lane q holds workers q and q + 32
  int sidx_lo = 0, sidx_hi = 0, stg_lo = 0, stg_hi = 0;
  long long applied = 0, rejected = 0;
  int diverged = -1;
  // per chunk: lane l's call as (worker << 8 | buffer), and the warp-uniform
  // masks of its applies and pulls
  struct Chunk { int wb; unsigned ma, mp; };
  auto number = [&](long long base, Chunk& c) {
    const long long i = base + lane;
    int kind = -1, worker = 0, buf = 0;
    if (i < n) {
      const int2 kw = *reinterpret_cast<const int2*>(&a.calls[i].kind);
      kind = kw.x;
      worker = kw.y;
    }
    const bool okw = worker >= 0 && worker < P;
    const bool isa = okw && kind == kCallApply, isp = okw && kind == kCallPull;
    c.ma = __ballot_sync(kFull, isa);
    c.mp = __ballot_sync(kFull, isp);
    const unsigned peers = __match_any_sync(kFull, isa ? worker : isp ? 64 + worker : 128 + lane);
    const int rank = __popc(peers & lt);
    const int wq = worker & 31;
    const int s_lo = __shfl_sync(kFull, sidx_lo, wq), s_hi = __shfl_sync(kFull, sidx_hi, wq);
    const int g_lo = __shfl_sync(kFull, stg_lo, wq), g_hi = __shfl_sync(kFull, stg_hi, wq);
    if (isa) buf = ((worker < 32 ? s_lo : s_hi) + rank) % nsyn;
    if (isp) buf = (worker < 32 ? g_lo : g_hi) ^ ((rank + 1) & 1);
    c.wb = (okw ? worker : 0) << 8 | buf;
    for (int q = 0; q < P; ++q) {
      const int na = __popc(__ballot_sync(kFull, isa && worker == q));
      const int np = __popc(__ballot_sync(kFull, isp && worker == q));
      if (lane == (q & 31)) {
        if (q < 32) { sidx_lo += na; stg_lo ^= np & 1; }
        else { sidx_hi += na; stg_hi ^= np & 1; }
      }
    }
  };
  auto slice_of = [&](const Chunk& c, int l) {
    const int wb = __shfl_sync(kFull, c.wb, l);
    return reinterpret_cast<const float4*>(a.synth + ((long long)(wb >> 8) * nsyn + (wb & 255)) * a.dpad);
  };
  // x * 0 is 0 for finite x and NaN otherwise: one FFMA per component
  auto acc_nonfinite = [](float acc, const float4& v) {
    return __fmaf_rn(v.w, 0.f, __fmaf_rn(v.z, 0.f, __fmaf_rn(v.y, 0.f, __fmaf_rn(v.x, 0.f, acc))));
  };
  auto scan = [&](const Chunk& c, long long chunk) {
    unsigned m = c.ma;
    unsigned badbits = 0;
    while (m) {
      int ls[K];
      float4 r[K][VV];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        ls[k] = -1;
        if (m) {
          ls[k] = __ffs(m) - 1;
          m &= m - 1;
          if constexpr (V > 0) load_slice<V, true>(r[k], slice_of(c, ls[k]), lo, hi, lane);
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (ls[k] < 0) break;
        float acc = 0.f;
        if constexpr (V > 0) {
#pragma unroll
          for (int u = 0; u < V; ++u) acc = acc_nonfinite(acc, r[k][u]);
        } else {
          const float4* src = slice_of(c, ls[k]);
          for (long long j = lo + lane; j < hi; j += 32) acc = acc_nonfinite(acc, ld_stream(src + j));
        }
        if (__any_sync(kFull, acc != acc)) badbits |= 1u << ls[k];
      }
    }
    if (lane == 0 && chunk * 32 < n) {
      unsigned long long* w = &s_ring[chunk & (kRingChunks - 1)];
      if (badbits) atomicOr(w, (unsigned long long)badbits);
      const unsigned long long old = atomicAdd(w, 1ull << 32);
      if ((unsigned)(old >> 32) == (unsigned)warps_here - 1) {  // last warp of this CTA
        const unsigned long long bits = atomicExch(w, 0ull) & 0xffffffffull;
        if (bits) atomicOr(&gchunk[chunk], bits);
        atomicAdd(&gchunk[chunk], 1ull << 32);
      }
    }
  };
  Chunk c0, c1, c2;
  number(0, c0);
  scan(c0, 0);
  number(32, c1);
  scan(c1, 1);
  bool stop = false;
  for (long long base = 0, chunk = 0; base < n && !stop; base += 32, ++chunk) {
    // polls for this chunk, issued before the lookahead work hides them
    unsigned long long wm = 0, cv = 0;
    if (lane == 0) {
      wm = ld_relaxed_u64(&a.out->validated);
      cv = ld_relaxed_u64(&gchunk[chunk]);
    }
    number(base + 64, c2);
    scan(c2, chunk + 2);
    const long long need = n - base < 32 ? n : base + 32;
    if (lane == 0) {
      // the gate warp's watermark: calls validated so far (| 1 once done).
      // Relaxed is enough: no data is published under it.
      unsigned backoff = 32;
      while ((wm >> 1) < (unsigned long long)need && !(wm & 1ull)) {
        if (globaltimer_ns() - t0 > a.timeout_ns) { wm = ~0ull; break; }
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
        wm = ld_relaxed_u64(&a.out->validated);
      }
      // every data CTA has scanned this chunk
      while (wm != ~0ull && (unsigned)(cv >> 32) < a.n_ctas) {
        if (globaltimer_ns() - t0 > a.timeout_ns) { wm = ~0ull; break; }
        __nanosleep(20);
        cv = ld_relaxed_u64(&gchunk[chunk]);
      }
    }
    wm = __shfl_sync(kFull, wm, 0);
    const unsigned bits = (unsigned)__shfl_sync(kFull, cv, 0);
    if (wm == ~0ull) {
      if (lane == 0) atomicCAS(&a.out->status, PS_OK, PS_E_TIMEOUT);
      return;
    }
    long long upto = (long long)(wm >> 1);
    if (upto < need) stop = true;  // the gate stopped inside this chunk
    else upto = need;
    const int m = upto > base ? (int)(upto - base) : 0;
    const unsigned live = m >= 32 ? kFull : ((1u << m) - 1u);
    // pulls and applies in call order (decides are the gate warp's), KG calls
    // at a time with every update slice of the group loaded up front
    bool dbad = false;
    unsigned calls = (c0.ma | c0.mp) & live;
    while (calls) {
      int idx[KG];
      float4 g[KG][VV];
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        idx[k] = -1;
        if (calls) {
          const int i = __ffs(calls) - 1;
          calls &= calls - 1;
          idx[k] = i;
          if constexpr (V > 0)
            if (((c0.ma & ~bits) >> i) & 1u) load_slice<V, true>(g[k], slice_of(c0, i), lo, hi, lane);
        }
      }
      if constexpr (V > 0) {
        // branch-light: every slot of the group runs the same straight-line
        // code under warp-uniform predicates, so address math and shuffles
        // of later calls overlap the stores / math of earlier ones
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          const int i = idx[k];
          const unsigned bit = i >= 0 ? (1u << i) : 0u;
          const int wb = __shfl_sync(kFull, c0.wb, i & 31);
          const int w = wb >> 8, buf = wb & 255;
          if (c0.mp & bit) {
            float4* dst = reinterpret_cast<float4*>(a.rep + ((long long)w * 2 + buf) * a.dpad);
#pragma unroll
            for (int u = 0; u < V; ++u) {
              const long long j = lo + lane + 32ll * u;
              if (j < hi) dst[j] = wr[u];
            }
          }
          if (c0.ma & ~bits & bit) {
            float acc = 0.f;
#pragma unroll
            for (int u = 0; u < V; ++u) {
              wr[u] = apply4(wr[u], a.lr, g[k][u]);
              acc = acc_nonfinite(acc, wr[u]);
            }
            if (acc != acc && !dbad) { dbad = true; diverged = w; }
            applied += 1;
          }
          if (c0.ma & bits & bit) rejected += 1;
        }
      } else {
        for (int k = 0; k < KG; ++k) {
          const int i = idx[k];
          if (i < 0) break;
          const int wb = __shfl_sync(kFull, c0.wb, i);
          const int w = wb >> 8, buf = wb & 255;
          if ((c0.mp >> i) & 1u) {
            float4* dst = reinterpret_cast<float4*>(a.rep + ((long long)w * 2 + buf) * a.dpad);
            for (long long j = lo + lane; j < hi; j += 32) dst[j] = W[j];
          } else if ((bits >> i) & 1u) {
            rejected += 1;
          } else {
            float acc = 0.f;
            const float4* gp = reinterpret_cast<const float4*>(a.synth + ((long long)w * nsyn + buf) * a.dpad);
            for (long long j = lo + lane; j < hi; j += 32) {
              const float4 r = apply4(W[j], a.lr, gp[j]);
              acc = acc_nonfinite(acc, r);
              W[j] = r;
            }
            if (acc != acc && !dbad) { dbad = true; diverged = w; }
            applied += 1;
          }
        }
      }
    }
    // a non-finite result (server.py:38-41): the run stops with the worker named
    if (__any_sync(kFull, dbad)) {
      const int src = __ffs(__ballot_sync(kFull, dbad)) - 1;
      const int wdiv = __shfl_sync(kFull, diverged, src);
      if (lane == 0 && atomicCAS(&a.out->status, PS_OK, PS_E_DIVERGED) == PS_OK) a.out->diverged_worker = wdiv;
    }
    c0 = c1;
    c1 = c2;
  }
  if constexpr (V > 0) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long j = lo + lane + 32ll * u;
      if (j < hi) W[j] = wr[u];
    }
  }
  if (lane == 0) atomicMax(&a.out->t_data_done, globaltimer_ns());
  if (dw == 0 && lane == 0) {
    a.out->applied = applied;
    a.out->rejected = rejected;
  }
}

// Speculative replay data warp (register-resident slices, V > 0). Same call
// numbering as data_warp_replay, but no separate finiteness pass: a chunk is
// executed as soon as the gate's watermark allows, every update is checked
// while it is applied, and the chunk's non-finite-update bits are published
// (CTA-aggregated, one global word per chunk) only afterwards. The weights
// before each of the last L+1 chunks are kept in registers; when a chunk's
// global verdict comes back (L chunks later, so nobody waits for it in the
// common case) with a rejected update (server.py:65-67) the warp restores
// the checkpoint and re-executes that chunk and the later ones with their
// final verdicts -- pulls included, so every replica ends up exactly as the
// in-order server would have written it.
template <int V, int KG4 = 2>
__device__ void data_warp_replay_spec(const SimArgs& a, unsigned dw, unsigned* s_ring32, int warps_here) {
  static_assert(V > 0 && V <= 4, "register-resident slices of at most 4 float4 per lane");
#ifndef PS_REPLAY_KG2
#define PS_REPLAY_KG2 8
#endif
  constexpr int KG = V == 1 ? 16 : V == 2 ? PS_REPLAY_KG2 : KG4;  // calls per group
#ifndef PS_REPLAY_LAG
#define PS_REPLAY_LAG 3
#endif
  constexpr int L = V <= 2 ? PS_REPLAY_LAG : 2;  // chunks executed before their verdict is read
  constexpr int kRingChunks = kRing / 2;
  unsigned long long* s_ring = reinterpret_cast<unsigned long long*>(s_ring32);
  unsigned long long* gchunk = reinterpret_cast<unsigned long long*>(a.gword);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int P = a.P, nsyn = a.n_synth;
  const long long n = a.n_data;  // the gate publishes the data calls (DataEmit)
  const long long per = (a.nv + a.n_data_warps - 1) / a.n_data_warps;
  const long long lo = (long long)dw * per < a.nv ? (long long)dw * per : a.nv;
  const long long hi = lo + per < a.nv ? lo + per : a.nv;
  float4* W = reinterpret_cast<float4*>(a.W);
  const float4* const synth4 = reinterpret_cast<const float4*>(a.synth);
  float4* const rep4 = reinterpret_cast<float4*>(a.rep);
  float4 wr[V];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    wr[u] = j < hi ? W[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // this lane's element u is float4 lo + lane + 32u of every buffer
  const float4* const sbase = synth4 + lo + lane;
  float4* const rbase = rep4 + lo + lane;
  const int span = (int)(hi - lo) - lane;  // element u is in the slice iff 32u < span
  (void)sbase; (void)rbase; (void)span;
  const unsigned long long t0 = globaltimer_ns();
  long long applied = 0, rejected = 0;
  int diverged = -1;  // worker of the first non-finite result seen by this warp
  bool timed_out = false;
  // per call: (worker << 8 | buffer), and the float4 offset of its slice in
  // the resident updates (apply) or the replicas (pull) -- 32 bits suffice for
  // the slice widths this path serves (V <= 4)
  struct Chunk { int wb; unsigned ma, mp, off; };
  const unsigned dv4 = (unsigned)(a.dpad >> 2);
  // one data call per lane from the gate's descriptor stream (DataEmit)
  auto decode = [&](unsigned d, bool in, Chunk& c) {
    const bool isp = in && ((d >> 16) & 1u), isa = in && !((d >> 16) & 1u);
    c.ma = __ballot_sync(kFull, isa);
    c.mp = __ballot_sync(kFull, isp);
    const int worker = (int)((d >> 8) & 127u), buf = (int)(d & 255u);
    c.wb = worker << 8 | buf;
    c.off = isa ? (unsigned)(worker * nsyn + buf) * dv4 : isp ? (unsigned)(worker * 2 + buf) * dv4 : 0u;
  };
  // descriptors [base, upto): each word carries the run's tag, so a word not
  // yet written by this run is re-polled (rare: the watermark said it is there)
  const unsigned tag = a.tag;
  auto load_desc = [&](long long base, long long upto) -> unsigned long long {
    const long long i = base + lane;
    return i < upto ? ld_relaxed_u64(a.dstream + i) : ((unsigned long long)tag << 32);
  };
  auto settle = [&](unsigned long long v, long long base, long long upto) -> unsigned {
    while (__any_sync(kFull, (unsigned)(v >> 32) != tag)) {
      if ((unsigned)(v >> 32) != tag) v = load_desc(base, upto);
      if (globaltimer_ns() - t0 > a.timeout_ns) { timed_out = true; break; }
    }
    return (unsigned)v;
  };
  auto acc_nonfinite = [](float acc, const float4& v) {
    return __fmaf_rn(v.w, 0.f, __fmaf_rn(v.z, 0.f, __fmaf_rn(v.y, 0.f, __fmaf_rn(v.x, 0.f, acc))));
  };
  // execute the live calls of a chunk with the rejected set `rej`; returns the
  // calls whose update (gb) / result (rb) holds a non-finite value in this slice
  auto exec = [&](const Chunk& c, unsigned live, unsigned rej, unsigned& gb, unsigned& rb) {
    // per-lane bits, one warp reduction per chunk (not a vote per apply)
    unsigned lrb = 0;
    unsigned calls = (c.ma | c.mp) & live;
#ifndef PS_REPLAY_BRANCHED_SLOTS
    // straight-line slots: every slot runs the same predicated code, so the
    // compiler can interleave the slots of a group. A slot that is not a live
    // apply loads nothing and keeps g = +0, and w - lr*(+0) == w bit for bit
    // (also for -0, inf and NaN), so its apply is an exact identity; its
    // result is not checked.
    const unsigned mapp = c.ma & ~rej;
    // the descriptor stream holds only data calls, in order: slot s is lane s
    const int ncalls = 32 - __clz(calls);
    for (int s0 = 0; s0 < ncalls; s0 += KG) {
      unsigned bitk[KG];
      float4 g[KG][V];
      unsigned offk[KG];
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        const int i = s0 + k;  // <= 31: s0 < ncalls <= 32 and KG divides 32
        bitk[k] = calls & (1u << i);
        offk[k] = __shfl_sync(kFull, c.off, i);
        const bool ld = (mapp & bitk[k]) != 0u;
#pragma unroll
        for (int u = 0; u < V; ++u) g[k][u] = ld_keep_if(ld && 32 * u < span, sbase + offk[k] + 32 * u);
      }
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        const bool pl = (c.mp & bitk[k]) != 0u;
#pragma unroll
        for (int u = 0; u < V; ++u) st_f4_if(pl && 32 * u < span, rbase + offk[k] + 32 * u, wr[u]);
        float ra = 0.f;
#pragma unroll
        for (int u = 0; u < V; ++u) {
          wr[u] = apply4(wr[u], a.lr, g[k][u]);
          ra = acc_nonfinite(ra, wr[u]);
        }
        lrb |= (ra != ra) ? (mapp & bitk[k]) : 0u;
      }
    }
#else
    while (calls) {
      int idx[KG];
      unsigned offk[KG];
      float4 g[KG][V];
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        idx[k] = -1;
        offk[k] = 0;
        if (calls) {
          const int i = __ffs(calls) - 1;
          calls &= calls - 1;
          idx[k] = i;
          offk[k] = __shfl_sync(kFull, c.off, i);
          if (((c.ma & ~rej) >> i) & 1u) load_slice<V, true>(g[k], synth4 + offk[k], lo, hi, lane);
        }
      }
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        const int i = idx[k];
        const unsigned bit = i >= 0 ? (1u << i) : 0u;
        if (c.mp & bit) {
          float4* dst = rep4 + offk[k];
#pragma unroll
          for (int u = 0; u < V; ++u) {
            const long long j = lo + lane + 32ll * u;
            if (j < hi) dst[j] = wr[u];
          }
        }
        if (c.ma & ~rej & bit) {
          // only the result is checked here: a non-finite update always
          // gives a non-finite result (lr > 0), and the rare non-finite
          // result is classified below
          float ra = 0.f;
#pragma unroll
          for (int u = 0; u < V; ++u) {
            wr[u] = apply4(wr[u], a.lr, g[k][u]);
            ra = acc_nonfinite(ra, wr[u]);
          }
          if (ra != ra) lrb |= bit;
        }
      }
    }
#endif
    rb = __reduce_or_sync(kFull, lrb);
    gb = 0;
    // rare: which of the non-finite results come from a non-finite update
    // (a rejection, server.py:65-67) rather than from the weights
    for (unsigned m = rb; m; m &= m - 1) {
      const int i = __ffs(m) - 1;
      const int wb = __shfl_sync(kFull, c.wb, i);
      float4 r[V];
      load_slice<V>(r, reinterpret_cast<const float4*>(
                           a.synth + ((long long)(wb >> 8) * nsyn + (wb & 255)) * a.dpad),
                    lo, hi, lane);
      float ga = 0.f;
#pragma unroll
      for (int u = 0; u < V; ++u) ga = acc_nonfinite(ga, r[u]);
      if (__any_sync(kFull, ga != ga)) gb |= 1u << i;
    }
  };
  // CTA aggregation in shared memory: per ring slot a bits word and an
  // arrival count, both native 32-bit shared atomics (a 64-bit shared atomic
  // add is a compare-and-swap loop, and the CTA's warps all hit the same slot)
  auto publish = [&](long long chunk, unsigned bits) {
    if (lane == 0) {
      unsigned* w = &s_ring32[2 * (chunk & (kRingChunks - 1))];
      if (bits) atomicOr(w, bits);
      __threadfence_block();  // the bits before the arrival
      if (atomicAdd(w + 1, 1u) == (unsigned)warps_here - 1) {  // last warp of this CTA
        __threadfence_block();
        const unsigned b = atomicExch(w, 0u);
        atomicExch(w + 1, 0u);
        if (b) atomicOr(&gchunk[chunk], (unsigned long long)b);
        atomicAdd(&gchunk[chunk], 1ull << 32);
      }
    }
  };
  // `first`: a sample of the chunk's word loaded ahead (have_first), so the
  // common case -- the verdict is long final -- costs no load latency here
  auto verdict = [&](long long chunk, unsigned long long first = 0ull, bool have_first = false) -> unsigned {
    unsigned long long v = 0;
    if (lane == 0) {
      v = have_first ? first : ld_relaxed_u64(&gchunk[chunk]);
      while ((unsigned)(v >> 32) < a.n_ctas) {
        if (globaltimer_ns() - t0 > a.timeout_ns) { timed_out = true; break; }
        __nanosleep(20);
        v = ld_relaxed_u64(&gchunk[chunk]);
      }
    }
    timed_out = __shfl_sync(kFull, (int)timed_out, 0) != 0;
    return (unsigned)__shfl_sync(kFull, v, 0);
  };
  // pending chunks, newest at index 0: calls, live mask, weights before the
  // chunk, local non-finite-result bits, already final?
  Chunk C[L + 1];
  float4 ck[L + 1][V];
  unsigned LV[L + 1], RB[L + 1];
  bool FIN[L + 1];
#pragma unroll
  for (int j = 0; j <= L; ++j) { LV[j] = 0; RB[j] = 0; FIN[j] = true; C[j].wb = 0; C[j].ma = 0; C[j].mp = 0; }
  // resolve pending entry J (chunk number `chunk - J`): commit it, or roll
  // back to its checkpoint and replay it and everything newer with verdicts
  auto resolve = [&](auto J_, long long chunk, unsigned long long first = 0ull, bool have_first = false) {
    constexpr int J = decltype(J_)::value;
    if (FIN[J]) return;
    const unsigned bits = verdict(chunk - J, first, have_first) & LV[J];
    if (timed_out) return;
    if (!(bits & C[J].ma)) {
      applied += __popc(C[J].ma & LV[J]);
      if ((RB[J] & LV[J]) && diverged < 0) diverged = __shfl_sync(kFull, C[J].wb, __ffs(RB[J] & LV[J]) - 1) >> 8;
      FIN[J] = true;
      return;
    }
#pragma unroll
    for (int u = 0; u < V; ++u) wr[u] = ck[J][u];
#pragma unroll
    for (int jj = L; jj >= 0; --jj) {
      if (jj > J || FIN[jj]) continue;
      const unsigned rj = (jj == J ? bits : verdict(chunk - jj) & LV[jj]) & C[jj].ma;
      if (timed_out) return;
      unsigned gb, rb;
      exec(C[jj], LV[jj], rj, gb, rb);
      applied += __popc(C[jj].ma & LV[jj] & ~rj);
      rejected += __popc(rj);
      if ((rb & LV[jj]) && diverged < 0) diverged = __shfl_sync(kFull, C[jj].wb, __ffs(rb & LV[jj]) - 1) >> 8;
      FIN[jj] = true;
    }
  };
  bool stop = false;
  long long chunk = 0;
  unsigned long long wm = 0;  // the gate's data watermark, loaded a chunk ahead
  if (lane == 0) wm = ld_relaxed_u64(&a.out->dvalid);
  unsigned long long dnext = 0;  // the next chunk's descriptors, when already published
  bool have_next = false;
  for (long long base = 0; base < n && !stop && !timed_out; base += 32, ++chunk) {
    // the verdict word of the oldest pending chunk, in flight while this one is decoded
    unsigned long long vpre = 0;
    const bool vhave = lane == 0 && !FIN[L] && chunk - 1 - L >= 0;
    if (vhave) vpre = ld_relaxed_u64(&gchunk[chunk - 1 - L]);
    const long long need = n - base < 32 ? n : base + 32;
    if (lane == 0) {
      unsigned backoff = 32;
      while ((wm >> 1) < (unsigned long long)need && !(wm & 1ull)) {
        if (globaltimer_ns() - t0 > a.timeout_ns) { wm = ~0ull; break; }
        __nanosleep(backoff);
        backoff = backoff < 256 ? backoff * 2 : 256;
        wm = ld_relaxed_u64(&a.out->dvalid);
      }
    }
    wm = __shfl_sync(kFull, wm, 0);
    if (wm == ~0ull) { timed_out = true; break; }
    long long upto = (long long)(wm >> 1);
    if (upto < need) stop = true;  // the gate stopped inside this chunk
    else upto = need;
    const int m = upto > base ? (int)(upto - base) : 0;
    const unsigned live = m >= 32 ? kFull : ((1u << m) - 1u);
    Chunk cur;
    decode(settle(have_next ? dnext : load_desc(base, upto), base, upto), lane < m, cur);
    if (timed_out) break;
    {
      const long long nb = base + 32, nneed = n - nb < 32 ? n : nb + 32;
      have_next = !stop && nb < n && (long long)(wm >> 1) >= nneed;
      if (have_next) dnext = load_desc(nb, nneed);  // in flight while this chunk runs
    }
    // the oldest pending chunk must be final before its slot is reused
    resolve(std::integral_constant<int, L>{}, chunk - 1, vpre, vhave);
#pragma unroll
    for (int j = L; j > 0; --j) {
      C[j] = C[j - 1]; LV[j] = LV[j - 1]; RB[j] = RB[j - 1]; FIN[j] = FIN[j - 1];
#pragma unroll
      for (int u = 0; u < V; ++u) ck[j][u] = ck[j - 1][u];
    }
    C[0] = cur; LV[0] = live; FIN[0] = false;
#pragma unroll
    for (int u = 0; u < V; ++u) ck[0][u] = wr[u];
    unsigned gb, rb;
    exec(cur, live, 0u, gb, rb);
    RB[0] = rb;
    publish(chunk, gb);
    if (lane == 0) wm = ld_relaxed_u64(&a.out->dvalid);  // for the next chunk
  }
  // drain: every pending chunk final, oldest first
  if (!timed_out) {
    const long long newest = chunk - 1;
    if constexpr (L >= 4) resolve(std::integral_constant<int, (L >= 4 ? 4 : 0)>{}, newest);
    if constexpr (L >= 3) resolve(std::integral_constant<int, (L >= 3 ? 3 : 0)>{}, newest);
    resolve(std::integral_constant<int, 2>{}, newest);
    resolve(std::integral_constant<int, 1>{}, newest);
    resolve(std::integral_constant<int, 0>{}, newest);
  }
  if (timed_out) {
    if (lane == 0) atomicCAS(&a.out->status, PS_OK, PS_E_TIMEOUT);
    return;
  }
  // a non-finite result (server.py:38-41): the run stops with the worker named
  if (__any_sync(kFull, diverged >= 0) && lane == 0)
    if (atomicCAS(&a.out->status, PS_OK, PS_E_DIVERGED) == PS_OK) a.out->diverged_worker = diverged;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    if (j < hi) W[j] = wr[u];
  }
  if (lane == 0) atomicMax(&a.out->t_data_done, globaltimer_ns());
  if (dw == 0 && lane == 0) {
    a.out->applied = applied;
    a.out->rejected = rejected;
  }
}

// V: float4 per lane of register-resident weights (0 = in HBM);
// CTL: control tables in registers -- 2/4/8: scalar, replicated in every lane
// (fastest for few workers, ctl_regs.cuh); 32: one worker per lane
// (ctl_lanes.cuh); 0: shared memory (any P <= 64).
template <int V, int CTL>
__global__ void __launch_bounds__(kSimThreads) k_sim(SimArgs a) {
  __shared__ CtlState s;
  __shared__ __align__(8) unsigned s_ring[kRing];
  for (int i = threadIdx.x; i < kRing; i += blockDim.x) s_ring[i] = 0;
  __syncthreads();
  // CTA 0 is the control warp alone: no data warp competes with it for its
  // SM sub-partition's issue slot (the scheduler favours higher warp ids).
  if (blockIdx.x == 0) {
    if (threadIdx.x >= 32) {
      if (a.mode == 1 && threadIdx.x < 64) emit_warp_replay(a);  // beside the gate warp
      if constexpr (CTL == 2 || CTL == 4 || CTL == 8)
        if (a.mode == 1 && threadIdx.x >= 64 && threadIdx.x < 96) predict_warp_replay<CTL>(a);
      return;
    }
    if (a.mode == 1) {
      if constexpr (CTL == 2 || CTL == 4 || CTL == 8) gate_warp_replay<CTL>(a, &s.gate);
      else gate_warp_replay<0>(a, &s.gate);
      return;
    }
    if constexpr (CTL == 32) control_warp_lanes(a);
    else if constexpr (CTL > 0) control_warp_regs<CTL>(a);
    else control_warp(a, s);
    return;
  }
  const unsigned dw = ((blockIdx.x - 1) * kSimThreads + threadIdx.x) >> 5;
  if (a.mode == 1) {
    // speculation keeps L+1 checkpoints of the slice in registers: for the
    // wide slices (V >= 8) the scan-ahead path is the one without spills
    if constexpr (V > 0 && V <= 4) data_warp_replay_spec<V>(a, dw, s_ring, kSimThreads / 32);
    else data_warp_replay<V>(a, dw, s_ring, kSimThreads / 32);
  }
  else data_warp<V>(a, dw, s_ring, kSimThreads / 32);
}

// The replay alone with NT threads per CTA (select_replay_nt): fewer, wider
// data warps per SM -- the per-call control of a warp is the same whatever
// its slice width, so wider slices spend it on more data.
template <int V, int CTL, int NT, int KG4>
__global__ void __launch_bounds__(NT, 1) k_replay_nt(SimArgs a) {
  __shared__ ps_gate_state sg;
  __shared__ __align__(8) unsigned s_ring[kRing];
  for (int i = threadIdx.x; i < kRing; i += blockDim.x) s_ring[i] = 0;
  __syncthreads();
  if (blockIdx.x == 0) {
    if (threadIdx.x >= 32) {
      if (threadIdx.x < 64) emit_warp_replay(a);  // beside the gate warp
      else if (threadIdx.x < 96) predict_warp_replay<CTL>(a);
      return;
    }
    gate_warp_replay<CTL>(a, &sg);
    return;
  }
  const unsigned dw = ((blockIdx.x - 1) * NT + threadIdx.x) >> 5;
  data_warp_replay_spec<V, KG4>(a, dw, s_ring, NT / 32);
}

// ps_replay_ceiling: the replay's data warps with the control taken out (see
// include/dssp_ps.h). Same slice layout and load / store instructions as
// data_warp_replay_spec; the call stream is fixed (apply, pull, apply, ...).
template <int V>
__global__ void __launch_bounds__(kSimThreads, 1) k_replay_ceiling(const float4* W, float4* rep, const float4* upd,
                                                                long long nv, long long dv4, int pulls,
                                                                int applies, float lr, float4* sink,
                                                                unsigned n_data_warps) {
  if (blockIdx.x == 0) return;  // the replay's CTA 0 is the gate
  const int lane = threadIdx.x & 31;
  const long long dw = ((long long)(blockIdx.x - 1) * blockDim.x + threadIdx.x) >> 5;
  const long long per = (nv + n_data_warps - 1) / n_data_warps;
  const long long lo = dw * per < nv ? dw * per : nv, hi = lo + per < nv ? lo + per : nv;
  float4 w[V];
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long j = lo + lane + 32ll * u;
    w[u] = j < hi ? W[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const int n = pulls > applies ? pulls : applies;
  for (int c = 0; c < n; ++c) {
    if (c < applies) {
      float4 g[V];
      load_slice<V, true>(g, upd + (long long)(c & 7) * dv4, lo, hi, lane);
#pragma unroll
      for (int u = 0; u < V; ++u) w[u] = apply4(w[u], lr, g[u]);
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

// After the run: fold the data side's counters into the control block.
__global__ void k_sim_finish(Ctrl* ctrl, SimOut* out) {
  ctrl->gate.version += out->applied;
  ctrl->gate.rejected += out->rejected;
}

template <typename T>
__global__ void k_to_f32(const T* src, float* dst, long long n, long long dpad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < dpad; i += stride)
    dst[i] = i < n ? (float)src[i] : 0.f;
}

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
  ~DevGuard() { cudaSetDevice(prev); }
};

template <typename T>
int grow(ps_server* h, T** p, size_t* cap, size_t need) {
  if (*cap >= need && *p) return PS_OK;
  cudaFree(*p);
  *p = nullptr;
  PS_CK(h, cudaMalloc((void**)p, need * sizeof(T)));
  *cap = need;
  return PS_OK;
}

// One CTA per SM; the weight slice of every data warp lives in registers when
// it fits V float4 per lane (V in {1,2,4,8,16}), else in HBM (V = 0); the
// control warp's layout follows P (see k_sim).
int select_loop_kernel(ps_server* h, int P, int data_ctas, int* grid_out, const void** kern_out) {
  int grid = data_ctas > 0 ? data_ctas + 1 : h->sm_count;
  if (grid > h->sm_count) grid = h->sm_count;
  if (grid < 2) grid = 2;
  const long long dwarps = (long long)(grid - 1) * (kSimThreads / 32);
  const long long per = (h->nv + dwarps - 1) / dwarps;
  const long long need_v = (per + 31) / 32;
  const int vi = need_v <= 1 ? 0 : need_v <= 2 ? 1 : need_v <= 4 ? 2 : need_v <= 8 ? 3 : need_v <= 16 ? 4 : 5;
  const int pi = P <= 2 ? 0 : P <= 4 ? 1 : P <= 8 ? 2 : P <= kLaneP ? 3 : 4;
  static const void* const table[6][5] = {
      {(const void*)k_sim<1, 2>, (const void*)k_sim<1, 4>, (const void*)k_sim<1, 8>, (const void*)k_sim<1, 32>, (const void*)k_sim<1, 0>},
      {(const void*)k_sim<2, 2>, (const void*)k_sim<2, 4>, (const void*)k_sim<2, 8>, (const void*)k_sim<2, 32>, (const void*)k_sim<2, 0>},
      {(const void*)k_sim<4, 2>, (const void*)k_sim<4, 4>, (const void*)k_sim<4, 8>, (const void*)k_sim<4, 32>, (const void*)k_sim<4, 0>},
      {(const void*)k_sim<8, 2>, (const void*)k_sim<8, 4>, (const void*)k_sim<8, 8>, (const void*)k_sim<8, 32>, (const void*)k_sim<8, 0>},
      {(const void*)k_sim<16, 2>, (const void*)k_sim<16, 4>, (const void*)k_sim<16, 8>, (const void*)k_sim<16, 32>, (const void*)k_sim<16, 0>},
      {(const void*)k_sim<0, 2>, (const void*)k_sim<0, 4>, (const void*)k_sim<0, 8>, (const void*)k_sim<0, 32>, (const void*)k_sim<0, 0>}};
  const void* kern = table[vi][pi];
  // the occupancy of each instantiation, queried once per process (it is a
  // driver round trip on every run otherwise)
  static int occupancy[6][5] = {{-1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1},
                                {-1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1}, {-1, -1, -1, -1, -1}};
  int per_sm = occupancy[vi][pi];
  if (per_sm < 0) {
    PS_CK(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSimThreads, 0));
    occupancy[vi][pi] = per_sm;
  }
  if (grid > per_sm * h->sm_count) grid = per_sm * h->sm_count;
  if (grid < 2) return ps_fail(h, PS_E_CUDA, "k_sim cannot be resident");
  *grid_out = grid;
  *kern_out = kern;
  return PS_OK;
}

// PS_REPLAY_NT=128: the replay on 4 data warps per CTA with twice the slice
// each (P <= 8, V <= 4). With branched call slots it beat the 8-warp k_sim
// (0.431 vs 0.445 ms, profiles/r2_c2_replay_narrow_cta.txt); with the
// straight-line slots the 8-warp kernel is faster again (0.36-0.37 vs 0.41
// ms, profiles/r2_c2_replay_straight_slots.txt), so this is opt-in.
bool select_replay_nt(ps_server* h, int P, int data_ctas, int* grid_out, const void** kern_out, int* nt_out) {
  const char* v = getenv("PS_REPLAY_NT");
  if (!v || atoi(v) != 128 || P > 8) return false;
  int grid = data_ctas > 0 ? data_ctas + 1 : h->sm_count;
  if (grid > h->sm_count) grid = h->sm_count;
  if (grid < 2) grid = 2;
  const long long dwarps = (long long)(grid - 1) * 4;
  const long long need_v = ((h->nv + dwarps - 1) / dwarps + 31) / 32;
  if (need_v > 4) return false;
  const int vi = need_v <= 2 ? 0 : 1;
  const int pi = P <= 2 ? 0 : P <= 4 ? 1 : 2;
  static const void* const table[2][3] = {
      {(const void*)k_replay_nt<2, 2, 128, 2>, (const void*)k_replay_nt<2, 4, 128, 2>, (const void*)k_replay_nt<2, 8, 128, 2>},
      {(const void*)k_replay_nt<4, 2, 128, 2>, (const void*)k_replay_nt<4, 4, 128, 2>, (const void*)k_replay_nt<4, 8, 128, 2>}};
  static int occupancy[2][3] = {{-1, -1, -1}, {-1, -1, -1}};
  const void* kern = table[vi][pi];
  int per_sm = occupancy[vi][pi];
  if (per_sm < 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0) != cudaSuccess) {
      cudaGetLastError();
      per_sm = 0;
    }
    occupancy[vi][pi] = per_sm;
  }
  if (per_sm < 1 || grid > per_sm * h->sm_count) return false;
  *grid_out = grid;
  *kern_out = kern;
  *nt_out = 128;
  return true;
}

}  // namespace

extern "C" {

int ps_sim_run(ps_server* h, const ps_sim_config* sc, ps_sim_result* res) {
  DevGuard guard(h->dev);
  if (int prc = ps_resident_pause(h)) return prc;
  std::memset(res, 0, sizeof(*res));
  const int P = h->cfg.worker_count;
  if (sc->budget < 0) return ps_fail(h, PS_E_VALUE, "budget must be >= 0");
  if (sc->mode != 0 && sc->mode != 2) return ps_fail(h, PS_E_VALUE, "mode must be 0 or 2");
  if (sc->mode == 2 && (P > kLaneP || !(sc->time_scale > 0)))
    return ps_fail(h, PS_E_VALUE, "free-running runs need P <= 32 and time_scale > 0");
  if (sc->mode == 2 && !h->habort) {
    PS_CK(h, cudaHostAlloc((void**)&h->habort, sizeof(int), cudaHostAllocMapped));
    PS_CK(h, cudaHostGetDevicePointer((void**)&h->habort_dev, h->habort, 0));
  }
  if (h->habort) *(volatile int*)h->habort = 0;
  if (sc->grad_kind == PS_GRAD_SYNTHETIC && (!sc->synthetic || sc->n_synthetic < 1))
    return ps_fail(h, PS_E_VALUE, "synthetic updates need a device buffer");
  if (sc->grad_kind == PS_GRAD_BOWL && !sc->center) return ps_fail(h, PS_E_VALUE, "bowl needs a center");
  if (!sc->compute_time && sc->budget > 0) return ps_fail(h, PS_E_VALUE, "compute_time missing");
  ps_sim_buffers& b = h->sim;
  const size_t budget = (size_t)sc->budget;
  const size_t slots = (size_t)P * budget + 1;
  const size_t ops = (size_t)P * (3 * budget + 2) + 8;
  int rc;
  size_t cap;
  if (b.ops_cap < ops || !b.ops) {
    cudaFree(b.ops);
    b.ops = nullptr;
    PS_CK(h, cudaMalloc(&b.ops, ops * sizeof(Op)));
    PS_CK(h, cudaMemsetAsync(b.ops, 0, ops * sizeof(Op), h->stream));  // tag 0 = never valid
    b.ops_cap = ops;
    b.tag = 0;
  }
  b.tag = (b.tag + 1) & 0xffffu;
  if (b.tag == 0) {  // tag space wrapped: clear stale words once
    PS_CK(h, cudaMemsetAsync(b.ops, 0, b.ops_cap * sizeof(Op), h->stream));
    b.tag = 1;
  }
  cap = b.slots_cap;
  if (cap < slots || !b.gcount) {
    cudaFree(b.gcount);
    b.gcount = nullptr;
    PS_CK(h, cudaMalloc(&b.gcount, slots * sizeof(unsigned)));
    b.slots_cap = slots;
  }
  if (!b.out) PS_CK(h, cudaMalloc(&b.out, sizeof(SimOut)));
  if (b.P != P || !b.rep) {
    cudaFree(b.rep); cudaFree(b.gbuf);
    b.rep = nullptr; b.gbuf = nullptr;
    PS_CK(h, cudaMalloc(&b.rep, (size_t)P * 2 * h->dpad * sizeof(float)));
    PS_CK(h, cudaMalloc(&b.gbuf, (size_t)P * h->dpad * sizeof(float)));
    PS_CK(h, cudaMemsetAsync(b.rep, 0, (size_t)P * 2 * h->dpad * sizeof(float), h->stream));
    b.P = P;
  }
  if (!b.center) {
    PS_CK(h, cudaMalloc(&b.center, h->dpad * sizeof(float)));
    PS_CK(h, cudaMemsetAsync(b.center, 0, h->dpad * sizeof(float), h->stream));
  }
  if (sc->grad_kind == PS_GRAD_BOWL) {
    const size_t esz = sc->center_dtype == PS_F64 ? 8 : 4;
    void* tmp = nullptr;
    PS_CK(h, cudaMalloc(&tmp, h->d * esz));
    PS_CK(h, cudaMemcpyAsync(tmp, sc->center, h->d * esz, cudaMemcpyHostToDevice, h->stream));
    if (esz == 8)
      k_to_f32<double><<<h->sm_count * 4, 256, 0, h->stream>>>((const double*)tmp, b.center, h->d, h->dpad);
    else
      k_to_f32<float><<<h->sm_count * 4, 256, 0, h->stream>>>((const float*)tmp, b.center, h->d, h->dpad);
    PS_CK(h, cudaStreamSynchronize(h->stream));
    cudaFree(tmp);
  }
  const size_t nct = (size_t)P * budget + 1;
  cap = b.ctime_cap; if ((rc = grow(h, &b.ctime, &cap, nct))) return rc; b.ctime_cap = cap;
  if (budget) PS_CK(h, cudaMemcpyAsync(b.ctime, sc->compute_time, (size_t)P * budget * sizeof(double),
                                       cudaMemcpyHostToDevice, h->stream));
  // trace rows: every event yields one row; events <= P*(5*budget+2)
  const size_t trace_need = sc->record_trace ? (size_t)P * (5 * budget + 2) + 8 : 1;
  cap = b.trace_cap; if ((rc = grow(h, &b.trace, &cap, trace_need))) return rc; b.trace_cap = cap;
  const size_t loss_need = sc->loss_every > 0 ? (size_t)P * budget / sc->loss_every + 2 : 1;
  cap = b.loss_cap; if ((rc = grow(h, &b.losses, &cap, loss_need))) return rc; b.loss_cap = cap;
  PS_CK(h, cudaMemsetAsync(b.gcount, 0, slots * sizeof(unsigned), h->stream));
  PS_CK(h, cudaMemsetAsync(b.out, 0, sizeof(SimOut), h->stream));
  PS_CK(h, cudaMemsetAsync(b.losses, 0, loss_need * sizeof(double), h->stream));

  int grid = 0;
  const void* kern = nullptr;
  if ((rc = select_loop_kernel(h, P, sc->data_ctas, &grid, &kern))) return rc;

  SimArgs a{};
  a.P = P;
  a.budget = sc->budget;
  a.grad_kind = sc->grad_kind;
  a.n_synth = sc->n_synthetic > 0 ? sc->n_synthetic : 1;
  a.loss_every = sc->loss_every;
  a.record_trace = sc->record_trace;
  a.reset_gate = sc->reset_gate;
  a.nv = h->nv;
  a.dpad = h->dpad;
  a.max_events = sc->max_events;
  a.trace_cap = (long long)trace_need;
  a.loss_cap = (long long)loss_need;
  a.ops_cap = (long long)ops;
  a.comm_delay = sc->comm_delay;
  a.lr = (float)h->cfg.learning_rate;
  a.W = h->w[h->cur];
  a.rep = b.rep;
  a.gbuf = b.gbuf;
  a.center = b.center;
  a.synth = sc->synthetic;
  a.ctime = b.ctime;
  a.ops = (Op*)b.ops;
  a.gword = b.gcount;
  a.tag = b.tag;
  a.n_ctas = (unsigned)(grid - 1);  // CTA 0 is the control warp alone
  a.trace = b.trace;
  a.losses = b.losses;
  a.ctrl = h->ctrl;
  a.out = (SimOut*)b.out;
  a.n_data_warps = (unsigned)((grid - 1) * (kSimThreads / 32));
  a.timeout_ns = 20ull * 1000 * 1000 * 1000;
  a.base_version = h->hctrl->gate.version;
  b.last_base_version = a.base_version;
  a.mode = sc->mode;
  a.time_scale = sc->mode == 2 ? sc->time_scale : 1.0;
  a.deadline_ns = sc->mode == 2 && sc->deadline_s > 0 ? (unsigned long long)(sc->deadline_s * 1e9)
                                                      : 0xffffffffffffull;
  a.abort_flag = sc->mode == 2 ? h->habort_dev : nullptr;
  if (sc->mode == 2) a.timeout_ns = a.deadline_ns + 20ull * 1000 * 1000 * 1000;
  void* args[] = {&a};
  PS_CK(h, cudaEventRecord(h->ev0, h->stream));
  if ((rc = ps_order_after_producer(h))) return rc;  // resident updates may come from the caller's stream
  PS_CK(h, cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kSimThreads), args, 0, h->stream));
  PS_CK(h, cudaEventRecord(h->ev1, h->stream));
  k_sim_finish<<<1, 1, 0, h->stream>>>(h->ctrl, (SimOut*)b.out);
  PS_CK(h, cudaGetLastError());
  SimOut o{};
  PS_CK(h, cudaMemcpyAsync(&o, b.out, sizeof(SimOut), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->last_ms = ms;
  PS_CK(h, cudaMemcpy(h->hctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  h->cur = h->hctrl->cur;
  res->events = o.events;
  res->pushes = o.pushes;
  res->applied = o.applied;
  res->rejected = o.rejected;
  res->trace_rows = o.trace_rows < a.trace_cap ? o.trace_rows : a.trace_cap;
  res->loss_samples = sc->loss_every > 0 ? o.applied / sc->loss_every : 0;
  res->unfinished = o.unfinished;
  res->status = o.status;
  res->diverged_worker = o.diverged_worker;
  res->device_ms = ms;
  res->control_ms = o.t_control_done > o.t_start ? (o.t_control_done - o.t_start) * 1e-6 : 0.0;
  res->data_ms = o.t_data_done > o.t_start ? (o.t_data_done - o.t_start) * 1e-6 : 0.0;
  b.last_trace_rows = res->trace_rows;
  b.last_loss_samples = res->loss_samples < a.loss_cap ? res->loss_samples : a.loss_cap;
  b.last_loss_every = sc->loss_every;
  if (o.status == PS_E_TIMEOUT) {
    if (sc->mode == 2)
      return ps_fail(h, PS_E_TIMEOUT, "free-running run aborted (deadline or abort) with workers unfinished");
    return ps_fail(h, PS_E_TIMEOUT, "device watchdog fired in ps_sim_run");
  }
  if (o.status == PS_E_DIVERGED)
    return ps_fail(h, PS_E_DIVERGED, "weights went non-finite on worker " + std::to_string(o.diverged_worker));
  if (o.status == PS_E_BUDGET)
    return ps_fail(h, PS_E_BUDGET, "event budget " + std::to_string(sc->max_events) + " exceeded");
  if (o.status == PS_E_PROTOCOL) return ps_fail(h, PS_E_PROTOCOL, "protocol violation in device run");
  if (o.unfinished) {
    res->status = PS_E_DEADLOCK;
    return ps_fail(h, PS_E_DEADLOCK, "simulation deadlocked");
  }
  return PS_OK;
}

int ps_replay_run(ps_server* h, const ps_replay_call* calls, int64_t n, const float* synthetic,
                  int32_t n_synthetic, int32_t reset_gate, int32_t data_ctas, ps_sim_result* res) {
  DevGuard guard(h->dev);
  if (int prc = ps_resident_pause(h)) return prc;
  std::memset(res, 0, sizeof(*res));
  const int P = h->cfg.worker_count;
  if (n < 0 || (n > 0 && !calls)) return ps_fail(h, PS_E_VALUE, "bad call list");
  if (!synthetic || n_synthetic < 1) return ps_fail(h, PS_E_VALUE, "replay needs resident updates");
  // a decision word carries the released set in bits 8..63
  if (P > 55) return ps_fail(h, PS_E_VALUE, "replay supports at most 55 workers");
  // the data warps address a slice by a 32-bit float4 offset
  if ((unsigned long long)P * (unsigned long long)(n_synthetic > 2 ? n_synthetic : 2) * (unsigned long long)(h->dpad / 4) >= (1ull << 32))
    return ps_fail(h, PS_E_VALUE, "resident updates beyond 2^32 float4 (64 GB)");
  ps_sim_buffers& b = h->sim;
  int rc;
  size_t cap;
  // (no op log: the data warps number the calls themselves)
  // replay verdicts: one {CTAs done, non-finite bits} pair per 32-call chunk
  const size_t slots = 2 * ((size_t)n / 32 + 4);
  if (b.slots_cap < slots || !b.gcount) {
    cudaFree(b.gcount);
    b.gcount = nullptr;
    PS_CK(h, cudaMalloc(&b.gcount, slots * sizeof(unsigned)));
    b.slots_cap = slots;
  }
  if (!b.out) PS_CK(h, cudaMalloc(&b.out, sizeof(SimOut)));
  if (b.P != P || !b.rep) {
    cudaFree(b.rep); cudaFree(b.gbuf);
    b.rep = nullptr; b.gbuf = nullptr;
    PS_CK(h, cudaMalloc(&b.rep, (size_t)P * 2 * h->dpad * sizeof(float)));
    PS_CK(h, cudaMalloc(&b.gbuf, (size_t)P * h->dpad * sizeof(float)));
    b.P = P;
  }
  cap = b.calls_cap;
  if ((rc = grow(h, (ReplayCall**)&b.calls, &cap, (size_t)n + 1))) return rc;
  b.calls_cap = cap;
  cap = b.dec_cap;
  if ((rc = grow(h, &b.decisions, &cap, (size_t)n + 1))) return rc;
  b.dec_cap = cap;
  long long n_data = 0;  // pulls + applies: the most descriptors the gate can publish
  for (int64_t i = 0; i < n; ++i) n_data += (calls[i].kind == PS_CALL_PULL || calls[i].kind == PS_CALL_APPLY);
  cap = b.dstream_cap;
  // + the emitter's per-chunk prefix counts (8 B) and masks (4 B)
  if ((rc = grow(h, &b.dstream, &cap, (size_t)n_data + 32 + 2 * ((size_t)n / 32 + 3)))) return rc;
  if (cap != b.dstream_cap) {  // fresh words: no tag of any run
    PS_CK(h, cudaMemsetAsync(b.dstream, 0, cap * sizeof(unsigned long long), h->stream));
    b.dtag = 0;
  }
  b.dstream_cap = cap;
  cap = b.pred_cap;
  if ((rc = grow(h, &b.pred, &cap, (size_t)n + 32))) return rc;
  if (cap != b.pred_cap) PS_CK(h, cudaMemsetAsync(b.pred, 0, cap * sizeof(unsigned long long), h->stream));
  b.pred_cap = cap;
  if (++b.dtag == 0) {  // 32-bit tag space wrapped: clear stale words once
    PS_CK(h, cudaMemsetAsync(b.dstream, 0, b.dstream_cap * sizeof(unsigned long long), h->stream));
    PS_CK(h, cudaMemsetAsync(b.pred, 0, b.pred_cap * sizeof(unsigned long long), h->stream));
    b.dtag = 1;
  }
  if (n) PS_CK(h, cudaMemcpyAsync(b.calls, calls, (size_t)n * sizeof(ReplayCall), cudaMemcpyHostToDevice,
                                  h->stream));
  PS_CK(h, cudaMemsetAsync(b.gcount, 0, slots * sizeof(unsigned), h->stream));
  PS_CK(h, cudaMemsetAsync(b.out, 0, sizeof(SimOut), h->stream));
  int grid = 0, nt = kSimThreads;
  const void* kern = nullptr;
  if (!select_replay_nt(h, P, data_ctas, &grid, &kern, &nt))
    if ((rc = select_loop_kernel(h, P, data_ctas, &grid, &kern))) return rc;
  SimArgs a{};
  a.mode = 1;
  a.P = P;
  a.grad_kind = PS_GRAD_SYNTHETIC;
  a.n_synth = n_synthetic;
  a.reset_gate = reset_gate;
  a.nv = h->nv;
  a.dpad = h->dpad;
  a.trace_cap = (long long)b.dec_cap;
  a.ops_cap = 0;
  a.lr = (float)h->cfg.learning_rate;
  a.W = h->w[h->cur];
  a.rep = b.rep;
  a.gbuf = b.gbuf;
  a.synth = synthetic;
  a.ops = nullptr;
  a.gword = b.gcount;
  a.n_ctas = (unsigned)(grid - 1);
  a.calls = (const ReplayCall*)b.calls;
  a.n_calls = n;
  a.dstream = b.dstream;
  a.n_data = n_data;
  a.pred = b.pred;
  {
    const char* v = getenv("PS_REPLAY_CTL_AHEAD");
    a.pred_ahead = v ? atoi(v) != 0 : 1;
  }
  a.tag = b.dtag;  // the descriptor words of this run
  a.decisions = b.decisions;
  a.ctrl = h->ctrl;
  a.out = (SimOut*)b.out;
  a.n_data_warps = (unsigned)((grid - 1) * (nt / 32));
  a.timeout_ns = 20ull * 1000 * 1000 * 1000;
  a.base_version = h->hctrl->gate.version;
  {
    const char* v = getenv("PS_REPLAY_GATE_SCAN");
    a.gate_scan = v ? atoi(v) != 0 : 1;
  }
  void* args[] = {&a};
  PS_CK(h, cudaEventRecord(h->ev0, h->stream));
  if ((rc = ps_order_after_producer(h))) return rc;  // resident updates may come from the caller's stream
  PS_CK(h, cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(nt), args, 0, h->stream));
  PS_CK(h, cudaEventRecord(h->ev1, h->stream));
  k_sim_finish<<<1, 1, 0, h->stream>>>(h->ctrl, (SimOut*)b.out);
  PS_CK(h, cudaGetLastError());
  SimOut o{};
  PS_CK(h, cudaMemcpyAsync(&o, b.out, sizeof(SimOut), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->last_ms = ms;
  PS_CK(h, cudaMemcpy(h->hctrl, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  h->cur = h->hctrl->cur;
  res->events = o.events;
  res->pushes = o.pushes;
  res->applied = o.applied;
  res->rejected = o.rejected;
  res->trace_rows = o.trace_rows;
  res->status = o.status;
  res->diverged_worker = o.diverged_worker;
  res->device_ms = ms;
  res->control_ms = o.t_control_done > o.t_start ? (o.t_control_done - o.t_start) * 1e-6 : 0.0;
  res->data_ms = o.t_data_done > o.t_start ? (o.t_data_done - o.t_start) * 1e-6 : 0.0;
  b.last_decisions = o.trace_rows;
  if (o.status == PS_E_TIMEOUT) return ps_fail(h, PS_E_TIMEOUT, "device watchdog fired in ps_replay_run");
  if (o.status == PS_E_DIVERGED)
    return ps_fail(h, PS_E_DIVERGED, "weights went non-finite on worker " + std::to_string(o.diverged_worker));
  if (o.status == PS_E_PROTOCOL) return ps_fail(h, PS_E_PROTOCOL, "protocol violation in the replayed calls");
  return PS_OK;
}

int ps_replay_ceiling(ps_server* h, int32_t pulls, int32_t applies, int32_t reps, double* best_ms) {
  DevGuard guard(h->dev);
  if (pulls < 0 || applies < 0 || reps < 1) return ps_fail(h, PS_E_VALUE, "pulls, applies >= 0 and reps >= 1");
  int grid = 0, nt = kSimThreads;
  const void* kern = nullptr;
  int rc = PS_OK;
  // the replay's own grid and CTA shape for this vector (P = 4: the C2 shape)
  if (!select_replay_nt(h, 4, 0, &grid, &kern, &nt))
    if ((rc = select_loop_kernel(h, 4, 0, &grid, &kern))) return rc;
  const long long dwarps = (long long)(grid - 1) * (nt / 32);
  const long long need_v = ((h->nv + dwarps - 1) / dwarps + 31) / 32;
  if (need_v > 4) return ps_fail(h, PS_E_VALUE, "the ceiling probe covers register-resident slices (V <= 4)");
  float4 *scratch = nullptr;
  const size_t dv4 = (size_t)h->dpad / 4;
  PS_CK(h, cudaMalloc(&scratch, (17 * dv4) * sizeof(float4)));  // 8 replicas, 8 updates, 1 sink
  double best = 1e30;
  if (cudaMemsetAsync(scratch, 0, 17 * dv4 * sizeof(float4), h->stream) != cudaSuccess) rc = PS_E_CUDA;
  for (int r = 0; r < reps && rc == PS_OK; ++r) {
    cudaEventRecord(h->ev0, h->stream);
    const float4* W = reinterpret_cast<const float4*>(h->w[h->cur]);
    float4* rep = scratch;
    const float4* upd = scratch + 8 * dv4;
    float4* sink = scratch + 16 * dv4;
    const float lr = (float)h->cfg.learning_rate;
    const unsigned ndw = (unsigned)dwarps;
    if (need_v <= 1) k_replay_ceiling<1><<<grid, nt, 0, h->stream>>>(W, rep, upd, h->nv, dv4, pulls, applies, lr, sink, ndw);
    else if (need_v <= 2) k_replay_ceiling<2><<<grid, nt, 0, h->stream>>>(W, rep, upd, h->nv, dv4, pulls, applies, lr, sink, ndw);
    else k_replay_ceiling<4><<<grid, nt, 0, h->stream>>>(W, rep, upd, h->nv, dv4, pulls, applies, lr, sink, ndw);
    cudaEventRecord(h->ev1, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess) { rc = PS_E_CUDA; break; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    if (ms < best) best = ms;
  }
  cudaFree(scratch);
  if (rc) return ps_fail(h, rc, "replay ceiling probe failed");
  *best_ms = best;
  return PS_OK;
}

int ps_replay_decisions(ps_server* h, int64_t* out, int64_t cap, int64_t* n) {
  DevGuard guard(h->dev);
  *n = h->sim.last_decisions;
  const int64_t m = h->sim.last_decisions < cap ? h->sim.last_decisions : cap;
  if (m > 0) PS_CK(h, cudaMemcpy(out, h->sim.decisions, m * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_replay_read_replica(ps_server* h, int32_t worker, int32_t buf, float* dst_host) {
  DevGuard guard(h->dev);
  if (!h->sim.rep || worker < 0 || worker >= h->sim.P || buf < 0 || buf > 1 || !dst_host)
    return ps_fail(h, PS_E_VALUE, "no such replica (run a replay or simulation first)");
  const float* src = h->sim.rep + ((size_t)worker * 2 + buf) * h->dpad;
  PS_CK(h, cudaMemcpyAsync(dst_host, src, h->d * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  PS_CK(h, cudaStreamSynchronize(h->stream));
  return PS_OK;
}

int ps_sim_trace(ps_server* h, ps_trace_row* rows, int64_t cap, int64_t* n) {
  DevGuard guard(h->dev);
  const int64_t m = h->sim.last_trace_rows < cap ? h->sim.last_trace_rows : cap;
  *n = h->sim.last_trace_rows;
  if (m > 0) PS_CK(h, cudaMemcpy(rows, h->sim.trace, m * sizeof(ps_trace_row), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_sim_losses(ps_server* h, int64_t* versions, double* losses, int64_t cap, int64_t* n) {
  DevGuard guard(h->dev);
  const int64_t m = h->sim.last_loss_samples < cap ? h->sim.last_loss_samples : cap;
  *n = h->sim.last_loss_samples;
  if (m > 0) PS_CK(h, cudaMemcpy(losses, h->sim.losses, m * sizeof(double), cudaMemcpyDeviceToHost));
  const int64_t le = h->sim.last_loss_every;
  for (int64_t i = 0; i < m; ++i) versions[i] = (h->sim.last_base_version / le + i + 1) * le;
  return PS_OK;
}

}  // extern "C"
