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
// each). A whole run of steps is ONE persistent cooperative kernel on every
// rank (k_shard_run), with no host in the loop and no collective; per step:
//
//   push              CTA 0 of rank r: once every owner's slice of worker r's
//                     previous pull has landed, release-store ready = t into
//                     every owner's flag array.
//   data CTAs         owner r waits for all G ready flags, then streams its
//                     shard once: w' = w - lr*g_p for p in ticket order, each
//                     g_p slice read straight from worker p's HBM over NVLink
//                     (P2P loads, payload crosses once), w' written to the back
//                     buffer AND stored into every worker's replica (the pull,
//                     handle_pull server.py:84-91, as P2P stores -- no gather
//                     pass). Per-element order == global push order, no atomics
//                     on weights. While streaming it scans the update slices;
//                     the last CTA exchanges these verdicts with the other
//                     owners (an update with ANY non-finite element is
//                     rejected whole, server.py:65-67), commits by flipping the
//                     buffers (or, rarely, redoes its slice without the
//                     rejected updates; a non-finite result leaves w unchanged,
//                     server.py:38-41) and flags pulled = t to every worker.
//   gate CTA          one extra CTA runs the replicated gate (gate.cuh) for the
//                     group from shared memory while the data CTAs stream --
//                     every rank decides the same group from the same inputs,
//                     so no gate traffic crosses NVLink.
//
// Waits are only ever on flags written by OTHER GPUs' kernels that never wait
// on the waiter's later work, so the protocol cannot deadlock; every spin has a
// watchdog that aborts the kernel instead of hanging the GPU.
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "gate.cuh"

using namespace dssp;

namespace {

constexpr int kMaxRanks = 16;
constexpr int kSchedStride = 2 + kMaxRanks;  // ps_shard_run_groups row: n, pull mask, order
constexpr int kThreads = 256;
// per-rank flag words written by peers: ready[G] | V(t) in slot t % 4 [4][G]
// | F(t) redo done [G] | D first diverged step [G]. Four V slots: with the
// one-step-deep pipeline an owner can publish V(t+2) before a slow reader has
// read V(t), never V(t+4).
constexpr int kFlagWords = 7 * kMaxRanks;
constexpr int kVSlots = 4;
// streaming-loop shape (build-time knobs for tuning experiments): minimum
// resident CTAs per SM the register budget must allow, and float4 per thread
// per trip for G <= 2 / <= 4 / more
#ifndef PS_SHARD_MINB
#define PS_SHARD_MINB 2
#endif
#ifndef PS_SHARD_U2
#define PS_SHARD_U2 4
#endif
#ifndef PS_SHARD_U4
#define PS_SHARD_U4 2
#endif
#ifndef PS_SHARD_U8
#define PS_SHARD_U8 1
#endif
// cache policy of the streaming loop's accesses (build-time knob): 0 = default;
// 1 = replica stores evict-first (st.global.cs: nobody on this GPU reads them
// back in the run); 2 = also the shard loads L1::no_allocate
#ifndef PS_SHARD_CACHE
#define PS_SHARD_CACHE 0
#endif
__device__ __forceinline__ float4 shard_ld(const float4* p) {
  if constexpr (PS_SHARD_CACHE >= 2) {
    // coherent (not .nc: the rotation rewrites this buffer within the kernel)
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
  }
  return *p;
}
__device__ __forceinline__ void shard_st_w(float4* p, const float4& v) { *p = v; }
__device__ __forceinline__ void shard_st_rep(float4* p, const float4& v) {
  if constexpr (PS_SHARD_CACHE >= 1) __stcs(p, v);
  else *p = v;
}
__host__ __device__ constexpr int shard_unroll(int g) { return g <= 2 ? PS_SHARD_U2 : g <= 4 ? PS_SHARD_U4 : PS_SHARD_U8; }
constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct ShardPtrs {
  const float* w[kMaxRanks];            // each shard's weights (peer mappings)
  const float* upd[kMaxRanks];          // each worker's update buffer
  float* rep[kMaxRanks];                // each worker's replica (pull destination)
  unsigned long long* flags[kMaxRanks]; // each rank's flags: ready[G], pulled[G], verdict[G]
  long long lo[kMaxRanks];
};

struct ShardCtl {
  ps_gate_state gate;
  uint32_t bad;       // this step's non-finite bits (per ticket) and result bit 31
  int32_t status;
  int32_t _pad;
  unsigned long long trace_n;
  // Ticket order of the current push group: the seq order in which the
  // previous group's decisions scheduled the workers' GRANT_DELIVER events
  // (grant -> pusher first, then released ids ascending; simnet.py:192-201),
  // which every later event of the homogeneous chain inherits.
  int32_t order[2][kMaxRanks];  // [step parity]: this group's order, the next one's
  int32_t cur;  // which shard buffer holds the current weights
  int32_t _pad2;
  unsigned long long arrive_total;  // data-CTA arrivals over all steps (election)
  unsigned long long gate_done;     // last step whose decisions and next order are written
  unsigned long long committed;     // unused (kept for the host marks layout)
  unsigned long long redo_total;    // data-CTA arrivals at rejection redos (election)
  unsigned long long arrive_par[2]; // data-CTA arrivals of this run's even / odd steps
  uint32_t badp[2];                 // per-parity step verdict bits (see k_shard_run)
  int32_t div_sticky;               // a step of this server diverged
  int32_t no_lag;                   // PS_SHARD_NO_LAG: resolve every step in full
};

__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Profiling build only (-DPS_SHARD_PROFILE, tools/libdssp_ps_prof.so): sums
// of per-step phase durations on this rank, printed at the end of a run.
#ifdef PS_SHARD_PROFILE
__device__ unsigned long long g_prof[8];
__device__ unsigned long long g_t_resolved;
#define SPROF(stmt) stmt
#else
#define SPROF(stmt)
#endif

struct IpcBlob {
  cudaIpcMemHandle_t w, upd, rep, flags;
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
      __nanosleep(20);
    }
    if (acc_bad && (v & 1ull)) bad |= 1ull << q;
  }
  if (acc_bad) *acc_bad = bad;
  return true;
}

// One owner's streaming pass over its shard for one push group (the body of
// every step of k_shard_run, and of the one-sided NVLink probe): apply the
// live pushers' slices (`src[i]`, ticket order; G-1 of every G read over
// NVLink) to the shard in one read of it, write the new shard and store it
// into every pulling worker's replica (G-1 of them over NVLink), scanning the
// update slices and results for non-finite values. U consecutive float4 per
// thread per trip with all slices loaded first: U*G independent 128-bit loads
// in flight.
template <int G_MAX, int U>
__device__ __forceinline__ void stream_pass(const float4* wsrc, float4* wdst, const float4* const (&src)[G_MAX],
                                            unsigned live, unsigned pullm, const ShardPtrs& P, int G,
                                            long long lo, float lr, long long first, long long stride,
                                            long long nv, unsigned& gbad, unsigned& dbad) {
  for (long long base = first; base < nv; base += stride) {
    float4 g[U][G_MAX];
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * kThreads;
      if (j < nv) {
#pragma unroll
        for (int i = 0; i < G_MAX; ++i)
          if ((live >> i) & 1u) g[u][i] = ld_stream(src[i] + j);
        x[u] = shard_ld(wsrc + j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long j = base + (long long)u * kThreads;
      if (j < nv) {
#pragma unroll
        for (int i = 0; i < G_MAX; ++i)
          if ((live >> i) & 1u) {
            gbad |= nonfinite4(g[u][i]) ? (1u << i) : 0u;
            x[u] = apply4(x[u], lr, g[u][i]);
          }
        dbad |= nonfinite4(x[u]) ? 1u : 0u;
        shard_st_w(wdst + j, x[u]);
        // every worker's pull of this slice (handle_pull, server.py:84-91):
        // stored straight into each replica, G-1 of them over NVLink
#pragma unroll
        for (int q = 0; q < G_MAX; ++q)
          if (q < G && ((pullm >> q) & 1u)) shard_st_rep(reinterpret_cast<float4*>(P.rep[q] + lo) + j, x[u]);
      }
    }
  }
}

// Diagnostics only (ps_shard_stream_probe): this owner's streaming pass of a
// push group by every worker, repeated `reps` times, with NO flags and no
// peer participation -- so ncu can replay it in one process while the other
// ranks idle, and read its NVLink byte counters. It writes the shard's spare
// buffer and every replica's slice of this shard (the replicas' contents are
// not preserved: run it on a throwaway server).
template <int G_MAX>
__global__ void __launch_bounds__(kThreads, PS_SHARD_MINB)
k_shard_stream_probe(const float* __restrict__ w, float* __restrict__ spare, long long n_local, ShardPtrs P,
                     int G, int me, float lr, int reps) {
  constexpr int U = shard_unroll(G_MAX);
  const long long nv = (n_local + 3) >> 2;
  const long long lo = P.lo[me];
  const long long stride = (long long)gridDim.x * kThreads * U;
  const long long first = (long long)blockIdx.x * kThreads * U + threadIdx.x;
  const float4* src[G_MAX];
  unsigned live = 0;
#pragma unroll
  for (int i = 0; i < G_MAX; ++i) {
    src[i] = reinterpret_cast<const float4*>(P.upd[i < G ? i : 0] + lo);
    if (i < G) live |= 1u << i;
  }
  const unsigned pullm = G >= 32 ? 0xffffffffu : ((1u << G) - 1u);
  unsigned gbad = 0, dbad = 0;
  for (int r = 0; r < reps; ++r)
    stream_pass<G_MAX, U>(reinterpret_cast<const float4*>(w), reinterpret_cast<float4*>(spare), src, live, pullm,
                          P, G, lo, lr, first, stride, nv, gbad, dbad);
  if (gbad == 0xdeadbeefu) spare[0] = (float)dbad;  // keep the pass observable
}

template <int G_MAX>
__global__ void __launch_bounds__(kThreads, PS_SHARD_MINB)
k_shard_run(float* __restrict__ w0, float* __restrict__ w1, float* __restrict__ w2, long long n_local, ShardPtrs P, int G,
            int me, unsigned long long t0, int steps, float lr, ShardCtl* ctl, const double* now,
            ps_trace_row* trace, long long trace_cap, const int* sched) {
  const int ndata = gridDim.x - 1;
  // sched (optional): per step {pushers n, pull mask, ticket order[kMaxRanks]}
  // -- any push group and any set of pulling workers (heterogeneous
  // schedules); without it every worker pushes and pulls every step and the
  // ticket order follows the gate's previous grants (homogeneous schedule)
  // ---- the gate CTA: the replicated decisions, one group per step --------
  // They depend only on (worker, now) and the gate tables, never on the data,
  // so this CTA runs them from shared memory while the data CTAs stream.
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x >= 32) return;
    __shared__ ps_gate_state sg;
    {
      const unsigned long long* s = reinterpret_cast<const unsigned long long*>(&ctl->gate);
      unsigned long long* d = reinterpret_cast<unsigned long long*>(&sg);
      for (int i = threadIdx.x; i < (int)(sizeof(ps_gate_state) / 8); i += 32) d[i] = s[i];
    }
    __syncwarp();
    int status = PS_OK;
    for (int i = 0; i < steps && status == PS_OK; ++i) {
      const unsigned long long t = t0 + i;
      const int co = (int)(t & 1);
      if (threadIdx.x == 0 && !sched) {
        // order[co ^ 1] is read by every data CTA at the start of step t-1
        // (into shared memory); all of them have once they arrived there
        const unsigned long long s0 = globaltimer_ns();
        // every data CTA arrived at step i-1 of this run (per-parity counters)
        while (i > 0 && ld_acquire_u64(&ctl->arrive_par[(i - 1) & 1]) <
                            (unsigned long long)((i - 1) / 2 + 1) * (unsigned long long)ndata) {
          // the data side stopped (divergence / a peer's watchdog): so do we
          if (ld_relaxed_s32(&ctl->status) != PS_OK) { status = PS_E_TIMEOUT; break; }
          if (globaltimer_ns() - s0 > kTimeoutNs) { atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT); break; }
          __nanosleep(32);
        }
      }
      if (__shfl_sync(kFull, status, 0) != PS_OK) break;
      __syncwarp();
      int next[kMaxRanks];
      int n_next = 0;
      SPROF(const unsigned long long tg0 = globaltimer_ns());
      const int* row = sched ? sched + (long long)i * kSchedStride : nullptr;
      const int n_push = row ? row[0] : G;
      for (int k = 0; k < n_push; ++k) {
        const int p = row ? row[2 + k] : ctl->order[co][k];
        const GateResult r = gate_on_push(&sg, p, now[i]);
        if (threadIdx.x == 0) {
          if (r.status != PS_OK) status = r.status;
          if (r.status == PS_OK && r.outcome == 0) {
            next[n_next++] = p;
            for (int q = 0; q < G; ++q)
              if ((r.released >> q) & 1ull) next[n_next++] = q;
          }
          const unsigned long long n = ctl->trace_n++;
          if ((long long)n < trace_cap) {
            ps_trace_row row;
            row.time = now[i];
            row.worker = p;
            row.kind = PS_EV_PUSH_ARRIVE;
            row.count = sg.clocks[p];
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
        if (!sched && status == PS_OK && n_next != G) status = PS_E_PROTOCOL;
        if (status != PS_OK) atomicCAS(&ctl->status, PS_OK, status);
        if (!sched)
          for (int k = 0; k < n_next && k < G; ++k) ctl->order[co ^ 1][k] = next[k];
        st_release_u64(&ctl->gate_done, t);
        SPROF(g_prof[4] += globaltimer_ns() - tg0);
      }
      status = __shfl_sync(kFull, status, 0);
    }
    // tables back (version / rejected belong to the committing CTA)
    for (int q = threadIdx.x; q < G; q += 32) {
      ctl->gate.clocks[q] = sg.clocks[q];
      ctl->gate.latest[q] = sg.latest[q];
      ctl->gate.previous[q] = sg.previous[q];
      ctl->gate.populated[q] = sg.populated[q];
      ctl->gate.credits[q] = sg.credits[q];
    }
    if (threadIdx.x == 0) {
      ctl->gate.deferred = sg.deferred;
      ctl->gate.decisions = sg.decisions;
    }
    return;
  }
  // ---- data CTAs: one push group per step ---------------------------------
  // Per step ONE cross-GPU hop: after streaming step t, owner s publishes
  // V(t) = (t << 32 | diverged << 31 | rejected-worker bits seen in its slice)
  // into every rank's flag array. V(t) from every owner is, at once, "every
  // pull of step t has landed" (s wrote its slice into every replica before
  // the release) and the global verdict (the union of the bits).
  //
  // The shard is triple buffered: step k of the run reads buffer (c0 + k) % 3
  // and writes (c0 + k + 1) % 3. The first step of a run is resolved in full
  // before the second starts (the rejected set R of this run's update buffers
  // is then known -- they do not change during a run -- and a rejection is
  // redone without the rejected updates, server.py:65-67). In the homogeneous
  // schedule every later step skips R up front and needs only the divergence
  // verdict, so it is resolved one step LATE: step k starts once every owner
  // finished step k-2, overlapping the tail of step k-1 (the slowest CTAs, the
  // election, the fence and the cross-GPU flag hop) with step k's streaming.
  // A non-finite result at step j (server.py:38-41) is published in D[s] = j
  // before V(j); every rank then stops with the weights of buffer
  // (c0 + j - t0) % 3 -- intact, because no step past j + 1 can have started.
  // Heterogeneous schedules (sched != nullptr) resolve every step in full.
  __shared__ unsigned s_bits;
  __shared__ int s_stop, s_div;
  __shared__ unsigned long long s_rej, s_tdiv;
  __shared__ int s_order[2][kMaxRanks];
  __shared__ int s_n[2];           // pushers of the step in this slot
  __shared__ unsigned s_pull[2];   // workers whose replica the step writes
  const long long nv = (n_local + 3) >> 2;
  const long long lo = P.lo[me];
  constexpr int U = shard_unroll(G_MAX);
  const long long stride = (long long)ndata * kThreads * U;
  const long long first = (long long)blockIdx.x * kThreads * U + threadIdx.x;
  // buffer i of the rotation, by selects (a dynamically indexed array would
  // live in local memory)
  auto wb = [&](int i) -> float* { return i == 0 ? w0 : (i == 1 ? w1 : w2); };
  const int c0 = ld_relaxed_s32(&ctl->cur);  // the committed buffer at launch, identical in every CTA
  long long redo_n = 0;                      // redo rounds so far (election targets)
  const int steps_total = steps;
  const bool lag = steps > 2 && ld_relaxed_s32(&ctl->no_lag) == 0;
  // workers whose update of this run has been judged (by a full resolve):
  // a step whose pushers are all known carries no new rejection, so the next
  // step may start before its verdict (heterogeneous schedules meet new
  // pushers in their first groups, homogeneous ones only at step 0)
  unsigned long long K = 0;
  auto pushers_of = [&](int slot) {
    unsigned long long m = 0;
    for (int i = 0; i < s_n[slot]; ++i) m |= 1ull << s_order[slot][i];
    return m;
  };
  unsigned long long R = 0;                  // rejected workers of this run (lag mode)
  // commit step t (relative index k): buffer (c0 + k + 1) % 3 becomes current
  // (the rejected updates of step t: its own verdict bits plus every pusher of
  // the step already known to be rejected this run -- those were skipped)
  auto commit = [&](unsigned long long t, unsigned long long rej) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const int k = (int)(t - t0);
      ctl->cur = (c0 + k + 1) % 3;
      const int co = (int)(t & 1);
      unsigned long long pushers = 0;
      for (int i = 0; i < s_n[co]; ++i) pushers |= 1ull << s_order[co][i];
      const unsigned long long eff = (rej | R) & pushers;
      ctl->gate.version += s_n[co] - __popcll(eff);
      ctl->gate.rejected += __popcll(eff);
    }
  };
  auto stop_diverged = [&](unsigned long long tdiv) {
    // the weights stay at the input of step tdiv (server.py:38-41)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ctl->cur = (c0 + (int)(tdiv - t0)) % 3;
      atomicCAS(&ctl->status, PS_OK, PS_E_DIVERGED);
    }
  };
  // Full resolve of step t: wait for V(t) of every owner; redo this CTA's part
  // of the slice without rejected updates if any; stop on divergence; commit.
  auto resolve = [&](unsigned long long t) -> bool {
    if (threadIdx.x == 0) {
      SPROF(const unsigned long long tr0 = globaltimer_ns());
      unsigned long long rej = 0;
      int div = 0, stop = 0;
      const unsigned long long s0 = globaltimer_ns();
      for (int s = 0; s < G && !stop; ++s) {
        unsigned long long v;
        while (((v = ld_acquire_sys_u64(P.flags[me] + G + (int)(t % kVSlots) * G + s)) >> 32) < t) {
          if (globaltimer_ns() - s0 > kTimeoutNs) { atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT); stop = 1; break; }
          __nanosleep(20);
        }
        rej |= v & 0x7fffffffull;
        div |= (int)((v >> 31) & 1ull);
      }
      s_rej = rej; s_div = div; s_stop = stop;
      SPROF(if (blockIdx.x == 0) { const unsigned long long tn = globaltimer_ns(); g_prof[0] += tn - tr0; g_t_resolved = tn; })
    }
    __syncthreads();
    if (s_stop) return false;
    const unsigned long long rej = s_rej;
    const int co = (int)(t & 1);
    const int k = (int)(t - t0);
    if (rej) {
      // rare path: this CTA's part of the slice again, without the rejected
      // updates (server.py:65-67), into the back buffer and every replica;
      // the optimistic pass's divergence bit is void (it included them)
      const float4* wsrc = reinterpret_cast<const float4*>(wb((c0 + k) % 3));
      float4* wdst = reinterpret_cast<float4*>(wb((c0 + k + 1) % 3));
      unsigned redo_bad = 0;
      for (long long base = first; base < nv; base += stride)
        for (int u = 0; u < U; ++u) {
          const long long j = base + (long long)u * kThreads;
          if (j >= nv) break;
          float4 x = wsrc[j];
          for (int i = 0; i < s_n[co]; ++i) {
            const int p = s_order[co][i];
            if (!((rej >> p) & 1ull)) x = apply4(x, lr, reinterpret_cast<const float4*>(P.upd[p] + lo)[j]);
          }
          redo_bad |= nonfinite4(x) ? 1u : 0u;
          wdst[j] = x;
          for (int q = 0; q < G; ++q)
            if ((s_pull[co] >> q) & 1u) reinterpret_cast<float4*>(P.rep[q] + lo)[j] = x;
        }
      redo_bad = __syncthreads_or(redo_bad);
      redo_n += 1;
      if (threadIdx.x == 0) {
        if (redo_bad) atomicOr(&ctl->bad, 1u);
        const unsigned long long prev = atom_add_acq_rel_gpu_u64(&ctl->redo_total, 1ull);
        if (prev == (unsigned long long)(redo_n * ndata) - 1) {  // last CTA: F(t) to every rank
          const unsigned long long dv = atomicExch(&ctl->bad, 0u) & 1u;
          __threadfence_system();
          for (int s = 0; s < G; ++s) st_relaxed_sys_u64(P.flags[s] + (1 + kVSlots) * G + me, (t << 32) | dv);
        }
        int div = 0, stop = 0;
        const unsigned long long s0 = globaltimer_ns();
        for (int s = 0; s < G && !stop; ++s) {
          unsigned long long v;
          while (((v = ld_acquire_sys_u64(P.flags[me] + (1 + kVSlots) * G + s)) >> 32) < t) {
            if (globaltimer_ns() - s0 > kTimeoutNs) { atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT); stop = 1; break; }
            __nanosleep(20);
          }
          div |= (int)(v & 1ull);
        }
        s_div = div; s_stop = stop;
      }
      __syncthreads();
      if (s_stop) return false;
    }
    if (s_div) {
      stop_diverged(t);
      return false;
    }
    R |= rej;
    commit(t, rej);
    return true;
  };
  // Lagged resolve of step t (lag mode, t > t0): wait for V(>= t) of every
  // owner; a divergence at or before t stops the run at its first step.
  auto resolve_lag = [&](unsigned long long t) -> bool {
    if (threadIdx.x == 0) {
      SPROF(const unsigned long long tr0 = globaltimer_ns());
      int stop = 0;
      unsigned long long tdiv = 0;
      const unsigned long long s0 = globaltimer_ns();
      for (int s = 0; s < G && !stop; ++s) {
        unsigned long long v;
        while (((v = ld_acquire_sys_u64(P.flags[me] + G + (int)(t % kVSlots) * G + s)) >> 32) < t) {
          if (globaltimer_ns() - s0 > kTimeoutNs) { atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT); stop = 1; break; }
          __nanosleep(20);
        }
        if ((v >> 31) & 1ull) {
          // sticky: owner s diverged at step D[s] <= v's step (published first)
          const unsigned long long d = ld_acquire_sys_u64(P.flags[me] + (2 + kVSlots) * G + s);
          if (d && d <= t && (!tdiv || d < tdiv)) tdiv = d;
        }
      }
      s_tdiv = tdiv; s_stop = stop;
      SPROF(if (blockIdx.x == 0) { const unsigned long long tn = globaltimer_ns(); g_prof[0] += tn - tr0; g_t_resolved = tn; })
    }
    __syncthreads();
    if (s_stop) return false;
    if (s_tdiv) {
      stop_diverged(s_tdiv);
      return false;
    }
    commit(t, R);
    return true;
  };
  unsigned long long resolved = t0 - 1;  // last step resolved by this CTA
  for (int step = 0; step < steps_total; ++step) {
    const unsigned long long t = t0 + step;
    const int co = (int)(t & 1);
    if (!lag) {
      if (step > 0 && !resolve(t - 1)) return;
      resolved = t - 1;
    } else if (step >= 1) {
      const unsigned long long prev_pushers = pushers_of((int)((t - 1) & 1));
      if (step >= 2 && t - 2 > resolved) {
        if (!resolve_lag(t - 2)) return;
        resolved = t - 2;
      }
      if (prev_pushers & ~K) {
        // step t-1 met pushers not yet judged: its verdict (and any redo
        // without the rejected ones) before step t runs
        if (!resolve(t - 1)) return;
        resolved = t - 1;
        K |= prev_pushers;
      }
    }
    if (threadIdx.x == 0) {
      s_bits = 0;
      bool ok = true;
      if (step == 0) {
        // the run's first push: worker `me`'s update is in place (stream
        // order on this rank); every owner starts once all workers pushed
        if (blockIdx.x == 0) {
          __threadfence_system();
          for (int s = 0; s < G; ++s) st_relaxed_sys_u64(P.flags[s] + me, t);
        }
        ok = wait_flags(P.flags[me], G, t, nullptr, ctl);
      }
      // this group's ticket order is final once the gate finished step t-1
      // (with a schedule it is given)
      const unsigned long long s0 = globaltimer_ns();
      SPROF(const unsigned long long tw0 = globaltimer_ns());
      while (ok && !sched && ld_acquire_u64(&ctl->gate_done) + 1 < t) {
        if (globaltimer_ns() - s0 > kTimeoutNs) { atomicCAS(&ctl->status, PS_OK, PS_E_TIMEOUT); ok = false; }
        if (ld_relaxed_s32(&ctl->status) != PS_OK) ok = false;  // the gate stopped (protocol)
        __nanosleep(32);
      }
      SPROF(if (blockIdx.x == 0) g_prof[5] += globaltimer_ns() - tw0);
      if (ok) {
        if (sched) {
          const int* row = sched + (long long)step * kSchedStride;
          s_n[co] = row[0];
          s_pull[co] = (unsigned)row[1];
          for (int i = 0; i < row[0]; ++i) s_order[co][i] = row[2 + i];
        } else {
          s_n[co] = G;
          s_pull[co] = G >= 32 ? 0xffffffffu : ((1u << G) - 1u);
          for (int i = 0; i < G; ++i) s_order[co][i] = ctl->order[co][i];
        }
      }
      s_stop = !ok;
    }
    __syncthreads();
    if (s_stop) return;  // watchdog fired
    const float4* wsrc = reinterpret_cast<const float4*>(wb((c0 + step) % 3));
    float4* wdst = reinterpret_cast<float4*>(wb((c0 + step + 1) % 3));
    const int n_push = s_n[co];
    const unsigned pullm = s_pull[co];
    // in lag mode the rejected workers of this run are known after step 0:
    // their slices are not even loaded (rejected every push, server.py:65-67)
    unsigned live = 0;
    const float4* src[G_MAX];
#pragma unroll
    for (int i = 0; i < G_MAX; ++i) {
      const int p = i < n_push ? s_order[co][i] : 0;
      src[i] = reinterpret_cast<const float4*>(P.upd[p] + lo);
      if (i < n_push && !((R >> p) & 1ull)) live |= 1u << i;
    }
    unsigned dbad = 0;
    unsigned gbad = 0;  // bit i: the update of pusher order[i] holds a non-finite value here
    stream_pass<G_MAX, U>(wsrc, wdst, src, live, pullm, P, G, lo, lr, first, stride, nv, gbad, dbad);
    gbad = __reduce_or_sync(kFull, gbad);
    dbad = __reduce_or_sync(kFull, dbad);
    if ((threadIdx.x & 31) == 0 && (gbad | dbad)) atomicOr(&s_bits, gbad | (dbad << 31));
    __syncthreads();
    if (threadIdx.x == 0) {
      // per-parity verdict words and arrival counters: in lag mode CTAs of
      // steps t and t+1 arrive interleaved, never those of t and t+2
      if (s_bits) atomicOr(&ctl->badp[co], s_bits);
      // this CTA's stores (local and to peers; the barrier orders every warp's
      // before this thread) are released at GPU scope; the winner acquires
      // them all and its fence.sc.sys orders them before V(t) at system scope
      // (causality order is transitive across scopes) -- one system fence
      // per step instead of one per warp
      const unsigned long long prev = atom_add_acq_rel_gpu_u64(&ctl->arrive_par[step & 1], 1ull);
      SPROF(if (blockIdx.x == 0) g_prof[1] += globaltimer_ns() - g_t_resolved);
      if (prev == (unsigned long long)(step / 2 + 1) * (unsigned long long)ndata - 1) {
        SPROF(const unsigned long long te = globaltimer_ns(); g_prof[2] += te - g_t_resolved);
        // last data CTA of the step: V(t) to every rank
        const unsigned b = atomicExch(&ctl->badp[co], 0u);
        const unsigned div = (b >> 31) | (unsigned)ctl->div_sticky;
        // a step that also saw a rejected update carries a void divergence
        // bit (the optimistic pass included the update); its full resolve
        // redoes it, so only a clean step's non-finite result is sticky
        if ((b >> 31) && !(b & 0x7fffffffu) && !ctl->div_sticky) {
          ctl->div_sticky = 1;
          // D(me) = the first diverged step, published before V(t)
          for (int s = 0; s < G; ++s) st_relaxed_sys_u64(P.flags[s] + (2 + kVSlots) * G + me, t);
        }
        unsigned long long v = (t << 32) | ((unsigned long long)div << 31);
        for (int i = 0; i < s_n[co]; ++i)
          if ((b >> i) & 1u) v |= 1ull << s_order[co][i];
        __threadfence_system();
        for (int s = 0; s < G; ++s) st_relaxed_sys_u64(P.flags[s] + G + (int)(t % kVSlots) * G + me, v);
        SPROF(g_prof[3] += globaltimer_ns() - te; g_prof[6] += 1);
      }
    }
  }
  // the last steps' verdicts: this rank's replica is complete and committed
  // when the kernel exits
  const unsigned long long t_last = t0 + steps_total - 1;
  if (!lag) {
    resolve(t_last);
  } else {
    for (unsigned long long t = resolved + 1; t <= t_last; ++t) {
      const unsigned long long p = pushers_of((int)(t & 1));
      if (!((p & ~K) ? resolve(t) : resolve_lag(t))) break;
      K |= p;
    }
  }
#ifdef PS_SHARD_PROFILE
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const double n = g_prof[6] ? (double)g_prof[6] : 1.0;
    printf("[shard-prof rank %d] per step us: resolve_wait %.2f cta0_stream %.2f last_arrival %.2f "
           "publish_V %.2f gate %.2f gate_wait %.2f (steps %llu, data CTAs %d)\n", me,
           g_prof[0] * 1e-3 / n, g_prof[1] * 1e-3 / n, g_prof[2] * 1e-3 / n, g_prof[3] * 1e-3 / n,
           g_prof[4] * 1e-3 / n, g_prof[5] * 1e-3 / n, g_prof[6], ndata);
    for (int i = 0; i < 8; ++i) g_prof[i] = 0;
  }
#endif
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
  int* sched_dev = nullptr;  // ps_shard_run_groups: device copy of the groups
  size_t sched_cap = 0;
  int world = 1, rank = 0, dev = 0, sm_count = 148;
  cudaStream_t stream = nullptr;
  long long d = 0, S = 0, lo = 0, hi = 0, n_local = 0, dpad = 0;
  float* w = nullptr;                 // local shard (padded to a multiple of 4), buffer 0
  float* w_alt = nullptr;             // buffer 1 (ShardCtl::cur says which is current)
  float* w_3 = nullptr;               // buffer 2 (the lagged pipeline keeps three)
  double* now_dev = nullptr;          // per-step push instants of the current run
  int now_cap = 0;
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
  cudaEvent_t pev[4] = {nullptr, nullptr, nullptr, nullptr};
  int profile = 0;
  double phase_ms[3] = {0, 0, 0};   // ready / apply / pull, summed over profiled steps
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
  // Every buffer a peer maps through CUDA IPC gets its own 2 MB-granular
  // allocation: small allocations are carved out of shared blocks, and an IPC
  // mapping of a block outlives the buffer it was opened for (measured: a
  // later server's replica mapped through a stale block of an earlier one).
  auto ipc_bytes = [](size_t b) { return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1); };
  if ((e = cudaMalloc(&h->w, ipc_bytes(shard_bytes))) || (e = cudaMalloc(&h->w_alt, shard_bytes)) ||
      (e = cudaMalloc(&h->w_3, shard_bytes)))
    return bail("shard");
  // every initialization is ordered on the server's own (non-blocking)
  // stream: a plain cudaMemset runs on the legacy stream, which does not
  // order against it -- measured, a late memset zeroed part of a shard after
  // its w0 load
  if ((e = cudaMemsetAsync(h->w, 0, shard_bytes, h->stream)) || (e = cudaMemsetAsync(h->w_alt, 0, shard_bytes, h->stream)) ||
      (e = cudaMemsetAsync(h->w_3, 0, shard_bytes, h->stream)))
    return bail("shard memset");
  if ((e = cudaMalloc(&h->upd, ipc_bytes(h->dpad * sizeof(float))))) return bail("update buffer");
  if ((e = cudaMemsetAsync(h->upd, 0, h->dpad * sizeof(float), h->stream))) return bail("update memset");
  if ((e = cudaMalloc(&h->rep, ipc_bytes(h->dpad * sizeof(float))))) return bail("replica");
  if ((e = cudaMemsetAsync(h->rep, 0, h->dpad * sizeof(float), h->stream))) return bail("replica memset");
  if ((e = cudaMalloc(&h->flags, ipc_bytes(kFlagWords * sizeof(unsigned long long))))) return bail("flags");
  if ((e = cudaMemsetAsync(h->flags, 0, kFlagWords * sizeof(unsigned long long), h->stream))) return bail("flags memset");
  if ((e = cudaMalloc(&h->ctl, sizeof(ShardCtl)))) return bail("ctl");
  if ((e = cudaMallocHost(&h->hctl, sizeof(ShardCtl)))) return bail("hctl");
  std::memset(h->hctl, 0, sizeof(ShardCtl));
  ps_gate_state& gs = h->hctl->gate;
  gs.paradigm = cfg->paradigm;
  gs.worker_count = cfg->worker_count;
  gs.s_lower = cfg->s_lower;
  gs.r_max = cfg->r_max;
  gs.threshold = cfg->paradigm == PS_BSP ? 0 : cfg->s_lower;
  for (int r = 0; r < kMaxRanks; ++r) h->hctl->order[1][r] = r;  // step 1: initial pulls arrive in worker order
  if ((e = cudaMemcpy(h->ctl, h->hctl, sizeof(ShardCtl), cudaMemcpyHostToDevice))) return bail("ctl upload");
  // w0: full-length initial weights; bit 0 of w0_flags = on device, bit 1 = fp64.
  // The shard gets its range; the worker's replica starts as the whole vector
  // (the worker's first pull, simnet.py:135-138, before it computes anything).
  if (w0) {
    const bool on_dev = w0_flags & 1, f64 = w0_flags & 2;
    const size_t esz = f64 ? 8 : 4;
    const char* src = (const char*)w0;
    void* tmp = nullptr;
    if (!on_dev) {
      if ((e = cudaMalloc(&tmp, h->d * esz + 16))) return bail("w0 staging");
      // on the server's stream: a pageable cudaMemcpy may return before its
      // DMA lands, and the legacy stream does not order against h->stream
      if ((e = cudaMemcpyAsync(tmp, src, h->d * esz, cudaMemcpyHostToDevice, h->stream))) return bail("w0 upload");
      src = (const char*)tmp;
    }
    const char* mine = src + (size_t)h->lo * esz;
    if (f64) {
      if (h->n_local > 0)
        k_shard_load<double><<<h->sm_count * 2, 256, 0, h->stream>>>((const double*)mine, h->w, h->n_local);
      k_shard_load<double><<<h->sm_count * 2, 256, 0, h->stream>>>((const double*)src, h->rep, h->d);
    } else {
      if (h->n_local > 0)
        k_shard_load<float><<<h->sm_count * 2, 256, 0, h->stream>>>((const float*)mine, h->w, h->n_local);
      k_shard_load<float><<<h->sm_count * 2, 256, 0, h->stream>>>((const float*)src, h->rep, h->d);
    }
    if ((e = cudaStreamSynchronize(h->stream))) return bail("w0 convert");
    if (tmp) cudaFree(tmp);
  }
  if ((e = cudaStreamSynchronize(h->stream))) return bail("initialization");
  *out = h;
  return PS_OK;
}

// First half of a collective shutdown: unmap every peer buffer this rank
// opened. A peer must not free memory another process still has mapped (CUDA
// IPC: undefined behaviour -- measured, a later server's mapping then
// aliased stale pages), so every rank disconnects, the ranks synchronize,
// and only then does each free its own buffers (ps_shard_destroy).
int ps_shard_disconnect(ps_shard_server* h) {
  if (!h) return PS_OK;
  Dev guard(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->opened) cudaIpcCloseMemHandle(p);
  h->opened.clear();
  for (int r = 0; r < kMaxRanks; ++r)
    if (r != h->rank) { h->ptrs.w[r] = nullptr; h->ptrs.upd[r] = nullptr; h->ptrs.rep[r] = nullptr; h->ptrs.flags[r] = nullptr; }
  return PS_OK;
}

void ps_shard_destroy(ps_shard_server* h) {
  if (!h) return;
  Dev guard(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->opened) cudaIpcCloseMemHandle(p);
  cudaFree(h->w); cudaFree(h->w_alt); cudaFree(h->w_3); cudaFree(h->now_dev); cudaFree(h->upd); cudaFree(h->rep); cudaFree(h->flags); cudaFree(h->ctl);
  cudaFree(h->trace);
  cudaFree(h->sched_dev);
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
  SCK(h, cudaIpcGetMemHandle(&b.rep, h->rep));
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
      h->ptrs.rep[r] = h->rep;
      h->ptrs.flags[r] = h->flags;
      continue;
    }
    void *pw = nullptr, *pu = nullptr, *pr = nullptr, *pf = nullptr;
    SCK(h, cudaIpcOpenMemHandle(&pw, b[r].w, cudaIpcMemLazyEnablePeerAccess));
    SCK(h, cudaIpcOpenMemHandle(&pu, b[r].upd, cudaIpcMemLazyEnablePeerAccess));
    SCK(h, cudaIpcOpenMemHandle(&pr, b[r].rep, cudaIpcMemLazyEnablePeerAccess));
    SCK(h, cudaIpcOpenMemHandle(&pf, b[r].flags, cudaIpcMemLazyEnablePeerAccess));
    h->opened.push_back(pw);
    h->opened.push_back(pu);
    h->opened.push_back(pr);
    h->opened.push_back(pf);
    h->ptrs.w[r] = (const float*)pw;
    h->ptrs.upd[r] = (const float*)pu;
    h->ptrs.rep[r] = (float*)pr;
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

// Device pointer of this rank's replica: the worker's copy of the weights,
// written by every owner at each pull (a worker may keep its model
// parameters right here and compute on them between runs).
int ps_shard_replica_buffer(ps_shard_server* h, void** ptr, int64_t* padded_len) {
  *ptr = h->rep;
  *padded_len = h->dpad;
  return PS_OK;
}

// Enqueue `steps` push groups starting at step index t0 (1-based tickets) and
// wait for them. now[i] is the virtual push time of step i. Every owner writes
// its slice of the new weights straight into each worker's (engine-owned)
// replica; dst (device, fp32, may be NULL) additionally receives a copy of
// this rank's replica after the last step.
namespace {
int shard_run(ps_shard_server* h, int64_t t0, int32_t steps, const double* now, const int32_t* groups,
              void* dst, double* ms);
}  // namespace

int ps_shard_run(ps_shard_server* h, int64_t t0, int32_t steps, const double* now, void* dst,
                 double* ms) {
  return shard_run(h, t0, steps, now, nullptr, dst, ms);
}

// Any push groups: row i of `groups` (PS_SHARD_GROUP_STRIDE int32 each) is
// {n pushers, pull mask, ticket order[n]} of step i.
int ps_shard_run_groups(ps_shard_server* h, int64_t t0, int32_t steps, const double* now,
                        const int32_t* groups, void* dst, double* ms) {
  if (steps >= 1 && !groups) return sfail(h, PS_E_VALUE, "groups missing");
  for (int i = 0; i < steps; ++i) {
    const int32_t* row = groups + (long long)i * kSchedStride;
    if (row[0] < 0 || row[0] > h->world) return sfail(h, PS_E_VALUE, "group size out of range");
    if (h->world < 32 && ((unsigned)row[1] >> h->world)) return sfail(h, PS_E_VALUE, "pull mask names an unknown worker");
    unsigned seen = 0;
    for (int k = 0; k < row[0]; ++k) {
      const int p = row[2 + k];
      if (p < 0 || p >= h->world || ((seen >> p) & 1u)) return sfail(h, PS_E_VALUE, "bad ticket order");
      seen |= 1u << p;
    }
  }
  return shard_run(h, t0, steps, now, groups, dst, ms);
}

namespace {
int shard_run(ps_shard_server* h, int64_t t0, int32_t steps, const double* now, const int32_t* groups,
              void* dst, double* ms) {
  Dev guard(h->dev);
  if (steps < 1) return PS_OK;
  const long long need = (long long)(t0 + steps) * h->world + 8;
  if (need > h->trace_cap) {
    // grow, keeping the rows of earlier runs (the trace is cumulative)
    const long long cap = need * 2;
    ps_trace_row* grown = nullptr;
    SCK(h, cudaMalloc(&grown, cap * sizeof(ps_trace_row)));
    if (h->trace) {
      SCK(h, cudaMemcpyAsync(grown, h->trace, h->trace_cap * sizeof(ps_trace_row), cudaMemcpyDeviceToDevice,
                             h->stream));
      SCK(h, cudaStreamSynchronize(h->stream));
      cudaFree(h->trace);
    }
    h->trace = grown;
    h->trace_cap = cap;
  }
  const int G = h->world, me = h->rank;
  const float lr = (float)h->cfg.learning_rate;
  // One persistent cooperative launch runs all the steps: CTAs per SM of the
  // streaming loop (tuning knob, default 2, clamped to co-residency -- CTAs
  // wait on each other and on peers), plus one gate CTA.
  static const int per_sm_env = [] {
    const char* v = getenv("PS_SHARD_CTAS_PER_SM");
    const int n = v ? atoi(v) : 2;
    return n > 0 && n <= 16 ? n : 2;
  }();
  // PS_SHARD_GMAX (test knob): run a wider instantiation than G needs, so the
  // G <= 8 / 16 code paths are exercised on a box with fewer GPUs
  static const int gmax_env = [] {
    const char* v = getenv("PS_SHARD_GMAX");
    return v ? atoi(v) : 0;
  }();
  const int gsel = G > gmax_env ? G : gmax_env;
  const void* kern = gsel <= 2 ? (const void*)k_shard_run<2> : gsel <= 4 ? (const void*)k_shard_run<4>
                   : gsel <= 8 ? (const void*)k_shard_run<8> : (const void*)k_shard_run<16>;
  static int occupancy[4] = {-1, -1, -1, -1};  // per instantiation, queried once
  const int oi = gsel <= 2 ? 0 : gsel <= 4 ? 1 : gsel <= 8 ? 2 : 3;
  int resident = occupancy[oi];
  if (resident < 0) {
    SCK(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, kThreads, 0));
    occupancy[oi] = resident;
  }
  int total = h->sm_count * (per_sm_env < resident ? per_sm_env : resident);
  // no more streaming CTAs than one trip over the shard needs: idle CTAs
  // would only lengthen every step's election and polling
  {
    const int U = shard_unroll(gsel);  // float4 per thread per trip (k_shard_run)
    const long long nv = (h->n_local + 3) / 4;
    const long long need_ctas = (nv + (long long)kThreads * U - 1) / ((long long)kThreads * U);
    if (need_ctas + 1 < total) total = (int)(need_ctas > 0 ? need_ctas : 1) + 1;
  }
  const int data_ctas = total - 1;
  if (data_ctas < 1) return sfail(h, PS_E_CUDA, "k_shard_run cannot be resident");
  if (h->now_cap < steps) {
    cudaFree(h->now_dev);
    h->now_dev = nullptr;
    SCK(h, cudaMalloc(&h->now_dev, steps * sizeof(double)));
    h->now_cap = steps;
  }
  SCK(h, cudaMemcpyAsync(h->now_dev, now, steps * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  const int* schedp = nullptr;
  if (groups) {
    const size_t need_ints = (size_t)steps * kSchedStride;
    if (h->sched_cap < need_ints) {
      cudaFree(h->sched_dev);
      h->sched_dev = nullptr;
      SCK(h, cudaMalloc(&h->sched_dev, need_ints * sizeof(int)));
      h->sched_cap = need_ints;
    }
    SCK(h, cudaMemcpyAsync(h->sched_dev, groups, need_ints * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    schedp = h->sched_dev;
  }
  // election counter and step marks continue from ticket t0 - 1
  const unsigned long long marks[4] = {(unsigned long long)(t0 - 1) * (unsigned long long)data_ctas,
                                       (unsigned long long)(t0 - 1), (unsigned long long)(t0 - 1), 0ull};
  SCK(h, cudaMemcpyAsync(&h->ctl->arrive_total, marks, sizeof(marks), cudaMemcpyHostToDevice, h->stream));
  // this run's per-parity arrival counters and verdict words start at zero;
  // PS_SHARD_NO_LAG=1 resolves every step in full (the round-1 protocol)
  static const int no_lag_env = [] {
    const char* v = getenv("PS_SHARD_NO_LAG");
    return v && v[0] == '1' ? 1 : 0;
  }();
  // (staged in the pinned host mirror, which nothing else touches until the
  // run's own read-back at the end)
  h->hctl->arrive_par[0] = h->hctl->arrive_par[1] = 0;
  h->hctl->badp[0] = h->hctl->badp[1] = 0;
  h->hctl->div_sticky = 0;
  h->hctl->no_lag = no_lag_env;
  const size_t tail = offsetof(ShardCtl, no_lag) + sizeof(int32_t) - offsetof(ShardCtl, arrive_par);
  SCK(h, cudaMemcpyAsync(&h->ctl->arrive_par, &h->hctl->arrive_par, tail, cudaMemcpyHostToDevice, h->stream));
  float* w0p = h->w;
  float* w1p = h->w_alt;
  float* w2p = h->w_3;
  long long nl = h->n_local;
  ShardPtrs ptrs = h->ptrs;
  ShardCtl* ctl = h->ctl;
  ps_trace_row* trace = h->trace;
  long long tcap = h->trace_cap;
  int Gv = G, mev = me, nsteps = steps;
  unsigned long long t0v = (unsigned long long)t0;
  float lrv = lr;
  const double* nowp = h->now_dev;
  void* args[] = {&w0p, &w1p, &w2p, &nl, &ptrs, &Gv, &mev, &t0v, &nsteps, &lrv, &ctl, &nowp, &trace, &tcap, &schedp};
  SCK(h, cudaEventRecord(h->ev0, h->stream));
  SCK(h, cudaLaunchCooperativeKernel(kern, dim3(total), dim3(kThreads), args, 0, h->stream));
  if (h->profile) SCK(h, cudaEventRecord(h->pev[0], h->stream));
  SCK(h, cudaEventRecord(h->ev1, h->stream));
  if (h->profile) SCK(h, cudaEventRecord(h->pev[1], h->stream));
  if (dst) SCK(h, cudaMemcpyAsync(dst, h->rep, h->d * sizeof(float), cudaMemcpyDeviceToDevice, h->stream));
  SCK(h, cudaMemcpyAsync(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  float e = 0.f;
  cudaEventElapsedTime(&e, h->ev0, h->ev1);
  if (ms) *ms = e;
  if (h->profile) {
    float k = 0.f, wt = 0.f;
    cudaEventElapsedTime(&k, h->ev0, h->pev[0]);
    cudaEventElapsedTime(&wt, h->pev[0], h->pev[1]);
    h->phase_ms[0] += k;
    h->phase_ms[1] += wt;
  }
  const int st = h->hctl->status;
  if (st == PS_E_TIMEOUT) return sfail(h, PS_E_TIMEOUT, "device watchdog fired waiting for a peer");
  if (st == PS_E_DIVERGED) return sfail(h, PS_E_DIVERGED, "non-finite weights in the sharded server");
  if (st == PS_E_PROTOCOL) return sfail(h, PS_E_PROTOCOL, "protocol violation in the replicated gate");
  return PS_OK;
}

}  // namespace

// Profiling: bracket each of the three kernels with events (serializes the
// host with every step, so only for diagnosis, never for the timed numbers).
int ps_shard_set_profiling(ps_shard_server* h, int32_t on) {
  Dev guard(h->dev);
  if (on && !h->pev[0])
    for (int k = 0; k < 4; ++k) SCK(h, cudaEventCreate(&h->pev[k]));
  h->profile = on ? 1 : 0;
  h->phase_ms[0] = h->phase_ms[1] = h->phase_ms[2] = 0.0;
  return PS_OK;
}

int ps_shard_phase_ms(ps_shard_server* h, double* out3) {
  for (int k = 0; k < 3; ++k) out3[k] = h->phase_ms[k];
  return PS_OK;
}

int ps_shard_stream_probe(ps_shard_server* h, int32_t reps, double* ms) {
  Dev guard(h->dev);
  if (reps < 1) return sfail(h, PS_E_VALUE, "reps must be >= 1");
  const int G = h->world;
  const void* kern = G <= 2 ? (const void*)k_shard_stream_probe<2> : G <= 4 ? (const void*)k_shard_stream_probe<4>
                   : G <= 8 ? (const void*)k_shard_stream_probe<8> : (const void*)k_shard_stream_probe<16>;
  int resident = 0;
  SCK(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, kern, kThreads, 0));
  const int grid = h->sm_count * (resident < 2 ? resident : 2);
  // the spare buffer: whichever of the three is neither current nor next
  SCK(h, cudaMemcpy(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost));
  float* bufs[3] = {h->w, h->w_alt, h->w_3};
  const float* w = bufs[h->hctl->cur % 3];
  float* spare = bufs[(h->hctl->cur + 2) % 3];
  long long nl = h->n_local;
  ShardPtrs ptrs = h->ptrs;
  int Gv = G, mev = h->rank, r = reps;
  float lr = (float)h->cfg.learning_rate;
  void* args[] = {&w, &spare, &nl, &ptrs, &Gv, &mev, &lr, &r};
  SCK(h, cudaEventRecord(h->ev0, h->stream));
  SCK(h, cudaLaunchKernel(kern, dim3(grid), dim3(kThreads), args, 0, h->stream));
  SCK(h, cudaEventRecord(h->ev1, h->stream));
  SCK(h, cudaStreamSynchronize(h->stream));
  float e = 0.f;
  cudaEventElapsedTime(&e, h->ev0, h->ev1);
  if (ms) *ms = e;
  return PS_OK;
}

int ps_shard_read_shard(ps_shard_server* h, void* dst_host, int64_t* n) {
  Dev guard(h->dev);
  *n = h->n_local;
  SCK(h, cudaMemcpy(h->hctl, h->ctl, sizeof(ShardCtl), cudaMemcpyDeviceToHost));
  const float* bufs[3] = {h->w, h->w_alt, h->w_3};
  const float* cur = bufs[h->hctl->cur % 3];
  if (h->n_local > 0) SCK(h, cudaMemcpy(dst_host, cur, h->n_local * sizeof(float), cudaMemcpyDeviceToHost));
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
