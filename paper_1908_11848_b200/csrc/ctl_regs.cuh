// ctl_regs.cuh -- the run loop's control warp with every table in registers.
//
// For P <= PM workers (PM = 8 covers the benchmark and corpus schedules) the
// whole control state -- the event per worker ((time, seq) ordered, one in
// flight per worker), the worker bookkeeping and the DSSP gate tables
// (clocks, two-deep push history, credits, deferred mask) -- lives in
// registers, replicated identically in all 32 lanes of the warp. Every lane
// runs the same scalar event loop in lockstep (no broadcasts needed); the
// controller's (r_max+1)^2 grid is the one place the lanes split the work
// (gate.cuh controller_grid). Only lane 0 writes memory (trace rows, op words).
// Dynamic worker indices go through unrolled select loops so nothing spills
// to local memory.
//
// Semantics are those of gate.cuh / policy.py:84-206 and simnet.py:127-201;
// the trace-parity tests hold both control paths to the reference.
#pragma once

#include "gate.cuh"

namespace dssp {

#ifdef PS_SIM_PROFILE
__device__ long long g_ctl_calls, g_ctl_cycles;
#endif

template <int PM, typename T>
__device__ __forceinline__ T rget(const T (&a)[PM], int i) {
  T r = a[0];
#pragma unroll
  for (int q = 1; q < PM; ++q)
    if (q == i) r = a[q];
  return r;
}

template <int PM, typename T>
__device__ __forceinline__ void rset(T (&a)[PM], int i, T v) {
#pragma unroll
  for (int q = 0; q < PM; ++q)
    if (q == i) a[q] = v;
}

template <int PM>
struct RegGate {
  int paradigm, P, s_lower, r_max, threshold;
  int clocks[PM];
  double latest[PM], previous[PM];
  int populated[PM];
  int credits[PM];
  unsigned long long deferred;
  long long decisions;

  __device__ __forceinline__ void load(const ps_gate_state& g, bool reset) {
    paradigm = g.paradigm; P = g.worker_count; s_lower = g.s_lower; r_max = g.r_max;
    threshold = g.threshold;
#pragma unroll
    for (int q = 0; q < PM; ++q) {
      const bool z = reset || q >= P;
      clocks[q] = z ? 0 : (int)g.clocks[q];
      latest[q] = z ? 0.0 : g.latest[q];
      previous[q] = z ? 0.0 : g.previous[q];
      populated[q] = z ? 0 : (int)g.populated[q];
      credits[q] = z ? 0 : (int)g.credits[q];
    }
    deferred = reset ? 0ull : g.deferred;
    decisions = g.decisions;
  }

  __device__ __forceinline__ void store(ps_gate_state& g) const {
#pragma unroll
    for (int q = 0; q < PM; ++q) {
      if (q < P) {
        g.clocks[q] = clocks[q]; g.latest[q] = latest[q]; g.previous[q] = previous[q];
        g.populated[q] = populated[q]; g.credits[q] = credits[q];
      }
    }
    g.deferred = deferred;
    g.decisions = decisions;
  }

  __device__ __forceinline__ int min_clock() const {
    int m = clocks[0];
#pragma unroll
    for (int q = 1; q < PM; ++q)
      if (q < P && clocks[q] < m) m = clocks[q];
    return m;
  }
  __device__ __forceinline__ int max_clock() const {
    int m = clocks[0];
#pragma unroll
    for (int q = 1; q < PM; ++q)
      if (q < P && clocks[q] > m) m = clocks[q];
    return m;
  }
  __device__ __forceinline__ int slowest() const {
    const int m = min_clock();
    int s = 0;
#pragma unroll
    for (int q = PM - 1; q >= 0; --q)
      if (q < P && clocks[q] == m) s = q;
    return s;
  }
  __device__ __forceinline__ void record(int q, double t) {
#pragma unroll
    for (int i = 0; i < PM; ++i)
      if (i == q) { previous[i] = latest[i]; latest[i] = t; populated[i] += 1; }
  }
  __device__ __forceinline__ unsigned long long release_ready(int low) {
    if (!deferred) return 0ull;
    unsigned long long ready = 0ull;
#pragma unroll
    for (int q = 0; q < PM; ++q)
      if (q < P && ((deferred >> q) & 1ull) && clocks[q] - low <= threshold) ready |= 1ull << q;
    deferred &= ~ready;
    return ready;
  }

  // policy.py:152-206, warp-uniform (every lane holds the same tables).
  // Every paradigm records the push in the history (policy.py:158-195; the
  // controller records before it reads it), so the record is done once, up
  // front, and the minimum clock once for the gap test and the release scan.
  __device__ __forceinline__ GateResult on_push(int p, double now) {
    GateResult r{PS_OK, 0, 0ull};
    if (p < 0 || p >= P || ((deferred >> p) & 1ull)) { r.status = PS_E_PROTOCOL; return r; }
    const int count = rget<PM>(clocks, p) + 1;
    rset<PM>(clocks, p, count);
    decisions += 1;
    record(p, now);
    if (paradigm == PS_ASP) return r;  // grant, no release scan
    const int low = min_clock();
    int outcome;
    if (paradigm == PS_DSSP) {
      const int cred = rget<PM>(credits, p);
      const int gap = count - low;
      if (cred > 0) {
        rset<PM>(credits, p, cred - 1);
        outcome = 0;
      } else if (gap <= s_lower) {
        outcome = 0;
      } else if (!(count >= max_clock())) {
        outcome = 1;
      } else {
        int pred = 0;
        if (r_max > 0) {
          const int sl = slowest();
          if (rget<PM>(populated, p) >= 2 && rget<PM>(populated, sl) >= 2) {
#ifdef PS_SIM_PROFILE
            const long long tc = clock64();
#endif
            pred = controller_grid(rget<PM>(latest, p), rget<PM>(previous, p), rget<PM>(latest, sl),
                                   rget<PM>(previous, sl), r_max);
#ifdef PS_SIM_PROFILE
            if ((threadIdx.x & 31) == 0) { g_ctl_calls += 1; g_ctl_cycles += clock64() - tc; }
#endif
          }
        }
        int headroom = s_lower + r_max - gap;
        if (headroom < 0) headroom = 0;
        const int c = pred < headroom ? pred : headroom;
        rset<PM>(credits, p, c);
        outcome = c > 0 ? 0 : 1;
      }
    } else {
      outcome = (count - low <= threshold) ? 0 : 1;
    }
    r.outcome = outcome;
    if (outcome == 1) deferred |= 1ull << p;
    else r.released = release_ready(low);
    return r;
  }
};

}  // namespace dssp
