// ctl_lanes.cuh -- the run loop's control warp, one worker per lane.
//
// For P <= 32 workers, lane q holds worker q's whole state in registers: its
// in-flight event ((time, seq, kind); the reference keeps at most one per
// worker), its bookkeeping (iterations, active/staged replica, update slot,
// next compute draw) and its row of the DSSP gate tables (clock, two-deep push
// history, credit). Table-wide questions are single warp instructions:
//   min/max clock         __reduce_min_sync / __reduce_max_sync (policy.py:60-64)
//   slowest (ties -> id)  ballot + ffs                          (policy.py:66-69)
//   release scan          one ballot, ascending by construction (policy.py:197-206)
//   next event            three reductions over (time bits, seq): non-negative
//                         doubles order like their IEEE bit patterns, so the
//                         (time, seq) heap pop of simnet.py:106-108 is exact.
// Scalars (deferred mask, counters) are warp-uniform. The controller grid
// (gate.cuh controller_grid) is the only place the lanes split other work.
// Trace rows are written by five lanes with one store (one 8-byte field each).
//
// Semantics are those of gate.cuh / policy.py:84-206 and simnet.py:127-201;
// the trace-parity tests hold this path to the reference byte for byte.
#pragma once

#include "gate.cuh"

namespace dssp {

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

template <typename T>
__device__ __forceinline__ T from_lane(T v, int lane) {
  return __shfl_sync(kFull, v, lane);
}

// One DSSP gate whose per-worker tables live one row per lane.
struct LaneGate {
  int paradigm, P, s_lower, r_max, threshold;
  unsigned deferred;  // warp-uniform
  long long decisions;
  // this lane's row
  int clock, populated, credits;
  double latest, previous;

  __device__ __forceinline__ bool mine(int lane) const { return lane < P; }
  __device__ __forceinline__ int min_clock(int lane) const {
    return __reduce_min_sync(kFull, mine(lane) ? clock : 0x7fffffff);
  }
  __device__ __forceinline__ int max_clock(int lane) const {
    return __reduce_max_sync(kFull, mine(lane) ? clock : (int)0x80000000);
  }
  __device__ __forceinline__ void record(int lane, int q, double t) {
    if (lane == q) { previous = latest; latest = t; populated += 1; }
  }

  // policy.py:152-206, warp-collective; every lane returns the same result.
  __device__ __forceinline__ GateResult on_push(int lane, int p, double now) {
    GateResult r{PS_OK, 0, 0ull};
    if (p < 0 || p >= P || ((deferred >> p) & 1u)) { r.status = PS_E_PROTOCOL; return r; }
    const int c = from_lane(clock, p) + 1;
    if (lane == p) clock = c;
    decisions += 1;
    if (paradigm == PS_ASP) {
      record(lane, p, now);
      return r;  // grant, no release scan
    }
    int outcome;
    if (paradigm == PS_DSSP) {
      const int cred = from_lane(credits, p);
      if (cred > 0) {
        if (lane == p) credits = cred - 1;
        record(lane, p, now);
        outcome = 0;
      } else {
        const int gap = c - min_clock(lane);
        if (gap <= s_lower) {
          record(lane, p, now);
          outcome = 0;
        } else if (c < max_clock(lane)) {  // not the fastest (ties count as fastest)
          record(lane, p, now);
          outcome = 1;
        } else {
          record(lane, p, now);  // the controller records first (policy.py:121)
          int pred = 0;
          if (r_max > 0) {
            const int low = min_clock(lane);
            const int sl = __ffs(__ballot_sync(kFull, mine(lane) && clock == low)) - 1;
            const int pop_p = from_lane(populated, p), pop_s = from_lane(populated, sl);
            if (pop_p >= 2 && pop_s >= 2)
              pred = controller_grid(from_lane(latest, p), from_lane(previous, p),
                                     from_lane(latest, sl), from_lane(previous, sl), r_max);
          }
          int headroom = s_lower + r_max - gap;
          if (headroom < 0) headroom = 0;
          const int cr = pred < headroom ? pred : headroom;
          if (lane == p) credits = cr;
          outcome = cr > 0 ? 0 : 1;
        }
      }
    } else {
      record(lane, p, now);
      outcome = (c - min_clock(lane) <= threshold) ? 0 : 1;
    }
    r.outcome = outcome;
    if (outcome == 1) {
      deferred |= 1u << p;
    } else if (deferred) {
      const int low = min_clock(lane);
      const unsigned ready =
          __ballot_sync(kFull, mine(lane) && ((deferred >> lane) & 1u) && clock - low <= threshold);
      deferred &= ~ready;
      r.released = ready;
    }
    return r;
  }
};

}  // namespace dssp
