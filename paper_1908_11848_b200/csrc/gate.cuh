// gate.cuh -- the device-resident DSSP synchronization gate.
//
// One warp runs one decision: lane 0 owns the state machine (clock table,
// two-deep push history, credits, deferred mask) and all 32 lanes share the
// controller's (r_max+1)^2 fp64 grid. BSP, ASP and SSP are the degenerate
// settings of the same machine, exactly as in the reference:
//
//   policy.py:84-90    record / interval (floor 1e-9)
//   policy.py:60-73    minimum / maximum / slowest (ties -> smallest id) / is_fastest (ties count)
//   policy.py:108-132  synchronization_controller
//   policy.py:152-170  on_push        policy.py:172-195  _dssp_decide
//   policy.py:197-206  _release (only on GRANT, ascending ids)
//
// Bit-exactness: every controller product and sum is an explicitly rounded
// __dmul_rn / __dadd_rn / __dsub_rn (numpy evaluates r*I then latest + that,
// never an FMA), the per-r minimum is exact, and the argmin keeps the smallest
// r among equal minima (numpy argmin returns the first occurrence).
#pragma once

#include <stdint.h>
#include "../../include/dssp_ps.h"

namespace dssp {

constexpr double kIntervalFloor = 1e-9;  // policy.py:26
constexpr unsigned kFull = 0xffffffffu;

struct GateResult {
  int status;                 // PS_OK or PS_E_PROTOCOL
  int outcome;                // 0 grant, 1 defer
  unsigned long long released;
};

__device__ __forceinline__ double interval_of(double latest, double prev) {
  double d = __dsub_rn(latest, prev);
  return (kIntervalFloor > d) ? kIntervalFloor : d;  // Python max(d, floor)
}

// Warp-collective controller grid; every lane passes the same arguments.
__device__ __forceinline__ int controller_grid(double lp, double pp, double ls, double ps, int r_max) {
  const int lane = threadIdx.x & 31;
  const double ip = interval_of(lp, pp);
  const double is = interval_of(ls, ps);
  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int best_r = 0x7fffffff;
  // slow(k) = ls + (k+1)*is is non-decreasing in k (is > 0 and round-to-
  // nearest is monotone), so |slow(k) - cand| is minimized at the last k with
  // slow(k) <= cand or the one after it: a binary search finds that pair and
  // the per-r minimum equals the brute-force min over all k bit for bit.
  if (r_max <= 16) {
    // small grids: the reference's brute force, literally -- r_max+1
    // independent evaluations per lane pipeline better than the search's
    // dependent steps (policy.py:127-132)
    if (lane <= r_max) {
      const double cand = __dadd_rn(lp, __dmul_rn((double)lane, ip));
      const double inf = __longlong_as_double(0x7ff0000000000000ll);
      // all distances first (independent), then a min tree: no serial chain
      // through 17 dependent fp64 min operations
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k)
        v[k] = k <= r_max ? fabs(__dsub_rn(__dadd_rn(ls, __dmul_rn((double)(k + 1), is)), cand)) : inf;
#pragma unroll
      for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) v[k] = fmin(v[k], v[k + w]);
      // k = 16 (r_max == 16) is the one entry the tree does not hold
      best = r_max >= 16 ? fmin(v[0], fabs(__dsub_rn(__dadd_rn(ls, __dmul_rn(17.0, is)), cand))) : v[0];
      best_r = lane;
    }
  } else
  for (int r = lane; r <= r_max; r += 32) {
    const double cand = __dadd_rn(lp, __dmul_rn((double)r, ip));
    int lo = -1, hi = r_max + 1;  // slow(lo) <= cand < slow(hi), virtual ends
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__dadd_rn(ls, __dmul_rn((double)(mid + 1), is)) <= cand) lo = mid;
      else hi = mid;
    }
    double m = __longlong_as_double(0x7ff0000000000000ll);
    if (lo >= 0) m = fabs(__dsub_rn(__dadd_rn(ls, __dmul_rn((double)(lo + 1), is)), cand));
    if (hi <= r_max) {
      const double gh = fabs(__dsub_rn(__dadd_rn(ls, __dmul_rn((double)(hi + 1), is)), cand));
      if (gh < m) m = gh;
    }
    if (m < best) { best = m; best_r = r; }
  }
  // argmin over the lanes, first index wins on ties: the bit pattern of a
  // non-negative double orders like its value, so three integer redux
  // steps (high word, low word, r) replace a 5-round shuffle tree
  const unsigned long long bits = (unsigned long long)__double_as_longlong(best);
  const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
  return (int)__reduce_min_sync(kFull, (hi == mhi && lo == mlo) ? (unsigned)best_r : 0x7fffffffu);
}

// One lane's own controller (same arguments and result as controller_grid),
// for a warp that evaluates up to 32 decisions at once.
// cand(r) = lp + r*ip and slow(k) = ls + (k+1)*is are both non-decreasing
// (positive intervals, monotone rounding), so the last k with slow(k) <= cand
// -- the crossing, where |slow(k) - cand| is smallest, at it or the next k --
// only moves forward as r grows: one forward sweep over k for all r, each
// distance with controller_grid's exact rounded expressions, the first r on
// ties. `ok` is always set (kept for the caller's exact fallback hook).
__device__ __forceinline__ int controller_lane(double lp, double pp, double ls, double ps, int r_max, bool& ok) {
  const double ip = interval_of(lp, pp);
  const double is = interval_of(ls, ps);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double best = inf;
  int best_r = 0;
  int lo = -1;                                   // last k with slow(k) <= cand (-1: none)
  double s_lo = inf;                             // slow(lo)
  double s_hi = __dadd_rn(ls, __dmul_rn(1.0, is));  // slow(lo + 1) (inf past r_max)
  for (int r = 0; r <= r_max; ++r) {
    const double cand = __dadd_rn(lp, __dmul_rn((double)r, ip));
    while (lo < r_max && s_hi <= cand) {
      ++lo;
      s_lo = s_hi;
      s_hi = lo < r_max ? __dadd_rn(ls, __dmul_rn((double)(lo + 2), is)) : inf;
    }
    double m = lo >= 0 ? fabs(__dsub_rn(s_lo, cand)) : inf;
    if (lo < r_max) m = fmin(m, fabs(__dsub_rn(s_hi, cand)));
    if (m < best) { best = m; best_r = r; }
  }
  ok = true;
  return best_r;
}

__device__ __forceinline__ void record(ps_gate_state* s, int q, double t) {
  s->previous[q] = s->latest[q];
  s->latest[q] = t;
  s->populated[q] += 1;
}

__device__ __forceinline__ long long min_clock(const ps_gate_state* s) {
  long long m = s->clocks[0];
  for (int q = 1; q < s->worker_count; ++q) m = s->clocks[q] < m ? s->clocks[q] : m;
  return m;
}

__device__ __forceinline__ long long max_clock(const ps_gate_state* s) {
  long long m = s->clocks[0];
  for (int q = 1; q < s->worker_count; ++q) m = s->clocks[q] > m ? s->clocks[q] : m;
  return m;
}

__device__ __forceinline__ int slowest(const ps_gate_state* s) {
  const long long m = min_clock(s);
  for (int q = 0; q < s->worker_count; ++q)
    if (s->clocks[q] == m) return q;
  return 0;
}

__device__ __forceinline__ unsigned long long release_ready(ps_gate_state* s) {
  if (!s->deferred) return 0ull;
  const long long low = min_clock(s);
  unsigned long long ready = 0ull;
  for (int q = 0; q < s->worker_count; ++q)
    if (((s->deferred >> q) & 1ull) && s->clocks[q] - low <= s->threshold) ready |= 1ull << q;
  s->deferred &= ~ready;
  return ready;
}

// Warp-collective SyncPolicy.on_push. Only lane 0 touches *s; the result is
// broadcast to every lane.
__device__ inline GateResult gate_on_push(ps_gate_state* s, int p, double now) {
  const int lane = threadIdx.x & 31;
  int status = PS_OK, outcome = 0, stage = 0;  // stage 1: DSSP mint needs the controller grid
  long long gap = 0;
  double lp = 0, pp = 0, ls = 0, ps = 0;
  int r_max = 0;
  if (lane == 0) {
    if (p < 0 || p >= s->worker_count) {
      status = PS_E_PROTOCOL;                       // unknown worker
    } else if ((s->deferred >> p) & 1ull) {
      status = PS_E_PROTOCOL;                       // pushed while deferred
    } else {
      const long long count = ++s->clocks[p];
      if (s->paradigm == PS_ASP) {
        record(s, p, now);
        outcome = 0;
        stage = 3;                                  // grant, no release scan
      } else if (s->paradigm == PS_DSSP) {
        if (s->credits[p] > 0) {
          s->credits[p] -= 1;
          record(s, p, now);
          outcome = 0;
        } else {
          gap = count - min_clock(s);
          if (gap <= s->s_lower) {
            record(s, p, now);
            outcome = 0;
          } else if (!(s->clocks[p] >= max_clock(s))) {
            record(s, p, now);
            outcome = 1;
          } else {
            record(s, p, now);                      // the controller records first
            r_max = s->r_max;
            stage = 2;                              // pred = 0 unless the grid runs
            if (r_max > 0) {
              const int sl = slowest(s);
              if (s->populated[p] >= 2 && s->populated[sl] >= 2) {
                lp = s->latest[p]; pp = s->previous[p];
                ls = s->latest[sl]; ps = s->previous[sl];
                stage = 1;
              }
            }
          }
        }
      } else {
        record(s, p, now);
        outcome = (count - min_clock(s) <= s->threshold) ? 0 : 1;
      }
    }
  }
  stage = __shfl_sync(kFull, stage, 0);
  int pred = 0;
  if (stage == 1) {
    lp = __shfl_sync(kFull, lp, 0); pp = __shfl_sync(kFull, pp, 0);
    ls = __shfl_sync(kFull, ls, 0); ps = __shfl_sync(kFull, ps, 0);
    r_max = __shfl_sync(kFull, r_max, 0);
    pred = controller_grid(lp, pp, ls, ps, r_max);
  }
  unsigned long long released = 0ull;
  if (lane == 0 && status == PS_OK) {
    if (stage == 1 || stage == 2) {
      long long headroom = (long long)s->s_lower + s->r_max - gap;
      if (headroom < 0) headroom = 0;
      const long long c = (long long)pred < headroom ? (long long)pred : headroom;
      s->credits[p] = c;
      outcome = c > 0 ? 0 : 1;
    }
    if (outcome == 1) {
      s->deferred |= 1ull << p;
    } else if (stage != 3) {
      released = release_ready(s);
    }
    s->decisions += 1;
  }
  GateResult r;
  r.status = __shfl_sync(kFull, status, 0);
  r.outcome = __shfl_sync(kFull, outcome, 0);
  r.released = __shfl_sync(kFull, released, 0);
  return r;
}

__device__ __forceinline__ void gate_init(ps_gate_state* s, int paradigm, int workers, int s_lower,
                                          int r_max) {
  s->paradigm = paradigm;
  s->worker_count = workers;
  s->s_lower = s_lower;
  s->r_max = r_max;
  s->threshold = paradigm == PS_BSP ? 0 : s_lower;
}

}  // namespace dssp
