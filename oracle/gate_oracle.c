/*
 * oracle/gate_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C CPU restatement of the reference's hot-path arithmetic, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check the
 * CUDA engine. Nothing in paper_1908_11848_b200/ links or calls this file.
 *
 * Restated from (paths relative to /root/reference/pkg/src/stalesync/):
 *   policy.py:84-90    PushHistoryTable.record / interval (INTERVAL_FLOOR 1e-9, :26)
 *   policy.py:60-73    IterationClockTable.minimum / maximum / slowest / is_fastest
 *   policy.py:108-132  synchronization_controller ((r_max+1)^2 grid, first argmin)
 *   policy.py:138-170  SyncPolicy.__init__ / on_push
 *   policy.py:172-195  SyncPolicy._dssp_decide (credit spend, mint, headroom cap)
 *   policy.py:197-206  SyncPolicy._release (ascending ids, only on grant)
 *   server.py:29-42    apply_update (w - lr*g: a rounded multiply then a rounded
 *                      subtract; no FMA -- built with -ffp-contract=off)
 *   server.py:58-69    ParameterServer.apply_gradient finite checks
 *
 * Pinned against the tests/golden fixtures, which tests/golden/make_golden.py
 * produced by running the reference itself.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORC_MAX_WORKERS 64
enum { ORC_BSP = 0, ORC_ASP = 1, ORC_SSP = 2, ORC_DSSP = 3 };
enum { ORC_GRANT = 0, ORC_DEFER = 1, ORC_E_UNKNOWN = -1, ORC_E_DEFERRED = -2 };

typedef struct {
    int32_t paradigm, worker_count, s_lower, r_max, threshold, _pad;
    int64_t clocks[ORC_MAX_WORKERS];
    double latest[ORC_MAX_WORKERS];
    double previous[ORC_MAX_WORKERS];
    int64_t populated[ORC_MAX_WORKERS];
    int64_t credits[ORC_MAX_WORKERS];
    uint64_t deferred;
} orc_gate;

static const double INTERVAL_FLOOR = 1e-9; /* policy.py:26 */

int orc_sizeof_gate(void) { return (int)sizeof(orc_gate); }

/* policy.py:138-150 */
int orc_gate_init(orc_gate* g, int paradigm, int workers, int s_lower, int r_max) {
    if (workers < 1 || workers > ORC_MAX_WORKERS) return -3;
    memset(g, 0, sizeof(*g));
    g->paradigm = paradigm;
    g->worker_count = workers;
    g->s_lower = s_lower;
    g->r_max = r_max;
    g->threshold = (paradigm == ORC_BSP) ? 0 : s_lower;
    return 0;
}

/* policy.py:84-87 */
static void record(orc_gate* g, int q, double t) {
    g->previous[q] = g->latest[q];
    g->latest[q] = t;
    g->populated[q] += 1;
}

/* policy.py:89-90: Python max(d, floor) returns d unless floor > d */
static double interval_of(double latest, double prev) {
    double d = latest - prev;
    return (INTERVAL_FLOOR > d) ? INTERVAL_FLOOR : d;
}

static int64_t min_clock(const orc_gate* g) {
    int64_t m = g->clocks[0];
    for (int q = 1; q < g->worker_count; q++) if (g->clocks[q] < m) m = g->clocks[q];
    return m;
}

static int64_t max_clock(const orc_gate* g) {
    int64_t m = g->clocks[0];
    for (int q = 1; q < g->worker_count; q++) if (g->clocks[q] > m) m = g->clocks[q];
    return m;
}

/* policy.py:66-69: minimum count, ties to the smallest id */
static int slowest(const orc_gate* g) {
    int64_t m = min_clock(g);
    for (int q = 0; q < g->worker_count; q++) if (g->clocks[q] == m) return q;
    return 0;
}

/* policy.py:127-132 restated as explicit loops (tests/oracles.py:10-28 form):
 * cand(r) = latest_p + r*I_p, slow(k) = latest_s + (k+1)*I_s, each a rounded
 * multiply then a rounded add; argmin over r of min_k |slow(k) - cand(r)|
 * with strict '<' so the first (smallest) r wins ties. */
int orc_controller(double latest_p, double prev_p, double latest_s, double prev_s, int r_max) {
    if (r_max <= 0) return 0;
    double ip = interval_of(latest_p, prev_p);
    double is = interval_of(latest_s, prev_s);
    int best_r = 0;
    double best = INFINITY;
    for (int r = 0; r <= r_max; r++) {
        double cand = latest_p + (double)r * ip;
        double m = INFINITY;
        for (int k = 0; k <= r_max; k++) {
            double slow = latest_s + (double)(k + 1) * is;
            double gap = fabs(slow - cand);
            if (gap < m) m = gap;
        }
        if (m < best) { best = m; best_r = r; }
    }
    return best_r;
}

/* policy.py:108-132: records push_time first, then cold start / grid */
static int controller(orc_gate* g, int p, double now) {
    record(g, p, now);
    if (g->r_max <= 0) return 0;
    int s = slowest(g);
    if (g->populated[p] < 2 || g->populated[s] < 2) return 0;
    return orc_controller(g->latest[p], g->previous[p], g->latest[s], g->previous[s], g->r_max);
}

/* policy.py:172-195 */
static int dssp_decide(orc_gate* g, int p, double now, int64_t count) {
    if (g->credits[p] > 0) {
        g->credits[p] -= 1;
        record(g, p, now);
        return ORC_GRANT;
    }
    int64_t gap = count - min_clock(g);
    if (gap <= g->s_lower) { record(g, p, now); return ORC_GRANT; }
    if (!(g->clocks[p] >= max_clock(g))) { record(g, p, now); return ORC_DEFER; }
    int64_t predicted = controller(g, p, now);
    int64_t headroom = (int64_t)g->s_lower + g->r_max - gap;
    if (headroom < 0) headroom = 0;
    g->credits[p] = predicted < headroom ? predicted : headroom;
    return g->credits[p] > 0 ? ORC_GRANT : ORC_DEFER;
}

/* policy.py:197-206 */
static uint64_t release_ready(orc_gate* g) {
    if (!g->deferred) return 0;
    int64_t low = min_clock(g);
    uint64_t ready = 0;
    for (int q = 0; q < g->worker_count; q++)
        if ((g->deferred >> q) & 1ull)
            if (g->clocks[q] - low <= g->threshold) ready |= (1ull << q);
    g->deferred &= ~ready;
    return ready;
}

/* policy.py:152-170. Returns ORC_GRANT / ORC_DEFER or a negative protocol error. */
int orc_gate_on_push(orc_gate* g, int p, double now, uint64_t* released) {
    *released = 0;
    if (p < 0 || p >= g->worker_count) return ORC_E_UNKNOWN;
    if ((g->deferred >> p) & 1ull) return ORC_E_DEFERRED;
    int64_t count = ++g->clocks[p];
    int outcome;
    if (g->paradigm == ORC_ASP) {
        record(g, p, now);
        return ORC_GRANT;
    } else if (g->paradigm == ORC_DSSP) {
        outcome = dssp_decide(g, p, now, count);
    } else {
        record(g, p, now);
        outcome = (count - min_clock(g) <= g->threshold) ? ORC_GRANT : ORC_DEFER;
    }
    if (outcome == ORC_DEFER) {
        g->deferred |= (1ull << p);
        return ORC_DEFER;
    }
    *released = release_ready(g);
    return ORC_GRANT;
}

/* server.py:36-37 in fp32: w - lr*g as two rounded ops. Returns 0 when every
 * g is finite and every result is finite; 1 = non-finite gradient (nothing
 * written, server.py:65-67); 2 = non-finite result (nothing written,
 * server.py:38-41). out may alias w. */
int orc_apply_f32(const float* w, const float* g, float lr, float* out, int64_t n) {
    for (int64_t i = 0; i < n; i++) if (!isfinite(g[i])) return 1;
    for (int64_t i = 0; i < n; i++) {
        float t = lr * g[i];
        if (!isfinite(w[i] - t)) return 2;
    }
    for (int64_t i = 0; i < n; i++) { float t = lr * g[i]; out[i] = w[i] - t; }
    return 0;
}

int orc_apply_f64(const double* w, const double* g, double lr, double* out, int64_t n) {
    for (int64_t i = 0; i < n; i++) if (!isfinite(g[i])) return 1;
    for (int64_t i = 0; i < n; i++) {
        double t = lr * g[i];
        if (!isfinite(w[i] - t)) return 2;
    }
    for (int64_t i = 0; i < n; i++) { double t = lr * g[i]; out[i] = w[i] - t; }
    return 0;
}
