/*
 * dssp_ps.h -- C-ABI of the B200 parameter-server engine (push / pull / DSSP gate).
 *
 * Plain pointers, sizes and POD structs only: no torch or CUDA types cross this
 * boundary, so the reference's Python host side (or any FFI) can bind it. The
 * binding the reference would add is shown in INTEGRATION.md; the Python shim in
 * paper_1908_11848_b200/ uses ctypes.
 *
 * Every entry point replaces one reference interface (paths relative to
 * /root/reference/pkg/src/stalesync/):
 *
 *   ps_create           ParameterServer.__init__ + SyncPolicy.__init__   server.py:45-52, policy.py:138-150
 *   ps_apply            ParameterServer.apply_gradient / apply_update     server.py:58-69, :29-42
 *   ps_decide           ParameterServer.decide_push -> SyncPolicy.on_push server.py:71-78, policy.py:152-206
 *   ps_push             ParameterServer.handle_push (apply, then decide)  server.py:80-82
 *   ps_pull             ParameterServer.handle_pull (materialized copy)   server.py:84-91
 *   ps_read_weights     ParameterServer.weights.values / .version         server.py:47, config.py:54-68
 *   ps_get_state/peek   SyncPolicy.clocks / .history / .credits / .deferred  policy.py:43-105
 *   ps_set_state        direct table writes the reference tests perform   tests/test_policy.py:156-166, :209-220
 *   ps_controller_batch synchronization_controller (pure grid, oracle hook)  policy.py:108-132
 *   ps_apply_vectors    apply_update on plain vectors (stateless)          server.py:29-42
 *   ps_sim_run          Simulation.run event loop, device-resident          simnet.py:127-201
 *   ps_sim_trace        Simulation.entries (TraceEntry rows)               simnet.py:110-112, trace.py:28-37
 *   ps_replay_run       the server answering a recorded handle_pull / apply_gradient /
 *                       decide_push stream in one launch                   simnet.py:135-138, :183-201
 *   ps_replay_read_replica  the snapshots those handle_pull calls returned  server.py:84-91
 *   ps_workers_* / ps_bind_worker_stream / ps_enqueue_iteration
 *                       ThreadedRun worker loop, lock and release events  runner.py:168-291
 *
 *   ps_shard_*          the same push/pull/gate over G GPUs (one process per
 *                       GPU, contiguous-range shards, P2P over NVLink)
 *
 * Threading: like the reference ("callers serialize on_push calls",
 * policy.py:136), calls on one handle must be serialized by the caller.
 * Status codes: PS_OK (0), PS_REJECTED (1: non-finite gradient, counted, not an
 * error -- server.py:65-67), negative values map 1:1 onto the reference's
 * exceptions; ps_last_error() returns the message of the last failure.
 */
#ifndef DSSP_PS_H
#define DSSP_PS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_MAX_WORKERS 64

enum ps_paradigm { PS_BSP = 0, PS_ASP = 1, PS_SSP = 2, PS_DSSP = 3 };

enum ps_status {
  PS_OK = 0,
  PS_REJECTED = 1,       /* non-finite gradient: rejected_updates += 1 (server.py:65-67) */
  PS_E_PROTOCOL = -1,    /* ProtocolError (policy.py:29-30, :153-156; server.py:87-90) */
  PS_E_VALUE = -2,       /* ValueError: dimension mismatch, lr <= 0, bad config (server.py:31-35, :61-64) */
  PS_E_DIVERGED = -3,    /* DivergenceError (server.py:20-21, :38-41) */
  PS_E_CUDA = -4,        /* CUDA runtime failure */
  PS_E_DEADLOCK = -5,    /* DeadlockError (simnet.py:28-31, :150-153) */
  PS_E_BUDGET = -6,      /* event budget exceeded (simnet.py:131-132) */
  PS_E_TIMEOUT = -7      /* a device wait exceeded its watchdog (multi-GPU flags) */
};

enum ps_dtype { PS_F32 = 0, PS_F64 = 1 };

typedef struct ps_config {
  int32_t paradigm;      /* enum ps_paradigm */
  int32_t worker_count;  /* P, 1..PS_MAX_WORKERS */
  int32_t s_lower;       /* normalized as validate_config does (config.py:304-308) */
  int32_t r_max;
  double learning_rate;  /* > 0 */
  int64_t dimension;     /* d >= 1 */
  int32_t device;        /* CUDA ordinal of the (single-GPU) server */
  int32_t reserved[7];
} ps_config;

/* Host mirror of the device control block (policy.py:43-105 tables). */
typedef struct ps_gate_state {
  int32_t paradigm, worker_count, s_lower, r_max, threshold, _pad;
  int64_t clocks[PS_MAX_WORKERS];
  double latest[PS_MAX_WORKERS];
  double previous[PS_MAX_WORKERS];
  int64_t populated[PS_MAX_WORKERS];
  int64_t credits[PS_MAX_WORKERS];
  uint64_t deferred;      /* bit q set: worker q is deferred */
  int64_t version;        /* applied updates (WeightVector.version) */
  int64_t rejected;       /* rejected_updates */
  int64_t decisions;      /* on_push calls decided */
} ps_gate_state;

typedef struct ps_server ps_server;

/* Lifecycle. w0 is the initial weight vector on the host (PS_F64 as the
 * reference draws it, server.py:24-26, or PS_F32); it is rounded to fp32. */
int ps_create(const ps_config* cfg, const void* w0_host, int32_t w0_dtype, ps_server** out);
void ps_destroy(ps_server* h);
const char* ps_last_error(const ps_server* h); /* h may be NULL (last create failure) */
int ps_device_count(int32_t* n);

/* Push path. g is d values in g_dtype, on the host or (g_on_device=1) in the
 * server's device memory, borrowed for the call. *applied = 0 when rejected. */
int ps_apply(ps_server* h, int32_t worker, const void* g, int32_t g_dtype, int32_t g_on_device,
             int32_t* applied);
int ps_decide(ps_server* h, int32_t worker, double now, int32_t* granted, uint64_t* released);
int ps_push(ps_server* h, int32_t worker, const void* g, int32_t g_dtype, int32_t g_on_device,
            double now, int32_t* applied, int32_t* granted, uint64_t* released);

/* Pull path: materializes the current weights into dst (d values). */
int ps_pull(ps_server* h, int32_t worker, void* dst, int32_t dst_dtype, int32_t dst_on_device,
            int64_t* version);
int ps_read_weights(ps_server* h, void* dst, int32_t dst_dtype, int32_t dst_on_device,
                    int64_t* version);

/* Gate state. ps_get_state synchronizes with the device; ps_peek_state returns
 * the host mirror refreshed by the last synchronous call (no device traffic). */
int ps_get_state(ps_server* h, ps_gate_state* out);
int ps_peek_state(const ps_server* h, ps_gate_state* out);
int ps_set_state(ps_server* h, const ps_gate_state* in);

/* Oracle hooks. tables: n rows of (latest_p, prev_p, latest_s, prev_s). */
int ps_controller_batch(int32_t device, const double* tables, const int32_t* r_max, int32_t n,
                        int32_t* out);
int ps_apply_vectors(int32_t device, const void* w, const void* g, int32_t dtype, int64_t n,
                     double lr, void* out, int32_t* status);

/* ------------------------------------------------------------------------
 * Device-resident simulation (simnet.py:127-201): the whole event loop,
 * gate decisions, pulls, gradient production and applies run in ONE
 * persistent kernel; the host only launches it and reads the trace.
 * ---------------------------------------------------------------------- */
enum ps_grad_kind { PS_GRAD_BOWL = 0, PS_GRAD_SYNTHETIC = 1 };
enum ps_event_kind {
  PS_EV_COMPUTE_DONE = 0, PS_EV_PUSH_ARRIVE = 1, PS_EV_GRANT_DELIVER = 2,
  PS_EV_PULL_ARRIVE = 3, PS_EV_PULL_RETURN = 4   /* trace.py:19-25 */
};

typedef struct ps_sim_config {
  int32_t budget;              /* pushes per worker (engine.py:243-248) */
  int32_t grad_kind;           /* enum ps_grad_kind */
  int32_t loss_every;          /* 0: no loss sampling (simnet.py:118-125) */
  int32_t n_synthetic;         /* synthetic update buffers per worker */
  double comm_delay;           /* TimingSpec.comm_delay */
  const double* compute_time;  /* host [P * budget]: the k-th compute draw of worker p */
  const void* center;          /* host [d] bowl center (PS_GRAD_BOWL) */
  int32_t center_dtype;
  int32_t record_trace;        /* 1: keep TraceEntry rows */
  const float* synthetic;      /* device [P][n_synthetic][round_up(d,4)] (PS_GRAD_SYNTHETIC) */
  int64_t max_events;          /* 0: unbounded */
  int32_t data_ctas;           /* 0: one per SM minus the control CTA */
  int32_t reset_gate;          /* 1: zero the gate tables first (a fresh run) */
  int32_t mode;                /* 0: virtual time (simnet.py); 2: free-running on the wall clock
                                  (runner.py: each push is apply -> decide on its own, decided at
                                  the time it actually arrives; P <= 8) */
  int32_t _pad;
  double time_scale;           /* mode 2: wall-clock seconds per schedule second */
  double deadline_s;           /* mode 2: watchdog (deadline_guard, runner.py:294-298); 0 = none */
} ps_sim_config;

typedef struct ps_sim_result {
  int64_t events;              /* events processed */
  int64_t pushes;              /* push decisions */
  int64_t applied;             /* updates applied (final version delta) */
  int64_t rejected;
  int64_t trace_rows;
  int64_t loss_samples;
  uint64_t unfinished;         /* DeadlockError workers */
  int32_t status;              /* enum ps_status */
  int32_t diverged_worker;
  double device_ms;            /* kernel time, CUDA events on the launch stream */
  double control_ms;           /* control warp: start -> last op emitted (%globaltimer) */
  double data_ms;              /* start -> last data warp done (%globaltimer) */
} ps_sim_result;

typedef struct ps_trace_row {
  double time;
  int32_t worker;
  int32_t kind;                /* enum ps_event_kind */
  int64_t count;               /* clocks[worker] at the event (trace.py:32) */
  int32_t decision;            /* -1 none, 0 grant, 1 defer */
  int32_t _pad;
  uint64_t released;           /* ascending ids as a bit mask */
} ps_trace_row;

int ps_sim_run(ps_server* h, const ps_sim_config* sc, ps_sim_result* out);
/* Abort a free-running ps_sim_run from another host thread (ThreadedRun.abort,
 * runner.py:110-111): the run stops, returns PS_E_TIMEOUT and reports its
 * unfinished workers in ps_sim_result.unfinished. */
int ps_abort(ps_server* h);

/* Replay: the server serving a recorded request stream -- the reference's
 * boundary call sequence (handle_pull / apply_gradient / decide_push, in the
 * order the simulator issues them) executed in one persistent kernel: pulls
 * and applies as data ops, every decide through the device gate (decisions
 * retrievable with ps_replay_decisions as (released << 8) | outcome, hence at
 * most 55 workers). Updates are resident: apply k of worker p uses
 * synthetic[p][k % n_synthetic]. A protocol violation stops the data at the
 * offending call (PS_E_PROTOCOL); a non-finite update is rejected and
 * counted (ps_sim_result.rejected). */
enum { PS_CALL_PULL = 0, PS_CALL_APPLY = 1, PS_CALL_DECIDE = 2 };
typedef struct ps_replay_call {
  double now;       /* PS_CALL_DECIDE: the push instant */
  int32_t kind;
  int32_t worker;
} ps_replay_call;
int ps_replay_run(ps_server* h, const ps_replay_call* calls, int64_t n, const float* synthetic,
                  int32_t n_synthetic, int32_t reset_gate, int32_t data_ctas, ps_sim_result* out);
int ps_replay_decisions(ps_server* h, int64_t* out, int64_t cap, int64_t* n);
/* The pulled weights a run left in worker p's replicas (handle_pull's
 * snapshot, server.py:84-91): a replay writes pull k (k = 0, 1, ...) of
 * worker p into buffer (k + 1) % 2, so the two buffers hold that worker's last two pulls;
 * a simulation keeps its staging (PULL_ARRIVE) and active (PULL_RETURN)
 * copies there. dst_host receives d fp32 values. */
int ps_replay_read_replica(ps_server* h, int32_t worker, int32_t buf, float* dst_host);
/* Measurement only (no reference counterpart): the replay's data side with
 * no control at all -- every data warp streams `pulls` stores of its
 * register-resident slice into 8 rotating scratch replicas and `applies`
 * loads + applies from 8 rotating scratch updates, interleaved, on the
 * replay's own grid and slice layout. The best of `reps` device times is the
 * ceiling ps_replay_run's data warps are measured against. */
int ps_replay_ceiling(ps_server* h, int32_t pulls, int32_t applies, int32_t reps, double* best_ms);
int ps_sim_trace(ps_server* h, ps_trace_row* rows, int64_t cap, int64_t* n);
/* Loss samples of the last run: (version, 0.5*||w - c||^2 in fp64). */
int ps_sim_losses(ps_server* h, int64_t* versions, double* losses, int64_t cap, int64_t* n);

/* Device time (CUDA events on the server stream) of the last launch, in ms:
 * always for ps_sim_run, for the per-op calls only with profiling on (the
 * events cost two API calls per op, so they are off on the hot path). */
int ps_last_kernel_ms(ps_server* h, double* ms);
int ps_set_profiling(ps_server* h, int32_t on);
/* The same bracket around an empty kernel: the floor every per-op figure
 * above contains (launch as the GPU sees it + the two timestamps). */
int ps_profile_floor(ps_server* h, double* ms);

/* Device-pointer updates and pull destinations are usually produced/consumed
 * on the caller's own CUDA stream (a cudaStream_t passed as an opaque
 * pointer; NULL = none; the legacy default stream is cudaStreamLegacy,
 * (void*)1, since its handle 0 would read as "none"). Every later push/pull
 * is stream-ordered after the work already enqueued there (an event edge, no
 * host synchronization). */
int ps_set_producer_stream(ps_server* h, void* cuda_stream);

/* Resident mode: `ctas` > 0 keeps a persistent kernel of that many CTAs on
 * the GPU that serves ps_apply / ps_decide / ps_push / ps_pull /
 * ps_read_weights from a pinned, host-mapped mailbox -- no launch and no
 * stream synchronization per call (the reference's per-call API,
 * server.py:58-91, at mailbox latency). 0 turns it off. The kernel retires
 * itself after ~2 s without requests and the next call relaunches it; every
 * other entry point (state writes, run loops, free-running workers) pauses
 * it first. Device updates from a producer stream are waited for on the host
 * (an event synchronization), since no launch carries the stream edge. */
int ps_set_resident(ps_server* h, int32_t ctas);

/* ------------------------------------------------------------------------
 * Free-running workers on device flags (the threaded runner without the host:
 * runner.py:168-291). Every worker is a CUDA stream; an iteration is the
 * worker's own forward/backward, then ps_enqueue_iteration's three stream
 * items: a push kernel (ticket, apply in ticket order, gate decision at the
 * device clock -- apply_gradient -> decide_push under the runner's lock,
 * runner.py:226-249 -- and the go flags of the granted / released workers,
 * policy.py:197-206), a stream memory wait on the worker's go flag (a
 * deferred worker's stream blocks there, runner.py:255-263, occupying no SM
 * and no host thread), and a pull kernel (ticket, the weights into the bound
 * parameter buffer, runner.py:273-284). All state is device-resident and per
 * worker, so the iteration can be captured once in a CUDA graph and replayed
 * with no host work. The per-op calls above must not be used while workers
 * run. Streams that wait must not share a hardware queue with streams they
 * wait for: raise CUDA_DEVICE_MAX_CONNECTIONS (e.g. 32) before CUDA starts.
 * ---------------------------------------------------------------------- */
typedef struct ps_workers_report {
  int64_t tickets;             /* pushes + pulls served */
  int64_t decisions;           /* pushes decided */
  int64_t pulls;
  uint64_t go_mask;            /* workers currently allowed past their wait */
  int32_t status;              /* PS_OK, PS_E_DIVERGED, PS_E_PROTOCOL, PS_E_TIMEOUT */
  int32_t diverged_worker;
  int32_t aborted;
  int32_t _pad;
} ps_workers_report;

typedef struct ps_worker_decision {   /* one decided push, in ticket order */
  uint64_t ticket;
  double now;                  /* gate seconds since ps_workers_start (device clock x scale) */
  int32_t worker;
  int32_t outcome;             /* 0 grant, 1 defer */
  uint64_t released;           /* bit q: worker q released by this grant */
  int64_t version;             /* weights version after this push */
  int32_t applied;             /* 0: non-finite update, rejected (server.py:65-67) */
  int32_t _pad;
} ps_worker_decision;

typedef struct ps_worker_pull {
  uint64_t ticket;
  double now;
  int32_t worker;
  int32_t _pad;
  int64_t version;             /* version of the snapshot the worker received */
} ps_worker_pull;

/* Reset the ticket counter, go flags and logs (log_cap rows each) and start
 * the gate clock: now = (device time since this call) x time_scale seconds. */
int ps_workers_start(ps_server* h, int64_t log_cap, double time_scale);
/* Bind worker p to its stream and flat fp32 buffers (device, 16-B aligned,
 * >= round_up(d,4) floats): the push reads `grad`, the pull writes `params`. */
int ps_bind_worker_stream(ps_server* h, int32_t worker, void* cuda_stream, const float* grad,
                          float* params);
/* Enqueue push -> wait(go[p]) -> pull on `cuda_stream` (NULL: the bound one;
 * pass the capturing stream inside a CUDA-graph capture). throttle_ns > 0
 * first busy-waits that long on the device (runner.py:185-189 spin_compute;
 * the 1x/2x/4x throttle of BASELINE configs[3]). */
int ps_enqueue_iteration(ps_server* h, int32_t worker, void* cuda_stream, uint64_t throttle_ns);
/* Diagnostics: copy every update worker p pushes into ring[k % capacity]
 * (device, [capacity][round_up(d,4)] fp32); NULL turns it off. */
int ps_worker_record(ps_server* h, int32_t worker, float* ring, int64_t capacity);
int ps_workers_status(ps_server* h, ps_workers_report* out);
int ps_workers_log(ps_server* h, ps_worker_decision* dec, int64_t dec_cap, ps_worker_pull* pulls,
                   int64_t pull_cap, int64_t* n_dec, int64_t* n_pull);
/* Abort a free-running run from the host (ThreadedRun.abort, runner.py:110-111):
 * raises every go flag so no stream stays blocked; later kernels only
 * advance the ticket. */
int ps_workers_abort(ps_server* h);

/* ------------------------------------------------------------------------
 * Sharded server: G GPUs, one process (rank) per GPU, one worker per rank.
 * Shard r owns [r*S, min(d,(r+1)*S)), S = ceil(d/G) rounded up to 4. Ranks
 * exchange the opaque blobs of ps_shard_ipc_handles (any host transport --
 * the Python side uses torch.distributed.all_gather_object) and call
 * ps_shard_connect; afterwards every step moves data only over NVLink P2P
 * and synchronizes only through device flags (no collective, no host).
 * Replaces the same reference interfaces as the single-GPU server, for the
 * sharded layout of SURVEY.md section 8(e).
 * ---------------------------------------------------------------------- */
typedef struct ps_shard_server ps_shard_server;

int ps_shard_range(int64_t d, int32_t world, int32_t rank, int64_t* lo, int64_t* hi);
/* w0: full-length initial weights; w0_flags bit 0 = device pointer, bit 1 = fp64. */
int ps_shard_create(const ps_config* cfg, int32_t world, int32_t rank, const void* w0,
                    int64_t w0_flags, ps_shard_server** out);
/* Collective shutdown: every rank calls ps_shard_disconnect (unmaps its
 * peers' buffers), the ranks synchronize, then every rank calls
 * ps_shard_destroy (frees its own). A process must not free memory a peer
 * still has mapped. */
int ps_shard_disconnect(ps_shard_server* h);
void ps_shard_destroy(ps_shard_server* h);
const char* ps_shard_last_error(const ps_shard_server* h);
int ps_shard_ipc_handles(ps_shard_server* h, void* out, int64_t cap); /* returns blob size */
int ps_shard_connect(ps_shard_server* h, const void* blobs, int64_t len);
/* Any push groups (heterogeneous schedules): row i of `groups`, with
 * PS_SHARD_GROUP_STRIDE int32 per row, is {n pushers, pull mask, ticket
 * order[n]} of step i -- the workers that push at that instant in the order
 * the reference's event loop serves them (simnet.py:167-201), and the workers
 * whose pull arrives before the next group (their replica receives the
 * weights after this group). ps_shard_run is the homogeneous special case
 * (every worker pushes and pulls every step). */
#define PS_SHARD_GROUP_STRIDE 18
int ps_shard_run_groups(ps_shard_server* h, int64_t t0, int32_t steps, const double* now,
                        const int32_t* groups, void* dst, double* ms);
/* The worker's update buffer (device, fp32, padded_len >= d): push source. */
int ps_shard_update_buffer(ps_shard_server* h, void** ptr, int64_t* padded_len);
/* The worker's replica (device, fp32): starts as w0 and is rewritten by every
 * owner at each pull (handle_pull, server.py:84-91); a GPU-resident worker can
 * keep its model parameters in it. */
int ps_shard_replica_buffer(ps_shard_server* h, void** ptr, int64_t* padded_len);
/* Run `steps` push groups (tickets t0..t0+steps-1, one push per rank each,
 * applied in rank order then decided in rank order at virtual time now[i]),
 * each followed by this rank's pull into dst (device fp32, >= round_up(d,4)
 * floats; NULL = internal replica). Blocks until done; *ms = device time. */
int ps_shard_run(ps_shard_server* h, int64_t t0, int32_t steps, const double* now, void* dst,
                 double* ms);
int ps_shard_read_shard(ps_shard_server* h, void* dst_host, int64_t* n);
int ps_shard_read_replica(ps_shard_server* h, void* dst_host);
int ps_shard_get_state(ps_shard_server* h, ps_gate_state* out);
int ps_shard_trace(ps_shard_server* h, ps_trace_row* rows, int64_t cap, int64_t* n);
/* Diagnosis only: this owner's streaming pass (every worker's update slice in,
 * the new shard into every replica) `reps` times with no flags and no peer
 * participation, so a profiler can replay it in one process and read its
 * NVLink counters. Destroys the replicas' contents. *ms = device time. */
int ps_shard_stream_probe(ps_shard_server* h, int32_t reps, double* ms);
/* Diagnosis only: per-kernel event timing (ready / apply / pull, ms summed). */
int ps_shard_set_profiling(ps_shard_server* h, int32_t on);
int ps_shard_phase_ms(ps_shard_server* h, double* out3);

#ifdef __cplusplus
}
#endif
#endif /* DSSP_PS_H */
