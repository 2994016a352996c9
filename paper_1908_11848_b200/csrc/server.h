// server.h -- host-side state of one single-GPU parameter server handle.
#pragma once

#include <cuda_runtime.h>
#include <string>
#include "common.cuh"

struct ps_sim_buffers {
  size_t ops_cap = 0, slots_cap = 0, trace_cap = 0, loss_cap = 0, ctime_cap = 0;
  int P = 0;
  void* ops = nullptr;                 // Op[ops_cap] (tagged 64-bit words)
  unsigned tag = 0;                    // run tag of the op words
  unsigned* gcount = nullptr;          // [slots_cap] per-update finiteness words
  float* rep = nullptr;                // [P][2][dpad] worker replicas
  float* gbuf = nullptr;               // [P][dpad] worker gradients
  float* center = nullptr;             // [dpad]
  double* ctime = nullptr;             // [P][budget]
  ps_trace_row* trace = nullptr;
  double* losses = nullptr;
  void* out = nullptr;                 // SimOut
  void* calls = nullptr;               // replay: ps_replay_call[calls_cap]
  long long* decisions = nullptr;      // replay: one word per decide
  unsigned long long* dstream = nullptr;  // replay: the gate's data-call descriptors (tagged)
  unsigned dtag = 0;                   // replay: run tag of the descriptor words
  unsigned long long* pred = nullptr;  // replay: controller results by call (tagged)
  size_t pred_cap = 0;
  size_t calls_cap = 0, dec_cap = 0, dstream_cap = 0;
  int64_t last_decisions = 0;
  int64_t last_trace_rows = 0, last_loss_samples = 0, last_loss_every = 0, last_base_version = 0;
};

struct ps_worker_rt;  // ps_workers.cu: free-running workers on device flags
struct ps_resident;   // ps_server.cu: the persistent per-call server (ps_set_resident)

struct ps_server {
  ps_config cfg{};
  int dev = 0;
  cudaStream_t stream = nullptr;
  int64_t d = 0, nv = 0, dpad = 0;     // elements, float4 count, padded length
  float* w[2] = {nullptr, nullptr};    // double-buffered fp32 weights (device)
  dssp::Ctrl* ctrl = nullptr;          // device control block
  dssp::Ctrl* hctrl_dev = nullptr;     // device alias of the mapped host mirror hctrl
  int profile = 0;                     // 1: bracket each launch with CUDA events
  int* habort = nullptr;               // mapped host flag: abort a free-running run
  int* habort_dev = nullptr;
  cudaStream_t producer = nullptr;     // caller's stream that writes updates / reads pulls
  cudaEvent_t ev_in = nullptr;         // orders the server stream after `producer`
  dssp::Ctrl* hctrl = nullptr;         // pinned host mirror
  int cur = 0;                         // host mirror of ctrl->cur
  void* stage = nullptr;               // device staging for host-side gradients
  void* hstage = nullptr;              // pinned host staging
  size_t stage_bytes = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int sm_count = 148;
  std::string err;
  ps_sim_buffers sim;
  ps_worker_rt* wrt = nullptr;
  ps_resident* res = nullptr;
};

// Stop the resident per-call kernel (if running) before any other use of the
// server's device state; the next per-call op relaunches it.
int ps_resident_pause(ps_server* h);

void ps_workers_free(ps_server* h);

int ps_fail(ps_server* h, int code, const std::string& msg);
// Order h->stream after the caller's producer stream (ps_set_producer_stream).
int ps_order_after_producer(ps_server* h);
int ps_cuda_fail(ps_server* h, cudaError_t e, const char* what);

#define PS_CK(h, call)                                          \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return ps_cuda_fail((h), _e, #call); \
  } while (0)
