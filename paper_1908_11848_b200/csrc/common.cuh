// common.cuh -- shared device helpers: control block, memory-order primitives,
// 128-bit streaming loads/stores and the fp32 apply arithmetic.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/dssp_ps.h"

namespace dssp {

// Device control block of one server (lives in the server GPU's HBM).
struct Ctrl {
  ps_gate_state gate;          // policy tables + version / rejected counters
  uint32_t arrive;             // last-CTA election counter of the apply kernel
  uint32_t bad;                // per-CTA flag counts riding on the arrival (8-aligned pair)
  int32_t cur;                 // which of the two weight buffers is current
  int32_t status;              // result of the last op (enum ps_status)
  int32_t applied;
  int32_t granted;
  uint64_t released;
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// System scope (peer GPUs over NVLink, other processes through CUDA IPC).
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Fence-based release to peers: one fence.sc.sys, then plain relaxed stores.
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Arrival at a GPU-wide election: releases this thread's (and, through the
// preceding bar.sync, its CTA's) writes; the winner acquires everyone's.
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu_u64(unsigned long long* p,
                                                                      unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu_u32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int ld_volatile_s32_(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}
// System scope: also observed by stream memory operations (cuStreamWaitValue32)
__device__ __forceinline__ void st_release_u32_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Streaming 128-bit accesses: read-once operands skip L1 allocation.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// Read-only 128-bit loads that a warp repeats many times in one kernel (the
// replay's resident update slices): kept in L1, so the repeats are L1 hits.
__device__ __forceinline__ float4 ld_keep(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// Predicated forms (no branch): the load leaves +0 when p is false; the
// store does nothing.
__device__ __forceinline__ float4 ld_keep_if(bool p, const float4* ptr) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q ld.global.nc.L1::evict_last.v4.f32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w) : "l"(ptr), "r"((int)p));
  return v;
}
__device__ __forceinline__ void st_f4_if(bool p, float4* ptr, const float4& v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t"
               "@q st.global.v4.f32 [%1], {%2,%3,%4,%5};\n\t}"
               :: "r"((int)p), "l"(ptr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ld_f4(const float4* p) { return *p; }
__device__ __forceinline__ void st_f4(float4* p, const float4& v) { *p = v; }

__device__ __forceinline__ bool nonfinite(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}
__device__ __forceinline__ bool nonfinite4(const float4& v) {
  return nonfinite(v.x) | nonfinite(v.y) | nonfinite(v.z) | nonfinite(v.w);
}

// server.py:37 in fp32: a rounded multiply, then a rounded subtract (no FMA).
__device__ __forceinline__ float apply1(float w, float lr, float g) {
  return __fsub_rn(w, __fmul_rn(lr, g));
}
__device__ __forceinline__ float4 apply4(const float4& w, float lr, const float4& g) {
  return make_float4(apply1(w.x, lr, g.x), apply1(w.y, lr, g.y), apply1(w.z, lr, g.z),
                     apply1(w.w, lr, g.w));
}

}  // namespace dssp
