// Shared helpers for libdlrmb200: error plumbing, launch accounting, small
// device utilities.  Every exported entry point returns 0 / 1 (invalid
// argument) / 2 (CUDA error) and leaves a thread-local message.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <string>
#include <utility>

#include "dlrm_b200.h"

namespace dlrm {

void set_error(const std::string& msg);
void count_launch(int n = 1);

inline cudaStream_t as_stream(dlrm_stream_t s) {
  return reinterpret_cast<cudaStream_t>(s);
}

bool debug_sync();

// Launch-site check: captures the launch error (never synchronises, except
// with DLRM_DEBUG_SYNC=1 set in the environment, for debugging).
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug_sync()) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return 2;
  }
  count_launch();
  return 0;
}

#define DLRM_REQUIRE(cond, msg)          \
  do {                                   \
    if (!(cond)) {                       \
      ::dlrm::set_error(msg);            \
      return 1;                          \
    }                                    \
  } while (0)

#define DLRM_CUDA(call)                                                    \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) {                                               \
      ::dlrm::set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
      return 2;                                                            \
    }                                                                      \
  } while (0)

constexpr int kNumSMs = 148;

// Programmatic dependent launch (PDL).  Every kernel of the library is
// launched with programmatic stream serialization allowed, and starts with
// pdl_entry(): it lets the NEXT kernel in the stream be scheduled as soon as
// all of this grid's CTAs are resident (griddepcontrol.launch_dependents),
// then waits for the PREVIOUS grid to complete and flush its memory
// (griddepcontrol.wait) before touching any data.  The next kernel's launch
// latency and prologue therefore overlap this kernel's tail.  Kernels whose
// prologue does not read dependent data (tc_gemm: barrier init, TMEM alloc,
// tensor-map prefetch) call pdl_trigger() / pdl_wait() separately.
// DLRM_PDL=0 in the environment launches without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_entry() {
  pdl_trigger();
  pdl_wait();
}

bool pdl_enabled();

// ---- parameter updates (dlrm_update, see the header) ----------------------
struct Upd {
  int32_t kind;
  float lr;
  float eps;
  int64_t delta;  // accumulator = parameter + delta (floats), Adagrad only
};

inline Upd sgd_rule(float lr) { return Upd{DLRM_UPD_SGD, lr, 0.f, 0}; }
inline Upd upd_rule(const dlrm_update* u) { return Upd{u->kind, u->lr, u->eps, u->accum_delta}; }

// new value of parameter w (stored at p) for gradient g; Adagrad also
// updates the accumulator at p + delta
__device__ __forceinline__ float upd_apply(const Upd& u, float* p, float w, float g) {
  if (u.kind == DLRM_UPD_ADAGRAD) {
    float* a = p + u.delta;
    const float G = __fadd_rn(*a, __fmul_rn(g, g));
    *a = G;
    return __fsub_rn(w, __fdiv_rn(__fmul_rn(u.lr, g), __fadd_rn(__fsqrt_rn(G), u.eps)));
  }
  return __fsub_rn(w, __fmul_rn(u.lr, g));
}

__device__ __forceinline__ float4 upd_apply4(const Upd& u, float* p, float4 w, float4 g) {
  if (u.kind == DLRM_UPD_ADAGRAD) {
    float4* ap = reinterpret_cast<float4*>(p + u.delta);
    float4 a = *ap;
    a.x = __fadd_rn(a.x, __fmul_rn(g.x, g.x));
    a.y = __fadd_rn(a.y, __fmul_rn(g.y, g.y));
    a.z = __fadd_rn(a.z, __fmul_rn(g.z, g.z));
    a.w = __fadd_rn(a.w, __fmul_rn(g.w, g.w));
    *ap = a;
    return make_float4(
        __fsub_rn(w.x, __fdiv_rn(__fmul_rn(u.lr, g.x), __fadd_rn(__fsqrt_rn(a.x), u.eps))),
        __fsub_rn(w.y, __fdiv_rn(__fmul_rn(u.lr, g.y), __fadd_rn(__fsqrt_rn(a.y), u.eps))),
        __fsub_rn(w.z, __fdiv_rn(__fmul_rn(u.lr, g.z), __fadd_rn(__fsqrt_rn(a.z), u.eps))),
        __fsub_rn(w.w, __fdiv_rn(__fmul_rn(u.lr, g.w), __fadd_rn(__fsqrt_rn(a.w), u.eps))));
  }
  return make_float4(__fsub_rn(w.x, __fmul_rn(u.lr, g.x)), __fsub_rn(w.y, __fmul_rn(u.lr, g.y)),
                     __fsub_rn(w.z, __fmul_rn(u.lr, g.z)), __fsub_rn(w.w, __fmul_rn(u.lr, g.w)));
}

// cp.async helpers (16 B per lane, zero fill when !ok)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool ok) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = ok ? 16 : 0;  // src-size 0 -> zero fill
#ifndef DLRM_CP_CA
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n)
               : "memory");
#else
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n)
               : "memory");
#endif
}
// the same through L1 (cp.async.ca): repeated rows hit in L1
__device__ __forceinline__ void cp_async16_l1(void* smem, const void* gmem, bool ok) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = ok ? 16 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) {
  return (a + b - 1) / b;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Tables passed by value as a kernel parameter (CUDA 12.1+ allows up to
// 32 KB of parameters; 128 x 64 B = 8 KB here).
struct TableSet {
  dlrm_table_desc t[DLRM_MAX_TABLES];
  int64_t cap_base[DLRM_MAX_TABLES + 1];  // prefix of capacities
  int32_t nt;
};

struct FeatureSet {
  const float* feat[DLRM_MAX_FEATURES];
  int64_t stride[DLRM_MAX_FEATURES];
};

struct GradFeatureSet {
  float* feat[DLRM_MAX_FEATURES];
  int64_t stride[DLRM_MAX_FEATURES];
};

}  // namespace dlrm
