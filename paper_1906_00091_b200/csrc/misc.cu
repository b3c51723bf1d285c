// Library bookkeeping: thread-local error message, launch counter, build
// info, and the dense SGD kernel (ref optim.py:31-35).
#include <stdlib.h>

#include "common.cuh"

namespace dlrm {

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
bool debug_sync() {
  static const bool on = [] {
    const char* v = getenv("DLRM_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  return on;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("DLRM_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {

// p -= fl(lr * g) (SGD) or the Adagrad rule (upd_apply*): __fmul_rn /
// __fsub_rn keep nvcc from contracting to an FMA, matching numpy's rounding.
__global__ void update_dense_kernel(float* __restrict__ p, const float* __restrict__ g,
                                    int64_t n, Upd u, const int32_t* err_flag) {
  pdl_entry();
  if (err_flag && *err_flag) return;
  const int64_t n4 = n / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4* pw = reinterpret_cast<float4*>(p) + i;
    *pw = upd_apply4(u, reinterpret_cast<float*>(pw), *pw,
                     reinterpret_cast<const float4*>(g)[i]);
  }
  for (int64_t i = n4 * 4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = upd_apply(u, p + i, p[i], g[i]);
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

extern "C" const char* dlrm_last_error(void) { return g_last_error.c_str(); }

extern "C" int64_t dlrm_launch_count(void) { return g_launches.load(); }

extern "C" const char* dlrm_build_info(void) {
  return "libdlrmb200 sm_100a";
}

static int update_dense(float* p, const float* g, int64_t n, const Upd& u,
                        const int32_t* err_flag, dlrm_stream_t stream) {
  DLRM_REQUIRE(n >= 0, "negative length");
  if (n == 0) return 0;
  DLRM_REQUIRE(reinterpret_cast<uintptr_t>(p) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(g) % 16 == 0 &&
                   (u.kind != DLRM_UPD_ADAGRAD || u.delta % 4 == 0),
               "dense update needs 16-byte aligned buffers");
  const int64_t blocks = ceil_div(ceil_div(n, 4), 256);
  launch(update_dense_kernel, unsigned(blocks < 4 * kNumSMs ? blocks : 4 * kNumSMs), 256, 0,
         as_stream(stream), p, g, n, u, err_flag);
  return check_launch("update_dense_kernel");
}

extern "C" int dlrm_h2d_async(void* dst, const void* src, size_t bytes, void* wait_ev,
                              void* ev1, void* ev2, dlrm_stream_t stream) {
  DLRM_REQUIRE(dst && src, "bad h2d arguments");
  cudaStream_t s = as_stream(stream);
  if (wait_ev) DLRM_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(wait_ev), 0));
  DLRM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  if (ev1) DLRM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev1), s));
  if (ev2) DLRM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev2), s));
  return 0;
}

extern "C" int dlrm_d2d_async(void* dst, const void* src, size_t bytes, void* wait_ev, void* ev,
                              dlrm_stream_t stream) {
  DLRM_REQUIRE(dst && src, "bad d2d arguments");
  cudaStream_t s = as_stream(stream);
  if (wait_ev) DLRM_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(wait_ev), 0));
  DLRM_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  if (ev) DLRM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), s));
  return 0;
}

extern "C" int dlrm_step_result_copy(void* host_dst, const void* res, size_t res_bytes,
                                     void* prob_dst, const void* prob, size_t prob_bytes,
                                     void* ev, dlrm_stream_t stream) {
  DLRM_REQUIRE(host_dst && res, "bad result copy arguments");
  cudaStream_t s = as_stream(stream);
  DLRM_CUDA(cudaMemcpyAsync(host_dst, res, res_bytes, cudaMemcpyDeviceToHost, s));
  if (prob_dst && prob_bytes)
    DLRM_CUDA(cudaMemcpyAsync(prob_dst, prob, prob_bytes, cudaMemcpyDeviceToDevice, s));
  if (ev) DLRM_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), s));
  return 0;
}

extern "C" int dlrm_sgd_dense(float* p, const float* g, int64_t n, float lr,
                              const int32_t* err_flag, dlrm_stream_t stream) {
  return update_dense(p, g, n, sgd_rule(lr), err_flag, stream);
}

extern "C" int dlrm_update_dense(float* p, const float* g, int64_t n, const dlrm_update* upd,
                                 const int32_t* err_flag, dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(upd->eps >= 0.f, "eps must be nonnegative");
  return update_dense(p, g, n, upd_rule(upd), err_flag, stream);
}
