// Loss head: the top MLP's last (N = 1) layer fused with sigmoid, binary
// cross-entropy from logits, the logit gradient and the accuracy count; and
// its backward (dA, dw, db) with the SGD step fused.
//
// Reference (dlrmkit):
//   mlp_forward last layer  model.py:152      z = a w^T + b (identity act)
//   bce_from_logits         model.py:448-461  per = max(z,0) - z y + log1p(e^-|z|)
//                                             grad = (sigmoid(z) - y) / n
//   _sigmoid                dense.py:123-130  evaluated on the non-overflow side
//   accuracy                parallel.py:286   mean((p > .5) == (y > .5))
//   mlp_backward_trace      model.py:173-179  grad_a = gz W ; * relu'(z_prev)
#include "common.cuh"
#include "gemm.cuh"

namespace dlrm {
namespace {

__device__ __forceinline__ float stable_sigmoid(float z) {
  if (z >= 0.f) return 1.f / (1.f + expf(-z));
  const float e = expf(z);
  return e / (1.f + e);
}

// One warp per sample; block-level partials of (sum loss, #correct) written
// to part[block] in a fixed order.
__global__ void __launch_bounds__(256)
bce_head_kernel(const float* __restrict__ A, int64_t lda,
                const float* __restrict__ w, const float* __restrict__ b,
                int64_t M, int64_t K, const float* __restrict__ y,
                float n_total, float* logits, float* prob, float* grad_z,
                float* per_sample, float2* part) {
  pdl_entry();
  __shared__ float s_loss[8], s_ok[8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t m = int64_t(blockIdx.x) * 8 + warp;
  float per = 0.f, ok = 0.f;
  if (m < M) {
    const float* a = A + m * lda;
    float acc = 0.f;
    if ((K % 4) == 0 && (lda % 4) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0 &&
        (reinterpret_cast<uintptr_t>(w) % 16) == 0) {
      for (int64_t k = 4 * lane; k < K; k += 128) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(a + k));
        const float4 v = __ldg(reinterpret_cast<const float4*>(w + k));
        acc = fmaf(x.x, v.x, acc);
        acc = fmaf(x.y, v.y, acc);
        acc = fmaf(x.z, v.z, acc);
        acc = fmaf(x.w, v.w, acc);
      }
    } else {
      for (int64_t k = lane; k < K; k += 32) acc = fmaf(__ldg(a + k), __ldg(w + k), acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float z = acc + b[0];
      const float yy = y[m];
      per = fmaxf(z, 0.f) - z * yy + log1pf(expf(-fabsf(z)));
      const float p = stable_sigmoid(z);
      ok = ((p > 0.5f) == (yy > 0.5f)) ? 1.f : 0.f;
      if (logits) logits[m] = z;
      if (prob) prob[m] = p;
      if (per_sample) per_sample[m] = per;
      grad_z[m] = __fdiv_rn(p - yy, n_total);
    }
  }
  if (lane == 0) { s_loss[warp] = per; s_ok[warp] = ok; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float l = 0.f, c = 0.f;
    for (int i = 0; i < 8; ++i) { l += s_loss[i]; c += s_ok[i]; }
    part[blockIdx.x] = make_float2(l, c);
  }
}

__global__ void bce_final_kernel(const float2* __restrict__ part, int64_t nb,
                                 float* stats) {
  pdl_entry();
  __shared__ float s_l[256], s_c[256];
  float l = 0.f, c = 0.f;
  for (int64_t i = threadIdx.x; i < nb; i += 256) { l += part[i].x; c += part[i].y; }
  s_l[threadIdx.x] = l;
  s_c[threadIdx.x] = c;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s_l[threadIdx.x] += s_l[threadIdx.x + o];
      s_c[threadIdx.x] += s_c[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { stats[0] = s_l[0]; stats[1] = s_c[0]; }
}

// dA[m, k] = g[m] * w[k] * (A[m, k] > 0)
__global__ void head_dA_kernel(const float* __restrict__ A, int64_t lda,
                               const float* __restrict__ w,
                               const float* __restrict__ g, int64_t M,
                               int64_t K, float* __restrict__ dA, int64_t ldda,
                               int relu_mask) {
  pdl_entry();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * K) return;
  const int64_t m = e / K, k = e - m * K;
  const float v = g[m] * w[k];
  dA[m * ldda + k] = relu_mask ? v * (A[m * lda + k] > 0.f ? 1.f : 0.f) : v;
}

__global__ void relu_grad_kernel(const float* __restrict__ g, int64_t ldg,
                                 const float* __restrict__ a, int64_t lda,
                                 float* __restrict__ out, int64_t ldo, int64_t M,
                                 int64_t N) {
  pdl_entry();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t m = e / N, n = e - m * N;
  out[m * ldo + n] = g[m * ldg + n] * (a[m * lda + n] > 0.f ? 1.f : 0.f);
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

extern "C" int dlrm_relu_grad(const float* g, int64_t ldg, const float* act,
                              int64_t lda, float* out, int64_t ldo, int64_t M,
                              int64_t N, dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 0 && N >= 1, "bad relu_grad shape");
  if (M == 0) return 0;
  launch(relu_grad_kernel, unsigned(ceil_div(M * N, 256)), 256, 0, as_stream(stream), g, ldg, act, lda, out, ldo, M, N);
  return check_launch("relu_grad_kernel");
}

extern "C" size_t dlrm_bce_head_workspace_size(int64_t M) {
  return size_t(ceil_div(M > 0 ? M : 1, 8)) * sizeof(float2) + 256;
}

extern "C" int dlrm_bce_head(const float* A, int64_t lda, const float* w,
                             const float* b, int64_t M, int64_t K,
                             const float* y, float n_total, float* logits,
                             float* prob, float* grad_z, float* per_sample,
                             float* stats, void* workspace, size_t ws_bytes,
                             dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 1 && K >= 1 && lda >= K && grad_z && stats && y,
               "bad bce_head arguments");
  DLRM_REQUIRE(workspace && ws_bytes >= dlrm_bce_head_workspace_size(M),
               "bce_head workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t nb = ceil_div(M, 8);
  float2* part = static_cast<float2*>(workspace);
  launch(bce_head_kernel, unsigned(nb), 256, 0, s, A, lda, w, b, M, K, y, n_total,
                                                 logits, prob, grad_z, per_sample, part);
  if (int rc = check_launch("bce_head_kernel")) return rc;
  launch(bce_final_kernel, 1, 256, 0, s, part, nb, stats);
  return check_launch("bce_final_kernel");
}

static int head_bwd(const float* A, int64_t lda, const float* w, const float* g, int64_t M,
                    int64_t K, float* dA, int64_t ldda, int32_t relu_mask, float* dw, float* db,
                    float* w_upd, float* b_upd, const Upd& u, const int32_t* err_flag,
                    void* workspace, size_t ws_bytes, dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 1 && K >= 1 && lda >= K, "bad head_bwd arguments");
  cudaStream_t s = as_stream(stream);
  if (dA) {
    launch(head_dA_kernel, unsigned(ceil_div(M * K, 256)), 256, 0, s, A, lda, w, g, M, K, dA,
           ldda, relu_mask);
    if (int rc = check_launch("head_dA_kernel")) return rc;
  }
  float* ws = static_cast<float*>(workspace);
  const size_t wf = ws_bytes / sizeof(float);
  if (dw || w_upd) {
    if (int rc = colreduce(A, lda, g, M, K, dw, w_upd, u, err_flag, ws, wf, s)) return rc;
  }
  if (db || b_upd) {
    if (int rc = colreduce(g, 1, nullptr, M, 1, db, b_upd, u, err_flag, ws, wf, s)) return rc;
  }
  return 0;
}

extern "C" int dlrm_head_bwd(const float* A, int64_t lda, const float* w,
                             const float* g, int64_t M, int64_t K, float* dA,
                             int64_t ldda, int32_t relu_mask, float* dw,
                             float* db, float* w_upd,
                             float* b_upd, float lr, const int32_t* err_flag,
                             void* workspace, size_t ws_bytes,
                             dlrm_stream_t stream) {
  return head_bwd(A, lda, w, g, M, K, dA, ldda, relu_mask, dw, db, w_upd, b_upd, sgd_rule(lr),
                  err_flag, workspace, ws_bytes, stream);
}

extern "C" int dlrm_head_bwd_upd(const float* A, int64_t lda, const float* w, const float* g,
                                 int64_t M, int64_t K, float* dA, int64_t ldda,
                                 int32_t relu_mask, float* dw, float* db, float* w_upd,
                                 float* b_upd, const dlrm_update* upd,
                                 const int32_t* err_flag, void* workspace, size_t ws_bytes,
                                 dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(upd->eps >= 0.f, "eps must be nonnegative");
  return head_bwd(A, lda, w, g, M, K, dA, ldda, relu_mask, dw, db, w_upd, b_upd, upd_rule(upd),
                  err_flag, workspace, ws_bytes, stream);
}

extern "C" size_t dlrm_head_bwd_workspace_size(int64_t M, int64_t K) {
  return size_t(ceil_div(M > 0 ? M : 1, 64) + 1) * size_t(K > 1 ? K : 1) *
             sizeof(float) + 256;
}
