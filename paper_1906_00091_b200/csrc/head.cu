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

// ---------------------------------------------------------------------------
// Fused head step: forward of the N = 1 layer + BCE + logit gradient + the
// layer's backward in one pass over A.  A CTA owns HR rows; each warp takes
// HR/8 of them: z = A[m].w + b (warp reduction), sigma / loss / correct /
// g = (p - y)/n by lane 0, then dA[m] = g w (* ReLU mask) and the row's
// contribution g A[m] to dw, all while A[m] is in registers (K <= 32*4*KV).
// Per-CTA partials (dw [K], sum g, sum loss, #correct) go to the workspace in
// a fixed order; head_final reduces them in CTA order and applies the update.
constexpr int HR = 16;  // rows per CTA

template <int KV>  // float4 per lane per row: K <= 128 * KV
__global__ void __launch_bounds__(256)
head_fused_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ w,
                  const float* __restrict__ b, int64_t M, int64_t K,
                  const float* __restrict__ y, float n_total, float* prob, float* grad_z,
                  float* __restrict__ dA, int64_t ldda, int relu_mask,
                  float* __restrict__ part) {
  pdl_entry();
  __shared__ float4 s_dw[8][32 * KV];
  __shared__ float s_sc[8][3];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t kv = K / 4;
  float4 wv[KV], dw[KV];
#pragma unroll
  for (int j = 0; j < KV; ++j) {
    const int64_t c = lane + 32 * j;
    wv[j] = c < kv ? __ldg(reinterpret_cast<const float4*>(w) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    dw[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float sg = 0.f, sl = 0.f, sok = 0.f;
  for (int r = warp; r < HR; r += 8) {
    const int64_t m = int64_t(blockIdx.x) * HR + r;
    if (m >= M) break;
    const float4* a = reinterpret_cast<const float4*>(A + m * lda);
    float4 av[KV];
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      const int64_t c = lane + 32 * j;
      av[j] = c < kv ? __ldg(a + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      acc = fmaf(av[j].x, wv[j].x, acc);
      acc = fmaf(av[j].y, wv[j].y, acc);
      acc = fmaf(av[j].z, wv[j].z, acc);
      acc = fmaf(av[j].w, wv[j].w, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    float g = 0.f;
    if (lane == 0) {
      const float z = acc + b[0];
      const float yy = y[m];
      const float per = fmaxf(z, 0.f) - z * yy + log1pf(expf(-fabsf(z)));
      const float p = stable_sigmoid(z);
      if (prob) prob[m] = p;
      g = __fdiv_rn(p - yy, n_total);
      if (grad_z) grad_z[m] = g;
      sl += per;
      sok += ((p > 0.5f) == (yy > 0.5f)) ? 1.f : 0.f;
      sg += g;
    }
    g = __shfl_sync(0xffffffffu, g, 0);
    float4* da = reinterpret_cast<float4*>(dA + m * ldda);
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      const int64_t c = lane + 32 * j;
      if (c < kv) {
        float4 v = make_float4(g * wv[j].x, g * wv[j].y, g * wv[j].z, g * wv[j].w);
        if (relu_mask) {
          v.x *= av[j].x > 0.f ? 1.f : 0.f; v.y *= av[j].y > 0.f ? 1.f : 0.f;
          v.z *= av[j].z > 0.f ? 1.f : 0.f; v.w *= av[j].w > 0.f ? 1.f : 0.f;
        }
        if (dA) da[c] = v;
        dw[j].x = fmaf(g, av[j].x, dw[j].x);
        dw[j].y = fmaf(g, av[j].y, dw[j].y);
        dw[j].z = fmaf(g, av[j].z, dw[j].z);
        dw[j].w = fmaf(g, av[j].w, dw[j].w);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < KV; ++j) s_dw[warp][lane + 32 * j] = dw[j];
  if (lane == 0) { s_sc[warp][0] = sg; s_sc[warp][1] = sl; s_sc[warp][2] = sok; }
  __syncthreads();
  // CTA partial, warps summed in order: part[cta] = [dw (K) | sum g | loss | ok]
  float* pc = part + int64_t(blockIdx.x) * (K + 3);
  for (int64_t c = threadIdx.x; c < kv; c += blockDim.x) {
    float4 t = s_dw[0][c];
    for (int q = 1; q < 8; ++q) {
      const float4 u = s_dw[q][c];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    pc[4 * c] = t.x; pc[4 * c + 1] = t.y; pc[4 * c + 2] = t.z; pc[4 * c + 3] = t.w;
  }
  if (threadIdx.x < 3) {
    float t = 0.f;
    for (int q = 0; q < 8; ++q) t += s_sc[q][threadIdx.x];
    pc[K + threadIdx.x] = t;
  }
}

// dw[k] / db / stats reduced over the CTA partials in a fixed order; optional
// outputs and the fused update (skipped when *err_flag).
__global__ void __launch_bounds__(256)
head_final_kernel(const float* __restrict__ part, int64_t nparts, int64_t K, float* dw,
                  float* db, float* stats, float* w_upd, float* b_upd, Upd u,
                  const int32_t* err_flag) {
  // 32 columns per block; warp w sums partials [16w, 16w + 16) + 128 j (all
  // 16 loads of a chunk in flight before the in-order sum), then warp 0 adds
  // the 8 warp sums in order
  pdl_entry();
  __shared__ float s_t[8][33];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t c = int64_t(blockIdx.x) * 32 + lane;  // 0..K+2
  const int64_t ncol = K + 3;
  float t = 0.f;
  if (c < ncol) {
    for (int64_t i0 = 16 * warp; i0 < nparts; i0 += 128) {
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = i0 + j < nparts ? part[(i0 + j) * ncol + c] : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) t += v[j];
    }
  }
  s_t[warp][lane] = t;
  __syncthreads();
  if (warp != 0 || c >= ncol) return;
  t = s_t[0][lane];
#pragma unroll
  for (int w = 1; w < 8; ++w) t += s_t[w][lane];
  const bool upd = !(err_flag && *err_flag);
  if (c < K) {
    if (dw) dw[c] = t;
    if (w_upd && upd) w_upd[c] = upd_apply(u, w_upd + c, w_upd[c], t);
  } else if (c == K) {
    if (db) db[0] = t;
    if (b_upd && upd) b_upd[0] = upd_apply(u, b_upd, b_upd[0], t);
  } else if (stats) {
    stats[c - K - 1] = t;  // [0] loss sum, [1] correct count
  }
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

extern "C" size_t dlrm_head_step_workspace_size(int64_t M, int64_t K) {
  return size_t(ceil_div(M > 0 ? M : 1, HR)) * size_t(K + 3) * sizeof(float) + 256;
}

static int head_partials(const float* A, int64_t lda, const float* w, const float* b,
                         int64_t M, int64_t K, const float* y, float n_total, float* prob,
                         float* grad_z, float* dA, int64_t ldda, int32_t relu_mask,
                         void* workspace, size_t ws_bytes, cudaStream_t s) {
  DLRM_REQUIRE(M >= 1 && K >= 4 && K % 4 == 0 && K <= 128 * 8 && lda % 4 == 0 &&
                   (!dA || ldda % 4 == 0),
               "head_step needs K in [4, 1024], K % 4 == 0 and 16-byte rows");
  DLRM_REQUIRE(reinterpret_cast<uintptr_t>(A) % 16 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0 &&
                   (!dA || reinterpret_cast<uintptr_t>(dA) % 16 == 0),
               "head_step needs 16-byte aligned A / w / dA");
  DLRM_REQUIRE(workspace && ws_bytes >= dlrm_head_step_workspace_size(M, K),
               "head_step workspace too small");
  float* part = static_cast<float*>(workspace);
  const int64_t nb = ceil_div(M, HR);
  const int kvl = int(ceil_div(K / 4, 32));
  auto go = [&](auto kern) {
    launch(kern, unsigned(nb), 256, 0, s, A, lda, w, b, M, K, y, n_total, prob, grad_z, dA,
           ldda, relu_mask, part);
  };
  if (kvl <= 2) go(head_fused_kernel<2>);
  else if (kvl <= 4) go(head_fused_kernel<4>);
  else go(head_fused_kernel<8>);
  return check_launch("head_fused_kernel");
}

static int head_reduce(int64_t M, int64_t K, float* stats, float* dw, float* db, float* w_upd,
                       float* b_upd, const dlrm_update* upd, const int32_t* err_flag,
                       void* workspace, size_t ws_bytes, cudaStream_t s) {
  DLRM_REQUIRE(M >= 1 && K >= 4 && K <= 128 * 8, "head_step needs K in [4, 1024]");
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(workspace && ws_bytes >= dlrm_head_step_workspace_size(M, K),
               "head_step workspace too small");
  launch(head_final_kernel, unsigned(ceil_div(K + 3, 32)), 256, 0, s,
         static_cast<const float*>(workspace), ceil_div(M, HR), K, dw, db, stats, w_upd, b_upd,
         upd_rule(upd), err_flag);
  return check_launch("head_final_kernel");
}

extern "C" int dlrm_head_step(const float* A, int64_t lda, const float* w, const float* b,
                              int64_t M, int64_t K, const float* y, float n_total, float* prob,
                              float* grad_z, float* stats, float* dA, int64_t ldda,
                              int32_t relu_mask, float* dw, float* db, float* w_upd,
                              float* b_upd, const dlrm_update* upd, const int32_t* err_flag,
                              void* workspace, size_t ws_bytes, dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  cudaStream_t s = as_stream(stream);
  if (int rc = head_partials(A, lda, w, b, M, K, y, n_total, prob, grad_z, dA, ldda, relu_mask,
                             workspace, ws_bytes, s))
    return rc;
  return head_reduce(M, K, stats, dw, db, w_upd, b_upd, upd, err_flag, workspace, ws_bytes, s);
}

extern "C" int dlrm_head_step_partials(const float* A, int64_t lda, const float* w,
                                       const float* b, int64_t M, int64_t K, const float* y,
                                       float n_total, float* prob, float* grad_z, float* dA,
                                       int64_t ldda, int32_t relu_mask, void* workspace,
                                       size_t ws_bytes, dlrm_stream_t stream) {
  return head_partials(A, lda, w, b, M, K, y, n_total, prob, grad_z, dA, ldda, relu_mask,
                       workspace, ws_bytes, as_stream(stream));
}

extern "C" int dlrm_head_step_reduce(int64_t M, int64_t K, float* stats, float* dw, float* db,
                                     float* w_upd, float* b_upd, const dlrm_update* upd,
                                     const int32_t* err_flag, void* workspace, size_t ws_bytes,
                                     dlrm_stream_t stream) {
  return head_reduce(M, K, stats, dw, db, w_upd, b_upd, upd, err_flag, workspace, ws_bytes,
                     as_stream(stream));
}

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
