// C-ABI entry points for the MLP layers: forward (bias + activation fused),
// data gradient (ReLU mask fused), weight/bias gradients (split-K with a
// fixed-order reduction, SGD fused).  Shapes the tcgen05 path accepts go
// there (gemm_tc.cu); everything else runs on the SIMT kernels.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_tc.cuh"

namespace dlrm {
namespace {

int choose_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(N, 64) * ceil_div(K, 64);
  int64_t s = ceil_div(2 * kNumSMs, tiles);
  const int64_t cap = M / 256 > 1 ? M / 256 : 1;
  if (s > cap) s = cap;
  if (s > 64) s = 64;
  return int(s < 1 ? 1 : s);
}

size_t colreduce_ws_floats(int64_t R, int64_t C) {
  return size_t(ceil_div(R, 64) + 1) * size_t(C);
}

// ---------------------------------------------------------------------------
// Weight + bias gradient of a NARROW layer input (K <= 32, e.g. the 13 dense
// features): dW[n][k] = sum_m gZ[m][n] X[m][k], db[n] = sum_m gZ[m][n].  The
// batch is cut into S row slabs; thread n of a (column block, slab) CTA
// keeps the K + 1 sums of column n over its slab in registers (X rows staged
// in shared memory, gZ rows read coalesced), then a second kernel adds the
// slab partials in slab order and applies the update.  Deterministic; both
// GEMM paths waste >= half their tile on such a shape (measured 37-40 us at
// 2048 x 512 x 13 vs a few us here).
constexpr int kSkinnyRows = 64;  // X rows staged per batch

int skinny_slabs(int64_t M, int64_t N) {
  const int64_t cb = ceil_div(N, 128);
  int64_t s = ceil_div(kNumSMs, cb);
  const int64_t cap = ceil_div(M, 32);
  if (s > cap) s = cap;
  return int(s < 1 ? 1 : s);
}

int skinny_v_slabs(int64_t M, int64_t N);

// DLRM_SKINNY_V=0: the scalar narrow-input kernels only (A/B switch)
bool skinny_v_enabled() {
  static const bool on = !getenv("DLRM_SKINNY_V") || atoi(getenv("DLRM_SKINNY_V")) != 0;
  return on;
}

size_t skinny_ws_floats(int64_t M, int64_t N, int64_t K) {
  const int km = K <= 16 ? 16 : 32;
  const int64_t s = std::max<int64_t>(skinny_slabs(M, N), skinny_v_slabs(M, N));
  return size_t(s) * size_t(N) * size_t(km + 1);
}

template <int KM>
__global__ void __launch_bounds__(128)
skinny_wgrad_partial_kernel(const float* __restrict__ gZ, int64_t ldg,
                            const float* __restrict__ X, int64_t ldx, int64_t M, int64_t N,
                            int K, int64_t rows_per_slab, float* __restrict__ part) {
  pdl_entry();
  __shared__ float xs[kSkinnyRows][KM + 1];
  const int64_t n = int64_t(blockIdx.x) * 128 + threadIdx.x;
  const int64_t m0 = int64_t(blockIdx.y) * rows_per_slab;
  const int64_t m1 = m0 + rows_per_slab < M ? m0 + rows_per_slab : M;
  float acc[KM + 1];
#pragma unroll
  for (int k = 0; k <= KM; ++k) acc[k] = 0.f;
  for (int64_t mb = m0; mb < m1; mb += kSkinnyRows) {
    const int cnt = int(m1 - mb < kSkinnyRows ? m1 - mb : kSkinnyRows);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * KM; e += 128) {
      const int r = e / KM, k = e - r * KM;
      xs[r][k] = k < K ? __ldg(X + (mb + r) * ldx + k) : 0.f;
    }
    __syncthreads();
    if (n < N) {
#pragma unroll 8
      for (int r = 0; r < cnt; ++r) {
        const float g = __ldg(gZ + (mb + r) * ldg + n);
#pragma unroll
        for (int k = 0; k < KM; ++k) acc[k] = fmaf(g, xs[r][k], acc[k]);
        acc[KM] += g;
      }
    }
  }
  if (n < N) {
    float* p = part + (int64_t(blockIdx.y) * N + n) * (KM + 1);
#pragma unroll
    for (int k = 0; k <= KM; ++k) p[k] = acc[k];
  }
}

template <int KM>
__global__ void __launch_bounds__(256)
skinny_wgrad_final_kernel(const float* __restrict__ part, int S, int64_t N, int K,
                          float* dW, int64_t lddw, float* Wu, int64_t ldw, float* db,
                          float* bu, Upd u, const int32_t* err_flag) {
  pdl_entry();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // n * (KM + 1) + k
  if (e >= N * (KM + 1)) return;
  const int64_t n = e / (KM + 1);
  const int k = int(e - n * (KM + 1));
  if (k < KM && k >= K) return;
  float t = 0.f;  // slabs in order, 8 loads in flight
  const int64_t stride = N * (KM + 1);
  int sl = 0;
  for (; sl + 8 <= S; sl += 8) {
    float q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = part[int64_t(sl + j) * stride + e];
#pragma unroll
    for (int j = 0; j < 8; ++j) t += q[j];
  }
  for (; sl < S; ++sl) t += part[int64_t(sl) * stride + e];
  const bool upd = !(err_flag && *err_flag);
  if (k < KM) {
    if (dW) dW[n * lddw + k] = t;
    if (Wu && upd) {
      float* w = Wu + n * ldw + k;
      *w = upd_apply(u, w, *w, t);
    }
  } else {
    if (db) db[n] = t;
    if (bu && upd) bu[n] = upd_apply(u, bu + n, bu[n], t);
  }
}

// ---- vector variant (gZ rows 16-byte aligned): 512 threads per CTA = four
// row phases x 128 column threads of 4 columns each (float4 gZ loads, four
// rows unrolled: 64 KB of loads in flight per SM, where the scalar kernel
// above kept 4 KB and ran latency-bound at 0.75 TB/s at c4's 32768 x 512 x
// 13).  One CTA per (512-column block, slab), one slab per SM; the four
// phases are added in phase order in shared memory, the slab partials by
// skinny_wgrad_final4_kernel (a warp per output, fixed-order tree).
constexpr int kSkVCols = 512, kSkVPhases = 4;
#ifndef DLRM_SKV_U
#define DLRM_SKV_U 8
#endif
#ifndef DLRM_SKV_ROWS
#define DLRM_SKV_ROWS 128
#endif
constexpr int kSkVU = DLRM_SKV_U;        // gZ rows in flight per thread
constexpr int kSkVRows = DLRM_SKV_ROWS;  // X rows staged per chunk

int skinny_v_slabs(int64_t M, int64_t N) {
  const int64_t cb = ceil_div(N, kSkVCols);
  int64_t s = ceil_div(kNumSMs, cb);
  const int64_t cap = ceil_div(M, kSkinnyRows);
  if (s > cap) s = cap;
  return int(s < 1 ? 1 : s);
}

template <int KM>
__global__ void __launch_bounds__(128 * kSkVPhases, 1)
skinny_wgrad_partial4_kernel(const float* __restrict__ gZ, int64_t ldg,
                             const float* __restrict__ X, int64_t ldx, int64_t M, int64_t N,
                             int K, int64_t rows_per_slab, float* __restrict__ part) {
  pdl_entry();
  extern __shared__ float sk_smem[];
  float* xs = sk_smem;                               // [kSkVRows][KM + 1]
  float* red = sk_smem + kSkVRows * (KM + 1);        // [128][4 (KM + 1)]
  const int ph = threadIdx.x >> 7, ct = threadIdx.x & 127;
  const int64_t n = int64_t(blockIdx.x) * kSkVCols + 4 * ct;
  const int64_t m0 = int64_t(blockIdx.y) * rows_per_slab;
  const int64_t m1 = m0 + rows_per_slab < M ? m0 + rows_per_slab : M;
  const bool full = n + 3 < N;
  float acc[4][KM + 1];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int k = 0; k <= KM; ++k) acc[j][k] = 0.f;
  for (int64_t mb = m0; mb < m1; mb += kSkVRows) {
    const int cnt = int(m1 - mb < kSkVRows ? m1 - mb : kSkVRows);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * KM; e += 128 * kSkVPhases) {
      const int r = e / KM, k = e - r * KM;
      xs[r * (KM + 1) + k] = k < K ? __ldg(X + (mb + r) * ldx + k) : 0.f;
    }
    __syncthreads();
    if (n < N) {
      // rows ph, ph + 4, ... of the chunk; four loads issued before use
      for (int r0 = ph; r0 < cnt; r0 += kSkVU * kSkVPhases) {
        float4 g[kSkVU];
#pragma unroll
        for (int u = 0; u < kSkVU; ++u) {
          const int r = r0 + u * kSkVPhases;
          const float* src = gZ + (mb + (r < cnt ? r : 0)) * ldg + n;
          if (r >= cnt) {
            g[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else if (full) {
            g[u] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            g[u].x = __ldg(src);
            g[u].y = n + 1 < N ? __ldg(src + 1) : 0.f;
            g[u].z = n + 2 < N ? __ldg(src + 2) : 0.f;
            g[u].w = 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < kSkVU; ++u) {
          const int r = r0 + u * kSkVPhases;
          if (r >= cnt) break;
          const float* xr = xs + r * (KM + 1);
          const float gv[4] = {g[u].x, g[u].y, g[u].z, g[u].w};
#pragma unroll
          for (int k = 0; k < KM; ++k) {
            const float xv = xr[k];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j][k] = fmaf(gv[j], xv, acc[j][k]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[j][KM] += gv[j];
        }
      }
    }
  }
  // phases 3, 2, 1 hand their sums to phase 0 in turn (fixed order)
  for (int p = kSkVPhases - 1; p >= 1; --p) {
    __syncthreads();
    if (ph == p) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k <= KM; ++k) red[(j * (KM + 1) + k) * 128 + ct] = acc[j][k];
    }
    __syncthreads();
    if (ph == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int k = 0; k <= KM; ++k) acc[j][k] += red[(j * (KM + 1) + k) * 128 + ct];
    }
  }
  if (ph == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (n + j >= N) break;
      float* p = part + (int64_t(blockIdx.y) * N + n + j) * (KM + 1);
#pragma unroll
      for (int k = 0; k <= KM; ++k) p[k] = acc[j][k];
    }
  }
}

// dW / db from the slab partials: one warp per output (lane l adds slabs
// l, l + 32, ... in order, then an xor-shuffle tree), then the update
template <int KM>
__global__ void __launch_bounds__(256)
skinny_wgrad_final4_kernel(const float* __restrict__ part, int S, int64_t N, int K, float* dW,
                           int64_t lddw, float* Wu, int64_t ldw, float* db, float* bu, Upd u,
                           const int32_t* err_flag) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int64_t e = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // n * (KM + 1) + k
  if (e >= N * (KM + 1)) return;
  const int64_t n = e / (KM + 1);
  const int k = int(e - n * (KM + 1));
  if (k < KM && k >= K) return;
  const int64_t stride = N * (KM + 1);
  float t = 0.f;
  for (int sl = lane; sl < S; sl += 32) t += part[int64_t(sl) * stride + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane != 0) return;
  const bool upd = !(err_flag && *err_flag);
  if (k < KM) {
    if (dW) dW[n * lddw + k] = t;
    if (Wu && upd) {
      float* w = Wu + n * ldw + k;
      *w = upd_apply(u, w, *w, t);
    }
  } else {
    if (db) db[n] = t;
    if (bu && upd) bu[n] = upd_apply(u, bu + n, bu[n], t);
  }
}

template <int KM>
int skinny_wgrad4(const float* gZ, int64_t ldg, const float* X, int64_t ldx, int64_t M, int64_t N,
                  int64_t K, float* dW, int64_t lddw, float* db, float* W_upd, int64_t ldw,
                  float* b_upd, const Upd& u, const int32_t* err_flag, float* ws,
                  cudaStream_t s) {
  const int S = skinny_v_slabs(M, N);
  const int64_t rows = ceil_div(M, S);
  auto kp = skinny_wgrad_partial4_kernel<KM>;
  const size_t smem = size_t(kSkVRows * (KM + 1) + 128 * 4 * (KM + 1)) * 4;
  static bool attr = false;
  if (!attr) {
    DLRM_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  launch(kp, dim3(unsigned(ceil_div(N, kSkVCols)), unsigned(S)), 128 * kSkVPhases, smem, s, gZ,
         ldg, X, ldx, M, N, int(K), rows, ws);
  if (int rc = check_launch("skinny_wgrad_partial4_kernel")) return rc;
  launch(skinny_wgrad_final4_kernel<KM>, unsigned(ceil_div(N * (KM + 1) * 32, 256)), 256, 0, s,
         ws, S, N, int(K), dW, lddw, W_upd, ldw, db, b_upd, u, err_flag);
  return check_launch("skinny_wgrad_final4_kernel");
}

// ---- forward of a narrow input (K <= 16): Y = act(X W^T + b), padded
// columns zero.  Thread (phase, ct) of a CTA owns output columns
// 4ct..4ct+3 of a 512-column block, with their 4 x 16 weights and bias in
// registers, and makes rows phase, phase + 2, ... of its row range: per row
// four float4 reads of the staged X row (broadcast) and one float4 store.
// (The tensor-core kernel spends a whole 32-deep k-block per 13 inputs and is
// bound by its epilogue: 36 us at 32768 x 512 x 13 for 64 MB of output;
// weights read from shared memory per row made this kernel shared-memory
// bound at 30 us; this one takes 27.7 us, issue-bound at 16 warps per SM —
// three CTAs per SM spill and take 41 us.)
constexpr int kSkFwdK = 16;

__global__ void __launch_bounds__(256)
skinny_fwd_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ W,
                  int64_t ldw, const float* __restrict__ b, float* __restrict__ Y, int64_t ldy,
                  int64_t M, int64_t N, int K, int64_t ng, int act, int64_t rows_per_cta) {
  pdl_entry();
  __shared__ __align__(16) float xs[kSkinnyRows][kSkFwdK];
  __shared__ float ws[kSkVCols][kSkFwdK + 1];  // the block's weight rows, coalesced
  const int ph = threadIdx.x >> 7, ct = threadIdx.x & 127;
  const int64_t c0 = int64_t(blockIdx.x) * kSkVCols;
  const int64_t n = c0 + 4 * ct;
  for (int e = threadIdx.x; e < kSkVCols * kSkFwdK; e += 256) {
    const int c = e / kSkFwdK, k = e - c * kSkFwdK;
    ws[c][k] = (c0 + c < N && k < K) ? __ldg(W + (c0 + c) * ldw + k) : 0.f;
  }
  __syncthreads();
  float w[4][kSkFwdK];
  float bias[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bias[j] = n + j < N ? __ldg(b + n + j) : 0.f;
#pragma unroll
    for (int k = 0; k < kSkFwdK; ++k) w[j][k] = ws[4 * ct + j][k];
  }
  const int64_t m0 = int64_t(blockIdx.y) * rows_per_cta;
  const int64_t m1 = m0 + rows_per_cta < M ? m0 + rows_per_cta : M;
  for (int64_t mb = m0; mb < m1; mb += kSkinnyRows) {
    const int cnt = int(m1 - mb < kSkinnyRows ? m1 - mb : kSkinnyRows);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * kSkFwdK; e += 256) {
      const int r = e / kSkFwdK, k = e - r * kSkFwdK;
      xs[r][k] = k < K ? __ldg(X + (mb + r) * ldx + k) : 0.f;
    }
    __syncthreads();
    if (n >= ng) continue;
    for (int r = ph; r < cnt; r += 2) {
      float x[kSkFwdK];
#pragma unroll
      for (int q = 0; q < kSkFwdK / 4; ++q) {
        const float4 v = *reinterpret_cast<const float4*>(&xs[r][4 * q]);
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
      }
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float a = 0.f;
#pragma unroll
        for (int k = 0; k < kSkFwdK; ++k) a = fmaf(x[k], w[j][k], a);
        float v = a + bias[j];
        if (act == DLRM_ACT_RELU) v = fmaxf(v, 0.f);
        o[j] = n + j < N ? v : 0.f;  // columns >= N are padding
      }
      float* y = Y + (mb + r) * ldy + n;
      if (n + 3 < ng) {
        *reinterpret_cast<float4*>(y) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
        y[0] = o[0];
        if (n + 1 < ng) y[1] = o[1];
        if (n + 2 < ng) y[2] = o[2];
      }
    }
  }
}

int skinny_fwd(const float* X, int64_t ldx, const float* W, int64_t ldw, const float* b,
               float* Y, int64_t ldy, int64_t M, int64_t N, int64_t K, int64_t ng, int act,
               cudaStream_t s) {
  const int64_t cb = ceil_div(ng, kSkVCols);
  const int64_t ctas = ceil_div(2 * kNumSMs, cb);
  int64_t rows = ceil_div(M, ctas);
  rows = rows < 64 ? 64 : rows;  // the weight staging is amortised over >= 64 rows
  launch(skinny_fwd_kernel, dim3(unsigned(cb), unsigned(ceil_div(M, rows))), 256, 0, s, X, ldx,
         W, ldw, b, Y, ldy, M, N, int(K), ng, act, rows);
  return check_launch("skinny_fwd_kernel");
}

template <int KM>
int skinny_wgrad(const float* gZ, int64_t ldg, const float* X, int64_t ldx, int64_t M, int64_t N,
                 int64_t K, float* dW, int64_t lddw, float* db, float* W_upd, int64_t ldw,
                 float* b_upd, const Upd& u, const int32_t* err_flag, float* ws,
                 cudaStream_t s) {
  // (K <= 16: the four-column accumulators of K + 1 sums fit the registers
  // of a 512-thread CTA; 17..32 inputs stay on the scalar kernel)
  // (and long batches: at M = 2048 the scalar kernel is faster, 12.7 vs 17.7 us)
  if (KM == 16 && M >= 8192 && ldg % 4 == 0 && (reinterpret_cast<uintptr_t>(gZ) % 16) == 0 &&
      skinny_v_enabled())
    return skinny_wgrad4<KM>(gZ, ldg, X, ldx, M, N, K, dW, lddw, db, W_upd, ldw, b_upd, u,
                             err_flag, ws, s);
  const int S = skinny_slabs(M, N);
  const int64_t rows = ceil_div(M, S);
  launch(skinny_wgrad_partial_kernel<KM>, dim3(unsigned(ceil_div(N, 128)), unsigned(S)), 128, 0,
         s, gZ, ldg, X, ldx, M, N, int(K), rows, ws);
  if (int rc = check_launch("skinny_wgrad_partial_kernel")) return rc;
  launch(skinny_wgrad_final_kernel<KM>, unsigned(ceil_div(N * (KM + 1), 256)), 256, 0, s, ws,
         S, N, int(K), dW, lddw, W_upd, ldw, db, b_upd, u, err_flag);
  return check_launch("skinny_wgrad_final_kernel");
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

namespace dlrm {
namespace {
// N = 1 layer (the top MLP's last, identity layer): one warp per row with
// EXACTLY the loss head's dot order (head.cu bce_head_kernel /
// head_fused_kernel: lane l folds float4 chunks l, l+32, ... with fmaf, then
// an xor-shuffle tree), so mlp_forward's logits and dlrm_forward's
// probabilities are bitwise those of the fused training step.
__global__ void __launch_bounds__(256)
linear_n1_kernel(const float* __restrict__ X, int64_t ldx, const float* __restrict__ w,
                 const float* __restrict__ b, float* __restrict__ Y, int64_t ldy, int64_t M,
                 int64_t K, int64_t ng, int act) {
  pdl_entry();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t m = int64_t(blockIdx.x) * 8 + warp;
  if (m >= M) return;
  const float* a = X + m * ldx;
  float acc = 0.f;
  if ((K % 4) == 0 && (ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(X) % 16) == 0 &&
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
  float z = acc + (b ? b[0] : 0.f);
  if (act == DLRM_ACT_RELU) z = fmaxf(z, 0.f);
  for (int64_t c = lane; c < ng; c += 32) Y[m * ldy + c] = c == 0 ? z : 0.f;
}
}  // namespace
}  // namespace dlrm

namespace dlrm {
namespace {
int linear_fwd(const float* X, int64_t ldx, const float* W, const float* W_lo, int64_t ldw,
               const float* b, float* Y, int64_t ldy, int64_t M, int64_t N, int64_t K,
               int64_t pad_n, int32_t act, dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 0 && N >= 1 && K >= 1 && ldx >= K && ldw >= K && ldy >= N,
               "bad linear_fwd shape");
  DLRM_REQUIRE(act == DLRM_ACT_IDENTITY || act == DLRM_ACT_RELU, "bad activation");
  if (M == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const int64_t ng = pad_n > N ? pad_n : N;
  if (N == 1) {
    launch(linear_n1_kernel, unsigned(ceil_div(M, 8)), 256, 0, s, X, ldx, W, b, Y, ldy, M,
           K, ng, int(act));
    return check_launch("linear_n1_kernel");
  }
  // narrow input over a long batch (c4's 32768 x 13): the SIMT kernel below;
  // at M = 2048 the tensor-core kernel is faster (6.4 vs 10.6 us)
  if (K <= kSkFwdK && M >= 8192 && b && ldy % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(Y) % 16) == 0 && skinny_v_enabled())
    return skinny_fwd(X, ldx, W, ldw, b, Y, ldy, M, N, K, ng, act, s);
  if (tc_linear_fwd_ok(X, ldx, W, ldw, Y, ldy, M, N, K, ng))
    return tc_linear_fwd(X, ldx, W, ldw, b, Y, ldy, M, N, K, ng, act, s, W_lo);
  GemmEpilogue ep{EPI_BIAS_ACT, act, Y, ldy, b, nullptr, 0, ng, M};
  return gemm_simt(X, ldx, 1, W, ldw, 1, M, N, K, 1, ep, ng, s);
}

int linear_bwd_data(const float* gZ, int64_t ldg, const float* W, const float* W_lo,
                    int64_t ldw, const float* mask, int64_t ldm, float* dX, int64_t ldx,
                    int64_t M, int64_t N, int64_t K, dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 0 && N >= 1 && K >= 1 && ldg >= N && ldw >= K && ldx >= K,
               "bad linear_bwd_data shape");
  if (M == 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (tc_linear_bwd_data_ok(gZ, ldg, W, ldw, dX, ldx, M, N, K))
    return tc_linear_bwd_data(gZ, ldg, W, ldw, mask, ldm, dX, ldx, M, N, K, s, W_lo);
  GemmEpilogue ep{EPI_MASK, 0, dX, ldx, nullptr, mask, ldm, K, M};
  // dX(M x K) = gZ(M x N) W(N x K): A(m,k') = gZ[m*ldg+k'], B(k',n') = W[k'*ldw+n']
  return gemm_simt(gZ, ldg, 1, W, 1, ldw, M, K, N, 1, ep, K, s);
}
}  // namespace
}  // namespace dlrm

extern "C" int dlrm_linear_fwd(const float* X, int64_t ldx, const float* W,
                               int64_t ldw, const float* b, float* Y,
                               int64_t ldy, int64_t M, int64_t N, int64_t K,
                               int64_t pad_n, int32_t act,
                               dlrm_stream_t stream) {
  return dlrm::linear_fwd(X, ldx, W, nullptr, ldw, b, Y, ldy, M, N, K, pad_n, act, stream);
}

extern "C" int dlrm_linear_fwd_wlo(const float* X, int64_t ldx, const float* W,
                                   const float* W_lo, int64_t ldw, const float* b, float* Y,
                                   int64_t ldy, int64_t M, int64_t N, int64_t K,
                                   int64_t pad_n, int32_t act, dlrm_stream_t stream) {
  return dlrm::linear_fwd(X, ldx, W, W_lo, ldw, b, Y, ldy, M, N, K, pad_n, act, stream);
}

extern "C" int dlrm_linear_bwd_data_wlo(const float* gZ, int64_t ldg, const float* W,
                                        const float* W_lo, int64_t ldw, const float* mask,
                                        int64_t ldm, float* dX, int64_t ldx, int64_t M,
                                        int64_t N, int64_t K, dlrm_stream_t stream) {
  return dlrm::linear_bwd_data(gZ, ldg, W, W_lo, ldw, mask, ldm, dX, ldx, M, N, K, stream);
}

extern "C" int dlrm_tf32_split_lo(const float* x, float* lo, int64_t n,
                                  dlrm_stream_t stream) {
  DLRM_REQUIRE(n >= 0, "bad split_lo size");
  return dlrm::tc_split_lo(x, lo, n, dlrm::as_stream(stream));
}

extern "C" int dlrm_linear_bwd_data(const float* gZ, int64_t ldg,
                                    const float* W, int64_t ldw,
                                    const float* mask, int64_t ldm, float* dX,
                                    int64_t ldx, int64_t M, int64_t N,
                                    int64_t K, dlrm_stream_t stream) {
  return dlrm::linear_bwd_data(gZ, ldg, W, nullptr, ldw, mask, ldm, dX, ldx, M, N, K, stream);
}

extern "C" size_t dlrm_linear_bwd_weight_workspace_size(int64_t M, int64_t N,
                                                        int64_t K) {
  // SIMT path: split-K partials + bias column-reduce partials (the tcgen05
  // path reduces inside a cluster and needs none); narrow inputs: slab partials
  const int sp = choose_splits(M, N, K);
  size_t f = size_t(sp) * N * K + colreduce_ws_floats(M, N);
  if (K <= 32 && skinny_ws_floats(M, N, K) > f) f = skinny_ws_floats(M, N, K);
  return f * sizeof(float) + 256;
}

namespace dlrm {
namespace {
int linear_bwd_weight(const float* gZ, int64_t ldg, const float* X, int64_t ldx, int64_t M,
                      int64_t N, int64_t K, float* dW, int64_t lddw, float* db, float* W_upd,
                      int64_t ldw, float* b_upd, const Upd& u, const int32_t* err_flag,
                      void* workspace, size_t ws_bytes, dlrm_stream_t stream) {
  DLRM_REQUIRE(M >= 0 && N >= 1 && K >= 1 && ldg >= N && ldx >= K,
               "bad linear_bwd_weight shape");
  cudaStream_t s = as_stream(stream);
  if (M == 0) return 0;
  if (K <= 32) {
    DLRM_REQUIRE(ws_bytes >= dlrm_linear_bwd_weight_workspace_size(M, N, K) &&
                     workspace != nullptr,
                 "linear_bwd_weight workspace too small");
    float* ws = static_cast<float*>(workspace);
    return K <= 16 ? skinny_wgrad<16>(gZ, ldg, X, ldx, M, N, K, dW, lddw, db, W_upd, ldw, b_upd,
                                      u, err_flag, ws, s)
                   : skinny_wgrad<32>(gZ, ldg, X, ldx, M, N, K, dW, lddw, db, W_upd, ldw, b_upd,
                                      u, err_flag, ws, s);
  }
  if (tc_linear_bwd_weight_ok(gZ, ldg, X, ldx, M, N, K))
    return tc_linear_bwd_weight(gZ, ldg, X, ldx, M, N, K, dW, lddw, W_upd, ldw, db, b_upd,
                                u, err_flag, s);
  DLRM_REQUIRE(ws_bytes >= dlrm_linear_bwd_weight_workspace_size(M, N, K) &&
                   workspace != nullptr,
               "linear_bwd_weight workspace too small");
  float* ws = static_cast<float*>(workspace);
  const int sp = choose_splits(M, N, K);
  GemmEpilogue ep{EPI_PARTIAL, 0, ws, 0, nullptr, nullptr, 0, K, N};
  // dW(N x K) = gZ^T X: A(m',k') = gZ[k'*ldg + m'], B(k',n') = X[k'*ldx + n']
  int used = 1;
  if (int rc = gemm_simt(gZ, 1, ldg, X, 1, ldx, N, K, M, sp, ep, K, s, &used))
    return rc;
  if (int rc = splitk_reduce(ws, N, K, used, dW, lddw, W_upd, ldw, u, err_flag, s))
    return rc;
  if (db || b_upd) {
    float* cws = ws + size_t(sp) * N * K;
    return colreduce(gZ, ldg, nullptr, M, N, db, b_upd, u, err_flag, cws,
                     colreduce_ws_floats(M, N), s);
  }
  return 0;
}
}  // namespace
}  // namespace dlrm

extern "C" int dlrm_linear_bwd_weight(const float* gZ, int64_t ldg,
                                      const float* X, int64_t ldx, int64_t M,
                                      int64_t N, int64_t K, float* dW,
                                      int64_t lddw, float* db, float* W_upd,
                                      int64_t ldw, float* b_upd, float lr,
                                      const int32_t* err_flag, void* workspace,
                                      size_t ws_bytes, dlrm_stream_t stream) {
  return linear_bwd_weight(gZ, ldg, X, ldx, M, N, K, dW, lddw, db, W_upd, ldw, b_upd,
                           sgd_rule(lr), err_flag, workspace, ws_bytes, stream);
}

extern "C" int dlrm_linear_bwd_weight_upd(const float* gZ, int64_t ldg, const float* X,
                                          int64_t ldx, int64_t M, int64_t N, int64_t K,
                                          float* dW, int64_t lddw, float* db, float* W_upd,
                                          int64_t ldw, float* b_upd, const dlrm_update* upd,
                                          const int32_t* err_flag, void* workspace,
                                          size_t ws_bytes, dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(upd->eps >= 0.f, "eps must be nonnegative");
  return linear_bwd_weight(gZ, ldg, X, ldx, M, N, K, dW, lddw, db, W_upd, ldw, b_upd,
                           upd_rule(upd), err_flag, workspace, ws_bytes, stream);
}
