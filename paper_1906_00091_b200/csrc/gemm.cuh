// GEMM epilogues shared by the SIMT fallback and the tcgen05 kernels.
#pragma once

#include "common.cuh"

namespace dlrm {

enum EpiMode : int {
  EPI_BIAS_ACT = 0,  // Y = act(acc + bias[n]); zero pad columns [N, pad_n)
  EPI_MASK = 1,      // dX = acc * (mask[m, n] > 0)   (mask may be NULL)
  EPI_PARTIAL = 2,   // part[z][m][n] = acc             (split-K partials)
};

struct GemmEpilogue {
  int mode;
  int act;
  float* out;
  int64_t ldo;
  const float* bias;
  const float* mask;
  int64_t ldm;
  int64_t pad_n;
  int64_t M;    // for EPI_PARTIAL slab stride
  int vec = 0;  // 1: out/bias/mask rows are 16-byte aligned (float4 epilogue)
};

__device__ __forceinline__ void apply_epilogue(const GemmEpilogue& ep, int64_t m,
                                               int64_t n, int64_t N, float acc,
                                               int z) {
  if (ep.mode == EPI_BIAS_ACT) {
    if (n < N) {
      float v = acc + ep.bias[n];
      if (ep.act == DLRM_ACT_RELU) v = fmaxf(v, 0.f);
      ep.out[m * ep.ldo + n] = v;
    } else if (n < ep.pad_n) {
      ep.out[m * ep.ldo + n] = 0.f;
    }
  } else if (ep.mode == EPI_MASK) {
    if (n < N) {
      float v = acc;
      if (ep.mask) v = acc * (ep.mask[m * ep.ldm + n] > 0.f ? 1.f : 0.f);
      ep.out[m * ep.ldo + n] = v;
    }
  } else {
    if (n < N) ep.out[(int64_t(z) * ep.M + m) * N + n] = acc;
  }
}

// Four consecutive columns n..n+3 of row m (vector path when aligned and
// fully inside [0, N); otherwise per element).
__device__ __forceinline__ void apply_epilogue4(const GemmEpilogue& ep, int64_t m,
                                                int64_t n, int64_t N, float4 v, int z) {
  if (ep.vec && n + 3 < N) {
    if (ep.mode == EPI_BIAS_ACT) {
      const float4 b = *reinterpret_cast<const float4*>(ep.bias + n);
      v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
      if (ep.act == DLRM_ACT_RELU) {
        v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f);
        v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
      }
      *reinterpret_cast<float4*>(ep.out + m * ep.ldo + n) = v;
    } else if (ep.mode == EPI_MASK) {
      if (ep.mask) {
        const float4 k = *reinterpret_cast<const float4*>(ep.mask + m * ep.ldm + n);
        v.x *= k.x > 0.f ? 1.f : 0.f; v.y *= k.y > 0.f ? 1.f : 0.f;
        v.z *= k.z > 0.f ? 1.f : 0.f; v.w *= k.w > 0.f ? 1.f : 0.f;
      }
      *reinterpret_cast<float4*>(ep.out + m * ep.ldo + n) = v;
    } else {
      *reinterpret_cast<float4*>(ep.out + (int64_t(z) * ep.M + m) * N + n) = v;
    }
    return;
  }
  apply_epilogue(ep, m, n, N, v.x, z);
  apply_epilogue(ep, m, n + 1, N, v.y, z);
  apply_epilogue(ep, m, n + 2, N, v.z, z);
  apply_epilogue(ep, m, n + 3, N, v.w, z);
}

int gemm_simt(const float* a, int64_t a_outer, int64_t a_k, const float* b,
              int64_t b_outer, int64_t b_k, int64_t M, int64_t N, int64_t K,
              int splits, const GemmEpilogue& ep, int64_t n_grid,
              cudaStream_t s, int* used_splits = nullptr);

int colreduce(const float* X, int64_t ldx, const float* scale, int64_t R,
              int64_t C, float* out, float* upd, const Upd& u,
              const int32_t* err_flag, float* ws, size_t ws_floats,
              cudaStream_t s);

int splitk_reduce(const float* part, int64_t M, int64_t N, int splits,
                  float* dW, int64_t lddw, float* Wu, int64_t ldw, const Upd& u,
                  const int32_t* err_flag, cudaStream_t s);

}  // namespace dlrm
