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
  int64_t M;  // for EPI_PARTIAL slab stride
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

int gemm_simt(const float* a, int64_t a_outer, int64_t a_k, const float* b,
              int64_t b_outer, int64_t b_k, int64_t M, int64_t N, int64_t K,
              int splits, const GemmEpilogue& ep, int64_t n_grid,
              cudaStream_t s, int* used_splits = nullptr);

int colreduce(const float* X, int64_t ldx, const float* scale, int64_t R,
              int64_t C, float* out, float* upd, float lr,
              const int32_t* err_flag, float* ws, size_t ws_floats,
              cudaStream_t s);

int splitk_reduce(const float* part, int64_t M, int64_t N, int splits,
                  float* dW, int64_t lddw, float* Wu, int64_t ldw, float lr,
                  const int32_t* err_flag, cudaStream_t s);

}  // namespace dlrm
