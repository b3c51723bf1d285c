// tcgen05 (5th-gen tensor core) GEMM path: fp32-accurate 3xTF32 with TMEM
// accumulators.  Each *_ok predicate says whether a shape/stride set is one
// the tensor-core kernels take; otherwise the SIMT path runs.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace dlrm {

// false after dlrm_gemm_mode(1): every tensor-core kernel (GEMMs and the
// interaction) is replaced by its SIMT fp32 counterpart (A/B tests)
bool tc_enabled();
// dlrm_gemm_mode: 0 default, 1 SIMT only, 2 tensor cores wherever legal
int tc_mode();

// 2D fp32 tensor map (row-major, ld_elems per row) for TMA loads of
// box_inner x box_outer boxes; swizzle 0 none, 1 128B (K-major MMA tiles),
// 2 128B with 32-byte atoms (MN-major tf32 tiles).  False if not encodable.
bool tma_encode_2d(CUtensorMap* map, const float* base, int64_t inner, int64_t outer,
                   int64_t ld_elems, int box_inner, int box_outer, int swizzle);

bool tc_linear_fwd_ok(const float* X, int64_t ldx, const float* W, int64_t ldw,
                      const float* Y, int64_t ldy, int64_t M, int64_t N,
                      int64_t K, int64_t n_grid);
// W_lo (optional): lo_tf32(W - hi(W)) in W's layout (dlrm_tf32_split_lo),
// loaded by TMA instead of being converted per tile
int tc_linear_fwd(const float* X, int64_t ldx, const float* W, int64_t ldw,
                  const float* b, float* Y, int64_t ldy, int64_t M, int64_t N,
                  int64_t K, int64_t n_grid, int act, cudaStream_t s,
                  const float* W_lo = nullptr);

bool tc_linear_bwd_data_ok(const float* gZ, int64_t ldg, const float* W,
                           int64_t ldw, const float* dX, int64_t ldx, int64_t M,
                           int64_t N, int64_t K);
int tc_linear_bwd_data(const float* gZ, int64_t ldg, const float* W,
                       int64_t ldw, const float* mask, int64_t ldm, float* dX,
                       int64_t ldx, int64_t M, int64_t N, int64_t K,
                       cudaStream_t s, const float* W_lo = nullptr);
// lo[i] = lo_tf32(x[i] - hi(x[i])): the B_lo operand the GEMM splitter would
// make, for weights reused by many GEMM tiles
int tc_split_lo(const float* x, float* lo, int64_t n, cudaStream_t s);
bool blo_enabled();

bool tc_linear_bwd_weight_ok(const float* gZ, int64_t ldg, const float* X,
                             int64_t ldx, int64_t M, int64_t N, int64_t K);
// dW / W update and the bias gradient / update in one launch (split-K
// reduced inside a thread-block cluster); needs no workspace.
int tc_linear_bwd_weight(const float* gZ, int64_t ldg, const float* X,
                         int64_t ldx, int64_t M, int64_t N, int64_t K,
                         float* dW, int64_t lddw, float* W_upd, int64_t ldw,
                         float* db, float* b_upd, const Upd& u,
                         const int32_t* err_flag, cudaStream_t s);

}  // namespace dlrm
