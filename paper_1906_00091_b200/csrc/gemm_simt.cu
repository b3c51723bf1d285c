// fp32 SIMT GEMM path for the MLP layers (generic shapes/strides) plus the
// deterministic column reductions used by the weight/bias gradients.
//
// Reference (dlrmkit, pkg/src/dlrmkit/model.py):
//   mlp_forward         142-156  z = a W^T + b ; a' = act(z)
//   mlp_backward_trace  159-180  gz = grad_a * act'(z) ; grad_a' = gz W
//   mlp_backward        191-208  dW = sum_b gz_b^T x_b ; db = sum_b gz_b
// The reference sums dW/db through exact float64 "grid components" so that
// data-parallel shards reproduce serial bits; here the batch reduction is a
// plain fp32 reduction with a FIXED split order (deterministic run to run).
//
// This file is the generic fallback used for shapes the tcgen05 kernels do
// not take (odd K/N, unaligned strides).  Tile 64x64x16, 256 threads, 4x4
// register micro-tile.
#include "common.cuh"
#include "gemm.cuh"

namespace dlrm {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

struct Operand {
  const float* p;
  int64_t s_outer;  // stride of the non-K dim
  int64_t s_k;      // stride of the K dim
};

// Load a (ROWS x BK) tile of an operand whose element (r, k) lives at
// p[r*s_outer + k*s_k] into smem laid out [BK][ROWS].
template <int ROWS>
__device__ __forceinline__ void load_tile(float (*dst)[ROWS + 4], const Operand& op,
                                          int64_t r0, int64_t k0, int64_t R,
                                          int64_t K, bool k_contig) {
  for (int e = threadIdx.x; e < ROWS * BK; e += blockDim.x) {
    int r, k;
    if (k_contig) { r = e / BK; k = e - r * BK; }
    else { k = e / ROWS; r = e - k * ROWS; }
    const int64_t gr = r0 + r, gk = k0 + k;
    dst[k][r] = (gr < R && gk < K) ? __ldg(op.p + gr * op.s_outer + gk * op.s_k) : 0.f;
  }
}

__global__ void __launch_bounds__(256)
gemm_simt_kernel(Operand A, Operand B, int64_t M, int64_t N, int64_t K,
                 int64_t k_chunk, GemmEpilogue ep) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
  const int64_t kb = int64_t(blockIdx.z) * k_chunk;
  const int64_t ke = kb + k_chunk < K ? kb + k_chunk : K;
  const bool a_kc = A.s_k == 1, b_kc = B.s_k == 1;
  float acc[4][4] = {};
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    load_tile<BM>(As, A, m0, k0, M, ke, a_kc);
    load_tile<BN>(Bs, B, n0, k0, N, ke, b_kc);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      apply_epilogue(ep, m, n, N, acc[i][j], blockIdx.z);
    }
  }
}

// Deterministic column reduction, stage 1: partial[z][c] = sum over rows of
// chunk z of scale[r] * X[r, c]  (scale == NULL -> 1), in ascending row order
// within 8 interleaved lanes then a fixed-order combine.
__global__ void __launch_bounds__(256)
colreduce_partial_kernel(const float* __restrict__ X, int64_t ldx,
                         const float* __restrict__ scale, int64_t R, int64_t C,
                         int64_t rows_per_chunk, float* __restrict__ partial) {
  __shared__ float red[8][33];
  const int cx = threadIdx.x % 32, ry = threadIdx.x / 32;
  const int64_t c = int64_t(blockIdx.x) * 32 + cx;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = r0 + rows_per_chunk < R ? r0 + rows_per_chunk : R;
  float a = 0.f;
  if (c < C) {
    for (int64_t r = r0 + ry; r < r1; r += 8) {
      const float x = __ldg(X + r * ldx + c);
      a = scale ? fmaf(__ldg(scale + r), x, a) : a + x;
    }
  }
  red[ry][cx] = a;
  __syncthreads();
  if (ry == 0 && c < C) {
    float s = red[0][cx];
#pragma unroll
    for (int i = 1; i < 8; ++i) s += red[i][cx];
    partial[int64_t(blockIdx.y) * C + c] = s;
  }
}

// stage 2: out[c] = sum_z partial[z][c] (ascending z); optional store and
// fused SGD (p -= fl(lr*g)), skipped when *err_flag.
__global__ void colreduce_final_kernel(const float* __restrict__ partial,
                                       int64_t C, int splits, float* out,
                                       float* upd, float lr,
                                       const int32_t* err_flag) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = partial[c];
  for (int z = 1; z < splits; ++z) s += partial[int64_t(z) * C + c];
  if (out) out[c] = s;
  if (upd && !(err_flag && *err_flag)) upd[c] = __fsub_rn(upd[c], __fmul_rn(lr, s));
}

// dW split-K reduction: dW[m, n] = sum_z part[z][m][n]; optional SGD.
__global__ void splitk_final_kernel(const float* __restrict__ part, int64_t M,
                                    int64_t N, int splits, float* dW,
                                    int64_t lddw, float* Wu, int64_t ldw,
                                    float lr, const int32_t* err_flag) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t m = e / N, n = e - m * N;
  float s = part[e];
  for (int z = 1; z < splits; ++z) s += part[int64_t(z) * M * N + e];
  if (dW) dW[m * lddw + n] = s;
  if (Wu && !(err_flag && *err_flag))
    Wu[m * ldw + n] = __fsub_rn(Wu[m * ldw + n], __fmul_rn(lr, s));
}

}  // namespace

int gemm_simt(const float* a, int64_t a_outer, int64_t a_k, const float* b,
              int64_t b_outer, int64_t b_k, int64_t M, int64_t N, int64_t K,
              int splits, const GemmEpilogue& ep, int64_t n_grid,
              cudaStream_t s, int* used_splits) {
  Operand A{a, a_outer, a_k}, B{b, b_outer, b_k};
  const int64_t k_chunk = ceil_div(ceil_div(K, splits), BK) * BK;
  const int64_t z = K == 0 ? 1 : ceil_div(K, k_chunk);
  if (used_splits) *used_splits = int(z);
  dim3 grid(unsigned(ceil_div(n_grid, BN)), unsigned(ceil_div(M, BM)), unsigned(z));
  gemm_simt_kernel<<<grid, 256, 0, s>>>(A, B, M, N, K, k_chunk, ep);
  return check_launch("gemm_simt_kernel");
}

int colreduce(const float* X, int64_t ldx, const float* scale, int64_t R,
              int64_t C, float* out, float* upd, float lr,
              const int32_t* err_flag, float* ws, size_t ws_floats,
              cudaStream_t s) {
  int64_t splits = ceil_div(R, 256);
  const int64_t col_blocks = ceil_div(C, 32);
  if (splits * col_blocks > 4 * kNumSMs) splits = ceil_div(4 * kNumSMs, col_blocks);
  if (splits < 1) splits = 1;
  while (splits > 1 && size_t(splits * C) > ws_floats) --splits;
  DLRM_REQUIRE(size_t(splits * C) <= ws_floats, "column-reduction workspace too small");
  const int64_t rpc = R == 0 ? 1 : ceil_div(R, splits);
  splits = R == 0 ? 1 : ceil_div(R, rpc);
  colreduce_partial_kernel<<<dim3(unsigned(col_blocks), unsigned(splits)), 256, 0, s>>>(
      X, ldx, scale, R, C, rpc, ws);
  if (int rc = check_launch("colreduce_partial_kernel")) return rc;
  colreduce_final_kernel<<<unsigned(ceil_div(C, 256)), 256, 0, s>>>(
      ws, C, int(splits), out, upd, lr, err_flag);
  return check_launch("colreduce_final_kernel");
}

int splitk_reduce(const float* part, int64_t M, int64_t N, int splits, float* dW,
                  int64_t lddw, float* Wu, int64_t ldw, float lr,
                  const int32_t* err_flag, cudaStream_t s) {
  splitk_final_kernel<<<unsigned(ceil_div(M * N, 256)), 256, 0, s>>>(
      part, M, N, splits, dW, lddw, Wu, ldw, lr, err_flag);
  return check_launch("splitk_final_kernel");
}

}  // namespace dlrm
