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
  pdl_entry();
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
  pdl_entry();
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

// Vectorised variant (C % 4 == 0, 16-byte aligned rows): a block covers 128
// columns (32 lanes x float4) and 8 row-groups; 4 independent row streams
// per thread keep 4 loads in flight.  Same fixed combine order.
__global__ void __launch_bounds__(256)
colreduce_partial4_kernel(const float* __restrict__ X, int64_t ldx,
                          const float* __restrict__ scale, int64_t R, int64_t C,
                          int64_t rows_per_chunk, float* __restrict__ partial) {
  pdl_entry();
  __shared__ float4 red[8][32];
  const int cx = threadIdx.x % 32, ry = threadIdx.x / 32;
  const int64_t c4 = int64_t(blockIdx.x) * 32 + cx;  // float4 column index
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = r0 + rows_per_chunk < R ? r0 + rows_per_chunk : R;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (4 * c4 < C) {
    const float4* Xv = reinterpret_cast<const float4*>(X);
    const int64_t ld4 = ldx / 4;
    int64_t r = r0 + ry;
    for (; r + 24 < r1; r += 32) {
      float4 v[4];
      float sc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = __ldg(Xv + (r + 8 * u) * ld4 + c4);
        sc[u] = scale ? __ldg(scale + r + 8 * u) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a.x = fmaf(sc[u], v[u].x, a.x);
        a.y = fmaf(sc[u], v[u].y, a.y);
        a.z = fmaf(sc[u], v[u].z, a.z);
        a.w = fmaf(sc[u], v[u].w, a.w);
      }
    }
    for (; r < r1; r += 8) {
      const float4 v = __ldg(Xv + r * ld4 + c4);
      const float sc = scale ? __ldg(scale + r) : 1.f;
      a.x = fmaf(sc, v.x, a.x);
      a.y = fmaf(sc, v.y, a.y);
      a.z = fmaf(sc, v.z, a.z);
      a.w = fmaf(sc, v.w, a.w);
    }
  }
  red[ry][cx] = a;
  __syncthreads();
  if (ry == 0 && 4 * c4 < C) {
    float4 t = red[0][cx];
#pragma unroll
    for (int i = 1; i < 8; ++i) {
      t.x += red[i][cx].x;
      t.y += red[i][cx].y;
      t.z += red[i][cx].z;
      t.w += red[i][cx].w;
    }
    reinterpret_cast<float4*>(partial + int64_t(blockIdx.y) * C)[c4] = t;
  }
}

// stage 2: out[c] = sum_z partial[z][c] (ascending z); optional store and
// fused update (SGD / Adagrad), skipped when *err_flag.
__global__ void colreduce_final_kernel(const float* __restrict__ partial,
                                       int64_t C, int splits, float* out,
                                       float* upd, Upd u,
                                       const int32_t* err_flag) {
  pdl_entry();
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = partial[c];
  for (int z = 1; z < splits; ++z) s += partial[int64_t(z) * C + c];
  if (out) out[c] = s;
  if (upd && !(err_flag && *err_flag)) upd[c] = upd_apply(u, upd + c, upd[c], s);
}

// dW split-K reduction, 4 consecutive columns per thread (N % 4 == 0).
__global__ void splitk_final4_kernel(const float* __restrict__ part, int64_t M,
                                     int64_t N, int splits, float* dW,
                                     int64_t lddw, float* Wu, int64_t ldw,
                                     Upd u, const int32_t* err_flag) {
  pdl_entry();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // float4 index
  const int64_t n4 = N / 4;
  if (e >= M * n4) return;
  const int64_t m = e / n4, c = (e - m * n4) * 4;
  const float4* P = reinterpret_cast<const float4*>(part);
  float4 s = P[e];
  for (int z = 1; z < splits; ++z) {
    const float4 v = P[int64_t(z) * M * n4 + e];
    s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
  }
  if (dW) {
    dW[m * lddw + c] = s.x; dW[m * lddw + c + 1] = s.y;
    dW[m * lddw + c + 2] = s.z; dW[m * lddw + c + 3] = s.w;
  }
  if (Wu && !(err_flag && *err_flag)) {
    float4* w = reinterpret_cast<float4*>(Wu + m * ldw + c);
    *w = upd_apply4(u, reinterpret_cast<float*>(w), *w, s);
  }
}

// dW split-K reduction: dW[m, n] = sum_z part[z][m][n]; optional SGD.
__global__ void splitk_final_kernel(const float* __restrict__ part, int64_t M,
                                    int64_t N, int splits, float* dW,
                                    int64_t lddw, float* Wu, int64_t ldw,
                                    Upd u, const int32_t* err_flag) {
  pdl_entry();
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const int64_t m = e / N, n = e - m * N;
  float s = part[e];
  for (int z = 1; z < splits; ++z) s += part[int64_t(z) * M * N + e];
  if (dW) dW[m * lddw + n] = s;
  if (Wu && !(err_flag && *err_flag))
    Wu[m * ldw + n] = upd_apply(u, Wu + m * ldw + n, Wu[m * ldw + n], s);
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
  launch(gemm_simt_kernel, grid, 256, 0, s, A, B, M, N, K, k_chunk, ep);
  return check_launch("gemm_simt_kernel");
}

int colreduce(const float* X, int64_t ldx, const float* scale, int64_t R,
              int64_t C, float* out, float* upd, const Upd& u,
              const int32_t* err_flag, float* ws, size_t ws_floats,
              cudaStream_t s) {
  const bool vec = C % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(ws) & 15) == 0;
  const int64_t col_blocks = vec ? ceil_div(C, 128) : ceil_div(C, 32);
  // >= 64 rows per chunk, ~2 waves of blocks
  int64_t splits = ceil_div(R, 64);
  if (splits * col_blocks > 2 * kNumSMs) splits = ceil_div(2 * kNumSMs, col_blocks);
  if (splits < 1) splits = 1;
  while (splits > 1 && size_t(splits * C) > ws_floats) --splits;
  DLRM_REQUIRE(size_t(splits * C) <= ws_floats, "column-reduction workspace too small");
  const int64_t rpc = R == 0 ? 1 : ceil_div(R, splits);
  splits = R == 0 ? 1 : ceil_div(R, rpc);
  if (vec) {
    launch(colreduce_partial4_kernel, dim3(unsigned(ceil_div(C, 128)), unsigned(splits)), 256, 0, s, X, ldx, scale, R, C, rpc, ws);
  } else {
    launch(colreduce_partial_kernel, dim3(unsigned(ceil_div(C, 32)), unsigned(splits)), 256, 0, s, X, ldx, scale, R, C, rpc, ws);
  }
  if (int rc = check_launch("colreduce_partial_kernel")) return rc;
  launch(colreduce_final_kernel, unsigned(ceil_div(C, 256)), 256, 0, s, ws, C, int(splits), out, upd, u, err_flag);
  return check_launch("colreduce_final_kernel");
}

int splitk_reduce(const float* part, int64_t M, int64_t N, int splits, float* dW,
                  int64_t lddw, float* Wu, int64_t ldw, const Upd& u,
                  const int32_t* err_flag, cudaStream_t s) {
  const bool v4 = N % 4 == 0 && (ldw % 4 == 0 || !Wu) &&
                  (u.kind != DLRM_UPD_ADAGRAD || u.delta % 4 == 0) &&
                  (reinterpret_cast<uintptr_t>(part) & 15) == 0 &&
                  (!Wu || (reinterpret_cast<uintptr_t>(Wu) & 15) == 0);
  if (v4) {
    launch(splitk_final4_kernel, unsigned(ceil_div(M * N / 4, 256)), 256, 0, s, part, M, N, splits, dW, lddw, Wu, ldw, u, err_flag);
  } else {
    launch(splitk_final_kernel, unsigned(ceil_div(M * N, 256)), 256, 0, s, part, M, N, splits, dW, lddw, Wu, ldw, u, err_flag);
  }
  return check_launch("splitk_final_kernel");
}

}  // namespace dlrm
