// Pairwise dot-product interaction on the 5th-generation tensor cores
// (tcgen05, fp32-accurate 3xTF32), forward and backward.
//
// Reference (dlrmkit, pkg/src/dlrmkit/model.py):
//   interact           218-242  out = [z0 | z_i . z_j for i < j, row-major]
//   interact_backward  245-268  g_i = [i==0] gout[:, :d] + sum_{j!=i} g_ij z_j
//
// Both directions stack S samples' feature rows into one R = S*nf row tile
// (S chosen so the tile and its operands fit TMEM / shared memory) and run
// ONE 128-row MMA chain per tile; only the S diagonal nf x nf blocks of the
// products are used (the tensor pipe has ample headroom at these sizes: the
// op is HBM-bound).  Operands are split x = hi + lo with hi =
// x truncated to TF32 (what the tensor core reads of a raw fp32 operand) and
// lo = nearest-TF32(x - hi); the dropped lo*lo term is 2^-22 relative.
//
// Forward, per tile (A and B both K-major over the embedding dim d):
//   B = [Z | Z_lo] (2*Rp rows), A = Z (the raw rows are the hi operand)
//   D = Z_hi [Z_hi | Z_lo]^T  ->  columns [0, Rp): hh_ij, [Rp, 2Rp): X_ij
//   z_i . z_j = hh_ij + X_ij + X_ji      (X_ji = z_j,hi . z_i,lo)
// so one N = 2Rp MMA per k-step gives all three 3xTF32 products.
//
// Backward, per tile (A = the block-diagonal symmetric pair-gradient matrix
// M = G + G^T in TMEM, K-major; B = Z, MN-major, rows = stacked features):
//   D = [M_hi Z_hi | M_hi Z_lo + M_lo Z_hi]  (hh chain and the small terms in
//   separate TMEM columns, added in the epilogue), then g_0 += gout[:, :d] and
//   the bottom MLP's ReLU mask on feature 0 (training step only).
//
// Feature f of sample b is read at feat[f] + b*stride[f] (the pooled-embedding
// buffer or the all-to-all receive buffer in place), with 16-byte cp.async
// into the swizzled operand layouts.  One persistent CTA per SM:
//   warps 0-3  epilogue (TMEM lane quarters); backward: also build A in TMEM
//   warps 4-7  loaders (cp.async) + lo split
//   warp  8    TMEM allocator + MMA issuer (one thread)
#include <stdlib.h>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "tc_util.cuh"

namespace dlrm {

bool interact_tc_fwd_ok(const FeatureSet& fs, int nf, int64_t dim, int64_t ld_out,
                        const float* out);
int interact_tc_fwd(const FeatureSet& fs, int nf, int64_t dim, int64_t batch, float* out,
                    int64_t ld_out, int64_t pad_to, cudaStream_t s);
bool interact_tc_bwd_ok(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                        const float* gout, int64_t ld_gout);
int interact_tc_bwd(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                    int64_t batch, const float* gout, int64_t ld_gout, int mask_f0,
                    cudaStream_t s);

namespace {
using namespace tcu;

constexpr int IA_EPI = 128;      // epilogue warps 0-3
constexpr uint32_t IA_TMEM_COLS = 512;
constexpr size_t IA_SMEM_MAX = 220 * 1024;

// host-computed tile geometry (passed by value)
struct IaGeom {
  int nf, d, S, R, P;
  int Pp;            // bwd: P rounded up to 4 (pair-gradient row pitch)
  int Rp;            // fwd: R rounded up to 16 (B rows, MMA N; lo lanes of A at Rp)
  int rows;          // fwd: rows per K-chunk region (= Rp)
  int kchunks;       // fwd: ceil(d / 32)
  int tma;           // 1: features are rows of one [batch * nf, d] matrix, loaded by TMA
  int Kq;            // bwd: R rounded up to 16 (A slot columns)
  int Kp;            // bwd: R rounded up to 8 (MMA K)
  int nst;           // stages
  uint32_t stage_bytes;
  uint32_t b_bytes;  // bwd: operand bytes of a stage (the rest: pair gradients)
  uint32_t a_base;   // bwd: TMEM column of the A slots
  uint32_t idesc;
};

__device__ __forceinline__ void ia_pair(int p, int nf, int& i, int& j) {
  int row = 0, base = 0;
  while (p >= base + (nf - 1 - row)) {
    base += nf - 1 - row;
    ++row;
  }
  i = row;
  j = row + 1 + (p - base);
}

__device__ __forceinline__ float4 split_lo4(float4 v) {
  return make_float4(
      __uint_as_float(tf32_rna(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u))),
      __uint_as_float(tf32_rna(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u))),
      __uint_as_float(tf32_rna(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u))),
      __uint_as_float(tf32_rna(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u))));
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// Loader pipeline over this CTA's tiles (blockIdx.x, + gridDim.x, ...):
// issue(it, tile) starts the copies of local tile `it` (one cp.async group),
// finish(it, tile) completes it once its group has landed; up to IA_AHEAD
// later tiles stay in flight meanwhile (bounded by the stage count).
#ifndef DLRM_IA_AHEAD
#define DLRM_IA_AHEAD 3
#endif
constexpr int IA_AHEAD = DLRM_IA_AHEAD;

// DLRM_IA_PROF builds (measurements only): clock64 time per role / phase of
// the backward kernel, summed over CTAs, read with dlrm_ia_prof()
#ifdef DLRM_IA_PROF
__device__ unsigned long long g_ia_prof[32];
#define IA_T0(n) const long long _t##n = clock64();
#define IA_T1(n, k) prof[k] += (unsigned long long)(clock64() - _t##n);
#else
#define IA_T0(n)
#define IA_T1(n, k)
#endif

template <class Issue, class Finish>
__device__ __forceinline__ void ia_pipeline(int64_t ntiles, int nst, Issue issue, Finish finish) {
  const int ahead = nst - 1 < IA_AHEAD ? nst - 1 : IA_AHEAD;
  int issued = 0;
  int64_t next = blockIdx.x;
  for (; issued < ahead && next < ntiles; ++issued, next += gridDim.x) issue(issued, next);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    // groups still allowed in flight: the ones issued after tile `it`
    const int pending = issued - it - 1;
    if (pending >= 3) cp_async_wait<3>();
    else if (pending >= 2) cp_async_wait<2>();
    else if (pending == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    finish(it, tile);
    // the next tile's copies only now: its stage is the one the MMA of an
    // earlier tile read, and waiting for that MMA before finishing this tile
    // would serialise the loaders with the tensor core
    if (next < ntiles) {
      issue(issued++, next);
      next += gridDim.x;
    }
  }
}

// ---------------------------------------------------------------------------
// forward
//
// Per tile of S samples (R = S*nf feature rows, Rp = R rounded up to 16,
// Rp + R <= 128):
//   A (TMEM, K-major: lane = row, column = k) = [Z_hi rows 0..R) ; Z_lo rows
//     Rp..Rp+R)], written by the splitter warps from the landed tile;
//   B (smem, K-major 128B swizzle) = the raw Z rows (the hi operand);
//   D = A B^T (N = Rp): rows [0, R) hh_ij = z_i,hi . z_j,hi,
//                       rows [Rp, Rp+R) Y_ij = z_i,lo . z_j,hi,
//   z_i . z_j = hh_ij + Y_ij + Y_ji.
// Stage: kchunks regions of Rp rows x 128 B (16-byte piece j of row r at
// (j ^ (r & 7))).  TMEM: D buffers [0, 64) / [64, 128), A slots from 128.
// Roles: warps 0-3 epilogue, 4-7 splitters (TMEM lane quarters), 8 MMA
// issuer, 9 loader (TMA, or cp.async for non-uniform feature pointers).
constexpr int IF_WARPS = 10;
constexpr int IF_THREADS = 32 * IF_WARPS;

__global__ void __launch_bounds__(IF_THREADS, 1)
interact_tc_fwd_kernel(const __grid_constant__ CUtensorMap tmZ, FeatureSet fs, IaGeom g,
                       int64_t batch, float* __restrict__ out, int64_t ld_out, int64_t pad_to) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* stages = smem;
  float* H = reinterpret_cast<float*>(smem + size_t(g.nst) * g.stage_bytes);  // [R][nf]
  float* Y = H + g.R * g.nf;                                                   // [R][nf]
  int* pairs = reinterpret_cast<int*>(Y + g.R * g.nf);                         // [P]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(pairs + g.P) + 7) & ~uintptr_t(7));
  uint64_t* land = bars;        // [nst] tile landed (TMA tx / 32 cp.async lanes)
  uint64_t* empty = bars + 4;   // [nst] MMA done with the stage
  uint64_t* afull = bars + 8;   // [2] A slot written (4 splitter warps)
  uint64_t* aempty = bars + 10; // [2] A slot consumed
  uint64_t* tfull = bars + 12;  // [2] D buffer ready
  uint64_t* tempty = bars + 14; // [2] D buffer drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nf = g.nf, d = g.d, S = g.S, R = g.R, Rp = g.Rp;
  const int64_t ntiles = ceil_div(batch, S);
  const int W = d + g.P;

  for (int p = threadIdx.x; p < g.P; p += blockDim.x) {
    int i, j;
    ia_pair(p, nf, i, j);
    pairs[p] = (i << 16) | j;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.nst; ++s) {
      mbar_init(&land[s], g.tma ? 1 : 32);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 4);
      mbar_init(&aempty[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) tmem_alloc_warp(tmem_slot, IA_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  auto piece = [&](uint8_t* base, int r, int p) {  // 16-byte piece p (4 floats) of row r
    return base + size_t(p >> 3) * Rp * 128 + r * 128 + (((p & 7) ^ (r & 7)) << 4);
  };

  if (warp == 9) {
    // ---- loader: the tile's R rows into stage it % nst
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % g.nst;
      if (it >= g.nst) mbar_wait(&empty[st], ((it / g.nst) - 1) & 1);
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      const int64_t b0 = tile * S;
      if (g.tma) {
        if (lane == 0) {  // consecutive rows of the [batch * nf, d] matrix (past the end: zeros)
          mbar_expect_tx(&land[st], uint32_t(g.kchunks * R * 128));
          for (int kc = 0; kc < g.kchunks; ++kc)
            tma_load_2d(base + size_t(kc) * Rp * 128, &tmZ, &land[st], 32 * kc, int(b0 * nf));
        }
      } else {
        const int ns = int(batch - b0 < S ? batch - b0 : S);
        const int nv = d / 4;
        for (int e = lane; e < ns * nf * nv; e += 32) {
          const int r = e / nv, p = e - r * nv, sm = r / nf, f = r - sm * nf;
          cp_async16(piece(base, r, p), fs.feat[f] + (b0 + sm) * fs.stride[f] + 4 * p, true);
        }
        cp_async_commit();
        cp_async_wait<0>();
        fence_async_smem();
        mbar_arrive(&land[st]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---- splitters: lane r of A = row r's hi (r < R) or row r - Rp's lo
    const int q = warp - 4, r = 32 * q + lane;
    const bool hi_row = r < R, lo_row = r >= Rp && r < Rp + R;
    const int row = hi_row ? r : (lo_row ? r - Rp : 0);
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % g.nst, ab = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      mbar_wait(&land[st], (it / g.nst) & 1);
      if (it >= 2) mbar_wait(&aempty[ab], ((it - 2) >> 1) & 1);
      tc_fence_after();
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      const uint32_t slot = tmem + lane_off + 128u + uint32_t(ab * d);
      // feature-0 rows also give the output's z0 columns (exact copy)
      const int sm = row / nf;
      float* z0 = (hi_row && row - sm * nf == 0 && sm < ns) ? out + (b0 + sm) * ld_out : nullptr;
      for (int c0 = 0; c0 < d; c0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 x = *reinterpret_cast<const float4*>(piece(base, row, c0 / 4 + k));
          if (z0) *reinterpret_cast<float4*>(z0 + c0 + 4 * k) = x;
          const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t hb = __float_as_uint(xs[e]) & 0xFFFFE000u;
            v[4 * k + e] = lo_row ? tf32_rna(xs[e] - __uint_as_float(hb)) : hb;
          }
        }
        tmem_st16(slot + uint32_t(c0), v);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
      if (q == 0 && pad_to > W)  // zero pad columns of the output rows
        for (int e = lane; e < ns * int(pad_to - W); e += 32) {
          const int s2 = e / int(pad_to - W);
          out[(b0 + s2) * ld_out + W + (e - s2 * int(pad_to - W))] = 0.f;
        }
    }
  } else if (warp == 8) {
    // ---- MMA issuer
    if (lane == 0) {
      const int ksteps = d / 8;
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % g.nst, ab = it & 1;
        mbar_wait(&land[st], (it / g.nst) & 1);
        mbar_wait(&afull[ab], (it >> 1) & 1);
        if (it >= 2) mbar_wait(&tempty[ab], ((it - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(64 * ab);
        const uint32_t a = tmem + 128u + uint32_t(ab * d);
        const uint32_t base = smem_u32(stages + size_t(st) * g.stage_bytes);
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t b = smem_desc(base + uint32_t((ks >> 2) * Rp * 128 + (ks & 3) * 32), 16,
                                       1024, 2);
          mma_tf32_ts(dt, a + uint32_t(8 * ks), b, g.idesc, ks > 0 ? 1u : 0u);
        }
        mma_commit(&empty[st]);
        mma_commit(&aempty[ab]);
        mma_commit(&tfull[ab]);
      }
    }
  } else {
    // ---- epilogue (warps 0-3 = TMEM lane quarters): D rows -> H / Y, then
    // the pair columns of the output rows
    const int q = warp, r = 32 * q + lane;
    const bool hi_row = r < R, lo_row = r >= Rp && r < Rp + R;
    const int i = hi_row ? r : (lo_row ? r - Rp : -1);
    float* dst = hi_row ? H : Y;
    const int blk = i >= 0 ? (i / nf) * nf : 0;
    // column window of this warp's rows (the union of their samples' blocks)
    int lo_c = i >= 0 ? blk : 1 << 30, hi_c = i >= 0 ? blk + nf : 0;
    for (int o = 16; o > 0; o >>= 1) {
      lo_c = min(lo_c, __shfl_xor_sync(0xffffffffu, lo_c, o));
      hi_c = max(hi_c, __shfl_xor_sync(0xffffffffu, hi_c, o));
    }
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      mbar_wait(&tfull[ab], (it >> 1) & 1);
      tc_fence_after();
      const bool valid = i >= 0 && i / nf < ns;
      for (int c0 = lo_c & ~15; c0 < hi_c; c0 += 16) {
        uint32_t v[16];
        tmem_ld16_issue(tmem + lane_off + uint32_t(64 * ab + c0), v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int j = c0 + k;
          if (valid && j >= blk && j < blk + nf) dst[i * nf + (j - blk)] = __uint_as_float(v[k]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
      named_bar(2, IA_EPI);
      for (int s2 = 0; s2 < ns; ++s2) {
        float* orow = out + (b0 + s2) * ld_out + d;
        const float* Hs = H + s2 * nf * nf;
        const float* Ys = Y + s2 * nf * nf;
        for (int p = threadIdx.x; p < g.P; p += IA_EPI) {
          const int pr = pairs[p], pi = pr >> 16, pj = pr & 0xffff;
          orow[p] = (Hs[pi * nf + pj] + Ys[pi * nf + pj]) + Ys[pj * nf + pi];
        }
      }
      named_bar(2, IA_EPI);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, IA_TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// backward
//
// Per tile of S samples (R rows, Kp = R rounded up to 8, Kq = to 16):
//   A (TMEM, K-major) = [M_hi | M_lo], M = blockdiag over the samples of the
//     symmetric pair-gradient matrix G + G^T (zero diagonal), built by the
//     loader warps from the tile's gout[b, d + p];
//   B (smem, MN-major, SWIZZLE_128B_BASE32B: 32-wide column chunks of Kp
//     rows x 128 B, 32-byte atom a of row k at (a ^ (k & 3))) = [Z | Z_lo];
//   D = M_lo Z_hi + M_hi Z_lo (first: the small terms, against a small
//     accumulator) + M_hi Z_hi, one TMEM chain of d columns;
// then g_0 += gout[b, :d] and the bottom MLP's ReLU mask on feature 0.
// TMEM: D buffers [0, d) / [d, 2d), A slots [A_hi | A_lo] from a_base.
// Roles: warps 0-3 epilogue (TMEM -> gradient rows, straight from
// registers), 4-7 loaders (TMA or cp.async, lo split, A build; TMEM lane
// quarters), 8 MMA issuer.
__device__ __forceinline__ uint32_t mn_off(int k, int n) {
  // byte offset of element (k, n) inside the chunk set (without chunk stride)
  return uint32_t(k * 128 + ((((n & 31) >> 3) ^ (k & 3)) << 5) + ((n & 7) << 2));
}

constexpr int IB_EW = 8;                  // epilogue warps 0-7 (2 per lane quarter)
constexpr int IB_LW = 8;                  // loader warps 8-15 (2 per lane quarter)
constexpr int IB_MMA = IB_EW + IB_LW;     // MMA warp
constexpr int IB_THREADS = 32 * (IB_MMA + 1);
constexpr int IB_ET = 32 * IB_EW, IB_LT = 32 * IB_LW;

__global__ void __launch_bounds__(IB_THREADS, 1)
interact_tc_bwd_kernel(const __grid_constant__ CUtensorMap tmZ, FeatureSet fs,
                       GradFeatureSet gs, IaGeom g, int64_t batch,
                       const float* __restrict__ gout, int64_t ld_gout, int mask_f0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* stages = smem;
  // feature 0's extra terms of the tile's samples (gout[b, :d] and z0 for
  // the mask), prefetched by the epilogue warps: [2 buffers][S][2d]
  float* gz = reinterpret_cast<float*>(smem + size_t(g.nst) * g.stage_bytes);
  // the tile's symmetric pair-gradient matrices [R][mp] and the pair table
  const int mp = g.nf + 1;
  float* Ms = gz + size_t(2) * g.S * 2 * g.d;
  int* pairs = reinterpret_cast<int*>(Ms + size_t(g.R) * mp);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(pairs + g.P) + 7) & ~uintptr_t(7));
  uint64_t* land = bars;        // [nst] TMA landed (tx count)
  uint64_t* empty = bars + 4;   // [nst] MMA done with the stage
  uint64_t* afull = bars + 8;   // [2] A slot + B_lo ready (4 loader warps)
  uint64_t* aempty = bars + 10; // [2] A slot consumed
  uint64_t* dfull = bars + 12;  // [2] D buffer ready
  uint64_t* dempty = bars + 14; // [2] D buffer drained (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nf = g.nf, d = g.d, S = g.S, P = g.P, Pp = g.Pp;
  const int64_t ntiles = ceil_div(batch, S);
  const uint32_t lbo = uint32_t(g.Kp) * 128;  // column-chunk stride
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int pi, pj;
    ia_pair(p, nf, pi, pj);
    pairs[p] = (pi << 16) | pj;
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < g.nst; ++s) {
      mbar_init(&land[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], IB_LW);
      mbar_init(&aempty[b], 1);
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], IB_EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == IB_MMA) tmem_alloc_warp(tmem_slot, IA_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp >= IB_EW && warp < IB_MMA) {
    // ---- loaders (lane quarter q, half lh of the A columns)
    const int t = threadIdx.x - IB_ET, lw = warp - IB_EW, q = lw & 3, lh = lw >> 2;
    const int nv = d / 4;
    // pair gradients by 16-byte cp.async (the padded row holds Pp floats)
    const bool g16 = (reinterpret_cast<uintptr_t>(gout) % 16) == 0 && ld_gout % 4 == 0 &&
                     d % 4 == 0 && ld_gout >= d + Pp;
    const int i = 32 * q + lane;  // this thread's row of A
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    unsigned long long prof[8] = {0};
    IA_T0(all)
    auto issue = [&](int it, int64_t tile) {
      const int st = it % g.nst;
      IA_T0(e)
      if (it >= g.nst) mbar_wait(&empty[st], ((it / g.nst) - 1) & 1);
      IA_T1(e, 0)
      IA_T0(w)
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      float* gp = reinterpret_cast<float*>(base + g.b_bytes);
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const int rv = ns * nf;
      if (g.tma) {
        // Kp consecutive rows of the [batch * nf, d] matrix, one 32-column
        // box each: rows past the tile hold the next samples' (finite)
        // features, which meet zero columns of A; past the batch: zeros
        if (t == 0) {
          mbar_expect_tx(&land[st], uint32_t((d / 32) * lbo));
          for (int c = 0; c < d / 32; ++c)
            tma_load_2d(base + size_t(c) * lbo, &tmZ, &land[st], 32 * c, int(b0 * nf));
        }
      } else {
        // a 16-byte piece per lane (zero past the valid rows: A is zero
        // there, and 0 * garbage could be NaN)
        for (int r = lw; r < g.Kp; r += IB_LW) {
          const bool ok = r < rv;
          const int sm = ok ? r / nf : 0, f = ok ? r - sm * nf : 0;
          const float* src = fs.feat[f] + (b0 + sm) * fs.stride[f];
          for (int p = lane; p < nv; p += 32) {
            const int n = 4 * p;
            cp_async16(base + size_t(n >> 5) * lbo + mn_off(r, n), ok ? src + n : fs.feat[0], ok);
          }
        }
      }
      // pair gradients of the tile's samples
      if (g16) {
        const int pq = Pp / 4;
        for (int e = t; e < ns * pq; e += IB_LT) {
          const int sm = e / pq, c = e - sm * pq;
          cp_async16(gp + sm * Pp + 4 * c, gout + (b0 + sm) * ld_gout + d + 4 * c, true);
        }
      } else {
        for (int sm = 0; sm < ns; ++sm)
          for (int e = t; e < P; e += IB_LT) gp[sm * Pp + e] = __ldg(gout + (b0 + sm) * ld_gout + d + e);
      }
      cp_async_commit();
      IA_T1(w, 1)
    };
    auto finish = [&](int it, int64_t tile) {
      const int st = it % g.nst, ab = it & 1;
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      const float* gp = reinterpret_cast<const float*>(base + g.b_bytes);
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      IA_T0(l)
      if (g.tma) mbar_wait(&land[st], (it / g.nst) & 1);
      IA_T1(l, 2)
      IA_T0(b)
      named_bar(1, IB_LT);
      IA_T1(b, 3)
      IA_T0(o)
      // lo columns [d, 2d)
      for (int r = lw; r < g.Kp; r += IB_LW)
        for (int p = lane; p < nv; p += 32) {
          const int n = 4 * p, nl = d + n;
          const float4 v = *reinterpret_cast<const float4*>(base + size_t(n >> 5) * lbo + mn_off(r, n));
          *reinterpret_cast<float4*>(base + size_t(nl >> 5) * lbo + mn_off(r, nl)) = split_lo4(v);
        }
      fence_async_smem();
      IA_T1(o, 4)
      // the tile's symmetric M_s = G_s + G_s^T (zero diagonal) in smem,
      // row pitch mp, so that A row i reads its nf values contiguously
      for (int e = t; e < ns * nf; e += IB_LT) Ms[(e / nf) * nf * mp + (e % nf) * (mp + 1)] = 0.f;
      for (int e = t; e < ns * P; e += IB_LT) {
        const int sm = e / P, p = e - sm * P, pr = pairs[p], pi = pr >> 16, pj = pr & 0xffff;
        const float v = gp[sm * Pp + p];
        Ms[(sm * nf + pi) * mp + pj] = v;
        Ms[(sm * nf + pj) * mp + pi] = v;
      }
      named_bar(1, IB_LT);
      // A row i: M_s[fi][fk] over this sample's block, split hi / lo (this
      // warp: the 16-column groups of parity lh)
      IA_T0(a)
      if (it >= 2) mbar_wait(&aempty[ab], ((it - 2) >> 1) & 1);
      IA_T1(a, 5)
      IA_T0(c)
      tc_fence_after();
      const bool valid = i < ns * nf;
      const int blk = (i / nf) * nf;
      const float* mrow = Ms + size_t(i) * mp;
      const uint32_t slot = tmem + lane_off + g.a_base + uint32_t(2 * g.Kq * ab);
      for (int c0 = 16 * lh; c0 < g.Kq; c0 += 32) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int fk = c0 + k - blk;
          const float m = (valid && fk >= 0 && fk < nf) ? mrow[fk] : 0.f;
          hi[k] = __float_as_uint(m) & 0xFFFFE000u;
          lo[k] = tf32_rna(m - __uint_as_float(hi[k]));
        }
        tmem_st16(slot + uint32_t(c0), hi);
        tmem_st16(slot + uint32_t(g.Kq + c0), lo);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
      IA_T1(c, 6)
    };
    ia_pipeline(ntiles, g.nst, issue, finish);
    IA_T1(all, 7)
#ifdef DLRM_IA_PROF
    if (threadIdx.x == IB_ET)
      for (int k = 0; k < 8; ++k) atomicAdd(&g_ia_prof[k], prof[k]);
#endif
  } else if (warp == IB_MMA) {
    // ---- MMA issuer
    if (lane == 0) {
      const int ksteps = g.Kp / 8;
      unsigned long long prof[8] = {0};
      IA_T0(all)
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % g.nst, ab = it & 1;
        IA_T0(a)
        mbar_wait(&afull[ab], (it >> 1) & 1);
        IA_T1(a, 0)
        IA_T0(d)
        if (it >= 2) mbar_wait(&dempty[ab], ((it - 2) >> 1) & 1);
        IA_T1(d, 1)
        tc_fence_after();
        const uint32_t base = smem_u32(stages + size_t(st) * g.stage_bytes);
        const uint32_t a_hi = tmem + g.a_base + uint32_t(2 * g.Kq * ab), a_lo = a_hi + g.Kq;
        const uint32_t dt = tmem + uint32_t(d * ab);
        const uint32_t lo_off = uint32_t(d / 32) * lbo + uint32_t(d % 32 ? 64 : 0);
        // the small terms first, into a fresh accumulator, then hi x hi
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint32_t kb = base + uint32_t(ks * 1024);
          mma_tf32_ts(dt, a_lo + uint32_t(8 * ks), smem_desc(kb, lbo, 512, 1), g.idesc,
                      ks > 0 ? 1u : 0u);
          mma_tf32_ts(dt, a_hi + uint32_t(8 * ks), smem_desc(kb + lo_off, lbo, 512, 1), g.idesc,
                      1u);
        }
        for (int ks = 0; ks < ksteps; ++ks)
          mma_tf32_ts(dt, a_hi + uint32_t(8 * ks),
                      smem_desc(base + uint32_t(ks * 1024), lbo, 512, 1), g.idesc, 1u);
        mma_commit(&empty[st]);
        mma_commit(&aempty[ab]);
        mma_commit(&dfull[ab]);
      }
      IA_T1(all, 7)
#ifdef DLRM_IA_PROF
      for (int k = 0; k < 8; ++k) atomicAdd(&g_ia_prof[8 + k], prof[k]);
#endif
    }
  } else {
    // ---- epilogue (TMEM lane quarter q, half h of the columns): row i of D
    // is feature fi of sample s; written straight from registers
    const int q = warp & 3, h = warp >> 2, i = 32 * q + lane;
    const int ecols = d >= 32 ? d / 2 : d;
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    const int sm = i / nf, fi = i - sm * nf;
    const int nv = d / 4;
    unsigned long long prof[8] = {0};
    IA_T0(all)
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const bool valid = i < ns * nf;
      IA_T0(p)
      const int64_t b = b0 + (valid ? sm : 0);
      float* dst = gs.feat[valid ? fi : 0] + b * gs.stride[valid ? fi : 0];
      // gout[b, :d] / z0 of the tile's samples: the loads are in flight while
      // the MMAs run, then land in this tile's buffer
      float* gzb = gz + size_t(ab) * S * 2 * d;
      float4 pre[2];
      int npre = 0;
      for (int e = threadIdx.x; e < ns * 2 * nv && npre < 2; e += IB_ET, ++npre) {
        const int sm2 = e / (2 * nv), c = e - sm2 * 2 * nv;
        pre[npre] = c < nv ? __ldg(reinterpret_cast<const float4*>(gout + (b0 + sm2) * ld_gout) + c)
                           : __ldg(reinterpret_cast<const float4*>(fs.feat[0] + (b0 + sm2) *
                                                                     fs.stride[0]) + (c - nv));
      }
      IA_T1(p, 0)
      IA_T0(f)
      mbar_wait(&dfull[ab], (it >> 1) & 1);
      IA_T1(f, 1)
      IA_T0(g)
      npre = 0;
      for (int e = threadIdx.x; e < ns * 2 * nv && npre < 2; e += IB_ET, ++npre)
        reinterpret_cast<float4*>(gzb)[e] = pre[npre];
      for (int e = threadIdx.x + 2 * IB_ET; e < ns * 2 * nv; e += IB_ET) {
        const int sm2 = e / (2 * nv), c = e - sm2 * 2 * nv;
        reinterpret_cast<float4*>(gzb)[e] =
            c < nv ? __ldg(reinterpret_cast<const float4*>(gout + (b0 + sm2) * ld_gout) + c)
                   : __ldg(reinterpret_cast<const float4*>(fs.feat[0] + (b0 + sm2) * fs.stride[0]) +
                           (c - nv));
      }
      named_bar(2, IB_ET);
      IA_T1(g, 2)
      IA_T0(m)
      const float* g0 = gzb + size_t(valid ? sm : 0) * 2 * d;
      const float* z0 = g0 + d;
      tc_fence_after();
      if (32 * q < ns * nf) {
        for (int c0 = h * ecols; c0 < (h + 1) * ecols && c0 < d; c0 += 16) {
          uint32_t v[16];
          tmem_ld16_issue(tmem + lane_off + uint32_t(d * ab + c0), v);
          tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int k = 0; k < 16; k += 4) {
              float4 o = make_float4(__uint_as_float(v[k]), __uint_as_float(v[k + 1]),
                                     __uint_as_float(v[k + 2]), __uint_as_float(v[k + 3]));
              if (fi == 0) {
                const float4 a = *reinterpret_cast<const float4*>(g0 + c0 + k);
                o.x = a.x + o.x; o.y = a.y + o.y; o.z = a.z + o.z; o.w = a.w + o.w;
                if (mask_f0) {
                  const float4 zz = *reinterpret_cast<const float4*>(z0 + c0 + k);
                  o.x *= zz.x > 0.f ? 1.f : 0.f; o.y *= zz.y > 0.f ? 1.f : 0.f;
                  o.z *= zz.z > 0.f ? 1.f : 0.f; o.w *= zz.w > 0.f ? 1.f : 0.f;
                }
              }
              *reinterpret_cast<float4*>(dst + c0 + k) = o;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[ab]);
      IA_T1(m, 3)
    }
    IA_T1(all, 7)
#ifdef DLRM_IA_PROF
    if (threadIdx.x == 0)
      for (int k = 0; k < 8; ++k) atomicAdd(&g_ia_prof[16 + k], prof[k]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == IB_MMA) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, IA_TMEM_COLS);
  }
}

uint32_t ceil_to(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

bool fwd_geom(int nf, int d, IaGeom* g) {
  if (nf < 2 || nf > 64 || d < 8 || d > 128 || d % 8) return false;
  const int P = nf * (nf - 1) / 2;
  const int kchunks = (d + 31) / 32;
  // Rp: R rounded up to 16 (the MMA's N = Rp needs N % 16 == 0 at M = 128);
  // A holds the hi rows at lanes [0, R) and the lo rows at [Rp, Rp + R)
  int S = 128 / nf;
  while (S > 1 && int(ceil_to(S * nf, 16)) + S * nf > 128) --S;
  const int R = S * nf, Rp = int(ceil_to(R, 16));
  if (Rp + R > 128) return false;
  const uint32_t stage = uint32_t(kchunks) * Rp * 128;
  const size_t scratch = size_t(2) * R * nf * 4 + size_t(P) * 4 + 256;
  int nst = int((IA_SMEM_MAX - 1024 - scratch) / stage);
  if (nst > 4) nst = 4;
  if (nst < 2) return false;
  *g = IaGeom{};
  g->nf = nf; g->d = d; g->S = S; g->R = R; g->P = P; g->Rp = Rp; g->rows = Rp;
  g->kchunks = kchunks; g->nst = nst; g->stage_bytes = stage;
  g->idesc = instr_desc(Rp, false, false);
  return true;
}

bool bwd_geom(int nf, int d, IaGeom* g) {
  // the lo half of B starts at column d: a whole 32-column chunk, or (d = 16)
  // the upper half of chunk 0, so one descriptor addresses it
  if (nf < 2 || nf > 64 || d < 16 || d > 128 || (d % 32 && d != 16)) return false;
  const int P = nf * (nf - 1) / 2;
  const uint32_t a_base = ceil_to(uint32_t(2 * d), 32);  // after the two D buffers
  for (int S = 128 / nf; S >= 1; --S) {
    const int R = S * nf, Kq = int(ceil_to(R, 16)), Kp = int(ceil_to(R, 8));
    if (a_base + 4u * Kq > IA_TMEM_COLS) continue;
    const uint32_t nchunk = (2 * d + 31) / 32;
    const uint32_t b_bytes = nchunk * Kp * 128;
    const int Pp = int(ceil_to(P, 4));
    const uint32_t stage = ceil_to(b_bytes + uint32_t(S) * Pp * 4, 1024);
    int nst = int((IA_SMEM_MAX - 1024 - 256 - size_t(16) * S * d - size_t(R) * (nf + 1) * 4 -
                   size_t(P) * 4) / stage);
    if (nst > 4) nst = 4;
    if (nst < 2) continue;
    *g = IaGeom{};
    g->nf = nf; g->d = d; g->S = S; g->R = R; g->P = P; g->Pp = Pp; g->Kq = Kq; g->Kp = Kp;
    g->nst = nst; g->stage_bytes = stage; g->b_bytes = b_bytes; g->a_base = a_base;
    g->idesc = instr_desc(d, false, true);
    return true;
  }
  return false;
}

size_t fwd_smem(const IaGeom& g) {
  return 1024 + size_t(g.nst) * g.stage_bytes + size_t(2) * g.R * g.nf * 4 + size_t(g.P) * 4 +
         8 + 24 * 8;
}
size_t bwd_smem(const IaGeom& g) {
  return 1024 + size_t(g.nst) * g.stage_bytes + size_t(2) * g.S * 2 * g.d * 4 +
         size_t(g.R) * (g.nf + 1) * 4 + size_t(g.P) * 4 + 8 + 24 * 8;
}

// features f at feat[0] + f*d with row stride nf*d (the training engine's
// [B, nf, d] buffer): the tile rows are consecutive rows of one matrix
bool uniform_rows(const FeatureSet& fs, int nf, int64_t dim) {
  if (dim % 32 || getenv("DLRM_IA_NO_TMA")) return false;
  for (int f = 0; f < nf; ++f)
    if (fs.feat[f] != fs.feat[0] + f * dim || fs.stride[f] != nf * dim) return false;
  return true;
}

bool tc_ia_enabled() {
  static const bool off = getenv("DLRM_IA_SIMT") != nullptr;
  return !off && tc_enabled();
}

}  // namespace

bool interact_tc_fwd_ok(const FeatureSet& fs, int nf, int64_t dim, int64_t ld_out,
                        const float* out) {
  IaGeom g;
  if (!tc_ia_enabled() || !fwd_geom(nf, int(dim), &g)) return false;
  if (reinterpret_cast<uintptr_t>(out) % 16 || ld_out % 4) return false;
  for (int f = 0; f < nf; ++f)
    if (reinterpret_cast<uintptr_t>(fs.feat[f]) % 16 || fs.stride[f] % 4) return false;
  return true;
}

int interact_tc_fwd(const FeatureSet& fs, int nf, int64_t dim, int64_t batch, float* out,
                    int64_t ld_out, int64_t pad_to, cudaStream_t s) {
  IaGeom g;
  DLRM_REQUIRE(fwd_geom(nf, int(dim), &g), "interaction shape not supported by tcgen05 path");
  const size_t smem = fwd_smem(g);
  static bool configured = false;
  if (!configured) {
    DLRM_CUDA(cudaFuncSetAttribute(interact_tc_fwd_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(IA_SMEM_MAX + 4096)));
    configured = true;
  }
  CUtensorMap tm{};
  g.tma = uniform_rows(fs, nf, dim) &&
          tma_encode_2d(&tm, fs.feat[0], dim, batch * nf, dim, 32, g.R, 1);
  const int64_t ntiles = ceil_div(batch, g.S);
  const unsigned grid = unsigned(ntiles < kNumSMs ? ntiles : kNumSMs);
  launch(interact_tc_fwd_kernel, grid, IF_THREADS, smem, s, tm, fs, g, batch, out, ld_out,
         pad_to);
  return check_launch("interact_tc_fwd_kernel");
}

bool interact_tc_bwd_ok(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                        const float* gout, int64_t ld_gout) {
  IaGeom g;
  if (!tc_ia_enabled() || !bwd_geom(nf, int(dim), &g)) return false;
  if (reinterpret_cast<uintptr_t>(gout) % 16 || ld_gout % 4) return false;
  for (int f = 0; f < nf; ++f)
    if (reinterpret_cast<uintptr_t>(fs.feat[f]) % 16 || fs.stride[f] % 4 ||
        reinterpret_cast<uintptr_t>(gs.feat[f]) % 16 || gs.stride[f] % 4)
      return false;
  return true;
}

int interact_tc_bwd(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                    int64_t batch, const float* gout, int64_t ld_gout, int mask_f0,
                    cudaStream_t s) {
  IaGeom g;
  DLRM_REQUIRE(bwd_geom(nf, int(dim), &g), "interaction shape not supported by tcgen05 path");
  const size_t smem = bwd_smem(g);
  static bool configured = false;
  if (!configured) {
    DLRM_CUDA(cudaFuncSetAttribute(interact_tc_bwd_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(IA_SMEM_MAX + 4096)));
    configured = true;
  }
  CUtensorMap tm{};
  g.tma = uniform_rows(fs, nf, dim) &&
          tma_encode_2d(&tm, fs.feat[0], dim, batch * nf, dim, 32, g.Kp, 2);
  const int64_t ntiles = ceil_div(batch, g.S);
  const unsigned grid = unsigned(ntiles < kNumSMs ? ntiles : kNumSMs);
  launch(interact_tc_bwd_kernel, grid, IB_THREADS, smem, s, tm, fs, gs, g, batch, gout, ld_gout,
         mask_f0);
  return check_launch("interact_tc_bwd_kernel");
}

}  // namespace dlrm

#ifdef DLRM_IA_PROF
extern "C" int dlrm_ia_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dlrm::g_ia_prof, sizeof(unsigned long long) * 32);
  static const unsigned long long zero[32] = {0};
  cudaMemcpyToSymbol(dlrm::g_ia_prof, zero, sizeof(zero));
  return 0;
}
#endif
