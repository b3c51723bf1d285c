// Pairwise dot-product interaction on the 5th-generation tensor cores
// (tcgen05, fp32-accurate 3xTF32), forward and backward.
//
// Reference (dlrmkit, pkg/src/dlrmkit/model.py):
//   interact           218-242  out = [z0 | z_i . z_j for i < j, row-major]
//   interact_backward  245-268  g_i = [i==0] gout[:, :d] + sum_{j!=i} g_ij z_j
//
// Operands are split x = hi + lo with hi = x truncated to TF32 (what the
// tensor core reads of a raw fp32 operand) and lo = nearest-TF32(x - hi);
// the dropped lo*lo term is 2^-22 relative.  The tensor pipe has ample
// headroom at these sizes (the op is HBM-bound), so both
// directions spend MMA work on zero padding to keep the data movement simple.
//
// Forward: S samples' feature rows stacked into one R = S*nf row tile, ONE
// 128-row MMA chain per tile over the embedding dim (A = [Z_hi ; Z_lo] rows
// in TMEM, B = the raw rows), keeping only the S diagonal nf x nf blocks:
//   z_i . z_j = hh_ij + Y_ij + Y_ji   (Y_ij = z_i,lo . z_j,hi).
//
// Backward: per sample D = Z^T M (M = G + G^T, zero diagonal) with the
// embedding dim on the TMEM lanes, so each warp store of the epilogue is 32
// consecutive floats of one gradient row; see interact_tc_bwd_kernel.
//
// Feature f of sample b is read at feat[f] + b*stride[f] (the pooled-embedding
// buffer or the all-to-all receive buffer in place): by TMA when the features
// are the rows of one [batch * nf, d] matrix, else by 16-byte cp.async.  One
// persistent CTA per SM, warp-specialised (roles listed at each kernel).
#include <stdlib.h>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "tc_util.cuh"

namespace dlrm {

bool interact_tc_fwd_ok(const FeatureSet& fs, int nf, int64_t dim, int64_t batch,
                        int64_t ld_out, const float* out);
int interact_tc_fwd(const FeatureSet& fs, int nf, int64_t dim, int64_t batch, float* out,
                    int64_t ld_out, int64_t pad_to, cudaStream_t s);
bool interact_tc_bwd_ok(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                        int64_t batch, const float* gout, int64_t ld_gout);
int interact_tc_bwd(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                    int64_t batch, const float* gout, int64_t ld_gout, int mask_f0,
                    cudaStream_t s);

namespace {
using namespace tcu;

constexpr int IA_EPI = 128;      // forward epilogue warps 0-3
constexpr uint32_t IA_TMEM_COLS = 512;
constexpr size_t IA_SMEM_MAX = 220 * 1024;

// host-computed forward tile geometry (passed by value)
struct IaGeom {
  int nf, d, S, R, P;
  int Rp;            // R rounded up to 16 (B rows, MMA N; lo lanes of A at Rp)
  int rows;          // rows per K-chunk region (= Rp)
  int kchunks;       // ceil(d / 32)
  int tma;           // 1: features are rows of one [batch * nf, d] matrix, loaded by TMA
  int nst;           // stages
  uint32_t stage_bytes;
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

__host__ __device__ constexpr uint32_t ceil_to32(int x) { return uint32_t((x + 31) & ~31); }

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// DLRM_IA_PROF builds (measurements only): clock64 cycles each role's
// first thread spends in each barrier wait, and its total, summed over CTAs
// (read with dlrm_ia_prof; scripts/ia_prof.py)
#ifdef DLRM_IA_PROF
__device__ unsigned long long g_ia_prof[24];
#define IB_WAIT(bar, par, k)                                   \
  do {                                                         \
    const long long t0_ = clock64();                           \
    mbar_wait(bar, par);                                       \
    prof[k] += (unsigned long long)(clock64() - t0_);          \
  } while (0)
#define IB_PROF_BEGIN const long long pt0_ = clock64();
#define IB_PROF_END(cond, k)                                                    \
  if (lane == 0 && (cond)) {                                                    \
    prof[k] += (unsigned long long)(clock64() - pt0_);                        \
    for (int i_ = 0; i_ < 24; ++i_)                                             \
      if (prof[i_]) atomicAdd(&g_ia_prof[i_], prof[i_]);                        \
  }
#define IB_PROF_DECL unsigned long long prof[24] = {0};
#else
#define IB_WAIT(bar, par, k) mbar_wait(bar, par)
#define IB_PROF_BEGIN
#define IB_PROF_END(cond, k)
#define IB_PROF_DECL
#endif

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
// Role profile at c4 (DLRM_IF_PROF, scripts/if_prof.py): splitters busy 94 %
// and epilogue 86 % of the kernel; eight splitter warps (two per lane
// quarter, half the columns each) cut the MMA's wait for them from 72k to
// 12k cycles per CTA but left the epilogue at 95 % busy and the kernel no
// faster (179 vs 172 us); eight splitter AND eight epilogue warps: 197 us,
// every role ~95 % busy — the SM's issue slots are the limit, so four each.
constexpr int IF_WARPS = 10;
constexpr int IF_THREADS = 32 * IF_WARPS;

#ifdef DLRM_IF_PROF
__device__ unsigned long long g_if_prof[16];
#define IF_WAIT(bar, par, k)                                  \
  do {                                                        \
    const long long t0_ = clock64();                          \
    mbar_wait(bar, par);                                      \
    ifp[k] += (unsigned long long)(clock64() - t0_);          \
  } while (0)
#define IF_FLUSH(k)                                                          \
  do {                                                                       \
    ifp[k] += (unsigned long long)(clock64() - ift0);                        \
    if (lane == 0)                                                           \
      for (int i_ = 0; i_ < 16; ++i_)                                        \
        if (ifp[i_]) atomicAdd(&g_if_prof[i_], ifp[i_]);                     \
  } while (0)
#else
#define IF_WAIT(bar, par, k) mbar_wait(bar, par)
#define IF_FLUSH(k)
#endif
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
#ifdef DLRM_IF_PROF
  unsigned long long ifp[16] = {0};
  const long long ift0 = clock64();
#endif
  auto piece = [&](uint8_t* base, int r, int p) {  // 16-byte piece p (4 floats) of row r
    return base + size_t(p >> 3) * Rp * 128 + r * 128 + (((p & 7) ^ (r & 7)) << 4);
  };

  if (warp == 9) {
    // ---- loader: the tile's R rows into stage it % nst
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % g.nst;
      if (it >= g.nst) IF_WAIT(&empty[st], ((it / g.nst) - 1) & 1, 0);
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
      IF_WAIT(&land[st], (it / g.nst) & 1, 2);
      if (it >= 2) IF_WAIT(&aempty[ab], ((it - 2) >> 1) & 1, 3);
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
        IF_WAIT(&land[st], (it / g.nst) & 1, 5);
        IF_WAIT(&afull[ab], (it >> 1) & 1, 6);
        if (it >= 2) IF_WAIT(&tempty[ab], ((it - 2) >> 1) & 1, 7);
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
      IF_WAIT(&tfull[ab], (it >> 1) & 1, 9);
      tc_fence_after();
      const bool valid = i >= 0 && i / nf < ns;
      // the window's column chunks (at most 4 of 16: Rp <= 64) loaded with
      // one wait instead of a load-wait round trip per chunk
      const int cb = lo_c & ~15;
      const int nch = (hi_c - cb + 15) >> 4;
      uint32_t v[4][16];
#pragma unroll
      for (int ch = 0; ch < 4; ++ch)
        if (ch < nch) tmem_ld16_issue(tmem + lane_off + uint32_t(64 * ab + cb + 16 * ch), v[ch]);
      tmem_wait_ld();
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        if (ch >= nch) break;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int j = cb + 16 * ch + k;
          if (valid && j >= blk && j < blk + nf) dst[i * nf + (j - blk)] = __uint_as_float(v[ch][k]);
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
#ifdef DLRM_IF_PROF
  if (warp == 9) IF_FLUSH(1);
  else if (warp == 4) IF_FLUSH(4);
  else if (warp == 8) IF_FLUSH(8);
  else if (warp == 0) { if (lane == 0) ifp[11] = 1; IF_FLUSH(10); }
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, IA_TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// backward (transposed form)
//
// g_i = [i==0] gout[:, :d] + sum_k M_ik z_k with M = G + G^T (zero diagonal)
// is computed per sample as D = Z^T M (D[n][i] = g_i[n]): the embedding dim n
// is the MMA's M dimension (TMEM lanes), so
//   A (TMEM) = Z^T split hi / lo: lane n, column k = feature k of the sample
//     (nfq = nf rounded up to 16 columns each, zero past nf), written by the
//     splitter warps from the landed Z tile (plain row-major rows of d floats);
//   B (smem, K-major 128B swizzle) = [M_hi ; M_lo] (2 nfq rows x 128 B per
//     sample; pad rows / columns and the diagonal stay zero), built by the
//     builder warps straight from gout[b, d + p];
//   D = [A_hi M_hi^T | A_hi M_lo^T + A_lo M_hi^T]: one N = 2 nfq MMA and one
//     N = nfq MMA per k-step, hh chain and small terms in separate columns;
// and the epilogue writes row i of sample b from lane n: every warp store is
// 32 consecutive floats of one gradient row.  For d < 128 the 128 / d
// samples of a lane group share A's columns at different lanes; each sample
// has its own B and D (the other lanes of its D are not read).
// Roles: warps 0-7 epilogue (TMEM lane quarter, half of the lane groups),
// 8-11 splitters (lane quarters), 12-15 builders, 16 MMA issuer + TMEM
// allocator, 17 TMA / cp.async loader.
constexpr int JB_EW = 8, JB_SPL = 8, JB_BLD = 12, JB_MMA = 16, JB_LD = 17;
constexpr int JB_THREADS = 32 * (JB_LD + 1);
constexpr int JB_BT = 32 * (JB_MMA - JB_BLD);  // builder threads
constexpr int JB_MAXV = 8;    // pair gradients per builder thread per tile
constexpr int JB_G0 = 4;      // gout[b, :d] values per builder thread per tile

struct IbGeom {
  int nf, d, P;
  int gg;          // samples per TMEM lane group (128 / d)
  int S, groups;   // samples per tile, lane groups per tile
  int nst;         // Z stages
  uint32_t zbytes; // Z stage bytes
  uint32_t bbytes; // B bytes per sample (2 nfq rows x 128 B)
  uint32_t a_base; // TMEM column of the A slots (after the two D buffers)
  uint32_t tmem_cols;
  uint32_t idesc2, idesc1;  // N = 2 nfq / N = nfq
  int tma;
};

// byte offset of element (row, k) of a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return uint32_t(row * 128 + ((((k >> 2) ^ (row & 7)) << 4) | ((k & 3) << 2)));
}

template <int NFQ>
__global__ void __launch_bounds__(JB_THREADS, 1)
interact_tc_bwd_kernel(const __grid_constant__ CUtensorMap tmZ, FeatureSet fs,
                       GradFeatureSet gs, IbGeom g, int64_t batch,
                       const float* __restrict__ gout, int64_t ld_gout, int mask_f0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* stages = smem;
  uint8_t* bslots = smem + size_t(g.nst) * g.zbytes;  // [2][S][bbytes]
  const uint32_t bslot_bytes = uint32_t(g.S) * g.bbytes;
  // per pair-gradient slot e = s * P + p of a tile: .x its offset in the
  // tile's gout rows, .y the byte offsets of M[i][j] | M[j][i] << 16 in the
  // sample's B (hi rows; the lo rows are NFQ * 128 bytes further)
  uint2* btab = reinterpret_cast<uint2*>(bslots + size_t(2) * bslot_bytes);
  // feature 0's extra terms of a tile (gout[b, :d] from the builders, z0 for
  // the mask from the splitters), 4 tiles deep: [4][S][d] each
  float* g0buf = reinterpret_cast<float*>(btab + g.S * g.P);
  float* z0buf = g0buf + 4 * g.S * g.d;
  uint64_t* bars = reinterpret_cast<uint64_t*>(z0buf + 4 * g.S * g.d);
  uint64_t* zfull = bars;         // [nst] Z tile landed
  uint64_t* zempty = bars + 4;    // [nst] splitters done with the Z tile
  uint64_t* afull = bars + 8;     // [2] A slot written (4 splitter warps)
  uint64_t* bfull = bars + 10;    // [2] B slot written (2 builder warps)
  uint64_t* opempty = bars + 12;  // [2] MMAs done with the A / B slots
  uint64_t* dfull = bars + 14;    // [2] D buffer ready
  uint64_t* dempty = bars + 16;   // [2] D buffer drained (8 epilogue warps)
  uint64_t* gzfull = bars + 18;   // [4] g0 / z0 of a tile staged
  uint64_t* gzempty = bars + 22;  // [4] the epilogue is done with them
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nf = g.nf, d = g.d, S = g.S, P = g.P;
  const int64_t ntiles = ceil_div(batch, S);
  const uint32_t dcols = uint32_t(S) * 2 * NFQ;          // one D buffer
  const uint32_t acols = uint32_t(g.groups) * 2 * NFQ;   // one A slot

  for (int e = threadIdx.x; e < S * P; e += blockDim.x) {
    const int s = e / P, p = e - s * P;
    int pi, pj;
    ia_pair(p, nf, pi, pj);
    const uint32_t base = uint32_t(s) * g.bbytes;
    btab[e] = make_uint2(uint32_t(s * ld_gout + d + p),
                         (base + sw128_off(pi, pj)) | ((base + sw128_off(pj, pi)) << 16));
  }
  // B slots: zero once (pad rows / columns and the diagonal are never written)
  for (uint32_t e = threadIdx.x; e < 2 * bslot_bytes / 16; e += blockDim.x)
    reinterpret_cast<float4*>(bslots)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
  fence_async_smem();
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.nst; ++s) {
      mbar_init(&zfull[s], g.tma ? 1 : 32);
      mbar_init(&zempty[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 4);
      mbar_init(&bfull[b], JB_BT / 32);
      mbar_init(&opempty[b], 1);
      mbar_init(&dfull[b], 1);
      mbar_init(&dempty[b], JB_EW);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&gzfull[b], 4 + JB_BT / 32);
      mbar_init(&gzempty[b], JB_EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == JB_MMA) tmem_alloc_warp(tmem_slot, g.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  IB_PROF_DECL
  IB_PROF_BEGIN

  if (warp == JB_LD) {
    // ---- loader: the tile's S * nf feature rows, row-major, d floats each
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % g.nst;
      if (it >= g.nst) IB_WAIT(&zempty[st], ((it / g.nst) - 1) & 1, 0);
      uint8_t* zs = stages + size_t(st) * g.zbytes;
      const int64_t b0 = tile * S;
      if (g.tma) {
        if (lane == 0) {  // rows past the batch: zeros
          mbar_expect_tx(&zfull[st], uint32_t(S * nf * d * 4));
          tma_load_2d(zs, &tmZ, &zfull[st], 0, int(b0 * nf));
        }
      } else {
        const int ns = int(batch - b0 < S ? batch - b0 : S);
        const int nv = d / 4;
        for (int e = lane; e < ns * nf * nv; e += 32) {
          const int r = e / nv, p = e - r * nv, sm = r / nf, f = r - sm * nf;
          cp_async16(zs + (size_t(r) * d + 4 * p) * 4, fs.feat[f] + (b0 + sm) * fs.stride[f] + 4 * p,
                     true);
        }
        cp_async_commit();
        cp_async_wait<0>();
        mbar_arrive(&zfull[st]);
      }
    }
  } else if (warp >= JB_SPL && warp < JB_SPL + 4) {
    // ---- splitters: A lane L = (sample L / d of the group, dim L % d)
    const int q = warp - JB_SPL, L = 32 * q + lane, sl = L / d, n = L - sl * d;
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int st = it % g.nst, ab = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      IB_WAIT(&zfull[st], (it / g.nst) & 1, 1);
      if (it >= 2) IB_WAIT(&opempty[ab], ((it - 2) >> 1) & 1, 2);
      tc_fence_after();
      const float* zs = reinterpret_cast<const float*>(stages + size_t(st) * g.zbytes);
      const uint32_t slot = tmem + lane_off + g.a_base + uint32_t(ab) * acols;
      if (it >= 4) IB_WAIT(&gzempty[it & 3], ((it - 4) >> 2) & 1, 9);
      float* z0s = z0buf + (it & 3) * S * d;
      for (int gi = 0; gi < g.groups && gi * g.gg < ns; ++gi) {
        const int s = gi * g.gg + sl;
        if (s >= ns) continue;  // warp-uniform (d >= 32)
        const float* zr = zs + size_t(s) * nf * d + n;
        if (mask_f0) z0s[s * d + n] = zr[0];
#pragma unroll
        for (int c0 = 0; c0 < NFQ; c0 += 16) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float x = c0 + k < nf ? zr[(c0 + k) * d] : 0.f;
            hi[k] = __float_as_uint(x) & 0xFFFFE000u;
            lo[k] = tf32_rna(x - __uint_as_float(hi[k]));
          }
          tmem_st16(slot + uint32_t(gi * 2 * NFQ + c0), hi);
          tmem_st16(slot + uint32_t(gi * 2 * NFQ + NFQ + c0), lo);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&zempty[st]);
        mbar_arrive(&afull[ab]);
        mbar_arrive(&gzfull[it & 3]);
      }
    }
  } else if (warp >= JB_BLD && warp < JB_MMA) {
    // ---- builders: [M_hi ; M_lo] of each sample from its pair gradients;
    // two register sets, so one tile's gradients load while the previous
    // tile's are stored
    const int t = threadIdx.x - 32 * JB_BLD;
    float va[JB_MAXV + JB_G0], vb[JB_MAXV + JB_G0];
    auto load = [&](int64_t tile, float* v) {
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const float* src = gout + b0 * ld_gout;
#pragma unroll
      for (int k = 0; k < JB_MAXV; ++k) {
        const int e = t + JB_BT * k;
        v[k] = e < ns * P ? __ldg(src + btab[e].x) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < JB_G0; ++k) {  // gout[b, :d]
        const int e = t + JB_BT * k, sm = e / d;
        v[JB_MAXV + k] = e < ns * d ? __ldg(src + sm * ld_gout + (e - sm * d)) : 0.f;
      }
    };
    auto store = [&](int it, int64_t tile, const float* v) {
      const int ab = it & 1;
      const int64_t b0 = tile * S;
      const int nsp = int(batch - b0 < S ? batch - b0 : S) * P;
      if (it >= 2) IB_WAIT(&opempty[ab], ((it - 2) >> 1) & 1, 3);
      uint8_t* bs = bslots + size_t(ab) * bslot_bytes;
#pragma unroll
      for (int k = 0; k < JB_MAXV; ++k) {
        const int e = t + JB_BT * k;
        if (e < nsp) {
          const uint32_t o = btab[e].y, o1 = o & 0xffffu, o2 = o >> 16;
          const uint32_t h = __float_as_uint(v[k]) & 0xFFFFE000u;
          const uint32_t l = tf32_rna(v[k] - __uint_as_float(h));
          *reinterpret_cast<uint32_t*>(bs + o1) = h;
          *reinterpret_cast<uint32_t*>(bs + o2) = h;
          *reinterpret_cast<uint32_t*>(bs + o1 + NFQ * 128) = l;
          *reinterpret_cast<uint32_t*>(bs + o2 + NFQ * 128) = l;
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bfull[ab]);
      if (it >= 4) IB_WAIT(&gzempty[it & 3], ((it - 4) >> 2) & 1, 10);
      float* g0s = g0buf + (it & 3) * S * d;
#pragma unroll
      for (int k = 0; k < JB_G0; ++k) {
        const int e = t + JB_BT * k;
        if (e < nsp / P * d) g0s[e] = v[JB_MAXV + k];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&gzfull[it & 3]);
    };
    int it = 0;
    int64_t tile = blockIdx.x;
    if (tile < ntiles) load(tile, va);
    while (tile < ntiles) {
      if (tile + gridDim.x < ntiles) load(tile + gridDim.x, vb);
      store(it++, tile, va);
      tile += gridDim.x;
      if (tile >= ntiles) break;
      if (tile + gridDim.x < ntiles) load(tile + gridDim.x, va);
      store(it++, tile, vb);
      tile += gridDim.x;
    }
  } else if (warp == JB_MMA) {
    // ---- MMA issuer
    if (lane == 0) {
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int ab = it & 1;
        const int64_t b0 = tile * S;
        const int ns = int(batch - b0 < S ? batch - b0 : S);
        IB_WAIT(&afull[ab], (it >> 1) & 1, 4);
        IB_WAIT(&bfull[ab], (it >> 1) & 1, 5);
        if (it >= 2) IB_WAIT(&dempty[ab], ((it - 2) >> 1) & 1, 6);
        tc_fence_after();
        const uint32_t bbase = smem_u32(bslots + size_t(ab) * bslot_bytes);
        for (int s = 0; s < ns; ++s) {
          const uint32_t a_hi = tmem + g.a_base + uint32_t(ab) * acols + uint32_t(s / g.gg) * 2 * NFQ;
          const uint32_t dt = tmem + uint32_t(ab) * dcols + uint32_t(s) * 2 * NFQ;
          const uint32_t bb = bbase + uint32_t(s) * g.bbytes;
#pragma unroll
          for (int ks = 0; ks < NFQ / 8; ++ks) {
            const uint64_t bd = smem_desc(bb + uint32_t(32 * ks), 16, 1024, 2);
            mma_tf32_ts(dt, a_hi + uint32_t(8 * ks), bd, g.idesc2, ks > 0 ? 1u : 0u);
            mma_tf32_ts(dt + NFQ, a_hi + NFQ + uint32_t(8 * ks), bd, g.idesc1, 1u);
          }
        }
        mma_commit(&opempty[ab]);
        mma_commit(&dfull[ab]);
      }
    }
  } else if (warp < JB_EW) {
    // ---- epilogue: lane L of D = dim n of sample (group gi, L / d); this
    // warp takes the groups gi = h, h + 2
    const int q = warp & 3, h = warp >> 2, L = 32 * q + lane, sl = L / d, n = L - sl * d;
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int ab = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      IB_WAIT(&dfull[ab], (it >> 1) & 1, 7);
      IB_WAIT(&gzfull[it & 3], (it >> 2) & 1, 11);
      const float* g0s = g0buf + (it & 3) * S * d;
      const float* z0s = z0buf + (it & 3) * S * d;
      tc_fence_after();
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int s = (h + 2 * u) * g.gg + sl;
        if (h + 2 * u >= g.groups || s >= ns) continue;  // warp-uniform
        const uint32_t dt = tmem + lane_off + uint32_t(ab) * dcols + uint32_t(s) * 2 * NFQ;
        uint32_t hh[NFQ], sm[NFQ];
#pragma unroll
        for (int c0 = 0; c0 < NFQ; c0 += 16) {
          tmem_ld16_issue(dt + uint32_t(c0), hh + c0);
          tmem_ld16_issue(dt + uint32_t(NFQ + c0), sm + c0);
        }
        tmem_wait_ld();
        const int64_t b = b0 + s;
#pragma unroll
        for (int f = 0; f < NFQ; ++f) {
          if (f < nf) {
            float v = __uint_as_float(hh[f]) + __uint_as_float(sm[f]);
            if (f == 0) {
              v = g0s[s * d + n] + v;
              if (mask_f0) v *= z0s[s * d + n] > 0.f ? 1.f : 0.f;
            }
            gs.feat[f][b * gs.stride[f] + n] = v;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&dempty[ab]);
        mbar_arrive(&gzempty[it & 3]);
      }
    }
  }
  IB_PROF_END(warp == JB_LD || warp == JB_SPL || warp == JB_BLD || warp == JB_MMA || warp == 0,
              16 + (warp == JB_LD ? 0 : warp == JB_SPL ? 1 : warp == JB_BLD ? 2 : warp == JB_MMA ? 3 : 4))
  tc_fence_before();
  __syncthreads();
  if (warp == JB_MMA) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, g.tmem_cols);
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

bool bwd_geom(int nf, int d, IbGeom* g) {
  // lanes = the embedding dim: d in {32, 64, 128}; nf <= 32 (one K block)
  if (nf < 2 || nf > 32 || d < 32 || d > 128 || 128 % d) return false;
  const int P = nf * (nf - 1) / 2;
  const int nfq = nf <= 16 ? 16 : 32, gg = 128 / d;
  for (int S = 8; S >= 1; --S) {
    const int groups = (S + gg - 1) / gg;
    const uint32_t cols = uint32_t(2 * S * 2 * nfq + 2 * groups * 2 * nfq);
    if (groups > 4 || cols > IA_TMEM_COLS || S * P > JB_BT * JB_MAXV || S * d > JB_BT * JB_G0 ||
        S * 2 * nfq * 128 > 65536)
      continue;
    const uint32_t zbytes = ceil_to(uint32_t(S * nf * d * 4), 1024);
    const uint32_t bbytes = uint32_t(2 * nfq * 128);
    const size_t fixed = 1024 + size_t(2) * S * bbytes + size_t(S) * P * 8 + size_t(32) * S * d +
                         32 * 8;
    int nst = int((IA_SMEM_MAX - fixed) / zbytes);
    if (nst > 4) nst = 4;
    if (nst < 2) continue;
    uint32_t tc = 32;
    while (tc < cols) tc *= 2;
    *g = IbGeom{};
    g->nf = nf; g->d = d; g->P = P; g->gg = gg; g->S = S; g->groups = groups; g->nst = nst;
    g->zbytes = zbytes; g->bbytes = bbytes; g->a_base = uint32_t(2 * S * 2 * nfq);
    g->tmem_cols = tc;
    g->idesc2 = instr_desc(2 * nfq, false, false);
    g->idesc1 = instr_desc(nfq, false, false);
    return true;
  }
  return false;
}

size_t fwd_smem(const IaGeom& g) {
  return 1024 + size_t(g.nst) * g.stage_bytes + size_t(2) * g.R * g.nf * 4 + size_t(g.P) * 4 +
         8 + 24 * 8;
}
size_t bwd_smem(const IbGeom& g) {
  return 1024 + size_t(g.nst) * g.zbytes + size_t(2) * g.S * g.bbytes + size_t(g.S) * g.P * 8 +
         size_t(32) * g.S * g.d + 32 * 8;
}

// features f at feat[0] + f*d with row stride nf*d (the training engine's
// [B, nf, d] buffer): the tile rows are consecutive rows of one matrix
bool uniform_rows(const FeatureSet& fs, int nf, int64_t dim) {
  if (dim % 32 || getenv("DLRM_IA_NO_TMA")) return false;
  for (int f = 0; f < nf; ++f)
    if (fs.feat[f] != fs.feat[0] + f * dim || fs.stride[f] != nf * dim) return false;
  return true;
}

// Default dispatch (scripts/ia_matrix.py, profiles/round2/ia_matrix.jsonl):
// the SIMT kernels cost ~pairs x d FMAs per sample, the tensor-core ones
// are bound by their per-tile data movement.  With many features (nf = 27,
// d >= 64: Criteo-shaped) the tensor cores win at every batch (1.5-1.8x at
// d = 128); with few (nf = 9, 36 pairs: the Big Basin shape) or narrow rows
// (d = 32) the SIMT kernels are faster at every batch.  So: tensor cores
// when nf (nf - 1) / 2 >= 100 and d >= 64; dlrm_gemm_mode(2) forces them,
// DLRM_IA_SIMT (or mode 1) disables them.
bool tc_ia_enabled(int nf, int64_t dim) {
  static const bool off = getenv("DLRM_IA_SIMT") != nullptr;
  if (off || !tc_enabled()) return false;
  return tc_mode() == 2 || (nf * (nf - 1) / 2 >= 100 && dim >= 64);
}

}  // namespace

bool interact_tc_fwd_ok(const FeatureSet& fs, int nf, int64_t dim, int64_t batch,
                        int64_t ld_out, const float* out) {
  IaGeom g;
  (void)batch;
  if (!tc_ia_enabled(nf, dim) || !fwd_geom(nf, int(dim), &g)) return false;
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
                        int64_t batch, const float* gout, int64_t ld_gout) {
  IbGeom g;
  (void)batch;
  if (!tc_ia_enabled(nf, dim) || !bwd_geom(nf, int(dim), &g)) return false;
  if (reinterpret_cast<uintptr_t>(gout) % 16 || ld_gout % 4) return false;
  for (int f = 0; f < nf; ++f)
    if (reinterpret_cast<uintptr_t>(fs.feat[f]) % 16 || fs.stride[f] % 4) return false;
  (void)gs;  // gradient rows are written with 4-byte stores
  return true;
}

int interact_tc_bwd(const FeatureSet& fs, const GradFeatureSet& gs, int nf, int64_t dim,
                    int64_t batch, const float* gout, int64_t ld_gout, int mask_f0,
                    cudaStream_t s) {
  IbGeom g;
  DLRM_REQUIRE(bwd_geom(nf, int(dim), &g), "interaction shape not supported by tcgen05 path");
  const size_t smem = bwd_smem(g);
  auto k = nf <= 16 ? interact_tc_bwd_kernel<16> : interact_tc_bwd_kernel<32>;
  static bool configured[2] = {false, false};
  if (!configured[nf > 16]) {
    DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(IA_SMEM_MAX + 4096)));
    configured[nf > 16] = true;
  }
  CUtensorMap tm{};
  g.tma = uniform_rows(fs, nf, dim) &&
          tma_encode_2d(&tm, fs.feat[0], dim, batch * nf, dim, int(dim), g.S * nf, 0);
  const int64_t ntiles = ceil_div(batch, g.S);
  const unsigned grid = unsigned(ntiles < kNumSMs ? ntiles : kNumSMs);
  launch(k, grid, JB_THREADS, smem, s, tm, fs, gs, g, batch, gout, ld_gout, mask_f0);
  return check_launch("interact_tc_bwd_kernel");
}

}  // namespace dlrm

#ifdef DLRM_IA_PROF
extern "C" int dlrm_ia_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dlrm::g_ia_prof, sizeof(unsigned long long) * 24);
  static const unsigned long long zero[24] = {0};
  cudaMemcpyToSymbol(dlrm::g_ia_prof, zero, sizeof(zero));
  return 0;
}
#endif

#ifdef DLRM_IF_PROF
extern "C" int dlrm_if_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, dlrm::g_if_prof, sizeof(unsigned long long) * 16);
  static const unsigned long long zero[16] = {0};
  cudaMemcpyToSymbol(dlrm::g_if_prof, zero, sizeof(zero));
  return 0;
}
#endif
