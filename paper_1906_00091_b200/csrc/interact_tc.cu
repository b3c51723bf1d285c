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

// ablation switches for measurements (scripts/build_variant.py): 1 = no
// epilogue work, 2 = no MMAs, 3 = no lo split, 4 = no output stores
#ifndef DLRM_IA_ABL
#define DLRM_IA_ABL 0
#endif
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

// DLRM_IA_PROF builds (measurements only): clock64 time per role / phase of
// the forward kernel, summed over CTAs, read with dlrm_ia_prof()
#ifdef DLRM_IA_PROF
__device__ unsigned long long g_ia_prof[32];
#define IA_TIC(n) const long long _tic##n = clock64();
#define IA_TOC(n, k) pc[k] += (unsigned long long)(clock64() - _tic##n);
#else
#define IA_TIC(n)
#define IA_TOC(n, k)
#endif

#ifndef DLRM_IA_LOADER_WARPS
#define DLRM_IA_LOADER_WARPS 4
#endif
constexpr int IA_LW = DLRM_IA_LOADER_WARPS;  // loader warps 4 .. 4 + IA_LW - 1
constexpr int IA_MMA_WARP = 4 + IA_LW;
constexpr int IA_WARPS = IA_MMA_WARP + 1;
constexpr int IA_THREADS = 32 * IA_WARPS;
constexpr int IA_LOADERS = 32 * IA_LW;
constexpr int IA_EPI = 128;      // warps 0-3
constexpr uint32_t IA_TMEM_COLS = 512;
constexpr size_t IA_SMEM_MAX = 220 * 1024;

// host-computed tile geometry (passed by value)
struct IaGeom {
  int nf, d, S, R, P;
  int Pp;            // bwd: P rounded up to 4 (pair-gradient row pitch)
  int Rp;            // R rounded up to 8 (fwd: B rows of one operand half)
  int rows;          // fwd: rows per K-chunk region, max(2 Rp, 128)
  int kchunks;       // fwd: ceil(d / 32)
  int Kq;            // bwd: R rounded up to 16 (A slot columns)
  int Kp;            // bwd: R rounded up to 8 (MMA K)
  int nst;           // stages
  uint32_t stage_bytes;
  uint32_t b_bytes;  // bwd: operand bytes of a stage (the rest: pair gradients)
  uint32_t a_base;   // bwd: TMEM column of the A slots
  uint32_t idesc, idesc2;
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
#define DLRM_IA_AHEAD 2
#endif
constexpr int IA_AHEAD = DLRM_IA_AHEAD;

template <class Issue, class Finish>
__device__ __forceinline__ void ia_pipeline(int64_t ntiles, int nst, Issue issue, Finish finish,
                                            unsigned long long* pc = nullptr) {
  (void)pc;
  const int ahead = nst - 1 < IA_AHEAD ? nst - 1 : IA_AHEAD;
  int issued = 0;
  int64_t next = blockIdx.x;
  for (; issued < ahead && next < ntiles; ++issued, next += gridDim.x) issue(issued, next);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    if (next < ntiles) {
      issue(issued++, next);
      next += gridDim.x;
    }
    // groups still allowed in flight: the ones issued after tile `it`
    const int pending = issued - it - 1;
    IA_TIC(w)
    if (pending >= 3) cp_async_wait<3>();
    else if (pending >= 2) cp_async_wait<2>();
    else if (pending == 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    IA_TOC(w, 2)
    finish(it, tile);
  }
}

// ---------------------------------------------------------------------------
// forward
//
// Stage: kchunks regions of `rows` x 128 B (K-major, 128B swizzle: 16-byte
// piece j of row r at (j ^ (r & 7))); Z rows at [0, R), lo rows at [Rp, Rp+R).
// TMEM: two D buffers of 256 columns (tile it in buffer it % 2).
__global__ void __launch_bounds__(IA_THREADS, 1)
interact_tc_fwd_kernel(FeatureSet fs, IaGeom g, int64_t batch, float* __restrict__ out,
                       int64_t ld_out, int64_t pad_to) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* stages = smem;
  float* H = reinterpret_cast<float*>(smem + size_t(g.nst) * g.stage_bytes);  // [R][nf]
  float* X = H + g.R * g.nf;                                                   // [R][nf]
  int* pairs = reinterpret_cast<int*>(X + g.R * g.nf);                         // [P]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(pairs + g.P) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;                 // [nst] loaders done (128 arrivals)
  uint64_t* empty = bars + 4;            // [nst] MMA done with the stage
  uint64_t* tfull = bars + 8;            // [2] D buffer ready
  uint64_t* tempty = bars + 10;          // [2] D buffer drained (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nf = g.nf, d = g.d, S = g.S;
  const int64_t ntiles = ceil_div(batch, S);

  for (int p = threadIdx.x; p < g.P; p += blockDim.x) {
    int i, j;
    ia_pair(p, nf, i, j);
    pairs[p] = (i << 16) | j;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < g.nst; ++s) {
      mbar_init(&full[s], IA_LOADERS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == IA_MMA_WARP) tmem_alloc_warp(tmem_slot, IA_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  unsigned long long pc[16] = {0};
  IA_TIC(all)

  if (warp >= 4 && warp < IA_MMA_WARP) {
    // ---- loaders: raw rows by cp.async (IA_AHEAD tiles in flight), then the
    // lo rows and the z0 / pad columns of the output of the oldest landed
    // tile.  One warp per feature row, one 16-byte piece per lane.
    const int lw = warp - 4;
    const int nv = d / 4;
    auto piece = [&](uint8_t* base, int r, int p) {
      return base + size_t(p >> 3) * g.rows * 128 + r * 128 + (((p & 7) ^ (r & 7)) << 4);
    };
    auto issue = [&](int it, int64_t tile) {
      const int st = it % g.nst;
      IA_TIC(e)
      if (it >= g.nst) mbar_wait(&empty[st], ((it / g.nst) - 1) & 1);
      IA_TOC(e, 0)
      IA_TIC(i)
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      for (int s = 0; s < ns; ++s)
        for (int f = lw; f < nf; f += IA_LW) {
          const int r = s * nf + f;
          const float* src = fs.feat[f] + (b0 + s) * fs.stride[f];
          for (int p = lane; p < nv; p += 32) cp_async16(piece(base, r, p), src + 4 * p, true);
        }
      cp_async_commit();
      IA_TOC(i, 1)
    };
    const int W = d + g.P;
    const int tw = int(pad_to > W ? pad_to : W);
    auto finish = [&](int it, int64_t tile) {
      const int st = it % g.nst;
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      IA_TIC(b)
      named_bar(1, IA_LOADERS);  // every loader's copies of this tile landed
      IA_TOC(b, 3)
      IA_TIC(l)
      for (int r = lw; r < (DLRM_IA_ABL == 3 ? 0 : ns * nf); r += IA_LW)
        for (int p = lane; p < nv; p += 32) {
          uint8_t* src = piece(base, r, p);
          *reinterpret_cast<float4*>(src + g.Rp * 128) = split_lo4(*reinterpret_cast<float4*>(src));
        }
      fence_async_smem();
      mbar_arrive(&full[st]);
      IA_TOC(l, 4)
      IA_TIC(z)
      // output columns [0, d) (z0, exact copy) and the zero pad [W, tw)
      for (int s = lw; s < ns; s += IA_LW) {
        float* orow = out + (b0 + s) * ld_out;
        for (int p = lane; p < nv; p += 32)
          *reinterpret_cast<float4*>(orow + 4 * p) =
              *reinterpret_cast<const float4*>(piece(base, s * nf, p));
        for (int c = W + lane; c < tw; c += 32) orow[c] = 0.f;
      }
      IA_TOC(z, 5)
    };
    ia_pipeline(ntiles, g.nst, issue, finish, pc);
  } else if (warp == IA_MMA_WARP) {
    // ---- MMA issuer
    if (lane == 0) {
      const int ksteps = d / 8;
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % g.nst, buf = it & 1;
        IA_TIC(f)
        mbar_wait(&full[st], (it / g.nst) & 1);
        IA_TOC(f, 6)
        IA_TIC(t)
        if (it >= 2) mbar_wait(&tempty[buf], ((it - 2) >> 1) & 1);
        IA_TOC(t, 7)
        tc_fence_after();
        const uint32_t dt = tmem + uint32_t(256 * buf);
        const uint32_t base = smem_u32(stages + size_t(st) * g.stage_bytes);
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint32_t a = base + uint32_t((ks >> 2) * g.rows * 128 + (ks & 3) * 32);
          const uint64_t desc = smem_desc(a, 16, 1024, 2);
          if (DLRM_IA_ABL != 2) mma_tf32_ss(dt, desc, desc, g.idesc, ks > 0 ? 1u : 0u);
        }
        mma_commit(&empty[st]);
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ---- epilogue (warps 0-3 = TMEM lane quarters)
    const int q = warp;
    const int i = 32 * q + lane;  // tile row
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const int rv = ns * nf;  // valid rows
      IA_TIC(q)
      mbar_wait(&tfull[buf], (it >> 1) & 1);
      IA_TOC(q, 9)
      IA_TIC(m)
      tc_fence_after();
      if (DLRM_IA_ABL != 1 && 32 * q < rv) {
        const int r_hi = 32 * q + 31 < rv - 1 ? 32 * q + 31 : rv - 1;
        const int c_lo = ((32 * q) / nf * nf) & ~15, c_end = (r_hi / nf + 1) * nf;
        const int blk = (i / nf) * nf;
        const bool valid = i < rv;
        const uint32_t lrow = tmem + (uint32_t(32 * q) << 16) + uint32_t(256 * buf);
        for (int c0 = c_lo; c0 < c_end; c0 += 16) {
          uint32_t hv[16], xv[16];
          tmem_ld16_issue(lrow + uint32_t(c0), hv);
          tmem_ld16_issue(lrow + uint32_t(g.Rp + c0), xv);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int j = c0 + k;
            if (valid && j >= blk && j < blk + nf) {
              H[i * nf + (j - blk)] = __uint_as_float(hv[k]);
              X[i * nf + (j - blk)] = __uint_as_float(xv[k]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      IA_TOC(m, 10)
      IA_TIC(c)
      named_bar(2, IA_EPI);
      IA_TOC(c, 11)
      IA_TIC(o)
      // pair columns [d, d + P) of the tile's rows (z0 and the pad were
      // written by the loaders)
      for (int s = 0; s < (DLRM_IA_ABL == 1 || DLRM_IA_ABL == 4 ? 0 : ns); ++s) {
        float* orow = out + (b0 + s) * ld_out + d;
        const float* Hs = H + s * nf * nf;
        const float* Xs = X + s * nf * nf;
        for (int p = threadIdx.x; p < g.P; p += IA_EPI) {
          const int pr = pairs[p], pi = pr >> 16, pj = pr & 0xffff;
          orow[p] = (Hs[pi * nf + pj] + Xs[pi * nf + pj]) + Xs[pj * nf + pi];
        }
      }
      IA_TOC(o, 12)
      named_bar(2, IA_EPI);
    }
  }
#ifdef DLRM_IA_PROF
  IA_TOC(all, 15)
  if (lane == 0 && (warp == 0 || warp == 4 || warp == IA_MMA_WARP))
    for (int k = 0; k < 16; ++k)
      if (pc[k]) atomicAdd(&g_ia_prof[k + (k == 15 ? (warp == 0 ? 0 : warp == 4 ? 1 : 2) : 0)], pc[k]);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == IA_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, IA_TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// backward
//
// Stage: the B operand [Z | Z_lo] MN-major (SWIZZLE_128B_BASE32B: 32-wide
// column chunks of Kp rows x 128 B, 32-byte atom a of row k at (a ^ (k & 3));
// Z columns [0, d), lo columns [d, 2d)), rows past the valid samples zero;
// then the tile's pair gradients gout[b, d + p] (S x P floats).
// TMEM: D = [hh | small] (2d columns), then two A slots [A_hi | A_lo] of Kq
// columns each from a_base.
__device__ __forceinline__ uint32_t mn_off(int k, int n) {
  // byte offset of element (k, n) inside the chunk set (without chunk stride)
  return uint32_t(k * 128 + ((((n & 31) >> 3) ^ (k & 3)) << 5) + ((n & 7) << 2));
}

__global__ void __launch_bounds__(IA_THREADS, 1)
interact_tc_bwd_kernel(FeatureSet fs, GradFeatureSet gs, IaGeom g, int64_t batch,
                       const float* __restrict__ gout, int64_t ld_gout, int mask_f0) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* stages = smem;
  // [R][d + 4]: the pitch keeps each 8-lane phase of the row-per-lane float4
  // stores on distinct banks
  const int yp = g.d + 4;
  float* Y = reinterpret_cast<float*>(smem + size_t(g.nst) * g.stage_bytes);
  float* G0 = Y + size_t(g.R) * yp;       // [S][d] gout[b, :d] of the tile
  float* Z0 = G0 + size_t(g.S) * g.d;     // [S][d] z0 of the tile (mask)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Z0 + size_t(g.S) * g.d);
  uint64_t* full = bars;       // [nst] (128 loader arrivals)
  uint64_t* empty = bars + 4;  // [nst]
  uint64_t* afull = bars + 8;  // [2] A slot built (4 warps)
  uint64_t* aempty = bars + 10;  // [2] A slot consumed
  uint64_t* dfull = bars + 12;
  uint64_t* dempty = bars + 13;  // (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nf = g.nf, d = g.d, S = g.S, P = g.P, Pp = g.Pp;
  const int64_t ntiles = ceil_div(batch, S);
  const uint32_t lbo = uint32_t(g.Kp) * 128;  // column-chunk stride

  if (threadIdx.x == 0) {
    for (int s = 0; s < g.nst; ++s) {
      mbar_init(&full[s], IA_LOADERS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&afull[b], 4);
      mbar_init(&aempty[b], 1);
    }
    mbar_init(dfull, 1);
    mbar_init(dempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == IA_MMA_WARP) tmem_alloc_warp(tmem_slot, IA_TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp >= 4 && warp < IA_MMA_WARP) {
    // ---- loaders (IA_AHEAD tiles in flight)
    const int t = threadIdx.x - 128, lw = warp - 4;
    const int nv = d / 4;
    const int pv = P / 4, prem = P - 4 * pv;
    const bool g16 = (reinterpret_cast<uintptr_t>(gout) % 16) == 0 && ld_gout % 4 == 0 &&
                     d % 4 == 0;
    auto issue = [&](int it, int64_t tile) {
      const int st = it % g.nst;
      if (it >= g.nst) mbar_wait(&empty[st], ((it / g.nst) - 1) & 1);
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      float* gp = reinterpret_cast<float*>(base + g.b_bytes);
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const int rv = ns * nf;
      // Z rows, one warp per row, a 16-byte piece per lane (zero past the
      // valid rows: the block-diagonal A is zero there, and 0 * garbage
      // could be NaN)
      for (int r = lw; r < g.Kp; r += IA_LW) {
        const bool ok = r < rv;
        const int s = ok ? r / nf : 0, f = ok ? r - s * nf : 0;
        const float* src = fs.feat[f] + (b0 + s) * fs.stride[f];
        for (int p = lane; p < nv; p += 32) {
          const int n = 4 * p;
          cp_async16(base + size_t(n >> 5) * lbo + mn_off(r, n), ok ? src + n : fs.feat[0], ok);
        }
      }
      // pair gradients of the tile's samples
      for (int s = 0; s < ns; ++s) {
        const float* src = gout + (b0 + s) * ld_gout + d;
        if (g16) {
          for (int e = t; e < pv; e += IA_LOADERS) cp_async16(gp + s * Pp + 4 * e, src + 4 * e, true);
          for (int e = t; e < prem; e += IA_LOADERS) gp[s * Pp + 4 * pv + e] = __ldg(src + 4 * pv + e);
        } else {
          for (int e = t; e < P; e += IA_LOADERS) gp[s * Pp + e] = __ldg(src + e);
        }
      }
      cp_async_commit();
    };
    auto finish = [&](int it, int64_t tile) {
      (void)tile;
      const int st = it % g.nst;
      uint8_t* base = stages + size_t(st) * g.stage_bytes;
      named_bar(1, IA_LOADERS);
      // lo columns [d, 2d)
      for (int r = lw; r < g.Kp; r += IA_LW)
        for (int p = lane; p < nv; p += 32) {
          const int n = 4 * p, nl = d + n;
          const float4 v = *reinterpret_cast<const float4*>(base + size_t(n >> 5) * lbo + mn_off(r, n));
          *reinterpret_cast<float4*>(base + size_t(nl >> 5) * lbo + mn_off(r, nl)) = split_lo4(v);
        }
      fence_async_smem();
      mbar_arrive(&full[st]);
    };
    ia_pipeline(ntiles, g.nst, issue, finish);
  } else if (warp == IA_MMA_WARP) {
    // ---- MMA issuer
    if (lane == 0) {
      const int ksteps = g.Kp / 8;
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % g.nst, ab = it & 1;
        mbar_wait(&full[st], (it / g.nst) & 1);
        mbar_wait(&afull[ab], (it >> 1) & 1);
        if (it >= 1) mbar_wait(dempty, (it - 1) & 1);
        tc_fence_after();
        const uint32_t base = smem_u32(stages + size_t(st) * g.stage_bytes);
        const uint32_t a_hi = tmem + g.a_base + uint32_t(2 * g.Kq * ab), a_lo = a_hi + g.Kq;
        const uint32_t hh = tmem, small = tmem + uint32_t(d);
        // the small terms first (own columns), then the hi x hi chain
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t braw = smem_desc(base + uint32_t(ks * 1024), lbo, 512, 1);
          const uint64_t blo = smem_desc(base + uint32_t(ks * 1024) + uint32_t(d / 32) * lbo +
                                             uint32_t(d % 32 ? 64 : 0),
                                         lbo, 512, 1);
          mma_tf32_ts(small, a_lo + uint32_t(8 * ks), braw, g.idesc, ks > 0 ? 1u : 0u);
          mma_tf32_ts(small, a_hi + uint32_t(8 * ks), blo, g.idesc, 1u);
        }
        for (int ks = 0; ks < ksteps; ++ks) {
          const uint64_t braw = smem_desc(base + uint32_t(ks * 1024), lbo, 512, 1);
          mma_tf32_ts(hh, a_hi + uint32_t(8 * ks), braw, g.idesc, ks > 0 ? 1u : 0u);
        }
        mma_commit(&empty[st]);
        mma_commit(&aempty[ab]);
        mma_commit(dfull);
      }
    }
  } else {
    // ---- A builder + epilogue (warps 0-3 = TMEM lane quarters)
    const int q = warp;
    const int i = 32 * q + lane;
    const uint32_t lane_off = uint32_t(32 * q) << 16;
    auto build = [&](int it, int64_t tile) {
      const int st = it % g.nst, ab = it & 1;
      mbar_wait(&full[st], (it / g.nst) & 1);
      if (it >= 2) mbar_wait(&aempty[ab], ((it - 2) >> 1) & 1);
      tc_fence_after();
      const float* gp =
          reinterpret_cast<const float*>(stages + size_t(st) * g.stage_bytes + g.b_bytes);
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const bool valid = i < ns * nf;
      const int s = i / nf, fi = i - s * nf, blk = s * nf;
      const uint32_t slot = tmem + lane_off + g.a_base + uint32_t(2 * g.Kq * ab);
      for (int c0 = 0; c0 < g.Kq; c0 += 16) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int fk = c0 + k - blk;
          float m = 0.f;
          if (valid && fk >= 0 && fk < nf && fk != fi) {
            const int a = fi < fk ? fi : fk, b = fi < fk ? fk : fi;
            m = gp[s * Pp + a * (2 * nf - a - 1) / 2 + (b - a - 1)];
          }
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
    };
    int it = 0;
    int64_t tile = blockIdx.x;
    if (tile < ntiles) build(0, tile);
    for (; tile < ntiles; tile += gridDim.x, ++it) {
      if (tile + gridDim.x < ntiles) build(it + 1, tile + gridDim.x);
      const int64_t b0 = tile * S;
      const int ns = int(batch - b0 < S ? batch - b0 : S);
      const int rv = ns * nf;
      // feature 0's extra terms (gout[b, :d] and, for the mask, z0) of the
      // tile's samples into smem while the MMAs run
      const int nv = d / 4;
      for (int e = threadIdx.x; e < ns * nv; e += IA_EPI) {
        const int s = e / nv, c = e - s * nv;
        reinterpret_cast<float4*>(G0)[e] =
            __ldg(reinterpret_cast<const float4*>(gout + (b0 + s) * ld_gout) + c);
        if (mask_f0)
          reinterpret_cast<float4*>(Z0)[e] =
              __ldg(reinterpret_cast<const float4*>(fs.feat[0] + (b0 + s) * fs.stride[0]) + c);
      }
      mbar_wait(dfull, it & 1);
      tc_fence_after();
      if (32 * q < rv) {
        for (int c0 = 0; c0 < d; c0 += 16) {
          uint32_t hv[16], sv[16];
          tmem_ld16_issue(tmem + lane_off + uint32_t(c0), hv);
          tmem_ld16_issue(tmem + lane_off + uint32_t(d + c0), sv);
          tmem_wait_ld();
          if (i < rv) {
#pragma unroll
            for (int k = 0; k < 16; k += 4)
              *reinterpret_cast<float4*>(Y + size_t(i) * yp + c0 + k) = make_float4(
                  __uint_as_float(hv[k]) + __uint_as_float(sv[k]),
                  __uint_as_float(hv[k + 1]) + __uint_as_float(sv[k + 1]),
                  __uint_as_float(hv[k + 2]) + __uint_as_float(sv[k + 2]),
                  __uint_as_float(hv[k + 3]) + __uint_as_float(sv[k + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dempty);
      named_bar(2, IA_EPI);
      // feature rows out: one warp per row, float4 per lane
      for (int s = 0; s < ns; ++s)
        for (int f = warp; f < nf; f += 4) {
          const int r = s * nf + f;
          float4* dst = reinterpret_cast<float4*>(gs.feat[f] + (b0 + s) * gs.stride[f]);
          for (int c = lane; c < nv; c += 32) {
            float4 v = *reinterpret_cast<const float4*>(Y + size_t(r) * yp + 4 * c);
            if (f == 0) {
              const float4 g0 = reinterpret_cast<const float4*>(G0)[s * nv + c];
              v.x = g0.x + v.x; v.y = g0.y + v.y; v.z = g0.z + v.z; v.w = g0.w + v.w;
              if (mask_f0) {
                const float4 z0 = reinterpret_cast<const float4*>(Z0)[s * nv + c];
                v.x *= z0.x > 0.f ? 1.f : 0.f; v.y *= z0.y > 0.f ? 1.f : 0.f;
                v.z *= z0.z > 0.f ? 1.f : 0.f; v.w *= z0.w > 0.f ? 1.f : 0.f;
              }
            }
            dst[c] = v;
          }
        }
      named_bar(2, IA_EPI);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == IA_MMA_WARP) {
    tc_fence_after();
    tmem_dealloc_warp(tmem, IA_TMEM_COLS);
  }
}

uint32_t ceil_to(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

bool fwd_geom(int nf, int d, IaGeom* g) {
  if (nf < 2 || nf > 64 || d < 8 || d > 128 || d % 8) return false;
  const int P = nf * (nf - 1) / 2;
  const int kchunks = (d + 31) / 32;
  for (int S = 128 / nf; S >= 1; --S) {
    const int R = S * nf, Rp = int(ceil_to(R, 8));
    const int rows = 2 * Rp > 128 ? 2 * Rp : 128;
    const uint32_t stage = uint32_t(kchunks) * rows * 128;
    if (stage > 64 * 1024 && S > 1) continue;
    const size_t scratch = size_t(2) * R * nf * 4 + size_t(P) * 4 + 256;
    int nst = int((IA_SMEM_MAX - 1024 - scratch) / stage);
    if (nst > 4) nst = 4;
    if (nst < 2) continue;
    *g = IaGeom{};
    g->nf = nf; g->d = d; g->S = S; g->R = R; g->P = P; g->Rp = Rp; g->rows = rows;
    g->kchunks = kchunks; g->nst = nst; g->stage_bytes = stage;
    g->idesc = instr_desc(2 * Rp, false, false);
    return true;
  }
  return false;
}

bool bwd_geom(int nf, int d, IaGeom* g) {
  // the lo half of B starts at column d: a whole 32-column chunk, or (d = 16)
  // the upper half of chunk 0, so one descriptor addresses it
  if (nf < 2 || nf > 64 || d < 16 || d > 128 || (d % 32 && d != 16)) return false;
  const int P = nf * (nf - 1) / 2;
  const uint32_t a_base = ceil_to(uint32_t(2 * d), 32);
  for (int S = 128 / nf; S >= 1; --S) {
    const int R = S * nf, Kq = int(ceil_to(R, 16)), Kp = int(ceil_to(R, 8));
    if (a_base + 4u * Kq > IA_TMEM_COLS) continue;
    const uint32_t nchunk = (2 * d + 31) / 32;
    const uint32_t b_bytes = nchunk * Kp * 128;
    const int Pp = int(ceil_to(P, 4));
    const uint32_t stage = ceil_to(b_bytes + uint32_t(S) * Pp * 4, 1024);
    const size_t scratch = size_t(R) * (d + 4) * 4 + size_t(2) * S * d * 4 + 256;
    int nst = int((IA_SMEM_MAX - 1024 - scratch) / stage);
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
         8 + 16 * 8;
}
size_t bwd_smem(const IaGeom& g) {
  return 1024 + size_t(g.nst) * g.stage_bytes + size_t(g.R) * (g.d + 4) * 4 +
         size_t(2) * g.S * g.d * 4 + 16 * 8;
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
  const int64_t ntiles = ceil_div(batch, g.S);
  const unsigned grid = unsigned(ntiles < kNumSMs ? ntiles : kNumSMs);
  launch(interact_tc_fwd_kernel, grid, IA_THREADS, smem, s, fs, g, batch, out, ld_out, pad_to);
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
  const int64_t ntiles = ceil_div(batch, g.S);
  const unsigned grid = unsigned(ntiles < kNumSMs ? ntiles : kNumSMs);
  launch(interact_tc_bwd_kernel, grid, IA_THREADS, smem, s, fs, gs, g, batch, gout, ld_gout,
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
