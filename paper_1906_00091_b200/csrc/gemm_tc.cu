// fp32-accurate MLP GEMMs on the 5th-generation tensor cores (tcgen05).
//
//   D[M x N] = sum_k A(m, k) * B(n, k)        (fp32 in, fp32 out)
//
// computed as 3xTF32: x = hi + lo with hi = x truncated to TF32 and lo =
// x - hi (exact in fp32).  The tensor core itself ignores the low 13 mantissa
// bits of a kind::tf32 operand, so the TMA-landed fp32 tile IS the hi operand
// and only lo is materialised (by the splitter warps),
// then D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulated in TMEM.  The A
// operands (the 128-row side) are held in TMEM, not shared memory: the
// splitter warps read each landed A tile once and tcgen05.st its hi / lo
// halves into a TMEM slot, so neither A_lo stores nor the MMAs' A reads touch
// the shared-memory port, which bounds this kernel (TMA fill + splitter +
// MMA operand reads).  Single
// TF32 fails the reference tolerance on updated weights (SURVEY Appendix A:
// 6e-2); 3xTF32 matches fp32 (1.6e-7 loss, 9e-7 weights).
//
// Accuracy vs plain fp32 (scripts/tc_vs_simt.py, normwise vs float64, 2048 x
// 1024 x 1024): this kernel 3.6e-6, the SIMT fp32 GEMM 1.3e-6.  The gap is
// the tensor core's fp32 accumulation, which truncates: a TMEM chain of K/8
// steps drifts by up to (K/8) 2^-23.  Draining every 32-wide k-block into
// registers with round-to-nearest adds (fresh TMEM partials, ping-pong) was
// built and measured: 2.2e-7 — better than SIMT fp32 — but 45% slower (the
// splitter warps must wait for each k-block's MMAs before splitting the
// next), so it is not used; the 3x-of-fp32 error is far inside the
// north-star tolerance (tests/test_gpu_fullsize.py).
//
// Operands are fetched by TMA (cp.async.bulk.tensor, 128B swizzle) straight
// from the row-major activations/weights, K-major or MN-major as each GEMM
// needs (tcgen05 kind::tf32 accepts MN-major descriptors), so no transposed
// copies exist anywhere:
//   forward      Y  = X W^T      A = X  (K-major)   B = W (K-major)
//   data grad    dX = gZ W       A = gZ (K-major)   B = W (MN-major)
//   weight grad  dW = gZ^T X     A = gZ (MN-major)  B = X (MN-major)
//
// CTA = 10 warps, one 128 x BN output tile; a 4-stage TMA ring of raw tiles
// and a ring of TMEM A slots [A_hi | A_lo] (32 + 32 columns):
//   warp 0     TMA producer (one thread)
//   warp 1     TMEM allocator + MMA issuer (one thread)
//   warps 2-9  splitter for each landed stage (A -> TMEM slot, B_lo -> smem),
//              then the epilogue (tcgen05.ld 32x32b -> bias/ReLU/mask -> global)
// Barriers: full[t] (TMA tx), empty_t[t] / empty_l[l] (tcgen05.commit),
// conv[l] (8 splitter warps), acc_full (commit after the last k-block).
#include <cuda.h>
#include <stdlib.h>

#include "gemm.cuh"
#include "gemm_tc.cuh"
#include "tc_util.cuh"

namespace dlrm {
namespace {
using namespace tcu;

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 per 128-byte swizzle row
// TSTAGES shared-memory stages of [A raw | B_hi | B_lo] (TMA covers the L2
// latency of a tile load).
constexpr int TSTAGES = 4;
// splitter warps = epilogue warps: 2 per TMEM lane quarter
constexpr int SPLIT_WARPS = 8;
constexpr int EPI_WARPS = 8;
// bias row sums: k-row partials per tile row in the bias scratch
constexpr int kBiasRows = 8;
constexpr int THREADS = 64 + 32 * SPLIT_WARPS;
// lo = x - trunc_tf32(x) is fed to the tensor core, which truncates it to
// TF32 in turn (a 2^-22 relative bias per operand); DLRM_GEMM_RNA rounds it
// to the nearest TF32 instead (integer form, see tc_util.cuh)
#ifdef DLRM_GEMM_RNA
__device__ __forceinline__ uint32_t lo_bits(float x) { return tf32_rna(x); }
#else
__device__ __forceinline__ uint32_t lo_bits(float x) { return __float_as_uint(x); }
#endif

struct WgradFuse {
  int on;    // 1: fused wgrad epilogue (cluster of gridDim.z split-K CTAs)
  int bias;  // 1: bias gradient from the row sums of A
  float* dW;
  int64_t lddw;
  float* Wu;
  int64_t ldw;
  float* db;
  float* bu;
  Upd upd;  // SGD / Adagrad rule for W and b
  const int32_t* err_flag;
  int vec;  // dW / W rows 16-byte aligned
  int generic;  // 1: split-K forward / data gradient: the reduced tile goes
                // through the GemmEpilogue (bias / ReLU / mask) instead
};

struct TcArgs {
  int64_t M, N, K;
  int k_tiles_per_split;
  int k_tiles;
  GemmEpilogue ep;
  int a3d, b3d;  // MN-major operand described as a 3D tensor: one TMA box per tile
  WgradFuse wf;
  int blo;  // 1: B_lo comes from memory (third tensor map, same geometry as B) instead of
            // being converted from B_hi by the splitter warps
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// B tile of one k-block (BN columns at n0, BK k-rows at k0) into dst
template <bool B_MN, int BN>
__device__ __forceinline__ void load_b_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                            bool b3d, int64_t n0, int k0) {
  if (B_MN && b3d) {
    tma_load_3d(dst, map, bar, 0, k0, int(n0 / 32));
  } else if (B_MN) {
#pragma unroll
    for (int c = 0; c < BN / 32; ++c)
      tma_load_2d(dst + c * 32 * BK * 4, map, bar, int(n0 + 32 * c), k0);
    if (BN % 32)  // BN == 16: a single 16-wide box
      tma_load_2d(dst, map, bar, int(n0), k0);
  } else {
    tma_load_2d(dst, map, bar, k0, int(n0));
  }
}

// ---------------------------------------------------------------------------
// Fused weight-gradient epilogue (linear_bwd_weight): the split-K CTAs of one
// output tile form a thread-block cluster along z.  Each keeps its partial
// tile in its own shared memory; after a cluster barrier CTA z reduces rows
// [z*R, (z+1)*R) of the tile over the cluster ranks 0..S-1 in order (DSMEM
// loads, deterministic), writes dW and / or applies W -= lr * dW, and the
// n-tile-0 cluster does the same for the bias gradient (row sums of the A
// operand accumulated by the splitter warps).  No partial sums in global
// memory, no reduction kernel, no counters.
constexpr uint32_t kBiasScratch = 32 * 20 * 4 * 8;  // bias sums after the transpose tiles

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ float ld_dsmem1(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

// Executed by every thread of every CTA of the cluster (see WgradFuse).
template <int BN>
__device__ __forceinline__ void wgrad_cluster_reduce(const TcArgs& args, const uint8_t* ptile,
                                                     const uint8_t* bscratch, int64_t m0,
                                                     int64_t n0) {
  const WgradFuse& wf = args.wf;
  constexpr int P = BN + 4, C4 = BN / 4;
  // cluster (1, 1, S): the split k of this tile has cluster rank k
  const int S = int(gridDim.z), z = int(blockIdx.z);
  cluster_sync_all();  // every partial tile / bias scratch of the cluster is written
  const bool upd = wf.Wu != nullptr && !(wf.err_flag && *wf.err_flag);
  const int R = (BM + S - 1) / S, r0 = z * R, r1 = r0 + R < BM ? r0 + R : BM;
  const float* pt = reinterpret_cast<const float*>(ptile);
  const uint32_t base0 = dsmem_addr(pt, 0);
  const uint32_t rank_stride = S > 1 ? dsmem_addr(pt, 1) - base0 : 0;
  // generic: zero-padded output columns [N, pad_n) are written too
  const int64_t ncols = wf.generic && args.ep.pad_n > args.N ? args.ep.pad_n : args.N;
  for (int e = threadIdx.x; e < (r1 - r0) * C4; e += blockDim.x) {
    const int r = r0 + e / C4, c = (e % C4) * 4;
    const int64_t row = m0 + r, col = n0 + c;
    if (row >= args.M || col >= ncols) continue;
    const uint32_t off = uint32_t(r * P + c) * 4;
    float4 acc = ld_dsmem4(base0 + off);
    for (int k = 1; k < S; ++k) {
      const float4 v = ld_dsmem4(base0 + uint32_t(k) * rank_stride + off);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (wf.generic) {
      apply_epilogue4(args.ep, row, col, args.N, acc, 0);
      continue;
    }
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
    if (wf.vec && col + 3 < args.N) {
      if (wf.dW) *reinterpret_cast<float4*>(wf.dW + row * wf.lddw + col) = acc;
      if (upd) {
        float4* w = reinterpret_cast<float4*>(wf.Wu + row * wf.ldw + col);
        *w = upd_apply4(wf.upd, reinterpret_cast<float*>(w), *w, acc);
      }
    } else {
      for (int i = 0; i < 4 && col + i < args.N; ++i) {
        if (wf.dW) wf.dW[row * wf.lddw + col + i] = a[i];
        if (upd) {
          float* w = wf.Wu + row * wf.ldw + col + i;
          *w = upd_apply(wf.upd, w, *w, a[i]);
        }
      }
    }
  }
  if (wf.bias && n0 == 0) {
    const bool bupd = wf.bu != nullptr && !(wf.err_flag && *wf.err_flag);
    const float* bs = reinterpret_cast<const float*>(bscratch);
    const uint32_t bb0 = dsmem_addr(bs, 0);
    const uint32_t bstride = S > 1 ? dsmem_addr(bs, 1) - bb0 : 0;
    for (int r = r0 + int(threadIdx.x); r < r1; r += int(blockDim.x)) {
      const int64_t row = m0 + r;
      if (row >= args.M) continue;
      float acc = 0.f;  // ranks in order, k-rows in order
      for (int k = 0; k < S; ++k)
        for (int kr = 0; kr < kBiasRows; ++kr)
          acc += ld_dsmem1(bb0 + uint32_t(k) * bstride + uint32_t(kr * BM + r) * 4);
      if (wf.db) wf.db[row] = acc;
      if (bupd) wf.bu[row] = upd_apply(wf.upd, wf.bu + row, wf.bu[row], acc);
    }
  }
  cluster_sync_all();  // no CTA leaves while others still read its shared memory
}

// One CTA computes a BM x BN tile of the fp32-accurate product with 3xTF32
// tcgen05 MMAs.  Per k-step: a TMA stage [A raw | B_hi | B_lo] in shared
// memory (the raw fp32 B tile is the hi operand; the splitter writes B_lo
// right behind it) and a TMEM slot [A_hi | A_lo] written by the splitter
// (A operands from TMEM must be K-major there: lane = tile row, column = k,
// whatever the global layout — the splitter's per-row loads transpose
// MN-major tiles for free).  With B_lo adjacent to B_hi, the two products
// that share A_hi are ONE MMA of N = 2*BN (A_hi x [B_hi | B_lo]); the third,
// A_lo x B_hi, is an N = BN MMA.  Accumulators in TMEM: [big | small] pairs
// of BN columns; for BN <= 64 two pairs, k-block it going to pair it % 2, so
// each truncating TMEM accumulation chain is half as long (tensor-core fp32
// accumulation truncates; the error grows with the chain).  TMEM columns:
// accumulators, then ASLOTS x 64 A slots.
template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(THREADS, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmBl, TcArgs args) {
  constexpr bool FUSE = BN >= 32;            // BN = 16 (MN-major 64-byte boxes): 3 MMAs
  constexpr uint32_t A_BYTES = BM * BK * 4;  // 16 KB
  constexpr uint32_t B_BYTES = BN * BK * 4;
  constexpr uint32_t STAGE_BYTES = A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMA_BYTES = A_BYTES + B_BYTES;
  constexpr int NACC = BN >= 128 ? 1 : 2;
  constexpr uint32_t ACC_COLS = 2 * NACC * BN;
  // BN >= 64: > 113 KB of shared memory, one CTA per SM, all 512 columns;
  // narrower tiles may share an SM and take 256
  constexpr int ASLOTS = BN >= 64 ? 4 : 2;
  constexpr uint32_t TMEM_COLS = BN >= 64 ? 512 : 256;
  static_assert(ACC_COLS + 64 * ASLOTS <= TMEM_COLS, "TMEM overflow");
  constexpr uint32_t IDESC = instr_desc(BN, false, B_MN);
  constexpr uint32_t IDESC2 = instr_desc(FUSE ? 2 * BN : BN, false, B_MN);
  // epilogue scratch (transpose tiles, bias row sums) behind the dW partial
  // tile, inside the (by then idle) stage ring
  constexpr uint32_t PTILE_BYTES = (BM * (BN + 4) * 4 + 1023) / 1024 * 1024;
  static_assert(PTILE_BYTES + kBiasScratch + kBiasRows * BM * 4 <= TSTAGES * STAGE_BYTES,
                "epilogue scratch exceeds the stage ring");

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned for the 128B swizzle; offsetting the __shared__ array
  // (not casting through an integer) keeps every derived pointer in the
  // shared window, so the splitter / epilogue accesses compile to LDS / STS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;                                // TSTAGES x STAGE_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TSTAGES * STAGE_BYTES);
  uint64_t* full = bars;                               // TMA landed        [T]
  uint64_t* empty_t = bars + TSTAGES;                  // MMA done, stage   [T]
  uint64_t* conv = bars + 2 * TSTAGES;                 // A slot + B_lo set [L]
  uint64_t* empty_l = bars + 2 * TSTAGES + ASLOTS;     // MMA done, A slot  [L]
  uint64_t* acc_full = bars + 2 * TSTAGES + 2 * ASLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  uint8_t* epi = ring + PTILE_BYTES;                   // epilogue scratch

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
  const int kt0 = blockIdx.z * args.k_tiles_per_split;
  const int kt1 = min(args.k_tiles, kt0 + args.k_tiles_per_split);
  const int nk = kt1 - kt0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty_t[s], 1);
    }
    for (int s = 0; s < ASLOTS; ++s) {
      mbar_init(&conv[s], SPLIT_WARPS);
      mbar_init(&empty_l[s], 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Dependents are released only once this CTA HOLDS its TMEM: a PDL-launched
  // successor that allocates TMEM and then spins in griddepcontrol.wait can
  // therefore never keep a CTA of this grid (or, through it, a cluster
  // sibling on another stream) from allocating.  The prologue above touches
  // no data of the previous kernel.
  pdl_trigger();
  pdl_wait();  // operands / epilogue inputs come from earlier kernels

  if (warp == 0) {
    // ---- TMA producer: raw fp32 tiles (the tensor core reads them as the
    // hi operand: kind::tf32 ignores the low 13 mantissa bits)
    if (lane == 0) {
      for (int it = 0; it < nk; ++it) {
        const int s = it % TSTAGES;
        if (it >= TSTAGES) mbar_wait(&empty_t[s], ((it / TSTAGES) - 1) & 1);
        uint8_t* st = ring + s * STAGE_BYTES;
        const int k0 = (kt0 + it) * BK;
        mbar_expect_tx(&full[s], TMA_BYTES + (args.blo ? B_BYTES : 0u));
        if (A_MN && args.a3d) {
          tma_load_3d(st, &tmA, &full[s], 0, k0, int(m0 / 32));
        } else if (A_MN) {
#pragma unroll
          for (int c = 0; c < BM / 32; ++c)
            tma_load_2d(st + c * 32 * BK * 4, &tmA, &full[s], int(m0 + 32 * c), k0);
        } else {
          tma_load_2d(st, &tmA, &full[s], k0, int(m0));
        }
        load_b_tile<B_MN, BN>(st + A_BYTES, &tmB, &full[s], args.b3d, n0, k0);
        if (args.blo) load_b_tile<B_MN, BN>(st + A_BYTES + B_BYTES, &tmBl, &full[s], args.b3d, n0, k0);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    if (lane == 0) {
      for (int it = 0; it < nk; ++it) {
        const int t = it % TSTAGES, l = it % ASLOTS;
        mbar_wait(&conv[l], (it / ASLOTS) & 1);
        tc_fence_after();
        const uint32_t b_hi = smem_u32(ring + t * STAGE_BYTES) + A_BYTES;
        const uint32_t b_lo = b_hi + B_BYTES;
        const uint32_t a_hi = tmem + ACC_COLS + uint32_t(64 * l);  // TMEM slot
        const uint32_t a_lo = a_hi + 32;
        const uint32_t big = tmem + uint32_t((it % NACC) * 2 * BN);
        const uint32_t small = big + uint32_t(BN);
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          // B K-major: advance 32 B inside the swizzle row; MN-major: 8 k-rows.
          // A: 8 TMEM columns per k-step.
          const uint32_t bo = B_MN ? kk * 1024 : kk * 32;
          const uint32_t b_lbo = B_MN ? 32 * BK * 4 : 16, b_sbo = B_MN ? 512 : 1024;
          const uint32_t b_lay = B_MN ? 1 : 2;
          const uint64_t dbh = smem_desc(b_hi + bo, b_lbo, b_sbo, b_lay);
          const uint32_t first = (it >= NACC || kk > 0) ? 1u : 0u;
          if (FUSE) {
            mma_tf32_ts(big, a_hi + 8 * kk, dbh, IDESC2, first);  // [big | small] = A_hi x [B_hi | B_lo]
          } else {
            const uint64_t dbl = smem_desc(b_lo + bo, b_lbo, b_sbo, b_lay);
            mma_tf32_ts(big, a_hi + 8 * kk, dbh, IDESC, first);
            mma_tf32_ts(small, a_hi + 8 * kk, dbl, IDESC, first);
          }
          mma_tf32_ts(small, a_lo + 8 * kk, dbh, IDESC, 1u);      // small += A_lo x B_hi
        }
        mma_commit(&empty_t[t]);
        mma_commit(&empty_l[l]);
      }
      mma_commit(acc_full);
    }
  } else {
    // ---- splitter warps (2..9), per landed stage:
    //  A: warp (quarter q = warp % 4, half h) owns TMEM lanes / tile rows
    //     [32q, 32q+32) and k columns [16h, 16h+16): each thread loads its
    //     row's 16 values, tcgen05.st's hi = trunc_tf32(x) and lo = x - hi
    //     into the A slot.  Fused weight gradient, n-tile 0: the same loads
    //     accumulate the row sums of A (the bias gradient), 4 partials by k % 4.
    //  B: lo = x - trunc_tf32(x) written right behind B_hi in the stage.
    const int ct = threadIdx.x - 64;  // 0 .. 32*SPLIT_WARPS-1
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int arow = 32 * q + lane;
    const bool do_bias = A_MN && args.wf.on && args.wf.bias && blockIdx.x == 0;
    float bsum[4] = {0.f, 0.f, 0.f, 0.f};
    constexpr int B_F4 = int(B_BYTES / 16);
    constexpr int NSPLIT = 32 * SPLIT_WARPS;
    constexpr int NJ = (B_F4 + NSPLIT - 1) / NSPLIT;
    const uint32_t a_taddr = tmem + (uint32_t(32 * q) << 16) + ACC_COLS + uint32_t(16 * h);
    for (int it = 0; it < nk; ++it) {
      const int t = it % TSTAGES, l = it % ASLOTS;
      mbar_wait(&full[t], (it / TSTAGES) & 1);
      if (it >= ASLOTS) mbar_wait(&empty_l[l], ((it / ASLOTS) - 1) & 1);
      tc_fence_after();
      const uint8_t* st = ring + t * STAGE_BYTES;
      float x[16];
      if (A_MN) {  // [chunk q][k-row][32 rows, 32-byte atoms XOR k-row % 4]
        const float* src = reinterpret_cast<const float*>(st + q * 32 * BK * 4);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int kr = 16 * h + i;
          x[i] = src[kr * 32 + 8 * ((lane >> 3) ^ (kr & 3)) + (lane & 7)];
        }
      } else {  // row arow: 128 bytes, 16-byte chunk c at c ^ (row % 8)
        const float4* src = reinterpret_cast<const float4*>(st + arow * 128);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = src[(4 * h + c) ^ (arow & 7)];
          x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
      }
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        hi[i] = __float_as_uint(x[i]) & 0xFFFFE000u;
        lo[i] = lo_bits(x[i] - __uint_as_float(hi[i]));
      }
      if (do_bias) {
#pragma unroll
        for (int i = 0; i < 16; ++i) bsum[i & 3] += x[i];
      }
      const uint32_t slot = a_taddr + uint32_t(64 * l);
      tmem_st16(slot, hi);
      tmem_st16(slot + 32, lo);
      const float4* src_b = reinterpret_cast<const float4*>(st + A_BYTES);
      float4* dst_b = reinterpret_cast<float4*>(const_cast<uint8_t*>(st) + A_BYTES + B_BYTES);
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int i = ct + NSPLIT * j;
        if (!args.blo && (B_F4 % NSPLIT == 0 || i < B_F4)) {
          const float4 v = src_b[i];
          dst_b[i] = make_float4(__uint_as_float(lo_bits(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u))),
                                 __uint_as_float(lo_bits(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u))),
                                 __uint_as_float(lo_bits(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u))),
                                 __uint_as_float(lo_bits(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u))));
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[l]);
    }
    // ---- epilogue: TMEM lanes [32q, 32q+32) are readable by warps with
    // warp%4 == q; the two warps of a quarter take half of the columns each.
    // Per 32x16 block: all accumulator loads in flight, one wait, sum,
    // registers -> smem (transpose) -> float4 row-segment stores (4 lanes per
    // 64-byte row segment, 8 rows per instruction).
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int half = warp - 2 < EPI_WARPS ? (warp - 2) / 4 : 2;  // extra splitter warps: none
    float* tile = reinterpret_cast<float*>(epi) + (warp - 2) * (32 * 20);
    const GemmEpilogue& ep = args.ep;
    const int used = nk < NACC ? nk : NACC;
    constexpr int CW = BN / 2 < 16 ? 16 : BN / 2;  // columns per warp
#pragma unroll 1
    for (int c0 = half * CW; c0 < BN && c0 < (half + 1) * CW; c0 += 16) {
      uint32_t ra[2 * NACC][16];
      const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16) + uint32_t(c0);
#pragma unroll
      for (int j = 0; j < 2 * NACC; ++j) tmem_ld16_issue(lane_base + uint32_t(j * BN), ra[j]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(ra[0][i]) + __uint_as_float(ra[1][i]);
      if constexpr (NACC > 1) {
        if (used > 1) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            v[i] += __uint_as_float(ra[2][i]) + __uint_as_float(ra[3][i]);
        }
      }
      if (args.wf.on) {  // fused weight gradient: the partial tile stays in smem
        float* prow = reinterpret_cast<float*>(ring) + (32 * q + lane) * (BN + 4) + c0;
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(prow + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        continue;
      }
#pragma unroll
      for (int i = 0; i < 16; i += 4)
        *reinterpret_cast<float4*>(tile + lane * 20 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      __syncwarp();
      const int c4 = (lane & 3) * 4;
#pragma unroll
      for (int r = lane >> 2; r < 32; r += 8) {
        const int64_t row = m0 + 32 * q + r;
        if (row < args.M)
          apply_epilogue4(ep, row, n0 + c0 + c4, args.N,
                          *reinterpret_cast<const float4*>(tile + r * 20 + c4), blockIdx.z);
      }
      __syncwarp();
    }
    if (do_bias) {  // per-thread row-sum partials -> [k-row partial][m] scratch
      float* bs = reinterpret_cast<float*>(epi + kBiasScratch);
#pragma unroll
      for (int j = 0; j < 4; ++j) bs[(4 * h + j) * BM + arow] = bsum[j];
    }
  }
  if (args.wf.on) wgrad_cluster_reduce<BN>(args, ring, epi + kBiasScratch, m0, n0);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// Persistent variant for tile grids larger than the SMs (the B = 32768 MLPs):
// one CTA per SM walks output tiles tile = blockIdx.x, + gridDim.x, ... (the
// n tiles of an m row back to back, so the CTAs in flight share A rows in L2)
// with the same producer / MMA / splitter roles as tc_gemm_kernel (BN = 128,
// stage and A-slot counters running across tiles, so the producer fills the
// next tile's stages while this tile finishes), plus 8 epilogue warps: they
// drain the tile's [big | small] accumulators from TMEM into registers,
// release TMEM to the MMA issuer (acc_empty) and only then do the smem
// transpose and global stores — the next tile's MMAs overlap the stores.
constexpr int P_EPI_WARPS = 8;
constexpr int P_THREADS = THREADS + 32 * P_EPI_WARPS;

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(P_THREADS, 1)
tc_gemm_persistent_kernel(const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmBl, TcArgs args, int64_t n_tiles,
                          int64_t tiles) {
  constexpr int BN = 128;
  constexpr uint32_t A_BYTES = BM * BK * 4;
  constexpr uint32_t B_BYTES = BN * BK * 4;
  constexpr uint32_t STAGE_BYTES = A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMA_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t ACC_COLS = 2 * BN;  // one [big | small] pair
  constexpr int ASLOTS = 4;
  constexpr uint32_t TMEM_COLS = 512;
  static_assert(ACC_COLS + 64 * ASLOTS <= TMEM_COLS, "TMEM overflow");
  constexpr uint32_t IDESC = instr_desc(BN, false, B_MN);
  constexpr uint32_t IDESC2 = instr_desc(2 * BN, false, B_MN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = smem;                                // TSTAGES x STAGE_BYTES
  float* etile = reinterpret_cast<float*>(smem + TSTAGES * STAGE_BYTES);  // [8 warps][32][20]
  uint64_t* bars = reinterpret_cast<uint64_t*>(etile + P_EPI_WARPS * 32 * 20);
  uint64_t* full = bars;                               // TMA landed        [T]
  uint64_t* empty_t = bars + TSTAGES;                  // MMA done, stage   [T]
  uint64_t* conv = bars + 2 * TSTAGES;                 // A slot + B_lo set [L]
  uint64_t* empty_l = bars + 2 * TSTAGES + ASLOTS;     // MMA done, A slot  [L]
  uint64_t* acc_full = bars + 2 * TSTAGES + 2 * ASLOTS;  // tile accumulated
  uint64_t* acc_empty = acc_full + 1;                    // accumulators drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = args.k_tiles;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < TSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty_t[s], 1);
    }
    for (int s = 0; s < ASLOTS; ++s) {
      mbar_init(&conv[s], SPLIT_WARPS);
      mbar_init(&empty_l[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, P_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();  // after the TMEM allocation (see tc_gemm_kernel)
  pdl_wait();

  if (warp == 0) {
    // ---- TMA producer, k-blocks of all this CTA's tiles back to back
    if (lane == 0) {
      int g = 0;
      for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
        for (int it = 0; it < nk; ++it, ++g) {
          const int s = g % TSTAGES;
          if (g >= TSTAGES) mbar_wait(&empty_t[s], ((g / TSTAGES) - 1) & 1);
          uint8_t* st = ring + s * STAGE_BYTES;
          const int k0 = it * BK;
          mbar_expect_tx(&full[s], TMA_BYTES + (args.blo ? B_BYTES : 0u));
          if (A_MN && args.a3d) {
            tma_load_3d(st, &tmA, &full[s], 0, k0, int(m0 / 32));
          } else if (A_MN) {
#pragma unroll
            for (int c = 0; c < BM / 32; ++c)
              tma_load_2d(st + c * 32 * BK * 4, &tmA, &full[s], int(m0 + 32 * c), k0);
          } else {
            tma_load_2d(st, &tmA, &full[s], k0, int(m0));
          }
          load_b_tile<B_MN, BN>(st + A_BYTES, &tmB, &full[s], args.b3d, n0, k0);
          if (args.blo)
            load_b_tile<B_MN, BN>(st + A_BYTES + B_BYTES, &tmBl, &full[s], args.b3d, n0, k0);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    if (lane == 0) {
      int g = 0, ti = 0;
      for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++ti) {
        // the epilogue warps have drained the previous tile's accumulators
        if (ti >= 1) mbar_wait(acc_empty, (ti - 1) & 1);
        tc_fence_after();
        for (int it = 0; it < nk; ++it, ++g) {
          const int t = g % TSTAGES, l = g % ASLOTS;
          mbar_wait(&conv[l], (g / ASLOTS) & 1);
          tc_fence_after();
          const uint32_t b_hi = smem_u32(ring + t * STAGE_BYTES) + A_BYTES;
          const uint32_t a_hi = tmem + ACC_COLS + uint32_t(64 * l);
          const uint32_t a_lo = a_hi + 32;
          const uint32_t big = tmem, small = tmem + uint32_t(BN);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t bo = B_MN ? kk * 1024 : kk * 32;
            const uint32_t b_lbo = B_MN ? 32 * BK * 4 : 16, b_sbo = B_MN ? 512 : 1024;
            const uint32_t b_lay = B_MN ? 1 : 2;
            const uint64_t dbh = smem_desc(b_hi + bo, b_lbo, b_sbo, b_lay);
            const uint32_t first = (it > 0 || kk > 0) ? 1u : 0u;
            mma_tf32_ts(big, a_hi + 8 * kk, dbh, IDESC2, first);  // [big | small] = A_hi x [B_hi | B_lo]
            mma_tf32_ts(small, a_lo + 8 * kk, dbh, IDESC, 1u);    // small += A_lo x B_hi
          }
          mma_commit(&empty_t[t]);
          mma_commit(&empty_l[l]);
        }
        mma_commit(acc_full);
      }
    }
  } else if (warp < 2 + SPLIT_WARPS) {
    // ---- splitter warps (2..9), as in tc_gemm_kernel
    const int ct = threadIdx.x - 64;
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int arow = 32 * q + lane;
    constexpr int B_F4 = int(B_BYTES / 16);
    constexpr int NSPLIT = 32 * SPLIT_WARPS;
    constexpr int NJ = (B_F4 + NSPLIT - 1) / NSPLIT;
    const uint32_t a_taddr = tmem + (uint32_t(32 * q) << 16) + ACC_COLS + uint32_t(16 * h);
    int g = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      for (int it = 0; it < nk; ++it, ++g) {
        const int t = g % TSTAGES, l = g % ASLOTS;
        mbar_wait(&full[t], (g / TSTAGES) & 1);
        if (g >= ASLOTS) mbar_wait(&empty_l[l], ((g / ASLOTS) - 1) & 1);
        tc_fence_after();
        const uint8_t* st = ring + t * STAGE_BYTES;
        float x[16];
        if (A_MN) {
          const float* src = reinterpret_cast<const float*>(st + q * 32 * BK * 4);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int kr = 16 * h + i;
            x[i] = src[kr * 32 + 8 * ((lane >> 3) ^ (kr & 3)) + (lane & 7)];
          }
        } else {
          const float4* src = reinterpret_cast<const float4*>(st + arow * 128);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 v = src[(4 * h + c) ^ (arow & 7)];
            x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
          }
        }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          hi[i] = __float_as_uint(x[i]) & 0xFFFFE000u;
          lo[i] = lo_bits(x[i] - __uint_as_float(hi[i]));
        }
        const uint32_t slot = a_taddr + uint32_t(64 * l);
        tmem_st16(slot, hi);
        tmem_st16(slot + 32, lo);
        const float4* src_b = reinterpret_cast<const float4*>(st + A_BYTES);
        float4* dst_b = reinterpret_cast<float4*>(const_cast<uint8_t*>(st) + A_BYTES + B_BYTES);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int i = ct + NSPLIT * j;
          if (!args.blo && (B_F4 % NSPLIT == 0 || i < B_F4)) {
            const float4 v = src_b[i];
            dst_b[i] = make_float4(__uint_as_float(lo_bits(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u))),
                                   __uint_as_float(lo_bits(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u))),
                                   __uint_as_float(lo_bits(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u))),
                                   __uint_as_float(lo_bits(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u))));
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[l]);
      }
    }
  } else {
    // ---- epilogue warps (10..17): TMEM lane quarter q = warp % 4, column
    // half by warp; the whole 32 x 64 block is drained into registers before
    // the accumulators are released
    const int ew = warp - 2 - SPLIT_WARPS;  // 0..7
    const int q = warp & 3, half = ew >> 2;
    float* tile_s = etile + ew * (32 * 20);
    const GemmEpilogue& ep = args.ep;
    constexpr int CW = BN / 2;  // 64 columns per warp
    int ti = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++ti) {
      const int64_t m0 = (tile / n_tiles) * BM, n0 = (tile % n_tiles) * BN;
      mbar_wait(acc_full, ti & 1);
      tc_fence_after();
      float v[CW];
      const uint32_t lane_base = tmem + (uint32_t(32 * q) << 16) + uint32_t(half * CW);
#pragma unroll
      for (int c = 0; c < CW; c += 16) {
        uint32_t rb[16], rs[16];
        tmem_ld16_issue(lane_base + uint32_t(c), rb);
        tmem_ld16_issue(lane_base + uint32_t(BN + c), rs);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) v[c + i] = __uint_as_float(rb[i]) + __uint_as_float(rs[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);  // the next tile's MMAs may start
#pragma unroll
      for (int c = 0; c < CW; c += 16) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(tile_s + lane * 20 + i) =
              make_float4(v[c + i], v[c + i + 1], v[c + i + 2], v[c + i + 3]);
        __syncwarp();
        const int c4 = (lane & 3) * 4;
        // rolled: 4 inlined epilogues, not 16 (fully unrolled, the kernel's
        // SASS doubled and the epilogue stalled on instruction fetch)
#pragma unroll 1
        for (int r = lane >> 2; r < 32; r += 8) {
          const int64_t row = m0 + 32 * q + r;
          if (row < args.M)
            apply_epilogue4(ep, row, n0 + half * CW + c + c4, args.N,
                            *reinterpret_cast<const float4*>(tile_s + r * 20 + c4), 0);
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// host side

int g_tc_mode = 0;  // 0: use tcgen05 where the shape allows; 1: never

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library does not link libcuda (it must dlopen on GPU-less build hosts).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

bool encode(CUtensorMap* map, const float* base, int64_t inner, int64_t outer,
            int64_t ld_elems, int box_inner, int box_outer, CUtensorMapSwizzle swz) {
  EncodeTiledFn cuTensorMapEncodeTiled = encode_fn();
  if (!cuTensorMapEncodeTiled) return false;
  cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  cuuint64_t strides[1] = {cuuint64_t(ld_elems) * 4};
  cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                      const_cast<float*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

constexpr size_t smem_bytes(int bn) {
  return size_t(TSTAGES) * (BM * BK * 4 + 2 * bn * BK * 4) + 1024 + 256;
}

template <bool A_MN, bool B_MN, int BN>
int launch_bn(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& bl,
              const TcArgs& args, int64_t n_grid, int splits, cudaStream_t s) {
  auto k = tc_gemm_kernel<A_MN, B_MN, BN>;
  const size_t sm = smem_bytes(BN);
  static bool configured = false;
  if (!configured) {
    DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    configured = true;
  }
  const dim3 grid(unsigned(ceil_div(n_grid, BN)), unsigned(ceil_div(args.M, BM)),
                  unsigned(splits));
  const int64_t tiles = int64_t(grid.x) * grid.y;
  static const bool persist_ok = !getenv("DLRM_GEMM_PERSIST") ||
                                 atoi(getenv("DLRM_GEMM_PERSIST")) != 0;
  if (BN == 128 && !args.wf.on && splits == 1 && tiles > kNumSMs && persist_ok) {
    // more tiles than SMs: persistent CTAs, the next tile's loads and MMAs
    // overlap this tile's epilogue
    auto kp = tc_gemm_persistent_kernel<A_MN, B_MN>;
    const size_t psm = sm + size_t(P_EPI_WARPS) * 32 * 20 * 4;
    static bool pconf = false;
    if (!pconf) {
      DLRM_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(psm)));
      pconf = true;
    }
    launch(kp, unsigned(tiles < kNumSMs ? tiles : kNumSMs), P_THREADS, psm, s, a, b, bl, args,
           int64_t(grid.x), tiles);
    return check_launch("tc_gemm_persistent_kernel");
  }
  if (!args.wf.on) {
    launch(k, grid, THREADS, sm, s, a, b, bl, args);
    return check_launch("tc_gemm_kernel");
  }
  // fused weight gradient: the split-K CTAs of a tile are one cluster
  static bool nonportable = false;
  if (splits > 8 && !nonportable) {
    DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    nonportable = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = unsigned(splits);
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, k, a, b, bl, args);
  return check_launch("tc_gemm_kernel(cluster)");
}

// Concurrently resident clusters of (1, 1, cz) CTAs of the BN-wide kernel
// (the split-K clusters of the fused weight gradient); cached per (BN, cz).
template <bool A_MN, bool B_MN, int BN>
int max_clusters(int cz) {
  static int cache[17] = {0};
  if (cz < 1 || cz > 16) return 1;
  if (cache[cz]) return cache[cz];
  auto k = tc_gemm_kernel<A_MN, B_MN, BN>;
  const size_t sm = smem_bytes(BN);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  if (cz > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1, 1, unsigned(cz));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = unsigned(cz);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = cz > 8 ? 0 : kNumSMs / cz;  // a non-portable size that does not fit: unused
  }
  cache[cz] = n;
  return n;
}

#ifndef DLRM_MAX_SPLIT
#define DLRM_MAX_SPLIT 16
#endif
constexpr int kMaxSplit = DLRM_MAX_SPLIT;

// Tile plan: the N tile and the split-K (cluster) size.
struct TcPlan {
  int bn;
  int splits;
};

template <bool A_MN, bool B_MN>
int launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& bl, const TcArgs& args,
           int64_t n_grid, int bn, int splits, cudaStream_t s) {
  switch (bn) {
    case 16: return launch_bn<A_MN, B_MN, 16>(a, b, bl, args, n_grid, splits, s);
    case 32: return launch_bn<A_MN, B_MN, 32>(a, b, bl, args, n_grid, splits, s);
    case 64: return launch_bn<A_MN, B_MN, 64>(a, b, bl, args, n_grid, splits, s);
    default: return launch_bn<A_MN, B_MN, 128>(a, b, bl, args, n_grid, splits, s);
  }
}

// MN-major operand whose MN extent is a multiple of 32, seen as the 3D
// tensor (32 [stride 1], k [stride ld], mn/32 [stride 32]): one box
// {32, BK, rows/32} lands exactly the [chunk][k][32] tile layout.
bool encode3(CUtensorMap* map, const float* base, int64_t mn, int64_t k, int64_t ld,
             int rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {32, cuuint64_t(k), cuuint64_t(mn / 32)};
  cuuint64_t strides[2] = {cuuint64_t(ld) * 4, 128};
  cuuint32_t box[3] = {32, cuuint32_t(BK), cuuint32_t(rows / 32)};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

bool use3d(bool mn_major, int64_t mn, int rows) {
  return mn_major && mn % 32 == 0 && rows % 32 == 0 && rows >= 32 && !getenv("DLRM_NO_TMA3D");
}

// TMA boxes: K-major operand -> box {BK, rows}; MN-major -> box {32 (or 16), BK}
bool map_operand(CUtensorMap* m, const float* p, bool mn_major, int64_t mn, int64_t k,
                 int64_t ld, int rows) {
  if (!aligned16(p) || (ld % 4) != 0) return false;
  if (use3d(mn_major, mn, rows)) return encode3(m, p, mn, k, ld, rows);
  if (mn_major)
    return encode(m, p, mn, k, ld, rows < 32 ? rows : 32, BK,
                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  return encode(m, p, k, mn, ld, BK, rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Split-K plan for the cluster-reduced kernels (fused weight gradient; and
// forward / data gradient when a tile grid is too small to fill the SMs):
// BN and the split-K cluster size from the tile time model, waves counted
// against the number of co-resident clusters.  Returns splits = 1 when
// splitting does not pay.
template <bool A_MN, bool B_MN>
TcPlan cluster_plan(int64_t m_rows, int64_t n_grid, int64_t kt, int min_bn,
                    bool one_per_sm = false) {
  constexpr double F = 9000, C0 = 600, C1 = 7.5;
  const int64_t mt = ceil_div(m_rows, BM);
  TcPlan best{128, 1};
  double best_t = 1e30;
  for (int bn : {128, 64, 32, 16}) {
    if (bn < min_bn) continue;
    if (bn > 16 && n_grid <= bn / 2) continue;  // mostly empty tile
    const int64_t tiles = mt * ceil_div(n_grid, bn);
    // up to 16 split-K CTAs per cluster (non-portable size above 8): the
    // weight gradients of narrow layers over long batches (c4: 128 x 256
    // outputs over K = 32768) have only a few output tiles
    // (16 only over long K — >= 256 k-blocks, c4's B = 32768; at B = 2048 the
    // wider clusters measured no faster and cost a little at c2)
    const int64_t lim = kt >= 256 ? kMaxSplit : (kMaxSplit < 8 ? kMaxSplit : 8);
    int64_t smax = kt / 4 < lim ? kt / 4 : lim;
    if (smax < 1) smax = 1;
    for (int64_t sp = 1; sp <= smax; ++sp) {
      const int cap_occ = bn == 128 ? max_clusters<A_MN, B_MN, 128>(int(sp))
                    : bn == 64  ? max_clusters<A_MN, B_MN, 64>(int(sp))
                    : bn == 32  ? max_clusters<A_MN, B_MN, 32>(int(sp))
                                : max_clusters<A_MN, B_MN, 16>(int(sp));
      if (cap_occ < 1) continue;
      // one_per_sm: narrow tiles sharing an SM also share its tensor core
      const int cap = one_per_sm && cap_occ > kNumSMs / int(sp) ? kNumSMs / int(sp) : cap_occ;
      const double waves = double(ceil_div(tiles, cap));
      const double t = waves * (F + double(ceil_div(kt, sp)) * (C0 + C1 * bn)) +
                       (sp > 1 ? 400.0 * double(sp) : 0.0);
      if (t < best_t) {
        best_t = t;
        best = TcPlan{bn, int(sp)};
      }
    }
  }
  return best;
}

// Fused weight gradient: m = N (MN-major gZ), n = K, k = M.
TcPlan weight_plan(int64_t M, int64_t N, int64_t K) {
  // DLRM_WGRAD_PLAN="bn,splits": measurement override
  if (const char* e = getenv("DLRM_WGRAD_PLAN")) {
    int bn = 0, sp = 0;
    if (sscanf(e, "%d,%d", &bn, &sp) == 2 && (bn == 32 || bn == 64 || bn == 128) && sp >= 1 &&
        sp <= kMaxSplit)
      return TcPlan{bn, sp};
  }
  return cluster_plan<true, true>(N, K, ceil_div(M, BK), 32);
}

__global__ void __launch_bounds__(256) split_lo_kernel(const float4* __restrict__ x,
                                                       float4* __restrict__ lo, int64_t n4) {
  pdl_entry();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    lo[i] = make_float4(__uint_as_float(lo_bits(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u))),
                        __uint_as_float(lo_bits(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u))),
                        __uint_as_float(lo_bits(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u))),
                        __uint_as_float(lo_bits(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u))));
  }
}

}  // namespace

// DLRM_GEMM_BLO=0: the splitter converts B_lo per tile even when W_lo is given
bool blo_enabled() {
  static const bool on = !getenv("DLRM_GEMM_BLO") || atoi(getenv("DLRM_GEMM_BLO")) != 0;
  return on;
}

int tc_split_lo(const float* x, float* lo, int64_t n, cudaStream_t s) {
  DLRM_REQUIRE(n % 4 == 0 && aligned16(x) && aligned16(lo), "split_lo needs float4 rows");
  const int64_t n4 = n / 4;
  int64_t blocks = ceil_div(n4, 256);
  if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
  if (blocks < 1) return 0;
  launch(split_lo_kernel, unsigned(blocks), 256, 0, s, reinterpret_cast<const float4*>(x),
         reinterpret_cast<float4*>(lo), n4);
  return check_launch("split_lo_kernel");
}

bool tc_enabled() { return g_tc_mode != 1; }
int tc_mode() { return g_tc_mode; }

bool tma_encode_2d(CUtensorMap* map, const float* base, int64_t inner, int64_t outer,
                   int64_t ld_elems, int box_inner, int box_outer, int swizzle) {
  if (!aligned16(base) || (ld_elems % 4) != 0) return false;
  const CUtensorMapSwizzle swz = swizzle == 1   ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle == 2 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  return encode(map, base, inner, outer, ld_elems, box_inner, box_outer, swz);
}

namespace {
// split-K clusters of a forward / data-gradient GEMM: partial tiles reduced
// over DSMEM, then the normal epilogue
WgradFuse cluster_epilogue() {
  WgradFuse w{};
  w.on = 1;
  w.generic = 1;
  return w;
}
}  // namespace

bool tc_linear_fwd_ok(const float* X, int64_t ldx, const float* W, int64_t ldw, const float* Y,
                      int64_t ldy, int64_t M, int64_t N, int64_t K, int64_t n_grid) {
  (void)Y;
  (void)ldy;
  return tc_enabled() && M >= 1 && N >= 16 && K >= 1 && aligned16(X) && aligned16(W) &&
         ldx % 4 == 0 && ldw % 4 == 0 && n_grid >= N;
}

int tc_linear_fwd(const float* X, int64_t ldx, const float* W, int64_t ldw, const float* b,
                  float* Y, int64_t ldy, int64_t M, int64_t N, int64_t K, int64_t n_grid,
                  int act, cudaStream_t s, const float* W_lo) {
  // split-K over a thread-block cluster when the tile grid alone cannot
  // fill the SMs (bias / ReLU applied after the DSMEM reduction)
  const TcPlan pl = cluster_plan<false, false>(M, n_grid, ceil_div(K, BK), 16, true);
  const int bn = pl.bn;
  CUtensorMap ma, mb;
  DLRM_REQUIRE(map_operand(&ma, X, false, M, K, ldx, BM) &&
                   map_operand(&mb, W, false, N, K, ldw, bn),
               "tensor map encoding failed (linear_fwd)");
  TcArgs a{M, N, K, 0, 0, GemmEpilogue{EPI_BIAS_ACT, act, Y, ldy, b, nullptr, 0, n_grid, M,
                                        aligned16(Y) && ldy % 4 == 0 && aligned16(b)},
           0, 0};
  a.k_tiles = int(ceil_div(K, BK));
  a.k_tiles_per_split = int(ceil_div(a.k_tiles, pl.splits));
  const int used = int(ceil_div(a.k_tiles, a.k_tiles_per_split));
  if (used > 1) a.wf = cluster_epilogue();
  CUtensorMap ml = mb;
  if (W_lo && blo_enabled() && bn >= 32) {
    DLRM_REQUIRE(map_operand(&ml, W_lo, false, N, K, ldw, bn), "tensor map encoding failed (W_lo)");
    a.blo = 1;
  }
  return launch<false, false>(ma, mb, ml, a, n_grid, bn, used, s);
}

bool tc_linear_bwd_data_ok(const float* gZ, int64_t ldg, const float* W, int64_t ldw,
                           const float* dX, int64_t ldx, int64_t M, int64_t N, int64_t K) {
  (void)dX;
  (void)ldx;
  return tc_enabled() && M >= 1 && K >= 1 && N >= 1 && aligned16(gZ) && aligned16(W) &&
         ldg % 4 == 0 && ldw % 4 == 0;
}

int tc_linear_bwd_data(const float* gZ, int64_t ldg, const float* W, int64_t ldw,
                       const float* mask, int64_t ldm, float* dX, int64_t ldx, int64_t M,
                       int64_t N, int64_t K, cudaStream_t s, const float* W_lo) {
  // dX (M x K) = gZ (M x N) W (N x K): GEMM n = K (MN-major in W), k = N
  const TcPlan pl = cluster_plan<false, true>(M, K, ceil_div(N, BK), 32, true);
  const int bn = pl.bn;
  CUtensorMap ma, mb;
  DLRM_REQUIRE(map_operand(&ma, gZ, false, M, N, ldg, BM) &&
                   map_operand(&mb, W, true, K, N, ldw, bn),
               "tensor map encoding failed (linear_bwd_data)");
  TcArgs a{M, K, N, 0, 0, GemmEpilogue{EPI_MASK, 0, dX, ldx, nullptr, mask, ldm, K, M,
                                        aligned16(dX) && ldx % 4 == 0 &&
                                            (!mask || (aligned16(mask) && ldm % 4 == 0))},
           0, use3d(true, K, bn)};
  a.k_tiles = int(ceil_div(N, BK));
  a.k_tiles_per_split = int(ceil_div(a.k_tiles, pl.splits));
  const int used = int(ceil_div(a.k_tiles, a.k_tiles_per_split));
  if (used > 1) a.wf = cluster_epilogue();
  CUtensorMap ml = mb;
  if (W_lo && blo_enabled() && bn >= 32) {
    DLRM_REQUIRE(map_operand(&ml, W_lo, true, K, N, ldw, bn), "tensor map encoding failed (W_lo)");
    a.blo = 1;
  }
  return launch<false, true>(ma, mb, ml, a, K, bn, used, s);
}

bool tc_linear_bwd_weight_ok(const float* gZ, int64_t ldg, const float* X, int64_t ldx,
                             int64_t M, int64_t N, int64_t K) {
  // any K: a narrow input (the 13 dense features) lands as one zero-filled
  // 32-wide MN-major box per k-step; with cluster split-K this beats the
  // SIMT split-K path end to end (c2 0.241 -> 0.233 ms/step)
  return tc_enabled() && M >= 1 && N >= 1 && K >= 1 && aligned16(gZ) && aligned16(X) &&
         ldg % 4 == 0 && ldx % 4 == 0;
}


int tc_linear_bwd_weight(const float* gZ, int64_t ldg, const float* X, int64_t ldx, int64_t M,
                         int64_t N, int64_t K, float* dW, int64_t lddw, float* W_upd,
                         int64_t ldw, float* db, float* b_upd, const Upd& u,
                         const int32_t* err_flag, cudaStream_t s) {
  // dW (N x K) = gZ^T X: GEMM m = N (MN-major in gZ), n = K (MN-major in X), k = M;
  // db (N) = row sums of the A operand; both reduced over the split-K cluster
  const TcPlan pl = weight_plan(M, N, K);
  const int bn = pl.bn;
  CUtensorMap ma, mb;
  DLRM_REQUIRE(map_operand(&ma, gZ, true, N, M, ldg, BM) &&
                   map_operand(&mb, X, true, K, M, ldx, bn),
               "tensor map encoding failed (linear_bwd_weight)");
  TcArgs a{N, K, M, 0, 0, GemmEpilogue{}, use3d(true, N, BM), use3d(true, K, bn)};
  a.k_tiles = int(ceil_div(M, BK));
  a.k_tiles_per_split = int(ceil_div(a.k_tiles, pl.splits));
  const int used = int(ceil_div(a.k_tiles, a.k_tiles_per_split));
  const bool vec = (!dW || (aligned16(dW) && lddw % 4 == 0)) &&
                   (!W_upd || (aligned16(W_upd) && ldw % 4 == 0)) &&
                   (u.kind != DLRM_UPD_ADAGRAD || u.delta % 4 == 0);
  a.wf = WgradFuse{1, (db || b_upd) ? 1 : 0, dW, lddw, W_upd, ldw, db, b_upd, u, err_flag,
                   vec ? 1 : 0};

  return launch<true, true>(ma, mb, mb, a, K, bn, used, s);
}

}  // namespace dlrm

extern "C" int dlrm_gemm_mode(int32_t mode) {
  dlrm::g_tc_mode = mode;
  return 0;
}

extern "C" int dlrm_gemm_mode_get(void) { return dlrm::g_tc_mode; }
