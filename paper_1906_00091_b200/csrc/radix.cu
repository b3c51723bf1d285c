// Stable LSD radix sort of (uint32 key, uint32 value) pairs for the sparse
// backward: the index-only "prepare" half of embedding.py:182-210's
// lookup_backward (np.add.at order = ascending row, then ascending position,
// so the sort must be stable).  An alternative to the library onesweep sort
// (cub::DeviceRadixSort, the default), whose decoupled look-back chain over
// ~100-200 tiles makes each 8-bit pass latency-bound at ~1 M keys (15-21 us
// per pass on B200, three passes for 23-bit keys).  Selected with
// DLRM_SORT=radix8 / radix12.  Measured at c3 (827 k keys):
// prepare alone 70 us vs 80 us for the library sort, but the training step
// 0.428 vs 0.420 ms (it shares the SMs with the lookups on the side stream),
// so the library sort stays the default.
//
// Here: at most 12-bit digits, so 23-bit keys take two passes; every kernel is
// fully parallel (no inter-CTA chain).  Per pass, over tiles of TILE
// consecutive keys:
//   rs_hist_kernel     per-tile digit histograms H[digit][tile] (smem atomics)
//   rs_prefix_kernel   H -> exclusive prefix over the tiles of each digit (in
//                      place, one warp per digit) and the digit totals
//   rs_scatter_kernel  the digit bases (a block scan of the totals, redone by
//                      every CTA), then each warp walks its own contiguous
//                      1024-key slice of the tile (held in registers) in
//                      order: warp-private
//                      cursors per digit (the warps' counts prefix-summed in
//                      warp order), ranks among equal digits of the same 32
//                      keys from __match_any_sync — input order is kept
//                      within every digit, i.e. the pass is stable.
// Keys past n do not exist (tiles are clipped); the caller's sentinel keys
// (all ones in the sorted bits) simply sort last.
#include <stdlib.h>

#include "common.cuh"
#include "radix.cuh"

namespace dlrm {
namespace {

// Two shapes (digit_bits): 8-bit digits (256 buckets, 4096-key tiles,
// small CTAs) or 12-bit digits (4096 buckets, 8192-key tiles, one pass less).
template <int DB, int WARPS_, int SLICE_>
struct RsCfg {
  static constexpr int WARPS = WARPS_;
  static constexpr int SLICE = SLICE_;   // keys per warp per tile
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int TILE = WARPS * SLICE;
  static constexpr int NB = 1 << DB;
};

// Per-tile digit histograms, digit-major: H[digit * ntiles + tile].
template <class C>
__global__ void __launch_bounds__(C::THREADS)
rs_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift, int nbits,
               uint32_t* __restrict__ H, int64_t ntiles) {
  pdl_entry();
  __shared__ uint32_t h[C::NB];
  const int nb = 1 << nbits;
  const uint32_t mask = uint32_t(nb - 1);
  for (int b = threadIdx.x; b < nb; b += C::THREADS) h[b] = 0;
  const int64_t t0 = int64_t(blockIdx.x) * C::TILE;
  constexpr int PER = C::TILE / C::THREADS;  // keys per thread, all loads in flight
  uint32_t k[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t i = t0 + j * C::THREADS + threadIdx.x;
    k[j] = i < n ? __ldg(keys + i) : 0xffffffffu;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (t0 + j * C::THREADS + threadIdx.x < n) atomicAdd(&h[(k[j] >> shift) & mask], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += C::THREADS) H[int64_t(b) * ntiles + blockIdx.x] = h[b];
}

// one warp per digit: H[b][t] <- sum over tiles t' < t of H[b][t'], and the
// digit total
__global__ void __launch_bounds__(256)
rs_prefix_kernel(uint32_t* __restrict__ H, int64_t ntiles, int nbits, uint32_t* __restrict__ total) {
  pdl_entry();
  const int nb = 1 << nbits;
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (b >= nb) return;
  uint32_t* h = H + int64_t(b) * ntiles;
  uint32_t carry = 0;
  for (int64_t t = 0; t < ntiles; t += 32) {
    const uint32_t c = t + lane < ntiles ? h[t + lane] : 0u;
    uint32_t incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (t + lane < ntiles) h[t + lane] = carry + incl - c;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) total[b] = carry;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS)
rs_scatter_kernel(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                  uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int64_t n, int shift,
                  int nbits, const uint32_t* __restrict__ H, int64_t ntiles,
                  const uint32_t* __restrict__ total) {
  pdl_entry();
  extern __shared__ uint32_t rs_smem[];
  uint32_t* base = rs_smem;                     // [NB] digit bases
  uint32_t* cur = rs_smem + C::NB;              // [WARPS][NB] per-warp cursors
  const int nb = 1 << nbits;
  const uint32_t mask = uint32_t(nb - 1);
  __shared__ uint32_t wsum[C::WARPS];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // this warp's slice of the tile, into registers (all loads in flight)
  constexpr int R = C::SLICE / 32;
  const int64_t s0 = int64_t(blockIdx.x) * C::TILE + int64_t(warp) * C::SLICE;
  uint32_t k[R], v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t i = s0 + r * 32 + lane;
    k[r] = i < n ? __ldg(kin + i) : 0u;
    v[r] = i < n ? __ldg(vin + i) : 0u;
  }

  // digit bases: exclusive scan of the totals (each thread a run of nb/256)
  const int per = nb / C::THREADS > 0 ? nb / C::THREADS : 1;
  const int b0 = threadIdx.x * per;
  uint32_t s = 0;
  for (int j = 0; j < per; ++j)
    if (b0 + j < nb) s += total[b0 + j];
  uint32_t incl = s;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) wsum[warp] = incl;
  for (int e = threadIdx.x; e < C::WARPS * nb; e += C::THREADS) cur[e] = 0;
  __syncthreads();
  uint32_t run = incl - s;
  for (int w = 0; w < warp; ++w) run += wsum[w];
  for (int j = 0; j < per; ++j)
    if (b0 + j < nb) {
      base[b0 + j] = run;
      run += total[b0 + j];
    }
  // per-warp digit counts of the warp's slice
  uint32_t* wc = cur + warp * nb;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (s0 + r * 32 + lane < n) atomicAdd(&wc[(k[r] >> shift) & mask], 1u);
  __syncthreads();
  // cursors: base + this tile's offset + the counts of earlier warps
  for (int b = threadIdx.x; b < nb; b += C::THREADS) {
    uint32_t c = base[b] + H[int64_t(b) * ntiles + blockIdx.x];
    for (int w = 0; w < C::WARPS; ++w) {
      const uint32_t x = cur[w * nb + b];
      cur[w * nb + b] = c;
      c += x;
    }
  }
  __syncthreads();
  // scatter, in input order
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool ok = s0 + r * 32 + lane < n;
    const uint32_t dg = ok ? (k[r] >> shift) & mask : uint32_t(nb + lane);  // past n: own digit
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    uint32_t pos = 0;
    if (ok) pos = wc[dg] + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) wc[dg] += __popc(peers);  // the lowest peer advances
    if (ok) {
      kout[pos] = k[r];
      vout[pos] = v[r];
    }
    __syncwarp();
  }
}

template <class C>
int sort_passes(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_out, uint32_t* vals_out,
                int64_t n, int end_bit, void* scratch, int db, cudaStream_t s) {
  const int64_t ntiles = (n + C::TILE - 1) / C::TILE;
  uint32_t* kt = reinterpret_cast<uint32_t*>(scratch);
  uint32_t* vt = kt + ((n + 63) & ~int64_t(63));
  uint32_t* H = vt + ((n + 63) & ~int64_t(63));
  uint32_t* total = H + ntiles * C::NB;
  const int passes = (end_bit + db - 1) / db;
  const size_t smem = size_t(1 + C::WARPS) * C::NB * 4;
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    DLRM_CUDA(cudaFuncSetAttribute(rs_scatter_kernel<C>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  // ping-pong between the input and the scratch copy, the last pass into the output
  uint32_t* sk = keys_a;
  uint32_t* sv = vals_a;
  int shift = 0;
  for (int p = 0; p < passes; ++p) {
    const bool last = p == passes - 1;
    uint32_t* dk = last ? keys_out : (sk == kt ? keys_a : kt);
    uint32_t* dv = last ? vals_out : (sv == vt ? vals_a : vt);
    const int nbits = (end_bit - shift + (passes - p) - 1) / (passes - p);
    const int nb = 1 << nbits;
    launch(rs_hist_kernel<C>, unsigned(ntiles), C::THREADS, 0, s, sk, n, shift, nbits, H, ntiles);
    if (int rc = check_launch("rs_hist_kernel")) return rc;
    launch(rs_prefix_kernel, unsigned((nb * 32 + 255) / 256), 256, 0, s, H, ntiles, nbits, total);
    if (int rc = check_launch("rs_prefix_kernel")) return rc;
    launch(rs_scatter_kernel<C>, unsigned(ntiles), C::THREADS, smem, s, sk, sv, dk, dv, n, shift,
           nbits, H, ntiles, total);
    if (int rc = check_launch("rs_scatter_kernel")) return rc;
    sk = dk;
    sv = dv;
    shift += nbits;
  }
  return 0;
}

using Rs8 = RsCfg<8, 8, 512>;
using Rs12 = RsCfg<12, 8, 1024>;

}  // namespace

size_t stable_sort_scratch(int64_t n) {
  const int64_t t = n > 0 ? n : 1;
  const int64_t h8 = (t + Rs8::TILE - 1) / Rs8::TILE * Rs8::NB;
  const int64_t h12 = (t + Rs12::TILE - 1) / Rs12::TILE * Rs12::NB;
  // key / value ping-pong + histograms + digit totals
  return size_t(2) * size_t((t + 63) & ~int64_t(63)) * 4 + size_t(h8 > h12 ? h8 : h12) * 4 +
         size_t(Rs12::NB) * 4 + 1024;
}

int stable_sort_pairs(uint32_t* keys_a, uint32_t* vals_a, uint32_t* keys_out, uint32_t* vals_out,
                      int64_t n, int end_bit, int digit_bits, void* scratch, cudaStream_t s) {
  if (n <= 0) return 0;
  DLRM_REQUIRE(end_bit >= 1 && end_bit <= 32, "sort: bad key width");
  if (digit_bits == 12)
    return sort_passes<Rs12>(keys_a, vals_a, keys_out, vals_out, n, end_bit, scratch, 12, s);
  return sort_passes<Rs8>(keys_a, vals_a, keys_out, vals_out, n, end_bit, scratch, 8, s);
}

}  // namespace dlrm
