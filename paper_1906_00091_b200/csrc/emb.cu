// Embedding-bag kernels: pooled lookup (forward) and the sorted, deterministic
// sparse backward fused with the SGD row update.
//
// Reference semantics (dlrmkit, pkg/src/dlrmkit/embedding.py):
//   lookup_batch    155-179  strict ascending-position fold per bag, rows
//                            scaled by the per-index weight first (165-166)
//   check_bounds    117-124  lowest offending flat position is reported
//   lookup_backward 182-210  np.unique rows (ascending) + np.add.at, i.e. per
//                            row an ascending-position fold starting at +0.0
//   sgd_step_rows   optim.py:38-46   W[rows] -= lr * values (product first)
//
// HBM layout: all tables of a rank live in ONE row-major fp32 buffer W_all
// (row_base per table); pooled rows go to out[out_offset_t + j*out_stride].
// Gathers are 128-bit (float4) per lane, LPB = min(32, d/4) lanes per bag,
// indices loaded coalesced by the sub-warp and broadcast with shuffles, 4 row
// loads in flight per lane.
#include <stdlib.h>
#include <string.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "radix.cuh"

namespace dlrm {

namespace {

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
};
template <>
struct VecT<1> {
  using T = float;
};

__device__ __forceinline__ float4 ldg_vec(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float ldg_vec(const float* p) { return __ldg(p); }

__device__ __forceinline__ float4 vzero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

__device__ __forceinline__ float4 vmul(float a, float4 v) {
  return make_float4(__fmul_rn(a, v.x), __fmul_rn(a, v.y), __fmul_rn(a, v.z),
                     __fmul_rn(a, v.w));
}
__device__ __forceinline__ float vmul(float a, float v) { return __fmul_rn(a, v); }
__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y),
                     __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
// row update (SGD / Adagrad, see dlrm_update): new value of the parameter
// vector stored at p whose current value is w
__device__ __forceinline__ float4 vupd(const Upd& u, float4* p, float4 w, float4 g) {
  return upd_apply4(u, reinterpret_cast<float*>(p), w, g);
}
__device__ __forceinline__ float vupd(const Upd& u, float* p, float w, float g) {
  return upd_apply(u, p, w, g);
}
template <typename V>
__device__ __forceinline__ V vzero();
template <>
__device__ __forceinline__ float4 vzero<float4>() { return vzero4(); }
template <>
__device__ __forceinline__ float vzero<float>() { return 0.f; }

__device__ __forceinline__ void record_error(int64_t* err_pos, int32_t* err_flag,
                                             int t, int64_t pos) {
  atomicMin(reinterpret_cast<unsigned long long*>(err_pos + t),
            static_cast<unsigned long long>(pos));
  atomicExch(err_flag, 1);
}

template <int LPB>
__device__ __forceinline__ unsigned subgroup_mask() {
  if constexpr (LPB == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31;
    return ((1u << LPB) - 1u) << (lane & ~(LPB - 1));
  }
}

// ---------------------------------------------------------------------------
// forward: one LPB-lane sub-warp per bag; NV vectors of VEC floats per lane.
#ifndef DLRM_EMB_U1
#define DLRM_EMB_U1 4
#define DLRM_EMB_MINB1 4
#endif
template <int VEC, int LPB, int NV>
__global__ void __launch_bounds__(256, NV == 1 ? DLRM_EMB_MINB1 : 2)
emb_fwd_kernel(const float* __restrict__ W, int64_t dim, TableSet ts,
               int64_t num_bags, float* __restrict__ out, int64_t out_stride,
               int64_t* err_pos, int32_t* err_flag) {
  pdl_entry();
  using V = typename VecT<VEC>::T;
  constexpr int U = NV == 1 ? DLRM_EMB_U1 : (NV == 2 ? 4 : 2);  // rows in flight per lane
  const int lane = threadIdx.x & (LPB - 1);
  const int64_t group = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LPB;
  const int64_t total = num_bags * ts.nt;
  if (group >= total) return;
  const unsigned mask = subgroup_mask<LPB>();
  const int t = int(group / num_bags);
  const int64_t j = group - int64_t(t) * num_bags;
  const int64_t* offs = ts.t[t].offsets;
  const int64_t* idxp = ts.t[t].indices;
  const float* wts = ts.t[t].weights;
  const int64_t row_base = ts.t[t].row_base;
  const int64_t num_rows = ts.t[t].num_rows;
  const int64_t lo = __ldg(offs + j), hi = __ldg(offs + j + 1);
  const int64_t nvec = dim / VEC;

  V acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = vzero<V>();
  bool first = true;

  // indices of the next LPB positions are prefetched one chunk ahead
  int64_t nxt_idx = 0;
  float nxt_w = 1.f;
  if (lo + lane < hi) {
    nxt_idx = __ldg(idxp + lo + lane);
    if (wts) nxt_w = __ldg(wts + lo + lane);
  }
  for (int64_t p0 = lo; p0 < hi; p0 += LPB) {
    const int64_t my = p0 + lane;
    const int64_t myidx = nxt_idx;
    const float myw = nxt_w;
    if (my < hi && (myidx < 0 || myidx >= num_rows)) record_error(err_pos, err_flag, t, my);
    if (p0 + LPB + lane < hi) {
      nxt_idx = __ldg(idxp + p0 + LPB + lane);
      if (wts) nxt_w = __ldg(wts + p0 + LPB + lane);
    }
    const int cnt = int(hi - p0 < LPB ? hi - p0 : LPB);
    for (int q = 0; q < cnt; q += U) {
      V r[U][NV];
      float wq[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int src = min(q + u, cnt - 1);
        const int64_t ri = __shfl_sync(mask, myidx, src, LPB);
        wq[u] = __shfl_sync(mask, myw, src, LPB);
        const bool ok = (q + u < cnt) && ri >= 0 && ri < num_rows;
        const V* rowp = reinterpret_cast<const V*>(W + (row_base + ri) * dim);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int64_t v = lane + int64_t(i) * LPB;
          r[u][i] = (ok && v < nvec) ? ldg_vec(rowp + v) : vzero<V>();
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (q + u < cnt) {
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const V val = wts ? vmul(wq[u], r[u][i]) : r[u][i];
            acc[i] = first ? val : vadd(acc[i], val);
          }
          first = false;
        }
      }
    }
  }
  V* o = reinterpret_cast<V*>(out + ts.t[t].out_offset + j * out_stride);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int64_t v = lane + int64_t(i) * LPB;
    if (v < nvec) o[v] = acc[i];
  }
}

// forward for multi-hot bags: one WARP per bag.  A row is LPB = d/4 lanes,
// so one warp-wide load instruction fetches RPI = 32/LPB consecutive rows of
// the bag (U instructions in flight); rows are then folded in strict
// ascending position order by broadcasting each row's float4 with shuffles
// (every lane group keeps the same accumulator).  No divergence between bags
// sharing a warp, 2..8x more rows in flight per warp than one sub-warp/bag.
#ifndef DLRM_EMBW_U
#define DLRM_EMBW_U 4
#endif
template <int LPB>
__global__ void __launch_bounds__(256, 4)
emb_fwd_warp_kernel(const float* __restrict__ W, int64_t dim, TableSet ts,
                    int64_t num_bags, float* __restrict__ out, int64_t out_stride,
                    int64_t* err_pos, int32_t* err_flag) {
  pdl_entry();
  constexpr int RPI = 32 / LPB;
  constexpr int U = RPI >= 4 ? DLRM_EMBW_U / 2 : DLRM_EMBW_U;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPB, col = lane % LPB;
  const int64_t total = num_bags * ts.nt;
  const int64_t nwarps = int64_t(gridDim.x) * (blockDim.x / 32);
  const float4* Wv = reinterpret_cast<const float4*>(W);
  const int64_t nvec = dim / 4;

  // persistent: each warp walks bags bag, bag + nwarps, ...; the next bag's
  // bounds are fetched while the current one is being folded
  int64_t bag = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  int64_t nlo = 0, nhi = 0;
  if (bag < total) {
    const int t0 = int(bag / num_bags);
    const int64_t j0 = bag - int64_t(t0) * num_bags;
    nlo = __ldg(ts.t[t0].offsets + j0);
    nhi = __ldg(ts.t[t0].offsets + j0 + 1);
  }
  for (; bag < total; bag += nwarps) {
    const int t = int(bag / num_bags);
    const int64_t j = bag - int64_t(t) * num_bags;
    const int64_t* idxp = ts.t[t].indices;
    const float* wts = ts.t[t].weights;
    const int64_t row_base = ts.t[t].row_base;
    const int64_t num_rows = ts.t[t].num_rows;
    const int64_t lo = nlo, hi = nhi;
    const int64_t nb = bag + nwarps;
    if (nb < total) {
      const int tn = int(nb / num_bags);
      const int64_t jn = nb - int64_t(tn) * num_bags;
      nlo = __ldg(ts.t[tn].offsets + jn);
      nhi = __ldg(ts.t[tn].offsets + jn + 1);
    }
    float4 acc = vzero4();
    bool first = true;
    int64_t nxt_idx = 0;
    float nxt_w = 1.f;
    if (lo + lane < hi) {
      nxt_idx = __ldg(idxp + lo + lane);
      if (wts) nxt_w = __ldg(wts + lo + lane);
    }
    for (int64_t p0 = lo; p0 < hi; p0 += 32) {
      const int64_t myidx = nxt_idx;
      const float myw = nxt_w;
      if (p0 + lane < hi && (myidx < 0 || myidx >= num_rows))
        record_error(err_pos, err_flag, t, p0 + lane);
      if (p0 + 32 + lane < hi) {
        nxt_idx = __ldg(idxp + p0 + 32 + lane);
        if (wts) nxt_w = __ldg(wts + p0 + 32 + lane);
      }
      const int cnt = int(hi - p0 < 32 ? hi - p0 : 32);
      for (int q = 0; q < cnt; q += RPI * U) {
        float4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int pos = q + u * RPI + sub;
          const int src = pos < cnt ? pos : cnt - 1;
          const int64_t ri = __shfl_sync(0xffffffffu, myidx, src);
          const bool ok = pos < cnt && ri >= 0 && ri < num_rows;
          r[u] = ok ? __ldg(Wv + (row_base + ri) * nvec + col) : vzero4();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int s = 0; s < RPI; ++s) {
            const int pos = q + u * RPI + s;
            const int from = s * LPB + col;
            float4 v;
            v.x = __shfl_sync(0xffffffffu, r[u].x, from);
            v.y = __shfl_sync(0xffffffffu, r[u].y, from);
            v.z = __shfl_sync(0xffffffffu, r[u].z, from);
            v.w = __shfl_sync(0xffffffffu, r[u].w, from);
            const float w = __shfl_sync(0xffffffffu, myw, pos < cnt ? pos : 0);
            if (pos < cnt) {
              if (wts) v = vmul(w, v);
              acc = first ? v : vadd(acc, v);
              first = false;
            }
          }
        }
      }
    }
    if (sub == 0 && col < nvec)
      reinterpret_cast<float4*>(out + ts.t[t].out_offset + j * out_stride)[col] = acc;
  }
}

// ---------------------------------------------------------------------------
// forward, streaming variant (the default for 16-byte-aligned rows).
//
// Work split: the positions of all tables form one space (table t's slots at
// pre[t] + [0, nnz_t)); warp w of nwarps owns the bags whose first position
// falls in [w, w+1) * P / nwarps, i.e. a CONTIGUOUS run of bags balanced by
// rows, found with a 32-ary search over the offsets.  The warp then streams
// that run's rows through an S-slot cp.async ring of CH-row chunks without
// draining at bag boundaries (indices are fetched two chunks ahead, bag ends
// one 32-bag window ahead), and folds every chunk in strict ascending
// position order, emitting a bag when the position reaches its end offset.
constexpr uint32_t kBadRow = 0xffffffffu;  // stream path: tables have < 2^32 - 1 rows

struct StreamIdx {
  int64_t ix;
  float w;
};

// first global bag g = t * nb + j with pre[t] + offs_t[j] >= a (nt * nb if none)
__device__ __forceinline__ int64_t stream_bag_at(const TableSet& ts, int64_t nb,
                                                 const int64_t* pre, const int64_t* last,
                                                 int64_t a) {
  const int lane = threadIdx.x & 31;
  int t = -1;
  for (int base = 0; base < ts.nt && t < 0; base += 32) {
    const int tt = base + lane;
    const bool hit = tt < ts.nt && pre[tt] + last[tt] >= a;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m) t = base + __ffs(m) - 1;
  }
  if (t < 0) return int64_t(ts.nt) * nb;
  const int64_t* offs = ts.t[t].offsets;
  const int64_t target = a - pre[t];
  int64_t lo = 0, hi = nb - 1;  // offs[hi] >= target; answer in [lo, hi]
  while (hi > lo) {
    const int64_t step = (hi - lo + 30) / 31;  // lane 31 probes >= hi
    const int64_t jk = lo + int64_t(lane) * step;
    const bool ge = jk >= hi || __ldg(offs + jk) >= target;
    const int k = __ffs(__ballot_sync(0xffffffffu, ge)) - 1;
    const int64_t nhi = lo + int64_t(k) * step < hi ? lo + int64_t(k) * step : hi;
    lo = k == 0 ? lo : lo + int64_t(k - 1) * step + 1;
    hi = nhi;
  }
  return int64_t(t) * nb + lo;
}

template <int NVM, int CH, int S, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 1)
emb_fwd_stream_kernel(const float* __restrict__ W, int64_t dim, TableSet ts, int64_t nb,
                      float* __restrict__ out, int64_t out_stride, int64_t* err_pos,
                      int32_t* err_flag) {
  pdl_entry();
  constexpr int SLOT = CH * NVM;                  // float4 per ring slot
  constexpr int PER_LANE = (SLOT + 31) / 32;      // 16-byte copies per lane per chunk
  constexpr int NL = NVM >= 32 ? NVM / 32 : 1;    // float4 columns per lane
  constexpr int CW = NVM >= 32 ? 32 : NVM;        // lanes per row
  extern __shared__ float4 smem[];
  __shared__ int64_t pre[DLRM_MAX_TABLES + 1], last[DLRM_MAX_TABLES];
  const int lane = threadIdx.x & 31, wib = threadIdx.x / 32;
  float4* ring = smem + size_t(wib) * S * SLOT;
  float* wring = reinterpret_cast<float*>(smem + size_t(WARPS) * S * SLOT) + wib * S * CH;
  const float4* Wv = reinterpret_cast<const float4*>(W);
  const int64_t nvec = dim / 4;

  if (threadIdx.x < ts.nt) {
    pre[threadIdx.x + 1] = __ldg(ts.t[threadIdx.x].offsets + nb);
    last[threadIdx.x] = __ldg(ts.t[threadIdx.x].offsets + nb - 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pre[0] = 0;
    for (int t = 0; t < ts.nt; ++t) pre[t + 1] += pre[t];
  }
  __syncthreads();
  const int64_t P = pre[ts.nt];
  const int64_t nwarps = int64_t(gridDim.x) * WARPS;
  const int64_t gw = int64_t(blockIdx.x) * WARPS + wib;
  const int64_t g0 = gw == 0 ? 0 : stream_bag_at(ts, nb, pre, last, P * gw / nwarps);
  const int64_t g1 = gw == nwarps - 1 ? int64_t(ts.nt) * nb
                                      : stream_bag_at(ts, nb, pre, last, P * (gw + 1) / nwarps);

  for (int64_t g = g0; g < g1;) {
    const int t = int(g / nb);
    const int64_t j0 = g - int64_t(t) * nb;
    const int64_t j1 = (g1 - int64_t(t) * nb) < nb ? g1 - int64_t(t) * nb : nb;
    g = int64_t(t) * nb + j1;
    const int64_t* offs = ts.t[t].offsets;
    const int64_t* idxp = ts.t[t].indices;
    const float* wts = ts.t[t].weights;
    const int64_t row_base = ts.t[t].row_base;
    const int64_t num_rows = ts.t[t].num_rows;
    float* obase = out + ts.t[t].out_offset;
    const int64_t P0 = __ldg(offs + j0), P1 = __ldg(offs + j1);
    const int nch = int(ceil_div(P1 - P0, CH));
    const float4* Wt = Wv + row_base * NVM;

    // bag ends: lane k of win holds offs[wb + 1 + k]; win_nx the next window
    int64_t wb = j0;
    auto load_win = [&](int64_t base) -> int64_t {
      const int64_t jj = base + 1 + lane;
      return jj <= j1 ? __ldg(offs + jj) : P1;
    };
    int64_t win = load_win(wb), win_nx = load_win(wb + 32);
    int64_t j = j0;
    int64_t bend = __shfl_sync(0xffffffffu, win, 0);

    // index prefetch queue: q0 feeds the next issue, q1 the one after
    auto load_idx = [&](int c) -> StreamIdx {
      StreamIdx r{0, 1.f};
      const int64_t p = P0 + int64_t(c) * CH + lane;
      if (lane < CH && c < nch && p < P1) {
        r.ix = __ldg(idxp + p);
        if (wts) r.w = __ldg(wts + p);
      }
      return r;
    };
    StreamIdx q0 = load_idx(0), q1 = load_idx(1);
    int issued = 0, islot = 0, hot = 0;
    auto issue = [&]() {
      if (issued < nch) {
        const int64_t p0 = P0 + int64_t(issued) * CH;
        const int cnt = int(P1 - p0 < CH ? P1 - p0 : CH);
        // one validated 32-bit row id per lane; kBadRow lanes are zero-filled
        const int64_t ix = q0.ix;
        uint32_t myrow = kBadRow;
        if (lane < cnt) {
          if (ix < 0 || ix >= num_rows) record_error(err_pos, err_flag, t, p0 + lane);
          else myrow = uint32_t(ix);
        }
        float4* slot = ring + islot * SLOT;
        if (wts && lane < CH) wring[islot * CH + lane] = q0.w;
        // Skew detector: a row repeated inside one chunk means a hot working
        // set (e.g. Zipf indices), whose rows all SMs would otherwise fetch
        // from the same few L2 slices; such a warp loads through L1 for the
        // next 8 chunks, where the hot rows hit.  Uniform indices essentially
        // never repeat within a chunk and keep the L1-bypassing path.
        const unsigned peers = __match_any_sync(0xffffffffu, lane < cnt ? myrow : ~0u - lane);
        if (__any_sync(0xffffffffu, lane < cnt && __popc(peers) > 1)) hot = 8;
        else if (hot > 0) --hot;
        if (hot > 0) {
#pragma unroll
          for (int i = 0; i < PER_LANE; ++i) {
            const int e = lane + 32 * i;
            const int r = e / NVM, cc = e % NVM;
            const uint32_t rr = __shfl_sync(0xffffffffu, myrow, r < CH ? r : 0);
            const bool ok = rr != kBadRow;
            if (e < SLOT) cp_async16_l1(slot + e, Wt + size_t(ok ? rr : 0u) * NVM + cc, ok);
          }
        } else {
#pragma unroll
          for (int i = 0; i < PER_LANE; ++i) {
            const int e = lane + 32 * i;
            const int r = e / NVM, cc = e % NVM;
            const uint32_t rr = __shfl_sync(0xffffffffu, myrow, r < CH ? r : 0);
            const bool ok = rr != kBadRow;
            if (e < SLOT) cp_async16(slot + e, Wt + size_t(ok ? rr : 0u) * NVM + cc, ok);
          }
        }
      }
      cp_async_commit();
      ++issued;
      islot = islot == S - 1 ? 0 : islot + 1;
      q0 = q1;
      q1 = load_idx(issued + 1);
    };

    float4 acc[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) acc[k] = vzero4();
    bool first = true;
    auto emit = [&]() {
      float4* o = reinterpret_cast<float4*>(obase + j * out_stride);
#pragma unroll
      for (int k = 0; k < NL; ++k) {
        const int col = lane % CW + 32 * k;
        if (lane < CW && col < nvec) o[col] = acc[k];
        acc[k] = vzero4();
      }
      first = true;
      ++j;
      if (j - wb == 32) {
        wb += 32;
        win = win_nx;
        win_nx = load_win(wb + 32);
      }
      bend = __shfl_sync(0xffffffffu, win, int(j - wb));
    };

#pragma unroll
    for (int k = 0; k < S - 1; ++k) issue();
    for (int c = 0, cs = 0; c < nch; ++c, cs = cs == S - 1 ? 0 : cs + 1) {
      issue();
      cp_async_wait<S - 1>();
      __syncwarp();
      const int64_t p0 = P0 + int64_t(c) * CH;
      const int cnt = int(P1 - p0 < CH ? P1 - p0 : CH);
      const float4* sp = ring + cs * SLOT + lane % CW;  // zero-filled past cnt / bad rows
      const float* wsl = wring + cs * CH;
      auto row = [&](int r, float4 (&v)[NL]) {
#pragma unroll
        for (int k = 0; k < NL; ++k) {
          v[k] = sp[r * NVM + 32 * k];
          if (wts) v[k] = vmul(wsl[r], v[k]);
        }
      };
      int r = 0;
      while (r < cnt) {
        while (p0 + r == bend) emit();
        const int rend = bend - p0 < cnt ? int(bend - p0) : cnt;
        if (first) {
          float4 v[NL];
          row(r, v);
#pragma unroll
          for (int k = 0; k < NL; ++k) acc[k] = v[k];
          first = false;
          ++r;
        }
        for (; r + 4 <= rend; r += 4) {
          float4 v[4][NL];
#pragma unroll
          for (int u = 0; u < 4; ++u) row(r + u, v[u]);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < NL; ++k) acc[k] = vadd(acc[k], v[u][k]);
        }
        for (; r < rend; ++r) {
          float4 v[NL];
          row(r, v);
#pragma unroll
          for (int k = 0; k < NL; ++k) acc[k] = vadd(acc[k], v[k]);
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
    while (j < j1) emit();
  }
}

// ---------------------------------------------------------------------------
// backward, stage 1: one (key = global row, value = slot) pair per index slot
// plus the bag of each live slot.  Slots past a table's nnz get the sentinel
// key so a capacity-sized (graph-static) sort leaves them at the end.
// Blocks [0, bag_blocks) walk bags (LPB lanes per bag, positions strided over
// the lanes: no per-slot search for the bag); the remaining blocks walk the
// capacity and fill the padding slots.
template <int LPB>
__global__ void __launch_bounds__(256)
emb_keys_kernel(TableSet ts, int64_t num_bags, int64_t total_slots, int64_t bag_blocks,
                uint32_t sentinel, uint32_t* __restrict__ keys,
                uint32_t* __restrict__ vals, int32_t* __restrict__ bag_of, int by_bag,
                int64_t* err_pos, int32_t* err_flag) {
  pdl_entry();
  if (blockIdx.x < bag_blocks) {
    const int64_t gb = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LPB;
    const int lane = threadIdx.x % LPB;
    if (gb >= num_bags * ts.nt) return;
    const int t = int(gb / num_bags);
    const int64_t j = gb - int64_t(t) * num_bags;
    const int64_t* offs = ts.t[t].offsets;
    const int64_t lo = __ldg(offs + j), hi = __ldg(offs + j + 1);
    const int64_t* idxp = ts.t[t].indices;
    const int64_t nrows = ts.t[t].num_rows, rbase = ts.t[t].row_base;
    const int64_t cb = ts.cap_base[t], cap = ts.t[t].capacity;
    for (int64_t k = lo + lane; k < hi; k += LPB) {
      if (k >= cap) {  // more indices than the declared capacity: reported, not sorted
        record_error(err_pos, err_flag, t, k);
        break;
      }
      const int64_t idx = __ldg(idxp + k);
      uint32_t key = sentinel;
      if (idx >= 0 && idx < nrows) key = uint32_t(rbase + idx);
      else record_error(err_pos, err_flag, t, k);
      keys[cb + k] = key;
      if (by_bag) {
        vals[cb + k] = uint32_t(j);
      } else {
        vals[cb + k] = uint32_t(cb + k);
        bag_of[cb + k] = int32_t(j);
      }
    }
    return;
  }
  const int64_t s = (int64_t(blockIdx.x) - bag_blocks) * blockDim.x + threadIdx.x;
  if (s >= total_slots) return;
  int lo = 0, hi = ts.nt - 1;  // table of slot s: largest t with cap_base[t] <= s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts.cap_base[mid] <= s) lo = mid; else hi = mid - 1;
  }
  const int64_t k = s - ts.cap_base[lo];
  if (k < __ldg(ts.t[lo].offsets + num_bags)) return;  // live: written by its bag
  keys[s] = sentinel;
  vals[s] = by_bag ? 0u : uint32_t(s);
  if (!by_bag) bag_of[s] = 0;
}

__device__ __forceinline__ int table_of_row(const TableSet& ts, uint32_t row) {
  int lo = 0, hi = ts.nt - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ts.t[mid].row_base <= int64_t(row)) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Run-start flags for the coalesce path.
__global__ void run_flags_kernel(const uint32_t* __restrict__ keys, int64_t n,
                                 uint32_t sentinel, uint32_t* __restrict__ flags) {
  pdl_entry();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = keys[i];
  flags[i] = (k != sentinel && (i == 0 || keys[i - 1] != k)) ? 1u : 0u;
}

__global__ void count_unique_kernel(const uint32_t* uid, const uint32_t* flags,
                                    int64_t n, int64_t* num_unique) {
  pdl_entry();
  if (threadIdx.x == 0 && blockIdx.x == 0)
    *num_unique = n ? int64_t(uid[n - 1]) + int64_t(flags[n - 1]) : 0;
}

// ---------------------------------------------------------------------------
// backward, stage 3: deterministic segmented fold over the sorted slots.
// Chunk c of CH sorted slots belongs to one sub-warp, which owns every run
// (equal-row segment) that STARTS inside the chunk — following it past the
// chunk end if needed.  Per run: acc = +0; acc += g[bag]*a in ascending slot
// order (== ascending position); then either W[row] -= lr*acc (SGD mode) or
// rows_out/values_out[uid] = (row, acc) (coalesce mode).
struct FoldArgs {
  const uint32_t* keys;  // sorted
  const uint32_t* vals;  // sorted by key (stable): bags (by_bag) or slots
  const int32_t* bag_of;  // slot -> bag (slot values only)
  int by_bag;             // 1: no table is weighted, the sort carried the bag itself
  int64_t n;
  uint32_t sentinel;
  const float* grad;
  int64_t grad_stride;
  float* W;  // update mode
  Upd upd;
  const int32_t* err_flag;
  const uint32_t* uid;  // coalesce mode
  int64_t* rows_out;
  float* values_out;
  uint32_t* long_count;  // runs longer than kLongRun are deferred here
  uint4* long_runs;      // (start, end, row, 0)
};

// Runs (equal-row segments) longer than kLongRun slots are folded by the
// segment path (a whole warp per 256-slot segment, 8-32 rows in flight)
// instead of by the one sub-warp that owns the run start (4 rows in flight).
// The fold order within a segment is the same strict order, so results do
// not depend on the threshold; 16 measured best (Kaggle-shaped step 0.234 ->
// 0.201 ms: its small tables make many 20-700-slot runs; c3 unchanged).
#ifndef DLRM_LONG_RUN
#define DLRM_LONG_RUN 16
#endif
constexpr int kLongRun = DLRM_LONG_RUN;
// ring depth of the fold's cp.async fast path (0: register batches only)
// (measured at the c3 shape: 4 -> step 0.413 ms; register batches 0.425;
// 8 -> 0.420; 12 -> 0.440); narrow rows (<= 16 floats) keep the register
// batches (Kaggle-shaped step 0.197 vs 0.202 ms)
#ifndef DLRM_FOLD_RING
#define DLRM_FOLD_RING 4
#endif

template <int LPB>
constexpr int fold_groups() { return 256 / LPB < 32 ? 256 / LPB : 32; }

// Rows up to 128 floats (NV == 1): registers capped for 4 blocks (32 warps)
// per SM — the apply is bound by the rows in flight; measured on B200 at the
// c3 shape (8 x 1M x 64, 827K lookups): 127 us at 3 blocks/SM (80 registers),
// 102 us at 4 (64 registers, a few bytes of spills).
// CH sorted slots per chunk (and per staged batch): 32, or 8 when the
// lookups are few (the chunks are the kernel's only parallelism: at the
// Kaggle shape, 53 k one-index bags, CH = 32 left 52 CTAs).
template <int VEC, int LPB, int NV, bool COALESCE, int CH>
__global__ void __launch_bounds__(fold_groups<LPB>() * LPB, NV == 1 ? 4 : 1)
emb_fold_kernel(FoldArgs fa, TableSet ts, int64_t dim) {
  pdl_entry();
  using V = typename VecT<VEC>::T;
  constexpr int U = COALESCE ? 8 : 4;  // gradient rows in flight per lane
  constexpr int GROUPS = fold_groups<LPB>();
  __shared__ uint32_t s_key[GROUPS][CH];
  __shared__ int64_t s_goff[GROUPS][CH];
  __shared__ float s_w[GROUPS][CH];

  const int lane = threadIdx.x & (LPB - 1);
  const int g = threadIdx.x / LPB;
  const unsigned mask = subgroup_mask<LPB>();
  const int64_t chunk = int64_t(blockIdx.x) * GROUPS + g;
  const int64_t start = chunk * CH;
  if (start >= fa.n) return;
  if (!COALESCE && fa.err_flag && *fa.err_flag) return;
  const int64_t limit = start + CH < fa.n ? start + CH : fa.n;  // owned run starts
  const int64_t nvec = dim / VEC;

  // stage keys, gradient-row offsets and weights of slots [base, base+CH)
  auto stage = [&](int64_t base) -> int {
    const int cnt = int(fa.n - base < CH ? fa.n - base : CH);
    __syncwarp(mask);
    for (int i = lane; i < cnt; i += LPB) {
      const uint32_t k = fa.keys[base + i];
      s_key[g][i] = k;
      int64_t goff = 0;
      float w = 1.f;
      if (k != fa.sentinel) {
        const int t = table_of_row(ts, k);
        const uint32_t v = fa.vals[base + i];
        if (fa.by_bag) {  // one memory level less on the staging path
          goff = ts.t[t].out_offset + int64_t(v) * fa.grad_stride;
        } else {
          goff = ts.t[t].out_offset + int64_t(fa.bag_of[v]) * fa.grad_stride;
          if (ts.t[t].weights) w = __ldg(ts.t[t].weights + (v - ts.cap_base[t]));
        }
      }
      s_goff[g][i] = goff;
      s_w[g][i] = w;
    }
    __syncwarp(mask);
    return cnt;
  };

  int64_t base = start;
  int cnt = stage(base);
  int i = 0;
  if (start > 0) {  // skip the tail of a run that started in an earlier chunk
    const uint32_t prev = fa.keys[start - 1];
    while (i < cnt && s_key[g][i] == prev) ++i;
  }
  if (i >= cnt) return;
  uint32_t cur = s_key[g][i];
  if (cur == fa.sentinel) return;
  int64_t run_start = base + i;

#if DLRM_FOLD_RING > 0
  if constexpr (!COALESCE && VEC == 4 && NV == 1 && LPB >= 8) {
    // SGD / Adagrad fast path (rows <= 128 floats): a per-sub-warp ring of
    // RR slots in shared memory, each the gradient row of one sorted slot and
    // (for a run start) its table row, filled by cp.async RR slots ahead of
    // the fold — RR rows in flight per sub-warp without holding them in
    // registers.  Same arithmetic, same order as the register path below.
    constexpr int RR = DLRM_FOLD_RING;
    extern __shared__ float4 fold_ring[];
    float4* rg = fold_ring + (size_t(g) * RR * 2) * LPB;  // [RR][LPB] gradient rows
    float4* rw = rg + size_t(RR) * LPB;                    // [RR][LPB] table rows
    const bool col_ok = lane < nvec;
    float4 acc4 = vzero4(), w4 = vzero4();
    bool first = true;
    // issue slot jj of the staged chunk into ring position q
    auto issue = [&](int jj, int q, uint32_t prevk, bool first_slot) {
      if (jj < cnt) {
        const uint32_t k = s_key[g][jj];
        const bool live = k != fa.sentinel;
        const bool starts = live && (first_slot || k != prevk);
        const float4* src = reinterpret_cast<const float4*>(fa.grad + s_goff[g][jj]) + lane;
        cp_async16(rg + q * LPB + lane, live && col_ok ? src : reinterpret_cast<const float4*>(fa.grad),
                   live && col_ok);
        const float4* wsrc = reinterpret_cast<const float4*>(fa.W + int64_t(k) * dim) + lane;
        cp_async16(rw + q * LPB + lane, starts && col_ok ? wsrc : reinterpret_cast<const float4*>(fa.W),
                   starts && col_ok);
      }
      cp_async_commit();
    };
    auto flush4 = [&](uint32_t row) {
      float4* wrow = reinterpret_cast<float4*>(fa.W + int64_t(row) * dim);
      if (col_ok) wrow[lane] = vupd(fa.upd, wrow + lane, w4, acc4);
    };
    while (true) {
      // prologue: RR slots in flight
      const int j0 = i;
      for (int r = 0; r < RR; ++r)
        issue(j0 + r, r, j0 + r > 0 ? s_key[g][j0 + r - 1] : cur, first && r == 0);
      for (int jj = j0, q = 0; jj < cnt; ++jj, q = q == RR - 1 ? 0 : q + 1) {
        cp_async_wait<RR - 1>();
        __syncwarp(mask);
        const uint32_t k = s_key[g][jj];
        if (first) {
          w4 = rw[q * LPB + lane];
          first = false;
        } else if (k != cur) {
          flush4(cur);
          if (k == fa.sentinel || base + jj >= limit) {
            cp_async_wait<0>();
            return;
          }
          cur = k;
          run_start = base + jj;
          acc4 = vzero4();
          w4 = rw[q * LPB + lane];
        }
        const float4 r4 = rg[q * LPB + lane];
        acc4 = vadd(acc4, vmul(s_w[g][jj], r4));
        __syncwarp(mask);
        issue(jj + RR, q, s_key[g][jj + RR - 1 < cnt ? jj + RR - 1 : 0], false);
      }
      cp_async_wait<0>();
      base += CH;
      if (base >= fa.n) break;
      if (fa.keys[base] != cur) break;  // our last run ends exactly here
      if (base - run_start >= CH) {
        int64_t lo2 = base, step = CH;
        int64_t hi2 = base + step;
        while (hi2 < fa.n && fa.keys[hi2] == cur) {
          lo2 = hi2;
          step *= 2;
          hi2 = lo2 + step;
        }
        if (hi2 > fa.n) hi2 = fa.n;
        while (hi2 - lo2 > 1) {
          const int64_t mid = (lo2 + hi2) >> 1;
          if (fa.keys[mid] == cur) lo2 = mid; else hi2 = mid;
        }
        const int64_t run_end = lo2 + 1;
        if (run_end - run_start > kLongRun) {
          if (lane == 0) {
            const uint32_t slot = atomicAdd(fa.long_count, 1u);
            fa.long_runs[slot] = make_uint4(uint32_t(run_start), uint32_t(run_end), cur, 0u);
          }
          return;
        }
      }
      cnt = stage(base);
      i = 0;
    }
    flush4(cur);
    return;
  }
#endif

  V acc[NV], wcur[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = vzero<V>();
  // SGD mode: the table row of each run is prefetched when the run's first
  // element is loaded, so the read-modify-write at the run's end does not
  // wait a full memory latency per row
  if constexpr (!COALESCE) {
    const V* wr0 = reinterpret_cast<const V*>(fa.W + int64_t(cur) * dim);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int64_t c = lane + int64_t(v) * LPB;
      wcur[v] = c < nvec ? wr0[c] : vzero<V>();
    }
  }

  auto flush = [&](uint32_t row, int64_t rs) {
    if constexpr (COALESCE) {
      const uint32_t u = fa.uid[rs];
      const int t = table_of_row(ts, row);
      if (lane == 0) fa.rows_out[u] = int64_t(row) - ts.t[t].row_base;
      V* dst = reinterpret_cast<V*>(fa.values_out + int64_t(u) * dim);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = lane + int64_t(v) * LPB;
        if (c < nvec) dst[c] = acc[v];
      }
    } else {
      V* wrow = reinterpret_cast<V*>(fa.W + int64_t(row) * dim);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = lane + int64_t(v) * LPB;
        if (c < nvec) wrow[c] = vupd(fa.upd, wrow + c, wcur[v], acc[v]);
      }
    }
  };

  // Runs starting in [start, limit) are ours; the last one is followed past
  // `limit` batch by batch (a long run of a hot row keeps U rows in flight).
  while (true) {
    for (; i < cnt; i += U) {
      V r[U][NV];
      V wr[COALESCE ? 1 : U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ii = i + u < cnt ? i + u : cnt - 1;
        const uint32_t k = s_key[g][ii];
        const bool live = (i + u < cnt) && k != fa.sentinel;
        const V* src = reinterpret_cast<const V*>(fa.grad + s_goff[g][ii]);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int64_t c = lane + int64_t(v) * LPB;
          r[u][v] = (live && c < nvec) ? ldg_vec(src + c) : vzero<V>();
        }
        if constexpr (!COALESCE) {
          const uint32_t prev = (i + u == 0) ? cur : s_key[g][ii - (ii > 0 ? 1 : 0)];
          const bool starts = live && (i + u == 0 ? k != cur : k != prev);
          const V* wsrc = reinterpret_cast<const V*>(fa.W + int64_t(k) * dim);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int64_t c = lane + int64_t(v) * LPB;
            wr[u][v] = (starts && c < nvec) ? wsrc[c] : vzero<V>();
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ii = i + u;
        if (ii >= cnt) break;
        const uint32_t k = s_key[g][ii];
        if (k != cur) {
          flush(cur, run_start);
          if (k == fa.sentinel || base + ii >= limit) return;
          cur = k;
          run_start = base + ii;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            acc[v] = vzero<V>();
            if constexpr (!COALESCE) wcur[v] = wr[u][v];
          }
        }
        const float w = s_w[g][ii];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = vadd(acc[v], vmul(w, r[u][v]));  // fl(1*x)==x
      }
    }
    base += CH;
    if (base >= fa.n) break;
    if (fa.keys[base] != cur) break;  // our last run ends exactly here
    if (base - run_start >= CH) {
      // a hot row: find the run end (galloping search on the sorted keys);
      // a long run is handed to emb_long_run_kernel, which folds it with a
      // whole CTA (the strict order is kept there), and dropped here
      int64_t lo2 = base, step = CH;
      int64_t hi2 = base + step;
      while (hi2 < fa.n && fa.keys[hi2] == cur) {
        lo2 = hi2;
        step *= 2;
        hi2 = lo2 + step;
      }
      if (hi2 > fa.n) hi2 = fa.n;
      while (hi2 - lo2 > 1) {  // keys[lo2] == cur, keys[hi2] != cur (or end)
        const int64_t mid = (lo2 + hi2) >> 1;
        if (fa.keys[mid] == cur) lo2 = mid; else hi2 = mid;
      }
      const int64_t run_end = lo2 + 1;
      if (run_end - run_start > kLongRun) {
        if (lane == 0) {
          const uint32_t slot = atomicAdd(fa.long_count, 1u);
          fa.long_runs[slot] = make_uint4(uint32_t(run_start), uint32_t(run_end), cur, 0u);
        }
        return;
      }
    }
    cnt = stage(base);
    i = 0;
  }
  flush(cur, run_start);
}

// One CTA per deferred long run (a hot row): stage CHUNK gradient rows at a
// time into shared memory with all threads, then fold them in strict
// ascending slot order (lanes = columns) — the same result as the per-run
// fold, with the loads of a hot row spread over a whole CTA.
template <bool COALESCE>
__global__ void __launch_bounds__(256)
emb_long_run_kernel(FoldArgs fa, TableSet ts, int64_t dim, uint32_t max_runs) {
  pdl_entry();
  constexpr int CHUNK = 64;
  extern __shared__ float s_rows[];  // [CHUNK][dim]
  __shared__ int64_t s_goff[CHUNK];
  __shared__ float s_w[CHUNK];
  if (!COALESCE && fa.err_flag && *fa.err_flag) return;
  const uint32_t nruns = min(*fa.long_count, max_runs);
  for (uint32_t r = blockIdx.x; r < nruns; r += gridDim.x) {
  const uint4 run = fa.long_runs[r];
  const int64_t s0 = run.x, s1 = run.y;
  const uint32_t row = run.z;
  const int t = table_of_row(ts, row);
  float acc = 0.f;  // thread c < dim owns column c
  for (int64_t p0 = s0; p0 < s1; p0 += CHUNK) {
    const int cnt = int(s1 - p0 < CHUNK ? s1 - p0 : CHUNK);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const uint32_t v = fa.vals[p0 + threadIdx.x];
      const int64_t bag = fa.by_bag ? int64_t(v) : int64_t(fa.bag_of[v]);
      s_goff[threadIdx.x] = ts.t[t].out_offset + bag * fa.grad_stride;
      s_w[threadIdx.x] = (!fa.by_bag && ts.t[t].weights)
                             ? __ldg(ts.t[t].weights + (v - ts.cap_base[t])) : 1.f;
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < int64_t(cnt) * dim; e += blockDim.x) {
      const int i = int(e / dim), c = int(e - int64_t(i) * dim);
      s_rows[e] = __ldg(fa.grad + s_goff[i] + c);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < dim; c += blockDim.x) {
      float a = acc;
      for (int i = 0; i < cnt; ++i) a = __fadd_rn(a, __fmul_rn(s_w[i], s_rows[i * dim + c]));
      acc = a;
    }
  }
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    if constexpr (COALESCE) {
      const uint32_t u = fa.uid[s0];
      fa.values_out[int64_t(u) * dim + c] = acc;
      if (c == 0) fa.rows_out[u] = int64_t(row) - ts.t[t].row_base;
    } else {
      float* w = fa.W + int64_t(row) * dim + c;
      *w = upd_apply(fa.upd, w, *w, acc);
    }
  }
  }  // runs (grid-stride)
}

__global__ void err_reset_kernel(int64_t* err_pos, int32_t nt, int32_t* err_flag) {
  pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nt) err_pos[i] = INT64_MAX;
  if (i == 0 && err_flag) *err_flag = 0;
}

// The offending index VALUE of each table's first bad position, read on the
// device from the batch that ran (the host's copy of the indices may already
// hold the next batch when the step was pipelined).
__global__ void err_resolve_kernel(TableSet ts, const int64_t* __restrict__ err_pos,
                                   const int32_t* __restrict__ err_flag,
                                   int64_t* __restrict__ err_val) {
  pdl_entry();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ts.nt) return;
  const int64_t p = err_pos[t];
  int64_t v = 0;
  if (*err_flag && p != INT64_MAX && p >= 0 && p < ts.t[t].capacity) v = ts.t[t].indices[p];
  err_val[t] = v;
}

template <int VEC>
__global__ void sgd_rows_kernel(float* __restrict__ W, int64_t dim,
                                const int64_t* __restrict__ rows,
                                const float* __restrict__ values, int64_t n,
                                Upd u) {
  pdl_entry();
  using V = typename VecT<VEC>::T;
  const int64_t nvec = dim / VEC;
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * nvec) return;
  const int64_t i = e / nvec, c = e - i * nvec;
  V* w = reinterpret_cast<V*>(W + rows[i] * dim) + c;
  const V g = reinterpret_cast<const V*>(values + i * dim)[c];
  *w = vupd(u, w, *w, g);
}

// Hot rows (deferred long runs) are reduced in three steps so that a single
// row's contributions are spread over many warps:
//   seg_plan:    one CTA: segment counts ceil(len / kSeg) -> prefix seg_base,
//                and seg_run[segment] = run
//   seg_fold:    one warp per segment: strict ascending fold of its kSeg
//                slots (RPI rows per warp instruction, U in flight, folded in
//                order through shuffles) -> partial[segment]
//   seg_combine: one CTA per run: partials added in ascending segment order,
//                then the SGD row update (or the coalesced output).
// A run of <= kSeg slots is one segment, i.e. bit-identical to the strict
// fold; hotter rows become a fixed tree of strict folds (deterministic).
constexpr int kSeg = 256;

__global__ void seg_plan_kernel(FoldArgs fa, uint32_t max_runs, uint32_t max_segs,
                                uint32_t* seg_base, uint32_t* seg_run) {
  pdl_entry();
  __shared__ uint32_t s_tot[1024];
  const uint32_t nruns = min(*fa.long_count, max_runs);
  // per-thread contiguous run range -> local counts -> block scan
  const uint32_t per = (nruns + blockDim.x - 1) / blockDim.x;
  const uint32_t r0 = threadIdx.x * per, r1 = min(nruns, r0 + per);
  uint32_t cnt = 0;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint4 run = fa.long_runs[r];
    cnt += (run.y - run.x + kSeg - 1) / kSeg;
  }
  s_tot[threadIdx.x] = cnt;
  __syncthreads();
  for (int o = 1; o < int(blockDim.x); o <<= 1) {  // inclusive scan
    const uint32_t v = threadIdx.x >= unsigned(o) ? s_tot[threadIdx.x - o] : 0u;
    __syncthreads();
    s_tot[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t base = s_tot[threadIdx.x] - cnt;
  for (uint32_t r = r0; r < r1; ++r) {
    const uint4 run = fa.long_runs[r];
    const uint32_t ns = (run.y - run.x + kSeg - 1) / kSeg;
    seg_base[r] = base;
    for (uint32_t k = 0; k < ns && base + k < max_segs; ++k) seg_run[base + k] = r;
    base += ns;
  }
  if (threadIdx.x == blockDim.x - 1) seg_base[max_runs] = min(s_tot[threadIdx.x], max_segs);
}

#ifndef DLRM_SEG_U
#define DLRM_SEG_U 32  // cap; Zipf c5 point d = 64: apply 127 -> 115 us (16 rows), d = 128: 164 -> 160 us
#endif
template <int LPB, int NV>
__global__ void __launch_bounds__(256)
seg_fold_kernel(FoldArgs fa, TableSet ts, int64_t dim, uint32_t max_runs,
                const uint32_t* seg_base, const uint32_t* seg_run, float* partial) {
  pdl_entry();
  constexpr int RPI = 32 / LPB;
  // U * RPI gradient rows in flight per warp: the whole 32-slot batch
  constexpr int U = NV == 1 ? (32 / RPI < DLRM_SEG_U ? 32 / RPI : DLRM_SEG_U) : 2;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPB, col = lane % LPB;
  const uint32_t nseg = seg_base[max_runs];
  const uint32_t nwarps = gridDim.x * blockDim.x / 32;
  for (uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) / 32; seg < nseg; seg += nwarps) {
  const uint32_t r = seg_run[seg];
  const uint4 run = fa.long_runs[r];
  const uint32_t row = run.z;
  const int t = table_of_row(ts, row);
  const int64_t nvec = dim / 4;
  const int64_t a = int64_t(run.x) + int64_t(seg - seg_base[r]) * kSeg;
  const int64_t b = a + kSeg < int64_t(run.y) ? a + kSeg : int64_t(run.y);
  const float* wts = ts.t[t].weights;
  const float4* G = reinterpret_cast<const float4*>(fa.grad);
  float4 acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = vzero4();
  for (int64_t p0 = a; p0 < b; p0 += 32) {
    const int cnt = int(b - p0 < 32 ? b - p0 : 32);
    int64_t goff = 0;  // float4 offset of this lane's slot's gradient row
    float w = 1.f;
    if (lane < cnt) {
      const uint32_t v = fa.vals[p0 + lane];
      const int64_t bag = fa.by_bag ? int64_t(v) : int64_t(fa.bag_of[v]);
      goff = (ts.t[t].out_offset + bag * fa.grad_stride) / 4;
      if (wts && !fa.by_bag) w = __ldg(wts + (v - ts.cap_base[t]));
    }
    for (int q = 0; q < cnt; q += RPI * U) {
      float4 rr[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int pos = q + u * RPI + sub;
        const int64_t go = __shfl_sync(0xffffffffu, goff, pos < cnt ? pos : 0);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int64_t c = col + int64_t(v) * LPB;
          rr[u][v] = (pos < cnt && c < nvec) ? __ldg(G + go + c) : vzero4();
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int si = 0; si < RPI; ++si) {
          const int pos = q + u * RPI + si;
          const float wp = __shfl_sync(0xffffffffu, w, pos < cnt ? pos : 0);
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            float4 x;
            const int from = si * LPB + col;
            x.x = __shfl_sync(0xffffffffu, rr[u][v].x, from);
            x.y = __shfl_sync(0xffffffffu, rr[u][v].y, from);
            x.z = __shfl_sync(0xffffffffu, rr[u][v].z, from);
            x.w = __shfl_sync(0xffffffffu, rr[u][v].w, from);
            if (pos < cnt) acc[v] = vadd(acc[v], vmul(wp, x));
          }
        }
      }
    }
  }
  if (sub == 0) {
    if (run.y - run.x <= uint32_t(kSeg)) {
      // a single-segment run is finished here (seg_combine skips it): the
      // combine of one partial is the partial itself
      if (fa.values_out) {  // coalesce mode (lookup_backward)
        const uint32_t u = fa.uid[run.x];
        if (col == 0) fa.rows_out[u] = int64_t(row) - ts.t[t].row_base;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int64_t c = col + int64_t(v) * LPB;
          if (c < nvec) reinterpret_cast<float4*>(fa.values_out + int64_t(u) * dim)[c] = acc[v];
        }
      } else if (!(fa.err_flag && *fa.err_flag)) {
        float4* wrow = reinterpret_cast<float4*>(fa.W + int64_t(row) * dim);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int64_t c = col + int64_t(v) * LPB;
          if (c < nvec) wrow[c] = vupd(fa.upd, wrow + c, wrow[c], acc[v]);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t c = col + int64_t(v) * LPB;
        if (c < nvec) reinterpret_cast<float4*>(partial + int64_t(seg) * dim)[c] = acc[v];
      }
    }
  }
  }  // segments (grid-stride)
}

template <bool COALESCE>
__global__ void __launch_bounds__(128)
seg_combine_kernel(FoldArgs fa, TableSet ts, int64_t dim, uint32_t max_runs,
                   const uint32_t* seg_base, const float* partial) {
  pdl_entry();
  if (!COALESCE && fa.err_flag && *fa.err_flag) return;
  const uint32_t nruns = min(*fa.long_count, max_runs);
  for (uint32_t r = blockIdx.x; r < nruns; r += gridDim.x) {
  const uint4 run = fa.long_runs[r];
  const uint32_t row = run.z;
  const int t = table_of_row(ts, row);
  const uint32_t g0 = seg_base[r];
  const uint32_t ns = (run.y - run.x + kSeg - 1) / kSeg;
  if (ns <= 1) continue;  // finished by seg_fold_kernel
  for (int64_t c = threadIdx.x; c < dim; c += blockDim.x) {
    // partials added in segment order; loads issued 8 ahead of the adds
    const float* pc = partial + int64_t(g0) * dim + c;
    float v = pc[0];
    uint32_t k = 1;
    for (; k + 8 <= ns; k += 8) {
      float q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = pc[int64_t(k + j) * dim];
#pragma unroll
      for (int j = 0; j < 8; ++j) v = __fadd_rn(v, q[j]);
    }
    for (; k < ns; ++k) v = __fadd_rn(v, pc[int64_t(k) * dim]);
    if constexpr (COALESCE) {
      const uint32_t u = fa.uid[run.x];
      fa.values_out[int64_t(u) * dim + c] = v;
      if (c == 0) fa.rows_out[u] = int64_t(row) - ts.t[t].row_base;
    } else {
      float* w = fa.W + int64_t(row) * dim + c;
      *w = upd_apply(fa.upd, w, *w, v);
    }
  }
  }  // runs (grid-stride)
}

// ---------------------------------------------------------------------------
// dispatch helpers

int fill_tableset(TableSet& ts, const dlrm_table_desc* tables, int32_t nt) {
  DLRM_REQUIRE(tables != nullptr && nt >= 1 && nt <= DLRM_MAX_TABLES,
               "table count must be in [1, DLRM_MAX_TABLES]");
  ts.nt = nt;
  ts.cap_base[0] = 0;
  for (int i = 0; i < nt; ++i) {
    ts.t[i] = tables[i];
    DLRM_REQUIRE(i == 0 || tables[i].row_base >= tables[i - 1].row_base,
                 "table row_base must be nondecreasing");
    DLRM_REQUIRE(tables[i].capacity >= 0, "negative capacity");
    ts.cap_base[i + 1] = ts.cap_base[i] + tables[i].capacity;
  }
  for (int i = nt; i < DLRM_MAX_TABLES; ++i) ts.t[i] = dlrm_table_desc{};
  return 0;
}

bool vec4_ok(int64_t dim, const void* a, int64_t stride, int64_t off) {
  return dim % 4 == 0 && (reinterpret_cast<uintptr_t>(a) % 16) == 0 &&
         stride % 4 == 0 && off % 4 == 0;
}

template <int VEC, int LPB, int NV>
void launch_fwd(const float* W, int64_t dim, const TableSet& ts, int64_t nb,
                float* out, int64_t stride, int64_t* ep, int32_t* ef,
                cudaStream_t s) {
  const int64_t threads = nb * ts.nt * LPB;
  launch(emb_fwd_kernel<VEC, LPB, NV>, unsigned(ceil_div(threads, 256)), 256, 0, s, W, dim, ts, nb, out, stride, ep, ef);
}

template <int NVM, int CH, int S, int WARPS>
int launch_stream(const float* W, int64_t dim, const TableSet& ts, int64_t nb, float* out,
                  int64_t stride, int64_t* ep, int32_t* ef, cudaStream_t s) {
  const size_t smem = size_t(WARPS) * S * (CH * NVM * 16 + CH * 4);
  auto kern = emb_fwd_stream_kernel<NVM, CH, S, WARPS>;
  static bool attr = false;
  if (!attr) {
    DLRM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  // DLRM_EMB_FWD_CTAS: measurement override of the persistent grid
  static const int ctas = getenv("DLRM_EMB_FWD_CTAS") ? atoi(getenv("DLRM_EMB_FWD_CTAS")) : kNumSMs;
  launch(kern, unsigned(ctas > 0 && ctas <= kNumSMs ? ctas : kNumSMs), 32 * WARPS, smem, s, W,
         dim, ts, nb, out, stride, ep, ef);
  return check_launch("emb_fwd_stream_kernel");
}

struct WsLayout {
  size_t keys_a, keys_b, vals_a, vals_b, bag, flags, uid, err, longs, segb, segr, part,
      temp, total, temp_bytes;
  uint32_t max_long, max_segs;
};

WsLayout ws_layout(int64_t n, int64_t dim) {
  WsLayout L{};
  size_t sort_bytes = 0, scan_bytes = 0;
  // keys_a/vals_a -> keys_b/vals_b (CUB, or radix.cu with DLRM_SORT=radix*,
  // keeps its ping-pong buffers in temp); sized for the widest key range
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                  (uint32_t*)nullptr, int(n > 0 ? n : 1), 0, 32);
  if (stable_sort_scratch(n) > sort_bytes) sort_bytes = stable_sort_scratch(n);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (uint32_t*)nullptr,
                                (uint32_t*)nullptr, int(n > 0 ? n : 1));
  const size_t a = 256, e = align_up(size_t(n > 0 ? n : 1) * 4, a);
  L.keys_a = 0;
  L.keys_b = L.keys_a + e;
  L.vals_a = L.keys_b + e;
  L.vals_b = L.vals_a + e;
  L.bag = L.vals_b + e;
  L.flags = L.bag + e;
  L.uid = L.flags + e;
  L.err = L.uid + e;
  L.longs = L.err + align_up((DLRM_MAX_TABLES + 1) * 8, a);
  L.max_long = uint32_t((n > 0 ? n : 1) / kLongRun + 1);
  L.max_segs = uint32_t((n > 0 ? n : 1) / kSeg + L.max_long + 1);
  L.segb = L.longs + align_up(16 + size_t(L.max_long) * 16, a);
  L.segr = L.segb + align_up(size_t(L.max_long + 1) * 4, a);
  L.part = L.segr + align_up(size_t(L.max_segs) * 4, a);
  L.temp = L.part + align_up(size_t(L.max_segs) * size_t(dim > 0 ? dim : 1) * 4, a);
  L.temp_bytes = align_up(sort_bytes > scan_bytes ? sort_bytes : scan_bytes, a);
  L.total = L.temp + L.temp_bytes;
  return L;
}

int end_bit_for(int64_t total_rows) {
  int b = 1;
  while (b < 32 && (int64_t(1) << b) <= total_rows) ++b;
  return b;  // total_rows < 2^b, so sentinel = 2^b - 1 > every real row
}

// The sort's value: the bag of the lookup when no table is weighted (the
// backward then reads the gradient row without a slot -> bag lookup), else
// the slot (for its weight) with the bag in bag_of.  The sort is stable, so
// either way equal rows keep ascending-position order.
int by_bag_values(const TableSet& ts) {
  for (int t = 0; t < ts.nt; ++t)
    if (ts.t[t].weights) return 0;
  return 1;
}

// Sort (row, slot) pairs of all tables into keys_b / vals_b of the workspace.
int sort_pairs(const TableSet& ts, int64_t nb, char* ws, const WsLayout& L, int64_t n,
               int64_t* err_pos, int32_t* err_flag, uint32_t sentinel, int end_bit,
               cudaStream_t s) {
  uint32_t* ka = reinterpret_cast<uint32_t*>(ws + L.keys_a);
  uint32_t* kb = reinterpret_cast<uint32_t*>(ws + L.keys_b);
  uint32_t* va = reinterpret_cast<uint32_t*>(ws + L.vals_a);
  uint32_t* vb = reinterpret_cast<uint32_t*>(ws + L.vals_b);
  int32_t* bag = reinterpret_cast<int32_t*>(ws + L.bag);
  {
    // lanes per bag from the capacity-average pooling factor
    const double avg = double(n) / double(nb * ts.nt > 0 ? nb * ts.nt : 1);
    const int lpb = avg >= 12.0 ? 32 : (avg >= 3.0 ? 8 : 1);
    const int64_t bag_blocks = ceil_div(nb * ts.nt * lpb, 256);
    const unsigned grid = unsigned(bag_blocks + ceil_div(n, 256));
    if (lpb == 32)
      launch(emb_keys_kernel<32>, grid, 256, 0, s, ts, nb, n, bag_blocks, sentinel, ka, va, bag, by_bag_values(ts), err_pos, err_flag);
    else if (lpb == 8)
      launch(emb_keys_kernel<8>, grid, 256, 0, s, ts, nb, n, bag_blocks, sentinel, ka, va, bag, by_bag_values(ts), err_pos, err_flag);
    else
      launch(emb_keys_kernel<1>, grid, 256, 0, s, ts, nb, n, bag_blocks, sentinel, ka, va, bag, by_bag_values(ts), err_pos, err_flag);
    if (int rc = check_launch("emb_keys_kernel")) return rc;
  }
  // the hand-written radix sort (radix.cu) on request; the library onesweep
  // sort measured faster inside the step (see radix.cu)
  const char* alt = getenv("DLRM_SORT");
  if (alt && strncmp(alt, "radix", 5) == 0)
    return stable_sort_pairs(ka, va, kb, vb, n, end_bit, atoi(alt + 5) == 12 ? 12 : 8,
                             ws + L.temp, s);
  size_t tb = L.temp_bytes;
  DLRM_CUDA(cub::DeviceRadixSort::SortPairs(ws + L.temp, tb, ka, kb, va, vb, int(n), 0, end_bit, s));
  count_launch(end_bit / 8 + 2);
  return 0;
}

template <int VEC, int LPB, int NV, bool CO>
void launch_fold(const FoldArgs& fa, const TableSet& ts, int64_t dim,
                 cudaStream_t s) {
  constexpr int GROUPS = fold_groups<LPB>();
  // fewer than ~1k threads per SM with 32-slot chunks: 8-slot chunks
  const bool ring = DLRM_FOLD_RING > 0 && !CO && VEC == 4 && NV == 1 && LPB >= 8;
  const size_t smem = ring ? size_t(GROUPS) * 2 * (DLRM_FOLD_RING > 0 ? DLRM_FOLD_RING : 1) * LPB * 16 : 0;
  auto go = [&](auto kern, int64_t chunks) {
    static bool attr = false;
    if (smem > 0 && !attr) {  // dynamic + the static staging arrays may pass 48 KB
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      attr = true;
    }
    launch(kern, unsigned(ceil_div(chunks, GROUPS)), GROUPS * LPB, smem, s, fa, ts, dim);
  };
  if (ceil_div(fa.n, 32) * LPB < int64_t(kNumSMs) * 1024)
    go(emb_fold_kernel<VEC, LPB, NV, CO, 8>, ceil_div(fa.n, 8));
  else
    go(emb_fold_kernel<VEC, LPB, NV, CO, 32>, ceil_div(fa.n, 32));
}

template <bool CO>
int dispatch_fold(const FoldArgs& fa, const TableSet& ts, int64_t dim, bool v4,
                  cudaStream_t s);

// fold + deferred long runs (hot rows)
template <bool CO>
int run_fold(FoldArgs fa, const TableSet& ts, int64_t dim, bool v4, char* ws,
             const WsLayout& L, cudaStream_t s) {
  fa.long_count = reinterpret_cast<uint32_t*>(ws + L.longs);
  fa.long_runs = reinterpret_cast<uint4*>(ws + L.longs + 16);
  DLRM_CUDA(cudaMemsetAsync(fa.long_count, 0, sizeof(uint32_t), s));
  if (int rc = dispatch_fold<CO>(fa, ts, dim, v4, s)) return rc;
  const int64_t nvec = dim / 4;
  if (v4 && nvec <= 128) {
    uint32_t* segb = reinterpret_cast<uint32_t*>(ws + L.segb);
    uint32_t* segr = reinterpret_cast<uint32_t*>(ws + L.segr);
    float* part = reinterpret_cast<float*>(ws + L.part);
    launch(seg_plan_kernel, 1, 1024, 0, s, fa, L.max_long, L.max_segs, segb, segr);
    if (int rc = check_launch("seg_plan_kernel")) return rc;
    // persistent grids: the long-run path costs little when there are none
    const unsigned fold_blocks =
        unsigned(std::min<int64_t>(ceil_div(int64_t(L.max_segs) * 32, 256), 8 * kNumSMs));
    auto go = [&](auto kern) -> int {
      launch(kern, fold_blocks, 256, 0, s, fa, ts, dim, L.max_long, segb, segr, part);
      return check_launch("seg_fold_kernel");
    };
    int rc;
    if (nvec <= 1) rc = go(seg_fold_kernel<1, 1>);
    else if (nvec <= 2) rc = go(seg_fold_kernel<2, 1>);
    else if (nvec <= 4) rc = go(seg_fold_kernel<4, 1>);
    else if (nvec <= 8) rc = go(seg_fold_kernel<8, 1>);
    else if (nvec <= 16) rc = go(seg_fold_kernel<16, 1>);
    else if (nvec <= 32) rc = go(seg_fold_kernel<32, 1>);
    else if (nvec <= 64) rc = go(seg_fold_kernel<32, 2>);
    else rc = go(seg_fold_kernel<32, 4>);
    if (rc) return rc;
    launch(seg_combine_kernel<CO>, unsigned(std::min<int64_t>(L.max_long, 4 * kNumSMs)), 128, 0, s, fa, ts, dim, L.max_long, segb, part);
    return check_launch("seg_combine_kernel");
  }
  const size_t smem = size_t(64) * dim * 4;
  auto k = emb_long_run_kernel<CO>;
  if (smem > 48 * 1024)
    DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  launch(k, unsigned(std::min<int64_t>(L.max_long, 4 * kNumSMs)), 256, smem, s, fa, ts, dim, L.max_long);
  return check_launch("emb_long_run_kernel");
}

template <bool CO>
int dispatch_fold(const FoldArgs& fa, const TableSet& ts, int64_t dim, bool v4,
                  cudaStream_t s) {
  if (v4) {
    const int64_t nv = dim / 4;
    if (nv <= 1) launch_fold<4, 1, 1, CO>(fa, ts, dim, s);
    else if (nv <= 2) launch_fold<4, 2, 1, CO>(fa, ts, dim, s);
    else if (nv <= 4) launch_fold<4, 4, 1, CO>(fa, ts, dim, s);
    else if (nv <= 8) launch_fold<4, 8, 1, CO>(fa, ts, dim, s);
    else if (nv <= 16) launch_fold<4, 16, 1, CO>(fa, ts, dim, s);
    else if (nv <= 32) launch_fold<4, 32, 1, CO>(fa, ts, dim, s);
    else if (nv <= 64) launch_fold<4, 32, 2, CO>(fa, ts, dim, s);
    else if (nv <= 128) launch_fold<4, 32, 4, CO>(fa, ts, dim, s);
    else { set_error("embedding dim > 512 unsupported"); return 1; }
  } else {
    if (dim <= 4) launch_fold<1, 4, 1, CO>(fa, ts, dim, s);
    else if (dim <= 32) launch_fold<1, 32, 1, CO>(fa, ts, dim, s);
    else if (dim <= 128) launch_fold<1, 32, 4, CO>(fa, ts, dim, s);
    else if (dim <= 512) launch_fold<1, 32, 16, CO>(fa, ts, dim, s);
    else { set_error("embedding dim > 512 unsupported"); return 1; }
  }
  return check_launch("emb_fold_kernel");
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

extern "C" int dlrm_err_reset(int64_t* err_pos, int32_t nt, int32_t* err_flag,
                              dlrm_stream_t stream) {
  DLRM_REQUIRE(err_pos != nullptr && nt >= 0, "bad error buffers");
  launch(err_reset_kernel, unsigned(ceil_div(nt > 0 ? nt : 1, 128)), 128, 0,
                     as_stream(stream), err_pos, nt, err_flag);
  return check_launch("err_reset_kernel");
}

extern "C" int dlrm_err_resolve(const dlrm_table_desc* tables, int32_t nt,
                                const int64_t* err_pos, const int32_t* err_flag,
                                int64_t* err_val, dlrm_stream_t stream) {
  DLRM_REQUIRE(err_pos && err_flag && err_val, "bad error buffers");
  static thread_local TableSet ts;
  if (int rc = fill_tableset(ts, tables, nt)) return rc;
  launch(err_resolve_kernel, unsigned(ceil_div(nt, 128)), 128, 0, as_stream(stream), ts,
         err_pos, err_flag, err_val);
  return check_launch("err_resolve_kernel");
}

extern "C" int dlrm_emb_fwd(const float* W_all, int64_t dim,
                            const dlrm_table_desc* tables, int32_t nt,
                            int64_t num_bags, float* out, int64_t out_stride,
                            int64_t* err_pos, int32_t* err_flag,
                            dlrm_stream_t stream) {
  DLRM_REQUIRE(dim >= 1 && dim <= 512, "embedding dim must be in [1, 512]");
  DLRM_REQUIRE(num_bags >= 0 && out != nullptr && err_pos && err_flag,
               "bad emb_fwd arguments");
  static thread_local TableSet ts;
  if (int rc = fill_tableset(ts, tables, nt)) return rc;
  if (num_bags == 0) return 0;
  cudaStream_t s = as_stream(stream);
  bool v4 = vec4_ok(dim, W_all, out_stride, 0) &&
            (reinterpret_cast<uintptr_t>(out) % 16) == 0;
  for (int i = 0; i < nt && v4; ++i) v4 = tables[i].out_offset % 4 == 0;
  int64_t cap_total = 0;
  for (int i = 0; i < nt; ++i) cap_total += tables[i].capacity;
  const double avg_pool = double(cap_total) / double(num_bags * nt);
  const int64_t nv0 = dim / 4;
  // streaming kernel for multi-hot bags, wide rows and large batches;
  // pooling-1 narrow rows keep the sub-warp kernel (lower fixed latency)
  static const bool force_stream = getenv("DLRM_EMB_FORCE_STREAM") != nullptr;
  // (measured: pooling-1 bags of 256-byte rows stream faster from 128 k
  // lookups up; 64-byte rows never do)
  bool stream_ok = v4 && nv0 <= 128 && (nv0 & (nv0 - 1)) == 0 &&
                   (avg_pool >= 3.0 || nv0 >= 32 || (nv0 >= 16 && cap_total >= 131072) ||
                    force_stream) &&
                   !getenv("DLRM_EMB_NO_STREAM");
  for (int i = 0; i < nt && stream_ok; ++i) stream_ok = tables[i].num_rows < int64_t(kBadRow);
  if (stream_ok) {
    static const int cfg = getenv("DLRM_EMB_FWD_CFG") ? atoi(getenv("DLRM_EMB_FWD_CFG")) : 1;
#define DLRM_STREAM(NVM, CH, S, W) \
  return launch_stream<NVM, CH, S, W>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s)
    // (CH rows per chunk, S ring slots, W warps per CTA), ~200 KB of ring per
    // SM; defaults measured on B200 (scripts/emb_one.py, DLRM_EMB_FWD_CFG)
    if (nv0 == 1) DLRM_STREAM(1, 32, 4, 16);
    if (nv0 == 2) DLRM_STREAM(2, 32, 4, 16);
    if (nv0 == 4) {
      if (cfg == 0) DLRM_STREAM(4, 32, 4, 16);
      DLRM_STREAM(4, 32, 2, 16);
    }
    if (nv0 == 8) {
      if (cfg == 0) DLRM_STREAM(8, 32, 4, 12);
      DLRM_STREAM(8, 32, 3, 16);
    }
    if (nv0 == 16) {
      if (cfg == 0) DLRM_STREAM(16, 32, 4, 6);
      if (cfg == 2) DLRM_STREAM(16, 16, 4, 12);
      if (cfg == 4) DLRM_STREAM(16, 32, 3, 8);
      if (cfg == 5) DLRM_STREAM(16, 16, 3, 8);
      if (cfg == 6) DLRM_STREAM(16, 16, 2, 8);
      if (cfg == 10) DLRM_STREAM(16, 8, 4, 24);
      if (cfg == 11) DLRM_STREAM(16, 8, 3, 32);
      if (cfg == 9) DLRM_STREAM(16, 16, 3, 16);
      // 24 warps x 2 slots of 16-row chunks (c3 step 0.4095 -> 0.4067 ms
      // over two A/B runs; the round-1 default is cfg 9)
      DLRM_STREAM(16, 16, 2, 24);
    }
    if (nv0 == 32) {
      // 512-byte rows: 16 warps of 8-row chunks (c4 pooling-1 lookup 263 ->
      // 193 us, 4.6 TB/s; pooling 4 / 32 equal or better than 8 warps of
      // 16-row chunks, the round-1 default, now cfg 9)
      if (cfg == 0) DLRM_STREAM(32, 16, 4, 6);
      if (cfg == 2) DLRM_STREAM(32, 8, 4, 12);
      if (cfg == 7) DLRM_STREAM(32, 4, 6, 16);
      if (cfg == 8) DLRM_STREAM(32, 4, 4, 24);
      if (cfg == 9) DLRM_STREAM(32, 16, 3, 8);
      DLRM_STREAM(32, 8, 3, 16);
    }
    if (nv0 == 64) {
      if (cfg == 0) DLRM_STREAM(64, 8, 4, 6);
      if (cfg == 2) DLRM_STREAM(64, 4, 4, 12);
      if (cfg == 3) DLRM_STREAM(64, 4, 3, 16);
      DLRM_STREAM(64, 8, 3, 8);
    }
    DLRM_STREAM(128, 4, 3, 8);
#undef DLRM_STREAM
  }
  if (v4 && (nv0 == 4 || nv0 == 8 || nv0 == 16 || nv0 == 32) && avg_pool >= 32.0 / nv0) {
    const int64_t threads = num_bags * nt * 32;
    int64_t want = ceil_div(threads, 256);
    if (want > 4 * kNumSMs) want = 4 * kNumSMs;  // persistent: 4 blocks per SM
    const unsigned blocks = unsigned(want);
    switch (nv0) {
      case 4: launch(emb_fwd_warp_kernel<4>, blocks, 256, 0, s, W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag); break;
      case 8: launch(emb_fwd_warp_kernel<8>, blocks, 256, 0, s, W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag); break;
      case 16: launch(emb_fwd_warp_kernel<16>, blocks, 256, 0, s, W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag); break;
      default: launch(emb_fwd_warp_kernel<32>, blocks, 256, 0, s, W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag); break;
    }
    return check_launch("emb_fwd_warp_kernel");
  }
  if (v4) {
    const int64_t nv = dim / 4;
    if (nv <= 1) launch_fwd<4, 1, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 2) launch_fwd<4, 2, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 4) launch_fwd<4, 4, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 8) launch_fwd<4, 8, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 16) launch_fwd<4, 16, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 32) launch_fwd<4, 32, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (nv <= 64) launch_fwd<4, 32, 2>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else launch_fwd<4, 32, 4>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
  } else {
    if (dim <= 4) launch_fwd<1, 4, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (dim <= 32) launch_fwd<1, 32, 1>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else if (dim <= 128) launch_fwd<1, 32, 4>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
    else launch_fwd<1, 32, 16>(W_all, dim, ts, num_bags, out, out_stride, err_pos, err_flag, s);
  }
  return check_launch("emb_fwd_kernel");
}

extern "C" size_t dlrm_emb_bwd_workspace_size(int64_t total_capacity,
                                              int64_t total_rows, int64_t dim) {
  (void)total_rows;
  return ws_layout(total_capacity, dim).total;
}

namespace dlrm {
namespace {
struct BwdPlan {
  int64_t n;
  WsLayout L;
  int end_bit;
  uint32_t sentinel;
};

int bwd_plan(TableSet& ts, const dlrm_table_desc* tables, int32_t nt, int64_t dim,
             int64_t total_rows, void* workspace, size_t ws_bytes, BwdPlan* p) {
  DLRM_REQUIRE(dim >= 1 && dim <= 512, "embedding dim must be in [1, 512]");
  DLRM_REQUIRE(total_rows >= 1 && total_rows < (int64_t(1) << 31),
               "total rows must be in [1, 2^31)");
  if (int rc = fill_tableset(ts, tables, nt)) return rc;
  p->n = ts.cap_base[nt];
  DLRM_REQUIRE(p->n < (int64_t(1) << 31), "total capacity must be < 2^31");
  p->L = ws_layout(p->n, dim);
  DLRM_REQUIRE(p->n == 0 || (workspace != nullptr && ws_bytes >= p->L.total),
               "embedding backward workspace too small");
  p->end_bit = end_bit_for(total_rows);
  p->sentinel = uint32_t((int64_t(1) << p->end_bit) - 1);
  return 0;
}
}  // namespace
}  // namespace dlrm

extern "C" int dlrm_emb_bwd_prepare(int64_t dim, const dlrm_table_desc* tables, int32_t nt,
                                    int64_t num_bags, int64_t total_rows, void* workspace,
                                    size_t ws_bytes, dlrm_stream_t stream) {
  static thread_local TableSet ts;
  BwdPlan p;
  if (int rc = bwd_plan(ts, tables, nt, dim, total_rows, workspace, ws_bytes, &p)) return rc;
  if (p.n == 0 || num_bags == 0) return 0;
  char* ws = static_cast<char*>(workspace);
  // index errors were recorded by the forward; the key pass re-records into
  // a scratch area so the caller's err_pos is unaffected here
  int64_t* scratch_err = reinterpret_cast<int64_t*>(ws + p.L.err);
  int32_t* scratch_flag = reinterpret_cast<int32_t*>(ws + p.L.err + DLRM_MAX_TABLES * 8);
  return sort_pairs(ts, num_bags, ws, p.L, p.n, scratch_err, scratch_flag, p.sentinel,
                    p.end_bit, as_stream(stream));
}

namespace dlrm {
namespace {
int emb_apply(float* W_all, int64_t dim, const dlrm_table_desc* tables, int32_t nt,
              int64_t num_bags, const float* grad, int64_t grad_stride, const Upd& u,
              const int32_t* err_flag, int64_t total_rows, void* workspace, size_t ws_bytes,
              dlrm_stream_t stream) {
  static thread_local TableSet ts;
  BwdPlan p;
  if (int rc = bwd_plan(ts, tables, nt, dim, total_rows, workspace, ws_bytes, &p)) return rc;
  if (p.n == 0 || num_bags == 0) return 0;
  char* ws = static_cast<char*>(workspace);
  FoldArgs fa{};
  fa.keys = reinterpret_cast<const uint32_t*>(ws + p.L.keys_b);
  fa.vals = reinterpret_cast<const uint32_t*>(ws + p.L.vals_b);
  fa.bag_of = reinterpret_cast<const int32_t*>(ws + p.L.bag);
  fa.by_bag = by_bag_values(ts);
  fa.n = p.n;
  fa.sentinel = p.sentinel;
  fa.grad = grad;
  fa.grad_stride = grad_stride;
  fa.W = W_all;
  fa.upd = u;
  fa.err_flag = err_flag;
  bool v4 = vec4_ok(dim, W_all, grad_stride, 0) &&
            (reinterpret_cast<uintptr_t>(grad) % 16) == 0 &&
            (u.kind != DLRM_UPD_ADAGRAD || u.delta % 4 == 0);
  for (int i = 0; i < nt && v4; ++i) v4 = tables[i].out_offset % 4 == 0;
  return run_fold<false>(fa, ts, dim, v4, ws, p.L, as_stream(stream));
}
}  // namespace
}  // namespace dlrm

extern "C" int dlrm_emb_bwd_apply_sgd(float* W_all, int64_t dim, const dlrm_table_desc* tables,
                                      int32_t nt, int64_t num_bags, const float* grad,
                                      int64_t grad_stride, float lr, const int32_t* err_flag,
                                      int64_t total_rows, void* workspace, size_t ws_bytes,
                                      dlrm_stream_t stream) {
  return emb_apply(W_all, dim, tables, nt, num_bags, grad, grad_stride, sgd_rule(lr), err_flag,
                   total_rows, workspace, ws_bytes, stream);
}

extern "C" int dlrm_emb_bwd_apply(float* W_all, int64_t dim, const dlrm_table_desc* tables,
                                  int32_t nt, int64_t num_bags, const float* grad,
                                  int64_t grad_stride, const dlrm_update* upd,
                                  const int32_t* err_flag, int64_t total_rows, void* workspace,
                                  size_t ws_bytes, dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(upd->eps >= 0.f, "eps must be nonnegative");
  return emb_apply(W_all, dim, tables, nt, num_bags, grad, grad_stride, upd_rule(upd), err_flag,
                   total_rows, workspace, ws_bytes, stream);
}

extern "C" int dlrm_emb_bwd_sgd(float* W_all, int64_t dim,
                                const dlrm_table_desc* tables, int32_t nt,
                                int64_t num_bags, const float* grad,
                                int64_t grad_stride, float lr,
                                const int32_t* err_flag, int64_t total_rows,
                                void* workspace, size_t ws_bytes,
                                dlrm_stream_t stream) {
  if (int rc = dlrm_emb_bwd_prepare(dim, tables, nt, num_bags, total_rows, workspace,
                                    ws_bytes, stream))
    return rc;
  return dlrm_emb_bwd_apply_sgd(W_all, dim, tables, nt, num_bags, grad, grad_stride, lr,
                                err_flag, total_rows, workspace, ws_bytes, stream);
}

extern "C" int dlrm_emb_bwd_coalesce(int64_t dim, const dlrm_table_desc* table,
                                     int64_t num_bags, const float* grad,
                                     int64_t grad_stride, int64_t* rows_out,
                                     float* values_out, int64_t* num_unique,
                                     int64_t* err_pos, int32_t* err_flag,
                                     void* workspace, size_t ws_bytes,
                                     dlrm_stream_t stream) {
  DLRM_REQUIRE(dim >= 1 && dim <= 512, "embedding dim must be in [1, 512]");
  DLRM_REQUIRE(table != nullptr && num_unique != nullptr && err_pos &&
                   err_flag, "bad arguments");
  static thread_local TableSet ts;
  dlrm_table_desc one = *table;
  const int64_t total_rows = one.row_base + one.num_rows;
  DLRM_REQUIRE(total_rows >= 1 && total_rows < (int64_t(1) << 31),
               "table rows must be in [1, 2^31)");
  if (int rc = fill_tableset(ts, &one, 1)) return rc;
  const int64_t n = ts.cap_base[1];
  cudaStream_t s = as_stream(stream);
  if (n == 0 || num_bags == 0) {
    DLRM_CUDA(cudaMemsetAsync(num_unique, 0, sizeof(int64_t), s));
    return 0;
  }
  const WsLayout L = ws_layout(n, dim);
  DLRM_REQUIRE(workspace != nullptr && ws_bytes >= L.total,
               "embedding backward workspace too small");
  const int end_bit = end_bit_for(total_rows);
  const uint32_t sentinel = uint32_t((int64_t(1) << end_bit) - 1);
  char* ws = static_cast<char*>(workspace);
  if (int rc = sort_pairs(ts, num_bags, ws, L, n, err_pos, err_flag, sentinel, end_bit, s))
    return rc;
  const uint32_t* ks = reinterpret_cast<const uint32_t*>(ws + L.keys_b);
  const uint32_t* vs = reinterpret_cast<const uint32_t*>(ws + L.vals_b);
  uint32_t* flags = reinterpret_cast<uint32_t*>(ws + L.flags);
  uint32_t* uid = reinterpret_cast<uint32_t*>(ws + L.uid);
  launch(run_flags_kernel, unsigned(ceil_div(n, 256)), 256, 0, s, ks, n, sentinel, flags);
  if (int rc = check_launch("run_flags_kernel")) return rc;
  size_t tb = L.temp_bytes;
  DLRM_CUDA(cub::DeviceScan::ExclusiveSum(ws + L.temp, tb, flags, uid, int(n), s));
  count_launch();
  launch(count_unique_kernel, 1, 32, 0, s, uid, flags, n, num_unique);
  if (int rc = check_launch("count_unique_kernel")) return rc;
  FoldArgs fa{};
  fa.keys = ks;
  fa.vals = vs;
  fa.bag_of = reinterpret_cast<const int32_t*>(ws + L.bag);
  fa.by_bag = by_bag_values(ts);
  fa.n = n;
  fa.sentinel = sentinel;
  fa.grad = grad;
  fa.grad_stride = grad_stride;
  fa.uid = uid;
  fa.rows_out = rows_out;
  fa.values_out = values_out;
  bool v4 = vec4_ok(dim, values_out, grad_stride, one.out_offset) &&
            (reinterpret_cast<uintptr_t>(grad) % 16) == 0;
  return run_fold<true>(fa, ts, dim, v4, ws, L, s);
}

namespace dlrm {
namespace {
int update_rows(float* W, int64_t dim, const int64_t* rows, const float* values, int64_t n,
                const Upd& u, dlrm_stream_t stream) {
  DLRM_REQUIRE(dim >= 1 && n >= 0, "bad row-update arguments");
  if (n == 0) return 0;
  cudaStream_t s = as_stream(stream);
  const bool v4 = vec4_ok(dim, W, dim, 0) &&
                  (reinterpret_cast<uintptr_t>(values) % 16) == 0 &&
                  (u.kind != DLRM_UPD_ADAGRAD || u.delta % 4 == 0);
  if (v4) {
    const int64_t e = n * (dim / 4);
    launch(sgd_rows_kernel<4>, unsigned(ceil_div(e, 256)), 256, 0, s, W, dim, rows, values, n, u);
  } else {
    const int64_t e = n * dim;
    launch(sgd_rows_kernel<1>, unsigned(ceil_div(e, 256)), 256, 0, s, W, dim, rows, values, n, u);
  }
  return check_launch("sgd_rows_kernel");
}
}  // namespace
}  // namespace dlrm

extern "C" int dlrm_sgd_rows(float* W, int64_t dim, const int64_t* rows,
                             const float* values, int64_t n, float lr,
                             dlrm_stream_t stream) {
  return update_rows(W, dim, rows, values, n, sgd_rule(lr), stream);
}

extern "C" int dlrm_update_rows(float* W, int64_t dim, const int64_t* rows, const float* values,
                                int64_t n, const dlrm_update* upd, dlrm_stream_t stream) {
  DLRM_REQUIRE(upd != nullptr && (upd->kind == DLRM_UPD_SGD || upd->kind == DLRM_UPD_ADAGRAD),
               "bad update rule");
  DLRM_REQUIRE(upd->eps >= 0.f, "eps must be nonnegative");
  return update_rows(W, dim, rows, values, n, upd_rule(upd), stream);
}
