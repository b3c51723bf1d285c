// Pairwise dot-product feature interaction: C-ABI entry points, dispatching
// to the tcgen05 kernels (interact_tc.cu) and the SIMT fallback below
// (shapes the tensor-core path does not take: d % 8 / d % 16, d > 128,
// nf > 64, unaligned features; DLRM_IA_SIMT=1 forces it).
//
// Reference (dlrmkit, pkg/src/dlrmkit/model.py):
//   interact           218-242  out = [z0 | z_i . z_j for i < j, row-major]
//                               (upper triangle, (0,1),(0,2),...,(1,2),...)
//   interact_backward  245-268  g_i = [i==0] gout[:, :d] + sum_{j!=i} g_ij z_j
//
// Feature f of sample b is read from feat[f] + b*stride[f], so the kernel can
// consume the all-to-all receive buffer (features grouped by source rank) and
// the pooled-embedding buffer in place.  A CTA stages S samples' feature
// rows in shared memory (row pitch d+4 floats: conflict-free float4 reads),
// then each thread computes dot products / gradient columns from smem.
#include "common.cuh"

namespace dlrm {

// tcgen05 path (interact_tc.cu): used whenever the shape / alignment allows
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

// 512 threads per CTA: at the Terabyte shape (27 features, d = 128, B = 32768)
// the backward takes 361 vs 446 us with 256 (scripts/interact_bench.py);
// 1024 is slower (register-limited); small shapes are unchanged
#ifndef DLRM_IA_THREADS
#define DLRM_IA_THREADS 512
#endif
#ifndef DLRM_IA_BUDGET_KB
#define DLRM_IA_BUDGET_KB 96
#endif
constexpr int kIaThreads = DLRM_IA_THREADS;

__device__ __forceinline__ void pair_of(int p, int nf, int& i, int& j) {
  // row-major upper triangle: row i holds nf-1-i pairs
  int row = 0, base = 0;
  while (p >= base + (nf - 1 - row)) { base += nf - 1 - row; ++row; }
  i = row;
  j = row + 1 + (p - base);
}

template <bool V4>
__global__ void __launch_bounds__(kIaThreads)
interact_fwd_kernel(FeatureSet fs, int nf, int64_t dim, int64_t batch, int S,
                    float* __restrict__ out, int64_t ld_out, int64_t pad_to) {
  pdl_entry();
  extern __shared__ float4 smem4[];
  float* z = reinterpret_cast<float*>(smem4);
  const int pitch = int(dim) + 4;
  const int npairs = nf * (nf - 1) / 2;
  int* pairs = reinterpret_cast<int*>(z + size_t(S) * nf * pitch);
  for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
    int i, j;
    pair_of(p, nf, i, j);
    pairs[p] = (i << 16) | j;
  }
  const int64_t b0 = int64_t(blockIdx.x) * S;
  const int ns = int(batch - b0 < S ? batch - b0 : S);
  // stage features
  if (V4) {  // cp.async: every 16-byte piece of the tile in flight at once
    const int nv = int(dim / 4);
    for (int e = threadIdx.x; e < ns * nf * nv; e += blockDim.x) {
      const int s = e / (nf * nv), r = e - s * nf * nv, f = r / nv, c = r - f * nv;
      cp_async16(z + (size_t(s) * nf + f) * pitch + 4 * c,
                 reinterpret_cast<const float4*>(fs.feat[f] + (b0 + s) * fs.stride[f]) + c, true);
    }
    cp_async_commit();
    cp_async_wait<0>();
  } else {
    for (int e = threadIdx.x; e < ns * nf * int(dim); e += blockDim.x) {
      const int s = e / (nf * int(dim)), r = e - s * nf * int(dim), f = r / int(dim),
                c = r - f * int(dim);
      z[(size_t(s) * nf + f) * pitch + c] = __ldg(fs.feat[f] + (b0 + s) * fs.stride[f] + c);
    }
  }
  __syncthreads();
  const int width = int(dim) + npairs;
  const int total_w = int(pad_to > width ? pad_to : width);
  if (V4) {
    // z0 copy and zero pad columns
    const int extra = total_w - width;
    for (int e = threadIdx.x; e < ns * (int(dim) + extra); e += blockDim.x) {
      const int s = e / (int(dim) + extra), col = e - s * (int(dim) + extra);
      out[(b0 + s) * ld_out + (col < dim ? col : width + (col - int(dim)))] =
          col < dim ? z[size_t(s) * nf * pitch + col] : 0.f;
    }
    // pair dots in 4x4 feature blocks (bi <= bj), each block split over 4
    // consecutive lanes by column residue j = c % 4: lane j keeps the j-th of
    // the four interleaved partial sums of all 16 pairs, and the lanes combine
    // them as (p0 + p1) + (p2 + p3) — the same rounding as one thread with
    // four partials, with 4x the parallelism.  Staged rows are re-read nf/4
    // instead of nf times.
    const int nbk = (nf + 3) / 4, ntile = nbk * (nbk + 1) / 2;
    const int total = ns * ntile * 4;
    const int lane = threadIdx.x & 31;
    for (int base = threadIdx.x & ~31; base < total; base += blockDim.x) {
      const int e = base + lane;
      const bool active = e < total;
      const int item = active ? e >> 2 : 0, j = e & 3;
      const int s = item / ntile;
      int t = item - s * ntile, bi = 0;
      while (t >= nbk - bi) { t -= nbk - bi; ++bi; }
      const int bj = bi + t;
      const float* zs = z + size_t(s) * nf * pitch;
      const float* ri[4];
      const float* rj[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        ri[k] = zs + min(4 * bi + k, nf - 1) * pitch + j;
        rj[k] = zs + min(4 * bj + k, nf - 1) * pitch + j;
      }
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
      if (active) {
        for (int c = 0; c < dim; c += 4) {
          float x[4], y[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            x[k] = ri[k][c];
            y[k] = rj[k][c];
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(x[a], y[b], acc[a][b]);
        }
      }
      float* orow = out + (b0 + s) * ld_out + dim;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          float v = acc[a][b];
          v = v + __shfl_xor_sync(0xffffffffu, v, 1);  // lanes j, j^1: p0 + p1 / p2 + p3
          v = v + __shfl_xor_sync(0xffffffffu, v, 2);  // (p0 + p1) + (p2 + p3)
          const int i = 4 * bi + a, jj = 4 * bj + b;
          if (active && j == 0 && i < jj && jj < nf)
            orow[i * (2 * nf - i - 1) / 2 + (jj - i - 1)] = v;
        }
    }
    return;
  }
  for (int e = threadIdx.x; e < ns * total_w; e += blockDim.x) {
    const int s = e / total_w, col = e - s * total_w;
    const float* zs = z + size_t(s) * nf * pitch;
    float v;
    if (col < dim) {
      v = zs[col];
    } else if (col < width) {
      const int pr = pairs[col - int(dim)];
      const float* zi = zs + (pr >> 16) * pitch;
      const float* zj = zs + (pr & 0xffff) * pitch;
      float a = 0.f;
      for (int c = 0; c < dim; ++c) a = fmaf(zi[c], zj[c], a);
      v = a;
    } else {
      v = 0.f;
    }
    out[(b0 + s) * ld_out + col] = v;
  }
}

template <bool V4>
__global__ void __launch_bounds__(kIaThreads)
interact_bwd_kernel(FeatureSet fs, GradFeatureSet gs, int nf, int64_t dim,
                    int64_t batch, int S, const float* __restrict__ gout,
                    int64_t ld_gout, int mask_f0) {
  pdl_entry();
  extern __shared__ float4 smem4[];
  float* z = reinterpret_cast<float*>(smem4);
  const int pitch = int(dim) + 4;
  const int gp = (nf + 3) & ~3;  // pitch of the symmetric gradient matrix (float4 rows)
  float* G = z + size_t(S) * nf * pitch;
  const int npairs = nf * (nf - 1) / 2;
  const int64_t b0 = int64_t(blockIdx.x) * S;
  const int ns = int(batch - b0 < S ? batch - b0 : S);
  const int id = int(dim);
  if (V4) {  // cp.async staging (see forward)
    const int nv = id / 4;
    for (int e = threadIdx.x; e < ns * nf * nv; e += blockDim.x) {
      const int s = e / (nf * nv), r = e - s * nf * nv, f = r / nv, c = r - f * nv;
      cp_async16(z + (size_t(s) * nf + f) * pitch + 4 * c,
                 reinterpret_cast<const float4*>(fs.feat[f] + (b0 + s) * fs.stride[f]) + c, true);
    }
    cp_async_commit();
  } else {
    for (int e = threadIdx.x; e < ns * nf * id; e += blockDim.x) {
      const int s = e / (nf * id), r = e - s * nf * id, f = r / id, c = r - f * id;
      z[(size_t(s) * nf + f) * pitch + c] = __ldg(fs.feat[f] + (b0 + s) * fs.stride[f] + c);
    }
  }
  // symmetric pair gradients, zero diagonal
  for (int e = threadIdx.x; e < ns * nf; e += blockDim.x) {
    const int s = e / nf, f = e - s * nf;
    G[(size_t(s) * nf + f) * gp + f] = 0.f;
  }
#pragma unroll 4
  for (int e = threadIdx.x; e < ns * npairs; e += blockDim.x) {
    const int s = e / npairs, p = e - s * npairs;
    int i, j;
    pair_of(p, nf, i, j);
    const float g = __ldg(gout + (b0 + s) * ld_gout + id + p);
    G[(size_t(s) * nf + i) * gp + j] = g;
    G[(size_t(s) * nf + j) * gp + i] = g;
  }
  if (V4) cp_async_wait<0>();
  __syncthreads();
  if (V4) {
    // 4 features x 4 columns per thread: one float4 of G (symmetric, so row j
    // holds G[f0..f3][j]) and one float4 of Z feed 16 FMAs
    const int nv = id / 4, nbk = (nf + 3) / 4;
    for (int e = threadIdx.x; e < ns * nbk * nv; e += blockDim.x) {
      const int s = e / (nbk * nv), r = e - s * nbk * nv, fb = r / nv, c = r - fb * nv;
      const float* zs = z + size_t(s) * nf * pitch + 4 * c;
      const float* gs0 = G + size_t(s) * nf * gp + 4 * fb;
      float4 a[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (fb == 0) a[0] = __ldg(reinterpret_cast<const float4*>(gout + (b0 + s) * ld_gout) + c);
      for (int j = 0; j < nf; ++j) {
        const float4 g = *reinterpret_cast<const float4*>(gs0 + j * gp);
        const float4 x = *reinterpret_cast<const float4*>(zs + j * pitch);
        const float gk[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          a[k].x = fmaf(gk[k], x.x, a[k].x);
          a[k].y = fmaf(gk[k], x.y, a[k].y);
          a[k].z = fmaf(gk[k], x.z, a[k].z);
          a[k].w = fmaf(gk[k], x.w, a[k].w);
        }
      }
      if (fb == 0 && mask_f0) {
        const float4 z0 = *reinterpret_cast<const float4*>(zs);
        a[0].x *= z0.x > 0.f ? 1.f : 0.f;
        a[0].y *= z0.y > 0.f ? 1.f : 0.f;
        a[0].z *= z0.z > 0.f ? 1.f : 0.f;
        a[0].w *= z0.w > 0.f ? 1.f : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int f = 4 * fb + k;
        if (f < nf) reinterpret_cast<float4*>(gs.feat[f] + (b0 + s) * gs.stride[f])[c] = a[k];
      }
    }
  } else {
    for (int e = threadIdx.x; e < ns * nf * id; e += blockDim.x) {
      const int s = e / (nf * id), r = e - s * nf * id, f = r / id, c = r - f * id;
      const float* zs = z + size_t(s) * nf * pitch + c;
      const float* gr = G + (size_t(s) * nf + f) * gp;
      float a = f == 0 ? __ldg(gout + (b0 + s) * ld_gout + c) : 0.f;
      for (int j = 0; j < nf; ++j) a = fmaf(gr[j], zs[j * pitch], a);
      if (f == 0 && mask_f0) a *= zs[0] > 0.f ? 1.f : 0.f;
      gs.feat[f][(b0 + s) * gs.stride[f] + c] = a;
    }
  }
}

// Samples per CTA: enough CTAs for >= 2 per SM (the op is latency-bound at
// DLRM sizes: a few MB of features), capped by the shared-memory budget.
int pick_samples(int nf, int64_t dim, int64_t batch, size_t extra_per_sample, size_t fixed,
                 size_t budget) {
  const size_t per = size_t(nf) * (dim + 4) * 4 + extra_per_sample;
  int S = int((budget - fixed) / per);
  const int64_t want = batch / (2 * kNumSMs);
  if (S > want) S = int(want);
  if (S > 32) S = 32;
  return S < 1 ? 1 : S;
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

static int fill_features(FeatureSet& fs, const dlrm_features* feats, int32_t nf,
                         int64_t dim, bool* v4) {
  DLRM_REQUIRE(feats != nullptr && nf >= 1 && nf <= DLRM_MAX_FEATURES,
               "feature count must be in [1, DLRM_MAX_FEATURES]");
  *v4 = dim % 4 == 0;
  for (int f = 0; f < nf; ++f) {
    fs.feat[f] = feats->feat[f];
    fs.stride[f] = feats->feat_stride[f];
    *v4 = *v4 && reinterpret_cast<uintptr_t>(fs.feat[f]) % 16 == 0 &&
          fs.stride[f] % 4 == 0;
  }
  return 0;
}

extern "C" int dlrm_interact_fwd(const dlrm_features* feats, int32_t nf,
                                 int64_t dim, int64_t batch, float* out,
                                 int64_t ld_out, int64_t pad_to,
                                 dlrm_stream_t stream) {
  DLRM_REQUIRE(dim >= 1 && dim <= 1024 && batch >= 0, "bad interaction shape");
  static thread_local FeatureSet fs;
  bool v4;
  if (int rc = fill_features(fs, feats, nf, dim, &v4)) return rc;
  if (batch == 0) return 0;
  if (interact_tc_fwd_ok(fs, nf, dim, batch, ld_out, out))
    return interact_tc_fwd(fs, nf, dim, batch, out, ld_out, pad_to, as_stream(stream));
  const int npairs = nf * (nf - 1) / 2;
  const size_t fixed = align_up(size_t(npairs) * 4, 16);
  const int S = pick_samples(nf, dim, batch, 0, fixed, DLRM_IA_BUDGET_KB * 1024);
  const size_t smem = size_t(S) * nf * (dim + 4) * 4 + fixed;
  DLRM_REQUIRE(smem <= 200 * 1024, "interaction tile exceeds shared memory");
  cudaStream_t s = as_stream(stream);
  auto k = v4 ? interact_fwd_kernel<true> : interact_fwd_kernel<false>;
  DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  launch(k, unsigned(ceil_div(batch, S)), kIaThreads, smem, s, fs, nf, dim, batch, S, out,
                                                     ld_out, pad_to);
  return check_launch("interact_fwd_kernel");
}

extern "C" int dlrm_interact_bwd(const dlrm_features* feats, int32_t nf,
                                 int64_t dim, int64_t batch, const float* gout,
                                 int64_t ld_gout, float* const* grad_feat,
                                 const int64_t* grad_stride,
                                 int32_t relu_mask_f0, dlrm_stream_t stream) {
  DLRM_REQUIRE(dim >= 1 && dim <= 1024 && batch >= 0, "bad interaction shape");
  DLRM_REQUIRE(grad_feat != nullptr && grad_stride != nullptr, "null grads");
  static thread_local FeatureSet fs;
  static thread_local GradFeatureSet gs;
  bool v4;
  if (int rc = fill_features(fs, feats, nf, dim, &v4)) return rc;
  for (int f = 0; f < nf; ++f) {
    gs.feat[f] = grad_feat[f];
    gs.stride[f] = grad_stride[f];
    v4 = v4 && reinterpret_cast<uintptr_t>(grad_feat[f]) % 16 == 0 &&
         grad_stride[f] % 4 == 0;
  }
  v4 = v4 && reinterpret_cast<uintptr_t>(gout) % 16 == 0 && ld_gout % 4 == 0;
  if (batch == 0) return 0;
  if (interact_tc_bwd_ok(fs, gs, nf, dim, batch, gout, ld_gout))
    return interact_tc_bwd(fs, gs, nf, dim, batch, gout, ld_gout, relu_mask_f0,
                           as_stream(stream));
  const size_t extra = size_t(nf) * ((nf + 3) & ~3) * 4;
  const int S = pick_samples(nf, dim, batch, extra, 0, DLRM_IA_BUDGET_KB * 1024);
  const size_t smem = size_t(S) * (nf * (dim + 4) * 4 + extra);
  DLRM_REQUIRE(smem <= 200 * 1024, "interaction tile exceeds shared memory");
  cudaStream_t s = as_stream(stream);
  auto k = v4 ? interact_bwd_kernel<true> : interact_bwd_kernel<false>;
  DLRM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  launch(k, unsigned(ceil_div(batch, S)), kIaThreads, smem, s, fs, gs, nf, dim, batch, S,
                                                     gout, ld_gout, relu_mask_f0);
  return check_launch("interact_bwd_kernel");
}
