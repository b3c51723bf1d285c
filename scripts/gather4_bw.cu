// Random-row gather bandwidth through TMA gather4 (cp.async.bulk.tensor
// .tile::gather4: 4 arbitrary rows of a 2-D tensor per instruction) vs the
// plain-load ceiling of scripts/gather_bw.cu: 831k uniformly random 256-byte
// rows of a 2 GiB table, L2 flushed before each rep.  Per CTA one producer
// thread keeps STAGES stages of G gather4 ops in flight; 4 consumer warps
// reduce each landed stage (the pooled lookup's access pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gather4_bw scripts/gather4_bw.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}

template <int ROWF, int G, int STAGES>
__global__ void __launch_bounds__(160) g4(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx,
                                         int64_t n, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int STAGE_BYTES = G * 4 * ROWF * 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t per = 4 * G;                            // rows per stage
  const int64_t chunks = (n + per - 1) / per;
  if (warp == 4) {
    // the whole producer warp loads a stage's indices (one per lane, G <= 8
    // gives <= 32 rows), lanes 0..G-1 each issue one gather4; next stage's
    // indices are loaded before waiting for its slot
    static_assert(4 * G <= 32, "one index per lane");
    int it = 0;
    int64_t c = blockIdx.x;
    int cur = c < chunks ? int(idx[min(c * per + lane, n - 1)]) : 0;
    for (; c < chunks; c += gridDim.x, ++it) {
      const int64_t cn = c + gridDim.x;
      const int nxt = cn < chunks ? int(idx[min(cn * per + lane, n - 1)]) : 0;
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
      if (lane == 0) mbar_expect(&full[s], STAGE_BYTES);
      __syncwarp();
      int r[4];
      for (int q = 0; q < 4; ++q) r[q] = __shfl_sync(0xffffffffu, cur, (4 * lane + q) & 31);
      if (lane < G) {
        uint8_t* dst = smem + s * STAGE_BYTES + lane * 4 * ROWF * 4;
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                     ::"r"(sa(dst)), "l"(&tm), "r"(sa(&full[s])), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                     "r"(r[3])
                     : "memory");
      }
      cur = nxt;
    }
  } else {
    float acc = 0.f;
    int it = 0;
    for (int64_t c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const float4* src = reinterpret_cast<const float4*>(smem + s * STAGE_BYTES);
      for (int e = threadIdx.x; e < STAGE_BYTES / 16; e += 128) {
        const float4 v = src[e];
        acc += v.x + v.y + v.z + v.w;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 123.f) out[threadIdx.x] = acc;
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int ROWF, int G, int STAGES, int CPS>
void run(float* W, int64_t rows, uint32_t* idx, int64_t n, float* out, char* flush) {
  static Enc enc = nullptr;
  if (!enc) {
    void* p; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = (Enc)p;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {ROWF, cuuint64_t(rows)};
  cuuint64_t str[1] = {ROWF * 4};
  cuuint32_t box[2] = {ROWF, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return; }
  constexpr int smem = STAGES * G * 4 * ROWF * 4 + 2 * STAGES * 8 + 1024;
  auto k = g4<ROWF, G, STAGES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148 * CPS, 160, smem>>>(tm, idx + 5 * n, n, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int w = 0; w < 5; ++w) {
    cudaMemsetAsync(flush, w, 256 << 20);
    cudaEventRecord(a);
    k<<<148 * CPS, 160, smem>>>(tm, idx + w * n, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); ms += t;
  }
  ms /= 5;
  printf("gather4 row %4d B, %2d x4 rows/stage, %2d stages, %d CTA/SM: %7.1f us %6.0f GB/s  (%s)\n", ROWF * 4, G, STAGES, CPS,
         ms * 1e3, double(n) * ROWF * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t table_bytes = 2LL << 30;
  float* W; cudaMalloc(&W, table_bytes); cudaMemset(W, 0, table_bytes);
  const int64_t n = 831077;
  uint32_t* idx; cudaMalloc(&idx, 6 * n * 4);
  uint32_t* h = (uint32_t*)malloc(6 * n * 4);
  float* out; cudaMalloc(&out, 1 << 20);
  char* flush; cudaMalloc(&flush, 256 << 20);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
#define SW(ROWF) { int64_t rows = table_bytes / (ROWF * 4); for (int64_t i = 0; i < 6 * n; ++i) h[i] = rnd() % rows; \
  cudaMemcpy(idx, h, 6 * n * 4, cudaMemcpyHostToDevice); \
  run<ROWF, 8, 4, 1>(W, rows, idx, n, out, flush); run<ROWF, 8, 8, 1>(W, rows, idx, n, out, flush); \
  run<ROWF, 8, 4, 4>(W, rows, idx, n, out, flush); run<ROWF, 4, 8, 4>(W, rows, idx, n, out, flush); \
  run<ROWF, 8, 6, 3>(W, rows, idx, n, out, flush); run<ROWF, 2, 16, 6>(W, rows, idx, n, out, flush); }
  SW(64) SW(32) SW(128)
  return 0;
}
