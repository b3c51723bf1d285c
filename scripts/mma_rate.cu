// Microbenchmark: issue rate of tcgen05.mma kind::tf32 / kind::f16 from smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// MN-major SWIZZLE_128B_BASE32B: LBO = 32 fp32 x 32 rows = 4096 B, SBO = 512 B
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(512 >> 4) << 32) | (uint64_t(1) << 46) | (uint64_t(1) << 61);
}
template <int KIND, int N, int AMN = 0, int BMN = 0, int ROT = 0>
__global__ void mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  // idesc: f32 accum; kind tf32 (a/b fmt 2) or f16 with bf16 (fmt 1)
  const uint32_t fmt = KIND == 0 ? 2u : 1u;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(AMN) << 15) | (uint32_t(BMN) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    uint64_t a = AMN ? desc_mn(smem_u32(smem)) : desc(smem_u32(smem));
    uint64_t b = BMN ? desc_mn(smem_u32(smem + 32768)) : desc(smem_u32(smem + 32768));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (ROT) {  // fresh operands every MMA: 3 stages x 4 k-offsets (A at 0..48K, B at 48K..96K)
        const uint32_t st = uint32_t(i >> 2) % 3u, kk = uint32_t(i) & 3u;
        a = desc(smem_u32(smem) + st * 16384 + kk * 32);
        b = desc(smem_u32(smem) + 49152 + st * 16384 + kk * 32);
      }
      if (KIND == 0)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(i));
      else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int KIND, int N, int AMN = 0, int BMN = 0, int ROT = 0>
void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto k = mma_loop<KIND, N, AMN, BMN, ROT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  int iters = 4096;
  k<<<148, 128, 200000>>>(iters, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 200000>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[148]; cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  int K = KIND == 0 ? 8 : 16;
  double flops = 2.0 * 128 * N * K * iters * 148;
  printf("%s%s N=%d A_MN=%d B_MN=%d: %.1f cycles/mma, %.1f TFLOP/s (err=%s)\n", name, ROT ? " rotating" : "", N, AMN, BMN, double(c[0]) / iters,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main_pair();
int main() {
  run<0, 128, 0, 0, 1>("tf32"); run<0, 256, 0, 0, 1>("tf32"); run<1, 128, 0, 0, 1>("bf16");
  main_pair();
  run<0, 128>("tf32"); run<0, 256>("tf32"); run<0, 64>("tf32");
  run<0, 128, 0, 1>("tf32"); run<0, 128, 1, 1>("tf32"); run<0, 128, 1, 0>("tf32"); run<0, 64, 1, 1>("tf32");
  run<1, 128>("bf16"); run<1, 256>("bf16");
  return 0;
}

// ---- CTA-pair variant: cluster (2,1,1), cta_group::2, M = 256, issued by rank 0
template <int N, int ROT = 0>
__global__ void mma_pair_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); }
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
  long long t0 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    uint64_t a = desc(smem_u32(smem));
    uint64_t b = desc(smem_u32(smem + 32768));
    for (int i = 0; i < iters; ++i) {
      if (ROT) {
        const uint32_t st = uint32_t(i >> 2) % 3u, kk = uint32_t(i) & 3u;
        a = desc(smem_u32(smem) + st * 16384 + kk * 32);
        b = desc(smem_u32(smem) + 49152 + st * 8192 + kk * 32);
      }
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3));
  }
  if (threadIdx.x == 0) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int ROT = 0>
void run_pair() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto k = mma_pair_loop<N, ROT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  int iters = 4096;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 100000;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c[148]; cudaMemcpy(c, d, sizeof(c), cudaMemcpyDeviceToHost);
  double flops = 2.0 * 256 * N * 8 * iters * 74;
  printf("tf32 pair%s M=256 N=%d: %.1f cycles/mma, %.1f TFLOP/s (err=%s)\n", ROT ? " rotating" : "", N, double(c[0]) / iters,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main_pair() { run_pair<128>(); run_pair<256>(); run_pair<128, 1>(); run_pair<256, 1>(); return 0; }
