// Achievable random-row gather bandwidth on this GPU: every LPB-lane group
// reads R random rows of `row_bytes` (float4 per lane) with R loads in
// flight and reduces them; sweeps row size.  Reference ceiling for the
// pooled-lookup kernel (whose access pattern this is).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int LPB, int R>
__global__ void gather(const float4* __restrict__ W, const uint32_t* __restrict__ idx, int64_t nrows_total,
                       int64_t n, float4* out) {
  int lane = threadIdx.x % LPB;
  int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LPB;
  int64_t groups = int64_t(gridDim.x) * blockDim.x / LPB;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t base = g * R; base < n; base += groups * R) {
    float4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = base + r;
      v[r] = i < n ? __ldg(W + int64_t(__ldg(idx + i)) * LPB + lane) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) { acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w; }
  }
  if (acc.x == 123.f) out[g] = acc;
}
template <int LPB, int R>
void run(const float4* W, uint32_t* idx, int64_t rows, int64_t n, float4* out) {
  int blocks = 148 * 8;
  // fresh indices per rep (idx holds 6 sets) and L2 flushed before each rep
  static char* flush = nullptr;
  if (!flush) cudaMalloc(&flush, 256 << 20);
  gather<LPB, R><<<blocks, 256>>>(W, idx + 5 * n, rows, n, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int w = 0; w < 5; ++w) {
    cudaMemsetAsync(flush, w, 256 << 20);
    cudaEventRecord(a);
    gather<LPB, R><<<blocks, 256>>>(W, idx + w * n, rows, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); ms += t;
  }
  ms /= 5;
  double bytes = double(n) * LPB * 16;
  printf("row %4d B, %2d rows in flight/group: %7.1f us  %6.0f GB/s\n", LPB * 16, R, ms * 1e3, bytes / ms / 1e6);
}
int main() {
  const int64_t table_bytes = 2LL << 30;
  float4* W; cudaMalloc(&W, table_bytes); cudaMemset(W, 0, table_bytes);
  const int64_t n = 831077;
  uint32_t* idx; cudaMalloc(&idx, 6 * n * 4);
  uint32_t* h = (uint32_t*)malloc(6 * n * 4);
  float4* out; cudaMalloc(&out, 1 << 24);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
#define SWEEP(LPB) { int64_t rows = table_bytes / (LPB * 16); for (int64_t i = 0; i < 6 * n; ++i) h[i] = rnd() % rows; \
    cudaMemcpy(idx, h, 6 * n * 4, cudaMemcpyHostToDevice); run<LPB, 4>(W, idx, rows, n, out); run<LPB, 8>(W, idx, rows, n, out); run<LPB, 16>(W, idx, rows, n, out); }
  SWEEP(4) SWEEP(8) SWEEP(16) SWEEP(32)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
