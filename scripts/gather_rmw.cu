// Row read-modify-write bandwidth (the sparse apply's pattern: read a table
// row, add a gradient row, write it back) over a 8M x 256 B table, for
// ~800K distinct rows visited in SORTED order (what the apply does after the
// radix sort) vs a random order, next to the read-only gather of the same
// rows.  Bytes counted: read (+ write) of every visited row.
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
constexpr int LPB = 16;  // 16 lanes x float4 = 256-byte row
template <int R, bool WRITE>
__global__ void rmw(float4* __restrict__ W, const uint32_t* __restrict__ idx, int64_t n,
                    const float4* __restrict__ g, float4* out) {
  int lane = threadIdx.x % LPB;
  int64_t grp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / LPB;
  int64_t groups = int64_t(gridDim.x) * blockDim.x / LPB;
  float4 acc = make_float4(0, 0, 0, 0);
  // contiguous chunk of the index list per group (sorted order stays local)
  const int64_t per = (n + groups - 1) / groups;
  const int64_t b0 = grp * per, b1 = b0 + per < n ? b0 + per : n;
  for (int64_t base = b0; base < b1; base += R) {
    float4 v[R];
    uint32_t r_[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t i = base + r;
      r_[r] = i < b1 ? __ldg(idx + i) : 0xffffffffu;
      v[r] = r_[r] != 0xffffffffu ? W[int64_t(r_[r]) * LPB + lane] : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (WRITE) {
        if (r_[r] != 0xffffffffu) {
          float4 gg = g[(r_[r] & 1023) * LPB + lane];
          W[int64_t(r_[r]) * LPB + lane] = make_float4(v[r].x - 0.1f * gg.x, v[r].y - 0.1f * gg.y,
                                                       v[r].z - 0.1f * gg.z, v[r].w - 0.1f * gg.w);
        }
      } else {
        acc.x += v[r].x; acc.y += v[r].y; acc.z += v[r].z; acc.w += v[r].w;
      }
    }
  }
  if (acc.x == 123.f) out[grp] = acc;
}
template <int R, bool WRITE>
void run(const char* name, float4* W, uint32_t* idx, int64_t n, const float4* g, float4* out, char* flush) {
  int blocks = 148 * 8;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms = 0;
  for (int w = 0; w < 6; ++w) {
    cudaMemsetAsync(flush, w, 256 << 20);
    cudaEventRecord(a);
    rmw<R, WRITE><<<blocks, 256>>>(W, idx, n, g, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); if (w) ms += t;
  }
  ms /= 5;
  double bytes = double(n) * 256 * (WRITE ? 2 : 1);
  printf("%-8s %s R=%2d: %7.1f us  %6.0f GB/s\n", name, WRITE ? "rmw   " : "gather", R, ms * 1e3, bytes / ms / 1e6);
}
int main() {
  const int64_t rows = 8 << 20;
  float4* W; cudaMalloc(&W, rows * 256); cudaMemset(W, 0, rows * 256);
  float4* g; cudaMalloc(&g, 1024 * 256); cudaMemset(g, 0, 1024 * 256);
  float4* out; cudaMalloc(&out, 1 << 24);
  char* flush; cudaMalloc(&flush, 256 << 20);
  // ~800K distinct rows: 827K random draws, deduplicated
  std::vector<uint32_t> h(827000);
  uint64_t s = 88172645463325252ull;
  auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
  for (auto& x : h) x = uint32_t(rnd() % rows);
  std::sort(h.begin(), h.end());
  h.erase(std::unique(h.begin(), h.end()), h.end());
  const int64_t n = int64_t(h.size());
  std::vector<uint32_t> perm(h);
  for (int64_t i = n - 1; i > 0; --i) std::swap(perm[i], perm[rnd() % (i + 1)]);
  uint32_t *ds, *dr;
  cudaMalloc(&ds, n * 4); cudaMalloc(&dr, n * 4);
  cudaMemcpy(ds, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, perm.data(), n * 4, cudaMemcpyHostToDevice);
  printf("%lld distinct rows of %lld (256 B)\n", (long long)n, (long long)rows);
  run<8, false>("sorted", W, ds, n, g, out, flush);
  run<8, false>("random", W, dr, n, g, out, flush);
  run<4, true>("sorted", W, ds, n, g, out, flush);
  run<8, true>("sorted", W, ds, n, g, out, flush);
  run<16, true>("sorted", W, ds, n, g, out, flush);
  run<8, true>("random", W, dr, n, g, out, flush);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
