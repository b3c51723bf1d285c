// Host-side input generation: the variable-length bags of the reference's
// random source, bit-identical to numpy, in native code.
//
// The reference CLI's random source (dlrmkit cli.py:294-314 over datagen.py
// gen_sparse_batch 79-96) draws, per table and sample j, a length
// n = Generator.integers(1, k + 1) and then n indices Generator.integers(0,
// m, size=n) from ONE numpy Philox stream — 2 numpy calls per sample, i.e.
// ~16k Python-level calls per Big-Basin batch (rng.RandomBatchSource; 0.3 s
// per batch).  This file replays exactly what numpy does underneath, so the
// same Generator state yields the same bags:
//   * Philox4x64-10 (Random123 constants), 4 x uint64 per counter block,
//     counter incremented before each block (numpy philox_next);
//   * next_uint32: the upper half of a 64-bit output is cached for the next
//     32-bit draw (has_uint32 / uinteger);
//   * integers(low, high) with high - low - 1 < 2^32: Lemire's bounded
//     32-bit method with rejection (numpy buffered_bounded_lemire_uint32);
//     a range of one value consumes nothing.
// The caller passes numpy's Philox state (Generator.bit_generator.state) in
// and gets the advanced state back.
#include <stdint.h>
#include <string.h>

#include "dlrm_b200.h"

namespace {

struct Philox {
  uint64_t ctr[4], key[2], buf[4];
  int64_t pos;        // buffer position (4 = empty)
  int64_t has32;      // a cached upper half is pending
  uint64_t u32;       // the cached upper half
};

inline void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  const unsigned __int128 p = (unsigned __int128)a * b;
  *hi = uint64_t(p >> 64);
  *lo = uint64_t(p);
}

void philox_block(const uint64_t in[4], const uint64_t k_in[2], uint64_t out[4]) {
  uint64_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint64_t k0 = k_in[0], k1 = k_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

inline uint64_t next64(Philox& s) {
  if (s.pos < 4) return s.buf[s.pos++];
  if (++s.ctr[0] == 0 && ++s.ctr[1] == 0 && ++s.ctr[2] == 0) ++s.ctr[3];
  philox_block(s.ctr, s.key, s.buf);
  s.pos = 1;
  return s.buf[0];
}

inline uint32_t next32(Philox& s) {
  if (s.has32) {
    s.has32 = 0;
    return uint32_t(s.u32);
  }
  const uint64_t v = next64(s);
  s.has32 = 1;
  s.u32 = v >> 32;
  return uint32_t(v & 0xFFFFFFFFULL);
}

// off + uniform integer in [0, rng] (rng < 2^32 - 1), numpy's Lemire path
inline int64_t bounded(Philox& s, int64_t off, uint32_t rng) {
  if (rng == 0) return off;
  const uint32_t excl = rng + 1;
  uint64_t m = uint64_t(next32(s)) * excl;
  uint32_t left = uint32_t(m);
  if (left < excl) {
    const uint32_t threshold = (0xFFFFFFFFu - rng) % excl;
    while (left < threshold) {
      m = uint64_t(next32(s)) * excl;
      left = uint32_t(m);
    }
  }
  return off + int64_t(m >> 32);
}

}  // namespace

// Variable-length bags of `nt` tables (table t: rows[t]) for `batch` samples,
// lengths uniform in [1, k]: offsets_out[t * (batch + 1) + j] (CSR with the
// terminal entry), indices of table t at indices_out + t * batch * k, counts
// in nnz_out[t].  state: numpy Philox state as 13 uint64 (counter[4], key[2],
// buffer[4], buffer_pos, has_uint32, uinteger), advanced in place.  Host
// pointers; returns 0, or 1 for bad arguments (message in dlrm_last_error).
extern "C" int dlrm_random_bags(uint64_t* state, const int64_t* rows, int32_t nt, int64_t batch,
                                int64_t k, int64_t* offsets_out, int64_t* indices_out,
                                int64_t* nnz_out) {
  if (!state || !rows || nt < 1 || batch < 0 || k < 1 || k > (int64_t(1) << 31) ||
      !offsets_out || !indices_out || !nnz_out)
    return 1;
  for (int t = 0; t < nt; ++t)
    if (rows[t] < 1 || rows[t] >= (int64_t(1) << 32)) return 1;
  Philox s;
  memcpy(s.ctr, state, 4 * 8);
  memcpy(s.key, state + 4, 2 * 8);
  memcpy(s.buf, state + 6, 4 * 8);
  s.pos = int64_t(state[10]);
  s.has32 = int64_t(state[11]);
  s.u32 = state[12];
  for (int t = 0; t < nt; ++t) {
    int64_t* off = offsets_out + int64_t(t) * (batch + 1);
    int64_t* idx = indices_out + int64_t(t) * batch * k;
    const uint32_t rng_len = uint32_t(k - 1), rng_row = uint32_t(rows[t] - 1);
    off[0] = 0;
    int64_t n = 0;
    for (int64_t j = 0; j < batch; ++j) {
      const int64_t len = bounded(s, 1, rng_len);
      for (int64_t i = 0; i < len; ++i) idx[n + i] = bounded(s, 0, rng_row);
      n += len;
      off[j + 1] = n;
    }
    nnz_out[t] = n;
  }
  memcpy(state, s.ctr, 4 * 8);
  memcpy(state + 4, s.key, 2 * 8);
  memcpy(state + 6, s.buf, 4 * 8);
  state[10] = uint64_t(s.pos);
  state[11] = uint64_t(s.has32);
  state[12] = s.u32;
  return 0;
}

// ---------------------------------------------------------------------------
// One batch of the reference's host arrays packed into a step's input block
// (pipeline.InputLayout): dense rows float64 -> fp32 (row pitch ldx), labels
// float64 -> fp32, per-table offsets / indices int64 (and weights float64 ->
// fp32).  The copies run on `nthreads` native threads, without the Python
// GIL (the Prefetcher's worker calls this through ctypes).
#include <emmintrin.h>

#include <algorithm>
#include <thread>
#include <vector>

extern "C" int dlrm_pack_batch(uint8_t* dst, const int64_t* sec /* x, labels, offsets, indices,
                               iweights byte offsets */, int64_t batch, int64_t k0, int64_t ldx,
                               int32_t nt, const int64_t* cap_base, const double* dense,
                               int64_t ld_dense, const double* labels,
                               const int64_t* const* offsets, const int64_t* const* indices,
                               const int64_t* nnz, const double* const* weights,
                               int32_t nthreads) {
  if (!dst || !sec || batch < 0 || k0 < 0 || ldx < k0 || nt < 1 || !cap_base || !dense ||
      !labels || !offsets || !indices || !nnz)
    return 1;
  for (int t = 0; t < nt; ++t)
    if (nnz[t] < 0 || nnz[t] > cap_base[t + 1] - cap_base[t] || !offsets[t] ||
        (nnz[t] > 0 && !indices[t]))
      return 1;
  float* x = reinterpret_cast<float*>(dst + sec[0]);
  float* lab = reinterpret_cast<float*>(dst + sec[1]);
  int64_t* offs = reinterpret_cast<int64_t*>(dst + sec[2]);
  int64_t* idx = reinterpret_cast<int64_t*>(dst + sec[3]);
  float* iw = sec[4] >= 0 ? reinterpret_cast<float*>(dst + sec[4]) : nullptr;
  const int nth = std::max(1, std::min(int(nthreads), 64));
  // work items: dense row slabs, then tables.  The block is written with
  // streaming (non-temporal) stores: it is only read again by the H2D DMA,
  // and regular stores would first read every destination line (the host's
  // memory bandwidth is what the input pipeline is bound by, shared with
  // that DMA).
  const int64_t slabs = std::min<int64_t>(nth, std::max<int64_t>(1, batch / 64));
  const int64_t items = slabs + nt;
  auto work = [&](int64_t it) {
    if (it < slabs) {
      const int64_t r0 = batch * it / slabs, r1 = batch * (it + 1) / slabs;
      for (int64_t r = r0; r < r1; ++r) {
        const double* s = dense + r * ld_dense;
        float* d = x + r * ldx;
        int64_t c = 0;
        if ((reinterpret_cast<uintptr_t>(d) & 15) == 0)
          for (; c + 4 <= k0; c += 4) {
            const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(s + c));
            const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(s + c + 2));
            _mm_stream_ps(d + c, _mm_movelh_ps(lo, hi));
          }
        for (; c < k0; ++c) d[c] = float(s[c]);
      }
      if (it == 0)
        for (int64_t r = 0; r < batch; ++r) lab[r] = float(labels[r]);
      _mm_sfence();
      return;
    }
    const int t = int(it - slabs);
    memcpy(offs + int64_t(t) * (batch + 1), offsets[t], size_t(batch + 1) * 8);
    if (nnz[t] > 0) {
      int64_t* d = idx + cap_base[t];
      const int64_t* src = indices[t];
      int64_t i = 0, n = nnz[t];
      if ((reinterpret_cast<uintptr_t>(d) & 15) != 0 && n > 0) d[i] = src[i], ++i;
      for (; i + 2 <= n; i += 2)
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i),
                         _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i)));
      for (; i < n; ++i) d[i] = src[i];
      _mm_sfence();
    }
    if (iw) {
      float* w = iw + cap_base[t];
      const double* src = weights ? weights[t] : nullptr;
      for (int64_t i = 0; i < nnz[t]; ++i) w[i] = src ? float(src[i]) : 1.f;
    }
  };
  if (nth == 1 || items == 1) {
    for (int64_t it = 0; it < items; ++it) work(it);
    return 0;
  }
  std::vector<std::thread> pool;
  const int nuse = int(std::min<int64_t>(nth, items));
  for (int w = 0; w < nuse; ++w)
    pool.emplace_back([&, w] {
      for (int64_t it = w; it < items; it += nuse) work(it);
    });
  for (auto& th : pool) th.join();
  return 0;
}
