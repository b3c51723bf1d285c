// Criteo TSV ingestion (ref datagen.py:318-371 parse_criteo / _hash_token):
// host code, multithreaded over lines, writing straight into the caller's
// (pinned) batch buffers.
//
// Record: label \t 13 integer fields \t 26 categorical tokens.  Empty fields
// are legal (label 0, dense 0.0, index 0).  Dense: log1p(max(x, 0)) in double,
// rounded to fp32.  Categorical: 64-bit BLAKE2b (digest size 8, no key, the
// digest read little-endian) of the token's bytes, mod the table's vocabulary.
// BLAKE2b is written here from RFC 7693.  Lines end at '\n' — or, in
// universal-newline mode (files, as the reference's text-mode read_criteo
// sees them), at '\n', '\r' or "\r\n"; whitespace-only lines are skipped but
// counted for line numbers.  The first
// malformed line (lowest line number) is reported as "line k: ..." exactly as
// the reference's CriteoFormatError messages.
#include <math.h>
#include <sched.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace dlrm {
namespace {

constexpr int kDense = 13, kCat = 26, kFields = 1 + kDense + kCat;

// ---------------------------------------------------------------- BLAKE2b
constexpr uint64_t kIV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                             0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                             0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
constexpr uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

inline void mix(uint64_t* v, int a, int b, int c, int d, uint64_t x, uint64_t y) {
  v[a] = v[a] + v[b] + x;
  v[d] = rotr(v[d] ^ v[a], 32);
  v[c] = v[c] + v[d];
  v[b] = rotr(v[b] ^ v[c], 24);
  v[a] = v[a] + v[b] + y;
  v[d] = rotr(v[d] ^ v[a], 16);
  v[c] = v[c] + v[d];
  v[b] = rotr(v[b] ^ v[c], 63);
}

void compress(uint64_t* h, const uint8_t* block, uint64_t t, bool last) {
  uint64_t m[16], v[16];
  for (int i = 0; i < 16; ++i) {
    uint64_t w = 0;
    for (int j = 7; j >= 0; --j) w = (w << 8) | block[8 * i + j];  // little-endian words
    m[i] = w;
  }
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = kIV[i];
  }
  v[12] ^= t;  // byte counter (tokens are far below 2^64 bytes: high word 0)
  if (last) v[14] = ~v[14];
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kSigma[r];
    mix(v, 0, 4, 8, 12, m[s[0]], m[s[1]]);
    mix(v, 1, 5, 9, 13, m[s[2]], m[s[3]]);
    mix(v, 2, 6, 10, 14, m[s[4]], m[s[5]]);
    mix(v, 3, 7, 11, 15, m[s[6]], m[s[7]]);
    mix(v, 0, 5, 10, 15, m[s[8]], m[s[9]]);
    mix(v, 1, 6, 11, 12, m[s[10]], m[s[11]]);
    mix(v, 2, 7, 8, 13, m[s[12]], m[s[13]]);
    mix(v, 3, 4, 9, 14, m[s[14]], m[s[15]]);
  }
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// BLAKE2b with an 8-byte digest; the digest's bytes read little-endian are h[0]
uint64_t blake2b64(const uint8_t* p, size_t n) {
  uint64_t h[8];
  for (int i = 0; i < 8; ++i) h[i] = kIV[i];
  h[0] ^= 0x01010000ull ^ 8ull;  // depth 1, fanout 1, no key, outlen 8
  uint8_t block[128];
  uint64_t t = 0;
  while (n > 128) {
    t += 128;
    compress(h, p, t, false);
    p += 128;
    n -= 128;
  }
  memset(block, 0, sizeof(block));
  if (n) memcpy(block, p, n);
  t += n;
  compress(h, block, t, true);
  return h[0];
}

// ---------------------------------------------------------------- parsing
struct Line {
  const char* p;
  int64_t n;       // without the '\n'
  int64_t lineno;  // 1-based, counting blank lines
};

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v'; }

// Python int(tok) for the label: optional surrounding whitespace and sign
bool parse_label(const char* p, int64_t n, int* out) {
  int64_t i = 0, j = n;
  while (i < j && is_space(p[i])) ++i;
  while (j > i && is_space(p[j - 1])) --j;
  bool neg = false;
  if (i < j && (p[i] == '+' || p[i] == '-')) {
    neg = p[i] == '-';
    ++i;
  }
  if (i == j) return false;
  long long v = 0;
  for (int64_t k = i; k < j; ++k) {
    if (p[k] < '0' || p[k] > '9') return false;
    v = v * 10 + (p[k] - '0');
    if (v > 1000) v = 1000;  // anything but 0 / 1 is rejected anyway
  }
  *out = int(neg ? -v : v);
  return true;
}

// Python float(tok) for decimal / integer tokens (hex floats are rejected as
// Python does; underscores are not accepted)
bool parse_double(const char* p, int64_t n, double* out) {
  std::string s(p, size_t(n));
  size_t i = 0;
  while (i < s.size() && is_space(s[i])) ++i;
  size_t k = i;
  if (k < s.size() && (s[k] == '+' || s[k] == '-')) ++k;
  if (k + 1 < s.size() && s[k] == '0' && (s[k + 1] == 'x' || s[k + 1] == 'X')) return false;
  char* end = nullptr;
  const double v = strtod(s.c_str() + i, &end);
  if (end == s.c_str() + i) return false;
  while (*end && is_space(*end)) ++end;
  if (*end) return false;
  *out = v;
  return true;
}

struct Out {
  float* labels;
  float* dense;
  int64_t ld_dense;
  int64_t* cat;
  int64_t ld_cat;
  const int64_t* vocab;
};

// returns "" or the reference's error message for this line
std::string parse_line(const Line& L, int64_t r, const Out& o) {
  const char* f[kFields + 1];
  int64_t len[kFields + 1];
  int nf = 0;
  const char* s = L.p;
  const char* e = L.p + L.n;
  const char* q = s;
  for (const char* c = s;; ++c) {
    if (c == e || *c == '\t') {
      if (nf <= kFields) {
        f[nf] = q;
        len[nf] = c - q;
      }
      ++nf;
      q = c + 1;
      if (c == e) break;
    }
  }
  if (nf != kFields)
    return "line " + std::to_string(L.lineno) + ": expected " + std::to_string(kFields) +
           " tab-separated fields, got " + std::to_string(nf);
  int label = 0;
  if (len[0] && !parse_label(f[0], len[0], &label))
    return "line " + std::to_string(L.lineno) + ": unparsable label '" + std::string(f[0], size_t(len[0])) + "'";
  if (label != 0 && label != 1) return "line " + std::to_string(L.lineno) + ": label must be 0 or 1";
  o.labels[r] = float(label);
  for (int i = 0; i < kDense; ++i) {
    double v = 0.0;
    if (len[1 + i]) {
      double x;
      if (!parse_double(f[1 + i], len[1 + i], &x))
        return "line " + std::to_string(L.lineno) + ": unparsable dense field " + std::to_string(i) +
               ": '" + std::string(f[1 + i], size_t(len[1 + i])) + "'";
      v = log1p(0.0 > x ? 0.0 : x);  // Python max(x, 0.0): x unless 0.0 > x (NaN, -0.0 kept)
    }
    o.dense[r * o.ld_dense + i] = float(v);
  }
  for (int i = 0; i < kCat; ++i) {
    int64_t idx = 0;
    const int64_t n = len[1 + kDense + i];
    if (n) {
      const uint64_t hv = blake2b64(reinterpret_cast<const uint8_t*>(f[1 + kDense + i]), size_t(n));
      idx = int64_t(hv % uint64_t(o.vocab[i]));
    }
    o.cat[int64_t(i) * o.ld_cat + r] = idx;
  }
  return "";
}

}  // namespace
}  // namespace dlrm

using namespace dlrm;

extern "C" uint64_t dlrm_blake2b64(const void* data, int64_t nbytes) {
  return blake2b64(static_cast<const uint8_t*>(data), size_t(nbytes < 0 ? 0 : nbytes));
}

extern "C" int64_t dlrm_criteo_parse(const char* text, int64_t nbytes, const int64_t* vocab_sizes,
                                     int64_t max_records, float* labels, float* dense,
                                     int64_t ld_dense, int64_t* cat, int64_t ld_cat,
                                     int64_t first_lineno, int64_t* consumed, int32_t flags) {
  const int nthreads = flags >> 8;
  const bool universal = flags & 1;
  if (!text || nbytes < 0 || !vocab_sizes || !labels || !dense || !cat || ld_dense < kDense ||
      max_records < 0 || ld_cat < max_records) {
    set_error("dlrm_criteo_parse: bad arguments");
    return -1;
  }
  for (int i = 0; i < kCat; ++i)
    if (vocab_sizes[i] < 1) {
      set_error("dlrm_criteo_parse: vocabulary sizes must be positive");
      return -1;
    }
  // split into lines (records up to max_records); a final line without a
  // terminator counts as a line.  universal: '\n', '\r' and "\r\n" end a line
  // (Python's text-mode files, as the reference's read_criteo opens them)
  std::vector<Line> lines;
  int64_t pos = 0, lineno = first_lineno, used = 0;
  while (pos < nbytes && int64_t(lines.size()) < max_records) {
    const char* p = text + pos;
    int64_t n = 0, term = 0;
    if (universal) {
      while (pos + n < nbytes && p[n] != '\n' && p[n] != '\r') ++n;
      if (pos + n < nbytes) term = (p[n] == '\r' && pos + n + 1 < nbytes && p[n + 1] == '\n') ? 2 : 1;
    } else {
      const char* nl = static_cast<const char*>(memchr(p, '\n', size_t(nbytes - pos)));
      n = nl ? nl - p : nbytes - pos;
      term = nl ? 1 : 0;
    }
    bool blank = true;
    for (int64_t k = 0; k < n && blank; ++k) blank = is_space(p[k]);
    if (!blank) lines.push_back(Line{p, n, lineno});
    pos += n + term;
    used = pos;
    ++lineno;
  }
  if (consumed) *consumed = used;
  const int64_t nrec = int64_t(lines.size());
  Out o{labels, dense, ld_dense, cat, ld_cat, vocab_sizes};
  int nt = nthreads;
  if (nt <= 0) {  // the CPUs this process may run on
    cpu_set_t set;
    nt = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set)
                                                       : int(sysconf(_SC_NPROCESSORS_ONLN));
  }
  if (nt > 64) nt = 64;
  if (nt < 1) nt = 1;
  if (nrec < 4096) nt = 1;
  std::vector<std::string> errs(static_cast<size_t>(nt));
  std::vector<int64_t> err_line(size_t(nt), INT64_MAX);
  auto work = [&](int w) {
    const int64_t a = nrec * w / nt, b = nrec * (w + 1) / nt;
    for (int64_t r = a; r < b; ++r) {
      std::string m = parse_line(lines[size_t(r)], r, o);
      if (!m.empty()) {  // first bad line of this slice
        errs[size_t(w)] = m;
        err_line[size_t(w)] = lines[size_t(r)].lineno;
        return;
      }
    }
  };
  if (nt == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int w = 0; w < nt; ++w) th.emplace_back(work, w);
    for (auto& t : th) t.join();
  }
  const auto it = std::min_element(err_line.begin(), err_line.end());
  if (*it != INT64_MAX) {
    set_error(errs[size_t(it - err_line.begin())]);
    return -2;
  }
  return nrec;
}
