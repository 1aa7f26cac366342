// Graph ingest: OpenFst-style text -> state-major CSR on the
// host, with the reference's parsing rules (fst.py:204-275 parse_text_fst:
// `src dst ilabel olabel [weight]` arc lines, `state [weight]` final lines,
// `#` comments, the first line names the start state, arc order inside a
// state = line order) and its graph fingerprint (fst.py:194-201: sha256 over
// "start num_states", "il ol dst repr(w)" per arc, "f state repr(w)" per final
// state), plus a binary cache of the result.
#pragma once
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>
#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace ab {

static const uint32_t SHA256_K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

#if defined(__x86_64__)
// SHA-256 compression with the x86 SHA extensions (runtime-dispatched).
__attribute__((target("sha,sse4.1,ssse3"))) inline void sha256_ni(uint32_t st[8], const unsigned char *data,
                                                                  size_t nblocks) {
  const __m128i MASK = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
  __m128i tmp = _mm_loadu_si128((const __m128i *)&st[0]);
  __m128i s1 = _mm_loadu_si128((const __m128i *)&st[4]);
  tmp = _mm_shuffle_epi32(tmp, 0xB1);
  s1 = _mm_shuffle_epi32(s1, 0x1B);
  __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);
  s1 = _mm_blend_epi16(s1, tmp, 0xF0);
  for (; nblocks; --nblocks, data += 64) {
    const __m128i abef = s0, cdgh = s1;
    __m128i w[4];
    for (int i = 0; i < 16; ++i) {
      __m128i m;
      if (i < 4) {
        m = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i *)(data + 16 * i)), MASK);
      } else {
        const __m128i a = _mm_sha256msg1_epu32(w[(i - 4) & 3], w[(i - 3) & 3]);
        const __m128i b = _mm_add_epi32(a, _mm_alignr_epi8(w[(i - 1) & 3], w[(i - 2) & 3], 4));
        m = _mm_sha256msg2_epu32(b, w[(i - 1) & 3]);
      }
      w[i & 3] = m;
      __m128i k = _mm_add_epi32(m, _mm_loadu_si128((const __m128i *)&SHA256_K[4 * i]));
      s1 = _mm_sha256rnds2_epu32(s1, s0, k);
      k = _mm_shuffle_epi32(k, 0x0E);
      s0 = _mm_sha256rnds2_epu32(s0, s1, k);
    }
    s0 = _mm_add_epi32(s0, abef);
    s1 = _mm_add_epi32(s1, cdgh);
  }
  tmp = _mm_shuffle_epi32(s0, 0x1B);
  s1 = _mm_shuffle_epi32(s1, 0xB1);
  s0 = _mm_blend_epi16(tmp, s1, 0xF0);
  s1 = _mm_alignr_epi8(s1, tmp, 8);
  _mm_storeu_si128((__m128i *)&st[0], s0);
  _mm_storeu_si128((__m128i *)&st[4], s1);
}
inline bool have_sha_ni() {
  static const int v = __builtin_cpu_supports("sha") ? 1 : 0;
  return v != 0;
}
#endif

// ASCII whitespace as Python's str.split() / str.strip() see it
inline bool py_space(char c) { return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f); }

// ------------------------------------------------------------------ sha256
struct Sha256 {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  unsigned char buf[64];
  size_t n = 0;
  uint64_t bits = 0;
  static uint32_t rotr(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }
  void block(const unsigned char *p) { blocks(p, 1); }
  void blocks(const unsigned char *p, size_t nb) {
#if defined(__x86_64__)
    if (have_sha_ni()) {
      sha256_ni(h, p, nb);
      return;
    }
#endif
    for (; nb; --nb, p += 64) block_portable(p);
  }
  void block_portable(const unsigned char *p) {
    const uint32_t *K = SHA256_K;
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = k + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      k = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
  }
  void update(const char *p, size_t len) {
    bits += (uint64_t)len * 8;
    if (n) {
      const size_t take = std::min(len, 64 - n);
      memcpy(buf + n, p, take);
      n += take;
      p += take;
      len -= take;
      if (n < 64) return;
      block(buf);
      n = 0;
    }
    if (len >= 64) { // whole blocks in place
      const size_t nb = len / 64;
      blocks((const unsigned char *)p, nb);
      p += 64 * nb;
      len -= 64 * nb;
    }
    memcpy(buf, p, len);
    n = len;
  }
  std::string hex() {
    unsigned char pad[72] = {0x80};
    const uint64_t b = bits;
    const size_t padlen = (n < 56 ? 56 - n : 120 - n);
    update((const char *)pad, padlen);
    unsigned char len8[8];
    for (int i = 0; i < 8; ++i) len8[i] = (unsigned char)(b >> (56 - 8 * i));
    update((const char *)len8, 8);
    char out[65];
    for (int i = 0; i < 8; ++i) snprintf(out + 8 * i, 9, "%08x", h[i]);
    return std::string(out, 64);
  }
};

// Python repr() of a float (shortest round trip; fixed notation when the
// decimal point position is in (-4, 16], else d.ddde+XX).
inline std::string py_float_repr(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
  char sci[64];
  const auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  std::string s(sci, r.ptr);
  std::string sign;
  if (s[0] == '-') {
    sign = "-";
    s.erase(0, 1);
  }
  const size_t epos = s.find('e');
  const int exp10 = atoi(s.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (s[i] != '.') digits += s[i];
  const int decpt = exp10 + 1;
  const int nd = (int)digits.size();
  std::string out;
  if (decpt > -4 && decpt <= 16) {
    if (decpt <= 0) out = "0." + std::string((size_t)-decpt, '0') + digits;
    else if (decpt >= nd) out = digits + std::string((size_t)(decpt - nd), '0') + ".0";
    else out = digits.substr(0, (size_t)decpt) + "." + digits.substr((size_t)decpt);
  } else {
    out = digits.substr(0, 1);
    if (nd > 1) out += "." + digits.substr(1);
    char e[16];
    snprintf(e, sizeof(e), "e%c%02d", exp10 < 0 ? '-' : '+', exp10 < 0 ? -exp10 : exp10);
    out += e;
  }
  return sign + out;
}

// py_float_repr into `out` (>= 32 bytes free); returns the end.
inline char *py_float_repr_to(double x, char *out) {
  if (std::isfinite(x) && x != 0) {
    char sci[40];
    const auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
    const char *s = sci, *end = r.ptr;
    char *o = out;
    if (*s == '-') *o++ = *s++;
    const char *ep = s;
    while (ep < end && *ep != 'e') ++ep;
    int exp10 = 0;
    std::from_chars(ep + 1 + (ep[1] == '+'), end, exp10);
    char digits[24];
    int nd = 0;
    for (const char *q = s; q < ep; ++q)
      if (*q != '.') digits[nd++] = *q;
    const int decpt = exp10 + 1;
    if (decpt > -4 && decpt <= 16) {
      if (decpt <= 0) {
        *o++ = '0';
        *o++ = '.';
        for (int i = 0; i < -decpt; ++i) *o++ = '0';
        for (int i = 0; i < nd; ++i) *o++ = digits[i];
      } else if (decpt >= nd) {
        for (int i = 0; i < nd; ++i) *o++ = digits[i];
        for (int i = nd; i < decpt; ++i) *o++ = '0';
        *o++ = '.';
        *o++ = '0';
      } else {
        for (int i = 0; i < decpt; ++i) *o++ = digits[i];
        *o++ = '.';
        for (int i = decpt; i < nd; ++i) *o++ = digits[i];
      }
      return o;
    }
  }
  const std::string t = py_float_repr(x);
  memcpy(out, t.data(), t.size());
  return out + t.size();
}

struct HostFst {
  int32_t start = 0;
  int64_t num_states = 0;
  std::vector<int64_t> ro;
  std::vector<int32_t> il, ol, ns;
  std::vector<double> w;
  std::vector<int32_t> fstate; // sorted
  std::vector<double> fcost;
  std::string fingerprint;

  void compute_fingerprint() {
    Sha256 h;
    std::string line = std::to_string(start) + " " + std::to_string(num_states) + "\n";
    h.update(line.data(), line.size());
    // arc lines formatted in parallel, hashed in order (rounds of T blocks)
    const int64_t A = (int64_t)il.size();
    const int T = (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 64u);
    const int64_t BLK = 1 << 16;
    std::vector<std::vector<char>> bufs((size_t)T);
    for (int64_t r0 = 0; r0 < A; r0 += BLK * T) {
      auto fmt = [&](int t) {
        std::vector<char> &buf = bufs[(size_t)t];
        buf.clear();
        const int64_t b0 = r0 + (int64_t)t * BLK, b1 = std::min(A, b0 + BLK);
        if (b0 >= b1) return;
        buf.resize((size_t)(b1 - b0) * 72);
        char *p = buf.data();
        for (int64_t a = b0; a < b1; ++a) {
          p = std::to_chars(p, p + 12, il[a]).ptr;
          *p++ = ' ';
          p = std::to_chars(p, p + 12, ol[a]).ptr;
          *p++ = ' ';
          p = std::to_chars(p, p + 12, ns[a]).ptr;
          *p++ = ' ';
          p = py_float_repr_to(w[a], p);
          *p++ = '\n';
        }
        buf.resize((size_t)(p - buf.data()));
      };
      if (T == 1 || A - r0 <= BLK) {
        fmt(0);
        for (int t = 1; t < T; ++t) bufs[(size_t)t].clear();
      } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(fmt, t);
        for (auto &th : pool) th.join();
      }
      for (int t = 0; t < T; ++t) h.update(bufs[(size_t)t].data(), bufs[(size_t)t].size());
    }
    std::vector<char> fb;
    fb.reserve(1 << 20);
    for (size_t i = 0; i < fstate.size(); ++i) {
      char tmp[64];
      char *p = tmp;
      *p++ = 'f';
      *p++ = ' ';
      p = std::to_chars(p, p + 12, fstate[i]).ptr;
      *p++ = ' ';
      p = py_float_repr_to(fcost[i], p);
      *p++ = '\n';
      fb.insert(fb.end(), tmp, p);
      if (fb.size() > (1 << 20)) {
        h.update(fb.data(), fb.size());
        fb.clear();
      }
    }
    h.update(fb.data(), fb.size());
    fingerprint = h.hex();
  }
};

// Python int() / float() on one whitespace-free field (underscores between
// digits allowed, as Python does).
inline bool py_int(const char *b, const char *e, int64_t &v) {
  { // fast path: plain decimal digits
    const char *p = b;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    if (p < e && e - p <= 18) {
      int64_t x = 0;
      const char *q = p;
      for (; q < e && *q >= '0' && *q <= '9'; ++q) x = x * 10 + (*q - '0');
      if (q == e) {
        v = neg ? -x : x;
        return true;
      }
    }
  }
  std::string t;
  const char *p = b;
  if (p < e && (*p == '+' || *p == '-')) t += *p++;
  if (p == e) return false;
  bool prev_digit = false;
  for (; p < e; ++p) {
    if (*p >= '0' && *p <= '9') {
      t += *p;
      prev_digit = true;
    } else if (*p == '_' && prev_digit && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
      prev_digit = false;
    } else {
      return false;
    }
  }
  errno = 0;
  char *end = nullptr;
  const long long x = strtoll(t.c_str(), &end, 10);
  if (*end || errno) return false;
  v = x;
  return true;
}
inline bool py_float(const char *b, const char *e, double &v) {
  { // fast path: no underscores / sign prefix / hex (std::from_chars, exact like strtod)
    const char *p = b;
    bool plain = p < e && *p != '+';
    for (const char *q = b; q < e && plain; ++q) plain = *q != '_' && *q != 'x' && *q != 'X';
    if (plain) {
      const auto r = std::from_chars(p, e, v);
      if (r.ec == std::errc() && r.ptr == e) return true;
    }
  }
  std::string t;
  for (const char *p = b; p < e; ++p) {
    if (*p == '_') {
      if (p == b || p + 1 == e || !isdigit((unsigned char)p[-1]) || !isdigit((unsigned char)p[1])) return false;
      continue;
    }
    t += *p;
  }
  if (t.empty()) return false;
  char *end = nullptr;
  v = strtod(t.c_str(), &end);
  if (*end) return false;
  // Python rejects hex floats and "infinity"-like spellings strtod accepts only partly
  for (char c : t)
    if (c == 'x' || c == 'X' || c == 'p' || c == 'P') return false;
  return true;
}

// parse_text_fst + build_csr.  Returns 0, or 1 (parse error) / 2 (structure
// error) with `err` set to the reference's message.
struct ParsedRow {
  int32_t src, dst, il, ol;
  double w;
};
// Lines of one chunk of the text (line numbers from first_line).
struct ParseChunk {
  std::vector<ParsedRow> rows;
  std::vector<std::pair<int32_t, double>> finals;
  std::vector<std::pair<int32_t, int64_t>> final_line;
  bool have_start = false;
  int32_t start = 0;
  int64_t max_state = -1;
  int64_t err_line = -1; // first error of the chunk
  std::string err;
};

inline void parse_chunk(const char *text, size_t pos, size_t len, int64_t lineno, ParseChunk &R) {
  auto fail = [&](int64_t ln, const std::string &why, const char *b, const char *e) {
    std::string raw(b, e);
    if (!raw.empty() && raw.back() == '\r') raw.pop_back();
    R.err = "line " + std::to_string(ln) + ": " + why + ": '" + raw + "'";
    R.err_line = ln;
  };
  while (pos < len) {
    const char *nl = (const char *)memchr(text + pos, '\n', len - pos);
    const size_t eol = nl ? (size_t)(nl - text) : len;
    const char *lb = text + pos, *le = text + eol;
    pos = eol + 1;
    const char *b = lb, *e = le;
    while (b < e && py_space(*b)) ++b;
    while (e > b && py_space(e[-1])) --e;
    if (b == e || *b == '#') {
      ++lineno;
      continue;
    }
    const char *fb[6], *fe[6];
    int nf = 0;
    for (const char *p = b; p < e;) {
      while (p < e && py_space(*p)) ++p;
      if (p == e) break;
      const char *q = p;
      while (q < e && !py_space(*q)) ++q;
      if (nf < 6) {
        fb[nf] = p;
        fe[nf] = q;
      }
      ++nf;
      p = q;
    }
    if (nf == 4 || nf == 5) {
      int64_t v[4];
      for (int i = 0; i < 4; ++i)
        if (!py_int(fb[i], fe[i], v[i]))
          return fail(lineno, "invalid literal for int() with base 10: '" + std::string(fb[i], fe[i]) + "'", lb, le);
      double wv = 0.0;
      if (nf == 5 && !py_float(fb[4], fe[4], wv))
        return fail(lineno, "could not convert string to float: '" + std::string(fb[4], fe[4]) + "'", lb, le);
      if (std::min(std::min(v[0], v[1]), std::min(v[2], v[3])) < 0) return fail(lineno, "negative field", lb, le);
      if (!std::isfinite(wv)) return fail(lineno, "non-finite weight", lb, le);
      for (int i = 0; i < 4; ++i)
        if (v[i] > INT32_MAX) return fail(lineno, "field out of range", lb, le);
      R.rows.push_back(ParsedRow{(int32_t)v[0], (int32_t)v[1], (int32_t)v[2], (int32_t)v[3], wv});
      R.max_state = std::max(R.max_state, std::max(v[0], v[1]));
    } else if (nf == 1 || nf == 2) {
      int64_t st;
      if (!py_int(fb[0], fe[0], st))
        return fail(lineno, "invalid literal for int() with base 10: '" + std::string(fb[0], fe[0]) + "'", lb, le);
      double wv = 0.0;
      if (nf == 2 && !py_float(fb[1], fe[1], wv))
        return fail(lineno, "could not convert string to float: '" + std::string(fb[1], fe[1]) + "'", lb, le);
      if (st < 0) return fail(lineno, "negative state", lb, le);
      if (!std::isfinite(wv)) return fail(lineno, "non-finite weight", lb, le);
      if (st > INT32_MAX) return fail(lineno, "field out of range", lb, le);
      R.finals.emplace_back((int32_t)st, wv);
      R.final_line.emplace_back((int32_t)st, lineno);
      R.max_state = std::max(R.max_state, st);
    } else {
      return fail(lineno, "expected 1, 2, 4 or 5 fields, got " + std::to_string(nf), lb, le);
    }
    if (!R.have_start) {
      int64_t s0 = 0;
      py_int(fb[0], fe[0], s0);
      R.start = (int32_t)s0;
      R.have_start = true;
    }
    ++lineno;
  }
}

// parse_text_fst + build_csr.  Returns 0, or 1 (parse error) / 2 (structure
// error) with `err` set to the reference's message.  Large texts are parsed
// in newline-aligned chunks on several threads (line numbers and the first
// error are the same as a sequential parse).
inline int parse_text_fst(const char *text, size_t len, int64_t hint, HostFst &F, std::string &err) {
  int T = (int)std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), 64);
  if (len < ((size_t)1 << 22)) T = 1;
  std::vector<size_t> cut((size_t)T + 1, len);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {
    size_t c = std::max(cut[(size_t)t - 1], len / (size_t)T * (size_t)t);
    const char *nl = c < len ? (const char *)memchr(text + c, '\n', len - c) : nullptr;
    cut[(size_t)t] = nl ? (size_t)(nl - text) + 1 : len;
  }
  std::vector<int64_t> lines((size_t)T + 1, 1);
  std::vector<ParseChunk> parts((size_t)T);
  auto run = [&](auto fn) {
    if (T == 1) {
      fn(0);
      return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(fn, t);
    for (auto &th : pool) th.join();
  };
  std::vector<int64_t> nls((size_t)T, 0);
  run([&](int t) { // newlines per chunk -> first line number of each chunk
    int64_t n = 0;
    for (size_t p = cut[(size_t)t]; p < cut[(size_t)t + 1];) {
      const char *nl = (const char *)memchr(text + p, '\n', cut[(size_t)t + 1] - p);
      if (!nl) break;
      ++n;
      p = (size_t)(nl - text) + 1;
    }
    nls[(size_t)t] = n;
  });
  for (int t = 0; t < T; ++t) lines[(size_t)t + 1] = lines[(size_t)t] + nls[(size_t)t];
  run([&](int t) { parse_chunk(text, cut[(size_t)t], cut[(size_t)t + 1], lines[(size_t)t], parts[(size_t)t]); });
  for (const ParseChunk &c : parts)
    if (c.err_line >= 0) { // chunks are in line order: the first erroring chunk holds the first error
      err = c.err;
      return 1;
    }
  bool have_start = false;
  int64_t max_state = -1;
  size_t nrows = 0;
  for (const ParseChunk &c : parts) {
    if (!have_start && c.have_start) {
      F.start = c.start;
      have_start = true;
    }
    max_state = std::max(max_state, c.max_state);
    nrows += c.rows.size();
  }
  std::vector<ParsedRow> rows;
  std::vector<std::pair<int32_t, double>> finals;
  std::vector<std::pair<int32_t, int64_t>> final_line;
  if (T == 1) {
    rows.swap(parts[0].rows);
    finals.swap(parts[0].finals);
    final_line.swap(parts[0].final_line);
  } else {
    rows.reserve(nrows);
    for (ParseChunk &c : parts) {
      rows.insert(rows.end(), c.rows.begin(), c.rows.end());
      finals.insert(finals.end(), c.finals.begin(), c.finals.end());
      final_line.insert(final_line.end(), c.final_line.begin(), c.final_line.end());
      std::vector<ParsedRow>().swap(c.rows);
    }
  }
  if (!have_start) {
    err = "no start state: input contains no arc or final lines";
    return 1;
  }
  int64_t S = max_state + 1;
  if (hint >= 0) {
    if (hint < S) {
      err = "num_states_hint " + std::to_string(hint) + " smaller than highest referenced state " +
            std::to_string(max_state);
      return 2;
    }
    S = hint;
  }
  F.num_states = S;
  // duplicate finals (reported at the second occurrence, in line order)
  {
    std::vector<std::pair<int32_t, int64_t>> sorted = final_line;
    std::stable_sort(sorted.begin(), sorted.end(),
                     [](const std::pair<int32_t, int64_t> &a, const std::pair<int32_t, int64_t> &b) {
                       return a.first < b.first;
                     });
    int64_t bad_line = -1;
    int32_t bad_state = 0;
    for (size_t i = 1; i < sorted.size(); ++i)
      if (sorted[i].first == sorted[i - 1].first && (bad_line < 0 || sorted[i].second < bad_line)) {
        bad_line = sorted[i].second;
        bad_state = sorted[i].first;
      }
    if (bad_line >= 0) {
      err = "line " + std::to_string(bad_line) + ": duplicate final line for state " + std::to_string(bad_state);
      return 1;
    }
  }
  // state-major CSR, line order inside a state (stable counting sort)
  F.ro.assign((size_t)S + 1, 0);
  for (const ParsedRow &r : rows) F.ro[(size_t)r.src + 1]++;
  for (int64_t s = 0; s < S; ++s) F.ro[(size_t)s + 1] += F.ro[(size_t)s];
  const size_t A = rows.size();
  F.il.resize(A);
  F.ol.resize(A);
  F.ns.resize(A);
  F.w.resize(A);
  std::vector<int64_t> at(F.ro.begin(), F.ro.end() - 1);
  for (const ParsedRow &r : rows) {
    const int64_t g = at[(size_t)r.src]++;
    F.il[(size_t)g] = r.il;
    F.ol[(size_t)g] = r.ol;
    F.ns[(size_t)g] = r.dst;
    F.w[(size_t)g] = r.w;
  }
  std::sort(finals.begin(), finals.end(),
            [](const std::pair<int32_t, double> &a, const std::pair<int32_t, double> &b) { return a.first < b.first; });
  F.fstate.resize(finals.size());
  F.fcost.resize(finals.size());
  for (size_t i = 0; i < finals.size(); ++i) {
    F.fstate[i] = finals[i].first;
    F.fcost[i] = finals[i].second;
  }
  F.compute_fingerprint();
  return 0;
}

// Binary cache: magic, sizes, the source's (size, mtime) it was built from,
// the fingerprint, then the arrays.
struct CacheHeader {
  char magic[8];
  int64_t start, num_states, num_arcs, num_finals, src_size, src_mtime_ns;
  char fingerprint[64];
};

inline bool save_cache(const char *path, const HostFst &F, int64_t src_size, int64_t src_mtime) {
  FILE *f = fopen(path, "wb");
  if (!f) return false;
  CacheHeader h;
  memcpy(h.magic, "ABCSR01\0", 8);
  h.start = F.start;
  h.num_states = F.num_states;
  h.num_arcs = (int64_t)F.il.size();
  h.num_finals = (int64_t)F.fstate.size();
  h.src_size = src_size;
  h.src_mtime_ns = src_mtime;
  memcpy(h.fingerprint, F.fingerprint.data(), 64);
  bool ok = fwrite(&h, sizeof(h), 1, f) == 1;
  auto put = [&](const void *p, size_t n) { ok = ok && (n == 0 || fwrite(p, 1, n, f) == n); };
  put(F.ro.data(), F.ro.size() * 8);
  put(F.il.data(), F.il.size() * 4);
  put(F.ol.data(), F.ol.size() * 4);
  put(F.ns.data(), F.ns.size() * 4);
  put(F.w.data(), F.w.size() * 8);
  put(F.fstate.data(), F.fstate.size() * 4);
  put(F.fcost.data(), F.fcost.size() * 8);
  ok = (fclose(f) == 0) && ok;
  return ok;
}

inline bool load_cache(const char *path, HostFst &F, int64_t src_size, int64_t src_mtime) {
  FILE *f = fopen(path, "rb");
  if (!f) return false;
  CacheHeader h;
  bool ok = fread(&h, sizeof(h), 1, f) == 1 && memcmp(h.magic, "ABCSR01\0", 8) == 0 &&
            h.src_size == src_size && h.src_mtime_ns == src_mtime && h.num_states >= 0 && h.num_arcs >= 0 &&
            h.num_finals >= 0;
  if (ok) {
    F.start = (int32_t)h.start;
    F.num_states = h.num_states;
    F.ro.resize((size_t)h.num_states + 1);
    F.il.resize((size_t)h.num_arcs);
    F.ol.resize((size_t)h.num_arcs);
    F.ns.resize((size_t)h.num_arcs);
    F.w.resize((size_t)h.num_arcs);
    F.fstate.resize((size_t)h.num_finals);
    F.fcost.resize((size_t)h.num_finals);
    auto get = [&](void *p, size_t n) { ok = ok && (n == 0 || fread(p, 1, n, f) == n); };
    get(F.ro.data(), F.ro.size() * 8);
    get(F.il.data(), F.il.size() * 4);
    get(F.ol.data(), F.ol.size() * 4);
    get(F.ns.data(), F.ns.size() * 4);
    get(F.w.data(), F.w.size() * 8);
    get(F.fstate.data(), F.fstate.size() * 4);
    get(F.fcost.data(), F.fcost.size() * 8);
    F.fingerprint.assign(h.fingerprint, 64);
  }
  fclose(f);
  return ok;
}

} // namespace ab
