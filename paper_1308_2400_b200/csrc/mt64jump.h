// mt64jump.h -- jump-ahead for the MT19937-64 stream (host side), so the
// device can generate the reference's ONE std::mt19937_64 stream
// (random.hpp:111-129) in parallel: every CTA starts at its own offset of the
// same stream instead of one CTA walking it serially.
//
// The generator's state transition is linear over GF(2). Its 19937-bit
// relevant state has a primitive characteristic polynomial phi (degree
// D = 19937), so every bit of the raw (untempered) words v_k obeys the linear
// recurrence with characteristic polynomial phi for k >= 312 (the words the
// generator produced itself; the seeded words' unused low bits drop out).
// Hence, with p(x) = x^J mod phi = sum_i c_i x^i,
//
//     v_{k+J} = XOR_{i : c_i = 1} v_{k+i}          for every k >= 312,
//
// so the 312-word window at stream offset k+J is a GF(2) convolution of the
// ~20k words following offset k -- computed on the device (generate.cu,
// k_mt_jump). This header only finds phi (Berlekamp-Massey over the stream's
// low output bit) and the jump polynomials x^J mod phi (Barrett reduction over
// carry-less products); both are computed once per process.
//
// Window convention shared with generate.cu: the window at output offset p
// is the raw words whose tempered values are outputs p .. p+311, i.e.
// v[312+p .. 624+p) in the numbering where v[0..312) is the seeded state.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>
#if defined(__PCLMUL__)
#include <wmmintrin.h>
#endif

namespace mt64jump {

constexpr int kN = 312, kM = 156;  // words of state, middle offset
constexpr int kD = 19937;          // degree of phi
constexpr int kW = 312;            // 64-bit words of a polynomial of degree <= kD
constexpr uint64_t kA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

using Poly = std::vector<uint64_t>;  // bit i = coefficient of x^i

inline uint64_t mix(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t x = (a & kUpper) | (b & kLower);
  return c ^ (x >> 1) ^ ((x & 1ull) ? kA : 0ull);
}

// std::mt19937_64(seed)'s state, then one twist: the window at offset 0.
inline void seed_window(uint64_t seed, uint64_t* win) {
  uint64_t st[kN];
  st[0] = seed;
  for (uint64_t i = 1; i < (uint64_t)kN; ++i)
    st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + i;
  // v[312 + i] = f(v[i], v[i+1], v[i+156]) over the linear stream
  uint64_t v[2 * kN];
  std::memcpy(v, st, sizeof st);
  for (int i = 0; i < kN; ++i) v[kN + i] = mix(v[i], v[i + 1], v[i + kM]);
  std::memcpy(win, v + kN, kN * sizeof(uint64_t));
}

// ---- GF(2)[x] arithmetic ----------------------------------------------------

inline void clmul(uint64_t a, uint64_t b, uint64_t* lo, uint64_t* hi) {
#if defined(__PCLMUL__)
  const __m128i r = _mm_clmulepi64_si128(_mm_set_epi64x(0, (long long)a),
                                         _mm_set_epi64x(0, (long long)b), 0);
  *lo = (uint64_t)_mm_cvtsi128_si64(r);
  *hi = (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(r, r));
#else
  // 4-bit windows of b: 16 multiples of a (as 128-bit values)
  uint64_t tl[16], th[16];
  tl[0] = th[0] = 0;
  for (int u = 1; u < 16; ++u) {
    const int t = 31 - __builtin_clz((unsigned)u);  // top bit of u (u < 16)
    const int rest = u ^ (1 << t);
    tl[u] = tl[rest] ^ (a << t);
    th[u] = th[rest] ^ (t ? a >> (64 - t) : 0);
  }
  uint64_t l = 0, h = 0;
  for (int s = 60; s >= 0; s -= 4) {
    h = (h << 4) | (l >> 60);
    l <<= 4;
    const unsigned u = (unsigned)(b >> s) & 15u;
    l ^= tl[u];
    h ^= th[u];
  }
  *lo = l;
  *hi = h;
#endif
}

// r = a * b, r sized na + nb words
inline Poly mul(const Poly& a, const Poly& b) {
  Poly r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    if (!a[i]) continue;
    for (size_t j = 0; j < b.size(); ++j) {
      uint64_t lo, hi;
      clmul(a[i], b[j], &lo, &hi);
      r[i + j] ^= lo;
      r[i + j + 1] ^= hi;
    }
  }
  return r;
}

inline bool bit(const Poly& p, uint64_t i) {
  return (i >> 6) < p.size() && ((p[i >> 6] >> (i & 63)) & 1ull);
}

// p >> s (division by x^s, floor), into `words` words
inline Poly shr(const Poly& p, uint64_t s, size_t words) {
  Poly r(words, 0);
  const uint64_t w = s >> 6, b = s & 63;
  for (size_t i = 0; i < words; ++i) {
    const uint64_t k = i + w;
    uint64_t x = k < p.size() ? p[k] >> b : 0;
    if (b && k + 1 < p.size()) x |= p[k + 1] << (64 - b);
    r[i] = x;
  }
  return r;
}

// a ^= b << s (b shifted left by s bits), a large enough
inline void xor_shl(Poly& a, const Poly& b, uint64_t s) {
  const uint64_t w = s >> 6, bs = s & 63;
  for (size_t i = 0; i < b.size(); ++i) {
    if (!b[i]) continue;
    if (i + w < a.size()) a[i + w] ^= b[i] << bs;
    if (bs && i + w + 1 < a.size()) a[i + w + 1] ^= b[i] >> (64 - bs);
  }
}

inline void trim_to_degree_below(Poly& p, uint64_t bits) {
  const size_t words = (bits + 63) / 64;
  p.resize(words, 0);
  if (bits & 63) p[words - 1] &= (1ull << (bits & 63)) - 1;
}

// ---- the characteristic polynomial (Berlekamp-Massey) ----------------------

// Minimal polynomial of the low output bit of std::mt19937_64 (tempering is
// an invertible linear map of each word, so that bit sequence obeys phi);
// returned as phi itself (monic, degree kD) -- the reciprocal of the
// connection polynomial BM finds.
inline Poly charpoly() {
  const uint64_t nbits = 2 * (uint64_t)kD + 256;
  const size_t nw = (nbits + 63) / 64 + 4;
  // s reversed: rs bit t = s[nbits - 1 - t], so the discrepancy of step n is
  // a word-aligned dot product of C with rs from bit (nbits - 1 - n)
  Poly rs(nw, 0);
  std::mt19937_64 g(20130811ull);
  for (uint64_t n = 0; n < nbits; ++n) {
    if (g() & 1ull) {
      const uint64_t t = nbits - 1 - n;
      rs[t >> 6] |= 1ull << (t & 63);
    }
  }
  const size_t cw = (nbits + 63) / 64 + 2;
  Poly C(cw, 0), B(cw, 0), T;
  C[0] = B[0] = 1;
  uint64_t L = 0, m = 1;
  for (uint64_t n = 0; n < nbits; ++n) {
    const uint64_t off = nbits - 1 - n;  // rs bit of s[n]; s[n-i] at off + i
    const uint64_t ow = off >> 6, ob = off & 63;
    const size_t words = (size_t)(L / 64 + 1);
    uint64_t acc = 0;
    for (size_t k = 0; k < words; ++k) {
      uint64_t x = rs[ow + k] >> ob;
      if (ob) x |= rs[ow + k + 1] << (64 - ob);
      acc ^= x & C[k];
    }
    // C has no coefficient beyond degree L, so the dot product covers i <= L
    if (!(__builtin_popcountll(acc) & 1)) {
      ++m;
      continue;
    }
    if (2 * L <= n) {
      T = C;
      xor_shl(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shl(C, B, m);
      ++m;
    }
  }
  // phi_j = C_{L-j}
  Poly phi((size_t)(L / 64 + 1), 0);
  for (uint64_t j = 0; j <= L; ++j)
    if (bit(C, L - j)) phi[j >> 6] |= 1ull << (j & 63);
  return phi;  // degree L (== kD for MT19937-64; checked by the caller)
}

// ---- reduction mod phi ------------------------------------------------------

struct Field {
  Poly phi;  // degree kD, kW words (bit kD lies in word 311)
  Poly mu;   // floor(x^(2 kD) / phi), degree kD
  bool ok = false;

  Field() {
    phi = charpoly();
    uint64_t deg = 0;
    for (uint64_t i = 0; i < (uint64_t)phi.size() * 64; ++i)
      if (bit(phi, i)) deg = i;
    ok = deg == (uint64_t)kD && bit(phi, 0);
    phi.resize(kW, 0);
    // long division of x^(2D) by phi: quotient bits D..0
    Poly r((2 * kD) / 64 + 2, 0);
    r[(2 * kD) >> 6] |= 1ull << ((2 * kD) & 63);
    mu.assign(kW, 0);
    for (int64_t pos = 2 * kD; pos >= kD; --pos) {
      if (!bit(r, (uint64_t)pos)) continue;
      xor_shl(r, phi, (uint64_t)(pos - kD));
      const uint64_t q = (uint64_t)(pos - kD);
      mu[q >> 6] |= 1ull << (q & 63);
    }
  }

  // a mod phi for deg a < 2 kD - 1 (Barrett: exact for polynomials)
  Poly reduce(const Poly& a) const {
    const Poly hi = shr(a, kD, kW);           // floor(a / x^D), degree < D - 1
    const Poly q = shr(mul(hi, mu), kD, kW);  // floor(hi * mu / x^D)
    Poly r = a;
    r.resize(2 * kW + 2, 0);
    const Poly qp = mul(q, phi);
    for (size_t i = 0; i < qp.size() && i < r.size(); ++i) r[i] ^= qp[i];
    trim_to_degree_below(r, kD);
    r.resize(kW, 0);
    return r;
  }

  Poly mulmod(const Poly& a, const Poly& b) const { return reduce(mul(a, b)); }

  // x^J mod phi (left-to-right square and multiply by x)
  Poly xpow(uint64_t J) const {
    Poly p(kW, 0);
    p[0] = 1;
    if (J == 0) return p;
    int top = 63 - __builtin_clzll(J);
    for (int b = top; b >= 0; --b) {
      p = mulmod(p, p);
      if ((J >> b) & 1ull) {  // p *= x
        uint64_t carry = 0;
        for (int i = 0; i < kW; ++i) {
          const uint64_t nc = p[i] >> 63;
          p[i] = (p[i] << 1) | carry;
          carry = nc;
        }
        if (bit(p, kD))
          for (int i = 0; i < kW; ++i) p[i] ^= phi[i];
      }
    }
    return p;
  }
};

inline const Field& field() {
  static const Field f;  // thread-safe one-time init (~tens of ms)
  return f;
}

// Host application of a jump polynomial (tests; the device does it in
// generate.cu): the window at offset k + J from the window at offset k.
inline void apply_jump(const Poly& c, const uint64_t* win, uint64_t* out) {
  std::vector<uint64_t> v((size_t)kN * 65);
  std::memcpy(v.data(), win, kN * sizeof(uint64_t));
  for (size_t k = kN; k < v.size(); ++k) v[k] = mix(v[k - kN], v[k - kN + 1], v[k - kN + kM]);
  for (int w = 0; w < kN; ++w) out[w] = 0;
  for (uint64_t i = 0; i < (uint64_t)kD; ++i) {
    if (!bit(c, i)) continue;
    for (int w = 0; w < kN; ++w) out[w] ^= v[i + w];
  }
}

}  // namespace mt64jump
