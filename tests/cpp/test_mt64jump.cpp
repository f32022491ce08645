// CPU check of the MT19937-64 jump-ahead (paper_1308_2400_b200/csrc/mt64jump.h):
// the characteristic polynomial has degree 19937, and a window jumped by J
// equals std::mt19937_64's outputs J .. J+311 (discard(J) then 312 draws) --
// from offset 0 and chained from another jumped window.
#include <cstdio>
#include <random>

#include "mt64jump.h"

static uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

static int check(const char* what, uint64_t seed, uint64_t off, const uint64_t* win) {
  std::mt19937_64 g(seed);
  g.discard(off);
  for (int w = 0; w < mt64jump::kN; ++w) {
    const uint64_t want = g();
    if (temper(win[w]) != want) {
      std::printf("FAIL %s seed %llu offset %llu word %d\n", what, (unsigned long long)seed,
                  (unsigned long long)off, w);
      return 1;
    }
  }
  return 0;
}

int main() {
  const auto& f = mt64jump::field();
  if (!f.ok) {
    std::printf("FAIL characteristic polynomial degree\n");
    return 1;
  }
  int bad = 0;
  const uint64_t seeds[] = {0ull, 5489ull, 0xFFFFFFFFFFFFFFFFull};
  const uint64_t jumps[] = {1, 311, 312, 313, 19937, 100003, 638976, 3 * 638976 + 17};
  for (uint64_t seed : seeds) {
    uint64_t w0[312], w1[312], w2[312];
    mt64jump::seed_window(seed, w0);
    bad += check("window 0", seed, 0, w0);
    for (uint64_t J : jumps) {
      mt64jump::apply_jump(f.xpow(J), w0, w1);
      bad += check("jump", seed, J, w1);
    }
    // chained: 638976 then 2 * 638976 (the tree's composition)
    mt64jump::apply_jump(f.xpow(638976), w0, w1);
    mt64jump::apply_jump(f.xpow(2 * 638976), w1, w2);
    bad += check("chained", seed, 3 * 638976, w2);
    // x^(a+b) = x^a x^b mod phi
    const auto p = f.mulmod(f.xpow(638976), f.xpow(2 * 638976));
    mt64jump::apply_jump(p, w0, w1);
    bad += check("mulmod", seed, 3 * 638976, w1);
  }
  std::printf(bad ? "FAILED %d\n" : "ok\n", bad);
  return bad ? 1 : 0;
}
