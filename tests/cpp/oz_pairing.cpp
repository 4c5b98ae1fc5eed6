// Harness for the INT8 Gram's CTA-pair item list (csrc/k_ozaki.cu oz_pair_order / oz_pair_items, host
// code): every lower 128 x 128 tile of an nbI x nbI tile grid is produced exactly once, both CTAs of an
// item share the B column block, and the count matches.  The functions are spliced in by the test
// (tests/test_ozaki_scheme.py) from the product source, between the OZ_PAIR_SRC markers below.
#include <algorithm>
#include <cstdio>
#include <set>
#include <utility>
#include <vector>
struct int2 {
  int x, y;
};
static int2 make_int2(int x, int y) { return {x, y}; }
// OZ_PAIR_SRC
int main() {
  for (int nbI = 1; nbI <= 160; ++nbI) {
    for (int B : {1, 3, 6}) {
      std::vector<int2> o(size_t(nbI) * nbI + 2);
      const int n = oz_pair_order(nbI, B, o.data());
      if (n != oz_pair_items(nbI)) { std::printf("FAIL count nbI %d\n", nbI); return 1; }
      std::multiset<std::pair<int, int>> seen;
      for (int i = 0; i < n; ++i) {
        const int a0 = o[i].x >> 16, a1 = o[i].x & 0xFFFF, b = o[i].y;
        for (int a : {a0, a1 == 0xFFFF ? -1 : a1}) {
          if (a < 0) continue;
          if (a >= nbI || b >= nbI) { std::printf("FAIL range\n"); return 1; }
          seen.insert(a >= b ? std::make_pair(a, b) : std::make_pair(b, a));
        }
      }
      for (int a = 0; a < nbI; ++a)
        for (int c = 0; c <= a; ++c)
          if (seen.count({a, c}) != 1) { std::printf("FAIL tile %d %d nbI %d\n", a, c, nbI); return 1; }
      if (int(seen.size()) != nbI * (nbI + 1) / 2) { std::printf("FAIL extra\n"); return 1; }
      if (2 * n > nbI * (nbI + 1) / 2 + nbI) { std::printf("FAIL not paired nbI %d\n", nbI); return 1; }
    }
  }
  std::printf("PASS\n");
  return 0;
}
