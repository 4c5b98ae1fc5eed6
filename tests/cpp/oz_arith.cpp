// Host restatement of the INT8 path's scalar arithmetic (csrc/k_ozaki.cu) -- test infrastructure:
//   exp_sig     branch-free Cody-Waite + degree-13 Taylor exp of the sigmoid epilogue: <= 1 ulp vs std::exp
//   i51_to_f64  exact int64 -> double by the 1.5 * 2^52 magic add (|t| < 2^51)
//   digits      balanced base-256 digit bytes by the 0x808080808080 bias trick == the per-digit loop
// Exit code 0 and "PASS" on success.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

static double as_d(uint64_t b) { double d; std::memcpy(&d, &b, 8); return d; }
static uint64_t as_u(double d) { uint64_t b; std::memcpy(&b, &d, 8); return b; }
static double pow2i(int e) { return as_d(static_cast<uint64_t>(e + 1023) << 52); }

static double exp_sig(double t) {
  const double kb = std::fma(t, 0x1.71547652b82fep0, 0x1.8p52);
  const int k = static_cast<int>(static_cast<uint32_t>(as_u(kb)));
  const double kd = kb - 0x1.8p52;
  double r = std::fma(-kd, 0x1.62e42fefa39efp-1, t);
  r = std::fma(-kd, 0x1.abc9e3b39803fp-56, r);
  const double c[14] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
                        1.0 / 40320.0, 1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0, 1.0};
  double q = c[0];
  for (int i = 1; i < 14; ++i) q = std::fma(q, r, c[i]);
  const int k1 = k >> 1;
  const double v = (q * pow2i(k1)) * pow2i(k - k1);
  return t > 709.782712893384 ? INFINITY : (t < -745.1332191019412 ? 0.0 : v);
}

static double i51_to_f64(long long t) {
  const double m = 0x1.8p52;
  return as_d(as_u(m) + static_cast<uint64_t>(t)) - m;
}

int main() {
  std::mt19937_64 g(7);
  int fails = 0;
  // exp_sig
  std::uniform_real_distribution<double> wide(-746.0, 710.0), mid(-40.0, 40.0);
  double maxulp = 0.0;
  for (int i = 0; i < 4000000; ++i) {
    const double t = (i & 1) ? wide(g) : mid(g);
    const double a = exp_sig(t), b = std::exp(t);
    if (std::isinf(b) || b < 2.3e-308) {  // overflow / subnormal range: inf, or a value whose 1 + e rounds to 1
      if (std::isinf(b) != std::isinf(a) || (!std::isinf(b) && a > 2.3e-308)) ++fails;
      continue;
    }
    const double ulp = std::fabs(a - b) / (std::nextafter(b, INFINITY) - b);
    if (ulp > maxulp) maxulp = ulp;
  }
  if (maxulp > 1.0) ++fails;
  if (!std::isnan(exp_sig(NAN)) || exp_sig(800.0) != INFINITY || exp_sig(-800.0) != 0.0) ++fails;
  // i51_to_f64
  std::uniform_int_distribution<long long> ints(-(1LL << 51) + 1, (1LL << 51) - 1);
  for (int i = 0; i < 1000000; ++i) {
    const long long t = ints(g);
    if (i51_to_f64(t) != static_cast<double>(t)) ++fails;
  }
  // digit bytes: bias trick vs the balanced-digit loop (7 planes, |X| < 2^54)
  std::uniform_int_distribution<long long> xs(-(1LL << 54) + 1, (1LL << 54) - 1);
  for (int i = 0; i < 1000000; ++i) {
    const long long X0 = (i % 97 == 0) ? 0 : xs(g);
    long long X = X0;
    int8_t loop[7];
    for (int p = 6; p >= 1; --p) {
      const long long d = ((X + 128) & 255) - 128;
      X = (X - d) >> 8;
      loop[p] = static_cast<int8_t>(d);
    }
    loop[0] = static_cast<int8_t>(X);
    const uint64_t kBias = 0x808080808080ull;
    const uint64_t V = (static_cast<uint64_t>(X0) + kBias) ^ kBias;
    for (int b = 0; b < 7; ++b)
      if (static_cast<int8_t>(V >> (8 * b)) != loop[6 - b]) ++fails;
    if (loop[0] < -64 || loop[0] > 64) ++fails;
  }
  std::printf("exp_sig max ulp %.3f; %d failures\n%s\n", maxulp, fails, fails ? "FAIL" : "PASS");
  return fails ? 1 : 0;
}
