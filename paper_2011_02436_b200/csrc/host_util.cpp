// Host-only utilities of the C ABI: init_hidden, accuracy, and the seeded
// synthetic-data generators used by tests and bench.py.
//
// init_hidden restates elm.cpp:20-25,74-91 exactly: mt19937_64(seed), W filled
// row-major (input i outer, node j inner) then b, each draw (gen()>>11)*2^-53
// mapped to [-1, 1].  std::mt19937_64 is fully specified by the C++ standard,
// so W and b are bit-identical to the reference's on every platform.
#include "../../include/rbpelm_b200.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

void set_status(rbpg_status* st, int code, const std::string& msg) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->code = code;
  std::snprintf(st->message, sizeof st->message, "%s", msg.c_str());
}

inline double unit53(std::mt19937_64& gen) { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }

// Box-Muller, cosine branch only; u1 in (0, 1] so the log is finite.
inline double normal01(std::mt19937_64& gen) {
  const double u1 = (static_cast<double>(gen() >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = unit53(gen);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

// std::mt19937_64 (the C++ standard's parameters: n = 312, m = 156, r = 31,
// a = 0xB5026F5AA96619E9, tempering u = 29 / d = 0x5555555555555555, s = 17 / b = 0x71D67FFFEDA60000,
// t = 37 / c = 0xFFF7EEE000000000, l = 43, seeding f = 6364136223846793005), generated a whole
// 312-word block at a time: the twist and the tempering are straight loops the compiler
// vectorises.  Output-identical to std::mt19937_64 (pinned in the CPU tests); init_hidden sits on
// the end-to-end critical path (the hidden build waits for W).
class Mt64Block {
 public:
  explicit Mt64Block(std::uint64_t seed) {
    mt_[0] = seed;
    for (int i = 1; i < kN; ++i) mt_[i] = 6364136223846793005ull * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
    pos_ = kN;
  }
  std::uint64_t operator()() {
    if (pos_ == kN) refill();
    return out_[pos_++];
  }

 private:
  static constexpr int kN = 312, kM = 156;
  static constexpr std::uint64_t kA = 0xB5026F5AA96619E9ull, kUpper = 0xFFFFFFFF80000000ull,
                                 kLower = 0x7FFFFFFFull;
  static inline std::uint64_t twist(std::uint64_t a, std::uint64_t b, std::uint64_t c) {
    const std::uint64_t y = (a & kUpper) | (b & kLower);
    return c ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
  }
  void refill() {
    for (int i = 0; i < kN - kM; ++i) mt_[i] = twist(mt_[i], mt_[i + 1], mt_[i + kM]);
    for (int i = kN - kM; i < kN - 1; ++i) mt_[i] = twist(mt_[i], mt_[i + 1], mt_[i + kM - kN]);
    mt_[kN - 1] = twist(mt_[kN - 1], mt_[0], mt_[kM - 1]);
    for (int i = 0; i < kN; ++i) {
      std::uint64_t z = mt_[i];
      z ^= (z >> 29) & 0x5555555555555555ull;
      z ^= (z << 17) & 0x71D67FFFEDA60000ull;
      z ^= (z << 37) & 0xFFF7EEE000000000ull;
      z ^= z >> 43;
      out_[i] = z;
    }
    pos_ = 0;
  }
  std::uint64_t mt_[kN];
  std::uint64_t out_[kN];
  int pos_;
};

constexpr std::size_t kBlockRows = 65536;
inline std::uint64_t block_seed(std::uint64_t seed, std::size_t block) {
  return seed ^ (0x9E3779B97F4A7C15ull * static_cast<std::uint64_t>(block + 1));
}

}  // namespace

extern "C" {

const char* rbpg_version(void) { return "rbpelm-b200 0.1 (sm_100a)"; }

int rbpg_init_hidden(size_t inputs, size_t hidden, size_t outputs, uint64_t seed, double* w, double* b,
                     rbpg_status* st) {
  if (inputs < 1 || hidden < 1 || outputs < 1) {
    set_status(st, RBPG_INVALID_ARGUMENT, "ElmParams: inputs, hidden_nodes and outputs must be >= 1");
    return RBPG_INVALID_ARGUMENT;
  }
  Mt64Block gen(seed);
  for (size_t i = 0; i < inputs; ++i)
    for (size_t j = 0; j < hidden; ++j) w[i * hidden + j] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
  for (size_t j = 0; j < hidden; ++j) b[j] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
  set_status(st, RBPG_OK, "");
  return RBPG_OK;
}

int rbpg_accuracy(const double* pred, size_t rows, size_t cols, const double* y, size_t yrows, size_t ycols,
                  double* out, rbpg_status* st) {
  if (rows != yrows || cols != ycols) {
    set_status(st, RBPG_SHAPE_ERROR,
               "accuracy: shapes differ, " + std::to_string(rows) + "x" + std::to_string(cols) + " vs " +
                   std::to_string(yrows) + "x" + std::to_string(ycols));
    return RBPG_SHAPE_ERROR;
  }
  size_t hits = 0;
  for (size_t i = 0; i < rows; ++i) {
    size_t ap = 0, ay = 0;
    for (size_t j = 1; j < cols; ++j) {
      if (pred[i * cols + j] > pred[i * cols + ap]) ap = j;
      if (y[i * cols + j] > y[i * cols + ay]) ay = j;
    }
    hits += (ap == ay);
  }
  *out = static_cast<double>(hits) / static_cast<double>(rows);
  set_status(st, RBPG_OK, "");
  return RBPG_OK;
}

int rbpg_synth_classification(size_t row0, size_t n, size_t d, size_t m, uint64_t seed, uint64_t teacher_seed,
                              double noise_sigma, double* x, double* t, rbpg_status* st) {
  if (d < 1 || m < 1) {
    set_status(st, RBPG_INVALID_ARGUMENT, "synth: d and m must be >= 1");
    return RBPG_INVALID_ARGUMENT;
  }
  std::vector<double> v(d * m);
  {
    std::mt19937_64 tg(teacher_seed);
    for (auto& e : v) e = normal01(tg);
  }
  std::vector<double> xr(d), logits(m);
  size_t row = row0;
  const size_t end = row0 + n;
  while (row < end) {
    const size_t blk = row / kBlockRows;
    std::mt19937_64 gen(block_seed(seed, blk));
    const size_t bstart = blk * kBlockRows, bend = std::min(end, bstart + kBlockRows);
    for (size_t r = bstart; r < bend; ++r) {
      for (size_t k = 0; k < d; ++k) xr[k] = unit53(gen);
      for (size_t c = 0; c < m; ++c) logits[c] = noise_sigma * normal01(gen);
      if (r < row) continue;  // rows before the requested range inside this block
      for (size_t c = 0; c < m; ++c) {
        double s = 0.0;
        for (size_t k = 0; k < d; ++k) s += xr[k] * v[k * m + c];
        logits[c] += s;
      }
      size_t am = 0;
      for (size_t c = 1; c < m; ++c)
        if (logits[c] > logits[am]) am = c;
      const size_t o = r - row0;
      std::memcpy(x + o * d, xr.data(), sizeof(double) * d);
      for (size_t c = 0; c < m; ++c) t[o * m + c] = (c == am) ? 1.0 : 0.0;
    }
    row = bend;
  }
  set_status(st, RBPG_OK, "");
  return RBPG_OK;
}

// Config 3 inputs: X = [B, B C] with B iid U[0,1] (n x base) and C iid U[-1,1] (base x base, from
// mix_seed); T one-hot from the teacher on the full X.
int rbpg_synth_rank_deficient(size_t n, size_t base, size_t m, uint64_t seed, uint64_t mix_seed,
                              uint64_t teacher_seed, double noise_sigma, double* x, double* t, rbpg_status* st) {
  const size_t d = 2 * base;
  std::vector<double> bm(n * base), tb(n * m);
  int rc = rbpg_synth_classification(0, n, base, m, seed, teacher_seed, noise_sigma, bm.data(), tb.data(), st);
  if (rc) return rc;
  std::vector<double> cm(base * base);
  {
    std::mt19937_64 g(mix_seed);
    for (auto& e : cm) e = 2.0 * unit53(g) - 1.0;
  }
  std::vector<double> v(d * m);
  {
    std::mt19937_64 tg(teacher_seed ^ 0x5bd1e995ull);
    for (auto& e : v) e = normal01(tg);
  }
  std::mt19937_64 ng(seed ^ 0xc2b2ae3d27d4eb4full);
  std::vector<double> logits(m);
  for (size_t r = 0; r < n; ++r) {
    double* xr = x + r * d;
    for (size_t k = 0; k < base; ++k) xr[k] = bm[r * base + k];
    for (size_t k = 0; k < base; ++k) {
      double s = 0.0;
      for (size_t q = 0; q < base; ++q) s += bm[r * base + q] * cm[q * base + k];
      xr[base + k] = s;
    }
    for (size_t c = 0; c < m; ++c) {
      double s = noise_sigma * normal01(ng);
      for (size_t k = 0; k < d; ++k) s += xr[k] * v[k * m + c];
      logits[c] = s;
    }
    size_t am = 0;
    for (size_t c = 1; c < m; ++c)
      if (logits[c] > logits[am]) am = c;
    for (size_t c = 0; c < m; ++c) t[r * m + c] = (c == am) ? 1.0 : 0.0;
  }
  set_status(st, RBPG_OK, "");
  return RBPG_OK;
}

// Overwrite `ndup` hidden nodes with exact copies (W column and bias) of distinct other nodes.
// Positions come from a seeded Fisher-Yates shuffle: perm[0:ndup] are the targets, perm[ndup:2ndup]
// their sources.  target_out/source_out (ndup each) may be NULL.
int rbpg_duplicate_nodes(double* w, double* b, size_t d, size_t l, size_t ndup, uint64_t seed, size_t* target_out,
                         size_t* source_out, rbpg_status* st) {
  if (2 * ndup > l) {
    set_status(st, RBPG_INVALID_ARGUMENT, "duplicate_nodes: need 2*ndup <= L");
    return RBPG_INVALID_ARGUMENT;
  }
  std::vector<size_t> perm(l);
  for (size_t i = 0; i < l; ++i) perm[i] = i;
  std::mt19937_64 g(seed);
  for (size_t i = l - 1; i > 0; --i) {
    const size_t j = static_cast<size_t>(g() % (i + 1));
    std::swap(perm[i], perm[j]);
  }
  for (size_t q = 0; q < ndup; ++q) {
    const size_t tgt = perm[q], src = perm[ndup + q];
    for (size_t i = 0; i < d; ++i) w[i * l + tgt] = w[i * l + src];
    b[tgt] = b[src];
    if (target_out) target_out[q] = tgt;
    if (source_out) source_out[q] = src;
  }
  set_status(st, RBPG_OK, "");
  return RBPG_OK;
}

}  // extern "C"
