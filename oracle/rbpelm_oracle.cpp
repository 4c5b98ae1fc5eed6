// ============================================================================
// TEST INFRASTRUCTURE -- NOT PRODUCT CODE.
//
// CPU oracle for the RBP-ELM training hot path: an Eigen-free C++ restatement
// of the reference's algorithm (arXiv 2011.02436 artefact, /root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load this library, and only as the checker or the timed CPU baseline.
// The product path (paper_2011_02436_b200) never links or calls it.
//
// Why a restatement: the reference needs Eigen 3 (proj/CMakeLists.txt:12),
// which is not installed in this image or on the GPU box, so the reference
// library cannot be compiled here.  Every function below
// cites the reference file:line it follows.  Bit-level parity with Eigen's
// kernels is unpinned (no golden vectors exist in the reference);
// the oracle is pinned by porting the reference's own known-answer and
// tolerance tests (tests/test_oracle_*.py).
//
// Floating-point contract: compiled with -ffp-contract=off so that every
// a*b+c is a rounded multiply followed by a rounded add, as in the reference's
// SSE2 build (no -march, proj/CMakeLists.txt:23-24).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <atomic>
#include <thread>

namespace oracle {

constexpr double kEps = std::numeric_limits<double>::epsilon();

// ---- error model (reference: matrix.hpp:11-14, linalg.hpp:15-20, elm.hpp:67-72)
struct ShapeError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct SingularMatrix : std::runtime_error {
  SingularMatrix(std::size_t i, double v)
      : std::runtime_error("non-positive pivot " + std::to_string(v) + " at index " + std::to_string(i) +
                           " in symmetric factorization"),
        index(i), value(v) {}
  std::size_t index;
  double value;
};
struct SingularSplit : std::runtime_error {
  explicit SingularSplit(int b)
      : std::runtime_error(std::string("singular ") + (b == 0 ? "A" : "D") + " block after ridge retry"), block(b) {}
  int block;  // 0 = A, 1 = D
};

// ---- minimal row-major matrix (reference DenseMatrix, matrix.hpp:18-51)
struct Mat {
  std::size_t r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(std::size_t rows, std::size_t cols, double fill = 0.0) : r(rows), c(cols), v(rows * cols, fill) {}
  double& operator()(std::size_t i, std::size_t j) { return v[i * c + j]; }
  double operator()(std::size_t i, std::size_t j) const { return v[i * c + j]; }
  std::string shape() const { return std::to_string(r) + "x" + std::to_string(c); }
};

static Mat from_ptr(const double* p, std::size_t r, std::size_t c) {
  Mat m(r, c);
  std::memcpy(m.v.data(), p, sizeof(double) * r * c);
  return m;
}

static bool all_finite(const Mat& m) {
  for (double x : m.v)
    if (!std::isfinite(x)) return false;
  return true;
}

static int g_threads = 1;

// Dynamic-schedule parallel loop over [0, count).  Each index is processed by
// exactly one thread with the same arithmetic as the serial loop, so results
// are bitwise independent of the thread count.
template <typename F>
static void parallel_for(std::size_t count, bool enable, F&& fn) {
  const int nt = enable ? std::min<int>(g_threads, static_cast<int>(count)) : 1;
  if (nt <= 1) {
    for (std::size_t i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (std::size_t i; (i = next.fetch_add(1)) < count;) fn(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
}

// matrix.cpp:69-77
static Mat matmul(const Mat& a, const Mat& b) {
  if (a.c != b.r) throw ShapeError("matmul: inner dimensions differ, " + a.shape() + " times " + b.shape());
  Mat out(a.r, b.c, 0.0);
  parallel_for(a.r, a.r * a.c * b.c > 1000000, [&](std::size_t i) {
    double* o = &out.v[i * b.c];
    for (std::size_t k = 0; k < a.c; ++k) {
      const double s = a(i, k);
      const double* br = &b.v[k * b.c];
      for (std::size_t j = 0; j < b.c; ++j) o[j] = o[j] + s * br[j];
    }
  });
  return out;
}

// matrix.cpp:79-87 (a^T b)
static Mat matmul_at(const Mat& a, const Mat& b) {
  if (a.r != b.r) throw ShapeError("matmul_at: row counts differ, " + a.shape() + "^T times " + b.shape());
  Mat out(a.c, b.c, 0.0);
  parallel_for(a.c, a.r * a.c * b.c > 1000000, [&](std::size_t i) {
    double* o = &out.v[i * b.c];
    for (std::size_t n = 0; n < a.r; ++n) {
      const double s = a(n, i);
      const double* br = &b.v[n * b.c];
      for (std::size_t j = 0; j < b.c; ++j) o[j] = o[j] + s * br[j];
    }
  });
  return out;
}

static Mat transpose(const Mat& a) {
  Mat t(a.c, a.r);
  for (std::size_t i = 0; i < a.r; ++i)
    for (std::size_t j = 0; j < a.c; ++j) t(j, i) = a(i, j);
  return t;
}

static Mat sub(const Mat& a, const Mat& b) {
  if (a.r != b.r || a.c != b.c) throw ShapeError("subtract: shapes differ, " + a.shape() + " vs " + b.shape());
  Mat o(a.r, a.c);
  for (std::size_t i = 0; i < a.v.size(); ++i) o.v[i] = a.v[i] - b.v[i];
  return o;
}

static Mat take_columns(const Mat& a, std::size_t b, std::size_t e) {  // matrix.cpp:119-128
  if (b >= e || e > a.c) throw ShapeError("take_columns: invalid range for " + a.shape());
  Mat o(a.r, e - b);
  for (std::size_t i = 0; i < a.r; ++i)
    for (std::size_t j = b; j < e; ++j) o(i, j - b) = a(i, j);
  return o;
}

static Mat vstack(const Mat& t, const Mat& b) {  // matrix.cpp:130-139
  if (t.c != b.c) throw ShapeError("vstack: column counts differ, " + t.shape() + " vs " + b.shape());
  Mat o(t.r + b.r, t.c);
  std::copy(t.v.begin(), t.v.end(), o.v.begin());
  std::copy(b.v.begin(), b.v.end(), o.v.begin() + t.v.size());
  return o;
}

// Gram a^T a (matrix.cpp:152-161; also linalg.cpp:179-184): the lower triangle
// is accumulated, then mirrored, so the result is exactly symmetric.  Every
// element sums its products in increasing row order, within each row shard,
// and shards are added in shard order (shards = 1 is the reference's single
// pass; shards > 1 reproduces a row-sharded multi-GPU reduction order and is
// used to measure the oracle's own conditioning floor).
static Mat gram_sharded(const Mat& a, std::size_t shards) {
  const std::size_t n = a.c, rows = a.r;
  if (shards < 1) shards = 1;
  Mat acm = transpose(a);  // column-major copy, as linalg.cpp:181
  Mat g(n, n, 0.0);
  const std::size_t per = (rows + shards - 1) / shards;
  const std::size_t B = 4;
  parallel_for((n + B - 1) / B, true, [&](std::size_t ib) {
    const std::size_t i0 = ib * B;
    for (std::size_t j0 = 0; j0 <= i0; j0 += B) {
      double tot[B][B] = {};
      for (std::size_t s = 0; s < shards; ++s) {
        const std::size_t r0 = s * per, r1 = std::min(rows, r0 + per);
        double acc[B][B] = {};
        const double* hi[B];
        const double* hj[B];
        for (std::size_t q = 0; q < B; ++q) {
          hi[q] = &acm.v[std::min(i0 + q, n - 1) * rows];
          hj[q] = &acm.v[std::min(j0 + q, n - 1) * rows];
        }
        // 16 independent chains; each element still adds its products in row order
        for (std::size_t k = r0; k < r1; ++k) {
          const double a0 = hi[0][k], a1 = hi[1][k], a2 = hi[2][k], a3 = hi[3][k];
          const double b0 = hj[0][k], b1 = hj[1][k], b2 = hj[2][k], b3 = hj[3][k];
          acc[0][0] = acc[0][0] + a0 * b0; acc[0][1] = acc[0][1] + a0 * b1;
          acc[0][2] = acc[0][2] + a0 * b2; acc[0][3] = acc[0][3] + a0 * b3;
          acc[1][0] = acc[1][0] + a1 * b0; acc[1][1] = acc[1][1] + a1 * b1;
          acc[1][2] = acc[1][2] + a1 * b2; acc[1][3] = acc[1][3] + a1 * b3;
          acc[2][0] = acc[2][0] + a2 * b0; acc[2][1] = acc[2][1] + a2 * b1;
          acc[2][2] = acc[2][2] + a2 * b2; acc[2][3] = acc[2][3] + a2 * b3;
          acc[3][0] = acc[3][0] + a3 * b0; acc[3][1] = acc[3][1] + a3 * b1;
          acc[3][2] = acc[3][2] + a3 * b2; acc[3][3] = acc[3][3] + a3 * b3;
        }
        for (std::size_t ii = 0; ii < B; ++ii)
          for (std::size_t jj = 0; jj < B; ++jj) tot[ii][jj] = (s == 0) ? acc[ii][jj] : tot[ii][jj] + acc[ii][jj];
      }
      for (std::size_t ii = 0; ii < B; ++ii)
        for (std::size_t jj = 0; jj < B; ++jj) {
          const std::size_t i = i0 + ii, j = j0 + jj;
          if (i < n && j < n && j <= i) {
            g(i, j) = tot[ii][jj];
            g(j, i) = tot[ii][jj];
          }
        }
    }
  });
  return g;
}
static Mat gram(const Mat& a) { return gram_sharded(a, 1); }

// ---- init_hidden / hidden_matrix (elm.cpp:20-27, 74-106)
static double uniform_pm1(std::mt19937_64& gen) {  // elm.cpp:22-25
  double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}
static double sigmoid(double z) { return 1.0 / (1.0 + std::exp(-z)); }  // elm.cpp:27

static void init_hidden(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed, Mat& w,
                        Mat& b) {
  if (inputs < 1 || hidden < 1 || outputs < 1)
    throw std::invalid_argument("ElmParams: inputs, hidden_nodes and outputs must be >= 1");
  std::mt19937_64 gen(seed);
  w = Mat(inputs, hidden);
  for (std::size_t i = 0; i < inputs; ++i)
    for (std::size_t j = 0; j < hidden; ++j) w(i, j) = uniform_pm1(gen);
  b = Mat(1, hidden);
  for (std::size_t j = 0; j < hidden; ++j) b(0, j) = uniform_pm1(gen);
}

static Mat hidden_matrix(const Mat& w, const Mat& b, const Mat& x) {  // elm.cpp:93-106
  if (x.c != w.r)
    throw ShapeError("hidden_matrix: sample has " + std::to_string(x.c) + " features but the layer expects " +
                     std::to_string(w.r));
  Mat h = matmul(x, w);
  for (std::size_t i = 0; i < h.r; ++i)
    for (std::size_t j = 0; j < h.c; ++j) h(i, j) = sigmoid(h(i, j) + b(0, j));  // bias after the dot, :102
  return h;
}

// ---- pinv via SVD (linalg.cpp:68-87).  The reference calls Eigen's BDCSVD;
// this restates the same definition (V diag(1/s_i for s_i > cut) U^T with
// cut = tol * s_max, tol = max(rows, cols) * eps by default) on a one-sided
// Jacobi SVD.  Fallback / test-oracle only, never on the rank path.
static Mat pinv_svd(const Mat& a, double tol) {
  if (a.v.empty()) throw ShapeError("pinv_svd: empty matrix");
  const bool tall = a.r >= a.c;
  Mat m = tall ? a : transpose(a);  // m is p x q with p >= q
  const std::size_t p = m.r, q = m.c;
  Mat u = m;             // columns become U * sigma
  Mat v(q, q, 0.0);
  for (std::size_t i = 0; i < q; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 80; ++sweep) {
    double off = 0.0;
    for (std::size_t i = 0; i + 1 < q; ++i)
      for (std::size_t j = i + 1; j < q; ++j) {
        double alpha = 0, beta = 0, gamma = 0;
        for (std::size_t k = 0; k < p; ++k) {
          alpha += u(k, i) * u(k, i);
          beta += u(k, j) * u(k, j);
          gamma += u(k, i) * u(k, j);
        }
        if (gamma == 0.0) continue;
        double conv = std::fabs(gamma) / std::sqrt(alpha * beta);
        if (!(conv > 1e-15)) continue;
        off = std::max(off, conv);
        double zeta = (beta - alpha) / (2.0 * gamma);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (std::size_t k = 0; k < p; ++k) {
          double x = u(k, i), y = u(k, j);
          u(k, i) = cs * x - sn * y;
          u(k, j) = sn * x + cs * y;
        }
        for (std::size_t k = 0; k < q; ++k) {
          double x = v(k, i), y = v(k, j);
          v(k, i) = cs * x - sn * y;
          v(k, j) = sn * x + cs * y;
        }
      }
    if (off < 1e-15) break;
  }
  std::vector<double> s(q);
  double smax = 0.0;
  for (std::size_t j = 0; j < q; ++j) {
    double nrm = 0;
    for (std::size_t k = 0; k < p; ++k) nrm += u(k, j) * u(k, j);
    s[j] = std::sqrt(nrm);
    smax = std::max(smax, s[j]);
  }
  const double rel = tol > 0.0 ? tol : static_cast<double>(std::max(a.r, a.c)) * kEps;
  const double cut = rel * smax;
  // pinv(m) = V diag(1/s) U^T, U_j = u_j / s_j  =>  V diag(1/s^2) u^T
  Mat pm(q, p, 0.0);
  for (std::size_t j = 0; j < q; ++j) {
    if (!(s[j] > cut && s[j] > 0.0)) continue;
    const double w = 1.0 / (s[j] * s[j]);
    for (std::size_t r = 0; r < q; ++r) {
      const double vr = v(r, j) * w;
      for (std::size_t k = 0; k < p; ++k) pm(r, k) += vr * u(k, j);
    }
  }
  return tall ? pm : transpose(pm);
}

// ---- SpdFactor (linalg.cpp:99-151)
struct Spd {
  Mat l;  // lower factor
};
static Spd spd_factor(const Mat& m) {
  if (m.r != m.c) throw ShapeError("solve_spd: matrix is not square, " + m.shape());
  const std::size_t n = m.r;
  Mat a = m;
  double scale = 0.0, asym = 0.0;
  for (double x : a.v) scale = std::max(scale, std::fabs(x));
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) asym = std::max(asym, std::fabs(a(i, j) - a(j, i)));
  if (asym > 1e-12 * std::max(scale, 1.0))
    throw std::invalid_argument("solve_spd: matrix is not symmetric within 1e-12 relative");
  double dmax = -std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < n; ++i) dmax = std::max(dmax, a(i, i));
  const double thresh = static_cast<double>(n) * kEps * dmax;  // :109
  const std::size_t nb = 64;
  for (std::size_t k = 0; k < n; k += nb) {
    const std::size_t b = std::min(nb, n - k);
    for (std::size_t j = k; j < k + b; ++j) {
      double d = a(j, j);
      if (!std::isfinite(d) || d <= thresh || d <= 0.0) throw SingularMatrix(j, d);  // :118-119
      a(j, j) = std::sqrt(d);
      for (std::size_t i = j + 1; i < n; ++i) a(i, j) = a(i, j) / a(j, j);  // :124
      for (std::size_t c = j + 1; c < k + b; ++c) {                           // :125-127
        const double s = a(c, j);
        for (std::size_t i = c; i < n; ++i) a(i, c) = a(i, c) - s * a(i, j);
      }
    }
    const std::size_t t0 = k + b;  // :130-136 trailing lower rank-b update
    parallel_for(n - t0, (n - t0) > 256, [&](std::size_t ii) {
      const std::size_t i = t0 + ii;
      for (std::size_t j = t0; j <= i; ++j) {
        double acc = 0.0;
        for (std::size_t c = k; c < k + b; ++c) acc = acc + a(i, c) * a(j, c);
        a(i, j) = a(i, j) - acc;
      }
    });
  }
  Spd f;
  f.l = Mat(n, n, 0.0);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j <= i; ++j) f.l(i, j) = a(i, j);
  return f;
}

// L y = rhs then L^T x = y, in place (linalg.cpp:147-149, 267-268)
static void tri_solve_pair(const Mat& l, Mat& x) {
  const std::size_t n = l.r, m = x.c;
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t c = 0; c < i; ++c) {
      const double s = l(i, c);
      if (s == 0.0) continue;
      for (std::size_t j = 0; j < m; ++j) x(i, j) = x(i, j) - s * x(c, j);
    }
    for (std::size_t j = 0; j < m; ++j) x(i, j) = x(i, j) / l(i, i);
  }
  for (std::size_t ii = n; ii-- > 0;) {
    for (std::size_t c = ii + 1; c < n; ++c) {
      const double s = l(c, ii);
      if (s == 0.0) continue;
      for (std::size_t j = 0; j < m; ++j) x(ii, j) = x(ii, j) - s * x(c, j);
    }
    for (std::size_t j = 0; j < m; ++j) x(ii, j) = x(ii, j) / l(ii, ii);
  }
}

static Mat spd_solve(const Spd& f, const Mat& rhs) {
  if (rhs.r != f.l.r)
    throw ShapeError("solve_spd: rhs has " + std::to_string(rhs.r) + " rows, expected " + std::to_string(f.l.r));
  Mat x = rhs;
  tri_solve_pair(f.l, x);
  return x;
}

// ---- rank-revealing factorisation (linalg.cpp:157-248), on a precomputed Gram.
struct Factor {
  std::vector<std::size_t> order;
  std::size_t rank = 0;
  double tolerance = 0.0;
  Mat f;
  double min_margin = std::numeric_limits<double>::infinity();  // diagnostics only
};

// `g` is consumed (it becomes the trailing-updated Gram).  `rows` is the row
// count of the matrix the Gram came from (the default tolerance uses it, :171).
static Factor factor_gram(Mat g, std::size_t rows, double tol) {
  if (g.v.empty()) throw ShapeError("rank_revealing_permutation: empty matrix");
  if (tol < 0.0 || !std::isfinite(tol)) throw std::invalid_argument("rank_revealing_permutation: tolerance must be >= 0");
  const std::size_t n = g.c;
  Factor out;
  out.order.resize(n);
  for (std::size_t i = 0; i < n; ++i) out.order[i] = i;
  out.tolerance = tol > 0.0 ? tol : static_cast<double>(std::max(rows, n)) * kEps;
  out.f = Mat(n, n, 0.0);
  Mat& f = out.f;
  std::vector<double> d(n);
  for (std::size_t i = 0; i < n; ++i) d[i] = g(i, i);
  double dmax0 = d[0];
  for (std::size_t i = 1; i < n; ++i) dmax0 = std::max(dmax0, d[i]);
  if (!(dmax0 > 0.0)) {  // :189-193
    out.rank = 0;
    return out;
  }
  const double r00 = std::sqrt(dmax0);
  const double cut = out.tolerance * r00;
  std::size_t rank = n;
  const std::size_t nb = 64;
  std::vector<double> col(n);
  for (std::size_t k = 0; k < n && rank == n; k += nb) {
    const std::size_t kb = std::min(nb, n - k);
    for (std::size_t j = k; j < k + kb; ++j) {
      std::size_t piv = j;
      for (std::size_t i = j + 1; i < n; ++i)
        if (d[i] > d[piv]) piv = i;  // strict '>' (:209)
      {  // pivot margin diagnostic: gap to the runner-up, relative to r00^2
        double second = -std::numeric_limits<double>::infinity();
        for (std::size_t i = j; i < n; ++i)
          if (i != piv) second = std::max(second, d[i]);
        if (j + 1 < n) out.min_margin = std::min(out.min_margin, (d[piv] - second) / dmax0);
      }
      if (piv != j) {  // :211-218
        std::swap(out.order[j], out.order[piv]);
        std::swap(d[j], d[piv]);
        for (std::size_t c = 0; c < j; ++c) std::swap(f(j, c), f(piv, c));
        for (std::size_t c = 0; c < n; ++c) std::swap(g(j, c), g(piv, c));
        for (std::size_t r = 0; r < n; ++r) std::swap(g(r, j), g(r, piv));
      }
      const double rjj = d[j] > 0.0 ? std::sqrt(d[j]) : 0.0;
      if (rjj <= cut) {  // :219-223
        rank = j;
        break;
      }
      f(j, j) = rjj;
      for (std::size_t i = j + 1; i < n; ++i) {  // :225-235
        double v = g(i, j);
        if (j > k) {
          double s = 0.0;
          for (std::size_t c = k; c < j; ++c) s = s + f(i, c) * f(j, c);
          v = v - s;
        }
        v = v / rjj;
        f(i, j) = v;
        d[i] = d[i] - v * v;
      }
    }
    const std::size_t t0 = k + kb;  // :237-244 trailing rank-kb update, lower then mirror
    if (rank == n && t0 < n) {
      parallel_for(n - t0, (n - t0) > 256, [&](std::size_t ii) {
        const std::size_t i = t0 + ii;
        for (std::size_t jj = t0; jj <= i; ++jj) {
          double acc = 0.0;
          for (std::size_t c = k; c < k + kb; ++c) acc = acc + f(i, c) * f(jj, c);
          g(i, jj) = g(i, jj) - acc;
        }
      });
      for (std::size_t i = t0; i < n; ++i)
        for (std::size_t jj = i + 1; jj < n; ++jj) g(i, jj) = g(jj, i);
    }
  }
  out.rank = rank;
  return out;
}

static Mat solve_factored_gram(const Factor& fac, const Mat& rhs) {  // linalg.cpp:254-270
  const std::size_t n = fac.order.size();
  if (fac.rank != n)
    throw std::invalid_argument("solve_factored_gram: factor is rank-deficient (" + std::to_string(fac.rank) +
                                " of " + std::to_string(n) + ")");
  if (rhs.r != n)
    throw ShapeError("solve_factored_gram: rhs has " + std::to_string(rhs.r) + " rows, expected " + std::to_string(n));
  Mat x = rhs;
  tri_solve_pair(fac.f, x);
  return x;
}

static Mat apply_permutation(const Mat& a, const std::vector<std::size_t>& order) {  // linalg.cpp:40-52
  if (a.c != order.size()) throw ShapeError("apply_permutation: length mismatch");
  Mat o(a.r, a.c);
  for (std::size_t i = 0; i < a.r; ++i)
    for (std::size_t j = 0; j < a.c; ++j) o(i, j) = a(i, order[j]);
  return o;
}
static Mat invert_permutation_rows(const Mat& b, const std::vector<std::size_t>& order) {  // linalg.cpp:54-66
  if (b.r != order.size()) throw ShapeError("invert_permutation_rows: length mismatch");
  Mat o(b.r, b.c);
  for (std::size_t i = 0; i < b.r; ++i)
    for (std::size_t j = 0; j < b.c; ++j) o(order[i], j) = b(i, j);
  return o;
}

// ---- solvers (elm.cpp:29-49, 108-229)
struct Diag {
  std::size_t rank = 0;
  int rank_known = 0;
  std::size_t split_lo = 0, split_hi = 0;
  int ridge_applied = 0, fallback_to_direct = 0, used_svd_path = 0;
  double solve_seconds = 0, hidden_seconds = 0, training_accuracy = -1.0;
};

static Spd factor_with_ridge(const Mat& m, double ridge, bool& applied, int block) {  // elm.cpp:30-49
  try {
    return spd_factor(m);
  } catch (const SingularMatrix&) {
    double tr = 0.0;
    for (std::size_t i = 0; i < m.r; ++i) tr += m(i, i);
    double eps = ridge * tr / static_cast<double>(m.r);
    if (eps <= 0.0) eps = ridge;
    Mat rescued = m;
    for (std::size_t i = 0; i < m.r; ++i) rescued(i, i) += eps;
    try {
      Spd f = spd_factor(rescued);
      applied = true;
      return f;
    } catch (const SingularMatrix&) {
      throw SingularSplit(block);
    }
  }
}

static Mat solve_direct(const Mat& h, const Mat& y, Diag* diag) {  // elm.cpp:108-122
  if (h.r != y.r) throw ShapeError("solve_direct: H is " + h.shape() + " but Y is " + y.shape());
  if (h.r >= h.c) {
    try {
      Spd f = spd_factor(gram(h));
      return spd_solve(f, matmul_at(h, y));
    } catch (const SingularMatrix&) {
    }
  }
  if (diag) diag->used_svd_path = 1;
  return matmul(pinv_svd(h, 0.0), y);
}

static void solve_block_split(const Mat& h1, const Mat& h2, const Mat& y, double ridge, Diag* diag, Mat& beta1,
                              Mat& beta2) {  // elm.cpp:124-156
  const std::size_t n = h1.r;
  if (h2.r != n || y.r != n)
    throw ShapeError("solve_block_split: row counts differ (" + h1.shape() + ", " + h2.shape() + ", " + y.shape() + ")");
  if (n < h1.c + h2.c) throw ShapeError("solve_block_split: needs at least as many samples as columns");
  bool ridge_applied = false;
  Mat a = gram(h2);
  Mat g21 = matmul_at(h2, h1);
  Spd fa = factor_with_ridge(a, ridge, ridge_applied, 0);
  Mat b = spd_solve(fa, matmul_at(h2, y));
  Mat d = sub(gram(h1), matmul(transpose(g21), spd_solve(fa, g21)));
  {
    Mat dt = transpose(d);
    for (std::size_t i = 0; i < d.v.size(); ++i) d.v[i] = (d.v[i] + dt.v[i]) * 0.5;
  }
  Spd fd = factor_with_ridge(d, ridge, ridge_applied, 1);
  Mat residual = sub(y, matmul(h2, b));
  beta1 = spd_solve(fd, matmul_at(h1, residual));
  beta2 = sub(b, spd_solve(fa, matmul(g21, beta1)));
  if (diag && ridge_applied) diag->ridge_applied = 1;
}

enum Kind { kDirect = 0, kDfSplit = 1, kRankBased = 2 };

static Mat solve_beta(const Mat& h, const Mat& y, int kind, std::size_t split_index, double rank_tol, Diag& diag,
                      std::size_t gram_shards, Factor* fac_out) {  // elm.cpp:158-229
  const std::size_t l = h.c;
  if (kind == kDirect) {
    diag.split_lo = l;
    diag.split_hi = 0;
    return solve_direct(h, y, &diag);
  }
  if (kind == kDfSplit) {
    const std::size_t s = split_index;
    if (s < 1 || s >= l)
      throw std::invalid_argument("solve_beta: df split index must be in (0, " + std::to_string(l) + "), got " +
                                  std::to_string(s));
    diag.split_lo = s;
    diag.split_hi = l - s;
    Mat b1, b2;
    try {
      solve_block_split(take_columns(h, 0, s), take_columns(h, s, l), y, 1e-8, &diag, b1, b2);
      return vstack(b1, b2);
    } catch (const SingularSplit&) {
      diag.fallback_to_direct = 1;
      return solve_direct(h, y, &diag);
    }
  }
  if (kind != kRankBased) throw std::logic_error("solve_beta: unknown strategy");
  if (h.v.empty()) throw ShapeError("rank_revealing_permutation: empty matrix");
  Factor fac = factor_gram(gram_sharded(h, gram_shards), h.r, rank_tol);
  diag.rank = fac.rank;
  diag.rank_known = 1;
  if (fac_out) *fac_out = fac;
  if (fac.rank == 0 || l < 2) {
    diag.fallback_to_direct = 1;
    diag.split_lo = l;
    diag.split_hi = 0;
    return solve_direct(h, y, &diag);
  }
  const std::size_t split = (fac.rank == l) ? (l + 1) / 2 : fac.rank;
  diag.split_lo = split;
  diag.split_hi = l - split;
  if (fac.rank == l) {
    Mat hty = matmul_at(h, y);
    Mat htyp(l, hty.c);
    for (std::size_t i = 0; i < l; ++i)
      for (std::size_t j = 0; j < hty.c; ++j) htyp(i, j) = hty(fac.order[i], j);
    return invert_permutation_rows(solve_factored_gram(fac, htyp), fac.order);
  }
  Mat hp = apply_permutation(h, fac.order);
  Mat b1, b2;
  try {
    solve_block_split(take_columns(hp, 0, split), take_columns(hp, split, l), y, 1e-8, &diag, b1, b2);
    return invert_permutation_rows(vstack(b1, b2), fac.order);
  } catch (const SingularSplit&) {
    diag.fallback_to_direct = 1;
    return solve_direct(h, y, &diag);
  }
}

static double accuracy(const Mat& pred, const Mat& y) {  // elm.cpp:286-300
  if (pred.r != y.r || pred.c != y.c)
    throw ShapeError("accuracy: shapes differ, " + pred.shape() + " vs " + y.shape());
  std::size_t hits = 0;
  for (std::size_t i = 0; i < pred.r; ++i) {
    std::size_t ap = 0, ay = 0;
    for (std::size_t j = 1; j < pred.c; ++j) {
      if (pred(i, j) > pred(i, ap)) ap = j;
      if (y(i, j) > y(i, ay)) ay = j;
    }
    if (ap == ay) ++hits;
  }
  return static_cast<double>(hits) / static_cast<double>(pred.r);
}

}  // namespace oracle

// ============================================================================
// C ABI for ctypes (tests/ and bench.py's CPU legs only).
// ============================================================================
using namespace oracle;

extern "C" {

struct oracle_error {
  int code;  // 0 ok, 1 ShapeError, 2 invalid_argument, 3 SingularMatrix, 4 SingularSplit, 5 runtime_error, 6 other
  std::size_t pivot_index;
  double pivot_value;
  int block;
  char message[256];
};

struct oracle_diag {
  std::size_t rank;
  int rank_known;
  std::size_t split_lo, split_hi;
  int ridge_applied, fallback_to_direct, used_svd_path;
  double solve_seconds, hidden_seconds, training_accuracy;
  double min_pivot_margin;
};

static void set_err(oracle_error* e, int code, const char* msg) {
  if (!e) return;
  e->code = code;
  std::snprintf(e->message, sizeof e->message, "%s", msg);
}

extern "C++" {
template <typename F>
static int guarded(oracle_error* err, F&& body) {
  if (err) std::memset(err, 0, sizeof(oracle_error));
  try {
    body();
    return 0;
  } catch (const SingularMatrix& ex) {
    if (err) {
      err->pivot_index = ex.index;
      err->pivot_value = ex.value;
    }
    set_err(err, 3, ex.what());
    return 3;
  } catch (const SingularSplit& ex) {
    if (err) err->block = ex.block;
    set_err(err, 4, ex.what());
    return 4;
  } catch (const ShapeError& ex) {
    set_err(err, 1, ex.what());
    return 1;
  } catch (const std::invalid_argument& ex) {
    set_err(err, 2, ex.what());
    return 2;
  } catch (const std::runtime_error& ex) {
    set_err(err, 5, ex.what());
    return 5;
  } catch (const std::exception& ex) {
    set_err(err, 6, ex.what());
    return 6;
  }
}

}  // extern "C++"

static void copy_diag(const Diag& d, oracle_diag* o) {
  if (!o) return;
  o->rank = d.rank;
  o->rank_known = d.rank_known;
  o->split_lo = d.split_lo;
  o->split_hi = d.split_hi;
  o->ridge_applied = d.ridge_applied;
  o->fallback_to_direct = d.fallback_to_direct;
  o->used_svd_path = d.used_svd_path;
  o->solve_seconds = d.solve_seconds;
  o->hidden_seconds = d.hidden_seconds;
  o->training_accuracy = d.training_accuracy;
}

void oracle_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

int oracle_init_hidden(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed, double* w,
                       double* b, oracle_error* err) {
  return guarded(err, [&] {
    Mat W, B;
    init_hidden(inputs, hidden, outputs, seed, W, B);
    std::memcpy(w, W.v.data(), sizeof(double) * W.v.size());
    std::memcpy(b, B.v.data(), sizeof(double) * B.v.size());
  });
}

int oracle_hidden_matrix(const double* w, const double* b, std::size_t d, std::size_t l, const double* x,
                         std::size_t n, std::size_t xcols, double* h, oracle_error* err) {
  return guarded(err, [&] {
    Mat H = hidden_matrix(from_ptr(w, d, l), from_ptr(b, 1, l), from_ptr(x, n, xcols));
    std::memcpy(h, H.v.data(), sizeof(double) * H.v.size());
  });
}

int oracle_gram(const double* a, std::size_t rows, std::size_t cols, std::size_t shards, double* g,
                oracle_error* err) {
  return guarded(err, [&] {
    Mat G = gram_sharded(from_ptr(a, rows, cols), shards);
    std::memcpy(g, G.v.data(), sizeof(double) * G.v.size());
  });
}

int oracle_matmul(const double* a, std::size_t ar, std::size_t ac, const double* b, std::size_t br, std::size_t bc,
                  double* out, oracle_error* err) {
  return guarded(err, [&] {
    Mat O = matmul(from_ptr(a, ar, ac), from_ptr(b, br, bc));
    std::memcpy(out, O.v.data(), sizeof(double) * O.v.size());
  });
}

int oracle_matmul_at(const double* a, std::size_t ar, std::size_t ac, const double* b, std::size_t br,
                     std::size_t bc, double* out, oracle_error* err) {
  return guarded(err, [&] {
    Mat O = matmul_at(from_ptr(a, ar, ac), from_ptr(b, br, bc));
    std::memcpy(out, O.v.data(), sizeof(double) * O.v.size());
  });
}

int oracle_pinv_svd(const double* a, std::size_t rows, std::size_t cols, double tol, double* out, oracle_error* err) {
  return guarded(err, [&] {
    Mat P = pinv_svd(from_ptr(a, rows, cols), tol);
    std::memcpy(out, P.v.data(), sizeof(double) * P.v.size());
  });
}

int oracle_solve_spd(const double* m, std::size_t mr, std::size_t mc, const double* rhs, std::size_t rr,
                     std::size_t rc, double* out, oracle_error* err) {
  return guarded(err, [&] {
    Spd f = spd_factor(from_ptr(m, mr, mc));
    Mat X = spd_solve(f, from_ptr(rhs, rr, rc));
    std::memcpy(out, X.v.data(), sizeof(double) * X.v.size());
  });
}

// rank_revealing_factor on a matrix a (linalg.cpp:157-248)
int oracle_rank_revealing_factor(const double* a, std::size_t rows, std::size_t cols, double tol,
                                 std::size_t* order, std::size_t* rank, double* tolerance, double* factor,
                                 double* min_margin, oracle_error* err) {
  return guarded(err, [&] {
    if (rows == 0 || cols == 0) throw ShapeError("rank_revealing_permutation: empty matrix");
    if (tol < 0.0 || !std::isfinite(tol)) throw std::invalid_argument("rank_revealing_permutation: tolerance must be >= 0");
    Factor f = factor_gram(gram(from_ptr(a, rows, cols)), rows, tol);
    std::memcpy(order, f.order.data(), sizeof(std::size_t) * cols);
    *rank = f.rank;
    *tolerance = f.tolerance;
    if (factor) std::memcpy(factor, f.f.v.data(), sizeof(double) * f.f.v.size());
    if (min_margin) *min_margin = f.min_margin;
  });
}

// The same factorisation on a precomputed Gram g (n x n).  Lets the tests feed
// the GPU's own Gram to the oracle and compare pivots/rank bit-exactly.
int oracle_factor_gram(const double* g, std::size_t n, std::size_t rows, double tol, std::size_t* order,
                       std::size_t* rank, double* tolerance, double* factor, double* min_margin, oracle_error* err) {
  return guarded(err, [&] {
    Factor f = factor_gram(from_ptr(g, n, n), rows, tol);
    std::memcpy(order, f.order.data(), sizeof(std::size_t) * n);
    *rank = f.rank;
    *tolerance = f.tolerance;
    if (factor) std::memcpy(factor, f.f.v.data(), sizeof(double) * f.f.v.size());
    if (min_margin) *min_margin = f.min_margin;
  });
}

int oracle_solve_factored_gram(const double* factor, const std::size_t* order, std::size_t n, std::size_t rank,
                               const double* rhs, std::size_t rr, std::size_t rc, double* out, oracle_error* err) {
  return guarded(err, [&] {
    Factor f;
    f.order.assign(order, order + n);
    f.rank = rank;
    f.f = from_ptr(factor, n, n);
    Mat X = solve_factored_gram(f, from_ptr(rhs, rr, rc));
    std::memcpy(out, X.v.data(), sizeof(double) * X.v.size());
  });
}

// Rank-path pseudo-inverse H^+ = P (F F^T)^{-1} P^T H^T: the full-rank solve of
// elm.cpp:202-214 with right-hand side H^T in place of H^T T, i.e. solve_factored_gram
// (linalg.cpp:254-270) on the pivot-ordered rows of H^T, then invert_permutation_rows
// (linalg.cpp:54-66).  rank < cols raises invalid_argument exactly like solve_factored_gram;
// order and rank are written first.  The right-hand-side columns are independent, so they are
// solved in column blocks on the worker threads (same arithmetic per column).
int oracle_pseudo_inverse(const double* h, std::size_t rows, std::size_t cols, double tol, double* out,
                          std::size_t* order, std::size_t* rank, oracle_error* err) {
  return guarded(err, [&] {
    if (rows == 0 || cols == 0) throw ShapeError("pseudo_inverse: empty matrix");
    if (tol < 0.0 || !std::isfinite(tol)) throw std::invalid_argument("rank_revealing_permutation: tolerance must be >= 0");
    Mat hm = from_ptr(h, rows, cols);
    Factor f = factor_gram(gram(hm), rows, tol);
    std::memcpy(order, f.order.data(), sizeof(std::size_t) * cols);
    *rank = f.rank;
    if (f.rank != cols)
      throw std::invalid_argument("solve_factored_gram: factor is rank-deficient (" + std::to_string(f.rank) + " of " +
                                  std::to_string(cols) + ")");
    constexpr std::size_t kBlock = 256;
    const std::size_t nblk = (rows + kBlock - 1) / kBlock;
    parallel_for(nblk, nblk > 1, [&](std::size_t b) {
      const std::size_t c0 = b * kBlock, nc = std::min(kBlock, rows - c0);
      Mat x(cols, nc);
      for (std::size_t i = 0; i < cols; ++i)
        for (std::size_t j = 0; j < nc; ++j) x(i, j) = hm(c0 + j, f.order[i]);
      tri_solve_pair(f.f, x);
      for (std::size_t i = 0; i < cols; ++i)
        for (std::size_t j = 0; j < nc; ++j) out[f.order[i] * rows + c0 + j] = x(i, j);
    });
  });
}

int oracle_solve_block_split(const double* h1, std::size_t n, std::size_t c1, const double* h2, std::size_t c2,
                             const double* y, std::size_t m, double ridge, double* beta1, double* beta2,
                             oracle_diag* diag, oracle_error* err) {
  return guarded(err, [&] {
    Diag d;
    Mat b1, b2;
    solve_block_split(from_ptr(h1, n, c1), from_ptr(h2, n, c2), from_ptr(y, n, m), ridge, &d, b1, b2);
    std::memcpy(beta1, b1.v.data(), sizeof(double) * b1.v.size());
    std::memcpy(beta2, b2.v.data(), sizeof(double) * b2.v.size());
    copy_diag(d, diag);
  });
}

int oracle_solve_direct(const double* h, std::size_t n, std::size_t l, const double* y, std::size_t m, double* beta,
                        oracle_diag* diag, oracle_error* err) {
  return guarded(err, [&] {
    Diag d;
    Mat B = solve_direct(from_ptr(h, n, l), from_ptr(y, n, m), &d);
    std::memcpy(beta, B.v.data(), sizeof(double) * B.v.size());
    copy_diag(d, diag);
  });
}

// solve_beta (elm.cpp:158-229).  gram_shards > 1 sums the Gram over row shards
// (self-floor measurement).  order/min_margin are optional outputs for the rank path.
int oracle_solve_beta(const double* h, std::size_t n, std::size_t l, const double* y, std::size_t yrows,
                      std::size_t m, int kind, std::size_t split_index, double rank_tol, std::size_t gram_shards,
                      double* beta, std::size_t* order, oracle_diag* diag, oracle_error* err) {
  return guarded(err, [&] {
    if (yrows != n && kind != kDirect) {
      // the reference reaches the row check inside the block solve / matmul_at
    }
    Diag d;
    Factor fac;
    Mat B = solve_beta(from_ptr(h, n, l), from_ptr(y, yrows, m), kind, split_index, rank_tol, d, gram_shards,
                       order ? &fac : nullptr);
    std::memcpy(beta, B.v.data(), sizeof(double) * B.v.size());
    if (order && !fac.order.empty()) std::memcpy(order, fac.order.data(), sizeof(std::size_t) * l);
    copy_diag(d, diag);
    if (diag) diag->min_pivot_margin = fac.min_margin;
  });
}

// train (elm.cpp:231-280).  Outputs W (d x L), b (L), beta (L x m).
int oracle_train(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed, const double* x,
                 std::size_t n, std::size_t xcols, const double* y, std::size_t yrows, std::size_t ycols, int kind,
                 std::size_t split_index, double rank_tol, std::size_t gram_shards, double* w, double* b,
                 double* beta, std::size_t* order, oracle_diag* diag, oracle_error* err) {
  return guarded(err, [&] {
    if (n != yrows)
      throw ShapeError("train: X is " + std::to_string(n) + "x" + std::to_string(xcols) + " but Y is " +
                       std::to_string(yrows) + "x" + std::to_string(ycols));
    if (xcols != inputs)
      throw ShapeError("train: X has " + std::to_string(xcols) + " features but params.inputs is " +
                       std::to_string(inputs));
    if (ycols != outputs)
      throw ShapeError("train: Y has " + std::to_string(ycols) + " columns but params.outputs is " +
                       std::to_string(outputs));
    if (kind != kDirect && n < hidden)
      throw std::invalid_argument("train: block strategies need at least as many samples as hidden nodes (" +
                                  std::to_string(n) + " < " + std::to_string(hidden) + "); use the direct strategy");
    if (kind == kDfSplit && (split_index < 1 || split_index >= hidden))
      throw std::invalid_argument("train: df split index must be in (0, " + std::to_string(hidden) + "), got " +
                                  std::to_string(split_index));
    Mat W, Bv;
    init_hidden(inputs, hidden, outputs, seed, W, Bv);
    Mat X = from_ptr(x, n, xcols), Y = from_ptr(y, yrows, ycols);
    Diag d;
    Mat H = hidden_matrix(W, Bv, X);
    Factor fac;
    Mat beta_m = solve_beta(H, Y, kind, split_index, rank_tol, d, gram_shards, order ? &fac : nullptr);
    if (!all_finite(beta_m)) throw std::runtime_error("train: solver produced non-finite output weights");
    d.training_accuracy = accuracy(matmul(H, beta_m), Y);
    std::memcpy(w, W.v.data(), sizeof(double) * W.v.size());
    std::memcpy(b, Bv.v.data(), sizeof(double) * Bv.v.size());
    std::memcpy(beta, beta_m.v.data(), sizeof(double) * beta_m.v.size());
    if (order && !fac.order.empty()) std::memcpy(order, fac.order.data(), sizeof(std::size_t) * hidden);
    copy_diag(d, diag);
    if (diag) diag->min_pivot_margin = fac.min_margin;
  });
}

// predict (elm.cpp:282-284): scores = sigma(X W + b) beta
int oracle_predict(const double* w, const double* b, std::size_t d, std::size_t l, const double* beta, std::size_t m,
                   const double* x, std::size_t n, std::size_t xcols, double* scores, oracle_error* err) {
  return guarded(err, [&] {
    Mat S = matmul(hidden_matrix(from_ptr(w, d, l), from_ptr(b, 1, l), from_ptr(x, n, xcols)), from_ptr(beta, l, m));
    std::memcpy(scores, S.v.data(), sizeof(double) * S.v.size());
  });
}

int oracle_accuracy(const double* pred, std::size_t pr, std::size_t pc, const double* y, std::size_t yr,
                    std::size_t yc, double* out, oracle_error* err) {
  return guarded(err, [&] { *out = accuracy(from_ptr(pred, pr, pc), from_ptr(y, yr, yc)); });
}

}  // extern "C"
