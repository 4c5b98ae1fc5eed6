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
// which is not installed in this image or on the GPU box, so the reference's
// own build cannot run here.  Every function below cites
// the reference file:line it follows.
//
// Pinning: PINNED AGAINST THE REFERENCE'S OWN CODE.  oracle/_ref/librbpelm_ref.so
// is proj/src/{matrix,linalg,elm}.cpp compiled unedited against a stand-in for
// the Eigen subset they use (oracle/eigen_standin; `make reflib`), and
// tests/test_oracle_vs_reference.py checks this restatement against it bit for
// bit (C1, C2 at full size, rank-deficient twins, df splits, ties, SPD solves,
// error messages).  Golden vectors written by that library
// (tests/golden/reference_golden.json) are checked on CPU and on the B200.
// The reference's known-answer and tolerance tests are also ported
// (tests/test_reference_suite.py), and the blocked/threaded loops are pinned
// bitwise against the scalar-loop transcription (tests/golden/oracle_digests.json).
// Not pinned: the rounding of real Eigen's blocked kernels (no Eigen build exists).
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
#include <chrono>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include <emmintrin.h>

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

// Persistent worker pool behind parallel_for (thread start-up per call would dominate the many
// short parallel loops of the blocked Gram and factorisation).
class Pool {
 public:
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // fn() on `nt` threads (the caller included); returns when all have finished
  void run(int nt, const std::function<void()>& fn) {
    std::lock_guard<std::mutex> run_lk(run_mu_);
    while (static_cast<int>(th_.size()) < nt - 1) {
      const int idx = static_cast<int>(th_.size());
      th_.emplace_back([this, idx] { worker(idx); });
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      want_ = nt - 1;
      pending_ = nt - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void worker(int idx) {
    std::size_t seen = 0;
    for (;;) {
      const std::function<void()>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        if (idx >= want_) continue;
        job = job_;
      }
      (*job)();
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void()>* job_ = nullptr;
  std::size_t gen_ = 0;
  int want_ = 0, pending_ = 0;
  bool stop_ = false;
};
static Pool& pool() {
  static Pool p;
  return p;
}

// Dynamic-schedule parallel loop over [0, count).  Each index is processed by
// exactly one thread with the same arithmetic as the serial loop, so results
// are bitwise independent of the thread count.
static thread_local bool t_in_parallel = false;  // nested loops run serially on their thread
template <typename F>
static void parallel_for(std::size_t count, bool enable, F&& fn) {
  const int nt = (enable && !t_in_parallel) ? std::min<int>(g_threads, static_cast<int>(count)) : 1;
  if (nt <= 1) {
    for (std::size_t i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<std::size_t> next{0};
  const std::function<void()> worker = [&] {
    t_in_parallel = true;
    for (std::size_t i; (i = next.fetch_add(1)) < count;) fn(i);
    t_in_parallel = false;
  };
  pool().run(nt, worker);
}

// 4 x 4 block of products over k in increasing order: acc[a][b] = acc[a][b] + A[k][a] * B[k][b]
// with A, B packed as [k][4].  SSE2 (baseline x86-64) multiplies and adds are the separately
// rounded IEEE operations of the scalar loop, so every element equals the scalar sum bitwise.
static inline void mk44(const double* A4, const double* B4, std::size_t K, __m128d acc[4][2]) {
  for (std::size_t k = 0; k < K; ++k) {
    const __m128d b01 = _mm_loadu_pd(B4 + 4 * k), b23 = _mm_loadu_pd(B4 + 4 * k + 2);
    for (int a = 0; a < 4; ++a) {
      const __m128d av = _mm_set1_pd(A4[4 * k + a]);
      acc[a][0] = _mm_add_pd(acc[a][0], _mm_mul_pd(av, b01));
      acc[a][1] = _mm_add_pd(acc[a][1], _mm_mul_pd(av, b23));
    }
  }
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

// matrix.cpp:79-87 (a^T b).  Each output element sums a(n, i) * b(n, j) over n in increasing
// order; output rows go in blocks of 8 so that a row of `a` is read one cache line at a time.
static Mat matmul_at(const Mat& a, const Mat& b) {
  if (a.r != b.r) throw ShapeError("matmul_at: row counts differ, " + a.shape() + "^T times " + b.shape());
  Mat out(a.c, b.c, 0.0);
  constexpr std::size_t kI = 8;
  parallel_for((a.c + kI - 1) / kI, a.r * a.c * b.c > 1000000, [&](std::size_t ib) {
    const std::size_t i0 = ib * kI, i1 = std::min(a.c, i0 + kI);
    for (std::size_t n = 0; n < a.r; ++n) {
      const double* br = &b.v[n * b.c];
      for (std::size_t i = i0; i < i1; ++i) {
        const double s = a(n, i);
        double* o = &out.v[i * b.c];
        for (std::size_t j = 0; j < b.c; ++j) o[j] = o[j] + s * br[j];
      }
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
// Loop structure: rows go in chunks of kKC packed as 4-column blocks [block][row][4]; every lower
// 4 x 4 block of G carries its running sums across chunks (a stored double is exact, so the
// chunking does not change any value).
static Mat gram_sharded(const Mat& a, std::size_t shards) {
  const std::size_t n = a.c, rows = a.r;
  if (shards < 1) shards = 1;
  constexpr std::size_t kKC = 256;
  const std::size_t nb = (n + 3) / 4, nblk = nb * (nb + 1) / 2;
  std::vector<double> acc(nblk * 16, 0.0), tot;
  std::vector<double> q(nb * kKC * 4);
  const std::size_t per = (rows + shards - 1) / shards;
  for (std::size_t s = 0; s < shards; ++s) {
    const std::size_t r0 = std::min(rows, s * per), r1 = std::min(rows, r0 + per);
    if (s > 0) std::fill(acc.begin(), acc.end(), 0.0);
    for (std::size_t c0 = r0; c0 < r1; c0 += kKC) {
      const std::size_t kc = std::min(kKC, r1 - c0);
      parallel_for(nb, n * kc > 65536, [&](std::size_t cb) {
        double* dst = &q[cb * kKC * 4];
        for (std::size_t k = 0; k < kc; ++k) {
          const double* src = &a.v[(c0 + k) * n];
          for (std::size_t t = 0; t < 4; ++t) dst[4 * k + t] = (4 * cb + t < n) ? src[4 * cb + t] : 0.0;
        }
      });
      parallel_for(nb, n * kc > 65536, [&](std::size_t rev) {
        const std::size_t ib = nb - 1 - rev;  // longest block rows first
        for (std::size_t jb = 0; jb <= ib; ++jb) {
          double* ap = &acc[(ib * (ib + 1) / 2 + jb) * 16];
          __m128d r[4][2];
          for (int x = 0; x < 4; ++x) {
            r[x][0] = _mm_loadu_pd(ap + 4 * x);
            r[x][1] = _mm_loadu_pd(ap + 4 * x + 2);
          }
          mk44(&q[ib * kKC * 4], &q[jb * kKC * 4], kc, r);
          for (int x = 0; x < 4; ++x) {
            _mm_storeu_pd(ap + 4 * x, r[x][0]);
            _mm_storeu_pd(ap + 4 * x + 2, r[x][1]);
          }
        }
      });
    }
    if (s == 0) {
      tot = acc;
    } else {
      for (std::size_t e = 0; e < tot.size(); ++e) tot[e] = tot[e] + acc[e];
    }
  }
  if (shards == 1 && tot.empty()) tot = acc;
  Mat g(n, n, 0.0);
  parallel_for(nb, n > 256, [&](std::size_t ib) {
    for (std::size_t jb = 0; jb <= ib; ++jb) {
      const double* ap = &tot[(ib * (ib + 1) / 2 + jb) * 16];
      for (std::size_t x = 0; x < 4; ++x)
        for (std::size_t y = 0; y < 4; ++y) {
          const std::size_t i = 4 * ib + x, j = 4 * jb + y;
          if (i < n && j <= i) {
            g(i, j) = ap[4 * x + y];
            g(j, i) = ap[4 * x + y];
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

// L y = rhs then L^T x = y, in place (linalg.cpp:147-149, 267-268).  Right-hand-side columns are
// independent, so they go in column blocks on the worker threads (same arithmetic per column); the
// backward sweep reads L^T row-wise from a transposed copy.
static void tri_solve_pair(const Mat& l, Mat& x) {
  const std::size_t n = l.r, m = x.c;
  if (n == 0 || m == 0) return;
  Mat lt(n, n);
  parallel_for(n, n > 512, [&](std::size_t i) {
    for (std::size_t j = 0; j < n; ++j) lt(j, i) = l(i, j);
  });
  const std::size_t w = std::max<std::size_t>(1, std::min<std::size_t>(8, m / std::max(1, g_threads)));
  parallel_for((m + w - 1) / w, n * n * m > 4000000, [&](std::size_t blk) {
    const std::size_t j0 = blk * w, j1 = std::min(m, j0 + w);
    for (std::size_t i = 0; i < n; ++i) {
      const double* li = &l.v[i * n];
      double* xi = &x.v[i * m];
      for (std::size_t c = 0; c < i; ++c) {
        const double s = li[c];
        if (s == 0.0) continue;
        const double* xc = &x.v[c * m];
        for (std::size_t j = j0; j < j1; ++j) xi[j] = xi[j] - s * xc[j];
      }
      for (std::size_t j = j0; j < j1; ++j) xi[j] = xi[j] / li[i];
    }
    for (std::size_t ii = n; ii-- > 0;) {
      const double* lr = &lt.v[ii * n];
      double* xi = &x.v[ii * m];
      for (std::size_t c = ii + 1; c < n; ++c) {
        const double s = lr[c];
        if (s == 0.0) continue;
        const double* xc = &x.v[c * m];
        for (std::size_t j = j0; j < j1; ++j) xi[j] = xi[j] - s * xc[j];
      }
      for (std::size_t j = j0; j < j1; ++j) xi[j] = xi[j] / lr[ii];
    }
  });
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
  // Loop structure only (not arithmetic) differs from a literal transcription of :186-247:
  //  * within a panel the G swaps (:215-216) are tracked as a position -> row map `lab` into the
  //    panel-start G (exactly symmetric, so column j of the swapped G is row lab[j] gathered at
  //    lab[i]); rows and columns before the panel are never read again, so nothing else observes
  //    the physical swaps;
  //  * the trailing update writes the next panel's G (position order, both triangles, i.e. the
  //    reference's lower update plus mirror) into a second buffer, in 4 x 4 blocks on the worker
  //    threads, from the panel's factor columns packed as [row block][column][4];
  //  * column-update rows go four at a time so their dot-product chains overlap.
  // Every element still sums its products in increasing column order from 0.0 with separately
  // rounded multiplies and adds, so F, the order and the rank are bitwise those of the scalar
  // loops (pinned by the CPU tests).
  //  * the panel's own factor columns live in a compact n x 64 array `pc` during the panel (the
  //    same values F receives at panel end).
  Mat g2(n, n, 0.0);
  std::vector<std::size_t> lab(n);
  std::vector<double> pk, pc(n * nb);
  for (std::size_t k = 0; k < n && rank == n; k += nb) {
    const std::size_t kb = std::min(nb, n - k);
    for (std::size_t i = k; i < n; ++i) lab[i] = i;
    std::fill(pc.begin(), pc.end(), 0.0);
    std::size_t jend = k + kb;  // columns of this panel written
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
        for (std::size_t c = 0; c < k; ++c) std::swap(f(j, c), f(piv, c));
        for (std::size_t c = 0; c < j - k; ++c) std::swap(pc[j * nb + c], pc[piv * nb + c]);
        std::swap(lab[j], lab[piv]);  // G row and column swap
      }
      const double rjj = d[j] > 0.0 ? std::sqrt(d[j]) : 0.0;
      if (rjj <= cut) {  // :219-223
        rank = j;
        jend = j;
        break;
      }
      pc[j * nb + (j - k)] = rjj;  // f(j, j)
      // :225-235 -- col = (G[i,j] - F[i,k:j] F[j,k:j]^T) / rjj, d -= col^2
      const double* fj = &pc[j * nb] - k;
      const double* grow = &g.v[lab[j] * n];
      auto finish = [&](std::size_t i, double s) {
        double v = grow[lab[i]];
        if (j > k) v = v - s;
        v = v / rjj;
        pc[i * nb + (j - k)] = v;
        d[i] = d[i] - v * v;
      };
      constexpr std::size_t kRows = 512;  // rows per work item (one item per thread wake-up)
      const std::size_t nrow = n - (j + 1);
      parallel_for((nrow + kRows - 1) / kRows, nrow * (j - k) > 262144, [&](std::size_t item) {
        std::size_t i = j + 1 + item * kRows;
        const std::size_t iend = std::min(n, i + kRows);
        for (; i + 4 <= iend; i += 4) {
          const double* f0 = &pc[i * nb] - k;
          const double* f1 = f0 + nb;
          const double* f2 = f1 + nb;
          const double* f3 = f2 + nb;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          for (std::size_t c = k; c < j; ++c) {
            s0 = s0 + f0[c] * fj[c];
            s1 = s1 + f1[c] * fj[c];
            s2 = s2 + f2[c] * fj[c];
            s3 = s3 + f3[c] * fj[c];
          }
          finish(i, s0);
          finish(i + 1, s1);
          finish(i + 2, s2);
          finish(i + 3, s3);
        }
        for (; i < iend; ++i) {
          const double* fi = &pc[i * nb] - k;
          double s = 0.0;
          for (std::size_t c = k; c < j; ++c) s = s + fi[c] * fj[c];
          finish(i, s);
        }
      });
    }
    parallel_for(n - k, n - k > 256, [&](std::size_t ii) {
      const std::size_t i = k + ii;
      for (std::size_t c = k; c < jend; ++c) f(i, c) = pc[i * nb + (c - k)];
    });
    const std::size_t t0 = k + kb;  // :237-244 trailing rank-kb update, lower then mirror
    if (rank == n && t0 < n) {
      const std::size_t nt = n - t0, nbk = (nt + 3) / 4;
      pk.assign(nbk * kb * 4, 0.0);
      parallel_for(nbk, nt > 256, [&](std::size_t bi) {
        for (std::size_t t = 0; t < 4; ++t) {
          const std::size_t i = t0 + 4 * bi + t;
          if (i >= n) break;
          for (std::size_t c = 0; c < kb; ++c) pk[(bi * kb + c) * 4 + t] = pc[i * nb + c];
        }
      });
      parallel_for(nbk, nt > 256, [&](std::size_t rev) {
        const std::size_t bi = nbk - 1 - rev;
        for (std::size_t bj = 0; bj <= bi; ++bj) {
          __m128d r[4][2];
          for (int x = 0; x < 4; ++x) r[x][0] = r[x][1] = _mm_setzero_pd();
          mk44(&pk[bi * kb * 4], &pk[bj * kb * 4], kb, r);
          double acc[4][4];
          for (int x = 0; x < 4; ++x) {
            _mm_storeu_pd(&acc[x][0], r[x][0]);
            _mm_storeu_pd(&acc[x][2], r[x][1]);
          }
          for (std::size_t x = 0; x < 4; ++x) {
            const std::size_t ii = t0 + 4 * bi + x;
            if (ii >= n) break;
            const double* gr = &g.v[lab[ii] * n];
            for (std::size_t y = 0; y < 4; ++y) {
              const std::size_t jj = t0 + 4 * bj + y;
              if (jj > ii) break;
              const double v = gr[lab[jj]] - acc[x][y];
              g2(ii, jj) = v;
              g2(jj, ii) = v;
            }
          }
        }
      });
      std::swap(g.v, g2.v);
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

// ---- synthetic BASELINE inputs; the same generator definition as the product's
// rbpg_synth_classification, restated here so that the CPU legs of bench.py never load the product
// library.  X iid U[0,1] from mt19937_64 per 65536-row block (seed ^ golden * (block + 1)); one-hot
// T = argmax(X V + eps), V ~ N(0,1) (d x m, teacher_seed), eps ~ N(0, sigma) drawn after each row's
// features; Gaussians by Box-Muller (cosine branch, u1 in (0, 1]); ties go to the lowest index.
static double unit53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
static double normal01(std::mt19937_64& g) {
  const double u1 = (static_cast<double>(g() >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = unit53(g);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}
static void synth_classification(std::size_t row0, std::size_t n, std::size_t d, std::size_t m, std::uint64_t seed,
                                 std::uint64_t teacher_seed, double sigma, double* x, double* t) {
  constexpr std::size_t kBlockRows = 65536;
  std::vector<double> v(d * m);
  {
    std::mt19937_64 tg(teacher_seed);
    for (auto& e : v) e = normal01(tg);
  }
  const std::size_t end = row0 + n;
  const std::size_t b0 = row0 / kBlockRows, b1 = n ? (end - 1) / kBlockRows + 1 : b0;
  // blocks are independent streams: generate them on the worker threads
  parallel_for(b1 - b0, b1 - b0 > 1, [&](std::size_t bi) {
    const std::size_t blk = b0 + bi;
    std::mt19937_64 gen(seed ^ (0x9E3779B97F4A7C15ull * static_cast<std::uint64_t>(blk + 1)));
    std::vector<double> xr(d), logits(m);
    const std::size_t bstart = blk * kBlockRows, bend = std::min(end, bstart + kBlockRows);
    for (std::size_t r = bstart; r < bend; ++r) {
      for (std::size_t k = 0; k < d; ++k) xr[k] = unit53(gen);
      for (std::size_t c = 0; c < m; ++c) logits[c] = sigma * normal01(gen);
      if (r < row0) continue;
      for (std::size_t c = 0; c < m; ++c) {
        double s = 0.0;
        for (std::size_t k = 0; k < d; ++k) s += xr[k] * v[k * m + c];
        logits[c] += s;
      }
      std::size_t am = 0;
      for (std::size_t c = 1; c < m; ++c)
        if (logits[c] > logits[am]) am = c;
      const std::size_t o = r - row0;
      std::memcpy(x + o * d, xr.data(), sizeof(double) * d);
      for (std::size_t c = 0; c < m; ++c) t[o * m + c] = (c == am) ? 1.0 : 0.0;
    }
  });
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

int oracle_synth_classification(std::size_t row0, std::size_t n, std::size_t d, std::size_t m, std::uint64_t seed,
                                std::uint64_t teacher_seed, double sigma, double* x, double* t, oracle_error* err) {
  return guarded(err, [&] {
    if (d < 1 || m < 1) throw std::invalid_argument("synth: d and m must be >= 1");
    synth_classification(row0, n, d, m, seed, teacher_seed, sigma, x, t);
  });
}

// Phase timings of train(rank) on a row sample, for bench.py's CPU legs (a bounded sample of a
// workload too large for the CPU): times[0] hidden_matrix of the sample rows, [1] their Gram and
// H^T T, [2] the rank-revealing factorisation of an L x L Gram, [3] the full-rank solve
// (gather, two triangular solves, scatter), [4] the training-accuracy pass over the sample.
// Phases 0, 1 and 4 are linear in the row count; 2 and 3 do not depend on it.  When the sample has
// fewer rows than L its Gram is rank-deficient, so the factorisation is timed on the sample Gram
// plus ridge * max(diag) * I (full rank; the pivoted Cholesky's work does not depend on the values
// once no pivot stops early).  out_rank receives the factorisation's rank.
int oracle_train_phase_times(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed,
                             const double* x, std::size_t rows, const double* y, double ridge, double* times,
                             std::size_t* out_rank, oracle_error* err) {
  return guarded(err, [&] {
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    Mat W, Bv;
    init_hidden(inputs, hidden, outputs, seed, W, Bv);
    Mat X = from_ptr(x, rows, inputs), Y = from_ptr(y, rows, outputs);
    auto t0 = now();
    Mat H = hidden_matrix(W, Bv, X);
    auto t1 = now();
    Mat G = gram(H);
    Mat hty = matmul_at(H, Y);
    auto t2 = now();
    if (rows < hidden) {
      double dmax = 0.0;
      for (std::size_t i = 0; i < hidden; ++i) dmax = std::max(dmax, G(i, i));
      for (std::size_t i = 0; i < hidden; ++i) G(i, i) = G(i, i) + ridge * dmax;
    }
    Factor fac = factor_gram(std::move(G), std::max(rows, hidden), 0.0);
    auto t3 = now();
    *out_rank = fac.rank;
    Mat beta_m(hidden, outputs, 0.0);
    if (fac.rank == hidden) {
      Mat htyp(hidden, outputs);
      for (std::size_t i = 0; i < hidden; ++i)
        for (std::size_t j = 0; j < outputs; ++j) htyp(i, j) = hty(fac.order[i], j);
      beta_m = invert_permutation_rows(solve_factored_gram(fac, htyp), fac.order);
    }
    auto t4 = now();
    volatile double acc = accuracy(matmul(H, beta_m), Y);
    (void)acc;
    auto t5 = now();
    times[0] = sec(t0, t1);
    times[1] = sec(t1, t2);
    times[2] = sec(t2, t3);
    times[3] = sec(t3, t4);
    times[4] = sec(t4, t5);
  });
}

}  // extern "C"
