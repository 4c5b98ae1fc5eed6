// Drop-in check of the C++ surface: the same calls the reference's own tests and
// tools make (proj/tests/test_linalg.cpp, test_elm.cpp, tools/rbpelm_main.cpp),
// compiled against include/rbpelm_b200.hpp and linked to librbpelm_b200.so.
// Exit code 0 = all checks passed.
#include "rbpelm_b200.hpp"

#include <cmath>
#include <cstdio>
#include <random>

using namespace rbpelm;

static int failures = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      std::printf("CHECK failed: %s (line %d)\n", #c, __LINE__);    \
      ++failures;                                                   \
    }                                                               \
  } while (0)

int main() {
  // solve_spd known answer and failing pivot (test_linalg.cpp:60-90)
  DenseMatrix rhs(2, 1, {8, 27});
  DenseMatrix x = solve_spd(DenseMatrix(2, 2, {4, 0, 0, 9}), rhs);
  CHECK(std::fabs(x(0, 0) - 2.0) < 1e-12 && std::fabs(x(1, 0) - 3.0) < 1e-12);
  try {
    solve_spd(DenseMatrix(2, 2, {1, 0, 0, 0}), DenseMatrix(2, 1, {1, 1}));
    CHECK(false);
  } catch (const SingularMatrix& e) {
    CHECK(e.pivot_index == 1);
  }
  try {
    solve_spd(DenseMatrix(2, 3, 0.0), rhs);
    CHECK(false);
  } catch (const ShapeError&) {
  }

  // train / predict with the rank strategy (tools/rbpelm_main.cpp:209-251)
  std::mt19937_64 gen(7);
  const std::size_t n = 600, d = 8, L = 64, m = 3;
  DenseMatrix X(n, d, 0.0), Y(n, m, 0.0);
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t j = 0; j < d; ++j) X(i, j) = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    Y(i, gen() % m) = 1.0;
  }
  ElmParams params{d, L, m, Activation::Sigmoid, 42};
  auto [model, diag] = train(params, X, Y, SolverStrategy::rank_based());
  CHECK(diag.strategy == "rank");
  CHECK(diag.rank_known && diag.rank == L);
  CHECK(diag.split_lo == (L + 1) / 2 && diag.split_hi == L / 2);
  CHECK(model.beta.rows() == L && model.beta.cols() == m && model.beta.all_finite());
  DenseMatrix scores = predict(model, X);
  CHECK(std::fabs(accuracy(scores, Y) - diag.training_accuracy) < 1e-15);

  // rank-revealing factor: F F^T == P^T G P (test_linalg.cpp:143-157)
  DenseMatrix H = hidden_matrix(model.hidden, X);
  RankRevealingFactor f = rank_revealing_factor(H);
  DenseMatrix G = gram(H);
  double worst = 0.0;
  for (std::size_t i = 0; i < L; ++i)
    for (std::size_t j = 0; j < L; ++j) {
      double s = 0.0;
      for (std::size_t c = 0; c < L; ++c) s += f.factor(i, c) * f.factor(j, c);
      worst = std::fmax(worst, std::fabs(s - G(f.permutation.order[i], f.permutation.order[j])) /
                                   (1.0 + std::fabs(G(i, j))));
    }
  CHECK(worst < 1e-10);

  // rank-path pseudo-inverse extension: H^+ Y reproduces the rank-path beta
  ColumnPermutation pp;
  DenseMatrix Hp = pseudo_inverse(H, 0.0, &pp);
  CHECK(Hp.rows() == L && Hp.cols() == n && pp.rank == L && pp.order == f.permutation.order);
  double dmax = 0.0, bmax = 0.0;
  for (std::size_t i = 0; i < L; ++i)
    for (std::size_t j = 0; j < m; ++j) {
      double s = 0.0;
      for (std::size_t r = 0; r < n; ++r) s += Hp(i, r) * Y(r, j);
      dmax = std::fmax(dmax, std::fabs(s - model.beta(i, j)));
      bmax = std::fmax(bmax, std::fabs(model.beta(i, j)));
    }
  CHECK(dmax <= 1e-8 * bmax);

  // N < L with a block strategy names the direct strategy (elm.cpp:248-253)
  try {
    train(ElmParams{d, 1000, m, Activation::Sigmoid, 1}, X, Y, SolverStrategy::rank_based());
    CHECK(false);
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()).find("direct") != std::string::npos);
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "ok", failures);
  return failures ? 1 : 0;
}
