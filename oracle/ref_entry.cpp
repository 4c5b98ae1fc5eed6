// ============================================================================
// TEST INFRASTRUCTURE -- NOT PRODUCT CODE.
//
// C ABI over the REFERENCE's own library code.  oracle/Makefile (target
// `reflib`) compiles /root/reference/proj/src/{matrix,linalg,elm}.cpp where they
// lie, unedited, against oracle/eigen_standin (Eigen is absent here; see that
// header) and links them with this file into oracle/_ref/librbpelm_ref.so.
// Every entry below only marshals plain pointers into the reference's
// DenseMatrix / ElmParams and calls the reference's public functions
// (proj/include/rbpelm/{matrix,linalg,elm}.hpp).  The signatures mirror
// liboracle_rbpelm.so's (oracle_* -> ref_*), so oracle/ref.py drives both with
// the same Python and tests/test_oracle_vs_reference.py can compare the
// restatement with the reference's code on identical inputs.
// ============================================================================
#include "rbpelm/elm.hpp"
#include "rbpelm/linalg.hpp"
#include "rbpelm/matrix.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

using rbpelm::DenseMatrix;

namespace {

DenseMatrix wrap(const double* p, std::size_t r, std::size_t c) {
  return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}
void put(const DenseMatrix& m, double* out) {
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}
rbpelm::SolverStrategy strategy_of(int kind, std::size_t split_index, double rank_tol) {
  switch (kind) {
    case 0: return rbpelm::SolverStrategy::direct();
    case 1: return rbpelm::SolverStrategy::df_split(split_index);
    default: return rbpelm::SolverStrategy::rank_based(rank_tol);
  }
}

}  // namespace

extern "C" {

// same layouts as oracle_error / oracle_diag (oracle/rbpelm_oracle.cpp)
struct ref_error {
  int code;  // 0 ok, 1 ShapeError, 2 invalid_argument, 3 SingularMatrix, 4 SingularSplit, 5 runtime_error, 6 other
  std::size_t pivot_index;
  double pivot_value;
  int block;
  char message[256];
};
struct ref_diag {
  std::size_t rank;
  int rank_known;
  std::size_t split_lo, split_hi;
  int ridge_applied, fallback_to_direct, used_svd_path;
  double solve_seconds, hidden_seconds, training_accuracy;
  double min_pivot_margin;  // not produced by the reference: NaN
};

}  // extern "C"

namespace {

void set_err(ref_error* e, int code, const char* msg) {
  if (!e) return;
  e->code = code;
  std::snprintf(e->message, sizeof e->message, "%s", msg);
}

template <typename F>
int guarded(ref_error* err, F&& body) {
  if (err) std::memset(err, 0, sizeof(ref_error));
  try {
    body();
    return 0;
  } catch (const rbpelm::SingularMatrix& ex) {
    if (err) {
      err->pivot_index = ex.pivot_index;
      err->pivot_value = ex.pivot_value;
    }
    set_err(err, 3, ex.what());
    return 3;
  } catch (const rbpelm::SingularSplit& ex) {
    if (err) err->block = ex.which == rbpelm::SingularSplit::Block::A ? 0 : 1;
    set_err(err, 4, ex.what());
    return 4;
  } catch (const rbpelm::ShapeError& ex) {
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

void copy_diag(const rbpelm::SolveDiagnostics& d, ref_diag* o) {
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
  o->min_pivot_margin = std::numeric_limits<double>::quiet_NaN();
}

// The reference's solve_beta / train do not return the pivot order; the rank path's order is
// rank_revealing_permutation(H, tol) (elm.cpp calls rank_revealing_factor on the same H and tol).
void order_of(const DenseMatrix& h, double tol, std::size_t* order) {
  rbpelm::ColumnPermutation p = rbpelm::rank_revealing_permutation(h, tol);
  for (std::size_t i = 0; i < p.order.size(); ++i) order[i] = p.order[i];
}

}  // namespace

extern "C" {

void ref_set_threads(int) {}  // the reference is single-threaded

int ref_init_hidden(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed, double* w,
                    double* b, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::ElmParams p;
    p.inputs = inputs;
    p.hidden_nodes = hidden;
    p.outputs = outputs;
    p.seed = seed;
    rbpelm::HiddenLayer hl = rbpelm::init_hidden(p);
    put(hl.weights, w);
    put(hl.biases, b);
  });
}

int ref_hidden_matrix(const double* w, const double* b, std::size_t d, std::size_t l, const double* x, std::size_t n,
                      std::size_t xcols, double* h, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::HiddenLayer hl{wrap(w, d, l), wrap(b, 1, l)};
    put(rbpelm::hidden_matrix(hl, wrap(x, n, xcols)), h);
  });
}

int ref_gram(const double* a, std::size_t rows, std::size_t cols, std::size_t /*shards*/, double* g, ref_error* err) {
  return guarded(err, [&] { put(rbpelm::gram(wrap(a, rows, cols)), g); });
}

int ref_matmul(const double* a, std::size_t ar, std::size_t ac, const double* b, std::size_t br, std::size_t bc,
               double* out, ref_error* err) {
  return guarded(err, [&] { put(rbpelm::matmul(wrap(a, ar, ac), wrap(b, br, bc)), out); });
}

int ref_matmul_at(const double* a, std::size_t ar, std::size_t ac, const double* b, std::size_t br, std::size_t bc,
                  double* out, ref_error* err) {
  return guarded(err, [&] { put(rbpelm::matmul_at(wrap(a, ar, ac), wrap(b, br, bc)), out); });
}

int ref_pinv_svd(const double* a, std::size_t rows, std::size_t cols, double tol, double* out, ref_error* err) {
  return guarded(err, [&] { put(rbpelm::pinv_svd(wrap(a, rows, cols), tol), out); });
}

int ref_solve_spd(const double* m, std::size_t mr, std::size_t mc, const double* rhs, std::size_t rr, std::size_t rc,
                  double* out, ref_error* err) {
  return guarded(err, [&] { put(rbpelm::solve_spd(wrap(m, mr, mc), wrap(rhs, rr, rc)), out); });
}

int ref_rank_revealing_factor(const double* a, std::size_t rows, std::size_t cols, double tol, std::size_t* order,
                              std::size_t* rank, double* tolerance, double* factor, double* min_margin,
                              ref_error* err) {
  return guarded(err, [&] {
    rbpelm::RankRevealingFactor f = rbpelm::rank_revealing_factor(wrap(a, rows, cols), tol);
    for (std::size_t i = 0; i < f.permutation.order.size(); ++i) order[i] = f.permutation.order[i];
    *rank = f.permutation.rank;
    *tolerance = f.permutation.tolerance;
    if (factor) put(f.factor, factor);
    if (min_margin) *min_margin = std::numeric_limits<double>::quiet_NaN();
  });
}

int ref_solve_factored_gram(const double* factor, const std::size_t* order, std::size_t n, std::size_t rank,
                            const double* rhs, std::size_t rr, std::size_t rc, double* out, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::RankRevealingFactor f;
    f.permutation.order.assign(order, order + n);
    f.permutation.rank = rank;
    f.factor = wrap(factor, n, n);
    put(rbpelm::solve_factored_gram(f, wrap(rhs, rr, rc)), out);
  });
}

int ref_solve_block_split(const double* h1, std::size_t n, std::size_t c1, const double* h2, std::size_t c2,
                          const double* y, std::size_t m, double ridge, double* beta1, double* beta2, ref_diag* diag,
                          ref_error* err) {
  return guarded(err, [&] {
    rbpelm::SolveDiagnostics d;
    auto pr = rbpelm::solve_block_split(wrap(h1, n, c1), wrap(h2, n, c2), wrap(y, n, m), ridge, &d);
    put(pr.first, beta1);
    put(pr.second, beta2);
    copy_diag(d, diag);
  });
}

int ref_solve_direct(const double* h, std::size_t n, std::size_t l, const double* y, std::size_t m, double* beta,
                     ref_diag* diag, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::SolveDiagnostics d;
    put(rbpelm::solve_direct(wrap(h, n, l), wrap(y, n, m), &d), beta);
    copy_diag(d, diag);
  });
}

int ref_solve_beta(const double* h, std::size_t n, std::size_t l, const double* y, std::size_t yrows, std::size_t m,
                   int kind, std::size_t split_index, double rank_tol, std::size_t /*gram_shards*/, double* beta,
                   std::size_t* order, ref_diag* diag, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::SolveDiagnostics d;
    DenseMatrix hm = wrap(h, n, l);
    put(rbpelm::solve_beta(hm, wrap(y, yrows, m), strategy_of(kind, split_index, rank_tol), d), beta);
    if (order && kind == 2 && d.rank_known) order_of(hm, rank_tol, order);
    copy_diag(d, diag);
  });
}

int ref_train(std::size_t inputs, std::size_t hidden, std::size_t outputs, std::uint64_t seed, const double* x,
              std::size_t n, std::size_t xcols, const double* y, std::size_t yrows, std::size_t ycols, int kind,
              std::size_t split_index, double rank_tol, std::size_t /*gram_shards*/, double* w, double* b, double* beta,
              std::size_t* order, ref_diag* diag, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::ElmParams p;
    p.inputs = inputs;
    p.hidden_nodes = hidden;
    p.outputs = outputs;
    p.seed = seed;
    DenseMatrix xm = wrap(x, n, xcols);
    auto res = rbpelm::train(p, xm, wrap(y, yrows, ycols), strategy_of(kind, split_index, rank_tol));
    put(res.first.hidden.weights, w);
    put(res.first.hidden.biases, b);
    put(res.first.beta, beta);
    if (order && kind == 2 && res.second.rank_known)
      order_of(rbpelm::hidden_matrix(res.first.hidden, xm), rank_tol, order);
    copy_diag(res.second, diag);
  });
}

int ref_predict(const double* w, const double* b, std::size_t d, std::size_t l, const double* beta, std::size_t m,
                const double* x, std::size_t n, std::size_t xcols, double* scores, ref_error* err) {
  return guarded(err, [&] {
    rbpelm::ElmModel model;
    model.params.inputs = d;
    model.params.hidden_nodes = l;
    model.params.outputs = m;
    model.hidden = rbpelm::HiddenLayer{wrap(w, d, l), wrap(b, 1, l)};
    model.beta = wrap(beta, l, m);
    put(rbpelm::predict(model, wrap(x, n, xcols)), scores);
  });
}

int ref_accuracy(const double* pred, std::size_t pr, std::size_t pc, const double* y, std::size_t yr, std::size_t yc,
                 double* out, ref_error* err) {
  return guarded(err, [&] { *out = rbpelm::accuracy(wrap(pred, pr, pc), wrap(y, yr, yc)); });
}

}  // extern "C"
