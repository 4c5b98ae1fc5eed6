// Host C++ drop-in API (include/rbpelm_b200.hpp) over the C ABI.
// Value semantics and checks follow the reference (matrix.cpp:28-179,
// linalg.cpp:34-66, elm.cpp:53-72, 231-300); numerical work goes to the device.
#include "../../include/rbpelm_b200.hpp"
#include "../../include/rbpelm_b200.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <sstream>

namespace rbpelm {

namespace {

std::mutex g_mu;
rbpg_context* g_ctx = nullptr;
int g_device = 0;

rbpg_context* ctx() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx) {
    rbpg_status st;
    if (rbpg_context_create(g_device, &g_ctx, &st) != RBPG_OK) throw std::runtime_error(st.message);
  }
  return g_ctx;
}

// status record -> the reference's exception types
void raise(const rbpg_status& st) {
  switch (st.code) {
    case RBPG_OK:
      return;
    case RBPG_SHAPE_ERROR:
      throw ShapeError(st.message);
    case RBPG_INVALID_ARGUMENT:
      throw std::invalid_argument(st.message);
    case RBPG_SINGULAR_MATRIX:
      throw SingularMatrix(st.pivot_index, st.pivot_value);
    case RBPG_SINGULAR_SPLIT:
      throw SingularSplit(st.block == 0 ? SingularSplit::Block::A : SingularSplit::Block::D);
    default:
      throw std::runtime_error(st.message);
  }
}

rbpg_strategy to_c(const SolverStrategy& s) {
  rbpg_strategy c;
  c.kind = s.kind == SolverStrategy::Kind::Direct ? RBPG_DIRECT
           : s.kind == SolverStrategy::Kind::DfSplit ? RBPG_DF_SPLIT
                                                     : RBPG_RANK_BASED;
  c.split_index = s.split_index;
  c.rank_tol = s.rank_tol;
  return c;
}

void from_c(const rbpg_diagnostics& d, SolveDiagnostics& o) {
  o.rank = d.rank;
  o.rank_known = d.rank_known != 0;
  o.split_lo = d.split_lo;
  o.split_hi = d.split_hi;
  o.ridge_applied = d.ridge_applied != 0;
  o.fallback_to_direct = d.fallback_to_direct != 0;
  o.used_svd_path = d.used_svd_path != 0;
  o.solve_seconds = d.solve_seconds;
  o.hidden_seconds = d.hidden_seconds;
  o.training_accuracy = d.training_accuracy;
}

}  // namespace

namespace b200 {
void set_device(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx && device != g_device) {
    rbpg_context_destroy(g_ctx);
    g_ctx = nullptr;
  }
  g_device = device;
}

std::pair<ElmModel, SolveDiagnostics> train_multi(const ElmParams& params, const DenseMatrix& x, const DenseMatrix& y,
                                                  const SolverStrategy& strategy, const std::vector<int>& devices,
                                                  bool fixed_order) {
  static std::mutex mu;
  static std::map<int, rbpg_context*> ctxs;  // one context per device, process lifetime
  std::vector<rbpg_context*> list;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (int dv : devices) {
      auto it = ctxs.find(dv);
      if (it == ctxs.end()) {
        rbpg_context* c = nullptr;
        rbpg_status st;
        if (rbpg_context_create(dv, &c, &st) != RBPG_OK) throw std::runtime_error(st.message);
        it = ctxs.emplace(dv, c).first;
      }
      list.push_back(it->second);
    }
  }
  ElmModel model;
  model.params = params;
  SolveDiagnostics diag;
  diag.strategy = strategy.describe();
  const std::size_t L = std::max<std::size_t>(params.hidden_nodes, 1);
  model.hidden.weights = DenseMatrix(std::max<std::size_t>(params.inputs, 1), L, 0.0);
  model.hidden.biases = DenseMatrix(1, L, 0.0);
  model.beta = DenseMatrix(L, std::max<std::size_t>(params.outputs, 1), 0.0);
  rbpg_strategy s = to_c(strategy);
  rbpg_diagnostics d;
  rbpg_status st;
  rbpg_train_multi(list.data(), list.size(), params.inputs, params.hidden_nodes, params.outputs, params.seed, x.data(),
                   x.rows(), x.cols(), y.data(), y.rows(), y.cols(), &s, fixed_order ? 1 : 0,
                   model.hidden.weights.data(), model.hidden.biases.data(), model.beta.data(), nullptr, &d, &st);
  raise(st);
  from_c(d, diag);
  return {std::move(model), std::move(diag)};
}
}  // namespace b200

// ---- DenseMatrix ------------------------------------------------------------
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, double fill) : r_(rows), c_(cols), v_(rows * cols, fill) {
  if (rows == 0 || cols == 0) throw ShapeError("DenseMatrix dimensions must be positive, got " + shape_str());
  if (!std::isfinite(fill)) throw std::invalid_argument("DenseMatrix fill value must be finite");
}
DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data)
    : r_(rows), c_(cols), v_(std::move(data)) {
  if (rows == 0 || cols == 0) throw ShapeError("DenseMatrix dimensions must be positive, got " + shape_str());
  if (v_.size() != rows * cols)
    throw ShapeError("DenseMatrix data length " + std::to_string(v_.size()) + " does not match shape " + shape_str());
  if (!all_finite()) throw std::invalid_argument("DenseMatrix data contains non-finite entries");
}
DenseMatrix DenseMatrix::identity(std::size_t n) {
  DenseMatrix m(n, n, 0.0);
  for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}
bool DenseMatrix::all_finite() const {
  return std::all_of(v_.begin(), v_.end(), [](double x) { return std::isfinite(x); });
}
std::string DenseMatrix::shape_str() const { return std::to_string(r_) + "x" + std::to_string(c_); }

// Dense products: host loops for small operands, the DMMA GEMM above kDeviceFlops (the reference's
// acceptance test predicts through matmul(hidden_matrix(...), beta), acceptance.cpp:152-153).
namespace {
constexpr double kDeviceFlops = 2e6;
}
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.cols() != b.rows())
    throw ShapeError("matmul: inner dimensions differ, " + a.shape_str() + " times " + b.shape_str());
  DenseMatrix o(a.rows(), b.cols(), 0.0);
  if (2.0 * a.rows() * a.cols() * b.cols() >= kDeviceFlops) {
    rbpg_status st;
    rbpg_matmul(ctx(), a.data(), a.rows(), a.cols(), 0, b.data(), b.rows(), b.cols(), o.data(), &st);
    raise(st);
    return o;
  }
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t k = 0; k < a.cols(); ++k) {
      const double s = a(i, k);
      for (std::size_t j = 0; j < b.cols(); ++j) o(i, j) += s * b(k, j);
    }
  return o;
}
DenseMatrix matmul_at(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.rows() != b.rows())
    throw ShapeError("matmul_at: row counts differ, " + a.shape_str() + "^T times " + b.shape_str());
  DenseMatrix o(a.cols(), b.cols(), 0.0);
  if (2.0 * a.rows() * a.cols() * b.cols() >= kDeviceFlops) {
    rbpg_status st;
    rbpg_matmul(ctx(), a.data(), a.rows(), a.cols(), 1, b.data(), b.rows(), b.cols(), o.data(), &st);
    raise(st);
    return o;
  }
  for (std::size_t n = 0; n < a.rows(); ++n)
    for (std::size_t i = 0; i < a.cols(); ++i) {
      const double s = a(n, i);
      for (std::size_t j = 0; j < b.cols(); ++j) o(i, j) += s * b(n, j);
    }
  return o;
}
DenseMatrix transpose(const DenseMatrix& a) {
  DenseMatrix o(a.cols(), a.rows(), 0.0);
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < a.cols(); ++j) o(j, i) = a(i, j);
  return o;
}
static DenseMatrix zip(const DenseMatrix& a, const DenseMatrix& b, const char* what, double sb) {
  if (!a.same_shape(b)) throw ShapeError(std::string(what) + ": shapes differ, " + a.shape_str() + " vs " + b.shape_str());
  DenseMatrix o(a.rows(), a.cols(), 0.0);
  for (std::size_t i = 0; i < a.size(); ++i) o.data()[i] = a.data()[i] + sb * b.data()[i];
  return o;
}
DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b) { return zip(a, b, "add", 1.0); }
DenseMatrix subtract(const DenseMatrix& a, const DenseMatrix& b) {
  if (!a.same_shape(b)) throw ShapeError("subtract: shapes differ, " + a.shape_str() + " vs " + b.shape_str());
  DenseMatrix o(a.rows(), a.cols(), 0.0);
  for (std::size_t i = 0; i < a.size(); ++i) o.data()[i] = a.data()[i] - b.data()[i];
  return o;
}
DenseMatrix scale(const DenseMatrix& a, double s) {
  DenseMatrix o(a.rows(), a.cols(), 0.0);
  for (std::size_t i = 0; i < a.size(); ++i) o.data()[i] = a.data()[i] * s;
  return o;
}
DenseMatrix take_columns(const DenseMatrix& a, std::size_t begin, std::size_t end) {
  if (begin >= end || end > a.cols())
    throw ShapeError("take_columns: invalid range [" + std::to_string(begin) + ", " + std::to_string(end) + ") for " +
                     a.shape_str());
  DenseMatrix o(a.rows(), end - begin, 0.0);
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = begin; j < end; ++j) o(i, j - begin) = a(i, j);
  return o;
}
DenseMatrix vstack(const DenseMatrix& top, const DenseMatrix& bottom) {
  if (top.cols() != bottom.cols())
    throw ShapeError("vstack: column counts differ, " + top.shape_str() + " vs " + bottom.shape_str());
  DenseMatrix o(top.rows() + bottom.rows(), top.cols(), 0.0);
  std::copy(top.data(), top.data() + top.size(), o.data());
  std::copy(bottom.data(), bottom.data() + bottom.size(), o.data() + top.size());
  return o;
}
DenseMatrix hstack(const DenseMatrix& left, const DenseMatrix& right) {
  if (left.rows() != right.rows())
    throw ShapeError("hstack: row counts differ, " + left.shape_str() + " vs " + right.shape_str());
  DenseMatrix o(left.rows(), left.cols() + right.cols(), 0.0);
  for (std::size_t i = 0; i < left.rows(); ++i) {
    for (std::size_t j = 0; j < left.cols(); ++j) o(i, j) = left(i, j);
    for (std::size_t j = 0; j < right.cols(); ++j) o(i, left.cols() + j) = right(i, j);
  }
  return o;
}
DenseMatrix gram(const DenseMatrix& a) {
  DenseMatrix g(a.cols(), a.cols(), 0.0);
  rbpg_status st;
  rbpg_gram(ctx(), a.data(), a.rows(), a.cols(), g.data(), &st);
  raise(st);
  return g;
}
double frobenius_norm(const DenseMatrix& a) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a.data()[i] * a.data()[i];
  return std::sqrt(s);
}
double max_abs(const DenseMatrix& a) {
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a.data()[i]));
  return m;
}
double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b) {
  if (!a.same_shape(b)) throw ShapeError("max_abs_diff: shapes differ, " + a.shape_str() + " vs " + b.shape_str());
  double m = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a.data()[i] - b.data()[i]));
  return m;
}

// ---- linalg -------------------------------------------------------------------
SingularMatrix::SingularMatrix(std::size_t index, double value)
    : std::runtime_error("non-positive pivot " + std::to_string(value) + " at index " + std::to_string(index) +
                         " in symmetric factorization"),
      pivot_index(index),
      pivot_value(value) {}

DenseMatrix apply_permutation(const DenseMatrix& a, const ColumnPermutation& p) {
  if (a.cols() != p.order.size())
    throw ShapeError("apply_permutation: matrix has " + std::to_string(a.cols()) +
                     " columns but permutation length is " + std::to_string(p.order.size()));
  DenseMatrix o(a.rows(), a.cols(), 0.0);
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < a.cols(); ++j) o(i, j) = a(i, p.order[j]);
  return o;
}
DenseMatrix invert_permutation_rows(const DenseMatrix& b, const ColumnPermutation& p) {
  if (b.rows() != p.order.size())
    throw ShapeError("invert_permutation_rows: matrix has " + std::to_string(b.rows()) +
                     " rows but permutation length is " + std::to_string(p.order.size()));
  DenseMatrix o(b.rows(), b.cols(), 0.0);
  for (std::size_t i = 0; i < b.rows(); ++i)
    for (std::size_t j = 0; j < b.cols(); ++j) o(p.order[i], j) = b(i, j);
  return o;
}

// The factor lives on the device (rbpg_spd): factored once at construction -- SingularMatrix is
// raised there, as by the reference constructor (linalg.cpp:99-139) -- and reused by every solve.
struct SpdFactor::Impl {
  rbpg_spd* f = nullptr;
  ~Impl() { rbpg_spd_destroy(f); }
};
SpdFactor::SpdFactor(const DenseMatrix& m) : impl_(new Impl) {
  rbpg_status st;
  rbpg_spd_create(ctx(), m.data(), m.rows(), m.cols(), &impl_->f, &st);
  raise(st);
}
SpdFactor::~SpdFactor() = default;
SpdFactor::SpdFactor(SpdFactor&&) noexcept = default;
SpdFactor& SpdFactor::operator=(SpdFactor&&) noexcept = default;
std::size_t SpdFactor::dim() const { return rbpg_spd_dim(impl_->f); }
DenseMatrix SpdFactor::solve(const DenseMatrix& rhs) const {
  if (rhs.rows() != dim())
    throw ShapeError("solve_spd: rhs has " + std::to_string(rhs.rows()) + " rows, expected " + std::to_string(dim()));
  DenseMatrix out(rhs.rows(), rhs.cols(), 0.0);
  rbpg_status st;
  rbpg_spd_solve(impl_->f, rhs.data(), rhs.rows(), rhs.cols(), out.data(), &st);
  raise(st);
  return out;
}
DenseMatrix solve_spd(const DenseMatrix& m, const DenseMatrix& rhs) { return SpdFactor(m).solve(rhs); }
DenseMatrix pinv_svd(const DenseMatrix& a, double tol) {
  if (a.empty()) throw ShapeError("pinv_svd: empty matrix");
  DenseMatrix out(a.cols(), a.rows(), 0.0);
  rbpg_status st;
  rbpg_pinv_svd(ctx(), a.data(), a.rows(), a.cols(), tol, out.data(), &st);
  raise(st);
  return out;
}

RankRevealingFactor rank_revealing_factor(const DenseMatrix& a, double tol) {
  RankRevealingFactor out;
  if (a.empty()) throw ShapeError("rank_revealing_permutation: empty matrix");
  out.permutation.order.resize(a.cols());
  out.factor = DenseMatrix(a.cols(), a.cols(), 0.0);
  rbpg_status st;
  rbpg_rank_revealing_factor(ctx(), a.data(), a.rows(), a.cols(), tol, out.permutation.order.data(),
                             &out.permutation.rank, &out.permutation.tolerance, out.factor.data(), &st);
  raise(st);
  return out;
}
ColumnPermutation rank_revealing_permutation(const DenseMatrix& a, double tol) {
  return rank_revealing_factor(a, tol).permutation;
}
DenseMatrix solve_factored_gram(const RankRevealingFactor& f, const DenseMatrix& rhs) {
  const std::size_t n = f.permutation.order.size();
  DenseMatrix out(std::max<std::size_t>(rhs.rows(), 1), std::max<std::size_t>(rhs.cols(), 1), 0.0);
  rbpg_status st;
  rbpg_solve_factored_gram(ctx(), f.factor.data(), f.permutation.order.data(), n, f.permutation.rank, rhs.data(),
                           rhs.rows(), rhs.cols(), out.data(), &st);
  raise(st);
  return out;
}

DenseMatrix pseudo_inverse(const DenseMatrix& h, double tol, ColumnPermutation* perm) {
  if (h.empty()) throw ShapeError("pseudo_inverse: empty matrix");
  DenseMatrix out(h.cols(), h.rows(), 0.0);
  std::vector<std::size_t> order(h.cols());
  std::size_t rank = 0;
  rbpg_status st;
  rbpg_pseudo_inverse(ctx(), h.data(), h.rows(), h.cols(), tol, out.data(), order.data(), &rank, &st);
  if (perm) {
    perm->order = order;
    perm->rank = rank;
    perm->tolerance = tol > 0.0 ? tol : static_cast<double>(std::max(h.rows(), h.cols())) * 2.220446049250313e-16;
  }
  raise(st);
  return out;
}

// ---- elm ---------------------------------------------------------------------
std::string SolverStrategy::describe() const {  // elm.cpp:53-67
  switch (kind) {
    case Kind::Direct:
      return "direct";
    case Kind::DfSplit:
      return "df:" + std::to_string(split_index);
    case Kind::RankBased: {
      if (rank_tol <= 0.0) return "rank";
      std::ostringstream os;
      os << "rank:" << rank_tol;
      return os.str();
    }
  }
  return "?";
}

SingularSplit::SingularSplit(Block b)
    : std::runtime_error(std::string("singular ") + (b == Block::A ? "A" : "D") + " block after ridge retry"),
      which(b) {}

HiddenLayer init_hidden(const ElmParams& params) {
  if (params.inputs < 1 || params.hidden_nodes < 1 || params.outputs < 1)
    throw std::invalid_argument("ElmParams: inputs, hidden_nodes and outputs must be >= 1");
  HiddenLayer h{DenseMatrix(params.inputs, params.hidden_nodes, 0.0), DenseMatrix(1, params.hidden_nodes, 0.0)};
  rbpg_status st;
  rbpg_init_hidden(params.inputs, params.hidden_nodes, params.outputs, params.seed, h.weights.data(),
                   h.biases.data(), &st);
  raise(st);
  return h;
}

DenseMatrix hidden_matrix(const HiddenLayer& hidden, const DenseMatrix& x) {
  if (x.cols() != hidden.weights.rows())
    throw ShapeError("hidden_matrix: sample has " + std::to_string(x.cols()) + " features but the layer expects " +
                     std::to_string(hidden.weights.rows()));
  DenseMatrix h(x.rows(), hidden.weights.cols(), 0.0);
  rbpg_status st;
  rbpg_hidden_matrix(ctx(), hidden.weights.data(), hidden.biases.data(), hidden.weights.rows(),
                     hidden.weights.cols(), x.data(), x.rows(), x.cols(), h.data(), &st);
  raise(st);
  return h;
}

DenseMatrix solve_beta(const DenseMatrix& h, const DenseMatrix& y, const SolverStrategy& strategy,
                       SolveDiagnostics& diag) {
  diag.strategy = strategy.describe();
  DenseMatrix beta(h.cols(), y.cols(), 0.0);
  rbpg_strategy s = to_c(strategy);
  rbpg_diagnostics d;
  rbpg_status st;
  rbpg_solve_beta(ctx(), h.data(), h.rows(), h.cols(), y.data(), y.rows(), y.cols(), &s, beta.data(), &d, &st);
  raise(st);
  const double keep_acc = diag.training_accuracy;
  from_c(d, diag);
  diag.training_accuracy = keep_acc;
  diag.solve_seconds = diag.hidden_seconds = 0.0;
  return beta;
}

std::pair<DenseMatrix, DenseMatrix> solve_block_split(const DenseMatrix& h1, const DenseMatrix& h2,
                                                      const DenseMatrix& y, double ridge, SolveDiagnostics* diag) {
  DenseMatrix b1(std::max<std::size_t>(h1.cols(), 1), std::max<std::size_t>(y.cols(), 1), 0.0);
  DenseMatrix b2(std::max<std::size_t>(h2.cols(), 1), std::max<std::size_t>(y.cols(), 1), 0.0);
  rbpg_diagnostics d;
  rbpg_status st;
  rbpg_solve_block_split(ctx(), h1.data(), h1.rows(), h1.cols(), h2.data(), h2.rows(), h2.cols(), y.data(), y.rows(),
                         y.cols(), ridge, b1.data(), b2.data(), &d, &st);
  raise(st);
  if (diag && d.ridge_applied) diag->ridge_applied = true;
  return {std::move(b1), std::move(b2)};
}

DenseMatrix solve_direct(const DenseMatrix& h, const DenseMatrix& y, SolveDiagnostics* diag) {
  SolveDiagnostics local;
  DenseMatrix b = solve_beta(h, y, SolverStrategy::direct(), diag ? *diag : local);
  return b;
}

std::pair<ElmModel, SolveDiagnostics> train(const ElmParams& params, const DenseMatrix& x, const DenseMatrix& y,
                                            const SolverStrategy& strategy) {
  ElmModel model;
  model.params = params;
  SolveDiagnostics diag;
  diag.strategy = strategy.describe();
  const std::size_t L = std::max<std::size_t>(params.hidden_nodes, 1);
  model.hidden.weights = DenseMatrix(std::max<std::size_t>(params.inputs, 1), L, 0.0);
  model.hidden.biases = DenseMatrix(1, L, 0.0);
  model.beta = DenseMatrix(L, std::max<std::size_t>(params.outputs, 1), 0.0);
  rbpg_strategy s = to_c(strategy);
  rbpg_diagnostics d;
  rbpg_status st;
  rbpg_train(ctx(), params.inputs, params.hidden_nodes, params.outputs, params.seed, x.data(), x.rows(), x.cols(),
             y.data(), y.rows(), y.cols(), &s, model.hidden.weights.data(), model.hidden.biases.data(),
             model.beta.data(), nullptr, &d, &st);
  raise(st);
  from_c(d, diag);
  return {std::move(model), std::move(diag)};
}

DenseMatrix predict(const ElmModel& model, const DenseMatrix& x) {
  const auto& w = model.hidden.weights;
  if (x.cols() != w.rows())
    throw ShapeError("hidden_matrix: sample has " + std::to_string(x.cols()) + " features but the layer expects " +
                     std::to_string(w.rows()));
  DenseMatrix s(x.rows(), model.beta.cols(), 0.0);
  rbpg_status st;
  rbpg_predict(ctx(), w.data(), model.hidden.biases.data(), w.rows(), w.cols(), model.beta.data(), model.beta.cols(),
               x.data(), x.rows(), x.cols(), s.data(), &st);
  raise(st);
  return s;
}

double accuracy(const DenseMatrix& pred, const DenseMatrix& y) {
  double out = 0.0;
  rbpg_status st;
  rbpg_accuracy(pred.data(), pred.rows(), pred.cols(), y.data(), y.rows(), y.cols(), &out, &st);
  raise(st);
  return out;
}

}  // namespace rbpelm
