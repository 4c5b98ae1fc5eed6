// rbpelm_b200.hpp -- host C++ drop-in surface for the B200 build.
//
// Source-compatible with the reference's public API for the training hot path
// (proj/include/rbpelm/matrix.hpp, linalg.hpp, elm.hpp): same namespace, type
// names, signatures, value semantics and exception types.  Every numerical
// entry point forwards to the C ABI in rbpelm_b200.h (device work on the
// process-wide default context of device 0, or the one installed with
// rbpelm::b200::set_device); status records are rethrown as the reference's
// exceptions.  pinv_svd runs the device block one-sided Jacobi SVD (the same SVD
// serves solve_direct's pseudo-inverse branch) -- see INTEGRATION.md.
//
// Reference callers include "rbpelm/matrix.hpp", "rbpelm/elm.hpp", ... : the forwarding headers in
// include/rbpelm/ map each of them onto this file, so they compile unedited with -I include.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace rbpelm {

// ---- matrix.hpp -----------------------------------------------------------
class ShapeError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(std::size_t rows, std::size_t cols, double fill = 0.0);
  DenseMatrix(std::size_t rows, std::size_t cols, std::vector<double> data);
  static DenseMatrix identity(std::size_t n);

  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  std::size_t size() const { return v_.size(); }
  bool empty() const { return v_.empty(); }
  double& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  bool all_finite() const;
  bool same_shape(const DenseMatrix& o) const { return r_ == o.r_ && c_ == o.c_; }
  bool operator==(const DenseMatrix& o) const { return same_shape(o) && v_ == o.v_; }
  std::string shape_str() const;

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix matmul_at(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix transpose(const DenseMatrix& a);
DenseMatrix add(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix subtract(const DenseMatrix& a, const DenseMatrix& b);
DenseMatrix scale(const DenseMatrix& a, double s);
DenseMatrix take_columns(const DenseMatrix& a, std::size_t begin, std::size_t end);
DenseMatrix vstack(const DenseMatrix& top, const DenseMatrix& bottom);
DenseMatrix hstack(const DenseMatrix& left, const DenseMatrix& right);
DenseMatrix gram(const DenseMatrix& a);  // device SYRK (K2)
double frobenius_norm(const DenseMatrix& a);
double max_abs(const DenseMatrix& a);
double max_abs_diff(const DenseMatrix& a, const DenseMatrix& b);

// ---- linalg.hpp -----------------------------------------------------------
class SingularMatrix : public std::runtime_error {
 public:
  SingularMatrix(std::size_t pivot_index, double pivot_value);
  std::size_t pivot_index;
  double pivot_value;
};

struct ColumnPermutation {
  std::vector<std::size_t> order;
  std::size_t rank = 0;
  double tolerance = 0.0;
};

DenseMatrix apply_permutation(const DenseMatrix& a, const ColumnPermutation& p);
DenseMatrix invert_permutation_rows(const DenseMatrix& b, const ColumnPermutation& p);

class SpdFactor {
 public:
  explicit SpdFactor(const DenseMatrix& m);
  ~SpdFactor();
  SpdFactor(SpdFactor&&) noexcept;
  SpdFactor& operator=(SpdFactor&&) noexcept;
  SpdFactor(const SpdFactor&) = delete;
  SpdFactor& operator=(const SpdFactor&) = delete;
  DenseMatrix solve(const DenseMatrix& rhs) const;
  std::size_t dim() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

DenseMatrix solve_spd(const DenseMatrix& m, const DenseMatrix& rhs);
DenseMatrix pinv_svd(const DenseMatrix& a, double tol = 0.0);
ColumnPermutation rank_revealing_permutation(const DenseMatrix& a, double tol = 0.0);

struct RankRevealingFactor {
  ColumnPermutation permutation;
  DenseMatrix factor;
};
RankRevealingFactor rank_revealing_factor(const DenseMatrix& a, double tol = 0.0);
DenseMatrix solve_factored_gram(const RankRevealingFactor& f, const DenseMatrix& rhs);
// Extension (no reference counterpart): the rank-path pseudo-inverse
// H^+ = P (F F^T)^{-1} P^T H^T (L x N) of a full-rank h; rank < L throws std::invalid_argument
// like solve_factored_gram.  `perm` (optional) receives the pivot order and rank.
DenseMatrix pseudo_inverse(const DenseMatrix& h, double tol = 0.0, ColumnPermutation* perm = nullptr);

// ---- elm.hpp --------------------------------------------------------------
enum class Activation { Sigmoid };

struct ElmParams {
  std::size_t inputs = 1;
  std::size_t hidden_nodes = 1;
  std::size_t outputs = 1;
  Activation activation = Activation::Sigmoid;
  std::uint64_t seed = 0;
};

struct HiddenLayer {
  DenseMatrix weights;  // inputs x L
  DenseMatrix biases;   // 1 x L
};

struct ElmModel {
  ElmParams params;
  HiddenLayer hidden;
  DenseMatrix beta;  // L x m, original node order
};

struct SolverStrategy {
  enum class Kind { Direct, DfSplit, RankBased };
  Kind kind = Kind::Direct;
  std::size_t split_index = 0;
  double rank_tol = 0.0;
  static SolverStrategy direct() { return {Kind::Direct, 0, 0.0}; }
  static SolverStrategy df_split(std::size_t split) { return {Kind::DfSplit, split, 0.0}; }
  static SolverStrategy rank_based(double tol = 0.0) { return {Kind::RankBased, 0, tol}; }
  std::string describe() const;
};

struct SolveDiagnostics {
  std::string strategy;
  std::size_t rank = 0;
  bool rank_known = false;
  std::size_t split_lo = 0;
  std::size_t split_hi = 0;
  bool ridge_applied = false;
  bool fallback_to_direct = false;
  bool used_svd_path = false;
  double solve_seconds = 0.0;
  double hidden_seconds = 0.0;
  double training_accuracy = -1.0;
};

class SingularSplit : public std::runtime_error {
 public:
  enum class Block { A, D };
  explicit SingularSplit(Block which);
  Block which;
};

HiddenLayer init_hidden(const ElmParams& params);
DenseMatrix hidden_matrix(const HiddenLayer& hidden, const DenseMatrix& x);
DenseMatrix solve_direct(const DenseMatrix& h, const DenseMatrix& y, SolveDiagnostics* diag = nullptr);
std::pair<DenseMatrix, DenseMatrix> solve_block_split(const DenseMatrix& h1, const DenseMatrix& h2,
                                                      const DenseMatrix& y, double ridge = 1e-8,
                                                      SolveDiagnostics* diag = nullptr);
DenseMatrix solve_beta(const DenseMatrix& h, const DenseMatrix& y, const SolverStrategy& strategy,
                       SolveDiagnostics& diag);
std::pair<ElmModel, SolveDiagnostics> train(const ElmParams& params, const DenseMatrix& x, const DenseMatrix& y,
                                            const SolverStrategy& strategy);
DenseMatrix predict(const ElmModel& model, const DenseMatrix& x);
double accuracy(const DenseMatrix& pred, const DenseMatrix& y);

// ---- data.hpp (host-side data formats feeding train()) ----
/// Feature matrix plus one-hot targets; classes in first-appearance order; feature_ranges holds
/// the per-feature (min, max) captured by normalize() (empty for raw datasets).
struct Dataset {
  DenseMatrix x;  // N x n
  DenseMatrix y;  // N x m, one-hot rows
  std::vector<std::string> class_names;
  std::vector<std::pair<double, double>> feature_ranges;
  std::size_t samples() const { return x.rows(); }
  std::size_t features() const { return x.cols(); }
  std::size_t classes() const { return y.cols(); }
};

class DataError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

/// Comma-separated numeric features and one label column (label_column < 0: the last one).
Dataset load_csv(const std::string& path, int label_column = -1, bool has_header = false);
/// Sparse "label idx:val ..." lines, 1-based indices, absent entries 0.
Dataset load_libsvm(const std::string& path);
/// libsvm text with round-trip-exact values.
void save_libsvm(const Dataset& ds, const std::string& path);
/// Per-feature min-max map onto [-1, 1]; constant features map to 0.
Dataset normalize(const Dataset& ds);
Dataset normalize_with(const Dataset& ds, const std::vector<std::pair<double, double>>& ranges);
/// Deterministic Gaussian-cluster dataset (one cluster per class), normalized.
Dataset synth(std::size_t samples, std::size_t features, std::size_t classes, std::uint64_t seed);

// ---- bench.hpp (trial protocol and report formats) ----------
struct TrialRecord {
  std::uint64_t seed = 0;
  double total_seconds = 0.0;   // H construction through beta completion (host wall clock)
  double solve_seconds = 0.0;   // beta computation (device time)
  double hidden_seconds = 0.0;  // H construction (device time)
  double accuracy = 0.0;
  std::size_t rank = 0;
  bool rank_known = false;
  bool ridge_applied = false;
  bool fallback_to_direct = false;
};

struct TrialStats {
  std::string strategy;
  std::size_t hidden_nodes = 0;
  std::size_t trials = 0;
  double mean_seconds = 0.0;
  double min_seconds = 0.0;
  double max_seconds = 0.0;
  double stddev_seconds = 0.0;
  double mean_solve_seconds = 0.0;
  double mean_accuracy = 0.0;
  std::vector<TrialRecord> records;
};

struct DatasetInfo {
  std::string name;
  std::size_t samples = 0;
  std::size_t features = 0;
  std::size_t classes = 0;
};

struct BenchmarkReport {
  std::string machine;
  DatasetInfo dataset;
  std::vector<std::size_t> node_counts;
  std::vector<std::size_t> split_points;
  std::vector<TrialStats> stats;
};

struct SweepResult {
  std::vector<TrialStats> stats;
  std::size_t best_index = 0;   // argmin of mean_seconds
  std::size_t worst_index = 0;  // argmax of mean_seconds
};

/// `trials` trainings reseeded with base seed + index, after one discarded warm-up trial.
TrialStats run_trials(const Dataset& ds, const ElmParams& params_template, const SolverStrategy& strategy,
                      std::size_t trials);
SweepResult sweep_df_splits(const Dataset& ds, const ElmParams& params_template,
                            const std::vector<std::size_t>& split_points, std::size_t trials);
BenchmarkReport sweep_nodes(const Dataset& ds, const ElmParams& params_template,
                            const std::vector<std::size_t>& node_counts,
                            const std::vector<SolverStrategy>& strategies, std::size_t trials,
                            const std::string& machine = "", const std::string& dataset_name = "");
/// format "json" (schema 1) or "csv".
void emit_report(const BenchmarkReport& report, const std::string& format, const std::string& path);
/// One tab-separated series per strategy: path_prefix.<strategy>.tsv (hidden_nodes, mean, min, max).
std::vector<std::string> emit_plot_data(const BenchmarkReport& report, const std::string& path_prefix);
std::string report_to_json(const BenchmarkReport& report);
BenchmarkReport report_from_json(const std::string& text);

// ---- checks.hpp (test-scale algebra cross-checks; reference checks.hpp:12-41) ----------
/// C = I - H2 (H2^T H2)^{-1} H2^T (N x N): the projector the production block solve never forms.
DenseMatrix materialize_projector(const DenseMatrix& h2);
/// D = H1^T C H1 through the explicit projector.
DenseMatrix materialize_schur(const DenseMatrix& h1, const DenseMatrix& h2);
/// Beta from the explicitly assembled 2 x 2 block inverse of [H1 H2]^T [H1 H2], applied to
/// [H1^T Y; H2^T Y] (L x m, [H1 H2] column order).
DenseMatrix u_block_beta(const DenseMatrix& h1, const DenseMatrix& h2, const DenseMatrix& y);

struct PropertyResult {
  std::string name;
  double max_error = 0.0;
  double tolerance = 0.0;
  bool pass = true;
  std::uint64_t failing_seed = 0;  // seed of the first failing instance
};

/// Randomized property suite over the solver algebra (block vs SVD equivalence, U-block route,
/// projector / Schur structure, Penrose conditions, rank vs SVD count, permutation round trip, df vs
/// rank label equality), `cases` instances seeded from `seed`; inject_fault perturbs one result so a
/// harness can prove it detects failures.
std::vector<PropertyResult> run_verification(std::uint64_t seed, std::size_t cases, bool inject_fault = false);

// ---- B200 extras ----------------------------------------------------------
namespace b200 {
/// Select the CUDA device used by the calls above (default 0).
void set_device(int device);
/// train() row-sharded over several GPUs of this process (rbpg_train_multi): one NCCL all-reduce of
/// the packed augmented Gram, replicated solve; fixed_order: all-gather + rank-order sum instead.
std::pair<ElmModel, SolveDiagnostics> train_multi(const ElmParams& params, const DenseMatrix& x, const DenseMatrix& y,
                                                  const SolverStrategy& strategy, const std::vector<int>& devices,
                                                  bool fixed_order = false);
}  // namespace b200

}  // namespace rbpelm
