/*
 * rbpelm_b200.h -- C ABI of the B200-native RBP-ELM training hot path.
 *
 * This is the drop-in boundary: plain C types, host or device pointers with
 * explicit sizes, an error record instead of C++ exceptions.  The host C++
 * API in rbpelm_b200.hpp (namespace rbpelm, same signatures as the reference's
 * proj/include/rbpelm/{matrix,linalg,elm}.hpp) is implemented on top of these
 * entry points and rethrows the reference's exception types from the record.
 *
 * All matrices are row-major fp64.  "ld" arguments are leading dimensions in
 * elements.  Host-pointer entry points copy in/out around the device work;
 * *_device entry points take device pointers and run on the context's stream.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).
 */
#ifndef RBPELM_B200_H
#define RBPELM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ layer maps them onto the reference's exceptions */
enum {
  RBPG_OK = 0,
  RBPG_SHAPE_ERROR = 1,       /* rbpelm::ShapeError            (matrix.hpp:11-14)  */
  RBPG_INVALID_ARGUMENT = 2,  /* std::invalid_argument                              */
  RBPG_SINGULAR_MATRIX = 3,   /* rbpelm::SingularMatrix{pivot}  (linalg.hpp:15-20) */
  RBPG_SINGULAR_SPLIT = 4,    /* rbpelm::SingularSplit{block}   (elm.hpp:67-72)    */
  RBPG_RUNTIME_ERROR = 5,     /* std::runtime_error (e.g. non-finite beta)          */
  RBPG_CUDA_ERROR = 6,        /* device failure                                     */
  RBPG_NOT_SUPPORTED = 7      /* path not implemented on device (SVD fallback)      */
};

/* strategy kinds (elm.hpp:36-48) */
enum { RBPG_DIRECT = 0, RBPG_DF_SPLIT = 1, RBPG_RANK_BASED = 2 };

typedef struct rbpg_status {
  int code;
  size_t pivot_index;   /* SingularMatrix::pivot_index */
  double pivot_value;   /* SingularMatrix::pivot_value */
  int block;            /* SingularSplit::which: 0 = A, 1 = D */
  char message[256];
} rbpg_status;

typedef struct rbpg_strategy {  /* SolverStrategy (elm.hpp:36-48) */
  int kind;
  size_t split_index;
  double rank_tol;
} rbpg_strategy;

typedef struct rbpg_diagnostics {  /* SolveDiagnostics (elm.hpp:51-63) */
  size_t rank;
  int rank_known;
  size_t split_lo, split_hi;
  int ridge_applied;
  int fallback_to_direct;
  int used_svd_path;
  double solve_seconds;
  double hidden_seconds;
  double training_accuracy;
} rbpg_diagnostics;

typedef struct rbpg_context rbpg_context;

/* ---- context (one per device; per-call stream-safe when not shared across threads) */
int rbpg_context_create(int device, rbpg_context** out, rbpg_status* st);
void rbpg_context_destroy(rbpg_context* ctx);
/* stream the device entry points run on (cudaStream_t); NULL = the context's own non-blocking stream
 * (pass cudaStreamLegacy, 0x1, for the legacy default stream) */
int rbpg_context_set_stream(rbpg_context* ctx, void* stream, rbpg_status* st);
int rbpg_context_synchronize(rbpg_context* ctx, rbpg_status* st);
/* number of kernels this context has launched (evidence counter for bench.py) */
uint64_t rbpg_context_launch_count(const rbpg_context* ctx);
const char* rbpg_version(void);
/* per-kernel-class device timing with CUDA events on the context stream (off by default);
 * enabling/disabling resets the counters.  Names: "hidden_kernel", "syrk_kernel", "syrk_trailing",
 * "panel_kernel", "trsm_pair_kernel", "gemm_kernel", ... */
int rbpg_context_set_profiling(rbpg_context* ctx, int enable, rbpg_status* st);
int rbpg_context_profile_get(rbpg_context* ctx, const char* name, double* total_ms, uint64_t* count,
                             rbpg_status* st);

/* ---- host utilities (no device work) */
/* init_hidden (elm.cpp:74-91): W (inputs x hidden), b (hidden) from mt19937_64(seed) */
int rbpg_init_hidden(size_t inputs, size_t hidden, size_t outputs, uint64_t seed, double* w, double* b,
                     rbpg_status* st);
/* accuracy (elm.cpp:286-300): fraction of rows with argmax(pred) == argmax(y) */
int rbpg_accuracy(const double* pred, size_t rows, size_t cols, const double* y, size_t yrows, size_t ycols,
                  double* out, rbpg_status* st);
/* Synthetic classification data: X iid U[0,1] (N x d), one-hot T (N x m) from
 * argmax(X V + eps), V ~ N(0,1) (d x m) from teacher_seed, eps ~ N(0, noise_sigma).  Rows are
 * generated in 65536-row blocks seeded from (seed, block), so any row range [row0, row0+N)
 * of the global matrix can be generated independently (row sharding). */
int rbpg_synth_classification(size_t row0, size_t n, size_t d, size_t m, uint64_t seed, uint64_t teacher_seed,
                              double noise_sigma, double* x, double* t, rbpg_status* st);

/* Config-3 inputs: X = [B, B C] (n x 2*base), B iid U[0,1], C iid U[-1,1] (mix_seed); one-hot T. */
int rbpg_synth_rank_deficient(size_t n, size_t base, size_t m, uint64_t seed, uint64_t mix_seed,
                              uint64_t teacher_seed, double noise_sigma, double* x, double* t, rbpg_status* st);
/* Overwrite ndup hidden nodes (W column + bias) with copies of distinct other nodes (seeded). */
int rbpg_duplicate_nodes(double* w, double* b, size_t d, size_t l, size_t ndup, uint64_t seed, size_t* target_out,
                         size_t* source_out, rbpg_status* st);

/* ---- host-buffer entry points (reference-facing; copy in, compute on device, copy out) */

/* hidden_matrix (elm.cpp:93-106): H (n x L) = sigmoid(X W + b) */
int rbpg_hidden_matrix(rbpg_context* ctx, const double* w, const double* b, size_t d, size_t l, const double* x,
                       size_t n, size_t xcols, double* h, rbpg_status* st);
/* gram (matrix.cpp:152-161): G (cols x cols) = A^T A, exactly symmetric */
int rbpg_gram(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double* g, rbpg_status* st);
/* rank_revealing_factor (linalg.cpp:157-248); factor may be NULL (= rank_revealing_permutation) */
int rbpg_rank_revealing_factor(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double tol,
                               size_t* order, size_t* rank, double* tolerance, double* factor, rbpg_status* st);
/* solve_factored_gram (linalg.cpp:254-270): out (n x m) = (F F^T)^{-1} rhs in permuted coordinates */
int rbpg_solve_factored_gram(rbpg_context* ctx, const double* factor, const size_t* order, size_t n, size_t rank,
                             const double* rhs, size_t rrows, size_t m, double* out, rbpg_status* st);
/* Rank-path pseudo-inverse (not a reference entry point -- the reference forms
 * beta = H^+ T without materialising H^+): out (l x n) = P (F F^T)^{-1} P^T H^T, i.e. the
 * full-rank solve of elm.cpp:202-214 / solve_factored_gram (linalg.cpp:254-270) with right-hand
 * side H^T.  order (l) and rank are written; rank < l fails with RBPG_INVALID_ARGUMENT like
 * solve_factored_gram (linalg.cpp:256-260).  tol as rank_revealing_factor. */
int rbpg_pseudo_inverse(rbpg_context* ctx, const double* h, size_t n, size_t l, double tol, double* out,
                        size_t* order, size_t* rank, rbpg_status* st);
/* pinv_svd (linalg.cpp:68-87): out (cols x rows) = V diag(1/s) U^T over s > rel * s_max,
 * rel = tol > 0 ? tol : max(rows, cols) * eps.  Device block one-sided Jacobi SVD (k_svd.cu); the
 * same SVD serves solve_direct's pseudo-inverse branch (elm.cpp:119-121) inside solve_beta/train. */
int rbpg_pinv_svd(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double tol, double* out,
                  rbpg_status* st);
/* solve_spd (linalg.cpp:99-155): out = m^{-1} rhs through a blocked Cholesky */
int rbpg_solve_spd(rbpg_context* ctx, const double* m, size_t mrows, size_t mcols, const double* rhs, size_t rrows,
                   size_t rcols, double* out, rbpg_status* st);
/* solve_beta (elm.cpp:158-229) on a host H (n x L), Y (n x m) */
int rbpg_solve_beta(rbpg_context* ctx, const double* h, size_t n, size_t l, const double* y, size_t yrows, size_t m,
                    const rbpg_strategy* strategy, double* beta, rbpg_diagnostics* diag, rbpg_status* st);
/* train (elm.cpp:231-280): outputs W (inputs x L), b (L), beta (L x m); order (L) optional */
int rbpg_train(rbpg_context* ctx, size_t inputs, size_t hidden, size_t outputs, uint64_t seed, const double* x,
               size_t n, size_t xcols, const double* y, size_t yrows, size_t ycols, const rbpg_strategy* strategy,
               double* w, double* b, double* beta, size_t* order, rbpg_diagnostics* diag, rbpg_status* st);
/* Multi-GPU train() in ONE process ("the multi-GPU variant takes a device count";
 * §8(e)): contexts on ndev distinct devices; rows [r0_i, r0_i + n_i) go to device i (contiguous
 * shards, the first n % ndev shards one row longer); each device builds its augmented Gram
 * [H T]^T [H T]; ONE NCCL all-reduce (ncclCommInitAll over the devices, libnccl.so.2 resolved at run
 * time) of its packed lower triangle, or with fixed_order != 0 an all-gather plus a rank-order sum
 * (exact twin ties survive sharding); every device runs the identical solve (default tolerance with
 * the GLOBAL n, linalg.cpp:171); hits are summed.  Outputs as rbpg_train (beta and order from
 * device 0); diag->hidden_seconds = upload + H build + Gram, solve_seconds = exchange + solve +
 * accuracy (host wall clock). */
int rbpg_train_multi(rbpg_context* const* ctxs, size_t ndev, size_t inputs, size_t hidden, size_t outputs,
                     uint64_t seed, const double* x, size_t n, size_t xcols, const double* y, size_t yrows,
                     size_t ycols, const rbpg_strategy* strategy, int fixed_order, double* w, double* b,
                     double* beta, size_t* order, rbpg_diagnostics* diag, rbpg_status* st);
/* predict (elm.cpp:282-284): scores (n x m) = sigmoid(X W + b) beta */
int rbpg_predict(rbpg_context* ctx, const double* w, const double* b, size_t d, size_t l, const double* beta,
                 size_t m, const double* x, size_t n, size_t xcols, double* scores, rbpg_status* st);

/* solve_block_split (elm.cpp:124-156, elm.hpp:86-93): beta1 (c1 x m), beta2 (c2 x m) of the block solve
 * of [H1 H2] against Y through the Gram of H2 and the Schur complement, one relative ridge retry per
 * block (ridge, elm.cpp:30-49; 1e-8 in the reference's callers).  Row-count mismatch or n < c1 + c2:
 * RBPG_SHAPE_ERROR; a block still singular after the retry: RBPG_SINGULAR_SPLIT (block 0 = A, 1 = D).
 * diag->ridge_applied reports the retry. */
int rbpg_solve_block_split(rbpg_context* ctx, const double* h1, size_t n, size_t c1, const double* h2, size_t n2,
                           size_t c2, const double* y, size_t yrows, size_t m, double ridge, double* beta1,
                           double* beta2, rbpg_diagnostics* diag, rbpg_status* st);
/* SpdFactor (linalg.cpp:99-151, linalg.hpp:45-60): the Cholesky factor of m stays on the device and is
 * reused by every solve.  create fails with RBPG_SINGULAR_MATRIX (pivot index / value in st) like the
 * reference constructor; solve checks the right-hand-side row count (RBPG_SHAPE_ERROR). */
typedef struct rbpg_spd rbpg_spd;
int rbpg_spd_create(rbpg_context* ctx, const double* m, size_t mrows, size_t mcols, rbpg_spd** out, rbpg_status* st);
int rbpg_spd_solve(const rbpg_spd* f, const double* rhs, size_t rrows, size_t rcols, double* out, rbpg_status* st);
size_t rbpg_spd_dim(const rbpg_spd* f);
void rbpg_spd_destroy(rbpg_spd* f);
/* matmul (matrix.cpp:69-77; trans_a = 0) and matmul_at (matrix.cpp:79-87; trans_a = 1): out = op(a) b on
 * the DMMA GEMM; the shape errors of the reference's matmul / matmul_at */
int rbpg_matmul(rbpg_context* ctx, const double* a, size_t ar, size_t ac, int trans_a, const double* b, size_t br,
                size_t bc, double* out, rbpg_status* st);

/* ---- device-pointer stage API (torch plumbing, row-sharded multi-GPU)
 * Stage 1 (per shard): G (L x L, ld ldg) and HtT (L x m, ld ldt) of the local rows.  If keep_h,
 * H stays resident in the context for stage 3.  accumulate != 0 adds into G/HtT. */
int rbpg_gram_stage_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                           size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw, const double* db,
                           double* dg, size_t ldg, double* dhtt, size_t ldt, int accumulate, int keep_h,
                           rbpg_status* st);
/* Stage 2 (replicated): beta (L x m, ld ldb) from the (all-reduced) G, HtT.  n_total is the global
 * row count (default tolerance, linalg.cpp:171).  order_out (host, L) optional. */
int rbpg_solve_stage_device(rbpg_context* ctx, const double* dg, size_t ldg, const double* dhtt, size_t ldt,
                            size_t l, size_t m, size_t n_total, const rbpg_strategy* strategy, double* dbeta,
                            size_t ldb, size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st);
/* Augmented form of stages 1 and 2: stage 1 writes (adds, with accumulate) the whole
 * (L+m) x (L+m) Gram of [H T] (ld ldga >= L+m), so a sharded job all-reduces ONE buffer; stage 2
 * then factors it with the targets carried along (forward substitution inside the factorisation,
 * backward sweep only) -- the single-GPU train() pipeline. */
int rbpg_gram_stage_device_aug(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                               size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw, const double* db,
                               double* dgaug, size_t ldga, int accumulate, int keep_h, rbpg_status* st);
int rbpg_solve_stage_device_aug(rbpg_context* ctx, const double* dgaug, size_t ldga, size_t l, size_t m,
                                size_t n_total, const rbpg_strategy* strategy, double* dbeta, size_t ldb,
                                size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st);
/* Stage 3 (per shard): number of local rows whose argmax(H beta) equals argmax(T).  Uses the H kept
 * by stage 1 when available, otherwise rebuilds it from X. */
int rbpg_accuracy_stage_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                               size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw,
                               const double* db, const double* dbeta, size_t ldb, uint64_t* hits, rbpg_status* st);
/* gram on a device matrix: G (cols x cols, ld ldg) (+)= A^T A, exactly symmetric (matrix.cpp:152-161) */
int rbpg_gram_device(rbpg_context* ctx, const double* da, size_t lda, size_t rows, size_t cols, double* dg, size_t ldg,
                     int accumulate, rbpg_status* st);
/* The train path's Gram kernel on an arbitrary device matrix: G (cols x cols, ld ldg) (+)= A^T A on the
 * INT8 tensor cores (exact digit planes, fp64 combination; lower triangle + mirror, exactly symmetric).
 * Same contract as rbpg_gram_device; accuracy: |G - exact| <= ~2^-53 sqrt(G_aa G_bb) (tests/test_ozaki_gpu.py). */
int rbpg_gram_int8_device(rbpg_context* ctx, const double* da, size_t lda, size_t rows, size_t cols, double* dg,
                          size_t ldg, int accumulate, rbpg_status* st);
/* Row-sharded pseudo-inverse: from the (all-reduced) Gram of all n_total rows, writes this shard's
 * column block dout (l x n_local, ld ldo) = H^+[:, local rows] for the local rows dh (n_local x l).
 * order/rank (host) optional. */
int rbpg_pseudo_inverse_stage_device(rbpg_context* ctx, const double* dg, size_t ldg, size_t n_total,
                                     const double* dh, size_t ldh, size_t n_local, size_t l, double tol, double* dout,
                                     size_t ldo, size_t* order, size_t* rank, rbpg_status* st);
/* Batched predict (elm.cpp:282-284) on device X (n x d): fused sigma(X W + b) beta (H never stored),
 * optional scores (n x m, ld lds) and/or arg-max labels (int32, strict '>' with the lowest index on
 * ties, elm.cpp:291-296).  m <= 128 (RBPG_NOT_SUPPORTED otherwise; rbpg_predict handles any m). */
int rbpg_predict_device(rbpg_context* ctx, const double* dx, size_t ldx, size_t n, size_t d, const double* dw,
                        size_t ldw, const double* db, size_t l, const double* dbeta, size_t ldb, size_t m,
                        double* dscores, size_t lds, int* dlabels, rbpg_status* st);
/* Row-sharded exchange helpers: the all-reduce carries the packed lower triangle of the
 * (augmented) Gram, n(n+1)/2 doubles (element (i, j <= i) at i(i+1)/2 + j); unpack rebuilds the
 * exactly symmetric matrix.  sum_parts: out[e] = ((p_0[e] + p_1[e]) + p_2[e]) + ... over nparts
 * partials stride apart (an all-gather plus this fixed-order sum keeps exact twin ties, C3). */
int rbpg_pack_lower_device(rbpg_context* ctx, const double* dg, size_t ldg, size_t n, double* dpacked,
                           rbpg_status* st);
int rbpg_unpack_lower_device(rbpg_context* ctx, const double* dpacked, size_t n, double* dg, size_t ldg,
                             rbpg_status* st);
int rbpg_sum_parts_device(rbpg_context* ctx, const double* dparts, size_t stride, size_t nparts, size_t count,
                          double* dout, rbpg_status* st);
/* Whole train() on device-resident X, T (W, b host arrays from init_hidden). */
int rbpg_train_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in, size_t n,
                      size_t d, size_t l, size_t m, const double* w, const double* b, const rbpg_strategy* strategy,
                      double* dbeta, size_t ldb, size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st);

#ifdef __cplusplus
}
#endif
#endif /* RBPELM_B200_H */
