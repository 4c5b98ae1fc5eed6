// Kernel parameter blocks and host-side launcher declarations shared by the
// kernel translation units and the engine.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rbpg {

// Opt kernel `fn` into `smem` bytes of dynamic shared memory (and, with nonportable_cluster,
// cluster sizes above 8) on the CURRENT device.  Function attributes are per device, so the setting
// is remembered per (device, kernel): contexts on several GPUs in one process each get it.
cudaError_t ensure_attrs(const void* fn, size_t smem, bool nonportable_cluster = false);

// CTA tile for the TMA-fed DMMA kernels (K1 hidden build, K2 Gram/trailing SYRK)
constexpr int kTile = 128;   // rows x cols of the output tile
constexpr int kBK = 16;      // reduction rows per pipeline stage
constexpr int kStages = 4;   // TMA pipeline depth
constexpr int kGemmThreads = 256;
constexpr size_t kTmaSmemBytes = size_t(kStages) * 2 * kTile * kBK * sizeof(double) + 1024 + 256;

// ---- K1: H = sigmoid(X W + b)   (reference elm.cpp:93-106)
struct HiddenParams {
  int N, d, L;
  const double* bias;
  double* H;
  long long ldh;
  int transposed;  // 0: H = sigmoid(XW + b); 1: plain product stored transposed, H[c][r] = (XW)[r][c]
  const double* T;  // optional (transposed == 0): targets copied into H[:, L:L+m] (augmented [H T] rows)
  long long ldt;
  int m;
};

// ---- K2: lower-tile SYRK C = A^T A (+ A^T B tiles), TN layout (A is K x M row-major)
enum SyrkMode : int {
  kSyrkDirect = 0,   // write lower tile + mirror into G, HtT tiles into HtT
  kSyrkPartial = 1,  // raw tiles into per-split workspaces (reduced by finish kernel)
  kSyrkTrailing = 2  // G_new[off+a][off+b] = G_old[lab[a]][lab[b]] - acc, lower + mirror
};
struct SyrkParams {
  int M;                 // columns of A (= L, or trailing size)
  int mB;                // columns of B (T) for A^T B tiles
  int nbI;               // ceil(M / kTile)
  int nGram;             // nbI*(nbI+1)/2 lower tiles
  int nbT;               // ceil(mB / kTile) (0: no A^T B tiles)
  long long kRows;       // reduction length (rows of A)
  long long kPerSplit;   // multiple of kBK
  int mode;
  double* G;
  long long ldg;
  double* HtT;
  long long ldt;
  double* ws;            // partial: split s writes ws + s*wsStride (ld = ldg)
  long long wsStride;
  double* wsT;           // partial HtT: wsT + s*wsTStride (ld = ldt)
  long long wsTStride;
  const double* Gold;    // trailing: source Gram (panel-start coordinates)
  long long ldgo;        // trailing: leading dimension of Gold
  const int* lab;        // trailing: lab[p] = source index of position p (absolute)
  int off;               // trailing: first trailing position
  int split0;            // partial: index of this launch's first split in ws (row-blocked Grams)
  unsigned long long* tl; int tl_slot;  // optional device timeline
  int late_trigger;      // trailing: release the dependent launch only after the panel before has completed
  int mirror;            // trailing: also write the upper triangle (the next panel reads whole rows)
};

// ---- K2i: Gram on the INT8 tensor cores by exact digit planes (k_ozaki.cu)
// INT8 Gram accumulator groups (k_ozaki.cu): group 0 = weights 2 .. kOzGramW0G1 - 1, group 1 = the rest
// up to 8 (at most 4 weights = 512 TMEM columns each); group 0 reads planes 1 .. kOzGramPlanesG0.
// The 3 + 4 split (kOzGramW0G1 = 5: 9 % fewer plane bytes per k-step) measured no faster
// (profiles/r02/oz_split_experiment.txt), so 4 + 3 it is.
constexpr int kOzGramW0G1 = 6;
constexpr int kOzGramPlanesG0 = kOzGramW0G1 - 2;

struct OzParams {
  int M;              // columns of A
  int nbI;            // 128-wide tile rows
  int nTiles;         // (pair, column) blocks in p.tiles
  int splits;
  int Mpad;           // plane row length (whole tile-row pairs)
  long long Npad;     // plane rows (multiple of 64)
  long long ksteps;   // Npad / 32
  long long kPerSplit;  // k-steps per split (<= 512)
  const int* exps;
  const int2* tiles;  // (pair P, column J) blocks in launch order (oz_pair_order)
  double* ws;         // packed partial slots: slot (split * 2 + group) at ws + slot * wsStride
  long long wsStride;
  int max_stages;     // 0: as many as fit (diagnostic override)
  int dbg_notma;      // diagnostic only (tools/ozaki_test): skip the operand loads
  unsigned long long* dbg;  // diagnostic cycle counters (tools/ozaki_test), null in production
};

// ---- K1i: hidden build on the INT8 tensor cores (k_ozaki.cu): H = sigmoid(X W + b) from the digit
// planes of W (column exponents) and X^T (row exponents of X), 28 exact int8 products per k-step
struct OzHidParams {
  int N, L;           // rows of X / H, hidden nodes
  int nP, nJ;         // 256-node pair tiles of W's columns, 128-row tiles of X
  int ksteps;         // padded d / 32
  const int* rexp;    // exponent of each X row (max |X[r][:]| < 2^e)
  const int* cexp;    // exponent of each W column
  const double* bias;
  double* H;
  long long ldh;
  unsigned long long* cmax;  // optional: atomic max of each H column (as ordered bits) for the Gram's scan
};

// ---- K6i: accuracy pass on the INT8 tensor cores (k_ozaki.cu): scores = H beta from the Gram's digit
// planes of H (column exponents folded into beta) and the digit planes of the folded beta; the
// arg-max of each row's scores compared with the row's target label, hits counted
struct OzScoresParams {
  int rows;            // rows of this Gram part
  int m;               // classes (<= 128)
  int nP;              // 256-row pair tiles
  int ksteps;          // plane row length / 32 (the contraction over the columns of [H T])
  const double* cscale;  // [128] 2^(f_j - 60): the class exponents of the folded beta
  const int* labels;   // optional: target label (arg-max of the T row) of each row, for the hit count
  unsigned long long* hits;
  int* out_labels;     // optional: arg-max class of each row (predict)
  double* S;           // optional: the scores (rows x m, ld lds)
  long long lds;
};

// ---- generic DMMA GEMM: C = alpha * op(A) op(B) + beta * C (row-major)
struct GemmParams {
  int M, N, K;
  const double* A; long long lda; int transA;
  const double* B; long long ldb; int transB;
  double* C; long long ldc;
  double alpha, beta;
};

// ---- K6: scores = H beta (+ fused arg-max hit count)
struct ScoresParams {
  int N, L, m;
  double* S; long long lds;            // optional score output (N x m)
  const double* T; long long ldt;      // optional targets for the hit count
  unsigned long long* hits;
};

// ---- K6b: fused predict, scores = sigmoid(X W + b) beta with the arg-max epilogue (k_predict.cu)
struct PredictParams {
  int N, d, L, m;
  const double* bias;
  double* S; long long lds;            // optional scores (N x m)
  int* labels;                         // optional arg-max labels (N)
  const double* T; long long ldt;      // optional one-hot targets for the hit count
  unsigned long long* hits;
};

// ---- K3: pivoted-Cholesky panel (reference linalg.cpp:186-247)
struct FactorState {
  int rank;          // L until the stop rule fires
  int stopped;       // factorisation finished early (rank < L) or failed (spd)
  int fail;          // spd mode: SingularMatrix raised
  int fail_index;
  double fail_value;
  double dmax0;      // max diag of the initial Gram
  double cut;        // tolerance * sqrt(dmax0)   (pivoted mode)
  double thresh;     // n * eps * maxdiag         (spd mode, linalg.cpp:109)
  double tolerance;
  double min_margin; // not used on device (diagnostic placeholder)
};

struct __align__(16) PivotSlot {
  double val;
  int pos;
  int label;
  unsigned int epoch;
  int pad[3];
};

struct PanelParams {
  const double* G;  long long ldg;     // Gram in panel-start position coordinates
  const double* d_in; double* d_out;   // running diagonal by position
  const int* ord_in; int* ord_out;     // position -> original column
  int k, kb, n;
  FactorState* st;
  double* Pg;                           // [n][64] panel columns by label (global mirror)
  double* PcT; long long ldp;           // [64][ldp] remaining rows, by new position - (k+kb)
  int* lab_out;                         // [n] position -> panel-start label (for trailing gather)
  PivotSlot* slots;                     // [2][gridDim.x]
  double* Fo; long long ldf;            // factor rows by original column
  int pivoting;                         // 1 = rank-revealing (diag pivot), 0 = SpdFactor (no pivot)
  int rows_per_cta;
  int neligible;                        // labels >= neligible are never pivots (augmented right-hand sides)
  unsigned long long* trace;                   // optional per-phase cycle counters (CTA 0, thread 0)
  unsigned long long* tl; int tl_slot;         // optional device timeline
};

}  // namespace rbpg
