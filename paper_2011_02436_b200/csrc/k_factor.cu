// Rank-revealing factorisation and solve kernels.
//
//   factor_setup_kernel : d = diag(G), order = identity, r00/cut/threshold
//                         -- reference linalg.cpp:167-195 (pivoted) / :103-109 (SpdFactor)
//   panel_kernel (K3)   : one 64-column panel of the diagonal-pivoted blocked Cholesky,
//                         persistent + cooperative, one inter-CTA exchange per column
//                         -- reference linalg.cpp:197-236 (pivot search :207-210,
//                         swaps :211-218, stop rule :219-223, column update :225-235)
//   gather_factor_kernel: factor rows by final position (the reference's F, linalg.hpp:77-80)
//   permute kernels     : row gather/scatter   -- reference elm.cpp:208-213, linalg.cpp:54-66
//   accuracy_kernel     : argmax(pred) == argmax(y) count -- reference elm.cpp:286-300
//
// Pivot bookkeeping without data movement: the reference physically swaps G rows and
// columns, F row heads and d entries.  Here every panel works on *labels* (the column's
// position at panel start).  P (the panel's F columns), d and the G reads are indexed by
// label; positions are tracked by two replicated maps (lab_at: position -> label, pos_of:
// label -> position) that every CTA updates identically.  The arg-max compares
// (d desc, position asc), which is exactly the reference's strict '>' scan over positions.
// At panel end the trailing SYRK gathers G through lab_at, so G is re-laid in position
// order once per panel instead of being swapped per column.
#include "common.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cfloat>
#include <climits>

namespace cg = cooperative_groups;

namespace rbpg {

constexpr int kPanelThreads = 256;
constexpr double kEps = 2.220446049250313e-16;

// ---------------------------------------------------------------------------
// neligible <= n: only the first neligible columns are pivot candidates (and set the tolerance);
// the rest are augmented right-hand sides carried through the factorisation.
__global__ void factor_setup_kernel(const double* G, long long ldg, int n, int neligible, long long rows, double tol,
                                    int pivoting, double* d, int* ord, FactorState* st) {
  __shared__ double red[kPanelThreads];
  double mx = -DBL_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = G[(long long)i * ldg + i];
    d[i] = v;
    ord[i] = i;
    if (i < neligible) mx = fmax(mx, v);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double dmax0 = red[0];
    st->dmax0 = dmax0;
    st->fail = 0;
    st->fail_index = -1;
    st->fail_value = 0.0;
    st->rank = neligible;
    st->stopped = 0;
    const double rmax = static_cast<double>(rows > neligible ? rows : neligible);
    st->tolerance = tol > 0.0 ? tol : rmax * kEps;   // linalg.cpp:171
    if (pivoting) {
      if (!(dmax0 > 0.0)) {                           // linalg.cpp:189-193: rank 0, identity order
        st->rank = 0;
        st->stopped = 1;
      }
      st->cut = st->tolerance * sqrt(dmax0 > 0.0 ? dmax0 : 0.0);
    } else {
      st->thresh = static_cast<double>(neligible) * kEps * dmax0;  // linalg.cpp:109
    }
  }
}

// factor rows by final position: F[a][:] = Fo[order[a]][:]
// F[a][c] = Fo[ord[a]][c] on the computed part (c <= a, c < rank); zero elsewhere, so Fo needs no
// clearing (entries above the diagonal or past an early stop are never written by the panels)
__global__ void gather_factor_kernel(const double* Fo, long long ldf, const int* ord, int n, double* F,
                                     long long ldF, const FactorState* st) {
  const long long r = st->rank;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long a = e / n, c = e % n;
    F[a * ldF + c] = (c <= a && c < r) ? Fo[(long long)ord[a] * ldf + c] : 0.0;
  }
}

// out[i][:] = in[ord[i]][:]  (elm.cpp:208-213)
__global__ void gather_rows_kernel(const double* in, long long ldin, const int* ord, int n, int m, double* out,
                                   long long ldout) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    out[i * ldout + j] = in[(long long)ord[i] * ldin + j];
  }
}
// out[ord[i]][:] = in[i][:]  (linalg.cpp:54-66)
__global__ void scatter_rows_kernel(const double* in, long long ldin, const int* ord, int n, int m, double* out,
                                    long long ldout) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    out[(long long)ord[i] * ldout + j] = in[i * ldin + j];
  }
}

// hits = #{i : argmax(pred_i) == argmax(y_i)}, strict '>' so ties go to the lowest index
__global__ void accuracy_kernel(const double* pred, long long ldp, const double* y, long long ldy, long long rows,
                                int m, unsigned long long* hits) {
  unsigned long long local = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
       i += (long long)gridDim.x * blockDim.x) {
    int ap = 0, ay = 0;
    const double* pr = pred + i * ldp;
    const double* yr = y + i * ldy;
    for (int j = 1; j < m; ++j) {
      if (pr[j] > pr[ap]) ap = j;
      if (yr[j] > yr[ay]) ay = j;
    }
    local += (ap == ay);
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(hits, local);
}

// copy a strided sub-block and add ridge to the diagonal (elm.cpp:39-40)
__global__ void add_diag_kernel(double* A, long long lda, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    A[(long long)i * lda + i] = add_rn(A[(long long)i * lda + i], v);
}

// B[i][j] = A[rows[i]][cols[j]]  (Gram sub-block by original index lists)
__global__ void gather_block_kernel(const double* A, long long lda, const int* rows, int nr, const int* cols, int nc,
                                    double* B, long long ldb) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)nr * nc;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / nc, j = e % nc;
    B[i * ldb + j] = A[(long long)rows[i] * lda + cols[j]];
  }
}

// D = (D + D^T) / 2 (elm.cpp:147), lower pass writes both
__global__ void symmetrize_kernel(double* D, long long ldd, int n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / n, j = e % n;
    if (j >= i) continue;
    const double a = D[i * ldd + j], b = D[j * ldd + i];
    const double v1 = mul_rn(add_rn(a, b), 0.5);
    const double v2 = mul_rn(add_rn(b, a), 0.5);
    D[i * ldd + j] = v1;
    D[j * ldd + i] = v2;
  }
}

// trace of a square block (single CTA, fixed order)
__global__ void trace_kernel(const double* A, long long lda, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr = add_rn(tr, A[(long long)i * lda + i]);
    *out = tr;
  }
}

// flag = 1 if any entry of the n x m block is not finite (elm.cpp:275-277)
__global__ void nonfinite_kernel(const double* A, long long lda, int n, int m, int* flag) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * m;
       e += (long long)gridDim.x * blockDim.x) {
    if (!isfinite(A[(e / m) * lda + e % m])) *flag = 1;
  }
}

// out = A - B (n x m)
__global__ void axpy_rows_kernel(const double* A, long long lda, const double* B, long long ldb, int n, int m,
                                 double* out, long long ldo) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    out[i * ldo + j] = sub_rn(A[i * lda + j], B[i * ldb + j]);
  }
}

// ============================================================================
// launchers
// ============================================================================
cudaError_t launch_factor_setup(const double* G, long long ldg, int n, int neligible, long long rows, double tol,
                                int pivoting, double* d, int* ord, FactorState* st, cudaStream_t s) {
  factor_setup_kernel<<<1, kPanelThreads, 0, s>>>(G, ldg, n, neligible, rows, tol, pivoting, d, ord, st);
  return cudaGetLastError();
}

cudaError_t launch_gather_factor(const double* Fo, long long ldf, const int* ord, int n, double* F, long long ldF,
                                 const FactorState* st,
                                 int num_sms, cudaStream_t s) {
  gather_factor_kernel<<<num_sms * 4, 256, 0, s>>>(Fo, ldf, ord, n, F, ldF, st);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* in, long long ldin, const int* ord, int n, int m, double* out,
                               long long ldout, cudaStream_t s) {
  gather_rows_kernel<<<256, 256, 0, s>>>(in, ldin, ord, n, m, out, ldout);
  return cudaGetLastError();
}
cudaError_t launch_scatter_rows(const double* in, long long ldin, const int* ord, int n, int m, double* out,
                                long long ldout, cudaStream_t s) {
  scatter_rows_kernel<<<256, 256, 0, s>>>(in, ldin, ord, n, m, out, ldout);
  return cudaGetLastError();
}

cudaError_t launch_accuracy(const double* pred, long long ldp, const double* y, long long ldy, long long rows, int m,
                            unsigned long long* hits, int num_sms, cudaStream_t s) {
  accuracy_kernel<<<num_sms * 2, 256, 0, s>>>(pred, ldp, y, ldy, rows, m, hits);
  return cudaGetLastError();
}

cudaError_t launch_add_diag(double* A, long long lda, int n, double v, cudaStream_t s) {
  add_diag_kernel<<<64, 256, 0, s>>>(A, lda, n, v);
  return cudaGetLastError();
}
cudaError_t launch_gather_block(const double* A, long long lda, const int* rows, int nr, const int* cols, int nc,
                                double* B, long long ldb, cudaStream_t s) {
  gather_block_kernel<<<512, 256, 0, s>>>(A, lda, rows, nr, cols, nc, B, ldb);
  return cudaGetLastError();
}
cudaError_t launch_symmetrize(double* D, long long ldd, int n, cudaStream_t s) {
  symmetrize_kernel<<<512, 256, 0, s>>>(D, ldd, n);
  return cudaGetLastError();
}
cudaError_t launch_nonfinite(const double* A, long long lda, int n, int m, int* flag, cudaStream_t s) {
  nonfinite_kernel<<<128, 256, 0, s>>>(A, lda, n, m, flag);
  return cudaGetLastError();
}
cudaError_t launch_axpy_rows(const double* A, long long lda, const double* B, long long ldb, int n, int m,
                             double* out, long long ldo, cudaStream_t s) {
  axpy_rows_kernel<<<128, 256, 0, s>>>(A, lda, B, ldb, n, m, out, ldo);
  return cudaGetLastError();
}
cudaError_t launch_trace(const double* A, long long lda, int n, double* out, cudaStream_t s) {
  trace_kernel<<<1, 32, 0, s>>>(A, lda, n, out);
  return cudaGetLastError();
}

}  // namespace rbpg

namespace rbpg {
// out += in (rows x cols), fixed element-wise order
__global__ void add_block_kernel(double* out, long long ldo, const double* in, long long ldi, long long rows,
                                 long long cols) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e % cols;
    out[i * ldo + j] = add_rn(out[i * ldo + j], in[i * ldi + j]);
  }
}
cudaError_t launch_add_block(double* out, long long ldo, const double* in, long long ldi, long long rows,
                             long long cols, cudaStream_t s) {
  add_block_kernel<<<512, 256, 0, s>>>(out, ldo, in, ldi, rows, cols);
  return cudaGetLastError();
}
}  // namespace rbpg

// ---------------------------------------------------------------------------
// Row-sharded exchange helpers: the all-reduce moves the packed lower triangle of the
// (augmented) Gram, n(n+1)/2 doubles, instead of the full n x n buffer.
// ---------------------------------------------------------------------------
namespace rbpg {
// packed[i(i+1)/2 + j] = G[i][j], j <= i; one CTA per row (coalesced on both sides)
__global__ void pack_lower_kernel(const double* G, long long ldg, int n, double* packed) {
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const double* gr = G + (long long)i * ldg;
    double* pr = packed + (long long)i * (i + 1) / 2;
    for (int j = threadIdx.x; j <= i; j += blockDim.x) pr[j] = gr[j];
  }
}
// G[i][j] = G[j][i] = packed[i(i+1)/2 + j]: one CTA per 32 x 32 block of the lower triangle, the
// mirrored block written as a transpose through shared memory (coalesced rows both ways)
__global__ void __launch_bounds__(256) unpack_lower_kernel(const double* packed, int n, double* G, long long ldg) {
  __shared__ double blk[32][33];
  const int nb = (n + 31) / 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (long long b = blockIdx.x; b < (long long)nb * (nb + 1) / 2; b += gridDim.x) {
    int bi = static_cast<int>((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while ((long long)bi * (bi + 1) / 2 > b) --bi;
    while ((long long)(bi + 1) * (bi + 2) / 2 <= b) ++bi;
    const int bj = static_cast<int>(b - (long long)bi * (bi + 1) / 2);
    const int i0 = bi * 32, j0 = bj * 32;
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int i = i0 + r, j = j0 + tx;
      double v = 0.0;
      if (i < n && j <= i) {
        v = packed[(long long)i * (i + 1) / 2 + j];
        G[(long long)i * ldg + j] = v;
      }
      blk[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // G[j0 + r][i0 + tx] = blk[tx][r] (strictly upper part)
      const int j = j0 + r, i = i0 + tx;
      if (i < n && j < n && j < i) G[(long long)j * ldg + i] = blk[tx][r];
    }
  }
}
// out[e] = ((parts[0][e] + parts[1][e]) + parts[2][e]) + ... : a fixed-order sum of row-shard partials
// (all-gathered), so the reduction order -- and exact ties between twin Gram columns -- does not
// depend on the collective's internal order
__global__ void sum_parts_kernel(const double* parts, long long stride, int nparts, long long count, double* out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    double v = parts[e];
    for (int p = 1; p < nparts; ++p) v = add_rn(v, parts[p * stride + e]);
    out[e] = v;
  }
}
cudaError_t launch_pack_lower(const double* G, long long ldg, int n, double* packed, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pack_lower_kernel<<<n < 4096 ? n : 4096, 256, 0, s>>>(G, ldg, n, packed);
  return cudaGetLastError();
}
cudaError_t launch_unpack_lower(const double* packed, int n, double* G, long long ldg, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const long long nb = (n + 31) / 32, blocks = nb * (nb + 1) / 2;
  unpack_lower_kernel<<<static_cast<unsigned>(blocks < 65535 ? blocks : 65535), 256, 0, s>>>(packed, n, G, ldg);
  return cudaGetLastError();
}
cudaError_t launch_sum_parts(const double* parts, long long stride, int nparts, long long count, double* out,
                             cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  sum_parts_kernel<<<1184, 256, 0, s>>>(parts, stride, nparts, count, out);
  return cudaGetLastError();
}
}  // namespace rbpg
