// K7: SVD pseudo-inverse for the solve_direct fallback (reference elm.cpp:108-122 ->
// pinv_svd, linalg.cpp:68-87: thin SVD, cut = rel * s_max with rel = tol or max(rows, cols) * eps,
// pinv = V diag(1/s) U^T over s > cut).
//
// Block one-sided Jacobi on an M x K row-major matrix A (M >= K; the wide case runs on H^T).
// Columns are grouped in blocks of 16; a round pairs the blocks by the round-robin ("circle")
// ordering, so every round rotates K/32 disjoint 32-column pairs [A_I A_J] independently:
//   svd_gram_kernel : S = [A_I A_J]^T [A_I A_J] (32 x 32), row splits -> per-split partials
//   svd_eig_kernel  : fixed-order sum of the partials; if some column pair of S is not yet
//                     orthogonal, S = Q diag Q^T by cyclic two-sided Jacobi in shared memory
//   svd_apply_kernel: [A_I A_J] <- [A_I A_J] Q and [V_I V_J] <- [V_I V_J] Q, row tiles
// Each round re-forms S from the current columns, so the orthogonality test and the rotation
// angles always come from the actual columns (the one-sided Jacobi property); a sweep is K/16 - 1
// rounds and the host stops after a sweep in which no pair rotated.  Then s_j = ||a_j||,
// U_j = a_j / s_j and  pinv(A) Y = V diag(w) A^T Y  with w_j = 1/s_j^2 over the kept s_j.
//
// This is a fallback path (rank 0 / singular Gram / SingularSplit): correctness and
// determinism first; the heavy products it feeds (A^T Y, V C) run on the DMMA GEMM.
#include "common.cuh"
#include "kernels.cuh"

namespace rbpg {

namespace {

constexpr int kSB = 16;  // column block
constexpr int kPW = 32;  // pair width
constexpr int kRowTile = 64;
constexpr int kInnerSweeps = 16;

// round-robin pairing of n (even) items, round r in [0, n-1), slot k in [0, n/2)
__device__ __forceinline__ void rr_pair(int n, int r, int k, int& a, int& b) {
  if (k == 0) {
    a = r;
    b = n - 1;
  } else {
    a = (r + k) % (n - 1);
    b = (r - k + (n - 1)) % (n - 1);
  }
}

__device__ __forceinline__ int pair_col(int bi, int bj, int c) {
  return c < kSB ? bi * kSB + c : bj * kSB + (c - kSB);
}

// 64 rows x 32 pair columns of M (rows [r0, r1) valid) into X[64][33]
__device__ __forceinline__ void load_tile(const double* M, long long ld, long long rb, long long r1, int bi, int bj,
                                          double (*X)[kPW + 1]) {
#pragma unroll
  for (int k = 0; k < kRowTile * kPW / 256; ++k) {
    const int e = threadIdx.x + 256 * k, rr = e >> 5, c = e & 31;
    const long long gr = rb + rr;
    X[rr][c] = gr < r1 ? M[gr * ld + pair_col(bi, bj, c)] : 0.0;
  }
}

}  // namespace

__global__ void __launch_bounds__(256) svd_gram_kernel(const double* A, long long lda, long long M, int nb, int round,
                                                       long long rows_per_split, double* ws) {
  __shared__ double X[kRowTile][kPW + 1];
  int bi, bj;
  rr_pair(nb, round, blockIdx.x, bi, bj);
  const long long r0 = blockIdx.y * rows_per_split;
  const long long r1 = r0 + rows_per_split < M ? r0 + rows_per_split : M;
  const int tid = threadIdx.x, i = tid >> 3, j0 = (tid & 7) * 4;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (long long rb = r0; rb < r1; rb += kRowTile) {
    load_tile(A, lda, rb, r1, bi, bj, X);
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < kRowTile; ++rr) {
      const double xi = X[rr][i];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(xi, X[rr][j0 + q], acc[q]);
    }
    __syncthreads();
  }
  double* o = ws + ((long long)blockIdx.x * gridDim.y + blockIdx.y) * (kPW * kPW);
#pragma unroll
  for (int q = 0; q < 4; ++q) o[i * kPW + j0 + q] = acc[q];
}

// Pair (p, q) of the current columns needs a rotation: not orthogonal relative to the column norms
// (tol ~ sqrt(M) eps, the accumulated-dot-product noise), and above the absolute rounding floor of
// the rotated columns (noise ~ eps ||A||_F times the larger norm).  The floor keeps a column at
// the noise level from stagnating against a large one; the resulting accuracy is the absolute
// eps * s_max class of a bidiagonalisation SVD.
__device__ __forceinline__ bool needs_rotation(double spp, double sqq, double spq, double tol, double noise) {
  const double a = fabs(spq);
  return a > 0.0 && a > tol * sqrt(spp) * sqrt(sqq) && a > noise * sqrt(spp > sqq ? spp : sqq);
}

__global__ void __launch_bounds__(256) svd_eig_kernel(const double* ws, int splits, int nb, int round, double tol,
                                                      double noise, double* Q, int* flags, int* rotated) {
  __shared__ double S[kPW][kPW + 1];
  __shared__ double Qs[kPW][kPW + 1];
  __shared__ double cs[kPW / 2], sn[kPW / 2];
  __shared__ int need, any;
  const int tid = threadIdx.x, pair = blockIdx.x;
  const double* src = ws + (long long)pair * splits * (kPW * kPW);
  for (int e = tid; e < kPW * kPW; e += 256) {
    double s = 0.0;
    for (int sp = 0; sp < splits; ++sp) s += src[(long long)sp * (kPW * kPW) + e];  // fixed order
    S[e >> 5][e & 31] = s;
    Qs[e >> 5][e & 31] = (e >> 5) == (e & 31) ? 1.0 : 0.0;
  }
  if (tid == 0) need = 0;
  __syncthreads();
  for (int e = tid; e < kPW * kPW; e += 256) {
    const int p = e >> 5, q = e & 31;
    if (p < q && needs_rotation(S[p][p], S[q][q], S[p][q], tol, noise)) need = 1;
  }
  __syncthreads();
  if (!need) {
    if (tid == 0) flags[pair] = 0;
    return;
  }
  // cyclic two-sided Jacobi: S <- R^T S R, Qs <- Qs R, 16 disjoint rotations per round
  for (int sweep = 0; sweep < kInnerSweeps; ++sweep) {
    __syncthreads();  // every thread has read `any` of the previous sweep
    if (tid == 0) any = 0;
    __syncthreads();
    for (int r = 0; r < kPW - 1; ++r) {
      if (tid < kPW / 2) {
        int p, q;
        rr_pair(kPW, r, tid, p, q);
        if (p > q) { const int t = p; p = q; q = t; }
        const double alpha = S[p][p], beta = S[q][q], gamma = S[p][q];
        double c = 1.0, s = 0.0;
        if (gamma != 0.0 && fabs(gamma) > 1e-15 * sqrt(alpha) * sqrt(beta)) {
          const double zeta = (beta - alpha) / (2.0 * gamma);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          any = 1;
        }
        cs[tid] = c;
        sn[tid] = s;
      }
      __syncthreads();
      for (int e = tid; e < (kPW / 2) * kPW; e += 256) {  // rows p, q
        const int k = e >> 5, col = e & 31;
        int p, q;
        rr_pair(kPW, r, k, p, q);
        if (p > q) { const int t = p; p = q; q = t; }
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        const double x = S[p][col], y = S[q][col];
        S[p][col] = c * x - s * y;
        S[q][col] = s * x + c * y;
      }
      __syncthreads();
      for (int e = tid; e < (kPW / 2) * kPW; e += 256) {  // columns p, q of S and Qs
        const int k = e >> 5, row = e & 31;
        int p, q;
        rr_pair(kPW, r, k, p, q);
        if (p > q) { const int t = p; p = q; q = t; }
        const double c = cs[k], s = sn[k];
        if (s == 0.0) continue;
        double x = S[row][p], y = S[row][q];
        S[row][p] = c * x - s * y;
        S[row][q] = s * x + c * y;
        x = Qs[row][p];
        y = Qs[row][q];
        Qs[row][p] = c * x - s * y;
        Qs[row][q] = s * x + c * y;
      }
      __syncthreads();
    }
    if (!any) break;
  }
  double* qo = Q + (long long)pair * (kPW * kPW);
  for (int e = tid; e < kPW * kPW; e += 256) qo[e] = Qs[e >> 5][e & 31];
  if (tid == 0) {
    flags[pair] = 1;
    atomicAdd(rotated, 1);
  }
}

// [M_I M_J] <- [M_I M_J] Q on row splits of A (blockIdx.z = 0) and V (blockIdx.z = 1)
__global__ void __launch_bounds__(256) svd_apply_kernel(double* A, long long lda, long long M, double* V,
                                                        long long ldv, long long K, int nb, int round,
                                                        long long rows_a, long long rows_v, const double* Q,
                                                        const int* flags) {
  const int pair = blockIdx.x;
  if (!flags[pair]) return;
  __shared__ double Qs[kPW][kPW + 1];
  __shared__ double X[kRowTile][kPW + 1];
  int bi, bj;
  rr_pair(nb, round, pair, bi, bj);
  double* Mt = blockIdx.z == 0 ? A : V;
  const long long ld = blockIdx.z == 0 ? lda : ldv;
  const long long per = blockIdx.z == 0 ? rows_a : rows_v;
  const long long nrows = blockIdx.z == 0 ? M : K;
  const long long r0 = blockIdx.y * per;
  if (r0 >= nrows) return;
  const long long r1 = r0 + per < nrows ? r0 + per : nrows;
  const int tid = threadIdx.x;
  const double* qi = Q + (long long)pair * (kPW * kPW);
  for (int e = tid; e < kPW * kPW; e += 256) Qs[e >> 5][e & 31] = qi[e];
  const int row = tid >> 2, c0 = (tid & 3) * 8;
  for (long long rb = r0; rb < r1; rb += kRowTile) {
    __syncthreads();
    load_tile(Mt, ld, rb, r1, bi, bj, X);
    __syncthreads();
    double out[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) out[c] = 0.0;
#pragma unroll 8
    for (int k = 0; k < kPW; ++k) {
      const double x = X[row][k];
#pragma unroll
      for (int c = 0; c < 8; ++c) out[c] = fma(x, Qs[k][c0 + c], out[c]);
    }
    const long long gr = rb + row;
    if (gr < r1) {
#pragma unroll
      for (int c = 0; c < 8; ++c) Mt[gr * ld + pair_col(bi, bj, c0 + c)] = out[c];
    }
  }
}

// out[j] = sum_k A[k][j]^2 (fixed order: 8 row lanes, then a fixed combine)
__global__ void __launch_bounds__(256) col_sumsq_kernel(const double* A, long long lda, long long M, int K,
                                                        double* out) {
  __shared__ double part[8][33];
  const int c = threadIdx.x & 31, lane_row = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + c;
  double s = 0.0;
  if (j < K)
    for (long long r = lane_row; r < M; r += 8) {
      const double v = A[r * lda + j];
      s = fma(v, v, s);
    }
  part[lane_row][c] = s;
  __syncthreads();
  if (lane_row == 0 && j < K) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += part[q][c];
    out[j] = t;
  }
}

// C[i][:] *= w[i]
__global__ void scale_rows_kernel(double* C, long long ldc, int n, int m, const double* w) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    C[i * ldc + j] *= w[i];
  }
}

// C[:][j] *= w[j]
__global__ void scale_cols_kernel(double* C, long long ldc, long long n, int m, const double* w) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n * m;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / m, j = e % m;
    C[i * ldc + j] *= w[j];
  }
}

// out (cols x rows, ld ldo; columns >= rows zero-filled up to ncols_out) = in^T, in rows x cols
__global__ void transpose_kernel(const double* in, long long ldi, long long rows, long long cols, double* out,
                                 long long ldo, long long ncols_out) {
  __shared__ double t[32][33];
  const long long r0 = blockIdx.y * 32LL, c0 = blockIdx.x * 32LL;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long r = r0 + k, c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < rows && c < cols) ? in[r * ldi + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long oc = r0 + threadIdx.x, orow = c0 + k;  // out[orow][oc] = in[oc][orow]
    if (orow < cols && oc < ncols_out) out[orow * ldo + oc] = t[threadIdx.x][k];
  }
}

cudaError_t launch_svd_round(double* A, long long lda, long long M, double* V, long long ldv, long long K, int nb,
                             int round, int splits, long long rows_per_split, int vsplits, long long rows_v,
                             double tol, double noise, double* ws, double* Q, int* flags, int* rotated,
                             cudaStream_t s) {
  const int npairs = nb / 2;
  svd_gram_kernel<<<dim3(npairs, splits), 256, 0, s>>>(A, lda, M, nb, round, rows_per_split, ws);
  svd_eig_kernel<<<npairs, 256, 0, s>>>(ws, splits, nb, round, tol, noise, Q, flags, rotated);
  const int ys = splits > vsplits ? splits : vsplits;
  svd_apply_kernel<<<dim3(npairs, ys, 2), 256, 0, s>>>(A, lda, M, V, ldv, K, nb, round, rows_per_split, rows_v, Q,
                                                        flags);
  return cudaGetLastError();
}

cudaError_t launch_col_sumsq(const double* A, long long lda, long long M, int K, double* out, cudaStream_t s) {
  col_sumsq_kernel<<<(K + 31) / 32, 256, 0, s>>>(A, lda, M, K, out);
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(double* C, long long ldc, int n, int m, const double* w, cudaStream_t s) {
  const long long e = (long long)n * m;
  int blocks = static_cast<int>((e + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  scale_rows_kernel<<<blocks, 256, 0, s>>>(C, ldc, n, m, w);
  return cudaGetLastError();
}

cudaError_t launch_scale_cols(double* C, long long ldc, long long n, int m, const double* w, cudaStream_t s) {
  const long long e = n * m;
  long long blocks = (e + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 8192) blocks = 8192;
  scale_cols_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(C, ldc, n, m, w);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double* in, long long ldi, long long rows, long long cols, double* out,
                             long long ldo, long long ncols_out, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((ncols_out + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, ldi, rows, cols, out, ldo, ncols_out);
  return cudaGetLastError();
}

}  // namespace rbpg
