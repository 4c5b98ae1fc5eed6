// Rank-revealing factorisation and solve kernels.
//
//   factor_setup_kernel : d = diag(G), order = identity, r00/cut/threshold
//                         -- reference linalg.cpp:167-195 (pivoted) / :103-109 (SpdFactor)
//   panel_kernel (K3)   : one 64-column panel of the diagonal-pivoted blocked Cholesky,
//                         persistent + cooperative, one inter-CTA exchange per column
//                         -- reference linalg.cpp:197-236 (pivot search :207-210,
//                         swaps :211-218, stop rule :219-223, column update :225-235)
//   gather_factor_kernel: factor rows by final position (the reference's F, linalg.hpp:77-80)
//   trsm_pair_kernel(K4): F y = b, F^T x = y   -- reference linalg.cpp:254-270 / 141-151
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

constexpr int kPanel = 64;
constexpr int kPanelThreads = 256;
constexpr double kEps = 2.220446049250313e-16;

// ---------------------------------------------------------------------------
__global__ void factor_setup_kernel(const double* G, long long ldg, int n, long long rows, double tol,
                                    int pivoting, double* d, int* ord, FactorState* st) {
  __shared__ double red[kPanelThreads];
  double mx = -DBL_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = G[(long long)i * ldg + i];
    d[i] = v;
    ord[i] = i;
    mx = fmax(mx, v);
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
    st->rank = n;
    st->stopped = 0;
    const double rmax = static_cast<double>(rows > n ? rows : n);
    st->tolerance = tol > 0.0 ? tol : rmax * kEps;   // linalg.cpp:171
    if (pivoting) {
      if (!(dmax0 > 0.0)) {                           // linalg.cpp:189-193: rank 0, identity order
        st->rank = 0;
        st->stopped = 1;
      }
      st->cut = st->tolerance * sqrt(dmax0 > 0.0 ? dmax0 : 0.0);
    } else {
      st->thresh = static_cast<double>(n) * kEps * dmax0;  // linalg.cpp:109
    }
  }
}

// ---------------------------------------------------------------------------
// Panel kernel.  Grid: C CTAs (cooperative launch => co-resident), CTA c owns labels
// [k + c*R, k + (c+1)*R).  Dynamic smem: lab_at[nl], pos_of[nl] (int) + PsT[64][R] + dl[R].
// ---------------------------------------------------------------------------
struct BestCand {
  double val;
  int pos;
  int label;
};
__device__ __forceinline__ bool better(double v1, int p1, double v2, int p2) {
  return v1 > v2 || (v1 == v2 && p1 < p2);
}

__global__ void __launch_bounds__(kPanelThreads, 1) panel_kernel(PanelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = p.n, k = p.k, kb = p.kb, nl = n - k;
  const int R = p.rows_per_cta;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int C = gridDim.x, cta = blockIdx.x;

  double* PsT = reinterpret_cast<double*>(smem_raw);          // [64][R]
  double* dl = PsT + kPanel * R;                              // [R]
  int* lab_at = reinterpret_cast<int*>(dl + R);               // [nl] position-k -> label
  int* pos_of = lab_at + nl;                                  // [nl] label-k -> position
  __shared__ double prow[kPanel];
  __shared__ BestCand win;
  __shared__ double red_v[kPanelThreads / 32];
  __shared__ int red_p[kPanelThreads / 32], red_l[kPanelThreads / 32];
  __shared__ int s_stop;

  FactorState* st = p.st;
  if (st->stopped) {  // an earlier panel ended the factorisation: carry the order through
    if (cta == 0)
      for (int i = tid; i < n; i += blockDim.x) p.ord_out[i] = p.ord_in[i];
    return;
  }

  const int lbeg = k + cta * R;
  const int lend = min(n, lbeg + R);
  const int nown = max(0, lend - lbeg);

  for (int i = tid; i < nl; i += blockDim.x) {
    lab_at[i] = k + i;
    pos_of[i] = k + i;
  }
  for (int i = tid; i < kPanel * R; i += blockDim.x) PsT[i] = 0.0;
  for (int i = tid; i < R; i += blockDim.x) dl[i] = (i < nown) ? p.d_in[lbeg + i] : -DBL_MAX;
  if (tid == 0) s_stop = 0;
  __syncthreads();

  const double cut = st->cut;
  const double thresh = st->thresh;

  // local arg-max over owned alive labels -> publish slot for step j
  auto publish = [&](int j) {
    double bv = -DBL_MAX;
    int bp = INT_MAX, bl = -1;
    if (p.pivoting) {
      for (int i = tid; i < nown; i += blockDim.x) {
        const int x = lbeg + i;
        const int pos = pos_of[x - k];
        if (pos < j) continue;  // already pivoted
        const double v = dl[i];
        if (better(v, pos, bv, bp)) { bv = v; bp = pos; bl = x; }
      }
    } else {
      // SpdFactor: no pivoting; the candidate for step j is label j itself
      if (j >= lbeg && j < lend && tid == 0) { bv = dl[j - lbeg]; bp = j; bl = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; bl = ol; }
    }
    if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; red_l[warp] = bl; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kPanelThreads / 32; ++w)
        if (better(red_v[w], red_p[w], bv, bp)) { bv = red_v[w]; bp = red_p[w]; bl = red_l[w]; }
      PivotSlot* sl = p.slots + (j & 1) * C + cta;
      sl->val = bv;
      sl->pos = bp;
      sl->label = bl;
      __threadfence();
      st_release_u32(&sl->epoch, static_cast<unsigned int>(j + 1));
    }
  };

  publish(k);

  int steps = 0;
  for (int c = 0; c < kb; ++c) {
    const int j = k + c;
    // ---- gather all CTAs' candidates for step j and pick the winner (identical in every CTA)
    if (warp == 0) {
      double bv = -DBL_MAX;
      int bp = INT_MAX, bl = -1;
      const PivotSlot* base = p.slots + (j & 1) * C;
      for (int i = lane; i < C; i += 32) {
        while (ld_acquire_u32(&base[i].epoch) != static_cast<unsigned int>(j + 1)) {
        }
        const double v = ld_volatile_f64(&base[i].val);
        const int ps = *reinterpret_cast<const volatile int*>(&base[i].pos);
        const int lb = *reinterpret_cast<const volatile int*>(&base[i].label);
        if (better(v, ps, bv, bp)) { bv = v; bp = ps; bl = lb; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (better(ov, op, bv, bp)) { bv = ov; bp = op; bl = ol; }
      }
      if (lane == 0) {
        win.val = bv;
        win.pos = bp;
        win.label = bl;
        // swap positions j and piv (linalg.cpp:211-218) in the replicated maps
        const int piv = bp, xp = bl;
        if (piv != j) {
          const int y = lab_at[j - k];
          lab_at[j - k] = xp;
          lab_at[piv - k] = y;
          pos_of[xp - k] = j;
          pos_of[y - k] = piv;
        }
        // stop / failure rule
        const double dj = bv;
        if (p.pivoting) {
          const double rjj = dj > 0.0 ? sqrt(dj) : 0.0;
          if (rjj <= cut) s_stop = 1;                                   // linalg.cpp:219-223
        } else {
          if (!isfinite(dj) || dj <= thresh || dj <= 0.0) s_stop = 2;   // linalg.cpp:118-119
        }
      }
    }
    __syncthreads();
    if (s_stop) {
      if (cta == 0 && tid == 0) {
        st->stopped = 1;
        st->rank = j;
        if (s_stop == 2) {
          st->fail = 1;
          st->fail_index = j;
          st->fail_value = win.val;
        }
      }
      break;
    }
    const int xp = win.label;
    const double rjj = sqrt(win.val);
    // pivot row of the panel so far (written by its owner in earlier steps; L2 read)
    if (tid < c) prow[tid] = __ldcg(p.Pg + (long long)(xp - k) * kPanel + tid);
    if (xp >= lbeg && xp < lend && tid == 0) {
      PsT[c * R + (xp - lbeg)] = rjj;   // F(j, j) = rjj
      p.Pg[(long long)(xp - k) * kPanel + c] = rjj;
    }
    __syncthreads();

    // ---- column update for owned alive labels: quad (4 lanes) per label
    const double* grow = p.G + (long long)xp * p.ldg;
    for (int base = 0; base < nown; base += kPanelThreads / 4) {
      const int li = base + (tid >> 2);
      const int q = tid & 3;
      const bool active = li < nown;
      const int x = lbeg + li;
      bool alive = false;
      if (active) alive = pos_of[x - k] > j;
      double s = 0.0;
      if (alive) {
        const int cb = q * 16, ce = min(c, cb + 16);
        for (int cc = cb; cc < ce; ++cc) s = add_rn(s, mul_rn(PsT[cc * R + li], prow[cc]));
      }
      // fixed combine order ((s0 + s1) + s2) + s3
      const double s1 = __shfl_down_sync(0xffffffffu, s, 1, 4);
      const double s2 = __shfl_down_sync(0xffffffffu, s, 2, 4);
      const double s3 = __shfl_down_sync(0xffffffffu, s, 3, 4);
      if (alive && q == 0) {
        const double tot = add_rn(add_rn(add_rn(s, s1), s2), s3);
        const double gv = grow[x];
        const double col = (c > 0 ? sub_rn(gv, tot) : gv) / rjj;
        PsT[c * R + li] = col;
        p.Pg[(long long)(x - k) * kPanel + c] = col;
        dl[li] = sub_rn(dl[li], mul_rn(col, col));
      }
    }
    steps = c + 1;
    __syncthreads();
    if (c + 1 < kb) publish(j + 1);
  }
  __syncthreads();

  // ---- write back: factor rows by original column, compacted trailing panel, d, order
  for (int e = tid; e < nown * kPanel; e += blockDim.x) {
    const int li = e / kPanel, cc = e % kPanel;
    if (cc >= kb) continue;
    const int x = lbeg + li;
    const int orig = p.ord_in[x];
    p.Fo[(long long)orig * p.ldf + k + cc] = PsT[cc * R + li];
  }
  const bool stopped = s_stop != 0;
  if (!stopped) {
    const int t0 = k + kb;
    for (int e = tid; e < nown * kPanel; e += blockDim.x) {
      const int li = e / kPanel, cc = e % kPanel;
      if (cc >= kb) continue;
      const int x = lbeg + li;
      const int pos = pos_of[x - k];
      if (pos < t0) continue;
      p.PcT[(long long)cc * p.ldp + (pos - t0)] = PsT[cc * R + li];
    }
    for (int li = tid; li < nown; li += blockDim.x) {
      const int pos = pos_of[lbeg + li - k];
      if (pos >= t0) p.d_out[pos] = dl[li];
    }
  }
  // order / label maps: positions split across CTAs
  for (int pos = cta * blockDim.x + tid; pos < n; pos += C * blockDim.x) {
    if (pos < k) {
      p.ord_out[pos] = p.ord_in[pos];
    } else {
      const int lb = lab_at[pos - k];
      p.ord_out[pos] = p.ord_in[lb];
      p.lab_out[pos] = lb;
    }
  }
  (void)steps;
}

// factor rows by final position: F[a][:] = Fo[order[a]][:]
__global__ void gather_factor_kernel(const double* Fo, long long ldf, const int* ord, int n, double* F,
                                     long long ldF) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long a = e / n, c = e % n;
    F[a * ldF + c] = Fo[(long long)ord[a] * ldf + c];
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

// ---------------------------------------------------------------------------
// K4: F y = b then F^T x = y, in place on X (n x m), F lower (n x n).
// Cooperative: every CTA solves the 64x64 diagonal block redundantly in shared memory
// (identical arithmetic), then updates its contiguous slice of the remaining rows; one
// grid barrier per block.
// ---------------------------------------------------------------------------
constexpr int kTB = 64;
__global__ void __launch_bounds__(256) trsm_pair_kernel(const double* F, long long ldf, double* X, long long ldx,
                                                        int n, int m, int do_forward, int do_backward) {
  extern __shared__ __align__(16) double tsm[];
  double* Fd = tsm;                 // [64][65]
  double* Y = Fd + kTB * (kTB + 1); // [64][m]
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int nblk = (n + kTB - 1) / kTB;

  auto load_block = [&](int i0, int nb) {
    for (int e = tid; e < kTB * kTB; e += blockDim.x) {
      const int r = e / kTB, c = e % kTB;
      Fd[r * (kTB + 1) + c] = (r < nb && c < nb) ? F[(long long)(i0 + r) * ldf + i0 + c] : 0.0;
    }
    for (int e = tid; e < kTB * m; e += blockDim.x) {
      const int r = e / m, c = e % m;
      Y[r * m + c] = (r < nb) ? __ldcg(X + (long long)(i0 + r) * ldx + c) : 0.0;
    }
    __syncthreads();
  };

  if (do_forward) {
    for (int b = 0; b < nblk; ++b) {
      const int i0 = b * kTB, nb = min(kTB, n - i0);
      load_block(i0, nb);
      for (int r = 0; r < nb; ++r) {
        for (int c = tid; c < m; c += blockDim.x) Y[r * m + c] = Y[r * m + c] / Fd[r * (kTB + 1) + r];
        __syncthreads();
        for (int e = tid; e < (nb - r - 1) * m; e += blockDim.x) {
          const int rr = r + 1 + e / m, c = e % m;
          Y[rr * m + c] = sub_rn(Y[rr * m + c], mul_rn(Fd[rr * (kTB + 1) + r], Y[r * m + c]));
        }
        __syncthreads();
      }
      if (blockIdx.x == 0)
        for (int e = tid; e < nb * m; e += blockDim.x) X[(long long)(i0 + e / m) * ldx + e % m] = Y[e];
      // trailing rows [i0+nb, n): contiguous slice per CTA, warp per row, lanes over RHS columns
      const int rows = n - (i0 + nb);
      const int per = (rows + gridDim.x - 1) / gridDim.x;
      const int rb = i0 + nb + blockIdx.x * per, re = min(n, rb + per);
      for (int r = rb + warp; r < re; r += nwarps) {
        const double* frow = F + (long long)r * ldf + i0;
        for (int c = lane; c < m; c += 32) {
          double s = 0.0;
          for (int q = 0; q < nb; ++q) s = add_rn(s, mul_rn(frow[q], Y[q * m + c]));
          X[(long long)r * ldx + c] = sub_rn(__ldcg(X + (long long)r * ldx + c), s);
        }
      }
      grid.sync();
    }
  }
  if (do_backward) {
    for (int b = nblk - 1; b >= 0; --b) {
      const int i0 = b * kTB, nb = min(kTB, n - i0);
      load_block(i0, nb);
      for (int r = nb - 1; r >= 0; --r) {
        for (int c = tid; c < m; c += blockDim.x) Y[r * m + c] = Y[r * m + c] / Fd[r * (kTB + 1) + r];
        __syncthreads();
        for (int e = tid; e < r * m; e += blockDim.x) {
          const int rr = e / m, c = e % m;
          Y[rr * m + c] = sub_rn(Y[rr * m + c], mul_rn(Fd[r * (kTB + 1) + rr], Y[r * m + c]));
        }
        __syncthreads();
      }
      if (blockIdx.x == 0)
        for (int e = tid; e < nb * m; e += blockDim.x) X[(long long)(i0 + e / m) * ldx + e % m] = Y[e];
      const int rows = i0;
      const int per = (rows + gridDim.x - 1) / gridDim.x;
      const int rb = blockIdx.x * per, re = min(i0, rb + per);
      for (int r = rb + warp; r < re; r += nwarps) {
        for (int c = lane; c < m; c += 32) {
          double s = 0.0;
          for (int q = 0; q < nb; ++q) s = add_rn(s, mul_rn(F[(long long)(i0 + q) * ldf + r], Y[q * m + c]));
          X[(long long)r * ldx + c] = sub_rn(__ldcg(X + (long long)r * ldx + c), s);
        }
      }
      grid.sync();
    }
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
cudaError_t launch_factor_setup(const double* G, long long ldg, int n, long long rows, double tol, int pivoting,
                                double* d, int* ord, FactorState* st, cudaStream_t s) {
  factor_setup_kernel<<<1, kPanelThreads, 0, s>>>(G, ldg, n, rows, tol, pivoting, d, ord, st);
  return cudaGetLastError();
}

size_t panel_smem_bytes(int nl, int R) {
  return size_t(kPanel) * R * sizeof(double) + size_t(R) * sizeof(double) + size_t(2) * nl * sizeof(int);
}

cudaError_t launch_panel(const PanelParams& p, int ctas, cudaStream_t s) {
  const int nl = p.n - p.k;
  const size_t smem = panel_smem_bytes(nl, p.rows_per_cta);
  cudaError_t e = cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  PanelParams pp = p;
  void* args[] = {&pp};
  return cudaLaunchCooperativeKernel((void*)panel_kernel, dim3(ctas), dim3(kPanelThreads), args, smem, s);
}

int panel_max_ctas(int nl, int R, int num_sms) {
  int per_sm = 0;
  const size_t smem = panel_smem_bytes(nl, R);
  cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panel_kernel, kPanelThreads, smem);
  return per_sm * num_sms;
}

cudaError_t launch_gather_factor(const double* Fo, long long ldf, const int* ord, int n, double* F, long long ldF,
                                 int num_sms, cudaStream_t s) {
  gather_factor_kernel<<<num_sms * 4, 256, 0, s>>>(Fo, ldf, ord, n, F, ldF);
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

cudaError_t launch_trsm_pair(const double* F, long long ldf, double* X, long long ldx, int n, int m, int fwd, int bwd,
                             int num_sms, cudaStream_t s) {
  const size_t smem = (size_t(kTB) * (kTB + 1) + size_t(kTB) * m) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(trsm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, trsm_pair_kernel, 256, smem);
  int blocks = num_sms * (per_sm > 0 ? 1 : 0);
  const int nblk = (n + kTB - 1) / kTB;
  // small systems need few CTAs (barrier cost grows with the grid)
  const int want = (n * m) / (4 * 1024) + 1;
  if (blocks > want) blocks = want;
  if (blocks < 1) blocks = 1;
  (void)nblk;
  void* args[] = {(void*)&F, (void*)&ldf, (void*)&X, (void*)&ldx, (void*)&n, (void*)&m, (void*)&fwd, (void*)&bwd};
  return cudaLaunchCooperativeKernel((void*)trsm_pair_kernel, dim3(blocks), dim3(256), args, smem, s);
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
