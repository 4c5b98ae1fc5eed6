// K4: the two triangular solves of solve_factored_gram / SpdFactor::solve
// (reference linalg.cpp:254-270, 141-151): F y = b, then F^T x = y, for an n x n
// lower factor F and an n x m right-hand side (m <= 128 per launch).
//
// Structure (latency-bound problem: n/64 strictly sequential block steps):
//   tri_inv_kernel   : the 64x64 diagonal blocks of F are inverted once, all blocks
//                      in parallel (one CTA each), so a block step is a small product
//                      instead of 64 dependent substitution steps.
//   trsm_cluster_kernel: m <= 32 right-hand sides, one thread-block cluster, block solutions
//                      pushed between CTAs over distributed shared memory (below);
//   trsm_step_kernel : any m, one launch per 64-row block step (engine trsm_blocked_dev).
#include "common.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>

namespace cg = cooperative_groups;

namespace rbpg {

constexpr int kTB = 64;    // diagonal block

__global__ void __launch_bounds__(64) tri_inv_kernel(const double* F, long long ldf, int n, double* Dinv) {
  extern __shared__ __align__(16) double tsm[];
  double(*Fs)[kTB + 1] = reinterpret_cast<double(*)[kTB + 1]>(tsm);
  double(*Zs)[kTB + 1] = reinterpret_cast<double(*)[kTB + 1]>(tsm + kTB * (kTB + 1));
  const int b = blockIdx.x, i0 = b * kTB, nb = min(kTB, n - i0);
  const int j = threadIdx.x;
  for (int r = 0; r < kTB; ++r) {
    Fs[r][j] = (r < nb && j < nb && j <= r) ? F[(long long)(i0 + r) * ldf + i0 + j] : 0.0;
    Zs[r][j] = 0.0;
  }
  __syncthreads();
  // column j of the inverse: forward substitution on e_j
  if (j < nb) {
    Zs[j][j] = 1.0 / Fs[j][j];
    for (int i = j + 1; i < nb; ++i) {
      double s = 0.0;
      for (int c = j; c < i; ++c) s = fma(Fs[i][c], Zs[c][j], s);
      Zs[i][j] = -s / Fs[i][i];
    }
  }
  __syncthreads();
  double* D = Dinv + (long long)b * kTB * kTB;
  for (int r = 0; r < kTB; ++r) D[r * kTB + j] = Zs[r][j];
}

// ---------------------------------------------------------------------------
// Cluster variant for small right-hand sides (m <= 32, all owned rows fit in shared memory):
// one thread-block cluster; 64-row block b is owned by CTA b % CL, which alone updates and
// solves it.  The only exchange is the block solution Y_b, pushed by its owner into every
// CTA's ring buffer with st.async (bytes complete on the receiver's mbarrier) -- no grid
// barrier.  A cluster barrier every kSyncEvery steps bounds the skew below the ring depth.
// ---------------------------------------------------------------------------
constexpr int kRing = 8;
constexpr int kSyncEvery = 4;
constexpr int kClusterMaxM = 32;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc), "r"(src_bytes)
               : "memory");
}

constexpr int kPadT = kTB + 2;  // 16-byte aligned padded tile rows

// 64 x 64 block of F starting at (row0, col0) into T[64][kPadT] by cp.async; rows >= nrows and
// columns >= ncols are zero-filled (F beyond n is never read: ld padding holds garbage).
__device__ __forceinline__ void load_tile_async(double* T, const double* F, long long ldf, int row0, int nrows,
                                                int col0, int ncols, int tid, int nt) {
  for (int e = tid; e < kTB * (kTB / 2); e += nt) {
    const int r = e / (kTB / 2), ch = e % (kTB / 2);
    const int c = 2 * ch;
    uint32_t bytes = 0;
    if (r < nrows && c < ncols) bytes = (c + 1 < ncols) ? 16u : 8u;
    const double* src = bytes ? F + (long long)(row0 + r) * ldf + col0 + c : F;
    cp_async16(T + r * kPadT + c, src, bytes);
  }
}

// C[64][m] = A * B  (or C -= A * B), A 64x64 with A(r, k) = aT ? A[k*lda + r] : A[r*lda + k],
// B 64 x m row-major (ld m), on FP64 tensor cores: one (m16, n8) output tile per warp pass,
// two interleaved accumulator chains over K = 64.
__device__ __forceinline__ void mma64(const double* A, int lda, bool aT, const double* B, int m, double* Cm,
                                      bool subtract, int tid) {
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int nt8 = (m + 7) / 8;
  for (int tile = warp; tile < 4 * nt8; tile += 8) {
    const int m0 = (tile / nt8) * 16, n0 = (tile % nt8) * 8;
    double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
    const int col = n0 + g;
#pragma unroll 4
    for (int k0 = 0; k0 < kTB; k0 += 8) {
      const int ka = k0 + t, kb = k0 + 4 + t;
      const double a0 = aT ? A[ka * lda + m0 + g] : A[(m0 + g) * lda + ka];
      const double a1 = aT ? A[ka * lda + m0 + g + 8] : A[(m0 + g + 8) * lda + ka];
      const double b0 = col < m ? B[ka * m + col] : 0.0;
      const double a2 = aT ? A[kb * lda + m0 + g] : A[(m0 + g) * lda + kb];
      const double a3 = aT ? A[kb * lda + m0 + g + 8] : A[(m0 + g + 8) * lda + kb];
      const double b1 = col < m ? B[kb * m + col] : 0.0;
      dmma_16x8x4(c0, a0, a1, b0);
      dmma_16x8x4(c1, a2, a3, b1);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = m0 + g + 8 * h;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int cc = n0 + 2 * t + q;
        if (cc >= m) continue;
        const double v = c0[2 * h + q] + c1[2 * h + q];
        if (subtract)
          Cm[r * m + cc] -= v;
        else
          Cm[r * m + cc] = v;
      }
    }
  }
}

// Inverse of the lower-triangular 64 x 64 tile T (rows/cols >= nb zero) into Dinv (64 x 64, row-major).
// Column j is a forward substitution on e_j, shared by the two threads (j, h) of a lane pair: thread h
// keeps the partial sums of rows 32h..32h+31 in registers; the owner of row c forms z_c and passes it
// to its partner.  Same operation order as tri_inv_kernel (s_i accumulates F[i][c] z_c over
// increasing c by fma; z_i = -s_i / F[i][i], z_j = 1 / F[j][j]).
__device__ __forceinline__ void invert_tile(const double* T, int nb, double* Dinv, int tid) {
  if (tid >= 2 * kTB) return;  // warps 0-3, fully active (shuffles)
  const int j = tid >> 1, h = tid & 1, lane = tid & 31;
  const double* Th = T + h * 32 * kPadT;
  double sacc[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) sacc[r] = 0.0;
#pragma unroll
  for (int c = 0; c < kTB; ++c) {
    const double zl = ((c == j ? 1.0 : 0.0) - sacc[c & 31]) / T[c * kPadT + c];
    const double z0 = __shfl_sync(0xffffffffu, zl, (lane & ~1) | (c >> 5));
    const double z = (c >= j && c < nb) ? z0 : 0.0;
    if (h == (c >> 5)) Dinv[c * kTB + j] = z;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (h * 32 + r > c) sacc[r] = fma(Th[r * kPadT + c], z, sacc[r]);
  }
}

// Steps [s_begin, s_end) of the 2 * nblk block steps: forward steps s < nblk solve block s, backward
// steps s >= nblk solve block 2 * nblk - 1 - s (s_begin = nblk: backward substitution only, the
// right-hand side already forward-solved -- e.g. by the augmented factorisation).
__global__ void __launch_bounds__(256, 1) trsm_cluster_kernel(const double* F, long long ldf, double* Dinv,
                                                              double* X, long long ldx, int n, int m, int s_begin,
                                                              int s_end) {
  extern __shared__ __align__(16) double csm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), cta = static_cast<int>(cl.block_rank());
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nblk = (n + kTB - 1) / kTB;
  const int nown = (nblk - cta + C - 1) / C;  // owned blocks: cta, cta + C, ...
  const int nown_max = (nblk + C - 1) / C;   // identical layout in every CTA (remote addresses)
  double* Rown = csm;                                 // [nown_max][64][m]  rhs -> solutions
  double* Ring = Rown + (size_t)nown_max * kTB * m;   // [kRing][64][m] block solutions
  double* Ds = Ring + kRing * kTB * m;                // [2][64][kPadT] diagonal-block inverses
  double* Tc = Ds + 2 * kTB * kPadT;                  // [64][kPadT] critical F tile (prefetched)
  double* To = Tc + kTB * kPadT;                      // [64][kPadT] other F tiles
  __shared__ __align__(8) uint64_t rbar[kRing];
  if (tid < kRing) mbar_init(&rbar[tid], 1);
  if (tid == 0) fence_mbar_init();
  for (int e = tid; e < nown * kTB * m; e += nt) {
    const int ob = e / (kTB * m), rem = e % (kTB * m), q = rem / m, c = rem % m;
    const int row = (cta + ob * C) * kTB + q;
    Rown[e] = row < n ? X[(long long)row * ldx + c] : 0.0;
  }
  // inverses of the owned diagonal blocks (only the owner ever reads them), first-needed first
  for (int oi = 0; oi < nown; ++oi) {
    const int ob = s_begin == 0 ? oi : nown - 1 - oi;
    const int b = cta + ob * C, nb = min(kTB, n - b * kTB);
    load_tile_async(To, F, ldf, b * kTB, nb, b * kTB, nb, tid, nt);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    invert_tile(To, nb, Dinv + (long long)b * kTB * kTB, tid);
    __syncthreads();
  }
  cl.sync();
  const uint32_t ybytes = static_cast<uint32_t>(kTB * m * sizeof(double));
  auto block_of = [&](int s) { return s < nblk ? s : 2 * nblk - 1 - s; };
  auto owns = [&](int b) { return b % C == cta; };

  // Y_s = D_b^{-1} R_b (forward steps) or D_b^{-T} R_b (backward), pushed to every CTA's ring slot
  auto solve_and_push = [&](int s, const double* D) {
    const bool bwd = s >= nblk;
    const int b = block_of(s);
    double* Rb = Rown + (size_t)(b / C) * kTB * m;
    const int slot = (s - s_begin) % kRing;
    double* Y = Ring + slot * kTB * m;
    mma64(D, kPadT, bwd, Rb, m, Y, false, tid);
    __syncthreads();
    const uint32_t yl = smem_u32(Y), bl = smem_u32(&rbar[slot]);
    if (tid < C - 1) {
      // one bulk DSMEM copy per destination (TMA engine), issued by C - 1 threads in parallel and
      // in step order: the owner of the next block (the critical consumer) is served first
      const int d = bwd ? (cta - 1 - tid + 2 * C) % C : (cta + 1 + tid) % C;
      fence_proxy_async();
      bulk_wait_read0();  // this thread's earlier push has finished reading its ring slot
      bulk_s2s_cluster(mapa_u32(yl, d), yl, ybytes, mapa_u32(bl, d));
      bulk_commit();
    }
    if (tid == 32)  // the own copy was written in place
      asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;\n" ::"r"(bl), "r"(ybytes) : "memory");
    for (int e = tid; e < kTB * m; e += nt) Rb[e] = Y[e];  // the block's solution
  };
  // R_bp -= F-tile * Y (forward: tile = F[bp rows][b cols]; backward: tile = F[b rows][bp cols]^T)
  auto update = [&](int bp, const double* T, bool bwd, const double* Yb) {
    double* Rp = Rown + (size_t)(bp / C) * kTB * m;
    mma64(T, kPadT, bwd, Yb, m, Rp, true, tid);
  };
  auto issue_tile = [&](double* T, int b, int bp, bool bwd) {
    if (!bwd) load_tile_async(T, F, ldf, bp * kTB, min(kTB, n - bp * kTB), b * kTB, min(kTB, n - b * kTB), tid, nt);
    else load_tile_async(T, F, ldf, b * kTB, min(kTB, n - b * kTB), bp * kTB, min(kTB, n - bp * kTB), tid, nt);
  };
  auto issue_dinv = [&](double* D, int b) {
    const double* src = Dinv + (long long)b * kTB * kTB;
    for (int e = tid; e < kTB * (kTB / 2); e += nt) {
      const int r = e / (kTB / 2), c = 2 * (e % (kTB / 2));
      cp_async16(D + r * kPadT + c, src + r * kTB + c, 16u);
    }
  };

  // the first step's solution needs no update
  if (owns(block_of(s_begin))) {
    issue_dinv(Ds, block_of(s_begin));
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
  }
  if (tid < kRing && tid == 0) mbar_arrive_expect_tx(&rbar[0], ybytes);
  __syncthreads();
  if (owns(block_of(s_begin))) solve_and_push(s_begin, Ds);

  for (int s = s_begin; s < s_end; ++s) {
    const int u = s - s_begin;
    const bool bwd = s >= nblk;
    const int b = block_of(s);
    const int slot = u % kRing;
    const bool last = s + 1 == s_end;
    const int bn = last ? -1 : block_of(s + 1);
    const bool bwd_n = s + 1 >= nblk;
    // does the next step's block need this step's Y? (not at the forward -> backward turn)
    const bool crit = !last && owns(bn) && (bwd ? bn < b : bn > b) && bwd_n == bwd;
    // prefetch (independent of Y_s): the critical tile, the first non-critical tile and the
    // next diagonal inverse
    if (crit) issue_tile(Tc, b, bn, bwd);
    int first_other = -1;
    for (int ob = 0; ob < nown; ++ob) {
      const int bp = cta + ob * C;
      if ((bwd ? bp >= b : bp <= b) || (crit && bp == bn)) continue;
      first_other = bp;
      break;
    }
    if (first_other >= 0) issue_tile(To, b, first_other, bwd);
    if (!last && owns(bn)) issue_dinv(Ds + ((u + 1) & 1) * kTB * kPadT, bn);
    cp_async_commit();
    if (!last && tid == 0) mbar_arrive_expect_tx(&rbar[(u + 1) % kRing], ybytes);
    if ((u + 1) % kSyncEvery == 0) cl.sync();  // skew < kRing steps
    mbar_wait(&rbar[slot], (u / kRing) & 1);
    const double* Yb = Ring + slot * kTB * m;
    cp_async_wait_all();
    __syncthreads();
    if (!last && owns(bn)) {  // critical path: update the next block, solve it, push
      if (crit) update(bn, Tc, bwd, Yb);
      __syncthreads();
      solve_and_push(s + 1, Ds + ((u + 1) & 1) * kTB * kPadT);
    }
    for (int ob = 0; ob < nown; ++ob) {  // remaining updates off the critical path

      const int bp = cta + ob * C;
      if (bwd ? bp >= b : bp <= b) continue;
      if (crit && bp == bn) continue;
      if (bp != first_other) {  // prefetched above otherwise
        __syncthreads();
        issue_tile(To, b, bp, bwd);
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
      }
      update(bp, To, bwd, Yb);
    }
    __syncthreads();
  }
  cl.sync();  // no CTA exits while remote stores may still target it
  for (int e = tid; e < nown * kTB * m; e += nt) {
    const int ob = e / (kTB * m), rem = e % (kTB * m), q = rem / m, c = rem % m;
    const int row = (cta + ob * C) * kTB + q;
    if (row < n) X[(long long)row * ldx + c] = Rown[e];
  }
}

static size_t trsm_cluster_smem(int n, int m, int C) {
  const int nblk = (n + kTB - 1) / kTB;
  const int nown = (nblk + C - 1) / C;
  return (size_t(nown) * kTB * m + size_t(kRing) * kTB * m + 4 * size_t(kTB) * kPadT) * sizeof(double);
}

// One block step of the blocked TRSM pair (engine trsm_blocked_dev), fused: every CTA forms the
// block solution W = op(D_b) S_b for its NC-column slice (D_b = inverse of the 64 x 64 diagonal
// block, op = transpose on the backward sweep; recomputed per CTA instead of a second launch), then
// row-tile CTAs apply the rank-64 update of the rows still to solve,
//   backward: src[R, :] -= F[r0 : r0+nb, R]^T W      (R in [0, r0))
//   forward:  src[R, :] -= F[R, r0 : r0+nb] W        (R in [r0+nb, n))
// and CTA row 0 stores W into dst[r0 : r0+nb, :].  Grid (ceil(m/NC), 1 + row tiles of 64), 256
// threads; NC = 128 for m > 64 keeps the grid to one wave at n = 8192.
template <int NC>
__global__ void __launch_bounds__(256) trsm_step_kernel(const double* __restrict__ F, long long ldf,
                                                        const double* __restrict__ Db, double* src, long long lds,
                                                        double* dst, long long ldd, int n, int m, int r0, int nb,
                                                        int bwd) {
  constexpr int SP = NC + 2, DP = 66;   // padded smem rows (doubles)
  constexpr int NF = NC / 16;           // n8 fragments per warp (warp tile 16 x NC/2)
  constexpr int NE = 64 * NC / 256;     // S / W elements per thread
  extern __shared__ __align__(16) double tsm[];
  double(*S)[SP] = reinterpret_cast<double(*)[SP]>(tsm);                  // S_b slice [k][c]
  double(*Wt)[SP] = reinterpret_cast<double(*)[SP]>(tsm + 64 * SP);       // W [k][c]
  double(*D)[DP] = reinterpret_cast<double(*)[DP]>(tsm + 128 * SP);       // D_b [row][col]
  double(*A)[DP] = reinterpret_cast<double(*)[DP]>(tsm + 128 * SP + 64 * DP);  // A(i, k) at [k][i]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int j0 = blockIdx.x * NC, y = blockIdx.y;
  const int R0 = bwd ? (y - 1) * 64 : r0 + nb + (y - 1) * 64;
  const int Rend = bwd ? r0 : n;
  // every load of this thread in flight at once (a load-store loop would serialise the round trips)
  double sv[NE], dv[16], av[16];
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = tid + 256 * i, r = e / NC, c = e % NC;
    sv[i] = (r < nb && j0 + c < m) ? src[(long long)(r0 + r) * lds + j0 + c] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = tid + 256 * i, r = e >> 6, c = e & 63;
    dv[i] = (r < nb && c < nb) ? Db[r * 64 + c] : 0.0;
    av[i] = 0.0;
    if (y > 0) {  // bwd: A(i, k) = F[r0 + k][R0 + i] (coalesced in i); fwd: A(i, k) = F[R0 + i][r0 + k]
      if (bwd) {
        if (r < nb && R0 + c < Rend) av[i] = F[(long long)(r0 + r) * ldf + R0 + c];
      } else {
        if (c < nb && R0 + r < Rend) av[i] = F[(long long)(R0 + r) * ldf + r0 + c];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NE; ++i) {
    const int e = tid + 256 * i;
    S[e / NC][e % NC] = sv[i];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int e = tid + 256 * i, r = e >> 6, c = e & 63;
    D[r][c] = dv[i];
    if (bwd) A[r][c] = av[i]; else A[c][r] = av[i];
  }
  __syncthreads();
  // warp tile: rows 16 * (warp & 3) .. +16, cols (NC / 2) * (warp >> 2) .. + NC / 2
  const int wi = 16 * (warp & 3), wc = (NC / 2) * (warp >> 2);
  double acc[NF][4];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[f][q] = 0.0;
#pragma unroll 4
  for (int k = 0; k < 64; k += 4) {
    // W(i, c) = sum_k op(D)(i, k) S[k][c]; op(D)(i, k) = D[k][i] (bwd) or D[i][k] (fwd)
    const double a0 = bwd ? D[k + t][wi + g] : D[wi + g][k + t];
    const double a1 = bwd ? D[k + t][wi + g + 8] : D[wi + g + 8][k + t];
#pragma unroll
    for (int f = 0; f < NF; ++f) dmma_16x8x4(acc[f], a0, a1, S[k + t][wc + 8 * f + g]);
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int c = wc + 8 * f + 2 * t;
    Wt[wi + g][c] = acc[f][0];
    Wt[wi + g][c + 1] = acc[f][1];
    Wt[wi + g + 8][c] = acc[f][2];
    Wt[wi + g + 8][c + 1] = acc[f][3];
  }
  __syncthreads();
  if (y == 0) {
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = tid + 256 * i, r = e / NC, c = e % NC;
      if (r < nb && j0 + c < m) dst[(long long)(r0 + r) * ldd + j0 + c] = Wt[r][c];
    }
    return;
  }
  // read every old value first (the stores could alias later loads as far as the compiler knows);
  // the loads fly under the update DMMAs
  double old[NF][4];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int c = j0 + wc + 8 * f + 2 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = R0 + wi + g + 8 * h;
      const double* row = src + (long long)r * lds;
      old[f][2 * h] = (r < Rend && c < m) ? row[c] : 0.0;
      old[f][2 * h + 1] = (r < Rend && c + 1 < m) ? row[c + 1] : 0.0;
    }
  }
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[f][q] = 0.0;
#pragma unroll 4
  for (int k = 0; k < 64; k += 4) {
    const double a0 = A[k + t][wi + g], a1 = A[k + t][wi + g + 8];
#pragma unroll
    for (int f = 0; f < NF; ++f) dmma_16x8x4(acc[f], a0, a1, Wt[k + t][wc + 8 * f + g]);
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int c = j0 + wc + 8 * f + 2 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = R0 + wi + g + 8 * h;
      if (r >= Rend) continue;
      double* row = src + (long long)r * lds;
      if (c < m) row[c] = old[f][2 * h] - acc[f][2 * h];
      if (c + 1 < m) row[c + 1] = old[f][2 * h + 1] - acc[f][2 * h + 1];
    }
  }
}

cudaError_t launch_trsm_step(const double* F, long long ldf, const double* Db, double* src, long long lds,
                             double* dst, long long ldd, int n, int m, int r0, int nb, int bwd, cudaStream_t s) {
  const int rows = bwd ? r0 : n - r0 - nb;
  constexpr int kNC = 32;  // columns per CTA (measured best at C5's m = 100 against 64 / 128)
  const size_t smem = (size_t(128) * (kNC + 2) + size_t(128) * 66) * sizeof(double);
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(trsm_step_kernel<kNC>), smem);
  if (e != cudaSuccess) return e;
  dim3 grid((m + kNC - 1) / kNC, 1 + (rows + 63) / 64);
  trsm_step_kernel<kNC><<<grid, 256, smem, s>>>(F, ldf, Db, src, lds, dst, ldd, n, m, r0, nb, bwd);
  return cudaGetLastError();
}

// The 64 x 64 diagonal-block inverses of F (blocked TRSM path of the engine).
cudaError_t launch_tri_inv(const double* F, long long ldf, int n, double* dinv, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  constexpr size_t kInvSmem = size_t(2) * kTB * (kTB + 1) * sizeof(double);
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(tri_inv_kernel), kInvSmem);
  if (e != cudaSuccess) return e;
  tri_inv_kernel<<<(n + kTB - 1) / kTB, kTB, kInvSmem, s>>>(F, ldf, n, dinv);
  return cudaGetLastError();
}

// Whether launch_trsm_pair runs its cluster kernel for n rows and m right-hand sides.
bool trsm_cluster_fits(int n, int m) {
  if (m > kClusterMaxM) return false;
  const int nblk = (n + kTB - 1) / kTB;
  return trsm_cluster_smem(n, m, std::min(16, nblk)) <= 220 * 1024;
}

// Cluster TRSM pair (the caller checks trsm_cluster_fits; larger problems go through the blocked
// step kernels).  The cluster kernel inverts its diagonal blocks itself into dinv_ws.
cudaError_t launch_trsm_pair(const double* F, long long ldf, double* X, long long ldx, int n, int m, int fwd, int bwd,
                             int num_sms, double* dinv_ws, cudaStream_t s) {
  (void)num_sms;
  if (n <= 0 || m <= 0 || !(fwd || bwd)) return cudaSuccess;
  if (!trsm_cluster_fits(n, m)) return cudaErrorInvalidValue;
  const int nblk = (n + kTB - 1) / kTB;
  const int C = std::min(16, nblk);
  const size_t csmem = trsm_cluster_smem(n, m, C);
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(trsm_cluster_kernel), csmem, true);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = csmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int s_begin = fwd ? 0 : nblk, s_end = bwd ? 2 * nblk : nblk;
  return cudaLaunchKernelEx(&cfg, trsm_cluster_kernel, F, ldf, dinv_ws, X, ldx, n, m, s_begin, s_end);
}

}  // namespace rbpg
