// K4: the two triangular solves of solve_factored_gram / SpdFactor::solve
// (reference linalg.cpp:254-270, 141-151): F y = b, then F^T x = y, for an n x n
// lower factor F and an n x m right-hand side (m <= 128 per launch).
//
// Structure (latency-bound problem: n/64 strictly sequential block steps):
//   tri_inv_kernel   : the 64x64 diagonal blocks of F are inverted once, all blocks
//                      in parallel (one CTA each), so a block step is a small product
//                      instead of 64 dependent substitution steps.
//   trsm_sweep_kernel: cooperative; per block step every CTA forms the block solution
//                      Y_b = D_b^{-1} R_b (forward) or D_b^{-T} R_b (backward) in shared
//                      memory, CTA (b mod C) stores it, and all CTAs update their share of
//                      the remaining rows from 32-row F tiles staged in shared memory
//                      (coalesced 512-byte row segments); one grid barrier per block.
#include "common.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>

#include <algorithm>

namespace cg = cooperative_groups;

namespace rbpg {

constexpr int kTB = 64;    // diagonal block
constexpr int kTR = 32;    // update row tile

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

__global__ void __launch_bounds__(256) trsm_sweep_kernel(const double* F, long long ldf, const double* Dinv, double* X,
                                                         long long ldx, int n, int m, int backward) {
  extern __shared__ __align__(16) double sm[];
  double* Rb = sm;                      // [64][m]      right-hand side block
  double* Yb = Rb + kTB * m;            // [64][m]      block solution
  double* Ds = Yb + kTB * m;            // [64][65]     diagonal-block inverse
  double* Ft = Ds + kTB * (kTB + 1);    // [32][65]     F tile of the row update
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nblk = (n + kTB - 1) / kTB;

  auto load_tile = [&](int i0, int nb, int r0, int nr) {
    if (!backward) {
      for (int e = tid; e < kTR * kTB; e += nt) {
        const int rr = e / kTB, q = e % kTB;
        Ft[rr * (kTB + 1) + q] = (rr < nr && q < nb) ? __ldg(F + (long long)(r0 + rr) * ldf + i0 + q) : 0.0;
      }
    } else {
      for (int e = tid; e < kTR * kTB; e += nt) {
        const int q = e / kTR, rr = e % kTR;
        Ft[rr * (kTB + 1) + q] = (rr < nr && q < nb) ? __ldg(F + (long long)(i0 + q) * ldf + r0 + rr) : 0.0;
      }
    }
  };

  // The owner stores block b's solution only after the step's grid barrier (deferred to the
  // start of step s+1): every CTA reads block b's right-hand side from X during step s.
  auto store_solution = [&](int bb) {
    const int j0 = bb * kTB, jb = min(kTB, n - j0);
    for (int e = tid; e < jb * m; e += nt) X[(long long)(j0 + e / m) * ldx + e % m] = Yb[e];
  };
  for (int s = 0; s < nblk; ++s) {
    const int b = backward ? nblk - 1 - s : s;
    if (s > 0) {
      const int bp = backward ? b + 1 : b - 1;
      if (blockIdx.x == bp % gridDim.x) store_solution(bp);
    }
    const int i0 = b * kTB, nb = min(kTB, n - i0);
    const int rlo = backward ? 0 : i0 + nb;  // rows updated by this block: forward [i0+nb, n), backward [0, i0)
    const int rhi = backward ? i0 : n;
    const int ntiles = (rhi - rlo + kTR - 1) / kTR;
    // all loads of the step issued together: D_b, R_b and the first F tile
    const double* D = Dinv + (long long)b * kTB * kTB;
    for (int e = tid; e < kTB * kTB; e += nt) Ds[(e / kTB) * (kTB + 1) + e % kTB] = __ldg(D + e);
    for (int e = tid; e < kTB * m; e += nt) {
      const int q = e / m, c = e - q * m;
      Rb[e] = q < nb ? __ldcg(X + (long long)(i0 + q) * ldx + c) : 0.0;
    }
    if (blockIdx.x < ntiles) load_tile(i0, nb, rlo + blockIdx.x * kTR, min(kTR, rhi - (rlo + blockIdx.x * kTR)));
    __syncthreads();
    for (int e = tid; e < nb * m; e += nt) {
      const int i = e / m, c = e - i * m;
      double acc = 0.0;
      if (!backward) {
        for (int q = 0; q <= i; ++q) acc = fma(Ds[i * (kTB + 1) + q], Rb[q * m + c], acc);
      } else {
        for (int q = i; q < nb; ++q) acc = fma(Ds[q * (kTB + 1) + i], Rb[q * m + c], acc);
      }
      Yb[e] = acc;
    }
    __syncthreads();

    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int r0 = rlo + t * kTR, nr = min(kTR, rhi - r0);
      if (t != blockIdx.x) {
        __syncthreads();
        load_tile(i0, nb, r0, nr);
        __syncthreads();
      }
      for (int e = tid; e < nr * m; e += nt) {
        const int rr = e / m, c = e - rr * m;
        const double* fr = Ft + rr * (kTB + 1);
        double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
        for (int q = 0; q < kTB; q += 2) {
          a0 = fma(fr[q], Yb[q * m + c], a0);
          a1 = fma(fr[q + 1], Yb[(q + 1) * m + c], a1);
        }
        double* xp = X + (long long)(r0 + rr) * ldx + c;
        *xp = __ldcg(xp) - (a0 + a1);
      }
    }
    grid.sync();
  }
  const int blast = backward ? 0 : nblk - 1;
  if (nblk > 0 && blockIdx.x == blast % gridDim.x) store_solution(blast);
}

// ---------------------------------------------------------------------------
cudaError_t launch_trsm_pair(const double* F, long long ldf, double* X, long long ldx, int n, int m, int fwd, int bwd,
                             int num_sms, double* dinv_ws, cudaStream_t s) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  const int nblk = (n + kTB - 1) / kTB;
  constexpr size_t kInvSmem = size_t(2) * kTB * (kTB + 1) * sizeof(double);
  static bool inv_attr = false;
  if (!inv_attr) {
    cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kInvSmem);
    inv_attr = true;
  }
  tri_inv_kernel<<<nblk, kTB, kInvSmem, s>>>(F, ldf, n, dinv_ws);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t smem = (size_t(2) * kTB * m + size_t(kTB + kTR) * (kTB + 1)) * sizeof(double);
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    e = cudaFuncSetAttribute(trsm_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_smem = smem;
  }
  int blocks = std::min(num_sms, std::max(1, (n + kTB - 1) / kTB));
  const double* Dc = dinv_ws;
  for (int dir = 0; dir < 2; ++dir) {
    if ((dir == 0 && !fwd) || (dir == 1 && !bwd)) continue;
    int backward = dir;
    void* args[] = {(void*)&F, (void*)&ldf, (void*)&Dc, (void*)&X, (void*)&ldx, (void*)&n, (void*)&m, (void*)&backward};
    e = cudaLaunchCooperativeKernel((void*)trsm_sweep_kernel, dim3(blocks), dim3(256), args, smem, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rbpg
