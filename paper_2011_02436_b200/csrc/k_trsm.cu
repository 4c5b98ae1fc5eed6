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
  double* Rb = sm;                 // [64][m]   right-hand side block
  double* Yb = Rb + kTB * m;       // [64][m]   block solution
  double* Ft = Yb + kTB * m;       // [64][kTB+1] F tile (forward: [32][65] rows x q; backward: [64][33])
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nblk = (n + kTB - 1) / kTB;

  for (int s = 0; s < nblk; ++s) {
    const int b = backward ? nblk - 1 - s : s;
    const int i0 = b * kTB, nb = min(kTB, n - i0);
    for (int e = tid; e < kTB * m; e += nt) {
      const int q = e / m, c = e - (e / m) * m;
      Rb[e] = q < nb ? __ldcg(X + (long long)(i0 + q) * ldx + c) : 0.0;
    }
    __syncthreads();
    const double* D = Dinv + (long long)b * kTB * kTB;
    for (int e = tid; e < nb * m; e += nt) {
      const int i = e / m, c = e - (e / m) * m;
      double acc = 0.0;
      if (!backward) {
        for (int q = 0; q <= i; ++q) acc = fma(__ldg(D + i * kTB + q), Rb[q * m + c], acc);
      } else {
        for (int q = i; q < nb; ++q) acc = fma(__ldg(D + q * kTB + i), Rb[q * m + c], acc);
      }
      Yb[e] = acc;
    }
    __syncthreads();
    if (blockIdx.x == b % gridDim.x)
      for (int e = tid; e < nb * m; e += nt) X[(long long)(i0 + e / m) * ldx + e % m] = Yb[e];

    // remaining rows: forward [i0+nb, n), backward [0, i0)
    const int rlo = backward ? 0 : i0 + nb;
    const int rhi = backward ? i0 : n;
    const int ntiles = (rhi - rlo + kTR - 1) / kTR;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int r0 = rlo + t * kTR, nr = min(kTR, rhi - r0);
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
      __syncthreads();
      for (int e = tid; e < nr * m; e += nt) {
        const int rr = e / m, c = e - (e / m) * m;
        const double* fr = Ft + rr * (kTB + 1);
        double acc = 0.0;
#pragma unroll 8
        for (int q = 0; q < kTB; ++q) acc = fma(fr[q], Yb[q * m + c], acc);
        double* xp = X + (long long)(r0 + rr) * ldx + c;
        *xp = __ldcg(xp) - acc;
      }
      __syncthreads();
    }
    grid.sync();
  }
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
  const size_t smem = (size_t(2) * kTB * m + size_t(kTB) * (kTB + 1)) * sizeof(double);
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
