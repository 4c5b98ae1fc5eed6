// Bitwise check of oz_slice_kernel (bias-and-transpose digits) against the digit loop it replaced.
#include "../paper_2011_02436_b200/csrc/k_ozaki.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
namespace rbpg {
cudaError_t ensure_attrs(const void* fn, size_t smem, bool) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}
}
using namespace rbpg;
__global__ void old_slice(const double* A, long long lda, long long N, int M, const int* exps, int8_t* S,
                          long long ps, int Mpad, long long Npad) {
  const int groups = Mpad / 8;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < Npad * groups; it += (long long)gridDim.x * blockDim.x) {
    const long long r = it / groups;
    const int c0 = (int)(it - r * groups) * 8;
    unsigned long long w[7] = {0, 0, 0, 0, 0, 0, 0};
    if (r < N)
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + q;
        long long X = 0;
        if (c < M) X = __double2ll_rn(ldexp(A[r * lda + c], 54 - exps[c]));
        for (int p = 6; p >= 1; --p) {
          const long long dgt = ((X + 128) & 255) - 128;
          X = (X - dgt) >> 8;
          w[p] |= ((unsigned long long)dgt & 255ull) << (8 * q);
        }
        w[0] |= ((unsigned long long)X & 255ull) << (8 * q);
      }
    for (int p = 0; p < 7; ++p) *(unsigned long long*)(S + p * ps + r * Mpad + c0) = w[p];
  }
}
int main() {
  const long long N = 3001; const int M = 203, Mpad = 256; const long long Npad = 3008, lda = 204;
  std::vector<double> a(N * lda, 0.0);
  srand(5);
  for (long long r = 0; r < N; ++r)
    for (int c = 0; c < M; ++c) {
      double u = (rand() + 0.5) / (RAND_MAX + 1.0) - 0.3;
      int sc = (c % 11) * 37 - 150;
      if (c == 7) sc = -1060;  // tiny column: 54 - e > 1023
      if (c == 9) sc = 900;    // huge column: 54 - e < 0
      a[r * lda + c] = ldexp(u, sc) * ((r % 5 == 0) ? 1e-9 : 1.0);
      if (c == 3) a[r * lda + c] = 0.0;
    }
  double* dA; unsigned long long* cmax; int* exps; int8_t *S1, *S2;
  cudaMalloc(&dA, 8 * N * lda); cudaMalloc(&cmax, 8 * M); cudaMalloc(&exps, 4 * Mpad);
  cudaMalloc(&S1, 7 * Mpad * Npad); cudaMalloc(&S2, 7 * Mpad * Npad);
  cudaMemcpy(dA, a.data(), 8 * N * lda, cudaMemcpyHostToDevice);
  launch_oz_colmax(dA, lda, N, M, cmax, 148, 0);
  launch_oz_slice(dA, lda, N, M, cmax, exps, Mpad, Npad, S1, 0);
  old_slice<<<256, 256>>>(dA, lda, N, M, exps, S2, (long long)Mpad * Npad, Mpad, Npad);
  cudaDeviceSynchronize();
  std::vector<int8_t> h1(7 * Mpad * Npad), h2(7 * Mpad * Npad);
  cudaMemcpy(h1.data(), S1, h1.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), S2, h2.size(), cudaMemcpyDeviceToHost);
  long long diff = 0;
  for (size_t i = 0; i < h1.size(); ++i) diff += h1[i] != h2[i];
  printf("slice_check: %lld differing plane bytes of %zu (%s)\n", diff, h1.size(), cudaGetErrorString(cudaGetLastError()));
  return diff != 0;
}
