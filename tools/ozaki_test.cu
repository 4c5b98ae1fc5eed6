// Standalone check and timing of the INT8 (Ozaki-I) Gram kernel (csrc/k_ozaki.cu).
//   ozaki_test check N M      : random [0,1) sigmoid-like columns (+ one-hot, zero and twin columns),
//                               Gram vs a long-double CPU reference
//   ozaki_test time N M reps  : device-generated columns, kernel timing only
#include "../paper_2011_02436_b200/csrc/k_ozaki.cu"
constexpr long long kOzChunkRows = 16384;

#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <map>
#include <chrono>
#include <string>

namespace rbpg {
cudaError_t ensure_attrs(const void* fn, size_t smem, bool) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}
}
using namespace rbpg;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void gen_kernel(double* H, long long N, int M, long long ld, unsigned long long seed) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = N * (long long)M;
  for (; i < tot; i += (long long)gridDim.x * blockDim.x) {
    long long r = i / M; int c = (int)(i % M);
    unsigned long long z = (unsigned long long)(r * 1000003 + c) * 0x9E3779B97F4A7C15ull + seed;
    z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29; z *= 0x94D049BB133111EBull; z ^= z >> 32;
    double u = (z >> 11) * 0x1.0p-53;
    double zz = (u - 0.5) * 12.0 + 0.37 * (c % 17) - 3.0;
    H[r * ld + c] = 1.0 / (1.0 + exp(-zz));
  }
}

int main(int argc, char** argv) {
  const bool check = argc > 1 && std::string(argv[1]) == "check";
  const long long N = argc > 2 ? atoll(argv[2]) : 5000;
  const int M = argc > 3 ? atoi(argv[3]) : 300;
  const int reps = argc > 4 ? atoi(argv[4]) : 3;
  const int splits_arg = argc > 5 ? atoi(argv[5]) : 0;
  const long long ld = (M + 1) & ~1;
  double* dH;
  CK(cudaMalloc(&dH, sizeof(double) * N * ld));
  std::vector<double> H;
  if (check) {
    H.assign(N * ld, 0.0);
    srand(7);
    for (long long r = 0; r < N; ++r)
      for (int c = 0; c < M; ++c) {
        double u = (rand() + 0.5) / (RAND_MAX + 1.0);
        double zz = (u - 0.5) * 10.0 + 0.5 * (c % 13) - 4.0;
        H[r * ld + c] = 1.0 / (1.0 + std::exp(-zz));
      }
    // column 3 all zero, column 5 = twin of column 2, last 3 columns one-hot, column 7 negative
    for (long long r = 0; r < N; ++r) {
      H[r * ld + 3] = 0.0;
      H[r * ld + 5] = H[r * ld + 2];
      H[r * ld + 7] = -H[r * ld + 7] * 1e-3;
      for (int j = 0; j < 3; ++j) H[r * ld + M - 3 + j] = (r % 3 == j) ? 1.0 : 0.0;
    }
    CK(cudaMemcpy(dH, H.data(), sizeof(double) * N * ld, cudaMemcpyHostToDevice));
  } else {
    gen_kernel<<<4096, 256>>>(dH, N, M, ld, 12345);
    CK(cudaGetLastError());
  }
  int nsm = 148;
  (void)nsm;
  const int nbI = (M + 127) / 128, Mpad = (nbI + 1) / 2 * 2 * 128;
  const long long Npad = (N + 63) / 64 * 64;
  std::vector<int2> order((size_t)nbI * nbI + 2);
  const int nTiles = oz_pair_order(nbI, getenv("OZ_PBLOCK") ? atoi(getenv("OZ_PBLOCK")) : 3, order.data());
  const long long ksteps = Npad / 32;
  const long long per = getenv("OZ_KPER") ? atoll(getenv("OZ_KPER")) : kOzChunkRows / 32;
  const int splits = (int)((ksteps + per - 1) / per);
  unsigned long long* cmax; int* exps; int8_t* S; double* ws; double* G; int2* dtiles;
  CK(cudaMalloc(&cmax, 8 * M));
  CK(cudaMalloc(&exps, 4 * Mpad));
  CK(cudaMalloc(&S, (size_t)kOzPlanes * Mpad * Npad));
  const long long wsStride = (long long)(nbI * (nbI + 1) / 2) * 16384;
  CK(cudaMalloc(&ws, sizeof(double) * wsStride * 2 * splits));
  CK(cudaMalloc(&G, sizeof(double) * M * M));
  CK(cudaMalloc(&dtiles, sizeof(int2) * nTiles));
  CK(cudaMemcpy(dtiles, order.data(), sizeof(int2) * nTiles, cudaMemcpyHostToDevice));
  CUtensorMap maps[4];
  for (int g = 0; g < 2; ++g)
    for (int ab = 0; ab < 2; ++ab) {
      cuuint64_t d3[3] = {(cuuint64_t)Mpad, (cuuint64_t)Npad, (cuuint64_t)kOzPlanes};
      cuuint64_t s3[2] = {(cuuint64_t)Mpad, (cuuint64_t)Mpad * Npad};
      cuuint32_t b3[3] = {ab ? 64u : 128u, 32u, g ? 7u : (cuuint32_t)kOzGramPlanesG0};
      cuuint32_t e3[3] = {1, 1, 1};
      CUresult cr = cuTensorMapEncodeTiled(&maps[2 * g + ab], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, S, d3, s3, b3, e3,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           ab ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    }
  OzParams p{M, nbI, nTiles, splits, Mpad, Npad, ksteps, per, exps, dtiles, ws, wsStride,
             getenv("OZ_STAGES") ? atoi(getenv("OZ_STAGES")) : 0, getenv("OZ_NOTMA") ? atoi(getenv("OZ_NOTMA")) : 0,
             nullptr};
  unsigned long long* ddbg = nullptr;
  if (getenv("OZ_DBG")) { CK(cudaMalloc(&ddbg, 64)); CK(cudaMemset(ddbg, 0, 64)); p.dbg = ddbg; }
  cudaEvent_t e0, e1, e2, e3;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  float best_slice = 1e30f, best_gram = 1e30f;
  for (int rep = 0; rep < reps; ++rep) {
    cudaEventRecord(e0);
    CK(launch_oz_colmax(dH, ld, N, M, cmax, nsm, 0));
    CK(launch_oz_slice(dH, ld, N, M, cmax, exps, Mpad, Npad, S, 0));
    cudaEventRecord(e1);
    CK(launch_oz_gram2(maps, p, 0));
    cudaEventRecord(e2);
    CK(cudaEventSynchronize(e2));
    CK(cudaGetLastError());
    float a, b;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&b, e1, e2);
    if (a < best_slice) best_slice = a;
    if (b < best_gram) best_gram = b;
  }
  CK(cudaDeviceSynchronize());
  if (ddbg) {
    unsigned long long h[8];
    CK(cudaMemcpy(h, ddbg, 64, cudaMemcpyDeviceToHost));
    printf("dbg (summed over clusters, all reps): MMA tempty-wait %.3g cyc, full-wait %.3g, total %.3g, ksteps %llu, items %llu; "
           "epi tfull-wait %.3g, readout %.3g (per warp-item: %.0f)\n", (double)h[0], (double)h[1], (double)h[2], h[3], h[4],
           (double)h[5], (double)h[6], (double)h[6] / (h[4] * 16.0));
  }
  const double fl = (double)N * M * (M + 1);  // algorithmic flops of the lower-triangle Gram
  const double iops = 28.0 * 2.0 * 128 * 128 * (double)Npad * (nbI * (nbI + 1) / 2);  // lower tiles only
  printf("N=%lld M=%d tiles=%d splits=%d items=%d  slice %.3f ms  gram %.3f ms  => %.2f FP64-equiv TF/s, %.1f int8 TOPS\n",
         N, M, nTiles, splits, 2 * nTiles * splits, best_slice, best_gram, fl / best_gram * 1e-9, iops / best_gram * 1e-9);
  CK(launch_oz_finish(ws, wsStride, 2 * splits, M, G, M, 0, 0));
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<double> g((size_t)M * M);
    CK(cudaMemcpy(g.data(), G, sizeof(double) * M * M, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxrel_seq = 0;
    std::vector<long double> dg(M);
    for (int a = 0; a < M; ++a) { long double s = 0; for (long long r = 0; r < N; ++r) s += (long double)H[r*ld+a]*H[r*ld+a]; dg[a] = s; }
    for (int a = 0; a < M; ++a)
      for (int b = 0; b <= a; ++b) {
        long double s = 0; double sq = 0;
        for (long long r = 0; r < N; ++r) { s += (long double)H[r * ld + a] * H[r * ld + b]; sq += H[r*ld+a]*H[r*ld+b]; }
        long double scale = sqrtl(dg[a] * dg[b]);
        if (scale == 0) scale = 1;
        double rel = (double)(fabsl((long double)g[(size_t)a * M + b] - s) / scale);
        double rels = (double)(fabsl((long double)sq - s) / scale);
        if (rel > maxrel) maxrel = rel;
        if (rels > maxrel_seq) maxrel_seq = rels;
        if (g[(size_t)a * M + b] != g[(size_t)b * M + a]) { printf("asym %d %d\n", a, b); return 1; }
      }
    bool twin = g[2 * M + 2] == g[5 * M + 5] && g[5 * M + 2] == g[2 * M + 2];
    for (int c = 0; c < M; ++c) twin = twin && g[(size_t)c * M + 2] == g[(size_t)c * M + 5];
    printf("check: max |G - exact| / sqrt(Gaa Gbb) = %.3e (sequential fp64 sum: %.3e); twins bit-equal %d; zero col %g\n",
           maxrel, maxrel_seq, (int)twin, g[3 * M + 3]);
    if (maxrel > 4e-16 || !twin) { printf("FAIL\n"); return 1; }
    printf("PASS\n");
  }
  return 0;
}
