// FP64 peak probe for the B200 roofline denominator (MEASURED_PEAKS.json has no
// FP64 entry).  Measures, with CUDA events after warm-up:
//   * DMMA (mma.sync f64) issue-bound throughput for m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16,
//   * DFMA throughput (independent FMA chains),
//   * cuBLAS DGEMM 8192^3, best of 10 (the "measured FP64 GEMM" roofline peak),
// and prints one JSON object.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/fp64_peak.cu -lcublas -o tools/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int ACC = 8;  // independent accumulator tiles per warp

__global__ void dmma_k4(double* out) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = a0 - 1;
  double c[ACC][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < ACC; ++s)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};"
                   : "+d"(c[s][0]), "+d"(c[s][1]), "+d"(c[s][2]), "+d"(c[s][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double acc = 0;
  for (int s = 0; s < ACC; ++s) acc += c[s][0] + c[s][1] + c[s][2] + c[s][3];
  if (acc == 12345.678) out[0] = acc;
}

__global__ void dmma_k8(double* out) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 0.5; b[1] = 0.25;
  double c[ACC][4] = {};
  for (int it = 0; it < ITERS / 2; ++it) {
#pragma unroll
    for (int s = 0; s < ACC; ++s)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
                   : "+d"(c[s][0]), "+d"(c[s][1]), "+d"(c[s][2]), "+d"(c[s][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double acc = 0;
  for (int s = 0; s < ACC; ++s) acc += c[s][0] + c[s][1] + c[s][2] + c[s][3];
  if (acc == 12345.678) out[0] = acc;
}

__global__ void dmma_k16(double* out) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 * i;
  double c[ACC][4] = {};
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int s = 0; s < ACC; ++s)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};"
                   : "+d"(c[s][0]), "+d"(c[s][1]), "+d"(c[s][2]), "+d"(c[s][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double acc = 0;
  for (int s = 0; s < ACC; ++s) acc += c[s][0] + c[s][1] + c[s][2] + c[s][3];
  if (acc == 12345.678) out[0] = acc;
}

__global__ void dmma_m8k4(double* out) {
  double a0 = threadIdx.x * 1e-3, b0 = a0 - 1;
  double c[2 * ACC][2] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < 2 * ACC; ++s)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};"
                   : "+d"(c[s][0]), "+d"(c[s][1]) : "d"(a0), "d"(b0));
  }
  double acc = 0;
  for (int s = 0; s < 2 * ACC; ++s) acc += c[s][0] + c[s][1];
  if (acc == 12345.678) out[0] = acc;
}

__global__ void dfma_chain(double* out) {
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  const double m = 0.999999, a = 1e-7;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], m, a);
  }
  double acc = 0;
  for (int i = 0; i < 16; ++i) acc += x[i];
  if (acc == 12345.678) out[0] = acc;
}

template <typename K>
static float time_kernel(K kern, int blocks, int threads, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, 64));
  const int blocks = sms * 4, threads = 256;  // 8 warps x 4 CTAs per SM
  const double warps = blocks * (threads / 32.0);
  float t;
  printf("{\"sms\": %d", sms);
  t = time_kernel(dmma_k4, blocks, threads, out);
  printf(", \"dmma_m16n8k4_tflops\": %.3f", warps * ITERS * ACC * 16 * 8 * 4 * 2.0 / (t * 1e-3) / 1e12);
  t = time_kernel(dmma_k8, blocks, threads, out);
  printf(", \"dmma_m16n8k8_tflops\": %.3f", warps * (ITERS / 2) * ACC * 16 * 8 * 8 * 2.0 / (t * 1e-3) / 1e12);
  t = time_kernel(dmma_k16, blocks, threads, out);
  printf(", \"dmma_m16n8k16_tflops\": %.3f", warps * (ITERS / 4) * ACC * 16 * 8 * 16 * 2.0 / (t * 1e-3) / 1e12);
  t = time_kernel(dmma_m8k4, blocks, threads, out);
  printf(", \"dmma_m8n8k4_tflops\": %.3f", warps * ITERS * 2 * ACC * 8 * 8 * 4 * 2.0 / (t * 1e-3) / 1e12);
  t = time_kernel(dfma_chain, blocks, threads, out);
  printf(", \"dfma_tflops\": %.3f", blocks * (double)threads * ITERS * 16 * 2.0 / (t * 1e-3) / 1e12);

  // cuBLAS DGEMM 8192^3
  const int n = 8192;
  double *A, *B, *C;
  CK(cudaMalloc(&A, sizeof(double) * n * n));
  CK(cudaMalloc(&B, sizeof(double) * n * n));
  CK(cudaMalloc(&C, sizeof(double) * n * n));
  cudaMemset(A, 0, sizeof(double) * n * n);
  cudaMemset(B, 0, sizeof(double) * n * n);
  cublasHandle_t h; cublasCreate(&h);
  double one = 1.0, zero = 0.0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf(", \"cublas_dgemm_8192_tflops\": %.3f", 2.0 * n * n * (double)n / (best * 1e-3) / 1e12);
  // sustained: back to back for ~3 s
  cudaEventRecord(e0);
  int reps = 0;
  float el = 0;
  while (el < 3000.f) {
    for (int r = 0; r < 10; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
    reps += 10;
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&el, e0, e1);
  }
  printf(", \"cublas_dgemm_8192_sustained_tflops\": %.3f", 2.0 * n * n * (double)n * reps / (el * 1e-3) / 1e12);
  printf("}\n");
  CK(cudaGetLastError());
  return 0;
}
