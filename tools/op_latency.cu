// Dependent-chain latency (cycles) of the ops on the pivot step's critical path.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/op_latency.cu -o tools/op_latency
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  __shared__ int smi[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; smi[i] = (i * 7 + 3) & 1023; }
  __syncthreads();
  double x = seed, y = 1.0000001;
  long long t0, t1;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9); t1 = clock64(); cyc[0] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x + y; t1 = clock64(); cyc[1] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N / 16; ++i) x = sqrt(x) + 1.0; t1 = clock64(); cyc[2] = (t1 - t0) / (N / 16);
  t0 = clock64(); for (int i = 0; i < N / 16; ++i) x = 1.0 / x + 1.0; t1 = clock64(); cyc[3] = (t1 - t0) / (N / 16);
  int p = 0;
  t0 = clock64(); for (int i = 0; i < N; ++i) p = smi[p]; t1 = clock64(); cyc[4] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9; t1 = clock64(); cyc[5] = (t1 - t0) / N;
  unsigned u = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < N; ++i) u = __reduce_max_sync(0xffffffffu, u) + threadIdx.x; t1 = clock64(); cyc[6] = (t1 - t0) / N;
  t0 = clock64(); for (int i = 0; i < N / 16; ++i) x = x / (y + x); t1 = clock64(); cyc[7] = (t1 - t0) / (N / 16);
  double z = seed;
  t0 = clock64(); for (int i = 0; i < N; ++i) z = sm[((int)z) & 1023]; t1 = clock64(); cyc[8] = (t1 - t0) / N;
  out[threadIdx.x] = x + p + u + z;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
  lat<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, c, 9 * 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma\": %lld, \"dadd\": %lld, \"dsqrt+add\": %lld, \"drcp+add\": %lld, \"lds_int_chase\": %lld, \"shfl+dadd\": %lld, \"redux+iadd\": %lld, \"ddiv\": %lld, \"lds_f64_chase\": %lld}\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
  return 0;
}
