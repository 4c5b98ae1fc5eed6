// Latency probe for the sequential-step kernels (panel factorisation, TRSM sweeps):
// cluster barrier, DSMEM load, global-flag grid barrier, L2 pointer chase, __syncthreads.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/latency_probe.cu -o tools/latency_probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int IT = 20000;

template <int CL>
__global__ void cluster_sync_loop(long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / IT;
}

template <int CL>
__global__ void cluster_split_loop(long long* out) {  // arrive.release / wait.acquire pair
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / IT;
}

template <int CL>
__global__ void dsmem_chase(long long* out) {
  __shared__ int nxt[1024];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i * 97 + 13) & 1023;
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    int* rem = cl.map_shared_rank(nxt, CL - 1);
    int p = 0;
    long long t0 = clock64();
    for (int i = 0; i < 2000; ++i) p = rem[p];
    long long t1 = clock64();
    out[2] = (t1 - t0) / 2000 + (p == -1);
  }
  cl.sync();
}

__global__ void l2_chase(const int* next, long long* out, int hops) {
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < hops; ++i) p = __ldcg(next + p);
  long long t1 = clock64();
  out[3] = (t1 - t0) / hops + (p == -1);
}

__global__ void syncthreads_loop(long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < IT; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / IT;
}

// grid barrier through per-CTA epoch flags (as the grid panel variant), C CTAs
__global__ void flag_barrier_loop(unsigned int* flags, long long* out, int iters) {
  const int C = gridDim.x;
  long long t0 = clock64();
  for (int e = 1; e <= iters; ++e) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(flags + blockIdx.x * 32), "r"(e) : "memory");
    if (threadIdx.x < 32) {
      for (int i = threadIdx.x; i < C; i += 32) {
        unsigned int v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flags + i * 32) : "memory");
        } while (v < (unsigned)e);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[5] = (t1 - t0) / iters;
}

__global__ void grid_sync_loop(long long* out, int iters) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[6] = (t1 - t0) / iters;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  long long h[16] = {};
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sm_clock_khz\": %d", clk);
  auto launch_cl = [&](void (*k)(long long*), int cl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
    cudaDeviceSynchronize();
    return e;
  };
#define CL_CASE(N)                                                                                           \
  launch_cl(cluster_sync_loop<N>, N);                                                                        \
  launch_cl(cluster_split_loop<N>, N);                                                                       \
  launch_cl(dsmem_chase<N>, N);                                                                              \
  cudaMemcpy(h, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);                                          \
  printf(", \"cluster%d_sync_cyc\": %lld, \"cluster%d_arrive_wait_cyc\": %lld, \"cluster%d_dsmem_load_cyc\": %lld", N, \
         h[0], N, h[1], N, h[2]);
  CL_CASE(2) CL_CASE(4) CL_CASE(8) CL_CASE(16)
  // L2 chase over 8 MB
  const int n = 2 * 1024 * 1024;
  int* nx;
  cudaMalloc(&nx, n * sizeof(int));
  int* hn = new int[n];
  for (int i = 0; i < n; ++i) hn[i] = (int)((i + 4099LL * 33) % n);
  cudaMemcpy(nx, hn, n * sizeof(int), cudaMemcpyHostToDevice);
  l2_chase<<<1, 1>>>(nx, d, 1000);
  cudaDeviceSynchronize();
  l2_chase<<<1, 1>>>(nx, d, 4000);
  syncthreads_loop<<<1, 256>>>(d);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf(", \"l2_load_cyc\": %lld, \"syncthreads256_cyc\": %lld", h[3], h[4]);
  unsigned int* flags;
  cudaMalloc(&flags, 148 * 32 * 4);
  for (int C : {8, 16, 32, 64, 148}) {
    cudaMemset(flags, 0, 148 * 32 * 4);
    int iters = 2000;
    void* args[] = {&flags, &d, &iters};
    cudaLaunchCooperativeKernel((void*)flag_barrier_loop, dim3(C), dim3(256), args, 0, 0);
    void* args2[] = {&d, &iters};
    cudaLaunchCooperativeKernel((void*)grid_sync_loop, dim3(C), dim3(256), args2, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 8 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf(", \"flagbar%d_cyc\": %lld, \"gridsync%d_cyc\": %lld", C, h[5], C, h[6]);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
