// tcgen05.mma kind::i8 issue-rate probe: one CTA per SM issues back-to-back MMAs from constant shared
// memory (no TMA) into TMEM; reports int8 TOPS for K-major vs MN-major operands, N = 64/128/256.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int MN, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* s = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(s)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tslot;
  // descriptors
  const uint32_t a = su32(s), b = su32(s + 32768);
  uint64_t da, db;
  if (MN) {  // MN-major SW128: K rows of 128 B, 8-row groups 1024 B apart; B: N/128 atoms 4096 B apart
    da = ((a >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
    db = ((b >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
  } else {  // K-major SW128: rows of 128 B (4 k-steps), 8-row groups 1024 B apart
    da = ((a >> 4) & 0x3FFF) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
    db = ((b >> 4) & 0x3FFF) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
  }
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (MN ? (1u << 15) | (1u << 16) : 0u) | ((uint32_t)(N >> 3) << 17) |
                         ((128u >> 4) << 24);
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const uint32_t acc = it > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tb),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
}
template <int MN, int N>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 20000;
  cudaFuncSetAttribute(probe<MN, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  probe<MN, N><<<148, 128, 70 * 1024>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MN, N><<<148, 128, 70 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double ops = 2.0 * 128 * N * 32 * (double)iters * 148;
  printf("%s N=%d: %.1f cycles/MMA (floor %d), %.0f TOPS (kernel %.3f ms) err=%s\n", name, N, (double)cyc / iters,
         128 * N / 256, ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0, 128>("K-major ");
  run<1, 128>("MN-major");
  run<0, 256>("K-major ");
  run<1, 256>("MN-major");
  run<0, 64>("K-major ");
  run<1, 64>("MN-major");
  return 0;
}
