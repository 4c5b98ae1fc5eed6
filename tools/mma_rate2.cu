// tcgen05 kind::i8 issue-rate probe, part 2: (a) the Ozaki k-step pattern (18 MMAs over 3 accumulators,
// 14 operand tiles, commit per step) on 1 CTA; (b) the same with cta_group::2 (M = 256, N = 128 per pair).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t dsw128(uint32_t a) {
  return ((a >> 4) & 0x3FFF) | (uint64_t(4096 >> 4) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t dsw64(uint32_t a) {
  return ((a >> 4) & 0x3FFF) | (uint64_t(2048 >> 4) << 16) | (uint64_t(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
}
template <int CG>
__global__ void __launch_bounds__(128, 1) probe(int steps, int commit_every, unsigned long long* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t fullb[8], emptyb[8];
  unsigned char* s = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 60 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(s)[i] = 0x01010101u * (i & 3);
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&fullb[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&emptyb[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  if (threadIdx.x < 32) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tb = tslot;
  const uint32_t base = su32(s);
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) |
                         ((uint32_t)(CG == 2 ? 256 : 128) >> 4 << 24);
  unsigned long long t0 = clock64();
  int ncommit = 0;
  if (mode >= 2 && threadIdx.x == 32 && rank == 0) {  // producer: wait empty, arrive full
    for (int st = 0; st < steps; ++st) {
      const int s5 = st % 5;
      if (st >= 5) asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&emptyb[s5])), "r"((st / 5 - 1) & 1));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&fullb[s5])) : "memory");
    }
  }
  if (threadIdx.x == 0 && rank == 0) {
    for (int st = 0; st < steps; ++st) {
      if (mode >= 2) {
        const int s5 = st % 5;
        asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&fullb[s5])), "r"((st / 5) & 1));
      }
      if (mode >= 1) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const bool g0 = mode == 3 || (mode == 4 && (st & 1));
      const int wlo = g0 ? 2 : 6, whi = g0 ? 5 : 8, pl = g0 ? 4 : 7;
#pragma unroll
      for (int w = 2; w <= 8; ++w)
#pragma unroll
        for (int i = 1; i < w; ++i) {
          const int j = w - i;
          if (i > 7 || j > 7) continue;
          if (w < wlo || w > whi || i > pl || j > pl) continue;
          const uint64_t da = dsw128(base + (i - 1) * 4096);
          const uint64_t db = CG == 2 ? dsw64(base + 28672 + (j - 1) * 2048) : dsw128(base + 28672 + (j - 1) * 4096);
          const uint32_t acc = (st > 0 || i > 1);
          if (CG == 1)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                             tb + (w - wlo) * 128), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                             tb + (w - wlo) * 128), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      if (mode >= 2) {
        const int s5 = st % 5;
        if (CG == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&emptyb[s5])) : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(su32(&emptyb[s5])), "h"((unsigned short)1) : "memory");
      } else if (commit_every && (st % commit_every) == commit_every - 1) {
        if (CG == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(su32(&bar)), "h"((unsigned short)1) : "memory");
        ++ncommit;
      }
    }
    if (CG == 1)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(su32(&bar)), "h"((unsigned short)1) : "memory");
    ++ncommit;
    // wait for the last commit's phase
    const uint32_t par = (ncommit - 1) & 1;
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&bar)), "r"(par));
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  else __syncthreads();
  if (threadIdx.x < 32) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tb));
  }
}
template <int CG>
void run(int commit_every, int mode) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int steps = 2000;
  auto k = probe<CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 64 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, 10, commit_every, d, mode);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, steps, commit_every, d, mode);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  // per step: 18 MMAs of 128 x 128 x 32 per SM
  double ops = 2.0 * 128 * 128 * 32 * 18.0 * steps * 148;
  printf("mode %d cta_group::%d commit every %d: %.1f cycles/step (floor 1152), %.0f TOPS, err=%s\n", mode, CG, commit_every,
         (double)cyc / steps, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<2>(1, 2); run<2>(1, 3); run<2>(1, 4); run<1>(1, 3);
  return 0;
}
