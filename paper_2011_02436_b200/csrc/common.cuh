// Shared device helpers for the sm_100a RBP-ELM kernels: FP64 DMMA fragments,
// TMA (cp.async.bulk.tensor) + mbarrier primitives, and small utilities.
//
// FP64 on Blackwell: tcgen05.mma has no f64 kind, so FP64 tensor-core work is
// the warp-level DMMA (mma.sync ... .f64, SASS DMMA.8x8x4).  Operands are staged
// in shared memory by TMA and fed to DMMA from registers; accumulators live in
// registers (TMEM is not addressable by DMMA).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rbpg {

// ---------------------------------------------------------------------------
// DMMA m16n8k4 (row.col): D = A(16x4) * B(4x8) + C, per-thread fragments:
//   a0 = A[g][t], a1 = A[g+8][t];  b0 = B[t][g];
//   c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1]
// with g = lane/4, t = lane%4.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
// mbarrier + TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---------------------------------------------------------------------------
// distributed shared memory: cluster address of a local smem address in CTA `rank`, and
// asynchronous remote stores that complete their bytes on the receiver's mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mapa_u32(uint32_t smem_addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2f64(uint32_t cluster_addr, double a, double b, uint32_t cluster_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                   cluster_addr),
               "d"(a), "d"(b), "r"(cluster_mbar)
               : "memory");
}
__device__ __forceinline__ void st_async_v2b64(uint32_t cluster_addr, unsigned long long a, unsigned long long b,
                                               uint32_t cluster_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n" ::"r"(
                   cluster_addr),
               "l"(a), "l"(b), "r"(cluster_mbar)
               : "memory");
}

// ---------------------------------------------------------------------------
// gpu-scope release/acquire helpers for inter-CTA flag exchange
// ---------------------------------------------------------------------------
// bulk copy (TMA engine) of `bytes` (multiple of 16) from this CTA's shared memory into another
// cluster CTA's shared memory; the bytes complete on the receiver's mbarrier.  The source must be
// made visible to the async proxy first (fence_proxy_async after the writes).
__device__ __forceinline__ void bulk_s2s_cluster(uint32_t cluster_dst, uint32_t src, uint32_t bytes,
                                                 uint32_t cluster_mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          cluster_dst),
      "r"(src), "r"(bytes), "r"(cluster_mbar)
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// programmatic dependent launch: a kernel launched with the programmatic-serialization attribute
// may start while its predecessor runs; pdl_wait() blocks until the predecessor grid has completed
// and its writes are visible (a no-op without the attribute).  pdl_trigger() lets this grid's
// dependent start launching now.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_volatile_f64(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Exactly-rounded mul / sub that the compiler may not contract into an FMA
// (the reference build is SSE2 without FMA; see oracle header).
// 1 / x for x >= 1 (x = 1 + exp(-z) in the sigmoid) without the XU pipe: an integer-subtraction
// seed on the bit pattern (relative error < 5.1%), then four Newton-Raphson steps on DFMA
// (error 5e-2 -> 2.6e-3 -> 6.5e-6 -> 4e-11 -> ~1e-21 before rounding), the last one giving the
// correctly rounded quotient in all tested cases.  The DP reciprocal seed (MUFU.RCP64H) is the
// bottleneck of the sigmoid epilogue on sm_100 (XU pipe ~90% busy), DFMA is not.
// For x >= 2^1020 (z below about -707: 1/x is subnormal or nearly so) the seed's exponent difference
// has no room and the iteration returned NaN; such x are scaled by 2^-64 first (exact) and the quotient
// is scaled back with one rounding onto the subnormal grid.
__device__ __forceinline__ double recip_ge1(double x) {
  const bool big = x >= 0x1p1020;
  const double xs = big ? x * 0x1p-64 : x;
  double y = __longlong_as_double(0x7FDE623822FC16E6LL - __double_as_longlong(xs));
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double e = fma(-xs, y, 1.0);
    y = fma(y, e, y);
  }
  y = big ? y * 0x1p-64 : y;
  return x <= 1.7976931348623157e308 ? y : (x > 0.0 ? 0.0 : x);  // 1/inf = 0, NaN propagates
}

// 2^e for a normal exponent (-1022 <= e <= 1023)
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double(static_cast<long long>(e + 1023) << 52); }
// e^t without branches for the sigmoid epilogue (~1 ulp, like exp): t = k ln2 + r with k = rint(t / ln2)
// read from the bits of the magic-shifted product (no F2I), r by two FMAs (|r| <= ln2 / 2), e^r by its
// degree-13 Taylor polynomial (truncation < 2^-57; coefficients in constant memory, so every DFMA takes
// its operand from the constant bank), 2^k as two exact factors; t > 709.78 -> inf and t < -745.14 -> 0
// by selects.  Branch-free, so the unrolled epilogue interleaves many of them.
static __constant__ double c_exp_taylor[14] = {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
                                        1.0 / 362880.0,     1.0 / 40320.0,     1.0 / 5040.0,     1.0 / 720.0,
                                        1.0 / 120.0,        1.0 / 24.0,        1.0 / 6.0,        0.5,
                                        1.0,                1.0};
__device__ __forceinline__ double exp_sig(double t) {
  const double kb = fma(t, 0x1.71547652b82fep0, 0x1.8p52);
  const int k = __double2loint(kb);
  const double kd = kb - 0x1.8p52;
  double r = fma(-kd, 0x1.62e42fefa39efp-1, t);
  r = fma(-kd, 0x1.abc9e3b39803fp-56, r);
  double q = c_exp_taylor[0];
#pragma unroll
  for (int i = 1; i < 14; ++i) q = fma(q, r, c_exp_taylor[i]);
  const int k1 = k >> 1;
  const double v = (q * pow2i(k1)) * pow2i(k - k1);
  return t > 709.782712893384 ? __longlong_as_double(0x7ff0000000000000LL) : (t < -745.1332191019412 ? 0.0 : v);
}
// The epilogue's sigmoid for |z| <= 700 (finite): bit for bit recip_ge1(1.0 + exp_sig(-z)), with the
// selects that can never fire in that range left out -- e^t neither overflows nor underflows (|k| <= 1010:
// q 2^k is a normal double, so adding k to q's exponent field equals the two exact power-of-two products),
// and 1 + e^t is finite.  The caller checks the range with one integer maximum over the high words of its
// z values and redoes the rare out-of-range block through sigmoid_exact.
__device__ __forceinline__ double sigmoid_in_range(double z) {
  const double t = -z;
  const double kb = fma(t, 0x1.71547652b82fep0, 0x1.8p52);
  const int k = __double2loint(kb);
  const double kd = kb - 0x1.8p52;
  double r = fma(-kd, 0x1.62e42fefa39efp-1, t);
  r = fma(-kd, 0x1.abc9e3b39803fp-56, r);
  double q = c_exp_taylor[0];
#pragma unroll
  for (int i = 1; i < 14; ++i) q = fma(q, r, c_exp_taylor[i]);
  const double e = __hiloint2double(__double2hiint(q) + (k << 20), __double2loint(q));
  const double x = 1.0 + e;
  double y = __longlong_as_double(0x7FDE623822FC16E6LL - __double_as_longlong(x));
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double d = fma(-x, y, 1.0);
    y = fma(y, d, y);
  }
  return y;
}
// every z, including non-finite ones: the reference arithmetic with all its selects (out of line: it runs
// only for blocks holding |z| > 700, and for the last, partial row block of the matrix)
static __device__ __noinline__ double sigmoid_exact(double z) { return recip_ge1(1.0 + exp_sig(-z)); }
constexpr int kSigmoidRangeHi = 0x4085E000;  // high word of 700.0
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// Optional device timeline (RBPG_DEVICE_TIMELINE): slot s of tl holds {first entry, first start
// of work, last exit} over a launch's CTAs, in globaltimer nanoseconds.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int slot, int phase) {
  if (tl == nullptr || threadIdx.x != 0) return;
  const unsigned long long t = gtimer();
  if (phase < 2) atomicMin(&tl[3 * slot + phase], t);
  else atomicMax(&tl[3 * slot + 2], t);
}

}  // namespace rbpg
