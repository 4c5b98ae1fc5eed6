// K2i: the Gram of the augmented rows [H T] on the INT8 tensor cores (tcgen05.mma kind::i8), exact
// to FP64 accuracy by integer splitting (Ozaki scheme I) -- the same product as syrk_kernel
// (reference linalg.cpp:179-184: G = H^T H, lower triangle + mirror; H^T T in the last tile row).
//
// Splitting.  Column c of A (N x M, fp64) gets the exponent e_c with max_k |A[k][c]| < 2^e_c.
// Every element becomes the 54-bit integer X = rint(A * 2^(54 - e_c)) (|X| < 2^54: the rounding is
// at 2^-54 of the column maximum, finer than fp64's own 2^-53 relative spacing at that maximum),
// written in 7 balanced base-256 digits
//     X = sum_{i=1..7} d_i 256^(7-i),   d_2..d_7 in [-128, 127],  d_1 in [-64, 64],
// so that A[k][c] = 2^(e_c - 54) X exactly up to that one rounding.  The digit planes D_i (int8,
// N x M) keep A's row-major layout, [plane][row][column]: MN-major MMA operands, so a TMA box row is
// 128 contiguous bytes.
//
// Products.  G[a][b] = 2^(e_a + e_b) sum_{i,j} 2^(4 - 8(i + j)) (D_i^T D_j)[a][b].  Terms with
// i + j >= 9 are below 2^-56 of the scale max_a max_b per row and zero-mean (balanced digits): they
// are dropped, which leaves 28 INT8 products per 32-row k-step, grouped by weight w = i + j into int32
// accumulators in tensor memory: group 0 = w 2..5 (10 products, 4 accumulators, planes 1..4), group
// 1 = w 6..8 (18 products, 3 accumulators, planes 1..7).  An item is one (256 x 128 block, group,
// split of at most 512 k-steps) -- 512 k-steps is the int32 headroom (7 pairs x 32 rows x 2^14 x 512
// < 2^31) -- read out once: Horner's rule over the weights in fp64 (exact for group 1, one rounding
// for group 0), scaled by the column exponents, stored into the item's packed partial tile.  The
// fixed-order reduction (oz_finish_kernel) sums the partials and mirrors: the result is exactly
// symmetric and, integer arithmetic being exact, identical columns give bit-identical Gram entries
// wherever they sit (the exact twin ties of C3 survive).
//
// Execution (oz_gram2_kernel): persistent CTA pairs (tcgen05 cta_group::2, M = 256, N = 128); per
// pair one producer warp per CTA (3-D TMA, one box per operand and k-step), one MMA warp (rank 0),
// eight epilogue warps per CTA.  Measured (tools/ozaki_test, one B200): C5 shard 413 ms = 2.38 int8
// POP/s (83 FP64-equivalent TF/s), C4 L = 8000 68 ms; operands-resident ceiling 3.5 POP/s; the MMA
// pattern itself 4.5 POP/s (tools/mma_rate2.cu).
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <vector>

namespace rbpg {

namespace {

constexpr int kOzPlanes = 7;
constexpr int kOzMaxStages = 12;
constexpr uint32_t kOzRing = 224 * 1024;  // operand ring: as many whole k-step stages as fit
constexpr uint32_t kOzTileBytes = 128 * 32;  // one plane tile: 32 rows x 128 columns (bytes)

// shared-memory matrix descriptor, MN-major, 128-byte swizzle: a K row of 128 bytes (the whole 128-wide
// M / N extent, one swizzle atom wide), 8-row K groups 1024 B apart (stride byte offset); the leading
// byte offset (next 128-element MN atom) is unused at M = N = 128
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(4096 >> 4) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

// Group G: number of weights, first weight, planes used, and the (i, j) pairs in issue order
template <int G>
struct OzGroup {
  static constexpr int kW = G == 0 ? 4 : 3;
  static constexpr int kW0 = G == 0 ? 2 : 6;
  static constexpr int kPlanes = G == 0 ? 4 : 7;
};
// The Gram's weight split (kOzGramW0G1 = first weight of group 1, kernels.cuh): group 0 = weights
// 2 .. kOzGramW0G1 - 1 on planes 1 .. kOzGramW0G1 - 2, group 1 = kOzGramW0G1 .. 8 on planes 1 .. 7
template <int G>
struct OzGramGroup {
  static constexpr int kW = G == 0 ? kOzGramW0G1 - 2 : 9 - kOzGramW0G1;
  static constexpr int kW0 = G == 0 ? 2 : kOzGramW0G1;
  static constexpr int kPlanes = G == 0 ? kOzGramPlanesG0 : 7;
};

}  // namespace

// max |A[k][c]| per column as ordered bits (atomicMax on the non-negative double's pattern)
__global__ void __launch_bounds__(256) oz_colmax_kernel(const double* __restrict__ A, long long lda, long long N,
                                                        int M, unsigned long long* cmax) {
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ty = threadIdx.x >> 5;
  double m = 0.0;
  if (c < M)
    for (long long r = static_cast<long long>(blockIdx.y) * 8 + ty; r < N; r += static_cast<long long>(gridDim.y) * 8)
      m = fmax(m, fabs(A[r * lda + c]));
  __shared__ double red[8][33];
  red[ty][threadIdx.x & 31] = m;
  __syncthreads();
  if (ty == 0 && c < M) {
    for (int i = 1; i < 8; ++i) m = fmax(m, red[i][threadIdx.x & 31]);
    atomicMax(cmax + c, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// column exponents e_c (max < 2^e_c; 0 for an all-zero column) for columns < Mpad (padding: 0)
__global__ void oz_exps_kernel(const unsigned long long* cmax, int M, int Mpad, int* exps) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= Mpad) return;
  int e = 0;
  if (c < M && cmax[c] != 0ull) {
    const double v = __longlong_as_double(static_cast<long long>(cmax[c]));
    frexp(v, &e);  // v = f 2^e, f in [0.5, 1): v < 2^e
  }
  exps[c] = e;
}

// Digit planes, [plane][row][column] with the padded extents (rows >= N, columns >= M: zeros).
// One thread per 8 consecutive columns of a row: 64 bytes of A in, 8 bytes per plane out.
// Balanced digits without a digit loop: adding B = 0x808080808080 (128 in each of the six low bytes)
// turns X = sum_i d_i 256^i (d_0..d_5 in [-128, 127]) into X + B = sum_{i<6} (d_i + 128) 256^i +
// d_6 256^6 with every d_i + 128 in [0, 255] -- byte i of X + B is d_i + 128, i.e. d_i ^ 0x80 as a
// signed byte, and (X + B) >> 48 is the top digit d_6.  So V = (X + B) ^ B holds all seven digit bytes
// (byte i: plane 6 - i), and the 8 x 8 byte transpose of a thread's 8 values into its 8-byte plane
// words takes four 4 x 4 PRMT transposes.

__device__ __forceinline__ void byte_transpose4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&r)[4]) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  r[0] = __byte_perm(t0, t2, 0x5410);
  r[1] = __byte_perm(t0, t2, 0x7632);
  r[2] = __byte_perm(t1, t3, 0x5410);
  r[3] = __byte_perm(t1, t3, 0x7632);
}

// Grid: x over 128-thread blocks of 8-column groups (a thread's 8 columns and their scales are fixed),
// y strides the rows -- no index division in the loop; 16-byte loads when the row segment is aligned.
__global__ void __launch_bounds__(128) oz_slice_kernel(const double* __restrict__ A, long long lda, long long N, int M,
                                                       const int* __restrict__ exps, int8_t* __restrict__ S,
                                                       long long plane_stride, int Mpad, long long Npad) {
  constexpr unsigned long long kBias = 0x808080808080ull;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= Mpad / 8) return;
  const int c0 = g * 8;
  // A 2^(54 - e) exactly (|.| < 2^54): one power-of-two factor, two when 54 - e exceeds the normal
  // exponent range (columns with max < 2^-969); a result below 2^-1022 rounds to 0 either way
  double f1[8], f2[8];
  bool live[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int c = c0 + q;
    live[q] = c < M;
    const int k = live[q] ? 54 - exps[c] : 0;
    f1[q] = pow2i(min(k, 1023));
    f2[q] = k > 1023 ? pow2i(k - 1023) : 1.0;
  }
  const bool full = c0 + 8 <= M;
  for (long long r = blockIdx.y; r < Npad; r += gridDim.y) {
    double a[8];
    const double* row = A + r * lda + c0;
    if (r < N && full && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(row + q));
        a[q] = t.x;
        a[q + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (r < N && live[q]) ? row[q] : 0.0;
    }
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long X = __double2ll_rn((a[q] * f1[q]) * f2[q]);
      const unsigned long long V = (static_cast<unsigned long long>(X) + kBias) ^ kBias;
      lo[q] = static_cast<uint32_t>(V);
      hi[q] = static_cast<uint32_t>(V >> 32);
    }
    uint32_t l0[4], l1[4], h0[4], h1[4];  // [byte] words of columns 0-3 / 4-7
    byte_transpose4(lo[0], lo[1], lo[2], lo[3], l0);
    byte_transpose4(lo[4], lo[5], lo[6], lo[7], l1);
    byte_transpose4(hi[0], hi[1], hi[2], hi[3], h0);
    byte_transpose4(hi[4], hi[5], hi[6], hi[7], h1);
    int8_t* dst = S + r * Mpad + c0;
#pragma unroll
    for (int i = 0; i < 7; ++i) {  // byte i -> plane 6 - i
      const uint32_t w0 = i < 4 ? l0[i & 3] : h0[i & 3], w1 = i < 4 ? l1[i & 3] : h1[i & 3];
      *reinterpret_cast<uint2*>(dst + (kOzPlanes - 1 - i) * plane_stride) = make_uint2(w0, w1);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 128 block
// -- tile rows 2P (CTA rank 0) and 2P + 1 (rank 1) against tile column J -- as ONE M = 256, N = 128
// MMA stream issued by rank 0.  Each CTA stages its own 128 A rows (box {128, 32}, 128-byte swizzle)
// and HALF of the B columns (box {64, 32}, 64-byte swizzle): per SM the tensor core reads 6 KB of
// shared memory per 64-cycle MMA instead of 8 KB, and the L2 delivers 6 KB per plane instead of 8.
// Every CTA's TMA bytes complete on rank 0's full barrier; rank 0's commits arrive on both CTAs'
// empty / tmem-full barriers (multicast); both epilogues arrive on rank 0's tmem-empty barrier.  The
// accumulator rows live in the TMEM of the CTA that owns them, so the epilogue is unchanged.  The
// block (2P, 2P + 1) is above the diagonal: computed, not stored.
// ---------------------------------------------------------------------------------------------
namespace {
constexpr uint32_t kOzBHalfBytes = 64 * 32;  // B half-tile: 32 rows x 64 columns
// instruction descriptor: M = 256, N = 128, MN-major, s8 x s8 -> s32
constexpr uint32_t kOzIdesc2 =
    (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
// MN-major, 64-byte swizzle: K rows of 64 bytes (this CTA's 64 columns, one swizzle atom), 8-row
// groups 512 B apart
__device__ __forceinline__ uint64_t oz_desc64(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(2048 >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(4) << 61);
}
// Executed by the whole (converged) MMA warp with warp-uniform operands, so the descriptors stay in
// uniform registers; one elected lane issues.  (Issued from a single-lane branch, every MMA needed a
// register -> uniform-register broadcast loop: ~1.5x the 64-cycle MMA time at 10 MMAs per k-step.)
__device__ __forceinline__ void oz_mma2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kOzIdesc2), "r"(acc));
}
__device__ __forceinline__ void oz_commit2(uint64_t* bar) {  // arrive on `bar` in both CTAs of the pair
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];\n" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void named_bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

template <class Grp>
__device__ __forceinline__ void oz_mma_kstep2(uint32_t tbase, uint32_t sa, uint32_t sb, bool first) {
#pragma unroll
  for (int w = Grp::kW0; w < Grp::kW0 + Grp::kW; ++w) {
#pragma unroll
    for (int i = 1; i < w; ++i) {
      const int j = w - i;
      if (i > Grp::kPlanes || j > Grp::kPlanes) continue;
      oz_mma2(tbase + (w - Grp::kW0) * 128, oz_desc(sa + (i - 1) * kOzTileBytes),
              oz_desc64(sb + (j - 1) * kOzBHalfBytes), (first && i == 1) ? 0u : 1u);
    }
  }
}
}  // namespace

// x 2^e without a libm call: two exact power-of-two factors, each inside the normal exponent range
// for |e| <= 2044 (column exponents of finite data)
__device__ __forceinline__ double scale2(double x, int e) {
  const int e1 = e / 2;
  return (x * pow2i(e1)) * pow2i(e - e1);
}
// exact int64 -> fp64 for |t| < 2^51 on the integer and FP64 pipes (I2F.F64 runs on the XU pipe, which
// the sigmoid epilogue would saturate): the bits of 1.5 * 2^52 plus t are the double 1.5 * 2^52 + t
__device__ __forceinline__ double i51_to_f64(long long t) {
  constexpr double kMagic = 0x1.8p52;
  return __longlong_as_double(__double_as_longlong(kMagic) + t) - kMagic;
}
// mbarrier wait that suspends the thread (up to the hint) instead of spinning: the producer and MMA
// warps of oz_hidden_kernel share the SM sub-partitions with the epilogue's FP64 math
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// One chunk's read-out for one epilogue thread (row `quarter * 32 + lane`, 64 columns from `col0`):
// Horner over the group's weights, added to the fp64 running sums in registers.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// One chunk's read-out for one epilogue thread (row `quarter * 32 + lane`, 64 columns from `col0`):
// Horner over the group's weights, added to the fp64 running sums in registers.
// Read-out of one item's accumulators by one epilogue thread (tile row `quarter * 32 + lane`, all 128
// columns, 8 at a time): Horner over the group's weights in fp64 (exact for group 1, one rounding for
// group 0), times 2^(e_row + e_col + 4 - 8 w0), stored to the item's packed partial tile.  Every
// TMEM load of the item is done before the caller releases the accumulators; the stores drain after.
template <int G>
__device__ __forceinline__ void oz_readout(uint32_t trow, const OzParams& p, int I, int J, int quarter, int lane,
                                           int col0, const int* ecol, double* tile_out, bool trans) {
  constexpr int kW = OzGramGroup<G>::kW, kW0 = OzGramGroup<G>::kW0;
  const int rl = quarter * 32 + lane, r = I * 128 + rl;
  const bool rok = r < p.M;
  const int er = (rok ? p.exps[r] : 0) + 4 - 8 * kW0;
  double* dst = tile_out + rl * 128;
#pragma unroll 2
  for (int cb = col0 / 8; cb < col0 / 8 + 8; ++cb) {
    double v[8];
    int c[8];
    tmem_ld8(trow + (kW - 1) * 128 + cb * 8, c);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = i51_to_f64(c[q]);
#pragma unroll
    for (int a = kW - 2; a >= 0; --a) {
      tmem_ld8(trow + a * 128 + cb * 8, c);
      tmem_wait_ld();
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = fma(v[q], 0x1.0p-8, i51_to_f64(c[q]));
    }
    if (rok && !trans) {
#pragma unroll
      for (int q = 0; q < 8; q += 2)
        *reinterpret_cast<double2*>(dst + cb * 8 + q) =
            make_double2(scale2(v[q], er + ecol[cb * 8 + q]), scale2(v[q + 1], er + ecol[cb * 8 + q + 1]));
    } else if (rok) {  // transposed: the warp's 32 rows are 32 consecutive entries of a stored row
#pragma unroll
      for (int q = 0; q < 8; ++q) tile_out[(cb * 8 + q) * 128 + rl] = scale2(v[q], er + ecol[cb * 8 + q]);
    }
  }
}

constexpr int kOz2Threads = 320;  // producer warp, MMA warp, 8 epilogue warps (2 per TMEM lane quarter)
constexpr uint32_t kOz2Stage = kOzPlanes * (kOzTileBytes + kOzBHalfBytes);  // 42 KB: a group-1 k-step
constexpr int kOz2Stages = static_cast<int>(kOzRing / kOz2Stage);

// Persistent: cluster c of C processes items c, c + C, ... (group-1 items first, then group 0; split-
// major; pair blocks in the host's order).  An item is at most one int32-safe chunk (512 k-steps), so
// its accumulators are read out once, straight into the item's own packed partial tile (no
// read-modify-write); the fixed-order reduction (oz_finish_kernel) sums the partials.  The stage ring
// and the accumulator barriers run on across items: the producer streams the next item's operands
// while the epilogue drains the previous item's accumulators (released after its last TMEM load).
__global__ void __launch_bounds__(kOz2Threads, 1) __cluster_dims__(2, 1, 1)
    oz_gram2_kernel(const __grid_constant__ CUtensorMap tmA3g0, const __grid_constant__ CUtensorMap tmB3g0,
                    const __grid_constant__ CUtensorMap tmA3g1, const __grid_constant__ CUtensorMap tmB3g1, OzParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzRing);
  uint64_t* empty = full + kOzMaxStages;
  uint64_t* tfull = empty + kOzMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int per = p.nTiles * p.splits;
  const int nitems = 2 * per;
  const int nst = min(p.max_stages > 0 ? p.max_stages : kOz2Stages, kOz2Stages);

  struct Item {
    int G, split, I, J, nk;
    bool valid;  // this CTA's tile is stored (rank 1 of a single-tile item is idle)
    long long kb;
  };
  auto item_of = [&](int it) {
    Item t;
    t.G = it < per ? 1 : 0;
    const int r = it < per ? it : it - per;
    t.split = r / p.nTiles;
    const int2 pj = p.tiles[r % p.nTiles];  // (a0 << 16 | a1, b): oz_pair_order
    const int a0 = pj.x >> 16, a1 = pj.x & 0xFFFF;
    t.valid = rank == 0 || a1 != 0xFFFF;
    t.I = (rank == 0 || !t.valid) ? a0 : a1;
    t.J = pj.y;
    t.kb = static_cast<long long>(t.split) * p.kPerSplit;
    const long long ke = min(p.ksteps, t.kb + p.kPerSplit);
    t.nk = ke > t.kb ? static_cast<int>(ke - t.kb) : 0;
    return t;
  };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA3g0);
    tma_prefetch_desc(&tmB3g0);
    tma_prefetch_desc(&tmA3g1);
    tma_prefetch_desc(&tmB3g1);
    for (int s = 0; s < kOzMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t leader_full0 = mapa_u32(smem_u32(&full[0]), 0);
  const uint32_t leader_tempty = mapa_u32(smem_u32(tempty), 0);

  if (warp == 0) {
    if (lane == 0) {
      long long gk = 0;  // k-steps issued by this CTA over all its items
      for (int it = cl; it < nitems; it += ncl) {
        const Item t = item_of(it);
        const int planes = t.G ? OzGramGroup<1>::kPlanes : OzGramGroup<0>::kPlanes;
        const uint32_t a_bytes = planes * kOzTileBytes, bytes = planes * (kOzTileBytes + kOzBHalfBytes);
        for (int k = 0; k < t.nk; ++k, ++gk) {
          const int s = static_cast<int>(gk % nst);
          if (gk >= nst) mbar_wait(&empty[s], static_cast<uint32_t>((gk / nst) - 1) & 1);
          if (p.dbg_notma) {
            if (rank == 0) mbar_arrive(&full[s]);
            continue;
          }
          unsigned char* st = smem + s * kOz2Stage;
          const int kr = static_cast<int>((t.kb + k) * 32);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * bytes);
          const uint32_t bar = leader_full0 + s * 8;
          tma_load_3d_pair(st, t.G ? &tmA3g1 : &tmA3g0, bar, t.I * 128, kr, 0);
          tma_load_3d_pair(st + a_bytes, t.G ? &tmB3g1 : &tmB3g0, bar, t.J * 128 + 64 * rank, kr, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // the whole warp runs the issue loop (uniform operands); oz_mma2 elects one lane
      long long gk = 0, gi = 0;  // k-steps and non-empty items so far
      long long t_te = 0, t_full = 0, t_all = clock64();
      for (int it = cl; it < nitems; it += ncl) {
        const Item t = item_of(it);
        if (t.nk == 0) continue;
        const uint32_t a_bytes = (t.G ? OzGramGroup<1>::kPlanes : OzGramGroup<0>::kPlanes) * kOzTileBytes;
        long long c0 = p.dbg ? clock64() : 0;
        if (gi > 0) mbar_wait(tempty, static_cast<uint32_t>(gi - 1) & 1);  // previous item read out
        if (p.dbg) t_te += clock64() - c0;
        tc_fence_after();
        for (int k = 0; k < t.nk; ++k, ++gk) {
          const int s = static_cast<int>(gk % nst);
          c0 = p.dbg ? clock64() : 0;
          mbar_wait(&full[s], static_cast<uint32_t>(gk / nst) & 1);
          if (p.dbg) t_full += clock64() - c0;
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kOz2Stage);
          if (t.G == 0) oz_mma_kstep2<OzGramGroup<0>>(tbase, sa, sa + a_bytes, k == 0);
          else oz_mma_kstep2<OzGramGroup<1>>(tbase, sa, sa + a_bytes, k == 0);
          oz_commit2(&empty[s]);
        }
        oz_commit2(tfull);
        ++gi;
      }
      if (p.dbg && lane == 0) {
        atomicAdd(p.dbg + 0, static_cast<unsigned long long>(t_te));
        atomicAdd(p.dbg + 1, static_cast<unsigned long long>(t_full));
        atomicAdd(p.dbg + 2, static_cast<unsigned long long>(clock64() - t_all));
        atomicAdd(p.dbg + 3, static_cast<unsigned long long>(gk));
        atomicAdd(p.dbg + 4, static_cast<unsigned long long>(gi));
      }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const uint32_t trow = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
    int* ecol = reinterpret_cast<int*>(tslot + 4) + 64 * half;  // this warp pair's 64 column exponents
    long long gi = 0;
    for (int it = cl; it < nitems; it += ncl) {
      const Item t = item_of(it);
      const bool store = t.valid;
      // the accumulator is G[rows I][columns J]; above the diagonal (a leftover computed as its
      // transpose) it is stored transposed into packed tile (J, I)
      const bool trans = t.I < t.J;
      const int PI = trans ? t.J : t.I, PJ = trans ? t.I : t.J;
      double* tile_out = p.ws + static_cast<long long>(t.split * 2 + t.G) * p.wsStride +
                         static_cast<long long>(store ? PI * (PI + 1) / 2 + PJ : 0) * 16384;
      if (t.nk == 0) {  // empty split: a zero partial
        if (store)
          for (int c = half * 64; c < half * 64 + 64; ++c) {
            const int rl = quarter * 32 + lane;
            tile_out[trans ? c * 128 + rl : rl * 128 + c] = 0.0;
          }
        continue;
      }
      // column exponents of this item, staged while the MMAs run (the previous item's read-out by this
      // warp pair is complete: warps of one pair cover disjoint quarters, so sync the pair)
      named_bar_sync_n(1 + half, 128);
      if (quarter == 0 || quarter == 1) {  // two of the pair's four warps fill its 64 entries
        const int c = t.J * 128 + half * 64 + (quarter & 1) * 32 + lane;
        ecol[(quarter & 1) * 32 + lane] = p.exps[min(c, p.Mpad - 1)];
      }
      named_bar_sync_n(1 + half, 128);
      long long c1 = (p.dbg && lane == 0) ? clock64() : 0;
      mbar_wait(tfull, static_cast<uint32_t>(gi) & 1);
      tc_fence_after();
      long long c2 = (p.dbg && lane == 0) ? clock64() : 0;
      OzParams q = p;
      if (!store) q.M = 0;
      if (t.G == 0) oz_readout<0>(trow, q, t.I, t.J, quarter, lane, half * 64, ecol - 64 * half, tile_out, trans);
      else oz_readout<1>(trow, q, t.I, t.J, quarter, lane, half * 64, ecol - 64 * half, tile_out, trans);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty);
      if (p.dbg && lane == 0) {
        atomicAdd(p.dbg + 5, static_cast<unsigned long long>(c2 - c1));
        atomicAdd(p.dbg + 6, static_cast<unsigned long long>(clock64() - c2));
      }
      ++gi;
    }
  }
  tc_fence_before();
  cluster_sync_all();  // all MMAs consumed, all remote arrivals delivered
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

// ---------------------------------------------------------------------------------------------
// K1i: the hidden build H = sigmoid(X W + b) on the INT8 tensor cores -- reference elm.cpp:93-106
// (XW at matrix.cpp:69-77, bias added after the full dot product elm.cpp:102, sigmoid elm.cpp:27).
// Same digit-plane product as the Gram with W's columns and X's rows as the scaled dimensions:
// W[k][c] = 2^(f_c - 54) sum_i dw_i 256^(7-i), X[r][k] = 2^(e_r - 54) sum_j dx_j 256^(7-j), so
// (XW)[r][c] = 2^(f_c + e_r - 60) sum_{w=2..8} a_w 256^(8-w), a_w = sum_{i+j=w} (DW_i^T DX_j^T)[c][r]
// (int32, exact while 7 d 2^14 < 2^31: d <= 16384).  The combination is exact up to one rounding:
// v0 = sum_{w<=5} a_w 256^(5-w) < 2^50 and v1 = sum_{w>=6} a_w 256^(8-w) < 2^41 are exact integers (int64
// Horner, converted exactly without I2F),
// z = fma(v0, 2^24, v1) rounds once, the power-of-two scale is exact.
// The accumulator is H^T: TMEM lane = hidden node, column = sample row, so an epilogue warp holds 32
// consecutive hidden nodes of one row per store (coalesced 256-byte rows of H) and keeps its node's
// exponent and bias in registers.
// Execution: persistent CTA pairs as oz_gram2_kernel (M = 256 hidden nodes, N = 128 rows per item);
// an item runs group 1 (w 6..8, planes 1..7, 3 accumulators, 18 products) over the whole k range,
// then group 0 (w 2..5, planes 1..4, 4 accumulators = all 512 TMEM columns, 10 products).  The
// epilogue reads group 1 into registers (v1, 64 rows per thread), adds group 0, releases TMEM -- the
// next item's group-1 MMAs start -- and runs bias, sigmoid and the stores while they execute.
// Operands: A = planes of W ([plane][k][node], MN-major), B = planes of X^T ([plane][k][row]).
// ---------------------------------------------------------------------------------------------
constexpr int kOzHidThreads = 576;  // producer warp, MMA warp, 16 epilogue warps (4 per TMEM lane quarter)
__global__ void __launch_bounds__(kOzHidThreads, 1) __cluster_dims__(2, 1, 1)
    oz_hidden_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                     OzHidParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzRing);
  uint64_t* empty = full + kOzMaxStages;
  uint64_t* tfull = empty + kOzMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* s_frow = reinterpret_cast<double*>(tslot + 4);  // [128] 2^(row exponent) of this item's rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nitems = p.nP * p.nJ;
  const int nst = kOz2Stages;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA0);
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmA1);
    tma_prefetch_desc(&tmB1);
    for (int s = 0; s < kOzMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 32);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t leader_full0 = mapa_u32(smem_u32(&full[0]), 0);
  const uint32_t leader_tempty = mapa_u32(smem_u32(tempty), 0);
  // item it: row tile J = it / nP (consecutive items share the X rows), node pair P = it % nP

  if (warp == 0) {
    if (lane == 0) {
      long long gk = 0;
      for (int it = cl; it < nitems; it += ncl) {
        const int J = it / p.nP, P = it - J * p.nP;
        for (int ph = 0; ph < 2; ++ph) {
          const int g = 1 - ph;  // group 1 (18 products) first: its MMAs overlap the previous item's math
          const int planes = g ? OzGroup<1>::kPlanes : OzGroup<0>::kPlanes;
          const uint32_t a_bytes = planes * kOzTileBytes, bytes = planes * (kOzTileBytes + kOzBHalfBytes);
          for (int k = 0; k < p.ksteps; ++k, ++gk) {
            const int s = static_cast<int>(gk % nst);
            if (gk >= nst) mbar_wait_sleep(&empty[s], static_cast<uint32_t>((gk / nst) - 1) & 1);
            unsigned char* st = smem + s * kOz2Stage;
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * bytes);
            const uint32_t bar = leader_full0 + s * 8;
            tma_load_3d_pair(st, g ? &tmA1 : &tmA0, bar, (2 * P + rank) * 128, k * 32, 0);
            tma_load_3d_pair(st + a_bytes, g ? &tmB1 : &tmB0, bar, J * 128 + 64 * rank, k * 32, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // whole warp: uniform descriptors, oz_mma2 elects the issuing lane
      long long gk = 0, q = 0;  // k-steps, accumulator phases (two per item)
      for (int it = cl; it < nitems; it += ncl) {
        for (int ph = 0; ph < 2; ++ph, ++q) {
          const int g = 1 - ph;
          if (q > 0) mbar_wait_sleep(tempty, static_cast<uint32_t>(q - 1) & 1);  // previous phase read out
          tc_fence_after();
          const uint32_t a_bytes = (g ? OzGroup<1>::kPlanes : OzGroup<0>::kPlanes) * kOzTileBytes;
          for (int k = 0; k < p.ksteps; ++k, ++gk) {
            const int s = static_cast<int>(gk % nst);
            mbar_wait_sleep(&full[s], static_cast<uint32_t>(gk / nst) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * kOz2Stage);
            if (g == 0) oz_mma_kstep2<OzGroup<0>>(tbase, sa, sa + a_bytes, k == 0);
            else oz_mma_kstep2<OzGroup<1>>(tbase, sa, sa + a_bytes, k == 0);
            oz_commit2(&empty[s]);
          }
          oz_commit2(tfull);
        }
      }
    }
  } else {
    // 16 epilogue warps: warp w reads TMEM lane quarter w % 4; part = (w - 2) / 4 picks 32 of the item's
    // 128 rows, so a thread holds 32 partial sums (64 registers) and the math of four warps per SM
    // sub-partition interleaves
    const int quarter = warp & 3, part = (warp - 2) >> 2;
    const uint32_t trow = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + part * 32;
    long long q = 0;
    for (int it = cl; it < nitems; it += ncl) {
      const int J = it / p.nP, P = it - J * p.nP;
      const int c = (2 * P + rank) * 128 + quarter * 32 + lane;  // this thread's hidden node
      const int r0 = J * 128 + part * 32;                          // its 32 rows
      // this part's 32 row scales (the previous item's stores by these four warps are done)
      named_bar_sync_n(1 + part, 128);
      if (quarter == 0) {
        const int r = r0 + lane;
        s_frow[part * 32 + lane] = pow2i(r < p.N ? min(max(p.rexp[r], -1022), 1023) : 0);
      }
      named_bar_sync_n(1 + part, 128);
      double v[32];
      // group 1 (first): v1 = (a6 256 + a7) 256 + a8, exact (< 2^41)
      mbar_wait(tfull, static_cast<uint32_t>(q) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        int a6[8], a7[8], a8[8];
        tmem_ld8(trow + 0 * 128 + cb * 8, a6);
        tmem_ld8(trow + 1 * 128 + cb * 8, a7);
        tmem_ld8(trow + 2 * 128 + cb * 8, a8);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[cb * 8 + i] = i51_to_f64(((static_cast<long long>(a6[i]) << 8) + a7[i]) * 256 + a8[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty);
      ++q;
      // group 0: v0 = ((a2 256 + a3) 256 + a4) 256 + a5, exact (< 2^50); z = v0 2^24 + v1 (one rounding)
      mbar_wait(tfull, static_cast<uint32_t>(q) & 1);
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        int a2[8], a3[8], a4[8], a5[8];
        tmem_ld8(trow + 0 * 128 + cb * 8, a2);
        tmem_ld8(trow + 1 * 128 + cb * 8, a3);
        tmem_ld8(trow + 2 * 128 + cb * 8, a4);
        tmem_ld8(trow + 3 * 128 + cb * 8, a5);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const long long t = (((static_cast<long long>(a2[i]) << 8) + a3[i]) * 256 + a4[i]) * 256 + a5[i];
          v[cb * 8 + i] = fma(i51_to_f64(t), 0x1.0p24, v[cb * 8 + i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty);  // the next item's group-1 MMAs may start
      ++q;
      // scale, bias after the full dot product, sigmoid (elm.cpp:102, :27), store: the warp writes 32
      // consecutive nodes of each row
      if (c < p.L) {
        // (XW)[r][c] = v 2^(f_c - 60) 2^(e_r): both factors exact powers of two (exponents clamped to the
        // normal range: rows / columns whose maximum is below 2^-962 are outside the supported inputs);
        // z = fma(v 2^(f_c - 60), 2^(e_r), b) rounds once, as the product then the bias addition would
        const double sc = pow2i(min(max(p.cexp[c] - 60, -1022), 1023));
        const double bc = p.bias[c];
        const int nr = min(32, p.N - r0);
        double* dst = p.H + static_cast<long long>(r0) * p.ldh + c;
        const double* frow = s_frow + part * 32;
        double hm = 0.0;  // column maximum of this thread's rows (h >= 0; fmax skips NaN like the scan)
        bool redo = nr < 32;
        if (!redo) {  // whole block, no per-row predicates; range checked once for the 32 values
          int zhi = 0;
          double* out = dst;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const double z = fma(v[i] * sc, frow[i], bc);
            zhi = max(zhi, __double2hiint(z) & 0x7fffffff);
            const double h = sigmoid_in_range(z);
            *out = h;
            out += p.ldh;
            hm = fmax(hm, h);
          }
          redo = zhi > kSigmoidRangeHi;  // some |z| > 700 (or not finite): recompute the block exactly
        }
        if (redo) {
          hm = 0.0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const double z = fma(v[i] * sc, frow[i], bc);
            const double h = sigmoid_exact(z);
            if (i < nr) {
              dst[static_cast<long long>(i) * p.ldh] = h;
              hm = fmax(hm, h);
            }
          }
        }
        // fused column scan of the Gram that follows (oz_colmax_kernel's result for these rows)
        if (p.cmax) atomicMax(p.cmax + c, static_cast<unsigned long long>(__double_as_longlong(hm)));
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

cudaError_t launch_oz_hidden(const CUtensorMap* maps, const OzHidParams& p, cudaStream_t s) {
  const size_t smem = size_t(kOzRing) + 3072;  // ring, barriers, TMEM slot, row scales, alignment (227 KB)
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(oz_hidden_kernel), smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int items = p.nP * p.nJ;
  const int clusters = std::min(items, nsm / 2);
  oz_hidden_kernel<<<2 * clusters, kOzHidThreads, smem, s>>>(maps[0], maps[1], maps[2], maps[3], p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K6i: the training-accuracy pass (elm.cpp:278, 286-300: hits = #rows with argmax(H beta) ==
// argmax(T), strict '>' scans, lowest index on ties) on the INT8 tensor cores.  The Gram's digit
// planes of [H T] (H[r][c] = 2^(e_c - 54) X_rc, column exponents e_c) are reused: folding 2^(e_c) into
// beta, beta'[c][j] = beta[c][j] 2^(e_c) (exact) = 2^(f_j - 54) Y_cj with class exponents f_j, gives
// scores[r][j] = 2^(f_j - 60) sum_{w=2..8} a_w 256^(8-w), a_w = sum_{i+j=w} (DX_i DY_j^T)[r][j]
// (int32: columns of [H T] <= 16384).  Rows of T's columns meet zero beta' rows, so the contraction
// runs over the whole plane row.  Both operands are K-major (the planes are [row][column] with the
// contraction index contiguous): 32-byte TMA boxes at 32-byte swizzle, one MMA k-step per stage.
// Execution: CTA pairs (M = 256 rows, N = 128 classes), an item per 256-row tile: group 1 (18 products)
// then group 0 (10) over the whole contraction; 8 epilogue warps (64 classes per thread), the arg-max
// of the two halves of a row combined through shared memory.
// ---------------------------------------------------------------------------------------------
namespace {
// K-major, 32-byte swizzle: 8-row groups of 32-byte rows 256 B apart (stride byte offset), leading byte
// offset unused (1)
__device__ __forceinline__ uint64_t oz_desc_k32(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(6) << 61);
}
// instruction descriptor: M = 256, N = 128, K-major A and B, s8 x s8 -> s32
constexpr uint32_t kOzIdescK = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
__device__ __forceinline__ void oz_mma2k(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kOzIdescK), "r"(acc));
}
template <int G>
__device__ __forceinline__ void oz_mma_kstep2k(uint32_t tbase, uint32_t sa, uint32_t sb, bool first) {
#pragma unroll
  for (int w = OzGroup<G>::kW0; w < OzGroup<G>::kW0 + OzGroup<G>::kW; ++w) {
#pragma unroll
    for (int i = 1; i < w; ++i) {
      const int j = w - i;
      if (i > OzGroup<G>::kPlanes || j > OzGroup<G>::kPlanes) continue;
      oz_mma2k(tbase + (w - OzGroup<G>::kW0) * 128, oz_desc_k32(sa + (i - 1) * kOzTileBytes),
               oz_desc_k32(sb + (j - 1) * kOzBHalfBytes), (first && i == 1) ? 0u : 1u);
    }
  }
}
}  // namespace

__global__ void __launch_bounds__(kOz2Threads, 1) __cluster_dims__(2, 1, 1)
    oz_scores_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                     const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                     OzScoresParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzRing);
  uint64_t* empty = full + kOzMaxStages;
  uint64_t* tfull = empty + kOzMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  double* s_best = reinterpret_cast<double*>(tslot + 4);  // [128] half 1's best score per row
  int* s_idx = reinterpret_cast<int*>(s_best + 128);       // [128] and its class
  unsigned int& s_hits = *reinterpret_cast<unsigned int*>(s_idx + 128);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nitems = p.nP;
  const int nst = kOz2Stages;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA0);
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmA1);
    tma_prefetch_desc(&tmB1);
    for (int s = 0; s < kOzMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);
    fence_mbar_init();
    s_hits = 0;
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t leader_full0 = mapa_u32(smem_u32(&full[0]), 0);
  const uint32_t leader_tempty = mapa_u32(smem_u32(tempty), 0);

  if (warp == 0) {
    if (lane == 0) {
      long long gk = 0;
      for (int it = cl; it < nitems; it += ncl) {
        for (int ph = 0; ph < 2; ++ph) {
          const int g = 1 - ph;
          const int planes = g ? OzGroup<1>::kPlanes : OzGroup<0>::kPlanes;
          const uint32_t a_bytes = planes * kOzTileBytes, bytes = planes * (kOzTileBytes + kOzBHalfBytes);
          for (int k = 0; k < p.ksteps; ++k, ++gk) {
            const int s = static_cast<int>(gk % nst);
            if (gk >= nst) mbar_wait_sleep(&empty[s], static_cast<uint32_t>((gk / nst) - 1) & 1);
            unsigned char* st = smem + s * kOz2Stage;
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * bytes);
            const uint32_t bar = leader_full0 + s * 8;
            tma_load_3d_pair(st, g ? &tmA1 : &tmA0, bar, k * 32, (2 * it + rank) * 128, 0);
            tma_load_3d_pair(st + a_bytes, g ? &tmB1 : &tmB0, bar, k * 32, 64 * rank, 0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      long long gk = 0, q = 0;
      for (int it = cl; it < nitems; it += ncl) {
        for (int ph = 0; ph < 2; ++ph, ++q) {
          const int g = 1 - ph;
          if (q > 0) mbar_wait_sleep(tempty, static_cast<uint32_t>(q - 1) & 1);
          tc_fence_after();
          const uint32_t a_bytes = (g ? OzGroup<1>::kPlanes : OzGroup<0>::kPlanes) * kOzTileBytes;
          for (int k = 0; k < p.ksteps; ++k, ++gk) {
            const int s = static_cast<int>(gk % nst);
            mbar_wait_sleep(&full[s], static_cast<uint32_t>(gk / nst) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + s * kOz2Stage);
            if (g == 0) oz_mma_kstep2k<0>(tbase, sa, sa + a_bytes, k == 0);
            else oz_mma_kstep2k<1>(tbase, sa, sa + a_bytes, k == 0);
            oz_commit2(&empty[s]);
          }
          oz_commit2(tfull);
        }
      }
    }
  } else {
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const uint32_t trow = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + half * 64;
    const int rl = quarter * 32 + lane;
    unsigned int my_hits = 0;
    long long q = 0;
    for (int it = cl; it < nitems; it += ncl) {
      const int r = (2 * it + rank) * 128 + rl;
      double v[64];
      mbar_wait(tfull, static_cast<uint32_t>(q) & 1);  // group 1: exact integers < 2^41
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 8; ++cb) {
        int a6[8], a7[8], a8[8];
        tmem_ld8(trow + 0 * 128 + cb * 8, a6);
        tmem_ld8(trow + 1 * 128 + cb * 8, a7);
        tmem_ld8(trow + 2 * 128 + cb * 8, a8);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[cb * 8 + i] = i51_to_f64(((static_cast<long long>(a6[i]) << 8) + a7[i]) * 256 + a8[i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty);
      ++q;
      mbar_wait(tfull, static_cast<uint32_t>(q) & 1);  // group 0: exact < 2^50; z = v0 2^24 + v1
      tc_fence_after();
#pragma unroll
      for (int cb = 0; cb < 8; ++cb) {
        int a2[8], a3[8], a4[8], a5[8];
        tmem_ld8(trow + 0 * 128 + cb * 8, a2);
        tmem_ld8(trow + 1 * 128 + cb * 8, a3);
        tmem_ld8(trow + 2 * 128 + cb * 8, a4);
        tmem_ld8(trow + 3 * 128 + cb * 8, a5);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const long long t = (((static_cast<long long>(a2[i]) << 8) + a3[i]) * 256 + a4[i]) * 256 + a5[i];
          v[cb * 8 + i] = fma(i51_to_f64(t), 0x1.0p24, v[cb * 8 + i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty);
      ++q;
      // arg-max over this thread's classes (strict '>' in increasing class order); scores stored on request
      double best = 0.0;
      int bi = -1;
      double* srow = (p.S && r < p.rows) ? p.S + static_cast<long long>(r) * p.lds : nullptr;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const int j = half * 64 + i;
        const double sv = v[i] * __ldg(p.cscale + j);
        if (j < p.m && (bi < 0 || sv > best)) {
          best = sv;
          bi = j;
        }
        if (srow && j < p.m) srow[j] = sv;
      }
      // the two halves of row rl: half 1 posts, half 0 combines (ties stay with the lower classes)
      named_bar_sync_n(1 + quarter, 64);
      if (half == 1) {
        s_best[rl] = best;
        s_idx[rl] = bi;
      }
      named_bar_sync_n(1 + quarter, 64);
      if (half == 0 && r < p.rows) {
        const int b1 = s_idx[rl];
        if (b1 >= 0 && (bi < 0 || s_best[rl] > best)) bi = b1;
        if (p.labels) my_hits += (bi == p.labels[r]) ? 1u : 0u;
        if (p.out_labels) p.out_labels[r] = bi;
      }
    }
    if (half == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_hits += __shfl_xor_sync(0xffffffffu, my_hits, o);
      if (lane == 0 && my_hits) atomicAdd(&s_hits, my_hits);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
  if (threadIdx.x == 0 && s_hits && p.hits) atomicAdd(p.hits, static_cast<unsigned long long>(s_hits));
}

// Digit planes of the folded beta (K-major, [plane][class][column], 128 class rows; rows >= m and
// columns >= L zero) and the class scales 2^(f_j - 60).  One CTA per class row: the exact maximum of
// |beta[c][j] 2^(e_c)|, then the 54-bit integers and their digits (as oz_slice_kernel).
__global__ void __launch_bounds__(256) oz_beta_planes_kernel(const double* __restrict__ beta, long long ldb, int L, int m,
                                                             const int* __restrict__ cexp, int Kpad, int8_t* S,
                                                             double* cscale) {
  const int j = blockIdx.x;
  __shared__ double red[256];
  double mx = 0.0;
  if (j < m)
    for (int c = threadIdx.x; c < L; c += 256) mx = fmax(mx, fabs(scale2(beta[static_cast<long long>(c) * ldb + j], cexp[c])));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  int f = 0;
  if (red[0] > 0.0) frexp(red[0], &f);
  if (threadIdx.x == 0) cscale[j] = pow2i(min(max(f - 60, -1022), 1023));
  constexpr unsigned long long kBias = 0x808080808080ull;
  const long long plane = 128LL * Kpad;
  for (int c = threadIdx.x; c < Kpad; c += 256) {
    long long X = 0;
    if (j < m && c < L) X = __double2ll_rn(scale2(beta[static_cast<long long>(c) * ldb + j], cexp[c] + 54 - f));
    const unsigned long long V = (static_cast<unsigned long long>(X) + kBias) ^ kBias;
#pragma unroll
    for (int i = 0; i < 7; ++i) S[(kOzPlanes - 1 - i) * plane + static_cast<long long>(j) * Kpad + c] = static_cast<int8_t>(V >> (8 * i));
  }
}

// target labels: argmax of each T row (strict '>', lowest index on ties; elm.cpp:291-296)
__global__ void oz_labels_kernel(const double* T, long long ldt, long long rows, int m, int* labels) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double* y = T + i * ldt;
    int a = 0;
    for (int j = 1; j < m; ++j)
      if (y[j] > y[a]) a = j;
    labels[i] = a;
  }
}

cudaError_t launch_oz_beta_planes(const double* beta, long long ldb, int L, int m, const int* cexp, int Kpad, int8_t* S,
                                  double* cscale, cudaStream_t s) {
  oz_beta_planes_kernel<<<128, 256, 0, s>>>(beta, ldb, L, m, cexp, Kpad, S, cscale);
  return cudaGetLastError();
}
cudaError_t launch_oz_labels(const double* T, long long ldt, long long rows, int m, int* labels, cudaStream_t s) {
  const long long blocks = std::min<long long>((rows + 255) / 256, 148LL * 8);
  oz_labels_kernel<<<static_cast<unsigned>(std::max<long long>(blocks, 1)), 256, 0, s>>>(T, ldt, rows, m, labels);
  return cudaGetLastError();
}
cudaError_t launch_oz_scores(const CUtensorMap* maps, const OzScoresParams& p, cudaStream_t s) {
  const size_t smem = size_t(kOzRing) + 3072;  // ring, barriers, TMEM slot, half-row arg-max exchange
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(oz_scores_kernel), smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int clusters = std::min(p.nP, nsm / 2);
  oz_scores_kernel<<<2 * clusters, kOz2Threads, smem, s>>>(maps[0], maps[1], maps[2], maps[3], p);
  return cudaGetLastError();
}

// Fixed-order reduction of the packed partial tiles: G[i][j] = G[j][i] = (acc ? G[i][j] : 0) +
// sum_{slot} part[slot][tile(i, j)][i % 128][j % 128] over the lower triangle (compensated), slots in increasing
// order (split-major, group 0 before group 1 within a split).  One CTA per 32 x 32 block, staged in
// shared memory for the mirrored (transposed) half.
__global__ void __launch_bounds__(256) oz_finish_kernel(const double* __restrict__ ws, long long wsStride, int slots,
                                                        int M, double* G, long long ldg, int accumulate) {
  __shared__ double blk[32][33];
  const int nb = (M + 31) / 32;
  const int b = blockIdx.x;
  int bi = static_cast<int>((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
  while (bi * (bi + 1) / 2 > b) --bi;
  while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
  const int bj = b - bi * (bi + 1) / 2;
  if (bi >= nb) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i0 = bi * 32, j0 = bj * 32;
  for (int rr = ty; rr < 32; rr += 8) {
    const int i = i0 + rr, j = j0 + tx;
    double v = 0.0;
    if (i < M && j <= i) {
      const int I = i >> 7, J = j >> 7;
      const long long off = static_cast<long long>(I * (I + 1) / 2 + J) * 16384 + (i & 127) * 128 + (j & 127);
      // compensated (TwoSum) fixed-order sum: the error stays ~1 ulp of the result however many split
      // partials a small Gram is cut into
      double sum = ws[off], comp = 0.0;
      for (int sl = 1; sl < slots; ++sl) {
        const double x = ws[sl * wsStride + off];
        const double t = add_rn(sum, x);
        const double bp = sub_rn(t, sum);
        comp = add_rn(comp, add_rn(sub_rn(sum, sub_rn(t, bp)), sub_rn(x, bp)));
        sum = t;
      }
      v = add_rn(sum, comp);
      if (accumulate) v = add_rn(G[static_cast<long long>(i) * ldg + j], v);
      G[static_cast<long long>(i) * ldg + j] = v;
    }
    blk[rr][tx] = v;
  }
  __syncthreads();
  for (int rr = ty; rr < 32; rr += 8) {  // mirror: G[j0 + rr][i0 + tx] = blk[tx][rr]
    const int j = j0 + rr, i = i0 + tx;
    if (i < M && j < M && (bi != bj || rr < tx)) G[static_cast<long long>(j) * ldg + i] = blk[tx][rr];
  }
}

cudaError_t launch_oz_finish(const double* ws, long long wsStride, int slots, int M, double* G, long long ldg,
                             int accumulate, cudaStream_t s) {
  const int nb = (M + 31) / 32;
  oz_finish_kernel<<<nb * (nb + 1) / 2, 256, 0, s>>>(ws, wsStride, slots, M, G, ldg, accumulate);
  return cudaGetLastError();
}

// Items of the CTA-pair Gram: two 128 x 128 tiles that share their B column block (one M = 256 x N = 128
// MMA stream), packed as x = (a0 << 16) | a1 (rank 0 reads tile rows a0, rank 1 tile rows a1; a1 = 0xFFFF:
// rank 1 idle), y = b (columns).  Every lower tile (a, c), a >= c, is produced exactly once: column c's
// tiles (c, c), (c + 1, c), ... pair up top-down; when their count nbI - c is odd, the bottom tile
// (nbI - 1, c) is left over and computed as its transpose (rows c, columns nbI - 1), so the leftovers of
// all columns share one B block and pair up too.  (Pairing adjacent tile rows instead computes a tile
// above the diagonal in every diagonal pair block and a padding tile row when nbI is odd: C5's 65 tile
// rows took 1122 items, this takes 1073.)  A transposed item's integer accumulators are the transpose
// of the normal ones (the weight sums include both (i, j) and (j, i)), so the Gram is bitwise the same.
// Launch order: square blocks of B tile rows x B columns (L2 reuse of both operands), leftovers last.
int oz_pair_order(int nbI, int B, int2* out) {
  struct It {
    int a0, a1, b;
  };
  std::vector<It> its, tail;
  std::vector<int> left;
  for (int c = 0; c < nbI; ++c) {
    int a = c;
    for (; a + 1 < nbI; a += 2) its.push_back({a, a + 1, c});
    if (a < nbI) left.push_back(c);  // (nbI - 1, c) left over
  }
  for (size_t i = 0; i < left.size(); i += 2)
    tail.push_back({left[i], i + 1 < left.size() ? left[i + 1] : -1, nbI - 1});
  std::stable_sort(its.begin(), its.end(), [B](const It& u, const It& v) {
    if (u.a0 / B != v.a0 / B) return u.a0 / B < v.a0 / B;
    if (u.b / B != v.b / B) return u.b / B < v.b / B;
    if (u.a0 != v.a0) return u.a0 < v.a0;
    return u.b < v.b;
  });
  int n = 0;
  for (const It& t : its) out[n++] = make_int2((t.a0 << 16) | t.a1, t.b);
  for (const It& t : tail) out[n++] = make_int2((t.a0 << 16) | (t.a1 < 0 ? 0xFFFF : t.a1), t.b);
  return n;
}
// number of items oz_pair_order produces
int oz_pair_items(int nbI) {
  int n = 0, left = 0;
  for (int c = 0; c < nbI; ++c) {
    n += (nbI - c) / 2;
    left += (nbI - c) & 1;
  }
  return n + (left + 1) / 2;
}

cudaError_t launch_oz_gram2(const CUtensorMap* maps, const OzParams& p, cudaStream_t s) {
  const size_t smem = size_t(kOzRing) + 2048;  // ring, barriers, TMEM slot, 128 column exponents, alignment
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(oz_gram2_kernel), smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int items = 2 * p.nTiles * p.splits;
  const int clusters = std::min(items, nsm / 2);
  oz_gram2_kernel<<<2 * clusters, kOz2Threads, smem, s>>>(maps[0], maps[1], maps[2], maps[3], p);
  return cudaGetLastError();
}

cudaError_t launch_oz_colmax(const double* A, long long lda, long long N, int M, unsigned long long* cmax,
                             int num_sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * M, s);
  if (e != cudaSuccess) return e;
  const int cb = (M + 31) / 32;
  long long ry = (8LL * num_sms) / cb;  // up to 8 CTAs of 8 warps per SM in one wave: enough loads in flight
  const long long rmax = (N + 255) / 256;
  if (ry > rmax) ry = rmax;
  if (ry < 1) ry = 1;
  oz_colmax_kernel<<<dim3(cb, static_cast<unsigned>(ry)), 256, 0, s>>>(A, lda, N, M, cmax);
  return cudaGetLastError();
}

// column scan accumulated into cmax (no reset): the T columns of a hidden build whose H columns the
// hidden kernel scanned, or the H of the DMMA hidden kernel
cudaError_t launch_oz_colmax_acc(const double* A, long long lda, long long N, int M, unsigned long long* cmax,
                                 int num_sms, cudaStream_t s) {
  if (N <= 0 || M <= 0) return cudaSuccess;
  const int cb = (M + 31) / 32;
  long long ry = (8LL * num_sms) / cb;
  const long long rmax = (N + 255) / 256;
  if (ry > rmax) ry = rmax;
  if (ry < 1) ry = 1;
  oz_colmax_kernel<<<dim3(cb, static_cast<unsigned>(ry)), 256, 0, s>>>(A, lda, N, M, cmax);
  return cudaGetLastError();
}

cudaError_t launch_oz_slice(const double* A, long long lda, long long N, int M, const unsigned long long* cmax,
                            int* exps, int Mpad, long long Npad, int8_t* S, cudaStream_t s) {
  oz_exps_kernel<<<(Mpad + 255) / 256, 256, 0, s>>>(cmax, M, Mpad, exps);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int gx = (Mpad / 8 + 127) / 128;
  const long long gy = std::min<long long>(Npad, std::max<long long>(1, (148LL * 12 + gx - 1) / gx));
  oz_slice_kernel<<<dim3(gx, static_cast<unsigned>(gy)), 128, 0, s>>>(A, lda, N, M, exps, S,
                                                                     static_cast<long long>(Mpad) * Npad, Mpad, Npad);
  return cudaGetLastError();
}

}  // namespace rbpg
