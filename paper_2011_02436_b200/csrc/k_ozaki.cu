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
// N x M) keep A's row-major layout, [plane][row][column]: MN-major MMA operands, so one TMA box row
// is 128 contiguous bytes (a K-major box row would be 32: four times the L2 requests).
//
// Products.  G[a][b] = 2^(e_a + e_b) sum_{i,j} 2^(4 - 8(i + j)) (D_i^T D_j)[a][b].  Terms with
// i + j >= 9 are below 2^-56 of |G|'s scale and zero-mean (balanced digits): they are dropped, which
// leaves 28 INT8 products per 32-row k-step, grouped by weight w = i + j into int32 accumulators in
// tensor memory: group 0 = w 2..5 (10 products, 4 accumulators, planes 1..4), group 1 = w 6..8 (18
// products, 3 accumulators, planes 1..7).  One CTA computes one (128 x 128 tile, group, K-split)
// item; every 512 k-steps (16384 rows, the int32 headroom: 7 pairs x 32 rows x 2^14 x 512 < 2^31)
// the epilogue warps read the accumulators, combine the weights by Horner's rule in fp64 (exact but
// for the last addition) and add the chunk into the item's fp64 partial in global memory.  The
// fixed-order split reduction (syrk_finish_kernel) sums the partials and mirrors: the result is
// exactly symmetric and, as integer arithmetic is exact, identical columns give bit-identical Gram
// entries wherever they sit (the exact twin ties of C3 survive).
//
// Warp roles (192 threads): warp 0 issues TMA (4-stage ring of one k-step: one 4 KB box {128
// columns, 32 rows} per plane tile, 128-byte swizzle),
// warp 1 allocates TMEM and issues tcgen05.mma from one lane, warps 2-5 are the epilogue (warp w
// reads TMEM lanes 32 (w % 4) .. +31, i.e. tile rows).
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>

namespace rbpg {

namespace {

constexpr int kOzPlanes = 7;
constexpr int kOzMaxStages = 12;
constexpr uint32_t kOzRing = 224 * 1024;  // operand ring: as many whole k-step stages as fit
constexpr int kOzChunk = 512;  // k-steps between accumulator read-outs
constexpr uint32_t kOzTileBytes = 128 * 32;  // one plane tile: 32 rows x 128 columns (bytes)

// instruction descriptor: D s32, A s8, B s8, MN-major both (bits 15, 16), M = 128, N = 128
constexpr uint32_t kOzIdesc =
    (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

// shared-memory matrix descriptor, MN-major, 128-byte swizzle: a K row of 128 bytes (the whole 128-wide
// M / N extent, one swizzle atom wide), 8-row K groups 1024 B apart (stride byte offset); the leading
// byte offset (next 128-element MN atom) is unused at M = N = 128
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(4096 >> 4) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

__device__ __forceinline__ void oz_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kOzIdesc), "r"(acc));
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Group G: number of weights, first weight, planes used, and the (i, j) pairs in issue order
template <int G>
struct OzGroup {
  static constexpr int kW = G == 0 ? 4 : 3;
  static constexpr int kW0 = G == 0 ? 2 : 6;
  static constexpr int kPlanes = G == 0 ? 4 : 7;
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
__global__ void __launch_bounds__(256) oz_slice_kernel(const double* __restrict__ A, long long lda, long long N, int M,
                                                       const int* __restrict__ exps, int8_t* __restrict__ S,
                                                       long long plane_stride, int Mpad, long long Npad) {
  const int groups = Mpad / 8;
  const long long total = Npad * groups;
  for (long long it = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; it < total;
       it += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = it / groups;
    const int c0 = static_cast<int>(it - r * groups) * 8;
    unsigned long long w[kOzPlanes];
#pragma unroll
    for (int p = 0; p < kOzPlanes; ++p) w[p] = 0;
    if (r < N) {
      const double* row = A + r * lda;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = c0 + q;
        long long X = 0;
        if (c < M) X = __double2ll_rn(ldexp(row[c], 54 - exps[c]));
        // balanced base-256 digits from the least significant one
#pragma unroll
        for (int p = kOzPlanes - 1; p >= 1; --p) {
          const long long dgt = ((X + 128) & 255) - 128;
          X = (X - dgt) >> 8;
          w[p] |= (static_cast<unsigned long long>(dgt) & 255ull) << (8 * q);
        }
        w[0] |= (static_cast<unsigned long long>(X) & 255ull) << (8 * q);
      }
    }
#pragma unroll
    for (int p = 0; p < kOzPlanes; ++p)
      *reinterpret_cast<unsigned long long*>(S + p * plane_stride + r * Mpad + c0) = w[p];
  }
}

template <int G>
__device__ __forceinline__ void oz_mma_kstep(uint32_t tbase, uint32_t sa, uint32_t sb, bool first) {
  // pairs (i, j), i + j = w, in increasing w; the first pair of each weight starts its accumulator
  // on the first k-step of a chunk
#pragma unroll
  for (int w = OzGroup<G>::kW0; w < OzGroup<G>::kW0 + OzGroup<G>::kW; ++w) {
#pragma unroll
    for (int i = 1; i < w; ++i) {
      const int j = w - i;
      if (i > OzGroup<G>::kPlanes || j > OzGroup<G>::kPlanes) continue;
      const uint64_t da = oz_desc(sa + (i - 1) * kOzTileBytes);
      const uint64_t db = oz_desc(sb + (j - 1) * kOzTileBytes);
      oz_mma(tbase + (w - OzGroup<G>::kW0) * 128, da, db, (first && i == 1) ? 0u : 1u);
    }
  }
}

template <int G>
__device__ __forceinline__ void oz_epilogue_chunk(uint32_t tbase, int quarter, int lane, const OzParams& p, int I,
                                                  int J, double* part, bool first_chunk) {
  constexpr int kW = OzGroup<G>::kW, kW0 = OzGroup<G>::kW0;
  const int r = I * 128 + quarter * 32 + lane;
  const uint32_t trow = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
  const int er = r < p.M ? p.exps[r] : 0;
  for (int cb = 0; cb < 4; ++cb) {
    double v[32];
    int c32[32];
    tmem_ld32(trow + (kW - 1) * 128 + cb * 32, c32);
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = static_cast<double>(c32[q]);
#pragma unroll
    for (int a = kW - 2; a >= 0; --a) {
      tmem_ld32(trow + a * 128 + cb * 32, c32);
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = fma(v[q], 0x1.0p-8, static_cast<double>(c32[q]));
    }
    const int cbase = J * 128 + cb * 32;
    if (r < p.M) {
      double* dst = part + static_cast<long long>(r) * p.ldg + cbase;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int c = cbase + q;
        if (c < p.M) {
          const double s = ldexp(v[q], er + p.exps[c] + 4 - 8 * kW0);
          dst[q] = first_chunk ? s : dst[q] + s;
        }
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(192, 1) oz_gram_kernel(const __grid_constant__ CUtensorMap tmS, OzParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOzRing);
  uint64_t* empty = full + kOzMaxStages;
  uint64_t* tfull = empty + kOzMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // item decode: split-major; within a split the tiles in the host's order (square blocks of tiles, so
  // the CTAs of a wave share few operand panels), each tile's group-1 item (the longer) before its
  // group-0 item (both read planes 1..4 of the same panels)
  const int item = blockIdx.x;
  int split, G, ti;
  if (p.interleave) {
    split = item / (2 * p.nTiles);
    const int r2 = item % (2 * p.nTiles);
    G = (r2 & 1) ? 0 : 1;
    ti = r2 >> 1;
  } else {  // all group-1 items first (longest first), split-major
    const int per = p.nTiles * p.splits;
    G = item < per ? 1 : 0;
    const int r = item < per ? item : item - per;
    split = r / p.nTiles;
    ti = r % p.nTiles;
  }
  const int2 tij = p.tiles[ti];
  const int I = tij.x, J = tij.y;
  const bool diag = I == J;
  const long long kb = static_cast<long long>(split) * p.kPerSplit;
  const long long ke = min(p.ksteps, kb + p.kPerSplit);
  const int nk = ke > kb ? static_cast<int>(ke - kb) : 0;
  const int planes = G == 0 ? OzGroup<0>::kPlanes : OzGroup<1>::kPlanes;
  const uint32_t stage_bytes = (diag ? 1u : 2u) * planes * kOzTileBytes;
  const int nst = min(p.max_stages > 0 ? p.max_stages : kOzMaxStages, static_cast<int>(kOzRing / stage_bytes));

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmS);
    for (int s = 0; s < kOzMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  double* part = p.ws + static_cast<long long>(split * 2 + G) * p.wsStride;

  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < nk; ++k) {
        const int s = k % nst;
        if (k >= nst) mbar_wait(&empty[s], ((k / nst) - 1) & 1);
        unsigned char* st = smem + s * stage_bytes;
        const int kr = static_cast<int>((kb + k) * 32);
        mbar_arrive_expect_tx(&full[s], stage_bytes);
        for (int pl = 0; pl < planes; ++pl) {
          const int prow = static_cast<int>(pl * p.Npad + kr);
          tma_load_2d(st + pl * kOzTileBytes, &tmS, &full[s], I * 128, prow);
          if (!diag) tma_load_2d(st + (planes + pl) * kOzTileBytes, &tmS, &full[s], J * 128, prow);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int k = 0; k < nk; ++k) {
        const int s = k % nst;
        const int kc = k % kOzChunk;
        if (kc == 0 && k > 0) {  // the epilogue must have drained the previous chunk
          mbar_wait(tempty, ((k / kOzChunk) - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], (k / nst) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * stage_bytes);
        const uint32_t sb = diag ? sa : sa + planes * kOzTileBytes;
        if (G == 0) oz_mma_kstep<0>(tbase, sa, sb, kc == 0);
        else oz_mma_kstep<1>(tbase, sa, sb, kc == 0);
        oz_commit(&empty[s]);
        if (kc == kOzChunk - 1 || k == nk - 1) oz_commit(tfull);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int nchunks = (nk + kOzChunk - 1) / kOzChunk;
    for (int ch = 0; ch < nchunks; ++ch) {
      mbar_wait(tfull, ch & 1);
      tc_fence_after();
      if (G == 0) oz_epilogue_chunk<0>(tbase, quarter, lane, p, I, J, part, ch == 0);
      else oz_epilogue_chunk<1>(tbase, quarter, lane, p, I, J, part, ch == 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
    if (nchunks == 0) {  // empty split: the partial is zero
      const int r = I * 128 + quarter * 32 + lane;
      if (r < p.M)
        for (int c = J * 128; c < min(p.M, J * 128 + 128); ++c) part[static_cast<long long>(r) * p.ldg + c] = 0.0;
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

size_t oz_gram_smem() { return size_t(kOzRing) + 1024 + 256; }

// Lower-triangle tiles of an nbI x nbI tile grid in square blocks of B x B tiles (block rows and columns
// in lower-triangle order, tiles row-major inside a block): about num_sms consecutive tiles then read
// ~2 sqrt(num_sms) panels instead of up to nbI + 3.
void oz_tile_order(int nbI, int B, int2* out) {
  int n = 0;
  for (int bi = 0; bi * B < nbI; ++bi)
    for (int bj = 0; bj <= bi; ++bj)
      for (int i = bi * B; i < std::min(nbI, bi * B + B); ++i)
        for (int j = bj * B; j < std::min(i + 1, bj * B + B); ++j) out[n++] = make_int2(i, j);
}

cudaError_t launch_oz_colmax(const double* A, long long lda, long long N, int M, unsigned long long* cmax,
                             int num_sms, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * M, s);
  if (e != cudaSuccess) return e;
  const int cb = (M + 31) / 32;
  long long ry = (2LL * num_sms + cb - 1) / cb;
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
  const long long work = Npad * (Mpad / 8);
  const unsigned grid = static_cast<unsigned>(std::min<long long>((work + 255) / 256, 148LL * 16));
  oz_slice_kernel<<<grid, 256, 0, s>>>(A, lda, N, M, exps, S, static_cast<long long>(Mpad) * Npad, Mpad, Npad);
  return cudaGetLastError();
}

cudaError_t launch_oz_gram(const CUtensorMap& tmS, const OzParams& p, cudaStream_t s) {
  const size_t smem = oz_gram_smem();
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(oz_gram_kernel), smem);
  if (e != cudaSuccess) return e;
  oz_gram_kernel<<<2 * p.nTiles * p.splits, 192, smem, s>>>(tmS, p);
  return cudaGetLastError();
}

}  // namespace rbpg
