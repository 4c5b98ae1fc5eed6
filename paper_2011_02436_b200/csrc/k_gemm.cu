// FP64 tensor-core (DMMA) kernels fed by TMA:
//   K1 hidden_kernel : H = sigmoid(X W + b)      -- reference elm.cpp:93-106 (matmul at
//                      matrix.cpp:69-77, bias added after the dot at elm.cpp:102, sigmoid elm.cpp:27)
//   K2 syrk_kernel   : lower-tile G = H^T H (+ H^T T tiles), split-K with a fixed-order
//                      reduction -- reference linalg.cpp:179-184 (Gram), matrix.cpp:79-87
//                      (matmul_at for H^T T); trail_kernel: the rank-kb trailing update of the
//                      pivoted Cholesky (linalg.cpp:237-244)
//   gemm_kernel      : generic C = alpha op(A) op(B) + beta C for the small solve-side products
//
// Data layout: every matrix is row-major fp64 with an even leading dimension
// (16-byte TMA stride rule).  Output tiles are 128x128 per CTA, 8 warps each
// owning a 64x32 sub-tile as 4x4 m16n8k4 DMMA fragments (64 fp64 accumulators
// per thread).  Shared-memory operand tiles are stored "MN-major" ([k][mn], mn
// contiguous) and read as 16-byte pairs: MMA row g / g+8 (or n-tile pair)
// are mapped onto adjacent columns so each quarter-warp reads one 128-byte
// row, which is bank-conflict free without padding.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

#include <algorithm>
#include <cstdio>

namespace rbpg {

namespace {

// 128B-swizzled [row][16] fp64 tile written by TMA (CU_TENSOR_MAP_SWIZZLE_128B):
// the 16-byte chunk index inside each 128-byte row is XORed with (row & 7).
__device__ __forceinline__ int swz16(int row, int col) {
  return row * 16 + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}

// Round a dynamic-shared-memory pointer up to 1024 B (128B-swizzle atom) by pointer
// arithmetic on the shared base, so the compiler keeps shared-window addressing (LDS,
// not generic LD) for every derived pointer.
__device__ __forceinline__ unsigned char* align1024(unsigned char* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

}  // namespace

// ============================================================================
// K1: hidden-layer build.  Row tile 128 (samples) x column tile BN (hidden nodes).  BN = 64 keeps
// the accumulators at 32 per thread so two CTAs share an SM: one CTA's sigmoid epilogue (FP64
// CUDA-core pipe) overlaps the other's DMMA main loop (tensor pipe).  BN = 128 (one CTA per SM)
// serves the plain transposed product of the pseudo-inverse, which has no epilogue to hide.
// ============================================================================
template <int BN, int NS = 4>
__global__ void __launch_bounds__(kGemmThreads, BN == 32 ? 3 : (BN == 64 ? 2 : 1))
    hidden_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, HiddenParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  double* Xs = reinterpret_cast<double*>(smem);        // [stage][128 rows][16] swizzled
  // W rows padded by 4 doubles (TMA box {BN + 4, 16}): the k rows of a quarter-warp's 16-byte
  // fragment loads then start on different banks (an unpadded 512 / 1024-byte row stride maps
  // the 4 k rows onto the same banks: 4-way conflicts)
  constexpr int BNP = BN + 4;
  double* Ws = Xs + NS * kTile * kBK;             // [stage][16][BNP]
  uint64_t* full = reinterpret_cast<uint64_t*>(Ws + NS * kBK * BNP);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int l0 = blockIdx.x * BN, n0 = blockIdx.y * kTile;
  const int ktiles = (p.d + kBK - 1) / kBK;
  constexpr uint32_t kStageBytes = (kTile + BNP) * kBK * sizeof(double);

  if (tid == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < NS && s < ktiles; ++s) {
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(Xs + s * kTile * kBK, &tmX, &full[s], s * kBK, n0);
      tma_load_2d(Ws + s * kBK * BNP, &tmW, &full[s], l0, s * kBK);
    }
  }

  // warp tile: 64 x 32 (BN = 128: 2 x 4 warps), 32 x 32 (BN = 64: 4 x 2 warps) or 16 x 32 (BN = 32: 8 x 1)
  constexpr int MT = BN == 128 ? 4 : (BN == 64 ? 2 : 1);
  constexpr int WARPS_N = BN / 32;
  const int wm = (warp / WARPS_N) * (MT * 16), wn = (warp % WARPS_N) * 32;
  double acc[MT][4][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % NS;
    mbar_wait(&full[s], (kt / NS) & 1);
    const double* xs = Xs + s * kTile * kBK;
    const double* ws = Ws + s * kBK * BNP;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kc = ks * 4 + t;
      double a[MT][2], b[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        // MMA rows g, g + 8 <-> tile rows 2g, 2g + 1: a half-warp's 8-byte loads then cover the
        // 8 swizzled 16-byte chunks once (rows g, g + 1 would pair up on the same chunks)
        const int r = wm + mt * 16 + 2 * g;
        a[mt][0] = xs[swz16(r, kc)];
        a[mt][1] = xs[swz16(r + 1, kc)];
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(ws + kc * BNP + wn + pp * 16 + 2 * g);
        b[2 * pp] = w.x;
        b[2 * pp + 1] = w.y;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
    __syncthreads();
    if (tid == 0 && kt + NS < ktiles) {
      const int kn = kt + NS;
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(Xs + s * kTile * kBK, &tmX, &full[s], kn * kBK, n0);
      tma_load_2d(Ws + s * kBK * BNP, &tmW, &full[s], l0, kn * kBK);
    }
  }

  if (p.transposed) {  // plain product stored transposed: H[c][r] (pseudo-inverse H^+ = G^-1 H^T)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = n0 + wm + mt * 16 + 2 * g + (q >> 1);
          const int c = l0 + wn + (nt >> 1) * 16 + 4 * t + 2 * (q & 1) + (nt & 1);
          if (r < p.N && c < p.L) p.H[(long long)c * p.ldh + r] = acc[mt][nt][q];
        }
    return;
  }

  // augmented rows [H T]: the last column tile also copies this row tile's targets
  if (p.T && blockIdx.x == gridDim.x - 1) {
    for (int e = tid; e < kTile * p.m; e += kGemmThreads) {
      const int rr = e / p.m, j = e - rr * p.m, r = n0 + rr;
      if (r < p.N) p.H[(long long)r * p.ldh + p.L + j] = p.T[(long long)r * p.ldt + j];
    }
  }

  // epilogue: bias after the full dot product, then sigmoid (elm.cpp:102, :27)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int cb = l0 + wn + pp * 16 + 4 * t;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int r = n0 + wm + mt * 16 + 2 * g + half;
        if (r >= p.N) continue;
        double v[4] = {acc[mt][2 * pp][2 * half], acc[mt][2 * pp + 1][2 * half], acc[mt][2 * pp][2 * half + 1],
                       acc[mt][2 * pp + 1][2 * half + 1]};
        double h[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = cb + q;
          const double z = add_rn(v[q], c < p.L ? p.bias[c] : 0.0);
          h[q] = recip_ge1(1.0 + exp(-z));
        }
        double* dst = p.H + (long long)r * p.ldh + cb;
        if (cb + 3 < p.L) {
          reinterpret_cast<double2*>(dst)[0] = make_double2(h[0], h[1]);
          reinterpret_cast<double2*>(dst)[1] = make_double2(h[2], h[3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (cb + q < p.L) dst[q] = h[q];
        }
      }
    }
  }
}

// ============================================================================
// K2: SYRK-TN family.  A (kRows x M) row-major via tmA; B = A for Gram tiles,
// B = T (kRows x mB) via tmB for the H^T T tiles.
// ============================================================================
// PART 0: every lower tile (+ T tiles).  PART 1: off-diagonal lower tiles (+ T tiles) only -- the
// diagonal ones go to syrk_diag_kernel, which this grid overlaps as its programmatic dependent.
template <int TILE, int PART = 0>
__global__ void __launch_bounds__(TILE == 128 ? 256 : 128, 1)
    syrk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SyrkParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  // operand rows padded by 4 doubles (TMA box {TILE + 4, 16}): a quarter-warp's 16-byte fragment
  // loads from 4 consecutive k rows then start on different banks (no 4-way conflicts)
  constexpr int TP = TILE + 4;
  double* As = reinterpret_cast<double*>(smem);   // [stage][16][TP]
  double* Bs = As + kStages * kBK * TP;          // [stage][16][TP]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + kStages * kBK * TP);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;

  // ---- tile decode: lower-triangular Gram tiles first, then H^T T tiles
  const int bx = blockIdx.x;
  int I, J;
  bool isT;
  const int nLower = PART == 1 ? p.nbI * (p.nbI - 1) / 2 : p.nGram;
  if (bx < nLower) {
    int i = static_cast<int>((sqrt(8.0 * bx + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > bx) --i;
    while ((i + 1) * (i + 2) / 2 <= bx) ++i;
    I = i;
    J = bx - i * (i + 1) / 2;
    if (PART == 1) ++I;  // strictly lower: tile (i + 1, j), j <= i
    isT = false;
  } else {
    const int tt = bx - nLower;
    I = tt / p.nbT;
    J = tt % p.nbT;
    isT = true;
  }
  const CUtensorMap* mapB = isT ? &tmB : &tmA;
  const int i0 = I * TILE, j0 = J * TILE;

  const long long kbeg = (long long)blockIdx.y * p.kPerSplit;
  long long kend = kbeg + p.kPerSplit;
  if (kend > p.kRows) kend = p.kRows;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kBK - 1) / kBK) : 0;
  constexpr uint32_t kStageBytes = 2u * TP * kBK * sizeof(double);

  if (tid == 0) {
    tma_prefetch_desc(&tmA);
    if (isT) tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  tl_mark(p.tl, p.tl_slot, 0);
  pdl_trigger();  // PART 1: the diagonal-tile grid (this grid's dependent) may start launching
  if (PART == 0) pdl_wait();  // launched programmatic-dependent: the producer of A may still be finishing
  tl_mark(p.tl, p.tl_slot, 1);
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages && s < ktiles; ++s) {
      const int kr = static_cast<int>(kbeg + s * kBK);
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(As + s * kBK * TP, &tmA, &full[s], i0, kr);
      tma_load_2d(Bs + s * kBK * TP, mapB, &full[s], j0, kr);
    }
  }

  constexpr int WM = TILE / 2, WARPS_N = TILE / 32, MT = WM / 16;
  const int wm = (warp / WARPS_N) * WM, wn = (warp % WARPS_N) * 32;
  double acc[MT][4][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % kStages;
    mbar_wait(&full[s], (kt / kStages) & 1);
    const double* as = As + s * kBK * TP;
    const double* bs = Bs + s * kBK * TP;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kc = ks * 4 + t;
      double a[MT][2], b[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double2 v = *reinterpret_cast<const double2*>(as + kc * TP + wm + mt * 16 + 2 * g);
        a[mt][0] = v.x;   // MMA row g   <-> tile row 2g
        a[mt][1] = v.y;   // MMA row g+8 <-> tile row 2g+1
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(bs + kc * TP + wn + pp * 16 + 2 * g);
        b[2 * pp] = w.x;       // n-tile 2pp   col g <-> tile col 16pp + 2g
        b[2 * pp + 1] = w.y;   // n-tile 2pp+1 col g <-> tile col 16pp + 2g + 1
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
    __syncthreads();
    if (tid == 0 && kt + kStages < ktiles) {
      const int kr = static_cast<int>(kbeg + (long long)(kt + kStages) * kBK);
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(As + s * kBK * TP, &tmA, &full[s], i0, kr);
      tma_load_2d(Bs + s * kBK * TP, mapB, &full[s], j0, kr);
    }
  }

  // ---- epilogue.  Thread holds rows r, r+1 (r even) x cols c..c+3 per (mt, pp).
  const int split = p.split0 + blockIdx.y;

#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int r0 = i0 + wm + mt * 16 + 2 * g;
      const int c0 = j0 + wn + pp * 16 + 4 * t;
      double v[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        v[h][0] = acc[mt][2 * pp][2 * h];
        v[h][1] = acc[mt][2 * pp + 1][2 * h];
        v[h][2] = acc[mt][2 * pp][2 * h + 1];
        v[h][3] = acc[mt][2 * pp + 1][2 * h + 1];
      }
      if (isT) {
        double* out = (p.mode == kSyrkPartial) ? p.wsT + split * p.wsTStride : p.HtT;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + h;
          if (r >= p.M) continue;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q < p.mB) out[(long long)r * p.ldt + c0 + q] = v[h][q];
        }
        continue;
      }
      if (p.mode == kSyrkPartial) {
        double* out = p.ws + split * p.wsStride;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + h;
          if (r >= p.M) continue;
          double* dst = out + (long long)r * p.ldg + c0;
          if (c0 + 3 < p.M) {
            reinterpret_cast<double2*>(dst)[0] = make_double2(v[h][0], v[h][1]);
            reinterpret_cast<double2*>(dst)[1] = make_double2(v[h][2], v[h][3]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (c0 + q < p.M) dst[q] = v[h][q];
          }
        }
        continue;
      }
      // direct: lower element (r >= c) written at (r, c) and mirrored to (c, r)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + h;
        if (r >= p.M) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q;
          if (c >= p.M || c > r) continue;
          p.G[(long long)r * p.ldg + c] = v[h][q];
          p.G[(long long)c * p.ldg + r] = v[h][q];
        }
      }
    }
  }
  tl_mark(p.tl, p.tl_slot, 2);
}

// Fragment pairs of a diagonal 128-wide Gram tile: row group mt (16 rows) x column pair pp (two n8
// fragments, 16 columns) with pp <= mt, i.e. the 72 of 128 (m16, n8) fragments that touch the lower
// triangle.  SMSP s = warp & 3 owns row groups s and 7 - s: 9 pairs (18 fragments, equal tensor-pipe
// work per SMSP), 5 pairs for warp s and 4 for warp s + 4 (the SMSP's pipe is shared, so the split
// within it does not matter).  Whole pairs per warp let every B fragment load be one 16-byte load
// feeding two DMMAs (split pairs compiled to 8-byte loads with 4-way bank conflicts).
template <int DS, int DH>
struct DiagPairs {
  static constexpr int kFirst = DS + 1;  // pairs of row group DS
  static constexpr int kP0 = DH == 0 ? 0 : 5, kNP = DH == 0 ? 5 : 4;
  static __device__ __forceinline__ int mt(int P) { return P < kFirst ? DS : 7 - DS; }
  static __device__ __forceinline__ int pp(int P) { return P < kFirst ? P : P - kFirst; }
};

// One 16-deep k-slab for warp (DS, DH): its kNP pairs accumulate into acc[2i], acc[2i + 1].
template <int DS, int DH>
__device__ __forceinline__ void diag_step(double (&acc)[10][4], const double* as, const double* bs, int g, int t) {
  using DP = DiagPairs<DS, DH>;
#pragma unroll
  for (int ks = 0; ks < kBK / 4; ++ks) {
    const int kc = ks * 4 + t;
#pragma unroll
    for (int i = 0; i < DP::kNP; ++i) {
      const int P = DP::kP0 + i;
      const double2 a = *reinterpret_cast<const double2*>(as + kc * 132 + DP::mt(P) * 16 + 2 * g);
      const double2 bw = *reinterpret_cast<const double2*>(bs + kc * 132 + DP::pp(P) * 16 + 2 * g);
      dmma_16x8x4(acc[2 * i], a.x, a.y, bw.x);
      dmma_16x8x4(acc[2 * i + 1], a.x, a.y, bw.y);
    }
  }
}

// Diagonal 128 x 128 Gram tiles (direct or split-K partial): only the lower-triangle fragment pairs
// are computed.  Every element sees the same DMMA k-sequence as in a full tile (exact twin ties
// survive).
template <int DS, int DH>
__device__ __forceinline__ void diag_tile_loop(double (&acc)[10][4], double* As, double* Bs,
                                               uint64_t* full, const CUtensorMap* tmA, int i0, long long kbeg,
                                               int ktiles, int tid, int g, int t) {
  constexpr uint32_t kStageBytes = 2u * 132 * kBK * sizeof(double);
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % kStages;
    mbar_wait(&full[s], (kt / kStages) & 1);
    diag_step<DS, DH>(acc, As + s * kBK * 132, Bs + s * kBK * 132, g, t);
    __syncthreads();
    if (tid == 0 && kt + kStages < ktiles) {
      const int kr = static_cast<int>(kbeg + (long long)(kt + kStages) * kBK);
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(As + s * kBK * 132, tmA, &full[s], i0, kr);
      tma_load_2d(Bs + s * kBK * 132, tmA, &full[s], i0, kr);
    }
  }
}

template <int DS, int DH>
__device__ __forceinline__ void diag_store(const double (&acc)[10][4], double* out, const SyrkParams& p, int i0,
                                           int g, int t) {
  using DP = DiagPairs<DS, DH>;
#pragma unroll
  for (int i = 0; i < DP::kNP; ++i) {
    const int P = DP::kP0 + i, mt = DP::mt(P), pp = DP::pp(P);
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int nt = 2 * pp + f;
      // fragment (mt, nt): MMA row g / g+8 <-> tile row mt*16 + 2g / +1; MMA col j <-> tile col
      // (nt >> 1) * 16 + 2j + (nt & 1); lower elements only (mirrored in direct mode)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = i0 + mt * 16 + 2 * g + (e >> 1);
        const int c = i0 + (nt >> 1) * 16 + 2 * (2 * t + (e & 1)) + (nt & 1);
        if (r >= p.M || c > r) continue;
        out[(long long)r * p.ldg + c] = acc[2 * i + f][e];
        if (p.mode != kSyrkPartial) out[(long long)c * p.ldg + r] = acc[2 * i + f][e];
      }
    }
  }
}

__global__ void __launch_bounds__(256, 1)
    syrk_diag_kernel(const __grid_constant__ CUtensorMap tmA, SyrkParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  double* As = reinterpret_cast<double*>(smem);
  double* Bs = As + kStages * kBK * 132;  // padded rows, as in syrk_kernel
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + kStages * kBK * 132);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int I = blockIdx.x, i0 = I * 128;
  const long long kbeg = (long long)blockIdx.y * p.kPerSplit;
  long long kend = kbeg + p.kPerSplit;
  if (kend > p.kRows) kend = p.kRows;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kBK - 1) / kBK) : 0;
  constexpr uint32_t kStageBytes = 2u * 132 * kBK * sizeof(double);
  if (tid == 0) {
    tma_prefetch_desc(&tmA);
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages && s < ktiles; ++s) {
      const int kr = static_cast<int>(kbeg + s * kBK);
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(As + s * kBK * 132, &tmA, &full[s], i0, kr);
      tma_load_2d(Bs + s * kBK * 132, &tmA, &full[s], i0, kr);
    }
  }
  double acc[10][4];
#pragma unroll
  for (int i = 0; i < 10; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  switch (warp) {  // compile-time fragment lists per warp
    case 0: diag_tile_loop<0, 0>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 1: diag_tile_loop<1, 0>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 2: diag_tile_loop<2, 0>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 3: diag_tile_loop<3, 0>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 4: diag_tile_loop<0, 1>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 5: diag_tile_loop<1, 1>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    case 6: diag_tile_loop<2, 1>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
    default: diag_tile_loop<3, 1>(acc, As, Bs, full, &tmA, i0, kbeg, ktiles, tid, g, t); break;
  }
  pdl_wait();  // completes only after the off-diagonal grid (its primary): the reduction follows
  double* out = (p.mode == kSyrkPartial) ? p.ws + (p.split0 + blockIdx.y) * p.wsStride : p.G;
  switch (warp) {
    case 0: diag_store<0, 0>(acc, out, p, i0, g, t); break;
    case 1: diag_store<1, 0>(acc, out, p, i0, g, t); break;
    case 2: diag_store<2, 0>(acc, out, p, i0, g, t); break;
    case 3: diag_store<3, 0>(acc, out, p, i0, g, t); break;
    case 4: diag_store<0, 1>(acc, out, p, i0, g, t); break;
    case 5: diag_store<1, 1>(acc, out, p, i0, g, t); break;
    case 6: diag_store<2, 1>(acc, out, p, i0, g, t); break;
    default: diag_store<3, 1>(acc, out, p, i0, g, t); break;
  }
}

// Trailing update of the blocked pivoted Cholesky (K2 in trailing mode, behind every panel but
// the last): G_new[t0 + r][t0 + c] = G_old[lab[t0 + r]][lab[t0 + c]] - sum_cc PcT[cc][r] PcT[cc][c]
// for r >= c.  K = the panel width (<= 64), so every k-stage is loaded up front.  The G_old gathers
// (two dependent L2 round trips: label, then entry) are issued as cp.async into shared memory
// before the DMMAs, in a thread-interleaved layout (element e of thread t at [e][t]: conflict-free),
// so their latency hides under the tensor-core work.  G_old is read through its lower triangle
// (G[max][min]) and G_new is written lower-only unless p.mirror (the next panel reads whole rows).
// TILE 32 (64 threads) for the small late updates: four times the CTAs per DMMA of a 64-wide tile.
// KS: k-stages resident (4 = the whole rank-64 panel loaded up front; 2 or 1 = the panel streamed
// through fewer stages, reloaded as they are consumed, so three or four CTAs fit on an SM)
// NT: 2 * TILE threads (warps of (TILE / 2) x 32), or 4 * TILE (warps of (TILE / 4) x 32: twice the warps
// issuing DMMAs per tile -- a warp issues at most one DMMA per ~34 cycles, so the pipe needs several)
template <int TILE, int KS = kStages, int NT = 2 * TILE>
__global__ void __launch_bounds__(NT, NT == 4 * TILE ? 3 : 1)
    trail_kernel(const __grid_constant__ CUtensorMap tmP, SyrkParams p) {
  constexpr int TP = TILE + 4;      // padded smem rows (TMA box {TILE + 4, 16})
  constexpr int WARPS_N = TILE / 32;
  constexpr int WARPS_M = NT / 32 / WARPS_N;
  constexpr int MT = TILE / WARPS_M / 16;  // m16 fragments per warp
  constexpr int NG = MT * 2 * 2 * 4;  // G_old entries per thread
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  double* As = reinterpret_cast<double*>(smem);  // [stage][16][TP]
  double* Bs = As + KS * kBK * TP;               // [stage][16][TP]
  double* gsm = Bs + KS * kBK * TP;              // [NG][NT]
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + NG * NT);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  int I, J;
  {
    const int bx = blockIdx.x;
    int i = static_cast<int>((sqrtf(8.0f * bx + 1.0f) - 1.0f) * 0.5f);
    while (i * (i + 1) / 2 > bx) --i;
    while ((i + 1) * (i + 2) / 2 <= bx) ++i;
    I = i;
    J = bx - i * (i + 1) / 2;
  }
  const int i0 = I * TILE, j0 = J * TILE;
  const bool diag = I == J;
  const int ktiles = static_cast<int>((p.kRows + kBK - 1) / kBK);  // <= kStages (launcher checks)
  const uint32_t stage_bytes = (diag ? 1u : 2u) * TP * kBK * sizeof(double);
  if (tid == 0) {
    tma_prefetch_desc(&tmP);
    for (int s = 0; s < KS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  tl_mark(p.tl, p.tl_slot, 0);
  if (!p.late_trigger) pdl_trigger();
  pdl_wait();  // the panel that wrote PcT / lab may still be finishing
  if (p.late_trigger) pdl_trigger();
  tl_mark(p.tl, p.tl_slot, 1);
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < ktiles && s < KS; ++s) {
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      tma_load_2d(As + s * kBK * TP, &tmP, &full[s], i0, s * kBK);
      if (!diag) tma_load_2d(Bs + s * kBK * TP, &tmP, &full[s], j0, s * kBK);
    }
  }
  const int wm = (warp / WARPS_N) * (TILE / WARPS_M), wn = (warp % WARPS_N) * 32;
  const int M = p.M, off = p.off;
  {  // G_old gathers -> gsm
    int sr[MT][2], sc[2][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = i0 + wm + mt * 16 + 2 * g + h;
        sr[mt][h] = r < M ? __ldg(p.lab + off + r) : 0;
      }
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = j0 + wn + pp * 16 + 4 * t + q;
        sc[pp][q] = c < M ? __ldg(p.lab + off + c) : 0;
      }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int r = i0 + wm + mt * 16 + 2 * g + h, c = j0 + wn + pp * 16 + 4 * t + q;
            if (r < M && c <= r) {
              const int a = max(sr[mt][h], sc[pp][q]), b = min(sr[mt][h], sc[pp][q]);
              cp_async8(gsm + (((mt * 2 + pp) * 2 + h) * 4 + q) * NT + tid, p.Gold + (long long)a * p.ldgo + b);
            }
          }
    cp_async_commit();
  }

  double acc[MT][4][4];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;
  for (int kt = 0; kt < ktiles; ++kt) {
    if (KS < kStages && kt > 0 && kt % KS == 0) {  // stages consumed: the next k-tiles into them
      __syncthreads();
      if (tid == 0)
        for (int s = 0; s < KS && kt + s < ktiles; ++s) {
          mbar_arrive_expect_tx(&full[s], stage_bytes);
          tma_load_2d(As + s * kBK * TP, &tmP, &full[s], i0, (kt + s) * kBK);
          if (!diag) tma_load_2d(Bs + s * kBK * TP, &tmP, &full[s], j0, (kt + s) * kBK);
        }
    }
    mbar_wait(&full[kt % KS], (kt / KS) & 1);
    const double* as = As + (kt % KS) * kBK * TP;
    const double* bs = diag ? as : Bs + (kt % KS) * kBK * TP;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kc = ks * 4 + t;
      double a[MT][2], b[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const double2 v = *reinterpret_cast<const double2*>(as + kc * TP + wm + mt * 16 + 2 * g);
        a[mt][0] = v.x;
        a[mt][1] = v.y;
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(bs + kc * TP + wn + pp * 16 + 2 * g);
        b[2 * pp] = w.x;
        b[2 * pp + 1] = w.y;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
  }
  cp_async_wait_all();  // this thread's own gathers (it reads nothing another thread copied)

  // ---- epilogue.  Thread holds rows r, r+1 x cols c..c+3 per (mt, pp) (see syrk_kernel).
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = i0 + wm + mt * 16 + 2 * g + h, c0 = j0 + wn + pp * 16 + 4 * t;
        if (r >= M || c0 > r) continue;
        double v[4];
        v[0] = acc[mt][2 * pp][2 * h];
        v[1] = acc[mt][2 * pp + 1][2 * h];
        v[2] = acc[mt][2 * pp][2 * h + 1];
        v[3] = acc[mt][2 * pp + 1][2 * h + 1];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = sub_rn(gsm[(((mt * 2 + pp) * 2 + h) * 4 + q) * NT + tid], v[q]);
        double* dst = p.G + (long long)(off + r) * p.ldg + off + c0;
        if (c0 + 3 <= r) {
          reinterpret_cast<double2*>(dst)[0] = make_double2(v[0], v[1]);
          reinterpret_cast<double2*>(dst)[1] = make_double2(v[2], v[3]);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q <= r) dst[q] = v[q];
        }
        if (p.mirror) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (c0 + q < r) p.G[(long long)(off + c0 + q) * p.ldg + off + r] = v[q];
        }
      }
  tl_mark(p.tl, p.tl_slot, 2);
}

// Fixed-order split reduction: G[i][j] = G[j][i] = (acc ? G[i][j] : 0) + sum_s ws[s][i][j] over the
// lower triangle (i >= j), plus the H^T T partials.  One CTA per 32 x 32 block of the lower
// triangle: the summed block is staged in shared memory and written both ways with coalesced rows
// (the mirrored half is a transpose, not a column scatter).  Blocks past the triangle reduce the
// H^T T partials.
__global__ void __launch_bounds__(256) syrk_finish_kernel(SyrkParams p, int splits, int accumulate) {
  __shared__ double blk[32][33];
  const int M = p.M, nb = (M + 31) / 32, nlow = nb * (nb + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  int b = blockIdx.x;
  if (b < nlow) {
    int bi = static_cast<int>((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
    while (bi * (bi + 1) / 2 > b) --bi;
    while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
    const int bj = b - bi * (bi + 1) / 2;
    const int i0 = bi * 32, j0 = bj * 32;
    for (int r = ty; r < 32; r += 8) {
      const int i = i0 + r, j = j0 + tx;
      double v = 0.0;
      if (i < M && j < M && j <= i) {
        const long long off = (long long)i * p.ldg + j;
        v = p.ws[off];
        for (int sp = 1; sp < splits; ++sp) v = add_rn(v, p.ws[sp * p.wsStride + off]);
        if (accumulate) v = add_rn(p.G[off], v);
        p.G[off] = v;
      }
      blk[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // mirror: G[j0 + r][i0 + tx] = blk[tx][r]
      const int j = j0 + r, i = i0 + tx;
      if (i < M && j < M && (bi != bj || r < tx)) p.G[(long long)j * p.ldg + i] = blk[tx][r];
    }
    return;
  }
  b -= nlow;
  const long long totalT = (long long)p.M * p.mB;
  for (long long f = (long long)b * blockDim.x + threadIdx.x; f < totalT; f += (long long)(gridDim.x - nlow) * blockDim.x) {
    const long long i = f / p.mB, j = f % p.mB;
    double v = p.wsT[i * p.ldt + j];
    for (int sp = 1; sp < splits; ++sp) v = add_rn(v, p.wsT[sp * p.wsTStride + i * p.ldt + j]);
    if (accumulate) v = add_rn(p.HtT[i * p.ldt + j], v);
    p.HtT[i * p.ldt + j] = v;
  }
}

// ============================================================================
// Generic DMMA GEMM (64x64 tiles, 4 warps of 32x32), plain staged loads.
// Used for the small solve-side products (block path, scores).
// ============================================================================
constexpr int kGT = 64, kGK = 16, kGPad = 66;

__global__ void __launch_bounds__(128) gemm_kernel(GemmParams p) {
  __shared__ __align__(16) double As[kGK][kGPad];
  __shared__ __align__(16) double Bs[kGK][kGPad];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int m0 = blockIdx.y * kGT, n0 = blockIdx.x * kGT;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;

  for (int k0 = 0; k0 < p.K; k0 += kGK) {
    // A tile: op(A)(m, k) -> As[k][m]
    for (int e = tid; e < kGK * kGT; e += 128) {
      int kk, mm;
      if (!p.transA) { kk = e % kGK; mm = e / kGK; } else { mm = e % kGT; kk = e / kGT; }
      const int gm = m0 + mm, gk = k0 + kk;
      double v = 0.0;
      if (gm < p.M && gk < p.K) v = p.transA ? p.A[(long long)gk * p.lda + gm] : p.A[(long long)gm * p.lda + gk];
      As[kk][mm] = v;
    }
    // B tile: op(B)(k, n) -> Bs[k][n]
    for (int e = tid; e < kGK * kGT; e += 128) {
      int kk, nn;
      if (!p.transB) { nn = e % kGT; kk = e / kGT; } else { kk = e % kGK; nn = e / kGK; }
      const int gn = n0 + nn, gk = k0 + kk;
      double v = 0.0;
      if (gn < p.N && gk < p.K) v = p.transB ? p.B[(long long)gn * p.ldb + gk] : p.B[(long long)gk * p.ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kGK / 4; ++ks) {
      const int kc = ks * 4 + t;
      double a[2][2], b[4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double2 v = *reinterpret_cast<const double2*>(&As[kc][wm + mt * 16 + 2 * g]);
        a[mt][0] = v.x;
        a[mt][1] = v.y;
      }
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(&Bs[kc][wn + pp * 16 + 2 * g]);
        b[2 * pp] = w.x;
        b[2 * pp + 1] = w.y;
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x4(acc[mt][nt], a[mt][0], a[mt][1], b[nt]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int r0 = m0 + wm + mt * 16 + 2 * g;
      const int c0 = n0 + wn + pp * 16 + 4 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + h;
        if (r >= p.M) continue;
        const double v[4] = {acc[mt][2 * pp][2 * h], acc[mt][2 * pp + 1][2 * h], acc[mt][2 * pp][2 * h + 1],
                             acc[mt][2 * pp + 1][2 * h + 1]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q;
          if (c >= p.N) continue;
          double* dst = p.C + (long long)r * p.ldc + c;
          const double prod = p.alpha == 1.0 ? v[q] : p.alpha * v[q];
          *dst = p.beta == 0.0 ? prod : add_rn(p.beta == 1.0 ? *dst : p.beta * *dst, prod);
        }
      }
    }
}

// ============================================================================
// launchers
// ============================================================================
// bn = 32 (sigmoid build: 128 x 32 tiles, three CTAs per SM) or 128 (plain transposed product of the
// pseudo-inverse); tmW's box is {bn + 4, kBK}
cudaError_t launch_hidden(const CUtensorMap& tmX, const CUtensorMap& tmW, const HiddenParams& p, int bn,
                          cudaStream_t s) {
  dim3 grid((p.L + bn - 1) / bn, (p.N + kTile - 1) / kTile);
  if (bn == 32) {
    constexpr size_t kSmem32 = size_t(3) * (kTile + 36) * kBK * sizeof(double) + 1024 + 256;
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(hidden_kernel<32, 3>), kSmem32);
    if (e != cudaSuccess) return e;
    hidden_kernel<32, 3><<<grid, kGemmThreads, kSmem32, s>>>(tmX, tmW, p);
  } else if (bn == 128) {
    constexpr size_t kSmem128 = size_t(kStages) * (kTile + 132) * kBK * sizeof(double) + 1024 + 256;
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(hidden_kernel<128>), kSmem128);
    if (e != cudaSuccess) return e;
    hidden_kernel<128><<<grid, kGemmThreads, kSmem128, s>>>(tmX, tmW, p);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// The Gram (tile 128, 256 threads, one CTA per SM).  With two or more tile rows the diagonal tiles
// go to syrk_diag_kernel and the rest to syrk_kernel<128, 1>; a single tile row runs
// syrk_kernel<128>.  The tensor maps' boxes must be {tile + 4, kBK} (padded shared-memory rows).
constexpr size_t kSyrkSmem128 = size_t(kStages) * 2 * 132 * kBK * sizeof(double) + 1024 + 256;

cudaError_t launch_syrk(const CUtensorMap& tmA, const CUtensorMap& tmB, const SyrkParams& p, int splits, int tile,
                        cudaStream_t s, bool pdl) {
  if (tile != 128 || p.mode == kSyrkTrailing) return cudaErrorInvalidValue;
  if (p.nbI >= 2) {
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(syrk_diag_kernel), kSyrkSmem128);
    if (e == cudaSuccess) e = ensure_attrs(reinterpret_cast<const void*>(syrk_kernel<128, 1>), kSyrkSmem128);
    if (e != cudaSuccess) return e;
    // off-diagonal (long) CTAs first, the diagonal (short) ones as its programmatic dependent:
    // they fill the SMs the last off-diagonal wave leaves idle
    syrk_kernel<128, 1><<<dim3(p.nbI * (p.nbI - 1) / 2 + p.nbI * p.nbT, splits), 256, kSyrkSmem128, s>>>(tmA, tmB, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t c2 = {};
    c2.gridDim = dim3(p.nbI, splits);
    c2.blockDim = dim3(256);
    c2.dynamicSmemBytes = kSyrkSmem128;
    c2.stream = s;
    cudaLaunchAttribute a2[1];
    a2[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a2[0].val.programmaticStreamSerializationAllowed = 1;
    c2.attrs = a2;
    c2.numAttrs = 1;
    return cudaLaunchKernelEx(&c2, syrk_diag_kernel, tmA, p);
  }
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(syrk_kernel<128>), kSyrkSmem128);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.nGram + p.nbI * p.nbT, splits);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kSyrkSmem128;
  return cudaLaunchKernelEx(&cfg, syrk_kernel<128>, tmA, tmB, p);
}

template <int TILE, int KS = kStages>
constexpr size_t trail_smem() {
  return size_t(KS) * 2 * (TILE + 4) * kBK * sizeof(double) + size_t(TILE / 32) * 16 * 2 * TILE * sizeof(double) +
         1024 + 256;
}

// Trailing update (tile 32 or 64); the tensor map covers PcT with box {tile + 4, 16}.  64-wide tiles
// stream the rank-64 panel through one 16-deep stage reloaded four times (four CTAs per SM; C4
// L=8000: 9.1 ms of trailing updates, against 11.4 / 9.5 ms with the whole panel / halves resident).
cudaError_t launch_trail(const CUtensorMap& tmP, const SyrkParams& p, int tile, cudaStream_t s) {
  if (p.kRows > kStages * kBK) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.nbI * (p.nbI + 1) / 2);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (tile == 64) {
    // 256 threads (8 warps of 16 x 32) at 3 CTAs per SM: 24 DMMA-issuing warps per SM instead of 16
    // (C4 L = 8000 trailing 18.1 -> 16.0-16.5 ms, bitwise-identical results)
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(trail_kernel<64, 1, 256>), trail_smem<64, 1>());
    if (e != cudaSuccess) return e;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = trail_smem<64, 1>();
    return cudaLaunchKernelEx(&cfg, trail_kernel<64, 1, 256>, tmP, p);
  }
  if (tile == 32) {
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(trail_kernel<32>), trail_smem<32>());
    if (e != cudaSuccess) return e;
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = trail_smem<32>();
    return cudaLaunchKernelEx(&cfg, trail_kernel<32>, tmP, p);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_syrk_finish(const SyrkParams& p, int splits, int accumulate, int num_sms, cudaStream_t s) {
  const int nb = (p.M + 31) / 32;
  const int tblocks = p.mB > 0 ? num_sms : 0;
  syrk_finish_kernel<<<nb * (nb + 1) / 2 + tblocks, 256, 0, s>>>(p, splits, accumulate);
  return cudaGetLastError();
}

// ============================================================================
// K6: scores = H beta with a fused arg-max epilogue (training accuracy, predict).
// Skinny DMMA GEMM: CTA = 128 rows of H x all m (<= BN) columns, K = L streamed by TMA
// (H tile [128][16] 128B-swizzled, beta tile [16][BN]); 8 warps x 16 rows each.
// Epilogue: optional score store, per-row arg-max (strict '>', lowest index on ties,
// elm.cpp:291-296) compared with arg-max(T), hits accumulated per CTA.
// ============================================================================
template <int BN>
__global__ void __launch_bounds__(kGemmThreads)
    scores_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmB, ScoresParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024(smem_raw);
  constexpr int kS = 4;
  double* Hs = reinterpret_cast<double*>(smem);        // [stage][128][16] swizzled
  constexpr int BNP = BN + 4;                          // padded B rows (TMA box {BN + 4, 16})
  double* Bs = Hs + kS * kTile * kBK;                  // [stage][16][BNP]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + kS * kBK * BNP);
  double* sc = reinterpret_cast<double*>(smem);  // [128][BN+1], aliases the drained pipeline
  constexpr int SCL = BN + 1;
  __shared__ unsigned long long blk_hits;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kTile;
  const int ktiles = (p.L + kBK - 1) / kBK;
  constexpr uint32_t kStageBytes = (kTile * kBK + kBK * BNP) * sizeof(double);
  if (tid == 0) {
    tma_prefetch_desc(&tmH);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    blk_hits = 0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kS && s < ktiles; ++s) {
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(Hs + s * kTile * kBK, &tmH, &full[s], s * kBK, r0);
      tma_load_2d(Bs + s * kBK * BNP, &tmB, &full[s], 0, s * kBK);
    }
  }
  constexpr int NT = BN / 8;
  double acc[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.0;
  const int wm = warp * 16;
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % kS;
    mbar_wait(&full[s], (kt / kS) & 1);
    const double* hs = Hs + s * kTile * kBK;
    const double* bs = Bs + s * kBK * BNP;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int kc = ks * 4 + t;
      // MMA rows g, g + 8 <-> tile rows 2g, 2g + 1 (conflict-free swizzled loads, as in K1)
      const double a0 = hs[swz16(wm + 2 * g, kc)];
      const double a1 = hs[swz16(wm + 2 * g + 1, kc)];
#pragma unroll
      for (int pp = 0; pp < NT / 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(bs + kc * BNP + pp * 16 + 2 * g);
        dmma_16x8x4(acc[2 * pp], a0, a1, w.x);
        dmma_16x8x4(acc[2 * pp + 1], a0, a1, w.y);
      }
    }
    __syncthreads();
    if (tid == 0 && kt + kS < ktiles) {
      const int kn = kt + kS;
      mbar_arrive_expect_tx(&full[s], kStageBytes);
      tma_load_2d(Hs + s * kTile * kBK, &tmH, &full[s], kn * kBK, r0);
      tma_load_2d(Bs + s * kBK * BNP, &tmB, &full[s], 0, kn * kBK);
    }
  }
  // scatter the accumulators to smem in natural column order
#pragma unroll
  for (int pp = 0; pp < NT / 2; ++pp) {
    const int cb = pp * 16 + 4 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wm + 2 * g + h;
      sc[r * SCL + cb + 0] = acc[2 * pp][2 * h];
      sc[r * SCL + cb + 1] = acc[2 * pp + 1][2 * h];
      sc[r * SCL + cb + 2] = acc[2 * pp][2 * h + 1];
      sc[r * SCL + cb + 3] = acc[2 * pp + 1][2 * h + 1];
    }
  }
  __syncthreads();
  if (p.S)
    for (int e = tid; e < kTile * p.m; e += kGemmThreads) {
      const int r = e / p.m, c = e % p.m;
      if (r0 + r < p.N) p.S[(long long)(r0 + r) * p.lds + c] = sc[r * SCL + c];
    }
  if (p.T && tid < kTile && r0 + tid < p.N) {
    const double* tr = p.T + (long long)(r0 + tid) * p.ldt;
    int ap = 0, ay = 0;
    for (int j = 1; j < p.m; ++j) {
      if (sc[tid * SCL + j] > sc[tid * SCL + ap]) ap = j;
      if (tr[j] > tr[ay]) ay = j;
    }
    if (ap == ay) atomicAdd(&blk_hits, 1ull);
  }
  __syncthreads();
  if (tid == 0 && p.hits && blk_hits) atomicAdd(p.hits, blk_hits);
}

cudaError_t launch_scores(const CUtensorMap& tmH, const CUtensorMap& tmB, const ScoresParams& p, cudaStream_t s) {
  const int grid = (p.N + kTile - 1) / kTile;
  auto go = [&](auto kern, int bn) -> cudaError_t {
    const size_t pipe = size_t(4) * (kTile * kBK + kBK * (bn + 4)) * sizeof(double) + 64;
    const size_t scb = size_t(kTile) * (bn + 1) * sizeof(double);
    const size_t smem = (pipe > scb ? pipe : scb) + 1024;
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kGemmThreads, smem, s>>>(tmH, tmB, p);
    return cudaGetLastError();
  };
  // BN = m rounded up to 16 (pairs of n8 fragments): C5's m = 100 computes 112 columns, not 128
  switch ((p.m + 15) / 16) {
    case 1: return go(scores_kernel<16>, 16);
    case 2: return go(scores_kernel<32>, 32);
    case 3: return go(scores_kernel<48>, 48);
    case 4: return go(scores_kernel<64>, 64);
    case 5: return go(scores_kernel<80>, 80);
    case 6: return go(scores_kernel<96>, 96);
    case 7: return go(scores_kernel<112>, 112);
    case 8: return go(scores_kernel<128>, 128);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm(const GemmParams& p, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  dim3 grid((p.N + kGT - 1) / kGT, (p.M + kGT - 1) / kGT);
  gemm_kernel<<<grid, 128, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rbpg
