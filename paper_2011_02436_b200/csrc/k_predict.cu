// K6b: fused batched prediction -- reference predict (elm.cpp:282-284) and the arg-max rule of
// accuracy (elm.cpp:286-300):
//   scores = sigmoid(X W + b) beta,   label = argmax_j scores[i][j] (strict '>', lowest index wins)
// in one kernel: H is never written to HBM.  A CTA owns 128 rows of X and walks the hidden nodes in
// chunks of 32:
//   GEMM1  Z (128 x 32) = X (128 x d) W[:, chunk]   TMA ring over d (X tile 128x16, 128B-swizzled;
//                                                    W tile 16 x 36, padded rows), DMMA m16n8k4
//   epilogue  h = sigmoid(z + b), exactly K1's arithmetic (bias after the full dot product, DFMA
//             Newton reciprocal) -> shared memory, k-major, this warp's 16 rows only
//   GEMM2  S (128 x MP) += h (128 x 32) beta[chunk, :] (beta chunk 32 x (MP+4) by TMA, double-buffered)
// Each warp owns 16 rows in both products, so between them it only needs __syncwarp.  The k-steps
// of GEMM2 run in the same order as scores_kernel's (4-wide, increasing hidden index), so scores
// equal the unfused K1 + K6 path bitwise.  Epilogue: scores staged in shared memory, one thread per
// row scans them in index order (the reference's strict '>' scan), optional score / label stores
// and hit count against one-hot targets.
#include "common.cuh"
#include "kernels.cuh"

namespace rbpg {

namespace {
__device__ __forceinline__ int swz16p(int row, int col) {
  return row * 16 + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}
__device__ __forceinline__ unsigned char* align1024p(unsigned char* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}
}  // namespace

constexpr int kPBN = 32;          // hidden nodes per chunk
constexpr int kPNS = 3;           // GEMM1 ring stages
constexpr int kPWP = kPBN + 4;    // padded W tile rows
constexpr int kPHP = kTile + 4;   // padded H^T rows (k-major)
// row swizzle of the H^T chunk: rows XOR 0 / 4 / 8 / 12 by column group of 4
__device__ __forceinline__ int hsw(int col) { return ((col >> 2) & 3) << 2; }

template <int MP>
constexpr size_t predict_smem() {
  constexpr size_t ring = size_t(kPNS) * (kTile * kBK + kBK * kPWP) * sizeof(double);
  constexpr size_t hs = size_t(kPBN) * kPHP * sizeof(double);
  constexpr size_t bs = size_t(2) * kPBN * (MP + 4) * sizeof(double);
  constexpr size_t main = ring + hs + bs + 64;
  constexpr size_t sc = size_t(kTile) * (MP + 1) * sizeof(double);
  return (main > sc ? main : sc) + 1024;
}

template <int MP>
__global__ void __launch_bounds__(kGemmThreads, MP <= 48 ? 2 : 1)
    predict_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                   const __grid_constant__ CUtensorMap tmB, PredictParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = align1024p(smem_raw);
  double* Xs = reinterpret_cast<double*>(smem);            // [stage][128][16] swizzled
  double* Ws = Xs + kPNS * kTile * kBK;                    // [stage][16][36]
  double* Hs = Ws + kPNS * kBK * kPWP;                     // [32][132]  h^T of the chunk
  constexpr int BP = MP + 4;
  double* Bs = Hs + kPBN * kPHP;                           // [2][32][MP + 4]
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + 2 * kPBN * BP);  // [kPNS]
  uint64_t* bfull = full + kPNS;                                      // [2]
  double* sc = reinterpret_cast<double*>(smem);            // [128][MP + 1] after the main loop
  constexpr int SCL = MP + 1;
  __shared__ unsigned long long blk_hits;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kTile;
  const int ktiles = (p.d + kBK - 1) / kBK;
  const int nchunks = (p.L + kPBN - 1) / kPBN;
  const int total = nchunks * ktiles;
  constexpr uint32_t kStageBytes = (kTile * kBK + kBK * kPWP) * sizeof(double);
  constexpr uint32_t kBetaBytes = kPBN * BP * sizeof(double);

  auto issue_step = [&](int step) {
    const int c = step / ktiles, kt = step - c * ktiles, s = step % kPNS;
    mbar_arrive_expect_tx(&full[s], kStageBytes);
    tma_load_2d(Xs + s * kTile * kBK, &tmX, &full[s], kt * kBK, r0);
    tma_load_2d(Ws + s * kBK * kPWP, &tmW, &full[s], c * kPBN, kt * kBK);
  };
  auto issue_beta = [&](int c) {
    mbar_arrive_expect_tx(&bfull[c & 1], kBetaBytes);
    tma_load_2d(Bs + (c & 1) * kPBN * BP, &tmB, &bfull[c & 1], 0, c * kPBN);
  };
  if (tid == 0) {
    tma_prefetch_desc(&tmX);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kPNS; ++s) mbar_init(&full[s], 1);
    mbar_init(&bfull[0], 1);
    mbar_init(&bfull[1], 1);
    fence_mbar_init();
    blk_hits = 0;
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kPNS && s < total; ++s) issue_step(s);
    issue_beta(0);
    if (nchunks > 1) issue_beta(1);
  }

  constexpr int NT2 = MP / 8;
  double acc2[NT2][4];
#pragma unroll
  for (int i = 0; i < NT2; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc2[i][q] = 0.0;
  const int wm = warp * 16;

  for (int c = 0; c < nchunks; ++c) {
    double acc1[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc1[j][q] = 0.0;
    for (int kt = 0; kt < ktiles; ++kt) {
      const int step = c * ktiles + kt, s = step % kPNS;
      mbar_wait(&full[s], (step / kPNS) & 1);
      const double* xs = Xs + s * kTile * kBK;
      const double* ws = Ws + s * kBK * kPWP;
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        const int kc = ks * 4 + t;
        const double a0 = xs[swz16p(wm + 2 * g, kc)];
        const double a1 = xs[swz16p(wm + 2 * g + 1, kc)];
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
          const double2 w = *reinterpret_cast<const double2*>(ws + kc * kPWP + pp * 16 + 2 * g);
          dmma_16x8x4(acc1[2 * pp], a0, a1, w.x);
          dmma_16x8x4(acc1[2 * pp + 1], a0, a1, w.y);
        }
      }
      __syncthreads();
      if (tid == 0 && step + kPNS < total) issue_step(step + kPNS);
    }
    // epilogue 1: h = sigmoid(z + b) into Hs[col][row] (this warp's rows, rows 2g and 2g+1 as one
    // 16-byte store); nodes >= L give 0.  Rows are XOR-swizzled per column group (hsw), which keeps
    // the row pairs together and makes both these stores and GEMM2's fragment loads conflict-free.
    // The sigmoid is the K1i epilogue's (common.cuh): z in place over the accumulators, one integer
    // maximum over the high words of the thread's 16 values, then the select-free in-range form --
    // or, when some |z| > 700 (or is not finite), the out-of-line exact form for all 16.
    int zhi = 0;
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = c * kPBN + pp * 16 + 4 * t + q;
        const double bq = col < p.L ? p.bias[col] : 0.0;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          double& a = acc1[2 * pp + (q & 1)][2 * half + (q >> 1)];
          a = col < p.L ? add_rn(a, bq) : 0.0;
          zhi = max(zhi, __double2hiint(a) & 0x7fffffff);
        }
      }
    if (zhi <= kSigmoidRangeHi) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc1[j][e] = sigmoid_in_range(acc1[j][e]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc1[j][e] = sigmoid_exact(acc1[j][e]);
    }
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const int cb = pp * 16 + 4 * t;  // chunk column of acc1[2pp][*] / acc1[2pp+1][*]
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        // acc1[2pp + (q & 1)][2 * half + (q >> 1)] holds (row 2g + half, column cb + q)
        const bool live = c * kPBN + cb + q < p.L;
        const double h0 = live ? acc1[2 * pp + (q & 1)][q >> 1] : 0.0;
        const double h1 = live ? acc1[2 * pp + (q & 1)][2 + (q >> 1)] : 0.0;
        const int kc = cb + q;
        *reinterpret_cast<double2*>(Hs + kc * kPHP + ((wm + 2 * g) ^ hsw(kc))) = make_double2(h0, h1);
      }
    }
    __syncwarp();
    mbar_wait(&bfull[c & 1], (c >> 1) & 1);
    const double* bs = Bs + (c & 1) * kPBN * BP;
#pragma unroll
    for (int kk = 0; kk < kPBN; kk += 4) {
      const int kc = kk + t;
      const double2 a = *reinterpret_cast<const double2*>(Hs + kc * kPHP + ((wm + 2 * g) ^ hsw(kc)));
#pragma unroll
      for (int pp = 0; pp < NT2 / 2; ++pp) {
        const double2 w = *reinterpret_cast<const double2*>(bs + kc * BP + pp * 16 + 2 * g);
        dmma_16x8x4(acc2[2 * pp], a.x, a.y, w.x);
        dmma_16x8x4(acc2[2 * pp + 1], a.x, a.y, w.y);
      }
    }
    __syncthreads();  // every warp is done with Bs[c & 1] (and its Hs rows)
    if (tid == 0 && c + 2 < nchunks) issue_beta(c + 2);
  }

  // scores -> shared memory in natural column order (aliases the drained pipeline)
#pragma unroll
  for (int pp = 0; pp < NT2 / 2; ++pp) {
    const int cb = pp * 16 + 4 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = wm + 2 * g + h;
      sc[r * SCL + cb + 0] = acc2[2 * pp][2 * h];
      sc[r * SCL + cb + 1] = acc2[2 * pp + 1][2 * h];
      sc[r * SCL + cb + 2] = acc2[2 * pp][2 * h + 1];
      sc[r * SCL + cb + 3] = acc2[2 * pp + 1][2 * h + 1];
    }
  }
  __syncthreads();
  if (p.S)
    for (int e = tid; e < kTile * p.m; e += kGemmThreads) {
      const int r = e / p.m, cc = e - r * p.m;
      if (r0 + r < p.N) p.S[(long long)(r0 + r) * p.lds + cc] = sc[r * SCL + cc];
    }
  if (tid < kTile && r0 + tid < p.N) {
    int ap = 0;
    for (int j = 1; j < p.m; ++j)
      if (sc[tid * SCL + j] > sc[tid * SCL + ap]) ap = j;
    if (p.labels) p.labels[r0 + tid] = ap;
    if (p.T) {
      const double* tr = p.T + (long long)(r0 + tid) * p.ldt;
      int ay = 0;
      for (int j = 1; j < p.m; ++j)
        if (tr[j] > tr[ay]) ay = j;
      if (ap == ay) atomicAdd(&blk_hits, 1ull);
    }
  }
  if (p.hits) {
    __syncthreads();
    if (tid == 0 && blk_hits) atomicAdd(p.hits, blk_hits);
  }
}

// tmX: X (N x d) box {16, 128} 128B-swizzled; tmW: W (d x L) box {36, 16}; tmB: beta (L x m) box
// {MP + 4, 32} (out-of-bounds columns / rows read as zero)
int predict_mp(int m) { return m >= 1 && m <= 128 ? (m + 15) / 16 * 16 : 0; }  // pairs of n8 fragments

cudaError_t launch_predict(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmB,
                           const PredictParams& p, cudaStream_t s) {
  if (p.N <= 0) return cudaSuccess;
  const int grid = (p.N + kTile - 1) / kTile;
  auto go = [&](auto kern, size_t smem) -> cudaError_t {
    cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kGemmThreads, smem, s>>>(tmX, tmW, tmB, p);
    return cudaGetLastError();
  };
  switch (predict_mp(p.m)) {
    case 16: return go(predict_kernel<16>, predict_smem<16>());
    case 32: return go(predict_kernel<32>, predict_smem<32>());
    case 48: return go(predict_kernel<48>, predict_smem<48>());
    case 64: return go(predict_kernel<64>, predict_smem<64>());
    case 80: return go(predict_kernel<80>, predict_smem<80>());
    case 96: return go(predict_kernel<96>, predict_smem<96>());
    case 112: return go(predict_kernel<112>, predict_smem<112>());
    case 128: return go(predict_kernel<128>, predict_smem<128>());
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rbpg
