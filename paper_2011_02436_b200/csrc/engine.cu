// Host engine of the B200 RBP-ELM hot path: workspace, TMA descriptors, the
// solve dispatch of the reference's solve_beta (elm.cpp:158-229) and train()
// (elm.cpp:231-280), and the C ABI declared in include/rbpelm_b200.h.
//
// Pipeline of train() with the rank strategy, all on one stream:
//   K1 hidden_kernel   H = sigmoid(X W + b)               (elm.cpp:93-106)
//   K2 syrk_kernel     G = H^T H, HtT = H^T T              (linalg.cpp:179-184, elm.cpp:207)
//   K3 panel_kernel +  diagonal-pivoted blocked Cholesky  (linalg.cpp:186-247)
//      syrk_kernel(trailing)
//   K4 trsm_pair       beta = P F^-T F^-1 P^T HtT          (elm.cpp:202-214, linalg.cpp:254-270)
//   accuracy           argmax(H beta) vs argmax(T)         (elm.cpp:278, 286-300)
// If rank < L the Schur block solve (elm.cpp:124-156) runs on sub-blocks of the
// original Gram and HtT (no N-sized passes): H1^T(T - H2 B) = HtT[P1] - G[P1,P2] B.
#include "../../include/rbpelm_b200.h"
#include "common.cuh"
#include "kernels.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace rbpg {
cudaError_t ensure_attrs(const void* fn, size_t smem, bool nonportable_cluster) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, std::pair<size_t, bool>> done;  // (device, kernel) -> set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto& cur = done[{dev, fn}];
  if (smem > cur.first || (smem > 0 && cur.first == 0)) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cur.first = smem;
  }
  if (nonportable_cluster && !cur.second) {
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cur.second = true;
  }
  return cudaSuccess;
}
cudaError_t launch_hidden(const CUtensorMap&, const CUtensorMap&, const HiddenParams&, int, cudaStream_t);
cudaError_t launch_syrk(const CUtensorMap&, const CUtensorMap&, const SyrkParams&, int, int, cudaStream_t, bool = false);
cudaError_t launch_syrk_finish(const SyrkParams&, int, int, int, cudaStream_t);
cudaError_t launch_gemm(const GemmParams&, cudaStream_t);
cudaError_t launch_scores(const CUtensorMap&, const CUtensorMap&, const ScoresParams&, cudaStream_t);
cudaError_t launch_factor_setup(const double*, long long, int, int, long long, double, int, double*, int*,
                                FactorState*, cudaStream_t);
cudaError_t launch_panel(const PanelParams&, int, int*, cudaStream_t);
bool panel_is_reg(int nl);
int panel_width(int n, int k);
cudaError_t launch_trail(const CUtensorMap&, const SyrkParams&, int, cudaStream_t);
cudaError_t launch_gather_factor(const double*, long long, const int*, int, double*, long long, const FactorState*,
                                 int, cudaStream_t);
cudaError_t launch_gather_rows(const double*, long long, const int*, int, int, double*, long long, cudaStream_t);
cudaError_t launch_scatter_rows(const double*, long long, const int*, int, int, double*, long long, cudaStream_t);
cudaError_t launch_tri_inv(const double*, long long, int, double*, cudaStream_t);
cudaError_t launch_trsm_step(const double*, long long, const double*, double*, long long, double*, long long, int, int,
                             int, int, int, cudaStream_t);
bool trsm_cluster_fits(int n, int m);
cudaError_t launch_trsm_pair(const double*, long long, double*, long long, int, int, int, int, int, double*,
                             cudaStream_t);
cudaError_t launch_accuracy(const double*, long long, const double*, long long, long long, int, unsigned long long*,
                            int, cudaStream_t);
cudaError_t launch_add_diag(double*, long long, int, double, cudaStream_t);
cudaError_t launch_gather_block(const double*, long long, const int*, int, const int*, int, double*, long long,
                                cudaStream_t);
cudaError_t launch_symmetrize(double*, long long, int, cudaStream_t);
cudaError_t launch_trace(const double*, long long, int, double*, cudaStream_t);
cudaError_t launch_nonfinite(const double*, long long, int, int, int*, cudaStream_t);
cudaError_t launch_add_block(double*, long long, const double*, long long, long long, long long, cudaStream_t);
cudaError_t launch_svd_round(double*, long long, long long, double*, long long, long long, int, int, int, long long,
                             int, long long, double, double, double*, double*, int*, int*, cudaStream_t);
cudaError_t launch_col_sumsq(const double*, long long, long long, int, double*, cudaStream_t);
cudaError_t launch_scale_rows(double*, long long, int, int, const double*, cudaStream_t);
cudaError_t launch_scale_cols(double*, long long, long long, int, const double*, cudaStream_t);
cudaError_t launch_transpose(const double*, long long, long long, long long, double*, long long, long long,
                             cudaStream_t);
cudaError_t launch_axpy_rows(const double*, long long, const double*, long long, int, int, double*, long long,
                             cudaStream_t);
cudaError_t launch_predict(const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const PredictParams&, cudaStream_t);
int predict_mp(int m);
cudaError_t launch_pack_lower(const double*, long long, int, double*, cudaStream_t);
cudaError_t launch_unpack_lower(const double*, int, double*, long long, cudaStream_t);
cudaError_t launch_oz_colmax(const double*, long long, long long, int, unsigned long long*, int, cudaStream_t);
cudaError_t launch_oz_colmax_acc(const double*, long long, long long, int, unsigned long long*, int, cudaStream_t);
cudaError_t launch_oz_slice(const double*, long long, long long, int, const unsigned long long*, int*, int, long long,
                            int8_t*, cudaStream_t);
cudaError_t launch_oz_gram2(const CUtensorMap* maps, const OzParams&, cudaStream_t);
cudaError_t launch_oz_hidden(const CUtensorMap* maps, const OzHidParams&, cudaStream_t);
cudaError_t launch_oz_beta_planes(const double*, long long, int, int, const int*, int, int8_t*, double*, cudaStream_t);
cudaError_t launch_oz_labels(const double*, long long, long long, int, int*, cudaStream_t);
cudaError_t launch_oz_scores(const CUtensorMap* maps, const OzScoresParams&, cudaStream_t);
int oz_pair_order(int nbI, int B, int2* out);
int oz_pair_items(int nbI);
cudaError_t launch_oz_finish(const double*, long long, int, int, double*, long long, int, cudaStream_t);
cudaError_t launch_sum_parts(const double*, long long, int, long long, double*, cudaStream_t);
}  // namespace rbpg

using namespace rbpg;

// ============================================================================
// errors
// ============================================================================
namespace {
struct Fail {
  int code;
  std::string msg;
  size_t pivot_index = 0;
  double pivot_value = 0.0;
  int block = 0;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(RBPG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
std::string shp(size_t r, size_t c) { return std::to_string(r) + "x" + std::to_string(c); }
inline size_t even(size_t v) { return (v + 1) & ~size_t(1); }
inline size_t round_up(size_t v, size_t m) { return (v + m - 1) / m * m; }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
}  // namespace

struct rbpg_context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t copy = nullptr;  // host -> device input uploads, overlapped with the hidden build
  cudaStream_t aux = nullptr;   // hidden builds of late upload blocks, concurrent with the first Gram part
  cudaEvent_t chunk_ev[16] = {};
  cudaEvent_t aux_ev[8] = {};
  cudaStream_t stream = nullptr;
  std::map<std::string, std::pair<void*, size_t>> bufs;
  uint64_t launches = 0;
  EncodeTiledFn encode = nullptr;
  cudaEvent_t ev[8] = {};
  // H kept resident by the gram stage for the accuracy stage, valid only for the exact inputs that
  // built it (X, W, b pointers and leading dimensions, row and node counts)
  const double* kept_h = nullptr;
  size_t kept_n = 0, kept_l = 0, kept_ldh = 0;
  struct KeptKey {
    const double *x = nullptr, *w = nullptr, *b = nullptr;
    size_t ldx = 0, ldw = 0, d = 0;
    bool operator==(const KeptKey& o) const {
      return x == o.x && w == o.w && b == o.b && ldx == o.ldx && ldw == o.ldw && d == o.d;
    }
  } kept_key;
  // digit planes of [H T] written by the INT8 Gram, one record per Gram part (row range, planes, column
  // exponents); the records of the parts that built the kept H serve the INT8 accuracy pass
  struct OzPart {
    size_t r0 = 0, rows = 0, Mpad = 0, Npad = 0;
    int8_t* planes = nullptr;
    int* exps = nullptr;
  };
  std::vector<OzPart> oz_pending, oz_kept;
  const double* oz_kept_h = nullptr;
  void keep_h(const double* h, size_t n, size_t l, size_t ldh, const KeptKey& key) {
    oz_kept = oz_pending;
    oz_kept_h = h;
    kept_h = h;
    kept_n = n;
    kept_l = l;
    kept_ldh = ldh;
    kept_key = key;
  }
  bool kept_for(const KeptKey& key, size_t n, size_t l) const {
    return kept_h && kept_n == n && kept_l == l && kept_key == key;
  }
  size_t h_budget_bytes = size_t(48) << 30;
  // train-path Gram on the INT8 tensor cores (k_ozaki.cu); RBPG_GRAM_DMMA=1: the FP64 DMMA Gram
  bool gram_int8 = std::getenv("RBPG_GRAM_DMMA") == nullptr;
  int oz_tiles_nbI = -1;  // tile grid whose launch order is in the "oz_tiles" buffer
  int oz_tiles_n = 0;
  // hidden matrix + targets of the current solve when resident (train / solve_beta): the SVD
  // pseudo-inverse branch of solve_direct needs H itself, not only its Gram
  const double* src_h = nullptr;
  const double* src_y = nullptr;
  size_t src_n = 0, src_ldh = 0, src_ldy = 0;
  int svd_sweeps = 0;  // sweeps of the last SVD (diagnostics)
  std::mutex mu;

  void* buf(const std::string& name, size_t bytes) {
    auto it = bufs.find(name);
    if (it != bufs.end() && it->second.second >= bytes) return it->second.first;
    if (it != bufs.end()) {
      cudaStreamSynchronize(stream);
      cudaFree(it->second.first);
      bufs.erase(it);
      if (kept_h && name == "H") kept_h = nullptr;
    }
    void* p = nullptr;
    ck(cudaMalloc(&p, bytes < 256 ? 256 : bytes), ("cudaMalloc " + name).c_str());
    bufs[name] = {p, bytes};
    return p;
  }
  double* dbuf(const std::string& name, size_t elems) { return static_cast<double*>(buf(name, elems * 8)); }
  std::map<std::string, std::pair<void*, size_t>> hbufs;  // pinned host staging
  void* pinned(const std::string& name, size_t bytes) {
    auto it = hbufs.find(name);
    if (it != hbufs.end() && it->second.second >= bytes) return it->second.first;
    if (it != hbufs.end()) {
      cudaStreamSynchronize(stream);
      cudaFreeHost(it->second.first);
      hbufs.erase(it);
    }
    void* p = nullptr;
    ck(cudaMallocHost(&p, bytes < 64 ? 64 : bytes), ("cudaMallocHost " + name).c_str());
    hbufs[name] = {p, bytes};
    return p;
  }
  // per-kernel-class device timing (bench.py roofline evidence), off by default
  bool profile = false;
  struct Prof {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
    double ms = 0.0;
    uint64_t count = 0;
  };
  std::map<std::string, Prof> prof;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  }
  template <typename F>
  void run(const char* name, F&& launch) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (profile) {
      a = take_event();
      b = take_event();
      cudaEventRecord(a, stream);
    }
    ck(launch(), name);
    ++launches;
    if (profile) {
      cudaEventRecord(b, stream);
      prof[name].pending.emplace_back(a, b);
      if (timeline_on) timeline.push_back({name, a, b});
    }
  }
  // RBPG_TIMELINE=1 (with profiling on): per-launch start / duration / gap dump on stderr
  struct Mark {
    const char* name;
    cudaEvent_t a, b;
  };
  const bool timeline_on = std::getenv("RBPG_TIMELINE") != nullptr;
  std::vector<Mark> timeline;
  void dump_timeline() {
    if (timeline.empty()) return;
    float prev_end = 0.f;
    for (size_t i = 0; i < timeline.size(); ++i) {
      float st = 0.f, du = 0.f;
      cudaEventElapsedTime(&st, timeline[0].a, timeline[i].a);
      cudaEventElapsedTime(&du, timeline[i].a, timeline[i].b);
      std::fprintf(stderr, "TL %-22s start %9.1f us  dur %8.1f us  gap %6.1f us\n", timeline[i].name, st * 1e3,
                   du * 1e3, (st - prev_end) * 1e3);
      prev_end = st + du;
    }
    timeline.clear();
  }
  void collect() {
    cudaStreamSynchronize(stream);
    if (timeline_on) dump_timeline();
    for (auto& kv : prof) {
      for (auto& pr : kv.second.pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.first, pr.second);
        kv.second.ms += ms;
        kv.second.count += 1;
        ev_pool.push_back(pr.first);
        ev_pool.push_back(pr.second);
      }
      kv.second.pending.clear();
    }
  }
};

namespace {

CUtensorMap make_map(rbpg_context* ctx, const double* base, uint64_t cols, uint64_t rows, uint64_t ld,
                     uint32_t box_cols, uint32_t box_rows, bool swizzle128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * sizeof(double)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ctx->encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(RBPG_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ") dims " +
                              std::to_string(cols) + "x" + std::to_string(rows) + " ld " + std::to_string(ld));
  return m;
}

// ---------------------------------------------------------------------------
// device building blocks
// ---------------------------------------------------------------------------
// 3-D map over digit planes [7][rows][cols] (int8): boxes of {bc, 32, planes}, 128- or 64-byte swizzle
CUtensorMap plane_map(rbpg_context* ctx, int8_t* planes, size_t cols, size_t rows, uint32_t bc, uint32_t nplanes) {
  CUtensorMap m;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), 7};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(cols) * rows};
  cuuint32_t box[3] = {bc, 32u, nplanes};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = ctx->encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, planes, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, bc == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(RBPG_CUDA_ERROR, "cuTensorMapEncodeTiled (digit planes) failed (" + std::to_string(int(r)) + ")");
  return m;
}

// K1i (k_ozaki.cu): H = sigmoid(X W + b) on the INT8 tensor cores.  W (d x L) and X^T (d x N) are cut
// into digit planes with one exponent per W column / X row (the Gram's column scan + slice, on the
// transposed X), then one persistent CTA-pair kernel computes 256-node x 128-row blocks of H^T with the
// fused epilogue.  Scratch buffers are per stream: the e2e path builds row blocks on two streams.
constexpr size_t kOzHidMaxD = 16384;  // int32 headroom of one k range: 7 d 2^14 < 2^31
void hidden_oz_dev(rbpg_context* ctx, const double* dX, size_t ldx, size_t N, size_t d, const double* dW, size_t ldw,
                   const double* db, size_t L, double* dH, size_t ldh, unsigned long long* cmax = nullptr) {
  const size_t Nr = (N + 127) / 128 * 128, Kpad = (d + 31) / 32 * 32, Lp = (L + 255) / 256 * 256;
  const std::string sfx = "." + std::to_string(reinterpret_cast<uintptr_t>(ctx->stream));
  double* xt = ctx->dbuf("ozh.xt" + sfx, d * Nr);
  for (size_t r0 = 0; r0 < N; r0 += (size_t(1) << 20)) {  // X^T in row chunks (grid.y limit of the transpose)
    const size_t nr = std::min(N - r0, size_t(1) << 20);
    ctx->run("oz_hidden_prep", [&] {
      return launch_transpose(dX + r0 * ldx, static_cast<long long>(ldx), static_cast<long long>(nr),
                              static_cast<long long>(d), xt + r0, static_cast<long long>(Nr), static_cast<long long>(nr),
                              ctx->stream);
    });
  }
  auto* cmx = reinterpret_cast<unsigned long long*>(ctx->dbuf("ozh.cmx" + sfx, N));
  auto* cmw = reinterpret_cast<unsigned long long*>(ctx->dbuf("ozh.cmw" + sfx, L));
  int* ex = reinterpret_cast<int*>(ctx->buf("ozh.ex" + sfx, Nr * sizeof(int)));
  int* ew = reinterpret_cast<int*>(ctx->buf("ozh.ew" + sfx, Lp * sizeof(int)));
  auto* px = reinterpret_cast<int8_t*>(ctx->buf("ozh.px" + sfx, 7 * Kpad * Nr));
  auto* pw = reinterpret_cast<int8_t*>(ctx->buf("ozh.pw" + sfx, 7 * Kpad * Lp));
  ctx->run("oz_hidden_prep", [&] {
    return launch_oz_colmax(xt, static_cast<long long>(Nr), static_cast<long long>(d), static_cast<int>(N), cmx,
                            ctx->num_sms, ctx->stream);
  });
  ctx->run("oz_hidden_prep", [&] {
    return launch_oz_slice(xt, static_cast<long long>(Nr), static_cast<long long>(d), static_cast<int>(N), cmx, ex,
                           static_cast<int>(Nr), static_cast<long long>(Kpad), px, ctx->stream);
  });
  ctx->run("oz_hidden_prep", [&] {
    return launch_oz_colmax(dW, static_cast<long long>(ldw), static_cast<long long>(d), static_cast<int>(L), cmw,
                            ctx->num_sms, ctx->stream);
  });
  ctx->run("oz_hidden_prep", [&] {
    return launch_oz_slice(dW, static_cast<long long>(ldw), static_cast<long long>(d), static_cast<int>(L), cmw, ew,
                           static_cast<int>(Lp), static_cast<long long>(Kpad), pw, ctx->stream);
  });
  CUtensorMap maps[4] = {plane_map(ctx, pw, Lp, Kpad, 128, 4), plane_map(ctx, px, Nr, Kpad, 64, 4),
                         plane_map(ctx, pw, Lp, Kpad, 128, 7), plane_map(ctx, px, Nr, Kpad, 64, 7)};
  OzHidParams p{};
  p.N = static_cast<int>(N);
  p.L = static_cast<int>(L);
  p.nP = static_cast<int>(Lp / 256);
  p.nJ = static_cast<int>(Nr / 128);
  p.ksteps = static_cast<int>(Kpad / 32);
  p.rexp = ex;
  p.cexp = ew;
  p.bias = db;
  p.H = dH;
  p.ldh = static_cast<long long>(ldh);
  p.cmax = cmax;
  ctx->run("hidden_kernel", [&] { return launch_oz_hidden(maps, p, ctx->stream); });
}

// cmax (optional, m > 0 with T): the column maxima of the built rows of [H T] accumulated for the INT8
// Gram's scan (zeroed by the caller before the first block of a Gram part).
void hidden_dev(rbpg_context* ctx, const double* dX, size_t ldx, size_t N, size_t d, const double* dW, size_t ldw,
                const double* db, size_t L, double* dH, size_t ldh, const double* dT = nullptr, size_t ldt = 0,
                size_t m = 0, unsigned long long* cmax = nullptr) {
  if (N == 0) return;
  if (ctx->gram_int8 && d <= kOzHidMaxD && N < (size_t(1) << 31)) {
    hidden_oz_dev(ctx, dX, ldx, N, d, dW, ldw, db, L, dH, ldh, cmax);
    if (m > 0 && dT)  // augmented rows [H T]
      ck(cudaMemcpy2DAsync(dH + L, ldh * 8, dT, ldt * 8, m * 8, N, cudaMemcpyDeviceToDevice, ctx->stream), "append T");
    if (cmax && m > 0)
      ctx->run("oz_colmax", [&] {
        return launch_oz_colmax_acc(dH + L, static_cast<long long>(ldh), static_cast<long long>(N), static_cast<int>(m),
                                    cmax + L, ctx->num_sms, ctx->stream);
      });
    return;
  }
  CUtensorMap tmX = make_map(ctx, dX, d, N, ldx, 16, kTile, true);
  constexpr int bn = 32;  // 128 x 32 tiles, three CTAs per SM (k_gemm.cu)
  CUtensorMap tmW = make_map(ctx, dW, L, d, ldw, bn + 4, kBK, false);  // padded smem rows
  HiddenParams p{static_cast<int>(N), static_cast<int>(d), static_cast<int>(L), db, dH, static_cast<long long>(ldh),
                 0, m > 0 ? dT : nullptr, static_cast<long long>(ldt), static_cast<int>(m)};
  ctx->run("hidden_kernel", [&] { return launch_hidden(tmX, tmW, p, bn, ctx->stream); });
  if (cmax)  // the DMMA build has no fused scan: scan its rows of [H T]
    ctx->run("oz_colmax", [&] {
      return launch_oz_colmax_acc(dH, static_cast<long long>(ldh), static_cast<long long>(N),
                                  static_cast<int>(L + (dT ? m : 0)), cmax, ctx->num_sms, ctx->stream);
    });
}

// G (+)= A^T A over rows [0, N) of A (N x L, ld lda); HtT (+)= A^T T when m > 0.
// split-K count S for a Gram of N rows (uniform row splits for every tile, so every Gram element
// sees the same arithmetic): greedy list scheduling of the tile x split CTAs on the SMs --
// off-diagonal and H^T T tiles first, then the diagonal ones at ~0.56 of their work (72 of 128
// fragments) -- plus the fixed-order reduction of the S partials
// Large Grams (thousands of tiles, e.g. C5's 2145) are split too: with one split the tiles fill
// 14.05 waves and the last wave leaves most SMs idle (~5 %); two or three splits level it for one
// fixed-order reduction pass (~0.2 ms at L + m = 8292).
int gram_splits(rbpg_context* ctx, size_t N, size_t L, size_t m, int tiles, int nbI) {
  int splits = 1;
  {
    const int P = ctx->num_sms;
    const int nfull = tiles - (nbI >= 2 ? nbI : 0), ndiag = nbI >= 2 ? nbI : 0;
    const double us_per_row = 2.0 * kTile * kTile / (35.7e12 / P) * 1e6;
    // fixed-order reduction: ~1 us per partial at L + m = 1010 (measured), quadratic in L + m
    const double finish_us_per_split = double(L + m) * double(L + m) / (1010.0 * 1010.0);
    const double ws_bytes_per_split = double(L + m) * double(L + m) * 8.0;
    std::vector<std::pair<double, int>> cand;  // (modelled time, S)
    const int max_sp = tiles < 4 * P ? 40 : 4;
    for (int sp = 1; sp <= max_sp; ++sp) {
      if (sp > 1 && N / static_cast<size_t>(sp) < 768) break;
      if (sp > 1 && sp * ws_bytes_per_split > 2.0e9) break;  // split workspace <= 2 GB
      const double dur = double(N) / sp * us_per_row + 2.0;  // + per-CTA prologue / partial store
      // equal full-tile CTAs: every SM gets q or q + 1 of them; then the diagonal CTAs go, one
      // at a time, to the least-loaded SM (loads kept as a histogram of levels)
      const long long nf = 1LL * nfull * sp;
      std::map<double, long long> level;
      level[double(nf / P) * dur] += P - nf % P;
      if (nf % P) level[double(nf / P + 1) * dur] += nf % P;
      const double ddur = 0.5625 * (dur - 2.0) + 2.0;
      for (long long c = 0; c < 1LL * ndiag * sp; ++c) {
        auto it = level.begin();
        const double l = it->first;
        if (--it->second == 0) level.erase(it);
        level[l + ddur] += 1;
      }
      cand.emplace_back(level.rbegin()->first + (sp > 1 ? sp * finish_us_per_split + 3.0 : 0.0), sp);
    }
    // the greedy model misses the launch order of the two grids: among the near-best candidates
    // prefer the split count that fills the last off-diagonal wave (measured best at C2: S = 37,
    // 28 x 37 = 7 x 148)
    double tmin = 1e300;
    for (const auto& c : cand) tmin = std::min(tmin, c.first);
    long long best_rem = P + 1;
    for (const auto& c : cand) {
      if (c.first > 1.01 * tmin) continue;
      const long long rem = (1LL * nfull * c.second) % P;
      const long long waste = rem == 0 ? 0 : P - rem;
      if (waste < best_rem) {
        best_rem = waste;
        splits = c.second;
      }
    }
  }
  return splits;
}

void gram_dev(rbpg_context* ctx, const double* dA, size_t lda, size_t N, size_t L, const double* dT, size_t ldt_in,
              size_t m, double* dG, size_t ldg, double* dHtT, size_t ldt, bool accumulate) {
  SyrkParams p{};
  p.M = static_cast<int>(L);
  p.mB = static_cast<int>(m);
  p.nbI = static_cast<int>((L + kTile - 1) / kTile);
  p.nGram = p.nbI * (p.nbI + 1) / 2;
  p.nbT = m > 0 ? static_cast<int>((m + kTile - 1) / kTile) : 0;
  const int tiles = p.nGram + p.nbI * p.nbT;
  int splits = gram_splits(ctx, N, L, m, tiles, p.nbI);
  long long per = static_cast<long long>(round_up((N + splits - 1) / splits, kBK));
  if (per == 0) per = kBK;
  splits = static_cast<int>((N + per - 1) / per);
  if (splits < 1) splits = 1;
  p.kRows = static_cast<long long>(N);
  p.kPerSplit = per;
  p.G = dG;
  p.ldg = static_cast<long long>(ldg);
  p.HtT = dHtT;
  p.ldt = static_cast<long long>(ldt);
  const bool direct = splits == 1 && !accumulate;
  p.mode = direct ? kSyrkDirect : kSyrkPartial;
  if (!direct) {
    p.ws = ctx->dbuf("syrk_ws", size_t(splits) * L * ldg);
    p.wsStride = static_cast<long long>(L * ldg);
    if (m > 0) {
      p.wsT = ctx->dbuf("syrk_wsT", size_t(splits) * L * ldt);
      p.wsTStride = static_cast<long long>(L * ldt);
    }
  }
  if (N == 0) {
    if (!accumulate) {
      ck(cudaMemsetAsync(dG, 0, sizeof(double) * L * ldg, ctx->stream), "memset G");
      if (m > 0) ck(cudaMemsetAsync(dHtT, 0, sizeof(double) * L * ldt, ctx->stream), "memset HtT");
    }
    return;
  }
  CUtensorMap tmA = make_map(ctx, dA, L, N, lda, kTile + 4, kBK, false);  // padded smem rows
  CUtensorMap tmB = m > 0 ? make_map(ctx, dT, m, N, ldt_in, kTile + 4, kBK, false) : tmA;
  ctx->run("syrk_kernel", [&] { return launch_syrk(tmA, tmB, p, splits, kTile, ctx->stream); });
  if (p.nbI >= 2) ++ctx->launches;  // diagonal + off-diagonal grids
  if (!direct) ctx->run("syrk_finish", [&] { return launch_syrk_finish(p, splits, accumulate ? 1 : 0, ctx->num_sms, ctx->stream); });
}

// ---- Gram on the INT8 tensor cores (k_ozaki.cu): exact digit planes, FP64-accurate result.
// Row splits of at most 512 k-steps (16384 rows: the int32 headroom of one accumulation), so every
// CTA-pair item is read out once into its own packed partial tile set (2 slots per split: the two
// accumulator groups); the fixed-order reduction (oz_finish_kernel) sums the slots.
// k-steps (32 rows) per split: at most 512 (the int32 headroom).  A small Gram gets shorter splits when
// that shortens the persistent kernel: a list-scheduling model of the items (round robin over the CTA
// pairs, group-1 items of 18 MMAs per k-step first, then group 0 with 10; ~34 ns per MMA and ~6 us of
// read-out per item) plus the fixed-order reduction reading every partial slot (~5 TB/s).  (C4 L = 500:
// 84 items on 74 pairs at 512 k-steps, 0.62 -> 0.38 ms; C4 L = 8000 / C5: unchanged.)
long long oz_ksteps_per_split_model(size_t rows, size_t M, int num_sms);
long long oz_ksteps_per_split(size_t rows, size_t M, int num_sms) {  // memoised: called several times per train
  static std::mutex mu;
  static std::map<std::tuple<size_t, size_t, int>, long long> memo;
  const auto key = std::make_tuple((rows + 63) / 64, M, num_sms);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  const long long per = oz_ksteps_per_split_model(rows, M, num_sms);
  std::lock_guard<std::mutex> lk(mu);
  if (memo.size() > 4096) memo.clear();
  memo[key] = per;
  return per;
}
long long oz_ksteps_per_split_model(size_t rows, size_t M, int num_sms) {
  const long long ksteps = static_cast<long long>((rows + 63) / 64 * 64 / 32);
  const int nbI = static_cast<int>((M + 127) / 128);
  const long long tiles = oz_pair_items(nbI);  // CTA-pair items per split and group
  const int pairs = std::max(1, num_sms / 2);
  const long long base = std::max<long long>(1, (ksteps + 511) / 512);
  long long best_per = (ksteps + base - 1) / base;  // uniform splits
  if (2 * tiles * base >= 6LL * pairs) return std::min<long long>(best_per, 512);  // already >= 6 waves of items
  const double slot_bytes = double(nbI) * (nbI + 1) / 2 * 16384 * 8;
  double best = 1e30;
  for (long long sp = base; sp <= base * 16; ++sp) {
    const long long per = (ksteps + sp - 1) / sp;
    if (per < 32 && sp > base) break;
    const long long splits = (ksteps + per - 1) / per;
    const long long items = 2 * tiles * splits;
    if (items > 4 * 1024 * 1024) break;
    std::vector<double> load(static_cast<size_t>(std::min<long long>(pairs, items)), 0.0);
    for (long long it = 0; it < items; ++it) {  // the kernel's item order: group 1 first, split-major
      const bool g1 = it < tiles * splits;
      const long long r = g1 ? it : it - tiles * splits;
      const long long split = r / tiles;
      const long long nk = std::min(per, ksteps - split * per);
      load[static_cast<size_t>(it % static_cast<long long>(load.size()))] += (g1 ? 18 : 10) * nk * 34e-9 + 6e-6;
    }
    const double t = *std::max_element(load.begin(), load.end()) + 2.0 * splits * slot_bytes / 5e12;
    if (t < best * 0.98) {
      best = t;
      best_per = per;
    }
  }
  return std::min<long long>(best_per, 512);
}
int oz_splits(size_t rows, size_t M, int num_sms) {
  const long long per = oz_ksteps_per_split(rows, M, num_sms);
  const long long ksteps = static_cast<long long>((rows + 63) / 64 * 64 / 32);
  return static_cast<int>(std::max<long long>(1, (ksteps + per - 1) / per));
}
size_t oz_slot_doubles(size_t M) {
  const size_t nbI = (M + 127) / 128;
  return nbI * (nbI + 1) / 2 * 16384;  // lower 128 x 128 tiles, packed
}
// Partials of rows [0, rows) of A (rows x M, ld lda) into the 2 * oz_splits(rows) slots at ws.
// Part `part` (rows [r0, r0 + rows) of the Gram operand) keeps its own planes and exponents, recorded in
// ctx->oz_pending for the INT8 accuracy pass.
// cmax_ready: the column maxima of these rows already accumulated by their hidden builds (fused scan).
void oz_gram_part(rbpg_context* ctx, const double* dA, size_t lda, size_t rows, size_t M, double* ws, int part = 0,
                  size_t r0 = 0, const unsigned long long* cmax_ready = nullptr) {
  const int nbI = static_cast<int>((M + 127) / 128), Mpad = (nbI + 1) / 2 * 2 * 128;
  const long long Npad = static_cast<long long>((rows + 63) / 64 * 64);
  const std::string sfx = part ? "." + std::to_string(part) : std::string();
  auto* cmax = cmax_ready ? const_cast<unsigned long long*>(cmax_ready)
                          : reinterpret_cast<unsigned long long*>(ctx->dbuf("oz_cmax" + sfx, M));
  auto* exps = reinterpret_cast<int*>(ctx->dbuf("oz_exps" + sfx, (Mpad + 1) / 2));
  auto* planes = reinterpret_cast<int8_t*>(ctx->buf("oz_planes" + sfx, size_t(7) * Mpad * Npad));
  ctx->oz_pending.push_back({r0, rows, static_cast<size_t>(Mpad), static_cast<size_t>(Npad), planes, exps});
  if (!cmax_ready)
    ctx->run("oz_colmax", [&] {
      return launch_oz_colmax(dA, static_cast<long long>(lda), static_cast<long long>(rows), static_cast<int>(M), cmax,
                              ctx->num_sms, ctx->stream);
    });
  ctx->run("oz_slice", [&] {
    return launch_oz_slice(dA, static_cast<long long>(lda), static_cast<long long>(rows), static_cast<int>(M), cmax,
                           exps, Mpad, Npad, planes, ctx->stream);
  });
  // 3-D maps over the planes [plane][row][column]: one box per operand and k-step holds all the planes
  // a group needs (A: 128 columns, 128-byte swizzle; B: this CTA's 64 columns, 64-byte swizzle)
  CUtensorMap maps[4];
  for (int g = 0; g < 2; ++g)
    for (int ab = 0; ab < 2; ++ab) {
      cuuint64_t dims[3] = {static_cast<cuuint64_t>(Mpad), static_cast<cuuint64_t>(Npad), 7};
      cuuint64_t strides[2] = {static_cast<cuuint64_t>(Mpad), static_cast<cuuint64_t>(Mpad) * Npad};
      cuuint32_t box[3] = {ab ? 64u : 128u, 32u, g ? 7u : static_cast<cuuint32_t>(kOzGramPlanesG0)};
      cuuint32_t estr[3] = {1, 1, 1};
      CUresult r = ctx->encode(&maps[2 * g + ab], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, planes, dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, ab ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        fail(RBPG_CUDA_ERROR, "cuTensorMapEncodeTiled (digit planes) failed (" + std::to_string(int(r)) + ")");
    }
  if (ctx->oz_tiles_nbI != nbI) {  // (pair, column) block launch order, uploaded once per tile-grid size
    std::vector<int2> order(size_t(nbI) * nbI + 2);
    const int n = oz_pair_order(nbI, 3, order.data());
    order.resize(n);
    int2* dt = reinterpret_cast<int2*>(ctx->buf("oz_tiles", order.size() * sizeof(int2)));
    ck(cudaMemcpyAsync(dt, order.data(), order.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream),
       "upload tile order");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    ctx->oz_tiles_nbI = nbI;
    ctx->oz_tiles_n = n;
  }
  OzParams p{};
  p.tiles = reinterpret_cast<const int2*>(ctx->buf("oz_tiles", 0));
  p.M = static_cast<int>(M);
  p.nbI = nbI;
  p.nTiles = ctx->oz_tiles_n;
  p.Mpad = Mpad;
  p.Npad = Npad;
  p.ksteps = Npad / 32;
  p.splits = oz_splits(rows, M, ctx->num_sms);
  p.kPerSplit = oz_ksteps_per_split(rows, M, ctx->num_sms);
  p.exps = exps;
  p.ws = ws;
  p.wsStride = static_cast<long long>(oz_slot_doubles(M));
  ctx->run("oz_gram_kernel", [&] { return launch_oz_gram2(maps, p, ctx->stream); });
}
// G (+)= A^T A on the INT8 tensor cores (A: N x M); same contract as gram_dev with m = 0.
void gram_oz_dev(rbpg_context* ctx, const double* dA, size_t lda, size_t N, size_t M, double* dG, size_t ldg,
                 bool accumulate, const unsigned long long* cmax_ready = nullptr) {
  if (N == 0) {
    gram_dev(ctx, dA, lda, 0, M, nullptr, 0, 0, dG, ldg, nullptr, 0, accumulate);
    return;
  }
  const int splits = oz_splits(N, M, ctx->num_sms);
  double* ws = ctx->dbuf("syrk_ws", size_t(2) * splits * oz_slot_doubles(M));
  ctx->oz_pending.clear();
  oz_gram_part(ctx, dA, lda, N, M, ws, 0, 0, cmax_ready);
  ctx->run("syrk_finish", [&] {
    return launch_oz_finish(ws, static_cast<long long>(oz_slot_doubles(M)), 2 * splits, static_cast<int>(M), dG,
                            static_cast<long long>(ldg), accumulate ? 1 : 0, ctx->stream);
  });
}

// The augmented Gram of the train path: INT8 digit-plane Gram unless RBPG_GRAM_DMMA=1 selects the
// FP64 DMMA Gram (comparison / fallback for inputs whose exponents leave the fp64 normal range).
void gram_aug_dev(rbpg_context* ctx, const double* dA, size_t lda, size_t N, size_t M, double* dG, size_t ldg,
                  bool accumulate, const unsigned long long* cmax_ready = nullptr) {
  if (ctx->gram_int8) gram_oz_dev(ctx, dA, lda, N, M, dG, ldg, accumulate, cmax_ready);
  else gram_dev(ctx, dA, lda, N, M, nullptr, 0, 0, dG, ldg, nullptr, 0, accumulate);
}

// Row-blocked Gram G = A^T A over rows [0, N) for the e2e path: part q covers rows
// [ends[q-1], ends[q]) with its own uniform split count, every split writes its own partial slot
// (split0 offset), and one fixed-order reduction sums all parts' partials.  Each part is launched
// by `launch_part(q)` ordering: the caller interleaves its launches with the producers of its rows.
struct GramParts {
  SyrkParams p{};
  std::vector<size_t> ends;
  std::vector<int> splits, split0;
  std::vector<long long> per;
  int total = 0;
};
GramParts gram_parts_plan(rbpg_context* ctx, size_t L, const std::vector<size_t>& ends, double* dG, size_t ldg) {
  GramParts gp;
  gp.ends = ends;
  SyrkParams& p = gp.p;
  p.M = static_cast<int>(L);
  p.nbI = static_cast<int>((L + kTile - 1) / kTile);
  p.nGram = p.nbI * (p.nbI + 1) / 2;
  p.G = dG;
  p.ldg = static_cast<long long>(ldg);
  p.mode = kSyrkPartial;
  size_t r0 = 0;
  for (size_t e : ends) {
    const size_t rows = e - r0;
    if (ctx->gram_int8) {  // INT8 Gram: 2 packed partial slots per split
      const int sp = oz_splits(rows, L, ctx->num_sms);
      gp.split0.push_back(gp.total);
      gp.splits.push_back(sp);
      gp.per.push_back(0);
      gp.total += 2 * sp;
      r0 = e;
      continue;
    }
    int sp = gram_splits(ctx, rows, L, 0, p.nGram, p.nbI);
    long long per = static_cast<long long>(round_up((rows + sp - 1) / sp, kBK));
    if (per == 0) per = kBK;
    sp = static_cast<int>((rows + per - 1) / per);
    gp.split0.push_back(gp.total);
    gp.splits.push_back(sp);
    gp.per.push_back(per);
    gp.total += sp;
    r0 = e;
  }
  const size_t slot = ctx->gram_int8 ? oz_slot_doubles(L) : L * ldg;
  p.ws = ctx->dbuf("syrk_ws", size_t(gp.total) * slot);
  p.wsStride = static_cast<long long>(slot);
  return gp;
}
void gram_parts_launch(rbpg_context* ctx, GramParts& gp, int q, const double* dA, size_t lda,
                       const unsigned long long* cmax_ready = nullptr) {
  const size_t r0 = q == 0 ? 0 : gp.ends[q - 1], rows = gp.ends[q] - r0;
  if (ctx->gram_int8) {
    if (q == 0) ctx->oz_pending.clear();
    oz_gram_part(ctx, dA + r0 * lda, lda, rows, gp.p.M, gp.p.ws + gp.split0[q] * gp.p.wsStride, q, r0, cmax_ready);
    return;
  }
  SyrkParams p = gp.p;
  p.kRows = static_cast<long long>(rows);
  p.kPerSplit = gp.per[q];
  p.split0 = gp.split0[q];
  CUtensorMap tmA = make_map(ctx, dA + r0 * lda, p.M, rows, lda, kTile + 4, kBK, false);
  ctx->run("syrk_kernel", [&] { return launch_syrk(tmA, tmA, p, gp.splits[q], kTile, ctx->stream); });
  if (p.nbI >= 2) ++ctx->launches;
}
void gram_parts_finish(rbpg_context* ctx, GramParts& gp, bool accumulate) {
  if (ctx->gram_int8) {
    ctx->run("syrk_finish", [&] {
      return launch_oz_finish(gp.p.ws, gp.p.wsStride, gp.total, gp.p.M, gp.p.G, gp.p.ldg, accumulate ? 1 : 0,
                              ctx->stream);
    });
    return;
  }
  ctx->run("syrk_finish", [&] { return launch_syrk_finish(gp.p, gp.total, accumulate ? 1 : 0, ctx->num_sms, ctx->stream); });
}

void gemm_dev(rbpg_context* ctx, int M, int N, int K, const double* A, size_t lda, bool tA, const double* B,
              size_t ldb, bool tB, double* C, size_t ldc, double alpha, double beta,
              const char* name = "gemm_kernel") {
  GemmParams p{M, N, K, A, static_cast<long long>(lda), tA ? 1 : 0, B, static_cast<long long>(ldb), tB ? 1 : 0,
               C, static_cast<long long>(ldc), alpha, beta};
  ctx->run(name, [&] { return launch_gemm(p, ctx->stream); });
}

// Blocked TRSM pair for right-hand sides the cluster kernel cannot hold (m > 32, or n too large
// for its shared-memory ring): the 64 x 64 diagonal blocks of F are inverted once, then every block
// step is two DMMA GEMMs -- the block solution W_b = D_b^-1 X_b (D_b^-T backward) and the rank-64
// update of the rows still to solve.  Forward writes X -> W, backward W -> X (or X -> W, copied
// back), so the pair needs no copy.
void trsm_blocked_dev(rbpg_context* ctx, const double* F, size_t ldf, double* X, size_t ldx, size_t n, size_t m,
                      bool fwd, bool bwd) {
  const size_t nblk = (n + 63) / 64;
  double* dinv = ctx->dbuf("trsm.dinv", nblk * 64 * 64);
  ctx->run("trsm_pair_kernel", [&] { return launch_tri_inv(F, static_cast<long long>(ldf), static_cast<int>(n), dinv, ctx->stream); });
  const size_t ldw = even(m);
  double* W = ctx->dbuf("trsm.w", n * ldw);
  double* src = X;
  size_t lds = ldx;
  double* dst = W;
  size_t ldd = ldw;
  const int mi = static_cast<int>(m);
  const long long lf = static_cast<long long>(ldf);
  for (int dir = 0; dir < 2; ++dir) {
    if ((dir == 0 && !fwd) || (dir == 1 && !bwd)) continue;
    for (size_t i = 0; i < nblk; ++i) {
      const size_t b = dir == 0 ? i : nblk - 1 - i;
      const size_t r0 = b * 64, nb = std::min<size_t>(64, n - r0);
      ctx->run("trsm_pair_kernel", [&] {
        return launch_trsm_step(F, lf, dinv + b * 4096, src, static_cast<long long>(lds), dst,
                                static_cast<long long>(ldd), static_cast<int>(n), mi, static_cast<int>(r0),
                                static_cast<int>(nb), dir, ctx->stream);
      });
    }
    std::swap(src, dst);
    std::swap(lds, ldd);
  }
  if (src != X)
    ck(cudaMemcpy2DAsync(X, ldx * 8, src, lds * 8, m * 8, n, cudaMemcpyDeviceToDevice, ctx->stream), "trsm copy");
}

// X (n x m, ld ldx) <- (F F^T)^{-1} X: the cluster kernel for m <= 32 when its rows fit in shared
// memory, the blocked step kernels otherwise
void trsm_pair_dev(rbpg_context* ctx, const double* F, size_t ldf, double* X, size_t ldx, size_t n, size_t m,
                   bool fwd = true, bool bwd = true) {
  if (n == 0 || m == 0 || !(fwd || bwd)) return;
  if (!trsm_cluster_fits(static_cast<int>(n), static_cast<int>(m))) {
    trsm_blocked_dev(ctx, F, ldf, X, ldx, n, m, fwd, bwd);
    return;
  }
  double* dinv = ctx->dbuf("trsm.dinv", ((n + 63) / 64) * 64 * 64);
  ctx->run("trsm_pair_kernel", [&] {
    return launch_trsm_pair(F, static_cast<long long>(ldf), X, static_cast<long long>(ldx), static_cast<int>(n),
                            static_cast<int>(m), fwd ? 1 : 0, bwd ? 1 : 0, ctx->num_sms, dinv, ctx->stream);
  });
}

struct FactorResult {
  const double* F = nullptr;  // factor rows by final position (n x n, ld ldF)
  size_t ldF = 0;
  const int* ord = nullptr;   // device: position -> original column
  FactorState st{};           // host copy (valid after the stream reaches the factorisation's end)
  FactorState* dst = nullptr; // device state
  FactorState* hst = nullptr; // pinned host staging of the state
};

// Diagonal-pivoted (pivoting = 1, linalg.cpp:157-248) or unpivoted SpdFactor (pivoting = 0,
// linalg.cpp:99-139) blocked Cholesky of the symmetric dG (n x n, ld ldg).  dG is not modified.
// neligible < n: the trailing n - neligible columns are right-hand sides carried through the
// factorisation (never pivots): their factor rows become the forward-solved F^{-1} P^T b.
FactorResult factor_dev(rbpg_context* ctx, const double* dG, size_t ldg, size_t n, size_t rows_for_tol, double tol,
                        int pivoting, const std::string& tag, bool sync = true, size_t neligible = SIZE_MAX) {
  cudaStream_t s = ctx->stream;
  if (neligible > n) neligible = n;
  const size_t ldn = round_up(n, 8);
  double* Ga = ctx->dbuf(tag + ".Ga", n * ldn);
  double* Gb = ctx->dbuf(tag + ".Gb", n * ldn);
  double* Fo = ctx->dbuf(tag + ".Fo", n * ldn);
  double* F = ctx->dbuf(tag + ".F", n * ldn);
  double* dv[2] = {ctx->dbuf(tag + ".d0", n), ctx->dbuf(tag + ".d1", n)};
  int* ov[2] = {static_cast<int*>(ctx->buf(tag + ".o0", n * 4)), static_cast<int*>(ctx->buf(tag + ".o1", n * 4))};
  int* lab = static_cast<int*>(ctx->buf(tag + ".lab", n * 4));
  double* Pg = ctx->dbuf(tag + ".Pg", n * 64);
  const size_t ldp = even(n);
  double* PcT = ctx->dbuf(tag + ".PcT", 64 * ldp);
  const int max_ctas = ctx->num_sms;
  PivotSlot* slots = static_cast<PivotSlot*>(ctx->buf(tag + ".slots", sizeof(PivotSlot) * 2 * (max_ctas + 32)));
  FactorState* st = static_cast<FactorState*>(ctx->buf(tag + ".state", sizeof(FactorState)));


  unsigned long long* trace = nullptr;
  const bool trace_wide = std::getenv("RBPG_PANEL_TRACE") && std::string(std::getenv("RBPG_PANEL_TRACE")) == "wide";
  if (std::getenv("RBPG_PANEL_TRACE")) {
    trace = static_cast<unsigned long long*>(ctx->buf(tag + ".ptrace", 128));
    ck(cudaMemsetAsync(trace, 0, 128, s), "memset trace");
  }
  // RBPG_DEVICE_TIMELINE: {entry, start of work, exit} of every panel / trailing launch
  unsigned long long* tl = nullptr;
  const int tl_max = 512;
  int tl_n = 0;
  std::vector<char> tl_kind;
  if (std::getenv("RBPG_DEVICE_TIMELINE")) {
    tl = static_cast<unsigned long long*>(ctx->buf(tag + ".tl", sizeof(unsigned long long) * 3 * tl_max));
    std::vector<unsigned long long> init(3 * tl_max);
    for (int i = 0; i < tl_max; ++i) {
      init[3 * i] = init[3 * i + 1] = ~0ull;
      init[3 * i + 2] = 0;
    }
    ck(cudaMemcpyAsync(tl, init.data(), sizeof(unsigned long long) * 3 * tl_max, cudaMemcpyHostToDevice, s), "tl init");
    ck(cudaStreamSynchronize(s), "tl init sync");
  }
  if (n > 4096) {  // the grid panel variant's global mirror and exchange slots
    ck(cudaMemsetAsync(Pg, 0, sizeof(double) * n * 64, s), "memset Pg");
    ck(cudaMemsetAsync(slots, 0, sizeof(PivotSlot) * 2 * (max_ctas + 32), s), "memset slots");
  }
  ctx->run("factor_setup", [&] {
    return launch_factor_setup(dG, static_cast<long long>(ldg), static_cast<int>(n), static_cast<int>(neligible),
                               static_cast<long long>(rows_for_tol), tol, pivoting, dv[0], ov[0], st, s);
  });
  // the first panel and trailing update read the caller's G in place; later ones ping-pong Ga / Gb
  const double* gcur = dG;
  size_t ldcur = ldg;
  double* gnext = Ga;
  int cur = 0;
  for (size_t k = 0, kb = 0; k < neligible; k += kb) {
    // 64-wide panels, 32-wide while more than 4096 labels remain (k_panel.cu, wide variant)
    kb = std::min<size_t>(static_cast<size_t>(panel_width(static_cast<int>(n), static_cast<int>(k))),
                          neligible - k);
    PanelParams pp{};
    pp.G = gcur;
    pp.ldg = static_cast<long long>(ldcur);
    pp.d_in = dv[cur];
    pp.d_out = dv[1 - cur];
    pp.ord_in = ov[cur];
    pp.ord_out = ov[1 - cur];
    pp.k = static_cast<int>(k);
    pp.kb = static_cast<int>(kb);
    pp.n = static_cast<int>(n);
    pp.st = st;
    pp.Pg = Pg;
    pp.PcT = PcT;
    pp.ldp = static_cast<long long>(ldp);
    pp.lab_out = lab;
    pp.slots = slots;
    pp.Fo = Fo;
    pp.ldf = static_cast<long long>(ldn);
    pp.pivoting = pivoting;
    pp.rows_per_cta = 0;  // chosen by launch_panel
    pp.neligible = static_cast<int>(neligible);
    // RBPG_PANEL_TRACE=wide: only the 32-wide panels (more than 4096 labels left) are traced
    pp.trace = (trace && (!trace_wide || panel_width(static_cast<int>(n), static_cast<int>(k)) < 64)) ? trace : nullptr;
    if (tl && tl_n < tl_max) {
      pp.tl = tl;
      pp.tl_slot = tl_n++;
      tl_kind.push_back('P');
    }
    ctx->run("panel_kernel", [&] { return launch_panel(pp, ctx->num_sms, nullptr, s); });
    const size_t t0 = k + kb;
    if (t0 < neligible) {  // another panel follows
      const size_t nrem = n - t0;
      // 32-wide tiles while they fit in three waves (the late, small updates: their DMMA work per
      // SM is what bounds the update), 64-wide beyond.  (A 128-wide trailing SYRK, which gathers
      // G_old element by element in its epilogue, measured 1.5x slower at L = 8000.)
      const size_t nb32 = (nrem + 31) / 32;
      const int ttile = (nb32 * (nb32 + 1) / 2 <= size_t(3 * ctx->num_sms)) ? 32 : 64;
      CUtensorMap tm = make_map(ctx, PcT, nrem, static_cast<uint64_t>(kb), ldp, ttile + 4, kBK, false);
      SyrkParams sp{};
      sp.M = static_cast<int>(nrem);
      sp.nbI = static_cast<int>((nrem + ttile - 1) / ttile);
      sp.nGram = sp.nbI * (sp.nbI + 1) / 2;
      sp.nbT = 0;
      sp.kRows = static_cast<long long>(kb);
      sp.kPerSplit = static_cast<long long>(round_up(kb, kBK));
      sp.mode = kSyrkTrailing;
      sp.G = gnext;
      sp.ldg = static_cast<long long>(ldn);
      sp.Gold = gcur;
      sp.ldgo = static_cast<long long>(ldcur);
      sp.lab = lab;
      sp.off = static_cast<int>(t0);
      // every panel variant reads G through its lower triangle: no mirrored upper half
      sp.mirror = 0;
      if (tl && tl_n < tl_max) {
        sp.tl = tl;
        sp.tl_slot = tl_n++;
        tl_kind.push_back('T');
      }
      ctx->run("syrk_trailing", [&] { return launch_trail(tm, sp, ttile, s); });
      double* written = gnext;
      gnext = (written == Ga) ? Gb : Ga;
      gcur = written;
      ldcur = ldn;
    }
    cur = 1 - cur;
  }
  ctx->run("gather_factor", [&] { return launch_gather_factor(Fo, static_cast<long long>(ldn), ov[cur], static_cast<int>(n), F,
                                static_cast<long long>(ldn), st, ctx->num_sms, s); });
  FactorResult r;
  r.dst = st;
  // pinned staging so the state copy is truly asynchronous (sync = false: the caller reads it later)
  FactorState* hs = static_cast<FactorState*>(ctx->pinned("factor.state", sizeof(FactorState)));
  ck(cudaMemcpyAsync(hs, st, sizeof(FactorState), cudaMemcpyDeviceToHost, s), "read factor state");
  r.hst = hs;
  if (sync) {
    ck(cudaStreamSynchronize(s), "factor sync");
    r.st = *hs;
  }
  if (tl) {
    std::vector<unsigned long long> h(3 * tl_n);
    ck(cudaStreamSynchronize(s), "tl sync");
    ck(cudaMemcpy(h.data(), tl, sizeof(unsigned long long) * 3 * tl_n, cudaMemcpyDeviceToHost), "tl read");
    const unsigned long long base = h.empty() ? 0 : h[0];
    unsigned long long prev_end = base;
    for (int i = 0; i < tl_n; ++i) {
      std::fprintf(stderr, "[tl %s] %c%-3d entry %8.2f start %8.2f end %8.2f  dur %7.2f  gap %6.2f us\n", tag.c_str(),
                   tl_kind[i], i, (h[3 * i] - base) * 1e-3, (h[3 * i + 1] - base) * 1e-3, (h[3 * i + 2] - base) * 1e-3,
                   (double(h[3 * i + 2]) - double(h[3 * i + 1])) * 1e-3,
                   (double(h[3 * i + 1]) - double(prev_end)) * 1e-3);
      prev_end = h[3 * i + 2];
    }
  }
  if (trace) {
    unsigned long long h[16];
    cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost);
    const double st = double(h[9] ? h[9] : 1);
    std::fprintf(stderr, "[panel trace %s n=%zu] steps %llu cycles/step: pre+wait %.0f resolve %.0f dot %.0f "
                 "sqrt+stop %.0f rcp %.0f col(G) %.0f argmax %.0f bar %.0f publish %.0f (dot: first row chunk at %.0f)\n",
                 tag.c_str(), n, h[9], h[0] / st, h[1] / st, h[2] / st, h[3] / st, h[4] / st, h[5] / st, h[6] / st,
                 h[7] / st, h[8] / st, h[10] / st);
  }
  r.F = F;
  r.ldF = ldn;
  r.ord = ov[cur];
  return r;
}

// SpdFactor with the one-shot ridge rescue (elm.cpp:30-49).  Returns the factor; throws
// SingularSplit(block) if the ridge retry also fails.
FactorResult spd_with_ridge(rbpg_context* ctx, const double* dA, size_t lda, size_t n, double ridge, bool& applied,
                            int block, const std::string& tag) {
  FactorResult f = factor_dev(ctx, dA, lda, n, n, 0.0, 0, tag);
  if (!f.st.fail) return f;
  double* tr = ctx->dbuf(tag + ".trace", 1);
  ctx->run("trace", [&] { return launch_trace(dA, static_cast<long long>(lda), static_cast<int>(n), tr, ctx->stream); });
  double htr = 0.0;
  ck(cudaMemcpyAsync(&htr, tr, 8, cudaMemcpyDeviceToHost, ctx->stream), "read trace");
  ck(cudaStreamSynchronize(ctx->stream), "trace sync");
  double eps = ridge * htr / static_cast<double>(n);
  if (eps <= 0.0) eps = ridge;
  double* R = ctx->dbuf(tag + ".ridge", n * lda);
  ck(cudaMemcpyAsync(R, dA, sizeof(double) * n * lda, cudaMemcpyDeviceToDevice, ctx->stream), "copy ridge");
  ctx->run("add_diag", [&] { return launch_add_diag(R, static_cast<long long>(lda), static_cast<int>(n), eps, ctx->stream); });
  f = factor_dev(ctx, R, lda, n, n, 0.0, 0, tag);
  if (f.st.fail) {
    Fail e{RBPG_SINGULAR_SPLIT, std::string("singular ") + (block == 0 ? "A" : "D") + " block after ridge retry"};
    e.block = block;
    throw e;
  }
  applied = true;
  return f;
}

// ---------------------------------------------------------------------------
// SVD of H for pinv_svd (linalg.cpp:68-87) by block one-sided Jacobi (k_svd.cu).  Tall H (N >= L):
// A = H (N x L); wide H: A = H^T (L x N).  Columns padded with zeros to a multiple of 32.  After
// convergence A = U diag(s) (columns orthogonal), V accumulates the rotations, and w_j = 1/s_j^2
// for the kept s_j > cut = rel * s_max (rel = tol or max(rows, cols) * eps), else 0.
// ---------------------------------------------------------------------------
struct SvdResult {
  double* A = nullptr;  // M x Kp rotated columns (ld Kp)
  double* V = nullptr;  // Kp x Kp (ld Kp)
  double* w = nullptr;  // Kp weights 1/s^2 or 0 (device)
  size_t M = 0, K = 0, Kp = 0;
  bool tall = true;
};

SvdResult svd_dev(rbpg_context* ctx, const double* dH, size_t ldh, size_t N, size_t L, double tol) {
  cudaStream_t s = ctx->stream;
  constexpr double kEps = 2.220446049250313e-16;
  SvdResult r;
  r.tall = N >= L;
  r.M = r.tall ? N : L;
  r.K = r.tall ? L : N;
  r.Kp = round_up(r.K, 32);
  const size_t M = r.M, Kp = r.Kp;
  r.A = ctx->dbuf("svd.A", M * Kp);
  if (r.tall) {
    if (Kp > L) ck(cudaMemsetAsync(r.A, 0, sizeof(double) * M * Kp, s), "memset A");
    ck(cudaMemcpy2DAsync(r.A, Kp * 8, dH, ldh * 8, L * 8, N, cudaMemcpyDeviceToDevice, s), "copy H");
  } else {
    ctx->run("transpose", [&] {
      return launch_transpose(dH, static_cast<long long>(ldh), static_cast<long long>(N), static_cast<long long>(L),
                              r.A, static_cast<long long>(Kp), static_cast<long long>(Kp), s);
    });
  }
  r.V = ctx->dbuf("svd.V", Kp * Kp);
  ck(cudaMemsetAsync(r.V, 0, sizeof(double) * Kp * Kp, s), "memset V");
  ctx->run("add_diag", [&] { return launch_add_diag(r.V, static_cast<long long>(Kp), static_cast<int>(Kp), 1.0, s); });
  double* s2 = ctx->dbuf("svd.s2", Kp);
  double* hs2 = static_cast<double*>(ctx->pinned("svd.s2", Kp * 8));
  auto col_norms = [&] {
    ctx->run("col_sumsq", [&] {
      return launch_col_sumsq(r.A, static_cast<long long>(Kp), static_cast<long long>(M), static_cast<int>(Kp), s2, s);
    });
    ck(cudaMemcpyAsync(hs2, s2, Kp * 8, cudaMemcpyDeviceToHost, s), "read norms");
    ck(cudaStreamSynchronize(s), "svd sync");
  };
  col_norms();
  double fro2 = 0.0;
  for (size_t j = 0; j < Kp; ++j) fro2 += hs2[j];

  const int nb = static_cast<int>(Kp / 16), npairs = nb / 2;
  const size_t want = 2 * static_cast<size_t>(ctx->num_sms);
  auto split_rows = [&](size_t rows) {
    size_t sp = std::max<size_t>(1, (want + npairs - 1) / npairs);
    size_t per = round_up((rows + sp - 1) / sp, 64);
    return std::max<size_t>(per, 64);
  };
  const size_t rows_a = split_rows(M), rows_v = split_rows(Kp);
  const int splits = static_cast<int>((M + rows_a - 1) / rows_a);
  const int vsplits = static_cast<int>((Kp + rows_v - 1) / rows_v);
  double* ws = ctx->dbuf("svd.ws", static_cast<size_t>(npairs) * splits * 1024);
  double* Q = ctx->dbuf("svd.Q", static_cast<size_t>(npairs) * 1024);
  int* flags = static_cast<int*>(ctx->buf("svd.flags", npairs * 4));
  int* rot = static_cast<int*>(ctx->buf("svd.rot", 4));
  int* hrot = static_cast<int*>(ctx->pinned("svd.rot", 4));
  const double otol = 4.0 * kEps * std::sqrt(static_cast<double>(M));
  const double noise = 2.0 * kEps * std::sqrt(fro2);
  constexpr int kMaxSweeps = 60;
  int sweep = 0;
  if (nb >= 2 && fro2 > 0.0) {
    for (; sweep < kMaxSweeps; ++sweep) {
      ck(cudaMemsetAsync(rot, 0, 4, s), "memset rot");
      for (int rd = 0; rd < nb - 1; ++rd)
        ctx->run("svd_round", [&] {
          return launch_svd_round(r.A, static_cast<long long>(Kp), static_cast<long long>(M), r.V,
                                  static_cast<long long>(Kp), static_cast<long long>(Kp), nb, rd, splits,
                                  static_cast<long long>(rows_a), vsplits, static_cast<long long>(rows_v), otol,
                                  noise, ws, Q, flags, rot, s);
        });
      ck(cudaMemcpyAsync(hrot, rot, 4, cudaMemcpyDeviceToHost, s), "read rot");
      ck(cudaStreamSynchronize(s), "svd sweep sync");
      if (*hrot == 0) break;
    }
  }
  ctx->svd_sweeps = sweep + 1;
  col_norms();
  double smax = 0.0;
  std::vector<double> sv(Kp), w(Kp, 0.0);
  for (size_t j = 0; j < Kp; ++j) {
    sv[j] = std::sqrt(hs2[j]);
    smax = std::max(smax, sv[j]);
  }
  const double rel = tol > 0.0 ? tol : static_cast<double>(std::max(N, L)) * kEps;
  const double cut = rel * smax;
  for (size_t j = 0; j < Kp; ++j)
    if (sv[j] > cut && sv[j] > 0.0) w[j] = 1.0 / (sv[j] * sv[j]);
  r.w = ctx->dbuf("svd.w", Kp);
  ck(cudaMemcpyAsync(r.w, w.data(), Kp * 8, cudaMemcpyHostToDevice, s), "upload w");
  ck(cudaStreamSynchronize(s), "svd sync");  // w lives on the host stack
  return r;
}

// beta (L x m) = pinv(H) Y = V diag(w) A^T Y (tall) or A diag(w) V^T Y (wide)
void svd_solve_dev(rbpg_context* ctx, const double* dH, size_t ldh, size_t N, size_t L, const double* dY, size_t ldy,
                   size_t m, double* dBeta, size_t ldb) {
  SvdResult r = svd_dev(ctx, dH, ldh, N, L, 0.0);
  const size_t lm = even(m);
  double* C = ctx->dbuf("svd.C", r.Kp * lm);
  const int Kp = static_cast<int>(r.Kp);
  gemm_dev(ctx, Kp, static_cast<int>(m), static_cast<int>(N), r.tall ? r.A : r.V, r.Kp, true, dY, ldy, false, C, lm,
           1.0, 0.0);
  ctx->run("scale_rows", [&] { return launch_scale_rows(C, static_cast<long long>(lm), Kp, static_cast<int>(m), r.w, ctx->stream); });
  gemm_dev(ctx, static_cast<int>(L), static_cast<int>(m), Kp, r.tall ? r.V : r.A, r.Kp, false, C, lm, false, dBeta,
           ldb, 1.0, 0.0);
}

// pinv(H) (L x N, ld ldo) = V diag(w) A^T (tall) or A diag(w) V[0:N]^T (wide)
void svd_pinv_dev(rbpg_context* ctx, const double* dH, size_t ldh, size_t N, size_t L, double tol, double* dOut,
                  size_t ldo) {
  SvdResult r = svd_dev(ctx, dH, ldh, N, L, tol);
  ctx->run("scale_cols", [&] {
    return launch_scale_cols(r.A, static_cast<long long>(r.Kp), static_cast<long long>(r.M), static_cast<int>(r.Kp),
                             r.w, ctx->stream);
  });
  const int Kp = static_cast<int>(r.Kp);
  if (r.tall)
    gemm_dev(ctx, static_cast<int>(L), static_cast<int>(N), Kp, r.V, r.Kp, false, r.A, r.Kp, true, dOut, ldo, 1.0, 0.0);
  else
    gemm_dev(ctx, static_cast<int>(L), static_cast<int>(N), Kp, r.A, r.Kp, false, r.V, r.Kp, true, dOut, ldo, 1.0, 0.0);
}

// solve_direct (elm.cpp:108-122): SpdFactor(G) and two triangular solves; if N < L or the Gram
// is singular, beta = pinv_svd(H) Y (linalg.cpp:68-87) on the resident H (ctx->src_h).
void direct_dev(rbpg_context* ctx, const double* dG, size_t ldg, const double* dHtT, size_t ldt, size_t L, size_t m,
                size_t rows, double* dBeta, size_t ldb, rbpg_diagnostics* diag) {
  if (rows >= L) {
    FactorResult f = factor_dev(ctx, dG, ldg, L, L, 0.0, 0, "direct");
    if (!f.st.fail) {
      ck(cudaMemcpy2DAsync(dBeta, ldb * 8, dHtT, ldt * 8, m * 8, L, cudaMemcpyDeviceToDevice, ctx->stream),
         "copy rhs");
      trsm_pair_dev(ctx, f.F, f.ldF, dBeta, ldb, L, m);
      return;
    }
    if (diag) diag->used_svd_path = 1;
    if (f.st.dmax0 == 0.0) {  // every column of H is zero: pinv(H) = 0
      ck(cudaMemset2DAsync(dBeta, ldb * 8, 0, m * 8, L, ctx->stream), "zero beta");
      return;
    }
  } else {
    if (diag) diag->used_svd_path = 1;
  }
  if (!ctx->src_h || ctx->src_n != rows)
    fail(RBPG_NOT_SUPPORTED,
         "solve_direct: the SVD pseudoinverse branch needs the whole hidden matrix resident on one device "
         "(not available through the row-sharded stage API)");
  svd_solve_dev(ctx, ctx->src_h, ctx->src_ldh, rows, L, ctx->src_y, ctx->src_ldy, m, dBeta, ldb);
}

// RAII: the resident H / Y of the current call for the SVD branch
struct SourceScope {
  rbpg_context* ctx;
  SourceScope(rbpg_context* c, const double* h, size_t ldh, const double* y, size_t ldy, size_t n) : ctx(c) {
    c->src_h = h;
    c->src_ldh = ldh;
    c->src_y = y;
    c->src_ldy = ldy;
    c->src_n = n;
  }
  ~SourceScope() {
    ctx->src_h = nullptr;
    ctx->src_y = nullptr;
    ctx->src_n = 0;
  }
};

// Schur block solve (elm.cpp:124-156) on Gram sub-blocks.  ord: device position -> original
// column; the first `split` positions form H1, the rest H2.  Writes beta in ORIGINAL order.
void block_dev(rbpg_context* ctx, const double* dG, size_t ldg, const double* dHtT, size_t ldt, size_t L, size_t m,
               size_t rows, const int* ord, size_t split, double* dBeta, size_t ldb, rbpg_diagnostics* diag,
               double ridge_rel = 1e-8) {
  const size_t n1 = split, n2 = L - split;
  if (rows < L) fail(RBPG_SHAPE_ERROR, "solve_block_split: needs at least as many samples as columns");
  cudaStream_t s = ctx->stream;
  const int* P1 = ord;
  const int* P2 = ord + n1;
  const size_t l1 = even(n1), l2 = even(n2), lm = even(m);
  double* A = ctx->dbuf("blk.A", n2 * l2);
  double* G21 = ctx->dbuf("blk.G21", n2 * l1);
  double* D = ctx->dbuf("blk.D", n1 * l1);
  double* X = ctx->dbuf("blk.X", n2 * l1);
  double* Bm = ctx->dbuf("blk.B", n2 * lm);
  double* R1 = ctx->dbuf("blk.R1", n1 * lm);
  double* T2 = ctx->dbuf("blk.T2", n2 * lm);
  double* Bp = ctx->dbuf("blk.beta", L * lm);
  ctx->run("gather A", [&] { return launch_gather_block(dG, ldg, P2, n2, P2, n2, A, l2, s); });
  ctx->run("gather G21", [&] { return launch_gather_block(dG, ldg, P2, n2, P1, n1, G21, l1, s); });
  ctx->run("gather G11", [&] { return launch_gather_block(dG, ldg, P1, n1, P1, n1, D, l1, s); });
  ctx->run("gather H2tT", [&] { return launch_gather_rows(dHtT, ldt, P2, n2, m, Bm, lm, s); });
  ctx->run("gather H1tT", [&] { return launch_gather_rows(dHtT, ldt, P1, n1, m, R1, lm, s); });
  bool ridge = false;
  FactorResult fa = spd_with_ridge(ctx, A, l2, n2, ridge_rel, ridge, 0, "fa");
  trsm_pair_dev(ctx, fa.F, fa.ldF, Bm, lm, n2, m);                                  // B = A^-1 H2^T T
  ck(cudaMemcpy2DAsync(X, l1 * 8, G21, l1 * 8, n1 * 8, n2, cudaMemcpyDeviceToDevice, s), "copy G21");
  trsm_pair_dev(ctx, fa.F, fa.ldF, X, l1, n2, n1);                                  // A^-1 G21
  gemm_dev(ctx, n1, n1, n2, G21, l1, true, X, l1, false, D, l1, -1.0, 1.0);         // D = G11 - G21^T A^-1 G21
  ctx->run("symmetrize", [&] { return launch_symmetrize(D, l1, n1, s); });                          // (D + D^T)/2
  FactorResult fd = spd_with_ridge(ctx, D, l1, n1, ridge_rel, ridge, 1, "fd");
  gemm_dev(ctx, n1, m, n2, G21, l1, true, Bm, lm, false, R1, lm, -1.0, 1.0);        // H1^T(T - H2 B)
  trsm_pair_dev(ctx, fd.F, fd.ldF, R1, lm, n1, m);                                  // beta1
  gemm_dev(ctx, n2, m, n1, G21, l1, false, R1, lm, false, T2, lm, 1.0, 0.0);        // G21 beta1
  trsm_pair_dev(ctx, fa.F, fa.ldF, T2, lm, n2, m);                                  // A^-1 G21 beta1
  ck(cudaMemcpy2DAsync(Bp, lm * 8, R1, lm * 8, m * 8, n1, cudaMemcpyDeviceToDevice, s), "stack beta1");
  ctx->run("beta2", [&] { return launch_axpy_rows(Bm, lm, T2, lm, n2, m, Bp + n1 * lm, lm, s); });  // beta2 = B - ...
  ctx->run("unpermute beta", [&] { return launch_scatter_rows(Bp, lm, ord, L, m, dBeta, ldb, s); });
  if (ridge && diag) diag->ridge_applied = 1;
}

// solve_beta dispatch (elm.cpp:158-229) on device G (original coordinates) and HtT.
// gaug: dG is the whole augmented Gram [H T]^T [H T] ((L+m) x (L+m), ld ldg) with dHtT = dG + L.
// The rank path then factors it with the m target columns carried along as never-pivot labels, so
// the factorisation itself forward-solves F y = P^T H^T T (y = their factor rows) and only the
// backward substitution F^T x = y remains (cf. solve_factored_gram, linalg.cpp:254-270).
// post (optional): work enqueued behind the speculative full-rank solve before the single rank
// readback (train()'s finiteness check and accuracy pass); *post_valid tells the caller whether that
// work ran on the final beta (rank == L) or must be repeated after the fallback solve.
void solve_dev(rbpg_context* ctx, const double* dG, size_t ldg, const double* dHtT, size_t ldt, size_t L, size_t m,
               size_t rows, const rbpg_strategy& sg, double* dBeta, size_t ldb, size_t* order_out,
               rbpg_diagnostics* diag, bool gaug = false, const std::function<void()>* post = nullptr,
               bool* post_valid = nullptr) {
  if (post_valid) *post_valid = false;
  if (sg.kind == RBPG_DIRECT) {
    diag->split_lo = L;
    diag->split_hi = 0;
    direct_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, dBeta, ldb, diag);
    return;
  }
  if (sg.kind == RBPG_DF_SPLIT) {
    const size_t sidx = sg.split_index;
    if (sidx < 1 || sidx >= L)
      fail(RBPG_INVALID_ARGUMENT, "solve_beta: df split index must be in (0, " + std::to_string(L) + "), got " +
                                      std::to_string(sidx));
    diag->split_lo = sidx;
    diag->split_hi = L - sidx;
    std::vector<int> id(L);
    for (size_t i = 0; i < L; ++i) id[i] = static_cast<int>(i);
    int* dord = static_cast<int*>(ctx->buf("df.ord", L * 4));
    ck(cudaMemcpyAsync(dord, id.data(), L * 4, cudaMemcpyHostToDevice, ctx->stream), "upload identity");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    try {
      block_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, dord, sidx, dBeta, ldb, diag);
    } catch (const Fail& e) {
      if (e.code != RBPG_SINGULAR_SPLIT) throw;
      diag->fallback_to_direct = 1;
      direct_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, dBeta, ldb, diag);
    }
    return;
  }
  if (sg.kind != RBPG_RANK_BASED) fail(RBPG_RUNTIME_ERROR, "solve_beta: unknown strategy");
  if (sg.rank_tol < 0.0 || !std::isfinite(sg.rank_tol))
    fail(RBPG_INVALID_ARGUMENT, "rank_revealing_permutation: tolerance must be >= 0");
  const bool aug = gaug && m > 0 && m <= 32;
  FactorResult f = factor_dev(ctx, dG, ldg, aug ? L + m : L, rows, sg.rank_tol, 1, "rrf", false, L);
  // speculate the full-rank solve (elm.cpp:202-214) before the one host readback of the rank;
  // with rank < L its result is discarded
  const size_t lm = even(m);
  double* rhs = ctx->dbuf("rank.rhs", L * lm);
  if (aug) {  // y (forward-solved, position order) = rows L.. of the factor, transposed
    ctx->run("transpose y", [&] {
      return launch_transpose(f.F + L * f.ldF, static_cast<long long>(f.ldF), static_cast<long long>(m),
                              static_cast<long long>(L), rhs, static_cast<long long>(lm), static_cast<long long>(m),
                              ctx->stream);
    });
    trsm_pair_dev(ctx, f.F, f.ldF, rhs, lm, L, m, false, true);
  } else {
    ctx->run("gather rhs", [&] { return launch_gather_rows(dHtT, ldt, f.ord, L, m, rhs, lm, ctx->stream); });
    trsm_pair_dev(ctx, f.F, f.ldF, rhs, lm, L, m);
  }
  ctx->run("unpermute beta", [&] { return launch_scatter_rows(rhs, lm, f.ord, L, m, dBeta, ldb, ctx->stream); });
  int* ho = static_cast<int*>(ctx->pinned("order.out", L * 4));
  if (order_out) ck(cudaMemcpyAsync(ho, f.ord, L * 4, cudaMemcpyDeviceToHost, ctx->stream), "read order");
  if (post) (*post)();
  ck(cudaStreamSynchronize(ctx->stream), "factor sync");
  f.st = *f.hst;
  const size_t rank = static_cast<size_t>(f.st.rank);
  diag->rank = rank;
  diag->rank_known = 1;
  if (order_out)
    for (size_t i = 0; i < L; ++i) order_out[i] = static_cast<size_t>(ho[i]);
  if (rank == 0 || L < 2) {
    diag->fallback_to_direct = 1;
    diag->split_lo = L;
    diag->split_hi = 0;
    direct_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, dBeta, ldb, diag);
    return;
  }
  const size_t split = (rank == L) ? (L + 1) / 2 : rank;
  diag->split_lo = split;
  diag->split_hi = L - split;
  if (rank == L) {  // the speculated solve is the answer
    if (post_valid) *post_valid = post != nullptr;
    return;
  }
  try {
    block_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, f.ord, split, dBeta, ldb, diag);
  } catch (const Fail& e) {
    if (e.code != RBPG_SINGULAR_SPLIT) throw;
    diag->fallback_to_direct = 1;
    direct_dev(ctx, dG, ldg, dHtT, ldt, L, m, rows, dBeta, ldb, diag);
  }
}

// non-finite beta check (elm.cpp:275-277); with defer the flag lands in pinned memory and the
// caller tests it after its own synchronisation
const int* check_finite(rbpg_context* ctx, const double* dBeta, size_t ldb, size_t L, size_t m, bool defer = false) {
  int* flag = static_cast<int*>(ctx->buf("nonfinite", 4));
  ck(cudaMemsetAsync(flag, 0, 4, ctx->stream), "memset flag");
  ctx->run("nonfinite", [&] { return launch_nonfinite(dBeta, static_cast<long long>(ldb), static_cast<int>(L), static_cast<int>(m), flag,
                            ctx->stream); });
  int* h = static_cast<int*>(ctx->pinned("nonfinite", 4));
  ck(cudaMemcpyAsync(h, flag, 4, cudaMemcpyDeviceToHost, ctx->stream), "read flag");
  if (defer) return h;
  ck(cudaStreamSynchronize(ctx->stream), "sync");
  if (*h) fail(RBPG_RUNTIME_ERROR, "train: solver produced non-finite output weights");
  return h;
}

struct Padded {
  const double* p;
  size_t ld;
};
// device matrix with an even leading dimension and 16-byte aligned base (TMA rules)
Padded pad_device(rbpg_context* ctx, const std::string& name, const double* d, size_t ld, size_t rows, size_t cols) {
  if (ld % 2 == 0 && (reinterpret_cast<uintptr_t>(d) & 15) == 0) return {d, ld};
  const size_t nld = even(cols);
  double* q = ctx->dbuf(name, rows * nld);
  ck(cudaMemcpy2DAsync(q, nld * 8, d, ld * 8, cols * 8, rows, cudaMemcpyDeviceToDevice, ctx->stream), "pad copy");
  return {q, nld};
}
// host <-> device copies: one linear transfer when the rows are contiguous on both sides (a pitched
// 2D copy of many short rows runs at a fraction of the link bandwidth)
void copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
               cudaMemcpyKind kind, cudaStream_t s, const char* what) {
  if (!rows || !width) return;
  if (dpitch == width && spitch == width)
    ck(cudaMemcpyAsync(dst, src, width * rows, kind, s), what);
  else
    ck(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, s), what);
}
Padded upload(rbpg_context* ctx, const std::string& name, const double* h, size_t rows, size_t cols) {
  const size_t ld = even(cols);
  double* q = ctx->dbuf(name, std::max<size_t>(1, rows) * ld);
  copy_rows(q, ld * 8, h, cols * 8, cols * 8, rows, cudaMemcpyHostToDevice, ctx->stream, "upload");
  return {q, ld};
}
void download(rbpg_context* ctx, double* h, const double* d, size_t ld, size_t rows, size_t cols) {
  copy_rows(h, cols * 8, d, ld * 8, cols * 8, rows, cudaMemcpyDeviceToHost, ctx->stream, "download");
  ck(cudaStreamSynchronize(ctx->stream), "sync");
}

size_t h_chunk_rows(rbpg_context* ctx, size_t N, size_t ldh) {
  size_t rows = ctx->h_budget_bytes / (ldh * 8);
  rows = std::max<size_t>(rows / kTile * kTile, kTile);
  return std::min(rows, N);
}

// Stage 1: H build + Gram/HtT over the local rows (chunked when H exceeds the budget).
// Returns the summed K1 time (ms) when timing events are requested.
// The Gram is taken of the augmented rows [H | T] (N x (L+m)): its lower triangle holds H^T H and,
// mirrored, H^T T = Gaug[0:L, L:L+m], so the H^T T product rides in the SYRK's last tile row
// instead of 128-wide tiles that would carry only m useful columns.
// `ready` (optional): row blocks of X/T still being uploaded, as (end row, event recorded after the
// block's copy); the hidden build then runs per block behind its upload (one Gram over all rows).
struct RowReady {
  size_t end;
  cudaEvent_t ev;
};
float gram_stage(rbpg_context* ctx, const double* dX, size_t ldx, const double* dT, size_t ldt_in, size_t N,
                 size_t d, size_t L, size_t m, const double* dW, size_t ldw, const double* db, double* dGaug,
                 size_t ldga, bool accumulate, bool keep_h, bool timed,
                 const std::vector<RowReady>* ready = nullptr) {
  const size_t M = L + m;
  const size_t ldh = even(M);
  const size_t chunk = std::max<size_t>(1, h_chunk_rows(ctx, std::max<size_t>(N, 1), ldh));
  const rbpg_context::KeptKey key{dX, dW, db, ldx, ldw, d};
  ctx->kept_h = nullptr;  // the H buffer is rewritten below
  double* dH = ctx->dbuf("H", chunk * ldh);
  float hidden_ms = 0.f;
  if (N == 0) {
    gram_dev(ctx, dH, ldh, 0, M, nullptr, 0, 0, dGaug, ldga, nullptr, 0, accumulate);
    return 0.f;
  }
  // Gram parts behind the uploads: part 0 covers the first upload blocks and runs while the later
  // blocks arrive; their hidden builds go on the aux stream, concurrently with the Gram parts on
  // the main stream; part q > 0 starts once the aux stream has built its last block.
  // Default cuts (measured on one B200, PCIe ~40 GB/s): after block 2 when the Gram + hidden work
  // outlasts the upload (C2: 3.83 -> 3.74 ms e2e), every 2 blocks when the upload dominates
  // (C4 L = 250: 3.32 -> 2.96 ms).  Parts end after these upload-block counts (the last part
  // always ends at N).
  const double upload_s = double(N) * double(d + m) * 8.0 / 40e9;
  const double compute_s = (2.0 * N * d * L + double(N) * M * M) / 30e12;
  const std::vector<size_t> part_cuts =
      upload_s > compute_s ? std::vector<size_t>{2, 4, 6} : std::vector<size_t>{2};
  std::vector<size_t> cuts;  // block counts ending parts 0 .. P-2
  if (ready && chunk >= N && M >= 2 * kTile)
    for (size_t c : part_cuts)
      if (c < ready->size()) cuts.push_back(c);
  if (!cuts.empty()) {
    std::vector<size_t> ends;
    for (size_t c : cuts) ends.push_back((*ready)[c - 1].end);
    ends.push_back(N);
    GramParts gp = gram_parts_plan(ctx, M, ends, dGaug, ldga);
    if (timed) cudaEventRecord(ctx->ev[0], ctx->stream);
    ck(cudaEventRecord(ctx->aux_ev[0], ctx->stream), "event");  // H rows free (earlier work done)
    ck(cudaStreamWaitEvent(ctx->aux, ctx->aux_ev[0], 0), "wait");
    // column maxima of each part's rows of [H T], accumulated by the hidden builds (the INT8 Gram's scan)
    std::vector<unsigned long long*> pcm(cuts.size() + 1, nullptr);
    if (ctx->gram_int8)
      for (size_t qq = 0; qq <= cuts.size(); ++qq)
        pcm[qq] = reinterpret_cast<unsigned long long*>(ctx->dbuf("oz_hcmax." + std::to_string(qq), M));
    size_t r0 = 0, q = 0;
    for (size_t i = 0; i < ready->size(); ++i) {
      const RowReady& rr = (*ready)[i];
      const bool on_aux = i >= cuts[0];
      const size_t part = static_cast<size_t>(std::upper_bound(cuts.begin(), cuts.end(), i) - cuts.begin());
      ck(cudaStreamWaitEvent(on_aux ? ctx->aux : ctx->stream, rr.ev, 0), "wait upload");
      if (on_aux) std::swap(ctx->stream, ctx->aux);
      if (pcm[part] && i == (part == 0 ? 0 : cuts[part - 1]))  // first block of the part
        ck(cudaMemsetAsync(pcm[part], 0, M * sizeof(unsigned long long), ctx->stream), "zero column maxima");
      hidden_dev(ctx, dX + r0 * ldx, ldx, rr.end - r0, d, dW, ldw, db, L, dH + r0 * ldh, ldh, dT + r0 * ldt_in,
                 ldt_in, m, pcm[part]);
      if (on_aux) std::swap(ctx->stream, ctx->aux);
      r0 = rr.end;
      if (q < cuts.size() && i + 1 == cuts[q]) {  // part q's rows are built: launch it on the main stream
        if (q > 0) {
          ck(cudaEventRecord(ctx->aux_ev[1 + q], ctx->aux), "event");
          ck(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1 + q], 0), "wait hidden");
        }
        gram_parts_launch(ctx, gp, static_cast<int>(q), dH, ldh, pcm[q]);
        ++q;
      }
    }
    ck(cudaEventRecord(ctx->aux_ev[1], ctx->aux), "event");
    ck(cudaStreamWaitEvent(ctx->stream, ctx->aux_ev[1], 0), "wait hidden");
    if (timed) cudaEventRecord(ctx->ev[1], ctx->stream);
    gram_parts_launch(ctx, gp, static_cast<int>(cuts.size()), dH, ldh, pcm[cuts.size()]);
    gram_parts_finish(ctx, gp, accumulate);
    if (keep_h) {
      ctx->keep_h(dH, N, L, ldh, key);
    } else {
      ctx->kept_h = nullptr;
    }
    return 0.f;
  }
  if (ready && chunk >= N) {
    if (timed) cudaEventRecord(ctx->ev[0], ctx->stream);
    unsigned long long* cm = nullptr;
    if (ctx->gram_int8) {
      cm = reinterpret_cast<unsigned long long*>(ctx->dbuf("oz_hcmax.0", M));
      ck(cudaMemsetAsync(cm, 0, M * sizeof(unsigned long long), ctx->stream), "zero column maxima");
    }
    size_t r0 = 0;
    for (const RowReady& rr : *ready) {
      ck(cudaStreamWaitEvent(ctx->stream, rr.ev, 0), "wait upload");
      hidden_dev(ctx, dX + r0 * ldx, ldx, rr.end - r0, d, dW, ldw, db, L, dH + r0 * ldh, ldh, dT + r0 * ldt_in,
                 ldt_in, m, cm);
      r0 = rr.end;
    }
    if (timed) cudaEventRecord(ctx->ev[1], ctx->stream);
    // (a row-blocked Gram behind the uploads was measured slower: its per-block wave
    // quantisation costs more than the hidden upload tail)
    gram_aug_dev(ctx, dH, ldh, N, M, dGaug, ldga, accumulate, cm);
    if (keep_h) {
      ctx->keep_h(dH, N, L, ldh, key);
    } else {
      ctx->kept_h = nullptr;
    }
    return 0.f;
  }
  for (size_t r0 = 0; r0 < N; r0 += chunk) {
    const size_t nr = std::min(chunk, N - r0);
    // chunk 0 is timed by ev[0]/ev[1] without a sync (read by the caller after its own sync);
    // further chunks (H larger than the budget) synchronise on ev[4]/ev[5]
    cudaEvent_t ea = r0 == 0 ? ctx->ev[0] : ctx->ev[4], eb = r0 == 0 ? ctx->ev[1] : ctx->ev[5];
    if (timed) cudaEventRecord(ea, ctx->stream);
    unsigned long long* cm = nullptr;
    if (ctx->gram_int8) {
      cm = reinterpret_cast<unsigned long long*>(ctx->dbuf("oz_hcmax.0", M));
      ck(cudaMemsetAsync(cm, 0, M * sizeof(unsigned long long), ctx->stream), "zero column maxima");
    }
    hidden_dev(ctx, dX + r0 * ldx, ldx, nr, d, dW, ldw, db, L, dH, ldh, dT + r0 * ldt_in, ldt_in, m, cm);  // + T columns
    if (timed) {
      cudaEventRecord(eb, ctx->stream);
      if (r0 > 0) {
        cudaEventSynchronize(eb);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ea, eb);
        hidden_ms += ms;
      }
    }
    gram_aug_dev(ctx, dH, ldh, nr, M, dGaug, ldga, accumulate || r0 > 0, cm);
  }
  if (keep_h && chunk >= N) {
    ctx->keep_h(dH, N, L, ldh, key);
  } else {
    ctx->kept_h = nullptr;
  }
  return hidden_ms;
}

// Stage 3: hits = #rows with argmax(H beta) == argmax(T)
// K6: S (optional) = H beta and/or hits += #rows with argmax(H beta) == argmax(T); m <= 128.
void scores_dev(rbpg_context* ctx, const double* H, size_t ldh, size_t N, size_t L, const double* dBeta, size_t ldb,
                size_t m, double* S, size_t lds, const double* T, size_t ldt, unsigned long long* hits) {
  if (N == 0) return;
  Padded B = pad_device(ctx, "beta.pad", dBeta, ldb, L, m);
  const uint32_t bn = static_cast<uint32_t>((m + 15) / 16 * 16);  // scores_kernel<BN>, BN = m rounded up to 16
  CUtensorMap tmH = make_map(ctx, H, L, N, ldh, 16, kTile, true);
  CUtensorMap tmB = make_map(ctx, B.p, m, L, B.ld, bn + 4, kBK, false);  // padded smem rows
  ScoresParams p{static_cast<int>(N), static_cast<int>(L), static_cast<int>(m), S, static_cast<long long>(lds), T,
                 static_cast<long long>(ldt), hits};
  ctx->run("scores_kernel", [&] { return launch_scores(tmH, tmB, p, ctx->stream); });
}

// K6i (k_ozaki.cu): the training-accuracy pass on the INT8 tensor cores, from the digit planes the Gram
// of the kept H wrote (one launch per Gram part: each part has its own column exponents, folded into
// beta's planes).  Valid when those parts cover exactly the N kept rows and the plane rows (the columns
// of [H T]) fit the int32 headroom.
bool oz_scores_ready(rbpg_context* ctx, size_t N, size_t M) {
  if (!ctx->gram_int8 || ctx->oz_kept.empty() || ctx->oz_kept_h != ctx->kept_h) return false;
  size_t r = 0;
  for (const auto& pt : ctx->oz_kept) {
    if (pt.r0 != r || pt.Mpad > 16384 || pt.Mpad < M) return false;
    r += pt.rows;
  }
  return r == N;
}
// One Gram part's INT8 scores: beta folded with the part's column exponents and split per class, then
// the hit count (labels = targets), and / or the arg-max labels and the scores of the part's rows.
void oz_scores_part(rbpg_context* ctx, const rbpg_context::OzPart& pt, size_t L, size_t m, const double* dBeta,
                    size_t ldb, const int* tlabels, unsigned long long* hits, int* out_labels, double* S, size_t lds) {
  const size_t K = pt.Mpad;
  auto* bp = reinterpret_cast<int8_t*>(ctx->buf("ozs.bplanes", 7 * 128 * K));
  double* cs = ctx->dbuf("ozs.cscale", 128);
  ctx->run("scores_kernel", [&] {
    return launch_oz_beta_planes(dBeta, static_cast<long long>(ldb), static_cast<int>(L), static_cast<int>(m), pt.exps,
                                 static_cast<int>(K), bp, cs, ctx->stream);
  });
  auto map = [&](int8_t* base, size_t rows, uint32_t box_rows, uint32_t np) {
    CUtensorMap mp;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), 7};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(K) * rows};
    cuuint32_t box[3] = {32u, box_rows, np};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = ctx->encode(&mp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(RBPG_CUDA_ERROR, "cuTensorMapEncodeTiled (scores planes) failed (" + std::to_string(int(r)) + ")");
    return mp;
  };
  CUtensorMap maps[4] = {map(pt.planes, pt.Npad, 128, 4), map(bp, 128, 64, 4), map(pt.planes, pt.Npad, 128, 7),
                         map(bp, 128, 64, 7)};
  OzScoresParams p{};
  p.rows = static_cast<int>(pt.rows);
  p.m = static_cast<int>(m);
  p.nP = static_cast<int>((pt.rows + 255) / 256);
  p.ksteps = static_cast<int>(K / 32);
  p.cscale = cs;
  p.labels = tlabels ? tlabels + pt.r0 : nullptr;
  p.hits = hits;
  p.out_labels = out_labels ? out_labels + pt.r0 : nullptr;
  p.S = S ? S + pt.r0 * lds : nullptr;
  p.lds = static_cast<long long>(lds);
  ctx->run("scores_kernel", [&] { return launch_oz_scores(maps, p, ctx->stream); });
}
void oz_scores_dev(rbpg_context* ctx, size_t N, size_t L, size_t m, const double* dBeta, size_t ldb, const double* dT,
                   size_t ldt, unsigned long long* hits) {
  int* labels = reinterpret_cast<int*>(ctx->buf("ozs.labels", N * sizeof(int)));
  ctx->run("scores_kernel", [&] {
    return launch_oz_labels(dT, static_cast<long long>(ldt), static_cast<long long>(N), static_cast<int>(m), labels,
                            ctx->stream);
  });
  for (const auto& pt : ctx->oz_kept) oz_scores_part(ctx, pt, L, m, dBeta, ldb, labels, hits, nullptr, nullptr, 0);
}

// K6b: fused sigma(X W + b) beta with the arg-max epilogue (m <= 128): optional scores S, labels,
// and hits += #rows whose arg-max equals argmax(T).  H is never written.
void predict_dev(rbpg_context* ctx, const double* dX, size_t ldx, size_t N, size_t d, const double* dW, size_t ldw,
                 const double* db, size_t L, const double* dBeta, size_t ldb, size_t m, double* S, size_t lds,
                 int* labels, const double* T, size_t ldt, unsigned long long* hits) {
  if (N == 0) return;
  const int mp = predict_mp(static_cast<int>(m));
  if (mp == 0) fail(RBPG_INVALID_ARGUMENT, "predict_dev: more than 128 classes");
  // m > 48: the INT8 path (K1i hidden build of a row chunk with its column scan, digit planes, K6i
  // scores) -- the fused DMMA kernel below is FP64-bound on its scores product there
  if (ctx->gram_int8 && m > 48 && d <= kOzHidMaxD && (L + 255) / 256 * 256 <= 16384) {
    const size_t ldh = even(L);
    const size_t chunk = std::min<size_t>(N, std::max<size_t>(256, (size_t(8) << 30) / (ldh * 15)));
    double* dH = ctx->dbuf("pred.H", chunk * ldh);
    auto* cm = reinterpret_cast<unsigned long long*>(ctx->dbuf("pred.cmax", L));
    int* tl = nullptr;
    if (T && hits) {
      tl = reinterpret_cast<int*>(ctx->buf("pred.tlabels", N * sizeof(int)));
      ctx->run("scores_kernel", [&] {
        return launch_oz_labels(T, static_cast<long long>(ldt), static_cast<long long>(N), static_cast<int>(m), tl,
                                ctx->stream);
      });
    }
    for (size_t r0 = 0; r0 < N; r0 += chunk) {
      const size_t nr = std::min(chunk, N - r0);
      ck(cudaMemsetAsync(cm, 0, L * sizeof(unsigned long long), ctx->stream), "zero column maxima");
      hidden_oz_dev(ctx, dX + r0 * ldx, ldx, nr, d, dW, ldw, db, L, dH, ldh, cm);
      const int nbI = static_cast<int>((L + 127) / 128), Mpad = (nbI + 1) / 2 * 2 * 128;
      const long long Npad = static_cast<long long>((nr + 63) / 64 * 64);
      int* exps = reinterpret_cast<int*>(ctx->dbuf("pred.exps", (Mpad + 1) / 2));
      auto* planes = reinterpret_cast<int8_t*>(ctx->buf("pred.planes", size_t(7) * Mpad * Npad));
      ctx->run("oz_slice", [&] {
        return launch_oz_slice(dH, static_cast<long long>(ldh), static_cast<long long>(nr), static_cast<int>(L), cm, exps,
                               Mpad, Npad, planes, ctx->stream);
      });
      rbpg_context::OzPart pt{0, nr, static_cast<size_t>(Mpad), static_cast<size_t>(Npad), planes, exps};
      oz_scores_part(ctx, pt, L, m, dBeta, ldb, tl ? tl + r0 : nullptr, hits, labels ? labels + r0 : nullptr,
                     S ? S + r0 * lds : nullptr, lds);
    }
    return;
  }
  Padded X = pad_device(ctx, "pred.x", dX, ldx, N, d);
  Padded W = pad_device(ctx, "pred.w", dW, ldw, d, L);
  Padded B = pad_device(ctx, "beta.pad", dBeta, ldb, L, m);
  CUtensorMap tmX = make_map(ctx, X.p, d, N, X.ld, 16, kTile, true);
  CUtensorMap tmW = make_map(ctx, W.p, L, d, W.ld, 36, kBK, false);
  CUtensorMap tmB = make_map(ctx, B.p, m, L, B.ld, static_cast<uint32_t>(mp + 4), 32, false);
  PredictParams p{static_cast<int>(N), static_cast<int>(d), static_cast<int>(L), static_cast<int>(m), db,
                  S, static_cast<long long>(lds), labels, T, static_cast<long long>(ldt), hits};
  ctx->run("predict_kernel", [&] { return launch_predict(tmX, tmW, tmB, p, ctx->stream); });
}

uint64_t accuracy_stage(rbpg_context* ctx, const double* dX, size_t ldx, const double* dT, size_t ldt_in, size_t N,
                        size_t d, size_t L, size_t m, const double* dW, size_t ldw, const double* db,
                        const double* dBeta, size_t ldb, unsigned long long** deferred = nullptr) {
  unsigned long long* hits = static_cast<unsigned long long*>(ctx->buf("hits", 8));
  ck(cudaMemsetAsync(hits, 0, 8, ctx->stream), "memset hits");
  if (N > 0) {
    const size_t ldh = even(L);
    const bool kept = ctx->kept_for(rbpg_context::KeptKey{dX, dW, db, ldx, ldw, d}, N, L);
    if (!kept && m <= 128) {  // no resident H for these inputs: the fused predict kernel recomputes it
      predict_dev(ctx, dX, ldx, N, d, dW, ldw, db, L, dBeta, ldb, m, nullptr, 0, nullptr, dT, ldt_in, hits);
    } else {
      if (!kept) ctx->kept_h = nullptr;  // the H buffer is rebuilt from these inputs below
      const size_t chunk = kept ? N : h_chunk_rows(ctx, N, ldh);
      const size_t lm = even(m);
      double* S = ctx->dbuf("scores", chunk * lm);
      for (size_t r0 = 0; r0 < N; r0 += chunk) {
        const size_t nr = std::min(chunk, N - r0);
        const double* H = ctx->kept_h;
        size_t hld = ctx->kept_ldh;
        if (!kept) {
          double* dH = ctx->dbuf("H", chunk * ldh);
          hidden_dev(ctx, dX + r0 * ldx, ldx, nr, d, dW, ldw, db, L, dH, ldh);
          H = dH;
          hld = ldh;
        }
        // K6i on the Gram's digit planes for many classes: its cost (28 int8 products against the 128
        // padded classes per row) undercuts the DMMA K6 once m > 48, where K6 turns FP64-bound (C5,
        // m = 100: 31 -> 11 ms); below, K6 reads H once at HBM speed (C4, m = 10: 1.2 vs 2.7 ms)
        if (kept && m > 48 && m <= 128 && oz_scores_ready(ctx, N, L + m)) {
          oz_scores_dev(ctx, N, L, m, dBeta, ldb, dT, ldt_in, hits);
          break;
        }
        if (m <= 128) {  // K6: skinny DMMA GEMM with the fused arg-max / hit count, scores never stored
          scores_dev(ctx, H, hld, nr, L, dBeta, ldb, m, nullptr, 0, dT + r0 * ldt_in, ldt_in, hits);
        } else {
          gemm_dev(ctx, static_cast<int>(nr), static_cast<int>(m), static_cast<int>(L), H, hld, false, dBeta, ldb,
                   false, S, lm, 1.0, 0.0);
          ctx->run("accuracy", [&] {
            return launch_accuracy(S, static_cast<long long>(lm), dT + r0 * ldt_in, static_cast<long long>(ldt_in),
                                   static_cast<long long>(nr), static_cast<int>(m), hits, ctx->num_sms, ctx->stream);
          });
        }
      }
    }
  }
  unsigned long long* h = static_cast<unsigned long long*>(ctx->pinned("hits", 8));
  ck(cudaMemcpyAsync(h, hits, 8, cudaMemcpyDeviceToHost, ctx->stream), "read hits");
  if (deferred) {
    *deferred = h;
    return 0;
  }
  ck(cudaStreamSynchronize(ctx->stream), "sync");
  return *h;
}

// train() body on device-resident X, T (elm.cpp:231-280 after validation and init_hidden)
void train_core(rbpg_context* ctx, const double* dX, size_t ldx, const double* dT, size_t ldt_in, size_t N, size_t d,
                size_t L, size_t m, const double* w, const double* b, const rbpg_strategy& sg, double* dBeta,
                size_t ldb, size_t* order_out, rbpg_diagnostics* diag,
                const std::vector<RowReady>* ready = nullptr, bool wb_uploaded = false) {
  Padded X = pad_device(ctx, "X.pad", dX, ldx, N, d);
  Padded T = pad_device(ctx, "T.pad", dT, ldt_in, N, m);
  Padded W{ctx->dbuf("W", std::max<size_t>(1, d) * even(L)), even(L)};
  double* db = ctx->dbuf("b", L);
  if (!wb_uploaded) {  // else already on the device (uploaded by the caller ahead of the inputs)
    W = upload(ctx, "W", w, d, L);
    ck(cudaMemcpyAsync(db, b, L * 8, cudaMemcpyHostToDevice, ctx->stream), "upload b");
  }
  // augmented Gram [H T]^T [H T]: G = Gaug[0:L, 0:L], H^T T = Gaug[0:L, L:L+m] (same ld)
  const size_t ldg = round_up(L + m, 8), ldt = ldg;
  double* G = ctx->dbuf("G0", (L + m) * ldg);
  double* HtT = G + L;

  const auto wall0 = std::chrono::steady_clock::now();
  const int* bad = nullptr;
  unsigned long long* hits = nullptr;
  cudaEventRecord(ctx->ev[2], ctx->stream);
  float hidden_ms = gram_stage(ctx, X.p, X.ld, T.p, T.ld, N, d, L, m, W.p, W.ld, db, G, ldg, false, true, true, ready);
  {
    // [H T] stays resident (unless H exceeded the memory budget) for solve_direct's SVD branch
    const bool kept = ctx->kept_for(rbpg_context::KeptKey{X.p, W.p, db, X.ld, W.ld, d}, N, L);
    SourceScope src(ctx, kept ? ctx->kept_h : nullptr, ctx->kept_ldh, kept ? ctx->kept_h + L : nullptr,
                    ctx->kept_ldh, kept ? N : 0);
    // finiteness check and accuracy pass enqueued behind the (speculative) solve: one
    // synchronisation for the rank, the check and the hit count
    const std::function<void()> post = [&] {
      cudaEventRecord(ctx->ev[3], ctx->stream);
      bad = check_finite(ctx, dBeta, ldb, L, m, true);
      accuracy_stage(ctx, X.p, X.ld, T.p, T.ld, N, d, L, m, W.p, W.ld, db, dBeta, ldb, &hits);
    };
    bool done = false;
    solve_dev(ctx, G, ldg, HtT, ldt, L, m, N, sg, dBeta, ldb, order_out, diag, true, &post, &done);
    if (!done) post();  // other strategies, or the rank < L fallback changed beta
  }
  ck(cudaStreamSynchronize(ctx->stream), "sync");
  float total_ms = 0.f, first_hidden_ms = 0.f;
  cudaEventElapsedTime(&total_ms, ctx->ev[2], ctx->ev[3]);
  if (N > 0) cudaEventElapsedTime(&first_hidden_ms, ctx->ev[0], ctx->ev[1]);
  hidden_ms += first_hidden_ms;
  (void)wall0;
  diag->hidden_seconds = hidden_ms * 1e-3;
  diag->solve_seconds = std::max(0.f, total_ms - hidden_ms) * 1e-3;
  if (*bad) fail(RBPG_RUNTIME_ERROR, "train: solver produced non-finite output weights");
  diag->training_accuracy = N ? static_cast<double>(*hits) / static_cast<double>(N) : 0.0;
}

// ---------------------------------------------------------------------------
// Rank-path pseudo-inverse H^+ (SURVEY §8 a11).  For rank(H) = L it is the full-rank solve of
// elm.cpp:202-214 with right-hand side H^T: H^+ = P (F F^T)^{-1} P^T H^T.  Device form:
//   Z    = (F F^T)^{-1}             triangular-solve pair on the identity (L right-hand sides)
//   Ginv = P Z P^T                  gather (Ginv[a][b] = Z[pos a][pos b])
//   H^+  = Ginv H^T                 one DMMA product over the rows of H (hidden_kernel, plain
//                                   transposed epilogue): 2 L^2 N tensor-core flops instead of
//                                   N / 128 latency-bound triangular sweeps.
// The factorisation and Ginv depend only on G, so a row shard of H yields its column block of
// H^+ from the all-reduced Gram with no further exchange.
// ---------------------------------------------------------------------------
struct PinvFactor {
  const double* Ginv = nullptr;  // L x L (ld), original node order; null when rank < L
  size_t ld = 0;
  size_t rank = 0;
  std::vector<int> order;
};

PinvFactor pinv_factor_dev(rbpg_context* ctx, const double* dG, size_t ldg, size_t L, size_t rows_for_tol,
                           double tol) {
  if (tol < 0.0 || !std::isfinite(tol)) fail(RBPG_INVALID_ARGUMENT, "rank_revealing_permutation: tolerance must be >= 0");
  FactorResult f = factor_dev(ctx, dG, ldg, L, rows_for_tol, tol, 1, "pinv");
  PinvFactor r;
  r.rank = static_cast<size_t>(f.st.rank);
  r.order.resize(L);
  ck(cudaMemcpy(r.order.data(), f.ord, L * 4, cudaMemcpyDeviceToHost), "read order");
  if (r.rank != L) return r;
  const size_t ld = round_up(L, 8);
  double* Z = ctx->dbuf("pinv.Z", L * ld);
  ck(cudaMemsetAsync(Z, 0, sizeof(double) * L * ld, ctx->stream), "memset Z");
  ctx->run("add_diag", [&] { return launch_add_diag(Z, static_cast<long long>(ld), static_cast<int>(L), 1.0, ctx->stream); });
  trsm_pair_dev(ctx, f.F, f.ldF, Z, ld, L, L);
  std::vector<int> pos(L);
  for (size_t i = 0; i < L; ++i) pos[r.order[i]] = static_cast<int>(i);
  int* dpos = static_cast<int*>(ctx->buf("pinv.pos", L * 4));
  ck(cudaMemcpyAsync(dpos, pos.data(), L * 4, cudaMemcpyHostToDevice, ctx->stream), "upload pos");
  double* Ginv = ctx->dbuf("pinv.Ginv", L * ld);
  ctx->run("gather Ginv", [&] {
    return launch_gather_block(Z, static_cast<long long>(ld), dpos, static_cast<int>(L), dpos, static_cast<int>(L),
                               Ginv, static_cast<long long>(ld), ctx->stream);
  });
  ck(cudaStreamSynchronize(ctx->stream), "pinv sync");  // pos lives on the host stack
  r.Ginv = Ginv;
  r.ld = ld;
  return r;
}

// out (L x N, ld ldo) = Ginv (L x L) * H^T for H (N x L, ld ldh)
void pinv_apply_dev(rbpg_context* ctx, const double* Ginv, size_t ldgi, const double* dH, size_t ldh, size_t N, size_t L,
                    double* dOut, size_t ldo) {
  if (N == 0) return;
  CUtensorMap tmH = make_map(ctx, dH, L, N, ldh, 16, kTile, true);
  CUtensorMap tmG = make_map(ctx, Ginv, L, L, ldgi, kTile + 4, kBK, false);  // padded smem rows
  HiddenParams p{static_cast<int>(N), static_cast<int>(L), static_cast<int>(L), nullptr, dOut,
                 static_cast<long long>(ldo), 1};
  ctx->run("pinv_apply", [&] { return launch_hidden(tmH, tmG, p, kTile, ctx->stream); });
}

void rank_deficient_pinv(const PinvFactor& pf, size_t L) {
  fail(RBPG_INVALID_ARGUMENT, "solve_factored_gram: factor is rank-deficient (" + std::to_string(pf.rank) + " of " +
                                  std::to_string(L) + ")");
}

template <typename F>
int guarded(rbpg_context* ctx, rbpg_status* st, F&& body) {
  if (st) std::memset(st, 0, sizeof(*st));
  try {
    if (ctx) {
      std::lock_guard<std::mutex> lk(ctx->mu);
      ck(cudaSetDevice(ctx->device), "cudaSetDevice");
      body();
    } else {
      body();
    }
    return RBPG_OK;
  } catch (const Fail& e) {
    if (st) {
      st->code = e.code;
      st->pivot_index = e.pivot_index;
      st->pivot_value = e.pivot_value;
      st->block = e.block;
      std::snprintf(st->message, sizeof st->message, "%s", e.msg.c_str());
    }
    return e.code;
  } catch (const std::exception& e) {
    if (st) {
      st->code = RBPG_RUNTIME_ERROR;
      std::snprintf(st->message, sizeof st->message, "%s", e.what());
    }
    return RBPG_RUNTIME_ERROR;
  }
}

void zero_diag(rbpg_diagnostics* d) { std::memset(d, 0, sizeof(*d)); d->training_accuracy = -1.0; }

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int rbpg_context_create(int device, rbpg_context** out, rbpg_status* st) {
  return guarded(nullptr, st, [&] {
    int count = 0;
    ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count) fail(RBPG_CUDA_ERROR, "no such CUDA device " + std::to_string(device));
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      fail(RBPG_CUDA_ERROR, std::string("rbpelm-b200 is built for sm_100a (B200); device is ") + prop.name);
    auto* c = new rbpg_context();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    ck(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking), "copy stream");
    ck(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking), "aux stream");
    for (auto& e : c->chunk_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : c->aux_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    c->stream = c->own;
    for (auto& e : c->ev) ck(cudaEventCreate(&e), "event");
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q), "driver entry point");
    if (!fn || q != cudaDriverEntryPointSuccess) fail(RBPG_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    c->encode = reinterpret_cast<EncodeTiledFn>(fn);
    if (const char* e = std::getenv("RBPG_H_BUDGET_GB")) c->h_budget_bytes = size_t(std::atof(e) * (1ull << 30));
    *out = c;
  });
}

void rbpg_context_destroy(rbpg_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamSynchronize(ctx->copy);
  for (auto& kv : ctx->bufs) cudaFree(kv.second.first);
  for (auto& kv : ctx->hbufs) cudaFreeHost(kv.second.first);
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  for (auto& e : ctx->chunk_ev) cudaEventDestroy(e);
  for (auto& e : ctx->aux_ev) cudaEventDestroy(e);
  cudaStreamSynchronize(ctx->aux);
  cudaStreamDestroy(ctx->own);
  cudaStreamDestroy(ctx->copy);
  cudaStreamDestroy(ctx->aux);
  delete ctx;
}

int rbpg_context_set_stream(rbpg_context* ctx, void* stream, rbpg_status* st) {
  return guarded(ctx, st, [&] { ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own; });
}
int rbpg_context_synchronize(rbpg_context* ctx, rbpg_status* st) {
  return guarded(ctx, st, [&] { ck(cudaStreamSynchronize(ctx->stream), "sync"); });
}
uint64_t rbpg_context_launch_count(const rbpg_context* ctx) { return ctx ? ctx->launches : 0; }

int rbpg_context_set_profiling(rbpg_context* ctx, int enable, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    ctx->collect();
    ctx->prof.clear();
    ctx->profile = enable != 0;
  });
}

int rbpg_context_profile_get(rbpg_context* ctx, const char* name, double* total_ms, uint64_t* count,
                             rbpg_status* st) {
  return guarded(ctx, st, [&] {
    ctx->collect();
    auto it = ctx->prof.find(name);
    *total_ms = it == ctx->prof.end() ? 0.0 : it->second.ms;
    *count = it == ctx->prof.end() ? 0 : it->second.count;
  });
}

int rbpg_hidden_matrix(rbpg_context* ctx, const double* w, const double* b, size_t d, size_t l, const double* x,
                       size_t n, size_t xcols, double* h, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (xcols != d)
      fail(RBPG_SHAPE_ERROR, "hidden_matrix: sample has " + std::to_string(xcols) +
                                 " features but the layer expects " + std::to_string(d));
    Padded X = upload(ctx, "X.in", x, n, d);
    Padded W = upload(ctx, "W", w, d, l);
    double* db = ctx->dbuf("b", l);
    ck(cudaMemcpyAsync(db, b, l * 8, cudaMemcpyHostToDevice, ctx->stream), "upload b");
    const size_t ldh = even(l);
    double* H = ctx->dbuf("H", n * ldh);
    ctx->kept_h = nullptr;
    hidden_dev(ctx, X.p, X.ld, n, d, W.p, W.ld, db, l, H, ldh);
    download(ctx, h, H, ldh, n, l);
  });
}

int rbpg_gram(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double* g, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    Padded A = upload(ctx, "A.in", a, rows, cols);
    const size_t ldg = round_up(cols, 8);
    double* G = ctx->dbuf("G0", cols * ldg);
    gram_dev(ctx, A.p, A.ld, rows, cols, nullptr, 0, 0, G, ldg, nullptr, 0, false);
    download(ctx, g, G, ldg, cols, cols);
  });
}

int rbpg_rank_revealing_factor(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double tol,
                               size_t* order, size_t* rank, double* tolerance, double* factor, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (rows == 0 || cols == 0) fail(RBPG_SHAPE_ERROR, "rank_revealing_permutation: empty matrix");
    if (tol < 0.0 || !std::isfinite(tol))
      fail(RBPG_INVALID_ARGUMENT, "rank_revealing_permutation: tolerance must be >= 0");
    Padded A = upload(ctx, "A.in", a, rows, cols);
    const size_t ldg = round_up(cols, 8);
    double* G = ctx->dbuf("G0", cols * ldg);
    gram_dev(ctx, A.p, A.ld, rows, cols, nullptr, 0, 0, G, ldg, nullptr, 0, false);
    FactorResult f = factor_dev(ctx, G, ldg, cols, rows, tol, 1, "rrf");
    std::vector<int> o(cols);
    ck(cudaMemcpy(o.data(), f.ord, cols * 4, cudaMemcpyDeviceToHost), "read order");
    for (size_t i = 0; i < cols; ++i) order[i] = static_cast<size_t>(o[i]);
    *rank = static_cast<size_t>(f.st.rank);
    *tolerance = f.st.tolerance;
    if (factor) download(ctx, factor, f.F, f.ldF, cols, cols);
  });
}

int rbpg_solve_factored_gram(rbpg_context* ctx, const double* factor, const size_t* order, size_t n, size_t rank,
                             const double* rhs, size_t rrows, size_t m, double* out, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    (void)order;
    if (rank != n)
      fail(RBPG_INVALID_ARGUMENT, "solve_factored_gram: factor is rank-deficient (" + std::to_string(rank) + " of " +
                                      std::to_string(n) + ")");
    if (rrows != n)
      fail(RBPG_SHAPE_ERROR,
           "solve_factored_gram: rhs has " + std::to_string(rrows) + " rows, expected " + std::to_string(n));
    Padded F = upload(ctx, "F.in", factor, n, n);
    Padded X = upload(ctx, "rhs.in", rhs, n, m);
    trsm_pair_dev(ctx, F.p, F.ld, const_cast<double*>(X.p), X.ld, n, m);
    download(ctx, out, X.p, X.ld, n, m);
  });
}

int rbpg_pseudo_inverse(rbpg_context* ctx, const double* h, size_t n, size_t l, double tol, double* out,
                        size_t* order, size_t* rank, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (n == 0 || l == 0) fail(RBPG_SHAPE_ERROR, "pseudo_inverse: empty matrix");
    Padded H = upload(ctx, "A.in", h, n, l);
    const size_t ldg = round_up(l, 8);
    double* G = ctx->dbuf("G0", l * ldg);
    gram_dev(ctx, H.p, H.ld, n, l, nullptr, 0, 0, G, ldg, nullptr, 0, false);
    PinvFactor pf = pinv_factor_dev(ctx, G, ldg, l, n, tol);
    for (size_t i = 0; i < l; ++i) order[i] = static_cast<size_t>(pf.order[i]);
    *rank = pf.rank;
    if (pf.rank != l) rank_deficient_pinv(pf, l);
    const size_t ldo = even(n);
    double* O = ctx->dbuf("pinv.out", l * ldo);
    pinv_apply_dev(ctx, pf.Ginv, pf.ld, H.p, H.ld, n, l, O, ldo);
    download(ctx, out, O, ldo, l, n);
  });
}

int rbpg_pinv_svd(rbpg_context* ctx, const double* a, size_t rows, size_t cols, double tol, double* out,
                  rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (rows == 0 || cols == 0) fail(RBPG_SHAPE_ERROR, "pinv_svd: empty matrix");
    Padded A = upload(ctx, "A.in", a, rows, cols);
    const size_t ldo = even(rows);
    double* O = ctx->dbuf("pinv.out", cols * ldo);
    svd_pinv_dev(ctx, A.p, A.ld, rows, cols, tol, O, ldo);
    download(ctx, out, O, ldo, cols, rows);
  });
}

int rbpg_gram_device(rbpg_context* ctx, const double* da, size_t lda, size_t rows, size_t cols, double* dg, size_t ldg,
                     int accumulate, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (cols == 0) fail(RBPG_SHAPE_ERROR, "gram: empty matrix");
    Padded A = pad_device(ctx, "gram.a", da, lda, rows, cols);
    if (ldg % 2 == 0 && (reinterpret_cast<uintptr_t>(dg) & 15) == 0) {
      gram_dev(ctx, A.p, A.ld, rows, cols, nullptr, 0, 0, dg, ldg, nullptr, 0, accumulate != 0);
    } else {  // 16-byte vector stores: stage an odd leading dimension / unaligned base
      const size_t lds = round_up(cols, 8);
      double* S = ctx->dbuf("gram.stage", cols * lds);
      if (accumulate)
        ck(cudaMemcpy2DAsync(S, lds * 8, dg, ldg * 8, cols * 8, cols, cudaMemcpyDeviceToDevice, ctx->stream), "stage");
      gram_dev(ctx, A.p, A.ld, rows, cols, nullptr, 0, 0, S, lds, nullptr, 0, accumulate != 0);
      ck(cudaMemcpy2DAsync(dg, ldg * 8, S, lds * 8, cols * 8, cols, cudaMemcpyDeviceToDevice, ctx->stream), "store");
    }
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int rbpg_gram_int8_device(rbpg_context* ctx, const double* da, size_t lda, size_t rows, size_t cols, double* dg,
                          size_t ldg, int accumulate, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (cols == 0) fail(RBPG_SHAPE_ERROR, "gram: empty matrix");
    if (ldg < cols) fail(RBPG_SHAPE_ERROR, "gram: ldg < cols");
    gram_oz_dev(ctx, da, lda, rows, cols, dg, ldg, accumulate != 0);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int rbpg_pseudo_inverse_stage_device(rbpg_context* ctx, const double* dg, size_t ldg, size_t n_total,
                                     const double* dh, size_t ldh, size_t n_local, size_t l, double tol, double* dout,
                                     size_t ldo, size_t* order, size_t* rank, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (n_total == 0 || l == 0) fail(RBPG_SHAPE_ERROR, "pseudo_inverse: empty matrix");
    PinvFactor pf = pinv_factor_dev(ctx, dg, ldg, l, n_total, tol);
    if (order)
      for (size_t i = 0; i < l; ++i) order[i] = static_cast<size_t>(pf.order[i]);
    if (rank) *rank = pf.rank;
    if (pf.rank != l) rank_deficient_pinv(pf, l);
    Padded H = pad_device(ctx, "pinv.h", dh, ldh, n_local, l);
    pinv_apply_dev(ctx, pf.Ginv, pf.ld, H.p, H.ld, n_local, l, dout, ldo);
    ck(cudaStreamSynchronize(ctx->stream), "sync");
  });
}

int rbpg_solve_spd(rbpg_context* ctx, const double* mat, size_t mrows, size_t mcols, const double* rhs, size_t rrows,
                   size_t rcols, double* out, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (mrows != mcols) fail(RBPG_SHAPE_ERROR, "solve_spd: matrix is not square, " + shp(mrows, mcols));
    const size_t n = mrows;
    double scale = 0.0, asym = 0.0;  // linalg.cpp:104-107 (host validation)
    for (size_t i = 0; i < n * n; ++i) scale = std::max(scale, std::fabs(mat[i]));
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) asym = std::max(asym, std::fabs(mat[i * n + j] - mat[j * n + i]));
    if (asym > 1e-12 * std::max(scale, 1.0))
      fail(RBPG_INVALID_ARGUMENT, "solve_spd: matrix is not symmetric within 1e-12 relative");
    Padded M = upload(ctx, "M.in", mat, n, n);
    FactorResult f = factor_dev(ctx, M.p, M.ld, n, n, 0.0, 0, "spd");
    if (f.st.fail) {
      Fail e{RBPG_SINGULAR_MATRIX, "non-positive pivot " + std::to_string(f.st.fail_value) + " at index " +
                                       std::to_string(f.st.fail_index) + " in symmetric factorization"};
      e.pivot_index = static_cast<size_t>(f.st.fail_index);
      e.pivot_value = f.st.fail_value;
      throw e;
    }
    if (rrows != n)
      fail(RBPG_SHAPE_ERROR, "solve_spd: rhs has " + std::to_string(rrows) + " rows, expected " + std::to_string(n));
    Padded X = upload(ctx, "rhs.in", rhs, n, rcols);
    trsm_pair_dev(ctx, f.F, f.ldF, const_cast<double*>(X.p), X.ld, n, rcols);
    download(ctx, out, X.p, X.ld, n, rcols);
  });
}

int rbpg_solve_beta(rbpg_context* ctx, const double* h, size_t n, size_t l, const double* y, size_t yrows, size_t m,
                    const rbpg_strategy* strategy, double* beta, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    if (n == 0 || l == 0) fail(RBPG_SHAPE_ERROR, "solve_beta: empty hidden matrix");
    if (yrows != n) fail(RBPG_SHAPE_ERROR, "solve_beta: H is " + shp(n, l) + " but Y is " + shp(yrows, m));
    // [H | Y] in one buffer: one SYRK gives H^T H and H^T Y (see gram_stage)
    const size_t lda = even(l + m);
    double* A = ctx->dbuf("A.in", n * lda);
    ck(cudaMemcpy2DAsync(A, lda * 8, h, l * 8, l * 8, n, cudaMemcpyHostToDevice, ctx->stream), "upload H");
    ck(cudaMemcpy2DAsync(A + l, lda * 8, y, m * 8, m * 8, n, cudaMemcpyHostToDevice, ctx->stream), "upload Y");
    const size_t ldg = round_up(l + m, 8), ldt = ldg, lb = even(m);
    double* G = ctx->dbuf("G0", (l + m) * ldg);
    double* HtT = G + l;
    double* B = ctx->dbuf("beta", l * lb);
    gram_dev(ctx, A, lda, n, l + m, nullptr, 0, 0, G, ldg, nullptr, 0, false);
    SourceScope src(ctx, A, lda, A + l, lda, n);
    solve_dev(ctx, G, ldg, HtT, ldt, l, m, n, *strategy, B, lb, nullptr, diag, true);
    download(ctx, beta, B, lb, l, m);
  });
}

int rbpg_train(rbpg_context* ctx, size_t inputs, size_t hidden, size_t outputs, uint64_t seed, const double* x,
               size_t n, size_t xcols, const double* y, size_t yrows, size_t ycols, const rbpg_strategy* strategy,
               double* w, double* b, double* beta, size_t* order, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    // validation order of elm.cpp:234-258
    if (n != yrows) fail(RBPG_SHAPE_ERROR, "train: X is " + shp(n, xcols) + " but Y is " + shp(yrows, ycols));
    if (xcols != inputs)
      fail(RBPG_SHAPE_ERROR, "train: X has " + std::to_string(xcols) + " features but params.inputs is " +
                                 std::to_string(inputs));
    if (ycols != outputs)
      fail(RBPG_SHAPE_ERROR, "train: Y has " + std::to_string(ycols) + " columns but params.outputs is " +
                                 std::to_string(outputs));
    if (strategy->kind != RBPG_DIRECT && n < hidden)
      fail(RBPG_INVALID_ARGUMENT, "train: block strategies need at least as many samples as hidden nodes (" +
                                      std::to_string(n) + " < " + std::to_string(hidden) + "); use the direct strategy");
    if (strategy->kind == RBPG_DF_SPLIT && (strategy->split_index < 1 || strategy->split_index >= hidden))
      fail(RBPG_INVALID_ARGUMENT, "train: df split index must be in (0, " + std::to_string(hidden) + "), got " +
                                      std::to_string(strategy->split_index));
    // X and T go up in row blocks on the copy stream; the hidden build of each block waits only for
    // its own upload, and W, b are generated on the host meanwhile
    const size_t ldx = even(xcols), ldy = even(ycols);
    double* dX = ctx->dbuf("X.in", std::max<size_t>(1, n) * ldx);
    double* dY = ctx->dbuf("T.in", std::max<size_t>(1, n) * ldy);
    std::vector<RowReady> ready;
    {
      constexpr size_t max_blk = 7;  // upload blocks (10 or 14 measured slower at C2)
      const size_t nblk = std::min<size_t>(max_blk, std::max<size_t>(1, n / 4096));
      const size_t per = round_up((n + nblk - 1) / nblk, kTile);
      ck(cudaEventRecord(ctx->chunk_ev[15], ctx->stream), "event");  // buffers free (prior work done)
      ck(cudaStreamWaitEvent(ctx->copy, ctx->chunk_ev[15], 0), "wait");
      for (size_t r0 = 0, i = 0; r0 < n; r0 += per, ++i) {
        const size_t nr = std::min(per, n - r0);
        copy_rows(dX + r0 * ldx, ldx * 8, x + r0 * xcols, xcols * 8, xcols * 8, nr, cudaMemcpyHostToDevice,
                  ctx->copy, "upload X");
        copy_rows(dY + r0 * ldy, ldy * 8, y + r0 * ycols, ycols * 8, ycols * 8, nr, cudaMemcpyHostToDevice,
                  ctx->copy, "upload Y");
        if (i == 0) {  // W, b generated on the host while block 0 is in flight, then queued behind it
          rbpg_status s2;
          if (rbpg_init_hidden(inputs, hidden, outputs, seed, w, b, &s2)) fail(s2.code, s2.message);
          double* dW = ctx->dbuf("W", inputs * even(hidden));
          copy_rows(dW, even(hidden) * 8, w, hidden * 8, hidden * 8, inputs, cudaMemcpyHostToDevice, ctx->copy,
                    "upload W");
          ck(cudaMemcpyAsync(ctx->dbuf("b", hidden), b, hidden * 8, cudaMemcpyHostToDevice, ctx->copy), "upload b");
        }
        ck(cudaEventRecord(ctx->chunk_ev[i], ctx->copy), "event");
        ready.push_back({r0 + nr, ctx->chunk_ev[i]});
      }
    }
    if (ready.empty()) {  // no rows: W, b were not generated inside the loop
      rbpg_status s2;
      if (rbpg_init_hidden(inputs, hidden, outputs, seed, w, b, &s2)) fail(s2.code, s2.message);
    }
    const size_t lb = even(outputs);
    double* B = ctx->dbuf("beta", hidden * lb);
    train_core(ctx, dX, ldx, dY, ldy, n, inputs, hidden, outputs, w, b, *strategy, B, lb, order, diag, &ready,
               !ready.empty());
    download(ctx, beta, B, lb, hidden, outputs);
  });
}

int rbpg_predict(rbpg_context* ctx, const double* w, const double* b, size_t d, size_t l, const double* beta,
                 size_t m, const double* x, size_t n, size_t xcols, double* scores, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (xcols != d)
      fail(RBPG_SHAPE_ERROR, "hidden_matrix: sample has " + std::to_string(xcols) +
                                 " features but the layer expects " + std::to_string(d));
    Padded X = upload(ctx, "X.in", x, n, d);
    Padded W = upload(ctx, "W", w, d, l);
    Padded Bt = upload(ctx, "beta.in", beta, l, m);
    double* db = ctx->dbuf("b", l);
    ck(cudaMemcpyAsync(db, b, l * 8, cudaMemcpyHostToDevice, ctx->stream), "upload b");
    const size_t lm = even(m);
    double* S = ctx->dbuf("scores", std::max<size_t>(n, 1) * lm);
    if (m <= 128) {  // K6b: fused, H never stored
      predict_dev(ctx, X.p, X.ld, n, d, W.p, W.ld, db, l, Bt.p, Bt.ld, m, S, lm, nullptr, nullptr, 0, nullptr);
    } else {  // K1 into row chunks of H, then the DMMA GEMM
      const size_t ldh = even(l);
      const size_t chunk = h_chunk_rows(ctx, std::max<size_t>(n, 1), ldh);
      double* H = ctx->dbuf("H", chunk * ldh);
      ctx->kept_h = nullptr;
      for (size_t r0 = 0; r0 < n; r0 += chunk) {
        const size_t nr = std::min(chunk, n - r0);
        hidden_dev(ctx, X.p + r0 * X.ld, X.ld, nr, d, W.p, W.ld, db, l, H, ldh);
        gemm_dev(ctx, static_cast<int>(nr), static_cast<int>(m), static_cast<int>(l), H, ldh, false, Bt.p, Bt.ld,
                 false, S + r0 * lm, lm, 1.0, 0.0);
      }
    }
    download(ctx, scores, S, lm, n, m);
  });
}

int rbpg_predict_device(rbpg_context* ctx, const double* dx, size_t ldx, size_t n, size_t d, const double* dw,
                        size_t ldw, const double* db, size_t l, const double* dbeta, size_t ldb, size_t m,
                        double* dscores, size_t lds, int* dlabels, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (m > 128) fail(RBPG_NOT_SUPPORTED, "predict_device: at most 128 classes (use rbpg_predict)");
    if (n == 0 || l == 0 || m == 0) return;
    predict_dev(ctx, dx, ldx, n, d, dw, ldw, db, l, dbeta, ldb, m, dscores, lds, dlabels, nullptr, 0, nullptr);
  });
}

int rbpg_solve_block_split(rbpg_context* ctx, const double* h1, size_t n, size_t c1, const double* h2, size_t n2,
                           size_t c2, const double* y, size_t yrows, size_t m, double ridge, double* beta1,
                           double* beta2, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    if (n2 != n || yrows != n)  // elm.cpp:128-131
      fail(RBPG_SHAPE_ERROR, "solve_block_split: row counts differ (" + shp(n, c1) + ", " + shp(n2, c2) + ", " +
                                 shp(yrows, m) + ")");
    if (n < c1 + c2) fail(RBPG_SHAPE_ERROR, "solve_block_split: needs at least as many samples as columns");
    if (c1 == 0 || c2 == 0 || m == 0) fail(RBPG_SHAPE_ERROR, "solve_block_split: empty block");
    // [H1 H2 Y] in one buffer: one SYRK gives every Gram block the Schur solve needs
    const size_t L = c1 + c2, lda = even(L + m);
    double* A = ctx->dbuf("A.in", n * lda);
    ck(cudaMemcpy2DAsync(A, lda * 8, h1, c1 * 8, c1 * 8, n, cudaMemcpyHostToDevice, ctx->stream), "upload H1");
    ck(cudaMemcpy2DAsync(A + c1, lda * 8, h2, c2 * 8, c2 * 8, n, cudaMemcpyHostToDevice, ctx->stream), "upload H2");
    ck(cudaMemcpy2DAsync(A + L, lda * 8, y, m * 8, m * 8, n, cudaMemcpyHostToDevice, ctx->stream), "upload Y");
    const size_t ldg = round_up(L + m, 8), lb = even(m);
    double* G = ctx->dbuf("G0", (L + m) * ldg);
    gram_dev(ctx, A, lda, n, L + m, nullptr, 0, 0, G, ldg, nullptr, 0, false);
    std::vector<int> id(L);
    for (size_t i = 0; i < L; ++i) id[i] = static_cast<int>(i);
    int* dord = static_cast<int*>(ctx->buf("bs.ord", L * 4));
    ck(cudaMemcpyAsync(dord, id.data(), L * 4, cudaMemcpyHostToDevice, ctx->stream), "upload identity");
    double* B = ctx->dbuf("beta", L * lb);
    block_dev(ctx, G, ldg, G + L, ldg, L, m, n, dord, c1, B, lb, diag, ridge);
    download(ctx, beta1, B, lb, c1, m);
    download(ctx, beta2, B + c1 * lb, lb, c2, m);
  });
}

// SpdFactor (linalg.cpp:99-151) kept on the device: factor once, solve many right-hand sides
struct rbpg_spd {
  rbpg_context* ctx;
  double* F = nullptr;  // lower factor (n x ldF), owned
  size_t n = 0, ldF = 0;
};

int rbpg_spd_create(rbpg_context* ctx, const double* mat, size_t mrows, size_t mcols, rbpg_spd** out,
                    rbpg_status* st) {
  *out = nullptr;
  return guarded(ctx, st, [&] {
    if (mrows != mcols) fail(RBPG_SHAPE_ERROR, "solve_spd: matrix is not square, " + shp(mrows, mcols));
    const size_t n = mrows;
    double scale = 0.0, asym = 0.0;  // linalg.cpp:104-107 (host validation)
    for (size_t i = 0; i < n * n; ++i) scale = std::max(scale, std::fabs(mat[i]));
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) asym = std::max(asym, std::fabs(mat[i * n + j] - mat[j * n + i]));
    if (asym > 1e-12 * std::max(scale, 1.0))
      fail(RBPG_INVALID_ARGUMENT, "solve_spd: matrix is not symmetric within 1e-12 relative");
    Padded M = upload(ctx, "M.in", mat, n, n);
    FactorResult f = factor_dev(ctx, M.p, M.ld, n, n, 0.0, 0, "spd");
    if (f.st.fail) {
      Fail e{RBPG_SINGULAR_MATRIX, "non-positive pivot " + std::to_string(f.st.fail_value) + " at index " +
                                       std::to_string(f.st.fail_index) + " in symmetric factorization"};
      e.pivot_index = static_cast<size_t>(f.st.fail_index);
      e.pivot_value = f.st.fail_value;
      throw e;
    }
    auto* h = new rbpg_spd{ctx};
    h->n = n;
    h->ldF = f.ldF;
    if (cudaMalloc(&h->F, sizeof(double) * std::max<size_t>(1, n * f.ldF)) != cudaSuccess) {
      delete h;
      fail(RBPG_CUDA_ERROR, "cudaMalloc SpdFactor");
    }
    ck(cudaMemcpyAsync(h->F, f.F, sizeof(double) * n * f.ldF, cudaMemcpyDeviceToDevice, ctx->stream), "copy F");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    *out = h;
  });
}

int rbpg_spd_solve(const rbpg_spd* f, const double* rhs, size_t rrows, size_t rcols, double* out, rbpg_status* st) {
  return guarded(f->ctx, st, [&] {
    if (rrows != f->n)
      fail(RBPG_SHAPE_ERROR, "solve_spd: rhs has " + std::to_string(rrows) + " rows, expected " + std::to_string(f->n));
    if (rcols == 0) return;
    Padded X = upload(f->ctx, "rhs.in", rhs, f->n, rcols);
    trsm_pair_dev(f->ctx, f->F, f->ldF, const_cast<double*>(X.p), X.ld, f->n, rcols);
    download(f->ctx, out, X.p, X.ld, f->n, rcols);
  });
}

size_t rbpg_spd_dim(const rbpg_spd* f) { return f ? f->n : 0; }

void rbpg_spd_destroy(rbpg_spd* f) {
  if (!f) return;
  cudaSetDevice(f->ctx->device);
  cudaStreamSynchronize(f->ctx->stream);
  cudaFree(f->F);
  delete f;
}

// matmul (matrix.cpp:69-77) / matmul_at (matrix.cpp:79-87) on the DMMA GEMM
int rbpg_matmul(rbpg_context* ctx, const double* a, size_t ar, size_t ac, int trans_a, const double* b, size_t br,
                size_t bc, double* out, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    const size_t M = trans_a ? ac : ar, K = trans_a ? ar : ac;
    if (K != br) {
      if (trans_a)
        fail(RBPG_SHAPE_ERROR, "matmul_at: row counts differ, " + shp(ar, ac) + "^T times " + shp(br, bc));
      fail(RBPG_SHAPE_ERROR, "matmul: inner dimensions differ, " + shp(ar, ac) + " times " + shp(br, bc));
    }
    if (M == 0 || bc == 0) return;
    Padded A = upload(ctx, "mm.a", a, ar, ac);
    Padded B = upload(ctx, "mm.b", b, br, bc);
    const size_t ldc = even(bc);
    double* C = ctx->dbuf("mm.c", M * ldc);
    gemm_dev(ctx, static_cast<int>(M), static_cast<int>(bc), static_cast<int>(K), A.p, A.ld, trans_a != 0, B.p, B.ld,
             false, C, ldc, 1.0, 0.0);
    download(ctx, out, C, ldc, M, bc);
  });
}

int rbpg_pack_lower_device(rbpg_context* ctx, const double* dg, size_t ldg, size_t n, double* dpacked,
                           rbpg_status* st) {
  return guarded(ctx, st, [&] {
    ctx->run("pack_lower", [&] {
      return launch_pack_lower(dg, static_cast<long long>(ldg), static_cast<int>(n), dpacked, ctx->stream);
    });
  });
}

int rbpg_unpack_lower_device(rbpg_context* ctx, const double* dpacked, size_t n, double* dg, size_t ldg,
                             rbpg_status* st) {
  return guarded(ctx, st, [&] {
    ctx->run("unpack_lower", [&] {
      return launch_unpack_lower(dpacked, static_cast<int>(n), dg, static_cast<long long>(ldg), ctx->stream);
    });
  });
}

int rbpg_sum_parts_device(rbpg_context* ctx, const double* dparts, size_t stride, size_t nparts, size_t count,
                          double* dout, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (nparts == 0) fail(RBPG_INVALID_ARGUMENT, "sum_parts: no parts");
    ctx->run("sum_parts", [&] {
      return launch_sum_parts(dparts, static_cast<long long>(stride), static_cast<int>(nparts),
                              static_cast<long long>(count), dout, ctx->stream);
    });
  });
}

int rbpg_gram_stage_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                           size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw, const double* db,
                           double* dg, size_t ldg, double* dhtt, size_t ldt, int accumulate, int keep_h,
                           rbpg_status* st) {
  return guarded(ctx, st, [&] {
    Padded X = pad_device(ctx, "X.pad", dx, ldx, n, d);
    Padded T = pad_device(ctx, "T.pad", dt, ldt_in, n, m);
    Padded W = pad_device(ctx, "W.pad", dw, ldw, d, l);
    const size_t lda = round_up(l + m, 8);
    double* ga = ctx->dbuf("Gaug", (l + m) * lda);
    gram_stage(ctx, X.p, X.ld, T.p, T.ld, n, d, l, m, W.p, W.ld, db, ga, lda, false, keep_h != 0, false);
    if (accumulate) {  // add this block's partial sums to the caller's
      ctx->run("add_block", [&] { return launch_add_block(dg, ldg, ga, lda, l, l, ctx->stream); });
      if (m) ctx->run("add_block", [&] { return launch_add_block(dhtt, ldt, ga + l, lda, l, m, ctx->stream); });
    } else {
      ck(cudaMemcpy2DAsync(dg, ldg * 8, ga, lda * 8, l * 8, l, cudaMemcpyDeviceToDevice, ctx->stream), "store G");
      if (m)
        ck(cudaMemcpy2DAsync(dhtt, ldt * 8, ga + l, lda * 8, m * 8, l, cudaMemcpyDeviceToDevice, ctx->stream),
           "store HtT");
    }
  });
}

int rbpg_gram_stage_device_aug(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                               size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw, const double* db,
                               double* dgaug, size_t ldga, int accumulate, int keep_h, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    if (ldga < l + m) fail(RBPG_SHAPE_ERROR, "gram_stage_device_aug: leading dimension below l + m");
    Padded X = pad_device(ctx, "X.pad", dx, ldx, n, d);
    Padded T = pad_device(ctx, "T.pad", dt, ldt_in, n, m);
    Padded W = pad_device(ctx, "W.pad", dw, ldw, d, l);
    // the Gram kernels store 16-byte vectors: an odd leading dimension (or unaligned base) goes
    // through an aligned staging buffer
    if (ldga % 2 == 0 && (reinterpret_cast<uintptr_t>(dgaug) & 15) == 0) {
      gram_stage(ctx, X.p, X.ld, T.p, T.ld, n, d, l, m, W.p, W.ld, db, dgaug, ldga, accumulate != 0, keep_h != 0,
                 false);
      return;
    }
    const size_t M = l + m, lds = round_up(M, 8);
    double* S = ctx->dbuf("Gaug.stage", M * lds);
    if (accumulate)
      ck(cudaMemcpy2DAsync(S, lds * 8, dgaug, ldga * 8, M * 8, M, cudaMemcpyDeviceToDevice, ctx->stream), "stage G");
    gram_stage(ctx, X.p, X.ld, T.p, T.ld, n, d, l, m, W.p, W.ld, db, S, lds, accumulate != 0, keep_h != 0, false);
    ck(cudaMemcpy2DAsync(dgaug, ldga * 8, S, lds * 8, M * 8, M, cudaMemcpyDeviceToDevice, ctx->stream), "store G");
  });
}

int rbpg_solve_stage_device_aug(rbpg_context* ctx, const double* dgaug, size_t ldga, size_t l, size_t m,
                                size_t n_total, const rbpg_strategy* strategy, double* dbeta, size_t ldb,
                                size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    if (ldga < l + m) fail(RBPG_SHAPE_ERROR, "solve_stage_device_aug: leading dimension below l + m");
    solve_dev(ctx, dgaug, ldga, dgaug + l, ldga, l, m, n_total, *strategy, dbeta, ldb, order_out, diag, true);
    check_finite(ctx, dbeta, ldb, l, m);
  });
}

int rbpg_solve_stage_device(rbpg_context* ctx, const double* dg, size_t ldg, const double* dhtt, size_t ldt,
                            size_t l, size_t m, size_t n_total, const rbpg_strategy* strategy, double* dbeta,
                            size_t ldb, size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    solve_dev(ctx, dg, ldg, dhtt, ldt, l, m, n_total, *strategy, dbeta, ldb, order_out, diag);
    check_finite(ctx, dbeta, ldb, l, m);
  });
}

int rbpg_accuracy_stage_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in,
                               size_t n, size_t d, size_t l, size_t m, const double* dw, size_t ldw,
                               const double* db, const double* dbeta, size_t ldb, uint64_t* hits, rbpg_status* st) {
  return guarded(ctx, st, [&] {
    Padded X = pad_device(ctx, "X.pad", dx, ldx, n, d);
    Padded T = pad_device(ctx, "T.pad", dt, ldt_in, n, m);
    Padded W = pad_device(ctx, "W.pad", dw, ldw, d, l);
    *hits = accuracy_stage(ctx, X.p, X.ld, T.p, T.ld, n, d, l, m, W.p, W.ld, db, dbeta, ldb);
  });
}

int rbpg_train_device(rbpg_context* ctx, const double* dx, size_t ldx, const double* dt, size_t ldt_in, size_t n,
                      size_t d, size_t l, size_t m, const double* w, const double* b, const rbpg_strategy* strategy,
                      double* dbeta, size_t ldb, size_t* order_out, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(ctx, st, [&] {
    if (strategy->kind != RBPG_DIRECT && n < l)
      fail(RBPG_INVALID_ARGUMENT, "train: block strategies need at least as many samples as hidden nodes (" +
                                      std::to_string(n) + " < " + std::to_string(l) + "); use the direct strategy");
    train_core(ctx, dx, ldx, dt, ldt_in, n, d, l, m, w, b, *strategy, dbeta, ldb, order_out, diag);
  });
}

// ============================================================================
// Single-process multi-device train() (SURVEY §8(b) "the multi-GPU variant takes a device count",
// §8(e)): contiguous row shards, per-device augmented Gram, ONE NCCL all-reduce of its packed lower
// triangle, replicated solve.  NCCL is resolved at run time (dlopen of libnccl.so.2: the same library
// object torch may already have loaded), so the C ABI has no link-time NCCL dependency.
// ============================================================================
}  // extern "C"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.ErrorString = reinterpret_cast<decltype(api.ErrorString)>(sym("ncclGetErrorString"));
    if (api.CommInitAll && api.AllReduce && api.AllGather && api.GroupStart && api.GroupEnd && api.ErrorString)
      api.h = h;
  });
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(RBPG_CUDA_ERROR, std::string(what) + ": " + nccl().ErrorString(r));
}

// one communicator clique per device list, created once per process
const std::vector<ncclComm_t>& comms_for(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return it->second;
  std::vector<ncclComm_t> c(devs.size());
  nck(nccl().CommInitAll(c.data(), static_cast<int>(devs.size()), devs.data()), "ncclCommInitAll");
  return cache.emplace(devs, std::move(c)).first->second;
}

// run fn(i) for every device on its own host thread; the first failure is rethrown
void per_device(size_t ndev, const std::function<void(size_t)>& fn) {
  std::vector<Fail> fails(ndev);
  std::vector<char> failed(ndev, 0);
  std::vector<std::thread> th;
  for (size_t i = 0; i < ndev; ++i)
    th.emplace_back([&, i] {
      try {
        fn(i);
      } catch (const Fail& e) {
        fails[i] = e;
        failed[i] = 1;
      } catch (const std::exception& e) {
        fails[i] = Fail{RBPG_RUNTIME_ERROR, e.what()};
        failed[i] = 1;
      }
    });
  for (auto& t : th) t.join();
  for (size_t i = 0; i < ndev; ++i)
    if (failed[i]) throw fails[i];
}

}  // namespace

extern "C" {

int rbpg_train_multi(rbpg_context* const* ctxs, size_t ndev, size_t inputs, size_t hidden, size_t outputs,
                     uint64_t seed, const double* x, size_t n, size_t xcols, const double* y, size_t yrows,
                     size_t ycols, const rbpg_strategy* strategy, int fixed_order, double* w, double* b,
                     double* beta, size_t* order, rbpg_diagnostics* diag, rbpg_status* st) {
  rbpg_diagnostics local;
  if (!diag) diag = &local;
  zero_diag(diag);
  return guarded(nullptr, st, [&] {
    if (ndev == 0 || !ctxs) fail(RBPG_INVALID_ARGUMENT, "train_multi: no device contexts");
    std::vector<int> devs(ndev);
    for (size_t i = 0; i < ndev; ++i) {
      if (!ctxs[i]) fail(RBPG_INVALID_ARGUMENT, "train_multi: null context");
      devs[i] = ctxs[i]->device;
      for (size_t j = 0; j < i; ++j)
        if (devs[j] == devs[i]) fail(RBPG_INVALID_ARGUMENT, "train_multi: one context per device (NCCL ranks)");
    }
    // validation order of elm.cpp:234-258
    if (n != yrows) fail(RBPG_SHAPE_ERROR, "train: X is " + shp(n, xcols) + " but Y is " + shp(yrows, ycols));
    if (xcols != inputs)
      fail(RBPG_SHAPE_ERROR, "train: X has " + std::to_string(xcols) + " features but params.inputs is " +
                                 std::to_string(inputs));
    if (ycols != outputs)
      fail(RBPG_SHAPE_ERROR, "train: Y has " + std::to_string(ycols) + " columns but params.outputs is " +
                                 std::to_string(outputs));
    if (strategy->kind != RBPG_DIRECT && n < hidden)
      fail(RBPG_INVALID_ARGUMENT, "train: block strategies need at least as many samples as hidden nodes (" +
                                      std::to_string(n) + " < " + std::to_string(hidden) + "); use the direct strategy");
    if (strategy->kind == RBPG_DF_SPLIT && (strategy->split_index < 1 || strategy->split_index >= hidden))
      fail(RBPG_INVALID_ARGUMENT, "train: df split index must be in (0, " + std::to_string(hidden) + "), got " +
                                      std::to_string(strategy->split_index));
    if (ndev > 1 && !nccl().h) fail(RBPG_NOT_SUPPORTED, "train_multi: libnccl.so.2 not found");
    rbpg_status s2;
    if (rbpg_init_hidden(inputs, hidden, outputs, seed, w, b, &s2)) fail(s2.code, s2.message);
    const size_t L = hidden, m = outputs, d = inputs, M = L + m, ldga = round_up(M, 8);
    const size_t count = M * (M + 1) / 2;
    const size_t ldx = even(d), ldy = even(m), ldw = even(L), lb = even(m);
    std::vector<size_t> row0(ndev), rows(ndev);
    for (size_t i = 0, r = 0; i < ndev; ++i) {  // sharded.shard_rows: the first n % ndev shards get one more row
      rows[i] = n / ndev + (i < n % ndev ? 1 : 0);
      row0[i] = r;
      r += rows[i];
    }
    std::vector<double*> G(ndev), packed(ndev), parts(ndev), B(ndev);
    std::vector<const double*> X(ndev), T(ndev), W(ndev), bb(ndev);
    const auto t0 = std::chrono::steady_clock::now();
    // phase 1: every device uploads its rows and builds its augmented Gram, packed
    per_device(ndev, [&](size_t i) {
      rbpg_context* c = ctxs[i];
      std::lock_guard<std::mutex> lk(c->mu);
      ck(cudaSetDevice(c->device), "cudaSetDevice");
      double* dx = c->dbuf("multi.X", std::max<size_t>(1, rows[i]) * ldx);
      double* dy = c->dbuf("multi.T", std::max<size_t>(1, rows[i]) * ldy);
      double* dw = c->dbuf("multi.W", std::max<size_t>(1, d) * ldw);
      double* db = c->dbuf("multi.b", L);
      copy_rows(dx, ldx * 8, x + row0[i] * xcols, xcols * 8, xcols * 8, rows[i], cudaMemcpyHostToDevice, c->stream,
                "upload X");
      copy_rows(dy, ldy * 8, y + row0[i] * ycols, ycols * 8, ycols * 8, rows[i], cudaMemcpyHostToDevice, c->stream,
                "upload Y");
      copy_rows(dw, ldw * 8, w, L * 8, L * 8, d, cudaMemcpyHostToDevice, c->stream, "upload W");
      ck(cudaMemcpyAsync(db, b, L * 8, cudaMemcpyHostToDevice, c->stream), "upload b");
      X[i] = dx;
      T[i] = dy;
      W[i] = dw;
      bb[i] = db;
      G[i] = c->dbuf("multi.G", M * ldga);
      gram_stage(c, dx, ldx, dy, ldy, rows[i], d, L, m, dw, ldw, db, G[i], ldga, false, true, false);
      packed[i] = c->dbuf("multi.packed", count);
      if (fixed_order) parts[i] = c->dbuf("multi.parts", count * ndev);
      c->run("pack_lower", [&] { return launch_pack_lower(G[i], static_cast<long long>(ldga), static_cast<int>(M),
                                                          packed[i], c->stream); });
      ck(cudaStreamSynchronize(c->stream), "gram sync");
    });
    const auto t1 = std::chrono::steady_clock::now();
    // phase 2: the one exchange step
    if (ndev > 1) {
      const std::vector<ncclComm_t>& comms = comms_for(devs);
      nck(nccl().GroupStart(), "ncclGroupStart");
      for (size_t i = 0; i < ndev; ++i) {
        ck(cudaSetDevice(devs[i]), "cudaSetDevice");
        if (fixed_order)
          nck(nccl().AllGather(packed[i], parts[i], count, ncclDouble, comms[i], ctxs[i]->stream), "ncclAllGather");
        else
          nck(nccl().AllReduce(packed[i], packed[i], count, ncclDouble, ncclSum, comms[i], ctxs[i]->stream),
              "ncclAllReduce");
      }
      nck(nccl().GroupEnd(), "ncclGroupEnd");
    }
    // phase 3: replicated solve and the local hit counts
    std::vector<unsigned long long> hits(ndev, 0);
    std::vector<rbpg_diagnostics> dg(ndev);
    std::vector<std::vector<size_t>> ord(ndev, std::vector<size_t>(L));
    per_device(ndev, [&](size_t i) {
      rbpg_context* c = ctxs[i];
      std::lock_guard<std::mutex> lk(c->mu);
      ck(cudaSetDevice(c->device), "cudaSetDevice");
      if (ndev > 1 && fixed_order)
        c->run("sum_parts", [&] { return launch_sum_parts(parts[i], static_cast<long long>(count),
                                                          static_cast<int>(ndev), static_cast<long long>(count),
                                                          packed[i], c->stream); });
      c->run("unpack_lower", [&] { return launch_unpack_lower(packed[i], static_cast<int>(M), G[i],
                                                              static_cast<long long>(ldga), c->stream); });
      B[i] = c->dbuf("multi.beta", L * lb);
      zero_diag(&dg[i]);
      // the SVD branch of solve_direct needs all of H on one device: only with one device
      SourceScope src(c, ndev == 1 && c->kept_h ? c->kept_h : nullptr, c->kept_ldh,
                      ndev == 1 && c->kept_h ? c->kept_h + L : nullptr, c->kept_ldh, ndev == 1 ? n : 0);
      solve_dev(c, G[i], ldga, G[i] + L, ldga, L, m, n, *strategy, B[i], lb, ord[i].data(), &dg[i], true);
      check_finite(c, B[i], lb, L, m);
      hits[i] = accuracy_stage(c, X[i], ldx, T[i], ldy, rows[i], d, L, m, W[i], ldw, bb[i], B[i], lb);
    });
    const auto t2 = std::chrono::steady_clock::now();
    {
      rbpg_context* c = ctxs[0];
      std::lock_guard<std::mutex> lk(c->mu);
      ck(cudaSetDevice(c->device), "cudaSetDevice");
      download(c, beta, B[0], lb, L, m);
    }
    if (order) std::copy(ord[0].begin(), ord[0].end(), order);
    unsigned long long tot = 0;
    for (auto h : hits) tot += h;
    *diag = dg[0];
    diag->training_accuracy = n ? static_cast<double>(tot) / static_cast<double>(n) : 0.0;
    diag->hidden_seconds = std::chrono::duration<double>(t1 - t0).count();  // upload + H build + Gram
    diag->solve_seconds = std::chrono::duration<double>(t2 - t1).count();   // exchange + solve + accuracy
  });
}

}  // extern "C"
