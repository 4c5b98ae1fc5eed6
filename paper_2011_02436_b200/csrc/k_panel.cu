// K3: one panel (<= 64 columns) of the diagonal-pivoted blocked Cholesky of the Gram
// matrix -- reference linalg.cpp:197-236: pivot = first maximum of the running diagonal d
// over positions >= j (strict '>', :207-210), swaps (:211-218), stop rule rjj <= cut
// (:219-223), column update col = (G[:,j] - F[:,k:j] F[j,k:j]^T) / rjj and d -= col^2
// (:225-235).  With pivoting = 0 the same kernel is the unpivoted SpdFactor panel with the
// reference's singular-pivot rule (linalg.cpp:116-129).
//
// Labels instead of swaps: every CTA owns a contiguous range of labels (a label is the
// column's position at panel start) and keeps, in shared memory, its labels' running
// diagonal and panel columns (stored transposed, PsT[c][label]).  Positions are tracked by
// two replicated maps (lab_at, pos_of) that every CTA updates identically, so a swap is O(1).
// The arg-max key is (d, -position): an order-preserving 64-bit image of d reduced with three
// warp REDUX ops (max hi word, max lo word, min position), which is exactly the reference's
// first-maximum scan.
//
// Latency structure of one column step (the loop is strictly sequential over L columns):
//   exchange -> every warp reads all CTAs' candidates and resolves the winner itself
//   fetch    -> every warp loads the pivot's panel row and the G entries of its own labels
//   update   -> quad (4 lanes) per label, fused local arg-max, ONE __syncthreads, warp 0
//               combines the 8 warp candidates, applies the swap, publishes.
// Exchange variants:
//   * cluster (nl <= 16 * 256): the panel runs in ONE thread-block cluster; candidates sit in
//     each CTA's shared memory, one barrier.cluster per column, the pivot's panel row is read
//     from its owner through distributed shared memory;
//   * grid (larger panels): cooperative grid, candidates in global slots with release/acquire
//     epochs, the panel row mirrored to global memory.
#include "common.cuh"
#include "kernels.cuh"

#include <cooperative_groups.h>
#include <cfloat>
#include <climits>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace rbpg {

constexpr int kPanelW = 64;
constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kMaxCluster = 16;
constexpr int kMaxLabelsPerCta = 256;

// order-preserving image of a double (larger value <=> larger unsigned key)
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(u));
}

// warp arg-max: largest key, ties -> smallest position.  All lanes get the result.
__device__ __forceinline__ void warp_argmax(unsigned long long& key, int& pos) {
  const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(key >> 32));
  const unsigned lo =
      __reduce_max_sync(0xffffffffu, static_cast<unsigned>(key >> 32) == hi ? static_cast<unsigned>(key) : 0u);
  const unsigned long long best = (static_cast<unsigned long long>(hi) << 32) | lo;
  pos = static_cast<int>(__reduce_min_sync(0xffffffffu, key == best ? static_cast<unsigned>(pos) : 0x7fffffffu));
  key = best;
}

__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

struct __align__(16) Cand {
  unsigned long long key;
  int pos;
  int pad;
};

template <bool kCluster>
__global__ void __launch_bounds__(kPThreads, 1) panel_kernel_t(PanelParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = p.n, k = p.k, kb = p.kb, nl = n - k;
  const int R = p.rows_per_cta;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  int C, cta;
  if constexpr (kCluster) {
    cg::cluster_group cl = cg::this_cluster();
    C = static_cast<int>(cl.num_blocks());
    cta = static_cast<int>(cl.block_rank());
  } else {
    C = gridDim.x;
    cta = blockIdx.x;
  }

  double* PsT = reinterpret_cast<double*>(smem_raw);  // [64][R]
  double* dl = PsT + kPanelW * R;                      // [R]
  int* lab_at = reinterpret_cast<int*>(dl + R);       // [nl]  position-k -> label
  int* pos_of = lab_at + nl;                          // [nl]  label-k -> position
  // cluster: every CTA's candidate and its panel row, pushed by the owner before the barrier
  __shared__ Cand cand_all[2][kMaxCluster];
  __shared__ __align__(16) double rows_all[2][kMaxCluster][kPanelW];
  __shared__ __align__(8) uint64_t cand_full[2];  // tx-count barriers of the two candidate buffers
  __shared__ Cand wbest[kPWarps];
  __shared__ int s_stop;

  FactorState* st = p.st;
  if (st->stopped) {  // an earlier panel ended the factorisation: carry the order through
    if (cta == 0)
      for (int i = tid; i < n; i += blockDim.x) p.ord_out[i] = p.ord_in[i];
    return;
  }
  const int lbeg = k + cta * R;
  const int lend = min(n, lbeg + R);
  const int nown = max(0, lend - lbeg);

  for (int i = tid; i < nl; i += blockDim.x) {
    lab_at[i] = k + i;
    pos_of[i] = k + i;
  }
  for (int i = tid; i < kPanelW * R; i += blockDim.x) PsT[i] = 0.0;
  for (int i = tid; i < R; i += blockDim.x) dl[i] = (i < nown) ? p.d_in[lbeg + i] : -DBL_MAX;
  if (tid == 0) s_stop = 0;
  if constexpr (kCluster) {
    if (tid == 0) {
      mbar_init(&cand_full[0], 1);
      mbar_init(&cand_full[1], 1);
      fence_mbar_init();
    }
    cg::this_cluster().sync();  // every CTA's barriers exist before any remote st.async
  }
  __syncthreads();
  // bytes one step's exchange delivers into each CTA: C candidates + C panel rows
  const uint32_t kStepBytes = static_cast<uint32_t>(C) * (sizeof(Cand) + kPanelW * sizeof(double));
  const double cut = st->cut;
  const double thresh = st->thresh;

  // Combine the per-warp candidates and publish this CTA's candidate for step j.  (piv, y)
  // describe the swap of the step just finished, still pending in the maps (tid 0 applies it).
  // Cluster: every warp combines redundantly and pushes to destinations d = warp (mod 8):
  // (key, pos) and the candidate's panel row (columns 0..j-k-1) by st.async, which completes
  // on the receiver's mbarrier.  Grid: warp 0 writes the global slot with a release epoch.
  auto combine_publish = [&](int j, int piv, int y) {
    unsigned long long key = 0;
    int pos = INT_MAX;
    if (lane < kPWarps) {
      key = wbest[lane].key;
      pos = wbest[lane].pos;
    }
    warp_argmax(key, pos);
    if constexpr (kCluster) {
      const int cvalid = j - k;  // panel columns already computed
      double2 rv = make_double2(0.0, 0.0);
      if (pos != INT_MAX) {
        const int lab = (pos == piv) ? y : lab_at[pos - k];
        const int lib = lab - lbeg;
        if (2 * lane < cvalid) rv.x = PsT[(2 * lane) * R + lib];
        if (2 * lane + 1 < cvalid) rv.y = PsT[(2 * lane + 1) * R + lib];
      }
      const int par = (j - k) & 1;
      const uint32_t row_l = smem_u32(&rows_all[par][cta][2 * lane]);
      const uint32_t cand_l = smem_u32(&cand_all[par][cta]);
      const uint32_t bar_l = smem_u32(&cand_full[par]);
      for (int d = warp; d < C; d += kPWarps) {
        const uint32_t rbar = mapa_u32(bar_l, d);
        st_async_v2f64(mapa_u32(row_l, d), rv.x, rv.y, rbar);
        if (lane == 0) st_async_v2b64(mapa_u32(cand_l, d), key, static_cast<unsigned long long>(pos), rbar);
      }
    } else if (warp == 0 && lane == 0) {
      PivotSlot* sl = p.slots + (j & 1) * C + cta;
      *reinterpret_cast<unsigned long long*>(&sl->val) = key;
      sl->pos = pos;
      st_release_u32(&sl->epoch, static_cast<unsigned int>(j + 1));
    }
  };

  // ---- initial candidates for step k
  {
    unsigned long long key = 0;
    int pos = INT_MAX;
    if (p.pivoting) {
      for (int i = tid; i < nown && lbeg + i < p.neligible; i += kPThreads) {
        const unsigned long long kk = dkey(dl[i]);
        if (kk > key || (kk == key && lbeg + i < pos)) {
          key = kk;
          pos = lbeg + i;
        }
      }
    } else if (k >= lbeg && k < lend && tid == 0) {
      key = dkey(dl[k - lbeg]);
      pos = k;
    }
    warp_argmax(key, pos);
    if (lane == 0) {
      wbest[warp].key = key;
      wbest[warp].pos = pos;
    }
    __syncthreads();
    combine_publish(k, -1, -1);
  }

  unsigned long long* trace = p.trace;
  long long tacc[6] = {0, 0, 0, 0, 0, 0};
  __shared__ unsigned long long s_wkey;
  __shared__ int s_piv, s_xp, s_y, s_src;
  __shared__ double prow_g[kPanelW];  // grid variant: pivot panel row staged from global
  // sqrt(d) <= cut  <=>  d <= cut^2 up to rounding: values above cut^2 (1 + 2^-30) never stop
  const double cut_sq_hi = cut * cut * (1.0 + 0x1.0p-30);
  for (int c = 0; c < kb; ++c) {
    const int j = k + c;
    long long t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0;
    if (trace) t0 = clock64();
    // ---------------- exchange: warp 0 resolves the winner
    if constexpr (kCluster) {
      if (warp == 0) {
        // arm this step's buffer (remote bytes may already have landed: the tx-count may be
        // transiently negative within the phase), then wait for all C candidates + rows
        if (lane == 0) mbar_arrive_expect_tx(&cand_full[c & 1], kStepBytes);
        mbar_wait(&cand_full[c & 1], (c >> 1) & 1);
      }
    }
    if (trace) t1 = clock64();
    if (warp == 0) {
      unsigned long long wkey = 0;
      int wpos = INT_MAX;
      unsigned long long ck = 0;
      int cp = INT_MAX;
      if constexpr (kCluster) {
        if (lane < C) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&cand_all[c & 1][lane]);
          ck = v.x;
          cp = static_cast<int>(v.y & 0xffffffffull);
        }
        wkey = ck;
        wpos = cp;
      } else {
        const PivotSlot* base = p.slots + (j & 1) * C;
        for (int i = lane; i < C; i += 32) {
          while (ld_acquire_u32(&base[i].epoch) != static_cast<unsigned int>(j + 1)) {
          }
          const unsigned long long kk = __ldcg(reinterpret_cast<const unsigned long long*>(&base[i].val));
          const int ps = __ldcg(&base[i].pos);
          if (kk > wkey || (kk == wkey && ps < wpos)) {
            wkey = kk;
            wpos = ps;
          }
        }
      }
      warp_argmax(wkey, wpos);
      const int xpw = lab_at[wpos - k];
      int src = 0;
      if constexpr (kCluster) {
        const unsigned msk = __ballot_sync(0xffffffffu, lane < C && ck == wkey && cp == wpos);
        src = __ffs(msk) - 1;
      } else {
        const double* rp = p.Pg + (long long)(xpw - k) * kPanelW;
        prow_g[lane] = lane < c ? __ldcg(rp + lane) : 0.0;
        prow_g[lane + 32] = lane + 32 < c ? __ldcg(rp + lane + 32) : 0.0;
      }
      if (lane == 0) {
        s_wkey = wkey;
        s_piv = wpos;
        s_xp = xpw;
        s_y = lab_at[j - k];
        s_src = src;
      }
      named_bar_arrive(1, kPThreads);  // winner known to the CTA
    } else {
      named_bar_sync(1, kPThreads);
    }
    const int piv = s_piv, xp = s_xp, y = s_y;
    const double dj = dkey_inv(s_wkey);
    const double* prow;
    if constexpr (kCluster) {
      prow = rows_all[c & 1][s_src];
    } else {
      prow = prow_g;
    }
    // this warp's first-pass G entries, issued before the FP64 math
    // G through its lower triangle (the trailing updates write only that half)
    auto gat = [&](int xl) { return p.G[(long long)max(xp, xl) * p.ldg + min(xp, xl)]; };
    double gpre = 0.0;
    {
      const int li0 = warp * 8 + (lane >> 2);
      if ((lane & 3) == 0 && li0 < nown) gpre = gat(lbeg + li0);
    }
    bool stop;
    if (p.pivoting) {
      stop = !(dj > cut_sq_hi) && (dj > 0.0 ? sqrt(dj) : 0.0) <= cut;  // linalg.cpp:219-223
    } else {
      stop = !isfinite(dj) || dj <= thresh || dj <= 0.0;               // linalg.cpp:118-119
    }
    if (stop) {
      __syncthreads();  // every warp has read the maps for this step
      if (tid == 0) {
        // the swap at step j happens before the stop test in the reference
        if (piv != j) {
          lab_at[j - k] = xp;
          lab_at[piv - k] = y;
          pos_of[xp - k] = j;
          pos_of[y - k] = piv;
        }
        s_stop = p.pivoting ? 1 : 2;
        if (cta == 0) {
          st->stopped = 1;
          st->rank = j;
          if (!p.pivoting) {
            st->fail = 1;
            st->fail_index = j;
            st->fail_value = dj;
          }
        }
      }
      __syncthreads();
      break;
    }
    const double rjj = sqrt(dj);
    const double inv_rjj = 1.0 / rjj;
    if (tid == 0 && (xp - k) / R == cta) {
      const int oli = (xp - k) % R;
      PsT[c * R + oli] = rjj;  // F(j, j) = rjj
      if constexpr (!kCluster) p.Pg[(long long)(xp - k) * kPanelW + c] = rjj;
    }
    if (trace) t2 = clock64();

    // ---------------- update: quad (4 lanes) per label; warp w owns labels w*8 + 64*pass + lane/4
    unsigned long long bkey = 0;
    int bpos = INT_MAX;
    for (int base = warp * 8; base < nown; base += kPThreads / 4) {
      const int li = base + (lane >> 2);
      const int q = lane & 3;
      const int x = lbeg + li;
      // position after this step's swap, without touching the shared maps
      int pos = -1;
      if (li < nown) pos = (x == y) ? piv : (x == xp ? j : pos_of[x - k]);
      const bool alive = pos > j;
      const double gv = (alive && q == 0) ? (base == warp * 8 ? gpre : gat(x)) : 0.0;
      double s = 0.0;
      if (alive) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int cc = q;
        for (; cc + 12 < c; cc += 16) {
          a0 = fma(PsT[cc * R + li], prow[cc], a0);
          a1 = fma(PsT[(cc + 4) * R + li], prow[cc + 4], a1);
          a2 = fma(PsT[(cc + 8) * R + li], prow[cc + 8], a2);
          a3 = fma(PsT[(cc + 12) * R + li], prow[cc + 12], a3);
        }
        for (; cc < c; cc += 4) a0 = fma(PsT[cc * R + li], prow[cc], a0);
        s = (a0 + a1) + (a2 + a3);
      }
      const double s1 = __shfl_down_sync(0xffffffffu, s, 1, 4);
      const double s2 = __shfl_down_sync(0xffffffffu, s, 2, 4);
      const double s3 = __shfl_down_sync(0xffffffffu, s, 3, 4);
      if (alive && q == 0) {
        const double tot = (s + s1) + (s2 + s3);
        const double col = (gv - tot) * inv_rjj;
        PsT[c * R + li] = col;
        if constexpr (!kCluster) p.Pg[(long long)(x - k) * kPanelW + c] = col;
        const double dn = fma(-col, col, dl[li]);
        dl[li] = dn;
        const unsigned long long kk = dkey(dn);
        if (p.pivoting) {
          if (x < p.neligible && (kk > bkey || (kk == bkey && pos < bpos))) {
            bkey = kk;
            bpos = pos;
          }
        } else if (pos == j + 1) {
          bkey = kk;
          bpos = pos;
        }
      }
    }
    if (trace) t3 = clock64();
    warp_argmax(bkey, bpos);
    if (lane == 0) {
      wbest[warp].key = bkey;
      wbest[warp].pos = bpos;
    }
    __syncthreads();
    if (trace) t4 = clock64();
    if (c + 1 < kb) combine_publish(j + 1, piv, y);
    if (tid == 0 && piv != j) {  // apply the swap (linalg.cpp:211-218) to the replicated maps
      lab_at[j - k] = xp;
      lab_at[piv - k] = y;
      pos_of[xp - k] = j;
      pos_of[y - k] = piv;
    }
    __syncwarp();
    if (trace) {
      const long long t5 = clock64();
      tacc[0] += t1 - t0;
      tacc[1] += t2 - t1;
      tacc[2] += t3 - t2;
      tacc[3] += t4 - t3;
      tacc[4] += t5 - t4;
      tacc[5] += 1;
    }
  }
  __syncthreads();
  if (trace && cta == 0 && tid == 0)
    for (int i = 0; i < 6; ++i) atomicAdd(&trace[i], static_cast<unsigned long long>(tacc[i]));
  if constexpr (kCluster) cg::this_cluster().sync();  // no CTA leaves while its smem may be read
  __syncthreads();

  // ---- write back: factor rows by original column, compacted trailing panel, d, order
  for (int e = tid; e < nown * kPanelW; e += blockDim.x) {
    const int li = e / kPanelW, cc = e % kPanelW;
    if (cc >= kb) continue;
    const int x = lbeg + li;
    p.Fo[(long long)p.ord_in[x] * p.ldf + k + cc] = PsT[cc * R + li];
  }
  if (!s_stop) {
    const int t0 = k + kb;
    for (int e = tid; e < nown * kPanelW; e += blockDim.x) {
      const int li = e / kPanelW, cc = e % kPanelW;
      if (cc >= kb) continue;
      const int pos = pos_of[lbeg + li - k];
      if (pos >= t0) p.PcT[(long long)cc * p.ldp + (pos - t0)] = PsT[cc * R + li];
    }
    for (int li = tid; li < nown; li += blockDim.x) {
      const int pos = pos_of[lbeg + li - k];
      if (pos >= t0) p.d_out[pos] = dl[li];
    }
  }
  for (int pos = cta * blockDim.x + tid; pos < n; pos += C * blockDim.x) {
    if (pos < k) {
      p.ord_out[pos] = p.ord_in[pos];
    } else {
      const int lb = lab_at[pos - k];
      p.ord_out[pos] = p.ord_in[lb];
      p.lab_out[pos] = lb;
    }
  }
}

// ---------------------------------------------------------------------------
// Quad-per-label cluster variant (nl <= 16 * 64 * LPQ): one label per quad (4 lanes) and layer; lane
// q of the quad owns its label's panel columns q, q+4, ..., kept in the CTA's shared memory in the
// padded "lane-major" order (row[q*kRQ + i] = P[label][q + 4i]) in which candidate rows also travel
// and are consumed.  The owner lane stores each new column with one 8-byte store (a register copy
// would need a select over all slots, the slot being a run-time value), the label's row is re-read
// (issued before the exchange wait) for the dot product, and the CTA's candidate row is pushed
// straight from this array.
// Arithmetic is identical in the 4 lanes of a quad (xor-shuffle sums), so every lane holds the
// same col and d; the reduction order is fixed and label-independent (exact twin ties persist).
// Template: LPQ labels per quad, NT threads, PW panel width (64; 32 for the wide panels of more
// than 4096 labels, whose rows would not fit in shared memory at 64), MapT the type of the
// replicated position maps (short when n < 32768 keeps 8192 labels' maps within shared memory).
// ---------------------------------------------------------------------------
template <int NT, int PW>
struct RegPanel {
  static constexpr int kWarps = NT / 32;
  static constexpr int kQuads = NT / 4;          // labels per layer (one per quad)
  static constexpr int kQ = PW / 4;              // panel columns per lane and label
  static constexpr int kRQ = kQ + 2;             // padded quarter of a lane-major row
  static constexpr int kRL = 4 * kRQ;            // padded row
  static constexpr int kCPQ = kQ / 2;            // 16-byte chunks per quarter
  static constexpr size_t kLayerBytes = size_t(kQuads) * kRL * sizeof(double);
};

// kTrace: per-phase cycle counters (RBPG_PANEL_TRACE), compiled out of the production variant
template <bool kTrace, int LPQ, int NT = kPThreads, int PW = kPanelW, typename MapT = int>
__global__ void __launch_bounds__(NT, 1) panel_reg_kernel(PanelParams p) {
  using RP = RegPanel<NT, PW>;
  constexpr int kWarps = RP::kWarps, kQuads = RP::kQuads, kQ = RP::kQ, kRQ = RP::kRQ, kRL = RP::kRL;
  constexpr int kCPQ = RP::kCPQ;
  constexpr int kLabels = kQuads * LPQ;  // labels per CTA
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = p.n, k = p.k, kb = p.kb, nl = n - k;
  const int R = p.rows_per_cta;  // <= kLabels
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks()), cta = static_cast<int>(cl.block_rank());
  double (*qrow)[kRL] = reinterpret_cast<double (*)[kRL]>(smem_raw);       // [kLabels] own rows
  MapT* lab_at = reinterpret_cast<MapT*>(smem_raw + RP::kLayerBytes * LPQ);  // [nl]
  MapT* pos_of = lab_at + nl;                                                 // [nl]
  __shared__ Cand cand_all[2][kMaxCluster];
  // candidate rows, lane-major with a padded quarter stride (row[q*kRQ + i] = P[label][q + 4i]):
  // the 4 distinct quarters a warp reads per step land on different banks
  __shared__ __align__(16) double rows_all[2][kMaxCluster][kRL];
  __shared__ __align__(8) uint64_t cand_full[2];
  __shared__ Cand wbest[kWarps];
  __shared__ int s_stop;

  tl_mark(p.tl, p.tl_slot, 0);
  pdl_trigger();
  pdl_wait();  // the previous trailing update / panel may still be finishing
  tl_mark(p.tl, p.tl_slot, 1);
  FactorState* st = p.st;
  if (st->stopped) {
    if (cta == 0)
      for (int i = tid; i < n; i += blockDim.x) p.ord_out[i] = p.ord_in[i];
    tl_mark(p.tl, p.tl_slot, 2);
    return;
  }
  const int lbeg = k + cta * R;
  const int nown = max(0, min(n, lbeg + R) - lbeg);
  const int qi = tid >> 2, q = tid & 3;
  // quad qi holds labels lbeg + qi + kQuads * l (l < LPQ): consecutive quads, consecutive labels
  int x[LPQ];
  bool mine[LPQ];
  double* myrow[LPQ];  // this lane's kQ slots of each of its labels' rows
  double dl[LPQ];
#pragma unroll
  for (int l = 0; l < LPQ; ++l) {
    const int li = qi + kQuads * l;
    x[l] = lbeg + li;
    mine[l] = li < nown;
    myrow[l] = &qrow[li][q * kRQ];
    dl[l] = mine[l] ? p.d_in[x[l]] : -DBL_MAX;
  }

  for (int i = tid; i < nl; i += blockDim.x) {
    lab_at[i] = static_cast<MapT>(k + i);
    pos_of[i] = static_cast<MapT>(k + i);
  }
  if (tid == 0) {
    s_stop = 0;
    mbar_init(&cand_full[0], 1);
    mbar_init(&cand_full[1], 1);
    fence_mbar_init();
  }
  cl.sync();
  const double cut = st->cut;
  const double thresh = st->thresh;
  for (int i = tid; i < 2 * kMaxCluster * kRL; i += blockDim.x) (&rows_all[0][0][0])[i] = 0.0;
  for (int i = tid; i < kLabels * kRL; i += blockDim.x) (&qrow[0][0])[i] = 0.0;
  __syncthreads();

  // the CTA row index (label - lbeg) of this warp's best candidate (any valid row when none)
  // (myl: which of the lane's labels the lane's own candidate is)
  auto best_row = [&](unsigned long long key, int pos, int mypos, unsigned long long mykey, int myl) {
    const unsigned who = __ballot_sync(0xffffffffu, q == 0 && mykey == key && mypos == pos && pos != INT_MAX);
    if constexpr (LPQ == 1) {
      return who ? warp * 8 + ((__ffs(who) - 1) >> 2) : 0;
    } else {
      const int src = who ? __ffs(who) - 1 : 0;
      const int bl = __shfl_sync(0xffffffffu, myl, src);
      return who ? warp * 8 + (src >> 2) + kQuads * bl : 0;
    }
  };
  // the lane's best candidate over its LPQ labels: larger key, then smaller position
  auto lane_best = [](unsigned long long& key, int& pos, int& bl, unsigned long long kk, int pp, int l) {
    if (kk > key || (kk == key && pp < pos)) {
      key = kk;
      pos = pp;
      bl = l;
    }
  };
  // publish for step j: the CTA's candidate and its row's first nch slot chunks (the receiving
  // step reads no later chunk; columns beyond those are zero or not yet summed)
  auto combine_publish = [&](int j, int nch) {
    unsigned long long key = 0, k0 = 0;
    int pos = INT_MAX, p0 = INT_MAX;
    if (lane < kWarps) {
      k0 = key = wbest[lane].key;
      p0 = pos = wbest[lane].pos;
    }
    warp_argmax(key, pos);
    const int wsrc = __ffs(__ballot_sync(0xffffffffu, lane < kWarps && k0 == key && p0 == pos)) - 1;
    const int par = (j - k) & 1;
    // lane's 16-byte chunk of the padded row (4 quarters x kCPQ chunks; lanes beyond push nothing)
    const bool row_lane = lane < 4 * kCPQ;
    const int roff = row_lane ? (lane / kCPQ) * kRQ + 2 * (lane % kCPQ) : 0;
    const double2 rv = *reinterpret_cast<const double2*>(&qrow[wbest[wsrc].pad][roff]);
    const uint32_t row_l = smem_u32(&rows_all[par][cta][roff]);
    const uint32_t cand_l = smem_u32(&cand_all[par][cta]);
    const uint32_t bar_l = smem_u32(&cand_full[par]);
    const bool push_row = row_lane && ((lane % kCPQ) >> 1) < nch;
    for (int d = warp; d < C; d += kWarps) {
      const uint32_t rbar = mapa_u32(bar_l, d);
      if (push_row) st_async_v2f64(mapa_u32(row_l, d), rv.x, rv.y, rbar);
      if (lane == 0) st_async_v2b64(mapa_u32(cand_l, d), key, static_cast<unsigned long long>(pos), rbar);
    }
  };

  // ---- initial candidates (rows are still zero)
  {
    unsigned long long key = 0;
    int pos = INT_MAX, bl = 0;
#pragma unroll
    for (int l = 0; l < LPQ; ++l) {
      if (mine[l] && q == 0 && x[l] < p.neligible) {
        if (p.pivoting) {
          lane_best(key, pos, bl, dkey(dl[l]), x[l], l);
        } else if (x[l] == k) {
          lane_best(key, pos, bl, dkey(dl[l]), k, l);
        }
      }
    }
    const unsigned long long mk = key;
    const int mp = pos;
    warp_argmax(key, pos);
    const int brow = best_row(key, pos, mp, mk, bl);
    if (lane == 0) {
      wbest[warp].key = key;
      wbest[warp].pos = pos;
      wbest[warp].pad = brow;
    }
    __syncthreads();
    combine_publish(k, 0);
  }

  // kTrace: stamps T0..T9 per step (values forced in consumption order), deltas accumulated
  long long tacc[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long ts[11];
#define PANEL_TS(i) \
  do {              \
    if (kTrace) ts[i] = clock64(); \
  } while (0)
#define PANEL_FORCE(v)                                                           \
  do {                                                                           \
    if (kTrace && __double_as_longlong(double(v)) == 0x7ff0deadbeefll) p.trace[15] = 1; \
  } while (0)
  // Every warp resolves the winner itself from the exchanged candidates (no intra-CTA broadcast).
  // The position swap of step c is written by tid 0 after step c's barrier, so a warp reading the
  // maps during step c + 1 applies that last swap itself (pivp <-> jp, labels xpp / ypp).
  int pivp = -1, xpp = -1, ypp = -1;
  // Steps run in PW/16 groups of 16 (the outer loop is unrolled, so the group ch is a compile-time
  // constant): group ch writes only slot chunk ch of the rows, so the label's own row stays in
  // registers and only that chunk (plus, on entry, the previous one) is re-read per step.
  double2 own[LPQ][kQ / 2];
#pragma unroll
  for (int l = 0; l < LPQ; ++l)
#pragma unroll
    for (int i = 0; i < kQ / 2; ++i) own[l][i] = make_double2(0.0, 0.0);
#pragma unroll
  for (int ch = 0; ch < PW / 16; ++ch) {
#pragma unroll 1
  for (int u = 0; u < 16; ++u) {
    const int c = 16 * ch + u;
    if (c >= kb) goto panel_done;
    const int j = k + c;
    PANEL_TS(0);
    const int jp = j - 1;
    auto lab_eff = [&](int ps) { return ps == jp ? xpp : (ps == pivp ? ypp : static_cast<int>(lab_at[ps - k])); };
    auto pos_eff = [&](int lb) { return lb == xpp ? jp : (lb == ypp ? pivp : static_cast<int>(pos_of[lb - k])); };
    int mypos[LPQ];
#pragma unroll
    for (int l = 0; l < LPQ; ++l) mypos[l] = mine[l] ? pos_eff(x[l]) : -1;  // before the exchange wait
    const int y = lab_eff(j);
    // this label's row: the chunk written by this group (and the previous group's last column)
#pragma unroll
    for (int l = 0; l < LPQ; ++l) {
      own[l][2 * ch] = reinterpret_cast<const double2*>(myrow[l])[2 * ch];
      own[l][2 * ch + 1] = reinterpret_cast<const double2*>(myrow[l])[2 * ch + 1];
      if (ch > 0 && u == 0) {
        own[l][2 * ch - 1] = reinterpret_cast<const double2*>(myrow[l])[2 * ch - 1];
        own[l][2 * ch - 2] = reinterpret_cast<const double2*>(myrow[l])[2 * ch - 2];
      }
    }
    if (warp == 0 && lane == 0)
      mbar_arrive_expect_tx(&cand_full[c & 1],
                            static_cast<uint32_t>(C) * (sizeof(Cand) + (c == 0 ? 0u : 128u * (((c - 1) >> 4) + 1))));
    mbar_wait(&cand_full[c & 1], (c >> 1) & 1);
    PANEL_TS(1);
    unsigned long long ck = 0;
    int cp = INT_MAX;
    if (lane < C) {
      ck = cand_all[c & 1][lane].key;
      cp = cand_all[c & 1][lane].pos;
    }
    unsigned long long wkey = ck;
    int piv = cp;
    warp_argmax(wkey, piv);
    const int src = __ffs(__ballot_sync(0xffffffffu, lane < C && ck == wkey && cp == piv)) - 1;
    const int xp = lab_eff(piv);
    PANEL_FORCE(xp);
    PANEL_TS(2);
    const double dj = dkey_inv(wkey);
    // this quad's label: position after this step's swap and G entry (load issued first)
    int pos[LPQ];
    bool alive[LPQ];
    double gv[LPQ];
#pragma unroll
    for (int l = 0; l < LPQ; ++l) {
      pos[l] = -1;
      if (mine[l]) pos[l] = (x[l] == y) ? piv : (x[l] == xp ? j : mypos[l]);
      alive[l] = pos[l] > j;
      // G through its lower triangle (trailing updates behind this variant write only that half)
      gv[l] = alive[l] ? p.G[(long long)max(xp, x[l]) * p.ldg + min(xp, x[l])] : 0.0;
    }
    // the dot product and sqrt(dj) go before the stop test: one basic block, so their latency
    // chains interleave (dj <= 0 or NaN always stops; rjj is then unused)
    const double* prow = rows_all[c & 1][src];  // lane-major: prow[q*kRQ + i] = P[xp][q + 4i]
    // ---- update: dot over columns cc = q + 4i < c from registers.  Entries at and beyond c are
    // zero in both operands, so whole 16-column chunks are summed unpredicated; a chunk is skipped
    // (warp-uniform) once c <= its first column.
    double a0[LPQ], a1[LPQ], a2[LPQ], a3[LPQ];
#pragma unroll
    for (int l = 0; l < LPQ; ++l) a0[l] = a1[l] = a2[l] = a3[l] = 0.0;
    const double2* pv = reinterpret_cast<const double2*>(prow + q * kRQ);
    if (kTrace) {  // diagnostic split of the dot phase: first row chunk landed
      const double2 t = pv[0];
      PANEL_FORCE(t.x + t.y);
      PANEL_TS(10);
    }
#pragma unroll
    for (int i = 0; i < kQ; i += 4) {
      if (i / 4 < ch || (i / 4 == ch && u > 0)) {  // == (c > 4 * i)
        const double2 v0 = pv[i / 2], v1 = pv[i / 2 + 1];
#pragma unroll
        for (int l = 0; l < LPQ; ++l) {
          const double2 u0 = own[l][i / 2], u1 = own[l][i / 2 + 1];
          a0[l] = fma(u0.x, v0.x, a0[l]);
          a1[l] = fma(u0.y, v0.y, a1[l]);
          a2[l] = fma(u1.x, v1.x, a2[l]);
          a3[l] = fma(u1.y, v1.y, a3[l]);
        }
      }
    }
    double sq[LPQ];
#pragma unroll
    for (int l = 0; l < LPQ; ++l) {
      sq[l] = (a0[l] + a1[l]) + (a2[l] + a3[l]);
      sq[l] = sq[l] + __shfl_xor_sync(0xffffffffu, sq[l], 1);
      sq[l] = sq[l] + __shfl_xor_sync(0xffffffffu, sq[l], 2);
    }
    PANEL_FORCE(sq[0]);
    PANEL_TS(3);
    const double rjj = sqrt(dj);
    bool stop;
    if (p.pivoting) {
      stop = (dj > 0.0 ? rjj : 0.0) <= cut;            // linalg.cpp:219-223
    } else {
      stop = !isfinite(dj) || dj <= thresh || dj <= 0.0;   // linalg.cpp:118-119
    }
    if (stop) {
      __syncthreads();
      if (tid == 0) {
        if (piv != j) {
          lab_at[j - k] = static_cast<MapT>(xp);
          lab_at[piv - k] = static_cast<MapT>(y);
          pos_of[xp - k] = static_cast<MapT>(j);
          pos_of[y - k] = static_cast<MapT>(piv);
        }
        s_stop = p.pivoting ? 1 : 2;
        if (cta == 0) {
          st->stopped = 1;
          st->rank = j;
          if (!p.pivoting) {
            st->fail = 1;
            st->fail_index = j;
            st->fail_value = dj;
          }
        }
      }
      __syncthreads();
      goto panel_done;
    }
    PANEL_TS(4);
    const double inv_rjj = 1.0 / rjj;
    PANEL_FORCE(inv_rjj);
    PANEL_TS(5);
    const int slot = c >> 2, owner_lane = c & 3;
    unsigned long long bkey = 0;
    int bpos = INT_MAX, bl = 0;
    double col[LPQ];
#pragma unroll
    for (int l = 0; l < LPQ; ++l) col[l] = (gv[l] - sq[l]) * inv_rjj;
    PANEL_FORCE(col[0]);
    PANEL_TS(6);
#pragma unroll
    for (int l = 0; l < LPQ; ++l) {
      // branch-free write of the new column (alive labels) or of F(j, j) = rjj (the pivot)
      const bool is_piv = mine[l] && x[l] == xp;
      const bool wr = (alive[l] || is_piv) && q == owner_lane;
      const double wv = alive[l] ? col[l] : rjj;
      if (wr) myrow[l][slot] = wv;  // read by this step's publication (after the barrier) and later steps
      if (alive[l]) {
        dl[l] = fma(-col[l], col[l], dl[l]);
        if (q == 0 && x[l] < p.neligible && (p.pivoting || pos[l] == j + 1))
          lane_best(bkey, bpos, bl, dkey(dl[l]), pos[l], l);
      }
    }
    const unsigned long long mk = bkey;
    const int mp = bpos;
    warp_argmax(bkey, bpos);
    PANEL_FORCE(bpos);
    PANEL_TS(7);
    const int brow = best_row(bkey, bpos, mp, mk, bl);
    if (lane == 0) {
      wbest[warp].key = bkey;
      wbest[warp].pos = bpos;
      wbest[warp].pad = brow;
    }
    __syncthreads();
    PANEL_TS(8);
    if (c + 1 < kb) combine_publish(j + 1, ch + 1);
    PANEL_TS(9);
    if (kTrace) {
#pragma unroll
      for (int i = 0; i < 9; ++i) tacc[i] += ts[i + 1] - ts[i];
      tacc[9] += 1;
      tacc[10] += ts[10] - ts[2];
    }
    if (tid == 0 && piv != j) {
      lab_at[j - k] = static_cast<MapT>(xp);
      lab_at[piv - k] = static_cast<MapT>(y);
      pos_of[xp - k] = static_cast<MapT>(j);
      pos_of[y - k] = static_cast<MapT>(piv);
    }
    pivp = piv;
    xpp = xp;
    ypp = y;
  }
  }
panel_done:
  __syncthreads();
  if (p.trace && cta == 0 && tid == 0)
    for (int i = 0; i < 11; ++i) atomicAdd(&p.trace[i], static_cast<unsigned long long>(tacc[i]));
  cl.sync();  // no CTA leaves while remote st.async may target it

  // ---- write back: Fo rows by original column, trailing panel, d, order
#pragma unroll
  for (int l = 0; l < LPQ; ++l) {
    if (!mine[l]) continue;
    const int orig = p.ord_in[x[l]];
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      const int cc = q + 4 * i;
      if (cc < kb) p.Fo[(long long)orig * p.ldf + k + cc] = myrow[l][i];
    }
    if (!s_stop) {
      const int t0 = k + kb;
      const int ps = pos_of[x[l] - k];
      if (ps >= t0) {
#pragma unroll
        for (int i = 0; i < kQ; ++i) {
          const int cc = q + 4 * i;
          if (cc < kb) p.PcT[(long long)cc * p.ldp + (ps - t0)] = myrow[l][i];
        }
        if (q == 0) p.d_out[ps] = dl[l];
      }
    }
  }
  for (int ps = cta * blockDim.x + tid; ps < n; ps += C * blockDim.x) {
    if (ps < k) {
      p.ord_out[ps] = p.ord_in[ps];
    } else {
      const int lb = lab_at[ps - k];
      p.ord_out[ps] = p.ord_in[lb];
      p.lab_out[ps] = lb;
    }
  }
  tl_mark(p.tl, p.tl_slot, 2);
}

// ---------------------------------------------------------------------------
size_t panel_smem_bytes(int nl, int R) {
  return size_t(kPanelW) * R * sizeof(double) + size_t(R) * sizeof(double) + size_t(2) * nl * sizeof(int);
}

// Cluster size for a panel of nl labels (0 = use the grid variant).
int panel_cluster_size(int nl) {
  if (nl <= 256) return nl <= 64 ? 1 : (nl <= 128 ? 2 : 4);
  if (nl <= 512) return 8;
  if (nl <= kMaxCluster * kMaxLabelsPerCta) return kMaxCluster;
  return 0;
}

// Labels per quad of panel_reg_kernel (256 threads, 64-wide) for a panel of nl labels (0: another
// variant).  Up to 4 labels per quad: 256 per CTA, 4096 per 16-CTA cluster.
int panel_reg_lpq(int nl) {
  const int CL = panel_cluster_size(nl);
  if (CL <= 0) return 0;
  const int R = (nl + CL - 1) / CL;
  constexpr int kQuads = RegPanel<kPThreads, kPanelW>::kQuads;
  return R <= kQuads ? 1 : (R <= 2 * kQuads ? 2 : (R <= 4 * kQuads ? 4 : 0));
}

// Wide panels (4096 < nl <= 8192 labels): a 16-CTA cluster of 512-thread CTAs, 4 labels per quad
// (512 per CTA), 32 panel columns (the rows of 512 labels at 64 columns would not fit in shared
// memory), 16-bit position maps.  Replaces the cooperative-grid panel there (about 6 us per pivot
// step through global-memory exchange slots).
constexpr int kWideThreads = 512, kWideWidth = 32, kWideLabels = kMaxCluster * (kWideThreads / 4) * 4;
bool panel_is_wide(int n, int k) { return n - k > kMaxCluster * kMaxLabelsPerCta && n - k <= kWideLabels && n < 32768; }
// Panel width the factorisation uses at panel start k of an n-label factorisation.
int panel_width(int n, int k) { return panel_is_wide(n, k) ? kWideWidth : kPanelW; }

// Whether a panel of nl labels runs a register variant (which reads G through its lower triangle).
bool panel_is_reg(int nl) { return panel_reg_lpq(nl) > 0 || (nl > kMaxCluster * kMaxLabelsPerCta && nl <= kWideLabels); }

template <typename K>
static cudaError_t launch_cluster_panel(K kern, const PanelParams& pp, int CL, int threads, size_t smem,
                                        cudaStream_t s) {
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(kern), smem > 0 ? smem : 16, true);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, pp);
}

cudaError_t launch_panel(const PanelParams& p, int num_sms, int* ctas_used, cudaStream_t s) {
  const int nl = p.n - p.k;
  PanelParams pp = p;
  const int CL = panel_cluster_size(nl);
  if (const int lpq = panel_reg_lpq(nl)) {
    pp.rows_per_cta = (nl + CL - 1) / CL;
    const size_t smem = RegPanel<kPThreads, kPanelW>::kLayerBytes * lpq + size_t(2) * nl * sizeof(int);
    auto kern = lpq == 1 ? (p.trace ? panel_reg_kernel<true, 1> : panel_reg_kernel<false, 1>)
                : lpq == 2 ? (p.trace ? panel_reg_kernel<true, 2> : panel_reg_kernel<false, 2>)
                           : (p.trace ? panel_reg_kernel<true, 4> : panel_reg_kernel<false, 4>);
    if (ctas_used) *ctas_used = CL;
    return launch_cluster_panel(kern, pp, CL, kPThreads, smem, s);
  }
  if (panel_is_wide(p.n, p.k)) {
    if (p.kb > kWideWidth) return cudaErrorInvalidValue;
    pp.rows_per_cta = (nl + kMaxCluster - 1) / kMaxCluster;
    const size_t smem = RegPanel<kWideThreads, kWideWidth>::kLayerBytes * 4 + size_t(2) * nl * sizeof(short);
    auto kern = p.trace ? panel_reg_kernel<true, 4, kWideThreads, kWideWidth, short>
                        : panel_reg_kernel<false, 4, kWideThreads, kWideWidth, short>;
    if (ctas_used) *ctas_used = kMaxCluster;
    return launch_cluster_panel(kern, pp, kMaxCluster, kWideThreads, smem, s);
  }
  // grid variant: ~ceil(nl / num_sms) labels per CTA, every CTA co-resident (cooperative launch)
  int R = (nl + num_sms - 1) / num_sms;
  if (R < 32) R = 32;
  if (R > kMaxLabelsPerCta) return cudaErrorInvalidValue;  // n > 256 * num_sms unsupported
  const int C = (nl + R - 1) / R;
  pp.rows_per_cta = R;
  const size_t smem = panel_smem_bytes(nl, R);
  cudaError_t e = ensure_attrs(reinterpret_cast<const void*>(panel_kernel_t<false>), smem);
  if (e != cudaSuccess) return e;
  if (ctas_used) *ctas_used = C;
  void* args[] = {&pp};
  return cudaLaunchCooperativeKernel((void*)panel_kernel_t<false>, dim3(C), dim3(kPThreads), args, smem, s);
}

}  // namespace rbpg
