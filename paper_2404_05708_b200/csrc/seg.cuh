// seg.cuh — segmented two-column kernel for batches of single-band pairs
// (SURVEY §8(a) a1–a6; BASELINE configs 2 and 1-like shapes).
//
// What: δ_dF of every pair, Eq. (1) M_ij = max{min{M_{i-1,j}, M_{i-1,j-1},
// M_{i,j-1}}, d_ij}, linear state (Theorem 1; Alg. 5,
// L229–L248), for pairs whose longer curve has at most 512 points.
//
// How — the all-pairs kernel's structure (cdist.cu), made to
// work on independent pairs:
//   * A warp is G = 32/W segments of W lanes (W = 16 or 32).  A segment holds
//     one pair's rows (the LONGER curve, padded to W·R rows by repeating its
//     last point: exact, PAPER L259 footnote), lane s rows [sR, sR+R), and
//     processes stream positions 2(t−s), 2(t−s)+1 at warp step t: two columns
//     per step, the second column's chain trailing the first by one row, so the
//     shuffle + min/max chain latency is paid once per two columns.
//   * A work ITEM is G·L pairs of the same (W, R) and nearly the same column
//     count; every pair's stream is padded to the item's period 2H (sentinel +
//     columns + repeats of its last column: exact for δ_dF), segment h runs
//     pairs h, h+G, h+2G, … back to back.  All segments therefore switch pairs
//     at the same steps: the result of pair k leaves at step H(k+1)+W−1, the
//     corner value enters at step Hk, and lane s takes pair k's rows at step
//     Hk+s — one predicated shared-memory load per row vector in a W-step
//     window, no divergent per-lane events.
//   * Row strips of the next pair are staged in shared memory (cp.async, then
//     converted: int input is translated by the pair's first row point into
//     the fp32-exact window) during the current pair.
//   * Column points are fetched one 32-position chunk ahead into registers and
//     written into a per-warp ring (one LDS.128 per column per lane).
//   * Items come from a list sorted by (shape, period), largest first (PAPER
//     L261–L262), popped by persistent warps.
#pragma once
#include "prep.cuh"
#include "strip.cuh"

namespace ffd {

constexpr int kSegL = 2;           // pairs per segment per item (default; FFD_SEG_L = 2 … 8 at run time:
                                   // larger items put more shapes in flight at once and thrash the
                                   // instruction cache — L = 8 measured 3.7 against 2.6 ms on config 2)
constexpr int kSegMaxL = 8;
constexpr int kSegMaxItemPairs = 2 * kSegMaxL;  // G·L ≤ 16
constexpr int kSegRows = 512;      // rows per warp: G·W·R ≤ 512
constexpr int kSegHStep = 4;       // period buckets of 4 steps
constexpr int kSegHB = 65;         // H ≤ 257 (columns ≤ 512)
constexpr int kSegShapes = 16;     // W = 16: R ∈ {2, 4, …, 16};  W = 32: R ∈ {9, …, 16}
constexpr int kSegBins = kSegShapes * kSegHB;
constexpr int kSegLag = 32;        // H ≥ W + kSegLag: a pair's row staging finishes in its predecessor
static_assert(kSegBins == kSegBinsP, "prep.cuh bin count");

__host__ __device__ inline void seg_shape(int idx, int& W, int& R) {
  if (idx < 8) {
    W = 16;
    R = 2 * (idx + 1);
  } else {
    W = 32;
    R = idx + 1;
  }
}
// (W, R) shape for a rows curve of `rows` ≤ 512 points: rows padded to a multiple of 32
__host__ __device__ inline int seg_shape_for(int rows) {
  if (rows <= 256) {
    int R = (rows + 15) / 16;
    R += R & 1;
    return R / 2 - 1;
  }
  return (rows + 31) / 32 - 1;
}
__host__ __device__ inline int seg_period(int cols) { return (cols + 2) / 2; }  // H: 2H ≥ 1 + cols
// seg key of a Fréchet pair (n, m), or −1 if it stays on the batch kernel
__host__ __device__ inline int seg_bin(int n, int m) {
  const int rows = n > m ? n : m, cols = n > m ? m : n;
  if (rows > kSegRows) return -1;
  int W, R;
  const int sh = seg_shape_for(rows);
  seg_shape(sh, W, R);
  const int H = seg_period(cols);
  if (H < W + kSegLag) return -1;
  return sh * kSegHB + (H - 1) / kSegHStep;
}
__host__ __device__ inline int seg_item_pairs(int bin, int L) {
  int W, R;
  seg_shape(bin / kSegHB, W, R);
  return (kWarp / W) * L;
}

struct SegItem {
  int start;      // first pair in the seg-sorted list
  int16_t count;  // pairs (≤ G·L)
  int16_t shape;  // (W, R) index
};

struct SegProblem {
  const void* p;
  const void* q;
  const PairDesc* sorted;  // seg-sorted pairs (rows = the longer curve)
  const SegItem* items;
  const int* n_items;
  int* counter;
  void* out;
  int* fb_list;  // int input: pairs that left the fp32-exact window (exact int64 tier)
  int* fb_count;
};

template <int KIND, int D, bool INT_IN>
struct alignas(16) SegSmem {
  using C = SCfg<float, KIND, D, INT_IN>;
  uint4 ring[128 * C::EW];               // 128 positions (G = 1) or 2 × 64 (G = 2)
  float stage[C::NS][kSegRows];          // next pair's row strips, [c][h·W·RP + s·RP + r]
  int32_t raw[INT_IN ? kSegRows * D : 4];  // int input: raw points (cp.async target)
  const void* rows_ptr[kSegMaxItemPairs];
  const void* cols_ptr[kSegMaxItemPairs];
  int nrows[kSegMaxItemPairs];
  int ncols[kSegMaxItemPairs];
  int idx[kSegMaxItemPairs];
  int bad[kSegMaxItemPairs];
  int center[kSegMaxItemPairs][D];
};

template <int KIND, int D, bool INT_IN, int FIN, int W, int R>
struct SegRunner {
  using C = SCfg<float, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  using Sm = SegSmem<KIND, D, INT_IN>;
  static constexpr int G = kWarp / W;     // segments per warp
  static constexpr int RING = 128 / G;    // ring positions per segment
  static constexpr int RP = (R + 3) & ~3; // lane stride in the stage arrays (16-B aligned)
  static constexpr int NS = C::NS;
  static constexpr int EW = C::EW;
  static_assert(G * W * RP <= kSegRows, "stage arrays");
  static_assert(!INT_IN || G * W * R <= kSegRows, "raw stage");

  Sm& sm;
  const SegProblem& pb;
  const int lane, s, h;
  int count, H, Lh;

  __device__ SegRunner(Sm& m, const SegProblem& p, int l)
      : sm(m), pb(p), lane(l), s(l % W), h(l / W) {}

  // pair slot of segment hh in sequence position k (a missing pair reads pair 0)
  __device__ __forceinline__ int slot(int hh, int k) const {
    const int j = hh + G * k;
    return j < count ? j : 0;
  }

  // one input point of pair j translated into the fp32-exact window (int input)
  __device__ __forceinline__ bool conv(const In (&a)[D], int j, float (&v)[D]) const {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < D; c++) {
      if constexpr (INT_IN) {
        const long long t = (long long)a[c] - (long long)sm.center[j][c];
        ok &= (t >= -C::LIM) && (t <= C::LIM);
        v[c] = (float)(int)t;
      } else {
        v[c] = (float)a[c];
      }
    }
    return ok;
  }

  // ---- row strips: stage pair k of every segment (cp.async), then convert ----
  __device__ __forceinline__ void stage_issue(int k) {
    for (int i = lane; i < G * W * R; i += kWarp) {
      const int hh = i / (W * R), rr = i - hh * (W * R);
      const int j = slot(hh, k);
      const int row = min(rr, sm.nrows[j] - 1);
      const In* src = reinterpret_cast<const In*>(sm.rows_ptr[j]) + (int64_t)row * D;
#pragma unroll
      for (int c = 0; c < D; c++) {
        uint32_t dst;
        if constexpr (INT_IN) dst = (uint32_t)__cvta_generic_to_shared(&sm.raw[i * D + c]);
        else dst = (uint32_t)__cvta_generic_to_shared(&sm.stage[c][hh * W * RP + (rr / R) * RP + rr % R]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src + c) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void stage_finish(int k) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if constexpr (INT_IN || C::XSQ) {
      for (int i = lane; i < G * W * R; i += kWarp) {
        const int hh = i / (W * R), rr = i - hh * (W * R);
        const int j = slot(hh, k);
        In a[D];
        float v[D];
#pragma unroll
        for (int c = 0; c < D; c++) {
          if constexpr (INT_IN) a[c] = sm.raw[i * D + c];
          else a[c] = sm.stage[c][hh * W * RP + (rr / R) * RP + rr % R];
        }
        const bool ok = conv(a, j, v);
        if (!ok) sm.bad[j] = 1;
        const int o = hh * W * RP + (rr / R) * RP + rr % R;
#pragma unroll
        for (int c = 0; c < D; c++) sm.stage[c][o] = v[c];
        if constexpr (C::XSQ) {
          int pp = 0;
#pragma unroll
          for (int c = 0; c < D; c++) pp += (int)v[c] * (int)v[c];
          sm.stage[D][o] = (float)pp;
        }
      }
      __syncwarp();
    }
  }
  // lanes with p take their strip from the stage arrays (one predicated vector
  // load per 4 rows); sa: shared address of this lane's strip of coordinate 0
  __device__ __forceinline__ void take_rows(float (&x)[NS][R], uint32_t sa, int p) const {
#pragma unroll
    for (int c = 0; c < NS; c++) pred_lds_strip<R>(x[c], sa + c * kSegRows * 4, p);
  }

  // ---- column stream of segment hh: position pos → element ------------------
  struct Raw {
    In a[D];
    int j;     // pair slot
    int kind;  // 0 point, 1 sentinel / past the end
  };
  __device__ __forceinline__ void fetch(int pos, Raw& r) const {
#pragma unroll
    for (int c = 0; c < D; c++) r.a[c] = (In)0;
    const int k = pos / (2 * H), loc = pos - k * 2 * H;
    r.j = slot(h, k < Lh ? k : 0);
    if (k >= Lh || loc == 0) {
      r.kind = 1;
      return;
    }
    r.kind = 0;
    const int col = min(loc - 1, sm.ncols[r.j] - 1);
    const In* src = reinterpret_cast<const In*>(sm.cols_ptr[r.j]) + (int64_t)col * D;
#pragma unroll
    for (int c = 0; c < D; c++) r.a[c] = __ldg(src + c);
  }
  // ring slot of position pos: the even and the odd positions in separate halves,
  // so that the lanes of a step (positions 2(t−s), 2(t−s)+1) read consecutive
  // 16-byte elements (interleaving them made every element load a 2-way bank conflict)
  static __device__ __forceinline__ int rslot(int pos) {
    return (((pos & 1) * (RING / 2) + ((pos >> 1) & (RING / 2 - 1))) * G);
  }
  __device__ __forceinline__ void store(int pos, const Raw& r) {
    alignas(16) float e[C::EBYTES / 4];
#pragma unroll
    for (int i = 0; i < C::EBYTES / 4; i++) e[i] = 0.f;
    if (r.kind != 0) {
      if constexpr (C::XSQ) e[D] = finf();
      else {
#pragma unroll
        for (int c = 0; c < D; c++) e[c] = finf();
      }
    } else {
      float v[D];
      if (!conv(r.a, r.j, v)) sm.bad[r.j] = 1;
      if constexpr (C::XSQ) {
        int qq = 0;
#pragma unroll
        for (int c = 0; c < D; c++) {
          qq += (int)v[c] * (int)v[c];
          e[c] = -2.f * v[c];
        }
        e[D] = (float)qq;
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) e[c] = v[c];
      }
    }
    uint4* dst = sm.ring + (rslot(pos) + h) * EW;
#pragma unroll
    for (int w = 0; w < EW; w++) dst[w] = reinterpret_cast<const uint4*>(e)[w];
  }

  // ---- result of the pair in slot (h, k): the segment's last lane ------------
  __device__ __forceinline__ void emit(int k, float v) {
    const int j = h + G * k;
    if (s != W - 1 || j >= count) return;
    const int idx = sm.idx[j];
    if constexpr (INT_IN) {
      if (sm.bad[j]) {
        pb.fb_list[atomicAdd(pb.fb_count, 1)] = idx;
        return;
      }
      reinterpret_cast<long long*>(pb.out)[idx] = (long long)v;
    } else {
      if constexpr (FIN == F_SQRT) v = sqrt_result(v);
      reinterpret_cast<float*>(pb.out)[idx] = v;
    }
  }

  __device__ void run() {
    const int NT = H * Lh;         // steps until lane 0 has consumed every position
    const int total = NT + W - 1;  // the segment's last lane finishes W − 1 steps later
    float x[NS][R], c[R];
    // rows of the first pair of every segment
    stage_issue(0);
    stage_finish(0);
#pragma unroll
    for (int cc = 0; cc < NS; cc++)
#pragma unroll
      for (int r = 0; r < R; r++) x[cc][r] = sm.stage[cc][h * W * RP + s * RP + r];
#pragma unroll
    for (int r = 0; r < R; r++) c[r] = finf();
    // column ring: positions [0, 32) of every segment stored, [32, 64) prefetched
    Raw pre[G];
#pragma unroll
    for (int e = 0; e < G; e++) {
      Raw r0;
      fetch(s * G + e, r0);
      store(s * G + e, r0);
      fetch(32 + s * G + e, pre[e]);
    }
    __syncwarp();
    __syncwarp();  // stage arrays read by every lane before the next staging overwrites them

    float diag = finf(), b0v = finf();
    // one step on positions 2g, 2g+1 of this segment; top0: what the segment's
    // first lane sees above its first row in the first column (the corner 0 on
    // a sentinel, +∞ otherwise; the second column is never a sentinel)
    auto step = [&](int t, float top0) {
      const int g = t - s;
      alignas(16) float e0[C::EBYTES / 4], e1[C::EBYTES / 4];
      {
        const uint4* s0 = sm.ring + (rslot(2 * g) + h) * EW;
        const uint4* s1 = sm.ring + (rslot(2 * g + 1) + h) * EW;
#pragma unroll
        for (int w = 0; w < EW; w++) {
          reinterpret_cast<uint4*>(e0)[w] = s0[w];
          reinterpret_cast<uint4*>(e1)[w] = s1[w];
        }
      }
      const float upv0 = __shfl_up_sync(0xffffffffu, b0v, 1, W);
      const float upv1 = __shfl_up_sync(0xffffffffu, c[R - 1], 1, W);
      const float up0 = (s == 0) ? top0 : upv0;
      const float up1 = (s == 0) ? finf() : upv1;
      float d0[R], d1[R];
      cell_dists<float, KIND, D, R, INT_IN>(x, e0, d0);
      cell_dists<float, KIND, D, R, INT_IN>(x, e1, d1);
      {
        float u = up0, dg = diag;
#pragma unroll
        for (int r = 0; r < R; r++) {
          const float nv = fmaxf(fminf(fminf(u, dg), c[r]), d0[r]);
          dg = c[r];
          c[r] = nv;
          u = nv;
        }
      }
      b0v = c[R - 1];
      {
        float u = up1, dg = up0;
#pragma unroll
        for (int r = 0; r < R; r++) {
          const float nv = fmaxf(fminf(fminf(u, dg), c[r]), d1[r]);
          dg = c[r];
          c[r] = nv;
          u = nv;
        }
      }
      diag = up1;
    };
    int next_refill = 16;  // 32 positions per segment per refill
    int stage_k = 1;       // next pair (sequence position) to stage
    bool staging = false;  // cp.async of stage_k − 1 in flight
    // every 16 steps: the chunk of positions [2t, 2t+32) is stored, the next one
    // prefetched; the row staging of the next pair is issued at the first refill
    // after the current pair's window and finished at the one after that
    auto refill = [&](int t) {
#pragma unroll
      for (int e = 0; e < G; e++) {
        store(2 * t + s * G + e, pre[e]);
        fetch(2 * t + 32 + s * G + e, pre[e]);
      }
      if (staging) {
        stage_finish(stage_k - 1);
        staging = false;
      } else if (stage_k < Lh && t >= H * (stage_k - 1) + W) {
        stage_issue(stage_k);
        ++stage_k;
        staging = true;
      }
      next_refill += 16;
      __syncwarp();
    };
    const uint32_t stage_sa = (uint32_t)__cvta_generic_to_shared(&sm.stage[0][h * W * RP + s * RP]);
    float res = finf();  // the segment's last lane: result of the pair before the window
    int t = 0;
    for (int k = 0; k < Lh; k++) {
      const int t0 = H * k, tw = t0 + W, t1 = t0 + H;
      // step Hk: the sentinel of pair k reaches lane 0 (corner value 0 above its first row)
      if (t == next_refill) refill(t);
      if (k > 0) take_rows(x, stage_sa, s == 0);
      step(t, 0.f);
      ++t;
      if (k > 0) {
        // the rest of the window: lane s takes pair k's rows at step Hk + s; the
        // last lane keeps its value of pair k − 1 (complete before its switch)
        while (t < tw) {
          const int stop = min(next_refill, tw);
#pragma unroll 2
          for (; t < stop; ++t) {
            const int p = s == t - t0;
            res = p ? c[R - 1] : res;
            take_rows(x, stage_sa, p);
            step(t, finf());
          }
          if (t == next_refill && t < tw) refill(t);
        }
        emit(k - 1, res);
      }
      while (t < t1) {
        const int stop = min(next_refill, t1);
#pragma unroll 2
        for (; t < stop; ++t) step(t, finf());
        if (t == next_refill && t < t1) refill(t);
      }
    }
    for (; t < total; t++) {  // drain: positions past the stream's end
      if (t == next_refill) refill(t);
      step(t, finf());
    }
    emit(Lh - 1, c[R - 1]);
    __syncwarp();
  }
};

template <int KIND, int D, bool INT_IN, int FIN>
__global__ void __launch_bounds__(kWarp* kWarpsPerCta, 4) seg_kernel(const SegProblem pb) {
  using Sm = SegSmem<KIND, D, INT_IN>;
  extern __shared__ uint4 seg_dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Sm& sm = reinterpret_cast<Sm*>(seg_dyn)[warp];
  for (int i = lane; i < 128 * SCfg<float, KIND, D, INT_IN>::EW; i += kWarp) sm.ring[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
  const int n_items = *pb.n_items;
  while (true) {
    int item = 0;
    if (lane == 0) item = atomicAdd(pb.counter, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const SegItem it = pb.items[item];
    int m = 0;
    if (lane < it.count) {
      const PairDesc d = pb.sorted[it.start + lane];
      using In = typename std::conditional<INT_IN, int32_t, float>::type;
      const In* rp = reinterpret_cast<const In*>(d.swap ? pb.q : pb.p) + d.row_off * D;
      const In* cp = reinterpret_cast<const In*>(d.swap ? pb.p : pb.q) + d.col_off * D;
      sm.rows_ptr[lane] = rp;
      sm.cols_ptr[lane] = cp;
      sm.nrows[lane] = d.n_rows;
      sm.ncols[lane] = d.m_cols;
      sm.idx[lane] = d.idx;
      sm.bad[lane] = 0;
      if constexpr (INT_IN) {
#pragma unroll
        for (int c = 0; c < D; c++) sm.center[lane][c] = (int)rp[c];
      }
      m = d.m_cols;
    }
    const int H = seg_period(__reduce_max_sync(0xffffffffu, m));
    __syncwarp();
    auto go = [&](auto& run) {
      run.count = it.count;
      run.H = H;
      run.Lh = (it.count + run.G - 1) / run.G;
      run.run();
    };
#define FFD_SEG_CASE(IDX, WW, RR)                              \
  case IDX: {                                                  \
    SegRunner<KIND, D, INT_IN, FIN, WW, RR> run(sm, pb, lane); \
    go(run);                                                   \
    break;                                                     \
  }
    switch (it.shape) {
      FFD_SEG_CASE(0, 16, 2)
      FFD_SEG_CASE(1, 16, 4)
      FFD_SEG_CASE(2, 16, 6)
      FFD_SEG_CASE(3, 16, 8)
      FFD_SEG_CASE(4, 16, 10)
      FFD_SEG_CASE(5, 16, 12)
      FFD_SEG_CASE(6, 16, 14)
      FFD_SEG_CASE(7, 16, 16)
      FFD_SEG_CASE(8, 32, 9)
      FFD_SEG_CASE(9, 32, 10)
      FFD_SEG_CASE(10, 32, 11)
      FFD_SEG_CASE(11, 32, 12)
      FFD_SEG_CASE(12, 32, 13)
      FFD_SEG_CASE(13, 32, 14)
      FFD_SEG_CASE(14, 32, 15)
      FFD_SEG_CASE(15, 32, 16)
      default:
        break;
    }
#undef FFD_SEG_CASE
    __syncwarp();
  }
}

// ---- host side (seg.cu) ------------------------------------------------------
struct SegWs {
  PairDesc* sorted;  // [B]
  SegItem* items;    // [seg_max_items(B)]
  int* item_off;     // [kSegBins] first item of each bin (descending bin order)
};
__host__ __device__ inline int64_t seg_max_items(int64_t B) { return B / 2 + kSegBins + 1; }  // L ≥ 2
int seg_items_per_segment();  // L: FFD_SEG_L (2 … 8), default kSegL
// the seg kernel is built for this (kind, dim, int input, finalisation)
bool seg_supported(int kind, int dim, int int_in, int fin);
cudaError_t launch_seg(const SegProblem& pb, int kind, int dim, int int_in, int fin, int sms, cudaStream_t st);

}  // namespace ffd
