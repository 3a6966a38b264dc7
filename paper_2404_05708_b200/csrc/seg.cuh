// seg.cuh — segmented two-column kernel for batches of single-band pairs
// (SURVEY §8(a) a1–a6; BASELINE config 2 and every 2-D pair ≤ 512 points).
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
//   * A GROUP is G pairs of the same (W, R) and nearly the same column count
//     (the prep sorts pairs by (shape, period)); its streams are padded to the
//     group's period 2H (sentinel + columns + repeats of the last column: exact
//     for δ_dF), one pair per segment.  A warp runs a STREAM of groups of one
//     shape back to back: group k occupies steps [T_k, T_k + H_k) of lane 0, so
//     every segment switches pairs at the same steps — the corner value enters
//     at T_k, lane s takes group k's rows at T_k + s (one predicated shared
//     load per 4 rows in a W-step window), and group k − 1's result is complete
//     in the segment's last lane before T_k + W − 1.  Only a change of shape
//     (or the end of the list) drains the lane pipeline (W − 1 steps).
//   * Groups are popped one ahead (atomic counter; the group record holds its
//     pair descriptors, so one dependent load), accepted at the first ring
//     refill of the previous group, and their rows staged in shared memory
//     (cp.async, then converted: int input is translated by the pair's first row
//     point into the fp32-exact window) after its window.
//   * Column points are fetched one 32-position chunk ahead into registers and
//     written into a per-warp ring (one LDS.128 per column per lane).
//   * Groups come from a list sorted by (shape, period), largest first (PAPER
//     L261–L262): all warps move through it together, so an SM runs few shapes
//     at a time (their code shares the instruction cache).
#pragma once
#include "prep.cuh"
#include "strip.cuh"

namespace ffd {

constexpr int kSegRows = 512;      // longest rows curve of a segmented pair
constexpr int kSegRowsBig = 1024;  // stage rows of the big kernel (2 segments × 16 lanes × R ≤ 32)
constexpr int kSegHStep = 4;       // period buckets of 4 steps
constexpr int kSegHB = 65;         // H ≤ 257 (columns ≤ 512)
constexpr int kSegShapes = 24;     // 0–7: W = 16, R ∈ {2, 4, …, 16};  8–15: W = 32, R ∈ {9, …, 16};
                                   // 16–23 (the big kernel): W = 16, R ∈ {18, 20, …, 32}
constexpr int kSegSmallShapes = 16;
constexpr int kSegBins = kSegShapes * kSegHB;
constexpr int kSegLag = 32;        // H ≥ W + kSegLag: a group's rows are staged inside its predecessor
constexpr int kSegSlots = 4;       // group records per warp (current, next, two finished)
static_assert(kSegBins == kSegBinsP, "prep.cuh bin count");

__host__ __device__ inline void seg_shape(int idx, int& W, int& R) {
  if (idx < 8) {
    W = 16;
    R = 2 * (idx + 1);
  } else if (idx < 16) {
    W = 32;
    R = idx + 1;
  } else {
    W = 16;
    R = 2 * (idx - 7);
  }
}
// (W, R) shape for a rows curve of `rows` ≤ 512 points: rows padded to a multiple
// of 32.  big: rows above 256 take two 16-lane segments of up to 32 rows per lane
// (the big kernel) instead of one 32-lane segment of up to 16
__host__ __device__ inline int seg_shape_for(int rows, bool big) {
  if (rows <= 256 || big) {
    int R = (rows + 15) / 16;
    R += R & 1;
    return R <= 16 ? R / 2 - 1 : R / 2 + 7;
  }
  return (rows + 31) / 32 - 1;
}
__host__ __device__ inline int seg_period(int cols) { return (cols + 2) / 2; }  // H: 2H ≥ 1 + cols
// seg key of a Fréchet pair (n, m), or −1 if it stays on the batch kernel
__host__ __device__ inline int seg_bin(int n, int m, bool big) {
  const int rows = n > m ? n : m, cols = n > m ? m : n;
  if (rows > kSegRows) return -1;
  int W, R;
  const int sh = seg_shape_for(rows, big);
  seg_shape(sh, W, R);
  const int H = seg_period(cols);
  if (H < W + kSegLag) return -1;
  return sh * kSegHB + (H - 1) / kSegHStep;
}
__host__ __device__ inline int seg_group_pairs(int bin) {
  int W, R;
  seg_shape(bin / kSegHB, W, R);
  return kWarp / W;
}

// one group: G ≤ 2 pair descriptors (rows = the longer curve) and its shape
struct alignas(16) SegGroup {
  PairDesc d[2];
  int count;  // pairs (1 … G)
  int shape;  // (W, R) index
  int pad[2];
};
static_assert(sizeof(SegGroup) == 80, "SegGroup");

struct SegProblem {
  const void* p;
  const void* q;
  const SegGroup* groups;
  const int* n_groups;
  const int* shape_info;  // [16][3]: first group, end, work (float bits) of each shape
  int* shape_ctr;         // [2] groups popped by the small and the big kernel
  void* out;
  int* fb_list;  // int input: pairs that left the fp32-exact window (exact int64 tier)
  int* fb_count;
};

// a popped group, held in registers until it is accepted into a stream
struct SegLook {
  PairDesc d;  // lanes < G: pair `lane` of the group
  int count;   // 0: no group (the list is exhausted)
  int shape;
};

template <int D>
struct SegSlot {
  const void* rows_ptr[2];
  const void* cols_ptr[2];
  int nrows[2];
  int ncols[2];
  int idx[2];
  int bad[2];
  int center[2][D];
  int count;
};

template <int KIND, int D, bool INT_IN, int ROWS>
struct alignas(16) SegSmem {
  using C = SCfg<float, KIND, D, INT_IN>;
  uint4 ring[128 * C::EW];  // 128 positions (G = 1) or 2 × 64 (G = 2)
  float stage[C::NS][ROWS]; // the next group's row strips, [c][h·W·RP + s·RP + r] (int input:
                            // copied as int32 bits, converted in place)
  SegSlot<D> slot[kSegSlots];
};

// Pop the next group of this kernel's shapes [LO, LO + NSH): the list holds them
// contiguously (descending shape index), from the first group of the highest
// shape to the end of the lowest; one atomic counter per kernel (lane 0), the
// record's loads are left in flight.  All warps move through the list together,
// so an SM runs few shapes at a time (measured: spreading the SMs over the
// shapes by their work lost 2.49 -> 2.65 ms on config 2).
template <int LO, int NSH>
__device__ __forceinline__ void seg_pop(const SegProblem& pb, int lane, SegLook& L) {
  int g = 0, end = 0;
  if (lane == 0) {
    const int first = pb.shape_info[3 * (LO + NSH - 1)];
    end = pb.shape_info[3 * LO + 1];
    g = first + atomicAdd(pb.shape_ctr + (LO > 0 ? 1 : 0), 1);
  }
  g = __shfl_sync(0xffffffffu, g, 0);
  end = __shfl_sync(0xffffffffu, end, 0);
  L.count = 0;
  L.shape = -1;
  if (g < end) {
    const SegGroup* gp = pb.groups + g;
    L.d = gp->d[lane & 1];
    L.count = gp->count;
    L.shape = gp->shape;
  }
}

template <int KIND, int D, bool INT_IN, int FIN, int W, int R, int ROWS, int LO, int NSH>
struct SegRunner {
  using C = SCfg<float, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  using Sm = SegSmem<KIND, D, INT_IN, ROWS>;
  static constexpr int G = kWarp / W;     // segments per warp
  static constexpr int RING = 128 / G;    // ring positions per segment
  static constexpr int RP = (R + 3) & ~3; // lane stride in the stage arrays (16-B aligned)
  static constexpr int NS = C::NS;
  static constexpr int EW = C::EW;
  static constexpr int SHAPE = W == 32 ? R - 1 : (R <= 16 ? R / 2 - 1 : R / 2 + 7);
  static_assert(G * W * RP <= ROWS, "stage arrays");

  Sm& sm;
  const SegProblem& pb;
  const int lane, s, h;

  __device__ SegRunner(Sm& m, const SegProblem& p, int l) : sm(m), pb(p), lane(l), s(l % W), h(l / W) {}

  // the group record L into slot j
  __device__ __forceinline__ void accept(const SegLook& L, int j) {
    SegSlot<D>& S = sm.slot[j];
    if (lane < L.count) {
      const PairDesc& d = L.d;
      const In* rp = reinterpret_cast<const In*>(d.swap ? pb.q : pb.p) + d.row_off * D;
      const In* cp = reinterpret_cast<const In*>(d.swap ? pb.p : pb.q) + d.col_off * D;
      S.rows_ptr[lane] = rp;
      S.cols_ptr[lane] = cp;
      S.nrows[lane] = d.n_rows;
      S.ncols[lane] = d.m_cols;
      S.idx[lane] = d.idx;
      S.bad[lane] = 0;
      if constexpr (INT_IN) {
#pragma unroll
        for (int c = 0; c < D; c++) S.center[lane][c] = (int)rp[c];
      }
    }
    if (lane == 0) S.count = L.count;
    __syncwarp();
  }
  // period of the group in slot j (uniform)
  __device__ __forceinline__ int period(int j) const {
    const int m = lane < sm.slot[j].count ? sm.slot[j].ncols[lane] : 0;
    return seg_period(__reduce_max_sync(0xffffffffu, m));
  }

  // pair of segment hh in slot j (a segment without a pair reads pair 0)
  __device__ __forceinline__ int pair_of(int j, int hh) const { return hh < sm.slot[j].count ? hh : 0; }

  // one input point of pair (j, pr) translated into the fp32-exact window (int input)
  __device__ __forceinline__ bool conv(const In (&a)[D], int j, int pr, float (&v)[D]) const {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < D; c++) {
      if constexpr (INT_IN) {
        const long long t = (long long)a[c] - (long long)sm.slot[j].center[pr][c];
        ok &= (t >= -C::LIM) && (t <= C::LIM);
        v[c] = (float)(int)t;
      } else {
        v[c] = (float)a[c];
      }
    }
    return ok;
  }

  // ---- row strips: stage the group in slot j (cp.async), then convert --------
  __device__ __forceinline__ void stage_issue(int j) {
    for (int i = lane; i < G * W * R; i += kWarp) {
      const int hh = i / (W * R), rr = i - hh * (W * R);
      const int pr = pair_of(j, hh);
      const int row = min(rr, sm.slot[j].nrows[pr] - 1);
      const In* src = reinterpret_cast<const In*>(sm.slot[j].rows_ptr[pr]) + (int64_t)row * D;
#pragma unroll
      for (int c = 0; c < D; c++) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&sm.stage[c][hh * W * RP + (rr / R) * RP + rr % R]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src + c) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void stage_finish(int j) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    if constexpr (INT_IN) {
      for (int i = lane; i < G * W * R; i += kWarp) {
        const int hh = i / (W * R), rr = i - hh * (W * R);
        const int pr = pair_of(j, hh);
        const int o = hh * W * RP + (rr / R) * RP + rr % R;
        In a[D];
        float v[D];
#pragma unroll
        for (int c = 0; c < D; c++) a[c] = __float_as_int(sm.stage[c][o]);
        if (!conv(a, j, pr, v)) sm.slot[j].bad[pr] = 1;
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
    for (int c = 0; c < NS; c++) pred_lds_strip<R>(x[c], sa + c * ROWS * 4, p);
  }

  // ---- column stream of this segment: position pos → element ----------------
  struct Raw {
    In a[D];
    int j, pr;  // slot, pair
    int kind;   // 0 point, 1 sentinel
  };
  // pos lies in group k (slot jk, from step Tk) or — when the next group is
  // accepted (Tn ≥ 0) — possibly in it (slot jn, from step Tn).  Positions past
  // the stream's last group repeat its last column (they only reach the drain).
  __device__ __forceinline__ void fetch(int pos, int jk, int Tk, int jn, int Tn, Raw& r) const {
#pragma unroll
    for (int c = 0; c < D; c++) r.a[c] = (In)0;
    const bool nxt = Tn >= 0 && pos >= 2 * Tn;
    r.j = nxt ? jn : jk;
    r.pr = pair_of(r.j, h);
    const int loc = pos - 2 * (nxt ? Tn : Tk);
    if (loc == 0) {
      r.kind = 1;
      return;
    }
    r.kind = 0;
    const int col = min(loc - 1, sm.slot[r.j].ncols[r.pr] - 1);
    const In* src = reinterpret_cast<const In*>(sm.slot[r.j].cols_ptr[r.pr]) + (int64_t)col * D;
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
      if (!conv(r.a, r.j, r.pr, v)) sm.slot[r.j].bad[r.pr] = 1;
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

  // ---- result of this segment's pair in slot j: the segment's last lane ------
  __device__ __forceinline__ void emit(int j, float v) {
    if (s != W - 1 || h >= sm.slot[j].count) return;
    const int idx = sm.slot[j].idx[h];
    if constexpr (INT_IN) {
      if (sm.slot[j].bad[h]) {
        pb.fb_list[atomicAdd(pb.fb_count, 1)] = idx;
        return;
      }
      reinterpret_cast<long long*>(pb.out)[idx] = (long long)v;
    } else {
      if constexpr (FIN == F_SQRT) v = sqrt_result(v);
      reinterpret_cast<float*>(pb.out)[idx] = v;
    }
  }

  // One stream: `look` holds its first group (of this shape); groups of the same
  // shape follow until the list ends or a group of another shape is popped —
  // that one is left in `look` for the caller.
  __device__ void stream(SegLook& look) {
    constexpr int SM = kSegSlots - 1;
    float x[NS][R], c[R];
    accept(look, 0);  // group 0 → slot 0
    int H = period(0);
    seg_pop<LO, NSH>(pb, lane, look);  // the next group, in flight
    stage_issue(0);
    stage_finish(0);
#pragma unroll
    for (int cc = 0; cc < NS; cc++)
#pragma unroll
      for (int r = 0; r < R; r++) x[cc][r] = sm.stage[cc][h * W * RP + s * RP + r];
#pragma unroll
    for (int r = 0; r < R; r++) c[r] = finf();
    // stream state (uniform): group k in slot k & SM from step Tk with period H;
    // the next group (once accepted) from step Tn (−1: not decided, or none)
    int k = 0, Tk = 0, Tn = -1;
    bool decided = false, last = false;  // next group decided; group k is the stream's last
    bool staging = false, stage_due = false;
    // column ring: positions [0, 32) of every segment stored, [32, 64) prefetched
    Raw pre[G];
#pragma unroll
    for (int e = 0; e < G; e++) {
      Raw r0;
      fetch(s * G + e, 0, 0, 0, -1, r0);
      store(s * G + e, r0);
      fetch(32 + s * G + e, 0, 0, 0, -1, pre[e]);
    }
    __syncwarp();

    float diag = finf(), b0v = finf();
    // one step on positions 2g, 2g+1 of this segment; top0: what the segment's
    // first lane sees above its first row in the first column (the corner 0 on
    // a sentinel, +∞ otherwise; the second column is never a sentinel)
    const float pass_a = s == 0 ? 0.f : 1.f, pass_b = s == 0 ? finf() : 0.f;
    auto step = [&](int t, float top0, auto sent_tag) {
      constexpr bool SENT = decltype(sent_tag)::value;
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
      float up0, up1;
      if constexpr (SENT) {
        up0 = (s == 0) ? top0 : upv0;
        up1 = (s == 0) ? finf() : upv1;
      } else {
        // the segment's first lane sees +∞ above its first row: fma(v, 0, +∞) is
        // +∞, or NaN when v = +∞, and min3 ignores a NaN operand exactly as it
        // ignores +∞; every other lane gets fma(v, 1, 0) = v exactly.  (FMA pipe:
        // a select would take the ALU pipe, the min/max recurrence's bottleneck)
        up0 = __fmaf_rn(upv0, pass_a, pass_b);
        up1 = __fmaf_rn(upv1, pass_a, pass_b);
      }
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
    // every 16 steps: positions [2t, 2t+32) stored, the next chunk prefetched.
    // Group k + 1 is accepted (or the stream's end decided) at the first refill
    // of group k, its rows staged at the first refill after group k's window and
    // converted at the next one (H ≥ W + 32: done before group k + 1 starts).
    auto refill = [&](int t) {
      if (staging) {
        stage_finish((k + 1) & SM);
        staging = false;
      } else if (stage_due && t >= Tk + W) {
        stage_issue((k + 1) & SM);
        staging = true;
        stage_due = false;
      }
      if (!decided) {
        decided = true;
        if (look.count > 0 && look.shape == SHAPE) {
          accept(look, (k + 1) & SM);
          Tn = Tk + H;
          stage_due = true;
          seg_pop<LO, NSH>(pb, lane, look);  // the group after it, in flight
        } else {
          last = true;
        }
      }
#pragma unroll
      for (int e = 0; e < G; e++) {
        store(2 * t + s * G + e, pre[e]);
        fetch(2 * t + 32 + s * G + e, k & SM, Tk, (k + 1) & SM, last ? -1 : Tn, pre[e]);
      }
      next_refill += 16;
      __syncwarp();
    };
    const uint32_t stage_sa = (uint32_t)__cvta_generic_to_shared(&sm.stage[0][h * W * RP + s * RP]);
    float res = finf();  // the segment's last lane: result of the group before the window
    int t = 0;
    while (true) {
      const int t0 = Tk, tw = t0 + W, t1 = t0 + H;
      // step Tk: the sentinel of group k reaches lane 0 (corner value 0 above its first row)
      if (t == next_refill) refill(t);
      if (k > 0) take_rows(x, stage_sa, s == 0);
      step(t, 0.f, std::true_type{});
      ++t;
      if (k > 0) {
        // the rest of the window: lane s takes group k's rows at step Tk + s; the
        // last lane keeps its value of group k − 1 (complete before its switch)
        while (t < tw) {
          const int stop = min(next_refill, tw);
#pragma unroll 2
          for (; t < stop; ++t) {
            const int p = s == t - t0;
            res = p ? c[R - 1] : res;
            take_rows(x, stage_sa, p);
            step(t, finf(), std::false_type{});
          }
          if (t == next_refill && t < tw) refill(t);
        }
        emit((k - 1) & SM, res);
      }
      while (t < t1) {
        const int stop = min(next_refill, t1);
#pragma unroll 2
        for (; t < stop; ++t) step(t, finf(), std::false_type{});
        if (t == next_refill && t < t1) refill(t);
      }
      if (last) break;
      // the next group: its rows staged, its first positions already in the ring
      ++k;
      Tk = Tn;
      H = period(k & SM);
      Tn = -1;
      decided = false;
    }
    // drain: positions past the stream's end reach the last lanes
    for (const int total = t + W - 1; t < total; t++) {
      if (t == next_refill) refill(t);
      step(t, finf(), std::false_type{});
    }
    emit(k & SM, c[R - 1]);
    __syncwarp();
  }
};

// BIG = false: shapes 0–15 (≤ 16 rows per lane, 4 CTAs/SM); BIG = true: shapes
// 16–23 (18–32 rows per lane, 2 CTAs/SM for their registers)
template <int KIND, int D, bool INT_IN, int FIN, bool BIG>
__global__ void __launch_bounds__(kWarp* kWarpsPerCta, BIG ? 2 : 4) seg_kernel(const SegProblem pb) {
  constexpr int ROWS = BIG ? kSegRowsBig : kSegRows;
  constexpr int LO = BIG ? kSegSmallShapes : 0, NSH = BIG ? kSegShapes - kSegSmallShapes : kSegSmallShapes;
  using Sm = SegSmem<KIND, D, INT_IN, ROWS>;
  extern __shared__ uint4 seg_dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Sm& sm = reinterpret_cast<Sm*>(seg_dyn)[warp];
  for (int i = lane; i < 128 * SCfg<float, KIND, D, INT_IN>::EW; i += kWarp) sm.ring[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
  SegLook look;
  seg_pop<LO, NSH>(pb, lane, look);
  while (look.count > 0) {
#define FFD_SEG_CASE(IDX, WW, RR)                                                   \
  case IDX: {                                                                       \
    SegRunner<KIND, D, INT_IN, FIN, WW, RR, ROWS, LO, NSH> run(sm, pb, lane);       \
    run.stream(look);                                                               \
    break;                                                                          \
  }
    if constexpr (BIG) {
      switch (look.shape) {
        FFD_SEG_CASE(16, 16, 18)
        FFD_SEG_CASE(17, 16, 20)
        FFD_SEG_CASE(18, 16, 22)
        FFD_SEG_CASE(19, 16, 24)
        FFD_SEG_CASE(20, 16, 26)
        FFD_SEG_CASE(21, 16, 28)
        FFD_SEG_CASE(22, 16, 30)
        FFD_SEG_CASE(23, 16, 32)
        default:
          look.count = 0;
          break;
      }
    } else {
      switch (look.shape) {
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
          look.count = 0;
          break;
      }
    }
#undef FFD_SEG_CASE
    __syncwarp();
  }
}

// ---- host side (seg.cu, seg_*.cu) -----------------------------------------------
// launch one instantiation: a persistent grid of SMs × occupancy CTAs (cached per device)
template <int KIND, int D, bool INT_IN, int FIN, bool BIG>
cudaError_t seg_launch_one(const SegProblem& pb, int sms, cudaStream_t st) {
  auto k = seg_kernel<KIND, D, INT_IN, FIN, BIG>;
  const size_t smem = sizeof(SegSmem<KIND, D, INT_IN, BIG ? kSegRowsBig : kSegRows>) * kWarpsPerCta;
  int dev = 0;
  cudaGetDevice(&dev);
  static int occ_cache[64] = {0};
  int occ = dev < 64 ? occ_cache[dev] : 0;
  if (occ == 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarp * kWarpsPerCta, smem);
    if (occ < 1) occ = 1;
    if (dev < 64) occ_cache[dev] = occ;
  }
  k<<<sms * occ, kWarp * kWarpsPerCta, smem, st>>>(pb);
  return cudaGetLastError();
}
// big: the big kernel (shapes 16–23) first, then the small one
template <int KIND, int D, bool INT_IN, int FIN>
cudaError_t seg_launch_k(const SegProblem& pb, int sms, cudaStream_t st, bool big) {
  if (big) {
    const cudaError_t e = seg_launch_one<KIND, D, INT_IN, FIN, true>(pb, sms, st);
    if (e != cudaSuccess) return e;
  }
  return seg_launch_one<KIND, D, INT_IN, FIN, false>(pb, sms, st);
}
__host__ __device__ inline int64_t seg_max_groups(int64_t B) { return B + kSegBins + 1; }
// the seg kernel is built for this (kind, dim, int input, finalisation)
bool seg_supported(int kind, int dim, int int_in, int fin);
bool seg_big();       // rows above 256 on the big kernel (FFD_SEG_BIG=1)
cudaError_t launch_seg(const SegProblem& pb, int kind, int dim, int int_in, int fin, int sms, cudaStream_t st,
                       int64_t* launches);

}  // namespace ffd
