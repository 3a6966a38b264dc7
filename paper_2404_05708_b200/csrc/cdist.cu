// cdist.cu — all-pairs discrete Fréchet distances between two dense curve sets.
//
// out[a - row_begin][b] = δ_dF(A_a, B_b) (PAPER Eq. (1), evaluated as
// in strip.cuh).  B200 design (DESIGN.md §"cdist kernel"):
//   * A warp is split into 32/W segments of W lanes; each segment keeps one
//     A-curve (the rows, ≤ W·R points) in registers for the whole work item —
//     rows are loaded once, never reloaded.  Lane s of a segment owns rows
//     [sR, sR+R) and processes column t − s at step t; boundary values move
//     down the segment with __shfl_up_sync(width = W).
//   * All segments of a warp stream the same tile of B curves through a
//     per-warp shared-memory ring (each element read with a broadcast LDS):
//     [sentinel, B_b0 points, sentinel, B_b0+1 points, …, sentinel].  The
//     sentinel column (+inf) resets the DP between B curves; the top lane of
//     each segment sees the corner value 0 at the sentinel.
//   * All B curves have the same length, so the stream is periodic with
//     period P = lenB + 1: the step at which a segment's last lane holds a
//     finished δ is known to the whole warp, and the results are stored with
//     one predicated store per period (no per-lane event checks).
//   * Work items (4 A-curves × a tile of B curves) are popped dynamically by
//     persistent warps; a rank's shard is a contiguous row range of A.
#include <climits>

#include <cstdio>
#include <cstdlib>

#include "cdist.cuh"
#include "ffd.h"
#include "strip.cuh"

namespace ffd {

constexpr int kCdTile = 128;  // B curves per work item

struct CdistProblem {
  const float* A;
  const float* B;
  int64_t nA, nB;
  int lenA, lenB;
  int64_t row_begin, row_end;
  OutSpec dst;
  int* counter;
  int64_t n_items;
  int64_t tiles_b;
  int self;  // B is A (ffd_cdist_self): evaluate each unordered pair once inside the shard
};

// one result to every destination (local matrix and/or NVLink peer matrices)
__device__ __forceinline__ void put_result(const OutSpec& d, int64_t row, int64_t col, float v) {
#pragma unroll 1
  for (int i = 0; i < d.n; i++)
    reinterpret_cast<float*>(d.out[i])[(row - d.row_base) * d.ld + col] = v;
}

constexpr int kCdMinCtasPerSm = 4;  // 128 registers/thread: the W=8, R=16 shape needs ~100
                                    // (R = 32 shapes: 3 CTAs/SM, 168 registers)

template <int KIND, int D, int W, int R, int FIN>
__global__ void __launch_bounds__(kWarp* kWarpsPerCta, (R > 16) ? 3 : kCdMinCtasPerSm)
    cdist_kernel(const CdistProblem pb) {
  using C = SCfg<float, KIND, D, false>;
  static_assert(!C::XSQ, "cdist: fp32 inputs");
  constexpr int SEG = kWarp / W;
  constexpr int EW = C::EW;
  __shared__ uint4 ring_all[kWarpsPerCta][kRing * EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = lane % W;        // lane index inside the segment
  const int seg = lane / W;      // segment index inside the warp
  uint4* ring = ring_all[warp];
  const int P = pb.lenB + 1;     // stream period

  while (true) {
    int64_t item = 0;
    if (lane == 0) item = atomicAdd(pb.counter, 1);
    item = __shfl_sync(0xffffffffu, (long long)item, 0);
    if (item >= pb.n_items) break;
    const int64_t ablk = item / pb.tiles_b;
    const int64_t tb = item % pb.tiles_b;
    const int64_t a = pb.row_begin + ablk * SEG + seg;        // this segment's A curve
    const bool a_ok = a < pb.row_end;
    const int64_t b0 = tb * kCdTile;
    const int nb = (int)min((int64_t)kCdTile, pb.nB - b0);
    if (pb.self) {
      // every (a, b) of this item has b < a with b inside the shard: it is written
      // by the mirror of (b, a) — skip the whole item (δ is symmetric)
      const int64_t a_first = pb.row_begin + ablk * SEG;
      const int64_t bb0 = pb.dst.col_off + b0;  // B index → A index
      if (bb0 + nb <= a_first && bb0 >= pb.row_begin) continue;
    }
    const int S = nb * P + 1;                                  // stream positions

    // rows of this segment's A curve (padded by repeating the last point)
    float x[C::NS][R];
    {
      const float* ap = pb.A + (a_ok ? a : pb.row_begin) * (int64_t)pb.lenA * D;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int row = min(s * R + r, pb.lenA - 1);
#pragma unroll
        for (int c = 0; c < D; c++) x[c][r] = __ldg(ap + (int64_t)row * D + c);
      }
    }
    // column element loader: position pos -> sentinel or B point
    const float* bbase = pb.B + b0 * (int64_t)pb.lenB * D;
    auto load_pt = [&](int pos, float (&v)[D]) {
      if (pos < S) {
        const int b = pos / P, k = pos - b * P;
        if (k == 0) {
#pragma unroll
          for (int c = 0; c < D; c++) v[c] = finf();
        } else {
          const float* bp = bbase + ((int64_t)b * pb.lenB + (k - 1)) * D;
#pragma unroll
          for (int c = 0; c < D; c++) v[c] = __ldg(bp + c);
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) v[c] = finf();
      }
    };
    auto store_el = [&](int pos, const float (&v)[D]) {
      alignas(16) float e[C::EBYTES / 4];
#pragma unroll
      for (int i = 0; i < C::EBYTES / 4; i++) e[i] = 0.f;
#pragma unroll
      for (int c = 0; c < D; c++) e[c] = v[c];
      uint4* dst = ring + (pos & kRingMask) * EW;
#pragma unroll
      for (int w = 0; w < EW; w++) dst[w] = reinterpret_cast<const uint4*>(e)[w];
    };
    float pre[D];
    {
      float v0[D];
      load_pt(lane, v0);
      store_el(lane, v0);
      load_pt(32 + lane, pre);
    }
    __syncwarp();

    float c[R];
#pragma unroll
    for (int r = 0; r < R; r++) c[r] = finf();
    float diag = finf();
    // one step: element, boundary value from the lane above, R cells.  `top` is
    // what the segment's first lane sees above its first row: the corner value
    // 0 on a sentinel column (t ≡ 0 mod P), +inf otherwise.
    auto step = [&](int t, float top) {
      const int g = t - s;
      alignas(16) float e[C::EBYTES / 4];
      {
        const uint4* src = ring + (g & kRingMask) * EW;
#pragma unroll
        for (int w = 0; w < EW; w++) reinterpret_cast<uint4*>(e)[w] = src[w];
      }
      const float upv = __shfl_up_sync(0xffffffffu, c[R - 1], 1, W);
      const float up = (s == 0) ? top : upv;
      float dist[R];
      cell_dists<float, KIND, D, R, false>(x, e, dist);
      float u = up, dg = diag;
      diag = up;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const float m = fminf(fminf(u, dg), c[r]);
        const float nv = fmaxf(m, dist[r]);
        dg = c[r];
        c[r] = nv;
        u = nv;
      }
    };
    const int total = S + W - 1;
    int next_out = P + W - 1;  // segment-last lanes enter the sentinel after B curve out_b
    int out_b = 0;
    int next_refill = 32;
    int next_sent = 0;         // segment-first lanes on a sentinel column
    int t = 0;
    while (t < total) {
      const int stop = min(min(min(next_refill, next_out), next_sent), total);
#pragma unroll 2
      for (; t < stop; ++t) step(t, finf());
      if (t >= total) break;
      if (t == next_refill) {
        store_el(t + lane, pre);
        load_pt(t + 32 + lane, pre);
        next_refill += 32;
        __syncwarp();
      }
      if (t == next_out) {
        // segment-last lanes hold δ(A_a, B_{b0+out_b}): column P·(out_b+1) − 1 is done
        if (s == W - 1 && a_ok) {
          float v = c[R - 1];
          if constexpr (FIN == F_SQRT) v = sqrt_result(v);
          const int64_t b = pb.dst.col_off + b0 + out_b;  // column of the result
          const bool in_shard = pb.self && b >= pb.row_begin && b < pb.row_end;
          // self mode: (a, b) with b < a inside the shard is the mirror's job
          if (!(in_shard && b < a)) put_result(pb.dst, a, b, v);
          if ((in_shard && b > a) || (pb.dst.mirror && !pb.self)) put_result(pb.dst, b, a, v);
        }
        ++out_b;
        next_out += P;
      }
      if (t == next_sent) {
        step(t, 0.f);
        ++t;
        next_sent += P;
      }
    }
    __syncwarp();
  }
  // results stored into NVLink peers' matrices: order them before whatever the
  // host sequences after this kernel (the barrier that publishes the matrix)
  if (pb.dst.n > 1) __threadfence_system();
}

// ---- two columns per step ------------------------------------------------------
// The same work items with each segment lane processing positions 2(t−s) and
// 2(t−s)+1 per step (strip.cuh step2_compute): the second column's min/max chain
// trails the first by one row, so the two chains interleave and the shuffle +
// chain latency is paid once per two columns.  Every B curve's stream segment
// is padded to an even period P2 = sentinel + lenB columns (+ one more copy of
// the last column when lenB + 1 is odd: a repeated point leaves δ unchanged,
// PAPER L259 footnote), so a sentinel is always a step's first column and a
// curve's last column a step's second: the corner value and the result need no
// per-column case.  Unlike the batch kernel there are no transition windows
// (the A curve of a segment is fixed for the item), so nothing pays for the
// longer step.
template <int KIND, int D, int W, int R, int FIN>
__global__ void __launch_bounds__(kWarp* kWarpsPerCta, (R > 16) ? 3 : kCdMinCtasPerSm)
    cdist_kernel2(const CdistProblem pb) {
  using C = SCfg<float, KIND, D, false>;
  static_assert(!C::XSQ, "cdist: fp32 inputs");
  constexpr int SEG = kWarp / W;
  constexpr int EW = C::EW;
  __shared__ uint4 ring_all[kWarpsPerCta][kRing * EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = lane % W;        // lane index inside the segment
  const int seg = lane / W;      // segment index inside the warp
  uint4* ring = ring_all[warp];
  const int P2 = (pb.lenB + 2) & ~1;  // even stream period
  const int H = P2 >> 1;              // steps per period

  while (true) {
    int64_t item = 0;
    if (lane == 0) item = atomicAdd(pb.counter, 1);
    item = __shfl_sync(0xffffffffu, (long long)item, 0);
    if (item >= pb.n_items) break;
    const int64_t ablk = item / pb.tiles_b;
    const int64_t tb = item % pb.tiles_b;
    const int64_t a = pb.row_begin + ablk * SEG + seg;
    const bool a_ok = a < pb.row_end;
    const int64_t b0 = tb * kCdTile;
    const int nb = (int)min((int64_t)kCdTile, pb.nB - b0);
    if (pb.self) {
      const int64_t a_first = pb.row_begin + ablk * SEG;
      const int64_t bb0 = pb.dst.col_off + b0;
      if (bb0 + nb <= a_first && bb0 >= pb.row_begin) continue;
    }
    const int S = nb * P2 + 2;  // positions: the periods, then a final sentinel and one more

    float x[C::NS][R];
    {
      const float* ap = pb.A + (a_ok ? a : pb.row_begin) * (int64_t)pb.lenA * D;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const int row = min(s * R + r, pb.lenA - 1);
#pragma unroll
        for (int c = 0; c < D; c++) x[c][r] = __ldg(ap + (int64_t)row * D + c);
      }
    }
    const float* bbase = pb.B + b0 * (int64_t)pb.lenB * D;
    auto load_pt = [&](int pos, float (&v)[D]) {
      const int b = pos / P2, k = pos - b * P2;
      if (pos < S - 2 && k != 0) {
        const float* bp = bbase + ((int64_t)b * pb.lenB + min(k - 1, pb.lenB - 1)) * D;
#pragma unroll
        for (int c = 0; c < D; c++) v[c] = __ldg(bp + c);
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) v[c] = finf();
      }
    };
    auto store_el = [&](int pos, const float (&v)[D]) {
      alignas(16) float e[C::EBYTES / 4];
#pragma unroll
      for (int i = 0; i < C::EBYTES / 4; i++) e[i] = 0.f;
#pragma unroll
      for (int c = 0; c < D; c++) e[c] = v[c];
      uint4* dst = ring + (pos & kRingMask) * EW;
#pragma unroll
      for (int w = 0; w < EW; w++) dst[w] = reinterpret_cast<const uint4*>(e)[w];
    };
    float pre[D];
    {
      float v0[D];
      load_pt(lane, v0);
      store_el(lane, v0);
      load_pt(32 + lane, pre);
    }
    __syncwarp();

    float c[R];
#pragma unroll
    for (int r = 0; r < R; r++) c[r] = finf();
    float diag = finf(), b0v = finf();
    // one step on positions 2g, 2g+1; `top0` is what the segment's first lane sees
    // above its first row in the first column: the corner 0 on a sentinel (t ≡ 0
    // mod H), +∞ otherwise (the second column is never a sentinel)
    auto step = [&](int t, float top0) {
      const int g = t - s;
      alignas(16) float e0[C::EBYTES / 4], e1[C::EBYTES / 4];
      {
        const uint4* src = ring + ((2 * g) & kRingMask) * EW;
#pragma unroll
        for (int w = 0; w < EW; w++) {
          reinterpret_cast<uint4*>(e0)[w] = src[w];
          reinterpret_cast<uint4*>(e1)[w] = src[EW + w];
        }
      }
      const float upv0 = __shfl_up_sync(0xffffffffu, b0v, 1, W);
      const float upv1 = __shfl_up_sync(0xffffffffu, c[R - 1], 1, W);
      const float up0 = (s == 0) ? top0 : upv0;
      const float up1 = (s == 0) ? finf() : upv1;
      float d0[R], d1[R];
      cell_dists<float, KIND, D, R, false>(x, e0, d0);
      cell_dists<float, KIND, D, R, false>(x, e1, d1);
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
    const int total = (S >> 1) + W - 1;
    int next_out = H + W - 1;  // segment-last lanes have finished B curve out_b (after step next_out − 1)
    int out_b = 0;
    int next_refill = 16;      // 32 positions per refill
    int next_sent = 0;         // segment-first lanes on a sentinel step
    int t = 0;
    while (t < total) {
      const int stop = min(min(min(next_refill, next_out), next_sent), total);
#pragma unroll 2
      for (; t < stop; ++t) step(t, finf());
      if (t >= total) break;
      if (t == next_refill) {
        store_el(2 * t + lane, pre);
        load_pt(2 * t + 32 + lane, pre);
        next_refill += 16;
        __syncwarp();
      }
      if (t == next_out) {
        if (s == W - 1 && a_ok && out_b < nb) {
          float v = c[R - 1];
          if constexpr (FIN == F_SQRT) v = sqrt_result(v);
          const int64_t b = pb.dst.col_off + b0 + out_b;
          const bool in_shard = pb.self && b >= pb.row_begin && b < pb.row_end;
          if (!(in_shard && b < a)) put_result(pb.dst, a, b, v);
          if ((in_shard && b > a) || (pb.dst.mirror && !pb.self)) put_result(pb.dst, b, a, v);
        }
        ++out_b;
        next_out += H;
      }
      if (t == next_sent) {
        step(t, 0.f);
        ++t;
        next_sent += H;
      }
    }
    __syncwarp();
  }
  if (pb.dst.n > 1) __threadfence_system();
}

// ---- dispatch ----------------------------------------------------------------
#ifndef FFD_CDIST_COLS
#define FFD_CDIST_COLS 2
#endif
template <int KIND, int D, int W, int R, int FIN>
static cudaError_t launch_one(const CdistProblem& pb, int sms, cudaStream_t st) {
  // columns per step: FFD_CDIST_COLS at build time, overridable by the environment (testing)
  static const int cols = getenv("FFD_CDIST_COLS") ? atoi(getenv("FFD_CDIST_COLS")) : FFD_CDIST_COLS;
  auto k = cols == 2 ? cdist_kernel2<KIND, D, W, R, FIN> : cdist_kernel<KIND, D, W, R, FIN>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarp * kWarpsPerCta, 0);
  if (occ < 1) occ = 1;
  k<<<sms * occ, kWarp * kWarpsPerCta, 0, st>>>(pb);
  return cudaGetLastError();
}

// shapes: (W, R) with W·R ≥ lenA; pick the first (smallest capacity) in pick_shape's order
template <int KIND, int D, int FIN>
static cudaError_t launch_shape(const CdistProblem& pb, int sms, cudaStream_t st, int W, int R) {
#define FFD_CD(WW, RR) \
  if (W == WW && R == RR) return launch_one<KIND, D, WW, RR, FIN>(pb, sms, st);
  FFD_CD(8, 4) FFD_CD(8, 8) FFD_CD(8, 16) FFD_CD(16, 12) FFD_CD(16, 16) FFD_CD(32, 12)
  FFD_CD(32, 16) FFD_CD(4, 32)
#undef FFD_CD
  return cudaErrorInvalidValue;
}

// (4, 32) before (8, 16): the same 128 rows with twice the rows per lane halves
// the per-step shuffle/select/load overhead per cell; at 3 CTAs/SM (168
// registers) config 4 runs at 5.50 against 5.26 T cells/s
static void pick_shape(int rows, int& W, int& R) {
  static const int shapes[][2] = {{8, 4}, {8, 8}, {4, 32}, {8, 16}, {16, 12}, {16, 16}, {32, 12}, {32, 16}};
  for (auto& sh : shapes)
    if (sh[0] * sh[1] >= rows) {
      W = sh[0];
      R = sh[1];
      return;
    }
  W = 0;
  R = 0;
}

size_t cdist_workspace_bytes() { return 256; }

int launch_cdist(const CdistArgs& a, int sms, cudaStream_t st, int64_t* launches) {
  if (a.dtype != FFD_F32) return FFD_ERR_UNSUPPORTED;
  if (a.dim != 2 && a.dim != 3) return FFD_ERR_UNSUPPORTED;
  int W = 0, R = 0;
  pick_shape(a.lenA, W, R);
  if (const char* env = getenv("FFD_CDIST_SHAPE")) {  // testing: force a built "W,R" shape
    int w = 0, r = 0;
    if (sscanf(env, "%d,%d", &w, &r) == 2 && w * r >= a.lenA) W = w, R = r;
  }
  if (!W) return FFD_ERR_UNSUPPORTED;  // rows longer than one warp band
  if ((int64_t)a.lenB + 1 > INT_MAX / (kCdTile + 1)) return FFD_ERR_UNSUPPORTED;
  CdistProblem pb{};
  pb.A = reinterpret_cast<const float*>(a.A);
  pb.B = reinterpret_cast<const float*>(a.B);
  pb.nA = a.nA;
  pb.nB = a.nB;
  pb.lenA = a.lenA;
  pb.lenB = a.lenB;
  pb.row_begin = a.row_begin;
  pb.row_end = a.row_end;
  pb.dst = a.dst;
  pb.counter = reinterpret_cast<int*>(a.workspace);
  pb.self = a.self;
  const int seg = kWarp / W;
  const int64_t rows = a.row_end - a.row_begin;
  pb.tiles_b = (a.nB + kCdTile - 1) / kCdTile;
  pb.n_items = ((rows + seg - 1) / seg) * pb.tiles_b;
  if (pb.n_items > INT_MAX) return FFD_ERR_UNSUPPORTED;
  if (cudaMemsetAsync(pb.counter, 0, sizeof(int), st) != cudaSuccess) return FFD_ERR_CUDA;
  cudaError_t e = cudaErrorInvalidValue;
  const int kind = a.norm == FFD_L1 ? K_L1 : (a.norm == FFD_LINF ? K_LINF : K_SQ);
  const bool sq = (a.norm == FFD_L2);
  if (a.dim == 2) {
    if (kind == K_SQ) e = sq ? launch_shape<K_SQ, 2, F_SQRT>(pb, sms, st, W, R)
                             : launch_shape<K_SQ, 2, F_NONE>(pb, sms, st, W, R);
    else if (kind == K_L1) e = launch_shape<K_L1, 2, F_NONE>(pb, sms, st, W, R);
    else e = launch_shape<K_LINF, 2, F_NONE>(pb, sms, st, W, R);
  } else {
    if (kind == K_SQ) e = sq ? launch_shape<K_SQ, 3, F_SQRT>(pb, sms, st, W, R)
                             : launch_shape<K_SQ, 3, F_NONE>(pb, sms, st, W, R);
    else if (kind == K_L1) e = launch_shape<K_L1, 3, F_NONE>(pb, sms, st, W, R);
    else e = launch_shape<K_LINF, 3, F_NONE>(pb, sms, st, W, R);
  }
  ++*launches;
  return e == cudaSuccess ? FFD_OK : FFD_ERR_CUDA;
}

}  // namespace ffd
