// longpair.cu — one very long pair spread over the whole GPU.
//
// What: δ_dF of a pair with n rows (shorter curve) and m columns, Eq. (1)
// (PAPER L159–L163), linear memory (Theorem 1): every warp keeps only
// its strip of rows and one column of DP state in registers.
//
// How (DESIGN.md §"long-pair kernel"):
//   * The rows are cut into bands of 32·R rows; band b runs on one warp as the
//     lane-strip wavefront of strip.cuh (lane ℓ: rows [ℓR, ℓR+R), column t−ℓ at
//     step t), streaming all m columns once.
//   * Band b's bottom row (lane 31's value, one per column) is the top input
//     of band b+1.  Inside a CTA of 8 warps (8 consecutive bands) it moves
//     through shared-memory rings; between CTAs through global-memory rings
//     (L2) with release/acquire progress counters.  Both rings are bounded
//     buffers with flow control (the consumer publishes how far it has read).
//   * The consumer copies top values into its column ring 8 columns at a time,
//     so consecutive bands run ≈ 8 + 31 steps apart (+ the L2 hop between CTAs).
//   * One persistent CTA per SM, cooperative launch (all CTAs co-resident, so
//     spinning on another CTA's progress cannot deadlock); bands beyond one
//     wave are processed in rounds, and progress counters are absolute stream
//     positions, so rounds and successive pairs need no grid barrier.
#include <climits>
#include <cstdlib>

#include "ffd.h"
#include "longpair.cuh"
#include "strip.cuh"

namespace ffd {

constexpr int kLWarps = 8;        // warps (bands) per CTA
constexpr int kLSmemRing = 256;   // shared link ring (floats)
constexpr int kLGlobRing = 4096;  // global link ring (floats) per CTA slot
constexpr int kTopChunk = 8;      // top values copied per refill
constexpr int kMaxLongCtas = 1024;

struct LongProblem {
  const void* p;
  const void* q;
  const int64_t* offsets;
  const int32_t* lengths;
  int64_t num_pairs;
  const int* list;
  const int* list_count;
  void* out;
  float* gring;        // [G][kLGlobRing]
  long long* gprod;    // [G] absolute positions published by CTA slot's last band
  long long* gcons;    // [G] absolute positions consumed from CTA slot's link
  int* bad;            // per long pair: left the fp32-exact window (int input)
};

__device__ __forceinline__ long long ld_acquire(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int KIND, int D, bool INT_IN, int FIN, int R>
struct LongRunner {
  using T = float;
  using C = SCfg<T, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  static constexpr int NS = C::NS;

  uint4* ring;                 // this warp's column ring [kRing * EW]
  float* slink;                // shared link rings [kLWarps][kLSmemRing]
  volatile int* sprod;         // [kLWarps] positions published into slink[w]
  volatile int* scons;         // [kLWarps] positions consumed from slink[w]
  const LongProblem& pb;
  int lane, warp;

  // ---- pair description --------------------------------------------------
  const In* rows;
  const In* cols;
  int n, m;
  int center[D];

  __device__ bool conv(const In (&a)[D], float (&v)[D]) const {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < D; c++) {
      if constexpr (INT_IN) {
        long long t = (long long)a[c] - center[c];
        ok &= (t >= -C::LIM) && (t <= C::LIM);
        v[c] = (float)(int)t;
      } else {
        v[c] = a[c];
      }
    }
    return ok;
  }

  // coordinates of column element `pos` (0 = sentinel) written without its top field
  __device__ void store_coords(const In (&a)[D], int kind, int pos, bool& ok) {
    float f[C::EBYTES / 4];
#pragma unroll
    for (int i = 0; i < C::EBYTES / 4; i++) f[i] = 0.f;
    if (kind != 0) {
      if constexpr (C::XSQ) {
        f[D] = finf();
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) f[c] = finf();
      }
    } else {
      float v[D];
      ok &= conv(a, v);
      if constexpr (C::XSQ) {
        int qq = 0;
#pragma unroll
        for (int c = 0; c < D; c++) {
          qq += (int)v[c] * (int)v[c];
          f[c] = -2.f * v[c];
        }
        f[D] = (float)qq;
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) f[c] = v[c];
      }
    }
    float* dst = reinterpret_cast<float*>(ring + (pos & kRingMask) * C::EW);
#pragma unroll
    for (int i = 0; i < C::EBYTES / 4; i++)
      if (i != C::I_TOP) dst[i] = f[i];
  }

  __device__ void fetch(int pos, int S, In (&a)[D], int& kind) const {
#pragma unroll
    for (int c = 0; c < D; c++) a[c] = (In)0;
    if (pos >= S) {
      kind = 2;
    } else if (pos == 0) {
      kind = 1;
    } else {
      kind = 0;
#pragma unroll
      for (int c = 0; c < D; c++) a[c] = __ldg(cols + (int64_t)(pos - 1) * D + c);
    }
  }

  // one band of 32·R rows starting at row r0; top: 0 sentinel-derived, 1 shared, 2 global
  __device__ bool run_band(int r0, int top_kind, int bot_kind, long long gbase_in, int gslot_in,
                           long long gbase_out, int gslot_out, bool last_band, int out_idx,
                           int* bad_flag) {
    const int S = m + 1;
    bool ok = true;
    float x[NS][R], c[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int row = min(r0 + lane * R + r, n - 1);
      In a[D];
#pragma unroll
      for (int cc = 0; cc < D; cc++) a[cc] = __ldg(rows + (int64_t)row * D + cc);
      float v[D];
      ok &= conv(a, v);
#pragma unroll
      for (int cc = 0; cc < D; cc++) x[cc][r] = v[cc];
      if constexpr (C::XSQ) {
        int pp = 0;
#pragma unroll
        for (int cc = 0; cc < D; cc++) pp += (int)v[cc] * (int)v[cc];
        x[D][r] = (float)pp;
      }
      c[r] = finf();
    }
    if constexpr (INT_IN) {
      if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicExch(bad_flag, 1);
    }
    float diag = finf();
    float* top_f = reinterpret_cast<float*>(ring);
    // column prologue: positions [0,32) stored, [32,64) prefetched
    In a[D];
    int kind;
    fetch(lane, S, a, kind);
    store_coords(a, kind, lane, ok);
    fetch(32 + lane, S, a, kind);
    int next_refill = 32, next_top = 0;
    const float* sl_in = slink + (warp - 1) * kLSmemRing;     // valid when top_kind == 1
    float* sl_out = slink + warp * kLSmemRing;                 // valid when bot_kind == 1
    float* gr_in = pb.gring + (size_t)gslot_in * kLGlobRing;
    float* gr_out = pb.gring + (size_t)gslot_out * kLGlobRing;
    long long published = 0;  // positions published by this band (relative)
    long long cons_seen = 0;  // consumer progress seen (relative), for flow control
    __syncwarp();

    const int total = S + 31;
    int t = 0;
    while (t < total) {
      // -- top values for positions [t, t+8) (lanes 0..7), before lane 0 needs them
      if (t == next_top) {
        const int need = min(t + kTopChunk, S);
        if (top_kind == 1) {
          if (lane == 0)
            while (sprod[warp - 1] < need) __nanosleep(32);
          __syncwarp();
          __threadfence_block();
        } else if (top_kind == 2) {
          if (lane == 0)
            while (ld_acquire(pb.gprod + gslot_in) < gbase_in + need) __nanosleep(64);
          __syncwarp();
        }
        if (lane < kTopChunk && t + lane < S + kTopChunk) {
          const int pos = t + lane;
          float tv;
          if (top_kind == 0) tv = (pos == 0) ? 0.f : finf();
          else if (pos >= S) tv = finf();
          else if (top_kind == 1) tv = sl_in[pos % kLSmemRing];
          else tv = __ldcg(gr_in + (gbase_in + pos) % kLGlobRing);
          top_f[(pos & kRingMask) * C::EW * 4 + C::I_TOP] = tv;
        }
        __syncwarp();
        if (lane == 0) {
          if (top_kind == 1) {
            __threadfence_block();
            scons[warp - 1] = need;
          } else if (top_kind == 2) {
            st_release(pb.gcons + gslot_in, gbase_in + need);
          }
        }
        next_top += kTopChunk;
      }
      // -- flow control for the bottom-row ring: positions up to t-31+8 will be written
      if (bot_kind != 0 && (t & (kTopChunk - 1)) == 0) {
        const long long hi = (long long)(t - 31 + kTopChunk);
        const int ringsz = bot_kind == 1 ? kLSmemRing : kLGlobRing;
        if (hi > cons_seen + ringsz) {
          if (lane == 31) {
            if (bot_kind == 1) {
              while (scons[warp] + ringsz < hi) __nanosleep(32);
            } else {
              while (ld_acquire(pb.gcons + gslot_out) - gbase_out + ringsz < hi) __nanosleep(64);
            }
          }
          __syncwarp();
          cons_seen = hi - ringsz;
        }
      }
      if (t == next_refill) {
        store_coords(a, kind, t + lane, ok);
        fetch(t + 32 + lane, S, a, kind);
        next_refill += 32;
      }
      __syncwarp();
      const int stop = min(min(next_refill, next_top), total);
      int g = t - lane;
#pragma unroll 1
      for (; t < stop; ++t, ++g) {
        warp_step<float, KIND, D, R, INT_IN>(c, diag, x, ring, g, lane);
        if (bot_kind != 0 && lane == 31 && g >= 0 && g < S) {
          if (bot_kind == 1) sl_out[g % kLSmemRing] = c[R - 1];
          else __stcg(gr_out + (gbase_out + g) % kLGlobRing, c[R - 1]);
        }
      }
      // -- publish the bottom row every 8 steps (positions complete: g+1 of lane 31)
      if (bot_kind != 0 && (t & (kTopChunk - 1)) == 0) {
        const long long done = min((long long)(t - 31), (long long)S);
        if (done > published) {
          if (lane == 31) {
            if (bot_kind == 1) {
              __threadfence_block();
              sprod[warp] = (int)done;
            } else {
              __threadfence();
              st_release(pb.gprod + gslot_out, gbase_out + done);
            }
          }
          published = done;
        }
      }
    }
    // final publish (all S positions)
    if (bot_kind != 0 && lane == 31) {
      if (bot_kind == 1) {
        __threadfence_block();
        sprod[warp] = S;
      } else {
        __threadfence();
        st_release(pb.gprod + gslot_out, gbase_out + S);
      }
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    if (last_band && lane == 31) {
      if constexpr (INT_IN) {
        __threadfence();
        const bool bad = !all_ok || *reinterpret_cast<volatile int*>(bad_flag) != 0;
        reinterpret_cast<long long*>(pb.out)[out_idx] = bad ? LLONG_MIN : (long long)c[R - 1];
      } else {
        float f = c[R - 1];
        if constexpr (FIN == F_SQRT) f = __fsqrt_rn(f);
        reinterpret_cast<float*>(pb.out)[out_idx] = f;
      }
    }
    __syncwarp();
    return all_ok;
  }
};

// Every band of a pair must be resident at once (bounded link rings + a band
// waiting on the next one would otherwise form a cycle), so the rows per lane
// R ∈ {8, 16, 32} are chosen per pair such that ⌈bands / 8⌉ ≤ CTAs; a pair
// whose shorter curve exceeds 8·32·32·CTAs points (≈1.2M on 148 SMs) gets the
// invalid value (NaN / INT64_MIN) and is reported by ffd_validate_batch users.
template <int KIND, int D, bool INT_IN, int FIN>
__global__ void __launch_bounds__(kWarp* kLWarps, 1) long_kernel(const LongProblem pb) {
  using C = SCfg<float, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  __shared__ uint4 rings[kLWarps][kRing * C::EW];
  __shared__ float slink[kLWarps * kLSmemRing];
  __shared__ int sprod[kLWarps], scons[kLWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  LongRunner<KIND, D, INT_IN, FIN, 8> run8{rings[warp], slink, sprod, scons, pb, lane, warp};
  LongRunner<KIND, D, INT_IN, FIN, 16> run16{rings[warp], slink, sprod, scons, pb, lane, warp};
  LongRunner<KIND, D, INT_IN, FIN, 32> run32{rings[warp], slink, sprod, scons, pb, lane, warp};
  const int npairs = *pb.list_count;
  long long base = 0;  // absolute stream position of the current pair on every global link
  for (int li = 0; li < npairs; li++) {
    const int k = pb.list[li];
    const int64_t B = pb.num_pairs;
    const int n0 = pb.lengths[k], m0 = pb.lengths[B + k];
    const bool swap = n0 > m0;
    const int n = swap ? m0 : n0, m = swap ? n0 : m0;
    const In* rows = reinterpret_cast<const In*>(swap ? pb.q : pb.p) +
                     (swap ? pb.offsets[B + k] : pb.offsets[k]) * D;
    const In* cols = reinterpret_cast<const In*>(swap ? pb.p : pb.q) +
                     (swap ? pb.offsets[k] : pb.offsets[B + k]) * D;
    int R = 0;
    for (int rr = 8; rr <= 32; rr *= 2) {
      const int nb = (n + kWarp * rr - 1) / (kWarp * rr);
      if ((nb + kLWarps - 1) / kLWarps <= G) {
        R = rr;
        break;
      }
    }
    const int S = m + 1;
    if (R == 0) {
      if (cta == 0 && threadIdx.x == 0) {
        if constexpr (INT_IN) reinterpret_cast<long long*>(pb.out)[k] = LLONG_MIN;
        else reinterpret_cast<float*>(pb.out)[k] = __int_as_float(0x7fc00000);
      }
      continue;
    }
    const int band_rows = kWarp * R;
    const int nb = (n + band_rows - 1) / band_rows;
    if (threadIdx.x < kLWarps) {
      sprod[threadIdx.x] = 0;
      scons[threadIdx.x] = 0;
    }
    __syncthreads();
    const int b = cta * kLWarps + warp;
    if (b < nb) {
      int top_kind = 0, gslot_in = (cta + G - 1) % G;
      if (b > 0) top_kind = (warp > 0) ? 1 : 2;
      int bot_kind = 0;
      if (b + 1 < nb) bot_kind = (warp < kLWarps - 1) ? 1 : 2;
      auto go = [&](auto& run) {
        run.n = n;
        run.m = m;
        run.rows = rows;
        run.cols = cols;
        if constexpr (INT_IN) {
#pragma unroll
          for (int c = 0; c < D; c++) run.center[c] = (int)rows[c];
        }
        run.run_band(b * band_rows, top_kind, bot_kind, base, gslot_in, base, cta, b == nb - 1, k,
                     pb.bad + li);
      };
      if (R == 8) go(run8);
      else if (R == 16) go(run16);
      else go(run32);
    }
    __syncthreads();
    base += S;  // every link's absolute position advances by one stream per pair
  }
}

// ---- host dispatch ---------------------------------------------------------------
struct LongWs {
  float* gring;
  long long* gprod;
  long long* gcons;
  int* bad;
};

// One persistent CTA (8 bands) per SM.  BASELINE config 5 (n = 262,144) runs as
// 128 CTAs of 8 bands × 256 rows (R = 8).  One instantiation per (kind, dim, input).
template <int KIND, int D, bool INT_IN, int FIN>
static cudaError_t launch_long_k(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w) {
  auto k = long_kernel<KIND, D, INT_IN, FIN>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarp * kLWarps, 0);
  if (occ < 1) return cudaErrorLaunchOutOfResources;
  int G = sms;
  if (const char* env = getenv("FFD_LONG_CTAS")) {  // testing: fewer CTAs -> larger R
    const int g = atoi(env);
    if (g > 0 && g < G) G = g;
  }
  if (G > kMaxLongCtas) G = kMaxLongCtas;
  LongProblem pb{a.p, a.q, a.offsets, a.lengths, a.num_pairs, a.list, a.list_count, a.out,
                 w.gring, w.gprod, w.gcons, w.bad};
  void* args[] = {&pb};
  return cudaLaunchCooperativeKernel((const void*)k, dim3(G), dim3(kWarp * kLWarps), args, 0, st);
}

cudaError_t launch_long_pairs(const LongArgs& a, int sms, cudaStream_t st, int64_t* launches) {
  // workspace (stream-ordered, pooled): global link rings + counters, zeroed
  const size_t ring_b = (size_t)kMaxLongCtas * kLGlobRing * sizeof(float);
  const size_t ctr_b = (size_t)kMaxLongCtas * sizeof(long long);
  const size_t bad_b = (size_t)(a.num_pairs > 0 ? a.num_pairs : 1) * sizeof(int);
  const size_t total = ring_b + 2 * ctr_b + bad_b;
  char* buf = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), total, st);
  if (e != cudaSuccess) return e;
  LongWs w{reinterpret_cast<float*>(buf), reinterpret_cast<long long*>(buf + ring_b),
           reinterpret_cast<long long*>(buf + ring_b + ctr_b),
           reinterpret_cast<int*>(buf + ring_b + 2 * ctr_b)};
  e = cudaMemsetAsync(buf + ring_b, 0, 2 * ctr_b + bad_b, st);
  if (e == cudaSuccess) {
    const bool i = a.dtype == FFD_I32;
    const int kind = i ? (a.norm == FFD_SQL2 ? K_XSQ : (a.norm == FFD_L1 ? K_L1 : K_LINF))
                       : (a.norm == FFD_L1 ? K_L1 : (a.norm == FFD_LINF ? K_LINF : K_SQ));
    const bool sq = a.norm == FFD_L2;
    e = cudaErrorInvalidValue;
#define FFD_LONG_F(DD)                                                                  \
  if (a.dim == DD) {                                                                    \
    if (!i && kind == K_SQ) e = sq ? launch_long_k<K_SQ, DD, false, F_SQRT>(a, sms, st, w) \
                                   : launch_long_k<K_SQ, DD, false, F_NONE>(a, sms, st, w); \
    else if (!i && kind == K_L1) e = launch_long_k<K_L1, DD, false, F_NONE>(a, sms, st, w); \
    else if (!i && kind == K_LINF) e = launch_long_k<K_LINF, DD, false, F_NONE>(a, sms, st, w); \
    else if (i && kind == K_XSQ) e = launch_long_k<K_XSQ, DD, true, F_NONE>(a, sms, st, w); \
    else if (i && kind == K_L1) e = launch_long_k<K_L1, DD, true, F_NONE>(a, sms, st, w); \
    else if (i && kind == K_LINF) e = launch_long_k<K_LINF, DD, true, F_NONE>(a, sms, st, w); \
  }
    FFD_LONG_F(1)
    FFD_LONG_F(2)
    FFD_LONG_F(3)
    FFD_LONG_F(4)
#undef FFD_LONG_F
    ++*launches;
  }
  cudaFreeAsync(buf, st);
  return e;
}

}  // namespace ffd
