// longpair_kernel.cuh — very long pairs spread over the whole GPU
// (BASELINE config 5).
//
// What: δ_dF of a pair with n rows (the shorter curve) and m columns, Eq. (1)
// in linear memory (Theorem 1): every warp keeps only
// its strip of rows and one column of DP state in registers.  Any n and m.
//
// How:
//   * The rows are cut into bands of 32·R rows; band b runs on one warp as the
//     lane-strip wavefront of strip.cuh (lane ℓ: rows [ℓR, ℓR+R), column t−ℓ at
//     step t) and streams all m columns once.
//   * Band b's bottom row (lane 31's value, one per column) is band b+1's top
//     input.  It moves through LINKS: rings of 8-byte slots {payload, tag}
//     written by lane 31 (tag = absolute stream position + 1; an int64 value
//     takes two slots, each with the tag).  The consumer polls the slot itself,
//     so data and "ready" arrive together and no fence or flag is needed (the
//     low-latency protocol NCCL calls LL).  Inside a CTA the ring is in shared
//     memory; between the CTAs of a cluster in the consumer's shared memory
//     (DSMEM); between clusters in global memory (L2).
//   * The consumer prefetches the slots of the next 32 columns one chunk ahead
//     (like the column points), checks the tags when it stores them into its
//     column ring, and re-polls only the slots that were not ready.  It
//     publishes how far it has consumed; the producer checks that counter (also
//     prefetched) before reusing slots: bounded rings, no overwrite.
//   * Slots are indexed by the ABSOLUTE stream position (tag base + position) so
//     that the slot reuse distance is exactly the ring size across successive
//     streams — the flow-control test (consumed + capacity > absolute position)
//     is only valid then.
//   * Any length (multi-pass): a group of Gg CTAs has NBP = 8·Gg band SLOTS;
//     band b runs on slot b mod NBP in pass ⌊b / NBP⌋.  The last slot's output
//     link WRAPS to the first slot, so pass k+1's first band reads pass k's
//     last band: the passes form one continuous wavefront with no grid barrier.
//     Slot 0 finishes pass k (a whole stream) before it consumes pass k+1's
//     input, so the wrap link must buffer one whole stream: it is a ring in HBM
//     of ≥ S positions (the batch workspace's band scratch, 156 MB on B200:
//     16M fp32 / 8M int64 positions),
//     and a multi-pass pair puts its LONGER curve on the rows so that the
//     buffered stream is the shorter curve (linear memory, Theorem 1).  Every
//     link carries one stream per pass; the wrap link's stream of pass k+1 is
//     written in pass k, so its producer tags it with the next pass's base.
//   * Exact integers: the fp32 tier evaluates int32 input in fp32-exact integer
//     arithmetic and flags a pair whose points leave the exact
//     window; the int64 tier (the same kernel with 64-bit state, launched after
//     it) recomputes exactly the flagged pairs.
//   * One persistent CTA of 8 warps per SM, cooperative launch: all slots are
//     co-resident, so spinning on a neighbour cannot deadlock.  Counters and
//     tags are absolute positions, so successive passes and pairs need no grid
//     barrier.
//   * A spin that sees no progress for ~2.5 s sets a global abort flag (every
//     other spin then gives up at once) and the pair's result becomes NaN /
//     INT64_MIN: a hang is never turned into a plausible number.
#pragma once
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "longpair.cuh"
#include "strip.cuh"

namespace ffd {

#ifndef FFD_LWARPS
#define FFD_LWARPS 8
#endif
constexpr int kLWarps = FFD_LWARPS;  // warps (band slots) per CTA
constexpr int kLSmemRing = 1024;    // slots per intra-CTA link (8 KB; the producer may run
                                    // ~500 steps ahead, far beyond the ~47 the consumer needs)
constexpr int kLGlobRing = 2048;    // slots per inter-CTA link
constexpr int kMaxLongCtas = 1024;
#ifndef FFD_LONG_COLS
#define FFD_LONG_COLS 2
#endif
// columns per warp step of the fp32 tier (2 or 4).  Four halve the steps per column but measured
// slower on config 5 (39.5 against 33 ms per norm: the step time doubled), so two stay the default.
constexpr int kLCols = FFD_LONG_COLS;
#ifndef FFD_LONG_UNROLL
#define FFD_LONG_UNROLL 8  // steps per iteration of the steady loop (8, 4 or 2): config 5 takes
                           // 93.0 / 94.5 / 98.2 ms per three norms (fewer branch stalls)
#endif
#ifndef FFD_LONG_R16
#define FFD_LONG_R16 1
#endif
constexpr bool kLR16 = FFD_LONG_R16 != 0;  // build the R = 16 bands (fp32 tier)
// a spin on a link that has not advanced for this many SM cycles (≈ 2.5 s)
// reports the link state with printf, sets the abort flag and gives up
constexpr long long kWatchdogCycles = 5000000000LL;
constexpr long long kAbortCheckCycles = 1LL << 20;  // spins read the abort flag only after ~0.5 ms
constexpr long long kAbortRecheckCycles = 1LL << 15;  // ... and then every ~17 µs

struct LongProblem {
  const void* p;
  const void* q;
  const int64_t* offsets;
  const int32_t* lengths;
  int64_t num_pairs;
  const int* list;
  const int* list_count;
  void* out;
  uint2* gring;    // [G][kLGlobRing] slots of the link CTA g → g+1 (zeroed per launch)
  unsigned* gcons; // [G + 1] consumer progress on the link CTA g → g+1, [G]: the wrap link
  uint2* wrap;     // multi-pass wrap link ring (HBM; the batch workspace's band scratch)
  unsigned wrap_slots;  // its capacity in slots (a power of two)
  int* bad;        // per long pair: a point left the fp32-exact window (int input, fp32 tier)
  int* abort;      // a watchdog fired: every spin gives up, results become NaN / INT64_MIN
  int trace;       // FFD_LONG_TRACE=1: print each band's start/end time
  int force_r;     // FFD_LONG_R (testing): rows per lane instead of the automatic choice
  // ffd_long_pair_shard (one pair, its rows curve split over GPUs): this launch
  // computes rows [row_begin, row_end); its first band reads its top input from
  // ext_in (a ring in this GPU's memory that the previous GPU writes over NVLink)
  // and its last band writes its bottom row into ext_out (the next GPU's ring).
  // The rings hold a whole stream, so no flow control crosses GPUs.
  int shard;
  int row_begin, row_end;
  uint2* ext_in;
  unsigned ext_in_mask, ext_in_tb;
  uint2* ext_out;
  unsigned ext_out_mask, ext_out_tb;
  unsigned* ext_cons;  // [2]: the consumer's progress (unread), the producer's (stays at ext_out_tb)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// slot accesses; `sys` selects system scope for links whose ring is written by
// another GPU over NVLink (the cross-GPU links of ffd_long_pair_shard)
__device__ __forceinline__ uint2 ld_slot(const uint2* p, int sys = 0) {
  uint2 v;
  if (sys)
    asm volatile("ld.relaxed.sys.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_slot4(const uint2* p, int sys = 0) {
  uint4 v;
  if (sys)
    asm volatile("ld.relaxed.sys.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
  else
    asm volatile("ld.relaxed.gpu.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
  return v;
}
// one predicated 16-byte store {a, b, c, d} (no divergent branch per step)
__device__ __forceinline__ void st_v4_pred(uint2* p, unsigned a, unsigned b, unsigned c, unsigned d,
                                           int pred, int sys = 0) {
  if (sys)
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t@q st.relaxed.sys.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
        "r"(a), "r"(b), "r"(c), "r"(d), "r"(pred)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t@q st.relaxed.gpu.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
        "r"(a), "r"(b), "r"(c), "r"(d), "r"(pred)
        : "memory");
}
__device__ __forceinline__ unsigned ld_ctr(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_ctr(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ bool aborted(const int* abort) {
  return *reinterpret_cast<const volatile int*>(abort) != 0;
}
// The abort flag is an L2 round trip: a spin reads it after ~0.5 ms of waiting,
// then every ~17 µs — not on every poll, where a band waiting out the pipeline
// fill would see its producer's slot up to one round trip late, a delay that
// adds up along the chain of bands (round 2: every poll after 0.5 ms read it).
struct AbortPoll {
  long long due;
  __device__ __forceinline__ explicit AbortPoll(long long t0) : due(t0 + kAbortCheckCycles) {}
  __device__ __forceinline__ bool fired(long long now, const int* abort) {
    if (now < due) return false;
    due = now + kAbortRecheckCycles;
    return aborted(abort);
  }
};

// How a DP value of type T moves through {payload, tag} slots.  A = absolute
// stream position (tag base + position), tag = A + 1.
template <typename T>
struct Slots;
template <>
struct Slots<float> {  // one slot per position
  static constexpr unsigned SPP = 1;
  using Pre = uint2;
  static __device__ __forceinline__ Pre load(const uint2* ring, unsigned mask, unsigned A, int sys = 0) {
    return ld_slot(ring + (A & mask), sys);
  }
  static __device__ __forceinline__ bool ready(const Pre& v, unsigned want) { return v.y == want; }
  static __device__ __forceinline__ float value(const Pre& v) { return __uint_as_float(v.x); }
  static __device__ __forceinline__ Pre none() { return make_uint2(0u, 0u); }
  // positions A (even) and A+1 in one 16-byte store
  static __device__ __forceinline__ void put2(uint2* ring, unsigned mask, unsigned A, float v0, float v1,
                                              int pred, int sys = 0) {
    st_v4_pred(ring + (A & mask & ~1u), __float_as_uint(v0), A + 1u, __float_as_uint(v1), A + 2u, pred, sys);
  }
};
template <>
struct Slots<long long> {  // two slots per position: {lo, tag}, {hi, tag}
  static constexpr unsigned SPP = 2;
  using Pre = uint4;
  static __device__ __forceinline__ Pre load(const uint2* ring, unsigned mask, unsigned A, int sys = 0) {
    return ld_slot4(ring + ((2u * A) & mask), sys);
  }
  static __device__ __forceinline__ bool ready(const Pre& v, unsigned want) {
    return v.y == want && v.w == want;
  }
  static __device__ __forceinline__ long long value(const Pre& v) {
    return (long long)(((unsigned long long)v.z << 32) | v.x);
  }
  static __device__ __forceinline__ Pre none() { return make_uint4(0u, 0u, 0u, 0u); }
  static __device__ __forceinline__ void put2(uint2* ring, unsigned mask, unsigned A, long long v0,
                                              long long v1, int pred, int sys = 0) {
    uint2* s = ring + ((2u * A) & mask);  // 32-byte aligned: A is even
    const unsigned long long u0 = (unsigned long long)v0, u1 = (unsigned long long)v1;
    st_v4_pred(s, (unsigned)u0, A + 1u, (unsigned)(u0 >> 32), A + 1u, pred, sys);
    st_v4_pred(s + 2, (unsigned)u1, A + 2u, (unsigned)(u1 >> 32), A + 2u, pred, sys);
  }
};

// one link endpoint: ring of slots (mask = slots − 1) and the consumer counter
struct Link {
  uint2* ring;
  unsigned mask;
  unsigned* cons;
  int sys;  // written by another GPU (system-scope accesses)
};

constexpr int kLRing = 256;  // column-ring positions per warp: lane 31 trails lane 0 by 31·K ≤ 124
constexpr int kLRingMask = kLRing - 1;
// A pair's column stream with K columns per step: `lead` sentinel positions
// (1 … K) so that its length lead + m is a multiple of K, then the m columns.  A
// second sentinel in front changes nothing (both reset every row to +∞); the
// corner value 0 sits at position lead − 1.  Padding in front, not behind,
// keeps the last column the last position, which DTW needs (a repeated column
// would add to its sums).
template <int K>
__host__ __device__ inline int stream_lead(int m) {
  const int r = m % K;
  return r ? K - r : K;
}
template <int K>
__host__ __device__ inline int stream_len(int m) {
  return stream_lead<K>(m) + m;
}

// ring slot of stream position p with K columns per step: lane ℓ reads positions
// K(t−ℓ)+k, so consecutive lanes would be K·16 B apart (a 2K-way shared-memory
// bank conflict on every element load); grouping the slots by p mod K makes
// their reads consecutive (conflict-free)
template <int K>
__device__ __forceinline__ int lring(int p) {
  return (p & (K - 1)) * (kLRing / K) + ((p / K) & (kLRing / K - 1));
}

// K columns per warp step (K = 2 or 4): lane ℓ at step t works on positions
// K(t−ℓ) … K(t−ℓ)+K−1.  Column k's chain trails column k−1's by one row (cell
// (r, k) needs (r, k−1) and (r−1, k)), so the K chains interleave and the
// shuffle + chain latency is paid once per K columns.  Lane ℓ hands lane ℓ+1 its
// bottom value after each of the K columns (K shuffles per step).  Software-
// pipelined: the distances of step g+1 are computed during
// step g's chains and the ring elements of step g+2 are loaded.
template <typename T, int KIND, int D, int R, bool INT_IN, int K, bool DTW = false>
struct PipeK {
  using C = SCfg<T, KIND, D, INT_IN>;
  static constexpr int N = C::EBYTES / sizeof(T);
  T d[K][R];   // distances of the step to execute next
  T top[K];    // its top values (lane 0)
  alignas(16) T nxt[K][N];  // the elements of the step after it

  __device__ __forceinline__ void load(T (&el)[K][N], const uint4* __restrict__ ring, int g) const {
#pragma unroll
    for (int k = 0; k < K; k++) {
      const uint4* src = ring + lring<K>(K * g + k) * C::EW;
#pragma unroll
      for (int w = 0; w < C::EW; w++) reinterpret_cast<uint4*>(el[k])[w] = src[w];
    }
  }

  __device__ __forceinline__ void prime(const T (&x)[C::NS][R], const uint4* __restrict__ ring, int g) {
    alignas(16) T el[K][N];
    load(el, ring, g);
#pragma unroll
    for (int k = 0; k < K; k++) {
      cell_dists<T, KIND, D, R, INT_IN>(x, el[k], d[k]);
      top[k] = el[k][C::I_TOP];
    }
    load(nxt, ring, g + 1);
  }

  __device__ __forceinline__ void step(T (&c)[R], T& diag, T (&b)[K], const T (&x)[C::NS][R],
                                       const uint4* __restrict__ ring, int g, int lane) {
    T up[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const T upv = __shfl_up_sync(0xffffffffu, b[k], 1);
      up[k] = (lane == 0) ? top[k] : upv;
    }
#pragma unroll
    for (int k = 0; k < K; k++) {
      T u = up[k], dg = (k == 0) ? diag : up[k - 1];
#pragma unroll
      for (int r = 0; r < R; r++) {
        const T m = tmin(tmin(u, dg), c[r]);
        T nv;
        if constexpr (DTW) nv = m + d[k][r];  // PAPER Appendix B: min3 + d
        else nv = tmax(m, d[k][r]);
        dg = c[r];
        c[r] = nv;
        u = nv;
      }
      b[k] = c[R - 1];
    }
    diag = up[K - 1];
#pragma unroll
    for (int k = 0; k < K; k++) {
      cell_dists<T, KIND, D, R, INT_IN>(x, nxt[k], d[k]);
      top[k] = nxt[k][C::I_TOP];
    }
    load(nxt, ring, g + 2);
  }
};

template <typename T, int KIND, int D, bool INT_IN, int FIN, int R>
struct LongRunner {
  using C = SCfg<T, KIND, D, INT_IN>;
  using SL = Slots<T>;
  using Pre = typename SL::Pre;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  static constexpr int NS = C::NS;

  uint4* ring;  // this warp's column ring [kLRing * EW]
  const LongProblem& pb;
  int lane;

  // ---- pair description --------------------------------------------------
  const In* rows;
  const In* cols;
  int n, m;
  int center[D];

  // input point → cell coordinates (fp32 tier with int input: translated by the
  // pair's first row point, false if it leaves the fp32-exact window)
  __device__ bool conv(const In (&a)[D], T (&v)[D]) const {
    bool ok = true;
#pragma unroll
    for (int c = 0; c < D; c++) {
      if constexpr (INT_IN && C::F) {
        long long t = (long long)a[c] - center[c];
        ok &= (t >= -C::LIM) && (t <= C::LIM);
        v[c] = (float)(int)t;
      } else {
        v[c] = (T)a[c];
      }
    }
    return ok;
  }

  // column element of position `pos` (0 = sentinel), written with its top value
  template <int K>
  __device__ void store_elem(const In (&a)[D], int kind, int pos, T top, bool& ok) {
    alignas(16) T f[C::EBYTES / sizeof(T)];
#pragma unroll
    for (int i = 0; i < (int)(C::EBYTES / sizeof(T)); i++) f[i] = (T)0;
    if (kind != 0) {
      if constexpr (!C::F) {
        f[C::I_SENT] = (T)1;
      } else if constexpr (C::XSQ) {
        f[D] = finf();
      } else {
#pragma unroll
        for (int c = 0; c < D; c++) f[c] = finf();
      }
    } else {
      T v[D];
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
    f[C::I_TOP] = top;
    uint4* dst = ring + lring<K>(pos) * C::EW;
#pragma unroll
    for (int w = 0; w < C::EW; w++) dst[w] = reinterpret_cast<const uint4*>(f)[w];
  }

  // positions: [0, lead) sentinels, lead + j = column j (stream_lead above)
  __device__ void fetch(int pos, int S2, int lead, In (&a)[D], int& kind) const {
#pragma unroll
    for (int c = 0; c < D; c++) a[c] = (In)0;
    if (pos >= S2) {
      kind = 2;
    } else if (pos < lead) {
      kind = 1;
    } else {
      kind = 0;
      const int64_t col = pos - lead;
#pragma unroll
      for (int c = 0; c < D; c++) a[c] = __ldg(cols + col * D + c);
    }
  }

  // top value of position `pos` for this band: the corner/border for band 0,
  // else the producer's slot (spinning until its tag shows up)
  __device__ __forceinline__ T top_of(int pos, int S2, int lead, bool has_in, const Link& in, unsigned tb,
                                      Pre pre) const {
    if (pos >= S2) return tinf<T>();
    if (!has_in) return pos == lead - 1 ? (T)0 : tinf<T>();
    const unsigned want = tb + (unsigned)pos + 1u;
    if (!SL::ready(pre, want)) {
      const long long t0 = clock64();
      AbortPoll ap(t0);
      while (!SL::ready(pre, want)) {
        pre = SL::load(in.ring, in.mask, tb + (unsigned)pos, in.sys);
        const long long now = clock64();
        if (ap.fired(now, pb.abort)) break;
        if (now - t0 > kWatchdogCycles) {  // a link that never delivers: report, abort
          printf("ffd long_kernel watchdog: consumer cta %d lane %d pos %d want tag %u (tb %u)\n",
                 (int)blockIdx.x, lane, pos, want, tb);
          atomicExch(pb.abort, 1);
          break;
        }
      }
    }
    return SL::value(pre);
  }

  // Wait (lane 0 only, with backoff) until the producer has published position
  // `pos`: it writes positions in order, so the earlier slots of the chunk are
  // then ready too and the other lanes find their tags at the first look.  This
  // keeps waiting warps from hammering shared memory / L2 with 32-lane polls,
  // which slowed the producers they wait for.
  __device__ __forceinline__ void wait_chunk(int pos, int S2, bool has_in, const Link& in,
                                             unsigned tb) const {
    if (has_in && lane == 0) {
      pos = min(pos, S2 - 1);
      const unsigned want = tb + (unsigned)pos + 1u;
      if (!SL::ready(SL::load(in.ring, in.mask, tb + (unsigned)pos, in.sys), want)) {
        const long long t0 = clock64();
        AbortPoll ap(t0);
        while (!SL::ready(SL::load(in.ring, in.mask, tb + (unsigned)pos, in.sys), want)) {
          __nanosleep(64);
          const long long now = clock64();
          if (ap.fired(now, pb.abort)) break;
          if (now - t0 > kWatchdogCycles) {
            printf("ffd long_kernel watchdog: chunk wait cta %d pos %d want tag %u (tb %u)\n",
                   (int)blockIdx.x, pos, want, tb);
            atomicExch(pb.abort, 1);
            break;
          }
        }
      }
    }
    __syncwarp();
  }

  // one band of 32·R rows starting at row r0, K columns per warp step (PipeK).
  // tbi / tbo: tag bases of the input / output link streams.
  // SYS: the band has a cross-GPU link (ffd_long_pair_shard): its per-step slot
  // accesses use system scope (a compile-time choice: a runtime branch in the
  // per-step store cost config 5 15 %)
  template <int K, bool SYS>
  __device__ bool run_band(int r0, bool has_in, Link in, unsigned tbi, bool has_out, Link out,
                           unsigned tbo, bool last_band, int out_idx, int* bad_flag) {
    static_assert(K == 2 || K == 4, "K columns per step");
    constexpr int P = 32 / K;                  // steps per 32-position chunk
    const int lead = stream_lead<K>(m);
    const int S2 = lead + m;                   // positions (a multiple of K)
    const int NT = S2 / K;                     // steps
    bool ok = true;
    T x[NS][R], c[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int row = min(r0 + lane * R + r, n - 1);
      In a[D];
#pragma unroll
      for (int cc = 0; cc < D; cc++) a[cc] = __ldg(rows + (int64_t)row * D + cc);
      T v[D];
      ok &= conv(a, v);
#pragma unroll
      for (int cc = 0; cc < D; cc++) x[cc][r] = v[cc];
      if constexpr (C::XSQ) {
        int pp = 0;
#pragma unroll
        for (int cc = 0; cc < D; cc++) pp += (int)v[cc] * (int)v[cc];
        x[D][r] = (float)pp;
      }
      c[r] = tinf<T>();
    }
    if constexpr (INT_IN && C::F) {
      if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicExch(bad_flag, 1);
    }
    T diag = tinf<T>(), b[K];
#pragma unroll
    for (int k = 0; k < K; k++) b[k] = tinf<T>();
    // prologue: positions [0, 32) stored; column points of [32, 64) and [64, 96)
    // in flight (two chunks ahead: one chunk does not cover the L2/HBM latency of
    // a latency-bound warp); link slots of [32, 64) in flight
    In a[D], a2[D];
    int kind, kind2;
    fetch(lane, S2, lead, a, kind);
    wait_chunk(31, S2, has_in, in, tbi);
    Pre pre = (has_in && lane < S2) ? SL::load(in.ring, in.mask, tbi + (unsigned)lane, SYS) : SL::none();
    store_elem<K>(a, kind, lane, top_of(lane, S2, lead, has_in, in, tbi, pre), ok);
    fetch(32 + lane, S2, lead, a, kind);
    fetch(64 + lane, S2, lead, a2, kind2);
    pre = (has_in && 32 + lane < S2) ? SL::load(in.ring, in.mask, tbi + (unsigned)(32 + lane), SYS) : SL::none();
    __syncwarp();
    if (has_in && lane == 0) st_ctr(in.cons, tbi + (unsigned)min(32, S2));
    const unsigned cap = (out.mask + 1u) / SL::SPP;  // output ring capacity in positions
    unsigned cons_seen = 0, cons_next = 0;
    if (has_out) cons_seen = cons_next = ld_ctr(out.cons);

    const int total = NT + 31;
    const int pown = (has_out && lane == kWarp - 1) ? 1 : 0;
    // DTW: the lane holding row n − 1 reads its value right after its last
    // position (step NT − 1 + lane); later steps run it over the stream's end
    // (d = +∞), which a sum does not survive
    const int cap_lane = (n - 1 - r0) / R, cap_reg = (n - 1 - r0) - cap_lane * R;
    const int t_cap = (FIN == F_DTW && last_band) ? NT + cap_lane : total + 1;
    T dtw_val = tinf<T>();
    int t = 0, next_refill = P;
    while (t < total) {
      if (t == next_refill) {
        // the slots of this chunk were prefetched one chunk ago: when every tag
        // is already there, go on without touching the link (a blocking poll of
        // an L2 link costs ~700 cycles per chunk); else wait on lane 0 first
        const int p0 = K * t;
        if (p0 < S2 && has_in) {
          const int pos = p0 + lane;
          const bool ready = pos >= S2 || SL::ready(pre, tbi + (unsigned)pos + 1u);
          if (!__all_sync(0xffffffffu, ready)) wait_chunk(p0 + 31, S2, has_in, in, tbi);
        }
        store_elem<K>(a, kind, p0 + lane, top_of(p0 + lane, S2, lead, has_in, in, tbi, pre), ok);
#pragma unroll
        for (int cc = 0; cc < D; cc++) a[cc] = a2[cc];
        kind = kind2;
        fetch(p0 + 64 + lane, S2, lead, a2, kind2);
        const int pn = p0 + 32 + lane;
        pre = (has_in && pn < S2) ? SL::load(in.ring, in.mask, tbi + (unsigned)pn, SYS) : SL::none();
        __syncwarp();
        if (has_in && lane == 0) st_ctr(in.cons, tbi + (unsigned)min(p0 + 32, S2));
        next_refill += P;
      }
      if (has_out && (t % P) == 0) {
        // lane 31 writes positions < K·t during the next P steps: their slots
        // must be consumed (cons + capacity > tbo + K·t).  The counter is read a
        // chunk ahead.
        if (lane == kWarp - 1) {
          cons_seen = cons_next;
          if ((int)(cons_seen + cap - (tbo + (unsigned)(K * t))) <= 0) {
            const long long t0 = clock64();
            AbortPoll ap(t0);
            while ((int)(cons_seen + cap - (tbo + (unsigned)(K * t))) <= 0) {
              __nanosleep(64);
              cons_seen = ld_ctr(out.cons);
              const long long now = clock64();
              if (ap.fired(now, pb.abort)) break;
              if (now - t0 > kWatchdogCycles) {
                printf("ffd long_kernel watchdog: producer cta %d warp %d t %d cons %u tb %u cap %u\n",
                       (int)blockIdx.x, (int)(threadIdx.x >> 5), t, cons_seen, tbo, cap);
                atomicExch(pb.abort, 1);
                break;
              }
            }
          }
          cons_next = ld_ctr(out.cons);
        }
      }
      __syncwarp();
      const int stop = min(min(next_refill, total), t < t_cap ? t_cap : total);
      int g = t - lane;
      // primed again after every refill (its look-ahead may read unstored slots)
      PipeK<T, KIND, D, R, INT_IN, K, FIN == F_DTW> pipe;
      pipe.prime(x, ring, g);
      // lane 31 publishes its K bottom-row values {value, tag} of every step with
      // predicated 16-byte stores (no divergent branch per step)
      auto one = [&](int gg) {
        pipe.step(c, diag, b, x, ring, gg, lane);
        const int pr = pown & ((unsigned)gg < (unsigned)NT);
#pragma unroll
        for (int k = 0; k < K; k += 2)
          SL::put2(out.ring, out.mask, tbo + (unsigned)(K * gg + k), b[k], b[k + 1], pr, SYS);
      };
#if FFD_LONG_UNROLL == 8
#pragma unroll 1
      for (; t + 8 <= stop; t += 8, g += 8) {
#pragma unroll
        for (int u = 0; u < 8; u++) one(g + u);
      }
#endif
#if FFD_LONG_UNROLL >= 4
#pragma unroll 1
      for (; t + 4 <= stop; t += 4, g += 4) {
        one(g);
        one(g + 1);
        one(g + 2);
        one(g + 3);
      }
#endif
#pragma unroll 1
      for (; t + 2 <= stop; t += 2, g += 2) {
        one(g);
        one(g + 1);
      }
      if (t < stop) {
        one(g);
        ++t;
      }
      if constexpr (FIN == F_DTW) {
        if (t == t_cap && lane == cap_lane) dtw_val = pick_reg<R>(c, cap_reg);
      }
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    if constexpr (FIN == F_DTW) {
      // DTW: rows repeated below row n − 1 are not neutral for a sum, so the lane
      // that holds row n − 1 emits, from its register (n − 1) mod R
      if (last_band && lane == cap_lane) {
        __threadfence();
        const float f = (float)dtw_val;
        reinterpret_cast<float*>(pb.out)[out_idx] = aborted(pb.abort) ? __int_as_float(0x7fc00000) : f;
      }
    } else if (last_band && lane == kWarp - 1) {
      __threadfence();
      const bool dead = aborted(pb.abort);
      if constexpr (INT_IN) {
        bool bad = dead;
        if constexpr (C::F) bad = bad || !all_ok || *reinterpret_cast<volatile int*>(bad_flag) != 0;
        // an fp32-tier pair flagged here is recomputed by the int64 tier
        reinterpret_cast<long long*>(pb.out)[out_idx] = bad ? LLONG_MIN : (long long)c[R - 1];
      } else {
        float f = c[R - 1];
        if constexpr (FIN == F_SQRT) f = sqrt_result(f);
        reinterpret_cast<float*>(pb.out)[out_idx] = dead ? __int_as_float(0x7fc00000) : f;
      }
    }
    if constexpr (INT_IN && C::F) {
      // a column point outside the window (seen by any band): flag for the int64 tier
      if (!all_ok && lane == 0) atomicExch(bad_flag, 1);
    }
    __syncwarp();
    return all_ok;
  }
};

// Rows per lane for a pair whose rows curve has n points, on a group of G
// co-resident CTAs: the smallest built R whose bands all fit at once
// (⌈bands / 8⌉ ≤ G: one pass, returns true); else false and the multi-pass R.
// (R = 32 is not built: its registers spilled and, the kernel's register count
// being the maximum over its R paths, slowed every R.)
template <typename T>
__host__ __device__ inline bool long_rows_fit(int n, int G, int& R) {
  constexpr bool F = std::is_same<T, float>::value;
  const int rs_f[4] = {4, 7, 8, 16};  // the R the fp32 tier is built for
  const int rs_i[2] = {4, 8};         // the R the int64 tier is built for
  const int* rs = F ? rs_f : rs_i;
  const int nr = F ? (kLR16 ? 4 : 3) : 2;
  for (int i = 0; i < nr; i++) {
    R = rs[i];
    const int nb = (n + kWarp * R - 1) / (kWarp * R);
    if ((nb + kLWarps - 1) / kLWarps <= G) return true;
  }
  R = F && kLR16 ? 16 : 8;
  return false;
}

template <typename T, int KIND, int D, bool INT_IN, int FIN>
__global__ void __launch_bounds__(kWarp* kLWarps, 1) long_kernel(const LongProblem pb) {
  using C = SCfg<T, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  constexpr bool TIER64 = !C::F;  // int64 tier: only the pairs the fp32 tier flagged
  // dynamic shared memory: [kLWarps][kLSmemRing] link slots, [kLWarps][kLRing·EW]
  // column rings, [kLWarps] consumer counters
  extern __shared__ uint4 lsm[];
  uint2 (*slink)[kLSmemRing] = reinterpret_cast<uint2(*)[kLSmemRing]>(lsm);
  uint4 (*rings)[kLRing * C::EW] =
      reinterpret_cast<uint4(*)[kLRing * C::EW]>(lsm + kLWarps * kLSmemRing / 2);
  unsigned* scons = reinterpret_cast<unsigned*>(lsm + kLWarps * kLSmemRing / 2 + kLWarps * kLRing * C::EW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int npairs = *pb.list_count;
  // the pairs this launch computes: all long pairs (fp32 tier), or the flagged
  // ones (int64 tier); every CTA derives the same selection
  auto selected = [&](int li) { return !TIER64 || pb.bad[li] != 0; };
  int nsel = 0;
  for (int li = 0; li < npairs; li++) nsel += selected(li) ? 1 : 0;
  // nothing to do (the common case of a batch without long pairs): leave before
  // initialising 64 KB of link rings; every CTA takes the same exit, so no
  // cluster barrier is left waiting
  if (nsel == 0) return;
  // Thread-block cluster: consecutive CTAs of a cluster link warp 7 → next CTA's
  // warp 0 through DISTRIBUTED shared memory (the producer stores {value, tag}
  // slots straight into the consumer CTA's smem ring slink[7], which warp 7 of
  // that CTA does not use itself; the consumer publishes its progress into its
  // own scons[7], which the producer reads remotely).  Links between clusters,
  // and the wrap link of a group, go through L2.
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  for (int i = threadIdx.x; i < kLWarps * kLSmemRing; i += blockDim.x)
    (&slink[0][0])[i] = make_uint2(0u, 0u);
  if (threadIdx.x < kLWarps) scons[threadIdx.x] = 0u;
  // this launch's global link state: tags restart at 1 every launch, so a slot
  // left from an earlier launch must read as empty — zeroed here (instead of a
  // memset on every batch call, most of which have no long pair) before the
  // grid barrier
  for (int i = threadIdx.x; i < kLGlobRing; i += blockDim.x)
    pb.gring[(size_t)cta * kLGlobRing + i] = make_uint2(0u, 0u);
  if (threadIdx.x == 0) pb.gcons[cta] = 0u;
  if constexpr (!TIER64) {
    for (int i = cta * (int)blockDim.x + (int)threadIdx.x; i < npairs; i += G * (int)blockDim.x) pb.bad[i] = 0;
    if (cta == 0 && threadIdx.x == 0) *pb.abort = 0;
  }
  __syncthreads();
  cl.sync();  // every CTA of the cluster has initialised its rings before any remote access
  cg::this_grid().sync();  // and every CTA its global ring before any consumer polls it
  // CTA groups: several long pairs run side by side, each on a contiguous group
  // of Gg CTAs (selected pair lj on group lj mod NG).  Gg is what the largest
  // pair needs at R = 16 (int64 tier: 8); a single very long pair (config 5) keeps the whole
  // grid.  Every CTA computes the same NG from the same lengths.
  int need = 1;
  for (int li = 0; li < npairs; li++) {
    if (!selected(li)) continue;
    const int k = pb.list[li];
    const int n0 = pb.lengths[k], m0 = pb.lengths[pb.num_pairs + k];
    const int rows = n0 < m0 ? n0 : m0;
    constexpr int RN = C::F && kLR16 ? 16 : 8;  // the tallest built band
    const int nbn = (rows + kWarp * RN - 1) / (kWarp * RN);
    need = max(need, (nbn + kLWarps - 1) / kLWarps);
  }
  need = min(need, G);
  const int NG = max(1, min(G / need, nsel));
  const int Gg = G / NG;
  // rows per lane of a pair whose shorter curve has n points; false: multi-pass
  auto choose_r = [&](int n, int& R) {
    bool fit = long_rows_fit<T>(n, Gg, R);
    if (pb.force_r && C::F && (pb.force_r == 4 || pb.force_r == 7 || pb.force_r == 8 || (kLR16 && pb.force_r == 16))) {
      R = pb.force_r;  // testing: a built R; multi-pass if its bands do not fit at once
      const int nbf = (n + kWarp * R - 1) / (kWarp * R);
      fit = (nbf + kLWarps - 1) / kLWarps <= Gg;
    }
    return fit;
  };
  // Multi-pass pairs (only possible with one group: every pair fits one pass on
  // a group of `need` CTAs) stream their SHORTER curve as columns through the
  // HBM wrap link, whose ring is sized once per launch to the longest such
  // stream (wrap_mask + 1 slots) and zeroed here: tags restart every launch.
  unsigned wrap_mask = 0;
  for (int li = 0; li < npairs && NG == 1; li++) {
    if (!selected(li)) continue;
    const int k = pb.list[li];
    const int n0 = pb.lengths[k], m0 = pb.lengths[pb.num_pairs + k];
    int Rx;
    if (choose_r(pb.shard ? pb.row_end - pb.row_begin : min(n0, m0), Rx)) continue;
    // (+64: the producer's flow-control test looks up to 62 positions past the stream)
    const unsigned long long need_slots =
        (unsigned long long)(stream_len<C::F ? kLCols : 2>(pb.shard ? max(n0, m0) : min(n0, m0)) + 64) *
        Slots<T>::SPP;
    unsigned long long cap = 2;
    while (cap < need_slots) cap <<= 1;
    if (cap <= pb.wrap_slots) wrap_mask = max(wrap_mask, (unsigned)(cap - 1ull));
  }
  if (wrap_mask)
    for (size_t i = (size_t)cta * blockDim.x + threadIdx.x; i <= (size_t)wrap_mask; i += (size_t)G * blockDim.x)
      pb.wrap[i] = make_uint2(0u, 0u);
  if (cta == 0 && threadIdx.x == 0) {
    pb.gcons[G] = 0u;
    if (pb.shard) pb.ext_cons[1] = pb.ext_out_tb;  // the next GPU's ring never needs flow control
  }
  if constexpr (!TIER64) {
    for (int i = cta * (int)blockDim.x + (int)threadIdx.x; i < npairs; i += G * (int)blockDim.x) pb.bad[i] = 0;
    if (cta == 0 && threadIdx.x == 0) *pb.abort = 0;
  }
  __syncthreads();
  cl.sync();  // every CTA of the cluster has initialised its rings before any remote access
  cg::this_grid().sync();  // and every CTA its global ring before any consumer polls it
  const int grp = cta / Gg, local = cta - grp * Gg;
  const int last = grp * Gg + Gg - 1;    // the group's last CTA
  const int NBP = Gg * kLWarps;          // band slots of the group
  const int j = local * kLWarps + warp;  // this warp's slot
  const Link wrapL{pb.wrap, wrap_mask, pb.gcons + G};  // multi-pass: last slot → slot 0
  // the links of this slot (fixed for the launch): input from slot j − 1 (slot
  // 0: the wrap link from the group's last slot), output to slot j + 1 (the last
  // slot: the wrap link)
  Link in{}, out{};
  if (warp > 0) {
    in = Link{slink[warp - 1], kLSmemRing - 1u, &scons[warp - 1]};
  } else if (local > 0 && crank > 0) {  // DSMEM link from the previous CTA of this cluster
    in = Link{slink[kLWarps - 1], kLSmemRing - 1u, &scons[kLWarps - 1]};
  } else {  // L2 link from the previous CTA of the group (local 0: the wrap link)
    const int src = local > 0 ? cta - 1 : last;
    in = Link{pb.gring + (size_t)src * kLGlobRing, kLGlobRing - 1u, pb.gcons + src};
  }
  if (warp < kLWarps - 1) {
    out = Link{slink[warp], kLSmemRing - 1u, &scons[warp]};
  } else if (local + 1 < Gg && crank + 1 < csize) {  // DSMEM link into the next CTA of this cluster
    out = Link{cl.map_shared_rank(slink[kLWarps - 1], crank + 1), kLSmemRing - 1u,
               cl.map_shared_rank(&scons[kLWarps - 1], crank + 1)};
  } else {
    out = Link{pb.gring + (size_t)cta * kLGlobRing, kLGlobRing - 1u, pb.gcons + cta};
  }
  unsigned tb = 0;  // tag base: absolute stream position of the current pass on every link
  int li = -1, lsel = -1;  // li: list index of the lsel-th selected pair
  for (int lj = grp; lj < nsel && grp < NG; lj += NG) {
    while (lsel < lj) {
      ++li;
      if (selected(li)) ++lsel;
    }
    const int k = pb.list[li];
    const int64_t B = pb.num_pairs;
    const int n0 = pb.lengths[k], m0 = pb.lengths[B + k];
    int R;
    // one pass: the shorter curve on the rows; multi-pass: the longer one (the
    // wrap link then buffers the shorter curve's stream)
    // shard: the shorter curve on the rows always (every GPU must agree), its
    // rows [row_begin, row_end) here
    const bool multi = !choose_r(pb.shard ? pb.row_end - pb.row_begin : (n0 < m0 ? n0 : m0), R);
    const bool swap = (multi && !pb.shard) ? n0 < m0 : n0 > m0;
    const int n = swap ? m0 : n0, m = swap ? n0 : m0;
    const In* rows = reinterpret_cast<const In*>(swap ? pb.q : pb.p) +
                     (swap ? pb.offsets[B + k] : pb.offsets[k]) * D;
    const In* cols = reinterpret_cast<const In*>(swap ? pb.p : pb.q) +
                     (swap ? pb.offsets[k] : pb.offsets[B + k]) * D;
    constexpr int KC = TIER64 ? 2 : kLCols;  // columns per step of this instantiation
    const unsigned S = (unsigned)stream_len<KC>(m);  // stream positions of this pair (see run_band)
    if (multi && (unsigned long long)(S + 64) * Slots<T>::SPP > (unsigned long long)wrap_mask + 1ull) {
      // the wrap ring cannot buffer this stream (both curves longer than the
      // band scratch holds: > 16M points, int64 tier 8M): documented limit, no plausible value
      if (local == 0 && threadIdx.x == 0) {
        if constexpr (INT_IN) reinterpret_cast<long long*>(pb.out)[k] = LLONG_MIN;
        else reinterpret_cast<float*>(pb.out)[k] = __int_as_float(0x7fc00000);
      }
      continue;
    }
    const int band_rows = kWarp * R;
    const int rb = pb.shard ? pb.row_begin : 0, re = pb.shard ? pb.row_end : n;  // rows of this launch
    const int nb = (re - rb + band_rows - 1) / band_rows;
    const int passes = (nb + NBP - 1) / NBP;
    const Link lin = (multi && j == 0) ? wrapL : in;
    const Link lout = (multi && j == NBP - 1) ? wrapL : out;
    const Link ext_in{pb.ext_in, pb.ext_in_mask, pb.ext_cons, 1};
    const Link ext_out{pb.ext_out, pb.ext_out_mask, pb.ext_cons + 1, 1};
    for (int pass = 0; pass < passes; pass++) {
      const int b = pass * NBP + j;  // band of this slot in this pass
      if (!(b < nb && b > 0) && lane == 0) {
        // this slot does not consume its input link in this pass: nobody writes
        // that stream either, so mark it consumed — otherwise the producer of a
        // later stream would wait on a stale counter
        st_ctr(lin.cons, tb + S);
      }
      if (b < nb) {
        // the shard's first / last band link to the neighbouring GPUs
        const bool x_in = b == 0 && rb > 0, x_out = b + 1 == nb && re < n;
        const bool has_in = b > 0 || x_in, has_out = b + 1 < nb || x_out;
        // the wrap link's stream belongs to the next pass (its consumer, slot 0, reads it then)
        const unsigned tbo = x_out ? pb.ext_out_tb : (j == NBP - 1) ? tb + S : tb;
        const unsigned tbi = x_in ? pb.ext_in_tb : tb;
        const Link lin_b = x_in ? ext_in : lin, lout_b = x_out ? ext_out : lout;
        auto go = [&](auto& run) {
          run.n = re;  // rows past the shard repeat its last row: exact for δ_dF (PAPER L259 footnote)
          run.m = m;
          run.rows = rows;
          run.cols = cols;
          if constexpr (INT_IN) {
#pragma unroll
            for (int c = 0; c < D; c++) run.center[c] = (int)rows[c];
          }
          const unsigned long long t0 = pb.trace ? gtimer() : 0ull;
          // fp32: four columns per step; int64 tier: two (its 64-bit state doubles the registers)
          if (x_in || x_out)
            run.template run_band<KC, true>(rb + b * band_rows, has_in, lin_b, tbi, has_out, lout_b, tbo,
                                            b == nb - 1 && re == n, k, pb.bad + li);
          else
            run.template run_band<KC, false>(rb + b * band_rows, has_in, lin_b, tbi, has_out, lout_b, tbo,
                                             b == nb - 1 && re == n, k, pb.bad + li);
          if (pb.trace && lane == 0)
            printf("ffdtrace band %d cta %d warp %d start %llu end %llu\n", b, cta, warp, t0, gtimer());
        };
        if constexpr (TIER64) {
          if (R == 4) {
            LongRunner<T, KIND, D, INT_IN, FIN, 4> run{rings[warp], pb, lane};
            go(run);
          } else {
            LongRunner<T, KIND, D, INT_IN, FIN, 8> run{rings[warp], pb, lane};
            go(run);
          }
        } else {
          if (R == 4) {
            LongRunner<T, KIND, D, INT_IN, FIN, 4> run{rings[warp], pb, lane};
            go(run);
          } else if (R == 7) {
            LongRunner<T, KIND, D, INT_IN, FIN, 7> run{rings[warp], pb, lane};
            go(run);
          } else if (R == 8) {
            LongRunner<T, KIND, D, INT_IN, FIN, 8> run{rings[warp], pb, lane};
            go(run);
          } else if constexpr (kLR16) {
            LongRunner<T, KIND, D, INT_IN, FIN, 16> run{rings[warp], pb, lane};
            go(run);
          }
        }
      }
      __syncwarp();
      tb += S;  // every link's absolute position advances by one stream per pass
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while a cluster neighbour may still access its smem
}

struct LongWs {
  uint2* gring;
  unsigned* gcons;
  int* bad;
  int* abort;
};

// One persistent CTA (8 band slots) per SM, cooperative launch.  BASELINE
// config 5 (n = 262,144) runs as 147 CTAs of 8 bands × 224 rows (R = 7).
template <typename T, int KIND, int D, bool INT_IN, int FIN>
cudaError_t launch_long_k(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G) {
  auto k = long_kernel<T, KIND, D, INT_IN, FIN>;
  using C = SCfg<T, KIND, D, INT_IN>;
  const size_t smem = sizeof(uint2) * kLWarps * kLSmemRing + sizeof(uint4) * kLWarps * kLRing * C::EW +
                      sizeof(unsigned) * kLWarps;
  // per-device caches: attribute, occupancy and the cluster shape for this grid
  // (the host-side queries would otherwise cost tens of µs on every call)
  int dev = 0;
  cudaGetDevice(&dev);
  static int occ_cache[64] = {0};
  static int clu_cache_g[64] = {0}, clu_cache_c[64] = {0}, clu_cache_bg[64] = {0};
  int occ = dev < 64 ? occ_cache[dev] : 0;
  if (occ == 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kWarp * kLWarps, smem);
    if (dev < 64) occ_cache[dev] = occ;
  }
  if (occ < 1) return cudaErrorLaunchOutOfResources;
  if (G > sms * occ) G = sms * occ;
  static const int trace = getenv("FFD_LONG_TRACE") ? atoi(getenv("FFD_LONG_TRACE")) : 0;
  unsigned wrap_slots = 0;  // the largest power of two of slots the wrap buffer holds
  for (unsigned long long c = 1; c * sizeof(uint2) <= a.wrap_bytes && c <= 0x80000000ull; c <<= 1)
    wrap_slots = (unsigned)c;
  static const int force_r = getenv("FFD_LONG_R") ? atoi(getenv("FFD_LONG_R")) : 0;
  LongProblem pb{a.p,     a.q,     a.offsets, a.lengths,  a.num_pairs, a.list, a.list_count, a.out,
                 w.gring, w.gcons, reinterpret_cast<uint2*>(a.wrap), wrap_slots, w.bad, w.abort, trace,
                 force_r};
  pb.shard = a.shard;
  pb.row_begin = a.row_begin;
  pb.row_end = a.row_end;
  pb.ext_in = reinterpret_cast<uint2*>(a.ext_in);
  pb.ext_in_mask = a.ext_in_slots ? (unsigned)(a.ext_in_slots - 1) : 0u;
  pb.ext_in_tb = a.ext_in_tb;
  pb.ext_out = reinterpret_cast<uint2*>(a.ext_out);
  pb.ext_out_mask = a.ext_out_slots ? (unsigned)(a.ext_out_slots - 1) : 0u;
  pb.ext_out_tb = a.ext_out_tb;
  pb.ext_cons = a.ext_cons;
  void* args[] = {&pb};
  // cluster size: the largest of 8/4/2 whose clusters can all be co-resident
  // for the whole grid (a smaller grid forces taller bands); FFD_LONG_CLUSTER=c
  // forces c (1: none).
  // Measured on config 5: clusters of 2–4 ≈ 32 ms per norm against ≈ 42 ms without
  // (clusters of 8 fit only 128 CTAs and force R = 8).
  static const int env_c = getenv("FFD_LONG_CLUSTER") ? atoi(getenv("FFD_LONG_CLUSTER")) : 0;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = 1;
  cfg.blockDim = dim3(kWarp * kLWarps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attrs;
  int best_c = 1, best_g = 0;
  const bool cached = dev < 64 && clu_cache_g[dev] == G && clu_cache_c[dev] > 0;
  if (cached) {
    best_c = clu_cache_c[dev];
    best_g = clu_cache_bg[dev];
  }
  for (int csz = 8; csz >= 2 && !cached; csz /= 2) {
    if (env_c > 0 && csz != env_c) continue;
    attrs[0].val.clusterDim.x = csz;
    cfg.numAttrs = 1;  // the occupancy query takes the cluster shape only
    cfg.gridDim = dim3((G / csz) * csz);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      continue;
    }
    const int g = (nclusters < G / csz ? nclusters : G / csz) * csz;
    // only a shape that keeps the whole grid: fewer CTAs would force taller bands
    if (g == G) {
      best_g = g;
      best_c = csz;
      break;
    }
  }
  if (!cached && dev < 64) {
    clu_cache_g[dev] = G;
    clu_cache_c[dev] = best_c;
    clu_cache_bg[dev] = best_g;
  }
  if (best_c > 1 && best_g > 0) {
    attrs[0].val.clusterDim.x = best_c;
    cfg.gridDim = dim3(best_g);
    cfg.numAttrs = 2;
    if (cudaLaunchKernelExC(&cfg, (const void*)k, args) == cudaSuccess) return cudaSuccess;
    (void)cudaGetLastError();  // clear a failed cluster launch; use the plain grid
  }
  return cudaLaunchCooperativeKernel((const void*)k, dim3(G), dim3(kWarp * kLWarps), args, smem, st);
}

// per-dimension dispatch (longpair_d<D>.cu)
cudaError_t launch_long_dim1(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G, int64_t* n);
cudaError_t launch_long_dim2(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G, int64_t* n);
cudaError_t launch_long_dim3(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G, int64_t* n);
cudaError_t launch_long_dim4(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G, int64_t* n);

// fp32 input: one launch.  int32 input: the fp32-exact tier, then the exact
// int64 tier over the pairs it flagged (a launch that exits at once when none is).
// DTW (a.measure = 1, fp32 only): the + cell, sqrt per cell under L2.
template <int D>
cudaError_t launch_long_dim(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G,
                            int64_t* launches) {
  ++*launches;
  if (a.measure == 1) {
    if (a.norm == 1) return launch_long_k<float, K_L1, D, false, F_DTW>(a, sms, st, w, G);
    if (a.norm == 3) return launch_long_k<float, K_LINF, D, false, F_DTW>(a, sms, st, w, G);
    if (a.norm == 2) return launch_long_k<float, K_SQRT, D, false, F_DTW>(a, sms, st, w, G);
    return launch_long_k<float, K_SQ, D, false, F_DTW>(a, sms, st, w, G);
  }
  if (a.dtype != 1) {
    if (a.norm == 1) return launch_long_k<float, K_L1, D, false, F_NONE>(a, sms, st, w, G);
    if (a.norm == 3) return launch_long_k<float, K_LINF, D, false, F_NONE>(a, sms, st, w, G);
    if (a.norm == 2) return launch_long_k<float, K_SQ, D, false, F_SQRT>(a, sms, st, w, G);
    return launch_long_k<float, K_SQ, D, false, F_NONE>(a, sms, st, w, G);
  }
  cudaError_t e;
  if (a.norm == 4) e = launch_long_k<float, K_XSQ, D, true, F_NONE>(a, sms, st, w, G);
  else if (a.norm == 1) e = launch_long_k<float, K_L1, D, true, F_NONE>(a, sms, st, w, G);
  else e = launch_long_k<float, K_LINF, D, true, F_NONE>(a, sms, st, w, G);
  if (e != cudaSuccess) return e;
  ++*launches;
  if (a.norm == 4) return launch_long_k<long long, K_SQ, D, true, F_NONE>(a, sms, st, w, G);
  if (a.norm == 1) return launch_long_k<long long, K_L1, D, true, F_NONE>(a, sms, st, w, G);
  return launch_long_k<long long, K_LINF, D, true, F_NONE>(a, sms, st, w, G);
}

}  // namespace ffd
