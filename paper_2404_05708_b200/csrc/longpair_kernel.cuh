// longpair_kernel.cuh — one very long pair spread over the whole GPU
// (BASELINE config 5).
//
// What: δ_dF of a pair with n rows (the shorter curve) and m columns, Eq. (1)
// in linear memory (Theorem 1): every warp keeps only
// its strip of rows and one column of DP state in registers.
//
// How:
//   * The rows are cut into bands of 32·R rows; band b runs on one warp as the
//     lane-strip wavefront of strip.cuh (lane ℓ: rows [ℓR, ℓR+R), column t−ℓ at
//     step t) and streams all m columns once.
//   * Band b's bottom row (lane 31's value, one per column) is band b+1's top
//     input.  It moves through LINKS: rings of 8-byte slots {value, tag} written
//     by lane 31 with one 64-bit store, tag = absolute stream position + 1.  The
//     consumer polls the slot itself, so data and "ready" arrive together and no
//     fence or flag is needed (the low-latency protocol NCCL calls LL).  Inside
//     a CTA the ring is in shared memory; between CTAs (warp 7 → next CTA's
//     warp 0) it is in global memory (L2).
//   * The consumer prefetches the slots of the next 32 columns one chunk ahead
//     (like the column points), checks the tags when it stores them into its
//     column ring, and re-polls only the slots that were not ready.  It
//     publishes how far it has consumed; the producer checks that counter (also
//     prefetched) before reusing slots: bounded rings, no overwrite.
//   * Slots are indexed by the ABSOLUTE stream position (tag base + position) so
//     that slot reuse distance is exactly the ring size across successive pairs —
//     the flow-control test (consumed + ring > absolute position) is only valid
//     then.  (Indexing by the position within a pair let a producer that had
//     moved on to the next pair overwrite the previous pair's last unconsumed
//     slots whenever a stream length was not a multiple of the ring size: a hang.)
//   * One persistent CTA of 8 warps per SM, cooperative launch: all bands are
//     co-resident, so spinning on a neighbour cannot deadlock.  Counters and
//     tags are absolute positions, so successive long pairs need no grid barrier.
#pragma once
#include <climits>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "longpair.cuh"
#include "strip.cuh"

namespace ffd {

constexpr int kLWarps = 8;          // warps (bands) per CTA
constexpr int kLSmemRing = 1024;    // slots per intra-CTA link (8 KB; the producer may run
                                    // ~500 steps ahead, far beyond the ~47 the consumer needs)
constexpr int kLGlobRing = 2048;    // slots per inter-CTA link
constexpr int kMaxLongCtas = 1024;
// a spin on a link that has not advanced for this many SM cycles (≈ 2.5 s)
// reports the link state with printf and gives up instead of hanging the GPU
constexpr long long kWatchdogCycles = 5000000000LL;

struct LongProblem {
  const void* p;
  const void* q;
  const int64_t* offsets;
  const int32_t* lengths;
  int64_t num_pairs;
  const int* list;
  const int* list_count;
  void* out;
  uint2* gring;    // [G][kLGlobRing] slots of the link CTA g → g+1 (zeroed per call)
  unsigned* gcons; // [G] consumer progress on the link CTA g → g+1 (zeroed per call)
  int* bad;        // per long pair: a point left the fp32-exact window (int input)
  int trace;       // FFD_LONG_TRACE=1: print each band's start/first-step/end time
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint2 ld_slot(const uint2* p) {
  uint2 v;
  asm volatile("ld.relaxed.gpu.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_slot(uint2* p, float v, unsigned tag) {
  asm volatile("st.relaxed.gpu.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(__float_as_uint(v)), "r"(tag)
               : "memory");
}
__device__ __forceinline__ void st_slot_pred(uint2* p, float v, unsigned tag, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\t@q st.relaxed.gpu.v2.u32 [%0], {%1, %2};\n\t}" ::"l"(p),
      "r"(__float_as_uint(v)), "r"(tag), "r"(pred)
      : "memory");
}
// two adjacent slots {v0, tag}, {v1, tag + 1} in one predicated 16-byte store
__device__ __forceinline__ void st_slot2_pred(uint2* p, float v0, float v1, unsigned tag, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t@q st.relaxed.gpu.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
      "r"(__float_as_uint(v0)), "r"(tag), "r"(__float_as_uint(v1)), "r"(tag + 1u), "r"(pred));
}
__device__ __forceinline__ unsigned ld_ctr(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_ctr(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// one link endpoint: ring of slots (mask = size − 1) and the consumer counter
struct Link {
  uint2* ring;
  unsigned mask;
  unsigned* cons;
};

template <int KIND, int D, bool INT_IN, int FIN, int R>
struct LongRunner {
  using T = float;
  using C = SCfg<T, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  static constexpr int NS = C::NS;

  uint4* ring;  // this warp's column ring [kRing * EW]
  const LongProblem& pb;
  int lane;

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

  // column element of position `pos` (0 = sentinel), written with its top value
  __device__ void store_elem(const In (&a)[D], int kind, int pos, float top, bool& ok) {
    alignas(16) float f[C::EBYTES / 4];
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
    f[C::I_TOP] = top;
    uint4* dst = ring + (pos & kRingMask) * C::EW;
#pragma unroll
    for (int w = 0; w < C::EW; w++) dst[w] = reinterpret_cast<const uint4*>(f)[w];
  }

  // positions: 0 = sentinel, p ∈ [1, m] = column p − 1, and when m + 1 is odd one
  // more copy of the last column (repeating a point leaves δ unchanged, PAPER
  // L259 footnote) so the stream has an even length S2 (two columns per step)
  __device__ void fetch(int pos, int S2, In (&a)[D], int& kind) const {
#pragma unroll
    for (int c = 0; c < D; c++) a[c] = (In)0;
    if (pos >= S2) {
      kind = 2;
    } else if (pos == 0) {
      kind = 1;
    } else {
      kind = 0;
      const int64_t col = min(pos - 1, m - 1);
#pragma unroll
      for (int c = 0; c < D; c++) a[c] = __ldg(cols + col * D + c);
    }
  }

  // top value of position `pos` for this band: the corner/border for band 0,
  // else the producer's slot (spinning until its tag shows up)
  __device__ __forceinline__ float top_of(int pos, int S2, bool has_in, const Link& in, unsigned tb,
                                          uint2 pre) const {
    if (pos >= S2) return finf();
    if (!has_in) return pos == 0 ? 0.f : finf();
    const unsigned want = tb + (unsigned)pos + 1u;
    if (pre.y != want) {
      const long long t0 = clock64();
      while (pre.y != want) {
        pre = ld_slot(in.ring + ((tb + (unsigned)pos) & in.mask));
        if (clock64() - t0 > kWatchdogCycles) {  // a link that never delivers: report, give up
          printf("ffd long_kernel watchdog: consumer cta %d lane %d pos %d want tag %u saw %u (tb %u)\n",
                 (int)blockIdx.x, lane, pos, want, pre.y, tb);
          break;
        }
      }
    }
    return __uint_as_float(pre.x);
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
      const uint2* slot = in.ring + ((tb + (unsigned)pos) & in.mask);
      if (ld_slot(slot).y != want) {
        const long long t0 = clock64();
        while (ld_slot(slot).y != want) {
          __nanosleep(64);
          if (clock64() - t0 > kWatchdogCycles) {
            printf("ffd long_kernel watchdog: chunk wait cta %d pos %d want tag %u (tb %u)\n",
                   (int)blockIdx.x, pos, want, tb);
            break;
          }
        }
      }
    }
    __syncwarp();
  }

  // one band of 32·R rows starting at row r0, two columns per warp step
  // (strip.cuh warp_step2: lane ℓ at step t works on columns 2(t−ℓ), 2(t−ℓ)+1)
  __device__ bool run_band(int r0, bool has_in, Link in, bool has_out, Link out, bool last_band,
                           int out_idx, int* bad_flag, unsigned tb) {
    const int S2 = (m + 2) & ~1;  // positions (even)
    const int NT = S2 / 2;        // steps
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
    float diag = finf(), b0 = finf();
    const uint2 none = make_uint2(0u, 0u);
    // prologue: positions [0, 32) stored; column points of [32, 64) and [64, 96)
    // in flight (two chunks ahead: one 16-step chunk does not cover the L2/HBM
    // latency of a latency-bound warp); link slots of [32, 64) in flight
    In a[D], a2[D];
    int kind, kind2;
    fetch(lane, S2, a, kind);
    wait_chunk(31, S2, has_in, in, tb);
    uint2 pre = (has_in && lane < S2) ? ld_slot(in.ring + ((tb + (unsigned)lane) & in.mask)) : none;
    store_elem(a, kind, lane, top_of(lane, S2, has_in, in, tb, pre), ok);
    fetch(32 + lane, S2, a, kind);
    fetch(64 + lane, S2, a2, kind2);
    pre = (has_in && 32 + lane < S2) ? ld_slot(in.ring + ((tb + (unsigned)(32 + lane)) & in.mask)) : none;
    __syncwarp();
    if (has_in && lane == 0) st_ctr(in.cons, tb + (unsigned)min(32, S2));
    unsigned cons_seen = 0, cons_next = 0;
    if (has_out) cons_seen = cons_next = ld_ctr(out.cons);

    const int total = NT + 31;
    const int pown = (has_out && lane == kWarp - 1) ? 1 : 0;
    const unsigned omask = out.mask & ~1u;
    int t = 0, next_refill = 16;
    while (t < total) {
      if (t == next_refill) {
        // the slots of this chunk were prefetched one chunk ago: when every tag
        // is already there, go on without touching the link (a blocking poll of
        // an L2 link costs ~700 cycles per chunk); else wait on lane 0 first
        if (2 * t < S2 && has_in) {
          const int pos = 2 * t + lane;
          const bool ready = pos >= S2 || pre.y == tb + (unsigned)pos + 1u;
          if (!__all_sync(0xffffffffu, ready)) wait_chunk(2 * t + 31, S2, has_in, in, tb);
        }
        store_elem(a, kind, 2 * t + lane, top_of(2 * t + lane, S2, has_in, in, tb, pre), ok);
#pragma unroll
        for (int cc = 0; cc < D; cc++) a[cc] = a2[cc];
        kind = kind2;
        fetch(2 * t + 64 + lane, S2, a2, kind2);
        const int pn = 2 * t + 32 + lane;
        pre = (has_in && pn < S2) ? ld_slot(in.ring + ((tb + (unsigned)pn) & in.mask)) : none;
        __syncwarp();
        if (has_in && lane == 0) st_ctr(in.cons, tb + (unsigned)min(2 * t + 32, S2));
        next_refill += 16;
      }
      if (has_out && (t & 15) == 0) {
        // lane 31 writes positions < 2t during the next 16 steps: their slots
        // must be consumed (cons + ring > tb + 2t).  The counter is read a chunk ahead.
        if (lane == kWarp - 1) {
          cons_seen = cons_next;
          if ((int)(cons_seen + out.mask + 1u - (tb + 2u * (unsigned)t)) <= 0) {
            const long long t0 = clock64();
            while ((int)(cons_seen + out.mask + 1u - (tb + 2u * (unsigned)t)) <= 0) {
              __nanosleep(64);
              cons_seen = ld_ctr(out.cons);
              if (clock64() - t0 > kWatchdogCycles) {
                printf("ffd long_kernel watchdog: producer cta %d warp %d t %d cons %u tb %u ring %u\n",
                       (int)blockIdx.x, (int)(threadIdx.x >> 5), t, cons_seen, tb, out.mask + 1u);
                break;
              }
            }
          }
          cons_next = ld_ctr(out.cons);
        }
      }
      __syncwarp();
      const int stop = min(next_refill, total);
      int g = t - lane;
      // the ring elements of the next step are loaded one step ahead (the
      // volatile link store would otherwise pin each load next to its use)
      // software-pipelined steps (strip.cuh Pipe2): the distances of step g+1 are
      // computed during step g's chain and the ring element of g+2 is loaded;
      // primed again after every refill (its look-ahead may read unstored slots)
      Pipe2<float, KIND, D, R, INT_IN> pipe;
      pipe.prime(x, ring, g);
      // lane 31 publishes its two bottom-row values {value, tag} of every step
      // with one predicated 16-byte store (no divergent branch per step)
      auto one = [&](int gg) {
        pipe.step(c, diag, b0, x, ring, gg, lane);
        st_slot2_pred(out.ring + ((tb + 2u * (unsigned)gg) & omask), b0, c[R - 1],
                      tb + 2u * (unsigned)gg + 1u, pown & ((unsigned)gg < (unsigned)NT));
      };
#pragma unroll 1
      for (; t + 2 <= stop; t += 2, g += 2) {
        one(g);
        one(g + 1);
      }
      if (t < stop) {
        one(g);
        ++t;
      }
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    if (last_band && lane == kWarp - 1) {
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

// rows per lane for a pair with n rows on G co-resident CTAs: the smallest
// built R whose bands all fit at once (⌈bands / 8⌉ ≤ G); 0 if none does
__host__ __device__ inline int long_rows_per_lane(int n, int G) {
  const int rs[5] = {4, 7, 8, 16, 32};  // the R the long kernel is built for
  for (int i = 0; i < 5; i++) {
    const int R = rs[i];
    const int nb = (n + kWarp * R - 1) / (kWarp * R);
    if ((nb + kLWarps - 1) / kLWarps <= G) return R;
  }
  return 0;
}

template <int KIND, int D, bool INT_IN, int FIN>
__global__ void __launch_bounds__(kWarp* kLWarps, 1) long_kernel(const LongProblem pb) {
  using C = SCfg<float, KIND, D, INT_IN>;
  using In = typename std::conditional<INT_IN, int32_t, float>::type;
  // dynamic shared memory: [kLWarps][kLSmemRing] link slots, [kLWarps][kRing·EW]
  // column rings, [kLWarps] consumer counters
  extern __shared__ uint4 lsm[];
  uint2 (*slink)[kLSmemRing] = reinterpret_cast<uint2(*)[kLSmemRing]>(lsm);
  uint4 (*rings)[kRing * C::EW] =
      reinterpret_cast<uint4(*)[kRing * C::EW]>(lsm + kLWarps * kLSmemRing / 2);
  unsigned* scons = reinterpret_cast<unsigned*>(lsm + kLWarps * kLSmemRing / 2 + kLWarps * kRing * C::EW);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  // Thread-block cluster: consecutive CTAs of a cluster link warp 7 → next CTA's
  // warp 0 through DISTRIBUTED shared memory (the producer stores {value, tag}
  // slots straight into the consumer CTA's smem ring slink[7], which warp 7 of
  // that CTA does not use itself; the consumer publishes its progress into its
  // own scons[7], which the producer reads remotely).  Only the link between
  // clusters goes through L2.
  // nothing to do (the common case of a batch without long pairs): leave before
  // initialising 64 KB of link rings; every CTA takes the same exit, so no
  // cluster barrier is left waiting
  if (*pb.list_count == 0) return;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int csize = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  const int npairs = *pb.list_count;
  for (int i = threadIdx.x; i < kLWarps * kLSmemRing; i += blockDim.x)
    (&slink[0][0])[i] = make_uint2(0u, 0u);
  if (threadIdx.x < kLWarps) scons[threadIdx.x] = 0u;
  // this call's global link state: tags restart at 1 every call, so a slot left
  // from an earlier call must read as empty — zeroed here (instead of a memset
  // on every batch call, most of which have no long pair) before the grid barrier
  for (int i = threadIdx.x; i < kLGlobRing; i += blockDim.x)
    pb.gring[(size_t)cta * kLGlobRing + i] = make_uint2(0u, 0u);
  if (threadIdx.x == 0) pb.gcons[cta] = 0u;
  for (int i = cta * (int)blockDim.x + (int)threadIdx.x; i < npairs; i += G * (int)blockDim.x) pb.bad[i] = 0;
  __syncthreads();
  cl.sync();  // every CTA of the cluster has initialised its rings before any remote access
  cg::this_grid().sync();  // and every CTA its global ring before any consumer polls it
  // CTA groups: several long pairs run side by side, each on a contiguous group
  // of Gg CTAs (pair li on group li mod NG).  Gg is what the largest pair needs
  // at R = 16; a single very long pair (config 5) keeps the whole grid.  Every
  // CTA computes the same NG from the same lengths.
  int need = 1;
  for (int li = 0; li < npairs; li++) {
    const int k = pb.list[li];
    const int n0 = pb.lengths[k], m0 = pb.lengths[pb.num_pairs + k];
    const int rows = n0 < m0 ? n0 : m0;
    const int nb16 = (rows + kWarp * 16 - 1) / (kWarp * 16);
    need = max(need, (nb16 + kLWarps - 1) / kLWarps);
  }
  need = min(need, G);
  const int NG = max(1, min(G / need, npairs));
  const int Gg = G / NG;
  const int grp = cta / Gg, local = cta - grp * Gg;
  unsigned tb = 0;  // tag base: absolute stream position of the current pair on every link
  for (int li = grp; li < npairs && grp < NG; li += NG) {
    const int k = pb.list[li];
    const int64_t B = pb.num_pairs;
    const int n0 = pb.lengths[k], m0 = pb.lengths[B + k];
    const bool swap = n0 > m0;
    const int n = swap ? m0 : n0, m = swap ? n0 : m0;
    const In* rows = reinterpret_cast<const In*>(swap ? pb.q : pb.p) +
                     (swap ? pb.offsets[B + k] : pb.offsets[k]) * D;
    const In* cols = reinterpret_cast<const In*>(swap ? pb.p : pb.q) +
                     (swap ? pb.offsets[k] : pb.offsets[B + k]) * D;
    const int R = long_rows_per_lane(n, Gg);
    const int S = (m + 2) & ~1;  // stream positions of this pair (even, see run_band)
    if (R == 0) {
      if (local == 0 && threadIdx.x == 0) {
        if constexpr (INT_IN) reinterpret_cast<long long*>(pb.out)[k] = LLONG_MIN;
        else reinterpret_cast<float*>(pb.out)[k] = __int_as_float(0x7fc00000);
      }
      continue;
    }
    const int band_rows = kWarp * R;
    const int nb = (n + band_rows - 1) / band_rows;
    const int b = local * kLWarps + warp;  // band of this warp within the group's pair
    if (!(b < nb && b > 0) && lane == 0 && b > 0) {
      // this warp does not consume its input link for this pair: its producer
      // (if any) writes nothing of it either, so mark the whole stream consumed —
      // otherwise the producer of a later pair would wait on a stale counter
      unsigned* cons = (warp > 0) ? &scons[warp - 1]
                                  : (crank > 0 ? &scons[kLWarps - 1] : pb.gcons + (cta - 1));
      st_ctr(cons, tb + (unsigned)S);
    }
    if (b < nb) {
      const bool has_in = b > 0, has_out = b + 1 < nb;
      Link in{}, out{};
      // b > 0 with warp 0 means local > 0: the previous CTA is in this group
      if (warp > 0) {
        in = Link{slink[warp - 1], kLSmemRing - 1u, &scons[warp - 1]};
      } else if (b > 0 && crank > 0) {  // DSMEM link from the previous CTA of this cluster
        in = Link{slink[kLWarps - 1], kLSmemRing - 1u, &scons[kLWarps - 1]};
      } else if (b > 0) {
        const int src = cta - 1;
        in = Link{pb.gring + (size_t)src * kLGlobRing, kLGlobRing - 1u, pb.gcons + src};
      }
      // has_out with warp 7 means the next CTA (local + 1 < Gg) is in this group
      if (warp < kLWarps - 1) {
        out = Link{slink[warp], kLSmemRing - 1u, &scons[warp]};
      } else if (has_out && crank + 1 < csize) {  // DSMEM link into the next CTA of this cluster
        out = Link{cl.map_shared_rank(slink[kLWarps - 1], crank + 1), kLSmemRing - 1u,
                   cl.map_shared_rank(&scons[kLWarps - 1], crank + 1)};
      } else {
        out = Link{pb.gring + (size_t)cta * kLGlobRing, kLGlobRing - 1u, pb.gcons + cta};
      }
      auto go = [&](auto& run) {
        run.n = n;
        run.m = m;
        run.rows = rows;
        run.cols = cols;
        if constexpr (INT_IN) {
#pragma unroll
          for (int c = 0; c < D; c++) run.center[c] = (int)rows[c];
        }
        const unsigned long long t0 = pb.trace ? gtimer() : 0ull;
        run.run_band(b * band_rows, has_in, in, has_out, out, b == nb - 1, k, pb.bad + li, tb);
        if (pb.trace && lane == 0)
          printf("ffdtrace band %d cta %d warp %d start %llu end %llu\n", b, cta, warp, t0, gtimer());
      };
      if (R == 4) {
        LongRunner<KIND, D, INT_IN, FIN, 4> run{rings[warp], pb, lane};
        go(run);
      } else if (R == 7) {
        LongRunner<KIND, D, INT_IN, FIN, 7> run{rings[warp], pb, lane};
        go(run);
      } else if (R == 8) {
        LongRunner<KIND, D, INT_IN, FIN, 8> run{rings[warp], pb, lane};
        go(run);
      } else if (R == 16) {
        LongRunner<KIND, D, INT_IN, FIN, 16> run{rings[warp], pb, lane};
        go(run);
      } else {
        LongRunner<KIND, D, INT_IN, FIN, 32> run{rings[warp], pb, lane};
        go(run);
      }
    }
    __syncthreads();
    tb += (unsigned)S;  // every link's absolute position advances by one stream per pair
  }
  cl.sync();  // no CTA leaves while a cluster neighbour may still access its smem
}

struct LongWs {
  uint2* gring;
  unsigned* gcons;
  int* bad;
};

// One persistent CTA (8 bands) per SM, cooperative launch.  BASELINE config 5
// (n = 262,144) runs as 147 CTAs of 8 bands × 224 rows (R = 7).
template <int KIND, int D, bool INT_IN, int FIN>
cudaError_t launch_long_k(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G) {
  auto k = long_kernel<KIND, D, INT_IN, FIN>;
  using C = SCfg<float, KIND, D, INT_IN>;
  const size_t smem = sizeof(uint2) * kLWarps * kLSmemRing + sizeof(uint4) * kLWarps * kRing * C::EW +
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
  LongProblem pb{a.p,      a.q,       a.offsets, a.lengths, a.num_pairs, a.list,
                 a.list_count, a.out, w.gring,   w.gcons,   w.bad, trace};
  void* args[] = {&pb};
  // clusters of 8 CTAs (DSMEM links inside a cluster), cooperative so that every
  // CTA is co-resident; falls back to plain cooperative CTAs if the device
  // cannot co-schedule the clusters (FFD_LONG_CLUSTER=1 forces that)
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
    // (or leave a pair that needs every CTA without a feasible R)
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
cudaError_t launch_long_dim1(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G);
cudaError_t launch_long_dim2(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G);
cudaError_t launch_long_dim3(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G);
cudaError_t launch_long_dim4(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G);

template <int D>
cudaError_t launch_long_dim(const LongArgs& a, int sms, cudaStream_t st, const LongWs& w, int G) {
  const bool i = a.dtype == 1;
  if (!i) {
    if (a.norm == 1) return launch_long_k<K_L1, D, false, F_NONE>(a, sms, st, w, G);
    if (a.norm == 3) return launch_long_k<K_LINF, D, false, F_NONE>(a, sms, st, w, G);
    if (a.norm == 2) return launch_long_k<K_SQ, D, false, F_SQRT>(a, sms, st, w, G);
    return launch_long_k<K_SQ, D, false, F_NONE>(a, sms, st, w, G);
  }
  if (a.norm == 4) return launch_long_k<K_XSQ, D, true, F_NONE>(a, sms, st, w, G);
  if (a.norm == 1) return launch_long_k<K_L1, D, true, F_NONE>(a, sms, st, w, G);
  return launch_long_k<K_LINF, D, true, F_NONE>(a, sms, st, w, G);
}

}  // namespace ffd
