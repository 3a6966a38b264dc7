// prep.cu — per-call preparation of a batch: band shape of every pair and a
// counting sort of the pairs by shape, longest first ("sorting
// the curves by their respective lengths before assigning them to batches").
//
// key = (nb − 1)·16 + (R − 1) where the pair's rows curve (the shorter one; δ is
// symmetric) is covered by nb bands of 32·R rows, R ≤ 16.  Pairs with a length
// < 1 get their invalid-output value here and are dropped; pairs too long for
// the batch kernel's band scratch go to the long-pair list.
#include "prep.cuh"
#include "seg.cuh"

namespace ffd {

// the invalid-output value of pair k: INT64_MIN (int64 out), NaN (float or double out)
// out_kind (the `int_out` argument): 0 float, 1 int64, 2 double
__device__ __forceinline__ void write_invalid(void* out, int64_t k, int out_kind) {
  if (out_kind == 1) reinterpret_cast<long long*>(out)[k] = LLONG_MIN;
  else if (out_kind == 2) reinterpret_cast<double*>(out)[k] = __longlong_as_double(0x7ff8000000000000ll);
  else reinterpret_cast<float*>(out)[k] = __int_as_float(0x7fc00000);
}

// shape key of pair k, and its descriptor; −1 when the pair is dropped (its
// invalid-output value written, or sent to the long-pair list)
__device__ __forceinline__ int pair_key(const int64_t* __restrict__ offsets,
                                        const int32_t* __restrict__ lengths, int64_t B, int64_t k,
                                        int int_out, int long_ok, void* __restrict__ out, PairDesc& d,
                                        int* __restrict__ long_list, int* __restrict__ long_count,
                                        int seg = 0) {
  const int n = lengths[k], m = lengths[B + k];
  if (n < 1 || m < 1) {
    write_invalid(out, k, int_out);
    return -1;
  }
  if (seg && long_ok > 0) {
    // the segmented kernel (seg.cuh): single-band Fréchet pairs, the longer curve on the rows
    const int bin = seg_bin(n, m, seg == 2);
    if (bin >= 0) {
      int W, R;
      seg_shape(bin / kSegHB, W, R);
      const bool swap = n < m;
      d.row_off = swap ? offsets[B + k] : offsets[k];
      d.col_off = swap ? offsets[k] : offsets[B + k];
      d.n_rows = swap ? m : n;
      d.m_cols = swap ? n : m;
      d.idx = (int)k;
      d.R = (uint8_t)R;
      d.nb = 1;
      d.swap = swap;
      d.pad = 0;
      return kNumKeys + bin;
    }
  }
  // Orientation: the rows (held in registers, R per lane) are the shorter curve,
  // unless a Fréchet pair is estimated cheaper with the LONGER curve as rows —
  // fewer column steps, each with more rows to spread the step's fixed
  // shuffle/select/load cost over (always so when the longer curve fits one band).  δ_dF
  // is symmetric and its value is one of the d_ij, so either orientation gives
  // the same bits; DTW (long_ok < 0) sums, so it keeps one orientation (the
  // fp32 mirror's).
  bool tall = false;
  if (long_ok > 0) {
    // estimated issue cost nb · (cols + 32 window steps) · (9.5 + 3.5·R) of each
    // orientation (the step's fixed part + ~3.5 instructions per cell-row)
    const int lo = n < m ? n : m, hi = n < m ? m : n;
    auto cost = [](int r, int c) {
      const int b = (r + kWarp * kMaxR - 1) / (kWarp * kMaxR);
      const int rr = (r + kWarp * b - 1) / (kWarp * b);
      return (float)b * (float)(c + kWarp) * (9.5f + 3.5f * (float)rr);
    };
    tall = hi <= kWarp * kMaxR * kMaxBands && cost(hi, lo) < cost(lo, hi);
  }
  const bool swap = tall ? n < m : n > m;
  const int rows = swap ? m : n, cols = swap ? n : m;
  const int nb = (rows + kWarp * kMaxR - 1) / (kWarp * kMaxR);
  // DTW (long_ok < 0): only the pairs the batch kernel cannot hold go to the
  // long-pair kernel; Fréchet (long_ok > 0) also sends the medium ones
  if (long_ok == -2 || (long_ok > 0 ? pair_goes_long(n, m, long_ok) : pair_too_long(n, m))) {
    if (long_ok && long_list) {
      long_list[atomicAdd(long_count, 1)] = (int)k;
    } else {  // no long-pair path requested (or its launch ruled out by the caller's length bounds): NaN
      write_invalid(out, k, int_out);
    }
    return -1;
  }
  const int R = (rows + kWarp * nb - 1) / (kWarp * nb);
  d.row_off = swap ? offsets[B + k] : offsets[k];
  d.col_off = swap ? offsets[k] : offsets[B + k];
  d.n_rows = rows;
  d.m_cols = cols;
  d.idx = (int)k;
  d.R = (uint8_t)R;
  d.nb = (uint8_t)nb;
  d.swap = swap;
  d.pad = 0;
  return (nb - 1) * kMaxR + (R - 1);
}

__global__ void prep_keys_kernel(const int64_t* __restrict__ offsets,
                                 const int32_t* __restrict__ lengths, int64_t B, int int_out, int long_ok,
                                 void* __restrict__ out, PairDesc* __restrict__ tmp,
                                 int16_t* __restrict__ keys, int* __restrict__ hist,
                                 int* __restrict__ long_list, int* __restrict__ long_count, int seg) {
  __shared__ int h[kAllKeys];
  const int nk = seg ? kAllKeys : kNumKeys;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < B;
       k += (int64_t)gridDim.x * blockDim.x) {
    PairDesc d;
    const int key = pair_key(offsets, lengths, B, k, int_out, long_ok, out, d, long_list, long_count, seg);
    if (key >= 0) {
      tmp[k] = d;
      atomicAdd(&h[key], 1);
    }
    keys[k] = (int16_t)key;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nk; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// Small batches (B ≤ kPrepSmallMax): the whole preparation in ONE block of
// kNumKeys·4 threads — counters zeroed, keys and histogram, the descending scan,
// the scatter — in place of the memset and three launches of the general path
// (for config 1's 16 pairs that chain is pure launch latency).  Each thread
// keeps its pairs' keys and descriptors in registers between the phases.
constexpr int kPrepSmallThreads = 1024;
constexpr int kPrepSmallPer = 4;  // pairs per thread

__global__ void __launch_bounds__(kPrepSmallThreads)
    prep_small_kernel(const int64_t* __restrict__ offsets, const int32_t* __restrict__ lengths,
                      int64_t B, int int_out, int long_ok, void* __restrict__ out,
                      int* __restrict__ counters, int* __restrict__ long_list,
                      PairDesc* __restrict__ sorted) {
  __shared__ int h[kNumKeys];
  __shared__ int s[kNumKeys];
  __shared__ int long_count;
  for (int i = threadIdx.x; i < kNumKeys; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) long_count = 0;
  __syncthreads();
  PairDesc d[kPrepSmallPer];
  int key[kPrepSmallPer];
#pragma unroll
  for (int u = 0; u < kPrepSmallPer; u++) {
    const int64_t k = threadIdx.x + (int64_t)u * blockDim.x;
    key[u] = -1;
    if (k < B) {
      key[u] = pair_key(offsets, lengths, B, k, int_out, long_ok, out, d[u], long_list, &long_count);
      if (key[u] >= 0) atomicAdd(&h[key[u]], 1);
    }
  }
  __syncthreads();
  // descending exclusive scan over the bins (as prep_scan_kernel)
  const int i = threadIdx.x;
  if (i < kNumKeys) s[i] = h[kNumKeys - 1 - i];
  __syncthreads();
  for (int o = 1; o < kNumKeys; o <<= 1) {
    const int v = (i < kNumKeys && i >= o) ? s[i - o] : 0;
    __syncthreads();
    if (i < kNumKeys) s[i] += v;
    __syncthreads();
  }
  int total = s[kNumKeys - 1];
  __syncthreads();
  if (i < kNumKeys) {
    const int bin = kNumKeys - 1 - i;
    h[bin] = s[i] - h[bin];  // h becomes the bin cursors
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kPrepSmallPer; u++)
    if (key[u] >= 0) sorted[atomicAdd(&h[key[u]], 1)] = d[u];
  if (threadIdx.x < kNumCtr)
    counters[threadIdx.x] = threadIdx.x == kCtrNumSorted ? total
                            : threadIdx.x == kCtrLong    ? long_count
                                                         : 0;
}

// one block of kNumKeys threads: descending-key exclusive scan -> bin cursors
__global__ void prep_scan_kernel(const int* __restrict__ hist, int* __restrict__ cursor,
                                 int* __restrict__ num_sorted) {
  __shared__ int s[kNumKeys];
  const int i = threadIdx.x;
  // position in descending order: bin i gets Σ_{j > i} hist[j]
  s[i] = hist[kNumKeys - 1 - i];
  __syncthreads();
  for (int o = 1; o < kNumKeys; o <<= 1) {
    int v = (i >= o) ? s[i - o] : 0;
    __syncthreads();
    s[i] += v;
    __syncthreads();
  }
  // s[i] = inclusive sum over reversed bins 0..i  ->  exclusive for bin (K-1-i)
  const int bin = kNumKeys - 1 - i;
  cursor[bin] = s[i] - hist[bin];
  if (i == kNumKeys - 1) *num_sorted = s[i];
}

__global__ void prep_scatter_kernel(const PairDesc* __restrict__ tmp,
                                    const int16_t* __restrict__ keys, int64_t B,
                                    int* __restrict__ cursor, PairDesc* __restrict__ sorted,
                                    PairDesc* __restrict__ seg_sorted) {
  // warp-aggregated: the lanes holding the same key take one atomicAdd for all
  // of them (a batch has only a handful of distinct shapes, so per-pair atomics
  // on one cursor serialise)
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < B; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = base + threadIdx.x;
    const int key = k < B ? keys[k] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int pos = 0;
    if (key >= 0 && lane == leader) pos = atomicAdd(&cursor[key], __popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader);
    if (key >= 0) (key >= kNumKeys ? seg_sorted : sorted)[pos + rank] = tmp[k];
  }
}


// exclusive scan of a[0, n) in shared memory by every thread of the block; returns the total
__device__ int block_scan_excl(int* a, int n) {
  __shared__ int wsum[32];
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = (n + blockDim.x - 1) / blockDim.x, b = threadIdx.x * P;
  int loc = 0;
  for (int i = 0; i < P; i++)
    if (b + i < n) loc += a[b + i];
  int v = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    int x = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    wsum[lane] = x;
  }
  __syncthreads();
  int excl = v - loc + (w > 0 ? wsum[w - 1] : 0);
  const int total = wsum[nw - 1];
  for (int i = 0; i < P; i++)
    if (b + i < n) {
      const int t = a[b + i];
      a[b + i] = excl;
      excl += t;
    }
  __syncthreads();
  return total;
}

// one block of 1024 threads: the batch kernel's bins (descending) as
// prep_scan_kernel, then the segmented kernel's bins (descending: the largest
// shape and period first) -> pair cursors (and a copy: the bin starts), and its
// groups (G pairs of one bin each) -> first group per bin (in rank order) and
// the group count.  off: [kSegBins] first group per rank, [kSegBins] bin starts
__global__ void __launch_bounds__(1024) prep_scan_seg_kernel(const int* __restrict__ hist, int* __restrict__ cursor,
                                                             int* __restrict__ off, int* __restrict__ counters) {
  __shared__ int s[kSegBins];
  for (int r = threadIdx.x; r < kNumKeys; r += blockDim.x) s[r] = hist[kNumKeys - 1 - r];
  const int total = block_scan_excl(s, kNumKeys);
  for (int r = threadIdx.x; r < kNumKeys; r += blockDim.x) cursor[kNumKeys - 1 - r] = s[r];
  __syncthreads();
  for (int r = threadIdx.x; r < kSegBins; r += blockDim.x) s[r] = hist[kNumKeys + kSegBins - 1 - r];
  block_scan_excl(s, kSegBins);
  for (int r = threadIdx.x; r < kSegBins; r += blockDim.x) {
    cursor[kNumKeys + kSegBins - 1 - r] = s[r];
    off[kSegBins + kSegBins - 1 - r] = s[r];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < kSegBins; r += blockDim.x) {
    const int bin = kSegBins - 1 - r, cnt = hist[kNumKeys + bin], gp = seg_group_pairs(bin);
    s[r] = (cnt + gp - 1) / gp;
  }
  const int groups = block_scan_excl(s, kSegBins);
  for (int r = threadIdx.x; r < kSegBins; r += blockDim.x) off[r] = s[r];
  __syncthreads();
  // per shape: its groups are contiguous (bins are shape-major): [first, end), and
  // its work Σ pairs · (W·R rows) · H (the kernel spreads the SMs over the shapes by it)
  if (threadIdx.x < kSegShapes) {
    const int sh = threadIdx.x;
    int W, R;
    seg_shape(sh, W, R);
    const int r_lo = kSegBins - 1 - (sh * kSegHB + kSegHB - 1);  // rank of the shape's highest bin
    int ng = 0;
    float work = 0.f;
    for (int b = 0; b < kSegHB; b++) {
      const int bin = sh * kSegHB + b, cnt = hist[kNumKeys + bin];
      ng += (cnt + kWarp / W - 1) / (kWarp / W);
      work += (float)cnt * (float)(W * R) * (float)((b + 1) * kSegHStep);
    }
    off[2 * kSegBins + 3 * sh] = off[r_lo];
    off[2 * kSegBins + 3 * sh + 1] = off[r_lo] + ng;
    off[2 * kSegBins + 3 * sh + 2] = __float_as_int(work);
  }
  if (threadIdx.x == 0) {
    counters[kCtrNumSorted] = total;
    counters[kCtrSegItems] = groups;
  }
}

// group i (after the scatter) -> its pair descriptors and shape: the bin whose
// group range holds i
__global__ void prep_seg_groups_kernel(const int* __restrict__ hist, const int* __restrict__ off,
                                       const int* __restrict__ counters, const PairDesc* __restrict__ seg_sorted,
                                       SegGroup* __restrict__ groups, int64_t max_groups) {
  const int n = counters[kCtrSegItems];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n && i < max_groups;
       i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = kSegBins;  // first rank with a first group > i
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (off[mid] <= i) lo = mid + 1;
      else hi = mid;
    }
    const int r = lo - 1, bin = kSegBins - 1 - r;
    const int gp = seg_group_pairs(bin), local = (int)i - off[r];
    const int cnt = hist[kNumKeys + bin];
    const int start = off[kSegBins + bin] + local * gp;
    SegGroup g;
    g.count = min(gp, cnt - local * gp);
    g.shape = bin / kSegHB;
    g.pad[0] = g.pad[1] = 0;
    g.d[0] = seg_sorted[start];
    g.d[1] = g.count > 1 ? seg_sorted[start + 1] : g.d[0];
    groups[i] = g;
  }
}

cudaError_t launch_prep(const int64_t* offsets, const int32_t* lengths, int64_t B, int int_out,
                        int long_ok, void* out, const BatchWs& ws, int num_sms, cudaStream_t st,
                        int64_t* launches, bool seg, bool long_run) {
  if (B == 0) return cudaSuccess;
  int* const long_list = long_run ? ws.long_list : nullptr;
  if (B <= kPrepSmallMax) {
    prep_small_kernel<<<1, kPrepSmallThreads, 0, st>>>(offsets, lengths, B, int_out, long_ok, out,
                                                       ws.counters, long_list, ws.sorted);
    *launches += 1;
    return cudaGetLastError();
  }
  if (cudaMemsetAsync(ws.counters, 0,
                      reinterpret_cast<char*>(ws.cursor) - reinterpret_cast<char*>(ws.counters),
                      st) != cudaSuccess)
    return cudaGetLastError();
  const int threads = 256;
  int64_t blocks = (B + threads - 1) / threads;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  prep_keys_kernel<<<(int)blocks, threads, 0, st>>>(offsets, lengths, B, int_out, long_ok, out, ws.tmp,
                                                    ws.keys, ws.hist, long_list,
                                                    ws.counters + kCtrLong, seg ? (seg_big() ? 2 : 1) : 0);
  if (seg) prep_scan_seg_kernel<<<1, 1024, 0, st>>>(ws.hist, ws.cursor, ws.seg_off, ws.counters);
  else prep_scan_kernel<<<1, kNumKeys, 0, st>>>(ws.hist, ws.cursor, ws.counters + kCtrNumSorted);
  prep_scatter_kernel<<<(int)blocks, threads, 0, st>>>(ws.tmp, ws.keys, B, ws.cursor, ws.sorted, ws.seg_sorted);
  *launches += 3;
  if (seg) {
    const int64_t mg = seg_max_groups(B);
    const int gb = (int)((mg + 255) / 256 < (int64_t)num_sms * 4 ? (mg + 255) / 256 : (int64_t)num_sms * 4);
    prep_seg_groups_kernel<<<gb, 256, 0, st>>>(ws.hist, ws.seg_off, ws.counters, ws.seg_sorted,
                                               reinterpret_cast<SegGroup*>(ws.seg_groups), mg);
    *launches += 1;
  }
  return cudaGetLastError();
}

}  // namespace ffd
