// api.cu — the C ABI of include/ffd.h: argument checks, workspace layout,
// dispatch to the compiled kernel instantiations, stream-ordered launches.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "cdist.cuh"
#include "distsum.cuh"
#include "ffd.h"
#include "longpair.cuh"
#include "prep.cuh"
#include "registry.h"
#include "seg.cuh"
#include "strip.cuh"
#include "validate.cuh"

namespace ffd {

// ---- registry -------------------------------------------------------------
static std::vector<BatchEntry>& registry() {
  static std::vector<BatchEntry> r;
  return r;
}
static std::mutex& reg_mutex() {
  static std::mutex m;
  return m;
}
void register_batch(const BatchEntry& e) {
  std::lock_guard<std::mutex> g(reg_mutex());
  registry().push_back(e);
}
const BatchEntry* find_batch(const BatchKey& k) {
  std::lock_guard<std::mutex> g(reg_mutex());
  for (auto& e : registry())
    if (e.key.tier == k.tier && e.key.kind == k.kind && e.key.dim == k.dim &&
        e.key.int_in == k.int_in && e.key.fin == k.fin)
      return &e;
  return nullptr;
}

// ---- device facts -----------------------------------------------------------
struct DevInfo {
  int sms = 0;
};
static DevInfo dev_info() {
  static DevInfo cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DevInfo{148};
  if (cache[dev].sms == 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev].sms = sms;
  }
  return cache[dev];
}

static thread_local int64_t g_launches = 0;

// ---- profiling hook: event pairs around the dominant kernel -----------------
static std::mutex g_prof_mu;
static std::atomic<int> g_prof_on{0};
struct ProfRec {
  int tag;  // which kernel: 0 batch main tier, 1 exact int64 tier, 2 long pair, 3 cdist
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof_events;

struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  int tag;
  ProfScope(cudaStream_t s, int t) : st(s), tag(t) {
    if (!g_prof_on.load()) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_events.push_back(ProfRec{tag, a, b});
  }
};

constexpr int kMaxCtasMain = kMinCtasPerSm > 4 ? kMinCtasPerSm : 4;  // cap on resident CTAs/SM used to size scratch
constexpr int kCtasFb = 1;

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace layout for a batch of B pairs on a device with `sms` SMs
static BatchWs batch_layout(void* base, int64_t B, int sms) {
  BatchWs w{};
  size_t off = 0;
  char* b = reinterpret_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  w.counters = reinterpret_cast<int*>(take(sizeof(int) * kNumCtr));
  w.hist = reinterpret_cast<int*>(take(sizeof(int) * kAllKeys));
  w.cursor = reinterpret_cast<int*>(take(sizeof(int) * kAllKeys));
  w.tmp = reinterpret_cast<PairDesc*>(take(sizeof(PairDesc) * (size_t)B));
  w.sorted = reinterpret_cast<PairDesc*>(take(sizeof(PairDesc) * (size_t)B));
  w.keys = reinterpret_cast<int16_t*>(take(sizeof(int16_t) * (size_t)B));
  w.fb_list = reinterpret_cast<int*>(take(sizeof(int) * (size_t)B));
  w.long_list = reinterpret_cast<int*>(take(sizeof(int) * (size_t)B));
  const size_t warps_main = (size_t)sms * kMaxCtasMain * kWarpsPerCta;
  const size_t warps_fb = (size_t)sms * kCtasFb * kWarpsPerCta;
  w.scratch_main = reinterpret_cast<float*>(take(warps_main * 2 * kScratchCols * sizeof(float)));
  w.scratch_fb = reinterpret_cast<long long*>(take(warps_fb * 2 * kScratchCols * sizeof(long long)));
  w.seg_sorted = reinterpret_cast<PairDesc*>(take(sizeof(PairDesc) * (size_t)B));
  w.seg_groups = take(sizeof(SegGroup) * (size_t)seg_max_groups(B));
  w.seg_off = reinterpret_cast<int*>(take(sizeof(int) * (2 * kSegBins + 3 * kSegShapes)));
  w.bytes = off;
  return w;
}

static int kind_for(int norm, int dtype) {
  if (dtype == FFD_I32) return norm == FFD_SQL2 ? K_XSQ : (norm == FFD_L1 ? K_L1 : K_LINF);
  return norm == FFD_L1 ? K_L1 : (norm == FFD_LINF ? K_LINF : K_SQ);
}

static int check_common(int32_t dim, int32_t norm, int32_t dtype) {
  if (dim < 1 || dim > 4) return FFD_ERR_ARG;
  if (norm < FFD_L1 || norm > FFD_SQL2) return FFD_ERR_ARG;
  if (dtype != FFD_F32 && dtype != FFD_I32) return FFD_ERR_ARG;
  if (dtype == FFD_I32 && norm == FFD_L2) return FFD_ERR_ARG;
  return FFD_OK;
}

// measure: 0 discrete Fréchet (Eq. (1)), 1 DTW (Appendix B), 2 DTW in fp64
static int batch_impl(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                      int64_t B, int32_t dim, int32_t norm, int32_t dtype, void* out,
                      void* workspace, size_t ws_bytes, cudaStream_t st, int measure = 0,
                      bool long_possible = true) {
  int s = check_common(dim, norm, dtype);
  if (s) return s;
  if (measure != 0 && dtype != FFD_F32) return FFD_ERR_UNSUPPORTED;
  if (B < 0) return FFD_ERR_ARG;
  if (B == 0) return FFD_OK;
  if (!p || !q || !offsets || !lengths || !out) return FFD_ERR_ARG;
  if (B > INT_MAX / 2) return FFD_ERR_UNSUPPORTED;
  const DevInfo di = dev_info();
  BatchWs ws = batch_layout(workspace, B, di.sms);
  if (!workspace || ws_bytes < ws.bytes) return FFD_ERR_WORKSPACE;

  const int int_in = dtype == FFD_I32;
  int kind = kind_for(norm, dtype);
  int fin = (norm == FFD_L2) ? F_SQRT : F_NONE;
  if (measure != 0) {  // DTW: L2 needs the per-cell square root (sums do not commute with it)
    if (norm == FFD_L2) kind = K_SQRT;
    fin = F_DTW;
  }
  const BatchEntry* main_e = find_batch(BatchKey{measure == 2 ? 2 : 0, kind, dim, int_in, fin});
  if (!main_e) return FFD_ERR_UNSUPPORTED;
  const BatchEntry* fb_e = nullptr;
  if (int_in) {
    const int fkind = norm == FFD_SQL2 ? K_SQ : (norm == FFD_L1 ? K_L1 : K_LINF);
    fb_e = find_batch(BatchKey{1, fkind, dim, 1, F_NONE});
    if (!fb_e) return FFD_ERR_UNSUPPORTED;
  }

  // Fréchet: pairs too long for the bands, and the medium ones, go to the long-pair
  // kernel; DTW (−1): only those too long for the bands (its sums keep one orientation)
  const bool dtw_all_long = measure == 1 && getenv("FFD_DTW_LONG") != nullptr;  // testing: every DTW pair long
  // (the fp64 DTW tier has no long-pair path: 0, such pairs get NaN)
  const int long_ok = measure == 0 ? medium_rows_for(B, di.sms) : measure == 2 ? 0 : (dtw_all_long ? -2 : -1);
  const int out_kind = int_in ? 1 : (measure == 2 ? 2 : 0);
  // single-band Fréchet pairs of the built cells go to the segmented kernel (seg.cuh)
  const bool use_seg = measure == 0 && B > kPrepSmallMax && seg_supported(kind, dim, int_in, fin);
  if (launch_prep(offsets, lengths, B, out_kind, long_ok, out, ws, di.sms, st, &g_launches, use_seg,
                  long_possible && measure != 2) !=
      cudaSuccess)
    return FFD_ERR_CUDA;

  Problem pb{};
  pb.p = p;
  pb.q = q;
  pb.offsets = offsets;
  pb.lengths = lengths;
  pb.num_pairs = B;
  pb.sorted = ws.sorted;
  pb.num_sorted = ws.counters + kCtrNumSorted;
  pb.counter = ws.counters + kCtrChunkMain;
  pb.out = out;
  pb.scratch = ws.scratch_main;
  pb.fb_list = ws.fb_list;
  pb.fb_count = ws.counters + kCtrFb;
  std::memcpy(pb.rmap, main_e->rmap, sizeof(pb.rmap));
  int occ = main_e->occupancy();
  if (occ < 1) occ = 1;
  if (occ > kMaxCtasMain) occ = kMaxCtasMain;
  // fp64 DTW: 8-byte band scratch in the float-sized buffer holds half the warps
  if (measure == 2 && occ > kMaxCtasMain / 2) occ = kMaxCtasMain / 2;
  {
    // chunk size: kChunkPairs, unless the batch is too small to give every
    // resident warp at least one chunk (then fewer pairs per chunk)
    const int64_t warps = (int64_t)di.sms * occ * kWarpsPerCta;
    int64_t ch = (B + warps - 1) / warps;
    pb.chunk = (int)(ch < 1 ? 1 : (ch > kChunkPairs ? kChunkPairs : ch));
  }
  {
    ProfScope prof(st, 0);
    // no more CTAs than there are chunks to take (a small batch would otherwise
    // start hundreds of CTAs that only find the chunk counter exhausted)
    const int64_t chunks = (B + pb.chunk - 1) / pb.chunk;
    const int64_t need = (chunks + kWarpsPerCta - 1) / kWarpsPerCta;
    const int ctas = (int)(need < (int64_t)di.sms * occ ? need : (int64_t)di.sms * occ);
    if (main_e->launch(pb, ctas, st) != cudaSuccess) return FFD_ERR_CUDA;
    ++g_launches;
    if (use_seg) {
      SegProblem sp{};
      sp.p = p;
      sp.q = q;
      sp.groups = reinterpret_cast<const SegGroup*>(ws.seg_groups);
      sp.n_groups = ws.counters + kCtrSegItems;
      sp.shape_info = ws.seg_off + 2 * kSegBins;
      sp.shape_ctr = ws.counters + kCtrSegShape;
      sp.out = out;
      sp.fb_list = ws.fb_list;
      sp.fb_count = ws.counters + kCtrFb;
      if (launch_seg(sp, kind, dim, int_in, fin, di.sms, st, &g_launches) != cudaSuccess) return FFD_ERR_CUDA;
    }
  }

  if (fb_e) {
    Problem fb = pb;
    fb.list = ws.fb_list;
    fb.list_count = ws.counters + kCtrFb;
    fb.counter = ws.counters + kCtrChunkFb;
    fb.chunk = kChunkPairs;
    fb.scratch = reinterpret_cast<float*>(ws.scratch_fb);
    fb.fb_list = nullptr;
    fb.fb_count = nullptr;
    std::memcpy(fb.rmap, fb_e->rmap, sizeof(fb.rmap));
    ProfScope prof(st, 1);
    if (fb_e->launch(fb, di.sms * kCtasFb, st) != cudaSuccess) return FFD_ERR_CUDA;
    ++g_launches;
  }

  if (!long_possible || measure == 2) return FFD_OK;  // no pair is long (caller saw every length), or fp64 DTW
  // pairs too long for the band scratch of the batch kernel: cross-CTA wavefront
  LongArgs la{};
  la.p = p;
  la.q = q;
  la.offsets = offsets;
  la.lengths = lengths;
  la.num_pairs = B;
  la.dim = dim;
  la.norm = norm;
  la.dtype = dtype;
  la.measure = measure;
  la.list = ws.long_list;
  la.list_count = ws.counters + kCtrLong;
  la.out = out;
  // the band scratch of the batch kernel (done with it: stream order) buffers
  // the wrap link of multi-pass pairs
  la.wrap = ws.scratch_main;
  la.wrap_bytes = (size_t)(reinterpret_cast<char*>(ws.scratch_fb) - reinterpret_cast<char*>(ws.scratch_main));
  ProfScope prof(st, 2);
  if (launch_long_pairs(la, di.sms, st, &g_launches) != cudaSuccess) return FFD_ERR_CUDA;
  return FFD_OK;
}

// ---- all-pairs shapes the dedicated cdist kernel does not cover -------------
// (int32 input, dim 1 or 4, A-curves longer than 512 points): the block is
// evaluated as chunked batches of (a, b) pairs by the batch kernels.  Pair lists
// are generated on the device; scratch comes from the stream-ordered pool.
__global__ void cdist_pairs_kernel(int64_t first, int64_t n, int64_t row_begin, int64_t nB,
                                   int32_t lenA, int32_t lenB, int64_t* offsets,
                                   int32_t* lengths) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = first + k;
    const int64_t a = row_begin + idx / nB, b = idx % nB;
    offsets[k] = a * lenA;
    offsets[n + k] = b * lenB;
    lengths[k] = lenA;
    lengths[n + k] = lenB;
  }
}

// results of pairs [first, first + n) of the row-major (rows × nB) block to every
// destination of `d` (and, with d.mirror, to the transposed places)
template <typename O>
__global__ void cdist_scatter_kernel(int64_t first, int64_t n, int64_t row_begin, int64_t nB, const O* src,
                                     OutSpec d) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = first + k;
    const int64_t a = row_begin + idx / nB, b = d.col_off + idx % nB;
    for (int i = 0; i < d.n; i++) {
      reinterpret_cast<O*>(d.out[i])[(a - d.row_base) * d.ld + b] = src[k];
      if (d.mirror) reinterpret_cast<O*>(d.out[i])[(b - d.row_base) * d.ld + a] = src[k];
    }
  }
  if (d.n > 1) __threadfence_system();
}

static int cdist_via_batch(const CdistArgs& a, cudaStream_t st) {
  const int64_t rows = a.row_end - a.row_begin;
  const int64_t total = rows * a.nB;
  const int64_t CH = total < (int64_t)(1 << 20) ? total : (int64_t)(1 << 20);
  const size_t osz = a.dtype == FFD_I32 ? 8 : 4;
  const size_t wsb = batch_layout(nullptr, CH, dev_info().sms).bytes;
  const size_t off_b = (size_t)CH * 2 * sizeof(int64_t), len_b = (size_t)CH * 2 * sizeof(int32_t);
  char* buf = nullptr;
  const size_t total_b = off_b + len_b + (size_t)CH * osz + wsb + 1024;
  if (cudaMallocAsync(reinterpret_cast<void**>(&buf), total_b, st) != cudaSuccess) return FFD_ERR_CUDA;
  int64_t* offsets = reinterpret_cast<int64_t*>(buf);
  int32_t* lengths = reinterpret_cast<int32_t*>(buf + off_b);
  char* tmp = buf + ((off_b + len_b + 255) / 256) * 256;
  char* ws = tmp + (((size_t)CH * osz + 255) / 256) * 256;
  int rc = FFD_OK;
  for (int64_t first = 0; first < total && rc == FFD_OK; first += CH) {
    const int64_t n = (total - first < CH) ? total - first : CH;
    const int blocks = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    cdist_pairs_kernel<<<blocks, 256, 0, st>>>(first, n, a.row_begin, a.nB, a.lenA, a.lenB, offsets,
                                               lengths);
    ++g_launches;
    rc = batch_impl(a.A, a.B, offsets, lengths, n, a.dim, a.norm, a.dtype, tmp, ws, wsb, st, 0,
                    pair_goes_long(a.lenA, a.lenB, medium_rows_for(n, dev_info().sms)));
    if (rc != FFD_OK) break;
    if (osz == 8)
      cdist_scatter_kernel<long long><<<blocks, 256, 0, st>>>(
          first, n, a.row_begin, a.nB, reinterpret_cast<const long long*>(tmp), a.dst);
    else
      cdist_scatter_kernel<float><<<blocks, 256, 0, st>>>(first, n, a.row_begin, a.nB,
                                                          reinterpret_cast<const float*>(tmp), a.dst);
    ++g_launches;
    if (cudaGetLastError() != cudaSuccess) rc = FFD_ERR_CUDA;
  }
  cudaFreeAsync(buf, st);
  return rc;
}

static int cdist_dispatch(const CdistArgs& a, cudaStream_t st) {
  const int rc = launch_cdist(a, dev_info().sms, st, &g_launches);
  if (rc != FFD_ERR_UNSUPPORTED) return rc;
  return cdist_via_batch(a, st);  // shapes outside the dedicated kernel
}

}  // namespace ffd

using namespace ffd;

extern "C" {

int ffd_version(void) { return 100; }

const char* ffd_status_string(int s) {
  switch (s) {
    case FFD_OK: return "ok";
    case FFD_ERR_ARG: return "invalid argument";
    case FFD_ERR_UNSUPPORTED: return "unsupported";
    case FFD_ERR_CUDA: return "CUDA error";
    case FFD_ERR_EMPTY: return "curve with length < 1";
    case FFD_ERR_NONFINITE: return "non-finite coordinate";
    case FFD_ERR_OVERFLOW: return "integer distance overflows int64";
    case FFD_ERR_RANGE: return "offsets/lengths out of range";
    case FFD_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int ffd_profile_enable(int on) {
  g_prof_on.store(on ? 1 : 0);
  return FFD_OK;
}

int ffd_profile_take(double* total_ms, int64_t* launches) {
  std::vector<ProfRec> ev;
  {
    std::lock_guard<std::mutex> g(g_prof_mu);
    ev.swap(g_prof_events);
  }
  double sum[4] = {0, 0, 0, 0};
  int64_t cnt[4] = {0, 0, 0, 0};
  int rc = FFD_OK;
  for (auto& e : ev) {
    float ms = 0.f;
    if (cudaEventSynchronize(e.b) != cudaSuccess || cudaEventElapsedTime(&ms, e.a, e.b) != cudaSuccess)
      rc = FFD_ERR_CUDA;
    sum[e.tag] += ms;
    cnt[e.tag] += 1;
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  int top = 0;
  for (int i = 1; i < 4; i++)
    if (sum[i] > sum[top]) top = i;
  if (total_ms) *total_ms = sum[top];
  if (launches) *launches = cnt[top];
  return rc;
}

int64_t ffd_take_launch_count(void) {
  int64_t n = g_launches;
  g_launches = 0;
  return n;
}

size_t ffd_batch_workspace_bytes(int64_t num_pairs) {
  if (num_pairs < 0) return 0;
  return batch_layout(nullptr, num_pairs, dev_info().sms).bytes;
}

int ffd_batch(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
              int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, void* out,
              void* workspace, size_t workspace_bytes, ffd_stream_t stream) {
  return batch_impl(p, q, offsets, lengths, num_pairs, dim, norm, dtype, out, workspace,
                    workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int ffd_batch_maxlen(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                     int64_t num_pairs, int64_t max_n, int64_t max_m, int32_t dim, int32_t norm,
                     int32_t dtype, void* out, void* workspace, size_t workspace_bytes,
                     ffd_stream_t stream) {
  if (max_n < 0 || max_m < 0) return FFD_ERR_ARG;
  // pair_goes_long is monotone in (n, m): a pair within the bounds goes long
  // only if a pair of the bounds' sizes would
  const int64_t cap = int64_t(1) << 30;  // above every threshold, no overflow in the band count
  const bool long_possible =
      pair_goes_long((int)(max_n < cap ? max_n : cap), (int)(max_m < cap ? max_m : cap),
                     medium_rows_for(num_pairs, dev_info().sms));
  return batch_impl(p, q, offsets, lengths, num_pairs, dim, norm, dtype, out, workspace,
                    workspace_bytes, reinterpret_cast<cudaStream_t>(stream), 0, long_possible);
}

int ffd_batch_dtw(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                  int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, void* out,
                  void* workspace, size_t workspace_bytes, ffd_stream_t stream) {
  return batch_impl(p, q, offsets, lengths, num_pairs, dim, norm, dtype, out, workspace,
                    workspace_bytes, reinterpret_cast<cudaStream_t>(stream), 1);
}

int ffd_batch_dtw_f64(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                      int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, double* out,
                      void* workspace, size_t workspace_bytes, ffd_stream_t stream) {
  return batch_impl(p, q, offsets, lengths, num_pairs, dim, norm, dtype, out, workspace,
                    workspace_bytes, reinterpret_cast<cudaStream_t>(stream), 2);
}

int ffd_dist_sum(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                 int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, double* out,
                 ffd_stream_t stream) {
  int s = check_common(dim, norm, dtype);
  if (s) return s;
  if (dtype != FFD_F32) return FFD_ERR_UNSUPPORTED;
  if (num_pairs < 0) return FFD_ERR_ARG;
  if (num_pairs == 0) return FFD_OK;
  if (!p || !q || !offsets || !lengths || !out) return FFD_ERR_ARG;
  return launch_dist_sum(static_cast<const float*>(p), static_cast<const float*>(q), offsets,
                         lengths, num_pairs, dim, norm, out, dev_info().sms,
                         reinterpret_cast<cudaStream_t>(stream), &g_launches);
}

// a second stream per device for the host path's uploads (created once)
static cudaStream_t copy_stream() {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!streams[dev]) cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
  return streams[dev];
}

int ffd_batch_host(const void* p_host, int64_t np, const void* q_host, int64_t nq,
                   const int64_t* offsets_host, const int32_t* lengths_host, int64_t num_pairs,
                   int32_t dim, int32_t norm, int32_t dtype, void* out_host, ffd_stream_t stream) {
  int s = check_common(dim, norm, dtype);
  if (s) return s;
  if (num_pairs < 0 || np < 0 || nq < 0) return FFD_ERR_ARG;
  if (num_pairs == 0) return FFD_OK;
  if (!p_host || !q_host || !offsets_host || !lengths_host || !out_host) return FFD_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  static std::once_flag pool_once;
  std::call_once(pool_once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  const int64_t B = num_pairs;
  const size_t esz = 4, ptb = (size_t)dim * esz;  // bytes per point
  const size_t pb = (size_t)np * ptb, qb = (size_t)nq * ptb;
  const size_t osz = dtype == FFD_I32 ? 8 : 4;
  const size_t ob = (size_t)B * osz;
  const size_t offb = (size_t)B * 2 * sizeof(int64_t);
  const size_t lenb = (size_t)B * 2 * sizeof(int32_t);
  const size_t wsb = ffd_batch_workspace_bytes(B);
  const int sms = dev_info().sms;
  const int medium_rows = medium_rows_for(B, sms);
  // Pipelined upload: the pairs are cut into K chunks; chunk j starts as soon as
  // the point prefixes its pairs reach are on the device, while the copy stream
  // moves the next points (the points dominate the call: 514 MB for config 2).
  const int K = (pb + qb >= (64u << 20) && B >= 64)
                    ? (int)std::min<int64_t>(8, std::max<int64_t>(2, (int64_t)((pb + qb) >> 26)))
                    : 1;
  void *dp = nullptr, *dq = nullptr, *doff = nullptr, *dlen = nullptr, *dout = nullptr, *dws = nullptr;
  void *coff = nullptr, *clen = nullptr;
  int rc = FFD_OK;
  if (cudaMallocAsync(&dp, pb ? pb : 16, st) || cudaMallocAsync(&dq, qb ? qb : 16, st) ||
      cudaMallocAsync(&doff, offb, st) || cudaMallocAsync(&dlen, lenb, st) ||
      cudaMallocAsync(&dout, ob, st) || cudaMallocAsync(&dws, wsb, st) ||
      (K > 1 && (cudaMallocAsync(&coff, offb, st) || cudaMallocAsync(&clen, lenb, st)))) {
    rc = FFD_ERR_CUDA;
  }
  if (rc == FFD_OK && K == 1) {
    if (cudaMemcpyAsync(dp, p_host, pb, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(dq, q_host, qb, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(doff, offsets_host, offb, cudaMemcpyHostToDevice, st) ||
        cudaMemcpyAsync(dlen, lengths_host, lenb, cudaMemcpyHostToDevice, st))
      rc = FFD_ERR_CUDA;
    bool any_long = false;  // the lengths are on the host: skip the long-pair launch if none is
    for (int64_t k = 0; k < B && !any_long; k++)
      any_long = lengths_host[k] >= 1 && lengths_host[B + k] >= 1 &&
                 pair_goes_long(lengths_host[k], lengths_host[B + k], medium_rows);
    if (rc == FFD_OK)
      rc = batch_impl(dp, dq, reinterpret_cast<int64_t*>(doff), reinterpret_cast<int32_t*>(dlen), B, dim,
                      norm, dtype, dout, dws, wsb, st, 0, any_long);
  } else if (rc == FFD_OK) {
    cudaStream_t cs = copy_stream();
    std::vector<cudaEvent_t> ev(K + 1, nullptr);
    for (auto& e : ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) rc = FFD_ERR_CUDA;
    // the allocations above are stream-ordered on `st`: the copy stream waits for them
    if (rc == FFD_OK && (cudaEventRecord(ev[K], st) || cudaStreamWaitEvent(cs, ev[K], 0) ||
                         cudaMemcpyAsync(doff, offsets_host, offb, cudaMemcpyHostToDevice, cs) ||
                         cudaMemcpyAsync(dlen, lengths_host, lenb, cudaMemcpyHostToDevice, cs)))
      rc = FFD_ERR_CUDA;
    int64_t have_p = 0, have_q = 0, need_p = 0, need_q = 0;
    for (int j = 0; j < K && rc == FFD_OK; j++) {
      const int64_t k0 = B * j / K, k1 = B * (j + 1) / K, bc = k1 - k0;
      const int medium_rows_c = medium_rows_for(bc, sms);
      bool any_long = false;
      for (int64_t k = k0; k < k1; k++) {
        const int32_t n = lengths_host[k], m = lengths_host[B + k];
        if (n < 1 || m < 1) continue;
        need_p = std::max<int64_t>(need_p, offsets_host[k] + n);
        need_q = std::max<int64_t>(need_q, offsets_host[B + k] + m);
        any_long = any_long || pair_goes_long(n, m, medium_rows_c);
      }
      need_p = std::min<int64_t>(need_p, np);
      need_q = std::min<int64_t>(need_q, nq);
      if (j == K - 1) need_p = np, need_q = nq;  // whatever is left
      if (need_p > have_p &&
          cudaMemcpyAsync(static_cast<char*>(dp) + have_p * ptb, static_cast<const char*>(p_host) + have_p * ptb,
                          (size_t)(need_p - have_p) * ptb, cudaMemcpyHostToDevice, cs))
        rc = FFD_ERR_CUDA;
      if (need_q > have_q &&
          cudaMemcpyAsync(static_cast<char*>(dq) + have_q * ptb, static_cast<const char*>(q_host) + have_q * ptb,
                          (size_t)(need_q - have_q) * ptb, cudaMemcpyHostToDevice, cs))
        rc = FFD_ERR_CUDA;
      have_p = std::max(have_p, need_p);
      have_q = std::max(have_q, need_q);
      if (rc != FFD_OK || cudaEventRecord(ev[j], cs) || cudaStreamWaitEvent(st, ev[j], 0)) {
        rc = FFD_ERR_CUDA;
        break;
      }
      // this chunk's [2·bc] offsets / lengths: two slices of the full arrays
      int64_t* co = static_cast<int64_t*>(coff) + 2 * k0;
      int32_t* cl = static_cast<int32_t*>(clen) + 2 * k0;
      const int64_t* fo = static_cast<const int64_t*>(doff);
      const int32_t* fl = static_cast<const int32_t*>(dlen);
      if (cudaMemcpyAsync(co, fo + k0, bc * sizeof(int64_t), cudaMemcpyDeviceToDevice, st) ||
          cudaMemcpyAsync(co + bc, fo + B + k0, bc * sizeof(int64_t), cudaMemcpyDeviceToDevice, st) ||
          cudaMemcpyAsync(cl, fl + k0, bc * sizeof(int32_t), cudaMemcpyDeviceToDevice, st) ||
          cudaMemcpyAsync(cl + bc, fl + B + k0, bc * sizeof(int32_t), cudaMemcpyDeviceToDevice, st)) {
        rc = FFD_ERR_CUDA;
        break;
      }
      rc = batch_impl(dp, dq, co, cl, bc, dim, norm, dtype, static_cast<char*>(dout) + k0 * osz, dws, wsb,
                      st, 0, any_long);
    }
    if (cudaStreamSynchronize(cs) != cudaSuccess && rc == FFD_OK) rc = FFD_ERR_CUDA;
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  if (rc == FFD_OK && cudaMemcpyAsync(out_host, dout, ob, cudaMemcpyDeviceToHost, st))
    rc = FFD_ERR_CUDA;
  for (void* ptr : {dp, dq, doff, dlen, dout, dws, coff, clen})
    if (ptr) cudaFreeAsync(ptr, st);
  if (cudaStreamSynchronize(st) != cudaSuccess && rc == FFD_OK) rc = FFD_ERR_CUDA;
  return rc;
}

size_t ffd_cdist_workspace_bytes(void) { return cdist_workspace_bytes(); }

static int cdist_common(const void* setA, int64_t nA, int32_t lenA, const void* setB, int64_t nB,
                        int32_t lenB, int32_t dim, int32_t norm, int32_t dtype, int64_t row_begin,
                        int64_t row_end, int self, const OutSpec& dst, void* workspace,
                        size_t workspace_bytes, ffd_stream_t stream) {
  int s = check_common(dim, norm, dtype);
  if (s) return s;
  if (nA < 0 || nB < 0 || row_begin < 0 || row_end < row_begin || row_end > nA) return FFD_ERR_ARG;
  if (dst.n < 1 || dst.n > kMaxOuts || dst.col_off < 0 || dst.row_base < 0) return FFD_ERR_ARG;
  if (row_end == row_begin || nB == 0) return FFD_OK;
  if (!setA || !setB || lenA < 1 || lenB < 1) return FFD_ERR_ARG;
  for (int i = 0; i < dst.n; i++)
    if (!dst.out[i]) return FFD_ERR_ARG;
  if (workspace_bytes < cdist_workspace_bytes() || (!workspace && cdist_workspace_bytes() > 0))
    return FFD_ERR_WORKSPACE;
  CdistArgs a{};
  a.A = setA;
  a.B = setB;
  a.nA = nA;
  a.nB = nB;
  a.lenA = lenA;
  a.lenB = lenB;
  a.dim = dim;
  a.norm = norm;
  a.dtype = dtype;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.dst = dst;
  a.workspace = workspace;
  a.self = self;
  ProfScope prof(reinterpret_cast<cudaStream_t>(stream), 3);
  return cdist_dispatch(a, reinterpret_cast<cudaStream_t>(stream));
}

int ffd_cdist(const void* setA, int64_t nA, int32_t lenA, const void* setB, int64_t nB,
              int32_t lenB, int32_t dim, int32_t norm, int32_t dtype, int64_t row_begin,
              int64_t row_end, void* out, int64_t ld_out, void* workspace, size_t workspace_bytes,
              ffd_stream_t stream) {
  if (ld_out < nB) return FFD_ERR_ARG;
  if (!out && row_end > row_begin && nB > 0) return FFD_ERR_ARG;
  OutSpec d{};
  d.out[0] = out;
  d.n = 1;
  d.row_base = row_begin;
  d.ld = ld_out;
  return cdist_common(setA, nA, lenA, setB, nB, lenB, dim, norm, dtype, row_begin, row_end, 0, d,
                      workspace, workspace_bytes, stream);
}

int ffd_cdist_self(const void* setA, int64_t nA, int32_t lenA, int32_t dim, int32_t norm,
                   int32_t dtype, int64_t row_begin, int64_t row_end, void* out, int64_t ld_out,
                   void* workspace, size_t workspace_bytes, ffd_stream_t stream) {
  if (ld_out < nA) return FFD_ERR_ARG;
  if (!out && row_end > row_begin) return FFD_ERR_ARG;
  OutSpec d{};
  d.out[0] = out;
  d.n = 1;
  d.row_base = row_begin;
  d.ld = ld_out;
  return cdist_common(setA, nA, lenA, setA, nA, lenA, dim, norm, dtype, row_begin, row_end, 1, d,
                      workspace, workspace_bytes, stream);
}

int ffd_cdist_to(const void* setA, int64_t nA, int32_t lenA, const void* setB, int64_t nB,
                 int32_t lenB, int32_t dim, int32_t norm, int32_t dtype, int64_t row_begin,
                 int64_t row_end, int32_t self, int64_t col_offset, int32_t mirror,
                 void* const* outs_host, int32_t n_outs, int64_t ld_out, void* workspace,
                 size_t workspace_bytes, ffd_stream_t stream) {
  if (!outs_host || n_outs < 1 || n_outs > kMaxOuts) return FFD_ERR_ARG;
  if (self && mirror) return FFD_ERR_ARG;
  if (self && lenB != lenA) return FFD_ERR_ARG;  // self: B is A's rows [col_offset, col_offset + nB)
  if (ld_out < col_offset + nB || (mirror && ld_out < nA) || (self && ld_out < nA)) return FFD_ERR_ARG;
  OutSpec d{};
  for (int i = 0; i < n_outs; i++) d.out[i] = outs_host[i];
  d.n = n_outs;
  d.row_base = 0;
  d.col_off = col_offset;
  d.ld = ld_out;
  d.mirror = mirror ? 1 : 0;
  return cdist_common(setA, nA, lenA, setB, nB, lenB, dim, norm, dtype, row_begin, row_end, self ? 1 : 0, d,
                      workspace, workspace_bytes, stream);
}

size_t ffd_long_pair_ring_bytes(int32_t n, int32_t m) {
  if (n < 1 || m < 1) return 0;
  return long_shard_ring_slots(n > m ? n : m) * 8;
}

int32_t ffd_long_pair_row_align(void) { return kWarp * kMaxR; }

int ffd_long_pair_shard(const void* p, int32_t n, const void* q, int32_t m, int32_t dim, int32_t norm,
                        int32_t dtype, int32_t row_begin, int32_t row_end, void* in_ring, size_t in_ring_bytes,
                        uint32_t in_tag_base, void* out_ring, size_t out_ring_bytes, uint32_t out_tag_base,
                        void* out, ffd_stream_t stream) {
  int s = check_common(dim, norm, dtype);
  if (s) return s;
  if (dtype != FFD_F32) return FFD_ERR_UNSUPPORTED;
  if (!p || !q || !out || n < 1 || m < 1) return FFD_ERR_ARG;
  const int rows = n < m ? n : m;  // the shorter curve is the rows curve (p on a tie)
  const int align = ffd_long_pair_row_align();
  if (row_begin < 0 || row_end <= row_begin || row_end > rows) return FFD_ERR_ARG;
  if (row_begin % align || (row_end != rows && row_end % align)) return FFD_ERR_ARG;
  const size_t need = ffd_long_pair_ring_bytes(n, m);
  if (row_begin > 0 && (!in_ring || in_ring_bytes < need)) return FFD_ERR_ARG;
  if (row_end < rows && (!out_ring || out_ring_bytes < need)) return FFD_ERR_ARG;
  LongArgs la{};
  la.p = p;
  la.q = q;
  la.dim = dim;
  la.norm = norm;
  la.dtype = dtype;
  la.out = out;
  la.row_begin = row_begin;
  la.row_end = row_end;
  la.ext_in = row_begin > 0 ? in_ring : nullptr;
  la.ext_in_slots = row_begin > 0 ? need / 8 : 0;
  la.ext_in_tb = in_tag_base;
  la.ext_out = row_end < rows ? out_ring : nullptr;
  la.ext_out_slots = row_end < rows ? need / 8 : 0;
  la.ext_out_tb = out_tag_base;
  ProfScope prof(reinterpret_cast<cudaStream_t>(stream), 2);
  return launch_long_shard(la, n, m, dev_info().sms, reinterpret_cast<cudaStream_t>(stream), &g_launches) ==
                 cudaSuccess
             ? FFD_OK
             : FFD_ERR_CUDA;
}

int ffd_validate_batch(const void* p, int64_t np, const void* q, int64_t nq,
                       const int64_t* offsets, const int32_t* lengths, int64_t num_pairs,
                       int32_t dim, int32_t dtype, ffd_stream_t stream) {
  if (dim < 1 || dim > 4 || (dtype != FFD_F32 && dtype != FFD_I32) || num_pairs < 0 || np < 0 ||
      nq < 0)
    return FFD_ERR_ARG;
  if (num_pairs == 0) return FFD_OK;
  if (!offsets || !lengths || (np > 0 && !p) || (nq > 0 && !q)) return FFD_ERR_ARG;
  return validate_batch(p, np, q, nq, offsets, lengths, num_pairs, dim, dtype,
                        reinterpret_cast<cudaStream_t>(stream), &g_launches);
}

}  // extern "C"
