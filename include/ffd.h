/* ffd.h — C ABI of the B200-native discrete Fréchet distance library (libffd.so).
 *
 * Method: arxiv 2404.05708 ("Walking Your Frog Fast in 4 LoC"), PAPER.md.
 *   δ_dF(p, q) for curves p ∈ R^{P×D}, q ∈ R^{Q×D} is M_PQ of
 *   the recurrence Eq. (1), M_ij = max{min{M_{i-1,j}, M_{i-1,j-1}, M_{i,j-1}}, d_ij}
 *   (L159–L163), evaluated iteratively, branch-free and in linear memory
 *   (Alg. 2 / Alg. 5) with d_ij = ‖p_i − q_j‖ evaluated
 *   lazily (Theorem 1).  Batching over independent pairs follows PAPER
 *   L259–L262 (padding by repeated points, sorting by length).
 *
 * General conventions (every entry point):
 *   - Pointers named *_host are host memory; every other pointer is DEVICE memory
 *     owned by the caller.  Nothing is retained after the call returns.
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) unless stated otherwise, reentrant and thread-safe.
 *   - Host-checkable argument errors return a status synchronously and launch
 *     nothing.  CUDA launch failures return FFD_ERR_CUDA.  Device-data
 *     preconditions (lengths ≥ 1, offsets in range, finite coordinates) are NOT
 *     checked by the asynchronous calls; ffd_validate_batch checks them.  A pair
 *     with a length < 1 gets NaN (fp32) / INT64_MIN (int) and reads nothing.
 *   - Integer inputs give exact results: every int32-coordinate result equals the
 *     exact int64 value whenever D·(max |coordinate difference|)² ≤ 2^63 − 1.
 *   - fp32 inputs: per-cell distances in fp32 with the operation order given in
 *     DESIGN.md §"fp32 arithmetic"; L2 takes one square root at the end (exact:
 *     sqrt is monotone).  Relative error ≤ 1e-5 of the exact value.
 */
#ifndef FFD_H
#define FFD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ffd_stream_t; /* == cudaStream_t */

typedef enum {
  FFD_OK = 0,
  FFD_ERR_ARG = -1,         /* bad argument (null pointer, bad dim/norm/dtype, sizes) */
  FFD_ERR_UNSUPPORTED = -2, /* valid request the library does not implement */
  FFD_ERR_CUDA = -3,        /* a CUDA call failed */
  FFD_ERR_EMPTY = -4,       /* validate: a curve has length < 1 */
  FFD_ERR_NONFINITE = -5,   /* validate: NaN / ±Inf coordinate */
  FFD_ERR_OVERFLOW = -6,    /* validate: int32 input with D·range² > 2^63 − 1 */
  FFD_ERR_RANGE = -7,       /* validate: offsets + lengths outside the point arrays */
  FFD_ERR_WORKSPACE = -8    /* workspace smaller than the *_workspace_bytes() value */
} ffd_status;

typedef enum {
  FFD_L1 = 1,   /* Σ|Δ_k|                                   */
  FFD_L2 = 2,   /* sqrt(Σ Δ_k²) — Euclidean      */
  FFD_LINF = 3, /* max |Δ_k|                                  */
  FFD_SQL2 = 4  /* Σ Δ_k²  (squared Euclidean; same coupling as L2) */
} ffd_norm;

typedef enum {
  FFD_F32 = 0, /* coordinates float32; out float32                          */
  FFD_I32 = 1  /* coordinates int32; out int64 (norms SQL2, L1, LINF only)   */
} ffd_dtype;

/* ---------------------------------------------------------------------------
 * ffd_batch — discrete Fréchet distance of B independent curve pairs.
 *   out[k] = δ_dF(p[offsets[k] .. offsets[k]+lengths[k]),
 *                 q[offsets[B+k] .. offsets[B+k]+lengths[B+k]])   under `norm`.
 *   p: [Σn, dim] points, q: [Σm, dim] points, array-of-structures, row-major,
 *      element type per `dtype`, naturally aligned.
 *   offsets: int64[2B] (in points; first the B p-offsets, then the B q-offsets).
 *   lengths: int32[2B] (same order), each ≥ 1 by precondition.
 *   dim ∈ {1,2,3,4}.  out: float[B] (FFD_F32) or int64[B] (FFD_I32).
 *   workspace: device scratch of at least ffd_batch_workspace_bytes(B) bytes,
 *   16-byte aligned, owned by the caller, not read before being written.
 *   Pairs are processed in an order sorted by length; the
 *   result does not depend on that order.  Any lengths n, m ≥ 1: a pair too
 *   long for one warp band is pipelined over groups of CTAs, in as many passes
 *   as it takes when its bands exceed what the GPU holds at once (linear
 *   memory, Theorem 1).  Returns FFD_OK once the work is queued; a
 *   long pair whose pipeline stalls for seconds (a hardware fault, never seen)
 *   gets NaN / INT64_MIN rather than a plausible value.
 * ------------------------------------------------------------------------- */
int ffd_batch(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
              int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, void* out,
              void* workspace, size_t workspace_bytes, ffd_stream_t stream);
size_t ffd_batch_workspace_bytes(int64_t num_pairs);

/* ffd_batch_maxlen — ffd_batch with caller-known length bounds: every
 *   lengths[k] ≤ max_n and lengths[B+k] ≤ max_m (k < B; the max_seqlen idea of
 *   variable-length attention kernels).  Same operation, arguments, layout,
 *   workspace and stream semantics as ffd_batch.  When no pair within the bounds
 *   needs the long-pair kernel (pair_goes_long is monotone in the lengths), its
 *   cooperative clustered launch is skipped: config 1 runs 2 launches instead
 *   of 3, with results identical to ffd_batch's.  A pair that breaks its bound
 *   and would need the long-pair kernel gets NaN / INT64_MIN (never a silent
 *   wrong value); with the point counts of p and q as bounds nothing is ever
 *   excluded.  max_n or max_m < 0 → FFD_ERR_ARG.                                */
int ffd_batch_maxlen(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                     int64_t num_pairs, int64_t max_n, int64_t max_m, int32_t dim, int32_t norm,
                     int32_t dtype, void* out, void* workspace, size_t workspace_bytes,
                     ffd_stream_t stream);

/* ffd_batch_dtw — dynamic time warping of B pairs (PAPER Appendix B:
 *   Alg. 2 with max replaced by +, i.e. C[i][j] = min{C[i−1][j], C[i−1][j−1],
 *   C[i][j−1]} + d_ij, result C[P][Q]).  Same arguments, layout, workspace and
 *   stream semantics as ffd_batch.  dtype must be FFD_F32 (FFD_ERR_UNSUPPORTED
 *   otherwise); FFD_L2 evaluates sqrt per cell; sums are accumulated in fp32 in
 *   the DP's own order (relative error ≤ (n+m+D+2)·2⁻²⁴ of the exact value).
 *   Any lengths: pairs too long for the batch kernel's bands (more than 16
 *   bands of 512 rows, or more than one band with the longer curve above 8254
 *   points) run on the long-pair kernel with the DTW cell (the shorter curve
 *   on the rows).                                                               */
int ffd_batch_dtw(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                  int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, void* out,
                  void* workspace, size_t workspace_bytes, ffd_stream_t stream);

/* ffd_batch_dtw_f64 — DTW of B pairs with the sums (and every distance) in
 *   fp64: the accumulation option of Appendix B's DTW.  Each
 *   d_ij is evaluated in fp64 from the fp32 coordinates (Δ in fp64, squares
 *   summed left to right, L2 one square root per cell) and every DP sum is one
 *   fp64 rounding, so out[k] equals the fp64 oracle bit for bit.  dtype must be
 *   FFD_F32; out: double[B]; same layout, workspace and stream semantics as
 *   ffd_batch.  Limits: pairs too long for the batch kernel's bands (see
 *   ffd_batch_dtw) get NaN — the long-pair kernel has no fp64 tier.           */
int ffd_batch_dtw_f64(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                      int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, double* out,
                      void* workspace, size_t workspace_bytes, ffd_stream_t stream);

/* ffd_dist_sum — Σ_i Σ_j d(p_i, q_j) of each of B pairs: the paper's "upper
 *   limit" baseline, the distances of the DP workload
 *   (FFD_L2 takes a square root per cell, the paper's hypot L271) without the
 *   recurrence.  A calibration kernel: how close the DP comes to the cost of
 *   its distances alone.  Layout, offsets (one-vs-many allowed) and stream
 *   semantics as ffd_batch; dtype must be FFD_F32 (FFD_ERR_UNSUPPORTED
 *   otherwise); out: double[B], deterministic (fixed summation order), relative
 *   error ≤ (35 + 2·dim)·2⁻²⁴ of the exact sum; NaN for a pair with a length
 *   < 1.  Needs no workspace (scratch from the stream-ordered pool).          */
int ffd_dist_sum(const void* p, const void* q, const int64_t* offsets, const int32_t* lengths,
                 int64_t num_pairs, int32_t dim, int32_t norm, int32_t dtype, double* out,
                 ffd_stream_t stream);

/* ffd_batch_host — the same computation from HOST buffers (end-to-end path).
 *   p_host: [np, dim], q_host: [nq, dim]; offsets_host/lengths_host as above;
 *   out_host: float[B] / int64[B].  Host buffers should be pinned for overlap.
 *   Copies in, computes and copies out on `stream` using device memory from a
 *   stream-ordered pool; synchronises `stream` before returning.  With ≥ 64 MB
 *   of points the pairs run in up to 8 chunks, each starting as soon as the
 *   point prefixes its pairs reach have been uploaded by an internal per-device
 *   copy stream (offsets need not be sorted; unsorted ones just wait longer).
 *   The host lengths also decide whether the long-pair kernel is launched.     */
int ffd_batch_host(const void* p_host, int64_t np, const void* q_host, int64_t nq,
                   const int64_t* offsets_host, const int32_t* lengths_host, int64_t num_pairs,
                   int32_t dim, int32_t norm, int32_t dtype, void* out_host, ffd_stream_t stream);

/* ---------------------------------------------------------------------------
 * ffd_cdist — all-pairs distances between two dense curve sets (one shard).
 *   The paper evaluates δ_dF of a batch of curves against one curve (PAPER
 *   L259); this is the same pair function (Eq. (1), with lazily
 *   evaluated d, Theorem 1) over every (A_a, B_b) of two sets — the
 *   independent pairs the paper parallelises over (L259) — written as a matrix
 *   block so that W ranks can each compute a block of rows (BASELINE.json
 *   north_star (3)).
 *   out[(a - row_begin)*ld_out + b] = δ_dF(A_a, B_b)  for a ∈ [row_begin, row_end),
 *   b ∈ [0, nB).  setA: [nA, lenA, dim], setB: [nB, lenB, dim] dense row-major.
 *   out: float (FFD_F32) or int64 (FFD_I32), ld_out ≥ nB elements.
 *   [row_begin, row_end) is the caller's shard (one rank's block of rows).
 *   workspace: ≥ ffd_cdist_workspace_bytes() bytes (may be NULL if that is 0).
 *   fp32 input with dim 2–3 and lenA ≤ 512 runs the dedicated all-pairs kernel;
 *   every other dtype/dim/length is evaluated as chunked batches of (a, b)
 *   pairs by ffd_batch's kernels (scratch from the stream-ordered pool).
 * ------------------------------------------------------------------------- */
int ffd_cdist(const void* setA, int64_t nA, int32_t lenA, const void* setB, int64_t nB,
              int32_t lenB, int32_t dim, int32_t norm, int32_t dtype, int64_t row_begin,
              int64_t row_end, void* out, int64_t ld_out, void* workspace,
              size_t workspace_bytes, ffd_stream_t stream);
size_t ffd_cdist_workspace_bytes(void);

/* ffd_cdist_self — the same for a set against ITSELF (B = A, nB = nA):
 *   out[(a − row_begin)*ld_out + b] = δ_dF(A_a, A_b), a ∈ [row_begin, row_end),
 *   b ∈ [0, nA).  δ is symmetric (a metric; bit-exactly so in fp32,
 *   DESIGN.md reading 15), so each unordered pair with both curves inside the
 *   shard is evaluated once and written to both places: the full range costs
 *   about half of ffd_cdist(A, A).  Same dtype/norm/workspace/stream rules.     */
int ffd_cdist_self(const void* setA, int64_t nA, int32_t lenA, int32_t dim, int32_t norm,
                   int32_t dtype, int64_t row_begin, int64_t row_end, void* out, int64_t ld_out,
                   void* workspace, size_t workspace_bytes, ffd_stream_t stream);

/* ffd_cdist_to — the all-pairs block written straight into one or more FULL
 *   matrices: this GPU's and, through NVLink, its peers' (north_star (3): the
 *   fused distribution that replaces the trailing all-gather).
 *   Rows a ∈ [row_begin, row_end) of setA against the nB curves of setB, whose
 *   curve b is column col_offset + b.  Every result goes to
 *     outs_host[i][a*ld_out + col_offset + b]   for i < n_outs (≤ 8),
 *   and, with mirror = 1, also to outs_host[i][(col_offset + b)*ld_out + a]
 *   (δ is symmetric: the lower triangle of a self matrix).
 *   self = 1: setB is setA's rows [col_offset, col_offset + nB) (lenB = lenA);
 *   each unordered pair with both curves inside [row_begin, row_end) is
 *   evaluated once and written to both places, as ffd_cdist_self.
 *   outs_host: a HOST array of n_outs DEVICE pointers — local memory or peer
 *   memory mapped into this context (CUDA IPC / symmetric memory) — each the
 *   base of a row-major matrix with ld_out elements per row, owned by the
 *   caller.  The kernel ends with a system-scope fence, so that a barrier
 *   sequenced after it on `stream` (e.g. an NCCL all-reduce or a symmetric-
 *   memory barrier) publishes the results to every peer.  Same dtype / norm /
 *   workspace / stream rules as ffd_cdist.                                     */
int ffd_cdist_to(const void* setA, int64_t nA, int32_t lenA, const void* setB, int64_t nB,
                 int32_t lenB, int32_t dim, int32_t norm, int32_t dtype, int64_t row_begin,
                 int64_t row_end, int32_t self, int64_t col_offset, int32_t mirror,
                 void* const* outs_host, int32_t n_outs, int64_t ld_out, void* workspace,
                 size_t workspace_bytes, ffd_stream_t stream);

/* ---------------------------------------------------------------------------
 * ffd_long_pair_shard — one very long pair over several GPUs.
 *   The rows curve (the shorter of p, q; p on a tie) is split into row ranges,
 *   one per GPU; each GPU runs this call on its range [row_begin, row_end) and
 *   the band chain of Eq. (1) (linear memory: Theorem 1)
 *   continues across GPUs: the first band of a range reads its top input from
 *   in_ring (in THIS GPU's memory, written by the GPU of the range above over
 *   NVLink) and the last band writes its bottom row into out_ring (the NEXT
 *   GPU's in_ring, a peer pointer mapped into this context: CUDA IPC or torch
 *   symmetric memory).  Rings hold a whole stream of ffd_long_pair_ring_bytes()
 *   bytes, so a GPU never waits for its consumer: the calls may run
 *   concurrently (pipelined over NVLink) or one after another (the same
 *   result).  The GPU whose range ends at the last row writes out[0] = δ_dF.
 *   p: [n, dim], q: [m, dim] fp32 (FFD_F32 only), device pointers, identical on
 *   every GPU.  row_begin is a multiple of ffd_long_pair_row_align() (512) and
 *   so is row_end unless it is the last row.  Tag bases: both ends of a link
 *   pass the same in/out tag base per call and advance it by at least the
 *   ring's slot count (bytes / 8) from one call to the next; a ring must be
 *   zeroed before its first use.  Returns FFD_ERR_ARG for bad ranges or rings.  */
size_t ffd_long_pair_ring_bytes(int32_t n, int32_t m);
int32_t ffd_long_pair_row_align(void);
int ffd_long_pair_shard(const void* p, int32_t n, const void* q, int32_t m, int32_t dim, int32_t norm,
                        int32_t dtype, int32_t row_begin, int32_t row_end, void* in_ring, size_t in_ring_bytes,
                        uint32_t in_tag_base, void* out_ring, size_t out_ring_bytes, uint32_t out_tag_base,
                        void* out, ffd_stream_t stream);

/* ---------------------------------------------------------------------------
 * ffd_validate_batch — SYNCHRONOUS device-data precondition check of a batch:
 *   lengths ≥ 1 (FFD_ERR_EMPTY), offsets+lengths within [0, np)/[0, nq)
 *   (FFD_ERR_RANGE), finite fp32 coordinates (FFD_ERR_NONFINITE), and for int32
 *   input D·(max |coordinate difference within a pair|)² ≤ 2^63−1
 *   (FFD_ERR_OVERFLOW).  Returns the first violated code in that order, FFD_OK
 *   otherwise.  Uses no caller workspace.
 * ------------------------------------------------------------------------- */
int ffd_validate_batch(const void* p, int64_t np, const void* q, int64_t nq,
                       const int64_t* offsets, const int32_t* lengths, int64_t num_pairs,
                       int32_t dim, int32_t dtype, ffd_stream_t stream);

/* ---------------------------------------------------------------------------
 * Profiling hook (benchmarks): while enabled, every ffd_batch / ffd_cdist call
 * records a CUDA event pair on its stream around each of its DP kernels (batch
 * main tier, exact int64 tier, long-pair wavefront, cdist).  ffd_profile_take()
 * waits for the recorded events and writes, for the DOMINANT kernel (the one
 * with the largest summed time), its summed milliseconds and its number of
 * timed launches; then it clears the record.  Host-side, thread-safe.
 * ------------------------------------------------------------------------- */
int ffd_profile_enable(int on);
int ffd_profile_take(double* total_ms, int64_t* launches);

/* human-readable name of a status code (static storage) */
const char* ffd_status_string(int status);

/* number of kernels the library launched on this thread since the last call
 * (for launch accounting in benchmarks); resets the counter. */
int64_t ffd_take_launch_count(void);

/* library version: major*10000 + minor*100 + patch */
int ffd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FFD_H */
