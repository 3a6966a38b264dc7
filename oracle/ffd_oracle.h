/* ffd_oracle.h — plain, slow, obviously-correct CPU oracle for the discrete
 * Fréchet distance (arxiv 2404.05708, "Walking Your Frog Fast in 4 LoC").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2404_05708_b200/, include/ffd.h) never links or calls it.
 * It shares no code, header, table or constant with the CUDA path.
 *
 * Notation follows the paper: curves p ∈ R^{P×D}, q ∈ R^{Q×D} (PAPER.md L67,
 * L124); point distance d_ij = f(p_i, q_j) (L132, L137); recurrence Eq. (1)
 * M_ij = max{min{M_{i-1,j}, M_{i-1,j-1}, M_{i,j-1}}, d_ij}, δ_dF = M_PQ
 * (L159–L163).  Indices here are 0-based; the (P+1)×(Q+1) padded table with
 * C[0][0]=0 and +inf on the rest of row 0 / column 0 is the branch-free
 * restatement of Alg. 3's four cases (L184–L192), see DESIGN.md "Readings".
 *
 * Arithmetic: fp32 coordinates are widened exactly to fp64 and every d_ij is
 * evaluated in fp64; int32 coordinates are evaluated exactly in int64 (with an
 * __int128 overflow check).  Functions with suffix _f32mirror instead evaluate
 * in fp32 with a documented operation order.
 *
 * Status codes: 0 ok, -1 bad argument, -4 empty curve, -5 non-finite
 * coordinate, -6 integer overflow of the exact int64 distance.
 */
#ifndef FFD_ORACLE_H
#define FFD_ORACLE_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_EMPTY (-4)
#define ORC_ERR_NONFINITE (-5)
#define ORC_ERR_OVERFLOW (-6)

/* norm ids (same numeric meaning as the product ABI, defined independently) */
#define ORC_L1 1
#define ORC_L2 2
#define ORC_LINF 3
#define ORC_SQL2 4

#ifdef __cplusplus
extern "C" {
#endif

/* ---- point distance f(p_i, q_j) (PAPER L67 ‖·‖_S, L271 Euclidean) ---------- */
double orc_point_dist_f32(const float* a, const float* b, int dim, int norm);
int orc_point_dist_i32(const int32_t* a, const int32_t* b, int dim, int norm, int64_t* out);

/* distance matrix d ∈ R^{P×Q}, row-major */
int orc_dist_matrix_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                        double* d);
int orc_dist_matrix_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                        int64_t* d);

/* ---- δ_dF from a given distance matrix d (P×Q, row-major) ------------------
 * _table   : Alg. 3 / Eq. (1) bottom-up over the padded (P+1)×(Q+1) table.
 * _linear  : Alg. 5, one row v ∈ R^Q.
 * _alg2    : Alg. 2 literally: fold of fréchet_next over rows, each a scan of
 *            fréchet_maxmin (Alg. 6/7 L333–L373).
 * _inplace : Alg. 4 on a copy of d.
 * _brute   : min over all monotone couplings of the max d along the coupling
 *            (definition), exponential: P,Q ≤ 10 only.       */
double orc_frechet_table_d(const double* d, int64_t P, int64_t Q);
double orc_frechet_linear_d(const double* d, int64_t P, int64_t Q);
double orc_frechet_alg2_d(const double* d, int64_t P, int64_t Q);
double orc_frechet_inplace_d(const double* d, int64_t P, int64_t Q);
double orc_frechet_brute_d(const double* d, int64_t P, int64_t Q);
int64_t orc_frechet_table_i(const int64_t* d, int64_t P, int64_t Q);
int64_t orc_frechet_linear_i(const int64_t* d, int64_t P, int64_t Q);
int64_t orc_frechet_brute_i(const int64_t* d, int64_t P, int64_t Q);
/* the full (P+1)×(Q+1) table itself (prefix semantics) */
void orc_frechet_full_table_d(const double* d, int64_t P, int64_t Q, double* C);

/* discrete Hausdorff distance of d (δ_dF ≥ Hausdorff) */
double orc_hausdorff_d(const double* d, int64_t P, int64_t Q);

/* ---- δ_dF of one curve pair with lazily evaluated d (Theorem 1) ------
 * table form with O(PQ) memory; linear form with O(Q) memory.              */
int orc_pair_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                 double* out);
int orc_pair_linear_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                        double* out);
int orc_pair_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                 int64_t* out);
int orc_pair_linear_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                        int64_t* out);
/* fp32 arithmetic with the documented operation order (DESIGN.md §fp32 mirror) */
int orc_pair_f32mirror(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                       float* out);

/* ---- batches: out[k] = δ(p[offsets[k]..+lengths[k]], q[offsets[B+k]..+lengths[B+k]])
 * offsets: int64[2B] in points, lengths: int32[2B]; OpenMP over pairs (timing only).
 * A pair with a precondition violation gets NaN / INT64_MIN and the first
 * violated status is returned.                                               */
int orc_batch_f32(const float* p, const float* q, const int64_t* offsets, const int32_t* lengths,
                  int64_t B, int dim, int norm, double* out, int threads);
int orc_batch_f32mirror(const float* p, const float* q, const int64_t* offsets,
                        const int32_t* lengths, int64_t B, int dim, int norm, float* out,
                        int threads);
int orc_batch_i32(const int32_t* p, const int32_t* q, const int64_t* offsets,
                  const int32_t* lengths, int64_t B, int dim, int norm, int64_t* out, int threads);

/* ---- sampled all-pairs entries: out[k] = δ(A[ia[k]], B[ib[k]]), dense sets
 * A: [nA, lenA, dim], B: [nB, lenB, dim] (only the sampled curves are read). */
int orc_cdist_entries_f32(const float* A, int32_t lenA, const float* B, int32_t lenB, int dim,
                          int norm, const int64_t* ia, const int64_t* ib, int64_t count,
                          double* out, int threads);
int orc_cdist_entries_f32mirror(const float* A, int32_t lenA, const float* B, int32_t lenB,
                                int dim, int norm, const int64_t* ia, const int64_t* ib,
                                int64_t count, float* out, int threads);

/* ---- DTW (PAPER Appendix B): max replaced by + ------------------ */
double orc_dtw_table_d(const double* d, int64_t P, int64_t Q);
double orc_dtw_alg_d(const double* d, int64_t P, int64_t Q);
/* DTW by definition (min over monotone couplings of the sum of d), P,Q ≤ 10 */
double orc_dtw_brute_d(const double* d, int64_t P, int64_t Q);
/* DTW of curve pairs: fp64 table with lazily evaluated d, and the fp32 mirror
 * of the kernels' operation order (L2: sqrt per cell) — DESIGN.md §DTW       */
int orc_pair_dtw_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                     double* out);
int orc_pair_dtw_f32mirror(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                           float* out);
int orc_batch_dtw_f32(const float* p, const float* q, const int64_t* offsets,
                      const int32_t* lengths, int64_t B, int dim, int norm, double* out,
                      int threads);
int orc_batch_dtw_f32mirror(const float* p, const float* q, const int64_t* offsets,
                            const int32_t* lengths, int64_t B, int dim, int norm, float* out,
                            int threads);

/* ---- Σ_ij d_ij: the paper's "upper limit" baseline --
 * The sum over all P·Q point distances of a pair, with the same d_ij as the DP
 * (L2 = sqrt per cell, the paper's hypot workload L271), in fp64 in row-major
 * order.  It is what the paper's SIMD DP "comes close" to: the cost of the
 * distances alone, without the recurrence. */
int orc_pair_dist_sum_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                          double* out);
int orc_batch_dist_sum_f32(const float* p, const float* q, const int64_t* offsets,
                           const int32_t* lengths, int64_t B, int dim, int norm, double* out,
                           int threads);

#ifdef __cplusplus
}
#endif
#endif
