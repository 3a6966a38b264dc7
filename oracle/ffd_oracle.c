/* ffd_oracle.c — plain CPU oracle for the discrete Fréchet distance.
 *
 * TEST INFRASTRUCTURE ONLY (see ffd_oracle.h).  Written from PAPER.md
 * (arxiv 2404.05708) alone; no blocking, fusion or reordering beyond what the
 * cited algorithm states.  Every function names the passage it follows.
 *
 * Parity pins (tests/test_oracle_*.py, all `-m "not gpu"`): brute-force
 * enumeration of couplings (definition), hand-derived worked examples
 * (tests/golden/worked_examples.json), closed forms (length-1 curves,
 * translation), invariants (symmetry, reversal, repeated points, membership,
 * Hausdorff and endpoint bounds, triangle inequality, norm ordering) and
 * bit-exact agreement of the table, Alg. 4, Alg. 5 and Alg. 2 forms.
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fopenmp -shared -fPIC -lm
 */
#include "ffd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static double dmin2(double a, double b) { return a < b ? a : b; }
static double dmax2(double a, double b) { return a > b ? a : b; }
static double dmin3(double a, double b, double c) { return dmin2(dmin2(a, b), c); }
static int64_t imin2(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t imax2(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t imin3(int64_t a, int64_t b, int64_t c) { return imin2(imin2(a, b), c); }

/* ------------------------------------------------------------------------- */
/* point distance f(p_i, q_j): PAPER L67 (‖·‖_S), L271 (Euclidean via hypot). */
/* L2 is the plain Euclidean norm sqrt(Σ Δ²) (reading 1); SQL2 is   */
/* Σ Δ²; L1 is Σ|Δ|; LINF is max|Δ|.  fp32 inputs are widened to fp64.       */
/* ------------------------------------------------------------------------- */
double orc_point_dist_f32(const float* a, const float* b, int dim, int norm) {
  double acc = 0.0;
  for (int k = 0; k < dim; k++) {
    double delta = (double)a[k] - (double)b[k];
    if (norm == ORC_L1) acc += fabs(delta);
    else if (norm == ORC_LINF) acc = dmax2(acc, fabs(delta));
    else acc += delta * delta;
  }
  if (norm == ORC_L2) acc = sqrt(acc);
  return acc;
}

int orc_point_dist_i32(const int32_t* a, const int32_t* b, int dim, int norm, int64_t* out) {
  __int128 acc = 0;
  for (int k = 0; k < dim; k++) {
    __int128 delta = (__int128)a[k] - (__int128)b[k];
    __int128 mag = delta < 0 ? -delta : delta;
    if (norm == ORC_L1) acc += mag;
    else if (norm == ORC_LINF) acc = acc > mag ? acc : mag;
    else if (norm == ORC_SQL2) acc += delta * delta;
    else return ORC_ERR_ARG; /* L2 (a square root) is not an integer result */
  }
  if (acc > (__int128)INT64_MAX) return ORC_ERR_OVERFLOW;
  *out = (int64_t)acc;
  return ORC_OK;
}

static int check_norm_f(int dim, int norm) {
  if (dim < 1 || dim > 4) return ORC_ERR_ARG;
  if (norm != ORC_L1 && norm != ORC_L2 && norm != ORC_LINF && norm != ORC_SQL2) return ORC_ERR_ARG;
  return ORC_OK;
}

static int check_finite(const float* x, int64_t npts, int dim) {
  for (int64_t i = 0; i < npts * dim; i++)
    if (!isfinite(x[i])) return ORC_ERR_NONFINITE;
  return ORC_OK;
}

int orc_dist_matrix_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                        double* d) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  for (int64_t i = 0; i < P; i++)
    for (int64_t j = 0; j < Q; j++)
      d[i * Q + j] = orc_point_dist_f32(p + i * dim, q + j * dim, dim, norm);
  return ORC_OK;
}

int orc_dist_matrix_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                        int64_t* d) {
  if (dim < 1 || dim > 4) return ORC_ERR_ARG;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  for (int64_t i = 0; i < P; i++)
    for (int64_t j = 0; j < Q; j++) {
      int st = orc_point_dist_i32(p + i * dim, q + j * dim, dim, norm, &d[i * Q + j]);
      if (st) return st;
    }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Alg. 3 / Eq. (1), padded-table restatement:   */
/*   C[0][0] = 0, C[0][j>0] = C[i>0][0] = +inf,                               */
/*   C[i][j] = max(min(C[i-1][j], C[i-1][j-1], C[i][j-1]), d[i-1][j-1]).      */
/* With every d ≥ 0 the four branches of Alg. 3 are exactly these cells.      */
/* ------------------------------------------------------------------------- */
void orc_frechet_full_table_d(const double* d, int64_t P, int64_t Q, double* C) {
  const int64_t W = Q + 1;
  C[0] = 0.0;
  for (int64_t j = 1; j <= Q; j++) C[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    C[i * W] = INFINITY;
    for (int64_t j = 1; j <= Q; j++) {
      double up = C[(i - 1) * W + j], diag = C[(i - 1) * W + (j - 1)], left = C[i * W + (j - 1)];
      C[i * W + j] = dmax2(dmin3(up, diag, left), d[(i - 1) * Q + (j - 1)]);
    }
  }
}

double orc_frechet_table_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  double* C = (double*)malloc(sizeof(double) * (size_t)(P + 1) * (size_t)(Q + 1));
  if (!C) return NAN;
  orc_frechet_full_table_d(d, P, Q, C);
  double r = C[P * (Q + 1) + Q];
  free(C);
  return r;
}

int64_t orc_frechet_table_i(const int64_t* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return INT64_MIN;
  const int64_t W = Q + 1;
  int64_t* C = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P + 1) * (size_t)W);
  if (!C) return INT64_MIN;
  C[0] = 0;
  for (int64_t j = 1; j <= Q; j++) C[j] = INT64_MAX;
  for (int64_t i = 1; i <= P; i++) {
    C[i * W] = INT64_MAX;
    for (int64_t j = 1; j <= Q; j++) {
      int64_t up = C[(i - 1) * W + j], diag = C[(i - 1) * W + (j - 1)], left = C[i * W + (j - 1)];
      C[i * W + j] = imax2(imin3(up, diag, left), d[(i - 1) * Q + (j - 1)]);
    }
  }
  int64_t r = C[P * W + Q];
  free(C);
  return r;
}

/* ------------------------------------------------------------------------- */
/* Alg. 4, in place on (a copy of) d:                       */
/*   d[:,1] ← max\(d[:,1]);  d[1,:] ← max\(d[1,:]);                           */
/*   for i=2..P, j=2..Q: d_ij ← max(min(d_{i-1,j}, d_{i-1,j-1}, d_{i,j-1}), d_ij) */
/* ------------------------------------------------------------------------- */
double orc_frechet_inplace_d(const double* d_in, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  double* d = (double*)malloc(sizeof(double) * (size_t)P * (size_t)Q);
  if (!d) return NAN;
  memcpy(d, d_in, sizeof(double) * (size_t)P * (size_t)Q);
  for (int64_t i = 1; i < P; i++) d[i * Q] = dmax2(d[(i - 1) * Q], d[i * Q]);       /* L210 */
  for (int64_t j = 1; j < Q; j++) d[j] = dmax2(d[j - 1], d[j]);                     /* L211 */
  for (int64_t i = 1; i < P; i++)                                                   /* L213 */
    for (int64_t j = 1; j < Q; j++)                                                 /* L214 */
      d[i * Q + j] = dmax2(dmin3(d[(i - 1) * Q + j], d[(i - 1) * Q + (j - 1)], d[i * Q + (j - 1)]),
                           d[i * Q + j]);                                           /* L215 */
  double r = d[P * Q - 1];
  free(d);
  return r;
}

/* ------------------------------------------------------------------------- */
/* Alg. 5, linear memory, written for a given row source.   */
/*   v ← max\(f(p_1, q))                                              (L234)  */
/*   for i = 2..P:                                                            */
/*     v_{2..Q} ← min(v_{1..Q-1}, v_{2..Q})  (simultaneous, reading 3) (L237) */
/*     v_1 ← max(v_1, f(p_i, q_1))                                     (L239) */
/*     for j = 2..Q: v_j ← max(min(v_{j-1}, v_j), f(p_i, q_j))         (L241) */
/*   return v_Q                                                        (L245) */
/* The simultaneous element-wise min is realised by sweeping j downwards so   */
/* that every min reads the pre-update v_{j-1}.                               */
/* ------------------------------------------------------------------------- */
#define ALG5_BODY(T, MIN2, MAX2, ROW_D)                                         \
  for (int64_t j = 0; j < Q; j++) {                                            \
    T dij = ROW_D(0, j);                                                       \
    v[j] = (j == 0) ? dij : MAX2(v[j - 1], dij);                               \
  }                                                                            \
  for (int64_t i = 1; i < P; i++) {                                            \
    for (int64_t j = Q - 1; j >= 1; j--) v[j] = MIN2(v[j - 1], v[j]);          \
    v[0] = MAX2(v[0], ROW_D(i, 0));                                            \
    for (int64_t j = 1; j < Q; j++) v[j] = MAX2(MIN2(v[j - 1], v[j]), ROW_D(i, j)); \
  }

double orc_frechet_linear_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  double* v = (double*)malloc(sizeof(double) * (size_t)Q);
  if (!v) return NAN;
#define D_FROM_MATRIX(i, j) d[(i) * Q + (j)]
  ALG5_BODY(double, dmin2, dmax2, D_FROM_MATRIX)
  double r = v[Q - 1];
  free(v);
  return r;
}

int64_t orc_frechet_linear_i(const int64_t* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return INT64_MIN;
  int64_t* v = (int64_t*)malloc(sizeof(int64_t) * (size_t)Q);
  if (!v) return INT64_MIN;
  ALG5_BODY(int64_t, imin2, imax2, D_FROM_MATRIX)
#undef D_FROM_MATRIX
  int64_t r = v[Q - 1];
  free(v);
  return r;
}

/* ------------------------------------------------------------------------- */
/* Alg. 2 literally with the scan/fold operators of         */
/* Alg. 6/7 (L333–L373).                                                      */
/*   fréchet_maxmin(a, x) = max{min{a, x_1}, x_2}                      (L141) */
/*   fréchet_next(a, x):  a_{2..Q} ← min{a_{1..Q-1}, a_{2..Q}}         (L145) */
/*                        return fréchet_maxmin\(max{a_1,x_1}, [a_{2..Q}|x_{2..Q}]) (L146) */
/*   fréchet_distance(d) = [fréchet_next/(max\(d_1), d_{2..P})]_Q      (L150) */
/* scan prepends its initial value (L126, L339); same-type scan/fold take the */
/* first element as initial value (L127, L350, L369).                         */
/* ------------------------------------------------------------------------- */
static double frechet_maxmin(double a, const double x[2]) { return dmax2(dmin2(a, x[0]), x[1]); }

/* Alg. 6, general form: y_1 = t0; t ← f(t, x_i); y_{i+1} = t.  x has N rows. */
static void scan_maxmin(double t0, const double (*x)[2], int64_t N, double* y) {
  y[0] = t0;
  double t = t0;
  for (int64_t i = 0; i < N; i++) {
    t = frechet_maxmin(t, x[i]);
    y[i + 1] = t;
  }
}

/* Alg. 6, same-type form for max: max\(x) = max\(x_1, x_{2..N}). */
static void scan_max(const double* x, int64_t N, double* y) {
  y[0] = x[0];
  double t = x[0];
  for (int64_t i = 1; i < N; i++) {
    t = dmax2(t, x[i]);
    y[i] = t;
  }
}

/* fréchet_next(a, x) -> result written to out (length Q) */
static void frechet_next(const double* a_in, const double* x, int64_t Q, double* out,
                         double* a, double (*stack)[2]) {
  memcpy(a, a_in, sizeof(double) * (size_t)Q);
  /* L145: a_{2..Q} ← min{a_{1..Q-1}, a_{2..Q}}, element-wise on the old values */
  for (int64_t j = 1; j < Q; j++) a[j] = dmin2(a_in[j - 1], a_in[j]);
  /* L146: stack [a_{2..Q} | x_{2..Q}] into a (Q-1)×2 matrix, scan row-wise */
  for (int64_t j = 1; j < Q; j++) {
    stack[j - 1][0] = a[j];
    stack[j - 1][1] = x[j];
  }
  scan_maxmin(dmax2(a[0], x[0]), (const double (*)[2])stack, Q - 1, out);
}

double orc_frechet_alg2_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  double* t = (double*)malloc(sizeof(double) * (size_t)Q);
  double* nxt = (double*)malloc(sizeof(double) * (size_t)Q);
  double* a = (double*)malloc(sizeof(double) * (size_t)Q);
  double (*stack)[2] = (double (*)[2])malloc(sizeof(double) * 2 * (size_t)(Q > 1 ? Q - 1 : 1));
  if (!t || !nxt || !a || !stack) { free(t); free(nxt); free(a); free(stack); return NAN; }
  /* L150: fold (Alg. 7) of fréchet_next with t0 = max\(d_1) over rows d_2..d_P */
  scan_max(d, Q, t);
  for (int64_t i = 1; i < P; i++) {
    frechet_next(t, d + i * Q, Q, nxt, a, stack);
    memcpy(t, nxt, sizeof(double) * (size_t)Q);
  }
  double r = t[Q - 1]; /* [·]_Q */
  free(t); free(nxt); free(a); free(stack);
  return r;
}

/* ------------------------------------------------------------------------- */
/* Definition (PAPER; Eiter–Mannila): δ_dF = min over monotone        */
/* couplings from (1,1) to (P,Q) with steps (1,0), (0,1), (1,1) of the max    */
/* d along the coupling.  Exhaustive depth-first enumeration; tiny inputs.    */
/* ------------------------------------------------------------------------- */
static double brute_rec_d(const double* d, int64_t P, int64_t Q, int64_t i, int64_t j, double cur) {
  if (i == P - 1 && j == Q - 1) return cur;
  double best = INFINITY;
  if (i + 1 < P) best = dmin2(best, brute_rec_d(d, P, Q, i + 1, j, dmax2(cur, d[(i + 1) * Q + j])));
  if (j + 1 < Q) best = dmin2(best, brute_rec_d(d, P, Q, i, j + 1, dmax2(cur, d[i * Q + j + 1])));
  if (i + 1 < P && j + 1 < Q)
    best = dmin2(best, brute_rec_d(d, P, Q, i + 1, j + 1, dmax2(cur, d[(i + 1) * Q + j + 1])));
  return best;
}

double orc_frechet_brute_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1 || P > 10 || Q > 10) return NAN;
  return brute_rec_d(d, P, Q, 0, 0, d[0]);
}

static int64_t brute_rec_i(const int64_t* d, int64_t P, int64_t Q, int64_t i, int64_t j, int64_t cur) {
  if (i == P - 1 && j == Q - 1) return cur;
  int64_t best = INT64_MAX;
  if (i + 1 < P) best = imin2(best, brute_rec_i(d, P, Q, i + 1, j, imax2(cur, d[(i + 1) * Q + j])));
  if (j + 1 < Q) best = imin2(best, brute_rec_i(d, P, Q, i, j + 1, imax2(cur, d[i * Q + j + 1])));
  if (i + 1 < P && j + 1 < Q)
    best = imin2(best, brute_rec_i(d, P, Q, i + 1, j + 1, imax2(cur, d[(i + 1) * Q + j + 1])));
  return best;
}

int64_t orc_frechet_brute_i(const int64_t* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1 || P > 10 || Q > 10) return INT64_MIN;
  return brute_rec_i(d, P, Q, 0, 0, d[0]);
}

/* discrete Hausdorff: max(max_i min_j d_ij, max_j min_i d_ij) */
double orc_hausdorff_d(const double* d, int64_t P, int64_t Q) {
  double h = 0.0;
  for (int64_t i = 0; i < P; i++) {
    double m = INFINITY;
    for (int64_t j = 0; j < Q; j++) m = dmin2(m, d[i * Q + j]);
    h = dmax2(h, m);
  }
  for (int64_t j = 0; j < Q; j++) {
    double m = INFINITY;
    for (int64_t i = 0; i < P; i++) m = dmin2(m, d[i * Q + j]);
    h = dmax2(h, m);
  }
  return h;
}

/* ------------------------------------------------------------------------- */
/* Pair-level forms with lazily evaluated d_ij (Theorem 1).       */
/* ------------------------------------------------------------------------- */
int orc_pair_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                 double* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  /* padded table, two rows at a time would be Alg. 5; keep the whole table.  */
  const int64_t W = Q + 1;
  double* C = (double*)malloc(sizeof(double) * (size_t)(P + 1) * (size_t)W);
  if (!C) return ORC_ERR_ARG;
  C[0] = 0.0;
  for (int64_t j = 1; j <= Q; j++) C[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    C[i * W] = INFINITY;
    for (int64_t j = 1; j <= Q; j++) {
      double dij = orc_point_dist_f32(p + (i - 1) * dim, q + (j - 1) * dim, dim, norm);
      C[i * W + j] = dmax2(dmin3(C[(i - 1) * W + j], C[(i - 1) * W + j - 1], C[i * W + j - 1]), dij);
    }
  }
  *out = C[P * W + Q];
  free(C);
  return ORC_OK;
}

int orc_pair_linear_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                        double* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  double* v = (double*)malloc(sizeof(double) * (size_t)Q);
  if (!v) return ORC_ERR_ARG;
#define D_LAZY_F(i, j) orc_point_dist_f32(p + (i) * dim, q + (j) * dim, dim, norm)
  ALG5_BODY(double, dmin2, dmax2, D_LAZY_F)
#undef D_LAZY_F
  *out = v[Q - 1];
  free(v);
  return ORC_OK;
}

int orc_pair_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                 int64_t* out) {
  if (dim < 1 || dim > 4) return ORC_ERR_ARG;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  const int64_t W = Q + 1;
  int64_t* C = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P + 1) * (size_t)W);
  if (!C) return ORC_ERR_ARG;
  C[0] = 0;
  for (int64_t j = 1; j <= Q; j++) C[j] = INT64_MAX;
  for (int64_t i = 1; i <= P; i++) {
    C[i * W] = INT64_MAX;
    for (int64_t j = 1; j <= Q; j++) {
      int64_t dij;
      int st = orc_point_dist_i32(p + (i - 1) * dim, q + (j - 1) * dim, dim, norm, &dij);
      if (st) { free(C); return st; }
      C[i * W + j] = imax2(imin3(C[(i - 1) * W + j], C[(i - 1) * W + j - 1], C[i * W + j - 1]), dij);
    }
  }
  *out = C[P * W + Q];
  free(C);
  return ORC_OK;
}

static int64_t dist_i_or_flag(const int32_t* a, const int32_t* b, int dim, int norm, int* bad) {
  int64_t r = 0;
  if (orc_point_dist_i32(a, b, dim, norm, &r)) { *bad = 1; return INT64_MAX; }
  return r;
}

int orc_pair_linear_i32(const int32_t* p, int64_t P, const int32_t* q, int64_t Q, int dim, int norm,
                        int64_t* out) {
  if (dim < 1 || dim > 4) return ORC_ERR_ARG;
  if (norm == ORC_L2) return ORC_ERR_ARG;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  int64_t* v = (int64_t*)malloc(sizeof(int64_t) * (size_t)Q);
  if (!v) return ORC_ERR_ARG;
  int bad = 0;
#define D_LAZY_I(i, j) dist_i_or_flag(p + (i) * dim, q + (j) * dim, dim, norm, &bad)
  ALG5_BODY(int64_t, imin2, imax2, D_LAZY_I)
#undef D_LAZY_I
  *out = v[Q - 1];
  free(v);
  return bad ? ORC_ERR_OVERFLOW : ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* fp32 mirror: the table DP evaluated in fp32 with */
/* the operation order documented for the kernels:                            */
/*   Δ_k = p_k − q_k (fp32);  SQL2/L2: s = Δ_0·Δ_0; s = fmaf(Δ_k, Δ_k, s) k≥1 */
/*   L1: s = |Δ_0| + |Δ_1| + … (left to right);  LINF: s = max_k |Δ_k|        */
/*   L2 reports sqrtf(δ_SQL2): the square root is taken once at the end       */
/*   (monotone, reading 11).  min/max only select, so the DP adds   */
/*   no rounding.  Compiled with -ffp-contract=off.                           */
/* ------------------------------------------------------------------------- */
static float mirror_dist(const float* a, const float* b, int dim, int norm) {
  float s = 0.0f;
  for (int k = 0; k < dim; k++) {
    float delta = a[k] - b[k];
    if (norm == ORC_L1) s = (k == 0) ? fabsf(delta) : s + fabsf(delta);
    else if (norm == ORC_LINF) s = (k == 0) ? fabsf(delta) : fmaxf(s, fabsf(delta));
    else s = (k == 0) ? delta * delta : fmaf(delta, delta, s);
  }
  return s;
}

int orc_pair_f32mirror(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                       float* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  /* two table rows suffice (Alg. 3 order); kept as a plain row-by-row table  */
  float* prev = (float*)malloc(sizeof(float) * (size_t)(Q + 1));
  float* cur = (float*)malloc(sizeof(float) * (size_t)(Q + 1));
  if (!prev || !cur) { free(prev); free(cur); return ORC_ERR_ARG; }
  prev[0] = 0.0f;
  for (int64_t j = 1; j <= Q; j++) prev[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    cur[0] = INFINITY;
    for (int64_t j = 1; j <= Q; j++) {
      float dij = mirror_dist(p + (i - 1) * dim, q + (j - 1) * dim, dim, norm);
      cur[j] = fmaxf(fminf(fminf(prev[j], prev[j - 1]), cur[j - 1]), dij);
    }
    float* t = prev; prev = cur; cur = t;
  }
  float r = prev[Q];
  free(prev); free(cur);
  *out = (norm == ORC_L2) ? sqrtf(r) : r;
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Batches and sampled all-pairs entries: one independent pair at a time.     */
/* ------------------------------------------------------------------------- */
static int threads_or_default(int threads) {
#ifdef _OPENMP
  return threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
  return 1;
#endif
}

int orc_batch_f32(const float* p, const float* q, const int64_t* offsets, const int32_t* lengths,
                  int64_t B, int dim, int norm, double* out, int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    double r = NAN;
    int st = orc_pair_f32(p + offsets[k] * dim, lengths[k], q + offsets[B + k] * dim,
                          lengths[B + k], dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

int orc_batch_f32mirror(const float* p, const float* q, const int64_t* offsets,
                        const int32_t* lengths, int64_t B, int dim, int norm, float* out,
                        int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    float r = NAN;
    int st = orc_pair_f32mirror(p + offsets[k] * dim, lengths[k], q + offsets[B + k] * dim,
                                lengths[B + k], dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

int orc_batch_i32(const int32_t* p, const int32_t* q, const int64_t* offsets,
                  const int32_t* lengths, int64_t B, int dim, int norm, int64_t* out, int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    int64_t r = INT64_MIN;
    int st = (norm == ORC_L2) ? ORC_ERR_ARG
                              : orc_pair_i32(p + offsets[k] * dim, lengths[k],
                                             q + offsets[B + k] * dim, lengths[B + k], dim, norm, &r);
    out[k] = st ? INT64_MIN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

int orc_cdist_entries_f32(const float* A, int32_t lenA, const float* B, int32_t lenB, int dim,
                          int norm, const int64_t* ia, const int64_t* ib, int64_t count,
                          double* out, int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < count; k++) {
    double r = NAN;
    int st = orc_pair_f32(A + ia[k] * lenA * dim, lenA, B + ib[k] * lenB * dim, lenB, dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

int orc_cdist_entries_f32mirror(const float* A, int32_t lenA, const float* B, int32_t lenB,
                                int dim, int norm, const int64_t* ia, const int64_t* ib,
                                int64_t count, float* out, int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < count; k++) {
    float r = NAN;
    int st = orc_pair_f32mirror(A + ia[k] * lenA * dim, lenA, B + ib[k] * lenB * dim, lenB, dim,
                                norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

/* ------------------------------------------------------------------------- */
/* DTW (PAPER Appendix B): "replacing max with summation".         */
/* Table: D[0][0]=0, borders +inf, D[i][j] = d + min(D[i-1][j], D[i-1][j-1], D[i][j-1]). */
/* Alg. (L386–L397): dtw_min(a,x) = min{a,x_1}+x_2;                            */
/*   dtw_next(a,x): a_{2..Q} ← min{a_{1..Q-1}, a_{2..Q}};                      */
/*                  return dtw_min\(a_1 + x_1, [a_{2..Q} | x_{2..Q}]);         */
/*   dtw_distance(d) = [dtw_next/(+\d_1, d_{2..P})]_Q  (the closing ]_Q is    */
/*   missing in the source, reading 14).                            */
/* ------------------------------------------------------------------------- */
double orc_dtw_table_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  const int64_t W = Q + 1;
  double* C = (double*)malloc(sizeof(double) * (size_t)(P + 1) * (size_t)W);
  if (!C) return NAN;
  C[0] = 0.0;
  for (int64_t j = 1; j <= Q; j++) C[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    C[i * W] = INFINITY;
    for (int64_t j = 1; j <= Q; j++)
      C[i * W + j] = d[(i - 1) * Q + j - 1] + dmin3(C[(i - 1) * W + j], C[(i - 1) * W + j - 1], C[i * W + j - 1]);
  }
  double r = C[P * W + Q];
  free(C);
  return r;
}

double orc_dtw_alg_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1) return NAN;
  double* t = (double*)malloc(sizeof(double) * (size_t)Q);
  double* a = (double*)malloc(sizeof(double) * (size_t)Q);
  if (!t || !a) { free(t); free(a); return NAN; }
  /* +\d_1: same-type scan of + over the first row */
  t[0] = d[0];
  for (int64_t j = 1; j < Q; j++) t[j] = t[j - 1] + d[j];
  for (int64_t i = 1; i < P; i++) {
    const double* x = d + i * Q;
    for (int64_t j = 1; j < Q; j++) a[j] = dmin2(t[j - 1], t[j]); /* element-wise on old values */
    a[0] = t[0];
    /* scan of dtw_min with initial value a_1 + x_1 over [a_{2..Q} | x_{2..Q}] */
    double acc = a[0] + x[0];
    t[0] = acc;
    for (int64_t j = 1; j < Q; j++) {
      acc = dmin2(acc, a[j]) + x[j];
      t[j] = acc;
    }
  }
  double r = t[Q - 1];
  free(t); free(a);
  return r;
}

/* ------------------------------------------------------------------------- */
/* DTW by definition, for pinning: min over all monotone couplings (the same  */
/* couplings as the Fréchet brute force) of the SUM of d along */
/* the coupling.  Exponential: P, Q ≤ 10 only.                                */
/* ------------------------------------------------------------------------- */
static double dtw_brute_rec(const double* d, int64_t P, int64_t Q, int64_t i, int64_t j, double acc) {
  acc += d[i * Q + j];
  if (i == P - 1 && j == Q - 1) return acc;
  double best = INFINITY;
  if (i + 1 < P) best = dmin2(best, dtw_brute_rec(d, P, Q, i + 1, j, acc));
  if (j + 1 < Q) best = dmin2(best, dtw_brute_rec(d, P, Q, i, j + 1, acc));
  if (i + 1 < P && j + 1 < Q) best = dmin2(best, dtw_brute_rec(d, P, Q, i + 1, j + 1, acc));
  return best;
}

double orc_dtw_brute_d(const double* d, int64_t P, int64_t Q) {
  if (P < 1 || Q < 1 || P > 10 || Q > 10) return NAN;
  return dtw_brute_rec(d, P, Q, 0, 0, 0.0);
}

/* DTW of one pair with lazily evaluated d (fp64; table rows of Appendix B's   */
/* recurrence): C[0][0]=0, borders +inf,                      */
/* C[i][j] = d(p_{i-1}, q_{j-1}) + min(C[i-1][j], C[i-1][j-1], C[i][j-1]).     */
int orc_pair_dtw_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                     double* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  double* prev = (double*)malloc(sizeof(double) * (size_t)(Q + 1));
  double* cur = (double*)malloc(sizeof(double) * (size_t)(Q + 1));
  if (!prev || !cur) { free(prev); free(cur); return ORC_ERR_ARG; }
  prev[0] = 0.0;
  for (int64_t j = 1; j <= Q; j++) prev[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    cur[0] = INFINITY;
    for (int64_t j = 1; j <= Q; j++)
      cur[j] = orc_point_dist_f32(p + (i - 1) * dim, q + (j - 1) * dim, dim, norm) +
               dmin3(prev[j], prev[j - 1], cur[j - 1]);
    double* t = prev; prev = cur; cur = t;
  }
  *out = prev[Q];
  free(prev); free(cur);
  return ORC_OK;
}

/* DTW fp32 mirror: the same table in fp32 with the kernels' operation order: */
/* d as in mirror_dist (L2: sqrtf of the squared sum, per cell — a sum of     */
/* distances cannot take the root once at the end), c = min(min(up, diag),    */
/* left) + d with one fp32 rounding per cell.                                  */
int orc_pair_dtw_f32mirror(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                           float* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  float* prev = (float*)malloc(sizeof(float) * (size_t)(Q + 1));
  float* cur = (float*)malloc(sizeof(float) * (size_t)(Q + 1));
  if (!prev || !cur) { free(prev); free(cur); return ORC_ERR_ARG; }
  prev[0] = 0.0f;
  for (int64_t j = 1; j <= Q; j++) prev[j] = INFINITY;
  for (int64_t i = 1; i <= P; i++) {
    cur[0] = INFINITY;
    for (int64_t j = 1; j <= Q; j++) {
      float dij = mirror_dist(p + (i - 1) * dim, q + (j - 1) * dim, dim, norm);
      if (norm == ORC_L2) dij = sqrtf(dij);
      cur[j] = fminf(fminf(prev[j], prev[j - 1]), cur[j - 1]) + dij;
    }
    float* t = prev; prev = cur; cur = t;
  }
  *out = prev[Q];
  free(prev); free(cur);
  return ORC_OK;
}

int orc_batch_dtw_f32(const float* p, const float* q, const int64_t* offsets,
                      const int32_t* lengths, int64_t B, int dim, int norm, double* out,
                      int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    double r = NAN;
    int st = orc_pair_dtw_f32(p + offsets[k] * dim, lengths[k], q + offsets[B + k] * dim,
                              lengths[B + k], dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

int orc_batch_dtw_f32mirror(const float* p, const float* q, const int64_t* offsets,
                            const int32_t* lengths, int64_t B, int dim, int norm, float* out,
                            int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    float r = NAN;
    int st = orc_pair_dtw_f32mirror(p + offsets[k] * dim, lengths[k], q + offsets[B + k] * dim,
                                    lengths[B + k], dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}

/* ---- Σ_ij d_ij ------------------------------------- */
int orc_pair_dist_sum_f32(const float* p, int64_t P, const float* q, int64_t Q, int dim, int norm,
                          double* out) {
  int st = check_norm_f(dim, norm);
  if (st) return st;
  if (P < 1 || Q < 1) return ORC_ERR_EMPTY;
  if (check_finite(p, P, dim) || check_finite(q, Q, dim)) return ORC_ERR_NONFINITE;
  double s = 0.0;
  for (int64_t i = 0; i < P; i++)
    for (int64_t j = 0; j < Q; j++) s += orc_point_dist_f32(p + i * dim, q + j * dim, dim, norm);
  *out = s;
  return ORC_OK;
}

int orc_batch_dist_sum_f32(const float* p, const float* q, const int64_t* offsets,
                           const int32_t* lengths, int64_t B, int dim, int norm, double* out,
                           int threads) {
  int first = ORC_OK;
  int nt = threads_or_default(threads);
  (void)nt;
#pragma omp parallel for schedule(dynamic, 8) num_threads(nt)
  for (int64_t k = 0; k < B; k++) {
    double r = NAN;
    int st = orc_pair_dist_sum_f32(p + offsets[k] * dim, lengths[k], q + offsets[B + k] * dim,
                                   lengths[B + k], dim, norm, &r);
    out[k] = st ? NAN : r;
    if (st) {
#pragma omp critical
      if (first == ORC_OK) first = st;
    }
  }
  return first;
}
