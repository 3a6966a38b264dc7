/* ffd_gen.c — seeded synthetic random-walk curves (the only code shared by the
 * oracle-side tests and the CUDA-side bench/tests).  It holds none of the
 * method's arithmetic: no distances, no DP.
 *
 * Workload shapes follow PAPER.md L268–L271 (random walks; steps uniform in
 * {−1,0,+1} per coordinate) and BASELINE.json configs 1–5 (Gaussian steps,
 * uniform integer steps, per-curve Gaussian start offsets, uniform lengths).
 *
 * Generator: counter-based SplitMix64.  Curve c of stream `tag` draws its
 * k-th 64-bit word as splitmix64(key(seed, tag, c) + (k+1)·γ), so any curve
 * is generated independently of the others (parallel and reproducible).
 * Gaussians: Box–Muller in fp64 (two normals per pair of uniforms); walks are
 * accumulated in fp64 and rounded to fp32 per point.
 */
#include <math.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define GAMMA 0x9E3779B97F4A7C15ULL

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static uint64_t curve_key(uint64_t seed, uint64_t tag, uint64_t c) {
  return mix64(mix64(seed ^ mix64(tag + GAMMA)) + c * GAMMA);
}

typedef struct {
  uint64_t key, k;
  int have_spare;
  double spare;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed, uint64_t tag, uint64_t c) {
  r->key = curve_key(seed, tag, c);
  r->k = 0;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_next(rng_t* r) {
  r->k++;
  return mix64(r->key + r->k * GAMMA);
}

/* uniform in (0, 1] with 53 bits */
static double rng_u01(rng_t* r) { return ((double)(rng_next(r) >> 11) + 1.0) * 0x1.0p-53; }

static double rng_normal(rng_t* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_u01(r), u2 = rng_u01(r);
  double rad = sqrt(-2.0 * log(u1));
  double ang = 6.283185307179586476925286766559 * u2;
  r->spare = rad * sin(ang);
  r->have_spare = 1;
  return rad * cos(ang);
}

/* integer uniformly in [lo, hi] (inclusive) via 64x64->128 multiply-high */
static int64_t rng_int(rng_t* r, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo) + 1ULL;
  unsigned __int128 m = (unsigned __int128)rng_next(r) * span;
  return lo + (int64_t)(m >> 64);
}

/* lengths[i] ~ U{lo..hi} for curve ids first..first+count-1, one word per curve */
void ffdgen_lengths(uint64_t seed, uint64_t tag, int64_t first, int64_t count, int32_t lo,
                    int32_t hi, int32_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; i++) {
    rng_t r;
    rng_init(&r, seed, tag, (uint64_t)(first + i));
    out[i] = (int32_t)rng_int(&r, lo, hi);
  }
}

/* Gaussian walks, fp32 output.  Curve i (global id first+i) has lengths[i]
 * points written at out + offsets[i]*dim.  Point 0 = start ~ N(0, start_sigma^2)
 * per coordinate (start_sigma = 0: origin); point t = point t-1 + N(0, sigma^2). */
void ffdgen_walks_f32(uint64_t seed, uint64_t tag, int64_t first, int64_t count,
                      const int32_t* lengths, const int64_t* offsets, int32_t dim, double sigma,
                      double start_sigma, float* out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < count; i++) {
    rng_t r;
    rng_init(&r, seed, tag, (uint64_t)(first + i));
    double pos[8];
    for (int k = 0; k < dim; k++) pos[k] = start_sigma > 0.0 ? start_sigma * rng_normal(&r) : 0.0;
    float* o = out + offsets[i] * dim;
    for (int32_t t = 0; t < lengths[i]; t++) {
      if (t > 0)
        for (int k = 0; k < dim; k++) pos[k] += sigma * rng_normal(&r);
      for (int k = 0; k < dim; k++) o[(int64_t)t * dim + k] = (float)pos[k];
    }
  }
}

/* integer walks from the origin, steps ~ U{step_lo..step_hi} per coordinate */
void ffdgen_walks_i32(uint64_t seed, uint64_t tag, int64_t first, int64_t count,
                      const int32_t* lengths, const int64_t* offsets, int32_t dim, int32_t step_lo,
                      int32_t step_hi, int32_t* out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < count; i++) {
    rng_t r;
    rng_init(&r, seed, tag, (uint64_t)(first + i));
    int64_t pos[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int32_t* o = out + offsets[i] * dim;
    for (int32_t t = 0; t < lengths[i]; t++) {
      if (t > 0)
        for (int k = 0; k < dim; k++) pos[k] += rng_int(&r, step_lo, step_hi);
      for (int k = 0; k < dim; k++) o[(int64_t)t * dim + k] = (int32_t)pos[k];
    }
  }
}

/* the paper's walks: steps uniform in {-1,0,+1} per coordinate, fp32 */
void ffdgen_walks_unit_f32(uint64_t seed, uint64_t tag, int64_t first, int64_t count,
                           const int32_t* lengths, const int64_t* offsets, int32_t dim, float* out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < count; i++) {
    rng_t r;
    rng_init(&r, seed, tag, (uint64_t)(first + i));
    double pos[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float* o = out + offsets[i] * dim;
    for (int32_t t = 0; t < lengths[i]; t++) {
      if (t > 0)
        for (int k = 0; k < dim; k++) pos[k] += (double)rng_int(&r, -1, 1);
      for (int k = 0; k < dim; k++) o[(int64_t)t * dim + k] = (float)pos[k];
    }
  }
}

/* uniform sample of `count` indices in [0, n) (with replacement), for sampled parity */
void ffdgen_indices(uint64_t seed, uint64_t tag, int64_t count, int64_t n, int64_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; i++) {
    rng_t r;
    rng_init(&r, seed, tag, (uint64_t)i);
    out[i] = rng_int(&r, 0, n - 1);
  }
}

int ffdgen_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
