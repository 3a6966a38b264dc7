// Per-SM issue/pipe throughput microbenchmark for the SASS ops the discrete
// Frechet DP cell is made of (SURVEY.md §2.5 N9, §8(d) "measured-pipe roofline").
//
// Each test runs NCHAIN independent dependency chains per thread, enough warps
// per SM to hide latency, and reports warp-instructions per SM clock measured
// with clock64() inside the kernel (so the result does not depend on the clock
// frequency).  The "cell" tests run the real DP cell arithmetic on R rows held
// in registers against a synthetic column stream held in registers (no LDS,
// no SHFL), giving the best-case cells/clk/SM for each formulation.
//
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
// Run:    ./pipes            (prints one JSON line per test)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int NCHAIN = 8;
constexpr int UNROLL = 4;

__device__ __forceinline__ uint64_t pack(float a, float b) {
  return (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(b) << 32);
}

// ---- single-op tests: each macro body updates x[u] from x[u] and y,z -------
template <int OP>
__global__ void op_kernel(float* out, long long* cyc, int iters) {
  float x[NCHAIN];
  int xi[NCHAIN];
  uint64_t x2[NCHAIN];
  float y = 1.0001f + threadIdx.x * 1e-7f, z = 0.9999f - threadIdx.x * 1e-7f;
  int yi = threadIdx.x | 1, zi = (threadIdx.x * 7) ^ 5;
  uint64_t y2 = pack(y, z), z2 = pack(z, y);
#pragma unroll
  for (int u = 0; u < NCHAIN; u++) {
    x[u] = threadIdx.x * 0.001f + u;
    xi[u] = threadIdx.x * 3 + u;
    x2[u] = pack(x[u], x[u] + 1.f);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < UNROLL; r++) {
#pragma unroll
      for (int u = 0; u < NCHAIN; u++) {
        if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[u]) : "f"(y), "f"(z));
        if (OP == 1) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x[u]) : "f"(y));
        if (OP == 2) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(x[u]) : "f"(y));
        if (OP == 3) asm volatile("min.f32 %0, %0, %1;" : "+f"(x[u]) : "f"(y));
        if (OP == 4) { float t; asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(x[u]), "f"(y), "f"(z)); x[u] = t; }
        if (OP == 5) asm volatile("add.s32 %0, %0, %1;" : "+r"(xi[u]) : "r"(yi));
        if (OP == 6) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(xi[u]) : "r"(yi), "r"(zi));
        if (OP == 7) asm volatile("min.s32 %0, %0, %1;" : "+r"(xi[u]) : "r"(yi));
        if (OP == 8) xi[u] = __vimin3_s32(xi[u], yi, zi);
        if (OP == 9) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x2[u]) : "l"(y2));
        if (OP == 10) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x2[u]) : "l"(y2), "l"(z2));
        if (OP == 11) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x2[u]) : "l"(y2));
        if (OP == 12) asm volatile("max.f32 %0, %0, %1;" : "+f"(x[u]) : "f"(y));
        if (OP == 13) x[u] = __shfl_up_sync(0xffffffffu, x[u], 1);
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < NCHAIN; u++) s += x[u] + (float)xi[u] + __uint_as_float((uint32_t)x2[u]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// ---- mixed independent streams: do two op types share one pipe? ----------
// MIX 0: FFMA2+FMNMX3  1: FFMA2+FMNMX  2: FFMA+FMNMX  3: FADD2+FFMA2+FMNMX3+FMNMX
// (the fp32 2-D cell mix, 7 slots on one shared pipe)  4: FADD2+2 FFMA2+2 FMNMX3+
// 2 FMNMX (two exact-int XSQ cells, 12 slots)  5: FMNMX3+FMNMX  6: FFMA2+IADD3
// 7: FMNMX3+IADD3.  instr_per_unit is the number of instructions per chain unit.
template <int MIX>
__global__ void mix_kernel(float* out, long long* cyc, int iters) {
  float a[NCHAIN], b[NCHAIN], x_acc[NCHAIN], y_acc[NCHAIN];
  int ia[NCHAIN];
  uint64_t p[NCHAIN], q[NCHAIN];
  float y = 1.0001f + threadIdx.x * 1e-7f, z = 0.9999f - threadIdx.x * 1e-7f;
  int yi = threadIdx.x | 1;
  uint64_t y2 = pack(y, z), z2 = pack(z, y);
#pragma unroll
  for (int u = 0; u < NCHAIN; u++) {
    a[u] = threadIdx.x * 0.001f + u;
    b[u] = threadIdx.x * 0.002f - u;
    x_acc[u] = 0.f;
    y_acc[u] = 0.f;
    ia[u] = threadIdx.x * 3 + u;
    p[u] = pack(a[u], a[u] + 1.f);
    q[u] = pack(b[u], b[u] + 2.f);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int r = 0; r < UNROLL; r++) {
#pragma unroll
      for (int u = 0; u < NCHAIN; u++) {
        if (MIX == 0 || MIX == 1 || MIX == 3 || MIX == 4 || MIX == 6)
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[u]) : "l"(y2), "l"(z2));
        if (MIX == 3 || MIX == 4)
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(q[u]) : "l"(y2));
        if (MIX == 4)
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[u]) : "l"(z2), "l"(y2));
        if (MIX == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(b[u]) : "f"(y), "f"(z));
        if (MIX == 0 || MIX == 3 || MIX == 4 || MIX == 5 || MIX == 7) {
          float t;
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(a[u]), "f"(y), "f"(z));
          a[u] = t;
        }
        if (MIX == 4) {
          float t;
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(b[u]), "f"(z), "f"(y));
          b[u] = t;
        }
        if (MIX == 1 || MIX == 2 || MIX == 3 || MIX == 4 || MIX == 5)
          asm volatile("max.f32 %0, %0, %1;" : "+f"(b[u]) : "f"(y));
        if (MIX == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[u]) : "f"(z));
        if (MIX == 6 || MIX == 7) asm volatile("add.s32 %0, %0, %1;" : "+r"(ia[u]) : "r"(yi));
        if (MIX == 8) {  // fp32 3-D SQ, two cells: 3 FADD2, FMUL2, 2 FFMA2, 2 FMNMX3, 2 FMNMX
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[u]) : "l"(y2));
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(q[u]) : "l"(y2));
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[u]) : "l"(z2));
          asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(q[u]) : "l"(z2));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[u]) : "l"(y2), "l"(z2));
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(q[u]) : "l"(z2), "l"(y2));
        }
        if (MIX == 8) {  // 2 x (FMNMX3 + FMNMX) on two chains
          float t;
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(a[u]), "f"(y), "f"(z));
          a[u] = t;
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(b[u]), "f"(z), "f"(y));
          b[u] = t;
          asm volatile("max.f32 %0, %0, %1;" : "+f"(a[u]) : "f"(z));
          asm volatile("max.f32 %0, %0, %1;" : "+f"(b[u]) : "f"(y));
        }
        if (MIX == 9 || MIX == 10) {  // fp32 2-D L1 / Linf, two cells: 2 FADD2 + 2 (|a| op |b|)
          // + 2 x (FMNMX3 + FMNMX); the distance feeds the max, as in the DP cell
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[u]) : "l"(y2));
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(q[u]) : "l"(z2));
          float r1, r2, t;
          if (MIX == 9) {
            asm volatile("{.reg .f32 l, h, al, ah; mov.b64 {l, h}, %1; abs.f32 al, l; abs.f32 ah, h; add.rn.f32 %0, al, ah;}"
                         : "=f"(r1) : "l"(p[u]));
            asm volatile("{.reg .f32 l, h, al, ah; mov.b64 {l, h}, %1; abs.f32 al, l; abs.f32 ah, h; add.rn.f32 %0, al, ah;}"
                         : "=f"(r2) : "l"(q[u]));
          } else {
            asm volatile("{.reg .f32 l, h, al, ah; mov.b64 {l, h}, %1; abs.f32 al, l; abs.f32 ah, h; max.f32 %0, al, ah;}"
                         : "=f"(r1) : "l"(p[u]));
            asm volatile("{.reg .f32 l, h, al, ah; mov.b64 {l, h}, %1; abs.f32 al, l; abs.f32 ah, h; max.f32 %0, al, ah;}"
                         : "=f"(r2) : "l"(q[u]));
          }
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(a[u]), "f"(y), "f"(z));
          a[u] = t;
          asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(b[u]), "f"(z), "f"(y));
          b[u] = t;
          asm volatile("max.f32 %0, %0, %1;" : "+f"(a[u]) : "f"(r1));
          asm volatile("max.f32 %0, %0, %1;" : "+f"(b[u]) : "f"(r2));
        }
      }
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < NCHAIN; u++)
    s += a[u] + b[u] + x_acc[u] + y_acc[u] + (float)ia[u] + __uint_as_float((uint32_t)p[u]) + __uint_as_float((uint32_t)q[u]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- cell tests: R rows in registers, one column per step ------------------
// q comes from a shared-memory ring (one LDS.128 per step, as in the real
// kernel); SHF=1 adds the lane-to-lane __shfl_up_sync of the real pipeline.
// VAR 0: fp32 2-D L2sq, scalar   (FADD FADD FMUL FFMA FMNMX3 FMNMX)
// VAR 1: fp32 2-D L2sq, packed f32x2 distance (FADD2 FADD2 FMUL2 FFMA2 per 2 rows)
// VAR 2: int32 2-D sqL2, standard (IADD3 IADD3 IMAD IMAD VIMNMX3 VIMNMX)
// VAR 3: int32 2-D sqL2, expansion |p|^2+|q|^2-2pq (IADD3 IMAD IMAD VIMNMX3 VIMNMX)
template <int VAR, int R, int SHF>
__global__ void cell_kernel(float* out, long long* cyc, int steps) {
  __shared__ float4 ring[4][128];
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 3;
  for (int i = lane; i < 128; i += 32)
    ring[w][i] = make_float4(i * 0.37f - 3.f, 1.5f - i * 0.21f, __int_as_float(i * 3 - 7), __int_as_float(5 - i));
  float px[R], py[R], pq[R], c[R];
  int ipx[R], ipy[R], ipp[R], ic[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    px[r] = lane * 0.37f + r; py[r] = r * 0.11f - lane; pq[r] = px[r] * px[r] + py[r] * py[r];
    c[r] = 1e30f;
    ipx[r] = lane * 3 + r; ipy[r] = r - lane; ipp[r] = ipx[r] * ipx[r] + ipy[r] * ipy[r];
    ic[r] = 0x7fffffff;
  }
  float b0_f = 0.f, diag_f = 0.f;
  int diag_i = 0;
  __syncthreads();
  long long t0 = clock64();
  int g = lane;
  for (int s = 0; s < steps; s++) {
    float4 e = ring[w][g & 127];
    g -= 1;
    if (VAR == 0) {
      float qx = e.x, qy = e.y;
      float upv = SHF ? __shfl_up_sync(0xffffffffu, c[R - 1], 1) : c[R - 1];
      float up = lane == 0 ? e.x : upv, dg = diag_f;
      diag_f = up;
#pragma unroll
      for (int r = 0; r < R; r++) {
        float dx = px[r] - qx, dy = py[r] - qy;
        float d = fmaf(dy, dy, dx * dx);
        float m = fminf(fminf(up, dg), c[r]);
        float nv = fmaxf(m, d);
        dg = c[r]; c[r] = nv; up = nv;
      }
    } else if (VAR == 1) {
      float upv = SHF ? __shfl_up_sync(0xffffffffu, c[R - 1], 1) : c[R - 1];
      float up = lane == 0 ? e.x : upv, dg = diag_f;
      diag_f = up;
      uint64_t q2x = pack(e.x, e.x), q2y = pack(e.y, e.y);
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        uint64_t p2x = pack(px[r], px[r + 1]), p2y = pack(py[r], py[r + 1]);
        uint64_t dx, dy, s2;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dx) : "l"(p2x), "l"(q2x));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(dy) : "l"(p2y), "l"(q2y));
        asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(s2) : "l"(dx));
        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(s2) : "l"(dy), "l"(s2));
        float d0 = __uint_as_float((uint32_t)s2), d1 = __uint_as_float((uint32_t)(s2 >> 32));
        float m0 = fminf(fminf(up, dg), c[r]);
        float n0 = fmaxf(m0, d0);
        float m1 = fminf(fminf(n0, c[r]), c[r + 1]);
        float n1 = fmaxf(m1, d1);
        dg = c[r + 1]; c[r] = n0; c[r + 1] = n1; up = n1;
      }
    } else if (VAR == 2) {
      int iqx = __float_as_int(e.z), iqy = __float_as_int(e.w);
      int upv = SHF ? __shfl_up_sync(0xffffffffu, ic[R - 1], 1) : ic[R - 1];
      int up = lane == 0 ? iqx : upv, dg = diag_i;
      diag_i = up;
#pragma unroll
      for (int r = 0; r < R; r++) {
        int dx = ipx[r] - iqx, dy = ipy[r] - iqy;
        int d = dx * dx + dy * dy;
        int m = __vimin3_s32(up, dg, ic[r]);
        int nv = max(m, d);
        dg = ic[r]; ic[r] = nv; up = nv;
      }
    } else if (VAR == 4 || VAR == 5 || VAR == 6) {
      // the c2 cell: int input in fp32-exact arithmetic, d = (pp + qq) + p'·(−2q')
      // on two rows at once (FADD2 + 2 FFMA2); VAR 4: chain FMNMX3 + FMNMX per row;
      // VAR 5: m = min(diag, left) off the chain, chain FMNMX + FMNMX (ptxas may fuse);
      // VAR 6: as 5 with m by an integer min on the (non-negative) float bits, which
      // ptxas cannot fuse into the chain's FMNMX
      float upv = SHF ? __shfl_up_sync(0xffffffffu, c[R - 1], 1) : c[R - 1];
      float up = lane == 0 ? e.w : upv, dg = diag_f;
      diag_f = up;
      const uint64_t q2x = pack(e.x, e.x), q2y = pack(e.y, e.y), qq2 = pack(e.z, e.z);
      float m[R];
      if (VAR != 4) {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const float left = c[r], above = r ? c[r - 1] : dg;
          if (VAR == 6) m[r] = __int_as_float(min(__float_as_int(above), __float_as_int(left)));
          else m[r] = fminf(above, left);
        }
      }
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        uint64_t acc;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(pack(pq[r], pq[r + 1])), "l"(qq2));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pack(px[r], px[r + 1])), "l"(q2x));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pack(py[r], py[r + 1])), "l"(q2y));
        const float d0 = __uint_as_float((uint32_t)acc), d1 = __uint_as_float((uint32_t)(acc >> 32));
        float n0, n1;
        if (VAR == 4) {
          n0 = fmaxf(fminf(fminf(up, dg), c[r]), d0);
          n1 = fmaxf(fminf(fminf(n0, c[r]), c[r + 1]), d1);
        } else {
          n0 = fmaxf(fminf(up, m[r]), d0);
          n1 = fmaxf(fminf(n0, m[r + 1]), d1);
        }
        dg = c[r + 1]; c[r] = n0; c[r + 1] = n1; up = n1;
      }
    } else if (VAR == 7) {
      // the c2 cell, TWO columns per step (strip.cuh Pipe2 layout): the second
      // column's chain trails the first by one row, so the two chains interleave
      const float4 e1 = ring[w][(g + 64) & 127];
      const float upv0 = SHF ? __shfl_up_sync(0xffffffffu, b0_f, 1) : b0_f;
      const float upv1 = SHF ? __shfl_up_sync(0xffffffffu, c[R - 1], 1) : c[R - 1];
      const float up0 = lane == 0 ? e.w : upv0, up1 = lane == 0 ? e1.w : upv1;
      float dist0[R], dist1[R];
      const uint64_t q2x = pack(e.x, e.x), q2y = pack(e.y, e.y), qq2 = pack(e.z, e.z);
      const uint64_t r2x = pack(e1.x, e1.x), r2y = pack(e1.y, e1.y), rq2 = pack(e1.z, e1.z);
#pragma unroll
      for (int r = 0; r < R; r += 2) {
        uint64_t acc, acc1;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(pack(pq[r], pq[r + 1])), "l"(qq2));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pack(px[r], px[r + 1])), "l"(q2x));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pack(py[r], py[r + 1])), "l"(q2y));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(acc1) : "l"(pack(pq[r], pq[r + 1])), "l"(rq2));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc1) : "l"(pack(px[r], px[r + 1])), "l"(r2x));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc1) : "l"(pack(py[r], py[r + 1])), "l"(r2y));
        dist0[r] = __uint_as_float((uint32_t)acc); dist0[r + 1] = __uint_as_float((uint32_t)(acc >> 32));
        dist1[r] = __uint_as_float((uint32_t)acc1); dist1[r + 1] = __uint_as_float((uint32_t)(acc1 >> 32));
      }
      float u = up0, dg = diag_f;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const float nv = fmaxf(fminf(fminf(u, dg), c[r]), dist0[r]);
        dg = c[r]; c[r] = nv; u = nv;
      }
      b0_f = c[R - 1];
      u = up1; dg = up0;
#pragma unroll
      for (int r = 0; r < R; r++) {
        const float nv = fmaxf(fminf(fminf(u, dg), c[r]), dist1[r]);
        dg = c[r]; c[r] = nv; u = nv;
      }
      diag_f = up1;
    } else {
      int m2x = __float_as_int(e.x), m2y = __float_as_int(e.y), qq = __float_as_int(e.z);
      int upv = SHF ? __shfl_up_sync(0xffffffffu, ic[R - 1], 1) : ic[R - 1];
      int up = lane == 0 ? __float_as_int(e.w) : upv, dg = diag_i;
      diag_i = up;
#pragma unroll
      for (int r = 0; r < R; r++) {
        int d = ipp[r] + qq + ipx[r] * m2x + ipy[r] * m2y;
        int m = __vimin3_s32(up, dg, ic[r]);
        int nv = max(m, d);
        dg = ic[r]; ic[r] = nv; up = nv;
      }
    }
  }
  long long t1 = clock64();
  float sacc = 0.f;
#pragma unroll
  for (int r = 0; r < R; r++) sacc += c[r] + (float)ic[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sacc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static int nsm;

static const char* g_only = nullptr;  // argv[1]: run only the tests whose name contains it

template <typename K>
static int run(const char* name, K kern, int blocks_per_sm, int threads, int iters,
               double instr_per_thread_iter, const char* unit) {
  if (g_only && !strstr(name, g_only)) return 0;
  int blocks = nsm * blocks_per_sm;
  float* out; long long* cyc;
  CK(cudaMalloc(&out, sizeof(float) * blocks * threads));
  CK(cudaMalloc(&cyc, sizeof(long long) * blocks));
  kern<<<blocks, threads>>>(out, cyc, iters / 10);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, cyc, iters);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[blocks];
  CK(cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
  double mx = 0, sum = 0;
  for (int i = 0; i < blocks; i++) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
  // per SM: blocks_per_sm blocks ran concurrently for ~max cycles
  double warps_per_sm = blocks_per_sm * threads / 32.0;
  double per_clk = warps_per_sm * iters * instr_per_thread_iter / mx;
  printf("{\"test\": \"%s\", \"per_clk_per_sm\": %.3f, \"unit\": \"%s\", \"warps_per_sm\": %.0f, "
         "\"max_cycles\": %.0f, \"mean_cycles\": %.0f, \"ms\": %.3f, \"clk_mhz_est\": %.0f}\n",
         name, per_clk, unit, warps_per_sm, mx, sum / blocks, ms, mx / (ms * 1e3));
  delete[] h;
  cudaFree(out); cudaFree(cyc);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) g_only = argv[1];
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", prop.name, nsm, prop.major, prop.minor);
  const int IT = 20000;
  const double per = NCHAIN * UNROLL;
  const char* names[] = {"FFMA", "FADD", "FMUL", "FMNMX", "FMNMX3", "IADD3", "IMAD", "VIMNMX",
                         "VIMNMX3", "FADD2", "FFMA2", "FMUL2", "FMNMX(max)", "SHFL.UP"};
  run(names[0], op_kernel<0>, 4, 256, IT, per, "warp-instr");
  run(names[1], op_kernel<1>, 4, 256, IT, per, "warp-instr");
  run(names[2], op_kernel<2>, 4, 256, IT, per, "warp-instr");
  run(names[3], op_kernel<3>, 4, 256, IT, per, "warp-instr");
  run(names[4], op_kernel<4>, 4, 256, IT, per, "warp-instr(pairs of min fused?)");
  run(names[5], op_kernel<5>, 4, 256, IT, per, "warp-instr");
  run(names[6], op_kernel<6>, 4, 256, IT, per, "warp-instr");
  run(names[7], op_kernel<7>, 4, 256, IT, per, "warp-instr");
  run(names[8], op_kernel<8>, 4, 256, IT, per, "warp-instr");
  run(names[9], op_kernel<9>, 4, 256, IT, per, "warp-instr");
  run(names[10], op_kernel<10>, 4, 256, IT, per, "warp-instr");
  run(names[11], op_kernel<11>, 4, 256, IT, per, "warp-instr");
  run(names[12], op_kernel<12>, 4, 256, IT, per, "warp-instr");
  run(names[13], op_kernel<13>, 4, 256, IT / 4, per, "warp-instr");
  // mixed streams (warp-instructions of all kinds per clock per SM)
  run("mix_FFMA2+FMNMX3", mix_kernel<0>, 4, 256, IT, per * 2, "warp-instr");
  run("mix_FFMA2+FMNMX", mix_kernel<1>, 4, 256, IT, per * 2, "warp-instr");
  run("mix_FFMA+FMNMX", mix_kernel<2>, 4, 256, IT, per * 2, "warp-instr");
  run("mix_cell_f32_FADD2+FFMA2+FMNMX3+FMNMX", mix_kernel<3>, 4, 256, IT, per * 4, "warp-instr");
  run("mix_cell_xsq_2cells_FADD2+2FFMA2+2FMNMX3+2FMNMX", mix_kernel<4>, 4, 256, IT, per * 7, "warp-instr");
  run("mix_FMNMX3+FMNMX", mix_kernel<5>, 4, 256, IT, per * 2, "warp-instr");
  run("mix_FFMA2+IADD3", mix_kernel<6>, 4, 256, IT, per * 2, "warp-instr");
  run("mix_FMNMX3+IADD3", mix_kernel<7>, 4, 256, IT, per * 2, "warp-instr");
  // the same mixes reported as cells per clock per SM (32 lanes x cells per unit)
  run("mixcells_f32_d2_sq", mix_kernel<3>, 4, 256, IT, per * 32, "cells");
  run("mixcells_xsq_d2", mix_kernel<4>, 4, 256, IT, per * 64, "cells");
  run("mixcells_f32_d3_sq", mix_kernel<8>, 4, 256, IT, per * 64, "cells");
  run("mixcells_f32_d2_l1", mix_kernel<9>, 4, 256, IT, per * 64, "cells");
  run("mixcells_f32_d2_linf", mix_kernel<10>, 4, 256, IT, per * 64, "cells");
  run("mixcells_xsq_d2_w16", mix_kernel<4>, 2, 256, IT, per * 64, "cells");
  run("mixcells_f32_d2_sq_w16", mix_kernel<3>, 2, 256, IT, per * 32, "cells");
  // cells per clock per SM: per thread-step = R cells; lanes x warps
  const int ST = 4000;
  int wl[3] = {8, 16, 32};
  for (int wi = 0; wi < 3; wi++) {
    int bps = wl[wi] / 4;  // 128-thread blocks
    char nm[96];
#define CELL2(V, RR, S, TAG) snprintf(nm, 96, "cell_%s_R%d_shfl%d_w%d", TAG, RR, S, wl[wi]); \
    run(nm, cell_kernel<V, RR, S>, bps, 128, ST, 2 * RR * 32.0, "cells");
#define CELL(V, RR, S, TAG) snprintf(nm, 96, "cell_%s_R%d_shfl%d_w%d", TAG, RR, S, wl[wi]); \
    run(nm, cell_kernel<V, RR, S>, bps, 128, ST, RR * 32.0, "cells");
    CELL(0, 16, 0, "f32_scalar") CELL(0, 16, 1, "f32_scalar") CELL(0, 8, 1, "f32_scalar")
    CELL(1, 16, 0, "f32_packed") CELL(1, 16, 1, "f32_packed") CELL(1, 8, 1, "f32_packed")
    CELL(2, 16, 0, "i32_std") CELL(2, 16, 1, "i32_std") CELL(2, 8, 1, "i32_std")
    CELL(3, 16, 0, "i32_expand") CELL(3, 16, 1, "i32_expand") CELL(3, 8, 1, "i32_expand")
    CELL(3, 4, 1, "i32_expand") CELL(0, 4, 1, "f32_scalar")
    CELL(4, 12, 1, "xsq_fmnmx3") CELL(5, 12, 1, "xsq_split") CELL(6, 12, 1, "xsq_split_int")
    CELL(4, 16, 1, "xsq_fmnmx3") CELL(5, 16, 1, "xsq_split") CELL(6, 16, 1, "xsq_split_int")
    CELL(4, 8, 1, "xsq_fmnmx3") CELL(5, 8, 1, "xsq_split") CELL(6, 8, 1, "xsq_split_int")
    CELL2(7, 12, 1, "xsq_2col") CELL2(7, 16, 1, "xsq_2col") CELL2(7, 8, 1, "xsq_2col")
  }
  return 0;
}
