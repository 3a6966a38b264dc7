// Cycles per warp step of the library's DP step functions (strip.cuh) for ONE
// warp alone on an SM: the latency-bound floor that the long-pair pipeline and
// lightly loaded SMs run at.  Variants isolate the shuffle, the ring loads and
// the two-column form.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I ../../paper_2404_05708_b200/csrc -I ../../include -o step step.cu
#include <cstdio>

#include "strip.cuh"

using namespace ffd;
constexpr int KIND = K_SQ, D = 2;
using C = SCfg<float, KIND, D, false>;

// VAR 0: warp_step2 (load + compute), 1: step2_compute_pf (pipelined loads),
// 2: warp_step (one column), 3: step2 compute without ring loads (element reused),
// 4: Pipe2 (the long kernel's step), 5–8: Pipe2 + lane 31's per-step 16-byte link
// store as the long kernel issues it: 5 st.relaxed.gpu generic -> smem,
// 6 st.shared (explicit), 7 st.relaxed.gpu -> global, 8 st.relaxed.gpu generic -> smem
// of ANOTHER buffer with the ring loads unchanged (same as 5, different slot stride)
__device__ __forceinline__ void st_gen_v4(void* p, float v0, float v1, unsigned tag, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t@q st.relaxed.gpu.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
      "r"(__float_as_uint(v0)), "r"(tag), "r"(__float_as_uint(v1)), "r"(tag + 1u), "r"(pred));
}
__device__ __forceinline__ void st_sh_v4(unsigned a, float v0, float v1, unsigned tag, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %5, 0;\n\t@q st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"r"(a),
      "r"(__float_as_uint(v0)), "r"(tag), "r"(__float_as_uint(v1)), "r"(tag + 1u), "r"(pred));
}

template <int VAR, int R>
__global__ void step_kernel(float* out, long long* cyc, int steps, uint4* gbuf) {
  __shared__ uint4 ring[kRing * C::EW];
  __shared__ uint4 link[512];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kRing * C::EW; i += 32)
    ring[i] = make_uint4(__float_as_uint(i * 0.1f), __float_as_uint(1.f - i * 0.01f), 0u,
                         __float_as_uint(1e30f));
  __syncwarp();
  float x[C::NS][R], c[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    x[0][r] = lane * 0.3f + r;
    x[1][r] = r * 0.2f - lane;
    c[r] = 1e30f;
  }
  float diag = 1e30f, b0 = 1e30f;
  Elem2<float, KIND, D, false> el;
  load_elem2<float, KIND, D, false>(el, ring, 0);
  Pipe2<float, KIND, D, R, false> pipe;
  pipe.prime(x, ring, -lane);
  __syncwarp();
  long long t0 = clock64();
  for (int g = 0; g < steps; g++) {
    if (VAR == 0) warp_step2<float, KIND, D, R, false>(c, diag, b0, x, ring, g - lane, lane);
    if (VAR == 1) step2_compute_pf<float, KIND, D, R, false>(c, diag, b0, x, el, lane, ring, g + 1 - lane);
    if (VAR == 2) warp_step<float, KIND, D, R, false>(c, diag, x, ring, g - lane, lane);
    if (VAR == 3) step2_compute<float, KIND, D, R, false>(c, diag, b0, x, el, lane);
    if (VAR == 4) pipe.step(c, diag, b0, x, ring, g - lane, lane);
    if (VAR >= 5) {
      pipe.step(c, diag, b0, x, ring, g - lane, lane);
      const int pown = lane == 31;
      if (VAR == 5 || VAR == 8) st_gen_v4(&link[g & 511], b0, c[R - 1], 2u * g + 1u, pown);
      if (VAR == 6) st_sh_v4((unsigned)__cvta_generic_to_shared(&link[g & 511]), b0, c[R - 1], 2u * g + 1u, pown);
      if (VAR == 7) st_gen_v4(&gbuf[g & 511], b0, c[R - 1], 2u * g + 1u, pown);
    }
  }
  long long t1 = clock64();
  float s = diag + b0;
#pragma unroll
  for (int r = 0; r < R; r++) s += c[r];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int VAR, int R>
static void run(const char* name) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  uint4* gbuf;
  cudaMalloc(&gbuf, 512 * 16);
  const int steps = 20000;
  step_kernel<VAR, R><<<1, 32>>>(out, cyc, steps / 10, gbuf);
  step_kernel<VAR, R><<<1, 32>>>(out, cyc, steps, gbuf);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"test\": \"step_%s_R%d\", \"cycles_per_step\": %.1f}\n", name, R, (double)h / steps);
  cudaFree(out);
  cudaFree(cyc);
  cudaFree(gbuf);
}

int main() {
  run<4, 4>("pipe2");
  run<5, 4>("pipe2+st_generic_smem");
  run<6, 4>("pipe2+st_shared");
  run<7, 4>("pipe2+st_global");
  run<4, 7>("pipe2");
  run<5, 7>("pipe2+st_generic_smem");
  run<6, 7>("pipe2+st_shared");
  run<7, 7>("pipe2+st_global");
  run<0, 1>("warp_step2");
  run<0, 4>("warp_step2");
  run<0, 8>("warp_step2");
  run<1, 4>("step2_pf");
  run<1, 8>("step2_pf");
  run<2, 4>("warp_step_1col");
  run<2, 8>("warp_step_1col");
  run<3, 4>("step2_noload");
  run<3, 8>("step2_noload");
  run<4, 1>("pipe2");
  run<4, 4>("pipe2");
  run<4, 7>("pipe2");
  run<4, 8>("pipe2");
  run<4, 16>("pipe2");
  run<0, 16>("warp_step2");
  return 0;
}
