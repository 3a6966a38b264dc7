// Dependent-chain latency of the SASS ops on the DP critical path (one warp,
// one chain): FMNMX3, FMNMX, the FMNMX3 -> FMNMX pair of the Fréchet cell,
// FSEL, SHFL.UP, LDS.  Reports SM cycles per dependent op (clock64 in-kernel).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency latency.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256;  // ops per timed chain (unrolled)

template <int OP>
__global__ void lat_kernel(float* out, long long* cyc, float y, float z, int iters) {
  __shared__ float sm[64];
  const int lane = threadIdx.x & 31;
  sm[lane] = (float)lane;
  sm[32 + lane] = (float)lane;
  __syncwarp();
  float a = threadIdx.x * 1e-3f;
  int ia = lane;
  long long best = 1LL << 60;
  for (int it = 0; it < iters; it++) {
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < N; k++) {
      if (OP == 0) {  // FMNMX3 chain
        float t;
        asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(a), "f"(y), "f"(z));
        a = t;
      } else if (OP == 1) {  // FMNMX chain
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(y));
      } else if (OP == 2) {  // cell: FMNMX3 then FMNMX (2 ops per k)
        float t;
        asm volatile("min.f32 %0, %1, %2;\n\tmin.f32 %0, %0, %3;" : "=f"(t) : "f"(a), "f"(y), "f"(z));
        asm volatile("max.f32 %0, %0, %1;" : "+f"(t) : "f"(y));
        a = t;
      } else if (OP == 3) {  // SHFL.UP chain
        a = __shfl_up_sync(0xffffffffu, a, 1);
      } else if (OP == 4) {  // LDS chain (address depends on the previous load)
        ia = __float_as_int(sm[ia & 63]) & 63;
      } else if (OP == 5) {  // SHFL + FSEL (lane 0 selects its own) as in the step
        float u = __shfl_up_sync(0xffffffffu, a, 1);
        a = (lane == 0) ? y : u;
      } else if (OP == 6) {  // FADD chain
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a) : "f"(y));
      }
    }
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
  }
  out[threadIdx.x] = a + (float)ia;
  if (threadIdx.x == 0) cyc[0] = best;
}

template <int OP>
static void run(const char* name, int ops_per_k) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 8);
  lat_kernel<OP><<<1, 32>>>(out, cyc, 1.0001f, 0.9999f, 20);
  cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"test\": \"lat_%s\", \"cycles_per_op\": %.2f}\n", name, (double)h / (N * ops_per_k));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("FMNMX3", 1);
  run<1>("FMNMX", 1);
  run<2>("FMNMX3+FMNMX_pair", 1);
  run<3>("SHFL.UP", 1);
  run<4>("LDS", 1);
  run<5>("SHFL.UP+FSEL", 1);
  run<6>("FADD", 1);
  return 0;
}
