// FFMA vs FFMA2 (fma.rn.f32x2, sm_100a) and FADD vs FADD2 issue rates: 32 warps per SM,
// 8 independent accumulator chains per thread, time per warp instruction from clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ffma2_rate scripts/ffma2_rate.cu
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2(float a, float b) { return (u64)__float_as_uint(a) | ((u64)__float_as_uint(b) << 32); }
template <int MODE>
__global__ void k(float *out, long long *cyc, int n, float m0) {
  // per-thread multiplier (a plain register, not a uniform / constant operand:
  // FFMA with a uniform or immediate operand issues at twice the 3-register rate)
  const float m = m0 + threadIdx.x * 1e-9f;
  float a[16];
  u64 p[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = f2(a[2 * i], a[2 * i + 1]);
  const u64 mm = f2(m, m * 1.5f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    if (MODE == 0) {  // 16 FFMA
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], m, 0.5f * m);
    } else if (MODE == 1) {  // 8 FFMA2 (16 fp32 FMAs)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(p[i]) : "l"(mm));
    } else if (MODE == 2) {  // 16 FADD
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = __fadd_rn(a[i], m);
    } else {  // 8 FADD2
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(mm));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float((uint32_t)p[i]) + __uint_as_float((uint32_t)(p[i] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float *o; long long *c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  const int n = 4096;
  const char *nm[4] = {"FFMA  (16/iter)", "FFMA2 (8/iter, 16 fma)", "FADD  (16/iter)", "FADD2 (8/iter, 16 add)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 1024>>>(o, c, n, 0.999f);
      if (mode == 1) k<1><<<148, 1024>>>(o, c, n, 0.999f);
      if (mode == 2) k<2><<<148, 1024>>>(o, c, n, 0.999f);
      if (mode == 3) k<3><<<148, 1024>>>(o, c, n, 0.999f);
    }
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const int ninstr = (mode & 1) ? 8 : 16;
    // 32 warps per SM over 4 SMSPs: 8 warps per SMSP
    const double per = (double)h / ((double)n * ninstr * 8);
    printf("%-24s cycles per warp-instr per SMSP = %.3f ; fp32 ops/cycle/SM = %.1f  (%s)\n", nm[mode], per,
           4 * 32.0 * ((mode & 1) ? 2 : 1) / per, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
