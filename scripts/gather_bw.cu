// Microbenchmark: random 256-B row gathers (the attention's access pattern)
// with cp.async into shared memory, vs CTA count / warps / stages.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gather_bw scripts/gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
template <int N> __device__ __forceinline__ void wait_g() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// each warp: rows [w*per, (w+1)*per) of its CTA's list; batch of 8 rows (K and V = 16 rows of 256 B)
template <int STAGES>
__global__ void gather(const uint8_t *kp, const uint8_t *vp, const uint32_t *rows, int rows_per_cta, int warps,
                       unsigned long long *sink, int stride) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w >= warps) return;
  const uint32_t *lst = rows + (size_t)blockIdx.x * rows_per_cta;
  const int per = rows_per_cta / warps;
  const int lo = w * per;
  const int nb = per / 8;
  uint8_t *ring = sm + (size_t)w * STAGES * 4096;
  auto issue = [&](int j) {
    uint8_t *st = ring + (j % STAGES) * 4096;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int q = lane + 32 * m, rr = q >> 4, ch = q & 15;
      const size_t off = (size_t)lst[lo + j * 8 + rr] * stride + ch * 16;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(st + rr * 256 + ch * 16);
      cp16(dst, kp + off);
      cp16(dst + 2048, vp + off);
    }
  };
  for (int s = 0; s < STAGES - 1; ++s) { if (s < nb) issue(s); commit(); }
  unsigned long long acc = 0;
  for (int j = 0; j < nb; ++j) {
    if (j + STAGES - 1 < nb) issue(j + STAGES - 1);
    commit();
    wait_g<STAGES - 1>();
    __syncwarp();
    acc += *(const uint32_t *)(ring + (j % STAGES) * 4096 + lane * 128);
    __syncwarp();
  }
  if (acc == 0x123456789ull) *sink = acc;
}

__global__ void flush_read(const uint4 *p, size_t n, unsigned long long *sink) {
  uint4 a = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    a.x ^= v.x; a.y ^= v.y;
  }
  if (a.x == 0x12345 && a.y == 0x777) *sink = a.x;
}

int main() {
  const size_t units = 128, k = 2048, S = 32768, P = 16, Hkv = 8;
  const size_t pages = units / Hkv * (S / P);   // B * S/P pages, each [Hkv][P][256 B]
  const size_t pool_rows = pages * Hkv * P;
  uint8_t *kp, *vp; uint32_t *rows; unsigned long long *sink;
  // INTERLEAVE=1: K and V rows of a token adjacent (one 512-B row), else two pools of 256-B rows
  const int inter = getenv("INTERLEAVE") && atoi(getenv("INTERLEAVE"));
  const int stride = inter ? 512 : 256;
  if (inter) {
    cudaMalloc(&kp, pool_rows * 512); cudaMemset(kp, 1, pool_rows * 512); vp = kp + 256;
  } else {
    cudaMalloc(&kp, pool_rows * 256); cudaMalloc(&vp, pool_rows * 256);
    cudaMemset(kp, 1, pool_rows * 256); cudaMemset(vp, 1, pool_rows * 256);
  }
  printf("layout: %s\n", inter ? "interleaved K|V 512-B rows" : "separate K and V pools, 256-B rows");
  cudaMalloc(&sink, 8);
  std::mt19937_64 g(1);
  // per unit: k random distinct tokens, random page permutation -> pool rows
  std::vector<uint32_t> hrows(units * k);
  std::vector<uint32_t> perm(S / P);
  for (size_t u = 0; u < units; ++u) {
    size_t b = u / Hkv, h = u % Hkv;
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = b * (S / P) + i;
    std::shuffle(perm.begin(), perm.end(), g);
    std::vector<uint32_t> toks(S); for (size_t t = 0; t < S; ++t) toks[t] = t;
    std::shuffle(toks.begin(), toks.end(), g);
    std::sort(toks.begin(), toks.begin() + k);
    for (size_t i = 0; i < k; ++i) { size_t t = toks[i]; hrows[u * k + i] = (perm[t / P] * Hkv + h) * P + t % P; }
  }
  cudaMalloc(&rows, hrows.size() * 4);
  cudaMemcpy(rows, hrows.data(), hrows.size() * 4, cudaMemcpyHostToDevice);
  // flush buffer
  uint8_t *fl; cudaMalloc(&fl, 512 << 20); cudaMemset(fl, 3, 512 << 20); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](int ctas, int warps, int stages) {
    const int rpc = (int)(units * k / ctas);
    size_t smem = (size_t)warps * stages * 4096;
    auto kern = stages == 2 ? gather<2> : stages == 3 ? gather<3> : gather<4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      flush_read<<<592, 512>>>((const uint4 *)fl, (512u << 20) / 16, sink);
      cudaEventRecord(e0);
      kern<<<ctas, warps * 32, smem>>>(kp, vp, rows, rpc, warps, sink, stride);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double bytes = (double)units * k * 512;
    printf("ctas %4d warps %2d stages %d smem %6zu KB: %7.2f us  %6.0f GB/s  (%s)\n", ctas, warps, stages, smem / 1024,
           best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  run(128, 16, 2); run(128, 16, 3); run(128, 8, 4); run(128, 24, 2);
  run(256, 16, 2); run(256, 8, 3); run(512, 8, 2); run(1024, 8, 2); run(2048, 4, 2);
  run(148 * 2, 16, 2);
  return 0;
}
