// Microbenchmark: the attention's row gathers (k random 256-B K rows + the
// same V rows per unit, through a random page order) at steady state
// (>= 1 GiB per launch), three ways of moving a row into shared memory:
//   cpasync : 16-B cp.async chunks spread over the warp (what decode_kernel does)
//   bulk    : one 256-B cp.async.bulk per row (lanes 0..15 of the warp each
//             issue one), completion on a per-stage mbarrier (complete_tx)
//   gather4 : cp.async.bulk.tensor.2d ... tile::gather4 over the pool viewed
//             as a 2-D [rows, 128] bf16 tensor map: 4 rows per instruction
//             (lanes 0..3 issue K rows 0-3, K 4-7, V 0-3, V 4-7)
// Every mode checks the gathered bytes (each 16-B chunk of a pool row holds
// its row id) and reports mismatches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_gather_bw scripts/tma_gather_bw.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

enum Mode { CPASYNC = 0, BULK = 1, GATHER4 = 2 };

__device__ __forceinline__ uint32_t sm32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void wait_g() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_row(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap *tm, int col, int r0, int r1, int r2, int r3,
                                        uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// each warp: rows [w*per, (w+1)*per) of its CTA's unit; batches of 8 tokens
// (8 K rows then 8 V rows = 4 KiB per stage)
template <int MODE, int STAGES>
__global__ void gather(const uint8_t *kp, const uint8_t *vp, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const uint32_t *rows, int k, int units, int warps,
                       unsigned long long *bad) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm);  // [warps][STAGES]
  uint8_t *ring0 = sm + 1024;
  if (threadIdx.x < warps * STAGES) mbar_init(sm32(bars + threadIdx.x), 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  if (w >= warps) return;
  unsigned long long nbad = 0;
  uint32_t phase[STAGES] = {};
  for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const uint32_t *lst = rows + (size_t)unit * k;
    const int per = k / warps, lo = w * per, nb = per / 8;
    uint8_t *ring = ring0 + (size_t)w * STAGES * 4096;
    auto issue = [&](int j) {
      const int s = j % STAGES;
      uint8_t *st = ring + s * 4096;
      const uint32_t bar = sm32(bars + w * STAGES + s);
      const uint32_t *rl = lst + lo + j * 8;
      if constexpr (MODE == CPASYNC) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const int q = lane + 32 * m, rr = q >> 4, ch = q & 15;
          const size_t off = (size_t)rl[rr] * 256 + ch * 16;
          const uint32_t dst = sm32(st + rr * 256 + ch * 16);
          cp16(dst, kp + off);
          cp16(dst + 2048, vp + off);
        }
      } else if constexpr (MODE == BULK) {
        if (lane == 0) mbar_expect(bar, 4096);
        __syncwarp();
        if (lane < 16) {
          const int rr = lane & 7;
          bulk_row(sm32(st + lane * 256), (lane < 8 ? kp : vp) + (size_t)rl[rr] * 256, 256, bar);
        }
      } else {
        if (lane == 0) mbar_expect(bar, 4096);
        __syncwarp();
        if (lane < 4) {
          const int h = (lane & 1) * 4;
          gather4(sm32(st + lane * 1024), lane < 2 ? &tk : &tv, 0, (int)rl[h], (int)rl[h + 1], (int)rl[h + 2],
                  (int)rl[h + 3], bar);
        }
      }
    };
    auto wait = [&](int j) {
      if constexpr (MODE == CPASYNC) {
        wait_g<STAGES - 1>();
      } else {
        const int s = j % STAGES;
        mbar_wait(sm32(bars + w * STAGES + s), phase[s]);
        phase[s] ^= 1u;
      }
      __syncwarp();
    };
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < nb) issue(s);
      if (MODE == CPASYNC) commit();
    }
    for (int j = 0; j < nb; ++j) {
      if (j + STAGES - 1 < nb) issue(j + STAGES - 1);
      if (MODE == CPASYNC) commit();
      wait(j);
      // check: chunk (lane & 15) of row (lane >> 4) of the K half and of the V half
      const uint8_t *st = ring + (j % STAGES) * 4096;
      const int rr = lane >> 4;
      const uint32_t want = lst[lo + j * 8 + rr];
      for (int rh = rr; rh < 8; rh += 2) {
        const uint32_t wv = lst[lo + j * 8 + rh];
        const uint32_t gk = *reinterpret_cast<const uint32_t *>(st + rh * 256 + (lane & 15) * 16);
        const uint32_t gv = *reinterpret_cast<const uint32_t *>(st + 2048 + rh * 256 + (lane & 15) * 16);
        nbad += (gk != wv) + (gv != (wv ^ 0x80000000u));
      }
      (void)want;
      __syncwarp();  // stage read before it is refilled
    }
    if (MODE == CPASYNC) wait_g<0>();
  }
  if (nbad) atomicAdd(bad, nbad);
}

__global__ void fill(uint32_t *p, size_t rows, uint32_t x) {  // every 16-B chunk of row i starts with i ^ x
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows * 16; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4 *>(p)[i] = make_uint4((uint32_t)(i >> 4) ^ x, 0, 0, 0);
}
__global__ void flush_read(const uint4 *p, size_t n, unsigned long long *sink) {
  uint4 a = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    a.x ^= v.x;
    a.y ^= v.y;
  }
  if (a.x == 0x12345 && a.y == 0x777) *sink = a.x;
}

int main(int argc, char **argv) {
  const size_t units = argc > 1 ? atoi(argv[1]) : 1024, k = 2048, S = 32768, P = 16, Hkv = 8;
  const size_t B = (units + Hkv - 1) / Hkv, pages = B * (S / P);
  const size_t pool_rows = pages * Hkv * P;
  uint8_t *kp, *vp;
  uint32_t *rows;
  unsigned long long *bad;
  if (cudaMalloc(&kp, pool_rows * 256) || cudaMalloc(&vp, pool_rows * 256)) {
    printf("alloc failed\n");
    return 1;
  }
  fill<<<4096, 256>>>((uint32_t *)kp, pool_rows, 0u);
  fill<<<4096, 256>>>((uint32_t *)vp, pool_rows, 0x80000000u);
  cudaMalloc(&bad, 8);
  std::mt19937_64 g(1);
  const int sorted = getenv("SORTED") && atoi(getenv("SORTED"));
  std::vector<uint32_t> hrows(units * k), perm(S / P), toks(S);
  for (size_t u = 0; u < units; ++u) {
    const size_t b = u / Hkv, h = u % Hkv;
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = (uint32_t)(b * (S / P) + i);
    std::shuffle(perm.begin(), perm.end(), g);
    for (size_t t = 0; t < S; ++t) toks[t] = (uint32_t)t;
    std::shuffle(toks.begin(), toks.end(), g);
    std::sort(toks.begin(), toks.begin() + k);
    for (size_t i = 0; i < k; ++i) {
      const size_t t = toks[i];
      hrows[u * k + i] = (uint32_t)((perm[t / P] * Hkv + h) * P + t % P);
    }
    if (sorted) std::sort(hrows.begin() + u * k, hrows.begin() + (u + 1) * k);
  }
  cudaMalloc(&rows, hrows.size() * 4);
  cudaMemcpy(rows, hrows.data(), hrows.size() * 4, cudaMemcpyHostToDevice);
  uint8_t *fl;
  cudaMalloc(&fl, 512 << 20);
  cudaMemset(fl, 3, 512 << 20);
  // tensor maps: the pools as 2-D [pool_rows, 128] 16-bit tensors, box {128, 1}
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  CUtensorMap tk, tv;
  const cuuint64_t dims[2] = {128, (cuuint64_t)pool_rows};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {128, 1}, es[2] = {1, 1};
  CUresult r1 = enc(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kp, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, vp, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("units %zu (%.2f GiB gathered per launch), rows %s, tensor maps: %d %d\n", units,
         units * k * 512.0 / (1 << 30), sorted ? "sorted by address" : "in token order", (int)r1, (int)r2);
  cudaDeviceSynchronize();
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *names[3] = {"cp.async 16B", "bulk per row", "tma gather4 "};
  auto run = [&](int mode, int ctas, int warps, int stages) {
    const size_t smem = 1024 + (size_t)warps * stages * 4096;
    using K = void (*)(const uint8_t *, const uint8_t *, const CUtensorMap, const CUtensorMap, const uint32_t *, int, int,
                       int, unsigned long long *);
    K tab[3][3] = {{gather<0, 2>, gather<0, 3>, gather<0, 4>},
                   {gather<1, 2>, gather<1, 3>, gather<1, 4>},
                   {gather<2, 2>, gather<2, 3>, gather<2, 4>}};
    K kern = tab[mode][stages - 2];
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaMemset(bad, 0, 8);
    float best = 1e9, sum = 0;
    const int reps = 5;
    for (int it = 0; it < reps; ++it) {
      flush_read<<<sms * 4, 512>>>((const uint4 *)fl, (512u << 20) / 16, bad + 0);
      cudaEventRecord(e0);
      kern<<<ctas, warps * 32, smem>>>(kp, vp, tk, tv, rows, (int)k, (int)units, warps, bad);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
      sum += ms;
    }
    unsigned long long nb = 0;
    cudaMemcpy(&nb, bad, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)units * k * 512;
    printf("%s ctas %5d warps %2d stages %d smem %3zu KB: best %8.2f us %6.0f GB/s  mean %6.0f GB/s  bad %llu (%s)\n",
           names[mode], ctas, warps, stages, smem / 1024, best * 1e3, bytes / best / 1e6, bytes / (sum / reps) / 1e6,
           nb, cudaGetErrorString(cudaGetLastError()));
  };
  if (getenv("GATHER_CTAS")) {  // e.g. GATHER_CTAS=128: the c3 kernel's grid (units on 128 of the SMs)
    const int c = atoi(getenv("GATHER_CTAS"));
    run(0, c, 16, 2);
    run(0, c, 16, 3);
    run(0, sms, 16, 2);
    return 0;
  }
  for (int mode = 0; mode < 3; ++mode) {
    run(mode, sms, 16, 2);
    run(mode, sms, 16, 3);
    run(mode, sms, 16, 4);
    run(mode, sms, 32, 2);
    run(mode, sms * 2, 16, 2);
    run(mode, sms * 2, 8, 4);
    run(mode, (int)units, 16, 2);
  }
  return 0;
}
