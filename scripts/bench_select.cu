// Isolated timing of the selection core (diagnostics): synthetic candidates
// staged in smem, 128 CTAs x 512 threads, like the last-arriver phase.
#include "../paper_2408_07092_b200/csrc/select.cu"
#include <cstdio>
#include <vector>

using namespace ds;

__global__ void __launch_bounds__(512) k_sel(int T, int keff, int32_t *idx, int32_t *rid, CacheView c, int reps,
                                             long long *cyc) {
  extern __shared__ __align__(16) uint32_t dyn[];
  __shared__ __align__(16) uint32_t bins[kBins];
  __shared__ uint32_t warp_tot[17], state[4];
  uint2 *stage = reinterpret_cast<uint2 *>(dyn);
  for (int i = threadIdx.x; i < T + 128; i += 512) {
    uint32_t x = (uint32_t)(i + 1) * 2654435761u ^ (blockIdx.x * 40503u);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    stage[i] = make_uint2(0x80000000u | (x >> 1), (uint32_t)i);
  }
  __syncthreads();
  const SelScratch scr{bins, warp_tot, state};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    select_core_staged<512>(stage, T, (uint32_t)keff, scr, idx + blockIdx.x * keff, rid + blockIdx.x * keff, c, 0, 0);
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int32_t *idx, *rid, *bt;
  long long *cyc;
  cudaMalloc(&idx, 128 * 4096 * 4);
  cudaMalloc(&rid, 128 * 4096 * 4);
  cudaMalloc(&bt, 1 << 20);
  cudaMemset(bt, 0, 1 << 20);
  cudaMalloc(&cyc, 128 * 8);
  CacheView c{};
  c.P = 16; c.Hkv = 8; c.maxp = 4096; c.block_table = bt;
  cudaFuncSetAttribute(k_sel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int T : {2048, 4600, 9000}) {
    for (int reps : {1, 5}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      k_sel<<<128, 512, (T + 256) * 8>>>(T, 2048 < T ? 2048 : T / 2, idx, rid, c, reps, cyc);
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) k_sel<<<128, 512, (T + 256) * 8>>>(T, 2048 < T ? 2048 : T / 2, idx, rid, c, reps, cyc);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      std::vector<long long> h(128);
      cudaMemcpy(h.data(), cyc, 128 * 8, cudaMemcpyDeviceToHost);
      printf("T=%5d reps=%d: %7.2f us/launch, in-kernel %8.0f cycles/rep (CTA 0), err=%s\n", T, reps, ms * 1000 / 20,
             (double)h[0] / reps, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
