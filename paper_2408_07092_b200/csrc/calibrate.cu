// calibrate.cu -- offline outlier-channel calibration (Sec. 4.1;
// modes of Table 3).  Offline and untimed.
//
// One CTA per KV head, one thread per channel c.  Thread c accumulates in
// fp64, in sample order n and group order g, sum|Q[n][hG+g][c]| and
// sum|K[n][h][c]| (reading R5: aggregate |S_i| over every calibration
// (query, key) pair = product of the two sums).  The top-r channels by
// importance (ties: lower channel) are found by rank counting and written
// ascending.  Random mode is one thread running a seeded splitmix64
// Fisher-Yates per head in head order.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

template <typename T>
__global__ void calibrate_kernel(const T *__restrict__ qc, const T *__restrict__ kc, int n, int Hq,
                                 int Hkv, int D, int mode, int r, int32_t *__restrict__ out) {
  extern __shared__ double imp[];  // [D] importance, then [D] int flags
  int *selflag = reinterpret_cast<int *>(imp + D);
  const int h = blockIdx.x, c = threadIdx.x;
  const int G = Hq / Hkv;
  if (c < D) {
    double qs = 0.0, ks = 0.0;
    for (int s = 0; s < n; ++s) {
      for (int g = 0; g < G; ++g)
        qs = qs + fabs((double)Elem<T>::to_f(qc[((size_t)s * Hq + (size_t)h * G + g) * D + c]));
      ks = ks + fabs((double)Elem<T>::to_f(kc[((size_t)s * Hkv + h) * D + c]));
    }
    imp[c] = mode == 0 ? qs * ks : (mode == 1 ? qs : ks);
  }
  __syncthreads();
  bool sel = false;
  if (c < D) {
    const double mine = imp[c];
    int rank = 0;
    for (int o = 0; o < D; ++o) {
      const double v = imp[o];
      rank += (v > mine) || (v == mine && o < c);
    }
    sel = rank < r;
    selflag[c] = sel;
  }
  __syncthreads();
  if (sel) {
    int before = 0;  // position among selected channels, ascending channel order
    for (int o = 0; o < c; ++o) before += selflag[o];
    out[(size_t)h * r + before] = c;
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t &s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void calibrate_random_kernel(int Hkv, int D, int r, uint64_t seed, int32_t *__restrict__ out) {
  extern __shared__ int32_t perm[];  // [D]
  if (threadIdx.x != 0) return;
  uint64_t st = seed;
  for (int h = 0; h < Hkv; ++h) {
    for (int i = 0; i < D; ++i) perm[i] = i;
    for (int i = D - 1; i >= 1; --i) {
      int j = (int)(splitmix64(st) % (uint64_t)(i + 1));
      int32_t t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
    // insertion sort of the first r ascending
    for (int i = 1; i < r; ++i) {
      int32_t v = perm[i];
      int j = i - 1;
      while (j >= 0 && perm[j] > v) {
        perm[j + 1] = perm[j];
        --j;
      }
      perm[j + 1] = v;
    }
    for (int i = 0; i < r; ++i) out[(size_t)h * r + i] = perm[i];
  }
}

cudaError_t launch_calibrate(const void *qc, const void *kc, int n, int Hq, int Hkv, int D, ds_dtype dt,
                             int mode, int r, uint64_t seed, int32_t *out, cudaStream_t st) {
  if (mode == 3) {
    calibrate_random_kernel<<<1, 32, D * sizeof(int32_t), st>>>(Hkv, D, r, seed, out);
    return cudaPeekAtLastError();
  }
  const int threads = ((D + 31) / 32) * 32;
  const size_t smem = D * (sizeof(double) + sizeof(int));
  switch (dt) {
    case DS_BF16:
      calibrate_kernel<__nv_bfloat16><<<Hkv, threads, smem, st>>>(
          (const __nv_bfloat16 *)qc, (const __nv_bfloat16 *)kc, n, Hq, Hkv, D, mode, r, out);
      break;
    case DS_FP16:
      calibrate_kernel<__half><<<Hkv, threads, smem, st>>>((const __half *)qc, (const __half *)kc, n, Hq,
                                                           Hkv, D, mode, r, out);
      break;
    default:
      calibrate_kernel<float><<<Hkv, threads, smem, st>>>((const float *)qc, (const float *)kc, n, Hq, Hkv,
                                                          D, mode, r, out);
  }
  return cudaPeekAtLastError();
}

}  // namespace ds
