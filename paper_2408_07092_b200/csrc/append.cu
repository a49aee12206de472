// append.cu -- a0: KV + label-cache append (Sec. 4.2).
//
// One warp per (b, new token i, KV head h): 16-byte vector copies of the K
// and V rows into their page slot, then the r label channels
// label[b][h][p][j] = k_new[b][i][h][C[h][j]] as a bit copy of the same
// element type (DS_LABEL_INT4: the row quantised to 4-bit codes + a scale,
// reading R16).  Bytes per unit and token: 2*d*e (KV) + r*e (label), or
// 2*d*e + ceil(r/2) + e.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"
#include "append_row.cuh"

namespace ds {

template <typename T>
__global__ void __launch_bounds__(128) append_kernel(CacheView c, const T *__restrict__ k_new,
                                                     const T *__restrict__ v_new,
                                                     const int32_t *__restrict__ positions,
                                                     int n_new) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int row = blockIdx.x * 4 + warp;  // over (i, h)
  pdl_wait();
  pdl_trigger();
  if (row >= n_new * c.Hkv) return;
  const int i = row / c.Hkv, h = row - i * c.Hkv;
  const int p = positions[b] + i;
  const size_t src = (((size_t)b * n_new + i) * c.Hkv + h) * (size_t)c.D;
  append_row_warp<T>(c, b, h, p, k_new + src, v_new + src, lane, true, nullptr, nullptr);
}

cudaError_t launch_append(const ds_cache *cc, const void *k_new, const void *v_new,
                          const int32_t *positions, int n_new, cudaStream_t st) {
  CacheView c = make_view(cc);
  PdlLaunch L(dim3((n_new * c.Hkv + 3) / 4, c.B), dim3(128), 0, st);
  switch (cc->dtype) {
    case DS_BF16:
      return L.run(append_kernel<__nv_bfloat16>, c, (const __nv_bfloat16 *)k_new, (const __nv_bfloat16 *)v_new,
                   positions, n_new);
    case DS_FP16:
      return L.run(append_kernel<__half>, c, (const __half *)k_new, (const __half *)v_new, positions, n_new);
    default:
      return L.run(append_kernel<float>, c, (const float *)k_new, (const float *)v_new, positions, n_new);
  }
}

}  // namespace ds
