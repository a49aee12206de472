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
  const int page = c.block_table[(size_t)b * c.maxp + p / c.P];
  const size_t dst = (((size_t)page * c.Hkv + h) * c.P + (p % c.P)) * c.D;
  const size_t src = (((size_t)b * n_new + i) * c.Hkv + h) * (size_t)c.D;
  const int nvec = c.D * (int)sizeof(T) / 16;
  const uint4 *ks = reinterpret_cast<const uint4 *>(k_new + src);
  const uint4 *vs = reinterpret_cast<const uint4 *>(v_new + src);
  uint4 *kd = reinterpret_cast<uint4 *>((T *)c.k_pool + dst);
  uint4 *vd = reinterpret_cast<uint4 *>((T *)c.v_pool + dst);
  for (int v = lane; v < nvec; v += 32) {
    kd[v] = ks[v];
    vd[v] = vs[v];
  }
  if (c.lnone) return;  // no label cache (Table 4 ablation)
  const int32_t *C = c.C + (size_t)h * c.r;
  const size_t lrow = ((size_t)b * c.Hkv + h) * c.Smax + p;
  if (!c.lq4) {
    T *lab = (T *)c.label + lrow * c.r;
    for (int j = lane; j < c.r; j += 32) lab[j] = k_new[src + C[j]];
    return;
  }
  // 4-bit label (reading R16): s = RNE_T(max|x| / 7) (1 for a zero
  // row or a zero rounding), c_j = clamp(round_half_away(x_j / s), -7, 7)
  float a = 0.0f;
  for (int j = lane; j < c.r; j += 32) a = fmaxf(a, fabsf(Elem<T>::to_f(k_new[src + C[j]])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
  T st = Elem<T>::from_f(a == 0.0f ? 1.0f : a / 7.0f);
  if (Elem<T>::to_f(st) == 0.0f) st = Elem<T>::from_f(1.0f);
  const float s = Elem<T>::to_f(st);
  uint8_t *cod = (uint8_t *)c.label + lrow * c.rb;
  for (int j0 = 0; j0 < c.r; j0 += 32) {  // 32 is even: code pairs never straddle rounds
    const int j = j0 + lane;
    int code = 0;
    if (j < c.r) code = (int)fminf(fmaxf(roundf(Elem<T>::to_f(k_new[src + C[j]]) / s), -7.0f), 7.0f);
    const int hi = __shfl_down_sync(0xffffffffu, code, 1);
    if (!(lane & 1) && j < c.r) cod[j >> 1] = (uint8_t)((code & 15) | ((j + 1 < c.r ? hi & 15 : 0) << 4));
  }
  if (lane == 0) ((T *)c.label_scale)[lrow] = st;
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
