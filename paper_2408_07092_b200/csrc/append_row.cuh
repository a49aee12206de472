// append_row.cuh -- a0 for one (b, KV head h, token p) by one warp:
// the K and V rows into the token's page slot and its label row -- a bit
// copy of the r channels (DS_LABEL_NATIVE, reading R8), 4-bit codes + scale
// (DS_LABEL_INT4, reading R16) or nothing (DS_LABEL_NONE).  Shared by
// append_kernel and the fused append of decode_kernel, so both write the
// same bytes.
#pragma once
#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

// write: store the rows (false: only report the label values).
// lab_out (nullable, r floats, shared memory): the values line 2 scores
// token p with -- the widened label values (native / none) or the codes as
// floats (int4, the scale in *scale_out).  The whole warp must call.
template <typename T>
__device__ __forceinline__ void append_row_warp(const CacheView &c, int b, int h, int p, const T *__restrict__ krow,
                                                const T *__restrict__ vrow, int lane, bool write, float *lab_out,
                                                float *scale_out) {
  if (write) {
    const int page = c.block_table[(size_t)b * c.maxp + p / c.P];
    const size_t dst = (((size_t)page * c.Hkv + h) * c.P + (p % c.P)) * c.D;
    const int nvec = c.D * (int)sizeof(T) / 16;
    const uint4 *ks = reinterpret_cast<const uint4 *>(krow);
    const uint4 *vs = reinterpret_cast<const uint4 *>(vrow);
    uint4 *kd = reinterpret_cast<uint4 *>((T *)c.k_pool + dst);
    uint4 *vd = reinterpret_cast<uint4 *>((T *)c.v_pool + dst);
    for (int v = lane; v < nvec; v += 32) {
      kd[v] = ks[v];
      vd[v] = vs[v];
    }
  }
  const int32_t *C = c.C + (size_t)h * c.r;
  const size_t lrow = ((size_t)b * c.Hkv + h) * c.Smax + p;
  if (!c.lq4) {
    T *lab = (T *)c.label + lrow * c.r;
    for (int j = lane; j < c.r; j += 32) {
      const T x = krow[C[j]];
      if (write && !c.lnone) lab[j] = x;
      if (lab_out) lab_out[j] = Elem<T>::to_f(x);
    }
    return;
  }
  // 4-bit label (reading R16): s = RNE_T(max|x| / 7) (1 for a zero
  // row or a zero rounding), c_j = clamp(round_half_away(x_j / s), -7, 7)
  float a = 0.0f;
  for (int j = lane; j < c.r; j += 32) a = fmaxf(a, fabsf(Elem<T>::to_f(krow[C[j]])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
  T st = Elem<T>::from_f(a == 0.0f ? 1.0f : a / 7.0f);
  if (Elem<T>::to_f(st) == 0.0f) st = Elem<T>::from_f(1.0f);
  const float s = Elem<T>::to_f(st);
  uint8_t *cod = (uint8_t *)c.label + lrow * c.rb;
  for (int j0 = 0; j0 < c.r; j0 += 32) {  // 32 is even: code pairs never straddle rounds
    const int j = j0 + lane;
    int code = 0;
    if (j < c.r) code = (int)fminf(fmaxf(roundf(Elem<T>::to_f(krow[C[j]]) / s), -7.0f), 7.0f);
    const int hi = __shfl_down_sync(0xffffffffu, code, 1);
    if (write && !(lane & 1) && j < c.r) cod[j >> 1] = (uint8_t)((code & 15) | ((j + 1 < c.r ? hi & 15 : 0) << 4));
    if (lab_out && j < c.r) lab_out[j] = (float)code;
  }
  if (lane == 0) {
    if (write) ((T *)c.label_scale)[lrow] = st;
    if (scale_out) *scale_out = s;
  }
}

}  // namespace ds
