// prefetch.cu -- a6, Double Sparsity-Offload: copy the selected
// K/V rows of every unit from the (host-resident) paged pools into a device
// slot, ascending by token, so the next layer's attention reads them from HBM.
//
// Grid (ceil(k / 64), units), 8 warps; a warp moves 8 rows per step (the
// 16-B loads of 8 K rows and 8 V rows are all in flight before any store:
// over the host link a load takes microseconds).  Bytes per unit: 2 * k_eff
// * d * e over the link, the same into HBM.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

constexpr int kGatherRows = 64;  // rows per CTA
constexpr int kGatherWarps = 8;

__global__ void __launch_bounds__(kGatherWarps * 32) gather_rows_kernel(CacheView c, ds_prefetch_slot s,
                                                                        int row_bytes) {
  const int unit = blockIdx.y;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_wait();  // the index list comes from the selection launch just before
  pdl_trigger();
  if (unit == 0 && blockIdx.x == 0)
    for (int i = threadIdx.x; i < c.B; i += blockDim.x) {
      s.count[i] = min(s.k, c.seq_lens[i]);
      s.table[i] = i;
    }
  const int kk = min(s.k, c.seq_lens[b]);
  const int cpr = row_bytes / 16;  // 16-B chunks per row
  const int32_t *idx = s.idx + (size_t)unit * s.k;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const uint8_t *kp = (const uint8_t *)c.k_pool, *vp = (const uint8_t *)c.v_pool;
  uint8_t *kd = (uint8_t *)s.k_rows + (size_t)unit * s.k * row_bytes;
  uint8_t *vd = (uint8_t *)s.v_rows + (size_t)unit * s.k * row_bytes;
  const int r0 = blockIdx.x * kGatherRows;
  const int r1 = min(r0 + kGatherRows, kk);
  const int total = (r1 - r0) * cpr;  // 16-B chunks of this CTA (per pool)
  for (int q0 = warp * 32 * 8; q0 < total; q0 += kGatherWarps * 32 * 8) {
    uint4 kv[8], vv[8];
    size_t dst[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u * 32 + lane;
      dst[u] = ~(size_t)0;
      if (q < total) {
        const int r = r0 + q / cpr, ch = q % cpr;
        const int t = idx[r];
        const size_t row = ((size_t)bt[t / c.P] * c.Hkv + h) * c.P + (t % c.P);
        kv[u] = *reinterpret_cast<const uint4 *>(kp + row * row_bytes + ch * 16);
        vv[u] = *reinterpret_cast<const uint4 *>(vp + row * row_bytes + ch * 16);
        dst[u] = (size_t)r * row_bytes + ch * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dst[u] != ~(size_t)0) {
        *reinterpret_cast<uint4 *>(kd + dst[u]) = kv[u];
        *reinterpret_cast<uint4 *>(vd + dst[u]) = vv[u];
      }
  }
}

cudaError_t launch_gather(const ds_cache *cc, const ds_prefetch_slot *slot, cudaStream_t st) {
  CacheView c = make_view(cc);
  const int eb = cc->dtype == DS_FP32 ? 4 : 2;
  PdlLaunch L(dim3((slot->k + kGatherRows - 1) / kGatherRows, cc->batch * cc->num_kv_heads),
              dim3(kGatherWarps * 32), 0, st);
  return L.run(gather_rows_kernel, c, *slot, cc->head_dim * eb);
}

}  // namespace ds
