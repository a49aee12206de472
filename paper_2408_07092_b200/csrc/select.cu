// select.cu -- a1..a3 of Algorithm 1: label-score GEMV and
// exact top-k selection, one thread-block cluster per (b, KV head) unit.
//
// Geometry: a unit's tokens [0, n) are split into CL contiguous ranges of
// `chunk` tokens (chunk = ceil(n/CL) rounded to 32), one CTA each.
//
//  a1  q_lab[j] = sum_g q[b][hG+g][C[h][j]]     (fp32, g order; reading R3)
//  a2  s_hat[t] = fma-chain_j(q_lab[j], L[t][j]) (fp32, j ascending, no
//      1/sqrt(d); reading R2) streamed from the contiguous label cache with
//      128-bit loads (one label row = r*e bytes, 16 B at r=8/16-bit), kept
//      on chip as a monotone u32 order key in shared memory.
//  a3  MSB-first radix select over the CL CTAs: per 8-bit digit a
//      warp-aggregated shared-memory histogram, a DSMEM all-reduce (every
//      CTA reads the CL histograms), an identical suffix scan in every CTA
//      -> digit of the k-th key; exits early as soon as the boundary bin
//      holds exactly the remaining count.  Then an ordered compaction:
//      token t goes to position  #gt(<t) + min(#eq(<t), remaining),
//      which yields the ascending index list with ties to the lower index
//      (reading R6) without sorting.  s_hat never touches HBM.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace cg = cooperative_groups;

namespace ds {

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kMaxR = 256;
constexpr int kSelMaxSmem = 200 * 1024;

// s_hat for one token (fma chain over j ascending).
template <typename T, int R>
__device__ __forceinline__ float label_score(const T *__restrict__ row, const float *qlab, int r) {
  float s = 0.0f;
  if constexpr (R > 0 && (R * sizeof(T)) % 16 == 0) {
    constexpr int NV = R * sizeof(T) / 16;
    uint4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = __ldg(reinterpret_cast<const uint4 *>(row) + i);
    const T *e = reinterpret_cast<const T *>(v);
#pragma unroll
    for (int j = 0; j < R; ++j) s = fmaf(qlab[j], Elem<T>::to_f(e[j]), s);
  } else {
    for (int j = 0; j < r; ++j) s = fmaf(qlab[j], Elem<T>::to_f(row[j]), s);
  }
  return s;
}

template <typename T, int R>
__global__ void __launch_bounds__(kSelThreads) score_select_kernel(SelectParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const CacheView &c = p.c;
  const int unit = blockIdx.x / CL;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = c.seq_lens[b];
  const int keff = min(p.k, n);
  const int r = R > 0 ? R : c.r;

  extern __shared__ uint32_t keys[];  // [cap]
  __shared__ uint32_t hist[2][256];
  __shared__ float qlab[kMaxR];
  __shared__ uint32_t wsum[kSelWarps];
  __shared__ uint32_t wgt[kSelWarps], weq[kSelWarps];
  __shared__ uint32_t cta_cnt[2];
  __shared__ uint32_t sel_state[3];

  int chunk = (n + CL - 1) / CL;
  chunk = (chunk + 31) & ~31;
  const int t0 = crank * chunk;
  const int nloc = max(0, min(chunk, n - t0));

  // ---- a1: query label (group sum, g order)
  for (int j = tid; j < r; j += kSelThreads) {
    const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)h * c.G) * c.D;
    const int ch = c.C[(size_t)h * c.r + j];
    float s = 0.0f;
    for (int g = 0; g < c.G; ++g) s = s + Elem<T>::to_f(qb[(size_t)g * c.D + ch]);
    qlab[j] = s;
  }
  __syncthreads();
  float ql[R > 0 ? R : 1];
  if constexpr (R > 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) ql[j] = qlab[j];
  }
  const float *qsrc = R > 0 ? ql : qlab;

  // ---- a2: stream the label rows, 4 tokens in flight per thread
  const T *lab = (const T *)c.label + (((size_t)b * c.Hkv + h) * c.Smax + t0) * (size_t)c.r;
  if (p.scores) {  // diagnostics entry: s_hat to HBM, no selection
    float *so = p.scores + ((size_t)b * c.Hkv + h) * c.Smax + t0;
    for (int i = tid; i < nloc; i += kSelThreads) so[i] = label_score<T, R>(lab + (size_t)i * r, qsrc, r);
    return;
  }
  {
    int i = tid;
    for (; i + 3 * kSelThreads < nloc; i += 4 * kSelThreads) {
      float s0 = label_score<T, R>(lab + (size_t)i * r, qsrc, r);
      float s1 = label_score<T, R>(lab + (size_t)(i + kSelThreads) * r, qsrc, r);
      float s2 = label_score<T, R>(lab + (size_t)(i + 2 * kSelThreads) * r, qsrc, r);
      float s3 = label_score<T, R>(lab + (size_t)(i + 3 * kSelThreads) * r, qsrc, r);
      keys[i] = order_key(s0);
      keys[i + kSelThreads] = order_key(s1);
      keys[i + 2 * kSelThreads] = order_key(s2);
      keys[i + 3 * kSelThreads] = order_key(s3);
    }
    for (; i < nloc; i += kSelThreads) keys[i] = order_key(label_score<T, R>(lab + (size_t)i * r, qsrc, r));
  }

  int32_t *idx_out = p.idx + (size_t)unit * p.k;
  // positions >= k_eff are -1
  if (crank == 0)
    for (int i = keff + tid; i < p.k; i += kSelThreads) idx_out[i] = -1;

  if (keff >= n) {  // every token is selected: ascending identity (no cluster traffic)
    for (int i = tid; i < nloc; i += kSelThreads) idx_out[t0 + i] = t0 + i;
    return;
  }

  // ---- a3: cluster radix select
  if (tid < 256) hist[0][tid] = 0;
  __syncthreads();
  uint32_t prefix = 0, mask = 0;
  int remaining = keff;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    uint32_t *hcur = hist[pass & 1];
    for (int base = 0; base < nloc; base += kSelThreads) {
      const int i = base + tid;
      uint32_t key = i < nloc ? keys[i] : 0u;
      const bool valid = (i < nloc) && ((key & mask) == prefix);
      const uint32_t dig = (key >> shift) & 255u;
      const uint32_t peers = __match_any_sync(0xffffffffu, valid ? dig : 0x100u);
      if (valid && lane == __ffs(peers) - 1) atomicAdd(&hcur[dig], (uint32_t)__popc(peers));
    }
    cluster.sync();  // every CTA's histogram is complete and visible
    uint32_t tot = 0;
    if (tid < 256) {
      for (int cr = 0; cr < CL; ++cr) tot += cluster.map_shared_rank(hcur, cr)[tid];
    }
    // suffix sum over bins: incl(d) = sum_{d' >= d} tot(d')
    uint32_t v = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t x = __shfl_down_sync(0xffffffffu, v, o);
      if (lane + o < 32) v += x;
    }
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (tid < 256) {
      uint32_t above_w = 0;
      for (int w = warp + 1; w < 256 / 32; ++w) above_w += wsum[w];
      const uint32_t incl = v + above_w;
      const uint32_t above = incl - tot;
      if (above < (uint32_t)remaining && incl >= (uint32_t)remaining) {
        sel_state[0] = tid;
        sel_state[1] = above;
        sel_state[2] = tot;
      }
    }
    // this pass's zeroing target was last read (remotely) before the
    // cluster.sync above, so it can be cleared now
    if (tid < 256) hist[(pass + 1) & 1][tid] = 0;
    __syncthreads();
    const uint32_t dstar = sel_state[0], above = sel_state[1], cnt = sel_state[2];
    remaining -= (int)above;
    prefix |= dstar << shift;
    mask |= 255u << shift;
    if ((int)cnt == remaining) break;  // take the whole boundary bin
  }

  // ---- ordered compaction
  int wchunk = (nloc + kSelWarps - 1) / kSelWarps;
  wchunk = (wchunk + 31) & ~31;
  const int wb = warp * wchunk, we = min(wb + wchunk, nloc);
  uint32_t ngt = 0, neq = 0;
  for (int base = wb; base < we; base += 32) {
    const int i = base + lane;
    const uint32_t km = (i < we ? keys[i] : 0u) & mask;
    const bool gt = i < we && km > prefix;
    const bool eq = i < we && km == prefix;
    ngt += __popc(__ballot_sync(0xffffffffu, gt));
    neq += __popc(__ballot_sync(0xffffffffu, eq));
  }
  if (lane == 0) {
    wgt[warp] = ngt;
    weq[warp] = neq;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t a = 0, e = 0;
    for (int w = 0; w < kSelWarps; ++w) {
      a += wgt[w];
      e += weq[w];
    }
    cta_cnt[0] = a;
    cta_cnt[1] = e;
  }
  cluster.sync();
  uint32_t gbase = 0, ebase = 0;
  for (int cr = 0; cr < crank; ++cr) {
    const uint32_t *rc = cluster.map_shared_rank(cta_cnt, cr);
    gbase += rc[0];
    ebase += rc[1];
  }
  for (int w = 0; w < warp; ++w) {
    gbase += wgt[w];
    ebase += weq[w];
  }
  const uint32_t lt = lanemask_lt();
  const uint32_t rem = (uint32_t)remaining;
  for (int base = wb; base < we; base += 32) {
    const int i = base + lane;
    const uint32_t km = (i < we ? keys[i] : 0u) & mask;
    const bool gt = i < we && km > prefix;
    const bool eq = i < we && km == prefix;
    const uint32_t gm = __ballot_sync(0xffffffffu, gt);
    const uint32_t em = __ballot_sync(0xffffffffu, eq);
    const uint32_t gb = gbase + __popc(gm & lt);
    const uint32_t eb = ebase + __popc(em & lt);
    if (gt) {
      idx_out[gb + min(eb, rem)] = t0 + i;
    } else if (eq && eb < rem) {
      idx_out[gb + eb] = t0 + i;
    }
    gbase += __popc(gm);
    ebase += __popc(em);
  }
  cluster.sync();  // no CTA leaves while its shared memory may still be read
}

SelectGeom select_geom(const ds_cache *c) {
  SelectGeom g;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * c->num_kv_heads;
  const int target = 4 * sms;
  int cl = 1;
  while (cl < 8 && units * cl < target) cl <<= 1;
  // keys must fit: cap * 4 B <= 96 KiB
  int cap = 0;
  for (;;) {
    cap = ((c->max_seq_len + cl - 1) / cl + 31) & ~31;
    if (cap * 4 <= 96 * 1024 || cl >= 16) break;
    cl <<= 1;
  }
  g.cl = cl;
  g.cap = cap;
  g.threads = kSelThreads;
  g.smem = (size_t)cap * 4;
  return g;
}

template <typename T, int R>
static cudaError_t launch_select_t(const SelectParams &p, const SelectGeom &g, int units, cudaStream_t st) {
  auto kern = score_select_kernel<T, R>;
  // kernel attributes are set once per process (thread-safe static init),
  // so no attribute call happens inside CUDA-graph capture
  static const cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(score_select_kernel<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSelMaxSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(score_select_kernel<T, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * g.cl);
  cfg.blockDim = dim3(g.threads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = g.cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_select(const ds_cache *c, const SelectParams &p, const SelectGeom &g, cudaStream_t st) {
  const int units = c->batch * c->num_kv_heads;
  const int rb = c->r * (c->dtype == DS_FP32 ? 4 : 2);
  switch (c->dtype) {
    case DS_BF16:
      return c->r == 8 ? launch_select_t<__nv_bfloat16, 8>(p, g, units, st)
                       : (c->r == 16 ? launch_select_t<__nv_bfloat16, 16>(p, g, units, st)
                                     : launch_select_t<__nv_bfloat16, 0>(p, g, units, st));
    case DS_FP16:
      return c->r == 8 ? launch_select_t<__half, 8>(p, g, units, st)
                       : (c->r == 16 ? launch_select_t<__half, 16>(p, g, units, st)
                                     : launch_select_t<__half, 0>(p, g, units, st));
    default:
      (void)rb;
      return c->r == 16 ? launch_select_t<float, 16>(p, g, units, st)
                        : (c->r == 8 ? launch_select_t<float, 8>(p, g, units, st)
                                     : launch_select_t<float, 0>(p, g, units, st));
  }
}

}  // namespace ds
