// attend.cu -- a4/a5 of Algorithm 1: exact softmax attention
// over the selected rows K_[i,:], V_[i,:] gathered from the paged KV cache,
// as split-K flash-decoding; plus the dense baseline on the same
// layout (rows = every token).
//
// Grid (nsplit, units).  A CTA owns `rows_per_cta` consecutive positions of
// the unit's (ascending) index list; its 4 warps each own a contiguous
// quarter and run an independent pipeline over batches of 16 rows:
//   * gather: cp.async 16-B chunks of the 256-B K and V rows (page lookup
//     through block_table), swizzled chunk^(row&7) into a per-warp smem ring
//     of NST stages (NST-1 batches in flight while one is computed);
//   * QK: 16-bit types on tensor cores, mma.sync m16n8k16 with the 16 rows
//     as M and the G<=8 query heads of the KV group as N (fp32 accumulate,
//     exact products); fp32 on CUDA cores;
//   * online softmax in base 2 (scale log2(e)/sqrt(d) folded in), fp32;
//   * PV on CUDA cores in fp32 (each lane owns d/32 output dims per head).
// Warps are merged in smem, CTAs write unnormalised partials (m, l, o) which
// the combine kernel reduces and rounds to the output dtype (RNE).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

constexpr int kAttnWarps = 4;
constexpr int kAttnThreads = 32 * kAttnWarps;
constexpr int kRows = 16;  // rows per warp batch
constexpr int kStages = 3;

template <typename T, int EPL>
__device__ __forceinline__ void load_lane(const uint8_t *p, float (&v)[EPL]) {
  if constexpr (sizeof(T) == 4) {
    if constexpr (EPL == 4) {
      float4 x = *reinterpret_cast<const float4 *>(p);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      float2 x = *reinterpret_cast<const float2 *>(p);
      v[0] = x.x; v[1] = x.y;
    }
  } else {
    if constexpr (EPL == 4) {
      uint2 x = *reinterpret_cast<const uint2 *>(p);
      float2 a = Elem<T>::unpack2(x.x), b = Elem<T>::unpack2(x.y);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
      float2 a = Elem<T>::unpack2(*reinterpret_cast<const uint32_t *>(p));
      v[0] = a.x; v[1] = a.y;
    }
  }
}

template <typename T, int D, int G>
struct AttnSmem {
  static constexpr int E = sizeof(T);
  static constexpr int CH = D * E / 16;
  static constexpr int ROWB = D * E;
  static constexpr int STAGE = 2 * kRows * ROWB;
  static constexpr int RING = kAttnWarps * kStages * STAGE;
  static constexpr int SC = kAttnWarps * G * kRows * 4;
  static constexpr int QF = (E == 4) ? G * D * 4 : 0;
  static constexpr int COMB = kAttnWarps * G * (D + 2) * 4;
  static constexpr int BYTES = (RING > COMB ? RING : COMB) + SC + QF;
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(kAttnThreads) attn_split_kernel(AttnParams p) {
  using SM = AttnSmem<T, D, G>;
  constexpr int E = SM::E, CH = SM::CH, ROWB = SM::ROWB, STAGE = SM::STAGE;
  constexpr int GI = (G + 1) / 2;
  constexpr int EPL = D / 32;
  static_assert(CH >= 8, "swizzle needs >= 8 chunks per row");
  const CacheView &c = p.c;
  const int unit = blockIdx.y, split = blockIdx.x;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int n_sel = p.idx ? min(p.k, c.seq_lens[b]) : c.seq_lens[b];
  const int row0 = split * p.rows_per_cta;
  if (row0 >= n_sel) return;
  const int row1 = min(row0 + p.rows_per_cta, n_sel);

  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int RINGB = SM::RING > SM::COMB ? SM::RING : SM::COMB;
  uint8_t *wst = smem + (size_t)warp * kStages * STAGE;
  float *sc = reinterpret_cast<float *>(smem + RINGB) + warp * G * kRows;
  float *qf = reinterpret_cast<float *>(smem + RINGB + SM::SC);

  const int nr = row1 - row0;
  int per = (nr + kAttnWarps - 1) / kAttnWarps;
  per = (per + kRows - 1) & ~(kRows - 1);
  const int wr0 = row0 + warp * per;
  const int wr1 = min(wr0 + per, row1);
  const int nb = wr1 > wr0 ? (wr1 - wr0 + kRows - 1) / kRows : 0;

  const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)h * G) * D;
  const int32_t *idx = p.idx ? p.idx + (size_t)unit * p.k : nullptr;
  const uint8_t *kp = (const uint8_t *)c.k_pool;
  const uint8_t *vp = (const uint8_t *)c.v_pool;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const float scale = p.scale_log2;

  // query operands
  uint32_t bq[(E == 2) ? D / 16 : 1][2];
  if constexpr (E == 2) {
    const int n = lane >> 2, kq = (lane & 3) * 2;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      if (n < G) {
        bq[kk][0] = *reinterpret_cast<const uint32_t *>(qb + (size_t)n * D + kk * 16 + kq);
        bq[kk][1] = *reinterpret_cast<const uint32_t *>(qb + (size_t)n * D + kk * 16 + kq + 8);
      } else {
        bq[kk][0] = 0u;
        bq[kk][1] = 0u;
      }
    }
  } else {
    for (int i = tid; i < G * D; i += kAttnThreads) qf[i] = Elem<T>::to_f(qb[i]);
    __syncthreads();
  }

  auto issue = [&](int j) {
    uint8_t *st = wst + (j % kStages) * STAGE;
    const int rbase = wr0 + j * kRows;
    const int rr = rbase + (lane & (kRows - 1));
    uint32_t rowid = 0;
    if (rr < wr1) {
      const int t = idx ? idx[rr] : rr;
      const int page = bt[t / c.P];
      rowid = ((uint32_t)page * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P + (uint32_t)(t % c.P);
    }
#pragma unroll
    for (int m = 0; m < CH / 2; ++m) {
      const int qq = lane + 32 * m;
      const int row = qq / CH, ch = qq % CH;
      const uint32_t rid = __shfl_sync(0xffffffffu, rowid, row);
      const bool rv = rbase + row < wr1;
      const size_t off = rv ? (size_t)rid * ROWB + (size_t)ch * 16 : 0;
      const uint32_t dst = smem_u32(st + row * ROWB + ((ch ^ (row & 7)) * 16));
      cp_async16(dst, kp + off, rv ? 16 : 0);
      cp_async16(dst + kRows * ROWB, vp + off, rv ? 16 : 0);
    }
  };

  float m_r[GI], l_r[GI], al_r[GI];
#pragma unroll
  for (int i = 0; i < GI; ++i) {
    m_r[i] = -INFINITY;
    l_r[i] = 0.f;
    al_r[i] = 1.f;
  }
  float acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nb) issue(s);
    cp_async_commit();
  }
  for (int j = 0; j < nb; ++j) {
    if (j + kStages - 1 < nb) issue(j + kStages - 1);
    cp_async_commit();
    cp_async_wait<kStages - 1>();
    __syncwarp();
    const uint8_t *st = wst + (j % kStages) * STAGE;
    const int nvalid = min(kRows, wr1 - (wr0 + j * kRows));

    // ---- QK^T -> sc[g][row] (log2 domain)
    if constexpr (E == 2) {
      float cf[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const int mi = lane >> 3;
        const int rowi = (lane & 7) + 8 * (mi & 1);
        const int ch = 2 * kk + (mi >> 1);
        uint32_t a[4];
        ldmatrix_x4(smem_u32(st + rowi * ROWB + ((ch ^ (rowi & 7)) * 16)), a[0], a[1], a[2], a[3]);
        Mma<T>::run(cf, a, bq[kk][0], bq[kk][1]);
      }
      const int r0 = lane >> 2, hh = (lane & 3) * 2;
      if (hh < G) {
        sc[hh * kRows + r0] = r0 < nvalid ? cf[0] * scale : -INFINITY;
        sc[hh * kRows + r0 + 8] = r0 + 8 < nvalid ? cf[2] * scale : -INFINITY;
      }
      if (hh + 1 < G) {
        sc[(hh + 1) * kRows + r0] = r0 < nvalid ? cf[1] * scale : -INFINITY;
        sc[(hh + 1) * kRows + r0 + 8] = r0 + 8 < nvalid ? cf[3] * scale : -INFINITY;
      }
    } else {
      const int row = lane >> 1, half = lane & 1;
      float dot[G];
#pragma unroll
      for (int g = 0; g < G; ++g) dot[g] = 0.f;
      const uint8_t *kr = st + row * ROWB;
#pragma unroll 4
      for (int cc = 0; cc < CH / 2; ++cc) {
        const int ch = half * (CH / 2) + cc;
        const float4 kv = *reinterpret_cast<const float4 *>(kr + ((ch ^ (row & 7)) * 16));
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 qv = *reinterpret_cast<const float4 *>(qf + g * D + ch * 4);
          dot[g] = fmaf(kv.x, qv.x, dot[g]);
          dot[g] = fmaf(kv.y, qv.y, dot[g]);
          dot[g] = fmaf(kv.z, qv.z, dot[g]);
          dot[g] = fmaf(kv.w, qv.w, dot[g]);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) dot[g] += __shfl_xor_sync(0xffffffffu, dot[g], 1);
      if (half == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) sc[g * kRows + row] = row < nvalid ? dot[g] * scale : -INFINITY;
      }
    }
    __syncwarp();

    // ---- online softmax: two heads per pass (lanes 0-15 / 16-31), 16 rows
#pragma unroll
    for (int it = 0; it < GI; ++it) {
      const int g = 2 * it + (lane >> 4), row = lane & 15;
      const float z = g < G ? sc[g * kRows + row] : -INFINITY;
      float bm = z;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
      const float mnew = fmaxf(m_r[it], bm);
      float alpha, pz;
      if (mnew == -INFINITY) {
        alpha = 1.f;
        pz = 0.f;
      } else {
        alpha = exp2f(m_r[it] - mnew);
        pz = exp2f(z - mnew);
      }
      if (g < G) sc[g * kRows + row] = pz;
      float ps = pz;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l_r[it] = l_r[it] * alpha + ps;
      m_r[it] = mnew;
      al_r[it] = alpha;
    }
    __syncwarp();

    // ---- PV (fp32): lane owns dims [lane*EPL, lane*EPL+EPL)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float a = __shfl_sync(0xffffffffu, al_r[g >> 1], (g & 1) * 16);
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[g][e] *= a;
    }
    {
      const int lbyte = lane * EPL * E;
      const int lch = lbyte >> 4, lin = lbyte & 15;
      const uint8_t *vb = st + kRows * ROWB;
#pragma unroll
      for (int row = 0; row < kRows; ++row) {
        float v[EPL];
        load_lane<T, EPL>(vb + row * ROWB + ((lch ^ (row & 7)) << 4) + lin, v);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float pg = sc[g * kRows + row];
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(pg, v[e], acc[g][e]);
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();

  // ---- merge the 4 warps, write this CTA's partial
  __syncthreads();
  float *wm = reinterpret_cast<float *>(smem);
  float *wl = wm + kAttnWarps * G;
  float *wo = wl + kAttnWarps * G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float mg = __shfl_sync(0xffffffffu, m_r[g >> 1], (g & 1) * 16);
    const float lg = __shfl_sync(0xffffffffu, l_r[g >> 1], (g & 1) * 16);
    if (lane == 0) {
      wm[warp * G + g] = mg;
      wl[warp * G + g] = lg;
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e) wo[(warp * G + g) * D + lane * EPL + e] = acc[g][e];
  }
  __syncthreads();
  const size_t pbase = ((size_t)unit * p.nsplit + split) * G;
  for (int i = tid; i < G * D; i += kAttnThreads) {
    const int g = i / D, dd = i - (i / D) * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, wm[w * G + g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < kAttnWarps; ++w) {
        const float sw = exp2f(wm[w * G + g] - M);
        L = fmaf(wl[w * G + g], sw, L);
        O = fmaf(wo[(w * G + g) * D + dd], sw, O);
      }
    }
    p.part_o[(pbase + g) * D + dd] = O;
    if (dd == 0) {
      p.part_ml[(pbase + g) * 2] = M;
      p.part_ml[(pbase + g) * 2 + 1] = L;
    }
  }
}

template <typename T, int D, int G>
__global__ void __launch_bounds__(128) combine_kernel(AttnParams p) {
  const CacheView &c = p.c;
  const int unit = blockIdx.x;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int n_sel = p.idx ? min(p.k, c.seq_lens[b]) : c.seq_lens[b];
  const int nvalid = min(p.nsplit, (n_sel + p.rows_per_cta - 1) / p.rows_per_cta);
  T *out = (T *)p.out + ((size_t)b * c.Hq + (size_t)h * G) * D;
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int g = i / D, dd = i - (i / D) * D;
    float M = -INFINITY;
    for (int s = 0; s < nvalid; ++s) M = fmaxf(M, p.part_ml[(((size_t)unit * p.nsplit + s) * G + g) * 2]);
    float y = 0.f;
    if (M != -INFINITY) {
      float L = 0.f, O = 0.f;
      for (int s = 0; s < nvalid; ++s) {
        const size_t pb = ((size_t)unit * p.nsplit + s) * G + g;
        const float sw = exp2f(p.part_ml[pb * 2] - M);
        L = fmaf(p.part_ml[pb * 2 + 1], sw, L);
        O = fmaf(p.part_o[pb * D + dd], sw, O);
      }
      y = O / L;
    }
    out[(size_t)g * D + dd] = Elem<T>::from_f(y);
  }
}

// ------------------------------------------------------------ dispatch
template <typename T, int D, int G>
static cudaError_t launch_attn_t(const AttnParams &p, const AttnGeom &g, int units, cudaStream_t st) {
  auto kern = attn_split_kernel<T, D, G>;
  const int smem = AttnSmem<T, D, G>::BYTES;
  static const cudaError_t attr =
      cudaFuncSetAttribute(attn_split_kernel<T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           AttnSmem<T, D, G>::BYTES);
  if (attr != cudaSuccess) return attr;
  kern<<<dim3(g.nsplit, units), kAttnThreads, smem, st>>>(p);
  return cudaPeekAtLastError();
}

template <typename T, int D, int G>
static cudaError_t launch_combine_t(const AttnParams &p, int units, cudaStream_t st) {
  combine_kernel<T, D, G><<<units, 128, 0, st>>>(p);
  return cudaPeekAtLastError();
}

template <typename T, int D>
static cudaError_t dispatch_g(const ds_cache *c, const AttnParams &p, const AttnGeom *g, cudaStream_t st) {
  const int units = c->batch * c->num_kv_heads;
  const int G = c->num_q_heads / c->num_kv_heads;
  switch (G) {
    case 1: return g ? launch_attn_t<T, D, 1>(p, *g, units, st) : launch_combine_t<T, D, 1>(p, units, st);
    case 2: return g ? launch_attn_t<T, D, 2>(p, *g, units, st) : launch_combine_t<T, D, 2>(p, units, st);
    case 4: return g ? launch_attn_t<T, D, 4>(p, *g, units, st) : launch_combine_t<T, D, 4>(p, units, st);
    default: return g ? launch_attn_t<T, D, 8>(p, *g, units, st) : launch_combine_t<T, D, 8>(p, units, st);
  }
}

template <typename T>
static cudaError_t dispatch_d(const ds_cache *c, const AttnParams &p, const AttnGeom *g, cudaStream_t st) {
  return c->head_dim == 64 ? dispatch_g<T, 64>(c, p, g, st) : dispatch_g<T, 128>(c, p, g, st);
}

static cudaError_t dispatch(const ds_cache *c, const AttnParams &p, const AttnGeom *g, cudaStream_t st) {
  switch (c->dtype) {
    case DS_BF16: return dispatch_d<__nv_bfloat16>(c, p, g, st);
    case DS_FP16: return dispatch_d<__half>(c, p, g, st);
    default: return dispatch_d<float>(c, p, g, st);
  }
}

cudaError_t launch_attn(const ds_cache *c, const AttnParams &p, const AttnGeom &g, cudaStream_t st) {
  return dispatch(c, p, &g, st);
}
cudaError_t launch_combine(const ds_cache *c, const AttnParams &p, cudaStream_t st) {
  return dispatch(c, p, nullptr, st);
}

AttnGeom attn_geom(const ds_cache *c, int n_rows) {
  AttnGeom g;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * c->num_kv_heads;
  const int target = 4 * sms;  // CTAs in flight
  int nsplit = (target + units - 1) / units;
  const int max_split = (n_rows + 63) / 64;
  if (nsplit > max_split) nsplit = max_split;
  if (nsplit < 1) nsplit = 1;
  int rows = (n_rows + nsplit - 1) / nsplit;
  rows = (rows + 63) & ~63;
  g.rows_per_cta = rows;
  g.nsplit = (n_rows + rows - 1) / rows;
  g.threads = kAttnThreads;
  g.smem = 0;
  return g;
}

}  // namespace ds
