// attend.cu -- a4/a5 of Algorithm 1: exact softmax attention
// over the selected rows K_[i,:], V_[i,:] gathered from the paged KV cache,
// as split-K flash-decoding; plus the dense baseline on the same
// layout (rows = every token).
//
// Grid (nsplit, units), cluster (nsplit, 1, 1): the nsplit CTAs of a unit
// form one cluster.  CTA s owns positions [s*R, (s+1)*R) of the unit's
// ascending index list (R = rows_per_cta), processed in tiles of kTile rows:
//   * prologue per tile: the tile's pool row ids (token -> page via
//     block_table) are resolved once into shared memory, so the gathers never
//     wait on dependent index loads;
//   * its 4 warps each own a contiguous quarter of the tile and run an
//     independent cp.async pipeline over batches of 16 rows: the 256-B K and
//     V rows are copied in 16-B chunks, swizzled chunk^(row&7), into a
//     per-warp ring of kStages stages (kStages-1 batches in flight);
//   * QK: 16-bit types on tensor cores, mma.sync m16n8k16 with the 16 rows as
//     M and the G<=8 query heads of the KV group as N (exact products, fp32
//     accumulate); fp32 on CUDA cores;
//   * online softmax in base 2 (scale log2(e)/sqrt(d) folded in), fp32;
//   * PV on CUDA cores in fp32 (each lane owns d/32 output dims per head).
// Warps merge in shared memory; the CTAs of the cluster then merge their
// (m, l, o) partials over DSMEM, each CTA finishing a slice of the G*d
// outputs, rounded once to the output dtype (RNE).  No HBM partials.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace cg = cooperative_groups;

namespace ds {

constexpr int kAttnWarps = 4;
constexpr int kAttnThreads = 32 * kAttnWarps;
constexpr int kRows = 16;  // rows per warp batch
constexpr int kStages = 3;
constexpr int kTile = 1024;  // rows per rowid tile
constexpr int kMaxSplit = 16;

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


// Sparse path: wait until the unit's selection is published (score_select
// kernel, possibly still running under PDL); the dense path waits for the
// predecessor grid.
__device__ __forceinline__ void wait_inputs(const uint32_t *ready, int unit, int n_sel) {
  if (ready) {
    pdl_trigger();
    if (n_sel > 0) {
      if (threadIdx.x == 0) {
        uint32_t v;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ready + unit) : "memory");
          if (v) break;
          __nanosleep(128);
        }
      }
      __syncthreads();
    }
  } else {
    pdl_wait();
    pdl_trigger();
  }
}

// Pool row ids of rows [tr0, tr0+tn) of a unit into smem: taken from the
// select kernel's list (sparse) or resolved through block_table (dense).
__device__ __forceinline__ void load_rowids(uint32_t *rowids, const int32_t *rid, const int32_t *bt,
                                            const CacheView &c, int h, int tr0, int tn, int nthreads,
                                            int me) {
  // batches of loads into registers before any smem store: the round trips
  // overlap instead of serialising on the stores
  constexpr int BU = 8;
  for (int i0 = me; i0 < tn; i0 += BU * nthreads) {
    uint32_t v[BU];
#pragma unroll
    for (int u = 0; u < BU; ++u) {
      const int i = i0 + u * nthreads;
      if (i < tn) {
        if (rid) {  // written by a kernel that may still be running (PDL): coherent L2 load
          v[u] = (uint32_t)__ldcg(rid + tr0 + i);
        } else {
          const int t = tr0 + i;
          v[u] = ((uint32_t)__ldg(bt + t / c.P) * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P +
                 (uint32_t)(t % c.P);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < BU; ++u)
      if (i0 + u * nthreads < tn) rowids[i0 + u * nthreads] = v[u];
  }
}

// Merge the (m, l, o) partials of the nsplit CTAs of a cluster over DSMEM;
// CTA s finishes outputs [s*P, (s+1)*P) of the unit's G*D, rounded once.
// cm = this CTA's partial: [G] m, [G] l, [G][D] o (log2 domain, unnormalised).
template <typename T, int D, int G>
__device__ __forceinline__ void cluster_merge(cg::cluster_group &cluster, float *cm, const AttnParams &p, int b,
                                              int h, int nthreads) {
  const int nsplit = (int)cluster.num_blocks();
  const int split = (int)cluster.block_rank();
  T *out = (T *)p.out + ((size_t)b * p.c.Hq + (size_t)h * G) * D;
  const int per_cta = (G * D + nsplit - 1) / nsplit;
  const int o0 = split * per_cta, o1 = min(o0 + per_cta, G * D);
  for (int i = o0 + (int)threadIdx.x; i < o1; i += nthreads) {
    const int g = i / D, dd = i - (i / D) * D;
    float M = -INFINITY;
    for (int s = 0; s < nsplit; ++s) M = fmaxf(M, cluster.map_shared_rank(cm, s)[g]);
    float y = 0.f;
    if (M != -INFINITY) {
      float L = 0.f, O = 0.f;
      for (int s = 0; s < nsplit; ++s) {
        const float *rm = cluster.map_shared_rank(cm, s);
        const float sw = exp2f(rm[g] - M);
        L = fmaf(rm[G + g], sw, L);
        O = fmaf(rm[2 * G + g * D + dd], sw, O);
      }
      y = O / L;
    }
    out[(size_t)g * D + dd] = Elem<T>::from_f(y);
  }
  cluster.sync();  // keep every partial alive until all readers are done
  if (p.ready && split == 0 && threadIdx.x == 0) p.ready[(size_t)b * p.c.Hkv + h] = 0u;  // consumed
}

// Merge nw warp partials (wm/wl [nw][G], wo [nw][G][D]) into the CTA partial cm.
template <int D, int G>
__device__ __forceinline__ void warp_merge(const float *wm, const float *wl, const float *wo, int nw, float *cm,
                                           int nthreads) {
  float *cl = cm + G, *co = cm + 2 * G;
  for (int i = threadIdx.x; i < G * D; i += nthreads) {
    const int g = i / D, dd = i - (i / D) * D;
    float M = -INFINITY;
    for (int w = 0; w < nw; ++w) M = fmaxf(M, wm[w * G + g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < nw; ++w) {
        const float sw = exp2f(wm[w * G + g] - M);
        L = fmaf(wl[w * G + g], sw, L);
        O = fmaf(wo[(w * G + g) * D + dd], sw, O);
      }
    }
    co[g * D + dd] = O;
    if (dd == 0) {
      cm[g] = M;
      cl[g] = L;
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
  // after the loop the ring area holds the warp partials then the CTA partial
  static constexpr int WPART = kAttnWarps * G * (D + 2) * 4;
  static constexpr int CPART = G * (D + 2) * 4;
  static constexpr int RINGB = RING > WPART + CPART ? RING : WPART + CPART;
  static constexpr int SC = kAttnWarps * G * kRows * 4;
  static constexpr int QF = (E == 4) ? G * D * 4 : 0;
  static constexpr int ROWID = kTile * 4;
  static constexpr int BYTES = RINGB + SC + QF + ROWID;
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(kAttnThreads) attn_simt_kernel(AttnParams p) {
  using SM = AttnSmem<T, D, G>;
  constexpr int E = SM::E, CH = SM::CH, ROWB = SM::ROWB, STAGE = SM::STAGE;
  constexpr int GI = (G + 1) / 2;
  constexpr int EPL = D / 32;
  static_assert(CH >= 8, "swizzle needs >= 8 chunks per row");
  cg::cluster_group cluster = cg::this_cluster();
  const int nsplit = (int)cluster.num_blocks();
  const int split = (int)cluster.block_rank();
  const CacheView &c = p.c;
  const int unit = blockIdx.y;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int n_sel = p.rowid ? min(p.k, c.seq_lens[b]) : c.seq_lens[b];
  const int row0 = min(split * p.rows_per_cta, n_sel);
  const int row1 = min(row0 + p.rows_per_cta, n_sel);

  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t *wst = smem + (size_t)warp * kStages * STAGE;
  float *sc = reinterpret_cast<float *>(smem + SM::RINGB) + warp * G * kRows;
  float *qf = reinterpret_cast<float *>(smem + SM::RINGB + SM::SC);
  uint32_t *rowids = reinterpret_cast<uint32_t *>(smem + SM::RINGB + SM::SC + SM::QF);

  const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)h * G) * D;
  const int32_t *rid = p.rowid ? p.rowid + (size_t)unit * p.k : nullptr;
  const uint8_t *kp = (const uint8_t *)c.k_pool;
  const uint8_t *vp = (const uint8_t *)c.v_pool;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const float scale = p.scale_log2;

  wait_inputs(p.ready, unit, n_sel);
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
  }

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

  for (int tr0 = row0; tr0 < row1; tr0 += kTile) {
    const int tn = min(kTile, row1 - tr0);
    __syncthreads();  // previous tile fully consumed
    load_rowids(rowids, rid, bt, c, h, tr0, tn, kAttnThreads, tid);
    __syncthreads();
    int per = (tn + kAttnWarps - 1) / kAttnWarps;
    per = (per + kRows - 1) & ~(kRows - 1);
    const int wr0 = min(warp * per, tn);
    const int wr1 = min(wr0 + per, tn);
    const int nb = (wr1 - wr0 + kRows - 1) / kRows;

    auto issue = [&](int j) {
      uint8_t *st = wst + (j % kStages) * STAGE;
      const int rbase = wr0 + j * kRows;
#pragma unroll
      for (int m = 0; m < CH / 2; ++m) {
        const int qq = lane + 32 * m;
        const int row = qq / CH, ch = qq % CH;
        const bool rv = rbase + row < wr1;
        const size_t off = rv ? (size_t)rowids[rbase + row] * ROWB + (size_t)ch * 16 : 0;
        const uint32_t dst = smem_u32(st + row * ROWB + ((ch ^ (row & 7)) * 16));
        cp_async16(dst, kp + off, rv ? 16 : 0);
        cp_async16(dst + kRows * ROWB, vp + off, rv ? 16 : 0);
      }
    };

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
  }

  // ---- merge the 4 warps into this CTA's partial (kept in smem for DSMEM)
  __syncthreads();
  float *wm = reinterpret_cast<float *>(smem);
  float *wl = wm + kAttnWarps * G;
  float *wo = wl + kAttnWarps * G;
  float *cm = reinterpret_cast<float *>(smem + SM::WPART);  // [G] m, [G] l, [G][D] o
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
  warp_merge<D, G>(wm, wl, wo, kAttnWarps, cm, kAttnThreads);
  cluster.sync();  // every CTA's partial is complete and visible
  cluster_merge<T, D, G>(cluster, cm, p, b, h, kAttnThreads);
}

// ====================================================================
// 16-bit path: cp.async row gathers + tensor-core QK and PV (TMA measured,
// not faster: profiles/r2_tma_gather.md).
//
// Per warp and batch of 16 rows: the 256-B K and V rows are copied with
// cp.async in 16-B chunks (one warp instruction = 512 B) into a padded stage
// (row stride d*2+16 B, so ldmatrix is bank-conflict free), kMmaStages-1
// batches in flight.  S^T = Q K^T with the query heads as M (16, zero-padded beyond
// G) and the rows as N: Q is a register-resident A operand, K comes in by
// ldmatrix as B.  The S fragments are exactly the P fragments of the next
// MMA (FA2 register reuse): O = P V with V by ldmatrix.trans as B; P is
// rounded once to the 16-bit type, l and m stay fp32.
constexpr int kMmaWarps = 8;
constexpr int kMmaThreads = 32 * kMmaWarps;
constexpr int kMmaStages = 3;
constexpr int kSub = 256;  // rows whose pool row ids a warp stages at a time

template <typename T, int D, int G>
struct MmaSmem {
  static constexpr int ROWB = D * 2;
  static constexpr int ROWP = ROWB + 16;
  static constexpr int STAGE = 2 * kRows * ROWP;
  static constexpr int RING = kMmaWarps * kMmaStages * STAGE;
  static constexpr int WPART = kMmaWarps * G * (D + 2) * 4;
  static constexpr int CPART = G * (D + 2) * 4;
  static constexpr int RINGB = RING > WPART + CPART ? RING : WPART + CPART;
  static constexpr int ROWID = kMmaWarps * kSub * 4;
  static constexpr int BYTES = RINGB + ROWID;
};

template <typename T, int D, int G>
__global__ void __launch_bounds__(kMmaThreads, 1) attn_mma_kernel(AttnParams p) {
  using SM = MmaSmem<T, D, G>;
  constexpr int ROWB = SM::ROWB, ROWP = SM::ROWP, STAGE = SM::STAGE;
  constexpr int NKS = D / 16, NDT = D / 8;
  constexpr int CHN = ROWB / 16, RPP = 32 / CHN;
  static_assert(G <= 8, "query heads per KV head must fit the 8 live rows of the M=16 tile");
  DS_TRACE_AT(2, 0);
  cg::cluster_group cluster = cg::this_cluster();
  const int split = (int)cluster.block_rank();
  const CacheView &c = p.c;
  const int unit = blockIdx.y;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int n_sel = p.rowid ? min(p.k, c.seq_lens[b]) : c.seq_lens[b];
  const int row0 = min(split * p.rows_per_cta, n_sel);
  const int row1 = min(row0 + p.rows_per_cta, n_sel);

  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  uint8_t *wst = smem + (size_t)warp * kMmaStages * STAGE;
  uint32_t *rowids = reinterpret_cast<uint32_t *>(smem + SM::RINGB) + warp * kSub;

  const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)h * G) * D;
  const int32_t *rid = p.rowid ? p.rowid + (size_t)unit * p.k : nullptr;
  const uint8_t *kp = (const uint8_t *)c.k_pool;
  const uint8_t *vp = (const uint8_t *)c.v_pool;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const float scale = p.scale_log2;

  // Q as the A operand (rows = heads; rows >= G and the upper 8 are zero)
  uint32_t qa[NKS][2];
#pragma unroll
  for (int kk = 0; kk < NKS; ++kk) {
    if (gq < G) {
      qa[kk][0] = *reinterpret_cast<const uint32_t *>(qb + (size_t)gq * D + kk * 16 + 2 * tq);
      qa[kk][1] = *reinterpret_cast<const uint32_t *>(qb + (size_t)gq * D + kk * 16 + 8 + 2 * tq);
    } else {
      qa[kk][0] = 0u;
      qa[kk][1] = 0u;
    }
  }
  float o[NDT][4];
#pragma unroll
  for (int nd = 0; nd < NDT; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  wait_inputs(p.ready, unit, n_sel);  // the row ids come from score_select_kernel

  // this warp's contiguous share of the CTA's rows, in sub-tiles of kSub
  int per = (row1 - row0 + kMmaWarps - 1) / kMmaWarps;
  per = (per + kRows - 1) & ~(kRows - 1);
  const int w_lo = min(row0 + warp * per, row1);
  const int w_hi = min(w_lo + per, row1);
  for (int s0 = w_lo; s0 < w_hi; s0 += kSub) {
    const int sn = min(kSub, w_hi - s0);
    __syncwarp();
    load_rowids(rowids, rid, bt, c, h, s0, sn, 32, lane);
    __syncwarp();
    const int nb = (sn + kRows - 1) / kRows;
    if (s0 == w_lo) DS_TRACE_AT(2, 1);

    // batch j: 16 rows x (K, V) x CHN chunks of 16 B; one warp instruction
    // moves 32 chunks.  Rows past the end are zero-filled (src size 0).
    auto issue = [&](int j) {
      uint8_t *st = wst + (j % kMmaStages) * STAGE;
      const int rb = j * kRows;
      const int ch = lane % CHN;
#pragma unroll
      for (int m = 0; m < kRows / RPP; ++m) {
        const int row = m * RPP + lane / CHN;
        const bool rv = rb + row < sn;
        const size_t off = rv ? (size_t)rowids[rb + row] * ROWB + (size_t)ch * 16 : 0;
        const uint32_t dst = smem_u32(st + row * ROWP + ch * 16);
        cp_async16(dst, kp + off, rv ? 16 : 0);
        cp_async16(dst + kRows * ROWP, vp + off, rv ? 16 : 0);
      }
    };

#pragma unroll
    for (int s = 0; s < kMmaStages - 1; ++s) {
      if (s < nb) issue(s);
      cp_async_commit();
    }
    for (int j = 0; j < nb; ++j) {
      if (j + kMmaStages - 1 < nb) issue(j + kMmaStages - 1);
      cp_async_commit();
      cp_async_wait<kMmaStages - 1>();
      __syncwarp();
      const uint8_t *st = wst + (j % kMmaStages) * STAGE;
      const int nvalid = min(kRows, sn - j * kRows);

      // ---- S^T = Q K^T : sf[nt] holds S[head gq][row nt*8 + 2tq + {0,1}]
      float sf[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        const int mi = lane >> 3;
        const int krow = (mi >> 1) * 8 + (lane & 7);
        const uint32_t kaddr = smem_u32(st + krow * ROWP + (mi & 1) * 16);
#pragma unroll
        for (int kk = 0; kk < NKS; ++kk) {
          uint32_t b00, b01, b10, b11;
          ldmatrix_x4(kaddr + kk * 32, b00, b01, b10, b11);
          const uint32_t a[4] = {qa[kk][0], 0u, qa[kk][1], 0u};
          Mma<T>::run(sf[0], a, b00, b01);
          Mma<T>::run(sf[1], a, b10, b11);
        }
      }
      // ---- online softmax (base 2) for head gq over the 16 rows
      float pv[2][2];
      float bmax = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = nt * 8 + 2 * tq + e;
          pv[nt][e] = r < nvalid ? sf[nt][e] * scale : -INFINITY;
          bmax = fmaxf(bmax, pv[nt][e]);
        }
      bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 1));
      bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 2));
      const float mnew = fmaxf(m_run, bmax);
      float alpha = 1.f, psum = 0.f;
      if (mnew == -INFINITY) {
        pv[0][0] = pv[0][1] = pv[1][0] = pv[1][1] = 0.f;
      } else {
        alpha = exp2f(m_run - mnew);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            pv[nt][e] = exp2f(pv[nt][e] - mnew);
            psum += pv[nt][e];
          }
      }
      l_run = l_run * alpha + psum;
      m_run = mnew;
#pragma unroll
      for (int nd = 0; nd < NDT; ++nd) {
        o[nd][0] *= alpha;
        o[nd][1] *= alpha;
      }
      // ---- O += P V
      // P as hi + lo 16-bit pairs (see decode.cu): ~16 significant bits in PV
      const uint32_t ph0 = pack2<T>(pv[0][0], pv[0][1]), ph1 = pack2<T>(pv[1][0], pv[1][1]);
      const float2 f0 = Elem<T>::unpack2(ph0), f1 = Elem<T>::unpack2(ph1);
      const uint32_t pa[4] = {ph0, 0u, ph1, 0u};
      const uint32_t pl[4] = {pack2<T>(pv[0][0] - f0.x, pv[0][1] - f0.y), 0u,
                              pack2<T>(pv[1][0] - f1.x, pv[1][1] - f1.y), 0u};
      {
        const int mi = lane >> 3;
        const int vrow = (mi & 1) * 8 + (lane & 7);
        const uint32_t vaddr = smem_u32(st + kRows * ROWP + vrow * ROWP + (mi >> 1) * 16);
#pragma unroll
        for (int nd2 = 0; nd2 < NDT / 2; ++nd2) {
          uint32_t v0, v1, v2, v3;
          ldmatrix_x4_trans(vaddr + nd2 * 32, v0, v1, v2, v3);
          Mma<T>::run(o[2 * nd2], pa, v0, v1);
          Mma<T>::run(o[2 * nd2 + 1], pa, v2, v3);
          Mma<T>::run(o[2 * nd2], pl, v0, v1);
          Mma<T>::run(o[2 * nd2 + 1], pl, v2, v3);
        }
      }
      __syncwarp();  // every lane is done with this stage before it is refilled
    }
    cp_async_wait<0>();
  }
  DS_TRACE_AT(2, 2);

  // ---- warp partials -> CTA partial (smem) -> cluster merge (DSMEM)
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  __syncthreads();
  float *wm = reinterpret_cast<float *>(smem);
  float *wl = wm + kMmaWarps * G;
  float *wo = wl + kMmaWarps * G;
  float *cm = reinterpret_cast<float *>(smem + SM::WPART);
  if (gq < G) {
    if (tq == 0) {
      wm[warp * G + gq] = m_run;
      wl[warp * G + gq] = l_run;
    }
#pragma unroll
    for (int nd = 0; nd < NDT; ++nd) {
      *reinterpret_cast<float2 *>(wo + (warp * G + gq) * D + nd * 8 + 2 * tq) = make_float2(o[nd][0], o[nd][1]);
    }
  }
  __syncthreads();
  warp_merge<D, G>(wm, wl, wo, kMmaWarps, cm, kMmaThreads);
  if (cluster.num_blocks() > 1) {
    cluster.sync();  // every CTA's partial is complete and visible
    DS_TRACE_AT(2, 3);
    cluster_merge<T, D, G>(cluster, cm, p, b, h, kMmaThreads);
  } else {  // single CTA per unit: normalise and store directly
    __syncthreads();
    T *out = (T *)p.out + ((size_t)b * c.Hq + (size_t)h * G) * D;
    for (int i = tid; i < G * D; i += kMmaThreads) {
      const int g = i / D;
      out[i] = Elem<T>::from_f(cm[g] == -INFINITY ? 0.f : cm[2 * G + i] / cm[G + g]);
    }
    if (p.ready && tid == 0) p.ready[unit] = 0u;  // consumed (every warp passed its loads)
  }
  DS_TRACE_AT(2, 4);
}

// ------------------------------------------------------------ dispatch
// 16-bit types take the tensor-core kernel, fp32 the CUDA-core one.
template <typename T, int D, int G>
struct AttnImpl {
  static constexpr int kThreads = kMmaThreads;
  static constexpr int kSmem = MmaSmem<T, D, G>::BYTES;
  static void (*kernel())(AttnParams) { return attn_mma_kernel<T, D, G>; }
};
template <int D, int G>
struct AttnImpl<float, D, G> {
  static constexpr int kThreads = kAttnThreads;
  static constexpr int kSmem = AttnSmem<float, D, G>::BYTES;
  static void (*kernel())(AttnParams) { return attn_simt_kernel<float, D, G>; }
};

template <typename T, int D, int G>
static cudaError_t set_attn_attrs() {
  static PerDeviceOnce once;
  return once([] {
    cudaError_t e = cudaFuncSetAttribute(AttnImpl<T, D, G>::kernel(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         AttnImpl<T, D, G>::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(AttnImpl<T, D, G>::kernel(), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  });
}

template <typename T, int D, int G>
static cudaLaunchConfig_t attn_cfg(int ns, int units, cudaLaunchAttribute *a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ns, units);
  cfg.blockDim = dim3(AttnImpl<T, D, G>::kThreads);
  cfg.dynamicSmemBytes = AttnImpl<T, D, G>::kSmem;
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = ns;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  return cfg;
}

template <typename T, int D, int G>
static AttnGeom attn_geom_t(const ds_cache *c, int n_rows) {
  AttnGeom best{};
  best.nsplit = 0;
  if (set_attn_attrs<T, D, G>() != cudaSuccess) return best;
  const int units = c->batch * c->num_kv_heads;
  double best_cost = 1e300;
  for (int ns = 1; ns <= kMaxSplit; ++ns) {
    int rows = (n_rows + ns - 1) / ns;
    rows = (rows + kRows - 1) & ~(kRows - 1);
    if ((n_rows + rows - 1) / rows != ns) continue;  // would leave an empty split
    cudaLaunchAttribute a[2];
    cudaLaunchConfig_t cfg = attn_cfg<T, D, G>(ns, units, a);
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, AttnImpl<T, D, G>::kernel(), &cfg) != cudaSuccess || ncl < 1) {
      cudaGetLastError();
      continue;
    }
    const double waves = (double)units / ncl;
    // time ~ (#waves, a partial last wave counted fully) x rows per CTA, plus
    // a fixed per-CTA cost (prologue, merge) of ~96 rows
    const double cost = ceil(waves) * (rows + 96.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best.nsplit = ns;
      best.rows_per_cta = rows;
    }
  }
  best.threads = AttnImpl<T, D, G>::kThreads;
  best.smem = AttnImpl<T, D, G>::kSmem;
  return best;
}

template <typename T, int D, int G>
static cudaError_t launch_attn_t(const AttnParams &p, const AttnGeom &g, int units, cudaStream_t st) {
  cudaError_t e = set_attn_attrs<T, D, G>();
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute a[2];
  cudaLaunchConfig_t cfg = attn_cfg<T, D, G>(g.nsplit, units, a);
  cfg.stream = st;
  return cudaLaunchKernelEx(&cfg, AttnImpl<T, D, G>::kernel(), p);
}

template <template <typename, int, int> class OP, typename R, typename... A>
static R dispatch(const ds_cache *c, A... args) {
  const int G = c->num_q_heads / c->num_kv_heads;
#define DS_G(T, D)                                      \
  switch (G) {                                          \
    case 1: return OP<T, D, 1>::run(c, args...);        \
    case 2: return OP<T, D, 2>::run(c, args...);        \
    case 4: return OP<T, D, 4>::run(c, args...);        \
    default: return OP<T, D, 8>::run(c, args...);       \
  }
#define DS_D(T)                 \
  if (c->head_dim == 64) {      \
    DS_G(T, 64)                 \
  } else {                      \
    DS_G(T, 128)                \
  }
  switch (c->dtype) {
    case DS_BF16: DS_D(__nv_bfloat16)
    case DS_FP16: DS_D(__half)
    default: DS_D(float)
  }
#undef DS_D
#undef DS_G
}

template <typename T, int D, int G>
struct GeomOp {
  static AttnGeom run(const ds_cache *c, int n) { return attn_geom_t<T, D, G>(c, n); }
};
template <typename T, int D, int G>
struct LaunchOp {
  static cudaError_t run(const ds_cache *c, const AttnParams *p, const AttnGeom *g, cudaStream_t st) {
    return launch_attn_t<T, D, G>(*p, *g, c->batch * c->num_kv_heads, st);
  }
};

AttnGeom attn_geom(const ds_cache *c, int n_rows) { return dispatch<GeomOp, AttnGeom>(c, n_rows); }

cudaError_t launch_attn(const ds_cache *c, const AttnParams &p, const AttnGeom &g, cudaStream_t st) {
  return dispatch<LaunchOp, cudaError_t>(c, &p, &g, st);
}

}  // namespace ds
