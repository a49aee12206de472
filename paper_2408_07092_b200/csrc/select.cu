// select.cu -- a1..a3 of Algorithm 1: label-score GEMV and exact
// top-k selection, fused in one kernel (score_select_kernel, grid chunks x
// units, 512 threads; see the kernel's comment for the three phases).
//   a1  q_lab[j] = sum_g q[b][hG+g][C[h][j]]      (fp32, g order; reading R3)
//   a2  s_hat[t] = fma-chain_j(q_lab[j], L[t][j])  (fp32, j ascending, no
//       1/sqrt(d); reading R2), streamed from the contiguous label cache with
//       eight 128-bit loads in flight per thread (one row = r*e = 16 B at
//       r=8 / 16-bit) into a monotone u32 order key (-0 == +0) in smem.
//   a3  i = argtopk(s_hat, k): exact, ties to the lower index, ascending
//       (reading R6).  Each chunk emits a candidate superset of its share of
//       the global top-k; the unit's last-arriving CTA selects exactly among
//       them (MSB radix 12+12+8 bits, equal keys by token order) and writes
//       the index list with each token's pool row id.  s_hat never leaves the
//       chip; the candidates (~k + a histogram bin per chunk) stay in L2.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

constexpr int kScoreThreads = 512;
constexpr int kScoreWarps = kScoreThreads / 32;
constexpr int kScoreUnroll = 8;
constexpr int kMaxChunks = 16;       // score CTAs per unit
constexpr int kMaxChunkLen = 16384;  // tokens per score CTA (keys kept in smem)
constexpr int kMaxDynSmem = 200 * 1024;
constexpr int kMaxR = 256;
constexpr int kDigitBits = 12;
constexpr int kBins = 1 << kDigitBits;
constexpr int kShift1 = 32 - kDigitBits;  // level-1 digit: top 12 key bits

// per-unit stride of the candidate workspace (>= nchunks * chunk for any geometry)
__host__ __device__ __forceinline__ size_t cand_stride(int smax) {
  return (size_t)smax + (size_t)kMaxChunks * 256;
}

// ------------------------------------------------------------ helpers
// Block-wide exclusive prefix of one u32 per thread (NT threads); *total =
// sum.  Two shuffle levels (warp, then warp 0 over the warp totals): 2
// barriers, no serial smem walks.  warp_tot needs NT/32 + 1 entries.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *warp_tot, uint32_t *total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // warp_tot may still be read by a previous scan
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t t = lane < NW ? warp_tot[lane] : 0u;
    uint32_t y = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    if (lane < NW) warp_tot[lane] = y - t;
    if (lane == NW - 1) warp_tot[NW] = y;
  }
  __syncthreads();
  *total = warp_tot[NW];
  return warp_tot[warp] + x - v;
}

// Boundary digit of a histogram bins[nb] (nb a multiple of NT): with `need`
// keys wanted from the top, the digit d with above(d) < need <= above(d) +
// bins[d]; every thread gets (d, above(d), bins[d]).
template <int NT>
__device__ __forceinline__ void find_boundary(const uint32_t *bins, int nb, uint32_t need, uint32_t *warp_tot,
                                              uint32_t *state, uint32_t &d, uint32_t &above, uint32_t &cnt) {
  const int per = nb / NT;  // thread t owns digits nb-1-per*t-j, descending
  uint32_t s = 0;
  for (int j = 0; j < per; ++j) s += bins[nb - 1 - per * (int)threadIdx.x - j];
  uint32_t tot;
  uint32_t run = block_excl_scan<NT>(s, warp_tot, &tot);
  for (int j = 0; j < per; ++j) {
    const int dd = nb - 1 - per * (int)threadIdx.x - j;
    const uint32_t v = bins[dd];
    if (run < need && run + v >= need) {
      state[0] = dd;
      state[1] = run;
      state[2] = v;
    }
    run += v;
  }
  __syncthreads();
  d = state[0];
  above = state[1];
  cnt = state[2];
  __syncthreads();
}

// ------------------------------------------------------------------ A
template <typename T, int R>
__device__ __forceinline__ float label_score(const T *__restrict__ row, const float *ql, int r) {
  float s = 0.0f;
  if constexpr (R > 0 && (R * sizeof(T)) % 16 == 0) {
    constexpr int NV = R * sizeof(T) / 16;
    uint4 v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = __ldg(reinterpret_cast<const uint4 *>(row) + i);
    const T *e = reinterpret_cast<const T *>(v);
#pragma unroll
    for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[j]), s);
  } else {
    for (int j = 0; j < r; ++j) s = fmaf(ql[j], Elem<T>::to_f(row[j]), s);
  }
  return s;
}

// Candidate sources for the unit's exact selection: staged in shared memory
// (the usual case) or read in place from the per-chunk segments in global
// memory (tie-heavy boundaries with more candidates than fit).
struct StagedSrc {
  const uint2 *a;
  __device__ __forceinline__ uint2 get(int s) const { return a[s]; }
};
struct GlobalSrc {
  const uint2 *g;
  const uint32_t *seg;
  int chunk;
  __device__ __forceinline__ uint2 get(int s) const {
    int q = 0;
    while ((int)seg[q + 1] <= s) ++q;
    return __ldcg(g + (size_t)q * chunk + (s - (int)seg[q]));
  }
};

struct SelScratch {
  uint32_t *bins;      // [kBins]
  uint32_t *warp_tot;  // [NW + 1]
  uint32_t *state;     // [4]
};

// Exact top-k_eff of T candidates (ascending token order) with ties to the
// lower index: MSB radix over 12 + 12 + 8 key bits for the k-th key, then
// one ordered pass writes the selected tokens (ascending) and their pool row
// ids.  NT threads.
template <int NT, class Src>
__device__ __forceinline__ void select_core(const Src &src, int T, uint32_t keff, const SelScratch &sc,
                                            int32_t *idx_out, int32_t *rid_out, const CacheView &c, int b,
                                            int h) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t need = keff, prefix = 0, mask = 0;
  bool whole = false;  // the boundary bin is taken entirely
  for (int lv = 0; lv < 3 && !whole; ++lv) {
    const int sh = lv == 0 ? 20 : (lv == 1 ? 8 : 0), nb = lv < 2 ? 4096 : 256;
    const uint32_t wm = (uint32_t)nb - 1u;
    const int nbz = nb < NT ? NT : nb;
    for (int i = tid; i < nbz; i += NT) sc.bins[i] = 0;
    __syncthreads();
#pragma unroll 4
    for (int s = tid; s < T; s += NT) {
      const uint32_t key = src.get(s).x;
      if ((key & mask) == prefix) atomicAdd(&sc.bins[(key >> sh) & wm], 1u);
    }
    __syncthreads();
    uint32_t d, above, cnt;
    find_boundary<NT>(sc.bins, nbz, need, sc.warp_tot, sc.state, d, above, cnt);
    need -= above;
    prefix |= d << sh;
    mask |= wm << sh;
    whole = cnt == need;
  }
  // ordered selection: masked key > prefix, or == prefix and (the whole bin
  // is taken, or it is among the first `need` equal keys in token order)
  int per = (T + NW - 1) / NW;
  per = (per + 31) & ~31;
  const int w0 = min(warp * per, T), w1 = min(w0 + per, T);
  const uint32_t lt = lanemask_lt();
  uint32_t tot, eq_base = 0;
  if (!whole) {
    uint32_t weq = 0;
#pragma unroll 4
    for (int base = w0; base < w1; base += 32) {
      const int s = base + lane;
      weq += __popc(__ballot_sync(0xffffffffu, s < w1 && (src.get(s).x & mask) == prefix));
    }
    eq_base = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? weq : 0u, sc.warp_tot, &tot), 0);
  }
  uint32_t wtake = 0, run = eq_base;
#pragma unroll 4
  for (int base = w0; base < w1; base += 32) {
    const int s = base + lane;
    const uint32_t km = s < w1 ? (src.get(s).x & mask) : 0u;
    const bool gt = s < w1 && km > prefix, eq = s < w1 && km == prefix;
    const uint32_t em = __ballot_sync(0xffffffffu, eq);
    const bool take = gt || (eq && (whole || run + __popc(em & lt) < need));
    wtake += __popc(__ballot_sync(0xffffffffu, take));
    run += __popc(em);
  }
  uint32_t pos = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? wtake : 0u, sc.warp_tot, &tot), 0);
  run = eq_base;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const bool pow2 = (c.P & (c.P - 1)) == 0;
  const int psh = __ffs(c.P) - 1;
#pragma unroll 2
  for (int base = w0; base < w1; base += 32) {
    const int s = base + lane;
    uint2 e = make_uint2(0u, 0u);
    if (s < w1) e = src.get(s);
    const uint32_t km = e.x & mask;
    const bool gt = s < w1 && km > prefix, eq = s < w1 && km == prefix;
    const uint32_t em = __ballot_sync(0xffffffffu, eq);
    const bool take = gt || (eq && (whole || run + __popc(em & lt) < need));
    const uint32_t tm = __ballot_sync(0xffffffffu, take);
    if (take) {
      const uint32_t o = pos + __popc(tm & lt);
      const int t = (int)e.y;
      const int pg = pow2 ? (t >> psh) : t / c.P;
      const int sl = pow2 ? (t & (c.P - 1)) : t - pg * c.P;
      idx_out[o] = t;
      rid_out[o] = (int32_t)(((uint32_t)__ldg(bt + pg) * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P + (uint32_t)sl);
    }
    pos += __popc(tm);
    run += __popc(em);
  }
}

// select_core for candidates staged in shared memory (16-B aligned, padded
// by 4 entries): warp w owns 128-candidate blocks; lane l handles candidates
// 4l..4l+3 of a block (two 128-bit loads), prefix sums by warp shuffles.
template <int NT>
__device__ __forceinline__ void select_core_staged(const uint2 *cand, int T, uint32_t keff, const SelScratch &sc,
                                                   int32_t *idx_out, int32_t *rid_out, const CacheView &c, int b,
                                                   int h) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int per = (T + NW - 1) / NW;
  per = (per + 127) & ~127;
  const int w0 = min(warp * per, T), w1 = min(w0 + per, T);
  auto load4 = [&](int base, uint32_t (&k)[4], uint32_t (&t)[4]) {
    const uint4 a = *reinterpret_cast<const uint4 *>(cand + base + 4 * lane);
    const uint4 bq = *reinterpret_cast<const uint4 *>(cand + base + 4 * lane + 2);
    k[0] = a.x; t[0] = a.y; k[1] = a.z; t[1] = a.w;
    k[2] = bq.x; t[2] = bq.y; k[3] = bq.z; t[3] = bq.w;
  };
  auto warp_excl = [&](uint32_t v, uint32_t &total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
  };
  uint32_t need = keff, prefix = 0, mask = 0;
  bool whole = false;
  for (int lv = 0; lv < 3 && !whole; ++lv) {
    const int sh = lv == 0 ? 20 : (lv == 1 ? 8 : 0), nb = lv < 2 ? 4096 : 256;
    const uint32_t wm = (uint32_t)nb - 1u;
    const int nbz = nb < NT ? NT : nb;
    for (int i = tid; i < nbz; i += NT) sc.bins[i] = 0;
    __syncthreads();
    for (int base = w0; base < w1; base += 128) {
      uint32_t k[4], t[4];
      load4(base, k, t);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (base + 4 * lane + e < w1 && (k[e] & mask) == prefix) atomicAdd(&sc.bins[(k[e] >> sh) & wm], 1u);
    }
    __syncthreads();
    uint32_t d, above, cnt;
    find_boundary<NT>(sc.bins, nbz, need, sc.warp_tot, sc.state, d, above, cnt);
    need -= above;
    prefix |= d << sh;
    mask |= wm << sh;
    whole = cnt == need;
  }
  uint32_t tot, eq_base = 0;
  if (!whole) {  // equal keys beyond the first `need` are dropped: their ordinals
    uint32_t weq = 0;
    for (int base = w0; base < w1; base += 128) {
      uint32_t k[4], t[4];
      load4(base, k, t);
#pragma unroll
      for (int e = 0; e < 4; ++e) weq += base + 4 * lane + e < w1 && (k[e] & mask) == prefix;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) weq += __shfl_xor_sync(0xffffffffu, weq, o);
    eq_base = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? weq : 0u, sc.warp_tot, &tot), 0);
  }
  // per lane: take flags for its 4 candidates (gt, or eq within the first `need`)
  auto takes = [&](int base, const uint32_t (&k)[4], uint32_t &run, bool (&tk)[4]) {
    bool eq[4];
    uint32_t ne = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool in = base + 4 * lane + e < w1;
      const uint32_t km = k[e] & mask;
      eq[e] = in && km == prefix;
      tk[e] = in && km > prefix;
      ne += eq[e];
    }
    uint32_t etot;
    uint32_t eo = run + (whole ? 0u : warp_excl(ne, etot));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      tk[e] = tk[e] || (eq[e] && (whole || eo < need));
      eo += eq[e];
    }
    if (!whole) run += etot;
  };
  uint32_t wtake = 0, run = eq_base;
  for (int base = w0; base < w1; base += 128) {
    uint32_t k[4], t[4];
    bool tk[4];
    load4(base, k, t);
    takes(base, k, run, tk);
    wtake += tk[0] + tk[1] + tk[2] + tk[3];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) wtake += __shfl_xor_sync(0xffffffffu, wtake, o);
  uint32_t pos = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? wtake : 0u, sc.warp_tot, &tot), 0);
  run = eq_base;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const bool pow2 = (c.P & (c.P - 1)) == 0;
  const int psh = __ffs(c.P) - 1;
  for (int base = w0; base < w1; base += 128) {
    uint32_t k[4], t[4];
    bool tk[4];
    load4(base, k, t);
    takes(base, k, run, tk);
    const uint32_t nt = tk[0] + tk[1] + tk[2] + tk[3];
    uint32_t ttot;
    uint32_t o = pos + warp_excl(nt, ttot);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (tk[e]) {
        const int tok = (int)t[e];
        const int pg = pow2 ? (tok >> psh) : tok / c.P;
        const int sl = pow2 ? (tok & (c.P - 1)) : tok - pg * c.P;
        idx_out[o] = tok;
        rid_out[o] = (int32_t)(((uint32_t)__ldg(bt + pg) * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P +
                               (uint32_t)sl);
        ++o;
      }
    pos += ttot;
  }
}

// Exact top-k of T staged candidates (ascending token order), fast path:
// level 1 = 4096 linear fp32 bins over [lo, hi] (the candidates' key range),
// so the boundary bin holds only a few keys; the boundary is found by one warp
// over a 64-bin coarse then a 64-bin fine scan; the boundary bin's members are
// ranked exactly by (key desc, token asc) by one warp; one ordered pass writes
// the selected tokens and their pool row ids.  Returns false (nothing
// written) when the boundary bin is too crowded (ties): the caller then runs
// the generic radix path.
constexpr int kMaxMembers = 256;
struct FastScratch {
  uint32_t *fine;      // [4096]
  uint32_t *coarse;    // [64]
  uint2 *members;      // [kMaxMembers] (key, slot)
  uint32_t *selbits;   // [T/32 + 1] selected boundary members, by slot
  uint32_t *warp_tot;  // [NW + 1]
  uint32_t *state;     // [8]
};

template <int NT>
__device__ __forceinline__ bool select_fast(const uint2 *cand, int T, uint32_t keff, uint32_t lo_key,
                                            uint32_t hi_key, const FastScratch &sc, int32_t *idx_out,
                                            int32_t *rid_out, const int32_t *btrow, const CacheView &c, int h) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float lo = key_to_float(lo_key), hi = key_to_float(hi_key);
  const float scale = 4096.0f / (hi - lo);
  auto binof = [&](uint32_t key) -> int {
    const float x = fminf(fmaxf((key_to_float(key) - lo) * scale, 0.0f), 4095.0f);
    return (int)x;
  };
  for (int i = tid; i < 4096; i += NT) sc.fine[i] = 0;
  if (tid < 64) sc.coarse[tid] = 0;
  for (int i = tid; i <= T / 32; i += NT) sc.selbits[i] = 0;
  if (tid == 0) sc.state[4] = 0;
  __syncthreads();
#pragma unroll 4
  for (int s = tid; s < T; s += NT) {
    const int bn = binof(cand[s].x);
    atomicAdd(&sc.fine[bn], 1u);
    atomicAdd(&sc.coarse[bn >> 6], 1u);
  }
  __syncthreads();
  if (warp == 0) {  // coarse then fine boundary, descending bins
    uint32_t above = 0;
    int cb = 0;
    {
      const uint32_t a = sc.coarse[63 - 2 * lane], bq = sc.coarse[62 - 2 * lane];
      uint32_t incl = a + bq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t ex = incl - a - bq;
      const bool h0 = ex < keff && ex + a >= keff;
      const bool h1 = !h0 && ex + a < keff && ex + a + bq >= keff;
      const uint32_t m = __ballot_sync(0xffffffffu, h0 || h1);
      const int src = __ffs(m) - 1;
      const bool sh1 = __shfl_sync(0xffffffffu, h1, src);
      cb = 63 - 2 * src - (sh1 ? 1 : 0);
      above = __shfl_sync(0xffffffffu, sh1 ? ex + a : ex, src);
    }
    {
      const int f0 = cb * 64;
      const uint32_t a = sc.fine[f0 + 63 - 2 * lane], bq = sc.fine[f0 + 62 - 2 * lane];
      uint32_t incl = a + bq;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t ex = above + incl - a - bq;
      const bool h0 = ex < keff && ex + a >= keff;
      const bool h1 = !h0 && ex + a < keff && ex + a + bq >= keff;
      const uint32_t m = __ballot_sync(0xffffffffu, h0 || h1);
      const int src = __ffs(m) - 1;
      if (lane == src) {
        sc.state[0] = f0 + 63 - 2 * lane - (h1 ? 1 : 0);
        sc.state[1] = h1 ? ex + a : ex;
        sc.state[2] = h1 ? bq : a;
      }
    }
  }
  __syncthreads();
  const int b1 = (int)sc.state[0];
  const uint32_t need = keff - sc.state[1], cnt = sc.state[2];
  const bool whole = cnt == need;
  if (!whole) {
    if (cnt > (uint32_t)kMaxMembers) return false;
    // members of the boundary bin -> list, ranked exactly by warp 0
#pragma unroll 4
    for (int s = tid; s < T; s += NT) {
      const uint32_t key = cand[s].x;
      if (binof(key) == b1) sc.members[atomicAdd(&sc.state[4], 1u)] = make_uint2(key, (uint32_t)s);
    }
    __syncthreads();
    if (warp == 0) {
      const int m = (int)sc.state[4];
      for (int i = lane; i < m; i += 32) {
        const uint2 me = sc.members[i];
        uint32_t rank = 0;
        for (int j = 0; j < m; ++j) {
          const uint2 o = sc.members[j];
          rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);  // slot order == token order
        }
        if (rank < need) atomicOr(&sc.selbits[me.y >> 5], 1u << (me.y & 31));
      }
    }
    __syncthreads();
  }
  // ---- ordered pass: warp w owns a contiguous slot range
  int per = (T + NW - 1) / NW;
  per = (per + 31) & ~31;
  const int w0 = min(warp * per, T), w1 = min(w0 + per, T);
  auto take = [&](int s, uint32_t key) {
    const int bn = binof(key);
    return bn > b1 || (bn == b1 && (whole || ((sc.selbits[s >> 5] >> (s & 31)) & 1u)));
  };
  uint32_t wt = 0;
#pragma unroll 4
  for (int base = w0; base < w1; base += 32) {
    const int s = base + lane;
    wt += __popc(__ballot_sync(0xffffffffu, s < w1 && take(s, cand[s].x)));
  }
  uint32_t tot;
  uint32_t pos = __shfl_sync(0xffffffffu, block_excl_scan<NT>(lane == 0 ? wt : 0u, sc.warp_tot, &tot), 0);
  const uint32_t lt = lanemask_lt();
  const bool pow2 = (c.P & (c.P - 1)) == 0;
  const int psh = __ffs(c.P) - 1;
#pragma unroll 2
  for (int base = w0; base < w1; base += 32) {
    const int s = base + lane;
    uint2 e = make_uint2(0u, 0u);
    if (s < w1) e = cand[s];
    const bool tk = s < w1 && take(s, e.x);
    const uint32_t tm = __ballot_sync(0xffffffffu, tk);
    if (tk) {
      const uint32_t o = pos + __popc(tm & lt);
      const int t = (int)e.y;
      const int pg = pow2 ? (t >> psh) : t / c.P;
      const int sl = pow2 ? (t & (c.P - 1)) : t - pg * c.P;
      idx_out[o] = t;
      rid_out[o] = (int32_t)(((uint32_t)btrow[pg] * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P + (uint32_t)sl);
    }
    pos += __popc(tm);
  }
  return true;
}

// Fused a1 + a2 + a3.  Grid (chunks, units), kScoreThreads threads.
//   1. stream this chunk's label rows -> keys (smem) + 12-bit digit histogram
//   2. emit, in token order, every token whose digit is >= the digit bounding
//      the chunk's local top-k: a superset of the chunk's share of the unit's
//      global top-k (any global top-k token is in its chunk's top-k)
//   3. the last CTA of the unit to arrive (global counter) selects exactly
//      among the unit's candidates, writes the index list and row ids, resets
//      the counter and publishes ready[unit] for the attention kernel
// counter[] and ready[] are zero between calls (zero-filled workspace on first
// use; restored by the last arriver and by the attention kernel).
template <typename T, int R>
__global__ void __launch_bounds__(kScoreThreads, 2) score_select_kernel(ScoreParams p) {
  extern __shared__ __align__(16) uint32_t keys[];  // [chunk] order keys; then staged candidates
  __shared__ float qlab[kMaxR];
  __shared__ __align__(16) uint32_t hist[kBins];
  __shared__ uint32_t warp_tot[kScoreWarps + 1], state[8], seg[kMaxChunks + 1];
  __shared__ uint32_t coarse[64], mm[2];
  __shared__ __align__(16) uint2 members[kMaxMembers];
  __shared__ int last;
  const CacheView &c = p.c;
  const int unit = blockIdx.y, part = blockIdx.x;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = c.seq_lens[b];
  const int t0 = part * p.chunk;
  const int nloc = min(p.chunk, n - t0);
  const int r = R > 0 ? R : c.r;
  const int keff = min(p.k, n);
  const int nparts = (n + p.chunk - 1) / p.chunk;
  DS_TRACE_AT(0, 0);
  for (int i = tid; i < kBins; i += kScoreThreads) hist[i] = 0;
  pdl_wait();  // the label rows may come from the preceding append
  pdl_trigger();
  if (n <= 0) {  // empty sequence: nothing selected (the attention writes zeros)
    if (part == 0 && !p.scores)
      for (int i = tid; i < p.k; i += kScoreThreads) {
        p.idx[(size_t)unit * p.k + i] = -1;
        p.rowid[(size_t)unit * p.k + i] = -1;
      }
    return;
  }
  if (nloc <= 0) return;
  for (int j = tid; j < r; j += kScoreThreads) {  // a1
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
  const float *qs = R > 0 ? ql : qlab;
  const T *lab = (const T *)c.label + (((size_t)b * c.Hkv + h) * c.Smax + t0) * (size_t)c.r;

  if (p.scores) {  // diagnostics entry (ds_approx_scores): s_hat to HBM
    float *so = p.scores + (size_t)unit * c.Smax + t0;
    for (int i = tid; i < nloc; i += kScoreThreads) so[i] = label_score<T, R>(lab + (size_t)i * r, qs, r);
    return;
  }
  // ---- a2: stream the label: keys + digit histogram
  int i0 = tid;
  if constexpr (R > 0 && R * sizeof(T) == 16) {
    constexpr int U = kScoreUnroll;
    for (; i0 + (U - 1) * kScoreThreads < nloc; i0 += U * kScoreThreads) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = __ldg(reinterpret_cast<const uint4 *>(lab) + (size_t)(i0 + u * kScoreThreads));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const T *e = reinterpret_cast<const T *>(&v[u]);
        float s = 0.0f;
#pragma unroll
        for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[j]), s);
        const uint32_t k0 = order_key(s);
        keys[i0 + u * kScoreThreads] = k0;
        atomicAdd(&hist[k0 >> kShift1], 1u);
      }
    }
  }
  for (int i = i0; i < nloc; i += kScoreThreads) {
    const uint32_t k0 = order_key(label_score<T, R>(lab + (size_t)i * r, qs, r));
    keys[i] = k0;
    atomicAdd(&hist[k0 >> kShift1], 1u);
  }
  __syncthreads();
  DS_TRACE_AT(0, 1);

  // ---- local candidates (ordered emission; warp w owns a contiguous range)
  uint32_t dmin = 0;
  if (keff < nloc) {
    uint32_t above, cnt;
    find_boundary<kScoreThreads>(hist, kBins, (uint32_t)keff, warp_tot, state, dmin, above, cnt);
  }
  {
    // warp w owns 128-token blocks [w0, w1); lane l holds tokens 4l..4l+3 of
    // a block (one 128-bit smem load); positions by warp-shuffle prefix sums
    int per = (nloc + kScoreWarps - 1) / kScoreWarps;
    per = (per + 127) & ~127;
    const int w0 = min(warp * per, nloc), w1 = min(w0 + per, nloc);
    uint32_t mine = 0, kmin = 0xffffffffu, kmax = 0u;
    if (tid == 0) {
      mm[0] = 0xffffffffu;
      mm[1] = 0u;
    }
#pragma unroll 2
    for (int base = w0; base < w1; base += 128) {
      const int i = base + 4 * lane;
      const uint4 kv = *reinterpret_cast<const uint4 *>(keys + i);
      const uint32_t kk[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (i + e < w1 && (kk[e] >> kShift1) >= dmin) {
          ++mine;
          kmin = min(kmin, kk[e]);
          kmax = max(kmax, kk[e]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mine += __shfl_xor_sync(0xffffffffu, mine, o);
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
      atomicMin(&mm[0], kmin);
      atomicMax(&mm[1], kmax);
    }
    uint32_t tot;
    uint32_t pos = __shfl_sync(0xffffffffu, block_excl_scan<kScoreThreads>(lane == 0 ? mine : 0u, warp_tot, &tot), 0);
    uint2 *out = p.cand + (size_t)unit * cand_stride(c.Smax) + (size_t)part * p.chunk;
#pragma unroll 2
    for (int base = w0; base < w1; base += 128) {
      const int i = base + 4 * lane;
      const uint4 kv = *reinterpret_cast<const uint4 *>(keys + i);
      const uint32_t kk[4] = {kv.x, kv.y, kv.z, kv.w};
      bool sel[4];
      uint32_t cnt = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sel[e] = i + e < w1 && (kk[e] >> kShift1) >= dmin;
        cnt += sel[e];
      }
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t o = pos + incl - cnt;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (sel[e]) out[o++] = make_uint2(kk[e], (uint32_t)(t0 + i + e));
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncthreads();
    if (tid == 0) {
      p.cand_count[unit * kMaxChunks + part] = tot;
      p.cand_minmax[(unit * kMaxChunks + part) * 2] = mm[0];
      p.cand_minmax[(unit * kMaxChunks + part) * 2 + 1] = mm[1];
    }
  }
  DS_TRACE_AT(0, 2);

  // ---- arrival: the unit's last CTA performs the selection
  __syncthreads();
  if (tid == 0) {
    __threadfence();  // release this CTA's candidates
    last = atomicAdd(p.counter + unit, 1u) == (uint32_t)(nparts - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();  // acquire the other chunks' candidates
  if (tid == 0) {
    uint32_t o = 0, lo = 0xffffffffu, hi = 0u;
    for (int q = 0; q < nparts; ++q) {
      seg[q] = o;
      o += __ldcg(p.cand_count + unit * kMaxChunks + q);
      lo = min(lo, __ldcg(p.cand_minmax + (unit * kMaxChunks + q) * 2));
      hi = max(hi, __ldcg(p.cand_minmax + (unit * kMaxChunks + q) * 2 + 1));
    }
    seg[nparts] = o;
    mm[0] = lo;
    mm[1] = hi;
  }
  __syncthreads();
  const int ncand = (int)seg[nparts];
  const uint2 *gc = p.cand + (size_t)unit * cand_stride(c.Smax);
  int32_t *idx_out = p.idx + (size_t)unit * p.k;
  int32_t *rid_out = p.rowid + (size_t)unit * p.k;
  for (int i = keff + tid; i < p.k; i += kScoreThreads) {  // positions >= k_eff
    idx_out[i] = -1;
    rid_out[i] = -1;
  }
  const SelScratch scr{hist, warp_tot, state};
  uint2 *stage = reinterpret_cast<uint2 *>(keys);  // the keys are no longer needed
  int32_t *btrow = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(keys) + (size_t)p.stage_cap * 8);
  uint32_t *selbits = reinterpret_cast<uint32_t *>(btrow + c.maxp);
  bool done = false;
  if (ncand + 128 <= p.stage_cap) {  // vector loads read up to 127 entries past the end
    // the block-table row (row ids) and every chunk's candidates: each thread
    // issues a batch of loads into registers before storing any of them, so
    // the L2 round trips overlap instead of serialising on the smem stores
    {
      const int np = (n + c.P - 1) / c.P;
      const int32_t *bt = c.block_table + (size_t)b * c.maxp;
      constexpr int BU = 8;
      for (int i0 = tid; i0 < np; i0 += BU * kScoreThreads) {
        int32_t v[BU];
#pragma unroll
        for (int u = 0; u < BU; ++u) v[u] = i0 + u * kScoreThreads < np ? __ldg(bt + i0 + u * kScoreThreads) : 0;
#pragma unroll
        for (int u = 0; u < BU; ++u)
          if (i0 + u * kScoreThreads < np) btrow[i0 + u * kScoreThreads] = v[u];
      }
      for (int s0 = tid; s0 < ncand; s0 += BU * kScoreThreads) {
        uint2 v[BU];
#pragma unroll
        for (int u = 0; u < BU; ++u) {
          const int s2 = s0 + u * kScoreThreads;
          if (s2 < ncand) {
            int q = 0;
            while ((int)seg[q + 1] <= s2) ++q;
            v[u] = __ldcg(gc + (size_t)q * p.chunk + (s2 - (int)seg[q]));
          }
        }
#pragma unroll
        for (int u = 0; u < BU; ++u)
          if (s0 + u * kScoreThreads < ncand) stage[s0 + u * kScoreThreads] = v[u];
      }
    }
    __syncthreads();
    DS_TRACE_AT(0, 3);
    const FastScratch fs{hist, coarse, members, selbits, warp_tot, state};
    done = select_fast<kScoreThreads>(stage, ncand, (uint32_t)keff, mm[0], mm[1], fs, idx_out, rid_out, btrow, c, h);
    if (!done) select_core_staged<kScoreThreads>(stage, ncand, (uint32_t)keff, scr, idx_out, rid_out, c, b, h);
  } else {
    select_core<kScoreThreads>(GlobalSrc{gc, seg, p.chunk}, ncand, (uint32_t)keff, scr, idx_out, rid_out, c, b, h);
  }
  DS_TRACE_AT(0, 4);
  // ---- publish
  __syncthreads();
  if (tid == 0) {
    p.counter[unit] = 0u;
    __threadfence();
    atomicExch(p.ready + unit, 1u);
  }
}

// ------------------------------------------------------------- launch
template <typename T, int R>
static cudaError_t launch_score_t(const ScoreParams &p, int units, int nchunks, size_t smem, cudaStream_t st) {
  static const cudaError_t attr = cudaFuncSetAttribute(score_select_kernel<T, R>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  if (attr != cudaSuccess) return attr;
  return PdlLaunch(dim3(nchunks, units), dim3(kScoreThreads), smem, st).run(score_select_kernel<T, R>, p);
}

SelectGeom select_geom(const ds_cache *c, int k) {
  SelectGeom g{};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * c->num_kv_heads;
  // CTAs per unit: enough for one wave at 2 CTAs/SM, but chunks of >= 4k
  // tokens so that each chunk's local top-k superset stays small (~k); each
  // chunk's keys fit in shared memory
  const int per_sm = 2;
  int nch = (per_sm * sms) / units;
  const int kk = k < 1 ? 1 : k;
  const int by_k = c->max_seq_len / (4 * kk);
  if (nch > by_k) nch = by_k;
  const int need = (c->max_seq_len + kMaxChunkLen - 1) / kMaxChunkLen;
  if (nch < need) nch = need;
  nch = nch < 1 ? 1 : (nch > kMaxChunks ? kMaxChunks : nch);
  int chunk = (c->max_seq_len + nch - 1) / nch;
  chunk = (chunk + 255) & ~255;
  g.chunk = chunk;
  g.nchunks = (c->max_seq_len + chunk - 1) / chunk;
  // dynamic smem holds the chunk's keys, then the unit's staged candidates
  // (expected ~nchunks * (k + a bin); the global path covers overflow)
  size_t stage = (size_t)g.nchunks * (kk + kk / 2) + 64;
  // the stage, the block-table row and the bitmap must fit kMaxDynSmem
  const size_t fixed = (size_t)c->max_pages_per_seq * 4 + 4096 + 1024;
  const size_t cap_max = (kMaxDynSmem - fixed) / (8 + 1);
  if (stage > cap_max) stage = cap_max;
  size_t bytes = (size_t)chunk * 4;
  if (stage * 8 > bytes) bytes = stage * 8;
  bytes += 1024;  // 128-bit loads run up to 127 keys / candidates past the end
  g.stage_cap = (int)(bytes / 8);
  // after the stage: the block-table row and the selected-members bitmap
  bytes += (size_t)c->max_pages_per_seq * 4 + ((size_t)g.stage_cap / 32 + 1) * 4;
  g.score_smem = (bytes + 15) & ~(size_t)15;
  g.threads = kScoreThreads;
  return g;
}

size_t select_workspace_cand(const ds_cache *c) {
  return (size_t)c->batch * c->num_kv_heads * cand_stride(c->max_seq_len) * 8;
}
size_t select_workspace_count(const ds_cache *c) { return (size_t)c->batch * c->num_kv_heads * kMaxChunks * 4; }

cudaError_t launch_score(const ds_cache *c, const ScoreParams &p, const SelectGeom &g, cudaStream_t st) {
  const int units = c->batch * c->num_kv_heads;
  if (g.chunk > kMaxChunkLen) return cudaErrorInvalidValue;
#define DS_SCORE(T, R) launch_score_t<T, R>(p, units, g.nchunks, g.score_smem, st)
  switch (c->dtype) {
    case DS_BF16:
      return c->r == 8 ? DS_SCORE(__nv_bfloat16, 8) : (c->r == 16 ? DS_SCORE(__nv_bfloat16, 16) : DS_SCORE(__nv_bfloat16, 0));
    case DS_FP16:
      return c->r == 8 ? DS_SCORE(__half, 8) : (c->r == 16 ? DS_SCORE(__half, 16) : DS_SCORE(__half, 0));
    default:
      return c->r == 16 ? DS_SCORE(float, 16) : (c->r == 8 ? DS_SCORE(float, 8) : DS_SCORE(float, 0));
  }
#undef DS_SCORE
}

}  // namespace ds
