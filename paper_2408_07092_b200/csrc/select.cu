// select.cu -- a1..a3 of Algorithm 1: label-score GEMV and exact
// top-k selection, as two kernels.
//
// score_kernel  (grid: chunks x units, no inter-CTA communication)
//   a1  q_lab[j] = sum_g q[b][hG+g][C[h][j]]      (fp32, g order; reading R3)
//   a2  s_hat[t] = fma-chain_j(q_lab[j], L[t][j])  (fp32, j ascending, no
//       1/sqrt(d); reading R2), streamed from the contiguous label cache with
//       eight 128-bit loads in flight per thread (one row = r*e = 16 B at
//       r=8 / 16-bit).  Each score becomes a monotone u32 order key (-0 == +0)
//       written to a workspace that stays in L2, plus a per-CTA histogram of
//       the key's top 11 bits (sign, exponent, 2 mantissa bits).
//
// select_kernel (grid: units, one 1024-thread CTA each; __syncthreads only)
//   a3  i = argtopk(s_hat, k): ties to the lower index, ascending (reading R6).
//       The unit's <= 8 partial histograms are summed -> boundary digit b1;
//       one pass over the L2-resident keys marks digit > b1 in a selection
//       bitmap and collects the boundary digit's (key, token) candidates;
//       these are resolved exactly by a second 11-bit level and an exact rank
//       of the few keys left in the second boundary digit.  A tie-heavy
//       boundary (more candidates than fit) takes an exact MSB radix select.
//       The bitmap is compacted in token order into the index list, and each
//       selected token's pool row id (block_table lookup) is written beside
//       it, so the attention kernel's gathers start after a single load.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace ds {

constexpr int kScoreThreads = 512;
constexpr int kScoreUnroll = 8;
constexpr int kMaxChunks = 8;  // score CTAs per unit (partial histograms)
constexpr int kMaxR = 256;
constexpr int kDigitBits = 12;             // radix digit width
constexpr int kBins = 1 << kDigitBits;      // digits per level
constexpr int kShift1 = 32 - kDigitBits;    // level 1: top 12 key bits
constexpr int kShift2 = kShift1 - kDigitBits;  // level 2: the next 12
constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kCandCap = 4096;

// per-unit stride of the key workspace: a multiple of 4 keys (16 B)
__host__ __device__ __forceinline__ size_t key_stride(int smax) { return ((size_t)smax + 3) & ~(size_t)3; }

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

template <typename T, int R>
__global__ void __launch_bounds__(kScoreThreads) score_kernel(ScoreParams p) {
  const CacheView &c = p.c;
  const int unit = blockIdx.y, part = blockIdx.x;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int tid = threadIdx.x;
  const int n = c.seq_lens[b];
  const int t0 = part * p.chunk;
  const int nloc = min(p.chunk, n - t0);
  const int r = R > 0 ? R : c.r;
  DS_TRACE_AT(0, 0);
  __shared__ float qlab[kMaxR];
  __shared__ __align__(16) uint32_t hist[kBins];
  for (int i = tid; i < kBins; i += kScoreThreads) hist[i] = 0;
  pdl_wait();  // the label rows may come from the preceding append
  pdl_trigger();
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
  const size_t obase = (size_t)unit * c.Smax + t0;

  if (p.scores) {  // diagnostics entry (ds_approx_scores): s_hat to HBM
    for (int i = tid; i < nloc; i += kScoreThreads) p.scores[obase + i] = label_score<T, R>(lab + (size_t)i * r, qs, r);
    return;
  }
  uint32_t *keys = p.keys + (size_t)unit * key_stride(c.Smax) + t0;
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
  uint4 *dst = reinterpret_cast<uint4 *>(p.part_hist + ((size_t)unit * kMaxChunks + part) * kBins);
  for (int i = tid; i < kBins / 4; i += kScoreThreads) dst[i] = reinterpret_cast<const uint4 *>(hist)[i];
  DS_TRACE_AT(0, 1);
}

// ------------------------------------------------------------------ B
struct SelSmem {
  uint32_t bins[kBins];
  uint32_t warp_tot[kSelWarps];
  uint32_t state[4];
  uint32_t ncand, nfinal;
  uint2 cand[kCandCap];  // (key, token)
};

// Block-wide exclusive prefix of one u32 per thread; *total gets the sum.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *warp_tot, uint32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint32_t before = 0, tot = 0;
  for (int w = 0; w < kSelWarps; ++w) {
    const uint32_t t = warp_tot[w];
    before += w < warp ? t : 0u;
    tot += t;
  }
  *total = tot;
  return before + x - v;
}

// Boundary digit of the histogram in sm.bins: with `need` keys wanted from the
// top, the digit d with above(d) < need <= above(d) + bins[d]; all threads get
// (d, above(d), bins[d]).
__device__ __forceinline__ void find_boundary(SelSmem &sm, uint32_t need, uint32_t &d, uint32_t &above,
                                              uint32_t &cnt) {
  constexpr int PER = kBins / kSelThreads;
  const int tid = threadIdx.x;
  uint32_t v[PER], s = 0;  // thread tid owns digits kBins-1-PER*tid-j (descending order)
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    v[j] = sm.bins[kBins - 1 - PER * tid - j];
    s += v[j];
  }
  uint32_t tot;
  uint32_t run = block_excl_scan(s, sm.warp_tot, &tot);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (run < need && run + v[j] >= need) {
      sm.state[0] = kBins - 1 - PER * tid - j;
      sm.state[1] = run;
      sm.state[2] = v[j];
    }
    run += v[j];
  }
  __syncthreads();
  d = sm.state[0];
  above = sm.state[1];
  cnt = sm.state[2];
  __syncthreads();
}

// Ordered compaction of the selection bitmap: token t -> position
// #selected(< t), with its pool row id.
__device__ __forceinline__ void compact(SelSmem &sm, const uint32_t *bm, int nwords, int32_t *idx_out,
                                        int32_t *rowid_out, const CacheView &c, const int32_t *bt, int h) {
  const int tid = threadIdx.x;
  const int per = (nwords + kSelThreads - 1) / kSelThreads;
  const int w0 = min(tid * per, nwords), w1 = min(w0 + per, nwords);
  uint32_t cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bm[w]);
  uint32_t tot;
  uint32_t pos = block_excl_scan(cnt, sm.warp_tot, &tot);
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = bm[w];
    while (bits) {  // up to 4 tokens at a time
      int tt[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tt[u] = bits ? w * 32 + __ffs(bits) - 1 : -1;
        bits &= bits - 1;
      }
      int pg[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) pg[u] = tt[u] >= 0 ? bt[tt[u] / c.P] : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (tt[u] < 0) break;
        idx_out[pos] = tt[u];
        rowid_out[pos] = (int32_t)(((uint32_t)pg[u] * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P +
                                   (uint32_t)(tt[u] % c.P));
        ++pos;
      }
    }
  }
}

// Spread the 8 bits of x to bit positions 0, 4, ..., 28.
__device__ __forceinline__ uint32_t spread4(uint32_t x) {
  x = (x | (x << 12)) & 0x000F000Fu;
  x = (x | (x << 6)) & 0x03030303u;
  x = (x | (x << 3)) & 0x11111111u;
  return x;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(SelectParams p) {
  extern __shared__ __align__(16) uint8_t dyn[];
  SelSmem &sm = *reinterpret_cast<SelSmem *>(dyn);
  uint32_t *bm = reinterpret_cast<uint32_t *>(dyn + sizeof(SelSmem));  // [Smax/32] selection bitmap
  int32_t *btrow = reinterpret_cast<int32_t *>(bm + ((p.c.Smax + 31) >> 5));  // [maxp] this sequence's pages
  const CacheView &c = p.c;
  const int unit = blockIdx.x;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31;
  const int n = c.seq_lens[b];
  const int keff = min(p.k, n);
  const int nwords = (n + 31) >> 5;
  int32_t *idx_out = p.idx + (size_t)unit * p.k;
  int32_t *rid_out = p.rowid + (size_t)unit * p.k;
  const uint32_t *keys = p.keys + (size_t)unit * key_stride(c.Smax);
  DS_TRACE_AT(1, 0);

  {
    const int np = (n + c.P - 1) / c.P;
    const int32_t *bt = c.block_table + (size_t)b * c.maxp;
    for (int i = tid; i < np; i += kSelThreads) btrow[i] = __ldg(bt + i);
  }
  for (int i = keff + tid; i < p.k; i += kSelThreads) {  // positions >= k_eff
    idx_out[i] = -1;
    rid_out[i] = -1;
  }
  if (tid == 0) {
    sm.ncand = 0;
    sm.nfinal = 0;
  }
  pdl_wait();  // keys and partial histograms come from score_kernel
  pdl_trigger();
  if (keff >= n) {  // every token selected (k >= S, or a short sequence)
    for (int w = tid; w < nwords; w += kSelThreads)
      bm[w] = (w == nwords - 1 && (n & 31)) ? (1u << (n & 31)) - 1u : 0xffffffffu;
    __syncthreads();
    compact(sm, bm, nwords, idx_out, rid_out, c, btrow, h);
    return;
  }

  // ---- level 1: sum the partial histograms of the score CTAs
  const int nparts = (n + p.chunk - 1) / p.chunk;
  for (int i = tid; i < kBins; i += kSelThreads) {
    uint32_t v[kMaxChunks];
#pragma unroll
    for (int q = 0; q < kMaxChunks; ++q)
      v[q] = q < nparts ? __ldcg(p.part_hist + ((size_t)unit * kMaxChunks + q) * kBins + i) : 0u;
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < kMaxChunks; ++q) s += v[q];
    sm.bins[i] = s;
  }
  __syncthreads();
  uint32_t b1, above1, cnt1;
  find_boundary(sm, (uint32_t)keff, b1, above1, cnt1);
  DS_TRACE_AT(1, 1);
  const uint32_t rem1 = (uint32_t)keff - above1;
  const bool take_all = cnt1 == rem1;

  if (take_all || cnt1 <= (uint32_t)kCandCap) {
    // ---- one pass over the keys: bitmap of digit > b1 (and == b1 when all of
    // it is taken), boundary candidates into smem.  A warp covers 32
    // consecutive tokens per round (one bitmap word).
    // A warp round covers 128 consecutive tokens: lane l holds tokens
    // base+4l .. base+4l+3 (one 128-bit load); the 4 bitmap words of the
    // round are assembled from 4 ballots.  RB rounds of loads in flight.
    constexpr int RB = 8, TPR = kSelThreads * 4;
    const int rounds = (n + TPR - 1) / TPR;
    for (int rd0 = 0; rd0 < rounds; rd0 += RB) {
      uint4 kv[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int t = (rd0 + u) * TPR + 4 * tid;
        kv[u] = t < n ? __ldcg(reinterpret_cast<const uint4 *>(keys + t)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        if (rd0 + u >= rounds) break;
        const int base = (rd0 + u) * TPR + (tid & ~31) * 4;
        const int tl = base + 4 * lane;
        const uint32_t kk[4] = {kv[u].x, kv[u].y, kv[u].z, kv[u].w};
        uint32_t sb[4], cb[4];
        int mycand = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const bool in = tl + e < n;
          const uint32_t d = kk[e] >> kShift1;
          sb[e] = __ballot_sync(0xffffffffu, in && (d > b1 || (take_all && d == b1)));
          const bool cand = !take_all && in && d == b1;
          cb[e] = __ballot_sync(0xffffffffu, cand);
          mycand += cand;
        }
        if (lane < 4 && base + 32 * lane < n) {
          uint32_t word = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) word |= spread4((sb[e] >> (8 * lane)) & 0xffu) << e;
          bm[(base >> 5) + lane] = word;
        }
        if ((cb[0] | cb[1] | cb[2] | cb[3]) != 0u) {
          // slots: warp-inclusive prefix of the per-lane candidate counts
          int incl = mycand;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          uint32_t slot = 0;
          if (lane == 31) slot = atomicAdd(&sm.ncand, (uint32_t)incl);
          slot = __shfl_sync(0xffffffffu, slot, 31) + (uint32_t)(incl - mycand);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t d = kk[e] >> kShift1;
            if (tl + e < n && d == b1) sm.cand[slot++] = make_uint2(kk[e], (uint32_t)(tl + e));
          }
        }
      }
    }
    __syncthreads();
    DS_TRACE_AT(1, 2);
    if (!take_all) {
      // ---- level 2 over the candidates: the next 11 bits
      const int nc = (int)sm.ncand;
      for (int i = tid; i < kBins; i += kSelThreads) sm.bins[i] = 0;
      __syncthreads();
      for (int i = tid; i < nc; i += kSelThreads) atomicAdd(&sm.bins[(sm.cand[i].x >> kShift2) & (kBins - 1)], 1u);
      __syncthreads();
      uint32_t b2, above2, cnt2;
      find_boundary(sm, rem1, b2, above2, cnt2);
      const uint32_t rem2 = rem1 - above2;
      uint2 *fin = sm.cand + nc;  // keys of digit b2 (when ranked) reuse the buffer tail
      const int fcap = kCandCap - nc;
      for (int i = tid; i < nc; i += kSelThreads) {
        const uint2 e = sm.cand[i];
        const uint32_t d2 = (e.x >> kShift2) & (kBins - 1);
        if (d2 > b2 || (cnt2 == rem2 && d2 == b2)) {
          atomicOr(&bm[e.y >> 5], 1u << (e.y & 31));
        } else if (d2 == b2) {
          const uint32_t s = atomicAdd(&sm.nfinal, 1u);
          if ((int)s < fcap) fin[s] = e;
        }
      }
      __syncthreads();
      if (cnt2 != rem2) {  // exact rank (key desc, token asc) inside digit b2
        const int nf = (int)sm.nfinal;
        const bool small = nf <= fcap;
        const uint2 *lst = small ? fin : sm.cand;
        const int nl = small ? nf : nc;
        for (int i = tid; i < nl; i += kSelThreads) {
          const uint2 me = lst[i];
          if (((me.x >> kShift2) & (kBins - 1)) != b2) continue;
          uint32_t rank = 0;
          for (int j = 0; j < nl; ++j) {
            const uint2 o = lst[j];
            if (((o.x >> kShift2) & (kBins - 1)) != b2) continue;
            rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);
          }
          if (rank < rem2) atomicOr(&bm[me.y >> 5], 1u << (me.y & 31));
        }
      }
      __syncthreads();
    }
  } else {
    // ---- exact MSB radix over the remaining 21 key bits (tie-heavy boundary)
    uint32_t prefix = b1 << kShift1, mask = 0xffffffffu << kShift1, rem = rem1;
    const int shs[3] = {kShift1 - 8, kShift1 - 16, 0}, nbs[3] = {8, 8, kShift1 - 16};
    for (int ps = 0; ps < 3; ++ps) {
      const int sh = shs[ps];
      const uint32_t dm = (1u << nbs[ps]) - 1u;
      for (int i = tid; i < 256; i += kSelThreads) sm.bins[i] = 0;
      __syncthreads();
      for (int t = tid; t < n; t += kSelThreads) {
        const uint32_t key = __ldcg(keys + t);
        if ((key & mask) == prefix) atomicAdd(&sm.bins[(key >> sh) & dm], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t above = 0;
        for (int dd = (int)dm; dd >= 0; --dd) {
          if (above + sm.bins[dd] >= rem) {
            sm.state[0] = dd;
            sm.state[1] = above;
            sm.state[2] = sm.bins[dd];
            break;
          }
          above += sm.bins[dd];
        }
      }
      __syncthreads();
      rem -= sm.state[1];
      prefix |= sm.state[0] << sh;
      mask |= dm << sh;
      const bool done = sm.state[2] == rem;
      __syncthreads();
      if (done) break;
    }
    // gt: (key & mask) > prefix; eq: == prefix, the first `rem` by token index
    uint32_t eq_before = 0;
    const int rounds = (n + kSelThreads - 1) / kSelThreads;
    for (int rd = 0; rd < rounds; ++rd) {
      const int base = rd * kSelThreads + (tid & ~31);
      const int t = base + lane;
      const uint32_t km = (t < n ? __ldcg(keys + t) : 0u) & mask;
      const bool gt = t < n && km > prefix;
      const bool eq = t < n && km == prefix;
      const uint32_t em = __ballot_sync(0xffffffffu, eq);
      uint32_t tot;
      const uint32_t wb = block_excl_scan(lane == 0 ? (uint32_t)__popc(em) : 0u, sm.warp_tot, &tot);
      const uint32_t rk = eq_before + __shfl_sync(0xffffffffu, wb, 0) + __popc(em & lanemask_lt());
      const uint32_t word = __ballot_sync(0xffffffffu, gt || (eq && rk < rem));
      if (lane == 0 && base < n) bm[base >> 5] = word;
      eq_before += tot;
    }
    __syncthreads();
  }
  DS_TRACE_AT(1, 3);
  compact(sm, bm, nwords, idx_out, rid_out, c, btrow, h);
  DS_TRACE_AT(1, 4);
}

// ------------------------------------------------------------- launch
template <typename T, int R>
static cudaError_t launch_score_t(const ScoreParams &p, int units, int nchunks, cudaStream_t st) {
  return PdlLaunch(dim3(nchunks, units), dim3(kScoreThreads), 0, st).run(score_kernel<T, R>, p);
}

SelectGeom select_geom(const ds_cache *c) {
  SelectGeom g{};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * c->num_kv_heads;
  // as many score CTAs per unit as fit in one wave (no straggler wave)
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, score_kernel<__nv_bfloat16, 8>, kScoreThreads, 0) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    per_sm = 2;
  }
  int nch = (per_sm * sms) / units;
  nch = nch < 1 ? 1 : (nch > kMaxChunks ? kMaxChunks : nch);
  int chunk = (c->max_seq_len + nch - 1) / nch;
  chunk = (chunk + 255) & ~255;
  g.chunk = chunk;
  g.nchunks = (c->max_seq_len + chunk - 1) / chunk;
  g.smem = sizeof(SelSmem) + (size_t)((c->max_seq_len + 31) / 32) * 4 + (size_t)c->max_pages_per_seq * 4;
  g.threads = kSelThreads;
  return g;
}

size_t select_workspace_keys(const ds_cache *c) {
  return (size_t)c->batch * c->num_kv_heads * key_stride(c->max_seq_len) * 4;
}
size_t select_workspace_hist(const ds_cache *c) {
  return (size_t)c->batch * c->num_kv_heads * kMaxChunks * kBins * 4;
}

cudaError_t launch_score(const ds_cache *c, const ScoreParams &p, const SelectGeom &g, cudaStream_t st) {
  const int units = c->batch * c->num_kv_heads;
  switch (c->dtype) {
    case DS_BF16:
      return c->r == 8 ? launch_score_t<__nv_bfloat16, 8>(p, units, g.nchunks, st)
                       : (c->r == 16 ? launch_score_t<__nv_bfloat16, 16>(p, units, g.nchunks, st)
                                     : launch_score_t<__nv_bfloat16, 0>(p, units, g.nchunks, st));
    case DS_FP16:
      return c->r == 8 ? launch_score_t<__half, 8>(p, units, g.nchunks, st)
                       : (c->r == 16 ? launch_score_t<__half, 16>(p, units, g.nchunks, st)
                                     : launch_score_t<__half, 0>(p, units, g.nchunks, st));
    default:
      return c->r == 16 ? launch_score_t<float, 16>(p, units, g.nchunks, st)
                        : (c->r == 8 ? launch_score_t<float, 8>(p, units, g.nchunks, st)
                                     : launch_score_t<float, 0>(p, units, g.nchunks, st));
  }
}

cudaError_t launch_select(const ds_cache *c, const SelectParams &p, const SelectGeom &g, cudaStream_t st) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (attr != cudaSuccess) return attr;
  return PdlLaunch(dim3(c->batch * c->num_kv_heads), dim3(kSelThreads), g.smem, st).run(select_kernel, p);
}

}  // namespace ds
