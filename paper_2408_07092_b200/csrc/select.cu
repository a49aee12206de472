// select.cu -- a1..a3 of Algorithm 1: label-score GEMV and exact
// top-k selection, fused in one kernel: score_select_kernel, grid
// (nch, units) with the nch CTAs of a (b, KV head) unit forming one thread-
// block cluster; each CTA owns a contiguous chunk of tokens.
//   a1  q_lab[j] = sum_g q[b][hG+g][C[h][j]]      (fp32, g order; reading R3)
//   a2  s_hat[t] = fma-chain_j(q_lab[j], L[t][j])  (fp32, j ascending, no
//       1/sqrt(d); reading R2), streamed from the contiguous label cache with
//       eight 128-bit loads in flight per thread (one row = r*e = 16 B at
//       r=8 / 16-bit), kept in shared memory as monotone u32 order keys
//       (-0 == +0) while a 12-bit histogram of the keys' top bits is built.
//       s_hat never leaves the chip.
//   a3  i = argtopk(s_hat, k): exact, ties to the lower index, ascending
//       (reading R6).  The selection is fixed by one boundary pair (kB, tB):
//       token t is selected  <=>  key > kB  or  (key == kB and t <= tB),
//       i.e. rank < k in the order (key desc, token asc).  It is found with
//       cluster barriers and a few KB of DSMEM reads:
//         S1  cluster histogram of bits 31..20 -> boundary digit D1
//         L2  one pass over the chunk: keys with digit D1 (a few hundred)
//             go to a candidate list and a 10-bit histogram of bits 19..10
//         S2  cluster histogram -> 22-bit boundary prefix P2
//         S3  the keys with prefix P2 (typically < 10) and per-CTA counts
//             are exchanged; every CTA ranks those members exactly
//         S4  exit guard; CTA 0 publishes the unit's ready flag
//       then each CTA writes its selected tokens, ascending, at its cluster
//       prefix offset together with their pool row ids (block_table), so the
//       attention kernel's gathers start after a single load.  If more than
//       kMaxMembers keys share P2 (massive ties), the last 10 bits and the
//       token order of equal keys are resolved with two more barriers.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ds_common.cuh"
#include "ds_internal.h"

namespace cg = cooperative_groups;

namespace ds {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 8;
constexpr int kMaxChunks = 16;       // CTAs (cluster size) per unit
constexpr int kMaxChunkLen = 16384;  // tokens per CTA (keys kept in smem)
constexpr int kMaxR = 256;
constexpr int kSh1 = 20, kD1 = 4096;  // level-1 digit: key bits 31..20
constexpr int kSh2 = 10, kD2 = 1024;  // level-2 digit: key bits 19..10
constexpr int kD3 = 1024;             // level-3 digit: key bits 9..0
constexpr int kCandCap = 1024;        // level-1 boundary keys listed per CTA
constexpr int kMaxMembers = 512;      // P2 keys ranked directly (cluster-wide)
constexpr int kMaxPageRow = 1024;     // block-table entries cached per CTA
constexpr int kMaxDynSmem = (kMaxChunkLen + 128) * 4 + kMaxPageRow * 4;

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

struct SelSh {
  float qlab[kMaxR];
  uint32_t h1[kD1];  // level-1 histogram (read remotely S1..S2); later the level-3 one
  uint32_t c1[64];   // 64-bin coarse sums of h1 (remote S1..S2)
  uint32_t h2[kD2];  // level-2 histogram (remote S2..S3)
  uint32_t c2[32];   // coarse sums of h2 (remote S2..S3)
  uint2 cand[kCandCap];         // (key, token) with digit1 == D1
  uint2 members[kMaxMembers];   // (key, token) with prefix P2 (remote S3..S4)
  uint2 gathered[kMaxMembers];
  uint32_t gtm[kMaxChunkLen / 32];  // per 32-token group: digit1 > D1 (>= D1 if taken whole)
  uint32_t eqm[kMaxChunkLen / 32];  // per 32-token group: digit1 == D1 (not whole)
  uint32_t wcnt[kWarps];  // per-warp scratch counts
  uint32_t cnt[4];        // [0] #digit1 > D1 (or >= if whole), [1] #(digit1 == D1, prefix > P2), [3] total
  uint32_t state[8];
  uint32_t ncand, nmem, lower_sel, pad;
};

// Cluster-wide boundary over a histogram of 64*64 (NC=64, coarse sums in c)
// or 32*32 (NC=32) bins, each CTA holding its own copy; warp 0 only.
template <int NC>
__device__ __forceinline__ Boundary<NC / 32> cluster_boundary(cg::cluster_group &cluster, int nch, uint32_t *h,
                                                              uint32_t *cs, uint32_t need) {
  constexpr int NPL = NC / 32;
  const int lane = threadIdx.x & 31;
  uint32_t v[NPL];
#pragma unroll
  for (int j = 0; j < NPL; ++j) v[j] = 0;
  for (int cr = 0; cr < nch; ++cr) {
    const uint32_t *rc = cluster.map_shared_rank(cs, cr);
#pragma unroll
    for (int j = 0; j < NPL; ++j) v[j] += rc[NC - 1 - NPL * lane - j];
  }
  const Boundary<NPL> cb = warp_boundary<NPL>(v, NC - 1, 0u, need);
#pragma unroll
  for (int j = 0; j < NPL; ++j) v[j] = 0;
  for (int cr = 0; cr < nch; ++cr) {
    const uint32_t *rf = cluster.map_shared_rank(h, cr) + cb.bin * NC;
#pragma unroll
    for (int j = 0; j < NPL; ++j) v[j] += rf[NC - 1 - NPL * lane - j];
  }
  return warp_boundary<NPL>(v, cb.bin * NC + NC - 1, cb.above, need);
}

// coarse sums: cs[i] = sum of h[i*NC .. i*NC+NC-1] for NC*NC bins (all threads)
template <int NC>
__device__ __forceinline__ void coarse_sums(const uint32_t *h, uint32_t *cs) {
  constexpr int kPer = NC * NC / kThreads;  // bins per thread: 8 (NC=64) or 2 (NC=32)
  constexpr int kLanes = NC / kPer;         // lanes per coarse bin: 8 or 16
  const int tid = threadIdx.x;
  uint32_t v = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) v += h[tid * kPer + j];
#pragma unroll
  for (int o = 1; o < kLanes; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((tid & (kLanes - 1)) == 0) cs[tid / kLanes] = v;
}

template <typename T, int R>
__global__ void __launch_bounds__(kThreads, 2) score_select_kernel(ScoreParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int nch = (int)cluster.num_blocks(), crank = (int)cluster.block_rank();
  extern __shared__ __align__(16) uint32_t keys[];  // [chunk + 128] order keys, then the page row
  __shared__ SelSh sh;
  const CacheView &c = p.c;
  const int unit = blockIdx.y;
  const int b = unit / c.Hkv, h = unit - (unit / c.Hkv) * c.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = c.seq_lens[b];
  const int keff = min(p.k, n);
  const int t0 = crank * p.chunk;
  const int nloc = max(0, min(p.chunk, n - t0));
  const int r = R > 0 ? R : c.r;
  int32_t *idx_out = p.idx ? p.idx + (size_t)unit * p.k : nullptr;
  int32_t *rid_out = p.rowid ? p.rowid + (size_t)unit * p.k : nullptr;
  int32_t *btrow = reinterpret_cast<int32_t *>(keys + p.chunk + 128);  // pages of this chunk
  const int pg0 = t0 / c.P;
  const bool bt_cached = p.chunk / c.P + 2 <= kMaxPageRow;
  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  DS_TRACE_AT(0, 0);
  pdl_wait();  // the label rows may come from the preceding append
  pdl_trigger();
  // (every branch below is uniform over the cluster: n, k, p.scores are)
  if (n <= 0) {  // empty sequence: nothing selected (the attention writes zeros)
    if (crank == 0 && idx_out)
      for (int i = tid; i < p.k; i += kThreads) {
        idx_out[i] = -1;
        rid_out[i] = -1;
      }
    return;
  }
  // ---- a1 + this chunk's block-table entries (issued early) + zeroing
  const int npg = nloc > 0 ? (t0 + nloc - 1) / c.P - pg0 + 1 : 0;
  if (!p.scores && bt_cached)
    for (int i = tid; i < npg; i += kThreads) btrow[i] = __ldg(bt + pg0 + i);
  const bool gmax = c.greduce == DS_GROUP_MAX;  // R17 (host-checked: G * r <= kMaxR)
  for (int i = tid; i < (gmax ? c.G * r : r); i += kThreads) {
    const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)h * c.G) * c.D;
    const int g0 = gmax ? i / r : 0, j = gmax ? i - g0 * r : i;
    const int ch = c.C[(size_t)h * c.r + j];
    float s = 0.0f;
    if (gmax) s = Elem<T>::to_f(qb[(size_t)g0 * c.D + ch]);  // per-head label q_g[C[j]]
    else
      for (int g = 0; g < c.G; ++g) s = s + Elem<T>::to_f(qb[(size_t)g * c.D + ch]);
    sh.qlab[i] = s;
  }
  for (int i = tid; i < kD1; i += kThreads) sh.h1[i] = 0;
  for (int i = tid; i < kD2; i += kThreads) sh.h2[i] = 0;
  if (tid < kWarps) sh.wcnt[tid] = 0;
  if (tid == 0) {
    sh.ncand = 0;
    sh.nmem = 0;
    sh.lower_sel = 0;
  }
  __syncthreads();
  float ql[R > 0 ? R : 1];
  if constexpr (R > 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) ql[j] = sh.qlab[j];
  }
  const float *qs = R > 0 ? ql : sh.qlab;
  const size_t lrow = ((size_t)b * c.Hkv + h) * c.Smax + t0;  // first label row of this CTA
  const T *lab = (const T *)c.label + lrow * (size_t)c.r;
  const uint8_t *cod = (const uint8_t *)c.label + lrow * (size_t)c.rb;  // 4-bit label (R16)
  const T *scl = (const T *)c.label_scale + lrow;
  auto head_score = [&](int i, const float *qv) {
    if (c.lnone) {  // no label cache (Table 4 ablation): the channels of the paged K row
      const int t = t0 + i;
      const T *kr = (const T *)c.k_pool +
                    (((size_t)__ldg(bt + t / c.P) * c.Hkv + h) * c.P + t % c.P) * (size_t)c.D;
      float s = 0.0f;
      for (int j = 0; j < r; ++j) s = fmaf(qv[j], Elem<T>::to_f(kr[c.C[(size_t)h * c.r + j]]), s);
      return s;
    }
    return c.lq4 ? q4_score<T>(cod + (size_t)i * c.rb, scl[i], qv, r) : label_score<T, R>(lab + (size_t)i * r, qv, r);
  };
  auto score_at = [&](int i) {
    if (!gmax) return head_score(i, qs);
    float m = -INFINITY;  // R17: max over the group's per-head scores
    for (int g = 0; g < c.G; ++g) m = fmaxf(m, head_score(i, sh.qlab + g * r));
    return m;
  };
  if (p.scores) {  // diagnostics entry (ds_approx_scores): s_hat to HBM
    float *so = p.scores + (size_t)unit * c.Smax + t0;
    for (int i = tid; i < nloc; i += kThreads) so[i] = score_at(i);
    return;
  }
  // ---- a2: stream the label -> keys + level-1 histogram
  int i0 = tid;
  if constexpr (R > 0 && R * sizeof(T) == 16) {
    constexpr int U = kUnroll;
    for (; !c.lq4 && !c.lnone && !gmax && i0 + (U - 1) * kThreads < nloc; i0 += U * kThreads) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const uint4 *>(lab) + (size_t)(i0 + u * kThreads));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const T *e = reinterpret_cast<const T *>(&v[u]);
        float s = 0.0f;
#pragma unroll
        for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[j]), s);
        const uint32_t k0 = order_key(s);
        keys[i0 + u * kThreads] = k0;
        atomicAdd(&sh.h1[k0 >> kSh1], 1u);
      }
    }
  }
  for (int i = i0; i < nloc; i += kThreads) {
    const uint32_t k0 = order_key(score_at(i));
    keys[i] = k0;
    atomicAdd(&sh.h1[k0 >> kSh1], 1u);
  }
  if (tid < 128) keys[nloc + tid] = 0u;  // pad: below every finite score's key
  DS_TRACE_AT(0, 1);

  const bool pow2 = (c.P & (c.P - 1)) == 0;
  const int psh = __ffs(c.P) - 1;
  auto rowid_of = [&](int t) -> int32_t {
    const int pg = pow2 ? (t >> psh) : t / c.P;
    const int sl = t - pg * c.P;
    const int32_t page = bt_cached ? btrow[pg - pg0] : __ldg(bt + pg);
    return (int32_t)(((uint32_t)page * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P + (uint32_t)sl);
  };
  // warp ranges: warp w owns local tokens [w0, w1), a multiple of 128 long
  int per = (nloc + kWarps - 1) / kWarps;
  per = (per + 127) & ~127;
  const int w0 = min(warp * per, nloc), w1 = min(w0 + per, nloc);

  // every token selected (k >= n): ascending identity
  if (keff >= n) {
    __syncthreads();
    if (crank == 0)
      for (int i = n + tid; i < p.k; i += kThreads) {
        idx_out[i] = -1;
        rid_out[i] = -1;
      }
    for (int i = tid; i < nloc; i += kThreads) {
      idx_out[t0 + i] = t0 + i;
      rid_out[t0 + i] = rowid_of(t0 + i);
    }
    cluster.sync();
    if (crank == 0 && tid == 0) {
      __threadfence();
      atomicExch(p.ready + unit, 1u);
    }
    return;
  }
  if (crank == 0)  // positions >= k_eff
    for (int i = keff + tid; i < p.k; i += kThreads) {
      idx_out[i] = -1;
      rid_out[i] = -1;
    }
  __syncthreads();
  coarse_sums<64>(sh.h1, sh.c1);

  // ---- S1: level-1 boundary digit D1
  cluster.sync();
  if (warp == 0) {
    const Boundary<2> d1 = cluster_boundary<64>(cluster, nch, sh.h1, sh.c1, (uint32_t)keff);
    if (lane == 0) {
      sh.state[0] = (uint32_t)d1.bin;
      sh.state[1] = d1.above;
      sh.state[2] = d1.cnt;
    }
  }
  __syncthreads();
  const uint32_t D1 = sh.state[0];
  const uint32_t need1 = (uint32_t)keff - sh.state[1];
  const bool whole1 = sh.state[2] == need1;
  const bool ovf = sh.h1[D1] > (uint32_t)kCandCap;  // my D1 keys do not fit the list
  DS_TRACE_AT(0, 2);

  // ---- L2: per 32-token group, ballot masks of digit1 > D1 (>= D1 when D1
  // is taken whole) and digit1 == D1 (keys past nloc are 0: below any
  // finite score's key)
  const uint32_t lt = lanemask_lt();
  const int ng = (w1 - w0 + 31) >> 5;  // this warp's groups (<= 32)
  const int grp = (w0 >> 5) + lane;    // lane-per-group passes: my group
  {
    const int gcmp = whole1 ? (int)D1 - 1 : (int)D1;
    const uint32_t ecmp = whole1 ? 0xffffffffu : D1;
    uint32_t g = 0;
    for (int base = w0; base < w1; base += 128) {
      uint32_t kk[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) kk[e] = keys[base + 32 * e + lane];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t d = kk[e] >> kSh1;
        const uint32_t mg = __ballot_sync(0xffffffffu, (int)d > gcmp);
        const uint32_t me = __ballot_sync(0xffffffffu, d == ecmp);
        if (lane == e) {
          sh.gtm[(base >> 5) + e] = mg;
          sh.eqm[(base >> 5) + e] = me;
        }
        g += __popc(mg);
      }
    }
    if (lane == 0) sh.wcnt[warp] = g;
    __syncwarp();
    // the D1 keys (a few hundred): candidate list + level-2 histogram
    if (!whole1) {
      uint32_t e = lane < ng ? sh.eqm[grp] : 0u;
      const uint32_t ne = __popc(e);
      uint32_t incl = ne;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t slot = 0;
      if (lane == 31 && incl && !ovf) slot = atomicAdd(&sh.ncand, incl);
      slot = __shfl_sync(0xffffffffu, slot, 31) + incl - ne;
      while (e) {
        const int bit = __ffs(e) - 1;
        e &= e - 1;
        const uint32_t key = keys[grp * 32 + bit];
        atomicAdd(&sh.h2[(key >> kSh2) & (kD2 - 1)], 1u);
        if (!ovf) sh.cand[slot++] = make_uint2(key, (uint32_t)(t0 + grp * 32 + bit));
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kWarps; ++w) s += sh.wcnt[w];
    sh.cnt[0] = s;
    sh.cnt[1] = 0;
  }
  coarse_sums<32>(sh.h2, sh.c2);
  DS_TRACE_AT(0, 3);

  // iterate this CTA's keys with digit1 == D1: the list, or a full scan
  auto for_each_cand = [&](auto &&f) {
    if (!ovf) {
      const int nc = (int)sh.ncand;
      for (int i = tid; i < nc; i += kThreads) f(sh.cand[i].x, (int)sh.cand[i].y);
    } else {
      for (int i = tid; i < nloc; i += kThreads) {
        const uint32_t key = keys[i];
        if ((key >> kSh1) == D1) f(key, t0 + i);
      }
    }
  };

  uint32_t kB = 0;   // boundary pair: selected <=> key > kB || (key == kB && t <= tB)
  int tB = 0x7fffffff;
  uint32_t base_sel = 0;  // selected tokens of the lower CTAs of the cluster
  if (whole1) {
    kB = D1 << kSh1;  // key >= kB
    cluster.sync();   // S2: counts
    for (int cr = 0; cr < crank; ++cr) base_sel += cluster.map_shared_rank(sh.cnt, cr)[0];
  } else {
    // ---- S2: level-2 boundary -> 22-bit prefix P2
    cluster.sync();
    if (warp == 0) {
      const Boundary<1> d2 = cluster_boundary<32>(cluster, nch, sh.h2, sh.c2, need1);
      if (lane == 0) {
        sh.state[3] = (uint32_t)d2.bin;
        sh.state[4] = d2.above;
        sh.state[5] = d2.cnt;
      }
    }
    __syncthreads();
    const uint32_t P2 = (D1 << (kSh1 - kSh2)) | sh.state[3];
    const uint32_t need2 = need1 - sh.state[4];
    const uint32_t cnt2 = sh.state[5];
    const bool whole2 = cnt2 == need2;
    const bool fits2 = cnt2 <= (uint32_t)kMaxMembers;
    // members pass over the candidates: prefix > P2 are selected (>= P2 when
    // P2 is taken whole); prefix == P2 -> member list
    for_each_cand([&](uint32_t key, int t) {
      const uint32_t pfx = key >> kSh2;
      if (pfx > P2 || (whole2 && pfx == P2)) {
        atomicAdd(&sh.cnt[1], 1u);
      } else if (pfx == P2 && fits2) {
        sh.members[atomicAdd(&sh.nmem, 1u)] = make_uint2(key, (uint32_t)t);
      }
    });
    DS_TRACE_AT(0, 4);
    // ---- S3: exchange members + counts
    cluster.sync();
    DS_TRACE_AT(0, 7);
    for (int cr = 0; cr < crank; ++cr) {
      const uint32_t *rc = cluster.map_shared_rank(sh.cnt, cr);
      base_sel += rc[0] + rc[1];
    }
    if (whole2) {
      kB = P2 << kSh2;
    } else if (fits2) {
      uint32_t off = 0;
      for (int cr = 0; cr < nch; ++cr) {
        const uint32_t m = cr == crank ? sh.nmem : cluster.map_shared_rank(&sh.nmem, cr)[0];
        const uint2 *rmem = cluster.map_shared_rank(sh.members, cr);
        for (int i = tid; i < (int)m; i += kThreads) sh.gathered[off + i] = rmem[i];
        off += m;
      }
      __syncthreads();
      const int nm = (int)cnt2;
      for (int i = tid; i < nm; i += kThreads) {
        const uint2 me = sh.gathered[i];
        uint32_t rank = 0;
        for (int j = 0; j < nm; ++j) {
          const uint2 o = sh.gathered[j];
          rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);
        }
        if (rank == need2 - 1) {
          sh.state[6] = me.x;
          sh.state[7] = me.y;
        }
        if (rank < need2 && (int)me.y < t0) atomicAdd(&sh.lower_sel, 1u);
      }
      __syncthreads();
      kB = sh.state[6];
      tB = (int)sh.state[7];
      base_sel += sh.lower_sel;
    } else {
      // ---- massive ties at P2: level-3 digit (bits 9..0) over the cluster,
      // then the token order among keys equal to kB
      uint32_t *h3 = sh.h1;  // h1 / c1 are no longer read by any CTA (after S2)
      uint32_t *c3 = sh.c1;
      for (int i = tid; i < kD3; i += kThreads) h3[i] = 0;
      __syncthreads();
      for_each_cand([&](uint32_t key, int t) {
        if ((key >> kSh2) == P2) atomicAdd(&h3[key & (kD3 - 1)], 1u);
      });
      __syncthreads();
      coarse_sums<32>(h3, c3);
      cluster.sync();
      if (warp == 0) {
        const Boundary<1> d3 = cluster_boundary<32>(cluster, nch, h3, c3, need2);
        if (lane == 0) {
          sh.state[6] = (uint32_t)d3.bin;
          sh.state[7] = d3.above;
        }
      }
      __syncthreads();
      const uint32_t D3 = sh.state[6];
      kB = (P2 << kSh2) | D3;
      const uint32_t rem = need2 - sh.state[7];  // keys == kB to take, in token order
      uint32_t eq_lower = 0;
      for (int cr = 0; cr < crank; ++cr) eq_lower += cluster.map_shared_rank(h3, cr)[D3];
      const uint32_t my_eq = h3[D3];
      const uint32_t take = rem > eq_lower ? min(rem - eq_lower, my_eq) : 0u;
      // tB = my take-th key equal to kB in token order (none: -1, all: max)
      if (take == 0) {
        tB = -1;
      } else if (take == my_eq) {
        tB = 0x7fffffff;
      } else {
        uint32_t e = 0;  // per-warp counts of keys == kB
        for (int base = w0; base < w1; base += 32)
          e += __popc(__ballot_sync(0xffffffffu, base + lane < w1 && keys[base + lane] == kB));
        __syncthreads();
        if (lane == 0) sh.wcnt[warp] = e;
        __syncthreads();
        uint32_t before = 0;
        for (int w = 0; w < warp; ++w) before += sh.wcnt[w];
        if (before < take && before + e >= take) {  // this warp holds the take-th one
          uint32_t run = before;
          for (int base = w0; base < w1; base += 32) {
            const bool q = base + lane < w1 && keys[base + lane] == kB;
            const uint32_t m = __ballot_sync(0xffffffffu, q);
            if (run + __popc(m) >= take) {
              const int sel = __fns(m, 0, (int)(take - run));
              if (lane == 0) sh.state[5] = (uint32_t)(t0 + base + sel);
              break;
            }
            run += __popc(m);
          }
        }
        __syncthreads();
        tB = (int)sh.state[5];
      }
      // per-warp selected counts and the CTA total, exchanged once more
      uint32_t g = 0;
      for (int base = w0; base < w1; base += 32) {
        const int li = base + lane;
        const uint32_t key = li < w1 ? keys[li] : 0u;
        g += __popc(__ballot_sync(0xffffffffu, li < w1 && (key > kB || (key == kB && t0 + li <= tB))));
      }
      __syncthreads();
      if (lane == 0) sh.wcnt[warp] = g;
      __syncthreads();
      if (tid == 0) {
        uint32_t s = 0;
        for (int w = 0; w < kWarps; ++w) s += sh.wcnt[w];
        sh.cnt[3] = s;
      }
      cluster.sync();
      base_sel = 0;
      for (int cr = 0; cr < crank; ++cr) base_sel += cluster.map_shared_rank(sh.cnt, cr)[3];
    }
  }
  DS_TRACE_AT(0, 8);

  // ---- ordered write of the selected tokens (ascending) + their row ids:
  // lane l of warp w owns the l-th 32-token group of the warp's range
  {
    uint32_t sel = 0;
    if (lane < ng) {
      sel = sh.gtm[grp];
      uint32_t e = sh.eqm[grp];
      while (e) {
        const int bit = __ffs(e) - 1;
        e &= e - 1;
        const uint32_t key = keys[grp * 32 + bit];
        if (key > kB || (key == kB && t0 + grp * 32 + bit <= tB)) sel |= 1u << bit;
      }
    }
    const uint32_t cntl = __popc(sel);
    uint32_t incl = cntl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    __syncthreads();  // wcnt is scratch of the passes above
    if (lane == 31) sh.wcnt[warp] = incl;
    __syncthreads();
    uint32_t pos = base_sel + incl - cntl;
    for (int w = 0; w < warp; ++w) pos += sh.wcnt[w];
    DS_TRACE_AT(0, 10);
    while (sel) {
      const int bit = __ffs(sel) - 1;
      sel &= sel - 1;
      const int t = t0 + grp * 32 + bit;
      idx_out[pos] = t;
      rid_out[pos] = rowid_of(t);
      ++pos;
    }
  }
  DS_TRACE_AT(0, 5);
  // ---- S4: exit guard (DSMEM lifetime) + every CTA's writes done; publish
  cluster.sync();
  if (crank == 0 && tid == 0) {
    __threadfence();
    atomicExch(p.ready + unit, 1u);
  }
  DS_TRACE_AT(0, 6);
}

// ------------------------------------------------------------- launch
template <typename T, int R>
static cudaError_t launch_score_t(const ScoreParams &p, int units, int nch, size_t smem, cudaStream_t st) {
  static PerDeviceOnce once;
  const cudaError_t attr = once([] {
    cudaError_t e = cudaFuncSetAttribute(score_select_kernel<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxDynSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(score_select_kernel<T, R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  });
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, units);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = nch;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, score_select_kernel<T, R>, p);
}

SelectGeom select_geom(const ds_cache *c) {
  SelectGeom g{};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * c->num_kv_heads;
  // cluster size: as many CTAs per unit as fill the GPU at 2 CTAs/SM (<= 8,
  // portable), more only if a chunk's keys would not fit in shared memory
  int nch = (2 * sms) / units;
  if (nch > 8) nch = 8;
  const int need = (c->max_seq_len + kMaxChunkLen - 1) / kMaxChunkLen;
  if (nch < need) nch = need;
  if (nch < 1) nch = 1;
  if (nch > kMaxChunks) nch = kMaxChunks;
  int chunk = (c->max_seq_len + nch - 1) / nch;
  chunk = (chunk + 255) & ~255;
  g.chunk = chunk;
  g.nchunks = (c->max_seq_len + chunk - 1) / chunk;
  // keys [chunk] + 128 pad + this chunk's block-table entries (if few enough)
  const int pages = chunk / c->page_size + 2;
  g.score_smem = ((size_t)chunk + 128) * 4 + (pages <= kMaxPageRow ? (size_t)pages * 4 : 0);
  g.score_smem = (g.score_smem + 15) & ~(size_t)15;
  g.threads = kThreads;
  return g;
}

cudaError_t launch_score(const ds_cache *c, const ScoreParams &p, const SelectGeom &g, cudaStream_t st) {
  const int units = c->batch * c->num_kv_heads;
  if (g.chunk > kMaxChunkLen || g.nchunks > kMaxChunks || g.score_smem > (size_t)kMaxDynSmem)
    return cudaErrorInvalidValue;
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
