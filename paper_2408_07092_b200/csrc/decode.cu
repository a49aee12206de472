// decode.cu -- Algorithm 1 in ONE kernel for the serving shape:
// many (b, KV head) units, S <= 32K tokens, 16-bit KV.  One 1024-thread CTA
// per unit keeps all S approximate scores on chip (128 KB of order keys),
// so the exact top-k needs only CTA barriers, and the K/V gathers of the
// attention start while the selection is still being finished:
//
//   a1  q_lab = group-summed q[C]                         (reading R3)
//   a2  s_hat[t] = fp32 fma chain over j (no 1/sqrt(d))  (reading R2), 32
//       warps streaming the contiguous label rows with eight 128-bit loads in
//       flight per thread; keys + a 12-bit histogram of their top bits.
//   a3  exact argtopk, ties to the lower index (reading R6):
//         D1 = boundary digit of bits 31..20  -> every token with a larger
//              digit is selected (typically ~60-90% of k), marked in 32-bit
//              ballot masks per 32-token group;
//         the D1 tokens (a few hundred) form a candidate list;
//       then the CTA splits into two roles
//         warps 16..31 (selection tail): 10-bit digit of bits 19..10 over the
//              candidates, exact ranking of the <= 512 keys sharing the 22-bit
//              boundary prefix, (ties: bits 9..0, then token order), marks the
//              selected candidates, writes the optional index list;
//         warps 0..15 (attention): a4/a5 over the rows already known to be
//              selected, then (named barrier) over the marked candidates.
//   a4  s = softmax(q K_i^T / sqrt(d)), a5 y = s V_i, flash-decoding style:
//       per warp, batches of 8 rows gathered with cp.async (16 B chunks,
//       XOR-swizzled, 2 stages) into the key buffer (free once the masks
//       exist); S = Q K^T on tensor cores (mma m16n8k16, heads as M), online
//       softmax in base 2, O^T += V^T P^T (mma m16n8k8, P re-used from the S
//       fragments), fp32 accumulators; the 16 warp partials merge in shared
//       memory and y is rounded once (RNE).
//
// Softmax and the output do not depend on the order in which the selected
// rows are visited (up to fp32 rounding), which is what lets the attention
// start before the boundary is resolved.
//
// Variants (runtime-uniform branches; everything after the order keys is
// shared): the label format (16-bit bit copy R8, 4-bit codes + scale R16, or
// none -- channels read from the K rows, the Table 4 ablation); the GQA
// reading (group sum R3, max / per query head R17); a fused a0 of the new
// token (ds_decode_attention_append); select-only for the offload prefetch
// (a6).  Few units or S > 32K: a thread-block cluster of CTAs per unit, the
// selection exchanging histograms and members over DSMEM.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

#include "ds_common.cuh"
#include "ds_internal.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ds {
namespace fused {

#ifdef DS_EXP_NOHIST  // timing experiment only (wrong results): no digit-1 histogram
#define DS_HIST_ADD(p) ((void)(p))
#else
#define DS_HIST_ADD(p) atomicAdd((p), 1u)
#endif

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kAttWarps = 16;  // warps [0, 16): attention; [16, 32): selection tail
constexpr int kAttThreads = kAttWarps * 32;
constexpr int kSelThreads = kThreads - kAttThreads;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kUnroll = 8;
constexpr int kMaxS = 32768;
constexpr int kMaxR = 256;
constexpr int kSh1 = 20, kD1 = 4096;  // digit 1: key bits 31..20
constexpr int kSh2 = 10, kD2 = 1024;  // digit 2: key bits 19..10
constexpr int kD3 = 1024;             // digit 3: key bits 9..0
constexpr int kCandCap = 2048;        // digit-1 boundary tokens listed
constexpr int kMaxMembers = 512;      // 22-bit-prefix boundary tokens ranked directly
constexpr int kListCap = 2048 + 64;   // pool rows per attention round (k = 2048 + batch alignment)
constexpr int kExtCap = 2 * kCandCap - 64;  // list positions continued in a dead candidate buffer
constexpr int kBatch = 8;             // rows per warp batch
constexpr int kBarAtt = 1, kBarSel = 2, kBarDone = 3, kBarRegs = 4;  // named barriers
// register split after the common phases (64 per thread at launch):
// attention warpgroups 0-3 grow, selection warpgroups 4-7 shrink
constexpr int kAttRegs = 88, kSelRegs = 40, kCommonRegs = 64;
static_assert(kThreads * kCommonRegs <= 65536, "launch register budget (__launch_bounds__(kThreads, 1))");
static_assert(kAttThreads * kAttRegs + kSelThreads * kSelRegs <= 65536, "register file");

struct alignas(128) Sh {
  float qlab[kMaxR];
  uint32_t h1[kD1];  // digit-1 histogram; the tie path re-uses it for digit 3
  uint32_t c1[64];
  uint32_t h2[kD2];
  uint32_t c2[32];
  uint2 cand[kCandCap];        // (key, token) with digit1 == D1
  uint2 members[kMaxMembers];  // (key, token) with the boundary 22-bit prefix
  uint32_t gtm[kMaxS / 32];    // per group: digit1 > D1 (>= D1 when D1 is taken whole)
  uint32_t eqm[kMaxS / 32];    // per group: digit1 == D1; the tie path: key == kB
  uint32_t selm[kMaxS / 32];   // per group: selected digit-1 boundary tokens
  uint32_t list[kListCap];     // pool row ids of the current attention round
  uint32_t wtot[kWarps];
  uint32_t state[16];
  uint32_t cnt[4];             // [3] this CTA's selected count (read remotely)
  uint32_t ncand, nmem, lower_sel, pad0;
  uint64_t xbar[4];            // cluster exchange barriers of the selection warps
  float newlab[kMaxR];         // fused append: the new token's label values (int4: codes)
  float newscale;              // fused append, int4: its scale
  int newpage;                 // fused append: the physical page of the new token (cp.async)
  alignas(16) uint8_t newkv[2 * 128 * 2];  // fused append: the new token's K row then V row (cp.async)
  alignas(16) uint8_t qt[8 * 128 * 2];  // query rows (heads >= G zero), 16-B chunks swizzled
};

template <int D>
struct Geo {
  static constexpr int ROWB = D * 2;                    // bytes per K / V row
  static constexpr int CHN = ROWB / 16;                 // 16-B chunks per row
  static constexpr int STAGE = 2 * kBatch * ROWB;       // K rows then V rows of a batch
  static constexpr int RING = kAttWarps * 2 * STAGE;    // 2 stages per attention warp
  // warp partials: m, l per head, O rows with a stride of D + 4 floats, so
  // the fragment stores of one warp (heads 2tq, 2tq + 1; columns gq) hit 32
  // distinct banks
  static constexpr int WOS = D + 4;
  static constexpr int PART = (2 * kAttWarps * 8 + kAttWarps * 8 * WOS) * 4;
  static constexpr int CPART = (16 + 8 * D + 8 * kAttWarps) * 4;          // then the CTA partial + weights
  static_assert(CHN >= 8, "row swizzle needs >= 8 chunks");
};

__device__ __forceinline__ uint32_t swz(int row, int ch) { return (uint32_t)((ch ^ (row & 7)) << 4); }

// cluster-wide exchange among the selection warps of the nch CTAs of a
// unit: mbarrier xb of every CTA expects one arrival per CTA.
__device__ __forceinline__ void xchg_arrive(uint64_t *xb, int nch) {
  const uint32_t a = smem_u32(xb);
  // one cluster-scope release (cumulative over the CTA's writes ordered
  // before it by the preceding barrier), then relaxed arrivals
  asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
  for (int cr = 0; cr < nch; ++cr) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(a), "r"(cr));
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra) : "memory");
  }
}
__device__ __forceinline__ void xchg_wait(uint64_t *xb) {
  const uint32_t a = smem_u32(xb);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a)
        : "memory");
}

// Cluster barrier without a release per thread (barrier.cluster.arrive
// defaults to .release, which costs every arriving thread a cluster-scope
// fence): one fence.acq_rel.cluster per warp by lane 0 -- cumulative over the
// warp's writes, ordered before it by __syncwarp -- then relaxed arrivals and
// the acquiring wait.  publish = false: the warp has nothing to release.
__device__ __forceinline__ void cluster_sync_warp(bool publish) {
  __syncwarp();
  if (publish && (threadIdx.x & 31) == 0) asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
  __syncwarp();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}

// cluster_sum of uint2 loads (both halves summed; one 8-B DSMEM load per CTA)
template <typename F>
__device__ __forceinline__ uint2 cluster_sum2(int nch, F &&load) {
  uint2 s = make_uint2(0u, 0u);
  for (int c0 = 0; c0 < nch; c0 += 8) {
    uint2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = c0 + j < nch ? load(c0 + j) : make_uint2(0u, 0u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s.x += v[j].x;
      s.y += v[j].y;
    }
  }
  return s;
}

// sum over the cluster's CTAs of load(cr): the DSMEM loads of up to 8 CTAs
// are issued together, so a reduction costs one round trip per 8 CTAs
template <typename F>
__device__ __forceinline__ uint32_t cluster_sum(int nch, F &&load) {
  uint32_t s = 0;
  for (int c0 = 0; c0 < nch; c0 += 8) {
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = c0 + j < nch ? load(c0 + j) : 0u;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  return s;
}

// CL: a cluster of CTAs per unit.  PV: the label format and the group-sum
// reading fixed at compile time -- 1: the 16-bit label (the serving
// variant), 2: the 4-bit label (R16) -- so the label-format / GQA branches
// are compiled out and the code is compact (the serial phases between the
// streams are otherwise slowed by instruction-cache misses); 0: every
// format and GQA reading chosen at run time
template <typename T, int R, int D, bool CL, int PV>
__global__ void __launch_bounds__(kThreads, 1) decode_kernel(FusedParams p) {
  using GE = Geo<D>;
  constexpr int ROWB = GE::ROWB, CHN = GE::CHN, STAGE = GE::STAGE;
  constexpr int NKS = D / 16;  // QK k-steps; also O^T m-tiles
  extern __shared__ __align__(128) uint8_t smem[];
  Sh &sh = *reinterpret_cast<Sh *>(smem);
  uint8_t *region = smem + sizeof(Sh);  // keys, then the attention ring, then the partials
  uint32_t *keys = reinterpret_cast<uint32_t *>(region);
  cg::cluster_group cluster = cg::this_cluster();
  const int nch = CL ? (int)cluster.num_blocks() : 1, crank = CL ? (int)cluster.block_rank() : 0;
  // shared memory of CTA cr of the cluster (the local array without a cluster)
  auto remote = [&](auto *ptr, int cr) {
    if constexpr (CL) return cluster.map_shared_rank(ptr, cr);
    else return ptr;
  };
  const CacheView &c = p.c;
  const bool lq4 = PV == 2 || (PV == 0 && c.lq4), lnone = PV == 0 && c.lnone;  // label format (R16 / Table 4)
  const int greduce = PV ? (int)DS_GROUP_SUM : (int)c.greduce;                 // GQA reading (R3 / R17)
  // a unit is one (b, KV head) -- or one (b, query head) for DS_GROUP_PER_HEAD
  // (reading R17: each query head selects on its own over its KV head's data)
  const bool perh = greduce == DS_GROUP_PER_HEAD;
  const int unit = blockIdx.y;
  const int nuh = perh ? c.Hq : c.Hkv;  // units per sequence
  const int b = unit / nuh, hu = unit - (unit / nuh) * nuh;
  const int h = perh ? hu / c.G : hu;    // the KV head
  const int G = perh ? 1 : c.G;          // query heads this unit serves
  const int hq0 = perh ? hu : h * c.G;   // the first of them
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  DS_TRACE_AT(1, 0);
  if (CL && tid == 0) {
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&sh.xbar[i])), "r"(nch) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // The label rows of this CTA's chunk (and its block-table slice) go to L2
  // before the wait: the preceding kernel does not produce them (it may
  // write one new row, which the L2 keeps coherent; they are read into
  // registers only after the wait), so their HBM reads overlap its drain.
  auto l2_prefetch_chunk = [&] {
    const int t0p = crank * p.chunk, mloc = max(0, min(p.chunk, c.Smax - t0p));
    const size_t lr0 = ((size_t)b * c.Hkv + h) * (size_t)c.Smax + t0p;
    if (!p.l2_prefetch) {
    } else if (tid == 0 && !lnone) {
      if (!lq4) {
        prefetch_l2((const T *)c.label + lr0 * (size_t)c.r, (size_t)mloc * c.r * sizeof(T));
      } else if (((lr0 * c.rb) & 15) == 0 && ((lr0 * sizeof(T)) & 15) == 0) {
        prefetch_l2((const uint8_t *)c.label + lr0 * c.rb, (size_t)mloc * c.rb);
        prefetch_l2((const T *)c.label_scale + lr0, (size_t)mloc * sizeof(T));
      }
    }
    // the block-table slice (the row ids of the gathers) always: a few KB,
    // L2-resident by the time the selected rows are looked up (c3 40.9 ->
    // 40.8 us)
    if (tid == 32) {
      const int pg0 = t0p / c.P, npg = (mloc + c.P - 1) / c.P + 1;
      const int32_t *btp = c.block_table + (size_t)b * c.maxp + pg0;
      if (((uintptr_t)btp & 15) == 0) prefetch_l2(btp, (size_t)min(npg, c.maxp - pg0) * 4 & ~(size_t)15);
    }
  };
  l2_prefetch_chunk();
  pdl_wait();  // label / KV rows may come from the preceding append
  // (dependents are released only after the register split below: a CTA of
  // the next kernel must not take the registers the selection warps free)
  DS_TRACE_AT(2, 2);
  // The prologue's own round trips (seq_lens, the channel set C) are issued
  // first and together, so they are one DRAM latency, not a chain of them
  const int n = c.seq_lens[b];
  const int r = R > 0 ? R : c.r;
  int chj = 0;
  if (tid < r) chj = __ldg(c.C + (size_t)h * c.r + tid);
  const int t0 = crank * p.chunk;  // this CTA's tokens [t0, t0 + nloc)
  const size_t lrow = ((size_t)b * c.Hkv + h) * (size_t)c.Smax + t0;  // first label row of this CTA
  const T *lab = (const T *)c.label + lrow * (size_t)c.r;
  const uint8_t *cod = (const uint8_t *)c.label + lrow * (size_t)c.rb;  // 4-bit label (R16)
  const T *scl = (const T *)c.label_scale + lrow;
  // the query tile goes first, straight into shared memory (cp.async; rows
  // >= G zero-filled), ahead of the label prefetch in the memory queues; it
  // is waited for before the prologue's first barrier
  const T *qb = (const T *)p.q + ((size_t)b * c.Hq + (size_t)hq0) * D;
  for (int i = tid; i < 8 * CHN; i += kThreads) {
    const int row = i / CHN, ch = i - (i / CHN) * CHN;
    cp_async16(smem_u32(sh.qt + row * ROWB + swz(row, ch)), qb + (size_t)min(row, G - 1) * D + ch * 8,
               row < G ? 16 : 0);
  }
  // fused append (a0 of the new token): its K and V rows are staged in shared
  // memory by cp.async with the query tile (no registers, no wait here); the
  // CTA whose chunk holds the token writes them, and its label row, after the
  // stream (the stream may read the old label row: that one key is re-scored)
  static_assert(2 * D * 2 <= (int)sizeof(Sh::newkv), "new K/V row buffer");
  if (p.k_new && tid < 2 * CHN) {
    const T *src = (const T *)(tid < CHN ? p.k_new : p.v_new) + ((size_t)b * c.Hkv + h) * D;
    cp_async16(smem_u32(sh.newkv + tid * 16), src + (tid % CHN) * 8, 16);
  }
  cp_async_commit();
  const int pn = p.k_new ? p.positions[b] : -1;  // the new token's position (uniform)
  // No label rows are requested before the prologue's own round trips
  // (seq_lens, C, the query tile) are back: a first batch of 16 MiB issued
  // ahead of them queued them behind it (c3: 2.0 us instead of 0.7 us until
  // n is known; decode 41.4 -> 40.6 us without it).  The 4-bit label loads
  // its first two code groups once n is known (its loop keeps two in flight).
  const int maxloc = max(0, min(p.chunk, c.Smax - t0));
  constexpr bool kVec16 = R > 0 && R * sizeof(T) == 16;  // one 16-B label row per token
  constexpr int U = kUnroll;
  const bool q4v = R == 8 && lq4 && (c.Smax & 3) == 0;  // 16-B code / 8-B scale vectors of 4 tokens
  // (int4: codes of the first two groups in pv[0..1], their scales in pv[2])
  uint4 pv[U];
  auto first_batch = [&] {
    if (!lnone && greduce != DS_GROUP_MAX && lq4 && q4v) {
      const int mg = maxloc >> 2;
      const uint2 z2 = make_uint2(0, 0);
      uint2 a2 = z2, b2 = z2;
      pv[0] = pv[1] = make_uint4(0, 0, 0, 0);
      if (tid < mg) pv[0] = ldg_nc_v4(reinterpret_cast<const uint4 *>(cod) + tid), a2 = ldg_nc_v2(reinterpret_cast<const uint2 *>(scl) + tid);
      if (tid + kThreads < mg)
        pv[1] = ldg_nc_v4(reinterpret_cast<const uint4 *>(cod) + tid + kThreads),
        b2 = ldg_nc_v2(reinterpret_cast<const uint2 *>(scl) + tid + kThreads);
      pv[2] = make_uint4(a2.x, a2.y, b2.x, b2.y);
    }
  };
  const int keff = min(p.k, n);
  DS_TRACE_AT(2, 3);
  const int nloc = max(0, min(p.chunk, n - t0));
  T *outp = (T *)p.out + ((size_t)b * c.Hq + (size_t)hq0) * D;
  int32_t *idx = p.idx ? p.idx + (size_t)unit * p.k : nullptr;
  if (n <= 0) {  // empty sequence: y = 0, nothing selected (uniform over the cluster)
    cp_async_wait<0>();
    if (crank == 0) {
      if (!p.select_only)
        for (int i = tid; i < G * D; i += kThreads) outp[i] = Elem<T>::from_f(0.f);
      if (idx)
        for (int i = tid; i < p.k; i += kThreads) idx[i] = -1;
    }
    return;
  }
  first_batch();

  // ---- a1, query tile, zeroing (the tile and C are loaded together; q_lab
  // is then summed from the tile in shared memory)
  for (int i = tid; i < kD1; i += kThreads) sh.h1[i] = 0;
  for (int i = tid; i < kD2; i += kThreads) sh.h2[i] = 0;
  for (int i = tid; i < kMaxS / 32; i += kThreads) sh.selm[i] = 0;
  if (tid < 4) sh.cnt[tid] = 0;
  if (tid == 0) {
    sh.ncand = 0;
    sh.nmem = 0;
    sh.lower_sel = 0;
  }
  // DS_LABEL_NONE: the chunk's block-table entries (cand is free until the masks)
  int32_t *btc = reinterpret_cast<int32_t *>(sh.cand);
  const int pg0 = t0 / c.P;
  const int npg = nloc > 0 ? (t0 + nloc - 1) / c.P - pg0 + 1 : 0;
  const bool btc_ok = lnone && npg <= (int)(sizeof(sh.cand) / 4);
  if (btc_ok)
    for (int i = tid; i < npg; i += kThreads) btc[i] = __ldg(c.block_table + (size_t)b * c.maxp + pg0 + i);
  cp_async_wait<0>();  // this thread's part of the query tile (and the new K / V rows)
  __syncthreads();
  DS_TRACE_AT(2, 4);
  // fused append, owner CTA: the new token's page entry (waited for after the
  // stream) and its r label values from the staged K row
  const bool own_new = pn >= t0 && pn < t0 + nloc;
  if (own_new) {
    if (tid == 0) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(&sh.newpage)),
                   "l"(c.block_table + (size_t)b * c.maxp + pn / c.P)
                   : "memory");
      cp_async_commit();
    }
    const T *kn = reinterpret_cast<const T *>(sh.newkv);
    static_assert(kMaxR <= kThreads, "one label channel per thread");
    if (tid < r) sh.newlab[tid] = Elem<T>::to_f(kn[chj]);
  }
  auto qtile = [&](int g, int ch) {  // q[g][ch] from the swizzled tile
    return Elem<T>::to_f(*reinterpret_cast<const T *>(sh.qt + g * ROWB + swz(g, ch >> 3) + (ch & 7) * 2));
  };
  const bool gmax = greduce == DS_GROUP_MAX;
  if (gmax) {  // R17: per-head query labels q_g[C[j]] at qlab[g * r + j]
    for (int i = tid; i < G * r; i += kThreads) {
      const int g = i / r, j = i - (i / r) * r;
      sh.qlab[i] = qtile(g, c.C[(size_t)h * c.r + j]);
    }
  } else {
    if (tid < r) {  // Q_label[j] = sum_g q[g][C[j]], g ascending (R3); thread j = channel j
      float s = 0.0f;
      for (int g = 0; g < G; ++g) s = s + qtile(g, chj);
      sh.qlab[tid] = s;
    }
  }
  __syncthreads();
  float ql[R > 0 ? R : 1];
  if constexpr (R > 0) {
#pragma unroll
    for (int j = 0; j < R; ++j) ql[j] = sh.qlab[j];
  }
  const float *qs = R > 0 ? ql : sh.qlab;

  DS_TRACE_AT(1, 12);
  // ---- a2: stream this CTA's label rows -> order keys + digit-1 histogram
  const T *kp = (const T *)c.k_pool;
  const int32_t *btb = c.block_table + (size_t)b * c.maxp;
  auto krow = [&](int t) -> const T * {  // token t's paged K row (DS_LABEL_NONE)
    const int pg = t / c.P;
    const int32_t page = btc_ok ? btc[pg - pg0] : __ldg(btb + pg);
    return kp + (((size_t)page * c.Hkv + h) * c.P + (t - pg * c.P)) * (size_t)D;
  };
  if (gmax) {
    // R17: s_hat[t] = max_g (fma chain of q_g[C[j]] * L[t][j]) -- a plain
    // loop (diagnostic variant), every label format
    for (int i = tid; i < nloc; i += kThreads) {
      const T *kr = lnone ? krow(t0 + i) : nullptr;
      float m = -INFINITY;
      for (int g = 0; g < G; ++g) {
        const float *qv = sh.qlab + g * r;
        float s;
        if (lq4) {
          s = q4_score<T>(cod + (size_t)i * c.rb, scl[i], qv, r);
        } else {
          s = 0.0f;
          for (int j = 0; j < r; ++j)
            s = fmaf(qv[j], Elem<T>::to_f(lnone ? kr[c.C[(size_t)h * c.r + j]] : lab[(size_t)i * r + j]), s);
        }
        m = fmaxf(m, s);
      }
      const uint32_t k0 = order_key(m);
      keys[i] = k0;
      DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
    }
  } else if (lnone) {
    // no label cache (the Table 4 ablation): the r channels are
    // read straight from each token's paged K row -- 2-byte reads scattered
    // over the 256-B row, one DRAM sector or more per channel
    int i0 = tid;
    if constexpr (R > 0) {
      int chs[R];
#pragma unroll
      for (int j = 0; j < R; ++j) chs[j] = __ldg(c.C + (size_t)h * c.r + j);
      constexpr int UN = 4;
      for (; i0 + (UN - 1) * kThreads < nloc; i0 += UN * kThreads) {
        T e[UN][R];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          const T *kr = krow(t0 + i0 + u * kThreads);
#pragma unroll
          for (int j = 0; j < R; ++j) e[u][j] = __ldg(kr + chs[j]);
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[u][j]), s);
          const uint32_t k0 = order_key(s);
          keys[i0 + u * kThreads] = k0;
          DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
        }
      }
    }
    for (int i = i0; i < nloc; i += kThreads) {
      const T *kr = krow(t0 + i);
      float s = 0.0f;
      for (int j = 0; j < r; ++j) s = fmaf(qs[j], Elem<T>::to_f(kr[c.C[(size_t)h * c.r + j]]), s);
      const uint32_t k0 = order_key(s);
      keys[i] = k0;
      DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
    }
  } else if (lq4) {
    // 4-bit label (reading R16): ceil(r/2) code bytes + one scale per
    // token; s_hat = (fma chain of q_label[j] * c_j) * s
    int i0 = tid;
    if (q4v) {
      const uint4 *cv = reinterpret_cast<const uint4 *>(cod);
      const uint2 *sv = reinterpret_cast<const uint2 *>(scl);
      const int ng = nloc >> 2;
      u64 qp[8];  // {q_label[j], q_label[j]} for the packed-pair chains (R == 8 here)
#pragma unroll
      for (int j = 0; j < 8; ++j) qp[j] = pack_u2(__float_as_uint(ql[R == 8 ? j : 0]), __float_as_uint(ql[R == 8 ? j : 0]));
      auto grp = [&](int g, const uint4 &v, const uint2 &w) {
        // tokens (0, 1) and (2, 3) of the group as fp32 pairs: s_hat = chain * s
        const T *se = reinterpret_cast<const T *>(&w);
        const float2 d01 = q4_pair_dot(v.x, v.y, qp), d23 = q4_pair_dot(v.z, v.w, qp);
        const float2 p01 = unpack_f2(fmul2(pack_u2(__float_as_uint(d01.x), __float_as_uint(d01.y)),
                                           pack_u2(__float_as_uint(Elem<T>::to_f(se[0])), __float_as_uint(Elem<T>::to_f(se[1])))));
        const float2 p23 = unpack_f2(fmul2(pack_u2(__float_as_uint(d23.x), __float_as_uint(d23.y)),
                                           pack_u2(__float_as_uint(Elem<T>::to_f(se[2])), __float_as_uint(Elem<T>::to_f(se[3])))));
        const uint32_t kk[4] = {order_key(p01.x), order_key(p01.y), order_key(p23.x), order_key(p23.y)};
#pragma unroll
        for (int e = 0; e < 4; ++e) DS_HIST_ADD(&sh.h1[kk[e] >> kSh1]);
        *reinterpret_cast<uint4 *>(keys + 4 * g) = make_uint4(kk[0], kk[1], kk[2], kk[3]);
      };
      // two groups per thread in flight while the previous two are scored
      uint4 v0 = pv[0], v1 = pv[1];
      uint2 w0 = make_uint2(pv[2].x, pv[2].y), w1 = make_uint2(pv[2].z, pv[2].w);
      int g0 = tid;
      for (; g0 < ng; g0 += 2 * kThreads) {
        uint4 n0 = v0, n1 = v1;
        uint2 m0 = w0, m1 = w1;
        if (g0 + 2 * kThreads < ng) n0 = ldg_nc_v4(cv + g0 + 2 * kThreads), m0 = ldg_nc_v2(sv + g0 + 2 * kThreads);
        if (g0 + 3 * kThreads < ng) n1 = ldg_nc_v4(cv + g0 + 3 * kThreads), m1 = ldg_nc_v2(sv + g0 + 3 * kThreads);
        grp(g0, v0, w0);
        if (g0 + kThreads < ng) grp(g0 + kThreads, v1, w1);
        v0 = n0, v1 = n1, w0 = m0, w1 = m1;
      }
      i0 = 4 * ng + tid;
    }
    for (int i = i0; i < nloc; i += kThreads) {
      const uint32_t k0 = order_key(q4_score<T>(cod + (size_t)i * c.rb, scl[i], qs, r));
      keys[i] = k0;
      DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
    }
  } else {
    int i0 = tid;
    if constexpr (kVec16) {
      auto rows8 = [&](int ib, const uint4 (&v)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const T *e = reinterpret_cast<const T *>(&v[u]);
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[j]), s);
          const uint32_t k0 = order_key(s);
          keys[ib + u * kThreads] = k0;
          DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
        }
      };
      for (; i0 + (U - 1) * kThreads < nloc; i0 += U * kThreads) {
#pragma unroll
        for (int u = 0; u < U; ++u) pv[u] = __ldg(reinterpret_cast<const uint4 *>(lab) + (size_t)(i0 + u * kThreads));
        rows8(i0, pv);
      }
      if (i0 < nloc) {  // the last, partial batch: all its rows in flight at once (S = 4K: the only batch)
#pragma unroll
        for (int u = 0; u < U; ++u)
          pv[u] = i0 + u * kThreads < nloc ? __ldg(reinterpret_cast<const uint4 *>(lab) + (size_t)(i0 + u * kThreads))
                                           : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (i0 + u * kThreads >= nloc) break;
          const T *e = reinterpret_cast<const T *>(&pv[u]);
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < R; ++j) s = fmaf(ql[j], Elem<T>::to_f(e[j]), s);
          const uint32_t k0 = order_key(s);
          keys[i0 + u * kThreads] = k0;
          DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
        }
        i0 = nloc;
      }
    }
    for (int i = i0; i < nloc; i += kThreads) {
      const T *row = lab + (size_t)i * r;
      float s = 0.0f;
      for (int j = 0; j < r; ++j) s = fmaf(qs[j], Elem<T>::to_f(row[j]), s);
      const uint32_t k0 = order_key(s);
      keys[i] = k0;
      DS_HIST_ADD(&sh.h1[k0 >> kSh1]);
    }
  }
  DS_TRACE_AT(1, 13);
  if (tid < 128) keys[nloc + tid] = 0u;  // pad: below every finite score's key
  __syncthreads();
  const int pnew = pn;
  if (own_new) {  // fused append: write the new token's rows, re-score its key
    if (warp == 0) {
      // K / V rows and the 16-bit label row from the staged copies (per-head
      // mode: the G units of a KV head all write the identical bytes, and
      // each CTA's own gathers read them after the barrier below)
      if (lane == 0) cp_async_wait<0>();  // the page entry
      __syncwarp();
      const size_t dst = (((size_t)sh.newpage * c.Hkv + h) * c.P + (pnew % c.P)) * (size_t)D;
      const uint4 *src = reinterpret_cast<const uint4 *>(sh.newkv);
      for (int v = lane; v < 2 * CHN; v += 32) {
        if (v < CHN) reinterpret_cast<uint4 *>((T *)c.k_pool + dst)[v] = src[v];
        else reinterpret_cast<uint4 *>((T *)c.v_pool + dst)[v - CHN] = src[v];
      }
      if (!lq4 && !lnone) {
        const T *kn = reinterpret_cast<const T *>(sh.newkv);
        T *lr = (T *)c.label + (((size_t)b * c.Hkv + h) * c.Smax + pnew) * c.r;
        for (int j = lane; j < c.r; j += 32) lr[j] = kn[c.C[(size_t)h * c.r + j]];
      }
    }
    if (tid == 0) {
      if (lq4) {  // R16, the arithmetic of append_row_warp: codes replace the values in newlab
        float a = 0.0f;
        for (int j = 0; j < r; ++j) a = fmaxf(a, fabsf(sh.newlab[j]));
        T st = Elem<T>::from_f(a == 0.0f ? 1.0f : a / 7.0f);
        if (Elem<T>::to_f(st) == 0.0f) st = Elem<T>::from_f(1.0f);
        const float s = Elem<T>::to_f(st);
        for (int j = 0; j < r; ++j) sh.newlab[j] = fminf(fmaxf(roundf(sh.newlab[j] / s), -7.0f), 7.0f);
        sh.newscale = s;
        {  // (per-head mode: every unit of the KV head writes the same bytes)
          const size_t lr = ((size_t)b * c.Hkv + h) * c.Smax + pnew;
          uint8_t *cod = (uint8_t *)c.label + lr * c.rb;
          for (int j = 0; j < r; j += 2) {
            const int lo = (int)sh.newlab[j], hi = j + 1 < r ? (int)sh.newlab[j + 1] : 0;
            cod[j >> 1] = (uint8_t)((lo & 15) | ((hi & 15) << 4));
          }
          ((T *)c.label_scale)[lr] = st;
        }
      }
      const bool gm = greduce == DS_GROUP_MAX;
      float sc = -INFINITY;
      for (int g = 0; g < (gm ? G : 1); ++g) {
        const float *qv = sh.qlab + (gm ? g * r : 0);
        float acc = 0.0f;
        for (int j = 0; j < r; ++j) acc = fmaf(qv[j], sh.newlab[j], acc);
        if (lq4) acc = acc * sh.newscale;
        sc = gm ? fmaxf(sc, acc) : acc;
      }
      const int i = pnew - t0;
      const uint32_t stale = keys[i], fresh = order_key(sc);
      if (fresh != stale) {
        atomicSub(&sh.h1[stale >> kSh1], 1u);
        atomicAdd(&sh.h1[fresh >> kSh1], 1u);
        keys[i] = fresh;
      }
    }
    __syncthreads();
  }
  DS_TRACE_AT(1, 1);

  // ---- a3 level 1: boundary digit D1 of the cluster histogram
  const bool all_sel = keff >= n;  // (uniform over the cluster)
  // every CTA's mbarriers are initialised and its h1 / c1 complete (read
  // remotely until the first exchange) before any CTA goes on
  if (CL && !all_sel) {
    const uint4 f = reinterpret_cast<const uint4 *>(sh.h1)[tid];  // 64 coarse bins of 64
    uint32_t v = f.x + f.y + f.z + f.w;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 15) == 0) sh.c1[tid >> 4] = v;
  }
  if constexpr (CL) cluster_sync_warp(true);
  const int ngrp = (nloc + 31) >> 5;
  uint32_t D1 = 0, need1 = 0;
  bool whole1 = true, ovf = false;
  uint32_t nd1 = 0;  // this CTA's D1 tokens (an upper bound of its selected candidates)
  if (!all_sel) {
    if (!CL) {  // 64 coarse bins of 64: 4 bins per thread, 16 lanes per coarse bin
      const uint4 f = reinterpret_cast<const uint4 *>(sh.h1)[tid];
      uint32_t v = f.x + f.y + f.z + f.w;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((tid & 15) == 0) sh.c1[tid >> 4] = v;
      __syncthreads();
    }
    if (warp == 0) {
      // lane l: bins 63-2l, 62-2l of the (coarse, then fine) histogram, as one u64
      const uint2 *c1p = reinterpret_cast<const uint2 *>(sh.c1) + 31 - lane;
      uint32_t v[2];
      uint2 w = cluster_sum2(nch, [&](int cr) { return *remote(c1p, cr); });  // one round trip per 8 CTAs
      v[0] = w.y;
      v[1] = w.x;
      const Boundary<2> cb = warp_boundary<2>(v, 63, 0u, (uint32_t)keff);
      const uint2 *h1p = reinterpret_cast<const uint2 *>(sh.h1 + cb.bin * 64) + 31 - lane;
      w = cluster_sum2(nch, [&](int cr) { return *remote(h1p, cr); });
      v[0] = w.y;
      v[1] = w.x;
      const Boundary<2> fb = warp_boundary<2>(v, cb.bin * 64 + 63, cb.above, (uint32_t)keff);
      if (lane == 0) {
        sh.state[0] = (uint32_t)fb.bin;
        sh.state[1] = fb.above;
        sh.state[2] = fb.cnt;
      }
    }
    __syncthreads();
    D1 = sh.state[0];
    need1 = (uint32_t)keff - sh.state[1];
    whole1 = sh.state[2] == need1;
    nd1 = whole1 ? 0u : sh.h1[D1];
    ovf = nd1 > (uint32_t)kCandCap;  // this CTA's D1 tokens do not fit the list
  }
  DS_TRACE_AT(1, 7);
  const bool tail = !all_sel && !whole1;

  // ---- masks: per 32-token group, ballot of digit1 > D1 (>= D1 when D1 is
  // taken whole) and digit1 == D1; warp w owns groups of [w*per, w*per+per)
  {
    int per = (nloc + kWarps - 1) / kWarps;
    per = (per + 127) & ~127;
    const int w0 = min(warp * per, nloc), w1 = min(w0 + per, nloc);
    if (all_sel) {
      for (int g = tid; g < ngrp; g += kThreads) {
        const int rem = nloc - g * 32;
        sh.gtm[g] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
        sh.eqm[g] = 0u;
      }
    } else {
      // digit1 > D1 (>= D1 taken whole) <=> key >= gthr; digit1 >= D1 <=>
      // key >= elo, so digit1 == D1 is the XOR of the two (empty when D1 is
      // taken whole: gthr = elo)
      // (D1 = 4095 not taken whole: nothing lies above the top digit; the
      // all-ones threshold admits no finite score's key, R6)
      const uint32_t gthr = !whole1 && D1 == (uint32_t)(kD1 - 1) ? 0xffffffffu : (whole1 ? D1 : D1 + 1) << kSh1;
      const uint32_t elo = D1 << kSh1;
      // this warp's <= 32 groups, four at a time: a load, two compares and
      // two ballots per group, lane 0 stores the four gt words and the four
      // ge words with one 16-B store each (eqm holds digit1 >= D1 until the
      // candidate pass below turns it into digit1 == D1) -- the pass is bound
      // by the ALU pipe (2 cycles per warp instruction)
      static_assert(kMaxS / 32 / kWarps <= 32, "one group per lane in the candidate pass");
      const int g0 = w0 >> 5, ng = (w1 - w0 + 31) >> 5;  // (g0 is a multiple of 4: per is)
      const uint32_t *kw = keys + (size_t)g0 * 32 + lane;
      uint4 *gtp = reinterpret_cast<uint4 *>(sh.gtm + g0), *eqp = reinterpret_cast<uint4 *>(sh.eqm + g0);
      const bool l0 = lane == 0;
      int gi = 0;
#pragma unroll 4
      for (; gi + 4 <= ng; gi += 4) {
        uint32_t kk[4], mg[4], me[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) kk[u] = kw[(gi + u) * 32];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          mg[u] = __ballot_sync(0xffffffffu, kk[u] >= gthr);
          me[u] = __ballot_sync(0xffffffffu, kk[u] >= elo);
        }
        if (l0) {
          gtp[gi >> 2] = make_uint4(mg[0], mg[1], mg[2], mg[3]);
          eqp[gi >> 2] = make_uint4(me[0], me[1], me[2], me[3]);
        }
      }
      for (; gi < ng; ++gi) {
        const uint32_t key = kw[gi * 32];
        const uint32_t mg = __ballot_sync(0xffffffffu, key >= gthr);
        const uint32_t me = __ballot_sync(0xffffffffu, key >= elo);
        if (lane == 0) {
          sh.gtm[g0 + gi] = mg;
          sh.eqm[g0 + gi] = me;
        }
      }
      __syncwarp();
      DS_TRACE_AT(1, 8);
      if (!whole1) {  // the D1 tokens: candidate list + digit-2 histogram (lane per group)
        const int ng = (w1 - w0 + 31) >> 5, grp = (w0 >> 5) + lane;
        uint32_t e = lane < ng ? sh.eqm[grp] ^ sh.gtm[grp] : 0u;  // digit1 == D1
        if (lane < ng) sh.eqm[grp] = e;
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
  }
  DS_TRACE_AT(1, 9);
  __syncthreads();
  DS_TRACE_AT(1, 2);

  const int32_t *bt = c.block_table + (size_t)b * c.maxp;
  const bool pow2 = (c.P & (c.P - 1)) == 0;
  const int psh = __ffs(c.P) - 1;
  auto row_of = [&](int t) -> uint32_t {  // pool row id of token t (block table lookup)
    const int pg = pow2 ? (t >> psh) : t / c.P;
    const int sl = t - pg * c.P;
    return ((uint32_t)__ldg(bt + pg) * (uint32_t)c.Hkv + (uint32_t)h) * (uint32_t)c.P + (uint32_t)sl;
  };
  // list positions >= kListCap: the candidate buffer of the cluster-local
  // tail (h1) or this CTA's own candidate list (past the 32 words the list
  // building uses as scratch) -- both dead once every mark is in selm, and
  // neither read by another CTA by then
  static_assert(sizeof(Sh::h1) / 4 >= kExtCap && sizeof(Sh::cand) / 4 - 64 >= kExtCap, "extended list");
  // more certain rows than the list holds: the whole selection still fits
  // the list + its extension (this CTA selects at most its nd1 D1 tokens
  // beyond the certain rows), so no attention rounds
  auto ext_fits = [&](uint32_t n_gt) {
    return ((n_gt + kBatch - 1) & ~(uint32_t)(kBatch - 1)) + nd1 <= (uint32_t)(kListCap + kExtCap);
  };
  auto ext_list = [&](bool loc) -> uint32_t * {
    return loc ? reinterpret_cast<uint32_t *>(sh.h1) : reinterpret_cast<uint32_t *>(sh.cand) + 64;
  };
  if (tid == 0) {
    sh.state[14] = 0u;  // candidate rows not listed yet (read by the attention warps)
    sh.state[15] = 0u;  // the attention warps' batch cursor
  }
  __syncthreads();

  if (warp >= kAttWarps) {
    // ================================================ selection tail
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kSelRegs));
    named_sync(kBarRegs, kThreads);  // the attention warps hold their registers
    pdl_trigger();
    const int stid = tid - kAttThreads, sw = warp - kAttWarps;
    // Cluster-local tail (uniform over the cluster): when the cluster's D1
    // tokens fit one list, every CTA copies all of them (one exchange, one
    // pass of DSMEM reads) into h1 -- free once every CTA is past D1 -- and
    // finishes the selection on its own, marking its own tokens: no further
    // exchanges.  Otherwise the CTAs exchange histograms and members.
    const bool loc = CL && tail && sh.state[2] <= (uint32_t)kCandCap;
    uint2 *const gcand = loc ? reinterpret_cast<uint2 *>(sh.h1) : sh.cand;
    static_assert(sizeof(sh.h1) >= kCandCap * sizeof(uint2), "cluster candidate buffer");
    const int nchx = loc ? 1 : nch;  // CTAs whose histograms / members are combined
    auto for_each_cand = [&](auto &&f) {  // (key, global token) with digit1 == D1: this CTA's, or the cluster's
      if (loc) {
        const int nc = (int)sh.state[2];
        for (int i = stid; i < nc; i += kSelThreads) f(gcand[i].x, (int)gcand[i].y);
      } else if (!ovf) {
        const int nc = (int)sh.ncand;
        for (int i = stid; i < nc; i += kSelThreads) f(sh.cand[i].x, (int)sh.cand[i].y);
      } else {  // more D1 tokens than the list holds: scan the keys
        for (int i = stid; i < nloc; i += kSelThreads) {
          const uint32_t key = keys[i];
          if ((key >> kSh1) == D1) f(key, t0 + i);
        }
      }
    };
    auto mine = [&](int t) { return t >= t0 && t < t0 + nloc; };
    auto mark = [&](int t) {
      if (mine(t)) atomicOr(&sh.selm[(t - t0) >> 5], 1u << ((t - t0) & 31));
    };
    auto sel_sync = [&] { named_sync(kBarSel, kSelThreads); };
    // cluster exchange point x: publish this CTA's data, wait for every CTA's
    auto exchange = [&](int x) {
      sel_sync();
      DS_TRACE_BY(0, 2 * x, kAttThreads);  // (trace build: the fused kernel borrows kind 0's slots)
      if constexpr (CL) {
        if (stid == 0) xchg_arrive(&sh.xbar[x], nch);
        xchg_wait(&sh.xbar[x]);
      }
      DS_TRACE_BY(0, 2 * x + 1, kAttThreads);
    };
    // sum of a word over the CTAs whose data is combined (just the local one
    // in the cluster-local mode)
    auto csum = [&](int n, const uint32_t *p) {
      return loc ? (n > 0 ? *p : 0u) : cluster_sum(n, [&](int cr) { return *remote(p, cr); });
    };
    // boundary of a 1024-bin histogram (32 coarse sums of 32 per CTA), over
    // the cluster or (local mode) this CTA alone
    auto boundary1024 = [&](uint32_t *hh, uint32_t *cc, uint32_t need, uint32_t *st, int x) {
      uint32_t v = hh[2 * stid] + hh[2 * stid + 1];
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((stid & 15) == 0) cc[stid >> 4] = v;
      if (loc) sel_sync();
      else exchange(x);
      if (sw == 0) {
        uint32_t w[1];
        w[0] = csum(nchx, cc + 31 - lane);
        const Boundary<1> cb = warp_boundary<1>(w, 31, 0u, need);
        w[0] = csum(nchx, hh + cb.bin * 32 + 31 - lane);
        const Boundary<1> fb = warp_boundary<1>(w, cb.bin * 32 + 31, cb.above, need);
        if (lane == 0) {
          st[0] = (uint32_t)fb.bin;
          st[1] = fb.above;
          st[2] = fb.cnt;
        }
      }
      DS_TRACE_BY(0, 8 + x, kAttThreads);
      sel_sync();
      DS_TRACE_BY(0, 11 + x, kAttThreads);
    };
    if (loc) {
      // every CTA's candidate list is complete and every CTA is past D1
      // (h1 is no longer read remotely): copy the cluster's candidates
      exchange(0);
      if (sw == 0) {
        const uint32_t m = lane < nch ? remote(&sh.ncand, lane)[0] : 0u;
        uint32_t incl = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        sh.c2[lane] = incl - m;  // exclusive offset of CTA lane's candidates
      }
      for (int i = stid; i < kD2; i += kSelThreads) sh.h2[i] = 0;  // (rebuilt over the cluster's candidates)
      sel_sync();
      const int nc = (int)sh.state[2];
      for (int i = stid; i < nc; i += kSelThreads) {
        int cr = 0;
        for (int j = 1; j < nch; ++j) cr += (uint32_t)i >= sh.c2[j] ? 1 : 0;
        const uint2 e = remote(sh.cand, cr)[i - (int)sh.c2[cr]];
        gcand[i] = e;
        atomicAdd(&sh.h2[(e.x >> kSh2) & (kD2 - 1)], 1u);
      }
      sel_sync();
    }
#ifdef DS_TRACE  // (trace build: the D1-bin candidate count this CTA's tail ranks)
    if (stid == 0 && blockIdx.x + blockIdx.y * gridDim.x < (unsigned)ds::kTraceCtas)
      ds::g_trace[2][blockIdx.x + blockIdx.y * gridDim.x][7] =
          1000000ull + (loc ? sh.state[2] : (!ovf ? sh.ncand : 999999u)) + (tail ? 0ull : 2000000ull);
#endif
    if (tail) {
      boundary1024(sh.h2, sh.c2, need1, sh.state + 3, 0);
      DS_TRACE_BY(1, 14, kAttThreads);
      const uint32_t P2 = (D1 << (kSh1 - kSh2)) | sh.state[3];
      const uint32_t need2 = need1 - sh.state[4];
      const uint32_t cnt2 = sh.state[5];
      const bool whole2 = cnt2 == need2;
      const bool fits2 = cnt2 <= (uint32_t)kMaxMembers;
      for_each_cand([&](uint32_t key, int t) {
        const uint32_t pfx = key >> kSh2;
        if (pfx > P2 || (whole2 && pfx == P2)) mark(t);
        else if (pfx == P2 && fits2) sh.members[atomicAdd(&sh.nmem, 1u)] = make_uint2(key, (uint32_t)t);
      });
      DS_TRACE_BY(0, 14, kAttThreads);
      if (!whole2 && fits2) {
        const uint2 *gathered = sh.members;  // (local mode: the cluster's members are all here)
        if (!loc) {
          exchange(1);  // every CTA's members are listed
          // the cluster's members land in h2 (no CTA reads it after exchange 1)
          uint2 *gm = reinterpret_cast<uint2 *>(sh.h2);
          static_assert(sizeof(sh.h2) >= kMaxMembers * sizeof(uint2), "member buffer");
          // every CTA's member count in one round trip (lane cr of warp 0), the
          // offsets in c2 (free after exchange 1), then every CTA's members in
          // one pass so the remote reads of all CTAs overlap
          if (sw == 0) {
            const uint32_t m = lane < nch ? remote(&sh.nmem, lane)[0] : 0u;
            uint32_t incl = m;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            sh.c2[lane] = incl - m;  // exclusive offset of CTA lane
          }
          sel_sync();
          for (int i = stid; i < (int)cnt2; i += kSelThreads) {
            int cr = 0;
            for (int j = 1; j < nch; ++j) cr += (uint32_t)i >= sh.c2[j] ? 1 : 0;
            gm[i] = remote(sh.members, cr)[i - (int)sh.c2[cr]];
          }
          gathered = gm;
        }
        sel_sync();
        DS_TRACE_BY(1, 15, kAttThreads);
        const int nm = (int)cnt2;  // rank by (key desc, token asc)
        for (int i = stid; i < nm; i += kSelThreads) {
          const uint2 me = gathered[i];
          if (!mine((int)me.y)) continue;
          uint32_t rank = 0;
          for (int j = 0; j < nm; ++j) {
            const uint2 o = gathered[j];
            rank += (o.x > me.x) || (o.x == me.x && o.y < me.y);
          }
          if (rank < need2) mark((int)me.y);
        }
      } else if (!whole2) {
        // massive ties at the 22-bit prefix: digit 3, then token order among
        // the keys equal to kB (h1 / c1 and eqm are no longer read by anyone;
        // local mode: h1 holds the candidates, members are unused here)
        uint32_t *h3 = loc ? reinterpret_cast<uint32_t *>(sh.members) : sh.h1, *c3 = sh.c1;
        static_assert(sizeof(sh.members) >= kD3 * sizeof(uint32_t), "digit-3 histogram");
        for (int i = stid; i < kD3; i += kSelThreads) h3[i] = 0;
        for (int g = stid; g < ngrp; g += kSelThreads) sh.eqm[g] = 0;
        if (stid == 0) sh.lower_sel = sh.cnt[1] = 0;
        sel_sync();
        for_each_cand([&](uint32_t key, int t) {
          if ((key >> kSh2) == P2 && (loc || mine(t))) atomicAdd(&h3[key & (kD3 - 1)], 1u);
        });
        sel_sync();
        boundary1024(h3, c3, need2, sh.state + 6, 2);
        const uint32_t kB = (P2 << kSh2) | sh.state[6];
        const uint32_t rem = need2 - sh.state[7];  // keys == kB taken, lowest tokens first
        for_each_cand([&](uint32_t key, int t) {
          if ((key >> kSh2) == P2 && key > kB) mark(t);
          else if (key == kB) {
            if (mine(t)) {
              atomicOr(&sh.eqm[(t - t0) >> 5], 1u << ((t - t0) & 31));
              if (loc) atomicAdd(&sh.cnt[1], 1u);
            } else if (t < t0) {
              atomicAdd(&sh.lower_sel, 1u);  // (local mode: a lower CTA's key == kB)
            }
          }
        });
        sel_sync();
        // keys == kB in lower CTAs (h3 is final on every CTA after exchange 2)
        uint32_t eq_lower = 0u, my_eq = 0u;
        if (loc) {
          eq_lower = sh.lower_sel;
          my_eq = sh.cnt[1];
        } else {
          eq_lower = cluster_sum(crank, [&](int cr) { return remote(h3, cr)[kB & (kD3 - 1)]; });
          my_eq = h3[kB & (kD3 - 1)];
        }
        const uint32_t take = rem > eq_lower ? min(rem - eq_lower, my_eq) : 0u;
        sel_sync();
        if (sw == 0 && take > 0) {  // the take-th local key == kB, token order
          uint32_t run = 0;
          for (int g0 = 0; g0 < ngrp; g0 += 32) {
            const int g = g0 + lane;
            const uint32_t m = g < ngrp ? sh.eqm[g] : 0u;
            const uint32_t cnt = __popc(m);
            uint32_t incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += y;
            }
            if (run + incl >= take && run + incl - cnt < take) {
              uint32_t mm = m;  // drop the set bits before the wanted one
              for (uint32_t q = run + incl - cnt + 1; q < take; ++q) mm &= mm - 1;
              sh.state[8] = (uint32_t)(g * 32 + __ffs(mm) - 1);
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            if (run + tot >= take) break;
            run += tot;
          }
        }
        sel_sync();
        const int lB = take == 0 ? -1 : (int)sh.state[8];  // local index of the last taken key == kB
        for (int g = stid; g < ngrp; g += kSelThreads) {
          const uint32_t m = sh.eqm[g];
          const int l0 = g * 32;
          const uint32_t le = l0 + 31 <= lB ? 0xffffffffu : (l0 > lB ? 0u : ((2u << (lB - l0)) - 1u));
          if (m & le) atomicOr(&sh.selm[g], m & le);
        }
      }
      sel_sync();  // every mark is in selm
    }
    if (ovf) {
      named_arrive(kBarDone, kThreads);  // the attention warps wait for the keys buffer
    } else {
      // the selected candidates' row ids go to list positions [n_gt, n_gt + n_sel),
      // behind the attention warps' own list of the certain rows; then a flag
      // (no CTA barrier: each attention warp picks them up when it is done)
      const int ga = sw * 64 + lane, gb = ga + 32;  // warp sw: groups [64 sw, 64 sw + 64)
      const uint32_t ma = (tail && ga < ngrp) ? sh.selm[ga] : 0u;
      const uint32_t mb = (tail && gb < ngrp) ? sh.selm[gb] : 0u;
      uint32_t gt = (ga < ngrp ? __popc(sh.gtm[ga]) : 0u) + (gb < ngrp ? __popc(sh.gtm[gb]) : 0u);
      const uint32_t ca = __popc(ma), cb = __popc(mb);
      uint32_t ia = ca, ib = cb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
          ia += ya;
          ib += yb;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gt += __shfl_xor_sync(0xffffffffu, gt, o);
      const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
      if (lane == 0) {
        sh.wtot[kAttWarps + sw] = ta + tb;
        sh.cand[sw].x = gt;  // (the candidate list is no longer read)
      }
      sel_sync();
      uint32_t base = 0, n_sel = 0, n_gt = 0;
      for (int w = 0; w < kSelWarps; ++w) {
        const uint32_t x = sh.wtot[kAttWarps + w];
        if (w < sw) base += x;
        n_sel += x;
        n_gt += sh.cand[w].x;
      }
      const uint32_t p0 = (n_gt + kBatch - 1) & ~(uint32_t)(kBatch - 1);  // batch-aligned start
      // positions past the list continue in a dead candidate buffer (split-S
      // units select ~k / nch rows per CTA, which can exceed the list)
      uint32_t *const xl = ext_list(loc);
      // (n_gt > kListCap without ext_fits: the attention warps run the
      // certain rows in rounds of the list, and the candidates after them,
      // from selm)
      const bool fits = (n_gt <= (uint32_t)kListCap || ext_fits(n_gt)) && p0 + n_sel <= (uint32_t)(kListCap + kExtCap);
      if (fits && n_gt > (uint32_t)kListCap) {
        // the certain rows past the list, at the positions the attention
        // warps' list order gives them (warp sw = attention warp sw's groups)
        const uint32_t xa = ga < ngrp ? sh.gtm[ga] : 0u, xb = gb < ngrp ? sh.gtm[gb] : 0u;
        const uint32_t za = __popc(xa), zb = __popc(xb);
        uint32_t ja = za, jb = zb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t ya = __shfl_up_sync(0xffffffffu, ja, o);
          const uint32_t yb = __shfl_up_sync(0xffffffffu, jb, o);
          if (lane >= o) {
            ja += ya;
            jb += yb;
          }
        }
        const uint32_t sa = __shfl_sync(0xffffffffu, ja, 31);
        uint32_t gbase = 0;
        for (int w = 0; w < sw; ++w) gbase += sh.cand[w].x;
        uint32_t qa = gbase + ja - za, qb = gbase + sa + jb - zb;
        for (uint32_t m = xa; m; m &= m - 1, ++qa)
          if (qa >= (uint32_t)kListCap) xl[qa - kListCap] = row_of(t0 + ga * 32 + __ffs(m) - 1);
        for (uint32_t m = xb; m; m &= m - 1, ++qb)
          if (qb >= (uint32_t)kListCap) xl[qb - kListCap] = row_of(t0 + gb * 32 + __ffs(m) - 1);
      }
      if (fits) {
        uint32_t pa = p0 + base + ia - ca, pb = p0 + base + ta + ib - cb;
        for (uint32_t m = ma; m; m &= m - 1, ++pa) {
          const uint32_t rw = row_of(t0 + ga * 32 + __ffs(m) - 1);
          if (pa < (uint32_t)kListCap) sh.list[pa] = rw;
          else xl[pa - kListCap] = rw;
        }
        for (uint32_t m = mb; m; m &= m - 1, ++pb) {
          const uint32_t rw = row_of(t0 + gb * 32 + __ffs(m) - 1);
          if (pb < (uint32_t)kListCap) sh.list[pb] = rw;
          else xl[pb - kListCap] = rw;
        }
      }
      sel_sync();
      if (stid == 0) {
        sh.state[12] = p0;
        sh.state[13] = n_sel;
        __threadfence_block();
        *reinterpret_cast<volatile uint32_t *>(&sh.state[14]) = fits ? 1u : 2u;
      }
    }
    DS_TRACE_BY(1, 3, kAttThreads);
    // ---- optional index list: ascending selected tokens, -1 past k_eff
    if (idx) {
      const int ga = sw * 64 + lane, gb = ga + 32;  // warp sw: groups [64 sw, 64 sw + 64)
      const uint32_t ma = ga < ngrp ? (sh.gtm[ga] | sh.selm[ga]) : 0u;
      const uint32_t mb = gb < ngrp ? (sh.gtm[gb] | sh.selm[gb]) : 0u;
      const uint32_t ca = __popc(ma), cb = __popc(mb);
      uint32_t ia = ca, ib = cb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) {
          ia += ya;
          ib += yb;
        }
      }
      const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
      if (lane == 0) sh.wtot[kAttWarps + sw] = ta + tb;
      sel_sync();
      uint32_t base = 0, mine = 0;
      for (int w = 0; w < kSelWarps; ++w) {
        const uint32_t x = sh.wtot[kAttWarps + w];
        if (w < sw) base += x;
        mine += x;
      }
      if (stid == 0) sh.cnt[3] = mine;  // this CTA's selected tokens
      exchange(3);
      base += cluster_sum(crank, [&](int cr) { return remote(sh.cnt, cr)[3]; });
      uint32_t pa = base + ia - ca, pb = base + ta + ib - cb;
      for (uint32_t m = ma; m; m &= m - 1) idx[pa++] = t0 + ga * 32 + __ffs(m) - 1;
      for (uint32_t m = mb; m; m &= m - 1) idx[pb++] = t0 + gb * 32 + __ffs(m) - 1;
      if (crank == 0)
        for (int i = keff + stid; i < p.k; i += kSelThreads) idx[i] = -1;
    }
    if constexpr (CL) {  // the attention warps merge the cluster's partials
      cluster_sync_warp(false);
      cluster_sync_warp(false);
    }
  } else {
    // ================================================== attention warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kAttRegs));
    named_arrive(kBarRegs, kThreads);
    pdl_trigger();
    if (p.select_only) {  // a6 prefetch: the selection warps write the index list
      if (ovf) named_sync(kBarDone, kThreads);  // (matches their arrive)
      if constexpr (CL) {
        cluster_sync_warp(false);
        cluster_sync_warp(false);
      }
      return;
    }
    const int aw = warp;
    const int gq = lane >> 2, tq = lane & 3;
    const uint8_t *kp = (const uint8_t *)c.k_pool;
    const uint8_t *vp = (const uint8_t *)c.v_pool;
    const float scale = p.scale_log2;
    uint8_t *ring = region + (size_t)aw * 2 * STAGE;
    const uint32_t qbase = smem_u32(sh.qt) + (lane & 7) * ROWB;
    float o[NKS][4];
#pragma unroll
    for (int mt = 0; mt < NKS; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;

    // one batch of <= 8 rows from stage st (K rows then V rows)
    auto compute = [&](const uint8_t *st, int nvalid) {
      float sf[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t kb = smem_u32(st) + (lane & 7) * ROWB;
#pragma unroll
      for (int j = 0; j < NKS / 2; ++j) {
        const int ch = 4 * j + (lane >> 3);
        uint32_t b0, b1, b2, b3, a0, a2, a0n, a2n;
        ldmatrix_x4(kb + swz(lane, ch), b0, b1, b2, b3);
        ldmatrix_x4(qbase + swz(lane, ch), a0, a2, a0n, a2n);
        const uint32_t A0[4] = {a0, 0u, a2, 0u};
        const uint32_t A1[4] = {a0n, 0u, a2n, 0u};
        Mma<T>::run(sf, A0, b0, b1);
        Mma<T>::run(sf, A1, b2, b3);
      }
      // online softmax (base 2) for head gq over rows 2tq, 2tq+1
      const float z0 = 2 * tq < nvalid ? sf[0] * scale : -INFINITY;
      const float z1 = 2 * tq + 1 < nvalid ? sf[1] * scale : -INFINITY;
      float bm = fmaxf(z0, z1);
      bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 1));
      bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
      const float mnew = fmaxf(m_run, bm);  // finite: row 0 of a batch is valid
      const float alpha = exp2f(m_run - mnew);
      const float p0 = exp2f(z0 - mnew), p1 = exp2f(z1 - mnew);
      l_run = l_run * alpha + p0 + p1;
      m_run = mnew;
      const float alo = __shfl_sync(0xffffffffu, alpha, 8 * tq);
      const float ahi = __shfl_sync(0xffffffffu, alpha, 8 * tq + 4);
#pragma unroll
      for (int mt = 0; mt < NKS; ++mt) {
        o[mt][0] *= alo;
        o[mt][1] *= ahi;
        o[mt][2] *= alo;
        o[mt][3] *= ahi;
      }
      // P as a hi + lo pair of 16-bit values (hi = RNE(p), lo = RNE(p - hi)):
      // ~16 significant bits, so the PV product is not limited by the 8-bit
      // bf16 mantissa (R14 holds for peaked softmaxes too)
      const uint32_t bp = pack2<T>(p0, p1);
      const float2 ph = Elem<T>::unpack2(bp);
      const uint32_t bl = pack2<T>(p0 - ph.x, p1 - ph.y);
      const uint32_t vb = smem_u32(st + kBatch * ROWB) + (lane & 7) * ROWB;
#pragma unroll
      for (int j = 0; j < NKS / 2; ++j) {
        uint32_t v0, v1, v2, v3;
        ldmatrix_x4_trans(vb + swz(lane, 4 * j + (lane >> 3)), v0, v1, v2, v3);
        Mma8<T>::run(o[2 * j], v0, v1, bp);
        Mma8<T>::run(o[2 * j + 1], v2, v3, bp);
        Mma8<T>::run(o[2 * j], v0, v1, bl);
        Mma8<T>::run(o[2 * j + 1], v2, v3, bl);
      }
    };

    // attention over list positions [lo, hi): batches of 8 rows, 2 cp.async stages
    auto gather_range = [&](int lo, int hi) {
      const int nb = (hi - lo + kBatch - 1) / kBatch;
      auto issue = [&](int j) {
        uint8_t *st = ring + (j & 1) * STAGE;
        const int rb = lo + j * kBatch;
#pragma unroll
        for (int m = 0; m < kBatch * CHN / 32; ++m) {
          const int q = lane + 32 * m;
          const int rr = q / CHN, ch = q % CHN;
          const bool rv = rb + rr < hi;
          const size_t off = rv ? (size_t)sh.list[rb + rr] * ROWB + (size_t)ch * 16 : 0;
          const uint32_t dst = smem_u32(st + rr * ROWB + swz(rr, ch));
          cp_async16(dst, kp + off, rv ? 16 : 0);
          cp_async16(dst + kBatch * ROWB, vp + off, rv ? 16 : 0);
        }
      };
      if (nb > 0) issue(0);
      cp_async_commit();
      for (int j = 0; j < nb; ++j) {
        if (j + 1 < nb) issue(j + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        compute(ring + (j & 1) * STAGE, min(kBatch, hi - (lo + j * kBatch)));
        __syncwarp();  // stage fully read before it is refilled
      }
      cp_async_wait<0>();
    };
    auto split = [&](int n, int &lo, int &hi) {  // this warp's share of n rows (multiples of 8)
      int per = (n + kAttWarps - 1) / kAttWarps;
      per = (per + kBatch - 1) & ~(kBatch - 1);
      lo = min(aw * per, n);
      hi = min(lo + per, n);
    };

    // attention over this CTA's rows whose group masks are mask(g), in rounds of
    // kListCap; final_sync: end with an attention-warp barrier
    auto run_rows = [&](auto &&mask, bool final_sync) {
      const int ga = aw * 64 + lane, gb = ga + 32;  // warp aw: groups [64 aw, 64 aw + 64)
      const uint32_t ma = ga < ngrp ? mask(ga) : 0u;
      const uint32_t mb = gb < ngrp ? mask(gb) : 0u;
      const uint32_t ca = __popc(ma), cb = __popc(mb);
      uint32_t ia = ca, ib = cb;
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o2);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o2);
        if (lane >= o2) {
          ia += ya;
          ib += yb;
        }
      }
      const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
      if (lane == 0) sh.wtot[aw] = ta + tb;
      named_sync(kBarAtt, kAttThreads);
      uint32_t base = 0, total = 0;
      for (int w = 0; w < kAttWarps; ++w) {
        const uint32_t x = sh.wtot[w];
        if (w < aw) base += x;
        total += x;
      }
      named_sync(kBarAtt, kAttThreads);  // wtot read by all before any reuse
      for (uint32_t r0 = 0; r0 < total; r0 += kListCap) {
        // row ids of list positions [r0, r0 + kListCap)
        uint32_t pa = base + ia - ca, pb = base + ta + ib - cb;
        for (uint32_t m = ma; m; m &= m - 1, ++pa)
          if (pa >= r0 && pa < r0 + kListCap) sh.list[pa - r0] = row_of(t0 + ga * 32 + __ffs(m) - 1);
        for (uint32_t m = mb; m; m &= m - 1, ++pb)
          if (pb >= r0 && pb < r0 + kListCap) sh.list[pb - r0] = row_of(t0 + gb * 32 + __ffs(m) - 1);
        named_sync(kBarAtt, kAttThreads);
        int lo, hi;
        split((int)min((uint32_t)kListCap, total - r0), lo, hi);
        gather_range(lo, hi);
        if (final_sync || r0 + kListCap < total) named_sync(kBarAtt, kAttThreads);  // list consumed
      }
    };

    if (!ovf) {
      // the certain rows (digit1 > D1) at list positions [0, n_gt)
      const int ga = aw * 64 + lane, gb = ga + 32;  // warp aw: groups [64 aw, 64 aw + 64)
      const uint32_t ma = ga < ngrp ? sh.gtm[ga] : 0u;
      const uint32_t mb = gb < ngrp ? sh.gtm[gb] : 0u;
      const uint32_t ca = __popc(ma), cb = __popc(mb);
      uint32_t ia = ca, ib = cb;
#pragma unroll
      for (int o2 = 1; o2 < 32; o2 <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ia, o2);
        const uint32_t yb = __shfl_up_sync(0xffffffffu, ib, o2);
        if (lane >= o2) {
          ia += ya;
          ib += yb;
        }
      }
      const uint32_t ta = __shfl_sync(0xffffffffu, ia, 31), tb = __shfl_sync(0xffffffffu, ib, 31);
      if (lane == 0) sh.wtot[aw] = ta + tb;
      named_sync(kBarAtt, kAttThreads);
      uint32_t base = 0, n_gt = 0;
      for (int w = 0; w < kAttWarps; ++w) {
        const uint32_t x = sh.wtot[w];
        if (w < aw) base += x;
        n_gt += x;
      }
      if (n_gt <= (uint32_t)kListCap || ext_fits(n_gt)) {
        // certain rows at list positions [0, n_gt): those past the list are
        // written by the selection warps with the candidates (below)
        uint32_t pa = base + ia - ca, pb = base + ta + ib - cb;
        for (uint32_t m = ma; m && pa < (uint32_t)kListCap; m &= m - 1) sh.list[pa++] = row_of(t0 + ga * 32 + __ffs(m) - 1);
        for (uint32_t m = mb; m && pb < (uint32_t)kListCap; m &= m - 1) sh.list[pb++] = row_of(t0 + gb * 32 + __ffs(m) - 1);
        named_sync(kBarAtt, kAttThreads);  // the list of certain rows is complete
        const uint32_t *const xl = ext_list(CL && tail && sh.state[2] <= (uint32_t)kCandCap);  // (loc)
        // batches of 8 list positions handed out by a shared cursor: batches
        // below nb1 are certain rows; the selected candidates follow from
        // position 8 * nb1 once the selection warps raise the flag
        const int nb1 = ((int)n_gt + kBatch - 1) / kBatch;
        auto grab = [&](int &nvalid) -> int {  // next batch (or -1) and its valid rows
          int j = 0, nv = 0;
          if (lane == 0) {
            j = (int)atomicAdd(&sh.state[15], 1u);
            if (j < nb1 && (j + 1) * kBatch <= kListCap) {
              nv = min(kBatch, (int)n_gt - j * kBatch);
            } else if (j < nb1) {  // certain rows past the list: listed with the candidates
              while (*reinterpret_cast<volatile uint32_t *>(&sh.state[14]) == 0u) __nanosleep(64);
              __threadfence_block();
              nv = min(kBatch, (int)n_gt - j * kBatch);
            } else {
              uint32_t f;
              while ((f = *reinterpret_cast<volatile uint32_t *>(&sh.state[14])) == 0u) __nanosleep(64);
              __threadfence_block();
              const int lim = (int)sh.state[12] + (int)sh.state[13];
              if (f != 1u || j * kBatch >= lim) j = -1;
              else nv = min(kBatch, lim - j * kBatch);
            }
          }
          nvalid = __shfl_sync(0xffffffffu, nv, 0);
          return __shfl_sync(0xffffffffu, j, 0);
        };
        auto issue = [&](int j, int nv, int stg) {
          uint8_t *st = ring + stg * STAGE;
          const int rb = j * kBatch;
#pragma unroll
          for (int m = 0; m < kBatch * CHN / 32; ++m) {
            const int q = lane + 32 * m;
            const int rr = q / CHN, ch = q % CHN;
            const bool rv = rr < nv;
            const int pos = rb + rr;
            const uint32_t rid = !rv ? 0u : pos < kListCap ? sh.list[pos] : xl[pos - kListCap];
            const size_t off = (size_t)rid * ROWB + (size_t)ch * 16;
            const uint32_t dst = smem_u32(st + rr * ROWB + swz(rr, ch));
            cp_async16(dst, kp + off, rv ? 16 : 0);
            cp_async16(dst + kBatch * ROWB, vp + off, rv ? 16 : 0);
          }
        };
        int nv_cur = 0, stg = 0;
        int cur = grab(nv_cur);
        if (cur >= 0) issue(cur, nv_cur, 0);
        cp_async_commit();
        while (cur >= 0) {
          int nv_nxt = 0;
          const int nxt = grab(nv_nxt);
          if (nxt >= 0) issue(nxt, nv_nxt, stg ^ 1);
          cp_async_commit();
          cp_async_wait<1>();
          __syncwarp();
          compute(ring + stg * STAGE, nv_cur);
          __syncwarp();  // stage fully read before it is refilled
          cur = nxt;
          nv_cur = nv_nxt;
          stg ^= 1;
        }
        cp_async_wait<0>();
      } else {  // more certain rows than one list: rounds
        named_sync(kBarAtt, kAttThreads);
        run_rows([&](int g) { return sh.gtm[g]; }, false);
      }
      DS_TRACE_AT(1, 4);
      if (lane == 0)  // (the flag: set by now in the cursor path)
        while (*reinterpret_cast<volatile uint32_t *>(&sh.state[14]) == 0u) __nanosleep(64);
      __syncwarp();
      __threadfence_block();
      if (*reinterpret_cast<volatile uint32_t *>(&sh.state[14]) != 1u && tail) {
        // the candidates did not fit behind the certain rows: a list of their own
        named_sync(kBarAtt, kAttThreads);
        run_rows([&](int g) { return sh.selm[g]; }, true);
      }
    } else {  // the tail still scans the keys in this buffer: wait, then all rows
      named_sync(kBarDone, kThreads);
      run_rows([&](int g) { return sh.gtm[g] | sh.selm[g]; }, true);
    }
    DS_TRACE_AT(1, 5);
    // ---- warp partials (m, l per head; O^T fragments) -> CTA partial
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    float *wm = reinterpret_cast<float *>(region);  // [16][8]
    float *wl = wm + kAttWarps * 8;                 // [16][8]
    float *wo = wl + kAttWarps * 8;                 // [16][8][WOS]
    constexpr int WOS = GE::WOS;
    named_sync(kBarAtt, kAttThreads);               // ring no longer read
    if (tq == 0) {
      wm[aw * 8 + gq] = m_run;
      wl[aw * 8 + gq] = l_run;
    }
    // (only the G real heads: rows >= G of the tile are padding)
    const bool h0ok = 2 * tq < G, h1ok = 2 * tq + 1 < G;
#pragma unroll
    for (int mt = 0; mt < NKS; ++mt) {
      float *w0 = wo + (size_t)(aw * 8 + 2 * tq) * WOS + 16 * mt + gq;
      if (h0ok) {
        w0[0] = o[mt][0];
        w0[8] = o[mt][2];
      }
      if (h1ok) {
        w0[WOS] = o[mt][1];
        w0[WOS + 8] = o[mt][3];
      }
    }
    named_sync(kBarAtt, kAttThreads);
    DS_TRACE_AT(1, 10);
    float *cm = reinterpret_cast<float *>(region + GE::PART);  // [8] m, [8] l, [8][D] o of this CTA
    float *wsc = cm + 16 + 8 * D;                              // [8][16] per-warp weights
    if constexpr (!CL) {
      // one CTA: every output thread folds the 16 warp partials of its head
      // itself (M, then the weights 2^(m_w - M)), no weights phase and barrier
      for (int i = tid; i < G * D; i += kAttThreads) {
        const int g = i / D, dd = i - (i / D) * D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w) M = fmaxf(M, wm[w * 8 + g]);  // finite: >= 1 row (n >= 1)
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w) {
          const float e = exp2f(wm[w * 8 + g] - M);  // 0 for a warp without rows (m = -inf)
          L = fmaf(wl[w * 8 + g], e, L);
          O = fmaf(wo[(size_t)(w * 8 + g) * WOS + dd], e, O);
        }
        outp[i] = Elem<T>::from_f(O / L);
      }
    }
    if (CL && aw < G) {  // warp g: head g's weights over the 16 warps (lane w, w + 16)
      const int g = aw;
      const float m0 = lane < kAttWarps ? wm[lane * 8 + g] : -INFINITY;
      float M = m0;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
      const float e0 = (lane < kAttWarps && M != -INFINITY) ? exp2f(m0 - M) : 0.f;
      float L = lane < kAttWarps ? wl[lane * 8 + g] * e0 : 0.f;
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o2);
      // cluster: unnormalised weights; (M, L) go to the merge
      if (lane < kAttWarps) wsc[g * kAttWarps + lane] = e0;
      if (lane == 0) {
        cm[g] = M;
        cm[8 + g] = L;
      }
    }
    // ---- the cluster's partials -> y (CTA cr finishes a slice of the G*D outputs)
    if constexpr (CL) {
      named_sync(kBarAtt, kAttThreads);
      DS_TRACE_AT(1, 11);
      for (int i = tid; i < G * D; i += kAttThreads) {
        const int g = i / D, dd = i - (i / D) * D;
        float O = 0.f;
#pragma unroll
        for (int w = 0; w < kAttWarps; ++w) O = fmaf(wo[(size_t)(w * 8 + g) * WOS + dd], wsc[g * kAttWarps + w], O);
        cm[16 + i] = O;
      }
      cluster_sync_warp(true);  // every CTA's partial is complete
      const float *cm0 = reinterpret_cast<const float *>(region + GE::PART);
      const int per_cta = (G * D + nch - 1) / nch;
      const int i0 = crank * per_cta, i1 = min(i0 + per_cta, G * D);
      for (int i = i0 + tid; i < i1; i += kAttThreads) {
        const int g = i / D;
        float M = -INFINITY, L = 0.f, O = 0.f;
        for (int c0 = 0; c0 < nch; c0 += 8) {  // online merge, 8 CTAs' loads in flight
          float mm[8], ll[8], oo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (c0 + j < nch) {
              const float *rm = cluster.map_shared_rank(cm0, c0 + j);
              mm[j] = rm[g];
              ll[j] = rm[8 + g];
              oo[j] = rm[16 + i];
            } else {
              mm[j] = -INFINITY;
              ll[j] = oo[j] = 0.f;
            }
          }
          float Mn = M;
#pragma unroll
          for (int j = 0; j < 8; ++j) Mn = fmaxf(Mn, mm[j]);
          if (Mn == -INFINITY) continue;  // no rows in these CTAs yet
          const float a = exp2f(M - Mn);  // M = -inf at first: a = 0 and L = O = 0 anyway
          L *= a;
          O *= a;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float sw = exp2f(mm[j] - Mn);
            L = fmaf(ll[j], sw, L);
            O = fmaf(oo[j], sw, O);
          }
          M = Mn;
        }
        outp[i] = Elem<T>::from_f(O / L);
      }
      cluster_sync_warp(true);  // partials and exchange data stay alive until every reader is done
    }
  }
  DS_TRACE_AT(1, 6);
}

template <typename T, int R, int D>
static size_t smem_bytes(int chunk) {
  size_t region = ((size_t)chunk + 128) * 4;
  region = region > (size_t)Geo<D>::RING ? region : (size_t)Geo<D>::RING;
  region = region > (size_t)(Geo<D>::PART + Geo<D>::CPART) ? region : (size_t)(Geo<D>::PART + Geo<D>::CPART);
  return sizeof(Sh) + region;
}

template <typename T, int R, int D, bool CL, int PV>
static cudaError_t launch_cl(const ds_cache *c, const FusedParams &p, int nch, cudaStream_t st) {
  const size_t smem = smem_bytes<T, R, D>(p.chunk);
  static PerDeviceOnce once;
  const cudaError_t attr = once([] {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, R, D, CL, PV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedMaxSmem);
    if (e == cudaSuccess && CL)
      e = cudaFuncSetAttribute(decode_kernel<T, R, D, CL, PV>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  });
  if (attr != cudaSuccess) return attr;
  if (smem > (size_t)kFusedMaxSmem) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, c->batch * (c->group_reduce == DS_GROUP_PER_HEAD ? c->num_q_heads : c->num_kv_heads));
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
  cfg.attrs = CL ? a : a + 1;  // no cluster attribute for one CTA per unit
  cfg.numAttrs = CL ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, decode_kernel<T, R, D, CL, PV>, p);
}

template <typename T, int R, int D>
static cudaError_t launch_t(const ds_cache *c, const FusedParams &p, int nch, cudaStream_t st) {
  // the group-sum reading with the 16-bit or the 4-bit label (r = 8) has its
  // own compact instance
  if constexpr (R > 0) {
    if (c->group_reduce == DS_GROUP_SUM && c->label_format == DS_LABEL_NATIVE)
      return nch > 1 ? launch_cl<T, R, D, true, 1>(c, p, nch, st) : launch_cl<T, R, D, false, 1>(c, p, nch, st);
    if (c->group_reduce == DS_GROUP_SUM && c->label_format == DS_LABEL_INT4)
      return nch > 1 ? launch_cl<T, R, D, true, 2>(c, p, nch, st) : launch_cl<T, R, D, false, 2>(c, p, nch, st);
  }
  return nch > 1 ? launch_cl<T, R, D, true, 0>(c, p, nch, st) : launch_cl<T, R, D, false, 0>(c, p, nch, st);
}

// Can a cluster of nch CTAs (1024 threads, ~200 KB of shared memory each) be
// resident at all?  Portable sizes (<= 8) always can on B200; 9..16 need the
// non-portable opt-in and enough free SMs in one GPC, so ask the occupancy API.
template <typename T, int R, int D>
static bool cluster_fits_t(int nch, int chunk) {
  if (nch <= 8) return true;
  static PerDeviceOnce once;
  if (once([] {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel<T, R, D, true, 0>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedMaxSmem);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(decode_kernel<T, R, D, true, 0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e;
      }) != cudaSuccess)
    return false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nch, 1);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes<T, R, D>(chunk);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = nch;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, decode_kernel<T, R, D, true, 0>, &cfg) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of the query
    return false;
  }
  return nclusters > 0;
}

// How many clusters of n CTAs can be co-resident (1 CTA per SM at the fused
// kernel's footprint; a cluster lives in one GPC, so this is GPC-limited, not
// SMs / n).  Queried once per device for n = 2..16 -- every instance of
// decode_kernel has the same footprint (1024 threads, ~200 KB of shared
// memory, whole SM).  0 when the query fails.
static int max_active_clusters(int n) {
  static PerDeviceOnce once;
  static int mac[kMaxDevices][17];
  int dev = 0;
  if (n < 2 || n > 16 || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  const cudaError_t e = once([dev] {
    auto kern = decode_kernel<__nv_bfloat16, 8, 128, true, 0>;
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedMaxSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int m = 2; m <= 16 && r == cudaSuccess; ++m) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(m, 1);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = smem_bytes<__nv_bfloat16, 8, 128>(kMaxS);
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = m;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int nc = 0;
      r = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
      mac[dev][m] = nc;
    }
    if (r != cudaSuccess) cudaGetLastError();  // (not sticky)
    return r;
  });
  return e == cudaSuccess ? mac[dev][n] : 0;
}

}  // namespace fused

// CTAs per unit (one thread-block cluster): enough to cover the SMs when
// there are few units, enough to hold S keys on chip when S is long.
int fused_cluster(const ds_cache *c) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = c->batch * (c->group_reduce == DS_GROUP_PER_HEAD ? c->num_q_heads : c->num_kv_heads);
  // A cluster of CTAs per unit when the units cover < 3/4 of the SMs and the
  // sequences are long enough: the largest n <= 16 whose clusters of every
  // unit are co-resident in one wave (units * n <= SMs and units <= the
  // clusters of n the GPCs can hold) with chunks of >= 4K tokens.  Past the
  // co-residency limit a second wave doubles the time (16 units of S=32K:
  // 4/5/6 CTAs 20.4/19.9/19.3 us, 7 and 8 CTAs 35.5/34.7 us; 16 units of
  // S=128K: 4/6 CTAs 43.1/34.7 us, 7 CTAs 60.3 us).  Short sequences (<= 8K)
  // stay on one CTA: a cluster's fixed exchange cost outweighs the split
  // streaming/gather time (c2 S=4K: 12.6 us on one CTA, 14.0 on 4; S=16K:
  // 4 CTAs 17.3 us vs 18.9 on 2 and 22.1 on 1).
  int nch = 1;
  if (units * 4 < sms * 3 && c->max_seq_len > 8192) {
    for (int n = min(16, sms / units); n >= 2; --n) {
      if ((c->max_seq_len + n - 1) / n < 4096) continue;
      if (fused::max_active_clusters(n) < units) continue;
      nch = n;
      break;
    }
  }
  const int need = (c->max_seq_len + fused::kMaxS - 1) / fused::kMaxS;
#ifdef DS_EXP_NCH_ENV  // timing experiments only (never in libds.so): DS_NCH forces the cluster size
  if (const char *e = getenv("DS_NCH")) {
    const int v = atoi(e);
    if (v >= need && v >= 1 && v <= 16) return v;
  }
#endif
  if (nch < need) nch = need;
  if (nch < 1) nch = 1;
  return nch;
}

static int fused_chunk(const ds_cache *c, int nch) {
  int chunk = (c->max_seq_len + nch - 1) / nch;
  return (chunk + 127) & ~127;
}

bool fused_applicable(const ds_cache *c) {
  if (c->dtype != DS_BF16 && c->dtype != DS_FP16) return false;
  if (c->r > fused::kMaxR) return false;
  const int nch = fused_cluster(c);
  if (nch > 16) return false;
  const int chunk = fused_chunk(c, nch);
  if (chunk > fused::kMaxS) return false;
  using namespace fused;
#define DS_F(T)                                                                                                 \
  if (c->head_dim == 64) return c->r == 8 ? cluster_fits_t<T, 8, 64>(nch, chunk) : cluster_fits_t<T, 0, 64>(nch, chunk); \
  return c->r == 8 ? cluster_fits_t<T, 8, 128>(nch, chunk) : cluster_fits_t<T, 0, 128>(nch, chunk);
  if (c->dtype == DS_BF16) {
    DS_F(__nv_bfloat16)
  }
  DS_F(__half)
#undef DS_F
}

cudaError_t launch_fused(const ds_cache *c, FusedParams p, cudaStream_t st) {
  using namespace fused;
  const int nch = fused_cluster(c);
  const int chunk = fused_chunk(c, nch);
  if (chunk > kMaxS) return cudaErrorInvalidValue;
  p.chunk = chunk;
  {
    // label L2 prefetch before the PDL wait: measured to help when CTAs start
    // in several waves (c4: 512 units) or as clusters (c5), and to cost
    // ~1 us when every unit has one CTA of a single wave (c3: the burst
    // delays the first demand loads)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long units = (long)c->batch * (c->group_reduce == DS_GROUP_PER_HEAD ? c->num_q_heads : c->num_kv_heads);
#ifdef DS_EXP_L2PF  // timing experiment: force the phase-0 L2 prefetch on (1) or off (0)
    p.l2_prefetch = DS_EXP_L2PF;
#else
    p.l2_prefetch = nch > 1 || units * nch > sms;
#endif
  }
#define DS_F(T)                                                                                         \
  if (c->head_dim == 64) return c->r == 8 ? launch_t<T, 8, 64>(c, p, nch, st) : launch_t<T, 0, 64>(c, p, nch, st); \
  return c->r == 8 ? launch_t<T, 8, 128>(c, p, nch, st) : launch_t<T, 0, 128>(c, p, nch, st);
  if (c->dtype == DS_BF16) {
    DS_F(__nv_bfloat16)
  }
  DS_F(__half)
#undef DS_F
}

}  // namespace ds
