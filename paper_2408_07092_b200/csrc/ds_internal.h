// ds_internal.h -- host<->kernel plumbing shared by the libds.so sources.
#pragma once
#include <cuda_runtime_api.h>
#include <stdint.h>

#include <atomic>

#include "ds.h"

namespace ds {

// Flat, by-value view of a ds_cache passed to every kernel.
struct CacheView {
  int B, Hq, Hkv, D, G, P, num_pages, maxp, Smax, r;
  const void *k_pool, *v_pool;
  const int32_t *block_table, *seq_lens;
  const void *label;
  const int32_t *C;
  int lq4, rb;              // DS_LABEL_INT4; code bytes per label row (ceil(r/2))
  int lnone;                // DS_LABEL_NONE: line 2 reads the channels from the K pool
  int greduce;              // ds_group_reduce
  const void *label_scale;  // DS_LABEL_INT4: [B][Hkv][Smax] of the cache dtype
};

// score_select_kernel: a1 + a2 + a3 -> index list + pool row ids per unit.
struct ScoreParams {
  CacheView c;
  const void *q;         // [B][Hq][D]
  int k;
  uint32_t *ready;       // [units] selection published (0 between calls)
  int32_t *idx;          // [units][k] ascending token indices (-1 past k_eff)
  int32_t *rowid;        // [units][k] pool row ids of the same tokens
  float *scores;         // non-null: ds_approx_scores mode (s_hat [units][Smax] only)
  int chunk;             // tokens per CTA (cluster = nchunks CTAs per unit)
};

struct AttnParams {
  CacheView c;
  const void *q;            // [B][Hq][D]
  const int32_t *rowid;     // [units][k] pool rows (sparse) or nullptr (dense: every token)
  uint32_t *ready;          // sparse: per-unit selection flags to wait on (reset after use)
  int k;                    // selection size (sparse); ignored for dense
  int rows_per_cta;         // rows of the index list per CTA (cluster = nsplit CTAs)
  float scale_log2;         // log2(e) / sqrt(D)
  void *out;                // [B][Hq][D]
};

// decode_kernel (decode.cu): the whole of Algorithm 1 per unit in one CTA.
struct FusedParams {
  CacheView c;
  const void *q;     // [B][Hq][D]
  int k;
  void *out;         // [B][Hq][D]
  int32_t *idx;      // nullable [units][k]
  float scale_log2;  // log2(e) / sqrt(D)
  int chunk;         // tokens per CTA (cluster of ceil(S / chunk) CTAs per unit)
  int select_only;   // a6 prefetch: lines 1-3 only (idx written, no attention, out unused)
  // fused a0 (ds_decode_attention_append): one new token per sequence at
  // positions[b], k_new / v_new [B][1][Hkv][D]; nullptr = no append
  const void *k_new, *v_new;
  const int32_t *positions;
  // L2 prefetch of each CTA's label rows before griddepcontrol.wait (set by
  // launch_fused when the grid has more CTAs than SMs or clusters)
  int l2_prefetch;
};
constexpr int kFusedMaxSmem = 227 * 1024;
bool fused_applicable(const ds_cache *c);
cudaError_t launch_fused(const ds_cache *c, FusedParams p, cudaStream_t st);
cudaError_t launch_gather(const ds_cache *c, const ds_prefetch_slot *slot, cudaStream_t st);
int fused_cluster(const ds_cache *c);

// Launch-geometry decisions (deterministic functions of the cache shape).
struct SelectGeom {
  int chunk, nchunks;  // score CTAs per unit (one cluster)
  int threads;
  size_t score_smem;   // dynamic smem (a chunk's keys + its block-table entries)
};
SelectGeom select_geom(const ds_cache *c);

struct AttnGeom {
  int rows_per_cta, nsplit, threads;
  size_t smem;
};
AttnGeom attn_geom(const ds_cache *c, int n_rows);

// Workspace layout: ready flags | idx | rowid.
struct Workspace {
  uint32_t *ready;
  int32_t *idx, *rowid;
  size_t bytes;
};
Workspace carve_workspace(const ds_cache *c, int k, void *base);

// Kernel launchers (defined in the .cu files); return cudaError_t.
cudaError_t launch_append(const ds_cache *c, const void *k_new, const void *v_new,
                          const int32_t *positions, int n_new, cudaStream_t st);
cudaError_t launch_calibrate(const void *qc, const void *kc, int n, int Hq, int Hkv, int D,
                             ds_dtype dt, int mode, int r, uint64_t seed, int32_t *out,
                             cudaStream_t st);
cudaError_t launch_score(const ds_cache *c, const ScoreParams &p, const SelectGeom &g, cudaStream_t st);
cudaError_t launch_attn(const ds_cache *c, const AttnParams &p, const AttnGeom &g, cudaStream_t st);

CacheView make_view(const ds_cache *c);

// Kernel attributes (dynamic shared memory size, non-portable cluster size)
// belong to a device context, so a process driving several GPUs must set
// them once per device, not once per process.  One instance per kernel
// instantiation; f() is idempotent, so callers racing on a first use may
// both run it.
constexpr int kMaxDevices = 64;
struct PerDeviceOnce {
  std::atomic<int> done[kMaxDevices] = {};
  template <typename F>
  cudaError_t operator()(F &&f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return f();
    if (done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) done[dev].store(1, std::memory_order_release);
    return e;
  }
};

// cudaLaunchKernelEx with programmatic stream serialization (PDL): the kernel
// may start while its predecessor drains (see pdl_wait / pdl_trigger).
struct PdlLaunch {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[1];
  PdlLaunch(dim3 grid, dim3 block, size_t smem, cudaStream_t st) : cfg{} {
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  template <typename... KArgs, typename... Args>
  cudaError_t run(void (*kern)(KArgs...), Args... args) {
    return cudaLaunchKernelEx(&cfg, kern, args...);
  }
};

}  // namespace ds
