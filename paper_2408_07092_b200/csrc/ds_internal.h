// ds_internal.h -- host<->kernel plumbing shared by the libds.so sources.
#pragma once
#include <cuda_runtime_api.h>
#include <stdint.h>

#include "ds.h"

namespace ds {

// Flat, by-value view of a ds_cache passed to every kernel.
struct CacheView {
  int B, Hq, Hkv, D, G, P, num_pages, maxp, Smax, r;
  const void *k_pool, *v_pool;
  const int32_t *block_table, *seq_lens;
  const void *label;
  const int32_t *C;
};

struct SelectParams {
  CacheView c;
  const void *q;       // [B][Hq][D]
  int k;
  int32_t *idx;        // [B*Hkv][k]
  float *scores;       // non-null: ds_approx_scores mode (write s_hat, no select)
  int cap;             // key capacity per CTA (smem)
};

struct AttnParams {
  CacheView c;
  const void *q;            // [B][Hq][D]
  const int32_t *idx;       // [B*Hkv][k] or nullptr for dense
  int k;                    // selection size (sparse) ; ignored for dense
  int rows_per_cta;
  int nsplit;
  float scale_log2;         // log2(e) / sqrt(D)
  float *part_o;            // [units][nsplit][G][D]
  float *part_ml;           // [units][nsplit][G][2]
  void *out;                // [B][Hq][D]
};

// Launch-geometry decisions (deterministic functions of the cache shape).
struct SelectGeom {
  int cl;      // cluster size (CTAs per unit)
  int cap;     // keys per CTA (multiple of 32)
  int threads;
  size_t smem;
};
SelectGeom select_geom(const ds_cache *c);

struct AttnGeom {
  int rows_per_cta, nsplit, threads;
  size_t smem;
};
AttnGeom attn_geom(const ds_cache *c, int n_rows);

// Workspace layout.
struct Workspace {
  int32_t *idx;
  float *part_o, *part_ml;
  size_t bytes;
};
Workspace carve_workspace(const ds_cache *c, int k, int nsplit, void *base);

// Kernel launchers (defined in the .cu files); return cudaError_t.
cudaError_t launch_append(const ds_cache *c, const void *k_new, const void *v_new,
                          const int32_t *positions, int n_new, cudaStream_t st);
cudaError_t launch_calibrate(const void *qc, const void *kc, int n, int Hq, int Hkv, int D,
                             ds_dtype dt, int mode, int r, uint64_t seed, int32_t *out,
                             cudaStream_t st);
cudaError_t launch_select(const ds_cache *c, const SelectParams &p, const SelectGeom &g,
                          cudaStream_t st);
cudaError_t launch_attn(const ds_cache *c, const AttnParams &p, const AttnGeom &g, cudaStream_t st);
cudaError_t launch_combine(const ds_cache *c, const AttnParams &p, cudaStream_t st);

CacheView make_view(const ds_cache *c);

}  // namespace ds
