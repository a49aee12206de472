// api.cu -- the extern "C" boundary of libds.so (declared in include/ds.h).
// Host-side validation, workspace carving and launch orchestration only;
// every step of the method runs in the kernels of select.cu / attend.cu /
// append.cu / calibrate.cu.
#include <cmath>
#include <cstdint>

#include "ds.h"
#include "ds_internal.h"

namespace ds {

CacheView make_view(const ds_cache *c) {
  CacheView v;
  v.B = c->batch;
  v.Hq = c->num_q_heads;
  v.Hkv = c->num_kv_heads;
  v.D = c->head_dim;
  v.G = c->num_q_heads / c->num_kv_heads;
  v.P = c->page_size;
  v.num_pages = c->num_pages;
  v.maxp = c->max_pages_per_seq;
  v.Smax = c->max_seq_len;
  v.r = c->r;
  v.k_pool = c->k_pool;
  v.v_pool = c->v_pool;
  v.block_table = c->block_table;
  v.seq_lens = c->seq_lens;
  v.label = c->label;
  v.C = c->channel_idx;
  return v;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

Workspace carve_workspace(const ds_cache *c, int k, int nsplit, void *base) {
  const size_t units = (size_t)c->batch * c->num_kv_heads;
  const int G = c->num_q_heads / c->num_kv_heads;
  Workspace w;
  size_t off = 0;
  const size_t idx_b = align256(units * (size_t)(k > 0 ? k : 0) * sizeof(int32_t));
  const size_t po_b = align256(units * nsplit * G * (size_t)c->head_dim * sizeof(float));
  const size_t pm_b = align256(units * nsplit * G * 2 * sizeof(float));
  char *p = (char *)base;
  w.idx = (int32_t *)(p ? p + off : nullptr);
  off += idx_b;
  w.part_o = (float *)(p ? p + off : nullptr);
  off += po_b;
  w.part_ml = (float *)(p ? p + off : nullptr);
  off += pm_b;
  w.bytes = off;
  return w;
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static ds_status validate_cache(const ds_cache *c) {
  if (!c) return DS_ERR_INVALID_ARGUMENT;
  if (c->batch < 1 || c->num_q_heads < 1 || c->num_kv_heads < 1 || c->head_dim < 1 || c->page_size < 1 ||
      c->num_pages < 1 || c->max_pages_per_seq < 1 || c->max_seq_len < 1 || c->r < 1)
    return DS_ERR_INVALID_ARGUMENT;
  if (c->num_q_heads % c->num_kv_heads != 0) return DS_ERR_INVALID_ARGUMENT;
  if (c->r > c->head_dim) return DS_ERR_INVALID_ARGUMENT;
  if ((long long)c->max_pages_per_seq * c->page_size < c->max_seq_len) return DS_ERR_INVALID_ARGUMENT;
  if (c->dtype != DS_FP16 && c->dtype != DS_BF16 && c->dtype != DS_FP32) return DS_ERR_UNSUPPORTED;
  if (c->head_dim != 64 && c->head_dim != 128) return DS_ERR_UNSUPPORTED;
  const int G = c->num_q_heads / c->num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return DS_ERR_UNSUPPORTED;
  if (c->r > 256) return DS_ERR_UNSUPPORTED;
  // pool row ids are 32-bit inside the kernels
  if ((long long)c->num_pages * c->num_kv_heads * c->page_size >= (1ll << 31)) return DS_ERR_UNSUPPORTED;
  if (!c->k_pool || !c->v_pool || !c->block_table || !c->seq_lens || !c->label || !c->channel_idx)
    return DS_ERR_INVALID_ARGUMENT;
  if (!aligned16(c->k_pool) || !aligned16(c->v_pool) || !aligned16(c->label)) return DS_ERR_INVALID_ARGUMENT;
  return DS_OK;
}

static ds_status cuda_status(cudaError_t e) { return e == cudaSuccess ? DS_OK : DS_ERR_CUDA; }

}  // namespace ds

using namespace ds;

extern "C" {

const char *ds_status_string(ds_status s) {
  switch (s) {
    case DS_OK: return "DS_OK";
    case DS_ERR_INVALID_ARGUMENT: return "DS_ERR_INVALID_ARGUMENT";
    case DS_ERR_UNSUPPORTED: return "DS_ERR_UNSUPPORTED";
    case DS_ERR_GQA_INCOMPATIBLE: return "DS_ERR_GQA_INCOMPATIBLE (k-outlier calibration is N/A for GQA)";
    case DS_ERR_WORKSPACE_TOO_SMALL: return "DS_ERR_WORKSPACE_TOO_SMALL";
    case DS_ERR_CUDA: return "DS_ERR_CUDA";
  }
  return "DS_ERR_UNKNOWN";
}

const char *ds_version(void) { return "ds-b200 0.1 sm_100a"; }

ds_status ds_calibrate_channels(const void *q_calib, const void *k_calib, int32_t n, int32_t num_q_heads,
                                int32_t num_kv_heads, int32_t head_dim, ds_dtype dtype, ds_calib_mode mode,
                                int32_t r, uint64_t seed, int32_t *channel_idx_out, cudaStream_t stream) {
  if (num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || head_dim < 1 || head_dim > 1024 ||
      r < 1 || r > head_dim || !channel_idx_out)
    return DS_ERR_INVALID_ARGUMENT;
  if (mode < DS_CALIB_QK || mode > DS_CALIB_RANDOM) return DS_ERR_INVALID_ARGUMENT;
  if (dtype != DS_FP16 && dtype != DS_BF16 && dtype != DS_FP32) return DS_ERR_UNSUPPORTED;
  if (mode == DS_CALIB_K && num_q_heads != num_kv_heads) return DS_ERR_GQA_INCOMPATIBLE;
  if (mode != DS_CALIB_RANDOM && (n < 1 || !q_calib || !k_calib)) return DS_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_calibrate(q_calib, k_calib, n, num_q_heads, num_kv_heads, head_dim, dtype, (int)mode,
                                      r, seed, channel_idx_out, stream));
}

ds_status ds_append_kv(const ds_cache *c, const void *k_new, const void *v_new, const int32_t *positions,
                       int32_t n_new, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (n_new < 0 || n_new > c->max_seq_len || !positions) return DS_ERR_INVALID_ARGUMENT;
  if (n_new == 0) return DS_OK;
  if (!k_new || !v_new || !aligned16(k_new) || !aligned16(v_new)) return DS_ERR_INVALID_ARGUMENT;
  return cuda_status(launch_append(c, k_new, v_new, positions, n_new, stream));
}

size_t ds_decode_workspace_size(const ds_cache *c, int32_t k) {
  if (validate_cache(c) != DS_OK || k < 1 || k > c->max_seq_len) return 0;
  AttnGeom g = attn_geom(c, k);
  return carve_workspace(c, k, g.nsplit, nullptr).bytes;
}

ds_status ds_decode_attention(const ds_cache *c, const void *q, int32_t k, void *out, int32_t *topk_idx_out,
                              void *workspace, size_t workspace_bytes, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (k < 1 || k > c->max_seq_len || !q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  AttnGeom ag = attn_geom(c, k);
  Workspace w = carve_workspace(c, k, ag.nsplit, workspace);
  if (!workspace || workspace_bytes < w.bytes) return DS_ERR_WORKSPACE_TOO_SMALL;
  SelectGeom sg = select_geom(c);
  if (sg.smem > 200 * 1024) return DS_ERR_UNSUPPORTED;
  SelectParams sp;
  sp.c = make_view(c);
  sp.q = q;
  sp.k = k;
  sp.idx = topk_idx_out ? topk_idx_out : w.idx;
  sp.scores = nullptr;
  sp.cap = sg.cap;
  cudaError_t e = launch_select(c, sp, sg, stream);
  if (e != cudaSuccess) return DS_ERR_CUDA;
  AttnParams ap;
  ap.c = sp.c;
  ap.q = q;
  ap.idx = sp.idx;
  ap.k = k;
  ap.rows_per_cta = ag.rows_per_cta;
  ap.nsplit = ag.nsplit;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
  ap.part_o = w.part_o;
  ap.part_ml = w.part_ml;
  ap.out = out;
  e = launch_attn(c, ap, ag, stream);
  if (e != cudaSuccess) return DS_ERR_CUDA;
  return cuda_status(launch_combine(c, ap, stream));
}

ds_status ds_approx_scores(const ds_cache *c, const void *q, float *scores_out, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (!q || !scores_out || !aligned16(q)) return DS_ERR_INVALID_ARGUMENT;
  SelectGeom sg = select_geom(c);
  SelectParams sp;
  sp.c = make_view(c);
  sp.q = q;
  sp.k = 1;
  sp.idx = nullptr;
  sp.scores = scores_out;
  sp.cap = sg.cap;
  return cuda_status(launch_select(c, sp, sg, stream));
}

size_t ds_dense_workspace_size(const ds_cache *c) {
  if (validate_cache(c) != DS_OK) return 0;
  AttnGeom g = attn_geom(c, c->max_seq_len);
  return carve_workspace(c, 0, g.nsplit, nullptr).bytes;
}

ds_status ds_dense_decode_attention(const ds_cache *c, const void *q, void *out, void *workspace,
                                    size_t workspace_bytes, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (!q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  AttnGeom ag = attn_geom(c, c->max_seq_len);
  Workspace w = carve_workspace(c, 0, ag.nsplit, workspace);
  if (!workspace || workspace_bytes < w.bytes) return DS_ERR_WORKSPACE_TOO_SMALL;
  AttnParams ap;
  ap.c = make_view(c);
  ap.q = q;
  ap.idx = nullptr;
  ap.k = 0;
  ap.rows_per_cta = ag.rows_per_cta;
  ap.nsplit = ag.nsplit;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
  ap.part_o = w.part_o;
  ap.part_ml = w.part_ml;
  ap.out = out;
  cudaError_t e = launch_attn(c, ap, ag, stream);
  if (e != cudaSuccess) return DS_ERR_CUDA;
  return cuda_status(launch_combine(c, ap, stream));
}

}  // extern "C"
