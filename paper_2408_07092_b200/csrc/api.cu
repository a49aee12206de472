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
  v.lq4 = c->label_format == DS_LABEL_INT4;
  v.lnone = c->label_format == DS_LABEL_NONE;
  v.greduce = (int)c->group_reduce;
  v.rb = (c->r + 1) / 2;
  v.label_scale = c->label_scale;
  return v;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

Workspace carve_workspace(const ds_cache *c, int k, void *base) {
  const size_t units = (size_t)c->batch * c->num_kv_heads;
  const size_t kb = align256(units * (size_t)(k > 0 ? k : 0) * sizeof(int32_t));
  const size_t flag_b = align256(units * sizeof(uint32_t));
  char *p = (char *)base;
  size_t off = 0;
  Workspace w;
  auto take = [&](size_t n) {
    char *q = p ? p + off : nullptr;
    off += n;
    return q;
  };
  w.ready = (uint32_t *)take(flag_b);
  w.idx = (int32_t *)take(kb);
  w.rowid = (int32_t *)take(kb);
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
  if (c->label_format != DS_LABEL_NATIVE && c->label_format != DS_LABEL_INT4 && c->label_format != DS_LABEL_NONE)
    return DS_ERR_INVALID_ARGUMENT;
  if (c->group_reduce != DS_GROUP_SUM && c->group_reduce != DS_GROUP_MAX && c->group_reduce != DS_GROUP_PER_HEAD)
    return DS_ERR_INVALID_ARGUMENT;
  if (c->group_reduce != DS_GROUP_SUM && c->dtype == DS_FP32) return DS_ERR_UNSUPPORTED;
  if (c->group_reduce == DS_GROUP_MAX && (c->num_q_heads / c->num_kv_heads) * c->r > 256) return DS_ERR_UNSUPPORTED;
  const bool lab = c->label_format != DS_LABEL_NONE;
  if (!c->k_pool || !c->v_pool || !c->block_table || !c->seq_lens || (lab && !c->label) || !c->channel_idx)
    return DS_ERR_INVALID_ARGUMENT;
  if (!aligned16(c->k_pool) || !aligned16(c->v_pool) || (lab && !aligned16(c->label))) return DS_ERR_INVALID_ARGUMENT;
  if (c->label_format == DS_LABEL_INT4 && (!c->label_scale || !aligned16(c->label_scale)))
    return DS_ERR_INVALID_ARGUMENT;
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
  return carve_workspace(c, k, nullptr).bytes;
}

int32_t ds_decode_launches(const ds_cache *c, int32_t k) {
  if (validate_cache(c) != DS_OK || k < 1 || k > c->max_seq_len) return 0;
  return fused_applicable(c) ? 1 : 2;
}

static void fill_attn(AttnParams &ap, const ds_cache *c, const void *q, const int32_t *rowid, int k,
                      const AttnGeom &ag, void *out) {
  ap.c = make_view(c);
  ap.q = q;
  ap.rowid = rowid;
  ap.ready = nullptr;
  ap.k = k;
  ap.rows_per_cta = ag.rows_per_cta;
  ap.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
  ap.out = out;
}

ds_status ds_decode_attention(const ds_cache *c, const void *q, int32_t k, void *out, int32_t *topk_idx_out,
                              void *workspace, size_t workspace_bytes, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (k < 1 || k > c->max_seq_len || !q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  Workspace w = carve_workspace(c, k, workspace);
  if (!workspace || workspace_bytes < w.bytes || !aligned16(workspace)) return DS_ERR_WORKSPACE_TOO_SMALL;
  if (fused_applicable(c)) {  // serving shape: one kernel, one CTA per unit
    FusedParams fp;
    fp.c = make_view(c);
    fp.q = q;
    fp.k = k;
    fp.out = out;
    fp.idx = topk_idx_out;
    fp.select_only = 0;
    fp.k_new = fp.v_new = nullptr;
    fp.positions = nullptr;
    fp.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
    return cuda_status(launch_fused(c, fp, stream));
  }
  // the two-kernel path has no per-query-head units (R17 per head)
  if (c->group_reduce == DS_GROUP_PER_HEAD) return DS_ERR_UNSUPPORTED;
  SelectGeom sg = select_geom(c);
  AttnGeom ag = attn_geom(c, k);
  if (ag.nsplit < 1) return DS_ERR_UNSUPPORTED;
  ScoreParams sc;
  sc.c = make_view(c);
  sc.q = q;
  sc.k = k;
  sc.ready = w.ready;
  sc.idx = topk_idx_out ? topk_idx_out : w.idx;
  sc.rowid = w.rowid;
  sc.scores = nullptr;
  sc.chunk = sg.chunk;
  if (launch_score(c, sc, sg, stream) != cudaSuccess) return DS_ERR_CUDA;
  AttnParams ap;
  fill_attn(ap, c, q, w.rowid, k, ag, out);
  ap.ready = w.ready;
  return cuda_status(launch_attn(c, ap, ag, stream));
}

ds_status ds_decode_attention_append(const ds_cache *c, const void *k_new, const void *v_new,
                                     const int32_t *positions, const void *q, int32_t k, void *out,
                                     int32_t *topk_idx_out, void *workspace, size_t workspace_bytes,
                                     cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (!positions || !k_new || !v_new || !aligned16(k_new) || !aligned16(v_new)) return DS_ERR_INVALID_ARGUMENT;
  if (k < 1 || k > c->max_seq_len || !q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  Workspace w = carve_workspace(c, k, workspace);
  if (!workspace || workspace_bytes < w.bytes || !aligned16(workspace)) return DS_ERR_WORKSPACE_TOO_SMALL;
  if (!fused_applicable(c)) {  // fp32: the append kernel, then the two-kernel decode
    if (c->group_reduce == DS_GROUP_PER_HEAD) return DS_ERR_UNSUPPORTED;
    if (launch_append(c, k_new, v_new, positions, 1, stream) != cudaSuccess) return DS_ERR_CUDA;
    return ds_decode_attention(c, q, k, out, topk_idx_out, workspace, workspace_bytes, stream);
  }
  FusedParams fp;
  fp.c = make_view(c);
  fp.q = q;
  fp.k = k;
  fp.out = out;
  fp.idx = topk_idx_out;
  fp.select_only = 0;
  fp.k_new = k_new;
  fp.v_new = v_new;
  fp.positions = positions;
  fp.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)c->head_dim));
  return cuda_status(launch_fused(c, fp, stream));
}

ds_status ds_approx_scores(const ds_cache *c, const void *q, float *scores_out, cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (c->group_reduce == DS_GROUP_PER_HEAD) return DS_ERR_UNSUPPORTED;
  if (!q || !scores_out || !aligned16(q)) return DS_ERR_INVALID_ARGUMENT;
  SelectGeom sg = select_geom(c);
  ScoreParams sc;
  sc.c = make_view(c);
  sc.q = q;
  sc.k = 1;
  sc.ready = nullptr;
  sc.idx = nullptr;
  sc.rowid = nullptr;
  sc.scores = scores_out;
  sc.chunk = sg.chunk;
  return cuda_status(launch_score(c, sc, sg, stream));
}

static ds_status check_slot(const ds_cache *c, const ds_prefetch_slot *slot) {
  if (!slot || slot->k < 1 || slot->k > c->max_seq_len) return DS_ERR_INVALID_ARGUMENT;
  if (!slot->idx || !slot->count || !slot->table || !slot->k_rows || !slot->v_rows) return DS_ERR_INVALID_ARGUMENT;
  if (!aligned16(slot->k_rows) || !aligned16(slot->v_rows)) return DS_ERR_INVALID_ARGUMENT;
  if ((long long)c->batch * c->num_kv_heads * slot->k >= (1ll << 31)) return DS_ERR_UNSUPPORTED;
  return DS_OK;
}

ds_status ds_prefetch_next_layer(const ds_cache *next, const void *q_pred, int32_t k, const ds_prefetch_slot *slot,
                                 cudaStream_t side_stream) {
  ds_status s = validate_cache(next);
  if (s != DS_OK) return s;
  if (!q_pred || !aligned16(q_pred)) return DS_ERR_INVALID_ARGUMENT;
  if ((s = check_slot(next, slot)) != DS_OK) return s;
  if (k != slot->k) return DS_ERR_INVALID_ARGUMENT;
  if (!fused_applicable(next) || next->group_reduce == DS_GROUP_PER_HEAD) return DS_ERR_UNSUPPORTED;
  FusedParams fp;
  fp.c = make_view(next);
  fp.q = q_pred;
  fp.k = k;
  fp.out = nullptr;
  fp.idx = slot->idx;
  fp.scale_log2 = 0.f;
  fp.select_only = 1;
  fp.k_new = fp.v_new = nullptr;
  fp.positions = nullptr;
  if (launch_fused(next, fp, side_stream) != cudaSuccess) return DS_ERR_CUDA;
  return cuda_status(launch_gather(next, slot, side_stream));
}

ds_status ds_decode_attention_prefetched(const ds_cache *c, const void *q, const ds_prefetch_slot *slot, void *out,
                                         cudaStream_t stream) {
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (!q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  if ((s = check_slot(c, slot)) != DS_OK) return s;
  // the slot as a paged cache: one page of k rows per sequence, page b = b
  ds_cache v = *c;
  v.page_size = slot->k;
  v.num_pages = c->batch;
  v.max_pages_per_seq = 1;
  v.max_seq_len = slot->k;
  v.k_pool = slot->k_rows;
  v.v_pool = slot->v_rows;
  v.block_table = slot->table;
  v.seq_lens = slot->count;
  AttnGeom ag = attn_geom(&v, v.max_seq_len);
  if (ag.nsplit < 1) return DS_ERR_UNSUPPORTED;
  AttnParams ap;
  fill_attn(ap, &v, q, nullptr, 0, ag, out);
  return cuda_status(launch_attn(&v, ap, ag, stream));
}

size_t ds_dense_workspace_size(const ds_cache *c) {
  (void)c;
  return 0;  // the dense path merges its splits on chip
}

ds_status ds_dense_decode_attention(const ds_cache *c, const void *q, void *out, void *workspace,
                                    size_t workspace_bytes, cudaStream_t stream) {
  (void)workspace;
  (void)workspace_bytes;
  ds_status s = validate_cache(c);
  if (s != DS_OK) return s;
  if (!q || !out || !aligned16(q) || !aligned16(out)) return DS_ERR_INVALID_ARGUMENT;
  AttnGeom ag = attn_geom(c, c->max_seq_len);
  if (ag.nsplit < 1) return DS_ERR_UNSUPPORTED;
  AttnParams ap;
  fill_attn(ap, c, q, nullptr, 0, ag, out);
  return cuda_status(launch_attn(c, ap, ag, stream));
}

}  // extern "C"
