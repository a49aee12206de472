/*
 * ds.h -- C ABI of libds.so: the Double Sparsity decode-attention hot path
 * (arXiv 2408.07092) as hand-written CUDA for NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" is line n of the paper text (/root/reference/PAPER.md,
 * v1 LaTeX), with the section / algorithm line it falls in.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Ownership: every buffer is allocated by the caller (e.g. a torch
 *    tensor's data_ptr()).  The library never allocates, frees or retains
 *    a pointer past the call, and keeps no mutable global state (only a
 *    once-initialised kernel-attribute setup).  Calls are thread-safe.
 *  - Asynchrony: every call only validates on the host and enqueues
 *    kernels on the caller's stream; results are visible in stream order.
 *    All calls are legal inside CUDA-graph capture.
 *  - Pointers are device pointers unless stated otherwise (host-mapped
 *    pinned memory is a valid device pointer).  All tensors are dense,
 *    row-major, 16-byte aligned.
 *  - Errors: a ds_status return code, never an exception or exit().
 *    Host-checkable preconditions (shapes, dtypes, alignment, ranges of
 *    scalars, workspace size) return DS_ERR_INVALID_ARGUMENT /
 *    DS_ERR_UNSUPPORTED / DS_ERR_WORKSPACE_TOO_SMALL before anything is
 *    enqueued.  A failed launch returns DS_ERR_CUDA.  Data-dependent
 *    preconditions that live in device memory (channel ids < head_dim and
 *    ascending, block-table entries < num_pages, seq_lens <= max_seq_len,
 *    append positions in range, finite inputs) are the caller's contract
 *    and are not checked: violating them is undefined behaviour.
 *  - dtype: q, K, V, the label cache and out share one element type.  The
 *    default (DS_LABEL_NATIVE) label cache has the same 16-bit (or 32-bit)
 *    type as K, so "label == channel gather of K" holds bit for bit (DESIGN
 *    reading R8).  DS_LABEL_INT4 stores it in 4 bits (reading R16).
 *  - Supported shapes: head_dim in {64, 128}; G = num_q_heads /
 *    num_kv_heads in {1, 2, 4, 8}; 1 <= r <= head_dim; page_size >= 1.
 *    Others return DS_ERR_UNSUPPORTED.
 */
#ifndef DS_H_
#define DS_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DS_OK = 0,
  DS_ERR_INVALID_ARGUMENT = 1,
  DS_ERR_UNSUPPORTED = 2,
  DS_ERR_GQA_INCOMPATIBLE = 3, /* k-outlier calibration with GQA, P:298 (Table 3) */
  DS_ERR_WORKSPACE_TOO_SMALL = 4,
  DS_ERR_CUDA = 5
} ds_status;

typedef enum { DS_FP16 = 0, DS_BF16 = 1, DS_FP32 = 2 } ds_dtype;

/* Label-cache storage ("Since approximate attention is not
 * sensitive to precision, we can store the label cache in 4-bit"):
 *   DS_LABEL_NATIVE: label [batch][num_kv_heads][max_seq_len][r] of dtype,
 *                    a bit copy of K's r channels (reading R8).
 *   DS_LABEL_INT4  : reading R16, symmetric per-token quantisation.  For
 *                    the r channel values x_j of a token:
 *                      s   = RNE_dtype(max_j |x_j| / 7)  (fp32 divide; 1 if
 *                            max is 0 or the rounding gives 0)
 *                      c_j = clamp(round_half_away(x_j / s), -7, 7)
 *                    label       : uint8 [batch][num_kv_heads][max_seq_len][ceil(r/2)],
 *                                  byte i = c_{2i} (low nibble) | c_{2i+1} << 4,
 *                                  4-bit two's complement, an odd r pads 0;
 *                    label_scale : dtype [batch][num_kv_heads][max_seq_len] = s.
 *                    Line 2 becomes s_hat[t] = (fp32 fma chain over j of
 *                    q_label[j] * c_j) * s_t.  Per token ceil(r/2) + e bytes
 *                    instead of r * e (6 instead of 16 at r = 8, 16-bit).
 *   DS_LABEL_NONE  : no label cache (the ablation of Appendix B.1, Table 4,
 *                    P:517-544): line 2 reads the r channels of each token
 *                    straight from its paged K row (2-byte reads scattered
 *                    over the row); label and label_scale are ignored and
 *                    may be NULL.  Scores are the same values as with the
 *                    native label (a bit copy of those channels). */
typedef enum { DS_LABEL_NATIVE = 0, DS_LABEL_INT4 = 1, DS_LABEL_NONE = 2 } ds_label_format;

/* GQA selection granularity (the paper runs GQA models, Table 3 P:308-310,
 * without saying how a KV head's G query heads share the selection):
 *   DS_GROUP_SUM     : reading R3 (default) -- one top-k set per (b, KV
 *                      head), scored with the group-summed query label
 *                      Q_label[j] = sum_g q_g[C[j]] (g ascending, fp32).
 *   DS_GROUP_MAX     : reading R17 -- one set per (b, KV head), scored with
 *                      max_g of the per-head scores s_g[t] (each the fp32 fma
 *                      chain of q_g[C[j]] * L[t][j]).  Needs G * r <= 256.
 *   DS_GROUP_PER_HEAD: reading R17 -- one set per (b, query head): every
 *                      query head runs Algorithm 1 on its KV head's label and
 *                      K/V (the layer treated as MHA over shared K/V);
 *                      topk_idx_out is then [batch][num_q_heads][k].
 * MAX and PER_HEAD run on 16-bit caches only (fp32 -> DS_ERR_UNSUPPORTED);
 * PER_HEAD has no prefetch (DS_ERR_UNSUPPORTED) nor ds_approx_scores. */
typedef enum { DS_GROUP_SUM = 0, DS_GROUP_MAX = 1, DS_GROUP_PER_HEAD = 2 } ds_group_reduce;

/* Outlier-channel modes of Table 3: qk (default), q, k, random. */
typedef enum { DS_CALIB_QK = 0, DS_CALIB_Q = 1, DS_CALIB_K = 2, DS_CALIB_RANDOM = 3 } ds_calib_mode;

/* One layer's cache (the full KV cache is kept; plus the label
 * cache).  All pointers are device pointers.
 *   k_pool, v_pool : [num_pages][num_kv_heads][page_size][head_dim]
 *                    token t of sequence b, head h lives in page
 *                    block_table[b][t / page_size], slot t % page_size.
 *   block_table    : int32 [batch][max_pages_per_seq]
 *   seq_lens       : int32 [batch]; attention reads tokens t < seq_lens[b]
 *                    (the caller appends the current token first, reading R10)
 *   label          : [batch][num_kv_heads][max_seq_len][r]   K_label
 *                    (DS_LABEL_INT4: packed codes, see ds_label_format)
 *   channel_idx    : int32 [num_kv_heads][r] = C, ascending, distinct.
 *   label_format   : ds_label_format (0 = native: a zero-initialised
 *                    struct keeps the 16-bit label)
 *   label_scale    : DS_LABEL_INT4 only: dtype [batch][num_kv_heads][max_seq_len],
 *                    16-B aligned; ignored (may be NULL) for native labels.
 *   group_reduce   : ds_group_reduce (0 = DS_GROUP_SUM, reading R3). */
typedef struct {
  int32_t batch, num_q_heads, num_kv_heads, head_dim;
  int32_t page_size, num_pages, max_pages_per_seq, max_seq_len, r;
  ds_dtype dtype;
  void *k_pool, *v_pool;
  const int32_t *block_table;
  const int32_t *seq_lens;
  void *label;
  const int32_t *channel_idx;
  ds_label_format label_format;
  void *label_scale;
  ds_group_reduce group_reduce;
} ds_cache;

/* Human-readable name of a status code (static string, never NULL). */
const char *ds_status_string(ds_status s);

/* Library version string, e.g. "ds-b200 0.1 sm_100a". */
const char *ds_version(void);

/* Offline calibration, Sec. 4.1: A = sum_i S_i, S_i = Q_i*K_i;
 * pick the r channels with the largest aggregated |S_i| per KV head
 * (readings R4, R5: per KV head, group's q heads summed; fp64 sums of
 * |Q| and |K| over the n calibration samples, importance = product for
 * qk mode, the |Q| sum for q mode, the |K| sum for k mode; random mode is
 * a seeded splitmix64 Fisher-Yates draw).  Ties go to the lower channel;
 * output is ascending.
 *   q_calib [n][num_q_heads][head_dim], k_calib [n][num_kv_heads][head_dim]
 *   channel_idx_out int32 [num_kv_heads][r] (device).
 * Errors: DS_ERR_GQA_INCOMPATIBLE for k mode with num_q_heads != num_kv_heads. */
ds_status ds_calibrate_channels(const void *q_calib, const void *k_calib, int32_t n,
                                int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                                ds_dtype dtype, ds_calib_mode mode, int32_t r, uint64_t seed,
                                int32_t *channel_idx_out, cudaStream_t stream);

/* Label-cache append, Sec. 4.2: "During the prefilling stage, all
 * heavy channel values from the Key cache are stored in the label cache;
 * in the decoding phase, only the heavy channel values of new tokens are
 * added."  For every b < batch, i < n_new, h: token p = positions[b] + i
 * gets K/V rows k_new[b][i][h][:], v_new[b][i][h][:] written into its
 * page slot and label[b][h][p][j] = k_new[b][i][h][C[h][j]] (a bit copy;
 * DS_LABEL_INT4: the row's codes and scale quantised from those values,
 * reading R16).
 *   k_new, v_new : [batch][n_new][num_kv_heads][head_dim]
 *   positions    : int32 [batch] (device), first write position per
 *                  sequence; p < max_seq_len and its page must be mapped.
 * Does not modify seq_lens (the caller owns it). */
ds_status ds_append_kv(const ds_cache *c, const void *k_new, const void *v_new,
                       const int32_t *positions, int32_t n_new, cudaStream_t stream);

/* Bytes of workspace ds_decode_attention needs for this cache and k
 * (0 on invalid arguments). */
size_t ds_decode_workspace_size(const ds_cache *c, int32_t k);

/* Algorithm 1 "Double Sparsity Decode", one decode query per
 * sequence, every (b, KV head) unit independently:
 *   1  Q_label <- Q_[C]                (group-summed for GQA, reading R3)
 *   2  s_hat   <- Q_label . K_label^T  (fp32 fma chain over j ascending,
 *                                       no 1/sqrt(d), reading R2)
 *   3  i       <- argtopk(s_hat, k_eff), k_eff = min(k, seq_lens[b]);
 *                 ties to the lower index, ascending (reading R6)
 *   4  s       <- softmax(Q . K_[i,:]^T / sqrt(d_h))   (fp32)
 *   5  y       <- s . V_[i,:]          -> out, rounded to dtype (RNE)
 *   q   : [batch][num_q_heads][head_dim]
 *   out : [batch][num_q_heads][head_dim]
 *   topk_idx_out : nullable int32 [batch][num_kv_heads][k] ([batch][num_q_heads][k]
 *                  for DS_GROUP_PER_HEAD); positions
 *                  >= k_eff are set to -1.
 *   workspace    : >= ds_decode_workspace_size(c, k) bytes of device memory,
 *                  16-byte aligned, ZERO-FILLED before its first use; every
 *                  call leaves its synchronisation words zeroed again, so it
 *                  can be reused by later calls on the same stream (not by
 *                  concurrent calls).  It holds the selected index lists,
 *                  their pool row ids and per-unit ready flags through which
 *                  the attention of a (b, KV head) unit starts as soon as that
 *                  unit's selection is published.
 * Errors: DS_ERR_INVALID_ARGUMENT if k < 1 or k > max_seq_len. A sequence
 * with seq_lens[b] == 0 yields out = 0. */
ds_status ds_decode_attention(const ds_cache *c, const void *q, int32_t k, void *out,
                              int32_t *topk_idx_out, void *workspace, size_t workspace_bytes,
                              cudaStream_t stream);

/* Number of kernels one ds_decode_attention call with this cache and k
 * enqueues (0 on invalid arguments): 1 when the whole of Algorithm 1 runs
 * as one kernel (16-bit KV: one CTA per (b, KV head) unit, or a thread-block
 * cluster of up to 16 CTAs per unit when units are few or max_seq_len >
 * 32768 -- up to 512K tokens; when units are few, the largest cluster size
 * whose clusters of all units the occupancy API says are co-resident in one
 * wave; above 8 CTAs only where one can be resident), else 2 (fp32, or a
 * cluster that cannot be resident: score+select with the CTAs of a unit in
 * one thread-block cluster, then the attention).  Results are identical up to the fp32
 * summation order of the attention.  DS_GROUP_PER_HEAD exists only on the
 * one-kernel path (DS_ERR_UNSUPPORTED from the decode calls otherwise). */
int32_t ds_decode_launches(const ds_cache *c, int32_t k);

/* ---------------------------------------------------------------------
 * Double Sparsity-Offload, Sec. 5.1: "The complete KV cache is
 * stored on the CPU, while the GPU maintains only the label cache and a
 * double buffer.  [...] each layer processes its embeddings through the next
 * layer's query projection to generate an approximate query for the
 * subsequent layer [...] the tokens corresponding to the approximate
 * attention results for the next layer are offloaded to the GPU" (reading
 * R15: the predicted query is an input).
 *
 * A slot is one half of the double buffer (caller-allocated device memory):
 *   idx    int32 [batch][num_kv_heads][k]  selected tokens, ascending, -1 past k_eff
 *   count  int32 [batch]                   k_eff = min(k, seq_lens[b])
 *   table  int32 [batch]                   written as 0..batch-1 (the slot's page table)
 *   k_rows, v_rows [batch][num_kv_heads][k][head_dim]  the gathered K / V rows
 */
typedef struct {
  int32_t k;
  int32_t *idx, *count, *table;
  void *k_rows, *v_rows;
} ds_prefetch_slot;

/* Lines 1-3 of Algorithm 1 with the predicted query q_pred [batch][Hq][d]
 * against next's device-resident label cache, then the k_eff selected K/V
 * rows of every unit are copied from next's pools -- pinned host memory
 * (cudaHostAlloc / torch pin_memory; read over the host link through unified
 * addressing) or device memory -- into the slot, ascending by token.  Enqueued
 * on side_stream (typically overlapping the current layer's attention); the
 * caller orders the consumer after it (an event).  16-bit dtypes only
 * (DS_ERR_UNSUPPORTED otherwise). */
ds_status ds_prefetch_next_layer(const ds_cache *next, const void *q_pred, int32_t k,
                                 const ds_prefetch_slot *slot, cudaStream_t side_stream);

/* Lines 4-5 of Algorithm 1 with the layer's true query q over the rows a
 * prefetch put in slot: y = softmax(q K_slot^T / sqrt(d)) V_slot, exact, over
 * the count[b] rows of each unit.  c supplies the shape (its pools are not
 * read).  out [batch][Hq][d]. */
ds_status ds_decode_attention_prefetched(const ds_cache *c, const void *q, const ds_prefetch_slot *slot,
                                         void *out, cudaStream_t stream);

/* One decode step of a layer in one launch: ds_append_kv of one new token
 * per sequence (n_new = 1; "in the decoding phase, only the heavy
 * channel values of new tokens are added") followed by ds_decode_attention
 * (Algorithm 1), with the same results and the same cache contents as the
 * two calls in sequence.  The caller sets seq_lens[b] to include the new
 * token (positions[b] < seq_lens[b], reading R10) before the call.
 *   k_new, v_new : [batch][1][num_kv_heads][head_dim] (device, 16-B aligned)
 *   positions    : int32 [batch] (device), the new token's position
 *   q, k, out, topk_idx_out, workspace : as ds_decode_attention.
 * On the single-kernel path the CTA whose chunk holds the new token writes
 * its K/V and label rows and scores it from the values it wrote; fp32
 * caches run the append kernel and then the two-kernel decode.
 * Errors: as ds_append_kv and ds_decode_attention. */
ds_status ds_decode_attention_append(const ds_cache *c, const void *k_new, const void *v_new,
                                     const int32_t *positions, const void *q, int32_t k, void *out,
                                     int32_t *topk_idx_out, void *workspace, size_t workspace_bytes,
                                     cudaStream_t stream);

/* Lines 1-2 of Algorithm 1 only, for diagnostics and tests:
 * scores_out fp32 [batch][num_kv_heads][max_seq_len]; entries t >=
 * seq_lens[b] are left untouched.  Same arithmetic as ds_decode_attention. */
ds_status ds_approx_scores(const ds_cache *c, const void *q, float *scores_out,
                           cudaStream_t stream);

/* Dense decode attention baseline on the same paged layout, Sec. 2.1
 * (P:43): y = softmax(q K^T / sqrt(d_h)) V over every token t < seq_lens[b]. */
size_t ds_dense_workspace_size(const ds_cache *c);
ds_status ds_dense_decode_attention(const ds_cache *c, const void *q, void *out, void *workspace,
                                    size_t workspace_bytes, cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DS_H_ */
