/*
 * oracle/ds_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * Double Sparsity decode hot path (arXiv 2408.07092).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * code.  The product (paper_2408_07092_b200/, libds.so) never links,
 * imports or executes it, and it shares no source, header, table or helper
 * with the CUDA path.
 *
 * Every function below follows a passage of /root/reference/PAPER.md
 * ("P:n" = line n) in the paper's order and notation; where the paper is
 * silent the DESIGN.md reading it takes is named (R1..R16, which extend
 * SURVEY.md 8(c)).  Floating point is fp32 as BASELINE.json's north_star
 * fixes ("a plain, slow CPU oracle in fp32"); calibration statistics are
 * accumulated in fp64.  No blocking, fusion or reordering beyond what the
 * definitions state.  Compile with -O2 -ffp-contract=off (no fast-math):
 * every multiply and add below is an IEEE fp32 operation in source order.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): worked examples from
 * SPEC.md, closed forms, brute-force rank definitions, library routines
 * (torch SDPA in fp64, numpy fancy indexing) and invariants.  Nothing in
 * this file is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* a0  Label cache (Sec. 4.2): "all heavy channel values from
 *     the Key cache are stored in the label cache".
 *     L[t][j] = K[t][C[j]]  for t < S, j < r.                          */
void oracle_label_gather(const float *K, int S, int d, const int32_t *C,
                         int r, float *L) {
  for (int t = 0; t < S; ++t)
    for (int j = 0; j < r; ++j) L[(size_t)t * r + j] = K[(size_t)t * d + C[j]];
}

/* ------------------------------------------------------------------ */
/* a1  Alg. 1 line 1: Q_label <- Q_[C].
 *     GQA reading R3: one selection per KV head, the group's query heads
 *     are summed channel-wise, left to right in g order, in fp32.       */
void oracle_query_label(const float *q /*[G][d]*/, int G, int d,
                        const int32_t *C, int r, float *qlab /*[r]*/) {
  for (int j = 0; j < r; ++j) {
    float s = 0.0f;
    for (int g = 0; g < G; ++g) s = s + q[(size_t)g * d + C[j]];
    qlab[j] = s;
  }
}

/* a2  Alg. 1 line 2: s_hat <- Q_label . K_label   (reading R1:
 *     one score per token, q_C . K_label^T; reading R2: no 1/sqrt(d), no
 *     softmax).  The dot product is the fp32 fma chain over j in
 *     ascending order (reading R2/R13: a defined order so the selection
 *     is reproducible).                                                 */
void oracle_approx_scores(const float *qlab, const float *L, int S, int r,
                          float *shat) {
  for (int t = 0; t < S; ++t) {
    float s = 0.0f;
    for (int j = 0; j < r; ++j) s = fmaf(qlab[j], L[(size_t)t * r + j], s);
    shat[t] = s;
  }
}

/* f2  4-bit label cache ("Since approximate attention is not
 *     sensitive to precision, we can store the label cache in 4-bit").
 *     The paper names no scheme; reading R16 (symmetric
 *     per-row quantisation, codes in [-7, 7]) with the scale stored in the
 *     cache's own element type:
 *       a    = max_j |L[t][j]|
 *       s32  = a / 7 in fp32 (1 when a == 0)
 *       s    = s32 rounded to nearest-even in the scale type (fp16 / bf16 /
 *              fp32: scale_dtype 0 / 1 / 2, the ds_dtype numbering), then
 *              widened; s = 1 if that rounding gives 0
 *       c_j  = clamp(round_half_away_from_zero(L[t][j] / s), -7, 7), the
 *              quotient in fp32
 *     The dequantised label value is c_j * s.                            */
static float oracle_round_to_dtype(float x, int scale_dtype) {
  if (scale_dtype == 0) return (float)(_Float16)x; /* IEEE binary16, RNE */
  if (scale_dtype == 1) return (float)(__bf16)x;   /* bfloat16, RNE */
  return x;
}

void oracle_quantize_label_4bit(const float *L /*[S][r]*/, int S, int r,
                                int scale_dtype, int8_t *codes /*[S][r]*/,
                                float *scale /*[S]*/) {
  for (int t = 0; t < S; ++t) {
    const float *row = L + (size_t)t * r;
    float a = 0.0f;
    for (int j = 0; j < r; ++j)
      if (fabsf(row[j]) > a) a = fabsf(row[j]);
    float s32 = a == 0.0f ? 1.0f : a / 7.0f;
    float s = oracle_round_to_dtype(s32, scale_dtype);
    if (s == 0.0f) s = 1.0f;
    for (int j = 0; j < r; ++j) {
      float v = row[j] / s;
      double c = v < 0.0f ? -floor(-(double)v + 0.5) : floor((double)v + 0.5);
      if (c > 7.0) c = 7.0;
      if (c < -7.0) c = -7.0;
      codes[(size_t)t * r + j] = (int8_t)c;
    }
    scale[t] = s;
  }
}

/* The stored code layout (reading R16, SPEC int4 packing): row t holds
 * ceil(r/2) bytes; byte i carries code 2i in its low nibble and code
 * 2i+1 in its high nibble, each as a 4-bit two's complement number; an
 * odd r leaves the last high nibble 0.                                  */
void oracle_pack_int4(const int8_t *codes, int S, int r, uint8_t *out) {
  int rb = (r + 1) / 2;
  for (int t = 0; t < S; ++t)
    for (int i = 0; i < rb; ++i) {
      int lo = codes[(size_t)t * r + 2 * i];
      int hi = 2 * i + 1 < r ? codes[(size_t)t * r + 2 * i + 1] : 0;
      out[(size_t)t * rb + i] = (uint8_t)((lo & 15) | ((hi & 15) << 4));
    }
}

/* a2 over a 4-bit label (reading R16): the fp32 fma chain over j of
 * q_label[j] * c_j (exact small integers), then one multiply by the
 * row's scale:  s_hat[t] = (fma-chain_j qlab[j] * c_j) * s_t.  Up to
 * rounding this is q_label . (c * s), the dequantised label.            */
void oracle_approx_scores_q4(const float *qlab, const int8_t *codes,
                             const float *scale, int S, int r, float *shat) {
  for (int t = 0; t < S; ++t) {
    float acc = 0.0f;
    for (int j = 0; j < r; ++j) acc = fmaf(qlab[j], (float)codes[(size_t)t * r + j], acc);
    shat[t] = acc * scale[t];
  }
}

/* a3  Alg. 1 line 3: i <- argtopk(s_hat, k).
 *     Reading R6: ties go to the lower index, output ascending; -0 == +0
 *     under float comparison.  Implemented as a full sort of
 *     (score desc, index asc) pairs, then the first k indices are sorted
 *     ascending.  k > S is clamped (reading R7, k_eff = min(k, S)).      */
typedef struct {
  float s;
  int32_t t;
} oracle_pair;

static int oracle_pair_cmp(const void *a, const void *b) {
  const oracle_pair *x = (const oracle_pair *)a, *y = (const oracle_pair *)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  return (x->t < y->t) ? -1 : (x->t > y->t);
}

static int oracle_int_cmp(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int oracle_argtopk(const float *scores, int S, int k, int32_t *idx,
                   float *tau_out) {
  int keff = k < S ? k : S;
  if (keff <= 0) return 0;
  oracle_pair *p = (oracle_pair *)malloc(sizeof(oracle_pair) * (size_t)S);
  for (int t = 0; t < S; ++t) {
    p[t].s = scores[t];
    p[t].t = t;
  }
  qsort(p, (size_t)S, sizeof(oracle_pair), oracle_pair_cmp);
  for (int i = 0; i < keff; ++i) idx[i] = p[i].t;
  if (tau_out) *tau_out = p[keff - 1].s;
  free(p);
  qsort(idx, (size_t)keff, sizeof(int32_t), oracle_int_cmp);
  return keff;
}

/* a4-a5  Alg. 1 lines 4-5:
 *     s <- softmax(Q . K_[i,:]^T / sqrt(d_h));  y <- s . V_[i,:]
 *     fp32, max subtraction (reading R11), two passes, no online
 *     rescaling; the weights are normalised first, then V is summed in
 *     index order.                                                      */
void oracle_attend(const float *q /*[d]*/, const float *K /*[S][d]*/,
                   const float *V /*[S][d]*/, int d, const int32_t *idx,
                   int n, float *y /*[d]*/) {
  for (int c = 0; c < d; ++c) y[c] = 0.0f;
  if (n <= 0) return;
  float *z = (float *)malloc(sizeof(float) * (size_t)n);
  float sq = sqrtf((float)d);
  float m = -INFINITY;
  for (int i = 0; i < n; ++i) {
    const float *kr = K + (size_t)idx[i] * d;
    float dot = 0.0f;
    for (int c = 0; c < d; ++c) dot = dot + q[c] * kr[c];
    z[i] = dot / sq;
    if (z[i] > m) m = z[i];
  }
  float l = 0.0f;
  for (int i = 0; i < n; ++i) {
    z[i] = expf(z[i] - m);
    l = l + z[i];
  }
  for (int i = 0; i < n; ++i) {
    float s = z[i] / l;
    const float *vr = V + (size_t)idx[i] * d;
    for (int c = 0; c < d; ++c) y[c] = y[c] + s * vr[c];
  }
  free(z);
}

/* Dense attention, Sec. 2.1: y = softmax(q K^T / sqrt(d_h)) V,
 * i.e. oracle_attend over every token 0..S-1.                            */
void oracle_dense_attention(const float *q, const float *K, const float *V,
                            int S, int d, float *y) {
  int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  for (int t = 0; t < S; ++t) idx[t] = t;
  oracle_attend(q, K, V, d, idx, S, y);
  free(idx);
}

/* Algorithm 1 end to end for one (batch, KV head) unit.
 *   q_attn [G][d]: the true query heads of the group (line 4).
 *   q_sel  [G][d]: the query used for selection (lines 1-3); equal to
 *                  q_attn for Double Sparsity, the predicted next-layer
 *                  query for Double Sparsity-Offload.
 *   K, V   [S][d], L [S][r], C [r].
 *   codes [S][r], scale [S]: a 4-bit label (reading R16) used for line 2
 *                  instead of L when scale is not NULL.
 * Outputs y [G][d]; optional idx [k_eff], shat [S], tau.               */
int oracle_ds_decode_unit(const float *q_attn, const float *q_sel, int G,
                          const float *K, const float *V, const float *L,
                          const int8_t *codes, const float *scale,
                          const int32_t *C, int S, int d, int r, int k,
                          float *y, int32_t *idx_out, float *shat_out,
                          float *tau_out) {
  float *qlab = (float *)malloc(sizeof(float) * (size_t)r);
  float *shat = (float *)malloc(sizeof(float) * (size_t)(S > 0 ? S : 1));
  int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  oracle_query_label(q_sel, G, d, C, r, qlab);              /* line 1 */
  if (scale)                                                /* line 2 */
    oracle_approx_scores_q4(qlab, codes, scale, S, r, shat);   /* 4-bit label (R16) */
  else
    oracle_approx_scores(qlab, L, S, r, shat);
  float tau = 0.0f;
  int keff = oracle_argtopk(shat, S, k, idx, &tau);         /* line 3 */
  for (int g = 0; g < G; ++g)                               /* lines 4-5 */
    oracle_attend(q_attn + (size_t)g * d, K, V, d, idx, keff, y + (size_t)g * d);
  if (idx_out) memcpy(idx_out, idx, sizeof(int32_t) * (size_t)keff);
  if (shat_out) memcpy(shat_out, shat, sizeof(float) * (size_t)S);
  if (tau_out) *tau_out = tau;
  free(qlab);
  free(shat);
  free(idx);
  return keff;
}

/* GQA selection granularity, reading R17 (the paper runs
 * GQA models, Table 3, without saying how the G query heads of a
 * KV head share the selection).  mode 0 = group sum (reading R3, exactly
 * oracle_ds_decode_unit), 1 = max over the heads of the per-head scores,
 * 2 = per head (each query head runs Algorithm 1 alone on the shared
 * label/K/V).  Outputs: y [G][d]; idx_out [k_eff] (modes 0, 1) or
 * [G][k] with -1 past each head's k_eff (mode 2); shat_out [S] (modes 0, 1)
 * or [G][S] (mode 2).  Returns k_eff.                                    */
int oracle_ds_decode_unit_group(const float *q_attn, const float *q_sel, int G,
                                const float *K, const float *V, const float *L,
                                const int8_t *codes, const float *scale,
                                const int32_t *C, int S, int d, int r, int k,
                                int mode, float *y, int32_t *idx_out,
                                float *shat_out) {
  if (mode == 0)
    return oracle_ds_decode_unit(q_attn, q_sel, G, K, V, L, codes, scale, C, S, d, r, k, y,
                                 idx_out, shat_out, NULL);
  int keff = k < S ? k : S;
  if (mode == 2) {
    for (int g = 0; g < G; ++g) {
      int32_t *ig = idx_out ? idx_out + (size_t)g * k : NULL;
      oracle_ds_decode_unit(q_attn + (size_t)g * d, q_sel + (size_t)g * d, 1, K, V, L, codes,
                            scale, C, S, d, r, k, y + (size_t)g * d, ig,
                            shat_out ? shat_out + (size_t)g * S : NULL, NULL);
      if (ig)
        for (int i = keff; i < k; ++i) ig[i] = -1;
    }
    return keff;
  }
  /* mode 1: s_hat[t] = max_g s_g[t], g ascending from -inf */
  float *qlab = (float *)malloc(sizeof(float) * (size_t)r);
  float *sg = (float *)malloc(sizeof(float) * (size_t)(S > 0 ? S : 1));
  float *shat = (float *)malloc(sizeof(float) * (size_t)(S > 0 ? S : 1));
  int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
  for (int t = 0; t < S; ++t) shat[t] = -INFINITY;
  for (int g = 0; g < G; ++g) {
    oracle_query_label(q_sel + (size_t)g * d, 1, d, C, r, qlab);  /* line 1, head g */
    if (scale)                                                     /* line 2, head g */
      oracle_approx_scores_q4(qlab, codes, scale, S, r, sg);
    else
      oracle_approx_scores(qlab, L, S, r, sg);
    for (int t = 0; t < S; ++t) shat[t] = fmaxf(shat[t], sg[t]);
  }
  keff = oracle_argtopk(shat, S, k, idx, NULL);                   /* line 3 */
  for (int g = 0; g < G; ++g)                                     /* lines 4-5 */
    oracle_attend(q_attn + (size_t)g * d, K, V, d, idx, keff, y + (size_t)g * d);
  if (idx_out) memcpy(idx_out, idx, sizeof(int32_t) * (size_t)keff);
  if (shat_out) memcpy(shat_out, shat, sizeof(float) * (size_t)S);
  free(qlab);
  free(sg);
  free(shat);
  free(idx);
  return keff;
}

/* ------------------------------------------------------------------ */
/* Batched driver over units (b, h): dense tensors
 *   q [B][Hq][d], K,V [B][Hkv][Smax][d], L [B][Hkv][Smax][r],
 *   C [Hkv][r], seq_lens [B]; y [B][Hq][d]; idx [B][Hkv][k] (-1 padded).
 * mode 0 = Double Sparsity (Alg. 1), mode 1 = dense attention.
 * codes [B][Hkv][Smax][r] + scale [B][Hkv][Smax] (nullable): 4-bit label.
 * nthreads > 1 statically partitions the independent units over pthreads
 * (the per-unit code is unchanged); it exists only for the cpu_baseline. */
typedef struct {
  const float *q, *qsel, *K, *V, *L;
  const int8_t *codes;
  const float *scale;
  const int32_t *C, *seq_lens;
  int B, Hq, Hkv, Smax, d, r, k, mode;
  float *y;
  int32_t *idx;
  int u0, u1;
} oracle_job;

static void *oracle_run_units(void *arg) {
  oracle_job *j = (oracle_job *)arg;
  int G = j->Hq / j->Hkv;
  for (int u = j->u0; u < j->u1; ++u) {
    int b = u / j->Hkv, h = u % j->Hkv;
    int S = j->seq_lens[b];
    const float *q = j->q + ((size_t)b * j->Hq + (size_t)h * G) * j->d;
    const float *qs = j->qsel + ((size_t)b * j->Hq + (size_t)h * G) * j->d;
    size_t kv = ((size_t)b * j->Hkv + h) * (size_t)j->Smax;
    float *y = j->y + ((size_t)b * j->Hq + (size_t)h * G) * j->d;
    if (j->mode == 1) {
      for (int g = 0; g < G; ++g)
        oracle_dense_attention(q + (size_t)g * j->d, j->K + kv * j->d,
                               j->V + kv * j->d, S, j->d, y + (size_t)g * j->d);
    } else {
      int32_t *idx = j->idx ? j->idx + ((size_t)b * j->Hkv + h) * j->k : NULL;
      int keff = oracle_ds_decode_unit(q, qs, G, j->K + kv * j->d, j->V + kv * j->d,
                                       j->L + kv * j->r,
                                       j->codes ? j->codes + kv * j->r : NULL,
                                       j->scale ? j->scale + kv : NULL,
                                       j->C + (size_t)h * j->r, S,
                                       j->d, j->r, j->k, y, idx, NULL, NULL);
      if (idx)
        for (int i = keff; i < j->k; ++i) idx[i] = -1;
    }
  }
  return NULL;
}

int oracle_decode_batch(const float *q, const float *qsel, const float *K,
                        const float *V, const float *L, const int8_t *codes,
                        const float *scale, const int32_t *C,
                        const int32_t *seq_lens, int B, int Hq, int Hkv,
                        int Smax, int d, int r, int k, int mode, float *y,
                        int32_t *idx, int nthreads) {
  if (Hkv <= 0 || Hq % Hkv != 0) return -1;
  int units = B * Hkv;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > units) nthreads = units;
  oracle_job *jobs = (oracle_job *)calloc((size_t)nthreads, sizeof(oracle_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    oracle_job j = {q, qsel ? qsel : q, K, V, L, codes, scale, C, seq_lens, B, Hq, Hkv,
                    Smax, d, r, k, mode, y, idx,
                    (int)((long)units * i / nthreads),
                    (int)((long)units * (i + 1) / nthreads)};
    jobs[i] = j;
  }
  for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, oracle_run_units, &jobs[i]);
  oracle_run_units(&jobs[0]);
  for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Offline calibration, Sec. 4.1: A = sum_i S_i with
 * S_i = Q_i * K_i; the critical channels are argmax_i S_i.  Reading R5:
 * aggregate |S_i| over every calibration (query, key) pair, which
 * factorises into (sum_n |Q_n,i|) * (sum_m |K_m,i|); reading R4: per KV
 * head, the group's query heads summed.  Modes follow Table 3:
 *   0 = qk outlier, 1 = q outlier, 2 = k outlier (N/A for GQA),
 *   3 = random channel (splitmix64 Fisher-Yates, seeded).
 * fp64 accumulation in sample order; top-r by importance desc, ties to
 * the lower channel; written ascending.  Returns 0, or
 * -2 for k mode with GQA, -1 for bad arguments.                        */
static uint64_t oracle_splitmix64(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int oracle_calibrate(const float *Qc /*[n][Hq][d]*/, const float *Kc /*[n][Hkv][d]*/,
                     int n, int Hq, int Hkv, int d, int mode, int r,
                     uint64_t seed, int32_t *C_out /*[Hkv][r]*/,
                     double *imp_out /*nullable [Hkv][d]*/) {
  if (Hkv <= 0 || Hq % Hkv != 0 || r < 1 || r > d) return -1;
  int G = Hq / Hkv;
  if (mode == 2 && G != 1) return -2;
  if (mode < 0 || mode > 3) return -1;
  double *imp = (double *)malloc(sizeof(double) * (size_t)d);
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)d);
  uint64_t state = seed;
  for (int h = 0; h < Hkv; ++h) {
    int32_t *C = C_out + (size_t)h * r;
    if (mode == 3) {
      for (int i = 0; i < d; ++i) perm[i] = i;
      for (int i = d - 1; i >= 1; --i) {
        int j = (int)(oracle_splitmix64(&state) % (uint64_t)(i + 1));
        int32_t tmp = perm[i];
        perm[i] = perm[j];
        perm[j] = tmp;
      }
      for (int i = 0; i < r; ++i) C[i] = perm[i];
      qsort(C, (size_t)r, sizeof(int32_t), oracle_int_cmp);
      if (imp_out)
        for (int c = 0; c < d; ++c) imp_out[(size_t)h * d + c] = 0.0;
      continue;
    }
    for (int c = 0; c < d; ++c) {
      double qs = 0.0, ks = 0.0;
      for (int s = 0; s < n; ++s) {
        for (int g = 0; g < G; ++g)
          qs = qs + fabs((double)Qc[((size_t)s * Hq + (size_t)h * G + g) * d + c]);
        ks = ks + fabs((double)Kc[((size_t)s * Hkv + h) * d + c]);
      }
      imp[c] = mode == 0 ? qs * ks : (mode == 1 ? qs : ks);
    }
    if (imp_out) memcpy(imp_out + (size_t)h * d, imp, sizeof(double) * (size_t)d);
    /* top-r by (importance desc, channel asc): repeated arg-max */
    char *taken = (char *)calloc((size_t)d, 1);
    for (int i = 0; i < r; ++i) {
      int best = -1;
      for (int c = 0; c < d; ++c)
        if (!taken[c] && (best < 0 || imp[c] > imp[best])) best = c;
      taken[best] = 1;
    }
    int o = 0;
    for (int c = 0; c < d; ++c)
      if (taken[c]) C[o++] = c;
    free(taken);
  }
  free(imp);
  free(perm);
  return 0;
}
