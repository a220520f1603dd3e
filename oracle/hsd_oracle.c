/*
 * hsd_oracle.c — CPU ORACLE (test infrastructure only; see hsd_oracle.h).
 *
 * Compiled with -O2 -ffp-contract=off (oracle/Makefile) so that every a*b+c is
 * two correctly-rounded IEEE operations, exactly like the reference built at
 * -O2 without -march=native.
 */
#include "hsd_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/hsd/hsd_synth.h"

/* ======================================================================== */
/* retrieval                                                                 */
/* ======================================================================== */

/* store.cpp:29-34 — `for i: s += a[i] * b[i]` in fp64. */
double hsdo_dot_f32(const float* a, const float* b, int dim) {
  double s = 0.0;
  for (int i = 0; i < dim; ++i) s += (double)a[i] * (double)b[i];
  return s;
}

/* (score desc, id asc) total order of store.cpp:67-70. */
static int better(double sa, int64_t ia, double sb, int64_t ib) {
  if (sa != sb) return sa > sb;
  return ia < ib;
}

/* Insert (s, id) into the sorted top-k list (len = current length). */
static void topk_insert(double* sc, int64_t* id, int* len, int k, double s, int64_t i) {
  if (*len == k && !better(s, i, sc[k - 1], id[k - 1])) return;
  int pos = (*len < k) ? *len : k - 1;
  while (pos > 0 && better(s, i, sc[pos - 1], id[pos - 1])) {
    sc[pos] = sc[pos - 1];
    id[pos] = id[pos - 1];
    --pos;
  }
  sc[pos] = s;
  id[pos] = i;
  if (*len < k) ++(*len);
}

/* store.cpp:59-73.  A full sort followed by truncation to k equals a bounded
 * insertion under the same total order. */
int hsdo_search_topk_exact(const float* keys, int64_t n, int dim, const float* query, int k, double* scores,
                           int64_t* ids) {
  if (k < 1) return -HSDO_INVALID_INPUT; /* store.cpp:60 */
  int len = 0;
  for (int64_t r = 0; r < n; ++r) {
    double s = hsdo_dot_f32(query, keys + (size_t)r * (size_t)dim, dim);
    topk_insert(scores, ids, &len, k, s, r);
  }
  return len;
}

/* `kind` may carry HSDO_KEYS_BF16: the stored key is the bf16 rounding
 * (RN-even) of the fp32 key, widened back to fp32 (bf16 collections). */
static void gen_key_row(int kind, uint64_t kbase, int64_t row, int dim, float* out, int64_t* scratch) {
  const int bf16 = (kind & HSDO_KEYS_BF16) != 0;
  kind &= ~HSDO_KEYS_BF16;
  int64_t src = hsd_key_src_row(kind, row);
  if (kind == HSD_SYNTH_EXACT) {
    for (int c = 0; c < dim; ++c) out[c] = hsd_exact_val(hsd_hash_at(kbase, (uint64_t)src * (uint64_t)dim + c));
  } else {
    int64_t ss = 0;
    for (int c = 0; c < dim; ++c) {
      scratch[c] = hsd_key_raw_kind(kind, kbase, src, dim, c);
      ss += scratch[c] * scratch[c];
    }
    for (int c = 0; c < dim; ++c) out[c] = hsd_norm_val(scratch[c], ss);
  }
  if (bf16)
    for (int c = 0; c < dim; ++c) out[c] = hsd_bf16_val(hsd_bf16_bits(out[c]));
}

void hsdo_gen_keys(int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim, float* out) {
  uint64_t kbase = hsd_stream_base(db_seed, HSD_TAG_KEYS);
  int64_t* scratch = (int64_t*)malloc(sizeof(int64_t) * (size_t)dim);
  for (int64_t r = 0; r < n; ++r) gen_key_row(kind, kbase, row0 + r, dim, out + (size_t)r * dim, scratch);
  free(scratch);
}

void hsdo_gen_queries(int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B, int dim,
                      float* out) {
  int64_t* raw = (int64_t*)malloc(sizeof(int64_t) * (size_t)dim);
  for (int b = 0; b < B; ++b) {
    int64_t q = q0 + b;
    int64_t row = hsd_query_row(q_seed, kind, q, n_rows);
    float* o = out + (size_t)b * dim;
    if (kind == HSD_SYNTH_EXACT) {
      for (int c = 0; c < dim; ++c) o[c] = hsd_query_exact(q_seed, db_seed, q, row, dim, c);
      continue;
    }
    int64_t ss = 0;
    for (int c = 0; c < dim; ++c) {
      raw[c] = hsd_query_raw_kind(kind, q_seed, db_seed, q, row, dim, c);
      ss += raw[c] * raw[c];
    }
    for (int c = 0; c < dim; ++c) o[c] = hsd_norm_val(raw[c], ss);
  }
  free(raw);
}

int hsdo_search_synth(int kind, uint64_t db_seed, int64_t n, int dim, const float* queries, int B, int k,
                      double* scores, int64_t* ids, int threads) {
  if (k < 1) return -HSDO_INVALID_INPUT;
  int nt = 1;
#ifdef _OPENMP
  nt = threads > 0 ? threads : omp_get_max_threads();
#else
  (void)threads;
#endif
  double* psc = (double*)malloc(sizeof(double) * (size_t)nt * B * k);
  int64_t* pid = (int64_t*)malloc(sizeof(int64_t) * (size_t)nt * B * k);
  int* plen = (int*)calloc((size_t)nt * B, sizeof(int));
  uint64_t kbase = hsd_stream_base(db_seed, HSD_TAG_KEYS);
#ifdef _OPENMP
#pragma omp parallel num_threads(nt)
#endif
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    float* row = (float*)malloc(sizeof(float) * (size_t)dim);
    int64_t* scratch = (int64_t*)malloc(sizeof(int64_t) * (size_t)dim);
    int64_t chunk = (n + nt - 1) / nt;
    int64_t r0 = chunk * t, r1 = r0 + chunk < n ? r0 + chunk : n;
    for (int64_t r = r0; r < r1; ++r) {
      gen_key_row(kind, kbase, r, dim, row, scratch);
      for (int b = 0; b < B; ++b) {
        double s = hsdo_dot_f32(queries + (size_t)b * dim, row, dim);
        size_t o = ((size_t)t * B + b);
        topk_insert(psc + o * k, pid + o * k, &plen[o], k, s, r);
      }
    }
    free(row);
    free(scratch);
  }
  int len = 0;
  for (int b = 0; b < B; ++b) {
    int l = 0;
    for (int t = 0; t < nt; ++t) {
      size_t o = ((size_t)t * B + b);
      for (int j = 0; j < plen[o]; ++j) topk_insert(scores + (size_t)b * k, ids + (size_t)b * k, &l, k, psc[o * k + j], pid[o * k + j]);
    }
    len = l;
  }
  free(psc);
  free(pid);
  free(plen);
  return len;
}

/* ======================================================================== */
/* actions                                                                   */
/* ======================================================================== */

/* actions.cpp:32-50 (validate :17-26, check_k :28-30). */
int hsdo_quantize(const double* a7, const double* lo7, const double* hi7, int k_bins, int* bins7) {
  if (k_bins < 2) return -HSDO_CONFIG;
  for (int i = 0; i < 7; ++i) {
    if (!isfinite(lo7[i]) || !isfinite(hi7[i])) return -HSDO_CONFIG;
    if (!(lo7[i] < hi7[i])) return -HSDO_CONFIG;
  }
  for (int i = 0; i < 7; ++i) {
    const double v = a7[i];
    if (!isfinite(v)) return -HSDO_INVALID_INPUT;
    const double lo = lo7[i], hi = hi7[i];
    const double clamped = v < lo ? lo : (hi < v ? hi : v); /* std::clamp */
    const double t = (clamped - lo) / (hi - lo);
    int bin = (int)floor(t * (k_bins - 1));
    if (bin < 0) bin = 0;
    if (bin > k_bins - 1) bin = k_bins - 1;
    bins7[i] = bin;
  }
  return 0;
}

void hsdo_synth_tokens(uint64_t db_seed, int64_t row, uint8_t* tok21) {
  double lo[7], hi[7], a[7];
  int bins[7];
  for (int i = 0; i < 7; ++i) {
    lo[i] = -1.0;
    hi[i] = 1.0;
  }
  for (int s = 0; s < 3; ++s) {
    for (int j = 0; j < 7; ++j) a[j] = hsd_action_val(db_seed, row, s, j);
    hsdo_quantize(a, lo, hi, 256, bins);
    for (int j = 0; j < 7; ++j) tok21[s * 7 + j] = (uint8_t)bins[j];
  }
}

void hsdo_gen_features(uint64_t seed, int64_t e0, int E, int d_f, float* now, float* prev) {
  int64_t* raw = (int64_t*)malloc(sizeof(int64_t) * (size_t)d_f);
  for (int e = 0; e < E; ++e) {
    for (int which = 0; which < 2; ++which) {
      int64_t ss = 0;
      for (int c = 0; c < d_f; ++c) {
        raw[c] = hsd_feat_raw(seed, e0 + e, which, d_f, c);
        ss += raw[c] * raw[c];
      }
      float* o = (which ? prev : now) + (size_t)e * d_f;
      for (int c = 0; c < d_f; ++c) o[c] = hsd_norm_val(raw[c], ss);
    }
  }
  free(raw);
}

void hsdo_gen_logits(uint64_t db_seed, uint64_t seed, const int64_t* rows, int64_t e0, int E, int L, float* out) {
  uint8_t tok[21];
  for (int e = 0; e < E; ++e) {
    int64_t ee = e0 + e;
    int64_t row = rows ? rows[e] : -1;
    if (row >= 0) hsdo_synth_tokens(db_seed, row, tok);
    for (int p = 0; p < L; ++p) {
      int draft = row >= 0 ? tok[p]
                           : (int)(hsd_hash_at(hsd_stream_base(seed, HSD_TAG_LOGITS), ((uint64_t)ee << 8) ^ (0xD000u + p)) &
                                   0xFFu);
      int g = hsd_logit_greedy_bin(seed, ee, p, draft);
      int tie = hsd_logit_tie_bin(seed, ee, p);
      float* o = out + ((size_t)e * L + p) * 256;
      for (int b = 0; b < 256; ++b) o[b] = (b == g || b == tie) ? 8.0f : hsd_logit_background(seed, ee, p, b);
    }
  }
}

/* ======================================================================== */
/* verification                                                              */
/* ======================================================================== */

int hsdo_token_bias(int draft_bin, int verify_bin) { return abs(draft_bin - verify_bin); }

/* SPEC.md:430-439.  Gripper groups: accept iff bias == 0.  Otherwise, with
 * relaxation on: accept iff sum(bias) <= bias_seq_max and every bias <=
 * bias_token_max; relaxation off: accept iff all biases are 0 (Eq. 2-2). */
int hsdo_accept_sequence(const int* draft, const int* verify, int n, int is_gripper, const hsdo_accept_params* p) {
  int sum = 0, mx = 0;
  for (int i = 0; i < n; ++i) {
    int b = hsdo_token_bias(draft[i], verify[i]);
    sum += b;
    if (b > mx) mx = b;
  }
  if (is_gripper || !p->enabled) return mx == 0;
  return sum <= p->bias_seq_max && mx <= p->bias_token_max;
}

int hsdo_argmax(const float* logits, int nbins) {
  int best = 0;
  for (int b = 1; b < nbins; ++b)
    if (logits[b] > logits[best]) best = b;
  return best;
}

/* Knuth TwoSum. */
static void two_sum(double a, double b, double* s, double* e) {
  double x = a + b;
  double bv = x - a;
  double av = x - bv;
  *e = (a - av) + (b - bv);
  *s = x;
}

/* Double-double accumulation of exact fp64 products of fp32 inputs; the
 * result is the correctly rounded dot except within ~2^-100 relative. */
double hsdo_feature_cos(const float* a, const float* b, int dim) {
  double hi = 0.0, lo = 0.0;
  for (int i = 0; i < dim; ++i) {
    double p = (double)a[i] * (double)b[i]; /* exact */
    double s, e;
    two_sum(hi, p, &s, &e);
    hi = s;
    lo += e;
  }
  double s, e;
  two_sum(hi, lo, &s, &e);
  return s;
}

/* SPEC.md:458-466. */
int hsdo_should_skip(double cos_now_prev, const hsdo_skip_state* s, int gap_d, int history) {
  if (gap_d < 1 || history < gap_d) return 0;
  return gap_d <= s->O_dist && cos_now_prev >= s->min_S;
}

/* Group layout of one action slice (actions.hpp:11-12):
 * pos = dims 0-2, rot = 3-5, grip = 6. */
static int group_count(int L) { return (L / 7) * 3; }
static void group_at(int g, int* start, int* len, int* grip) {
  int s = g / 3, kind = g % 3;
  *start = s * 7 + (kind == 0 ? 0 : (kind == 1 ? 3 : 6));
  *len = kind == 2 ? 1 : 3;
  *grip = kind == 2;
}

/* Accepted prefix (in tokens) of one chain against the greedy tokens. */
static int chain_prefix(const int* chain, int L, const int* greedy, const hsdo_accept_params* p) {
  int acc = 0, G = group_count(L);
  for (int g = 0; g < G; ++g) {
    int st, ln, gr;
    group_at(g, &st, &ln, &gr);
    if (!hsdo_accept_sequence(chain + st, greedy + st, ln, gr, p)) break;
    acc += ln;
  }
  return acc;
}

/* Brute-force DFS enumeration of the sequence-wise tree
 * under the gripper-isolation invariant: every gripper
 * level links only to a same-rank parent and child, so every level after pos0
 * carries one rank b; pos0 may come from any rank a.  Children are visited
 * best-rank-first; identical token sequences are emitted once (per-level dedup
 * keeping the best rank leaves the chain language unchanged). */
int hsdo_enumerate_chains(const int* drafts, int n_cand, int L, int cap, int* chains_out, int* a_out, int* b_out) {
  int count = 0;
  int* tmp = (int*)malloc(sizeof(int) * (size_t)L);
  for (int a = 0; a < n_cand && count < cap; ++a) {
    for (int b = 0; b < n_cand && count < cap; ++b) {
      for (int t = 0; t < L; ++t) tmp[t] = (t < 3) ? drafts[a * L + t] : drafts[b * L + t];
      int dup = 0;
      for (int c = 0; c < count && !dup; ++c) dup = memcmp(chains_out + (size_t)c * L, tmp, sizeof(int) * L) == 0;
      if (dup) continue;
      memcpy(chains_out + (size_t)count * L, tmp, sizeof(int) * L);
      a_out[count] = a;
      b_out[count] = b;
      ++count;
    }
  }
  free(tmp);
  return count;
}

void hsdo_verify_round(const int* drafts, int n_cand, int L, const int* greedy, int skip, int cap,
                       const hsdo_accept_params* p, hsdo_outcome* out) {
  memset(out, 0, sizeof(*out));
  if (n_cand <= 0) { /* empty shard: autoregressive step */
    out->fallback = 1;
    out->calls = 1;
    out->n_emit = 1;
    out->tokens[0] = greedy[0];
    out->win_a = out->win_b = -1;
    return;
  }
  if (skip) { /* skipped drafts count as fully accepted */
    out->skipped = 1;
    out->accept_len = L;
    out->n_emit = L;
    for (int t = 0; t < L; ++t) out->tokens[t] = drafts[t];
    return;
  }
  int* chains = (int*)malloc(sizeof(int) * (size_t)cap * L);
  int* as = (int*)malloc(sizeof(int) * (size_t)cap);
  int* bs = (int*)malloc(sizeof(int) * (size_t)cap);
  int n = hsdo_enumerate_chains(drafts, n_cand, L, cap, chains, as, bs);
  int best = -1, best_len = -1;
  for (int c = 0; c < n; ++c) {
    int len = chain_prefix(chains + (size_t)c * L, L, greedy, p);
    if (len > best_len) { /* earliest chain wins ties */
      best_len = len;
      best = c;
    }
  }
  out->calls = n;
  out->win_a = as[best];
  out->win_b = bs[best];
  out->accept_len = best_len;
  if (best_len == 0) { /* SPEC.md:443 fallback: one greedy verifier token */
    out->fallback = 1;
    out->n_emit = 1;
    out->tokens[0] = greedy[0];
  } else {
    out->n_emit = best_len;
    for (int t = 0; t < best_len; ++t) out->tokens[t] = chains[(size_t)best * L + t];
  }
  free(chains);
  free(as);
  free(bs);
}

/* verify_tree with teacher-forced per-chain verifier output
 * (VerifierModel::verify_chain, models.hpp:34-37): chain c of the brute-force
 * enumeration above is compared with its own greedy tokens
 * chain_greedy[c][0..L); the fallback / empty-shard token is greedy_ctx =
 * greedy_next(context) (models.hpp:38-39).  Otherwise as hsdo_verify_round. */
void hsdo_verify_round_chains(const int* drafts, int n_cand, int L, const int* chain_greedy, int greedy_ctx, int skip,
                              int cap, const hsdo_accept_params* p, hsdo_outcome* out) {
  memset(out, 0, sizeof(*out));
  if (n_cand <= 0) {
    out->fallback = 1;
    out->calls = 1;
    out->n_emit = 1;
    out->tokens[0] = greedy_ctx;
    out->win_a = out->win_b = -1;
    return;
  }
  if (skip) {
    out->skipped = 1;
    out->accept_len = L;
    out->n_emit = L;
    for (int t = 0; t < L; ++t) out->tokens[t] = drafts[t];
    return;
  }
  int* chains = (int*)malloc(sizeof(int) * (size_t)cap * L);
  int* as = (int*)malloc(sizeof(int) * (size_t)cap);
  int* bs = (int*)malloc(sizeof(int) * (size_t)cap);
  int n = hsdo_enumerate_chains(drafts, n_cand, L, cap, chains, as, bs);
  int best = -1, best_len = -1;
  for (int c = 0; c < n; ++c) {
    int len = chain_prefix(chains + (size_t)c * L, L, chain_greedy + (size_t)c * L, p);
    if (len > best_len) {
      best_len = len;
      best = c;
    }
  }
  out->calls = n;
  out->win_a = as[best];
  out->win_b = bs[best];
  out->accept_len = best_len;
  if (best_len == 0) {
    out->fallback = 1;
    out->n_emit = 1;
    out->tokens[0] = greedy_ctx;
  } else {
    out->n_emit = best_len;
    for (int t = 0; t < best_len; ++t) out->tokens[t] = chains[(size_t)best * L + t];
  }
  free(chains);
  free(as);
  free(bs);
}

void hsdo_calibrate_init(hsdo_calib* c) {
  c->min_S = INFINITY;
  c->O_dist = 0;
  c->found = 0;
}

/* SPEC.md:449-457 / PAPER.md:258-265 with the spec's reading (min_S starts at
 * +inf, all pairs (i, i+d), d >= 1): first strict minimum of S > T in (i, d)
 * loop order. */
void hsdo_calibrate_accumulate(hsdo_calib* c, const double* sims, int n, double T) {
  for (int i = 0; i < n - 1; ++i) {
    for (int d = 1; i + d < n; ++d) {
      double S = sims[(size_t)i * n + (i + d)];
      if (S > T && S < c->min_S) {
        c->min_S = S;
        c->O_dist = d;
        c->found = 1;
      }
    }
  }
}

int hsdo_calibrate_finish(const hsdo_calib* c, double* min_S, int* O_dist) {
  if (!c->found) return -HSDO_CALIBRATION;
  *min_S = c->min_S;
  *O_dist = c->O_dist;
  return 0;
}

/* literal Alg. 1 arithmetic, optional inversion, clamp [T, 1]. */
void hsdo_update_skip_state(hsdo_skip_state* s, int success, double S_c, double min_S_h) {
  double adj = s->delta * fabs(S_c - min_S_h);
  double sign = success ? 1.0 : -1.0;
  if (s->inverted) sign = -sign;
  s->min_S += sign * adj;
  if (success)
    s->O_dist += 1;
  else
    s->O_dist = s->O_dist - 1 < 1 ? 1 : s->O_dist - 1;
  if (s->min_S < s->T) s->min_S = s->T;
  if (s->min_S > 1.0) s->min_S = 1.0;
}

/* ======================================================================== */
/* kinematics (Eigen-free restatement of kinematics.cpp)                     */
/* ======================================================================== */

/* Cyclic Jacobi eigen-decomposition of a symmetric 3x3 matrix; eigenvalues
 * ascending with matching eigenvector columns (Eigen's SelfAdjointEigenSolver
 * ordering, kinematics.cpp:57-60). */
static void eig3_sym(const double A_in[3][3], double w[3], double V[3][3]) {
  double A[3][3];
  memcpy(A, A_in, sizeof(A));
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    double scale = fabs(A[0][0]) + fabs(A[1][1]) + fabs(A[2][2]);
    if (off == 0.0 || off <= 1e-300 || off <= scale * 1e-18) break;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) { /* A = J^T A J */
          double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
    }
  }
  int idx[3] = {0, 1, 2};
  double d[3] = {A[0][0], A[1][1], A[2][2]};
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (d[idx[j]] < d[idx[i]]) {
        int t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
      }
  double Vs[3][3];
  for (int c = 0; c < 3; ++c) {
    w[c] = d[idx[c]];
    for (int r = 0; r < 3; ++r) Vs[r][c] = V[r][idx[c]];
  }
  memcpy(V, Vs, sizeof(Vs));
}

static int all_finite3(const double* xyz, int n) {
  for (int i = 0; i < 3 * n; ++i)
    if (!isfinite(xyz[i])) return 0;
  return 1;
}

/* kinematics.cpp:38-76 */
int hsdo_project_window(const double* xyz, int n, double* uv) {
  if (n < 3) return -HSDO_INVALID_INPUT;
  if (!all_finite3(xyz, n)) return -HSDO_INVALID_INPUT;
  double mean[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) mean[j] += xyz[3 * i + j];
  for (int j = 0; j < 3; ++j) mean[j] /= (double)n;
  double C[3][3] = {{0}};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += (xyz[3 * i + a] - mean[a]) * (xyz[3 * i + b] - mean[b]);
      C[a][b] = s;
    }
  double w[3], V[3][3];
  eig3_sym(C, w, V);
  double u[3] = {V[0][2], V[1][2], V[2][2]};
  double v[3] = {V[0][1], V[1][1], V[2][1]};
  double* axes[2] = {u, v};
  for (int k = 0; k < 2; ++k) { /* canonical sign, kinematics.cpp:63-69 */
    double* ax = axes[k];
    int lead = 0;
    for (int j = 1; j < 3; ++j)
      if (fabs(ax[j]) > fabs(ax[lead])) lead = j;
    if (ax[lead] < 0.0)
      for (int j = 0; j < 3; ++j) ax[j] = -ax[j];
  }
  for (int i = 0; i < n; ++i) {
    double c0 = xyz[3 * i] - mean[0], c1 = xyz[3 * i + 1] - mean[1], c2 = xyz[3 * i + 2] - mean[2];
    uv[2 * i] = c0 * u[0] + c1 * u[1] + c2 * u[2];
    uv[2 * i + 1] = c0 * v[0] + c1 * v[1] + c2 * v[2];
  }
  return 0;
}

/* RadiusObjective::eval, kinematics.cpp:90-103 */
static double radius_objective(const double* uv, int n, double cx, double cy) {
  double mu = 0.0;
  for (int i = 0; i < n; ++i) mu += hypot(uv[2 * i] - cx, uv[2 * i + 1] - cy);
  mu /= (double)n;
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    double r = hypot(uv[2 * i] - cx, uv[2 * i + 1] - cy);
    s += (r - mu) * (r - mu);
  }
  return s;
}

/* LDLT (diagonal pivoting) solve of the SPD 2x2 system M x = rhs. */
static void ldlt2_solve(double a, double b, double c, double r0, double r1, double* x0, double* x1) {
  int swap = fabs(c) > fabs(a);
  double A00 = swap ? c : a, A11 = swap ? a : c;
  double q0 = swap ? r1 : r0, q1 = swap ? r0 : r1;
  double d0 = A00;
  double l = b / d0;
  double d1 = A11 - l * b;
  double y0 = q0, y1 = q1 - l * y0;
  double z0 = y0 / d0, z1 = y1 / d1;
  double s1 = z1, s0 = z0 - l * s1;
  *x0 = swap ? s1 : s0;
  *x1 = swap ? s0 : s1;
}

/* kinematics.cpp:107-207 */
int hsdo_fit_circle_center(const double* uv, int n, double* cu, double* cv, int* degenerate, int* iterations) {
  if (n < 3) return -HSDO_INVALID_INPUT;
  for (int i = 0; i < 2 * n; ++i)
    if (!isfinite(uv[i])) return -HSDO_INVALID_INPUT;
  double cx = 0.0, cy = 0.0;
  for (int i = 0; i < n; ++i) {
    cx += uv[2 * i];
    cy += uv[2 * i + 1];
  }
  cx /= (double)n;
  cy /= (double)n;
  double spread = 0.0; /* max_pairwise_distance, :78-86 */
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double dd = hypot(uv[2 * i] - uv[2 * j], uv[2 * i + 1] - uv[2 * j + 1]);
      if (dd > spread) spread = dd;
    }
  *iterations = 0;
  *degenerate = 0;
  if (spread < 1e-9) {
    *cu = cx;
    *cv = cy;
    *degenerate = 1;
    return 0;
  }
  /* 2x2 scatter and its minor eigenpair (:135-144) */
  double sa = 0, sb = 0, sc = 0;
  for (int i = 0; i < n; ++i) {
    double dx = uv[2 * i] - cx, dy = uv[2 * i + 1] - cy;
    sa += dx * dx;
    sb += dx * dy;
    sc += dy * dy;
  }
  double half_tr = 0.5 * (sa + sc), half_diff = 0.5 * (sa - sc);
  double rad = sqrt(half_diff * half_diff + sb * sb);
  double l1 = half_tr + rad;
  double l0 = half_tr - rad;
  double ex, ey; /* eigenvector of l0 */
  if (sb == 0.0) {
    if (sa <= sc) {
      ex = 1.0;
      ey = 0.0;
    } else {
      ex = 0.0;
      ey = 1.0;
    }
  } else if (fabs(l0 - sa) >= fabs(l0 - sc)) {
    ex = sb;
    ey = l0 - sa;
  } else {
    ex = l0 - sc;
    ey = sb;
  }
  double en = sqrt(ex * ex + ey * ey);
  ex /= en;
  ey /= en;
  double x = cx, y = cy;
  if (l0 <= 1e-12 * l1) {
    x += ex * spread;
    y += ey * spread;
  }
  double lambda = 1e-6;
  double objective = radius_objective(uv, n, x, y);
  double radii[64], ux[64], uy[64];
  for (int iter = 0; iter < 100; ++iter) {
    *iterations = iter + 1;
    double mu = 0.0, mux = 0.0, muy = 0.0;
    for (int i = 0; i < n; ++i) {
      double dx = uv[2 * i] - x, dy = uv[2 * i + 1] - y;
      double r = sqrt(dx * dx + dy * dy); /* Vector2d::norm */
      radii[i] = r;
      ux[i] = r > 0.0 ? dx / r : 0.0;
      uy[i] = r > 0.0 ? dy / r : 0.0;
      mu += r;
    }
    mu /= (double)n;
    for (int i = 0; i < n; ++i) {
      mux += ux[i];
      muy += uy[i];
    }
    mux /= (double)n;
    muy /= (double)n;
    double j00 = 0, j01 = 0, j11 = 0, g0 = 0, g1 = 0;
    for (int i = 0; i < n; ++i) {
      double jx = -ux[i] + mux, jy = -uy[i] + muy;
      double f = radii[i] - mu;
      j00 += jx * jx;
      j01 += jx * jy;
      j11 += jy * jy;
      g0 += jx * f;
      g1 += jy * f;
    }
    int moved = 0;
    for (int attempt = 0; attempt < 25; ++attempt) {
      double s0, s1;
      ldlt2_solve(j00 + lambda, j01, j11 + lambda, -g0, -g1, &s0, &s1);
      if (!isfinite(s0) || !isfinite(s1)) {
        lambda *= 10.0;
        continue;
      }
      double nx = x + s0, ny = y + s1;
      double cand = radius_objective(uv, n, nx, ny);
      if (cand <= objective) {
        x = nx;
        y = ny;
        objective = cand;
        lambda = lambda * 0.3 > 1e-12 ? lambda * 0.3 : 1e-12;
        moved = sqrt(s0 * s0 + s1 * s1) >= 1e-10;
        if (!moved) {
          *cu = x;
          *cv = y;
          return 0;
        }
        break;
      }
      lambda *= 10.0;
    }
    if (!moved) break;
  }
  *cu = x;
  *cv = y;
  return 0;
}

/* kinematics.cpp:209-218 */
int hsdo_curvature_radius(const double* xyz, int n, double r_cap, double* R) {
  if (!(r_cap > 0.0)) return -HSDO_CONFIG;
  if (n > 64) return -HSDO_INVALID_INPUT; /* oracle buffer bound */
  double uv[128];
  int rc = hsdo_project_window(xyz, n, uv);
  if (rc) return rc;
  double cu, cv;
  int deg, it;
  rc = hsdo_fit_circle_center(uv, n, &cu, &cv, &deg, &it);
  if (rc) return rc;
  if (deg) {
    *R = 0.0;
    return 0;
  }
  double m = 0.0;
  for (int i = 0; i < n; ++i) m += hypot(uv[2 * i] - cu, uv[2 * i + 1] - cv);
  m /= (double)n;
  *R = m < r_cap ? m : r_cap;
  return 0;
}

/* kinematics.cpp:220-230 */
int hsdo_cumulative_displacement(const double* xyz, int n, double* D) {
  if (n < 2) return -HSDO_INVALID_INPUT;
  if (!all_finite3(xyz, n)) return -HSDO_INVALID_INPUT;
  double total = 0.0;
  for (int i = 0; i + 1 < n; ++i) {
    double dx = xyz[3 * i] - xyz[3 * i + 3], dy = xyz[3 * i + 1] - xyz[3 * i + 4], dz = xyz[3 * i + 2] - xyz[3 * i + 5];
    total += sqrt(dx * dx + dy * dy + dz * dz); /* Vec3::norm, geometry.hpp:17 */
  }
  *D = total;
  return 0;
}

/* kinematics.cpp:232-236 (lo > hi95 is the caller's InvalidInput) */
double hsdo_normalize(double x, double lo, double hi95) {
  if (lo == hi95) return 0.0;
  double t = (x - lo) / (hi95 - lo);
  return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* kinematics.cpp:238-247 (nearest rank) */
int hsdo_percentile_bounds(const double* samples, int n, double* lo, double* p95) {
  if (n <= 0) return -HSDO_INVALID_INPUT;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(s, samples, sizeof(double) * (size_t)n);
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  size_t rank = (size_t)ceil(0.95 * (double)n);
  if (rank < 1) rank = 1;
  size_t idx = rank - 1 < (size_t)n - 1 ? rank - 1 : (size_t)n - 1;
  *lo = s[0];
  *p95 = s[idx];
  free(s);
  return 0;
}

double hsdo_fused_metric(double R, double D, const hsdo_metric_params* p, const hsdo_norm_bounds* b) {
  double nr = hsdo_normalize(R, b->r_min, b->r_max95);
  double nd = hsdo_normalize(D, b->d_min, b->d_max95);
  return p->alpha * nr + (1.0 - p->alpha) * nd;
}

int hsdo_classify(double F, double threshold) { return F > threshold ? 1 : 0; }

int hsdo_window_features(const double* xyz, int n, const hsdo_metric_params* p, const hsdo_norm_bounds* b, double* R,
                         double* D, double* F, int* decision) {
  if (n != p->w) return -HSDO_INVALID_INPUT;
  int rc = hsdo_curvature_radius(xyz, n, p->r_cap, R);
  if (rc) return rc;
  rc = hsdo_cumulative_displacement(xyz, n, D);
  if (rc) return rc;
  *F = hsdo_fused_metric(*R, *D, p, b);
  *decision = hsdo_classify(*F, p->threshold);
  return 0;
}

#define HSD_MODE_HYBRID_O 0
#define HSD_K_MAX_O 32
#define HSD_HYB_MAX_EMIT_O 28

/* ------------------------------------------------------- hybrid loop (config 5)
 * SPEC.md:508-578 run_step per robot and round:
 *   decide_sd: window_features over the trailing w points
 *     (kinematics.cpp:261-273), cold start (< w points) -> drafter; pure modes
 *     override;
 *   retrieval_sd: retrieve_drafts (search_topk_exact over the
 *     stored keys, payload = the demonstration policy tokens) -> should_skip
 *      -> verify_tree;
 *   drafter_sd: drafter_generate (toy drafter) -> verify;
 *   emit + autoregressive completion of the action slice, ToyEnv position,
 *   trajectory history, cost model. */
static void hyb_window(const double* ring, int w, int n, double* out) {
  for (int i = 0; i < w; ++i) {
    int src = n >= w ? (n - w + i) % w : (i < n ? i : (n > 0 ? n - 1 : 0));
    out[i * 3 + 0] = ring[src * 3 + 0];
    out[i * 3 + 1] = ring[src * 3 + 1];
    out[i * 3 + 2] = ring[src * 3 + 2];
  }
}

static void hyb_query(const hsdo_hybrid_params* p, int64_t qid, int64_t row, int dim, float* q, int64_t* raw) {
  const int kind = p->key_kind & ~HSDO_KEYS_BF16;
  if (kind == HSD_SYNTH_EXACT) {
    for (int c = 0; c < dim; ++c) q[c] = hsd_query_exact(p->seed, p->db_seed, qid, row, dim, c);
    return;
  }
  int64_t ss = 0;
  for (int c = 0; c < dim; ++c) {
    raw[c] = hsd_query_raw(p->seed, p->db_seed, qid, row, dim, c);
    ss += raw[c] * raw[c];
  }
  for (int c = 0; c < dim; ++c) q[c] = hsd_norm_val(raw[c], ss);
}

int hsdo_hybrid_run(const hsdo_hybrid_params* p, int64_t n_rows, int dim, int rounds, hsdo_step_record* trace,
                    double* pos, hsdo_episode_report* rep) {
  const int R = p->robots, w = p->metric.w, k = p->k, L = p->drafter_L;
  const int64_t n_demo = n_rows / p->traj_T;
  double* ring = (double*)calloc((size_t)R * w * 3, sizeof(double));
  int* hist_n = (int*)calloc((size_t)R, sizeof(int));
  int64_t* act = (int64_t*)calloc((size_t)R, sizeof(int64_t));
  int* nrounds = (int*)calloc((size_t)R, sizeof(int));
  int* modes = (int*)calloc((size_t)R, sizeof(int));
  double* Fv = (double*)calloc((size_t)R, sizeof(double));
  int* ret = (int*)malloc(sizeof(int) * (size_t)R);
  float* qs = (float*)malloc(sizeof(float) * (size_t)R * dim);
  int64_t* raw = (int64_t*)malloc(sizeof(int64_t) * (size_t)(dim > p->d_f ? dim : p->d_f) + 8);
  double* sc = (double*)malloc(sizeof(double) * (size_t)R * k);
  int64_t* ids = (int64_t*)malloc(sizeof(int64_t) * (size_t)R * k);
  float* fn = (float*)malloc(sizeof(float) * (size_t)(p->d_f > 0 ? p->d_f : 1));
  float* fp = (float*)malloc(sizeof(float) * (size_t)(p->d_f > 0 ? p->d_f : 1));
  hsdo_outcome* outs = (hsdo_outcome*)malloc(sizeof(hsdo_outcome) * (size_t)R);
  const hsdo_accept_params ap = {p->relaxed, p->bias_seq_max, p->bias_token_max};
  const hsdo_skip_state ss = {0.0, p->min_S, p->O_dist, 0.0, 0};
  double win[3 * 32];
  for (int r = 0; r < R; ++r) {
    for (int d = 0; d < 3; ++d) pos[r * 3 + d] = ring[(size_t)r * w * 3 + d] = hsd_robot_start(p->seed, r, d);
    hist_n[r] = 1;
    memset(&rep[r], 0, sizeof(rep[r]));
  }
  for (int round = 0; round < rounds; ++round) {
    int nr = 0;
    for (int r = 0; r < R; ++r) {  /* decide_sd */
      double Rk = 0, Dk = 0, F = 0;
      int dec = 0;
      hyb_window(ring + (size_t)r * w * 3, w, hist_n[r], win);
      hsdo_window_features(win, w, &p->metric, &p->bounds, &Rk, &Dk, &F, &dec);
      if (hist_n[r] < w) dec = 0; /* cold start */
      Fv[r] = F;
      if (p->mode == HSD_MODE_HYBRID_O)
        modes[r] = dec == 1 ? 1 : 0;
      else
        modes[r] = p->mode == 1 ? 1 : (p->mode == 2 ? 0 : 2);
      if (modes[r] == 1) ret[nr++] = r;
    }
    /* retrieve_drafts: one batched exact search over the stored keys */
    for (int i = 0; i < nr; ++i) {
      const int r = ret[i];
      const int64_t e = hsd_robot_episode(p->seed, r, n_demo);
      const int64_t row = hsd_hybrid_query_row(e, act[r], p->traj_T, n_demo, n_rows);
      hyb_query(p, hsd_hybrid_qid(r, round), row, dim, qs + (size_t)i * dim, raw);
    }
    if (nr > 0) hsdo_search_synth(p->key_kind, p->db_seed, n_rows, dim, qs, nr, k, sc, ids, 0);
    for (int i = 0; i < nr; ++i) { /* should_skip + verify_tree */
      const int r = ret[i];
      const int64_t e = hsd_robot_episode(p->seed, r, n_demo);
      int greedy[21], drafts[HSD_K_MAX_O * 21], nc = 0;
      for (int q = 0; q < 21; ++q) greedy[q] = hsd_robot_greedy(p->db_seed, p->seed, r, e, act[r] + q / 7, q % 7);
      for (int c = 0; c < k; ++c) {
        const int64_t id = ids[(size_t)i * k + c];
        if (id < 0) continue;
        for (int q = 0; q < 21; ++q)
          drafts[nc * 21 + q] = hsd_policy_token(p->db_seed, id / p->traj_T, id % p->traj_T + q / 7, q % 7);
        ++nc;
      }
      int skip = 0;
      if (p->skip_enabled) {
        hsdo_gen_features(p->seed, hsd_hybrid_qid(r, round), 1, p->d_f, fn, fp);
        skip = hsdo_should_skip(hsdo_feature_cos(fn, fp, p->d_f), &ss, p->gap_d, nrounds[r]);
      }
      if (nc == 0) { /* empty shard: autoregressive for the step */
        memset(&outs[r], 0, sizeof(outs[r]));
        outs[r].calls = 1;
        outs[r].fallback = 1;
        outs[r].n_emit = 1;
        outs[r].tokens[0] = greedy[0];
      } else {
        hsdo_verify_round(drafts, nc, 21, greedy, skip, p->chain_cap, &ap, &outs[r]);
      }
    }
    for (int r = 0; r < R; ++r) { /* drafter_generate + verify */
      if (modes[r] != 0) continue;
      const int64_t e = hsd_robot_episode(p->seed, r, n_demo);
      int greedy[21], draft[21];
      for (int q = 0; q < L; ++q) {
        greedy[q] = hsd_robot_greedy(p->db_seed, p->seed, r, e, act[r] + q / 7, q % 7);
        draft[q] = hsd_drafter_token(p->seed, r, round, q, greedy[q], p->drafter_p_pct);
      }
      hsdo_verify_round(draft, 1, L, greedy, 0, p->chain_cap, &ap, &outs[r]);
    }
    for (int r = 0; r < R; ++r) { /* emit, ToyEnv, history, cost */
      const int m = modes[r];
      const int64_t e = hsd_robot_episode(p->seed, r, n_demo);
      int toks[HSD_HYB_MAX_EMIT_O], n = 0, accepted = 0, calls = 0, skipped = 0, fallback = 0;
      double cost = 0.0;
      if (m == 0 || m == 1) {
        const hsdo_outcome* o = &outs[r];
        for (int i = 0; i < o->n_emit; ++i) toks[n++] = o->tokens[i];
        accepted = o->accept_len;
        calls = o->calls;
        skipped = o->skipped;
        fallback = o->fallback;
        cost = m == 1 ? p->cost_retrieval : p->cost_drafter_token * (double)L;
      }
      const int target = n == 0 ? 7 : ((n + 6) / 7) * 7;
      while (n < target) {
        toks[n] = hsd_robot_greedy(p->db_seed, p->seed, r, e, act[r] + n / 7, n % 7);
        ++n;
        ++calls;
      }
      cost = cost + (double)calls * p->cost_verifier;
      double* rg = ring + (size_t)r * w * 3;
      for (int a = 0; a < n / 7; ++a) {
        for (int d = 0; d < 3; ++d) pos[r * 3 + d] = pos[r * 3 + d] + HSD_ENV_SCALE * hsd_dequantize_bin(toks[a * 7 + d], -1.0, 1.0, 256);
        const int sw = hist_n[r] % w;
        rg[sw * 3 + 0] = pos[r * 3 + 0];
        rg[sw * 3 + 1] = pos[r * 3 + 1];
        rg[sw * 3 + 2] = pos[r * 3 + 2];
        ++hist_n[r];
      }
      act[r] += n / 7;
      nrounds[r] += 1;
      rep[r].rounds += 1;
      rep[r].tokens += n;
      rep[r].accepted += accepted;
      rep[r].verifier_calls += calls;
      rep[r].cost += cost;
      rep[r].n_retrieval += m == 1;
      rep[r].n_drafter += m == 0;
      rep[r].n_skipped += skipped;
      rep[r].n_fallback += fallback;
      if (trace) {
        hsdo_step_record* t = &trace[(size_t)round * R + r];
        t->F = m == 2 ? -1.0f : (float)Fv[r];
        t->accept_len = (int16_t)accepted;
        t->verifier_calls = (int16_t)calls;
        t->n_emit = (int16_t)n;
        t->mode = (int8_t)m;
        t->skipped = (int8_t)skipped;
        t->cost = (float)cost;
      }
    }
  }
  free(ring);
  free(hist_n);
  free(act);
  free(nrounds);
  free(modes);
  free(Fv);
  free(ret);
  free(qs);
  free(raw);
  free(sc);
  free(ids);
  free(fn);
  free(fp);
  free(outs);
  return 0;
}

int hsdo_policy_token(uint64_t db_seed, int64_t e, int64_t j, int d) { return hsd_policy_token(db_seed, e, j, d); }
int hsdo_robot_greedy(uint64_t db_seed, uint64_t seed, int64_t r, int64_t n_demo, int64_t j, int d) {
  return hsd_robot_greedy(db_seed, seed, r, hsd_robot_episode(seed, r, n_demo), j, d);
}
double hsdo_robot_start(uint64_t seed, int64_t r, int d) { return hsd_robot_start(seed, r, d); }
double hsdo_dequantize_bin(int bin, double lo, double hi, int k_bins) { return hsd_dequantize_bin(bin, lo, hi, k_bins); }

/* Windowed finite-difference kinematics (diagnostics beside R/D/F): mean
 * |v|, |a|, |j| per step, v_i = P_{i+1} - P_i, a_i = v_{i+1} - v_i, j_i = a_{i+1} - a_i. */
void hsdo_window_derivatives(const double* xyz, int n, double* out3) {
  double sv = 0, sa = 0, sj = 0;
  for (int i = 0; i + 1 < n; ++i) {
    double v[3], a[3], j[3];
    for (int d = 0; d < 3; ++d) v[d] = xyz[(i + 1) * 3 + d] - xyz[i * 3 + d];
    sv += sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (i + 2 < n) {
      for (int d = 0; d < 3; ++d) {
        double v1 = xyz[(i + 2) * 3 + d] - xyz[(i + 1) * 3 + d];
        a[d] = v1 - v[d];
      }
      sa += sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
      if (i + 3 < n) {
        for (int d = 0; d < 3; ++d) {
          double v1 = xyz[(i + 2) * 3 + d] - xyz[(i + 1) * 3 + d];
          double v2 = xyz[(i + 3) * 3 + d] - xyz[(i + 2) * 3 + d];
          j[d] = (v2 - v1) - a[d];
        }
        sj += sqrt(j[0] * j[0] + j[1] * j[1] + j[2] * j[2]);
      }
    }
  }
  out3[0] = n > 1 ? sv / (double)(n - 1) : 0.0;
  out3[1] = n > 2 ? sa / (double)(n - 2) : 0.0;
  out3[2] = n > 3 ? sj / (double)(n - 3) : 0.0;
}
