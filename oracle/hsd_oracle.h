/*
 * hsd_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference's algorithms on the HeiSD
 * retrieval-side hot path, used ONLY by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg as the checker.  The product
 * (libhsd_gpu.so) never links, loads or calls anything in this directory.
 *
 * Parity anchors:
 *   - search / quantize are pinned against the reference itself, compiled from
 *     /root/reference/proj/src/{store,actions,hnsw}.cpp into oracle/_ref/
 *     (oracle/Makefile) and driven through oracle/ref_shim.cpp;
 *   - verification / drafting / decide_sd are spec-only in the reference
 *      and are pinned by every SPEC golden vector
 *     (tests/test_oracle_golden.py);
 *   - kinematics.cpp needs Eigen, which is not vendored (proj/.gitignore:2), so
 *     it is restated Eigen-free and pinned by the SPEC/PAPER fixtures at the
 *     reference's stated tolerances.
 */
#ifndef HSD_ORACLE_H
#define HSD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror errors.hpp:10-50 (and include/hsd/hsd_gpu.h) */
enum { HSDO_OK = 0, HSDO_INVALID_INPUT = 1, HSDO_CONFIG = 2, HSDO_SCHEMA = 3, HSDO_CALIBRATION = 7 };

/* ---------------------------------------------------------------- retrieval */
/* cosine_similarity, store.cpp:29-34: sequential fp64 sum of a[i]*b[i]. */
double hsdo_dot_f32(const float* a, const float* b, int dim);

/* Collection::search_topk_exact, store.cpp:59-73, over fp32 keys widened to
 * fp64.  Returns the hit count min(k, n) or -HSDO_INVALID_INPUT when k < 1. */
int hsdo_search_topk_exact(const float* keys, int64_t n, int dim, const float* query, int k, double* scores,
                           int64_t* ids);

/* Same contract over a counter-generated DB (include/hsd/hsd_synth.h) that is
 * never materialised: every row is generated once and scored against all B
 * queries.  `threads` <= 0 uses all cores.  Results are independent of the
 * thread count. */
int hsdo_search_synth(int kind, uint64_t db_seed, int64_t n, int dim, const float* queries, int B, int k,
                      double* scores, int64_t* ids, int threads);

/* Key-storage flag OR-ed into `kind` of hsdo_search_synth / hsdo_gen_keys:
 * the DB stores bf16 keys (RN-even rounding of the fp32 synthetic key), as a
 * bf16 collection does (include/hsd/hsd_synth.h hsd_bf16_bits). */
#define HSDO_KEYS_BF16 0x100

/* Generate rows [row0, row0+n) of a synthetic DB / a query batch (fp32). */
void hsdo_gen_keys(int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim, float* out);
void hsdo_gen_queries(int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B, int dim,
                      float* out);

/* Verifier features (f_now, f_prev) of episodes [e0, e0+E) and logits
 * [E][L][256] whose greedy bins track the draft tokens of DB row rows[e]
 * (-1 = random draft), as generated on the device (hsd_synth.h). */
void hsdo_gen_features(uint64_t seed, int64_t e0, int E, int d_f, float* now, float* prev);
void hsdo_gen_logits(uint64_t db_seed, uint64_t seed, const int64_t* rows, int64_t e0, int E, int L, float* out);

/* ------------------------------------------------------------------ actions */
/* quantize, actions.cpp:32-50 (uniform bounds lo/hi on all 7 dims).  Returns
 * 0, or -HSDO_CONFIG / -HSDO_INVALID_INPUT. */
int hsdo_quantize(const double* a7, const double* lo7, const double* hi7, int k_bins, int* bins7);
/* Payload tokens of synthetic record `row`: quantize(next_actions[s]) for
 * s = 0..2 with bounds [-1, 1], K = 256 -> 21 bins. */
void hsdo_synth_tokens(uint64_t db_seed, int64_t row, uint8_t* tok21);

/* ------------------------------------------------------------- verification */
typedef struct {
  int enabled;        /* relaxed acceptance on */
  int bias_seq_max;   /* 30 (PAPER §4.2) */
  int bias_token_max; /* 15 */
} hsdo_accept_params;

typedef struct {
  double T;
  double min_S;
  int O_dist;
  double delta;
  int inverted; /* update_direction = inverted */
} hsdo_skip_state;

int hsdo_token_bias(int draft_bin, int verify_bin);
/* accept_sequence.  is_gripper selects zero tolerance. */
int hsdo_accept_sequence(const int* draft, const int* verify, int n, int is_gripper, const hsdo_accept_params* p);
/* argmax over `nbins` logits, lowest index on ties (Eq. 2-1). */
int hsdo_argmax(const float* logits, int nbins);

/* Exactly-rounded (double-double) dot of two fp32 feature vectors. */
double hsdo_feature_cos(const float* a, const float* b, int dim);
/* should_skip, SPEC.md:458-466 (history = number of stored features). */
int hsdo_should_skip(double cos_now_prev, const hsdo_skip_state* s, int gap_d, int history);

typedef struct {
  int accept_len;    /* accepted draft tokens (excludes the fallback token) */
  int win_a;         /* winning chain: pos0 from candidate a ... */
  int win_b;         /* ... everything after pos0 from candidate b */
  int fallback;      /* empty prefix -> 1 greedy verifier token */
  int calls;         /* verifier_calls (unique chains visited) */
  int skipped;       /* verify-skip fired: whole rank-0 draft emitted */
  int n_emit;        /* tokens emitted */
  int tokens[64];    /* emitted tokens */
} hsdo_outcome;

/* One retrieval-mode decode round for one episode (CS-1):
 *   drafts   : n_cand x L tokens (rank order, L = 7 or 21)
 *   greedy   : L verifier greedy tokens (teacher-forced, context-free)
 *   skip     : result of should_skip for this step
 * chains = (a, b) label assignments, enumerated in DFS /
 * lexicographic order, duplicates (identical token sequences) dropped, capped
 * at `cap`.  Longest accepted prefix wins, earliest chain on ties. */
void hsdo_verify_round(const int* drafts, int n_cand, int L, const int* greedy, int skip, int cap,
                       const hsdo_accept_params* p, hsdo_outcome* out);

/* Brute-force DFS enumerator used to pin the fast path above. */
void hsdo_verify_round_chains(const int* drafts, int n_cand, int L, const int* chain_greedy /* cap x L */,
                              int greedy_ctx, int skip, int cap, const hsdo_accept_params* p, hsdo_outcome* out);
int hsdo_enumerate_chains(const int* drafts, int n_cand, int L, int cap, int* chains_out /* cap x L */,
                          int* a_out, int* b_out);

/* offline_calibrate_skip, SPEC.md:449-457 over a cosine matrix per trajectory.
 * sims: n x n similarity matrix (row-major) of one trajectory; returns 0 and
 * (min_S, O_dist) or -HSDO_CALIBRATION.  Multiple trajectories: call
 * hsdo_calibrate_accumulate then hsdo_calibrate_finish. */
typedef struct {
  double min_S;
  int O_dist;
  int found;
} hsdo_calib;
void hsdo_calibrate_init(hsdo_calib* c);
void hsdo_calibrate_accumulate(hsdo_calib* c, const double* sims, int n, double T);
int hsdo_calibrate_finish(const hsdo_calib* c, double* min_S, int* O_dist);
/* update_skip_state */
void hsdo_update_skip_state(hsdo_skip_state* s, int success, double S_c, double min_S_h);

/* --------------------------------------------------------------- kinematics */
typedef struct {
  double alpha;
  int w;
  double threshold;
  double r_cap;
} hsdo_metric_params;

typedef struct {
  double d_min, d_max95, r_min, r_max95;
} hsdo_norm_bounds;

/* project_window, kinematics.cpp:38-76. xyz: n x 3; uv: n x 2 */
int hsdo_project_window(const double* xyz, int n, double* uv);
/* fit_circle_center, kinematics.cpp:107-207 */
int hsdo_fit_circle_center(const double* uv, int n, double* cu, double* cv, int* degenerate, int* iterations);
/* curvature_radius, kinematics.cpp:209-218 */
int hsdo_curvature_radius(const double* xyz, int n, double r_cap, double* R);
/* cumulative_displacement, kinematics.cpp:220-230 */
int hsdo_cumulative_displacement(const double* xyz, int n, double* D);
double hsdo_normalize(double x, double lo, double hi95);                                /* :232-236 */
int hsdo_percentile_bounds(const double* samples, int n, double* lo, double* p95);      /* :238-247 */
double hsdo_fused_metric(double R, double D, const hsdo_metric_params* p, const hsdo_norm_bounds* b); /* :249-255 */
int hsdo_classify(double F, double threshold); /* :257-259; 1 = retrieval_sd, 0 = drafter_sd */
/* window_features, kinematics.cpp:261-273; decision = decide_sd
 * with history >= w. */
int hsdo_window_features(const double* xyz, int n, const hsdo_metric_params* p, const hsdo_norm_bounds* b, double* R,
                         double* D, double* F, int* decision);

/* Windowed finite-difference kinematics: mean |v|, |a|, |j| per step (out3). */
void hsdo_window_derivatives(const double* xyz, int n, double* out3);

/* ------------------------------------------------------- hybrid loop (config 5)
 * run_step / run_episode of the SPEC scheduler for R robots,
 * sequentially, over the counter-based harness of hsd_synth.h (demonstration
 * policy rows, robots, toy drafter, ToyEnv).  Restates the device loop
 * (k_hybrid.cu + api.cu hsd_hybrid_step) for parity; the record layouts are
 * those of include/hsd/hsd_gpu.h. */
typedef struct {
  int robots, k, mode, traj_T, drafter_p_pct, drafter_L, gap_d, d_f;
  uint64_t seed, db_seed;
  int key_kind;  /* may carry HSDO_KEYS_BF16 */
  int relaxed, bias_seq_max, bias_token_max, skip_enabled, O_dist, chain_cap;
  double min_S;
  hsdo_metric_params metric;
  hsdo_norm_bounds bounds;
  double cost_verifier, cost_drafter_token, cost_retrieval;
} hsdo_hybrid_params;

typedef struct {
  float F;
  int16_t accept_len, verifier_calls, n_emit;
  int8_t mode, skipped;
  float cost;
} hsdo_step_record;

typedef struct {
  int64_t rounds, tokens, accepted, verifier_calls;
  double cost;
  int32_t n_retrieval, n_drafter, n_skipped, n_fallback;
} hsdo_episode_report;

/* DB: n_rows synthetic rows of family key_kind (dim) with TRAJ payloads.
 * Outputs: trace [rounds][R] (or NULL), pos [R][3], reports [R]. */
/* Demonstration policy token (hsd_synth.h hsd_policy_token). */
int hsdo_policy_token(uint64_t db_seed, int64_t e, int64_t j, int d);
int hsdo_robot_greedy(uint64_t db_seed, uint64_t seed, int64_t r, int64_t n_demo, int64_t j, int d);
double hsdo_robot_start(uint64_t seed, int64_t r, int d);
/* dequantize of one bin, actions.cpp:52-66 */
double hsdo_dequantize_bin(int bin, double lo, double hi, int k_bins);
int hsdo_hybrid_run(const hsdo_hybrid_params* p, int64_t n_rows, int dim, int rounds, hsdo_step_record* trace,
                    double* pos, hsdo_episode_report* reports);

#ifdef __cplusplus
}
#endif
#endif
