/*
 * hsd_gpu.h — C ABI of the B200-native HeiSD retrieval-side hot path.
 *
 * Drop-in boundary for the reference's C++ API in proj/include/hsd (see
 * INTEGRATION.md for the reference-side binding and include/hsd/gpu.hpp for
 * the header-only C++ wrapper that re-exposes the reference signatures).
 *
 *   hot-path step (CS-5):
 *     hsd_window_features  -> drafter/retrieval decision per robot  (K5)
 *     hsd_search_topk_exact-> top-k records per query                (K1+K2)
 *     hsd_verify_round     -> gather + verify-skip + relaxed accept  (K4)
 *     hsd_step             -> all of the above on one stream
 *
 * Conventions
 *   - Plain pointers and sizes; no C++ or torch types.  Unless stated
 *     otherwise array arguments are DEVICE pointers on the collection's GPU and
 *     work is enqueued asynchronously on `stream` (a cudaStream_t, NULL = the
 *     legacy default stream).
 *   - Every call returns an hsd_status; the status codes mirror the
 *     reference's exception taxonomy (errors.hpp:10-50) so the C++ wrapper can
 *     rethrow the matching hsd:: exception.  hsd_last_error() returns a
 *     thread-local message for the last failing call on this thread.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point returns HSD_ERR_NO_DEVICE.
 */
#ifndef HSD_GPU_H
#define HSD_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSD_ABI_VERSION 1
#define HSD_K_MAX 32        /* largest k served by the device top-k */
#define HSD_TOKENS_STRIDE 32 /* bytes per record in the device token table (21 used) */

typedef enum hsd_status {
  HSD_OK = 0,
  HSD_ERR_INVALID_INPUT = 1, /* hsd::InvalidInputError (errors.hpp:15) */
  HSD_ERR_CONFIG = 2,        /* hsd::ConfigError       (errors.hpp:20) */
  HSD_ERR_SCHEMA = 3,        /* hsd::SchemaError       (errors.hpp:25) */
  HSD_ERR_IO = 4,            /* hsd::IoError           (errors.hpp:30) */
  HSD_ERR_PARSE = 5,         /* hsd::ParseError        (errors.hpp:35) */
  HSD_ERR_VERSION = 6,       /* hsd::VersionError      (errors.hpp:43) */
  HSD_ERR_CALIBRATION = 7,   /* hsd::CalibrationError  (errors.hpp:48) */
  HSD_ERR_CUDA = 100,
  HSD_ERR_NCCL = 101,
  HSD_ERR_OOM = 102,
  HSD_ERR_NO_DEVICE = 103,
} hsd_status;

/* Key storage type of a collection. */
typedef enum hsd_dtype {
  HSD_DTYPE_F32 = 0,  /* fp32 keys (the reference's fp64 embeddings rounded once to fp32) */
  HSD_DTYPE_BF16 = 1, /* bf16 keys (RN-even from fp32): half the HBM bytes per scan */
} hsd_dtype;

const char* hsd_last_error(void);
/* 1-based line of the last HSD_ERR_PARSE from a file reader (hsd::ParseError
 * line_number, errors.hpp:35-40); 0 when not applicable. */
long hsd_last_error_line(void);
int hsd_abi_version(void);
/* Number of visible sm_100 devices (0 when none). */
hsd_status hsd_device_count(int* n);

/* ------------------------------------------------------------------------
 * Collection — one task shard of the trajectory DB resident in HBM.
 * Replaces hsd::Collection (store.hpp:59-96): same dim rule (store.cpp:36-38),
 * dense ids in insertion order (store.cpp:53), insert-time schema checks
 * (store.cpp:44-57).  Keys are stored fp32 row-major [capacity][dim]; payload
 * next_actions are quantized at insert (actions.cpp:32-50, bounds [-1,1],
 * K = 256) into a uint8 token table [capacity][32] (21 used: 3 slices x 7).
 * ---------------------------------------------------------------------- */
typedef struct hsd_collection hsd_collection;

hsd_status hsd_collection_create(int device, int dim, int64_t capacity, hsd_collection** out);
/* Same with an explicit key storage type (hsd_dtype).  bf16 collections round
 * keys once to bf16 (RN-even) at insert/generate; searches over them are exact
 * (bit-identical to the reference's fp64 dot) with respect to the STORED bf16
 * keys, and their recall against an fp32 DB is what the bf16 mode reports.
 * bf16 needs dim % 8 == 0 -> HSD_ERR_CONFIG otherwise. */
hsd_status hsd_collection_create_ex(int device, int dim, int64_t capacity, int dtype, hsd_collection** out);
hsd_status hsd_collection_destroy(hsd_collection* c);
hsd_status hsd_collection_size(const hsd_collection* c, int64_t* n);
hsd_status hsd_collection_dim(const hsd_collection* c, int* dim);
hsd_status hsd_collection_device(const hsd_collection* c, int* device);
/* Device pointers of the resident arrays (read-only views); the fp32 key view
 * fails with HSD_ERR_INVALID_INPUT on a bf16 collection. */
hsd_status hsd_collection_keys(const hsd_collection* c, const float** keys, const uint8_t** tokens);
hsd_status hsd_collection_dtype(const hsd_collection* c, int* dtype);

/* Filter mode of an fp32 collection.  HSD_FILTER_BF16_COPY keeps a bf16 copy
 * of the keys resident (+50% HBM) that the tensor-core filter streams at half
 * the bytes per scan; the exact fp64 rescoring still reads the fp32 keys, so
 * ids and scores stay bit-identical to the reference (the filter margin widens
 * to the bf16 x bf16 error bound).  Kept current by insert / generate. */
enum { HSD_FILTER_NATIVE = 0, HSD_FILTER_BF16_COPY = 1 };
hsd_status hsd_collection_set_filter(hsd_collection* c, int filter);
hsd_status hsd_collection_get_filter(const hsd_collection* c, int* filter);
/* Untyped key view (fp32 or bf16 bits per hsd_collection_dtype). */
hsd_status hsd_collection_data(const hsd_collection* c, const void** keys, const uint8_t** tokens);

/* Collection::insert (store.cpp:44-57) of n records.  HOST pointers:
 *   emb          fp32 [n][dim]
 *   next_actions fp64 [n][3][7]  (Payload::next_actions, store.hpp:31)
 *   episode_idx, step_idx int32 [n] or NULL (0); negative -> HSD_ERR_SCHEMA.
 * Non-finite actions -> HSD_ERR_INVALID_INPUT (actions.cpp:38-40).
 * *first_id receives the id of the first inserted record.  Synchronous. */
hsd_status hsd_collection_insert(hsd_collection* c, const float* emb, const double* next_actions,
                                 const int32_t* episode_idx, const int32_t* step_idx, int64_t n, int64_t* first_id);

/* Record::feature (store.hpp:40-42) of records [row0, row0 + n): fp32 HOST
 * [n][d_f], has uint8 [n] (NULL = all present; absent rows stay zero).  The
 * first call fixes d_f; another length -> HSD_ERR_SCHEMA.  Synchronous.  The
 * device table feeds hsd_calibrate_skip (offline Alg. 1) directly. */
hsd_status hsd_collection_set_features(hsd_collection* c, int64_t row0, int64_t n, int d_f, const float* feat,
                                       const uint8_t* has);
/* Device view of the feature table: fp32 [capacity][d_f], presence [capacity]
 * (NULL / d_f = 0 when no record carries a feature). */
hsd_status hsd_collection_features(const hsd_collection* c, const float** feat, const uint8_t** has, int* d_f);

/* Append n counter-generated records (include/hsd/hsd_synth.h, family
 * `kind`) generated on the device; synchronous.  Record i of the collection
 * holds synthetic row i. */
hsd_status hsd_collection_generate(hsd_collection* c, int kind, uint64_t db_seed, int64_t n);
/* Same, appending synthetic rows [row0, row0 + n) of the global stream (the
 * local shard of a row-sharded DB; local id j holds global row row0 + j). */
hsd_status hsd_collection_generate_rows(hsd_collection* c, int kind, uint64_t db_seed, int64_t row0, int64_t n);

/* ------------------------------------------------------------------------
 * Exact top-k search — Collection::search_topk_exact (store.cpp:59-73) for a
 * batch of B fp32 queries [B][dim].  Outputs [B][k]: fp64 scores and int32
 * record ids, ordered (score desc, id asc); when k > size the trailing
 * entries are id -1 / score -inf.  Scores are the reference's sequential fp64
 * dot product of the (fp32-widened) query and key, bit for bit.
 * k < 1 -> HSD_ERR_INVALID_INPUT (store.cpp:60).  k > HSD_K_MAX is served
 * by a separate exact path (every row's score, then a stable radix sort per
 * query; stream-ordered scratch of ~24 bytes per row) and needs dim <= ~17000.
 * An empty collection yields all -1 (no error).
 * `queries` is a device pointer, 16-byte aligned (HSD_ERR_INVALID_INPUT
 * otherwise; rows are dim * 4 bytes apart with dim % 4 == 0).
 * ---------------------------------------------------------------------- */
hsd_status hsd_search_topk_exact(hsd_collection* c, const float* queries, int B, int k, double* scores,
                                 int32_t* ids, void* stream);

/* Same, restricted to the record range [row_begin, row_end) (a per-task
 * shard inside one device array); ids stay collection-global. */
hsd_status hsd_search_topk_range(hsd_collection* c, const float* queries, int B, int k, int64_t row_begin,
                                 int64_t row_end, double* scores, int32_t* ids, void* stream);

/* Search statistics of `stream`, accumulated since the last reset:
 *   stats3[0] queries that needed the exact range fallback (a filter list
 *             could not bound its rows: runs of near-duplicate records);
 *   stats3[1] pooled candidates rescored exactly;
 *   stats3[2] filter lists rescanned by the fallback.
 * Results are exact either way; the fallback only costs time.  Synchronizes
 * `stream`; reset != 0 zeroes the counters afterwards. */
hsd_status hsd_search_stats(hsd_collection* c, void* stream, int reset, int* stats3);
/* stats3[0] of hsd_search_stats (kept for ABI version 1 callers). */
hsd_status hsd_search_overflow_count(hsd_collection* c, void* stream, int* count);

/* Diagnostics: the tcgen05 filter's approximate scores of B <= 256 queries
 * against every record, fp32 [B][size] (device); variant 1 = the stored keys
 * (TF32 over fp32 keys, bf16 over bf16 keys), 4 = the bf16 filter copy of an
 * fp32 collection.  Used by the tests to check the error bounds the exact
 * rescoring relies on. */
hsd_status hsd_debug_sim_scores(hsd_collection* c, const float* queries, int B, int variant, float* out,
                                void* stream);
/* Search path switch, process-wide: 0 auto (exact scan of every row when the
 * cost model prefers it — small rows x batch, B <= 4 — else the tensor-core
 * filter + exact rescoring, CTA-pair kernels above 128 queries), 1 filter with
 * single-CTA wide kernels only (also HSD_WIDE_PAIR=0), 2 filter + rescoring
 * only, 3 exact scan wherever it applies (B <= 4, k <= 32).  Every path
 * returns the same bits. */
/* Diagnostics: returns and clears the CUDA runtime's pending (non-sticky)
 * error of the calling thread — the tests check that no entry point, destroy
 * included, leaves one behind. */
int hsd_debug_last_cuda_error(void);
hsd_status hsd_set_sim_path(int path);
/* The path a search of B queries (top-k) over `rows` rows (-1: the whole
 * collection) takes under the current switch: *exact_scan = 1 for the exact
 * scan (K1x), 0 for the tensor-core filter + exact rescoring (K1 + K2), 2 for
 * the same filter whose fp32 key tiles are converted to bf16 on chip (CTA
 * pairs, 129..1024 queries over fp32 keys without the bf16 filter copy). */
hsd_status hsd_search_plan(hsd_collection* c, int B, int k, int64_t rows, int* exact_scan);

/* ------------------------------------------------------------------------
 * Approximate index — the device stand-in for the reference's HNSW index:
 * Collection::build_hnsw(HnswParams) (store.cpp:75-80, hnsw.cpp:58-169) and
 * the index branch of Collection::search_topk (store.cpp:82-92).
 *
 * An inverted file (IVF-flat): nlist unit-norm centroids (spherical k-means,
 * n_iter Lloyd iterations whose assignment is the collection's own exact
 * search; deterministic), each record in the list of its best centroid
 * (score desc, id asc), the lists read in place from the keys.  A search
 * scores every centroid, scans the rows of the nprobe best lists, keeps the
 * 32 best candidates by their fp32-accumulated scores (over the stored keys,
 * or the bf16 filter copy when the collection keeps one) and returns
 * the top k of those by the EXACT score: every returned score is the
 * reference's cosine_similarity of the returned id (store.cpp:86-90), ranked
 * (score desc, id asc).  Recall against search_topk_exact is reported by the
 * tests and the bench, not guaranteed.
 *
 * hsd_index_build: empty collection -> HSD_ERR_INVALID_INPUT ("cannot index
 * an empty collection", store.cpp:76); nlist is clamped to the row count.
 * The index holds the collection (which must outlive it); a later insert or
 * generate makes it stale, and a stale index searches exactly (the reference
 * drops the index on insert and search_topk falls back to the exact scan).
 * ---------------------------------------------------------------------- */
typedef struct hsd_ivf_params {
  int nlist;  /* inverted lists, 1..16384 (clamped to the row count) */
  int n_iter; /* Lloyd iterations after the strided seeds, 0..1000 */
} hsd_ivf_params;
typedef struct hsd_index hsd_index;
hsd_status hsd_index_build(hsd_collection* c, const hsd_ivf_params* params, hsd_index** out);
hsd_status hsd_index_destroy(hsd_index* x);
/* nlist, indexed rows, longest list, stale (1 when the collection changed) */
hsd_status hsd_index_info(const hsd_index* x, int* nlist, int64_t* n_rows, int* max_list, int* stale);
/* Host copies (any may be NULL): offs [nlist + 1], perm [n_rows] (list
 * order -> record id, ascending within each list), centroids fp32 [nlist][dim]. */
hsd_status hsd_index_lists(const hsd_index* x, int32_t* offs, int32_t* perm, float* centroids);
/* Approximate top-k of B queries (device, 16-byte aligned) over the nprobe
 * (1..32, clamped to nlist) best lists; scores / ids as
 * hsd_search_topk_exact (-inf / -1 past the candidates found).  probes
 * (device [B][nprobe], optional) receives the probed list ids.  k >
 * HSD_K_MAX answers with the exact top-k (probes untouched). */
hsd_status hsd_search_topk_index(hsd_index* x, const float* queries, int B, int k, int nprobe, double* scores,
                                 int32_t* ids, int32_t* probes, void* stream);

/* ------------------------------------------------------------------------
 * Verification — fused gather + verify-skip + sequence-wise relaxed
 * acceptance + accepted length (spec-only in the reference).
 * ---------------------------------------------------------------------- */
typedef struct hsd_verify_params {
  int32_t relaxed;        /* RelaxedAcceptanceParams::enabled */
  int32_t bias_seq_max;   /* 30 (PAPER §4.2) */
  int32_t bias_token_max; /* 15 */
  int32_t skip_enabled;   /* verify-skip on (Alg. 1, retrieval mode only) */
  double min_S;           /* VerifySkipState::min_S */
  int32_t O_dist;         /* VerifySkipState::O_dist */
  int32_t chain_cap;      /* enumerate_chains cap (default 64) */
} hsd_verify_params;

typedef struct hsd_outcome {
  int32_t accept_len; /* accepted draft tokens (VerifyOutcome::accept_length) */
  int16_t win_a;      /* winning chain: pos0 from candidate rank a ...        */
  int16_t win_b;      /* ... every later group from candidate rank b          */
  int16_t calls;      /* verifier_calls (unique chains visited)               */
  int8_t fallback;    /* empty prefix -> one greedy verifier token            */
  int8_t skipped;     /* verify-skip fired                                    */
  int16_t n_emit;     /* tokens emitted                                       */
  int16_t greedy0;    /* verifier greedy token at position 0                  */
  float cos_sim;      /* skip-check similarity (diagnostic; -2 when not run)  */
} hsd_outcome;

/* One decode round for E episodes:
 *   ids       int32 [E][k] retrieved record ids (rank order; -1 = none)
 *   logits    fp32 [E][L][256] verifier logits (teacher-forced greedy = argmax,
 *             lowest bin on ties), L in {7, 21} (1 or 3 action slices)
 *   feat_now, feat_prev fp32 [E][d_f] verifier features (may be NULL when no
 *             parameter set enables skipping)
 *   history   int32 [E] number of stored features (NULL = unbounded)
 *   gap_d     candidate step gap d of should_skip
 *   params    HOST array of P parameter sets (a tolerance / threshold sweep
 *             reads the inputs once)
 * Outputs (device): out [P][E] outcomes, tokens [P][E][L] emitted tokens. */
hsd_status hsd_verify_round(hsd_collection* c, const int32_t* ids, int E, int k, int L, const float* logits,
                            const float* feat_now, const float* feat_prev, int d_f, const int32_t* history, int gap_d,
                            const hsd_verify_params* params, int P, hsd_outcome* out, uint8_t* tokens, void* stream);

/* Same over pre-gathered draft records (drafts uint8 [E][k][32], e.g. from
 * hsd_search_topk_sharded); ids only mark valid candidates (-1 = none). */
hsd_status hsd_verify_round_drafts(int device, const int32_t* ids, const uint8_t* drafts, int E, int k, int L,
                                   const float* logits, const float* feat_now, const float* feat_prev, int d_f,
                                   const int32_t* history, int gap_d, const hsd_verify_params* params, int P,
                                   hsd_outcome* out, uint8_t* tokens, void* stream);

/* ------------------------------------------------------------------------
 * verify_tree with a real verifier: VerifierModel::verify_chain returns, per
 * chain, greedy tokens TEACHER-FORCED on that chain (models.hpp:34-37), so
 * every chain has its own greedy tokens.  Two calls:
 *
 * 1. hsd_enumerate_chains: the chains verify_tree visits (
 *    unique token sequences "pos0 of candidate a + later groups
 *    of candidate b" in DFS = lexicographic (a, b) order, at most `cap`).
 *    Outputs (device): n_chains int32 [E]; chain_ab int16 [E][cap][2] (a, b);
 *    chain_tokens uint8 [E][cap][L] — the inputs of the caller's verifier.
 * 2. hsd_verify_round_chains: the verifier's output for those chains, either
 *    chain_greedy uint8 [E][cap][L] (verify_chain's tokens) or chain_logits
 *    fp32 [E][cap][L][256] (greedy = std::max_element over the bins), plus
 *    greedy_ctx int32 [E] = greedy_next(context) (models.hpp:38-39), the token
 *    emitted on fallback / for an empty shard.  Verify-skip as in
 *    hsd_verify_round; one parameter set (its chain_cap must equal `cap`).
 *    Outputs: out [E] and tokens [E][L] as hsd_verify_round.
 * Candidates come from the collection's token table by id (c != NULL) or
 * from pre-gathered drafts uint8 [E][k][32] (then `device` names the GPU). */
hsd_status hsd_enumerate_chains(hsd_collection* c, int device, const int32_t* ids, const uint8_t* drafts, int E,
                                int k, int L, int cap, int32_t* n_chains, int16_t* chain_ab, uint8_t* chain_tokens,
                                void* stream);
hsd_status hsd_verify_round_chains(hsd_collection* c, int device, const int32_t* ids, const uint8_t* drafts, int E,
                                   int k, int L, int cap, const uint8_t* chain_greedy, const float* chain_logits,
                                   const int32_t* greedy_ctx, const float* feat_now, const float* feat_prev, int d_f,
                                   const int32_t* history, int gap_d, const hsd_verify_params* params,
                                   hsd_outcome* out, uint8_t* tokens, void* stream);

/* ------------------------------------------------------------------------
 * Kinematic fused metric — window_features + classify_segment + decide_sd
 * (kinematics.cpp:38-273) for W windows of w points.
 * ---------------------------------------------------------------------- */
typedef struct hsd_metric_params {
  double alpha;     /* FusedMetricParams (kinematics.hpp:38-45) */
  int32_t w;
  double threshold;
  double r_cap;
} hsd_metric_params;

typedef struct hsd_norm_bounds {
  double d_min, d_max95, r_min, r_max95; /* NormalizationBounds (kinematics.hpp:29-36) */
} hsd_norm_bounds;

/* xyz fp64 [W][w][3]; history int32 [W] (NULL = warm) -> R, D, F fp64 [W],
 * decision int32 [W]: 1 retrieval_sd, 0 drafter_sd (cold start history < w is
 * drafter), -1 non-finite window (InvalidInputError).  Params
 * are validated like FusedMetricParams/NormalizationBounds::validate
 * (kinematics.cpp:13-24) -> HSD_ERR_CONFIG. */
hsd_status hsd_window_features(int device, const double* xyz, int W, const hsd_metric_params* params,
                               const hsd_norm_bounds* bounds, const int32_t* history, double* R, double* D, double* F,
                               int32_t* decision, void* stream);

/* compute_percentile_bounds (kinematics.cpp:238-247): (min, nearest-rank
 * 95th percentile) of n > 0 DEVICE fp64 samples, returned to the HOST.
 * n < 1 or a non-finite sample -> HSD_ERR_INVALID_INPUT.  Synchronizes `stream`. */
hsd_status hsd_percentile_bounds(int device, const double* samples, int64_t n, double* min_out, double* p95_out,
                                 void* stream);
/* NormalizationBounds of a task suite (the norm-bounds computation, SPEC.md:205,
 * Appendix D): R and D of every window xyz fp64 [W][w][3] (device), then
 * (r_min, r_max95) and (d_min, d_max95) with hsd_percentile_bounds.  HOST
 * output.  Synchronizes `stream`. */
hsd_status hsd_norm_bounds_from_windows(int device, const double* xyz, int W, const hsd_metric_params* params,
                                        hsd_norm_bounds* out, void* stream);

/* Same, plus the windowed finite-difference kinematics of each window in the
 * same pass: vaj fp64 [W][3] (may be NULL) = mean |velocity|, mean
 * |acceleration|, mean |jerk| per action step (v_i = P_{i+1} - P_i,
 * a_i = v_{i+1} - v_i, j_i = a_{i+1} - a_i; 0 when the window is too short).
 * Diagnostics named by the north star; the reference's decision uses R/D/F. */
hsd_status hsd_window_features_ex(int device, const double* xyz, int W, const hsd_metric_params* params,
                                  const hsd_norm_bounds* bounds, const int32_t* history, double* R, double* D,
                                  double* F, int32_t* decision, double* vaj, void* stream);

/* quantize (actions.cpp:32-50) of n action slices fp64 [n][7] with per-dim
 * bounds lo7/hi7 (HOST) into int32 bins [n][7]; status[n] (int32, device):
 * 0 ok, 1 non-finite input.  Bad bounds / K < 2 -> HSD_ERR_CONFIG. */
hsd_status hsd_quantize(int device, const double* actions, int64_t n, const double* lo7, const double* hi7, int k_bins,
                        int32_t* bins, int32_t* status, void* stream);

/* ------------------------------------------------------------------------
 * Fused decode-round step (CS-5): kinematics + search -> verify, ordered on
 * `stream` (the kinematic metric runs on an engine-owned side stream forked
 * from and joined back into `stream`, overlapping the DB scan).  All episodes
 * are searched; decision[] reports the drafter/retrieval boundary.
 * ---------------------------------------------------------------------- */
typedef struct hsd_engine hsd_engine;

hsd_status hsd_engine_create(hsd_collection* c, int max_B, int k, int L, int d_f, int w, hsd_engine** out);
hsd_status hsd_engine_destroy(hsd_engine* e);

typedef struct hsd_step_io {
  /* inputs [B]-major; device pointers for hsd_step, host for hsd_step_host */
  const float* queries;   /* [B][dim] */
  const float* logits;    /* [B][L][256] */
  const float* feat_now;  /* [B][d_f] or NULL */
  const float* feat_prev; /* [B][d_f] or NULL */
  const double* xyz;      /* [B][w][3] or NULL (skip kinematics) */
  const int32_t* history; /* [B] or NULL */
  /* outputs */
  double* scores;         /* [B][k] */
  int32_t* ids;           /* [B][k] */
  hsd_outcome* out;       /* [B] */
  uint8_t* tokens;        /* [B][L] */
  double* R;              /* [B] or NULL */
  double* D;
  double* F;
  int32_t* decision;
} hsd_step_io;

hsd_status hsd_step(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                    const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream);
/* hsd_step replayed from a CUDA graph: the first call with a given (B, io
 * pointers, parameters, stream) runs eagerly and captures the round; later
 * identical calls launch the graph (one launch instead of ~10: for small,
 * launch-bound batches such as config 1's B = 1).  Needs a non-NULL stream. */
hsd_status hsd_step_graph(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                          const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream);
/* Stage timing of the next `max_steps` hsd_step calls with CUDA events on the
 * step's stream (0 disables).  hsd_engine_stage_times synchronizes and returns
 * the summed milliseconds of [kinematics, similarity, select, verify, total]
 * over the recorded steps, then resets the recorder. */
hsd_status hsd_engine_enable_timing(hsd_engine* e, int max_steps);
hsd_status hsd_engine_stage_times(hsd_engine* e, int* n_steps, double ms[5]);
/* Per recorded step of `e`: the times (ms) of its [start, after similarity,
 * after select, end] events relative to the first recorded start event of
 * `ref` (another engine on the same device, or e itself) — marks [n][4].
 * With steps of several engines interleaved this gives the similarity
 * kernel's completion-to-completion interval inside a timed region.  Call
 * before hsd_engine_stage_times (which resets the recorder); synchronizes. */
hsd_status hsd_engine_stage_marks(hsd_engine* e, const hsd_engine* ref, int max_n, double* marks, int* n);
/* The engine's search statistics (as hsd_search_stats; the engine owns its
 * scratch).  Synchronizes the device. */
hsd_status hsd_engine_stats(hsd_engine* e, int reset, int* stats3);

/* Same with HOST buffers: H2D of the inputs and D2H of the outputs happen
 * inside the call (device staging owned by the engine); synchronous. */
hsd_status hsd_step_host(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                         const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream);
/* Asynchronous hsd_step_host: enqueue and return.  Two steps may be in flight
 * (double-buffered device staging): the uploads of step i+1 and the downloads
 * of step i-1 run on engine copy streams under step i's kernels.  Host buffers
 * should be pinned, must stay valid and unmodified until hsd_engine_sync, and
 * the outputs are complete after it returns. */
hsd_status hsd_step_host_async(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                               const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream);
hsd_status hsd_engine_sync(hsd_engine* e);

/* ------------------------------------------------------------------------
 * Multi-GPU: row-sharded collection (rank r owns a contiguous id range) with a
 * per-rank local top-k, an NCCL all-gather of the B x k records over NVLink
 * and a k-way merge; bit-identical to the single-GPU result.
 * ---------------------------------------------------------------------- */
typedef struct hsd_comm hsd_comm;
#define HSD_UNIQUE_ID_BYTES 128
hsd_status hsd_comm_unique_id(uint8_t id[HSD_UNIQUE_ID_BYTES]);
hsd_status hsd_comm_create(const uint8_t id[HSD_UNIQUE_ID_BYTES], int world, int rank, int device, hsd_comm** out);
hsd_status hsd_comm_destroy(hsd_comm* comm);
/* Contiguous shard [begin, end) of n_total rows for `rank` of `world`. */
hsd_status hsd_shard_range(int64_t n_total, int world, int rank, int64_t* begin, int64_t* end);
/* Local search of this rank's collection (ids offset by id_offset) followed by
 * the all-gather + merge; every rank receives the global [B][k] result and,
 * when `drafts` is non-null, the matching payload tokens [B][k][32] (the
 * records' drafts travel with them, so verification needs no remote lookup). */
hsd_status hsd_search_topk_sharded(hsd_collection* c, hsd_comm* comm, int64_t id_offset, const float* queries, int B,
                                   int k, double* scores, int32_t* ids, uint8_t* drafts, void* stream);
/* Same; reserve_sms SMs are left to work running concurrently on another
 * stream (e.g. the kinematic metric of the rank's episodes). */
hsd_status hsd_search_topk_sharded_ex(hsd_collection* c, hsd_comm* comm, int64_t id_offset, const float* queries,
                                      int B, int k, double* scores, int32_t* ids, uint8_t* drafts, int reserve_sms,
                                      void* stream);

/* Peer-memory exchange instead of the NCCL all-gather: every rank exports the
 * CUDA IPC handle of its receive window (sized for up to max_B queries and
 * k_max), the caller all-gathers the world x HSD_IPC_HANDLE_BYTES handles (any
 * transport) and imports them.  hsd_search_topk_sharded then publishes each
 * rank's B x k records straight into every peer's window (stores over
 * NVLink / NVSwitch + a system-scope release flag per epoch) and merges once
 * all G flags of its own window arrived — results identical to the NCCL
 * path.  A peer that never publishes is reported by hsd_comm_p2p_status
 * (bounded wait, no hang). */
#define HSD_IPC_HANDLE_BYTES 64
/* A communicator for the peer-memory exchange only (no NCCL communicator). */
hsd_status hsd_comm_create_p2p(int world, int rank, int device, hsd_comm** out);
hsd_status hsd_comm_p2p_export(hsd_comm* comm, int max_B, int k_max, uint8_t handle[HSD_IPC_HANDLE_BYTES]);
hsd_status hsd_comm_p2p_import(hsd_comm* comm, const uint8_t* handles /* [world][HSD_IPC_HANDLE_BYTES] */);
hsd_status hsd_comm_p2p_status(hsd_comm* comm, int* peer_timeout);

/* K3 merge on the device: G per-shard exact top-k lists (g_scores fp64 /
 * g_ids int32 [G][B][k], ids already global; optional g_drafts uint8
 * [G][B][k][32]) -> the global [B][k] in (score desc, id asc) order.  Used by
 * hsd_search_topk_sharded after the all-gather, and directly for task shards
 * searched separately on one GPU. */
hsd_status hsd_merge_topk(int device, const double* g_scores, const int32_t* g_ids, const uint8_t* g_drafts, int G,
                          int B, int k, double* scores, int32_t* ids, uint8_t* drafts, void* stream);

/* ------------------------------------------------------------------------
 * DB ingest: load_collection (store.cpp:152-191) of the
 * reference's JSONL v1 file, parsed natively (strict JSON, multi-threaded by
 * line) into a host columnar image, then uploaded like hsd_collection_insert.
 * Errors follow store.cpp: HSD_ERR_IO (cannot open), HSD_ERR_PARSE with
 * hsd_last_error_line() (missing / malformed header, no integer version,
 * metric != "cosine", malformed record, missing or mis-sized embedding,
 * missing payload, bad payload fields, negative indices), HSD_ERR_VERSION
 * (version != 1), HSD_ERR_CONFIG (dim < 1).  Additions: features of one file
 * must share one length (HSD_ERR_SCHEMA with the line).
 * ---------------------------------------------------------------------- */
typedef struct hsd_jsonl_db hsd_jsonl_db;
/* Host-only (no device needed).  threads <= 0: all cores. */
hsd_status hsd_jsonl_read(const char* path, int threads, hsd_jsonl_db** out);
hsd_status hsd_jsonl_free(hsd_jsonl_db* db);
hsd_status hsd_jsonl_info(const hsd_jsonl_db* db, int64_t* n, int* dim, int* d_f, const char** name);
/* Host views: emb fp32 [n][dim] (fp32 rounding of the file's doubles),
 * next_actions fp64 [n][21], episode/step idx int32 [n], features fp32
 * [n][d_f] (NULL when no record has one; zeros where absent), has_feature [n]. */
hsd_status hsd_jsonl_data(const hsd_jsonl_db* db, const float** emb, const double** next_actions,
                          const int32_t** episode_idx, const int32_t** step_idx, const float** features,
                          const uint8_t** has_feature);
hsd_status hsd_collection_from_jsonl(const hsd_jsonl_db* db, int device, int dtype, hsd_collection** out);
hsd_status hsd_collection_load_jsonl(const char* path, int device, int dtype, hsd_collection** out);
/* Binary columnar device image (keys as stored, quantized tokens, max row
 * norm) for fast reload of a shard; synchronous, streamed through pinned 64 MB
 * chunks.  Bad magic / truncated -> HSD_ERR_PARSE, version -> HSD_ERR_VERSION. */
hsd_status hsd_collection_save_image(hsd_collection* c, const char* path);
hsd_status hsd_collection_load_image(const char* path, int device, hsd_collection** out);

/* ------------------------------------------------------------------------
 * Verify-skip lifecycle (Alg. 1).
 * ---------------------------------------------------------------------- */
typedef struct hsd_skip_state { /* VerifySkipState */
  double T;         /* pre-sampled similarity boundary */
  double min_S;
  int32_t O_dist;
  double delta;     /* feedback step */
  int32_t inverted; /* update_direction = inverted */
} hsd_skip_state;

/* offline_calibrate_skip over n_traj trajectories: rows [offsets[t],
 * offsets[t+1]) of the DEVICE feature matrix fp32 [n][d_f] (offsets: HOST
 * int64 [n_traj + 1]).  S(i, i+d) is the exactly rounded feature dot (the
 * similarity should_skip uses); the minimum S > T wins, ties to the first pair
 * in (trajectory, i, d) order.  Batched per-trajectory Gram tiles on the fp64
 * pipe (double-double, bit-exact).  No pair above T -> HSD_ERR_CALIBRATION
 * (skipping stays disabled).  Synchronizes `stream`. */
hsd_status hsd_calibrate_skip(int device, const float* features, int d_f, const int64_t* offsets, int n_traj,
                              double T, double* min_S, int* O_dist, void* stream);
/* update_skip_state: host arithmetic, literal Alg. 1
 * directions, optional inversion, min_S clamped to [T, 1], O_dist >= 1. */
hsd_status hsd_update_skip_state(hsd_skip_state* s, int success, double S_c, double min_S_h);

/* ------------------------------------------------------------------------
 * Hybrid decoding loop (config 5): the SPEC scheduler's run_step / run_episode
 * for R robots at once, device-resident.  Per round and
 * robot: decide_sd (kinematic fused metric over the trailing w points; cold
 * start -> drafter) -> retrieval (top-K_top drafts, 21 tokens, verify-skip,
 * verify_tree with relaxed acceptance) or toy drafter (L tokens, verified) ->
 * emitted tokens + autoregressive completion of the action slice -> ToyEnv
 * position += HSD_ENV_SCALE * dequantize(xyz bins) -> trajectory ring; cost
 * model, StepRecord trace and EpisodeReport counters.  The
 * synthetic harness (demonstration policy, robots, drafter) is the
 * counter-based one of hsd_synth.h.  The DB must hold HSD_PAYLOAD_TRAJ rows
 * (row = e * traj_T + j).  With a communicator the DB is row-sharded: every
 * rank runs all robots (replicated state), searches its shard and merges the
 * all-gathered top-k; results are identical on every rank.
 * ---------------------------------------------------------------------- */
enum { HSD_MODE_HYBRID = 0, HSD_MODE_PURE_RETRIEVAL = 1, HSD_MODE_PURE_DRAFTER = 2, HSD_MODE_AUTOREGRESSIVE = 3 };
#define HSD_HYB_RET_L 21    /* retrieval draft: 3 action slices */
#define HSD_HYB_MAX_EMIT 28 /* 21 accepted + completion to the slice boundary */

typedef struct hsd_hybrid_params {
  int32_t robots;           /* R */
  int32_t k;                /* K_top retrieved drafts (SPEC.md:379 default 3) */
  int32_t mode;             /* HSD_MODE_* (HybridConfig.mode) */
  int32_t traj_T;           /* demonstration length of the DB rows */
  int32_t drafter_p_pct;    /* toy drafter accuracy p in percent (85) */
  int32_t drafter_L;        /* drafter draft length (7) */
  int32_t gap_d;            /* should_skip gap d (1) */
  int32_t d_f;              /* verifier feature dim of the skip check (0: skip off) */
  uint64_t seed;            /* robots, drafter, logits, features */
  uint64_t db_seed;         /* DB keys + demonstration policy */
  int32_t key_kind;         /* synthetic key family of the DB (HSD_SYNTH_*) */
  int32_t record_trace;     /* keep the per-round StepRecord trace on the device */
  hsd_verify_params verify; /* acceptance caps + verify-skip state (retrieval mode) */
  hsd_metric_params metric; /* FusedMetricParams */
  hsd_norm_bounds bounds;   /* NormalizationBounds */
  double cost_verifier;     /* CostModel: verifier call 1.0 */
  double cost_drafter_token;/*            drafter token 0.1 */
  double cost_retrieval;    /*            retrieval query 0.37 */
} hsd_hybrid_params;

typedef struct hsd_step_record { /* StepRecord */
  float F;                /* fused metric (-1 in autoregressive mode) */
  int16_t accept_len;     /* accepted draft tokens */
  int16_t verifier_calls; /* chains verified + autoregressive completion tokens */
  int16_t n_emit;         /* tokens emitted (multiple of 7) */
  int8_t mode;            /* 1 retrieval_sd, 0 drafter_sd, 2 autoregressive */
  int8_t skipped;         /* verify-skip fired */
  float cost;             /* cost units of the round */
} hsd_step_record;

typedef struct hsd_episode_report { /* EpisodeReport counters */
  int64_t rounds, tokens, accepted, verifier_calls;
  double cost;
  int32_t n_retrieval, n_drafter, n_skipped, n_fallback;
} hsd_episode_report;

typedef struct hsd_hybrid hsd_hybrid;
/* comm may be NULL (single GPU: the collection holds rows [0, n_total_rows)). */
hsd_status hsd_hybrid_create(hsd_collection* c, hsd_comm* comm, int64_t id_offset, int64_t n_total_rows,
                             const hsd_hybrid_params* p, int max_rounds, hsd_hybrid** out);
hsd_status hsd_hybrid_destroy(hsd_hybrid* h);
/* Run n decode rounds for all robots on `stream` (one host sync per round:
 * the retrieval/drafter robot counts size the launches). */
hsd_status hsd_hybrid_step(hsd_hybrid* h, int n_rounds, void* stream);
/* Host copies: positions [R][3], reports [R], trace [rounds][R] (rounds
 * recorded so far, <= max_rounds), retrieval queries / drafter rounds so far. */
hsd_status hsd_hybrid_positions(hsd_hybrid* h, double* xyz);
hsd_status hsd_hybrid_reports(hsd_hybrid* h, hsd_episode_report* out);
hsd_status hsd_hybrid_trace(hsd_hybrid* h, hsd_step_record* out, int* rounds);
hsd_status hsd_hybrid_counts(hsd_hybrid* h, int64_t* retrieval_queries, int64_t* drafter_rounds);
/* CUDA-event stage times summed over the rounds since the last call (ms):
 * [decide (windows + K5 + compaction), search (queries, logits, K1+K2[+K3]),
 *  verify (K4 retrieval + drafter), emit, total]; synchronizes. */
hsd_status hsd_hybrid_stage_times(hsd_hybrid* h, int* rounds, double ms[5]);

/* Generate with an explicit payload family (HSD_PAYLOAD_*): TRAJ rows hold the
 * demonstration policy of episode row / traj_T from action row % traj_T. */
hsd_status hsd_collection_generate_ex(hsd_collection* c, int kind, uint64_t db_seed, int64_t row0, int64_t n,
                                      int payload, int traj_T);

/* ------------------------------------------------------------------------
 * Synthetic workload generators on the device (include/hsd/hsd_synth.h).
 * ---------------------------------------------------------------------- */
hsd_status hsd_gen_queries(int device, int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B,
                           int dim, float* out, void* stream);
/* logits [E][L][256] whose greedy bins are draft tokens of record rows[e]
 * (+ hsd_logit_greedy_bin deltas); rows may hold -1 (random draft). */
hsd_status hsd_gen_logits(hsd_collection* c, uint64_t seed, const int64_t* rows, int E, int L, float* out,
                          void* stream);
hsd_status hsd_gen_features(int device, uint64_t seed, int E, int d_f, float* now, float* prev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HSD_GPU_H */
