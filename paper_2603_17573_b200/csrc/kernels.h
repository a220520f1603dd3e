// kernels.h — host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hsd/hsd_gpu.h"

namespace hsd {

// ---- K0 synthetic generators (k_synth.cu) ------------------------------------
// keys: fp32 or bf16 (key_dtype = HSD_DTYPE_*) row-major [n][dim]
// payload: HSD_PAYLOAD_RANDOM (quantized hsd_action_val) or HSD_PAYLOAD_TRAJ
// (demonstration policy tokens, rows of traj_T actions per episode)
cudaError_t launch_gen_keys(int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim, void* keys, int key_dtype,
                            uint8_t* tokens, unsigned long long* maxnorm_bits, int payload, int traj_T,
                            cudaStream_t s);
cudaError_t launch_row_norms(const void* keys, int key_dtype, int64_t row0, int64_t n, int dim,
                             unsigned long long* maxnorm_bits, cudaStream_t s);
cudaError_t launch_to_bf16(const float* in, int64_t n, uint16_t* out, cudaStream_t s);
cudaError_t launch_gen_queries(int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B, int dim,
                               float* out, cudaStream_t s);
cudaError_t launch_gen_logits(const uint8_t* tokens, uint64_t seed, const int64_t* rows, int E, int L, float* out,
                              cudaStream_t s);
cudaError_t launch_gen_features(uint64_t seed, int E, int d_f, float* now, float* prev, cudaStream_t s);
cudaError_t launch_quantize(const double* actions, int64_t n, const double* lohi_dev /*[14] lo7 then hi7*/,
                            int k_bins, int32_t* bins, int32_t* status, cudaStream_t s);
cudaError_t launch_quantize_tokens(const double* actions /*[n][21]*/, int64_t n, uint8_t* tokens /*[n][32]*/,
                                   int32_t* bad, cudaStream_t s);

// ---- K1 similarity + per-list candidate lists --------------------------------
// partial: [lists][B][kCandLocal] u64 candidate keys (the filter's top-32 of
// each list's rows per query).
constexpr int kMaxBatchPass = 1024;  // queries per K1 pass

// Rows covered by filter list l of a pass (what the exact fallback rescans):
// blocks first + j * stride (j < count) of 128 rows, clipped to row_end, with
//   stride 1 (one CTA / cluster per list): first = l * per, count = min(per, nb - first)
//   stride 2 (CTA pairs, list 2u + h):     blocks u*per + h, u*per + h + 2, ... < min((u+1)*per, nb)
struct ListGeom {
  int64_t row_begin, row_end;
  int64_t per;
  int stride;
};

// K1 wide tcgen05 filter (k_sim_wide.cu): up to 256 queries per pass (UMMA
// N = 64/128/256), fp32 keys read as TF32 or bf16 keys (kind::f16); same
// partial-list contract.  scratch: sim_wide_scratch_bytes(dim).
int sim_wide_max_batch();
void sim_wide_set_single(bool single);  // ablation: no CTA-pair kernels
// partial lists (= persistent CTAs, or clusters when B > 256) of a wide pass
int sim_wide_lists(int B, int64_t rows, int num_sms);
double sim_wide_gamma(int dim, int key_dtype);
// true when a pass of B queries over fp32 keys converts the key tiles to bf16
// on chip (the CTA-pair kernel): its filter bound is the bf16-copy one
bool sim_wide_converts(int key_dtype, int B, int dim);
size_t sim_wide_scratch_bytes(int dim);
cudaError_t launch_sim_wide(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin, int64_t row_end,
                            int dim, const float* queries, int B, int lists, void* scratch, uint64_t* partial,
                            float* dump, cudaStream_t s, ListGeom* geom = nullptr);

// ---- K1x exact scan (k_exact.cu): every row's reference fp64 chain + top-k ----
// For small (rows x batch): replaces K1 + K2.  scratch: exact_scan_scratch_bytes,
// zeroed once at allocation (a ticket the last CTA resets).
constexpr int kScanMaxBatch = 4;
bool exact_scan_supported(int B, int dim, int key_dtype, int k);
size_t exact_scan_scratch_bytes(int B, int num_sms);
double exact_scan_cost_us(int64_t rows, int dim, int key_dtype, int B);
cudaError_t launch_exact_scan(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin,
                              int64_t row_end, int dim, const float* queries, int B, int k, void* scratch,
                              int num_sms, double* scores, int32_t* ids, cudaStream_t s);
// k > HSD_K_MAX: the same scan writes every row's order key, a stable radix
// sort per query orders (key, id); stream-ordered allocations (cudaMallocAsync).
bool exact_topk_large_supported(int dim, int key_dtype);
cudaError_t launch_exact_topk_large(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin,
                                    int64_t row_end, int dim, const float* queries, int B, int k, int num_sms,
                                    double* scores, int32_t* ids, cudaStream_t s);

// ---- K2 select: exact top-k from the filter lists -----------------------------
// Four launches (candidates + threshold, pooled rescoring, exact range
// fallback, rank; k_select.cu); scratch: select_scratch_bytes(B), B <= kMaxBatchPass.
// stats (device, accumulated): [0] queries that needed the range fallback,
// [1] pooled candidates rescored, [2] fallback lists rescanned.
size_t select_scratch_bytes(int B);
int select_max_lists();
// pub != nullptr: the rank kernel publishes the top-k records (global ids +
// draft tokens) into every peer's window instead of writing scores / ids.
struct P2PPublish;
cudaError_t launch_select(const uint64_t* partial, int lists, int B, int k, const void* keys, int key_dtype, int dim,
                          const float* queries, const unsigned long long* maxnorm_bits, double gamma,
                          const ListGeom& geom, double* scores, int32_t* ids, int* stats, void* scratch, int num_sms,
                          cudaStream_t s, const P2PPublish* pub = nullptr);

// Exact rescoring + rank of externally pooled candidates (the IVF index):
// pool [B][C] u64 candidate keys (kEmpty = none, ids = rows of `keys`),
// C <= 32; scratch: select_scratch_bytes(B), B <= kMaxBatchPass.
cudaError_t launch_rescore_pool(const uint64_t* pool, int C, int B, int k, const void* keys, int key_dtype, int dim,
                                const float* queries, double* scores, int32_t* ids, int* stats, void* scratch,
                                cudaStream_t s);

// K3 merge of G gathered per-rank top-k records (sharded search); tokens
// [G][B][k][32] are permuted alongside when non-null.
cudaError_t launch_merge_ranks(const double* g_scores, const int32_t* g_ids, const uint8_t* g_tok, int G, int B, int k,
                               double* scores, int32_t* ids, uint8_t* tok, cudaStream_t s);

// K3 over peer memory (k_p2p.cu): receive windows shared by CUDA IPC; publish
// writes this rank's B x k records into every peer's window + a release flag,
// merge waits for all G flags of its own window and merges.  err set on a
// peer that never published (bounded spin, no hang).
constexpr int kMaxP2P = 8;
struct P2PWindows {
  void* base[kMaxP2P];  // window of each rank as mapped in this process (own = local allocation)
  size_t off_flags, off_scores, off_ids, off_toks;
  int Bmax, kmax;
};
// Fused publish (K2's rank kernel writes its final records straight into the
// peers' windows): what the rank kernel needs to do it.
struct P2PPublish {
  P2PWindows w;
  int rank, G;
  uint64_t epoch;
  int64_t id_offset;      // local id -> global id
  int q_offset;           // query index of this pass's first query
  const uint8_t* tokens;  // local token table [n][32] (drafts travel with the records)
};
size_t p2p_window_bytes(int G, int Bmax, int kmax, P2PWindows* layout);
// Standalone publish from local buffers (empty shards) + the flag-synchronised merge.
cudaError_t launch_p2p_publish(const P2PWindows& w, int rank, int G, int B, int k, uint64_t epoch, const double* ls,
                               const int32_t* li, const uint8_t* lt, cudaStream_t s);
cudaError_t launch_p2p_merge(const P2PWindows& w, int rank, int G, int B, int k, uint64_t epoch, double* scores,
                             int32_t* ids, uint8_t* tok, int* err, cudaStream_t s);

// ---- approximate index: IVF-flat (k_ivf.cu; host side in api.cu) ---------------
// Scan units: mode 0 (coarse) unit u = (query u / per_q, rows [(u % per_q) span, +span)
// of [0, n_rows)); mode 1 (fine) pairs p = b * nprobe + j own units
// [upre[p], upre[p + 1]), spans of list probe[p] = [offs[l], offs[l+1]).
struct IvfUnits {
  int mode;
  int ur;    // rows per scoring chunk: 32 or 128
  int span;  // rows per unit: a multiple of ur (a unit loops over its chunks)
  int per_q, n_q;
  int64_t n_rows;
  int n_pairs, nprobe;
  const int32_t* upre;
  const int32_t* probe;
  const int32_t* offs;
};
constexpr int kIvfMaxLists = 16384;
size_t ivf_part_bytes(int64_t units);
// per-unit top-32 (u64 candidate keys; ids = row_id[pos] or pos) of bf16 (rows_bf16) or fp32 rows
cudaError_t launch_ivf_scan(const void* rows, int rows_bf16, int64_t stride, const int32_t* row_id, int dim,
                            const float* queries, const IvfUnits& su, int64_t max_units, int grid, uint64_t* part,
                            cudaStream_t s);
cudaError_t launch_ivf_merge(const uint64_t* part, const IvfUnits& su, int B, uint64_t* pool, cudaStream_t s);
cudaError_t launch_ivf_probe(const uint64_t* pool, int B, int nprobe, const int32_t* offs, int span, int32_t* probe,
                             int32_t* upre, cudaStream_t s);
// build: seeds (sum <- seed rows), centroids (sum <- list sums when perm; cent <- sum / |sum|)
cudaError_t launch_ivf_seed(const void* keys, int key_dtype, int dim, int64_t n, int nlist, double* sum,
                            cudaStream_t s);
cudaError_t launch_ivf_centroids(const void* keys, int key_dtype, int dim, int nlist, const int32_t* perm,
                                 const int32_t* offs, double* sum, float* cent, cudaStream_t s);
cudaError_t launch_ivf_widen(const uint16_t* in, int64_t n, float* out, cudaStream_t s);
// stable counting sort of rows by list: bh scratch [ivf_sort_blocks(n)][nlist]
int64_t ivf_sort_blocks(int64_t n, int64_t* chunk);
cudaError_t launch_ivf_sort(const int32_t* assign, int64_t n, int nlist, int32_t* bh, int32_t* offs, int32_t* perm,
                            cudaStream_t s);
// ---- K4 gather + verify-skip + relaxed acceptance ----------------------------
// Draft tokens come from the collection's table by id, or pre-gathered
// cand_tokens [E][k][32] when non-null (sharded search records).
cudaError_t launch_verify(const int32_t* ids, int E, int k, int L, const uint8_t* tokens, const uint8_t* cand_tokens,
                          const float* logits, const float* feat_now, const float* feat_prev, int d_f,
                          const int32_t* history, int gap_d, const hsd_verify_params* params_dev, int P, int need_cos,
                          hsd_outcome* out, uint8_t* tok_out, cudaStream_t s, const double* cos_in = nullptr,
                          bool early = false);
// early: K4 is the programmatic dependent of the search's last kernel and
// reduces its logits / features (inputs of the step) before it waits for the
// search grid; only the ids -> token rows -> acceptance sweep follow it.
// should_skip similarity [E] (exactly rounded, same bits as K4's in-kernel dot) as a separate pass
cudaError_t launch_cos(const float* feat_now, const float* feat_prev, int E, int d_f, double* cos_out,
                       cudaStream_t s);
cudaError_t launch_gather_tokens(const uint8_t* tokens, const int32_t* ids, int n, uint8_t* out, cudaStream_t s);

// ---- verify_tree with per-chain (teacher-forced) verifier output (k_chains.cu)
cudaError_t launch_chain_argmax(const float* logits, int64_t rows, uint8_t* greedy, cudaStream_t s);
cudaError_t launch_enumerate_chains(const int32_t* ids, int E, int k, int L, const uint8_t* tokens,
                                    const uint8_t* cand_tokens, int cap, int32_t* n_chains, int16_t* chain_ab,
                                    uint8_t* chain_tokens, cudaStream_t s);
cudaError_t launch_verify_chains(const int32_t* ids, int E, int k, int L, const uint8_t* tokens,
                                 const uint8_t* cand_tokens, int cap, const uint8_t* chain_greedy,
                                 const int32_t* greedy_ctx, const float* feat_now, const float* feat_prev, int d_f,
                                 const int32_t* history, int gap_d, const hsd_verify_params* params_dev,
                                 hsd_outcome* out, uint8_t* tok_out, cudaStream_t s);

// ---- K5 kinematics -------------------------------------------------------------
// vaj (optional) [W][3]: mean |velocity|, |acceleration|, |jerk| per step over the window
cudaError_t launch_kinematics(const double* xyz, int W, const hsd_metric_params& mp, const hsd_norm_bounds& nb,
                              const int32_t* history, double* R, double* D, double* F, int32_t* decision,
                              cudaStream_t s, double* vaj = nullptr);

// compute_percentile_bounds (k_bounds.cu): out2 (device) <- (min, p95); bad (device) += non-finite count
cudaError_t launch_percentile_bounds(const double* samples, int64_t n, double* out2, int* bad, cudaStream_t s);

// ---- verify-skip offline calibration (k_calib.cu) --------------------------------
size_t calib_scratch_bytes(int n_traj, int max_tiles);
cudaError_t launch_calibrate(const float* feat, int d_f, const int64_t* off_dev, int n_traj, int max_len, double T,
                             void* scratch, double* min_S_out, int* O_dist_out, int* found_out, cudaStream_t s);

// ---- hybrid decoding loop (k_hybrid.cu) ----------------------------------------
struct HybridArgs {
  int R, w, dim, d_f, key_kind, traj_T, drafter_p_pct, drafter_L;
  uint64_t seed, db_seed;
  int64_t n_demo, n_rows;
  double cost_verifier, cost_drafter_token, cost_retrieval;
  double* pos;       // [R][3]
  double* ring;      // [R][w][3]
  int32_t* hist_n;   // [R] points appended (ring index = hist_n % w)
  int64_t* act;      // [R] actions emitted (next action index j)
  int32_t* rounds;   // [R] decode rounds (stored skip features)
  hsd_episode_report* report;  // [R]
};
cudaError_t launch_hyb_init(const HybridArgs& a, cudaStream_t s);
cudaError_t launch_hyb_windows(int R, int w, const double* ring, const int32_t* hist_n, double* xyz, int32_t* histw,
                               cudaStream_t s);
cudaError_t launch_hyb_compact(int R, int mode, const int32_t* decision, int32_t* modes, int32_t* slot,
                               int32_t* ret_idx, int32_t* drf_idx, int32_t* counts, cudaStream_t s);
cudaError_t launch_hyb_prep_ret(const HybridArgs& a, int round, const int32_t* ret_idx, int n, float* queries,
                                float* fnow, float* fprev, int32_t* hist_c, cudaStream_t s);
cudaError_t launch_hyb_logits(const HybridArgs& a, int round, const int32_t* idx, int n, int L, float* out,
                              cudaStream_t s);
cudaError_t launch_hyb_drafts(const HybridArgs& a, int round, const int32_t* idx, int n, int L, uint8_t* drafts,
                              int32_t* ids, cudaStream_t s);
cudaError_t launch_hyb_emit(const HybridArgs& a, int round, const int32_t* modes, const int32_t* slot,
                            const hsd_outcome* out_r, const uint8_t* tok_r, const hsd_outcome* out_d,
                            const uint8_t* tok_d, const double* F, hsd_step_record* trace, cudaStream_t s);

}  // namespace hsd
