// k_hybrid.cu — kernels of the device-resident hybrid decoding loop (config 5):
// run_step / run_episode of the SPEC scheduler for R robots
// at once, around the hot-path kernels K1-K5.
//
// One round (hsd_hybrid_step, api.cu):
//   hyb_windows     trailing w-point window of every robot's trajectory ring
//   K5              window_features + decide_sd (cold start < w -> drafter)
//   hyb_compact     retrieval / drafter robot lists (pure modes override)
//   hyb_prep_ret    per retrieval robot: query embedding (near-duplicate of its
//                   demonstration row), skip-check features
//   hyb_logits      verifier logits whose greedy bins are the robot's policy
//   K1+K2 (+K3)     top-k retrieval of K_top drafts (sharded: all-gather+merge)
//   K4              gather + verify-skip + relaxed acceptance (L = 21)
//   hyb_drafts      toy drafter drafts (L = 7) ; K4 again with k = 1
//   hyb_emit        emitted tokens + autoregressive completion of the action
//                   slice -> dequantize -> ToyEnv position -> trajectory ring;
//                   cost model + StepRecord trace + EpisodeReport counters
// The synthetic harness (policy, robots, drafter, ToyEnv scale) is the
// counter-based one of include/hsd/hsd_synth.h, restated on the host by the
// oracle (oracle/hsd_oracle.c hsdo_hybrid_run) for parity.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "hsd/hsd_synth.h"
#include "kernels.h"

namespace hsd {
namespace {

constexpr int kMaxW = 32;

__global__ void hyb_windows_kernel(int R, int w, const double* __restrict__ ring, const int32_t* __restrict__ hist_n,
                                   double* __restrict__ xyz, int32_t* __restrict__ histw) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int n = hist_n[r];
  const double* rg = ring + (size_t)r * w * 3;
  double* out = xyz + (size_t)r * w * 3;
  // chronological order: the oldest of the last w points first
  for (int i = 0; i < w; ++i) {
    int src;
    if (n >= w)
      src = (n - w + i) % w;
    else
      src = i < n ? i : (n > 0 ? n - 1 : 0);
    out[i * 3 + 0] = rg[src * 3 + 0];
    out[i * 3 + 1] = rg[src * 3 + 1];
    out[i * 3 + 2] = rg[src * 3 + 2];
  }
  histw[r] = n;
}

// One CTA: mode per robot and the compacted retrieval / drafter lists.
// modes: 1 retrieval_sd, 0 drafter_sd, 2 autoregressive.
__global__ void __launch_bounds__(1024) hyb_compact_kernel(int R, int mode, const int32_t* __restrict__ decision,
                                                           int32_t* __restrict__ modes, int32_t* __restrict__ slot,
                                                           int32_t* __restrict__ ret_idx,
                                                           int32_t* __restrict__ drf_idx, int32_t* __restrict__ counts) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base_r, base_d;
  if (threadIdx.x == 0) base_r = base_d = 0;
  __syncthreads();
  for (int r0 = 0; r0 < R; r0 += 1024) {
    const int r = r0 + threadIdx.x;
    int m = -1;
    if (r < R) {
      if (mode == HSD_MODE_HYBRID)
        m = decision[r] == 1 ? 1 : 0;  // -1 (non-finite window) degrades to the drafter
      else
        m = mode == HSD_MODE_PURE_RETRIEVAL ? 1 : (mode == HSD_MODE_PURE_DRAFTER ? 0 : 2);
      modes[r] = m;
    }
    const int is_r = m == 1, is_d = m == 0;
    int pr, pd, tr, td;
    Scan(tmp).ExclusiveSum(is_r, pr, tr);
    __syncthreads();
    Scan(tmp).ExclusiveSum(is_d, pd, td);
    if (r < R) {
      if (is_r) {
        ret_idx[base_r + pr] = r;
        slot[r] = base_r + pr;
      } else if (is_d) {
        drf_idx[base_d + pd] = r;
        slot[r] = base_d + pd;
      } else {
        slot[r] = -1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      base_r += tr;
      base_d += td;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    counts[0] = base_r;
    counts[1] = base_d;
  }
}

// Per retrieval robot (one CTA each): query embedding and skip features.
__global__ void __launch_bounds__(256) hyb_prep_ret_kernel(HybridArgs a, int round, const int32_t* __restrict__ ret_idx,
                                                           float* __restrict__ queries, float* __restrict__ fnow,
                                                           float* __restrict__ fprev, int32_t* __restrict__ hist_c) {
  using BR = cub::BlockReduce<long long, 256>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ long long s_ss;
  const int i = blockIdx.x;
  const int r = ret_idx[i];
  const int64_t e = hsd_robot_episode(a.seed, r, a.n_demo);
  const int64_t j = a.act[r];
  const int64_t row = hsd_hybrid_query_row(e, j, a.traj_T, a.n_demo, a.n_rows);
  const int64_t qid = hsd_hybrid_qid(r, round);
  float* q = queries + (size_t)i * a.dim;
  if (a.key_kind == HSD_SYNTH_EXACT) {
    for (int c = threadIdx.x; c < a.dim; c += 256) q[c] = hsd_query_exact(a.seed, a.db_seed, qid, row, a.dim, c);
  } else {
    long long ss = 0;
    for (int c = threadIdx.x; c < a.dim; c += 256) {
      const long long v = hsd_query_raw(a.seed, a.db_seed, qid, row, a.dim, c);
      ss += v * v;
    }
    ss = BR(tmp).Sum(ss);
    if (threadIdx.x == 0) s_ss = ss;
    __syncthreads();
    ss = s_ss;
    for (int c = threadIdx.x; c < a.dim; c += 256)
      q[c] = hsd_norm_val(hsd_query_raw(a.seed, a.db_seed, qid, row, a.dim, c), ss);
    __syncthreads();
  }
  if (a.d_f > 0) {
    for (int which = 0; which < 2; ++which) {
      long long ss = 0;
      for (int c = threadIdx.x; c < a.d_f; c += 256) {
        const long long v = hsd_feat_raw(a.seed, qid, which, a.d_f, c);
        ss += v * v;
      }
      ss = BR(tmp).Sum(ss);
      if (threadIdx.x == 0) s_ss = ss;
      __syncthreads();
      ss = s_ss;
      float* f = (which ? fprev : fnow) + (size_t)i * a.d_f;
      for (int c = threadIdx.x; c < a.d_f; c += 256) f[c] = hsd_norm_val(hsd_feat_raw(a.seed, qid, which, a.d_f, c), ss);
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) hist_c[i] = a.rounds[r];
}

// Verifier logits [n][L][256] of listed robots: greedy bin = the robot's policy
// token at stream position act*7 + p (8.0), background multiples of 1/64.
__global__ void __launch_bounds__(256) hyb_logits_kernel(HybridArgs a, int round, const int32_t* __restrict__ idx, int L,
                                                         float* __restrict__ out) {
  const int i = blockIdx.x, p = blockIdx.y, b = threadIdx.x;
  const int r = idx[i];
  const int64_t e = hsd_robot_episode(a.seed, r, a.n_demo);
  const int g = hsd_robot_greedy(a.db_seed, a.seed, r, e, a.act[r] + p / 7, p % 7);
  const int64_t qid = hsd_hybrid_qid(r, round);
  out[((size_t)i * L + p) * 256 + b] = b == g ? 8.0f : hsd_logit_background(a.seed, qid, p, b);
}

// Toy-drafter drafts (k = 1 candidate, L tokens) of listed robots.
__global__ void hyb_drafts_kernel(HybridArgs a, int round, const int32_t* __restrict__ idx, int n, int L,
                                  uint8_t* __restrict__ drafts, int32_t* __restrict__ ids) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * HSD_TOKENS_STRIDE) return;
  const int i = t / HSD_TOKENS_STRIDE, p = t % HSD_TOKENS_STRIDE;
  const int r = idx[i];
  uint8_t v = 0;
  if (p < L) {
    const int64_t e = hsd_robot_episode(a.seed, r, a.n_demo);
    const int g = hsd_robot_greedy(a.db_seed, a.seed, r, e, a.act[r] + p / 7, p % 7);
    v = (uint8_t)hsd_drafter_token(a.seed, r, round, p, g, a.drafter_p_pct);
  }
  drafts[(size_t)i * HSD_TOKENS_STRIDE + p] = v;
  if (p == 0) ids[i] = 0;
}

// Emit: tokens of the round (+ autoregressive completion of the action slice)
// -> actions -> ToyEnv -> trajectory ring; cost model, trace, report counters.
__global__ void hyb_emit_kernel(HybridArgs a, int round, const int32_t* __restrict__ modes,
                                const int32_t* __restrict__ slot, const hsd_outcome* __restrict__ out_r,
                                const uint8_t* __restrict__ tok_r, const hsd_outcome* __restrict__ out_d,
                                const uint8_t* __restrict__ tok_d, const double* __restrict__ F,
                                hsd_step_record* __restrict__ trace) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  const int m = modes[r];
  const int64_t e = hsd_robot_episode(a.seed, r, a.n_demo);
  const int64_t j0 = a.act[r];
  uint8_t toks[HSD_HYB_MAX_EMIT];
  int n = 0, accepted = 0, calls = 0, skipped = 0, fallback = 0;
  double cost = 0.0;
  if (m == 1 || m == 0) {
    const int s = slot[r];
    const hsd_outcome o = m == 1 ? out_r[s] : out_d[s];
    const uint8_t* t = m == 1 ? tok_r + (size_t)s * HSD_HYB_RET_L : tok_d + (size_t)s * a.drafter_L;
    for (int i = 0; i < o.n_emit; ++i) toks[n++] = t[i];
    accepted = o.accept_len;
    calls = o.calls;
    skipped = o.skipped;
    fallback = o.fallback;
    cost = m == 1 ? a.cost_retrieval : HSD_MUL(a.cost_drafter_token, (double)a.drafter_L);
  }
  // autoregressive completion to the action-slice boundary (AR mode: 7 tokens)
  const int target = n == 0 ? 7 : ((n + 6) / 7) * 7;
  while (n < target) {
    toks[n] = (uint8_t)hsd_robot_greedy(a.db_seed, a.seed, r, e, j0 + n / 7, n % 7);
    ++n;
    ++calls;
  }
  cost = HSD_ADD(cost, HSD_MUL((double)calls, a.cost_verifier));
  // apply the completed actions
  double* pos = a.pos + (size_t)r * 3;
  double* ring = a.ring + (size_t)r * a.w * 3;
  int hn = a.hist_n[r];
  for (int act = 0; act < n / 7; ++act) {
    for (int d = 0; d < 3; ++d) {
      const double dq = hsd_dequantize_bin(toks[act * 7 + d], -1.0, 1.0, 256);
      pos[d] = HSD_ADD(pos[d], HSD_MUL(HSD_ENV_SCALE, dq));
    }
    const int slot_w = hn % a.w;
    ring[slot_w * 3 + 0] = pos[0];
    ring[slot_w * 3 + 1] = pos[1];
    ring[slot_w * 3 + 2] = pos[2];
    ++hn;
  }
  a.hist_n[r] = hn;
  a.act[r] = j0 + n / 7;
  a.rounds[r] += 1;
  hsd_episode_report& rep = a.report[r];
  rep.rounds += 1;
  rep.tokens += n;
  rep.accepted += accepted;
  rep.verifier_calls += calls;
  rep.cost = HSD_ADD(rep.cost, cost);
  rep.n_retrieval += m == 1;
  rep.n_drafter += m == 0;
  rep.n_skipped += skipped;
  rep.n_fallback += fallback;
  if (trace) {
    hsd_step_record& t = trace[(size_t)round * a.R + r];
    t.F = m == 2 ? -1.0f : (float)F[r];
    t.accept_len = (int16_t)accepted;
    t.verifier_calls = (int16_t)calls;
    t.n_emit = (int16_t)n;
    t.mode = (int8_t)m;
    t.skipped = (int8_t)skipped;
    t.cost = (float)cost;
  }
}

__global__ void hyb_init_kernel(HybridArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  for (int d = 0; d < 3; ++d) {
    const double v = hsd_robot_start(a.seed, r, d);
    a.pos[(size_t)r * 3 + d] = v;
    a.ring[(size_t)r * a.w * 3 + d] = v;  // the start pose is the first trajectory point
  }
  a.hist_n[r] = 1;
  a.act[r] = 0;
  a.rounds[r] = 0;
  a.report[r] = hsd_episode_report{};
}

}  // namespace

cudaError_t launch_hyb_init(const HybridArgs& a, cudaStream_t s) {
  hyb_init_kernel<<<(a.R + 127) / 128, 128, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_hyb_windows(int R, int w, const double* ring, const int32_t* hist_n, double* xyz, int32_t* histw,
                               cudaStream_t s) {
  if (w > kMaxW) return cudaErrorInvalidValue;
  hyb_windows_kernel<<<(R + 127) / 128, 128, 0, s>>>(R, w, ring, hist_n, xyz, histw);
  return cudaGetLastError();
}

cudaError_t launch_hyb_compact(int R, int mode, const int32_t* decision, int32_t* modes, int32_t* slot,
                               int32_t* ret_idx, int32_t* drf_idx, int32_t* counts, cudaStream_t s) {
  hyb_compact_kernel<<<1, 1024, 0, s>>>(R, mode, decision, modes, slot, ret_idx, drf_idx, counts);
  return cudaGetLastError();
}

cudaError_t launch_hyb_prep_ret(const HybridArgs& a, int round, const int32_t* ret_idx, int n, float* queries,
                                float* fnow, float* fprev, int32_t* hist_c, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  hyb_prep_ret_kernel<<<n, 256, 0, s>>>(a, round, ret_idx, queries, fnow, fprev, hist_c);
  return cudaGetLastError();
}

cudaError_t launch_hyb_logits(const HybridArgs& a, int round, const int32_t* idx, int n, int L, float* out,
                              cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  hyb_logits_kernel<<<dim3(n, L), 256, 0, s>>>(a, round, idx, L, out);
  return cudaGetLastError();
}

cudaError_t launch_hyb_drafts(const HybridArgs& a, int round, const int32_t* idx, int n, int L, uint8_t* drafts,
                              int32_t* ids, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int t = n * HSD_TOKENS_STRIDE;
  hyb_drafts_kernel<<<(t + 255) / 256, 256, 0, s>>>(a, round, idx, n, L, drafts, ids);
  return cudaGetLastError();
}

cudaError_t launch_hyb_emit(const HybridArgs& a, int round, const int32_t* modes, const int32_t* slot,
                            const hsd_outcome* out_r, const uint8_t* tok_r, const hsd_outcome* out_d,
                            const uint8_t* tok_d, const double* F, hsd_step_record* trace, cudaStream_t s) {
  hyb_emit_kernel<<<(a.R + 127) / 128, 128, 0, s>>>(a, round, modes, slot, out_r, tok_r, out_d, tok_d, F, trace);
  return cudaGetLastError();
}

}  // namespace hsd
