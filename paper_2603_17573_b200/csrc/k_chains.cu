// k_chains.cu — verify_tree with TEACHER-FORCED per-chain verifier output
// (VerifierModel::verify_chain, /root/reference/proj/include/hsd/models.hpp:34-37:
// "Greedy token for every position of `chain` in one call. Position i is
// conditioned on (context, chain[0..i))").
//
// K4 (k_verify.cu) serves the context-free case: one logit block per episode
// whose greedy tokens are the same for every chain.  A real verifier gives
// each chain its own greedy tokens, so verify_tree has to
// compare chain c's draft tokens with chain c's greedy tokens.  Kernels:
//
//   chain_argmax   greedy token of every (episode, chain, position) from
//                  per-chain logits [E][cap][L][256] (std::max_element's rule,
//                  dev::warp_argmax256): one warp per 256-bin row, streaming
//   enumerate      the chains verify_tree visits, per episode: unique token
//                  sequences (pos0 of candidate a, later groups of candidate b)
//                  in DFS = lexicographic (a, b) order, capped (SPEC.md:351-368,
//                  frozen reading DESIGN.md §3) -> (a, b) and the chain's tokens,
//                  so the caller can run its verifier on each chain
//   chains         one warp per episode: dedup, verify-skip,
//                  per-chain group acceptance against the
//                  chain's own greedy tokens, longest accepted prefix, earliest
//                  chain on ties, fallback = greedy_next(context) (models.hpp:38-39)
//
// Chain c of an episode with nA distinct pos0 groups and nB distinct later
// parts is (alpha, beta) = (c / nB, c % nB) over the canonical (first-seen)
// candidates: the first occurrence of a token sequence in lexicographic (a, b)
// order is (first a with its pos0, first b with its later part), so this is
// exactly the brute-force enumeration with duplicates removed
// (oracle: hsdo_enumerate_chains).
#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

constexpr int kCThreads = 64;  // 2 episodes (warps) per CTA
constexpr int kCWarps = kCThreads / 32;
constexpr int kTokRow = 24;

struct ChainWarp {
  uint8_t tok[HSD_K_MAX][kTokRow];
  uint8_t repA[HSD_K_MAX], repB[HSD_K_MAX];
};

// Candidate tokens of episode e into W.tok; distinct pos0 groups (repA, nA)
// and distinct later parts (repB, nB) in first-seen order.  Returns n_cand.
__device__ __forceinline__ int load_and_dedup(int e, int k, int L, const int32_t* __restrict__ ids,
                                              const uint8_t* __restrict__ tokens,
                                              const uint8_t* __restrict__ cand_tokens, ChainWarp& W, int& nA,
                                              int& nB) {
  const int lane = threadIdx.x & 31;
  const int id = lane < k ? ids[(size_t)e * k + lane] : -1;
  const int n_cand = __popc(__ballot_sync(0xffffffffu, id >= 0));  // rank order, -1 padding last
  if (id >= 0) {
    const uint8_t* row = cand_tokens ? cand_tokens + ((size_t)e * k + lane) * HSD_TOKENS_STRIDE
                                     : tokens + (size_t)id * HSD_TOKENS_STRIDE;
    const uint32_t* r4 = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
    for (int i = 0; i < kTokRow / 4; ++i) reinterpret_cast<uint32_t*>(W.tok[lane])[i] = r4[i];
  }
  __syncwarp();
  bool isA = false, isB = false;
  if (lane < n_cand) {
    const uint8_t* me = W.tok[lane];
    isA = isB = true;
    for (int c = 0; c < lane; ++c) {
      const uint8_t* o = W.tok[c];
      if (o[0] == me[0] && o[1] == me[1] && o[2] == me[2]) isA = false;
      bool same = true;
      for (int t = 3; t < L; ++t) same &= (o[t] == me[t]);
      if (same) isB = false;
    }
  }
  const unsigned mA = __ballot_sync(0xffffffffu, isA), mB = __ballot_sync(0xffffffffu, isB);
  nA = __popc(mA);
  nB = __popc(mB);
  if (isA) W.repA[__popc(mA & ((1u << lane) - 1))] = (uint8_t)lane;
  if (isB) W.repB[__popc(mB & ((1u << lane) - 1))] = (uint8_t)lane;
  __syncwarp();
  return n_cand;
}

__device__ __forceinline__ uint8_t chain_tok(const ChainWarp& W, int a, int b, int t) {
  return t < 3 ? W.tok[a][t] : W.tok[b][t];
}

__global__ void __launch_bounds__(256) chain_argmax_kernel(const float* __restrict__ logits, int64_t rows,
                                                           uint8_t* __restrict__ greedy) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float4* row = reinterpret_cast<const float4*>(logits + r * 256);
  const float4 a = __ldcs(row + 2 * lane), c = __ldcs(row + 2 * lane + 1);
  const int g = dev::warp_argmax256(a, c, lane);
  if (lane == 0) greedy[r] = (uint8_t)g;
}

__global__ void __launch_bounds__(kCThreads) enumerate_kernel(const int32_t* __restrict__ ids, int E, int k, int L,
                                                              const uint8_t* __restrict__ tokens,
                                                              const uint8_t* __restrict__ cand_tokens, int cap,
                                                              int32_t* __restrict__ n_chains,
                                                              int16_t* __restrict__ chain_ab,
                                                              uint8_t* __restrict__ chain_tokens) {
  __shared__ ChainWarp sw[kCWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kCWarps + warp;
  if (e >= E) return;
  ChainWarp& W = sw[warp];
  int nA, nB;
  const int n_cand = load_and_dedup(e, k, L, ids, tokens, cand_tokens, W, nA, nB);
  const int n = n_cand ? min(cap, nA * nB) : 0;
  if (lane == 0) n_chains[e] = n;
  for (int c = lane; c < n; c += 32) {
    const int a = W.repA[c / nB], b = W.repB[c % nB];
    chain_ab[((size_t)e * cap + c) * 2] = (int16_t)a;
    chain_ab[((size_t)e * cap + c) * 2 + 1] = (int16_t)b;
    uint8_t* dst = chain_tokens + ((size_t)e * cap + c) * L;
    for (int t = 0; t < L; ++t) dst[t] = chain_tok(W, a, b, t);
  }
}

__global__ void __launch_bounds__(kCThreads) chains_kernel(
    const int32_t* __restrict__ ids, int E, int k, int L, const uint8_t* __restrict__ tokens,
    const uint8_t* __restrict__ cand_tokens, int cap, const uint8_t* __restrict__ chain_greedy,
    const int32_t* __restrict__ greedy_ctx, const float* __restrict__ feat_now, const float* __restrict__ feat_prev,
    int d_f, const int32_t* __restrict__ history, int gap_d, const hsd_verify_params* __restrict__ params,
    hsd_outcome* __restrict__ out, uint8_t* __restrict__ tok_out) {
  __shared__ ChainWarp sw[kCWarps];
  dev::pdl_wait();
  dev::pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kCWarps + warp;
  if (e >= E) return;
  ChainWarp& W = sw[warp];
  const hsd_verify_params p = *params;
  int nA, nB;
  const int n_cand = load_and_dedup(e, k, L, ids, tokens, cand_tokens, W, nA, nB);
  double cosv = -2.0;
  if (p.skip_enabled && feat_now && feat_prev)
    cosv = dev::warp_dd_dot(feat_now + (size_t)e * d_f, feat_prev + (size_t)e * d_f, d_f, lane);
  const int hist = history ? history[e] : 0x7fffffff;
  const bool skip = p.skip_enabled && n_cand > 0 && gap_d >= 1 && hist >= gap_d && gap_d <= p.O_dist &&
                    cosv >= p.min_S;
  const int g0 = greedy_ctx[e];
  const int n = n_cand ? min(cap, nA * nB) : 0;
  // per chain: accepted prefix against the chain's own greedy tokens
  int best_len = -1, best_c = 0x7fffffff;
  if (!skip)
    for (int c = lane; c < n; c += 32) {
      const int a = W.repA[c / nB], b = W.repB[c % nB];
      const uint8_t* g = chain_greedy + ((size_t)e * cap + c) * L;
      int len = 0;
      for (int grp = 0; grp < (L / 7) * 3; ++grp) {
        const int s = grp / 3, kind = grp % 3;
        const int st = s * 7 + (kind == 0 ? 0 : (kind == 1 ? 3 : 6)), ln = kind == 2 ? 1 : 3;
        int sum = 0, mx = 0;
        for (int i = 0; i < ln; ++i) {
          const int bias = abs((int)chain_tok(W, a, b, st + i) - (int)g[st + i]);
          sum += bias;
          mx = bias > mx ? bias : mx;
        }
        const bool ok = (kind == 2 || !p.relaxed) ? mx == 0 : (sum <= p.bias_seq_max && mx <= p.bias_token_max);
        if (!ok) break;
        len += ln;
      }
      if (len > best_len) {  // c ascends per lane: the first maximum is the earliest
        best_len = len;
        best_c = c;
      }
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int ol = __shfl_xor_sync(0xffffffffu, best_len, o);
    const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
    if (ol > best_len || (ol == best_len && oc < best_c)) {
      best_len = ol;
      best_c = oc;
    }
  }
  hsd_outcome o;
  o.accept_len = 0;
  o.win_a = -1;
  o.win_b = -1;
  o.calls = 0;
  o.fallback = 0;
  o.skipped = 0;
  o.n_emit = 0;
  o.greedy0 = (int16_t)g0;
  o.cos_sim = (float)cosv;
  uint8_t* my = tok_out + (size_t)e * L;
  int wa = 0, wb = 0, emit = 0;  // emitted draft prefix from chain (wa, wb)
  if (skip) {  // the rank-0 draft counts as fully accepted
    o.accept_len = L;
    o.win_a = o.win_b = 0;
    o.skipped = 1;
    emit = L;
  } else if (n_cand == 0) {  // empty shard: one autoregressive step
    o.fallback = 1;
    o.calls = 1;
  } else {
    o.calls = (int16_t)n;
    wa = W.repA[best_c / nB];
    wb = W.repB[best_c % nB];
    o.win_a = (int16_t)wa;
    o.win_b = (int16_t)wb;
    if (best_len <= 0) {
      o.fallback = 1;
    } else {
      o.accept_len = best_len;
      emit = best_len;
    }
  }
  o.n_emit = (int16_t)(o.fallback ? 1 : emit);
  if (lane < L) my[lane] = o.fallback ? (lane == 0 ? (uint8_t)g0 : 0) : (lane < emit ? chain_tok(W, wa, wb, lane) : 0);
  if (lane == 0) out[e] = o;
}

}  // namespace

cudaError_t launch_chain_argmax(const float* logits, int64_t rows, uint8_t* greedy, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  chain_argmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(logits, rows, greedy);
  return cudaGetLastError();
}

cudaError_t launch_enumerate_chains(const int32_t* ids, int E, int k, int L, const uint8_t* tokens,
                                    const uint8_t* cand_tokens, int cap, int32_t* n_chains, int16_t* chain_ab,
                                    uint8_t* chain_tokens, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  enumerate_kernel<<<(E + kCWarps - 1) / kCWarps, kCThreads, 0, s>>>(ids, E, k, L, tokens, cand_tokens, cap,
                                                                      n_chains, chain_ab, chain_tokens);
  return cudaGetLastError();
}

cudaError_t launch_verify_chains(const int32_t* ids, int E, int k, int L, const uint8_t* tokens,
                                 const uint8_t* cand_tokens, int cap, const uint8_t* chain_greedy,
                                 const int32_t* greedy_ctx, const float* feat_now, const float* feat_prev, int d_f,
                                 const int32_t* history, int gap_d, const hsd_verify_params* params_dev,
                                 hsd_outcome* out, uint8_t* tok_out, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  return launch_pdl(chains_kernel, dim3((E + kCWarps - 1) / kCWarps), dim3(kCThreads), 0, s, ids, E, k, L, tokens,
                    cand_tokens, cap, chain_greedy, greedy_ctx, feat_now, feat_prev, d_f, history, gap_d, params_dev,
                    out, tok_out);
}

}  // namespace hsd
