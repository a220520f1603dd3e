// k_verify.cu — K4: fused draft gather + verify-skip + sequence-wise relaxed
// acceptance + accepted length, one warp per episode.
//
// Spec-only in the reference; semantics frozen in the oracle
// (oracle/hsd_oracle.c: hsdo_verify_round) and DESIGN.md:
//   - retrieve_drafts: gather the k candidates' pre-quantized
//     payload tokens (L = 7: next_actions[0]; L = 21: all three slices);
//   - greedy verifier token per position = argmax over 256 bins, lowest bin
//     on ties (Eq. 2-1);
//   - should_skip: d <= O_dist, history >= d and
//     cos(f_now, f_prev) >= min_S (double-double dot, exactly rounded);
//   - sequence groups pos/rot/grip; accept_sequence
//     (SPEC.md:430-439): gripper zero tolerance, else sum <= 30 and max <= 15;
//   - chains (a, b): pos0 from rank a, every later group from rank b (gripper
//     isolation), DFS = lexicographic order over distinct
//     token sequences, capped; longest accepted prefix wins,
//     earliest chain on ties; empty prefix -> fallback greedy token
//     (SPEC.md:440-448).
// All parameter sets of a sweep are evaluated from the same registers; the
// logits, tokens and features are read once.
#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

constexpr int kThreads = 64;  // 2 warps (episodes) per CTA: finer CTAs balance C3's 4096 episodes over 148 SMs
constexpr int kWarps = kThreads / 32;
constexpr int kTokStride = 24;  // bytes per candidate row in shared memory
constexpr int kPairs = 256;     // (parameter set, candidate) pairs per warp per chunk
constexpr int kFeatUnroll = 4;  // feature float4 pairs loaded per lane before accumulation

__device__ __forceinline__ int group_count(int L) { return (L / 7) * 3; }
__device__ __forceinline__ void group_at(int g, int& st, int& ln, bool& grip) {
  const int s = g / 3, kind = g % 3;
  st = s * 7 + (kind == 0 ? 0 : (kind == 1 ? 3 : 6));
  ln = kind == 2 ? 1 : 3;
  grip = kind == 2;
}

__device__ __forceinline__ bool accept_group(const uint8_t* draft, const int* greedy, int st, int ln, bool grip,
                                             const hsd_verify_params& p) {
  int sum = 0, mx = 0;
  for (int i = 0; i < ln; ++i) {
    const int b = abs((int)draft[st + i] - greedy[st + i]);
    sum += b;
    mx = b > mx ? b : mx;
  }
  if (grip || !p.relaxed) return mx == 0;
  return sum <= p.bias_seq_max && mx <= p.bias_token_max;
}

// Per-warp shared scratch of one episode.
struct WarpScratch {
  uint8_t tok[HSD_K_MAX][kTokStride];
  int greedy[32];
  uint8_t pair[kPairs];  // per (set, candidate): rest | pos0-accepted << 7
  int8_t len[kPairs], bb[kPairs];
  int rankA[HSD_K_MAX], rankB[HSD_K_MAX];
};

// verify-skip similarity of one episode on one warp: exactly rounded dot
// (double-double; the result is the exact sum rounded once, so the order is
// free).  kFeatUnroll float4 pairs per lane are requested (volatile loads,
// all issued) before any is accumulated.
__device__ __forceinline__ double episode_cos(const float* fnE, const float* fpE, int d_f, int lane) {
  const float4* a4 = reinterpret_cast<const float4*>(fnE);
  const float4* b4 = reinterpret_cast<const float4*>(fpE);
  const int n4 = d_f / 4;
  // two independent double-double accumulators (x / z and y / w components)
  double hv[2] = {0.0, 0.0}, lv[2] = {0.0, 0.0};
  for (int t0 = lane; t0 < n4; t0 += 32 * kFeatUnroll) {
    float4 xa[kFeatUnroll], yb[kFeatUnroll];
#pragma unroll
    for (int u = 0; u < kFeatUnroll; ++u) {
      const int t = min(t0 + 32 * u, n4 - 1);
      xa[u] = dev::ldg_stream(a4 + t);
      yb[u] = dev::ldg_stream(b4 + t);
    }
#pragma unroll
    for (int u = 0; u < kFeatUnroll; ++u) {
      if (t0 + 32 * u >= n4) {
        xa[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        yb[u] = xa[u];
      }
      const double pr[4] = {(double)xa[u].x * (double)yb[u].x, (double)xa[u].y * (double)yb[u].y,
                            (double)xa[u].z * (double)yb[u].z, (double)xa[u].w * (double)yb[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double s, er;
        dev::two_sum(hv[i & 1], pr[i], s, er);
        hv[i & 1] = s;
        lv[i & 1] = __dadd_rn(lv[i & 1], er);
      }
    }
  }
  double hi = hv[0], lo = lv[0];
  {
    double s, er;
    dev::two_sum(hi, hv[1], s, er);
    hi = s;
    lo = __dadd_rn(__dadd_rn(lo, lv[1]), er);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ohi = __shfl_xor_sync(0xffffffffu, hi, o);
    const double olo = __shfl_xor_sync(0xffffffffu, lo, o);
    double s, er;
    dev::two_sum(hi, ohi, s, er);
    hi = s;
    lo = __dadd_rn(__dadd_rn(lo, olo), er);
  }
  double s, er;
  dev::two_sum(hi, lo, s, er);
  return s;
}

// The same similarity, fast: plain fp64 sums (every fp32 x fp32 product is
// exact in fp64; two FMA chains per lane, then the butterfly) plus a
// rigorous bound on their error, from an fp32 sum of |products|.  Whenever
// the bound cannot settle the result — the float cos_sim output or any
// enabled set's `cos >= min_S` decision could differ from the exactly
// rounded similarity's — the exact double-double pass (episode_cos) decides
// instead.  The returned value is then only used through those two, so it is
// interchangeable with the exact one.  Half the fp64 instructions of the
// double-double loop on the common path.
__device__ __forceinline__ void cos_accum(const float4 (&xa)[kFeatUnroll], const float4 (&yb)[kFeatUnroll],
                                          double& s0, double& s1, float& ab) {
#pragma unroll
  for (int u = 0; u < kFeatUnroll; ++u) {
    s0 = fma((double)xa[u].x, (double)yb[u].x, s0);
    s1 = fma((double)xa[u].y, (double)yb[u].y, s1);
    s0 = fma((double)xa[u].z, (double)yb[u].z, s0);
    s1 = fma((double)xa[u].w, (double)yb[u].w, s1);
    ab = fmaf(fabsf(xa[u].x), fabsf(yb[u].x), ab);
    ab = fmaf(fabsf(xa[u].y), fabsf(yb[u].y), ab);
    ab = fmaf(fabsf(xa[u].z), fabsf(yb[u].z), ab);
    ab = fmaf(fabsf(xa[u].w), fabsf(yb[u].w), ab);
  }
}

// Chunk c of a lane's feature elements: float4 index c * 32U + 32u + lane
// (volatile loads: every load of the chunk is issued before any is used).
__device__ __forceinline__ void cos_load_regs(const float4* a4, const float4* b4, int n4, int c, int lane,
                                              float4 (&xa)[kFeatUnroll], float4 (&yb)[kFeatUnroll]) {
#pragma unroll
  for (int u = 0; u < kFeatUnroll; ++u) {
    const int t = min(c * 32 * kFeatUnroll + 32 * u + lane, n4 - 1);
    xa[u] = dev::ldg_stream(a4 + t);
    yb[u] = dev::ldg_stream(b4 + t);
  }
#pragma unroll
  for (int u = 0; u < kFeatUnroll; ++u)
    if (c * 32 * kFeatUnroll + 32 * u + lane >= n4) {
      xa[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      yb[u] = xa[u];
    }
}

__device__ __forceinline__ double episode_cos_fast(const float* fnE, const float* fpE, int d_f, int lane,
                                                   const hsd_verify_params* __restrict__ params, int P) {
  const float4* a4 = reinterpret_cast<const float4*>(fnE);
  const float4* b4 = reinterpret_cast<const float4*>(fpE);
  const int n4 = d_f / 4;
  const int nch = (n4 + 32 * kFeatUnroll - 1) / (32 * kFeatUnroll);
  double s0 = 0.0, s1 = 0.0;
  float ab = 0.f;
  for (int c = 0; c < nch; ++c) {
    float4 xa[kFeatUnroll], yb[kFeatUnroll];
    cos_load_regs(a4, b4, n4, c, lane, xa, yb);
    cos_accum(xa, yb, s0, s1, ab);
  }
  double sv = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // butterfly: every lane ends with the same bits
    sv += __shfl_xor_sync(0xffffffffu, sv, o);
    ab += __shfl_xor_sync(0xffffffffu, ab, o);
  }
  // A term passes through <= d_f / 32 + 8 roundings (its chain, the join, 5
  // butterfly levels): |sv - S| <= m u sum|p| (1 + O(mu)).  The fp32 sum of
  // |p| (m_f roundings, every term rounded at most once more) is a lower
  // estimate within m_f 2^-24; fp32 underflow loses < 2^-149 per term.
  const double m = (double)(d_f / 32 + 8);
  const double abs_sum = (double)ab * (1.0 + (m + 2.0) * 0x1p-23) + (double)d_f * 0x1p-148;
  const double err = abs_sum * m * 0x1p-53 * (1.0 + 0x1p-30) + (double)d_f * 0x1p-1074;
  const double e2 = err * (1.0 + 0x1p-50) + fabs(sv) * 0x1p-51;  // + the final rounding of the exact value
  bool amb = !isfinite(sv) || !isfinite(e2) || (float)(sv - e2) != (float)(sv + e2);
  for (int p = 0; p < P; ++p)
    if (params[p].skip_enabled) amb |= fabs(sv - params[p].min_S) <= e2 + fabs(params[p].min_S) * 0x1p-51;
  return amb ? episode_cos(fnE, fpE, d_f, lane) : sv;
}

// Candidate dedup (chain language): lane c < n_cand gets the
// first candidate with its pos0 group (bytes 0-2) and the first with its
// later groups (bytes 3..L-1).  Token rows live in registers (NW words) and
// are compared through shuffles, all lanes in step.
template <int NW>
__device__ __forceinline__ void dedup_rows(const WarpScratch& W, int n_cand, int L, int lane, int& ca, int& cb) {
  uint32_t w[NW], mk[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    w[i] = lane < n_cand ? reinterpret_cast<const uint32_t*>(W.tok[lane])[i] : 0u;
    uint32_t m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int t = 4 * i + b;
      if (t >= 3 && t < L) m |= 0xFFu << (8 * b);
    }
    mk[i] = m;
  }
  ca = lane;
  cb = lane;
  for (int c = 0; c < n_cand; ++c) {
    uint32_t dA = 0, dB = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint32_t x = __shfl_sync(0xffffffffu, w[i], c) ^ w[i];
      if (i == 0) dA = x & 0xFFFFFFu;
      dB |= x & mk[i];
    }
    if (c < lane) {
      if (ca == lane && dA == 0) ca = c;
      if (cb == lane && dB == 0) cb = c;
    }
  }
}

// One episode's decode round on one warp.  lgE: its logits [L][256]; fnE /
// fpE: its features [d_f] (or null).
//
// Phase order.  C3's 4096 episodes fit in one wave of warps (32 per SM), so
// the kernel lasts as long as one warp's whole round.  The two halves of the
// round — streaming the 32-KB feature pair (HBM-bound) and the logits +
// dedup + acceptance sweep (latency-bound, little traffic) — are independent
// until the outcome step needs the similarity.  Even warps stream their
// features first, odd warps last, so on every SM half the warps keep HBM busy
// while the other half run their sweeps, instead of every warp reaching the
// feature phase at the same time.  (A persistent variant streaming the next
// episode into shared memory with bulk copies measured 3.7x slower: with 2
// warps per SM the short dependent global reads of ids / tokens / params are
// no longer hidden.  One CTA of 4 warps per episode with every load issued up
// front measured 1.7x slower: its 128 registers left 4 episodes per SM, each
// serialising its sweep on one warp.)
__device__ __forceinline__ void verify_episode(int e, int E, int k, int L, const int32_t* __restrict__ ids,
                                               const uint8_t* __restrict__ tokens,
                                               const uint8_t* __restrict__ cand_tokens, const float* lgE,
                                               const float* fnE, const float* fpE, int d_f,
                                               const int32_t* __restrict__ history, int gap_d,
                                               const hsd_verify_params* __restrict__ params, int P, int need_cos,
                                               const double* __restrict__ cos_in, hsd_outcome* __restrict__ out,
                                               uint8_t* __restrict__ tok_out, WarpScratch& W, bool early) {
  const int lane = threadIdx.x & 31;
  // early: launched (PDL) while the search still runs — the features and
  // logits (inputs of the step) are reduced first, then the warp waits for
  // the search grid and only the ids -> token rows -> sweep remain after it
  const bool feat_first = early || ((threadIdx.x >> 5) & 1) == 0;
  const bool own_cos = need_cos && !cos_in && fnE && fpE;
  // The candidate ids (and then their token rows) do not depend on the logits
  // or the features: issue them first so their round trips overlap the
  // logits / feature phases instead of following them.
  const int32_t* my_ids = ids + (size_t)e * k;
  int id = -1;
  if (!early) id = lane < k ? my_ids[lane] : -1;
  double cosv = -2.0;
  if (need_cos && cos_in) cosv = cos_in[e];  // cos_kernel's pass (off the critical path in the engine step)
  // ---- the candidates' draft tokens: cp.async into this warp's staging rows
  //      (waited for before the dedup)
  auto stage_tokens = [&]() {
    if (id >= 0) {
      const uint8_t* row = cand_tokens ? cand_tokens + ((size_t)e * k + lane) * HSD_TOKENS_STRIDE
                                       : tokens + (size_t)id * HSD_TOKENS_STRIDE;
#pragma unroll
      for (int i = 0; i < kTokStride / 4; ++i) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(&W.tok[lane][4 * i]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(row + 4 * i) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // Two phases in parity order (see above): the feature stream, and the
  // logits + token gather + dedup.  One code site each.
  int n_cand = 0, nA = 0, nB = 0;
  // odd warps run the sweep before their features: skip decisions are deferred
  const bool defer = own_cos && !feat_first;
  const int hist = history ? history[e] : 0x7fffffff;
  const int hist_ok = gap_d >= 1 && hist >= gap_d;
  auto skip_cond = [&](const hsd_verify_params& pp) {  // should_skip without the similarity test
    return pp.skip_enabled && n_cand > 0 && hist_ok && gap_d <= pp.O_dist;
  };
  const int* greedy = W.greedy;  // positions < L (shared memory, no per-thread copy)
  for (int ph = 0; ph < 2; ++ph) {
    if ((ph == 0) == feat_first) {
      if (ph == 0 && !early) stage_tokens();  // even warps: the token rows land under the feature stream
      if (own_cos) cosv = episode_cos_fast(fnE, fpE, d_f, lane, params, P);
      continue;
    }
    // ---- greedy tokens: argmax per position, lowest index on ties.  Four
    //      positions are loaded before any is reduced (4 KB in flight per warp).
    const float4* lg = reinterpret_cast<const float4*>(lgE);
    for (int p0 = 0; p0 < L; p0 += 4) {
      float4 a[4], c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = min(p0 + u, L - 1);
        a[u] = lg[p * 64 + lane * 2];
        c[u] = lg[p * 64 + lane * 2 + 1];
      }
      if (ph == 0 && p0 == 0) stage_tokens();  // odd warps: the id has arrived under the logit loads
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int bi = dev::warp_argmax256(a[u], c[u], lane);
        if (lane == 0 && p0 + u < L) W.greedy[p0 + u] = bi;
      }
    }
    if (early) {  // the search's ids are complete and visible past this point
      dev::pdl_wait();
      id = lane < k ? my_ids[lane] : -1;
      stage_tokens();
    }
    // ---- the gathered draft tokens have landed: dedup (independent of params)
    n_cand = __popc(__ballot_sync(0xffffffffu, id >= 0));  // ids are rank-ordered, -1 padding last
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    int ca, cb;
    if (L <= 8)
      dedup_rows<2>(W, n_cand, L, lane, ca, cb);
    else
      dedup_rows<6>(W, n_cand, L, lane, ca, cb);
    const bool isA = lane < n_cand && ca == lane;
    const bool isB = lane < n_cand && cb == lane;
    const unsigned mA = __ballot_sync(0xffffffffu, isA), mB = __ballot_sync(0xffffffffu, isB);
    nA = __popc(mA);
    nB = __popc(mB);
    if (lane < n_cand) {
      W.rankA[lane] = isA ? __popc(mA & ((1u << lane) - 1)) : -1;
      W.rankB[lane] = isB ? __popc(mB & ((1u << lane) - 1)) : -1;
    }
    __syncwarp();

  // ---- per parameter set (a tolerance / threshold sweep): lane-parallel over
  //      (set, candidate) pairs, processed in chunks of kPairs pairs.
  //      A: group acceptance of every candidate (pos0 accepted?, length of the
  //         accepted run of later groups);
  //      B: for every canonical pos0 candidate a, the best later-group source b
  //         among the enumerated chains (DFS order: rank_a * nB + rank_b < cap);
  //      C: one lane per set: longest chain, earliest on ties -> outcome.
  const int G = group_count(L);
  const int nc = n_cand > 0 ? n_cand : 1;
  const int chunk = kPairs / nc;  // sets per chunk (>= 1: n_cand <= 32)
  for (int p0 = 0; p0 < P; p0 += chunk) {
    const int pc = min(chunk, P - p0);
    const int npairs = pc * n_cand;
    for (int idx = lane; idx < npairs; idx += 32) {  // A
      const int pi = p0 + idx / n_cand, c = idx % n_cand;
      const hsd_verify_params& pp = params[pi];
      const uint8_t* me = W.tok[c];
      int st, ln;
      bool gr;
      group_at(0, st, ln, gr);
      const int a0 = accept_group(me, greedy, st, ln, gr, pp) ? 1 : 0;
      int rest = 0;
      for (int g = 1; g < G; ++g) {
        group_at(g, st, ln, gr);
        if (!accept_group(me, greedy, st, ln, gr, pp)) break;
        rest += ln;
      }
      W.pair[idx] = (uint8_t)(rest | (a0 << 7));
    }
    __syncwarp();
    for (int idx = lane; idx < npairs; idx += 32) {  // B
      const int pi = p0 + idx / n_cand, a = idx % n_cand, base = idx - a;
      const int rA = W.rankA[a];
      int len = -1, bb = -1;
      if (rA >= 0) {
        const int cap = params[pi].chain_cap > 0 ? params[pi].chain_cap : 64;
        const int limit = cap - rA * nB;  // b's with rankB < limit are enumerated
        if (limit > 0) {
          int br = -1;
          for (int b = 0; b < n_cand; ++b) {
            const int rb = W.rankB[b];
            if (rb < 0 || rb >= limit) continue;
            const int r = W.pair[base + b] & 0x7F;
            if (r > br) {
              br = r;
              bb = b;
            }
          }
          len = (W.pair[idx] >> 7) ? 3 + br : 0;
        }
      }
      W.len[idx] = (int8_t)len;
      W.bb[idx] = (int8_t)bb;
    }
    __syncwarp();
    for (int q = lane; q < pc; q += 32) {  // C
      const int pi = p0 + q;
      const hsd_verify_params& pp = params[pi];
      hsd_outcome o;
      o.accept_len = 0;
      o.win_a = -1;
      o.win_b = -1;
      o.calls = 0;
      o.fallback = 0;
      o.skipped = 0;
      o.n_emit = 0;
      o.greedy0 = (int16_t)greedy[0];
      o.cos_sim = (float)cosv;
      uint8_t* my_tok = tok_out + ((size_t)pi * E + e) * L;
      const bool skip = !defer && skip_cond(pp) && cosv >= pp.min_S;
      if (skip) {  // the retrieved draft is emitted as fully accepted
        o.accept_len = L;
        o.win_a = 0;
        o.win_b = 0;
        o.skipped = 1;
        o.n_emit = (int16_t)L;
        for (int t = 0; t < L; ++t) my_tok[t] = W.tok[0][t];
      } else if (n_cand == 0) {  // empty shard: autoregressive step
        o.fallback = 1;
        o.calls = 1;
        o.n_emit = 1;
        my_tok[0] = (uint8_t)greedy[0];
        for (int t = 1; t < L; ++t) my_tok[t] = 0;
      } else {
        const int cap = pp.chain_cap > 0 ? pp.chain_cap : 64;
        int wl = -1, wa = 0, wr = 1 << 20, wb = -1;  // longest, then the earliest chain (smallest rank of a)
        for (int a = 0; a < n_cand; ++a) {
          const int l = W.len[q * n_cand + a];
          const int ra = W.rankA[a] >= 0 ? W.rankA[a] : (1 << 20);
          if (l > wl || (l == wl && ra < wr)) {
            wl = l;
            wa = a;
            wr = ra;
            wb = W.bb[q * n_cand + a];
          }
        }
        const long long chains = (long long)nA * nB;
        o.calls = (int16_t)(chains < cap ? chains : cap);
        if (wl <= 0) {  // every chain rejected at pos0 -> first chain, fallback token
          o.win_a = 0;
          o.win_b = 0;
          o.fallback = 1;
          o.n_emit = 1;
          my_tok[0] = (uint8_t)greedy[0];
          for (int t = 1; t < L; ++t) my_tok[t] = 0;
        } else {
          o.win_a = (int16_t)wa;
          o.win_b = (int16_t)wb;
          o.accept_len = wl;
          o.n_emit = (int16_t)wl;
          for (int t = 0; t < L; ++t)
            my_tok[t] = t < wl ? (t < 3 ? W.tok[wa][t] : W.tok[wb][t]) : (uint8_t)0;
        }
      }
      out[(size_t)pi * E + e] = o;
    }
    __syncwarp();
  }
  }  // the logits / logic phase
  // ---- odd warps streamed their features after the sweep: apply the skip
  //      decisions now (a skipped set's outcome is replaced) and the similarity
  if (defer) {
    __syncwarp();
    for (int q = lane; q < P; q += 32) {
      const hsd_verify_params& pp = params[q];
      hsd_outcome* op = out + (size_t)q * E + e;
      if (skip_cond(pp) && cosv >= pp.min_S) {
        hsd_outcome o;
        o.accept_len = L;
        o.win_a = 0;
        o.win_b = 0;
        o.calls = 0;
        o.fallback = 0;
        o.skipped = 1;
        o.n_emit = (int16_t)L;
        o.greedy0 = (int16_t)W.greedy[0];
        o.cos_sim = (float)cosv;
        *op = o;
        uint8_t* my_tok = tok_out + ((size_t)q * E + e) * L;
        for (int t = 0; t < L; ++t) my_tok[t] = W.tok[0][t];
      } else {
        op->cos_sim = (float)cosv;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1024 / kThreads) verify_kernel(const int32_t* __restrict__ ids, int E, int k, int L,
                                                             const uint8_t* __restrict__ tokens,
                                                             const uint8_t* __restrict__ cand_tokens,
                                                             const float* __restrict__ logits,
                                                             const float* __restrict__ feat_now,
                                                             const float* __restrict__ feat_prev, int d_f,
                                                             const int32_t* __restrict__ history, int gap_d,
                                                             const hsd_verify_params* __restrict__ params, int P,
                                                             int need_cos, const double* __restrict__ cos_in,
                                                             hsd_outcome* __restrict__ out,
                                                             uint8_t* __restrict__ tok_out, int early) {
  __shared__ WarpScratch sw[kWarps];
  // early != 0: every input but the ids predates the previous kernel, so
  // verify_episode waits only before the ids (see there); the PDL trigger of
  // the previous grid then lets the logits / feature phases run under it
  if (!early) dev::pdl_wait();  // the retrieved ids (K2)
  dev::pdl_trigger();
  const int warp = threadIdx.x >> 5;
  const int e = blockIdx.x * kWarps + warp;
  if (e >= E) {
    if (early) dev::pdl_wait();  // no access, but no grid outlives its predecessor's inputs either
    return;
  }
  verify_episode(e, E, k, L, ids, tokens, cand_tokens, logits + (size_t)e * L * 256,
                 feat_now ? feat_now + (size_t)e * d_f : nullptr, feat_prev ? feat_prev + (size_t)e * d_f : nullptr,
                 d_f, history, gap_d, params, P, need_cos, cos_in, out, tok_out, sw[warp], early != 0);
}

// should_skip's similarity for every episode as its own pass: one CTA per
// episode, all 2 x d_f x 4 bytes in flight at once (8 float4 pairs per thread
// at d_f = 4096) instead of one warp's serial round trips.  Same exactly
// rounded double-double sum as verify_episode, so either path gives the same
// bits.
constexpr int kCosThreads = 128;
constexpr int kCosUnroll = 8;

__global__ void __launch_bounds__(kCosThreads) cos_kernel(const float* __restrict__ feat_now,
                                                          const float* __restrict__ feat_prev, int d_f,
                                                          double* __restrict__ cos_out) {
  const int e = blockIdx.x;
  const float4* a4 = reinterpret_cast<const float4*>(feat_now + (size_t)e * d_f);
  const float4* b4 = reinterpret_cast<const float4*>(feat_prev + (size_t)e * d_f);
  const int n4 = d_f / 4;
  double hi = 0.0, lo = 0.0;
  for (int t0 = threadIdx.x; t0 < n4; t0 += kCosThreads * kCosUnroll) {
    float4 xa[kCosUnroll], yb[kCosUnroll];
#pragma unroll
    for (int u = 0; u < kCosUnroll; ++u) {
      const int t = t0 + kCosThreads * u;
      xa[u] = t < n4 ? __ldcs(a4 + t) : make_float4(0.f, 0.f, 0.f, 0.f);
      yb[u] = t < n4 ? __ldcs(b4 + t) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kCosUnroll; ++u) {
      const double pr[4] = {(double)xa[u].x * (double)yb[u].x, (double)xa[u].y * (double)yb[u].y,
                            (double)xa[u].z * (double)yb[u].z, (double)xa[u].w * (double)yb[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double sm, er;
        dev::two_sum(hi, pr[i], sm, er);
        hi = sm;
        lo = __dadd_rn(lo, er);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ohi = __shfl_xor_sync(0xffffffffu, hi, o);
    const double olo = __shfl_xor_sync(0xffffffffu, lo, o);
    double sm, er;
    dev::two_sum(hi, ohi, sm, er);
    hi = sm;
    lo = __dadd_rn(__dadd_rn(lo, olo), er);
  }
  __shared__ double rh[kCosThreads / 32], rl[kCosThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    rh[threadIdx.x >> 5] = hi;
    rl[threadIdx.x >> 5] = lo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    hi = rh[0];
    lo = rl[0];
    for (int w = 1; w < kCosThreads / 32; ++w) {
      double sm, er;
      dev::two_sum(hi, rh[w], sm, er);
      hi = sm;
      lo = __dadd_rn(__dadd_rn(lo, rl[w]), er);
    }
    double sm, er;
    dev::two_sum(hi, lo, sm, er);
    cos_out[e] = sm;
  }
}

}  // namespace

cudaError_t launch_cos(const float* feat_now, const float* feat_prev, int E, int d_f, double* cos_out,
                       cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  cos_kernel<<<E, kCosThreads, 0, s>>>(feat_now, feat_prev, d_f, cos_out);
  return cudaGetLastError();
}

cudaError_t launch_verify(const int32_t* ids, int E, int k, int L, const uint8_t* tokens, const uint8_t* cand_tokens,
                          const float* logits, const float* feat_now, const float* feat_prev, int d_f,
                          const int32_t* history, int gap_d, const hsd_verify_params* params_dev, int P, int need_cos,
                          hsd_outcome* out, uint8_t* tok_out, cudaStream_t s, const double* cos_in, bool early) {
  if (E <= 0) return cudaSuccess;
  return launch_pdl(verify_kernel, dim3((E + kWarps - 1) / kWarps), dim3(kThreads), 0, s, ids, E, k, L, tokens,
                    cand_tokens, logits, feat_now, feat_prev, d_f, history, gap_d, params_dev, P, need_cos, cos_in, out,
                    tok_out, early ? 1 : 0);
}

// Pre-gather the payload tokens of a [n] id list (sharded search records).
__global__ void gather_tokens_kernel(const uint8_t* __restrict__ tokens, const int32_t* __restrict__ ids, int n,
                                     uint8_t* __restrict__ out) {
  const int i = blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8;
  const int w = threadIdx.x & 7;
  if (i >= n) return;
  const int id = ids[i];
  const uint32_t v = id >= 0 ? reinterpret_cast<const uint32_t*>(tokens + (size_t)id * HSD_TOKENS_STRIDE)[w] : 0u;
  reinterpret_cast<uint32_t*>(out + (size_t)i * HSD_TOKENS_STRIDE)[w] = v;
}

cudaError_t launch_gather_tokens(const uint8_t* tokens, const int32_t* ids, int n, uint8_t* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  gather_tokens_kernel<<<(n + 31) / 32, 256, 0, s>>>(tokens, ids, n, out);
  return cudaGetLastError();
}

}  // namespace hsd
