/*
 * hsd_synth.h — counter-based synthetic workload generators for the HeiSD
 * retrieval-side hot path (SURVEY.md §8(d) "Synthetic inputs").
 *
 * Every value is a pure function of (seed, stream tag, counter) and is built
 * from integer hashing plus IEEE operations that are correctly rounded on both
 * the host and the device (integer ops, +, *, /, sqrt; no libm transcendentals,
 * no FMA-contractible expressions).  The CUDA generator kernels and the CPU
 * oracle therefore produce bit-identical inputs without shipping 16 GB of keys
 * across PCIe.
 *
 * Two key families:
 *   HSD_SYNTH_EXACT : key = ((h mod 17) - 8) / 16.  Exact in bf16/TF32/fp32;
 *                     every dot product of two such vectors is exact in fp32 in
 *                     any summation order (|sum| <= 1024 in units of 2^-8), so
 *                     scores tie often and the (score desc, id asc) rule of
 *                     store.cpp:67-70 is exercised.  Every 997th row duplicates
 *                     its predecessor (forced exact ties).
 *   HSD_SYNTH_REAL  : Irwin-Hall(4) integer vector, L2-normalised exactly:
 *                     sum of squares in int64 (order-independent), sqrt and the
 *                     divide in fp64, then rounded once to fp32.
 *   HSD_SYNTH_CLUSTER: REAL rows, except that each 512-row block may open with
 *                     a run of 64-512 consecutive rows around one centre: a
 *                     near-duplicate run (64 * centre + noise, pairwise cosine
 *                     ~0.9999: the steps of a demonstration, SPEC.md:602,
 *                     608-613) or a run of identical rows (a stationary
 *                     segment).  Queries near such a run see hundreds of rows
 *                     within the filter's error window of the k-th score.
 *
 * This header is plain C99 and compiles as CUDA (__host__ __device__).
 */
#ifndef HSD_SYNTH_H
#define HSD_SYNTH_H

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define HSD_HD __host__ __device__ __forceinline__
#else
#define HSD_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HSD_SYNTH_EXACT = 0,
  HSD_SYNTH_REAL = 1,
  HSD_SYNTH_CLUSTER = 2,
};

/* stream tags */
enum {
  HSD_TAG_KEYS = 1,
  HSD_TAG_QUERY = 2,
  HSD_TAG_LOGITS = 3,
  HSD_TAG_TRAJ = 4,
  HSD_TAG_FEAT = 5,
  HSD_TAG_ACTIONS = 6,
  HSD_TAG_QNOISE = 7,
  HSD_TAG_QPICK = 8,
  HSD_TAG_POLICY = 9,
  HSD_TAG_ROBOT = 10,
  HSD_TAG_DRAFTER = 11,
};

/* Payload families of generated records (hsd_collection_generate_ex). */
enum {
  HSD_PAYLOAD_RANDOM = 0, /* next_actions uniform in [-1, 1) (hsd_action_val) */
  HSD_PAYLOAD_TRAJ = 1,   /* demonstration rows: row = e * T + j holds next_actions[s] = policy(e, j + s) */
};

HSD_HD uint64_t hsd_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Base of one (seed, tag) counter stream. */
HSD_HD uint64_t hsd_stream_base(uint64_t seed, uint32_t tag) {
  return hsd_splitmix64(seed * 0xD1342543DE82EF95ull + (uint64_t)tag * 0x2545F4914F6CDD1Dull);
}

HSD_HD uint64_t hsd_hash_at(uint64_t base, uint64_t idx) { return hsd_splitmix64(base ^ (idx * 0x9E3779B97F4A7C15ull)); }

/* Row that a DB row's key is generated from (duplicate rows, EXACT family). */
HSD_HD int64_t hsd_key_src_row(int kind, int64_t row) {
  if (kind == HSD_SYNTH_EXACT && row > 0 && (row % 997) == 996) return row - 1;
  return row;
}

/* Irwin-Hall(4) centred integer in [-131070, 131070]. */
HSD_HD int32_t hsd_ih4(uint64_t h) {
  int32_t s = (int32_t)(h & 0xFFFFu) + (int32_t)((h >> 16) & 0xFFFFu) + (int32_t)((h >> 32) & 0xFFFFu) +
              (int32_t)((h >> 48) & 0xFFFFu);
  return s - 131070;
}

/* EXACT-family element value. */
HSD_HD float hsd_exact_val(uint64_t h) { return (float)((int32_t)(h % 17u) - 8) * 0.0625f; }

/* REAL-family raw (un-normalised) integer of key (row, col). */
HSD_HD int32_t hsd_key_raw(uint64_t kbase, int64_t src_row, int dim, int col) {
  return hsd_ih4(hsd_hash_at(kbase, (uint64_t)src_row * (uint64_t)dim + (uint64_t)col));
}

/* CLUSTER family: block g = row / HSD_CLUSTER_BLOCK opens with a run of
 * hsd_cluster_len rows of kind hsd_cluster_type (0 none, 1 near-duplicate,
 * 2 identical). */
#define HSD_CLUSTER_BLOCK 512
HSD_HD uint64_t hsd_cluster_hash(uint64_t kbase, int64_t g) {
  return hsd_hash_at(kbase ^ 0xC2B2AE3D27D4EB4Full, (uint64_t)g);
}
HSD_HD int hsd_cluster_type(uint64_t kbase, int64_t g) {
  const uint32_t t = (uint32_t)(hsd_cluster_hash(kbase, g) & 3u);
  return t <= 1u ? 1 : (t == 2u ? 2 : 0);
}
HSD_HD int hsd_cluster_len(uint64_t kbase, int64_t g) {
  return 64 + (int)((hsd_cluster_hash(kbase, g) >> 8) % 449u);
}
/* Raw (un-normalised) integer of key (row, col) of family `kind` (REAL or
 * CLUSTER; |raw| < 2^24, so dim * raw^2 fits int64 for dim < 2^14). */
HSD_HD int64_t hsd_key_raw_kind(int kind, uint64_t kbase, int64_t row, int dim, int col) {
  if (kind == HSD_SYNTH_CLUSTER) {
    const int64_t g = row / HSD_CLUSTER_BLOCK, p = row % HSD_CLUSTER_BLOCK;
    const int type = hsd_cluster_type(kbase, g);
    if (type != 0 && p < hsd_cluster_len(kbase, g)) {
      const int64_t centre =
          hsd_ih4(hsd_hash_at(kbase ^ 0x165667B19E3779F9ull, (uint64_t)g * (uint64_t)dim + (uint64_t)col));
      if (type == 2) return centre;
      return 64 * centre + hsd_key_raw(kbase, row, dim, col);
    }
  }
  return hsd_key_raw(kbase, row, dim, col);
}

/* Exactly-rounded normalisation of one raw element given the int64 sum of squares. */
HSD_HD float hsd_norm_val(int64_t raw, int64_t sumsq) {
  double n = sqrt((double)sumsq);
  return (float)((double)raw / n);
}

/* ---- bf16 key storage (bf16 collections) ----------------------------------
 * fp32 -> bf16 round-to-nearest-even on the bit pattern (finite inputs; the
 * generators and insert reject non-finite values), identical on host and
 * device, and the exact widening back to fp32. */
HSD_HD uint16_t hsd_bf16_bits(float f) {
  union {
    float f;
    uint32_t u;
  } v;
  v.f = f;
  uint32_t u = v.u;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
HSD_HD float hsd_bf16_val(uint16_t b) {
  union {
    float f;
    uint32_t u;
  } v;
  v.u = (uint32_t)b << 16;
  return v.f;
}

/* ---- queries -------------------------------------------------------------
 * Query q of a batch is one of:
 *   EXACT: 25% an exact copy of DB row r (r hashed), else a fresh EXACT vector.
 *   REAL : 50% near-duplicate 3*raw_key(r) + noise (top-1 cosine ~0.95, in line
 *          with PAPER.md:852), else pure noise (random unit vector).
 * hsd_query_mode() returns the picked row for copy/near-dup queries, -1 else. */
HSD_HD int64_t hsd_query_row(uint64_t seed, int kind, int64_t q, int64_t n_rows) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_QPICK), (uint64_t)q);
  uint32_t sel = (uint32_t)(h & 0xFFu);
  int hit = (kind == HSD_SYNTH_EXACT) ? (sel < 64u) : (sel < 128u);
  if (!hit || n_rows <= 0) return -1;
  return (int64_t)((h >> 8) % (uint64_t)n_rows);
}

/* REAL / CLUSTER raw query element (needs the picked row).  Near-duplicate
 * queries of CLUSTER rows scale the noise like the row (64x inside a run). */
HSD_HD int64_t hsd_query_raw_kind(int kind, uint64_t seed, uint64_t db_seed, int64_t q, int64_t row, int dim,
                                  int col) {
  int64_t noise = hsd_ih4(hsd_hash_at(hsd_stream_base(seed, HSD_TAG_QNOISE), (uint64_t)q * (uint64_t)dim + col));
  if (row < 0) return noise;
  const uint64_t kbase = hsd_stream_base(db_seed, HSD_TAG_KEYS);
  int64_t k = hsd_key_raw_kind(kind, kbase, hsd_key_src_row(kind, row), dim, col);
  if (kind == HSD_SYNTH_CLUSTER) {
    const int64_t g = row / HSD_CLUSTER_BLOCK;
    if (hsd_cluster_type(kbase, g) == 1 && row % HSD_CLUSTER_BLOCK < hsd_cluster_len(kbase, g)) noise *= 64;
  }
  return 3 * k + noise;
}
HSD_HD int64_t hsd_query_raw(uint64_t seed, uint64_t db_seed, int64_t q, int64_t row, int dim, int col) {
  return hsd_query_raw_kind(HSD_SYNTH_REAL, seed, db_seed, q, row, dim, col);
}

/* EXACT-family query element. */
HSD_HD float hsd_query_exact(uint64_t seed, uint64_t db_seed, int64_t q, int64_t row, int dim, int col) {
  if (row >= 0)
    return hsd_exact_val(hsd_hash_at(hsd_stream_base(db_seed, HSD_TAG_KEYS),
                                     (uint64_t)hsd_key_src_row(HSD_SYNTH_EXACT, row) * (uint64_t)dim + col));
  return hsd_exact_val(hsd_hash_at(hsd_stream_base(seed, HSD_TAG_QNOISE), (uint64_t)q * (uint64_t)dim + col));
}

/* ---- payload actions (Payload::next_actions, store.hpp:31) ---------------
 * next_actions[s][j] for record `row`: uniform in [-1, 1) with ~1.2% of values
 * forced to the boundary (1.0) or outside the bounds (1.5, -1.25) so that the
 * clamp of actions.cpp:42 is exercised.  Exact doubles. */
HSD_HD double hsd_action_val(uint64_t seed, int64_t row, int s, int j) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_ACTIONS), (uint64_t)row * 21u + (uint64_t)(s * 7 + j));
  uint32_t sel = (uint32_t)(h & 0xFFu);
  if (sel == 0u) return 1.0;
  if (sel == 1u) return 1.5;
  if (sel == 2u) return -1.25;
  return (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

/* ---- verifier logits ------------------------------------------------------
 * logits[e][p][b] (fp32).  Background: multiples of 1/64 in [-2, 2).  The
 * greedy bin is draft_bin + delta with delta = 0 (50%), |delta| <= 15 (30%),
 * |delta| in [16, 64] (20%), clamped to [0, 255]; it gets 8.0.  1% of positions
 * get a second bin at exactly 8.0 (argmax tie -> lowest index wins). */
HSD_HD int hsd_logit_greedy_bin(uint64_t seed, int64_t e, int p, int draft_bin) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_LOGITS), ((uint64_t)e << 8) ^ (uint64_t)(0xF000u + p));
  uint32_t sel = (uint32_t)(h % 100u);
  int delta = 0;
  if (sel < 50u) {
    delta = 0;
  } else if (sel < 80u) {
    delta = (int)((h >> 8) % 31u) - 15;
  } else {
    int mag = 16 + (int)((h >> 8) % 49u);
    delta = ((h >> 20) & 1u) ? mag : -mag;
  }
  int g = draft_bin + delta;
  if (g < 0) g = 0;
  if (g > 255) g = 255;
  return g;
}

HSD_HD int hsd_logit_tie_bin(uint64_t seed, int64_t e, int p) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_LOGITS), ((uint64_t)e << 8) ^ (uint64_t)(0xE000u + p));
  if ((h % 100u) != 0u) return -1;
  return (int)((h >> 8) & 0xFFu);
}

HSD_HD float hsd_logit_background(uint64_t seed, int64_t e, int p, int b) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_LOGITS), ((uint64_t)e * 64u + (uint64_t)p) * 256u + (uint64_t)b);
  return (float)((int32_t)(h & 0xFFu) - 128) * 0.015625f;
}

/* ---- verifier features for the verify-skip check (Alg. 1) ----------------
 * f_now = normalise(IH4 noise); f_prev = normalise(a * raw_now + noise) with the
 * mixing weight a swept per episode in [1, 48] so cos(f_now, f_prev) straddles
 * typical min_S values (0.7 .. 0.9998). */
HSD_HD int32_t hsd_feat_mix(uint64_t seed, int64_t e) {
  uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_FEAT), (uint64_t)e ^ 0xABCDEF0000000000ull);
  return 1 + (int32_t)(h % 48u);
}

HSD_HD int64_t hsd_feat_raw(uint64_t seed, int64_t e, int which, int dim, int col) {
  uint64_t base = hsd_stream_base(seed, HSD_TAG_FEAT);
  int64_t now = hsd_ih4(hsd_hash_at(base, ((uint64_t)e * 2u) * (uint64_t)dim + (uint64_t)col));
  if (which == 0) return now;
  int64_t noise = hsd_ih4(hsd_hash_at(base, ((uint64_t)e * 2u + 1u) * (uint64_t)dim + (uint64_t)col));
  return (int64_t)hsd_feat_mix(seed, e) * now + noise;
}

/* ---- trajectory harness (config 5: the hybrid decoding loop) -------------
 * Stand-in for the SPEC harness (ToyEnv + OracleVLA +
 * recorded demonstrations).  Demonstration episode e follows a piecewise
 * policy of HSD_SEG_LEN-action segments that alternate
 *   transport (even segments): straight, fast (|v| <= 0.8), gripper open;
 *   approach  (odd segments) : the velocity turns by a fixed rational rotation
 *                              (cos, sin) = ((1-u^2)/(1+u^2), 2u/(1+u^2)) per
 *                              action in one axis plane, slow (|v| ~ 0.3),
 *                              gripper closed;
 * so the fused metric (kinematics.cpp) sees straight/fast windows (retrieval)
 * and tight slow arcs (drafter).  Values use +, *, / with explicit rounding
 * (no FMA contraction, no libm transcendentals): host and device agree bit for
 * bit.  Tokens are the reference quantize (actions.cpp:32-50) of the values. */
#define HSD_SEG_LEN 24
#define HSD_ENV_SCALE 0.01 /* ToyEnv: position += HSD_ENV_SCALE * dequantize(xyz bins) */

#if defined(__CUDA_ARCH__)
#define HSD_MUL(a, b) __dmul_rn((a), (b))
#define HSD_ADD(a, b) __dadd_rn((a), (b))
#define HSD_SUB(a, b) __dsub_rn((a), (b))
#define HSD_DIV(a, b) __ddiv_rn((a), (b))
#else
#define HSD_MUL(a, b) ((a) * (b))
#define HSD_ADD(a, b) ((a) + (b))
#define HSD_SUB(a, b) ((a) - (b))
#define HSD_DIV(a, b) ((a) / (b))
#endif

/* quantize of one value, actions.cpp:42-47 (bounds [lo, hi], K bins). */
HSD_HD int hsd_quantize_bin(double v, double lo, double hi, int k_bins) {
  const double c = v < lo ? lo : (hi < v ? hi : v);
  const double t = HSD_DIV(HSD_SUB(c, lo), HSD_SUB(hi, lo));
  int bin = (int)floor(HSD_MUL(t, (double)(k_bins - 1)));
  bin = bin < 0 ? 0 : bin;
  return bin > k_bins - 1 ? k_bins - 1 : bin;
}

/* dequantize of one bin, actions.cpp:60-63: lo + bin / (K - 1) * span. */
HSD_HD double hsd_dequantize_bin(int bin, double lo, double hi, int k_bins) {
  return HSD_ADD(lo, HSD_MUL(HSD_DIV((double)bin, (double)(k_bins - 1)), HSD_SUB(hi, lo)));
}

/* Policy action value of demonstration episode e at action index j, dim d. */
HSD_HD double hsd_policy_val(uint64_t seed, int64_t e, int64_t j, int d) {
  const int64_t seg = j / HSD_SEG_LEN;
  const int64_t jj = j - seg * HSD_SEG_LEN;
  const uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_POLICY), (uint64_t)e * 0x100000001B3ull + (uint64_t)seg);
  const int arc = (int)(seg & 1);
  if (d == 6) return arc ? 1.0 : -1.0; /* gripper closed while approaching */
  if (d >= 3) /* rotation: piecewise-constant small values */
    return HSD_MUL(0.0625, (double)((int)((h >> (8 * d)) % 5u) - 2));
  if (!arc) { /* transport: constant direction, components in [-0.8, 0.8) */
    return HSD_DIV((double)((int)((h >> (8 * d)) & 0xFFu) - 128), 160.0);
  }
  /* approach: rotate (cx, cy) by the rational angle of u, jj times */
  const int plane = (int)((h >> 24) % 3u); /* (0,1) (1,2) (0,2) */
  const int ax = plane == 1 ? 1 : 0, ay = plane == 0 ? 1 : 2;
  if (d != ax && d != ay) return 0.0;
  const double u = HSD_ADD(0.15, HSD_DIV((double)((h >> 32) & 0xFFu), 1700.0)); /* 0.15 .. 0.30 */
  const double u2 = HSD_MUL(u, u);
  const double den = HSD_ADD(1.0, u2);
  const double cr = HSD_DIV(HSD_SUB(1.0, u2), den), sr = HSD_DIV(HSD_MUL(2.0, u), den);
  const double w = HSD_SUB(HSD_DIV((double)((h >> 40) & 0xFFu), 127.5), 1.0); /* start angle parameter */
  const double w2 = HSD_MUL(w, w);
  double cx = HSD_DIV(HSD_SUB(1.0, w2), HSD_ADD(1.0, w2)), cy = HSD_DIV(HSD_MUL(2.0, w), HSD_ADD(1.0, w2));
  for (int64_t i = 0; i < jj; ++i) {
    const double nx = HSD_SUB(HSD_MUL(cr, cx), HSD_MUL(sr, cy));
    const double ny = HSD_ADD(HSD_MUL(sr, cx), HSD_MUL(cr, cy));
    cx = nx;
    cy = ny;
  }
  const double sp = HSD_ADD(0.25, HSD_DIV((double)((h >> 48) & 0xFFu), 2550.0)); /* 0.25 .. 0.35 */
  return HSD_MUL(sp, d == ax ? cx : cy);
}

HSD_HD int hsd_policy_token(uint64_t seed, int64_t e, int64_t j, int d) {
  return hsd_quantize_bin(hsd_policy_val(seed, e, j, d), -1.0, 1.0, 256);
}

/* Robot r of the hybrid loop: the demonstration episode it replays (>= n_demo
 * -> an episode absent from the DB: "unseen instance", ~1/8 of robots) and its
 * per-dim bin bias (1/4 of seen robots deviate by 1..6 bins on pos/rot dims:
 * inside the relaxed caps 30/15, rejected by strict acceptance). */
HSD_HD int64_t hsd_robot_episode(uint64_t seed, int64_t r, int64_t n_demo) {
  const uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_ROBOT), (uint64_t)r);
  if (n_demo <= 0 || (h & 7u) == 0u) return n_demo + (int64_t)((h >> 8) % 1000003u); /* unseen */
  return (int64_t)((h >> 8) % (uint64_t)n_demo);
}
HSD_HD int hsd_robot_bias(uint64_t seed, int64_t r, int d) {
  const uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_ROBOT), (uint64_t)r ^ 0x5A5A000000000000ull);
  if (d == 6 || (h & 3u) != 0u) return 0;
  const int mag = 1 + (int)((h >> (4 + 6 * d)) % 6u);
  return ((h >> (40 + d)) & 1u) ? mag : -mag;
}
/* Verifier (OracleVLA stand-in) greedy token of robot r (replaying episode e)
 * at action j, dim d: the policy token (policy_seed = the DB seed) plus the
 * robot's bias (robot_seed = the loop seed), clamped to [0, 255]. */
HSD_HD int hsd_robot_greedy(uint64_t policy_seed, uint64_t robot_seed, int64_t r, int64_t e, int64_t j, int d) {
  int t = hsd_policy_token(policy_seed, e, j, d) + hsd_robot_bias(robot_seed, r, d);
  return t < 0 ? 0 : (t > 255 ? 255 : t);
}
/* DB row a robot's retrieval query near-duplicates: its demonstration row
 * (e, j) when that row exists, else -1 (a query with no near neighbour). */
HSD_HD int64_t hsd_hybrid_query_row(int64_t e, int64_t j, int64_t T, int64_t n_demo, int64_t n_rows) {
  if (e < 0 || e >= n_demo || j < 0 || j >= T) return -1;
  const int64_t row = e * T + j;
  return row < n_rows ? row : -1;
}
/* ToyEnv start position of robot r (exact binary fractions in [-0.125, 0.125)). */
HSD_HD double hsd_robot_start(uint64_t seed, int64_t r, int d) {
  const uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_ROBOT), (uint64_t)r ^ 0xA5A5000000000000ull);
  return (double)((int)((h >> (8 * d)) & 0xFFu) - 128) / 1024.0;
}
/* Counter id of robot r's round-`round` query / features / logits streams. */
HSD_HD int64_t hsd_hybrid_qid(int64_t r, int64_t round) { return (r << 24) + round; }
/* Toy drafter: the verifier's greedy token with probability
 * p_pct/100, else a uniformly random different bin. */
HSD_HD int hsd_drafter_token(uint64_t seed, int64_t r, int64_t step, int p, int greedy, int p_pct) {
  const uint64_t h = hsd_hash_at(hsd_stream_base(seed, HSD_TAG_DRAFTER), ((uint64_t)r << 24) ^ ((uint64_t)step << 5) ^ (uint64_t)p);
  if ((int)(h % 100u) < p_pct) return greedy;
  return (greedy + 1 + (int)((h >> 8) % 255u)) & 255;
}

#ifdef __cplusplus
}
#endif

#endif /* HSD_SYNTH_H */
