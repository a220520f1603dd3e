// k_synth.cu — K0: counter-based synthetic DB / query / logit / feature
// generation on the device (bit-identical to the host formulas in
// include/hsd/hsd_synth.h), the device quantizer (actions.cpp:32-50) and the
// per-row norm pass feeding the top-k error bound.
#include <cub/block/block_reduce.cuh>

#include <algorithm>

#include "common.cuh"
#include "hsd/hsd_synth.h"
#include "kernels.h"

namespace hsd {
namespace {

constexpr int kGenThreads = 256;

// quantize one value, actions.cpp:36-48 (IEEE ops, no contraction)
__device__ __forceinline__ int quantize_one(double v, double lo, double hi, int k_bins) {
  const double clamped = v < lo ? lo : (hi < v ? hi : v);
  const double t = __ddiv_rn(__dsub_rn(clamped, lo), __dsub_rn(hi, lo));
  int bin = (int)floor(__dmul_rn(t, (double)(k_bins - 1)));
  bin = bin < 0 ? 0 : bin;
  bin = bin > k_bins - 1 ? k_bins - 1 : bin;
  return bin;
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* bits, double v) {
  atomicMax(bits, (unsigned long long)__double_as_longlong(v));
}

// Stored key element: fp32 as generated, or bf16 (RN-even) for bf16 collections.
__device__ __forceinline__ float store_key(float* p, float v) {
  *p = v;
  return v;
}
__device__ __forceinline__ float store_key(uint16_t* p, float v) {
  const uint16_t b = hsd_bf16_bits(v);
  *p = b;
  return hsd_bf16_val(b);
}

// One CTA per DB row: key row (EXACT or exactly-normalised REAL), the norm of
// the stored row, and the 21 payload tokens quantize(next_actions[s]).
template <typename KT>
__global__ void __launch_bounds__(kGenThreads) gen_keys_kernel(int kind, uint64_t db_seed, int64_t row0, int dim,
                                                               KT* __restrict__ keys, uint8_t* __restrict__ tokens,
                                                               unsigned long long* maxnorm_bits, int payload,
                                                               int traj_T) {
  using BR = cub::BlockReduce<long long, kGenThreads>;
  using BRD = cub::BlockReduce<double, kGenThreads>;
  __shared__ union {
    typename BR::TempStorage i;
    typename BRD::TempStorage d;
  } tmp;
  __shared__ long long s_ss;
  const int64_t row = row0 + blockIdx.x;
  const int64_t src = hsd_key_src_row(kind, row);
  const uint64_t kbase = hsd_stream_base(db_seed, HSD_TAG_KEYS);
  KT* out = keys + (size_t)blockIdx.x * (size_t)dim;
  double nrm2 = 0.0;
  if (kind == HSD_SYNTH_EXACT) {
    for (int c = threadIdx.x; c < dim; c += kGenThreads) {
      const float v = store_key(out + c, hsd_exact_val(hsd_hash_at(kbase, (uint64_t)src * (uint64_t)dim + c)));
      nrm2 += (double)v * (double)v;
    }
  } else {
    long long ss = 0;
    for (int c = threadIdx.x; c < dim; c += kGenThreads) {
      long long r = hsd_key_raw_kind(kind, kbase, src, dim, c);
      ss += r * r;
    }
    ss = BR(tmp.i).Sum(ss);
    if (threadIdx.x == 0) s_ss = ss;
    __syncthreads();
    ss = s_ss;
    for (int c = threadIdx.x; c < dim; c += kGenThreads) {
      const float v = store_key(out + c, hsd_norm_val(hsd_key_raw_kind(kind, kbase, src, dim, c), ss));
      nrm2 += (double)v * (double)v;
    }
    __syncthreads();
  }
  nrm2 = BRD(tmp.d).Sum(nrm2);
  if (threadIdx.x == 0) atomic_max_nonneg(maxnorm_bits, sqrt(nrm2));
  if (threadIdx.x < HSD_TOKENS_STRIDE) {
    uint8_t t = 0;
    if (threadIdx.x < 21) {
      const int s = threadIdx.x / 7, j = threadIdx.x % 7;
      if (payload == HSD_PAYLOAD_TRAJ)  // demonstration row (e, jj): next_actions[s] = policy(e, jj + s)
        t = (uint8_t)hsd_policy_token(db_seed, row / traj_T, row % traj_T + s, j);
      else
        t = (uint8_t)quantize_one(hsd_action_val(db_seed, row, s, j), -1.0, 1.0, 256);
    }
    tokens[(size_t)blockIdx.x * HSD_TOKENS_STRIDE + threadIdx.x] = t;
  }
}

__device__ __forceinline__ double key_val(float x) { return (double)x; }
__device__ __forceinline__ double key_val(uint16_t b) { return (double)hsd_bf16_val(b); }

template <typename KT>
__global__ void __launch_bounds__(kGenThreads) row_norm_kernel(const KT* __restrict__ keys, int dim,
                                                               unsigned long long* maxnorm_bits) {
  using BRD = cub::BlockReduce<double, kGenThreads>;
  __shared__ typename BRD::TempStorage tmp;
  const KT* r = keys + (size_t)blockIdx.x * (size_t)dim;
  double s = 0.0;
  for (int c = threadIdx.x; c < dim; c += kGenThreads) s += key_val(r[c]) * key_val(r[c]);
  s = BRD(tmp).Sum(s);
  if (threadIdx.x == 0) atomic_max_nonneg(maxnorm_bits, sqrt(s));
}

__global__ void __launch_bounds__(kGenThreads) gen_queries_kernel(int kind, uint64_t q_seed, uint64_t db_seed,
                                                                  int64_t n_rows, int64_t q0, int dim,
                                                                  float* __restrict__ out) {
  using BR = cub::BlockReduce<long long, kGenThreads>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ long long s_ss;
  const int64_t q = q0 + blockIdx.x;
  const int64_t row = hsd_query_row(q_seed, kind, q, n_rows);
  float* o = out + (size_t)blockIdx.x * (size_t)dim;
  if (kind == HSD_SYNTH_EXACT) {
    for (int c = threadIdx.x; c < dim; c += kGenThreads) o[c] = hsd_query_exact(q_seed, db_seed, q, row, dim, c);
    return;
  }
  long long ss = 0;
  for (int c = threadIdx.x; c < dim; c += kGenThreads) {
    long long r = hsd_query_raw_kind(kind, q_seed, db_seed, q, row, dim, c);
    ss += r * r;
  }
  ss = BR(tmp).Sum(ss);
  if (threadIdx.x == 0) s_ss = ss;
  __syncthreads();
  ss = s_ss;
  for (int c = threadIdx.x; c < dim; c += kGenThreads)
    o[c] = hsd_norm_val(hsd_query_raw_kind(kind, q_seed, db_seed, q, row, dim, c), ss);
}

// One CTA per (episode, position): 256 threads = 256 bins.
__global__ void __launch_bounds__(256) gen_logits_kernel(const uint8_t* __restrict__ tokens, uint64_t seed,
                                                         const int64_t* __restrict__ rows, int L,
                                                         float* __restrict__ out) {
  const int e = blockIdx.x / L, p = blockIdx.x % L;
  const int64_t row = rows ? rows[e] : -1;
  int draft;
  if (row >= 0) {
    draft = tokens[(size_t)row * HSD_TOKENS_STRIDE + p];
  } else {
    draft = (int)(hsd_hash_at(hsd_stream_base(seed, HSD_TAG_LOGITS), ((uint64_t)e << 8) ^ (0xD000u + p)) & 0xFFu);
  }
  const int g = hsd_logit_greedy_bin(seed, e, p, draft);
  const int tie = hsd_logit_tie_bin(seed, e, p);
  const int b = threadIdx.x;
  const float v = (b == g || b == tie) ? 8.0f : hsd_logit_background(seed, e, p, b);
  out[(size_t)blockIdx.x * 256 + b] = v;
}

// One CTA per (episode, which): which 0 = f_now, 1 = f_prev.
__global__ void __launch_bounds__(kGenThreads) gen_features_kernel(uint64_t seed, int d_f, float* __restrict__ now,
                                                                   float* __restrict__ prev) {
  using BR = cub::BlockReduce<long long, kGenThreads>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ long long s_ss;
  const int64_t e = blockIdx.x >> 1;
  const int which = blockIdx.x & 1;
  long long ss = 0;
  for (int c = threadIdx.x; c < d_f; c += kGenThreads) {
    long long r = hsd_feat_raw(seed, e, which, d_f, c);
    ss += r * r;
  }
  ss = BR(tmp).Sum(ss);
  if (threadIdx.x == 0) s_ss = ss;
  __syncthreads();
  ss = s_ss;
  float* o = (which ? prev : now) + (size_t)e * d_f;
  for (int c = threadIdx.x; c < d_f; c += kGenThreads) o[c] = hsd_norm_val(hsd_feat_raw(seed, e, which, d_f, c), ss);
}

__global__ void quantize_kernel(const double* __restrict__ a, int64_t n, const double* __restrict__ lohi, int k_bins,
                                int32_t* __restrict__ bins, int32_t* __restrict__ status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int bad = 0;
  int out[7];
#pragma unroll
  for (int d = 0; d < 7; ++d) {
    const double v = a[i * 7 + d];
    if (!isfinite(v)) bad = 1;
    out[d] = quantize_one(v, lohi[d], lohi[7 + d], k_bins);
  }
#pragma unroll
  for (int d = 0; d < 7; ++d) bins[i * 7 + d] = bad ? 0 : out[d];
  if (status) status[i] = bad;
}

__global__ void quantize_tokens_kernel(const double* __restrict__ a, int64_t n, uint8_t* __restrict__ tokens,
                                       int32_t* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int j = threadIdx.x & 31;
  if (i >= n) return;
  uint8_t t = 0;
  if (j < 21) {
    const double v = a[i * 21 + j];
    if (!isfinite(v)) atomicExch(bad, 1);
    t = (uint8_t)quantize_one(v, -1.0, 1.0, 256);
  }
  tokens[i * HSD_TOKENS_STRIDE + j] = t;
}

}  // namespace

cudaError_t launch_gen_keys(int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim, void* keys, int key_dtype,
                            uint8_t* tokens, unsigned long long* maxnorm_bits, int payload, int traj_T,
                            cudaStream_t s) {
  constexpr int64_t kChunk = 1 << 20;
  for (int64_t r = 0; r < n; r += kChunk) {
    const int64_t m = n - r < kChunk ? n - r : kChunk;
    if (key_dtype == HSD_DTYPE_BF16)
      gen_keys_kernel<uint16_t><<<(unsigned)m, kGenThreads, 0, s>>>(
          kind, db_seed, row0 + r, dim, (uint16_t*)keys + (size_t)r * dim, tokens + (size_t)r * HSD_TOKENS_STRIDE,
          maxnorm_bits, payload, traj_T);
    else
      gen_keys_kernel<float><<<(unsigned)m, kGenThreads, 0, s>>>(
          kind, db_seed, row0 + r, dim, (float*)keys + (size_t)r * dim, tokens + (size_t)r * HSD_TOKENS_STRIDE,
          maxnorm_bits, payload, traj_T);
  }
  return cudaGetLastError();
}

cudaError_t launch_row_norms(const void* keys, int key_dtype, int64_t row0, int64_t n, int dim,
                             unsigned long long* maxnorm_bits, cudaStream_t s) {
  constexpr int64_t kChunk = 1 << 20;
  for (int64_t r = 0; r < n; r += kChunk) {
    const int64_t m = n - r < kChunk ? n - r : kChunk;
    if (key_dtype == HSD_DTYPE_BF16)
      row_norm_kernel<uint16_t><<<(unsigned)m, kGenThreads, 0, s>>>((const uint16_t*)keys + (size_t)(row0 + r) * dim,
                                                                   dim, maxnorm_bits);
    else
      row_norm_kernel<float><<<(unsigned)m, kGenThreads, 0, s>>>((const float*)keys + (size_t)(row0 + r) * dim, dim,
                                                                maxnorm_bits);
  }
  return cudaGetLastError();
}

// fp32 -> bf16 (RN-even, hsd_bf16_bits) of n elements (bf16 collection insert).
__global__ void to_bf16_kernel(const float* __restrict__ in, int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hsd_bf16_bits(in[i]);
}

cudaError_t launch_to_bf16(const float* in, int64_t n, uint16_t* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  to_bf16_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_queries(int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B, int dim,
                               float* out, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  gen_queries_kernel<<<B, kGenThreads, 0, s>>>(kind, q_seed, db_seed, n_rows, q0, dim, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_logits(const uint8_t* tokens, uint64_t seed, const int64_t* rows, int E, int L, float* out,
                              cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  gen_logits_kernel<<<E * L, 256, 0, s>>>(tokens, seed, rows, L, out);
  return cudaGetLastError();
}

cudaError_t launch_gen_features(uint64_t seed, int E, int d_f, float* now, float* prev, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  gen_features_kernel<<<2 * E, kGenThreads, 0, s>>>(seed, d_f, now, prev);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const double* actions, int64_t n, const double* lohi_dev, int k_bins, int32_t* bins,
                            int32_t* status, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  quantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(actions, n, lohi_dev, k_bins, bins, status);
  return cudaGetLastError();
}

cudaError_t launch_quantize_tokens(const double* actions, int64_t n, uint8_t* tokens, int32_t* bad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  quantize_tokens_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(actions, n, tokens, bad);
  return cudaGetLastError();
}

}  // namespace hsd
