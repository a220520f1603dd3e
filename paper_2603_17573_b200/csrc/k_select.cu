// k_select.cu — K2 select and K3 shard merge.
//
// K2, one CTA per query:
//   1. merge the per-CTA candidate lists (sorted u64 keys) into the global
//      approximate top-32 (warp bitonic merges) -> A_k, the k-th best approx
//      score;
//   2. margin: every record whose EXACT score can reach the exact k-th score
//      has approx >= A_k - 2E, E = gamma * max|key| * |q| (forward error bound
//      of the approximate path).  Collect all such candidates; flag overflow
//      if a per-CTA list was exhausted above the margin;
//   3. rescore the candidates with the reference's arithmetic — cosine_similarity
//      (store.cpp:29-34): s += q[i] * k[i] sequentially in fp64 — so scores are
//      bit-identical to the reference;
//   4. order (score desc, id asc) (store.cpp:67-70), truncate to k (:71).
// K3: k-way merge of G ranks' exact top-k lists (multi-GPU all-gather result).
#include "common.cuh"
#include "hsd/hsd_synth.h"
#include "kernels.h"

namespace hsd {
namespace {

using dev::cand_id;
using dev::cand_score;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPool = 512;
constexpr int kCandMax = 256;  // rescored candidates (one thread each)
// Rescoring staging ring: 2 buffers of n rows x (W + 4) floats (16-B aligned
// rows for cp.async, +4 floats spreads rows over banks), W = 512 for n <= 32,
// 64 for n <= 256.
constexpr int kRowsFloats = 2 * 256 * (64 + 4);  // >= 2 * 32 * (512 + 4)
static_assert(kRowsFloats >= 2 * 32 * (512 + 4), "staging ring too small");
constexpr int kMaxW = 512;

__device__ __forceinline__ double widen(float x) { return (double)x; }
__device__ __forceinline__ double widen(uint16_t b) { return (double)hsd_bf16_val(b); }  // bf16 key -> exact fp64

struct SelectSmem {
  uint64_t top[kWarps][32];
  uint64_t pool[kPool];
  __align__(16) float rows[kRowsFloats];  // staging ring, reinterpreted as KT
  __align__(16) double q[2][kMaxW];
  double exact[kCandMax];
  uint32_t id[kCandMax];
  double red[kWarps];
  int pool_n;
  int over;
};

template <typename KT>  // float (fp32 collection) or uint16_t (bf16 bits)
__global__ void __launch_bounds__(kThreads) select_kernel(const uint64_t* __restrict__ partial, int lists, int B, int k,
                                                          const KT* __restrict__ keys, int dim,
                                                          const float* __restrict__ queries,
                                                          const unsigned long long* __restrict__ maxnorm_bits,
                                                          double gamma, double* __restrict__ scores,
                                                          int32_t* __restrict__ ids, int* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SelectSmem& S = *reinterpret_cast<SelectSmem*>(smem_raw);
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* qrow = queries + (size_t)b * dim;

  // 1. approximate global top-32 (4 list loads in flight per warp)
  uint64_t top = kEmpty;
  for (int l0 = warp; l0 < lists; l0 += 4 * kWarps) {
    uint64_t x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int l = l0 + u * kWarps;
      x[u] = l < lists ? partial[((size_t)l * B + b) * kCandLocal + lane] : kEmpty;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) top = dev::warp_merge_top32(top, x[u]);
  }
  S.top[warp][lane] = top;
  double qq = 0.0;
  for (int i = tid; i < dim; i += kThreads) qq += (double)qrow[i] * (double)qrow[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  if (lane == 0) S.red[warp] = qq;
  if (tid == 0) {
    S.pool_n = 0;
    S.over = 0;
  }
  __syncthreads();
  if (warp == 0) {
    uint64_t t = S.top[0][lane];
    for (int w = 1; w < kWarps; ++w) t = dev::warp_merge_top32(t, S.top[w][lane]);
    S.top[0][lane] = t;
  }
  __syncthreads();
  double qn2 = 0.0;
  for (int w = 0; w < kWarps; ++w) qn2 += S.red[w];
  const uint64_t kth = S.top[0][k - 1];
  const double maxnorm = __longlong_as_double((long long)*maxnorm_bits);
  const double E = gamma * maxnorm * sqrt(qn2) * 1.000001 + 1e-300;
  const double T = (kth == kEmpty) ? -INFINITY : (double)cand_score(kth) - 2.0 * E;

  // 2. margin candidates
  for (int l = tid; l < lists; l += kThreads) {
    const uint64_t* lst = partial + ((size_t)l * B + b) * kCandLocal;
    int j = 0;
    for (; j < kCandLocal; ++j) {
      const uint64_t key = lst[j];
      if (key == kEmpty || (double)cand_score(key) < T) break;
      const int slot = atomicAdd(&S.pool_n, 1);
      if (slot < kPool) S.pool[slot] = key;
    }
    if (j == kCandLocal) S.over = 1;  // list exhausted above the margin
  }
  __syncthreads();
  int n = S.pool_n;
  if (n > kPool) {
    n = kPool;
    if (tid == 0) S.over = 1;
  }
  if (n > kCandMax) {  // keep the best kCandMax by approximate score
    if (warp == 0) {
      uint64_t v[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) v[s] = s * 32 + lane < n ? S.pool[s * 32 + lane] : kEmpty;
      dev::warp_sort<16>(v);
#pragma unroll
      for (int s = 0; s < 8; ++s) S.pool[s * 32 + lane] = v[s];
    }
    n = kCandMax;
    if (tid == 0) S.over = 1;
  }
  __syncthreads();
  if (tid < n) S.id[tid] = cand_id(S.pool[tid]);
  __syncthreads();

  // 3. exact rescoring in the reference's order.  Candidate rows stream
  //    through a double-buffered cp.async ring of wide column chunks (the
  //    next chunk lands while this one is consumed); each thread then runs
  //    the sequential fp64 chain of its candidate out of shared memory.
  // widest chunk (in elements) whose double buffer fits; rows are padded by
  // 16 B (spreads them over banks, keeps cp.async destinations aligned)
  constexpr int kPad = 16 / (int)sizeof(KT);
  constexpr int kRingElems = kRowsFloats * 4 / (int)sizeof(KT);
  const int W = 2 * n * (kMaxW + kPad) <= kRingElems ? kMaxW
                : 2 * n * (256 + kPad) <= kRingElems ? 256
                : 2 * n * (128 + kPad) <= kRingElems ? 128
                                                     : 64;
  const int stride = W + kPad;
  const int nchunk = (dim + W - 1) / W;
  const int v16 = W / kPad;  // 16-B copies per row chunk
  KT* ring = reinterpret_cast<KT*>(S.rows);
  auto issue = [&](int ch) {
    KT* dst = ring + (ch & 1) * n * stride;
    const int c0 = ch * W;
    for (int i = tid; i < n * v16; i += kThreads) {
      const int c = i / v16, j16 = i - c * v16;
      const int col = c0 + j16 * kPad;
      const KT* src = keys + (size_t)S.id[c] * dim + col;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + c * stride + j16 * kPad);
      const int bytes = col < dim ? 16 : 0;  // dim is a multiple of kPad; zero-fill past the end
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
    }
    for (int j = tid; j < W; j += kThreads) S.q[ch & 1][j] = c0 + j < dim ? (double)qrow[c0 + j] : 0.0;
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc = 0.0;
  issue(0);
  for (int ch = 0; ch < nchunk; ++ch) {
    if (ch + 1 < nchunk) {
      issue(ch + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int w = dim - ch * W < W ? dim - ch * W : W;
    if (tid < n) {
      // acc = fl(acc + fl(q*k)) of store.cpp:32; the fp32 x fp32 (or fp32 x
      // bf16) product is exact in fp64, so the fused form fl(acc + q*k) is
      // bit-identical and leaves one dependent op per element on the chain.
      const KT* r = ring + (ch & 1) * n * stride + tid * stride;
      const double* qc = S.q[ch & 1];
#pragma unroll 16
      for (int j = 0; j < w; ++j) acc = __fma_rn(qc[j], widen(r[j]), acc);
    }
    __syncthreads();
  }
  if (tid < n) S.exact[tid] = acc;
  __syncthreads();

  // 4. rank by (score desc, id asc) and emit the first k
  if (tid < n) {
    const double s = S.exact[tid];
    const uint32_t me = S.id[tid];
    int rank = 0;
    for (int c = 0; c < n; ++c) {
      const double o = S.exact[c];
      rank += (o > s) || (o == s && S.id[c] < me);
    }
    if (rank < k) {
      scores[(size_t)b * k + rank] = s;
      ids[(size_t)b * k + rank] = (int32_t)me;
    }
  }
  for (int r = n + tid; r < k; r += kThreads) {
    scores[(size_t)b * k + r] = -INFINITY;
    ids[(size_t)b * k + r] = -1;
  }
  if (tid == 0 && S.over) atomicAdd(overflow, 1);
}

// K3: G sorted lists [G][B][k] -> global [B][k].
__global__ void merge_ranks_kernel(const double* __restrict__ gs, const int32_t* __restrict__ gi,
                                   const uint8_t* __restrict__ gt, int G, int B, int k, double* __restrict__ scores,
                                   int32_t* __restrict__ ids, uint8_t* __restrict__ tok) {
  const int b = blockIdx.x;
  const int n = G * k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int g = i / k, j = i % k;
    const int32_t me = gi[((size_t)g * B + b) * k + j];
    if (me < 0) continue;
    const double s = gs[((size_t)g * B + b) * k + j];
    int rank = 0;
    for (int c = 0; c < n; ++c) {
      const int gg = c / k, jj = c % k;
      const int32_t o = gi[((size_t)gg * B + b) * k + jj];
      if (o < 0) continue;
      const double os = gs[((size_t)gg * B + b) * k + jj];
      rank += (os > s) || (os == s && o < me);
    }
    if (rank < k) {
      scores[(size_t)b * k + rank] = s;
      ids[(size_t)b * k + rank] = me;
      if (tok) {
        const uint4* src = reinterpret_cast<const uint4*>(gt + (((size_t)g * B + b) * k + j) * HSD_TOKENS_STRIDE);
        uint4* dst = reinterpret_cast<uint4*>(tok + ((size_t)b * k + rank) * HSD_TOKENS_STRIDE);
        dst[0] = src[0];
        dst[1] = src[1];
      }
    }
  }
  // ranks beyond the number of valid entries
  __shared__ int valid;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (gi[((size_t)(i / k) * B + b) * k + (i % k)] >= 0) atomicAdd(&valid, 1);
  __syncthreads();
  for (int r = valid + threadIdx.x; r < k; r += blockDim.x) {
    scores[(size_t)b * k + r] = -INFINITY;
    ids[(size_t)b * k + r] = -1;
  }
}

}  // namespace

cudaError_t launch_select(const uint64_t* partial, int lists, int B, int k, const void* keys, int key_dtype, int dim,
                          const float* queries, const unsigned long long* maxnorm_bits, double gamma, double* scores,
                          int32_t* ids, int* overflow, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  const size_t smem = sizeof(SelectSmem);
  if (key_dtype == HSD_DTYPE_BF16) {
    if (dim % 8) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(select_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    select_kernel<uint16_t><<<B, kThreads, smem, s>>>(partial, lists, B, k, (const uint16_t*)keys, dim, queries,
                                                      maxnorm_bits, gamma, scores, ids, overflow);
  } else {
    cudaError_t e = cudaFuncSetAttribute(select_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    select_kernel<float><<<B, kThreads, smem, s>>>(partial, lists, B, k, (const float*)keys, dim, queries,
                                                   maxnorm_bits, gamma, scores, ids, overflow);
  }
  return cudaGetLastError();
}

cudaError_t launch_merge_ranks(const double* g_scores, const int32_t* g_ids, const uint8_t* g_tok, int G, int B, int k,
                               double* scores, int32_t* ids, uint8_t* tok, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  merge_ranks_kernel<<<B, 256, 0, s>>>(g_scores, g_ids, g_tok, G, B, k, scores, ids, tok);
  return cudaGetLastError();
}

}  // namespace hsd
