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

#include <atomic>
#include "p2p.cuh"

namespace hsd {
namespace {

using dev::cand_id;
using dev::cand_score;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPool = 512;
constexpr int kCandMax = 256;   // rescored candidates per query
constexpr int kPerWide = 32;    // candidates rescored per CTA (lanes of warp 0) from 9 queries up
constexpr int kPerNarrow = 8;   // ... and for 1-8 queries (more CTAs, more rows in flight)
constexpr int kRThreads = 128;  // rescoring CTA: all threads stage rows, warp 0 runs the fp64 chains

__device__ __forceinline__ double widen(float x) { return (double)x; }
__device__ __forceinline__ double widen(uint16_t b) { return (double)hsd_bf16_val(b); }  // bf16 key -> exact fp64

// Per-query scratch between the three K2 kernels.
struct SelScratch {
  uint32_t id[kCandMax];
  double exact[kCandMax];
  int n;
  int over;
};

struct CandSmem {
  uint64_t top[kWarps][32];
  uint64_t pool[kPool];
  double red[kWarps];
  int pool_n;
  int over;
};

// K2a, one CTA per query: approximate global top-32 of the per-CTA lists ->
// A_k; every record whose exact score can reach the exact k-th has approx >=
// A_k - 2E (E = gamma * max|key| * |q|): collect them (best kCandMax by
// approximate score), flag an overflow if a per-CTA list ran out above the
// margin.
__global__ void __launch_bounds__(kThreads) select_cand_kernel(const uint64_t* __restrict__ partial, int lists, int B,
                                                               int k, int dim, const float* __restrict__ queries,
                                                               const unsigned long long* __restrict__ maxnorm_bits,
                                                               double gamma, SelScratch* __restrict__ scr) {
  __shared__ CandSmem S;
  dev::pdl_wait();  // K1's partial lists
  dev::pdl_trigger();
  const int b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* qrow = queries + (size_t)b * dim;

  // kListBatch list loads in flight per warp: the merge is latency-bound on
  // these L2 round trips (~18 lists per warp at 144 lists)
  constexpr int kListBatch = 8;
  uint64_t top = kEmpty;
  for (int l0 = warp; l0 < lists; l0 += kListBatch * kWarps) {
    uint64_t x[kListBatch];
#pragma unroll
    for (int u = 0; u < kListBatch; ++u) {
      const int l = l0 + u * kWarps;
      x[u] = l < lists ? partial[((size_t)l * B + b) * kCandLocal + lane] : kEmpty;
    }
#pragma unroll
    for (int u = 0; u < kListBatch; ++u) top = dev::warp_merge_top32(top, x[u]);
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
  SelScratch& o = scr[b];
  if (tid < n) o.id[tid] = cand_id(S.pool[tid]);
  if (tid == 0) {
    o.n = n;
    o.over = S.over;
  }
}

// K2b, one CTA per (query, kPer candidates): exact rescoring in the
// reference's order (store.cpp:32): acc = fma(q_i, k_i, acc), i = 0..dim-1, in
// fp64 — the fp32 (or bf16) x fp32 product is exact in fp64, so the fused form
// is bit-identical to s += a[i]*b[i].
// Rows and the query stream through a double-buffered cp.async ring of
// kW-element chunks (all 128 threads copy); the query chunk is widened to fp64
// once per chunk CTA-wide; lane c of warp 0 runs candidate c's chain with the
// operands of the next kPipe steps loaded ahead of the current kPipe DFMAs.
// Shape (tools/rescore_lab.cu, config-2 shape, L2 flushed): 32 chains per CTA
// run at 52 us where 8 chains per CTA took 90-110 us — the chain's per-step
// F2F widening and DFMA are issued per warp instruction, so full warps of
// chains cost 4x fewer issue slots per SM than quarter-filled ones.  At 1-8
// queries the SMs are idle anyway, and 8 chains per CTA (more CTAs, more rows
// in flight) measured 41.5 us against 47.5 us for 32 (100 candidates).
constexpr int kW = 256;    // elements per chunk
constexpr int kPipe = 8;   // chain steps whose operands are loaded ahead

template <typename KT, int kPer>
constexpr size_t rescore_smem() {
  return sizeof(KT) * 2 * kPer * (kW + 16 / sizeof(KT)) + sizeof(float) * 2 * kW + sizeof(double) * kW;
}

template <typename KT, int kPer>
__global__ void __launch_bounds__(kRThreads) rescore_kernel(const KT* __restrict__ keys, int dim,
                                                            const float* __restrict__ queries,
                                                            SelScratch* __restrict__ scr) {
  constexpr int kPad = 16 / (int)sizeof(KT);
  constexpr int kStride = kW + kPad;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  auto& rows = *reinterpret_cast<KT(*)[2][kPer][kStride]>(smem_raw);
  auto& qs = *reinterpret_cast<float(*)[2][kW]>(smem_raw + sizeof(KT) * 2 * kPer * kStride);
  auto& qd = *reinterpret_cast<double(*)[kW]>(smem_raw + sizeof(KT) * 2 * kPer * kStride + sizeof(float) * 2 * kW);
  __shared__ uint32_t ids[kPer];
  dev::pdl_wait();  // the candidate lists
  dev::pdl_trigger();
  const int b = blockIdx.x, c0 = blockIdx.y * kPer;
  SelScratch& o = scr[b];
  const int n = min(o.n - c0, kPer);
  if (n <= 0) return;
  const int tid = threadIdx.x;
  if (tid < n) ids[tid] = o.id[c0 + tid];
  __syncthreads();
  const float* qrow = queries + (size_t)b * dim;
  const int nchunk = (dim + kW - 1) / kW;
  constexpr int v16 = kW / kPad;  // 16-B copies per row chunk
  auto issue = [&](int ch) {
    const int cbase = ch * kW;
    for (int i = tid; i < n * v16; i += kRThreads) {
      const int c = i / v16, j16 = i - c * v16;
      const int col = cbase + j16 * kPad;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(&rows[ch & 1][c][j16 * kPad]);
      const int bytes = col < dim ? 16 : 0;  // dim is a multiple of kPad; zero-fill past the end
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(keys + (size_t)ids[c] * dim + col),
                   "r"(bytes)
                   : "memory");
    }
    for (int j4 = tid; j4 < kW / 4; j4 += kRThreads) {
      const int col = cbase + j4 * 4;
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(&qs[ch & 1][j4 * 4]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(qrow + col), "r"(col < dim ? 16 : 0)
                   : "memory");
    }
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
    for (int j = tid; j < kW; j += kRThreads) qd[j] = (double)qs[ch & 1][j];
    __syncthreads();
    const int w = min(dim - ch * kW, kW);
    if (tid < n) {
      const KT* r = rows[ch & 1][tid];
      if (w == kW) {
        double qa[kPipe], ra[kPipe];
#pragma unroll
        for (int u = 0; u < kPipe; ++u) {
          qa[u] = qd[u];
          ra[u] = widen(r[u]);
        }
        for (int j = 0; j < kW; j += kPipe) {
          double qb[kPipe], rb[kPipe];
          const int jn = j + kPipe < kW ? j + kPipe : j;
#pragma unroll
          for (int u = 0; u < kPipe; ++u) {
            qb[u] = qd[jn + u];
            rb[u] = widen(r[jn + u]);
          }
#pragma unroll
          for (int u = 0; u < kPipe; ++u) acc = __fma_rn(qa[u], ra[u], acc);
#pragma unroll
          for (int u = 0; u < kPipe; ++u) {
            qa[u] = qb[u];
            ra[u] = rb[u];
          }
        }
      } else {
#pragma unroll 16
        for (int j = 0; j < w; ++j) acc = __fma_rn(qd[j], widen(r[j]), acc);
      }
    }
    __syncthreads();
  }
  if (tid < n) o.exact[c0 + tid] = acc;
}

// K2c, one CTA per query: rank by (score desc, id asc) and emit the first k
// (store.cpp:67-71).
// With a publish descriptor (sharded search over peer memory) the final
// records go straight into every peer's receive window — global id, fp64
// score and the 32-byte draft tokens — followed by the per-query flag: the
// local top-k and the exchange are one kernel.
__global__ void __launch_bounds__(kThreads) rank_kernel(const SelScratch* __restrict__ scr, int k,
                                                        double* __restrict__ scores, int32_t* __restrict__ ids,
                                                        int* __restrict__ overflow, P2PPublish pub, int publish) {
  // integer order keys: the branch-free 64-bit compare loop runs in half the
  // time of the fp64 (x > s) || (x == s && ...) form (6 vs 12 us at n ~ 100)
  __shared__ uint64_t key[kCandMax];
  __shared__ uint32_t id[kCandMax];
  dev::pdl_wait();  // the exact scores
  dev::pdl_trigger();
  const int b = blockIdx.x, tid = threadIdx.x;
  const SelScratch& o = scr[b];
  const int n = o.n;
  double s = 0.0;
  uint32_t me = 0;
  uint64_t mk = 0;
  if (tid < n) {
    s = o.exact[tid];
    me = o.id[tid];
    mk = dev::score_desc_key(s);
    key[tid] = mk;
    id[tid] = me;
  }
  __syncthreads();
  if (tid < n) {
    int rank = 0;
#pragma unroll 8
    for (int c = 0; c < n; ++c) {
      const uint64_t x = key[c];
      rank += (x < mk) | ((x == mk) & (id[c] < me));
    }
    if (rank < k) {
      if (publish) {
        const int qb = pub.q_offset + b;
        for (int g = 0; g < pub.G; ++g)
          p2p_put_record(pub.w, g, pub.rank, pub.G, qb, rank, pub.epoch, s, (int32_t)(me + pub.id_offset),
                         pub.tokens + (size_t)me * HSD_TOKENS_STRIDE);
      } else {
        scores[(size_t)b * k + rank] = s;
        ids[(size_t)b * k + rank] = (int32_t)me;
      }
    }
  }
  for (int r = n + tid; r < k; r += kThreads) {
    if (publish) {
      for (int g = 0; g < pub.G; ++g)
        p2p_put_record(pub.w, g, pub.rank, pub.G, pub.q_offset + b, r, pub.epoch, -INFINITY, -1, nullptr);
    } else {
      scores[(size_t)b * k + r] = -INFINITY;
      ids[(size_t)b * k + r] = -1;
    }
  }
  if (publish) {
    __syncthreads();
    if (tid < pub.G) p2p_put_flag(pub.w, tid, pub.rank, pub.G, pub.q_offset + b, pub.epoch);
  }
  if (tid == 0 && o.over) atomicAdd(overflow, 1);
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

size_t select_scratch_bytes(int B) { return (size_t)B * sizeof(SelScratch); }

cudaError_t launch_select(const uint64_t* partial, int lists, int B, int k, const void* keys, int key_dtype, int dim,
                          const float* queries, const unsigned long long* maxnorm_bits, double gamma, double* scores,
                          int32_t* ids, int* overflow, void* scratch, cudaStream_t s, const P2PPublish* pub) {
  if (B <= 0) return cudaSuccess;
  if (key_dtype == HSD_DTYPE_BF16 && dim % 8) return cudaErrorInvalidValue;
  SelScratch* scr = reinterpret_cast<SelScratch*>(scratch);
  cudaError_t e = launch_pdl(select_cand_kernel, dim3(B), dim3(kThreads), 0, s, partial, lists, B, k, dim, queries,
                             maxnorm_bits, gamma, scr);
  if (e != cudaSuccess) return e;
  // function attributes are per device: set them once for each device used
  // (the kernels' occupancy is set by shared memory: ask for the full carveout)
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  cudaGetDevice(&dev);
  auto attrs = [](auto kern, size_t smem) {
    cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return r;
  };
  if (dev < 64 && !(configured.load() >> dev & 1)) {
    e = attrs(rescore_kernel<uint16_t, kPerWide>, rescore_smem<uint16_t, kPerWide>());
    if (e == cudaSuccess) e = attrs(rescore_kernel<float, kPerWide>, rescore_smem<float, kPerWide>());
    if (e == cudaSuccess) e = attrs(rescore_kernel<uint16_t, kPerNarrow>, rescore_smem<uint16_t, kPerNarrow>());
    if (e == cudaSuccess) e = attrs(rescore_kernel<float, kPerNarrow>, rescore_smem<float, kPerNarrow>());
    if (e != cudaSuccess) return e;
    configured.fetch_or(1ull << dev);
  }
  auto go = [&](auto kern, size_t smem, int per, const auto* kp) {
    return launch_pdl(kern, dim3(B, kCandMax / per), dim3(kRThreads), smem, s, kp, dim, queries, scr);
  };
  const bool narrow = B <= 8;
  if (key_dtype == HSD_DTYPE_BF16)
    e = narrow ? go(rescore_kernel<uint16_t, kPerNarrow>, rescore_smem<uint16_t, kPerNarrow>(), kPerNarrow,
                    (const uint16_t*)keys)
               : go(rescore_kernel<uint16_t, kPerWide>, rescore_smem<uint16_t, kPerWide>(), kPerWide,
                    (const uint16_t*)keys);
  else
    e = narrow ? go(rescore_kernel<float, kPerNarrow>, rescore_smem<float, kPerNarrow>(), kPerNarrow,
                    (const float*)keys)
               : go(rescore_kernel<float, kPerWide>, rescore_smem<float, kPerWide>(), kPerWide, (const float*)keys);
  if (e != cudaSuccess) return e;
  P2PPublish pb{};
  if (pub) pb = *pub;
  return launch_pdl(rank_kernel, dim3(B), dim3(kThreads), 0, s, scr, k, scores, ids, overflow, pb, pub ? 1 : 0);
}

cudaError_t launch_merge_ranks(const double* g_scores, const int32_t* g_ids, const uint8_t* g_tok, int G, int B, int k,
                               double* scores, int32_t* ids, uint8_t* tok, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  merge_ranks_kernel<<<B, 256, 0, s>>>(g_scores, g_ids, g_tok, G, B, k, scores, ids, tok);
  return cudaGetLastError();
}

}  // namespace hsd
