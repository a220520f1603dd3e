// k_select.cu — K2 select (exact top-k from K1's filter lists) and K3 shard merge.
//
// K2 reproduces Collection::search_topk_exact (store.cpp:59-73) bit for bit
// from K1's per-list approximate top-32s.  Four launches per pass, chained by
// programmatic dependent launch:
//
//   select_cand  one CTA per query.
//     1. merge the per-list candidate lists (sorted u64 keys) into the global
//        approximate top-32; its first k rows are the filter's top-k;
//     2. threshold.  A parallel fp64 dot of those k rows (error ~dim 2^-53)
//        gives L, a lower bound of the reference's k-th best score S_k (k
//        distinct rows score at least L).  A row r of the reference's top-k
//        has s_r >= S_k >= L, so its filter score is >= T = L - E - delta,
//        E = gamma max|key| |q| (+ absolute underflow slack) the filter's
//        forward error bound (sim_wide_gamma), delta the fp64 slack.
//        T >= A_k - 2E always, and ~A_k - E in practice: half the window
//        of the plain A_k - 2E margin;
//     3. collect.  A list that still holds a row >= T in its last slot may
//        have dropped other rows >= T: the list goes to the range fallback
//        (its entries are not pooled).  Every other list contributes its
//        entries >= T.  If more than kCandMax such entries remain, every list
//        holding one goes to the fallback instead.
//   rescore      one CTA per (query, 8 or 32 pooled candidates): the
//                reference's arithmetic, cosine_similarity (store.cpp:29-34),
//                s += q[i] * k[i] sequentially in fp64 (bit-identical).
//   fallback     persistent; exit at once when no query needs it.  Otherwise
//                rescore EVERY row of each fallback list (32-row chunks, the
//                same fp64 chain) and merge each chunk into the query's exact
//                top-k under a per-query lock.  Exact for any input, however
//                many near-duplicates a list range holds.
//   rank         one CTA per query: order pooled + fallback rows by
//                (score desc, id asc) (store.cpp:67-70), truncate to k (:71).
//
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
constexpr int kCandMax = 256;   // pooled (rescored) candidates per query
constexpr int kMaxLists = 256;  // filter lists per pass (<= SMs)
constexpr int kPerWide = 32;    // candidates rescored per CTA (lanes of warp 0) from 9 queries up
constexpr int kPerNarrow = 8;   // ... and for 1-8 queries (more CTAs, more rows in flight)
constexpr int kRThreads = 128;  // rescoring CTA: all threads stage rows, warp 0 runs the fp64 chains
constexpr int kFbChunk = 32;    // fallback rows per chain round (lanes of warp 0)

__device__ __forceinline__ double widen(float x) { return (double)x; }
__device__ __forceinline__ double widen(uint16_t b) { return (double)hsd_bf16_val(b); }  // bf16 key -> exact fp64

// Per-query scratch between the K2 kernels.
struct SelScratch {
  uint32_t id[kCandMax];
  double exact[kCandMax];
  int n;       // pooled candidates
  int n_fb;    // fallback lists
  int lock;    // fallback merge lock
  int pad;
  uint16_t fb_list[kMaxLists];
  // exact top-k of the fallback rows, ascending (order key, id)
  uint64_t fb_key[dev::kCandLocal];
  uint32_t fb_id[dev::kCandLocal];
  double fb_score[dev::kCandLocal];
};

struct CandSmem {
  uint64_t top[kWarps][32];
  uint64_t pool[kCandMax];
  double red[kWarps];
  double fast[dev::kCandLocal];
  uint8_t cnt[kMaxLists];
  int pool_n;
  int n_fb;
  int above;  // entries >= T in non-exhausted lists
};

// Rows of filter list l (ListGeom, kernels.h): blocks first + j * stride,
// j < count, of 128 rows each (clipped to row_end).
struct ListRows {
  int64_t first, count;
};
__device__ __forceinline__ ListRows list_rows(const ListGeom& g, int l) {
  const int64_t nb = (g.row_end - g.row_begin + 127) / 128;
  ListRows r;
  if (g.stride == 1) {
    r.first = (int64_t)l * g.per;
    r.count = max((int64_t)0, min(g.per, nb - r.first));
  } else {  // CTA pairs: list 2u + h walks blocks blk0 + h, blk0 + h + 2, ... of unit u's range
    const int64_t blk0 = (int64_t)(l >> 1) * g.per, blk1 = min(blk0 + g.per, nb);
    r.first = blk0 + (l & 1);
    r.count = r.first < blk1 ? (blk1 - r.first + 1) / 2 : 0;
  }
  return r;
}

// Parallel fp64 dot of one stored row with the query (one warp): every
// product is exact in fp64, the sum carries <= (dim/32 + 5) roundings.
template <typename KT>
__device__ __forceinline__ double warp_dot(const KT* __restrict__ row, const float* __restrict__ q, int dim, int lane) {
  double acc = 0.0;
  if constexpr (sizeof(KT) == 4) {
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const int n4 = dim / 4;
    for (int i0 = lane; i0 < n4; i0 += 32 * 4) {
      float4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u;
        a[u] = i < n4 ? __ldg(r4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
        b[u] = i < n4 ? __ldg(q4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc = __fma_rn((double)a[u].x, (double)b[u].x, acc);
        acc = __fma_rn((double)a[u].y, (double)b[u].y, acc);
        acc = __fma_rn((double)a[u].z, (double)b[u].z, acc);
        acc = __fma_rn((double)a[u].w, (double)b[u].w, acc);
      }
    }
  } else {  // bf16 keys, dim % 8 == 0
    const uint4* r8 = reinterpret_cast<const uint4*>(row);
    const float4* q4 = reinterpret_cast<const float4*>(q);
    const int n8 = dim / 8;
    for (int i0 = lane; i0 < n8; i0 += 32 * 2) {
      uint4 a[2];
      float4 b[4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = i0 + 32 * u;
        a[u] = i < n8 ? __ldg(r8 + i) : make_uint4(0, 0, 0, 0);
        b[2 * u] = i < n8 ? __ldg(q4 + 2 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
        b[2 * u + 1] = i < n8 ? __ldg(q4 + 2 * i + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const uint32_t w[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
        const float qv[8] = {b[2 * u].x, b[2 * u].y, b[2 * u].z, b[2 * u].w,
                             b[2 * u + 1].x, b[2 * u + 1].y, b[2 * u + 1].z, b[2 * u + 1].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          acc = __fma_rn((double)hsd_bf16_val((uint16_t)(w[t] & 0xFFFFu)), (double)qv[2 * t], acc);
          acc = __fma_rn((double)hsd_bf16_val((uint16_t)(w[t] >> 16)), (double)qv[2 * t + 1], acc);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// K2a, one CTA per query (see the file header).
template <typename KT>
__global__ void __launch_bounds__(kThreads) select_cand_kernel(const uint64_t* __restrict__ partial, int lists, int B,
                                                               int k, int dim, const float* __restrict__ queries,
                                                               const KT* __restrict__ keys,
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
    S.n_fb = 0;
    S.above = 0;
  }
  __syncthreads();
  if (warp == 0) {
    uint64_t t = S.top[0][lane];
    for (int w = 1; w < kWarps; ++w) t = dev::warp_merge_top32(t, S.top[w][lane]);
    S.top[0][lane] = t;
  }
  __syncthreads();
  const uint64_t kth = S.top[0][k - 1];
  // fp64 dots of the filter's top-k rows -> L (lower bound of the k-th exact score)
  if (kth != kEmpty)
    for (int r = warp; r < k; r += kWarps) {
      const double d = warp_dot(keys + (size_t)cand_id(S.top[0][r]) * dim, qrow, dim, lane);
      if (lane == 0) S.fast[r] = d;
    }
  __syncthreads();
  double qn2 = 0.0;
  for (int w = 0; w < kWarps; ++w) qn2 += S.red[w];
  const double qn = sqrt(qn2) * 1.000001;
  const double mn = __longlong_as_double((long long)*maxnorm_bits) * 1.000001;
  // filter error vs the real dot: relative (gamma) + absolute (subnormal
  // rounding / flush-to-zero of products and accumulators)
  const double E = gamma * mn * qn + (dim + 16.0) * 0x1p-124 * (1.0 + mn + qn);
  // fp64 slack: the parallel dot and the reference's sequential sum each
  // differ from the real dot by <= (dim + 64) 2^-53 max|k| |q|
  const double delta = 4.0 * (dim + 64.0) * 0x1p-53 * mn * qn + 0x1p-1000;
  double T = -INFINITY;
  if (kth != kEmpty) {
    double L = S.fast[0];
    for (int r = 1; r < k; ++r) L = fmin(L, S.fast[r]);
    T = L - E - delta;
  }

  // count the entries >= T of every list; exhausted lists go to the fallback
  for (int l = tid; l < lists; l += kThreads) {
    const uint64_t* lst = partial + ((size_t)l * B + b) * kCandLocal;
    int j = 0;
    for (; j < kCandLocal; ++j) {
      const uint64_t key = lst[j];
      if (key == kEmpty || (double)cand_score(key) < T) break;
    }
    S.cnt[l] = (uint8_t)j;
    if (j < kCandLocal && j > 0) atomicAdd(&S.above, j);
  }
  __syncthreads();
  const bool all_fb = S.above > kCandMax;  // too many to pool: every list with a candidate goes to the fallback
  SelScratch& o = scr[b];
  for (int l = tid; l < lists; l += kThreads) {
    const int j = S.cnt[l];
    if (j == kCandLocal || (all_fb && j > 0)) {
      o.fb_list[atomicAdd(&S.n_fb, 1)] = (uint16_t)l;
    } else if (j > 0) {
      const uint64_t* lst = partial + ((size_t)l * B + b) * kCandLocal;
      const int slot = atomicAdd(&S.pool_n, j);
      for (int i = 0; i < j; ++i) S.pool[slot + i] = lst[i];
    }
  }
  __syncthreads();
  const int n = S.pool_n;
  for (int i = tid; i < n; i += kThreads) o.id[i] = cand_id(S.pool[i]);
  if (tid < kCandLocal) {
    o.fb_key[tid] = kEmpty;
    o.fb_id[tid] = 0xFFFFFFFFu;
  }
  if (tid == 0) {
    o.n = n;
    o.n_fb = S.n_fb;
    o.lock = 0;
  }
}

// Exact rescoring of `n` <= kPer rows (ids in smem) against one query, in the
// reference's order (store.cpp:32): acc = fma(q_i, k_i, acc), i = 0..dim-1, in
// fp64 — the fp32 (or bf16) x fp32 product is exact in fp64, so the fused form
// is bit-identical to s += a[i]*b[i].  Returns lane c's (c < n) score in warp 0.
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
__device__ __forceinline__ double rescore_rows(const KT* __restrict__ keys, int dim, const float* __restrict__ qrow,
                                               const uint32_t* ids, int n, uint8_t* smem_raw) {
  constexpr int kPad = 16 / (int)sizeof(KT);
  constexpr int kStride = kW + kPad;
  auto& rows = *reinterpret_cast<KT(*)[2][kPer][kStride]>(smem_raw);
  auto& qs = *reinterpret_cast<float(*)[2][kW]>(smem_raw + sizeof(KT) * 2 * kPer * kStride);
  auto& qd = *reinterpret_cast<double(*)[kW]>(smem_raw + sizeof(KT) * 2 * kPer * kStride + sizeof(float) * 2 * kW);
  const int tid = threadIdx.x;
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
  return acc;
}

// K2b, one CTA per (query, kPer pooled candidates).
template <typename KT, int kPer>
__global__ void __launch_bounds__(kRThreads) rescore_kernel(const KT* __restrict__ keys, int dim,
                                                            const float* __restrict__ queries,
                                                            SelScratch* __restrict__ scr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ uint32_t ids[kPer];
  dev::pdl_wait();  // the candidate lists
  const int b = blockIdx.x, c0 = blockIdx.y * kPer;
  SelScratch& o = scr[b];
  const int n = min(o.n - c0, kPer);
  if (n <= 0) return;
  const int tid = threadIdx.x;
  if (tid < n) ids[tid] = o.id[c0 + tid];
  __syncthreads();
  const double acc = rescore_rows<KT, kPer>(keys, dim, queries + (size_t)b * dim, ids, n, smem_raw);
  // the fallback kernel (next) needs this kernel's shared memory: let it
  // launch only as the chains finish
  dev::pdl_trigger();
  if (tid < n) o.exact[c0 + tid] = acc;
}

// Lexicographic (order key, id) "better than" (score desc, id asc).
__device__ __forceinline__ bool better(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// K2c, fallback: exact rescoring of every row of the lists select_cand could
// not bound (see the file header).  Work units = (query, fallback list,
// 32-row chunk), spread over a persistent grid.
template <typename KT>
__global__ void __launch_bounds__(kRThreads) fallback_kernel(const KT* __restrict__ keys, int dim,
                                                             const float* __restrict__ queries, int B, int k,
                                                             ListGeom g, SelScratch* __restrict__ scr) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __shared__ int pre[kMaxBatchPass + 1];  // prefix of fallback lists over the pass's queries
  __shared__ uint32_t ids[kFbChunk];
  dev::pdl_wait();
  dev::pdl_trigger();
  const int tid = threadIdx.x, lane = tid & 31;
  // CTA-wide exclusive scan of n_fb over the B queries (B <= kMaxBatchPass)
  constexpr int kPerT = (kMaxBatchPass + kRThreads - 1) / kRThreads;
  int v[kPerT], run = 0;
#pragma unroll
  for (int u = 0; u < kPerT; ++u) {
    const int q = tid * kPerT + u;
    v[u] = q < B ? scr[q].n_fb : 0;
    run += v[u];
  }
  __shared__ int wsum[kRThreads / 32];
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[tid >> 5] = incl;
  __syncthreads();
  int base = incl - run;
  for (int w = 0; w < (tid >> 5); ++w) base += wsum[w];
  int total = 0;
  for (int w = 0; w < kRThreads / 32; ++w) total += wsum[w];
  if (total == 0) return;  // the common case: every query bounded by the pooled candidates
#pragma unroll
  for (int u = 0; u < kPerT; ++u) {
    const int q = tid * kPerT + u;
    if (q <= kMaxBatchPass) pre[q] = base;
    base += v[u];
  }
  if (tid == kRThreads - 1) pre[kMaxBatchPass] = total;
  __syncthreads();
  const int64_t U = 4 * ((g.per + g.stride - 1) / g.stride);  // 32-row chunks per list (upper bound)
  const int64_t units = (int64_t)total * U;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int item = (int)(u / U);
    const int64_t c = u - (int64_t)item * U;
    int lo = 0, hi = B;  // query b: pre[b] <= item < pre[b + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= item) lo = mid; else hi = mid;
    }
    const int b = lo;
    SelScratch& o = scr[b];
    const ListRows lr = list_rows(g, o.fb_list[item - pre[b]]);
    const int64_t j = c / 4;
    if (j >= lr.count) continue;
    const int64_t row0 = g.row_begin + (lr.first + j * g.stride) * 128 + (c % 4) * kFbChunk;
    const int n = (int)min((int64_t)kFbChunk, g.row_end - row0);
    if (n <= 0) continue;
    if (tid < n) ids[tid] = (uint32_t)(row0 + tid);
    __syncthreads();
    const double s = rescore_rows<KT, kFbChunk>(keys, dim, queries + (size_t)b * dim, ids, n, smem_raw);
    if (tid < 32) {
      uint64_t mk = lane < n ? dev::score_desc_key(s) : kEmpty;
      uint32_t mi = lane < n ? ids[lane] : 0xFFFFFFFFu;
      // skip the lock when no row beats the current k-th (it only improves)
      const uint64_t kk = *(volatile uint64_t*)&o.fb_key[k - 1];
      const uint32_t ki = *(volatile uint32_t*)&o.fb_id[k - 1];
      if (__any_sync(0xffffffffu, lane < n && better(mk, mi, kk, ki))) {
        if (lane == 0)
          while (atomicCAS(&o.lock, 0, 1) != 0) __nanosleep(64);
        __syncwarp();
        __threadfence();
        const uint64_t ok = lane < k ? __ldcg(&o.fb_key[lane]) : kEmpty;
        const uint32_t oi = lane < k ? __ldcg(&o.fb_id[lane]) : 0xFFFFFFFFu;
        const double os = lane < k ? __ldcg(&o.fb_score[lane]) : 0.0;
        // rank of each entry in the union (old k sorted + 32 new)
        int r_old = lane, r_new = 0;
        for (int t = 0; t < 32; ++t) {
          const uint64_t xk = dev::shfl_u64(mk, t);
          const uint32_t xi = __shfl_sync(0xffffffffu, mi, t);
          const uint64_t yk = dev::shfl_u64(ok, t);
          const uint32_t yi = __shfl_sync(0xffffffffu, oi, t);
          r_old += better(xk, xi, ok, oi);
          r_new += better(xk, xi, mk, mi) + better(yk, yi, mk, mi);
        }
        __syncwarp();
        if (lane < k && ok != kEmpty && r_old < k) {
          o.fb_key[r_old] = ok;
          o.fb_id[r_old] = oi;
          o.fb_score[r_old] = os;
        }
        if (lane < n && r_new < k) {
          o.fb_key[r_new] = mk;
          o.fb_id[r_new] = mi;
          o.fb_score[r_new] = s;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(&o.lock, 0);
      }
    }
    __syncthreads();  // ids / staging reuse
  }
}

// K2d, one CTA per query: rank pooled + fallback rows by (score desc, id asc)
// and emit the first k (store.cpp:67-71).
// With a publish descriptor (sharded search over peer memory) the final
// records go straight into every peer's receive window — global id, fp64
// score and the 32-byte draft tokens — followed by the per-query flag: the
// local top-k and the exchange are one kernel.
constexpr int kRankMax = kCandMax + dev::kCandLocal;
__global__ void __launch_bounds__(kThreads) rank_kernel(const SelScratch* __restrict__ scr, int k,
                                                        double* __restrict__ scores, int32_t* __restrict__ ids,
                                                        int* __restrict__ stats, P2PPublish pub, int publish) {
  // integer order keys: the branch-free 64-bit compare loop runs in half the
  // time of the fp64 (x > s) || (x == s && ...) form (6 vs 12 us at n ~ 100)
  __shared__ uint64_t key[kRankMax];
  __shared__ uint32_t id[kRankMax];
  __shared__ double sc[kRankMax];
  __shared__ int nfb;
  dev::pdl_wait();  // the exact scores
  dev::pdl_trigger();
  const int b = blockIdx.x, tid = threadIdx.x;
  const SelScratch& o = scr[b];
  const int np = o.n;
  if (tid == 0) {
    int c = 0;
    while (c < k && o.fb_key[c] != kEmpty) ++c;
    nfb = c;
  }
  for (int i = tid; i < np; i += kThreads) {
    sc[i] = o.exact[i];
    key[i] = dev::score_desc_key(sc[i]);
    id[i] = o.id[i];
  }
  __syncthreads();
  const int n = np + nfb;
  if (tid < nfb) {
    sc[np + tid] = o.fb_score[tid];
    key[np + tid] = o.fb_key[tid];
    id[np + tid] = o.fb_id[tid];
  }
  __syncthreads();
  for (int i = tid; i < n; i += kThreads) {
    const uint64_t mk = key[i];
    const uint32_t me = id[i];
    int rank = 0;
#pragma unroll 8
    for (int c = 0; c < n; ++c) {
      const uint64_t x = key[c];
      rank += (x < mk) | ((x == mk) & (id[c] < me));
    }
    if (rank < k) {
      const double s = sc[i];
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
  if (tid == 0) {
    if (o.n_fb) atomicAdd(&stats[0], 1);
    atomicAdd(&stats[1], np);
    atomicAdd(&stats[2], o.n_fb);
  }
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

template <typename KT>
cudaError_t select_typed(const uint64_t* partial, int lists, int B, int k, const KT* keys, int dim,
                         const float* queries, const unsigned long long* maxnorm_bits, double gamma,
                         const ListGeom& geom, double* scores, int32_t* ids, int* stats, SelScratch* scr, int fb_grid,
                         cudaStream_t s, const P2PPublish* pub) {
  cudaError_t e = launch_pdl(select_cand_kernel<KT>, dim3(B), dim3(kThreads), 0, s, partial, lists, B, k, dim,
                             queries, keys, maxnorm_bits, gamma, scr);
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
    e = attrs(rescore_kernel<KT, kPerWide>, rescore_smem<KT, kPerWide>());
    if (e == cudaSuccess) e = attrs(rescore_kernel<KT, kPerNarrow>, rescore_smem<KT, kPerNarrow>());
    if (e == cudaSuccess) e = attrs(fallback_kernel<KT>, rescore_smem<KT, kFbChunk>());
    if (e != cudaSuccess) return e;
    configured.fetch_or(1ull << dev);
  }
  if (B <= 8)
    e = launch_pdl(rescore_kernel<KT, kPerNarrow>, dim3(B, kCandMax / kPerNarrow), dim3(kRThreads),
                   rescore_smem<KT, kPerNarrow>(), s, keys, dim, queries, scr);
  else
    e = launch_pdl(rescore_kernel<KT, kPerWide>, dim3(B, kCandMax / kPerWide), dim3(kRThreads),
                   rescore_smem<KT, kPerWide>(), s, keys, dim, queries, scr);
  if (e != cudaSuccess) return e;
  e = launch_pdl(fallback_kernel<KT>, dim3(fb_grid), dim3(kRThreads), rescore_smem<KT, kFbChunk>(), s, keys, dim,
                 queries, B, k, geom, scr);
  if (e != cudaSuccess) return e;
  P2PPublish pb{};
  if (pub) pb = *pub;
  return launch_pdl(rank_kernel, dim3(B), dim3(kThreads), 0, s, scr, k, scores, ids, stats, pb, pub ? 1 : 0);
}

// Pooled candidates from an external filter (the IVF index, k_ivf.cu): one
// CTA per query copies the valid entries of pool[b][0..C) (u64 candidate
// keys: the filter's approximate order, global row ids) into the per-query
// scratch the rescoring and rank kernels read; no fallback lists.
__global__ void __launch_bounds__(kThreads) pool_kernel(const uint64_t* __restrict__ pool, int C,
                                                        SelScratch* __restrict__ scr) {
  __shared__ int n;
  dev::pdl_wait();
  dev::pdl_trigger();
  const int b = blockIdx.x, tid = threadIdx.x;
  SelScratch& o = scr[b];
  if (tid == 0) n = 0;
  __syncthreads();
  for (int i = tid; i < C; i += kThreads) {
    const uint64_t key = pool[(size_t)b * C + i];
    if (key != kEmpty) o.id[atomicAdd(&n, 1)] = cand_id(key);
  }
  if (tid < dev::kCandLocal) {
    o.fb_key[tid] = kEmpty;
    o.fb_id[tid] = 0xFFFFFFFFu;
  }
  __syncthreads();
  if (tid == 0) {
    o.n = n;
    o.n_fb = 0;
    o.lock = 0;
  }
}

template <typename KT>
cudaError_t rescore_pool_typed(const uint64_t* pool, int C, int B, int k, const KT* keys, int dim,
                               const float* queries, double* scores, int32_t* ids, int* stats, SelScratch* scr,
                               cudaStream_t s) {
  cudaError_t e = launch_pdl(pool_kernel, dim3(B), dim3(kThreads), 0, s, pool, C, scr);
  if (e != cudaSuccess) return e;
  const size_t smem = rescore_smem<KT, kPerNarrow>();
  e = cudaFuncSetAttribute(rescore_kernel<KT, kPerNarrow>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // C <= 32 candidates per query: (C / 8) CTAs of 8 chains each
  e = launch_pdl(rescore_kernel<KT, kPerNarrow>, dim3(B, (C + kPerNarrow - 1) / kPerNarrow), dim3(kRThreads), smem, s,
                 keys, dim, queries, scr);
  if (e != cudaSuccess) return e;
  return launch_pdl(rank_kernel, dim3(B), dim3(kThreads), 0, s, (const SelScratch*)scr, k, scores, ids, stats,
                    P2PPublish{}, 0);
}

}  // namespace

size_t select_scratch_bytes(int B) { return (size_t)B * sizeof(SelScratch); }
int select_max_lists() { return kMaxLists; }

cudaError_t launch_select(const uint64_t* partial, int lists, int B, int k, const void* keys, int key_dtype, int dim,
                          const float* queries, const unsigned long long* maxnorm_bits, double gamma,
                          const ListGeom& geom, double* scores, int32_t* ids, int* stats, void* scratch, int num_sms,
                          cudaStream_t s, const P2PPublish* pub) {
  if (B <= 0) return cudaSuccess;
  if (B > kMaxBatchPass || lists > kMaxLists || k > dev::kCandLocal) return cudaErrorInvalidValue;
  if (key_dtype == HSD_DTYPE_BF16 && dim % 8) return cudaErrorInvalidValue;
  SelScratch* scr = reinterpret_cast<SelScratch*>(scratch);
  const int fb_grid = 2 * num_sms;
  if (key_dtype == HSD_DTYPE_BF16)
    return select_typed(partial, lists, B, k, (const uint16_t*)keys, dim, queries, maxnorm_bits, gamma, geom, scores,
                        ids, stats, scr, fb_grid, s, pub);
  return select_typed(partial, lists, B, k, (const float*)keys, dim, queries, maxnorm_bits, gamma, geom, scores, ids,
                      stats, scr, fb_grid, s, pub);
}

cudaError_t launch_rescore_pool(const uint64_t* pool, int C, int B, int k, const void* keys, int key_dtype, int dim,
                                const float* queries, double* scores, int32_t* ids, int* stats, void* scratch,
                                cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (B > kMaxBatchPass || C < 1 || C > dev::kCandLocal || k > dev::kCandLocal) return cudaErrorInvalidValue;
  if (key_dtype == HSD_DTYPE_BF16 && dim % 8) return cudaErrorInvalidValue;
  SelScratch* scr = reinterpret_cast<SelScratch*>(scratch);
  if (key_dtype == HSD_DTYPE_BF16)
    return rescore_pool_typed(pool, C, B, k, (const uint16_t*)keys, dim, queries, scores, ids, stats, scr, s);
  return rescore_pool_typed(pool, C, B, k, (const float*)keys, dim, queries, scores, ids, stats, scr, s);
}

cudaError_t launch_merge_ranks(const double* g_scores, const int32_t* g_ids, const uint8_t* g_tok, int G, int B, int k,
                               double* scores, int32_t* ids, uint8_t* tok, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  merge_ranks_kernel<<<B, 256, 0, s>>>(g_scores, g_ids, g_tok, G, B, k, scores, ids, tok);
  return cudaGetLastError();
}

}  // namespace hsd
