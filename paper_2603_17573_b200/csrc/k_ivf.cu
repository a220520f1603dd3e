// k_ivf.cu — the approximate device index: an inverted
// file (IVF-flat) over the collection's keys, standing in for the reference's
// HNSW graph (hnsw.cpp:58-169) behind Collection::build_hnsw / search_topk
// (store.cpp:75-92).
//
// Why IVF and not a graph on a B200: a graph walk is a chain of dependent
// 16-KB row fetches (one hop per L2/HBM round trip), while an inverted list
// is a contiguous run of rows that streams at HBM rate with coalesced 128-bit
// loads.  Probing p of L lists reads p/L of the DB per query.
//
// Device layout (api.cu builds it):
//   centroids  fp32 [nlist][dim], unit norm (spherical k-means)
//   offs       int32 [nlist + 1]   list l = positions [offs[l], offs[l+1])
//   perm       int32 [n]           position -> record id, ascending within a list
// A list's rows are read in place from the collection's keys through perm:
// a row is dim * 4 (or 2) contiguous bytes, so the indirection costs no
// coalescing at dim >= 256, and no list-ordered copy is kept (a trajectory
// DB's lists are mostly runs of consecutive rows anyway).
//
// Search (B queries, nprobe lists each):
//   1. coarse scan: every centroid scored (fp32 SIMT over the fp32 centroids),
//      units of `span` rows (chunks of `ur`) -> per-unit top-32 -> per-query merge -> the nprobe
//      best lists (approximate order; ties by list id);
//   2. probe prefix: units of the probed lists (ceil(len / span) each; the
//      span bounds the unit count, so the per-unit lists stay small);
//   3. fine scan: the probed lists' rows (the stored keys, or the bf16 filter
//      copy of an fp32 collection when it keeps one) x the fp32 query, fp32
//      accumulation; per-unit top-32 keyed by RECORD id;
//   4. per-query merge -> the 32 best candidates by approximate score;
//   5. k_select's pooled rescoring: the reference's sequential fp64 sum over
//      the stored keys (store.cpp:29-34) and (score desc, id asc) ranking, so
//      every returned score is exactly cosine_similarity of the returned id, as
//      search_topk recomputes it for the HNSW ids (store.cpp:86-90).
//
// Build (index.cu): strided seeds, Lloyd iterations whose assignment step is
// the collection's own exact search (tcgen05 filter + fp64 rescoring) of the
// rows against the centroid set, a deterministic stable counting sort (per
// block histograms + a one-warp ballot scatter) and fp64 list means.
// Deterministic: the same collection and parameters
// give the same index bit for bit.
#include "common.cuh"
#include "hsd/hsd_synth.h"
#include "kernels.h"

namespace hsd {
namespace {

using dev::kEmpty;

constexpr int kIThreads = 256;
constexpr int kIWarps = kIThreads / 32;
constexpr int kUnitMax = 128;

// 8 bf16 (one 16-B load) against 8 fp32 query values
__device__ __forceinline__ float dot8(const uint4 a, const float4 q0, const float4 q1, float acc) {
  acc = fmaf(__uint_as_float(a.x << 16), q0.x, acc);
  acc = fmaf(__uint_as_float(a.x & 0xFFFF0000u), q0.y, acc);
  acc = fmaf(__uint_as_float(a.y << 16), q0.z, acc);
  acc = fmaf(__uint_as_float(a.y & 0xFFFF0000u), q0.w, acc);
  acc = fmaf(__uint_as_float(a.z << 16), q1.x, acc);
  acc = fmaf(__uint_as_float(a.z & 0xFFFF0000u), q1.y, acc);
  acc = fmaf(__uint_as_float(a.w << 16), q1.z, acc);
  acc = fmaf(__uint_as_float(a.w & 0xFFFF0000u), q1.w, acc);
  return acc;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Two rows' dots with one query (one warp; every lane ends with both sums).
// bf16 rows (dim % 8 == 0, as bf16 collections require).
__device__ __forceinline__ void dot2(const uint16_t* __restrict__ ra, const uint16_t* __restrict__ rb, bool vb,
                                     const float* __restrict__ q, int dim, int lane, float& sa, float& sb) {
  const uint4* a8 = reinterpret_cast<const uint4*>(ra);
  const uint4* b8 = reinterpret_cast<const uint4*>(rb);
  const float4* q4 = reinterpret_cast<const float4*>(q);
  const int n8 = dim / 8;
  float xa = 0.f, xb = 0.f;
  int i = lane;
  for (; i + 96 < n8; i += 128) {
    uint4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = dev::ldg_stream_u4(a8 + i + 32 * u);
      b[u] = vb ? dev::ldg_stream_u4(b8 + i + 32 * u) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 q0 = __ldg(q4 + 2 * (i + 32 * u)), q1 = __ldg(q4 + 2 * (i + 32 * u) + 1);
      xa = dot8(a[u], q0, q1, xa);
      xb = dot8(b[u], q0, q1, xb);
    }
  }
  for (; i < n8; i += 32) {
    const uint4 a = dev::ldg_stream_u4(a8 + i);
    const uint4 b = vb ? dev::ldg_stream_u4(b8 + i) : make_uint4(0, 0, 0, 0);
    const float4 q0 = __ldg(q4 + 2 * i), q1 = __ldg(q4 + 2 * i + 1);
    xa = dot8(a, q0, q1, xa);
    xb = dot8(b, q0, q1, xb);
  }
  sa = warp_sum(xa);
  sb = warp_sum(xb);
}

// fp32 rows (the centroids and fp32 collections; dim % 4 == 0).  Four
// 16-B loads per row in flight per lane.
__device__ __forceinline__ void dot2(const float* __restrict__ ra, const float* __restrict__ rb, bool vb,
                                     const float* __restrict__ q, int dim, int lane, float& sa, float& sb) {
  const float4* a4 = reinterpret_cast<const float4*>(ra);
  const float4* b4 = reinterpret_cast<const float4*>(rb);
  const float4* q4 = reinterpret_cast<const float4*>(q);
  const int n4 = dim / 4;
  float xa = 0.f, xb = 0.f;
  int i = lane;
  for (; i + 96 < n4; i += 128) {
    float4 a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = dev::ldg_stream(a4 + i + 32 * u);
      b[u] = vb ? dev::ldg_stream(b4 + i + 32 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4 qq = __ldg(q4 + i + 32 * u);
      xa = fmaf(a[u].x, qq.x, fmaf(a[u].y, qq.y, fmaf(a[u].z, qq.z, fmaf(a[u].w, qq.w, xa))));
      xb = fmaf(b[u].x, qq.x, fmaf(b[u].y, qq.y, fmaf(b[u].z, qq.z, fmaf(b[u].w, qq.w, xb))));
    }
  }
  for (; i < n4; i += 32) {
    const float4 a = dev::ldg_stream(a4 + i);
    const float4 b = vb ? dev::ldg_stream(b4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 qq = __ldg(q4 + i);
    xa = fmaf(a.x, qq.x, fmaf(a.y, qq.y, fmaf(a.z, qq.z, fmaf(a.w, qq.w, xa))));
    xb = fmaf(b.x, qq.x, fmaf(b.y, qq.y, fmaf(b.z, qq.z, fmaf(b.w, qq.w, xb))));
  }
  sa = warp_sum(xa);
  sb = warp_sum(xb);
}

// Unit -> (query, row range) of the coarse (identity ids) or fine (lists) scan.
struct Unit {
  int b;
  int64_t r0, r1;
};
__device__ __forceinline__ Unit unit_of(const IvfUnits& su, int64_t u) {
  Unit x;
  if (su.mode == 0) {
    x.b = (int)(u / su.per_q);
    x.r0 = (u - (int64_t)x.b * su.per_q) * su.span;
    x.r1 = min(x.r0 + su.span, su.n_rows);
    return x;
  }
  int lo = 0, hi = su.n_pairs;  // largest p with upre[p] <= u
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (su.upre[mid] <= u) lo = mid; else hi = mid;
  }
  const int l = su.probe[lo];
  x.b = lo / su.nprobe;
  x.r0 = su.offs[l] + (u - su.upre[lo]) * (int64_t)su.span;
  x.r1 = min(x.r0 + su.span, (int64_t)su.offs[l + 1]);
  return x;
}

__device__ __forceinline__ int64_t unit_count(const IvfUnits& su) {
  return su.mode == 0 ? (int64_t)su.per_q * su.n_q : (int64_t)su.upre[su.n_pairs];
}

// Scan: per unit, the 32 best (score desc, id asc) of its rows.
template <typename KT>
__global__ void __launch_bounds__(kIThreads) ivf_scan_kernel(const KT* __restrict__ rows, int64_t stride,
                                                             const int32_t* __restrict__ row_id, int dim,
                                                             const float* __restrict__ queries, IvfUnits su,
                                                             uint64_t* __restrict__ out) {
  __shared__ uint64_t sk[kUnitMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = unit_count(su);
  for (int64_t u = blockIdx.x; u < total; u += gridDim.x) {
    const Unit x = unit_of(su, u);
    const float* q = queries + (size_t)x.b * dim;
    uint64_t top = kEmpty;  // warp 0: the unit's running top-32 over its chunks of ur rows
    for (int64_t c0 = x.r0; c0 < x.r1; c0 += su.ur) {
      for (int rr = warp; rr < su.ur; rr += 2 * kIWarps) {
        const int64_t pa = c0 + rr, pb = pa + kIWarps;
        const bool va = pa < x.r1, vb = pb < x.r1;
        // the record behind each list position: its id and its stored key row
        const int64_t ia = va ? (row_id ? (int64_t)row_id[pa] : pa) : 0;
        const int64_t ib = vb ? (row_id ? (int64_t)row_id[pb] : pb) : ia;
        float sa = 0.f, sb = 0.f;
        if (va) dot2(rows + ia * stride, rows + ib * stride, vb, q, dim, lane, sa, sb);
        if (lane == 0) {
          sk[rr] = va ? dev::cand_key(sa, (uint32_t)ia) : kEmpty;
          sk[rr + kIWarps] = vb ? dev::cand_key(sb, (uint32_t)ib) : kEmpty;
        }
      }
      __syncthreads();
      if (warp == 0) {
        uint64_t v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) v[t] = t * 32 + lane < su.ur ? sk[t * 32 + lane] : kEmpty;
        dev::warp_sort<4>(v);
        top = dev::warp_merge_top32(top, v[0]);
      }
      __syncthreads();
    }
    if (warp == 0) out[(size_t)u * 32 + lane] = top;
  }
}

// Per query: merge its units' sorted top-32 lists into pool[b][0..32).
__global__ void __launch_bounds__(kIThreads) ivf_merge_kernel(const uint64_t* __restrict__ part, IvfUnits su,
                                                              uint64_t* __restrict__ pool) {
  __shared__ uint64_t wt[kIWarps][32];
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t u0, u1;
  if (su.mode == 0) {
    u0 = (int64_t)b * su.per_q;
    u1 = u0 + su.per_q;
  } else {
    u0 = su.upre[b * su.nprobe];
    u1 = su.upre[(b + 1) * su.nprobe];
  }
  uint64_t top = kEmpty;
  for (int64_t u = u0 + warp; u < u1; u += kIWarps) top = dev::warp_merge_top32(top, part[(size_t)u * 32 + lane]);
  wt[warp][lane] = top;
  __syncthreads();
  if (warp == 0) {
    top = wt[0][lane];
#pragma unroll
    for (int w = 1; w < kIWarps; ++w) top = dev::warp_merge_top32(top, wt[w][lane]);
    pool[(size_t)b * 32 + lane] = top;
  }
}

// Probe lists (the first nprobe of each query's coarse pool) and the fine
// scan's unit prefix upre[p] (ceil(len / span) units per probed list).  One CTA.
constexpr int kPThreads = 1024;
__global__ void __launch_bounds__(kPThreads) ivf_probe_kernel(const uint64_t* __restrict__ pool, int B, int nprobe,
                                                              const int32_t* __restrict__ offs, int span,
                                                              int32_t* __restrict__ probe,
                                                              int32_t* __restrict__ upre) {
  __shared__ int wsum[kPThreads / 32];
  const int n = B * nprobe, tid = threadIdx.x, lane = tid & 31;
  const int per = (n + kPThreads - 1) / kPThreads;
  const int p0 = min(n, tid * per), p1 = min(n, p0 + per);
  int run = 0;
  for (int p = p0; p < p1; ++p) {
    const uint64_t key = pool[(size_t)(p / nprobe) * 32 + (p % nprobe)];
    const int l = key == kEmpty ? -1 : (int)dev::cand_id(key);
    probe[p] = l < 0 ? 0 : l;
    run += l < 0 ? 0 : (offs[l + 1] - offs[l] + span - 1) / span;
  }
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
  for (int p = p0; p < p1; ++p) {
    const uint64_t key = pool[(size_t)(p / nprobe) * 32 + (p % nprobe)];
    const int l = key == kEmpty ? -1 : (int)dev::cand_id(key);
    upre[p] = base;
    base += l < 0 ? 0 : (offs[l + 1] - offs[l] + span - 1) / span;
  }
  if (tid == kPThreads - 1) upre[n] = base;
}

// ---- build ---------------------------------------------------------------------

__device__ __forceinline__ double widen(float x) { return (double)x; }
__device__ __forceinline__ double widen(uint16_t b) { return (double)hsd_bf16_val(b); }

// Seeds: row floor((2l + 1) n / (2 nlist)) of each of nlist equal strata.
template <typename KT>
__global__ void ivf_seed_kernel(const KT* __restrict__ keys, int dim, int64_t n, int nlist, double* __restrict__ sum) {
  const int l = blockIdx.x;
  const int64_t r = (int64_t)((2.0 * l + 1.0) * (double)n / (2.0 * nlist));
  for (int d = threadIdx.x; d < dim; d += blockDim.x) sum[(size_t)l * dim + d] = widen(keys[(size_t)r * dim + d]);
}

// fp64 column sums of each list's rows (ascending position order: deterministic).
template <typename KT>
__global__ void __launch_bounds__(256) ivf_sum_kernel(const KT* __restrict__ keys, int dim,
                                                      const int32_t* __restrict__ perm,
                                                      const int32_t* __restrict__ offs, double* __restrict__ sum) {
  const int l = blockIdx.x, d = blockIdx.y * 256 + threadIdx.x;
  if (d >= dim) return;
  const int j0 = offs[l], j1 = offs[l + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = j0;
  for (; j + 3 < j1; j += 4) {
    a0 += widen(keys[(size_t)perm[j] * dim + d]);
    a1 += widen(keys[(size_t)perm[j + 1] * dim + d]);
    a2 += widen(keys[(size_t)perm[j + 2] * dim + d]);
    a3 += widen(keys[(size_t)perm[j + 3] * dim + d]);
  }
  for (; j < j1; ++j) a0 += widen(keys[(size_t)perm[j] * dim + d]);
  sum[(size_t)l * dim + d] = (a0 + a1) + (a2 + a3);
}

// Centroid l <- sum / |sum| (fp32); an empty list or a zero sum keeps the old
// centroid.  offs == nullptr: seeds (every list non-empty).
__global__ void __launch_bounds__(256) ivf_norm_kernel(const double* __restrict__ sum, int dim,
                                                       const int32_t* __restrict__ offs, float* __restrict__ cent) {
  __shared__ double red[8];
  const int l = blockIdx.x, tid = threadIdx.x;
  if (offs && offs[l + 1] == offs[l]) return;
  double acc = 0.0;
  for (int d = tid; d < dim; d += 256) acc = fma(sum[(size_t)l * dim + d], sum[(size_t)l * dim + d], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < 8; ++w) t += red[w];
  if (!(t > 0.0) || !isfinite(t)) return;
  const double inv = 1.0 / sqrt(t);
  for (int d = tid; d < dim; d += 256) cent[(size_t)l * dim + d] = (float)(sum[(size_t)l * dim + d] * inv);
}

// bf16 collection rows -> fp32 (the assignment step's queries)
__global__ void ivf_widen_kernel(const uint16_t* __restrict__ in, int64_t n, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hsd_bf16_val(in[i]);
}

// Per-block list histograms bh[g][l] of assign over rows [g chunk, (g+1) chunk).
__global__ void ivf_hist_kernel(const int32_t* __restrict__ assign, int64_t n, int64_t chunk, int nlist,
                                int32_t* __restrict__ bh) {
  extern __shared__ int h[];
  for (int i = threadIdx.x; i < nlist; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) atomicAdd(&h[assign[r]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < nlist; i += blockDim.x) bh[(size_t)blockIdx.x * nlist + i] = h[i];
}

// One CTA: list sizes -> offs (exclusive scan) and bh[g][l] -> first position
// of block g's rows in list l.
__global__ void __launch_bounds__(kPThreads) ivf_lists_kernel(int32_t* __restrict__ bh, int G, int nlist,
                                                              int32_t* __restrict__ offs) {
  __shared__ int wsum[kPThreads / 32];
  constexpr int kPer = kIvfMaxLists / kPThreads;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int l = tid; l < nlist; l += kPThreads) {
    int t = 0;
    for (int g = 0; g < G; ++g) t += bh[(size_t)g * nlist + l];
    offs[l + 1] = t;  // size, scanned below
  }
  __syncthreads();
  const int per = (nlist + kPThreads - 1) / kPThreads;
  const int l0 = min(nlist, tid * per), l1 = min(nlist, l0 + per);
  int run = 0, sz[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    sz[i] = l0 + i < l1 ? offs[l0 + i + 1] : 0;
    run += sz[i];
  }
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
  __syncthreads();  // every thread holds the sizes it scans
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (l0 + i < l1) offs[l0 + i] = base;
    base += sz[i];
  }
  if (tid == kPThreads - 1) offs[nlist] = base;
  __syncthreads();
  for (int l = tid; l < nlist; l += kPThreads) {
    int run2 = offs[l];
    for (int g = 0; g < G; ++g) {
      const int t = bh[(size_t)g * nlist + l];
      bh[(size_t)g * nlist + l] = run2;
      run2 += t;
    }
  }
}

// Stable scatter: one warp per block walks its rows in order, 32 at a time;
// rows of one list within a tile are ranked by lane (match.any), so perm holds
// every list's record ids in ascending order.
__global__ void __launch_bounds__(32) ivf_scatter_kernel(const int32_t* __restrict__ assign, int64_t n,
                                                         int64_t chunk, int nlist, const int32_t* __restrict__ bh,
                                                         int32_t* __restrict__ perm) {
  extern __shared__ int cnt[];
  const int lane = threadIdx.x;
  for (int i = lane; i < nlist; i += 32) cnt[i] = bh[(size_t)blockIdx.x * nlist + i];
  __syncwarp();
  const int64_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  for (int64_t t = r0; t < r1; t += 32) {
    const int64_t r = t + lane;
    const bool valid = r < r1;
    const int l = valid ? assign[r] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const int rank = __popc(peers & ((1u << lane) - 1));
    const int base = valid ? cnt[l] : 0;
    __syncwarp();
    if (valid) {
      perm[base + rank] = (int32_t)r;
      if (rank == 0) cnt[l] = base + __popc(peers);
    }
    __syncwarp();
  }
}

}  // namespace

size_t ivf_part_bytes(int64_t units) { return (size_t)units * 32 * sizeof(uint64_t); }

cudaError_t launch_ivf_scan(const void* rows, int rows_bf16, int64_t stride, const int32_t* row_id, int dim,
                            const float* queries, const IvfUnits& su, int64_t max_units, int grid, uint64_t* part,
                            cudaStream_t s) {
  if ((su.ur != 32 && su.ur != kUnitMax) || su.span < su.ur || su.span % su.ur) return cudaErrorInvalidValue;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(max_units, grid));
  if (rows_bf16)
    ivf_scan_kernel<uint16_t><<<g, kIThreads, 0, s>>>((const uint16_t*)rows, stride, row_id, dim, queries, su, part);
  else
    ivf_scan_kernel<float><<<g, kIThreads, 0, s>>>((const float*)rows, stride, row_id, dim, queries, su, part);
  return cudaGetLastError();
}

cudaError_t launch_ivf_merge(const uint64_t* part, const IvfUnits& su, int B, uint64_t* pool, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  ivf_merge_kernel<<<B, kIThreads, 0, s>>>(part, su, pool);
  return cudaGetLastError();
}

cudaError_t launch_ivf_probe(const uint64_t* pool, int B, int nprobe, const int32_t* offs, int span, int32_t* probe,
                             int32_t* upre, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  if (nprobe < 1 || nprobe > 32) return cudaErrorInvalidValue;
  ivf_probe_kernel<<<1, kPThreads, 0, s>>>(pool, B, nprobe, offs, span, probe, upre);
  return cudaGetLastError();
}

cudaError_t launch_ivf_seed(const void* keys, int key_dtype, int dim, int64_t n, int nlist, double* sum,
                            cudaStream_t s) {
  if (key_dtype == HSD_DTYPE_BF16)
    ivf_seed_kernel<uint16_t><<<nlist, 256, 0, s>>>((const uint16_t*)keys, dim, n, nlist, sum);
  else
    ivf_seed_kernel<float><<<nlist, 256, 0, s>>>((const float*)keys, dim, n, nlist, sum);
  return cudaGetLastError();
}

cudaError_t launch_ivf_centroids(const void* keys, int key_dtype, int dim, int nlist, const int32_t* perm,
                                 const int32_t* offs, double* sum, float* cent, cudaStream_t s) {
  if (perm) {
    const dim3 grid(nlist, (dim + 255) / 256);
    if (key_dtype == HSD_DTYPE_BF16)
      ivf_sum_kernel<uint16_t><<<grid, 256, 0, s>>>((const uint16_t*)keys, dim, perm, offs, sum);
    else
      ivf_sum_kernel<float><<<grid, 256, 0, s>>>((const float*)keys, dim, perm, offs, sum);
  }
  ivf_norm_kernel<<<nlist, 256, 0, s>>>(sum, dim, perm ? offs : nullptr, cent);
  return cudaGetLastError();
}

cudaError_t launch_ivf_widen(const uint16_t* in, int64_t n, float* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
  ivf_widen_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, out);
  return cudaGetLastError();
}

int64_t ivf_sort_blocks(int64_t n, int64_t* chunk) {
  *chunk = 4096;
  return (n + *chunk - 1) / *chunk;
}

cudaError_t launch_ivf_sort(const int32_t* assign, int64_t n, int nlist, int32_t* bh, int32_t* offs, int32_t* perm,
                            cudaStream_t s) {
  int64_t chunk = 0;
  const int64_t G = ivf_sort_blocks(n, &chunk);
  const size_t smem = (size_t)nlist * sizeof(int);
  cudaError_t e = cudaFuncSetAttribute(ivf_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(ivf_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ivf_hist_kernel<<<(unsigned)G, 256, smem, s>>>(assign, n, chunk, nlist, bh);
  ivf_lists_kernel<<<1, kPThreads, 0, s>>>(bh, (int)G, nlist, offs);
  ivf_scatter_kernel<<<(unsigned)G, 32, smem, s>>>(assign, n, chunk, nlist, bh, perm);
  return cudaGetLastError();
}

}  // namespace hsd
