// k_sim_simt.cu — K1 (SIMT): approximate fp32 similarity S = Q·K^T streamed
// from HBM, fused with a per-CTA top-32 candidate filter per query.
//
// Replaces the hot loop of Collection::search_topk_exact (store.cpp:63-66):
// every key row is read exactly once per launch.  The scores produced here are
// only a FILTER: the select kernel (k_select.cu) rescoring recomputes the
// reference's sequential fp64 dot for the surviving candidates, so ids and
// scores end up bit-identical to the reference.
//
//   sim_rows<BP>  B <= 8   : warp-per-row-group GEMV, 128-bit streaming loads,
//                            queries in shared memory, warp reduce-scatter.
//   sim_tile      B <= 64  : 128-key x 64-query register-tiled SIMT GEMM
//                            (FFMA-bound; superseded by the tcgen05 kernel,
//                            k_sim_tc.cu, when available).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

using dev::cand_key;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ============================================================================
// sim_rows: B <= 8 queries.  Each warp owns R = 32/BP consecutive rows at a
// time; lane l streams float4 column slices l, l+32, ... of every row; the
// R x BP partial dots are reduce-scattered so that lane l ends with (row l/BP,
// query l%BP).  Warp-private candidate buffers (64 slots) are compacted to the
// best 32 when they fill.
// ============================================================================
template <int BP>
__global__ void __launch_bounds__(kThreads) sim_rows_kernel(const float* __restrict__ keys, int64_t row_begin,
                                                            int64_t row_end, int dim, const float* __restrict__ queries,
                                                            int B, int64_t rows_per_cta,
                                                            uint64_t* __restrict__ partial) {
  constexpr int R = 32 / BP;
  constexpr int kBuf = 64;
  extern __shared__ __align__(16) unsigned char smem[];
  const int dim4 = dim >> 2;
  float4* sq = reinterpret_cast<float4*>(smem);                                       // [BP][dim4]
  uint64_t* cbuf = reinterpret_cast<uint64_t*>(smem + (size_t)BP * dim4 * 16);         // [warps][BP][kBuf]
  uint64_t* thr = cbuf + kWarps * BP * kBuf;                                           // [warps][BP]
  int* cnt = reinterpret_cast<int*>(thr + kWarps * BP);                                // [warps][BP]

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < BP * dim4; i += kThreads) {
    const int q = i / dim4;
    sq[i] = q < B ? reinterpret_cast<const float4*>(queries)[(size_t)q * dim4 + (i % dim4)] : make_float4(0, 0, 0, 0);
  }
  for (int i = threadIdx.x; i < kWarps * BP; i += kThreads) {
    thr[i] = kEmpty;
    cnt[i] = 0;
  }
  __syncthreads();

  const int64_t r0 = row_begin + (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = std::min<int64_t>(r0 + rows_per_cta, row_end);
  const float4* k4 = reinterpret_cast<const float4*>(keys);
  uint64_t* my_buf = cbuf + warp * BP * kBuf;
  uint64_t* my_thr = thr + warp * BP;
  int* my_cnt = cnt + warp * BP;

  for (int64_t g = r0 + (int64_t)warp * R; g < r1; g += (int64_t)kWarps * R) {
    float acc[R * BP];
#pragma unroll
    for (int j = 0; j < R * BP; ++j) acc[j] = 0.f;
    for (int t = lane; t < dim4; t += 32) {
      float4 kv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t row = g + r;
        kv[r] = row < r1 ? dev::ldg_stream(k4 + (size_t)row * dim4 + t) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < BP; ++q) {
        const float4 qv = sq[q * dim4 + t];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float a = acc[r * BP + q];
          a = fmaf(kv[r].x, qv.x, a);
          a = fmaf(kv[r].y, qv.y, a);
          a = fmaf(kv[r].z, qv.z, a);
          a = fmaf(kv[r].w, qv.w, a);
          acc[r * BP + q] = a;
        }
      }
    }
    // reduce-scatter: lane l ends with the full sum of pair index l
#pragma unroll
    for (int off = 16, n = 32; off > 0; off >>= 1, n >>= 1) {
      const bool hi = (lane & off) != 0;
#pragma unroll
      for (int j = 0; j < n / 2; ++j) {
        const float send = hi ? acc[j] : acc[j + n / 2];
        const float keep = hi ? acc[j + n / 2] : acc[j];
        acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    const int r = lane / BP, q = lane % BP;
    const int64_t row = g + r;
    if (row < r1 && q < B) {
      const uint64_t key = cand_key(acc[0], (uint32_t)row);
      if (key < my_thr[q]) {
        const int slot = atomicAdd(&my_cnt[q], 1);
        my_buf[q * kBuf + slot] = key;
      }
    }
    __syncwarp();
#pragma unroll
    for (int qq = 0; qq < BP; ++qq) {
      if (my_cnt[qq] > kCandLocal) {  // warp-uniform
        uint64_t v[2];
        const int c = my_cnt[qq];
        v[0] = lane < c ? my_buf[qq * kBuf + lane] : kEmpty;
        v[1] = lane + 32 < c ? my_buf[qq * kBuf + lane + 32] : kEmpty;
        dev::warp_sort<2>(v);
        __syncwarp();
        my_buf[qq * kBuf + lane] = v[0];
        if (lane == 31) my_thr[qq] = v[0];
        if (lane == 0) my_cnt[qq] = kCandLocal;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // merge the warps' lists: warp w handles query w
  if (warp < BP && warp < B) {
    uint64_t v[8];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const int c = cnt[w * BP + warp];
      v[w] = lane < c ? cbuf[(w * BP + warp) * kBuf + lane] : kEmpty;
    }
    dev::warp_sort<8>(v);
    partial[((size_t)blockIdx.x * B + warp) * kCandLocal + lane] = v[0];
  }
}

// ============================================================================
// sim_tile: 8 < B <= 64.  Tile = 128 keys x 64 queries x 32-column chunk in
// shared memory (k-major, padded), 8x4 register micro-tile per thread,
// register prefetch of the next chunk.  CTA-level candidate buffers of
// 32 + 128 slots per query, compacted after every tile.
// ============================================================================
constexpr int kTM = 128, kTQ = 64, kTK = 32;
constexpr int kKS = kTM + 4;  // padded row stride (floats) of the key chunk
constexpr int kQS = kTQ + 4;
constexpr int kTileBuf = kCandLocal + kTM;

struct TileSmem {
  float ks[kTK][kKS];
  float qs[kTK][kQS];
  uint64_t cbuf[kTQ][kTileBuf];
  uint64_t thr[kTQ];
  int cnt[kTQ];
};

__global__ void __launch_bounds__(kThreads) sim_tile_kernel(const float* __restrict__ keys, int64_t row_begin,
                                                            int64_t row_end, int dim, const float* __restrict__ queries,
                                                            int B, int64_t tiles_per_cta,
                                                            uint64_t* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& S = *reinterpret_cast<TileSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;
  for (int i = tid; i < kTQ; i += kThreads) {
    S.thr[i] = kEmpty;
    S.cnt[i] = 0;
  }
  const int64_t n_tiles_total = (row_end - row_begin + kTM - 1) / kTM;
  const int64_t t0 = (int64_t)blockIdx.x * tiles_per_cta;
  const int64_t t1 = std::min<int64_t>(t0 + tiles_per_cta, n_tiles_total);
  const float4* k4 = reinterpret_cast<const float4*>(keys);
  const float4* q4 = reinterpret_cast<const float4*>(queries);
  const int dim4 = dim >> 2;
  const int nchunks = (dim4 + 7) / 8;  // a ragged last chunk is zero-filled
  __syncthreads();

  for (int64_t tile = t0; tile < t1; ++tile) {
    const int64_t base = row_begin + tile * kTM;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

    float4 pk[4], pq[2];
    auto load = [&](int chunk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + kThreads * i;  // 1024 float4 = 128 rows x 8
        const int64_t row = base + (idx >> 3);
        const int col4 = chunk * 8 + (idx & 7);
        pk[i] = (row < row_end && col4 < dim4) ? dev::ldg_stream(k4 + (size_t)row * dim4 + col4)
                                               : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int idx = tid + kThreads * i;  // 512 float4 = 64 queries x 8
        const int q = idx >> 3;
        const int col4 = chunk * 8 + (idx & 7);
        pq[i] = (q < B && col4 < dim4) ? __ldg(q4 + (size_t)q * dim4 + col4) : make_float4(0, 0, 0, 0);
      }
    };
    load(0);
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = tid + kThreads * i;
        const int row = idx >> 3, c = (idx & 7) * 4;
        S.ks[c + 0][row] = pk[i].x;
        S.ks[c + 1][row] = pk[i].y;
        S.ks[c + 2][row] = pk[i].z;
        S.ks[c + 3][row] = pk[i].w;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int idx = tid + kThreads * i;
        const int q = idx >> 3, c = (idx & 7) * 4;
        S.qs[c + 0][q] = pq[i].x;
        S.qs[c + 1][q] = pq[i].y;
        S.qs[c + 2][q] = pq[i].z;
        S.qs[c + 3][q] = pq[i].w;
      }
      __syncthreads();
      if (chunk + 1 < nchunks) load(chunk + 1);
#pragma unroll 8
      for (int kk = 0; kk < kTK; ++kk) {
        const float4 a = *reinterpret_cast<const float4*>(&S.ks[kk][tx * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&S.ks[kk][64 + tx * 4]);
        const float4 q = *reinterpret_cast<const float4*>(&S.qs[kk][ty * 4]);
        const float kv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        const float qv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(kv[i], qv[j], acc[i][j]);
      }
    }
    // epilogue: candidate filter
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = ty * 4 + j;
      if (q >= B) continue;
      const uint64_t t = S.thr[q];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = base + (i < 4 ? tx * 4 + i : 64 + tx * 4 + (i - 4));
        if (row >= row_end) continue;
        const uint64_t key = cand_key(acc[i][j], (uint32_t)row);
        if (key < t) {
          const int slot = atomicAdd(&S.cnt[q], 1);
          S.cbuf[q][slot] = key;
        }
      }
    }
    __syncthreads();
    for (int q = warp; q < B; q += kWarps) {
      const int c = S.cnt[q];
      if (c > kCandLocal) {
        uint64_t v[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const int i = s * 32 + lane;
          v[s] = i < c ? S.cbuf[q][i] : kEmpty;
        }
        dev::warp_sort<8>(v);
        __syncwarp();
        S.cbuf[q][lane] = v[0];
        if (lane == 31) S.thr[q] = v[0];
        if (lane == 0) S.cnt[q] = kCandLocal;
      }
    }
    __syncthreads();
  }
  // final: sort each query's <= 32 survivors and write them out
  for (int q = warp; q < B; q += kWarps) {
    const int c = S.cnt[q];
    uint64_t v[1];
    v[0] = lane < c ? S.cbuf[q][lane] : kEmpty;
    dev::warp_sort<1>(v);
    partial[((size_t)blockIdx.x * B + q) * kCandLocal + lane] = v[0];
  }
}


}  // namespace

SimPlan sim_plan(int B, int64_t rows, int dim, int num_sms) {
  SimPlan p{};
  // Forward error bound of an fp32 dot of `dim` terms in any order with FMA:
  // |approx - exact| <= gamma_dim * sum|k_i q_i|, gamma_n = n u / (1 - n u).
  const double u = 1.0 / 16777216.0;
  const double n = (double)dim + 4.0;
  p.gamma = n * u / (1.0 - n * u) * 1.0001;
  if (B <= 8) {
    p.lists = num_sms * 4;
  } else {
    const int64_t tiles = (rows + kTM - 1) / kTM;
    p.lists = (int)std::min<int64_t>(tiles, (int64_t)num_sms * 2);
  }
  if (p.lists < 1) p.lists = 1;
  return p;
}

cudaError_t launch_sim(const float* keys, int64_t row_begin, int64_t row_end, int dim, const float* queries, int B,
                       const SimPlan& plan, uint64_t* partial, cudaStream_t s) {
  const int64_t rows = row_end - row_begin;
  if (B <= 8) {
    const int BP = B <= 1 ? 1 : (B <= 2 ? 2 : (B <= 4 ? 4 : 8));
    const int dim4 = dim / 4;
    const size_t smem = (size_t)BP * dim4 * 16 + (size_t)kWarps * BP * (64 * 8 + 8 + 4);
    const int64_t rows_per_cta = (rows + plan.lists - 1) / plan.lists;
    cudaError_t e = cudaSuccess;
#define HSD_ROWS(BPV)                                                                                    \
  case BPV:                                                                                              \
    e = cudaFuncSetAttribute(sim_rows_kernel<BPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (e != cudaSuccess) return e;                                                                      \
    sim_rows_kernel<BPV><<<plan.lists, kThreads, smem, s>>>(keys, row_begin, row_end, dim, queries, B,   \
                                                            rows_per_cta, partial);                     \
    break;
    switch (BP) {
      HSD_ROWS(1)
      HSD_ROWS(2)
      HSD_ROWS(4)
      HSD_ROWS(8)
    }
#undef HSD_ROWS
    return cudaGetLastError();
  }
  const int64_t tiles = (rows + kTM - 1) / kTM;
  const int64_t tiles_per_cta = (tiles + plan.lists - 1) / plan.lists;
  const size_t smem = sizeof(TileSmem);
  cudaError_t e = cudaFuncSetAttribute(sim_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sim_tile_kernel<<<plan.lists, kThreads, smem, s>>>(keys, row_begin, row_end, dim, queries, B, tiles_per_cta,
                                                      partial);
  return cudaGetLastError();
}

}  // namespace hsd
