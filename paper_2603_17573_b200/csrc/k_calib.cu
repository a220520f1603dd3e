// k_calib.cu — verify-skip offline calibration (Alg. 1 offline stage,
// SPEC.md:449-457) as a batched per-trajectory Gram pass.
//
// For every trajectory t (rows [off[t], off[t+1]) of the feature matrix) and
// every pair (i, i+d), d >= 1, S = the exactly rounded dot of the two fp32
// feature vectors (the same similarity should_skip uses, k_verify.cu).  Among
// pairs with S > T the minimum S wins; ties go to the first pair in the
// oracle's loop order (trajectory, i, d) (oracle/hsd_oracle.c
// hsdo_calibrate_accumulate).  The result is (min_S, O_dist = d).
//
// The dot must be exact to the last bit (the selection compares S values), so
// the Gram tiles run on the fp64 pipe in double-double: fp32 x fp32 products
// are exact in fp64, two_sum keeps the rounding error, one rounding at the end.
// Tile: 32 x 32 pairs per CTA (upper-triangle tiles only), 64-dim feature
// chunks staged in shared memory, 4 pairs per thread.
#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

constexpr int kT = 32;        // tile edge (rows i, columns j)
constexpr int kChunk = 64;    // feature dims per shared-memory stage
constexpr int kThreads = 256; // 4 pairs per thread

struct CalibBest {
  double S;        // +inf when none
  uint64_t order;  // (traj << 42) | (i << 21) | d : the oracle's loop order
};

__device__ __forceinline__ bool better(double s, uint64_t o, double bs, uint64_t bo) {
  return s < bs || (s == bs && o < bo);
}

// grid.x = tile index within the trajectory's upper triangle, grid.y = trajectory
__global__ void __launch_bounds__(kThreads) calib_tiles_kernel(const float* __restrict__ feat, int d_f,
                                                               const int64_t* __restrict__ off, double T,
                                                               int max_tiles, CalibBest* __restrict__ best) {
  __shared__ float sa[kT][kChunk + 1], sb[kT][kChunk + 1];
  __shared__ double rs[kThreads];
  __shared__ uint64_t ro[kThreads];
  const int t = blockIdx.y;
  const int64_t r0 = off[t], n = off[t + 1] - r0;
  const int nt = (int)((n + kT - 1) / kT);
  // map blockIdx.x -> (bi, bj) with bj >= bi over the nt x nt tile triangle
  int b = blockIdx.x, bi = 0;
  while (bi < nt && b >= nt - bi) {
    b -= nt - bi;
    ++bi;
  }
  CalibBest mine{INFINITY, ~0ull};
  if (bi < nt) {
    const int bj = bi + b;
    const int tid = threadIdx.x;
    const int pi = tid / 8, pj0 = (tid % 8) * 4;  // thread: row pi, columns pj0..pj0+3
    double hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
    for (int c0 = 0; c0 < d_f; c0 += kChunk) {
      for (int x = tid; x < kT * kChunk; x += kThreads) {
        const int rr = x / kChunk, cc = x % kChunk;
        const int64_t ia = bi * kT + rr, ib = bj * kT + rr;
        sa[rr][cc] = (ia < n && c0 + cc < d_f) ? feat[(size_t)(r0 + ia) * d_f + c0 + cc] : 0.f;
        sb[rr][cc] = (ib < n && c0 + cc < d_f) ? feat[(size_t)(r0 + ib) * d_f + c0 + cc] : 0.f;
      }
      __syncthreads();
#pragma unroll 4
      for (int cc = 0; cc < kChunk; ++cc) {
        const double a = (double)sa[pi][cc];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double p = a * (double)sb[pj0 + u][cc];  // exact: fp32 x fp32 fits in fp64
          double s, e;
          dev::two_sum(hi[u], p, s, e);
          hi[u] = s;
          lo[u] = __dadd_rn(lo[u], e);
        }
      }
      __syncthreads();
    }
    const int64_t i = (int64_t)bi * kT + pi;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = (int64_t)bj * kT + pj0 + u;
      if (i < n && j < n && j > i) {
        double S, e;
        dev::two_sum(hi[u], lo[u], S, e);
        const uint64_t ord = ((uint64_t)t << 42) | ((uint64_t)i << 21) | (uint64_t)(j - i);
        if (S > T && better(S, ord, mine.S, mine.order)) {
          mine.S = S;
          mine.order = ord;
        }
      }
    }
  }
  // block reduction (deterministic: total order on (S, order))
  rs[threadIdx.x] = mine.S;
  ro[threadIdx.x] = mine.order;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w && better(rs[threadIdx.x + w], ro[threadIdx.x + w], rs[threadIdx.x], ro[threadIdx.x])) {
      rs[threadIdx.x] = rs[threadIdx.x + w];
      ro[threadIdx.x] = ro[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) best[(size_t)t * max_tiles + blockIdx.x] = CalibBest{rs[0], ro[0]};
}

__global__ void __launch_bounds__(1024) calib_reduce_kernel(const CalibBest* __restrict__ in, int64_t m,
                                                            CalibBest* __restrict__ out) {
  __shared__ double rs[1024];
  __shared__ uint64_t ro[1024];
  double s = INFINITY;
  uint64_t o = ~0ull;
  for (int64_t x = threadIdx.x; x < m; x += 1024)
    if (better(in[x].S, in[x].order, s, o)) {
      s = in[x].S;
      o = in[x].order;
    }
  rs[threadIdx.x] = s;
  ro[threadIdx.x] = o;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w && better(rs[threadIdx.x + w], ro[threadIdx.x + w], rs[threadIdx.x], ro[threadIdx.x])) {
      rs[threadIdx.x] = rs[threadIdx.x + w];
      ro[threadIdx.x] = ro[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = CalibBest{rs[0], ro[0]};
}

}  // namespace

size_t calib_scratch_bytes(int n_traj, int max_tiles) { return ((size_t)n_traj * max_tiles + 1) * sizeof(CalibBest); }

cudaError_t launch_calibrate(const float* feat, int d_f, const int64_t* off_dev, int n_traj, int max_len, double T,
                             void* scratch, double* min_S_out, int* O_dist_out, int* found_out, cudaStream_t s) {
  const int nt = (max_len + kT - 1) / kT;
  const int max_tiles = nt * (nt + 1) / 2;
  if (n_traj <= 0 || max_tiles <= 0) {
    *found_out = 0;
    return cudaSuccess;
  }
  CalibBest* tiles = reinterpret_cast<CalibBest*>(scratch);
  CalibBest* res = tiles + (size_t)n_traj * max_tiles;
  calib_tiles_kernel<<<dim3(max_tiles, n_traj), kThreads, 0, s>>>(feat, d_f, off_dev, T, max_tiles, tiles);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  calib_reduce_kernel<<<1, 1024, 0, s>>>(tiles, (int64_t)n_traj * max_tiles, res);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CalibBest h;
  e = cudaMemcpyAsync(&h, res, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *found_out = h.order != ~0ull;
  if (*found_out) {
    *min_S_out = h.S;
    *O_dist_out = (int)(h.order & ((1ull << 21) - 1));
  }
  return cudaSuccess;
}

}  // namespace hsd
