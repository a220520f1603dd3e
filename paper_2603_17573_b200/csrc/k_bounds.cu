// k_bounds.cu — compute_percentile_bounds (kinematics.cpp:238-247) on the
// device: (min, nearest-rank 95th percentile) of n fp64 samples, the value at
// index min(n - 1, max(ceil(0.95 n), 1) - 1) of the ascending sort.  Feeds
// the NormalizationBounds that K5 consumes (the norm-bounds CLI).
//
// The samples are mapped to order-preserving u64 keys (-0.0 shares +0.0's
// key: the reference's std::sort treats them as equal) and radix-sorted with
// CUB; non-finite samples are rejected first (std::sort with NaN is undefined).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

__global__ void order_keys_kernel(const double* __restrict__ x, int64_t n, uint64_t* __restrict__ keys,
                                  int* __restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    if (!isfinite(v)) atomicAdd(bad, 1);
    uint64_t u = (uint64_t)__double_as_longlong(v == 0.0 ? 0.0 : v);
    keys[i] = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  }
}

__global__ void pick_kernel(const uint64_t* __restrict__ sorted, int64_t idx, double* __restrict__ out) {
  auto val = [](uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)u);
  };
  out[0] = val(sorted[0]);
  out[1] = val(sorted[idx]);
}

}  // namespace

// out2 (device) <- (min, p95); bad (device) counts non-finite samples.
cudaError_t launch_percentile_bounds(const double* samples, int64_t n, double* out2, int* bad, cudaStream_t s) {
  if (n <= 0) return cudaErrorInvalidValue;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, n, 0, 64, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&k0, (size_t)n * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&k1, (size_t)n * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes, s);
  if (e == cudaSuccess) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    order_keys_kernel<<<blocks, 256, 0, s>>>(samples, n, k0, bad);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, n, 0, 64, s);
  if (e == cudaSuccess) {
    int64_t rank = (int64_t)ceil(0.95 * (double)n);  // kinematics.cpp:244
    rank = rank < 1 ? 1 : rank;
    const int64_t idx = std::min<int64_t>(n - 1, rank - 1);
    pick_kernel<<<1, 1, 0, s>>>(k1, idx, out2);
    e = cudaGetLastError();
  }
  if (k0) cudaFreeAsync(k0, s);
  if (k1) cudaFreeAsync(k1, s);
  if (tmp) cudaFreeAsync(tmp, s);
  return e;
}

}  // namespace hsd
