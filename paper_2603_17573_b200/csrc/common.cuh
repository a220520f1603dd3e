// common.cuh — shared device helpers for the HeiSD hot-path kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hsd {
namespace dev {

// ---- programmatic dependent launch (PDL) -------------------------------------
// The small kernels of the step (K2's three launches, K4) are launched with
// programmatic stream serialization: a kernel lets its dependent launch as
// soon as all its CTAs are resident (pdl_trigger at entry), and the dependent
// blocks in pdl_wait until the predecessor grid has completed and its memory
// is visible.  Every dependent calls pdl_wait before touching any input.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr int kWarp = 32;
constexpr int kCandLocal = 32;     // candidates kept per (CTA, query) by the similarity kernels
constexpr uint64_t kEmpty = ~0ull; // empty candidate slot (sorts last)

// ---- candidate keys ---------------------------------------------------------
// A candidate is (approx score f32, record id u32) packed so that ASCENDING u64
// order is the reference's (score desc, id asc) order (store.cpp:67-70).
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t cand_key(float s, uint32_t id) {
  if (s != s) s = -INFINITY;  // NaN ranks last
  return ((uint64_t)(~f2ord(s)) << 32) | (uint64_t)id;
}
__device__ __forceinline__ float cand_score(uint64_t k) { return ord2f(~(uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t cand_id(uint64_t k) { return (uint32_t)(k & 0xFFFFFFFFu); }

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

// ---- warp bitonic sort ------------------------------------------------------
// Sorts 32*V u64 keys ascending across a warp; element i lives in lane
// (i % 32), slot (i / 32).
template <int V>
__device__ __forceinline__ void warp_sort(uint64_t (&a)[V]) {
  const int lane = threadIdx.x & 31;
  constexpr int N = 32 * V;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int vs = stride / 32;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int pv = v ^ vs;
          if (pv > v) {
            const int i = v * 32 + lane;
            const bool asc = (i & size) == 0;
            uint64_t x = a[v], y = a[pv];
            const bool sw = asc ? (x > y) : (x < y);
            a[v] = sw ? y : x;
            a[pv] = sw ? x : y;
          }
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int i = v * 32 + lane;
          const bool asc = (i & size) == 0;
          const uint64_t y = shfl_xor_u64(a[v], stride);
          const bool lower = (lane & stride) == 0;
          const uint64_t mn = a[v] < y ? a[v] : y;
          const uint64_t mx = a[v] < y ? y : a[v];
          a[v] = (asc == lower) ? mn : mx;
        }
      }
    }
  }
}

// Merge a sorted-ascending 32-key list `x` (one per lane) into the running
// sorted top-32 `top` (one per lane): keeps the 32 smallest, sorted.
__device__ __forceinline__ uint64_t warp_merge_top32(uint64_t top, uint64_t x) {
  const int lane = threadIdx.x & 31;
  const uint64_t y = shfl_u64(x, 31 - lane);  // reverse -> bitonic with `top`
  uint64_t m = top < y ? top : y;              // lower half of the 64-element bitonic merge
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const uint64_t o = shfl_xor_u64(m, stride);
    const bool lower = (lane & stride) == 0;
    m = lower ? (m < o ? m : o) : (m < o ? o : m);
  }
  return m;
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ldg_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Knuth TwoSum (error-free transformation).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bv = __dsub_rn(s, a);
  double av = __dsub_rn(s, bv);
  e = __dadd_rn(__dsub_rn(a, av), __dsub_rn(b, bv));
}

// Greedy verifier token over 256 bins held 8 per lane (lane l: bins 8l..8l+7
// in a, c): std::max_element's result (the reference's greedy rule, PAPER.md
// Eq. 2-1), i.e. the sequential scan `if (v[b] > v[best]) best = b`: the
// lowest index among equal maxima; a NaN is never selected after bin 0, and a
// NaN in bin 0 is never replaced (every comparison with it is false).
__device__ __forceinline__ int warp_argmax256(const float4& a, const float4& c, int lane) {
  const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
  // the largest non-NaN value (fmaxf drops a NaN operand; NaN only if all are)
  float m = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  // the lowest bin holding it (-0.0 == +0.0, as the sequential > scan sees them)
  int first = 8;
#pragma unroll
  for (int i = 7; i >= 0; --i) first = v[i] == m ? i : first;
  const unsigned hit = __ballot_sync(0xffffffffu, first < 8);
  const int src = hit ? __ffs(hit) - 1 : 0;
  const int fi = __shfl_sync(0xffffffffu, first, src);
  const float v0 = __shfl_sync(0xffffffffu, a.x, 0);
  return (v0 != v0 || hit == 0) ? 0 : src * 8 + fi;
}

// should_skip's similarity over one warp: the double-double sum of the exact
// fp64 products of two fp32 vectors (d % 4 == 0), i.e. the exact dot rounded
// once (except within ~2^-100): the same bits as cos_kernel / K4.
__device__ __forceinline__ double warp_dd_dot(const float* a, const float* b, int d, int lane) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  double hi = 0.0, lo = 0.0;
  for (int t = lane; t < d / 4; t += 32) {
    const float4 x = a4[t], y = b4[t];
    const double pr[4] = {(double)x.x * (double)y.x, (double)x.y * (double)y.y, (double)x.z * (double)y.z,
                          (double)x.w * (double)y.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double s, e;
      two_sum(hi, pr[i], s, e);
      hi = s;
      lo = __dadd_rn(lo, e);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ohi = __shfl_xor_sync(0xffffffffu, hi, o);
    const double olo = __shfl_xor_sync(0xffffffffu, lo, o);
    double s, e;
    two_sum(hi, ohi, s, e);
    hi = s;
    lo = __dadd_rn(__dadd_rn(lo, olo), e);
  }
  double s, e;
  two_sum(hi, lo, s, e);
  return s;
}

// Order key of an exact fp64 score for (score desc) ranking with integer
// compares: a larger score gives a smaller key; -0.0 and +0.0 share a key
// (they compare equal, so the id decides, as with the reference's
// std::sort comparator).  Scores are finite.
__device__ __forceinline__ uint64_t score_desc_key(double d) {
  uint64_t u = (uint64_t)__double_as_longlong(d == 0.0 ? 0.0 : d);
  u = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  return ~u;
}

}  // namespace dev
}  // namespace hsd

namespace hsd {
// Launch `kern` as a programmatic dependent of the previous kernel on `s`.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace hsd
