// k_sim_tc1.cu — K1 (tensor cores, default path): TF32 similarity filter on
// tcgen05 + TMA, fused with the per-CTA top-32 candidate filter.
//
// The tensor cores only FILTER: S~ = K·Q^T with operands read as TF32 from
// the raw fp32 tiles.  |S - S~| <= gamma_tf32 * sum|k_i q_i| (sim_tc1_gamma),
// and the select kernel (k_select.cu) keeps every record whose S~ lies within
// 2E of the k-th best and rescores it with the reference's sequential fp64 dot
// — so the final ids/scores are bit-identical to store.cpp while the scan runs
// at the HBM roofline.  (k_sim_tc.cu holds the 3xTF32 variant with a ~10x
// tighter filter at ~1.5x the shared-memory traffic.)
//
// Per SM (persistent CTA over a contiguous range of 128-key blocks):
//   warp 0     TMA producer: key tiles 128 rows x 32 fp32 (16 KB, SWIZZLE_128B),
//              kKStages-deep ring (the HBM stream)
//   warp 3     TMA producer: query chunks 64 x 32 fp32 (8 KB, L2-resident)
//   warp 1     tcgen05.mma issuer: per stage 4 x (M128 N64 K8) kind::tf32 into
//              the accumulator of the stage's key block
//   warp 2     TMEM allocator (512 columns = 2 buffers x 4 blocks x 64 queries)
//   warps 4-7  epilogue: tcgen05.ld -> staging tile -> ballot filter against
//              the register-resident per-query top-32
// Accumulators are double-buffered, so the epilogue of group g overlaps the
// MMAs of group g+1; each staged query chunk is reused by 4 key tiles.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace hsd {
namespace {

using namespace sm100;
using dev::cand_key;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kBM = 128;   // keys per block (UMMA M)
constexpr int kBQ = 64;    // queries per slab (UMMA N)
constexpr int kBK = 32;    // fp32 per k-chunk (one 128-B swizzle atom)
constexpr int kGB = 4;     // key blocks per accumulator buffer (query-chunk reuse)
constexpr int kKStages = 9;
constexpr int kQStages = 4;
constexpr int kThreads = 256;
constexpr int kTmemCols = 512;
constexpr int kBufCols = kGB * kBQ;  // 256
constexpr int kKeyTile = kBM * kBK * 4;  // 16 KB
constexpr int kQTile = kBQ * kBK * 4;    // 8 KB
constexpr int kStg = kBQ + 1;

struct __align__(1024) Tc1Smem {
  float kbuf[kKStages][kBM * kBK];
  float qbuf[kQStages][kBQ * kBK];
  float stg[kBM * kStg];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t q_full[kQStages], q_empty[kQStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

template <bool kDump>
__global__ void __launch_bounds__(kThreads, 1)
    sim_tc1_kernel(const __grid_constant__ CUtensorMap keys_map, const __grid_constant__ CUtensorMap q_map,
                   int64_t row_begin, int64_t row_end, int dim, int B, int64_t blocks_per_cta,
                   uint64_t* __restrict__ partial, float* __restrict__ dump) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Tc1Smem& S = *reinterpret_cast<Tc1Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t blk0 = (int64_t)blockIdx.x * blocks_per_cta;
  const int64_t blk1 = std::min<int64_t>(blk0 + blocks_per_cta, n_blocks);
  const int nk = (dim + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&S.k_full[i], 1);
      mbar_init(&S.k_empty[i], 1);
    }
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.acc_full[i], 1);
      mbar_init(&S.acc_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ======================= key stream (HBM)
    if (lane == 0 && blk0 < blk1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&keys_map) : "memory");
      const uint64_t pol = policy_evict_first();
      int ks = 0;
      uint32_t kph = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB) {
        const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
        for (int kc = 0; kc < nk; ++kc)
          for (int m = 0; m < gb; ++m) {
            mbar_wait(&S.k_empty[ks], kph ^ 1);
            mbar_expect_tx(&S.k_full[ks], kKeyTile);
            tma_load_2d(&S.kbuf[ks][0], &keys_map, &S.k_full[ks], kc * kBK, (int)(row_begin + (g0 + m) * kBM), pol);
            if (++ks == kKStages) {
              ks = 0;
              kph ^= 1;
            }
          }
      }
    }
  } else if (warp == 3) {
    // ======================= query chunks (L2-resident, reused by gb key tiles)
    if (lane == 0 && blk0 < blk1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&q_map) : "memory");
      const uint64_t pol = policy_evict_last();
      int qs = 0;
      uint32_t qph = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB)
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.q_empty[qs], qph ^ 1);
          mbar_expect_tx(&S.q_full[qs], kQTile);
          tma_load_2d(&S.qbuf[qs][0], &q_map, &S.q_full[qs], kc * kBK, 0, pol);
          if (++qs == kQStages) {
            qs = 0;
            qph ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (whole warp; one lane elected in the asm)
    constexpr uint32_t idesc = tf32_idesc(kBM, kBQ);
    const uint64_t adesc0 = sw128_desc(&S.kbuf[0][0]);
    const uint64_t bdesc0 = sw128_desc(&S.qbuf[0][0]);
    int ks = 0, qs = 0;
    uint32_t kph = 0, qph = 0;
    int gi = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      const int buf = gi & 1;
      if (gi >= 2) {
        mbar_wait(&S.acc_empty[buf], ((gi >> 1) - 1) & 1);
        tc_fence_after();
      }
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&S.q_full[qs], qph);
        const uint64_t bdesc = bdesc0 + (uint64_t)(qs * (kQTile >> 4));
        for (int m = 0; m < gb; ++m) {
          mbar_wait(&S.k_full[ks], kph);
          tc_fence_after();
          const uint64_t adesc = adesc0 + (uint64_t)(ks * (kKeyTile >> 4));
          const uint32_t d = tmem + buf * kBufCols + m * kBQ;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk)  // +32 B per K-step of 8 tf32
            mma_ss(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
          tc_commit(&S.k_empty[ks]);
          if (++ks == kKStages) {
            ks = 0;
            kph ^= 1;
          }
        }
        tc_commit(&S.q_empty[qs]);
        if (++qs == kQStages) {
          qs = 0;
          qph ^= 1;
        }
      }
      tc_commit(&S.acc_full[buf]);
    }
  } else if (warp >= 4) {
    // ======================= epilogue
    const int ew = warp - 4;  // TMEM lane quadrant
    const int r = ew * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(ew * 32) << 16;
    constexpr int kMyQ = kBQ / 4;  // queries q = ew + 4 i owned by this warp
    uint64_t top[kMyQ];
#pragma unroll
    for (int i = 0; i < kMyQ; ++i) top[i] = kEmpty;
    int gi = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      const int buf = gi & 1;
      mbar_wait(&S.acc_full[buf], (gi >> 1) & 1);
      tc_fence_after();
      for (int m = 0; m < gb; ++m) {
        const int64_t base = row_begin + (g0 + m) * kBM;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t acc[32];
          TMEM_LD32(tmem + lane_addr + buf * kBufCols + m * kBQ + half * 32, acc);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s = __uint_as_float(acc[j]);
            if (kDump) {
              const int q = half * 32 + j;
              if (base + r < row_end && q < B) dump[(size_t)q * (row_end - row_begin) + (base + r - row_begin)] = s;
            } else {
              S.stg[r * kStg + half * 32 + j] = s;
            }
          }
        }
        if (m == gb - 1) {  // buffer drained: the MMAs of group gi+2 may reuse it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.acc_empty[buf]);
        }
        if (kDump) continue;
        named_sync(1, 128);
#pragma unroll
        for (int i = 0; i < kMyQ; ++i) {
          const int q = ew + 4 * i;
          if (q < B) {
            uint64_t key[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int rr = lane + 32 * j;
              key[j] = base + rr < row_end ? cand_key(S.stg[rr * kStg + q], (uint32_t)(base + rr)) : kEmpty;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t mask = __ballot_sync(0xffffffffu, key[j] < dev::shfl_u64(top[i], 31));
              while (mask) {
                const int src = __ffs(mask) - 1;
                mask &= mask - 1;
                const uint64_t x = dev::shfl_u64(key[j], src);
                const int pos = __popc(__ballot_sync(0xffffffffu, top[i] < x));
                if (pos < 32) {
                  const uint64_t up = dev::shfl_u64(top[i], (lane + 31) & 31);
                  top[i] = lane < pos ? top[i] : (lane == pos ? x : up);
                }
              }
            }
          }
        }
        named_sync(1, 128);
      }
    }
    if (!kDump) {
#pragma unroll
      for (int i = 0; i < kMyQ; ++i) {
        const int q = ew + 4 * i;
        if (q < B) partial[((size_t)blockIdx.x * B + q) * kCandLocal + lane] = top[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// Zero-padded copy of the query slab to 64 rows (the TMA box).
__global__ void pad_queries_kernel(const float* __restrict__ q, int B, int dim, float* __restrict__ out) {
  const int row = blockIdx.x;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) out[(size_t)row * dim + c] = row < B ? q[(size_t)row * dim + c] : 0.f;
}

}  // namespace

double sim_tc1_gamma(int dim) {
  // Operands read as TF32: |x - tf32(x)| <= 2^-10 |x| (truncation; 2^-11 if
  // rounded), so |kq - k'q'| <= (2^-10 + 2^-10 (1 + 2^-10)) |k||q| per
  // product; plus fp32 accumulation of dim products at <= 2^-23 relative each
  // (the tensor core accumulator is not round-to-nearest).
  return (2.0 + 1.0 / 1024.0) / 1024.0 * 1.0001 + (dim + 16.0) / 8388608.0;
}

size_t sim_tc1_scratch_bytes(int dim) { return (size_t)kBQ * dim * sizeof(float); }

cudaError_t launch_sim_tc1(const float* keys, int64_t n_keys_total, int64_t row_begin, int64_t row_end, int dim,
                           const float* queries, int B, int lists, float* scratch, uint64_t* partial, float* dump,
                           cudaStream_t s) {
  if (B < 1 || B > kBQ) return cudaErrorInvalidValue;
  pad_queries_kernel<<<kBQ, 256, 0, s>>>(queries, B, dim, scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap km, qm;
  if (!tc_make_map(&km, keys, (uint64_t)n_keys_total, (uint64_t)dim, kBM) ||
      !tc_make_map(&qm, scratch, kBQ, (uint64_t)dim, kBQ))
    return cudaErrorInvalidValue;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t per = (n_blocks + lists - 1) / lists;
  const size_t smem = sizeof(Tc1Smem) + 1024;
  if (dump) {
    e = cudaFuncSetAttribute(sim_tc1_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sim_tc1_kernel<true><<<lists, kThreads, smem, s>>>(km, qm, row_begin, row_end, dim, B, per, partial, dump);
  } else {
    e = cudaFuncSetAttribute(sim_tc1_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sim_tc1_kernel<false><<<lists, kThreads, smem, s>>>(km, qm, row_begin, row_end, dim, B, per, partial, dump);
  }
  return cudaGetLastError();
}

}  // namespace hsd
