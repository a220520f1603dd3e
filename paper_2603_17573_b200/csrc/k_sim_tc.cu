// k_sim_tc.cu — K1' (tensor cores): 3xTF32 similarity on tcgen05 + TMA,
// fused with the per-CTA top-32 candidate filter.
//
// S = K·Q^T for 128-key blocks against a 64-query slab, split-precision so the
// filter scores carry ~fp32 accuracy (error bound in sim_plan_tc):
//     K = Kh + Kl,  Q = Qh + Ql      (h = TF32-truncated, l = exact remainder)
//     S ~= Kh·Qh + (Kh·Ql + Kl·Qh)
//   MMA1 (SS): A = raw key tile (smem, TMA SWIZZLE_128B, read as TF32 = Kh),
//              B = [Qh | Ql] (N = 128)  -> TMEM cols [0,64) Kh·Qh, [64,128) Kh·Ql
//   MMA2 (TS): A = Kl (TMEM, written by the split warps with tcgen05.st),
//              B = Qh (N = 64)          -> accumulates into cols [64,128)
// Both products share one pass of the key tile through shared memory; Kl never
// touches shared memory.  Three accumulators (3 x 128 key rows) live in TMEM
// so each query chunk staged in smem is reused for 3 key tiles.
//
// Warp roles (384 threads, 1 CTA per SM, persistent over a contiguous range of
// key blocks):
//   warp 0      TMA producer (keys ring, query ring)
//   warp 1      tcgen05.mma issuer (single elected lane)
//   warp 2      TMEM allocator
//   warps 4-7   split: Kl = K - trunc_tf32(K) -> TMEM (tcgen05.st)
//   warps 8-11  epilogue: tcgen05.ld scores -> per-query candidate filter
// Every synchronisation is an mbarrier (TMA complete_tx, tcgen05.commit,
// thread arrivals); the epilogue warpgroup uses a named barrier.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace hsd {
namespace {

using dev::cand_key;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kBM = 128;       // keys per block (UMMA M)
constexpr int kBQ = 64;        // queries per slab
constexpr int kBK = 32;        // fp32 per k-chunk (one 128-B swizzle atom)
constexpr int kGB = 3;         // key blocks per group (accumulators in TMEM)
constexpr int kKStages = 9;    // key ring (16 KB per stage): 144 KB of HBM reads in flight per SM
constexpr int kQStages = 2;    // query ring (16 KB per stage: Qh rows 0-63, Ql rows 64-127)
constexpr int kLStages = 4;    // Kl stages in TMEM (32 columns each)
constexpr int kAccCols = 128;  // per key block
constexpr int kKlCol0 = kGB * kAccCols;  // 384
constexpr int kTmemCols = 512;
constexpr int kThreads = 384;
constexpr int kTileBytes = kBM * kBK * 4;  // 16 KB
constexpr int kStg = kBQ + 1;              // padded row of the score staging tile

// Candidate filter: the 4 epilogue warps own queries q % 4 == w; each keeps the
// running sorted top-32 of each of its queries in registers (one key per
// lane).  Per 128-key block the scores are staged through shared memory
// (row-major, padded: conflict-free), each warp tests its queries' 128 keys
// against the lane-31 threshold with one ballot, and inserts the (rare, ~32/n
// at the n-th block) survivors one by one with a shuffle shift.
struct __align__(1024) TcSmem {
  float kbuf[kKStages][kBM * kBK];
  float qbuf[kQStages][128 * kBK];
  float stg[kBM * kStg];
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t q_full[kQStages], q_empty[kQStages];
  uint64_t l_full[kLStages], l_empty[kLStages];
  uint64_t acc_full, acc_empty;
  uint32_t tmem_base;
};

// ------------------------------------------------------------------ PTX helpers
using namespace sm100;
// ------------------------------------------------------------------ kernel
template <bool kDump>
__global__ void __launch_bounds__(kThreads, 1)
    sim_tc_kernel(const __grid_constant__ CUtensorMap keys_map, const __grid_constant__ CUtensorMap qh_map,
                  const __grid_constant__ CUtensorMap ql_map, int64_t row_begin, int64_t row_end, int dim, int B,
                  int64_t blocks_per_cta, uint64_t* __restrict__ partial, float* __restrict__ dump) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // keep the pointer derived from the __shared__ array so accesses stay LDS/STS
  TcSmem& S = *reinterpret_cast<TcSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t blk0 = (int64_t)blockIdx.x * blocks_per_cta;
  const int64_t blk1 = std::min<int64_t>(blk0 + blocks_per_cta, n_blocks);
  const int nk = (dim + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&S.k_full[i], 1);
      mbar_init(&S.k_empty[i], 1 + 4);  // MMA commit + 4 split warps
    }
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], 1);
    }
    for (int i = 0; i < kLStages; ++i) {
      mbar_init(&S.l_full[i], 4);
      mbar_init(&S.l_empty[i], 1);
    }
    mbar_init(&S.acc_full, 1);
    mbar_init(&S.acc_empty, 4);
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

  if (warp == 3) {
    // ======================= TMA producer: query chunks (L2-resident, reused by gb key tiles)
    if (lane == 0 && blk0 < blk1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&qh_map) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&ql_map) : "memory");
      const uint64_t pol_q = policy_evict_last();
      int qs = 0;
      uint32_t qph = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB) {
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.q_empty[qs], qph ^ 1);
          mbar_expect_tx(&S.q_full[qs], kTileBytes);
          tma_load_2d(&S.qbuf[qs][0], &qh_map, &S.q_full[qs], kc * kBK, 0, pol_q);
          tma_load_2d(&S.qbuf[qs][64 * kBK], &ql_map, &S.q_full[qs], kc * kBK, 0, pol_q);
          if (++qs == kQStages) {
            qs = 0;
            qph ^= 1;
          }
        }
      }
    }
  } else if (warp == 0) {
    // ======================= TMA producer: key tiles (HBM stream, runs kKStages ahead)
    if (lane == 0 && blk0 < blk1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&keys_map) : "memory");
      const uint64_t pol_k = policy_evict_first();
      int ks = 0;
      uint32_t kph = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB) {
        const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
        for (int kc = 0; kc < nk; ++kc) {
          for (int m = 0; m < gb; ++m) {
            mbar_wait(&S.k_empty[ks], kph ^ 1);
            mbar_expect_tx(&S.k_full[ks], kTileBytes);
            tma_load_2d(&S.kbuf[ks][0], &keys_map, &S.k_full[ks], kc * kBK, (int)(row_begin + (g0 + m) * kBM), pol_k);
            if (++ks == kKStages) {
              ks = 0;
              kph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer
    constexpr uint32_t idesc1 = tf32_idesc(128, 128);
    constexpr uint32_t idesc2 = tf32_idesc(128, 64);
    int ks = 0, qs = 0, ls = 0;
    uint32_t kph = 0, qph = 0, lph = 0;
    int gi = 0;
    // stage s of a 16-KB ring sits 16384 B = 1024 descriptor units further
    const uint64_t adesc0 = sw128_desc(&S.kbuf[0][0]);
    const uint64_t bdesc0 = sw128_desc(&S.qbuf[0][0]);
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      if (gi > 0) {
        mbar_wait(&S.acc_empty, (gi - 1) & 1);
        tc_fence_after();
      }
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&S.q_full[qs], qph);
        const uint64_t bdesc = bdesc0 + (uint64_t)(qs * (kTileBytes >> 4));
        for (int m = 0; m < gb; ++m) {
          mbar_wait(&S.k_full[ks], kph);
          mbar_wait(&S.l_full[ls], lph);
          tc_fence_after();
          const uint64_t adesc = adesc0 + (uint64_t)(ks * (kTileBytes >> 4));
          const uint32_t d = tmem + m * kAccCols;
          const uint32_t kl = tmem + kKlCol0 + ls * kBK;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            // +32 B per K-step of 8 tf32 (descriptor address field is in 16-B units)
            mma_ss(d, adesc + 2 * kk, bdesc + 2 * kk, idesc1, (kc > 0 || kk > 0) ? 1u : 0u);
            mma_ts(d + 64, kl + 8 * kk, bdesc + 2 * kk, idesc2, 1u);
          }
          tc_commit(&S.k_empty[ks]);
          tc_commit(&S.l_empty[ls]);
          if (++ks == kKStages) {
            ks = 0;
            kph ^= 1;
          }
          if (++ls == kLStages) {
            ls = 0;
            lph ^= 1;
          }
        }
        tc_commit(&S.q_empty[qs]);
        if (++qs == kQStages) {
          qs = 0;
          qph ^= 1;
        }
      }
      tc_commit(&S.acc_full);
    }
  } else if (warp >= 4 && warp < 8) {
    // ======================= split: Kl = K - trunc_tf32(K) -> TMEM
    const int r = (warp - 4) * 32 + lane;  // key row within the tile == TMEM lane
    const uint32_t lane_addr = (uint32_t)((warp - 4) * 32) << 16;
    int ks = 0, ls = 0;
    uint32_t kph = 0, lph = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      for (int kc = 0; kc < nk; ++kc) {
        for (int m = 0; m < gb; ++m) {
          mbar_wait(&S.k_full[ks], kph);
          mbar_wait(&S.l_empty[ls], lph ^ 1);
          tc_fence_after();
          const unsigned char* row = reinterpret_cast<const unsigned char*>(&S.kbuf[ks][0]) + r * 128;
          uint32_t lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(row + ((c ^ (r & 7)) << 4));
            const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float h = __uint_as_float(__float_as_uint(x[j]) & 0xFFFFE000u);
              lo[c * 4 + j] = __float_as_uint(x[j] - h);
            }
          }
          TMEM_ST32(tmem + lane_addr + kKlCol0 + ls * kBK, lo);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&S.l_full[ls]);
            mbar_arrive(&S.k_empty[ks]);
          }
          if (++ks == kKStages) {
            ks = 0;
            kph ^= 1;
          }
          if (++ls == kLStages) {
            ls = 0;
            lph ^= 1;
          }
        }
      }
    }
  } else if (warp >= 8) {
    // ======================= epilogue: scores -> candidate filter
    const int ew = warp - 8;
    const int r = ew * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(ew * 32) << 16;
    constexpr int kMyQ = kBQ / 4;  // queries owned by this warp: q = ew + 4 i
    uint64_t top[kMyQ];
#pragma unroll
    for (int i = 0; i < kMyQ; ++i) top[i] = kEmpty;
    int gi = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      mbar_wait(&S.acc_full, gi & 1);
      tc_fence_after();
      for (int m = 0; m < gb; ++m) {
        const int64_t base = row_begin + (g0 + m) * kBM;
        // 1. TMEM -> registers -> staging tile (S~ = hi*hi + corrections)
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t hi[32], cr[32];
          TMEM_LD32(tmem + lane_addr + m * kAccCols + half * 32, hi);
          TMEM_LD32(tmem + lane_addr + m * kAccCols + 64 + half * 32, cr);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float s = __uint_as_float(hi[j]) + __uint_as_float(cr[j]);
            if (kDump) {
              const int q = half * 32 + j;
              if (base + r < row_end && q < B) dump[(size_t)q * (row_end - row_begin) + (base + r - row_begin)] = s;
            } else {
              S.stg[r * kStg + half * 32 + j] = s;
            }
          }
        }
        if (m == gb - 1) {  // accumulators drained: the next group's MMAs may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.acc_empty);
        }
        if (kDump) continue;
        named_sync(1, 128);
        // 2. filter: one ballot per (query, 32 keys); rare survivors inserted by shuffle shift
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

// Q [B][dim] -> Qh = trunc_tf32(Q), Ql = Q - Qh, zero-padded to 64 rows.
__global__ void split_queries_kernel(const float* __restrict__ q, int B, int dim, float* __restrict__ qh,
                                     float* __restrict__ ql) {
  const int row = blockIdx.x;
  for (int c = threadIdx.x; c < dim; c += blockDim.x) {
    const float x = row < B ? q[(size_t)row * dim + c] : 0.f;
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    qh[(size_t)row * dim + c] = h;
    ql[(size_t)row * dim + c] = x - h;
  }
}

bool make_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t dim, uint32_t box_rows) {
  return tc_make_map(m, base, rows, dim, box_rows);
}

}  // namespace

size_t sim_tc_scratch_bytes(int dim) { return 2ull * kBQ * dim * sizeof(float); }

double sim_tc_gamma(int dim) {
  // |S - S~| <= gamma * sum|k_i q_i|:  split/representation error 3 * 2^-20
  // (|Kl|,|Ql| < 2^-10 |.|, TF32 rounding of the remainders, dropped Kl*Ql)
  // plus fp32 accumulation of 3 * dim products at <= 2^-23 relative each.
  return 3.0 / 1048576.0 + (3.0 * dim + 16.0) / 8388608.0;
}

int sim_tc_lists(int64_t rows, int num_sms) {
  const int64_t blocks = (rows + kBM - 1) / kBM;
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, num_sms));
}

cudaError_t launch_sim_tc(const float* keys, int64_t n_keys_total, int64_t row_begin, int64_t row_end, int dim,
                          const float* queries, int B, int lists, float* scratch, uint64_t* partial, float* dump,
                          cudaStream_t s) {
  if (B < 1 || B > kBQ) return cudaErrorInvalidValue;
  float* qh = scratch;
  float* ql = scratch + (size_t)kBQ * dim;
  split_queries_kernel<<<kBQ, 256, 0, s>>>(queries, B, dim, qh, ql);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  CUtensorMap km, qhm, qlm;
  if (!make_map(&km, keys, (uint64_t)n_keys_total, (uint64_t)dim, kBM) || !make_map(&qhm, qh, kBQ, dim, kBQ) ||
      !make_map(&qlm, ql, kBQ, dim, kBQ))
    return cudaErrorInvalidValue;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t per = (n_blocks + lists - 1) / lists;
  const size_t smem = sizeof(TcSmem) + 1024;
  if (dump) {
    e = cudaFuncSetAttribute(sim_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sim_tc_kernel<true><<<lists, kThreads, smem, s>>>(km, qhm, qlm, row_begin, row_end, dim, B, per, partial, dump);
  } else {
    e = cudaFuncSetAttribute(sim_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sim_tc_kernel<false><<<lists, kThreads, smem, s>>>(km, qhm, qlm, row_begin, row_end, dim, B, per, partial, dump);
  }
  return cudaGetLastError();
}

}  // namespace hsd
