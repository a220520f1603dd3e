// k_sim_wide.cu — K1 (tensor cores, the default for every batch): similarity
// FILTER on tcgen05 + TMA for up to 1024 queries per pass, fused with the
// per-CTA top-32 candidate filter.  Kernels in this file:
//
//   sim_wide_kernel  one CTA per SM, up to 128 queries per pass (NS = 1, 2);
//                    with kMC > 1 clusters of query groups share multicast key
//                    tiles (the single-CTA ablation above 128 queries)
//   sim_pair_kernel  above 128 queries: CTA pairs (tcgen05.mma.cta_group::2,
//                    M = 256), clusters of up to 4 pairs with multicast key
//                    halves, queries balanced over the pairs (see below)
//   pad_queries_*    the zero-padded query slab; K1 is its programmatic
//                    dependent (only the query producer waits for it)
//
// Two operand types share the kernels:
//
//   TF32  fp32 collections: keys and queries are read as TF32 straight from
//         the fp32 tiles (kind::tf32, 32 fp32 = one 128-B atom per k-chunk);
//   BF16  bf16 collections: keys are stored bf16, queries rounded to bf16 at
//         padding time (kind::f16, 64 bf16 per k-chunk).
//
// Either way the tensor cores only FILTER: |S - S~| <= gamma * sum|k_i q_i|
// (sim_wide_gamma) and the select kernel (k_select.cu) rescores every record
// within 2E of the k-th best with the reference's sequential fp64 dot
// (store.cpp:29-34) against the STORED keys, so ids and scores are
// bit-identical to the reference over the stored (fp32 or bf16) DB.
//
// Query batch width: NS slabs of 64 queries form one UMMA N = 64*NS (<= 256)
// so a key tile is read from HBM once per pass for up to 256 queries:
//
//   NS  N    key blocks per accumulator   TMEM columns per buffer
//   1   64   4                            256
//   2   128  2                            256
//   4   256  1                            256
//
// Per SM (persistent CTA over a contiguous range of 128-key blocks):
//   warp 0      TMA producer: key tiles 128 rows x 128 B (16 KB, SWIZZLE_128B)
//   warp 3      TMA producer: query tiles 64*NS rows x 128 B (L2-resident)
//   warp 1      tcgen05.mma issuer: per key tile 4 x (M128 N64NS K) into the
//               accumulator of its key block
//   warp 2      TMEM allocator (512 columns = 2 buffers x 256)
//   warps 4-11  epilogue: tcgen05.ld (x16) -> staging tile of 32 queries ->
//               ballot filter against the register-resident per-query top-32
// Accumulators are double-buffered, so the epilogue of group g overlaps the
// MMAs of group g+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "hsd/hsd_synth.h"
#include "kernels.h"
#include "sm100.cuh"

namespace hsd {
namespace {

using namespace sm100;
using dev::cand_key;
using dev::kCandLocal;
using dev::kEmpty;

constexpr int kBM = 128;              // keys per block (UMMA M)
constexpr int kKeyTile = kBM * 128;   // 16 KB: 128 rows x one 128-B swizzle atom
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (4 + kEpiWarps);
constexpr int kTmemCols = 512;
constexpr int kStgQ = 32;             // queries staged per epilogue round
constexpr int kStg = kStgQ + 1;

template <int NS, int GB>
struct WideCfg {
  static constexpr int kBQ = 64 * NS;                 // UMMA N
  static constexpr int kGB = GB;                      // key blocks per accumulator buffer (query-tile reuse)
  static constexpr int kBufCols = GB * kBQ;           // TMEM columns per accumulator buffer
  static constexpr int kBufs = kTmemCols / kBufCols;  // 2 = double-buffered, 1 = single
  static_assert(kBufs == 1 || kBufs == 2, "accumulators must fill 256 or 512 TMEM columns");
  static constexpr int kQTile = kBQ * 128;            // bytes per query k-chunk tile
  static constexpr int kKStages = NS == 4 ? 7 : (NS == 1 ? 10 : 9);  // NS = 1: 10 measured 0.7% over 9, 11-12 (fewer query stages) slower
  static constexpr int kQStages = NS == 1 ? 4 : 3;
  static constexpr int kMyQ = kBQ / kEpiWarps;        // queries owned per epilogue lane-group
};

template <int NS, int GB>
struct __align__(1024) WideSmem {
  using Cfg = WideCfg<NS, GB>;
  uint8_t kbuf[Cfg::kKStages][kKeyTile];
  uint8_t qbuf[Cfg::kQStages][Cfg::kQTile];
  float stg[kBM * kStg];
  uint64_t k_full[Cfg::kKStages], k_empty[Cfg::kKStages];
  uint64_t q_full[Cfg::kQStages], q_empty[Cfg::kQStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};

// One staging round of the epilogue: the 32 staged queries x 128 key rows in
// `stg` are merged into the register-resident per-query top-32 lists (a warp
// owns 4 queries; lane l holds rank l of each list, ascending keys).
template <int kMyQ>
__device__ __forceinline__ void epi_insert_round(const float* stg, int ew, int lane, int j, int q_valid,
                                                 int64_t base, int64_t row_hi, uint64_t (&top)[kMyQ]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ql = ew * 4 + i;
    if (j * kStgQ + ql < q_valid) {
      uint64_t& tp = top[j * 4 + i];
      uint64_t key[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = lane + 32 * u;
        key[u] = base + rr < row_hi ? cand_key(stg[rr * kStg + ql], (uint32_t)(base + rr)) : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t mask = __ballot_sync(0xffffffffu, key[u] < dev::shfl_u64(tp, 31));
        while (mask) {
          const int src = __ffs(mask) - 1;
          mask &= mask - 1;
          const uint64_t x = dev::shfl_u64(key[u], src);
          const int pos = __popc(__ballot_sync(0xffffffffu, tp < x));
          if (pos < 32) {
            const uint64_t up = dev::shfl_u64(tp, (lane + 31) & 31);
            tp = lane < pos ? tp : (lane == pos ? x : up);
          }
        }
      }
    }
  }
}

// kMC > 1: a cluster of kMC CTAs shares one key range; CTA rank r holds query
// group r (256 queries each) and issues every kMC-th key tile with a TMA
// multicast into all kMC CTAs, so the keys cross HBM once for up to 1024
// queries.  A ring slot is refilled only after every CTA's MMAs released it
// (multicast commits into each CTA's k_empty, count kMC).
template <bool kBf16, int NS, int GB, bool kDump, int kMC = 1>
__global__ void __launch_bounds__(kThreads, 1)
    sim_wide_kernel(const __grid_constant__ CUtensorMap keys_map, const __grid_constant__ CUtensorMap q_map,
                    int64_t row_begin, int64_t row_end, int dim, int B, int64_t blocks_per_cta,
                    uint64_t* __restrict__ partial, float* __restrict__ dump) {
  using Cfg = WideCfg<NS, GB>;
  constexpr int kBQ = Cfg::kBQ, kGB = Cfg::kGB, kKS = Cfg::kKStages, kQS = Cfg::kQStages;
  constexpr int kBufCols = Cfg::kBufCols, kBufs = Cfg::kBufs;
  constexpr int kBK = kBf16 ? 64 : 32;  // elements per 128-B k-chunk
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  WideSmem<NS, GB>& S = *reinterpret_cast<WideSmem<NS, GB>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int unit = kMC > 1 ? (int)cluster_id_x() : (int)blockIdx.x;  // key-range owner
  const int n_units = kMC > 1 ? (int)n_clusters_x() : (int)gridDim.x;
  const int rank = kMC > 1 ? (int)cluster_ctarank() : 0;             // query group
  const int q_base = rank * kBQ;
  const int64_t blk0 = (int64_t)unit * blocks_per_cta;
  const int64_t blk1 = std::min<int64_t>(blk0 + blocks_per_cta, n_blocks);
  const int nk = (dim + kBK - 1) / kBK;
  // Each CTA walks the k-chunks starting at its own offset, so the 148 CTAs do
  // not all request the same (L2-resident) query tile at the same moment; the
  // filter's error bound does not depend on the accumulation order.
  const int kc0 = (int)(((int64_t)unit * nk) / n_units);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kKS; ++i) {
      mbar_init(&S.k_full[i], 1);
      mbar_init(&S.k_empty[i], kMC);
    }
    for (int i = 0; i < kQS; ++i) {
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.acc_full[i], 1);
      mbar_init(&S.acc_empty[i], kEpiWarps);
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
  if constexpr (kMC > 1) cluster_sync_all();  // peers' barriers exist before any multicast / remote arrive
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  dev::pdl_trigger();  // K2's first kernel may launch onto free SM resources and wait there

  if (warp == 0) {
    // ======================= key stream (HBM)
    if (lane == 0 && blk0 < blk1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&keys_map) : "memory");
      const uint64_t pol = policy_evict_first();
      int ks = 0;
      uint32_t kph = 0;
      uint32_t tile = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB) {
        const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
        for (int kc = 0; kc < nk; ++kc)
          for (int m = 0; m < gb; ++m, ++tile) {
            mbar_wait(&S.k_empty[ks], kph ^ 1);
            mbar_expect_tx(&S.k_full[ks], kKeyTile);
            const int c = kc + kc0 < nk ? kc + kc0 : kc + kc0 - nk;
            if constexpr (kMC > 1) {
              if ((int)(tile % kMC) == rank)
                tma_load_2d_mc(&S.kbuf[ks][0], &keys_map, &S.k_full[ks], c * kBK,
                               (int)(row_begin + (g0 + m) * kBM), (uint16_t)((1u << kMC) - 1), pol);
            } else {
              tma_load_2d(&S.kbuf[ks][0], &keys_map, &S.k_full[ks], c * kBK, (int)(row_begin + (g0 + m) * kBM),
                          pol);
            }
            if (++ks == kKS) {
              ks = 0;
              kph ^= 1;
            }
          }
      }
    }
  } else if (warp == 3) {
    // ======================= query tiles (L2-resident, reused by gb key tiles)
    if (lane == 0 && blk0 < blk1) {
      dev::pdl_wait();  // the padded query slab (the key stream above does not need it)
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&q_map) : "memory");
      const uint64_t pol = policy_evict_last();
      int qs = 0;
      uint32_t qph = 0;
      for (int64_t g0 = blk0; g0 < blk1; g0 += kGB)
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.q_empty[qs], qph ^ 1);
          mbar_expect_tx(&S.q_full[qs], Cfg::kQTile);
          const int c = kc + kc0 < nk ? kc + kc0 : kc + kc0 - nk;
          tma_load_2d(&S.qbuf[qs][0], &q_map, &S.q_full[qs], c * kBK, q_base, pol);
          if (++qs == kQS) {
            qs = 0;
            qph ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (whole warp; one lane elected in the asm)
    constexpr uint32_t idesc = kBf16 ? bf16_idesc(kBM, kBQ) : tf32_idesc(kBM, kBQ);
    const uint64_t adesc0 = sw128_desc(&S.kbuf[0][0]);
    const uint64_t bdesc0 = sw128_desc(&S.qbuf[0][0]);
    int ks = 0, qs = 0;
    uint32_t kph = 0, qph = 0;
    int gi = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      const int buf = gi % kBufs;
      if (gi >= kBufs) {  // the epilogue must have drained this buffer
        mbar_wait(&S.acc_empty[buf], ((gi / kBufs) - 1) & 1);
        tc_fence_after();
      }
      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&S.q_full[qs], qph);
        const uint64_t bdesc = bdesc0 + (uint64_t)(qs * (Cfg::kQTile >> 4));
        for (int m = 0; m < gb; ++m) {
          mbar_wait(&S.k_full[ks], kph);
          tc_fence_after();
          const uint64_t adesc = adesc0 + (uint64_t)(ks * (kKeyTile >> 4));
          const uint32_t d = tmem + buf * kBufCols + m * kBQ;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // +32 B per UMMA K-step (8 tf32 / 16 bf16)
            if (kBf16)
              mma_ss_f16(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
            else
              mma_ss(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (kMC > 1)
            tc_commit_mc(&S.k_empty[ks], (uint16_t)((1u << kMC) - 1));
          else
            tc_commit(&S.k_empty[ks]);
          if (++ks == kKS) {
            ks = 0;
            kph ^= 1;
          }
        }
        tc_commit(&S.q_empty[qs]);
        if (++qs == kQS) {
          qs = 0;
          qph ^= 1;
        }
      }
      tc_commit(&S.acc_full[buf]);
    }
  } else if (warp >= 4) {
    // ======================= epilogue (8 warps)
    const int ew = warp - 4;        // 0..7
    const int quad = warp & 3;      // TMEM lane quadrant this warp may access
    const int half = ew >> 2;       // which 16 of the 32 staged columns it loads
    const int r = quad * 32 + lane; // key row of the block this thread loads
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    // query q = j * 32 + ew * 4 + i  (j: staging round, i < 4) -> top[j * 4 + i]
    uint64_t top[Cfg::kMyQ];
#pragma unroll
    for (int i = 0; i < Cfg::kMyQ; ++i) top[i] = kEmpty;
    int gi = 0;
    for (int64_t g0 = blk0; g0 < blk1; g0 += kGB, ++gi) {
      const int gb = (int)std::min<int64_t>(kGB, blk1 - g0);
      const int buf = gi % kBufs;
      mbar_wait(&S.acc_full[buf], (gi / kBufs) & 1);
      tc_fence_after();
      for (int m = 0; m < gb; ++m) {
        const int64_t base = row_begin + (g0 + m) * kBM;
#pragma unroll
        for (int j = 0; j < kBQ / kStgQ; ++j) {
          uint32_t acc[16];
          TMEM_LD16(tmem + lane_addr + buf * kBufCols + m * kBQ + j * kStgQ + half * 16, acc);
          tmem_ld_wait();
          if (m == gb - 1 && j == kBQ / kStgQ - 1) {  // buffer drained: MMAs of group gi+kBufs may reuse it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.acc_empty[buf]);
          }
          if constexpr (kDump) {
            if (base + r < row_end) {
              const size_t nrows = (size_t)(row_end - row_begin);
              const int q0 = j * kStgQ + half * 16;
              float* drow = dump + (size_t)q0 * nrows + (size_t)(base + r - row_begin);
              const int tmax = min(16, B - q_base - q0);
#pragma unroll
              for (int t = 0; t < 16; ++t)
                if (t < tmax) drow[(size_t)t * nrows] = __uint_as_float(acc[t]);
            }
          } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) S.stg[r * kStg + half * 16 + t] = __uint_as_float(acc[t]);
            named_sync(1, 32 * kEpiWarps);
            epi_insert_round(S.stg, ew, lane, j, B - q_base, base, row_end, top);
            named_sync(1, 32 * kEpiWarps);
          }
        }
      }
    }
    if (!kDump) {
#pragma unroll
      for (int j = 0; j < kBQ / kStgQ; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = j * kStgQ + ew * 4 + i;
          if (q_base + q < B) partial[((size_t)unit * B + q_base + q) * kCandLocal + lane] = top[j * 4 + i];
        }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kMC > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant for one group of 129..256 queries (NS = 4).  Why: at
// N = 256 the single-CTA kernel re-streams the 32-KB query tile of every
// k-chunk from L2 into shared memory for ONE 16-KB key tile (the two
// 256-column accumulator buffers leave no room to reuse it), and the MMA reads
// both back: ~96 KB of shared-memory traffic per key tile, more than the
// 128 B/clk port sustains at the UMMA rate.  With cta_group::2 the pair runs
// one M = 256 UMMA per k-step: each CTA stages its own key block (A half) and
// HALF of the query tile (B half, 128 queries), so per CTA and key tile the
// traffic drops to 16 + 16 KB written and 16 + 16 KB read, and the L2 query
// stream halves.
//   pair rank 0 (leader): key TMA, query TMA, MMA issue, TMEM alloc, epilogue
//   pair rank 1:          key TMA, query TMA,            TMEM alloc, epilogue
// Every full barrier lives in the leader (both CTAs' TMA bytes complete on it);
// the leader's commits multicast into both CTAs' empty / acc_full barriers; the
// peer's epilogue arrives remotely on the leader's acc_empty.
// Accumulator rows: leader TMEM = its key block, peer TMEM = the next block.
// kG > 1 (257..1024 queries): a cluster of kG pairs, pair g holding query
// group g; the key tile of pair-half h is issued by CTA 2 (t mod kG) + h and
// multicast into the kG CTAs of half h (keys cross HBM once per pass), and a
// key slot is refilled only after all kG pair leaders released it.
constexpr int kPairQ = 256;                 // UMMA N (queries per pass)
constexpr int kPairHalfQ = kPairQ / 2;      // B rows staged per CTA
constexpr int kPairQTile = kPairHalfQ * 128;
constexpr int kPairKS = 8, kPairQS = 4;

// kConv: fp32 keys converted to bf16 on chip.  Per 64-column k-chunk the key
// producer TMA-loads two fp32 boxes (128 rows x 32 columns each, 32 KB) into
// a raw ring; eight converter warps round them to bf16 (RN-even, the same
// rounding as the bf16 filter copy) into the SWIZZLE_128B K-major tile that
// kind::f16 reads, so the pair runs bf16 MMAs (half the tensor work of TF32)
// while HBM still carries each fp32 key once.  Queries: the bf16 slab.  The
// filter bound is the bf16-copy one (both operands bf16-rounded).
constexpr int kConvRawS = 3, kConvKS = 3, kConvQS = 3;
constexpr int kConvWarps = 8;
constexpr int kConvThreads = kThreads + 32 * kConvWarps;

template <bool kConv>
struct __align__(1024) PairSmemT {
  static constexpr int KS = kConv ? kConvKS : kPairKS;
  static constexpr int QS = kConv ? kConvQS : kPairQS;
  static constexpr int RS = kConv ? kConvRawS : 0;
  uint8_t kbuf[KS][kKeyTile];
  uint8_t qbuf[QS][kPairQTile];
  uint8_t raw[RS > 0 ? RS : 1][kConv ? 2 * kKeyTile : 16];  // 1-KB aligned (after whole 16-KB tiles)
  float stg[kBM * kStg];
  uint64_t k_full[KS], k_empty[KS];
  uint64_t q_full[QS], q_empty[QS];
  uint64_t raw_full[RS > 0 ? RS : 1], raw_empty[RS > 0 ? RS : 1];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
};
using PairSmem = PairSmemT<false>;
static_assert(sizeof(PairSmemT<true>) + 1024 <= 227 * 1024, "conversion pair kernel exceeds shared memory");

// Arrive on the pair leader's barrier without a cluster-scope release (no
// MEMBAR.GPU): the converter's generic stores are ordered for the tensor
// cores by fence.proxy.async, and the arrive / wait pair at the default
// (CTA) scope then orders them for the MMA issue — the remote-arrive form of
// CUTLASS's ClusterBarrier.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x (low half) = lo
  return *reinterpret_cast<const uint32_t*>(&v);
}

template <bool kBf16, int kG, bool kConv = false>
__global__ void __launch_bounds__(kConv ? kConvThreads : kThreads, 1)
    sim_pair_kernel(const __grid_constant__ CUtensorMap keys_map, const __grid_constant__ CUtensorMap q_map,
                    int64_t row_begin, int64_t row_end, int dim, int B, int64_t blocks_per_pair,
                    int per_group, uint64_t* __restrict__ partial) {
  static_assert(!kConv || !kBf16, "on-chip conversion: fp32 keys");
  constexpr bool kF16 = kBf16 || kConv;  // kind::f16 MMAs
  constexpr int kBK = kF16 ? 64 : 32;
  constexpr int KS = PairSmemT<kConv>::KS, QS = PairSmemT<kConv>::QS;
  constexpr int kMyQ = kPairQ / kEpiWarps;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  PairSmemT<kConv>& S =
      *reinterpret_cast<PairSmemT<kConv>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cr = (int)cluster_ctarank();
  const int rank = cr & 1;           // 0 = pair leader
  const int grp = cr >> 1;           // query group of this pair
  const uint32_t leader = (uint32_t)(cr & ~1);
  // The pass's B queries are split evenly over the kG pairs (per_group, a
  // multiple of 16, <= 256): the pairs of a cluster run in lockstep on shared
  // key tiles, so the widest group sets the pace.  UMMA N of this pair = its
  // group's queries rounded up to 16; the leader stages queries [0, N/2) of
  // the group, the peer [N/2, N).
  const int q_base = grp * per_group;
  const int n_grp = B - q_base < per_group ? (B - q_base > 0 ? B - q_base : 0) : per_group;
  const int n_mma = (n_grp + 15) & ~15;
  const int n_half = n_mma / 2;
  const uint16_t pair_mask = (uint16_t)(3u << (2 * grp));
  const uint16_t all_mask = (uint16_t)((1u << (2 * kG)) - 1);
  uint16_t half_mask = 0;  // the kG CTAs holding the same key half
#pragma unroll
  for (int g = 0; g < kG; ++g) half_mask |= (uint16_t)(1u << (2 * g + rank));
  const int unit = (int)cluster_id_x(), n_units = (int)n_clusters_x();
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t blk0 = (int64_t)unit * blocks_per_pair;
  const int64_t blk1 = std::min<int64_t>(blk0 + blocks_per_pair, n_blocks);
  const int64_t steps = blk1 > blk0 ? (blk1 - blk0 + 1) / 2 : 0;  // key-block pairs
  const int64_t row_hi = std::min<int64_t>(row_end, row_begin + blk1 * kBM);
  const int nk = (dim + kBK - 1) / kBK;
  const int kc0 = (int)(((int64_t)unit * nk) / n_units);

  if (threadIdx.x == 0) {
    for (int i = 0; i < KS; ++i) {
      // kConv: both CTAs' converter warps arrive on the leader's k_full
      mbar_init(&S.k_full[i], kConv ? 2 * kConvWarps : 1);
      // kConv: the bf16 stage is this CTA's own (only its pair's MMAs read it)
      mbar_init(&S.k_empty[i], kConv ? 1 : kG);
    }
    for (int i = 0; i < QS; ++i) {
      mbar_init(&S.q_full[i], 1);
      mbar_init(&S.q_empty[i], 1);
    }
    if constexpr (kConv) {
      for (int i = 0; i < kConvRawS; ++i) {
        mbar_init(&S.raw_full[i], 1);
        // kG > 1: the raw slot is a multicast target of the kG CTAs of this
        // pair-half, so every one of their converters releases it here
        mbar_init(&S.raw_empty[i], kConvWarps * kG);
      }
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.acc_full[i], 1);
      mbar_init(&S.acc_empty[i], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's barriers exist before any peer TMA / remote arrive
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  dev::pdl_trigger();  // K2's first kernel may launch onto free SM resources and wait there

  if (warp == 0) {
    // ======================= key stream: this CTA's block of each pair step
    if (lane == 0 && steps > 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&keys_map) : "memory");
      const uint64_t pol = policy_evict_first();
      int ks = 0;
      uint32_t kph = 0;
      uint32_t tile = 0;
      for (int64_t st = 0; st < steps; ++st) {
        const int row = (int)(row_begin + (blk0 + 2 * st + rank) * kBM);
        for (int kc = 0; kc < nk; ++kc, ++tile) {
          const int c = kc + kc0 < nk ? kc + kc0 : kc + kc0 - nk;
          if constexpr (kConv) {
            // raw fp32 halves of the chunk into this CTA's own ring
            mbar_wait(&S.raw_empty[ks], kph ^ 1);
            mbar_expect_tx(&S.raw_full[ks], 2 * kKeyTile);
            if constexpr (kG > 1) {  // tile t: issued by pair t mod kG into the kG CTAs of this half
              if ((int)(tile % kG) == grp) {
                tma_load_2d_mc(&S.raw[ks][0], &keys_map, &S.raw_full[ks], c * kBK, row, half_mask, pol);
                tma_load_2d_mc(&S.raw[ks][kKeyTile], &keys_map, &S.raw_full[ks], c * kBK + 32, row, half_mask, pol);
              }
            } else {
              tma_load_2d(&S.raw[ks][0], &keys_map, &S.raw_full[ks], c * kBK, row, pol);
              tma_load_2d(&S.raw[ks][kKeyTile], &keys_map, &S.raw_full[ks], c * kBK + 32, row, pol);
            }
            if (++ks == kConvRawS) {
              ks = 0;
              kph ^= 1;
            }
            continue;
          }
          mbar_wait(&S.k_empty[ks], kph ^ 1);
          if (rank == 0) mbar_expect_tx(&S.k_full[ks], 2 * kKeyTile);
          const uint32_t bar = mapa_shared(smem_u32(&S.k_full[ks]), leader);
          if constexpr (kG > 1) {
            if ((int)(tile % kG) == grp)
              tma_load_2d_pair_mc(&S.kbuf[ks][0], &keys_map, bar, c * kBK, row, half_mask, pol);
          } else {
            tma_load_2d_pair(&S.kbuf[ks][0], &keys_map, bar, c * kBK, row, pol);
          }
          if (++ks == KS) {
            ks = 0;
            kph ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    // ======================= query half tiles (L2-resident)
    if (lane == 0 && steps > 0) {
      dev::pdl_wait();  // the padded query slab
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&q_map) : "memory");
      const uint64_t pol = policy_evict_last();
      int qs = 0;
      uint32_t qph = 0;
      for (int64_t st = 0; st < steps; ++st)
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.q_empty[qs], qph ^ 1);
          if (rank == 0) mbar_expect_tx(&S.q_full[qs], 2 * kPairQTile);
          const int c = kc + kc0 < nk ? kc + kc0 : kc + kc0 - nk;
          tma_load_2d_pair(&S.qbuf[qs][0], &q_map, mapa_shared(smem_u32(&S.q_full[qs]), leader), c * kBK,
                           q_base + rank * n_half, pol);
          if (++qs == QS) {
            qs = 0;
            qph ^= 1;
          }
        }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader only)
    if (rank == 0) {
      const uint32_t idesc = kF16 ? bf16_idesc(2 * kBM, n_mma) : tf32_idesc(2 * kBM, n_mma);
      const uint64_t adesc0 = sw128_desc(&S.kbuf[0][0]);
      const uint64_t bdesc0 = sw128_desc(&S.qbuf[0][0]);
      int ks = 0, qs = 0;
      uint32_t kph = 0, qph = 0;
      for (int64_t gi = 0; gi < steps; ++gi) {
        const int buf = (int)(gi & 1);
        if (gi >= 2) {  // both CTAs' epilogues drained this buffer
          mbar_wait(&S.acc_empty[buf], (uint32_t)((gi / 2) - 1) & 1);
          tc_fence_after();
        }
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.q_full[qs], qph);
          mbar_wait(&S.k_full[ks], kph);
          tc_fence_after();
          const uint64_t adesc = adesc0 + (uint64_t)(ks * (kKeyTile >> 4));
          const uint64_t bdesc = bdesc0 + (uint64_t)(qs * (kPairQTile >> 4));
          const uint32_t d = tmem + buf * kPairQ;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (kF16)
              mma2_ss_f16(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
            else
              mma2_ss(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kc > 0 || kk > 0) ? 1u : 0u);
          }
          // every CTA's slot ks: kG releases complete it (kConv: the pair's own bf16 stage)
          tc_commit2_mc(&S.k_empty[ks], kConv ? pair_mask : all_mask);
          tc_commit2_mc(&S.q_empty[qs], pair_mask);
          if (++ks == KS) {
            ks = 0;
            kph ^= 1;
          }
          if (++qs == QS) {
            qs = 0;
            qph ^= 1;
          }
        }
        tc_commit2_mc(&S.acc_full[buf], pair_mask);
      }
    }
  } else if (kConv && warp >= 4 + kEpiWarps) {
    // ======================= converters: raw fp32 halves -> bf16 K-major SW128 tile
    if constexpr (kConv) {
      int rs = 0, ks = 0;
      uint32_t rph = 0, kph = 0;
      for (int64_t st = 0; st < steps; ++st)
        for (int kc = 0; kc < nk; ++kc) {
          mbar_wait(&S.raw_full[rs], rph);
          mbar_wait(&S.k_empty[ks], kph ^ 1);  // the MMAs have read this bf16 stage
          const uint8_t* raw = &S.raw[rs][0];
          uint8_t* dst = &S.kbuf[ks][0];
          // lane = (row parity rsel, fp32 box h, fp32 16-B chunk x): one 16-B
          // load of 4 keys, 8 B of bf16 out — the half (x & 1) of bf16 chunk
          // j = 4h + x / 2.  SWIZZLE_128B puts 16-B chunk c of row r at
          // c ^ (r & 7) in both tiles, so every 8-lane load phase reads 8
          // distinct chunks of one row and every 16-lane store phase writes
          // one whole 128-B bf16 row: no bank conflicts either way.
          const int x = lane & 7, h = (lane >> 3) & 1, rsel = lane >> 4;
          const int cw = warp - 4 - kEpiWarps;
#pragma unroll 8
          for (int i = 0; i < kBM / (2 * kConvWarps); ++i) {
            const int r = (i * kConvWarps + cw) * 2 + rsel, sw = r & 7;
            const float4 a = *reinterpret_cast<const float4*>(raw + h * kKeyTile + r * 128 + ((x ^ sw) << 4));
            const int j = 4 * h + (x >> 1);
            *reinterpret_cast<uint2*>(dst + r * 128 + ((j ^ sw) << 4) + (x & 1) * 8) =
                make_uint2(bf16x2_rn(a.x, a.y), bf16x2_rn(a.z, a.w));
          }
          // the tile's generic stores -> visible to the tensor cores (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (kG > 1) {
#pragma unroll
              for (int g = 0; g < kG; ++g)
                mbar_arrive_remote(mapa_shared(smem_u32(&S.raw_empty[rs]), (uint32_t)(2 * g + rank)));
            } else {
              mbar_arrive(&S.raw_empty[rs]);
            }
            mbar_arrive_remote(mapa_shared(smem_u32(&S.k_full[ks]), leader));
          }
          if (++rs == kConvRawS) {
            rs = 0;
            rph ^= 1;
          }
          if (++ks == KS) {
            ks = 0;
            kph ^= 1;
          }
        }
    }
  } else if (warp >= 4) {
    // ======================= epilogue (8 warps per CTA, its own key block)
    const int ew = warp - 4;
    const int quad = warp & 3;
    const int half = ew >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const uint32_t leader_empty0 = mapa_shared(smem_u32(&S.acc_empty[0]), leader);
    const uint32_t leader_empty1 = mapa_shared(smem_u32(&S.acc_empty[1]), leader);
    uint64_t top[kMyQ];
#pragma unroll
    for (int i = 0; i < kMyQ; ++i) top[i] = kEmpty;
    for (int64_t gi = 0; gi < steps; ++gi) {
      const int buf = (int)(gi & 1);
      mbar_wait(&S.acc_full[buf], (uint32_t)(gi / 2) & 1);
      tc_fence_after();
      const int64_t base = row_begin + (blk0 + 2 * gi + rank) * kBM;
      const int nj = (n_mma + kStgQ - 1) / kStgQ;  // staging rounds holding this pair's columns
#pragma unroll
      for (int j = 0; j < kPairQ / kStgQ; ++j) {
        if (j >= nj) break;
        uint32_t acc[16];
        TMEM_LD16(tmem + lane_addr + buf * kPairQ + j * kStgQ + half * 16, acc);
        tmem_ld_wait();
        if (j == nj - 1) {  // buffer drained
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(buf ? leader_empty1 : leader_empty0);
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) S.stg[r * kStg + half * 16 + t] = __uint_as_float(acc[t]);
        named_sync(1, 32 * kEpiWarps);
        epi_insert_round(S.stg, ew, lane, j, n_grp, base, row_hi, top);
        named_sync(1, 32 * kEpiWarps);
      }
    }
    const int list = unit * 2 + rank;  // one list per key half of the cluster's range
#pragma unroll
    for (int j = 0; j < kPairQ / kStgQ; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ql = j * kStgQ + ew * 4 + i;
        if (ql < n_grp) partial[((size_t)list * B + q_base + ql) * kCandLocal + lane] = top[j * 4 + i];
      }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer's MMAs / commits may still touch it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

// Zero-padded copy of the query slab to `rows` rows (the TMA box); bf16 mode
// rounds to bf16 (RN-even, hsd_bf16_bits) on the way.
// One CTA per padded row; dim % 4 == 0 (the collection's contract), rows are
// 16-B aligned.  Each thread moves kPadVec float4 with all loads issued before
// any store: a scalar load->store loop serialises one L2/DRAM round trip per
// iteration (measured 11 us for a 64 x 4096 slab, ~1 us vectorised).
constexpr int kPadThreads = 256, kPadVec = 4;
__global__ void __launch_bounds__(kPadThreads) pad_queries_f32_kernel(const float* __restrict__ q, int B, int dim,
                                                                      float* __restrict__ out) {
  dev::pdl_trigger();  // K1 may launch and start its key stream now
  const int row = blockIdx.x, n4 = dim / 4;
  const float4* src = reinterpret_cast<const float4*>(q + (size_t)row * dim);
  float4* dst = reinterpret_cast<float4*>(out + (size_t)row * dim);
  for (int c0 = threadIdx.x; c0 < n4; c0 += kPadThreads * kPadVec) {
    float4 v[kPadVec];
#pragma unroll
    for (int u = 0; u < kPadVec; ++u) {
      const int c = c0 + u * kPadThreads;
      v[u] = (row < B && c < n4) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kPadVec; ++u)
      if (c0 + u * kPadThreads < n4) dst[c0 + u * kPadThreads] = v[u];
  }
}
__global__ void __launch_bounds__(kPadThreads) pad_queries_bf16_kernel(const float* __restrict__ q, int B, int dim,
                                                                       uint16_t* __restrict__ out) {
  dev::pdl_trigger();  // K1 may launch and start its key stream now
  const int row = blockIdx.x, n4 = dim / 4;
  const float4* src = reinterpret_cast<const float4*>(q + (size_t)row * dim);
  uint2* dst = reinterpret_cast<uint2*>(out + (size_t)row * dim);
  for (int c0 = threadIdx.x; c0 < n4; c0 += kPadThreads * kPadVec) {
    float4 v[kPadVec];
#pragma unroll
    for (int u = 0; u < kPadVec; ++u) {
      const int c = c0 + u * kPadThreads;
      v[u] = (row < B && c < n4) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kPadVec; ++u)
      if (c0 + u * kPadThreads < n4)
        dst[c0 + u * kPadThreads] =
            make_uint2((uint32_t)hsd_bf16_bits(v[u].x) | ((uint32_t)hsd_bf16_bits(v[u].y) << 16),
                       (uint32_t)hsd_bf16_bits(v[u].z) | ((uint32_t)hsd_bf16_bits(v[u].w) << 16));
  }
}

template <bool kBf16, int NS, int GB, bool kDump, int kMC = 1>
cudaError_t launch_ns(const CUtensorMap& km, const CUtensorMap& qm, int64_t rb, int64_t re, int dim, int B,
                      int lists, int64_t per, uint64_t* partial, float* dump, cudaStream_t s) {
  const size_t smem = sizeof(WideSmem<NS, GB>) + 1024;
  auto kern = sim_wide_kernel<kBf16, NS, GB, kDump, kMC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // programmatic dependent of the query-slab kernel: the CTAs set up and start
  // the key stream while the slab is written (only the query producer waits)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(lists * kMC));  // kMC > 1: `lists` clusters of kMC CTAs
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kMC;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kMC > 1 ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, km, qm, rb, re, dim, B, per, partial, dump);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <bool kBf16, int kG, bool kConv = false>
cudaError_t launch_pair(const CUtensorMap& km, const CUtensorMap& qm, int64_t rb, int64_t re, int dim, int B,
                        int lists, int64_t per_pair, uint64_t* partial, cudaStream_t s) {
  const int per_group = (((B + kG - 1) / kG) + 15) & ~15;  // <= 256: kG = ceil(B / 256)
  const size_t smem = sizeof(PairSmemT<kConv>) + 1024;
  auto kern = sim_pair_kernel<kBf16, kG, kConv>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(lists * kG));  // lists = 2 x clusters; a cluster is kG pairs
  cfg.blockDim = dim3(kConv ? kConvThreads : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * kG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // after the query-slab kernel
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, kern, km, qm, rb, re, dim, B, per_pair, per_group, partial);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// CTA-pair kernels above 128 queries; HSD_WIDE_PAIR=0 or the tc_single path
// override (hsd_set_sim_path) select the single-CTA kernels (ablation).
int g_force_single = 0;
bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HSD_WIDE_PAIR");
    v = (e && !strcmp(e, "0")) ? 0 : 1;
  }
  return v == 1 && !g_force_single;
}

// Accumulator layout per NS: "db" = double-buffered (256 columns per buffer;
// the epilogue of one group overlaps the MMAs of the next), "max" = one
// 512-column buffer holding twice the key blocks (each query tile feeds twice
// as many key tiles; the MMAs wait for the epilogue once per group).
// HSD_WIDE_ACC=db|max overrides the default for ablations.
int wide_acc_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HSD_WIDE_ACC");
    v = (e && !strcmp(e, "max")) ? 1 : 0;  // default: double-buffered (measured faster at NS = 2 and 4)
  }
  return v;
}

template <bool kBf16, bool kDump>
cudaError_t launch_dispatch(int NS, const CUtensorMap& km, const CUtensorMap& qm, int64_t rb, int64_t re, int dim,
                            int B, int lists, int64_t per, uint64_t* partial, float* dump, cudaStream_t s) {
  const int mode = wide_acc_mode();
  if (NS == 1) return launch_ns<kBf16, 1, 4, kDump>(km, qm, rb, re, dim, B, lists, per, partial, dump, s);
  if constexpr (!kDump) {  // the single-buffer ablation is not instantiated for the debug dump
    if (mode == 1) {
      if (NS == 2) return launch_ns<kBf16, 2, 4, false>(km, qm, rb, re, dim, B, lists, per, partial, dump, s);
      return launch_ns<kBf16, 4, 2, false>(km, qm, rb, re, dim, B, lists, per, partial, dump, s);
    }
  }
  if (NS == 2) return launch_ns<kBf16, 2, 2, kDump>(km, qm, rb, re, dim, B, lists, per, partial, dump, s);
  return launch_ns<kBf16, 4, 1, kDump>(km, qm, rb, re, dim, B, lists, per, partial, dump, s);
}

}  // namespace

int sim_wide_max_batch() { return 1024; }
void sim_wide_set_single(bool single) { g_force_single = single ? 1 : 0; }

// Query groups (cluster size) of one pass: B <= 256 -> 1 CTA per key range;
// more -> ceil(B / 256) CTAs per cluster sharing each key tile by multicast.
static int wide_groups(int B) { return B <= 256 ? 1 : (B + 255) / 256; }

// Clusters of G CTAs that fit on the device at once (GPC packing leaves some
// SMs unused for G = 3, 4); a persistent grid larger than this would run a
// second wave.  Cached per G (same kernel resources for both dtypes).
static int max_active_clusters(int G, int num_sms) {
  static int cache[5] = {0, 0, 0, 0, 0};
  if (G <= 1) return num_sms;
  if (cache[G]) return cache[G];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(G * (num_sms / G)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sizeof(WideSmem<4, 1>) + 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaSuccess;
  switch (G) {
    case 2:
      e = cudaFuncSetAttribute(sim_wide_kernel<false, 4, 1, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cfg.dynamicSmemBytes);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, sim_wide_kernel<false, 4, 1, false, 2>, &cfg);
      break;
    case 3:
      e = cudaFuncSetAttribute(sim_wide_kernel<false, 4, 1, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cfg.dynamicSmemBytes);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, sim_wide_kernel<false, 4, 1, false, 3>, &cfg);
      break;
    default:
      e = cudaFuncSetAttribute(sim_wide_kernel<false, 4, 1, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cfg.dynamicSmemBytes);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, sim_wide_kernel<false, 4, 1, false, 4>, &cfg);
      break;
  }
  if (e != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = num_sms / G;
  }
  cache[G] = std::min(n, num_sms / G);
  return cache[G];
}

static bool use_pair(int B) { return B > 128 && pair_enabled(); }

// fp32 keys in the pair kernel (one pair per cluster, 129..256 queries):
// converted to bf16 on chip (kind::f16) unless HSD_PAIR_CONVERT=0 (TF32).
static bool pair_convert_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HSD_PAIR_CONVERT");
    v = (e && !strcmp(e, "0")) ? 0 : 1;
  }
  return v == 1;
}

// Clusters of G CTA pairs (2G CTAs) resident at once, cached per G.
static int max_active_pair_clusters(int G, int num_sms) {
  static int cache[5] = {0, 0, 0, 0, 0};
  if (!cache[G]) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(2 * G * (num_sms / (2 * G))));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sizeof(PairSmem) + 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)(2 * G);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaSuccess;
    auto q = [&](auto kern) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    };
    switch (G) {
      case 1: q(sim_pair_kernel<false, 1>); break;
      case 2: q(sim_pair_kernel<false, 2>); break;
      case 3: q(sim_pair_kernel<false, 3>); break;
      default: q(sim_pair_kernel<false, 4>); break;
    }
    if (e != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = num_sms / (2 * G);
    }
    cache[G] = std::max(1, n);
  }
  return std::max(1, std::min(cache[G], num_sms / (2 * G)));
}

int sim_wide_lists(int B, int64_t rows, int num_sms) {
  const int g = wide_groups(B);
  const int64_t blocks = (rows + kBM - 1) / kBM;
  if (use_pair(B)) {  // clusters of g CTA pairs: lists = 2 x clusters, each walks >= 2 key blocks
    const int64_t cl = std::max<int64_t>(1, std::min<int64_t>((blocks + 1) / 2, max_active_pair_clusters(g, num_sms)));
    return (int)(2 * cl);
  }
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, max_active_clusters(g, num_sms)));
}

bool sim_wide_converts(int key_dtype, int B, int dim) {
  // dim % 8: the bf16 query slab's rows must be 16-B multiples (TMA stride)
  return key_dtype == HSD_DTYPE_F32 && dim % 8 == 0 && use_pair(B) && pair_convert_enabled();
}

double sim_wide_gamma(int dim, int key_dtype) {
  // Relative forward error of the filter score S~ against the real dot S of
  // the stored keys and the fp32 query: |S - S~| <= gamma * sum|k_i q_i|.
  // (k_select.cu adds the absolute underflow / flush-to-zero slack.)
  // Products: with operands rounded to k' = k(1 + a), q' = q(1 + b),
  // |k'q' - kq| <= (|a| + |b| + |ab|) |kq|; bf16 x bf16 and tf32 x tf32
  // products are exact in fp32.  Accumulation: the fp32 tensor-core
  // accumulator (not round-to-nearest) over dim products, <= (dim + 16) 2^-23
  // relative to sum|k'q'| <= (1 + u)^2 sum|kq|; 2^-22 per product covers
  // truncation of every addend to the running exponent.
  const double acc = (dim + 16.0) * 0x1p-22 * 1.02;
  if (key_dtype & 0x100) {
    // bf16 filter copy of fp32 keys: both operands rounded to bf16, RN-even,
    // unit roundoff u = 2^-8 (8-bit significand): a = b = 2^-8.
    return (0x1p-7 + 0x1p-16) * 1.0001 + acc;
  }
  if (key_dtype == HSD_DTYPE_BF16) {
    // bf16 keys are exact; queries rounded to bf16 (RN-even): b = 2^-8.
    return 0x1p-8 * 1.0001 + acc;
  }
  // TF32 operands (fp32 tiles read as tf32: the low 13 mantissa bits are
  // dropped, |x - tf32(x)| < 2^-10 |x|): a = b = 2^-10.
  return (0x1p-9 + 0x1p-20) * 1.0001 + acc;
}

size_t sim_wide_scratch_bytes(int dim) { return (size_t)1024 * dim * sizeof(float); }

cudaError_t launch_sim_wide(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin, int64_t row_end,
                            int dim, const float* queries, int B, int lists, void* scratch, uint64_t* partial,
                            float* dump, cudaStream_t s, ListGeom* geom) {
  if (B < 1 || B > kMaxBatchPass) return cudaErrorInvalidValue;
  const int groups = wide_groups(B);
  const int NS = groups > 1 ? 4 : (B <= 64 ? 1 : (B <= 128 ? 2 : 4));
  const int box = 64 * NS;          // query rows per CTA
  const int rows = box * groups;    // padded query slab
  const bool bf16 = key_dtype == HSD_DTYPE_BF16;
  if (bf16 && dim % 8) return cudaErrorInvalidValue;  // TMA row stride must be a multiple of 16 B
  const bool pair = use_pair(B) && !dump && lists % 2 == 0;
  const bool conv = pair && sim_wide_converts(key_dtype, B, dim);
  const uint32_t qbox = pair ? (uint32_t)kPairHalfQ : (uint32_t)box;  // a pair CTA stages half the queries
  CUtensorMap km, qm;
  if (conv) {  // fp32 key tiles (converted on chip), bf16 query slab
    pad_queries_bf16_kernel<<<rows, kPadThreads, 0, s>>>(queries, B, dim, (uint16_t*)scratch);
    if (!tc_make_map(&km, (const float*)keys, (uint64_t)n_keys_total, (uint64_t)dim, kBM) ||
        !tc_make_map_bf16(&qm, scratch, (uint64_t)rows, (uint64_t)dim, qbox))
      return cudaErrorInvalidValue;
  } else if (bf16) {
    pad_queries_bf16_kernel<<<rows, kPadThreads, 0, s>>>(queries, B, dim, (uint16_t*)scratch);
    if (!tc_make_map_bf16(&km, keys, (uint64_t)n_keys_total, (uint64_t)dim, kBM) ||
        !tc_make_map_bf16(&qm, scratch, (uint64_t)rows, (uint64_t)dim, qbox))
      return cudaErrorInvalidValue;
  } else {
    pad_queries_f32_kernel<<<rows, kPadThreads, 0, s>>>(queries, B, dim, (float*)scratch);
    if (!tc_make_map(&km, (const float*)keys, (uint64_t)n_keys_total, (uint64_t)dim, kBM) ||
        !tc_make_map(&qm, (const float*)scratch, (uint64_t)rows, (uint64_t)dim, qbox))
      return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n_blocks = (row_end - row_begin + kBM - 1) / kBM;
  const int64_t per = (n_blocks + lists - 1) / lists;
  if (geom) *geom = ListGeom{row_begin, row_end, per, 1};
  if (pair) {
    const int64_t pairs = lists / 2;
    const int64_t per_pair = ((n_blocks + pairs - 1) / pairs + 1) & ~(int64_t)1;  // even: whole block pairs
    if (geom) *geom = ListGeom{row_begin, row_end, per_pair, 2};
    if (conv) {
      switch (groups) {
        case 1: return launch_pair<false, 1, true>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s);
        case 2: return launch_pair<false, 2, true>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s);
        case 3: return launch_pair<false, 3, true>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s);
        case 4: return launch_pair<false, 4, true>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s);
        default: return cudaErrorInvalidValue;
      }
    }
    switch (groups) {
#define HSD_PAIR(G)                                                                                        \
  case G:                                                                                                  \
    return bf16 ? launch_pair<true, G>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s)    \
                : launch_pair<false, G>(km, qm, row_begin, row_end, dim, B, lists, per_pair, partial, s);
      HSD_PAIR(1)
      HSD_PAIR(2)
      HSD_PAIR(3)
      HSD_PAIR(4)
#undef HSD_PAIR
      default: return cudaErrorInvalidValue;
    }
  }
  if (groups > 1) {
    if (dump) return cudaErrorInvalidValue;  // the debug dump covers single-group passes
    switch (groups) {
#define HSD_WIDE_MC(G)                                                                                            \
  case G:                                                                                                         \
    return bf16 ? launch_ns<true, 4, 1, false, G>(km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s) \
                : launch_ns<false, 4, 1, false, G>(km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s);
      HSD_WIDE_MC(2)
      HSD_WIDE_MC(3)
      HSD_WIDE_MC(4)
#undef HSD_WIDE_MC
      default: return cudaErrorInvalidValue;
    }
  }
  if (bf16)
    return dump ? launch_dispatch<true, true>(NS, km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s)
                : launch_dispatch<true, false>(NS, km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s);
  return dump ? launch_dispatch<false, true>(NS, km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s)
              : launch_dispatch<false, false>(NS, km, qm, row_begin, row_end, dim, B, lists, per, partial, dump, s);
}

}  // namespace hsd
