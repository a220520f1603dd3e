// k_exact.cu — K1x exact scan: every row scored with the reference's own
// arithmetic, for searches whose (rows x queries) is small.
//
// Collection::search_topk_exact (store.cpp:59-73) scores every record with
// cosine_similarity (store.cpp:29-34): s += a[i] * b[i] sequentially in fp64,
// then orders by (score desc, id asc) and keeps k.  The default path (K1
// tensor-core filter + K2 exact rescoring of the candidates) pays K2's
// dim-step dependent fp64 chain AFTER the filter's scan.  For a small DB at
// batch 1..4 (config 1: 10k rows x 4096, one query) streaming the fp32 keys
// once costs about as much as that one chain, so this kernel runs the chain of
// EVERY row while the keys stream in, and the filter, the candidate pooling
// and the rescoring all disappear:
//
//   * one thread per row (lanes 0..lpw-1 of 4 compute warps, a tile of
//     R = 4 lpw rows per CTA, persistent over tiles), each running NQ <= 4
//     independent chains (one per query: NQ-way ILP on the DFMA latency),
//     16 B of its row per shared load, widened just before its DFMAs;
//   * warp 4 streams the tile's 128-B row segments (32 fp32 or 64 bf16
//     columns) by TMA into an S-stage SWIZZLE_128B ring; a thread's 16-B
//     shared loads of its own row hit 8 distinct bank groups per 8 rows
//     (conflict-free);
//   * the queries are widened to fp64 once per CTA into shared memory
//     (zero-padded to the chunk width: fma(0, 0, s) == s, and s is never
//     -0.0 since the chain starts at +0.0);
//   * acc = fma(q_i, k_i, acc), i ascending: the fp32 (or bf16) x fp32
//     product is exact in fp64, so this is bit-identical to s += a[i]*b[i];
//   * each warp keeps a sorted (order key, id) top-k per query in registers
//     (bitonic sort + merge; a batch that cannot enter is rejected with one
//     ballot), the CTA's 4 warp lists merge in shared memory, and the
//     CTAs' lists merge in two ticketed levels (groups of 12 CTAs, then the
//     groups) into the final top-k.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace hsd {
namespace {

using dev::kEmpty;
using namespace sm100;

// compute warps: one per scheduler.  (Two per scheduler with half the rows
// each measured 16% slower at config 1: the per-step instruction stream is
// issued per warp, so it doubles, while a chain's latency stays.)
__host__ __device__ constexpr int compute_warps(int) { return 4; }
constexpr uint32_t kNoId = 0xFFFFFFFFu;
constexpr int kSmemBudget = 225 * 1024;
constexpr int kGroup = 12;      // CTAs per first-level merge group (~sqrt of the grid)
constexpr int kSegPerStage = 4;

// (order key, id): ascending = the reference's (score desc, id asc).
__device__ __forceinline__ bool lt(uint64_t ak, uint32_t ai, uint64_t bk, uint32_t bi) {
  return ak < bk || (ak == bk && ai < bi);
}

// Bitonic sort of 32 (key, id) pairs, one per lane, ascending.
__device__ __forceinline__ void warp_sort_ki(uint64_t& k, uint32_t& i) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t ok = dev::shfl_xor_u64(k, stride);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, stride);
      const bool asc = (lane & size) == 0 || size == 32;
      const bool lower = (lane & stride) == 0;
      const bool other_less = lt(ok, oi, k, i);
      // ascending region: the lower lane keeps the smaller element
      if ((lower == asc) ? other_less : !other_less) {
        k = ok;
        i = oi;
      }
    }
  }
}

// Merge a sorted-ascending batch (b) into the sorted list (l): keeps the 32
// smallest of the union, sorted.
__device__ __forceinline__ void warp_merge_ki(uint64_t& lk, uint32_t& li, uint64_t bk, uint32_t bi) {
  const int lane = threadIdx.x & 31;
  const uint64_t rk = dev::shfl_u64(bk, 31 - lane);
  const uint32_t ri = __shfl_sync(0xffffffffu, bi, 31 - lane);
  if (lt(rk, ri, lk, li)) {
    lk = rk;
    li = ri;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    const uint64_t ok = dev::shfl_xor_u64(lk, stride);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, li, stride);
    const bool lower = (lane & stride) == 0;
    const bool other_less = lt(ok, oi, lk, li);
    if (lower ? other_less : !other_less) {
      lk = ok;
      li = oi;
    }
  }
}

// Offer one unsorted batch (one entry per lane) to the warp's top-k list.
__device__ __forceinline__ void warp_offer(uint64_t& lk, uint32_t& li, uint64_t ck, uint32_t ci, int k) {
  const uint64_t kk = dev::shfl_u64(lk, k - 1);
  const uint32_t ki = __shfl_sync(0xffffffffu, li, k - 1);
  if (!__any_sync(0xffffffffu, lt(ck, ci, kk, ki))) return;
  warp_sort_ki(ck, ci);
  warp_merge_ki(lk, li, ck, ci);
}

// Offer a sorted list (entries 0..k-1 valid, one per lane) to the warp's list.
__device__ __forceinline__ void warp_offer_sorted(uint64_t& lk, uint32_t& li, uint64_t ck, uint32_t ci, int k) {
  const uint64_t kk = dev::shfl_u64(lk, k - 1);
  const uint32_t ki = __shfl_sync(0xffffffffu, li, k - 1);
  const uint64_t hk = dev::shfl_u64(ck, 0);
  const uint32_t hi = __shfl_sync(0xffffffffu, ci, 0);
  if (!lt(hk, hi, kk, ki)) return;
  warp_merge_ki(lk, li, ck, ci);
}

__device__ __forceinline__ double key_score(uint64_t key) {  // inverse of score_desc_key (scores are never -0.0)
  uint64_t u = ~key;
  u = (u >> 63) ? (u & 0x7FFFFFFFFFFFFFFFull) : ~u;
  return __longlong_as_double((long long)u);
}

// The chain is latency-bound: one dependent DFMA per step (~8.6 cycles on
// sm_100) with one warp per scheduler.  The consumer loop is the plain one:
// per 16-B chunk of a thread's row segment one shared load, the widening and
// the chunk's DFMAs per query, with the broadcast query operands loaded
// beside them; the compiler schedules the loads a group ahead.  (A ping-pong
// variant that widened the whole next 32-column sub into fp64 registers while
// the current sub's chain ran used 190 registers and measured ~1 us slower per
// scan at config 1, r02q: 55.3 vs 54.4 us.)
constexpr int kSub = 32;  // columns per sub-segment (one 128-B fp32 segment, half a bf16 one)
constexpr int kVecPerSub(int key_bytes) { return kSub * key_bytes / 16; }  // 16-B loads per sub: 8 fp32, 4 bf16

struct ScanArgs {
  int dim, nchunk;               // 128-B row segments per row
  int64_t row_begin, row_end;    // rows scored
  int R, lpw, S;                 // tile rows (4 lpw), rows per warp, ring stages
  int seg;                       // 128-B row segments per stage (one barrier handshake each)
  int64_t ntiles;
  int k;
  const float* queries;          // [NQ][dim]
  uint64_t* lkey;                // [gridDim][NQ][32]
  uint32_t* lid;
  unsigned* ticket;              // zero between launches (the last CTA resets it)
  unsigned* gticket;             // [groups] per-group tickets (each group's last CTA resets its own)
  uint64_t* gkey;                // [groups][NQ][32] group lists
  uint32_t* gid;
  double* scores;                // [NQ][k]
  int32_t* ids;
  uint64_t* allkey;              // != nullptr: every row's order key [NQ][rows], no top-k (large k)
};

template <typename KT, int NQ, int kCW = compute_warps(NQ)>
__global__ void __launch_bounds__((kCW + 1) * 32, 1) exact_scan_kernel(const __grid_constant__ CUtensorMap km, ScanArgs a) {
  constexpr int CPC = 128 / (int)sizeof(KT);  // columns per 128-B segment
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B stages must sit on 1-KB boundaries (the plan reserves the slack)
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg_bytes = a.R * 128;
  const int stage_bytes = seg_bytes * a.seg;
  const int qlen = a.nchunk * CPC;
  uint8_t* ring = smem;
  double* q64 = reinterpret_cast<double*>(smem + (size_t)a.S * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(q64 + (size_t)NQ * qlen);
  uint64_t* empty = full + a.S;
  uint64_t* ck = empty + a.S;                          // [kCW][NQ][32] CTA merge staging
  uint32_t* ci = reinterpret_cast<uint32_t*>(ck + kCW * NQ * 32);
  __shared__ int s_last;

  if (tid == 0) {
    for (int s = 0; s < a.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  dev::pdl_wait();  // the queries may come from the previous kernel
  dev::pdl_trigger();  // an early K4 (engine step) may start its logits / feature phases under the scan

  if (warp == kCW) {
    // ---- TMA producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int slot = 0, n = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const int y = (int)(a.row_begin + t * a.R);
        for (int j = 0; j < a.nchunk; j += a.seg) {
          const int nseg = min(a.seg, a.nchunk - j);
          if (n >= a.S) mbar_wait(&empty[slot], ph ^ 1);
          ++n;
          mbar_expect_tx(&full[slot], (uint32_t)(nseg * seg_bytes));
          for (int s2 = 0; s2 < nseg; ++s2)
            tma_load_2d(ring + (size_t)slot * stage_bytes + (size_t)s2 * seg_bytes, &km, &full[slot], (j + s2) * CPC,
                        y, pol);
          if (++slot == a.S) slot = 0, ph ^= 1;
        }
      }
    }
  } else {
    // ---- compute warps: queries -> fp64 (zero-padded), then the chains
    {
      // all of a thread's 16-B query loads in flight at once (one L2 round
      // trip, not one per element), then the widened stores
      constexpr int kLd = 8;
      const int d4 = a.dim / 4, n4 = NQ * d4;
      const float4* q4 = reinterpret_cast<const float4*>(a.queries);
      for (int b0 = tid; b0 < n4; b0 += kCW * 32 * kLd) {
        float4 v[kLd];
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
          const int x = b0 + u * kCW * 32;
          v[u] = x < n4 ? __ldg(q4 + x) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kLd; ++u) {
          const int x = b0 + u * kCW * 32;
          if (x < n4) {
            const int q = x / d4, c = (x - q * d4) * 4;
            double* o = q64 + (size_t)q * qlen + c;
            o[0] = (double)v[u].x;
            o[1] = (double)v[u].y;
            o[2] = (double)v[u].z;
            o[3] = (double)v[u].w;
          }
        }
      }
      for (int x = tid; x < NQ * (qlen - a.dim); x += kCW * 32) {  // zero tail of the last segment
        const int q = x / (qlen - a.dim);
        q64[(size_t)q * qlen + a.dim + (x - q * (qlen - a.dim))] = 0.0;
      }
    }
    named_sync(1, kCW * 32);
    uint64_t lk[NQ];
    uint32_t li[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      lk[q] = kEmpty;
      li[q] = kNoId;
    }
    const int rr = warp * a.lpw + lane;
    const int swz = rr & 7;
    // ring positions: the next segment to wait for, the next to release
    int wslot = 0, rslot = 0;
    uint32_t wph = 0;
    constexpr int SUBS = CPC / kSub;  // subs per 128-B segment
    const uint8_t* rowbase = ring + (size_t)(lane < a.lpw ? rr : 0) * 128;
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      const int64_t row = a.row_begin + t * a.R + rr;
      const bool active = lane < a.lpw && row < a.row_end;
      double acc[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
      // per 16-B chunk of the row segment: one shared load, widen, the
      // chunk's DFMAs per query (broadcast query operands); the compiler
      // schedules the loads a group ahead.  A stage holds up to 4 segments
      // (128 fp32 columns) behind one barrier wait and one release: 47 vs
      // 49 us at 2.5k rows, 51 vs 53 us at config 1 (same box, r02q).
      constexpr int E = 16 / (int)sizeof(KT);  // keys per 16-B chunk
      constexpr int kVec = kVecPerSub((int)sizeof(KT));
      for (int j = 0; j < a.nchunk; j += a.seg) {  // one ring stage: nseg row segments, one handshake
        const int nseg = min(a.seg, a.nchunk - j);
        mbar_wait(&full[wslot], wph);
        for (int sg = 0; sg < nseg; ++sg) {
          const uint8_t* rowp = rowbase + (size_t)wslot * stage_bytes + (size_t)sg * seg_bytes;
#pragma unroll
          for (int h = 0; h < SUBS; ++h) {
            const double* qc = q64 + (size_t)((j + sg) * SUBS + h) * kSub;
#pragma unroll
            for (int c = 0; c < kVec; ++c) {
              const uint4 x = *reinterpret_cast<const uint4*>(rowp + (((h * kVec + c) ^ swz) << 4));
              double kv[E];
              if constexpr (sizeof(KT) == 4) {
                kv[0] = (double)__uint_as_float(x.x);
                kv[1] = (double)__uint_as_float(x.y);
                kv[2] = (double)__uint_as_float(x.z);
                kv[3] = (double)__uint_as_float(x.w);
              } else {
                const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  kv[2 * i] = (double)__uint_as_float(w[i] << 16);
                  kv[2 * i + 1] = (double)__uint_as_float(w[i] & 0xFFFF0000u);
                }
              }
#pragma unroll
              for (int q = 0; q < NQ; ++q) {
#pragma unroll
                for (int e = 0; e < E; e += 2) {
                  const double2 qq = *reinterpret_cast<const double2*>(qc + (size_t)q * qlen + c * E + e);
                  acc[q] = __fma_rn(qq.x, kv[e], acc[q]);
                  acc[q] = __fma_rn(qq.y, kv[e + 1], acc[q]);
                }
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rslot]);
        if (++rslot == a.S) rslot = 0;
        if (++wslot == a.S) wslot = 0, wph ^= 1;
      }
      if (a.allkey) {  // large k: the keys go to the radix sort (coalesced: consecutive rows per lane)
        if (active) {
          const int64_t rows = a.row_end - a.row_begin;
#pragma unroll
          for (int q = 0; q < NQ; ++q) a.allkey[(size_t)q * rows + (row - a.row_begin)] = dev::score_desc_key(acc[q]);
        }
        continue;
      }
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        warp_offer(lk[q], li[q], active ? dev::score_desc_key(acc[q]) : kEmpty, active ? (uint32_t)row : kNoId, a.k);
    }
    if (a.allkey) return;  // uniform over the compute warps; the producer's loads were all consumed
    // the CTA's list: warps 1..3 stage theirs, warp 0 merges
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      ck[(warp * NQ + q) * 32 + lane] = lk[q];
      ci[(warp * NQ + q) * 32 + lane] = li[q];
    }
    named_sync(1, kCW * 32);
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        for (int w = 1; w < kCW; ++w)
          warp_offer_sorted(lk[q], li[q], ck[(w * NQ + q) * 32 + lane], ci[(w * NQ + q) * 32 + lane], a.k);
        a.lkey[((size_t)blockIdx.x * NQ + q) * 32 + lane] = lk[q];
        a.lid[((size_t)blockIdx.x * NQ + q) * 32 + lane] = li[q];
      }
    }
  }
  if (a.allkey) return;  // the producer warp (large k: no merge)
  // ---- two-level merge.  The last CTA of each group of kGroup CTAs merges
  // the group's lists into a group list; the last group then merges the
  // group lists.  (One last CTA merging all ~140 lists chained ~28 dependent
  // warp merges per warp: 51.2 -> 49.2 us at config 1, same box, r02q.)
  constexpr int kWarps = kCW + 1;
  const int G = gridDim.x;
  const int ngroups = (G + kGroup - 1) / kGroup;
  const int grp = blockIdx.x / kGroup;
  const int first = grp * kGroup, members = min(kGroup, G - first);
  uint64_t lk[NQ];
  uint32_t li[NQ];
  auto merge_lists = [&](const uint64_t* __restrict__ key, const uint32_t* __restrict__ id, int lfirst, int count) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      lk[q] = kEmpty;
      li[q] = kNoId;
    }
    const int per_list = NQ * a.k;
    const int chunk = (int)((size_t)a.S * stage_bytes / ((size_t)per_list * 12));
    uint64_t* sk = reinterpret_cast<uint64_t*>(ring);
    uint32_t* si = reinterpret_cast<uint32_t*>(ring + (size_t)chunk * per_list * 8);
    for (int c0 = 0; c0 < count; c0 += chunk) {
      const int n = min(chunk, count - c0);
#pragma unroll 8
      for (int x = tid; x < n * per_list; x += kWarps * 32) {
        const int g = x / per_list, r = x - g * per_list, q = r / a.k, j = r - q * a.k;
        const size_t src = ((size_t)(lfirst + c0 + g) * NQ + q) * 32 + j;
        sk[x] = __ldcg(&key[src]);
        si[x] = __ldcg(&id[src]);
      }
      __syncthreads();
      for (int g = warp; g < n; g += kWarps) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int x = (g * NQ + q) * a.k + lane;
          warp_offer_sorted(lk[q], li[q], lane < a.k ? sk[x] : kEmpty, lane < a.k ? si[x] : kNoId, a.k);
        }
      }
      __syncthreads();
    }
    __syncthreads();
    if (warp > 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        ck[((warp - 1) * NQ + q) * 32 + lane] = lk[q];
        ci[((warp - 1) * NQ + q) * 32 + lane] = li[q];
      }
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        for (int w = 0; w < kWarps - 1; ++w)
          warp_offer_sorted(lk[q], li[q], ck[(w * NQ + q) * 32 + lane], ci[(w * NQ + q) * 32 + lane], a.k);
    }
  };
  auto write_final = [&]() {
    if (warp == 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (lane < a.k) {
          const bool ok = lk[q] != kEmpty;
          a.scores[(size_t)q * a.k + lane] = ok ? key_score(lk[q]) : -INFINITY;
          a.ids[(size_t)q * a.k + lane] = ok ? (int32_t)li[q] : -1;
        }
    }
  };
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&a.gticket[grp], 1u) == (unsigned)members - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  merge_lists(a.lkey, a.lid, first, members);
  if (ngroups == 1) {
    write_final();
    if (tid == 0) a.gticket[grp] = 0u;
    return;
  }
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      a.gkey[((size_t)grp * NQ + q) * 32 + lane] = lk[q];
      a.gid[((size_t)grp * NQ + q) * 32 + lane] = li[q];
    }
    if (lane == 0) a.gticket[grp] = 0u;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.ticket, 1u) == (unsigned)ngroups - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  merge_lists(a.gkey, a.gid, 0, ngroups);
  write_final();
  if (tid == 0) *a.ticket = 0u;
}

struct ScanPlan {
  int lpw, R, S, grid, seg;
  int64_t ntiles;
  size_t smem;
};

template <typename KT>
ScanPlan scan_plan(int64_t rows, int dim, int NQ, int nsm) {
  constexpr int CPC = 128 / (int)sizeof(KT);
  const int kCW = compute_warps(NQ);
  ScanPlan p{};
  const int nchunk = (dim + CPC - 1) / CPC;
  int lpw = (int)std::min<int64_t>(32, (((rows + nsm - 1) / nsm) + kCW - 1) / kCW);
  while ((kCW * lpw) % 8) ++lpw;  // a stage is a whole number of 1-KB swizzle atoms
  p.lpw = lpw;
  p.R = kCW * lpw;
  p.ntiles = (rows + p.R - 1) / p.R;
  p.grid = (int)std::min<int64_t>(p.ntiles, nsm);
  const size_t fixed = (size_t)NQ * nchunk * CPC * sizeof(double) + 64 * 16 +
                       (size_t)kCW * NQ * 32 * (sizeof(uint64_t) + sizeof(uint32_t)) + 1024;
  // Stages of up to kSegPerStage row segments: the consumers' barrier wait and
  // release (~120 cycles per handshake, tools/chain_lab.cu mode 14) are paid
  // once per stage; the ring keeps >= 4 stages.
  int seg = kSegPerStage;
  size_t stage = 0;
  int S = 0;
  for (;; seg >>= 1) {
    seg = std::max(1, std::min(seg, nchunk));
    stage = (size_t)p.R * 128 * seg;
    S = (int)std::min<size_t>(16, (kSmemBudget - fixed) / stage);
    if (S >= 4 || seg == 1) break;
  }
  p.seg = seg;
  p.S = S;
  p.smem = (size_t)S * stage + fixed;
  return p;
}

template <typename KT, int NQ>
cudaError_t launch_scan_t(const CUtensorMap& km, const ScanPlan& p, const ScanArgs& a, cudaStream_t s) {
  auto kern = exact_scan_kernel<KT, NQ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3((compute_warps(NQ) + 1) * 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, km, a);
}

}  // namespace

bool exact_scan_supported(int B, int dim, int key_dtype, int k) {
  if (B < 1 || B > kScanMaxBatch || k < 1 || k > 32) return false;
  if (key_dtype == HSD_DTYPE_BF16 ? dim % 8 : dim % 4) return false;  // TMA row stride: 16-B multiple
  const size_t q = (size_t)B * (size_t)(dim + 63) * sizeof(double);
  return q <= 136 * 1024;  // leaves room for a >= 4-stage ring of the widest tile
}

size_t exact_scan_scratch_bytes(int B, int num_sms) {
  const int nq = std::max(1, B);
  const int groups = (num_sms + kGroup - 1) / kGroup;
  return (size_t)(num_sms + groups) * nq * 32 * (sizeof(uint64_t) + sizeof(uint32_t)) + 256;
}

double exact_scan_cost_us(int64_t rows, int dim, int key_dtype, int B) {
  // streaming bound (fp32 / bf16 keys at ~6 TB/s) vs the dim-step DFMA chain
  // (~4.6 ns per step) + launch / merge overhead; measured on B200
  const double bytes = (double)rows * dim * (key_dtype == HSD_DTYPE_BF16 ? 2 : 4);
  const double stream = bytes / 6.0e6;
  const double chain = dim * 4.6e-3 * (B > 2 ? 1.15 : 1.0);
  return std::max(stream, chain) + 6.0;
}

cudaError_t launch_exact_scan(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin,
                              int64_t row_end, int dim, const float* queries, int B, int k,
                              void* scratch, int num_sms, double* scores,
                              int32_t* ids, cudaStream_t s) {
  if (!exact_scan_supported(B, dim, key_dtype, k) || row_end <= row_begin) return cudaErrorInvalidValue;
  const bool bf16 = key_dtype == HSD_DTYPE_BF16;
  const int NQ = B;
  const int64_t rows = row_end - row_begin;
  const ScanPlan p = bf16 ? scan_plan<uint16_t>(rows, dim, NQ, num_sms) : scan_plan<float>(rows, dim, NQ, num_sms);
  if (p.S < 2) return cudaErrorInvalidValue;
  CUtensorMap km;
  const bool ok = bf16 ? tc_make_map_bf16(&km, keys, (uint64_t)n_keys_total, (uint64_t)dim, (uint32_t)p.R)
                       : tc_make_map(&km, (const float*)keys, (uint64_t)n_keys_total, (uint64_t)dim, (uint32_t)p.R);
  if (!ok) return cudaErrorInvalidValue;
  uint8_t* sc = static_cast<uint8_t*>(scratch);
  ScanArgs a{};
  a.dim = dim;
  a.nchunk = bf16 ? (dim + 63) / 64 : (dim + 31) / 32;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.R = p.R;
  a.lpw = p.lpw;
  a.S = p.S;
  a.seg = p.seg;
  a.ntiles = p.ntiles;
  a.k = k;
  a.queries = queries;
  // [ticket | group tickets (<= 48) : 256 B][lkey][lid][gkey][gid]
  const int groups = (num_sms + kGroup - 1) / kGroup;
  if (groups > 48) return cudaErrorInvalidValue;
  a.ticket = reinterpret_cast<unsigned*>(sc);
  a.gticket = reinterpret_cast<unsigned*>(sc + 64);
  a.lkey = reinterpret_cast<uint64_t*>(sc + 256);
  a.lid = reinterpret_cast<uint32_t*>(sc + 256 + (size_t)num_sms * NQ * 32 * sizeof(uint64_t));
  a.gkey = reinterpret_cast<uint64_t*>(sc + 256 + (size_t)num_sms * NQ * 32 * 12);
  a.gid = reinterpret_cast<uint32_t*>(sc + 256 + (size_t)num_sms * NQ * 32 * 12 +
                                      (size_t)groups * NQ * 32 * sizeof(uint64_t));
  a.scores = scores;
  a.ids = ids;
  switch (NQ) {
#define HSD_SCAN(N)                                                                      \
  case N:                                                                                \
    return bf16 ? launch_scan_t<uint16_t, N>(km, p, a, s) : launch_scan_t<float, N>(km, p, a, s);
    HSD_SCAN(1)
    HSD_SCAN(2)
    HSD_SCAN(3)
    HSD_SCAN(4)
#undef HSD_SCAN
    default: return cudaErrorInvalidValue;
  }
}

// ---- large k (k > HSD_K_MAX): every row's key, then a stable radix sort ----
//
// The register top-k lists hold 32 entries.  For larger k the scan above
// writes every row's order key (its exact fp64 chain, bit-identical to
// cosine_similarity) and a stable LSD radix sort of (key, row id) with the
// ids in ascending order yields exactly the reference's (score desc, id asc)
// order (store.cpp:66-69); the first k entries are the result.
namespace {

__global__ void iota_ids_kernel(uint32_t* __restrict__ v, int64_t n, int64_t base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (uint32_t)(base + i);
}

__global__ void emit_topk_kernel(const uint64_t* __restrict__ key, const uint32_t* __restrict__ id, int64_t rows,
                                 int k, double* __restrict__ scores, int32_t* __restrict__ ids) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    const bool ok = j < rows;
    scores[j] = ok ? key_score(key[j]) : -INFINITY;
    ids[j] = ok ? (int32_t)id[j] : -1;
  }
}

}  // namespace

bool exact_topk_large_supported(int dim, int key_dtype) { return exact_scan_supported(1, dim, key_dtype, 1); }

cudaError_t launch_exact_topk_large(const void* keys, int key_dtype, int64_t n_keys_total, int64_t row_begin,
                                    int64_t row_end, int dim, const float* queries, int B, int k, int num_sms,
                                    double* scores, int32_t* ids, cudaStream_t s) {
  const int64_t rows = row_end - row_begin;
  if (B < 1 || k < 1 || rows < 1 || rows > INT32_MAX || !exact_topk_large_supported(dim, key_dtype))
    return cudaErrorInvalidValue;
  const bool bf16 = key_dtype == HSD_DTYPE_BF16;
  int G = kScanMaxBatch;  // queries per scan: the widest group whose fp64 query slab fits
  while (G > 1 && !exact_scan_supported(G, dim, key_dtype, 1)) --G;
  G = std::min(G, B);
  uint64_t *kin = nullptr, *kout = nullptr;
  uint32_t *vin = nullptr, *vout = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kin, kout, vin, vout, rows, 0, 64, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&kin, (size_t)G * rows * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&kout, (size_t)rows * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&vin, (size_t)rows * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&vout, (size_t)rows * 4, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tmp_bytes, s);
  const int blocks = (int)std::min<int64_t>((rows + 255) / 256, (int64_t)num_sms * 8);
  for (int b0 = 0; e == cudaSuccess && b0 < B; b0 += G) {
    const int nq = std::min(G, B - b0);
    const ScanPlan p = bf16 ? scan_plan<uint16_t>(rows, dim, nq, num_sms) : scan_plan<float>(rows, dim, nq, num_sms);
    if (p.S < 2) {
      e = cudaErrorInvalidValue;
      break;
    }
    CUtensorMap km;
    const bool ok = bf16 ? tc_make_map_bf16(&km, keys, (uint64_t)n_keys_total, (uint64_t)dim, (uint32_t)p.R)
                         : tc_make_map(&km, (const float*)keys, (uint64_t)n_keys_total, (uint64_t)dim, (uint32_t)p.R);
    if (!ok) {
      e = cudaErrorInvalidValue;
      break;
    }
    ScanArgs a{};
    a.dim = dim;
    a.nchunk = bf16 ? (dim + 63) / 64 : (dim + 31) / 32;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.R = p.R;
    a.lpw = p.lpw;
    a.S = p.S;
    a.seg = p.seg;
    a.ntiles = p.ntiles;
    a.k = 1;
    a.queries = queries + (size_t)b0 * dim;
    a.allkey = kin;
    switch (nq) {
#define HSD_SCAN(N)                                                                                  \
  case N:                                                                                            \
    e = bf16 ? launch_scan_t<uint16_t, N>(km, p, a, s) : launch_scan_t<float, N>(km, p, a, s);       \
    break;
      HSD_SCAN(1)
      HSD_SCAN(2)
      HSD_SCAN(3)
      HSD_SCAN(4)
#undef HSD_SCAN
      default: e = cudaErrorInvalidValue;
    }
    for (int q = 0; e == cudaSuccess && q < nq; ++q) {
      iota_ids_kernel<<<blocks, 256, 0, s>>>(vin, rows, row_begin);
      e = cudaGetLastError();
      if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin + (size_t)q * rows, kout, vin, vout, rows, 0, 64, s);
      if (e == cudaSuccess) {
        const size_t o = (size_t)(b0 + q) * k;
        emit_topk_kernel<<<(int)std::min<int64_t>((k + 255) / 256, (int64_t)num_sms * 8), 256, 0, s>>>(
            kout, vout, rows, k, scores + o, ids + o);
        e = cudaGetLastError();
      }
    }
  }
  if (kin) cudaFreeAsync(kin, s);
  if (kout) cudaFreeAsync(kout, s);
  if (vin) cudaFreeAsync(vin, s);
  if (vout) cudaFreeAsync(vout, s);
  if (tmp) cudaFreeAsync(tmp, s);
  return e;
}

}  // namespace hsd
