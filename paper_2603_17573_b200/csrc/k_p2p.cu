// k_p2p.cu — K3 over peer memory: the sharded search's exchange without NCCL.
//
// Every rank owns a receive window (cudaMalloc'd, shared by CUDA IPC handles)
// with two epoch-parity slots of [G][Bmax][k] records (fp64 score, int32 global
// id, 32-byte draft tokens) and [G][Bmax] per-query epoch flags.  A rank
//   publishes: K2's rank kernel (k_select.cu, fused) writes each query's final
//            top-k straight into slot (epoch & 1), row `rank`, of EVERY peer's
//            window (stores over NVLink / NVSwitch), then a system-scope
//            release fence and flag[rank][query] = epoch in each window;
//   merges:  query CTA b waits (acquire, bounded spin) until the G flags of
//            query b in its own window carry the epoch, then k-way merges the
//            G sorted lists in (score desc, id asc) order — bit-identical to
//            the NCCL path.
// Two parity slots suffice: a rank publishes epoch e + 2 into slot e & 1 only
// after its own merge of e + 1, which needed every peer's publish of e + 1,
// which each peer issued after finishing its merge of e.
#include "common.cuh"
#include "kernels.h"
#include "p2p.cuh"

namespace hsd {
namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Standalone publish from local buffers (used when a shard is empty): one CTA
// per (peer, query).
__global__ void p2p_publish_kernel(P2PWindows w, int rank, int G, int B, int k, uint64_t epoch,
                                   const double* __restrict__ ls, const int32_t* __restrict__ li,
                                   const uint8_t* __restrict__ lt) {
  const int peer = blockIdx.x, b = blockIdx.y;
  const int j = threadIdx.x;
  if (j < k) {
    const size_t i = (size_t)b * k + j;
    p2p_put_record(w, peer, rank, G, b, j, epoch, ls[i], li[i], lt ? lt + i * HSD_TOKENS_STRIDE : nullptr);
  }
  __syncthreads();
  if (j == 0) p2p_put_flag(w, peer, rank, G, b, epoch);
}

// One CTA per query: wait for every rank's records of this epoch, then merge.
__global__ void p2p_merge_kernel(P2PWindows w, int rank, int G, int B, int k, uint64_t epoch, double* __restrict__ scores,
                                 int32_t* __restrict__ ids, uint8_t* __restrict__ tok, int* __restrict__ err) {
  const int b = blockIdx.x;
  const int slot = (int)(epoch & 1);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(w.base[rank]);
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(base + w.off_flags) + (size_t)slot * G * w.Bmax;
    const long long t0 = clock64();
    int good = 1;
    for (int g = 0; g < G; ++g) {
      while (ld_acquire_sys(&flags[(size_t)g * w.Bmax + b]) < epoch) {
        if (clock64() - t0 > (1ll << 35)) {  // ~17 s: a peer never published -> report, do not hang
          good = 0;
          break;
        }
        __nanosleep(64);
      }
      if (!good) break;
    }
    ok = good;
    if (!good) *(volatile int*)err = 1;  // mapped host memory (api.cu): a plain store, same value from every writer
  }
  __syncthreads();
  if (!ok) {
    for (int r = threadIdx.x; r < k; r += blockDim.x) {
      scores[(size_t)b * k + r] = -INFINITY;
      ids[(size_t)b * k + r] = -1;
    }
    return;
  }
  const double* gs = reinterpret_cast<const double*>(base + w.off_scores) + (size_t)slot * G * w.Bmax * w.kmax;
  const int32_t* gi = reinterpret_cast<const int32_t*>(base + w.off_ids) + (size_t)slot * G * w.Bmax * w.kmax;
  const uint4* gt = reinterpret_cast<const uint4*>(base + w.off_toks) + (size_t)slot * G * w.Bmax * w.kmax * 2;
  const int n = G * k;
  auto at = [&](int c) { return ((size_t)(c / k) * w.Bmax + b) * w.kmax + (c % k); };
  __shared__ int valid;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    // the window is written by peers: read it from L2 (.cg), never from a stale L1 line
    const int32_t me = __ldcg(gi + at(i));
    if (me < 0) continue;
    atomicAdd(&valid, 1);
    const double s = __ldcg(gs + at(i));
    int r = 0;
    for (int c = 0; c < n; ++c) {
      const int32_t o = __ldcg(gi + at(c));
      if (o < 0) continue;
      const double os = __ldcg(gs + at(c));
      r += (os > s) || (os == s && o < me);
    }
    if (r < k) {
      scores[(size_t)b * k + r] = s;
      ids[(size_t)b * k + r] = me;
      if (tok) {
        uint4* dst = reinterpret_cast<uint4*>(tok + ((size_t)b * k + r) * HSD_TOKENS_STRIDE);
        dst[0] = __ldcg(gt + at(i) * 2);
        dst[1] = __ldcg(gt + at(i) * 2 + 1);
      }
    }
  }
  __syncthreads();
  for (int r = valid + threadIdx.x; r < k; r += blockDim.x) {
    scores[(size_t)b * k + r] = -INFINITY;
    ids[(size_t)b * k + r] = -1;
  }
}

}  // namespace

size_t p2p_window_bytes(int G, int Bmax, int kmax, P2PWindows* layout) {
  const size_t rec = (size_t)2 * G * Bmax * kmax;
  size_t off = 0;
  layout->off_flags = off;
  off += ((size_t)2 * G * Bmax * sizeof(uint64_t) + 255) & ~(size_t)255;
  layout->off_scores = off;
  off += (rec * sizeof(double) + 255) & ~(size_t)255;
  layout->off_ids = off;
  off += (rec * sizeof(int32_t) + 255) & ~(size_t)255;
  layout->off_toks = off;
  off += rec * HSD_TOKENS_STRIDE;
  layout->Bmax = Bmax;
  layout->kmax = kmax;
  return off;
}

cudaError_t launch_p2p_publish(const P2PWindows& w, int rank, int G, int B, int k, uint64_t epoch, const double* ls,
                               const int32_t* li, const uint8_t* lt, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  p2p_publish_kernel<<<dim3(G, B), 32, 0, s>>>(w, rank, G, B, k, epoch, ls, li, lt);
  return cudaGetLastError();
}

cudaError_t launch_p2p_merge(const P2PWindows& w, int rank, int G, int B, int k, uint64_t epoch, double* scores,
                             int32_t* ids, uint8_t* tok, int* err, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  p2p_merge_kernel<<<B, 128, 0, s>>>(w, rank, G, B, k, epoch, scores, ids, tok, err);
  return cudaGetLastError();
}

}  // namespace hsd
