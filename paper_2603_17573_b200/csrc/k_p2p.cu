// k_p2p.cu — K3 over peer memory: the sharded search's exchange without NCCL.
//
// Every rank owns a receive window (cudaMalloc'd, shared by CUDA IPC handles)
// with two epoch-parity slots of [G][Bmax][k] records (fp64 score, int32 global
// id, 32-byte draft tokens) and [G] epoch flags.  After its local top-k a rank
//   publish: writes its B x k records straight into slot (epoch & 1), row
//            `rank`, of EVERY peer's window (stores over NVLink / NVSwitch),
//            then a system-scope release fence and flag[rank] = epoch in each
//            peer's window;
//   merge:   waits (acquire, bounded spin) until all G flags of its own window
//            carry the epoch, then k-way merges the G sorted lists in
//            (score desc, id asc) order — bit-identical to the NCCL path.
// Two parity slots suffice: a rank publishes epoch e + 2 into slot e & 1 only
// after its own merge of e + 1, which needed every peer's publish of e + 1,
// which each peer issued after finishing its merge of e.
#include "common.cuh"
#include "kernels.h"

namespace hsd {
namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One CTA per destination peer.
__global__ void p2p_publish_kernel(P2PWindows w, int rank, int G, int B, int k, uint64_t epoch,
                                   const double* __restrict__ ls, const int32_t* __restrict__ li,
                                   const uint8_t* __restrict__ lt) {
  const int peer = blockIdx.x;
  const int slot = (int)(epoch & 1);
  uint8_t* base = reinterpret_cast<uint8_t*>(w.base[peer]);
  double* ds = reinterpret_cast<double*>(base + w.off_scores) + ((size_t)slot * G + rank) * w.Bmax * w.kmax;
  int32_t* di = reinterpret_cast<int32_t*>(base + w.off_ids) + ((size_t)slot * G + rank) * w.Bmax * w.kmax;
  uint4* dt = reinterpret_cast<uint4*>(base + w.off_toks) + ((size_t)slot * G + rank) * w.Bmax * w.kmax * 2;
  const int n = B * k;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int b = i / k, j = i % k;
    const size_t d = (size_t)b * w.kmax + j;
    ds[d] = ls[i];
    di[d] = li[i];
    const uint4* src = reinterpret_cast<const uint4*>(lt + (size_t)i * HSD_TOKENS_STRIDE);
    dt[d * 2] = src[0];
    dt[d * 2 + 1] = src[1];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t* flags = reinterpret_cast<uint64_t*>(base + w.off_flags) + (size_t)slot * G;
    st_release_sys(&flags[rank], epoch);
  }
}

// One CTA per query: wait for every rank's records of this epoch, then merge.
__global__ void p2p_merge_kernel(P2PWindows w, int rank, int G, int B, int k, uint64_t epoch, double* __restrict__ scores,
                                 int32_t* __restrict__ ids, uint8_t* __restrict__ tok, int* __restrict__ err) {
  const int b = blockIdx.x;
  const int slot = (int)(epoch & 1);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(w.base[rank]);
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const uint64_t* flags = reinterpret_cast<const uint64_t*>(base + w.off_flags) + (size_t)slot * G;
    const long long t0 = clock64();
    int good = 1;
    for (int g = 0; g < G; ++g) {
      while (ld_acquire_sys(&flags[g]) < epoch) {
        if (clock64() - t0 > (1ll << 35)) {  // ~17 s: a peer never published -> report, do not hang
          good = 0;
          break;
        }
        __nanosleep(64);
      }
      if (!good) break;
    }
    ok = good;
    if (!good) atomicExch(err, 1);
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
  off += ((size_t)2 * G * sizeof(uint64_t) + 255) & ~(size_t)255;
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

cudaError_t launch_p2p_exchange(const P2PWindows& w, int rank, int G, int B, int k, uint64_t epoch,
                                const double* ls, const int32_t* li, const uint8_t* lt, double* scores, int32_t* ids,
                                uint8_t* tok, int* err, cudaStream_t s) {
  p2p_publish_kernel<<<G, 256, 0, s>>>(w, rank, G, B, k, epoch, ls, li, lt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  p2p_merge_kernel<<<B, 128, 0, s>>>(w, rank, G, B, k, epoch, scores, ids, tok, err);
  return cudaGetLastError();
}

}  // namespace hsd
