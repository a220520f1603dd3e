// p2p.cuh — device helpers of the peer-memory exchange (k_p2p.cu layout):
// record / flag stores into a peer's receive window.
#pragma once

#include "kernels.h"

namespace hsd {

__device__ __forceinline__ void p2p_st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Record j of query b from `rank` into peer's window, slot epoch & 1.
__device__ __forceinline__ void p2p_put_record(const P2PWindows& w, int peer, int rank, int G, int b, int j,
                                               uint64_t epoch, double score, int32_t id, const uint8_t* tok32) {
  const int slot = (int)(epoch & 1);
  uint8_t* base = reinterpret_cast<uint8_t*>(w.base[peer]);
  const size_t d = (((size_t)slot * G + rank) * w.Bmax + b) * w.kmax + j;
  reinterpret_cast<double*>(base + w.off_scores)[d] = score;
  reinterpret_cast<int32_t*>(base + w.off_ids)[d] = id;
  uint4* dt = reinterpret_cast<uint4*>(base + w.off_toks) + d * 2;
  if (tok32) {
    const uint4* src = reinterpret_cast<const uint4*>(tok32);
    dt[0] = src[0];
    dt[1] = src[1];
  } else {
    dt[0] = make_uint4(0, 0, 0, 0);
    dt[1] = make_uint4(0, 0, 0, 0);
  }
}

// After a CTA's records of query b (all peers) are stored: fence, then
// flag[rank][b] = epoch in the peer's window (call from one thread).
__device__ __forceinline__ void p2p_put_flag(const P2PWindows& w, int peer, int rank, int G, int b, uint64_t epoch) {
  const int slot = (int)(epoch & 1);
  __threadfence_system();
  uint64_t* flags = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(w.base[peer]) + w.off_flags) +
                    ((size_t)slot * G + rank) * w.Bmax;
  p2p_st_release_sys(&flags[b], epoch);
}

}  // namespace hsd
