// api.cu — C ABI (include/hsd/hsd_gpu.h): collection handle, search / verify /
// kinematics entry points, fused step engine and the NCCL-sharded search.
// Host code only; kernels live in k_*.cu.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "hsd/hsd_gpu.h"
#include "hsd/hsd_synth.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;
thread_local long g_err_line = 0;

hsd_status fail(hsd_status st, const char* fmt, ...) {
  g_err_line = 0;
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

hsd_status cuda_fail(cudaError_t e, const char* what) {
  cudaGetLastError();  // clear sticky-free errors
  return fail(e == cudaErrorMemoryAllocation ? HSD_ERR_OOM : HSD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CU(x)                                     \
  do {                                            \
    cudaError_t e_ = (x);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x); \
  } while (0)

#define NC(x)                                                                         \
  do {                                                                                \
    ncclResult_t r_ = (x);                                                            \
    if (r_ != ncclSuccess) return fail(HSD_ERR_NCCL, "%s: %s", #x, ncclGetErrorString(r_)); \
  } while (0)

// Every compute entry point requires an sm_100 device; there is no CPU path.
hsd_status require_device(int device) {
  static int s_count = -1;
  static signed char s_ok[64] = {0};  // 0 unknown, 1 sm_100, -1 other
  if (s_count < 0) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    s_count = n;
  }
  if (s_count == 0) return fail(HSD_ERR_NO_DEVICE, "no CUDA device visible (the HeiSD hot path has no CPU fallback)");
  if (device < 0 || device >= s_count || device >= 64)
    return fail(HSD_ERR_INVALID_INPUT, "device %d out of range [0, %d)", device, s_count);
  if (s_ok[device] == 0) {
    int major = 0, minor = 0;
    CU(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CU(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    s_ok[device] = major == 10 ? 1 : -1;
    if (major != 10)
      return fail(HSD_ERR_NO_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a", device, major, minor);
  }
  if (s_ok[device] < 0) return fail(HSD_ERR_NO_DEVICE, "device %d is not sm_100", device);
  CU(cudaSetDevice(device));
  return HSD_OK;
}

constexpr int kMaxSms = 256;  // sizing bound of per-SM scratch

int num_sms(int device) {
  static int cache[64] = {0};
  if (device >= 0 && device < 64 && cache[device]) return cache[device];
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (device >= 0 && device < 64) cache[device] = v;
  return v;
}

__global__ void fill_empty_kernel(double* scores, int32_t* ids, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    scores[i] = -INFINITY;
    ids[i] = -1;
  }
}

__global__ void offset_ids_kernel(int32_t* ids, int n, int64_t off) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && ids[i] >= 0) ids[i] = (int32_t)(ids[i] + off);
}

// Device scratch of one search stream (or one engine): K1's filter lists, the
// padded query slab, K2's per-query state and the search statistics.
struct Scratch {
  uint64_t* partial = nullptr;
  size_t partial_cap = 0;  // bytes
  void* sel = nullptr;     // K2 per-query candidate / exact-score scratch
  size_t sel_cap = 0;
  void* qslab = nullptr;   // K1's padded query slab (TMA source)
  size_t qslab_cap = 0;
  int* stats = nullptr;    // [0] fallback queries, [1] pooled candidates, [2] fallback lists (accumulated)
  void* scan = nullptr;    // K1x exact scan: ticket + per-CTA lists (zeroed once; the ticket self-resets)
  bool fixed = false;      // engine-owned: never reallocated (captured graphs hold its pointers)
};

}  // namespace

struct hsd_collection {
  int device = 0;
  int dim = 0;
  int dtype = HSD_DTYPE_F32;
  int64_t n = 0;
  int64_t cap = 0;
  void* keys = nullptr;  // fp32 or bf16 [cap][dim]
  // Optional bf16 filter copy of an fp32 collection ([cap][dim], RN-even):
  // the tensor-core filter streams it (half the HBM bytes); the exact fp64
  // rescoring still reads the fp32 keys, so results are unchanged.
  uint16_t* shadow = nullptr;
  uint8_t* tokens = nullptr;
  unsigned long long* maxnorm = nullptr;  // fp64 bits of max row norm
  // Record::feature (store.hpp:40-42): verifier features captured at recording
  // time, fp32 [cap][d_f] + presence [cap] (allocated on first use; d_f fixed)
  float* feat = nullptr;
  uint8_t* has_feat = nullptr;
  int d_f = 0;
  // bumped by every row mutation: an approximate index built at an older
  // generation is stale (the reference drops its HNSW index on insert)
  uint64_t gen = 0;
  std::mutex mu;
  std::unordered_map<cudaStream_t, Scratch> scratch;
};

namespace {

size_t key_bytes(const hsd_collection* c) { return c->dtype == HSD_DTYPE_BF16 ? 2 : 4; }

hsd_status ensure_capacity(hsd_collection* c, int64_t need) {
  if (need <= c->cap) return HSD_OK;
  int64_t ncap = std::max<int64_t>(need, c->cap * 2);
  void* nk = nullptr;
  uint8_t* nt = nullptr;
  CU(cudaMalloc(&nk, (size_t)ncap * c->dim * key_bytes(c)));
  cudaError_t e = cudaMalloc(&nt, (size_t)ncap * HSD_TOKENS_STRIDE);
  if (e != cudaSuccess) {
    cudaFree(nk);
    return cuda_fail(e, "cudaMalloc(tokens)");
  }
  if (c->n > 0) {
    CU(cudaMemcpy(nk, c->keys, (size_t)c->n * c->dim * key_bytes(c), cudaMemcpyDeviceToDevice));
    CU(cudaMemcpy(nt, c->tokens, (size_t)c->n * HSD_TOKENS_STRIDE, cudaMemcpyDeviceToDevice));
  }
  if (c->shadow) {
    uint16_t* ns = nullptr;
    cudaError_t e2 = cudaMalloc(&ns, (size_t)ncap * c->dim * 2);
    if (e2 != cudaSuccess) {
      cudaFree(nk);
      cudaFree(nt);
      return cuda_fail(e2, "cudaMalloc(filter shadow)");
    }
    if (c->n > 0) CU(cudaMemcpy(ns, c->shadow, (size_t)c->n * c->dim * 2, cudaMemcpyDeviceToDevice));
    cudaFree(c->shadow);
    c->shadow = ns;
  }
  if (c->feat) {
    float* nf = nullptr;
    uint8_t* nh = nullptr;
    cudaError_t e2 = cudaMalloc(&nf, (size_t)ncap * c->d_f * 4);
    if (e2 == cudaSuccess) e2 = cudaMalloc(&nh, (size_t)ncap);
    if (e2 != cudaSuccess) {
      cudaFree(nk);
      cudaFree(nt);
      cudaFree(nf);
      return cuda_fail(e2, "cudaMalloc(features)");
    }
    CU(cudaMemset(nf, 0, (size_t)ncap * c->d_f * 4));
    CU(cudaMemset(nh, 0, (size_t)ncap));
    if (c->n > 0) {
      CU(cudaMemcpy(nf, c->feat, (size_t)c->n * c->d_f * 4, cudaMemcpyDeviceToDevice));
      CU(cudaMemcpy(nh, c->has_feat, (size_t)c->n, cudaMemcpyDeviceToDevice));
    }
    cudaFree(c->feat);
    cudaFree(c->has_feat);
    c->feat = nf;
    c->has_feat = nh;
  }
  cudaFree(c->keys);
  cudaFree(c->tokens);
  c->keys = nk;
  c->tokens = nt;
  c->cap = ncap;
  return HSD_OK;
}

// bf16 filter copy of rows [row0, row0 + n) of an fp32 collection.
hsd_status refresh_shadow(hsd_collection* c, int64_t row0, int64_t n) {
  if (!c->shadow || n <= 0) return HSD_OK;
  CU(hsd::launch_to_bf16((const float*)c->keys + (size_t)row0 * c->dim, n * c->dim,
                         c->shadow + (size_t)row0 * c->dim, 0));
  return HSD_OK;
}

// Scratch bytes of one search of B queries over `rows` rows on `nsm` SMs
// (all_sizes: of ANY search of up to B queries — an engine's fixed scratch).
// Every pass may use a different list count (pair clusters, the tail pass):
// the lists are sized for the largest lists(Bs) * Bs.
void scratch_need(int B, int64_t rows, int nsm, int dim, bool all_sizes, size_t* partial, size_t* sel,
                  size_t* qslab) {
  const int W = hsd::kMaxBatchPass;
  size_t p = 0;
  if (all_sizes) {
    for (int t = 1; t <= std::min(B, W); ++t) p = std::max(p, (size_t)hsd::sim_wide_lists(t, rows, nsm) * t);
  } else {
    for (int b0 = 0; b0 < B; b0 += W) {
      const int Bs = std::min(W, B - b0);
      p = std::max(p, (size_t)hsd::sim_wide_lists(Bs, rows, nsm) * Bs);
    }
  }
  *partial = p * hsd::dev::kCandLocal * sizeof(uint64_t);
  *sel = hsd::select_scratch_bytes(std::min(B, W));
  *qslab = hsd::sim_wide_scratch_bytes(dim);
}

hsd_status alloc_scratch(Scratch& sc, size_t partial_bytes, size_t sel_bytes, size_t qslab_bytes) {
  if (!sc.stats) {
    CU(cudaMalloc(&sc.stats, 4 * sizeof(int)));
    CU(cudaMemset(sc.stats, 0, 4 * sizeof(int)));
  }
  if (!sc.scan) {
    const size_t b = hsd::exact_scan_scratch_bytes(hsd::kScanMaxBatch, kMaxSms);
    CU(cudaMalloc(&sc.scan, b));
    CU(cudaMemset(sc.scan, 0, b));
  }
  auto grow = [&](void** p, size_t* cap, size_t need) -> cudaError_t {
    if (*cap >= need) return cudaSuccess;
    cudaFree(*p);  // implicit device synchronisation: no kernel still reads the old buffer
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e == cudaSuccess) *cap = need;
    return e;
  };
  CU(grow((void**)&sc.partial, &sc.partial_cap, partial_bytes));
  CU(grow(&sc.sel, &sc.sel_cap, sel_bytes));
  CU(grow(&sc.qslab, &sc.qslab_cap, qslab_bytes));
  return HSD_OK;
}

void free_scratch(Scratch& sc) {
  cudaFree(sc.partial);
  cudaFree(sc.sel);
  cudaFree(sc.qslab);
  cudaFree(sc.stats);
  cudaFree(sc.scan);
  sc = Scratch{};
}

hsd_status get_scratch(hsd_collection* c, cudaStream_t s, size_t partial_bytes, size_t sel_bytes, size_t qslab_bytes,
                       Scratch** out) {
  std::lock_guard<std::mutex> lk(c->mu);
  Scratch& sc = c->scratch[s];
  hsd_status st = alloc_scratch(sc, partial_bytes, sel_bytes, qslab_bytes);
  if (st != HSD_OK) return st;
  *out = &sc;
  return HSD_OK;
}

// Optional stage events (engine timing): marks[i] is recorded after stage i.
struct StageMarks {
  cudaEvent_t after_sim = nullptr;
  cudaEvent_t after_select = nullptr;
};

// Search path override (hsd_set_sim_path): 0 auto, 1 single-CTA wide
// kernels, 2 filter + rescoring only, 3 exact scan wherever it applies.
std::atomic<int> g_search_path{0};

// K1x (exact scan of every row) or K1 + K2 (filter + exact rescoring): the
// cheaper by the measured cost model.  The filter streams the
// bf16 copy (or the stored keys), then pays K2's chain after the scan; the
// exact scan streams the stored keys with the chains running underneath.
bool use_exact_scan(const hsd_collection* c, int B, int k, int64_t rows) {
  const int mode = g_search_path.load();
  if (mode == 1 || mode == 2) return false;
  if (!hsd::exact_scan_supported(B, c->dim, c->dtype, k)) return false;
  if (mode == 3) return true;
  const double fbytes = (double)rows * c->dim * (c->shadow ? 2 : (int)key_bytes(c));
  const double filter_us = fbytes / 6.5e6 + 12.0 + c->dim * 0.0095;
  return hsd::exact_scan_cost_us(rows, c->dim, c->dtype, B) < filter_us;
}

constexpr int kShadowGamma = 0x100;  // sim_wide_gamma flag: bf16-rounded keys (filter shadow)

// K1 + K2 over rows [rb, re) in passes of up to 1024 queries.
// own != nullptr: the engine's fixed scratch (sized at engine creation).
// pub != nullptr: sharded search over peer memory — the final per-query
// top-k records are published into the peers' windows by K2 (scores / ids
// are then scratch for an empty shard only).
hsd_status search_impl(hsd_collection* c, const float* queries, int B, int k, int64_t rb, int64_t re, double* scores,
                       int32_t* ids, cudaStream_t s, const StageMarks* marks = nullptr, int reserve_sms = 0,
                       const hsd::P2PPublish* pub = nullptr, Scratch* own = nullptr) {
  if (k < 1) return fail(HSD_ERR_INVALID_INPUT, "k must be >= 1");  // store.cpp:60
  // k > HSD_K_MAX: the exact scan of every row + a stable radix sort (a
  // plain search only; the engine, sharded and index paths keep k <= 32)
  const bool large_k = k > HSD_K_MAX;
  if (large_k && (pub || own || marks))
    return fail(HSD_ERR_INVALID_INPUT, "k = %d exceeds HSD_K_MAX = %d", k, HSD_K_MAX);
  if (B < 0) return fail(HSD_ERR_INVALID_INPUT, "negative batch");
  if (B == 0) return HSD_OK;
  if (!queries || !scores || !ids) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (reinterpret_cast<uintptr_t>(queries) % 16)  // 128-bit / cp.async / TMA staging of query rows
    return fail(HSD_ERR_INVALID_INPUT, "queries must be 16-byte aligned");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  rb = std::max<int64_t>(rb, 0);
  re = std::min<int64_t>(re, c->n);
  const int64_t rows = re - rb;
  if (rows <= 0) {  // empty collection -> empty result, no error (store.cpp:62-72)
    const int64_t n = (int64_t)B * k;
    fill_empty_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 64), 256, 0, s>>>(scores, ids, n);
    CU(cudaGetLastError());
    if (pub) CU(hsd::launch_p2p_publish(pub->w, pub->rank, pub->G, B, k, pub->epoch, scores, ids, nullptr, s));
    return HSD_OK;
  }
  if (large_k) {
    if (!hsd::exact_topk_large_supported(c->dim, c->dtype))
      return fail(HSD_ERR_INVALID_INPUT, "k = %d > HSD_K_MAX needs dim <= ~17000 (fp64 query slab), got %d", k, c->dim);
    CU(hsd::launch_exact_topk_large(c->keys, c->dtype, c->n, rb, re, c->dim, queries, B, k,
                                    std::min(num_sms(c->device), kMaxSms), scores, ids, s));
    return HSD_OK;
  }
  // reserve_sms: SMs left free for work running concurrently on another stream
  // (the engine's kinematics); the persistent tcgen05 kernel sizes its grid to
  // the rest so neither waits for the other's CTAs to retire.
  const int nsm = std::max(1, num_sms(c->device) - std::max(0, reserve_sms));
  size_t need_p = 0, need_s = 0, need_q = 0;
  scratch_need(B, rows, nsm, c->dim, false, &need_p, &need_s, &need_q);
  Scratch* sc = own;
  if (own) {
    if (own->partial_cap < need_p || own->sel_cap < need_s || own->qslab_cap < need_q)
      return fail(HSD_ERR_INVALID_INPUT, "engine scratch too small for this step (batch %d)", B);
  } else {
    st = get_scratch(c, s, need_p, need_s, need_q, &sc);
    if (st != HSD_OK) return st;
  }
  // the filter: the bf16 copy of an fp32 collection when present (half the
  // bytes; both operands bf16-rounded), else the stored keys (TF32 / bf16)
  const void* fkeys = c->shadow ? (const void*)c->shadow : c->keys;
  const int fdtype = c->shadow ? HSD_DTYPE_BF16 : c->dtype;
  const double gamma = c->shadow ? hsd::sim_wide_gamma(c->dim, HSD_DTYPE_BF16 | kShadowGamma)
                                 : hsd::sim_wide_gamma(c->dim, c->dtype);
  if (!pub && use_exact_scan(c, B, k, rows)) {
    // K1x: every row's exact chain while the keys stream (small rows x batch)
    CU(hsd::launch_exact_scan(c->keys, c->dtype, c->n, rb, re, c->dim, queries, B, k, sc->scan,
                              std::min(nsm, kMaxSms), scores, ids, s));
    if (marks && marks->after_sim) CU(cudaEventRecord(marks->after_sim, s));
    if (marks && marks->after_select) CU(cudaEventRecord(marks->after_select, s));
    return HSD_OK;
  }
  const int W = hsd::kMaxBatchPass;
  for (int b0 = 0; b0 < B; b0 += W) {
    const int Bs = std::min(W, B - b0);
    const int lists = hsd::sim_wide_lists(Bs, rows, nsm);
    if (lists > hsd::select_max_lists()) return fail(HSD_ERR_CONFIG, "%d filter lists exceed the select kernel", lists);
    const float* q = queries + (size_t)b0 * c->dim;
    hsd::ListGeom geom{};
    CU(hsd::launch_sim_wide(fkeys, fdtype, c->n, rb, re, c->dim, q, Bs, lists, sc->qslab, sc->partial, nullptr, s,
                            &geom));
    if (marks && marks->after_sim && b0 + W >= B) CU(cudaEventRecord(marks->after_sim, s));
    hsd::P2PPublish pb{};
    if (pub) {
      pb = *pub;
      pb.q_offset = b0;
    }
    // fp32 keys converted to bf16 on chip (CTA-pair passes): the bf16-copy bound
    const double g = !c->shadow && hsd::sim_wide_converts(fdtype, Bs, c->dim)
                         ? hsd::sim_wide_gamma(c->dim, HSD_DTYPE_BF16 | kShadowGamma)
                         : gamma;
    CU(hsd::launch_select(sc->partial, lists, Bs, k, c->keys, c->dtype, c->dim, q, c->maxnorm, g, geom,
                          scores + (size_t)b0 * k, ids + (size_t)b0 * k, sc->stats, sc->sel, nsm, s,
                          pub ? &pb : nullptr));
  }
  if (marks && marks->after_select) CU(cudaEventRecord(marks->after_select, s));
  return HSD_OK;
}

}  // namespace

extern "C" {

const char* hsd_last_error(void) { return g_err.c_str(); }
long hsd_last_error_line(void) { return g_err_line; }
int hsd_abi_version(void) { return HSD_ABI_VERSION; }

hsd_status hsd_device_count(int* n) {
  if (!n) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess) {
    cudaGetLastError();
    cnt = 0;
  }
  int ok = 0;
  for (int d = 0; d < cnt; ++d) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++ok;
  }
  *n = ok;
  return HSD_OK;
}

hsd_status hsd_collection_create(int device, int dim, int64_t capacity, hsd_collection** out) {
  return hsd_collection_create_ex(device, dim, capacity, HSD_DTYPE_F32, out);
}

hsd_status hsd_collection_create_ex(int device, int dim, int64_t capacity, int dtype, hsd_collection** out) {
  if (!out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *out = nullptr;
  if (dim < 1) return fail(HSD_ERR_CONFIG, "collection dim must be >= 1");  // store.cpp:37
  if (dtype != HSD_DTYPE_F32 && dtype != HSD_DTYPE_BF16) return fail(HSD_ERR_CONFIG, "unknown key dtype %d", dtype);
  if (dim % 4 != 0) return fail(HSD_ERR_CONFIG, "dim must be a multiple of 4 (128-bit loads), got %d", dim);
  if (dtype == HSD_DTYPE_BF16 && dim % 8 != 0)
    return fail(HSD_ERR_CONFIG, "bf16 collections need dim a multiple of 8 (16-B rows), got %d", dim);
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  auto* c = new hsd_collection();
  c->device = device;
  c->dim = dim;
  c->dtype = dtype;
  cudaError_t e = cudaMalloc(&c->maxnorm, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(c->maxnorm, 0, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(maxnorm)");
  }
  st = ensure_capacity(c, std::max<int64_t>(capacity, 1));
  if (st != HSD_OK) {
    hsd_collection_destroy(c);
    return st;
  }
  *out = c;
  return HSD_OK;
}

hsd_status hsd_collection_destroy(hsd_collection* c) {
  if (!c) return HSD_OK;
  cudaSetDevice(c->device);
  for (auto& kv : c->scratch) free_scratch(kv.second);
  cudaFree(c->keys);
  cudaFree(c->tokens);
  cudaFree(c->shadow);
  cudaFree(c->maxnorm);
  cudaFree(c->feat);
  cudaFree(c->has_feat);
  delete c;
  cudaGetLastError();
  return HSD_OK;
}

hsd_status hsd_collection_size(const hsd_collection* c, int64_t* n) {
  if (!c || !n) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *n = c->n;
  return HSD_OK;
}

hsd_status hsd_collection_dim(const hsd_collection* c, int* dim) {
  if (!c || !dim) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *dim = c->dim;
  return HSD_OK;
}

hsd_status hsd_collection_device(const hsd_collection* c, int* device) {
  if (!c || !device) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *device = c->device;
  return HSD_OK;
}

hsd_status hsd_collection_keys(const hsd_collection* c, const float** keys, const uint8_t** tokens) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (keys && c->dtype != HSD_DTYPE_F32) return fail(HSD_ERR_INVALID_INPUT, "fp32 key view of a bf16 collection");
  if (keys) *keys = (const float*)c->keys;
  if (tokens) *tokens = c->tokens;
  return HSD_OK;
}

hsd_status hsd_collection_set_filter(hsd_collection* c, int filter) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  if (filter != HSD_FILTER_NATIVE && filter != HSD_FILTER_BF16_COPY)
    return fail(HSD_ERR_CONFIG, "unknown filter mode %d", filter);
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  if (filter == HSD_FILTER_NATIVE) {
    CU(cudaDeviceSynchronize());
    cudaFree(c->shadow);
    c->shadow = nullptr;
    return HSD_OK;
  }
  if (c->dtype != HSD_DTYPE_F32) return fail(HSD_ERR_CONFIG, "the bf16 filter copy applies to fp32 collections");
  if (c->dim % 8) return fail(HSD_ERR_CONFIG, "the bf16 filter copy needs dim % 8 == 0");
  if (c->shadow) return HSD_OK;
  CU(cudaMalloc(&c->shadow, (size_t)c->cap * c->dim * 2));
  st = refresh_shadow(c, 0, c->n);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  return HSD_OK;
}

hsd_status hsd_collection_get_filter(const hsd_collection* c, int* filter) {
  if (!c || !filter) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *filter = c->shadow ? HSD_FILTER_BF16_COPY : HSD_FILTER_NATIVE;
  return HSD_OK;
}

hsd_status hsd_collection_dtype(const hsd_collection* c, int* dtype) {
  if (!c || !dtype) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *dtype = c->dtype;
  return HSD_OK;
}

hsd_status hsd_collection_data(const hsd_collection* c, const void** keys, const uint8_t** tokens) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (keys) *keys = c->keys;
  if (tokens) *tokens = c->tokens;
  return HSD_OK;
}

hsd_status hsd_collection_insert(hsd_collection* c, const float* emb, const double* next_actions,
                                 const int32_t* episode_idx, const int32_t* step_idx, int64_t n, int64_t* first_id) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  if (n < 0) return fail(HSD_ERR_INVALID_INPUT, "negative record count");
  if (first_id) *first_id = c->n;
  if (n == 0) return HSD_OK;
  if (!emb || !next_actions) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  for (int64_t i = 0; i < n; ++i)  // store.cpp:50-52
    if ((episode_idx && episode_idx[i] < 0) || (step_idx && step_idx[i] < 0))
      return fail(HSD_ERR_SCHEMA, "payload indices must be nonnegative");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  st = ensure_capacity(c, c->n + n);
  if (st != HSD_OK) return st;
  double* dact = nullptr;
  int32_t* dbad = nullptr;
  CU(cudaMalloc(&dact, (size_t)n * 21 * sizeof(double)));
  CU(cudaMalloc(&dbad, sizeof(int32_t)));
  int32_t bad = 0;
  cudaError_t e = cudaMemcpy(dact, next_actions, (size_t)n * 21 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(dbad, 0, sizeof(int32_t));
  if (e == cudaSuccess) e = hsd::launch_quantize_tokens(dact, n, c->tokens + (size_t)c->n * HSD_TOKENS_STRIDE, dbad, 0);
  if (e == cudaSuccess) e = cudaMemcpy(&bad, dbad, sizeof(int32_t), cudaMemcpyDeviceToHost);
  cudaFree(dact);
  cudaFree(dbad);
  if (e != cudaSuccess) return cuda_fail(e, "insert: quantize payload");
  if (bad) return fail(HSD_ERR_INVALID_INPUT, "non-finite action value in payload");  // actions.cpp:38-40
  if (c->dtype == HSD_DTYPE_BF16) {
    float* tmp = nullptr;
    CU(cudaMalloc(&tmp, (size_t)n * c->dim * sizeof(float)));
    e = cudaMemcpy(tmp, emb, (size_t)n * c->dim * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = hsd::launch_to_bf16(tmp, n * c->dim, (uint16_t*)c->keys + (size_t)c->n * c->dim, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "insert: bf16 keys");
  } else {
    CU(cudaMemcpy((float*)c->keys + (size_t)c->n * c->dim, emb, (size_t)n * c->dim * sizeof(float),
                  cudaMemcpyHostToDevice));
  }
  CU(hsd::launch_row_norms(c->keys, c->dtype, c->n, n, c->dim, c->maxnorm, 0));
  st = refresh_shadow(c, c->n, n);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  c->n += n;
  ++c->gen;
  return HSD_OK;
}

hsd_status hsd_collection_set_features(hsd_collection* c, int64_t row0, int64_t n, int d_f, const float* feat,
                                       const uint8_t* has) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  if (n < 0 || row0 < 0 || row0 + n > c->n) return fail(HSD_ERR_INVALID_INPUT, "feature rows outside the collection");
  if (d_f < 1) return fail(HSD_ERR_INVALID_INPUT, "feature dim must be >= 1");
  if (c->d_f && c->d_f != d_f)
    return fail(HSD_ERR_SCHEMA, "feature length %d differs from the collection's first feature (%d)", d_f, c->d_f);
  if (n > 0 && !feat) return fail(HSD_ERR_INVALID_INPUT, "null features");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  if (!c->feat) {
    CU(cudaMalloc(&c->feat, (size_t)c->cap * d_f * 4));
    CU(cudaMalloc(&c->has_feat, (size_t)c->cap));
    CU(cudaMemset(c->feat, 0, (size_t)c->cap * d_f * 4));
    CU(cudaMemset(c->has_feat, 0, (size_t)c->cap));
    c->d_f = d_f;
  }
  if (n == 0) return HSD_OK;
  CU(cudaMemcpy(c->feat + (size_t)row0 * d_f, feat, (size_t)n * d_f * 4, cudaMemcpyHostToDevice));
  if (has) {
    CU(cudaMemcpy(c->has_feat + row0, has, (size_t)n, cudaMemcpyHostToDevice));
  } else {
    CU(cudaMemset(c->has_feat + row0, 1, (size_t)n));
  }
  return HSD_OK;
}

hsd_status hsd_collection_features(const hsd_collection* c, const float** feat, const uint8_t** has, int* d_f) {
  if (!c || !feat || !d_f) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *feat = c->feat;
  if (has) *has = c->has_feat;
  *d_f = c->d_f;
  return HSD_OK;
}

hsd_status hsd_collection_generate(hsd_collection* c, int kind, uint64_t db_seed, int64_t n) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  return hsd_collection_generate_rows(c, kind, db_seed, c->n, n);
}

hsd_status hsd_collection_generate_rows(hsd_collection* c, int kind, uint64_t db_seed, int64_t row0, int64_t n) {
  return hsd_collection_generate_ex(c, kind, db_seed, row0, n, HSD_PAYLOAD_RANDOM, 0);
}

hsd_status hsd_collection_generate_ex(hsd_collection* c, int kind, uint64_t db_seed, int64_t row0, int64_t n,
                                      int payload, int traj_T) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  if (payload != HSD_PAYLOAD_RANDOM && payload != HSD_PAYLOAD_TRAJ)
    return fail(HSD_ERR_CONFIG, "unknown payload family %d", payload);
  if (payload == HSD_PAYLOAD_TRAJ && traj_T < 1) return fail(HSD_ERR_CONFIG, "traj_T must be >= 1");
  if (row0 < 0) return fail(HSD_ERR_INVALID_INPUT, "negative row offset");
  if (kind < HSD_SYNTH_EXACT || kind > HSD_SYNTH_CLUSTER) return fail(HSD_ERR_CONFIG, "unknown synthetic family %d", kind);
  if (n < 0) return fail(HSD_ERR_INVALID_INPUT, "negative record count");
  if (n == 0) return HSD_OK;
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  st = ensure_capacity(c, c->n + n);
  if (st != HSD_OK) return st;
  CU(hsd::launch_gen_keys(kind, db_seed, row0, n, c->dim, (uint8_t*)c->keys + (size_t)c->n * c->dim * key_bytes(c),
                          c->dtype, c->tokens + (size_t)c->n * HSD_TOKENS_STRIDE, c->maxnorm, payload, traj_T, 0));
  st = refresh_shadow(c, c->n, n);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  c->n += n;
  ++c->gen;
  return HSD_OK;
}

hsd_status hsd_search_topk_exact(hsd_collection* c, const float* queries, int B, int k, double* scores, int32_t* ids,
                                 void* stream) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  return search_impl(c, queries, B, k, 0, c->n, scores, ids, (cudaStream_t)stream);
}

hsd_status hsd_search_topk_range(hsd_collection* c, const float* queries, int B, int k, int64_t row_begin,
                                 int64_t row_end, double* scores, int32_t* ids, void* stream) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  if (row_begin > row_end) return fail(HSD_ERR_INVALID_INPUT, "row_begin > row_end");
  return search_impl(c, queries, B, k, row_begin, row_end, scores, ids, (cudaStream_t)stream);
}

hsd_status hsd_set_sim_path(int path) {
  if (path < 0 || path > 3)
    return fail(HSD_ERR_INVALID_INPUT,
                "path must be 0 (auto), 1 (single-CTA wide kernels, no CTA pairs), 2 (filter + rescoring only) "
                "or 3 (exact scan wherever it applies)");
  hsd::sim_wide_set_single(path == 1);
  g_search_path.store(path);
  return HSD_OK;
}

hsd_status hsd_search_plan(hsd_collection* c, int B, int k, int64_t rows, int* exact_scan) {
  if (!c || !exact_scan) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *exact_scan = use_exact_scan(c, B, k, rows < 0 ? c->n : rows) ? 1 : 0;
  const int Bs = std::min(B, hsd::kMaxBatchPass);
  if (!*exact_scan && !c->shadow && hsd::sim_wide_converts(c->dtype, Bs, c->dim)) *exact_scan = 2;
  return HSD_OK;
}

hsd_status hsd_debug_sim_scores(hsd_collection* c, const float* queries, int B, int variant, float* out,
                                void* stream) {
  if (!c || !queries || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (variant != 1 && variant != 4)
    return fail(HSD_ERR_INVALID_INPUT, "variant must be 1 (stored keys: TF32 / bf16) or 4 (bf16 filter copy)");
  if (variant == 4 && !c->shadow) return fail(HSD_ERR_INVALID_INPUT, "collection has no bf16 filter copy");
  if (B < 1 || B > 256) return fail(HSD_ERR_INVALID_INPUT, "debug dump supports 1 <= B <= 256");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  if (c->n == 0) return HSD_OK;
  const int nsm = num_sms(c->device);
  size_t need_p = 0, need_s = 0, need_q = 0;
  scratch_need(B, c->n, nsm, c->dim, false, &need_p, &need_s, &need_q);
  const int lists = hsd::sim_wide_lists(B, c->n, nsm);
  Scratch* sc = nullptr;
  st = get_scratch(c, (cudaStream_t)stream, need_p, need_s, need_q, &sc);
  if (st != HSD_OK) return st;
  if (variant == 4)
    CU(hsd::launch_sim_wide(c->shadow, HSD_DTYPE_BF16, c->n, 0, c->n, c->dim, queries, B, lists, sc->qslab,
                            sc->partial, out, (cudaStream_t)stream));
  else
    CU(hsd::launch_sim_wide(c->keys, c->dtype, c->n, 0, c->n, c->dim, queries, B, lists, sc->qslab, sc->partial, out,
                            (cudaStream_t)stream));
  return HSD_OK;
}

hsd_status hsd_search_stats(hsd_collection* c, void* stream, int reset, int* stats3) {
  if (!c || !stats3) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  stats3[0] = stats3[1] = stats3[2] = 0;
  int* dv = nullptr;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    auto it = c->scratch.find((cudaStream_t)stream);
    if (it == c->scratch.end()) return HSD_OK;
    dv = it->second.stats;
  }
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  CU(cudaMemcpy(stats3, dv, 3 * sizeof(int), cudaMemcpyDeviceToHost));
  if (reset) CU(cudaMemset(dv, 0, 4 * sizeof(int)));
  return HSD_OK;
}

hsd_status hsd_search_overflow_count(hsd_collection* c, void* stream, int* count) {
  if (!count) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  int v[3];
  hsd_status st = hsd_search_stats(c, stream, 0, v);
  *count = v[0];
  return st;
}

static hsd_status check_verify_params(const hsd_verify_params* params, int P) {
  if (!params || P < 1) return fail(HSD_ERR_INVALID_INPUT, "need at least one parameter set");
  for (int i = 0; i < P; ++i) {
    const hsd_verify_params& p = params[i];
    if (p.bias_seq_max < 0 || p.bias_token_max < 0 || p.bias_token_max > p.bias_seq_max)
      return fail(HSD_ERR_CONFIG, "acceptance caps must satisfy 0 <= bias_token_max <= bias_seq_max (SPEC.md:409)");
    if (p.skip_enabled && p.O_dist < 1) return fail(HSD_ERR_CONFIG, "O_dist must be >= 1 (SPEC.md:413)");
  }
  return HSD_OK;
}

// device copies of parameter arrays, cached per stream
namespace {
struct ParamCache {
  std::mutex mu;
  std::unordered_map<cudaStream_t, std::pair<hsd_verify_params*, std::vector<hsd_verify_params>>> m;
} g_params;

hsd_status device_params(int device, const hsd_verify_params* params, int P, cudaStream_t s,
                         const hsd_verify_params** out) {
  std::lock_guard<std::mutex> lk(g_params.mu);
  auto& ent = g_params.m[s];
  const bool same = ent.second.size() == (size_t)P &&
                    std::memcmp(ent.second.data(), params, sizeof(hsd_verify_params) * P) == 0;
  if (!same) {
    if (ent.second.size() < (size_t)P || !ent.first) {
      if (ent.first) {
        cudaStreamSynchronize(s);
        cudaFree(ent.first);
      }
      ent.first = nullptr;
      CU(cudaMalloc(&ent.first, sizeof(hsd_verify_params) * std::max(P, 16)));
    } else {
      cudaStreamSynchronize(s);  // the previous parameters may still be in use
    }
    CU(cudaMemcpy(ent.first, params, sizeof(hsd_verify_params) * P, cudaMemcpyHostToDevice));
    ent.second.assign(params, params + P);
  }
  (void)device;
  *out = ent.first;
  return HSD_OK;
}
}  // namespace

static hsd_status verify_impl(int device, hsd_collection* c, const uint8_t* drafts, const int32_t* ids, int E, int k,
                              int L, const float* logits, const float* feat_now, const float* feat_prev, int d_f,
                              const int32_t* history, int gap_d, const hsd_verify_params* params, int P,
                              hsd_outcome* out, uint8_t* tokens, void* stream, const double* cos_in = nullptr,
                              const hsd_verify_params* params_dev = nullptr, bool early = false) {
  if (L != 7 && L != 21) return fail(HSD_ERR_INVALID_INPUT, "draft length must be 7 or 21, got %d", L);
  if (k < 1 || k > HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "k must be in [1, %d]", HSD_K_MAX);
  if (E < 0) return fail(HSD_ERR_INVALID_INPUT, "negative episode count");
  hsd_status st = check_verify_params(params, P);
  if (st != HSD_OK) return st;
  if (E == 0) return HSD_OK;
  if (!ids || !logits || !out || !tokens) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  int need_cos = 0;
  for (int i = 0; i < P; ++i) need_cos |= params[i].skip_enabled;
  if (need_cos && (!feat_now || !feat_prev || d_f < 4 || d_f % 4))
    return fail(HSD_ERR_INVALID_INPUT, "verify-skip needs fp32 features with d_f a multiple of 4");
  st = require_device(device);
  if (st != HSD_OK) return st;
  const hsd_verify_params* dp = params_dev;  // an engine's own copy (stream-ordered / per captured graph)
  if (!dp) {
    st = device_params(device, params, P, (cudaStream_t)stream, &dp);
    if (st != HSD_OK) return st;
  }
  CU(hsd::launch_verify(ids, E, k, L, c ? c->tokens : nullptr, drafts, logits, feat_now, feat_prev, d_f, history, gap_d, dp, P,
                        need_cos, out, tokens, (cudaStream_t)stream, cos_in, early));
  return HSD_OK;
}

hsd_status hsd_verify_round(hsd_collection* c, const int32_t* ids, int E, int k, int L, const float* logits,
                            const float* feat_now, const float* feat_prev, int d_f, const int32_t* history, int gap_d,
                            const hsd_verify_params* params, int P, hsd_outcome* out, uint8_t* tokens, void* stream) {
  if (!c) return fail(HSD_ERR_INVALID_INPUT, "null collection");
  return verify_impl(c->device, c, nullptr, ids, E, k, L, logits, feat_now, feat_prev, d_f, history, gap_d, params, P,
                     out, tokens, stream);
}

hsd_status hsd_verify_round_drafts(int device, const int32_t* ids, const uint8_t* drafts, int E, int k, int L,
                                   const float* logits, const float* feat_now, const float* feat_prev, int d_f,
                                   const int32_t* history, int gap_d, const hsd_verify_params* params, int P,
                                   hsd_outcome* out, uint8_t* tokens, void* stream) {
  if (!drafts) return fail(HSD_ERR_INVALID_INPUT, "null drafts");
  return verify_impl(device, nullptr, drafts, ids, E, k, L, logits, feat_now, feat_prev, d_f, history, gap_d, params,
                     P, out, tokens, stream);
}

static hsd_status chains_common(hsd_collection* c, int* device, const int32_t* ids, const uint8_t* drafts, int E,
                                int k, int L, int cap) {
  if (c) *device = c->device;
  if (L != 7 && L != 21) return fail(HSD_ERR_INVALID_INPUT, "draft length must be 7 or 21, got %d", L);
  if (k < 1 || k > HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "k must be in [1, %d]", HSD_K_MAX);
  if (cap < 1 || cap > HSD_K_MAX * HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "chain cap must be in [1, 1024]");
  if (E < 0) return fail(HSD_ERR_INVALID_INPUT, "negative episode count");
  if (E > 0 && !ids) return fail(HSD_ERR_INVALID_INPUT, "null ids");
  if (!c && !drafts) return fail(HSD_ERR_INVALID_INPUT, "need a collection or pre-gathered drafts");
  return require_device(*device);
}

hsd_status hsd_enumerate_chains(hsd_collection* c, int device, const int32_t* ids, const uint8_t* drafts, int E,
                                int k, int L, int cap, int32_t* n_chains, int16_t* chain_ab, uint8_t* chain_tokens,
                                void* stream) {
  hsd_status st = chains_common(c, &device, ids, drafts, E, k, L, cap);
  if (st != HSD_OK || E == 0) return st;
  if (!n_chains || !chain_ab || !chain_tokens) return fail(HSD_ERR_INVALID_INPUT, "null output");
  CU(hsd::launch_enumerate_chains(ids, E, k, L, c ? c->tokens : nullptr, drafts, cap, n_chains, chain_ab,
                                  chain_tokens, (cudaStream_t)stream));
  return HSD_OK;
}

hsd_status hsd_verify_round_chains(hsd_collection* c, int device, const int32_t* ids, const uint8_t* drafts, int E,
                                   int k, int L, int cap, const uint8_t* chain_greedy, const float* chain_logits,
                                   const int32_t* greedy_ctx, const float* feat_now, const float* feat_prev, int d_f,
                                   const int32_t* history, int gap_d, const hsd_verify_params* params,
                                   hsd_outcome* out, uint8_t* tokens, void* stream) {
  hsd_status st = chains_common(c, &device, ids, drafts, E, k, L, cap);
  if (st != HSD_OK) return st;
  st = check_verify_params(params, 1);
  if (st != HSD_OK) return st;
  if ((params->chain_cap > 0 ? params->chain_cap : 64) != cap)
    return fail(HSD_ERR_CONFIG, "params.chain_cap (%d) must equal the enumeration cap (%d)", params->chain_cap, cap);
  if (E == 0) return HSD_OK;
  if (!!chain_greedy == !!chain_logits)
    return fail(HSD_ERR_INVALID_INPUT, "pass exactly one of chain_greedy / chain_logits");
  if (!greedy_ctx || !out || !tokens) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (params->skip_enabled && (!feat_now || !feat_prev || d_f < 4 || d_f % 4))
    return fail(HSD_ERR_INVALID_INPUT, "verify-skip needs fp32 features with d_f a multiple of 4");
  cudaStream_t s = (cudaStream_t)stream;
  const hsd_verify_params* dp = nullptr;
  st = device_params(device, params, 1, s, &dp);
  if (st != HSD_OK) return st;
  uint8_t* g = const_cast<uint8_t*>(chain_greedy);
  if (chain_logits) {  // greedy tokens of every (episode, chain, position), stream-ordered scratch
    const int64_t rows = (int64_t)E * cap * L;
    CU(cudaMallocAsync((void**)&g, (size_t)rows, s));
    cudaError_t e = hsd::launch_chain_argmax(chain_logits, rows, g, s);
    if (e != cudaSuccess) {
      cudaFreeAsync(g, s);
      return cuda_fail(e, "chain_argmax");
    }
  }
  cudaError_t e = hsd::launch_verify_chains(ids, E, k, L, c ? c->tokens : nullptr, drafts, cap, g, greedy_ctx,
                                            feat_now, feat_prev, d_f, history, gap_d, dp, out, tokens, s);
  if (chain_logits) cudaFreeAsync(g, s);
  CU(e);
  return HSD_OK;
}

static hsd_status check_metric(const hsd_metric_params* mp, const hsd_norm_bounds* nb) {
  if (!mp || !nb) return fail(HSD_ERR_INVALID_INPUT, "null parameters");
  // FusedMetricParams::validate (kinematics.cpp:19-24)
  if (!(mp->alpha >= 0.0 && mp->alpha <= 1.0)) return fail(HSD_ERR_CONFIG, "metric.alpha must lie in [0,1]");
  if (mp->w < 3) return fail(HSD_ERR_CONFIG, "metric.window must be >= 3");
  if (mp->w > 32) return fail(HSD_ERR_CONFIG, "metric.window must be <= 32 on the device path");
  if (!(mp->threshold >= 0.0 && mp->threshold <= 1.0)) return fail(HSD_ERR_CONFIG, "metric.threshold must lie in [0,1]");
  if (!(mp->r_cap > 0.0)) return fail(HSD_ERR_CONFIG, "metric.r_cap must be positive");
  // NormalizationBounds::validate (kinematics.cpp:13-17)
  if (!(nb->d_min >= 0.0) || !(nb->r_min >= 0.0)) return fail(HSD_ERR_CONFIG, "normalization bounds must be nonnegative");
  if (nb->d_min > nb->d_max95) return fail(HSD_ERR_CONFIG, "d_min exceeds d_max95");
  if (nb->r_min > nb->r_max95) return fail(HSD_ERR_CONFIG, "r_min exceeds r_max95");
  return HSD_OK;
}

hsd_status hsd_window_features(int device, const double* xyz, int W, const hsd_metric_params* params,
                               const hsd_norm_bounds* bounds, const int32_t* history, double* R, double* D, double* F,
                               int32_t* decision, void* stream) {
  hsd_status st = check_metric(params, bounds);
  if (st != HSD_OK) return st;
  if (W < 0) return fail(HSD_ERR_INVALID_INPUT, "negative window count");
  if (W == 0) return HSD_OK;
  if (!xyz || !R || !D || !F || !decision) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  st = require_device(device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_kinematics(xyz, W, *params, *bounds, history, R, D, F, decision, (cudaStream_t)stream));
  return HSD_OK;
}

hsd_status hsd_window_features_ex(int device, const double* xyz, int W, const hsd_metric_params* params,
                                  const hsd_norm_bounds* bounds, const int32_t* history, double* R, double* D,
                                  double* F, int32_t* decision, double* vaj, void* stream) {
  hsd_status st = check_metric(params, bounds);
  if (st != HSD_OK) return st;
  if (W < 0) return fail(HSD_ERR_INVALID_INPUT, "negative window count");
  if (W == 0) return HSD_OK;
  if (!xyz || !R || !D || !F || !decision) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  st = require_device(device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_kinematics(xyz, W, *params, *bounds, history, R, D, F, decision, (cudaStream_t)stream, vaj));
  return HSD_OK;
}

hsd_status hsd_percentile_bounds(int device, const double* samples, int64_t n, double* min_out, double* p95_out,
                                 void* stream) {
  if (n < 1) return fail(HSD_ERR_INVALID_INPUT, "percentile of empty sample set");  // kinematics.cpp:239
  if (!samples || !min_out || !p95_out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  void* buf = nullptr;  // [2] fp64 result + int non-finite count
  CU(cudaMallocAsync(&buf, 24, s));
  CU(cudaMemsetAsync((uint8_t*)buf + 16, 0, 4, s));
  cudaError_t e = hsd::launch_percentile_bounds(samples, n, (double*)buf, (int*)((uint8_t*)buf + 16), s);
  uint8_t host[24];
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, buf, 24, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(buf, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  CU(e);
  int bad;
  std::memcpy(&bad, host + 16, 4);
  if (bad) return fail(HSD_ERR_INVALID_INPUT, "%d non-finite samples", bad);
  std::memcpy(min_out, host, 8);
  std::memcpy(p95_out, host + 8, 8);
  return HSD_OK;
}

hsd_status hsd_norm_bounds_from_windows(int device, const double* xyz, int W, const hsd_metric_params* params,
                                        hsd_norm_bounds* out, void* stream) {
  if (!out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (W < 1) return fail(HSD_ERR_INVALID_INPUT, "percentile of empty sample set");
  const hsd_norm_bounds unit{0.0, 1.0, 0.0, 1.0};
  hsd_status st = check_metric(params, &unit);
  if (st != HSD_OK) return st;
  st = require_device(device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  double* rd = nullptr;  // R [W], D [W], F [W], decision [W]
  CU(cudaMallocAsync((void**)&rd, (size_t)W * 32, s));
  cudaError_t e = hsd::launch_kinematics(xyz, W, *params, unit, nullptr, rd, rd + W, rd + 2 * W,
                                         (int32_t*)(rd + 3 * W), s);
  if (e != cudaSuccess) {
    cudaFreeAsync(rd, s);
    return cuda_fail(e, "kinematics");
  }
  hsd_norm_bounds b{};
  st = hsd_percentile_bounds(device, rd, W, &b.r_min, &b.r_max95, stream);
  if (st == HSD_OK) st = hsd_percentile_bounds(device, rd + W, W, &b.d_min, &b.d_max95, stream);
  cudaFreeAsync(rd, s);
  if (st != HSD_OK) return st;
  *out = b;
  return HSD_OK;
}

hsd_status hsd_quantize(int device, const double* actions, int64_t n, const double* lo7, const double* hi7, int k_bins,
                        int32_t* bins, int32_t* status, void* stream) {
  if (k_bins < 2) return fail(HSD_ERR_CONFIG, "bin count must be >= 2, got %d", k_bins);  // actions.cpp:28-30
  if (!lo7 || !hi7) return fail(HSD_ERR_INVALID_INPUT, "null bounds");
  for (int i = 0; i < 7; ++i) {  // ActionSpaceBounds::validate (actions.cpp:17-26)
    if (!std::isfinite(lo7[i]) || !std::isfinite(hi7[i]))
      return fail(HSD_ERR_CONFIG, "action bounds must be finite (dim %d)", i);
    if (!(lo7[i] < hi7[i])) return fail(HSD_ERR_CONFIG, "degenerate action bounds on dim %d", i);
  }
  if (n < 0) return fail(HSD_ERR_INVALID_INPUT, "negative count");
  if (n == 0) return HSD_OK;
  if (!actions || !bins) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  double lohi[14];
  std::memcpy(lohi, lo7, 7 * sizeof(double));
  std::memcpy(lohi + 7, hi7, 7 * sizeof(double));
  double* d = nullptr;
  CU(cudaMalloc(&d, sizeof(lohi)));
  cudaError_t e = cudaMemcpy(d, lohi, sizeof(lohi), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = hsd::launch_quantize(actions, n, d, k_bins, bins, status, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "quantize");
  return HSD_OK;
}

// ----------------------------------------------------------------------- engine
}  // extern "C"

// Device staging of one host-buffer step (hsd_step_host[_async]); two slots
// let step i+1's uploads and step i-1's downloads overlap step i's kernels.
struct StageSlot {
  float *q = nullptr, *logits = nullptr, *fnow = nullptr, *fprev = nullptr;
  double* xyz = nullptr;
  int32_t* hist = nullptr;
  double* scores = nullptr;
  int32_t* ids = nullptr;
  hsd_outcome* out = nullptr;
  uint8_t* tok = nullptr;
  double *R = nullptr, *D = nullptr, *F = nullptr;
  int32_t* dec = nullptr;
  cudaEvent_t uploaded = nullptr, computed = nullptr, downloaded = nullptr;
  bool used = false;
};

// A captured decode round (hsd_step_graph): the launch sequence of one
// (shape, buffers, parameters, stream) combination replayed as one graph.
struct StepGraph {
  std::vector<uint8_t> key;
  cudaGraphExec_t exec = nullptr;
  hsd_verify_params* vp = nullptr;  // private device copy of the captured parameters
};

struct hsd_engine {
  hsd_collection* c = nullptr;
  int device = 0;  // the collection's device (destroy never dereferences c: it may be gone)
  int max_B = 0, k = 0, L = 0, d_f = 0, w = 0;
  std::vector<StepGraph> graphs;  // small LRU-less cache (cleared when full)
  StageSlot slot[2];
  int next_slot = 0;
  cudaStream_t up = nullptr, down = nullptr;  // H2D / D2H copy streams
  // stage timing, kStepEvents per step: [0] start, [1] after similarity,
  // [2] after select, [3] end (verify + join), [4]/[5] kinematics on the side stream
  std::vector<cudaEvent_t> ev;
  int max_steps = 0, recorded = 0;
  cudaStream_t side = nullptr;  // K5 and the verify-skip similarity run concurrently with K1
  cudaEvent_t fork = nullptr, join = nullptr;
  double* cos = nullptr;  // [max_B] should_skip similarity, computed on the side stream
  // Fixed device state of the engine's steps: K1/K2 scratch sized for max_B
  // at creation and never reallocated, and the eager steps' parameter copy
  // (updated stream-ordered).  Captured graphs hold these pointers, so one
  // engine issues its steps on one stream at a time.
  Scratch scr;
  hsd_verify_params* vp = nullptr;
  hsd_verify_params vp_last{};  // the values *vp holds (stream-ordered), valid when vp_set
  bool vp_set = false;
  void* vp_stream = nullptr;     // the stream that copied them
};

static constexpr int kStepEvents = 6;

extern "C" {

hsd_status hsd_engine_create(hsd_collection* c, int max_B, int k, int L, int d_f, int w, hsd_engine** out) {
  if (!c || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *out = nullptr;
  if (max_B < 1 || k < 1 || k > HSD_K_MAX || (L != 7 && L != 21) || d_f < 0 || d_f % 4 || w < 3 || w > 32)
    return fail(HSD_ERR_INVALID_INPUT, "bad engine shape");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  auto* e = new hsd_engine();
  e->c = c;
  e->device = c->device;
  e->max_B = max_B;
  e->k = k;
  e->L = L;
  e->d_f = d_f;
  e->w = w;
  cudaError_t r = cudaSuccess;
  auto alloc = [&](auto** p, size_t bytes) {
    if (r == cudaSuccess && bytes) r = cudaMalloc(p, bytes);
  };
  for (StageSlot& S : e->slot) {
    alloc(&S.q, (size_t)max_B * c->dim * 4);
    alloc(&S.logits, (size_t)max_B * L * 256 * 4);
    alloc(&S.fnow, (size_t)max_B * d_f * 4);
    alloc(&S.fprev, (size_t)max_B * d_f * 4);
    alloc(&S.xyz, (size_t)max_B * w * 3 * 8);
    alloc(&S.hist, (size_t)max_B * 4);
    alloc(&S.scores, (size_t)max_B * k * 8);
    alloc(&S.ids, (size_t)max_B * k * 4);
    alloc(&S.out, (size_t)max_B * sizeof(hsd_outcome));
    alloc(&S.tok, (size_t)max_B * L);
    alloc(&S.R, (size_t)max_B * 8);
    alloc(&S.D, (size_t)max_B * 8);
    alloc(&S.F, (size_t)max_B * 8);
    alloc(&S.dec, (size_t)max_B * 4);
    for (cudaEvent_t* ev : {&S.uploaded, &S.computed, &S.downloaded})
      if (r == cudaSuccess) r = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  }
  alloc(&e->cos, (size_t)max_B * 8);
  alloc(&e->vp, sizeof(hsd_verify_params));
  if (r == cudaSuccess) {
    size_t need_p = 0, need_s = 0, need_q = 0;
    scratch_need(max_B, INT64_MAX / 4, num_sms(c->device), c->dim, true, &need_p, &need_s, &need_q);
    if (alloc_scratch(e->scr, need_p, need_s, need_q) != HSD_OK) r = cudaErrorMemoryAllocation;
    e->scr.fixed = true;
  }
  if (r == cudaSuccess) r = cudaStreamCreateWithFlags(&e->up, cudaStreamNonBlocking);
  if (r == cudaSuccess) r = cudaStreamCreateWithFlags(&e->down, cudaStreamNonBlocking);
  if (r != cudaSuccess) {
    hsd_engine_destroy(e);
    return cuda_fail(r, "engine buffers");
  }
  *out = e;
  return HSD_OK;
}

hsd_status hsd_engine_enable_timing(hsd_engine* e, int max_steps) {
  if (!e || max_steps < 0) return fail(HSD_ERR_INVALID_INPUT, "bad arguments");
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  for (cudaEvent_t x : e->ev) cudaEventDestroy(x);
  e->ev.assign((size_t)max_steps * kStepEvents, nullptr);
  for (auto& x : e->ev) CU(cudaEventCreate(&x));
  e->max_steps = max_steps;
  e->recorded = 0;
  return HSD_OK;
}

hsd_status hsd_engine_stage_times(hsd_engine* e, int* n_steps, double* ms) {
  if (!e || !n_steps || !ms) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  for (int i = 0; i < 5; ++i) ms[i] = 0.0;
  for (int s = 0; s < e->recorded; ++s) {
    cudaEvent_t* v = &e->ev[(size_t)s * kStepEvents];
    CU(cudaEventSynchronize(v[3]));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, v[4], v[5]));  // kinematics (side stream, overlapped)
    ms[0] += t;
    CU(cudaEventElapsedTime(&t, v[0], v[1]));  // similarity
    ms[1] += t;
    CU(cudaEventElapsedTime(&t, v[1], v[2]));  // select
    ms[2] += t;
    CU(cudaEventElapsedTime(&t, v[2], v[3]));  // verify (+ join of the side stream)
    ms[3] += t;
    CU(cudaEventElapsedTime(&t, v[0], v[3]));  // step total
    ms[4] += t;
  }
  *n_steps = e->recorded;
  e->recorded = 0;
  return HSD_OK;
}

hsd_status hsd_engine_stage_marks(hsd_engine* e, const hsd_engine* ref, int max_n, double* marks, int* n) {
  if (!e || !ref || !marks || !n) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (ref->recorded < 1) return fail(HSD_ERR_INVALID_INPUT, "reference engine has no recorded step");
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  const int m = std::min(max_n, e->recorded);
  cudaEvent_t r0 = ref->ev[0];
  for (int s = 0; s < m; ++s) {
    const cudaEvent_t* v = &e->ev[(size_t)s * kStepEvents];
    CU(cudaEventSynchronize(v[3]));
    for (int j = 0; j < 4; ++j) {
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, r0, v[j]));
      marks[(size_t)s * 4 + j] = t;
    }
  }
  *n = m;
  return HSD_OK;
}

hsd_status hsd_engine_destroy(hsd_engine* e) {
  if (!e) return HSD_OK;
  cudaSetDevice(e->device);
  for (cudaEvent_t x : e->ev) cudaEventDestroy(x);
  cudaDeviceSynchronize();  // no step still reads the engine's buffers
  cudaFree(e->cos);
  if (e->side) {
    cudaStreamSynchronize(e->side);
    cudaStreamDestroy(e->side);
    cudaEventDestroy(e->fork);
    cudaEventDestroy(e->join);
  }
  if (e->up) cudaStreamSynchronize(e->up);
  if (e->down) cudaStreamSynchronize(e->down);
  for (StageSlot& S : e->slot) {
    void* ps[] = {S.q, S.logits, S.fnow, S.fprev, S.xyz, S.hist, S.scores, S.ids, S.out, S.tok, S.R, S.D, S.F, S.dec};
    for (void* p : ps) cudaFree(p);
    for (cudaEvent_t ev : {S.uploaded, S.computed, S.downloaded})
      if (ev) cudaEventDestroy(ev);
  }
  if (e->up) cudaStreamDestroy(e->up);
  if (e->down) cudaStreamDestroy(e->down);
  for (StepGraph& g : e->graphs) {
    cudaGraphExecDestroy(g.exec);
    cudaFree(g.vp);
  }
  free_scratch(e->scr);
  cudaFree(e->vp);
  delete e;
  cudaGetLastError();  // a destroy leaves no pending error behind
  return HSD_OK;
}

}  // extern "C"

// One decode round on `stream`; vp_dev: the device copy of *vp the verify
// kernel reads (the engine's eager copy, or a captured graph's own).
static hsd_status step_impl(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                            const hsd_verify_params* vp_dev, const hsd_metric_params* mp, const hsd_norm_bounds* nb,
                            int gap_d, void* stream) {
  hsd_status st = HSD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t* ev = (e->recorded < e->max_steps) ? &e->ev[(size_t)e->recorded * kStepEvents] : nullptr;
  if (ev) CU(cudaEventRecord(ev[0], s));
  // K5 (hybrid boundary, decide_sd) and should_skip's similarity do not depend
  // on the retrieval: run them on a side stream so they hide under K1 (K5's
  // Gauss-Newton loop is latency-bound; the similarity would otherwise be a
  // serial feature stream inside K4 after K2).
  // Small batches on the exact scan (K1x, config 1): K4 is launched as K1x's
  // programmatic dependent and runs its feature / logits phases while K1x
  // scans (the similarity in K4 itself), so only the ids -> sweep tail follows
  // the scan; K5 alone takes the side stream, joined after K4.
  static const bool no_early = getenv("HSD_NO_EARLY_VERIFY") != nullptr;  // A/B measurements only
  const bool early = !no_early && B <= hsd::kScanMaxBatch && use_exact_scan(e->c, B, e->k, e->c->n);
  const bool cos_side = !early && vp->skip_enabled && e->d_f > 0 && io->feat_now && io->feat_prev;
  const bool use_side = io->xyz || cos_side;
  if (use_side) {
    if (!e->side) {
      CU(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&e->join, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(e->fork, s));
    CU(cudaStreamWaitEvent(e->side, e->fork, 0));
    if (ev) CU(cudaEventRecord(ev[4], e->side));
    if (cos_side) CU(hsd::launch_cos(io->feat_now, io->feat_prev, B, e->d_f, e->cos, e->side));
    if (io->xyz) {
      st = hsd_window_features(e->c->device, io->xyz, B, mp, nb, io->history, io->R, io->D, io->F, io->decision,
                               e->side);
      if (st != HSD_OK) return st;
    }
    if (ev) CU(cudaEventRecord(ev[5], e->side));
    CU(cudaEventRecord(e->join, e->side));
  }
  StageMarks marks;
  if (ev) {
    marks.after_sim = ev[1];
    marks.after_select = ev[2];
  }
  const int k5_blocks = io->xyz ? (B + 15) / 16 : 0;  // K5 runs 16 windows per CTA
  st = search_impl(e->c, io->queries, B, e->k, 0, e->c->n, io->scores, io->ids, s, ev ? &marks : nullptr,
                   k5_blocks, nullptr, &e->scr);  // K1+K2
  if (st != HSD_OK) return st;
  if (use_side && !early) CU(cudaStreamWaitEvent(s, e->join, 0));
  st = verify_impl(e->c->device, e->c, nullptr, io->ids, B, e->k, e->L, io->logits, io->feat_now, io->feat_prev,
                   e->d_f, io->history, gap_d, vp, 1, io->out, io->tokens, stream, cos_side ? e->cos : nullptr,
                   vp_dev, early);  // K4
  if (st != HSD_OK) return st;
  if (use_side && early) CU(cudaStreamWaitEvent(s, e->join, 0));
  if (ev) {
    if (!use_side) {
      CU(cudaEventRecord(ev[4], s));
      CU(cudaEventRecord(ev[5], s));
    }
    CU(cudaEventRecord(ev[3], s));
    ++e->recorded;
  }
  return HSD_OK;
}

extern "C" {

hsd_status hsd_step(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                    const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream) {
  if (!e || !io || !vp) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (B < 0 || B > e->max_B) return fail(HSD_ERR_INVALID_INPUT, "batch %d outside [0, %d]", B, e->max_B);
  if (B == 0) return HSD_OK;
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  st = check_verify_params(vp, 1);
  if (st != HSD_OK) return st;
  // stream-ordered copy: the previous steps' verify kernels read their own
  // values first.  Unchanged parameters (every step of a run) skip it: a
  // pageable 64-B copy costs ~1.4 us of stream time at config 1.
  // (only on the stream that made the copy: another stream is not ordered after it)
  if (!e->vp_set || e->vp_stream != stream || std::memcmp(&e->vp_last, vp, sizeof *vp) != 0) {
    CU(cudaMemcpyAsync(e->vp, vp, sizeof *vp, cudaMemcpyHostToDevice, (cudaStream_t)stream));
    e->vp_last = *vp;
    e->vp_set = true;
    e->vp_stream = stream;
  }
  return step_impl(e, B, io, vp, e->vp, mp, nb, gap_d, stream);
}

hsd_status hsd_engine_stats(hsd_engine* e, int reset, int* stats3) {
  if (!e || !stats3) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(stats3, e->scr.stats, 3 * sizeof(int), cudaMemcpyDeviceToHost));
  if (reset) CU(cudaMemset(e->scr.stats, 0, 4 * sizeof(int)));
  return HSD_OK;
}

hsd_status hsd_step_graph(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                          const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream) {
  if (!e || !io || !vp) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (B < 0 || B > e->max_B) return fail(HSD_ERR_INVALID_INPUT, "batch %d outside [0, %d]", B, e->max_B);
  if (B == 0) return HSD_OK;
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (!s) return fail(HSD_ERR_INVALID_INPUT, "graph capture needs an explicit (non-legacy) stream");
  // key: everything the captured launches depend on
  std::vector<uint8_t> key;
  auto put = [&](const void* p, size_t n) {
    const uint8_t* b = (const uint8_t*)p;
    key.insert(key.end(), b, b + n);
  };
  put(&B, sizeof B);
  put(io, sizeof *io);
  put(vp, sizeof *vp);
  const hsd_metric_params mpz = mp ? *mp : hsd_metric_params{};
  const hsd_norm_bounds nbz = nb ? *nb : hsd_norm_bounds{};
  put(&mpz, sizeof mpz);
  put(&nbz, sizeof nbz);
  put(&gap_d, sizeof gap_d);
  put(&s, sizeof s);
  const int64_t n = e->c->n;
  put(&n, sizeof n);
  for (StepGraph& g : e->graphs)
    if (g.key == key) {
      CU(cudaGraphLaunch(g.exec, s));
      return HSD_OK;
    }
  // miss: run the round eagerly (warms every per-stream cache), then capture
  // the same launch sequence for the next calls, reading a private copy of
  // the parameters (the engine's scratch is fixed, so the graph's other
  // pointers stay valid)
  const int saved = e->max_steps;
  e->max_steps = 0;  // no stage-timing events inside graphs
  st = hsd_step(e, B, io, vp, mp, nb, gap_d, stream);
  hsd_verify_params* gvp = nullptr;
  if (st == HSD_OK) {
    CU(cudaMalloc(&gvp, sizeof *vp));
    CU(cudaMemcpy(gvp, vp, sizeof *vp, cudaMemcpyHostToDevice));
    cudaGraph_t g = nullptr;
    CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    st = step_impl(e, B, io, vp, gvp, mp, nb, gap_d, stream);
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (st == HSD_OK && ce != cudaSuccess) st = cuda_fail(ce, "cudaStreamEndCapture");
    if (st == HSD_OK) {
      cudaGraphExec_t x = nullptr;
      ce = cudaGraphInstantiate(&x, g, 0);
      if (ce != cudaSuccess) {
        st = cuda_fail(ce, "cudaGraphInstantiate");
      } else {
        if (e->graphs.size() >= 16) {
          CU(cudaStreamSynchronize(s));  // replays of the old graphs may still read their parameters
          for (StepGraph& old : e->graphs) {
            cudaGraphExecDestroy(old.exec);
            cudaFree(old.vp);
          }
          e->graphs.clear();
        }
        e->graphs.push_back({std::move(key), x, gvp});
        gvp = nullptr;
      }
    }
    if (g) cudaGraphDestroy(g);
  }
  if (gvp) cudaFree(gvp);
  e->max_steps = saved;
  return st;
}

hsd_status hsd_step_host_async(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                               const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream) {
  if (!e || !io) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (B < 0 || B > e->max_B) return fail(HSD_ERR_INVALID_INPUT, "batch %d outside [0, %d]", B, e->max_B);
  if (B == 0) return HSD_OK;
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream, up = e->up, down = e->down;
  StageSlot& S = e->slot[e->next_slot];
  e->next_slot ^= 1;
  const int dim = e->c->dim;
  // uploads: the slot's inputs were last read by the kernels of step i-2
  if (S.used) CU(cudaStreamWaitEvent(up, S.computed, 0));
  hsd_step_io d{};
  CU(cudaMemcpyAsync(S.q, io->queries, (size_t)B * dim * 4, cudaMemcpyHostToDevice, up));
  CU(cudaMemcpyAsync(S.logits, io->logits, (size_t)B * e->L * 256 * 4, cudaMemcpyHostToDevice, up));
  d.queries = S.q;
  d.logits = S.logits;
  if (io->feat_now && io->feat_prev && e->d_f) {
    CU(cudaMemcpyAsync(S.fnow, io->feat_now, (size_t)B * e->d_f * 4, cudaMemcpyHostToDevice, up));
    CU(cudaMemcpyAsync(S.fprev, io->feat_prev, (size_t)B * e->d_f * 4, cudaMemcpyHostToDevice, up));
    d.feat_now = S.fnow;
    d.feat_prev = S.fprev;
  }
  if (io->xyz) {
    CU(cudaMemcpyAsync(S.xyz, io->xyz, (size_t)B * e->w * 3 * 8, cudaMemcpyHostToDevice, up));
    d.xyz = S.xyz;
  }
  if (io->history) {
    CU(cudaMemcpyAsync(S.hist, io->history, (size_t)B * 4, cudaMemcpyHostToDevice, up));
    d.history = S.hist;
  }
  CU(cudaEventRecord(S.uploaded, up));
  d.scores = S.scores;
  d.ids = S.ids;
  d.out = S.out;
  d.tokens = S.tok;
  d.R = S.R;
  d.D = S.D;
  d.F = S.F;
  d.decision = S.dec;
  // kernels: after this step's uploads and after step i-2's downloads of the slot's outputs
  CU(cudaStreamWaitEvent(s, S.uploaded, 0));
  if (S.used) CU(cudaStreamWaitEvent(s, S.downloaded, 0));
  st = hsd_step(e, B, &d, vp, mp, nb, gap_d, stream);
  if (st != HSD_OK) return st;
  CU(cudaEventRecord(S.computed, s));
  // downloads overlap the next step's kernels
  CU(cudaStreamWaitEvent(down, S.computed, 0));
  if (io->scores) CU(cudaMemcpyAsync(io->scores, S.scores, (size_t)B * e->k * 8, cudaMemcpyDeviceToHost, down));
  if (io->ids) CU(cudaMemcpyAsync(io->ids, S.ids, (size_t)B * e->k * 4, cudaMemcpyDeviceToHost, down));
  if (io->out) CU(cudaMemcpyAsync(io->out, S.out, (size_t)B * sizeof(hsd_outcome), cudaMemcpyDeviceToHost, down));
  if (io->tokens) CU(cudaMemcpyAsync(io->tokens, S.tok, (size_t)B * e->L, cudaMemcpyDeviceToHost, down));
  if (io->xyz) {
    if (io->R) CU(cudaMemcpyAsync(io->R, S.R, (size_t)B * 8, cudaMemcpyDeviceToHost, down));
    if (io->D) CU(cudaMemcpyAsync(io->D, S.D, (size_t)B * 8, cudaMemcpyDeviceToHost, down));
    if (io->F) CU(cudaMemcpyAsync(io->F, S.F, (size_t)B * 8, cudaMemcpyDeviceToHost, down));
    if (io->decision) CU(cudaMemcpyAsync(io->decision, S.dec, (size_t)B * 4, cudaMemcpyDeviceToHost, down));
  }
  CU(cudaEventRecord(S.downloaded, down));
  S.used = true;
  return HSD_OK;
}

hsd_status hsd_engine_sync(hsd_engine* e) {
  if (!e) return fail(HSD_ERR_INVALID_INPUT, "null engine");
  hsd_status st = require_device(e->c->device);
  if (st != HSD_OK) return st;
  CU(cudaStreamSynchronize(e->down));  // the last download waits for every earlier step
  CU(cudaStreamSynchronize(e->up));
  return HSD_OK;
}

hsd_status hsd_step_host(hsd_engine* e, int B, const hsd_step_io* io, const hsd_verify_params* vp,
                         const hsd_metric_params* mp, const hsd_norm_bounds* nb, int gap_d, void* stream) {
  hsd_status st = hsd_step_host_async(e, B, io, vp, mp, nb, gap_d, stream);
  if (st != HSD_OK) return st;
  return hsd_engine_sync(e);
}

// ------------------------------------------------------------------ multi-GPU
}  // extern "C"

struct hsd_comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  double* gs = nullptr;
  int32_t* gi = nullptr;
  double* ls = nullptr;
  int32_t* li = nullptr;
  uint8_t* gt = nullptr;
  uint8_t* lt = nullptr;
  size_t cap = 0;  // entries per rank
  // peer-memory exchange (hsd_comm_p2p_*): receive window + mapped peers
  void* window = nullptr;
  hsd::P2PWindows win{};
  bool p2p = false;
  uint64_t epoch = 0;
  int* err = nullptr;    // device view of h_err (mapped pinned host memory)
  int* h_err = nullptr;  // set by the merge when a peer never published
};

extern "C" {

hsd_status hsd_comm_unique_id(uint8_t id[HSD_UNIQUE_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == HSD_UNIQUE_ID_BYTES, "NCCL unique id size");
  if (!id) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  ncclUniqueId u;
  NC(ncclGetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return HSD_OK;
}

hsd_status hsd_comm_create(const uint8_t id[HSD_UNIQUE_ID_BYTES], int world, int rank, int device, hsd_comm** out) {
  if (!id || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(HSD_ERR_INVALID_INPUT, "bad rank %d of %d", rank, world);
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  auto* c = new hsd_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HSD_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return HSD_OK;
}

hsd_status hsd_comm_destroy(hsd_comm* c) {
  if (!c) return HSD_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  if (c->comm) ncclCommDestroy(c->comm);
  for (int g = 0; g < c->world && g < hsd::kMaxP2P; ++g)
    if (c->p2p && g != c->rank && c->win.base[g]) cudaIpcCloseMemHandle(c->win.base[g]);
  void* ps[] = {c->gs, c->gi, c->ls, c->li, c->gt, c->lt, c->window};
  for (void* p : ps) cudaFree(p);
  if (c->h_err) cudaFreeHost(c->h_err);
  delete c;
  return HSD_OK;
}

hsd_status hsd_comm_create_p2p(int world, int rank, int device, hsd_comm** out) {
  if (!out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (world < 1 || rank < 0 || rank >= world) return fail(HSD_ERR_INVALID_INPUT, "bad rank %d of %d", rank, world);
  if (world > hsd::kMaxP2P) return fail(HSD_ERR_CONFIG, "peer exchange supports up to %d ranks", hsd::kMaxP2P);
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  auto* c = new hsd_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  *out = c;
  return HSD_OK;
}

hsd_status hsd_comm_p2p_export(hsd_comm* c, int max_B, int k_max, uint8_t handle[HSD_IPC_HANDLE_BYTES]) {
  if (!c || !handle) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (c->world > hsd::kMaxP2P) return fail(HSD_ERR_CONFIG, "peer exchange supports up to %d ranks", hsd::kMaxP2P);
  if (max_B < 1 || k_max < 1 || k_max > HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "bad window shape");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  static_assert(sizeof(cudaIpcMemHandle_t) == HSD_IPC_HANDLE_BYTES, "IPC handle size");
  if (!c->window) {
    const size_t bytes = hsd::p2p_window_bytes(c->world, max_B, k_max, &c->win);
    CU(cudaMalloc(&c->window, bytes));
    CU(cudaMemset(c->window, 0, bytes));  // flags start at epoch 0
    // the merge's timeout flag lives in mapped host memory: the next call reads
    // it without synchronising and fails instead of returning empty results
    CU(cudaHostAlloc((void**)&c->h_err, sizeof(int), cudaHostAllocMapped));
    *(volatile int*)c->h_err = 0;
    CU(cudaHostGetDevicePointer((void**)&c->err, c->h_err, 0));
    c->win.base[c->rank] = c->window;
  }
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, c->window));
  std::memcpy(handle, &h, sizeof h);
  return HSD_OK;
}

hsd_status hsd_comm_p2p_import(hsd_comm* c, const uint8_t* handles) {
  if (!c || !handles) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (!c->window) return fail(HSD_ERR_INVALID_INPUT, "call hsd_comm_p2p_export first");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  for (int g = 0; g < c->world; ++g) {
    if (g == c->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)g * HSD_IPC_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->win.base[g] = p;
  }
  CU(cudaDeviceSynchronize());
  c->p2p = true;
  return HSD_OK;
}

hsd_status hsd_comm_p2p_status(hsd_comm* c, int* peer_timeout) {
  if (!c || !peer_timeout) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *peer_timeout = 0;
  if (!c->h_err) return HSD_OK;
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  *peer_timeout = *(volatile int*)c->h_err;
  return HSD_OK;
}

hsd_status hsd_shard_range(int64_t n_total, int world, int rank, int64_t* begin, int64_t* end) {
  if (!begin || !end) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (world < 1 || rank < 0 || rank >= world || n_total < 0) return fail(HSD_ERR_INVALID_INPUT, "bad shard request");
  const int64_t base = n_total / world, rem = n_total % world;
  *begin = rank * base + std::min<int64_t>(rank, rem);
  *end = *begin + base + (rank < rem ? 1 : 0);
  return HSD_OK;
}

hsd_status hsd_search_topk_sharded(hsd_collection* col, hsd_comm* cm, int64_t id_offset, const float* queries, int B,
                                   int k, double* scores, int32_t* ids, uint8_t* drafts, void* stream) {
  return hsd_search_topk_sharded_ex(col, cm, id_offset, queries, B, k, scores, ids, drafts, 0, stream);
}

hsd_status hsd_search_topk_sharded_ex(hsd_collection* col, hsd_comm* cm, int64_t id_offset, const float* queries,
                                      int B, int k, double* scores, int32_t* ids, uint8_t* drafts, int reserve_sms,
                                      void* stream) {
  if (!col || !cm) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (k < 1 || k > HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "k must be in [1, %d]", HSD_K_MAX);
  if (B <= 0) return B == 0 ? HSD_OK : fail(HSD_ERR_INVALID_INPUT, "negative batch");
  hsd_status st = require_device(col->device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t need = (size_t)B * k;
  if (cm->cap < need) {
    void* ps[] = {cm->gs, cm->gi, cm->ls, cm->li, cm->gt, cm->lt};
    for (void* p : ps) cudaFree(p);
    cm->gs = nullptr;
    cm->gi = nullptr;
    cm->ls = nullptr;
    cm->li = nullptr;
    cm->gt = nullptr;
    cm->lt = nullptr;
    cm->cap = 0;
    CU(cudaMalloc(&cm->gs, need * cm->world * 8));
    CU(cudaMalloc(&cm->gi, need * cm->world * 4));
    CU(cudaMalloc(&cm->gt, need * cm->world * HSD_TOKENS_STRIDE));
    CU(cudaMalloc(&cm->ls, need * 8));
    CU(cudaMalloc(&cm->li, need * 4));
    CU(cudaMalloc(&cm->lt, need * HSD_TOKENS_STRIDE));
    cm->cap = need;
  }
  if (cm->p2p && cm->h_err && *(volatile int*)cm->h_err)  // a previous round's merge timed out
    return fail(HSD_ERR_NCCL, "peer exchange: a peer never published its records (merge timed out); the "
                              "communicator is unusable");
  if (cm->p2p) {  // local top-k whose K2 epilogue publishes into every peer's window, then the merge
    if (B > cm->win.Bmax || k > cm->win.kmax)
      return fail(HSD_ERR_INVALID_INPUT, "batch %d / k %d exceed the peer window (%d, %d)", B, k, cm->win.Bmax,
                  cm->win.kmax);
    ++cm->epoch;
    hsd::P2PPublish pub{};
    pub.w = cm->win;
    pub.rank = cm->rank;
    pub.G = cm->world;
    pub.epoch = cm->epoch;
    pub.id_offset = id_offset;
    pub.tokens = col->tokens;
    st = search_impl(col, queries, B, k, 0, col->n, cm->ls, cm->li, s, nullptr, reserve_sms, &pub);
    if (st != HSD_OK) return st;
    CU(hsd::launch_p2p_merge(cm->win, cm->rank, cm->world, B, k, cm->epoch, scores, ids, drafts, cm->err, s));
    return HSD_OK;
  }
  // local top-k over this rank's shard (K1 + K2), then the 32-B draft record
  st = search_impl(col, queries, B, k, 0, col->n, cm->ls, cm->li, s, nullptr, reserve_sms);
  if (st != HSD_OK) return st;
  CU(hsd::launch_gather_tokens(col->tokens, cm->li, (int)need, cm->lt, s));
  offset_ids_kernel<<<(int)((need + 255) / 256), 256, 0, s>>>(cm->li, (int)need, id_offset);
  CU(cudaGetLastError());
  // K3: exchange the B x k records over NVLink and merge (score desc, id asc)
  if (!cm->comm) return fail(HSD_ERR_INVALID_INPUT, "peer-memory communicator not imported (hsd_comm_p2p_import)");
  NC(ncclGroupStart());
  NC(ncclAllGather(cm->ls, cm->gs, need, ncclFloat64, cm->comm, s));
  NC(ncclAllGather(cm->li, cm->gi, need, ncclInt32, cm->comm, s));
  NC(ncclAllGather(cm->lt, cm->gt, need * HSD_TOKENS_STRIDE, ncclUint8, cm->comm, s));
  NC(ncclGroupEnd());
  CU(hsd::launch_merge_ranks(cm->gs, cm->gi, cm->gt, cm->world, B, k, scores, ids, drafts, s));
  return HSD_OK;
}

hsd_status hsd_merge_topk(int device, const double* g_scores, const int32_t* g_ids, const uint8_t* g_drafts, int G,
                          int B, int k, double* scores, int32_t* ids, uint8_t* drafts, void* stream) {
  if (G < 1 || B < 0 || k < 1 || k > HSD_K_MAX) return fail(HSD_ERR_INVALID_INPUT, "bad merge shape");
  if (!g_scores || !g_ids || !scores || !ids || (drafts && !g_drafts)) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (B == 0) return HSD_OK;
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_merge_ranks(g_scores, g_ids, drafts ? g_drafts : nullptr, G, B, k, scores, ids, drafts,
                             (cudaStream_t)stream));
  return HSD_OK;
}

// ------------------------------------------------------------------ generators
hsd_status hsd_gen_queries(int device, int kind, uint64_t q_seed, uint64_t db_seed, int64_t n_rows, int64_t q0, int B,
                           int dim, float* out, void* stream) {
  if (kind < HSD_SYNTH_EXACT || kind > HSD_SYNTH_CLUSTER) return fail(HSD_ERR_CONFIG, "unknown synthetic family %d", kind);
  if (B < 0 || dim < 1) return fail(HSD_ERR_INVALID_INPUT, "bad shape");
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_gen_queries(kind, q_seed, db_seed, n_rows, q0, B, dim, out, (cudaStream_t)stream));
  return HSD_OK;
}

hsd_status hsd_gen_logits(hsd_collection* c, uint64_t seed, const int64_t* rows, int E, int L, float* out,
                          void* stream) {
  if (!c || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (L < 1 || L > 21) return fail(HSD_ERR_INVALID_INPUT, "bad draft length");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_gen_logits(c->tokens, seed, rows, E, L, out, (cudaStream_t)stream));
  return HSD_OK;
}

hsd_status hsd_gen_features(int device, uint64_t seed, int E, int d_f, float* now, float* prev, void* stream) {
  if (!now || !prev || d_f < 1 || E < 0) return fail(HSD_ERR_INVALID_INPUT, "bad arguments");
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  CU(hsd::launch_gen_features(seed, E, d_f, now, prev, (cudaStream_t)stream));
  return HSD_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ hybrid loop (config 5)
struct hsd_hybrid {
  hsd_collection* c = nullptr;
  int device = 0;  // the collection's device (destroy never dereferences c)
  hsd_comm* comm = nullptr;
  int64_t id_offset = 0, n_total = 0;
  hsd_hybrid_params p{};
  int R = 0, w = 0, max_rounds = 0, round = 0;
  hsd::HybridArgs a{};
  // per-robot state (a.* pointers) + per-round scratch
  double *xyz = nullptr, *Rk = nullptr, *Dk = nullptr, *Fk = nullptr;
  int32_t *histw = nullptr, *dec = nullptr, *modes = nullptr, *slot = nullptr, *ret_idx = nullptr, *drf_idx = nullptr,
          *counts = nullptr, *hist_c = nullptr, *ids = nullptr, *ids_d = nullptr;
  float *q = nullptr, *fnow = nullptr, *fprev = nullptr, *lg_r = nullptr, *lg_d = nullptr;
  double* scores = nullptr;
  uint8_t *drafts = nullptr, *drafts_d = nullptr, *tok_r = nullptr, *tok_d = nullptr;
  hsd_outcome *out_r = nullptr, *out_d = nullptr;
  hsd_step_record* trace = nullptr;
  int32_t* h_counts = nullptr;  // pinned
  int64_t n_ret_queries = 0, n_drf_rounds = 0;
  std::vector<void*> allocs;
  // stage timing: two alternating event sets [start, decided, searched, verified, emitted]
  cudaEvent_t ev[2][5] = {};
  bool pending[2] = {false, false};
  double stage_ms[5] = {0, 0, 0, 0, 0};
  int timed_rounds = 0;
};

static void hybrid_collect(hsd_hybrid* h, int set) {
  if (!h->pending[set]) return;
  float t;
  cudaEvent_t* e = h->ev[set];
  for (int i = 0; i < 4; ++i)
    if (cudaEventElapsedTime(&t, e[i], e[i + 1]) == cudaSuccess) h->stage_ms[i] += t;
  if (cudaEventElapsedTime(&t, e[0], e[4]) == cudaSuccess) h->stage_ms[4] += t;
  h->pending[set] = false;
  ++h->timed_rounds;
}

extern "C" {

hsd_status hsd_hybrid_destroy(hsd_hybrid* h) {
  if (!h) return HSD_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (void* p : h->allocs) cudaFree(p);
  if (h->h_counts) cudaFreeHost(h->h_counts);
  for (auto& set : h->ev)
    for (cudaEvent_t e : set)
      if (e) cudaEventDestroy(e);
  delete h;
  cudaGetLastError();
  return HSD_OK;
}

hsd_status hsd_hybrid_create(hsd_collection* c, hsd_comm* comm, int64_t id_offset, int64_t n_total_rows,
                             const hsd_hybrid_params* p, int max_rounds, hsd_hybrid** out) {
  if (!c || !p || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *out = nullptr;
  if (p->robots < 1 || p->robots > (1 << 20)) return fail(HSD_ERR_CONFIG, "robots must lie in [1, 2^20]");
  if (p->k < 1 || p->k > HSD_K_MAX) return fail(HSD_ERR_CONFIG, "K_top must lie in [1, %d]", HSD_K_MAX);
  if (p->mode < HSD_MODE_HYBRID || p->mode > HSD_MODE_AUTOREGRESSIVE) return fail(HSD_ERR_CONFIG, "unknown mode");
  if (p->traj_T < 1) return fail(HSD_ERR_CONFIG, "traj_T must be >= 1");
  if (p->drafter_L != 7 && p->drafter_L != 21) return fail(HSD_ERR_CONFIG, "drafter L must be 7 or 21");
  if (p->drafter_p_pct < 0 || p->drafter_p_pct > 100) return fail(HSD_ERR_CONFIG, "drafter p must lie in [0, 100]");
  if (p->gap_d < 1) return fail(HSD_ERR_CONFIG, "gap d must be >= 1");
  if (p->d_f < 0 || p->d_f % 4) return fail(HSD_ERR_CONFIG, "d_f must be a nonnegative multiple of 4");
  if (p->verify.skip_enabled && p->d_f == 0) return fail(HSD_ERR_CONFIG, "verify-skip needs d_f > 0");
  if (!(p->cost_verifier >= 0 && p->cost_drafter_token >= 0 && p->cost_retrieval >= 0))
    return fail(HSD_ERR_CONFIG, "cost weights must be >= 0");  // CostModel invariant
  if (max_rounds < 0) return fail(HSD_ERR_INVALID_INPUT, "negative trace capacity");
  hsd_status st = check_metric(&p->metric, &p->bounds);
  if (st != HSD_OK) return st;
  st = check_verify_params(&p->verify, 1);
  if (st != HSD_OK) return st;
  st = require_device(c->device);
  if (st != HSD_OK) return st;
  auto* h = new hsd_hybrid();
  h->c = c;
  h->device = c->device;
  h->comm = comm;
  h->id_offset = id_offset;
  h->n_total = n_total_rows;
  h->p = *p;
  h->R = p->robots;
  h->w = p->metric.w;
  h->max_rounds = p->record_trace ? max_rounds : 0;
  const int R = h->R, w = h->w, k = p->k, L = p->drafter_L, dim = c->dim, d_f = p->d_f;
  cudaError_t e = cudaSuccess;
  auto alloc = [&](auto** ptr, size_t bytes) {
    if (e != cudaSuccess) return;
    e = cudaMalloc(ptr, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) h->allocs.push_back((void*)*ptr);
  };
  hsd::HybridArgs& a = h->a;
  alloc(&a.pos, (size_t)R * 3 * 8);
  alloc(&a.ring, (size_t)R * w * 3 * 8);
  alloc(&a.hist_n, (size_t)R * 4);
  alloc(&a.act, (size_t)R * 8);
  alloc(&a.rounds, (size_t)R * 4);
  alloc(&a.report, (size_t)R * sizeof(hsd_episode_report));
  alloc(&h->xyz, (size_t)R * w * 3 * 8);
  alloc(&h->histw, (size_t)R * 4);
  alloc(&h->Rk, (size_t)R * 8);
  alloc(&h->Dk, (size_t)R * 8);
  alloc(&h->Fk, (size_t)R * 8);
  alloc(&h->dec, (size_t)R * 4);
  alloc(&h->modes, (size_t)R * 4);
  alloc(&h->slot, (size_t)R * 4);
  alloc(&h->ret_idx, (size_t)R * 4);
  alloc(&h->drf_idx, (size_t)R * 4);
  alloc(&h->counts, 8);
  alloc(&h->hist_c, (size_t)R * 4);
  alloc(&h->q, (size_t)R * dim * 4);
  alloc(&h->fnow, (size_t)R * d_f * 4);
  alloc(&h->fprev, (size_t)R * d_f * 4);
  alloc(&h->lg_r, (size_t)R * HSD_HYB_RET_L * 256 * 4);
  alloc(&h->scores, (size_t)R * k * 8);
  alloc(&h->ids, (size_t)R * k * 4);
  alloc(&h->drafts, (size_t)R * k * HSD_TOKENS_STRIDE);
  alloc(&h->out_r, (size_t)R * sizeof(hsd_outcome));
  alloc(&h->tok_r, (size_t)R * HSD_HYB_RET_L);
  alloc(&h->lg_d, (size_t)R * L * 256 * 4);
  alloc(&h->drafts_d, (size_t)R * HSD_TOKENS_STRIDE);
  alloc(&h->ids_d, (size_t)R * 4);
  alloc(&h->out_d, (size_t)R * sizeof(hsd_outcome));
  alloc(&h->tok_d, (size_t)R * L);
  if (h->max_rounds) alloc(&h->trace, (size_t)h->max_rounds * R * sizeof(hsd_step_record));
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_counts, 2 * sizeof(int32_t));
  if (e != cudaSuccess) {
    hsd_hybrid_destroy(h);
    return cuda_fail(e, "hybrid buffers");
  }
  a.R = R;
  a.w = w;
  a.dim = dim;
  a.d_f = d_f;
  a.key_kind = p->key_kind;
  a.traj_T = p->traj_T;
  a.drafter_p_pct = p->drafter_p_pct;
  a.drafter_L = L;
  a.seed = p->seed;
  a.db_seed = p->db_seed;
  a.n_rows = n_total_rows;
  a.n_demo = n_total_rows / p->traj_T;
  a.cost_verifier = p->cost_verifier;
  a.cost_drafter_token = p->cost_drafter_token;
  a.cost_retrieval = p->cost_retrieval;
  for (auto& set : h->ev)
    for (cudaEvent_t& ev : set)
      if (e == cudaSuccess) e = cudaEventCreate(&ev);
  if (e == cudaSuccess) e = hsd::launch_hyb_init(a, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    hsd_hybrid_destroy(h);
    return cuda_fail(e, "hybrid init");
  }
  *out = h;
  return HSD_OK;
}

hsd_status hsd_hybrid_step(hsd_hybrid* h, int n_rounds, void* stream) {
  if (!h) return fail(HSD_ERR_INVALID_INPUT, "null hybrid loop");
  if (n_rounds < 0) return fail(HSD_ERR_INVALID_INPUT, "negative round count");
  hsd_status st = require_device(h->c->device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const hsd_hybrid_params& p = h->p;
  const int R = h->R, k = p.k, L = p.drafter_L;
  hsd_verify_params vp_drf = p.verify;
  vp_drf.skip_enabled = 0;  // verify-skip is retrieval-mode only
  for (int it = 0; it < n_rounds; ++it) {
    const int round = h->round;
    const int set = round & 1;
    cudaEvent_t* ev = h->ev[set];
    CU(cudaEventRecord(ev[0], s));
    // decide_sd for every robot (K5 over the trailing window; cold start -> drafter)
    CU(hsd::launch_hyb_windows(R, h->w, h->a.ring, h->a.hist_n, h->xyz, h->histw, s));
    CU(hsd::launch_kinematics(h->xyz, R, p.metric, p.bounds, h->histw, h->Rk, h->Dk, h->Fk, h->dec, s));
    CU(hsd::launch_hyb_compact(R, p.mode, h->dec, h->modes, h->slot, h->ret_idx, h->drf_idx, h->counts, s));
    CU(cudaMemcpyAsync(h->h_counts, h->counts, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(ev[1], s));
    CU(cudaStreamSynchronize(s));
    hybrid_collect(h, set ^ 1);  // the previous round has completed
    const int nr = h->h_counts[0], nd = h->h_counts[1];
    if (nr == 0) CU(cudaEventRecord(ev[2], s));
    if (nr > 0) {  // retrieval_sd robots: retrieve_drafts -> should_skip -> verify_tree
      CU(hsd::launch_hyb_prep_ret(h->a, round, h->ret_idx, nr, h->q, h->fnow, h->fprev, h->hist_c, s));
      CU(hsd::launch_hyb_logits(h->a, round, h->ret_idx, nr, HSD_HYB_RET_L, h->lg_r, s));
      const float* fn = p.d_f ? h->fnow : nullptr;
      const float* fp = p.d_f ? h->fprev : nullptr;
      if (h->comm) {
        st = hsd_search_topk_sharded(h->c, h->comm, h->id_offset, h->q, nr, k, h->scores, h->ids, h->drafts, s);
        if (st != HSD_OK) return st;
        CU(cudaEventRecord(ev[2], s));
        st = verify_impl(h->c->device, nullptr, h->drafts, h->ids, nr, k, HSD_HYB_RET_L, h->lg_r, fn, fp, p.d_f,
                         h->hist_c, p.gap_d, &p.verify, 1, h->out_r, h->tok_r, s);
      } else {
        st = search_impl(h->c, h->q, nr, k, 0, h->c->n, h->scores, h->ids, s);
        if (st != HSD_OK) return st;
        CU(cudaEventRecord(ev[2], s));
        st = verify_impl(h->c->device, h->c, nullptr, h->ids, nr, k, HSD_HYB_RET_L, h->lg_r, fn, fp, p.d_f, h->hist_c,
                         p.gap_d, &p.verify, 1, h->out_r, h->tok_r, s);
      }
      if (st != HSD_OK) return st;
    }
    if (nd > 0) {  // drafter_sd robots: drafter_generate -> verify (one candidate)
      CU(hsd::launch_hyb_drafts(h->a, round, h->drf_idx, nd, L, h->drafts_d, h->ids_d, s));
      CU(hsd::launch_hyb_logits(h->a, round, h->drf_idx, nd, L, h->lg_d, s));
      st = verify_impl(h->c->device, nullptr, h->drafts_d, h->ids_d, nd, 1, L, h->lg_d, nullptr, nullptr, 0, nullptr,
                       p.gap_d, &vp_drf, 1, h->out_d, h->tok_d, s);
      if (st != HSD_OK) return st;
    }
    CU(cudaEventRecord(ev[3], s));
    hsd_step_record* tr = round < h->max_rounds ? h->trace : nullptr;
    CU(hsd::launch_hyb_emit(h->a, round, h->modes, h->slot, h->out_r, h->tok_r, h->out_d, h->tok_d, h->Fk, tr, s));
    CU(cudaEventRecord(ev[4], s));
    h->pending[set] = true;
    h->n_ret_queries += nr;
    h->n_drf_rounds += nd;
    ++h->round;
  }
  return HSD_OK;
}

hsd_status hsd_hybrid_stage_times(hsd_hybrid* h, int* rounds, double* ms) {
  if (!h || !rounds || !ms) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(h->c->device);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  hybrid_collect(h, 0);
  hybrid_collect(h, 1);
  for (int i = 0; i < 5; ++i) {
    ms[i] = h->stage_ms[i];
    h->stage_ms[i] = 0;
  }
  *rounds = h->timed_rounds;
  h->timed_rounds = 0;
  return HSD_OK;
}

hsd_status hsd_hybrid_positions(hsd_hybrid* h, double* xyz) {
  if (!h || !xyz) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(h->c->device);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(xyz, h->a.pos, (size_t)h->R * 3 * 8, cudaMemcpyDeviceToHost));
  return HSD_OK;
}

hsd_status hsd_hybrid_reports(hsd_hybrid* h, hsd_episode_report* out) {
  if (!h || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(h->c->device);
  if (st != HSD_OK) return st;
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(out, h->a.report, (size_t)h->R * sizeof(hsd_episode_report), cudaMemcpyDeviceToHost));
  return HSD_OK;
}

hsd_status hsd_hybrid_trace(hsd_hybrid* h, hsd_step_record* out, int* rounds) {
  if (!h || !rounds) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(h->c->device);
  if (st != HSD_OK) return st;
  const int n = std::min(h->round, h->max_rounds);
  *rounds = n;
  if (out && n > 0) {
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(out, h->trace, (size_t)n * h->R * sizeof(hsd_step_record), cudaMemcpyDeviceToHost));
  }
  return HSD_OK;
}

hsd_status hsd_hybrid_counts(hsd_hybrid* h, int64_t* retrieval_queries, int64_t* drafter_rounds) {
  if (!h) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (retrieval_queries) *retrieval_queries = h->n_ret_queries;
  if (drafter_rounds) *drafter_rounds = h->n_drf_rounds;
  return HSD_OK;
}

}  // extern "C"

// Error plumbing for the host-only translation units (ingest.cpp): ParseError
// carries its 1-based line (errors.hpp:35-40) in the message and in
// hsd_last_error_line().
hsd_status hsd_internal_fail(hsd_status st, const char* msg, long line) {
  if (line > 0)
    fail(st, "%s (line %ld)", msg, line);
  else
    fail(st, "%s", msg);
  g_err_line = line;
  return st;
}

// ------------------------------------------------------------------ binary device image
// Columnar image of a collection for fast reload:
//   "HSDIMG01" | u32 version=1 | i32 dim | i32 dtype | i32 pad | i64 n | u64 maxnorm bits
//   | keys [n][dim] (fp32 or bf16) | tokens [n][32]
// Streamed through a pinned staging buffer in 64 MB chunks.
namespace {
constexpr char kImgMagic[8] = {'H', 'S', 'D', 'I', 'M', 'G', '0', '1'};
constexpr size_t kImgChunk = 64u << 20;

struct ImgHeader {
  char magic[8];
  uint32_t version;
  int32_t dim, dtype, pad;
  int64_t n;
  unsigned long long maxnorm;
};
static_assert(sizeof(ImgHeader) == 40, "image header layout");

hsd_status img_copy(FILE* f, void* dev, size_t bytes, bool to_file, void* pin) {
  for (size_t off = 0; off < bytes; off += kImgChunk) {
    const size_t m = std::min(kImgChunk, bytes - off);
    if (to_file) {
      CU(cudaMemcpy(pin, (uint8_t*)dev + off, m, cudaMemcpyDeviceToHost));
      if (fwrite(pin, 1, m, f) != m) return fail(HSD_ERR_IO, "image write failed");
    } else {
      if (fread(pin, 1, m, f) != m) return fail(HSD_ERR_PARSE, "truncated image");
      CU(cudaMemcpy((uint8_t*)dev + off, pin, m, cudaMemcpyHostToDevice));
    }
  }
  return HSD_OK;
}
}  // namespace

extern "C" {

hsd_status hsd_collection_save_image(hsd_collection* c, const char* path) {
  if (!c || !path) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  ImgHeader h{};
  std::memcpy(h.magic, kImgMagic, 8);
  h.version = 1;
  h.dim = c->dim;
  h.dtype = c->dtype;
  h.n = c->n;
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(&h.maxnorm, c->maxnorm, 8, cudaMemcpyDeviceToHost));
  FILE* f = fopen(path, "wb");
  if (!f) return fail(HSD_ERR_IO, "cannot open for writing: %s", path);
  void* pin = nullptr;
  cudaError_t e = cudaMallocHost(&pin, kImgChunk);
  if (e != cudaSuccess) {
    fclose(f);
    return cuda_fail(e, "pinned staging");
  }
  st = fwrite(&h, sizeof h, 1, f) == 1 ? HSD_OK : fail(HSD_ERR_IO, "image write failed");
  if (st == HSD_OK) st = img_copy(f, c->keys, (size_t)c->n * c->dim * key_bytes(c), true, pin);
  if (st == HSD_OK) st = img_copy(f, c->tokens, (size_t)c->n * HSD_TOKENS_STRIDE, true, pin);
  cudaFreeHost(pin);
  if (fclose(f) != 0 && st == HSD_OK) st = fail(HSD_ERR_IO, "image close failed");
  return st;
}

hsd_status hsd_collection_load_image(const char* path, int device, hsd_collection** out) {
  if (!path || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *out = nullptr;
  FILE* f = fopen(path, "rb");
  if (!f) return fail(HSD_ERR_IO, "cannot open for reading: %s", path);
  ImgHeader h{};
  if (fread(&h, sizeof h, 1, f) != 1 || std::memcmp(h.magic, kImgMagic, 8) != 0) {
    fclose(f);
    return fail(HSD_ERR_PARSE, "not an hsd device image: %s", path);
  }
  if (h.version != 1) {
    fclose(f);
    return fail(HSD_ERR_VERSION, "unsupported device image version %u", h.version);
  }
  if (h.n < 0) {
    fclose(f);
    return fail(HSD_ERR_PARSE, "corrupt image header");
  }
  hsd_collection* c = nullptr;
  hsd_status st = hsd_collection_create_ex(device, h.dim, std::max<int64_t>(h.n, 1), h.dtype, &c);
  if (st != HSD_OK) {
    fclose(f);
    return st;
  }
  void* pin = nullptr;
  cudaError_t e = cudaMallocHost(&pin, kImgChunk);
  if (e != cudaSuccess) {
    fclose(f);
    hsd_collection_destroy(c);
    return cuda_fail(e, "pinned staging");
  }
  st = img_copy(f, c->keys, (size_t)h.n * h.dim * key_bytes(c), false, pin);
  if (st == HSD_OK) st = img_copy(f, c->tokens, (size_t)h.n * HSD_TOKENS_STRIDE, false, pin);
  cudaFreeHost(pin);
  fclose(f);
  if (st == HSD_OK) {
    cudaError_t e2 = cudaMemcpy(c->maxnorm, &h.maxnorm, 8, cudaMemcpyHostToDevice);
    if (e2 != cudaSuccess) st = cuda_fail(e2, "maxnorm");
  }
  if (st != HSD_OK) {
    hsd_collection_destroy(c);
    return st;
  }
  c->n = h.n;
  *out = c;
  return HSD_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ verify-skip calibration (Alg. 1)
extern "C" {

hsd_status hsd_calibrate_skip(int device, const float* features, int d_f, const int64_t* offsets, int n_traj,
                              double T, double* min_S, int* O_dist, void* stream) {
  if (!features || !offsets || !min_S || !O_dist) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (n_traj < 1) return fail(HSD_ERR_INVALID_INPUT, "need at least one trajectory (SPEC.md:453)");
  if (d_f < 1) return fail(HSD_ERR_INVALID_INPUT, "feature dim must be >= 1");
  if (!std::isfinite(T)) return fail(HSD_ERR_CONFIG, "similarity boundary T must be finite");
  int64_t max_len = 0;
  for (int t = 0; t < n_traj; ++t) {
    if (offsets[t + 1] < offsets[t] || offsets[t] < 0)
      return fail(HSD_ERR_INVALID_INPUT, "trajectory offsets must be nondecreasing");
    max_len = std::max<int64_t>(max_len, offsets[t + 1] - offsets[t]);
  }
  if (max_len >= (1 << 20)) return fail(HSD_ERR_INVALID_INPUT, "trajectories longer than 2^20 points");
  if (n_traj > 65535) return fail(HSD_ERR_INVALID_INPUT, "at most 65535 trajectories per call");
  hsd_status st = require_device(device);
  if (st != HSD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = (int)((max_len + 31) / 32);
  const int max_tiles = nt * (nt + 1) / 2;
  int64_t* doff = nullptr;
  void* scratch = nullptr;
  CU(cudaMalloc(&doff, (size_t)(n_traj + 1) * sizeof(int64_t)));
  cudaError_t e = cudaMalloc(&scratch, hsd::calib_scratch_bytes(n_traj, std::max(max_tiles, 1)));
  int found = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(doff, offsets, (size_t)(n_traj + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = hsd::launch_calibrate(features, d_f, doff, n_traj, (int)max_len, T, scratch, min_S, O_dist, &found, s);
  cudaFree(doff);
  cudaFree(scratch);
  if (e != cudaSuccess) return cuda_fail(e, "calibrate");
  if (!found)  // no pair exceeds T -> calibration failed, skipping stays disabled
    return fail(HSD_ERR_CALIBRATION, "no feature pair exceeds the similarity boundary T = %.17g", T);
  return HSD_OK;
}

hsd_status hsd_update_skip_state(hsd_skip_state* s, int success, double S_c, double min_S_h) {
  if (!s) return fail(HSD_ERR_INVALID_INPUT, "null state");
  // literal Alg. 1 feedback, optional inversion, clamp [T, 1]
  const double adj = s->delta * std::fabs(S_c - min_S_h);
  double sign = success ? 1.0 : -1.0;
  if (s->inverted) sign = -sign;
  s->min_S += sign * adj;
  if (success)
    s->O_dist += 1;
  else
    s->O_dist = s->O_dist - 1 < 1 ? 1 : s->O_dist - 1;
  if (s->min_S < s->T) s->min_S = s->T;
  if (s->min_S > 1.0) s->min_S = 1.0;
  return HSD_OK;
}

}  // extern "C"

// ---- approximate index (IVF-flat; k_ivf.cu) ------------------------------------
// Collection::build_hnsw / search_topk (store.cpp:75-92), SURVEY §8(f) rank 4.

namespace {
struct IvfScratch {
  uint64_t* part = nullptr;  // per-unit top-32 lists (coarse and fine passes share it)
  size_t part_cap = 0;
  uint64_t* pool = nullptr;  // [kMaxBatchPass][32]
  int32_t* probe = nullptr;  // [kMaxBatchPass * 32]
  int32_t* upre = nullptr;   // [kMaxBatchPass * 32 + 1]
  void* sel = nullptr;       // k_select's per-query scratch
  int* stats = nullptr;
};
}  // namespace

struct hsd_index {
  hsd_collection* col = nullptr;  // indexed collection (not owned; destroy never dereferences it)
  int device = 0;
  uint64_t gen = 0;               // the collection's generation at build
  int64_t n = 0;
  int nlist = 0, dim = 0, max_list = 0;
  hsd_collection* cent = nullptr;  // owned: the centroids as an fp32 collection (the build's exact assignment)
  int32_t* offs = nullptr;
  int32_t* perm = nullptr;
  std::mutex mu;
  std::unordered_map<cudaStream_t, IvfScratch> scratch;
};

namespace {

void free_ivf_scratch(IvfScratch& s) {
  cudaFree(s.part);
  cudaFree(s.pool);
  cudaFree(s.probe);
  cudaFree(s.upre);
  cudaFree(s.sel);
  cudaFree(s.stats);
  s = IvfScratch{};
}

// Rows per scan unit: 128, or 32 when 128-row units would leave SMs idle.
int ivf_unit_rows(double units128, int nsm) { return units128 >= 2.0 * nsm ? 128 : 32; }

// Exact assignment of every row to its best centroid (score desc, id asc):
// the collection's own search over the centroid set, rows as queries.
hsd_status ivf_assign(hsd_collection* c, hsd_collection* cent, float* qtmp, int64_t qtmp_rows, double* sc,
                      int32_t* assign) {
  for (int64_t r0 = 0; r0 < c->n; r0 += qtmp_rows) {
    const int64_t m = std::min(qtmp_rows, c->n - r0);
    const float* q = nullptr;
    if (c->dtype == HSD_DTYPE_BF16) {
      CU(hsd::launch_ivf_widen((const uint16_t*)c->keys + (size_t)r0 * c->dim, m * c->dim, qtmp, 0));
      q = qtmp;
    } else {
      q = (const float*)c->keys + (size_t)r0 * c->dim;
    }
    hsd_status st = search_impl(cent, q, (int)m, 1, 0, cent->n, sc, assign + r0, 0);
    if (st != HSD_OK) return st;
  }
  return HSD_OK;
}

hsd_status ivf_set_centroid_rows(hsd_collection* cent) {
  CU(cudaMemsetAsync(cent->maxnorm, 0, sizeof(unsigned long long), 0));
  CU(hsd::launch_row_norms(cent->keys, HSD_DTYPE_F32, 0, cent->n, cent->dim, cent->maxnorm, 0));
  ++cent->gen;
  return HSD_OK;
}

}  // namespace

extern "C" {

hsd_status hsd_index_destroy(hsd_index* x) {
  if (!x) return HSD_OK;
  cudaSetDevice(x->device);
  for (auto& kv : x->scratch) free_ivf_scratch(kv.second);
  cudaFree(x->offs);
  cudaFree(x->perm);
  hsd_collection_destroy(x->cent);
  delete x;
  cudaGetLastError();
  return HSD_OK;
}

hsd_status hsd_index_build(hsd_collection* c, const hsd_ivf_params* p, hsd_index** out) {
  if (!c || !p || !out) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  *out = nullptr;
  if (c->n == 0) return fail(HSD_ERR_INVALID_INPUT, "cannot index an empty collection");  // store.cpp:76
  if (p->nlist < 1 || p->nlist > hsd::kIvfMaxLists)
    return fail(HSD_ERR_CONFIG, "nlist must be in [1, %d], got %d", hsd::kIvfMaxLists, p->nlist);
  if (p->n_iter < 0 || p->n_iter > 1000) return fail(HSD_ERR_CONFIG, "n_iter must be in [0, 1000], got %d", p->n_iter);
  if (c->n > INT32_MAX) return fail(HSD_ERR_CONFIG, "the index addresses at most 2^31 - 1 rows");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  auto* x = new hsd_index();
  x->col = c;
  x->device = c->device;
  x->gen = c->gen;
  x->n = c->n;
  x->dim = c->dim;
  x->nlist = (int)std::min<int64_t>(p->nlist, c->n);
  const int L = x->nlist, dim = c->dim;
  const int64_t n = c->n;
  double* sum = nullptr;
  double* sc = nullptr;
  int32_t* assign = nullptr;
  int32_t* bh = nullptr;
  float* qtmp = nullptr;
  int64_t chunk = 0;
  const int64_t G = hsd::ivf_sort_blocks(n, &chunk);
  const int64_t qrows = std::min<int64_t>(n, 1 << 16);
  auto done = [&](hsd_status r) {
    cudaFree(sum);
    cudaFree(sc);
    cudaFree(assign);
    cudaFree(bh);
    cudaFree(qtmp);
    if (r != HSD_OK) hsd_index_destroy(x);
    return r;
  };
#define IVF_CU(expr)                                     \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return done(cuda_fail(e_, #expr)); \
  } while (0)
  st = hsd_collection_create_ex(c->device, dim, L, HSD_DTYPE_F32, &x->cent);
  if (st != HSD_OK) return done(st);
  IVF_CU(cudaMalloc(&sum, (size_t)L * dim * sizeof(double)));
  IVF_CU(cudaMalloc(&sc, (size_t)qrows * sizeof(double)));
  IVF_CU(cudaMalloc(&assign, (size_t)n * sizeof(int32_t)));
  IVF_CU(cudaMalloc(&bh, (size_t)G * L * sizeof(int32_t)));
  IVF_CU(cudaMalloc(&x->offs, (size_t)(L + 1) * sizeof(int32_t)));
  IVF_CU(cudaMalloc(&x->perm, (size_t)n * sizeof(int32_t)));
  if (c->dtype == HSD_DTYPE_BF16) IVF_CU(cudaMalloc(&qtmp, (size_t)qrows * dim * sizeof(float)));
  float* cent = (float*)x->cent->keys;
  IVF_CU(cudaMemset(cent, 0, (size_t)L * dim * sizeof(float)));
  x->cent->n = L;
  // seeds: one row per stratum, normalized
  IVF_CU(hsd::launch_ivf_seed(c->keys, c->dtype, dim, n, L, sum, 0));
  IVF_CU(hsd::launch_ivf_centroids(nullptr, c->dtype, dim, L, nullptr, nullptr, sum, cent, 0));
  st = ivf_set_centroid_rows(x->cent);
  if (st != HSD_OK) return done(st);
  for (int it = 0; it <= p->n_iter; ++it) {
    st = ivf_assign(c, x->cent, qtmp, qrows, sc, assign);
    if (st != HSD_OK) return done(st);
    IVF_CU(hsd::launch_ivf_sort(assign, n, L, bh, x->offs, x->perm, 0));
    if (it == p->n_iter) break;  // the lists match the final centroids
    IVF_CU(hsd::launch_ivf_centroids(c->keys, c->dtype, dim, L, x->perm, x->offs, sum, cent, 0));
    st = ivf_set_centroid_rows(x->cent);
    if (st != HSD_OK) return done(st);
  }
  std::vector<int32_t> offs(L + 1);
  IVF_CU(cudaMemcpy(offs.data(), x->offs, (L + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int l = 0; l < L; ++l) x->max_list = std::max(x->max_list, offs[l + 1] - offs[l]);
  if (offs[L] != n) return done(fail(HSD_ERR_CUDA, "index build: %d of %lld rows placed", offs[L], (long long)n));
  IVF_CU(cudaDeviceSynchronize());
#undef IVF_CU
  *out = x;
  return done(HSD_OK);
}

hsd_status hsd_index_info(const hsd_index* x, int* nlist, int64_t* n_rows, int* max_list, int* stale) {
  if (!x) return fail(HSD_ERR_INVALID_INPUT, "null index");
  if (nlist) *nlist = x->nlist;
  if (n_rows) *n_rows = x->n;
  if (max_list) *max_list = x->max_list;
  if (stale) *stale = x->gen != x->col->gen;
  return HSD_OK;
}

hsd_status hsd_index_lists(const hsd_index* x, int32_t* offs, int32_t* perm, float* centroids) {
  if (!x) return fail(HSD_ERR_INVALID_INPUT, "null index");
  hsd_status st = require_device(x->col->device);
  if (st != HSD_OK) return st;
  if (offs) CU(cudaMemcpy(offs, x->offs, (x->nlist + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (perm) CU(cudaMemcpy(perm, x->perm, x->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (centroids)
    CU(cudaMemcpy(centroids, x->cent->keys, (size_t)x->nlist * x->dim * sizeof(float), cudaMemcpyDeviceToHost));
  return HSD_OK;
}

hsd_status hsd_search_topk_index(hsd_index* x, const float* queries, int B, int k, int nprobe, double* scores,
                                 int32_t* ids, int32_t* probes, void* stream) {
  if (!x) return fail(HSD_ERR_INVALID_INPUT, "null index");
  hsd_collection* c = x->col;
  cudaStream_t s = (cudaStream_t)stream;
  // an index older than the rows is dropped, as insert drops the HNSW index
  // (store.cpp:44-57): search_topk falls back to the exact search (:83)
  if (x->gen != c->gen) return search_impl(c, queries, B, k, 0, c->n, scores, ids, s);
  if (k < 1) return fail(HSD_ERR_INVALID_INPUT, "k must be >= 1");  // store.cpp:60
  // k > HSD_K_MAX: the exact top-k (the probed-list lists hold 32 entries);
  // the exact answer is also the best one an index can return
  if (k > HSD_K_MAX) return search_impl(c, queries, B, k, 0, c->n, scores, ids, s);
  if (nprobe < 1 || nprobe > 32) return fail(HSD_ERR_INVALID_INPUT, "nprobe must be in [1, 32], got %d", nprobe);
  if (B < 0) return fail(HSD_ERR_INVALID_INPUT, "negative batch");
  if (B == 0) return HSD_OK;
  if (!queries || !scores || !ids) return fail(HSD_ERR_INVALID_INPUT, "null pointer");
  if (reinterpret_cast<uintptr_t>(queries) % 16) return fail(HSD_ERR_INVALID_INPUT, "queries must be 16-byte aligned");
  hsd_status st = require_device(c->device);
  if (st != HSD_OK) return st;
  const int np = std::min(nprobe, x->nlist);
  const int nsm = num_sms(c->device);
  const int W = hsd::kMaxBatchPass;
  const int Bp = std::min(B, W);
  // rows per scoring chunk (ur) and per unit (span), coarse and fine, and the
  // unit bounds of one pass: spans grow so a pass has at most ~kUnitCap units
  // (the per-unit top-32 lists stay small whatever nlist / nprobe / B are)
  const int64_t kUnitCap = std::max<int64_t>(256LL * nsm, (int64_t)Bp * np);
  const int ur_c = ivf_unit_rows((double)Bp * ((x->nlist + 127) / 128), nsm);
  int span_c = ur_c;
  while ((int64_t)Bp * ((x->nlist + span_c - 1) / span_c) > kUnitCap) span_c *= 2;
  const int per_q = (x->nlist + span_c - 1) / span_c;
  const double avg = (double)x->n / x->nlist;
  const int ur_f = ivf_unit_rows((double)Bp * np * std::ceil(avg / 128.0), nsm);
  int span_f = ur_f;
  while ((int64_t)Bp * np * ((x->max_list + span_f - 1) / span_f) > kUnitCap) span_f *= 2;
  const int64_t fine_max = (int64_t)Bp * np * ((x->max_list + span_f - 1) / span_f);
  const int64_t units_max = std::max<int64_t>((int64_t)Bp * per_q, fine_max);
  IvfScratch* sc = nullptr;
  {
    std::lock_guard<std::mutex> lk(x->mu);
    sc = &x->scratch[s];
    if (!sc->pool) {
      CU(cudaMalloc(&sc->pool, (size_t)W * 32 * sizeof(uint64_t)));
      CU(cudaMalloc(&sc->probe, (size_t)W * 32 * sizeof(int32_t)));
      CU(cudaMalloc(&sc->upre, ((size_t)W * 32 + 1) * sizeof(int32_t)));
      CU(cudaMalloc(&sc->sel, hsd::select_scratch_bytes(W)));
      CU(cudaMalloc(&sc->stats, 4 * sizeof(int)));
      CU(cudaMemset(sc->stats, 0, 4 * sizeof(int)));
    }
    const size_t need = hsd::ivf_part_bytes(units_max);
    if (sc->part_cap < need) {
      cudaFree(sc->part);  // implicit synchronisation: no kernel still reads it
      sc->part = nullptr;
      sc->part_cap = 0;
      CU(cudaMalloc(&sc->part, need));
      sc->part_cap = need;
    }
  }
  const int grid = nsm * 8;
  for (int b0 = 0; b0 < B; b0 += W) {
    const int Bs = std::min(W, B - b0);
    const float* q = queries + (size_t)b0 * c->dim;
    hsd::IvfUnits cu{};
    cu.mode = 0;
    cu.ur = ur_c;
    cu.span = span_c;
    cu.per_q = per_q;
    cu.n_q = Bs;
    cu.n_rows = x->nlist;
    CU(hsd::launch_ivf_scan(x->cent->keys, 0, x->dim, nullptr, x->dim, q, cu, (int64_t)Bs * per_q, grid, sc->part, s));
    CU(hsd::launch_ivf_merge(sc->part, cu, Bs, sc->pool, s));
    CU(hsd::launch_ivf_probe(sc->pool, Bs, np, x->offs, span_f, sc->probe, sc->upre, s));
    if (probes) {
      CU(cudaMemcpy2DAsync(probes + (size_t)b0 * nprobe, nprobe * sizeof(int32_t), sc->probe, np * sizeof(int32_t),
                           np * sizeof(int32_t), Bs, cudaMemcpyDeviceToDevice, s));
    }
    hsd::IvfUnits fu{};
    fu.mode = 1;
    fu.ur = ur_f;
    fu.span = span_f;
    fu.n_pairs = Bs * np;
    fu.nprobe = np;
    fu.upre = sc->upre;
    fu.probe = sc->probe;
    fu.offs = x->offs;
    const int64_t fmax = (int64_t)Bs * np * ((x->max_list + span_f - 1) / span_f);
    // the fine scan streams the filter copy when the collection keeps one (half the bytes)
    const void* frows = c->shadow ? (const void*)c->shadow : c->keys;
    const int fbf16 = c->shadow || c->dtype == HSD_DTYPE_BF16;
    CU(hsd::launch_ivf_scan(frows, fbf16, x->dim, x->perm, x->dim, q, fu, fmax, grid, sc->part, s));
    CU(hsd::launch_ivf_merge(sc->part, fu, Bs, sc->pool, s));
    CU(hsd::launch_rescore_pool(sc->pool, 32, Bs, k, c->keys, c->dtype, c->dim, q, scores + (size_t)b0 * k,
                                ids + (size_t)b0 * k, sc->stats, sc->sel, s));
  }
  return HSD_OK;
}

}  // extern "C"

extern "C" int hsd_debug_last_cuda_error(void) { return (int)cudaGetLastError(); }

