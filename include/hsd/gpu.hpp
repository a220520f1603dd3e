// gpu.hpp — header-only C++20 drop-in for the reference's hot-path API
// (proj/include/hsd), backed by the B200 C ABI in hsd/hsd_gpu.h.
//
// A user of the reference keeps its own headers (hsd/store.hpp,
// hsd/kinematics.hpp, hsd/actions.hpp, hsd/errors.hpp) on the include path and
// swaps
//     hsd::Collection            -> hsd::gpu::Collection
//     hsd::window_features(...)  -> hsd::gpu::window_features(...)
//     hsd::quantize(...)         -> hsd::gpu::quantize(...)
// with the same signatures, value types and exception taxonomy (errors.hpp);
// batched variants are added for the GPU.  The verification ops, spec-only in
// the reference, are exposed as hsd::gpu::Verifier.
//
// Numerics: the device stores keys as fp32.  search_topk_exact returns, bit
// for bit, what store.cpp:59-73 returns for the fp32-rounded embeddings and
// query (the fp64 scores are the reference's sequential dot of the widened
// values); inputs that are already fp32-representable (the usual case: model
// activations) are therefore bit-identical end to end.  Any dim >= 1 is
// accepted: rows are zero-padded to a multiple of 8 on the device, and the
// trailing fma(0, 0, s) steps leave the sequential sum's bits unchanged (s
// starts at +0.0 and a sum of an +0.0 product never produces -0.0).  See
// INTEGRATION.md.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "hsd/actions.hpp"
#include "hsd/errors.hpp"
#include "hsd/hsd_gpu.h"
#include "hsd/kinematics.hpp"
#include "hsd/store.hpp"

namespace hsd::gpu {

// ---------------------------------------------------------------- errors
[[noreturn]] inline void throw_status(hsd_status st) {
  const std::string m = hsd_last_error();
  switch (st) {
    case HSD_ERR_INVALID_INPUT: throw InvalidInputError(m);
    case HSD_ERR_CONFIG: throw ConfigError(m);
    case HSD_ERR_SCHEMA: throw SchemaError(m);
    case HSD_ERR_IO: throw IoError(m);
    case HSD_ERR_PARSE: throw ParseError(m);
    case HSD_ERR_VERSION: throw VersionError(m);
    case HSD_ERR_CALIBRATION: throw CalibrationError(m);
    default: throw Error(m);  // CUDA / NCCL / OOM / no device
  }
}
inline void check(hsd_status st) {
  if (st != HSD_OK) throw_status(st);
}

// ---------------------------------------------------------------- device buffer
template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) { resize(n); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  ~DeviceBuffer() { cudaFree(p_); }
  void resize(size_t n) {
    if (n <= n_) return;
    cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
    if (cudaMalloc(&p_, n * sizeof(T)) != cudaSuccess) throw Error("cudaMalloc failed");
    n_ = n;
  }
  T* get() const { return p_; }
  void upload(const T* h, size_t n, cudaStream_t s = nullptr) {
    resize(n);
    if (n && cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s) != cudaSuccess) throw Error("H2D failed");
  }
  void download(T* h, size_t n, cudaStream_t s = nullptr) const {
    if (n && cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s) != cudaSuccess) throw Error("D2H failed");
    if (cudaStreamSynchronize(s) != cudaSuccess) throw Error("stream sync failed");
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// ---------------------------------------------------------------- Collection
// Same surface as hsd::Collection (store.hpp:59-96); records' payloads stay on
// the host (SearchHit carries them), keys and quantized payload tokens live in
// HBM.
class Collection {
 public:
  Collection() = default;
  Collection(std::string name, int dim, int device = 0, int64_t capacity = 1024)
      : name_(std::move(name)), dim_(dim), pdim_((dim + 7) / 8 * 8) {
    if (dim < 1) throw ConfigError("collection dim must be >= 1");  // store.cpp:37
    check(hsd_collection_create(device, pdim_, capacity, &h_));
    device_ = device;
  }
  Collection(Collection&& o) noexcept { *this = std::move(o); }
  Collection& operator=(Collection&& o) noexcept {
    std::swap(name_, o.name_);
    std::swap(dim_, o.dim_);
    std::swap(pdim_, o.pdim_);
    std::swap(device_, o.device_);
    std::swap(h_, o.h_);
    std::swap(index_, o.index_);
    std::swap(nprobe_, o.nprobe_);
    std::swap(records_, o.records_);
    std::swap(q_, o.q_);
    std::swap(s_, o.s_);
    std::swap(i_, o.i_);
    return *this;
  }
  ~Collection() {
    drop_index();
    hsd_collection_destroy(h_);
  }

  // Upload an existing reference collection (e.g. one built by load_collection).
  static Collection from(const hsd::Collection& c, int device = 0) {
    Collection g(c.name(), c.dim(), device, (int64_t)std::max<size_t>(c.size(), 1));
    g.insert_batch(c.records());
    return g;
  }

  const std::string& name() const { return name_; }
  int dim() const { return dim_; }
  size_t size() const { return records_.size(); }
  bool empty() const { return records_.empty(); }
  const Record& record(int id) const { return records_[static_cast<size_t>(id)]; }
  const std::vector<Record>& records() const { return records_; }
  hsd_collection* handle() const { return h_; }

  // Collection::insert (store.cpp:44-57): SchemaError on a dim mismatch or
  // negative payload indices; returns the dense record id.
  int insert(Embedding embedding, Payload payload, std::optional<std::vector<double>> feature = std::nullopt) {
    std::vector<Record> one;
    one.push_back({std::move(embedding), std::move(payload), std::move(feature)});
    return insert_batch(one);
  }

  // Bulk insert; returns the id of the first record.
  int insert_batch(const std::vector<Record>& recs) {
    const int64_t n = (int64_t)recs.size();
    std::vector<float> emb((size_t)n * pdim_, 0.0f);
    std::vector<double> act((size_t)n * 21);
    std::vector<int32_t> ep((size_t)n), st((size_t)n);
    int d_f = 0;
    for (int64_t i = 0; i < n; ++i) {
      const Record& r = recs[(size_t)i];
      if ((int)r.embedding.size() != dim_)
        throw SchemaError("embedding dim " + std::to_string(r.embedding.size()) + " does not match collection dim " +
                          std::to_string(dim_));
      for (int c = 0; c < dim_; ++c) emb[(size_t)i * pdim_ + c] = (float)r.embedding[(size_t)c];
      for (int s = 0; s < 3; ++s)
        for (int j = 0; j < 7; ++j) act[(size_t)i * 21 + s * 7 + j] = r.payload.next_actions[(size_t)s][(size_t)j];
      ep[(size_t)i] = r.payload.episode_idx;
      st[(size_t)i] = r.payload.step_idx;
      if (r.feature && !d_f) d_f = (int)r.feature->size();
    }
    int64_t first = 0;
    check(hsd_collection_insert(h_, emb.data(), act.data(), ep.data(), st.data(), n, &first));
    if (n) drop_index();  // stale after mutation (store.cpp:55)
    if (d_f) {  // Record::feature -> the device feature table (feeds calibrate_skip)
      std::vector<float> f((size_t)n * d_f, 0.0f);
      std::vector<uint8_t> has((size_t)n, 0);
      for (int64_t i = 0; i < n; ++i) {
        const auto& rf = recs[(size_t)i].feature;
        if (!rf) continue;
        if ((int)rf->size() != d_f) throw SchemaError("feature length differs from the collection's first feature");
        for (int c = 0; c < d_f; ++c) f[(size_t)i * d_f + c] = (float)(*rf)[(size_t)c];
        has[(size_t)i] = 1;
      }
      check(hsd_collection_set_features(h_, first, n, d_f, f.data(), has.data()));
    }
    records_.insert(records_.end(), recs.begin(), recs.end());
    return (int)first;
  }

  // offline_calibrate_skip over the collection's own
  // recorded features: a trajectory is a run of consecutive records with one
  // episode_idx (records without a feature stand alone and add no pair).
  // Returns (min_S, O_dist); CalibrationError when no pair exceeds T.
  std::pair<double, int> calibrate_skip(double T) const {
    const float* feat = nullptr;
    int d_f = 0;
    check(hsd_collection_features(h_, &feat, nullptr, &d_f));
    if (!d_f) throw CalibrationError("no record carries a verifier feature");
    std::vector<int64_t> off{0};
    for (size_t i = 1; i < records_.size(); ++i)
      if (records_[i].payload.episode_idx != records_[i - 1].payload.episode_idx || !records_[i].feature ||
          !records_[i - 1].feature)
        off.push_back((int64_t)i);
    off.push_back((int64_t)records_.size());
    double best = INFINITY;
    int best_d = 0;
    bool found = false;
    for (size_t t0 = 0; t0 + 1 < off.size(); t0 += 65535) {  // hsd_calibrate_skip's batch limit
      const size_t nt = std::min<size_t>(65535, off.size() - 1 - t0);
      std::vector<int64_t> o(off.begin() + (long)t0, off.begin() + (long)(t0 + nt + 1));
      const int64_t base = o.front();
      for (auto& v : o) v -= base;
      double m = 0.0;
      int d = 0;
      const hsd_status st =
          hsd_calibrate_skip(device_, feat + (size_t)base * d_f, d_f, o.data(), (int)nt, T, &m, &d, nullptr);
      if (st == HSD_ERR_CALIBRATION) continue;
      check(st);
      if (!found || m < best) {  // first strict minimum in trajectory order
        best = m;
        best_d = d;
        found = true;
      }
    }
    if (!found) throw CalibrationError("no feature pair exceeds the similarity boundary T");
    return {best, best_d};
  }

  // Collection::search_topk_exact (store.cpp:59-73).
  std::vector<SearchHit> search_topk_exact(const Embedding& query, int k) const {
    return search_topk_exact_batch(std::vector<Embedding>{query}, k).front();
  }
  // Collection::build_hnsw (store.cpp:75-80): the device's approximate index
  // is an inverted file (IVF-flat, hsd_index_*), not a graph.  HnswParams map
  // to it as  nlist = ceil(sqrt(N)) (<= 16384),  Lloyd iterations =
  // clamp(ef_construct / 10, 1, 20),  nprobe = clamp(ef_search / 4, 1, 32);
  // m (graph degree) has no IVF meaning.
  void build_hnsw(const HnswParams& params) {
    if (records_.empty()) throw InvalidInputError("cannot index an empty collection");  // store.cpp:76
    if (params.m < 2 || params.ef_construct < 1) throw ConfigError("invalid hnsw parameters");  // hnsw.cpp:42
    drop_index();
    const double n = (double)records_.size();
    hsd_ivf_params p{(int)std::min(16384.0, std::ceil(std::sqrt(n))), std::clamp(params.ef_construct / 10, 1, 20)};
    check(hsd_index_build(h_, &p, &index_));
    nprobe_ = std::clamp(params.ef_search / 4, 1, 32);
  }
  bool has_hnsw() const { return index_ != nullptr; }

  // Collection::search_topk (store.cpp:82-92): the index when built (the
  // returned scores are still cosine_similarity of the returned ids, :86-90),
  // else the exact search.
  std::vector<SearchHit> search_topk(const Embedding& query, int k) const {
    if (!index_) return search_topk_exact(query, k);
    if (k < 1) return {};  // HnswIndex::search returns no ids (hnsw.cpp:160)
    if ((int)query.size() != dim_) throw InvalidInputError("embedding dim mismatch in cosine");
    std::vector<float> q((size_t)pdim_, 0.0f);
    for (int c = 0; c < dim_; ++c) q[(size_t)c] = (float)query[(size_t)c];
    s_.resize((size_t)k);
    i_.resize((size_t)k);
    q_.upload(q.data(), q.size());
    check(hsd_search_topk_index(index_, q_.get(), 1, k, nprobe_, s_.get(), i_.get(), nullptr, nullptr));
    std::vector<double> sc((size_t)k);
    std::vector<int32_t> id((size_t)k);
    s_.download(sc.data(), sc.size());
    i_.download(id.data(), id.size());
    std::vector<SearchHit> out;
    for (int j = 0; j < k && id[(size_t)j] >= 0; ++j)
      out.push_back({sc[(size_t)j], id[(size_t)j], records_[(size_t)id[(size_t)j]].payload});
    return out;
  }

  // Batched search: one pass over the DB for all queries.
  std::vector<std::vector<SearchHit>> search_topk_exact_batch(const std::vector<Embedding>& queries, int k) const {
    if (k < 1) throw InvalidInputError("k must be >= 1");  // store.cpp:60
    const int B = (int)queries.size();
    std::vector<std::vector<SearchHit>> out((size_t)B);
    if (records_.empty() || B == 0) return out;  // empty collection -> empty result
    std::vector<float> q((size_t)B * pdim_, 0.0f);
    for (int b = 0; b < B; ++b) {
      if ((int)queries[(size_t)b].size() != dim_) throw InvalidInputError("embedding dim mismatch in cosine");
      for (int c = 0; c < dim_; ++c) q[(size_t)b * pdim_ + c] = (float)queries[(size_t)b][(size_t)c];
    }
    // device buffers persist across calls (grown on demand): no allocation per query
    s_.resize((size_t)B * k);
    i_.resize((size_t)B * k);
    q_.upload(q.data(), q.size());
    check(hsd_search_topk_exact(h_, q_.get(), B, k, s_.get(), i_.get(), nullptr));
    std::vector<double> sc((size_t)B * k);
    std::vector<int32_t> id((size_t)B * k);
    s_.download(sc.data(), sc.size());
    i_.download(id.data(), id.size());
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < k; ++j) {
        const int32_t r = id[(size_t)b * k + j];
        if (r < 0) break;
        out[(size_t)b].push_back({sc[(size_t)b * k + j], r, records_[(size_t)r].payload});
      }
    return out;
  }

 private:
  void drop_index() {
    hsd_index_destroy(index_);
    index_ = nullptr;
  }

  std::string name_;
  int dim_ = 0;
  int pdim_ = 0;  // device row length: dim rounded up to 8 (zero padding)
  int device_ = 0;
  hsd_collection* h_ = nullptr;
  hsd_index* index_ = nullptr;  // approximate index (build_hnsw), dropped on insert
  int nprobe_ = 25;
  std::vector<Record> records_;
  mutable DeviceBuffer<float> q_;
  mutable DeviceBuffer<double> s_;
  mutable DeviceBuffer<int32_t> i_;
};

// ---------------------------------------------------------------- kinematics
inline hsd_metric_params to_c(const FusedMetricParams& p) { return {p.alpha, p.w, p.threshold, p.r_cap}; }
inline hsd_norm_bounds to_c(const NormalizationBounds& b) { return {b.d_min, b.d_max95, b.r_min, b.r_max95}; }

// Batched window_features (kinematics.cpp:261-273) over windows of exactly
// params.w points; decisions[i] = classify_segment(F_i, params.threshold).
inline std::vector<WindowFeatures> window_features_batch(const std::vector<std::vector<TrajectoryPoint>>& windows,
                                                         const FusedMetricParams& params,
                                                         const NormalizationBounds& bounds,
                                                         std::vector<SdKind>* decisions = nullptr, int device = 0) {
  // FusedMetricParams/NormalizationBounds::validate (kinematics.cpp:13-24) are
  // applied by hsd_window_features (ConfigError) — their definitions live in
  // kinematics.cpp, which this header does not require.
  const int W = (int)windows.size();
  std::vector<WindowFeatures> out((size_t)W);
  if (W == 0) return out;
  std::vector<double> xyz((size_t)W * params.w * 3);
  for (int i = 0; i < W; ++i) {
    if ((int)windows[(size_t)i].size() != params.w) throw InvalidInputError("window_features expects exactly w points");
    for (int p = 0; p < params.w; ++p) {
      const TrajectoryPoint& t = windows[(size_t)i][(size_t)p];
      xyz[((size_t)i * params.w + p) * 3 + 0] = t.x;
      xyz[((size_t)i * params.w + p) * 3 + 1] = t.y;
      xyz[((size_t)i * params.w + p) * 3 + 2] = t.z;
    }
  }
  DeviceBuffer<double> dx, dR((size_t)W), dD((size_t)W), dF((size_t)W);
  DeviceBuffer<int32_t> dd((size_t)W);
  dx.upload(xyz.data(), xyz.size());
  const hsd_metric_params mp = to_c(params);
  const hsd_norm_bounds nb = to_c(bounds);
  check(hsd_window_features(device, dx.get(), W, &mp, &nb, nullptr, dR.get(), dD.get(), dF.get(), dd.get(), nullptr));
  std::vector<double> R((size_t)W), D((size_t)W), F((size_t)W);
  std::vector<int32_t> dec((size_t)W);
  dR.download(R.data(), R.size());
  dD.download(D.data(), D.size());
  dF.download(F.data(), F.size());
  dd.download(dec.data(), dec.size());
  if (decisions) decisions->resize((size_t)W);
  for (int i = 0; i < W; ++i) {
    if (dec[(size_t)i] < 0) throw InvalidInputError("non-finite trajectory point");  // kinematics.cpp:29-35
    out[(size_t)i] = {R[(size_t)i], D[(size_t)i], F[(size_t)i], params.w};
    if (decisions) (*decisions)[(size_t)i] = dec[(size_t)i] ? SdKind::retrieval_sd : SdKind::drafter_sd;
  }
  return out;
}

// window_features (kinematics.hpp:91-93), same signature.
inline WindowFeatures window_features(std::span<const TrajectoryPoint> points, const FusedMetricParams& params,
                                      const NormalizationBounds& bounds) {
  return window_features_batch({std::vector<TrajectoryPoint>(points.begin(), points.end())}, params, bounds).front();
}

// ---------------------------------------------------------------- actions
// quantize (actions.hpp:55), batched on the device with the reference formula.
inline std::vector<ActionBins> quantize_batch(const std::vector<ActionSlice>& a, const ActionSpaceBounds& bounds,
                                              int k_bins, int device = 0) {
  double lo[7], hi[7];
  for (int i = 0; i < 7; ++i) {
    lo[i] = bounds.dims[(size_t)i].lo;
    hi[i] = bounds.dims[(size_t)i].hi;
  }
  const int64_t n = (int64_t)a.size();
  std::vector<ActionBins> out((size_t)n);
  std::vector<double> h((size_t)n * 7);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < 7; ++j) h[(size_t)i * 7 + j] = a[(size_t)i][j];
  DeviceBuffer<double> da;
  DeviceBuffer<int32_t> db((size_t)std::max<int64_t>(n, 1) * 7), dst((size_t)std::max<int64_t>(n, 1));
  da.upload(h.data(), h.size());
  check(hsd_quantize(device, da.get(), n, lo, hi, k_bins, db.get(), dst.get(), nullptr));
  std::vector<int32_t> bins((size_t)n * 7), st((size_t)n);
  db.download(bins.data(), bins.size());
  dst.download(st.data(), st.size());
  for (int64_t i = 0; i < n; ++i) {
    if (st[(size_t)i]) throw InvalidInputError("non-finite action value");  // actions.cpp:38-40
    for (int j = 0; j < 7; ++j) out[(size_t)i][j] = bins[(size_t)i * 7 + j];
  }
  return out;
}
inline ActionBins quantize(const ActionSlice& a, const ActionSpaceBounds& bounds, int k_bins) {
  return quantize_batch({a}, bounds, k_bins).front();
}

// ---------------------------------------------------------------- verification
// Spec-only in the reference.  One decode round per episode:
// retrieved ids [E][k] -> VerifyOutcome-like results.
struct VerifyOutcome {
  std::vector<int> accepted_tokens;
  int accept_length = 0;
  int verifier_calls = 0;
  bool skipped = false;
  bool fallback_used = false;
};

class Verifier {
 public:
  Verifier(const Collection& c, int draft_len, hsd_verify_params params) : c_(&c), L_(draft_len), p_(params) {}

  // ids [E][k] (rank order, -1 padded), logits [E][L][256], optional features
  // [E][d_f] now/prev for should_skip; all host arrays.
  std::vector<VerifyOutcome> verify(const std::vector<int32_t>& ids, int E, int k, const std::vector<float>& logits,
                                    const float* feat_now = nullptr, const float* feat_prev = nullptr, int d_f = 0,
                                    int gap_d = 1) const {
    DeviceBuffer<int32_t> di;
    DeviceBuffer<float> dl, dn, dp;
    di.upload(ids.data(), (size_t)E * k);
    dl.upload(logits.data(), (size_t)E * L_ * 256);
    if (feat_now && feat_prev) {
      dn.upload(feat_now, (size_t)E * d_f);
      dp.upload(feat_prev, (size_t)E * d_f);
    }
    DeviceBuffer<hsd_outcome> dout((size_t)std::max(E, 1));
    DeviceBuffer<uint8_t> dtok((size_t)std::max(E, 1) * L_);
    check(hsd_verify_round(c_->handle(), di.get(), E, k, L_, dl.get(), dn.get(), dp.get(), d_f, nullptr, gap_d, &p_, 1,
                           dout.get(), dtok.get(), nullptr));
    std::vector<hsd_outcome> o((size_t)E);
    std::vector<uint8_t> tok((size_t)E * L_);
    dout.download(o.data(), o.size());
    dtok.download(tok.data(), tok.size());
    std::vector<VerifyOutcome> res((size_t)E);
    for (int e = 0; e < E; ++e) {
      VerifyOutcome& r = res[(size_t)e];
      r.accept_length = o[(size_t)e].accept_len;
      r.verifier_calls = o[(size_t)e].calls;
      r.skipped = o[(size_t)e].skipped != 0;
      r.fallback_used = o[(size_t)e].fallback != 0;
      for (int t = 0; t < o[(size_t)e].n_emit; ++t) r.accepted_tokens.push_back(tok[(size_t)e * L_ + t]);
    }
    return res;
  }

 private:
  const Collection* c_;
  int L_;
  hsd_verify_params p_;
};

}  // namespace hsd::gpu
