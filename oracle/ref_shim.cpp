// ref_shim.cpp — CPU ORACLE (test infrastructure only).
//
// extern "C" entry points over the REFERENCE implementation itself: this file
// is compiled together with the unmodified reference sources
// /root/reference/proj/src/{actions,store,hnsw}.cpp by oracle/Makefile into
// oracle/_ref/libhsdref.so.  No reference source is copied into this repo.
// Used to pin the C restatement (hsd_oracle.c) and as the `--impl reference`
// CPU arm of bench.py.
#include "hsd/actions.hpp"
#include "hsd/errors.hpp"
#include "hsd/store.hpp"

#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "hsd_oracle.h"
#include "hsd_synth.h"

namespace {

int map_exception() {
  try {
    throw;
  } catch (const hsd::InvalidInputError&) {
    return -1;
  } catch (const hsd::ConfigError&) {
    return -2;
  } catch (const hsd::SchemaError&) {
    return -3;
  } catch (const hsd::IoError&) {
    return -4;
  } catch (const hsd::ParseError&) {
    return -5;
  } catch (const hsd::VersionError&) {
    return -6;
  } catch (const hsd::CalibrationError&) {
    return -7;
  } catch (...) {
    return -99;
  }
}

hsd::ActionSpaceBounds bounds_of(const double* lo7, const double* hi7) {
  hsd::ActionSpaceBounds b;
  for (int i = 0; i < hsd::kActionDims; ++i) b.dims[static_cast<size_t>(i)] = {lo7[i], hi7[i]};
  return b;
}

void hit_tokens(const hsd::SearchHit& h, uint8_t* tok21) {
  const auto b = hsd::ActionSpaceBounds::uniform(-1.0, 1.0);
  for (int s = 0; s < 3; ++s) {
    hsd::ActionSlice a;
    for (int j = 0; j < hsd::kActionDims; ++j) a[j] = h.payload.next_actions[static_cast<size_t>(s)][static_cast<size_t>(j)];
    const hsd::ActionBins q = hsd::quantize(a, b, 256);
    for (int j = 0; j < hsd::kActionDims; ++j) tok21[s * 7 + j] = static_cast<uint8_t>(q[j]);
  }
}

}  // namespace

extern "C" {

void* hsdref_collection_new(int dim) {
  try {
    return new hsd::Collection("bench", dim);
  } catch (...) {
    return nullptr;
  }
}

void hsdref_collection_free(void* c) { delete static_cast<hsd::Collection*>(c); }

long hsdref_collection_size(void* c) { return static_cast<long>(static_cast<hsd::Collection*>(c)->size()); }

// Insert n records: embedding = fp32 rows widened to fp64, payload next_actions
// (n x 21 doubles), episode/step indices.
int hsdref_insert(void* c, const float* emb, const double* next_actions, int64_t n, int dim, int episode_idx) {
  auto* col = static_cast<hsd::Collection*>(c);
  try {
    for (int64_t r = 0; r < n; ++r) {
      hsd::Embedding e(static_cast<size_t>(dim));
      for (int i = 0; i < dim; ++i) e[static_cast<size_t>(i)] = emb[r * dim + i];
      hsd::Payload p;
      p.dataset_name = "synthetic";
      p.episode_idx = episode_idx;
      p.step_idx = static_cast<int>(col->size());
      for (int s = 0; s < 3; ++s)
        for (int j = 0; j < 7; ++j)
          p.next_actions[static_cast<size_t>(s)][static_cast<size_t>(j)] = next_actions[r * 21 + s * 7 + j];
      col->insert(std::move(e), std::move(p));
    }
  } catch (...) {
    return map_exception();
  }
  return 0;
}

// Insert rows [row0, row0+n) of a counter-generated DB (include/hsd/hsd_synth.h).
int hsdref_insert_synth(void* c, int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim) {
  std::vector<float> row(static_cast<size_t>(dim));
  std::vector<double> act(21);
  for (int64_t r = 0; r < n; ++r) {
    hsdo_gen_keys(kind, db_seed, row0 + r, 1, dim, row.data());
    for (int s = 0; s < 3; ++s)
      for (int j = 0; j < 7; ++j) act[static_cast<size_t>(s * 7 + j)] = hsd_action_val(db_seed, row0 + r, s, j);
    int rc = hsdref_insert(c, row.data(), act.data(), 1, dim, 0);
    if (rc) return rc;
  }
  return 0;
}

// Same, generating the rows on `threads` host threads (chunks of 2048 rows)
// while the reference's single-writer insert (store.cpp:44-57) appends them
// in order: a full 1M x 4096 Collection builds in seconds, not minutes.
int hsdref_insert_synth_mt(void* c, int kind, uint64_t db_seed, int64_t row0, int64_t n, int dim, int threads) {
  if (threads < 1) threads = 1;
  constexpr int64_t kChunk = 2048;
  std::vector<float> buf[2];
  for (auto& b : buf) b.resize(static_cast<size_t>(kChunk) * dim);
  auto gen = [&](std::vector<float>& b, int64_t r0, int64_t m) {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t]() {
        for (int64_t r = t; r < m; r += threads) hsdo_gen_keys(kind, db_seed, r0 + r, 1, dim, b.data() + r * dim);
      });
    for (auto& th : pool) th.join();
  };
  std::vector<double> act(static_cast<size_t>(kChunk) * 21);
  int64_t m0 = std::min(kChunk, n);
  gen(buf[0], row0, m0);
  for (int64_t c0 = 0, i = 0; c0 < n; c0 += kChunk, ++i) {
    const int64_t m = std::min(kChunk, n - c0);
    std::thread next;
    const int64_t c1 = c0 + kChunk;
    if (c1 < n) next = std::thread([&, c1]() { gen(buf[(i + 1) & 1], row0 + c1, std::min(kChunk, n - c1)); });
    for (int64_t r = 0; r < m; ++r)
      for (int s = 0; s < 3; ++s)
        for (int j = 0; j < 7; ++j) act[static_cast<size_t>(r * 21 + s * 7 + j)] = hsd_action_val(db_seed, row0 + c0 + r, s, j);
    const int rc = hsdref_insert(c, buf[i & 1].data(), act.data(), m, dim, 0);
    if (next.joinable()) next.join();
    if (rc) return rc;
  }
  return 0;
}

// Collection::search_topk_exact (store.cpp:59-73) for one fp64 query; also
// returns the quantized payload tokens (retrieve_drafts).
int hsdref_search(void* c, const double* query, int dim, int k, double* scores, int32_t* ids, uint8_t* tokens) {
  auto* col = static_cast<hsd::Collection*>(c);
  try {
    hsd::Embedding q(query, query + dim);
    auto hits = col->search_topk_exact(q, k);
    for (size_t i = 0; i < hits.size(); ++i) {
      scores[i] = hits[i].score;
      ids[i] = hits[i].record_id;
      if (tokens) hit_tokens(hits[i], tokens + i * 21);
    }
    return static_cast<int>(hits.size());
  } catch (...) {
    return map_exception();
  }
}

// B queries on `threads` host threads, one query per thread at a time (the
// reference has no batch API; concurrent const searches are safe).
int hsdref_search_batch(void* c, const float* queries, int B, int dim, int k, int threads, double* scores,
                        int32_t* ids, uint8_t* tokens) {
  std::atomic<int> next{0};
  std::atomic<int> err{0};
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&]() {
      std::vector<double> q(static_cast<size_t>(dim));
      for (int b = next++; b < B; b = next++) {
        for (int i = 0; i < dim; ++i) q[static_cast<size_t>(i)] = queries[static_cast<size_t>(b) * dim + i];
        int rc = hsdref_search(c, q.data(), dim, k, scores + static_cast<size_t>(b) * k, ids + static_cast<size_t>(b) * k,
                               tokens ? tokens + static_cast<size_t>(b) * k * 21 : nullptr);
        if (rc < 0) err = rc;
      }
    });
  }
  for (auto& th : pool) th.join();
  return err.load();
}

int hsdref_quantize(const double* a7, const double* lo7, const double* hi7, int k_bins, int* bins7) {
  try {
    hsd::ActionSlice a;
    for (int i = 0; i < 7; ++i) a[i] = a7[i];
    auto b = hsd::quantize(a, bounds_of(lo7, hi7), k_bins);
    for (int i = 0; i < 7; ++i) bins7[i] = b[i];
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int hsdref_dequantize(const int* bins7, const double* lo7, const double* hi7, int k_bins, double* a7) {
  try {
    hsd::ActionBins b;
    for (int i = 0; i < 7; ++i) b[i] = bins7[i];
    auto a = hsd::dequantize(b, bounds_of(lo7, hi7), k_bins);
    for (int i = 0; i < 7; ++i) a7[i] = a[i];
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int hsdref_l2_normalize(const double* v, int n, double* out) {
  try {
    auto r = hsd::l2_normalize(std::vector<double>(v, v + n));
    std::memcpy(out, r.data(), sizeof(double) * static_cast<size_t>(n));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

double hsdref_cosine(const double* a, const double* b, int n) {
  return hsd::cosine_similarity(std::vector<double>(a, a + n), std::vector<double>(b, b + n));
}

// ---- persistence (store.cpp:138-191), the reference's own JSONL v1 path ----
// hsdref_load: load_collection(path); returns 0 or the negative status of the
// thrown hsd:: exception (-99 for a non-hsd exception, e.g. nlohmann's), with
// ParseError's line number in *line.  On success *out holds the Collection.
int hsdref_load(const char* path, void** out, long* line) {
  *out = nullptr;
  *line = 0;
  try {
    *out = new hsd::Collection(hsd::load_collection(path));
    return 0;
  } catch (const hsd::ParseError& e) {
    *line = e.line_number;
    return -5;
  } catch (...) {
    return map_exception();
  }
}

int hsdref_save(void* c, const char* path) {
  try {
    hsd::save_collection(*static_cast<hsd::Collection*>(c), path);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int hsdref_dim(void* c) { return static_cast<hsd::Collection*>(c)->dim(); }

// Record r of a loaded collection: embedding [dim], next_actions [21],
// episode/step idx, feature length (-1 = none) and up to feat_cap values.
int hsdref_record(void* c, long r, double* emb, double* next21, int* ep, int* st, double* feat, int feat_cap) {
  const auto& rec = static_cast<hsd::Collection*>(c)->records().at(static_cast<size_t>(r));
  std::memcpy(emb, rec.embedding.data(), rec.embedding.size() * sizeof(double));
  for (int s = 0; s < 3; ++s)
    for (int j = 0; j < 7; ++j) next21[s * 7 + j] = rec.payload.next_actions[static_cast<size_t>(s)][static_cast<size_t>(j)];
  *ep = rec.payload.episode_idx;
  *st = rec.payload.step_idx;
  if (!rec.feature) return -1;
  const int n = static_cast<int>(rec.feature->size());
  for (int i = 0; i < n && i < feat_cap; ++i) feat[i] = (*rec.feature)[static_cast<size_t>(i)];
  return n;
}

}  // extern "C"
