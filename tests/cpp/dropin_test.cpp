// dropin_test.cpp — the reference's own C++ API next to the drop-in.
//
// Builds a reference hsd::Collection (store.cpp, compiled in place into
// oracle/_ref/libhsdref.so), uploads it with hsd::gpu::Collection::from, and
// checks that search_topk_exact returns identical SearchHits (score bits,
// record ids, payloads), that hsd::gpu::quantize matches hsd::quantize, that
// hsd::gpu::window_features matches the oracle restatement within 1e-5, and
// that errors surface as the reference's exception types.
// Built by tests/cpp/Makefile (needs /root/reference headers), run on the GPU
// box by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "hsd/gpu.hpp"

extern "C" {
#include "hsd_oracle.h"
}
#include "hsd_synth.h"

static int failures = 0;
#define CHECK(cond, ...)              \
  do {                                \
    if (!(cond)) {                    \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");              \
      ++failures;                     \
    }                                 \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  const int dim = 256, n = 5000, B = 40, k = 8;
  // ---- reference collection with synthetic records
  hsd::Collection ref("dropin", dim);
  std::vector<float> row((size_t)dim);
  for (int r = 0; r < n; ++r) {
    hsdo_gen_keys(HSD_SYNTH_REAL, 77, r, 1, dim, row.data());
    hsd::Payload p;
    p.dataset_name = "synthetic";
    p.episode_idx = r / 100;
    p.step_idx = r % 100;
    for (int s = 0; s < 3; ++s)
      for (int j = 0; j < 7; ++j) p.next_actions[(size_t)s][(size_t)j] = hsd_action_val(77, r, s, j);
    ref.insert(hsd::Embedding(row.begin(), row.end()), p);
  }
  hsd::gpu::Collection gpu = hsd::gpu::Collection::from(ref, 0);
  CHECK(gpu.size() == ref.size(), "size");

  // ---- search parity (single and batched)
  std::vector<float> q((size_t)B * dim);
  hsdo_gen_queries(HSD_SYNTH_REAL, 78, 77, n, 0, B, dim, q.data());
  std::vector<hsd::Embedding> queries;
  for (int b = 0; b < B; ++b) queries.emplace_back(q.begin() + (size_t)b * dim, q.begin() + (size_t)(b + 1) * dim);
  auto batch = gpu.search_topk_exact_batch(queries, k);
  for (int b = 0; b < B; ++b) {
    auto want = ref.search_topk_exact(queries[(size_t)b], k);
    auto got = b % 7 == 0 ? gpu.search_topk_exact(queries[(size_t)b], k) : batch[(size_t)b];
    CHECK(got.size() == want.size(), "hit count q=%d", b);
    for (size_t i = 0; i < std::min(got.size(), want.size()); ++i) {
      CHECK(got[i].record_id == want[i].record_id, "id q=%d rank=%zu", b, i);
      CHECK(std::memcmp(&got[i].score, &want[i].score, sizeof(double)) == 0, "score bits q=%d rank=%zu", b, i);
      CHECK(got[i].payload == want[i].payload, "payload q=%d rank=%zu", b, i);
    }
  }
  CHECK(gpu.search_topk(queries[0], HSD_K_MAX).size() == HSD_K_MAX, "k = HSD_K_MAX");
  // k > HSD_K_MAX: the large-k path (every row's score + a stable radix sort), any k as in store.cpp
  for (int kk : {HSD_K_MAX + 1, 500, n, n + 3}) {
    std::vector<hsd::Embedding> q3(queries.begin(), queries.begin() + 5);
    auto lb = gpu.search_topk_exact_batch(q3, kk);
    for (int b = 0; b < 5; ++b) {
      auto want = ref.search_topk_exact(queries[(size_t)b], kk);
      auto got = b == 0 ? gpu.search_topk_exact(queries[0], kk) : lb[(size_t)b];
      CHECK(got.size() == want.size(), "large-k hit count k=%d q=%d", kk, b);
      bool same = got.size() == want.size();
      for (size_t i = 0; same && i < got.size(); ++i)
        same = got[i].record_id == want[i].record_id &&
               std::memcmp(&got[i].score, &want[i].score, sizeof(double)) == 0 && got[i].payload == want[i].payload;
      CHECK(same, "large-k hits k=%d q=%d", kk, b);
    }
  }
  CHECK(throws<hsd::InvalidInputError>([&] { gpu.search_topk_exact(queries[0], 0); }), "k < 1 -> InvalidInputError");
  CHECK(throws<hsd::SchemaError>([&] { gpu.insert(hsd::Embedding(3, 0.0), hsd::Payload{}); }), "dim -> SchemaError");
  hsd::gpu::Collection empty("e", dim);
  CHECK(empty.search_topk_exact(queries[0], 5).empty(), "empty collection -> empty result");
  CHECK(throws<hsd::ConfigError>([&] { hsd::gpu::Collection bad("b", 0); }), "dim 0 -> ConfigError");

  // ---- approximate index: build_hnsw / has_hnsw / search_topk (store.cpp:75-92)
  {
    hsd::HnswParams hp;  // m 16, ef_construct 100, ef_search 100
    ref.build_hnsw(hp);
    gpu.build_hnsw(hp);
    CHECK(gpu.has_hnsw(), "has_hnsw after build");
    int common = 0, total = 0;
    for (int b = 0; b < B; ++b) {
      auto got = gpu.search_topk(queries[(size_t)b], k);
      auto hn = ref.search_topk(queries[(size_t)b], k);  // the reference's HNSW
      auto ex = ref.search_topk_exact(queries[(size_t)b], k);
      CHECK(!got.empty() && got.size() <= (size_t)k, "index hit count q=%d", b);
      for (size_t i = 0; i < got.size(); ++i) {
        // every score is the reference's cosine_similarity of the returned id (store.cpp:86-90)
        const double want = hsd::cosine_similarity(queries[(size_t)b], ref.record(got[i].record_id).embedding);
        CHECK(std::memcmp(&got[i].score, &want, sizeof(double)) == 0, "index score bits q=%d rank=%zu", b, i);
        CHECK(got[i].payload == ref.record(got[i].record_id).payload, "index payload q=%d", b);
        if (i) CHECK(got[i - 1].score > got[i].score || (got[i - 1].score == got[i].score &&
                                                          got[i - 1].record_id < got[i].record_id),
                     "index order q=%d rank=%zu", b, i);
      }
      // near-duplicate queries (the first half of a REAL batch) find their row at rank 0, as HNSW does
      if (hsd_query_row(78, HSD_SYNTH_REAL, b, n) >= 0) {
        CHECK(got[0].record_id == ex[0].record_id, "index top-1 q=%d", b);
        CHECK(hn.empty() || hn[0].record_id == ex[0].record_id, "reference hnsw top-1 q=%d", b);
      }
      for (const auto& h : got)
        for (const auto& e : ex) common += h.record_id == e.record_id;
      total += (int)ex.size();
    }
    std::printf("index recall@%d vs exact: %.3f\n", k, (double)common / total);
    CHECK(gpu.search_topk(queries[0], 0).empty(), "index k = 0 -> no hits (hnsw.cpp:160)");
    {  // k > HSD_K_MAX through the index: the exact top-k
      auto got = gpu.search_topk(queries[2], 100);
      auto want = ref.search_topk_exact(queries[2], 100);
      bool same = got.size() == want.size();
      for (size_t i = 0; same && i < got.size(); ++i)
        same = got[i].record_id == want[i].record_id && std::memcmp(&got[i].score, &want[i].score, 8) == 0;
      CHECK(same, "index k = 100 -> the exact top-100");
    }
    hsd::Payload p;
    gpu.insert(queries[0], p);  // mutation drops the index (store.cpp:55)
    CHECK(!gpu.has_hnsw(), "insert drops the index");
    auto after = gpu.search_topk(queries[1], k);
    auto exact = gpu.search_topk_exact(queries[1], k);
    CHECK(after.size() == exact.size() && after[0].record_id == exact[0].record_id, "no index -> exact search");
    hsd::gpu::Collection e2("e2", dim);
    CHECK(throws<hsd::InvalidInputError>([&] { e2.build_hnsw(hp); }), "empty collection -> InvalidInputError");
  }

  // ---- any dim: rows zero-padded to a multiple of 8 on the device, scores unchanged bit for bit
  for (int odd : {1, 3, 61, 130}) {
    hsd::Collection r2("odd", odd);
    std::mt19937_64 g((uint64_t)odd);
    std::normal_distribution<float> Nf(0.0f, 1.0f);
    for (int i = 0; i < 700; ++i) {
      hsd::Embedding e((size_t)odd);
      for (auto& v : e) v = (double)Nf(g);
      hsd::Payload p;
      p.episode_idx = i;
      r2.insert(std::move(e), p);
    }
    auto g2 = hsd::gpu::Collection::from(r2, 0);
    for (int t = 0; t < 5; ++t) {
      hsd::Embedding qq((size_t)odd);
      for (auto& v : qq) v = (double)Nf(g);
      auto want = r2.search_topk_exact(qq, 9);
      auto got = g2.search_topk_exact(qq, 9);
      CHECK(got.size() == want.size(), "odd dim %d hit count", odd);
      for (size_t i = 0; i < std::min(got.size(), want.size()); ++i) {
        CHECK(got[i].record_id == want[i].record_id, "odd dim %d id rank=%zu", odd, i);
        CHECK(std::memcmp(&got[i].score, &want[i].score, sizeof(double)) == 0, "odd dim %d score bits", odd);
      }
    }
  }

  // ---- Record::feature on the device -> offline calibration from the collection itself
  {
    const int df = 64, per_ep = 20, n_ep = 6;
    hsd::gpu::Collection fc("feat", 16);
    std::vector<hsd::Record> recs;
    std::vector<float> fall;
    std::mt19937_64 g(11);
    std::normal_distribution<double> Nd(0.0, 1.0);
    for (int e = 0; e < n_ep; ++e) {
      std::vector<double> base((size_t)df);
      for (auto& v : base) v = Nd(g);
      for (int i = 0; i < per_ep; ++i) {
        std::vector<double> f((size_t)df);
        double nn = 0.0;
        for (int c = 0; c < df; ++c) {
          f[(size_t)c] = base[(size_t)c] + 0.02 * i * Nd(g);
          nn += f[(size_t)c] * f[(size_t)c];
        }
        for (auto& v : f) v /= std::sqrt(nn);
        for (double v : f) fall.push_back((float)v);
        hsd::Payload p;
        p.episode_idx = e;
        p.step_idx = i;
        recs.push_back({hsd::Embedding(16, 0.25), p, (e == 3 && i == 7) ? std::nullopt : std::optional(f)});
      }
    }
    fc.insert_batch(recs);
    const double T = 0.9;
    auto got = fc.calibrate_skip(T);
    // oracle: exactly rounded dots of the stored fp32 features, trajectories split at the featureless record
    hsdo_calib cal;
    hsdo_calibrate_init(&cal);
    std::vector<std::pair<int, int>> runs;
    for (int e = 0; e < n_ep; ++e) {
      if (e == 3) {
        runs.push_back({e * per_ep, e * per_ep + 7});
        runs.push_back({e * per_ep + 8, (e + 1) * per_ep});
      } else {
        runs.push_back({e * per_ep, (e + 1) * per_ep});
      }
    }
    for (auto [a, b] : runs) {
      const int m = b - a;
      std::vector<double> sims((size_t)m * m, 0.0);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j)
          sims[(size_t)i * m + j] = hsdo_feature_cos(&fall[(size_t)(a + i) * df], &fall[(size_t)(a + j) * df], df);
      hsdo_calibrate_accumulate(&cal, sims.data(), m, T);
    }
    double mS = 0.0;
    int od = 0;
    CHECK(hsdo_calibrate_finish(&cal, &mS, &od) == 0, "oracle calibration");
    CHECK(got.first == mS && got.second == od, "calibrate_skip %.17g/%d vs %.17g/%d", got.first, got.second, mS, od);
    CHECK(throws<hsd::CalibrationError>([&] { fc.calibrate_skip(1.0); }), "T = 1 -> CalibrationError");
  }

  // ---- quantize parity against the reference
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> U(-1.4, 1.4);
  std::vector<hsd::ActionSlice> acts(3000);
  for (auto& a : acts)
    for (int j = 0; j < 7; ++j) a[j] = U(rng);
  acts[0] = hsd::ActionSlice{{-1, 1, 0, 1, -1, 0.5, 1}};
  const auto bounds = hsd::ActionSpaceBounds::uniform(-1.0, 1.0);
  auto got = hsd::gpu::quantize_batch(acts, bounds, 256);
  for (size_t i = 0; i < acts.size(); ++i) CHECK(got[i] == hsd::quantize(acts[i], bounds, 256), "quantize %zu", i);
  hsd::ActionSlice nan_a;
  nan_a[2] = NAN;
  CHECK(throws<hsd::InvalidInputError>([&] { hsd::gpu::quantize(nan_a, bounds, 256); }), "nan -> InvalidInputError");

  // ---- window_features vs the oracle restatement (reference needs Eigen)
  hsd::FusedMetricParams mp;  // alpha .5, w 15, theta .5, r_cap 1 (kinematics.hpp:39-42)
  hsd::NormalizationBounds nb{0.000009, 0.123381, 0.000001, 0.014989};
  std::vector<std::vector<hsd::TrajectoryPoint>> wins;
  std::normal_distribution<double> N(0.0, 0.004);
  for (int w = 0; w < 200; ++w) {
    std::vector<hsd::TrajectoryPoint> pts;
    double x = 0, y = 0, z = 0;
    for (int i = 0; i < 15; ++i) {
      if (w % 3 == 0) {
        const double th = 0.3 * i;
        x = 0.05 * std::cos(th) + 0.1 * w / 200.0;
        y = 0.05 * std::sin(th);
        z = 0.001 * i;
      } else {
        x += N(rng);
        y += N(rng);
        z += N(rng);
      }
      pts.push_back({x, y, z, i});
    }
    wins.push_back(pts);
  }
  std::vector<hsd::SdKind> dec;
  auto feats = hsd::gpu::window_features_batch(wins, mp, nb, &dec);
  hsdo_metric_params omp{mp.alpha, mp.w, mp.threshold, mp.r_cap};
  hsdo_norm_bounds onb{nb.d_min, nb.d_max95, nb.r_min, nb.r_max95};
  for (size_t w = 0; w < wins.size(); ++w) {
    double xyz[45], R, D, F;
    int d;
    for (int i = 0; i < 15; ++i) {
      xyz[3 * i] = wins[w][(size_t)i].x;
      xyz[3 * i + 1] = wins[w][(size_t)i].y;
      xyz[3 * i + 2] = wins[w][(size_t)i].z;
    }
    hsdo_window_features(xyz, 15, &omp, &onb, &R, &D, &F, &d);
    CHECK(std::fabs(feats[w].R - R) <= 1e-5 * std::max(1e-12, std::fabs(R)) + 1e-15, "R w=%zu %g %g", w, feats[w].R, R);
    CHECK(std::fabs(feats[w].D - D) <= 1e-5 * D + 1e-15, "D w=%zu", w);
    CHECK(std::fabs(feats[w].F - F) <= 1e-5, "F w=%zu", w);
    if (std::fabs(F - mp.threshold) > 1e-9)
      CHECK((dec[w] == hsd::SdKind::retrieval_sd) == (d == 1), "decision w=%zu", w);
  }
  auto one = hsd::gpu::window_features(std::span<const hsd::TrajectoryPoint>(wins[1]), mp, nb);
  CHECK(one.R == feats[1].R && one.w == 15, "single window");
  CHECK(throws<hsd::InvalidInputError>([&] {
          hsd::gpu::window_features(std::span<const hsd::TrajectoryPoint>(wins[0].data(), 14), mp, nb);
        }),
        "w mismatch -> InvalidInputError");
  hsd::FusedMetricParams badp;
  badp.alpha = 1.5;
  CHECK(throws<hsd::ConfigError>([&] { hsd::gpu::window_features_batch({wins[0]}, badp, nb); }), "alpha -> ConfigError");

  if (failures) {
    std::printf("DROPIN FAILED (%d)\n", failures);
    return 1;
  }
  std::printf("DROPIN OK: %d queries, %zu quantize, %zu windows\n", B, acts.size(), wins.size());
  return 0;
}
