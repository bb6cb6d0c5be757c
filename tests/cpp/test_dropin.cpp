// The reference's doctest cases for the hot path, restated against the C++
// drop-in (include/sparsim_b200.hpp) — the reference's own call sites compile
// unchanged against it.  Built by __graft_entry__.build(), run on the GPU by
// tests/test_gpu_cpp.py.  Exit code = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <set>

#include "sparsim_b200.hpp"

using namespace sparsim;

static int g_fail = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      ++g_fail;                                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                  \
  } while (0)
#define CHECK_THROWS_AS(expr, type) \
  do {                              \
    bool ok = false;                \
    try {                           \
      (void)(expr);                 \
    } catch (const type&) {         \
      ok = true;                    \
    } catch (...) {                 \
    }                               \
    CHECK(ok && #type);             \
  } while (0)

static GradientVector vec(std::initializer_list<double> xs) { return GradientVector(xs); }

int main() {
  int ndev = 0;
  if (micro_device_count(&ndev) != MICRO_OK || ndev == 0) {
    std::printf("no CUDA device\n");
    return 100;
  }
  // test_tensor.cpp:66-78
  CHECK(partition(8, 4, 0, 2) == (PartitionRange{4, 6, 2}));
  CHECK(partition(8, 1, 7, 0) == (PartitionRange{0, 8, 0}));
  CHECK(partition(10, 4, 1, 3) == (PartitionRange{0, 3, 3}));
  CHECK_THROWS_AS(partition(3, 4, 0, 0), std::invalid_argument);
  CHECK_THROWS_AS(partition(8, 4, 0, 4), std::invalid_argument);
  CHECK_THROWS_AS(partition(8, 0, 0, 0), std::invalid_argument);

  // test_sparsifier.cpp:47-69
  {
    const GradientVector acc = vec({1, -3, 0.5, 2});
    auto sel = select_by_threshold(acc, PartitionRange{0, 4, 0}, 1.5);
    CHECK((sel.indices == std::vector<Index>{1, 3}));
    CHECK((sel.values == std::vector<double>{-3, 2}));
    CHECK(select_by_threshold(acc, PartitionRange{0, 4, 0}, 100.0).count() == 0);
    const GradientVector z = vec({0, -0.25, 0, 7});
    CHECK((select_by_threshold(z, PartitionRange{0, 4, 0}, 0.0).indices == std::vector<Index>{1, 3}));
    const GradientVector five = vec({5, 5, 5, 5});
    CHECK((select_by_threshold(five, PartitionRange{1, 3, 0}, 0.0).indices == std::vector<Index>{1, 2}));
    CHECK_THROWS_AS(select_by_threshold(five, PartitionRange{0, 9, 0}, 0.0), std::invalid_argument);
    CHECK_THROWS_AS(select_by_threshold(five, PartitionRange{0, 4, 0}, -1.0), std::invalid_argument);
    CHECK((hard_threshold_select(vec({0.1, 0.9, 0.5}), 0.4).indices == std::vector<Index>{1, 2}));
  }
  // test_sparsifier.cpp:71-98 top-k, CLT-k, select_all (ties to the lower index)
  {
    const GradientVector acc = vec({1, -3, 0.5, 2});
    auto top = select_topk(acc, PartitionRange{0, 4, 0}, 2);
    CHECK((top.indices == std::vector<Index>{1, 3}));
    CHECK((top.values == std::vector<double>{-3, 2}));
    const GradientVector tied = vec({1, -1, 1, 1});
    CHECK((select_topk(tied, PartitionRange{0, 4, 0}, 2).indices == std::vector<Index>{0, 1}));
    CHECK((select_topk(tied, PartitionRange{1, 4, 0}, 2).indices == std::vector<Index>{1, 2}));
    CHECK(select_topk(acc, PartitionRange{0, 4, 0}, 4).count() == 4);
    CHECK(select_topk(acc, PartitionRange{0, 4, 0}, 0).count() == 0);
    CHECK_THROWS_AS(select_topk(acc, PartitionRange{0, 2, 0}, 3), std::invalid_argument);
    CHECK((cltk_select(acc, 1, 1, 5, 4).indices == std::vector<Index>{1}));
    CHECK_THROWS_AS(cltk_select(acc, 1, 0, 5, 4), std::logic_error);
    CHECK_THROWS_AS(cltk_select(acc, 9, 1, 5, 4), std::invalid_argument);
    CHECK(select_all(acc).count() == 4 && select_all(acc).values[1] == -3.0);
    CHECK(parse_sparsifier_kind("hard") == SparsifierKind::hard_threshold && to_string(SparsifierKind::cltk) == "cltk");
    CHECK_THROWS_AS(parse_sparsifier_kind("foo"), std::invalid_argument);
    // randomized against a host sort (|acc| desc, index asc)
    std::mt19937_64 r2(5);
    for (int rep = 0; rep < 20; ++rep) {
      const std::size_t n = 1 + r2() % 5000;
      GradientVector a(n);
      for (auto& v : a) v = (double)((int)(r2() % 9) - 4) * 0.25;  // many ties
      const std::size_t k = r2() % (n + 1);
      std::vector<Index> ord(n);
      for (std::size_t j = 0; j < n; ++j) ord[j] = (Index)j;
      std::sort(ord.begin(), ord.end(), [&](Index x, Index y) {
        const double ax = std::fabs(a[(std::size_t)x]), ay = std::fabs(a[(std::size_t)y]);
        return ax != ay ? ax > ay : x < y;
      });
      ord.resize(k);
      std::sort(ord.begin(), ord.end());
      CHECK(select_topk(a, PartitionRange{0, (Index)n, 0}, k).indices == ord);
    }
  }
  // test_sparsifier.cpp:100-112, 217-227
  CHECK(micro_update_threshold({1.0}, 100, 150, 0.1).delta == 1.1000000000000001);
  CHECK(micro_update_threshold({1.0}, 100, 100, 0.1).delta == 1.0);
  CHECK(std::fabs(micro_update_threshold({1.0}, 100, 40, 0.1).delta - 0.9) < 1e-15);
  CHECK(micro_update_threshold({0.0}, 10, 50, 0.1, 1e-12).delta == 1e-12);
  CHECK(micro_update_threshold({0.0}, 10, 3, 0.1).delta == 0.0);
  CHECK_THROWS_AS(micro_update_threshold({1.0}, 10, 5, 0.0), std::invalid_argument);
  CHECK(global_target_count(0.01, 10000) == 100);
  CHECK(global_target_count(0.001, 100) == 1);
  CHECK(per_worker_target_count(0.01, 10000, 4, PerWorkerTarget::split) == 25);
  CHECK(per_worker_target_count(0.01, 10000, 4, PerWorkerTarget::full) == 100);
  CHECK_THROWS_AS(global_target_count(1.5, 100), std::invalid_argument);

  // test_sparsifier.cpp:154-182 partition-filter invariance (seeded, double)
  {
    std::mt19937_64 rng(13);
    std::normal_distribution<double> unit(0.0, 1.0);
    std::uniform_real_distribution<double> thr(0.0, 2.5);
    for (int n : {1, 2, 4, 8}) {
      for (int rep = 0; rep < 10; ++rep) {
        const Index n_g = n + static_cast<Index>(rng() % 20000);
        GradientVector acc((std::size_t)n_g);
        for (auto& v : acc) v = unit(rng);
        const double delta = thr(rng);
        const auto t = static_cast<std::int64_t>(rng() % 50);
        const auto whole = select_by_threshold(acc, PartitionRange{0, n_g, 0}, delta);
        std::vector<SparseSelection> parts;
        for (int i = 0; i < n; ++i) parts.push_back(select_by_threshold(acc, partition(n_g, n, t, i), delta));
        const auto agg = all_gather_indices(parts);
        CHECK(agg.indices == whole.indices);
        CHECK(agg.total_selected() == whole.count());
        std::size_t scalar = 0;
        for (Index j = 0; j < n_g; ++j) scalar += std::abs(acc[(std::size_t)j]) > delta;
        CHECK(scalar == whole.count());
      }
    }
  }
  // test_error_feedback.cpp:26-65
  {
    const GradientVector g = vec({3, -1, 2});
    CHECK(accumulate(GradientVector(3, 0.0), 1.0, g) == g);
    CHECK(accumulate(vec({1, 1}), 0.5, vec({2, 0})) == vec({2, 1}));
    CHECK_THROWS_AS(accumulate(vec({1, 1}), 1.0, vec({1, 2, 3})), std::invalid_argument);
    CHECK_THROWS_AS(accumulate(vec({1, 1}), 0.0, vec({1, 2})), std::invalid_argument);
    const GradientVector acc = vec({3, 4, 5});
    SparseSelection everything{{0, 1, 2}, {3, 4, 5}};
    CHECK(compensate(acc, everything) == GradientVector(3, 0.0));
    CHECK(compensate(acc, SparseSelection{}) == acc);
    SparseSelection one{{1}, {4}};
    CHECK(compensate(acc, one) == vec({3, 0, 5}));
    SparseSelection bad{{7}, {0}};
    CHECK_THROWS_AS(compensate(acc, bad), std::invalid_argument);
  }
  // test_collectives.cpp:29-66
  {
    auto sel_of = [](std::vector<Index> ix) {
      SparseSelection s;
      s.indices = ix;
      s.values.assign(ix.size(), 1.0);
      return s;
    };
    auto d = all_gather_indices({sel_of({0, 1}), sel_of({2, 3})});
    CHECK((d.indices == std::vector<Index>{0, 1, 2, 3}));
    CHECK(d.total_selected() == 4);
    auto o = all_gather_indices({sel_of({0, 1}), sel_of({0, 1})});
    CHECK((o.indices == std::vector<Index>{0, 1}));
    CHECK(o.total_selected() == 4);
    const std::vector<GradientVector> accs{vec({1, 2}), vec({3, 4})};
    AggregatedSelection at1;
    at1.indices = {1};
    at1.per_worker_counts = {1, 0};
    const GradientVector g = all_reduce_sparse(accs, at1);
    CHECK(g[0] == 0.0 && g[1] == 6.0);
    CHECK((all_reduce_sparse_values(accs, at1) == std::vector<double>{6.0}));
    CHECK_THROWS_AS(all_reduce_sparse(std::vector<GradientVector>{vec({1, 2}), vec({1, 2, 3})}, at1),
                    std::invalid_argument);
  }
  // harness.cpp:121-224 via MicroEngine: exclusivity, conservation, density
  {
    const Index n_g = 100003;
    const int n = 4;
    SparsifierConfig sc;
    sc.density = 0.01;
    sc.initial_threshold = 0.02;
    MicroEngine eng(n_g, n, sc);
    std::mt19937_64 rng(42);
    std::normal_distribution<double> unit(0.0, 1.0);
    std::vector<double> G((std::size_t)(n * n_g));
    std::vector<double> want_norm, want_thr, want_density;
    for (int t = 0; t < 20; ++t) {
      for (auto& v : G) v = unit(rng);
      std::vector<double> summed;
      double thr = 0.0;
      for (const auto& d : eng.thresholds()) thr += d.delta;
      want_thr.push_back(thr / n);
      const auto agg = eng.step(G.data(), 0.01, t, &summed);
      want_density.push_back(actual_density(agg, n_g));
      std::vector<GradientVector> res;
      for (int i = 0; i < n; ++i) res.push_back(eng.residual(i));
      double ns = 0.0;  // error_feedback.hpp:41-48 with a sequential fp64 norm
      for (const auto& e : res) {
        double q = 0.0;
        for (double v : e) q += v * v;
        ns += std::sqrt(q);
      }
      want_norm.push_back(ns / n);
      CHECK(std::fabs(error_metric(res) - ns / n) <= 1e-12 * (ns / n));
      CHECK(agg.indices.size() == agg.total_selected());  // no build-up (acceptance.cpp:93-118)
      for (std::size_t k = 1; k < agg.indices.size(); ++k) CHECK(agg.indices[k - 1] < agg.indices[k]);
      CHECK(summed.size() == agg.indices.size());
      for (int i = 0; i < n; ++i) {
        const auto e = eng.residual(i);
        for (Index j : agg.indices) CHECK(e[(std::size_t)j] == 0.0);
      }
    }
    // IterationRecord (metrics.hpp:15-29) from the device history
    const auto recs = eng.records();
    CHECK(recs.size() == 20);
    for (std::size_t s = 0; s < recs.size(); ++s) {
      CHECK(recs[s].t == (std::int64_t)s);
      CHECK(recs[s].actual_density == want_density[s]);
      CHECK(recs[s].redundant_traffic_factor == 1.0);
      CHECK(recs[s].threshold == want_thr[s]);
      CHECK(std::fabs(recs[s].error_norm - want_norm[s]) <= 1e-12 * want_norm[s]);
    }
  }
  // non-finite gradient (harness.cpp:128-130): MicroEngine::step throws
  // std::runtime_error, keeps refusing until reset(), then steps again
  {
    const Index n_g = 4099;
    const int n = 2;
    SparsifierConfig sc;
    MicroEngine eng(n_g, n, sc);
    std::vector<double> G((std::size_t)(n * n_g), 0.5);
    eng.step(G.data(), 0.01, 0);
    G[(std::size_t)n_g + 7] = std::nan("");
    CHECK_THROWS_AS(eng.step(G.data(), 0.01, 1), std::runtime_error);
    G[(std::size_t)n_g + 7] = 0.5;
    CHECK_THROWS_AS(eng.step(G.data(), 0.01, 2), std::runtime_error);  // poisoned until reset
    eng.reset();
    const auto agg = eng.step(G.data(), 0.01, 0);
    CHECK(agg.per_worker_counts.size() == 2);
    G[3] = INFINITY;
    CHECK_THROWS_AS(eng.step(G.data(), 0.01, 1), std::runtime_error);
    bool is_logic = false;  // runtime_error, not invalid_argument / logic_error
    try {
      eng.step(G.data(), 0.01, 2);
    } catch (const std::logic_error&) {
      is_logic = true;
    } catch (const std::runtime_error&) {
    }
    CHECK(!is_logic);
  }
  // fp32 gradients into the fp64 engine (MICRO_GRAD_F32) == the fp64 engine
  // on the same values widened: selection, sums, residuals, bit for bit
  {
    const Index n_g = 70001;
    const int n = 3;
    SparsifierConfig sc;
    sc.density = 0.02;
    sc.initial_threshold = 0.02;
    MicroEngine e32(n_g, n, sc, true, MICRO_F64, MICRO_GRAD_F32);
    MicroEngine e64(n_g, n, sc, true, MICRO_F64);
    std::mt19937_64 rng(5);
    std::normal_distribution<float> unit(0.0f, 1.0f);
    std::vector<float> Gf((std::size_t)(n * n_g));
    std::vector<double> Gd(Gf.size());
    for (int t = 0; t < 6; ++t) {
      for (std::size_t j = 0; j < Gf.size(); ++j) Gd[j] = (double)(Gf[j] = unit(rng));
      std::vector<double> s32, s64;
      const auto a = e32.step(Gf.data(), 0.01, t, &s32);
      const auto b = e64.step(Gd.data(), 0.01, t, &s64);
      CHECK(a.indices == b.indices);
      CHECK(a.per_worker_counts == b.per_worker_counts);
      CHECK(s32 == s64);
    }
    for (int i = 0; i < n; ++i) CHECK(e32.residual(i) == e64.residual(i));
  }
  // MicroGroup (one process, one context per rank; here all on device 0)
  // == MicroEngine (single-device cluster), bit for bit
  {
    const Index n_g = 50001;
    const int n = 3;
    SparsifierConfig sc;
    sc.density = 0.02;
    sc.initial_threshold = 0.02;
    MicroEngine eng(n_g, n, sc, true, MICRO_F32);
    MicroGroup grp(n_g, std::vector<int>(n, 0), sc, true, MICRO_F32);
    std::mt19937_64 rng(9);
    std::normal_distribution<float> unit(0.0f, 1.0f);
    std::vector<float> G((std::size_t)(n * n_g));
    std::vector<void*> d(n);
    for (int r = 0; r < n; ++r) b200::check(micro_device_malloc(&d[r], (int64_t)n_g * 4, 0));
    for (int t = 0; t < 8; ++t) {
      for (auto& v : G) v = unit(rng);
      std::vector<double> summed;
      const auto agg = eng.step(G.data(), 0.01, t, &summed);
      for (int r = 0; r < n; ++r) b200::h2d(d[r], G.data() + (std::size_t)r * n_g, (std::size_t)n_g * 4);
      grp.step(std::vector<const void*>(d.begin(), d.end()), 0.01, t);
      grp.sync();
      for (int r = 0; r < n; ++r) {
        std::vector<int32_t> idx((std::size_t)n_g);
        std::vector<float> sums((std::size_t)n_g);
        int64_t K = 0;
        b200::check(micro_copy_union(grp.rank(r), idx.data(), sums.data(), n_g, &K));
        CHECK((std::size_t)K == agg.indices.size());
        bool same = (std::size_t)K == agg.indices.size();
        for (int64_t k = 0; same && k < K; ++k)
          same = idx[(std::size_t)k] == agg.indices[(std::size_t)k] && (double)sums[(std::size_t)k] == summed[(std::size_t)k];
        CHECK(same);
      }
    }
    for (int r = 0; r < n; ++r) micro_device_free(d[r]);
  }
  std::printf("%s: %d failed checks\n", g_fail ? "FAIL" : "OK", g_fail);
  return g_fail;
}
