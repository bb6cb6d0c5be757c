// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker / CPU baseline arm).
//
// An extern "C" face over the reference's own hot-path code, compiled
// VERBATIM from /root/reference/proj/src/{sparsifier,collectives,metrics}.cpp
// and its sparsim/*.hpp headers against oracle/eigen_shim (see
// oracle/Makefile).  Nothing here is copied from the reference: the wrappers
// only marshal plain pointers into the reference's value types and call its
// functions.  ref_cluster_* re-drives the MiCRO branch of run_iteration
// (proj/src/harness.cpp:121-224) in the same order with the same calls;
// harness.cpp itself cannot be built here because it pulls in task.cpp, which
// needs the full Eigen Dense API.
//
// Output lands only in oracle/_ref/ (git-ignored; travels to the GPU box).
#include "sparsim/collectives.hpp"
#include "sparsim/error_feedback.hpp"
#include "sparsim/metrics.hpp"
#include "sparsim/sparsifier.hpp"
#include "sparsim/tensor.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace sparsim;

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_msg = e.what();
    return 2;
  } catch (const std::runtime_error& e) {
    g_msg = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 8;
  }
}

GradientVector from_ptr(const double* p, std::int64_t n) {
  GradientVector v(n);
  if (n) std::memcpy(v.data(), p, static_cast<std::size_t>(n) * sizeof(double));
  return v;
}

void to_ptr(const GradientVector& v, double* out) {
  if (v.size()) std::memcpy(out, v.data(), static_cast<std::size_t>(v.size()) * sizeof(double));
}

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// Mirror of the ClusterState fields the MiCRO branch touches (harness.hpp:49-70).
struct RefCluster {
  Index n_g;
  int n;
  SparsifierConfig sc;
  bool error_feedback;
  std::vector<GradientVector> residuals;     // WorkerState::residual
  std::vector<ThresholdState> thresholds;    // WorkerState::threshold
  std::vector<GradientVector> accumulators;  // ClusterState::accumulators
  std::size_t k_global = 0, k_worker = 0;
  double phase[4] = {0, 0, 0, 0};  // accumulate, select, gather+reduce, threshold+compensate
  // bench options (ref_cluster_set_options): the dense averaged gradient
  // all_reduce_sparse(...) / n (collectives.cpp:51-57) each step, and host
  // threads for the per-worker loops (harness.cpp runs its workers one after
  // the other; with threads > 1 the same per-worker calls run concurrently)
  bool dense_on = false;
  GradientVector dense;
  int threads = 1;
};

// f(i) for every worker i, on up to `threads` host threads (workers are
// independent in the accumulate, select and compensate loops).
template <class F>
void for_workers(int n, int threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> err(static_cast<std::size_t>(n));
  const int T = threads < n ? threads : n;
  for (int w = 0; w < T; ++w)
    pool.emplace_back([&, w] {
      for (int i = w; i < n; i += T) {
        try {
          f(i);
        } catch (...) {
          err[static_cast<std::size_t>(i)] = std::current_exception();
        }
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

int ref_partition(std::int64_t n_g, int n, std::int64_t t, int worker, std::int64_t* start,
                  std::int64_t* end) {
  return guarded([&] {
    const PartitionRange r = partition(n_g, n, t, worker);
    *start = r.start;
    *end = r.end;
  });
}

int ref_global_target_count(double d, std::int64_t n_g, std::uint64_t* k) {
  return guarded([&] { *k = global_target_count(d, n_g); });
}

int ref_per_worker_target_count(double d, std::int64_t n_g, int n, int target, std::uint64_t* k) {
  return guarded([&] {
    *k = per_worker_target_count(d, n_g, n, target ? PerWorkerTarget::full : PerWorkerTarget::split);
  });
}

int ref_update_threshold(double* delta, std::uint64_t k_target, std::uint64_t k_selected,
                         double alpha, double min_threshold) {
  return guarded([&] {
    *delta = micro_update_threshold(ThresholdState{*delta}, k_target, k_selected, alpha,
                                    min_threshold)
                 .delta;
  });
}

int ref_select_by_threshold(const double* acc, std::int64_t n_g, std::int64_t start,
                            std::int64_t end, double delta, std::int64_t* idx, double* val,
                            std::int64_t* count) {
  return guarded([&] {
    const GradientVector a = from_ptr(acc, n_g);
    const SparseSelection s = select_by_threshold(a, PartitionRange{start, end, 0}, delta);
    for (std::size_t k = 0; k < s.count(); ++k) {
      idx[k] = s.indices[k];
      val[k] = s.values[k];
    }
    *count = static_cast<std::int64_t>(s.count());
  });
}

int ref_accumulate(const double* e, std::int64_t n_e, double eta, const double* g,
                   std::int64_t n_g, double* out) {
  return guarded([&] { to_ptr(accumulate(from_ptr(e, n_e), eta, from_ptr(g, n_g)), out); });
}

int ref_compensate(const double* acc, std::int64_t n, const std::int64_t* sel, std::int64_t k,
                   double* out) {
  return guarded([&] {
    std::vector<Index> s(sel, sel + k);
    to_ptr(compensate(from_ptr(acc, n), std::span<const Index>(s)), out);
  });
}

// selections: row i = counts[i] indices, rows concatenated in worker order.
int ref_all_gather_indices(int n, const std::int64_t* counts, const std::int64_t* concat,
                           std::int64_t* union_idx, std::int64_t* K, std::uint64_t* total) {
  return guarded([&] {
    std::vector<SparseSelection> sels(static_cast<std::size_t>(n));
    std::int64_t off = 0;
    for (int i = 0; i < n; ++i) {
      sels[i].indices.assign(concat + off, concat + off + counts[i]);
      sels[i].values.assign(static_cast<std::size_t>(counts[i]), 0.0);
      off += counts[i];
    }
    const AggregatedSelection agg = all_gather_indices(sels);
    std::copy(agg.indices.begin(), agg.indices.end(), union_idx);
    *K = static_cast<std::int64_t>(agg.indices.size());
    *total = agg.total_selected();
  });
}

int ref_all_reduce_sparse_values(const double* accs, int n, std::int64_t n_g,
                                 const std::int64_t* union_idx, std::int64_t K, double* sums) {
  return guarded([&] {
    std::vector<GradientVector> a;
    for (int i = 0; i < n; ++i) a.push_back(from_ptr(accs + static_cast<std::int64_t>(i) * n_g, n_g));
    AggregatedSelection agg;
    agg.indices.assign(union_idx, union_idx + K);
    const std::vector<double> v = all_reduce_sparse_values(a, agg);
    std::copy(v.begin(), v.end(), sums);
  });
}

int ref_all_reduce_sparse(const double* accs, int n, std::int64_t n_g,
                          const std::int64_t* union_idx, std::int64_t K, double* dense) {
  return guarded([&] {
    std::vector<GradientVector> a;
    for (int i = 0; i < n; ++i) a.push_back(from_ptr(accs + static_cast<std::int64_t>(i) * n_g, n_g));
    AggregatedSelection agg;
    agg.indices.assign(union_idx, union_idx + K);
    to_ptr(all_reduce_sparse(a, agg), dense);
  });
}

int ref_error_metric(const double* es, int n, std::int64_t n_g, double* out) {
  return guarded([&] {
    std::vector<GradientVector> r;
    for (int i = 0; i < n; ++i) r.push_back(from_ptr(es + static_cast<std::int64_t>(i) * n_g, n_g));
    *out = error_metric(r);
  });
}

// ---- run_iteration's MiCRO branch (harness.cpp:121-224) over the reference calls ----

void* ref_cluster_create(std::int64_t n_g, int n, double density, double delta0, double alpha,
                         double min_threshold, int target, int error_feedback) {
  auto* c = new RefCluster;
  c->n_g = n_g;
  c->n = n;
  c->sc.density = density;
  c->sc.initial_threshold = delta0;
  c->sc.scaling_factor = alpha;
  c->sc.min_threshold = min_threshold;
  c->sc.target = target ? PerWorkerTarget::full : PerWorkerTarget::split;
  c->error_feedback = error_feedback != 0;
  int rc = guarded([&] {
    if (n < 1 || n_g < n) throw std::invalid_argument("run config: bad worker count");
    c->residuals.assign(static_cast<std::size_t>(n), GradientVector::Zero(n_g));  // harness.cpp:95
    c->thresholds.assign(static_cast<std::size_t>(n), ThresholdState{delta0});   // harness.cpp:96
    c->accumulators.assign(static_cast<std::size_t>(n), GradientVector::Zero(n_g));
    c->k_global = global_target_count(density, n_g);                                // :106
    c->k_worker = per_worker_target_count(density, n_g, n, c->sc.target);           // :107
  });
  if (rc) {
    delete c;
    return nullptr;
  }
  return c;
}

void ref_cluster_destroy(void* h) { delete static_cast<RefCluster*>(h); }

// G: n*n_g doubles (worker-major).  Outputs: counts[n], union_idx[K], summed[K],
// *K, delta_used[n].  x (optional, n_g): the model, updated x -= summed/n.
int ref_cluster_step(void* h, const double* G, double eta, std::int64_t t, double* x,
                     std::int64_t* counts, std::int64_t* union_idx, double* summed,
                     std::int64_t* K, double* delta_used) {
  auto& cs = *static_cast<RefCluster*>(h);
  return guarded([&] {
    const int n = cs.n;
    const Index n_g = cs.n_g;
    auto t0 = Clock::now();
    // gradients and residual accumulation (harness.cpp:123-132)
    for (int i = 0; i < n; ++i) {
      const double* g = G + static_cast<std::int64_t>(i) * n_g;
      for (Index j = 0; j < n_g; ++j)
        if (!std::isfinite(g[j]))
          throw std::runtime_error("iteration " + std::to_string(t) +
                                   ": non-finite gradient on worker " + std::to_string(i));
    }
    for_workers(n, cs.threads, [&](int i) {
      // cs.accumulators[i] = w.residual + eta * grad; — evaluated in place like Eigen's
      // lazy assignment (no temporary), the same IEEE op per element.
      const double* g = G + static_cast<std::int64_t>(i) * n_g;
      double* acc = cs.accumulators[static_cast<std::size_t>(i)].data();
      const double* res = cs.residuals[static_cast<std::size_t>(i)].data();
      for (Index j = 0; j < n_g; ++j) acc[j] = res[j] + eta * g[j];
    });
    auto t1 = Clock::now();
    // selection (harness.cpp:139-151)
    std::vector<SparseSelection> selections(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) delta_used[i] = cs.thresholds[static_cast<std::size_t>(i)].delta;
    for_workers(n, cs.threads, [&](int i) {
      const auto range = partition(n_g, n, t, i);
      selections[static_cast<std::size_t>(i)] =
          select_by_threshold(cs.accumulators[static_cast<std::size_t>(i)], range, delta_used[i]);
    });
    auto t2 = Clock::now();
    // collectives (harness.cpp:185-186)
    const AggregatedSelection agg = all_gather_indices(selections);
    const std::vector<double> sums = all_reduce_sparse_values(cs.accumulators, agg);
    if (cs.dense_on) {  // the dense averaged gradient: all_reduce_sparse / n
      cs.dense = all_reduce_sparse(cs.accumulators, agg);
      if (n > 1)
        for (Index j = 0; j < n_g; ++j) cs.dense[j] /= n;
    }
    auto t3 = Clock::now();
    // threshold estimate (harness.cpp:201-208)
    for (int i = 0; i < n; ++i)
      cs.thresholds[static_cast<std::size_t>(i)] = micro_update_threshold(
          cs.thresholds[static_cast<std::size_t>(i)], cs.k_worker,
          selections[static_cast<std::size_t>(i)].count(), cs.sc.scaling_factor,
          cs.sc.min_threshold);
    // model update x - g/n (harness.cpp:212-215), one model (all workers' are identical)
    if (x)
      for (std::size_t k = 0; k < agg.indices.size(); ++k) x[agg.indices[k]] -= sums[k] / n;
    // compensate + swap (harness.cpp:219-224)
    for_workers(n, cs.threads, [&](int i) {
      auto& acc = cs.accumulators[static_cast<std::size_t>(i)];
      for (Index j : agg.indices) acc[j] = 0.0;
      if (!cs.error_feedback) acc.setZero();
      std::swap(cs.residuals[static_cast<std::size_t>(i)], acc);
    });
    auto t4 = Clock::now();
    cs.phase[0] += secs(t0, t1);
    cs.phase[1] += secs(t1, t2);
    cs.phase[2] += secs(t2, t3);
    cs.phase[3] += secs(t3, t4);
    for (int i = 0; i < n; ++i) counts[i] = static_cast<std::int64_t>(agg.per_worker_counts[i]);
    std::copy(agg.indices.begin(), agg.indices.end(), union_idx);
    std::copy(sums.begin(), sums.end(), summed);
    *K = static_cast<std::int64_t>(agg.indices.size());
  });
}

// The comparison sparsifiers of run_iteration (harness.cpp:152-181: top-k,
// CLT-k, hard threshold, dense; kind = SparsifierKind 1..4), then the same
// collectives, model update and compensate + swap as the MiCRO branch.
int ref_cluster_step_kind(void* h, int kind, const double* G, double eta, std::int64_t t, double* x,
                          std::int64_t* counts, std::int64_t* union_idx, double* summed, std::int64_t* K) {
  auto& cs = *static_cast<RefCluster*>(h);
  return guarded([&] {
    const int n = cs.n;
    const Index n_g = cs.n_g;
    for (int i = 0; i < n; ++i) {
      const double* g = G + static_cast<std::int64_t>(i) * n_g;
      for (Index j = 0; j < n_g; ++j)
        if (!std::isfinite(g[j]))
          throw std::runtime_error("iteration " + std::to_string(t) +
                                   ": non-finite gradient on worker " + std::to_string(i));
      double* acc = cs.accumulators[static_cast<std::size_t>(i)].data();
      const double* res = cs.residuals[static_cast<std::size_t>(i)].data();
      for (Index j = 0; j < n_g; ++j) acc[j] = res[j] + eta * g[j];
    }
    std::vector<SparseSelection> selections(static_cast<std::size_t>(n));
    const PartitionRange whole{0, n_g, 0};
    switch (kind) {
      case 1:
        for (int i = 0; i < n; ++i)
          selections[static_cast<std::size_t>(i)] =
              select_topk(cs.accumulators[static_cast<std::size_t>(i)], whole, cs.k_global);
        break;
      case 2: {
        const int leader = static_cast<int>(t % n);
        selections[static_cast<std::size_t>(leader)] =
            cltk_select(cs.accumulators[static_cast<std::size_t>(leader)], cs.k_global, leader, t, n);
        break;
      }
      case 3:
        for (int i = 0; i < n; ++i)
          selections[static_cast<std::size_t>(i)] =
              hard_threshold_select(cs.accumulators[static_cast<std::size_t>(i)], cs.sc.initial_threshold);
        break;
      case 4:
        for (int i = 0; i < n; ++i)
          selections[static_cast<std::size_t>(i)] = select_all(cs.accumulators[static_cast<std::size_t>(i)]);
        break;
      default:
        throw std::invalid_argument("ref_cluster_step_kind: kind must be 1..4");
    }
    const AggregatedSelection agg = all_gather_indices(selections);
    const std::vector<double> sums = all_reduce_sparse_values(cs.accumulators, agg);
    if (x)
      for (std::size_t k = 0; k < agg.indices.size(); ++k) x[agg.indices[k]] -= sums[k] / n;
    for (int i = 0; i < n; ++i) {
      auto& acc = cs.accumulators[static_cast<std::size_t>(i)];
      for (Index j : agg.indices) acc[j] = 0.0;
      if (!cs.error_feedback) acc.setZero();
      std::swap(cs.residuals[static_cast<std::size_t>(i)], acc);
    }
    for (int i = 0; i < n; ++i) counts[i] = static_cast<std::int64_t>(agg.per_worker_counts[i]);
    std::copy(agg.indices.begin(), agg.indices.end(), union_idx);
    std::copy(sums.begin(), sums.end(), summed);
    *K = static_cast<std::int64_t>(agg.indices.size());
  });
}

int ref_cluster_residual(void* h, int i, double* out) {
  auto& cs = *static_cast<RefCluster*>(h);
  return guarded([&] {
    if (i < 0 || i >= cs.n) throw std::invalid_argument("worker out of range");
    to_ptr(cs.residuals[static_cast<std::size_t>(i)], out);
  });
}

// Bench options: dense != 0 also forms the dense averaged gradient each step;
// threads > 1 runs the per-worker loops concurrently.
int ref_cluster_set_options(void* h, int dense, int threads) {
  auto& cs = *static_cast<RefCluster*>(h);
  cs.dense_on = dense != 0;
  cs.threads = threads < 1 ? 1 : threads;
  return 0;
}

// Overwrite worker i's state (residual, threshold): the bench transplants a
// converged state adapted at a smaller n_g (tiled) so the timed steps start
// in the stationary regime.
int ref_cluster_set_state(void* h, int i, const double* residual, double delta) {
  auto& cs = *static_cast<RefCluster*>(h);
  return guarded([&] {
    if (i < 0 || i >= cs.n) throw std::invalid_argument("worker out of range");
    std::memcpy(cs.residuals[static_cast<std::size_t>(i)].data(), residual,
                static_cast<std::size_t>(cs.n_g) * sizeof(double));
    cs.thresholds[static_cast<std::size_t>(i)] = ThresholdState{delta};
  });
}

int ref_cluster_dense(void* h, double* out) {
  auto& cs = *static_cast<RefCluster*>(h);
  return guarded([&] {
    if (!cs.dense_on || cs.dense.size() != cs.n_g) throw std::logic_error("dense output not formed");
    to_ptr(cs.dense, out);
  });
}

int ref_cluster_thresholds(void* h, double* out) {
  auto& cs = *static_cast<RefCluster*>(h);
  for (int i = 0; i < cs.n; ++i) out[i] = cs.thresholds[static_cast<std::size_t>(i)].delta;
  return 0;
}

void ref_cluster_phase_times(void* h, double* out4) {
  auto& cs = *static_cast<RefCluster*>(h);
  for (int k = 0; k < 4; ++k) out4[k] = cs.phase[k];
}

}  // extern "C"
