// sparsim_b200.hpp — header-only C++ drop-in for the reference's sparsifier
// API (namespace sparsim, /root/reference/proj/include/sparsim/*.hpp), backed
// by the B200 C ABI (micro.h).  Same names, argument meaning and exception
// types as the reference, so its callers and tests relink unchanged:
//
//   reference header                       here
//   tensor.hpp:25-32,48-63  PartitionRange, partition
//   sparsifier.hpp:21-46    SparsifierKind, PerWorkerTarget, SparseSelection, ThresholdState,
//                           SparsifierConfig
//   sparsifier.hpp:49-84    select_by_threshold, select_topk, micro_update_threshold,
//                           cltk_select, hard_threshold_select, select_all,
//                           global/per_worker_target_count, to_string / parse_*
//   error_feedback.hpp:17-48 accumulate, compensate, error_metric
//   collectives.hpp:15-43   AggregatedSelection, all_gather_indices,
//                           all_reduce_sparse(_values), buildup_factor,
//                           redundant_traffic_factor
//   metrics.cpp:7-10        actual_density
//   harness.cpp:121-224     MicroEngine (the per-iteration step for every SparsifierKind)
//   metrics.hpp:15-29       IterationRecord via MicroEngine::records
//
// Vectors are any contiguous container of double with .data()/.size() (e.g.
// Eigen::VectorXd or std::vector<double>); results are returned as
// `GradientVector`, std::vector<double> unless SPARSIM_B200_GRADIENT_VECTOR
// names another type (define it to Eigen::VectorXd before including).
// The value-level calls stage host data through device memory and run the
// fp64 kernels, which are bit-exact against the reference.  Link with
// -lmicro_b200 (paper_2310_00967_b200/lib).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "micro.h"

#ifndef SPARSIM_B200_GRADIENT_VECTOR
#define SPARSIM_B200_GRADIENT_VECTOR std::vector<double>
#endif

namespace sparsim {

using Index = std::ptrdiff_t;
using GradientVector = SPARSIM_B200_GRADIENT_VECTOR;

struct PartitionRange {
  Index start = 0;
  Index end = 0;
  int owner = 0;
  Index size() const { return end - start; }
  bool operator==(const PartitionRange&) const = default;
};

enum class SparsifierKind { micro, topk, cltk, hard_threshold, dense };
enum class PerWorkerTarget { split, full };

struct SparseSelection {
  std::vector<Index> indices;
  std::vector<double> values;
  std::size_t count() const { return indices.size(); }
};

struct ThresholdState {
  double delta = 0.0;
};

struct SparsifierConfig {
  SparsifierKind kind = SparsifierKind::micro;
  double density = 0.01;
  double initial_threshold = 0.01;
  double scaling_factor = 0.01;
  double min_threshold = 1e-12;
  PerWorkerTarget target = PerWorkerTarget::split;
};

struct AggregatedSelection {
  std::vector<Index> indices;
  std::vector<std::size_t> per_worker_counts;
  std::size_t total_selected() const {
    std::size_t s = 0;
    for (auto c : per_worker_counts) s += c;
    return s;
  }
};

namespace b200 {

// Status -> the reference's exception type.
[[noreturn]] inline void raise(int rc) {
  const std::string msg = micro_last_error();
  switch (rc) {
    case MICRO_EINVAL: throw std::invalid_argument(msg);
    case MICRO_ELOGIC: throw std::logic_error(msg);
    case MICRO_ENONFINITE: throw std::runtime_error(msg);
    default: throw std::runtime_error(std::string(micro_status_string(rc)) + ": " + msg);
  }
}
inline void check(int rc) {
  if (rc != MICRO_OK) raise(rc);
}

inline int& device() {
  static int d = 0;
  return d;
}

class DeviceBuffer {
 public:
  explicit DeviceBuffer(std::size_t bytes) { check(micro_device_malloc(&p_, (int64_t)bytes, device())); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  ~DeviceBuffer() { micro_device_free(p_); }
  void* get() const { return p_; }
  template <class T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
};

inline void h2d(void* d, const void* h, std::size_t bytes) { check(micro_memcpy(d, h, (int64_t)bytes, 0, nullptr)); }
inline void d2h(void* h, const void* d, std::size_t bytes) { check(micro_memcpy(h, d, (int64_t)bytes, 1, nullptr)); }

template <class V>
DeviceBuffer upload(const V& v) {
  DeviceBuffer b(sizeof(double) * (std::size_t)v.size());
  h2d(b.get(), v.data(), sizeof(double) * (std::size_t)v.size());
  return b;
}

inline GradientVector make_vector(Index n) { return GradientVector(static_cast<std::size_t>(n)); }

inline std::vector<int32_t> to_i32(const std::vector<Index>& ix) {
  std::vector<int32_t> out(ix.size());
  for (std::size_t k = 0; k < ix.size(); ++k) {
    if (ix[k] < INT32_MIN || ix[k] > INT32_MAX) throw std::invalid_argument("index out of range");
    out[k] = static_cast<int32_t>(ix[k]);
  }
  return out;
}

}  // namespace b200

inline PartitionRange partition(Index n_g, int n, std::int64_t t, int worker) {
  int64_t s = 0, e = 0;
  b200::check(micro_partition(n_g, n, t, worker, &s, &e));
  return PartitionRange{s, e, worker};
}

inline std::size_t global_target_count(double density, Index n_g) {
  uint64_t k = 0;
  b200::check(micro_global_target_count(density, n_g, &k));
  return k;
}

inline std::size_t per_worker_target_count(double density, Index n_g, int n, PerWorkerTarget target) {
  uint64_t k = 0;
  b200::check(micro_per_worker_target_count(density, n_g, n,
                                            target == PerWorkerTarget::full ? MICRO_TARGET_FULL : MICRO_TARGET_SPLIT, &k));
  return k;
}

inline ThresholdState micro_update_threshold(ThresholdState state, std::size_t k_target, std::size_t k_selected,
                                             double alpha, double min_threshold = 1e-12) {
  b200::check(::micro_update_threshold(&state.delta, k_target, k_selected, alpha, min_threshold));
  return state;
}

template <class V>
SparseSelection select_by_threshold(const V& acc, const PartitionRange& range, double delta) {
  const Index n_g = (Index)acc.size();
  const Index m = range.end > range.start ? range.end - range.start : 0;
  if (range.start < 0 || range.end < range.start || range.end > n_g) {
    b200::check(micro_select_by_threshold(MICRO_F64, nullptr, n_g, range.start, range.end, delta, nullptr, nullptr,
                                          0, nullptr, nullptr));  // raises the reference's message
  }
  auto d_acc = b200::upload(acc);
  b200::DeviceBuffer d_idx(sizeof(int32_t) * (std::size_t)(m + 1)), d_val(sizeof(double) * (std::size_t)(m + 1)),
      d_cnt(sizeof(int64_t));
  b200::check(micro_select_by_threshold(MICRO_F64, d_acc.get(), n_g, range.start, range.end, delta,
                                        d_idx.as<int32_t>(), d_val.get(), m, d_cnt.as<int64_t>(), nullptr));
  int64_t k = 0;
  b200::d2h(&k, d_cnt.get(), sizeof k);
  std::vector<int32_t> ix((std::size_t)k);
  SparseSelection out;
  out.values.resize((std::size_t)k);
  if (k) {
    b200::d2h(ix.data(), d_idx.get(), sizeof(int32_t) * (std::size_t)k);
    b200::d2h(out.values.data(), d_val.get(), sizeof(double) * (std::size_t)k);
  }
  out.indices.assign(ix.begin(), ix.end());
  return out;
}

// sparsifier.cpp:39-67 (device radix select; ties to the lower index)
template <class V>
SparseSelection select_topk(const V& acc, const PartitionRange& range, std::size_t k) {
  const Index n_g = (Index)acc.size();
  if (range.start < 0 || range.end < range.start || range.end > n_g)
    b200::check(micro_select_topk(MICRO_F64, nullptr, n_g, range.start, range.end, 0, nullptr, nullptr, 0, nullptr,
                                  nullptr));  // raises the range message
  const Index m = range.end - range.start;
  if ((Index)k > m)
    throw std::invalid_argument("select_topk: k=" + std::to_string(k) + " exceeds range size " + std::to_string(m));
  SparseSelection out;
  if (k == 0) return out;
  auto d_acc = b200::upload(acc);
  b200::DeviceBuffer d_idx(sizeof(int32_t) * (k + 1)), d_val(sizeof(double) * (k + 1)), d_cnt(sizeof(int64_t));
  b200::check(micro_select_topk(MICRO_F64, d_acc.get(), n_g, range.start, range.end, (int64_t)k,
                                d_idx.as<int32_t>(), d_val.get(), (int64_t)k, d_cnt.as<int64_t>(), nullptr));
  int64_t c = 0;
  b200::d2h(&c, d_cnt.get(), sizeof c);
  std::vector<int32_t> ix((std::size_t)c);
  out.values.resize((std::size_t)c);
  if (c) {
    b200::d2h(ix.data(), d_idx.get(), sizeof(int32_t) * (std::size_t)c);
    b200::d2h(out.values.data(), d_val.get(), sizeof(double) * (std::size_t)c);
  }
  out.indices.assign(ix.begin(), ix.end());
  return out;
}

// sparsifier.cpp:85-97
template <class V>
SparseSelection cltk_select(const V& acc_leader, std::size_t k_total, int leader, std::int64_t t, int n) {
  if (n < 1 || leader < 0 || leader >= n) throw std::invalid_argument("cltk_select: leader id out of range");
  if (t < 0 || t % n != leader)
    throw std::logic_error("cltk_select: worker " + std::to_string(leader) + " is not the leader at iteration " +
                           std::to_string(t) + " (leader cycles as t mod n)");
  if (k_total > (std::size_t)acc_leader.size()) throw std::invalid_argument("cltk_select: k exceeds gradient count");
  return select_topk(acc_leader, PartitionRange{0, (Index)acc_leader.size(), leader}, k_total);
}

// sparsifier.cpp:103-108: every index with its value (a copy; no arithmetic)
template <class V>
SparseSelection select_all(const V& acc) {
  SparseSelection out;
  out.indices.resize((std::size_t)acc.size());
  for (std::size_t j = 0; j < out.indices.size(); ++j) out.indices[j] = (Index)j;
  out.values.assign(acc.data(), acc.data() + acc.size());
  return out;
}

// sparsifier.cpp:127-160
inline std::string to_string(SparsifierKind kind) {
  switch (kind) {
    case SparsifierKind::micro: return "micro";
    case SparsifierKind::topk: return "topk";
    case SparsifierKind::cltk: return "cltk";
    case SparsifierKind::hard_threshold: return "hard";
    case SparsifierKind::dense: return "dense";
  }
  throw std::invalid_argument("unknown sparsifier kind");
}
inline SparsifierKind parse_sparsifier_kind(const std::string& name) {
  if (name == "micro") return SparsifierKind::micro;
  if (name == "topk") return SparsifierKind::topk;
  if (name == "cltk") return SparsifierKind::cltk;
  if (name == "hard" || name == "hard_threshold") return SparsifierKind::hard_threshold;
  if (name == "dense") return SparsifierKind::dense;
  throw std::invalid_argument("unknown sparsifier '" + name + "' (expected micro|topk|cltk|hard|dense)");
}
inline std::string to_string(PerWorkerTarget target) { return target == PerWorkerTarget::split ? "split" : "full"; }
inline PerWorkerTarget parse_per_worker_target(const std::string& name) {
  if (name == "split") return PerWorkerTarget::split;
  if (name == "full") return PerWorkerTarget::full;
  throw std::invalid_argument("unknown per-worker target '" + name + "' (expected split|full)");
}

template <class V>
SparseSelection hard_threshold_select(const V& acc, double delta_fixed) {
  return select_by_threshold(acc, PartitionRange{0, (Index)acc.size(), 0}, delta_fixed);
}

template <class V1, class V2>
GradientVector accumulate(const V1& residual, double eta, const V2& grad) {
  if (residual.size() != grad.size())
    throw std::invalid_argument("accumulate: length mismatch (" + std::to_string(residual.size()) + " vs " +
                                std::to_string(grad.size()) + ")");
  const Index n = (Index)residual.size();
  auto d_e = b200::upload(residual);
  auto d_g = b200::upload(grad);
  b200::DeviceBuffer d_out(sizeof(double) * (std::size_t)(n + 1));
  b200::check(micro_accumulate(MICRO_F64, d_e.get(), eta, d_g.get(), d_out.get(), n, nullptr));
  GradientVector out = b200::make_vector(n);
  b200::d2h(out.data(), d_out.get(), sizeof(double) * (std::size_t)n);
  return out;
}

template <class V>
GradientVector compensate(const V& acc, std::span<const Index> selected) {
  const Index n = (Index)acc.size();
  auto d_acc = b200::upload(acc);
  const auto ix = b200::to_i32(std::vector<Index>(selected.begin(), selected.end()));
  b200::DeviceBuffer d_ix(sizeof(int32_t) * (ix.size() + 1));
  if (!ix.empty()) b200::h2d(d_ix.get(), ix.data(), sizeof(int32_t) * ix.size());
  b200::check(micro_compensate(MICRO_F64, d_acc.get(), n, d_ix.as<int32_t>(), (int64_t)ix.size(), nullptr));
  GradientVector out = b200::make_vector(n);
  b200::d2h(out.data(), d_acc.get(), sizeof(double) * (std::size_t)n);
  return out;
}

template <class V>
GradientVector compensate(const V& acc, const SparseSelection& selected) {
  return compensate(acc, std::span<const Index>(selected.indices));
}

inline AggregatedSelection all_gather_indices(const std::vector<SparseSelection>& selections) {
  AggregatedSelection agg;
  std::vector<int64_t> counts;
  std::vector<Index> cat;
  for (const auto& s : selections) {
    counts.push_back((int64_t)s.count());
    agg.per_worker_counts.push_back(s.count());
    cat.insert(cat.end(), s.indices.begin(), s.indices.end());
  }
  if (cat.empty()) return agg;
  const auto c32 = b200::to_i32(cat);
  b200::DeviceBuffer d_cat(sizeof(int32_t) * c32.size()), d_u(sizeof(int32_t) * c32.size());
  b200::h2d(d_cat.get(), c32.data(), sizeof(int32_t) * c32.size());
  int64_t K = 0;
  b200::check(micro_all_gather_indices((int)counts.size(), counts.data(), d_cat.as<int32_t>(), d_u.as<int32_t>(), &K,
                                       nullptr));
  std::vector<int32_t> u((std::size_t)K);
  b200::d2h(u.data(), d_u.get(), sizeof(int32_t) * (std::size_t)K);
  agg.indices.assign(u.begin(), u.end());
  return agg;
}

namespace b200 {
template <class Acc>
std::vector<double> reduce(const std::vector<Acc>& accs, const AggregatedSelection& agg, GradientVector* dense) {
  if (accs.empty()) throw std::invalid_argument("all_reduce_sparse: no workers");
  const Index n_g = (Index)accs.front().size();
  for (const auto& a : accs)
    if ((Index)a.size() != n_g) throw std::invalid_argument("all_reduce_sparse: accumulator length mismatch");
  std::vector<DeviceBuffer> bufs;
  std::vector<const void*> ptrs;
  bufs.reserve(accs.size());
  for (const auto& a : accs) {
    bufs.push_back(upload(a));
    ptrs.push_back(bufs.back().get());
  }
  const auto u = to_i32(agg.indices);
  DeviceBuffer d_u(sizeof(int32_t) * (u.size() + 1)), d_out(sizeof(double) * ((std::size_t)n_g + u.size() + 1));
  if (!u.empty()) h2d(d_u.get(), u.data(), sizeof(int32_t) * u.size());
  std::vector<double> vals;
  if (dense) {
    check(micro_all_reduce_sparse(MICRO_F64, ptrs.data(), (int)ptrs.size(), n_g, d_u.as<int32_t>(), (int64_t)u.size(),
                                  d_out.get(), nullptr));
    *dense = make_vector(n_g);
    d2h(dense->data(), d_out.get(), sizeof(double) * (std::size_t)n_g);
  } else {
    check(micro_all_reduce_sparse_values(MICRO_F64, ptrs.data(), (int)ptrs.size(), n_g, d_u.as<int32_t>(),
                                         (int64_t)u.size(), d_out.get(), nullptr));
    vals.resize(u.size());
    if (!u.empty()) d2h(vals.data(), d_out.get(), sizeof(double) * u.size());
  }
  return vals;
}
}  // namespace b200

template <class Acc>
GradientVector all_reduce_sparse(const std::vector<Acc>& accumulators, const AggregatedSelection& agg) {
  GradientVector dense;
  b200::reduce(accumulators, agg, &dense);
  return dense;
}

template <class Acc>
std::vector<double> all_reduce_sparse_values(const std::vector<Acc>& accumulators, const AggregatedSelection& agg) {
  return b200::reduce(accumulators, agg, nullptr);
}

inline double buildup_factor(const AggregatedSelection& agg, std::size_t k_target_global) {
  if (agg.total_selected() == 0) return 0.0;
  if (k_target_global == 0) throw std::invalid_argument("buildup_factor: zero target count");
  return static_cast<double>(agg.indices.size()) / static_cast<double>(k_target_global);
}

inline double redundant_traffic_factor(const AggregatedSelection& agg) {
  const std::size_t total = agg.total_selected();
  if (total == 0) return 0.0;
  return static_cast<double>(total) / static_cast<double>(agg.indices.size());
}

inline double actual_density(const AggregatedSelection& agg, Index n_g) {
  if (n_g < 1) throw std::invalid_argument("actual_density: n_g must be positive");
  return static_cast<double>(agg.indices.size()) / static_cast<double>(n_g);
}

// harness.hpp:25-32 / harness.cpp:61-63, 109-110: the step-decay learning
// rate that run_iteration hands to each step (host arithmetic).
struct LrSchedule {
  double initial = 0.01;
  double decay_factor = 0.1;
  std::int64_t decay_at = -1;  // -1: resolved to 3/4 of the run
};
inline std::int64_t resolve_decay_at(const LrSchedule& lr, std::int64_t iterations) {
  return lr.decay_at >= 0 ? lr.decay_at : (3 * iterations) / 4;
}
inline double learning_rate_at(const LrSchedule& lr, std::int64_t decay_at, std::int64_t t) {
  return lr.initial * (t >= decay_at ? lr.decay_factor : 1.0);
}

// error_feedback.hpp:41-48: mean of the per-worker residual norms (each
// ||e_i||^2 a deterministic fp64 tree sum on the device; the reference's
// Eigen summation order is not pinned, so agreement is to ~1e-15 relative).
template <class Vec>
double error_metric(const std::vector<Vec>& residuals) {
  if (residuals.empty()) throw std::invalid_argument("error_metric: no workers");
  const Index n_g = (Index)residuals.front().size();
  std::vector<b200::DeviceBuffer> bufs;
  std::vector<const void*> ptrs;
  bufs.reserve(residuals.size());
  for (const auto& e : residuals) {
    if ((Index)e.size() != n_g) throw std::invalid_argument("error_metric: residual length mismatch");
    bufs.push_back(b200::upload(e));
    ptrs.push_back(bufs.back().get());
  }
  double out = 0.0;
  b200::check(micro_error_metric(MICRO_F64, ptrs.data(), (int)ptrs.size(), n_g, &out, nullptr));
  return out;
}

namespace b200 {
// metrics.hpp:15-29.  The MiCRO path fills t, the four scalars and the
// threshold; loss and the modeled phase times belong to the simulator's task
// and cost model (outside this path) and stay 0.  (Own type so that this
// header can sit next to the reference's metrics.hpp: MicroEngine::records
// fills the reference's sparsim::IterationRecord just as well.)
struct IterationRecord {
  std::int64_t t = 0;
  double actual_density = 0.0;
  double buildup_factor = 0.0;
  double redundant_traffic_factor = 0.0;
  double error_norm = 0.0;
  double threshold = 0.0;
  double loss = 0.0;
  double time_grad = 0.0;
  double time_select = 0.0;
  double time_comm = 0.0;
  double time_overhead = 0.0;
};
}  // namespace b200

// The per-iteration MiCRO step of run_iteration (harness.cpp:121-224) for
// `workers` in-process workers on one device, with their residuals and
// thresholds resident in HBM.  step() takes host gradients (workers * n_g,
// worker-major), returns the aggregated selection and the reduced sums
// (what all_gather_indices + all_reduce_sparse_values return), and leaves
// e_{i,t+1} and delta_{i,t+1} on the device.
class MicroEngine {
 public:
  // grad_dtype MICRO_GRAD_F32 (with dtype MICRO_F64): step() takes fp32
  // gradients; state and arithmetic stay fp64 (include/micro.h).
  MicroEngine(Index n_g, int workers, const SparsifierConfig& sc, bool error_feedback = true, int dtype = MICRO_F64,
              int grad_dtype = MICRO_GRAD_SAME)
      : n_g_(n_g), n_(workers), esz_(dtype == MICRO_F64 ? 8 : 4) {
    micro_config cfg;
    micro_config_default(&cfg);
    cfg.n_g = n_g;
    cfg.n_workers = workers;
    cfg.n_local = workers;
    cfg.dtype = dtype;
    cfg.grad_dtype = grad_dtype;
    cfg.density = sc.density;
    cfg.initial_threshold = sc.initial_threshold;
    cfg.scaling_factor = sc.scaling_factor;
    cfg.min_threshold = sc.min_threshold;
    cfg.target = sc.target == PerWorkerTarget::full ? MICRO_TARGET_FULL : MICRO_TARGET_SPLIT;
    cfg.error_feedback = error_feedback ? 1 : 0;
    cfg.sparsifier = (int32_t)sc.kind;  // SparsifierKind order == MICRO_MICRO..MICRO_DENSE
    cfg.device = b200::device();
    b200::check(micro_ctx_create(&ctx_, &cfg, nullptr));
  }
  MicroEngine(const MicroEngine&) = delete;
  MicroEngine& operator=(const MicroEngine&) = delete;
  ~MicroEngine() {
    micro_ctx_destroy(ctx_);
    micro_host_free(h_idx_);
    micro_host_free(h_sums_);
  }

  // h_grads: workers * n_g elements of the engine's dtype (double for MICRO_F64),
  // or float with grad_dtype MICRO_GRAD_F32.
  AggregatedSelection step(const void* h_grads, double eta, std::int64_t t, std::vector<double>* summed = nullptr) {
    if (!h_idx_) {  // pinned result buffers, allocated once (full-bandwidth D2H, no per-step zeroing)
      b200::check(micro_host_malloc(reinterpret_cast<void**>(&h_idx_), (int64_t)n_g_ * 4));
      b200::check(micro_host_malloc(&h_sums_, (int64_t)n_g_ * (int64_t)esz_));
    }
    int64_t K = 0;
    b200::check(micro_step_host(ctx_, h_grads, eta, t, h_idx_, h_sums_, n_g_, &K));
    const unsigned char* sums = static_cast<const unsigned char*>(h_sums_);
    AggregatedSelection agg;
    agg.indices.assign(h_idx_, h_idx_ + K);
    std::vector<int64_t> counts((std::size_t)n_);
    b200::check(micro_query(ctx_, nullptr, counts.data(), nullptr));
    for (auto c : counts) agg.per_worker_counts.push_back((std::size_t)c);
    if (summed) {
      summed->resize((std::size_t)K);
      for (int64_t k = 0; k < K; ++k)
        (*summed)[(std::size_t)k] = esz_ == 8 ? reinterpret_cast<const double*>(sums)[k]
                                              : reinterpret_cast<const float*>(sums)[k];
    }
    return agg;
  }

  // Back to t = 0 (residuals 0, thresholds delta_0).  Needed after a
  // non-finite gradient: the reference throws before its accumulator replaces
  // the residual (harness.cpp:128-130, :223); here K1 has already streamed the
  // NaN/Inf into e_{t+1}, so the engine refuses to step until reset.
  void reset() { b200::check(micro_ctx_reset(ctx_)); }

  std::vector<ThresholdState> thresholds() const {
    std::vector<double> d((std::size_t)n_);
    b200::check(micro_query(ctx_, nullptr, nullptr, d.data()));
    std::vector<ThresholdState> out;
    for (double v : d) out.push_back(ThresholdState{v});
    return out;
  }

  GradientVector residual(int worker) const {
    std::vector<unsigned char> raw((std::size_t)n_g_ * esz_);
    b200::check(micro_copy_residual(ctx_, worker, raw.data()));
    GradientVector out = b200::make_vector(n_g_);
    for (Index j = 0; j < n_g_; ++j)
      out[(std::size_t)j] = esz_ == 8 ? reinterpret_cast<const double*>(raw.data())[j]
                                      : reinterpret_cast<const float*>(raw.data())[j];
    return out;
  }

  // Records of the last min(max_steps, 4096) steps, oldest first; Rec is any
  // type with IterationRecord's field names (e.g. the reference's own).
  template <class Rec = b200::IterationRecord>
  std::vector<Rec> records(std::int64_t max_steps = 4096) const {
    std::vector<micro_record> raw((std::size_t)std::max<std::int64_t>(max_steps, 1));
    std::int64_t w = 0;
    b200::check(micro_records(ctx_, max_steps, raw.data(), &w));
    std::vector<Rec> out((std::size_t)w);
    for (std::int64_t s = 0; s < w; ++s) {
      const micro_record& r = raw[(std::size_t)s];
      Rec& o = out[(std::size_t)s];
      o.t = r.t;
      o.actual_density = r.actual_density;
      o.buildup_factor = r.buildup_factor;
      o.redundant_traffic_factor = r.redundant_traffic_factor;
      o.error_norm = r.error_norm;
      o.threshold = r.threshold;
    }
    return out;
  }

  micro_ctx* handle() const { return ctx_; }

 private:
  micro_ctx* ctx_ = nullptr;
  Index n_g_;
  int n_;
  std::size_t esz_;
  int32_t* h_idx_ = nullptr;  // pinned step results (lazily allocated)
  void* h_sums_ = nullptr;
};

// The same step with one GPU per worker, driven from one process
// (micro_group_*): rank r's context lives on devices[r]; the exchange reads
// the peers' buffers directly (NVLink) between event barriers.  step() takes
// one device gradient pointer per rank (on that rank's device) and enqueues
// the whole iteration without blocking; sync() waits for it.
class MicroGroup {
 public:
  MicroGroup(Index n_g, const std::vector<int>& devices, const SparsifierConfig& sc, bool error_feedback = true,
             int dtype = MICRO_F32, int grad_dtype = MICRO_GRAD_SAME)
      : n_((int)devices.size()) {
    if (n_ < 2) throw std::invalid_argument("MicroGroup: need at least two ranks");
    ctxs_.assign((std::size_t)n_, nullptr);
    for (int r = 0; r < n_; ++r) {
      micro_config cfg;
      micro_config_default(&cfg);
      cfg.n_g = n_g;
      cfg.n_workers = n_;
      cfg.n_local = 1;
      cfg.rank = r;
      cfg.dtype = dtype;
      cfg.grad_dtype = grad_dtype;
      cfg.density = sc.density;
      cfg.initial_threshold = sc.initial_threshold;
      cfg.scaling_factor = sc.scaling_factor;
      cfg.min_threshold = sc.min_threshold;
      cfg.target = sc.target == PerWorkerTarget::full ? MICRO_TARGET_FULL : MICRO_TARGET_SPLIT;
      cfg.error_feedback = error_feedback ? 1 : 0;
      cfg.device = devices[(std::size_t)r];
      b200::check(micro_ctx_create(&ctxs_[(std::size_t)r], &cfg, nullptr));
    }
    b200::check(micro_group_attach(ctxs_.data(), n_));
  }
  MicroGroup(const MicroGroup&) = delete;
  MicroGroup& operator=(const MicroGroup&) = delete;
  ~MicroGroup() {
    for (auto* c : ctxs_) micro_ctx_destroy(c);
  }

  void step(const std::vector<const void*>& d_grads, double eta, std::int64_t t) {
    if ((int)d_grads.size() != n_) throw std::invalid_argument("MicroGroup::step: one gradient per rank");
    b200::check(micro_group_step(ctxs_.data(), n_, d_grads.data(), eta, t));
  }
  void sync() {
    for (auto* c : ctxs_) b200::check(micro_sync(c));
  }
  micro_ctx* rank(int r) const { return ctxs_.at((std::size_t)r); }

 private:
  int n_;
  std::vector<micro_ctx*> ctxs_;
};

}  // namespace sparsim
