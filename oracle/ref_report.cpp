// ref_report.cpp — TEST INFRASTRUCTURE ONLY (the checker for report.py).
//
// An extern "C" face over the reference's own record writer,
// /root/reference/proj/src/report.cpp compiled VERBATIM (oracle/Makefile)
// with the nlohmann/json single header found in this image.  The wrapper
// only marshals plain arrays into the reference's RunConfig /
// IterationRecord and calls sparsim::emit.  task.cpp (which owns
// to_string(TaskKind)) needs the full Eigen Dense API and is not built, so
// the three task names are restated here (task.cpp:348-355).
#include "sparsim/harness.hpp"
#include "sparsim/report.hpp"

#include <cstdint>
#include <exception>
#include <string>
#include <vector>

namespace sparsim {
std::string_view to_string(TaskKind kind) {  // task.cpp:348-355
  switch (kind) {
    case TaskKind::quadratic: return "quadratic";
    case TaskKind::logistic_regression: return "logreg";
    case TaskKind::mlp2: return "mlp2";
  }
  return "?";
}
}  // namespace sparsim

using namespace sparsim;

extern "C" {

// cols: n rows of (actual_density, buildup_factor, redundant_traffic_factor,
// error_norm, threshold, loss, time_grad, time_select, time_comm,
// time_overhead); ints: workers, iterations, batch_size, seed, task,
// dimension, samples, target, decay_at, error_feedback, kind;
// dbls: density, delta0, alpha, eps_delta, lr, decay_factor,
// latency_per_collective, bytes_per_element, bandwidth, compute_time_per_op.
int ref_emit(int fmt, const char* path, const std::int64_t* t, const double* cols, std::int64_t n,
             const std::int64_t* ints, const double* dbls) {
  try {
    RunConfig c;
    c.workers = (int)ints[0];
    c.iterations = ints[1];
    c.batch_size = (Index)ints[2];
    c.seed = (std::uint64_t)ints[3];
    c.task = (TaskKind)ints[4];
    c.dimension = (Index)ints[5];
    c.samples = (Index)ints[6];
    c.sparsifier.target = (PerWorkerTarget)ints[7];
    c.lr.decay_at = ints[8];
    c.error_feedback = ints[9] != 0;
    c.sparsifier.kind = (SparsifierKind)ints[10];
    c.sparsifier.density = dbls[0];
    c.sparsifier.initial_threshold = dbls[1];
    c.sparsifier.scaling_factor = dbls[2];
    c.sparsifier.min_threshold = dbls[3];
    c.lr.initial = dbls[4];
    c.lr.decay_factor = dbls[5];
    c.cost_model.latency_per_collective = dbls[6];
    c.cost_model.bytes_per_element = dbls[7];
    c.cost_model.bandwidth = dbls[8];
    c.compute_time_per_op = dbls[9];
    std::vector<IterationRecord> recs((std::size_t)n);
    for (std::int64_t s = 0; s < n; ++s) {
      const double* r = cols + s * 10;
      IterationRecord& o = recs[(std::size_t)s];
      o.t = t[s];
      o.actual_density = r[0];
      o.buildup_factor = r[1];
      o.redundant_traffic_factor = r[2];
      o.error_norm = r[3];
      o.threshold = r[4];
      o.loss = r[5];
      o.time_grad = r[6];
      o.time_select = r[7];
      o.time_comm = r[8];
      o.time_overhead = r[9];
    }
    emit(c, recs, fmt == 0 ? RecordFormat::csv : RecordFormat::json, path);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"
