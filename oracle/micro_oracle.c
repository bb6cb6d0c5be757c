/*
 * micro_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C, scalar restatement of the reference's MiCRO hot path, written
 * once per element type (float = the GPU path's contract, double = the
 * reference's own precision).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library.
 *
 * Chain of trust:
 *   orc_*_f64  == reference TUs compiled verbatim (oracle/_ref) bit for bit
 *   orc_*_f32  == the GPU path bit for bit
 * Parity is pinned: tests/test_oracle_vs_ref.py runs both against the
 * reference's own compiled code and the golden vectors in tests/golden/.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  Build with -ffp-contract=off and
 * without -ffast-math/-march: `acc = e + eta*G` is two
 * roundings, never an FMA.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/micro_synth.h"

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENONFINITE 3
#define ORC_ENOMEM 7

static __thread char orc_msg[512];

const char* orc_last_error(void) { return orc_msg; }

static int orc_fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static int orc_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(orc_msg, sizeof orc_msg, fmt, ap);
  va_end(ap);
  return code;
}

/* include/sparsim/tensor.hpp:48-63 — cyclic balanced contiguous partition. */
int orc_partition(int64_t n_g, int n, int64_t t, int worker, int64_t* start, int64_t* end) {
  if (n < 1) return orc_fail(ORC_EINVAL, "partition: need at least one worker");
  if (n_g < n)
    return orc_fail(ORC_EINVAL, "partition: vector length %lld smaller than worker count %d",
                    (long long)n_g, n);
  if (worker < 0 || worker >= n)
    return orc_fail(ORC_EINVAL, "partition: worker id %d out of range", worker);
  if (t < 0) return orc_fail(ORC_EINVAL, "partition: negative iteration");
  const int64_t cycle = (t % n + worker) % n;          /* tensor.hpp:57 */
  const int64_t base = n_g / n, rem = n_g % n;         /* tensor.hpp:58-59 */
  const int64_t s = cycle * base + (cycle < rem ? cycle : rem);
  const int64_t len = base + (cycle < rem ? 1 : 0);    /* tensor.hpp:60-61 */
  *start = s;
  *end = s + len;
  return ORC_OK;
}

/* src/sparsifier.cpp:110-116 */
int orc_global_target_count(double density, int64_t n_g, uint64_t* k) {
  if (!(density > 0.0 && density <= 1.0)) return orc_fail(ORC_EINVAL, "density must lie in (0, 1]");
  if (n_g < 1) return orc_fail(ORC_EINVAL, "global_target_count: empty gradient vector");
  const long long r = llround(density * (double)n_g);
  *k = (uint64_t)(r > 1 ? r : 1);
  return ORC_OK;
}

/* src/sparsifier.cpp:118-125; target 0 = split, 1 = full */
int orc_per_worker_target_count(double density, int64_t n_g, int n, int target, uint64_t* k) {
  if (n < 1) return orc_fail(ORC_EINVAL, "per_worker_target_count: need at least one worker");
  if (target == 1) return orc_global_target_count(density, n_g, k);
  if (!(density > 0.0 && density <= 1.0)) return orc_fail(ORC_EINVAL, "density must lie in (0, 1]");
  const long long r = llround(density * (double)n_g / n);
  *k = (uint64_t)(r > 1 ? r : 1);
  return ORC_OK;
}

/* src/sparsifier.cpp:69-83 */
int orc_update_threshold(double* delta, uint64_t k_target, uint64_t k_selected, double alpha,
                         double min_threshold) {
  if (!(alpha > 0.0 && alpha < 1.0))
    return orc_fail(ORC_EINVAL, "micro_update_threshold: alpha must lie in (0, 1)");
  if (!(*delta >= 0.0)) return orc_fail(ORC_EINVAL, "micro_update_threshold: negative threshold");
  if (k_selected > k_target)
    *delta = *delta == 0.0 ? min_threshold : *delta * (1.0 + alpha);
  else if (k_selected < k_target)
    *delta *= 1.0 - alpha;
  return ORC_OK;
}

/* Host copy of the synthetic-gradient spec (include/micro_synth.h). */
void orc_gaussian(uint64_t seed, uint32_t worker, uint64_t t, int64_t n, float* out) {
  float z[4];
  for (int64_t q = 0; q * 4 < n; ++q) {
    ms_gaussian4(seed, worker, t, (uint64_t)q, z);
    for (int c = 0; c < 4 && q * 4 + c < n; ++c) out[q * 4 + c] = z[c];
  }
}

/* src/collectives.cpp:14-28 — concat in worker order, sort, unique.
 * sel_idx: n rows, row i holds counts[i] indices in ascending order (every
 * selection here is: sparsifier.cpp:29-35), so sort + unique of the
 * concatenation is the n-way merge of the rows with duplicates dropped —
 * the same sorted unique union in O(K n) instead of O(K log K).
 * Returns the union size in *K. */
int orc_all_gather_indices(int n, const int64_t* counts, const int64_t* const* sel_idx,
                           int64_t* union_idx, int64_t* K) {
  int64_t pos[64] = {0};
  int64_t w = 0;
  if (n > 64) return orc_fail(ORC_EINVAL, "all_gather_indices: at most 64 workers");
  for (;;) {
    int best = -1;
    int64_t v = 0;
    for (int i = 0; i < n; ++i)
      if (pos[i] < counts[i] && (best < 0 || sel_idx[i][pos[i]] < v)) {
        best = i;
        v = sel_idx[i][pos[i]];
      }
    if (best < 0) break;
    ++pos[best];
    if (w == 0 || union_idx[w - 1] != v) union_idx[w++] = v;
  }
  *K = w;
  return ORC_OK;
}

static int64_t* orc_union_idx = NULL;
static float* orc_union_sum_f32 = NULL;
static double* orc_union_sum_f64 = NULL;

/* The union kept by the last orc_step_* call made with union_idx == NULL. */
int orc_fetch_union_f32(int64_t* idx, float* sum, int64_t K) {
  if (K) { memcpy(idx, orc_union_idx, (size_t)K * 8); memcpy(sum, orc_union_sum_f32, (size_t)K * 4); }
  return ORC_OK;
}
int orc_fetch_union_f64(int64_t* idx, double* sum, int64_t K) {
  if (K) { memcpy(idx, orc_union_idx, (size_t)K * 8); memcpy(sum, orc_union_sum_f64, (size_t)K * 8); }
  return ORC_OK;
}

#define DEFINE_ORACLE(T, SUF, ABS, ISFINITE)                                                    \
  /* src/sparsifier.cpp:22-37: ascending scan, strict (double)|acc| > delta */                \
  int orc_select_##SUF(const T* acc, int64_t n_g, int64_t start, int64_t end, double delta,     \
                       int64_t* idx, T* val, int64_t* count) {                                  \
    if (start < 0 || end < start || end > n_g)                                                  \
      return orc_fail(ORC_EINVAL, "selection: range [%lld, %lld) invalid for vector of length %lld", \
                      (long long)start, (long long)end, (long long)n_g);                        \
    if (!(delta >= 0.0) || !isfinite(delta))                                                    \
      return orc_fail(ORC_EINVAL, "selection: threshold must be finite and nonnegative");       \
    int64_t k = 0;                                                                              \
    for (int64_t j = start; j < end; ++j) {                                                     \
      const T v = acc[j];                                                                       \
      if ((double)ABS(v) > delta) {                                                             \
        idx[k] = j;                                                                             \
        val[k] = v;                                                                             \
        ++k;                                                                                    \
      }                                                                                         \
    }                                                                                           \
    *count = k;                                                                                 \
    return ORC_OK;                                                                              \
  }                                                                                             \
                                                                                                \
  /* src/collectives.cpp:30-49: sum = 0; for every worker in order: sum += acc_i[j] */         \
  int orc_all_reduce_sparse_values_##SUF(const T* accs, int n, int64_t n_g,                     \
                                         const int64_t* union_idx, int64_t K, T* sums) {        \
    if (n < 1) return orc_fail(ORC_EINVAL, "all_reduce_sparse: no workers");                    \
    for (int64_t k = 0; k < K; ++k) {                                                           \
      const int64_t j = union_idx[k];                                                           \
      if (j < 0 || j >= n_g)                                                                    \
        return orc_fail(ORC_EINVAL, "all_reduce_sparse: index %lld out of range", (long long)j); \
      T s = (T)0;                                                                               \
      for (int i = 0; i < n; ++i) s += accs[(int64_t)i * n_g + j];                              \
      sums[k] = s;                                                                              \
    }                                                                                           \
    return ORC_OK;                                                                              \
  }                                                                                             \
                                                                                                \
  /* One MiCRO iteration for n in-process workers, src/harness.cpp:121-224 order.              \
   * e: n*n_g residuals (in: e_t, out: e_{t+1}); G: n*n_g gradients; delta: n thresholds      \
   * (in: delta_t, out: delta_{t+1}); x: optional n_g model (x -= sum/n at the union).        \
   * Outputs: counts[n] = k_i, union_idx/union_sum[K] (cap n_g), delta_used[n]. */             \
  int orc_step_##SUF(int64_t n_g, int n, double density, double alpha, double min_threshold,    \
                     int target, int error_feedback, int64_t t, double eta, T* e, const T* G,   \
                     double* delta, T* x, int64_t* counts, int64_t* union_idx, T* union_sum,    \
                     int64_t* K, double* delta_used) {                                          \
    if (n < 1 || n_g < n) return orc_fail(ORC_EINVAL, "run config: bad n_g/n");                 \
    uint64_t k_worker;                                                                          \
    int rc = orc_per_worker_target_count(density, n_g, n, target, &k_worker);                   \
    if (rc) return rc;                                                                          \
    const T eta_t = (T)eta;                                                                     \
    /* harness.cpp:123-132: finite check, acc_i = e_i + eta*G_i (two roundings, in place) */    \
    /* (all gradients are checked before any residual is touched: the reference's        \
     * accumulators are scratch, so a throw leaves e_t intact) */                              \
    for (int i = 0; i < n; ++i) {                                                               \
      const T* g = G + (int64_t)i * n_g;                                                        \
      for (int64_t j = 0; j < n_g; ++j)                                                         \
        if (!ISFINITE(g[j]))                                                                    \
          return orc_fail(ORC_ENONFINITE, "iteration %lld: non-finite gradient on worker %d",   \
                          (long long)t, i);                                                     \
    }                                                                                           \
    for (int i = 0; i < n; ++i) {                                                               \
      const T* g = G + (int64_t)i * n_g;                                                        \
      T* a = e + (int64_t)i * n_g;                                                              \
      for (int64_t j = 0; j < n_g; ++j) {                                                       \
        const T p = eta_t * g[j];                                                               \
        a[j] = a[j] + p;                                                                        \
      }                                                                                         \
    }                                                                                           \
    /* harness.cpp:139-151: select in the cyclic partition with this worker's delta    \
     * (buffers sized to the selection: one counting pass, then the scan itself) */       \
    int64_t total = 0;                                                                      \
    for (int i = 0; i < n; ++i) {                                                           \
      int64_t s, en;                                                                        \
      orc_partition(n_g, n, t, i, &s, &en);                                                 \
      if (!(delta[i] >= 0.0) || !isfinite(delta[i]))                                        \
        return orc_fail(ORC_EINVAL, "selection: threshold must be finite and nonnegative"); \
      const T* a = e + (int64_t)i * n_g;                                                    \
      for (int64_t j = s; j < en; ++j) total += (double)ABS(a[j]) > delta[i];               \
    }                                                                                       \
    int64_t* sel_idx = (int64_t*)malloc((size_t)(total + 1) * sizeof(int64_t));            \
    T* sel_val = (T*)malloc((size_t)(total + 1) * sizeof(T));                               \
    const int64_t** rows = (const int64_t**)malloc((size_t)n * sizeof(int64_t*));           \
    if (!sel_idx || !sel_val || !rows) {                                                    \
      free(sel_idx); free(sel_val); free(rows);                                             \
      return orc_fail(ORC_ENOMEM, "oracle: out of memory");                                 \
    }                                                                                       \
    int64_t off = 0;                                                                        \
    for (int i = 0; i < n; ++i) {                                                           \
      int64_t s, en, k;                                                                     \
      orc_partition(n_g, n, t, i, &s, &en);                                                 \
      delta_used[i] = delta[i];                                                             \
      rc = orc_select_##SUF(e + (int64_t)i * n_g, n_g, s, en, delta[i], sel_idx + off,      \
                            sel_val + off, &k);                                             \
      if (rc) { free(sel_idx); free(sel_val); free(rows); return rc; }                      \
      rows[i] = sel_idx + off;                                                              \
      counts[i] = k;                                                                        \
      off += k;                                                                             \
    }                                                                                       \
    /* harness.cpp:185-186: all_gather_indices, all_reduce_sparse_values.  With            \
     * union_idx == NULL the union is kept here (sized to it) for orc_fetch_union_*. */     \
    if (!union_idx) {                                                                       \
      free(orc_union_idx); free(orc_union_sum_##SUF);                                       \
      orc_union_idx = (int64_t*)malloc((size_t)(total + 1) * sizeof(int64_t));             \
      orc_union_sum_##SUF = (T*)malloc((size_t)(total + 1) * sizeof(T));                    \
      if (!orc_union_idx || !orc_union_sum_##SUF) {                                         \
        free(sel_idx); free(sel_val); free(rows);                                           \
        return orc_fail(ORC_ENOMEM, "oracle: out of memory");                               \
      }                                                                                     \
      union_idx = orc_union_idx;                                                            \
      union_sum = orc_union_sum_##SUF;                                                      \
    }                                                                                       \
    orc_all_gather_indices(n, counts, rows, union_idx, K);                                  \
    orc_all_reduce_sparse_values_##SUF(e, n, n_g, union_idx, *K, union_sum);                \
    /* harness.cpp:201-208: threshold estimate for t+1 with this iteration's count */           \
    for (int i = 0; i < n; ++i)                                                                 \
      orc_update_threshold(&delta[i], k_worker, (uint64_t)counts[i], alpha, min_threshold);     \
    /* harness.cpp:212-215: x[j] -= summed / n (true division) */                               \
    if (x)                                                                                      \
      for (int64_t k = 0; k < *K; ++k) x[union_idx[k]] -= union_sum[k] / (T)n;                 \
    /* harness.cpp:219-224: zero every union index on every worker; EF off -> zero all */       \
    for (int i = 0; i < n; ++i) {                                                               \
      T* a = e + (int64_t)i * n_g;                                                              \
      for (int64_t k = 0; k < *K; ++k) a[union_idx[k]] = (T)0;                                  \
      if (!error_feedback) memset(a, 0, (size_t)n_g * sizeof(T));                               \
    }                                                                                           \
    free(sel_idx); free(sel_val); free(rows);                                                   \
    return ORC_OK;                                                                              \
  }

DEFINE_ORACLE(float, f32, fabsf, isfinite)
DEFINE_ORACLE(double, f64, fabs, isfinite)
