// api.cu — the C ABI's engine half (include/micro.h): the MiCRO context,
// K1 launch plumbing, the single-device cluster, the comparison sparsifiers
// and the host-side bookkeeping around the sm_100a kernels.  No CPU compute
// path exists: every array operation is a device kernel; the host only
// validates, sizes launches and moves small scalars.
// (dist_api.cu: one rank of an n-GPU job; value_api.cu: stateless calls.)
#include <type_traits>
#include "internal.cuh"

using namespace micro;
using namespace micro::host;

// ---------------------------------------------------------------- errors --

namespace micro {
namespace host {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int check_dtype(int dtype) {
  if (dtype != MICRO_F32 && dtype != MICRO_F64) return fail(MICRO_EINVAL, "unknown dtype %d", dtype);
  return MICRO_OK;
}

int num_sms(int dev) {
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = v;
  return v;
}

// ---- pure host restatements (shared by the C ABI and the engine) ----

int h_partition(int64_t n_g, int n, int64_t t, int worker, int64_t* start, int64_t* end) {
  if (n < 1) return fail(MICRO_EINVAL, "partition: need at least one worker");
  if (n_g < n)
    return fail(MICRO_EINVAL, "partition: vector length %lld smaller than worker count %d",
                (long long)n_g, n);
  if (worker < 0 || worker >= n)
    return fail(MICRO_EINVAL, "partition: worker id %d out of range", worker);
  if (t < 0) return fail(MICRO_EINVAL, "partition: negative iteration");
  partition_range(n_g, n, t, worker, start, end);
  return MICRO_OK;
}

int h_global_target(double d, int64_t n_g, uint64_t* k) {
  if (!(d > 0.0 && d <= 1.0)) return fail(MICRO_EINVAL, "density must lie in (0, 1]");
  if (n_g < 1) return fail(MICRO_EINVAL, "global_target_count: empty gradient vector");
  const long long r = std::llround(d * static_cast<double>(n_g));
  *k = static_cast<uint64_t>(std::max(1LL, r));
  return MICRO_OK;
}

int h_worker_target(double d, int64_t n_g, int n, int target, uint64_t* k) {
  if (n < 1) return fail(MICRO_EINVAL, "per_worker_target_count: need at least one worker");
  if (target == MICRO_TARGET_FULL) return h_global_target(d, n_g, k);
  if (target != MICRO_TARGET_SPLIT) return fail(MICRO_EINVAL, "unknown per-worker target %d", target);
  if (!(d > 0.0 && d <= 1.0)) return fail(MICRO_EINVAL, "density must lie in (0, 1]");
  const long long r = std::llround(d * static_cast<double>(n_g) / n);
  *k = static_cast<uint64_t>(std::max(1LL, r));
  return MICRO_OK;
}

int h_update_threshold(double* delta, uint64_t k_target, uint64_t k_sel, double alpha, double eps) {
  if (!(alpha > 0.0 && alpha < 1.0))
    return fail(MICRO_EINVAL, "micro_update_threshold: alpha must lie in (0, 1)");
  if (!(*delta >= 0.0)) return fail(MICRO_EINVAL, "micro_update_threshold: negative threshold");
  if (k_sel > k_target)
    *delta = *delta == 0.0 ? eps : *delta * (1.0 + alpha);
  else if (k_sel < k_target)
    *delta *= 1.0 - alpha;
  return MICRO_OK;
}



int read_flags(micro_ctx* c, int* flags) {
  CU(cudaMemcpyAsync(flags, c->flags, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (*flags & 1) c->poisoned = true;
  return MICRO_OK;
}

unsigned grid_for(int64_t work, int dev) {
  const int64_t b = (work + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 8 * num_sms(dev)));
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}


int finalize_blocks(micro_ctx* c) {
  const int64_t want = ((int64_t)c->k_worker * c->n * 3 / 2 + 255) / 256;
  return (int)std::min<int64_t>(std::max<int64_t>(want, 1), 64 * num_sms(c->dev));
}

template <typename T>
int launch_finalize(micro_ctx* c, const int32_t* uidx, const void* usum, int k_from_counts) {
  FinalizeArgs f{};
  f.n = c->n;
  f.n_local = c->n_local;
  f.n_g = c->n_g;
  f.t = c->t_cur;
  f.counts = c->counts;
  f.delta = c->delta;
  f.k_target = c->k_worker;
  f.alpha = c->cfg.scaling_factor;
  f.min_threshold = c->cfg.min_threshold;
  f.k_from_counts = k_from_counts;
  f.cap = c->sel_cap;
  f.K = c->Kbuf + c->buf;
  f.union_idx = uidx;
  f.union_sum = usum;
  const int pb = c->buf ^ 1;
  if (c->ever_stepped && c->dense && !c->dense_fused) {
    f.prev_idx = c->sel_is_union ? c->sel_idx[pb][0] : c->uni_idx[pb];
    f.prev_K = c->Kbuf + pb;
  }
  f.dense = c->dense_fused ? nullptr : c->dense;  // fused: K1 maintained it
  // n = 1 with the streaming K1: k1_gather applied the model update
  f.model = c->sel_is_union ? nullptr : c->model;
  f.update_delta = c->kind == 0;
  if (c->vectors_done) {  // k_dense_all wrote the model and the dense g/n
    f.model = nullptr;
    f.dense = nullptr;
    f.prev_idx = nullptr;
    c->vectors_done = false;
  }
  f.slot = c->steps % kHistCap;
  f.hist_t = c->hist_t;
  f.hist_K = c->hist_K;
  f.hist_counts = c->hist_counts;
  f.hist_delta = c->hist_delta;
  f.hist_err = c->hist_err;
  f.norm_mode = norm_mode(c);
  f.slots = c->norm_slot;
  f.corr = c->n > 1 && c->kind == 0;
  const int blocks = (f.dense || f.model) ? finalize_blocks(c) : 1;  // grid-stride over the union
  if (c->fin_done) {
    // k1_gather already did the threshold update + history (n = 1, micro_step);
    // dense (fused into K1) and model (k1_gather) are done too
    c->fin_done = false;
  } else {
    bool waited = false;  // an event wait or a clear kernel sits between: launch normally
    if (c->clear_pending) {
      CU(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
      c->clear_pending = false;
      waited = true;
    } else if (f.prev_idx) {
      waited = true;
      k_dense_clear<T><<<blocks, 256, 0, c->stream>>>(f.prev_idx, f.prev_K, (T*)c->dense, c->n_g);
      CU(cudaGetLastError());
    }
    CU(launch_maybe_pdl(!waited, k_finalize<T>, dim3(blocks), dim3(256), c->stream, f));
  }
  if (!c->cfg.error_feedback && c->n > 1)
    for (int i = 0; i < c->n_local; ++i) CU(cudaMemsetAsync(c->resid[i], 0, c->n_g * c->esz, c->stream));
  c->steps++;
  c->ever_stepped = true;
  c->compressed = false;
  return MICRO_OK;
}

template int launch_finalize<float>(micro_ctx*, const int32_t*, const void*, int);
template int launch_finalize<double>(micro_ctx*, const int32_t*, const void*, int);



int bitmap_offsets(const unsigned* bitmap, int64_t nwords, int* off, int* tiles, cudaStream_t st, long long* total) {
  const int64_t nt = scan_tiles(nwords);
  k_scan_totals<true><<<(unsigned)nt, kScanThreads, 0, st>>>(bitmap, nwords, tiles);
  CU(cudaGetLastError());
  k_scan_top<<<1, kScanThreads, 0, st>>>(tiles, nt, total);
  CU(cudaGetLastError());
  k_scan_apply<true><<<(unsigned)nt, kScanThreads, 0, st>>>(bitmap, nwords, tiles, off);
  CU(cudaGetLastError());
  return MICRO_OK;
}

int check_ctx(micro_ctx* c) {
  if (!c) return fail(MICRO_EINVAL, "null context");
  return MICRO_OK;
}

int ensure_staging(micro_ctx* c) {
  if (c->staging) return MICRO_OK;
  c->staging_stride = ((size_t)c->n_g * c->gsz + 255) / 256 * 256;
  cudaError_t e = cudaMalloc(&c->staging, c->staging_stride * c->n_local);
  if (e != cudaSuccess) {
    c->staging = nullptr;
    return fail(MICRO_ENOMEM, "gradient staging: %s", cudaGetErrorString(e));
  }
  return MICRO_OK;
}

int check_poison(micro_ctx* c) {
  if (c->poisoned)
    return fail(MICRO_ENONFINITE,
                "context poisoned by a non-finite gradient at iteration %lld; call micro_ctx_reset",
                (long long)c->t_cur);
  return MICRO_OK;
}

}  // namespace host
}  // namespace micro

namespace {

SumSqSlots norm_slots(micro_ctx* c, int i) {
  SumSqSlots q{};
  q.part = c->norm_part;
  q.group = c->norm_group;
  q.ticket = c->norm_ticket;
  q.out = &c->norm_slot[i].sq;
  return q;
}


// ||resid_i||^2 by a standalone pass (K1 variants without the fused sum).
template <typename T>
int launch_sumsq(micro_ctx* c, int i) {
  const int64_t grid = std::min<int64_t>(c->norm_ctas, 4 * (int64_t)num_sms(c->dev));
  k_sumsq<T><<<(unsigned)grid, 256, 0, c->stream>>>((const T*)c->resid[i], c->n_g, norm_slots(c, i));
  CU(cudaGetLastError());
  return MICRO_OK;
}

// Steps whose streamed bytes (e, G read; e written) stay below this prefetch
// the model's selected lines during k1_stream (C1: 140 MB; C3: 1.66 GB does not).
constexpr int64_t kPrefetchStepBytes = 256ll << 20;

template <typename T, typename TG = T>
int launch_k1_stream(micro_ctx* c, int i, const void* grad, double eta, int64_t ps, int64_t pe,
                     const double* thr = nullptr, const long long* tie = nullptr, bool acc_in_e = false) {
  constexpr int UE = stream_unit_elems<T>();
  StreamArgs a{};
  a.grad = grad;
  a.resid = c->resid[i];
  a.n_g = (int)c->n_g;
  a.p_start = (int)ps;
  a.p_end = (int)pe;
  a.eta = eta;
  a.delta = thr ? thr : c->delta + i;
  a.tie_j = tie;
  a.unit_lo = (int)(ps / UE);
  a.unit_hi = (int)((pe - 1) / UE);
  a.stage_idx = c->stage_idx;
  a.stage_val = c->stage_val;
  a.unit_counts = c->unit_counts;
  a.flags = c->flags;
  a.dense = c->dense;
  a.dirty = c->dense_dirty;
  a.super_counts = c->super_counts + c->super_par * kMaxSupers;
  a.super_runs = c->super_runs;
  a.sq_part = c->norm_part;
  a.model = c->model;
  const int units = (int)((c->n_g + UE - 1) / UE);
  const unsigned grid = (unsigned)((units + kStreamWarps - 1) / kStreamWarps);
  const bool fd = c->dense_fused;
  cudaStream_t st = c->stream;
  // every timing_period-th launch (event records between kernels cost the step
  // a few µs at small sizes, so long runs sample)
  const bool timed = c->timing && c->t_next < kTimingCap && (c->t_seen++ % c->timing_period) == 0;
  if (timed) CU(cudaEventRecord(c->t_ev[2 * c->t_next], st));
  auto dispatch = [&](unsigned g) -> int {
#define K1S(MODE, D) \
    CU(launch_pdl(k1_stream<T, MODE, D, false, false, false, false, TG>, dim3(g), dim3(kStreamThreads), st, a))
#define K1N(D)                                                                                              \
    do {                                                                                                      \
      if (c->norm) CU(launch_pdl(k1_stream<T, kWriteZeroSel, D, true, false, false, false, TG>, dim3(g),      \
                                 dim3(kStreamThreads), st, a));                                            \
      else K1S(kWriteZeroSel, D);                                                                             \
    } while (0)
    if (c->norm && (int64_t)grid > c->norm_ctas) return fail(MICRO_ECAPACITY, "norm workspace too small");
    if (c->kind && !c->sel_is_union) {  // comparison sparsifiers: keep acc (the union is zeroed after the reduce)
      if constexpr (std::is_same<T, TG>::value) {  // (fp32 gradients are MiCRO only)
        if (acc_in_e)  // top-k: e holds acc already; compact only
          CU(launch_pdl(k1_stream<T, kWriteNone, false, false, true, true>, dim3(g),
                              dim3(kStreamThreads), st, a));
        else if (tie)
          CU(launch_pdl(k1_stream<T, kWriteAcc, false, false, true>, dim3(g), dim3(kStreamThreads), st, a));
        else K1S(kWriteAcc, false);
      }
    } else if (c->kind && acc_in_e) {  // top-k / CLT-k, one worker: compact acc (in e), zero it, dense g/n
      if constexpr (std::is_same<T, TG>::value) {
#define K1T(D, N) CU(launch_pdl(k1_stream<T, kWriteZeroSel, D, N, true, true>, dim3(g), dim3(kStreamThreads), st, a))
        if (fd && c->norm) K1T(true, true);
        else if (fd) K1T(true, false);
        else if (c->norm) K1T(false, true);
        else K1T(false, false);
#undef K1T
      }
    } else if (c->n > 1) {
      if (c->cfg.error_feedback) K1N(false);
      else K1S(kWriteAcc, false);
    } else if (c->cfg.error_feedback) {
      // small steps: prefetch x's selected lines into L2 for k1_gather's update
      const bool pf = c->model && (int64_t)c->n_g * (int64_t)c->esz * 3 <= kPrefetchStepBytes;
      if (pf) {
#define K1P(D, N) \
  CU(launch_pdl(k1_stream<T, kWriteZeroSel, D, N, false, false, true, TG>, dim3(g), dim3(kStreamThreads), st, a))
        if (fd && c->norm) K1P(true, true);
        else if (fd) K1P(true, false);
        else if (c->norm) K1P(false, true);
        else K1P(false, false);
#undef K1P
      } else if (fd) K1N(true);
      else K1N(false);
    } else {
      if (fd) K1S(kWriteNone, true);
      else K1S(kWriteNone, false);
    }
#undef K1S
#undef K1N
    CU(cudaGetLastError());
    return MICRO_OK;
  };
  if (c->h2d_chunks > 1 && c->sel_is_union && c->kind == 0) {
    // step_host: chunk k of the gradient landed on the copy stream -> stream
    // its CTAs while the next chunk is still in flight over PCIe
    const unsigned per = (grid + c->h2d_chunks - 1) / c->h2d_chunks;
    for (int k = 0; k < c->h2d_chunks; ++k) {
      const unsigned lo = std::min(grid, per * k), hi = std::min(grid, per * (k + 1));
      if (lo >= hi) break;
      CU(cudaStreamWaitEvent(st, c->h2d_ev[k], 0));
      a.cta_offset = (int)lo;
      TRY(dispatch(hi - lo));
    }
    a.cta_offset = 0;
  } else {
    TRY(dispatch(grid));
  }
  if (timed) CU(cudaEventRecord(c->t_ev[2 * c->t_next++ + 1], st));
  CompactArgs b{};
  b.stage_idx = c->stage_idx;
  b.stage_val = c->stage_val;
  b.run_counts = c->unit_counts;
  b.super_counts = a.super_counts;
  c->super_par ^= 1;
  b.super_clear = c->super_counts + c->super_par * kMaxSupers;
  b.super_len = kMaxSupers;
  b.num_runs = a.unit_hi / kStreamWarps - a.unit_lo / kStreamWarps + 1;
  b.super_runs = c->super_runs;
  b.run_stride = kStreamWarps * UE;
  b.sel_idx = c->sel_idx[c->buf][i];
  b.sel_val = c->sel_val[c->buf][i];
  b.cap = c->sel_cap;
  b.count = c->counts + i;
  b.flags = c->flags;
  b.model = c->sel_is_union ? c->model : nullptr;  // n = 1: the union is this selection, g/n = acc
  // (its values are then the union's sums: a selected -0 is stored as +0;
  // the value-level selections keep the raw acc)
  b.sum_from_zero = c->sel_is_union ? 1 : 0;
  if ((b.num_runs + b.super_runs - 1) / b.super_runs > kMaxSupers)
    return fail(MICRO_ECAPACITY, "super-block workspace too small");
  if (c->fuse_step) {
    b.fin_delta = c->delta + i;
    b.fin_fixed = c->kind != 0;
    b.k_target = c->k_worker;
    b.alpha = c->cfg.scaling_factor;
    b.min_threshold = c->cfg.min_threshold;
    b.fin_K = c->Kbuf + c->buf;
    b.fin_t = c->t_cur;
    b.fin_slot = c->steps % kHistCap;
    b.hist_t = c->hist_t;
    b.hist_K = c->hist_K;
    b.hist_counts = c->hist_counts;
    b.hist_delta = c->hist_delta;
    b.hist_err = c->hist_err;
    b.norm_mode = norm_mode(c);
    c->fin_done = true;
  }
  unsigned gblocks = (unsigned)((b.num_runs + kGatherWarps - 1) / kGatherWarps);
  if (c->norm && (c->kind == 0 || c->sel_is_union)) {  // one more CTA reduces k1_stream's per-CTA partials
    b.sq_part = c->norm_part;
    b.sq_parts = (int)grid;
    b.sq_out = &c->norm_slot[i].sq;
    b.hist_err = c->hist_err;
    b.fin_slot = c->steps % kHistCap;
    gblocks += 1;
  }
  if (c->cfg.density >= 0.05)
    CU(launch_pdl(k1_gather<T, false>, dim3(gblocks), dim3(kGatherWarps * 32), c->stream, b));
  else
    CU(launch_pdl(k1_gather<T, true>, dim3(gblocks), dim3(kGatherWarps * 32), c->stream, b));
  return MICRO_OK;
}


// One worker of a comparison sparsifier (harness.cpp:152-181).
template <typename T>
int launch_baseline(micro_ctx* c, int i, const void* grad, double eta, int64_t t) {
  cudaStream_t st = c->stream;
  const int kind = c->kind;
  const int64_t n_g = c->n_g;
  const bool selects = kind == 1 || kind == 3 || (kind == 2 && t % c->n == i);
  const unsigned agrid = grid_for(n_g, c->dev);
  auto accumulate_only = [&](long long count) -> int {
    k_accumulate_probe<T><<<agrid, 256, 0, st>>>((T*)c->resid[i], (const T*)grad, eta, n_g, c->flags);
    CU(cudaGetLastError());
    k_fill_i64<<<1, 32, 0, st>>>(c->counts + i, 1, count);
    CU(cudaGetLastError());
    return MICRO_OK;
  };
  if (!selects) return accumulate_only(kind == 4 ? n_g : 0);
  if (kind == 3) return launch_k1_stream<T>(c, i, grad, eta, 0, n_g);  // |acc| > delta_0 (c->delta[i])
  // top-k (and the CLT-k leader): k_global over the whole vector
  const long long k = (long long)c->k_global;
  if (k == 0) return accumulate_only(0);
  if (k >= n_g) return launch_k1_stream<T>(c, i, grad, eta, 0, n_g, c->minus_one);
  TopkState* ts = c->topk + i;
  k_topk_init<<<1, 1, 0, st>>>(ts, k);
  CU(cudaGetLastError());
  const int bits = KeyOf<T>::kBits;
  const unsigned hgrid = (unsigned)std::min<int64_t>((n_g + 255) / 256, 4 * (int64_t)num_sms(c->dev));
  T* acc = (T*)c->resid[i];
  for (int hi = bits; hi > 0; hi -= kDigitBits) {  // MSB-first digits of <= 11 bits
    const int width = std::min(kDigitBits, hi);
    const int shift = hi - width;
    if (hi == bits)  // the first pass forms acc = e + eta*G once and keeps it in e
      k_topk_hist<T><<<hgrid, 256, 0, st>>>(acc, (const T*)grad, eta, n_g, shift, width, ts, c->topk_hist, acc,
                                            c->flags);
    else  // later passes, ties and the compaction read acc alone
      k_topk_hist<T><<<hgrid, 256, 0, st>>>(acc, nullptr, eta, n_g, shift, width, ts, c->topk_hist);
    CU(cudaGetLastError());
    k_topk_digit<T><<<1, 1024, 0, st>>>(ts, c->topk_hist, shift, width, shift == 0, n_g);
    CU(cudaGetLastError());
  }
  const int64_t chunk = tie_chunk(n_g);
  const int nch = (int)((n_g + chunk - 1) / chunk);
  k_tie_count<T><<<nch, 256, 0, st>>>(acc, nullptr, eta, n_g, chunk, ts, c->tie_counts);
  CU(cudaGetLastError());
  k_tie_find<T><<<1, 1024, 0, st>>>(acc, nullptr, eta, n_g, chunk, nch, ts, c->tie_counts);
  CU(cudaGetLastError());
  return launch_k1_stream<T>(c, i, grad, eta, 0, n_g, &ts->pivot, &ts->tie_j, /*acc_in_e=*/true);
}

// Top-k on every worker of a single-device cluster at once (the batched
// kernels of baselines.cuh: one launch per radix pass for all workers), then
// each worker's compaction with the tie rule, as launch_baseline does.
template <typename T>
int launch_topk_batch(micro_ctx* c, const void* const* grads, double eta) {
  cudaStream_t st = c->stream;
  const int n = c->n_local;
  const int64_t n_g = c->n_g;
  const long long k = (long long)c->k_global;
  TopkBatch b{};
  for (int i = 0; i < n; ++i) {
    b.e[i] = c->resid[i];
    b.g[i] = grads[i];
  }
  k_topk_init_b<<<1, 64, 0, st>>>(c->topk, n, k);
  CU(cudaGetLastError());
  const int bits = KeyOf<T>::kBits;
  const unsigned hgrid = (unsigned)std::min<int64_t>((n_g + 255) / 256, 4 * (int64_t)num_sms(c->dev));
  for (int hi = bits; hi > 0; hi -= kDigitBits) {
    const int width = std::min(kDigitBits, hi);
    const int shift = hi - width;
    k_topk_hist_b<T><<<dim3(hgrid, n), 256, 0, st>>>(b, eta, n_g, shift, width, c->topk, c->topk_hist, hi == bits,
                                                      c->flags);
    CU(cudaGetLastError());
    k_topk_digit_b<T><<<n, 1024, 0, st>>>(c->topk, c->topk_hist, shift, width, shift == 0, n_g);
    CU(cudaGetLastError());
  }
  const int64_t chunk = tie_chunk(n_g);
  const int nch = (int)((n_g + chunk - 1) / chunk);
  k_tie_count_b<T><<<dim3(nch, n), 256, 0, st>>>(b, n_g, chunk, c->topk, c->tie_counts);
  CU(cudaGetLastError());
  k_tie_find_b<T><<<n, 1024, 0, st>>>(b, n_g, chunk, nch, c->topk, c->tie_counts);
  CU(cudaGetLastError());
  for (int i = 0; i < n; ++i) {
    TopkState* ts = c->topk + i;
    TRY(launch_k1_stream<T>(c, i, grads[i], eta, 0, n_g, &ts->pivot, &ts->tie_j, /*acc_in_e=*/true));
  }
  return MICRO_OK;
}

template <typename T>
int launch_k1(micro_ctx* c, int i, const void* grad, double eta, int64_t t) {
  if (c->kind) return launch_baseline<T>(c, i, grad, eta, t);  // grad realigned by micro_compress
  int64_t ps, pe;
  partition_range(c->n_g, c->n, t, c->cfg.rank + i, &ps, &pe);
  if constexpr (std::is_same<T, double>::value)
    if (c->gsz == 4) return launch_k1_stream<double, float>(c, i, grad, eta, ps, pe);  // fp32 gradients
  return launch_k1_stream<T>(c, i, grad, eta, ps, pe);
}

// Clear the previous union's sectors of the dense g/n on the aux stream, so
// the (small, latency-bound) clear overlaps the HBM-bound K1.
template <typename T>
int fork_dense_clear(micro_ctx* c) {
  if (!c->dense || c->dense_fused || !c->ever_stepped || !c->aux || c->kind == 4) return MICRO_OK;
  const int pb = c->buf ^ 1;
  const int32_t* prev = c->sel_is_union ? c->sel_idx[pb][0] : c->uni_idx[pb];
  CU(cudaEventRecord(c->ev_fork, c->stream));
  CU(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
  k_dense_clear<T><<<finalize_blocks(c), 256, 0, c->aux>>>(prev, c->Kbuf + pb, (T*)c->dense, c->n_g);
  CU(cudaGetLastError());
  CU(cudaEventRecord(c->ev_join, c->aux));
  c->clear_pending = true;
  return MICRO_OK;
}

// Union (sorted unique of overlapping selections), worker-order sums, the
// union zeroed everywhere, then the usual finalize without a threshold update.
template <typename T>
int aggregate_baseline(micro_ctx* c) {
  cudaStream_t st = c->stream;
  int32_t* uidx = c->uni_idx[c->buf];
  long long* K = c->Kbuf + c->buf;
  const unsigned grid = grid_for(c->n_g, c->dev);
  WorkerPtrs w{};
  for (int i = 0; i < c->n_local; ++i) w.resid[i] = c->resid[i];
  if (c->kind == 4) {  // one coalesced pass does the union, sums, model, dense g/n and zeroing
    k_dense_all<T><<<grid, 256, 0, st>>>(w, c->n, c->n_g, (T*)c->model, (T*)c->dense, uidx,
                                         (T*)c->uni_sum[c->buf], K);
    CU(cudaGetLastError());
    if (c->norm)
      for (int i = 0; i < c->n_local; ++i) TRY(launch_sumsq<T>(c, i));
    c->vectors_done = true;
    return launch_finalize<T>(c, uidx, c->uni_sum[c->buf], 0);
  } else {
    for (int i = 0; i < c->n_local; ++i) w.sel_idx[i] = c->sel_idx[c->buf][i];
    const unsigned mgrid = grid_for(std::min<int64_t>(c->sel_cap, 2 * (int64_t)c->k_global + 1024), c->dev);
    k_union_mark<<<dim3(mgrid, c->n_local), 256, 0, st>>>(w, c->counts, c->sel_cap, c->bitmap);
    CU(cudaGetLastError());
    TRY(bitmap_offsets(c->bitmap, c->nwords, c->word_off, c->scan_tmp, st, K));
    // Emission + worker-order sums: one pass over the bitmap's words when
    // the union is dense (K > 15 % of n_g: coalesced residual loads), else
    // the ordered emission and a gather per union entry.  The scan wrote K;
    // each path's kernels read it and the other path's return at once.
    const long long dense_above = (long long)c->nwords * 32 * 3 / 20;
    const unsigned wgrid = grid_for(c->nwords * 32 / kUnionWords, c->dev);  // a warp per kUnionWords words
    if (c->cfg.error_feedback)
      k_union_words<T, true><<<wgrid, 256, 0, st>>>(w, c->n, c->bitmap, c->nwords, c->word_off, uidx,
                                                     (T*)c->uni_sum[c->buf], K, dense_above);
    else
      k_union_words<T, false><<<wgrid, 256, 0, st>>>(w, c->n, c->bitmap, c->nwords, c->word_off, uidx,
                                                      (T*)c->uni_sum[c->buf], K, dense_above);
    CU(cudaGetLastError());
    k_bitmap_emit<<<grid_for(c->nwords, c->dev), 256, 0, st>>>(c->bitmap, c->nwords, c->word_off, uidx, K,
                                                                dense_above);
    CU(cudaGetLastError());
    if (c->cfg.error_feedback)
      k_union_reduce<T, true><<<grid, 256, 0, st>>>(w, c->n, uidx, K, (T*)c->uni_sum[c->buf], dense_above);
    else
      k_union_reduce<T, false><<<grid, 256, 0, st>>>(w, c->n, uidx, K, (T*)c->uni_sum[c->buf], dense_above);
    CU(cudaGetLastError());
  }
  if (!c->cfg.error_feedback)
    for (int i = 0; i < c->n_local; ++i) CU(cudaMemsetAsync(c->resid[i], 0, c->n_g * c->esz, st));
  else if (c->norm)
    for (int i = 0; i < c->n_local; ++i) TRY(launch_sumsq<T>(c, i));
  return launch_finalize<T>(c, uidx, c->uni_sum[c->buf], 0);
}

template <typename T>
int aggregate_cluster(micro_ctx* c) {
  if (c->kind && !c->sel_is_union) return aggregate_baseline<T>(c);
  if (c->n == 1) return launch_finalize<T>(c, c->sel_idx[c->buf][0], c->sel_val[c->buf][0], 1);
  WorkerPtrs w{};
  for (int i = 0; i < c->n; ++i) {
    w.sel_idx[i] = c->sel_idx[c->buf][i];
    w.sel_val[i] = c->sel_val[c->buf][i];
    w.resid[i] = c->resid[i];
  }
  const int64_t expect = std::max<int64_t>((int64_t)c->k_worker * 3 / 2, 256);
  const unsigned gx = (unsigned)std::min<int64_t>((expect + 255) / 256, 2048);
  const dim3 grid(gx, (unsigned)c->n);
  const long long* cnt = (const long long*)c->counts;
  NormSlot* slots = c->norm ? c->norm_slot : (NormSlot*)nullptr;
  int32_t* ui = c->uni_idx[c->buf];
  T* us = (T*)c->uni_sum[c->buf];
  const long long cap = c->sel_cap;
  if (c->cfg.error_feedback && c->n <= 8)
    CU(launch_pdl(k_cluster_reduce<T, true, true>, grid, dim3(256), c->stream, w, cnt, cap, c->n, (int64_t)c->t_cur, ui,
                  us, slots));
  else if (c->cfg.error_feedback)
    CU(launch_pdl(k_cluster_reduce<T, true>, grid, dim3(256), c->stream, w, cnt, cap, c->n, (int64_t)c->t_cur, ui, us,
                  slots));
  else
    CU(launch_pdl(k_cluster_reduce<T, false>, grid, dim3(256), c->stream, w, cnt, cap, c->n, (int64_t)c->t_cur, ui, us,
                  (NormSlot*)nullptr));
  CU(cudaGetLastError());
  return launch_finalize<T>(c, c->uni_idx[c->buf], c->uni_sum[c->buf], 1);
}

int validate_config(const micro_config* g) {
  if (!g) return fail(MICRO_EINVAL, "null config");
  TRY(check_dtype(g->dtype));
  if (g->n_workers < 1) return fail(MICRO_EINVAL, "run config: workers must be >= 1");
  if (g->sparsifier < MICRO_MICRO || g->sparsifier > MICRO_DENSE)
    return fail(MICRO_EINVAL, "unknown sparsifier kind %d", g->sparsifier);
  if (g->sparsifier != MICRO_MICRO && g->n_local != g->n_workers)
    return fail(MICRO_EINVAL, "the comparison sparsifiers run as a single-device cluster (n_local == n_workers)");
  if (g->n_workers > MICRO_MAX_WORKERS)
    return fail(MICRO_EINVAL, "run config: at most %d workers supported", MICRO_MAX_WORKERS);
  if (g->n_g < g->n_workers)
    return fail(MICRO_EINVAL, "run config: gradient length %lld smaller than worker count %d",
                (long long)g->n_g, g->n_workers);
  if (g->n_g >= (int64_t)INT32_MAX) return fail(MICRO_EINVAL, "n_g must be < 2^31 (int32 indices)");
  if (!(g->n_local == g->n_workers || (g->n_local == 1 && g->n_workers > 1)))
    return fail(MICRO_EINVAL, "n_local must equal n_workers or be 1");
  if (g->rank < 0 || g->rank + g->n_local > g->n_workers)
    return fail(MICRO_EINVAL, "rank %d out of range", g->rank);
  if (!(g->density > 0.0 && g->density <= 1.0)) return fail(MICRO_EINVAL, "run config: density must lie in (0, 1]");
  if (!(g->initial_threshold >= 0.0) || !std::isfinite(g->initial_threshold))
    return fail(MICRO_EINVAL, "run config: delta0 must be finite and nonnegative");
  if (!(g->scaling_factor > 0.0 && g->scaling_factor < 1.0))
    return fail(MICRO_EINVAL, "run config: alpha must lie in (0, 1)");
  if (!(g->min_threshold > 0.0)) return fail(MICRO_EINVAL, "run config: eps-delta must be positive");
  if (g->target != MICRO_TARGET_SPLIT && g->target != MICRO_TARGET_FULL)
    return fail(MICRO_EINVAL, "unknown per-worker target %d", g->target);
  if (g->selection_capacity < 0) return fail(MICRO_EINVAL, "negative selection capacity");
  if (g->grad_dtype != MICRO_GRAD_SAME && g->grad_dtype != MICRO_GRAD_F32)
    return fail(MICRO_EINVAL, "unknown gradient element type %d", g->grad_dtype);
  if (g->grad_dtype == MICRO_GRAD_F32 && (g->dtype != MICRO_F64 || g->sparsifier != MICRO_MICRO))
    return fail(MICRO_EINVAL, "fp32 gradients need fp64 state (dtype MICRO_F64) and the MiCRO sparsifier");
  return MICRO_OK;
}

int reset_state(micro_ctx* c) {
  DeviceGuard dg(c->dev);
  if (c->aux) CU(cudaStreamSynchronize(c->aux));
  c->clear_pending = false;
  for (int i = 0; i < c->n_local; ++i) CU(cudaMemsetAsync(c->resid[i], 0, c->n_g * c->esz, c->stream));
  // MiCRO: delta_0 per worker; hard threshold: the fixed delta_0; top-k, CLT-k,
  // dense: no threshold (the record's threshold is 0, harness.cpp:135)
  std::vector<double> d0(c->n_local, (c->kind == 0 || c->kind == 3) ? c->cfg.initial_threshold : 0.0);
  CU(cudaMemcpyAsync(c->delta, d0.data(), sizeof(double) * c->n_local, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemsetAsync(c->counts, 0, sizeof(long long) * c->n_local, c->stream));
  CU(cudaMemsetAsync(c->Kbuf, 0, sizeof(long long) * 2, c->stream));
  CU(cudaMemsetAsync(c->flags, 0, sizeof(int), c->stream));
  if (c->dense) CU(cudaMemsetAsync(c->dense, 0, c->n_g * c->esz, c->stream));
  if (c->dense_dirty) CU(cudaMemsetAsync(c->dense_dirty, 0, (c->n_g / 256 + 8) * 8, c->stream));
  if (c->super_counts) CU(cudaMemsetAsync(c->super_counts, 0, 2 * kMaxSupers * sizeof(int), c->stream));
  if (c->kind) {
    CU(cudaMemsetAsync(c->topk_hist, 0, sizeof(unsigned) * kBins * c->n_local, c->stream));
    CU(cudaMemsetAsync(c->bitmap, 0, sizeof(unsigned) * c->nwords, c->stream));
    const double m1 = -1.0;
    CU(cudaMemcpyAsync(c->minus_one, &m1, sizeof m1, cudaMemcpyHostToDevice, c->stream));
  }
  if (c->norm) {
    CU(cudaMemsetAsync(c->norm_ticket, 0, sizeof(unsigned) * (sumsq_groups(c->norm_ctas) + 1), c->stream));
    CU(cudaMemsetAsync(c->norm_slot, 0, sizeof(NormSlot) * c->n_local, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  c->steps = 0;
  c->t_cur = -1;
  c->buf = 0;
  c->compressed = false;
  c->poisoned = false;
  c->ever_stepped = false;
  return MICRO_OK;
}


}  // namespace

// ============================================================== C ABI ====

extern "C" {

int micro_abi_version(void) { return MICRO_ABI_VERSION; }

const char* micro_status_string(int s) {
  switch (s) {
    case MICRO_OK: return "MICRO_OK";
    case MICRO_EINVAL: return "MICRO_EINVAL (invalid_argument)";
    case MICRO_ELOGIC: return "MICRO_ELOGIC (logic_error)";
    case MICRO_ENONFINITE: return "MICRO_ENONFINITE (runtime_error: non-finite gradient)";
    case MICRO_ECUDA: return "MICRO_ECUDA";
    case MICRO_ENCCL: return "MICRO_ENCCL";
    case MICRO_ECAPACITY: return "MICRO_ECAPACITY";
    case MICRO_ENOMEM: return "MICRO_ENOMEM";
  }
  return "unknown status";
}

const char* micro_last_error(void) { return g_err.c_str(); }

int micro_partition(int64_t n_g, int n, int64_t t, int worker, int64_t* start, int64_t* end) {
  return h_partition(n_g, n, t, worker, start, end);
}

int micro_global_target_count(double density, int64_t n_g, uint64_t* k) {
  return h_global_target(density, n_g, k);
}

int micro_per_worker_target_count(double density, int64_t n_g, int n, int target, uint64_t* k) {
  return h_worker_target(density, n_g, n, target, k);
}

int micro_update_threshold(double* delta, uint64_t k_target, uint64_t k_selected, double alpha,
                           double min_threshold) {
  return h_update_threshold(delta, k_target, k_selected, alpha, min_threshold);
}

void micro_config_default(micro_config* g) {
  std::memset(g, 0, sizeof *g);
  g->n_workers = 1;
  g->n_local = 1;
  g->dtype = MICRO_F32;
  g->density = 0.01;
  g->initial_threshold = 0.01;
  g->scaling_factor = 0.01;
  g->min_threshold = 1e-12;
  g->target = MICRO_TARGET_SPLIT;
  g->error_feedback = 1;
  g->dense_output = 1;
  g->record_error_norm = 1;
}

int micro_ctx_create(micro_ctx** out, const micro_config* cfg, void* stream) {
  if (!out) return fail(MICRO_EINVAL, "null output pointer");
  *out = nullptr;
  TRY(validate_config(cfg));
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (cfg->device < 0 || cfg->device >= ndev)
    return fail(MICRO_EINVAL, "device %d out of range (%d devices)", cfg->device, ndev);
  auto* c = new micro_ctx;
  c->cfg = *cfg;
  c->dev = cfg->device;
  c->n = cfg->n_workers;
  c->n_local = cfg->n_local;
  c->n_g = cfg->n_g;
  c->esz = dtype_size(cfg->dtype);
  c->gsz = cfg->grad_dtype == MICRO_GRAD_F32 ? 4 : c->esz;
  c->cluster = c->n_local == c->n;
  c->kind = cfg->sparsifier;
  // one worker: the union is its selection, for MiCRO and the comparison
  // selections alike (hard threshold: the same step with delta_0 fixed;
  // top-k / CLT-k: the radix select, then the same compaction with the ties
  // and zeroing).  The sums are 0 + acc (a selected -0 becomes +0).  The
  // dense baseline keeps its one-pass kernel; top-k / CLT-k without error
  // feedback keep the general path (their first pass leaves acc in e, which
  // that path zeroes).
  c->sel_is_union = c->n == 1 && (c->kind == 0 || c->kind == 3 ||
                                   ((c->kind == 1 || c->kind == 2) && cfg->error_feedback));
  int rc = h_worker_target(cfg->density, cfg->n_g, cfg->n_workers, cfg->target, &c->k_worker);
  if (rc) { delete c; return rc; }
  DeviceGuard dg(c->dev);
  auto cleanup = [&](int code) {
    micro_ctx_destroy(c);
    return code;
  };
  c->stream = (cudaStream_t)stream;  // NULL = the legacy default stream, like every CUDA API
  // MiCRO selects inside its partition; the comparison sparsifiers over the whole vector
  const int64_t max_range = c->kind ? c->n_g : (c->n_g + c->n - 1) / c->n;
  c->sel_cap = cfg->selection_capacity ? std::min<int64_t>(cfg->selection_capacity, max_range) : max_range;
  c->uni_cap = std::min<int64_t>(c->n_g, (int64_t)c->n * c->sel_cap);
  c->dense_fused = c->sel_is_union && cfg->dense_output;
  const int nbuf = c->n == 1 ? 2 : 1;
  c->resid.assign(c->n_local, nullptr);
  for (int b = 0; b < 2; ++b) {
    c->sel_idx[b].assign(c->n_local, nullptr);
    c->sel_val[b].assign(c->n_local, nullptr);
  }
  for (int i = 0; i < c->n_local; ++i) {
    if ((rc = c->alloc(&c->resid[i], c->n_g * c->esz))) return cleanup(rc);
    for (int b = 0; b < nbuf; ++b) {
      if ((rc = c->alloc((void**)&c->sel_idx[b][i], c->sel_cap * 4))) return cleanup(rc);
      if ((rc = c->alloc(&c->sel_val[b][i], c->sel_cap * c->esz))) return cleanup(rc);
    }
    if (nbuf == 1) {
      c->sel_idx[1][i] = c->sel_idx[0][i];
      c->sel_val[1][i] = c->sel_val[0][i];
    }
  }
  if (!c->sel_is_union)
    for (int b = 0; b < 2; ++b) {
      if ((rc = c->alloc((void**)&c->uni_idx[b], c->uni_cap * 4))) return cleanup(rc);
      if ((rc = c->alloc(&c->uni_sum[b], c->uni_cap * c->esz))) return cleanup(rc);
    }
  if ((rc = c->alloc((void**)&c->counts, sizeof(long long) * c->n_local))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->delta, sizeof(double) * c->n_local))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->Kbuf, sizeof(long long) * 2))) return cleanup(rc);
  if (cfg->dense_output && (rc = c->alloc(&c->dense, c->n_g * c->esz))) return cleanup(rc);
  if (c->dense_fused && (rc = c->alloc((void**)&c->dense_dirty, (c->n_g / 256 + 8) * 8))) return cleanup(rc);
  {
    // K1 staging: one run slot of kStreamWarps units per k1_stream CTA that meets the range
    const int64_t ue = c->esz == 4 ? stream_unit_elems<float>() : stream_unit_elems<double>();
    const int64_t stage = (max_range / (kStreamWarps * ue) + 2) * kStreamWarps * ue;
    if ((rc = c->alloc((void**)&c->stage_idx, stage * 4))) return cleanup(rc);
    if ((rc = c->alloc(&c->stage_val, stage * c->esz))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->unit_counts, (max_range / 128 + 8) * sizeof(int)))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->super_counts, 2 * kMaxSupers * sizeof(int)))) return cleanup(rc);
    {
      // super blocks of S runs (S a multiple of the gather CTA's 8 runs), <= kMaxSupers of them
      const int64_t runs = max_range / (kStreamWarps * ue) + 2;
      const int64_t S = (runs + kMaxSupers - 1) / kMaxSupers;
      c->super_runs = (int)std::max<int64_t>(kGatherWarps, (S + kGatherWarps - 1) / kGatherWarps * kGatherWarps);
    }
  }
  if ((rc = c->alloc((void**)&c->flags, sizeof(int)))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->hist_t, sizeof(long long) * kHistCap))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->hist_K, sizeof(long long) * kHistCap))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->hist_counts, sizeof(long long) * kHistCap * c->n_local))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->hist_delta, sizeof(double) * kHistCap * c->n_local))) return cleanup(rc);
  if ((rc = c->alloc((void**)&c->hist_err, sizeof(double) * kHistCap * c->n_local))) return cleanup(rc);
  c->norm = cfg->record_error_norm && cfg->error_feedback;
  if (c->kind) {
    if ((rc = h_global_target(cfg->density, c->n_g, &c->k_global))) return cleanup(rc);
    c->nwords = (c->n_g + 31) / 32;
    if ((rc = c->alloc((void**)&c->topk, sizeof(TopkState) * c->n_local))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->topk_hist, sizeof(unsigned) * kBins * c->n_local))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->tie_counts, sizeof(unsigned) * kTieChunks * c->n_local))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->bitmap, sizeof(unsigned) * c->nwords))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->scan_tmp, sizeof(int) * scan_tiles(c->nwords)))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->word_off, sizeof(int) * c->nwords))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->minus_one, sizeof(double)))) return cleanup(rc);
  }
  if (c->norm) {
    // producing grids: k1_stream (one CTA per 8 units) or k_sumsq (4 per SM)
    const int64_t ue = c->esz == 4 ? stream_unit_elems<float>() : stream_unit_elems<double>();
    const int64_t units = (c->n_g + ue - 1) / ue;
    c->norm_ctas = std::max<int64_t>((units + kStreamWarps - 1) / kStreamWarps, 4 * (int64_t)num_sms(c->dev));
    const int64_t groups = sumsq_groups(c->norm_ctas);
    if ((rc = c->alloc((void**)&c->norm_part, sizeof(double) * c->norm_ctas))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->norm_group, sizeof(double) * groups))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->norm_ticket, sizeof(unsigned) * (groups + 1)))) return cleanup(rc);
    if ((rc = c->alloc((void**)&c->norm_slot, sizeof(NormSlot) * c->n_local))) return cleanup(rc);
  }
  cudaError_t e;
  if (c->dense && !c->dense_fused) {
    if ((e = cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming)) != cudaSuccess)
      return cleanup(fail(MICRO_ECUDA, "aux stream: %s", cudaGetErrorString(e)));
  }
  if ((rc = reset_state(c))) return cleanup(rc);
  *out = c;
  return MICRO_OK;
}

int micro_ctx_destroy(micro_ctx* c) {
  if (!c) return MICRO_OK;
  DeviceGuard dg(c->dev);
  cudaStreamSynchronize(c->stream);
  if (c->aux) cudaStreamSynchronize(c->aux);
  nccl_release(c);
  for (void* p : c->peer_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocs) cudaFree(p);
  for (cudaEvent_t ev : c->t_ev) cudaEventDestroy(ev);
  if (c->staging) cudaFree(c->staging);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->group_ev) cudaEventDestroy(c->group_ev);
  if (c->h2d_stream) {
    cudaStreamSynchronize(c->h2d_stream);
    for (cudaEvent_t ev : c->h2d_ev)
      if (ev) cudaEventDestroy(ev);
    if (c->h2d_free) cudaEventDestroy(c->h2d_free);
    cudaStreamDestroy(c->h2d_stream);
  }

  if (c->aux) cudaStreamDestroy(c->aux);
  delete c;
  return MICRO_OK;
}

int micro_ctx_reset(micro_ctx* c) {
  TRY(check_ctx(c));
  return reset_state(c);
}

void* micro_ctx_stream(micro_ctx* c) { return c ? (void*)c->stream : nullptr; }

int micro_set_model(micro_ctx* c, void* d_x) {
  TRY(check_ctx(c));
  if (d_x && ((uintptr_t)d_x % c->esz)) return fail(MICRO_EINVAL, "model pointer misaligned");
  c->model = d_x;
  return MICRO_OK;
}

int micro_compress(micro_ctx* c, const void* const* d_grads, double eta, int64_t t) {
  TRY(check_ctx(c));
  TRY(check_poison(c));
  if (!d_grads) return fail(MICRO_EINVAL, "null gradient array");
  if (!(eta > 0.0)) return fail(MICRO_EINVAL, "accumulate: eta must be positive");
  if (t < 0) return fail(MICRO_EINVAL, "partition: negative iteration");
  if (c->compressed) return fail(MICRO_ELOGIC, "micro_compress called twice without aggregation");
  for (int i = 0; i < c->n_local; ++i) {
    if (!d_grads[i]) return fail(MICRO_EINVAL, "null gradient for local worker %d", i);
    if ((uintptr_t)d_grads[i] % c->gsz) return fail(MICRO_EINVAL, "gradient %d misaligned for its dtype", i);
  }
  DeviceGuard dg(c->dev);
  c->t_cur = t;
  c->buf = (int)(c->steps & 1);
  TRY(c->esz == 4 ? fork_dense_clear<float>(c) : fork_dense_clear<double>(c));
  std::vector<const void*> gs(c->n_local);
  for (int i = 0; i < c->n_local; ++i) {
    const void* g = d_grads[i];
    if ((uintptr_t)g % 16) {
      // the streaming K1 reads 16-byte vectors: realign once (8 B/elem copy)
      TRY(ensure_staging(c));
      void* dst = (char*)c->staging + (size_t)i * c->staging_stride;
      if (dst != g) CU(cudaMemcpyAsync(dst, g, (size_t)c->n_g * c->gsz, cudaMemcpyDeviceToDevice, c->stream));
      g = dst;
    }
    gs[i] = g;
  }
  if (c->kind == 1 && c->n_local > 1 && c->k_global > 0 && (int64_t)c->k_global < c->n_g) {
    // top-k on several workers: every worker's radix select in the same launches
    if (c->esz == 4) TRY(launch_topk_batch<float>(c, gs.data(), eta));
    else TRY(launch_topk_batch<double>(c, gs.data(), eta));
  } else if ((c->kind == 2 || c->kind == 4) && c->n_local > 1) {
    // workers that only accumulate this step (CLT-k's non-leaders, dense: all)
    // in one launch; the CLT-k leader then selects as in launch_baseline
    const int leader = c->kind == 2 ? (int)(t % c->n) : -1;
    TopkBatch b{};
    for (int i = 0; i < c->n_local; ++i) {
      b.e[i] = c->resid[i];
      b.g[i] = gs[i];
    }
    const long long count = c->kind == 4 ? (long long)c->n_g : 0;
    const dim3 grid(grid_for(c->n_g, c->dev), c->n_local);
    if (c->esz == 4)
      k_accumulate_probe_b<float><<<grid, 256, 0, c->stream>>>(b, eta, c->n_g, c->flags, leader, c->counts, count);
    else
      k_accumulate_probe_b<double><<<grid, 256, 0, c->stream>>>(b, eta, c->n_g, c->flags, leader, c->counts, count);
    CU(cudaGetLastError());
    if (leader >= 0) {
      if (c->esz == 4) TRY(launch_k1<float>(c, leader, gs[leader], eta, t));
      else TRY(launch_k1<double>(c, leader, gs[leader], eta, t));
    }
  } else {
    for (int i = 0; i < c->n_local; ++i) {
      if (c->esz == 4) TRY(launch_k1<float>(c, i, gs[i], eta, t));
      else TRY(launch_k1<double>(c, i, gs[i], eta, t));
    }
  }
  c->compressed = true;
  return MICRO_OK;
}

int micro_aggregate(micro_ctx* c) {
  TRY(check_ctx(c));
  TRY(check_poison(c));
  if (!c->compressed) return fail(MICRO_ELOGIC, "micro_aggregate without a preceding micro_compress");
  if (!c->cluster) {
    if (c->nccl_comm) return nccl_aggregate(c);
    return fail(MICRO_ELOGIC,
                "micro_aggregate: multi-rank context without NCCL attached; use micro_dist_attach_nccl, "
                "or the micro_dist_* / micro_peer_* protocol");
  }
  DeviceGuard dg(c->dev);
  return c->esz == 4 ? aggregate_cluster<float>(c) : aggregate_cluster<double>(c);
}

int micro_step(micro_ctx* c, const void* const* d_grads, double eta, int64_t t) {
  TRY(check_ctx(c));
  // one-worker cluster, streaming K1: fold k_finalize into k1_gather
  c->fuse_step = c->cluster && c->sel_is_union && (!c->dense || c->dense_fused);
  const int rc = micro_compress(c, d_grads, eta, t);
  c->fuse_step = false;
  if (rc != MICRO_OK) {
    c->fin_done = false;
    return rc;
  }
  return micro_aggregate(c);
}

int micro_sync(micro_ctx* c) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  int flags = 0;
  TRY(read_flags(c, &flags));
  if (flags & 1) return check_poison(c);
  if (flags & 2) return fail(MICRO_ECAPACITY, "selection exceeded capacity %lld", (long long)c->sel_cap);
  return MICRO_OK;
}

int micro_step_host(micro_ctx* c, const void* h_grads, double eta, int64_t t, int32_t* h_idx,
                    void* h_sums, int64_t cap, int64_t* K) {
  TRY(check_ctx(c));
  if (!c->cluster) return fail(MICRO_ELOGIC, "micro_step_host: single-device clusters only");
  DeviceGuard dg(c->dev);
  TRY(ensure_staging(c));
  const size_t row = (size_t)c->n_g * c->gsz;
  std::vector<const void*> g(c->n_local);
  for (int i = 0; i < c->n_local; ++i) g[i] = (const char*)c->staging + (size_t)i * c->staging_stride;
  if (c->sel_is_union && c->kind == 0) {
    // copy/compute overlap: the gradient crosses PCIe in chunks of whole K1
    // CTAs on a copy stream; K1 streams each chunk as it lands
    if (!c->h2d_stream) {
      CU(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
      for (auto& ev : c->h2d_ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&c->h2d_free, cudaEventDisableTiming));
    }
    const int64_t cta_elems = (c->esz == 4 ? stream_unit_elems<float>() : stream_unit_elems<double>()) * kStreamWarps;
    const int64_t ctas = (c->n_g + cta_elems - 1) / cta_elems;
    const int64_t per = (ctas + micro_ctx::kH2DChunks - 1) / micro_ctx::kH2DChunks;
    CU(cudaEventRecord(c->h2d_free, c->stream));  // the last step's K1 has read the staging
    CU(cudaStreamWaitEvent(c->h2d_stream, c->h2d_free, 0));
    for (int k = 0; k < micro_ctx::kH2DChunks; ++k) {
      const int64_t lo = std::min<int64_t>(c->n_g, per * k * cta_elems);
      const int64_t hi = std::min<int64_t>(c->n_g, per * (k + 1) * cta_elems);
      if (hi > lo)
        CU(cudaMemcpyAsync((char*)c->staging + lo * c->gsz, (const char*)h_grads + lo * c->gsz,
                           (size_t)(hi - lo) * c->gsz, cudaMemcpyHostToDevice, c->h2d_stream));
      CU(cudaEventRecord(c->h2d_ev[k], c->h2d_stream));
    }
    c->h2d_chunks = micro_ctx::kH2DChunks;
    const int rc = micro_step(c, g.data(), eta, t);
    c->h2d_chunks = 0;
    TRY(rc);
  } else {
    CU(cudaMemcpy2DAsync(c->staging, c->staging_stride, h_grads, row, row, c->n_local, cudaMemcpyHostToDevice,
                         c->stream));
    TRY(micro_step(c, g.data(), eta, t));
  }
  return micro_copy_union(c, h_idx, h_sums, cap, K);
}

int micro_query(micro_ctx* c, micro_stats* st, int64_t* counts, double* deltas) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  int flags = 0;
  TRY(read_flags(c, &flags));
  long long K = 0;
  std::vector<long long> k(c->n_local);
  if (c->ever_stepped) {
    const int b = (int)((c->steps - 1) & 1);
    CU(cudaMemcpy(&K, c->Kbuf + b, sizeof K, cudaMemcpyDeviceToHost));
  }
  CU(cudaMemcpy(k.data(), c->counts, sizeof(long long) * c->n_local, cudaMemcpyDeviceToHost));
  if (counts)
    for (int i = 0; i < c->n_local; ++i) counts[i] = k[i];
  if (deltas) CU(cudaMemcpy(deltas, c->delta, sizeof(double) * c->n_local, cudaMemcpyDeviceToHost));
  if (st) {
    st->t = c->t_cur;
    st->steps = c->steps;
    st->K = K;
    long long tot = 0;
    for (long long v : k) tot += v;
    st->total_selected = c->cluster ? tot : K;
    st->nonfinite = flags & 1;
    st->overflow = (flags >> 1) & 1;
  }
  return MICRO_OK;
}

int micro_kernel_timing(micro_ctx* c, int enable) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  if (enable && c->t_ev.empty()) {
    c->t_ev.resize(2 * kTimingCap);
    for (auto& ev : c->t_ev) CU(cudaEventCreate(&ev));
  }
  if (enable < 0) return fail(MICRO_EINVAL, "timing period must be >= 0");
  c->timing = enable != 0;
  c->timing_period = enable > 0 ? enable : 1;
  c->t_seen = 0;
  c->t_next = 0;
  return MICRO_OK;
}

int micro_kernel_times(micro_ctx* c, float* ms, int max, int* written) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  CU(cudaStreamSynchronize(c->stream));
  const int n = std::min(max, c->t_next);
  for (int k = 0; k < n; ++k) CU(cudaEventElapsedTime(&ms[k], c->t_ev[2 * k], c->t_ev[2 * k + 1]));
  if (written) *written = n;
  return MICRO_OK;
}

int micro_history(micro_ctx* c, int64_t max, int64_t* t, int64_t* K, int64_t* counts,
                  double* delta_used, int64_t* written) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  CU(cudaStreamSynchronize(c->stream));
  const int64_t n = std::min<int64_t>(std::min<int64_t>(max, c->steps), kHistCap);
  std::vector<long long> ht(kHistCap), hk(kHistCap), hc(kHistCap * c->n_local);
  std::vector<double> hd(kHistCap * c->n_local);
  CU(cudaMemcpy(ht.data(), c->hist_t, sizeof(long long) * kHistCap, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hk.data(), c->hist_K, sizeof(long long) * kHistCap, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hc.data(), c->hist_counts, sizeof(long long) * hc.size(), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hd.data(), c->hist_delta, sizeof(double) * hd.size(), cudaMemcpyDeviceToHost));
  for (int64_t s = 0; s < n; ++s) {
    const int64_t step = c->steps - n + s;
    const int64_t slot = step % kHistCap;
    if (t) t[s] = ht[slot];
    if (K) K[s] = hk[slot];
    for (int i = 0; i < c->n_local; ++i) {
      if (counts) counts[s * c->n_local + i] = hc[slot * c->n_local + i];
      if (delta_used) delta_used[s * c->n_local + i] = hd[slot * c->n_local + i];
    }
  }
  if (written) *written = n;
  return MICRO_OK;
}

int micro_records(micro_ctx* c, int64_t max, micro_record* out, int64_t* written) {
  TRY(check_ctx(c));
  if (max < 0 || (max && !out)) return fail(MICRO_EINVAL, "bad record buffer");
  DeviceGuard dg(c->dev);
  CU(cudaStreamSynchronize(c->stream));
  const int64_t n = std::min<int64_t>(std::min<int64_t>(max, c->steps), kHistCap);
  const int nl = c->n_local;
  std::vector<long long> ht(kHistCap), hk(kHistCap), hc(kHistCap * nl);
  std::vector<double> hd(kHistCap * nl), he(kHistCap * nl);
  CU(cudaMemcpy(ht.data(), c->hist_t, sizeof(long long) * kHistCap, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hk.data(), c->hist_K, sizeof(long long) * kHistCap, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hc.data(), c->hist_counts, sizeof(long long) * hc.size(), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hd.data(), c->hist_delta, sizeof(double) * hd.size(), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(he.data(), c->hist_err, sizeof(double) * he.size(), cudaMemcpyDeviceToHost));
  uint64_t k_global = 0;
  TRY(h_global_target(c->cfg.density, c->n_g, &k_global));
  for (int64_t s = 0; s < n; ++s) {
    const int64_t slot = (c->steps - n + s) % kHistCap;
    micro_record r{};
    r.t = ht[slot];
    r.K = hk[slot];
    long long tot = 0;
    double dsum = 0.0, esum = 0.0;
    for (int i = 0; i < nl; ++i) {  // worker order, like the reference's loops
      tot += hc[slot * nl + i];
      dsum += hd[slot * nl + i];
      esum += he[slot * nl + i];
    }
    // a rank of an n-GPU job sees only its own k_i; the partitions are
    // disjoint, so sum_i k_i = |union| there
    r.total_selected = c->cluster ? tot : r.K;
    r.actual_density = (double)r.K / (double)c->n_g;                                   // metrics.cpp:7-10
    r.buildup_factor = r.total_selected == 0 ? 0.0 : (double)r.K / (double)k_global;   // collectives.cpp:59-63
    r.redundant_traffic_factor = r.total_selected == 0 ? 0.0 : (double)r.total_selected / (double)r.K;
    r.error_norm = esum / nl;                                                          // harness.cpp:230-235
    // MiCRO: the workers' mean (harness.cpp:149); the hard threshold records
    // delta_0 itself (:172), not a mean that need not round back to it
    r.threshold = c->kind == 3 ? c->cfg.initial_threshold : dsum / nl;
    out[s] = r;
  }
  if (written) *written = n;
  return MICRO_OK;
}

int micro_union_device(micro_ctx* c, const int32_t** d_idx, const void** d_sums, const int64_t** d_K) {
  TRY(check_ctx(c));
  const int b = c->ever_stepped ? (int)((c->steps - 1) & 1) : 0;
  if (d_idx) *d_idx = c->sel_is_union ? c->sel_idx[b][0] : c->uni_idx[b];
  if (d_sums) *d_sums = c->sel_is_union ? c->sel_val[b][0] : c->uni_sum[b];
  if (d_K) *d_K = (const int64_t*)(c->Kbuf + b);
  return MICRO_OK;
}

int micro_dense_device(micro_ctx* c, const void** d_dense) {
  TRY(check_ctx(c));
  if (!c->dense) return fail(MICRO_ELOGIC, "dense output disabled (micro_config.dense_output = 0)");
  *d_dense = c->dense;
  return MICRO_OK;
}

int micro_residual_device(micro_ctx* c, int i, void** d) {
  TRY(check_ctx(c));
  if (i < 0 || i >= c->n_local) return fail(MICRO_EINVAL, "local worker %d out of range", i);
  *d = c->resid[i];
  return MICRO_OK;
}

int micro_selection_device(micro_ctx* c, int i, const int32_t** d_idx, const void** d_val,
                           const int64_t** d_count) {
  TRY(check_ctx(c));
  if (i < 0 || i >= c->n_local) return fail(MICRO_EINVAL, "local worker %d out of range", i);
  if (d_idx) *d_idx = c->sel_idx[c->buf][i];
  if (d_val) *d_val = c->sel_val[c->buf][i];
  if (d_count) *d_count = (const int64_t*)(c->counts + i);
  return MICRO_OK;
}

int micro_threshold_device(micro_ctx* c, double** d) {
  TRY(check_ctx(c));
  *d = c->delta;
  return MICRO_OK;
}

int micro_copy_union(micro_ctx* c, int32_t* h_idx, void* h_sums, int64_t cap, int64_t* K) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->dev);
  int flags = 0;
  TRY(read_flags(c, &flags));
  if (flags & 1) return check_poison(c);
  if (flags & 2) return fail(MICRO_ECAPACITY, "selection exceeded capacity %lld", (long long)c->sel_cap);
  if (!c->ever_stepped) {
    if (K) *K = 0;
    return MICRO_OK;
  }
  const int32_t* di;
  const void* ds;
  const int64_t* dK;
  TRY(micro_union_device(c, &di, &ds, &dK));
  long long k = 0;
  CU(cudaMemcpy(&k, dK, sizeof k, cudaMemcpyDeviceToHost));
  if (K) *K = k;
  if (k > cap) return fail(MICRO_ECAPACITY, "union of %lld exceeds host capacity %lld", k, (long long)cap);
  if (k) {
    if (h_idx) CU(cudaMemcpyAsync(h_idx, di, (size_t)k * 4, cudaMemcpyDeviceToHost, c->stream));
    if (h_sums) CU(cudaMemcpyAsync(h_sums, ds, (size_t)k * c->esz, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  return MICRO_OK;
}

int micro_copy_residual(micro_ctx* c, int i, void* h) {
  TRY(check_ctx(c));
  if (i < 0 || i >= c->n_local) return fail(MICRO_EINVAL, "local worker %d out of range", i);
  DeviceGuard dg(c->dev);
  CU(cudaMemcpyAsync(h, c->resid[i], c->n_g * c->esz, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MICRO_OK;
}

int micro_copy_dense(micro_ctx* c, void* h) {
  TRY(check_ctx(c));
  if (!c->dense) return fail(MICRO_ELOGIC, "dense output disabled (micro_config.dense_output = 0)");
  DeviceGuard dg(c->dev);
  CU(cudaMemcpyAsync(h, c->dense, c->n_g * c->esz, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MICRO_OK;
}

// ---- one rank of a multi-GPU job ----

}  // extern "C"
