// dist_api.cu — one rank of an n-GPU job (include/micro.h micro_dist_* and
// micro_peer_*): the device halves of the NCCL protocol (dist.py) and the
// exchange over peer memory (peer.cuh).
#include "internal.cuh"

using namespace micro;
using namespace micro::host;

namespace micro {
namespace host {

int dist_ensure_buffers(micro_ctx* c) {
  if (c->dist_all_counts) return MICRO_OK;
  const size_t nk = (size_t)c->n * c->sel_cap;
  TRY(c->alloc((void**)&c->dist_all_counts, sizeof(long long) * c->n));
  TRY(c->alloc((void**)&c->dist_all_idx, 4 * nk));
  TRY(c->alloc(&c->dist_send, c->esz * nk));
  if (!c->recv) TRY(c->alloc(&c->recv, c->esz * nk));
  TRY(c->alloc(&c->dist_own_sums, c->esz * c->sel_cap));
  TRY(c->alloc(&c->dist_all_sums, c->esz * nk));
  CU(cudaMemsetAsync(c->dist_all_counts, 0, sizeof(long long) * c->n, c->stream));
  return MICRO_OK;
}

}  // namespace host
}  // namespace micro

extern "C" {

// ---- the collective protocol's device halves (fixed stride, device counts) ----

static int check_dist_ctx(micro_ctx* c, const char* what) {
  TRY(check_ctx(c));
  TRY(check_poison(c));
  if (c->cluster) return fail(MICRO_ELOGIC, "%s: context is a single-device cluster", what);
  if (!c->compressed) return fail(MICRO_ELOGIC, "%s before micro_compress", what);
  return MICRO_OK;
}

// grid rows sized for the expected selection (the kernels read the real count)
static unsigned dist_grid_x(micro_ctx* c) {
  return grid_for(std::min<int64_t>((int64_t)c->k_worker * 2, c->sel_cap), c->dev) / 4 + 1;
}

int micro_dist_buffers(micro_ctx* c, micro_dist_bufs* b) {
  TRY(check_ctx(c));
  if (c->cluster) return fail(MICRO_ELOGIC, "micro_dist_buffers: context is a single-device cluster");
  if (!b) return fail(MICRO_EINVAL, "null buffer descriptor");
  DeviceGuard dg(c->dev);
  TRY(dist_ensure_buffers(c));
  b->kcap = c->sel_cap;
  b->own_count = (const int64_t*)c->counts;
  b->own_idx = c->sel_idx[0][0];  // single-buffered at n > 1
  b->all_counts = (int64_t*)c->dist_all_counts;
  b->all_idx = c->dist_all_idx;
  b->send = c->dist_send;
  b->recv = c->recv;
  b->own_sums = c->dist_own_sums;
  b->all_sums = c->dist_all_sums;
  return MICRO_OK;
}

int micro_dist_gather_foreign(micro_ctx* c) {
  TRY(check_dist_ctx(c, "micro_dist_gather_foreign"));
  DeviceGuard dg(c->dev);
  TRY(dist_ensure_buffers(c));
  const dim3 grid(dist_grid_x(c), c->n);
  NormSlot* corr = c->norm ? c->norm_slot : nullptr;
  const int me = c->cfg.rank;
  const long long* cnt = c->dist_all_counts;
  if (c->esz == 4) {
    if (c->cfg.error_feedback)
      k_dist_gather_foreign<float, true><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, cnt, c->sel_cap, me,
                                                                      (float*)c->resid[0], (float*)c->dist_send, corr);
    else
      k_dist_gather_foreign<float, false><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, cnt, c->sel_cap, me,
                                                                       (float*)c->resid[0], (float*)c->dist_send, corr);
  } else {
    if (c->cfg.error_feedback)
      k_dist_gather_foreign<double, true><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, cnt, c->sel_cap, me,
                                                                       (double*)c->resid[0], (double*)c->dist_send, corr);
    else
      k_dist_gather_foreign<double, false><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, cnt, c->sel_cap, me,
                                                                        (double*)c->resid[0], (double*)c->dist_send, corr);
  }
  CU(cudaGetLastError());
  return MICRO_OK;
}

int micro_dist_owner_reduce(micro_ctx* c) {
  TRY(check_dist_ctx(c, "micro_dist_owner_reduce"));
  DeviceGuard dg(c->dev);
  TRY(dist_ensure_buffers(c));
  const unsigned grid = grid_for(std::min<int64_t>((int64_t)c->k_worker * 2, c->sel_cap), c->dev);
  const int me = c->cfg.rank;
  if (c->esz == 4)
    k_dist_owner_reduce<float><<<grid, 256, 0, c->stream>>>((const float*)c->sel_val[c->buf][0], c->dist_all_counts,
                                                            (const float*)c->recv, c->sel_cap, c->n, me,
                                                            (float*)c->dist_own_sums);
  else
    k_dist_owner_reduce<double><<<grid, 256, 0, c->stream>>>((const double*)c->sel_val[c->buf][0], c->dist_all_counts,
                                                             (const double*)c->recv, c->sel_cap, c->n, me,
                                                             (double*)c->dist_own_sums);
  CU(cudaGetLastError());
  return MICRO_OK;
}

int micro_dist_finalize(micro_ctx* c) {
  TRY(check_dist_ctx(c, "micro_dist_finalize"));
  DeviceGuard dg(c->dev);
  TRY(dist_ensure_buffers(c));
  const dim3 grid(dist_grid_x(c), c->n);
  if (c->esz == 4) {
    k_dist_build_union<float><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, (const float*)c->dist_all_sums,
                                                           c->dist_all_counts, c->sel_cap, c->n, c->t_cur,
                                                           c->uni_idx[c->buf], (float*)c->uni_sum[c->buf],
                                                           c->Kbuf + c->buf);
    CU(cudaGetLastError());
    return launch_finalize<float>(c, c->uni_idx[c->buf], c->uni_sum[c->buf], 0);
  }
  k_dist_build_union<double><<<grid, 256, 0, c->stream>>>(c->dist_all_idx, (const double*)c->dist_all_sums,
                                                          c->dist_all_counts, c->sel_cap, c->n, c->t_cur,
                                                          c->uni_idx[c->buf], (double*)c->uni_sum[c->buf],
                                                          c->Kbuf + c->buf);
  CU(cudaGetLastError());
  return launch_finalize<double>(c, c->uni_idx[c->buf], c->uni_sum[c->buf], 0);
}

// ---- peer-memory exchange (peer.cuh) ------------------------------------
namespace {
constexpr int kPeerBufs = 10;  // resid, counts, uidx x2, usum x2, norm corr, sel_idx x2, recv
static_assert(MICRO_PEER_HANDLE_BYTES == kPeerBufs * sizeof(cudaIpcMemHandle_t), "handle layout");

void* peer_buf(micro_ctx* c, int b) {
  switch (b) {
    case 0: return c->resid[0];
    case 1: return c->counts;
    case 2: return c->uni_idx[0];
    case 3: return c->uni_idx[1];
    case 4: return c->uni_sum[0];
    case 5: return c->uni_sum[1];
    case 6: return c->norm ? c->norm_slot : nullptr;
    case 7: return c->sel_idx[0][0];
    case 8: return c->sel_idx[1][0] != c->sel_idx[0][0] ? c->sel_idx[1][0] : nullptr;  // single-buffered
    default: return c->recv;
  }
}

int check_peer_ctx(micro_ctx* c) {
  TRY(check_ctx(c));
  TRY(check_poison(c));
  if (c->cluster || c->n_local != 1 || c->n < 2)
    return fail(MICRO_ELOGIC, "micro_peer_*: needs a rank context (n_local = 1 of n > 1 workers)");
  return MICRO_OK;
}
}  // namespace

int micro_peer_export(micro_ctx* c, void* out) {
  TRY(check_peer_ctx(c));
  if (!out) return fail(MICRO_EINVAL, "null handle buffer");
  DeviceGuard dg(c->dev);
  if (!c->recv) TRY(c->alloc(&c->recv, (size_t)c->n * c->sel_cap * c->esz));
  auto* h = (cudaIpcMemHandle_t*)out;
  for (int b = 0; b < kPeerBufs; ++b) {
    std::memset(&h[b], 0, sizeof h[b]);
    if (void* p = peer_buf(c, b)) CU(cudaIpcGetMemHandle(&h[b], p));
  }
  return MICRO_OK;
}

int micro_peer_import(micro_ctx* c, const void* all) {
  TRY(check_peer_ctx(c));
  if (!all) return fail(MICRO_EINVAL, "null handle array");
  if (c->peer_ready) return fail(MICRO_ELOGIC, "micro_peer_import called twice");
  DeviceGuard dg(c->dev);
  const auto* h = (const cudaIpcMemHandle_t*)all;
  const int me = c->cfg.rank;
  static const cudaIpcMemHandle_t zero{};
  for (int r = 0; r < c->n; ++r) {
    void* p[kPeerBufs] = {};
    for (int b = 0; b < kPeerBufs; ++b) {
      if (r == me) {
        p[b] = peer_buf(c, b);
        continue;
      }
      const cudaIpcMemHandle_t& hb = h[(size_t)r * kPeerBufs + b];
      if (std::memcmp(&hb, &zero, sizeof zero) == 0) continue;
      CU(cudaIpcOpenMemHandle(&p[b], hb, cudaIpcMemLazyEnablePeerAccess));
      c->peer_opened.push_back(p[b]);
    }
    if (!p[8]) p[8] = p[7];  // the rank's selection is single-buffered
    if (!p[0] || !p[1] || !p[2] || !p[3] || !p[4] || !p[5] || !p[7] || !p[9])
      return fail(MICRO_EINVAL, "rank %d exported incomplete handles", r);
    if (c->norm && !p[6]) return fail(MICRO_EINVAL, "rank %d does not record the error norm", r);
    c->peer_resid[r] = p[0];
    c->peer_counts[r] = (const long long*)p[1];
    c->peer_uidx[0][r] = (int32_t*)p[2];
    c->peer_uidx[1][r] = (int32_t*)p[3];
    c->peer_usum[0][r] = p[4];
    c->peer_usum[1][r] = p[5];
    c->peer_corr[r] = c->norm ? (NormSlot*)p[6] : nullptr;
    c->peer_sel[0][r] = (const int32_t*)p[7];
    c->peer_sel[1][r] = (const int32_t*)p[8];
    c->peer_recv[r] = p[9];
  }
  c->peer_ready = true;
  return MICRO_OK;
}

int micro_peer_exchange(micro_ctx* c) {
  TRY(check_peer_ctx(c));
  if (!c->peer_ready) return fail(MICRO_ELOGIC, "micro_peer_exchange before micro_peer_import");
  if (!c->compressed) return fail(MICRO_ELOGIC, "micro_peer_exchange before micro_compress");
  if (c->peer_phase) return fail(MICRO_ELOGIC, "micro_peer_exchange called twice");
  DeviceGuard dg(c->dev);
  PeerPtrs pp{};
  for (int r = 0; r < c->n; ++r) {
    pp.counts[r] = c->peer_counts[r];
    pp.resid[r] = c->peer_resid[r];
    pp.uidx[r] = c->peer_uidx[c->buf][r];
    pp.usum[r] = c->peer_usum[c->buf][r];
    pp.corr[r] = c->peer_corr[r];
  }
  // sized for the expected selection (the kernel reads the actual count)
  const unsigned grid = grid_for(std::min<int64_t>((int64_t)c->k_worker * 2, c->sel_cap), c->dev);
  const int me = c->cfg.rank;
  const bool ef = c->cfg.error_feedback != 0;
  long long* Kout = c->Kbuf + c->buf;
  if (c->esz == 4) {
    const float* v = (const float*)c->sel_val[c->buf][0];
    if (ef) k_peer_exchange<float, true><<<grid, 256, 0, c->stream>>>(pp, c->n, me, c->t_cur, c->sel_cap,
                                                                      c->sel_idx[c->buf][0], v, Kout);
    else k_peer_exchange<float, false><<<grid, 256, 0, c->stream>>>(pp, c->n, me, c->t_cur, c->sel_cap,
                                                                     c->sel_idx[c->buf][0], v, Kout);
  } else {
    const double* v = (const double*)c->sel_val[c->buf][0];
    if (ef) k_peer_exchange<double, true><<<grid, 256, 0, c->stream>>>(pp, c->n, me, c->t_cur, c->sel_cap,
                                                                       c->sel_idx[c->buf][0], v, Kout);
    else k_peer_exchange<double, false><<<grid, 256, 0, c->stream>>>(pp, c->n, me, c->t_cur, c->sel_cap,
                                                                      c->sel_idx[c->buf][0], v, Kout);
  }
  CU(cudaGetLastError());
  c->peer_phase = 2;
  return MICRO_OK;
}

PeerBulkPtrs bulk_ptrs(micro_ctx* c) {
  PeerBulkPtrs pb{};
  for (int r = 0; r < c->n; ++r) {
    pb.counts[r] = c->peer_counts[r];
    pb.sel_idx[r] = c->peer_sel[c->buf][r];
    pb.recv[r] = c->peer_recv[r];
    pb.uidx[r] = c->peer_uidx[c->buf][r];
    pb.usum[r] = c->peer_usum[c->buf][r];
  }
  return pb;
}

int micro_peer_contribute(micro_ctx* c) {
  TRY(check_peer_ctx(c));
  if (!c->peer_ready) return fail(MICRO_ELOGIC, "micro_peer_contribute before micro_peer_import");
  if (!c->compressed) return fail(MICRO_ELOGIC, "micro_peer_contribute before micro_compress");
  if (c->peer_phase) return fail(MICRO_ELOGIC, "micro_peer_contribute called twice");
  DeviceGuard dg(c->dev);
  const PeerBulkPtrs pb = bulk_ptrs(c);
  // per owner: CTAs of 8 warps x 32 lanes x kPeerILP entries for the expected selection
  const int64_t expect = std::min<int64_t>((int64_t)c->k_worker * 3 / 2 + 1, c->sel_cap);
  const int64_t per_cta = 8 * 32 * kPeerILP;
  const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((expect + per_cta - 1) / per_cta,
                                                                    2 * (int64_t)num_sms(c->dev))), c->n);
  NormSlot* corr = c->norm ? c->norm_slot : nullptr;
  const int me = c->cfg.rank;
  if (c->esz == 4) {
    if (c->cfg.error_feedback)
      k_peer_contribute<float, true><<<grid, 256, 0, c->stream>>>(pb, me, c->sel_cap, (float*)c->resid[0], corr);
    else
      k_peer_contribute<float, false><<<grid, 256, 0, c->stream>>>(pb, me, c->sel_cap, (float*)c->resid[0], corr);
  } else {
    if (c->cfg.error_feedback)
      k_peer_contribute<double, true><<<grid, 256, 0, c->stream>>>(pb, me, c->sel_cap, (double*)c->resid[0], corr);
    else
      k_peer_contribute<double, false><<<grid, 256, 0, c->stream>>>(pb, me, c->sel_cap, (double*)c->resid[0], corr);
  }
  CU(cudaGetLastError());
  c->peer_phase = 1;
  return MICRO_OK;
}

int micro_peer_reduce(micro_ctx* c) {
  TRY(check_peer_ctx(c));
  if (c->peer_phase != 1) return fail(MICRO_ELOGIC, "micro_peer_reduce before micro_peer_contribute");
  DeviceGuard dg(c->dev);
  const PeerBulkPtrs pb = bulk_ptrs(c);
  // two entries per thread for the expected selection (the kernel reads the real count)
  const unsigned grid = grid_for(std::min<int64_t>((int64_t)c->k_worker * 3 / 4 + 1, c->sel_cap), c->dev);
  long long* Kout = c->Kbuf + c->buf;
  if (c->esz == 4)
    k_peer_reduce_push<float><<<grid, 256, 0, c->stream>>>(pb, c->n, c->cfg.rank, c->t_cur, c->sel_cap,
                                                           c->sel_idx[c->buf][0],
                                                           (const float*)c->sel_val[c->buf][0], Kout);
  else
    k_peer_reduce_push<double><<<grid, 256, 0, c->stream>>>(pb, c->n, c->cfg.rank, c->t_cur, c->sel_cap,
                                                            c->sel_idx[c->buf][0],
                                                            (const double*)c->sel_val[c->buf][0], Kout);
  CU(cudaGetLastError());
  c->peer_phase = 2;
  return MICRO_OK;
}

int micro_peer_finalize(micro_ctx* c) {
  TRY(check_peer_ctx(c));
  if (c->peer_phase != 2) return fail(MICRO_ELOGIC, "micro_peer_finalize before the exchange");
  DeviceGuard dg(c->dev);
  c->peer_phase = 0;
  if (c->esz == 4) return launch_finalize<float>(c, c->uni_idx[c->buf], c->uni_sum[c->buf], 0);
  return launch_finalize<double>(c, c->uni_idx[c->buf], c->uni_sum[c->buf], 0);
}

// ---- device memory plumbing ----


// ---- one process driving all n ranks (peer access instead of CUDA IPC) ----

int micro_group_attach(micro_ctx* const* ctxs, int n) {
  if (!ctxs || n < 2 || n > MICRO_MAX_WORKERS) return fail(MICRO_EINVAL, "micro_group_attach: need 2..64 contexts");
  for (int r = 0; r < n; ++r) {
    TRY(check_peer_ctx(ctxs[r]));
    if (ctxs[r]->n != n || ctxs[r]->cfg.rank != r)
      return fail(MICRO_EINVAL, "micro_group_attach: context %d is not rank %d of %d", r, r, n);
    if (ctxs[r]->peer_ready) return fail(MICRO_ELOGIC, "micro_group_attach: context %d already attached", r);
    if (ctxs[r]->n_g != ctxs[0]->n_g || ctxs[r]->esz != ctxs[0]->esz || ctxs[r]->norm != ctxs[0]->norm)
      return fail(MICRO_EINVAL, "micro_group_attach: contexts disagree on n_g / dtype / error norm");
  }
  for (int r = 0; r < n; ++r) {  // peer access between distinct devices, receive slabs
    micro_ctx* c = ctxs[r];
    DeviceGuard dg(c->dev);
    for (int q = 0; q < n; ++q) {
      const int d = ctxs[q]->dev;
      if (d == c->dev) continue;
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, c->dev, d));
      if (!can) return fail(MICRO_ECUDA, "device %d cannot access device %d", c->dev, d);
      const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(MICRO_ECUDA, "cudaDeviceEnablePeerAccess(%d): %s", d, cudaGetErrorString(e));
      cudaGetLastError();  // clear "already enabled"
    }
    if (!c->recv) TRY(c->alloc(&c->recv, (size_t)c->n * c->sel_cap * c->esz));
    if (!c->group_ev) CU(cudaEventCreateWithFlags(&c->group_ev, cudaEventDisableTiming));
  }
  for (int r = 0; r < n; ++r) {
    micro_ctx* c = ctxs[r];
    for (int q = 0; q < n; ++q) {
      micro_ctx* o = ctxs[q];
      c->peer_resid[q] = o->resid[0];
      c->peer_counts[q] = o->counts;
      c->peer_uidx[0][q] = o->uni_idx[0];
      c->peer_uidx[1][q] = o->uni_idx[1];
      c->peer_usum[0][q] = o->uni_sum[0];
      c->peer_usum[1][q] = o->uni_sum[1];
      c->peer_corr[q] = c->norm ? o->norm_slot : nullptr;
      c->peer_sel[0][q] = o->sel_idx[0][0];
      c->peer_sel[1][q] = o->sel_idx[1][0];
      c->peer_recv[q] = o->recv;
    }
    c->peer_ready = true;
  }
  return MICRO_OK;
}

// every context's stream waits for every other's work so far (a device-side
// barrier built from events: the host never blocks)
static int group_barrier(micro_ctx* const* ctxs, int n) {
  for (int r = 0; r < n; ++r) {
    DeviceGuard dg(ctxs[r]->dev);
    CU(cudaEventRecord(ctxs[r]->group_ev, ctxs[r]->stream));
  }
  for (int r = 0; r < n; ++r) {
    DeviceGuard dg(ctxs[r]->dev);
    for (int q = 0; q < n; ++q)
      if (q != r) CU(cudaStreamWaitEvent(ctxs[r]->stream, ctxs[q]->group_ev, 0));
  }
  return MICRO_OK;
}

int micro_group_step(micro_ctx* const* ctxs, int n, const void* const* d_grads, double eta, int64_t t) {
  if (!ctxs || !d_grads || n < 2) return fail(MICRO_EINVAL, "micro_group_step: bad arguments");
  for (int r = 0; r < n; ++r)
    if (!ctxs[r] || !ctxs[r]->peer_ready) return fail(MICRO_ELOGIC, "micro_group_step before micro_group_attach");
  for (int r = 0; r < n; ++r) TRY(micro_compress(ctxs[r], d_grads + r, eta, t));
  TRY(group_barrier(ctxs, n));
  for (int r = 0; r < n; ++r) TRY(micro_peer_contribute(ctxs[r]));
  TRY(group_barrier(ctxs, n));
  for (int r = 0; r < n; ++r) TRY(micro_peer_reduce(ctxs[r]));
  TRY(group_barrier(ctxs, n));
  for (int r = 0; r < n; ++r) TRY(micro_peer_finalize(ctxs[r]));
  return MICRO_OK;
}

}  // extern "C"
