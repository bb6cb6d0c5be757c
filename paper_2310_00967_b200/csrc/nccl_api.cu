// nccl_api.cu — the n-GPU exchange behind the C ABI over NCCL (include/micro.h
// micro_dist_attach_nccl / micro_dist_init_nccl): a C++ host with one process
// per GPU runs the whole MiCRO iteration through micro_step on its rank
// context — no Python, and no host synchronisation inside the step.
//
// Two transports share the attach:
//   MICRO_XCHG_PEER  the bulk peer-memory exchange (peer.cuh: every NVLink
//                    transfer contiguous) with 4-byte ncclAllReduce barriers on
//                    the context's stream; the CUDA IPC handles of every rank's
//                    buffers are all-gathered over NCCL once, at attach.
//   MICRO_XCHG_NCCL  the collective protocol of SURVEY.md §8e with device-side
//                    counts and a fixed stride (exchange.cuh k_dist_*):
//                    all-gather counts + indices, grouped send/recv of the
//                    contributions, all-gather of the owners' sums.
// Reference semantics: collectives.cpp:14-57 (all_gather_indices,
// all_reduce_sparse_values, all_reduce_sparse), harness.cpp:185-224 order.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy the
// process already has, e.g. torch's), so the library itself loads on hosts
// without NCCL and reports MICRO_ENCCL only when an NCCL entry is called.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "internal.cuh"

using namespace micro;
using namespace micro::host;

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
  decltype(&ncclCommUserRank) CommUserRank = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

NcclApi load_nccl() {
  NcclApi a;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if loaded
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
    return a;
  }
  bool all = true;
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn) {
      all = false;
      a.why += std::string(a.why.empty() ? "" : ", ") + name;
    }
  };
  sym(a.GetUniqueId, "ncclGetUniqueId");
  sym(a.CommInitRank, "ncclCommInitRank");
  sym(a.CommDestroy, "ncclCommDestroy");
  sym(a.CommCount, "ncclCommCount");
  sym(a.CommUserRank, "ncclCommUserRank");
  sym(a.AllGather, "ncclAllGather");
  sym(a.AllReduce, "ncclAllReduce");
  sym(a.Send, "ncclSend");
  sym(a.Recv, "ncclRecv");
  sym(a.GroupStart, "ncclGroupStart");
  sym(a.GroupEnd, "ncclGroupEnd");
  sym(a.GetErrorString, "ncclGetErrorString");
  if (!all) a.why = "libnccl.so.2 lacks " + a.why;
  a.ok = all;
  return a;
}

const NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] { api = load_nccl(); });
  return &api;
}

#define NC(call)                                                                                          \
  do {                                                                                                    \
    const ncclResult_t _r = (call);                                                                       \
    if (_r != ncclSuccess)                                                                                \
      return fail(MICRO_ENCCL, "%s: %s (%s:%d)", #call, nccl_api()->GetErrorString(_r), __FILE__, __LINE__); \
  } while (0)

int need_nccl(const NcclApi** out) {
  const NcclApi* a = nccl_api();
  if (!a->ok) return fail(MICRO_ENCCL, "NCCL unavailable: %s", a->why.c_str());
  *out = a;
  return MICRO_OK;
}

ncclDataType_t value_type(const micro_ctx* c) { return c->esz == 8 ? ncclFloat64 : ncclFloat32; }

// 4-byte all-reduce on the context's stream: every rank's stream reaches
// this point before any rank's stream continues (stream-ordered, the host
// does not wait).
int barrier(micro_ctx* c) {
  const NcclApi* a = nccl_api();
  NC(a->AllReduce(c->nccl_bar, c->nccl_bar, 1, ncclInt32, ncclSum, (ncclComm_t)c->nccl_comm, c->stream));
  return MICRO_OK;
}

int check_rank_ctx(micro_ctx* c) {
  TRY(check_ctx(c));
  if (c->cluster || c->n_local != 1 || c->n < 2)
    return fail(MICRO_ELOGIC, "micro_dist_*_nccl: needs a rank context (n_local = 1 of n > 1 workers)");
  if (c->nccl_comm) return fail(MICRO_ELOGIC, "NCCL already attached to this context");
  return MICRO_OK;
}

int attach(micro_ctx* c, ncclComm_t comm, int transport, bool owned) {
  const NcclApi* a = nullptr;
  TRY(need_nccl(&a));
  if (transport != MICRO_XCHG_PEER && transport != MICRO_XCHG_NCCL)
    return fail(MICRO_EINVAL, "unknown exchange transport %d", transport);
  int count = 0, rank = -1;
  NC(a->CommCount(comm, &count));
  NC(a->CommUserRank(comm, &rank));
  if (count != c->n || rank != c->cfg.rank)
    return fail(MICRO_EINVAL, "communicator is rank %d of %d; the context is rank %d of %d", rank, count,
                c->cfg.rank, c->n);
  DeviceGuard dg(c->dev);
  if (!c->nccl_bar) TRY(c->alloc((void**)&c->nccl_bar, sizeof(int)));
  CU(cudaMemsetAsync(c->nccl_bar, 0, sizeof(int), c->stream));
  if (transport == MICRO_XCHG_PEER) {
    // every rank's IPC handle blob, all-gathered over NCCL (once)
    const size_t hb = MICRO_PEER_HANDLE_BYTES;
    std::vector<char> mine(hb), all(hb * c->n);
    TRY(micro_peer_export(c, mine.data()));
    char* dbuf = nullptr;
    CU(cudaMallocAsync((void**)&dbuf, hb * (c->n + 1), c->stream));
    CU(cudaMemcpyAsync(dbuf, mine.data(), hb, cudaMemcpyHostToDevice, c->stream));
    NC(a->AllGather(dbuf, dbuf + hb, hb, ncclChar, comm, c->stream));
    CU(cudaMemcpyAsync(all.data(), dbuf + hb, hb * c->n, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaFreeAsync(dbuf, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    TRY(micro_peer_import(c, all.data()));
  } else {
    TRY(dist_ensure_buffers(c));
  }
  c->nccl_comm = comm;
  c->nccl_owned = owned;
  c->xchg = transport;
  return MICRO_OK;
}

}  // namespace

namespace micro {
namespace host {

// micro_aggregate on a rank context with NCCL attached (api.cu)
int nccl_aggregate(micro_ctx* c) {
  const NcclApi* a = nullptr;
  TRY(need_nccl(&a));
  DeviceGuard dg(c->dev);
  const ncclComm_t comm = (ncclComm_t)c->nccl_comm;
  if (c->xchg == MICRO_XCHG_PEER) {
    TRY(barrier(c));  // every rank's K1 is done
    TRY(micro_peer_contribute(c));
    TRY(barrier(c));  // every contribution has landed in its owner's slab
    TRY(micro_peer_reduce(c));
    TRY(barrier(c));  // every owner has pushed its (index, sum) segment
    return micro_peer_finalize(c);
  }
  const int me = c->cfg.rank;
  const size_t kcap = (size_t)c->sel_cap;
  const ncclDataType_t vt = value_type(c);
  NC(a->GroupStart());
  NC(a->AllGather(c->counts, c->dist_all_counts, 1, ncclInt64, comm, c->stream));           // K2
  NC(a->AllGather(c->sel_idx[0][0], c->dist_all_idx, kcap, ncclInt32, comm, c->stream));     // K3
  NC(a->GroupEnd());
  TRY(micro_dist_gather_foreign(c));                                                        // K4
  NC(a->GroupStart());                                                                      // K5
  for (int r = 0; r < c->n; ++r) {
    if (r == me) continue;
    NC(a->Send((const char*)c->dist_send + r * kcap * c->esz, kcap, vt, r, comm, c->stream));
    NC(a->Recv((char*)c->recv + r * kcap * c->esz, kcap, vt, r, comm, c->stream));
  }
  NC(a->GroupEnd());
  TRY(micro_dist_owner_reduce(c));                                                          // K6
  NC(a->AllGather(c->dist_own_sums, c->dist_all_sums, kcap, vt, comm, c->stream));          // K7
  return micro_dist_finalize(c);                                                            // K8
}

void nccl_release(micro_ctx* c) {
  if (c->nccl_comm && c->nccl_owned && nccl_api()->ok) nccl_api()->CommDestroy((ncclComm_t)c->nccl_comm);
  c->nccl_comm = nullptr;
}

}  // namespace host
}  // namespace micro

extern "C" {

int micro_nccl_unique_id(void* out) {
  if (!out) return fail(MICRO_EINVAL, "null unique-id buffer");
  static_assert(sizeof(ncclUniqueId) == MICRO_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  const NcclApi* a = nullptr;
  TRY(need_nccl(&a));
  NC(a->GetUniqueId(reinterpret_cast<ncclUniqueId*>(out)));
  return MICRO_OK;
}

int micro_dist_init_nccl(micro_ctx* c, const void* unique_id, int transport) {
  TRY(check_rank_ctx(c));
  if (!unique_id) return fail(MICRO_EINVAL, "null unique id");
  const NcclApi* a = nullptr;
  TRY(need_nccl(&a));
  DeviceGuard dg(c->dev);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  ncclComm_t comm = nullptr;
  NC(a->CommInitRank(&comm, c->n, id, c->cfg.rank));
  const int rc = attach(c, comm, transport, true);
  if (rc != MICRO_OK) a->CommDestroy(comm);
  return rc;
}

int micro_dist_attach_nccl(micro_ctx* c, void* nccl_comm, int transport) {
  TRY(check_rank_ctx(c));
  if (!nccl_comm) return fail(MICRO_EINVAL, "null communicator");
  return attach(c, (ncclComm_t)nccl_comm, transport, false);
}

}  // extern "C"
