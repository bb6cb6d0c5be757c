// internal.cuh — shared by the library's translation units (api.cu: the
// engine; dist_api.cu: one rank of an n-GPU job; value_api.cu: the stateless
// value-level calls).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/micro.h"
#include "../../include/micro_synth.h"
#include "baselines.cuh"
#include "exchange.cuh"
#include "peer.cuh"
#include "scan.cuh"
#include "select_stream.cuh"

namespace micro {
namespace host {

// ---- errors: the message of the last failing call on this thread ----
extern thread_local std::string g_err;
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

#define CU(call)                                                                           \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return ::micro::host::fail(MICRO_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                                 __FILE__, __LINE__);                                      \
  } while (0)

#define TRY(call)                    \
  do {                               \
    int _rc = (call);                \
    if (_rc != MICRO_OK) return _rc; \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline size_t dtype_size(int dtype) { return dtype == MICRO_F64 ? 8 : 4; }
int check_dtype(int dtype);
int num_sms(int dev);
unsigned grid_for(int64_t work, int dev);
int current_device();

// pure host restatements (shared by the C ABI and the engine)
int h_partition(int64_t n_g, int n, int64_t t, int worker, int64_t* start, int64_t* end);
int h_global_target(double d, int64_t n_g, uint64_t* k);
int h_worker_target(double d, int64_t n_g, int n, int target, uint64_t* k);
int h_update_threshold(double* delta, uint64_t k_target, uint64_t k_sel, double alpha, double eps);

constexpr int64_t kHistCap = 4096;
constexpr int kTimingCap = 1024;

// Launch with programmatic stream serialization (PDL) when `pdl`: the kernel
// may begin while its predecessor drains and waits in pdl_wait().
template <typename... P, typename... A>
cudaError_t launch_maybe_pdl(bool pdl, void (*kern)(P...), dim3 grid, dim3 block, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

template <typename... P, typename... A>
cudaError_t launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, cudaStream_t st, A&&... args) {
  return launch_maybe_pdl(true, kern, grid, block, st, std::forward<A>(args)...);
}

}  // namespace host
}  // namespace micro

// (the translation units bring micro:: and micro::host:: into scope themselves)
namespace micro {
namespace host {
using namespace ::micro;
}  // namespace host
}  // namespace micro

// ------------------------------------------------------------ the context --

struct micro_ctx {
  micro_config cfg{};
  int dev = 0;
  cudaStream_t stream = nullptr;
  int n = 1, n_local = 1;
  int64_t n_g = 0;
  size_t esz = 4;
  size_t gsz = 4;  // gradient element size (esz, or 4 for fp32 gradients into fp64 state)
  uint64_t k_worker = 0;
  int64_t sel_cap = 0, uni_cap = 0;
  bool cluster = true;  // n_local == n
  // per local worker
  std::vector<void*> resid;
  std::vector<int32_t*> sel_idx[2];
  std::vector<void*> sel_val[2];
  long long* counts = nullptr;    // n_local
  double* delta = nullptr;        // n_local
  // union (n > 1), double-buffered for the dense sparse-clear
  int32_t* uni_idx[2] = {nullptr, nullptr};
  void* uni_sum[2] = {nullptr, nullptr};
  long long* Kbuf = nullptr;      // [2]
  void* dense = nullptr;
  void* model = nullptr;
  // K1 workspace (k1_stream -> k1_gather)
  int32_t* stage_idx = nullptr;  // per-CTA staging runs
  void* stage_val = nullptr;
  int* unit_counts = nullptr;    // selections per K1 unit / per k1_stream CTA run
  // k1_stream -> k1_gather: selections per super block of super_runs CTA
  // runs, two parities (a launch zeroes the other one for the next launch)
  int* super_counts = nullptr;
  int super_runs = 8;
  int super_par = 0;
  int* flags = nullptr;
  // history
  long long *hist_t = nullptr, *hist_K = nullptr, *hist_counts = nullptr;
  double* hist_delta = nullptr;
  double* hist_err = nullptr;
  // error norm (record_error_norm, EF on): ||e_{t+1}||^2 per worker, fused into K1
  bool norm = false;
  int64_t norm_ctas = 0;               // slots for the largest producing grid
  double* norm_part = nullptr;
  double* norm_group = nullptr;
  unsigned* norm_ticket = nullptr;     // norm_groups + 1
  micro::NormSlot* norm_slot = nullptr;  // n_local: ||e||^2 after K1 + the exchange's corrections (norm.cuh)
  // host-side step state
  int64_t steps = 0;      // completed aggregations
  int64_t t_cur = -1;     // iteration of the pending/last compress
  int buf = 0;            // buffer parity of the pending/last step
  bool compressed = false;
  bool poisoned = false;
  bool ever_stepped = false;
  void* staging = nullptr;  // gradient staging (lazy): host inputs, unaligned device inputs
  size_t staging_stride = 0;  // bytes per worker row (256-byte aligned)
  // the previous union's dense clear runs on `aux`, overlapping K1 (fork at
  // compress, join before finalize)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool clear_pending = false;
  // n = 1 with the streaming K1: the dense g/n is maintained inside K1
  // (k1_stream<..., kDense>) with one dirty bit per 32-byte sector
  bool dense_fused = false;
  // micro_step on a one-worker cluster with the streaming K1: k1_gather's
  // block 0 does the threshold update + history (no k_finalize launch)
  bool fuse_step = false;   // set for the duration of micro_step
  bool fin_done = false;    // this step's finalize already ran inside k1_gather
  // optional in-library kernel timing of K1's streaming pass (micro_kernel_times)
  // micro_step_host (n = 1): the gradient arrives in kH2DChunks pieces on
  // h2d_stream; K1 streams each piece's CTAs as soon as it has landed
  static constexpr int kH2DChunks = 8;
  int h2d_chunks = 0;        // > 1 only while micro_step_host runs
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t h2d_ev[kH2DChunks] = {};
  cudaEvent_t h2d_free = nullptr;  // the previous step is done with the staging buffer
  bool timing = false;
  int timing_period = 1;   // record every timing_period-th k1_stream launch
  int64_t t_seen = 0;
  int t_next = 0;
  std::vector<cudaEvent_t> t_ev;
  unsigned long long* dense_dirty = nullptr;
  std::vector<void*> allocs;
  // comparison sparsifiers (micro_config.sparsifier, baselines.cuh)
  int kind = 0;                 // 0 MiCRO, 1 top-k, 2 CLT-k, 3 hard threshold, 4 dense
  bool vectors_done = false;    // this step's model / dense g/n already written (dense kind)
  bool sel_is_union = false;    // n = 1 MiCRO: the union is worker 0's selection
  uint64_t k_global = 0;
  micro::TopkState* topk = nullptr;    // n_local
  unsigned* topk_hist = nullptr;
  unsigned* tie_counts = nullptr;
  unsigned* bitmap = nullptr;   // union of overlapping selections
  int* word_off = nullptr;
  int* scan_tmp = nullptr;      // block totals of the hand-written scan (scan.cuh)
  int64_t nwords = 0;
  double* minus_one = nullptr;  // threshold that selects everything (k >= n_g)
  // peer-memory exchange (micro_peer_*): every rank's buffers mapped here
  bool peer_ready = false;
  const long long* peer_counts[micro::kMaxWorkers] = {};
  void* peer_resid[micro::kMaxWorkers] = {};
  int32_t* peer_uidx[2][micro::kMaxWorkers] = {};
  void* peer_usum[2][micro::kMaxWorkers] = {};
  micro::NormSlot* peer_corr[micro::kMaxWorkers] = {};
  const int32_t* peer_sel[2][micro::kMaxWorkers] = {};
  void* peer_recv[micro::kMaxWorkers] = {};
  void* recv = nullptr;          // bulk exchange / collective protocol: receive slabs [source rank][sel_cap] (lazy)
  // the collective protocol (micro_dist_*, nccl_api.cu): fixed stride sel_cap per rank (lazy)
  long long* dist_all_counts = nullptr;  // [n]
  int32_t* dist_all_idx = nullptr;       // [n][sel_cap]
  void* dist_send = nullptr;             // [n][sel_cap]: segment o -> owner o
  void* dist_own_sums = nullptr;         // [sel_cap]
  void* dist_all_sums = nullptr;         // [n][sel_cap]
  int peer_phase = 0;            // 0 idle, 1 contributed (bulk), 2 exchanged (ready to finalize)
  cudaEvent_t group_ev = nullptr;  // micro_group_step barriers (one process, all ranks)
  // NCCL attached (nccl_api.cu): micro_aggregate runs the n-GPU exchange
  void* nccl_comm = nullptr;     // ncclComm_t
  bool nccl_owned = false;       // made by micro_dist_init_nccl: destroyed with the context
  int xchg = 0;                  // MICRO_XCHG_PEER / MICRO_XCHG_NCCL
  int* nccl_bar = nullptr;       // 4-byte barrier all-reduce buffer
  std::vector<void*> peer_opened;  // cudaIpcOpenMemHandle mappings to close

  int alloc(void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess)
      return micro::host::fail(MICRO_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    allocs.push_back(*p);
    return MICRO_OK;
  }
};

namespace micro {
namespace host {

// 0: error norm not recorded, 1: recorded (EF on), 2: residual is zero (EF off)
inline int norm_mode(const micro_ctx* c) { return !c->cfg.error_feedback ? 2 : c->norm ? 1 : 0; }
int check_ctx(micro_ctx* c);
int check_poison(micro_ctx* c);
int ensure_staging(micro_ctx* c);
int dist_ensure_buffers(micro_ctx* c);
int nccl_aggregate(micro_ctx* c);  // nccl_api.cu
void nccl_release(micro_ctx* c);
int read_flags(micro_ctx* c, int* flags);
// word offsets of a union bitmap: off[w] = popcount of words [0, w) (scan.cuh);
// `tiles` holds scan_tiles(nwords) ints of scratch
int bitmap_offsets(const unsigned* bitmap, int64_t nwords, int* off, int* tiles, cudaStream_t st,
                   long long* total = nullptr);
// threshold update, history, dense g/n and model after the union is formed
// (instantiated for float and double in api.cu)
template <typename T>
int launch_finalize(micro_ctx* c, const int32_t* uidx, const void* usum, int k_from_counts);

}  // namespace host
}  // namespace micro
