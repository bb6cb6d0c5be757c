/*
 * micro.h — C ABI of the B200-native MiCRO sparsify + aggregate path.
 *
 * Drop-in boundary for the reference's hot path (sparsim, /root/reference/proj):
 * every entry point below names the reference interface it replaces
 * (paths relative to /root/reference/proj).  Plain pointers and sizes only; no
 * torch or C++ types.  Device pointers are CUDA global-memory addresses on the
 * context's device; streams are cudaStream_t passed as void*.
 *
 * Status codes map 1:1 onto the reference's exception types:
 *   MICRO_EINVAL     <-> std::invalid_argument
 *   MICRO_ELOGIC     <-> std::logic_error
 *   MICRO_ENONFINITE <-> std::runtime_error ("non-finite gradient", harness.cpp:128-130)
 * The message of the last failing call on the calling thread is returned by
 * micro_last_error(); it carries the reference's message text where one exists.
 *
 * Element types: MICRO_F32 is the north-star contract (fp32 gradients,
 * fp32 residuals, fp64 thresholds); MICRO_F64 runs the identical kernels in the
 * reference's own precision and is bit-exact against its compiled code; with
 * micro_config.grad_dtype = MICRO_GRAD_F32 the fp64 engine takes fp32
 * gradients (widened exactly: the reference's result on the same values).
 */
#ifndef MICRO_H
#define MICRO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MICRO_ABI_VERSION 5  /* 5: micro_config.grad_dtype */
#define MICRO_MAX_WORKERS 64

typedef enum micro_status {
  MICRO_OK = 0,
  MICRO_EINVAL = 1,
  MICRO_ELOGIC = 2,
  MICRO_ENONFINITE = 3,
  MICRO_ECUDA = 4,
  MICRO_ENCCL = 5,
  MICRO_ECAPACITY = 6,
  MICRO_ENOMEM = 7
} micro_status;

typedef enum micro_dtype { MICRO_F32 = 0, MICRO_F64 = 1 } micro_dtype;

/* sparsifier.hpp:26 PerWorkerTarget */
typedef enum micro_target { MICRO_TARGET_SPLIT = 0, MICRO_TARGET_FULL = 1 } micro_target;

int micro_abi_version(void);
const char* micro_status_string(int status);
/* Message of the last non-OK return on this thread ("" if none). */
const char* micro_last_error(void);

/* ---- pure host functions (no device work) ------------------------------- */

/* tensor.hpp:48-63 partition(n_g, n, t, worker) -> [start, end) */
int micro_partition(int64_t n_g, int n, int64_t t, int worker, int64_t* start, int64_t* end);
/* sparsifier.cpp:110-116 global_target_count */
int micro_global_target_count(double density, int64_t n_g, uint64_t* k);
/* sparsifier.cpp:118-125 per_worker_target_count */
int micro_per_worker_target_count(double density, int64_t n_g, int n, int target, uint64_t* k);
/* sparsifier.cpp:69-83 micro_update_threshold (in/out *delta) */
int micro_update_threshold(double* delta, uint64_t k_target, uint64_t k_selected, double alpha,
                           double min_threshold);

/* ---- stateless device operations (value-level API) ---------------------- *
 * All pointers are device pointers; work is enqueued on `stream`; counts that
 * the host needs are returned through device memory (d_count) so nothing
 * synchronises unless stated.                                               */

/* error_feedback.hpp:17-23 accumulate: acc = e + eta*g (two roundings). */
int micro_accumulate(int dtype, const void* d_e, double eta, const void* d_g, void* d_acc,
                     int64_t n, void* stream);
/* sparsifier.cpp:22-37 select_by_threshold: ascending (idx, acc[idx]) with
 * |acc| > delta inside [start, end).  Writes at most `cap` pairs; *d_count
 * (device int64) receives the full count (> cap => MICRO_ECAPACITY at the next
 * synchronising call of this thread, see micro_sync). */
int micro_select_by_threshold(int dtype, const void* d_acc, int64_t n_g, int64_t start,
                              int64_t end, double delta, int32_t* d_idx, void* d_val,
                              int64_t cap, int64_t* d_count, void* stream);
/* sparsifier.cpp:39-67 select_topk: the k largest |acc| in [start, end),
 * ties to the lower index, ascending; k > end - start is MICRO_EINVAL.
 * (cltk_select is this over the whole vector; select_all is a copy.) */
int micro_select_topk(int dtype, const void* d_acc, int64_t n_g, int64_t start, int64_t end, int64_t k,
                      int32_t* d_idx, void* d_val, int64_t cap, int64_t* d_count, void* stream);
/* error_feedback.hpp:27-39 compensate (in place): acc[idx[k]] = 0. */
int micro_compensate(int dtype, void* d_acc, int64_t n_g, const int32_t* d_idx, int64_t k,
                     void* stream);
/* collectives.cpp:30-49 all_reduce_sparse_values: sums[k] = sum over workers
 * in order of accs[i][union[k]], starting from +0.  h_accs: host array of n
 * device pointers. */
int micro_all_reduce_sparse_values(int dtype, const void* const* h_accs, int n, int64_t n_g,
                                   const int32_t* d_union, int64_t K, void* d_sums, void* stream);
/* collectives.cpp:51-57 all_reduce_sparse: dense n_g result, sums at the union. */
int micro_all_reduce_sparse(int dtype, const void* const* h_accs, int n, int64_t n_g,
                            const int32_t* d_union, int64_t K, void* d_dense, void* stream);
/* collectives.cpp:14-28 all_gather_indices: sorted unique union of n sorted
 * index lists (device, concatenated in worker order, h_counts on host).
 * Synchronises; *K returns the union size. */
int micro_all_gather_indices(int n, const int64_t* h_counts, const int32_t* d_concat,
                             int32_t* d_union, int64_t* K, void* stream);
/* error_feedback.hpp:41-48 error_metric: (sum_i ||e_i||_2) / n over n device
 * residuals of n_g entries (h_res: host array of device pointers), norms
 * summed in worker order.  Each ||e_i||^2 is a deterministic fp64 tree sum
 * (the reference's Eigen summation order is not pinned).
 * Synchronises. */
int micro_error_metric(int dtype, const void* const* h_res, int n, int64_t n_g, double* out,
                       void* stream);

/* Device memory plumbing for hosts without the CUDA runtime (the C++
 * drop-in, sparsim_b200.hpp).  kind: 0 host->device, 1 device->host,
 * 2 device->device.  micro_memcpy synchronises `stream`. */
int micro_device_malloc(void** d_ptr, int64_t bytes, int device);
int micro_device_free(void* d_ptr);
/* Pinned (page-locked) host memory: full-bandwidth H2D/D2H for step_host. */
int micro_host_malloc(void** h_ptr, int64_t bytes);
int micro_host_free(void* h_ptr);
int micro_memcpy(void* dst, const void* src, int64_t bytes, int kind, void* stream);
/* The value-level calls above take their scratch (up to (4 + esz) bytes per
 * element of the range) from a library-owned stream-ordered pool per device
 * that keeps freed blocks reserved, so repeated calls do not re-map it;
 * this returns the reserve of `device` to the driver. */
int micro_value_workspace_trim(int device);
int micro_device_count(int* count);
/* The calling thread's current CUDA device (what micro_synth_gaussian and
 * the value-level calls launch on). */
int micro_set_device(int device);

/* Synthetic N(0,1) gradients of include/micro_synth.h (bench/test inputs). */
int micro_synth_gaussian(int dtype, uint64_t seed, uint32_t worker, uint64_t t, int64_t n,
                         void* d_out, void* stream);

/* ---- the MiCRO engine (run_iteration's MiCRO branch, harness.cpp:121-224) -- *
 * A context holds `n_local` workers of an n-worker cluster on one device: the
 * residuals e_i (harness.hpp:51), thresholds delta_i (:52), selection and
 * union buffers, the dense averaged gradient and the look-back workspace.
 *   n_local == n_workers : the whole cluster lives on this device (the
 *                          reference's in-process ClusterState); micro_step
 *                          runs the complete iteration.
 *   n_local == 1 < n     : one rank of a multi-GPU job (one process per GPU);
 *                          micro_compress runs K1, the host moves counts,
 *                          indices and values between ranks (NCCL), and the
 *                          micro_dist_* calls run the device halves.        */

typedef struct micro_ctx micro_ctx;

typedef struct micro_config {
  int64_t n_g;              /* gradient length */
  int32_t n_workers;        /* n */
  int32_t n_local;          /* n (single-device cluster) or 1 (one rank) */
  int32_t rank;             /* worker id of the (first) local worker */
  int32_t dtype;            /* micro_dtype */
  double density;           /* d in (0,1]            sparsifier.hpp:41 */
  double initial_threshold; /* delta_0 >= 0          sparsifier.hpp:42 */
  double scaling_factor;    /* alpha in (0,1)        sparsifier.hpp:43 */
  double min_threshold;     /* eps_delta > 0         sparsifier.hpp:44 */
  int32_t target;           /* micro_target          sparsifier.hpp:45 */
  int32_t error_feedback;   /* RunConfig::error_feedback, harness.hpp:46 */
  int32_t dense_output;     /* keep the dense averaged gradient g/n on device */
  int32_t device;           /* CUDA device ordinal */
  int64_t selection_capacity; /* pairs per worker; 0 = partition size (never overflows) */
  int32_t record_error_norm;  /* per-step error norm ||e_{t+1}||_2 (harness.cpp:230-235), fused
                                 into K1; 0 = not recorded (NaN in micro_records) */
  int32_t sparsifier;         /* SparsifierKind (sparsifier.hpp:21): MICRO_MICRO (default) or a
                                 comparison sparsifier of harness.cpp:152-181 (single-device
                                 cluster only) */
  int32_t grad_dtype;         /* element type of the gradients passed to micro_compress /
                                 micro_step / micro_step_host: MICRO_GRAD_SAME (0, default) = dtype;
                                 MICRO_GRAD_F32 = fp32 gradients (BASELINE's "fp32 gradient") into
                                 fp64 state and arithmetic (dtype MICRO_F64, MiCRO only).  (double)g
                                 is exact, so results equal the reference's run on the same gradient
                                 values; G moves 4 B per element instead of 8. */
} micro_config;

/* gradient element types (micro_config.grad_dtype) */
enum { MICRO_GRAD_SAME = 0, MICRO_GRAD_F32 = 1 };

/* sparsifier kinds (sparsifier.hpp:21) */
enum {
  MICRO_MICRO = 0,  /* threshold in the exclusive cyclic partition (the path)  */
  MICRO_TOPK = 1,   /* select_topk over the whole vector, ties -> lower index    */
  MICRO_CLTK = 2,   /* cltk_select: the leader t mod n's top-k only               */
  MICRO_HARD = 3,   /* hard_threshold_select: |acc| > initial_threshold (fixed)   */
  MICRO_DENSE = 4   /* select_all                                                 */
};

void micro_config_default(micro_config* cfg);

int micro_ctx_create(micro_ctx** ctx, const micro_config* cfg, void* stream);
int micro_ctx_destroy(micro_ctx* ctx);
/* Back to t = 0 state: residuals 0, thresholds delta_0, errors cleared. */
int micro_ctx_reset(micro_ctx* ctx);
void* micro_ctx_stream(micro_ctx* ctx);

/* Optional model x (device, n_g elements of dtype): every aggregation applies
 * x[j] -= sum_j / n at the union (harness.cpp:210-215).  NULL disables. */
int micro_set_model(micro_ctx* ctx, void* d_x);

/* K1 for each local worker: acc_i = e_i + eta*G_i over all n_g, select
 * |acc_i| > delta_i in partition(n_g, n, t, i), ordered compaction into
 * (index, value) pairs, own selections zeroed in the residual.  d_grads: host
 * array of n_local device pointers.  Asynchronous. */
int micro_compress(micro_ctx* ctx, const void* const* d_grads, double eta, int64_t t);
/* Single-device cluster: union + ordered all-worker reduce + foreign zeroing
 * + threshold update + dense g/n (+ model).  A rank context with NCCL
 * attached (micro_dist_attach_nccl): the n-GPU exchange + finalize.
 * Asynchronous. */
int micro_aggregate(micro_ctx* ctx);
/* micro_compress + micro_aggregate. */
int micro_step(micro_ctx* ctx, const void* const* d_grads, double eta, int64_t t);
/* End to end with host buffers: pinned host gradients (n_local * n_g) are
 * copied in, the step runs, and the union (indices + sums, at most cap) is
 * copied out.  Synchronises; returns MICRO_ENONFINITE / MICRO_ECAPACITY. */
int micro_step_host(micro_ctx* ctx, const void* h_grads, double eta, int64_t t,
                    int32_t* h_union_idx, void* h_union_sum, int64_t cap, int64_t* K);

/* Synchronise the context's stream and report deferred device errors
 * (non-finite gradient, capacity overflow).  After MICRO_ENONFINITE the
 * context is poisoned until micro_ctx_reset (residuals hold NaN/Inf). */
int micro_sync(micro_ctx* ctx);

typedef struct micro_stats {
  int64_t t;               /* iteration of the last step */
  int64_t steps;           /* completed steps since create/reset */
  int64_t K;               /* |union| of the last step */
  int64_t total_selected;  /* sum_i k_i of the last step (== K for MiCRO) */
  int32_t nonfinite;
  int32_t overflow;
} micro_stats;

/* Synchronises.  counts/deltas: n_local entries each (may be NULL):
 * k_i of the last step and delta_i for the NEXT step. */
int micro_query(micro_ctx* ctx, micro_stats* st, int64_t* counts, double* deltas);
/* Per-step history ring (last min(max, steps, 4096) steps), synchronises.
 * K[s], counts[s*n_local+i], delta_used[s*n_local+i]. Returns the number of
 * steps written in *written. */
int micro_history(micro_ctx* ctx, int64_t max, int64_t* t, int64_t* K, int64_t* counts,
                  double* delta_used, int64_t* written);

/* The reference's per-iteration record (IterationRecord, metrics.hpp:15-29;
 * filled at harness.cpp:226-236) for the MiCRO path's scalars; the task
 * loss and the modeled phase times are outside this path. */
typedef struct micro_record {
  int64_t t;
  int64_t K;                        /* |union| */
  int64_t total_selected;           /* sum_i k_i (this context's workers; K on a rank of n) */
  double actual_density;            /* K / n_g (metrics.cpp:7-10) */
  double buildup_factor;            /* K / k_global, 0 if nothing selected (collectives.cpp:59-63) */
  double redundant_traffic_factor;  /* total_selected / K, 0 if nothing (collectives.cpp:65-69) */
  double error_norm;                /* (sum_i ||e_{i,t+1}||_2) / n_local; NaN if not recorded */
  double threshold;                 /* (sum_i delta_i used) / n_local (harness.cpp:139-149) */
} micro_record;

/* Records of the last min(max, steps, 4096) steps, oldest first; synchronises. */
int micro_records(micro_ctx* ctx, int64_t max, micro_record* out, int64_t* written);

/* Diagnostics: CUDA-event timing of K1's streaming pass (k1_stream) inside
 * the library.  micro_kernel_timing(p), p >= 1, starts recording every p-th
 * launch (up to 1024 recorded, restarting the count; 0 stops);
 * micro_kernel_times synchronises and returns the per-launch durations in ms. */
int micro_kernel_timing(micro_ctx* ctx, int enable);
int micro_kernel_times(micro_ctx* ctx, float* ms, int max, int* written);

/* Device views, valid until the next step on this context. */
int micro_union_device(micro_ctx* ctx, const int32_t** d_idx, const void** d_sums,
                       const int64_t** d_K);
int micro_dense_device(micro_ctx* ctx, const void** d_dense);
int micro_residual_device(micro_ctx* ctx, int local_worker, void** d_resid);
int micro_selection_device(micro_ctx* ctx, int local_worker, const int32_t** d_idx,
                           const void** d_val, const int64_t** d_count);
int micro_threshold_device(micro_ctx* ctx, double** d_delta);
/* Host copies (synchronise). */
int micro_copy_union(micro_ctx* ctx, int32_t* h_idx, void* h_sums, int64_t cap, int64_t* K);
int micro_copy_residual(micro_ctx* ctx, int local_worker, void* h_out);
int micro_copy_dense(micro_ctx* ctx, void* h_out);

/* ---- one rank of a multi-GPU job (n_local == 1 < n_workers) -------------- *
 * The collective protocol (collectives.cpp:14-57 semantics,
 * harness.cpp:185-224 order) as device halves around host-driven
 * collectives.  Every buffer has a fixed stride kcap (the selection
 * capacity, micro_config.selection_capacity or the partition size) per rank
 * and every count stays on the device, so the host never reads one: the
 * whole iteration is stream-ordered.  A selection larger than kcap raises
 * the overflow flag (MICRO_ECAPACITY at the next synchronising call).
 *   micro_compress                              own_count, own_idx
 *   all-gather own_count -> all_counts[n]       (int64)
 *   all-gather own_idx   -> all_idx[n][kcap]    (int32)
 *   micro_dist_gather_foreign                   send[o][kcap]: own acc at owner o's
 *                                               indices (zeroed in the residual)
 *   all-to-all: send[o] -> rank o's recv[me]    (kcap values per pair)
 *   micro_dist_owner_reduce                     own_sums[kcap]: rank-ordered sums
 *   all-gather own_sums  -> all_sums[n][kcap]
 *   micro_dist_finalize                         union, dense g/n, model, delta, stats
 * micro_dist_attach_nccl / micro_dist_init_nccl run exactly this (or the peer
 * exchange below) inside micro_aggregate with NCCL; dist.py runs it over
 * torch.distributed. */
typedef struct micro_dist_bufs {
  int64_t kcap;
  const int64_t* own_count; /* [1]   this rank's k_i */
  const int32_t* own_idx;   /* [kcap] this rank's selection, ascending */
  int64_t* all_counts;      /* [n]   <- all-gather of own_count */
  int32_t* all_idx;         /* [n][kcap] <- all-gather of own_idx */
  void* send;               /* [n][kcap] segment o goes to rank o */
  void* recv;               /* [n][kcap] segment r <- rank r's send[me] */
  void* own_sums;           /* [kcap] */
  void* all_sums;           /* [n][kcap] <- all-gather of own_sums */
} micro_dist_bufs;
int micro_dist_buffers(micro_ctx* ctx, micro_dist_bufs* out);
int micro_dist_gather_foreign(micro_ctx* ctx);
int micro_dist_owner_reduce(micro_ctx* ctx);
int micro_dist_finalize(micro_ctx* ctx);

/* ---- the exchange behind the C ABI over NCCL (no Python, no host sync) ---- *
 * One process per GPU, one rank context each.  Either the host brings its
 * own communicator (micro_dist_attach_nccl; an ncclComm_t of n ranks, rank ==
 * the context's rank), or the library makes one: rank 0 calls
 * micro_nccl_unique_id, the host hands the 128 bytes to every rank (MPI, a
 * file, ...), each calls micro_dist_init_nccl.  Afterwards micro_aggregate /
 * micro_step on the rank context run the whole exchange on ctx's stream:
 *   MICRO_XCHG_PEER  the bulk peer-memory exchange below (NVLink P2P through
 *                    CUDA IPC mappings made at attach, handles all-gathered
 *                    over NCCL); the three barriers are 4-byte ncclAllReduce
 *                    calls on ctx's stream.  The default.
 *   MICRO_XCHG_NCCL  the collective protocol above: ncclAllGather of the
 *                    counts, indices and sums, grouped ncclSend/ncclRecv for
 *                    the contributions (kcap per pair).
 * NCCL is loaded at attach (libnccl.so.2, the process's copy if one is
 * loaded); MICRO_ENCCL reports its errors. */
#define MICRO_NCCL_UNIQUE_ID_BYTES 128
enum { MICRO_XCHG_PEER = 0, MICRO_XCHG_NCCL = 1 };
int micro_nccl_unique_id(void* out);
int micro_dist_init_nccl(micro_ctx* ctx, const void* unique_id, int transport);
int micro_dist_attach_nccl(micro_ctx* ctx, void* nccl_comm, int transport);

/* ---- the same exchange as ONE kernel over peer memory (NVLink) ----------- *
 * Replaces K2..K7 above (collectives.cpp:14-57 semantics, harness.cpp:185-224
 * order) with no NCCL data movement and no host round trip:
 *   setup:  micro_peer_export -> all-gather the handle blobs (any transport)
 *           -> micro_peer_import(all ranks' blobs in rank order)
 *   step:   micro_compress
 *           barrier #1 (every rank's compress complete; e.g. a 4-byte
 *                       ncclAllReduce on ctx's stream)
 *           micro_peer_exchange  (owner: peer reads of acc_r[j] in rank order,
 *                                 peer zeroing, push (j, s_j) to every rank)
 *           barrier #2
 *           micro_peer_finalize  (threshold, history, dense g/n, model)
 * The handle blob holds CUDA IPC handles of this rank's residual, counts,
 * union buffers and error-norm slot. */
#define MICRO_PEER_HANDLE_BYTES 640
int micro_peer_export(micro_ctx* ctx, void* out);
int micro_peer_import(micro_ctx* ctx, const void* all_handles);
int micro_peer_exchange(micro_ctx* ctx);
int micro_peer_finalize(micro_ctx* ctx);
/* Bulk variant (every NVLink transfer contiguous; one more barrier):
 *   micro_compress, barrier, micro_peer_contribute (gather own acc at every
 *   other owner's indices — read from the owner, contiguous — zero them, write
 *   the values into the owner's receive slab), barrier, micro_peer_reduce
 *   (owner: rank-order sums from its slabs, push (j, s_j) to every rank),
 *   barrier, micro_peer_finalize. */
int micro_peer_contribute(micro_ctx* ctx);
int micro_peer_reduce(micro_ctx* ctx);

/* One process driving all n ranks (SURVEY.md 8b "micro_aggregate_all"):
 * ctxs[r] is rank r's context (n_local = 1, on any device); attach maps the
 * buffers directly (peer access between distinct devices, no IPC), and
 * micro_group_step runs compress -> contribute -> reduce -> finalize on every
 * rank's stream with event barriers between the phases (no host sync). */
int micro_group_attach(micro_ctx* const* ctxs, int n);
int micro_group_step(micro_ctx* const* ctxs, int n, const void* const* d_grads, double eta, int64_t t);

#ifdef __cplusplus
}
#endif

#endif /* MICRO_H */
