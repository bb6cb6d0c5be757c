// exchange.cuh — the aggregation half of the MiCRO step (K4..K9).
//
// Reference semantics (paths relative to /root/reference/proj):
//   union U = sorted unique of all S_i          collectives.cpp:14-28
//     (MiCRO partitions are disjoint, so U is the concatenation of the S_i
//      in PARTITION order — no sort; acceptance.cpp:93-118)
//   s_j = 0; for i = 0..n-1: s_j += acc_i[j]    collectives.cpp:39-47 (P1, P2)
//   delta_i <- update(delta_i, k_w, k_i)        harness.cpp:201-208
//   x[j] -= s_j / n                             harness.cpp:212-215
//   acc_i[j] = 0 for j in U, every worker       harness.cpp:219-221 (P3)
#pragma once

#include "common.cuh"
#include "norm.cuh"

namespace micro {

struct WorkerPtrs {
  const int32_t* sel_idx[kMaxWorkers];
  const void* sel_val[kMaxWorkers];
  void* resid[kMaxWorkers];
};

// Single-device cluster, n > 1: one block row per partition p; the owner's
// own value comes from its K1 pairs (its residual entry is already zeroed),
// every other worker's from its accumulator, summed in worker order.
// Counts beyond the selection capacity were not stored (K1 raised the
// overflow flag, reported at the next sync); consumers read at most `cap`.
__device__ __forceinline__ long long clamp_count(long long k, long long cap) { return k < cap ? k : cap; }

template <typename T, bool kZero, bool kFew = false>
__global__ void __launch_bounds__(256) k_cluster_reduce(WorkerPtrs w, const long long* counts,
                                                        long long cap, int n, int64_t t,
                                                        int32_t* union_idx, T* union_sum,
                                                        NormSlot* sq_corr) {
  // sq_corr (kZero, error norm on): per worker, the squares of the residual
  // entries zeroed here (foreign union indices), subtracted from K1's
  // ||e||^2 by k_finalize.  kFew (n <= 8): each thread keeps one partial
  // per worker in registers and the warps reduce them once at the end;
  // otherwise lane r of each warp accumulates worker r (r + 32 in a second
  // register) with one warp reduction per worker and iteration.  Either way
  // the per-CTA partials are fixed by the grid shape, and one
  // order-independent fixed-point add (norm.cuh fx_add) per block and worker
  // makes the total independent of CTA timing.
  __shared__ double s_corr[8][kMaxWorkers];
  pdl_wait();  // the workers' K1 results are complete
  pdl_trigger();
  const int p = blockIdx.y;
  const int owner = partition_owner(p, n, t);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long off = 0;
  for (int q = 0; q < p; ++q) off += clamp_count(counts[partition_owner(q, n, t)], cap);
  const long long k = clamp_count(counts[owner], cap);
  const int32_t* __restrict__ idx = w.sel_idx[owner];
  const T* __restrict__ val = (const T*)w.sel_val[owner];
  const bool corr = kZero && sq_corr != nullptr;  // grid-uniform
  double c_lo = 0.0, c_hi = 0.0;
  double qt[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) qt[u] = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = (long long)blockIdx.x * blockDim.x; b < k; b += stride) {  // warp-uniform trip count
    const long long m = b + threadIdx.x;
    const bool act = m < k;
    const int32_t j = act ? idx[m] : 0;
    T s = (T)0;
    // eight workers' entries in flight per thread (random reads, 64-byte L2
    // fetches), then summed strictly in worker order
    for (int r0 = 0; r0 < n; r0 += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u;
        v[u] = (T)0;
        if (act && r < n) v[u] = r == owner ? val[m] : ld_rand((const T*)w.resid[r] + j);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u;
        if (r >= n) break;
        s = add_rn(s, v[u]);
        if (kZero && act && r != owner) ((T*)w.resid[r])[j] = (T)0;
        if (kFew) {
          if (corr && r != owner) qt[u] += (double)v[u] * (double)v[u];  // v = 0 when !act
        } else if (corr && r != owner) {
          const double q = warp_sum_f64(act ? (double)v[u] * (double)v[u] : 0.0);
          if (lane == (r & 31)) {
            if (r < 32) c_lo += q;
            else c_hi += q;
          }
        }
      }
      if (kFew) break;
    }
    if (act) {
      union_idx[off + m] = j;
      union_sum[off + m] = s;
    }
  }
  if (corr) {
    if (kFew) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double q = warp_sum_f64(qt[u]);
        if (lane == 0 && u < n) s_corr[wid][u] = q;
      }
    } else {
      if (lane < n) s_corr[wid][lane] = c_lo;
      if (lane + 32 < n) s_corr[wid][lane + 32] = c_hi;
    }
    __syncthreads();
    if ((int)threadIdx.x < n) {
      double tot = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += s_corr[q][threadIdx.x];
      if (tot != 0.0) fx_add(sq_corr + threadIdx.x, tot);
    }
  }
}

// ---- one rank of an n-GPU job: the collective protocol's device halves ----
// Buffers have a fixed stride kcap (the selection capacity) per rank, and
// every count is read from device memory (the all-gathered k_r), so the host
// never reads a count: the protocol is stream-ordered end to end (the NCCL
// calls of nccl_api.cu, or torch.distributed in dist.py, move the buffers).

// K4: gather own acc at every OTHER owner's indices into send[o][kcap] and
// zero them there (harness.cpp:219-221).
template <typename T, bool kZero>
__global__ void __launch_bounds__(256) k_dist_gather_foreign(const int32_t* all_idx, const long long* all_counts,
                                                             long long kcap, int me, T* resid, T* send,
                                                             NormSlot* sq_corr) {
  __shared__ double s_corr[8];
  const int o = blockIdx.y;
  if (o == me) return;  // block-uniform
  pdl_wait();
  const long long k = clamp_count(all_counts[o], kcap);
  const int32_t* __restrict__ idx = all_idx + (int64_t)o * kcap;
  T* __restrict__ out = send + (int64_t)o * kcap;
  double q = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long m0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; m0 < k; m0 += 4 * stride) {
    int32_t j[4];
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (m0 + u * stride < k) j[u] = idx[m0 + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)  // four random reads in flight
      if (m0 + u * stride < k) v[u] = ld_rand(resid + j[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (m0 + u * stride < k) {
        out[m0 + u * stride] = v[u];
        if (kZero) {
          resid[j[u]] = (T)0;
          q += (double)v[u] * (double)v[u];
        }
      }
  }
  if (kZero && sq_corr) {  // squares of the zeroed entries (error norm, see k_cluster_reduce)
    q = warp_sum_f64(q);
    if ((threadIdx.x & 31) == 0) s_corr[threadIdx.x >> 5] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_corr[w];
      if (tot != 0.0) fx_add(sq_corr, tot);
    }
  }
}

// K6: as owner, s = 0; for r in rank order: s += contribution_r (recv[r][kcap];
// its own value from the K1 pairs).
template <typename T>
__global__ void __launch_bounds__(256) k_dist_owner_reduce(const T* own_val, const long long* all_counts,
                                                           const T* recv, long long kcap, int n, int me, T* sums) {
  pdl_wait();
  const long long k = clamp_count(all_counts[me], kcap);
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < k;
       m += (long long)gridDim.x * blockDim.x) {
    T s = (T)0;
    for (int r = 0; r < n; ++r) s = add_rn(s, r == me ? own_val[m] : recv[(int64_t)r * kcap + m]);
    sums[m] = s;
  }
}

// K8: lay the all-gathered (index, sum) lists out as the union in partition
// order; K = sum of the (clamped) counts.
template <typename T>
__global__ void __launch_bounds__(256) k_dist_build_union(const int32_t* all_idx, const T* all_sums,
                                                          const long long* all_counts, long long kcap, int n,
                                                          int64_t t, int32_t* union_idx, T* union_sum,
                                                          long long* K_out) {
  pdl_wait();
  const int p = blockIdx.y;
  const int owner = partition_owner(p, n, t);
  long long off = 0, K = 0;
  for (int q = 0; q < n; ++q) {
    const long long kq = clamp_count(all_counts[partition_owner(q, n, t)], kcap);
    if (q < p) off += kq;
    K += kq;
  }
  if (p == 0 && blockIdx.x == 0 && threadIdx.x == 0) *K_out = K;
  const long long k = clamp_count(all_counts[owner], kcap);
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < k;
       m += (long long)gridDim.x * blockDim.x) {
    union_idx[off + m] = all_idx[(int64_t)owner * kcap + m];
    union_sum[off + m] = all_sums[(int64_t)owner * kcap + m];
  }
}

struct FinalizeArgs {
  int n;                      // cluster size (divisor of the average)
  int n_local;
  int64_t n_g;
  int64_t t;
  const long long* counts;    // n_local, this step's k_i
  double* delta;              // n_local, updated in place
  unsigned long long k_target;
  double alpha, min_threshold;
  int k_from_counts;          // 1: K = sum counts (single-device cluster)
  long long cap;              // selection capacity per worker
  long long* K;               // in (k_from_counts == 0) / out
  const int32_t* union_idx;
  const void* union_sum;
  const int32_t* prev_idx;    // previous union (dense sparse-clear), may be NULL
  const long long* prev_K;
  void* dense;                // n_g or NULL
  void* model;                // n_g or NULL
  // history ring
  int64_t slot;
  long long* hist_t;
  long long* hist_K;
  long long* hist_counts;
  double* hist_delta;
  double* hist_err;           // per worker ||e_{t+1}||_2 (error_norm record)
  int norm_mode;              // 0: not recorded (NaN), 1: sqrt(sq - corrections), 2: residual is zero (EF off)
  int update_delta;           // 0: comparison sparsifiers (no threshold estimate, harness.cpp:201)
  NormSlot* slots;            // per worker: ||e||^2 after K1 (own selections zeroed) + the exchange's corrections
  int corr;                   // 1: subtract (and clear) the corrections (n > 1 MiCRO)
};

__device__ __forceinline__ long long lower_bound_i32(const int32_t* a, long long n, int64_t key) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Threshold update + history (block 0), then the dense g/n maintenance with
// whole 32-byte sectors: after k_dense_clear the dense vector is zero outside
// the current union, so the full content of every sector the union touches
// is known — avg at union slots, 0 elsewhere.  Each such sector is written
// once, in full, by its owner thread (its first union entry): no
// partial-sector read-modify-write in HBM.  The optional model update
// x -= avg (harness.cpp:212-215) is done by the same owner.
template <typename T>
__global__ void __launch_bounds__(256) k_finalize(FinalizeArgs a) {
  constexpr int SEC = 32 / (int)sizeof(T);  // elements per 32-byte sector
  __shared__ long long s_K;
  pdl_wait();  // the union and counts are complete
  pdl_trigger();
  if (threadIdx.x == 0) {
    long long K;
    if (a.k_from_counts) {
      K = 0;
      for (int i = 0; i < a.n_local; ++i) K += clamp_count(a.counts[i], a.cap);
    } else {
      K = *a.K;
    }
    s_K = K;
  }
  __syncthreads();
  const long long K = s_K;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      if (a.k_from_counts) *a.K = K;
      a.hist_t[a.slot] = a.t;
      a.hist_K[a.slot] = K;
    }
    if (threadIdx.x < a.n_local) {
      const int i = threadIdx.x;
      const unsigned long long k = (unsigned long long)a.counts[i];
      double d = a.delta[i];
      a.hist_counts[a.slot * a.n_local + i] = (long long)k;
      a.hist_delta[a.slot * a.n_local + i] = d;
      double err = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not recorded
      if (a.norm_mode == 1) {
        const double sq = a.slots[i].sq - (a.corr ? fx_take(a.slots + i) : 0.0);
        err = sqrt(sq > 0.0 ? sq : 0.0);
      } else if (a.norm_mode == 2) {
        err = 0.0;
      }
      a.hist_err[a.slot * a.n_local + i] = err;
      // sparsifier.cpp:77-81
      if (a.update_delta) {
        if (k > a.k_target) d = d == 0.0 ? a.min_threshold : d * (1.0 + a.alpha);
        else if (k < a.k_target) d *= 1.0 - a.alpha;
        a.delta[i] = d;
      }
    }
  }
  if (!a.dense && !a.model) return;
  T* dense = (T*)a.dense;
  T* x = (T*)a.model;
  const T* sums = (const T*)a.union_sum;
  const int32_t* cur = a.union_idx;
  const T nf = (T)a.n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (x) {  // harness.cpp:212-215: x[j] -= s_j / n; four union entries per thread in flight
    for (long long m0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; m0 < K; m0 += 4 * stride) {
      int32_t j[4];
      T xv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (m0 + q * stride < K) {
          j[q] = cur[m0 + q * stride];
          xv[q] = ld_rand(x + j[q]);
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (m0 + q * stride < K) x[j[q]] = xv[q] - div_rn(sums[m0 + q * stride], nf);  // one rounding after /
    }
  }
  if (!dense) return;
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < K; m += stride) {
    const int64_t s = cur[m] / SEC;
    if (m > 0 && cur[m - 1] / SEC == s) continue;  // not the sector's owner
    T v[SEC];
#pragma unroll
    for (int c = 0; c < SEC; ++c) v[c] = (T)0;
    for (long long q = m; q < K && cur[q] / SEC == s; ++q) v[cur[q] % SEC] = div_rn(sums[q], nf);
    T* p = dense + s * SEC;
    if ((s + 1) * SEC <= a.n_g) {
      using V = typename Vec<T>::V;
      constexpr int VN = Vec<T>::N;
#pragma unroll
      for (int h = 0; h < SEC / VN; ++h) {
        V w;
#pragma unroll
        for (int c = 0; c < VN; ++c) set_comp(w, c, v[h * VN + c]);
        reinterpret_cast<V*>(p)[h] = w;
      }
    } else {
      for (int c = 0; c < SEC && s * SEC + c < a.n_g; ++c) p[c] = v[c];
    }
  }
}

// Clear the previous union's sectors of the dense g/n (whole 32-byte sectors,
// one owner per sector).  Launched before k_finalize, which then rewrites the
// sectors of the current union in full, so no membership test is needed.
template <typename T>
__global__ void __launch_bounds__(256) k_dense_clear(const int32_t* prev, const long long* prev_K,
                                                     T* dense, int64_t n_g) {
  constexpr int SEC = 32 / (int)sizeof(T);
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  const long long pK = *prev_K;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < pK; m += stride) {
    const int64_t s = prev[m] / SEC;
    if (m > 0 && prev[m - 1] / SEC == s) continue;
    T* p = dense + s * SEC;
    if ((s + 1) * SEC <= n_g) {
      V z;
#pragma unroll
      for (int c = 0; c < VN; ++c) set_comp(z, c, (T)0);
#pragma unroll
      for (int h = 0; h < SEC / VN; ++h) reinterpret_cast<V*>(p)[h] = z;
    } else {
      for (int c = 0; c < SEC && s * SEC + c < n_g; ++c) p[c] = (T)0;
    }
  }
}

}  // namespace micro
