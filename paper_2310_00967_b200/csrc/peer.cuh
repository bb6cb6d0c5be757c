// peer.cuh — the n-GPU exchange as ONE kernel over peer memory (NVLink /
// NVSwitch), replacing the NCCL protocol's K2..K7 (dist.py) and its host
// count round trip.
//
// Reference semantics: the union restricted to partition p is the selection
// of p's owner (exclusive partitions, acceptance.cpp:93-118), and every sum
// is s_j = 0; for r = 0..n-1: s_j += acc_r[j] (collectives.cpp:39-47).  So
// each rank, as owner of its own partition, after every rank's K1 is done
// (caller's barrier #1):
//   * reads every rank's k_r (peer loads) -> its segment offset in partition
//     order and K;
//   * for each of its selected j: reads acc_r[j] from every peer's residual in
//     rank order (its own value from the K1 pairs), sums from +0, and zeroes
//     the peers' entries (harness.cpp:219-221 — no races: j has one owner);
//   * pushes (j, s_j) into every rank's union buffer at its segment
//     (peer stores).
// After barrier #2 each rank finalizes locally (threshold, history, dense
// g/n, model) from its own union buffer.  No kernel ever waits on another
// rank's kernel: the two barriers are the caller's (a 4-byte NCCL
// all-reduce on the compute stream, or a host barrier in tests).
#pragma once

#include "common.cuh"
#include "norm.cuh"

namespace micro {

struct PeerPtrs {
  const long long* counts[kMaxWorkers];  // rank r's k_r (its counts[0])
  void* resid[kMaxWorkers];
  int32_t* uidx[kMaxWorkers];            // union buffers of this step's parity
  void* usum[kMaxWorkers];
  NormSlot* corr[kMaxWorkers];           // error-norm slots (NULL: not recorded)
};

__device__ __forceinline__ long long ld_volatile_i64(const long long* p) {
  return *reinterpret_cast<const volatile long long*>(p);
}

template <typename T, bool kZero>
__global__ void __launch_bounds__(256) k_peer_exchange(PeerPtrs p, int n, int me, int64_t t, long long cap,
                                                       const int32_t* __restrict__ own_idx,
                                                       const T* __restrict__ own_val, long long* K_out) {
  __shared__ long long s_off, s_k;
  __shared__ double s_corr[8][kMaxWorkers];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    const int pme = (int)((t % n + me) % n);  // my partition (tensor.hpp:57)
    long long off = 0, K = 0;
    for (int q = 0; q < n; ++q) {
      const long long kq = ld_volatile_i64(p.counts[partition_owner(q, n, t)]);
      const long long kc = kq < cap ? kq : cap;
      if (q < pme) off += kc;
      K += kc;
    }
    const long long km = ld_volatile_i64(p.counts[me]);
    s_off = off;
    s_k = km < cap ? km : cap;
    if (blockIdx.x == 0) *K_out = K;
  }
  __syncthreads();
  const long long off = s_off, k = s_k;
  const bool corr = kZero && p.corr[0] != nullptr;  // grid-uniform
  double c_lo = 0.0, c_hi = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long b = (long long)blockIdx.x * blockDim.x; b < k; b += stride) {  // warp-uniform trip count
    const long long m = b + threadIdx.x;
    const bool act = m < k;
    const int32_t j = act ? own_idx[m] : 0;
    T s = (T)0;
    // eight peers' entries in flight per thread, summed strictly in rank order
    for (int r0 = 0; r0 < n; r0 += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u;
        v[u] = (T)0;
        if (act && r < n) v[u] = r == me ? own_val[m] : ((const T*)p.resid[r])[j];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u;
        if (r >= n) break;
        s = add_rn(s, v[u]);
        if (kZero && act && r != me) ((T*)p.resid[r])[j] = (T)0;
        if (corr && r != me) {
          const double q = warp_sum_f64(act ? (double)v[u] * (double)v[u] : 0.0);
          if (lane == (r & 31)) {
            if (r < 32) c_lo += q;
            else c_hi += q;
          }
        }
      }
    }
    if (act)
      for (int q = 0; q < n; ++q) {
        p.uidx[q][off + m] = j;
        ((T*)p.usum[q])[off + m] = s;
      }
  }
  if (corr) {
    if (lane < n) s_corr[wid][lane] = c_lo;
    if (lane + 32 < n) s_corr[wid][lane + 32] = c_hi;
    __syncthreads();
    if ((int)threadIdx.x < n && (int)threadIdx.x != me) {
      double tot = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += s_corr[q][threadIdx.x];
      if (tot != 0.0) fx_add(p.corr[threadIdx.x], tot);
    }
  }
  __threadfence_system();  // peer stores visible before the caller's barrier
}

}  // namespace micro

namespace micro {

// ---- bulk variant: every NVLink transfer contiguous --------------------------
// Random 4-byte remote reads and stores (above) cost a whole NVLink request
// each; here the only random accesses are local HBM ones:
//   phase A (after barrier #1), every rank r for every other owner o: read
//     o's selected index list (remote, contiguous), gather its own acc_r at
//     those indices and zero them (local), write the values contiguously
//     into o's receive slab r (remote, contiguous);
//   phase B (after barrier #2), every owner: s = 0; s += contribution_r in
//     rank order (local, contiguous), push (j, s_j) into every rank's union
//     buffer (remote, contiguous);
//   finalize after barrier #3.
struct PeerBulkPtrs {
  const long long* counts[kMaxWorkers];
  const int32_t* sel_idx[kMaxWorkers];   // each owner's own selection (this step's parity)
  void* recv[kMaxWorkers];               // each owner's receive slabs: [source rank][cap]
  int32_t* uidx[kMaxWorkers];
  void* usum[kMaxWorkers];
};

template <typename T, bool kZero>
__global__ void __launch_bounds__(256) k_peer_contribute(PeerBulkPtrs p, int me, long long cap, T* __restrict__ resid,
                                                         NormSlot* corr) {
  const int o = blockIdx.y;
  if (o == me) return;  // block-uniform
  __shared__ double s_q[8];
  long long k = ld_volatile_i64(p.counts[o]);
  k = k < cap ? k : cap;
  const int32_t* __restrict__ idx = p.sel_idx[o];
  T* __restrict__ out = (T*)p.recv[o] + (long long)me * cap;
  double q = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long m0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; m0 < k; m0 += 4 * stride) {
    int32_t j[4];
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)  // four index reads (remote, coalesced) in flight
      if (m0 + u * stride < k) j[u] = idx[m0 + u * stride];
#pragma unroll
    for (int u = 0; u < 4; ++u)  // four local gathers in flight
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
  if (kZero && corr) {  // squares of the entries zeroed here (error norm)
    q = warp_sum_f64(q);
    if ((threadIdx.x & 31) == 0) s_q[threadIdx.x >> 5] = q;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_q[w];
      if (tot != 0.0) fx_add(corr, tot);
    }
  }
  __threadfence_system();
}

template <typename T>
__global__ void __launch_bounds__(256) k_peer_reduce_push(PeerBulkPtrs p, int n, int me, int64_t t, long long cap,
                                                          const int32_t* __restrict__ own_idx,
                                                          const T* __restrict__ own_val, long long* K_out) {
  __shared__ long long s_off, s_k;
  if (threadIdx.x == 0) {
    const int pme = (int)((t % n + me) % n);
    long long off = 0, K = 0;
    for (int q = 0; q < n; ++q) {
      const long long kq = ld_volatile_i64(p.counts[partition_owner(q, n, t)]);
      const long long kc = kq < cap ? kq : cap;
      if (q < pme) off += kc;
      K += kc;
    }
    const long long km = ld_volatile_i64(p.counts[me]);
    s_off = off;
    s_k = km < cap ? km : cap;
    if (blockIdx.x == 0) *K_out = K;
  }
  __syncthreads();
  const long long off = s_off, k = s_k;
  const T* __restrict__ recv = (const T*)p.recv[me];
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < k; m += (long long)gridDim.x * blockDim.x) {
    T s = (T)0;
    for (int r = 0; r < n; ++r) s = add_rn(s, r == me ? own_val[m] : recv[(long long)r * cap + m]);
    const int32_t j = own_idx[m];
    for (int q = 0; q < n; ++q) {
      p.uidx[q][off + m] = j;
      ((T*)p.usum[q])[off + m] = s;
    }
  }
  __threadfence_system();
}

}  // namespace micro
