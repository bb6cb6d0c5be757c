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

// The CTA's peer stores, released at system scope once: the barrier orders
// every thread's stores before thread 0's fence (cumulative).  The kernel
// boundary and the caller's barrier order them as well; the single fence
// keeps the protocol safe for a caller whose barrier is only a flag, at the
// cost of one membar.sys per CTA instead of one per thread (ncu: the
// per-thread fence was 70 % of the exchange kernels' stalls).
// Every rank's count (peer loads, one per lane, all in flight) -> this
// rank's segment offset in partition order, its own (clamped) count and K.
// Warp 0 only; results in *off, *km, *K (lane 0).
__device__ __forceinline__ void peer_offsets(const long long* const* counts, int n, int me, int64_t t, long long cap,
                                             long long* off, long long* km, long long* K) {
  const int lane = threadIdx.x & 31;
  const int pme = (int)((t % n + me) % n);  // my partition (tensor.hpp:57)
  long long o = 0, tot = 0;
  for (int q0 = 0; q0 < n; q0 += 32) {
    const int q = q0 + lane;  // partition q, owned by partition_owner(q)
    long long kc = 0;
    if (q < n) {
      const long long kq = ld_volatile_i64(counts[partition_owner(q, n, t)]);
      kc = kq < cap ? kq : cap;
    }
    o += (long long)warp_sum_u64((unsigned long long)(q < pme ? kc : 0));
    tot += (long long)warp_sum_u64((unsigned long long)kc);
  }
  if (lane == 0) {
    const long long k = ld_volatile_i64(counts[me]);
    *off = o;
    *km = k < cap ? k : cap;
    *K = tot;
  }
}

__device__ __forceinline__ void cta_release_system() {
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
}

template <typename T, bool kZero>
__global__ void __launch_bounds__(256) k_peer_exchange(PeerPtrs p, int n, int me, int64_t t, long long cap,
                                                       const int32_t* __restrict__ own_idx,
                                                       const T* __restrict__ own_val, long long* K_out) {
  __shared__ long long s_off, s_k, s_K;
  __shared__ double s_corr[8][kMaxWorkers];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid == 0) peer_offsets(p.counts, n, me, t, cap, &s_off, &s_k, &s_K);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *K_out = s_K;
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
  cta_release_system();  // peer stores visible before the caller's barrier
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

constexpr int kPeerILP = 8;  // entries per lane in flight in the bulk exchange kernels

// Grid: x = CTAs per owner (each warp takes 32 * kPeerILP consecutive
// entries of the owner's list per round), y = owner.
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
  const int lane = threadIdx.x & 31;
  constexpr long long kChunk = 32 * kPeerILP;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  double q = 0.0;
  for (long long base = warp * kChunk; base < k; base += nwarps * kChunk) {
    int32_t j[kPeerILP];
    T v[kPeerILP];
#pragma unroll
    for (int u = 0; u < kPeerILP; ++u)  // the owner's index list: remote, coalesced
      if (base + u * 32 + lane < k) j[u] = idx[base + u * 32 + lane];
#pragma unroll
    for (int u = 0; u < kPeerILP; ++u)  // own accumulator: local random reads, all in flight
      if (base + u * 32 + lane < k) v[u] = ld_rand(resid + j[u]);
#pragma unroll
    for (int u = 0; u < kPeerILP; ++u)
      if (base + u * 32 + lane < k) {
        out[base + u * 32 + lane] = v[u];  // the owner's receive slab: remote, coalesced
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
  cta_release_system();
}

// Owner: s = 0; s += contribution_r in rank order (all n values in flight,
// eight at a time), then the (index, sum) pair pushed to every rank.
template <typename T>
__global__ void __launch_bounds__(256) k_peer_reduce_push(PeerBulkPtrs p, int n, int me, int64_t t, long long cap,
                                                          const int32_t* __restrict__ own_idx,
                                                          const T* __restrict__ own_val, long long* K_out) {
  __shared__ long long s_off, s_k, s_K;
  if (threadIdx.x < 32) peer_offsets(p.counts, n, me, t, cap, &s_off, &s_k, &s_K);
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *K_out = s_K;
  const long long off = s_off, k = s_k;
  const T* __restrict__ recv = (const T*)p.recv[me];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long m0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; m0 < k; m0 += 2 * stride) {
    // two entries per thread, each with n contributions (eight at a time) in flight
    T s[2] = {(T)0, (T)0};
    int32_t j[2] = {0, 0};
    for (int r0 = 0; r0 < n; r0 += 8) {
      T v[2][8];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long long m = m0 + e * stride;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = r0 + u;
          v[e][u] = (T)0;
          if (m < k && r < n) v[e][u] = r == me ? own_val[m] : recv[(long long)r * cap + m];
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (r0 + u < n) s[e] = add_rn(s[e], v[e][u]);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
      if (m0 + e * stride < k) j[e] = own_idx[m0 + e * stride];
    for (int q = 0; q < n; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const long long m = m0 + e * stride;
        if (m < k) {
          p.uidx[q][off + m] = j[e];
          ((T*)p.usum[q])[off + m] = s[e];
        }
      }
  }
  cta_release_system();
}

}  // namespace micro
