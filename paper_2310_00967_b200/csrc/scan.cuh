// scan.cuh — hand-written exclusive prefix sum over 32-bit words (three
// passes: tile totals, a one-CTA scan of the totals, the tile scans with
// their offsets).  Used where selections may overlap and the union is formed
// from a bitmap (the comparison sparsifiers' union and the value-level
// all_gather_indices, collectives.cpp:14-28): the input is the bitmap itself
// and each word contributes its popcount, so the offsets come out of the scan
// with no separate popcount pass.  Off the MiCRO hot path (its partitions are
// disjoint and the union is formed in partition order without a scan).
#pragma once

#include "common.cuh"

namespace micro {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048 words per CTA

__host__ __device__ constexpr int64_t scan_tiles(int64_t n) { return (n + kScanTile - 1) / kScanTile; }

template <bool kPopc>
__device__ __forceinline__ int scan_item(const unsigned* in, int64_t i, int64_t n) {
  if (i >= n) return 0;
  const unsigned v = in[i];
  return kPopc ? __popc(v) : (int)v;
}

// CTA-wide exclusive scan of the tile held in s (kScanTile ints, in place);
// returns the tile total.  Each thread owns kScanItems consecutive entries.
__device__ __forceinline__ int cta_scan_tile(int* s) {
  __shared__ int s_warp[kScanThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int v[kScanItems], sum = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    v[q] = s[tid * kScanItems + q];
    sum += v[q];
  }
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int q = 0; q < kScanThreads / 32; ++q) {
    before += q < w ? s_warp[q] : 0;
    total += s_warp[q];
  }
  int run = before + incl - sum;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    s[tid * kScanItems + q] = run;
    run += v[q];
  }
  __syncthreads();
  return total;
}

template <bool kPopc>
__global__ void __launch_bounds__(kScanThreads) k_scan_totals(const unsigned* __restrict__ in, int64_t n,
                                                              int* __restrict__ totals) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  int v = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) v += scan_item<kPopc>(in, base + q * kScanThreads + threadIdx.x, n);
  __shared__ int s_warp[kScanThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
#pragma unroll
    for (int q = 0; q < kScanThreads / 32; ++q) t += s_warp[q];
    totals[blockIdx.x] = t;
  }
}

// One CTA: exclusive scan of the tile totals in place; the grand total goes
// to *grand (may be NULL).
static __global__ void __launch_bounds__(kScanThreads) k_scan_top(int* __restrict__ totals, int64_t ntiles,
                                                           long long* grand) {
  __shared__ int s[kScanTile];
  long long carry = 0;
  for (int64_t b = 0; b < ntiles; b += kScanTile) {
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
      const int64_t i = b + q * kScanThreads + threadIdx.x;
      s[q * kScanThreads + threadIdx.x] = i < ntiles ? totals[i] : 0;
    }
    __syncthreads();
    const int t = cta_scan_tile(s);
#pragma unroll
    for (int q = 0; q < kScanItems; ++q) {
      const int64_t i = b + q * kScanThreads + threadIdx.x;
      if (i < ntiles) totals[i] = (int)(carry + s[q * kScanThreads + threadIdx.x]);
    }
    carry += t;
    __syncthreads();
  }
  if (grand && threadIdx.x == 0) *grand = carry;
}

template <bool kPopc>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(const unsigned* __restrict__ in, int64_t n,
                                                             const int* __restrict__ offs, int* __restrict__ out) {
  __shared__ int s[kScanTile];
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q)
    s[q * kScanThreads + threadIdx.x] = scan_item<kPopc>(in, base + q * kScanThreads + threadIdx.x, n);
  __syncthreads();
  cta_scan_tile(s);
  const int off = offs[blockIdx.x];
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    const int64_t i = base + q * kScanThreads + threadIdx.x;
    if (i < n) out[i] = off + s[q * kScanThreads + threadIdx.x];
  }
}

}  // namespace micro
