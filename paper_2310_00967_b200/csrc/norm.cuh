// norm.cuh — deterministic fp64 sums of squares for the reference's
// per-iteration error norm: error_norm = (sum_i ||e_{i,t+1}||_2) / n
// (harness.cpp:230-235; error_metric, error_feedback.hpp:41-48).
//
// Every CTA of the producing grid reduces its threads' partial sums with a
// fixed butterfly (bit-identical in every lane) and publishes one double;
// the last CTA of each group of kSqGroup CTAs (atomic ticket) sums the
// group in index order, and the last group sums the groups.  The result
// depends only on the grid shape, never on CTA timing; tickets are reset by
// the CTAs that consume them, so the slots are ready for the next launch.
#pragma once

#include "common.cuh"

namespace micro {

constexpr int kSqGroup = 64;

struct SumSqSlots {
  double* part;       // one per CTA of the producing grid
  double* group;      // one per group of kSqGroup CTAs
  unsigned* ticket;   // groups + 1 (the last one is the top-level ticket); zero between launches
  double* out;        // the total
};

__host__ __device__ constexpr long long sumsq_groups(long long ctas) { return (ctas + kSqGroup - 1) / kSqGroup; }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-worker error-norm slot.  K1 leaves ||e_{t+1}||^2 (own selections
// zeroed) in `sq`; the exchange then zeroes the foreign union entries of the
// residual and subtracts their squares, which arrive from many CTAs — over
// peer memory from several GPUs — in no fixed order.  fp64 atomics would make
// the record depend on CTA timing (acceptance C11: identical runs, identical
// records), so each CTA's (deterministic) partial is added exactly and
// order-independently as a 128-bit fixed-point integer.  The fixed point is
// scaled by the power of two just above `sq` (every correction is a part of
// sq), so its resolution is relative to the norm — 2^-128 of it — whatever
// the residuals' magnitude, and the sum cannot overflow.  A partial outside
// that range (non-finite, or larger than sq) sets a sticky flag and the record
// reads NaN.  Slots that other GPUs update use system-scope atomics.
struct NormSlot {
  unsigned long long lo, hi;  // sum of corrections * 2^(64 - E) as hi + lo * 2^-64, E = ilogb(sq) + 2
  double sq;                  // ||e||^2 after K1
  unsigned long long bad;     // sticky
};

__device__ __forceinline__ void fx_add(NormSlot* s, double v) {
  if (v == 0.0) return;
  const double sq = *reinterpret_cast<volatile double*>(&s->sq);
  const double x = (sq > 0.0 && sq < INFINITY) ? ldexp(v, 64 - (ilogb(sq) + 2)) : -1.0;
  if (!(x >= 0.0 && x < 1.8e19)) {  // also NaN / inf partials
    atomicOr_system(&s->bad, 1ull);
    return;
  }
  const double h = floor(x);
  const unsigned long long hi = (unsigned long long)h;
  const unsigned long long lo = __double2ull_rz((x - h) * 18446744073709551616.0);
  const unsigned long long old = atomicAdd_system(&s->lo, lo);
  atomicAdd_system(&s->hi, hi + (old + lo < old ? 1ull : 0ull));
}

// The corrections' sum; clears it for the next step (single reader, after
// every contributor is done).
__device__ __forceinline__ double fx_take(NormSlot* s) {
  const unsigned long long lo = s->lo, hi = s->hi, bad = s->bad;
  s->lo = 0ull;
  s->hi = 0ull;
  s->bad = 0ull;
  if (bad) return __longlong_as_double(0x7ff8000000000000ll);
  if (!(s->sq > 0.0)) return 0.0;
  return ldexp((double)hi + (double)lo * 0x1p-64, (ilogb(s->sq) + 2) - 64);
}

// Called by every thread of the CTA (contains a __syncthreads) at the end of
// the kernel: after it returns, only warp 0 of the finishing CTAs has done
// anything further.
__device__ __forceinline__ void cta_sumsq_publish(double v, const SumSqSlots& s) {
  __shared__ double s_red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  v = warp_sum_f64(v);
  if (lane == 0) s_red[w] = v;
  __syncthreads();
  if (w != 0) return;
  double t = lane < nw ? s_red[lane] : 0.0;
  t = warp_sum_f64(t);
  const unsigned nblk = gridDim.x, b = blockIdx.x, g = b / kSqGroup;
  const unsigned gsize = min((unsigned)kSqGroup, nblk - g * kSqGroup);
  const unsigned ngroups = (nblk + kSqGroup - 1) / kSqGroup;
  unsigned prev = 0;
  if (lane == 0) {
    s.part[b] = t;
    __threadfence();
    prev = atomicAdd(s.ticket + g, 1u);
  }
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != gsize - 1) return;
  __threadfence();
  double gs = 0.0;
  for (unsigned q = lane; q < gsize; q += 32) gs += __ldcg(s.part + g * kSqGroup + q);
  gs = warp_sum_f64(gs);
  if (lane == 0) {
    s.group[g] = gs;
    s.ticket[g] = 0;
    __threadfence();
    prev = atomicAdd(s.ticket + ngroups, 1u);
  }
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != ngroups - 1) return;
  __threadfence();
  double tot = 0.0;
  for (unsigned q = lane; q < ngroups; q += 32) tot += __ldcg(s.group + q);
  tot = warp_sum_f64(tot);
  if (lane == 0) {
    *s.out = tot;
    s.ticket[ngroups] = 0;
  }
}

// Standalone sum of squares of one vector (the value-level error_metric):
// fixed grid, each thread sums its grid-stride elements in order —
// deterministic for a given n and grid.  fp32 reads 16-byte vectors (four in
// flight) then the scalar tail (scalar 4-byte loads reached 3.5 TB/s); fp64
// and unaligned vectors take the scalar loop (the vector form of the fp64
// sum measured 1.4x slower: its dependent adds sit behind each vector).
template <typename T>
__global__ void __launch_bounds__(256) k_sumsq(const T* __restrict__ x, int64_t n, SumSqSlots s) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N, U = 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  double v = 0.0;
  int64_t done = 0;
  if (sizeof(T) == 4 && ((uintptr_t)x & 15) == 0) {
    const int64_t nv = n / VN;
    const V* xv = reinterpret_cast<const V*>(x);
    for (int64_t q0 = tid; q0 < nv; q0 += U * stride) {
      V a[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < nv) a[u] = ld_nc_stream(xv + q0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < nv) {
#pragma unroll
          for (int c = 0; c < VN; ++c) {
            const double y = (double)comp(a[u], c);
            v += y * y;
          }
        }
    }
    done = nv * VN;
  }
  for (int64_t j = done + tid; j < n; j += stride) {
    const double y = (double)x[j];
    v += y * y;
  }
  cta_sumsq_publish(v, s);
}

}  // namespace micro
