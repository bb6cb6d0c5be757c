// baselines.cuh — the comparison sparsifiers of run_iteration
// (harness.cpp:152-181) on the device:
//   top-k  select_topk (sparsifier.cpp:39-67): the k largest |acc| over the
//          whole vector, ties to the lower index, ascending
//   CLT-k  cltk_select (sparsifier.cpp:85-97): the leader t mod n only
//   hard   hard_threshold_select (sparsifier.cpp:99-101): |acc| > delta_0
//   dense  select_all (sparsifier.cpp:103-108)
// followed by the general union (sorted unique of overlapping selections,
// collectives.cpp:14-28) and the worker-order sums (collectives.cpp:30-49).
//
// Top-k is a radix select on the magnitude bits (fp32: 31 bits in 11/11/9-bit
// digits; fp64: 63 bits in six digits), one histogram pass per digit over
// acc = e + eta*G recomputed from (e, G) with K1's exact arithmetic, a
// one-block digit pick after each pass (no host round trip), then — only if
// the pivot magnitude P is shared by more elements than are still needed —
// the index J of the last tie to keep (lowest indices first).  The selection
// {|acc| > P} ∪ {|acc| == P, j <= J} is then exactly the reference's, and it
// is compacted in order by K1's streaming kernel with a tie predicate.
// The union of overlapping selections is a bitmap (atomicOr), compacted in
// index order.
#pragma once

#include "common.cuh"
#include "exchange.cuh"  // WorkerPtrs

namespace micro {

struct TopkState {
  unsigned long long prefix;  // key bits fixed so far
  unsigned long long mask;    // which bits of the key are fixed
  long long k_rem;            // elements still to take at/below the prefix
  long long eq;               // elements in the last chosen bucket (== P after the last pass)
  long long tie_j;            // last tie index kept (n_g: all ties)
  double pivot;               // P as a value (threshold of the compaction)
  int need_tie;
};

template <typename T> struct KeyOf;
template <> struct KeyOf<float> {
  using K = unsigned int;
  static constexpr int kBits = 31;
  __device__ static K key(float a) { return __float_as_uint(a) & 0x7fffffffu; }
  __device__ static double value(unsigned long long k) { return (double)__uint_as_float((unsigned)k); }
};
template <> struct KeyOf<double> {
  using K = unsigned long long;
  static constexpr int kBits = 63;
  __device__ static K key(double a) { return (K)__double_as_longlong(a) & 0x7fffffffffffffffull; }
  __device__ static double value(unsigned long long k) { return __longlong_as_double((long long)k); }
};

constexpr int kDigitBits = 11;
constexpr int kTieChunks = 65536;  // tie counting granularity (k_tie_count / k_tie_find)
constexpr int64_t kTieMinChunk = 4096;  // >= 16 elements per k_tie_count thread (tiny CTAs were launch bound)

// Elements per tie-counting chunk: at most kTieChunks chunks, at least
// kTieMinChunk elements each (k_tie_find walks one chunk: <= a few passes).
inline int64_t tie_chunk(int64_t n) {
  const int64_t c = (n + kTieChunks - 1) / kTieChunks;
  return c > kTieMinChunk ? c : kTieMinChunk;
}

// acc = e + eta*G (K1's arithmetic), or acc itself (g == NULL: the value API)
template <typename T>
__device__ __forceinline__ T acc_at(const T* e, const T* g, T eta, int64_t j) {
  return g ? add_rn(e[j], mul_rn(eta, g[j])) : e[j];
}
constexpr int kBins = 1 << kDigitBits;

static __global__ void k_topk_init(TopkState* st, long long k) {
  st->prefix = 0;
  st->mask = 0;
  st->k_rem = k;
  st->eq = 0;
  st->tie_j = 0;
  st->pivot = 0.0;
  st->need_tie = 0;
}

// Histogram of the current digit over the elements whose higher digits match
// the prefix, in kHistCopies interleaved shared-memory copies (the top digit
// holds the exponent: a handful of bins take everything, so same-address
// atomics are the cost to spread).
constexpr int kHistCopies = 4;  // lane l counts into copy l % 4: at most 8 lanes share an address

template <typename T>
__device__ __forceinline__ void hist_add(unsigned* s_hist, T acc, unsigned long long prefix, unsigned long long mask,
                                         int shift, unsigned dmask, bool valid) {
  using KO = KeyOf<T>;
  if (valid) {
    const unsigned long long key = KO::key(absx(acc));
    if ((key & mask) == prefix)
      atomicAdd(&s_hist[((unsigned)(key >> shift) & dmask) * kHistCopies + (threadIdx.x & (kHistCopies - 1))], 1u);
  }
}

// 16-byte loads of e and G (the same acc = e + eta*G as K1), every lane
// keeping two vectors of each in flight.  With acc_out (the first digit of
// the engine's top-k) acc is also written back in place and G probed for
// non-finite values, so the later passes and the compaction read acc alone
// (4 instead of 8 bytes per element).
// vectors per thread in flight (warp-uniform grid-stride loops)
#ifndef MICRO_HIST_VECS
#define MICRO_HIST_VECS 8
#endif
#ifndef MICRO_HIST_VECS_G
#define MICRO_HIST_VECS_G 2
#endif
constexpr int kHistVecs = MICRO_HIST_VECS, kHistVecsG = MICRO_HIST_VECS_G;

template <typename T>
__device__ __forceinline__ void topk_hist_body(const T* e, const T* __restrict__ g, double eta_d, int64_t n_g,
                                                   int shift, int width, const TopkState* st,
                                                   unsigned* __restrict__ hist, T* acc_out = nullptr,
                                                   int* flags = nullptr) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  __shared__ unsigned s_hist[kBins * kHistCopies];
  for (int b = threadIdx.x; b < kBins * kHistCopies; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  const unsigned dmask = (1u << width) - 1u;
  const T eta = (T)eta_d;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto flush = [&]() {
    __syncthreads();
    for (int b = threadIdx.x; b <= (int)dmask; b += blockDim.x) {
      unsigned c = 0;
#pragma unroll
      for (int q = 0; q < kHistCopies; ++q) c += s_hist[b * kHistCopies + q];
      if (c) atomicAdd(&hist[b], c);
    }
  };
  T probe = (T)0;  // NaN iff some G is Inf/NaN (acc_out passes only)
  if (((uintptr_t)e % 16) || ((uintptr_t)g % 16)) {  // a range of the value API: scalar loads
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < n_g; j0 += stride) {
      const int64_t j = j0 + threadIdx.x;
      const bool ok = j < n_g;
      const T acc = ok ? acc_at(e, g, eta, j) : (T)0;
      if (ok && acc_out) {
        probe = probe + g[j] * (T)0;
        acc_out[j] = acc;
      }
      hist_add<T>(s_hist, acc, prefix, mask, shift, dmask, ok);
    }
    if (flags && probe != probe) atomicOr(flags, 1);
    flush();
    return;
  }
  const int64_t nv = n_g / VN;  // whole vectors (e, G 16-byte aligned: K1 staging / cudaMalloc)
  if (!g) {  // acc alone: kHistVecs vectors per thread in flight
    for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x * kHistVecs; v0 < nv; v0 += kHistVecs * stride) {
      V ev[kHistVecs];
      bool ok[kHistVecs];
#pragma unroll
      for (int u = 0; u < kHistVecs; ++u) {
        const int64_t v = v0 + u * blockDim.x + threadIdx.x;
        ok[u] = v < nv;
        if (ok[u]) ev[u] = ld_stream(reinterpret_cast<const V*>(e) + v);
      }
#pragma unroll
      for (int u = 0; u < kHistVecs; ++u)
#pragma unroll
        for (int c = 0; c < VN; ++c) hist_add<T>(s_hist, ok[u] ? comp(ev[u], c) : (T)0, prefix, mask, shift, dmask, ok[u]);
    }
  } else
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x * kHistVecsG; v0 < nv; v0 += kHistVecsG * stride) {
    V ev[kHistVecsG], gv[kHistVecsG];
    bool ok[kHistVecsG];
#pragma unroll
    for (int u = 0; u < kHistVecsG; ++u) {
      const int64_t v = v0 + u * blockDim.x + threadIdx.x;
      ok[u] = v < nv;
      if (ok[u]) {
        ev[u] = reinterpret_cast<const V*>(e)[v];
        if (g) gv[u] = ld_nc_stream(reinterpret_cast<const V*>(g) + v);
      }
    }
#pragma unroll
    for (int u = 0; u < kHistVecsG; ++u) {
      V av;
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const T acc = !ok[u] ? (T)0 : g ? add_rn(comp(ev[u], c), mul_rn(eta, comp(gv[u], c))) : comp(ev[u], c);
        set_comp(av, c, acc);
        if (acc_out && ok[u]) probe = probe + comp(gv[u], c) * (T)0;
        hist_add<T>(s_hist, acc, prefix, mask, shift, dmask, ok[u]);
      }
      if (acc_out && ok[u]) st_stream(reinterpret_cast<V*>(acc_out) + v0 + u * blockDim.x + threadIdx.x, av);
    }
  }
  // the tail (n_g % VN elements)
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const int64_t j = nv * VN + threadIdx.x;
    const bool ok = j < n_g;
    const T acc = ok ? acc_at(e, g, eta, j) : (T)0;
    if (ok && acc_out) {
      probe = probe + g[j] * (T)0;
      acc_out[j] = acc;
    }
    hist_add<T>(s_hist, acc, prefix, mask, shift, dmask, ok);
  }
  if (flags && probe != probe) atomicOr(flags, 1);
  flush();
}

// One block of 1024: pick the bucket holding the k_rem-th largest key, fold
// it into the prefix, clear the histogram.  last: also form the pivot and
// whether ties must be cut.
template <typename T>
__device__ __forceinline__ void topk_digit_body(TopkState* st, unsigned* hist, int shift, int width,
                                                     int last, int64_t n_g) {
  __shared__ long long s_w[32];
  __shared__ int s_bin;
  __shared__ long long s_above;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nb = 1 << width;
  // thread tid owns bins hi-2*tid and hi-2*tid-1 (descending order)
  const int b0 = nb - 1 - 2 * tid, b1 = b0 - 1;
  const long long c0 = b0 >= 0 ? hist[b0] : 0, c1 = b1 >= 0 ? hist[b1] : 0;
  const long long mine = c0 + c1;
  long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[w] = incl;
  if (tid == 0) s_bin = -1;
  __syncthreads();
  if (w == 0) {
    long long x = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_w[lane] = x;
  }
  __syncthreads();
  const long long k = st->k_rem;
  const long long excl = (w ? s_w[w - 1] : 0) + incl - mine;  // keys in bins above b0
  if (b0 >= 0 && excl < k && excl + c0 >= k) {
    s_bin = b0;
    s_above = excl;
  } else if (b1 >= 0 && excl + c0 < k && excl + c0 + c1 >= k) {
    s_bin = b1;
    s_above = excl + c0;
  }
  __syncthreads();
  if (tid == 0) {
    const int b = s_bin;  // always found: k_rem <= elements matching the prefix
    st->k_rem = k - s_above;
    st->eq = hist[b];
    st->prefix |= (unsigned long long)b << shift;
    st->mask |= (unsigned long long)((1u << width) - 1u) << shift;
    if (last) {
      st->pivot = KeyOf<T>::value(st->prefix);
      st->need_tie = st->k_rem < st->eq;
      st->tie_j = n_g;  // all ties (refined by k_tie_find when need_tie)
    }
  }
  __syncthreads();
  for (int b = tid; b < nb; b += blockDim.x) hist[b] = 0;
}

// Ties at the pivot per contiguous chunk (only when some must be cut).
template <typename T>
__device__ __forceinline__ void tie_count_body(const T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                   int64_t n_g, int64_t chunk, const TopkState* st,
                                                   unsigned* __restrict__ counts) {
  if (!st->need_tie) return;
  __shared__ unsigned s_c;
  if (threadIdx.x == 0) s_c = 0;
  __syncthreads();
  const T eta = (T)eta_d;
  const T P = (T)st->pivot;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(lo + chunk, n_g);
  unsigned c = 0;
#pragma unroll 4
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) c += absx(acc_at(e, g, eta, j)) == P;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s_c, c);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s_c;
}

// One block of 1024: the chunk holding the k_rem-th tie, then that tie's
// index (ties taken in index order).
// base: added to the index written (the value API selects inside a range).
template <typename T>
__device__ __forceinline__ void tie_find_body(const T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                   int64_t n_g, int64_t chunk, int nchunks, TopkState* st,
                                                   const unsigned* __restrict__ counts, int64_t base = 0) {
  if (!st->need_tie) return;
  __shared__ long long s_w[32];
  __shared__ long long s_rem;
  __shared__ int s_chunk;
  __shared__ long long s_j;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long k = st->k_rem;
  // thread tid owns chunks [tid*per, (tid+1)*per)
  const int per = (nchunks + 1023) / 1024;
  long long mine = 0;
  for (int q = tid * per; q < min(nchunks, (tid + 1) * per); ++q) mine += counts[q];
  long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    long long x = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_w[lane] = x;
  }
  __syncthreads();
  long long run = (w ? s_w[w - 1] : 0) + incl - mine;
  if (run < k && run + mine >= k) {
    for (int q = tid * per; q < min(nchunks, (tid + 1) * per); ++q) {
      if (run + counts[q] >= k) {
        s_chunk = q;
        s_rem = k - run;
        break;
      }
      run += counts[q];
    }
  }
  __syncthreads();
  // walk the chunk in index order, 1024 elements at a time
  const T eta = (T)eta_d;
  const T P = (T)st->pivot;
  const int64_t lo = (int64_t)s_chunk * chunk, hi = min(lo + chunk, n_g);
  long long rem = s_rem;
  if (tid == 0) s_j = -1;
  __syncthreads();
  for (int64_t b = lo; b < hi; b += 1024) {
    const int64_t j = b + tid;
    const bool tie = j < hi && absx(acc_at(e, g, eta, j)) == P;
    const unsigned bal = __ballot_sync(0xffffffffu, tie);
    if (lane == 0) s_w[w] = __popc(bal);
    __syncthreads();
    long long before = 0, total = 0;
    for (int q = 0; q < 32; ++q) {
      if (q < w) before += s_w[q];
      total += s_w[q];
    }
    before += __popc(bal & ((1u << lane) - 1u));
    if (tie && before + 1 == rem) s_j = j;
    __syncthreads();
    if (s_j >= 0 || total >= rem) break;
    rem -= total;
    __syncthreads();
  }
  if (tid == 0) st->tie_j = base + s_j;
}

// The single-range kernels (one worker, or a range of the value API).
template <typename T>
__global__ void __launch_bounds__(256, 4) k_topk_hist(const T* e, const T* __restrict__ g, double eta_d, int64_t n_g,
                                                   int shift, int width, const TopkState* st,
                                                   unsigned* __restrict__ hist, T* acc_out = nullptr,
                                                   int* flags = nullptr) {
  topk_hist_body<T>(e, g, eta_d, n_g, shift, width, st, hist, acc_out, flags);
}
template <typename T>
__global__ void __launch_bounds__(1024) k_topk_digit(TopkState* st, unsigned* hist, int shift, int width, int last,
                                                     int64_t n_g) {
  topk_digit_body<T>(st, hist, shift, width, last, n_g);
}
template <typename T>
__global__ void __launch_bounds__(256) k_tie_count(const T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                   int64_t n_g, int64_t chunk, const TopkState* st,
                                                   unsigned* __restrict__ counts) {
  tie_count_body<T>(e, g, eta_d, n_g, chunk, st, counts);
}
template <typename T>
__global__ void __launch_bounds__(1024) k_tie_find(const T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                   int64_t n_g, int64_t chunk, int nchunks, TopkState* st,
                                                   const unsigned* __restrict__ counts, int64_t base = 0) {
  tie_find_body<T>(e, g, eta_d, n_g, chunk, nchunks, st, counts, base);
}

// The same selection for every worker of a single-device cluster at once
// (blockIdx.y = worker): eight workers' radix passes, digit picks and tie
// searches share each launch instead of running one after another.  Worker
// y owns st[y], hist[y * kBins ..] and counts[y * kTieChunks ..]; its acc is
// formed in place in e[y] by the first pass, as in the per-worker path.
struct TopkBatch {
  void* e[kMaxWorkers];        // residual -> acc (in place)
  const void* g[kMaxWorkers];  // gradients (first pass only)
};

static __global__ void k_topk_init_b(TopkState* st, int n, long long k) {
  if ((int)threadIdx.x < n) {
    TopkState* s = st + threadIdx.x;
    s->prefix = 0;
    s->mask = 0;
    s->k_rem = k;
    s->eq = 0;
    s->tie_j = 0;
    s->pivot = 0.0;
    s->need_tie = 0;
  }
}
template <typename T>
__global__ void __launch_bounds__(256, 4) k_topk_hist_b(TopkBatch b, double eta_d, int64_t n_g, int shift, int width,
                                                     const TopkState* st, unsigned* __restrict__ hist, int first,
                                                     int* flags) {
  const int y = blockIdx.y;
  T* acc = (T*)b.e[y];
  topk_hist_body<T>(acc, first ? (const T*)b.g[y] : nullptr, eta_d, n_g, shift, width, st + y, hist + y * kBins,
                    first ? acc : nullptr, first ? flags : nullptr);
}
template <typename T>
__global__ void __launch_bounds__(1024) k_topk_digit_b(TopkState* st, unsigned* hist, int shift, int width, int last,
                                                       int64_t n_g) {
  topk_digit_body<T>(st + blockIdx.x, hist + blockIdx.x * kBins, shift, width, last, n_g);
}
template <typename T>
__global__ void __launch_bounds__(256) k_tie_count_b(TopkBatch b, int64_t n_g, int64_t chunk, const TopkState* st,
                                                     unsigned* __restrict__ counts) {
  const int y = blockIdx.y;
  tie_count_body<T>((const T*)b.e[y], nullptr, 1.0, n_g, chunk, st + y, counts + (int64_t)y * kTieChunks);
}
template <typename T>
__global__ void __launch_bounds__(1024) k_tie_find_b(TopkBatch b, int64_t n_g, int64_t chunk, int nchunks,
                                                     TopkState* st, const unsigned* __restrict__ counts) {
  const int y = blockIdx.x;
  tie_find_body<T>((const T*)b.e[y], nullptr, 1.0, n_g, chunk, nchunks, st + y, counts + (int64_t)y * kTieChunks);
}

// acc = e + eta*G in place with the non-finite probe (workers that select
// nothing this step: CLT-k non-leaders, dense).
template <typename T>
__device__ __forceinline__ void accumulate_probe_body(T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                      int64_t n_g, int* flags) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  constexpr int U = 4;  // vectors per thread in flight
  const T eta = (T)eta_d;
  T probe = (T)0;
  const int64_t nv = n_g / VN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += U * stride) {
    V ev[U], gv[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * stride < nv) {
        ev[u] = ld_stream(reinterpret_cast<const V*>(e) + v0 + u * stride);
        gv[u] = ld_nc_stream(reinterpret_cast<const V*>(g) + v0 + u * stride);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (v0 + u * stride < nv) {
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          probe = probe + comp(gv[u], c) * (T)0;
          set_comp(ev[u], c, add_rn(comp(ev[u], c), mul_rn(eta, comp(gv[u], c))));
        }
        st_stream(reinterpret_cast<V*>(e) + v0 + u * stride, ev[u]);
      }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t j = nv * VN; j < n_g; ++j) {
      probe = probe + g[j] * (T)0;
      e[j] = add_rn(e[j], mul_rn(eta, g[j]));
    }
  if (probe != probe) atomicOr(flags, 1);
}
template <typename T>
__global__ void __launch_bounds__(256) k_accumulate_probe(T* __restrict__ e, const T* __restrict__ g, double eta_d,
                                                          int64_t n_g, int* flags) {
  accumulate_probe_body<T>(e, g, eta_d, n_g, flags);
}
// Every worker of the cluster but `skip` (the CLT-k leader; -1: none) at
// once (blockIdx.y = worker), and their selection counts set to `count`.
template <typename T>
__global__ void __launch_bounds__(256) k_accumulate_probe_b(TopkBatch b, double eta_d, int64_t n_g, int* flags,
                                                            int skip, long long* counts, long long count) {
  const int y = blockIdx.y;
  if (y == skip) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[y] = count;
  accumulate_probe_body<T>((T*)b.e[y], (const T*)b.g[y], eta_d, n_g, flags);
}

// ---- union of overlapping selections: bitmap, then ordered emission ----
// blockIdx.y = worker: every worker's selection in one launch.
static __global__ void __launch_bounds__(256) k_union_mark(WorkerPtrs wp, const long long* counts, long long cap,
                                                    unsigned* __restrict__ bitmap) {
  const int32_t* __restrict__ idx = wp.sel_idx[blockIdx.y];
  const long long k = min(counts[blockIdx.y], cap);
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < k; m += (long long)gridDim.x * blockDim.x) {
    const int32_t j = idx[m];
    atomicOr(&bitmap[j >> 5], 1u << (j & 31));
  }
}

// off: exclusive prefix of the popcounts.  Writes the union in index order,
// K, and clears the bitmap for the next step.
static __global__ void __launch_bounds__(256) k_bitmap_emit(unsigned* __restrict__ bitmap, int64_t nwords,
                                                     const int* __restrict__ off, int32_t* __restrict__ uidx,
                                                     long long* K, long long dense_above = -1) {
  if (dense_above >= 0 && *K > dense_above) return;  // k_union_words emitted the union
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    unsigned bits = bitmap[w];
    int o = off[w];
    if (w == nwords - 1) *K = (long long)o + __popc(bits);
    if (!bits) continue;
    bitmap[w] = 0;
    while (bits) {
      const int b = __ffs(bits) - 1;
      uidx[o++] = (int32_t)(w * 32 + b);
      bits &= bits - 1;
    }
  }
}

// The union emission and the worker-order sums in one pass over the bitmap
// (for dense unions, instead of k_bitmap_emit + k_union_reduce): a warp takes four consecutive
// words, lane l element 32 w + l, so each worker's residual is read with
// coalesced loads (only the union's lanes load) — the unions of overlapping
// selections are dense enough (top-k build-up 7.5 %, hard threshold 35 % at
// n = 8) that a random gather per entry re-fetched the same lines.  Sums run
// s = 0; s += acc_r for r in worker order (collectives.cpp:44-45); the union
// lands at off[w] + rank in index order; the bitmap is cleared for the next
// step (K: the scan's total).
// 4 words per warp and iteration at <= 128 registers (2 CTAs per SM) measured
// best (profiles/README.md: 2 words at <= 64 registers, 4 at 143 slower)
constexpr int kUnionWords = 4;
template <typename T, bool kZero>
__global__ void __launch_bounds__(256, 2) k_union_words(WorkerPtrs wp, int n, unsigned* __restrict__ bitmap,
                                                     int64_t nwords, const int* __restrict__ off,
                                                     int32_t* __restrict__ uidx, T* __restrict__ usum, long long* K,
                                                     long long dense_above) {
  if (*K <= dense_above) return;  // sparse union: k_bitmap_emit + k_union_reduce
  constexpr int kW = kUnionWords;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned below = (1u << lane) - 1u;
  for (int64_t w0 = gw * kW; w0 < nwords; w0 += nw * kW) {
    unsigned bits[kW];
    int o[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      const bool in = w0 + q < nwords;
      bits[q] = in ? bitmap[w0 + q] : 0u;
      o[q] = in ? off[w0 + q] : 0;
    }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        if (bits[q]) bitmap[w0 + q] = 0u;
      }
    }
    unsigned any = 0;
#pragma unroll
    for (int q = 0; q < kW; ++q) any |= bits[q];
    if (!any) continue;
    T s[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) s[q] = (T)0;
    for (int r0 = 0; r0 < n; r0 += 8) {
      T v[kW][8];
#pragma unroll
      for (int q = 0; q < kW; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (r0 + u < n && ((bits[q] >> lane) & 1u)) v[q][u] = ((const T*)wp.resid[r0 + u])[(w0 + q) * 32 + lane];
#pragma unroll
      for (int q = 0; q < kW; ++q)
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (r0 + u < n && ((bits[q] >> lane) & 1u)) {
            s[q] = add_rn(s[q], v[q][u]);
            if (kZero) ((T*)wp.resid[r0 + u])[(w0 + q) * 32 + lane] = (T)0;
          }
    }
#pragma unroll
    for (int q = 0; q < kW; ++q)
      if ((bits[q] >> lane) & 1u) {
        const int pos = o[q] + __popc(bits[q] & below);
        uidx[pos] = (int32_t)((w0 + q) * 32 + lane);
        usum[pos] = s[q];
      }
  }
}

static __global__ void k_iota(int32_t* u, int64_t n, long long* K) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    u[j] = (int32_t)j;
  if (blockIdx.x == 0 && threadIdx.x == 0) *K = n;
}

static __global__ void k_fill_i64(long long* p, int n, long long v) {
  if ((int)threadIdx.x < n) p[threadIdx.x] = v;
}

// s_j = 0; for r in worker order: s_j += acc_r[j] (collectives.cpp:44-45), and
// the union zeroed on every worker (harness.cpp:219-221).
template <typename T, bool kZero>
__global__ void __launch_bounds__(256) k_union_reduce(WorkerPtrs w, int n, const int32_t* __restrict__ uidx,
                                                      const long long* K, T* __restrict__ usum,
                                                      long long dense_above = -1) {
  const long long k = *K;
  if (dense_above >= 0 && k > dense_above) return;  // k_union_words summed the union
  const long long stride = (long long)gridDim.x * blockDim.x;
  // eight workers' entries in flight per thread (random reads, 64-byte L2
  // fetches; as k_cluster_reduce), then summed strictly in worker order —
  // one worker per round left every round a full DRAM latency
  for (long long m = (long long)blockIdx.x * blockDim.x + threadIdx.x; m < k; m += stride) {
    const int32_t j = uidx[m];
    T s = (T)0;
    for (int r0 = 0; r0 < n; r0 += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (r0 + u < n) v[u] = ld_rand((const T*)w.resid[r0 + u] + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (r0 + u >= n) break;
        s = add_rn(s, v[u]);
        if (kZero) ((T*)w.resid[r0 + u])[j] = (T)0;
      }
    }
    usum[m] = s;
  }
}

}  // namespace micro

namespace micro {

// Dense (select_all): the union is every index, so the whole step is one
// coalesced pass — s_j = sum_r acc_r[j] in worker order, g/n = s_j / n into
// the model and the dense output, the union written as (j, s_j), and every
// residual zeroed (harness.cpp:210-224).
template <typename T>
__global__ void __launch_bounds__(256) k_dense_all(WorkerPtrs w, int n, int64_t n_g, T* __restrict__ x,
                                                   T* __restrict__ dense, int32_t* __restrict__ uidx,
                                                   T* __restrict__ usum, long long* K) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  constexpr int U = 4;  // vectors per thread in flight (the pass is write-heavy: keep loads deep)
  const T nf = (T)n;
  const int64_t nv = n_g / VN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += U * stride) {
    V s[U], xv[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ok[u] = v0 + u * stride < nv;
#pragma unroll
      for (int c = 0; c < VN; ++c) set_comp(s[u], c, (T)0);
      if (x && ok[u]) xv[u] = ld_stream(reinterpret_cast<const V*>(x) + v0 + u * stride);
    }
    for (int r = 0; r < n; ++r) {  // worker order
      V a[U];
      V* e = reinterpret_cast<V*>(w.resid[r]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) a[u] = ld_stream(e + v0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ok[u]) {
          V z;
#pragma unroll
          for (int c = 0; c < VN; ++c) {
            set_comp(s[u], c, add_rn(comp(s[u], c), comp(a[u], c)));
            set_comp(z, c, (T)0);
          }
          st_stream(e + v0 + u * stride, z);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t v = v0 + u * stride;
      st_stream(reinterpret_cast<V*>(usum) + v, s[u]);
      V avg;
#pragma unroll
      for (int c = 0; c < VN; ++c) set_comp(avg, c, div_rn(comp(s[u], c), nf));
      if (x) {
#pragma unroll
        for (int c = 0; c < VN; ++c) set_comp(xv[u], c, comp(xv[u], c) - comp(avg, c));
        st_stream(reinterpret_cast<V*>(x) + v, xv[u]);
      }
      if (dense) st_stream(reinterpret_cast<V*>(dense) + v, avg);
      if (VN == 4)
        __stcs(reinterpret_cast<int4*>(uidx) + v, make_int4((int)(v * 4), (int)(v * 4 + 1), (int)(v * 4 + 2), (int)(v * 4 + 3)));
      else
        __stcs(reinterpret_cast<int2*>(uidx) + v, make_int2((int)(v * 2), (int)(v * 2 + 1)));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the n_g % VN tail, and K
    for (int64_t j = nv * VN; j < n_g; ++j) {
      T s = (T)0;
      for (int r = 0; r < n; ++r) {
        T* e = (T*)w.resid[r] + j;
        s = add_rn(s, *e);
        *e = (T)0;
      }
      usum[j] = s;
      const T avg = div_rn(s, nf);
      if (x) x[j] = x[j] - avg;
      if (dense) dense[j] = avg;
      uidx[j] = (int32_t)j;
    }
    *K = n_g;
  }
}

}  // namespace micro
