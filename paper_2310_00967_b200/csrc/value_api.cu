// value_api.cu — the stateless value-level calls of include/micro.h (the
// reference's sparsim:: free functions on device arrays), device memory
// plumbing for hosts without the CUDA runtime, and the synthetic inputs.
#include <mutex>

#include "internal.cuh"

using namespace micro;
using namespace micro::host;

namespace {

// Workspace of the value-level calls: a library-owned stream-ordered pool per
// device whose freed blocks stay reserved (release threshold = max).  On the
// default pool a call's multi-GB staging (worst case: every element selected)
// went back to the driver at each synchronisation and was mapped again by the
// next call — 50-130 ms per select at C3 size.  micro_value_workspace_trim()
// hands the reserve back.
constexpr int kMaxPoolDevices = 64;
cudaMemPool_t g_pools[kMaxPoolDevices] = {};
std::mutex g_pool_mu;

cudaError_t value_pool(int dev, cudaMemPool_t* out) {
  if (dev < 0 || dev >= kMaxPoolDevices) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    cudaError_t e = cudaMemPoolCreate(&p, &props);
    if (e != cudaSuccess) return e;
    unsigned long long keep = ~0ull;
    e = cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) {
      cudaMemPoolDestroy(p);
      return e;
    }
    g_pools[dev] = p;
  }
  *out = g_pools[dev];
  return cudaSuccess;
}

// cudaMallocAsync from the library's pool on the stream's device (the
// legacy default stream: the current device)
cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = s ? cudaStreamGetDevice(s, &dev) : cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool = nullptr;
  if ((e = value_pool(dev, &pool)) != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

template <typename T>
__global__ void k_synth(uint64_t seed, uint32_t worker, uint64_t t, int64_t n, T* out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q * 4 >= n) return;
  float z[4];
  ms_gaussian4(seed, worker, t, (uint64_t)q, z);
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (q * 4 + c < n) out[q * 4 + c] = (T)z[c];
}

// acc = e + eta*g elementwise (two roundings).  fp32: 16-byte vectors, four
// per operand in flight per thread, when all three arrays are 16-byte aligned
// (scalar 4-byte loads reached 4.8 TB/s); fp64 keeps the scalar loop, which
// already streams at the copy peak (the vector form measured 5 % slower).
template <typename T>
__global__ void k_accumulate(const T* e, T eta, const T* g, T* acc, int64_t n) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N, U = 4;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (sizeof(T) == 4 && (((uintptr_t)e | (uintptr_t)g | (uintptr_t)acc) & 15) == 0) {
    const int64_t nv = n / VN;
    const V* ev = reinterpret_cast<const V*>(e);
    const V* gv = reinterpret_cast<const V*>(g);
    V* av = reinterpret_cast<V*>(acc);
    for (int64_t q0 = tid; q0 < nv; q0 += U * stride) {
      V a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < nv) {
          a[u] = ld_nc_stream(ev + q0 + u * stride);
          b[u] = ld_nc_stream(gv + q0 + u * stride);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < nv) {
          V r;
#pragma unroll
          for (int c = 0; c < VN; ++c) set_comp(r, c, add_rn(comp(a[u], c), mul_rn(eta, comp(b[u], c))));
          st_stream(av + q0 + u * stride, r);
        }
    }
    done = nv * VN;
  }
  for (int64_t j = done + tid; j < n; j += stride) acc[j] = add_rn(e[j], mul_rn(eta, g[j]));
}

template <typename T>
__global__ void k_compensate(T* acc, int64_t n_g, const int32_t* idx, int64_t k, int* bad) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < k;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = idx[m];
    if (j < 0 || j >= n_g) atomicOr(bad, 1);
    else acc[j] = (T)0;
  }
}

template <typename T>
__global__ void k_reduce_values(WorkerPtrs w, int n, int64_t n_g, const int32_t* uidx, int64_t K,
                                T* sums, T* dense, int* bad) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < K;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = uidx[m];
    if (j < 0 || j >= n_g) { atomicOr(bad, 1); continue; }
    T s = (T)0;
    for (int r = 0; r < n; ++r) s = add_rn(s, ((const T*)w.sel_val[r])[j]);
    if (sums) sums[m] = s;
    if (dense) dense[j] = s;
  }
}

// min / max of a concatenated index list (the bitmap's extent)
__global__ void k_index_extent(const int32_t* idx, int64_t n, int* mm) {
  int lo = INT32_MAX, hi = -1;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    const int j = idx[m];
    lo = min(lo, j);
    hi = max(hi, j);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void k_mark_indices(const int32_t* idx, int64_t n, unsigned* bitmap) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n; m += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = idx[m];
    atomicOr(&bitmap[j >> 5], 1u << (j & 31));
  }
}

}  // namespace

extern "C" {

int micro_device_count(int* count) {
  if (!count) return fail(MICRO_EINVAL, "null count");
  CU(cudaGetDeviceCount(count));
  return MICRO_OK;
}

int micro_set_device(int device) {
  CU(cudaSetDevice(device));
  return MICRO_OK;
}

int micro_value_workspace_trim(int device) {
  if (device < 0 || device >= kMaxPoolDevices) return fail(MICRO_EINVAL, "device %d out of range", device);
  cudaMemPool_t p = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    p = g_pools[device];
  }
  if (p) CU(cudaMemPoolTrimTo(p, 0));
  return MICRO_OK;
}

int micro_device_malloc(void** d, int64_t bytes, int device) {
  if (!d || bytes < 0) return fail(MICRO_EINVAL, "bad allocation request");
  *d = nullptr;
  DeviceGuard dg(device);
  cudaError_t e = cudaMalloc(d, bytes ? (size_t)bytes : 16);
  if (e != cudaSuccess) return fail(MICRO_ENOMEM, "cudaMalloc(%lld): %s", (long long)bytes, cudaGetErrorString(e));
  return MICRO_OK;
}

int micro_host_malloc(void** h, int64_t bytes) {
  if (!h || bytes < 0) return fail(MICRO_EINVAL, "micro_host_malloc: bad arguments");
  *h = nullptr;
  CU(cudaMallocHost(h, bytes ? (size_t)bytes : 16));
  return MICRO_OK;
}

int micro_host_free(void* h) {
  if (h) CU(cudaFreeHost(h));
  return MICRO_OK;
}

int micro_device_free(void* d) {
  if (d) CU(cudaFree(d));
  return MICRO_OK;
}

int micro_memcpy(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
  if (bytes < 0 || kind < 0 || kind > 2) return fail(MICRO_EINVAL, "bad copy request");
  if (!bytes) return MICRO_OK;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost
                                                                          : cudaMemcpyDeviceToDevice;
  CU(cudaMemcpyAsync(dst, src, (size_t)bytes, k, (cudaStream_t)stream));
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  return MICRO_OK;
}

// ---- stateless value-level operations ----

int micro_synth_gaussian(int dtype, uint64_t seed, uint32_t worker, uint64_t t, int64_t n, void* d_out,
                         void* stream) {
  TRY(check_dtype(dtype));
  if (n < 0 || (n && !d_out)) return fail(MICRO_EINVAL, "bad output");
  if (!n) return MICRO_OK;
  const int64_t q = (n + 3) / 4;
  const unsigned grid = (unsigned)((q + 255) / 256);
  if (dtype == MICRO_F32) k_synth<float><<<grid, 256, 0, (cudaStream_t)stream>>>(seed, worker, t, n, (float*)d_out);
  else k_synth<double><<<grid, 256, 0, (cudaStream_t)stream>>>(seed, worker, t, n, (double*)d_out);
  CU(cudaGetLastError());
  return MICRO_OK;
}

int micro_accumulate(int dtype, const void* d_e, double eta, const void* d_g, void* d_acc, int64_t n,
                     void* stream) {
  TRY(check_dtype(dtype));
  if (!(eta > 0.0)) return fail(MICRO_EINVAL, "accumulate: eta must be positive");
  if (n < 0) return fail(MICRO_EINVAL, "accumulate: negative length");
  if (!n) return MICRO_OK;
  const unsigned grid = grid_for(n, current_device());
  if (dtype == MICRO_F32)
    k_accumulate<float><<<grid, 256, 0, (cudaStream_t)stream>>>((const float*)d_e, (float)eta, (const float*)d_g,
                                                                (float*)d_acc, n);
  else
    k_accumulate<double><<<grid, 256, 0, (cudaStream_t)stream>>>((const double*)d_e, eta, (const double*)d_g,
                                                                 (double*)d_acc, n);
  CU(cudaGetLastError());
  return MICRO_OK;
}

}  // extern "C"

// Ordered compaction of {j in [start, end) : |acc_j| > thr} (thr = *d_thr or
// delta), plus, with d_tie, {|acc_j| == thr, j <= *d_tie} (top-k's ties):
// the engine's two kernels over the range only — k1_stream in its acc-only
// form (one 4-byte read per element, per-CTA staging runs) and k1_gather
// (ordered copy at each run's prefix) — with scratch from the stream-ordered
// allocator.
template <typename T>
static int select_stream_range(const void* d_acc, int64_t n_g, int64_t start, int64_t end, const double* d_thr,
                               double delta, const long long* d_tie, int32_t* d_idx, void* d_val, int64_t cap,
                               int64_t* d_count, cudaStream_t s) {
  constexpr int UE = stream_unit_elems<T>();
  const int64_t cta_lo = start / UE / kStreamWarps, cta_hi = (end - 1) / UE / kStreamWarps;
  const int64_t runs = cta_hi - cta_lo + 1;
  const int64_t per_run = (int64_t)kStreamWarps * UE;
  const int64_t sup = (runs + kMaxSupers - 1) / kMaxSupers;
  const int super_runs = (int)std::max<int64_t>(kGatherWarps, (sup + kGatherWarps - 1) / kGatherWarps * kGatherWarps);
  const size_t b_idx = sizeof(int32_t) * runs * per_run, b_val = sizeof(T) * runs * per_run;
  const size_t b_cnt = sizeof(int) * runs, b_sup = sizeof(int) * kMaxSupers;
  char* ws = nullptr;
  const size_t tail = (b_idx + b_val + b_cnt + b_sup + 15) / 16 * 16;
  CU(ws_alloc((void**)&ws, tail + 32, s));
  int32_t* stage_idx = (int32_t*)ws;
  T* stage_val = (T*)(ws + b_idx);
  int* counts = (int*)(ws + b_idx + b_val);
  int* supers = (int*)(ws + b_idx + b_val + b_cnt);
  int* flags = (int*)(ws + tail);
  double* thr = (double*)(ws + tail + 16);
  CU(cudaMemsetAsync(supers, 0, b_sup, s));
  CU(cudaMemsetAsync(flags, 0, sizeof(int), s));
  if (!d_thr) {
    long long bits;
    std::memcpy(&bits, &delta, sizeof bits);
    k_fill_i64<<<1, 32, 0, s>>>((long long*)thr, 1, bits);
    CU(cudaGetLastError());
    d_thr = thr;
  }
  StreamArgs a{};
  a.resid = const_cast<void*>(d_acc);  // acc, read only (kNoG, kWriteNone)
  a.n_g = (int)n_g;
  a.p_start = (int)start;
  a.p_end = (int)end;
  a.eta = 1.0;
  a.delta = d_thr;
  a.tie_j = d_tie;
  a.unit_lo = (int)(start / UE);
  a.unit_hi = (int)((end - 1) / UE);
  a.stage_idx = stage_idx;
  a.stage_val = stage_val;
  a.unit_counts = counts;
  a.flags = flags;
  a.super_counts = supers;
  a.super_runs = super_runs;
  a.cta_offset = (int)cta_lo;
  if (d_tie)
    k1_stream<T, kWriteNone, false, false, true, true><<<(unsigned)runs, kStreamThreads, 0, s>>>(a);
  else
    k1_stream<T, kWriteNone, false, false, false, true><<<(unsigned)runs, kStreamThreads, 0, s>>>(a);
  CU(cudaGetLastError());
  CompactArgs b{};
  b.stage_idx = stage_idx;
  b.stage_val = stage_val;
  b.run_counts = counts;
  b.super_counts = supers;
  b.super_clear = supers;
  b.super_len = 0;  // single use
  b.num_runs = (int)runs;
  b.super_runs = super_runs;
  b.run_stride = (int)per_run;
  b.sel_idx = d_idx;
  b.sel_val = d_val;
  b.cap = cap;
  b.count = (long long*)d_count;
  b.flags = flags;
  CU(launch_pdl(k1_gather<T>, dim3((unsigned)((runs + kGatherWarps - 1) / kGatherWarps)), dim3(kGatherWarps * 32), s, b));
  CU(cudaFreeAsync(ws, s));
  return MICRO_OK;
}

extern "C" {

static int select_range(int dtype, const void* d_acc, int64_t n_g, int64_t start, int64_t end, double delta,
                        const double* d_thr, const long long* d_tie, int32_t* d_idx, void* d_val, int64_t cap,
                        int64_t* d_count, void* stream) {
  TRY(check_dtype(dtype));
  if (start < 0 || end < start || end > n_g)
    return fail(MICRO_EINVAL, "selection: range [%lld, %lld) invalid for vector of length %lld",
                (long long)start, (long long)end, (long long)n_g);
  if (n_g >= (int64_t)INT32_MAX) return fail(MICRO_EINVAL, "n_g must be < 2^31 (int32 indices)");
  if (!d_count) return fail(MICRO_EINVAL, "null count pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (end == start) {
    CU(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    return MICRO_OK;
  }
  if ((uintptr_t)d_acc % 16) return fail(MICRO_EINVAL, "acc not 16-byte aligned");
  if (dtype == MICRO_F32)
    return select_stream_range<float>(d_acc, n_g, start, end, d_thr, delta, d_tie, d_idx, d_val, cap, d_count, s);
  return select_stream_range<double>(d_acc, n_g, start, end, d_thr, delta, d_tie, d_idx, d_val, cap, d_count, s);
}

int micro_select_by_threshold(int dtype, const void* d_acc, int64_t n_g, int64_t start, int64_t end,
                              double delta, int32_t* d_idx, void* d_val, int64_t cap, int64_t* d_count,
                              void* stream) {
  if (!(delta >= 0.0) || !std::isfinite(delta))
    return fail(MICRO_EINVAL, "selection: threshold must be finite and nonnegative");
  return select_range(dtype, d_acc, n_g, start, end, delta, nullptr, nullptr, d_idx, d_val, cap, d_count, stream);
}

}  // extern "C"

template <typename T>
static int topk_pivot(const T* acc, int64_t m, int64_t k, int64_t base, TopkState* st, unsigned* hist,
                      unsigned* tie_counts, int dev, cudaStream_t s) {
  k_topk_init<<<1, 1, 0, s>>>(st, k);
  CU(cudaGetLastError());
  const unsigned hgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 4 * (int64_t)num_sms(dev)));
  for (int hi = KeyOf<T>::kBits; hi > 0; hi -= kDigitBits) {
    const int width = std::min(kDigitBits, hi);
    const int shift = hi - width;
    k_topk_hist<T><<<hgrid, 256, 0, s>>>(acc, nullptr, 1.0, m, shift, width, st, hist);
    CU(cudaGetLastError());
    k_topk_digit<T><<<1, 1024, 0, s>>>(st, hist, shift, width, shift == 0, base + m);
    CU(cudaGetLastError());
  }
  const int64_t chunk = tie_chunk(m);
  const int nch = (int)((m + chunk - 1) / chunk);
  k_tie_count<T><<<nch, 256, 0, s>>>(acc, nullptr, 1.0, m, chunk, st, tie_counts);
  CU(cudaGetLastError());
  k_tie_find<T><<<1, 1024, 0, s>>>(acc, nullptr, 1.0, m, chunk, nch, st, tie_counts, base);
  CU(cudaGetLastError());
  return MICRO_OK;
}

extern "C" {

int micro_select_topk(int dtype, const void* d_acc, int64_t n_g, int64_t start, int64_t end, int64_t k,
                      int32_t* d_idx, void* d_val, int64_t cap, int64_t* d_count, void* stream) {
  TRY(check_dtype(dtype));
  if (start < 0 || end < start || end > n_g)
    return fail(MICRO_EINVAL, "selection: range [%lld, %lld) invalid for vector of length %lld",
                (long long)start, (long long)end, (long long)n_g);
  const int64_t m = end - start;
  if (k < 0 || k > m)
    return fail(MICRO_EINVAL, "select_topk: k=%lld exceeds range size %lld", (long long)k, (long long)m);
  if (!d_count) return fail(MICRO_EINVAL, "null count pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (k == 0) {
    CU(cudaMemsetAsync(d_count, 0, sizeof(int64_t), s));
    return MICRO_OK;
  }
  int dev = 0;
  CU(cudaGetDevice(&dev));
  // scratch: state, histogram, tie counts, the "everything" threshold
  const size_t bytes = 256 + sizeof(unsigned) * (kBins + kTieChunks);
  char* ws = nullptr;
  CU(ws_alloc((void**)&ws, bytes, s));
  CU(cudaMemsetAsync(ws, 0, bytes, s));
  auto* st = (TopkState*)ws;
  auto* m1 = (double*)(ws + 128);
  unsigned* hist = (unsigned*)(ws + 256);
  unsigned* ties = hist + kBins;
  int rc = MICRO_OK;
  if (k == m) {  // every index of the range (sparsifier.cpp:56: no nth_element)
    const double minus1 = -1.0;
    CU(cudaMemcpyAsync(m1, &minus1, sizeof minus1, cudaMemcpyHostToDevice, s));
    rc = select_range(dtype, d_acc, n_g, start, end, 0.0, m1, nullptr, d_idx, d_val, cap, d_count, stream);
  } else {
    if (dtype == MICRO_F32)
      rc = topk_pivot<float>((const float*)d_acc + start, m, k, start, st, hist, ties, dev, s);
    else
      rc = topk_pivot<double>((const double*)d_acc + start, m, k, start, st, hist, ties, dev, s);
    if (rc == MICRO_OK)
      rc = select_range(dtype, d_acc, n_g, start, end, 0.0, &st->pivot, &st->tie_j, d_idx, d_val, cap, d_count,
                        stream);
  }
  cudaFreeAsync(ws, s);
  return rc;
}

int micro_compensate(int dtype, void* d_acc, int64_t n_g, const int32_t* d_idx, int64_t k, void* stream) {
  TRY(check_dtype(dtype));
  if (k < 0) return fail(MICRO_EINVAL, "compensate: negative count");
  if (!k) return MICRO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = nullptr;
  CU(ws_alloc((void**)&bad, sizeof(int), s));
  CU(cudaMemsetAsync(bad, 0, sizeof(int), s));
  const unsigned grid = grid_for(k, current_device());
  if (dtype == MICRO_F32) k_compensate<float><<<grid, 256, 0, s>>>((float*)d_acc, n_g, d_idx, k, bad);
  else k_compensate<double><<<grid, 256, 0, s>>>((double*)d_acc, n_g, d_idx, k, bad);
  CU(cudaGetLastError());
  int hbad = 0;
  CU(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(bad, s));
  CU(cudaStreamSynchronize(s));
  if (hbad) return fail(MICRO_EINVAL, "compensate: index out of range");
  return MICRO_OK;
}

static int reduce_values(int dtype, const void* const* h_accs, int n, int64_t n_g, const int32_t* d_union,
                         int64_t K, void* d_sums, void* d_dense, void* stream) {
  TRY(check_dtype(dtype));
  if (n < 1 || !h_accs) return fail(MICRO_EINVAL, "all_reduce_sparse: no workers");
  if (n > kMaxWorkers) return fail(MICRO_EINVAL, "all_reduce_sparse: at most %d workers", kMaxWorkers);
  if (K < 0) return fail(MICRO_EINVAL, "all_reduce_sparse: negative union size");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t esz = dtype_size(dtype);
  if (d_dense) CU(cudaMemsetAsync(d_dense, 0, n_g * esz, s));
  if (!K) return MICRO_OK;
  WorkerPtrs w{};
  for (int r = 0; r < n; ++r) w.sel_val[r] = h_accs[r];
  int* bad = nullptr;
  CU(ws_alloc((void**)&bad, sizeof(int), s));
  CU(cudaMemsetAsync(bad, 0, sizeof(int), s));
  const unsigned grid = grid_for(K, current_device());
  if (dtype == MICRO_F32)
    k_reduce_values<float><<<grid, 256, 0, s>>>(w, n, n_g, d_union, K, (float*)d_sums, (float*)d_dense, bad);
  else
    k_reduce_values<double><<<grid, 256, 0, s>>>(w, n, n_g, d_union, K, (double*)d_sums, (double*)d_dense, bad);
  CU(cudaGetLastError());
  int hbad = 0;
  CU(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(bad, s));
  CU(cudaStreamSynchronize(s));
  if (hbad) return fail(MICRO_EINVAL, "all_reduce_sparse: index out of range");
  return MICRO_OK;
}

int micro_all_reduce_sparse_values(int dtype, const void* const* h_accs, int n, int64_t n_g,
                                   const int32_t* d_union, int64_t K, void* d_sums, void* stream) {
  return reduce_values(dtype, h_accs, n, n_g, d_union, K, d_sums, nullptr, stream);
}

int micro_all_reduce_sparse(int dtype, const void* const* h_accs, int n, int64_t n_g,
                            const int32_t* d_union, int64_t K, void* d_dense, void* stream) {
  if (!d_dense) return fail(MICRO_EINVAL, "null dense output");
  return reduce_values(dtype, h_accs, n, n_g, d_union, K, nullptr, d_dense, stream);
}

int micro_all_gather_indices(int n, const int64_t* h_counts, const int32_t* d_concat, int32_t* d_union,
                             int64_t* K, void* stream) {
  if (n < 0 || (n && !h_counts)) return fail(MICRO_EINVAL, "bad selection list");
  if (!K) return fail(MICRO_EINVAL, "null K");
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    if (h_counts[i] < 0) return fail(MICRO_EINVAL, "negative count");
    total += h_counts[i];
  }
  *K = 0;
  if (!total) return MICRO_OK;
  if (total >= (int64_t)INT32_MAX) return fail(MICRO_EINVAL, "too many indices");
  // sort + unique (collectives.cpp:25-26) as a bitmap over the index extent:
  // mark, popcount prefix (scan.cuh), emit in index order — the same sorted
  // unique union for any input order, duplicates included
  cudaStream_t s = (cudaStream_t)stream;
  const int dev = current_device();
  int* mm = nullptr;
  CU(ws_alloc((void**)&mm, 2 * sizeof(int), s));
  const int init[2] = {INT32_MAX, -1};
  CU(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s));
  k_index_extent<<<grid_for(total, dev), 256, 0, s>>>(d_concat, total, mm);
  CU(cudaGetLastError());
  int hmm[2] = {0, 0};
  CU(cudaMemcpyAsync(hmm, mm, sizeof hmm, cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(mm, s));
  CU(cudaStreamSynchronize(s));
  if (hmm[0] < 0) return fail(MICRO_EINVAL, "all_gather_indices: negative index %d", hmm[0]);
  const int64_t nwords = (int64_t)hmm[1] / 32 + 1;
  const int64_t nt = scan_tiles(nwords);
  char* ws = nullptr;
  const size_t bm = sizeof(unsigned) * nwords, ob = sizeof(int) * nwords, tb = sizeof(int) * nt;
  CU(ws_alloc((void**)&ws, bm + ob + tb + 16, s));
  unsigned* bitmap = (unsigned*)ws;
  int* off = (int*)(ws + bm);
  int* tiles = (int*)(ws + bm + ob);
  long long* dK = (long long*)(ws + ((bm + ob + tb + 7) / 8 * 8));
  CU(cudaMemsetAsync(bitmap, 0, bm, s));
  k_mark_indices<<<grid_for(total, dev), 256, 0, s>>>(d_concat, total, bitmap);
  CU(cudaGetLastError());
  TRY(bitmap_offsets(bitmap, nwords, off, tiles, s));
  k_bitmap_emit<<<grid_for(nwords, dev), 256, 0, s>>>(bitmap, nwords, off, d_union, dK);
  CU(cudaGetLastError());
  long long hk = 0;
  CU(cudaMemcpyAsync(&hk, dK, sizeof hk, cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(ws, s));
  CU(cudaStreamSynchronize(s));
  *K = hk;
  return MICRO_OK;
}

int micro_error_metric(int dtype, const void* const* h_res, int n, int64_t n_g, double* out, void* stream) {
  TRY(check_dtype(dtype));
  if (n < 1 || !h_res) return fail(MICRO_EINVAL, "error_metric: no workers");
  if (n_g < 0 || !out) return fail(MICRO_EINVAL, "error_metric: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((n_g + 255) / 256, 4 * (int64_t)num_sms(dev)));
  const int64_t groups = sumsq_groups(grid);
  // one scratch block: per-worker slots (part, group, ticket) + n totals
  const size_t bytes = sizeof(double) * (size_t)n * (grid + groups + 1) + sizeof(unsigned) * (size_t)n * (groups + 1);
  char* scratch = nullptr;
  CU(ws_alloc((void**)&scratch, bytes, s));
  CU(cudaMemsetAsync(scratch, 0, bytes, s));
  double* part = (double*)scratch;
  double* grp = part + (size_t)n * grid;
  double* tot = grp + (size_t)n * groups;
  unsigned* tick = (unsigned*)(tot + n);
  for (int i = 0; i < n; ++i) {
    if (n_g && !h_res[i]) {
      cudaFreeAsync(scratch, s);
      return fail(MICRO_EINVAL, "error_metric: null residual %d", i);
    }
    SumSqSlots q{part + (size_t)i * grid, grp + (size_t)i * groups, tick + (size_t)i * (groups + 1), tot + i};
    if (n_g == 0) continue;
    if (dtype == MICRO_F32) k_sumsq<float><<<(unsigned)grid, 256, 0, s>>>((const float*)h_res[i], n_g, q);
    else k_sumsq<double><<<(unsigned)grid, 256, 0, s>>>((const double*)h_res[i], n_g, q);
    CU(cudaGetLastError());
  }
  std::vector<double> h(n);
  CU(cudaMemcpyAsync(h.data(), tot, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  CU(cudaFreeAsync(scratch, s));
  CU(cudaStreamSynchronize(s));
  double sum = 0.0;  // error_feedback.hpp:44-47: norms summed in worker order, then / n
  for (int i = 0; i < n; ++i) sum += std::sqrt(h[i]);
  *out = sum / (double)n;
  return MICRO_OK;
}

}  // extern "C"
