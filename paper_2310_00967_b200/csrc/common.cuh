// common.cuh — shared device helpers for the MiCRO sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace micro {

constexpr int kMaxWorkers = 64;  // MICRO_MAX_WORKERS

// 16-byte vector of T: 4 floats or 2 doubles per load/store.
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using V = float4;
  static constexpr int N = 4;
};
template <>
struct Vec<double> {
  using V = double2;
  static constexpr int N = 2;
};

__device__ __forceinline__ float comp(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
__device__ __forceinline__ double comp(const double2& v, int c) { return c == 0 ? v.x : v.y; }
__device__ __forceinline__ void set_comp(float4& v, int c, float x) {
  if (c == 0) v.x = x; else if (c == 1) v.y = x; else if (c == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ void set_comp(double2& v, int c, double x) {
  if (c == 0) v.x = x; else v.y = x;
}

// Explicitly rounded arithmetic: never contracted into FMA.
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// The selection threshold in T such that |x| > thr  <=>  (double)|x| > delta
// for every x of type T (SURVEY.md §8c fp32 contract): round delta down.
__device__ __forceinline__ float threshold_as(double delta, float*) { return __double2float_rd(delta); }
__device__ __forceinline__ double threshold_as(double delta, double*) { return delta; }

__device__ __forceinline__ float absx(float x) { return fabsf(x); }
__device__ __forceinline__ double absx(double x) { return fabs(x); }

__device__ __forceinline__ bool finite(float x) { return isfinite(x); }
__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// Streaming loads/stores (data touched once per pass).
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
// read-only, no L1 allocation (the gradient: read once per pass)
__device__ __forceinline__ float4 ld_nc_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_nc_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(float4* p, const float4& v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, const double2& v) { __stcs(p, v); }

// ---- L2 eviction policies (createpolicy + .L2::cache_hint) ----
// The 12 B/elem streams go through L2 evict-first; the small K1 staging runs
// are written evict-last so the compaction reads them from L2, then are
// discarded without write-back (discard.global.L2).
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ld_hint(const float4* p, unsigned long long pol) {
  float4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, unsigned long long pol) {
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_nc_hint(const float4* p, unsigned long long pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_nc_hint(const double2* p, unsigned long long pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
  return r;
}
// The gradient's vector of VN elements (K1's G loads): the state's own
// vector, or VN fp32 values widened exactly to the fp64 state (float2 ->
// double2: 8 B per lane).
template <typename TG, int VN>
struct GradVec;
template <>
struct GradVec<float, 4> { using V = float4; };
template <>
struct GradVec<double, 2> { using V = double2; };
template <>
struct GradVec<float, 2> { using V = float2; };
template <typename V>
__device__ __forceinline__ V ld_grad(const V* p, unsigned long long pol) { return ld_nc_hint(p, pol); }
template <typename V>
__device__ __forceinline__ V ld_grad(const float2* p, unsigned long long pol) {
  float2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
               : "=f"(r.x), "=f"(r.y) : "l"(p), "l"(pol));
  return V{(double)r.x, (double)r.y};
}
__device__ __forceinline__ void st_hint(float4* p, const float4& v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2* p, const double2& v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(int* p, int v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float* p, float v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
// Scattered read-modify-write targets (the model x at the union): ask L2 to
// fetch only the 64-byte half around the word instead of its default span.
__device__ __forceinline__ float ld_rand(const float* p) {
  float v;
  asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_rand(const double* p) {
  double v;
  asm volatile("ld.global.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Programmatic dependent launch (PDL): a kernel launched with programmatic
// stream serialization may start while its predecessor drains; it must wait
// for the predecessor's completion (and memory) before touching its results.
// Both are no-ops for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Drop a 128-byte L2 line without writing it back (its content is dead).
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// gpu-scope relaxed 64-bit status words (look-back).
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// cycle = (t % n + worker) % n; balanced contiguous ranges, remainder first
// (tensor.hpp:48-63).  Device copy of the host function.
__host__ __device__ __forceinline__ void partition_range(int64_t n_g, int n, int64_t t, int worker,
                                                         int64_t* start, int64_t* end) {
  const int64_t cycle = (t % n + worker) % n;
  const int64_t base = n_g / n, rem = n_g % n;
  const int64_t s = cycle * base + (cycle < rem ? cycle : rem);
  *start = s;
  *end = s + base + (cycle < rem ? 1 : 0);
}

// Owner (worker id) of partition p at iteration t: (t % n + i) % n == p.
__host__ __device__ __forceinline__ int partition_owner(int p, int n, int64_t t) {
  return (int)(((int64_t)p - t % n + n) % n);
}

}  // namespace micro
