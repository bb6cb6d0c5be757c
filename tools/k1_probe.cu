// k1_probe.cu — isolates what limits the K1 streaming pass on B200.
// Variants of e = e + eta*G over n floats (12 B/elem), timed with events:
//   0: plain ld/st (torch-like)          1: st.global.cs stores
//   2: ld.global.cs e + st.global.cs     3: 0 + |acc|>thr mask + popc (no pairs)
//   4: 3 + zero selected in the store    5: 4 + warp scan of counts
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o k1_probe tools/k1_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void __launch_bounds__(256) probe(float4* e, const float4* g, long n4, float eta, float thr,
                                             unsigned* out) {
  unsigned cnt = 0;
  for (long i = blockIdx.x * 256L + threadIdx.x; i < n4; i += (long)gridDim.x * 256L) {
    float4 a = V >= 2 ? __ldcs(e + i) : e[i];
    const float4 b = __ldg(g + i);
    a.x = __fadd_rn(a.x, __fmul_rn(eta, b.x));
    a.y = __fadd_rn(a.y, __fmul_rn(eta, b.y));
    a.z = __fadd_rn(a.z, __fmul_rn(eta, b.z));
    a.w = __fadd_rn(a.w, __fmul_rn(eta, b.w));
    if (V >= 3) {
      const unsigned m = (fabsf(a.x) > thr) | (fabsf(a.y) > thr) << 1 | (fabsf(a.z) > thr) << 2 |
                         (fabsf(a.w) > thr) << 3;
      unsigned c = __popc(m);
      if (V >= 5) {
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, c, o);
          if ((threadIdx.x & 31) >= o) c += y;
        }
      }
      cnt += c;
      if (V >= 4) {
        if (m & 1) a.x = 0.f;
        if (m & 2) a.y = 0.f;
        if (m & 4) a.z = 0.f;
        if (m & 8) a.w = 0.f;
      }
    }
    if (V >= 1) __stcs(e + i, a); else e[i] = a;
  }
  if (cnt == 0xFFFFFFFFu) out[0] = cnt;
}

template <int V>
float run(float4* e, const float4* g, long n4, unsigned* out, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    probe<V><<<grid, 256>>>(e, g, n4, 0.01f, 0.03f, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 138000000L;
  const long n4 = n / 4;
  float4 *e, *g;
  unsigned* out;
  cudaMalloc(&e, n4 * 16);
  cudaMalloc(&g, n4 * 16);
  cudaMalloc(&out, 4);
  cudaMemset(e, 0, n4 * 16);
  cudaMemset(g, 0x3c, n4 * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {8, 32, 0}) {
    const int grid = mult ? sms * mult : (int)((n4 + 255) / 256);
    float t[6] = {run<0>(e, g, n4, out, grid), run<1>(e, g, n4, out, grid), run<2>(e, g, n4, out, grid),
                  run<3>(e, g, n4, out, grid), run<4>(e, g, n4, out, grid), run<5>(e, g, n4, out, grid)};
    for (int v = 0; v < 6; ++v)
      printf("grid %8d variant %d: %.1f us  %.0f GB/s\n", grid, v, t[v] * 1e3, 12.0 * n / (t[v] * 1e-3) / 1e9);
  }
  return 0;
}

// ---- access-pattern probes (same arithmetic as variant 0) ----
// P1: every warp streams its own contiguous range (units of 256 float4 = 32 lanes x 8)
// P2: every CTA streams a contiguous range, its warps round-robin over 32-float4 units
template <int PAT>
__global__ void __launch_bounds__(256) pattern(float4* e, const float4* g, long n4, float eta) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long GW = (long)gridDim.x * 8, gw = (long)blockIdx.x * 8 + w;
  constexpr int U = 64;  // float4 per unit (2 per lane)
  const long units = n4 / U;
  long u0, u1, step;
  if (PAT == 1) { u0 = units * gw / GW; u1 = units * (gw + 1) / GW; step = 1; }
  else { u0 = units * blockIdx.x / gridDim.x + w; u1 = units * (blockIdx.x + 1) / gridDim.x; step = 8; }
  for (long u = u0; u < u1; u += step) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const long idx = u * U + i * 32 + lane;
      float4 a = e[idx];
      const float4 b = __ldg(g + idx);
      a.x = __fadd_rn(a.x, __fmul_rn(eta, b.x));
      a.y = __fadd_rn(a.y, __fmul_rn(eta, b.y));
      a.z = __fadd_rn(a.z, __fmul_rn(eta, b.z));
      a.w = __fadd_rn(a.w, __fmul_rn(eta, b.w));
      e[idx] = a;
    }
  }
}

template <int PAT>
float runp(float4* e, const float4* g, long n4, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    pattern<PAT><<<grid, 256>>>(e, g, n4, 0.01f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < best) best = ms;
  }
  return best;
}

struct PatternMain {
  PatternMain() {
    const long n = 138000000L, n4 = n / 4;
    float4 *e, *g;
    cudaMalloc(&e, n4 * 16);
    cudaMalloc(&g, n4 * 16);
    cudaMemset(e, 0, n4 * 16);
    cudaMemset(g, 0x3c, n4 * 16);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mult : {1, 2, 4, 8}) {
      const int grid = sms * mult;
      const float t1 = runp<1>(e, g, n4, grid), t2 = runp<2>(e, g, n4, grid);
      printf("pattern grid %5d: per-warp ranges %.1f us %.0f GB/s | per-CTA window %.1f us %.0f GB/s\n", grid,
             t1 * 1e3, 12.0 * n / (t1 * 1e-3) / 1e9, t2 * 1e3, 12.0 * n / (t2 * 1e-3) / 1e9);
    }
    cudaFree(e);
    cudaFree(g);
  }
} pattern_main;
