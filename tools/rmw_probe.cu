// rmw_probe.cu — the floor of the sparse model update x[j] -= v on B200:
// K sorted random indices (density d) into an n-element fp32 vector.
//   0: one thread per index, plain RMW        1: 0 with ld.global.L2::64B
//   2: 4 indices per thread (ILP), 64B hint   3: write only x[j] = v
//   4: read only (sum x[j])                   5: 2 with ld.global.L2::128B
//   6: whole 32-byte sector writes at a random subset of sectors (the dense
//      g/n pattern), 7: the same sectors with streaming (.cs) stores
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o rmw_probe tools/rmw_probe.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ float ld64(const float* p) {
  float v;
  asm volatile("ld.global.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld128(const float* p) {
  float v;
  asm volatile("ld.global.L2::128B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <int V>
__global__ void __launch_bounds__(256) rmw(float* x, const int* idx, const float* val, long K, float* sink) {
  const long tid = blockIdx.x * 256L + threadIdx.x;
  if (V == 2 || V == 5) {
    const long b = tid * 4;
    if (b >= K) return;
    int j[4];
    float v[4], y[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      j[q] = b + q < K ? idx[b + q] : -1;
      v[q] = b + q < K ? val[b + q] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) y[q] = j[q] >= 0 ? (V == 2 ? ld64(x + j[q]) : ld128(x + j[q])) : 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j[q] >= 0) x[j[q]] = y[q] - v[q];
    return;
  }
  if (tid >= K) return;
  const int j = idx[tid];
  const float v = val[tid];
  if (V == 0) x[j] = x[j] - v;
  if (V == 1) x[j] = ld64(x + j) - v;
  if (V == 3) x[j] = v;
  if (V == 4) {
    const float y = x[j];
    if (y == 12345.f) sink[0] = y;
  }
}

template <int V>
__global__ void __launch_bounds__(256) secw(float* x, const int* sec, long K) {
  const long tid = blockIdx.x * 256L + threadIdx.x;
  if (tid >= K) return;
  float4* p = reinterpret_cast<float4*>(x) + 2L * sec[tid];
  const float4 z = make_float4(0.5f, 0.f, 0.f, 0.25f);
  if (V == 6) {
    p[0] = z;
    p[1] = z;
  } else {
    __stcs(p, z);
    __stcs(p + 1, z);
  }
}

template <int V>
float run_sec(float* x, const int* sec, long K, float* flush, size_t fbytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 12; ++r) {
    cudaMemsetAsync(flush, r, fbytes);
    cudaEventRecord(a);
    secw<V><<<(unsigned)((K + 255) / 256), 256>>>(x, sec, K);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) best = ms < best ? ms : best;
  }
  printf("  variant %d: %ld sectors, best %.1f us (%.0f GB/s of 32-byte writes)\n", V, K, best * 1e3,
         K * 32.0 / (best * 1e-3) / 1e9);
  return best;
}

template <int V>
float run(float* x, const int* idx, const float* val, long K, float* sink, float* flush, size_t fbytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const long per = (V == 2 || V == 5) ? 4 : 1;
  const unsigned grid = (unsigned)((K + 256 * per - 1) / (256 * per));
  float best = 1e9f, sum = 0.f;
  int cnt = 0;
  for (int r = 0; r < 12; ++r) {
    cudaMemsetAsync(flush, r, fbytes);  // evict x from L2
    cudaEventRecord(a);
    rmw<V><<<grid, 256>>>(x, idx, val, K, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) {
      best = std::min(best, ms);
      sum += ms;
      ++cnt;
    }
  }
  printf("  variant %d: best %.1f us  mean %.1f us  (%.0f GB/s at 64 B/access)\n", V, best * 1e3,
         sum / cnt * 1e3, K * 64.0 / (best * 1e-3) / 1e9);
  return best;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 138000000L;
  const double d = argc > 2 ? atof(argv[2]) : 0.0109;
  std::mt19937_64 rng(1);
  std::bernoulli_distribution pick(d);
  std::vector<int> hidx;
  for (long j = 0; j < n; ++j)
    if (pick(rng)) hidx.push_back((int)j);
  const long K = (long)hidx.size();
  std::vector<float> hval(K, 0.5f);
  float *x, *val, *sink, *flush;
  int* idx;
  const size_t fbytes = 512ull << 20;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&idx, K * 4);
  cudaMalloc(&val, K * 4);
  cudaMalloc(&sink, 4);
  cudaMalloc(&flush, fbytes);
  cudaMemset(x, 0, n * 4);
  cudaMemcpy(idx, hidx.data(), K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(val, hval.data(), K * 4, cudaMemcpyHostToDevice);
  printf("n = %ld, K = %ld (density %.4f %%)\n", n, K, 100.0 * K / n);
  run<0>(x, idx, val, K, sink, flush, fbytes);
  run<1>(x, idx, val, K, sink, flush, fbytes);
  run<2>(x, idx, val, K, sink, flush, fbytes);
  run<5>(x, idx, val, K, sink, flush, fbytes);
  run<3>(x, idx, val, K, sink, flush, fbytes);
  run<4>(x, idx, val, K, sink, flush, fbytes);
  {  // the dense g/n pattern: ~2 x 8.5 % of the sectors, whole 32-byte writes
    std::bernoulli_distribution pick_s(argc > 3 ? atof(argv[3]) : 0.17);
    std::vector<int> hs;
    for (long s = 0; s < n / 8; ++s)
      if (pick_s(rng)) hs.push_back((int)s);
    int* dsec;
    cudaMalloc(&dsec, hs.size() * 4);
    cudaMemcpy(dsec, hs.data(), hs.size() * 4, cudaMemcpyHostToDevice);
    run_sec<6>(x, dsec, (long)hs.size(), flush, fbytes);
    run_sec<7>(x, dsec, (long)hs.size(), flush, fbytes);
    cudaFree(dsec);
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
