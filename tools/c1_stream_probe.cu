// c1_stream_probe.cu — what bounds a K1-shaped stream at C1 size (11.7M
// elements, f64 e read+write, fp32 G read: 20 B/elem, L2 flushed between
// reps).  Variants, all computing e = e + eta*(double)g:
//   0  grid-stride, 4 vectors per operand in flight per thread (torch-like)
//   1  one warp per 256-element unit, 8 units per CTA, loads up front (K1's shape)
//   2  as 1, two units per warp, both units' loads up front
//   3  as 1 + a CTA barrier after the compute (K1's compaction sync)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o c1_stream_probe tools/c1_stream_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ldd(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float2 ldf(const float2* p) { return __ldcs(p); }

__global__ void v0(double2* e, const float2* g, long nv, double eta) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long q0 = blockIdx.x * (long)blockDim.x + threadIdx.x; q0 < nv; q0 += 4 * stride) {
    double2 a[4]; float2 b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) if (q0 + u * stride < nv) { a[u] = ldd(e + q0 + u * stride); b[u] = ldf(g + q0 + u * stride); }
#pragma unroll
    for (int u = 0; u < 4; ++u) if (q0 + u * stride < nv) {
      a[u].x = __dadd_rn(a[u].x, __dmul_rn(eta, (double)b[u].x));
      a[u].y = __dadd_rn(a[u].y, __dmul_rn(eta, (double)b[u].y));
      __stcs(e + q0 + u * stride, a[u]);
    }
  }
}

template <int UPW, bool SYNC>
__global__ void __launch_bounds__(256) vunit(double2* e, const float2* g, long nv, double eta) {
  // unit = 128 double2 vectors (256 elements); warp w of CTA b handles units (b*8*UPW + w + 8*k)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 a[UPW][4]; float2 b[UPW][4];
  long base[UPW];
#pragma unroll
  for (int k = 0; k < UPW; ++k) {
    base[k] = ((long)blockIdx.x * 8 * UPW + w + 8 * k) * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long q = base[k] + i * 32 + lane;
      if (q < nv) { a[k][i] = ldd(e + q); b[k][i] = ldf(g + q); }
    }
  }
#pragma unroll
  for (int k = 0; k < UPW; ++k) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[k][i].x = __dadd_rn(a[k][i].x, __dmul_rn(eta, (double)b[k][i].x));
      a[k][i].y = __dadd_rn(a[k][i].y, __dmul_rn(eta, (double)b[k][i].y));
    }
    if (SYNC) __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long q = base[k] + i * 32 + lane;
      if (q < nv) __stcs(e + q, a[k][i]);
    }
  }
}

__global__ void sweep(const int4* p, long n, int* sink) {  // read the flush buffer: its lines become clean
  int acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) acc ^= __ldcg(p + i).x;
  if (acc == 0x7fffffff) *sink = acc;
}

int main() {
  const long n = 11700000, nv = n / 2;
  double2* e; float2* g; char* flush;
  cudaMalloc(&e, n * 8); cudaMalloc(&g, n * 4); cudaMalloc(&flush, 512l << 20);
  cudaMemset(e, 0, n * 8); cudaMemset(g, 0, n * 4);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto time = [&](const char* name, auto launch) {
    float best = 1e9f, sum = 0; int reps = 30;
    for (int r = 0; r < reps + 3; ++r) {
      cudaMemsetAsync(flush, r & 0xff, 256l << 20);  // evict e and G from L2 ...
      sweep<<<sms * 8, 256>>>((const int4*)(flush + (256l << 20)), (256l << 20) / 16, (int*)flush);  // ... and leave it clean
      cudaEventRecord(t0); launch(); cudaEventRecord(t1); cudaEventSynchronize(t1);
      float ms; cudaEventElapsedTime(&ms, t0, t1);
      if (r >= 3) { best = ms < best ? ms : best; sum += ms; }
    }
    printf("%-44s best %7.2f us  mean %7.2f us  (%5.2f TB/s at 20 B/elem, best)\n", name, best * 1e3, sum / reps * 1e3,
           n * 20.0 / (best * 1e-3) / 1e12);
  };
  const double eta = 0.01;
  time("copy e -> e2 (cudaMemcpyAsync, 16 B/elem)", [&] { cudaMemcpyAsync(flush, e, n * 8, cudaMemcpyDeviceToDevice); });
  time("v0 grid-stride x4 (4 CTAs/SM x 256)", [&] { v0<<<sms * 8, 256>>>(e, g, nv, eta); });
  time("v0 grid-stride x4 (16 CTAs/SM)", [&] { v0<<<sms * 16, 256>>>(e, g, nv, eta); });
  const long units = (nv + 127) / 128;
  time("v1 unit/warp, 8 units/CTA", [&] { vunit<1, false><<<(units + 7) / 8, 256>>>(e, g, nv, eta); });
  time("v2 two units/warp", [&] { vunit<2, false><<<(units + 15) / 16, 256>>>(e, g, nv, eta); });
  time("v3 unit/warp + CTA barrier", [&] { vunit<1, true><<<(units + 7) / 8, 256>>>(e, g, nv, eta); });
  time("v3b two units/warp + CTA barriers", [&] { vunit<2, true><<<(units + 15) / 16, 256>>>(e, g, nv, eta); });
  return 0;
}
