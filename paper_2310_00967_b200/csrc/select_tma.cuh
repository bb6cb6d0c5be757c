// select_tma.cuh — K1, persistent TMA-staged variant (the production path).
//
// Same semantics as k1_fused_select (select.cuh; reference harness.cpp:131,
// sparsifier.cpp:22-37, harness.cpp:219-221), different schedule:
//
//  * one CTA per SM (grid = #SMs), persistent; 16 consumer warps + 1
//    producer warp;
//  * the producer streams e_t and G tiles (16 KB per operand) into a 4-stage
//    shared-memory ring with cp.async.bulk (the TMA bulk-copy engine),
//    completion tracked by mbarrier transaction counts, so 128 KB per SM are
//    always in flight independent of what the consumers are doing;
//  * consumers compute acc = e + eta*G, write e_{t+1} straight back to HBM
//    (coalesced 16-byte streaming stores), compact the selected (index,
//    value) pairs tile by tile into a per-CTA staging run (block scan, no
//    cross-CTA dependency inside the streaming loop);
//  * each CTA owns a contiguous, balanced slice of the partition's tiles (so
//    its staged run is globally ordered) plus a slice of the other tiles;
//    after its partition slice it publishes its count, resolves its global
//    offset with ONE decoupled look-back over the #SMs CTAs, and copies its
//    run into place while the producer keeps prefetching.
//
// Cost per worker: 12*n_g bytes (read e, G; write e) + 8 bytes per selected
// pair + 16 bytes per pair of staging round trip (0.16 B/elem at d = 1%).
#pragma once

#include "common.cuh"
#include "select.cuh"

namespace micro {

constexpr int kTmaConsumerWarps = 16;
constexpr int kTmaConsumers = kTmaConsumerWarps * 32;       // 512
constexpr int kTmaThreads = kTmaConsumers + 32;             // + producer warp
constexpr int kTmaStages = 4;
constexpr int kTmaTileBytes = 16384;                        // per operand per stage
constexpr int kTmaSmemBytes = kTmaStages * 2 * kTmaTileBytes + 1024;

template <typename T>
__host__ __device__ constexpr int tma_tile_elems() {
  return kTmaTileBytes / (int)sizeof(T);  // 4096 fp32 / 2048 fp64
}

struct TmaSelectArgs {
  const void* grad;
  void* resid;
  int64_t n_g;
  int64_t p_start, p_end;
  double eta;
  const double* delta;
  int32_t* sel_idx;
  void* sel_val;
  int64_t cap;
  long long* count;
  int32_t* stage_idx;          // staging runs, (ptile_hi - ptile_lo + 1) * TILE pairs
  void* stage_val;
  unsigned long long* status;  // >= status_len words
  int64_t status_len;
  unsigned int epoch;
  int* flags;
  int64_t num_tiles;
  int64_t ptile_lo, ptile_hi;  // tiles intersecting [p_start, p_end)
};

// ---- mbarrier / bulk-copy primitives (inline PTX, sm_90+) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {  // named barrier over the 512 consumer threads
  asm volatile("bar.sync 1, %0;" ::"n"(kTmaConsumers) : "memory");
}

// Tile sequence of CTA b: its slice of the partition tiles, then its slice of
// the remaining tiles.
struct TilePlan {
  int64_t p_lo, p_n;  // partition tiles [p_lo, p_lo + p_n)
  int64_t o_lo, o_n;  // index range in the outside-tile list
  int64_t gap_lo, gap_n;
  __device__ __forceinline__ int64_t count() const { return p_n + o_n; }
  __device__ __forceinline__ int64_t tile(int64_t k) const {
    if (k < p_n) return p_lo + k;
    const int64_t q = o_lo + (k - p_n);
    return q < gap_lo ? q : q + gap_n;  // skip over the partition tiles
  }
};

__device__ __forceinline__ TilePlan make_plan(const TmaSelectArgs& a, int b, int G) {
  TilePlan pl;
  const int64_t P = a.ptile_hi - a.ptile_lo + 1;
  const int64_t O = a.num_tiles - P;
  const int64_t p0 = P * b / G, p1 = P * (b + 1) / G;
  const int64_t o0 = O * b / G, o1 = O * (b + 1) / G;
  pl.p_lo = a.ptile_lo + p0;
  pl.p_n = p1 - p0;
  pl.o_lo = o0;
  pl.o_n = o1 - o0;
  pl.gap_lo = a.ptile_lo;
  pl.gap_n = P;
  return pl;
}

template <typename T, int kMode>
__global__ void __launch_bounds__(kTmaThreads, 1) k1_tma_select(TmaSelectArgs a) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  constexpr int TILE = tma_tile_elems<T>();
  constexpr int VPT = TILE / VN / kTmaConsumers;  // vectors per consumer thread per operand (2)
  static_assert(VPT * VN * kTmaConsumers == TILE, "tile/threads mismatch");

  extern __shared__ __align__(1024) unsigned char smem[];
  T* s_e = reinterpret_cast<T*>(smem);                                  // [stages][TILE]
  T* s_g = reinterpret_cast<T*>(smem + kTmaStages * kTmaTileBytes);     // [stages][TILE]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kTmaStages * kTmaTileBytes);
  uint64_t* empty = full + kTmaStages;
  __shared__ unsigned int s_warp[2][kTmaConsumerWarps];
  __shared__ long long s_excl;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x, G = gridDim.x;
  const TilePlan pl = make_plan(a, b, G);
  const int64_t ntiles = pl.count();
  const int64_t n_g = a.n_g;

  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kTmaConsumerWarps) {
    // ================= producer warp: one elected lane streams tiles =========
    if (lane == 0) {
      const T* E = (const T*)a.resid;
      const T* Gp = (const T*)a.grad;
      for (int64_t k = 0; k < ntiles; ++k) {
        const int s = (int)(k % kTmaStages);
        const uint32_t round = (uint32_t)(k / kTmaStages);
        if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
        const int64_t tile = pl.tile(k);
        const int64_t base = tile * TILE;
        int64_t elems = n_g - base < TILE ? n_g - base : TILE;
        const uint32_t bytes = (uint32_t)((elems * (int64_t)sizeof(T)) & ~(int64_t)15);
        mbar_arrive_expect_tx(&full[s], 2 * bytes);
        if (bytes) {
          bulk_g2s(s_e + (size_t)s * TILE, E + base, bytes, &full[s]);
          bulk_g2s(s_g + (size_t)s * TILE, Gp + base, bytes, &full[s]);
        }
      }
    }
    return;
  }

  // ================= consumers ===============================================
  const double delta = *a.delta;
  const T thr = threshold_as(delta, (T*)nullptr);
  const T eta = (T)a.eta;
  T* __restrict__ E = (T*)a.resid;
  const T* __restrict__ Gp = (const T*)a.grad;
  int32_t* __restrict__ st_idx = a.stage_idx;
  T* __restrict__ st_val = (T*)a.stage_val;
  const int64_t run_base = (pl.p_lo - a.ptile_lo) * TILE;  // this CTA's staging run
  long long run = 0;                                       // pairs staged so far
  bool bad = false;

  for (int64_t k = 0; k < ntiles; ++k) {
    const int s = (int)(k % kTmaStages);
    const uint32_t round = (uint32_t)(k / kTmaStages);
    const int64_t tile = pl.tile(k);
    const int64_t base = tile * TILE;
    const int64_t elems = n_g - base < TILE ? n_g - base : TILE;
    const int64_t vec_elems = ((elems * (int64_t)sizeof(T)) & ~(int64_t)15) / (int64_t)sizeof(T);
    mbar_wait(&full[s], round & 1);

    V e[VPT];
    unsigned mask[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int v = i * kTmaConsumers + tid;
      const int64_t off = (int64_t)v * VN;
      V g;
      if (off + VN <= vec_elems) {
        e[i] = reinterpret_cast<const V*>(s_e + (size_t)s * TILE)[v];
        g = reinterpret_cast<const V*>(s_g + (size_t)s * TILE)[v];
      } else {  // the vector's tail (last tile only): straight from global
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          const bool in = off + c < elems;
          set_comp(e[i], c, in ? E[base + off + c] : (T)0);
          set_comp(g, c, in ? Gp[base + off + c] : (T)0);
        }
      }
      mask[i] = 0;
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const int64_t j = base + off + c;
        const T gv = comp(g, c);
        bad |= (off + c < elems) && !finite(gv);
        const T acc = add_rn(comp(e[i], c), mul_rn(eta, gv));  // two roundings, no FMA
        set_comp(e[i], c, acc);
        mask[i] |= (unsigned)((j >= a.p_start) && (j < a.p_end) && (absx(acc) > thr)) << c;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s

    if (kMode != kWriteNone) {
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        const int v = i * kTmaConsumers + tid;
        const int64_t off = (int64_t)v * VN;
        V out = e[i];
        if (kMode == kWriteZeroSel) {
#pragma unroll
          for (int c = 0; c < VN; ++c)
            if (mask[i] & (1u << c)) set_comp(out, c, (T)0);
        }
        if (off + VN <= elems) {
          st_stream(reinterpret_cast<V*>(E + base + off), out);
        } else {
#pragma unroll
          for (int c = 0; c < VN; ++c)
            if (off + c < elems) E[base + off + c] = comp(out, c);
        }
      }
    }

    if (k < pl.p_n) {
      // ---- ordered compaction of this partition tile into the CTA's run ----
      unsigned packed = 0;
#pragma unroll
      for (int i = 0; i < VPT; ++i) packed |= (unsigned)__popc(mask[i]) << (16 * i);
      unsigned incl = packed;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int par = (int)(k & 1);
      if (lane == 31) s_warp[par][warp] = incl;
      consumer_sync();
      unsigned wpre = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kTmaConsumerWarps; ++w) {
        const unsigned x = s_warp[par][w];
        wpre += w < warp ? x : 0u;
        tot += x;
      }
      const unsigned excl = wpre + incl - packed;
      int cbase[VPT];
      int tcount = 0;
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        cbase[i] = tcount;
        tcount += (int)((tot >> (16 * i)) & 0xFFFFu);
      }
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        if (!mask[i]) continue;
        long long pos = run_base + run + cbase[i] + (long long)((excl >> (16 * i)) & 0xFFFFu);
        const int64_t j0 = base + (int64_t)(i * kTmaConsumers + tid) * VN;
#pragma unroll
        for (int c = 0; c < VN; ++c)
          if (mask[i] & (1u << c)) {
            st_idx[pos] = (int32_t)(j0 + c);
            st_val[pos] = comp(e[i], c);
            ++pos;
          }
      }
      run += tcount;
    }

    if (k + 1 == pl.p_n || (pl.p_n == 0 && k == 0)) {
      // ---- partition slice done: global offset by one look-back, copy run ----
      consumer_sync();  // staged pairs of all warps written
      if (warp == 0) {
        const long long ex = lookback(a.status, b, (unsigned long long)run, a.epoch, lane);
        if (lane == 0) {
          s_excl = ex;
          if (b == G - 1) {
            const long long total = ex + run;
            *a.count = total;
            if (total > a.cap) atomicOr(a.flags, 2);
            const unsigned long long ep = (unsigned long long)(a.epoch & 0xFFFFFFu) << 40;
            for (int64_t q = G; q < a.status_len; ++q) st_relaxed_u64(&a.status[q], ep);
          }
        }
      }
      consumer_sync();
      const long long dst0 = s_excl;
      int32_t* __restrict__ out_idx = a.sel_idx;
      T* __restrict__ out_val = (T*)a.sel_val;
      for (long long m = tid; m < run; m += kTmaConsumers) {
        const long long d = dst0 + m;
        if (d < a.cap) {
          out_idx[d] = st_idx[run_base + m];
          out_val[d] = st_val[run_base + m];
        }
      }
    }
  }
  if (ntiles == 0 && warp == 0) {  // CTA without tiles still closes its link of the chain
    const long long ex = lookback(a.status, b, 0ull, a.epoch, lane);
    if (lane == 0 && b == G - 1) {
      *a.count = ex;
      if (ex > a.cap) atomicOr(a.flags, 2);
      const unsigned long long ep = (unsigned long long)(a.epoch & 0xFFFFFFu) << 40;
      for (int64_t q = G; q < a.status_len; ++q) st_relaxed_u64(&a.status[q], ep);
    }
  }
  if (bad) atomicOr(a.flags, 1);
}

}  // namespace micro
