// select_tma.cuh — K1, persistent warp-streaming variant (the production path).
//
// Same semantics as k1_fused_select (select.cuh; reference harness.cpp:131,
// sparsifier.cpp:22-37, harness.cpp:219-221), different schedule:
//
//  * one CTA per SM (grid = #SMs), 8 warps, every warp an independent
//    streaming engine over its own contiguous range of the vector;
//  * each warp runs its own 4-stage shared-memory ring: its lane 0 streams
//    2 KB units of e_t and G with cp.async.bulk (the TMA bulk-copy engine),
//    completion tracked by per-warp mbarrier transaction counts, and refills
//    a stage as soon as the warp has read it — 16 KB per warp, 128 KB per SM
//    in flight, with no cross-warp synchronisation in the streaming loop;
//  * the warp computes acc = e + eta*G with explicitly rounded arithmetic,
//    writes e_{t+1} straight back with coalesced 16-byte streaming stores,
//    and compacts selected (index, value) pairs with one packed warp scan
//    per unit into its own staged run (ordered: warps own contiguous,
//    balanced slices of the partition, in (CTA, warp) order);
//  * after the partition slices every CTA sums its warps' runs, resolves its
//    global offset with ONE decoupled look-back over the #SMs CTAs, and each
//    warp copies its run into place; then the warps stream the units outside
//    the partition (accumulate only).
//
// ncu on the first TMA version (one CTA-wide ring, 16 consumer warps, a
// block scan + barrier per 16 KB tile) showed 56 instructions per element
// and an ALU pipe at 68 %: the consumers, not HBM, were the limit.  Here the
// inner loop is ~8 instructions per element and warps never wait on each
// other while streaming.
//
// Bytes per worker: 12*n_g (read e, G; write e) + 8 per selected pair
// + 16 per pair for the staging round trip (0.16 B/elem at d = 1%).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "select.cuh"

namespace micro {

// Streaming configuration: warps per CTA, ring stages per warp, bytes per
// unit (per operand).  Shared memory = WARPS * STAGES * 2 * UNIT_BYTES.
// TMA = false: the warps load straight from HBM with 16-byte LDGs instead of
// bulk copies (no ring); MINB CTAs per SM are then resident.
template <int WARPS_, int STAGES_, int UNIT_BYTES_, bool TMA_ = true, int MINB_ = 1>
struct WsCfg {
  static constexpr int WARPS = WARPS_;
  static constexpr int STAGES = STAGES_;
  static constexpr int UNIT_BYTES = UNIT_BYTES_;
  static constexpr bool TMA = TMA_;
  static constexpr int MINB = MINB_;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int SMEM = TMA ? WARPS * STAGES * 2 * UNIT_BYTES + WARPS * STAGES * 8 + 128 : 0;
};

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
  int32_t* stage_idx;          // staging, (unit_hi - unit_lo + 1) * UNIT pairs (unit-local runs)
  void* stage_val;
  int* unit_counts;            // selections per partition unit
  unsigned long long* status;  // >= status_len words
  int64_t status_len;
  unsigned int epoch;
  int* flags;
  int64_t num_units;
  int64_t unit_lo, unit_hi;    // units intersecting [p_start, p_end)
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
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ float nan_probe(float g, float acc) { return __fmaf_rn(g, 0.0f, acc); }
__device__ __forceinline__ double nan_probe(double g, double acc) { return __fma_rn(g, 0.0, acc); }

// Work plan.  CTA b owns a contiguous, balanced slice of the partition's
// units and a slice of the remaining units; inside the slice its warps take
// units round-robin (warp w: units w, w+W, w+2W, ...), so a CTA streams one
// contiguous window of HBM (DRAM-row friendly: a probe with per-warp
// contiguous ranges — 1184 scattered streams — capped at 3.5 TB/s, while
// the same arithmetic on one moving window reaches 6.6 TB/s).
struct WarpPlan {  // unit indices fit int32: n_g < 2^31 (checked on the host)
  int p_first, p_n;  // partition units p_first + k*W, k < p_n
  int o_first, o_n;  // outside-list indices o_first + k*W, k < o_n
  int gap_lo, gap_n;
  int W;
  __device__ __forceinline__ int count() const { return p_n + o_n; }
  __device__ __forceinline__ int unit(int k) const {
    if (k < p_n) return p_first + k * W;
    const int q = o_first + (k - p_n) * W;
    return q < gap_lo ? q : q + gap_n;
  }
};

template <typename T, int kMode, class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB) k1_tma_select(TmaSelectArgs a) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  constexpr int kWsWarps = Cfg::WARPS, kWsStages = Cfg::STAGES, kWsUnitBytes = Cfg::UNIT_BYTES;
  constexpr int UE = kWsUnitBytes / (int)sizeof(T);
  constexpr int VPL = UE / VN / 32;  // vectors per lane per operand per unit (4)
  static_assert(VPL * VN * 32 == UE, "unit/lanes mismatch");
  static_assert(VPL <= 4, "packed 8-bit counts hold 4 vectors");

  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ long long s_run[kWsWarps];
  __shared__ long long s_excl;
  __shared__ int s_wsum[kWsWarps];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int b = blockIdx.x, G = gridDim.x;

  // per-warp ring: [stage][e | g][UE]
  T* ring = reinterpret_cast<T*>(smem + (size_t)w * kWsStages * 2 * kWsUnitBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kWsWarps * kWsStages * 2 * kWsUnitBytes) +
                   w * kWsStages;

  WarpPlan pl;
  int cta_p0, cta_p1;  // this CTA's partition units [cta_p0, cta_p1)
  {
    const int64_t P = a.unit_hi - a.unit_lo + 1, O = a.num_units - P;
    cta_p0 = (int)(a.unit_lo + P * b / G);
    cta_p1 = (int)(a.unit_lo + P * (b + 1) / G);
    const int o0 = (int)(O * b / G), o1 = (int)(O * (b + 1) / G);
    pl.W = kWsWarps;
    pl.p_first = cta_p0 + w;
    pl.p_n = pl.p_first < cta_p1 ? (cta_p1 - pl.p_first + kWsWarps - 1) / kWsWarps : 0;
    pl.o_first = o0 + w;
    pl.o_n = pl.o_first < o1 ? (o1 - pl.o_first + kWsWarps - 1) / kWsWarps : 0;
    pl.gap_lo = (int)a.unit_lo;
    pl.gap_n = (int)P;
  }
  const int nk = pl.count();
  const int n_g = (int)a.n_g;
  const int p_start = (int)a.p_start, p_end = (int)a.p_end;
  const T* __restrict__ Gp = (const T*)a.grad;
  T* __restrict__ E = (T*)a.resid;

  if (Cfg::TMA && lane == 0) {
    for (int s = 0; s < kWsStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  auto issue = [&](int k) {  // lane 0 only
    const int s = k % kWsStages;
    const int base = pl.unit(k) * UE;
    const int elems = n_g - base < UE ? n_g - base : UE;
    const uint32_t bytes = (uint32_t)(elems * (int)sizeof(T)) & ~15u;
    mbar_arrive_expect_tx(&full[s], 2 * bytes);
    if (bytes) {
      bulk_g2s(ring + (size_t)(2 * s) * UE, E + base, bytes, &full[s]);
      bulk_g2s(ring + (size_t)(2 * s + 1) * UE, Gp + base, bytes, &full[s]);
    }
  };
  if (Cfg::TMA && lane == 0)
    for (int k = 0; k < nk && k < kWsStages; ++k) issue(k);

  const double delta = *a.delta;
  const T thr = threshold_as(delta, (T*)nullptr);
  const T eta = (T)a.eta;
  int32_t* __restrict__ st_idx = a.stage_idx;
  T* __restrict__ st_val = (T*)a.stage_val;
  int* __restrict__ ucount = a.unit_counts;
  const int unit_lo = (int)a.unit_lo;
  long long run = 0;  // pairs selected by this warp
  T probe = (T)0;  // becomes NaN iff some G is Inf/NaN

  // One unit: wait, read the stage, refill it, accumulate, store e_{t+1},
  // and (partition units) compact the selections into the warp's run.
  // FULL: a whole unit (every unit but the vector's last) — no bounds tests;
  // SEL: a partition unit; CHECK: per-element partition-range test (the two
  // boundary units of the partition only).
  auto body = [&](int k, int base, int elems, auto kFull, auto kSel, auto kCheck) {
    constexpr bool FULL = decltype(kFull)::value;
    constexpr bool SEL = decltype(kSel)::value;
    constexpr bool CHECK = decltype(kCheck)::value;
    const int s = k % kWsStages;
    const int vec_elems = FULL ? UE : (int)((elems * (int)sizeof(T)) & ~15) / (int)sizeof(T);
    if constexpr (Cfg::TMA) mbar_wait(&full[s], (uint32_t)(k / kWsStages) & 1u);
    [[maybe_unused]] const V* se = reinterpret_cast<const V*>(ring + (size_t)(2 * s) * UE);
    [[maybe_unused]] const V* sg = reinterpret_cast<const V*>(ring + (size_t)(2 * s + 1) * UE);
    V e[VPL], g[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int off = (i * 32 + lane) * VN;
      if (FULL || off + VN <= vec_elems) {
        if constexpr (Cfg::TMA) {
          e[i] = se[i * 32 + lane];
          g[i] = sg[i * 32 + lane];
        } else {
          e[i] = ld_stream(reinterpret_cast<const V*>(E + base + off));
          g[i] = ld_nc_stream(reinterpret_cast<const V*>(Gp + base + off));
        }
      } else {  // the last unit's tail: straight from global
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          const bool in = off + c < elems;
          set_comp(e[i], c, in ? E[base + off + c] : (T)0);
          set_comp(g[i], c, in ? Gp[base + off + c] : (T)0);
        }
      }
    }
    if constexpr (Cfg::TMA) {
      __syncwarp();
      if (lane == 0 && k + kWsStages < nk) {
        fence_proxy_async_smem();  // our generic reads of stage s precede the async refill
        issue(k + kWsStages);
      }
    }
    unsigned mask[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      mask[i] = 0;
      const int off = (i * 32 + lane) * VN;
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const T gv = comp(g[i], c);
        probe = nan_probe(gv, probe);
        const T acc = add_rn(comp(e[i], c), mul_rn(eta, gv));  // two roundings, no FMA
        set_comp(e[i], c, acc);
        if (SEL) {
          bool sel = absx(acc) > thr;
          if (CHECK) {
            const int j = base + off + c;
            sel = sel && j >= p_start && j < p_end;
          }
          mask[i] |= (unsigned)sel << c;
        }
      }
    }
    if (kMode != kWriteNone) {
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int off = (i * 32 + lane) * VN;
        V out = e[i];
        if (kMode == kWriteZeroSel && SEL) {
#pragma unroll
          for (int c = 0; c < VN; ++c)
            if (mask[i] & (1u << c)) set_comp(out, c, (T)0);
        }
        if (FULL || off + VN <= elems) {
          st_stream(reinterpret_cast<V*>(E + base + off), out);
        } else {
#pragma unroll
          for (int c = 0; c < VN; ++c)
            if (off + c < elems) E[base + off + c] = comp(out, c);
        }
      }
    }
    if (SEL) {
      // order inside a unit: (vector i, lane, component c); per-lane counts of
      // the VPL vectors packed as 8-bit fields (warp totals <= 128)
      unsigned packed = 0;
#pragma unroll
      for (int i = 0; i < VPL; ++i) packed |= (unsigned)__popc(mask[i]) << (8 * i);
      unsigned incl = packed;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
      // pairs of unit u are staged at [(u - unit_lo) * UE, + count)
      const long long run_base = (long long)(base / UE - unit_lo) * UE;
      unsigned unit_count = 0;
#pragma unroll
      for (int i = 0; i < VPL; ++i) unit_count += (tot >> (8 * i)) & 0xFFu;
      if (lane == 0) ucount[base / UE - unit_lo] = (int)unit_count;
      if (tot) {
        const unsigned excl = incl - packed;
        unsigned any = 0;
#pragma unroll
        for (int i = 0; i < VPL; ++i) any |= mask[i];
        if (any) {
        unsigned cb = 0;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (mask[i]) {
            long long pos = run_base + cb + ((excl >> (8 * i)) & 0xFFu);
            const int j0 = base + (i * 32 + lane) * VN;
#pragma unroll
            for (int c = 0; c < VN; ++c)
              if (mask[i] & (1u << c)) {
                st_idx[pos] = j0 + c;
                st_val[pos] = comp(e[i], c);
                ++pos;
              }
          }
          cb += (tot >> (8 * i)) & 0xFFu;
        }
        }
        run += unit_count;
      }
    }
  };
  using TT = std::true_type;
  using FF = std::false_type;
  auto process = [&](int k, bool in_partition) {
    const int base = pl.unit(k) * UE;
    const int elems = n_g - base < UE ? n_g - base : UE;
    const bool full_unit = elems == UE;
    if (in_partition) {
      const bool all_in = base >= p_start && base + elems <= p_end;
      if (full_unit && all_in) body(k, base, elems, TT{}, TT{}, FF{});
      else body(k, base, elems, FF{}, TT{}, TT{});
    } else {
      if (full_unit) body(k, base, elems, TT{}, FF{}, FF{});
      else body(k, base, elems, FF{}, FF{}, FF{});
    }
  };

  int k = 0;
  for (; k < pl.p_n; ++k) process(k, true);

  // ---- partition slices done: CTA offset by one look-back, runs into place ----
  if (lane == 0) s_run[w] = run;
  __syncthreads();
  if (w == 0) {
    long long cta = 0;
#pragma unroll
    for (int q = 0; q < kWsWarps; ++q) cta += s_run[q];
    const long long ex = lookback(a.status, b, (unsigned long long)cta, a.epoch, lane);
    if (lane == 0) {
      s_excl = ex;
      if (b == G - 1) {
        const long long total = ex + cta;
        *a.count = total;
        if (total > a.cap) atomicOr(a.flags, 2);
      }
    }
    if (b == G - 1) {  // stamp the unused look-back words with this epoch
      const unsigned long long ep = (unsigned long long)(a.epoch & 0xFFFFFFu) << 40;
      for (int64_t q = G + lane; q < a.status_len; q += 32) st_relaxed_u64(&a.status[q], ep);
    }
  }
  __syncthreads();
  {
    // copy the staged unit runs into place, in unit order: block-wide scan
    // of the per-unit counts, THREADS units at a time
    long long off = s_excl;
    int32_t* __restrict__ out_idx = a.sel_idx;
    T* __restrict__ out_val = (T*)a.sel_val;
    for (int u0 = cta_p0; u0 < cta_p1; u0 += Cfg::THREADS) {
      const int u = u0 + tid;
      const int cnt = u < cta_p1 ? ucount[u - unit_lo] : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wsum[w] = incl;
      __syncthreads();
      int wpre = 0, tot = 0;
#pragma unroll
      for (int q = 0; q < kWsWarps; ++q) {
        const int x = s_wsum[q];
        wpre += q < w ? x : 0;
        tot += x;
      }
      const long long dst = off + wpre + incl - cnt;
      const long long src = (long long)(u - unit_lo) * UE;
      for (int m = 0; m < cnt; ++m) {
        const long long d = dst + m;
        if (d < a.cap) {
          out_idx[d] = st_idx[src + m];
          out_val[d] = st_val[src + m];
        }
      }
      off += tot;
      __syncthreads();
    }
  }

  for (; k < nk; ++k) process(k, false);

  if (probe != probe) atomicOr(a.flags, 1);
}

}  // namespace micro
