// select_stream.cuh — K1 as two kernels: an unordered streaming pass and a
// small ordered compaction.
//
// Reference semantics (paths relative to /root/reference/proj):
//   acc_i = e_i + eta * G_i over ALL n_g            harness.cpp:131 (P4)
//   non-finite G  -> runtime_error                  harness.cpp:128-130
//   S_i = { j in partition : |acc_i[j]| > delta_i } sparsifier.cpp:22-37,
//         ascending, strict, (index, acc value)     tensor.hpp:48-63
//   e_{i,t+1}[j] = 0 for j in S_i (own part of the union zeroing)
//                                                   harness.cpp:219-221
// The same two kernels serve the value-level select_by_threshold /
// select_topk (acc only: kNoG, kWriteNone) over a range.
//
// K1a  k1_stream: one warp per 512-element unit (2 KB per operand), eight
//      units per CTA, ~32 warps resident per SM.  Each lane issues its eight
//      16-byte loads (e, G) up front, computes acc = e + eta*G with explicitly
//      rounded arithmetic, stores e_{t+1} (selected entries zeroed), and — for
//      units that intersect the partition — compacts the selected
//      (index, value) pairs with one packed warp scan into the unit's own
//      staging slot [(u - u_lo) * 512, + k_u), recording k_u.  No ordering,
//      no cross-warp or cross-CTA dependency: the pass runs at the HBM
//      roofline like a plain axpy (tools/k1_probe.cu: 6.2-7.0 TB/s).
//      Each CTA's run count is also added (one atomic) into its "super
//      block" of S consecutive runs (<= 1024 super blocks).
// K1b  k1_gather: one warp per run copies it, coalesced, to its final
//      position, giving the ascending (index, value) list.  A CTA's output
//      offset is the sum of the super blocks before its own plus the runs
//      before it inside its super block (<= 1024 + S L2 reads per CTA, no
//      scan kernel, no look-back); block 0 also forms k_i.
//
// Why not one pass: every single-pass variant we measured in round 1
// (per-tile decoupled look-back; persistent CTAs with TMA bulk-copy rings;
// per-warp rings; LDG streaming with per-warp ordered runs) stayed at
// 2.5-3.6 TB/s — the ordering machinery sat on the critical path of every
// tile (profiles/README.md, round 1).  The staging
// round trip costs 16 bytes per selected pair plus 4 bytes per 512
// elements (0.2 B/elem at d = 1%, vs 12 B/elem streamed).
#pragma once

#include "common.cuh"
#include "norm.cuh"

namespace micro {

enum WriteMode : int {
  kWriteZeroSel = 0,  // e <- acc with own selections zeroed (error feedback on)
  kWriteAcc = 1,      // e <- acc (error feedback off, n > 1: peers still read acc)
  kWriteNone = 2,     // no residual write (EF off at n = 1, or select-only)
};

constexpr int kStreamWarps = 8;                  // units per CTA
constexpr int kStreamThreads = kStreamWarps * 32;
constexpr int kStreamUnitBytes = 2048;            // per operand
// dense g/n write granularity: a chunk of kDenseLanes lanes (16 B each) is
// rewritten whole when any of its entries is (or was) selected
#ifndef MICRO_DENSE_LANES
#define MICRO_DENSE_LANES 2
#endif
constexpr int kDenseLanes = MICRO_DENSE_LANES;


template <typename T>
__host__ __device__ constexpr int stream_unit_elems() {
  return kStreamUnitBytes / (int)sizeof(T);  // 512 fp32 / 256 fp64
}

struct StreamArgs {
  const void* grad;
  void* resid;
  int n_g;                 // < 2^31 (checked on the host)
  int p_start, p_end;
  double eta;
  const double* delta;
  int unit_lo, unit_hi;    // units intersecting [p_start, p_end)
  int32_t* stage_idx;      // (unit_hi - unit_lo + 1) * UNIT pairs
  void* stage_val;
  int* unit_counts;        // unit_hi - unit_lo + 1
  int* flags;              // bit0 non-finite
  // single-worker dense g/n, fused (kDense): whole 32-byte sectors, one
  // "nonzero last step" bit per sector (64 per unit)
  void* dense;
  unsigned long long* dirty;
  int* super_counts;       // selections per super block of `super_runs` CTA runs (zeroed)
  int super_runs;
  double* sq_part;         // kNorm: per CTA, sum of e_{t+1}^2 (own selections zeroed); reduced by k1_gather
  const long long* tie_j;  // kTie (top-k baseline): also select |acc| == thr at j <= *tie_j
  int cta_offset;          // this launch covers CTAs [cta_offset, cta_offset + gridDim.x) (chunked H2D)
  const void* model;       // kPf: the model x whose selected lines k1_gather will read-modify-write
};

// L2 prefetch with the evict-last priority: the line survives the rest of
// the (evict-first) stream and k1_gather's read of it hits L2.
__device__ __forceinline__ void prefetch_l2_keep(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

__device__ __forceinline__ float nan_probe_s(float g, float acc) { return __fmaf_rn(g, 0.0f, acc); }
__device__ __forceinline__ double nan_probe_s(double g, double acc) { return __fma_rn(g, 0.0, acc); }

// Compress the 32 lane bits of a sector ballot (lanes 2k, 2k+1 share
// sector k) into 16 sector bits.
__device__ __forceinline__ unsigned even_bits(unsigned x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  x = (x | (x >> 8)) & 0x0000FFFFu;
  return x;
}

__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// kNoG (top-k baseline): e already holds acc (written by the first histogram
// pass), G is not read.
// kPf (small steps, n = 1 with the model update): the lines of x at this
// unit's selections are prefetched into L2 while the stream runs, taking the
// model's DRAM latency off k1_gather's critical path.
// TG: the gradient's element type.  TG = float with T = double: fp32
// gradients (BASELINE's "fp32 gradient") into the reference's fp64 state and
// arithmetic — (double)g is exact, so acc = e + eta*(double)g rounds exactly
// as the reference's e + eta*G on the same gradient values; G moves 4 B per
// element instead of 8.
template <typename T, int kMode, bool kDense, bool kNorm, bool kTie = false, bool kNoG = false, bool kPf = false,
          typename TG = T>
__global__ void __launch_bounds__(kStreamThreads, kNoG ? 5 : 4) k1_stream(StreamArgs a) {  // acc-only: 51 regs, 5 CTAs/SM
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  constexpr int UE = stream_unit_elems<T>();
  constexpr int VPL = UE / VN / 32;  // 4 vectors per lane per operand
  static_assert(VPL * VN * 32 == UE && VPL <= 4, "unit layout");

  __shared__ int s_cnt[kStreamWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int bx = (int)blockIdx.x + a.cta_offset;
  const int u = bx * kStreamWarps + w;
  pdl_wait();  // the previous step's gather / finalize (staging, counts, delta) is done
  const int base = u * UE;
  // warps past the vector's end idle but still meet the CTA barrier below
  const int elems = base >= a.n_g ? 0 : (a.n_g - base < UE ? a.n_g - base : UE);
  const bool live = elems > 0;
  const TG* __restrict__ Gp = (const TG*)a.grad + base;
  T* __restrict__ E = (T*)a.resid + base;

  const unsigned long long pol_stream = policy_evict_first();
  // kDense: last step's sector bits, loaded with e and G so the latency overlaps
  const unsigned long long dirty_prev = (kDense && live) ? a.dirty[u] : 0ull;
  V e[VPL], g[VPL];
  if (elems == UE) {  // (elems == 0 for dead warps: the guarded path below loads nothing)
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      e[i] = ld_hint(reinterpret_cast<const V*>(E) + i * 32 + lane, pol_stream);
      if (!kNoG) g[i] = ld_grad<V>(reinterpret_cast<const typename GradVec<TG, VN>::V*>(Gp) + i * 32 + lane, pol_stream);
    }
  } else {  // the vector's last, partial unit
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const int off = (i * 32 + lane) * VN + c;
        set_comp(e[i], c, off < elems ? E[off] : (T)0);
        set_comp(g[i], c, (!kNoG && off < elems) ? (T)Gp[off] : (T)0);
      }
  }

  const bool sel_unit = live && u >= a.unit_lo && u <= a.unit_hi;
  // (padding lanes of the last partial unit take the ranged path: a threshold < 0
  // would otherwise select their zeros)
  const bool all_in = base >= a.p_start && base + UE <= a.p_end;
  const T thr = threshold_as(*a.delta, (T*)nullptr);
  const long long tie_limit = kTie ? *a.tie_j : 0;
  const T eta = (T)a.eta;
  T probe = (T)0;  // becomes NaN iff some G is Inf/NaN
  // bit i * VN + c: element (vector i, lane, component c) is selected
  unsigned bits = 0;
  bool tie_seen = false;
  V out[VPL];  // e_{t+1} as stored (own selections zeroed when EF is on)
  // one element: acc, the compare, the stored value.  `ranged`: the unit
  // straddles the partition's ends (or is the vector's partial last unit).
  auto element = [&](int i, int c, bool ranged) {
    T acc;
    if (kNoG) {
      acc = comp(e[i], c);
    } else {
      const T gv = comp(g[i], c);
      probe = nan_probe_s(gv, probe);
      acc = add_rn(comp(e[i], c), mul_rn(eta, gv));  // two roundings, no FMA
    }
    set_comp(e[i], c, acc);
    bool sel = absx(acc) > thr;
    if (kTie) tie_seen |= absx(acc) == thr;
    if (ranged) {
      const int j = base + (i * 32 + lane) * VN + c;
      sel = sel && j >= a.p_start && j < a.p_end;
    }
    if (sel) bits |= 1u << (i * VN + c);
    set_comp(out[i], c, (kMode == kWriteZeroSel && sel) ? (T)0 : acc);
  };
  // warp-uniform branches: the common case (every element of the unit in the
  // partition) carries no index arithmetic
  if (sel_unit && all_in) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) element(i, c, false);
  } else if (sel_unit) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) element(i, c, true);
  } else {  // outside the partition: accumulate only
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        T acc;
        if (kNoG) {
          acc = comp(e[i], c);
        } else {
          const T gv = comp(g[i], c);
          probe = nan_probe_s(gv, probe);
          acc = add_rn(comp(e[i], c), mul_rn(eta, gv));
        }
        set_comp(e[i], c, acc);
        set_comp(out[i], c, acc);
      }
  }
  // top-k: ties at the pivot are selected up to index J.  They are rare, so
  // the index comparisons run only in the warps that hold one.
  if (kTie && __any_sync(0xffffffffu, tie_seen)) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const int j = base + (i * 32 + lane) * VN + c;
        const bool tie = sel_unit && absx(comp(e[i], c)) == thr && (long long)j <= tie_limit &&
                         (all_in || (j >= a.p_start && j < a.p_end));
        if (tie) {
          bits |= 1u << (i * VN + c);
          if (kMode == kWriteZeroSel) set_comp(out[i], c, (T)0);  // top-k at n = 1: ties are zeroed too
        }
      }
  }
  constexpr unsigned VMASK = (1u << VN) - 1u;

  if (kPf) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if ((bits >> (i * VN)) & VMASK) prefetch_l2_keep((const T*)a.model + base + (i * 32 + lane) * VN);
  }
  if (kMode != kWriteNone) {
    if (kNoG && kMode == kWriteZeroSel && elems == UE) {
      // e already holds acc (top-k, one worker): only the 32-byte sectors
      // holding a selection change; lanes 2k and 2k+1 share sector k
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const bool sec = ((bits >> (i * VN)) & VMASK) != 0;
        const bool peer = __shfl_xor_sync(0xffffffffu, sec, 1);
        if (sec || peer) st_hint(reinterpret_cast<V*>(E) + i * 32 + lane, out[i], pol_stream);
      }
    } else if (elems == UE) {
#pragma unroll
      for (int i = 0; i < VPL; ++i) st_hint(reinterpret_cast<V*>(E) + i * 32 + lane, out[i], pol_stream);
    } else {
#pragma unroll
      for (int i = 0; i < VPL; ++i)
#pragma unroll
        for (int c = 0; c < VN; ++c) {
          const int off = (i * 32 + lane) * VN + c;
          if (off < elems) E[off] = comp(out[i], c);
        }
    }
  }

  // kNorm: this lane's part of ||e_{t+1}||^2 (the stored values; zeros add nothing)
  double sq = 0.0;
  if (kNorm) {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
#pragma unroll
      for (int c = 0; c < VN; ++c) {
        const double y = (double)comp(out[i], c);
        sq += y * y;
      }
  }

  if (kDense && live) {  // live is warp-uniform: the shuffles below see every lane
    // n = 1: g/n = (0 + acc) / 1 = acc at the selections (never +-0: |acc| >
    // delta >= 0), 0 elsewhere.  A 32-byte sector is written in full when it
    // holds a selection now or held one last step; lanes 2k and 2k+1 own its
    // two 16-byte halves (sector k + 16 i of the unit).
    static_assert(VPL * 16 == 64, "64 sectors per unit");
    const unsigned long long prev = dirty_prev;
    unsigned long long now = 0;
    T* D = (T*)a.dense + base;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const unsigned m = (bits >> (i * VN)) & VMASK;
      bool sec = m != 0;  // the lanes of one kDenseLanes * 16-byte chunk agree (every lane shuffles)
#pragma unroll
      for (int o = 1; o < kDenseLanes; o <<= 1) {
        const bool peer = __shfl_xor_sync(0xffffffffu, sec, o);  // unconditional: no short-circuit
        sec = sec || peer;
      }
      const unsigned secbits = even_bits(__ballot_sync(0xffffffffu, sec));
      now |= (unsigned long long)secbits << (16 * i);
      if (sec || ((prev >> (16 * i + (lane >> 1))) & 1ull)) {
        V dv;
#pragma unroll
        // (0 + acc: the reference's sum from +0, so a selected -0 (top-k) is +0)
        for (int c = 0; c < VN; ++c) set_comp(dv, c, (m & (1u << c)) ? add_rn((T)0, comp(e[i], c)) : (T)0);
        if (elems == UE) {
          st_hint(reinterpret_cast<V*>(D) + i * 32 + lane, dv, pol_stream);
        } else {
#pragma unroll
          for (int c = 0; c < VN; ++c) {
            const int off = (i * 32 + lane) * VN + c;
            if (off < elems) D[off] = comp(dv, c);
          }
        }
      }
    }
    if (lane == 0 && now != prev) a.dirty[u] = now;
  }

  // ---- ordered compaction of the CTA's 8 units into one contiguous run ----
  // order inside a unit: (vector i, lane, component c); the VPL per-lane
  // counts are packed as 8-bit fields (warp totals <= 128); units in warp
  // order inside the CTA.  Runs live at staging slot (CTA - cta_lo) * 8 * UE.
  const int cta_lo = a.unit_lo / kStreamWarps, cta_hi = a.unit_hi / kStreamWarps;
  const bool sel_cta = bx >= cta_lo && bx <= cta_hi;  // CTA-uniform
  if (sel_cta) {
    unsigned packed = 0;
#pragma unroll
    for (int i = 0; i < VPL; ++i) packed |= (unsigned)__popc((bits >> (i * VN)) & VMASK) << (8 * i);  // 0 unless sel_unit
    unsigned incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    const unsigned excl = incl - packed;
    // first position of this lane's pairs of vector i: the warp's pairs of
    // vectors < i + this vector's pairs in lanes < this one (sums reach 512:
    // not packable in bytes)
    int first[VPL];
    int unit_count = 0;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      first[i] = unit_count + (int)((excl >> (8 * i)) & 0xFFu);
      unit_count += (int)((tot >> (8 * i)) & 0xFFu);
    }
    if (lane == 0) s_cnt[w] = unit_count;
    __syncthreads();
    int woff = 0, cta_count = 0;
#pragma unroll
    for (int q = 0; q < kStreamWarps; ++q) {
      const int x = s_cnt[q];
      woff += q < w ? x : 0;
      cta_count += x;
    }
    const int slot = bx - cta_lo;
    if (threadIdx.x == 0) {
      a.unit_counts[slot] = cta_count;
      if (cta_count) atomicAdd(a.super_counts + slot / a.super_runs, cta_count);
    }
    if (unit_count) {
      const unsigned long long pol_keep = policy_evict_last();  // read back by k1_gather, then discarded
      int32_t* __restrict__ si = a.stage_idx + (long long)slot * (kStreamWarps * UE) + woff;
      T* __restrict__ sv = (T*)a.stage_val + (long long)slot * (kStreamWarps * UE) + woff;
      // one iteration per selected component (a warp runs its lanes' maximum)
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        unsigned m = (bits >> (i * VN)) & VMASK;
        int pos = first[i];
        const int j0 = base + (i * 32 + lane) * VN;
        while (m) {
          const int c = __ffs(m) - 1;
          m &= m - 1;
          st_hint(si + pos, j0 + c, pol_keep);
          st_hint(sv + pos, comp(e[i], c), pol_keep);
          ++pos;
        }
      }
    }
  }
  if (probe != probe) atomicOr(a.flags, 1);
  pdl_trigger();  // this CTA's results are written: k1_gather may start launching
  if (kNorm) {  // the stored e_{t+1}: acc with the own selections zeroed (EF on)
    // CTA partial only: no fence, no ticket on the streaming pass (a
    // per-CTA release costs ~20 % of K1); k1_gather's extra CTA sums them
    __shared__ double s_sq[kStreamWarps];
    sq = warp_sum_f64(sq);
    if (lane == 0) s_sq[w] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < kStreamWarps; ++q) t += s_sq[q];
      a.sq_part[bx] = t;
    }
  }
}

struct CompactArgs {
  const int32_t* stage_idx;
  const void* stage_val;
  const int* run_counts;   // pairs per CTA run (k1_stream)
  const int* super_counts; // pairs per super block of `super_runs` runs (k1_stream)
  int* super_clear;        // the other parity's super counts: zeroed here for the next launch
  int super_len;           // entries of super_clear
  int num_runs;
  int super_runs;
  int run_stride;          // staging elements per run slot
  int32_t* sel_idx;
  void* sel_val;
  long long cap;
  long long* count;
  int* flags;              // bit1 capacity overflow
  void* model;             // n = 1: x -= g/n = acc at the selections (harness.cpp:212-215)
  // n = 1 single-call step (micro_step): block 0 also does what k_finalize
  // would — K, history, threshold update (sparsifier.cpp:77-81) — so the
  // iteration is two launches.  fin_delta == NULL: not fused.
  double* fin_delta;
  int sum_from_zero;       // the selection is the union (one worker): write 0 + v, the reference's sum
  int fin_fixed;           // the hard threshold (n = 1): record delta_0, never update it
  unsigned long long k_target;
  double alpha, min_threshold;
  long long* fin_K;
  long long fin_t, fin_slot;
  long long *hist_t, *hist_K, *hist_counts;
  double* hist_delta;
  double* hist_err;
  int norm_mode;           // as FinalizeArgs (no foreign entries at n = 1)
  // norm on: the grid's last CTA sums k1_stream's per-CTA partials in index
  // order into *sq_out (and, fused n = 1 step, hist_err[fin_slot])
  const double* sq_part;
  int sq_parts;
  double* sq_out;
};

__device__ __forceinline__ void gather_finalize(const CompactArgs& a, long long total) {
  const long long K = total < a.cap ? total : a.cap;
  *a.fin_K = K;
  a.hist_t[a.fin_slot] = a.fin_t;
  a.hist_K[a.fin_slot] = K;
  a.hist_counts[a.fin_slot] = total;
  double d = *a.fin_delta;
  a.hist_delta[a.fin_slot] = d;
  if (a.norm_mode != 1)  // mode 1: written by the reducing CTA
    a.hist_err[a.fin_slot] = a.norm_mode == 2 ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
  if (a.fin_fixed) return;
  const unsigned long long k = (unsigned long long)total;
  if (k > a.k_target) d = d == 0.0 ? a.min_threshold : d * (1.0 + a.alpha);
  else if (k < a.k_target) d *= 1.0 - a.alpha;
  *a.fin_delta = d;
}

constexpr int kGatherWarps = 8;   // runs per k1_gather CTA (divides super_runs)
constexpr int kMaxSupers = 1024;  // super blocks per launch

// CTA-wide sum of an int range [lo, hi) (256 threads).
__device__ __forceinline__ long long block_sum_range(const int* p, int lo, int hi, long long* s_part) {
  long long v = 0;
  for (int q = lo + (int)threadIdx.x; q < hi; q += kGatherWarps * 32) v += p[q];
  v = (long long)warp_sum_u64((unsigned long long)v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();  // s_part reuse
  if (lane == 0) s_part[w] = v;
  __syncthreads();
  long long t = 0;
#pragma unroll
  for (int q = 0; q < kGatherWarps; ++q) t += s_part[q];
  return t;
}

// One warp per CTA run: coalesced copy into the ordered output at the run's
// exclusive prefix, then the run's staging lines are dropped from L2 without
// write-back.  n = 1: the model update rides along.
// kWide: fetch the model's lines 64 B at a time (L2::64B: fewer DRAM
// transactions when the selections are sparse); dense selections (d >= 5 %)
// already touch most sectors, and plain sector loads move fewer bytes.
template <typename T, bool kWide = true>
__global__ void __launch_bounds__(kGatherWarps * 32) k1_gather(CompactArgs a) {
  __shared__ long long s_part[kGatherWarps];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  pdl_wait();  // k1_stream's runs and counts are complete and visible
  pdl_trigger();
  // norm on: CTA 0 (scheduled first, overlapping the copies) reduces
  // ||e_{t+1}||^2 in a fixed order; the copy CTAs are 1..
  if (a.sq_part && blockIdx.x == 0) {
    __shared__ double s_sq[kGatherWarps];
    double v = 0.0;
#pragma unroll 8
    for (int q = threadIdx.x; q < a.sq_parts; q += kGatherWarps * 32) v += a.sq_part[q];
    v = warp_sum_f64(v);
    if (lane == 0) s_sq[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < kGatherWarps; ++q) t += s_sq[q];
      *a.sq_out = t;
      if (a.fin_delta) a.hist_err[a.fin_slot] = sqrt(t);
    }
    return;
  }
  const int gb = (int)blockIdx.x - (a.sq_part ? 1 : 0);
  const int r0 = gb * kGatherWarps;
  const int sb = r0 / a.super_runs;
  const int r = r0 + w;
  // this CTA's run counts first (independent of the prefix below): one round
  // of L2 reads for everything the CTA needs
  const int mine = (r0 + lane < a.num_runs && lane < w) ? a.run_counts[r0 + lane] : 0;
  const int n = r < a.num_runs ? a.run_counts[r] : 0;
  // pairs before this CTA: super blocks [0, sb) + runs [sb * S, r0), summed in one pass
  long long base = 0;
  {
    const int nsup = sb, nrun = r0 - sb * a.super_runs;
    long long v = 0;
    for (int q = threadIdx.x; q < nsup + nrun; q += kGatherWarps * 32)
      v += q < nsup ? a.super_counts[q] : a.run_counts[sb * a.super_runs + (q - nsup)];
    v = (long long)warp_sum_u64((unsigned long long)v);
    if (lane == 0) s_part[w] = v;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kGatherWarps; ++q) base += s_part[q];
  }
  if (gb == 0) {
    const int nsup = (a.num_runs + a.super_runs - 1) / a.super_runs;
    const long long total = block_sum_range(a.super_counts, 0, nsup, s_part);
    if (threadIdx.x == 0) {
      *a.count = total;
      if (total > a.cap) atomicOr(a.flags, 2);
      if (a.fin_delta) gather_finalize(a, total);
    }
    for (int q = threadIdx.x; q < a.super_len; q += kGatherWarps * 32) a.super_clear[q] = 0;
  }
  // runs of this CTA before r (<= 7 L2 hits, loaded above)
  base += (long long)__reduce_add_sync(0xffffffffu, (unsigned)mine);
  if (r >= a.num_runs) return;
  if (!n) return;
  const long long off = base < a.cap ? base : a.cap;
  const long long src = (long long)r * a.run_stride;
  const int32_t* __restrict__ si = a.stage_idx + src;
  const T* __restrict__ sv = (const T*)a.stage_val + src;
  int32_t* __restrict__ oi = a.sel_idx + off;
  T* __restrict__ ov = (T*)a.sel_val + off;
  const long long room = a.cap - off;
  T* __restrict__ x = (T*)a.model;
  // kG entries per lane in flight: at high density a run holds hundreds of
  // pairs and the model's random read-modify-write is latency bound
  // (dense selections, !kWide: 8 in fp64 too — C5 d = 0.1 f64 10065 -> 9859
  // us/iter; 16 in fp32 was slower at 80 registers)
  constexpr int kG = kWide ? 32 / (int)sizeof(T) : 8;  // kWide: 8 fp32, 4 fp64 (registers: occupancy)
  const int lim = n < room ? n : (int)room;
  for (int m0 = lane; m0 < lim; m0 += 32 * kG) {
    int32_t j[kG];
    T v[kG], xv[kG];
#pragma unroll
    for (int q = 0; q < kG; ++q) {
      const int m = m0 + 32 * q;
      if (m < lim) {
        j[q] = si[m];
        v[q] = a.sum_from_zero ? add_rn((T)0, sv[m]) : sv[m];  // 0 + v = v, except a selected -0 (top-k) -> +0
        oi[m] = j[q];
        ov[m] = v[q];
      }
    }
    if (x) {  // n = 1: g/n = (0 + v) / 1
#pragma unroll
      for (int q = 0; q < kG; ++q)
        if (m0 + 32 * q < lim) xv[q] = kWide ? ld_rand(x + j[q]) : x[j[q]];
#pragma unroll
      for (int q = 0; q < kG; ++q)
        if (m0 + 32 * q < lim) x[j[q]] = xv[q] - v[q];
    }
  }
  __syncwarp();
  for (int o = lane * 128; o < n * 4; o += 32 * 128) discard_l2_line(reinterpret_cast<const char*>(si) + o);
  for (int o = lane * 128; o < n * (int)sizeof(T); o += 32 * 128)
    discard_l2_line(reinterpret_cast<const char*>(sv) + o);
}

}  // namespace micro
