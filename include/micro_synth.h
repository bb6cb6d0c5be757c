/*
 * micro_synth.h — the synthetic-gradient specification shared by the device
 * generator (paper_2310_00967_b200/csrc/synth.cu) and the CPU checker
 * (oracle/micro_oracle.c).
 *
 * SURVEY.md §8(d) "Identical inputs on host and device": G_{i,t}[j] ~ N(0,1)
 * drawn from a counter-based Philox4x32-10 stream keyed by (seed, worker) and
 * indexed by (t, j), turned into normals by a Box-Muller transform whose log,
 * sqrt and sin/cos are built from IEEE-rounded +, -, *, / and sqrt only.  Every
 * operation is spelled with the MS_F* macros below, which map to the
 * explicitly rounded __f*_rn intrinsics on the device (never contracted into
 * FMA) and to plain operators on the host (compiled with -ffp-contract=off),
 * so host and device produce bit-identical gradients.
 *
 * This is a data-generation spec, not a path under test: the reference
 * (sparsim) has its own gradient producers (proj/src/task.cpp), which are out
 * of scope, and BASELINE.json asks for synthetic Gaussians.
 */
#ifndef MICRO_SYNTH_H
#define MICRO_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define MS_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define MS_FADD(a, b) __fadd_rn((a), (b))
#define MS_FSUB(a, b) __fsub_rn((a), (b))
#define MS_FMUL(a, b) __fmul_rn((a), (b))
#define MS_FDIV(a, b) __fdiv_rn((a), (b))
#define MS_FSQRT(a) __fsqrt_rn(a)
#define MS_AS_UINT(x) __float_as_uint(x)
#define MS_AS_FLOAT(x) __uint_as_float(x)
#else
#define MS_FADD(a, b) ((a) + (b))
#define MS_FSUB(a, b) ((a) - (b))
#define MS_FMUL(a, b) ((a) * (b))
#define MS_FDIV(a, b) ((a) / (b))
#define MS_FSQRT(a) ms_host_sqrtf(a)
#define MS_AS_UINT(x) ms_host_as_uint(x)
#define MS_AS_FLOAT(x) ms_host_as_float(x)
#endif
#else
#define MS_HD static inline
#define MS_FADD(a, b) ((a) + (b))
#define MS_FSUB(a, b) ((a) - (b))
#define MS_FMUL(a, b) ((a) * (b))
#define MS_FDIV(a, b) ((a) / (b))
#define MS_FSQRT(a) ms_host_sqrtf(a)
#define MS_AS_UINT(x) ms_host_as_uint(x)
#define MS_AS_FLOAT(x) ms_host_as_float(x)
#endif

#if !defined(__CUDA_ARCH__)
#include <math.h>
#include <string.h>
static inline float ms_host_sqrtf(float x) { return sqrtf(x); } /* IEEE sqrtss */
static inline uint32_t ms_host_as_uint(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static inline float ms_host_as_float(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }
#endif

/* Philox4x32-10 (Salmon et al., SC'11): integer-only, so identical everywhere. */
MS_HD void ms_philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                            uint32_t k0, uint32_t k1, uint32_t out[4]) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 24-bit uniform in (0,1): ((x >> 8) + 0.5) * 2^-24, exact in fp32. */
MS_HD float ms_uniform(uint32_t x) {
  return MS_FMUL((float)(x >> 8) + 0.5f, 5.9604644775390625e-08f);
}

/* ln(u) for u in (0,1): u = m * 2^e, m in [sqrt(.5), sqrt(2)), atanh series. */
MS_HD float ms_log(float u) {
  uint32_t bits = MS_AS_UINT(u);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float m = MS_AS_FLOAT((bits & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) { m = MS_FMUL(m, 0.5f); e += 1; }
  const float f = MS_FSUB(m, 1.0f);
  const float s = MS_FDIV(f, MS_FADD(2.0f, f));
  const float s2 = MS_FMUL(s, s);
  float p = MS_FMUL(s2, 0.22222222f);
  p = MS_FMUL(s2, MS_FADD(0.28571429f, p));
  p = MS_FMUL(s2, MS_FADD(0.4f, p));
  p = MS_FMUL(s2, MS_FADD(0.66666667f, p));
  const float logm = MS_FMUL(s, MS_FADD(2.0f, p));
  return MS_FADD(MS_FMUL((float)e, 0.69314718f), logm);
}

/* sin and cos of x in [0, pi/2) by Taylor polynomials (error < 1e-7). */
MS_HD void ms_sincos_quarter(float x, float* s, float* c) {
  const float x2 = MS_FMUL(x, x);
  float ps = MS_FMUL(x2, -2.5052108e-08f);
  ps = MS_FMUL(x2, MS_FADD(2.7557319e-06f, ps));
  ps = MS_FMUL(x2, MS_FADD(-1.9841270e-04f, ps));
  ps = MS_FMUL(x2, MS_FADD(8.3333333e-03f, ps));
  ps = MS_FMUL(x2, MS_FADD(-1.6666667e-01f, ps));
  *s = MS_FMUL(x, MS_FADD(1.0f, ps));
  float pc = MS_FMUL(x2, 2.0876757e-09f);
  pc = MS_FMUL(x2, MS_FADD(-2.7557319e-07f, pc));
  pc = MS_FMUL(x2, MS_FADD(2.4801587e-05f, pc));
  pc = MS_FMUL(x2, MS_FADD(-1.3888889e-03f, pc));
  pc = MS_FMUL(x2, MS_FADD(4.1666667e-02f, pc));
  pc = MS_FMUL(x2, MS_FADD(-0.5f, pc));
  *c = MS_FADD(1.0f, pc);
}

/* Box-Muller: (u1, u2) -> two N(0,1) samples. */
MS_HD void ms_box_muller(float u1, float u2, float* z0, float* z1) {
  const float r = MS_FSQRT(MS_FMUL(-2.0f, ms_log(u1)));
  const float v = MS_FMUL(u2, 4.0f);
  const int q = (int)v;
  const float x = MS_FMUL(MS_FSUB(v, (float)q), 1.57079637f);
  float s, c;
  ms_sincos_quarter(x, &s, &c);
  float sn, cs;
  switch (q & 3) {
    case 0: sn = s; cs = c; break;
    case 1: sn = c; cs = -s; break;
    case 2: sn = -s; cs = -c; break;
    default: sn = -c; cs = s; break;
  }
  *z0 = MS_FMUL(r, cs);
  *z1 = MS_FMUL(r, sn);
}

/* Four consecutive gradient entries G[4q .. 4q+3] of worker `worker` at
 * iteration t, run seed `seed`. */
MS_HD void ms_gaussian4(uint64_t seed, uint32_t worker, uint64_t t, uint64_t q, float out[4]) {
  uint32_t x[4];
  ms_philox4x32_10((uint32_t)q, (uint32_t)(q >> 32), (uint32_t)t, (uint32_t)(t >> 32),
                   (uint32_t)seed, (uint32_t)(seed >> 32) ^ (worker * 0x85EBCA6Bu + 0x1B873593u), x);
  ms_box_muller(ms_uniform(x[0]), ms_uniform(x[1]), &out[0], &out[1]);
  ms_box_muller(ms_uniform(x[2]), ms_uniform(x[3]), &out[2], &out[3]);
}

#endif /* MICRO_SYNTH_H */
