// numpy's default_rng(seed) stream, bit for bit, on the device.
//
// The reference draws every arrival skeleton of the throughput simulator
// with numpy (throughput_sim.py:179-186):
//   g = np.random.default_rng(seed)
//   arrivals = np.cumsum(g.exponential(scale=1 / beta_per_ms, size=n))
//   idx      = g.integers(0, len(scenarios), size=n)
//   execs    = g.integers(1, exec_count_max + 1, size=n)
// A Monte-Carlo sweep (configs[3]) needs one such skeleton per scenario, so
// the engine generates them on the GPU -- one thread per skeleton -- with the
// same generator, the same distributions and the same floating-point
// operations as numpy 2.x:
//   * SeedSequence(seed).generate_state(4, uint64) (numpy/random/
//     bit_generator.pyx: hashmix / mix over a 4-word pool) -> PCG64 seeding
//     (pcg64.c pcg64_set_seed / pcg_setseq_128_srandom_r);
//   * PCG64 XSL-RR 128/64 (step, then output), 32-bit draws buffered from
//     64-bit ones low half first (pcg64_next32);
//   * exponential: scale * the ziggurat standard exponential (distributions.c
//     random_standard_exponential) over numpy's own tables (np_ziggurat.inc,
//     extracted from the wheel), the tail via log1p -- glibc's log1p,
//     restated op for op with its FMAs (glibc 2.39 x86_64 __log1p_fma, the
//     variant selected on FMA-capable hosts; tests/test_skeleton.py checks the
//     restatement against the host libm), the wedge test against exp();
//   * integers: Lemire's bounded 32-bit draw (buffered_bounded_lemire_uint32)
//     for ranges below 2^32.
// The wedge comparison `(fe[i-1] - fe[i]) * u + fe[i] < exp(-x)` uses CUDA's
// exp (<= 1 ulp from glibc's); it can only decide differently when the two
// sides are within an ulp of each other (probability ~1e-16 per draw).
//
// SP_HD functions compile for the host too (the CPU tests build them with
// g++ to check the restatement against numpy without a GPU).
#pragma once

#include <stdint.h>
#include <math.h>

// (SP_DT: functions that read the ziggurat tables -- device-only under nvcc,
// where the tables live in device memory)
#ifdef __CUDACC__
#define SP_HD __host__ __device__ __forceinline__
#define SP_DT __device__ __forceinline__
#ifndef SP_ZIG_QUAL
#define SP_ZIG_QUAL __device__ const
#endif
#else
#define SP_HD inline
#define SP_DT inline
#ifndef SP_ZIG_QUAL
#define SP_ZIG_QUAL static const
#endif
#endif

namespace sp {
namespace nprand {

#include "np_ziggurat.inc"

typedef unsigned __int128 u128;

// round-to-nearest primitives that are never contracted (device) / compiled
// with -ffp-contract=off (host test build)
SP_HD double r_add(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
SP_HD double r_sub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
SP_HD double r_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SP_HD double r_div(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
SP_HD double r_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}
SP_HD int32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  uint64_t b;
  __builtin_memcpy(&b, &x, 8);
  return (int32_t)(b >> 32);
#endif
}
SP_HD double with_hi_word(double x, int32_t h) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(h, __double2loint(x));
#else
  uint64_t b;
  __builtin_memcpy(&b, &x, 8);
  b = (b & 0xffffffffull) | ((uint64_t)(uint32_t)h << 32);
  __builtin_memcpy(&x, &b, 8);
  return x;
#endif
}

// ---------------------------------------------------------------------------
// SeedSequence (bit_generator.pyx) for an integer seed < 2^64 and no spawn
// key: entropy = the seed's 32-bit words, little end first ([0] for 0).

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

SP_HD uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> 16;
  return v;
}
SP_HD uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// generate_state(4, np.uint64) of SeedSequence(seed)
SP_HD void seed_sequence_state(uint64_t seed, uint64_t out[4]) {
  uint32_t ent[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const int n_ent = (seed >> 32) ? 2 : 1;
  uint32_t pool[4];
  uint32_t h = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], h));
  uint32_t w[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

// ---------------------------------------------------------------------------
// PCG64 (pcg64.h): 128-bit LCG, XSL-RR output of the stepped state

constexpr u128 kPcgMult = ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;

struct Pcg64 {
  u128 state, inc;
  uint32_t buf;  // pcg64_next32's buffered high half
  int has32;
};

SP_HD void pcg_step(Pcg64& g) { g.state = g.state * kPcgMult + g.inc; }

SP_HD Pcg64 pcg64_from_seed(uint64_t seed) {
  uint64_t v[4];
  seed_sequence_state(seed, v);
  const u128 s = ((u128)v[0] << 64) | v[1], q = ((u128)v[2] << 64) | v[3];
  Pcg64 g;
  g.state = 0;
  g.inc = (q << 1) | 1u;
  pcg_step(g);
  g.state += s;
  pcg_step(g);
  g.buf = 0;
  g.has32 = 0;
  return g;
}

SP_HD uint64_t next_u64(Pcg64& g) {
  pcg_step(g);
  const uint64_t x = (uint64_t)(g.state >> 64) ^ (uint64_t)g.state;
  const unsigned rot = (unsigned)(g.state >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
SP_HD uint32_t next_u32(Pcg64& g) {
  if (g.has32) {
    g.has32 = 0;
    return g.buf;
  }
  const uint64_t x = next_u64(g);
  g.has32 = 1;
  g.buf = (uint32_t)(x >> 32);
  return (uint32_t)x;
}
SP_HD double next_double(Pcg64& g) { return (double)(next_u64(g) >> 11) * (1.0 / 9007199254740992.0); }

// ---------------------------------------------------------------------------
// glibc 2.39 log1p (sysdeps/ieee754/dbl-64/s_log1p.c, x86_64 FMA build):
// the fdlibm algorithm with the polynomial in Estrin form and the FMAs the
// compiler formed there, restated op for op.

SP_HD double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = hi_word(x), ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) return ax < 0x3c900000 ? x : r_fma(-r_mul(x, x), 0.5, x);
    if (hx > 0 || hx < (int32_t)0xbfd2bec4) {
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return r_add(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = r_add(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? r_sub(1.0, r_sub(u, x)) : r_sub(x, r_sub(u, 1.0));
      c = r_div(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = r_sub(u, 1.0);
  }
  const double hfsq = r_mul(r_mul(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : r_fma(dk, ln2_hi, r_fma(dk, ln2_lo, c));
    const double R = r_mul(r_fma(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return r_sub(f, R);
    return r_fma(dk, ln2_hi, -r_sub(r_sub(R, r_fma(dk, ln2_lo, c)), f));
  }
  const double s = r_div(f, r_add(2.0, f));
  const double z = r_mul(s, s);
  const double R2 = r_fma(z, Lp3, Lp2), R3 = r_fma(z, Lp5, Lp4), R4 = r_fma(z, Lp7, Lp6);
  const double z2 = r_mul(z, z), z4 = r_mul(z2, z2), z6 = r_mul(z2, z4);
  const double R = r_fma(z6, R4, r_fma(z4, R3, r_fma(z, Lp1, r_mul(z2, R2))));
  const double t = r_mul(s, r_add(R, hfsq));
  if (k == 0) return r_sub(f, r_sub(hfsq, t));
  return r_fma(dk, ln2_hi, -r_sub(r_sub(hfsq, r_add(r_fma(dk, ln2_lo, c), t)), f));
}

// ---------------------------------------------------------------------------
// distributions (numpy/random/src/distributions/distributions.c)

SP_DT double standard_exponential(Pcg64& g) {
  for (;;) {
    uint64_t ri = next_u64(g);
    ri >>= 3;
    const int idx = (int)(ri & 0xFF);
    ri >>= 8;
    const double x = r_mul((double)ri, np_zig_we[idx]);
    if (ri < np_zig_ke[idx]) return x;  // 98.9 % of the draws
    if (idx == 0) return r_sub(np_zig_exp_r, glibc_log1p(-next_double(g)));
    const double u = next_double(g);
    if (r_add(r_mul(r_sub(np_zig_fe[idx - 1], np_zig_fe[idx]), u), np_zig_fe[idx]) < exp(-x)) return x;
  }
}

// integers(low, high) of a range rng = high - 1 - low < 2^32 - 1 (rng > 0)
SP_HD uint32_t bounded_lemire32(Pcg64& g, uint32_t rng) {
  const uint32_t excl = rng + 1u;
  uint64_t m = (uint64_t)next_u32(g) * excl;
  uint32_t left = (uint32_t)m;
  if (left < excl) {
    const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
    while (left < thr) {
      m = (uint64_t)next_u32(g) * excl;
      left = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

// g.integers(low, high) for high - low in [1, 2^32): Lemire, except that a
// single-value range draws nothing and the full 2^32 range is a raw draw
SP_HD int64_t integers(Pcg64& g, int64_t low, int64_t high) {
  const uint64_t rng = (uint64_t)(high - 1 - low);
  if (rng == 0) return low;
  if (rng == 0xFFFFFFFFull) return low + (int64_t)next_u32(g);
  return low + (int64_t)bounded_lemire32(g, (uint32_t)rng);
}

}  // namespace nprand
}  // namespace sp
