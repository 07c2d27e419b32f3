// ts_core.cuh - host/device core of the V(s) scoring path.
//
// Everything in this header compiles for both the host (C++17, the native
// greedy driver and candidate enumerator) and sm_100a (the featurize and
// generator kernels), so the integer nest math and the bit-exact float
// conversions have exactly one implementation.
//
//   * exact IEEE f64 primitives (no contraction on either side)
//   * glibc 2.39 __log2_fma restated (math.log2 in featurizer.py:55-58, :96-103)
//   * 256-bit unsigned integers with correctly rounded (half-even)
//     conversion and division to f64 (PyLong_AsDouble, int/int true division)
//   * the pipeline descriptor, per-stage loop nests (schedule_space.py:176-285)
//     and the 16-wide feature row (featurizer.py:44-107)
//   * candidate enumeration in the reference's order (schedule_space.py:361-452)
#pragma once

#include <stdint.h>
#include <string.h>
#ifndef __CUDACC__
#include <cmath>
#endif

#include "../../include/tensched_b200.h"
#include "glibc_log2_data.h"

#ifdef __CUDACC__
#define TS_HD __host__ __device__ __forceinline__
#else
#define TS_HD inline
#endif

namespace ts {

// ---------------------------------------------------------------- exact f64
// Device: explicit _rn intrinsics so nvcc never contracts or reorders.
// Host: the library is compiled with -ffp-contract=off.
TS_HD double fadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
TS_HD double fsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
TS_HD double fmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
TS_HD double fdiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
TS_HD double ffma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
TS_HD double as_double(uint64_t u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}
TS_HD uint64_t as_u64(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

// ------------------------------------------------------- glibc 2.39 log2
#ifdef __CUDACC__
// Global (not __constant__): the table index differs per lane, which the
// constant cache would serialize; __ldg keeps it in L1.
__device__ uint64_t d_log2_data[TS_LOG2_NDATA];
#define TS_HD_NOINLINE __host__ __device__ __noinline__
#else
#define TS_HD_NOINLINE inline
#endif

TS_HD double log2_c(int i) {
#ifdef __CUDA_ARCH__
  return as_double(__ldg(reinterpret_cast<const unsigned long long*>(d_log2_data) + i));
#else
  return as_double(ts_log2_data_bits[i]);
#endif
}

// Restatement of glibc 2.39 sysdeps/ieee754/dbl-64/e_log2.c as compiled in
// the x86-64 FMA ifunc variant (libm 0x79f90).  The
// contraction pattern below was read off that binary; all other ops are
// single IEEE operations.  Not correctly rounded - bit-compatibility with
// the reference's math.log2 is the point.  Powers of two short-circuit to
// their exponent: glibc returns them exactly (checked over all 2098 normal
// and subnormal powers, tests/test_host.py).
// Not inlined: the featurizer calls it from up to six sites, and one shared
// copy keeps the walk's code small enough for the instruction cache
// (featurize 12.14 -> 12.03 ms).
TS_HD_NOINLINE double glibc_log2(double x) {
  const uint64_t ix0 = as_u64(x);
  uint64_t ix = ix0;
  if ((ix & 0x000FFFFFFFFFFFFFull) == 0 && ix - 0x0010000000000000ull < 0x7FE0000000000000ull)
    return (double)((int)(ix >> 52) - 1023);
  // |x - 1| small: dedicated polynomial (wrapping unsigned compare).
  if (ix - 0x3feea4af00000000ull <= 0x210a9ffffffffull) {
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double invln2hi = log2_c(0), invln2lo = log2_c(1);
    const double r = fsub(x, 1.0);
    const double hi = fmul(invln2hi, r);
    const double r2 = fmul(r, r);
    const double r4 = fmul(r2, r2);
    const double lo = ffma(r, invln2lo, ffma(invln2hi, r, -hi));
    const double q = ffma(r, log2_c(9), log2_c(8));
    const double y = ffma(q, r2, hi);
    const double l2 = fadd(ffma(q, r2, fsub(hi, y)), lo);
    const double s1 = ffma(ffma(r, log2_c(13), log2_c(12)), r2, ffma(r, log2_c(11), log2_c(10)));
    const double s2 = ffma(ffma(r, log2_c(17), log2_c(16)), r2, ffma(r, log2_c(15), log2_c(14)));
    return fadd(y, ffma(ffma(s2, r4, s1), r4, l2));
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
    // zero, subnormal, negative, inf or nan (never reached by features)
    if ((ix << 1) == 0) return -1.0 / 0.0;
    if (ix == 0x7ff0000000000000ull) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);
    ix = as_u64(fmul(x, 4503599627370496.0));  // 0x1p52
    ix -= 52ull << 52;
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 46) & 63);
  const int k = (int)((int64_t)tmp >> 52);
  const double z = as_double(ix - (tmp & 0xfff0000000000000ull));
  const double invc = log2_c(18 + 2 * i), logc = log2_c(19 + 2 * i);
  const double invln2hi = log2_c(0), invln2lo = log2_c(1);
  const double r = ffma(z, invc, -1.0);
  const double t1 = fmul(r, invln2hi);
  const double t2 = ffma(r, invln2lo, ffma(invln2hi, r, -t1));
  const double t3 = fadd((double)k, logc);
  const double hi = fadd(t1, t3);
  const double lo = fadd(fadd(fsub(t3, hi), t1), t2);
  const double r2 = fmul(r, r);
  const double r4 = fmul(r2, r2);
  const double p = ffma(ffma(r, log2_c(7), log2_c(6)), r4,
                        ffma(ffma(r, log2_c(5), log2_c(4)), r2, ffma(r, log2_c(3), log2_c(2))));
  return fadd(ffma(r2, p, lo), hi);
}

// log2 of small integers from a table holding glibc_log2(i) for i < 4096,
// filled on the device by glibc_log2 itself at context creation (so it is
// bit-identical by construction); larger arguments compute.  Loop extents,
// vector widths and 1 + invocations mostly fall in the table.
constexpr int LOG2_TABLE = 4096;
#ifdef __CUDACC__
__device__ double d_log2_int[LOG2_TABLE];
#endif

TS_HD double log2_int(uint64_t v) {
#ifdef __CUDA_ARCH__
  if (v < (uint64_t)LOG2_TABLE) return __ldg(d_log2_int + v);
#endif
  return glibc_log2((double)v);
}

// ------------------------------------------------------------ 256-bit ints
// Invocation counts reach 133 bits on random VGG-16 states (inv*ppi 141,
// SURVEY.md 7 hard part 4); 256 bits with an overflow status.  All limb
// accesses use static indices (selects) so the device keeps them in
// registers.
struct u256 {
  uint64_t w[4];  // little-endian limbs
};

TS_HD u256 u256_from(uint64_t v) {
  u256 r;
  r.w[0] = v;
  r.w[1] = r.w[2] = r.w[3] = 0;
  return r;
}

TS_HD uint64_t limb(const u256& a, int i) {
  return i == 0 ? a.w[0] : i == 1 ? a.w[1] : i == 2 ? a.w[2] : i == 3 ? a.w[3] : 0;
}

TS_HD int clz64(uint64_t v) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)v);
#else
  return v ? __builtin_clzll(v) : 64;
#endif
}

TS_HD bool u256_small(const u256& a) { return (a.w[1] | a.w[2] | a.w[3]) == 0; }

TS_HD int u256_bitlen(const u256& a) {
  return a.w[3] ? 256 - clz64(a.w[3])
       : a.w[2] ? 192 - clz64(a.w[2])
       : a.w[1] ? 128 - clz64(a.w[1])
       : 64 - clz64(a.w[0]);
}

// a *= m; returns false on overflow past 256 bits
TS_HD bool u256_mul_u64(u256& a, uint64_t m) {
  unsigned __int128 carry = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned __int128 t = (unsigned __int128)a.w[i] * m + carry;
    a.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return carry == 0;
}

TS_HD bool u256_add_u64(u256& a, uint64_t v) {
  unsigned __int128 carry = v;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned __int128 t = (unsigned __int128)a.w[i] + carry;
    a.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return carry == 0;
}

// bits [lo, lo+64) of a, lo in [0, 256)
TS_HD uint64_t u256_bits64(const u256& a, int lo) {
  const int li = lo >> 6, sh = lo & 63;
  uint64_t v = limb(a, li) >> sh;
  if (sh) v |= limb(a, li + 1) << (64 - sh);
  return v;
}

// true iff any bit below position n (0 <= n <= 256) is set
TS_HD bool u256_any_below(const u256& a, int n) {
  bool any = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int base = 64 * i;
    const uint64_t m = n >= base + 64 ? ~0ull : (n <= base ? 0ull : ((1ull << (n - base)) - 1));
    any = any || (a.w[i] & m);
  }
  return any;
}

TS_HD u256 u256_shl(const u256& a, int s) {  // 0 <= s < 256
  u256 r;
  const int li = s >> 6, sh = s & 63;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint64_t v = limb(a, i - li) << sh;
    if (sh) v |= limb(a, i - li - 1) >> (64 - sh);
    r.w[i] = (i - li >= 0) ? v : 0;
  }
  return r;
}

TS_HD double u64_to_double(uint64_t v) {  // round to nearest even
#ifdef __CUDA_ARCH__
  return __ull2double_rn(v);
#else
  return (double)v;
#endif
}

// mant (53 bits, top bit at 52, or exactly 2^53 after rounding) * 2^e2, exact
TS_HD double make_double(uint64_t mant, int e2) {
  if (mant == (1ull << 53)) {
    mant >>= 1;
    e2 += 1;
  }
  const int64_t biased = (int64_t)e2 + 52 + 1023;
  if (biased >= 2047) return 1.0 / 0.0;
  if (biased <= 0) return 0.0;  // subnormal quotients do not occur on this path
  return as_double(((uint64_t)biased << 52) | (mant & ((1ull << 52) - 1)));
}

// Round q + f (0 <= f < 1, f > 0 iff sticky) to 53 bits half-even, times
// 2^e2.  Callers guarantee q has >= 55 bits whenever sticky is set.
// (by value: a reference would force the caller's u256 into local memory)
TS_HD_NOINLINE double round_u256(const u256 q, bool sticky, int e2) {
  const int bl = u256_bitlen(q);
  if (bl == 0) return 0.0;
  if (bl <= 53) {
    const int norm = 53 - bl;
    return make_double(q.w[0] << norm, e2 - norm);
  }
  const int sh = bl - 53;
  uint64_t mant = (u256_bits64(q, sh) & ((1ull << 53) - 1)) | (1ull << 52);
  const bool half = (u256_bits64(q, sh - 1) & 1ull) != 0;
  const bool below = sticky || u256_any_below(q, sh - 1);
  if (half && (below || (mant & 1ull))) mant += 1;
  return make_double(mant, e2 + sh);
}

// PyLong_AsDouble: correctly rounded, ties to even.
TS_HD double u256_to_double(const u256& a) {
  if (u256_small(a)) return u64_to_double(a.w[0]);
  return round_u256(a, false, 0);
}

// Division by an invariant normalized divisor with a precomputed reciprocal
// (Moller & Granlund 2011, "Improved division by invariant integers",
// Alg. 4): (u1:u0) / d with u1 < d, d >= 2^63, v = floor((2^128-1)/d) - 2^64.
TS_HD uint64_t div2by1(uint64_t u1, uint64_t u0, uint64_t d, uint64_t v, uint64_t& r) {
  unsigned __int128 q = (unsigned __int128)v * u1;
  q += ((unsigned __int128)(u1 + 1) << 64) | u0;
  uint64_t q1 = (uint64_t)(q >> 64);
  const uint64_t q0 = (uint64_t)q;
  uint64_t rr = u0 - q1 * d;
  if (rr > q0) {
    q1 -= 1;
    rr += d;
  }
  if (rr >= d) {
    q1 += 1;
    rr -= d;
  }
  r = rr;
  return q1;
}

// Invariant divisor: d = dn >> shift with dn normalized; inv from host.
struct Divisor {
  uint64_t d, dn, inv;
  int32_t shift;
};

inline Divisor make_divisor(uint64_t d) {  // host-side precomputation
  Divisor D;
  D.d = d;
  D.shift = clz64(d);
  D.dn = d << D.shift;
  D.inv = (uint64_t)((~(unsigned __int128)0) / D.dn - ((unsigned __int128)1 << 64));
  return D;
}

// q = a / d (quotient, 256 bits), returns whether the remainder is nonzero
TS_HD u256 u256_div(const u256& a, const Divisor& D, bool& inexact) {
  const int s = D.shift;
  // dividend << s as five limbs n4..n0
  uint64_t n[5];
#pragma unroll
  for (int i = 0; i < 4; ++i) n[i] = s ? (a.w[i] << s) | (i ? a.w[i - 1] >> (64 - s) : 0) : a.w[i];
  n[4] = s ? a.w[3] >> (64 - s) : 0;
  uint64_t r = n[4];
  u256 q;
#pragma unroll
  for (int i = 3; i >= 0; --i) q.w[i] = div2by1(r, n[i], D.dn, D.inv, r);
  inexact = r != 0;
  return q;
}

// CPython int/int true division (long_true_divide): correctly rounded n/d.
TS_HD_NOINLINE double u256_div_to_double_slow(const u256 n, const Divisor D) {
  const int a = u256_bitlen(n);
  if (a == 0) return 0.0;
  const int b = 64 - clz64(D.d);
  int k = 55 + b - a;  // scale so the quotient carries >= 55 bits
  const u256 N = k > 0 ? u256_shl(n, k) : n;
  if (k < 0) k = 0;
  bool inexact;
  const u256 q = u256_div(N, D, inexact);
  return round_u256(q, inexact, -k);
}

// a * m with overflow detection past 128 bits
TS_HD unsigned __int128 mul128_64(unsigned __int128 a, uint64_t m, bool& ok) {
  const unsigned __int128 lo = (unsigned __int128)(uint64_t)a * m;
  const unsigned __int128 hi = (unsigned __int128)(uint64_t)(a >> 64) * m;
  ok = ok && (hi >> 64) == 0;
  const unsigned __int128 r = lo + (hi << 64);
  ok = ok && r >= lo;
  return r;
}

TS_HD int bitlen128(unsigned __int128 a) {
  const uint64_t hi = (uint64_t)(a >> 64);
  return hi ? 128 - clz64(hi) : 64 - clz64((uint64_t)a);
}

// q (>= 55 bits) + fraction (sticky) rounded half-even to 53 bits, * 2^e2
TS_HD double round_u64(uint64_t q, bool sticky, int e2) {
  const int sh = 64 - clz64(q) - 53;
  uint64_t mant = q >> sh;
  const bool half = (q >> (sh - 1)) & 1ull;
  const bool below = sticky || (q & ((1ull << (sh - 1)) - 1)) != 0;
  if (half && (below || (mant & 1ull))) mant += 1;
  return make_double(mant, e2 + sh);
}

// Correctly rounded n / d for n < 2^128 (long_true_divide semantics): scale
// so the integer quotient carries 55-56 bits, one 128/64 division with the
// divisor's precomputed reciprocal, then half-even rounding with sticky.
TS_HD double div128_to_double(unsigned __int128 n, const Divisor& D) {
  if (n == 0) return 0.0;
  const int a = bitlen128(n);
  const int b = 64 - clz64(D.d);
  int k = 55 + b - a;
  unsigned __int128 N;
  bool sticky = false;
  if (k >= 0) {
    N = n << k;  // < 2^(55+b) <= 2^119
  } else {
    const int j = -k;
    N = n >> j;
    sticky = (n & (((unsigned __int128)1 << j) - 1)) != 0;
  }
  // N < d * 2^56, so N << shift fits 128 bits and the quotient fits 64
  const unsigned __int128 Nn = N << D.shift;
  uint64_t r;
  const uint64_t q = div2by1((uint64_t)(Nn >> 64), (uint64_t)Nn, D.dn, D.inv, r);
  return round_u64(q, sticky || r != 0, -k);
}

TS_HD double u256_div_to_double(const u256& n, const Divisor& D) {
  if (u256_small(n) && n.w[0] <= (1ull << 53) && D.d <= (1ull << 53))
    return fdiv(u64_to_double(n.w[0]), u64_to_double(D.d));  // both exact: IEEE division
  return u256_div_to_double_slow(n, D);
}

// ------------------------------------------------------------ descriptor
// Per stage, indexed by topological position (= feature row).
struct StageDesc {
  int32_t n_pure, n_red;
  int64_t ext[TS_MAX_PURE + TS_MAX_RED];  // all_dims order: pure then reduction
  uint64_t pure_points;                   // prod of pure extents
  uint64_t red_points;                    // prod of reduction extents
  uint64_t domain_points;                 // pure_points * red_points
  Divisor dp;                             // domain_points as an invariant divisor
  Divisor io;                             // 1 + input_bytes + output_bytes
  // schedule-invariant integers (pipeline_ir.py:241-252)
  uint64_t i_points, i_flops, i_in_bytes, i_out_bytes;
  int32_t n_inputs;
  int32_t ov_window, ov_stride;  // argmax of window / max(1, stride); window 0 = no edges
  int32_t consumer;              // sole consumer's topo index, -1 if none or several
  int32_t n_cedges;              // consumer edges reading this stage (hull, :218-224)
  int32_t cdim[2][TS_MAX_PURE];  // consumer dim per producer dim, -1 = constant
  int64_t cstride[2][TS_MAX_PURE];
  int64_t cwindow[2][TS_MAX_PURE];
  int32_t slot;  // nest slot (static liveness allocation), -1 = nest never read
  int32_t n_splittable;  // splittable pure dims: innermost two (schedule_space.py:399)
  double fast_c13;       // log2(red_points) - log2(domain_points) (FAST leg's f13, host libm)
};

struct PipelineDesc {
  int32_t n_stages;
  int32_t n_slots;
  StageDesc st[TS_MAX_STAGES];
};

// ------------------------------------------------------------------ nests
// Materialized loops of one scheduled stage (schedule_space.py:118-128),
// compact (80 bytes): what a producer anchored here needs.
struct Nest {
  u256 inv;                   // invocations
  uint32_t ext[TS_MAX_LOOPS]; // loop extents outermost first (< 2^31, descriptor-checked)
  uint8_t id[TS_MAX_LOOPS];   // loop ids (ts_decision.order encoding)
  int32_t n_loops;
  int32_t depth;
  // accessors shared with views of a nest stored elsewhere (the device's
  // shared-memory slots), so the nest math reads a consumer nest in place
  TS_HD uint64_t inv_w(int k) const { return inv.w[k]; }
  TS_HD uint32_t ext_at(int j) const { return ext[j]; }
  TS_HD uint8_t id_at(int j) const { return id[j]; }
  TS_HD int loops() const { return n_loops; }
  TS_HD int dep() const { return depth; }
};

TS_HD int loop_dim(uint8_t id, int n_pure) { return id < 8 ? (id >> 1) : n_pure + (id - 8); }

TS_HD int64_t sel4(const int64_t* a, int k) { return k == 0 ? a[0] : k == 1 ? a[1] : k == 2 ? a[2] : a[3]; }

// _anchor_ok (schedule_space.py:176-187): a level is illegal if it sits
// between the inner and the outer loop of a split dim.
TS_HD bool anchor_ok(const Nest& c, int lvl) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < TS_MAX_LOOPS; ++j) {
    const uint8_t id = c.id[j];
    if (j < c.n_loops && id < 8 && (id & 1) && j <= lvl) {  // inner loop at or above lvl
#pragma unroll
      for (int t = 0; t < TS_MAX_LOOPS; ++t)
        if (t < c.n_loops && c.id[t] == (uint8_t)(id - 1) && lvl < t) ok = false;
    }
  }
  return ok;
}

// Per-invocation pure extents, invocations and depth of stage `s` anchored
// at level `lvl` of its sole consumer's nest (schedule_space.py:190-225).
// Returns TS_OK / TS_ERR_OVERFLOW.
// kFast (device, tensor-core leg): invocations carried as a double in
// inv.w[0] (exact below 2^53, float-accurate beyond - they feed only the
// FAST leg's f13/f15 logarithms, see acquired_features<true>)
template <bool kFast = false, class CN>
TS_HD int anchored_extents(const StageDesc& s, const StageDesc& cs, const CN& cn, int lvl,
                           int64_t* pe, u256& inv, int& depth) {
  // invocations = consumer invocations * prod(outer loop extents up to lvl);
  // a 128-bit path covers all but the deepest chains (branch-uniform within
  // a warp far more often than a 64/256 split), 256 bits the rest
  bool ok = true;
#ifdef __CUDA_ARCH__
  if constexpr (kFast) {
    double v = __longlong_as_double((long long)cn.inv_w(0));
#pragma unroll
    for (int j = 0; j < TS_MAX_LOOPS; ++j)
      if (j <= lvl && j < cn.loops()) v *= (double)cn.ext_at(j);
    inv.w[0] = (uint64_t)__double_as_longlong(v);
    inv.w[1] = inv.w[2] = inv.w[3] = 0;
    ok = v < 1.157920892373162e77;  // 2^256: the exact leg's overflow bound
  } else
#endif
  {
    unsigned __int128 p = ((unsigned __int128)cn.inv_w(1) << 64) | cn.inv_w(0);
    bool fit = cn.inv_w(2) == 0 && cn.inv_w(3) == 0;
    // candidate_actions anchors at levels 0..2 (MAX_COMPUTE_AT_LEVELS); a
    // deeper level (legal for hand-written schedules) takes the long loop
    if (lvl < 3) {
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (j <= lvl && j < cn.loops()) p = mul128_64(p, cn.ext_at(j), fit);
    } else {
#pragma unroll
      for (int j = 0; j < TS_MAX_LOOPS; ++j)
        if (j <= lvl && j < cn.loops()) p = mul128_64(p, cn.ext_at(j), fit);
    }
    if (fit) {
      inv.w[0] = (uint64_t)p;
      inv.w[1] = (uint64_t)(p >> 64);
      inv.w[2] = inv.w[3] = 0;
    } else {
      for (int k = 0; k < 4; ++k) inv.w[k] = cn.inv_w(k);
#pragma unroll
      for (int j = 0; j < TS_MAX_LOOPS; ++j)
        if (j <= lvl && j < cn.loops()) ok = u256_mul_u64(inv, cn.ext_at(j)) && ok;
    }
  }
  // per-invocation consumer region: for each consumer dim read by an edge,
  // the product of that dim's loops strictly inside lvl.  Extents are below
  // 2^31 (descriptor-checked) and so are these products (<= full extents).
  // Consumer dim of every loop strictly inside lvl, a nibble per loop
  // (0xF: outside the region), and the loop extents; then per edge map
  // entry that reads a consumer dim (the stage's cdim: the same for every
  // state at this decision, so these branches are uniform on the device)
  // the product of that dim's inner extents.
  uint32_t dims = 0xFFFFFFFFu;
  uint32_t m[TS_MAX_LOOPS];
  const int nl = cn.loops();
#pragma unroll
  for (int j = 0; j < TS_MAX_LOOPS; ++j) {
    m[j] = cn.ext_at(j);
    const uint32_t dj = (uint32_t)loop_dim(cn.id_at(j), cs.n_pure) & 0xFu;
    if (j > lvl && j < nl) dims = (dims & ~(0xFu << (4 * j))) | (dj << (4 * j));
  }
#pragma unroll
  for (int k = 0; k < TS_MAX_PURE; ++k) pe[k] = -1;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (e >= s.n_cedges) continue;
#pragma unroll
    for (int k = 0; k < TS_MAX_PURE; ++k) {
      const int cd = s.cdim[e][k];
      int64_t ext = s.cwindow[e][k];
      if (cd >= 0) {
        uint32_t rv = 1u;
#pragma unroll
        for (int j = 0; j < TS_MAX_LOOPS; ++j) rv *= ((dims >> (4 * j)) & 0xFu) == (uint32_t)cd ? m[j] : 1u;
        ext += s.cstride[e][k] * ((int64_t)rv - 1);
      }
      pe[k] = ext > pe[k] ? ext : pe[k];
    }
  }
  depth = cn.dep() + lvl + 1;
  return ok ? TS_OK : TS_ERR_OVERFLOW;
}

// _nest_entry/_build_loops (schedule_space.py:228-274).  `cn` may be null
// for Root decisions; pe receives the per-invocation pure extents.
// inner_out (optional): the innermost loop's extent, taken from the value
// being stored (a later lookup ext[n_loops - 1] is a dynamic index, which
// would pin the Nest in local memory on the device).
template <bool kFast = false, class CN = Nest>
TS_HD int build_nest(const StageDesc& s, const StageDesc* cs, const CN* cn, const ts_decision& d,
                     Nest& out, int64_t* pe, uint32_t* inner_out = nullptr) {
  if (d.anchor >= 0) {
    if (!cn || !cs || d.anchor >= cn->loops()) return TS_ERR_ILLEGAL;
    const int rc = anchored_extents<kFast>(s, *cs, *cn, d.anchor, pe, out.inv, out.depth);
    if (rc) return rc;
  } else {
#pragma unroll
    for (int k = 0; k < TS_MAX_PURE; ++k) pe[k] = s.ext[k];
    out.inv = u256_from(kFast ? 0x3FF0000000000000ull : 1);  // kFast: 1.0 as a double
    out.depth = 0;
  }
  if (d.n_loops == 0 || d.n_loops > TS_MAX_LOOPS) return TS_ERR_ILLEGAL;
  out.n_loops = d.n_loops;
  bool bad = false;
  uint32_t inner = 0;
  uint32_t split4;  // split factors, a byte per pure dim
  memcpy(&split4, d.split, 4);
#pragma unroll
  for (int j = 0; j < TS_MAX_LOOPS; ++j) {
    const uint8_t id = d.order[j];
    out.id[j] = id;
    if (j >= d.n_loops) {
      out.ext[j] = 0;
      continue;
    }
    int64_t e;
    if (id < 8) {
      const int k = id >> 1;
      const int64_t f = (split4 >> (8 * k)) & 0xFFu;
      const int64_t p = sel4(pe, k);
      bad = bad || k >= s.n_pure || (!f && (id & 1));
      // extents < 2^31 (descriptor-checked): 32-bit division
      e = f ? ((id & 1) ? f : (int64_t)((uint32_t)p / (uint32_t)f)) : p;
    } else {
      const int r = id - 8;
      bad = bad || r >= s.n_red;
      e = r == 0 ? s.ext[s.n_pure] : r == 1 ? s.ext[s.n_pure + 1] : r == 2 ? s.ext[s.n_pure + 2]
                                                                            : s.ext[s.n_pure + 3];
    }
    out.ext[j] = (uint32_t)e;
    if (j == d.n_loops - 1) inner = (uint32_t)e;
  }
  if (inner_out) *inner_out = inner;
  return bad ? TS_ERR_ILLEGAL : TS_OK;
}

// 16-bit action code -> decision record for stage `s` (layout in
// include/tensched_b200.h, ts_score_states_coded): the candidate_actions
// space - splits of the innermost two pure dims by SPLIT_FACTORS, orders
// from _order_options (schedule_space.py:361-376: pure then reduction loops
// or the reverse, optionally with the last two exchanged), VEC_WIDTHS.
TS_HD ts_decision decode_action(const StageDesc& s, uint32_t code) {
  ts_decision d;
#pragma unroll
  for (int k = 0; k < 4; ++k) d.split[k] = 0;
  const int np = s.n_pure, nr = s.n_red;
  const int first = np >= 2 ? np - 2 : 0;  // splittable = dims[-2:]
  const uint32_t sc0 = (code >> 2) & 3u, sc1 = (code >> 4) & 3u;
  const uint8_t f0 = sc0 == 1 ? 8 : sc0 == 2 ? 32 : 0, f1 = sc1 == 1 ? 8 : sc1 == 2 ? 32 : 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < np) d.split[k] = k == first ? f0 : (k == first + 1 ? f1 : 0);
  // pure loop ids (k -> 2k, split: 2k, 2k+1) and reduction ids (8 + r) in
  // placement order, packed a byte per position (registers, not an array)
  uint64_t seq = 0;
  int n = 0;
  auto push = [&](uint32_t id) {
    if (n < TS_MAX_LOOPS) seq |= (uint64_t)id << (8 * n);
    ++n;
  };
  const bool outer = (code >> 6) & 1u;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    if ((pass == 0) == outer) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (r < nr) push(8 + r);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < np) {
          push(2 * k);
          if (d.split[k]) push(2 * k + 1);
        }
    }
  }
  if (((code >> 7) & 1u) && n >= 2 && n <= TS_MAX_LOOPS) {
    const int sa = 8 * (n - 2), sb = 8 * (n - 1);
    const uint64_t a = (seq >> sa) & 0xFFu, b = (seq >> sb) & 0xFFu;
    seq = (seq & ~(0xFFFFull << sa)) | (b << sa) | (a << sb);
  }
  if (n < TS_MAX_LOOPS) seq |= ~0ull << (8 * n);  // unused positions 0xFF
#pragma unroll
  for (int j = 0; j < TS_MAX_LOOPS; ++j) d.order[j] = (uint8_t)(seq >> (8 * j));
  // codes outside the space decode to an illegal record (n_loops 0), which
  // the featurizer reports as TS_ERR_ILLEGAL
  const bool bad = (code >> 11) != 0u || sc0 == 3u || sc1 == 3u || (np < 2 && sc1 != 0u) || np < 1 ||
                   n > TS_MAX_LOOPS;
  d.n_loops = bad ? 0 : (uint8_t)n;
  d.vec = ((code >> 8) & 1u) ? 8 : 1;
  d.flags = (uint8_t)(((code >> 9) & 1u) | (((code >> 10) & 1u) << 1));
  d.anchor = (int8_t)((int)(code & 3u) - 1);
  return d;
}

// Inverse of decode_action: the code whose decoding is `d`, or 0xFFFF when
// `d` lies outside candidate_actions' space.
TS_HD uint32_t encode_action(const StageDesc& s, const ts_decision& d) {
  if (d.anchor < -1 || d.anchor > 2 || d.flags > 3 || (d.vec != 1 && d.vec != 8)) return 0xFFFFu;
  const int np = s.n_pure;
  const int first = np >= 2 ? np - 2 : 0;
  uint32_t sc[2] = {0u, 0u};
  for (int k = 0; k < 4; ++k) {
    const uint32_t f = d.split[k];
    const uint32_t code = f == 0 ? 0u : f == 8 ? 1u : f == 32 ? 2u : 3u;
    if (k == first && k < np) {
      sc[0] = code;
    } else if (k == first + 1 && np >= 2) {
      sc[1] = code;
    } else if (f != 0) {
      return 0xFFFFu;
    }
  }
  if (sc[0] == 3u || sc[1] == 3u) return 0xFFFFu;
  const uint32_t base = (uint32_t)(d.anchor + 1) | (sc[0] << 2) | (sc[1] << 4) | ((d.vec == 8 ? 1u : 0u) << 8) |
                        ((uint32_t)(d.flags & 1u) << 9) | ((uint32_t)((d.flags >> 1) & 1u) << 10);
  uint32_t dw[4];
  memcpy(dw, &d, sizeof dw);
  // (placement, swap) in _order_options' order; the first variant that
  // reproduces the record wins (equal orders decode identically)
  for (uint32_t v = 0; v < 4; ++v) {
    const uint32_t code = base | ((v >> 1) << 6) | ((v & 1u) << 7);
    const ts_decision e = decode_action(s, code);
    uint32_t ew[4];
    memcpy(ew, &e, sizeof ew);
    if (ew[0] == dw[0] && ew[1] == dw[1] && ew[2] == dw[2] && ew[3] == dw[3]) return code;
  }
  return 0xFFFFu;
}

// check_action (schedule_space.py:288-347) on an encoded decision: null if
// legal, else the violated invariant.  Host only.
inline const char* check_decision(const StageDesc& s, const StageDesc* cs, const Nest* cn,
                                  const ts_decision& d) {
  if (d.anchor >= 0) {
    if (!cs || !cn) return "compute_at target must be the sole consumer";
    if (d.anchor >= cn->n_loops) return "compute_at loop level does not exist in the consumer's nest";
    if (!anchor_ok(*cn, d.anchor)) return "anchor level fixes a low-order split digit; anchored region would be strided";
  } else if (d.flags & TS_FLAG_STORE_AT) {
    return "store_at must be Root or the compute_at site";
  }
  int64_t pe[TS_MAX_PURE];
  if (d.anchor >= 0) {
    u256 inv;
    int depth;
    if (anchored_extents(s, *cs, *cn, d.anchor, pe, inv, depth)) return "integer exceeded 256 bits";
  } else {
    for (int k = 0; k < s.n_pure; ++k) pe[k] = s.ext[k];
  }
  for (int k = 0; k < TS_MAX_PURE; ++k) {
    const int f = d.split[k];
    if (!f) continue;
    if (k >= s.n_pure) return "cannot split non-pure dim";
    if (f < 2) return "split factor < 2";
    if (pe[k] % f != 0) return "split factor does not divide the dim's extent";
  }
  // order must be a permutation of the loops implied by the splits
  int seen[16] = {0};
  int expect = 0;
  for (int k = 0; k < s.n_pure; ++k) expect += d.split[k] ? 2 : 1;
  expect += s.n_red;
  if (d.n_loops != expect) return "order is not a permutation of the stage's loops";
  for (int j = 0; j < d.n_loops; ++j) {
    const int id = d.order[j];
    if (id >= 16) return "order is not a permutation of the stage's loops";
    if (id < 8) {
      const int k = id >> 1;
      if (k >= s.n_pure || ((id & 1) && !d.split[k])) return "order is not a permutation of the stage's loops";
    } else if (id - 8 >= s.n_red) {
      return "order is not a permutation of the stage's loops";
    }
    if (seen[id]++) return "order is not a permutation of the stage's loops";
  }
  Nest n;
  int64_t pe2[TS_MAX_PURE];
  if (build_nest(s, cs, cn, d, n, pe2)) return "order is not a permutation of the stage's loops";
  if (!(d.vec == 1 || d.vec == 4 || d.vec == 8 || d.vec == 16)) return "bad vectorize width";
  if (d.vec > 1) {
    if (n.id[n.n_loops - 1] >= 8) return "vectorized loop is a reduction dim";
    if (n.ext[n.n_loops - 1] % d.vec != 0) return "vector width does not divide innermost extent";
  }
  if ((d.flags & TS_FLAG_PARALLEL) && n.id[0] >= 8) return "parallel loop is a reduction dim";
  return nullptr;
}

#ifdef __CUDA_ARCH__
// log2 of a positive finite double to float accuracy: its exponent plus
// one MUFU lg2 of its mantissa
__device__ __forceinline__ double fast_log2_d(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  const int e = (int)((b >> 52) & 0x7FF) - 1023;
  const float m = (float)__longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
  return (double)e + (double)__log2f(m);
}

// log2 of a nonzero 64-bit integer to float accuracy (see fast_log2_u256)
__device__ __forceinline__ double fast_log2_u64(uint64_t v) {
  const int lz = __clzll((long long)v);
  const float m = (float)(uint32_t)((v << lz) >> 32) * 4.656612873077393e-10f;  // [1, 2)
  return (double)(63 - lz) + (double)__log2f(m);
}

// log2 of a nonzero 256-bit integer to float accuracy: bit length from the
// leading word, top 32 bits as the mantissa, one MUFU lg2 (|error| < 2^-21).
// The tensor-core (FAST) leg's recompute and invocation features only: its
// operands are rounded to f32 and split into 22-bit fp16 pairs anyway.
__device__ __forceinline__ double fast_log2_u256(const u256& a) {
  // leading word by selects (a dynamic a.w[k] would put the value in local memory)
  const int k = a.w[3] ? 3 : a.w[2] ? 2 : a.w[1] ? 1 : 0;
  const uint64_t hi = k == 3 ? a.w[3] : k == 2 ? a.w[2] : k == 1 ? a.w[1] : a.w[0];
  const uint64_t lo = k == 3 ? a.w[2] : k == 2 ? a.w[1] : k == 1 ? a.w[0] : 0;
  const int lz = __clzll((long long)hi);
  const uint64_t top = lz ? (hi << lz) | (lo >> (64 - lz)) : hi;  // leading 1 at bit 63
  const int e = 64 * k + 63 - lz;
  const float m = (float)(uint32_t)(top >> 32) * 4.656612873077393e-10f;  // [1, 2)
  return (double)e + (double)__log2f(m);
}
#endif

// Acquired features f8..f15 of a scheduled stage (featurizer.py:86-103),
// raw (not normalized).  kFast (device, tensor-core leg only): f13 and f15
// to float accuracy (fast_log2_u256) instead of the correctly rounded
// division and glibc's log2 - see k_featurize_rows<float>.
template <bool kFast = false>
TS_HD int acquired_features(const StageDesc& s, const Nest& n, const int64_t* pe, const ts_decision& d,
                            double* f, uint32_t inner) {
  f[0] = 1.0;
  f[1] = log2_int(d.vec);
  f[2] = (d.flags & TS_FLAG_PARALLEL) ? log2_int(n.ext[0]) : 0.0;
  f[3] = log2_int(inner);
  f[4] = (double)n.depth;
  // recompute factor = Fraction(inv * ppi, domain_points)  (cost_oracle.py:108-121)
  uint64_t region = 1;
#pragma unroll
  for (int k = 0; k < TS_MAX_PURE; ++k)
    if (k < s.n_pure) region *= (uint64_t)pe[k];
#ifdef __CUDA_ARCH__
  if constexpr (kFast) {
    // invocations as a double (anchored_extents<true>); log2(inv * region *
    // red_points / domain_points) = log2(inv) + log2(region) + the stage's
    // constant log2(red_points / domain_points)
    const double inv = __longlong_as_double((long long)n.inv.w[0]);
    if (!(inv * (double)region * (double)s.red_points < 1.157920892373162e77)) return TS_ERR_OVERFLOW;
    f[5] = fast_log2_d(inv) + fast_log2_u64(region) + s.fast_c13;
    const uint64_t pts = (d.flags & TS_FLAG_STORE_AT) ? region : s.pure_points;
    f[6] = pts <= 8192u ? 1.0 : 0.0;
    const double inv1 = inv + 1.0;  // exact below 2^53
    f[7] = inv1 < (double)LOG2_TABLE ? log2_int((uint64_t)inv1) : fast_log2_d(inv1);
    return TS_OK;
  }
#endif
  // inv * ppi below 2^128 (all but the deepest anchor chains): one
  // branch-uniform 128-bit correctly rounded division
  bool fit = n.inv.w[2] == 0 && n.inv.w[3] == 0;
  unsigned __int128 num128 = 0;
  if (fit) {
    num128 = mul128_64(((unsigned __int128)n.inv.w[1] << 64) | n.inv.w[0], region, fit);
    num128 = mul128_64(num128, s.red_points, fit);
  }
  if (fit) {
    f[5] = glibc_log2(div128_to_double(num128, s.dp));
  } else {
    u256 num = n.inv;
    bool ok = u256_mul_u64(num, region);
    ok = u256_mul_u64(num, s.red_points) && ok;
    if (!ok) return TS_ERR_OVERFLOW;
    f[5] = glibc_log2(u256_div_to_double(num, s.dp));
  }
  // working set at the store site (cost_oracle.py:162-169), cache 32768
  const uint64_t pts = (d.flags & TS_FLAG_STORE_AT) ? region : s.pure_points;
  f[6] = pts <= 8192u ? 1.0 : 0.0;  // 4 * pts <= 32768, overflow-free
  u256 inv1 = n.inv;
  if (!u256_add_u64(inv1, 1)) return TS_ERR_OVERFLOW;
  if (u256_small(inv1)) {
    f[7] = log2_int(inv1.w[0]);
  } else if (inv1.w[2] == 0 && inv1.w[3] == 0) {  // < 2^128: top 64 bits + sticky
    const int sh = 64 - clz64(inv1.w[1]);
    const uint64_t top = (inv1.w[1] << (64 - sh)) | (sh < 64 ? inv1.w[0] >> sh : 0);
    const bool sticky = sh < 64 ? (inv1.w[0] & ((1ull << sh) - 1)) != 0 : inv1.w[0] != 0;
    f[7] = glibc_log2(round_u64(top, sticky, sh));
  } else {
    f[7] = glibc_log2(u256_to_double(inv1));
  }
  return TS_OK;
}

TS_HD int acquired_features(const StageDesc& s, const Nest& n, const int64_t* pe, const ts_decision& d,
                            double* f) {
  uint32_t inner = 0;
#pragma unroll
  for (int j = 0; j < TS_MAX_LOOPS; ++j)
    if (j == n.n_loops - 1) inner = n.ext[j];
  return acquired_features(s, n, pe, d, f, inner);
}

// Intrinsic features f0..f7 (featurizer.py:44-65).
TS_HD void intrinsic_features(const StageDesc& s, double* f) {
  f[0] = glibc_log2(u256_to_double(u256_from(s.i_points + 1)));
  f[1] = glibc_log2(u256_to_double(u256_from(s.i_flops + 1)));
  f[2] = glibc_log2(u256_to_double(u256_from(s.i_in_bytes + 1)));
  f[3] = glibc_log2(u256_to_double(u256_from(s.i_out_bytes + 1)));
  f[4] = u256_div_to_double(u256_from(s.i_flops), s.io);
  f[5] = (double)s.n_inputs;
  f[6] = (double)s.n_red;
  f[7] = s.ov_window ? fdiv((double)s.ov_window, (double)(s.ov_stride > 1 ? s.ov_stride : 1)) : 0.0;
}

// ------------------------------------------------------- candidate actions
// Enumerates candidate_actions (schedule_space.py:379-452) for stage `s`
// given its sole consumer's nest (or null).  Calls emit(const ts_decision&)
// in the reference's order; returns the count (or -status on error).
template <typename Emit>
TS_HD int64_t enumerate_candidates(const StageDesc& s, const StageDesc* cs, const Nest* cn,
                                   Emit&& emit) {
  int anchors[1 + 3];
  int n_anchor = 0;
  anchors[n_anchor++] = -1;
  if (cn && cs) {
    const int lim = cn->n_loops < 3 ? cn->n_loops : 3;  // MAX_COMPUTE_AT_LEVELS
    for (int lvl = 0; lvl < lim; ++lvl)
      if (anchor_ok(*cn, lvl)) anchors[n_anchor++] = lvl;
  }
  const int n_pure = s.n_pure, n_red = s.n_red;
  const int first_split = n_pure >= 2 ? n_pure - 2 : 0;  // splittable = dims[-2:]
  int64_t count = 0;
  for (int ai = 0; ai < n_anchor; ++ai) {
    const int anchor = anchors[ai];
    int64_t pe[TS_MAX_PURE];
    if (anchor < 0) {
      for (int k = 0; k < n_pure; ++k) pe[k] = s.ext[k];
    } else {
      u256 inv;
      int depth;
      if (anchored_extents(s, *cs, *cn, anchor, pe, inv, depth)) return -TS_ERR_OVERFLOW;
    }
    // split options per splittable dim: None, 8, 32 (divisible and smaller)
    int opts[2][3];
    int n_opts[2] = {0, 0};
    const int n_sd = n_pure - first_split;
    for (int q = 0; q < n_sd; ++q) {
      const int64_t e = pe[first_split + q];
      opts[q][n_opts[q]++] = 0;
      if (e % 8 == 0 && 8 < e) opts[q][n_opts[q]++] = 8;
      if (e % 32 == 0 && 32 < e) opts[q][n_opts[q]++] = 32;
    }
    const int n_store = anchor < 0 ? 1 : 2;
    // itertools.product: last dim varies fastest
    const int n0 = n_opts[0], n1 = n_sd > 1 ? n_opts[1] : 1;
    for (int c0 = 0; c0 < n0; ++c0) {
      for (int c1 = 0; c1 < n1; ++c1) {
        int split[TS_MAX_PURE] = {0, 0, 0, 0};
        split[first_split] = opts[0][c0];
        if (n_sd > 1) split[first_split + 1] = opts[1][c1];
        // pure loop names in dim order, split dims expand to outer, inner
        uint8_t pure_ids[2 * TS_MAX_PURE];
        int64_t pure_ext[2 * TS_MAX_PURE];
        int np = 0;
        for (int k = 0; k < n_pure; ++k) {
          if (split[k]) {
            pure_ids[np] = (uint8_t)(2 * k);
            pure_ext[np++] = pe[k] / split[k];
            pure_ids[np] = (uint8_t)(2 * k + 1);
            pure_ext[np++] = split[k];
          } else {
            pure_ids[np] = (uint8_t)(2 * k);
            pure_ext[np++] = pe[k];
          }
        }
        const int nl = np + n_red;
        if (nl > TS_MAX_LOOPS) return -TS_ERR_PIPELINE;
        // _order_options (schedule_space.py:361-376)
        uint8_t seqs[4][TS_MAX_LOOPS];
        int64_t seq_ext[4][TS_MAX_LOOPS];
        int n_seq = 0;
        const int n_place = n_red ? 2 : 1;
        for (int pl = 0; pl < n_place; ++pl) {
          uint8_t base[TS_MAX_LOOPS];
          int64_t bext[TS_MAX_LOOPS];
          int t = 0;
          // t < nl <= TS_MAX_LOOPS (checked above); the bound is restated in
          // the loops so the compiler's range analysis sees it too
          if (pl == 0) {
            for (int j = 0; j < np && t < TS_MAX_LOOPS; ++j) { base[t] = pure_ids[j]; bext[t++] = pure_ext[j]; }
            for (int r = 0; r < n_red && t < TS_MAX_LOOPS; ++r) { base[t] = (uint8_t)(8 + r); bext[t++] = s.ext[n_pure + r]; }
          } else {
            for (int r = 0; r < n_red && t < TS_MAX_LOOPS; ++r) { base[t] = (uint8_t)(8 + r); bext[t++] = s.ext[n_pure + r]; }
            for (int j = 0; j < np && t < TS_MAX_LOOPS; ++j) { base[t] = pure_ids[j]; bext[t++] = pure_ext[j]; }
          }
          for (int sw = 0; sw < 2; ++sw) {
            uint8_t seq[TS_MAX_LOOPS];
            int64_t sext[TS_MAX_LOOPS];
            for (int j = 0; j < nl; ++j) { seq[j] = base[j]; sext[j] = bext[j]; }
            if (sw && nl >= 2) {
              uint8_t ti = seq[nl - 1]; seq[nl - 1] = seq[nl - 2]; seq[nl - 2] = ti;
              int64_t te = sext[nl - 1]; sext[nl - 1] = sext[nl - 2]; sext[nl - 2] = te;
            }
            bool dup = false;
            for (int q = 0; q < n_seq && !dup; ++q) {
              bool same = true;
              for (int j = 0; j < nl; ++j) same = same && seqs[q][j] == seq[j];
              dup = same;
            }
            if (!dup) {
              for (int j = 0; j < nl; ++j) { seqs[n_seq][j] = seq[j]; seq_ext[n_seq][j] = sext[j]; }
              ++n_seq;
            }
          }
        }
        for (int q = 0; q < n_seq; ++q) {
          const uint8_t inner = seqs[q][nl - 1];
          const bool inner_pure = inner < 8;
          const int n_vec = (inner_pure && seq_ext[q][nl - 1] % 8 == 0) ? 2 : 1;  // VEC_WIDTHS
          const bool outer_pure = seqs[q][0] < 8;
          const int n_par = outer_pure ? 2 : 1;
          for (int v = 0; v < n_vec; ++v) {
            for (int pr = 0; pr < n_par; ++pr) {
              for (int so = 0; so < n_store; ++so) {
                ts_decision dd;
                for (int k = 0; k < TS_MAX_PURE; ++k) dd.split[k] = (uint8_t)split[k];
                for (int j = 0; j < TS_MAX_LOOPS; ++j) dd.order[j] = j < nl ? seqs[q][j] : 0xFF;
                dd.n_loops = (uint8_t)nl;
                dd.vec = v ? 8 : 1;
                dd.flags = (uint8_t)((pr ? TS_FLAG_PARALLEL : 0) | (so ? TS_FLAG_STORE_AT : 0));
                dd.anchor = (int8_t)anchor;
                emit(dd);
                ++count;
              }
            }
          }
        }
      }
    }
  }
  return count;
}

// ------------------------------------------------------------ splitmix64
// SearchRng (search.py:30-58).
TS_HD uint64_t splitmix_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
TS_HD uint64_t rng_randrange(uint64_t& state, uint64_t n) {
  const uint64_t z = splitmix_next(state);
  return (uint64_t)(((unsigned __int128)z * n) >> 64);
}
// uniform(lo, hi) = lo + ((u64 >> 11) / 2^53) * (hi - lo)  (search.py:47-49)
TS_HD double rng_uniform(uint64_t& state, double lo, double hi) {
  const uint64_t z = splitmix_next(state);
  const double u = fmul((double)(z >> 11), 1.1102230246251565e-16);  // exact: * 2^-53
  return fadd(lo, fmul(u, fsub(hi, lo)));
}

}  // namespace ts
