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
__device__ __constant__ uint64_t d_log2_data[TS_LOG2_NDATA];
#endif

TS_HD double log2_c(int i) {
#ifdef __CUDA_ARCH__
  return as_double(d_log2_data[i]);
#else
  return as_double(ts_log2_data_bits[i]);
#endif
}

// Restatement of glibc 2.39 sysdeps/ieee754/dbl-64/e_log2.c as compiled in
// the x86-64 FMA ifunc variant (libm 0x79f90).  The
// contraction pattern below was read off that binary; all other ops are
// single IEEE operations.  Not correctly rounded - bit-compatibility with
// the reference's math.log2 is the point.
TS_HD double glibc_log2(double x) {
  const uint64_t ix0 = as_u64(x);
  uint64_t ix = ix0;
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

// ------------------------------------------------------------ 256-bit ints
struct u256 {
  uint64_t w[4];  // little-endian limbs
};

TS_HD u256 u256_from(uint64_t v) {
  u256 r;
  r.w[0] = v;
  r.w[1] = r.w[2] = r.w[3] = 0;
  return r;
}

TS_HD int clz64(uint64_t v) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)v);
#else
  return v ? __builtin_clzll(v) : 64;
#endif
}

TS_HD int u256_bitlen(const u256& a) {
  for (int i = 3; i >= 0; --i)
    if (a.w[i]) return 64 * i + 64 - clz64(a.w[i]);
  return 0;
}

// a *= m; returns false on overflow past 256 bits
TS_HD bool u256_mul_u64(u256& a, uint64_t m) {
  unsigned __int128 carry = 0;
  for (int i = 0; i < 4; ++i) {
    unsigned __int128 t = (unsigned __int128)a.w[i] * m + carry;
    a.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return carry == 0;
}

TS_HD bool u256_add_u64(u256& a, uint64_t v) {
  unsigned __int128 carry = v;
  for (int i = 0; i < 4; ++i) {
    unsigned __int128 t = (unsigned __int128)a.w[i] + carry;
    a.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return carry == 0;
}

// bits [lo, lo+64) of a (zero beyond 256)
TS_HD uint64_t u256_bits64(const u256& a, int lo) {
  if (lo >= 256) return 0;
  if (lo < 0) {
    // only used with lo >= -63: shift left
    return a.w[0] << (-lo);
  }
  const int li = lo >> 6, sh = lo & 63;
  uint64_t v = a.w[li] >> sh;
  if (sh && li + 1 < 4) v |= a.w[li + 1] << (64 - sh);
  return v;
}

// true iff any bit below position `n` is set
TS_HD bool u256_any_below(const u256& a, int n) {
  for (int i = 0; i < 4; ++i) {
    const int base = 64 * i;
    if (n <= base) break;
    if (n >= base + 64) {
      if (a.w[i]) return true;
    } else {
      if (a.w[i] & ((1ull << (n - base)) - 1)) return true;
    }
  }
  return false;
}

TS_HD u256 u256_shl(const u256& a, int s) {
  u256 r = u256_from(0);
  const int li = s >> 6, sh = s & 63;
  for (int i = 3; i >= li; --i) {
    uint64_t v = a.w[i - li] << sh;
    if (sh && i - li - 1 >= 0) v |= a.w[i - li - 1] >> (64 - sh);
    r.w[i] = v;
  }
  return r;
}

// Builds the double mant * 2^e2 for a 53-bit mant in [2^52, 2^53] (exact).
TS_HD double make_double(uint64_t mant, int e2) {
  if (mant == (1ull << 53)) {
    mant >>= 1;
    e2 += 1;
  }
  // value = mant * 2^e2, mant has its top bit at 52 -> exponent e2 + 52
  const int64_t biased = (int64_t)e2 + 52 + 1023;
  if (biased >= 2047) return 1.0 / 0.0;
  if (biased <= 0) {
    // subnormal: cannot happen for the quantities on this path; fall back
    // to an exact-as-possible scaling (flag via caller bounds)
    double d = (double)mant;
    for (int i = 0; i < -e2; ++i) d = fmul(d, 0.5);
    return d;
  }
  return as_double(((uint64_t)biased << 52) | (mant & ((1ull << 52) - 1)));
}

// Round the integer (q, sticky) - value q + f with 0 <= f < 1 and f > 0 iff
// sticky - to 53 bits half-even, scaled by 2^e2.
TS_HD double round_u256(const u256& q, bool sticky, int e2) {
  const int bl = u256_bitlen(q);
  if (bl == 0) return 0.0;
  if (bl <= 53 && !sticky) {
    const uint64_t m = q.w[0];
    const int norm = 53 - bl;
    return make_double(m << norm, e2 - norm);
  }
  if (bl <= 53) {
    // fraction bits below the integer: caller guarantees bl >= 55 when
    // sticky is set, so this branch is unreachable in practice
    const uint64_t m = q.w[0];
    const int norm = 53 - bl;
    return make_double(m << norm, e2 - norm);
  }
  const int sh = bl - 53;
  uint64_t mant = u256_bits64(q, sh) & ((1ull << 53) - 1);
  mant |= (1ull << 52);
  // rounding: bit sh-1 is the half bit, below it + sticky decide
  const bool half = (u256_bits64(q, sh - 1) & 1ull) != 0;
  const bool below = u256_any_below(q, sh - 1) || sticky;
  if (half && (below || (mant & 1ull))) mant += 1;
  return make_double(mant, e2 + sh);
}

// PyLong_AsDouble: correctly rounded, ties to even.
TS_HD double u256_to_double(const u256& a) { return round_u256(a, false, 0); }

// q = a / d, r = a % d (d > 0)
TS_HD u256 u256_divmod_u64(const u256& a, uint64_t d, uint64_t& rem) {
  u256 q;
  unsigned __int128 r = 0;
  for (int i = 3; i >= 0; --i) {
    const unsigned __int128 cur = (r << 64) | a.w[i];
    q.w[i] = (uint64_t)(cur / d);
    r = cur % d;
  }
  rem = (uint64_t)r;
  return q;
}

// CPython int/int true division (long_true_divide): correctly rounded n/d.
TS_HD double u256_div_u64_to_double(const u256& n, uint64_t d) {
  const int a = u256_bitlen(n);
  if (a == 0) return 0.0;
  const int b = 64 - clz64(d);
  int k = 55 + b - a;  // scale so the quotient carries >= 55 bits
  u256 N = n;
  if (k > 0) {
    N = u256_shl(n, k);
  } else {
    k = 0;
  }
  uint64_t rem;
  const u256 q = u256_divmod_u64(N, d, rem);
  return round_u256(q, rem != 0, -k);
}

// ------------------------------------------------------------ descriptor
// Per stage, indexed by topological position (= feature row).
struct StageDesc {
  int32_t n_pure, n_red;
  int64_t ext[TS_MAX_PURE + TS_MAX_RED];  // all_dims order: pure then reduction
  uint64_t pure_points;                   // prod of pure extents
  uint64_t red_points;                    // prod of reduction extents
  uint64_t domain_points;                 // pure_points * red_points
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
};

struct PipelineDesc {
  int32_t n_stages;
  int32_t n_slots;
  StageDesc st[TS_MAX_STAGES];
};

// ------------------------------------------------------------------ nests
// Materialized loops of one scheduled stage (schedule_space.py:118-128).
struct Nest {
  u256 inv;                    // invocations
  int64_t pe[TS_MAX_PURE];     // per-invocation pure extents
  int64_t ext[TS_MAX_LOOPS];   // loop extents outermost first
  uint8_t id[TS_MAX_LOOPS];    // loop ids (ts_decision.order encoding)
  int32_t n_loops;
  int32_t depth;
};

TS_HD int loop_dim(uint8_t id, int n_pure) { return id < 8 ? (id >> 1) : n_pure + (id - 8); }

// _anchor_ok (schedule_space.py:176-187): a level is illegal if it sits
// between the inner and the outer loop of a split dim.
TS_HD bool anchor_ok(const Nest& c, int lvl) {
  for (int j = 0; j < c.n_loops; ++j) {
    const uint8_t id = c.id[j];
    if (id < 8 && (id & 1)) {  // inner loop of split dim (id>>1)
      const int pi = j;
      int po = -1;
      for (int t = 0; t < c.n_loops; ++t)
        if (c.id[t] == (uint8_t)(id - 1)) po = t;
      if (po >= 0 && pi <= lvl && lvl < po) return false;
    }
  }
  return true;
}

// Per-invocation pure extents, invocations and depth of stage `s` anchored
// at level `lvl` of its sole consumer's nest (schedule_space.py:190-225).
// Returns TS_OK / TS_ERR_OVERFLOW.
TS_HD int anchored_extents(const StageDesc& s, const StageDesc& cs, const Nest& cn, int lvl,
                           int64_t* pe, u256& inv, int& depth) {
  inv = cn.inv;
  for (int j = 0; j <= lvl; ++j)
    if (!u256_mul_u64(inv, (uint64_t)cn.ext[j])) return TS_ERR_OVERFLOW;
  int64_t rem[TS_MAX_PURE + TS_MAX_RED];
  const int cdims = cs.n_pure + cs.n_red;
  for (int d = 0; d < cdims; ++d) rem[d] = 1;
  for (int j = lvl + 1; j < cn.n_loops; ++j) rem[loop_dim(cn.id[j], cs.n_pure)] *= cn.ext[j];
  for (int k = 0; k < s.n_pure; ++k) {
    int64_t best = -1;
    for (int e = 0; e < s.n_cedges; ++e) {
      const int cd = s.cdim[e][k];
      const int64_t ext = cd < 0 ? s.cwindow[e][k] : s.cstride[e][k] * (rem[cd] - 1) + s.cwindow[e][k];
      if (ext > best) best = ext;
    }
    pe[k] = best;
  }
  depth = cn.depth + lvl + 1;
  return TS_OK;
}

// _nest_entry/_build_loops (schedule_space.py:228-274).  `cn` may be null
// for Root decisions.  Returns a ts_status.
TS_HD int build_nest(const StageDesc& s, const StageDesc* cs, const Nest* cn, const ts_decision& d,
                     Nest& out) {
  if (d.anchor >= 0) {
    if (!cn || !cs || d.anchor >= cn->n_loops) return TS_ERR_ILLEGAL;
    const int rc = anchored_extents(s, *cs, *cn, d.anchor, out.pe, out.inv, out.depth);
    if (rc) return rc;
  } else {
    for (int k = 0; k < s.n_pure; ++k) out.pe[k] = s.ext[k];
    out.inv = u256_from(1);
    out.depth = 0;
  }
  if (d.n_loops == 0 || d.n_loops > TS_MAX_LOOPS) return TS_ERR_ILLEGAL;
  out.n_loops = d.n_loops;
  for (int j = 0; j < d.n_loops; ++j) {
    const uint8_t id = d.order[j];
    out.id[j] = id;
    if (id < 8) {
      const int k = id >> 1;
      if (k >= s.n_pure) return TS_ERR_ILLEGAL;
      const int64_t f = d.split[k];
      if (f) {
        out.ext[j] = (id & 1) ? f : out.pe[k] / f;
      } else {
        if (id & 1) return TS_ERR_ILLEGAL;
        out.ext[j] = out.pe[k];
      }
    } else {
      const int r = id - 8;
      if (r >= s.n_red) return TS_ERR_ILLEGAL;
      out.ext[j] = s.ext[s.n_pure + r];
    }
  }
  return TS_OK;
}

// check_action (schedule_space.py:288-347) on an encoded decision: null if
// legal, else the violated invariant.
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
  if (build_nest(s, cs, cn, d, n)) return "order is not a permutation of the stage's loops";
  if (!(d.vec == 1 || d.vec == 4 || d.vec == 8 || d.vec == 16)) return "bad vectorize width";
  if (d.vec > 1) {
    if (n.id[n.n_loops - 1] >= 8) return "vectorized loop is a reduction dim";
    if (n.ext[n.n_loops - 1] % d.vec != 0) return "vector width does not divide innermost extent";
  }
  if ((d.flags & TS_FLAG_PARALLEL) && n.id[0] >= 8) return "parallel loop is a reduction dim";
  return nullptr;
}

// Acquired features f8..f15 of a scheduled stage (featurizer.py:86-103),
// raw (not normalized).
TS_HD int acquired_features(const StageDesc& s, const Nest& n, const ts_decision& d, double* f) {
  f[0] = 1.0;
  f[1] = glibc_log2((double)d.vec);
  f[2] = (d.flags & TS_FLAG_PARALLEL) ? glibc_log2((double)n.ext[0]) : 0.0;
  f[3] = glibc_log2((double)n.ext[n.n_loops - 1]);
  f[4] = (double)n.depth;
  // recompute factor = Fraction(inv * ppi, domain_points)  (cost_oracle.py:108-121)
  uint64_t region = 1;
  for (int k = 0; k < s.n_pure; ++k) region *= (uint64_t)n.pe[k];
  u256 num = n.inv;
  if (!u256_mul_u64(num, region)) return TS_ERR_OVERFLOW;
  if (!u256_mul_u64(num, s.red_points)) return TS_ERR_OVERFLOW;
  f[5] = glibc_log2(u256_div_u64_to_double(num, s.domain_points));
  // working set at the store site (cost_oracle.py:162-169), cache 32768
  const uint64_t pts = (d.flags & TS_FLAG_STORE_AT) ? region : s.pure_points;
  const unsigned __int128 ws = (unsigned __int128)pts * 4u;
  f[6] = ws <= 32768u ? 1.0 : 0.0;
  u256 inv1 = n.inv;
  if (!u256_add_u64(inv1, 1)) return TS_ERR_OVERFLOW;
  f[7] = glibc_log2(u256_to_double(inv1));
  return TS_OK;
}

// Intrinsic features f0..f7 (featurizer.py:44-65).
TS_HD void intrinsic_features(const StageDesc& s, double* f) {
  f[0] = glibc_log2(u256_to_double(u256_from(s.i_points + 1)));
  f[1] = glibc_log2(u256_to_double(u256_from(s.i_flops + 1)));
  f[2] = glibc_log2(u256_to_double(u256_from(s.i_in_bytes + 1)));
  f[3] = glibc_log2(u256_to_double(u256_from(s.i_out_bytes + 1)));
  f[4] = u256_div_u64_to_double(u256_from(s.i_flops), 1 + s.i_in_bytes + s.i_out_bytes);
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
          if (pl == 0) {
            for (int j = 0; j < np; ++j) { base[t] = pure_ids[j]; bext[t++] = pure_ext[j]; }
            for (int r = 0; r < n_red; ++r) { base[t] = (uint8_t)(8 + r); bext[t++] = s.ext[n_pure + r]; }
          } else {
            for (int r = 0; r < n_red; ++r) { base[t] = (uint8_t)(8 + r); bext[t++] = s.ext[n_pure + r]; }
            for (int j = 0; j < np; ++j) { base[t] = pure_ids[j]; bext[t++] = pure_ext[j]; }
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
