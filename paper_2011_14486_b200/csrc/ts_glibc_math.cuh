// ts_glibc_math.cuh - glibc 2.39 exp and tanh restated for host and device.
//
// The reference's exact V is computed by its Cython kernel with libc `exp`
// and `tanh` (_recurrent_cy.pyx:10, :17-18, :58-60) and finished with CPython
// math.exp (value_model.py:154).  Neither glibc function is correctly
// rounded, so CUDA's exp/tanh agree with them only to ~1 ulp; these ports
// make the exact leg bit-identical by construction.  They follow the x86-64
// FMA ifunc builds this image's libm selects on FMA hosts, with the
// contraction pattern read off the binary (tools/extract_libm_exp.py):
//
//   glibc_exp    sysdeps/ieee754/dbl-64/e_exp.c as __exp_fma (libm 0x79b60)
//   glibc_expm1  fdlibm s_expm1.c as __expm1_fma (libm 0x7ac30)
//   glibc_tanh   fdlibm s_tanh.c (libm 0x31620, SSE2: no contraction) over glibc_expm1
//
// All other operations are single IEEE operations (fadd/fmul/fdiv, no
// contraction on either side).  Checked against the host libm bit for bit at
// context creation (self_test) and in tests/test_host.py.
#pragma once

#include "glibc_exp_data.h"
#include "ts_core.cuh"

namespace ts {

#ifdef __CUDACC__
__device__ uint64_t d_exp_tab[TS_EXP_NTAB];
#endif

TS_HD uint64_t exp_tab(int i) {
#ifdef __CUDA_ARCH__
  return __ldg(reinterpret_cast<const unsigned long long*>(d_exp_tab) + i);
#else
  return ts_exp_tab_bits[i];
#endif
}

// e_exp.c specialcase (tmp, sbits, ki) for |x| in [512, 1024): scale may
// overflow or land in the subnormal range (libm 0x79c60)
TS_HD double glibc_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {  // k > 0, the exponent of scale may overflow
    sbits -= 1009ull << 52;
    const double scale = as_double(sbits);
    return fmul(as_double(TS_EXP_TWO_1009_BITS), ffma(scale, tmp, scale));
  }
  // k < 0, subnormal results need special care
  sbits += 1022ull << 52;
  const double scale = as_double(sbits);
  const double st = fmul(scale, tmp);
  double y = fadd(scale, st);
  if (1.0 > y) {
    const double hi = fadd(y, 1.0);
    const double lo = fadd(fsub(scale, y), st);
    y = fsub(fadd(fadd(fadd(fsub(1.0, hi), y), lo), hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return fmul(as_double(TS_EXP_TWO_M1022_BITS), y);
}

TS_HD double glibc_exp(double x) {
  const uint64_t ux = as_u64(x);
  uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ffu;
  if (abstop - 0x3c9u > 0x3eu) {  // |x| < 2^-54, |x| >= 512, or not finite
    if ((int32_t)(abstop - 0x3c9u) < 0) return fadd(x, 1.0);  // tiny: 1 + x
    if (abstop > 0x408u) {  // |x| >= 1024
      if (ux == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return fadd(x, 1.0);
      return (ux >> 63) ? 0.0 : as_double(0x7ff0000000000000ull);  // __math_uflow / __math_oflow
    }
    abstop = 0;  // large |x|: the special case below
  }
  const double kds = ffma(x, as_double(TS_EXP_INVLN2N_BITS), as_double(TS_EXP_SHIFT_BITS));
  const uint64_t ki = as_u64(kds);
  const double kd = fsub(kds, as_double(TS_EXP_SHIFT_BITS));
  double r = ffma(kd, as_double(TS_EXP_NEGLN2HIN_BITS), x);
  r = ffma(kd, as_double(TS_EXP_NEGLN2LON_BITS), r);
  const int idx = 2 * (int)(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = as_double(exp_tab(idx));
  const uint64_t sbits = exp_tab(idx + 1) + top;
  const double p1 = ffma(r, as_double(TS_EXP_C3_BITS), as_double(TS_EXP_C2_BITS));
  const double t0 = fadd(r, tail);
  const double r2 = fmul(r, r);
  const double p2 = ffma(r, as_double(TS_EXP_C5_BITS), as_double(TS_EXP_C4_BITS));
  const double t1 = ffma(p1, r2, t0);
  const double r4 = fmul(r2, r2);
  const double tmp = ffma(r4, p2, t1);
  if (abstop == 0) return glibc_exp_special(tmp, sbits, ki);
  const double scale = as_double(sbits);
  return ffma(scale, tmp, scale);
}

// high word of y + (k << 20) (fdlibm SET_HIGH_WORD(y, high + (k << 20)))
TS_HD double add_exponent(double y, int k) {
  const uint64_t u = as_u64(y);
  const uint32_t hi = (uint32_t)(u >> 32) + ((uint32_t)k << 20);
  return as_double(((uint64_t)hi << 32) | (u & 0xffffffffull));
}

TS_HD double glibc_expm1(double x) {
  const uint64_t ux = as_u64(x);
  const uint32_t hx = (uint32_t)(ux >> 32) & 0x7fffffffu;
  const bool neg = (ux >> 63) != 0;
  double hi = 0.0, lo = 0.0, c = 0.0;
  int k = 0;
  if (hx > 0x40436879u) {  // |x| >= 56 ln2
    if (hx > 0x40862e41u) {  // |x| >= 709.78
      if (hx > 0x7fefffffu) {
        if (((hx & 0xfffffu) | (uint32_t)ux) != 0) return fadd(x, x);  // NaN
        return neg ? -1.0 : x;
      }
      if (x > 709.782712893384) return as_double(0x7ff0000000000000ull);  // overflow
    }
    if (neg) return fsub(as_double(TS_TANH_TINY_BITS), 1.0);  // tiny - one = -1
  }
  if (hx > 0x3fd62e42u) {  // |x| > 0.5 ln2: argument reduction
    if (hx < 0x3ff0a2b2u) {  // and |x| < 1.5 ln2
      if (!neg) {
        hi = fsub(x, as_double(TS_EM1_LN2_HI_BITS));
        lo = as_double(TS_EM1_LN2_LO_BITS);
        k = 1;
      } else {
        hi = fadd(x, as_double(TS_EM1_LN2_HI_BITS));
        lo = -as_double(TS_EM1_LN2_LO_BITS);
        k = -1;
      }
    } else {
      k = (int)fadd(neg ? -0.5 : 0.5, fmul(x, as_double(TS_EM1_INVLN2_BITS)));  // truncation
      const double t = (double)k;
      hi = ffma(-t, as_double(TS_EM1_LN2_HI_BITS), x);  // x - t ln2_hi, fused
      lo = fmul(t, as_double(TS_EM1_LN2_LO_BITS));
    }
    x = fsub(hi, lo);
    c = fsub(fsub(hi, x), lo);
  } else if (hx < 0x3c900000u) {  // |x| < 2^-54: x
    return x;
  }
  // x in the primary range
  const double hfx = fmul(x, 0.5);
  const double hxs = fmul(x, hfx);
  const double R2 = ffma(hxs, as_double(TS_EM1_Q3_BITS), as_double(TS_EM1_Q2_BITS));
  const double R3 = ffma(hxs, as_double(TS_EM1_Q5_BITS), as_double(TS_EM1_Q4_BITS));
  const double h2 = fmul(hxs, hxs);
  const double R1 = ffma(hxs, as_double(TS_EM1_Q1_BITS), 1.0);
  const double h4 = fmul(h2, h2);
  const double r1 = ffma(h4, R3, ffma(h2, R2, R1));
  double t = ffma(-r1, hfx, 3.0);
  double e = fmul(fdiv(fsub(r1, t), ffma(-x, t, 6.0)), hxs);
  if (k == 0) return fsub(x, ffma(e, x, -hxs));  // x - (x e - hxs), c = 0
  e = ffma(fsub(e, c), x, -c);                      // x (e - c) - c
  e = fsub(e, hxs);
  if (k == -1) return ffma(0.5, fsub(x, e), -0.5);  // 0.5 (x - e) - 0.5
  if (k == 1) {
    if (x < -0.25) return fmul(fsub(e, fadd(x, 0.5)), -2.0);
    return ffma(fsub(x, e), 2.0, 1.0);              // 1 + 2 (x - e)
  }
  if (k <= -2 || k > 56) {  // exp(x) - 1 from y = 1 - (e - x) scaled by 2^k
    const double y = fsub(1.0, fsub(e, x));
    return fsub(add_exponent(y, k), 1.0);
  }
  if (k < 20) {
    t = as_double((uint64_t)(0x3ff00000u - (0x200000u >> k)) << 32);  // 1 - 2^-k
    return add_exponent(fsub(t, fsub(e, x)), k);
  }
  t = as_double((uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);  // 2^-k
  return add_exponent(fadd(fsub(x, fadd(e, t)), 1.0), k);
}

TS_HD double glibc_tanh(double x) {
  const uint64_t ux = as_u64(x);
  const uint32_t jx = (uint32_t)(ux >> 32), ix = jx & 0x7fffffffu;
  const bool neg = (int32_t)jx < 0;
  if (ix > 0x7fefffffu) return neg ? fsub(fdiv(1.0, x), 1.0) : fadd(fdiv(1.0, x), 1.0);  // inf, NaN
  double z;
  if (ix > 0x4035ffffu) {  // |x| >= 22
    z = fsub(1.0, as_double(TS_TANH_TINY_BITS));
  } else {
    if ((ix | (uint32_t)ux) == 0) return x;  // +-0
    const double ax = as_double(ux & 0x7fffffffffffffffull);
    if (ix <= 0x3c7fffffu) return fmul(x, fadd(1.0, x));  // |x| < 2^-55
    if (ix > 0x3fefffffu) {                               // |x| >= 1
      const double t = glibc_expm1(fadd(ax, ax));
      z = fsub(1.0, fdiv(2.0, fadd(t, 2.0)));
    } else {
      const double t = glibc_expm1(fmul(ax, -2.0));
      z = fdiv(-t, fadd(t, 2.0));
    }
  }
  return neg ? -z : z;
}

// glibc_tanh without divergent branches, for the latency-bound exact LSTM
// kernels (a warp's lanes straddle |x| = 1 every timestep, and the branchy
// form then runs both halves, each with its own expm1 and division).  The two
// tanh forms call expm1 on 2|x| or -2|x|, so ONE expm1 evaluation with the
// argument, the reduction constants and the final assembly chosen per lane
// by selects performs exactly the operations the branchy code performs for
// that lane: bit-identical to glibc_tanh (checked at context creation and in
// tests/test_host.py).  Argument reduction: case 0.5 ln2 < |a| < 1.5 ln2 is
// the general reduction with k forced to +-1 (x - ln2_hi == fma(-1, ln2_hi, x),
// 1 * ln2_lo == ln2_lo); |a| <= 0.5 ln2 is k = 0 without reduction.  expm1's
// own special cases (|a| >= 56 ln2 negative, >= 709.78, |a| < 2^-54) cannot be
// reached from tanh: a = 2|x| in [2, 44) or -2|x| in (-2, -2^-54].
TS_HD double sel(bool p, double a, double b) { return p ? a : b; }

TS_HD double glibc_tanh_bf(double x) {
  const uint64_t ux = as_u64(x);
  const uint32_t ix = (uint32_t)(ux >> 32) & 0x7fffffffu;
  const double ax = as_double(ux & 0x7fffffffffffffffull);
  const bool big = ix > 0x3fefffffu;  // |x| >= 1: tanh = 1 - 2 / (expm1(2|x|) + 2)
  // ---- expm1(a), a = 2|x| or -2|x|
  const double a = big ? fadd(ax, ax) : fmul(ax, -2.0);
  const uint32_t ha = (uint32_t)(as_u64(a) >> 32) & 0x7fffffffu;
  const bool an = !big;               // a < 0
  const bool red = ha > 0x3fd62e42u;  // |a| > 0.5 ln2: reduce
  const bool k1 = ha < 0x3ff0a2b2u;   //   and |a| < 1.5 ln2: k = +-1
  int k = (int)fadd(an ? -0.5 : 0.5, fmul(a, as_double(TS_EM1_INVLN2_BITS)));
  k = red ? (k1 ? (an ? -1 : 1) : k) : 0;
  const double t = (double)k;
  const double hi = ffma(-t, as_double(TS_EM1_LN2_HI_BITS), a);
  const double lo = fmul(t, as_double(TS_EM1_LN2_LO_BITS));
  const double xr = red ? fsub(hi, lo) : a;
  const double c = red ? fsub(fsub(hi, xr), lo) : 0.0;
  const double hfx = fmul(xr, 0.5);
  const double hxs = fmul(xr, hfx);
  const double R2 = ffma(hxs, as_double(TS_EM1_Q3_BITS), as_double(TS_EM1_Q2_BITS));
  const double R3 = ffma(hxs, as_double(TS_EM1_Q5_BITS), as_double(TS_EM1_Q4_BITS));
  const double h2 = fmul(hxs, hxs);
  const double R1 = ffma(hxs, as_double(TS_EM1_Q1_BITS), 1.0);
  const double h4 = fmul(h2, h2);
  const double r1 = ffma(h4, R3, ffma(h2, R2, R1));
  const double tt = ffma(-r1, hfx, 3.0);
  const double e = fmul(fdiv(fsub(r1, tt), ffma(-xr, tt, 6.0)), hxs);
  const double e2 = fsub(ffma(fsub(e, c), xr, -c), hxs);
  // expm1(a): every lane evaluates the k = 0, +-1 and |k| >= 2 assemblies
  // and keeps its own (no divergence)
  const double ek = fsub(e2, xr);  // e - x
  const bool wide = k <= -2 || k > 56;
  const bool small = k < 20;
  const double tk = as_double(small ? (uint64_t)(0x3ff00000u - (0x200000u >> (k & 31))) << 32
                                    : (uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
  const double ya = wide ? fsub(1.0, ek) : (small ? fsub(tk, ek) : fadd(fsub(xr, fadd(e2, tk)), 1.0));
  const double ys = add_exponent(ya, k);
  double em = wide ? fsub(ys, 1.0) : ys;
  em = sel(k == -1, ffma(0.5, fsub(xr, e2), -0.5), em);
  em = sel(k == 1, sel(xr < -0.25, fmul(fsub(e2, fadd(xr, 0.5)), -2.0), ffma(fsub(xr, e2), 2.0, 1.0)), em);
  em = sel(k == 0, fsub(xr, ffma(e, xr, -hxs)), em);
  // ---- tanh
  const double q = fdiv(big ? 2.0 : -em, fadd(em, 2.0));
  double z = big ? fsub(1.0, q) : q;
  z = sel(ix > 0x4035ffffu, fsub(1.0, as_double(TS_TANH_TINY_BITS)), z);  // |x| >= 22
  z = (ux >> 63) ? -z : z;
  z = sel(ix <= 0x3c7fffffu, fmul(x, fadd(1.0, x)), z);  // |x| < 2^-55 (and +-0: x (1 + x) = x)
  if (ix > 0x7fefffffu) z = glibc_tanh(x);               // inf, NaN
  return z;
}

// the Cython kernel's sigmoid, 1 / (1 + exp(-x)) (_recurrent_cy.pyx:17-18)
TS_HD double glibc_sigmoid(double x) { return fdiv(1.0, fadd(1.0, glibc_exp(-x))); }

}  // namespace ts
