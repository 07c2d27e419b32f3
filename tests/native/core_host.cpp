// TEST INFRASTRUCTURE ONLY: host build of ts_core.cuh (the integer nest math,
// u256, correctly rounded conversions and the glibc-log2 port shared with the
// sm_100a kernels) so the CPU suite can check it against the reference's
// golden feature matrices without a GPU.  Never linked into the product.
#include <cstring>
#include <vector>

#include "../../paper_2011_14486_b200/csrc/ts_core.cuh"

using namespace ts;

extern "C" int core_featurize(const int64_t* desc, int64_t n_words, const ts_decision* rec,
                              const int64_t* offsets, int64_t n, double* out) {
  static PipelineDesc P;
  memset(&P, 0, sizeof P);
  const int T = (int)desc[1];
  P.n_stages = T;
  P.n_slots = (int)desc[2];
  for (int s = 0; s < T; ++s) {
    const int64_t* w = desc + 4 + 48 * s;
    StageDesc& sd = P.st[s];
    sd.n_pure = (int)w[0];
    sd.n_red = (int)w[1];
    for (int k = 0; k < 8; ++k) sd.ext[k] = w[2 + k];
    sd.pure_points = w[10]; sd.red_points = w[11]; sd.domain_points = w[12];
    sd.i_points = w[13]; sd.i_flops = w[14]; sd.i_in_bytes = w[15]; sd.i_out_bytes = w[16];
    sd.n_inputs = (int)w[17]; sd.ov_window = (int)w[18]; sd.ov_stride = (int)w[19];
    sd.consumer = (int)w[20]; sd.n_cedges = (int)w[21];
    for (int e = 0; e < 2; ++e)
      for (int k = 0; k < 4; ++k) {
        sd.cdim[e][k] = (int)w[22 + 4 * e + k];
        sd.cstride[e][k] = w[30 + 4 * e + k];
        sd.cwindow[e][k] = w[38 + 4 * e + k];
      }
    sd.slot = (int)w[46];
    sd.dp = make_divisor(sd.domain_points);
    sd.io = make_divisor(1 + sd.i_in_bytes + sd.i_out_bytes);
  }
  for (int64_t i = 0; i < n; ++i) {
    double* o = out + i * T * 16;
    for (int s = 0; s < T; ++s) {
      intrinsic_features(P.st[s], o + s * 16);
      for (int k = 8; k < 16; ++k) o[s * 16 + k] = 0.0;
    }
    std::vector<Nest> slots(16);
    const int d = (int)(offsets[i + 1] - offsets[i]);
    for (int j = 0; j < d; ++j) {
      const int s = T - 1 - j;
      const StageDesc& sd = P.st[s];
      const ts_decision& dec = rec[offsets[i] + j];
      const StageDesc* cs = dec.anchor >= 0 ? &P.st[sd.consumer] : nullptr;
      const Nest* cn = dec.anchor >= 0 ? &slots[cs->slot] : nullptr;
      Nest nn;
      int64_t pe[TS_MAX_PURE];
      int rc = build_nest(sd, cs, cn, dec, nn, pe);
      if (!rc) rc = acquired_features(sd, nn, pe, dec, o + s * 16 + 8);
      if (rc) return rc;
      if (sd.slot >= 0) slots[sd.slot] = nn;
    }
  }
  return 0;
}

extern "C" double core_log2(double x) { return glibc_log2(x); }

extern "C" double core_div(const uint64_t* n4, uint64_t d) {
  u256 a;
  for (int i = 0; i < 4; ++i) a.w[i] = n4[i];
  return u256_div_to_double(a, make_divisor(d));
}

extern "C" double core_to_double(const uint64_t* n4) {
  u256 a;
  for (int i = 0; i < 4; ++i) a.w[i] = n4[i];
  return u256_to_double(a);
}

extern "C" double core_div128(uint64_t lo, uint64_t hi, uint64_t d) {
  return div128_to_double(((unsigned __int128)hi << 64) | lo, make_divisor(d));
}

// f15 = log2(1 + inv) through acquired_features' conversion paths
extern "C" double core_log2_1p(uint64_t lo, uint64_t hi) {
  StageDesc s;
  memset(&s, 0, sizeof s);
  s.n_pure = 1;
  s.ext[0] = 1;
  s.pure_points = 1;
  s.red_points = 1;
  s.domain_points = 1;
  s.dp = make_divisor(1);
  Nest n;
  memset(&n, 0, sizeof n);
  n.inv.w[0] = lo;
  n.inv.w[1] = hi;
  n.n_loops = 1;
  n.ext[0] = 1;
  ts_decision d;
  memset(&d, 0, sizeof d);
  d.vec = 1;
  int64_t pe[4] = {1, 1, 1, 1};
  double f[8];
  if (acquired_features(s, n, pe, d, f)) return -1.0;
  return f[7];
}

#include "../../paper_2011_14486_b200/csrc/ts_glibc_math.cuh"

extern "C" void core_exp_tanh(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    out[2 * i] = glibc_exp(x[i]);
    out[2 * i + 1] = glibc_tanh(x[i]);
  }
}

extern "C" void core_tanh_bf(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = glibc_tanh_bf(x[i]);
}
