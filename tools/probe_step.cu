// Dependent latencies of the exact LSTM step's pieces on the B200 (one warp,
// clock64): fp64 add/fma chains, the glibc exp / sigmoid / branch-free tanh
// ports, a correctly rounded division, and one full k_children_exact_mw-style
// step chain (32 h terms -> tanh gate -> c -> tanh(c) -> h) without the
// barrier.  Tells how far the greedy's per-step time is from its latency floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -I paper_2011_14486_b200/csrc -o tools/probe_step.bin tools/probe_step.cu
#include <cstdio>

#include "ts_glibc_math.cuh"

using namespace ts;

// glibc_tanh_bf with its constants read from the constant bank (same
// operations, so the same bits) - does ptxas's immediate handling (UMOV
// pairs into uniform registers before each use) cost latency?
__constant__ double kc[12];
enum { C_INVLN2, C_LN2HI, C_LN2LO, C_Q1, C_Q2, C_Q3, C_Q4, C_Q5, C_TINY };
__device__ __forceinline__ double tanh_cb(double x) {
  const uint64_t ux = as_u64(x);
  const uint32_t ix = (uint32_t)(ux >> 32) & 0x7fffffffu;
  const double ax = as_double(ux & 0x7fffffffffffffffull);
  const bool big = ix > 0x3fefffffu;
  const double a = big ? ts::fadd(ax, ax) : ts::fmul(ax, -2.0);
  const uint32_t ha = (uint32_t)(as_u64(a) >> 32) & 0x7fffffffu;
  const bool an = !big;
  const bool red = ha > 0x3fd62e42u;
  const bool k1 = ha < 0x3ff0a2b2u;
  int k = (int)ts::fadd(an ? -0.5 : 0.5, ts::fmul(a, kc[C_INVLN2]));
  k = red ? (k1 ? (an ? -1 : 1) : k) : 0;
  const double t = (double)k;
  const double hi = ts::ffma(-t, kc[C_LN2HI], a);
  const double lo = ts::fmul(t, kc[C_LN2LO]);
  const double xr = red ? ts::fsub(hi, lo) : a;
  const double c = red ? ts::fsub(ts::fsub(hi, xr), lo) : 0.0;
  const double hfx = ts::fmul(xr, 0.5);
  const double hxs = ts::fmul(xr, hfx);
  const double R2 = ts::ffma(hxs, kc[C_Q3], kc[C_Q2]);
  const double R3 = ts::ffma(hxs, kc[C_Q5], kc[C_Q4]);
  const double h2 = ts::fmul(hxs, hxs);
  const double R1 = ts::ffma(hxs, kc[C_Q1], 1.0);
  const double h4 = ts::fmul(h2, h2);
  const double r1 = ts::ffma(h4, R3, ts::ffma(h2, R2, R1));
  const double tt = ts::ffma(-r1, hfx, 3.0);
  const double e = ts::fmul(ts::fdiv(ts::fsub(r1, tt), ts::ffma(-xr, tt, 6.0)), hxs);
  const double e2 = ts::fsub(ts::ffma(ts::fsub(e, c), xr, -c), hxs);
  const double ek = ts::fsub(e2, xr);
  const bool wide = k <= -2 || k > 56;
  const bool small = k < 20;
  const double tk = as_double(small ? (uint64_t)(0x3ff00000u - (0x200000u >> (k & 31))) << 32
                                    : (uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
  const double ya = wide ? ts::fsub(1.0, ek) : (small ? ts::fsub(tk, ek) : ts::fadd(ts::fsub(xr, ts::fadd(e2, tk)), 1.0));
  const double ys = add_exponent(ya, k);
  double em = wide ? ts::fsub(ys, 1.0) : ys;
  em = sel(k == -1, ts::ffma(0.5, ts::fsub(xr, e2), -0.5), em);
  em = sel(k == 1, sel(xr < -0.25, ts::fmul(ts::fsub(e2, ts::fadd(xr, 0.5)), -2.0), ts::ffma(ts::fsub(xr, e2), 2.0, 1.0)), em);
  em = sel(k == 0, ts::fsub(xr, ts::ffma(e, xr, -hxs)), em);
  const double q = ts::fdiv(big ? 2.0 : -em, ts::fadd(em, 2.0));
  double z = big ? ts::fsub(1.0, q) : q;
  z = sel(ix > 0x4035ffffu, ts::fsub(1.0, kc[C_TINY]), z);
  z = (ux >> 63) ? -z : z;
  z = sel(ix <= 0x3c7fffffu, ts::fmul(x, ts::fadd(1.0, x)), z);
  return z;
}

// tanh_cb with t = trunc(v) formed in fp64 (round-to-nearest by the 1.5 * 2^52
// shift, then a step toward zero) instead of F2I + I2F on the chain; k for
// the later selects still comes from F2I, off the chain
__device__ __forceinline__ double tanh_tr(double x) {
  const uint64_t ux = as_u64(x);
  const uint32_t ix = (uint32_t)(ux >> 32) & 0x7fffffffu;
  const double ax = as_double(ux & 0x7fffffffffffffffull);
  const bool big = ix > 0x3fefffffu;
  const double a = big ? ts::fadd(ax, ax) : ts::fmul(ax, -2.0);
  const uint32_t ha = (uint32_t)(as_u64(a) >> 32) & 0x7fffffffu;
  const bool an = !big;
  const bool red = ha > 0x3fd62e42u;
  const bool k1 = ha < 0x3ff0a2b2u;
  const double v = ts::fadd(an ? -0.5 : 0.5, ts::fmul(a, kc[C_INVLN2]));
  const double rn = ts::fsub(ts::fadd(v, 6755399441055744.0), 6755399441055744.0);
  const double tr = v >= 0.0 ? (rn > v ? ts::fsub(rn, 1.0) : rn) : (rn < v ? ts::fadd(rn, 1.0) : rn);
  const double t = red ? (k1 ? (an ? -1.0 : 1.0) : tr) : 0.0;
  int k = (int)v;
  k = red ? (k1 ? (an ? -1 : 1) : k) : 0;
  const double hi = ts::ffma(-t, kc[C_LN2HI], a);
  const double lo = ts::fmul(t, kc[C_LN2LO]);
  const double xr = red ? ts::fsub(hi, lo) : a;
  const double c = red ? ts::fsub(ts::fsub(hi, xr), lo) : 0.0;
  const double hfx = ts::fmul(xr, 0.5);
  const double hxs = ts::fmul(xr, hfx);
  const double R2 = ts::ffma(hxs, kc[C_Q3], kc[C_Q2]);
  const double R3 = ts::ffma(hxs, kc[C_Q5], kc[C_Q4]);
  const double h2 = ts::fmul(hxs, hxs);
  const double R1 = ts::ffma(hxs, kc[C_Q1], 1.0);
  const double h4 = ts::fmul(h2, h2);
  const double r1 = ts::ffma(h4, R3, ts::ffma(h2, R2, R1));
  const double tt = ts::ffma(-r1, hfx, 3.0);
  const double e = ts::fmul(ts::fdiv(ts::fsub(r1, tt), ts::ffma(-xr, tt, 6.0)), hxs);
  const double e2 = ts::fsub(ts::ffma(ts::fsub(e, c), xr, -c), hxs);
  const double ek = ts::fsub(e2, xr);
  const bool wide = k <= -2 || k > 56;
  const bool small = k < 20;
  const double tk = as_double(small ? (uint64_t)(0x3ff00000u - (0x200000u >> (k & 31))) << 32
                                    : (uint64_t)((uint32_t)(0x3ff - k) << 20) << 32);
  const double ya = wide ? ts::fsub(1.0, ek) : (small ? ts::fsub(tk, ek) : ts::fadd(ts::fsub(xr, ts::fadd(e2, tk)), 1.0));
  const double ys = add_exponent(ya, k);
  double em = wide ? ts::fsub(ys, 1.0) : ys;
  em = sel(k == -1, ts::ffma(0.5, ts::fsub(xr, e2), -0.5), em);
  em = sel(k == 1, sel(xr < -0.25, ts::fmul(ts::fsub(e2, ts::fadd(xr, 0.5)), -2.0), ts::ffma(ts::fsub(xr, e2), 2.0, 1.0)), em);
  em = sel(k == 0, ts::fsub(xr, ts::ffma(e, xr, -hxs)), em);
  const double q = ts::fdiv(big ? 2.0 : -em, ts::fadd(em, 2.0));
  double z = big ? ts::fsub(1.0, q) : q;
  z = sel(ix > 0x4035ffffu, ts::fsub(1.0, kc[C_TINY]), z);
  z = (ux >> 63) ? -z : z;
  z = sel(ix <= 0x3c7fffffu, ts::fmul(x, ts::fadd(1.0, x)), z);
  return z;
}

__global__ void k_lat(double seed, long long* cyc, double* out) {
  const int lane = threadIdx.x;
  double acc = 0.0;
  long long t0, t1;
  // DADD chain
  double a = seed + lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    a = ts::fadd(a, 1.0000001);
    a = ts::fadd(a, 1.0000001);
    a = ts::fadd(a, 1.0000001);
    a = ts::fadd(a, 1.0000001);
  }
  t1 = clock64();
  if (!lane) cyc[0] = t1 - t0;
  acc += a;
  // DFMA chain
  a = seed + lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    a = ts::ffma(a, 0.9999999, 1e-7);
    a = ts::ffma(a, 0.9999999, 1e-7);
    a = ts::ffma(a, 0.9999999, 1e-7);
    a = ts::ffma(a, 0.9999999, 1e-7);
  }
  t1 = clock64();
  if (!lane) cyc[1] = t1 - t0;
  acc += a;
  // fdiv
  double d = seed + 2.0 + lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) d = ts::fdiv(1.0, ts::fadd(d, 1.0));
  t1 = clock64();
  if (!lane) cyc[2] = t1 - t0;
  acc += d;
  // glibc exp
  double e = 0.3 + lane * 1e-3;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) e = glibc_exp(ts::fmul(e, 0.5));
  t1 = clock64();
  if (!lane) cyc[3] = t1 - t0;
  acc += e;
  // sigmoid
  double s = 0.3 + lane * 1e-3;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) s = glibc_sigmoid(s);
  t1 = clock64();
  if (!lane) cyc[4] = t1 - t0;
  acc += s;
  // tanh_bf (lanes straddle |x| = 1)
  double h = 0.5 + lane * 0.05;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) h = glibc_tanh_bf(ts::fadd(h, 0.7));
  t1 = clock64();
  if (!lane) cyc[5] = t1 - t0;
  acc += h;
  // one step chain: z = 32 sequential h terms, tanh gate, c, tanh(c), h
  __shared__ double hw[32];
  double wh[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) wh[k] = 0.01 * ((k * 7 + lane) % 13 - 6);
  double c = 0.1, hh = 0.05 * lane;
  hw[lane] = hh;
  __syncwarp();
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    double z = 0.1;
#pragma unroll
    for (int k = 0; k < 32; ++k) z = ts::fadd(z, ts::fmul(hw[k], wh[k]));
    const double g = glibc_tanh_bf(z);
    c = ts::fadd(ts::fmul(0.5, c), ts::fmul(0.5, g));
    hh = ts::fmul(0.5, glibc_tanh_bf(c));
    __syncwarp();
    hw[lane] = hh;
    __syncwarp();
  }
  t1 = clock64();
  if (!lane) cyc[6] = t1 - t0;
  acc += hh;
  // tanh_cb
  h = 0.5 + lane * 0.05;
  double hb = h;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) h = tanh_cb(ts::fadd(h, 0.7));
  t1 = clock64();
  if (!lane) cyc[7] = t1 - t0;
  acc += h;
  for (int i = 0; i < 256; ++i) {  // bit-identity check on this lane's sequence
    const double u = glibc_tanh_bf(ts::fadd(hb, 0.7)), v = tanh_cb(ts::fadd(hb, 0.7));
    if (as_u64(u) != as_u64(v)) cyc[8] = 1;
    hb = ts::fadd(u, -0.37 + 0.01 * i);
  }
  // tanh_tr
  h = 0.5 + lane * 0.05;
  hb = h;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) h = tanh_tr(ts::fadd(h, 0.7));
  t1 = clock64();
  if (!lane) cyc[9] = t1 - t0;
  acc += h;
  for (int i = 0; i < 4096; ++i) {
    const double xx = ts::fmul(ts::fadd(hb, -0.5), 12.0 + lane);
    const double u = glibc_tanh_bf(xx), v = tanh_tr(xx);
    if (as_u64(u) != as_u64(v)) cyc[10] = 1;
    hb = ts::fadd(u * 0.5 + 0.5, 0.001 * (i % 7));
  }
  // F2I + I2F chain
  double cv = 3.7 + lane;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) cv = (double)(int)ts::fadd(cv, 0.6);
  t1 = clock64();
  if (!lane) cyc[11] = t1 - t0;
  acc += cv;
  out[lane] = acc;
}

// The greedy step's structure: four warps, warp g one gate, a block barrier
// per step (k_children_exact_mw) ...
__global__ void k_step4(long long* cyc, double* out, int steps) {
  const int g = threadIdx.x >> 5, j = threadIdx.x & 31;
  __shared__ double hw[4][2][32], abuf[2][4][32];
  double wh[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) wh[k] = 0.01 * ((k * 7 + j + g) % 13 - 6);
  double c = 0.1;
  hw[g][0][j] = 0.05 * j;
  __syncthreads();
  int cur = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int t = 0; t < steps; ++t) {
    double z = 0.1;
#pragma unroll
    for (int k = 0; k < 32; ++k) z = ts::fadd(z, ts::fmul(hw[g][cur][k], wh[k]));
    abuf[cur][g][j] = g == 2 ? glibc_tanh_bf(z) : glibc_sigmoid(z);
    __syncthreads();
    c = ts::fadd(ts::fmul(abuf[cur][1][j], c), ts::fmul(abuf[cur][0][j], abuf[cur][2][j]));
    const double h = ts::fmul(abuf[cur][3][j], glibc_tanh_bf(c));
    hw[g][cur ^ 1][j] = h;
    __syncwarp();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = c;
}

// ... against one warp doing all four gates of its 32 units (four
// interleaved z chains, the recurrent weights in shared memory), no barrier
__global__ void k_step1(long long* cyc, double* out, int steps) {
  const int j = threadIdx.x & 31;
  __shared__ double W[32][128];
  __shared__ double hw[2][32];
  for (int e = j; e < 32 * 128; e += 32) W[e / 128][e % 128] = 0.01 * ((e * 7) % 13 - 6);
  double c = 0.1;
  hw[0][j] = 0.05 * j;
  __syncwarp();
  int cur = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int t = 0; t < steps; ++t) {
    double z0 = 0.1, z1 = 0.1, z2 = 0.1, z3 = 0.1;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double hk = hw[cur][k];
      z0 = ts::fadd(z0, ts::fmul(hk, W[k][j]));
      z1 = ts::fadd(z1, ts::fmul(hk, W[k][32 + j]));
      z2 = ts::fadd(z2, ts::fmul(hk, W[k][64 + j]));
      z3 = ts::fadd(z3, ts::fmul(hk, W[k][96 + j]));
    }
    const double gi = glibc_sigmoid(z0), gf = glibc_sigmoid(z1), gg = glibc_tanh_bf(z2), go = glibc_sigmoid(z3);
    c = ts::fadd(ts::fmul(gf, c), ts::fmul(gi, gg));
    const double h = ts::fmul(go, glibc_tanh_bf(c));
    hw[cur ^ 1][j] = h;
    __syncwarp();
    cur ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[1] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = c;
}

int main() {
  long long* cyc;
  double* out;
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMemcpyToSymbol(d_exp_tab, ts_exp_tab_bits, sizeof(uint64_t) * TS_EXP_NTAB);
  const uint64_t kb[9] = {TS_EM1_INVLN2_BITS, TS_EM1_LN2_HI_BITS, TS_EM1_LN2_LO_BITS, TS_EM1_Q1_BITS, TS_EM1_Q2_BITS,
                          TS_EM1_Q3_BITS, TS_EM1_Q4_BITS, TS_EM1_Q5_BITS, TS_TANH_TINY_BITS};
  cudaMemcpyToSymbol(kc, kb, sizeof kb);
  cyc[8] = 0;
  cyc[10] = 0;
  for (int r = 0; r < 3; ++r) k_lat<<<1, 32>>>(1.0, cyc, out);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 1;
  }
  long long* c2;
  cudaMallocManaged(&c2, 4 * sizeof(long long));
  double* o2;
  cudaMalloc(&o2, 64 * 128 * sizeof(double));
  for (int nb : {1, 40}) {
    for (int r = 0; r < 3; ++r) {
      k_step4<<<nb, 128>>>(c2, o2, 128);
      k_step1<<<nb, 32>>>(c2, o2, 128);
    }
    cudaDeviceSynchronize();
    printf("%d blocks: 4-warp step %.1f cycles, 1-warp all-gates step %.1f cycles\n", nb, c2[0] / 128.0,
           c2[1] / 128.0);
  }
  printf("DADD          %.1f cycles\n", cyc[0] / 1024.0);
  printf("DFMA          %.1f cycles\n", cyc[1] / 1024.0);
  printf("fdiv + DADD   %.1f cycles\n", cyc[2] / 256.0);
  printf("glibc_exp+DMUL %.1f cycles\n", cyc[3] / 256.0);
  printf("sigmoid       %.1f cycles\n", cyc[4] / 256.0);
  printf("tanh_bf+DADD  %.1f cycles\n", cyc[5] / 256.0);
  printf("tanh_cb+DADD  %.1f cycles (constant bank), mismatches %lld\n", cyc[7] / 256.0, cyc[8]);
  printf("tanh_tr+DADD  %.1f cycles (fp64 trunc), mismatches %lld\n", cyc[9] / 256.0, cyc[10]);
  printf("F2I+I2F+DADD  %.1f cycles\n", cyc[11] / 256.0);
  printf("step chain    %.1f cycles (no barrier)\n", cyc[6] / 64.0);
  return 0;
}
