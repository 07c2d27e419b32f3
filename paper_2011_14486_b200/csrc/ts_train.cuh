// ts_train.cuh - V training on the B200.
//
// value_model.gradients (value_model.py:182-210) = per-sequence
// lstm_forward_cached + lstm_backward (_recurrent_np.py:38-96) summed over the
// minibatch, then _clip (:213-220) and the SGD update (:267-271).  fp64
// throughout so the device trajectory tracks the reference's (the training
// loop is contractive: 1e-12 perturbations stay ~1e-13).
//
// Dataset layout: a sample is (rows, init, T, d): its input at timestep t is
// init[init_base + t] for t < T - d (unscheduled stages) and
// rows[row_base + (T - 1 - t)] otherwise (the scheduled stages' rows in
// decision order).  All prefixes of one complete schedule share its rows,
// so a bootstrap-style dataset of T+1 prefixes per schedule stores T rows.
//
//   k_train_fb     warp per sequence, lane per hidden unit: forward with the
//                  activation cache, d_raw = 2(raw + ts - log t)/n_total (or
//                  the caller's d_raw: backend.lstm_backward),
//                  BPTT; writes dz[b][t][4H] and keeps h_prev/h in the cache
//   k_train_wgrad  split-K weight gradients: block (p-tile, k-split) sums its
//                  (t, b) range in a fixed order into partials
//   k_train_reduce partials summed in split order -> grad
//   k_train_apply  one block: global L2 norm incl. b_out, clip, p -= lr g
//   k_train_fwd    warp per sequence: raw for _eval_split
//
// The gradient buffer is a plain device array between k_train_reduce and
// k_train_apply, so data-parallel training all-reduces it (NCCL) in between.
#pragma once

#include <cuda_runtime.h>

#include "ts_core.cuh"
#include "ts_lstm_tc.cuh"

namespace ts {
namespace tr {

constexpr int F = TS_FEATURE_WIDTH;

struct Layout {  // offsets into the flat parameter / gradient vector
  int H, G, oWx, oWh, ob, ow, obout, n;
  __host__ __device__ explicit Layout(int h)
      : H(h), G(4 * h), oWx(0), oWh(16 * 4 * h), ob(16 * 4 * h + h * 4 * h),
        ow(16 * 4 * h + h * 4 * h + 4 * h), obout(16 * 4 * h + h * 4 * h + 4 * h + h),
        n(16 * 4 * h + h * 4 * h + 4 * h + h + 1) {}
};

// cache per (sequence, timestep): i, f, g, o, c_prev, h_prev, tc, h  (x H)
constexpr int CACHE_FIELDS = 8;

__device__ __forceinline__ double sig(double x) { return fdiv(1.0, fadd(1.0, exp(-x))); }

struct Data {
  const double* rows;       // [n_rows][16] normalized
  const double* init;       // [n_init][16] normalized
  const int64_t* row_base;  // [N]
  const int32_t* init_base; // [N]
  const int32_t* Tlen;      // [N]
  const int32_t* depth;     // [N]
  const double* logt;       // [N]
  __device__ __forceinline__ const double* x(int64_t i, int t) const {
    const int T = Tlen[i], d = depth[i];
    return t < T - d ? init + (int64_t)(init_base[i] + t) * F : rows + (row_base[i] + (T - 1 - t)) * F;
  }
};

struct TrainArgs {
  Data D;
  const int* batch;     // [B] dataset indices
  const double* P;      // params
  double* cache;        // [B][Tmax][8][H]
  double* dz;           // [B][Tmax][4H]  (grouped kernels: packed pair rows, below)
  uint8_t* pvalid;      // grouped kernels: [Tmax * B] pair valid flags
  double* draw;         // [B]
  double* raw;          // [B]
  int B, Tmax, H;
  double target_scale;
  double n_total;       // global minibatch size n (value_model.py:193)
  double* partial;      // tensor-core weight gradients: [gridDim.x][n_params] per-CTA sums
  const double* draw_in;  // optional [B]: d_raw given by the caller (lstm_backward), else the loss's
};

__global__ void k_train_fb(TrainArgs a) {
  const int wb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wb >= a.B) return;
  const Layout L(a.H);
  const int H = a.H, G = L.G;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  const int idx = a.batch[wb];
  const int T = a.D.Tlen[idx];
  const double* Wx = a.P + L.oWx;
  const double* Wh = a.P + L.oWh;
  const double* bb = a.P + L.ob;
  const double* w = a.P + L.ow;
  double* cache = a.cache + (int64_t)wb * a.Tmax * CACHE_FIELDS * H;
  double h = 0.0, c = 0.0;
  double raw = fmul((double)T, a.P[L.obout]);
  // ---- forward with cache (_recurrent_np.py:38-59)
  for (int t = 0; t < T; ++t) {
    const double* X = a.D.x(idx, t);
    double zi = bb[j], zf = bb[H + j], zg = bb[2 * H + j], zo = bb[3 * H + j];
    for (int k = 0; k < F; ++k) {
      const double xv = X[k];
      const double* wr = Wx + k * G;
      zi = fadd(zi, fmul(xv, wr[j]));
      zf = fadd(zf, fmul(xv, wr[H + j]));
      zg = fadd(zg, fmul(xv, wr[2 * H + j]));
      zo = fadd(zo, fmul(xv, wr[3 * H + j]));
    }
    for (int k = 0; k < H; ++k) {
      const double hv = __shfl_sync(0xffffffffu, h, k);
      const double* wr = Wh + k * G;
      zi = fadd(zi, fmul(hv, wr[j]));
      zf = fadd(zf, fmul(hv, wr[H + j]));
      zg = fadd(zg, fmul(hv, wr[2 * H + j]));
      zo = fadd(zo, fmul(hv, wr[3 * H + j]));
    }
    double prod = 0.0;
    if (act) {
      const double gi = sig(zi), gf = sig(zf), gg = tanh(zg), go = sig(zo);
      const double c_prev = c, h_prev = h;
      c = fadd(fmul(gf, c), fmul(gi, gg));
      const double tc = tanh(c);
      h = fmul(go, tc);
      double* cc = cache + (int64_t)t * CACHE_FIELDS * H;
      cc[0 * H + j] = gi;
      cc[1 * H + j] = gf;
      cc[2 * H + j] = gg;
      cc[3 * H + j] = go;
      cc[4 * H + j] = c_prev;
      cc[5 * H + j] = h_prev;
      cc[6 * H + j] = tc;
      cc[7 * H + j] = h;
      prod = fmul(h, w[j]);
    }
    double acc = 0.0;
    for (int k = 0; k < H; ++k) acc = fadd(acc, __shfl_sync(0xffffffffu, prod, k));
    raw = fadd(raw, acc);
  }
  // d_raw = 2 (raw + ts - log t) / n  (value_model.py:201)
  const double d_raw = a.draw_in ? a.draw_in[wb]
                                 : fdiv(fmul(2.0, fsub(fadd(raw, a.target_scale), a.D.logt[idx])), a.n_total);
  if (lane == 0) {
    a.raw[wb] = raw;
    a.draw[wb] = d_raw;
  }
  // ---- BPTT (_recurrent_np.py:62-96)
  double dh_next = 0.0, dc_next = 0.0;
  double* dzb = a.dz + (int64_t)wb * a.Tmax * G;
  for (int t = T - 1; t >= 0; --t) {
    const double* cc = cache + (int64_t)t * CACHE_FIELDS * H;
    double dzi = 0.0, dzf = 0.0, dzg = 0.0, dzo = 0.0;
    if (act) {
      const double gi = cc[j], gf = cc[H + j], gg = cc[2 * H + j], go = cc[3 * H + j];
      const double c_prev = cc[4 * H + j], tc = cc[6 * H + j];
      const double dh = fadd(fmul(w[j], d_raw), dh_next);
      const double d_o = fmul(dh, tc);
      const double dc = fadd(dc_next, fmul(fmul(dh, go), fsub(1.0, fmul(tc, tc))));
      const double di = fmul(dc, gg), df = fmul(dc, c_prev), dg = fmul(dc, gi);
      dc_next = fmul(dc, gf);
      dzi = fmul(fmul(di, gi), fsub(1.0, gi));
      dzf = fmul(fmul(df, gf), fsub(1.0, gf));
      dzg = fmul(dg, fsub(1.0, fmul(gg, gg)));
      dzo = fmul(fmul(d_o, go), fsub(1.0, go));
      double* dzt = dzb + (int64_t)t * G;
      dzt[j] = dzi;
      dzt[H + j] = dzf;
      dzt[2 * H + j] = dzg;
      dzt[3 * H + j] = dzo;
    }
    // dh_next = dz @ Wh.T : lane k sums over the 4H gate columns in order
    double s = 0.0;
    for (int gsel = 0; gsel < 4; ++gsel) {
      const double dsel = gsel == 0 ? dzi : gsel == 1 ? dzf : gsel == 2 ? dzg : dzo;
      for (int jj = 0; jj < H; ++jj) {
        const double dv = __shfl_sync(0xffffffffu, dsel, jj);
        s = fadd(s, fmul(dv, Wh[j * G + gsel * H + jj]));
      }
    }
    dh_next = act ? s : 0.0;
  }
}

// Split-K weight gradients.  The reduction axis is the (t descending, b)
// sequence of valid (sequence, timestep) pairs; block y handles a fixed
// contiguous range of it (identical split for a given batch -> deterministic).
__global__ void k_train_wgrad(TrainArgs a, int ksplit, double* __restrict__ partial) {
  const Layout L(a.H);
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= L.n) return;
  const int H = a.H, G = L.G;
  const int64_t K = (int64_t)a.Tmax * a.B;
  const int64_t k0 = K * blockIdx.y / ksplit, k1 = K * (blockIdx.y + 1) / ksplit;
  double acc = 0.0;
  int kind, r, col;
  if (p < L.oWh) { kind = 0; r = p / G; col = p % G; }
  else if (p < L.ob) { kind = 1; r = (p - L.oWh) / G; col = (p - L.oWh) % G; }
  else if (p < L.ow) { kind = 2; r = 0; col = p - L.ob; }
  else if (p < L.obout) { kind = 3; r = p - L.ow; col = 0; }
  else { kind = 4; r = 0; col = 0; }
  for (int64_t kk = k0; kk < k1; ++kk) {
    const int t = a.Tmax - 1 - (int)(kk / a.B);
    const int b = (int)(kk % a.B);
    const int idx = a.batch[b];
    const int T = a.D.Tlen[idx];
    if (kind == 4) {  // db_out = sum_b T_b d_raw_b, counted once per sequence (at t = 0)
      if (t == 0) acc = fadd(acc, fmul((double)T, a.draw[b]));
      continue;
    }
    if (t >= T) continue;
    const int64_t bt = (int64_t)b * a.Tmax + t;
    if (kind == 0) {
      acc = fadd(acc, fmul(a.D.x(idx, t)[r], a.dz[bt * G + col]));
    } else if (kind == 1) {
      acc = fadd(acc, fmul(a.cache[(bt * CACHE_FIELDS + 5) * H + r], a.dz[bt * G + col]));
    } else if (kind == 2) {
      acc = fadd(acc, a.dz[bt * G + col]);
    } else {
      acc = fadd(acc, fmul(a.cache[(bt * CACHE_FIELDS + 7) * H + r], a.draw[b]));
    }
  }
  partial[(int64_t)blockIdx.y * L.n + p] = acc;
}

__global__ void k_train_reduce(const double* __restrict__ partial, int ksplit, int n, double* __restrict__ grad) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double acc = 0.0;
  int k = 0;
  for (; k + 8 <= ksplit; k += 8) {  // loads issued together, summed in order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = partial[(int64_t)(k + u) * n + p];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fadd(acc, v[u]);
  }
  for (; k < ksplit; ++k) acc = fadd(acc, partial[(int64_t)k * n + p]);
  grad[p] = acc;
}

// _clip + SGD (value_model.py:213-220, :267-271); one block of 1024 threads.
__global__ void k_train_apply(double* __restrict__ P, const double* __restrict__ grad, int n, double lr,
                              double max_norm, double* __restrict__ norm_out) {
  __shared__ double part[32];
  double sq = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sq = ffma(grad[i], grad[i], sq);
  for (int o = 16; o > 0; o >>= 1) sq = fadd(sq, __shfl_down_sync(0xffffffffu, sq, o));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fadd(t, part[w]);
    part[0] = sqrt(t);
  }
  __syncthreads();
  const double norm = part[0];
  const double scale = norm > max_norm ? fdiv(max_norm, norm) : 1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double g = norm > max_norm ? fmul(grad[i], scale) : grad[i];
    P[i] = fsub(P[i], fmul(lr, g));
  }
  if (threadIdx.x == 0 && norm_out) *norm_out = norm;
}

// ------------------------------------------------ H = 32: sequence groups
// The warp-per-sequence kernels above are latency-bound (one dependent fp64
// chain per lane, weights re-read through L1 every timestep).  For the
// model's H = 32 the batch is instead processed in groups of GS sequences per
// CTA with the weights resident in shared memory: every timestep is a small
// [GS x 48] x [48 x 128] product (thread = gate column, 8 sequences each) and
// the BPTT step a [GS x 128] x [128 x 32] product (thread = hidden unit, 2
// sequences), so each thread carries 8 (resp. 2) independent chains.  The
// products accumulate with fused multiply-adds in the same k order as the
// warp kernels (as BLAS dgemm kernels do); the gate and cell arithmetic is
// identical, so the two agree to rounding (tested at 1e-12).
//
// For the weight gradients the kernel also writes one packed row per valid
// (sequence, timestep) pair at its position kk = (Tmax-1-t)*B + b of the
// k_train_wgrad reduction order: [x_t (16) | h_{t-1} (32) | h_t (32) |
// dz_t (128)], flag pvalid[kk] = 1, so k_train_wgrad_group streams
// contiguous rows instead of chasing per-pair indices.
constexpr int GS = 16;
constexpr int PROW = 208;  // packed pair row (doubles)
constexpr int GTHREADS = 256;
constexpr int GH = 32, GG = 128, GK = 48;

struct GroupSmem {
  double W[GK][GG];    // rows 0..15 Wx, 16..47 Wh (the flat parameter order)
  double WhT[GG][GH];  // Wh transposed for dh_next
  double xh[GS][GK];   // [x_t | h_{t-1}] per sequence
  double zb[GS][GG];   // gate pre-activations (forward), dz (backward)
  double b[GG];
  double w[GH];
  const double* xinit[GS];  // per sequence: init rows (t < T - d)
  const double* xrows[GS];  //               scheduled rows, reversed (t >= T - d)
  int T[GS], Tu[GS];        // length, first scheduled timestep T - d
  uint64_t bar[2];          // tensor-core weight gradients: UMMA completion per operand buffer
  uint32_t tmem;            //                               TMEM accumulator base
};

// ------------------------------------------------ tensor-core weight gradients
// kTc = true (ts_train_set_mode(TS_TRAIN_TC)): the forward and BPTT
// recurrences stay fp64 (raw, d_raw and every dz are the exact kernel's), but
// the weight-gradient contraction - the one dense GEMM of training,
// [dWx; dWh; db]^T = sum over (sequence, timestep) of dz^T [x | h_prev | 1],
// K = B * T - runs on the tensor cores, fused into BPTT: at every timestep
// the CTA's 16 dz rows (A = dz^T, M = 128 gate columns, K = 16 sequences)
// and [x_t | h_{t-1} | 1] rows (B, N = 64) are split into TF32 hi/lo in
// shared memory (the forward weight tile's space, free during BPTT) and one
// thread issues six kind::tf32 UMMAs, A' = [hi | lo | hi] . B' = [hi | hi |
// lo] (3xTF32, ~22-bit operands), accumulating D[128 x 64] (fp32) in TMEM
// over the CTA's whole BPTT.  No pair rows go to HBM and the separate
// weight-gradient kernel disappears; the CTA writes its D (and the fp64 dw,
// db_out sums) as one partial, reduced in fixed order by k_train_reduce.
constexpr int TCN = 64;                          // UMMA N: x(16) | h_prev(32) | 1 | 0 x 15
constexpr int TC_CS_A = (GG / 8) * 128;          // A: bytes between K chunks = 2048
constexpr int TC_CS_B = (TCN / 8) * 128;         // B: 1024
constexpr int TC_A_BYTES = (GS / 4) * TC_CS_A;   // one K = 16 operand: 8192
constexpr int TC_B_BYTES = (GS / 4) * TC_CS_B;   // 4096
constexpr int TC_BUF = 2 * TC_A_BYTES + 2 * TC_B_BYTES;  // A_hi, A_lo, B_hi, B_lo = 24576
static_assert(2 * TC_BUF <= (int)sizeof(double) * GK * GG, "two operand buffers fit the W tile");
// kind::tf32, A = B = TF32, D = F32, K-major both, N = 64, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TCN >> 3) << 17) |
                              ((uint32_t)(GG >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(TC_IDESC), "r"(acc)
      : "memory");
}

// round to the nearest TF32 (ties away from zero) on the integer pipe - the
// bit pattern of cvt.rna.tf32.f32 for finite values, without the conversion
// unit; the tensor core reads the top 19 bits
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
}

// v = hi + lo + O(2^-22 |v|), both TF32 (fp32 bit patterns, low 13 bits 0);
// one f64 -> f32 conversion, the remainder f - hi is exact in fp32
__device__ __forceinline__ void split_tf32(double v, uint32_t& hi, uint32_t& lo) {
  const float f = (float)v;
  hi = tf32_rna(f);
  lo = tf32_rna(__fsub_rn(f, __uint_as_float(hi)));
}

// canonical K-major no-swizzle offset of element (row, k), 4-byte elements
__device__ __forceinline__ int tc_off(int row, int k, int cs) {
  return (k >> 2) * cs + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

template <bool kTc>
__global__ void __launch_bounds__(GTHREADS, 2) k_train_fb_group(TrainArgs a) {
  extern __shared__ __align__(16) double tr_dyn_smem[];
  GroupSmem& S = *reinterpret_cast<GroupSmem*>(tr_dyn_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Layout L(GH);
  const double* P = a.P;
  for (int e = tid; e < GK * GG; e += GTHREADS) (&S.W[0][0])[e] = P[L.oWx + e];
  for (int e = tid; e < GH * GG; e += GTHREADS) S.WhT[e % GG][e / GG] = P[L.oWh + e];
  for (int e = tid; e < GG; e += GTHREADS) S.b[e] = P[L.ob + e];
  if (tid < GH) S.w[tid] = P[L.ow + tid];
  for (int e = tid; e < GS * GK; e += GTHREADS) (&S.xh[0][0])[e] = 0.0;
  const int g0 = blockIdx.x * GS;
  if (tid < GS) {
    const int b = g0 + tid;
    int T = 0, Tu = 0;
    const double *xi = a.D.init, *xr = a.D.rows;
    if (b < a.B) {
      const int i = a.batch[b];
      T = a.D.Tlen[i];
      Tu = T - a.D.depth[i];
      xi = a.D.init + (int64_t)a.D.init_base[i] * F;
      xr = a.D.rows + (a.D.row_base[i] + (T - 1)) * F;  // row of timestep t: xr - t * F
    }
    S.T[tid] = T;
    S.Tu[tid] = Tu;
    S.xinit[tid] = xi;
    S.xrows[tid] = xr;
  }
  if constexpr (kTc) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       tc::smem_u32(&S.tmem)),
                   "r"(TCN)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
      tc::mbar_init(&S.bar[0], 1);
      tc::mbar_init(&S.bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
  }
  __syncthreads();
  if constexpr (kTc) tc::fence_after();
  int Tg = 0;
  for (int s = 0; s < GS; ++s) Tg = max(Tg, S.T[s]);
  // gate-phase ownership: sequence s = warp + 8q, hidden unit j = lane
  int Tq[2];
  double raw[2], c[2] = {0.0, 0.0};
  double* cache[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int s = warp + 8 * q, b = g0 + s;
    Tq[q] = S.T[s];
    raw[q] = fmul((double)Tq[q], P[L.obout]);
    cache[q] = a.cache + (int64_t)(b < a.B ? b : 0) * a.Tmax * CACHE_FIELDS * GH;
  }
  // ---- forward with cache
  for (int t = 0; t < Tg; ++t) {
    {  // x rows: one feature per thread
      const int s = tid >> 4, k = tid & 15;
      double v = 0.0;
      if (t < S.T[s]) {
        v = t < S.Tu[s] ? S.xinit[s][t * F + k] : S.xrows[s][k - t * F];
        if constexpr (!kTc) a.dz[((int64_t)(a.Tmax - 1 - t) * a.B + g0 + s) * PROW + k] = v;
      }
      S.xh[s][k] = v;
    }
    __syncthreads();
    {  // z = b + x Wx + h Wh, column n for sequences s0, s0+2, ..
      const int n = tid & (GG - 1), s0 = tid >> 7;
      double z[8];
      const double bn = S.b[n];
#pragma unroll
      for (int i = 0; i < 8; ++i) z[i] = bn;
#pragma unroll 2
      for (int k = 0; k < GK; k += 2) {  // k order kept; x pairs as 16-byte loads
        const double w0 = S.W[k][n], w1 = S.W[k + 1][n];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 xv = *reinterpret_cast<const double2*>(&S.xh[s0 + 2 * i][k]);
          z[i] = ffma(xv.y, w1, ffma(xv.x, w0, z[i]));
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) S.zb[s0 + 2 * i][n] = z[i];
    }
    __syncthreads();
    double hn[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int s = warp + 8 * q;
      if (t >= Tq[q]) continue;  // warp-uniform
      const double gi = sig(S.zb[s][lane]), gf = sig(S.zb[s][GH + lane]), gg = tanh(S.zb[s][2 * GH + lane]),
                   go = sig(S.zb[s][3 * GH + lane]);
      const double c_prev = c[q], h_prev = S.xh[s][16 + lane];
      c[q] = fadd(fmul(gf, c[q]), fmul(gi, gg));
      const double tc = tanh(c[q]);
      const double h = fmul(go, tc);
      double* cc = cache[q] + (int64_t)t * CACHE_FIELDS * GH;
      cc[0 * GH + lane] = gi;
      cc[1 * GH + lane] = gf;
      cc[2 * GH + lane] = gg;
      cc[3 * GH + lane] = go;
      cc[4 * GH + lane] = c_prev;
      cc[6 * GH + lane] = tc;
      if constexpr (kTc) {
        cc[7 * GH + lane] = h;  // h_prev of t + 1 as well
      } else {
        const int64_t kk = (int64_t)(a.Tmax - 1 - t) * a.B + g0 + s;
        double* pr = a.dz + kk * PROW;
        pr[16 + lane] = h_prev;
        pr[48 + lane] = h;
        if (lane == 0) a.pvalid[kk] = 1;
      }
      hn[q] = h;
      const double prod = fmul(h, S.w[lane]);
      double acc = 0.0;
      for (int k = 0; k < GH; ++k) acc = fadd(acc, __shfl_sync(0xffffffffu, prod, k));
      raw[q] = fadd(raw[q], acc);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q)
      if (t < Tq[q]) S.xh[warp + 8 * q][16 + lane] = hn[q];
  }
  // d_raw = 2 (raw + ts - log t) / n  (value_model.py:201)
  double d_raw[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int b = g0 + warp + 8 * q;
    d_raw[q] = 0.0;
    if (b >= a.B) continue;
    d_raw[q] = a.draw_in ? a.draw_in[b]
                         : fdiv(fmul(2.0, fsub(fadd(raw[q], a.target_scale), a.D.logt[a.batch[b]])), a.n_total);
    if (lane == 0) {
      a.raw[b] = raw[q];
      a.draw[b] = d_raw[q];
    }
  }
  // ---- BPTT; the cache row of the next (earlier) timestep is prefetched
  // into registers while the current dh_next product runs
  double dh_next[2] = {0.0, 0.0}, dc_next[2] = {0.0, 0.0};
  const double wj = S.w[lane];
  constexpr int NCV = kTc ? 8 : 6;
  double cv[2][NCV];
  auto load_cache = [&](int t) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (t < 0 || t >= Tq[q]) continue;
      const double* cc = cache[q] + (int64_t)t * CACHE_FIELDS * GH + lane;
      cv[q][0] = cc[0];
      cv[q][1] = cc[GH];
      cv[q][2] = cc[2 * GH];
      cv[q][3] = cc[3 * GH];
      cv[q][4] = cc[4 * GH];
      cv[q][5] = cc[6 * GH];
      if constexpr (kTc) {
        // h_t (dw) and h_{t-1} (the B operand): h_t is the previous call's
        // h_{t-1} except at a sequence's last timestep
        cv[q][7] = t == Tq[q] - 1 ? cc[7 * GH] : cv[q][6];
        cv[q][6] = t > 0 ? cc[7 * GH - CACHE_FIELDS * GH] : 0.0;
      }
    }
  };
  // tensor-core operands, two buffers in the (now unused) forward weight
  // tile, each [A_hi | A_lo | B_hi | B_lo] (K = 16 sequences); the UMMAs of
  // timestep t read buffer t & 1 while the next timestep fills the other
  uint8_t* tcbuf = reinterpret_cast<uint8_t*>(&S.W[0][0]);
  // per buffer (bit bf): phase parity and a commit in flight - at most one
  // per barrier, so a parity wait never skips a phase
  uint32_t phase = 0u, pending = 0u;
  int n_issued = 0;  // uniform: UMMA groups issued (TMEM holds a partial sum once > 0)
  double dw_acc[2] = {0.0, 0.0};
  if constexpr (kTc) {
    // B rows 49..63 stay zero in both buffers (row 48 is the ones column of db)
    for (int e = tid; e < 2 * 2 * 15 * 4; e += GTHREADS) {
      const int buf = e / 120, half = (e / 60) & 1, row = 49 + (e % 60) / 4, c4 = e % 4;
      *reinterpret_cast<uint4*>(tcbuf + buf * TC_BUF + 2 * TC_A_BYTES + half * TC_B_BYTES +
                                tc_off(row, 4 * c4, TC_CS_B)) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  load_cache(Tg - 1);
  for (int t = Tg - 1; t >= 0; --t) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int s = warp + 8 * q, b = g0 + s;
      if (t >= Tq[q]) {
        if constexpr (kTc) {  // this sequence adds nothing at t: zero operand rows
#pragma unroll
          for (int g = 0; g < 4; ++g) S.zb[s][g * GH + lane] = 0.0;
          S.xh[s][16 + lane] = 0.0;
          if (lane < 16) S.xh[s][lane] = 0.0;
        }
        continue;
      }
      const double gi = cv[q][0], gf = cv[q][1], gg = cv[q][2], go = cv[q][3];
      const double c_prev = cv[q][4], tc = cv[q][5];
      const double dh = fadd(fmul(wj, d_raw[q]), dh_next[q]);
      const double d_o = fmul(dh, tc);
      const double dc = fadd(dc_next[q], fmul(fmul(dh, go), fsub(1.0, fmul(tc, tc))));
      const double di = fmul(dc, gg), df = fmul(dc, c_prev), dg = fmul(dc, gi);
      dc_next[q] = fmul(dc, gf);
      const double dzi = fmul(fmul(di, gi), fsub(1.0, gi));
      const double dzf = fmul(fmul(df, gf), fsub(1.0, gf));
      const double dzg = fmul(dg, fsub(1.0, fmul(gg, gg)));
      const double dzo = fmul(fmul(d_o, go), fsub(1.0, go));
      if constexpr (kTc) {
        (void)b;
        // [x_t | h_{t-1}] of this sequence for the B operand
        S.xh[s][16 + lane] = cv[q][6];
        if (lane < 16) S.xh[s][lane] = t < S.Tu[s] ? S.xinit[s][t * F + lane] : S.xrows[s][lane - t * F];
        dw_acc[q] = ffma(cv[q][7], d_raw[q], dw_acc[q]);  // dw = sum_t h_t d_raw
      } else {
        double* dzt = a.dz + ((int64_t)(a.Tmax - 1 - t) * a.B + b) * PROW + 80;
        dzt[lane] = dzi;
        dzt[GH + lane] = dzf;
        dzt[2 * GH + lane] = dzg;
        dzt[3 * GH + lane] = dzo;
      }
      S.zb[s][lane] = dzi;
      S.zb[s][GH + lane] = dzf;
      S.zb[s][2 * GH + lane] = dzg;
      S.zb[s][3 * GH + lane] = dzo;
    }
    load_cache(t - 1);
    __syncthreads();
    if constexpr (kTc) {
      // operand tiles from S.zb / S.xh, one 16-byte chunk (4 sequences) per
      // item and segment, consecutive threads on consecutive rows (conflict
      // free); first the previous timestep's UMMAs must have read the tiles
      // buffer t & 1 was last read by the UMMAs of timestep t + 2: wait for
      // that commit (on the buffer's own barrier)
      const int bf = t & 1;
      if ((pending >> bf) & 1u) {
        tc::mbar_wait(&S.bar[bf], (phase >> bf) & 1u);
        phase ^= 1u << bf;
        pending &= ~(1u << bf);
      }
      uint8_t* At = tcbuf + (t & 1) * TC_BUF;
      uint8_t* Bt = At + 2 * TC_A_BYTES;
      for (int e = tid; e < GG * 4 + 49 * 4; e += GTHREADS) {
        const bool isa = e < GG * 4;
        const int e2 = isa ? e : e - GG * 4;
        const int row = isa ? (e2 & (GG - 1)) : e2 % 49, c4 = isa ? (e2 >> 7) : e2 / 49;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int sq = 4 * c4 + u;
          const double v = isa ? S.zb[sq][row] : (row < 48 ? S.xh[sq][row] : (t < S.T[sq] ? 1.0 : 0.0));
          split_tf32(v, hi[u], lo[u]);
        }
        const uint4 H4 = make_uint4(hi[0], hi[1], hi[2], hi[3]), L4 = make_uint4(lo[0], lo[1], lo[2], lo[3]);
        uint8_t* dst = isa ? At + tc_off(row, 4 * c4, TC_CS_A) : Bt + tc_off(row, 4 * c4, TC_CS_B);
        const int lo_off = isa ? TC_A_BYTES : TC_B_BYTES;
        *reinterpret_cast<uint4*>(dst) = H4;
        *reinterpret_cast<uint4*>(dst + lo_off) = L4;
      }
      tc::fence_async_smem();  // operand tiles visible to the tensor core
    }
    // dh_next = dz @ Wh.T in gate-column order; both sequences share the
    // Wh loads, dz pairs as 16-byte broadcasts
    {
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
      for (int col = 0; col < GG; col += 2) {
        const double w0 = S.WhT[col][lane], w1 = S.WhT[col + 1][lane];
        const double2 z0 = *reinterpret_cast<const double2*>(&S.zb[warp][col]);
        const double2 z1 = *reinterpret_cast<const double2*>(&S.zb[warp + 8][col]);
        acc0 = ffma(z0.y, w1, ffma(z0.x, w0, acc0));
        acc1 = ffma(z1.y, w1, ffma(z1.x, w0, acc1));
      }
      if (t < Tq[0]) dh_next[0] = acc0;
      if (t < Tq[1]) dh_next[1] = acc1;
    }
    __syncthreads();
    if constexpr (kTc) {
      if (tid == 0) {
        // 3xTF32: A_hi B_hi + A_lo B_hi + A_hi B_lo, two K = 8 steps each
        tc::fence_after();
        const uint32_t ab = tc::smem_u32(tcbuf + (t & 1) * TC_BUF), bb = ab + 2 * TC_A_BYTES;
#pragma unroll
        for (int pr = 0; pr < 3; ++pr) {
          const uint32_t a0 = ab + (pr == 1 ? TC_A_BYTES : 0), b0 = bb + (pr == 2 ? TC_B_BYTES : 0);
#pragma unroll
          for (int k = 0; k < 2; ++k)
            mma_tf32(S.tmem, tc::umma_desc(a0 + k * 2 * TC_CS_A, TC_CS_A, 128),
                     tc::umma_desc(b0 + k * 2 * TC_CS_B, TC_CS_B, 128), (n_issued > 0 || pr > 0 || k > 0) ? 1u : 0u);
        }
        tc::mma_commit(&S.bar[t & 1]);
      }
      pending |= 1u << (t & 1);
      ++n_issued;
    }
  }
  if constexpr (kTc) {
    // this CTA's weight-gradient partial: D (TMEM, fp32) -> dWx, dWh, db;
    // dw and db_out summed in fp64 over the CTA's sequences in fixed order
    double* out = a.partial + (int64_t)blockIdx.x * L.n;
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // S.xh is no operand source any more (tiles built)
      S.xh[warp + 8 * q][lane] = dw_acc[q];
      if (lane == 0) S.xh[warp + 8 * q][40] = g0 + warp + 8 * q < a.B ? fmul((double)Tq[q], d_raw[q]) : 0.0;
    }
    // drain the (up to two) outstanding commits
#pragma unroll
    for (int bf = 0; bf < 2; ++bf)
      if ((pending >> bf) & 1u) tc::mbar_wait(&S.bar[bf], (phase >> bf) & 1u);
    if (n_issued) tc::fence_after();
    __syncthreads();
    if (tid < GG) {
      const int m = tid;  // gate column = TMEM lane (warp w reads lanes 32w..32w+31)
      if (n_issued) {
        const uint32_t la = S.tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
        for (int c8 = 0; c8 < 7; ++c8) {  // columns 0..55 (x, h_prev, ones)
          float v[8];
          tc::tmem_ld8(la + c8 * 8, v);
          tc::tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int col = c8 * 8 + u;
            if (col < 16) out[L.oWx + col * GG + m] = (double)v[u];
            else if (col < 48) out[L.oWh + (col - 16) * GG + m] = (double)v[u];
            else if (col == 48) out[L.ob + m] = (double)v[u];
          }
        }
      } else {
        for (int k = 0; k < GK; ++k) out[k * GG + m] = 0.0;
        out[L.ob + m] = 0.0;
      }
    } else if (tid < GG + GH) {
      const int j = tid - GG;
      double acc = 0.0;
      for (int s2 = 0; s2 < GS; ++s2) acc = fadd(acc, S.xh[s2][j]);
      out[L.ow + j] = acc;
    } else if (tid == GG + GH) {
      double acc = 0.0;
      for (int s2 = 0; s2 < GS; ++s2) acc = fadd(acc, S.xh[s2][40]);
      out[L.obout] = acc;
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(S.tmem), "r"(TCN) : "memory");
  }
}

// Weight gradients, H = 32: one CTA per k-split range of the (t descending,
// b) pair sequence, all 6,305 parameters per CTA.  Chunks of WCH packed pair
// rows are staged in shared memory (the next chunk is prefetched into
// registers while the current one is consumed); thread (rg, cg) owns the
// 3 x 8 block rows rg + 16i, columns cg + 16j of [dWx; dWh], threads 0..127
// also db, 128..159 dw, 160 db_out.  Each parameter is accumulated in pair
// order (fused multiply-add).
constexpr int WCH = 16;
constexpr int WV = WCH * PROW / 2;                      // 16-byte vectors per chunk
constexpr int WPT = (WV + GTHREADS - 1) / GTHREADS;     // per thread
struct WgradSmem {
  double R[WCH][PROW];
  double dr[WCH];
  double tdr[WCH];     // T * d_raw (db_out term, rows with t == 0)
  int valid[WCH];
  int first[WCH];      // t == 0
};

__global__ void __launch_bounds__(GTHREADS) k_train_wgrad_group(TrainArgs a, int ksplit,
                                                                double* __restrict__ partial) {
  extern __shared__ __align__(16) double tr_dyn_smem[];
  WgradSmem& S = *reinterpret_cast<WgradSmem*>(tr_dyn_smem);
  const Layout L(GH);
  const int tid = threadIdx.x;
  const int rg = tid >> 4, cg = tid & 15;
  const int64_t K = (int64_t)a.Tmax * a.B;
  const int64_t k0 = K * blockIdx.x / ksplit, k1 = K * (blockIdx.x + 1) / ksplit;
  double acc[3][8];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  double extra = 0.0;
  // register prefetch of one chunk: rows [kb, kb + nk) are contiguous
  uint4 pf[WPT];
  int pf_valid = 0, pf_first = 0;
  double pf_dr = 0.0, pf_tdr = 0.0;
  auto fetch = [&](int64_t kb) {
    const int nk = (int)(k1 - kb < WCH ? k1 - kb : WCH);
    const uint4* src = reinterpret_cast<const uint4*>(a.dz + kb * PROW);
#pragma unroll
    for (int v = 0; v < WPT; ++v) {
      const int e = tid + v * GTHREADS;
      if (e < nk * (PROW / 2)) pf[v] = __ldcs(src + e);  // invalid rows: unused bytes
    }
    if (tid < nk) {
      const int64_t kk = kb + tid;
      const int t = a.Tmax - 1 - (int)(kk / a.B);
      const int b = (int)(kk % a.B);
      pf_valid = a.pvalid[kk];
      pf_first = t == 0;
      pf_dr = a.draw[b];
      pf_tdr = pf_first ? fmul((double)a.D.Tlen[a.batch[b]], pf_dr) : 0.0;
    }
  };
  if (k0 < k1) fetch(k0);
  for (int64_t kb = k0; kb < k1; kb += WCH) {
    const int nk = (int)(k1 - kb < WCH ? k1 - kb : WCH);
    __syncthreads();  // previous chunk consumed
    {
      uint4* dst = reinterpret_cast<uint4*>(&S.R[0][0]);
#pragma unroll
      for (int v = 0; v < WPT; ++v) {
        const int e = tid + v * GTHREADS;
        if (e < nk * (PROW / 2)) dst[e] = pf[v];
      }
      if (tid < nk) {
        S.valid[tid] = pf_valid;
        S.first[tid] = pf_first;
        S.dr[tid] = pf_dr;
        S.tdr[tid] = pf_tdr;
      }
    }
    __syncthreads();
    if (kb + WCH < k1) fetch(kb + WCH);
    for (int rr = 0; rr < nk; ++rr) {
      if (tid == GG + GH && S.first[rr]) extra = fadd(extra, S.tdr[rr]);
      if (!S.valid[rr]) continue;  // uniform
      double av[3], dv[8];
#pragma unroll
      for (int i = 0; i < 3; ++i) av[i] = S.R[rr][rg + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) dv[j] = S.R[rr][80 + cg + 16 * j];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = ffma(av[i], dv[j], acc[i][j]);
      if (tid < GG) extra = fadd(extra, S.R[rr][80 + tid]);
      else if (tid < GG + GH) extra = ffma(S.R[rr][48 + tid - GG], S.dr[rr], extra);
    }
  }
  double* out = partial + (int64_t)blockIdx.x * L.n;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) out[(rg + 16 * i) * GG + cg + 16 * j] = acc[i][j];
  if (tid < GG) out[L.ob + tid] = extra;
  else if (tid < GG + GH) out[L.ow + tid - GG] = extra;
  else if (tid == GG + GH) out[L.obout] = extra;
}

// raw for a list of sequences (eval, Cython order with the zero skip):
// warp per sequence
__global__ void k_train_fwd(TrainArgs a) {
  const int wb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wb >= a.B) return;
  const Layout L(a.H);
  const int H = a.H, G = L.G;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  const int idx = a.batch[wb];
  const int T = a.D.Tlen[idx];
  const double* Wx = a.P + L.oWx;
  const double* Wh = a.P + L.oWh;
  const double* bb = a.P + L.ob;
  const double* w = a.P + L.ow;
  double h = 0.0, c = 0.0;
  double raw = fmul((double)T, a.P[L.obout]);
  for (int t = 0; t < T; ++t) {
    const double* X = a.D.x(idx, t);
    double zi = bb[j], zf = bb[H + j], zg = bb[2 * H + j], zo = bb[3 * H + j];
    for (int k = 0; k < F; ++k) {
      const double xv = X[k];
      if (xv != 0.0) {
        const double* wr = Wx + k * G;
        zi = fadd(zi, fmul(xv, wr[j]));
        zf = fadd(zf, fmul(xv, wr[H + j]));
        zg = fadd(zg, fmul(xv, wr[2 * H + j]));
        zo = fadd(zo, fmul(xv, wr[3 * H + j]));
      }
    }
    for (int k = 0; k < H; ++k) {
      const double hv = __shfl_sync(0xffffffffu, h, k);
      if (hv != 0.0) {
        const double* wr = Wh + k * G;
        zi = fadd(zi, fmul(hv, wr[j]));
        zf = fadd(zf, fmul(hv, wr[H + j]));
        zg = fadd(zg, fmul(hv, wr[2 * H + j]));
        zo = fadd(zo, fmul(hv, wr[3 * H + j]));
      }
    }
    double prod = 0.0;
    if (act) {
      const double gi = sig(zi), gf = sig(zf), gg = tanh(zg), go = sig(zo);
      c = fadd(fmul(gf, c), fmul(gi, gg));
      h = fmul(go, tanh(c));
      prod = fmul(h, w[j]);
    }
    double acc = 0.0;
    for (int k = 0; k < H; ++k) acc = fadd(acc, __shfl_sync(0xffffffffu, prod, k));
    raw = fadd(raw, acc);
  }
  if (lane == 0) a.raw[wb] = raw;
}

}  // namespace tr
}  // namespace ts
