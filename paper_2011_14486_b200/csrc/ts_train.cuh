// ts_train.cuh - V training on the B200.
//
// value_model.gradients (value_model.py:182-210) = per-sequence
// lstm_forward_cached + lstm_backward (_recurrent_np.py:38-96) summed over the
// minibatch, then _clip (:213-220) and the SGD update (:267-271).  fp64
// throughout so the device trajectory tracks the reference's (the training
// loop is contractive: 1e-12 perturbations stay ~1e-13).
//
//   k_train_fb     warp per sequence, lane per hidden unit: forward with the
//                  activation cache, d_raw = 2(raw + ts - log t)/n_total,
//                  BPTT; writes dz[b][t][4H] and keeps h_prev/h in the cache
//   k_train_wgrad  thread per parameter: dWx = sum x^T dz, dWh = sum h_prev^T dz,
//                  db = sum dz, dw = sum h d_raw, db_out = sum_b T_b d_raw_b,
//                  reduced over (t descending, b) in a fixed order
//   k_train_apply  one block: global L2 norm incl. b_out, clip, p -= lr g
//   k_train_fwd    warp per sequence: raw for _eval_split
//
// The gradient buffer is a plain device array between k_train_wgrad and
// k_train_apply, so data-parallel training all-reduces it (NCCL) in between.
#pragma once

#include <cuda_runtime.h>

#include "ts_core.cuh"

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

struct TrainArgs {
  const double* X;      // [N][Tmax][16] normalized
  const int* Tlen;      // [N]
  const double* logt;   // [N]
  const int* batch;     // [B] dataset indices
  const double* P;      // params
  double* cache;        // [B][Tmax][8][H]
  double* dz;           // [B][Tmax][4H]
  double* draw;         // [B]
  double* raw;          // [B]
  int B, Tmax, H;
  double target_scale;
  double n_total;       // global minibatch size n (value_model.py:193)
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
  const int T = a.Tlen[idx];
  const double* X = a.X + (int64_t)idx * a.Tmax * F;
  const double* Wx = a.P + L.oWx;
  const double* Wh = a.P + L.oWh;
  const double* bb = a.P + L.ob;
  const double* w = a.P + L.ow;
  double* cache = a.cache + (int64_t)wb * a.Tmax * CACHE_FIELDS * H;
  double h = 0.0, c = 0.0;
  double raw = fmul((double)T, a.P[L.obout]);
  // ---- forward with cache (_recurrent_np.py:38-59)
  for (int t = 0; t < T; ++t) {
    double zi = bb[j], zf = bb[H + j], zg = bb[2 * H + j], zo = bb[3 * H + j];
    for (int k = 0; k < F; ++k) {
      const double xv = X[t * F + k];
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
  const double d_raw = fdiv(fmul(2.0, fsub(fadd(raw, a.target_scale), a.logt[idx])), a.n_total);
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

// Weight gradients: thread per parameter, fixed reduction order (t
// descending, then batch order) - deterministic for a given batch.
__global__ void k_train_wgrad(TrainArgs a, double* __restrict__ grad) {
  const Layout L(a.H);
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= L.n) return;
  const int H = a.H, G = L.G;
  double acc = 0.0;
  if (p < L.oWh) {  // dWx[k][c] = sum x[t][k] dz[t][c]
    const int k = p / G, c = p % G;
    for (int t = a.Tmax - 1; t >= 0; --t)
      for (int b = 0; b < a.B; ++b) {
        const int idx = a.batch[b];
        if (t >= a.Tlen[idx]) continue;
        acc = fadd(acc, fmul(a.X[((int64_t)idx * a.Tmax + t) * F + k], a.dz[((int64_t)b * a.Tmax + t) * G + c]));
      }
  } else if (p < L.ob) {  // dWh[k][c] = sum h_prev[t][k] dz[t][c]
    const int q = p - L.oWh, k = q / G, c = q % G;
    for (int t = a.Tmax - 1; t >= 0; --t)
      for (int b = 0; b < a.B; ++b) {
        if (t >= a.Tlen[a.batch[b]]) continue;
        const double hp = a.cache[(((int64_t)b * a.Tmax + t) * CACHE_FIELDS + 5) * H + k];
        acc = fadd(acc, fmul(hp, a.dz[((int64_t)b * a.Tmax + t) * G + c]));
      }
  } else if (p < L.ow) {  // db[c] = sum dz[t][c]
    const int c = p - L.ob;
    for (int t = a.Tmax - 1; t >= 0; --t)
      for (int b = 0; b < a.B; ++b) {
        if (t >= a.Tlen[a.batch[b]]) continue;
        acc = fadd(acc, a.dz[((int64_t)b * a.Tmax + t) * G + c]);
      }
  } else if (p < L.obout) {  // dw[j] = sum h[t][j] d_raw
    const int jj = p - L.ow;
    for (int t = a.Tmax - 1; t >= 0; --t)
      for (int b = 0; b < a.B; ++b) {
        if (t >= a.Tlen[a.batch[b]]) continue;
        const double hv = a.cache[(((int64_t)b * a.Tmax + t) * CACHE_FIELDS + 7) * H + jj];
        acc = fadd(acc, fmul(hv, a.draw[b]));
      }
  } else {  // db_out = sum_b T_b d_raw_b
    for (int b = 0; b < a.B; ++b) acc = fadd(acc, fmul((double)a.Tlen[a.batch[b]], a.draw[b]));
  }
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

// raw for a list of sequences (eval): warp per sequence
__global__ void k_train_fwd(TrainArgs a) {
  const int wb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wb >= a.B) return;
  const Layout L(a.H);
  const int H = a.H, G = L.G;
  const bool act = lane < H;
  const int j = act ? lane : 0;
  const int idx = a.batch[wb];
  const int T = a.Tlen[idx];
  const double* X = a.X + (int64_t)idx * a.Tmax * F;
  const double* Wx = a.P + L.oWx;
  const double* Wh = a.P + L.oWh;
  const double* bb = a.P + L.ob;
  const double* w = a.P + L.ow;
  double h = 0.0, c = 0.0;
  double raw = fmul((double)T, a.P[L.obout]);
  for (int t = 0; t < T; ++t) {
    double zi = bb[j], zf = bb[H + j], zg = bb[2 * H + j], zo = bb[3 * H + j];
    for (int k = 0; k < F; ++k) {
      const double xv = X[t * F + k];
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
