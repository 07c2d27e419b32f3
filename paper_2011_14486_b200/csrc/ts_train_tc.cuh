// ts_train_tc.cuh - V training with the forward AND backward recurrences on
// the 5th-gen tensor cores (ts_train_set_mode(TS_TRAIN_TCF), SURVEY.md 8
// a14-a15, _recurrent_np.py:38-96).
//
// A tile is 128 sequences of the minibatch (sequence = TMEM lane); a CTA of
// four warpgroups works one tile, each warpgroup covering all 128 rows for 8
// of the 32 hidden units.  Two kernels per minibatch, after the weights are
// re-packed for the current parameters (k_trc_pack):
//
//   k_trc_fwd   forward with the activation cache.  Per timestep one split-
//               fp16 UMMA group z = [x | h] . [Wx; Wh] + b (the FAST scoring
//               kernel's operand scheme: A' = [a_hi | a_lo | a_hi | 1],
//               B' = [W_hi; W_hi; W_lo; b], gate columns pre-scaled for ex2),
//               explicit gates on the MUFU pipe, the gates and the cell state
//               written to the cache (fp32), the readout summed in fp64;
//               then d_raw = 2 (raw + ts - log t) / n (value_model.py:201),
//               max |d_raw| (atomicMax on float bits), and the tile's dw =
//               sum_rows d_raw sum_t h_t and db_out = sum_rows T d_raw.
//   k_trc_bwd   BPTT in reverse time.  With S = 2^-e from max |d_raw| (the
//               scaled dz stay O(1), inside fp16's range; exact to undo) each
//               row forms its S dz from the cache (prefetched one timestep
//               ahead) and writes it ONCE into shared memory as split fp16
//               (hi, lo), in a layout that is the K-major A operand of
//                 (a) S dh_next = dz . Wh^T      (M = 128 rows, N = 32, K = 128 gates)
//               and, read MN-major, the A operand of
//                 (b) S [dWx; dWh; db]^T += dz^T . [x | h_prev | 1]
//                                                (M = 128 gates, N = 64, K = 128 rows)
//               [x | h_prev | 1] is written MN-major beside it.  Both products
//               are 3-term split-fp16 UMMAs (hi.hi + lo.hi + hi.lo) with fp32
//               accumulation in TMEM; (a) is read back every timestep, (b)
//               accumulates over the tile's whole BPTT and is flushed once,
//               divided by S, into this tile's fp64 partial gradient.
//   k_train_reduce (ts_train.cuh) sums the tiles' partials in fixed order.
//
// Precision: 22-bit operands, fp32 accumulation, MUFU gates - the gradient is
// fp32-accurate, not the fp64 trajectory of TS_TRAIN_EXACT: tested against
// the exact mode, every gradient block within 1e-5 of its norm (measured
// <= 3.6e-6), and the reference training run reproduces v0 (V within 1e-4,
// measured 5.4e-7; holdout R^2 within 5e-5).  H = 32 only.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ts_core.cuh"
#include "ts_f16.cuh"
#include "ts_lstm_tc.cuh"
#include "ts_train.cuh"

namespace ts {
namespace trc {

using tc::TM;
constexpr int H = 32, G = 128, NF = 5;  // cache fields: i, f, g, o, c
constexpr int FWD_SMEM = tc::TILE_BYTES + tc::A_BYTES + 128 + 4 * 128 * 8 + 32 * 129 * 4 + 128 * 8 + 64;
// backward operand buffers (bytes): dz hi/lo = [16 gate chunks][16 row groups][8][16 B]
constexpr int DZ_BYTES = (G / 8) * 2048;        // 32768 per hi / lo
constexpr int XH_BYTES = (64 / 8) * 2048;       // 16384 per hi / lo: [x 16 | h_prev 32 | 1 | 0 x 15]
constexpr int WT_CS = (H / 8) * 128;            // Wh^T image: bytes between K (gate) chunks = 512
constexpr int WT_BYTES = (G / 8) * WT_CS;       // 8192 per hi / lo
constexpr int BWD_SMEM = 2 * DZ_BYTES + 2 * XH_BYTES + 2 * WT_BYTES + 2048;
// kind::f16, D = f32; (a) K-major both, N = 32; (b) MN-major both, N = 64
constexpr uint32_t IDESC_DH = (1u << 4) | ((uint32_t)(H >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
constexpr uint32_t IDESC_WG = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) |
                              ((uint32_t)(TM >> 4) << 24);
constexpr int TMEM_COLS = 128;                  // bwd: dh at 0..31, dW accumulator at 64..127

struct Args {
  tr::Data D;
  const int* batch;        // [B] dataset indices
  int B, Tmax;
  const uint8_t* wimg;     // k_trc_pack output: forward B' image | w f32[32] | Wh^T hi | Wh^T lo
  const double* P;         // fp64 parameters (w, b_out)
  float* cache;            // [n_tiles][Tmax][NF][4][128][8]
  double* raw;             // [B]
  double* draw;            // [B]
  double target_scale;
  double n_total;
  const double* draw_in;   // optional caller d_raw (lstm_backward)
  unsigned* dmax;          // max |d_raw| as float bits (zeroed before k_trc_fwd)
  double* partial;         // [n_tiles][n_params]
  int rows;                // sequences per tile (<= 128; the rest of the tile's TMEM lanes idle):
                           // small batches spread over more SMs - the recurrences are latency-bound
};

__device__ __forceinline__ size_t cache_at(int tile, int t, int Tmax, int fld, int g8, int r) {
  return ((((size_t)tile * Tmax + t) * NF + fld) * 4 + g8) * (TM * 8) + (size_t)r * 8;
}

// ---------------------------------------------------------------- weights
// The forward image is tc::pack_weights' (gates pre-scaled by -log2 e, g by
// -2 log2 e); the backward Wh^T images hold the UNSCALED Wh, as B of (a):
// [N = 32 hidden units][K = 128 gates] K-major, hi and lo.
__global__ void k_trc_pack(const double* __restrict__ P, uint8_t* __restrict__ img) {
  const tr::Layout L(H);
  const double L2E = 1.4426950408889634074;
  uint8_t* fw = img;
  float* wout = reinterpret_cast<float*>(img + tc::TILE_BYTES);
  uint8_t* wt = img + tc::TILE_BYTES + 128;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < G * tc::KP; e += gridDim.x * blockDim.x) {
    const int n = e / tc::KP, k = e % tc::KP;
    const double scale = (n >= 64 && n < 96) ? -2.0 * L2E : -L2E;
    double wv = 0.0;
    int seg = 0;
    bool zero = false;
    if (k < 3 * tc::KA) {
      seg = k / tc::KA;
      const int kk = k % tc::KA;
      wv = scale * (kk < 16 ? P[L.oWx + kk * G + n] : P[L.oWh + (kk - 16) * G + n]);
    } else if (k == 3 * tc::KA || k == 3 * tc::KA + 1) {
      seg = k == 3 * tc::KA ? 0 : 2;
      wv = scale * P[L.ob + n];
    } else {
      zero = true;
    }
    const __half whi = __double2half(wv);
    const __half wlo = __double2half(wv - (double)__half2float(whi));
    const __half v = zero ? __float2half(0.0f) : (seg == 2 ? wlo : whi);
    const int kc = k / 8, q = k % 8;
    *reinterpret_cast<__half*>(fw + kc * tc::CHUNK_STRIDE + (n >> 3) * 128 + (n & 7) * 16 + q * 2) = v;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < H * G; e += gridDim.x * blockDim.x) {
    const int n = e / G, k = e % G;  // unit n, gate column k: Wh[n][k]
    const double wv = P[L.oWh + n * G + k];
    const __half whi = __double2half(wv);
    const __half wlo = __double2half(wv - (double)__half2float(whi));
    const int off = (k / 8) * WT_CS + (n >> 3) * 128 + (n & 7) * 16 + (k % 8) * 2;
    *reinterpret_cast<__half*>(wt + off) = whi;
    *reinterpret_cast<__half*>(wt + WT_BYTES + off) = wlo;
  }
  if (blockIdx.x == 0 && threadIdx.x < H) wout[threadIdx.x] = (float)P[L.ow + threadIdx.x];
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ float sigm_s(float u) { return tc::rcp(1.0f + tc::ex2(u)); }   // u = -log2e z
__device__ __forceinline__ float tanh_s(float v) { return fmaf(2.0f, tc::rcp(1.0f + tc::ex2(v)), -1.0f); }  // v = -2log2e z
constexpr float C2 = -2.0f * tc::LOG2E;

// x of row (sequence) at timestep t, raw f64 pairs: loads issued as a
// prefetch and converted only where used (converting at the load would
// stall on it right there)
__device__ __forceinline__ const double* row_src(const tr::Data& D, int idx, int T, int d, int t) {
  return t < T - d ? D.init + (int64_t)(D.init_base[idx] + t) * 16 : D.rows + (D.row_base[idx] + (T - 1 - t)) * 16;
}

// 4 features of row x (features 4 q .. 4 q + 3)
__device__ __forceinline__ void row_x4(const tr::Data& D, int idx, int T, int d, int t, int q, double2* x) {
  const double2* src = reinterpret_cast<const double2*>(row_src(D, idx, T, d, t) + 4 * q);
  x[0] = __ldg(src);
  x[1] = __ldg(src + 1);
}

// 4 floats -> split fp16 half-chunks (8 bytes each), hi at p, lo at p + lo_off
__device__ __forceinline__ void st_split4(uint8_t* p, int lo_off, const float* v) {
  const __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
  const float2 b0 = __half22float2(h0), b1 = __half22float2(h1);
  const __half2 l0 = __floats2half2_rn(v[0] - b0.x, v[1] - b0.y), l1 = __floats2half2_rn(v[2] - b1.x, v[3] - b1.y);
  *reinterpret_cast<uint2*>(p) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
  *reinterpret_cast<uint2*>(p + lo_off) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&l0), *reinterpret_cast<const uint32_t*>(&l1));
}

// 8 floats -> split fp16 chunks, stored at p (hi) and p + lo_off (lo)
__device__ __forceinline__ void st_split8(uint8_t* p, int lo_off, const float* v) {
  uint4 hi, lo;
  split8(v, hi, lo);
  *reinterpret_cast<uint4*>(p) = hi;
  *reinterpret_cast<uint4*>(p + lo_off) = lo;
}

// ---------------------------------------------------------------- forward
// NWG = 4 warpgroups per tile: every warpgroup covers the tile's 128 rows
// (TMEM lanes) for 8 of the 32 hidden units (its gate columns), so each
// timestep's MUFU / FMA epilogue is spread over 512 threads.
constexpr int NWG = 4;
constexpr int FWD_THREADS = NWG * TM;

__global__ void __launch_bounds__(FWD_THREADS, 1) k_trc_fwd(Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* Bw = smem;
  uint8_t* A = smem + tc::TILE_BYTES;
  float* wout = reinterpret_cast<float*>(smem + tc::TILE_BYTES + tc::A_BYTES);
  double* rawp = reinterpret_cast<double*>(wout + 32);       // [NWG][TM] partial readout sums
  float* hsum = reinterpret_cast<float*>(rawp + NWG * TM);   // [32 units][TM + 1] sum_t h_t
  double* drs = reinterpret_cast<double*>(hsum + 32 * (TM + 1));  // [TM] d_raw
  uint64_t* bar = reinterpret_cast<uint64_t*>(drs + TM);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, wg = tid / TM, r = tid % TM, warp = tid >> 5, tile = blockIdx.x;
  const int g8 = wg;  // this thread's 8 hidden units: 8 g8 .. 8 g8 + 7
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wimg);
    uint4* dst = reinterpret_cast<uint4*>(Bw);
    for (int i = tid; i < tc::TILE_BYTES / 16; i += FWD_THREADS) dst[i] = __ldg(src + i);
    if (tid < 32) wout[tid] = __ldg(reinterpret_cast<const float*>(a.wimg + tc::TILE_BYTES) + tid);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int b = tile * a.rows + r;
  int idx = 0, T = 0, d = 0;
  if (r < a.rows && b < a.B) {
    idx = a.batch[b];
    T = a.D.Tlen[idx];
    d = a.D.depth[idx];
  }
  double raw = 0.0;  // this warpgroup's units' readout, summed over timesteps
  float c[8], hs[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) c[u] = hs[u] = 0.0f;
  {
    const float z8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    tc::put_h8(A, r, g8, z8);
    if (wg == 0) tc::put_bias_ones(A, r);
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t a_base = tc::smem_u32(A), b_base = tc::smem_u32(Bw);
  uint32_t phase = 0;
  double2 x[2];  // features 4 g8 .. 4 g8 + 3 of x_t: each warpgroup writes a quarter of A's x part
  if (T > 0) row_x4(a.D, idx, T, d, 0, g8, x);
  uint8_t* xq = A + (g8 >> 1) * tc::CHUNK_STRIDE + (r >> 3) * 128 + (r & 7) * 16 + (g8 & 1) * 8;
  for (int t = 0; t < a.Tmax; ++t) {
    const bool act = t < T;
    {  // rows past their length feed zeros; their results are unused
      const float xz[4] = {act ? (float)x[0].x : 0.0f, act ? (float)x[0].y : 0.0f, act ? (float)x[1].x : 0.0f,
                           act ? (float)x[1].y : 0.0f};
      st_split4(xq, 6 * tc::CHUNK_STRIDE, xz);  // hi in chunk g8 / 2, lo in chunk 6 + g8 / 2
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
#pragma unroll
      for (int s = 0; s < tc::KSTEPS; ++s)
        tc::mma_f16(tmem, tc::umma_desc(a_base + tc::a_chunk(s) * tc::CHUNK_STRIDE, tc::CHUNK_STRIDE, 128),
                    tc::umma_desc(b_base + s * 2 * tc::CHUNK_STRIDE, tc::CHUNK_STRIDE, 128), s > 0);
      tc::mma_commit(bar);
    }
    if (t + 1 < T) row_x4(a.D, idx, T, d, t + 1, g8, x);  // next row in flight across the UMMA
    tc::mbar_wait(bar, phase);
    phase ^= 1u;
    tc::fence_after();
    float ui[8], uf[8], vg[8], uo[8];
    tc::tmem_ld8(lane_addr + 0 * 32 + g8 * 8, ui);
    tc::tmem_ld8(lane_addr + 1 * 32 + g8 * 8, uf);
    tc::tmem_ld8(lane_addr + 2 * 32 + g8 * 8, vg);
    tc::tmem_ld8(lane_addr + 3 * 32 + g8 * 8, uo);
    tc::tmem_wait_ld();
    float gi[8], gf[8], gg[8], go[8], h8[8];
    float acc = 0.0f;
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      // gates with shared reciprocals (Montgomery batch inversion: 1/a =
      // b/(ab)): (i, f) and (g, o) per unit, tanh(c) per pair of units -
      // 5 ex2 + 2.5 rcp per unit instead of 5 + 5; exponents clamped at 40
      // so the products stay finite (sigma >= 2^-40)
      float tcn[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int v = u + q;
        const float ti = 1.0f + tc::ex2(fminf(ui[v], 40.0f)), tf = 1.0f + tc::ex2(fminf(uf[v], 40.0f));
        const float tg = 1.0f + tc::ex2(fminf(vg[v], 40.0f)), to = 1.0f + tc::ex2(fminf(uo[v], 40.0f));
        const float r1 = tc::rcp(ti * tf), r2 = tc::rcp(tg * to);
        gi[v] = tf * r1;
        gf[v] = ti * r1;
        gg[v] = fmaf(2.0f, to * r2, -1.0f);
        go[v] = tg * r2;
        const float cn = fmaf(gf[v], c[v], gi[v] * gg[v]);
        c[v] = act ? cn : c[v];
        tcn[q] = 1.0f + tc::ex2(fminf(C2 * c[v], 40.0f));
      }
      const float r3 = tc::rcp(tcn[0] * tcn[1]);
      h8[u] = go[u] * fmaf(2.0f, tcn[1] * r3, -1.0f);
      h8[u + 1] = go[u + 1] * fmaf(2.0f, tcn[0] * r3, -1.0f);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        acc = fmaf(h8[u + q], wout[g8 * 8 + u + q], acc);
        hs[u + q] += act ? h8[u + q] : 0.0f;
      }
    }
    if (act) {
      float* cc = a.cache + cache_at(tile, t, a.Tmax, 0, g8, r);
      const size_t fs = (size_t)4 * TM * 8;  // field stride
      *reinterpret_cast<float4*>(cc) = make_float4(gi[0], gi[1], gi[2], gi[3]);
      *reinterpret_cast<float4*>(cc + 4) = make_float4(gi[4], gi[5], gi[6], gi[7]);
      *reinterpret_cast<float4*>(cc + fs) = make_float4(gf[0], gf[1], gf[2], gf[3]);
      *reinterpret_cast<float4*>(cc + fs + 4) = make_float4(gf[4], gf[5], gf[6], gf[7]);
      *reinterpret_cast<float4*>(cc + 2 * fs) = make_float4(gg[0], gg[1], gg[2], gg[3]);
      *reinterpret_cast<float4*>(cc + 2 * fs + 4) = make_float4(gg[4], gg[5], gg[6], gg[7]);
      *reinterpret_cast<float4*>(cc + 3 * fs) = make_float4(go[0], go[1], go[2], go[3]);
      *reinterpret_cast<float4*>(cc + 3 * fs + 4) = make_float4(go[4], go[5], go[6], go[7]);
      *reinterpret_cast<float4*>(cc + 4 * fs) = make_float4(c[0], c[1], c[2], c[3]);
      *reinterpret_cast<float4*>(cc + 4 * fs + 4) = make_float4(c[4], c[5], c[6], c[7]);
      raw = fadd(raw, (double)acc);
    }
    tc::put_h8(A, r, g8, h8);  // the UMMA that read A has completed
    tc::fence_before();
  }
  // raw = T b_out + the warpgroups' sums (fixed order), d_raw, and this
  // tile's dw = sum_rows d_raw sum_t h_t and db_out = sum_rows T d_raw
  const tr::Layout L(H);
  rawp[wg * TM + r] = raw;
#pragma unroll
  for (int u = 0; u < 8; ++u) hsum[(g8 * 8 + u) * (TM + 1) + r] = hs[u];
  __syncthreads();
  if (wg == 0) {
    double dr = 0.0;
    if (r < a.rows && b < a.B) {
      double rw = fmul((double)T, a.P[L.obout]);
      for (int q = 0; q < NWG; ++q) rw = fadd(rw, rawp[q * TM + r]);
      dr = a.draw_in ? a.draw_in[b] : fdiv(fmul(2.0, fsub(fadd(rw, a.target_scale), a.D.logt[idx])), a.n_total);
      a.raw[b] = rw;
      a.draw[b] = dr;
      atomicMax(a.dmax, __float_as_uint(fabsf((float)dr)));  // |d_raw| as float bits: monotonic
    }
    drs[r] = dr;
    rawp[r] = (double)T;  // (reused) this row's length
  }
  __syncthreads();
  double* out = a.partial + (size_t)tile * L.n;
  if (tid < H) {
    double acc = 0.0;
    for (int q = 0; q < TM; ++q) acc = fadd(acc, fmul((double)hsum[tid * (TM + 1) + q], drs[q]));
    out[L.ow + tid] = acc;
  } else if (tid == H) {
    double acc = 0.0;
    for (int q = 0; q < TM; ++q) acc = fadd(acc, fmul(rawp[q], drs[q]));
    out[L.obout] = acc;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
}

// ---------------------------------------------------------------- backward
// operand element offsets (bytes): dz[row r][gate m] (fp16) and
// xh[row r][feature n]: chunk (8 gates / features) stride 2048, row group 128
__device__ __forceinline__ int op_off(int chunk, int r) { return chunk * 2048 + (r >> 3) * 128 + (r & 7) * 16; }

// one thread's cache data for timestep t: its 8 units' gates and cell, and
// the previous timestep's o and c (h_{t-1} = o tanh c)
struct Rec {
  float4 gi[2], gf[2], gg[2], go[2], cc[2], op[2], cp[2];
};
__device__ __forceinline__ void load_rec(const float* cache, int tile, int t, int Tmax, int g8, int r, Rec& q) {
  const float* ce = cache + cache_at(tile, t, Tmax, 0, g8, r);
  const size_t fs = (size_t)4 * TM * 8;
  const float4* p = reinterpret_cast<const float4*>(ce);
  const size_t f4 = fs / 4;
  q.gi[0] = __ldcs(p); q.gi[1] = __ldcs(p + 1);
  q.gf[0] = __ldcs(p + f4); q.gf[1] = __ldcs(p + f4 + 1);
  q.gg[0] = __ldcs(p + 2 * f4); q.gg[1] = __ldcs(p + 2 * f4 + 1);
  q.go[0] = __ldcs(p + 3 * f4); q.go[1] = __ldcs(p + 3 * f4 + 1);
  q.cc[0] = __ldcs(p + 4 * f4); q.cc[1] = __ldcs(p + 4 * f4 + 1);
  if (t > 0) {
    const float4* pp = reinterpret_cast<const float4*>(cache + cache_at(tile, t - 1, Tmax, 0, g8, r));
    q.op[0] = __ldg(pp + 3 * f4); q.op[1] = __ldg(pp + 3 * f4 + 1);
    q.cp[0] = __ldg(pp + 4 * f4); q.cp[1] = __ldg(pp + 4 * f4 + 1);
  } else {
    q.op[0] = q.op[1] = q.cp[0] = q.cp[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
__device__ __forceinline__ float f4at(const float4* v, int u) {
  const float4 w = v[u >> 2];
  return (u & 3) == 0 ? w.x : (u & 3) == 1 ? w.y : (u & 3) == 2 ? w.z : w.w;
}

constexpr int BWD_THREADS = NWG * TM;

__global__ void __launch_bounds__(BWD_THREADS, 1) k_trc_bwd(Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* dzb = smem;                        // hi | lo
  uint8_t* xhb = smem + 2 * DZ_BYTES;         // hi | lo
  uint8_t* wtb = xhb + 2 * XH_BYTES;          // Wh^T hi | lo
  uint64_t* bar = reinterpret_cast<uint64_t*>(wtb + 2 * WT_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  float* wsh = reinterpret_cast<float*>(tmem_slot + 4);  // [H] readout weights (f32)
  const int tid = threadIdx.x, wg = tid / TM, r = tid % TM, warp = tid >> 5, tile = blockIdx.x;
  const int g8 = wg;
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wimg + tc::TILE_BYTES + 128);
    uint4* dst = reinterpret_cast<uint4*>(wtb);
    for (int i = tid; i < 2 * WT_BYTES / 16; i += BWD_THREADS) dst[i] = __ldg(src + i);
    if (tid < H) wsh[tid] = __ldg(reinterpret_cast<const float*>(a.wimg + tc::TILE_BYTES) + tid);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int b = tile * a.rows + r;
  int idx = 0, T = 0, d = 0;
  double dr = 0.0;
  if (r < a.rows && b < a.B) {
    idx = a.batch[b];
    T = a.D.Tlen[idx];
    d = a.D.depth[idx];
    dr = a.draw[b];
  }
  // S = 2^-e, 2^e the power of two just above max |d_raw| (k_trc_fwd's
  // atomicMax): the scaled dz stay O(1), inside fp16's range; exact to undo
  int e = 0;
  {
    const float m = __uint_as_float(*a.dmax);
    if (m > 0.0f && m < 1e30f) frexpf(m, &e);
    e = max(-100, min(100, e));
  }
  const float S = ldexpf(1.0f, -e), invS = ldexpf(1.0f, e);
  const float drs = (float)dr * S;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_dh = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t dz_base = tc::smem_u32(dzb), xh_base = tc::smem_u32(xhb), wt_base = tc::smem_u32(wtb);
  const uint32_t t_dh = tmem, t_dw = tmem + 64;
  // UMMA descriptor bases: (a) dz K-major [hi, lo], Wh^T [hi, lo];
  // (b) dz MN-major [hi, lo], [x | h | 1] MN-major [hi, lo]
  const uint64_t dA[2] = {tc::umma_desc(dz_base, 2048, 128), tc::umma_desc(dz_base + DZ_BYTES, 2048, 128)};
  const uint64_t dW[2] = {tc::umma_desc(wt_base, WT_CS, 128), tc::umma_desc(wt_base + WT_BYTES, WT_CS, 128)};
  const uint64_t dB[2] = {tc::umma_desc(dz_base, 128, 2048), tc::umma_desc(dz_base + DZ_BYTES, 128, 2048)};
  const uint64_t dX[2] = {tc::umma_desc(xh_base, 128, 2048), tc::umma_desc(xh_base + XH_BYTES, 128, 2048)};
  float dcn[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) dcn[u] = 0.0f;
  float wj[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) wj[u] = wsh[g8 * 8 + u];
  uint32_t phase = 0;
  Rec q;
  double2 x[2];  // features 4 g8 .. 4 g8 + 3 of x_t (each warpgroup writes a quarter of x)
  {
    const int t0 = a.Tmax - 1;
    if (t0 < T) {
      load_rec(a.cache, tile, t0, a.Tmax, g8, r, q);
      row_x4(a.D, idx, T, d, t0, g8, x);
    }
  }
  for (int t = a.Tmax - 1; t >= 0; --t) {
    const bool act = t < T;
    const bool have_dh = t < a.Tmax - 1;  // the previous step's dz . Wh^T is in TMEM
    float dh[8];
    if (have_dh) {
      tc::tmem_ld8(lane_dh + g8 * 8, dh);
      tc::tmem_wait_ld();
    }
    float zi[8], zf[8], zg[8], zo[8], hp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!act) {
        zi[u] = zf[u] = zg[u] = zo[u] = hp[u] = 0.0f;
        dcn[u] = 0.0f;
        continue;
      }
      const float gi = f4at(q.gi, u), gf = f4at(q.gf, u), gg = f4at(q.gg, u), go = f4at(q.go, u);
      const float c_t = f4at(q.cc, u), c_prev = f4at(q.cp, u);
      hp[u] = t > 0 ? f4at(q.op, u) * tanh_s(C2 * c_prev) : 0.0f;  // h_{t-1}
      const float tcv = tanh_s(C2 * c_t);
      const float dhv = fmaf(wj[u], drs, have_dh ? dh[u] : 0.0f);  // S dh
      const float d_o = dhv * tcv;
      const float dc = fmaf(dhv * go, fmaf(-tcv, tcv, 1.0f), dcn[u]);
      const float di = dc * gg, df = dc * c_prev, dg = dc * gi;
      dcn[u] = dc * gf;
      zi[u] = di * gi * (1.0f - gi);
      zf[u] = df * gf * (1.0f - gf);
      zg[u] = dg * fmaf(-gg, gg, 1.0f);
      zo[u] = d_o * go * (1.0f - go);
    }
    // dz (scaled) -> gate chunks g8 (i), 4 + g8 (f), 8 + g8 (g), 12 + g8 (o); h_{t-1} -> feature chunk 2 + g8
    st_split8(dzb + op_off(g8, r), DZ_BYTES, zi);
    st_split8(dzb + op_off(4 + g8, r), DZ_BYTES, zf);
    st_split8(dzb + op_off(8 + g8, r), DZ_BYTES, zg);
    st_split8(dzb + op_off(12 + g8, r), DZ_BYTES, zo);
    st_split8(xhb + op_off(2 + g8, r), XH_BYTES, hp);
    {  // a quarter of x_t (features 4 g8 ..), and the ones column (db) / zero padding
      const float xz[4] = {act ? (float)x[0].x : 0.0f, act ? (float)x[0].y : 0.0f, act ? (float)x[1].x : 0.0f,
                           act ? (float)x[1].y : 0.0f};
      st_split4(xhb + op_off(g8 >> 1, r) + (g8 & 1) * 8, XH_BYTES, xz);
      if (g8 < 2) {
        const float one[4] = {(act && g8 == 0) ? 1.0f : 0.0f, 0, 0, 0};
        st_split4(xhb + op_off(6, r) + g8 * 8, XH_BYTES, one);
      } else {
        const float zero4[4] = {0, 0, 0, 0};
        st_split4(xhb + op_off(7, r) + (g8 - 2) * 8, XH_BYTES, zero4);
      }
    }
    // the next (earlier) timestep's cache and x in flight across the UMMAs
    if (t > 0 && t - 1 < T) {
      load_rec(a.cache, tile, t - 1, a.Tmax, g8, r, q);
      row_x4(a.D, idx, T, d, t - 1, g8, x);
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after();
      // descriptors: the operand addresses are fixed, so each UMMA's pair is
      // a loop-invariant base plus a constant (the address field is addr >> 4)
#pragma unroll
      for (int p = 0; p < 3; ++p) {  // hi.hi, lo.hi, hi.lo
        const uint64_t da = dA[p == 1], dw = dW[p == 2];
#pragma unroll
        for (int s = 0; s < G / 16; ++s)
          // (a) S dh_next[rows x 32] = dz[rows x gates] . Wh^T: K = gates 16s..16s+15
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(t_dh),
              "l"(da + (uint64_t)(s * 2 * 2048 >> 4)), "l"(dw + (uint64_t)(s * 2 * WT_CS >> 4)), "r"(IDESC_DH),
              "r"((p > 0 || s > 0) ? 1u : 0u)
              : "memory");
      }
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const uint64_t da = dB[p == 1], dx = dX[p == 2];
#pragma unroll
        for (int s = 0; s < TM / 16; ++s) {
          // (b) S dW^T[gates x 64] += dz^T[gates x rows] . [x|h|1][rows x 64]: K = rows 16s..16s+15
          // (MN-major: K blocks of 8 rows are 128 B apart, MN blocks of 8 are 2048 B apart)
          const bool accum = (t < a.Tmax - 1) || p > 0 || s > 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(t_dw),
              "l"(da + (uint64_t)(s * 256 >> 4)), "l"(dx + (uint64_t)(s * 256 >> 4)), "r"(IDESC_WG),
              "r"(accum ? 1u : 0u)
              : "memory");
        }
      }
      tc::mma_commit(bar);
    }
    tc::mbar_wait(bar, phase);
    phase ^= 1u;
    tc::fence_after();
  }
  // ---- this tile's dW^T (TMEM lanes = gate columns) / S into its partial
  const tr::Layout L(H);
  double* out = a.partial + (size_t)tile * L.n;
  {
    const int m = r;  // TMEM lane = gate column
    const uint32_t la = t_dw + ((uint32_t)((warp & 3) * 32) << 16);
    for (int c8 = wg; c8 < 7; c8 += NWG) {
      float v[8];
      tc::tmem_ld8(la + c8 * 8, v);
      tc::tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = c8 * 8 + u;
        const double gv = (double)(v[u] * invS);
        if (col < 16) out[L.oWx + col * G + m] = gv;
        else if (col < 48) out[L.oWh + (col - 16) * G + m] = gv;
        else if (col == 48) out[L.ob + m] = gv;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

}  // namespace trc
}  // namespace ts
