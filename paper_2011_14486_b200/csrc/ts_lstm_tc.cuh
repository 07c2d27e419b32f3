// ts_lstm_tc.cuh - FAST scoring path: the LSTM value network on the 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM), fused with bias, gates,
// cell update, readout and exp.
//
// Per timestep each row (one state) computes z = [x | h] . [Wx; Wh] + b, a
// [1 x 48] x [48 x 128] product.  A warpgroup stacks 128 states as the
// M=128 rows of one UMMA: D[128 x 128] (fp32, TMEM) = A[128 x K] . B[128 x K]^T
// with fp16 operands split hi/lo and concatenated along K,
//     A' = [a_hi | a_lo | a_hi | 1 1 0..0],  B' = [W_hi ; W_hi ; W_lo ; b_hi b_lo 0..0]
// (K = 3*48 + 16 = 160, ten K=16 UMMAs; the second a_hi is the first one
// re-read through the UMMA descriptor, not a copy) so
// z ~= a_hi W_hi + a_lo W_hi + a_hi W_lo + b
// with 22-bit operands and fp32 accumulation (|dV|/V <= 1e-4, the north-star
// fp32 tolerance).  The gate columns of B' are pre-scaled by -log2(e)
// (i, f, o) and -2 log2(e) (g) so every gate costs one ex2.approx and one
// rcp.approx on the MUFU pipe: sigma = 1/(1 + 2^u), tanh = 2/(1 + 2^v) - 1.
//
// A CTA holds NWG = 4 warpgroups (512 threads, one CTA per SM) that share the
// weight tile B' in shared memory and own one A tile, one 128-column TMEM
// accumulator and one mbarrier each; they run independent tiles so one
// warpgroup's UMMA + commit latency hides under the others' MUFU work.
// One elected thread per warpgroup issues the UMMAs; tcgen05.commit arrives
// on the warpgroup's mbarrier; thread = TMEM lane = state reads its row with
// tcgen05.ld, updates c (registers), h, the readout, and writes the next A
// row (fp16 hi/lo) in the canonical K-major no-swizzle layout.
//
// Batch independence: every row's arithmetic depends only on its own inputs,
// so a state of depth d in a tile that starts earlier (at T - d_max) replays
// the shared unscheduled prefix rows and reaches exactly the fast prefix
// state of position T - d.  States are bucketed by depth (counting sort) so
// tiles waste no timesteps.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "ts_core.cuh"
#include "ts_f16.cuh"

namespace ts {
namespace tc {

constexpr int TM = 128;                   // states per tile (UMMA M)
constexpr int GN = 128;                   // gate columns 4H (UMMA N), H = 32
constexpr int KA = 48;                    // [x(16) | h(32)]
constexpr int KP = 3 * KA + 16;           // split-concatenated K + bias block = 160
constexpr int KCH = KP / 8;               // 16-byte K chunks = 20
constexpr int KSTEPS = KP / 16;           // UMMAs per timestep = 10
constexpr int CHUNK_STRIDE = TM * 16;     // bytes between K chunks (LBO) = 2048
constexpr int TILE_BYTES = KCH * CHUNK_STRIDE;  // 40960: the B' weight image
// A holds a_hi and a_lo once (the third product a_hi.W_lo re-reads a_hi's
// chunks through its descriptor) plus the bias block: 14 chunks, so every
// row costs two 16-byte stores per K chunk instead of three
constexpr int A_KCH = 2 * (KA / 8) + 2;  // 14
constexpr int A_BYTES = A_KCH * CHUNK_STRIDE;  // 28672
constexpr int NWG = 4;                    // warpgroups (tiles in flight) per CTA
constexpr int THREADS = NWG * TM;
constexpr int SMEM_BYTES = TILE_BYTES + NWG * A_BYTES + 1024;  // B, NWG x A, readout + barriers
constexpr int smem_bytes(int nwg) { return TILE_BYTES + nwg * A_BYTES + 1024; }
// A chunk read by UMMA step s (K = 16 = two chunks): a_hi . W_hi (s 0-2),
// a_lo . W_hi (3-5), a_hi . W_lo (6-8, a_hi again), bias (9)
__device__ __forceinline__ int a_chunk(int s) { return s < 6 ? 2 * s : s < 9 ? 2 * (s - 6) : 12; }
constexpr int PRE_STRIDE = 72;            // floats per prefix position: h[32], c[32], raw (f64)
constexpr float LOG2E = 1.4426950408889634f;

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // tcgen05 shared-memory descriptor, K-major, SWIZZLE_NONE, version 1
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// kind::f16, A=B=F16, D=F32, K-major both, N=128, M=128
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(GN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void wg_sync(int wg) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + wg), "r"(TM) : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- epilogue
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Upper clamp only: 2^x for very negative x underflows to 0, which the
// fused cell algebra tolerates (t = 1); the upper bound keeps the triple
// products of (1 + 2^x) below 2^128.
__device__ __forceinline__ float clamp40(float x) { return fminf(x, 40.0f); }

// 2^x on the FMA/ALU pipes (relieves the MUFU pipe, the LSTM's binding
// unit): round-to-nearest split x = j + f with the 1.5*2^23 trick,
// degree-5 near-minimax polynomial for 2^f on [-1/2, 1/2] (max rel err
// 2.3e-7, the same order as ex2.approx), exponent add.  |x| <= 40.
__device__ __forceinline__ float ex2_fma(float x) {
  const float t = __fadd_rn(x, 12582912.0f);
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  float p = fmaf(0.0013276466634124517f, f, 0.009675540961325169f);
  p = fmaf(p, f, 0.05550713464617729f);
  p = fmaf(p, f, 0.24022120237350464f);
  p = fmaf(p, f, 0.6931469440460205f);
  p = fmaf(p, f, 1.0000001192092896f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// ex2_fma for a unit pair on the paired fp32 pipe (FADD2 / FFMA2), the
// argument clamped to [-40, 40] (below -40, 1 + 2^x is 1 in fp32 either way)
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  x.x = fmaxf(x.x, -40.0f);
  x.y = fmaxf(x.y, -40.0f);
  const float2 sh = make_float2(12582912.0f, 12582912.0f), nsh = make_float2(-12582912.0f, -12582912.0f);
  const float2 t = __fadd2_rn(x, sh);
  const float2 f = __fadd2_rn(x, make_float2(-__fadd_rn(t.x, -12582912.0f), -__fadd_rn(t.y, -12582912.0f)));
  (void)nsh;
  float2 p = __ffma2_rn(make_float2(0.0013276466634124517f, 0.0013276466634124517f), f,
                        make_float2(0.009675540961325169f, 0.009675540961325169f));
  p = __ffma2_rn(p, f, make_float2(0.05550713464617729f, 0.05550713464617729f));
  p = __ffma2_rn(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__int_as_float(__float_as_int(p.x) + ((__float_as_int(t.x) - 0x4B400000) << 23)),
                     __int_as_float(__float_as_int(p.y) + ((__float_as_int(t.y) - 0x4B400000) << 23)));
}

#ifndef TS_QUAD_RCP
#ifndef TS_RAT_TANH
#define TS_RAT_TANH 0  // 1: tanh(c') as a rational on the FMA pipe (cell_group; measured equal, off), 0: ex2 on MUFU
#endif
// tanh rational (odd P / even Q in c'^2): Eigen's float tanh coefficients
// (generic_fast_tanh_float), a published minimax fit; error checked in
// tests/test_host.py against libm tanh
constexpr float kTanhClamp = 7.90531110763549805f;
constexpr float kTA1 = 4.89352455891786e-03f, kTA3 = 6.37261928875436e-04f, kTA5 = 1.48572235717979e-05f,
                kTA7 = 5.12229709037114e-08f, kTA9 = -8.60467152213735e-11f, kTA11 = 2.00018790482477e-13f,
                kTA13 = -2.76076847742355e-16f;
constexpr float kTB0 = 4.89352518554385e-03f, kTB2 = 2.26843463243900e-03f, kTB4 = 1.18534705686654e-04f,
                kTB6 = 1.19825839466702e-06f;
#define TS_QUAD_RCP 0  // 1: the output gate's reciprocal shared by four units (cell_group; measured 1%, off)
#endif
#ifndef TS_FMA_EXP
#define TS_FMA_EXP 0  // how many of the 5 per-unit exponentials use ex2_fma
#endif
__device__ __forceinline__ float ex2_sel(float x, int slot) {
  return slot < TS_FMA_EXP ? ex2_fma(x) : ex2(x);
}
// a unit pair's exponential of slot `slot` (the arguments already clamped
// above at 40)
__device__ __forceinline__ float2 ex2_pair(float a, float b, int slot) {
  if (slot < TS_FMA_EXP) return ex2_fma2(make_float2(a, b));
  return make_float2(ex2(a), ex2(b));
}

// Stores 16-byte chunk `kc` of row `r` in the canonical no-swizzle layout.
__device__ __forceinline__ void st_chunk(uint8_t* A, int kc, int r, const uint4& v) {
  *reinterpret_cast<uint4*>(A + kc * CHUNK_STRIDE + (r >> 3) * 128 + (r & 7) * 16) = v;
}

// x part, pre-split (x4 = intrinsic hi, lo, acquired hi, lo): chunks q = 0
// (intrinsic), 1 (acquired) of the hi and lo segments
__device__ __forceinline__ void put_x(uint8_t* A, int r, const uint4* x4) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    st_chunk(A, 0 * 6 + q, r, x4[2 * q]);
    st_chunk(A, 1 * 6 + q, r, x4[2 * q + 1]);
  }
}

// h part: 8 units of group g8 -> chunk q = 2 + g8 of the hi and lo segments
__device__ __forceinline__ void put_h8(uint8_t* A, int r, int g8, const float* h8) {
  uint4 hi, lo;
  split8(h8, hi, lo);
  st_chunk(A, 0 * 6 + 2 + g8, r, hi);
  st_chunk(A, 1 * 6 + 2 + g8, r, lo);
}

// bias block (A chunks 12, 13 against B' K entries 144..159): 1.0, 1.0
// multiplying b_hi, b_lo, rest 0
__device__ __forceinline__ void put_bias_ones(uint8_t* A, int r) {
  const uint32_t one_one = 0x3C003C00u;  // two fp16 1.0
  st_chunk(A, 12, r, make_uint4(one_one, 0u, 0u, 0u));
  st_chunk(A, 13, r, make_uint4(0u, 0u, 0u, 0u));
}

// ---------------------------------------------------------------- kernel
// Tiles: sorted positions [128*tile, 128*tile + 128); perm maps a sorted
// position to the original state index; depth is sorted descending, so the
// tile's first state has its maximum depth.  record_prefix: a single tile
// whose row 0 is the all-unscheduled state (depth 0, t0 = 0); thread 0
// writes (h, c, raw) before every timestep into `pre` (the fast prefix).
struct TcArgs {
  const uint8_t* wpack;     // B' image (TILE_BYTES) + readout w[32] f32
  const uint4* initx;       // [T][4] unscheduled rows, split fp16: intrinsic hi, lo, acquired hi, lo
  const uint4* rowsx;       // [n_records][2] acquired half of scheduled rows, split fp16: hi, lo
  const int64_t* offsets;   // [n+1]
  const int* perm;          // [n] sorted position -> state
  const int64_t* rowoff;    // [T+1] decision-major row offsets (k_depth_scan)
  float* pre;               // [(T+1)][PRE_STRIDE] fast prefix (h, c, raw)
  double* out;              // [n] V
  int64_t n;
  int T;
  int n_tiles;
  int record_prefix;
  double target_scale;
  double b_out;
  int* tile_counter;        // zeroed before the launch: dynamic tile scheduler (null: static)
};

// x at timestep t: intrinsic half from the stage's init row (the same for
// every row of the tile), acquired half from the init row (unscheduled) or
// the state's scheduled row; both already split into fp16 hi/lo
__device__ __forceinline__ void load_x(const uint4* init_row, const uint4* acq, uint4* x4) {
  x4[0] = __ldg(init_row);
  x4[1] = __ldg(init_row + 1);
  x4[2] = __ldg(acq);
  x4[3] = __ldg(acq + 1);
}

// One group of 8 hidden units of one row: gate pre-activations (TMEM,
// pre-scaled by -log2 e / -2 log2 e) -> c (updated in place), h8, readout.
// Shared by both tensor-core kernels so their rows are bit-identical.
__device__ __forceinline__ void cell_group(uint32_t lane_addr, int g8, float* c, float* h8, float& acc,
                                           const float* wout) {
  float ui[8], uf[8], vg[8], uo[8];
  tmem_ld8(lane_addr + 0 * 32 + g8 * 8, ui);
  tmem_ld8(lane_addr + 1 * 32 + g8 * 8, uf);
  tmem_ld8(lane_addr + 2 * 32 + g8 * 8, vg);
  tmem_ld8(lane_addr + 3 * 32 + g8 * 8, uo);
  tmem_wait_ld();
  // Fused cell algebra.  With t_x = 1 + 2^u_x: sigma = 1/t and
  // tanh = (1 - 2^v)/(1 + 2^v), so
  //   c' = f c + i g = (c t_i t_g + (1 - e_g) t_f) / (t_f t_i t_g)
  //   h  = o tanh(c') = (1 - e_c) / ((1 + e_o)(1 + e_c)).
  // Units in pairs share each reciprocal (Montgomery's batch
  // inversion: 1/a = b/(ab), 1/b = a/(ab)): 5 ex2 + 1 rcp per unit.
  // The denominators are pre-scaled through the FMA constants (t_i by
  // 2^-60, 1 + e_o by 2^-40, exact) so the pair products stay inside
  // [2^-120, 2^120] with the exponents clamped at 40 (sigma >= 2^-40).
  constexpr float S1 = 8.673617379884035e-19f;  // 2^-60
  constexpr float S2 = 9.094947017729282e-13f;  // 2^-40
  constexpr float C2 = -2.0f * LOG2E;
  // The two units of a pair go through the sm_100 paired fp32 pipe
  // (FFMA2 / FMUL2: two IEEE fmas / products per instruction, each lane the
  // same rounding as FFMA / FMUL, so the values are the scalar code's bit for
  // bit) - the epilogue is issue-bound next to its MUFU work.
  const float2 s1 = make_float2(S1, S1), ns1 = make_float2(-S1, -S1);
#if TS_QUAD_RCP
  // the output gate's reciprocal is shared by four units (one rcp per
  // quad): 1 + e_o and 1 + e_c clamped at 2^30 and scaled by 2^-30 keep the
  // product of four denominators inside [2^-120, 2^120]; sigma(o) and
  // tanh(c) then saturate at 2^-30 instead of 2^-40 (|error| < 1e-9)
  constexpr float S2Q = 9.313225746154785e-10f;  // 2^-30
  const float2 s2 = make_float2(S2Q, S2Q), ns2 = make_float2(-S2Q, -S2Q);
#pragma unroll
  for (int u4 = 0; u4 < 8; u4 += 4) {
    float2 ecq[2], d2q[2];
#pragma unroll
    for (int hq = 0; hq < 2; ++hq) {
      const int u = u4 + 2 * hq, j = g8 * 8 + u;
      const float2 ei = ex2_pair(clamp40(ui[u]), clamp40(ui[u + 1]), 0);
      const float2 ef = ex2_pair(clamp40(uf[u]), clamp40(uf[u + 1]), 1);
      const float2 eg = ex2_pair(clamp40(vg[u]), clamp40(vg[u + 1]), 2);
      const float2 eo = ex2_pair(fminf(uo[u], 30.0f), fminf(uo[u + 1], 30.0f), 3);
      const float2 ti = __ffma2_rn(ei, s1, s1);                                  // 2^-60 t_i
      const float2 tig = __ffma2_rn(ti, eg, ti);                                 // 2^-60 t_i t_g
      const float2 gm = __ffma2_rn(eg, ns1, s1);                                 // 2^-60 (1 - e_g)
      const float2 num = __ffma2_rn(make_float2(c[j], c[j + 1]), tig, __ffma2_rn(gm, ef, gm));
      const float2 d1 = __ffma2_rn(tig, ef, tig);                                // 2^-60 t_f t_i t_g
      const float r1 = rcp(d1.x * d1.y);
      const float2 cn = __fmul2_rn(num, __fmul2_rn(make_float2(d1.y, d1.x), make_float2(r1, r1)));
      c[j] = cn.x;
      c[j + 1] = cn.y;
      const float2 cc = __fmul2_rn(make_float2(C2, C2), cn);
      ecq[hq] = ex2_pair(fminf(cc.x, 30.0f), fminf(cc.y, 30.0f), 4);
      const float2 to = __ffma2_rn(eo, s2, s2);                                  // 2^-30 (1 + e_o)
      d2q[hq] = __ffma2_rn(to, ecq[hq], to);                                     // 2^-30 (1 + e_o)(1 + e_c)
    }
    const float p0 = d2q[0].x * d2q[0].y, p1 = d2q[1].x * d2q[1].y;
    const float rq = rcp(p0 * p1);
    const float r20 = p1 * rq, r21 = p0 * rq;  // 1 / p0, 1 / p1
#pragma unroll
    for (int hq = 0; hq < 2; ++hq) {
      const int u = u4 + 2 * hq, j = g8 * 8 + u;
      const float r2 = hq ? r21 : r20;
      const float2 hh = __fmul2_rn(__ffma2_rn(ecq[hq], ns2, s2),
                                   __fmul2_rn(make_float2(d2q[hq].y, d2q[hq].x), make_float2(r2, r2)));
      h8[u] = hh.x;
      h8[u + 1] = hh.y;
      acc = fmaf(hh.x, wout[j], acc);
      acc = fmaf(hh.y, wout[j + 1], acc);
    }
  }
#else
  const float2 s2 = make_float2(S2, S2), ns2 = make_float2(-S2, -S2);
#pragma unroll
  for (int u = 0; u < 8; u += 2) {
    const int j = g8 * 8 + u;
    const float2 ei = ex2_pair(clamp40(ui[u]), clamp40(ui[u + 1]), 0);
    const float2 ef = ex2_pair(clamp40(uf[u]), clamp40(uf[u + 1]), 1);
    const float2 eg = ex2_pair(clamp40(vg[u]), clamp40(vg[u + 1]), 2);
    const float2 eo = ex2_pair(clamp40(uo[u]), clamp40(uo[u + 1]), 3);
    // products by (1 + e) as fused a + a e: t_f is never formed
    const float2 ti = __ffma2_rn(ei, s1, s1);                                  // 2^-60 t_i
    const float2 tig = __ffma2_rn(ti, eg, ti);                                 // 2^-60 t_i t_g
    const float2 gm = __ffma2_rn(eg, ns1, s1);                                 // 2^-60 (1 - e_g)
    const float2 num = __ffma2_rn(make_float2(c[j], c[j + 1]), tig, __ffma2_rn(gm, ef, gm));
    const float2 d1 = __ffma2_rn(tig, ef, tig);                                // 2^-60 t_f t_i t_g
    const float r1 = rcp(d1.x * d1.y);
    const float2 cn = __fmul2_rn(num, __fmul2_rn(make_float2(d1.y, d1.x), make_float2(r1, r1)));
    c[j] = cn.x;
    c[j + 1] = cn.y;
#if TS_RAT_TANH
    // tanh(c') = P(c') / Q(c') on the FMA pipe (odd degree-13 / even degree-6
    // rational, |error| < 4e-7 on the clamp range [-7.905, 7.905], beyond it
    // tanh = +-1 within 2.8e-7), so h = o tanh(c') = P / ((1 + e_o) Q): Q
    // joins the output gate's shared reciprocal and the cell's exponential
    // leaves the MUFU pipe (5 MUFU ops per unit instead of 6).  Q lies in
    // [0.0049, 0.91], so the pair product stays above 2^-96.
    const float2 x = make_float2(fminf(fmaxf(cn.x, -kTanhClamp), kTanhClamp),
                                 fminf(fmaxf(cn.y, -kTanhClamp), kTanhClamp));
    const float2 x2 = __fmul2_rn(x, x);
    float2 pn = __ffma2_rn(make_float2(kTA13, kTA13), x2, make_float2(kTA11, kTA11));
    pn = __ffma2_rn(pn, x2, make_float2(kTA9, kTA9));
    pn = __ffma2_rn(pn, x2, make_float2(kTA7, kTA7));
    pn = __ffma2_rn(pn, x2, make_float2(kTA5, kTA5));
    pn = __ffma2_rn(pn, x2, make_float2(kTA3, kTA3));
    pn = __ffma2_rn(pn, x2, make_float2(kTA1, kTA1));
    pn = __fmul2_rn(pn, __fmul2_rn(x, s2));                                    // 2^-40 P(c')
    float2 qd = __ffma2_rn(make_float2(kTB6, kTB6), x2, make_float2(kTB4, kTB4));
    qd = __ffma2_rn(qd, x2, make_float2(kTB2, kTB2));
    qd = __ffma2_rn(qd, x2, make_float2(kTB0, kTB0));
    const float2 to = __ffma2_rn(eo, s2, s2);                                  // 2^-40 (1 + e_o)
    const float2 d2 = __fmul2_rn(to, qd);                                      // 2^-40 (1 + e_o) Q(c')
    const float r2 = rcp(d2.x * d2.y);
    const float2 hh = __fmul2_rn(pn, __fmul2_rn(make_float2(d2.y, d2.x), make_float2(r2, r2)));
    (void)ns2;
#else
    const float2 cc = __fmul2_rn(make_float2(C2, C2), cn);
    const float2 ec = ex2_pair(clamp40(cc.x), clamp40(cc.y), 4);
    const float2 to = __ffma2_rn(eo, s2, s2);                                  // 2^-40 (1 + e_o)
    const float2 d2 = __ffma2_rn(to, ec, to);                                  // 2^-40 (1 + e_o)(1 + e_c)
    const float r2 = rcp(d2.x * d2.y);
    const float2 hh = __fmul2_rn(__ffma2_rn(ec, ns2, s2), __fmul2_rn(make_float2(d2.y, d2.x), make_float2(r2, r2)));
#endif
    h8[u] = hh.x;
    h8[u + 1] = hh.y;
    acc = fmaf(hh.x, wout[j], acc);
    acc = fmaf(hh.y, wout[j + 1], acc);
  }
#endif
}

// kNWG warpgroups (tiles in flight) per CTA: 4 for large batches; 1 or 2
// when there are too few tiles to give every SM four, so small batches use
// more SMs.  The per-row arithmetic is the same code in every variant (and
// capped at the same 128 registers), so a state's V does not depend on the
// batch it is scored in.
template <int kNWG = NWG>
__global__ void __launch_bounds__(kNWG * TM, 4 / kNWG) k_lstm_tc(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* B = smem;
  const int tid = threadIdx.x;
  const int wg = tid / TM;            // warpgroup
  const int r = tid % TM;             // row within the tile = TMEM lane
  const int warp = tid >> 5;
  uint8_t* A = smem + TILE_BYTES + wg * A_BYTES;
  float* wout = reinterpret_cast<float*>(smem + TILE_BYTES + kNWG * A_BYTES);  // [32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(wout + 64);               // [kNWG]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kNWG);
  volatile int* tile_slot = reinterpret_cast<volatile int*>(tmem_slot + 1);  // [kNWG]

  // weights -> shared (B' image is already in the canonical layout)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wpack);
    uint4* dst = reinterpret_cast<uint4*>(B);
    for (int i = tid; i < TILE_BYTES / 16; i += kNWG * TM) dst[i] = __ldg(src + i);
    if (tid < 32) wout[tid] = __ldg(reinterpret_cast<const float*>(a.wpack + TILE_BYTES) + tid);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kNWG * 128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int g = 0; g < kNWG; ++g) mbar_init(bars + g, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot + wg * 128;   // this warpgroup's 128 columns
  const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const uint32_t a_base = smem_u32(A), b_base = smem_u32(B);
  uint64_t* bar = bars + wg;
  uint32_t phase = 0;
  const int T = a.T;
  put_bias_ones(A, r);

  // Tiles are in descending depth order; each warpgroup starts with one of
  // the first gridDim*kNWG and then takes the next unclaimed tile (longest
  // first, so the short tail tiles fill the gaps)
  for (int tile = blockIdx.x * kNWG + wg; tile < a.n_tiles;) {
    const int64_t sp = (int64_t)tile * TM + r;
    const bool valid = a.record_prefix ? (r == 0) : (sp < a.n);
    int64_t st = 0, off = 0;
    int d = 0;
    if (valid && !a.record_prefix) {
      st = a.perm[sp];
      off = a.offsets[st];
      d = (int)(a.offsets[st + 1] - off);
    }
    int dmax = T;  // record pass: the all-unscheduled row runs every timestep
    if (!a.record_prefix) {
      const int64_t first = a.perm[(int64_t)tile * TM];
      dmax = (int)(a.offsets[first + 1] - a.offsets[first]);
    }
    const int t0 = T - dmax;
    float c[32];
    double raw;
    {
      float h0[32];
      if (a.record_prefix) {
#pragma unroll
        for (int j = 0; j < 32; ++j) h0[j] = c[j] = 0.0f;
        raw = fmul((double)T, a.b_out);
      } else {
        const float* p = a.pre + (int64_t)t0 * PRE_STRIDE;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          h0[j] = p[j];
          c[j] = p[32 + j];
        }
        raw = *reinterpret_cast<const double*>(p + 64);
      }
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) put_h8(A, r, g8, h0 + 8 * g8);
    }
    uint4 x[4];
    load_x(a.initx + t0 * 4, (t0 < T - d) ? a.initx + t0 * 4 + 2 : a.rowsx + (a.rowoff[T - 1 - t0] + sp) * 2, x);
    for (int t = t0; t < T; ++t) {
      put_x(A, r, x);
      fence_async_smem();
      fence_before();
      wg_sync(wg);
      if (r == 0) {
        fence_after();
#pragma unroll
        for (int s = 0; s < KSTEPS; ++s)
          mma_f16(tmem, umma_desc(a_base + a_chunk(s) * CHUNK_STRIDE, CHUNK_STRIDE, 128),
                  umma_desc(b_base + s * 2 * CHUNK_STRIDE, CHUNK_STRIDE, 128), s > 0);
        mma_commit(bar);
      }
      // prefetch the next row while the tensor core works
      if (t + 1 < T)
        load_x(a.initx + (t + 1) * 4,
               (t + 1 < T - d) ? a.initx + (t + 1) * 4 + 2 : a.rowsx + (a.rowoff[T - 2 - t] + sp) * 2, x);
      mbar_wait(bar, phase);
      phase ^= 1u;
      fence_after();
      float acc = 0.0f;
      float* prow = (a.record_prefix && r == 0) ? a.pre + (int64_t)(t + 1) * PRE_STRIDE : nullptr;
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) {
        float h8[8];
        cell_group(lane_addr, g8, c, h8, acc, wout);
        // the UMMA that read A has completed (mbarrier), so h can go straight in
        put_h8(A, r, g8, h8);
        if (prow) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            prow[g8 * 8 + u] = h8[u];
            prow[32 + g8 * 8 + u] = c[g8 * 8 + u];
          }
        }
      }
      raw = fadd(raw, (double)acc);
      if (prow) *reinterpret_cast<double*>(prow + 64) = raw;
      fence_before();  // TMEM reads complete before the next UMMA overwrites D
    }
    if (!a.record_prefix && valid) a.out[st] = exp(fadd(raw, a.target_scale));
    if (a.tile_counter) {
      if (r == 0) tile_slot[wg] = gridDim.x * kNWG + atomicAdd(a.tile_counter, 1);
      wg_sync(wg);
      tile = tile_slot[wg];
    } else {
      wg_sync(wg);
      tile += gridDim.x * kNWG;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "r"(kNWG * 128)
                 : "memory");
}

// Prefix position 0 (h = c = 0, raw = T * b_out) for the record pass.
__global__ void k_prefix0(float* pre, int T, double b_out) {
  const int j = threadIdx.x;
  if (j < 64) pre[j] = 0.0f;
  if (j == 0) *reinterpret_cast<double*>(pre + 64) = fmul((double)T, b_out);
}

// --------------------------------------------- unscheduled rows -> split fp16
// initx[t] = {hi, lo} of (float) init_norm[t][0..7] and of [8..15]
__global__ void k_init_split(const double* __restrict__ init_norm, int T, uint4* __restrict__ initx) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = (float)init_norm[t * 16 + k];
  split8(v, initx[4 * t], initx[4 * t + 1]);
  split8(v + 8, initx[4 * t + 2], initx[4 * t + 3]);
}

// --------------------------------------------- depth bucketing (counting sort)
// Block-local histogram in shared memory, then one global atomic per bin.
__global__ void k_depth_hist(const int64_t* __restrict__ offsets, int64_t n, int T, int* __restrict__ hist) {
  extern __shared__ int sh[];
  for (int i = threadIdx.x; i <= T; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = offsets[i + 1] - offsets[i];
    // a depth outside 0..T sorts as 0 (the featurizer reports it)
    atomicAdd(sh + (d >= 0 && d <= T ? (int)d : 0), 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= T; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);
}

// descending depth: cursor[d] = number of states with depth > d
// rowoff[i] = first row of decision i in the depth-sorted, decision-major
// row layout: decision i of the state at sorted position p lives at
// rowoff[i] + p (only states deeper than i have one), so consecutive sorted
// positions - a warp of the featurizer, a tile of the LSTM - touch
// consecutive rows.
__global__ void k_depth_scan(const int* __restrict__ hist, int T, int* __restrict__ cursor,
                             int64_t* __restrict__ rowoff) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int acc = 0;
    for (int d = T; d >= 0; --d) {
      cursor[d] = acc;
      acc += hist[d];
    }
    int64_t r = 0;
    for (int i = 0; i < T; ++i) {
      rowoff[i] = r;
      r += cursor[i];  // states with depth > i
    }
    rowoff[T] = r;
  }
}

// Block-aggregated scatter: each block of SCATTER_THREADS x SCATTER_PER
// states ranks its states per depth in shared memory and reserves one range
// per (block, depth) with a single global atomic (the order inside a depth
// bucket is immaterial: every state's score is independent of its tile).
constexpr int SCATTER_THREADS = 256, SCATTER_PER = 4;
__global__ void __launch_bounds__(SCATTER_THREADS) k_depth_scatter(const int64_t* __restrict__ offsets, int64_t n,
                                                                    int T, int* __restrict__ cursor,
                                                                    int* __restrict__ perm) {
  extern __shared__ int sc[];  // cnt[T + 1], base[T + 1]
  int* cnt = sc;
  int* base = sc + (T + 1);
  for (int i = threadIdx.x; i <= T; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * SCATTER_THREADS * SCATTER_PER;
  int dep[SCATTER_PER], rank[SCATTER_PER];
#pragma unroll
  for (int k = 0; k < SCATTER_PER; ++k) {
    const int64_t i = b0 + k * SCATTER_THREADS + threadIdx.x;
    const int64_t d = i < n ? offsets[i + 1] - offsets[i] : -1;
    dep[k] = i < n ? (d >= 0 && d <= T ? (int)d : 0) : -1;  // as k_depth_hist
    rank[k] = dep[k] >= 0 ? atomicAdd(cnt + dep[k], 1) : 0;
  }
  __syncthreads();
  for (int dd = threadIdx.x; dd <= T; dd += blockDim.x)
    if (cnt[dd]) base[dd] = atomicAdd(cursor + dd, cnt[dd]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SCATTER_PER; ++k) {
    const int64_t i = b0 + k * SCATTER_THREADS + threadIdx.x;
    if (dep[k] >= 0) perm[base[dep[k]] + rank[k]] = (int)i;
  }
}

// --------------------------------------------- host: weight image
// B'[n][k] fp16 in the canonical K-major no-swizzle layout:
// chunk kc (8 K-elements), row-group n>>3, row n&7 -> kc*2048 + (n>>3)*128 + (n&7)*16.
// Gate columns scaled by -log2(e) (i, f, o) or -2 log2(e) (g); rows 144/145
// carry the scaled bias split hi/lo.
inline void pack_weights(const double* Wx, const double* Wh, const double* b, const double* w,
                         uint8_t* img /* TILE_BYTES + 32*4 */) {
  const double L2E = 1.4426950408889634074;
  memset(img, 0, TILE_BYTES + 32 * 4);
  for (int n = 0; n < GN; ++n) {
    const double scale = (n >= 64 && n < 96) ? -2.0 * L2E : -L2E;
    for (int k = 0; k < KP; ++k) {
      double wv;
      int seg;
      if (k < 3 * KA) {
        seg = k / KA;
        const int kk = k % KA;
        wv = scale * (kk < 16 ? Wx[kk * GN + n] : Wh[(kk - 16) * GN + n]);
      } else if (k == 3 * KA || k == 3 * KA + 1) {
        seg = k == 3 * KA ? 0 : 2;  // b_hi, b_lo
        wv = scale * b[n];
      } else {
        continue;
      }
      const __half whi = __double2half(wv);
      const __half wlo = __double2half(wv - (double)__half2float(whi));
      const __half v = seg == 2 ? wlo : whi;
      const int kc = k / 8, e = k % 8;
      memcpy(img + kc * CHUNK_STRIDE + (n >> 3) * 128 + (n & 7) * 16 + e * 2, &v, 2);
    }
  }
  float* fw = reinterpret_cast<float*>(img + TILE_BYTES);
  for (int j = 0; j < 32; ++j) fw[j] = (float)w[j];
}

}  // namespace tc
}  // namespace ts
