// ts_lstm_tc.cuh - FAST scoring path: the LSTM value network on the 5th-gen
// tensor cores (tcgen05.mma, accumulators in TMEM), fused with bias, gates,
// cell update, readout and exp.
//
// Per timestep each row (one state) computes z = [x | h] . [Wx; Wh] + b, a
// [1 x 48] x [48 x 128] product.  A CTA stacks 128 states as the M=128 rows
// of one UMMA: D[128 x 128] (fp32, TMEM) = A[128 x K] . B[128 x K]^T with
// fp16 operands split hi/lo and concatenated along K,
//     A' = [a_hi | a_lo | a_hi],  B' = [W_hi ; W_hi ; W_lo]   (K = 3*48 = 144)
// so a.W ~= a_hi W_hi + a_lo W_hi + a_hi W_lo with 22-bit operands and fp32
// accumulation (|dV|/V <= 1e-4, the north-star fp32 tolerance).  9 UMMAs of
// K=16 per timestep, issued by one thread, completion via tcgen05.commit on
// an mbarrier; the 128 epilogue threads (thread = TMEM lane = state) read
// their row with tcgen05.ld, apply the gates in fp32 (MUFU ex2/rcp), update
// c (registers) and h, and write the next A row (fp16 hi/lo) to shared
// memory in the canonical K-major no-swizzle layout.
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

namespace ts {
namespace tc {

constexpr int TM = 128;                   // states per tile (UMMA M)
constexpr int GN = 128;                   // gate columns 4H (UMMA N), H = 32
constexpr int KA = 48;                    // [x(16) | h(32)]
constexpr int KP = 3 * KA;                // split-concatenated K = 144
constexpr int KCH = KP / 8;               // 16-byte K chunks = 18
constexpr int CHUNK_STRIDE = TM * 16;     // bytes between K chunks (LBO) = 2048
constexpr int TILE_BYTES = KCH * CHUNK_STRIDE;  // 36864 per operand
constexpr int SMEM_BYTES = 2 * TILE_BYTES + 1024 + 1024;  // A, B, bias/readout, barriers
constexpr int PRE_STRIDE = 72;            // floats per prefix position: h[32], c[32], raw (as 2 floats) ...

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
__device__ __forceinline__ float sig_f(float x) { return __frcp_rn(1.0f + __expf(-x)); }
__device__ __forceinline__ float tanh_f(float x) { return fmaf(2.0f, sig_f(2.0f * x), -1.0f); }

// hi/lo fp16 split of 8 floats into two 16-byte chunks
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  __half2 h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half a = __float2half_rn(v[2 * i]), b = __float2half_rn(v[2 * i + 1]);
    h[i] = __halves2half2(a, b);
    l[i] = __halves2half2(__float2half_rn(v[2 * i] - __half2float(a)),
                          __float2half_rn(v[2 * i + 1] - __half2float(b)));
  }
  hi = *reinterpret_cast<uint4*>(h);
  lo = *reinterpret_cast<uint4*>(l);
}

// Stores a 16-byte chunk `kc` of row `r` in the canonical no-swizzle layout.
__device__ __forceinline__ void st_chunk(uint8_t* A, int kc, int r, const uint4& v) {
  *reinterpret_cast<uint4*>(A + kc * CHUNK_STRIDE + (r >> 3) * 128 + (r & 7) * 16) = v;
}

// Writes the x part (chunks q=0,1 of every segment) of row r.
__device__ __forceinline__ void put_x(uint8_t* A, int r, const float* x) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    uint4 hi, lo;
    split8(x + 8 * q, hi, lo);
    st_chunk(A, 0 * 6 + q, r, hi);
    st_chunk(A, 1 * 6 + q, r, lo);
    st_chunk(A, 2 * 6 + q, r, hi);
  }
}

// Writes the h part (chunks q=2..5) of row r.
__device__ __forceinline__ void put_h(uint8_t* A, int r, const float* h) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 hi, lo;
    split8(h + 8 * q, hi, lo);
    st_chunk(A, 0 * 6 + 2 + q, r, hi);
    st_chunk(A, 1 * 6 + 2 + q, r, lo);
    st_chunk(A, 2 * 6 + 2 + q, r, hi);
  }
}

// ---------------------------------------------------------------- kernel
// Tiles: sorted positions [128*tile, 128*tile + 128); perm maps a sorted
// position to the original state index; depth is sorted descending, so the
// tile's first state has its maximum depth.  record_prefix: a single tile
// whose row 0 is the all-unscheduled state (depth 0, t0 = 0); thread 0
// writes (h, c, raw) before every timestep into `pre` (the fast prefix).
struct TcArgs {
  const uint8_t* wpack;     // B' image (TILE_BYTES) + bias[128] f32 + w[32] f32
  const float* init32;      // [T][16] normalized unscheduled rows (fp32)
  const float* rows32;      // [n_records][16] normalized scheduled rows (fp32)
  const int64_t* offsets;   // [n+1]
  const int* perm;          // [n] sorted position -> state
  float* pre;               // [(T+1)][PRE_STRIDE] fast prefix (h, c, raw hi/lo)
  double* out;              // [n] V
  int64_t n;
  int T;
  int n_tiles;
  int record_prefix;
  double target_scale;
  double b_out;
};

__global__ void __launch_bounds__(TM, 1) k_lstm_tc(TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;
  uint8_t* B = smem + TILE_BYTES;
  float* bias = reinterpret_cast<float*>(smem + 2 * TILE_BYTES);  // [128]
  float* wout = bias + GN;                                       // [32]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * TILE_BYTES + 1024);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int r = threadIdx.x;
  const int warp = r >> 5;

  // weights -> shared (B' image is already in the canonical layout)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.wpack);
    uint4* dst = reinterpret_cast<uint4*>(B);
    for (int i = r; i < TILE_BYTES / 16; i += TM) dst[i] = __ldg(src + i);
    const float* fb = reinterpret_cast<const float*>(a.wpack + TILE_BYTES);
    bias[r] = __ldg(fb + r);
    if (r < 32) wout[r] = __ldg(fb + GN + r);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (r == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base = smem_u32(A), b_base = smem_u32(B);
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  uint32_t phase = 0;
  const int T = a.T;

  for (int tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x) {
    const int64_t sp = (int64_t)tile * TM + r;
    const bool valid = a.record_prefix ? (r == 0) : (sp < a.n);
    int64_t st = 0, off = 0;
    int d = 0;
    if (valid && !a.record_prefix) {
      st = a.perm[sp];
      off = a.offsets[st];
      d = (int)(a.offsets[st + 1] - off);
    }
    int dmax;
    if (a.record_prefix) {
      dmax = 0;
    } else {
      const int64_t first = a.perm[(int64_t)tile * TM];
      dmax = (int)(a.offsets[first + 1] - a.offsets[first]);
    }
    const int t0 = a.record_prefix ? 0 : T - dmax;
    float h[32], c[32];
    double raw;
    if (a.record_prefix) {
#pragma unroll
      for (int j = 0; j < 32; ++j) h[j] = c[j] = 0.0f;
      raw = fmul((double)T, a.b_out);
    } else {
      const float* p = a.pre + (int64_t)t0 * PRE_STRIDE;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        h[j] = p[j];
        c[j] = p[32 + j];
      }
      raw = *reinterpret_cast<const double*>(p + 64);
    }
    put_h(A, r, h);
    for (int t = t0; t < T; ++t) {
      if (a.record_prefix && r == 0) {
        float* p = a.pre + (int64_t)t * PRE_STRIDE;
        for (int j = 0; j < 32; ++j) {
          p[j] = h[j];
          p[32 + j] = c[j];
        }
        *reinterpret_cast<double*>(p + 64) = raw;
      }
      // x row for this timestep: own scheduled row or the shared prefix row
      float x[16];
      const float* src = (t < T - d) ? a.init32 + t * 16 : a.rows32 + (off + (T - 1 - t)) * 16;
      const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = __ldg(s4 + q);
        x[4 * q] = v.x;
        x[4 * q + 1] = v.y;
        x[4 * q + 2] = v.z;
        x[4 * q + 3] = v.w;
      }
      put_x(A, r, x);
      fence_async_smem();
      fence_before();
      __syncthreads();
      if (r == 0) {
        fence_after();
#pragma unroll
        for (int s = 0; s < KCH / 2; ++s)
          mma_f16(tmem, umma_desc(a_base + s * 2 * CHUNK_STRIDE, CHUNK_STRIDE, 128),
                  umma_desc(b_base + s * 2 * CHUNK_STRIDE, CHUNK_STRIDE, 128), s > 0);
        mma_commit(bar);
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
      fence_after();
      float acc = 0.0f;
#pragma unroll
      for (int g8 = 0; g8 < 4; ++g8) {
        float zi[8], zf[8], zg[8], zo[8];
        tmem_ld8(lane_addr + 0 * 32 + g8 * 8, zi);
        tmem_ld8(lane_addr + 1 * 32 + g8 * 8, zf);
        tmem_ld8(lane_addr + 2 * 32 + g8 * 8, zg);
        tmem_ld8(lane_addr + 3 * 32 + g8 * 8, zo);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = g8 * 8 + u;
          const float gi = sig_f(zi[u] + bias[j]);
          const float gf = sig_f(zf[u] + bias[32 + j]);
          const float gg = tanh_f(zg[u] + bias[64 + j]);
          const float go = sig_f(zo[u] + bias[96 + j]);
          c[j] = fmaf(gf, c[j], gi * gg);
          h[j] = go * tanh_f(c[j]);
          acc = fmaf(h[j], wout[j], acc);
        }
      }
      raw = fadd(raw, (double)acc);
      fence_before();
      put_h(A, r, h);
    }
    if (a.record_prefix) {
      if (r == 0) {
        float* p = a.pre + (int64_t)T * PRE_STRIDE;
        for (int j = 0; j < 32; ++j) {
          p[j] = h[j];
          p[32 + j] = c[j];
        }
        *reinterpret_cast<double*>(p + 64) = raw;
      }
    } else if (valid) {
      a.out[st] = exp(fadd(raw, a.target_scale));
    }
    __syncthreads();
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
}

// --------------------------------------------- featurize -> fp32 rows
__global__ void k_rows32(const double* __restrict__ rows64, int64_t n_words, float* __restrict__ rows32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_words) rows32[i] = (float)rows64[i];
}

// --------------------------------------------- depth bucketing (counting sort)
__global__ void k_depth_hist(const int64_t* __restrict__ offsets, int64_t n, int* __restrict__ hist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(hist + (int)(offsets[i + 1] - offsets[i]), 1);
}

// descending depth: cursor[d] = number of states with depth > d
__global__ void k_depth_scan(const int* __restrict__ hist, int T, int* __restrict__ cursor) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int acc = 0;
    for (int d = T; d >= 0; --d) {
      cursor[d] = acc;
      acc += hist[d];
    }
  }
}

__global__ void k_depth_scatter(const int64_t* __restrict__ offsets, int64_t n, int* __restrict__ cursor,
                                int* __restrict__ perm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int d = (int)(offsets[i + 1] - offsets[i]);
    perm[atomicAdd(cursor + d, 1)] = (int)i;
  }
}

// --------------------------------------------- host: weight image
// B'[n][k] fp16 in the canonical K-major no-swizzle layout:
// chunk kc (8 K-elements), row-group n>>3, row n&7 -> kc*2048 + (n>>3)*128 + (n&7)*16.
inline void pack_weights(const double* Wx, const double* Wh, const double* b, const double* w,
                         uint8_t* img /* TILE_BYTES + 160*4 */) {
  for (int n = 0; n < GN; ++n) {
    for (int k = 0; k < KP; ++k) {
      const int seg = k / KA, kk = k % KA;
      const double wv = kk < 16 ? Wx[kk * GN + n] : Wh[(kk - 16) * GN + n];
      const __half whi = __double2half(wv);
      const __half wlo = __double2half(wv - (double)__half2float(whi));
      const __half v = seg == 2 ? wlo : whi;
      const int kc = k / 8, e = k % 8;
      memcpy(img + kc * CHUNK_STRIDE + (n >> 3) * 128 + (n & 7) * 16 + e * 2, &v, 2);
    }
  }
  float* fb = reinterpret_cast<float*>(img + TILE_BYTES);
  for (int j = 0; j < GN; ++j) fb[j] = (float)b[j];
  for (int j = 0; j < 32; ++j) fb[GN + j] = (float)w[j];
}

}  // namespace tc
}  // namespace ts
