// Probe: tcgen05.mma kind::f16 with MN-major A and B (no swizzle), M=128,
// N=64, K=128 (8 instructions of K=16), against a CPU product.  The operand
// layout is the training kernel's: element (mn, k) of an MN-major operand at
//   (mn / 8) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (mn % 8) * 2
// (core matrix = 8 K-rows x 16 bytes of MN).  Tries both assignments of the
// two descriptor stride fields.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
constexpr int M = 128, N = 64, K = 128;
constexpr uint32_t IDESC = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__global__ void k(const __half* A, const __half* B, float* D, int variant) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* As = sm;                 // M x K : 16 mn-chunks x 2048
  uint8_t* Bs = sm + (M / 8) * 2048;  // N x K : 8 chunks x 2048
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int mn = e / K, kk = e % K;
    *reinterpret_cast<__half*>(As + (mn / 8) * 2048 + (kk / 8) * 128 + (kk % 8) * 16 + (mn % 8) * 2) = A[e];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int mn = e / K, kk = e % K;
    *reinterpret_cast<__half*>(Bs + (mn / 8) * 2048 + (kk / 8) * 128 + (kk % 8) * 16 + (mn % 8) * 2) = B[e];
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (tid == 0) {
    for (int s = 0; s < K / 16; ++s) {
      // K step s = rows 16s..16s+15 = two 8-row core blocks, 128 B apart
      const uint32_t ka = smem_u32(As) + s * 256, kb = smem_u32(Bs) + s * 256;
      uint64_t da, db;
      if (variant == 0) { da = desc(ka, 128, 2048); db = desc(kb, 128, 2048); }
      else { da = desc(ka, 2048, 128); db = desc(kb, 2048, 128); }
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm), "l"(da), "l"(db),
                   "r"(IDESC), "r"(s > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n\t.reg .pred done;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t@!done bra W_%=;\n\t}\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid >> 5, lane = tid & 31;
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) D[(warp * 32 + lane) * N + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(64));
}

int main() {
  std::vector<__half> A(M * K), B(N * K);
  std::vector<float> Af(M * K), Bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.0f; A[i] = __float2half(v); Af[i] = v; }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 13 - 6) / 4.0f; B[i] = __float2half(v); Bf[i] = v; }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (M / 8) * 2048 + (N / 8) * 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dD, 0, M * N * 4);
    k<<<1, 128, smem>>>(dA, dB, dD, variant);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(M * N);
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int kk = 0; kk < K; ++kk) s += (double)Af[m * K + kk] * Bf[n * K + kk];
        maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
      }
    printf("variant %d (%s): err=%s max abs err %.3e\n", variant, variant == 0 ? "LBO=128 (K), SBO=2048 (MN)" : "LBO=2048 (MN), SBO=128 (K)",
           cudaGetErrorString(e), maxerr);
  }
  return 0;
}
