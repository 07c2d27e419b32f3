// Microbenchmark: which pipe do fp32->fp16x2 packs (F2FP) issue on, and
// does the tensor core honour fp16 subnormal A operands?  Throughput of
// ex2.approx (MUFU), cvt.rn.f16x2.f32 (F2FP) and both interleaved; if the
// interleaved time is the sum, they share a pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe tools/probe_pipes.cu
#include <cstdio>
#include <cuda_fp16.h>

constexpr int ITERS = 4096;

__global__ void k_mufu(float* out, float seed) {
  float a = seed + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_f2fp(float* out, float seed) {
  float a = seed + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  unsigned acc = 0;
  for (int i = 0; i < ITERS; ++i) {
    unsigned r0, r1;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(a), "f"(b));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(c), "f"(d));
    acc ^= r0 ^ r1;
    a = __uint_as_float(__float_as_uint(a) ^ (acc & 1));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(b), "f"(c));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(d), "f"(a));
    acc ^= r0 ^ r1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

__global__ void k_both(float* out, float seed) {
  float a = seed + threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  float e = a + 4, f = a + 5, g = a + 6, h = a + 7;
  unsigned acc = 0;
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(c));
    asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(d));
    unsigned r0, r1;
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(e), "f"(f));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(g), "f"(h));
    acc ^= r0 ^ r1;
    e = __uint_as_float(__float_as_uint(e) ^ (acc & 1));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(f), "f"(g));
    asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(h), "f"(e));
    acc ^= r0 ^ r1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + (float)acc;
}

// integer/FMA-pipe fixed-point split (the LSTM's h operand): 4 FP + ~3.5 INT per value
__global__ void k_fixed(float* out, float seed) {
  float a = (seed + threadIdx.x) * 1e-3f, b = a * 0.5f, c = a * 0.25f, d = a * 0.125f;
  unsigned acc = 0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float x = q ? c : a, y = q ? d : b;
      const float ta = __fadd_rz(fabsf(x), 6144.0f), tb = __fadd_rz(fabsf(y), 6144.0f);
      const float la = fabsf(x) - (ta - 6144.0f), lb = fabsf(y) - (tb - 6144.0f);
      const float ua = fmaf(la, 4194304.0f, 12582912.0f), ub = fmaf(lb, 4194304.0f, 12582912.0f);
      const unsigned s = ((__float_as_uint(x) >> 16) & 0x8000u) | (__float_as_uint(y) & 0x80000000u);
      const unsigned hi = __byte_perm(__float_as_uint(ta), __float_as_uint(tb), 0x5410) | s;
      const unsigned lo = __byte_perm(__float_as_uint(ua), __float_as_uint(ub), 0x5410) | s;
      acc ^= hi + lo;
    }
    a = __uint_as_float(__float_as_uint(a) ^ (acc & 1));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 512 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(float*, float), double ops_per_thread) {
    k<<<148 * 8, 512>>>(out, 1.0f);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<148 * 8, 512>>>(out, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double thr = 5.0 * 148 * 8 * 512 * ops_per_thread / (ms * 1e-3) / 148 / 1.965e9;
    printf("%-8s %8.3f ms  %6.2f ops/clk/SM (at 1965 MHz)\n", name, ms / 5, thr);
  };
  run("mufu", k_mufu, 4.0 * ITERS);
  run("f2fp", k_f2fp, 4.0 * ITERS);
  run("both", k_both, 8.0 * ITERS);
  run("fixed", k_fixed, 4.0 * ITERS);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));

  // fp16 x fp16 subnormal products through the tensor path are covered by
  // the LSTM parity tests; here only the pipes.
  return 0;
}
