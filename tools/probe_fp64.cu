// Latency of dependent fp64 operations on the B200 (one warp, clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_fp64.bin tools/probe_fp64.cu
#include <cstdio>

__global__ void k_lat(double* out, double seed, long long* cyc) {
  double a = seed + threadIdx.x, b = 1.0000001;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
    a = __dadd_rn(a, b);
  }
  long long t1 = clock64();
  double e = seed + threadIdx.x * 1e-3;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) e = exp(e * 1e-3);
  long long t2 = clock64();
  double d = seed + 2.0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) d = __ddiv_rn(1.0, d + 1.0);
  long long t3 = clock64();
  double h = seed * 1e-3;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) h = tanh(h + 0.1);
  long long t4 = clock64();
  float f = seed;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    f = __fadd_rn(f, 1.0001f);
    f = __fadd_rn(f, 1.0001f);
    f = __fadd_rn(f, 1.0001f);
    f = __fadd_rn(f, 1.0001f);
  }
  long long t5 = clock64();
  out[threadIdx.x] = a + e + d + h + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  k_lat<<<1, 32>>>(out, 1.0, cyc);
  k_lat<<<1, 32>>>(out, 1.0, cyc);
  cudaDeviceSynchronize();
  printf("DADD dependent latency: %.1f cycles\n", cyc[0] / 4096.0);
  printf("exp(double) (+DMUL) dependent latency: %.1f cycles\n", cyc[1] / 256.0);
  printf("1/(d+1) DDIV (+DADD) dependent latency: %.1f cycles\n", cyc[2] / 256.0);
  printf("tanh(double) (+DADD) dependent latency: %.1f cycles\n", cyc[3] / 256.0);
  printf("FADD dependent latency: %.1f cycles\n", cyc[4] / 4096.0);
  return 0;
}
