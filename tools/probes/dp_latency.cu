// Dependent-chain latency of FP64 / conversion / shuffle instructions on this GPU (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, long long* cyc, double a, double b, float fa) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; i++) {
    x = fma(x, b, a);
    x = fma(x, b, a);
    x = fma(x, b, a);
    x = fma(x, b, a);
  }
  long long t1 = clock64();
  float f = fa;
  double y = a;
#pragma unroll 1
  for (int i = 0; i < 1024; i++) {
    y = (double)f + y;           // F2F + DADD chain through y
    f = (float)y;                // F2F back
  }
  long long t2 = clock64();
  double s = x;
#pragma unroll 1
  for (int i = 0; i < 1024; i++) s = __shfl_xor_sync(0xffffffffu, s, 1) + b;
  long long t3 = clock64();
  float g = fa;
#pragma unroll 1
  for (int i = 0; i < 1024; i++) {
    g = fmaf(g, fa, 1.0f);
    g = fmaf(g, fa, 1.0f);
    g = fmaf(g, fa, 1.0f);
    g = fmaf(g, fa, 1.0f);
  }
  long long t4 = clock64();
  out[threadIdx.x] = x + y + s;
  outf[threadIdx.x] = f + g;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 256); cudaMalloc(&of, 256); cudaMalloc(&c, 64);
  for (int r = 0; r < 3; r++) k<<<1, 32>>>(o, of, c, 1.0000001, 0.999999, 1.0001f);
  long long h[4];
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", h[0] / 4096.0);
  printf("F2F.F64.F32 + DADD + F2F.F32.F64 round trip: %.1f cycles\n", h[1] / 1024.0);
  printf("SHFL(double) + DADD: %.1f cycles\n", h[2] / 1024.0);
  printf("FFMA dependent latency: %.1f cycles\n", h[3] / 4096.0);
  return 0;
}
