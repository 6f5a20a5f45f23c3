// probe.cu — FP32 FFMA throughput probe (measurement utility for the roofline
// denominator: MEASURED_PEAKS.json has HBM and bf16 tensor peaks only, while the
// DiffMPC kernels run on the FP32 CUDA cores). Each thread runs 8 independent FMA
// chains; the kernel does blocks*threads*iters*8 FMAs = 2x that many flops.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) ffma_probe_kernel(int iters, float seed, float* out) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f;
  float a4 = a0 + 4.f, a5 = a0 + 5.f, a6 = a0 + 6.f, a7 = a0 + 7.f;
  const float b = 0.999f, c = 1e-3f;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  const float s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.f) out[blockIdx.x] = s;  // keep the chains alive
}

extern "C" int diffmpc_probe_ffma(int blocks, int iters, void* out, void* stream) {
  ffma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, 0.5f, (float*)out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
