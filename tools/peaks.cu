// Micro-benchmark of the non-tensor pipes that bound the pair kernels:
// FP32 FFMA (register and immediate forms), MUFU (rsqrt, ex2), FP64 DFMA.
// Prints one JSON line. Used for the roofline denominator (MEASURED_PEAKS has no FP32 entry).
#include <cstdio>
#include <cuda_runtime.h>

#define NCH 8
template <int MODE>
__global__ void k_pipe(float* out, int iters, float s) {
  float a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = threadIdx.x * 1e-7f + c;
  float b = s, cc = 1.0f - s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (MODE == 0) a[c] = fmaf(a[c], b, cc);          // FFMA 3-reg
        else if (MODE == 1) a[c] = fmaf(a[c], 0.9999f, 1e-6f);  // FFMA imm
        else if (MODE == 2) a[c] = rsqrtf(a[c] + 1.0f);  // MUFU.RSQ (+FADD)
        else if (MODE == 3) a[c] = exp2f(-a[c]);  // MUFU.EX2
      }
    }
  }
  float t = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) t += a[c];
  if (t == 12345.f) out[0] = t;
}
__global__ void k_dfma(double* out, int iters, double s) {
  double a[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) a[c] = threadIdx.x * 1e-7 + c;
  double b = s, cc = 1.0 - s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) a[c] = fma(a[c], b, cc);
    }
  }
  double t = 0;
  for (int c = 0; c < NCH; ++c) t += a[c];
  if (t == 12345.) out[0] = t;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float* d; cudaMalloc(&d, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256, iters = 4096;
  double res[5];
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k_pipe<0><<<blocks, threads>>>(d, iters, 0.999f);
      if (m == 1) k_pipe<1><<<blocks, threads>>>(d, iters, 0.999f);
      if (m == 2) k_pipe<2><<<blocks, threads>>>(d, iters / 4, 0.999f);
      if (m == 3) k_pipe<3><<<blocks, threads>>>(d, iters / 4, 0.999f);
      if (m == 4) k_dfma<<<blocks, threads>>>((double*)d, iters / 4, 0.999);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * (m >= 2 ? iters / 4 : iters) * 16 * NCH;
      res[m] = ops / (ms * 1e-3);  // ops/s (lane-ops)
    }
  }
  printf("{\"sms\": %d, \"clock_khz\": %d, \"ffma_reg_tflops\": %.2f, \"ffma_imm_tflops\": %.2f, "
         "\"mufu_rsq_gops\": %.1f, \"mufu_ex2_gops\": %.1f, \"dfma_tflops\": %.2f, "
         "\"nominal_fp32_tflops_at_max_clock\": %.2f}\n",
         sms, p.clockRate, res[0] * 2e-12, res[1] * 2e-12, res[2] * 1e-9, res[3] * 1e-9,
         res[4] * 2e-12, sms * 128.0 * 2 * p.clockRate * 1e3 * 1e-12);
  return 0;
}
