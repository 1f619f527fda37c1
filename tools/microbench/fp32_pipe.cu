// Microbenchmark: FP32 pipe throughput on sm_100a for scalar FFMA/FADD vs packed f32x2
// (FFMA2/FADD2/FMUL2), and the canonical 6-instruction distance body.
// Used once to fix the FP32 roofline denominator for the LeafToLeaf kernel.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void ffma_scalar(float *out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x0 = __fmaf_rn(x0, a, b); x1 = __fmaf_rn(x1, a, b); x2 = __fmaf_rn(x2, a, b); x3 = __fmaf_rn(x3, a, b);
      x4 = __fmaf_rn(x4, a, b); x5 = __fmaf_rn(x5, a, b); x6 = __fmaf_rn(x6, a, b); x7 = __fmaf_rn(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(a), "l"(b));
  return d;
}

__global__ void ffma_packed(float *out, float a, float b) {
  unsigned long long A, B;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
  unsigned long long x[8];
  for (int j = 0; j < 8; ++j) { float f = threadIdx.x + j; asm("mov.b64 %0, {%1, %1};" : "=l"(x[j]) : "f"(f)); }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = ffma2(x[q], A, B);
    }
  }
  float s = 0.f;
  for (int j = 0; j < 8; ++j) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[j])); s += lo + hi; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s SMs %d clock(kHz attr) %d\n", p.name, p.multiProcessorCount, clk);
  float *out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256;
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0); ffma_scalar<<<blocks, threads>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = double(blocks) * threads * ITERS * 32;  // lane-FMAs
    printf("scalar FFMA : %.3f ms  %.2f T lane-FMA/s  (%.1f TFLOP/s)\n", ms, lane_ops / ms / 1e9, 2 * lane_ops / ms / 1e9);
    cudaEventRecord(e0); ffma_packed<<<blocks, threads>>>(out, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    lane_ops = double(blocks) * threads * ITERS * 32 * 2;  // two FMAs per f32x2 op
    printf("packed FFMA2: %.3f ms  %.2f T lane-FMA/s  (%.1f TFLOP/s)\n", ms, lane_ops / ms / 1e9, 2 * lane_ops / ms / 1e9);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
