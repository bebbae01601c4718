// FP64 tensor-core (DMMA m8n8k4) throughput on B200, alone and concurrent with
// the vector FP64 pipe (DFMA): is the tensor path additive?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1;
}

__global__ void k_dfma(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  const double a = 0.999999, b = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// half the warps do DMMA, half DFMA
__global__ void k_mix(double* out, int iters_mma, int iters_fma) {
  if ((threadIdx.x >> 5) & 1) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
    const double a = 0.999999, b = 1e-7;
    for (int i = 0; i < iters_fma; ++i) {
#pragma unroll
      for (int r = 0; r < 32; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
    for (int i = 0; i < iters_mma; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
      }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + d0 + d1 + e0 + e1 + f0 + f1;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)sms * 8 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 2, threads = 512;
  float ms;
  const int it = 2000;
  k_dmma<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_dmma<<<blocks, threads>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double mma_flops = warps * it * 32 * 256 * 2;  // 32 mma per iter, 256 FMA each
  printf("DMMA m8n8k4 alone: %.2f TFLOP/s (%s)\n", mma_flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  k_dfma<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(out, it);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma_flops = (double)blocks * threads * it * 256 * 2;
  printf("DFMA alone:        %.2f TFLOP/s\n", fma_flops / ms / 1e9);
  // mixed: choose iteration counts so each half alone would take similar time
  for (int ratio : {1, 2, 4}) {
    const int im = it, ifm = it * ratio;
    cudaEventRecord(e0);
    k_mix<<<blocks, threads>>>(out, im, ifm);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double f = (warps / 2) * im * 32 * 256 * 2 + (double)blocks * threads / 2 * ifm * 256 * 2;
    printf("mixed (fma x%d):   %.2f TFLOP/s combined\n", ratio, f / ms / 1e9);
  }
  return 0;
}
