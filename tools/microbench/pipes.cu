// Pipe-throughput microbenchmarks used to pick the blind-rotation arithmetic
// (FP64 split FFT vs Goldilocks NTT). Register-only loops, all SMs busy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_dadd(double* out, double a) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void k_imad(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ uint64_t gl_mul(uint64_t a, uint64_t b) {
  const uint64_t Q = 0xFFFFFFFF00000001ull;
  uint64_t lo = a * b, hi = __umul64hi(a, b);
  uint64_t hh = hi >> 32, hl = hi & 0xFFFFFFFFull;
  uint64_t t = lo - hh; if (lo < hh) t -= 0xFFFFFFFFull;
  uint64_t u = (hl << 32) - hl;
  uint64_t s = t + u; if (s < t) s += 0xFFFFFFFFull;
  if (s >= Q) s -= Q;
  return s;
}

__global__ void k_glmul(uint64_t* out, uint64_t a) {
  uint64_t x0 = threadIdx.x + 12345, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = gl_mul(x0, a); x1 = gl_mul(x1, a); x2 = gl_mul(x2, a); x3 = gl_mul(x3, a);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}

__global__ void k_shfl(uint32_t* out) {
  uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = __shfl_xor_sync(0xffffffff, x0, 1); x1 = __shfl_xor_sync(0xffffffff, x1, 2);
      x2 = __shfl_xor_sync(0xffffffff, x2, 4); x3 = __shfl_xor_sync(0xffffffff, x3, 8);
      x4 = __shfl_xor_sync(0xffffffff, x4, 16); x5 = __shfl_xor_sync(0xffffffff, x5, 1);
      x6 = __shfl_xor_sync(0xffffffff, x6, 2); x7 = __shfl_xor_sync(0xffffffff, x7, 4);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// shared-memory 128-bit load bandwidth: each lane reads consecutive 16B
__global__ void k_lds128(double* out) {
  __shared__ double2 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_double2(i, i + 1);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int base = threadIdx.x & 1023;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 v = buf[(base + u * 128 + i) & 2047];
      acc.x += v.x; acc.y += v.y;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

template <typename F>
float time_kernel(F launch) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, threads = 512;
  const double nthreads = double(blocks) * threads;
  void* buf; cudaMalloc(&buf, nthreads * 8);
  printf("SMs %d  clock(kHz) %d\n", sms, clk);
  float ms;
  ms = time_kernel([&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0000001, 1e-9); });
  printf("DFMA  %.2f Tops/s  (%.2f TFLOP/s)  per-SM-clk %.1f\n", nthreads * ITERS * 32 / ms / 1e9, 2 * nthreads * ITERS * 32 / ms / 1e9,
         nthreads * ITERS * 32 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_dadd<<<blocks, threads>>>((double*)buf, 1e-9); });
  printf("DADD  %.2f Tops/s  per-SM-clk %.1f\n", nthreads * ITERS * 32 / ms / 1e9, nthreads * ITERS * 32 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_ffma<<<blocks, threads>>>((float*)buf, 1.0000001f, 1e-9f); });
  printf("FFMA  %.2f Tops/s  per-SM-clk %.1f\n", nthreads * ITERS * 32 / ms / 1e9, nthreads * ITERS * 32 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_imad<<<blocks, threads>>>((uint32_t*)buf, 1664525u, 1013904223u); });
  printf("IMAD  %.2f Tops/s  per-SM-clk %.1f\n", nthreads * ITERS * 32 / ms / 1e9, nthreads * ITERS * 32 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_glmul<<<blocks, threads>>>((uint64_t*)buf, 0x123456789abcdefull); });
  printf("GLMUL %.2f Gmodmul/s  per-SM-clk %.2f\n", nthreads * ITERS * 4 / ms / 1e6, nthreads * ITERS * 4 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_shfl<<<blocks, threads>>>((uint32_t*)buf); });
  printf("SHFL  %.2f Tlane/s  per-SM-clk %.1f lanes\n", nthreads * ITERS * 8 / ms / 1e9, nthreads * ITERS * 8 / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_kernel([&] { k_lds128<<<blocks, threads>>>((double*)buf); });
  printf("LDS128 %.2f TB/s  per-SM-clk %.1f B\n", nthreads * ITERS * 2 * 16 / ms / 1e9, nthreads * ITERS * 2 * 16 / (ms * 1e-3) / sms / (clk * 1e3));
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
