// TMEM / shared-memory / shuffle read throughput per SM (B200), to size the
// data-exchange budget of the blind rotation.  One CTA per SM,
// W warps; each loop iteration moves 4 KB per warp (TMEM: tcgen05.ld
// 32x32b.x32 = 32 lanes x 32 columns x 4 B; smem: 8 x LDS.128; shfl: 32 x
// SHFL.32 = 4 KB of lane-to-lane traffic).  Prints bytes per SM-clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmld tmld.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048

__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

template <int MODE>
__global__ void k_bw(uint32_t* out, long long* cyc) {
  __shared__ uint32_t slot;
  __shared__ __align__(16) uint4 sm[16 * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = threadIdx.x; t < 16 * 32; t += blockDim.x) sm[t] = make_uint4(t, t + 1, t + 2, t + 3);
  if (MODE == 0 && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = MODE == 0 ? slot + ((uint32_t)(32 * (warp & 3)) << 16) : 0;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    if constexpr (MODE == 0) {
      uint32_t r[32];
      tm_ld32(base + (uint32_t)(((i + warp) & 7) * 32), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];
    } else if constexpr (MODE == 1) {
      const uint4* p = sm + lane;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint4 v = p[((i + k + warp) & 15) * 32];
        acc += v.x ^ v.y ^ v.z ^ v.w;
      }
    } else if constexpr (MODE == 3) {
      if (warp & 1) {
        const uint4* p = sm + lane;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint4 v = p[((i + k + warp) & 15) * 32];
          acc += v.x ^ v.y ^ v.z ^ v.w;
        }
      } else {
        uint32_t v = acc + i;
#pragma unroll
        for (int k = 0; k < 32; ++k) v += __shfl_xor_sync(0xffffffffu, v, (k & 15) + 1);
        acc += v;
      }
    } else {
      uint32_t v = acc + i;
#pragma unroll
      for (int k = 0; k < 32; ++k) v += __shfl_xor_sync(0xffffffffu, v, (k & 15) + 1);
      acc += v;
    }
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (MODE == 0 && warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  k_bw<MODE><<<148, 32 * warps>>>(out, cyc);
  k_bw<MODE><<<148, 32 * warps>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)ITERS * warps * 4096.0;
  printf("%-6s warps=%2d  %8.1f bytes/SM-clock  (%s)\n", name, warps, bytes / mx,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<0>("tmem", w);
  for (int w : {4, 8, 16}) run<1>("smem", w);
  for (int w : {4, 8, 16}) run<2>("shfl", w);
  for (int w : {8, 16}) run<3>("mixed", w);
  return 0;
}
