// Warp transpose of the forward FFT (32 lanes x 16 complex doubles: lane l holds
// X[l][k], k = 0..15; lane 16b + k must end up with X[b + 2a][k], a = 0..15) two
// ways: through shared memory (16 STS.128 + 16 LDS.128, the kernel's swizzled tile)
// and through TMEM in two round trips (tcgen05.st 32x32b.x64 + 2x tcgen05.ld
// 16x256b.x8, twice).  Checks both results and prints cycles per transpose with
// W warps per CTA (W / 4 per TMEM sub-partition), one CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmtr tmtr.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 256

__device__ __forceinline__ void st64(uint32_t taddr, const uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
      "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, "
      "%57, %58, %59, %60, %61, %62, %63, %64};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]), "r"(r[36]),
      "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]), "r"(r[43]), "r"(r[44]), "r"(r[45]),
      "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]), "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]),
      "r"(r[55]), "r"(r[56]), "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63])
      : "memory");
}
// 16 lanes x 256 bits x 8: thread t gets, for rep m, {lane t/4: cols 8m + 2(t%4), +1;
// lane t/4 + 8: same cols} -> r[4m .. 4m+3]
__device__ __forceinline__ void ld16x256x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// word w of complex k of source lane l
__device__ __forceinline__ uint32_t val(int l, int k, int w) { return (uint32_t)((l << 8) | (k << 2) | w); }

// Trip A store layout: word q = 4 kk + w of complex k = 4j + kk -> column 8 (q / 2) + 2j + (q % 2).
// Trip A load (bases 0, 16; reps m): thread t (j = t % 4) receives from lane L = base + t/4 + 8 v1
// column 8m + 2j + e -> q = 2m + e of complex 4j + q/4 ... of source lane L.
// Trip B: thread s re-stores so final thread T = 4 (s % 8) + mm (mm = k % 4) finds its words at
// columns 8m' + 2mm + e; final load as trip A.
template <int MODE>  // 0 = smem, 1 = tmem
__global__ void k_tr(long long* cyc, int* bad, int iters) {
  __shared__ uint32_t slot;
  extern __shared__ __align__(16) double2 tiles[];  // [warp][16 * 32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
  uint32_t x[64];  // x[4k + w]
#pragma unroll
  for (int k = 0; k < 16; ++k)
#pragma unroll
    for (int w = 0; w < 4; ++w) x[4 * k + w] = val(lane, k, w);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      double2* tl = tiles + (size_t)warp * 16 * 32;
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int col = lane ^ ((k & 3) << 1);
        tl[k * 32 + col] = make_double2(__hiloint2double(x[4 * k + 1], x[4 * k]), __hiloint2double(x[4 * k + 3], x[4 * k + 2]));
      }
      __syncwarp();
      // the kernel's mapping (fft.cuh): target lane T = 2 k1 + b reads source lanes b + 2a at k1
      const int k1 = lane >> 1, b = lane & 1;
#pragma unroll
      for (int a = 0; a < 16; ++a) {
        const int col = (b + 2 * a) ^ ((k1 & 3) << 1);
        const double2 v = tl[k1 * 32 + col];
        x[4 * a] = __double2loint(v.x); x[4 * a + 1] = __double2hiint(v.x);
        x[4 * a + 2] = __double2loint(v.y); x[4 * a + 3] = __double2hiint(v.y);
      }
    } else {
      // ---- trip A ----
      uint32_t s[64];
      const int j = lane & 3;
      (void)j;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)          // complex k = 4 jj + kk
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const int q = 4 * kk + w;
            s[8 * (q / 2) + 2 * jj + (q % 2)] = x[4 * (4 * jj + kk) + w];
          }
      st64(tbase, s);
      wait_st();
      uint32_t r0[32], r1[32];
      ld16x256x8(tbase, r0);                    // lanes t/4 (+8)
      ld16x256x8(tbase + (16u << 16), r1);      // lanes 16 + t/4 (+8)
      wait_ld();
      // thread t now holds, for source lane L in {t/4, t/4+8, 16+t/4, 24+t/4} (index src = 2 half + v1),
      // the 16 words q = 2m + e of complexes 4j + q/4 (word q%4): r{half}[4m + 2 v1 + e]
      // ---- trip B: regroup by final thread T = 4 (t % 8) + mm, mm = complex % 4 ----
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1)
#pragma unroll
          for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int q = 2 * m + e, kk = q / 4, w = q % 4;  // complex 4j + kk, word w
              const int src = 2 * half + v1;                      // source index 0..3
              const uint32_t v = half ? r1[4 * m + 2 * v1 + e] : r0[4 * m + 2 * v1 + e];
              // destined for final thread with mm = kk; in its column group: word (src, w) -> q' = 4 src + w
              const int qq = 4 * src + w;
              s[8 * (qq / 2) + 2 * kk + (qq % 2)] = v;
            }
      st64(tbase, s);
      wait_st();
      ld16x256x8(tbase, r0);
      ld16x256x8(tbase + (16u << 16), r1);
      wait_ld();
      // final thread T: from intermediate s' (index src2 = 2 half + v1), words qq = 4 src + w of
      // the complex its source lane sent; map back to x[4a + w] with source lane b + 2a
#pragma unroll
      for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1)
#pragma unroll
          for (int m = 0; m < 8; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int qq = 2 * m + e, src = qq / 4, w = qq % 4;
              const int src2 = 2 * half + v1;
              // intermediate s' = T/4 + 8 src2 received source lane L = s'/4 + 8 ... (src: 2 half' + v1')
              // source lane l = b + 2a with a = (src2 + 4 * src) ordering fixed below
              const int a = src2 + 4 * src;
              const uint32_t v = half ? r1[4 * m + 2 * v1 + e] : r0[4 * m + 2 * v1 + e];
              x[4 * a + w] = v;
            }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  // check (ITERS even for smem-mode the transpose is an involution only on matching lanes, so check one pass)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
  (void)bad;
  // record x for host-side inspection of a single pass
  if (blockIdx.x == 0) {
    int nb = 0;
    const int k1 = MODE == 0 ? lane >> 1 : lane & 15, b = MODE == 0 ? lane & 1 : lane >> 4;
    for (int a = 0; a < 16; ++a)
      for (int w = 0; w < 4; ++w) {
        // after an odd number of passes? (validated with ITERS = 1 in the check kernel)
        nb += x[4 * a + w] != val(b + 2 * a, k1, w);
      }
    atomicAdd(bad + MODE, nb);
  }
}

int main() {
  long long* cyc;
  int* bad;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&bad, 2 * sizeof(int));
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8}) {
      cudaMemset(bad, 0, 2 * sizeof(int));
      // one pass: correctness (the transpose is not an involution); then ITERS passes: timing
      const int sm = warps * 16 * 32 * 16;
      cudaFuncSetAttribute(k_tr<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16 * 32 * 16);
      cudaFuncSetAttribute(k_tr<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16 * 32 * 16);
      if (mode == 0) k_tr<0><<<148, 32 * warps, sm>>>(cyc, bad, 1);
      else k_tr<1><<<148, 32 * warps, sm>>>(cyc, bad, 1);
      cudaDeviceSynchronize();
      int hb[2];
      cudaMemcpy(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost);
      if (mode == 0) k_tr<0><<<148, 32 * warps, sm>>>(cyc, bad, ITERS);
      else k_tr<1><<<148, 32 * warps, sm>>>(cyc, bad, ITERS);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%s warps=%d  %.1f cycles per transpose (per warp, all warps concurrent)  mismatches=%d  (%s)\n",
             mode ? "tmem" : "smem", warps, (double)mx / ITERS, hb[mode], cudaGetErrorString(e));
    }
  return 0;
}
