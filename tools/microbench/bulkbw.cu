// L2 -> shared-memory bulk-copy (cp.async.bulk) throughput when every SM
// streams the SAME 128 KB slab sequence (the v3 key pattern) vs distinct slabs,
// for several chunk sizes; plus an LDG.128 baseline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2306_11006_b200/csrc/mbarrier.cuh"
#include "../../paper_2306_11006_b200/csrc/ks_tc.cuh"
using namespace gw;
constexpr int SLAB = 131072;

__global__ void k_bulk(const unsigned char* src, int nslab, int chunk, int distinct, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SLAB);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nslab; ++s) {
      const int slab = distinct ? (s + blockIdx.x * 7) % nslab : s;
      mbar_expect_tx(bar, SLAB);
      for (int c = 0; c < SLAB; c += chunk) bulk_g2s(smem + c, src + (size_t)slab * SLAB + c, chunk, bar);
      mbar_wait(bar, s & 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void k_ldg(const uint4* src, int nslab, int distinct, long long* cyc, int* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint4* s4 = reinterpret_cast<uint4*>(smem);
  __syncthreads();
  long long t0 = clock64();
  for (int s = 0; s < nslab; ++s) {
    const int slab = distinct ? (s + blockIdx.x * 7) % nslab : s;
    const uint4* p = src + (size_t)slab * (SLAB / 16);
    for (int k = threadIdx.x; k < SLAB / 16; k += blockDim.x) s4[k] = __ldg(p + k);
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const int nslab = 630;
  unsigned char* src;
  long long* cyc;
  int* sink;
  cudaMalloc(&src, (size_t)nslab * SLAB);
  cudaMemset(src, 1, (size_t)nslab * SLAB);
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB + 64);
  cudaFuncSetAttribute(k_ldg, cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB + 64);
  long long h[148];
  for (int distinct = 0; distinct < 2; ++distinct) {
    for (int chunk : {131072, 32768, 8192, 2048}) {
      for (int rep = 0; rep < 2; ++rep) k_bulk<<<148, 32, SLAB + 64>>>(src, nslab, chunk, distinct, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (long long v : h) { mx = v > mx ? v : mx; sum += v; }
      printf("bulk  %s chunk %6d: %7.0f cyc/slab avg, %7.0f max  (%.1f B/clk/SM)  %s\n", distinct ? "distinct" : "same    ",
             chunk, (double)sum / 148 / nslab, (double)mx / nslab, SLAB / ((double)sum / 148 / nslab),
             cudaGetErrorString(cudaGetLastError()));
    }
    for (int thr : {128, 256, 512}) {
      for (int rep = 0; rep < 2; ++rep) k_ldg<<<148, thr, SLAB + 64>>>((const uint4*)src, nslab, distinct, cyc, sink);
      cudaDeviceSynchronize();
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long sum = 0;
      for (long long v : h) sum += v;
      printf("ldg   %s threads %4d: %7.0f cyc/slab avg (%.1f B/clk/SM)\n", distinct ? "distinct" : "same    ", thr,
             (double)sum / 148 / nslab, SLAB / ((double)sum / 148 / nslab));
    }
  }
  return 0;
}
