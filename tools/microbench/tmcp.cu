// Validates the tcgen05.cp .128x256b source layout used by br_v3.cuh:
// staging image [cidx 64][tmem lane 128][16 B], one instruction per cidx pair,
// descriptor lbo = 2048 (between the two 16-B column chunks), sbo = 128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2306_11006_b200/csrc/mbarrier.cuh"
#include "../../paper_2306_11006_b200/csrc/tmem.cuh"
#include "../../paper_2306_11006_b200/csrc/ks_tc.cuh"
using namespace gw;

__device__ __forceinline__ void tm_cp(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}

__global__ void k(const uint32_t* img, int* bad, int lbo, int sbo) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 131072 + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(slot, 512);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t base = *slot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar[0], 131072);
    bulk_g2s(smem, img, 131072, &bar[0]);
    mbar_wait(&bar[0], 0);
    const uint32_t s0 = smem_u32(smem);
    for (int j = 0; j < 32; ++j)
      tm_cp(base + 256 + 8 * j, umma_desc(s0 + j * 4096, lbo, sbo));
    umma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  tm_fence_after();
  int nbad = 0;
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t r[32];
    tm_ld_raw<32>(base + ((uint32_t)(32 * warp) << 16) + 256 + c0, r);
    tm_wait_ld();
    for (int k2 = 0; k2 < 32; ++k2) {
      const int col = c0 + k2, cidx = col / 4, wd = col % 4, tl = 32 * warp + lane;
      const uint32_t want = (uint32_t)(cidx * 100000 + tl * 10 + wd);
      if (r[k2] != want) {
        if (nbad < 3 && lane == 0) printf("warp %d lane %d col %d got %u want %u\n", warp, lane, col, r[k2], want);
        ++nbad;
      }
    }
  }
  atomicAdd(bad, nbad);
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(base, 512);
}

// throughput of the v3 TMA-mode key path: (a) 32 x tcgen05.cp.128x256b of a
// resident 128 KB slab, (b) cp.async.bulk of 128 KB, (c) both chained
__global__ void k_rate(const unsigned char* img, long long* out, int iters) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 131072 + 32);
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(slot, 512);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t base = *slot;
  if (threadIdx.x == 0) {
    const uint32_t s0 = smem_u32(smem);
    uint32_t ph0 = 0, ph1 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 32; ++j) tm_cp(base + 8 * j, umma_desc(s0 + j * 4096, 2048, 128));
      umma_commit(&bar[1]);
      mbar_wait(&bar[1], ph1); ph1 ^= 1;
    }
    long long t1 = clock64();
    for (int it = 0; it < iters; ++it) {
      mbar_expect_tx(&bar[0], 131072);
      bulk_g2s(smem, img + (size_t)(it % 64) * 131072, 131072, &bar[0]);
      mbar_wait(&bar[0], ph0); ph0 ^= 1;
    }
    long long t2 = clock64();
    for (int it = 0; it < iters; ++it) {
      mbar_expect_tx(&bar[0], 131072);
      bulk_g2s(smem, img + (size_t)(it % 64) * 131072, 131072, &bar[0]);
      mbar_wait(&bar[0], ph0); ph0 ^= 1;
      for (int j = 0; j < 32; ++j) tm_cp(base + 256 * (it & 1) + 8 * j, umma_desc(s0 + j * 4096, 2048, 128));
      umma_commit(&bar[1]);
      mbar_wait(&bar[1], ph1); ph1 ^= 1;
    }
    long long t3 = clock64();
    out[blockIdx.x * 3 + 0] = (t1 - t0) / iters;
    out[blockIdx.x * 3 + 1] = (t2 - t1) / iters;
    out[blockIdx.x * 3 + 2] = (t3 - t2) / iters;
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(base, 512);
}

int main() {
  uint32_t* h = new uint32_t[32768];
  for (int cidx = 0; cidx < 64; ++cidx)
    for (int tl = 0; tl < 128; ++tl)
      for (int wd = 0; wd < 4; ++wd) h[(cidx * 128 + tl) * 4 + wd] = cidx * 100000 + tl * 10 + wd;
  uint32_t* d;
  int* bad;
  cudaMalloc(&d, 131072);
  cudaMalloc(&bad, 4);
  cudaMemcpy(d, h, 131072, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 64);
  int combos[1][2] = {{2048, 128}};
  for (auto& cb : combos) {
    cudaMemset(bad, 0, 4);
    k<<<1, 128, 131072 + 64>>>(d, bad, cb[0], cb[1]);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = -1;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("lbo=%d sbo=%d: %s, mismatches %d\n", cb[0], cb[1], cudaGetErrorString(e), hb);
  }
  {
    unsigned char* img;
    long long* o;
    cudaMalloc(&img, (size_t)64 * 131072);
    cudaMemset(img, 3, (size_t)64 * 131072);
    cudaMalloc(&o, 148 * 3 * 8);
    cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 64);
    for (int grid : {1, 148}) {
      k_rate<<<grid, 128, 131072 + 64>>>(img, o, 200);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[3];
      cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
      printf("grid %3d (%s): tcgen05.cp 128 KB %lld cyc, bulk 128 KB %lld cyc, bulk+cp %lld cyc\n", grid,
             cudaGetErrorString(e), h[0], h[1], h[2]);
    }
  }
  return 0;
}
