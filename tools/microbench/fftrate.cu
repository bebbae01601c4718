// Achievable FP64 rate of the engine's own FFT code paths (csrc/fft.cuh):
//  A: in-register DIF+DIT DFT-16 pairs (no memory)      -> pure butterfly rate
//  B: full warp FFT-512 forward+inverse with smem transpose + shuffles
// Reported as FP64 warp-instructions per SM-cycle (peak 2.0 = 64 lanes/clk).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2306_11006_b200/csrc/fft.cuh"
using namespace gw;

template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_reg(double* out, int iters) {
  double2 x[16];
  for (int k = 0; k < 16; ++k) x[k] = make_double2(threadIdx.x * 0.001 + k, k * 0.5);
  for (int it = 0; it < iters; ++it) {
    dif<16, +1>(x);
    dit<16, -1>(x);
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = make_double2(x[k].x * 0.0625, x[k].y * 0.0625);
  }
  double s = 0;
  for (int k = 0; k < 16; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_fft(const double2* tables, double* out, int iters) {
  extern __shared__ double2 dyn[];
  double2* tw = dyn;
  double2 (*tiles)[512] = reinterpret_cast<double2 (*)[512]>(dyn + 512);
  for (int t = threadIdx.x; t < 512; t += blockDim.x) tw[t] = tables[2 * 512 + t];
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  double2 x[16];
  for (int k = 0; k < 16; ++k) x[k] = make_double2(threadIdx.x * 0.001 + k, k * 0.5);
  for (int it = 0; it < iters; ++it) {
    fft_forward<10, true>(x, tiles[w], tw, l);
    fft_inverse<10, true>(x, tiles[w], tw, l);
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = make_double2(x[k].x * (1.0 / 512), x[k].y * (1.0 / 512));
  }
  double s = 0;
  for (int k = 0; k < 16; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double2 roots[64];
  for (int t = 0; t < 64; ++t) roots[t] = make_double2(cos(2 * M_PI * t / 64), sin(2 * M_PI * t / 64));
  cudaMemcpyToSymbol(c_root64, roots, sizeof(roots));
  double2* tab;
  cudaMalloc(&tab, 3 * 512 * sizeof(double2));
  double2 h[3 * 512];
  for (int i = 0; i < 3 * 512; ++i) h[i] = make_double2(cos(i * 0.01), sin(i * 0.01));
  cudaMemcpy(tab, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, 148 * 1024 * sizeof(double));
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  auto run = [&](const char* name, auto launch, double fp64_per_iter_per_warp, int warps) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double cycles = ms * 1e-3 * clk * 1e3;
    double instr = fp64_per_iter_per_warp * iters * warps;  // per SM (grid = 148 CTAs)
    printf("%-28s warps/SM %2d  %.3f ms  FP64 warp-instr/SM-clk %.3f  (%.0f%% of peak)\n", name, warps, ms,
           instr / cycles, 100.0 * instr / cycles / 2.0);
  };
  // FP64 instruction counts per iteration per warp, from SASS (printed below by cuobjdump)
  const double reg_ops = 368;  // FP64 SASS instructions per iteration (cuobjdump)
  const double fft_ops = 968;
  run("reg DIF/DIT-16", [&] { k_reg<4><<<148, 128>>>(out, iters); }, reg_ops, 4);
  run("reg DIF/DIT-16", [&] { k_reg<8><<<148, 256>>>(out, iters); }, reg_ops, 8);
  run("reg DIF/DIT-16", [&] { k_reg<16><<<148, 512>>>(out, iters); }, reg_ops, 16);
  const size_t sm4 = (512 + 4 * 512) * 16, sm8 = (512 + 8 * 512) * 16, sm16 = (512 + 16 * 512) * 16;
  cudaFuncSetAttribute(k_fft<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
  cudaFuncSetAttribute(k_fft<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm8);
  cudaFuncSetAttribute(k_fft<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16);
  run("fft512 fwd+inv (smem)", [&] { k_fft<4><<<148, 128, sm4>>>(tab, out, iters); }, fft_ops, 4);
  run("fft512 fwd+inv (smem)", [&] { k_fft<8><<<148, 256, sm8>>>(tab, out, iters); }, fft_ops, 8);
  run("fft512 fwd+inv (smem)", [&] { k_fft<16><<<148, 512, sm16>>>(tab, out, iters); }, fft_ops, 16);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
