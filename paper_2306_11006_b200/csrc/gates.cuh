// gates.cuh -- gate prologue / epilogue kernels around the bootstrap.
//
// Reference: gatewave/cggi.py:785-854 (`eval_gate_batch`): the per-kind
// linear combination (_GATE_COMBO, :177-184), the MUX pair (:823-830), and
// the bootstrap-free kinds NOT (:812-814), COPY (:809-810), CONST (:801-807).
// Every kernel addresses ciphertext rows through (base, stride) pairs so the
// same code serves batched operand matrices and the device wire store.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "keyswitch.cuh"

namespace gw {

// Row counts go on grid.y, which CUDA caps at 65535: launches clamp it and the
// kernels loop over rows with a gridDim.y stride.
__host__ __device__ inline unsigned grid_rows(int64_t rows) {
  return (unsigned)(rows < 1 ? 1 : rows > 65535 ? 65535 : rows);
}


struct CheapUnit {     // bootstrap-free gate
  int32_t kind;        // 0 COPY, 1 NOT, 2 CONST0, 3 CONST1
  int32_t src;
  int32_t dst;
  int32_t pad;
};

__global__ void k_lin(const uint32_t* __restrict__ rows, int64_t stride, const LinJob* __restrict__ jobs,
                      int J, int W, uint32_t mu, uint32_t* __restrict__ lin, int64_t lin_stride) {
  // rows on grid.y with a grid-stride loop: gridDim.y is capped at 65535 (grid_rows())
  for (int j = blockIdx.y; j < J; j += gridDim.y) {
    const LinJob jb = jobs[j];
    const uint32_t* r0 = rows + (size_t)jb.src[0] * stride;
    const uint32_t* r1 = jb.src[1] >= 0 ? rows + (size_t)jb.src[1] * stride : nullptr;
    uint32_t* dst = lin + (size_t)j * lin_stride;
    for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < W; col += gridDim.x * blockDim.x) {
      uint32_t v = (uint32_t)jb.w[0] * r0[col];
      if (r1) v += (uint32_t)jb.w[1] * r1[col];
      if (col == W - 1) v += (uint32_t)jb.cmu * mu;
      dst[col] = v;
    }
  }
}

// Wire exchange: rows of a level's send list <-> a contiguous buffer (uint4 moves).
__global__ void k_xpack(const uint32_t* __restrict__ wires, int64_t stride, const int64_t* __restrict__ ids,
                        int64_t count, uint32_t* __restrict__ dst, int64_t dst_stride) {
  for (int64_t row = blockIdx.y; row < count; row += gridDim.y) {
    const uint4* s4 = reinterpret_cast<const uint4*>(wires + (size_t)ids[row] * stride);
    uint4* d4 = reinterpret_cast<uint4*>(dst + (size_t)row * dst_stride);
    for (int k = threadIdx.x; k < stride / 4; k += blockDim.x) d4[k] = s4[k];
  }
}
__global__ void k_xscatter(uint32_t* __restrict__ wires, int64_t stride, const int64_t* __restrict__ ids,
                           int64_t count, const uint32_t* __restrict__ src, int64_t src_stride) {
  for (int64_t row = blockIdx.y; row < count; row += gridDim.y) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + (size_t)row * src_stride);
    uint4* d4 = reinterpret_cast<uint4*>(wires + (size_t)ids[row] * stride);
    for (int k = threadIdx.x; k < stride / 4; k += blockDim.x) d4[k] = s4[k];
  }
}

__global__ void k_zero_units(const KsUnit* __restrict__ units, int U, uint32_t* out, int64_t stride, int W) {
  for (int u = blockIdx.y; u < U; u += gridDim.y) {
    uint32_t* row = out + (size_t)units[u].out_row * stride;
    for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < W; col += gridDim.x * blockDim.x) row[col] = 0;
  }
}

__global__ void k_cheap(const uint32_t* __restrict__ src_rows, int64_t src_stride, const CheapUnit* __restrict__ units,
                        int C, int W, uint32_t mu, uint32_t* dst_rows, int64_t dst_stride) {
  for (int u = blockIdx.y; u < C; u += gridDim.y) {
    const CheapUnit cu = units[u];
    uint32_t* dst = dst_rows + (size_t)cu.dst * dst_stride;
    const uint32_t* src = cu.src >= 0 ? src_rows + (size_t)cu.src * src_stride : nullptr;
    for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < W; col += gridDim.x * blockDim.x) {
      uint32_t v;
      switch (cu.kind) {
        case 0: v = src[col]; break;
        case 1: v = 0u - src[col]; break;
        case 2: v = (col == W - 1) ? 0u - mu : 0u; break;
        default: v = (col == W - 1) ? mu : 0u; break;
      }
      dst[col] = v;
    }
  }
}

// ext (B, N+1) -> pseudo accumulators (B, 2, N) whose extraction is ext
// (lets the seam-1 `_keyswitch_kernel` twin reuse the fused kernel).
__global__ void k_ext_to_acc(const uint32_t* __restrict__ ext, int64_t B, int N, uint32_t* __restrict__ acc) {
  for (int64_t g = blockIdx.y; g < B; g += gridDim.y) {
    const uint32_t* e = ext + g * (N + 1);
    uint32_t* a = acc + g * 2 * N;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < 2 * N; j += gridDim.x * blockDim.x) {
      uint32_t v = 0;
      if (j == 0) v = e[0];
      else if (j < N) v = 0u - e[N - j];
      else if (j == N) v = e[N];
      a[j] = v;
    }
  }
}

}  // namespace gw
