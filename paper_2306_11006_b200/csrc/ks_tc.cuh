// ks_tc.cuh -- keyswitch as an exact INT8 tensor-core GEMM (tcgen05.mma kind::i8).
//
// Reference: gatewave/cggi.py:670-692 `_keyswitch_kernel` (+ :695-704 extract,
// :842-846 MUX combine).  With digits d_{g,i,j} (MSB-first base-2^gamma digits
// of the rounded extracted sample) the keyswitch is
//     out[g][c] = b_g - sum_{i,j} ksk[i][j][d-1][c]        (d = 0 adds nothing)
//             = b_g - sum_k A[g][k] * K[k][c]   (mod 2^32)
// with a one-hot A (k = 4*(i*t+j) + d-1; the 4th value of each quadruple is a
// zero pad row) and K the key.  Splitting K into its four byte planes makes
// every product an exact u8 x u8 -> s32 tensor-core MMA (|partial| <= 2^21);
// the planes recombine as sum_p C_p << 8p mod 2^32, and split-K partials add
// with u32 atomics -- wrap-around addition is associative, so the result is
// bit-exact for any tiling.
//
// Tile: M = 128 samples (TMEM lanes) x N = 256 packed columns (64 output
// columns x 4 planes, int32 accumulators in 256 TMEM columns) x K blocks of
// 128 bytes (32 (i,j) pairs).  Warp roles: 0 = TMA producer of the key image
// (cp.async.bulk, one 32 KB block per stage), 1 = TMEM allocator + single-
// thread MMA issuer, 2..5 = one-hot A producers, then the epilogue.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "keyswitch.cuh"
#include "mbarrier.cuh"
#include "tmem.cuh"

namespace gw {

constexpr int KT_M = 128;
constexpr int KT_N = 256;
constexpr int KT_COLS = KT_N / 4;        // output columns per N tile
constexpr int KT_KB = 128;               // K bytes per stage
constexpr int KT_PAIRS = KT_KB / 4;      // (i,j) pairs per stage
constexpr int KT_STAGES = 4;
constexpr int KT_A_BYTES = KT_M * KT_KB;  // 16 KB
constexpr int KT_B_BYTES = KT_N * KT_KB;  // 32 KB
constexpr int KT_THREADS = 192;

struct KtArgs {
  const uint32_t* ut;      // (N, ut_stride): rounded samples u[g][i], transposed
  int64_t ut_stride;
  const uint32_t* body;    // (count): b term per sample
  const KsUnit* units;     // (count): output rows
  int count;
  const uint8_t* kimg;     // key image: [ntile][kblock][kc 8][n 256][16 B]
  int kblocks;             // total K blocks = N*t / 32
  int blocks_per_split;
  int t;                   // keyswitch levels
  int gamma;
  int W;                   // n + 1
  uint32_t* out;
  int64_t out_stride;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x
// 16 bytes; sbo = byte stride between 8-row groups, lbo = between 16-byte K chunks.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// kind::i8 instruction descriptor: D s32, A/B u8, both K-major, M=128, N=256.
constexpr uint32_t KT_IDESC = (2u << 4) | ((uint32_t)(KT_N >> 3) << 17) | ((uint32_t)(KT_M >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(KT_IDESC), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <int T>  // keyswitch levels t (divides 32): compile-time so the digit buffers stay in registers
__global__ void __launch_bounds__(KT_THREADS, 1) k_keyswitch_tc(KtArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint8_t* sA = smem;                                   // [stage][kc 8][m 128][16]
  uint8_t* sB = smem + KT_STAGES * KT_A_BYTES;          // [stage][kc 8][n 256][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + KT_STAGES * KT_B_BYTES);
  uint64_t* full_a = bars;
  uint64_t* full_b = bars + KT_STAGES;
  uint64_t* empty = bars + 2 * KT_STAGES;
  uint64_t* done = bars + 3 * KT_STAGES;
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(bars + 3 * KT_STAGES + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = blockIdx.x, nt = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * a.blocks_per_split;
  const int kb1 = min(a.kblocks, kb0 + a.blocks_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < KT_STAGES; ++s) {
      mbar_init(&full_a[s], 128);
      mbar_init(&full_b[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tm_alloc(tm_slot, 256);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tmem = *tm_slot;

  if (warp == 0) {
    // ---- TMA producer: key image blocks -----------------------------------
    if (lane == 0) {
      const uint8_t* src = a.kimg + ((size_t)nt * a.kblocks + kb0) * KT_B_BYTES;
      for (int k = 0; k < nkb; ++k) {
        const int s = k % KT_STAGES;
        mbar_wait(&empty[s], ((k / KT_STAGES) & 1) ^ 1);
        mbar_expect_tx(&full_b[s], KT_B_BYTES);
        bulk_g2s(sB + (size_t)s * KT_B_BYTES, src + (size_t)k * KT_B_BYTES, KT_B_BYTES, &full_b[s]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ---------------------------------------------------------
    if (lane == 0) {
      for (int k = 0; k < nkb; ++k) {
        const int s = k % KT_STAGES;
        const uint32_t par = (k / KT_STAGES) & 1;
        mbar_wait(&full_a[s], par);
        mbar_wait(&full_b[s], par);
        tm_fence_after();
        const uint32_t abase = smem_u32(sA + (size_t)s * KT_A_BYTES);
        const uint32_t bbase = smem_u32(sB + (size_t)s * KT_B_BYTES);
#pragma unroll
        for (int q = 0; q < KT_KB / 32; ++q) {  // K = 32 bytes per MMA = two 16-byte chunks
          const uint64_t da = umma_desc(abase + q * 2 * (KT_M * 16), KT_M * 16, 128);
          const uint64_t db = umma_desc(bbase + q * 2 * (KT_N * 16), KT_N * 16, 128);
          umma_i8(tmem, da, db, (k | q) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
  } else {
    // ---- one-hot A producers: thread m <-> sample row m ----------------------
    const int m = threadIdx.x - 64;  // 0..127
    const int g = mt * KT_M + m;
    const bool valid = g < a.count;
    const uint32_t dmask = (1u << a.gamma) - 1;
    const uint32_t* urow = a.ut + (valid ? g : 0);
    // A K block spans KT_PAIRS / t input coefficients (t divides 32, so at most
    // 32 when t = 1).  The samples of the next PD - 1 blocks are in flight while
    // block k is built (a register ring of PD blocks, PD * UMAX <= 32 words for
    // t >= 2), so the global-load latency is paid once per PD blocks, not per block.
    constexpr int UMAX = KT_PAIRS / T;  // coefficients per K block
    constexpr int PD = T >= 2 ? T : 2;  // ring depth (blocks)
    uint32_t ub[PD][UMAX];
    auto load_u = [&](int k, uint32_t (&dst)[UMAX]) {
      const int c0 = ((kb0 + k) * KT_PAIRS) / T;
#pragma unroll
      for (int q = 0; q < UMAX; ++q)
        dst[q] = (valid && k < nkb) ? __ldg(urow + (size_t)(c0 + q) * a.ut_stride) : 0u;
    };
#pragma unroll
    for (int d = 0; d < PD; ++d) load_u(d, ub[d]);
    for (int k0 = 0; k0 < nkb; k0 += PD) {
#pragma unroll
      for (int d = 0; d < PD; ++d) {
        const int k = k0 + d;
        if (k >= nkb) break;
        const int s = k % KT_STAGES;
        mbar_wait(&empty[s], ((k / KT_STAGES) & 1) ^ 1);
        uint8_t* dst = sA + (size_t)s * KT_A_BYTES + m * 16;
#pragma unroll
        for (int kc = 0; kc < KT_KB / 16; ++kc) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pl = kc * 4 + e;  // pair within the block; pairs of a coefficient are consecutive
            const int j = pl % T;
            const uint32_t u = ub[d][pl / T];
            const uint32_t dg = (u >> ((T - 1 - j) * a.gamma)) & dmask;
            w[e] = dg ? (1u << (8 * (dg - 1))) : 0u;
          }
          *reinterpret_cast<uint4*>(dst + kc * KT_M * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_async_smem();
        mbar_arrive(&full_a[s]);
        load_u(k + PD, ub[d]);
      }
    }
    // ---- epilogue: TMEM -> registers -> recombine planes -> atomics --------
    mbar_wait(done, 0);
    tm_fence_after();
    const int q4 = warp & 3;                 // TMEM sub-partition of this warp
    const int row = q4 * 32 + lane;          // accumulator lane = sample row
    const int gr = mt * KT_M + row;
    const bool vrow = gr < a.count;
    const KsUnit un = vrow ? a.units[gr] : KsUnit{0, -1, 0, 0u};
    uint32_t* orow = a.out + (size_t)un.out_row * a.out_stride;
#pragma unroll 1
    for (int cb = 0; cb < KT_N; cb += 32) {
      uint32_t v[32];
      tm_ld_raw<32>(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)cb, v);
      tm_wait_ld();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = nt * KT_COLS + cb / 4 + c;
        if (!vrow || col >= a.W) continue;
        uint32_t sum = v[4 * c] + (v[4 * c + 1] << 8) + (v[4 * c + 2] << 16) + (v[4 * c + 3] << 24);
        uint32_t val = 0u - sum;
        if (col == a.W - 1 && split == 0) val += a.body[gr];
        atomicAdd(orow + col, val);
      }
    }
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 1) tm_dealloc(tmem, 256);
}

// Rounded samples u = (ext[i] + 2^(31 - t*gamma)) >> (32 - t*gamma), transposed
// (N, ut_stride), and body terms, from the accumulators (fused extraction and
// MUX combine, cggi.py:695-704, 842-845).  Also zeroes the output rows the
// keyswitch's split-K atomics add into (one launch fewer per level).
__global__ void k_ks_prep(const uint32_t* __restrict__ acc, const KsUnit* __restrict__ units, int count, int N,
                          int tg, uint32_t* __restrict__ ut, int64_t ut_stride, uint32_t* __restrict__ body,
                          uint32_t* __restrict__ out, int64_t out_stride, int W) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (g >= count) return;
  const KsUnit un = units[g];
  for (int col = i; col < W; col += N) out[(size_t)un.out_row * out_stride + col] = 0u;
  const uint32_t* a0 = acc + (size_t)un.job0 * 2 * N;
  uint32_t x = (i == 0) ? a0[0] : 0u - a0[N - i];
  if (un.job1 >= 0) {
    const uint32_t* a1 = acc + (size_t)un.job1 * 2 * N;
    x += (i == 0) ? a1[0] : 0u - a1[N - i];
  }
  const uint32_t roff = 1u << (32 - tg - 1);
  ut[(size_t)i * ut_stride + g] = (uint32_t)(((uint64_t)x + roff) >> (32 - tg));
  if (i == 0) {
    uint32_t b = a0[N];
    if (un.job1 >= 0) b += acc[(size_t)un.job1 * 2 * N + N];
    body[g] = b + un.add_b;
  }
}

// One-time key image: ksk (N, t, V, Wp) u32 -> [ntile][kblock][kc][n][16 B]
// bytes, n = 4*column + plane, k = 4*(i*t+j) + v (v = V.. are zero pads).
__global__ void k_ksk_to_tc(const uint32_t* __restrict__ ksk, int N, int t, int V, int W, int Wp, int ntiles,
                            int kblocks, uint8_t* __restrict__ img) {
  const size_t chunk = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte chunk
  const size_t total = (size_t)ntiles * kblocks * (KT_KB / 16) * KT_N;
  if (chunk >= total) return;
  const int n = (int)(chunk % KT_N);
  const int kc = (int)((chunk / KT_N) % (KT_KB / 16));
  const int kb = (int)((chunk / ((size_t)KT_N * (KT_KB / 16))) % kblocks);
  const int nt = (int)(chunk / ((size_t)KT_N * (KT_KB / 16) * kblocks));
  const int col = nt * KT_COLS + n / 4, plane = n % 4;
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const int k = kb * KT_KB + kc * 16 + kk;
    const int pair = k / 4, v = k % 4;
    uint32_t byte = 0;
    if (v < V && col < W && pair < N * t) byte = (ksk[((size_t)pair * V + v) * Wp + col] >> (8 * plane)) & 0xFFu;
    w[kk / 4] |= byte << (8 * (kk % 4));
  }
  *reinterpret_cast<uint4*>(img + chunk * 16) = make_uint4(w[0], w[1], w[2], w[3]);
}

}  // namespace gw
