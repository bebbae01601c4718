// keyswitch.cuh -- fused sample-extract + keyswitch (+ MUX combine).
//
// Reference: gatewave/cggi.py:695-704 `_extract_rows`, :670-692
// `_keyswitch_kernel`, and the MUX recombination at :842-846.
//
//   ext[0] = acc0[0], ext[j] = -acc0[N-j] (0<j<N), ext[N] = acc1[0]
//   (MUX: ext = ext(job0) + ext(job1), ext[N] += mu)
//   u = (ext[i] + 2^(31-t*gamma)) >> (32 - t*gamma)
//   out = (0,...,0, ext[N]) - sum_{i<N, j<t, d_ij != 0} ksk[i][j][d_ij - 1][:]
//
// Grid = (gate tiles of GT) x (chunks of the N input coefficients).  Each
// thread owns 4 consecutive output columns (one uint4 of every KSK row), so a
// KSK row is read once per gate tile with fully coalesced 16-byte loads and
// reused from registers by all GT gates of the tile.  Partial sums of the
// chunks are combined with u32 atomics: wrap-around addition is associative,
// so the result is deterministic and bit-exact for any chunking.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gw {

struct KsUnit {       // one output sample
  int32_t job0;       // accumulator row (blind-rotation job) of the sample
  int32_t job1;       // second job for MUX, else -1
  int32_t out_row;    // destination row index
  uint32_t add_b;     // added to ext[N] (mu for MUX, else 0)
};

struct KsArgs {
  const uint32_t* acc;   // (jobs, 2, N)
  const KsUnit* units;   // (count)
  int count;
  const uint32_t* ksk;   // (N, t, V, Wp) u32
  int N;
  int t;
  int gamma;
  int W;                 // n + 1
  int Wp;                // padded row stride (multiple of 4)
  int chunk;             // input coefficients per CTA
  uint32_t* out;         // rows of out_stride words, zeroed beforehand
  int64_t out_stride;
};

template <int GT, int V>
__global__ void __launch_bounds__(160) k_keyswitch(KsArgs a) {
  extern __shared__ uint32_t ks_u[];  // [GT][chunk]
  const int tile0 = blockIdx.x * GT;
  const int i0 = blockIdx.y * a.chunk;
  const int iend = min(a.N, i0 + a.chunk);
  const int tg = a.t * a.gamma;
  const uint32_t roff = 1u << (32 - tg - 1);
  const int rsh = 32 - tg;
  const int N = a.N;

  for (int e = threadIdx.x; e < GT * a.chunk; e += blockDim.x) {
    const int gg = e / a.chunk, ii = e % a.chunk, i = i0 + ii;
    uint32_t u = 0;
    if (tile0 + gg < a.count && i < iend) {
      const KsUnit un = a.units[tile0 + gg];
      const uint32_t* acc0 = a.acc + (size_t)un.job0 * 2 * N;
      uint32_t x = (i == 0) ? acc0[0] : 0u - acc0[N - i];
      if (un.job1 >= 0) {
        const uint32_t* acc1 = a.acc + (size_t)un.job1 * 2 * N;
        x += (i == 0) ? acc1[0] : 0u - acc1[N - i];
      }
      u = (uint32_t)(((uint64_t)x + roff) >> rsh);
    }
    ks_u[e] = u;
  }
  __syncthreads();

  const int col4 = threadIdx.x;
  const int ncol4 = a.Wp >> 2;
  if (col4 >= ncol4) return;
  const uint4* ksk4 = reinterpret_cast<const uint4*>(a.ksk);
  const uint32_t dmask = (1u << a.gamma) - 1;
  const int Vr = (1 << a.gamma) - 1;

  uint4 sum[GT];
#pragma unroll
  for (int g = 0; g < GT; ++g) sum[g] = make_uint4(0, 0, 0, 0);

  for (int i = i0; i < iend; ++i) {
    for (int j = 0; j < a.t; ++j) {
      const size_t rowbase = ((size_t)i * a.t + j) * Vr;
      const int sh = (a.t - 1 - j) * a.gamma;
      if (V > 0) {
        uint4 rows[V > 0 ? V : 1];
#pragma unroll
        for (int v = 0; v < V; ++v) rows[v] = __ldg(ksk4 + (rowbase + v) * ncol4 + col4);
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          const uint32_t d = (ks_u[g * a.chunk + (i - i0)] >> sh) & dmask;
          uint4 r = make_uint4(0, 0, 0, 0);
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (d == (uint32_t)(v + 1)) r = rows[v];
          sum[g].x += r.x; sum[g].y += r.y; sum[g].z += r.z; sum[g].w += r.w;
        }
      } else {
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          const uint32_t d = (ks_u[g * a.chunk + (i - i0)] >> sh) & dmask;
          if (d) {
            const uint4 r = __ldg(ksk4 + (rowbase + d - 1) * ncol4 + col4);
            sum[g].x += r.x; sum[g].y += r.y; sum[g].z += r.z; sum[g].w += r.w;
          }
        }
      }
    }
  }

#pragma unroll
  for (int g = 0; g < GT; ++g) {
    if (tile0 + g >= a.count) break;
    const KsUnit un = a.units[tile0 + g];
    uint32_t* orow = a.out + (size_t)un.out_row * a.out_stride;
    uint32_t vals[4] = {sum[g].x, sum[g].y, sum[g].z, sum[g].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int col = col4 * 4 + q;
      if (col >= a.W) break;
      uint32_t v = 0u - vals[q];
      if (col == a.W - 1 && blockIdx.y == 0) {
        const uint32_t* acc0 = a.acc + (size_t)un.job0 * 2 * N;
        uint32_t b = acc0[N];
        if (un.job1 >= 0) b += a.acc[(size_t)un.job1 * 2 * N + N];
        v += b + un.add_b;
      }
      atomicAdd(orow + col, v);
    }
  }
}

}  // namespace gw
