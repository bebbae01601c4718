// blind_rotate.cuh -- fused batched blind rotation (reference:
// gatewave/cggi.py:592-667 `_blind_rotate_kernel`).
//
// One CTA holds GC gates for the whole n-step loop; the TRLWE accumulator of
// every gate stays in shared memory from the initial rotation to the end.
// Two warps serve one gate: warp c (c = 0, 1) owns accumulator component c,
// computes its l digit rows (rows c*l .. c*l+l-1, cggi.py:642-644) through the
// forward FFT, and after a pair barrier multiply-accumulates ALL 2l rows
// against the bootstrapping-key slab of component c (both 16-bit halves),
// inverse-transforms the two halves and adds lo + 2^16 hi into acc[c].
// Per step per gate: 2l forward + 4 inverse FFT-M, 2l*2*2*M complex MACs.
#pragma once
#include "fft.cuh"

namespace gw {

struct BrArgs {
  const uint32_t* lin;   // (B, lin_stride) u32: LWE rows [a_0..a_{n-1}, b]
  int64_t lin_stride;
  int B;
  int n;
  const uint32_t* tv;    // (2, N) test vector
  const double2* bk;     // native FFT layout, see bk_index()
  const double2* tables; // [tw1: P*L][twist: P*L]
  uint32_t* acc_out;     // (B, 2, N)
  int bg_bits;
  uint32_t offs;         // decomposition offset (cggi.py:516-522)
  int gates_per_cta;
  long long* prof;       // optional per-phase cycle counters (debug; nullptr = off)
  int ablate;            // debug timing ablations (0 = exact kernel); see br_tmem.cuh
  // rounding-margin probe (gw_set_margin_probe): max |x - rint(x)| over every
  // FP64 value the inverse transforms round, as the bits of a positive double
  unsigned long long* margin = nullptr;
  // fused gate prologue (v3): when jobs != nullptr, gate g's LWE row is
  // w0*rows[src0] + w1*rows[src1] (+ cmu*mu on the body) instead of lin[g]
  const LinJob* jobs = nullptr;
  const uint32_t* rows = nullptr;
  int64_t row_stride = 0;
  uint32_t mu = 0;
  // L2 warm-up of the next kernel's operand (v5): over the last kL2WarmSteps steps each CTA
  // prefetches its 1/gridDim share of these bytes (the keyswitch key image) into L2
  const char* l2warm = nullptr;
  uint64_t l2warm_bytes = 0;
};

// Bootstrapping key, FFT domain: [i][c][h][s][r][lane] complex, scaled by 1/M.
// One (i, c, h) slice is the contiguous slab one MAC warp consumes per step.
template <int LOGN, int LEV>
__host__ __device__ __forceinline__ size_t bk_index(int i, int c, int s, int r, int h, int l) {
  using G = Geo<LOGN>;
  return ((((size_t)(i * 2 + c) * 2 + h) * G::P + s) * (2 * LEV) + r) * G::L + l;
}

template <int LOGN, int LEV>
struct BrSmem {
  using G = Geo<LOGN>;
  static constexpr int TABLES = 2 * G::TILE;            // double2
  static constexpr int XBUF = 2 * LEV * G::TILE;         // double2 per gate (2 warps)
  static size_t bytes(int gc, int n) {
    const size_t lin_words = ((size_t)n + 1 + 3) & ~(size_t)3;
    return sizeof(double2) * (TABLES + (size_t)gc * XBUF) +
           (size_t)gc * (2 * G::N * sizeof(uint32_t) + lin_words * sizeof(uint32_t));
  }
};

template <int LOGN, int LEV>
__global__ void __launch_bounds__(256, 1) k_blind_rotate(BrArgs a) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, M = G::M, P = G::P, L = G::L, R = 2 * LEV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gc = a.gates_per_cta;
  const size_t lin_words = ((size_t)a.n + 1 + 3) & ~(size_t)3;
  double2* tw1 = reinterpret_cast<double2*>(smem_raw);
  double2* twist = tw1 + G::TILE;
  double2* xbuf_all = twist + G::TILE;
  uint32_t* acc_all = reinterpret_cast<uint32_t*>(xbuf_all + (size_t)gc * BrSmem<LOGN, LEV>::XBUF);
  uint32_t* lin_all = acc_all + (size_t)gc * 2 * N;

  for (int t = threadIdx.x; t < 2 * G::TILE; t += blockDim.x) tw1[t] = a.tables[t];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int l = lane & (L - 1);
  const int gl = warp >> 1;
  const int c = warp & 1;
  const int g = blockIdx.x * gc + gl;
  const bool active = gl < gc && g < a.B;

  uint32_t* lin_s = lin_all + (size_t)gl * lin_words;
  uint32_t* acc_g = acc_all + (size_t)gl * 2 * N;
  uint32_t* acc_c = acc_g + c * N;
  double2* xb_g = xbuf_all + (size_t)gl * BrSmem<LOGN, LEV>::XBUF;  // [warp c][lv][tile]
  double2* xb_mine = xb_g + (size_t)c * LEV * G::TILE;

  const uint32_t two_n_mask = 2 * N - 1;
  const uint32_t rshift = 32 - (LOGN + 1);
  const uint32_t radd = 1u << (32 - (LOGN + 1) - 1);

  if (active) {
    const uint32_t* src = a.lin + (size_t)g * a.lin_stride;
    for (int t = c * 32 + lane; t <= a.n; t += 64) lin_s[t] = src[t];
  }
  __syncthreads();
  if (!active) return;

  // acc <- tv * X^{-bbar}   (cggi.py:612-622)
  {
    const uint32_t bbar = ((lin_s[a.n] + radd) >> rshift) & two_n_mask;
    const uint32_t k = (2 * N - bbar) & two_n_mask;
    const uint32_t* tvc = a.tv + c * N;
    for (int j = lane; j < N; j += 32) {
      const uint32_t m = ((uint32_t)j - k) & two_n_mask;
      acc_c[j] = m < (uint32_t)N ? tvc[m] : 0u - tvc[m - N];
    }
  }
  __syncwarp();

  const int bar_id = 1 + gl;
  const uint32_t base_mask = (1u << a.bg_bits) - 1;
  const int32_t half_base = 1 << (a.bg_bits - 1);

  for (int i = 0; i < a.n; ++i) {
    const uint32_t abar = ((lin_s[i] + radd) >> rshift) & two_n_mask;
    // ---- rotate-subtract + gadget digits of acc[c] (cggi.py:627-644) ----
    // lane l owns coefficients j = L*m1 + l (real part) and j + M (imag part)
    uint32_t packed[LEV > 1 ? LEV - 1 : 1][P];
    double2 x[P];
#pragma unroll
    for (int m1 = 0; m1 < P; ++m1) {
      int32_t dg[2][LEV];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t j = (uint32_t)(L * m1 + l + hh * M);
        const uint32_t idx = (j - abar) & two_n_mask;
        const uint32_t v = acc_c[idx & (N - 1)];
        const uint32_t rot = (idx & N) ? 0u - v : v;
        const uint32_t buf = rot - acc_c[j] + a.offs;
#pragma unroll
        for (int lv = 0; lv < LEV; ++lv)
          dg[hh][lv] = (int32_t)((buf >> (32 - (lv + 1) * a.bg_bits)) & base_mask) - half_base;
      }
      const double2 tw = twist[m1 * L + l];
      x[bitrev_c<G::LOGP>(m1)] =
          cmul(make_double2(small_int_to_double(dg[0][0]), small_int_to_double(dg[1][0])), tw);
#pragma unroll
      for (int lv = 1; lv < LEV; ++lv)
        packed[lv - 1][m1] = ((uint32_t)dg[0][lv] & 0xFFFFu) | ((uint32_t)dg[1][lv] << 16);
    }
#pragma unroll
    for (int lv = 0; lv < LEV; ++lv) {
      double2* tile = xb_mine + lv * G::TILE;
      if (lv > 0) {
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) {
          const uint32_t pk = packed[lv - 1][m1];
          const int32_t d0 = (int32_t)(int16_t)(pk & 0xFFFFu);
          const int32_t d1 = (int32_t)pk >> 16;
          x[bitrev_c<G::LOGP>(m1)] = cmul(make_double2(small_int_to_double(d0), small_int_to_double(d1)),
                                          twist[m1 * L + l]);
        }
      }
      fft_forward<LOGN>(x, tile, tw1, l);
      __syncwarp();
#pragma unroll
      for (int s = 0; s < P; ++s) tile[s * L + l] = x[s];
    }
    named_barrier(bar_id, 64);
    // ---- MAC against BK_i slab of component c (cggi.py:648-657) ----
    double2 o0[P], o1[P];
    {
      const double2* bk0 = a.bk + bk_index<LOGN, LEV>(i, c, 0, 0, 0, l);
      const double2* bk1 = a.bk + bk_index<LOGN, LEV>(i, c, 0, 0, 1, l);
#pragma unroll
      for (int s = 0; s < P; ++s) {
        double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2 d = xb_g[(size_t)r * G::TILE + s * L + l];
          const double2 b0 = __ldg(bk0 + (size_t)(s * R + r) * L);
          const double2 b1 = __ldg(bk1 + (size_t)(s * R + r) * L);
          s0 = cfma(s0, d, b0);
          s1 = cfma(s1, d, b1);
        }
        o0[s] = s0;
        o1[s] = s1;
      }
    }
    named_barrier(bar_id, 64);
    // ---- inverse transforms, round, accumulate (cggi.py:658-666) ----
    double2* tile = xb_mine;
    // lanes >= L (N < 1024) duplicate lane l's work; only one copy updates acc
    const bool owner = lane < L;
    fft_inverse<LOGN>(o0, tile, tw1, l);
#pragma unroll
    for (int m1 = 0; m1 < P; ++m1) {
      const double2 v = cmulc(o0[m1], twist[m1 * L + l]);
      const uint32_t j = (uint32_t)(L * m1 + l);
      if (owner) {
        acc_c[j] += round_mod32(v.x);
        acc_c[j + M] += round_mod32(v.y);
      }
    }
    fft_inverse<LOGN>(o1, tile, tw1, l);
#pragma unroll
    for (int m1 = 0; m1 < P; ++m1) {
      const double2 v = cmulc(o1[m1], twist[m1 * L + l]);
      const uint32_t j = (uint32_t)(L * m1 + l);
      if (owner) {
        acc_c[j] += round_mod32(v.x) << 16;
        acc_c[j + M] += round_mod32(v.y) << 16;
      }
    }
    __syncwarp();
  }
  uint32_t* dst = a.acc_out + ((size_t)g * 2 + c) * N;
  for (int j = lane; j < N; j += 32) dst[j] = acc_c[j];
}

// Bootstrapping-key pre-transform (reference: cggi.py:283-285, BootstrappingKey
// keeps an NTT-domain copy).  One warp per (i, r, c, h): split the u32 key
// word into balanced 16-bit halves, fold, transform, scale by 1/M, store in
// the native layout.  Same fft_forward as the gate kernel => same ordering.
template <int LOGN, int LEV>
__global__ void __launch_bounds__(128) k_bk_to_fft(const uint32_t* __restrict__ bk_coeff,
                                                   int n, const double2* __restrict__ tables,
                                                   double2* __restrict__ bk_fft) {
  using G = Geo<LOGN>;
  constexpr int N = G::N, M = G::M, P = G::P, L = G::L, R = 2 * LEV;
  __shared__ double2 tw1[2 * G::TILE];
  __shared__ double2 tiles[4][G::TILE];
  double2* twist = tw1 + G::TILE;
  for (int t = threadIdx.x; t < 2 * G::TILE; t += blockDim.x) tw1[t] = tables[t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane & (L - 1);
  const long long job = (long long)blockIdx.x * 4 + warp;  // (((i*R + r)*2 + c)*2 + h)
  if (job >= (long long)n * R * 4) return;
  const int h = (int)(job & 1), c = (int)((job >> 1) & 1);
  const int r = (int)((job >> 2) % R);
  const int i = (int)((job >> 2) / R);
  const uint32_t* poly = bk_coeff + (((size_t)i * R + r) * 2 + c) * N;
  double2 x[P];
#pragma unroll
  for (int m1 = 0; m1 < P; ++m1) {
    int32_t part[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int32_t w = (int32_t)poly[L * m1 + l + hh * M];
      const int32_t lo = (int32_t)(int16_t)(w & 0xFFFF);
      part[hh] = h == 0 ? lo : (int32_t)(((int64_t)w - lo) >> 16);
    }
    x[bitrev_c<G::LOGP>(m1)] = cmul(make_double2((double)part[0], (double)part[1]), twist[m1 * L + l]);
  }
  fft_forward<LOGN>(x, tiles[warp], tw1, l);
  const double scale = 1.0 / (double)M;
#pragma unroll
  for (int s = 0; s < P; ++s)
    bk_fft[bk_index<LOGN, LEV>(i, c, s, r, h, l)] = make_double2(x[s].x * scale, x[s].y * scale);
}

}  // namespace gw
