// fft.cuh -- warp-level negacyclic FP64 FFT for the blind rotation.
//
// A real polynomial a(X) mod X^N + 1 is folded into M = N/2 complex points
//   z[m] = (a[m] + i a[m+M]) * e^{i pi m / N}
// whose length-M DFT (kernel e^{+2 pi i / M}) evaluates a at the N/2 roots
// e^{i pi (4k+1)/N}; the other N/2 roots are their conjugates (SURVEY.md
// Appendix B).  One warp owns one transform:
//   M = P * L with L = 2P lanes, P complex values per lane,
//   F1  in-register DIF DFT-P over m1 (input z[L*m1 + lane])
//   tw  lane twiddle e^{2 pi i lane k1 / M}
//   T   shared-memory transpose (XOR-swizzled, conflict-free 16-byte accesses)
//   F2  in-register DIF DFT-P
//   F3  radix-2 across lane pairs with half the values exchanged by shuffle.
// The forward output stays in this "native" per-lane order; the bootstrapping
// key is stored in the same order, and the inverse is the exact mirror, so no
// bit-reversal permutation is ever materialised.  tools/fft_model.py replays
// these index maps in numpy.
#pragma once
#include "gw_common.cuh"
#ifndef GW_ABL
#define GW_ABL 0  // timing-only ablations (tools): 1 decomposition, 2 transposes, 4 MAC, 8 atomics
#endif

namespace gw {

template <int LOGN>
struct Geo {
  static constexpr int N = 1 << LOGN;
  static constexpr int M = N / 2;
  static constexpr int LOGP = (LOGN - 2) / 2;  // M = 2 P^2
  static constexpr int P = 1 << LOGP;
  static constexpr int L = 2 * P;
  static_assert(2 * P * P == M, "ring dimension must be 4^k * 4 (64, 256, 1024)");
  static_assert(L <= 32, "one warp per transform");
  // smem elements (double2) of one P x L tile
  static constexpr int TILE = P * L;
  // e^{i pi L m1 / N} = c_root64[CSTEP * m1]: lane-independent part of the twist
  static constexpr int CSTEP = 32 * L / N;
};

template <int LOGP>
__device__ __forceinline__ constexpr int bitrev_c(int x) {
  int r = 0;
#pragma unroll
  for (int k = 0; k < LOGP; ++k) r |= ((x >> k) & 1) << (LOGP - 1 - k);
  return r;
}

// multiply by e^{SIGN * 2 pi i t / 64}
template <int SIGN>
__device__ __forceinline__ double2 rot64(double2 v, int t) {
  if (t == 0) return v;
  if (t == 16) return SIGN > 0 ? make_double2(-v.y, v.x) : make_double2(v.y, -v.x);
  const double2 w = c_root64[t];
  return SIGN > 0 ? cmul(v, w) : cmulc(v, w);
}

// One radix-2 stage of span LEN (compile-time, so every register index folds).
template <int P, int SIGN, int LEN>
__device__ __forceinline__ void dif_stage(double2 (&x)[P]) {
  constexpr int h = LEN / 2;
#pragma unroll
  for (int st = 0; st < P; st += LEN) {
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const double2 a = x[st + j], b = x[st + j + h];
      x[st + j] = cadd(a, b);
      x[st + j + h] = rot64<SIGN>(csub(a, b), j * (64 / LEN));
    }
  }
}

// DIT butterfly (a, b) <- (a + w b, a - w b), w = e^{SIGN 2 pi i t / 64}.
// Non-trivial twiddles use the tangent form w = s (1 + i r) (or s (r + i)),
// |r| <= 1: 6 FP64 ops instead of 8 (complex multiply + two complex adds).
template <int SIGN>
__device__ __forceinline__ void bfly(double2& a, double2& b, int t) {
  if (t == 0) {
    const double2 s = cadd(a, b), d = csub(a, b);
    a = s;
    b = d;
    return;
  }
  if (t == 16) {  // w = SIGN * i
    const double2 wb = SIGN > 0 ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
    const double2 s = cadd(a, wb), d = csub(a, wb);
    a = s;
    b = d;
    return;
  }
  const double2 cs = c_ts64[t];
  const bool case_a = (t % 32) <= 8 || (t % 32) >= 24;
  const double scale = (SIGN > 0 || case_a) ? cs.x : -cs.x;
  const double ratio = SIGN > 0 ? cs.y : -cs.y;
  double u, v;
  if (case_a) {
    u = fma(-ratio, b.y, b.x);
    v = fma(ratio, b.x, b.y);
  } else {
    u = fma(ratio, b.x, -b.y);
    v = fma(ratio, b.y, b.x);
  }
  const double2 s = make_double2(fma(scale, u, a.x), fma(scale, v, a.y));
  const double2 d = make_double2(fma(-scale, u, a.x), fma(-scale, v, a.y));
  a = s;
  b = d;
}

template <int P, int SIGN, int LEN>
__device__ __forceinline__ void dit_stage(double2 (&x)[P]) {
  constexpr int h = LEN / 2;
#pragma unroll
  for (int st = 0; st < P; st += LEN) {
#pragma unroll
    for (int j = 0; j < h; ++j) bfly<SIGN>(x[st + j], x[st + j + h], j * (64 / LEN));
  }
}

// Radix-2 DIF, natural order in, bit-reversed order out, kernel e^{SIGN 2 pi i / P}.
template <int P, int SIGN, int LEN = P>
__device__ __forceinline__ void dif(double2 (&x)[P]) {
  if constexpr (LEN >= 2) {
    dif_stage<P, SIGN, LEN>(x);
    dif<P, SIGN, LEN / 2>(x);
  }
}

// Radix-2 DIT, bit-reversed order in, natural order out, kernel e^{SIGN 2 pi i / P}.
template <int P, int SIGN, int LEN = 2>
__device__ __forceinline__ void dit(double2 (&x)[P]) {
  if constexpr (LEN <= P) {
    dit_stage<P, SIGN, LEN>(x);
    dit<P, SIGN, LEN * 2>(x);
  }
}

// Column of the transpose tile holding (row k1, logical column col).
__device__ __forceinline__ int swz(int k1, int col) { return col ^ ((k1 & 3) << 1); }

// Forward transform.  In: x[bitrev(m1)] = z[L*m1 + l] (l = lane & (L-1)).
// Out: x[s] = Z[k(l, s)], k = k1 + P*(c + P*d), k1 = l>>1, b = l&1,
//      c = b*P/2 + s%(P/2), d = s/(P/2).
// tw1: smem [k1][l] = e^{2 pi i l k1 / M}.  tile: smem scratch of Geo::TILE.
// TW0 = true: tw1 also carries the per-lane twist e^{i pi l / N} (then tw1[0][l]
// is not 1 and the caller multiplies by the lane-independent e^{i pi L m1 / N}).
// Lane-twiddle sources: a shared-memory table [k1][lane] or a register copy.
struct TwSmem {
  const double2* t;
  int L, l;
  __device__ __forceinline__ double2 operator()(int k1) const { return t[k1 * L + l]; }
};
template <int P>
struct TwRegs {
  const double2 (&r)[P];
  __device__ __forceinline__ double2 operator()(int k1) const { return r[k1]; }
};

template <int LOGN, bool TW0 = false, class TW>
__device__ __forceinline__ void fft_forward_tw(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l);
template <int LOGN, bool TW0 = false, class TW>
__device__ __forceinline__ void fft_inverse_tw(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l);

template <int LOGN, bool TW0 = false>
__device__ __forceinline__ void fft_forward(double2 (&x)[Geo<LOGN>::P], double2* tile,
                                            const double2* tw1, int l) {
  fft_forward_tw<LOGN, TW0>(x, tile, TwSmem{tw1, Geo<LOGN>::L, l}, l);
}
template <int LOGN, bool TW0 = false>
__device__ __forceinline__ void fft_inverse(double2 (&x)[Geo<LOGN>::P], double2* tile,
                                            const double2* tw1, int l) {
  fft_inverse_tw<LOGN, TW0>(x, tile, TwSmem{tw1, Geo<LOGN>::L, l}, l);
}

template <int LOGN, bool TW0, class TW>
__device__ __forceinline__ void fft_forward_tw(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l) {
  using G = Geo<LOGN>;
  constexpr int P = G::P, L = G::L, LOGP = G::LOGP;
  // Input in BIT-REVERSED register order: x[bitrev(m1)] = z[L*m1 + l].
  dit<P, +1>(x);  // x[k1] natural
#pragma unroll
  for (int k1 = TW0 ? 0 : 1; k1 < P; ++k1) x[k1] = cmul(x[k1], tw(k1));
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) tile[k1 * L + swz(k1, l)] = x[k1];
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int a = 0; a < P; ++a) x[bitrev_c<LOGP>(a)] = tile[k1 * L + swz(k1, b + 2 * a)];
  }
  __syncwarp();
  dit<P, +1>(x);  // x[c] = u_b[c], natural
  const bool hi = (l & 1) != 0;
  double2 y[P];
#pragma unroll
  for (int j = 0; j < P / 2; ++j) {
    const double2 ulo = x[j];
    const double2 uhi = x[j + P / 2];
    const double2 recv = shfl_xor_c(hi ? ulo : uhi, 1);
    double2 u0 = hi ? recv : ulo;
    // w^c with w = e^{2 pi i / 2P}, c = j + b*P/2: w^c = w^j * i^b (w^j lane-uniform)
    double2 u1 = mul_i_if(hi ? uhi : recv, hi);
    bfly<+1>(u0, u1, (32 / P) * j);
    y[j] = u0;
    y[j + P / 2] = u1;
  }
#pragma unroll
  for (int s = 0; s < P; ++s) x[s] = y[s];
}

// Inverse transform, exact mirror of fft_forward, scaled by M (no division):
// In: native layout.  Out: x[m1] = M * z[L*m1 + l].
template <int LOGN, bool TW0, class TW>
__device__ __forceinline__ void fft_inverse_tw(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l) {
  using G = Geo<LOGN>;
  constexpr int P = G::P, L = G::L, LOGP = G::LOGP;
  const bool hi = (l & 1) != 0;
  double2 u[P];
#pragma unroll
  for (int j = 0; j < P / 2; ++j) {
    const double2 X0 = x[j], X1 = x[j + P / 2];
    const double2 S = cadd(X0, X1);
    const double2 D = mul_mi_if(rot64<-1>(csub(X0, X1), (32 / P) * j), hi);
    const double2 recv = shfl_xor_c(hi ? S : D, 1);
    u[bitrev_c<LOGP>(j)] = hi ? recv : S;
    u[bitrev_c<LOGP>(j + P / 2)] = hi ? D : recv;
  }
  dit<P, -1>(u);  // u[a]
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int a = 0; a < P; ++a) tile[k1 * L + swz(k1, b + 2 * a)] = u[a];
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) x[bitrev_c<LOGP>(k1)] = tile[k1 * L + swz(k1, l)];
  __syncwarp();
#pragma unroll
  for (int k1 = TW0 ? 0 : 1; k1 < P; ++k1) {
    const int r = bitrev_c<LOGP>(k1);
    x[r] = cmulc(x[r], tw(k1));
  }
  dit<P, -1>(x);  // x[m1]
}

// ---- split transforms for the frequency-partitioned MAC (br_v3.cuh) --------
// The radix-2 stage across lane pairs (F3 above) is not done in registers:
// the forward "head" stops after F2 with x[c] = u_b[c] (lane l = 2*k1 + b),
// and the MAC phase, which gathers the values of all rows through shared
// memory anyway, applies  D(+/-) = u_0[c] +/- w^c u_1[c]  (w = e^{2 pi i/2P})
// for the (k1, c) pairs it owns.  The inverse "tail" starts from
// u[bitrev(c)] = u_b[c] (b = 0: O+ + O-, b = 1: (O+ - O-) conj(w^c)).
// No shuffles and no lane-parity selects remain in the transforms.
template <int LOGN, bool TW0, class TW>
__device__ __forceinline__ void fft_forward_head(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l) {
  using G = Geo<LOGN>;
  constexpr int P = G::P, L = G::L, LOGP = G::LOGP;
  dit<P, +1>(x);
#pragma unroll
  for (int k1 = TW0 ? 0 : 1; k1 < P; ++k1) x[k1] = cmul(x[k1], tw(k1));
#if !(GW_ABL & 2)
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) tile[k1 * L + swz(k1, l)] = x[k1];
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int a = 0; a < P; ++a) x[bitrev_c<LOGP>(a)] = tile[k1 * L + swz(k1, b + 2 * a)];
  }
  __syncwarp();
#endif
  dit<P, +1>(x);  // x[c] = u_b[c]
}

// In: x[bitrev(c)] = u_b[c].  Out: x[m1] = M * z[L*m1 + l] (in place).
template <int LOGN, bool TW0, class TW>
__device__ __forceinline__ void fft_inverse_tail(double2 (&x)[Geo<LOGN>::P], double2* tile, const TW& tw, int l) {
  using G = Geo<LOGN>;
  constexpr int P = G::P, L = G::L, LOGP = G::LOGP;
  dit<P, -1>(x);  // x[a]
#if !(GW_ABL & 2)
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int a = 0; a < P; ++a) tile[k1 * L + swz(k1, b + 2 * a)] = x[a];
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < P; ++k1) x[bitrev_c<LOGP>(k1)] = tile[k1 * L + swz(k1, l)];
  __syncwarp();
#endif
#pragma unroll
  for (int k1 = TW0 ? 0 : 1; k1 < P; ++k1) {
    const int r = bitrev_c<LOGP>(k1);
    x[r] = cmulc(x[r], tw(k1));
  }
  dit<P, -1>(x);  // x[m1]
}

}  // namespace gw
