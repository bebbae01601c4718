// gw_common.cuh -- shared device helpers for the B200 CGGI engine.
//
// Arithmetic convention: the negacyclic external product of the
// blind rotation is computed EXACTLY with an FP64 FFT.  Bootstrapping-key
// words are split into balanced 16-bit halves, so every convolution
// coefficient is an integer of magnitude <= 2l*N*2^(Bg-1)*2^15 (2^35 at the
// reference's parameters); the FP64 rounding error of the whole
// transform/MAC/inverse chain is < 1e-3 there, so rounding to the nearest
// integer reproduces the reference's Goldilocks-NTT result bit for bit.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gw {

// A bootstrap's input: lin = w0*row(s0) + w1*row(s1) + cmu*mu on the body word
// (cggi.py:816-830, the per-kind combination).  k_lin materialises it; the v3
// blind rotation computes it on the fly from the operand rows.
struct LinJob {
  int32_t src[2];
  int32_t w[2];
  int32_t cmu;
  int32_t pad;
};

// e^{2 pi i t / 64}, t in [0, 64): every root of unity the in-register DFTs
// use (sizes divide 64).  Filled from the host with correctly rounded values.
__constant__ double2 c_root64[64];
// Tangent-form twiddles for 6-op butterflies: for t with |cos| >= |sin|
// (t mod 32 in [0,8] or [24,32)) (cos, tan) of 2 pi t / 64, else (sin, cot).
__constant__ double2 c_ts64[64];

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
// a * b
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// acc + a * b
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}

// Exact small-int -> double without the (slow) I2F.F64 conversion:
// 1.5*2^52 + d has ulp 1, so reinterpreting and subtracting is exact.
__device__ __forceinline__ double small_int_to_double(int32_t d) {
  return __longlong_as_double(0x4338000000000000LL + (long long)d) - 6755399441055744.0;
}
// (double)((int)u - half) for small u, half: the offset folds into the magic constant.
__device__ __forceinline__ double digit_to_double(uint32_t u, int32_t half) {
  return __longlong_as_double((long long)(0x4338000000000000LL - half) + (long long)u) - 6755399441055744.0;
}
// Same value without 64-bit integer arithmetic: hi word 0x43380000, lo word u
// is exactly 1.5*2^52 + u; subtracting the (exact) constant 1.5*2^52 + half.
__device__ __forceinline__ double digit_to_double_lo(uint32_t u, double magic_plus_half) {
  return __hiloint2double(0x43380000, (int)u) - magic_plus_half;
}
// x * i^b for a lane-dependent bit b (integer sign flip + selects, no FP op).
__device__ __forceinline__ double2 mul_i_if(double2 t, bool b) {
  const double nty = __longlong_as_double(__double_as_longlong(t.y) ^ (long long)0x8000000000000000ULL);
  return make_double2(b ? nty : t.x, b ? t.x : t.y);
}
// x * (-i)^b
__device__ __forceinline__ double2 mul_mi_if(double2 t, bool b) {
  const double ntx = __longlong_as_double(__double_as_longlong(t.x) ^ (long long)0x8000000000000000ULL);
  return make_double2(b ? t.y : t.x, b ? ntx : t.y);
}
// Round-to-nearest integer of |x| < 2^51, returned mod 2^32.
__device__ __forceinline__ uint32_t round_mod32(double x) {
  return (uint32_t)__double_as_longlong(__dadd_rn(x, 6755399441055744.0));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void named_barrier(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double2 shfl_xor_c(double2 v, int m) {
  double2 r;
  r.x = __shfl_xor_sync(0xffffffffu, v.x, m);
  r.y = __shfl_xor_sync(0xffffffffu, v.y, m);
  return r;
}

__device__ __forceinline__ double2 sel_c(bool p, double2 a, double2 b) {
  return p ? a : b;
}

}  // namespace gw
