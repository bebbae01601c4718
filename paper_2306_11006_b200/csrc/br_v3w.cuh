// br_v3w.cuh -- blind rotation v3w: the v3 schedule (br_v3.cuh) with GW gates
// interleaved INSIDE every warp.  Reference: gatewave/cggi.py:592-667.
//
// v3 gives each warp one gate's row / frequency quarter / output and relies
// on several warps per SM sub-partition (one per gate) to hide the latency of
// its FP64 butterfly chains, transposes and TMEM loads.  The phase profile
// (profiles/r01_v3_phase_cycles.txt) shows that does not work well at 1-2
// gates per SM: one warp alone needs 2.8k cycles for a forward phase whose
// FP64 work is < 1k pipe cycles.  Here every compute warp carries GW
// independent gates through the same instruction stream, so the compiler
// interleaves GW independent dependency chains (ILP instead of TLP), and the
// MAC phase reads each bootstrapping-key value from TMEM ONCE for all GW
// gates (v3 reads it once per gate).
//
// CTA = GC groups x 4 compute warps (each warp: GW gates) + 4 key-loader
// warps; one CTA per SM (it owns all 512 TMEM columns); gates per CTA =
// GC * GW.  Per step i, for each gate of the warp's group:
//   F  warp r: rotate-subtract + gadget-decompose acc[r/2], fold + twist,
//      forward head -> U[r];
//   M  warp w: last forward radix-2 stage, 16 key MACs, first inverse stage
//      for the frequency pairs of TMEM sub-partition w;
//   I  warp o: inverse tail, untwist, round, acc[o/2] += v << 16(o%2).
// Data layouts (U slots, key image, TMEM ring, lane twiddles) are v3's.
#pragma once
#include "br_v3.cuh"

namespace gw {

struct V3W {
  // shared memory: per gate U (32 KB), acc (8 KB), digit exchange (4 KB)
  static size_t smem_bytes(int gates) {
    return (size_t)gates * (V3::UB * sizeof(double2) + 2 * V3::N * sizeof(uint32_t) + V3::XCHG * sizeof(uint32_t)) +
           128;
  }
};

// Forward head (fft.cuh fft_forward_head) of GW independent rows at once:
// every stage is issued for all rows before the next, so their chains overlap.
template <int GW>
__device__ __forceinline__ void fwd_head_multi(double2 (&x)[GW][V3::P], double2* const (&tile)[GW], uint32_t tm_tw,
                                               int l) {
  constexpr int P = V3::P, L = V3::L, LOGP = V3::G::LOGP;
#pragma unroll
  for (int j = 0; j < GW; ++j) dit<P, +1>(x[j]);
  // lane twiddles (twist folded in) from TMEM, 4 per load, shared by the GW rows
#pragma unroll
  for (int c = 0; c < P / 4; ++c) {
    uint32_t r[16];
    tm_ld_raw<16>(tm_tw + (uint32_t)(16 * c), r);
    tm_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 w = make_double2(__hiloint2double(r[4 * q + 1], r[4 * q]), __hiloint2double(r[4 * q + 3], r[4 * q + 2]));
#pragma unroll
      for (int j = 0; j < GW; ++j) x[j][4 * c + q] = cmul(x[j][4 * c + q], w);
    }
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < GW; ++j)
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) tile[j][k1 * L + swz(k1, l)] = x[j][k1];
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int j = 0; j < GW; ++j)
#pragma unroll
      for (int a = 0; a < P; ++a) x[j][bitrev_c<LOGP>(a)] = tile[j][k1 * L + swz(k1, b + 2 * a)];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < GW; ++j) dit<P, +1>(x[j]);  // x[c] = u_b[c]
}

// Inverse tail (fft.cuh fft_inverse_tail) of GW independent outputs at once.
template <int GW>
__device__ __forceinline__ void inv_tail_multi(double2 (&x)[GW][V3::P], double2* const (&tile)[GW], uint32_t tm_tw,
                                               int l) {
  constexpr int P = V3::P, L = V3::L, LOGP = V3::G::LOGP;
#pragma unroll
  for (int j = 0; j < GW; ++j) dit<P, -1>(x[j]);
  __syncwarp();
  {
    const int k1 = l >> 1, b = l & 1;
#pragma unroll
    for (int j = 0; j < GW; ++j)
#pragma unroll
      for (int a = 0; a < P; ++a) tile[j][k1 * L + swz(k1, b + 2 * a)] = x[j][a];
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < GW; ++j)
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) x[j][bitrev_c<LOGP>(k1)] = tile[j][k1 * L + swz(k1, l)];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < P / 4; ++c) {
    uint32_t r[16];
    tm_ld_raw<16>(tm_tw + (uint32_t)(16 * c), r);
    tm_wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double2 w = make_double2(__hiloint2double(r[4 * q + 1], r[4 * q]), __hiloint2double(r[4 * q + 3], r[4 * q + 2]));
      const int rr = bitrev_c<LOGP>(4 * c + q);
#pragma unroll
      for (int j = 0; j < GW; ++j) x[j][rr] = cmulc(x[j][rr], w);
    }
  }
#pragma unroll
  for (int j = 0; j < GW; ++j) dit<P, -1>(x[j]);  // x[m1]
}

#ifndef GW_V3W_LREG
#define GW_V3W_LREG 64
#endif

template <int GW, int GC, bool PROBE = false>
__global__ void __launch_bounds__(128 * GC + 128, 1) k_blind_rotate_v3w(BrArgs a) {
  constexpr int N = V3::N, M = V3::M, P = V3::P, L = V3::L, R = V3::R, LEV = V3::LEV, LOGN = V3::LOGN;
  constexpr int UB = V3::UB, CIDX = V3::CIDX;
  using G = V3::G;
  constexpr int NG = GW * GC;  // gates per CTA
  // register split (setmaxnreg): loaders LREG, compute warps what is left of the launch's pool
  constexpr int LREG = GW_V3W_LREG;
  constexpr int kPool = ((65536 / (128 * GC + 128)) & ~7) * (128 * GC + 128);
  constexpr int CREG0 = ((kPool - LREG * 128) / (128 * GC)) & ~7;
  constexpr int CREG = CREG0 > 248 ? 248 : CREG0;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double2* ubuf_all = reinterpret_cast<double2*>(smem_raw);                 // NG x UB
  uint32_t* acc_all = reinterpret_cast<uint32_t*>(ubuf_all + (size_t)NG * UB);  // NG x 2N
  uint32_t* xchg_all = acc_all + (size_t)NG * 2 * N;                          // NG x XCHG
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg_all + (size_t)NG * V3::XCHG);
  uint64_t* full_bar = bars;       // [2] loaders stored slab i into the ring
  uint64_t* empty_bar = bars + 2;  // [2] every compute warp finished MAC(i)
  uint64_t* go_bar = bars + 4;     // group 1 may start (stagger, GC = 2)
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(bars + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane;
  const int gl = warp >> 2, o = warp & 3;
  const bool loader = warp >= 4 * GC;

  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&full_bar[k], 4);
      mbar_init(&empty_bar[k], 4 * GC);
    }
    mbar_init(go_bar, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(tm_slot, 512);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm_base = *tm_slot;
  const uint32_t tm_warp = tm_base + ((uint32_t)(32 * o) << 16);
  const uint32_t tm_tw = tm_warp + (uint32_t)V3::TWCOL;
  if (!loader && gl == 0) {
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) tm_st4(tm_tw + (uint32_t)(4 * k1), __ldg(a.tables + 2 * G::TILE + k1 * L + l));
    tm_wait_st();
  }
  // key chunk q of step i lives in ring slot (4 i + q) mod 7
  auto kcol = [&](int slot_i, int q) -> uint32_t {
    const int sl = slot_i + q;
    return (uint32_t)((sl >= V3::RING ? sl - V3::RING : sl) * V3::CHUNK);
  };

  const uint32_t two_n_mask = 2 * N - 1;
  const uint32_t rshift = 32 - (LOGN + 1);
  const uint32_t radd = 1u << (32 - (LOGN + 1) - 1);
  const uint32_t base_mask = (1u << a.bg_bits) - 1;
  const int32_t half_base = 1 << (a.bg_bits - 1);
  const double dmagic = 6755399441055744.0 + (double)half_base;

  // this warp's gates: g = (blockIdx.x * GC + gl) * GW + j; inactive slots run
  // on row 0 and discard their results (the barrier protocol never depends on B)
  const uint32_t* lin_g[GW];
  bool active[GW];
  uint32_t* acc_g[GW];
  double2* U[GW];
  uint32_t* xg_g[GW];
#pragma unroll
  for (int j = 0; j < GW; ++j) {
    const int g = (blockIdx.x * GC + gl) * GW + j;
    active[j] = g < a.B;
    lin_g[j] = a.lin + (size_t)(active[j] ? g : 0) * a.lin_stride;
    const int s = gl * GW + j;  // gate slot in this CTA
    acc_g[j] = acc_all + (size_t)s * 2 * N;
    U[j] = ubuf_all + (size_t)s * UB;
    xg_g[j] = xchg_all + (size_t)s * V3::XCHG;
  }
  // acc <- tv * X^{-bbar} (cggi.py:612-622): warp o < 2 initialises component o
  if (!loader && o < 2) {
#pragma unroll
    for (int j = 0; j < GW; ++j) {
      const uint32_t bbar = ((lin_g[j][a.n] + radd) >> rshift) & two_n_mask;
      const uint32_t k = (2 * N - bbar) & two_n_mask;
      const uint32_t* tvc = a.tv + o * N;
      for (int jj = lane; jj < N; jj += 32) {
        const uint32_t m = ((uint32_t)jj - k) & two_n_mask;
        acc_g[j][o * N + jj] = m < (uint32_t)N ? tvc[m] : 0u - tvc[m - N];
      }
    }
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();

  if (loader) {
    // ---- loader warp: slab i -> ring slots of sub-partition o, ahead of the MAC ----
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(LREG));
    constexpr int RS = 16;  // 16-byte loads in flight per round (divides 48)
    const double2* src_w = a.bk + (size_t)32 * o + lane;
    int s_i = 0;
    for (int i = 0; i < a.n; ++i) {
      const double2* src = src_w + (size_t)i * CIDX * 128;
      if (o == 0 && lane == 0 && i + 2 < a.n) {  // L2 prefetch of the slab two steps ahead
        const char* pf = reinterpret_cast<const char*>(a.bk + (size_t)(i + 2) * CIDX * 128);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(V3::SLAB) : "memory");
      }
      if (i >= 2) {  // chunks 0-2 reuse the slots of slab i-2's chunks 1-3
        mbar_wait(&empty_bar[i & 1], (uint32_t)(((i - 2) >> 1) & 1));
        tm_fence_after();
      }
#pragma unroll 1
      for (int rnd = 0; rnd < 48 / RS; ++rnd) {
        double2 v[RS];
#pragma unroll
        for (int k = 0; k < RS; ++k) v[k] = ldg_stream(src + (size_t)(rnd * RS + k) * 128);
#pragma unroll
        for (int k = 0; k < RS; ++k) {
          const int cidx = rnd * RS + k;
          tm_st4(tm_warp + kcol(s_i, cidx >> 4) + (uint32_t)((cidx & 15) * 4), v[k]);
        }
      }
      if (i >= 1) {  // chunk 3 reuses the slot of slab i-1's chunk 0
        mbar_wait(&empty_bar[(i - 1) & 1], (uint32_t)(((i - 1) >> 1) & 1));
        tm_fence_after();
      }
      {
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = ldg_stream(src + (size_t)(48 + k) * 128);
#pragma unroll
        for (int k = 0; k < 16; ++k) tm_st4(tm_warp + kcol(s_i, 3) + (uint32_t)(k * 4), v[k]);
      }
      tm_wait_st();
      tm_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[i & 1]);
      s_i = s_i + 4 >= V3::RING ? s_i + 4 - V3::RING : s_i + 4;
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CREG));
    if (GC == 2 && gl == 1) mbar_wait(go_bar, 0);  // group 1 starts after group 0's F(0)
    const int mk1 = lane & 15;
    const int mc0 = 4 * o + 2 * (lane >> 4);
    const int pos = v3_pos(l);
    const int bar_id = 1 + gl;
    int sc = 0;
    uint32_t a_next[GW];
#pragma unroll
    for (int j = 0; j < GW; ++j) a_next[j] = __ldg(lin_g[j]);
    double worst = 0.0;
    double2* tiles[GW];
#pragma unroll
    for (int j = 0; j < GW; ++j) tiles[j] = U[j] + (size_t)o * P * L;

    for (int i = 0; i < a.n; ++i) {
      const int cur = i & 1;
      const int sn = sc + 4 >= V3::RING ? sc + 4 - V3::RING : sc + 4;
      uint32_t a_i[GW];
#pragma unroll
      for (int j = 0; j < GW; ++j) {
        a_i[j] = a_next[j];
        if (i + 1 < a.n) a_next[j] = __ldg(lin_g[j] + i + 1);
      }
      // ---------------- F: row r = o of every gate ----------------
      {
        const int cr = o / LEV, lv = o % LEV;
        const int sh_mine = 32 - (lv + 1) * a.bg_bits, sh_other = 32 - (2 - lv) * a.bg_bits;
        double2 x[GW][P];
        uint32_t mine[GW][P];
        // the two level-warps of component cr split the coefficients by half
        // (warp lv takes j + lv*M), extract BOTH levels and swap the other's digits
#pragma unroll
        for (int j = 0; j < GW; ++j) {
          const uint32_t* A = acc_g[j] + cr * N;
          const uint32_t abar = ((a_i[j] + radd) >> rshift) & two_n_mask;
          const uint32_t idxh = (((uint32_t)l - abar) & two_n_mask) + (uint32_t)(lv * M);
          uint32_t* to_partner = xg_g[j] + (size_t)cr * 2 * (P / 2) * 32 + (size_t)(1 - lv) * (P / 2) * 32;
#pragma unroll
          for (int m1 = 0; m1 < P; m1 += 2) {
            uint32_t oth[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t idx = (idxh + (uint32_t)(L * (m1 + q))) & two_n_mask;
              const uint32_t v = A[idx & (N - 1)];
              const uint32_t neg = 0u - ((idx >> LOGN) & 1u);
              const uint32_t buf = ((v ^ neg) - neg) - A[L * (m1 + q) + l + lv * M] + a.offs;
              mine[j][m1 + q] = (buf >> sh_mine) & base_mask;
              oth[q] = (buf >> sh_other) & base_mask;
            }
            to_partner[(m1 / 2) * 32 + lane] = oth[0] | (oth[1] << 16);
          }
        }
        named_barrier(5 + 2 * gl + cr, 64);
#pragma unroll
        for (int j = 0; j < GW; ++j) {
          const uint32_t* from_partner = xg_g[j] + (size_t)cr * 2 * (P / 2) * 32 + (size_t)lv * (P / 2) * 32;
#pragma unroll
          for (int m1 = 0; m1 < P; m1 += 2) {
            const uint32_t w = from_partner[(m1 / 2) * 32 + lane];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t rv = q ? (w >> 16) : (w & 0xFFFFu);
              const uint32_t re = lv ? rv : mine[j][m1 + q], im = lv ? mine[j][m1 + q] : rv;
              double2 v = make_double2(digit_to_double_lo(re, dmagic), digit_to_double_lo(im, dmagic));
              if (m1 + q > 0) v = cmul(v, c_root64[G::CSTEP * (m1 + q)]);
              x[j][bitrev_c<G::LOGP>(m1 + q)] = v;
            }
          }
        }
        fwd_head_multi<GW>(x, tiles, tm_tw, l);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < GW; ++j)
#pragma unroll
          for (int c = 0; c < P; ++c) tiles[j][c * L + pos] = x[j][c];
      }
      if (GC == 2 && i == 0 && gl == 0 && lane == 0) mbar_arrive(go_bar);
      named_barrier(bar_id, 128);  // U complete
      // ---------------- M: frequency pairs (mk1, mc0 + p) of all rows ----------------
      mbar_wait(&full_bar[cur], (uint32_t)((i >> 1) & 1));
      tm_fence_after();
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int c = mc0 + p;
        const double2 tw = c_root64[2 * c];  // e^{2 pi i c / 32}
        double2 D[GW][R][2];
#pragma unroll
        for (int j = 0; j < GW; ++j)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double2* row = U[j] + ((size_t)r * P + c) * L;
            const double2 u0 = row[v3_slot(mk1, 0)], u1 = row[v3_slot(mk1, 1)];
            const double2 t = cmul(u1, tw);
            D[j][r][0] = cadd(u0, t);
            D[j][r][1] = csub(u0, t);
          }
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // outputs 2hf, 2hf+1
          double2 O[GW][2][2];            // [gate][output of the pair][s]
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            uint32_t kw[32];  // 2 outputs x 4 rows of frequency (p, s): read ONCE for all GW gates
            tm_ld_raw<32>(tm_warp + kcol(sc, 2 * p + s) + (uint32_t)(hf * 32), kw);
            tm_wait_ld();
#pragma unroll
            for (int oi = 0; oi < 2; ++oi)
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const uint32_t* k4 = kw + (oi * 4 + r) * 4;
                const double2 kr = make_double2(__hiloint2double(k4[1], k4[0]), __hiloint2double(k4[3], k4[2]));
#pragma unroll
                for (int j = 0; j < GW; ++j)
                  O[j][oi][s] = r == 0 ? cmul(D[j][r][s], kr) : cfma(O[j][oi][s], D[j][r][s], kr);
              }
          }
#pragma unroll
          for (int j = 0; j < GW; ++j)
#pragma unroll
            for (int oi = 0; oi < 2; ++oi) {
              double2* row = U[j] + ((size_t)(2 * hf + oi) * P + c) * L;
              row[v3_slot(mk1, 0)] = cadd(O[j][oi][0], O[j][oi][1]);
              row[v3_slot(mk1, 1)] = cmulc(csub(O[j][oi][0], O[j][oi][1]), tw);
            }
        }
      }
      tm_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[cur]);
      named_barrier(bar_id, 128);  // V complete
      // ---------------- I: output o = (component o/2, half o%2) of every gate ----------------
      {
        double2 x[GW][P];
#pragma unroll
        for (int j = 0; j < GW; ++j)
#pragma unroll
          for (int c = 0; c < P; ++c) x[j][bitrev_c<G::LOGP>(c)] = tiles[j][c * L + pos];
        inv_tail_multi<GW>(x, tiles, tm_tw, l);
        const int shift = 16 * (o & 1);
#pragma unroll
        for (int j = 0; j < GW; ++j) {
          uint32_t* Ac = acc_g[j] + (o >> 1) * N;
#pragma unroll
          for (int m1 = 0; m1 < P; ++m1) {
            const double2 v = m1 == 0 ? x[j][0] : cmulc(x[j][m1], c_root64[G::CSTEP * m1]);
            const uint32_t jj = (uint32_t)(L * m1 + l);
            if constexpr (PROBE) worst = fmax(worst, fmax(fabs(v.x - rint(v.x)), fabs(v.y - rint(v.y))));
            atomicAdd(Ac + jj, round_mod32(v.x) << shift);
            atomicAdd(Ac + jj + M, round_mod32(v.y) << shift);
          }
        }
      }
      named_barrier(bar_id, 128);  // acc updated before the next decomposition
      sc = sn;
    }
    if constexpr (PROBE) {
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, d));
      if (lane == 0 && a.margin) atomicMax(a.margin, (unsigned long long)__double_as_longlong(worst));
    }
    if (o < 2) {
#pragma unroll
      for (int j = 0; j < GW; ++j) {
        if (!active[j]) continue;
        const int g = (blockIdx.x * GC + gl) * GW + j;
        uint32_t* dst = a.acc_out + ((size_t)g * 2 + o) * N;
        for (int jj = lane; jj < N; jj += 32) dst[jj] = acc_g[j][o * N + jj];
      }
    }
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(tm_base, 512);
}

}  // namespace gw
