// br_tmem.cuh -- blind rotation v2: 4 warps per gate, bootstrapping key
// double-buffered in Tensor Memory (reference: gatewave/cggi.py:592-667).
//
// CTA = GC gates x 4 warps.  Warp o (= its TMEM sub-partition) of a gate
//   * forward: row r = o of the 2l gadget-digit rows (cggi.py:627-647):
//     rotate-subtract + decompose acc[c_r] (smem), fold, FFT, D^_r -> smem;
//   * MAC (cggi.py:648-657): output o = (c, h): sum_r D^_r * BK_i[c][h][r]
//     with the key slab read from TMEM (tcgen05.ld), D^ from smem;
//   * inverse + round + acc[c] += v << 16h (cggi.py:658-666, smem atomics:
//     wrap-around adds commute, so the result is exact for any order).
// The key slab of step i+1 (one 32 KB (c,h) slice per sub-partition, 128 KB
// total) is streamed from L2 into the other TMEM buffer in four batches
// issued at the phase boundaries of step i, so its latency hides behind the
// FFTs; the GC warps of a sub-partition split the slice.
#pragma once
#include "blind_rotate.cuh"
#include "mbarrier.cuh"
#include "tmem.cuh"

namespace gw {

template <int LOGN, int LEV>
struct TmGeo {
  using G = Geo<LOGN>;
  static constexpr int R = 2 * LEV;
  static constexpr int COLS = G::P * R * 4;  // one buffer: [row][slot] complex (4 cols each)
  static constexpr int ALLOC = (2 * COLS) <= 32 ? 32 : (2 * COLS) <= 64 ? 64 : (2 * COLS) <= 128 ? 128
                               : (2 * COLS) <= 256 ? 256 : 512;
  static_assert(2 * COLS <= 512, "two key slabs must fit the 512 TMEM columns");
  // digit exchange between the two level-warps of one accumulator component
  static constexpr int XCHG = LEV == 2 ? 2 * 2 * (G::P / 2) * 32 : 0;  // u32 per gate
  static size_t smem_bytes(int gc, int n) {
    const size_t lin_words = ((size_t)n + 1 + 3) & ~(size_t)3;
    return 64 /*tmem slot + mbarriers*/ + sizeof(double2) * G::TILE /*tw1'*/ +
           (size_t)gc * (sizeof(double2) * R * G::TILE + 2 * G::N * sizeof(uint32_t) +
                         lin_words * sizeof(uint32_t) + XCHG * sizeof(uint32_t));
  }
};

template <int LOGN, int LEV, int GC>
__global__ void __launch_bounds__(128 * GC, 1) k_blind_rotate_tm(BrArgs a) {
  using G = Geo<LOGN>;
  using T = TmGeo<LOGN, LEV>;
  constexpr int N = G::N, M = G::M, P = G::P, L = G::L, R = T::R, COLS = T::COLS;
  // fill items per warp per step: its share of one (c,h) slice, streamed in
  // three groups (issued at a phase boundary, stored at the next one)
  constexpr int ITEMS = P * R / GC;        // complex values per lane
  constexpr int GS = (ITEMS + 2) / 3;      // items per group (register buffer)

  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(smem_raw);
  // key-slab buffer protocol: full[b] = all warps stored their share of the slab
  // in TMEM buffer b; empty[b] = all warps finished reading buffer b (MAC)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_raw + 8);
  uint64_t* empty_bar = full_bar + 2;
  uint64_t* go_bar = full_bar + 4;
  double2* tw1 = reinterpret_cast<double2*>(smem_raw + 64);
  double2* xbuf_all = tw1 + G::TILE;
  uint32_t* acc_all = reinterpret_cast<uint32_t*>(xbuf_all + (size_t)GC * R * G::TILE);
  const size_t lin_words = ((size_t)a.n + 1 + 3) & ~(size_t)3;
  uint32_t* lin_all = acc_all + (size_t)GC * 2 * N;
  uint32_t* xchg_all = lin_all + (size_t)GC * lin_words;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane & (L - 1);
  const int gl = warp >> 2, o = warp & 3;
  const int co = o >> 1, ho = o & 1;
  const int g = blockIdx.x * GC + gl;
  const bool active = g < a.B;

  for (int t = threadIdx.x; t < G::TILE; t += blockDim.x) tw1[t] = a.tables[2 * G::TILE + t];
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&full_bar[k], 4 * GC);
      mbar_init(&empty_bar[k], 4 * GC);
    }
    mbar_init(go_bar, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(tm_slot, T::ALLOC);

  uint32_t* lin_s = lin_all + (size_t)gl * lin_words;
  uint32_t* acc_g = acc_all + (size_t)gl * 2 * N;
  double2* xb = xbuf_all + (size_t)gl * R * G::TILE;  // [row][slot][lane]
  if (active) {
    const uint32_t* src = a.lin + (size_t)g * a.lin_stride;
    for (int t = o * 32 + lane; t <= a.n; t += 128) lin_s[t] = src[t];
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm_base = *tm_slot;
  const uint32_t tm_warp = tm_base + ((uint32_t)(32 * o) << 16);

  const uint32_t two_n_mask = 2 * N - 1;
  const uint32_t rshift = 32 - (LOGN + 1);
  const uint32_t radd = 1u << (32 - (LOGN + 1) - 1);
  const uint32_t base_mask = (1u << a.bg_bits) - 1;
  const int32_t half_base = 1 << (a.bg_bits - 1);

  // ---- key-slab streaming into TMEM ----------------------------------------
  // item t of this warp: slot s = (t / R) * GC + gl, row r = t % R.  Offsets
  // from the warp's (slot gl, row 0) base are compile-time constants.
  const size_t step_stride = (size_t)2 * 2 * P * R * L;  // complex per LWE index i
  const double2* fill_w = a.bk + bk_index<LOGN, LEV>(0, co, gl, 0, ho, l);
  const uint32_t col_w = tm_warp + (uint32_t)(gl * 4);  // slot gl of row 0
  double2 fb[GS];  // one group in flight
  auto issue = [&](int i, int grp) {
    const double2* src = fill_w + (size_t)i * step_stride;
#pragma unroll
    for (int k = 0; k < GS; ++k) {
      const int t = grp * GS + k;
      if (t < ITEMS) fb[k] = __ldg(src + ((t / R) * GC * R + t % R) * L);
    }
  };
  auto store = [&](int buf, int grp) {
#pragma unroll
    for (int k = 0; k < GS; ++k) {
      const int t = grp * GS + k;
      if (t < ITEMS) tm_st4(col_w + (uint32_t)(buf * COLS + ((t % R) * P + (t / R) * GC) * 4), fb[k]);
    }
  };

  // warp-level release of this warp's TMEM stores / loads to an mbarrier
  auto release = [&](uint64_t* bar) {
    tm_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  };
  // prologue: slab of step 0 into buffer 0 (all gates' warps, even inactive ones)
  for (int grp = 0; grp < 3; ++grp) {
    issue(0, grp);
    store(0, grp);
  }
  tm_wait_st();
  release(&full_bar[0]);
  // acc <- tv * X^{-bbar} (cggi.py:612-622): warp o < 2 initialises component o
  if (active && o < 2) {
    const uint32_t bbar = ((lin_s[a.n] + radd) >> rshift) & two_n_mask;
    const uint32_t k = (2 * N - bbar) & two_n_mask;
    const uint32_t* tvc = a.tv + o * N;
    for (int j = lane; j < N; j += 32) {
      const uint32_t m = ((uint32_t)j - k) & two_n_mask;
      acc_g[o * N + j] = m < (uint32_t)N ? tvc[m] : 0u - tvc[m - N];
    }
  }
  __syncthreads();
  // stagger: odd gates start once gate 0 has finished its first forward pass,
  // so neighbouring gates run different phases (FP64-heavy FFTs vs the
  // shared-memory-heavy MAC) at the same time
  if (GC > 1 && (gl & 1)) mbar_wait(go_bar, 0);

  const int bar_id = 1 + gl;
  const bool owner = L == 32 || lane < L;
  // lane twiddles: registers when the CTA is small enough to afford them
  // (saves 2 x 8 KB of shared-memory reads per warp per step), else smem
  // (measured on B200: the register copy costs more than the 2 x 8 KB of smem
  // reads it saves at GC=2 -- 4.76 vs 4.21 ms for 256 gates -- so it is off)
  constexpr bool TWREG = false;
  double2 twr[TWREG ? P : 1];
  if constexpr (TWREG) {
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) twr[k1] = tw1[k1 * L + l];
  }
  // phase accounting (debug): [warp o of gate 0 of CTA 0][phase] cycle sums
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && gl == 0 && lane == 0;
  long long pt[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
  auto mark = [&](int ph) {
    if (prof) {
      const long long t = clock64();
      pt[ph] += t - tprev;
      tprev = t;
    }
  };
  for (int i = 0; i < a.n; ++i) {
    const int cur = i & 1, nxt = cur ^ 1;
    const bool pre = i + 1 < a.n;
    const bool fill = pre && !(a.ablate & 4);  // debug ablation 4: no key streaming
    if (fill) issue(i + 1, 0);  // S0
    // ---- forward: row r = o, r < R ----
    if (active && o < R) {
      const int cr = o / LEV, lv = o % LEV;
      const uint32_t* A = acc_g + cr * N;
      const uint32_t abar = ((lin_s[i] + radd) >> rshift) & two_n_mask;
      const int sh = 32 - (lv + 1) * a.bg_bits;
      double2 x[P];
      const uint32_t idx0 = ((uint32_t)l - abar) & two_n_mask;
      if (a.ablate & 1) {  // debug: no decomposition
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) x[bitrev_c<G::LOGP>(m1)] = make_double2((double)(m1 + l), (double)abar);
      } else if constexpr (LEV == 2) {
        // The two level-warps of component cr split the coefficients by half
        // (warp lv takes j + lv*M), extract BOTH digit levels of their half,
        // and swap the other level's digits through shared memory.
        const int hh = lv;
        const int sh_mine = sh, sh_other = 32 - (2 - lv) * a.bg_bits;
        uint32_t* xg = xchg_all + (size_t)gl * T::XCHG + (size_t)cr * 2 * (P / 2) * 32;
        uint32_t* to_partner = xg + (size_t)(1 - lv) * (P / 2) * 32;
        const uint32_t* from_partner = xg + (size_t)lv * (P / 2) * 32;
        uint32_t mine[P];
#pragma unroll
        for (int m1 = 0; m1 < P; m1 += 2) {
          uint32_t oth[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t j = (uint32_t)(L * (m1 + q) + l + hh * M);
            const uint32_t idx = (idx0 + (uint32_t)(L * (m1 + q)) + (uint32_t)(hh * M)) & two_n_mask;
            const uint32_t v = A[idx & (N - 1)];
            const uint32_t neg = 0u - ((idx >> LOGN) & 1u);  // all ones past X^N
            const uint32_t buf = ((v ^ neg) - neg) - A[j] + a.offs;
            mine[m1 + q] = (buf >> sh_mine) & base_mask;
            oth[q] = (buf >> sh_other) & base_mask;
          }
          to_partner[(m1 / 2) * 32 + lane] = oth[0] | (oth[1] << 16);
        }
        named_barrier(5 + 2 * gl + cr, 64);
#pragma unroll
        for (int m1 = 0; m1 < P; m1 += 2) {
          const uint32_t w = from_partner[(m1 / 2) * 32 + lane];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint32_t rv = q ? (w >> 16) : (w & 0xFFFFu);
            const uint32_t re = hh ? rv : mine[m1 + q], im = hh ? mine[m1 + q] : rv;
            double2 v = make_double2(digit_to_double(re, half_base), digit_to_double(im, half_base));
            if (m1 + q > 0) v = cmul(v, c_root64[G::CSTEP * (m1 + q)]);
            x[bitrev_c<G::LOGP>(m1 + q)] = v;  // DIT forward takes bit-reversed input
          }
        }
      } else
#pragma unroll
      for (int m1 = 0; m1 < P; ++m1) {
        double dd[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t j = (uint32_t)(L * m1 + l + hh * M);
          const uint32_t idx = (idx0 + (uint32_t)(L * m1 + hh * M)) & two_n_mask;
          const uint32_t v = A[idx & (N - 1)];
          const uint32_t neg = 0u - ((idx >> LOGN) & 1u);  // all ones past X^N
          const uint32_t buf = ((v ^ neg) - neg) - A[j] + a.offs;
          dd[hh] = digit_to_double((buf >> sh) & base_mask, half_base);
        }
        // lane-independent part of the twist; the per-lane part lives in tw1'
        double2 v = make_double2(dd[0], dd[1]);
        if (m1 > 0) v = cmul(v, c_root64[G::CSTEP * m1]);
        x[bitrev_c<G::LOGP>(m1)] = v;
      }
      double2* tile = xb + (size_t)o * G::TILE;
      if (!(a.ablate & 16)) {
        if constexpr (TWREG) fft_forward_tw<LOGN, true>(x, tile, TwRegs<P>{twr}, l);
        else fft_forward<LOGN, true>(x, tile, tw1, l);
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < P; ++s) tile[s * L + l] = x[s];
    }
    if (GC > 1 && i == 0 && gl == 0 && lane == 0) mbar_arrive(go_bar);
    mark(0);
    if (pre) {  // S1: buffer nxt is free once every warp finished MAC(i-1)
      mbar_wait(&empty_bar[nxt], i == 0 ? 1u : (uint32_t)(((i - 1) >> 1) & 1));
      tm_fence_after();
      if (fill) {
        store(nxt, 0);
        issue(i + 1, 1);
      }
    }
    mark(1);
    named_barrier(bar_id, 128);
    mbar_wait(&full_bar[cur], (uint32_t)((i >> 1) & 1));
    tm_fence_after();
    mark(2);
    // ---- MAC: output (co, ho) over all R rows, key from TMEM ----
    double2 acc[P];
    // row-outer: the P slots are independent accumulation chains (ILP), the
    // key row arrives 8 slots per tcgen05.ld (32 columns)
    constexpr int SB = P < 8 ? P : 8;
    if (a.ablate & 2) {  // debug: no MAC
#pragma unroll
      for (int s = 0; s < P; ++s) acc[s] = make_double2((double)s, (double)i);
    } else
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int s0 = 0; s0 < P; s0 += SB) {
        uint32_t kw[4 * SB];
        tm_ld_raw<4 * SB>(tm_warp + (uint32_t)(cur * COLS + (r * P + s0) * 4), kw);
        tm_wait_ld();
#pragma unroll
        for (int q = 0; q < SB; ++q) {
          const int s = s0 + q;
          const double2 kr = make_double2(__hiloint2double(kw[4 * q + 1], kw[4 * q]),
                                          __hiloint2double(kw[4 * q + 3], kw[4 * q + 2]));
          const double2 d = xb[(size_t)r * G::TILE + s * L + l];
          acc[s] = r == 0 ? cmul(d, kr) : cfma(acc[s], d, kr);
        }
      }
    }
    release(&empty_bar[cur]);
    mark(3);
    named_barrier(bar_id, 128);
    if (fill) {  // S2
      store(nxt, 1);
      issue(i + 1, 2);
    }
    // ---- inverse, untwist, round, accumulate ----
    if (active) {
      if (!(a.ablate & 32)) {
        if constexpr (TWREG) fft_inverse_tw<LOGN, true>(acc, xb + (size_t)o * G::TILE, TwRegs<P>{twr}, l);
        else fft_inverse<LOGN, true>(acc, xb + (size_t)o * G::TILE, tw1, l);
      }
      uint32_t* Ac = acc_g + co * N;
      const int shift = 16 * ho;
#pragma unroll
      for (int m1 = 0; m1 < P; ++m1) {
        const double2 v = m1 == 0 ? acc[0] : cmulc(acc[m1], c_root64[G::CSTEP * m1]);
        const uint32_t j = (uint32_t)(L * m1 + l);
        if (owner && !(a.ablate & 8)) {
          atomicAdd(Ac + j, round_mod32(v.x) << shift);
          atomicAdd(Ac + j + M, round_mod32(v.y) << shift);
        }
      }
    }
    mark(4);
    if (pre) {  // S3
      if (fill) store(nxt, 2);
      tm_wait_st();
      release(&full_bar[nxt]);
    }
    named_barrier(bar_id, 128);  // acc of this gate updated before the next decomposition
    mark(5);
  }
  if (prof)
    for (int ph = 0; ph < 6; ++ph) a.prof[o * 6 + ph] = pt[ph];
  if (active && o < 2) {
    uint32_t* dst = a.acc_out + ((size_t)g * 2 + o) * N;
    for (int j = lane; j < N; j += 32) dst[j] = acc_g[o * N + j];
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(tm_base, T::ALLOC);
}

}  // namespace gw
