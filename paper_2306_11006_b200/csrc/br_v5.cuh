// br_v5.cuh -- blind rotation v5: the v3 structure (frequency-partitioned MAC,
// key streamed L2 -> loader warps -> TMEM ring, lane twiddles in TMEM) with the
// bootstrapping key held as ONE FFT image of its full 32-bit words instead of
// two 16-bit halves.  Reference: gatewave/cggi.py:592-667 (`_blind_rotate_kernel`),
// PARAM_128 / PARAM_110 geometry (N = 1024, l = 2: four gadget rows).
//
// Per step and gate the external product is 4 forward FFT-512 (one per gadget
// row, as in v3), 8 complex MACs per frequency (v3: 16) and 2 inverse FFT-512
// (one per accumulator component; v3: 4, one per component and key half).
// The key slab of a step is 64 KB (v3: 128 KB) and the HBM image 41 MB, the
// size of the reference's own NTT-domain key (cggi.py:283-285).
//
// Exactness: every coefficient the inverse transforms round is an
// integer of magnitude <= 2l N 2^(Bg-1) 2^31 = 2^51 at PARAM_128 / PARAM_110.
// The FP64 error of the transform chain is no longer provably below 1/2 at
// that magnitude; it is MEASURED (probe build, tests/test_gpu_margin.py):
// every rounded value lies within a few hundredths of an integer, so the
// outputs are bit-identical to the exact (split-key, v3) path and to the
// reference on every tested input.  The worst-case analytic bound still
// limits the phase deviation to < 2^24 raw units after n steps, far inside the
// 2^28 decryption margin (the north star's "stated noise bound").
// GATEWAVE_BR_EXACT=1 (gw_set_exact) selects the split-key v3 kernel.
//
// CTA = GC gates x 4 compute warps + 4 key-loader warps, one CTA per SM.
//   F  warp r: rotate-subtract, gadget digits, fold + twist, forward head of row r
//   M  warp w: frequency pairs (k1, c), c in [4w, 4w+4): last forward radix-2
//      stage of the 4 rows, 2 outputs x 4 rows complex MACs against the key
//      values in TMEM, first inverse radix-2 stage -> V rows 0, 1
//   I  warps (2c, 2c + 1) invert component c together (the paired inverse below:
//      each computes the even or odd outputs of both DFT-16 passes), untwist,
//      round, acc[c] += v with shared-memory RED.ADD.
// TMEM (512 columns): 3 key slabs of 128 columns (slab i in slot i mod 3), the
// forward lane twiddle table (64 columns) and the paired inverse's writer-side
// twiddles (2 x 32 columns).  The loader warps run up to two steps ahead of the
// MAC: slab i waits for MAC(i - 3) to release its slot.
#pragma once

#include "br_v3.cuh"

namespace gw {

struct V5 {
  static constexpr int LOGN = 10, LEV = 2;
  using G = Geo<LOGN>;
  static constexpr int N = G::N, M = G::M, P = G::P, L = G::L, R = 2 * LEV;
  static constexpr int CIDX = 32;                   // key complexes per TMEM lane per step: 4 freqs x (2 outputs x 4 rows)
  static constexpr int COLS = CIDX * 4;             // TMEM columns per slab (128)
  static constexpr int NSLOT = 3;                   // slabs resident in TMEM
  static constexpr int TWCOL = NSLOT * COLS;        // lane twiddles: columns 384..447
  static constexpr int TW4COL = TWCOL + 64;         // paired-inverse twiddles: columns 448..511
  static constexpr int UB = R * P * L;              // double2 per gate: U / V / transpose tiles (32 KB)
  static constexpr int XCHG = 2 * 2 * (P / 2) * 32; // u32 per gate: digit swap between level-warps
  static constexpr int SLAB = CIDX * 128 * 16;      // key bytes per step (64 KB)
  static size_t smem_bytes(int gc) {
    return (size_t)gc * (UB * sizeof(double2) + 2 * N * sizeof(uint32_t) + XCHG * sizeof(uint32_t)) + 256;
  }
};

// key image: [i][cidx][tmem lane] complex, cidx = q*8 + o*4 + r (q = 2p + s as in v3,
// o = accumulator component, r = gadget row), tmem lane = 32*w + lane.
__host__ __device__ __forceinline__ size_t v5_index(int i, int cidx, int tlane) {
  return ((size_t)i * V5::CIDX + cidx) * 128 + tlane;
}

// ---- design switches (compile-time; every default is a same-box A/B, profiles/r02_v5_*) ----
//
// The inverse is always the paired split inverse: two warps of a gate invert one
// accumulator component together, each doing the odd or even outputs of both DFT-16
// passes (decimation in frequency), with the lane twiddles applied by the writer of the
// transpose; warps (0, 1) take component 0, warps (2, 3) component 1.  Against two inverting
// warps per gate: GC = 1 5.78k -> 5.37k, GC = 2 7.99k -> 7.61k, GC = 3 10.40k -> 10.07k
// cycles per step (r02_v5_ipair_ab.txt, r02_v5_ipair_gc23_ab.txt).  Measured and not kept:
// four warps on quarter problems with a shuffle radix-2 (GC = 1 5.81k), pairs across the
// two gates of a CTA (GC = 2 8.23k), gate stagger (+0.1-2.8 %), loader nanosleep back-off
// (+0.7-1.7 % at GC = 2, 3), the forward transpose through TMEM (+2-6 %,
// r02_v5_tmem_transpose_rejected.txt), both pairs' MAC keys requested up front (+4.7 % at GC = 1).

// MAC lanes own the frequency pair (c', c' + 8) (c' = 2w + lane / 16) instead of (c, c + 1),
// so the MAC phase hands the paired inverse its DIF-split inputs directly: V[c'] + V[c'+8]
// in slot c' and (V[c'] - V[c'+8]) w16^(-c') in slot c'+8; each inverting warp reads 8
// values instead of 16.  Global (it changes the key image layout).  GC = 1 5.17k -> 4.97k,
// GC = 2 7.63k -> 7.40k, GC = 3 10.01k -> 9.78k (r02_v5_msplit_ab.txt)
#ifndef GW_V5_MSPLIT
#define GW_V5_MSPLIT 1
#endif
// End-of-step barrier of the inverting pair only (bit GC-1), with V_1 in U row 2 and each
// pair's scratch in its own odd row.  GC = 1 5.12k -> 5.03k, GC = 2 7.72k -> 7.59k,
// GC = 3 10.02k -> 9.93k (r02_v5_pair_b3_ab.txt)
#ifndef GW_V5_PAIR_B3
#define GW_V5_PAIR_B3 7
#endif
// Digit extraction with every accumulator load hoisted above the arithmetic and the
// partner stores (bit GC-1).  GC = 1 5.35k -> 5.23k, GC = 2 7.61k -> 7.66k (off there),
// GC = 3 10.07k -> 10.03k (r02_v5_digit_hoist_ab.txt)
#ifndef GW_V5_DIGITS_HOIST
#define GW_V5_DIGITS_HOIST 5
#endif
// MAC phase with the V stores of both frequency pairs after both MACs (bit GC-1; implied by
// GW_V5_MSPLIT).  GC = 1 5.22k -> 5.11k; GC = 2, 3 +0.2 % (r02_v5_mac_defer_ab.txt)
#ifndef GW_V5_M_DEFER
#define GW_V5_M_DEFER 1
#endif
// L2 bulk prefetch of the key slab GW_V5_L2PF steps ahead (v3 uses 2).  With v5's 64 KB
// slabs it does not pay: distance 0 vs 2: -0.8 / -0.4 / -0.3 % per step at GC = 1 / 2 / 3
// with the key L2-resident, +0.2 % bench value with L2 flushed between steps (r02_v5_l2pf_ab.txt)
#ifndef GW_V5_L2PF
#define GW_V5_L2PF 0
#endif
// F-phase digit conversion specialised on the warp's half (GC >= GW_V5_HH_BRANCH; 0 = never):
// one warp-uniform branch instead of 32 SELs.  GC = 1 +4 % (worse), GC = 2 -0.2 %, GC = 3 -0.6 %
// cycles per step (r02_v5_conv_ab.txt)
#ifndef GW_V5_HH_BRANCH
#define GW_V5_HH_BRANCH 2
#endif
// digit -> double as an integer subtract + I2F.F64 instead of the magic-number DADD, for
// GC >= GW_V5_CONV_I2F (0 = never).  Pays only together with the branch, at GC = 3: -0.3 %
// there, +0.7 / +1.3 % at GC = 2 / 1 (r02_v5_conv_ab.txt)
#ifndef GW_V5_CONV_I2F
#define GW_V5_CONV_I2F 3
#endif
// steps at the end of the blind rotation over which the loader warps warm L2 with the
// keyswitch key image (BrArgs::l2warm)
#ifndef GW_V5_L2WARM_STEPS
#define GW_V5_L2WARM_STEPS 32
#endif
// loader warps wait for a free key slot with a try_wait suspend-time hint (ns; 0 = plain
// try_wait loop; compiles to NANOSLEEP.SYNCS, woken by the barrier): GC = 1 -0.6 % per step,
// GC = 2, 3 neutral for hints 200-20000 ns (r02_v5_ldr_hint_ab.txt)
#ifndef GW_V5_LDR_HINT_NS
#define GW_V5_LDR_HINT_NS 200
#endif
// per-phase cycle counters (GATEWAVE_BR_PROFILE, tools/phase_profile.py) compiled in at
// every GC (default: GC = 2 only); the predicated-off clock reads still cost issue slots
#ifndef GW_V5_PHASE_PROF
#define GW_V5_PHASE_PROF 0
#endif
#ifndef GW_V5_MARK_MASK1
#define GW_V5_MARK_MASK1 0
#endif
#ifndef GW_V5_MARK_MASK2
#define GW_V5_MARK_MASK2 0x01
#endif
#ifndef GW_V5_MARK_MASK3
#define GW_V5_MARK_MASK3 0x10
#endif
#ifndef GW_V5_RED
#define GW_V5_RED 1  // accumulator updates as shared-memory RED.ADD (same-box A/B: -0.4 / -0.7 / -1 % at GC = 1 / 2 / 3 vs load-add-store, profiles/r02_v5_stagger_red_ab.txt)
#endif

#ifndef GW_V5_LREG2
#define GW_V5_LREG2 64
#endif
#ifndef GW_V5_LREG3
#define GW_V5_LREG3 56
#endif

template <int GC, bool PROBE = false>
__global__ void __launch_bounds__(128 * GC + 128, 1) k_blind_rotate_v5(BrArgs a) {
  static_assert(GC >= 1 && GC <= 3, "loader warps need registers the compute warps can spare");
  constexpr int LREG = GC == 1 ? 0 : GC == 2 ? GW_V5_LREG2 : GW_V5_LREG3;
  constexpr int kPool = ((65536 / (128 * GC + 128)) & ~7) * (128 * GC + 128);
  constexpr int CREG = GC == 1 ? 0 : ((kPool - LREG * 128) / (128 * GC)) & ~7;
  using G = V5::G;
  constexpr int N = V5::N, M = V5::M, P = V5::P, L = V5::L, R = V5::R, LEV = V5::LEV, LOGN = V5::LOGN;
  constexpr int UB = V5::UB, COLS = V5::COLS, CIDX = V5::CIDX, NSLOT = V5::NSLOT;
  constexpr int kL2WarmSteps = GW_V5_L2WARM_STEPS;
  constexpr int TWCOL = V5::TWCOL, TW4COL = V5::TW4COL;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double2* ubuf_all = reinterpret_cast<double2*>(smem_raw);  // GC x [row][c][pos]
  uint32_t* acc_all = reinterpret_cast<uint32_t*>(ubuf_all + (size_t)GC * UB);
  uint32_t* xchg_all = acc_all + (size_t)GC * 2 * N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg_all + (size_t)GC * V5::XCHG);
  uint64_t* full_bar = bars;           // [3] the loader warps stored slab i in slot i % 3
  uint64_t* empty_bar = bars + NSLOT;  // [3] every compute warp finished its MAC reads of slot i % 3
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSLOT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane;
  const int gl = warp >> 2, o = warp & 3;
  const int g = blockIdx.x * GC + gl;
  const bool active = g < a.B;
  // inactive gate slots (last CTA) run on row 0 and discard the result
  const uint32_t* lin_g = a.jobs ? nullptr : a.lin + (size_t)(active ? g : 0) * a.lin_stride;
  const uint32_t* src0 = nullptr;
  const uint32_t* src1 = nullptr;
  uint32_t w0 = 1, w1 = 0, body_add = 0;
  if (a.jobs) {  // fused gate prologue, as in v3
    const LinJob jb = a.jobs[active ? g : 0];
    src0 = a.rows + (size_t)jb.src[0] * a.row_stride;
    src1 = jb.src[1] >= 0 ? a.rows + (size_t)jb.src[1] * a.row_stride : src0;
    w0 = (uint32_t)jb.w[0];
    w1 = jb.src[1] >= 0 ? (uint32_t)jb.w[1] : 0u;
    body_add = (uint32_t)jb.cmu * a.mu;
  }
  auto lin_at = [&](int k) -> uint32_t {
    if (!a.jobs) return __ldg(lin_g + k);
    return w0 * __ldg(src0 + k) + w1 * __ldg(src1 + k) + (k == a.n ? body_add : 0u);
  };

  if (threadIdx.x == 0) {
    for (int k = 0; k < NSLOT; ++k) {
      mbar_init(&full_bar[k], 4);
      mbar_init(&empty_bar[k], 4 * GC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(tm_slot, 512);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm_base = *tm_slot;
  const uint32_t tm_warp = tm_base + ((uint32_t)(32 * o) << 16);
  const uint32_t tm_tw = tm_warp + (uint32_t)TWCOL;
  const uint32_t tm_tw4 = tm_warp + (uint32_t)TW4COL;
  if (gl == 0 && warp < 4 * GC) {
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) tm_st4(tm_tw + (uint32_t)(4 * k1), __ldg(a.tables + 2 * G::TILE + k1 * L + l));
    {
      // paired inverse, writer lane (k1, b) of role e: tw'(k1, b + 2 (2a' + e)), a' = 0..7
      // (both roles' tables in every sub-partition: columns TW4COL + 32 e)
      const int k1 = lane >> 1, b = lane & 1;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int a2 = 0; a2 < 8; ++a2)
          tm_st4(tm_tw4 + (uint32_t)(32 * e + 4 * a2), __ldg(a.tables + 2 * G::TILE + k1 * L + b + 2 * (2 * a2 + e)));
    }
    tm_wait_st();
  }

  const uint32_t two_n_mask = 2 * N - 1;
  const uint32_t rshift = 32 - (LOGN + 1);
  const uint32_t radd = 1u << (32 - (LOGN + 1) - 1);
  const uint32_t base_mask = (1u << a.bg_bits) - 1;
  const int32_t half_base = 1 << (a.bg_bits - 1);
  const double dmagic = 6755399441055744.0 + (double)half_base;

  uint32_t* acc_g = acc_all + (size_t)gl * 2 * N;
  double2* U = ubuf_all + (size_t)gl * UB;

  // acc <- tv * X^{-bbar} (cggi.py:612-622): warp o < 2 initialises component o
  if (warp < 4 * GC && o < 2) {
    const uint32_t bbar = ((lin_at(a.n) + radd) >> rshift) & two_n_mask;
    const uint32_t k = (2 * N - bbar) & two_n_mask;
    const uint32_t* tvc = a.tv + o * N;
    for (int j = lane; j < N; j += 32) {
      const uint32_t m = ((uint32_t)j - k) & two_n_mask;
      acc_g[o * N + j] = m < (uint32_t)N ? tvc[m] : 0u - tvc[m - N];
    }
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();

  const int mk1 = lane & 15;
  const int mc0 = 4 * o + 2 * (lane >> 4);
  // MAC-phase frequency of pair p owned by this lane (see GW_V5_MSPLIT)
  auto mfreq = [&](int p) { return GW_V5_MSPLIT ? 2 * o + (lane >> 4) + 8 * p : mc0 + p; };
  // U row that receives V_oo (the MAC output of accumulator component oo)
  constexpr bool kPairB3 = (GW_V5_PAIR_B3 >> (GC - 1)) & 1;
  auto v_row = [](int oo) { return kPairB3 ? 2 * oo : oo; };
  // the paired inverse's named barrier: warps (2 oo, 2 oo + 1) of gate gl
  // (ids: 1..GC per gate for B1-B3, 5..4+2GC the F level pairs)
  const int kPairQ = 2 * gl + (o >> 1);
  const int kPairBar = GC == 3 ? (kPairQ == 0 ? 4 : 10 + kPairQ) : 9 + kPairQ;
  const int pos = v3_pos(l);
  const int bar_id = 1 + gl;

  // the (predicated-off) clock reads of the phase profiler cost issue slots and steer
  // ptxas's schedule: without them GC = 1 / 3 run 3.9 / 1.7 % faster; at GC = 2 the first
  // one alone (after the forward phase) gives the best schedule, 1.9 % faster than all six
  // and 3.8 % faster than none; at GC = 3 the fifth alone (after the inverse), 0.75 % faster
  // than none (r02_v5_phase_marks_ab.txt).  -DGW_V5_PHASE_PROF=1 puts all
  // six back at every GC for tools/phase_profile.py.
  constexpr int kMarkMask = GW_V5_PHASE_PROF ? 0x3F : GC == 1 ? GW_V5_MARK_MASK1 : GC == 2 ? GW_V5_MARK_MASK2 : GW_V5_MARK_MASK3;
  constexpr bool kMarks = kMarkMask != 0;
  const bool prof = kMarks && a.prof != nullptr && blockIdx.x == 0 && gl == 0 && lane == 0;
  long long pt_[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
  auto mark = [&](int ph) {
    if (!((kMarkMask >> ph) & 1)) return;
    if (prof) {
      const long long t = clock64();
      pt_[ph] += t - tprev;
      tprev = t;
    }
  };

  if (warp >= 4 * GC) {
    // ---- loader warp: slab i -> TMEM slot i % 3 of sub-partition o ----
    if constexpr (GC >= 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(LREG));
    const double2* src_w = a.bk + (size_t)32 * o + lane;
    int slot = 0;
    for (int i = 0; i < a.n; ++i) {
      const double2* src = src_w + (size_t)i * CIDX * 128;
#if GW_V5_L2PF
      if (o == 0 && lane == 0 && i + GW_V5_L2PF < a.n) {
        const char* pf = reinterpret_cast<const char*>(a.bk + (size_t)(i + GW_V5_L2PF) * CIDX * 128);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(V5::SLAB) : "memory");
      }
#endif
      if (o == 3 && lane == 0 && a.l2warm_bytes && i >= a.n - kL2WarmSteps) {
        // this CTA's share of the keyswitch key image, one chunk per remaining step
        const uint64_t share = ((a.l2warm_bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
        const uint64_t chunk = ((share + kL2WarmSteps - 1) / kL2WarmSteps + 15) & ~15ull;
        const uint64_t lo = (uint64_t)blockIdx.x * share + (uint64_t)(i - (a.n - kL2WarmSteps)) * chunk;
        const uint64_t hi = min(min(lo + chunk, (uint64_t)(blockIdx.x + 1) * share), a.l2warm_bytes);
        for (uint64_t p = lo; p < hi; p += 65536) {
          const uint32_t len = (uint32_t)min(hi - p, (uint64_t)65536);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.l2warm + p), "r"(len) : "memory");
        }
      }
      if (i >= NSLOT) {
        if constexpr (GW_V5_LDR_HINT_NS > 0)
          mbar_wait_hint<GW_V5_LDR_HINT_NS>(&empty_bar[slot], (uint32_t)(((i - NSLOT) / NSLOT) & 1));
        else
          mbar_wait(&empty_bar[slot], (uint32_t)(((i - NSLOT) / NSLOT) & 1));
        tm_fence_after();
      }
      const uint32_t dst = tm_warp + (uint32_t)(slot * COLS);
#pragma unroll 1
      for (int rnd = 0; rnd < CIDX / 16; ++rnd) {
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = ldg_stream(src + (size_t)(rnd * 16 + k) * 128);
#pragma unroll
        for (int k = 0; k < 16; ++k) tm_st4(dst + (uint32_t)((rnd * 16 + k) * 4), v[k]);
      }
      tm_wait_st();
      tm_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[slot]);
      slot = slot + 1 == NSLOT ? 0 : slot + 1;
    }
  } else {
    if constexpr (GC >= 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CREG));
    uint32_t a_next = lin_at(0);
    double worst = 0.0;  // PROBE only
    int slot = 0;
    for (int i = 0; i < a.n; ++i) {
      const uint32_t a_i = a_next;
      if (i + 1 < a.n) a_next = lin_at(i + 1);
      // ---------------- F: row r = o (identical to v3) ----------------
      {
        const int cr = o / LEV, lv = o % LEV;
        const uint32_t* A = acc_g + cr * N;
        const uint32_t abar = ((a_i + radd) >> rshift) & two_n_mask;
        const uint32_t idx0 = ((uint32_t)l - abar) & two_n_mask;
        double2 x[P];
        const int hh = lv;
        const int sh_mine = 32 - (lv + 1) * a.bg_bits, sh_other = 32 - (2 - lv) * a.bg_bits;
        uint32_t* xg = xchg_all + (size_t)gl * V5::XCHG + (size_t)cr * 2 * (P / 2) * 32;
        uint32_t* to_partner = xg + (size_t)(1 - lv) * (P / 2) * 32;
        const uint32_t* from_partner = xg + (size_t)lv * (P / 2) * 32;
        uint32_t mine[P];
        const uint32_t idxh = idx0 + (uint32_t)(hh * M);
        if constexpr ((GW_V5_DIGITS_HOIST >> (GC - 1)) & 1) {
          // every accumulator read first, then the arithmetic, then the stores to the
          // partner: a store to the exchange area may not be moved above a later load of
          // acc by the compiler (it cannot prove the two regions disjoint), so with the
          // loads interleaved each coefficient pair would wait for the previous pair's
          // whole load -> digit -> store chain
          uint32_t vrot[P], vdir[P];
#pragma unroll
          for (int m1 = 0; m1 < P; ++m1) {
            const uint32_t idx = (idxh + (uint32_t)(L * m1)) & two_n_mask;
            vrot[m1] = A[idx & (N - 1)];
            vdir[m1] = A[L * m1 + l + hh * M];
          }
          uint32_t packed[P / 2];
#pragma unroll
          for (int m1 = 0; m1 < P; m1 += 2) {
            uint32_t oth[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t idx = (idxh + (uint32_t)(L * (m1 + q))) & two_n_mask;
              const uint32_t neg = 0u - ((idx >> LOGN) & 1u);
              const uint32_t buf = ((vrot[m1 + q] ^ neg) - neg) - vdir[m1 + q] + a.offs;
              mine[m1 + q] = (buf >> sh_mine) & base_mask;
              oth[q] = (buf >> sh_other) & base_mask;
            }
            packed[m1 / 2] = oth[0] | (oth[1] << 16);
          }
#pragma unroll
          for (int k = 0; k < P / 2; ++k) to_partner[k * 32 + lane] = packed[k];
        } else {
#pragma unroll
          for (int m1 = 0; m1 < P; m1 += 2) {
            uint32_t oth[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t idx = (idxh + (uint32_t)(L * (m1 + q))) & two_n_mask;
              const uint32_t v = A[idx & (N - 1)];
              const uint32_t neg = 0u - ((idx >> LOGN) & 1u);
              const uint32_t buf = ((v ^ neg) - neg) - A[L * (m1 + q) + l + hh * M] + a.offs;
              mine[m1 + q] = (buf >> sh_mine) & base_mask;
              oth[q] = (buf >> sh_other) & base_mask;
            }
            to_partner[(m1 / 2) * 32 + lane] = oth[0] | (oth[1] << 16);
          }
        }
        named_barrier(5 + 2 * gl + cr, 64);
        // digit (offset by half the base) -> double: the magic-number DADD, or (GW_V5_CONV_I2F)
        // an integer subtract and an int -> double conversion
        constexpr bool kI2F = GW_V5_CONV_I2F > 0 && GC >= GW_V5_CONV_I2F;
        constexpr bool kHHBranch = GW_V5_HH_BRANCH > 0 && GC >= GW_V5_HH_BRANCH;
        auto dconv = [&](uint32_t u) -> double {
          if constexpr (kI2F) return __int2double_rn((int)u - half_base);
          else return digit_to_double_lo(u, dmagic);
        };
        // (re, im) = (digit of j, digit of j + M): the level-warp of half hh computed its own
        // level's digits for half hh and received the partner's for the other half
        auto convert = [&](auto sel) {
          const bool upper = sel();
#pragma unroll
          for (int m1 = 0; m1 < P; m1 += 2) {
            const uint32_t w = from_partner[(m1 / 2) * 32 + lane];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t rv = q ? (w >> 16) : (w & 0xFFFFu);
              const uint32_t re = upper ? rv : mine[m1 + q], im = upper ? mine[m1 + q] : rv;
              double2 v = make_double2(dconv(re), dconv(im));
              if (m1 + q > 0) v = cmul(v, c_root64[G::CSTEP * (m1 + q)]);
              x[bitrev_c<G::LOGP>(m1 + q)] = v;
            }
          }
        };
        if constexpr (kHHBranch) {
          if (hh) convert([] { return true; });
          else convert([] { return false; });
        } else {
          convert([&] { return hh != 0; });
        }
        double2* tile = U + (size_t)o * P * L;
        fft_forward_head<LOGN, true>(x, tile, TwTmemHalves{tm_tw}, l);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < P; ++c) tile[c * L + pos] = x[c];
      }
      mark(0);
      named_barrier(bar_id, 128);  // U complete
      mark(1);
      // ---------------- M: frequency pairs (mk1, mc0 + p), 2 outputs x 4 rows ----------------
      mbar_wait(&full_bar[slot], (uint32_t)((i / NSLOT) & 1));
      tm_fence_after();
      const uint32_t tm_slab = tm_warp + (uint32_t)(slot * COLS);
      // GW_V5_M_DEFER: the V stores of both pairs after both MACs, so pair 1's loads need
      // not wait for pair 0's stores (the compiler keeps stores and later loads of U in order)
      constexpr bool kDefer = GW_V5_MSPLIT || ((GW_V5_M_DEFER >> (GC - 1)) & 1);
      double2 vout[2][2][2];  // [p][output][b], kDefer only
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int c = mfreq(p);
        const double2 tw = c_root64[2 * c];  // e^{2 pi i c / 32}
        uint32_t kw[2][32];
        // both s halves of this pair's keys: 2 x 32 columns (8 complex each)
#pragma unroll
        for (int s = 0; s < 2; ++s) tm_ld_raw<32>(tm_slab + (uint32_t)((2 * p + s) * 32), kw[s]);
        double2 D[R][2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double2* row = U + ((size_t)r * P + c) * L;
          const double2 u0 = row[v3_slot(mk1, 0)], u1 = row[v3_slot(mk1, 1)];
          const double2 t = cmul(u1, tw);
          D[r][0] = cadd(u0, t);
          D[r][1] = csub(u0, t);
        }
        tm_wait_ld();
        double2 O[2][2];  // [output][s]
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int oo = 0; oo < 2; ++oo)
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const uint32_t* k4 = kw[s] + (oo * 4 + r) * 4;
              const double2 kr = make_double2(__hiloint2double(k4[1], k4[0]), __hiloint2double(k4[3], k4[2]));
              O[oo][s] = r == 0 ? cmul(D[r][s], kr) : cfma(O[oo][s], D[r][s], kr);
            }
#pragma unroll
        for (int oo = 0; oo < 2; ++oo) {
          const double2 v0 = cadd(O[oo][0], O[oo][1]);
          const double2 v1 = cmulc(csub(O[oo][0], O[oo][1]), tw);
          if constexpr (kDefer) {
            vout[p][oo][0] = v0;
            vout[p][oo][1] = v1;
          } else {
            double2* row = U + ((size_t)v_row(oo) * P + c) * L;
            row[v3_slot(mk1, 0)] = v0;
            row[v3_slot(mk1, 1)] = v1;
          }
        }
      }
      if constexpr (GW_V5_MSPLIT) {
        // the paired inverse's DIF split of pass 1, done here: slot c' <- V[c'] + V[c'+8],
        // slot c'+8 <- (V[c'] - V[c'+8]) w16^(-c')
        const int c1 = mfreq(0);
#pragma unroll
        for (int oo = 0; oo < 2; ++oo)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const double2 dsum = cadd(vout[0][oo][b], vout[1][oo][b]);
            double2 ddif = csub(vout[0][oo][b], vout[1][oo][b]);
            if (c1 != 0) ddif = cmulc(ddif, c_root64[4 * c1]);
            U[((size_t)v_row(oo) * P + c1) * L + v3_slot(mk1, b)] = dsum;
            U[((size_t)v_row(oo) * P + c1 + 8) * L + v3_slot(mk1, b)] = ddif;
          }
      } else if constexpr (kDefer) {
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
          for (int oo = 0; oo < 2; ++oo) {
            double2* row = U + ((size_t)v_row(oo) * P + mc0 + p) * L;
            row[v3_slot(mk1, 0)] = vout[p][oo][0];
            row[v3_slot(mk1, 1)] = vout[p][oo][1];
          }
      }
      tm_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      mark(2);
      named_barrier(bar_id, 128);  // V complete
      mark(3);
      // ---------------- I: paired inverse, warps (2 oo, 2 oo + 1) -> component oo ----------------
      {
        // warps (2 oo, 2 oo + 1) invert component oo; role rr: even (0) / odd (1) outputs
        const int rr = o & 1, oo = o >> 1;
        const int pair_bar = kPairBar;
        const double2* tileV = U + (size_t)v_row(oo) * P * L;
        // the scratch row is free after M: rows 2, 3 (V in rows 0, 1), or row 2 oo + 1 when
        // V_oo sits in row 2 oo (GW_V5_PAIR_B3: each pair then touches only its own rows)
        double2* scratch = U + (size_t)(kPairB3 ? 2 * oo + 1 : 2 + oo) * P * L;
        uint32_t tw8[32];
        tm_ld_raw<32>(tm_tw4 + (uint32_t)(32 * rr), tw8);
        // pass 1, lane (k1, b): T[2a' + rr] = DFT-8_{c'} of (V[c'] +- V[c'+8]) w16^(-rr c')
        double2 x[8];
        if constexpr (GW_V5_MSPLIT) {  // the MAC phase wrote this role's DIF-split inputs
#pragma unroll
          for (int c2 = 0; c2 < 8; ++c2) x[bitrev_c<3>(c2)] = tileV[(8 * rr + c2) * L + pos];
        } else {
          double2 v[16];
#pragma unroll
          for (int c = 0; c < P; ++c) v[c] = tileV[c * L + pos];
#pragma unroll
          for (int c2 = 0; c2 < 8; ++c2)
            x[bitrev_c<3>(c2)] = rr == 0 ? cadd(v[c2], v[c2 + 8])
                                          : (c2 == 0 ? csub(v[0], v[8]) : cmulc(csub(v[c2], v[c2 + 8]), c_root64[4 * c2]));
        }
        dit<8, -1>(x);
        tm_wait_ld();
        {
          const int k1 = l >> 1, b = l & 1;
#pragma unroll
          for (int a2 = 0; a2 < 8; ++a2) {
            const uint32_t* w4 = tw8 + 4 * a2;
            const double2 tw = make_double2(__hiloint2double(w4[1], w4[0]), __hiloint2double(w4[3], w4[2]));
            scratch[k1 * L + swz(k1, b + 2 * (2 * a2 + rr))] = cmulc(x[a2], tw);
          }
        }
        named_barrier(pair_bar, 64);
        // pass 2, lane l: z[2m' + rr] = DFT-8_{k'} of (S[k'] +- S[k'+8]) w16^(-rr k')
        {
          double2 v[16];
#pragma unroll
          for (int k1 = 0; k1 < P; ++k1) v[k1] = scratch[k1 * L + swz(k1, l)];
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2)
            x[bitrev_c<3>(k2)] = rr == 0 ? cadd(v[k2], v[k2 + 8])
                                          : (k2 == 0 ? csub(v[0], v[8]) : cmulc(csub(v[k2], v[k2 + 8]), c_root64[4 * k2]));
        }
        dit<8, -1>(x);
        if (active) {
          uint32_t* Ac = acc_g + oo * N;
#pragma unroll
          for (int m2 = 0; m2 < 8; ++m2) {
            const int m1 = 2 * m2 + rr;
            const double2 v = m1 == 0 ? x[0] : cmulc(x[m2], c_root64[G::CSTEP * m1]);  // untwist
            const uint32_t j = (uint32_t)(L * m1 + l);
            if constexpr (PROBE) worst = fmax(worst, fmax(fabs(v.x - rint(v.x)), fabs(v.y - rint(v.y))));
#if GW_V5_RED
            atomicAdd(Ac + j, round_mod32(v.x));
            atomicAdd(Ac + j + M, round_mod32(v.y));
#else
            Ac[j] += round_mod32(v.x);
            Ac[j + M] += round_mod32(v.y);
#endif
          }
        }
      }
      mark(4);
      // acc updated before the next decomposition.  With GW_V5_PAIR_B3 only the pair that
      // updated component oo waits: the same two warps decompose component oo next, read
      // only acc[oo], and write only U rows 2 oo, 2 oo + 1, which no other warp reads before B1.
      if constexpr (kPairB3) named_barrier(kPairBar, 64); else named_barrier(bar_id, 128);
      mark(5);
      slot = slot + 1 == NSLOT ? 0 : slot + 1;
    }
    if constexpr (PROBE) {
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, d));
      if (lane == 0 && active && a.margin) atomicMax(a.margin, (unsigned long long)__double_as_longlong(worst));
    }
    if (prof)
      for (int ph = 0; ph < 6; ++ph) a.prof[o * 6 + ph] = pt_[ph];
    // component c is written back by warp 2c, one of the two warps that updated it (the
    // pair's last barrier orders their updates; with GW_V5_PAIR_B3 nothing else does)
    if (active && (o & 1) == 0) {
      const int cc = o >> 1;
      uint32_t* dst = a.acc_out + ((size_t)g * 2 + cc) * N;
      for (int j = lane; j < N; j += 32) dst[j] = acc_g[cc * N + j];
    }
  }
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(tm_base, 512);
}

// Key image for v5 (reference: cggi.py:283-285 keeps the NTT-domain copy).  One
// warp per (i, r, c) polynomial: the full signed 32-bit words, fold + twist, the
// forward head, the last radix-2 stage for every (k1, c) pair, scaled by 1/M and
// scattered to [i][cidx][tmem lane].
__global__ void __launch_bounds__(128) k_bk_to_v5(const uint32_t* __restrict__ bk_coeff, int n,
                                                  const double2* __restrict__ tables, double2* __restrict__ img) {
  using G = V5::G;
  constexpr int N = V5::N, M = V5::M, P = V5::P, L = V5::L, R = V5::R;
  __shared__ double2 tw1[P * L];
  __shared__ double2 tiles[4][P * L];
  for (int t = threadIdx.x; t < P * L; t += blockDim.x) tw1[t] = tables[2 * G::TILE + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane;
  const long long job = (long long)blockIdx.x * 4 + warp;  // (i*R + r)*2 + c
  if (job >= (long long)n * R * 2) return;
  const int c = (int)(job & 1);
  const int r = (int)((job >> 1) % R);
  const int i = (int)((job >> 1) / R);
  const uint32_t* poly = bk_coeff + (((size_t)i * R + r) * 2 + c) * N;
  double2 x[P];
#pragma unroll
  for (int m1 = 0; m1 < P; ++m1) {
    double2 v = make_double2((double)(int32_t)poly[L * m1 + l], (double)(int32_t)poly[L * m1 + l + M]);
    if (m1 > 0) v = cmul(v, c_root64[G::CSTEP * m1]);
    x[bitrev_c<G::LOGP>(m1)] = v;
  }
  double2* tile = tiles[warp];
  fft_forward_head<V5::LOGN, true>(x, tile, TwSmem{tw1, L, l}, l);
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < P; ++cc) tile[cc * L + v3_pos(l)] = x[cc];
  __syncwarp();
  const double scale = 1.0 / (double)M;
  const int k1 = lane & 15;
#pragma unroll
  for (int w = 0; w < 4; ++w)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int cf = GW_V5_MSPLIT ? 2 * w + (lane >> 4) + 8 * p : 4 * w + 2 * (lane >> 4) + p;
      const double2 u0 = tile[cf * L + v3_slot(k1, 0)], u1 = tile[cf * L + v3_slot(k1, 1)];
      const double2 t = cmul(u1, c_root64[2 * cf]);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double2 d = s ? csub(u0, t) : cadd(u0, t);
        const int cidx = (2 * p + s) * 8 + c * 4 + r;
        img[v5_index(i, cidx, 32 * w + lane)] = make_double2(d.x * scale, d.y * scale);
      }
    }
}

}  // namespace gw
