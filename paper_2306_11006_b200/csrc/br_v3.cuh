// br_v3.cuh -- blind rotation v3: frequency-partitioned MAC, bootstrapping key
// streamed L2 -> registers -> a TMEM ring, lane twiddles resident in TMEM.
// Reference: gatewave/cggi.py:592-667 (`_blind_rotate_kernel`), PARAM_128 /
// PARAM_110 geometry (N = 1024, l = 2: four gadget rows, four MAC outputs).
//
// CTA = GC gates x 4 compute warps (+ 4 key-loader warps for GC <= 3), one
// CTA per SM (it owns all 512 TMEM columns).
// Per step i, per gate:
//   F  warp r (row r = (component r/2, level r%2)): rotate-subtract +
//      gadget-decompose acc[r/2] (cggi.py:627-644), fold + twist, forward FFT
//      head (DFT-16, lane twiddle, transpose, DFT-16) -> u_b[c] into U[r].
//   M  warp w (TMEM sub-partition w) owns the frequency pairs (k1, c) with
//      c in [4w, 4w+4): it finishes the last radix-2 stage of all four rows
//      for its pairs, multiplies by the 16 key values of each of its 4
//      frequencies (read from TMEM, cggi.py:648-657), and applies the first
//      radix-2 stage of the four inverse transforms; results -> V (= U).
//   I  warp o (output o = (component o/2, key half o%2)): inverse FFT tail,
//      untwist, round, acc[o/2] += v << 16*(o%2) with shared-memory atomics
//      (cggi.py:658-666; wrap-around adds commute, so the result is exact).
// Compared to v2 (br_tmem.cuh), every shared-memory value is read once per
// step instead of four times, and the lane-pair radix-2 stage needs no
// shuffles or selects.  The key slab of a step (128 KB: 64 complex per TMEM
// lane, four 64-column chunks) lives in a 7-chunk TMEM ring next to the lane
// twiddle table (64 columns); see the KM modes below for who fills it.
#pragma once
#include "blind_rotate.cuh"
#include "ks_tc.cuh"
#include "mbarrier.cuh"
#include "tmem.cuh"

#ifndef GW_STAGGER2
#define GW_STAGGER2 1  // GC = 2: gate 1 starts after gate 0's decomposition (0), F (1) or M (2) of step 0
                        // (same-box A/B: 9.54k / 9.39k / 9.64k cycles per step)
#endif
// Loader-warp register budget and loads in flight per round at 2 / 3 gates per CTA.
// Same-box A/B (cycles per step): GC=2 LREG 64 + RS 16 9.40k, LREG 56 9.64k, LREG 104 +
// RS 24 9.76k; GC=3 LREG 56 12.64k, 64 12.94k, 40 13.17k, RS 8 14.7k, RS 12 17.7k.
#ifndef GW_LREG2
#define GW_LREG2 64
#endif
#ifndef GW_LREG3
#define GW_LREG3 56
#endif
#ifndef GW_RS2
#define GW_RS2 16
#endif
#ifndef GW_RS3
#define GW_RS3 16
#endif
// Loader warps: one thread per CTA prefetches the key slab GW_L2PF steps ahead into L2
// (cp.async.bulk.prefetch).  Same-box A/B, cycles per step: GC=2 9.41k -> 9.23k at distance
// 2, 4 or 6 (1 and 3 are 9-10 % slower); GC=1 -0.3 %, GC=3 neutral.  With the transform work
// ablated, GC=2 drops from 8.86k to 7.43k: the L2 latency of the key loads is what bounds the
// step once the compute gets faster.  Splitting the prefetch so each CTA requests only its
// 1/148 share of the slab is slower (GC=2 9.43k): every CTA prefetching the whole slab wins.
#ifndef GW_L2PF
#define GW_L2PF 2
#endif
#ifndef GW_TW_SMEM_GC
#define GW_TW_SMEM_GC 5  // smallest GC that keeps the lane twiddles in shared memory (none: TMEM measured faster at GC=4 too)
#endif

namespace gw {

struct V3 {
  static constexpr int LOGN = 10, LEV = 2;
  using G = Geo<LOGN>;
  static constexpr int N = G::N, M = G::M, P = G::P, L = G::L, R = 2 * LEV;
  static constexpr int CIDX = 64;                   // key complexes per TMEM lane per step: 4 freqs x (4 outputs x 4 rows)
  static constexpr int COLS = CIDX * 4;             // TMEM columns per step slab
  // TMEM: a ring of 7 key chunks (chunk = the 16 key values of one of a lane's
  // 4 frequencies = 64 columns) + the lane-twiddle table (16 complex = 64 columns)
  static constexpr int RING = 7, CHUNK = 64, TWCOL = RING * CHUNK;
  static constexpr int UB = R * P * L;              // double2 per gate: U / V / transpose tiles (32 KB)
  static constexpr int XCHG = 2 * 2 * (P / 2) * 32; // u32 per gate: digit swap between level-warps
  static constexpr int SLAB = CIDX * 128 * 16;      // key bytes per step (128 KB)
  // TMA mode stages the slab in shared memory (only where it fits: GC = 1)
  static size_t smem_bytes(int gc, bool tma) {
    return (tma ? (size_t)SLAB : 0) +
           (size_t)gc * (UB * sizeof(double2) + 2 * N * sizeof(uint32_t) + XCHG * sizeof(uint32_t)) +
           (gc >= GW_TW_SMEM_GC ? (size_t)P * L * sizeof(double2) : 0) + 128;
  }
};

// key image: [i][cidx][tmem lane] complex, cidx = q*16 + o*4 + r, tmem lane = 32*w + lane.
// Lane (w, lane) owns frequency pairs (k1 = lane & 15, c = 4w + 2*(lane >> 4) + p), q = 2p + s,
// s = 0: u_0 + w^c u_1, s = 1: u_0 - w^c u_1.
__host__ __device__ __forceinline__ size_t v3_index(int i, int cidx, int tlane) {
  return ((size_t)i * V3::CIDX + cidx) * 128 + tlane;
}

// Lane twiddles streamed from TMEM eight at a time (register-lean variant for
// GC >= 3): the transforms call tw(k1) for k1 = 0..15 in order.
#ifndef GW_TW_CHUNK
#define GW_TW_CHUNK 4  // complex twiddles per TMEM load in the register-lean variant (A/B: 4 > 2 > 8)
#endif
struct TwTmemHalves {
  static constexpr int C = GW_TW_CHUNK;
  uint32_t taddr;
  mutable uint32_t r[4 * C];
  __device__ __forceinline__ double2 operator()(int k1) const {
    if (k1 % C == 0) {
      tm_ld_raw<4 * C>(taddr + (uint32_t)((k1 / C) * 4 * C), r);
      tm_wait_ld();
    }
    const uint32_t* w = r + (k1 % C) * 4;
    return make_double2(__hiloint2double(w[1], w[0]), __hiloint2double(w[3], w[2]));
  }
};

// Slot of u_b[c] for k1 inside the 32-wide row c of U: 16 b + (k1 ^ 4b).  Both
// access patterns are conflict-free 16-byte accesses: a quarter-warp of the
// row warps (k1 in 4q..4q+3, b = 0, 1) and of the MAC warps (8 consecutive
// k1, fixed b) each touch 8 distinct bank groups.
__device__ __forceinline__ int v3_slot(int k1, int b) { return (b << 4) | (k1 ^ (b << 2)); }
__device__ __forceinline__ int v3_pos(int l) { return v3_slot(l >> 1, l & 1); }

__device__ __forceinline__ double2 ldg_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void tm_cp_128x256b(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}


// Key streaming modes (KM).  2, the default for GC <= 3: four loader warps
// (one per TMEM sub-partition) load each slab with 16-24 coalesced 16-byte
// loads in flight and store it with tcgen05.st, up to two steps ahead (chunks
// 0-2 of slab i wait for MAC(i-2), chunk 3 for MAC(i-1)); at GC = 2, 3
// setmaxnreg gives the compute warps CREG and the loaders LREG registers.
// 0 (GC = 4, or GATEWAVE_BR_LDR=0): the compute warps load their share at the
// four phase points of a step.  1 (GC = 1 with GATEWAVE_BR_GC1=tma): warp 0
// stages the slab through shared memory (cp.async.bulk -> tcgen05.cp), which
// costs 256 KB of shared-memory traffic per step (measured slower).
//
// KM = key streaming mode: 0 LDG by the compute warps, 1 TMA by warp 0, 2 four
// dedicated loader warps (one per TMEM sub-partition; GC = 1 only).
// PROBE: rounding-margin probe build (worst |x - rint(x)| before every rounding
// of the inverse transform) -- the exactness evidence.
template <int GC, int KM, bool PROBE = false>
__global__ void __launch_bounds__(128 * GC + (KM == 2 ? 128 : 0), 1) k_blind_rotate_v3(BrArgs a) {
  constexpr bool TMA = KM == 1, LDR = KM == 2;
  static_assert(!LDR || GC <= 3, "loader warps need registers the compute warps can spare");
  // with loader warps at GC >= 2 the register file is re-split with setmaxnreg:
  // compute warpgroups CREG, the loader warpgroup LREG (CREG*128*GC + LREG*128 <= 64K)
  constexpr int LREG = GC == 1 ? 0 : GC == 2 ? GW_LREG2 : GW_LREG3;
  // the register pool is what the launch allocated: (64K / threads) rounded down to 8, per thread
  constexpr int kPool = ((65536 / (128 * GC + 128)) & ~7) * (128 * GC + 128);
  constexpr int CREG = GC == 1 ? 0 : ((kPool - LREG * 128) / (128 * GC)) & ~7;
  using G = V3::G;
  constexpr int N = V3::N, M = V3::M, P = V3::P, L = V3::L, R = V3::R, LEV = V3::LEV, LOGN = V3::LOGN;
  constexpr int UB = V3::UB, COLS = V3::COLS, CIDX = V3::CIDX;
  // KM = 0: the slab is 8 groups of 8 cidx; warp (gl, w) owns groups gl, gl+GC, ...
  // and handles group list entry j at phase point j % 4 (GC = 1: two per point)
  constexpr int NG = (8 + GC - 1) / GC;     // max groups per warp
  constexpr int GPP = (NG + 3) / 4;         // groups per phase point

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stage = smem_raw;                                               // TMA mode: 128 KB slab
  double2* ubuf_all = reinterpret_cast<double2*>(smem_raw + (TMA ? V3::SLAB : 0));  // GC x [row][c][pos]
  uint32_t* acc_all = reinterpret_cast<uint32_t*>(ubuf_all + (size_t)GC * UB);
  uint32_t* xchg_all = acc_all + (size_t)GC * 2 * N;
  // GC = 4 (128 registers): lane twiddles from a shared-memory table; otherwise TMEM
  constexpr bool kTwSmem = GC >= GW_TW_SMEM_GC;
  double2* tw1 = reinterpret_cast<double2*>(xchg_all + (size_t)GC * V3::XCHG);
  uint64_t* bars = reinterpret_cast<uint64_t*>(tw1 + (kTwSmem ? P * L : 0));
  if constexpr (kTwSmem)
    for (int t = threadIdx.x; t < P * L; t += blockDim.x) tw1[t] = a.tables[2 * G::TILE + t];
  uint64_t* full_bar = bars;       // [2] every warp stored its share of the slab in TMEM buffer b
  uint64_t* empty_bar = bars + 2;  // [2] every warp finished its MAC reads of buffer b
  uint64_t* stage_bar = bars + 4;  // TMA mode: slab landed in shared memory
  uint64_t* go_bar = bars + 5;     // [2] stagger: gate 0 reached its start points for gates 1 / 2
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(bars + 7);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane;
  const int gl = warp >> 2, o = warp & 3;
  const int g = blockIdx.x * GC + gl;
  const bool active = g < a.B;
  // inactive gate slots (last CTA) run on row 0 and discard the result, so the
  // barrier protocol never depends on the batch size
  const uint32_t* lin_g = a.jobs ? nullptr : a.lin + (size_t)(active ? g : 0) * a.lin_stride;
  // fused gate prologue: the LWE row of a bootstrap is the gate's
  // linear combination of its operand rows, read straight from the wire store
  const uint32_t* src0 = nullptr;
  const uint32_t* src1 = nullptr;
  uint32_t w0 = 1, w1 = 0, body_add = 0;
  if (a.jobs) {
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
    for (int k = 0; k < 2; ++k) {
      mbar_init(&full_bar[k], TMA ? 1 : LDR ? 4 : 4 * GC);
      mbar_init(&empty_bar[k], 4 * GC);
    }
    mbar_init(stage_bar, 1);
    mbar_init(&go_bar[0], 4);
    mbar_init(&go_bar[1], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tm_alloc(tm_slot, 512);
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tm_base = *tm_slot;
  const uint32_t tm_warp = tm_base + ((uint32_t)(32 * o) << 16);
  const uint32_t tm_tw = tm_warp + (uint32_t)V3::TWCOL;
  // lane twiddles tw'[k1][l] -> TMEM columns TWCOL + 4 k1 of every sub-partition
  // (read with tcgen05.ld in the transforms instead of 32 LDS.128 per warp-step)
  if (!kTwSmem && gl == 0) {
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) tm_st4(tm_tw + (uint32_t)(4 * k1), __ldg(a.tables + 2 * G::TILE + k1 * L + l));
    tm_wait_st();
  }
  // key chunk q of step i: ring slot (4 i + q) mod 7 when the twiddles live in
  // TMEM; plain double buffering (slot 4 (i & 1) + q) when they do not (GC = 4:
  // the ring's chunk-3 reuse couples the gates of a CTA one step tighter)
  constexpr bool kRing = !kTwSmem;
  auto kcol = [&](int slot_i, int q) -> uint32_t {
    const int sl = slot_i + q;
    return (uint32_t)((kRing && sl >= V3::RING ? sl - V3::RING : sl) * V3::CHUNK);
  };

  // ---- key streaming ----
  const double2* kw_base = a.bk + (size_t)32 * o + lane;
  double2 kb[GPP][8];
  // LDG mode, phase point pt of step i: load / store this warp's groups
  auto kissue = [&](int i, int pt) {
    if constexpr (KM == 0) {
      const double2* src = kw_base + (size_t)i * CIDX * 128;
#pragma unroll
      for (int gg = 0; gg < GPP; ++gg) {
        const int j = pt * GPP + gg, grp = gl + GC * j;
        if (j < NG && grp < 8)
#pragma unroll
          for (int k = 0; k < 8; ++k) kb[gg][k] = ldg_stream(src + (size_t)(grp * 8 + k) * 128);
      }
    }
  };
  // store for step i+1 (ring base slot sn); its chunk 3 reuses the slot of step i's
  // chunk 0, so it waits until every warp has finished MAC(i) (empty barrier of step i)
  auto kstore = [&](int i, int sn, int pt) {
    if constexpr (KM == 0) {
#pragma unroll
      for (int gg = 0; gg < GPP; ++gg) {
        const int j = pt * GPP + gg, grp = gl + GC * j;
        if (j < NG && grp < 8) {
          if (kRing && grp >> 1 == 3) {
            mbar_wait(&empty_bar[i & 1], (uint32_t)((i >> 1) & 1));
            tm_fence_after();
          }
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tm_st4(tm_warp + kcol(sn, grp >> 1) + (uint32_t)(((grp & 1) * 8 + k) * 4), kb[gg][k]);
        }
      }
    }
  };
  auto release = [&](uint64_t* bar) {
    tm_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  };
  // TMA mode: slab -> TMEM buffer, 32 copies of 128 lanes x 8 columns (two cidx each)
  const uint32_t stage_s = smem_u32(stage);
  const unsigned char* img = reinterpret_cast<const unsigned char*>(a.bk);
  auto copy_to_tmem = [&](int buf, int sn) {
#pragma unroll 4
    for (int j = 0; j < COLS / 8; ++j)  // 8-column block j holds cidx 2j, 2j+1 (chunk j / 8)
      tm_cp_128x256b(tm_base + kcol(sn, j >> 3) + (uint32_t)((j & 7) * 8),
                     umma_desc(stage_s + j * 4096, 2048, 128));
    umma_commit(&full_bar[buf]);
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {  // prologue: slab 0 -> buffer 0
      mbar_expect_tx(stage_bar, V3::SLAB);
      bulk_g2s(stage, img, V3::SLAB, stage_bar);
      mbar_wait(stage_bar, 0);
      copy_to_tmem(0, 0);
    }
  } else if constexpr (KM == 0) {
    for (int pt = 0; pt < 4; ++pt) {  // prologue: slab 0 -> ring slots 0..3 (no chunk-3 wait)
      kissue(0, pt);
#pragma unroll
      for (int gg = 0; gg < GPP; ++gg) {
        const int j = pt * GPP + gg, grp = gl + GC * j;
        if (j < NG && grp < 8)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            tm_st4(tm_warp + kcol(0, grp >> 1) + (uint32_t)(((grp & 1) * 8 + k) * 4), kb[gg][k]);
      }
    }
    tm_wait_st();
    release(&full_bar[0]);
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
  // orders the twiddle-table tcgen05.st (and the prologue key stores) before
  // every warp's tcgen05.ld
  tm_fence_before();
  __syncthreads();
  tm_fence_after();

  // MAC-phase geometry of this lane: pairs (k1, c_p), p = 0, 1
  const int mk1 = lane & 15;
  const int mc0 = 4 * o + 2 * (lane >> 4);
  const int pos = v3_pos(l);
  const int bar_id = 1 + gl;
  int sc = 0;  // ring slot base of step i: (4 i) mod 7

  const bool prof = a.prof != nullptr && blockIdx.x == 0 && gl == 0 && lane == 0;
  long long pt_[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
  auto mark = [&](int ph) {
    if (prof) {
      const long long t = clock64();
      pt_[ph] += t - tprev;
      tprev = t;
    }
  };

  if (LDR && warp >= 4 * GC) {
    // ---- loader warp: slab i -> ring slots of sub-partition o, ahead of the MAC ----
    if constexpr (LDR && GC >= 2) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(LREG));
    constexpr int RS = GC == 1 ? 24 : GC == 2 ? GW_RS2 : GW_RS3;  // loads in flight per round (divides 48)
    const double2* src_w = a.bk + (size_t)32 * o + lane;
    int s_i = 0;
    for (int i = 0; i < a.n; ++i) {
      const double2* src = src_w + (size_t)i * CIDX * 128;
#if GW_L2PF
      // one thread per CTA asks L2 for slab i + GW_L2PF ahead of every SM's loads
      if (o == 0 && lane == 0 && i + GW_L2PF < a.n) {
        const char* pf = reinterpret_cast<const char*>(a.bk + (size_t)(i + GW_L2PF) * CIDX * 128);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(V3::SLAB) : "memory");
      }
#endif
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
      release(&full_bar[i & 1]);
      s_i = s_i + 4 >= V3::RING ? s_i + 4 - V3::RING : s_i + 4;
    }
  } else {
  if constexpr (LDR && GC >= 2) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CREG));
  // Stagger (measured: GC = 3 +1 %, GC = 2 +1.6-8 %): the gates of a CTA start at
  // different points of step 0 so they run different phases at once.  GC = 3:
  // gate 1 after gate 0's F(0), gate 2 after its M(0); GC = 2: gate 1 after gate
  // 0's F(0) (GW_STAGGER2).
  constexpr bool kStagger = LDR && (GC == 3 || GC == 2);
  if (kStagger && gl >= 1) mbar_wait(&go_bar[gl - 1], 0);
  uint32_t a_next = lin_at(0);
  uint32_t sink = 0;  // GW_ABL & 8 only
  double worst = 0.0;  // PROBE only
  for (int i = 0; i < a.n; ++i) {
    const int cur = i & 1, nxt = cur ^ 1;
    const int sn = kRing ? (sc + 4 >= V3::RING ? sc + 4 - V3::RING : sc + 4) : 4 - sc;  // slot base of step i+1
    const bool pre = i + 1 < a.n;
    const uint32_t a_i = a_next;
    if (pre) {
      a_next = lin_at(i + 1);
      kissue(i + 1, 0);
    }
    // ---------------- F: row r = o ----------------
    {
      const int cr = o / LEV, lv = o % LEV;
      const uint32_t* A = acc_g + cr * N;
      const uint32_t abar = ((a_i + radd) >> rshift) & two_n_mask;
      const uint32_t idx0 = ((uint32_t)l - abar) & two_n_mask;
      double2 x[P];
      // The two level-warps of component cr split the coefficients by half
      // (warp lv takes j + lv*M), extract BOTH digit levels of their half and
      // swap the other level's digits through shared memory.
      const int hh = lv;
      const int sh_mine = 32 - (lv + 1) * a.bg_bits, sh_other = 32 - (2 - lv) * a.bg_bits;
      uint32_t* xg = xchg_all + (size_t)gl * V3::XCHG + (size_t)cr * 2 * (P / 2) * 32;
      uint32_t* to_partner = xg + (size_t)(1 - lv) * (P / 2) * 32;
      const uint32_t* from_partner = xg + (size_t)lv * (P / 2) * 32;
      uint32_t mine[P];
      const uint32_t idxh = idx0 + (uint32_t)(hh * M);
#if GW_ABL & 1
#pragma unroll
      for (int m1 = 0; m1 < P; ++m1) mine[m1] = (idxh + (uint32_t)(7 * m1)) & base_mask;
#pragma unroll
      for (int m1 = 0; m1 < P; m1 += 2) {
        const uint32_t w = (mine[m1] * 3u) | (mine[m1 + 1] << 16);
#else
#pragma unroll
      for (int m1 = 0; m1 < P; m1 += 2) {
        uint32_t oth[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t idx = (idxh + (uint32_t)(L * (m1 + q))) & two_n_mask;
          const uint32_t v = A[idx & (N - 1)];
          const uint32_t neg = 0u - ((idx >> LOGN) & 1u);  // all ones past X^N
          const uint32_t buf = ((v ^ neg) - neg) - A[L * (m1 + q) + l + hh * M] + a.offs;
          mine[m1 + q] = (buf >> sh_mine) & base_mask;
          oth[q] = (buf >> sh_other) & base_mask;
        }
        to_partner[(m1 / 2) * 32 + lane] = oth[0] | (oth[1] << 16);
      }
      named_barrier(5 + 2 * gl + cr, 64);
#pragma unroll
      for (int m1 = 0; m1 < P; m1 += 2) {
        const uint32_t w = from_partner[(m1 / 2) * 32 + lane];
#endif
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const uint32_t rv = q ? (w >> 16) : (w & 0xFFFFu);
          const uint32_t re = hh ? rv : mine[m1 + q], im = hh ? mine[m1 + q] : rv;
          double2 v = make_double2(digit_to_double_lo(re, dmagic), digit_to_double_lo(im, dmagic));
          if (m1 + q > 0) v = cmul(v, c_root64[G::CSTEP * (m1 + q)]);
          x[bitrev_c<G::LOGP>(m1 + q)] = v;  // DIT forward takes bit-reversed input
        }
      }
      if (GC == 2 && GW_STAGGER2 == 0 && kStagger && i == 0 && gl == 0 && lane == 0) mbar_arrive(&go_bar[0]);
      double2* tile = U + (size_t)o * P * L;
      // lane twiddles streamed from TMEM in chunks during the twiddle multiply
      // (measured: GC = 1 -1.5 % per step against loading all 16 up front; GC = 2 neutral)
      if constexpr (!kTwSmem) {
        fft_forward_head<LOGN, true>(x, tile, TwTmemHalves{tm_tw}, l);
      } else {
        fft_forward_head<LOGN, true>(x, tile, TwSmem{tw1, L, l}, l);
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < P; ++c) tile[c * L + pos] = x[c];
    }
    if ((GC == 3 || (GC == 2 && GW_STAGGER2 == 1)) && kStagger && i == 0 && gl == 0 && lane == 0)
      mbar_arrive(&go_bar[0]);
    mark(0);
    if (KM == 0 && pre) {  // buffer nxt is free once every warp finished MAC(i-1)
      if (i >= 1) mbar_wait(&empty_bar[nxt], (uint32_t)(((i - 1) >> 1) & 1));
      tm_fence_after();
      kstore(i, sn, 0);
      kissue(i + 1, 1);
    }
    named_barrier(bar_id, 128);  // U complete
    mark(1);
    // ---------------- M: frequency pairs (mk1, mc0 + p) of all rows ----------------
    mbar_wait(&full_bar[cur], (uint32_t)((i >> 1) & 1));
    tm_fence_after();
    if (TMA && threadIdx.x == 0 && pre) {  // the copies of slab i are done: refill the staging buffer
      mbar_expect_tx(stage_bar, V3::SLAB);
      bulk_g2s(stage, img + (size_t)(i + 1) * V3::SLAB, V3::SLAB, stage_bar);
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int c = mc0 + p;
      const double2 tw = c_root64[2 * c];  // e^{2 pi i c / 32}
      double2 D[R][2];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double2* row = U + ((size_t)r * P + c) * L;
        const double2 u0 = row[v3_slot(mk1, 0)], u1 = row[v3_slot(mk1, 1)];
        const double2 t = cmul(u1, tw);
        D[r][0] = cadd(u0, t);
        D[r][1] = csub(u0, t);
      }
      double2 O[4][2];  // [output][s]
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#if GW_ABL & 4
#pragma unroll
        for (int oo = 0; oo < 4; ++oo) O[oo][s] = D[oo][s];
#else
        uint32_t kw[2][32];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
          tm_ld_raw<32>(tm_warp + kcol(sc, 2 * p + s) + (uint32_t)(hf * 32), kw[hf]);
        tm_wait_ld();
#pragma unroll
        for (int oo = 0; oo < 4; ++oo)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t* k4 = kw[oo >> 1] + ((oo & 1) * 4 + r) * 4;
            const double2 kr = make_double2(__hiloint2double(k4[1], k4[0]), __hiloint2double(k4[3], k4[2]));
            O[oo][s] = r == 0 ? cmul(D[r][s], kr) : cfma(O[oo][s], D[r][s], kr);
          }
#endif
      }
#pragma unroll
      for (int oo = 0; oo < 4; ++oo) {
        double2* row = U + ((size_t)oo * P + c) * L;
        row[v3_slot(mk1, 0)] = cadd(O[oo][0], O[oo][1]);
        row[v3_slot(mk1, 1)] = cmulc(csub(O[oo][0], O[oo][1]), tw);
      }
    }
    release(&empty_bar[cur]);
    if (kStagger && i == 0 && gl == 0 && lane == 0) mbar_arrive(&go_bar[1]);
    if (GC == 2 && GW_STAGGER2 == 2 && kStagger && i == 0 && gl == 0 && lane == 0) mbar_arrive(&go_bar[0]);
    mark(2);
    if (pre) {
      kstore(i, sn, 1);
      kissue(i + 1, 2);
    }
    named_barrier(bar_id, 128);  // V complete
    mark(3);
    // ---------------- I: output o = (component o/2, half o%2) ----------------
    {
      double2 x[P];
      double2* tile = U + (size_t)o * P * L;
#pragma unroll
      for (int c = 0; c < P; ++c) x[bitrev_c<G::LOGP>(c)] = tile[c * L + pos];
      if constexpr (!kTwSmem) {
        fft_inverse_tail<LOGN, true>(x, tile, TwTmemHalves{tm_tw}, l);
      } else {
        fft_inverse_tail<LOGN, true>(x, tile, TwSmem{tw1, L, l}, l);
      }
      if (pre) {
        kstore(i, sn, 2);
        kissue(i + 1, 3);
      }
      if (active) {
        uint32_t* Ac = acc_g + (o >> 1) * N;
        const int shift = 16 * (o & 1);
#pragma unroll
        for (int m1 = 0; m1 < P; ++m1) {
          const double2 v = m1 == 0 ? x[0] : cmulc(x[m1], c_root64[G::CSTEP * m1]);
          const uint32_t j = (uint32_t)(L * m1 + l);
          if constexpr (PROBE) worst = fmax(worst, fmax(fabs(v.x - rint(v.x)), fabs(v.y - rint(v.y))));
#if GW_ABL & 8
          sink ^= (round_mod32(v.x) << shift) + round_mod32(v.y);
          (void)j;
#else
          atomicAdd(Ac + j, round_mod32(v.x) << shift);
          atomicAdd(Ac + j + M, round_mod32(v.y) << shift);
#endif
        }
      }
    }
    mark(4);
    if (KM == 0 && pre) {
      kstore(i, sn, 3);
      tm_wait_st();
      release(&full_bar[nxt]);
    }
    // TMA mode, slab i+1: staging -> TMEM buffer nxt.  The whole of warp 0
    // waits (the bar.sync below is warp-aligned), one thread issues.
    if (TMA && warp == 0 && pre) {
      mbar_wait(stage_bar, (uint32_t)((i + 1) & 1));
      if (i >= 1) mbar_wait(&empty_bar[nxt], (uint32_t)(((i - 1) >> 1) & 1));
      mbar_wait(&empty_bar[cur], (uint32_t)((i >> 1) & 1));  // chunk 3 reuses step i's chunk-0 slot
      tm_fence_after();
      if (threadIdx.x == 0) copy_to_tmem(nxt, sn);
      __syncwarp();
    }
    named_barrier(bar_id, 128);  // acc updated before the next decomposition
    mark(5);
    sc = sn;
  }
#if GW_ABL & 8
  if (active) atomicXor(acc_g, sink);
#endif
  (void)sink;
  if constexpr (PROBE) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, d));
    if (lane == 0 && active && a.margin) atomicMax(a.margin, (unsigned long long)__double_as_longlong(worst));
  }
  if (prof)
    for (int ph = 0; ph < 6; ++ph) a.prof[o * 6 + ph] = pt_[ph];
  if (active && o < 2) {
    uint32_t* dst = a.acc_out + ((size_t)g * 2 + o) * N;
    for (int j = lane; j < N; j += 32) dst[j] = acc_g[o * N + j];
  }
  }  // compute warps
  tm_fence_before();
  __syncthreads();
  if (warp == 0) tm_dealloc(tm_base, 512);
}

// Key image for v3 (reference: cggi.py:283-285 keeps the NTT-domain copy).  One
// warp per (i, r, c, h) polynomial: balanced 16-bit split, fold + twist, the
// same forward head as the gate kernel, then the last radix-2 stage for every
// (k1, c) pair, scaled by 1/M and scattered to [i][cidx][tmem lane].
__global__ void __launch_bounds__(128) k_bk_to_v3(const uint32_t* __restrict__ bk_coeff, int n,
                                                  const double2* __restrict__ tables, double2* __restrict__ img) {
  using G = V3::G;
  constexpr int N = V3::N, M = V3::M, P = V3::P, L = V3::L, R = V3::R;
  __shared__ double2 tw1[P * L];
  __shared__ double2 tiles[4][P * L];
  for (int t = threadIdx.x; t < P * L; t += blockDim.x) tw1[t] = tables[2 * G::TILE + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane;
  const long long job = (long long)blockIdx.x * 4 + warp;  // ((i*R + r)*2 + c)*2 + h
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
    double2 v = make_double2((double)part[0], (double)part[1]);
    if (m1 > 0) v = cmul(v, c_root64[G::CSTEP * m1]);
    x[bitrev_c<G::LOGP>(m1)] = v;
  }
  double2* tile = tiles[warp];
  fft_forward_head<V3::LOGN, true>(x, tile, TwSmem{tw1, L, l}, l);
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < P; ++cc) tile[cc * L + v3_pos(l)] = x[cc];
  __syncwarp();
  const double scale = 1.0 / (double)M;
  const int oo = c * 2 + h;
  const int k1 = lane & 15;
#pragma unroll
  for (int w = 0; w < 4; ++w)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const int cf = 4 * w + 2 * (lane >> 4) + p;
      const double2 u0 = tile[cf * L + v3_slot(k1, 0)], u1 = tile[cf * L + v3_slot(k1, 1)];
      const double2 t = cmul(u1, c_root64[2 * cf]);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double2 d = s ? csub(u0, t) : cadd(u0, t);
        const int cidx = (2 * p + s) * 16 + oo * 4 + r;
        img[v3_index(i, cidx, 32 * w + lane)] = make_double2(d.x * scale, d.y * scale);
      }
    }
}

}  // namespace gw
