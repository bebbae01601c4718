// gw_api.cu -- C ABI of the B200 CGGI engine (include/gatewave_b200.h).
//
// Host-side responsibilities: parameter envelope, key upload + on-device FFT
// pre-transform, scratch management, descriptor building for gate batches
// and level plans, and the launch sequence per level:
//   k_lin -> k_blind_rotate -> k_zero_units -> k_keyswitch -> k_cheap
// All launches go to the context stream; only the host-pointer entry points
// synchronise (they must hand results back to the caller).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/gatewave_b200.h"
#include "blind_rotate.cuh"
#include "br_tmem.cuh"
#include "br_v3.cuh"
#include "br_v5.cuh"
#include "gates.cuh"
#include "keyswitch.cuh"
#include "ks_tc.cuh"

using namespace gw;

struct BatchDesc {
  void* mem = nullptr;
  LinJob* jobs = nullptr;
  KsUnit* units = nullptr;
  CheapUnit* cheap = nullptr;
  int J = 0, U = 0, C = 0;
};

struct gw_ctx {
  int device = 0;
  int sm_count = 148;
  int max_smem = 0;  // cudaDevAttrMaxSharedMemoryPerBlockOptin, cached
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  gw_params p{};
  bool have_params = false;
  bool have_keys = false;   // both keys present
  bool have_bk = false;
  bool have_ksk = false;
  int logn = 0;
  int Wp = 0;  // padded LWE row stride (words)
  // keys
  double2* bk_fft = nullptr;
  size_t bk_fft_count = 0;
  double2* bk_v3 = nullptr;    // v3 key image (br_v3.cuh), N = 1024 and l = 2 only
  double2* bk_v5 = nullptr;    // v5 single key image (br_v5.cuh), where v5 applies (v5_ok)
  uint32_t* ksk = nullptr;
  uint8_t* kimg = nullptr;     // keyswitch key as INT8 tensor-core B image (ks_tc.cuh)
  int kt_ntiles = 0, kt_kblocks = 0;
  size_t kimg_bytes = 0;
  bool ks_l2warm = true;        // v5 warms L2 with the key image before the keyswitch (GATEWAVE_KS_L2WARM)
  bool ks_tc = false;          // tensor-core keyswitch usable for these parameters
  int ks_variant = 1;          // 1: tensor cores when usable, 0: CUDA cores (GATEWAVE_KS_KERNEL=cuda)
  uint32_t* ks_ut = nullptr;   // (N, count) rounded samples
  size_t ks_ut_cap = 0;
  double2* tables = nullptr;
  uint32_t* tv_dev = nullptr;  // default test vector (0 | mu)
  // scratch
  uint32_t* lin = nullptr;
  size_t lin_cap = 0;  // rows
  uint32_t* acc = nullptr;
  size_t acc_cap = 0;  // rows (jobs)
  uint32_t* io = nullptr;
  size_t io_cap = 0;  // words
  void* desc = nullptr;
  size_t desc_cap = 0;  // bytes
  void* desc_host = nullptr;  // pinned
  size_t desc_host_cap = 0;
  cudaEvent_t desc_copied = nullptr;  // the last H2D copy out of desc_host
  // wire store
  uint32_t* wires = nullptr;
  int64_t wire_slots = 0;    // slots in use (0: no store)
  int64_t wires_cap = 0;     // slots allocated (owned stores are reused while they fit)
  bool wires_owned = true;   // false when attached to caller memory (torch)
  // device descriptors of homogeneous gate batches, keyed by (opcode, B)
  std::map<uint64_t, BatchDesc> batch_desc;
  // timing / accounting
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool profile = false;                       // per-stage event pairs (gw_set_profiling)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_ev[3];  // 0 blind rotate, 1 keyswitch, 2 other
  std::vector<cudaEvent_t> ev_pool;
  int64_t prof_items[3] = {0, 0, 0};
  int64_t launches = 0;
  long long* br_prof = nullptr;  // device buffer for phase cycle counters (GATEWAVE_BR_PROFILE=1)
  int br_ablate = 0;              // GATEWAVE_BR_ABLATE (debug timing only; results become wrong)
  // 2: v3 (frequency-partitioned MAC, TMA + tcgen05.cp key) where it applies (N = 1024, l = 2),
  // 1: v2 TMEM 4-warp kernel, 0: v1 2-warp kernel (GATEWAVE_BR_KERNEL=v3|v2|v1)
  int br_variant = 2;
  int br_gc = 0;  // v3 gates per CTA override (GATEWAVE_BR_GC, measurement only; 0 = by batch size)
  bool br_gc1_tma = false;  // GATEWAVE_BR_GC1=tma: one-gate CTAs stage the key through shared memory
  bool br_ldr = true;       // loader warps at GC = 2, 3 (GATEWAVE_BR_LDR=0: LDG by the compute warps)
  bool br_unfused = false;  // GATEWAVE_BR_UNFUSED=1: separate k_lin launch (A/B)
  bool br_exact = false;    // gw_set_exact / GATEWAVE_BR_EXACT=1: split-key v3 kernel instead of v5
  std::vector<cudaEvent_t> marks;  // device timeline (gw_timeline_*)
  void* nccl = nullptr;            // ncclComm_t owned by the context (gw_nccl_init)
  unsigned long long* margin = nullptr;  // rounding-margin probe accumulator (gw_set_margin_probe)
  int nccl_world = 0, nccl_rank = 0;
  std::string err;
};

struct gw_plan {
  int64_t n_levels = 0;
  std::vector<int> J, U, C;            // per segment counts
  std::vector<int64_t> seg_first;      // (n_levels + 1): first segment of each level
  std::vector<size_t> job_off, unit_off, cheap_off;
  LinJob* jobs = nullptr;
  KsUnit* units = nullptr;
  CheapUnit* cheap = nullptr;
  int max_jobs = 0;
  int64_t max_wire = -1;  // highest wire id the plan touches (checked against the store at run time)
};

namespace {

int fail(gw_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define GW_CUDA(ctx, expr)                                                             \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail((ctx), GW_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define GW_LAUNCHED(ctx)                                                               \
  do {                                                                                 \
    (ctx)->launches++;                                                                 \
    cudaError_t e_ = cudaGetLastError();                                               \
    if (e_ != cudaSuccess)                                                             \
      return fail((ctx), GW_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

int ilog2(int v) {
  int r = 0;
  while ((1 << r) < v) ++r;
  return (1 << r) == v ? r : -1;
}

template <typename T>
int ensure(gw_ctx* c, T** ptr, size_t* cap, size_t need, size_t elem_bytes) {
  if (*cap >= need && *ptr) return GW_OK;
  if (*ptr) {
    GW_CUDA(c, cudaStreamSynchronize(c->stream));  // in-flight work may still use it
    cudaFree(*ptr);
  }
  *ptr = nullptr;
  *cap = 0;
  size_t n = need < 16 ? 16 : need;
  n += n / 4;
  GW_CUDA(c, cudaMalloc((void**)ptr, n * elem_bytes));
  *cap = n;
  return GW_OK;
}

int ensure_desc(gw_ctx* c, size_t bytes) {
  if (c->desc_cap < bytes || !c->desc) {
    if (c->desc) cudaFree(c->desc);
    c->desc = nullptr;
    size_t n = bytes + bytes / 4 + 256;
    GW_CUDA(c, cudaMalloc(&c->desc, n));
    c->desc_cap = n;
  }
  if (c->desc_host_cap < bytes || !c->desc_host) {
    // the previous contents may still be in flight
    GW_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->desc_host) cudaFreeHost(c->desc_host);
    c->desc_host = nullptr;
    size_t n = bytes + bytes / 4 + 256;
    GW_CUDA(c, cudaMallocHost(&c->desc_host, n));
    c->desc_host_cap = n;
  }
  return GW_OK;
}

// cudaFuncSetAttribute / cudaDeviceGetAttribute cost microseconds per call: the
// dynamic shared-memory size set on a kernel and the device's opt-in limit are
// cached per (device, kernel).
int max_smem_optin(gw_ctx* c) {
  if (c->max_smem <= 0) cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  return c->max_smem;
}

template <typename K>
int set_smem(gw_ctx* c, K* kern, size_t bytes) {
  static std::map<std::pair<int, const void*>, size_t> applied;
  static std::mutex mtx;
  std::lock_guard<std::mutex> lk(mtx);
  const auto key = std::make_pair(c->device, (const void*)kern);
  auto it = applied.find(key);
  if (it != applied.end() && it->second >= bytes) return GW_OK;
  GW_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  applied[key] = bytes;
  return GW_OK;
}

// Host twiddle tables, long double -> correctly rounded-ish doubles.
void host_tables(int logn, std::vector<double2>& out) {
  const int N = 1 << logn, M = N / 2;
  const int P = 1 << ((logn - 2) / 2), L = 2 * P;
  out.resize(3 * P * L);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int k1 = 0; k1 < P; ++k1)
    for (int l = 0; l < L; ++l) {
      long double a = 2.0L * pi * (long double)(l * k1) / (long double)M;
      out[k1 * L + l] = make_double2((double)cosl(a), (double)sinl(a));
    }
  for (int m1 = 0; m1 < P; ++m1)
    for (int l = 0; l < L; ++l) {
      long double a = pi * (long double)(L * m1 + l) / (long double)N;
      out[P * L + m1 * L + l] = make_double2((double)cosl(a), (double)sinl(a));
    }
  // tw1'[k1][l] = e^{i pi l (1 + 4 k1) / N}: lane twiddle with the per-lane twist folded in
  for (int k1 = 0; k1 < P; ++k1)
    for (int l = 0; l < L; ++l) {
      long double a = pi * (long double)(l * (1 + 4 * k1)) / (long double)N;
      out[2 * P * L + k1 * L + l] = make_double2((double)cosl(a), (double)sinl(a));
    }
}

int upload_roots(gw_ctx* c) {
  double2 roots[64];
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int t = 0; t < 64; ++t) {
    long double a = 2.0L * pi * (long double)t / 64.0L;
    roots[t] = make_double2((double)cosl(a), (double)sinl(a));
  }
  // exact values where they exist
  roots[0] = make_double2(1.0, 0.0);
  roots[16] = make_double2(0.0, 1.0);
  roots[32] = make_double2(-1.0, 0.0);
  roots[48] = make_double2(0.0, -1.0);
  GW_CUDA(c, cudaMemcpyToSymbol(c_root64, roots, sizeof(roots)));
  double2 ts[64];
  for (int t = 0; t < 64; ++t) {
    const long double a = 2.0L * pi * (long double)t / 64.0L;
    const bool case_a = (t % 32) <= 8 || (t % 32) >= 24;  // |cos| >= |sin|
    ts[t] = case_a ? make_double2((double)cosl(a), (double)(sinl(a) / cosl(a)))
                   : make_double2((double)sinl(a), (double)(cosl(a) / sinl(a)));
  }
  GW_CUDA(c, cudaMemcpyToSymbol(c_ts64, ts, sizeof(ts)));
  return GW_OK;
}

// ---- kernel dispatch over (LOGN, LEV) --------------------------------------

template <int LOGN, int LEV>
int launch_br_t(gw_ctx* c, const BrArgs& a0) {
  BrArgs a = a0;
  int gc = (int)((a.B + c->sm_count - 1) / c->sm_count);
  if (gc < 1) gc = 1;
  if (gc > 4) gc = 4;
  const int max_smem = max_smem_optin(c);
  while (gc > 1 && BrSmem<LOGN, LEV>::bytes(gc, a.n) > (size_t)max_smem) --gc;
  const size_t smem = BrSmem<LOGN, LEV>::bytes(gc, a.n);
  if (smem > (size_t)max_smem)
    return fail(c, GW_ERR_PARAM, "LWE dimension too large for the on-chip blind rotation");
  if (int rc = set_smem(c, k_blind_rotate<LOGN, LEV>, smem)) return rc;
  a.gates_per_cta = gc;
  const int grid = (a.B + gc - 1) / gc;
  k_blind_rotate<LOGN, LEV><<<grid, 64 * gc, smem, c->stream>>>(a);
  GW_LAUNCHED(c);
  return GW_OK;
}

template <int LOGN, int LEV, int GC>
int launch_tm_g(gw_ctx* c, const BrArgs& a0, int max_smem) {
  BrArgs a = a0;
  const size_t smem = TmGeo<LOGN, LEV>::smem_bytes(GC, a.n);
  if (smem > (size_t)max_smem) return 1;  // caller falls back
  if (int rc = set_smem(c, k_blind_rotate_tm<LOGN, LEV, GC>, smem)) return rc;
  a.gates_per_cta = GC;
  const int grid = (a.B + GC - 1) / GC;
  k_blind_rotate_tm<LOGN, LEV, GC><<<grid, 128 * GC, smem, c->stream>>>(a);
  GW_LAUNCHED(c);
  return GW_OK;
}

// TMEM 4-warp kernel: one CTA per SM (it owns the TMEM), GC gates per CTA.
template <int LOGN, int LEV>
int launch_tm(gw_ctx* c, const BrArgs& a) {
  const int max_smem = max_smem_optin(c);
  const int per_sm = (int)((a.B + c->sm_count - 1) / c->sm_count);
  int rc = 1;
  if (per_sm >= 3) rc = launch_tm_g<LOGN, LEV, 4>(c, a, max_smem);
  if (rc == 1 && per_sm >= 2) rc = launch_tm_g<LOGN, LEV, 2>(c, a, max_smem);
  if (rc == 1) rc = launch_tm_g<LOGN, LEV, 1>(c, a, max_smem);
  if (rc == 1) return launch_br_t<LOGN, LEV>(c, a);
  return rc;
}

template <int GC, int KM, bool PROBE = false>
int launch_v3_g(gw_ctx* c, const BrArgs& a0) {
  BrArgs a = a0;
  a.bk = c->bk_v3;
  a.margin = PROBE ? c->margin : nullptr;
  const size_t smem = V3::smem_bytes(GC, KM == 1);
  if (int rc = set_smem(c, k_blind_rotate_v3<GC, KM, PROBE>, smem)) return rc;
  a.gates_per_cta = GC;
  const int grid = (a.B + GC - 1) / GC;
  k_blind_rotate_v3<GC, KM, PROBE><<<grid, 128 * GC + (KM == 2 ? 128 : 0), smem, c->stream>>>(a);
  GW_LAUNCHED(c);
  return GW_OK;
}

// v3: one CTA per SM holding GC gates.  GC minimises waves x step time, with the
// measured per-step cycles of each configuration (profiles/r01_v3_gc_sweep.txt):
// GC=1 7.8k (loader warps), GC=2 9.6k, GC=3 12.6k (loader warps + setmaxnreg + stagger),
// GC=4 17.7k (LDG key streaming by the compute warps).
int launch_v3(gw_ctx* c, const BrArgs& a) {
  static const double kStep[5] = {0, 7.8, 9.2, 12.6, 17.7};
  int gc = 1;
  double best = 1e300;
  for (int g = 1; g <= 4; ++g) {
    const double waves = (double)((a.B + (int64_t)c->sm_count * g - 1) / ((int64_t)c->sm_count * g));
    const double t = waves * kStep[g];
    if (t < best * 0.999) {
      best = t;
      gc = g;
    }
  }
  if (c->br_gc > 0) gc = c->br_gc;
  if (c->margin) {  // rounding-margin probe build: loader-warp variants only
    if (gc >= 3) return launch_v3_g<3, 2, true>(c, a);
    if (gc == 2) return launch_v3_g<2, 2, true>(c, a);
    return launch_v3_g<1, 2, true>(c, a);
  }
  if (gc >= 4) return launch_v3_g<4, 0>(c, a);
  if (gc == 3) return c->br_ldr ? launch_v3_g<3, 2>(c, a) : launch_v3_g<3, 0>(c, a);
  if (gc == 2) return c->br_ldr ? launch_v3_g<2, 2>(c, a) : launch_v3_g<2, 0>(c, a);
  return c->br_gc1_tma ? launch_v3_g<1, 1>(c, a) : launch_v3_g<1, 2>(c, a);
}

template <int GC, bool PROBE = false>
int launch_v5_g(gw_ctx* c, const BrArgs& a0) {
  BrArgs a = a0;
  a.bk = c->bk_v5;
  a.margin = PROBE ? c->margin : nullptr;
  const size_t smem = V5::smem_bytes(GC);
  if (int rc = set_smem(c, k_blind_rotate_v5<GC, PROBE>, smem)) return rc;
  a.gates_per_cta = GC;
  const int grid = (a.B + GC - 1) / GC;
  k_blind_rotate_v5<GC, PROBE><<<grid, 128 * GC + 128, smem, c->stream>>>(a);
  GW_LAUNCHED(c);
  return GW_OK;
}

// v5 (single key image): GC minimises waves x step time over the measured
// per-step cycles of each configuration.
int launch_v5(gw_ctx* c, const BrArgs& a) {
  static const double kStep[4] = {0, 4.75, 7.22, 9.45};  // k cycles per step, profiles/r02_v5_phase_marks_ab.txt
  int gc = 1;
  double best = 1e300;
  for (int g = 1; g <= 3; ++g) {
    const double waves = (double)((a.B + (int64_t)c->sm_count * g - 1) / ((int64_t)c->sm_count * g));
    const double t = waves * kStep[g];
    if (t < best * 0.999) {
      best = t;
      gc = g;
    }
  }
  if (c->br_gc > 0) gc = c->br_gc > 3 ? 3 : c->br_gc;
  if (c->margin) {
    if (gc == 3) return launch_v5_g<3, true>(c, a);
    if (gc == 2) return launch_v5_g<2, true>(c, a);
    return launch_v5_g<1, true>(c, a);
  }
  if (gc == 3) return launch_v5_g<3>(c, a);
  if (gc == 2) return launch_v5_g<2>(c, a);
  return launch_v5_g<1>(c, a);
}

// v5 applies at N = 1024, l = 2 when every convolution coefficient with the
// full 32-bit key word stays within 2^51 (the round_mod32 range): PARAM_128 / PARAM_110.
bool v5_ok(const gw_ctx* c) {
  return c->logn == 10 && c->p.l == 2 && std::log2(2.0 * c->p.l) + c->logn + (c->p.bg_bits - 1) + 31 <= 51.0 + 1e-9;
}

template <int LOGN>
int launch_br_n(gw_ctx* c, const BrArgs& a) {
  if (LOGN == 10 && c->p.l == 2 && c->br_variant == 2 && !c->br_exact && c->bk_v5) return launch_v5(c, a);
  if (LOGN == 10 && c->p.l == 2 && c->br_variant == 2 && c->bk_v3) return launch_v3(c, a);
  switch (c->p.l) {
    case 1: return c->br_variant ? launch_tm<LOGN, 1>(c, a) : launch_br_t<LOGN, 1>(c, a);
    case 2: return c->br_variant ? launch_tm<LOGN, 2>(c, a) : launch_br_t<LOGN, 2>(c, a);
    case 3: return launch_br_t<LOGN, 3>(c, a);
  }
  return fail(c, GW_ERR_PARAM, "gadget levels outside 1..3");
}

int launch_br(gw_ctx* c, const BrArgs& a) {
  switch (c->logn) {
    case 6: return launch_br_n<6>(c, a);
    case 8: return launch_br_n<8>(c, a);
    case 10: return launch_br_n<10>(c, a);
  }
  return fail(c, GW_ERR_PARAM, "ring dimension not supported");
}

template <int LOGN, int LEV>
int launch_bk_t(gw_ctx* c, const uint32_t* bk_dev) {
  const long long jobs = (long long)c->p.n * 2 * LEV * 4;
  const int grid = (int)((jobs + 3) / 4);
  k_bk_to_fft<LOGN, LEV><<<grid, 128, 0, c->stream>>>(bk_dev, c->p.n, c->tables, c->bk_fft);
  GW_LAUNCHED(c);
  return GW_OK;
}

template <int LOGN>
int launch_bk_n(gw_ctx* c, const uint32_t* bk) {
  switch (c->p.l) {
    case 1: return launch_bk_t<LOGN, 1>(c, bk);
    case 2: return launch_bk_t<LOGN, 2>(c, bk);
    case 3: return launch_bk_t<LOGN, 3>(c, bk);
  }
  return fail(c, GW_ERR_PARAM, "gadget levels outside 1..3");
}

int launch_bk(gw_ctx* c, const uint32_t* bk) {
  switch (c->logn) {
    case 6: return launch_bk_n<6>(c, bk);
    case 8: return launch_bk_n<8>(c, bk);
    case 10: return launch_bk_n<10>(c, bk);
  }
  return fail(c, GW_ERR_PARAM, "ring dimension not supported");
}

constexpr int KS_GT = 16;

int launch_ks(gw_ctx* c, const uint32_t* acc, const KsUnit* units, int U, uint32_t* out, int64_t out_stride) {
  if (U <= 0) return GW_OK;
  const int N = c->p.N, W = c->p.n + 1;
  if (!(c->ks_tc && c->ks_variant)) {  // the tensor-core path zeroes in k_ks_prep
    dim3 grid((W + 255) / 256, grid_rows(U));
    k_zero_units<<<grid, 256, 0, c->stream>>>(units, U, out, out_stride, W);
    GW_LAUNCHED(c);
  }
  if (c->ks_tc && c->ks_variant) {
    const int N = c->p.N;
    const size_t ut_stride = ((size_t)U + 31) & ~(size_t)31;
    int rc = ensure(c, &c->ks_ut, &c->ks_ut_cap, ut_stride * N + ut_stride, sizeof(uint32_t));
    if (rc) return rc;
    uint32_t* body = c->ks_ut + ut_stride * N;
    {
      dim3 grid((U + 127) / 128, N);
      k_ks_prep<<<grid, 128, 0, c->stream>>>(acc, units, U, N, c->p.ks_levels * c->p.ks_base_bits, c->ks_ut,
                                             (int64_t)ut_stride, body, out, out_stride, W);
      GW_LAUNCHED(c);
    }
    KtArgs k;
    k.ut = c->ks_ut;
    k.ut_stride = (int64_t)ut_stride;
    k.body = body;
    k.units = units;
    k.count = U;
    k.kimg = c->kimg;
    k.kblocks = c->kt_kblocks;
    k.t = c->p.ks_levels;
    k.gamma = c->p.ks_base_bits;
    k.W = W;
    k.out = out;
    k.out_stride = out_stride;
    const int mt = (U + KT_M - 1) / KT_M;
    int splits = c->sm_count / (mt * c->kt_ntiles);
    if (splits < 1) splits = 1;
    if (splits > c->kt_kblocks) splits = c->kt_kblocks;
    k.blocks_per_split = (c->kt_kblocks + splits - 1) / splits;
    splits = (c->kt_kblocks + k.blocks_per_split - 1) / k.blocks_per_split;
    const size_t smem = (size_t)KT_STAGES * (KT_A_BYTES + KT_B_BYTES) + 256;
    dim3 grid(mt, c->kt_ntiles, splits);
    auto go = [&](auto kern) -> int {
      if (int rc = set_smem(c, kern, smem)) return rc;
      kern<<<grid, KT_THREADS, smem, c->stream>>>(k);
      GW_LAUNCHED(c);
      return GW_OK;
    };
    switch (c->p.ks_levels) {
      case 1: return go(k_keyswitch_tc<1>);
      case 2: return go(k_keyswitch_tc<2>);
      case 4: return go(k_keyswitch_tc<4>);
      case 8: return go(k_keyswitch_tc<8>);
      case 16: return go(k_keyswitch_tc<16>);
      case 32: return go(k_keyswitch_tc<32>);
    }
    return fail(c, GW_ERR_PARAM, "tensor-core keyswitch needs t | 32");
  }
  KsArgs a;
  a.acc = acc;
  a.units = units;
  a.count = U;
  a.ksk = c->ksk;
  a.N = N;
  a.t = c->p.ks_levels;
  a.gamma = c->p.ks_base_bits;
  a.W = W;
  a.Wp = c->Wp;
  a.chunk = N < 64 ? N : 64;
  a.out = out;
  a.out_stride = out_stride;
  const int threads = ((c->Wp / 4) + 31) / 32 * 32;
  if (threads > 160) return fail(c, GW_ERR_PARAM, "LWE dimension too large for the keyswitch tile");
  dim3 grid((U + KS_GT - 1) / KS_GT, (N + a.chunk - 1) / a.chunk);
  const size_t smem = sizeof(uint32_t) * KS_GT * a.chunk;
  const int V = (1 << a.gamma) - 1;
  if (V == 3) k_keyswitch<KS_GT, 3><<<grid, threads, smem, c->stream>>>(a);
  else if (V == 1) k_keyswitch<KS_GT, 1><<<grid, threads, smem, c->stream>>>(a);
  else k_keyswitch<KS_GT, 0><<<grid, threads, smem, c->stream>>>(a);
  GW_LAUNCHED(c);
  return GW_OK;
}

int launch_lin(gw_ctx* c, const uint32_t* rows, int64_t stride, const LinJob* jobs, int J) {
  if (J <= 0) return GW_OK;
  const int W = c->p.n + 1;
  dim3 grid((W + 255) / 256, grid_rows(J));
  k_lin<<<grid, 256, 0, c->stream>>>(rows, stride, jobs, J, W, c->p.mu, c->lin, c->Wp);
  GW_LAUNCHED(c);
  return GW_OK;
}

int launch_cheap(gw_ctx* c, const uint32_t* src, int64_t src_stride, const CheapUnit* units, int C,
                 uint32_t* dst, int64_t dst_stride) {
  if (C <= 0) return GW_OK;
  const int W = c->p.n + 1;
  dim3 grid((W + 255) / 256, grid_rows(C));
  k_cheap<<<grid, 256, 0, c->stream>>>(src, src_stride, units, C, W, c->p.mu, dst, dst_stride);
  GW_LAUNCHED(c);
  return GW_OK;
}

cudaEvent_t pooled_event(gw_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// Stage bracket: records an event pair around `body` when profiling is on.
template <typename F>
int staged(gw_ctx* c, int stage, int64_t items, F&& body) {
  if (!c->profile) return body();
  cudaEvent_t a = pooled_event(c), b = pooled_event(c);
  cudaEventRecord(a, c->stream);
  int rc = body();
  cudaEventRecord(b, c->stream);
  c->prof_ev[stage].emplace_back(a, b);
  c->prof_items[stage] += items;
  return rc;
}

int ready(gw_ctx* c, bool need_bk = true, bool need_ksk = true) {
  if (!c) return GW_ERR_ARG;
  if (!c->have_params) return fail(c, GW_ERR_STATE, "parameters not set");
  if (need_bk && !c->have_bk) return fail(c, GW_ERR_STATE, "bootstrapping key not uploaded");
  if (need_ksk && !c->have_ksk) return fail(c, GW_ERR_STATE, "keyswitch key not uploaded");
  return GW_OK;
}

// One level over a row space: jobs/units/cheap are DEVICE descriptor arrays.
int run_level(gw_ctx* c, const uint32_t* src, int64_t src_stride, uint32_t* dst, int64_t dst_stride,
              const LinJob* jobs, int J, const KsUnit* units, int U, const CheapUnit* cheap, int C) {
  int rc;
  if (J > 0) {
    // v3 computes each bootstrap's linear combination in its prologue (fused
    // k_lin); the other kernels read materialised rows
    const bool fused = c->logn == 10 && c->p.l == 2 && c->br_variant == 2 && c->bk_v3 && !c->br_unfused;
    if ((rc = ensure(c, &c->acc, &c->acc_cap, (size_t)J * 2 * c->p.N, sizeof(uint32_t)))) return rc;
    if (!fused) {
      if ((rc = ensure(c, &c->lin, &c->lin_cap, (size_t)J * c->Wp, sizeof(uint32_t)))) return rc;
      if ((rc = staged(c, 2, 0, [&] { return launch_lin(c, src, src_stride, jobs, J); }))) return rc;
    }
    BrArgs a;
    if (fused) {
      a.jobs = jobs;
      a.rows = src;
      a.row_stride = src_stride;
      a.mu = c->p.mu;
    }
    a.lin = c->lin;
    a.lin_stride = c->Wp;
    a.B = J;
    a.n = c->p.n;
    a.tv = c->tv_dev;
    a.bk = c->bk_fft;
    a.tables = c->tables;
    a.acc_out = c->acc;
    a.bg_bits = c->p.bg_bits;
    uint64_t off = 1ull << (32 - c->p.l * c->p.bg_bits - 1);
    for (int j = 1; j <= c->p.l; ++j) off += (uint64_t)(1u << (c->p.bg_bits - 1)) << (32 - j * c->p.bg_bits);
    a.offs = (uint32_t)(off & 0xFFFFFFFFull);
    a.gates_per_cta = 1;
    a.prof = c->br_prof;
    a.ablate = c->br_ablate;
    // wide launches only: with a few CTAs each would prefetch megabytes, and the narrow
    // levels of config 2 measured 10 % slower with it (profiles/r02_keyswitch_ab.txt)
    if (c->ks_l2warm && c->ks_tc && c->ks_variant && c->kimg && J >= c->sm_count) {
      a.l2warm = reinterpret_cast<const char*>(c->kimg);
      a.l2warm_bytes = c->kimg_bytes;
    }
    if ((rc = staged(c, 0, J, [&] { return launch_br(c, a); }))) return rc;
    if ((rc = staged(c, 1, U, [&] { return launch_ks(c, c->acc, units, U, dst, dst_stride); }))) return rc;
  }
  if ((rc = staged(c, 2, 0, [&] { return launch_cheap(c, src, src_stride, cheap, C, dst, dst_stride); })))
    return rc;
  return GW_OK;
}

// Host-side descriptors for one gate (cggi.py:816-852 semantics).
void describe_gate(int op, int32_t s0, int32_t s1, int32_t s2, int32_t out, uint32_t mu,
                   std::vector<LinJob>& jobs, std::vector<KsUnit>& units, std::vector<CheapUnit>& cheap) {
  static const int combo[6][3] = {{-1, 1, 1}, {1, 1, 1}, {1, -1, -1}, {-1, -1, -1}, {2, 2, 2}, {-2, -2, -2}};
  if (op <= GW_XNOR) {
    LinJob j{};
    j.src[0] = s0; j.src[1] = s1;
    j.w[0] = combo[op][1]; j.w[1] = combo[op][2];
    j.cmu = combo[op][0];
    const int idx = (int)jobs.size();
    jobs.push_back(j);
    units.push_back(KsUnit{idx, -1, out, 0u});
  } else if (op == GW_BOOTSTRAP) {
    LinJob j{};
    j.src[0] = s0; j.src[1] = -1; j.w[0] = 1; j.w[1] = 0; j.cmu = 0;
    const int idx = (int)jobs.size();
    jobs.push_back(j);
    units.push_back(KsUnit{idx, -1, out, 0u});
  } else if (op == GW_MUX) {
    LinJob j1{}, j2{};
    j1.src[0] = s0; j1.src[1] = s1; j1.w[0] = 1; j1.w[1] = 1; j1.cmu = -1;   // sel + a - mu
    j2.src[0] = s2; j2.src[1] = s0; j2.w[0] = 1; j2.w[1] = -1; j2.cmu = -1;  // b - sel - mu
    const int idx = (int)jobs.size();
    jobs.push_back(j1);
    jobs.push_back(j2);
    units.push_back(KsUnit{idx, idx + 1, out, mu});  // pre.b += mu (cggi.py:845)
  } else {
    CheapUnit u{};
    u.kind = op == GW_COPY ? 0 : op == GW_NOT ? 1 : op == GW_CONST0 ? 2 : 3;
    u.src = s0;
    u.dst = out;
    cheap.push_back(u);
  }
}

int arity_of(int op) {
  if (op <= GW_XNOR) return 2;
  if (op == GW_NOT || op == GW_COPY || op == GW_BOOTSTRAP) return 1;
  if (op == GW_MUX) return 3;
  if (op == GW_CONST0 || op == GW_CONST1) return 0;
  return -1;
}

// Upload host descriptor vectors into the device descriptor arena.
int upload_desc(gw_ctx* c, const std::vector<LinJob>& jobs, const std::vector<KsUnit>& units,
                const std::vector<CheapUnit>& cheap, LinJob** dj, KsUnit** du, CheapUnit** dc) {
  const size_t bj = jobs.size() * sizeof(LinJob), bu = units.size() * sizeof(KsUnit),
               bc = cheap.size() * sizeof(CheapUnit);
  const size_t total = bj + bu + bc;
  int rc;
  // the pinned staging buffer may still feed the previous async copy: wait for
  // that copy only (an event), not for the whole stream
  if (c->desc_copied) GW_CUDA(c, cudaEventSynchronize(c->desc_copied));
  if ((rc = ensure_desc(c, total))) return rc;
  char* h = (char*)c->desc_host;
  if (bj) memcpy(h, jobs.data(), bj);
  if (bu) memcpy(h + bj, units.data(), bu);
  if (bc) memcpy(h + bj + bu, cheap.data(), bc);
  GW_CUDA(c, cudaMemcpyAsync(c->desc, h, total, cudaMemcpyHostToDevice, c->stream));
  if (!c->desc_copied) GW_CUDA(c, cudaEventCreateWithFlags(&c->desc_copied, cudaEventDisableTiming));
  GW_CUDA(c, cudaEventRecord(c->desc_copied, c->stream));
  char* d = (char*)c->desc;
  *dj = (LinJob*)d;
  *du = (KsUnit*)(d + bj);
  *dc = (CheapUnit*)(d + bj + bu);
  return GW_OK;
}

}  // namespace

namespace {
// libnccl is bound at run time (dlopen) so the engine has no link-time NCCL
// dependency: the one torch already loaded when present, else the system's.
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};
std::mutex g_nccl_mtx;
NcclApi g_nccl;

const NcclApi& nccl_api() {
  std::lock_guard<std::mutex> lk(g_nccl_mtx);
  if (g_nccl.tried) return g_nccl;
  g_nccl.tried = true;
  void* h = nullptr;
  if (const char* p = getenv("GATEWAVE_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already in the process (torch)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_nccl.why = std::string("libnccl.so.2 not found: ") + dlerror();
    return g_nccl;
  }
  bool ok = true;
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn) ok = false;
  };
  sym(g_nccl.GetUniqueId, "ncclGetUniqueId");
  sym(g_nccl.CommInitRank, "ncclCommInitRank");
  sym(g_nccl.CommDestroy, "ncclCommDestroy");
  sym(g_nccl.Send, "ncclSend");
  sym(g_nccl.Recv, "ncclRecv");
  sym(g_nccl.GroupStart, "ncclGroupStart");
  sym(g_nccl.GroupEnd, "ncclGroupEnd");
  sym(g_nccl.GetErrorString, "ncclGetErrorString");
  sym(g_nccl.GetVersion, "ncclGetVersion");
  g_nccl.ok = ok;
  if (!ok) g_nccl.why = "libnccl.so.2 lacks a required symbol";
  return g_nccl;
}

#define GW_NCCL(ctx, api, expr)                                                                   \
  do {                                                                                            \
    ncclResult_t r_ = (expr);                                                                     \
    if (r_ != ncclSuccess) return fail((ctx), GW_ERR_CUDA, std::string(#expr) + ": " + (api).GetErrorString(r_)); \
  } while (0)
}  // namespace

// ============================================================================
extern "C" {

int gw_version(void) { return 1; }

int gw_levels(const int64_t* pos, int64_t gates, int32_t* level) {
  if (gates < 0 || (gates > 0 && (!pos || !level))) return GW_ERR_ARG;
  for (int64_t k = 0; k < gates; ++k) {
    int32_t m = -1;
    for (int j = 0; j < 3; ++j) {
      const int64_t p = pos[3 * k + j];
      if (p < 0) continue;
      if (p >= k) return GW_ERR_ARG;
      if (level[p] > m) m = level[p];
    }
    level[k] = m + 1;
  }
  return GW_OK;
}

int gw_device_count(int* count) {
  if (!count) return GW_ERR_ARG;
  if (cudaGetDeviceCount(count) != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
  }
  return GW_OK;
}

int gw_create(int device, gw_ctx** out) {
  if (!out) return GW_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return GW_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) return GW_ERR_ARG;
  gw_ctx* c = new gw_ctx();
  c->device = device;
  int rc = GW_OK;
  if (cudaSetDevice(device) != cudaSuccess) rc = GW_ERR_CUDA;
  if (!rc && cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) rc = GW_ERR_CUDA;
  c->own_stream = true;
  if (!rc) cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (!rc && (cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess)) rc = GW_ERR_CUDA;
  if (!rc) rc = upload_roots(c);
  if (const char* v = getenv("GATEWAVE_BR_GC")) c->br_gc = atoi(v);
  if (const char* v = getenv("GATEWAVE_BR_GC1")) c->br_gc1_tma = strcmp(v, "tma") == 0;
  if (const char* v = getenv("GATEWAVE_BR_LDR")) c->br_ldr = atoi(v) != 0;
  if (const char* v = getenv("GATEWAVE_BR_UNFUSED")) c->br_unfused = atoi(v) != 0;
  if (const char* v = getenv("GATEWAVE_BR_EXACT")) c->br_exact = atoi(v) != 0;
  if (const char* v = getenv("GATEWAVE_KS_L2WARM")) c->ks_l2warm = atoi(v) != 0;

  if (const char* v = getenv("GATEWAVE_BR_KERNEL"))
    c->br_variant = strcmp(v, "v1") == 0 ? 0 : strcmp(v, "v2") == 0 ? 1 : 2;
  if (const char* v = getenv("GATEWAVE_KS_KERNEL")) c->ks_variant = strcmp(v, "cuda") == 0 ? 0 : 1;
  if (const char* v = getenv("GATEWAVE_BR_ABLATE")) c->br_ablate = atoi(v);
  if (const char* v = getenv("GATEWAVE_BR_PROFILE"))
    if (strcmp(v, "1") == 0 && cudaMalloc(&c->br_prof, 64 * sizeof(long long)) == cudaSuccess)
      cudaMemset(c->br_prof, 0, 64 * sizeof(long long));
  if (rc) {
    gw_destroy(c);
    return rc;
  }
  *out = c;
  return GW_OK;
}

int gw_destroy(gw_ctx* c) {
  if (!c) return GW_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->bk_fft);
  cudaFree(c->bk_v3);
  cudaFree(c->bk_v5);
  cudaFree(c->ksk);
  cudaFree(c->kimg);
  cudaFree(c->ks_ut);
  cudaFree(c->br_prof);
  cudaFree(c->margin);
  cudaFree(c->tables);
  cudaFree(c->tv_dev);
  cudaFree(c->lin);
  cudaFree(c->acc);
  cudaFree(c->io);
  cudaFree(c->desc);
  if (c->wires_owned) cudaFree(c->wires);
  for (auto& kv : c->batch_desc) cudaFree(kv.second.mem);
  if (c->desc_host) cudaFreeHost(c->desc_host);
  for (auto& v : c->prof_ev)
    for (auto& pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  for (auto e : c->marks) cudaEventDestroy(e);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->nccl) {
    const NcclApi& api = nccl_api();
    if (api.ok) api.CommDestroy((ncclComm_t)c->nccl);
  }
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->desc_copied) cudaEventDestroy(c->desc_copied);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return GW_OK;
}

const char* gw_last_error(const gw_ctx* c) { return c ? c->err.c_str() : "null context"; }

int gw_set_stream(gw_ctx* c, void* s) {
  if (!c) return GW_ERR_ARG;
  cudaSetDevice(c->device);
  if (c->stream) GW_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (s) {
    c->stream = (cudaStream_t)s;
    c->own_stream = false;
  } else {
    GW_CUDA(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  return GW_OK;
}

int gw_sync(gw_ctx* c) {
  if (!c) return GW_ERR_ARG;
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

int gw_set_params(gw_ctx* c, const gw_params* p) {
  if (!c || !p) return GW_ERR_ARG;
  // ParamSet.__post_init__ (cggi.py:86-110)
  if (p->n < 1) return fail(c, GW_ERR_PARAM, "LWE dimension must be positive");
  if (p->N < 2 || (p->N & (p->N - 1))) return fail(c, GW_ERR_PARAM, "ring dimension must be a power of two >= 2");
  if (!(p->bg_bits >= 1 && p->l >= 1 && p->l * p->bg_bits <= 32))
    return fail(c, GW_ERR_PARAM, "gadget levels * base bits must fit 32 bits");
  const int logn = ilog2(p->N);
  if (logn + p->bg_bits > 32) return fail(c, GW_ERR_PARAM, "gadget digits too wide for exact convolution");
  if (!(p->ks_base_bits >= 1 && p->ks_levels >= 1 && p->ks_levels * p->ks_base_bits <= 32))
    return fail(c, GW_ERR_PARAM, "keyswitch levels * base bits must fit 32 bits");
  if (p->mu == 0) return fail(c, GW_ERR_PARAM, "mu must be a nonzero uint32");
  // Engine envelope: warp-FFT geometry and FP64 exactness.
  if (!(logn == 6 || logn == 8 || logn == 10))
    return fail(c, GW_ERR_PARAM, "ring dimension not supported by the B200 engine (64, 256, 1024)");
  if (p->l > 3) return fail(c, GW_ERR_PARAM, "gadget levels > 3 not supported by the B200 engine");
  if (p->bg_bits > 16) return fail(c, GW_ERR_PARAM, "gadget base > 2^16 not supported by the B200 engine");
  // |coefficient| <= 2l * N * 2^(Bg-1) * 2^15 must stay <= 2^36: the largest
  // magnitude whose rounding margin is measured (Bg = 10, l = 2, N = 1024:
  // tests/test_gpu_margin.py); PARAM_128 / PARAM_110 sit at 2^35
  if (std::log2(2.0 * p->l) + logn + (p->bg_bits - 1) + 15 > 36.0 + 1e-9)
    return fail(c, GW_ERR_PARAM, "parameters outside the exact FP64 convolution envelope");
  if (p->ks_levels * p->ks_base_bits > 31)
    return fail(c, GW_ERR_PARAM, "keyswitch precision t*gamma > 31 not supported by the B200 engine");
  if (((p->n + 1 + 3) / 4) > 160) return fail(c, GW_ERR_PARAM, "LWE dimension > 639 not supported by the B200 engine");
  const bool same = c->have_params && memcmp(&c->p, p, sizeof(gw_params)) == 0;
  c->p = *p;
  c->logn = logn;
  c->Wp = (p->n + 1 + 3) & ~3;
  c->have_params = true;
  cudaSetDevice(c->device);
  if (!same) {
    c->have_keys = c->have_bk = c->have_ksk = false;
    // cached gate-batch descriptors carry mu (MUX units): drop them
    if (!c->batch_desc.empty()) {
      GW_CUDA(c, cudaStreamSynchronize(c->stream));
      for (auto& kv : c->batch_desc) cudaFree(kv.second.mem);
      c->batch_desc.clear();
    }
  }
  // tables + default test vector (cggi.py:712-713: a = 0, b = mu)
  std::vector<double2> t;
  host_tables(logn, t);
  cudaFree(c->tables);
  c->tables = nullptr;
  GW_CUDA(c, cudaMalloc(&c->tables, t.size() * sizeof(double2)));
  GW_CUDA(c, cudaMemcpy(c->tables, t.data(), t.size() * sizeof(double2), cudaMemcpyHostToDevice));
  std::vector<uint32_t> tv(2 * p->N, 0u);
  for (int j = 0; j < p->N; ++j) tv[p->N + j] = p->mu;
  cudaFree(c->tv_dev);
  c->tv_dev = nullptr;
  GW_CUDA(c, cudaMalloc(&c->tv_dev, tv.size() * sizeof(uint32_t)));
  GW_CUDA(c, cudaMemcpy(c->tv_dev, tv.data(), tv.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  return GW_OK;
}

int gw_upload_keys(gw_ctx* c, const uint32_t* bk_coeff, const uint32_t* ksk) {
  if (!c || (!bk_coeff && !ksk)) return GW_ERR_ARG;
  if (!c->have_params) return fail(c, GW_ERR_STATE, "parameters not set");
  cudaSetDevice(c->device);
  const int n = c->p.n, N = c->p.N, l = c->p.l, t = c->p.ks_levels, V = (1 << c->p.ks_base_bits) - 1;
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  if (bk_coeff) {
    c->have_bk = false;
    const size_t bk_words = (size_t)n * 2 * l * 2 * N;
    // bootstrapping key: upload coefficient domain, transform on device
    uint32_t* bk_dev = nullptr;
    GW_CUDA(c, cudaMalloc(&bk_dev, bk_words * sizeof(uint32_t)));
    cudaError_t e = cudaMemcpyAsync(bk_dev, bk_coeff, bk_words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream);
    if (e != cudaSuccess) {
      cudaFree(bk_dev);
      return fail(c, GW_ERR_CUDA, cudaGetErrorString(e));
    }
    const size_t nfft = (size_t)n * 2 * (2 * l) * 2 * (N / 2);
    if (c->bk_fft_count != nfft) {
      cudaFree(c->bk_fft);
      c->bk_fft = nullptr;
      c->bk_fft_count = 0;
      e = cudaMalloc(&c->bk_fft, nfft * sizeof(double2));
      if (e != cudaSuccess) {
        cudaFree(bk_dev);
        return fail(c, GW_ERR_CUDA, cudaGetErrorString(e));
      }
      c->bk_fft_count = nfft;
    }
    int rc = launch_bk(c, bk_dev);
    cudaFree(c->bk_v3);
    c->bk_v3 = nullptr;
    if (rc == GW_OK && c->logn == 10 && l == 2) {
      const size_t cnt = (size_t)n * V3::CIDX * 128;
      e = cudaMalloc(&c->bk_v3, cnt * sizeof(double2));
      if (e == cudaSuccess) {
        const long long jobs = (long long)n * 2 * l * 4;
        k_bk_to_v3<<<(unsigned)((jobs + 3) / 4), 128, 0, c->stream>>>(bk_dev, n, c->tables, c->bk_v3);
        e = cudaGetLastError();
        if (e == cudaSuccess) c->launches++;
      }
      if (e != cudaSuccess) rc = fail(c, GW_ERR_CUDA, std::string("v3 key image: ") + cudaGetErrorString(e));
    }
    cudaFree(c->bk_v5);
    c->bk_v5 = nullptr;
    if (rc == GW_OK && v5_ok(c)) {
      const size_t cnt = (size_t)n * V5::CIDX * 128;
      e = cudaMalloc(&c->bk_v5, cnt * sizeof(double2));
      if (e == cudaSuccess) {
        const long long jobs = (long long)n * 2 * l * 2;
        k_bk_to_v5<<<(unsigned)((jobs + 3) / 4), 128, 0, c->stream>>>(bk_dev, n, c->tables, c->bk_v5);
        e = cudaGetLastError();
        if (e == cudaSuccess) c->launches++;
      }
      if (e != cudaSuccess) rc = fail(c, GW_ERR_CUDA, std::string("v5 key image: ") + cudaGetErrorString(e));
    }


    cudaError_t es = cudaStreamSynchronize(c->stream);
    cudaFree(bk_dev);
    if (rc) return rc;
    if (es != cudaSuccess) return fail(c, GW_ERR_CUDA, cudaGetErrorString(es));
    c->have_bk = true;
  }
  if (ksk) {
    c->have_ksk = false;
    // keyswitch key: (N, t, V, n+1) -> padded rows of Wp words
    const size_t rows = (size_t)N * t * V;
    cudaFree(c->ksk);
    c->ksk = nullptr;
    GW_CUDA(c, cudaMalloc(&c->ksk, rows * c->Wp * sizeof(uint32_t)));
    GW_CUDA(c, cudaMemsetAsync(c->ksk, 0, rows * c->Wp * sizeof(uint32_t), c->stream));
    GW_CUDA(c, cudaMemcpy2DAsync(c->ksk, c->Wp * sizeof(uint32_t), ksk, (n + 1) * sizeof(uint32_t),
                                 (n + 1) * sizeof(uint32_t), rows, cudaMemcpyHostToDevice, c->stream));
    // tensor-core image: needs t | 32 (whole digit groups per K block), <= 3 nonzero digits
    cudaFree(c->kimg);
    c->kimg = nullptr;
    c->ks_tc = (32 % t == 0) && V <= 3 && ((size_t)N * t) % KT_PAIRS == 0;
    if (c->ks_tc) {
      c->kt_ntiles = (n + 1 + KT_COLS - 1) / KT_COLS;
      c->kt_kblocks = (int)((size_t)N * t / KT_PAIRS);
      const size_t bytes = (size_t)c->kt_ntiles * c->kt_kblocks * KT_B_BYTES;
      GW_CUDA(c, cudaMalloc(&c->kimg, bytes));
      c->kimg_bytes = bytes;
      const size_t chunks = bytes / 16;
      k_ksk_to_tc<<<(unsigned)((chunks + 255) / 256), 256, 0, c->stream>>>(c->ksk, N, t, V, n + 1, c->Wp,
                                                                           c->kt_ntiles, c->kt_kblocks, c->kimg);
      GW_LAUNCHED(c);
    }
    GW_CUDA(c, cudaStreamSynchronize(c->stream));
    c->have_ksk = true;
  }
  c->have_keys = c->have_bk && c->have_ksk;
  return GW_OK;
}

int gw_bk_fft_size(gw_ctx* c, int64_t* n_complex) {
  if (!c || !n_complex) return GW_ERR_ARG;
  if (!c->have_bk) return fail(c, GW_ERR_STATE, "bootstrapping key not uploaded");
  *n_complex = (int64_t)c->bk_fft_count;
  return GW_OK;
}

int gw_download_bk_fft(gw_ctx* c, double* out) {
  if (!c || !out) return GW_ERR_ARG;
  if (!c->have_bk) return fail(c, GW_ERR_STATE, "bootstrapping key not uploaded");
  cudaSetDevice(c->device);
  GW_CUDA(c, cudaMemcpyAsync(out, c->bk_fft, c->bk_fft_count * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

int gw_blind_rotate(gw_ctx* c, const uint32_t* lin, int64_t B, const uint32_t* tv, uint32_t* acc) {
  int rc = ready(c, true, false);
  if (rc) return rc;
  if (B < 0 || (B > 0 && (!lin || !tv || !acc))) return fail(c, GW_ERR_ARG, "null buffer");
  if (B == 0) return GW_OK;
  if (B > (1 << 30)) return fail(c, GW_ERR_ARG, "batch too large");
  cudaSetDevice(c->device);
  const int n = c->p.n, N = c->p.N;
  // io: lin rows (Wp stride) + tv
  const size_t need = (size_t)B * c->Wp + 2 * N;
  if ((rc = ensure(c, &c->io, &c->io_cap, need, sizeof(uint32_t)))) return rc;
  if ((rc = ensure(c, &c->acc, &c->acc_cap, (size_t)B * 2 * N, sizeof(uint32_t)))) return rc;
  uint32_t* dlin = c->io;
  uint32_t* dtv = c->io + (size_t)B * c->Wp;
  GW_CUDA(c, cudaMemcpy2DAsync(dlin, c->Wp * sizeof(uint32_t), lin, (n + 1) * sizeof(uint32_t),
                               (n + 1) * sizeof(uint32_t), B, cudaMemcpyHostToDevice, c->stream));
  GW_CUDA(c, cudaMemcpyAsync(dtv, tv, 2 * N * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  BrArgs a;
  a.lin = dlin;
  a.lin_stride = c->Wp;
  a.B = (int)B;
  a.n = n;
  a.tv = dtv;
  a.bk = c->bk_fft;
  a.tables = c->tables;
  a.acc_out = c->acc;
  a.bg_bits = c->p.bg_bits;
  uint64_t off = 1ull << (32 - c->p.l * c->p.bg_bits - 1);
  for (int j = 1; j <= c->p.l; ++j) off += (uint64_t)(1u << (c->p.bg_bits - 1)) << (32 - j * c->p.bg_bits);
  a.offs = (uint32_t)(off & 0xFFFFFFFFull);
  a.gates_per_cta = 1;
  a.prof = c->br_prof;
  a.ablate = c->br_ablate;
  if ((rc = launch_br(c, a))) return rc;
  GW_CUDA(c, cudaMemcpyAsync(acc, c->acc, (size_t)B * 2 * N * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

int gw_keyswitch(gw_ctx* c, const uint32_t* ext, int64_t B, uint32_t* out) {
  int rc = ready(c, false, true);
  if (rc) return rc;
  if (B < 0 || (B > 0 && (!ext || !out))) return fail(c, GW_ERR_ARG, "null buffer");
  if (B == 0) return GW_OK;
  cudaSetDevice(c->device);
  const int N = c->p.N, W = c->p.n + 1;
  const size_t ext_words = (size_t)B * (N + 1);
  const size_t need = ext_words + (size_t)B * c->Wp;
  if ((rc = ensure(c, &c->io, &c->io_cap, need, sizeof(uint32_t)))) return rc;
  if ((rc = ensure(c, &c->acc, &c->acc_cap, (size_t)B * 2 * N, sizeof(uint32_t)))) return rc;
  uint32_t* dext = c->io;
  uint32_t* dout = c->io + ext_words;
  GW_CUDA(c, cudaMemcpyAsync(dext, ext, ext_words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  {
    dim3 grid((2 * N + 255) / 256, grid_rows(B));
    k_ext_to_acc<<<grid, 256, 0, c->stream>>>(dext, B, N, c->acc);
    GW_LAUNCHED(c);
  }
  std::vector<LinJob> jobs;
  std::vector<KsUnit> units((size_t)B);
  std::vector<CheapUnit> cheap;
  for (int64_t g = 0; g < B; ++g) units[g] = KsUnit{(int32_t)g, -1, (int32_t)g, 0u};
  LinJob* dj;
  KsUnit* du;
  CheapUnit* dc;
  if ((rc = upload_desc(c, jobs, units, cheap, &dj, &du, &dc))) return rc;
  if ((rc = launch_ks(c, c->acc, du, (int)B, dout, c->Wp))) return rc;
  GW_CUDA(c, cudaMemcpy2DAsync(out, W * sizeof(uint32_t), dout, c->Wp * sizeof(uint32_t), W * sizeof(uint32_t), B,
                               cudaMemcpyDeviceToHost, c->stream));
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

// Gates per launch set of a homogeneous batch (the same cut as the level plans):
// whole waves of the blind rotation at 3 and 4 gates per CTA; bounds the
// scratch (lin rows + accumulators, ~130 MB) however large the batch.
constexpr int64_t kSegGates = 148 * 12 * 9;

static int eval_stacked(gw_ctx* c, int opcode, const uint32_t* stacked, int64_t in_stride, int arity, int64_t B,
                        uint32_t* d_out, int64_t out_stride) {
  for (int64_t g0 = 0; g0 < B; g0 += kSegGates) {
    const int64_t S = std::min<int64_t>(kSegGates, B - g0);
    // Descriptors of a homogeneous segment depend only on (opcode, S, B): cache
    // them on the device so repeated batches enqueue without any host round trip.
    // Operand k of gate g is stacked row k*B + g; the segment's rows are reached
    // by offsetting the base pointers by g0 rows.
    const uint64_t key = ((uint64_t)opcode << 56) | ((uint64_t)S << 28) | (uint64_t)B;
    auto it = c->batch_desc.find(key);
    if (it == c->batch_desc.end()) {
      std::vector<LinJob> jobs;
      std::vector<KsUnit> units;
      std::vector<CheapUnit> cheap;
      for (int64_t g = 0; g < S; ++g) {
        const int32_t s0 = arity > 0 ? (int32_t)g : -1;
        const int32_t s1 = arity > 1 ? (int32_t)(B + g) : -1;
        const int32_t s2 = arity > 2 ? (int32_t)(2 * B + g) : -1;
        describe_gate(opcode, s0, s1, s2, (int32_t)g, c->p.mu, jobs, units, cheap);
      }
      BatchDesc d;
      d.J = (int)jobs.size();
      d.U = (int)units.size();
      d.C = (int)cheap.size();
      const size_t bj = jobs.size() * sizeof(LinJob), bu = units.size() * sizeof(KsUnit),
                   bc = cheap.size() * sizeof(CheapUnit);
      if (c->batch_desc.size() > 64) {
        GW_CUDA(c, cudaStreamSynchronize(c->stream));
        for (auto& kv : c->batch_desc) cudaFree(kv.second.mem);
        c->batch_desc.clear();
      }
      GW_CUDA(c, cudaMalloc(&d.mem, bj + bu + bc + 16));
      char* m = (char*)d.mem;
      if (bj) GW_CUDA(c, cudaMemcpy(m, jobs.data(), bj, cudaMemcpyHostToDevice));
      if (bu) GW_CUDA(c, cudaMemcpy(m + bj, units.data(), bu, cudaMemcpyHostToDevice));
      if (bc) GW_CUDA(c, cudaMemcpy(m + bj + bu, cheap.data(), bc, cudaMemcpyHostToDevice));
      d.jobs = (LinJob*)m;
      d.units = (KsUnit*)(m + bj);
      d.cheap = (CheapUnit*)(m + bj + bu);
      it = c->batch_desc.emplace(key, d).first;
    }
    const BatchDesc& d = it->second;
    const uint32_t* src = stacked ? stacked + (size_t)g0 * in_stride : nullptr;
    int rc = run_level(c, src, in_stride, d_out + (size_t)g0 * out_stride, out_stride, d.jobs, d.J, d.units, d.U,
                       d.cheap, d.C);
    if (rc) return rc;
  }
  return GW_OK;
}

static int check_batch(gw_ctx* c, int opcode, int arity, int64_t B) {
  int rc = ready(c);
  if (rc) return rc;
  const int want = arity_of(opcode);
  if (want < 0) return fail(c, GW_ERR_ARG, "unknown opcode");
  if (arity != want) return fail(c, GW_ERR_DIM, "operand count does not match the gate arity");
  if (B < 0 || B > (1 << 26)) return fail(c, GW_ERR_ARG, "bad batch size");
  return GW_OK;
}

int gw_eval_gate_batch_device(gw_ctx* c, int opcode, const uint32_t* const* d_ops, int64_t in_stride, int arity,
                              int64_t B, uint32_t* d_out, int64_t out_stride) {
  int rc = check_batch(c, opcode, arity, B);
  if (rc) return rc;
  if (B == 0) return GW_OK;
  for (int k = 0; k < arity; ++k)
    if (!d_ops[k]) return fail(c, GW_ERR_ARG, "null operand");
  if (!d_out) return fail(c, GW_ERR_ARG, "null output");
  cudaSetDevice(c->device);
  const int W = c->p.n + 1;
  const uint32_t* stacked = nullptr;
  if (arity > 0) {
    // operands that already form one stacked (arity*B, Wp) block are used in place
    bool inplace = in_stride == c->Wp;
    for (int k = 1; k < arity && inplace; ++k) inplace = d_ops[k] == d_ops[0] + (size_t)k * B * c->Wp;
    if (inplace) {
      stacked = d_ops[0];
    } else {
      if ((rc = ensure(c, &c->io, &c->io_cap, (size_t)arity * B * c->Wp, sizeof(uint32_t)))) return rc;
      for (int k = 0; k < arity; ++k)
        GW_CUDA(c, cudaMemcpy2DAsync(c->io + (size_t)k * B * c->Wp, c->Wp * sizeof(uint32_t), d_ops[k],
                                     in_stride * sizeof(uint32_t), W * sizeof(uint32_t), B, cudaMemcpyDeviceToDevice,
                                     c->stream));
      stacked = c->io;
    }
  }
  return eval_stacked(c, opcode, stacked, c->Wp, arity, B, d_out, out_stride);
}

int gw_eval_gate_batch(gw_ctx* c, int opcode, const uint32_t* const* ops, int arity, int64_t B, uint32_t* out) {
  int rc = check_batch(c, opcode, arity, B);
  if (rc) return rc;
  if (B == 0) return GW_OK;
  for (int k = 0; k < arity; ++k)
    if (!ops[k]) return fail(c, GW_ERR_ARG, "null operand");
  if (!out) return fail(c, GW_ERR_ARG, "null output");
  cudaSetDevice(c->device);
  // Host rows are copied as they are (unpadded, stride W): one contiguous DMA per
  // operand and one for the result; the gate kernels take any row stride.
  const int W = c->p.n + 1;
  const size_t in_words = (size_t)arity * B * W;
  if ((rc = ensure(c, &c->io, &c->io_cap, in_words + (size_t)B * W, sizeof(uint32_t)))) return rc;
  for (int k = 0; k < arity; ++k)
    GW_CUDA(c, cudaMemcpyAsync(c->io + (size_t)k * B * W, ops[k], (size_t)B * W * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, c->stream));
  uint32_t* dout = c->io + in_words;
  if ((rc = eval_stacked(c, opcode, c->io, W, arity, B, dout, W))) return rc;
  GW_CUDA(c, cudaMemcpyAsync(out, dout, (size_t)B * W * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

// Owned wire stores are cached: a request that fits the allocated capacity reuses it, and
// releasing (slots = 0) keeps stores up to kWireKeepBytes (4 GB of the 180 GB: configs 2, 3
// and 5 stay resident; config 4's 30 GB store goes back to the driver).  cudaMalloc / cudaFree
// synchronise the device and were measured taking up to 0.8 s right after another
// process released GPU memory; a netlist evaluation allocates and releases its store
// every call (runtime.evaluate), so small stores must not go back to the driver.
constexpr size_t kWireKeepBytes = (size_t)4 << 30;

int gw_wires_alloc(gw_ctx* c, int64_t slots) {
  if (!c || slots < 0) return GW_ERR_ARG;
  if (!c->have_params) return fail(c, GW_ERR_STATE, "parameters not set");
  cudaSetDevice(c->device);
  const size_t row_bytes = (size_t)c->Wp * sizeof(uint32_t);
  if (c->wires_owned && c->wires && slots <= c->wires_cap &&
      (slots > 0 || (size_t)c->wires_cap * row_bytes <= kWireKeepBytes)) {
    c->wire_slots = slots;  // stream-ordered reuse: earlier work on the store precedes the memset
    if (slots) GW_CUDA(c, cudaMemsetAsync(c->wires, 0, (size_t)slots * row_bytes, c->stream));
    return GW_OK;
  }
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->wires_owned) cudaFree(c->wires);
  c->wires = nullptr;
  c->wire_slots = 0;
  c->wires_cap = 0;
  c->wires_owned = true;
  if (slots == 0) return GW_OK;
  GW_CUDA(c, cudaMalloc(&c->wires, (size_t)slots * row_bytes));
  GW_CUDA(c, cudaMemsetAsync(c->wires, 0, (size_t)slots * row_bytes, c->stream));
  c->wire_slots = slots;
  c->wires_cap = slots;
  return GW_OK;
}

int gw_wires_attach(gw_ctx* c, void* dev_ptr, int64_t slots, int64_t stride_words) {
  if (!c || slots < 0 || (slots > 0 && !dev_ptr)) return GW_ERR_ARG;
  if (!c->have_params) return fail(c, GW_ERR_STATE, "parameters not set");
  if (stride_words != c->Wp) return fail(c, GW_ERR_DIM, "wire rows must use the engine stride (n+1 rounded up to 4)");
  cudaSetDevice(c->device);
  if (slots > 0) {  // the kernels dereference it on this context's device: reject anything else
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, dev_ptr) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, GW_ERR_ARG, "wire store pointer is not CUDA memory");
    }
    if ((a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) || a.device != c->device)
      return fail(c, GW_ERR_ARG, "wire store must be device memory on GPU " + std::to_string(c->device));
  }
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->wires_owned) cudaFree(c->wires);
  c->wires = (uint32_t*)dev_ptr;
  c->wire_slots = slots;
  c->wires_cap = 0;
  c->wires_owned = false;
  return GW_OK;
}

int gw_wires_device_ptr(gw_ctx* c, void** ptr, int64_t* stride) {
  if (!c || !ptr || !stride) return GW_ERR_ARG;
  *ptr = c->wire_slots ? c->wires : nullptr;  // a released (cached) store is not handed out
  *stride = c->Wp;
  return GW_OK;
}

static int check_ids(gw_ctx* c, const int64_t* ids, int64_t count) {
  for (int64_t k = 0; k < count; ++k)
    if (ids[k] < 0 || ids[k] >= c->wire_slots) return fail(c, GW_ERR_WIRE, "wire id out of range: " + std::to_string(ids[k]));
  return GW_OK;
}

int gw_wires_put(gw_ctx* c, const int64_t* ids, const uint32_t* rows, int64_t count) {
  if (!c || count < 0 || (count > 0 && (!ids || !rows))) return GW_ERR_ARG;
  if (!c->wires || c->wire_slots == 0) return fail(c, GW_ERR_STATE, "wire store not allocated");
  int rc = check_ids(c, ids, count);
  if (rc) return rc;
  if (count == 0) return GW_OK;
  cudaSetDevice(c->device);
  const int W = c->p.n + 1;
  // stage contiguous rows, then scatter with a copy per contiguous id run
  int64_t k = 0;
  while (k < count) {
    int64_t run = 1;
    while (k + run < count && ids[k + run] == ids[k] + run) ++run;
    GW_CUDA(c, cudaMemcpy2DAsync(c->wires + (size_t)ids[k] * c->Wp, c->Wp * sizeof(uint32_t), rows + (size_t)k * W,
                                 W * sizeof(uint32_t), W * sizeof(uint32_t), run, cudaMemcpyHostToDevice, c->stream));
    k += run;
  }
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

int gw_wires_get(gw_ctx* c, const int64_t* ids, uint32_t* rows, int64_t count) {
  if (!c || count < 0 || (count > 0 && (!ids || !rows))) return GW_ERR_ARG;
  if (!c->wires || c->wire_slots == 0) return fail(c, GW_ERR_STATE, "wire store not allocated");
  int rc = check_ids(c, ids, count);
  if (rc) return rc;
  if (count == 0) return GW_OK;
  cudaSetDevice(c->device);
  const int W = c->p.n + 1;
  int64_t k = 0;
  while (k < count) {
    int64_t run = 1;
    while (k + run < count && ids[k + run] == ids[k] + run) ++run;
    GW_CUDA(c, cudaMemcpy2DAsync(rows + (size_t)k * W, W * sizeof(uint32_t), c->wires + (size_t)ids[k] * c->Wp,
                                 c->Wp * sizeof(uint32_t), W * sizeof(uint32_t), run, cudaMemcpyDeviceToHost, c->stream));
    k += run;
  }
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  return GW_OK;
}

int gw_plan_create(gw_ctx* c, int64_t n_levels, const int64_t* offs, const int32_t* opcodes, const int32_t* operands,
                   const int32_t* out_ids, gw_plan** out) {
  if (!c || !out || n_levels < 0 || (n_levels > 0 && (!offs || !opcodes || !operands || !out_ids))) return GW_ERR_ARG;
  if (!c->have_params) return fail(c, GW_ERR_STATE, "parameters not set");
  *out = nullptr;
  cudaSetDevice(c->device);
  gw_plan* p = new gw_plan();
  p->n_levels = n_levels;
  std::vector<LinJob> jobs;
  std::vector<KsUnit> units;
  std::vector<CheapUnit> cheap;
  // Every level is cut into segments of at most kSegGates gates (the gates of
  // a level are independent): a segment is one launch set, so scratch memory
  // stays bounded (~1 GB) however wide the level is.  kSegGates is a multiple
  // of 148 SMs x 3 and x 4 gates per CTA, i.e. whole waves of the blind rotation.
  for (int64_t lv = 0; lv < n_levels; ++lv) {
   p->seg_first.push_back((int64_t)p->J.size());
   for (int64_t s0 = offs[lv]; s0 < offs[lv + 1] || s0 == offs[lv]; s0 += kSegGates) {
    const int64_t s1 = std::min<int64_t>(offs[lv + 1], s0 + kSegGates);
    const size_t j0 = jobs.size(), u0 = units.size(), c0 = cheap.size();
    p->job_off.push_back(j0);
    p->unit_off.push_back(u0);
    p->cheap_off.push_back(c0);
    for (int64_t g = s0; g < s1; ++g) {
      const int op = opcodes[g];
      const int ar = arity_of(op);
      if (ar < 0) {
        delete p;
        return fail(c, GW_ERR_ARG, "unknown opcode in plan");
      }
      int32_t s[3] = {operands[3 * g], operands[3 * g + 1], operands[3 * g + 2]};
      for (int k = 0; k < ar; ++k)
        if (s[k] < 0 || s[k] >= c->wire_slots) {
          delete p;
          return fail(c, GW_ERR_WIRE, "operand wire out of range: " + std::to_string(s[k]));
        }
      if (out_ids[g] < 0 || out_ids[g] >= c->wire_slots) {
        delete p;
        return fail(c, GW_ERR_WIRE, "output wire out of range: " + std::to_string(out_ids[g]));
      }
      for (int k = 0; k < ar; ++k) p->max_wire = std::max<int64_t>(p->max_wire, s[k]);
      p->max_wire = std::max<int64_t>(p->max_wire, out_ids[g]);
      describe_gate(op, s[0], s[1], s[2], out_ids[g], c->p.mu, jobs, units, cheap);
    }
    // job indices inside units are level-local
    for (size_t u = u0; u < units.size(); ++u) {
      units[u].job0 -= (int32_t)j0;
      if (units[u].job1 >= 0) units[u].job1 -= (int32_t)j0;
    }
    p->J.push_back((int)(jobs.size() - j0));
    p->U.push_back((int)(units.size() - u0));
    p->C.push_back((int)(cheap.size() - c0));
    if (p->J.back() > p->max_jobs) p->max_jobs = p->J.back();
    if (s1 >= offs[lv + 1]) break;
   }
  }
  p->seg_first.push_back((int64_t)p->J.size());
  cudaError_t e = cudaSuccess;
  if (!jobs.empty()) e = cudaMalloc(&p->jobs, jobs.size() * sizeof(LinJob));
  if (e == cudaSuccess && !units.empty()) e = cudaMalloc(&p->units, units.size() * sizeof(KsUnit));
  if (e == cudaSuccess && !cheap.empty()) e = cudaMalloc(&p->cheap, cheap.size() * sizeof(CheapUnit));
  if (e == cudaSuccess && !jobs.empty())
    e = cudaMemcpy(p->jobs, jobs.data(), jobs.size() * sizeof(LinJob), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !units.empty())
    e = cudaMemcpy(p->units, units.data(), units.size() * sizeof(KsUnit), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !cheap.empty())
    e = cudaMemcpy(p->cheap, cheap.data(), cheap.size() * sizeof(CheapUnit), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    gw_plan_destroy(c, p);
    return fail(c, GW_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = p;
  return GW_OK;
}

int gw_plan_run_levels(gw_ctx* c, gw_plan* p, int64_t first, int64_t last) {
  int rc = ready(c);
  if (rc) return rc;
  if (!p) return fail(c, GW_ERR_ARG, "null plan");
  if (!c->wires || c->wire_slots == 0) return fail(c, GW_ERR_STATE, "wire store not allocated");
  // the store may have been re-allocated (smaller) since the plan was built
  if (p->max_wire >= c->wire_slots)
    return fail(c, GW_ERR_WIRE, "plan references wire " + std::to_string(p->max_wire) + " but the wire store has " +
                                    std::to_string(c->wire_slots) + " slots");
  if (first < 0) first = 0;
  if (last > p->n_levels) last = p->n_levels;
  if (first >= last) return GW_OK;
  cudaSetDevice(c->device);
  for (int64_t sg = p->seg_first[first]; sg < p->seg_first[last]; ++sg) {
    rc = run_level(c, c->wires, c->Wp, c->wires, c->Wp, p->jobs + p->job_off[sg], p->J[sg],
                   p->units + p->unit_off[sg], p->U[sg], p->cheap + p->cheap_off[sg], p->C[sg]);
    if (rc) return rc;
  }
  return GW_OK;
}

int gw_plan_run(gw_ctx* c, gw_plan* p) { return gw_plan_run_levels(c, p, 0, p ? p->n_levels : 0); }

int gw_plan_destroy(gw_ctx* c, gw_plan* p) {
  if (!p) return GW_OK;
  if (c) cudaSetDevice(c->device);
  cudaFree(p->jobs);
  cudaFree(p->units);
  cudaFree(p->cheap);
  delete p;
  return GW_OK;
}

// ---- multi-GPU wire exchange: point-to-point plan + native NCCL -------------
//
// counts[(level*world + src)*world + dst] = rows rank src produces at `level`
// that rank dst needs; ids in (level, src, dst) order.  Every rank passes the
// same arrays and keeps its own sends (src == rank, grouped by dst) and
// receives (dst == rank, grouped by src).  Send / receive staging buffers are
// owned by the plan, sized for the widest level.
struct gw_xplan {
  int64_t n_levels = 0;
  int world = 1, rank = 0;
  std::vector<int64_t> send_cnt, recv_cnt;      // [level][peer]
  std::vector<int64_t> send_off, recv_off;      // [level]: first row in the device id lists
  std::vector<int64_t> send_tot, recv_tot;      // [level]
  int64_t max_send = 0, max_recv = 0;
  int64_t* d_send_ids = nullptr;
  int64_t* d_recv_ids = nullptr;
  uint32_t* d_send = nullptr;
  uint32_t* d_recv = nullptr;
};


int gw_xplan_create(gw_ctx* c, int64_t n_levels, int32_t world, int32_t rank, const int64_t* counts,
                    const int64_t* ids, gw_xplan** out) {
  if (!c || !out || n_levels < 0 || world < 1 || rank < 0 || rank >= world) return GW_ERR_ARG;
  *out = nullptr;
  const int64_t cells = n_levels * world * world;
  if (cells > 0 && !counts) return GW_ERR_ARG;
  int64_t total = 0;
  for (int64_t k = 0; k < cells; ++k) {
    if (counts[k] < 0) return fail(c, GW_ERR_ARG, "exchange counts must be >= 0");
    total += counts[k];
  }
  if (total > 0 && !ids) return GW_ERR_ARG;
  for (int64_t k = 0; k < total; ++k)
    if (ids[k] < 0 || ids[k] >= c->wire_slots)
      return fail(c, GW_ERR_WIRE, "exchange wire id out of range: " + std::to_string(ids[k]));
  gw_xplan* x = new gw_xplan();
  x->n_levels = n_levels;
  x->world = world;
  x->rank = rank;
  std::vector<int64_t> sids, rids;
  x->send_cnt.assign(n_levels * world, 0);
  x->recv_cnt.assign(n_levels * world, 0);
  int64_t pos = 0;
  for (int64_t L = 0; L < n_levels; ++L) {
    x->send_off.push_back((int64_t)sids.size());
    x->recv_off.push_back((int64_t)rids.size());
    // (src, dst) cells of this level in order; rows of src -> dst are ids[pos .. pos + n)
    std::vector<std::pair<int64_t, int64_t>> cell(world * world);
    for (int q = 0; q < world; ++q)
      for (int r = 0; r < world; ++r) {
        const int64_t n = counts[(L * world + q) * world + r];
        cell[q * world + r] = {pos, n};
        pos += n;
      }
    for (int r = 0; r < world; ++r) {  // sends grouped by destination
      if (r == rank) continue;
      const auto& cl = cell[rank * world + r];
      sids.insert(sids.end(), ids + cl.first, ids + cl.first + cl.second);
      x->send_cnt[L * world + r] = cl.second;
    }
    for (int q = 0; q < world; ++q) {  // receives grouped by source
      if (q == rank) continue;
      const auto& cl = cell[q * world + rank];
      rids.insert(rids.end(), ids + cl.first, ids + cl.first + cl.second);
      x->recv_cnt[L * world + q] = cl.second;
    }
    x->send_tot.push_back((int64_t)sids.size() - x->send_off.back());
    x->recv_tot.push_back((int64_t)rids.size() - x->recv_off.back());
    x->max_send = std::max(x->max_send, x->send_tot.back());
    x->max_recv = std::max(x->max_recv, x->recv_tot.back());
  }
  cudaSetDevice(c->device);
  cudaError_t e = cudaSuccess;
  if (!sids.empty()) e = cudaMalloc(&x->d_send_ids, sids.size() * sizeof(int64_t));
  if (e == cudaSuccess && !sids.empty())
    e = cudaMemcpy(x->d_send_ids, sids.data(), sids.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !rids.empty()) e = cudaMalloc(&x->d_recv_ids, rids.size() * sizeof(int64_t));
  if (e == cudaSuccess && !rids.empty())
    e = cudaMemcpy(x->d_recv_ids, rids.data(), rids.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && x->max_send) e = cudaMalloc(&x->d_send, (size_t)x->max_send * c->Wp * sizeof(uint32_t));
  if (e == cudaSuccess && x->max_recv) e = cudaMalloc(&x->d_recv, (size_t)x->max_recv * c->Wp * sizeof(uint32_t));
  if (e != cudaSuccess) {
    gw_xplan_destroy(c, x);
    return fail(c, GW_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = x;
  return GW_OK;
}

int gw_xplan_peer_rows(gw_ctx* c, const gw_xplan* x, int64_t level, int64_t* send_rows, int64_t* recv_rows) {
  if (!c || !x || level < 0 || level >= x->n_levels || !send_rows || !recv_rows) return GW_ERR_ARG;
  for (int q = 0; q < x->world; ++q) {
    send_rows[q] = x->send_cnt[level * x->world + q];
    recv_rows[q] = x->recv_cnt[level * x->world + q];
  }
  return GW_OK;
}

int gw_xplan_buffers(gw_ctx* c, const gw_xplan* x, void** d_send, void** d_recv) {
  if (!c || !x || !d_send || !d_recv) return GW_ERR_ARG;
  *d_send = x->d_send;
  *d_recv = x->d_recv;
  return GW_OK;
}

int gw_exchange_pack(gw_ctx* c, const gw_xplan* x, int64_t level, uint32_t* d_send) {
  if (!c || !x || level < 0 || level >= x->n_levels) return GW_ERR_ARG;
  if (!c->wires || c->wire_slots == 0) return fail(c, GW_ERR_STATE, "wire store not allocated");
  const int64_t n = x->send_tot[level];
  if (n == 0) return GW_OK;
  if (!d_send) d_send = x->d_send;
  cudaSetDevice(c->device);
  k_xpack<<<dim3(1, grid_rows(n)), 160, 0, c->stream>>>(c->wires, c->Wp, x->d_send_ids + x->send_off[level], n,
                                                        d_send, c->Wp);
  GW_LAUNCHED(c);
  return GW_OK;
}

int gw_exchange_unpack(gw_ctx* c, const gw_xplan* x, int64_t level, const uint32_t* d_recv) {
  if (!c || !x || level < 0 || level >= x->n_levels) return GW_ERR_ARG;
  if (!c->wires || c->wire_slots == 0) return fail(c, GW_ERR_STATE, "wire store not allocated");
  const int64_t n = x->recv_tot[level];
  if (n == 0) return GW_OK;
  if (!d_recv) d_recv = x->d_recv;
  cudaSetDevice(c->device);
  k_xscatter<<<dim3(1, grid_rows(n)), 160, 0, c->stream>>>(c->wires, c->Wp, x->d_recv_ids + x->recv_off[level], n,
                                                           d_recv, c->Wp);
  GW_LAUNCHED(c);
  return GW_OK;
}

int gw_nccl_available(char* why, int64_t why_len) {
  const NcclApi& api = nccl_api();
  if (why && why_len > 0) {
    std::snprintf(why, (size_t)why_len, "%s", api.ok ? "" : api.why.c_str());
  }
  if (!api.ok) return 0;
  int v = 0;
  api.GetVersion(&v);
  return v > 0 ? v : 1;
}

int gw_nccl_unique_id(char* out /* NCCL_UNIQUE_ID_BYTES */) {
  if (!out) return GW_ERR_ARG;
  const NcclApi& api = nccl_api();
  if (!api.ok) return GW_ERR_STATE;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != ncclSuccess) return GW_ERR_CUDA;
  memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return GW_OK;
}

int gw_nccl_init(gw_ctx* c, int32_t world, int32_t rank, const char* unique_id) {
  if (!c || !unique_id || world < 1 || rank < 0 || rank >= world) return GW_ERR_ARG;
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(c, GW_ERR_STATE, "NCCL unavailable: " + api.why);
  cudaSetDevice(c->device);
  if (c->nccl) {
    api.CommDestroy((ncclComm_t)c->nccl);
    c->nccl = nullptr;
  }
  ncclUniqueId id;
  memcpy(id.internal, unique_id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t comm = nullptr;
  GW_NCCL(c, api, api.CommInitRank(&comm, world, id, rank));
  c->nccl = comm;
  c->nccl_world = world;
  c->nccl_rank = rank;
  return GW_OK;
}

int gw_exchange_enqueue(gw_ctx* c, const gw_xplan* x, int64_t level, void* nccl_comm) {
  if (!c || !x || level < 0 || level >= x->n_levels) return GW_ERR_ARG;
  ncclComm_t comm = (ncclComm_t)(nccl_comm ? nccl_comm : c->nccl);
  if (x->world == 1) return GW_OK;
  if (!comm) return fail(c, GW_ERR_STATE, "no NCCL communicator (gw_nccl_init or pass one)");
  const NcclApi& api = nccl_api();
  if (!api.ok) return fail(c, GW_ERR_STATE, "NCCL unavailable: " + api.why);
  int rc = gw_exchange_pack(c, x, level, nullptr);
  if (rc) return rc;
  if (x->send_tot[level] == 0 && x->recv_tot[level] == 0) return GW_OK;
  cudaSetDevice(c->device);
  const size_t row_bytes = (size_t)c->Wp * sizeof(uint32_t);
  // grouped point-to-point: each rank sends only the rows its peers read
  GW_NCCL(c, api, api.GroupStart());
  int64_t so = 0, ro = 0;
  for (int q = 0; q < x->world; ++q) {
    if (q == x->rank) continue;
    const int64_t ns = x->send_cnt[level * x->world + q], nr = x->recv_cnt[level * x->world + q];
    if (ns) {
      ncclResult_t r = api.Send((const char*)x->d_send + so * row_bytes, (size_t)ns * row_bytes, ncclUint8, q, comm,
                                c->stream);
      if (r != ncclSuccess) {
        api.GroupEnd();
        return fail(c, GW_ERR_CUDA, std::string("ncclSend: ") + api.GetErrorString(r));
      }
    }
    if (nr) {
      ncclResult_t r = api.Recv((char*)x->d_recv + ro * row_bytes, (size_t)nr * row_bytes, ncclUint8, q, comm,
                                c->stream);
      if (r != ncclSuccess) {
        api.GroupEnd();
        return fail(c, GW_ERR_CUDA, std::string("ncclRecv: ") + api.GetErrorString(r));
      }
    }
    so += ns;
    ro += nr;
  }
  GW_NCCL(c, api, api.GroupEnd());
  return gw_exchange_unpack(c, x, level, nullptr);
}

int gw_xplan_destroy(gw_ctx* c, gw_xplan* x) {
  if (!x) return GW_OK;
  if (c) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);  // staging buffers may still be in flight
  }
  cudaFree(x->d_send_ids);
  cudaFree(x->d_recv_ids);
  cudaFree(x->d_send);
  cudaFree(x->d_recv);
  delete x;
  return GW_OK;
}

// ---- device timeline: event marks on the context stream, read once ----------
int gw_timeline_reset(gw_ctx* c) {
  if (!c) return GW_ERR_ARG;
  for (auto e : c->marks) c->ev_pool.push_back(e);
  c->marks.clear();
  return GW_OK;
}

int gw_timeline_mark(gw_ctx* c) {
  if (!c) return GW_ERR_ARG;
  cudaEvent_t e = pooled_event(c);
  if (!e) return fail(c, GW_ERR_CUDA, "cudaEventCreate failed");
  GW_CUDA(c, cudaEventRecord(e, c->stream));
  c->marks.push_back(e);
  return GW_OK;
}

int gw_timeline_read(gw_ctx* c, float* ms, int64_t cap, int64_t* count) {
  if (!c || !count || (cap > 0 && !ms)) return GW_ERR_ARG;
  const int64_t n = c->marks.empty() ? 0 : (int64_t)c->marks.size() - 1;
  *count = n;
  if (n == 0) return GW_OK;
  GW_CUDA(c, cudaEventSynchronize(c->marks.back()));
  for (int64_t k = 0; k < n && k < cap; ++k) GW_CUDA(c, cudaEventElapsedTime(&ms[k], c->marks[k], c->marks[k + 1]));
  return GW_OK;
}

// All levels [first, last) with one event mark per level boundary and a single
// host synchronisation at the end; ms[k] = device time of level first + k.
int gw_plan_run_timed(gw_ctx* c, gw_plan* p, int64_t first, int64_t last, float* ms) {
  int rc = ready(c);
  if (rc) return rc;
  if (!p) return fail(c, GW_ERR_ARG, "null plan");
  if (first < 0) first = 0;
  if (last > p->n_levels) last = p->n_levels;
  if (first >= last) return GW_OK;
  if (!ms) return GW_ERR_ARG;
  gw_timeline_reset(c);
  if ((rc = gw_timeline_mark(c))) return rc;
  for (int64_t L = first; L < last; ++L) {
    if ((rc = gw_plan_run_levels(c, p, L, L + 1))) return rc;
    if ((rc = gw_timeline_mark(c))) return rc;
  }
  int64_t n = 0;
  rc = gw_timeline_read(c, ms, last - first, &n);
  gw_timeline_reset(c);
  return rc;
}

// Rounding-margin probe: blind rotations at N = 1024, l = 2 run the probe build
// of the kernel, which records max |x - rint(x)| over every value the inverse
// transforms round (exactness needs < 0.5).
int gw_set_margin_probe(gw_ctx* c, int on) {
  if (!c) return GW_ERR_ARG;
  cudaSetDevice(c->device);
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  if (on && !c->margin) {
    GW_CUDA(c, cudaMalloc(&c->margin, sizeof(unsigned long long)));
    GW_CUDA(c, cudaMemset(c->margin, 0, sizeof(unsigned long long)));
  } else if (!on && c->margin) {
    cudaFree(c->margin);
    c->margin = nullptr;
  }
  return GW_OK;
}

// Exact mode: the split-key v3 blind rotation (provable FP64 exactness) instead
// of v5 (single key image, measured exactness); DESIGN.md §3.
int gw_set_exact(gw_ctx* c, int on) {
  if (!c) return GW_ERR_ARG;
  c->br_exact = on != 0;
  return GW_OK;
}

int gw_get_exact(gw_ctx* c, int* on) {
  if (!c || !on) return GW_ERR_ARG;
  *on = c->br_exact ? 1 : 0;
  return GW_OK;
}

int gw_margin_read(gw_ctx* c, double* worst, int reset) {
  if (!c || !worst) return GW_ERR_ARG;
  if (!c->margin) return fail(c, GW_ERR_STATE, "margin probe off (gw_set_margin_probe)");
  cudaSetDevice(c->device);
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  unsigned long long bits = 0;
  GW_CUDA(c, cudaMemcpy(&bits, c->margin, sizeof(bits), cudaMemcpyDeviceToHost));
  memcpy(worst, &bits, sizeof(double));
  if (reset) GW_CUDA(c, cudaMemset(c->margin, 0, sizeof(unsigned long long)));
  return GW_OK;
}

int gw_timer_start(gw_ctx* c) {
  if (!c) return GW_ERR_ARG;
  GW_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  return GW_OK;
}

int gw_timer_stop(gw_ctx* c, float* ms) {
  if (!c || !ms) return GW_ERR_ARG;
  GW_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  GW_CUDA(c, cudaEventSynchronize(c->ev1));
  GW_CUDA(c, cudaEventElapsedTime(ms, c->ev0, c->ev1));
  return GW_OK;
}

int gw_set_profiling(gw_ctx* c, int on) {
  if (!c) return GW_ERR_ARG;
  c->profile = on != 0;
  return GW_OK;
}

int gw_stage_times(gw_ctx* c, double* ms /* [3] */, int64_t* items /* [3] */, int reset) {
  if (!c || !ms) return GW_ERR_ARG;
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < 3; ++k) {
    double tot = 0;
    for (auto& pr : c->prof_ev[k]) {
      float t = 0;
      GW_CUDA(c, cudaEventElapsedTime(&t, pr.first, pr.second));
      tot += t;
    }
    ms[k] = tot;
    if (items) items[k] = c->prof_items[k];
    if (reset) {
      for (auto& pr : c->prof_ev[k]) {
        c->ev_pool.push_back(pr.first);
        c->ev_pool.push_back(pr.second);
      }
      c->prof_ev[k].clear();
      c->prof_items[k] = 0;
    }
  }
  return GW_OK;
}

int gw_br_phase_cycles(gw_ctx* c, long long* out /* [4][6] */) {
  if (!c || !out) return GW_ERR_ARG;
  if (!c->br_prof) return fail(c, GW_ERR_STATE, "phase profiling off (GATEWAVE_BR_PROFILE=1)");
  GW_CUDA(c, cudaStreamSynchronize(c->stream));
  GW_CUDA(c, cudaMemcpy(out, c->br_prof, 24 * sizeof(long long), cudaMemcpyDeviceToHost));
  return GW_OK;
}

int gw_launch_count(gw_ctx* c, int64_t* count) {
  if (!c || !count) return GW_ERR_ARG;
  *count = c->launches;
  return GW_OK;
}

}  // extern "C"
