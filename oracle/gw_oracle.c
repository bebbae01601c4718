/*
 * gw_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's bootstrapped-gate hot path
 * (gatewave, /root/reference/pkg/src/gatewave/{torus,cggi}.py), used as the
 * parity checker for the CUDA engine and as the CPU baseline in bench.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product never does.
 *
 * It follows the reference algorithm literally: exact negacyclic NTT over the
 * Goldilocks prime Q = 2^64 - 2^32 + 1 with psi folded into the twiddles
 * (Harvey CT forward, GS inverse), gadget decomposition straight into
 * residues, LWE-index-outer blind rotation, constant-coefficient extraction
 * and MSB-first digit keyswitching.  Pinned against golden vectors produced
 * by the reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;
static const uint64_t Q = 0xFFFFFFFF00000001ULL;
static const uint64_t M32 = 0xFFFFFFFFULL;
static const uint64_t GENERATOR = 12037493425763644479ULL; /* torus.py:23 */

/* torus.py:74-88 (_mm): 128-bit product folded with 2^64 = 2^32 - 1 (mod Q).
 * The 64x64 -> 128 product is assembled from four 32x32 -> 64 partial
 * products (the reference's LLVM i128 multiply lowers the same way when it
 * vectorises), so gcc can vectorise the transform loops too. */
static inline uint64_t mm(uint64_t a, uint64_t b) {
  const uint64_t a0 = a & M32, a1 = a >> 32, b0 = b & M32, b1 = b >> 32;
  const uint64_t p00 = a0 * b0, p01 = a0 * b1, p10 = a1 * b0, p11 = a1 * b1;
  const uint64_t mid = (p00 >> 32) + (p01 & M32) + (p10 & M32);
  const uint64_t lo = (p00 & M32) | (mid << 32);
  const uint64_t hi = p11 + (p01 >> 32) + (p10 >> 32) + (mid >> 32);
  const uint64_t h_hi = hi >> 32, h_lo = hi & M32;
  uint64_t t = lo - h_hi;
  t = lo < h_hi ? t - M32 : t;
  uint64_t u = (h_lo << 32) - h_lo;
  uint64_t s = t + u;
  s = s < t ? s + M32 : s;
  return s >= Q ? s - Q : s;
}
/* torus.py:91-98 (_ma) */
static inline uint64_t ma(uint64_t a, uint64_t b) {
  uint64_t s = a + b;
  s = s < a ? s + M32 : s;
  return s >= Q ? s - Q : s;
}
/* torus.py:101-106 (_ms) */
static inline uint64_t ms(uint64_t a, uint64_t b) {
  uint64_t d = a - b;
  return a < b ? d - M32 : d;
}

static uint64_t powmod(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mm(r, b);
    b = mm(b, b);
    e >>= 1;
  }
  return r;
}


/* Minimal pthread parallel-for over independent gates (no OpenMP runtime in
 * this image).  Work items are handed out from one shared cursor. */
typedef void (*orc_task_fn)(void* ctx, int64_t idx, void* scratch);
typedef struct {
  orc_task_fn fn;
  void* ctx;
  int64_t count;
  int64_t next;
  size_t scratch_bytes;
  pthread_mutex_t mu;
  int failed;
} orc_pool;

static void* orc_worker(void* arg) {
  orc_pool* p = (orc_pool*)arg;
  void* scratch = p->scratch_bytes ? malloc(p->scratch_bytes) : NULL;
  if (p->scratch_bytes && !scratch) {
    pthread_mutex_lock(&p->mu);
    p->failed = 1;
    pthread_mutex_unlock(&p->mu);
    return NULL;
  }
  for (;;) {
    pthread_mutex_lock(&p->mu);
    int64_t idx = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (idx >= p->count) break;
    p->fn(p->ctx, idx, scratch);
  }
  free(scratch);
  return NULL;
}

static int orc_parallel_for(int64_t count, int threads, size_t scratch_bytes, orc_task_fn fn,
                            void* ctx) {
  orc_pool p;
  p.fn = fn; p.ctx = ctx; p.count = count; p.next = 0; p.scratch_bytes = scratch_bytes;
  p.failed = 0;
  pthread_mutex_init(&p.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads > 512) threads = 512;
  if (threads > count) threads = count > 0 ? (int)count : 1;
  pthread_t tids[512];
  int started = 0;
  for (int w = 1; w < threads; ++w)
    if (pthread_create(&tids[started], NULL, orc_worker, &p) == 0) ++started;
  orc_worker(&p);
  for (int w = 0; w < started; ++w) pthread_join(tids[w], NULL);
  pthread_mutex_destroy(&p.mu);
  return p.failed ? -2 : 0;
}

static int bitrev(int i, int bits) {
  int r = 0;
  for (int k = 0; k < bits; ++k) { r = (r << 1) | (i & 1); i >>= 1; }
  return r;
}

/* torus.py:233-270 (build_ntt_tables): psi = g^((Q-1)/2n), bit-reversed powers */
int orc_build_tables(int n, uint64_t* psi_brv, uint64_t* ipsi_brv, uint64_t* n_inv) {
  if (n < 1 || (n & (n - 1))) return -1;
  int log_n = 0;
  while ((1 << log_n) < n) ++log_n;
  uint64_t psi = powmod(GENERATOR, (Q - 1) / (2 * (uint64_t)n));
  uint64_t ipsi = powmod(psi, Q - 2);
  for (int i = 0; i < n; ++i) {
    int r = bitrev(i, log_n);
    psi_brv[i] = powmod(psi, (uint64_t)r);
    ipsi_brv[i] = powmod(ipsi, (uint64_t)r);
  }
  *n_inv = powmod((uint64_t)n, Q - 2);
  return 0;
}

/* torus.py:109-129 (_fwd_inplace): natural in, bit-reversed out */
static void ntt_fwd(uint64_t* a, int n, const uint64_t* psi_brv) {
  int t = n;
  for (int m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (int i = 0; i < m; ++i) {
      uint64_t w = psi_brv[m + i];
      int j1 = 2 * i * t;
      for (int j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j], v = mm(a[j + t], w);
        a[j] = ma(u, v);
        a[j + t] = ms(u, v);
      }
    }
  }
}

/* torus.py:132-152 (_inv_inplace): bit-reversed in, natural out, times n^-1 */
static void ntt_inv(uint64_t* a, int n, const uint64_t* ipsi_brv, uint64_t n_inv) {
  int t = 1;
  for (int m = n; m > 1; m >>= 1) {
    int h = m >> 1, j1 = 0;
    for (int i = 0; i < h; ++i) {
      uint64_t w = ipsi_brv[h + i];
      for (int j = j1; j < j1 + t; ++j) {
        uint64_t u = a[j], v = a[j + t];
        a[j] = ma(u, v);
        a[j + t] = mm(ms(u, v), w);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (int j = 0; j < n; ++j) a[j] = mm(a[j], n_inv);
}

void orc_ntt_forward(uint64_t* rows, int64_t count, int n, const uint64_t* psi_brv) {
  for (int64_t r = 0; r < count; ++r) ntt_fwd(rows + r * n, n, psi_brv);
}

void orc_ntt_inverse(uint64_t* rows, int64_t count, int n, const uint64_t* ipsi_brv, uint64_t n_inv) {
  for (int64_t r = 0; r < count; ++r) ntt_inv(rows + r * n, n, ipsi_brv, n_inv);
}

/* cggi.py:283-285 (BootstrappingKey.__init__): zero-extended u32 -> NTT domain */
void orc_bk_to_ntt(const uint32_t* bk, int64_t rows, int n, const uint64_t* psi_brv, uint64_t* out) {
  for (int64_t r = 0; r < rows; ++r) {
    uint64_t* o = out + r * n;
    for (int j = 0; j < n; ++j) o[j] = bk[r * n + j];
    ntt_fwd(o, n, psi_brv);
  }
}

/* cggi.py:516-522 (_decompose_offset) */
uint32_t orc_decompose_offset(int bg_bits, int levels) {
  uint64_t off = 1ULL << (32 - levels * bg_bits - 1);
  for (int j = 1; j <= levels; ++j) off += (uint64_t)(1u << (bg_bits - 1)) << (32 - j * bg_bits);
  return (uint32_t)(off & M32);
}

/*
 * cggi.py:592-667 (_blind_rotate_kernel), same loop order as the reference:
 * LWE index i outermost, gates inner, so the 64 KB NTT-domain key slice
 * BK_i stays cache-resident across the batch.  Each worker thread owns a
 * contiguous chunk of gates (results do not depend on the split).
 */
typedef struct {
  const uint32_t* cts; int64_t B; int n; const uint32_t* tv; int N; int log_n; const uint64_t* bk_ntt;
  int bg_bits; int levels; const uint64_t* psi_brv; const uint64_t* ipsi_brv; uint64_t n_inv;
  uint32_t* acc_out; int threads;
} br_args;

static void br_chunk(void* ctx, int64_t chunk, void* scratch) {
  br_args* a = (br_args*)ctx;
  const int N = a->N, n = a->n, levels = a->levels, bg_bits = a->bg_bits;
  const int two_n = 2 * N, rows = 2 * levels;
  const int64_t per = (a->B + a->threads - 1) / a->threads;
  const int64_t g0 = chunk * per, g1 = g0 + per < a->B ? g0 + per : a->B;
  if (g0 >= g1) return;
  uint64_t* resid = (uint64_t*)scratch;
  uint64_t* accntt = resid + (size_t)rows * N;
  const uint64_t rshift = 32 - (a->log_n + 1);
  const uint64_t radd = 1ULL << (32 - (a->log_n + 1) - 1);
  const uint64_t base_mask = (1ULL << bg_bits) - 1;
  const int64_t half_base = 1LL << (bg_bits - 1);
  const uint64_t offs = orc_decompose_offset(bg_bits, levels);
  const uint64_t two32 = 1ULL << 32;
  const uint64_t qhalf = Q / 2;
  /* :612-622 acc <- tv * X^{-bbar} */
  for (int64_t g = g0; g < g1; ++g) {
    const uint32_t* ct = a->cts + g * (n + 1);
    uint32_t* acc = a->acc_out + g * 2 * N;
    int bbar = (int)((((uint64_t)ct[n]) + radd) >> rshift) & (two_n - 1);
    int k = (two_n - bbar) & (two_n - 1);
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < N; ++j) {
        int m = (j - k) & (two_n - 1);
        acc[c * N + j] = m < N ? a->tv[c * N + m] : (uint32_t)((two32 - a->tv[c * N + m - N]) & M32);
      }
  }
  for (int i = 0; i < n; ++i) {
    const uint64_t* bk_i = a->bk_ntt + (size_t)i * rows * 2 * N;
    for (int64_t g = g0; g < g1; ++g) {
      uint32_t* acc = a->acc_out + g * 2 * N;
      int abar = (int)((((uint64_t)a->cts[g * (n + 1) + i]) + radd) >> rshift) & (two_n - 1);
      /* :627-644 rotate-subtract + decompose into residues */
      for (int c = 0; c < 2; ++c) {
        const uint32_t* row = acc + c * N;
        for (int j = 0; j < N; ++j) {
          int m = (j - abar) & (two_n - 1);
          uint64_t rot = m < N ? (uint64_t)row[m] : ((two32 - (uint64_t)row[m - N]) & M32);
          uint64_t buf = ((rot - (uint64_t)row[j]) + offs) & M32;
          for (int lv = 0; lv < levels; ++lv) {
            uint64_t sh = 32 - (lv + 1) * bg_bits;
            int64_t dig = (int64_t)((buf >> sh) & base_mask) - half_base;
            resid[(c * levels + lv) * N + j] = dig < 0 ? Q + (uint64_t)dig : (uint64_t)dig;
          }
        }
      }
      /* :645-647 forward transforms */
      for (int r = 0; r < rows; ++r) ntt_fwd(resid + r * N, N, a->psi_brv);
      /* :648-657 MAC against the TGSW rows */
      memset(accntt, 0, sizeof(uint64_t) * 2 * N);
      for (int r = 0; r < rows; ++r)
        for (int c2 = 0; c2 < 2; ++c2) {
          const uint64_t* bkrow = bk_i + ((size_t)r * 2 + c2) * N;
          uint64_t* arow = accntt + c2 * N;
          const uint64_t* dr = resid + r * N;
          for (int j = 0; j < N; ++j) arow[j] = ma(arow[j], mm(dr[j], bkrow[j]));
        }
      /* :658-666 inverse + accumulate */
      for (int c2 = 0; c2 < 2; ++c2) {
        uint64_t* arow = accntt + c2 * N;
        ntt_inv(arow, N, a->ipsi_brv, a->n_inv);
        uint32_t* out = acc + c2 * N;
        for (int j = 0; j < N; ++j) {
          uint64_t rr = arow[j];
          uint64_t tor = ((rr & M32) - (rr > qhalf ? 1ULL : 0ULL)) & M32;
          out[j] = (uint32_t)(((uint64_t)out[j] + tor) & M32);
        }
      }
    }
  }
}

int orc_blind_rotate(const uint32_t* cts, int64_t B, int n, const uint32_t* tv, int N,
                     const uint64_t* bk_ntt, int bg_bits, int levels, const uint64_t* psi_brv,
                     const uint64_t* ipsi_brv, uint64_t n_inv, uint32_t* acc_out, int threads) {
  int log_n = 0;
  while ((1 << log_n) < N) ++log_n;
  if ((1 << log_n) != N) return -1;
  if (threads < 1) threads = 1;
  if (threads > B) threads = (int)(B > 0 ? B : 1);
  br_args a = {cts, B, n, tv, N, log_n, bk_ntt, bg_bits, levels, psi_brv, ipsi_brv, n_inv, acc_out, threads};
  size_t scratch = sizeof(uint64_t) * (size_t)(2 * levels * N + 2 * N);
  return orc_parallel_for(threads, threads, scratch, br_chunk, &a);
}

/* cggi.py:695-704 (_extract_rows) */
void orc_extract(const uint32_t* acc, int64_t B, int N, uint32_t* out) {
  for (int64_t g = 0; g < B; ++g) {
    const uint32_t* a = acc + g * 2 * N;
    uint32_t* o = out + g * (N + 1);
    o[0] = a[0];
    for (int j = 1; j < N; ++j) o[j] = 0u - a[N - j];
    o[N] = a[N];
  }
}

/* cggi.py:670-692 (_keyswitch_kernel) */
typedef struct {
  const uint32_t* exts; int N; const uint32_t* ksk; int levels; int gamma; int width;
  uint32_t* out;
} ks_args;

static void ks_task(void* ctx, int64_t g, void* scratch) {
  (void)scratch;
  ks_args* a = (ks_args*)ctx;
  const int N = a->N, levels = a->levels, gamma = a->gamma, width = a->width;
  const int tg = levels * gamma;
  const uint64_t roff = 1ULL << (32 - tg - 1);
  const uint64_t rsh = 32 - tg;
  const uint64_t dmask = (1ULL << gamma) - 1;
  const int vmax = (1 << gamma) - 1;
  uint32_t* orow = a->out + g * width;
  memset(orow, 0, sizeof(uint32_t) * width);
  orow[width - 1] = a->exts[g * (N + 1) + N];
  for (int i = 0; i < N; ++i) {
    uint64_t u = ((uint64_t)a->exts[g * (N + 1) + i] + roff) >> rsh;
    for (int j = 0; j < levels; ++j) {
      uint64_t sh = (uint64_t)((levels - 1 - j) * gamma);
      int d = (int)((u >> sh) & dmask);
      if (d != 0) {
        const uint32_t* krow = a->ksk + (((size_t)i * levels + j) * vmax + (d - 1)) * width;
        for (int jj = 0; jj < width; ++jj) orow[jj] -= krow[jj];
      }
    }
  }
}

int orc_keyswitch(const uint32_t* exts, int64_t B, int N, const uint32_t* ksk, int levels,
                  int gamma, int width, uint32_t* out, int threads) {
  ks_args a = {exts, N, ksk, levels, gamma, width, out};
  return orc_parallel_for(B, threads, 0, ks_task, &a);
}
