/*
 * gatewave_b200.h -- C ABI of the B200-native CGGI gate-bootstrapping engine.
 *
 * Drop-in boundary for the hot path of the reference package `gatewave`
 * (/root/reference/pkg/src/gatewave).  The reference has no FFI of its own;
 * its seams are Python call sites resolved at call time.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - All buffers are C-contiguous, little-endian, BORROWED for the duration
 *     of the call.  Functions taking host pointers copy in/out and return
 *     after the result is on the host.  *_device variants take device
 *     pointers and only enqueue work on the context stream.
 *   - Return 0 on success, a negative GW_ERR_* code otherwise; the message is
 *     available from gw_last_error().  The Python layer maps codes onto the
 *     reference's exception types (ParameterError, DimensionError,
 *     EvaluateError, RuntimeError).
 *   - A context is bound to one CUDA device and one stream; it is not
 *     thread-safe (the reference's single-submitter model).
 */
#ifndef GATEWAVE_B200_H
#define GATEWAVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GW_OK 0
#define GW_ERR_PARAM (-1)  /* -> cggi.ParameterError */
#define GW_ERR_DIM (-2)    /* -> cggi.DimensionError */
#define GW_ERR_STATE (-3)  /* missing params / keys / wire store */
#define GW_ERR_CUDA (-4)   /* CUDA runtime failure -> RuntimeError */
#define GW_ERR_ARG (-5)    /* bad argument -> ValueError */
#define GW_ERR_WIRE (-6)   /* wire id out of range -> runtime.EvaluateError */

/* Gate opcodes: the order of gatewave.cggi.GateKind (cggi.py:142-153). */
enum gw_opcode {
  GW_AND = 0, GW_OR = 1, GW_NAND = 2, GW_NOR = 3, GW_XOR = 4, GW_XNOR = 5,
  GW_NOT = 6, GW_MUX = 7, GW_CONST0 = 8, GW_CONST1 = 9, GW_COPY = 10,
  GW_BOOTSTRAP = 11  /* arity 1: refresh one sample (cggi.py:770-777 gate_bootstrap) */
};

/* Mirrors the hot-path fields of gatewave.cggi.ParamSet (cggi.py:66-114). */
typedef struct gw_params {
  int32_t n;             /* LWE dimension */
  int32_t N;             /* ring dimension (64, 256 or 1024 on this engine) */
  int32_t bg_bits;       /* gadget base bits (Bg_bits) */
  int32_t l;             /* gadget levels (1..3 on this engine) */
  int32_t ks_base_bits;  /* keyswitch base bits (gamma) */
  int32_t ks_levels;     /* keyswitch levels (t) */
  uint32_t mu;           /* message amplitude (cggi.py:84) */
} gw_params;

typedef struct gw_ctx gw_ctx;
typedef struct gw_plan gw_plan;

int gw_version(void);

/* Host-only netlist helper (no GPU needed), replaces the FIFO level walk of
 * gatewave/scheduler.py:57-102 (partition_waves) for 10^7-gate netlists:
 * pos[3*k + j] is the gate POSITION (index in execution order) of operand j of
 * gate k, or -1 for a circuit input / unused slot; level[k] = 1 + max level of
 * its gate operands (0 if none).  Returns GW_ERR_ARG if an operand position is
 * not strictly before k (not a sequential form). */
int gw_levels(const int64_t* pos, int64_t gates, int32_t* level);
int gw_device_count(int* count);

/* Context life cycle.  `device` is the CUDA ordinal. */
int gw_create(int device, gw_ctx** out);
int gw_destroy(gw_ctx* ctx);
const char* gw_last_error(const gw_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream()); NULL = own stream. */
int gw_set_stream(gw_ctx* ctx, void* cuda_stream);
int gw_sync(gw_ctx* ctx);

/* ParamSet validation + engine envelope (cggi.py:86-110). */
int gw_set_params(gw_ctx* ctx, const gw_params* p);

/* Key upload (replaces EvalKey.build / BootstrappingKey.__init__,
 * cggi.py:277-285, 336-342): bk_coeff is bootstrapping_key.data
 * (n, 2l, 2, N) u32, ksk is keyswitch_key.data (N, t, 2^gamma-1, n+1) u32.
 * Either may be NULL (blind-rotation-only / keyswitch-only contexts).
 * The bootstrapping key is transformed into the FFT domain ON the device. */
int gw_upload_keys(gw_ctx* ctx, const uint32_t* bk_coeff, const uint32_t* ksk);
/* Device FFT-domain key, for the parity pin against bootstrapping_key.data. */
int gw_bk_fft_size(gw_ctx* ctx, int64_t* n_complex);
int gw_download_bk_fft(gw_ctx* ctx, double* out /* 2 * n_complex doubles */);

/* Seam 1 twins (cggi.py:592-667 `_blind_rotate_kernel`, cggi.py:670-692
 * `_keyswitch_kernel` with cggi.py:695-704 `_extract_rows` fused):
 *   lin (B, n+1) u32, tv (2, N) u32 -> acc (B, 2, N) u32
 *   ext (B, N+1) u32 -> out (B, n+1) u32 */
int gw_blind_rotate(gw_ctx* ctx, const uint32_t* lin, int64_t B, const uint32_t* tv, uint32_t* acc);
int gw_keyswitch(gw_ctx* ctx, const uint32_t* ext, int64_t B, uint32_t* out);

/* Seam 2 (cggi.py:785-854 `eval_gate_batch`): operands[k] is a (B, n+1)
 * u32 matrix per input position (arity = GATE_ARITY[kind]); out (B, n+1).
 * For CONST0/CONST1 arity is 0 and B is the requested count. */
int gw_eval_gate_batch(gw_ctx* ctx, int opcode, const uint32_t* const* operands, int arity,
                       int64_t B, uint32_t* out);
/* Same with device-resident operands/output (row strides in 32-bit words). */
int gw_eval_gate_batch_device(gw_ctx* ctx, int opcode, const uint32_t* const* d_operands,
                              int64_t in_stride, int arity, int64_t B, uint32_t* d_out,
                              int64_t out_stride);

/* Seam 3 support (runtime.py:76-222 `WireStore` + `evaluate`): a
 * device-resident wire store of `slots` rows and a level plan.  A plan holds,
 * per level, every gate's opcode, up to three operand wire ids (unused = -1)
 * and output wire id; gw_plan_run enqueues all levels on the stream without
 * host synchronisation (one fused launch set per level, all opcodes mixed).
 * gw_wires_alloc(ctx, slots) (re)sizes the store and zeroes the slots in use;
 * slots = 0 releases it.  An owned store is reused while it fits, and a released
 * store of up to 4 GB stays cached for the next call (cudaMalloc / cudaFree
 * synchronise the device); after release the store counts as absent. */
int gw_wires_alloc(gw_ctx* ctx, int64_t slots);
int gw_wires_put(gw_ctx* ctx, const int64_t* ids, const uint32_t* rows, int64_t count);
int gw_wires_get(gw_ctx* ctx, const int64_t* ids, uint32_t* rows, int64_t count);
int gw_wires_device_ptr(gw_ctx* ctx, void** ptr, int64_t* stride_words);
/* Use caller-owned device memory (e.g. a torch tensor) as the wire store:
 * `slots` rows of `stride_words` (= n+1 rounded up to 4) 32-bit words.  The
 * pointer must be device (or managed) memory on the context's GPU; host or
 * other-GPU memory is rejected with GW_ERR_ARG (cudaPointerGetAttributes). */
int gw_wires_attach(gw_ctx* ctx, void* dev_ptr, int64_t slots, int64_t stride_words);
int gw_plan_create(gw_ctx* ctx, int64_t n_levels, const int64_t* level_offsets,
                   const int32_t* opcodes, const int32_t* operands /* (count, 3) */,
                   const int32_t* out_ids, gw_plan** out);
int gw_plan_run(gw_ctx* ctx, gw_plan* plan);
int gw_plan_run_levels(gw_ctx* ctx, gw_plan* plan, int64_t first, int64_t last);
int gw_plan_destroy(gw_ctx* ctx, gw_plan* plan);

/* Multi-GPU wire exchange between levels (replaces the reference's per-wave
 * WireStore hand-off, runtime.py:166-190, for one process per GPU; SURVEY.md
 * §8(b) gw_exchange_enqueue).  Point-to-point plan: counts[(level*world +
 * src)*world + dst] is the number of wires rank src produces at `level` that
 * rank dst needs (reads in a later level, or circuit outputs); ids lists them
 * in (level, src, dst) order.  Every rank passes the same arrays and keeps its
 * own sends and receives; the plan owns device staging buffers.
 * gw_exchange_enqueue packs this rank's rows, runs one grouped ncclSend /
 * ncclRecv per peer (NCCL over NVLink / NVSwitch, only the rows each peer
 * reads) and scatters the received rows into the wire store -- all enqueued on
 * the context stream, no host synchronisation.  nccl_comm is an ncclComm_t
 * (NULL: the context's own, from gw_nccl_init).  libnccl.so.2 is bound at run
 * time (GATEWAVE_NCCL_LIB, else the copy already loaded, else the system's).
 * pack / unpack / peer_rows / buffers expose the same steps for a caller that
 * moves the staged rows itself (e.g. gloo on CPU). */
typedef struct gw_xplan gw_xplan;
int gw_xplan_create(gw_ctx* ctx, int64_t n_levels, int32_t world, int32_t rank, const int64_t* counts,
                    const int64_t* ids, gw_xplan** out);
int gw_xplan_peer_rows(gw_ctx* ctx, const gw_xplan* plan, int64_t level, int64_t* send_rows /* [world] */,
                       int64_t* recv_rows /* [world] */);
int gw_xplan_buffers(gw_ctx* ctx, const gw_xplan* plan, void** d_send, void** d_recv);
int gw_exchange_pack(gw_ctx* ctx, const gw_xplan* plan, int64_t level, uint32_t* d_send /* NULL: plan buffer */);
int gw_exchange_unpack(gw_ctx* ctx, const gw_xplan* plan, int64_t level, const uint32_t* d_recv /* NULL: plan buffer */);
int gw_exchange_enqueue(gw_ctx* ctx, const gw_xplan* plan, int64_t level, void* nccl_comm);
int gw_xplan_destroy(gw_ctx* ctx, gw_xplan* plan);
/* NCCL bootstrap: version (> 0) when libnccl is usable, else 0 and the reason in `why`. */
int gw_nccl_available(char* why, int64_t why_len);
int gw_nccl_unique_id(char* out /* 128 bytes, ncclUniqueId */);
int gw_nccl_init(gw_ctx* ctx, int32_t world, int32_t rank, const char* unique_id /* 128 bytes */);

/* Device timeline: event marks on the context stream, read after one sync:
 * ms[k] = time between mark k and mark k+1.  gw_plan_run_timed runs levels
 * [first, last) with a mark at every level boundary and returns the device
 * time of each level after a single host synchronisation. */
int gw_timeline_reset(gw_ctx* ctx);
int gw_timeline_mark(gw_ctx* ctx);
int gw_timeline_read(gw_ctx* ctx, float* ms, int64_t cap, int64_t* count);
int gw_plan_run_timed(gw_ctx* ctx, gw_plan* plan, int64_t first, int64_t last, float* ms /* last - first */);

/* CUDA-event timer on the context stream (milliseconds between start/stop). */
int gw_timer_start(gw_ctx* ctx);
int gw_timer_stop(gw_ctx* ctx, float* ms);
/* Optional per-stage CUDA-event accounting (roofline evidence): when on,
 * every blind-rotation / keyswitch / other launch is bracketed by events.
 * gw_stage_times syncs and returns summed milliseconds and processed items
 * (bootstraps, output samples, 0) per stage: [blind_rotate, keyswitch, other]. */
int gw_set_profiling(gw_ctx* ctx, int on);
int gw_stage_times(gw_ctx* ctx, double* ms, int64_t* items, int reset);
/* Debug: per-phase cycle sums of the last TMEM blind rotation, warps 0..3 of
 * its first gate, phases [forward, fill, barrier A, MAC, inverse, step end];
 * needs GATEWAVE_BR_PROFILE=1 at context creation. */
int gw_br_phase_cycles(gw_ctx* ctx, long long* out);
/* Rounding-margin probe (exactness evidence): when on, blind
 * rotations at N = 1024, l = 2 run a probe build that records the worst
 * |x - rint(x)| over every FP64 value the inverse transforms round to an
 * integer; gw_margin_read syncs and returns it (< 0.5 means every rounding
 * recovered the exact integer). */
int gw_set_margin_probe(gw_ctx* ctx, int on);
int gw_margin_read(gw_ctx* ctx, double* worst, int reset);
/* Exact mode.  Off (default): at N = 1024, l = 2 with every
 * convolution coefficient <= 2^51 (PARAM_128, PARAM_110) the blind rotation
 * uses ONE FFT image of the 32-bit key words (v5: half the inverse transforms
 * and MACs of the split key; exactness measured by the margin probe, not
 * proven).  On: the split-key kernel (v3), whose FP64 exactness is proven.
 * Also GATEWAVE_BR_EXACT=1 at context creation. */
int gw_set_exact(gw_ctx* ctx, int on);
int gw_get_exact(gw_ctx* ctx, int* on);
/* Number of engine kernel launches issued by this context so far. */
int gw_launch_count(gw_ctx* ctx, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* GATEWAVE_B200_H */
