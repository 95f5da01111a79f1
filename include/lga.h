/*
 * lga.h -- C ABI of the B200-native layered-gradient-accumulation (LGA) training step.
 *
 * Paper: "Layered gradient accumulation and modular pipeline parallelism: fast and
 * efficient training of large language models", arXiv 2106.02679.  Citations "P:L" are
 * line L of its text; DESIGN.md lists the readings taken where it is silent.
 *
 * What one lga_step computes:
 *   a dense stack of L pre-LN transformer layers (width d, `heads` heads, FFN 4d),
 *   trained with mixed precision and Adam on a training state partitioned over the D
 *   data-parallel replicas (ZeRO stage 3, P:67 footnote).  Every layer runs forward, and
 *   later recompute + backward, over ALL N micro-batches back to back ("we process all
 *   the micro-batches for a given layer before proceeding to the next one"); its
 *   parameters are all-gathered once per pass and its gradients reduce-scattered once per
 *   step ("the same bandwidth as without gradient accumulation"), overlapped with
 *   the neighbouring layer's compute on side streams (mixed buffering).  With
 *   P > 1, layer i lives on pipeline stage i mod P (modular pipeline) and
 *   activations / their gradients cross stages after every layer.
 *   LGA_FLAG_* select the memory-rich variants and the contiguous pipeline map.
 *
 * Rank grid: world = D * P ranks, one process per GPU.  stage = rank mod P,
 * replica = rank div P.  Replica r owns global micro-batches r*N ... r*N+N-1 and shard r
 * of every layer of its stage.
 *
 * Conventions (all functions):
 *   - Every function returns lga_status (0 = OK); no exceptions cross the ABI and the
 *     library never calls exit/abort.  lga_last_error() returns a thread-local detail
 *     string (file:line plus the CUDA / NCCL message) for the last failing call.
 *   - A bad argument returns LGA_ERR_INVALID_ARG (or _UNSUPPORTED / _SIZE_MISMATCH) with
 *     no side effects.  A CUDA or NCCL failure returns LGA_ERR_CUDA / LGA_ERR_NCCL and
 *     latches the handle: every later call except lga_destroy returns LGA_ERR_BAD_STATE.
 *   - Ownership: the caller owns every pointer it passes (x, target, out, init_params)
 *     and keeps it valid until the call returns (host buffers) or until the work ordered
 *     on `cuda_stream` completes (device buffers, like cudaMemcpyAsync).  The library owns
 *     its device arena and its NCCL communicators and frees both in lga_destroy.
 *   - Collective calls (lga_init, lga_step*, lga_grads, lga_params) must be made by all
 *     world ranks in the same order.  lga_comm_bytes, lga_layer_stage, lga_timing and
 *     lga_param_count are local.
 *   - A handle is single-threaded; one handle per process / GPU.
 */
#ifndef LGA_H_
#define LGA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LGA_ABI_VERSION 3u
#define LGA_NCCL_ID_BYTES 128

typedef enum {
  LGA_OK = 0,
  LGA_ERR_INVALID_ARG = 1,
  LGA_ERR_UNSUPPORTED = 2,
  LGA_ERR_OUT_OF_MEMORY = 3,
  LGA_ERR_CUDA = 4,
  LGA_ERR_NCCL = 5,
  LGA_ERR_SIZE_MISMATCH = 6,
  LGA_ERR_BAD_STATE = 7
} lga_status;

/* Arithmetic of the step.  LGA_FP32: every kernel computes and stores in fp32 (parity
 * mode; any head size).  LGA_BF16: the paper's mixed precision:
 * bf16 GEMM / attention operands on the tcgen05 tensor cores with fp32 accumulation,
 * fp32 residual stream and checkpoints (reading A-8), bf16 all-gather / reduce-scatter
 * (reading A-7), fp32 master weights and Adam state.  Requires d % 64 == 0 and
 * d / heads in {64, 128}. */
typedef enum { LGA_FP32 = 0, LGA_BF16 = 1 } lga_precision;

/* LGA_LAYERED: layer-major.  LGA_STANDARD: micro-batch-major gradient
 * accumulation with the same partition -- the comparison schedule, whose
 * all-gathers and reduce-scatters repeat per micro-batch.  STANDARD requires pp == 1. */
typedef enum { LGA_LAYERED = 0, LGA_STANDARD = 1 } lga_schedule;

/* flags */
#define LGA_FLAG_NO_COMM   0x1u  /* A/B timing only (exposed communication = T(step) - T(step without
                                    comm)): the first step communicates as usual, so the parameter slots
                                    hold real gathered weights; every later step skips every all-gather,
                                    reduce-scatter, all-reduce and pipeline transfer (the same kernels run,
                                    the results are then wrong); counters still count */
#define LGA_FLAG_NO_GRAPH  0x2u  /* run every step eagerly.  By default lga_step captures the whole step
                                    (all streams, NCCL calls included) into a CUDA graph at its second
                                    call and replays it while x / target keep their pointers; the first
                                    call and lga_step_host run eagerly */
#define LGA_FLAG_PROFILE   0x4u  /* record CUDA events around every GEMM / attention / AdamW launch
                                    (on the stream it is launched on) for lga_timing_last */
/* Memory-rich variants and the contiguous pipeline (N3).  All require
 * LGA_LAYERED (INVALID_ARG otherwise); results are the same gradient / update up to rounding. */
#define LGA_FLAG_KEEP_PARAMS   0x8u   /* N2a: keep each layer's forward all-gather until its backward
                                         (L/P gathered layers resident): 1 all-gather + 1 reduce-scatter
                                         per layer per step instead of 2 + 1 (reading A-6 relaxed) */
#define LGA_FLAG_NO_RECOMPUTE  0x10u  /* N2c: keep every layer's intermediates for all N micro-batches
                                         (about 28 d B per token per layer) and skip the backward's
                                         forward recompute; recompute_units = 0 */
#define LGA_FLAG_UNPARTITIONED 0x20u  /* N2b: no training-state partition: every replica holds the full
                                         fp32 master / m / v of its stage's layers and all-reduces each
                                         layer's gradient once per step; no all-gather */
#define LGA_FLAG_NCCL_DP       0x80u  /* baseline for A/B: data-parallel all-gather / reduce-scatter with NCCL.
                                         Default (partitioned LAYERED, D > 1): over NVLink peer memory --
                                         copy-engine all-gathers, reduce-scatter fused into the AdamW kernel
                                         (fixed rank order), per-layer peer flags */
#define LGA_FLAG_CONTIGUOUS_PP 0x40u  /* N3: contiguous pipeline map, layer i on stage i / (L/P) (the
                                         standard layout of P:71) instead of the modular i mod P;
                                         activations cross stages only at block boundaries */
#define LGA_FLAG_POST_LN       0x100u /* N4: post-LN layer of the original encoder (reading A-16),
                                         h1 = LN1(x + Attn(x)), y = LN2(h1 + FFN(h1)); same parameters and
                                         layout.  Default: pre-LN (reading A-1).  Any schedule / variant */

typedef struct {
  uint32_t abi_version;    /* must be LGA_ABI_VERSION */
  int32_t layers;          /* L  = d_l */
  int32_t d_model;         /* d  = d_m = d_a * d_h */
  int32_t heads;           /* d_a */
  int32_t seq_len;         /* s  = d_s */
  int32_t micro_batch;     /* b  = b_mu, sequences per micro-batch */
  int32_t n_micro;         /* N  = n_mu, micro-batches per replica per step */
  int32_t dp;              /* D  = n_b, data-parallel degree */
  int32_t pp;              /* P  = n_l, pipeline degree; L % P == 0, N >= P */
  int32_t ffn_mult;        /* n_I, must be 4 */
  int32_t precision;       /* lga_precision */
  int32_t schedule;        /* lga_schedule */
  int32_t causal;          /* 1 = causal self-attention (GPT), 0 = the paper's encoder */
  int32_t chunk;           /* micro-batches per kernel launch, 1..N (N/P when pp>1); 0 = auto: N when pp == 1,
                              else the largest divisor of N <= N/P with chunk * b * s <= 8192 tokens */
  float lr, beta1, beta2, adam_eps, weight_decay;   /* AdamW, torch semantics (reading A-4) */
  float ln_eps;            /* LayerNorm epsilon (biased variance), 1e-5 */
  int32_t retain_grads;    /* keep each step's reduced fp32 gradient shard for lga_grads */
  uint32_t flags;          /* LGA_FLAG_* */
} lga_config;

/* Exact per-rank integers (closed forms: DESIGN.md "Counters"; P:67, P:565, P:576, P:583,
 * P:598).  all-gather bytes = bytes this rank RECEIVES; reduce-scatter bytes = bytes it
 * SENDS; *_units count logical (micro-batch, layer) pairs regardless of `chunk`.
 * allreduce_calls counts the per-step loss all-reduce plus (LGA_FLAG_UNPARTITIONED) one
 * gradient all-reduce per layer; allreduce_bytes = bytes a rank SENDS in the gradient
 * all-reduces (ring: 2 (D-1)/D of the padded layer), the 8-byte loss excluded. */
typedef struct {
  uint64_t steps;
  uint64_t ag_calls, rs_calls, p2p_send_calls, p2p_recv_calls, allreduce_calls;
  uint64_t ag_bytes, rs_bytes, p2p_send_bytes, p2p_recv_bytes;
  uint64_t fwd_units, bwd_units, recompute_units;
  uint64_t allreduce_bytes;
} lga_comm_stats;

/* Device-measured timing of the last step (CUDA events on the library's streams). */
typedef struct {
  float step_ms;          /* caller-stream start to step completion */
  float comm_wait_ms;     /* exposed data-parallel communication: the sum of compute-stream stalls on
                             all-gathers, staging-buffer reuse, the peer loss all-reduce, and the
                             step-end join of the last reduce-scatter + AdamW (the tail) */
  float p2p_wait_ms;      /* sum of compute-stream stalls waiting on pipeline receives */
  float fwd_ms, bwd_ms;   /* compute-stream time of the forward / backward passes */
  /* Per kernel family, only with LGA_FLAG_PROFILE (else 0): summed device time of the
   * launches, launch count, and the ALGORITHMIC work they did (GEMM: 2 M N K flops per
   * launch; attention: 2 d_h s(s+1) per (sequence, head) forward for the causal triangle,
   * 2x that backward; AdamW: bytes = (g + 3x4 read + 3x4 written + param) per element). */
  float gemm_ms, attn_ms, adam_ms;
  uint32_t gemm_launches, attn_launches, adam_launches;
  double gemm_flop, attn_flop, adam_bytes;
  uint64_t kernel_launches;  /* every kernel this library launched in the step (NCCL excluded) */
  uint64_t graph_captures;   /* step graphs captured since lga_init (a small cache keyed by the x / target
                                pointers: alternating two input buffers captures twice, then replays) */
} lga_timing;

typedef struct lga_handle lga_handle;

uint32_t lga_abi_version(void);
const char* lga_status_string(lga_status s);
const char* lga_last_error(void);

/* Parameter counts: per_layer = P_l = 12 d^2 + 13 d, total = L * P_l.
 * Either output may be NULL. */
lga_status lga_param_count(const lga_config* cfg, uint64_t* per_layer, uint64_t* total);

/* The host-side plan of one rank, exactly as lga_init derives it (no device work; callable on a machine without
 * a GPU): its stage and replica (rank grid above), its local layers (first_layer, first_layer + layer_stride,
 * ... : i mod P = stage for the modular map P:127, a contiguous block with LGA_FLAG_CONTIGUOUS_PP), the
 * micro-batches per kernel launch (chunk), the per-step pipeline transfers it sends / receives in forward and
 * backward (the targets of its flag waits; their sum is lga_comm_stats.p2p_send_calls / p2p_recv_calls,
 * P:598), and its training-state shard (S = padded layer / D elements per layer, reading A-10).
 * Errors: as lga_init's configuration checks. */
typedef struct {
  int32_t stage, replica, local_layers, chunk;
  int32_t first_layer, layer_stride;
  uint64_t p2p_send_fwd, p2p_recv_fwd, p2p_send_bwd, p2p_recv_bwd;
  uint64_t shard_elems, layer_elems_padded;
} lga_rank_plan;
lga_status lga_plan(const lga_config* cfg, int32_t rank, int32_t world, lga_rank_plan* out);

/* Fill `out` (LGA_NCCL_ID_BYTES bytes, host) with a fresh NCCL unique id.  Rank 0 calls
 * it and the caller broadcasts the bytes to every rank (e.g. over torch.distributed)
 * before lga_init.  Needed only for the NCCL baseline (LGA_FLAG_NCCL_DP with dp > 1). */
lga_status lga_nccl_unique_id(uint8_t* out);

/* Host all-gather supplied by the caller for the bootstrap of a world > 1 (the CUDA IPC
 * handles of every rank's arena and their offsets): copy `bytes`
 * bytes from `send` into recv + r * bytes of EVERY rank r, in rank order, and return 0
 * (non-zero = failure, lga_init then returns LGA_ERR_INVALID_ARG).  Called only from
 * inside lga_init, on the calling thread; torch.distributed.all_gather_object over any
 * backend (gloo included) is a valid implementation.  `ctx` is passed through. */
typedef int32_t (*lga_allgather_fn)(void* ctx, const void* send, void* recv, uint64_t bytes);

/* Create the per-rank state.  Collective over all `world` ranks.
 *   cfg          configuration (copied).
 *   rank, world  this process's rank and the world size; world must equal dp * pp.
 *   device       CUDA device ordinal this rank uses (the library calls cudaSetDevice).
 *                Several ranks may share one device (CUDA IPC works between processes
 *                on one GPU; the peer-memory paths then run time-sliced).
 *   allgather,   host all-gather for the bootstrap; required when world > 1 unless
 *   allgather_ctx  nccl_id is given (the exchange then runs over NCCL); ignored if world == 1.
 *   nccl_id      LGA_NCCL_ID_BYTES from lga_nccl_unique_id on rank 0, or NULL.  Required
 *                only by LGA_FLAG_NCCL_DP with dp > 1 (INVALID_ARG otherwise); every
 *                other data path -- all-gathers, reduce-scatters, the unpartitioned
 *                all-reduce, pipeline transfers, the loss all-reduce -- runs over CUDA IPC
 *                peer memory, so one GPU can host several ranks.  (SURVEY 8(b) sketched a
 *                borrowed NCCL communicator; DESIGN.md "Boundary" records the change.)
 *   cuda_stream  borrowed cudaStream_t (0 = legacy default stream) the caller orders its
 *                work on; lga_step consumes inputs and publishes results on it.
 *   init_params  host fp32, canonical layout of ALL L layers (L * P_l floats, layout in
 *                DESIGN.md "Canonical parameter layout"; each rank keeps only its stage's
 *                layers and its shard); NULL = on-device seeded init ("train" recipe,
 *                DESIGN.md "Inputs") from `seed`.
 * On any error *out stays NULL and everything allocated so far is freed.
 * Errors: INVALID_ARG (d % heads, L % pp, world != dp*pp, N < pp, schedule/pp, chunk,
 *         a variant flag with LGA_STANDARD, no bootstrap for world > 1, a failing
 *         allgather, NCCL_DP without nccl_id),
 *         UNSUPPORTED (bf16 with d % 64 != 0 or head size not 64/128; ffn_mult != 4),
 *         OUT_OF_MEMORY, CUDA, NCCL. */
lga_status lga_init(const lga_config* cfg, int32_t rank, int32_t world, int32_t device,
                    lga_allgather_fn allgather, void* allgather_ctx, const uint8_t* nccl_id,
                    uintptr_t cuda_stream, const float* init_params, uint64_t seed, lga_handle** out);

/* One training step: forward + loss + recompute/backward + reduce-scatter + AdamW.
 *   x, target   DEVICE fp32 [N][b][s][d] (row-major, this replica's micro-batches).  x is
 *               read only by stage 0 and target only by the stage owning layer L-1; other
 *               stages may pass NULL.
 *   loss_out    if non-NULL, the step's global loss (mean over all D*N micro-batches of
 *               1/2 mean((y - T)^2), reading A-2) is written after a host sync; NULL keeps
 *               the call asynchronous with respect to the host. */
lga_status lga_step(lga_handle* h, const float* x, const float* target, double* loss_out);

/* Same as lga_step with HOST inputs: x and target (host, same layout, pinned or pageable)
 * are copied to the device inside the call; the end-to-end path of bench.py's "e2e".  The
 * call returns only after both copies have completed, so the caller may refill or free x
 * and target as soon as it returns (loss_out NULL or not). */
lga_status lga_step_host(lga_handle* h, const float* x, const float* target, double* loss_out);

/* The last step's reduced gradient dL/dtheta (fp32, canonical layout), requires
 * retain_grads.  pp == 1: all L layers (n = L * P_l); pp > 1: this stage's layers in
 * ascending order (n = (L/pp) * P_l).  Collective over all world ranks: the shards of the
 * replicas are read over peer memory between two device barriers.
 * out_on_device: 1 = `out` is a device pointer, 0 = host.  SIZE_MISMATCH if n differs. */
lga_status lga_grads(lga_handle* h, float* out, uint64_t n, int32_t out_on_device);

/* Current fp32 master parameters, same layout / size rules as lga_grads. */
lga_status lga_params(lga_handle* h, float* out, uint64_t n, int32_t out_on_device);

/* Checkpoint / resume of this rank's training state: a small header (configuration, rank, AdamW step t)
 * followed by the fp32 master shard, Adam m and v of its stage's layers ([3][L/P][S] floats, S = padded
 * layer / D, or the whole padded layer with LGA_FLAG_UNPARTITIONED).  lga_state_bytes gives the size;
 * lga_save_state copies the state into `host_out` after the last step completed; lga_load_state restores it
 * into a handle of the same configuration and rank (INVALID_ARG otherwise), refreshes the 16-bit parameter
 * shard and sets t, so the next lga_step continues the run bit for bit (SIZE_MISMATCH if `bytes` differs).
 * Every rank saves / loads its own shard between the same two steps.  lga_save_state is local;
 * lga_load_state is collective for world > 1: it returns after every rank has restored its shard (the
 * next step's all-gathers read peers' shards), LGA_ERR_CUDA if a peer does not arrive within 600 s. */
lga_status lga_state_bytes(const lga_handle* h, uint64_t* bytes);
lga_status lga_save_state(lga_handle* h, void* host_out, uint64_t bytes);
lga_status lga_load_state(lga_handle* h, const void* host_in, uint64_t bytes);

/* Counters for the last step and the running total (either may be NULL).  Host only. */
lga_status lga_comm_bytes(const lga_handle* h, lga_comm_stats* last_step, lga_comm_stats* total);

/* stage_of_layer[i] = i mod P for i < L (modular), or i / (L/P) with
 * LGA_FLAG_CONTIGUOUS_PP; n must equal L. */
lga_status lga_layer_stage(const lga_handle* h, int32_t* stage_of_layer, int32_t n);

/* Device timing of the last step (synchronises the step's completion event). */
lga_status lga_timing_last(lga_handle* h, lga_timing* out);

/* Free everything the handle owns.  Collective: waits for this rank's last step on the
 * caller stream, then for every rank to arrive (device barrier over peer memory, 60 s
 * timeout) before unmapping the peers' arenas and freeing its own, which peers write into. */
void lga_destroy(lga_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* LGA_H_ */
