// lga_host.cpp -- the C ABI (include/lga.h), the per-rank arena, the layer executor and the
// per-layer scheduler of the layered-gradient-accumulation step.
//
// Schedule:
//   s_comp  : layer compute, all micro-batches of a layer before the next layer
//   s_comm  : all-gather of layer l+1 ("Restore(i+1)") while s_comp runs layer l; in backward,
//             reduce-scatter + AdamW of layer l ("Reduce(i)") while s_comp runs layer l-1
//             (mixed buffering: 2 parameter slots, 1 fp32 accumulation buffer)
//   pipeline: layer i on stage i mod P; the FFN2 epilogue of layer i writes x_{i+1}
//             straight into stage (i+1) mod P's checkpoint buffer over NVLink (CUDA IPC), the
//             LN1 backward of layer i writes dX_i into stage (i-1) mod P's gradient buffer,
//             and a system-scope flag tells the receiver.
#include "../../include/lga.h"
#include "kernels.cuh"

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <string>
#include <vector>

namespace lga {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

static lga_status set_err(lga_status s, const char* file, int line, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  char full[1200];
  snprintf(full, sizeof(full), "%s:%d: %s", file, line, buf);
  g_last_error = full;
  return s;
}
#define ERR(s, ...) set_err((s), __FILE__, __LINE__, __VA_ARGS__)

struct StatusError {
  lga_status s;
};

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      ERR(LGA_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));                       \
      throw StatusError{LGA_ERR_CUDA};                                                  \
    }                                                                                   \
  } while (0)
#define NK(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) {                                                            \
      ERR(LGA_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_));                       \
      throw StatusError{LGA_ERR_NCCL};                                                  \
    }                                                                                   \
  } while (0)
#define KCHECK() CK(cudaGetLastError())

// ------------------------------------------------------------------ configuration
struct Cfg {
  int L, d, H, dh, s, b, N, D, P, f, M, c, Lloc;
  int64_t pl, plpad, S;
  bool bf16, layered, causal;
  DT E, G;      // compute storage type; reduce-scatter / gradient staging type
  float lr, b1, b2, eps, wd, ln_eps;
  bool retain, no_comm, profile;
  bool keep, norecomp, unpart, contig;   // LGA_FLAG_KEEP_PARAMS / NO_RECOMPUTE / UNPARTITIONED / CONTIGUOUS_PP
  bool graph_off;                        // LGA_FLAG_NO_GRAPH
  bool dp_ipc;                           // D > 1: all-gather / reduce-scatter / all-reduce over peer memory
  bool nccl_dp;                          // D > 1 with LGA_FLAG_NCCL_DP: the NCCL baseline
  bool post_ln;                          // LGA_FLAG_POST_LN (reading A-16)
  // canonical offsets
  int64_t o_ln1w, o_ln1b, o_wqkv, o_bqkv, o_wo, o_bo, o_ln2w, o_ln2b, o_w1, o_b1, o_w2, o_b2;
};

static lga_status validate(const lga_config* c, int world, Cfg* out) {
  if (!c) return ERR(LGA_ERR_INVALID_ARG, "cfg is NULL");
  if (c->abi_version != LGA_ABI_VERSION) return ERR(LGA_ERR_INVALID_ARG, "abi_version %u != %u", c->abi_version, LGA_ABI_VERSION);
  if (c->layers <= 0 || c->d_model <= 0 || c->heads <= 0 || c->seq_len <= 0 || c->micro_batch <= 0 || c->n_micro <= 0 ||
      c->dp <= 0 || c->pp <= 0)
    return ERR(LGA_ERR_INVALID_ARG, "non-positive dimension");
  if (c->d_model % c->heads) return ERR(LGA_ERR_INVALID_ARG, "d_model %% heads != 0");
  if (c->ffn_mult != 4) return ERR(LGA_ERR_UNSUPPORTED, "ffn_mult must be 4 (P:440)");
  if (c->layers % c->pp) return ERR(LGA_ERR_INVALID_ARG, "layers %% pp != 0 (reading A-11)");
  if (c->pp > 1 && c->n_micro < c->pp) return ERR(LGA_ERR_INVALID_ARG, "n_micro < pp (reading A-11)");
  if (world != c->dp * c->pp) return ERR(LGA_ERR_INVALID_ARG, "world %d != dp*pp %d", world, c->dp * c->pp);
  if (c->schedule != LGA_LAYERED && c->schedule != LGA_STANDARD) return ERR(LGA_ERR_INVALID_ARG, "bad schedule");
  if (c->schedule == LGA_STANDARD && c->pp != 1) return ERR(LGA_ERR_INVALID_ARG, "STANDARD requires pp == 1");
  if (c->precision != LGA_FP32 && c->precision != LGA_BF16) return ERR(LGA_ERR_INVALID_ARG, "bad precision");
  const int dh = c->d_model / c->heads;
  if (c->precision == LGA_BF16 && (c->d_model % 64 || (dh != 64 && dh != 128)))
    return ERR(LGA_ERR_UNSUPPORTED, "bf16 needs d %% 64 == 0 and head size 64 or 128 (got d=%d dh=%d)", c->d_model, dh);
  if (c->precision == LGA_FP32 && dh > 128) return ERR(LGA_ERR_UNSUPPORTED, "head size > 128");
  const int cmax = c->pp > 1 ? c->n_micro / c->pp : c->n_micro;
  if (c->chunk < 0 || c->chunk > cmax) return ERR(LGA_ERR_INVALID_ARG, "chunk %d not in [0, %d]", c->chunk, cmax);
  if (c->chunk > 0 && c->n_micro % c->chunk) return ERR(LGA_ERR_INVALID_ARG, "n_micro %% chunk != 0");
  if (!(c->lr >= 0.f) || !(c->beta1 >= 0.f && c->beta1 < 1.f) || !(c->beta2 >= 0.f && c->beta2 < 1.f) || !(c->adam_eps > 0.f) ||
      !(c->ln_eps > 0.f))
    return ERR(LGA_ERR_INVALID_ARG, "bad optimizer / LayerNorm hyper-parameter");
  if ((int64_t)c->micro_batch * c->seq_len * c->n_micro > (int64_t)1 << 30) return ERR(LGA_ERR_UNSUPPORTED, "batch too large");
  const uint32_t variants = LGA_FLAG_KEEP_PARAMS | LGA_FLAG_NO_RECOMPUTE | LGA_FLAG_UNPARTITIONED | LGA_FLAG_CONTIGUOUS_PP;
  if ((c->flags & variants) && c->schedule != LGA_LAYERED)
    return ERR(LGA_ERR_INVALID_ARG, "variant flags 0x%x require LGA_LAYERED", c->flags & variants);

  Cfg g{};
  g.L = c->layers; g.d = c->d_model; g.H = c->heads; g.dh = dh; g.s = c->seq_len; g.b = c->micro_batch;
  g.N = c->n_micro; g.D = c->dp; g.P = c->pp; g.f = 4 * g.d; g.M = g.b * g.s; g.Lloc = g.L / g.P;
  // default chunk: all micro-batches of a layer in one launch (P=1).  Under the pipeline, the largest divisor c of
  // N with c P <= N (the next stage must start before this one finishes the layer) and c b s <= 8192
  // tokens: fewer, larger launches than one micro-batch each (M = 2048-token GEMMs leave SMs idle) for a bubble of
  // (P-1) P c / (N L) -- measured at C4 (P = 4): c = 1 / 2 / 4 / 8 -> 1344 / 1221 / 1174 / 1186 ms (reading A-13)
  if (c->chunk > 0) {
    g.c = c->chunk;
  } else if (g.P > 1) {
    g.c = 1;
    for (int cc = g.N / g.P; cc >= 1; --cc)
      if (g.N % cc == 0 && (int64_t)cc * g.M <= 8192) { g.c = cc; break; }
  } else {
    g.c = g.N;
  }
  if (c->schedule == LGA_STANDARD) g.c = 1;
  g.pl = 12LL * g.d * g.d + 13LL * g.d;
  const int64_t q = 64LL * g.D;
  g.plpad = (g.pl + q - 1) / q * q;
  g.unpart = (c->flags & LGA_FLAG_UNPARTITIONED) != 0;
  g.S = g.unpart ? g.plpad : g.plpad / g.D;   // state elements per layer on this rank
  g.keep = (c->flags & LGA_FLAG_KEEP_PARAMS) != 0;
  g.norecomp = (c->flags & LGA_FLAG_NO_RECOMPUTE) != 0;
  g.contig = (c->flags & LGA_FLAG_CONTIGUOUS_PP) != 0;
  g.graph_off = (c->flags & LGA_FLAG_NO_GRAPH) != 0;
  g.bf16 = c->precision == LGA_BF16;
  g.layered = c->schedule == LGA_LAYERED;
  // N1: data parallelism over peer memory (every schedule and variant) unless LGA_FLAG_NCCL_DP asks for NCCL
  g.nccl_dp = g.D > 1 && (c->flags & LGA_FLAG_NCCL_DP) != 0;
  g.dp_ipc = g.D > 1 && !g.nccl_dp;
  g.post_ln = (c->flags & LGA_FLAG_POST_LN) != 0;
  g.causal = c->causal != 0;
  g.E = g.bf16 ? DT::BF16 : DT::F32;
  g.G = (g.bf16 && g.D > 1) ? DT::BF16 : DT::F32;   // 16-bit reduction only when there is a reduction (A-7)
  g.lr = c->lr; g.b1 = c->beta1; g.b2 = c->beta2; g.eps = c->adam_eps; g.wd = c->weight_decay; g.ln_eps = c->ln_eps;
  g.retain = c->retain_grads != 0;
  g.no_comm = (c->flags & LGA_FLAG_NO_COMM) != 0;
  g.profile = (c->flags & LGA_FLAG_PROFILE) != 0;
  const int64_t d = g.d, f = g.f;
  g.o_ln1w = 0; g.o_ln1b = d; g.o_wqkv = 2 * d; g.o_bqkv = g.o_wqkv + 3 * d * d; g.o_wo = g.o_bqkv + 3 * d;
  g.o_bo = g.o_wo + d * d; g.o_ln2w = g.o_bo + d; g.o_ln2b = g.o_ln2w + d; g.o_w1 = g.o_ln2b + d;
  g.o_b1 = g.o_w1 + d * f; g.o_w2 = g.o_b1 + f; g.o_b2 = g.o_w2 + f * d;
  if (g.o_b2 + d != g.pl) return ERR(LGA_ERR_INVALID_ARG, "internal layout error");
  *out = g;
  return LGA_OK;
}

// ------------------------------------------------------------------ arena (one allocation, M10 / P:96)
// Guard mode (env LGA_ARENA_GUARD=1; compute-sanitizer is unavailable on the GPU pool): every buffer is
// followed by a GUARD-byte canary filled with a pattern at init; lgatest_arena_guard_check counts the
// canary bytes a kernel overwrote -- an out-of-bounds write past the end of any arena buffer.
constexpr size_t GUARD = 4096;
constexpr unsigned char GUARD_BYTE = 0xA5;
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  bool planning = true;
  bool guard = false;
  std::vector<size_t> guards;   // offsets of the canaries (guard mode)
  template <typename T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    T* p = planning ? nullptr : reinterpret_cast<T*>(base + used);
    used += bytes;
    if (guard) {
      if (!planning) guards.push_back(used);
      used += GUARD;
    }
    return p;
  }
  void* take_bytes(size_t bytes) { return take<char>(bytes); }
};

// What a rank publishes about its arena at the bootstrap (exchanged with the caller's all-gather)
struct PeerInfo {
  cudaIpcMemHandle_t handle;
  uint64_t off_ckpt, off_dY, off_flags;   // pipeline
  uint64_t off_gst, off_psh, off_dpf;     // data parallelism over peer memory (N1)
  uint64_t off_master, off_gkeep;         // lga_params / lga_grads read the replicas' shards
  uint64_t off_wflags, off_loss;          // world counters (loss all-reduce, barrier), loss ring
  int32_t rank, world;                    // consistency check
  uint64_t pad;
};
static_assert(sizeof(PeerInfo) % 16 == 0, "PeerInfo size");

// Per-layer peer counters of the data-parallel group, dpf[kind * Lloc + j], each bumped by every replica:
//   GRAD  "my gradient of layer j is staged"        PARAM "my shard j is updated"
//   READ  "I read the shards of layer j" (gathers; unpartitioned: "I read the reduced slices")
//   RED   "my reduced slice of layer j is ready"    (unpartitioned all-reduce, between its two phases)
//   GREAD "I read my slice of your staging j"       (STANDARD: staging j is rewritten every micro-batch)
enum { DPF_GRAD = 0, DPF_PARAM = 1, DPF_READ = 2, DPF_RED = 3, DPF_GREAD = 4, DPF_KINDS = 5 };

// Forward intermediates of a chunk that the backward reads (pointers at the chunk's first token).
struct Ws {
  void *a = nullptr, *qkv = nullptr, *o = nullptr, *cn = nullptr, *u = nullptr, *g = nullptr;
  float *h1 = nullptr, *lse = nullptr;
  float2 *st1 = nullptr, *st2 = nullptr;
  // post-LN only: hn = LN1(s1) in fp32 (FFN2 residual; bf16 mode, else cn), s2 = h1 + FFN(h1) (LN2 input)
  float *hn = nullptr, *s2 = nullptr;
};

}  // namespace lga

using namespace lga;

struct lga_handle {
  Cfg c{};
  int rank = 0, world = 1, stage = 0, replica = 0, dev = 0;
  bool bad = false;
  cudaStream_t user = nullptr, s_comp = nullptr, s_comm = nullptr, s_copy = nullptr;
  bool tin_pending = false;   // lga_step_host: the target copy (on s_copy) not yet awaited by the loss
  bool x_split = false;       // lga_step_host: x copied per micro-batch on s_copy (ev_x[m]); layer 0 follows
  std::vector<cudaEvent_t> ev_x;
  ncclComm_t world_comm = nullptr, dp_comm = nullptr;
  Arena arena;
  // training state, per local layer j: [Lloc][S]
  float *master = nullptr, *mom = nullptr, *var = nullptr, *gkeep = nullptr, *gshard_acc = nullptr;
  void* pshard = nullptr;
  std::vector<void*> slot;   // gathered full layers: 2 (mixed buffering) or L/P (LGA_FLAG_KEEP_PARAMS)
  float* gacc = nullptr;
  void* gstage[2] = {nullptr, nullptr};   // staging of the reduced-precision layer gradient (alternating layers)
  void* gst_layers = nullptr;             // dp_ipc: one staging buffer per local layer [Lloc][plpad]
  // dp_ipc: per-layer counters [DPF_KINDS][Lloc] (gradient staged / shard updated / shard read / reduced slice
  // ready / staging read), written by the peers
  unsigned long long* dpf = nullptr;
  void** dp_gst_dev = nullptr;                   // device [D]: every DP peer's staging base (replica order)
  unsigned long long** dp_flag_dev = nullptr;    // device [D]: every DP peer's dpf
  std::vector<char*> dp_base;                    // host: IPC-mapped arena base of every DP peer (self: own)
  std::vector<char*> dp_psh;                     // host: every DP peer's pshard
  // world (bootstrap, loss all-reduce, barriers): every rank's arena mapped over CUDA IPC (self: own base)
  std::vector<char*> wbase;
  std::vector<PeerInfo> peers;
  bool connected = false;                        // every rank's arena mapped (world > 1)
  bool ready = false;                            // lga_init completed
  bool stepped = false;                          // ev_t1 recorded at least once
  // LGA_FLAG_NO_COMM A/B: the first step communicates (the parameter slots then hold real gathered weights,
  // so the A/B runs the same kernels on the same kind of data), every later step skips all transfers
  bool comm_off = false;
  unsigned long long* wflags = nullptr;          // [0] loss arrivals, [1] barrier arrivals (written by peers)
  double* loss_ring = nullptr;                   // [4][world] loss slots (written by peers)
  unsigned long long** w_flag_dev = nullptr;     // device [world]: every rank's wflags
  double** w_loss_dev = nullptr;                 // device [world]: every rank's loss_ring
  int* barrier_to = nullptr;                     // device: barrier timed out
  unsigned long long n_barrier = 0;              // barriers so far (collective, the same on every rank)
  // activations
  float* ckpt = nullptr;  // [Lloc][N][M][d]
  float* yout = nullptr;  // [N][M][d] on the stage owning layer L-1
  float* dY = nullptr;    // [N][M][d]
  float* dscratch = nullptr;  // [c][M][d] sink for dX of layer 0
  // forward intermediates the backward reads: one chunk-sized set, or (LGA_FLAG_NO_RECOMPUTE) one set
  // per local layer covering all N micro-batches
  std::vector<Ws> ws;
  // backward temporaries (chunk-sized)
  void *dYe = nullptr, *dh1e = nullptr, *dO = nullptr, *dqkv = nullptr;
  float *dC = nullptr, *dh1 = nullptr, *dsum = nullptr, *partial = nullptr;
  float* splitk_ws = nullptr;   // split-K partial sums of tile-starved GEMMs (small-d weight gradients)
  void* attn_ds = nullptr;      // dS^T of one chunk's attention backward (dQ from dS: 5 matmuls per block)
  int64_t splitk_floats = 0;
  double *mse_partial = nullptr, *loss_dev = nullptr, *loss_host = nullptr;
  float *xin = nullptr, *tin = nullptr;  // device copies for lga_step_host
  unsigned long long* flags = nullptr;   // [0] fwd receive count, [1] bwd receive count
  // pipeline peers
  float *next_ckpt = nullptr, *prev_dY = nullptr;
  unsigned long long *next_flags = nullptr, *prev_flags = nullptr;
  unsigned long long sent_fwd = 0, sent_bwd = 0, recv_fwd = 0, recv_bwd = 0;   // this step's transfers so far
  unsigned long long k_send_fwd = 0, k_send_bwd = 0, k_recv_fwd = 0, k_recv_bwd = 0;   // per step (stage map)
  long long* tstep = nullptr;   // device AdamW step t (from 1; restored by lga_load_state): bias corrections
  long long* tepoch = nullptr;  // device count of steps run by this handle: targets of every peer / pipeline flag
  // cross-step event waits are redundant (every step starts after the previous one completed) and illegal
  // inside a stream capture: only wait on events recorded earlier in the same step
  bool rec_adam[2] = {false, false};
  std::vector<char> rec_slot;
  // CUDA graph of lga_step (captured at the second call, replayed while x / target keep their pointers)
  bool capturing = false, graph_broken = false;
  int eager_steps = 0;
  // a small cache keyed by the (x, target) pointers: a data loader that double-buffers its inputs replays
  // two graphs instead of re-capturing every step
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    const float *x = nullptr, *T = nullptr;
    lga_comm_stats last{};
    int nwait = 0, nprof = 0;
    unsigned long long launches = 0, used = 0;
  };
  static constexpr int kGraphs = 2;
  StepGraph graphs[kGraphs];
  unsigned long long graph_clock = 0, graph_captures = 0;
  int64_t partial_floats = 0;
  // events
  std::vector<cudaEvent_t> ev_ag, ev_slot_free;   // per slot
  cudaEvent_t ev_in = nullptr, ev_tin = nullptr, ev_grad[2] = {}, ev_adam[2] = {}, ev_comm_end = nullptr,
              ev_comp_end = nullptr, ev_t0 = nullptr, ev_t1 = nullptr, ev_fwd_end = nullptr;
  std::vector<cudaEvent_t> ev_wait0, ev_wait1;   // stall accounting pairs (s_comp)
  std::vector<int> wait_kind;
  int n_wait = 0;
  // per-family profiling (LGA_FLAG_PROFILE): event pairs on the launching stream
  std::vector<cudaEvent_t> prof0, prof1;
  std::vector<int> prof_fam;
  std::vector<double> prof_work;
  int n_prof = 0;
  unsigned long long launches_at_start = 0, launches_last = 0;
  int64_t t = 0;  // AdamW step counter
  lga_comm_stats last{}, total{};
};

namespace lga {

// pipeline map: modular, layer i on stage i mod P; contiguous, stage i / (L/P)
static int stage_of(const Cfg& c, int64_t i) { return c.contig ? (int)(i / c.Lloc) : (int)(i % c.P); }
static int local_index(const Cfg& c, int64_t i) { return c.contig ? (int)(i % c.Lloc) : (int)(i / c.P); }
static int64_t local_to_global_s(const Cfg& c, int stage, int j) {
  return c.contig ? (int64_t)stage * c.Lloc + j : (int64_t)stage + (int64_t)j * c.P;
}
static int64_t local_to_global(const lga_handle* h, int j) { return local_to_global_s(h->c, h->stage, j); }
// Pipeline transfers per step of a stage (the flag epochs of the receive waits): N micro-batches at every
// layer boundary crossing to / from another stage, forward and backward.  Shared by lga_init and lga_plan.
static void plan_transfers(const Cfg& c, int stage, unsigned long long* send_fwd, unsigned long long* recv_fwd,
                           unsigned long long* send_bwd, unsigned long long* recv_bwd) {
  *send_fwd = *recv_fwd = *send_bwd = *recv_bwd = 0;
  for (int j = 0; j < c.Lloc && c.P > 1; ++j) {
    const int64_t i = local_to_global_s(c, stage, j);
    if (i > 0 && stage_of(c, i - 1) != stage) *recv_fwd += c.N, *send_bwd += c.N;
    if (i < c.L - 1 && stage_of(c, i + 1) != stage) *send_fwd += c.N, *recv_bwd += c.N;
  }
}
static bool owns_last(const lga_handle* h) { return stage_of(h->c, h->c.L - 1) == h->stage; }
static ncclDataType_t nccl_dt(DT t) { return t == DT::F32 ? ncclFloat32 : ncclBfloat16; }

static char* eoff(void* p, DT t, int64_t i) { return static_cast<char*>(p) + i * (int64_t)dt_size(t); }

static void plan_arena(lga_handle* h) {
  Arena& A = h->arena;
  const Cfg& c = h->c;
  const int64_t S = c.S, Ll = c.Lloc, T = (int64_t)c.c * c.M, d = c.d, f = c.f;
  const size_t e = dt_size(c.E);
  A.used = 0;
  h->master = A.take<float>(Ll * S);
  h->mom = A.take<float>(Ll * S);
  h->var = A.take<float>(Ll * S);
  h->pshard = A.take_bytes(Ll * S * e);
  h->gkeep = c.retain ? A.take<float>(Ll * S) : nullptr;
  h->gshard_acc = c.layered ? nullptr : A.take<float>(Ll * S);
  const int nslots = (c.D > 1 && !c.unpart) ? (c.keep ? (int)Ll : 2) : 0;
  h->slot.assign(nslots, nullptr);
  for (int k = 0; k < nslots; ++k) h->slot[k] = A.take_bytes(c.plpad * e);
  h->gacc = A.take<float>(c.plpad);
  if (c.dp_ipc) {   // a layer's staged gradient stays readable by the peers until the next step
    h->gst_layers = A.take_bytes(Ll * c.plpad * dt_size(c.G));
    h->dpf = A.take<unsigned long long>(DPF_KINDS * Ll);
    h->dp_gst_dev = A.take<void*>(c.D);
    h->dp_flag_dev = A.take<unsigned long long*>(c.D);
  } else {
    h->gstage[0] = A.take_bytes(c.plpad * dt_size(c.G));
    h->gstage[1] = A.take_bytes(c.plpad * dt_size(c.G));
  }
  const int64_t act = (int64_t)c.N * c.M * d;
  h->ckpt = A.take<float>(Ll * act);
  h->yout = A.take<float>(act);
  h->dY = A.take<float>(act);
  h->dscratch = A.take<float>(T * d);
  const int nws = c.norecomp ? (int)Ll : 1;
  const int64_t Tw = c.norecomp ? (int64_t)c.N * c.M : T;   // tokens per workspace set
  h->ws.assign(nws, Ws{});
  for (Ws& w : h->ws) {
    w.a = A.take_bytes(Tw * d * e);
    w.qkv = A.take_bytes(Tw * 3 * d * e);
    w.o = A.take_bytes(Tw * d * e);
    w.cn = A.take_bytes(Tw * d * e);
    w.u = A.take_bytes(Tw * f * e);
    w.g = A.take_bytes(Tw * f * e);
    w.h1 = A.take<float>(Tw * d);
    w.lse = A.take<float>(Tw / c.s * c.H * c.s);
    w.st1 = A.take<float2>(Tw);
    w.st2 = A.take<float2>(Tw);
    if (c.post_ln) {
      w.hn = c.bf16 ? A.take<float>(Tw * d) : nullptr;
      w.s2 = A.take<float>(Tw * d);
    }
  }
  h->dYe = A.take_bytes(T * d * e);
  h->dh1e = A.take_bytes(T * d * e);
  h->dO = A.take_bytes(T * d * e);
  h->dqkv = A.take_bytes(T * 3 * d * e);
  h->dC = A.take<float>(T * d);
  h->dh1 = A.take<float>(T * d);
  h->dsum = A.take<float>((int64_t)c.c * c.b * c.H * c.s);
  const int64_t pcol = (int64_t)colsum_blocks((int)T) * f;
  const int64_t pln = (int64_t)ln_bwd_blocks((int)T, (int)d) * 4 * d;   // 4 sums per block with `extra`
  const int64_t pgelu = (T + 31) / 32 * f;                                  // GELU-backward epilogue strips
  const int64_t pattn = (int64_t)c.c * c.b * ((c.s + 127) / 128) * 4 * 3 * d;   // attention-backward quadrants
  h->partial_floats = std::max(std::max(pcol, pln), std::max(pgelu, pattn));
  h->partial = A.take<float>(h->partial_floats);
  h->splitk_floats = c.bf16 ? std::min<int64_t>(16LL * 4 * d * d, (int64_t)1 << 25) : 0;
  h->splitk_ws = c.bf16 ? A.take<float>(h->splitk_floats) : nullptr;
  {   // bf16: [c b][heads][s128][s128] bf16 (LGA_ATTN_BWD=7 keeps the 7-matmul dQ kernel, no workspace)
    const char* v = getenv("LGA_ATTN_BWD");
    const bool seven = v && v[0] == '7';
    const int64_t s128 = (int64_t)(c.s + 127) / 128 * 128;
    h->attn_ds = (c.bf16 && !seven) ? A.take_bytes((size_t)c.c * c.b * c.H * s128 * s128 * 2) : nullptr;
  }
  h->mse_partial = A.take<double>(mse_blocks(act) + 64);
  h->loss_dev = A.take<double>(c.N + 8);
  h->xin = A.take<float>(act);
  h->tin = A.take<float>(act);
  h->flags = A.take<unsigned long long>(8);
  h->tstep = A.take<long long>(2);   // [0] AdamW step t, [1] steps run by this handle (flag epochs)
  h->tepoch = h->tstep ? h->tstep + 1 : nullptr;
  if (h->world > 1) {
    h->wflags = A.take<unsigned long long>(16);
    h->loss_ring = A.take<double>(4 * (int64_t)h->world);
    h->w_flag_dev = A.take<unsigned long long*>(h->world);
    h->w_loss_dev = A.take<double*>(h->world);
    h->barrier_to = A.take<int>(4);
  }
}

// timing events: plain records, or event-record nodes (cudaEventRecordExternal) inside a step capture
static void rec_time(lga_handle* h, cudaEvent_t ev, cudaStream_t st) {
  if (h->capturing) CK(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
  else CK(cudaEventRecord(ev, st));
}

// ------------------------------------------------------------------ profiling
enum { FAM_GEMM = 0, FAM_ATTN = 1, FAM_ADAM = 2 };
static int prof_begin(lga_handle* h, cudaStream_t st) {
  if (!h->c.profile) return -1;
  if (h->n_prof >= (int)h->prof0.size()) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    h->prof0.push_back(a);
    h->prof1.push_back(b);
    h->prof_fam.push_back(0);
    h->prof_work.push_back(0.0);
  }
  rec_time(h, h->prof0[h->n_prof], st);
  return h->n_prof++;
}
static void prof_end(lga_handle* h, int idx, cudaStream_t st, int fam, double work) {
  if (idx < 0) return;
  rec_time(h, h->prof1[idx], st);
  h->prof_fam[idx] = fam;
  h->prof_work[idx] = work;
}

// ------------------------------------------------------------------ GEMM dispatch
static void gemm(lga_handle* h, GemmArgs g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  const int p = prof_begin(h, st);
  if (h->c.bf16) {
    g.splitk_ws = h->splitk_ws;
    g.splitk_ws_floats = h->splitk_floats;
    CK(gemm_bf16_tc(g, st));
  } else {
    gemm_f32_simt(g, st);
  }
  KCHECK();
  prof_end(h, p, st, FAM_GEMM, 2.0 * g.M * (double)g.N * g.K);
}

// algorithmic attention flops of one forward over nseq sequences (causal triangle incl. diagonal)
static double attn_flops_fwd(const Cfg& c, int nseq) {
  const double s = c.s;
  const double pairs = c.causal ? s * (s + 1) / 2 : s * s;
  return 4.0 * c.dh * pairs * c.H * nseq;
}

// Gradient write mode of one chunk (reading A-3, subsystem (2)): where the chunk's gradient goes.
struct GradDst {
  const float* acc_in;  // fp32 accumulator to add (nullptr on the first chunk)
  void* out;            // fp32 accumulator (not last) or the staging buffer (last)
  DT out_dt;
};
// staging buffer of the gradient of local layer j: per layer (dp_ipc) or alternating
static void* stage_buf(lga_handle* h, int j) {
  if (h->gst_layers) return eoff(h->gst_layers, h->c.G, (int64_t)j * h->c.plpad);
  return h->gstage[j % 2];
}
static GradDst grad_dst(lga_handle* h, int chunk_idx, int nchunks, int j, int64_t off) {
  const bool first = chunk_idx == 0, last = chunk_idx == nchunks - 1;
  GradDst r;
  r.acc_in = first ? nullptr : h->gacc + off;
  if (last) {
    r.out = eoff(stage_buf(h, j), h->c.G, off);
    r.out_dt = h->c.G;
  } else {
    r.out = h->gacc + off;
    r.out_dt = DT::F32;
  }
  return r;
}

// LGA_TRACE=1: synchronise the compute stream and log after every layer pass (debugging hangs)
static bool trace_on() {
  static int t = -1;
  if (t < 0) {
    const char* v = getenv("LGA_TRACE");
    t = (v && v[0] == '1') ? 1 : 0;
  }
  return t == 1;
}
// NVTX ranges (env LGA_NVTX=1): "lga step t", "fwd layer i", "bwd layer i" around the host-side issue of each
// pass, so that ncu --nvtx-include / an NVTX-aware profiler can select one layer's kernels (eager steps; a
// replayed graph launches under the "lga step" range only)
static bool nvtx_on() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("LGA_NVTX");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}
struct NvtxRange {
  bool on;
  NvtxRange(const char* what, long long idx) : on(nvtx_on()) {
    if (!on) return;
    char buf[64];
    snprintf(buf, sizeof(buf), "%s %lld", what, idx);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};

static void trace(lga_handle* h, const char* what, int64_t layer) {
  if (!trace_on()) return;
  fprintf(stderr, "[lga rank %d stage %d] %s layer %lld issued\n", h->rank, h->stage, what, (long long)layer);
  CK(cudaStreamSynchronize(h->s_comp));
  fprintf(stderr, "[lga rank %d stage %d] %s layer %lld done\n", h->rank, h->stage, what, (long long)layer);
}

// ------------------------------------------------------------------ layer executor
// Forward of local layer j over micro-batches [m0, m0+c) (module docstring of kernels.cuh).
// x_in: [c][M][d] fp32; y_out: fp32 destination or nullptr (recompute: FFN2 not needed).
// cc: micro-batches in this launch (default the configured chunk c)
static void layer_fwd_post(lga_handle* h, const Ws& w, const void* W, const float* x_in, float* y_out, cudaStream_t st,
                           int cc);
static void layer_fwd(lga_handle* h, const Ws& w, const void* W, const float* x_in, float* y_out, cudaStream_t st,
                      int cc = -1) {
  const Cfg& c = h->c;
  if (cc < 0) cc = c.c;
  if (c.post_ln) return layer_fwd_post(h, w, W, x_in, y_out, st, cc);
  const int T = cc * c.M;
  const int d = c.d;
  const DT E = c.E;
  ln_fwd(x_in, eoff((void*)W, E, c.o_ln1w), eoff((void*)W, E, c.o_ln1b), E, w.a, E, w.st1, T, d, c.ln_eps, st);
  KCHECK();
  {  // qkv = a Wqkv + bqkv
    GemmArgs g;
    g.M = T; g.N = 3 * d; g.K = d;
    g.A = w.a; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wqkv); g.ldb = 3 * d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_bqkv); g.epi.bias_dt = E;
    g.epi.out = w.qkv; g.epi.ldo = 3 * d; g.epi.out_dt = E;
    gemm(h, g, st);
    trace(h, "  qkv gemm", -1);
  }
  {  // o = attention(q, k, v)
    AttnArgs a;
    a.nseq = cc * c.b; a.seq = c.s; a.heads = c.H; a.dh = c.dh; a.d = d; a.causal = c.causal;
    a.scale = 1.0f / sqrtf((float)c.dh);
    a.qkv = w.qkv; a.o = w.o; a.lse = w.lse;
    const int p = prof_begin(h, st);
    if (c.bf16) CK(attn_fwd_bf16(a, st)); else attn_fwd_f32(a, st);
    KCHECK();
    prof_end(h, p, st, FAM_ATTN, attn_flops_fwd(c, a.nseq));
    trace(h, "  attn fwd", -1);
  }
  {  // h1 = x + o Wo + bo
    GemmArgs g;
    g.M = T; g.N = d; g.K = d;
    g.A = w.o; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wo); g.ldb = d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_bo); g.epi.bias_dt = E;
    g.epi.res = x_in; g.epi.ldr = d;
    g.epi.out = w.h1; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
    trace(h, "  oproj gemm", -1);
  }
  ln_fwd(w.h1, eoff((void*)W, E, c.o_ln2w), eoff((void*)W, E, c.o_ln2b), E, w.cn, E, w.st2, T, d, c.ln_eps, st);
  KCHECK();
  {  // u = c W1 + b1 ; g = GELU(u).  u is read only by the backward's GELU': in the forward pass proper, when
     // the backward recomputes the layer, it is not stored (T x 4d x E bytes of HBM writes per layer)
    GemmArgs g;
    g.M = T; g.N = c.f; g.K = d;
    g.A = w.cn; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w1); g.ldb = c.f; g.b_kmajor = false;
    g.epi.kind = EPI_GELU_FWD; g.epi.bias = eoff((void*)W, E, c.o_b1); g.epi.bias_dt = E;
    g.epi.aux = (y_out && !c.norecomp) ? nullptr : w.u; g.epi.ldaux = c.f; g.epi.aux_dt = E;
    g.epi.out = w.g; g.epi.ldo = c.f; g.epi.out_dt = E;
    gemm(h, g, st);
    trace(h, "  ffn1 gemm", -1);
  }
  if (y_out) {  // y = h1 + g W2 + b2
    GemmArgs g;
    g.M = T; g.N = d; g.K = c.f;
    g.A = w.g; g.lda = c.f; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w2); g.ldb = d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_b2); g.epi.bias_dt = E;
    g.epi.res = w.h1; g.epi.ldr = d;
    g.epi.out = y_out; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
    trace(h, "  ffn2 gemm", -1);
  }
}

// Post-LN forward (reading A-16): a = x (cast to E for the QKV GEMM), s1 = x + Attn(a) Wo + bo (w.h1),
// h1 = LN1(s1) (E copy in cn, fp32 copy in hn), s2 = h1 + GELU(h1 W1 + b1) W2 + b2, y = LN2(s2).  The
// recompute (y_out == nullptr) still runs FFN2 and LN2: the LN2 backward reads s2 and its statistics.
static void layer_fwd_post(lga_handle* h, const Ws& w, const void* W, const float* x_in, float* y_out, cudaStream_t st,
                           int cc) {
  const Cfg& c = h->c;
  const int T = cc * c.M;
  const int d = c.d;
  const DT E = c.E;
  cast_f32(x_in, w.a, E, (int64_t)T * d, st);
  KCHECK();
  {  // qkv = x Wqkv + bqkv
    GemmArgs g;
    g.M = T; g.N = 3 * d; g.K = d;
    g.A = w.a; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wqkv); g.ldb = 3 * d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_bqkv); g.epi.bias_dt = E;
    g.epi.out = w.qkv; g.epi.ldo = 3 * d; g.epi.out_dt = E;
    gemm(h, g, st);
  }
  {  // o = attention(q, k, v)
    AttnArgs a;
    a.nseq = cc * c.b; a.seq = c.s; a.heads = c.H; a.dh = c.dh; a.d = d; a.causal = c.causal;
    a.scale = 1.0f / sqrtf((float)c.dh);
    a.qkv = w.qkv; a.o = w.o; a.lse = w.lse;
    const int p = prof_begin(h, st);
    if (c.bf16) CK(attn_fwd_bf16(a, st)); else attn_fwd_f32(a, st);
    KCHECK();
    prof_end(h, p, st, FAM_ATTN, attn_flops_fwd(c, a.nseq));
  }
  {  // s1 = x + o Wo + bo
    GemmArgs g;
    g.M = T; g.N = d; g.K = d;
    g.A = w.o; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wo); g.ldb = d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_bo); g.epi.bias_dt = E;
    g.epi.res = x_in; g.epi.ldr = d;
    g.epi.out = w.h1; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
  // h1 = LN1(s1): the E copy feeds FFN1; bf16 mode also keeps an fp32 copy for the FFN2 residual (the same
  // kernel on the same input: identical statistics)
  ln_fwd(w.h1, eoff((void*)W, E, c.o_ln1w), eoff((void*)W, E, c.o_ln1b), E, w.cn, E, w.st1, T, d, c.ln_eps, st);
  KCHECK();
  const float* hn = static_cast<const float*>(w.cn);
  if (c.bf16) {
    ln_fwd(w.h1, eoff((void*)W, E, c.o_ln1w), eoff((void*)W, E, c.o_ln1b), E, w.hn, DT::F32, w.st1, T, d, c.ln_eps, st);
    KCHECK();
    hn = w.hn;
  }
  {  // u = h1 W1 + b1 ; g = GELU(u)
    GemmArgs g;
    g.M = T; g.N = c.f; g.K = d;
    g.A = w.cn; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w1); g.ldb = c.f; g.b_kmajor = false;
    g.epi.kind = EPI_GELU_FWD; g.epi.bias = eoff((void*)W, E, c.o_b1); g.epi.bias_dt = E;
    g.epi.aux = (y_out && !c.norecomp) ? nullptr : w.u; g.epi.ldaux = c.f; g.epi.aux_dt = E;
    g.epi.out = w.g; g.epi.ldo = c.f; g.epi.out_dt = E;
    gemm(h, g, st);
  }
  {  // s2 = h1 + g W2 + b2
    GemmArgs g;
    g.M = T; g.N = d; g.K = c.f;
    g.A = w.g; g.lda = c.f; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w2); g.ldb = d; g.b_kmajor = false;
    g.epi.kind = EPI_STORE; g.epi.bias = eoff((void*)W, E, c.o_b2); g.epi.bias_dt = E;
    g.epi.res = hn; g.epi.ldr = d;
    g.epi.out = w.s2; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
  // y = LN2(s2) (recompute: statistics only, y into the backward's dC scratch)
  ln_fwd(w.s2, eoff((void*)W, E, c.o_ln2w), eoff((void*)W, E, c.o_ln2b), E, y_out ? y_out : h->dC, DT::F32, w.st2, T,
         d, c.ln_eps, st);
  KCHECK();
}

// wgrad: dW[i][j] (+)= sum_t X[t][i] dYm[t][j]  -> region at `off` with leading dim n
static void wgrad(lga_handle* h, const void* X, int64_t ldx, const void* Dy, int64_t ldy, int m, int n, int T,
                  const GradDst& dst, int64_t /*off*/, cudaStream_t st) {
  GemmArgs g;
  g.M = m; g.N = n; g.K = T;
  g.A = X; g.lda = ldx; g.a_kmajor = false;
  g.B = Dy; g.ldb = ldy; g.b_kmajor = false;
  g.epi.kind = EPI_STORE;
  g.epi.acc_in = dst.acc_in; g.epi.ldacc = n;
  g.epi.out = dst.out; g.epi.ldo = n; g.epi.out_dt = dst.out_dt;
  gemm(h, g, st);
}

// bias gradient from the column partials a producing kernel wrote into h->partial (nrows x n, fp32)
static void bias_from_partials(lga_handle* h, int64_t nrows, int n, const GradDst& dst, cudaStream_t st) {
  colsum_finish(h->partial, (int)nrows, n, n, dst.acc_in, dst.out, dst.out_dt, st);
  KCHECK();
}

static void bias_grad(lga_handle* h, const void* X, DT xdt, int64_t ldx, int n, int T, const GradDst& dst, cudaStream_t st) {
  const int nblk = colsum_partial(X, xdt, ldx, T, n, h->partial, st);
  KCHECK();
  colsum_finish(h->partial, nblk, n, n, dst.acc_in, dst.out, dst.out_dt, st);
  KCHECK();
}

// Attention backward -> dqkv (h->dO holds dO), and db_qkv = column sums of dqkv: on the tensor-core path the
// attention kernels emit per-quadrant partials next to their dqkv stores (no separate pass over dqkv)
static void attn_bwd_and_bias(lga_handle* h, const Ws& w, int T, const GradDst& bq, cudaStream_t st) {
  const Cfg& c = h->c;
  AttnArgs a;
  a.nseq = c.c * c.b; a.seq = c.s; a.heads = c.H; a.dh = c.dh; a.d = c.d; a.causal = c.causal;
  a.scale = 1.0f / sqrtf((float)c.dh);
  a.qkv = w.qkv; a.o = w.o; a.lse = w.lse; a.dO = h->dO; a.dsum = h->dsum; a.dqkv = h->dqkv;
  a.colsum = c.bf16 ? h->partial : nullptr;
  a.dsT = h->attn_ds;
  const int p = prof_begin(h, st);
  if (c.bf16) CK(attn_bwd_bf16(a, st)); else attn_bwd_f32(a, st);
  KCHECK();
  prof_end(h, p, st, FAM_ATTN, 2.0 * attn_flops_fwd(c, a.nseq));
  if (c.bf16) bias_from_partials(h, (int64_t)a.nseq * ((c.s + 127) / 128) * 4, 3 * c.d, bq, st);
  else bias_grad(h, h->dqkv, c.E, 3 * c.d, 3 * c.d, T, bq, st);
}

// Backward of local layer j over one chunk; the layer's intermediates are in the workspace
// (recomputed just before).  dY: fp32 [c][M][d] gradient of the layer output, read;
// dx_out: where dX goes (in place over dY, the previous stage's buffer, or a scratch sink).
// bf16: the GEMMs read dY as bf16 from h->dYe -- cast here unless dYe_ready (the previous layer's LN1
// backward already wrote it next to its fp32 dX); dx_e_out: also write dX as bf16 there (or nullptr).
static void layer_bwd_post(lga_handle* h, const Ws& w, const void* W, const float* dY, float* dx_out, int chunk_idx,
                           int nchunks, int jl, cudaStream_t st);
static void layer_bwd(lga_handle* h, const Ws& w, const void* W, const float* x_in, const float* dY, float* dx_out,
                      int chunk_idx, int nchunks, int jl, cudaStream_t st, bool dYe_ready = false,
                      void* dx_e_out = nullptr) {
  const Cfg& c = h->c;
  if (c.post_ln) return layer_bwd_post(h, w, W, dY, dx_out, chunk_idx, nchunks, jl, st);
  const int T = c.c * c.M;
  const int d = c.d, f = c.f;
  const DT E = c.E;
  const void* dYe = dY;
  if (c.bf16) {
    if (!dYe_ready) {
      cast_f32(dY, h->dYe, E, (int64_t)T * d, st);
      KCHECK();
    }
    dYe = h->dYe;
  }
  auto dst = [&](int64_t off) { return grad_dst(h, chunk_idx, nchunks, jl, off); };
  // ---- FFN2: y = h1 + g W2 + b2 (db2 = sum dY comes out of the LN2 backward below, which reads dY)
  wgrad(h, w.g, f, dYe, d, f, d, T, dst(c.o_w2), c.o_w2, st);
  {  // dU = (dY W2^T) * GELU'(u), written over u; bf16: the epilogue also emits db1 = sum dU per 32-row strip
    GemmArgs g;
    g.M = T; g.N = f; g.K = d;
    g.A = dYe; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w2); g.ldb = d; g.b_kmajor = true;
    g.epi.kind = EPI_GELU_BWD; g.epi.aux = w.u; g.epi.ldaux = f; g.epi.aux_dt = E;
    g.epi.out = w.u; g.epi.ldo = f; g.epi.out_dt = E;
    g.epi.colsum = c.bf16 ? h->partial : nullptr;
    gemm(h, g, st);
  }
  void* dU = w.u;
  if (c.bf16) bias_from_partials(h, (T + 31) / 32, f, dst(c.o_b1), st);
  else bias_grad(h, dU, E, f, f, T, dst(c.o_b1), st);
  // ---- FFN1: u = c W1 + b1
  wgrad(h, w.cn, d, dU, f, d, f, T, dst(c.o_w1), c.o_w1, st);
  {  // dC = dU W1^T
    GemmArgs g;
    g.M = T; g.N = d; g.K = f;
    g.A = dU; g.lda = f; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w1); g.ldb = f; g.b_kmajor = true;
    g.epi.out = h->dC; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
  // ---- LN2 backward + residual: dh1 = dY + LN2'(dC); its column partials also give db2 = sum dY (its
  // residual input) and db_o = sum dh1 (its output): no separate pass over dY / dh1
  {
    const int nblk = ln_bwd(h->dC, w.h1, w.st2, eoff((void*)W, E, c.o_ln2w), E, dY, h->dh1, c.bf16 ? h->dh1e : nullptr, E,
                            h->partial, T, d, st, /*extra=*/true);
    KCHECK();
    const int64_t o4[4] = {c.o_ln2w, c.o_ln2b, c.o_b2, c.o_bo};
    FinishSet fs;
    for (int k = 0; k < 4; ++k) {
      GradDst gd = dst(o4[k]);
      fs.o[fs.k++] = FinishOut{gd.acc_in, gd.out, gd.out_dt, (int64_t)k * d};
    }
    colsum_finish_multi(h->partial, nblk, 4LL * d, d, fs, st);
    KCHECK();
  }
  const void* dh1e = c.bf16 ? (const void*)h->dh1e : (const void*)h->dh1;
  // ---- O projection: h1 = x + o Wo + bo
  wgrad(h, w.o, d, dh1e, d, d, d, T, dst(c.o_wo), c.o_wo, st);
  {  // dO = dh1 Wo^T
    GemmArgs g;
    g.M = T; g.N = d; g.K = d;
    g.A = dh1e; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wo); g.ldb = d; g.b_kmajor = true;
    g.epi.out = h->dO; g.epi.ldo = d; g.epi.out_dt = E;
    gemm(h, g, st);
  }
  attn_bwd_and_bias(h, w, T, dst(c.o_bqkv), st);
  // ---- QKV: qkv = a Wqkv + bqkv
  wgrad(h, w.a, d, h->dqkv, 3 * d, d, 3 * d, T, dst(c.o_wqkv), c.o_wqkv, st);
  {  // dA = dqkv Wqkv^T  (into dC, free now)
    GemmArgs g;
    g.M = T; g.N = d; g.K = 3 * d;
    g.A = h->dqkv; g.lda = 3 * d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wqkv); g.ldb = 3 * d; g.b_kmajor = true;
    g.epi.out = h->dC; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
  // ---- LN1 backward + residual: dX = dh1 + LN1'(dA)
  {
    const int nblk = ln_bwd(h->dC, x_in, w.st1, eoff((void*)W, E, c.o_ln1w), E, h->dh1, dx_out, dx_e_out, E, h->partial,
                            T, d, st);
    KCHECK();
    GradDst gw = dst(c.o_ln1w), gbias = dst(c.o_ln1b);
    FinishSet fs;
    fs.o[fs.k++] = FinishOut{gw.acc_in, gw.out, gw.out_dt, 0};
    fs.o[fs.k++] = FinishOut{gbias.acc_in, gbias.out, gbias.out_dt, (int64_t)d};
    colsum_finish_multi(h->partial, nblk, 2LL * d, d, fs, st);
    KCHECK();
  }
}

// Post-LN backward (reading A-16; oracle.model.layer_backward_post): ds2 = LN2'(dY); FFN2 / FFN1 grads;
// dh1 = dU W1^T + ds2 (GEMM epilogue residual); ds1 = LN1'(dh1); O-projection and attention grads;
// dX = dqkv Wqkv^T + ds1.  dY is read only by the first kernel, so dx_out may alias it.
static void layer_bwd_post(lga_handle* h, const Ws& w, const void* W, const float* dY, float* dx_out, int chunk_idx,
                           int nchunks, int jl, cudaStream_t st) {
  const Cfg& c = h->c;
  const int T = c.c * c.M;
  const int d = c.d, f = c.f;
  const DT E = c.E;
  auto dst = [&](int64_t off) { return grad_dst(h, chunk_idx, nchunks, jl, off); };
  auto ln_back = [&](const float* dout, const float* xin, const float2* stats, int64_t ow, int64_t ob, int64_t osum) {
    // -> h->dh1 (fp32) and, bf16 mode, h->dh1e; gamma / beta gradients from the column partials, and the bias
    // whose gradient is the column sum of this output (osum: db2 = sum ds2, db_o = sum ds1)
    const int nblk = ln_bwd(dout, xin, stats, eoff((void*)W, E, ow), E, nullptr, h->dh1, c.bf16 ? h->dh1e : nullptr, E,
                            h->partial, T, d, st, /*extra=*/true);
    KCHECK();
    const int64_t o4[4] = {ow, ob, -1, osum};
    FinishSet fs;
    for (int k = 0; k < 4; ++k) {
      if (o4[k] < 0) continue;
      GradDst gd = dst(o4[k]);
      fs.o[fs.k++] = FinishOut{gd.acc_in, gd.out, gd.out_dt, (int64_t)k * d};
    }
    colsum_finish_multi(h->partial, nblk, 4LL * d, d, fs, st);
    KCHECK();
  };
  const void* dse = c.bf16 ? (const void*)h->dh1e : (const void*)h->dh1;   // ds2, then ds1, as GEMM operand
  // ---- LN2: y = LN2(s2)
  ln_back(dY, w.s2, w.st2, c.o_ln2w, c.o_ln2b, c.o_b2);
  // ---- FFN2: s2 = h1 + g W2 + b2
  wgrad(h, w.g, f, dse, d, f, d, T, dst(c.o_w2), c.o_w2, st);
  {  // dU = (ds2 W2^T) * GELU'(u), written over u (bf16: + the db1 strip partials)
    GemmArgs g;
    g.M = T; g.N = f; g.K = d;
    g.A = dse; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w2); g.ldb = d; g.b_kmajor = true;
    g.epi.kind = EPI_GELU_BWD; g.epi.aux = w.u; g.epi.ldaux = f; g.epi.aux_dt = E;
    g.epi.out = w.u; g.epi.ldo = f; g.epi.out_dt = E;
    g.epi.colsum = c.bf16 ? h->partial : nullptr;
    gemm(h, g, st);
  }
  void* dU = w.u;
  if (c.bf16) bias_from_partials(h, (T + 31) / 32, f, dst(c.o_b1), st);
  else bias_grad(h, dU, E, f, f, T, dst(c.o_b1), st);
  // ---- FFN1: u = h1 W1 + b1
  wgrad(h, w.cn, d, dU, f, d, f, T, dst(c.o_w1), c.o_w1, st);
  {  // dh1 = dU W1^T + ds2
    GemmArgs g;
    g.M = T; g.N = d; g.K = f;
    g.A = dU; g.lda = f; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_w1); g.ldb = f; g.b_kmajor = true;
    g.epi.res = h->dh1; g.epi.ldr = d;
    g.epi.out = h->dC; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
  // ---- LN1: h1 = LN1(s1)
  ln_back(h->dC, w.h1, w.st1, c.o_ln1w, c.o_ln1b, c.o_bo);
  // ---- O projection: s1 = x + o Wo + bo
  wgrad(h, w.o, d, dse, d, d, d, T, dst(c.o_wo), c.o_wo, st);
  {  // dO = ds1 Wo^T
    GemmArgs g;
    g.M = T; g.N = d; g.K = d;
    g.A = dse; g.lda = d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wo); g.ldb = d; g.b_kmajor = true;
    g.epi.out = h->dO; g.epi.ldo = d; g.epi.out_dt = E;
    gemm(h, g, st);
  }
  attn_bwd_and_bias(h, w, T, dst(c.o_bqkv), st);
  // ---- QKV: qkv = x Wqkv + bqkv
  wgrad(h, w.a, d, h->dqkv, 3 * d, d, 3 * d, T, dst(c.o_wqkv), c.o_wqkv, st);
  {  // dX = dqkv Wqkv^T + ds1
    GemmArgs g;
    g.M = T; g.N = d; g.K = 3 * d;
    g.A = h->dqkv; g.lda = 3 * d; g.a_kmajor = true;
    g.B = eoff((void*)W, E, c.o_wqkv); g.ldb = 3 * d; g.b_kmajor = true;
    g.epi.res = h->dh1; g.epi.ldr = d;
    g.epi.out = dx_out; g.epi.ldo = d; g.epi.out_dt = DT::F32;
    gemm(h, g, st);
  }
}

// ------------------------------------------------------------------ scheduler helpers
static void count_wait(lga_handle* h, cudaEvent_t ev, int kind) {
  // stall accounting: event pair around the compute stream's wait on a comm event (BJ metric)
  if (h->n_wait >= (int)h->ev_wait0.size()) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    h->ev_wait0.push_back(a);
    h->ev_wait1.push_back(b);
    h->wait_kind.push_back(kind);
  }
  h->wait_kind[h->n_wait] = kind;
  rec_time(h, h->ev_wait0[h->n_wait], h->s_comp);
  if (ev) CK(cudaStreamWaitEvent(h->s_comp, ev, 0));
  return;
}
static void count_wait_end(lga_handle* h) {
  rec_time(h, h->ev_wait1[h->n_wait], h->s_comp);
  h->n_wait++;
}

static const void* layer_weights(lga_handle* h, int j, int slot) {
  if (!h->slot.empty()) return h->slot[slot];
  return eoff(h->pshard, h->c.E, (int64_t)j * h->c.S);   // D == 1 or unpartitioned: the local full layer
}


static void all_gather(lga_handle* h, int j, int slot) {
  const Cfg& c = h->c;
  if (h->slot.empty()) return;
  h->last.ag_calls++;
  h->last.ag_bytes += (uint64_t)(c.D - 1) * c.S * dt_size(c.E);
  if (h->comm_off) return;
  if (c.dp_ipc) {
    // every replica's AdamW of layer j of the previous step is done (D (t-1) signals), then pull the D
    // shards over NVLink on the copy engines and tell each owner that its shard j has been read
    wait_flag(h->dpf + DPF_PARAM * c.Lloc + j, h->tepoch, (unsigned long long)c.D, 0ull, h->s_comm);
    KCHECK();
    const size_t bytes = (size_t)c.S * dt_size(c.E);
    for (int p = 0; p < c.D; ++p)
      CK(cudaMemcpyAsync(eoff(h->slot[slot], c.E, (int64_t)p * c.S), eoff(h->dp_psh[p], c.E, (int64_t)j * c.S), bytes,
                         cudaMemcpyDeviceToDevice, h->s_comm));
    dp_signal(h->dp_flag_dev, c.D, DPF_READ * c.Lloc + j, h->s_comm);
    KCHECK();
    return;
  }
  NK(ncclAllGather(eoff(h->pshard, c.E, (int64_t)j * c.S), h->slot[slot], (size_t)c.S, nccl_dt(c.E), h->dp_comm, h->s_comm));
}

// AdamW on this rank's shard of local layer j (update "as soon as possible", A-12)
static void adam_layer(lga_handle* h, int j, const void* g, DT gdt) {
  const Cfg& c = h->c;
  const float gscale = 1.0f / ((float)c.D * (float)c.N);   // gradient of the mean loss (A-3)
  const int64_t off = (int64_t)j * c.S;
  const int p = prof_begin(h, h->s_comm);
  adamw(g, gdt, gscale, h->master + off, h->mom + off, h->var + off, eoff(h->pshard, c.E, off), c.E,
        c.retain ? h->gkeep + off : nullptr, c.S, c.lr, c.b1, c.b2, c.eps, c.wd, h->tstep, h->s_comm);
  KCHECK();
  const double per = (double)dt_size(gdt) + 24.0 + (double)dt_size(c.E) + (c.retain ? 4.0 : 0.0);
  prof_end(h, p, h->s_comm, FAM_ADAM, per * (double)c.S);
}

// reduce-scatter of the staged gradient in place (once per layer per step); returns the shard.
// Unpartitioned (N2b): all-reduce of the whole layer in place instead (scatter-reduce + all-gather,
// P:565), every replica then updates the full layer.
static void* reduce_scatter(lga_handle* h, int j) {
  const Cfg& c = h->c;
  void* gs = stage_buf(h, j);
  if (c.unpart) {
    if (c.D > 1) {
      h->last.allreduce_calls++;
      h->last.allreduce_bytes += 2ull * (c.D - 1) * (uint64_t)(c.plpad / c.D) * dt_size(c.G);
      if (!h->comm_off) NK(ncclAllReduce(gs, gs, (size_t)c.plpad, nccl_dt(c.G), ncclSum, h->dp_comm, h->s_comm));
    }
    return gs;
  }
  void* shard_g = eoff(gs, c.G, (int64_t)h->replica * c.S);
  if (c.D > 1) {
    h->last.rs_calls++;
    h->last.rs_bytes += (uint64_t)(c.D - 1) * c.S * dt_size(c.G);
    if (!h->comm_off)
      NK(ncclReduceScatter(gs, shard_g, (size_t)c.S, nccl_dt(c.G), ncclSum, h->dp_comm, h->s_comm));
  }
  return shard_g;
}

// N1: reduce-scatter fused with AdamW over peer memory.  Announce this rank's staged gradient of layer j to
// every replica, wait until all D are staged (D t signals) and every replica has read this rank's shard j
// in this step (R D t; R = all-gathers of a layer per step), then sum the D slices in fixed rank order
// inside the AdamW kernel, and announce the updated shard.
static void rs_adam_peer(lga_handle* h, int j) {
  const Cfg& c = h->c;
  h->last.rs_calls++;
  h->last.rs_bytes += (uint64_t)(c.D - 1) * c.S * dt_size(c.G);
  const unsigned long long D = (unsigned long long)c.D, R = c.keep ? 1ull : 2ull;
  if (!h->comm_off) {
    dp_signal(h->dp_flag_dev, c.D, DPF_GRAD * c.Lloc + j, h->s_comm);
    KCHECK();
    wait_flag(h->dpf + DPF_GRAD * c.Lloc + j, h->tepoch, D, D, h->s_comm);
    KCHECK();
    wait_flag(h->dpf + DPF_READ * c.Lloc + j, h->tepoch, R * D, R * D, h->s_comm);
    KCHECK();
  }
  const float gscale = 1.0f / ((float)c.D * (float)c.N);   // gradient of the mean loss (A-3)
  const int64_t off = (int64_t)j * c.S;
  const int64_t goff = (int64_t)j * c.plpad + (int64_t)h->replica * c.S;
  const int p = prof_begin(h, h->s_comm);
  if (h->comm_off)
    adamw(eoff(stage_buf(h, j), c.G, (int64_t)h->replica * c.S), c.G, gscale, h->master + off, h->mom + off,
          h->var + off, eoff(h->pshard, c.E, off), c.E, c.retain ? h->gkeep + off : nullptr, c.S, c.lr, c.b1, c.b2,
          c.eps, c.wd, h->tstep, h->s_comm);
  else
    adamw_rs(h->dp_gst_dev, goff, c.D, c.G, gscale, h->master + off, h->mom + off, h->var + off,
             eoff(h->pshard, c.E, off), c.E, c.retain ? h->gkeep + off : nullptr, c.S, c.lr, c.b1, c.b2, c.eps, c.wd,
             h->tstep, h->s_comm);
  KCHECK();
  const double per = (double)c.D * dt_size(c.G) + 24.0 + (double)dt_size(c.E) + (c.retain ? 4.0 : 0.0);
  prof_end(h, p, h->s_comm, FAM_ADAM, per * (double)c.S);
  if (!h->comm_off) {
    dp_signal(h->dp_flag_dev, c.D, DPF_PARAM * c.Lloc + j, h->s_comm);
    KCHECK();
  }
}

// N2b over peer memory: the all-reduce of layer j's gradient as a reduce-scatter then an all-gather (the
// bandwidth-optimal 2 (D-1)/D of the layer per rank), then AdamW on the whole layer (every replica holds
// the full state).  (1) announce the staged gradient, wait for all D; (2) sum slice r of the D staging buffers in
// fixed rank order into this rank's own slice r (no peer reads slice r of this rank in this phase); (3) announce
// the reduced slice, wait for all D; (4) copy the D-1 other reduced slices from their owners (copy engines) and
// announce the reads, which the next step's backward of layer j waits for before it rewrites the staging.
static void allreduce_adam_peer(lga_handle* h, int j) {
  const Cfg& c = h->c;
  const int64_t Sr = c.plpad / c.D;   // slice of the reduce-scatter phase
  const size_t eg = dt_size(c.G);
  h->last.allreduce_calls++;
  h->last.allreduce_bytes += 2ull * (c.D - 1) * (uint64_t)Sr * eg;
  void* gs = stage_buf(h, j);
  if (!h->comm_off) {
    const unsigned long long D = (unsigned long long)c.D;
    dp_signal(h->dp_flag_dev, c.D, DPF_GRAD * c.Lloc + j, h->s_comm);
    KCHECK();
    wait_flag(h->dpf + DPF_GRAD * c.Lloc + j, h->tepoch, D, D, h->s_comm);
    KCHECK();
    const int64_t goff = (int64_t)j * c.plpad + (int64_t)h->replica * Sr;
    peer_reduce(h->dp_gst_dev, goff, c.D, c.G, nullptr, false, eoff(gs, c.G, (int64_t)h->replica * Sr), Sr, h->s_comm);
    KCHECK();
    dp_signal(h->dp_flag_dev, c.D, DPF_RED * c.Lloc + j, h->s_comm);
    KCHECK();
    wait_flag(h->dpf + DPF_RED * c.Lloc + j, h->tepoch, D, D, h->s_comm);
    KCHECK();
    for (int p = 0; p < c.D; ++p) {
      if (p == h->replica) continue;
      const int64_t o = (int64_t)p * Sr;
      const char* src = h->dp_base[p] + h->peers[p * c.P + h->stage].off_gst + ((int64_t)j * c.plpad + o) * eg;
      CK(cudaMemcpyAsync(eoff(gs, c.G, o), src, (size_t)Sr * eg, cudaMemcpyDeviceToDevice, h->s_comm));
    }
    dp_signal(h->dp_flag_dev, c.D, DPF_READ * c.Lloc + j, h->s_comm);
    KCHECK();
  }
  adam_layer(h, j, gs, c.G);
}

// STANDARD over peer memory: micro-batch m's gradient of layer j is reduce-scattered into this
// rank's fp32 shard accumulator (fixed rank order, (re)started at m = 0); the peers then announce that they read
// their slice of this rank's staging j (the next micro-batch's backward waits for that before rewriting it).
// After the last micro-batch: wait until every replica has done all of this step's 2 N gathers of shard j, then
// AdamW and announce the updated shard.
static void rs_acc_peer(lga_handle* h, int j, int m) {
  const Cfg& c = h->c;
  h->last.rs_calls++;
  h->last.rs_bytes += (uint64_t)(c.D - 1) * c.S * dt_size(c.G);
  const unsigned long long D = (unsigned long long)c.D, N = (unsigned long long)c.N;
  float* acc = h->gshard_acc + (int64_t)j * c.S;
  if (!h->comm_off) {
    dp_signal(h->dp_flag_dev, c.D, DPF_GRAD * c.Lloc + j, h->s_comm);
    KCHECK();
    wait_flag(h->dpf + DPF_GRAD * c.Lloc + j, h->tepoch, D * N, D * (unsigned long long)(m + 1), h->s_comm);
    KCHECK();
    peer_reduce(h->dp_gst_dev, (int64_t)j * c.plpad + (int64_t)h->replica * c.S, c.D, c.G, acc, m == 0, nullptr, c.S,
                h->s_comm);
    KCHECK();
    dp_signal(h->dp_flag_dev, c.D, DPF_GREAD * c.Lloc + j, h->s_comm);
    KCHECK();
  } else {
    shard_accumulate(eoff(stage_buf(h, j), c.G, (int64_t)h->replica * c.S), c.G, acc, c.S, m == 0, h->s_comm);
    KCHECK();
  }
  if (m == c.N - 1) {
    if (!h->comm_off) {
      wait_flag(h->dpf + DPF_READ * c.Lloc + j, h->tepoch, 2 * N * D, 2 * N * D, h->s_comm);
      KCHECK();
    }
    adam_layer(h, j, acc, DT::F32);
    if (!h->comm_off) {
      dp_signal(h->dp_flag_dev, c.D, DPF_PARAM * c.Lloc + j, h->s_comm);
      KCHECK();
    }
  }
}

static float* ckpt_ptr(lga_handle* h, int j, int m) {
  const Cfg& c = h->c;
  return h->ckpt + ((int64_t)j * c.N + m) * (int64_t)c.M * c.d;
}
static float* act_ptr(float* base, const Cfg& c, int m) { return base + (int64_t)m * c.M * c.d; }

// forward intermediates of local layer j, micro-batches [m0, m0 + c): the shared chunk set, or (no
// recompute) layer j's own set at token m0*M
static Ws chunk_ws(lga_handle* h, int j, int m0) {
  const Cfg& c = h->c;
  if (!c.norecomp) return h->ws[0];
  const Ws& b = h->ws[j];
  const int64_t t = (int64_t)m0 * c.M, d = c.d, f = c.f;
  const size_t e = dt_size(c.E);
  Ws w;
  w.a = static_cast<char*>(b.a) + t * d * e;
  w.qkv = static_cast<char*>(b.qkv) + t * 3 * d * e;
  w.o = static_cast<char*>(b.o) + t * d * e;
  w.cn = static_cast<char*>(b.cn) + t * d * e;
  w.u = static_cast<char*>(b.u) + t * f * e;
  w.g = static_cast<char*>(b.g) + t * f * e;
  w.h1 = b.h1 + t * d;
  w.lse = b.lse + (int64_t)m0 * c.b * c.H * c.s;
  w.st1 = b.st1 + t;
  w.st2 = b.st2 + t;
  w.hn = b.hn ? b.hn + t * d : nullptr;
  w.s2 = b.s2 ? b.s2 + t * d : nullptr;
  return w;
}

// lga_step_host copies the target on its own stream, overlapped with the forward; the first loss waits
static void await_target(lga_handle* h) {
  if (!h->tin_pending) return;
  CK(cudaStreamWaitEvent(h->s_comp, h->ev_tin, 0));
  h->tin_pending = false;
}

// ------------------------------------------------------------------ the step (LAYERED, any D, any P)
// Parameter slots: with mixed buffering (2 slots) the gather of layer j goes to slot agk % 2, agk counting
// gathers over the step; with LGA_FLAG_KEEP_PARAMS layer j has slot j, filled once in the forward.
static void step_layered(lga_handle* h, const float* x, const float* T) {
  const Cfg& c = h->c;
  const int nchunks = c.N / c.c;
  const int64_t mb = (int64_t)c.M * c.d;
  const bool dp_gather = !h->slot.empty();
  auto slot_of = [&](int j, int agk) { return c.keep ? j : agk % 2; };
  int agk = 0;  // running all-gather index
  // ---------------- forward: layer-major over all micro-batches
  if (dp_gather) {
    if (h->rec_slot[slot_of(0, 0)]) CK(cudaStreamWaitEvent(h->s_comm, h->ev_slot_free[slot_of(0, 0)], 0));
    all_gather(h, 0, slot_of(0, 0));
    CK(cudaEventRecord(h->ev_ag[slot_of(0, 0)], h->s_comm));
  }
  for (int j = 0; j < c.Lloc; ++j, ++agk) {
    const int sl = slot_of(j, agk);
    const int64_t i = local_to_global(h, j);
    NvtxRange nvtx_layer("fwd layer", i);
    if (dp_gather && j + 1 < c.Lloc) {  // prefetch Restore(next local layer) while computing layer i
      const int sn = slot_of(j + 1, agk + 1);
      if (h->rec_slot[sn]) CK(cudaStreamWaitEvent(h->s_comm, h->ev_slot_free[sn], 0));
      all_gather(h, j + 1, sn);
      CK(cudaEventRecord(h->ev_ag[sn], h->s_comm));
    }
    if (dp_gather) {
      count_wait(h, h->ev_ag[sl], 0);
      count_wait_end(h);
    }
    const void* W = layer_weights(h, j, sl);
    const bool recv = c.P > 1 && i > 0 && stage_of(c, i - 1) != h->stage;        // x_i from another stage
    const bool send = c.P > 1 && i < c.L - 1 && stage_of(c, i + 1) != h->stage;  // x_{i+1} to another stage
    const bool split0 = i == 0 && h->x_split;        // one micro-batch per launch, each after its copy
    const int cw = split0 ? 1 : c.c, nch = split0 ? c.N : nchunks;
    for (int k = 0; k < nch; ++k) {
      const int m0 = k * cw;
      const float* xin;
      if (i == 0) {
        xin = x + m0 * mb;   // layer 0 input is the caller's x (no copy)
        if (split0) CK(cudaStreamWaitEvent(h->s_comp, h->ev_x[k], 0));
      } else {
        xin = ckpt_ptr(h, j, m0);
        if (recv) {  // pipeline receive: x_i[m0..m0+c) written by the previous stage
          h->recv_fwd += cw;
          h->last.p2p_recv_calls += cw;
          h->last.p2p_recv_bytes += (uint64_t)cw * mb * 4;
          if (!h->comm_off) {
            count_wait(h, nullptr, 1);
            wait_flag(h->flags + 0, h->tepoch, h->k_recv_fwd, h->recv_fwd, h->s_comp);
            KCHECK();
            count_wait_end(h);
          }
        }
      }
      float* yo;
      if (i == c.L - 1) {
        yo = act_ptr(h->yout, c, m0);
      } else if (!send) {
        yo = ckpt_ptr(h, j + 1, m0);
      } else {  // write x_{i+1} straight into the next stage's checkpoint buffer (fused p2p)
        const int jn = local_index(c, i + 1);
        yo = h->comm_off ? h->dscratch : h->next_ckpt + ((int64_t)jn * c.N + m0) * mb;
      }
      layer_fwd(h, chunk_ws(h, j, m0), W, xin, yo, h->s_comp, cw);
      h->last.fwd_units += cw;
      if (send) {
        h->sent_fwd += cw;
        h->last.p2p_send_calls += cw;
        h->last.p2p_send_bytes += (uint64_t)cw * mb * 4;
        if (!h->comm_off) {
          set_flag(h->next_flags + 0, h->tepoch, h->k_send_fwd, h->sent_fwd, h->s_comp);
          KCHECK();
        }
      }
      if (i == c.L - 1) {  // loss of this chunk + seed gradient
        const int64_t n = (int64_t)cw * mb;
        await_target(h);
        mse_fwd_bwd(act_ptr(h->yout, c, m0), T + m0 * mb, act_ptr(h->dY, c, m0), h->mse_partial + 0, n,
                    1.0f / (float)mb, h->s_comp);
        KCHECK();
        // this chunk's sum of micro-batch losses -> loss_dev[1 + k] (summed in fixed order at the end)
        mse_finish(h->mse_partial, mse_blocks(n), 0.5 / (double)mb, h->loss_dev + 1 + k, h->s_comp);
        KCHECK();
      }
    }
    if (!c.keep) { CK(cudaEventRecord(h->ev_slot_free[sl], h->s_comp)); h->rec_slot[sl] = 1; }
    trace(h, "fwd", i);
  }
  rec_time(h, h->ev_fwd_end, h->s_comp);
  // ---------------- backward: layer-major, (recompute +) backward over all micro-batches
  if (dp_gather && !c.keep) {
    if (h->rec_slot[agk % 2]) CK(cudaStreamWaitEvent(h->s_comm, h->ev_slot_free[agk % 2], 0));
    all_gather(h, c.Lloc - 1, agk % 2);
    CK(cudaEventRecord(h->ev_ag[agk % 2], h->s_comm));
  }
  for (int j = c.Lloc - 1; j >= 0; --j, ++agk) {
    NvtxRange nvtx_layer("bwd layer", local_to_global(h, j));
    const int sl = slot_of(j, agk);
    const int64_t i = local_to_global(h, j);
    const int gb = j % 2;
    if (dp_gather && !c.keep && j - 1 >= 0) {
      if (h->rec_slot[(agk + 1) % 2]) CK(cudaStreamWaitEvent(h->s_comm, h->ev_slot_free[(agk + 1) % 2], 0));
      all_gather(h, j - 1, (agk + 1) % 2);
      CK(cudaEventRecord(h->ev_ag[(agk + 1) % 2], h->s_comm));
    }
    if (dp_gather && !c.keep) {
      count_wait(h, h->ev_ag[sl], 0);
      count_wait_end(h);
    }
    if (!c.dp_ipc && h->rec_adam[gb]) {   // staging gb free again (NCCL path: RS + AdamW of layer j + 2 done)
      count_wait(h, h->ev_adam[gb], 0);
      count_wait_end(h);
    }
    if (c.dp_ipc && c.unpart && !h->comm_off) {   // every replica read last step's reduced slices of staging j
      count_wait(h, nullptr, 0);
      wait_flag(h->dpf + DPF_READ * c.Lloc + j, h->tepoch, (unsigned long long)c.D, 0ull, h->s_comp);
      KCHECK();
      count_wait_end(h);
    }
    const void* W = layer_weights(h, j, sl);
    const bool recv = c.P > 1 && i < c.L - 1 && stage_of(c, i + 1) != h->stage;   // dY_i from another stage
    const bool send = c.P > 1 && i > 0 && stage_of(c, i - 1) != h->stage;         // dX_i to another stage
    // one chunk, and the next layer processed here is i-1: its bf16 dY comes out of this LN1 backward
    const bool fuse_e = c.bf16 && nchunks == 1;
    const bool dye_ready = fuse_e && i < c.L - 1 && !recv;
    void* dx_e = (fuse_e && i > 0 && !send) ? h->dYe : nullptr;
    for (int k = 0; k < nchunks; ++k) {
      const int m0 = k * c.c;
      const float* xin = (i == 0) ? x + m0 * mb : ckpt_ptr(h, j, m0);
      float* dYc = act_ptr(h->dY, c, m0);
      if (recv) {  // receive dY_i[m0..) from the next stage
        h->recv_bwd += c.c;
        h->last.p2p_recv_calls += c.c;
        h->last.p2p_recv_bytes += (uint64_t)c.c * mb * 4;
        if (!h->comm_off) {
          count_wait(h, nullptr, 1);
          wait_flag(h->flags + 1, h->tepoch, h->k_recv_bwd, h->recv_bwd, h->s_comp);
          KCHECK();
          count_wait_end(h);
        }
      }
      const Ws w = chunk_ws(h, j, m0);
      if (!c.norecomp) {
        layer_fwd(h, w, W, xin, nullptr, h->s_comp);   // recompute
        h->last.recompute_units += c.c;
      }
      float* dx;
      if (i == 0) dx = h->dscratch;
      else if (!send) dx = dYc;
      else dx = h->comm_off ? h->dscratch : h->prev_dY + m0 * mb;
      layer_bwd(h, w, W, xin, dYc, dx, k, nchunks, j, h->s_comp, dye_ready, dx_e);
      h->last.bwd_units += c.c;
      if (send) {
        h->sent_bwd += c.c;
        h->last.p2p_send_calls += c.c;
        h->last.p2p_send_bytes += (uint64_t)c.c * mb * 4;
        if (!h->comm_off) {
          set_flag(h->prev_flags + 1, h->tepoch, h->k_send_bwd, h->sent_bwd, h->s_comp);
          KCHECK();
        }
      }
    }
    { CK(cudaEventRecord(h->ev_slot_free[sl], h->s_comp)); h->rec_slot[sl] = 1; }
    trace(h, "bwd", i);
    CK(cudaEventRecord(h->ev_grad[gb], h->s_comp));
    CK(cudaStreamWaitEvent(h->s_comm, h->ev_grad[gb], 0));
    if (c.dp_ipc) {
      if (c.unpart) allreduce_adam_peer(h, j);
      else rs_adam_peer(h, j);
    } else {
      void* shard_g = reduce_scatter(h, j);
      adam_layer(h, j, shard_g, c.G);
    }
    { CK(cudaEventRecord(h->ev_adam[gb], h->s_comm)); h->rec_adam[gb] = true; }
  }
}

// ------------------------------------------------------------------ STANDARD (comparison, P = 1)
// for each micro-batch: for l: AG(l); fwd(l, m); loss(m); for l desc: AG(l); recompute+bwd(l, m);
// RS(l) -> shard, accumulate on the shard; AdamW after the last micro-batch.
static void step_standard(lga_handle* h, const float* x, const float* T) {
  const Cfg& c = h->c;
  const int64_t mb = (int64_t)c.M * c.d;
  // the layer used by each successive compute pass: per micro-batch, layers ascending then descending.  The
  // all-gather of use u+1 is prefetched into the other slot while use u computes (as in LAYERED: the
  // comparison schedule gets the same overlap; only its N-fold volume differs)
  std::vector<int> uses;
  uses.reserve((size_t)2 * c.N * c.L);
  for (int m = 0; m < c.N; ++m) {
    for (int j = 0; j < c.L; ++j) uses.push_back(j);
    for (int j = c.L - 1; j >= 0; --j) uses.push_back(j);
  }
  auto gather = [&](int u) {
    if (c.D <= 1 || u >= (int)uses.size()) return;
    const int sl = u % 2;
    if (h->rec_slot[sl]) CK(cudaStreamWaitEvent(h->s_comm, h->ev_slot_free[sl], 0));
    all_gather(h, uses[u], sl);
    CK(cudaEventRecord(h->ev_ag[sl], h->s_comm));
  };
  gather(0);
  int agk = 0;
  for (int m = 0; m < c.N; ++m) {
    for (int j = 0; j < c.L; ++j, ++agk) {
      const int sl = agk % 2;
      gather(agk + 1);
      if (c.D > 1) {
        count_wait(h, h->ev_ag[sl], 0);
        count_wait_end(h);
      }
      const float* xin = j == 0 ? x + m * mb : ckpt_ptr(h, j, m);
      float* yo = j == c.L - 1 ? act_ptr(h->yout, c, m) : ckpt_ptr(h, j + 1, m);
      layer_fwd(h, h->ws[0], layer_weights(h, j, sl), xin, yo, h->s_comp);
      h->last.fwd_units++;
      { CK(cudaEventRecord(h->ev_slot_free[sl], h->s_comp)); h->rec_slot[sl] = 1; }
    }
    await_target(h);
    mse_fwd_bwd(act_ptr(h->yout, c, m), T + m * mb, act_ptr(h->dY, c, m), h->mse_partial, mb, 1.0f / (float)mb, h->s_comp);
    KCHECK();
    mse_finish(h->mse_partial, mse_blocks(mb), 0.5 / (double)mb, h->loss_dev + 1 + m, h->s_comp);
    KCHECK();
    for (int j = c.L - 1; j >= 0; --j, ++agk) {
      const int sl = agk % 2;
      const int gb = j % 2;
      gather(agk + 1);
      if (c.D > 1) {
        count_wait(h, h->ev_ag[sl], 0);
        count_wait_end(h);
      }
      if (!c.dp_ipc && h->rec_adam[gb]) {   // staging gb free again (NCCL path)
        count_wait(h, h->ev_adam[gb], 0);
        count_wait_end(h);
      }
      if (c.dp_ipc && !h->comm_off) {   // every replica read its slice of the previous micro-batch's staging j
        count_wait(h, nullptr, 0);
        wait_flag(h->dpf + DPF_GREAD * c.Lloc + j, h->tepoch, (unsigned long long)c.D * c.N, (unsigned long long)c.D * m,
                  h->s_comp);
        KCHECK();
        count_wait_end(h);
      }
      const void* W = layer_weights(h, j, sl);
      const float* xin = j == 0 ? x + m * mb : ckpt_ptr(h, j, m);
      float* dYc = act_ptr(h->dY, c, m);
      layer_fwd(h, h->ws[0], W, xin, nullptr, h->s_comp);
      h->last.recompute_units++;
      layer_bwd(h, h->ws[0], W, xin, dYc, j == 0 ? h->dscratch : dYc, 0, 1, j, h->s_comp);
      h->last.bwd_units++;
      { CK(cudaEventRecord(h->ev_slot_free[sl], h->s_comp)); h->rec_slot[sl] = 1; }
      CK(cudaEventRecord(h->ev_grad[gb], h->s_comp));
      CK(cudaStreamWaitEvent(h->s_comm, h->ev_grad[gb], 0));
      if (c.dp_ipc) {
        rs_acc_peer(h, j, m);
      } else {   // reduce-scatter this micro-batch's gradient, accumulate it on the shard (fixed order over m)
        void* shard_g = reduce_scatter(h, j);
        float* acc = h->gshard_acc + (int64_t)j * c.S;
        shard_accumulate(shard_g, c.G, acc, c.S, m == 0, h->s_comm);
        KCHECK();
        if (m == c.N - 1) adam_layer(h, j, acc, DT::F32);
      }
      { CK(cudaEventRecord(h->ev_adam[gb], h->s_comm)); h->rec_adam[gb] = true; }
    }
  }
}

}  // namespace lga

// ================================================================== C ABI
using namespace lga;

#define ABI_TRY try {
#define ABI_CATCH                                      \
  }                                                    \
  catch (const StatusError& e) {                       \
    if (h) h->bad = true;                              \
    return e.s;                                        \
  }                                                    \
  catch (...) {                                        \
    if (h) h->bad = true;                              \
    return ERR(LGA_ERR_CUDA, "unexpected exception");  \
  }

extern "C" {

uint32_t lga_abi_version(void) { return LGA_ABI_VERSION; }

const char* lga_status_string(lga_status s) {
  switch (s) {
    case LGA_OK: return "LGA_OK";
    case LGA_ERR_INVALID_ARG: return "LGA_ERR_INVALID_ARG";
    case LGA_ERR_UNSUPPORTED: return "LGA_ERR_UNSUPPORTED";
    case LGA_ERR_OUT_OF_MEMORY: return "LGA_ERR_OUT_OF_MEMORY";
    case LGA_ERR_CUDA: return "LGA_ERR_CUDA";
    case LGA_ERR_NCCL: return "LGA_ERR_NCCL";
    case LGA_ERR_SIZE_MISMATCH: return "LGA_ERR_SIZE_MISMATCH";
    case LGA_ERR_BAD_STATE: return "LGA_ERR_BAD_STATE";
  }
  return "LGA_ERR_UNKNOWN";
}

const char* lga_last_error(void) { return g_last_error.c_str(); }

lga_status lga_param_count(const lga_config* cfg, uint64_t* per_layer, uint64_t* total) {
  if (!cfg) return ERR(LGA_ERR_INVALID_ARG, "cfg is NULL");
  if (cfg->d_model <= 0 || cfg->layers <= 0) return ERR(LGA_ERR_INVALID_ARG, "non-positive dimension");
  const uint64_t d = (uint64_t)cfg->d_model, n = (uint64_t)(cfg->ffn_mult > 0 ? cfg->ffn_mult : 4);
  const uint64_t pl = (4 + 2 * n) * d * d + 13 * d;
  if (per_layer) *per_layer = pl;
  if (total) *total = pl * (uint64_t)cfg->layers;
  return LGA_OK;
}

lga_status lga_plan(const lga_config* cfg, int32_t rank, int32_t world, lga_rank_plan* out) {
  if (!out) return ERR(LGA_ERR_INVALID_ARG, "out is NULL");
  Cfg c;
  lga_status s = validate(cfg, world, &c);
  if (s != LGA_OK) return s;
  if (rank < 0 || rank >= world) return ERR(LGA_ERR_INVALID_ARG, "rank %d out of [0, %d)", rank, world);
  lga_rank_plan p{};
  p.stage = rank % c.P;
  p.replica = rank / c.P;
  p.local_layers = c.Lloc;
  p.chunk = c.c;
  p.first_layer = (int32_t)local_to_global_s(c, p.stage, 0);
  p.layer_stride = c.contig ? 1 : c.P;
  unsigned long long sf, rf, sb, rb;
  plan_transfers(c, p.stage, &sf, &rf, &sb, &rb);
  p.p2p_send_fwd = sf; p.p2p_recv_fwd = rf; p.p2p_send_bwd = sb; p.p2p_recv_bwd = rb;
  p.shard_elems = (uint64_t)c.S;
  p.layer_elems_padded = (uint64_t)c.plpad;
  *out = p;
  return LGA_OK;
}

lga_status lga_nccl_unique_id(uint8_t* out) {
  if (!out) return ERR(LGA_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return ERR(LGA_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == LGA_NCCL_ID_BYTES, "nccl id size");
  memcpy(out, &id, sizeof(id));
  return LGA_OK;
}

// Device barrier of all world ranks over peer memory (collective; every rank calls it in the same order).
// Returns false if it timed out (a peer never arrived).
static bool world_sync(lga_handle* h, double timeout_s) {
  if (h->world <= 1 || !h->connected) return true;
  h->n_barrier += 1;
  CK(cudaMemsetAsync(h->barrier_to, 0, sizeof(int), h->s_comp));
  world_barrier(h->w_flag_dev, h->world, h->n_barrier * (unsigned long long)h->world, h->wflags + 1, h->barrier_to,
                (long long)(timeout_s * 1e9), h->s_comp);
  KCHECK();
  int to = 0;
  CK(cudaMemcpyAsync(&to, h->barrier_to, sizeof(int), cudaMemcpyDeviceToHost, h->s_comp));
  CK(cudaStreamSynchronize(h->s_comp));
  return to == 0;
}

static void free_handle(lga_handle* h) {
  if (!h) return;
  cudaSetDevice(h->dev);
  if (h->stepped && h->ev_t1) cudaEventSynchronize(h->ev_t1);   // the last step (graph replays run on the caller stream)
  if (h->s_comp) cudaStreamSynchronize(h->s_comp);
  if (h->s_comm) cudaStreamSynchronize(h->s_comm);
  if (h->s_copy) cudaStreamSynchronize(h->s_copy);
  // peers write into this arena (pipeline transfers, counters, loss slots): free it only after every rank is done
  if (h->ready && h->connected && !h->bad) {
    try {
      world_sync(h, 60.0);
    } catch (...) {
    }
  }
  cudaGetLastError();
  for (auto& gr : h->graphs)
    if (gr.exec) cudaGraphExecDestroy(gr.exec);
  for (size_t q = 0; q < h->wbase.size(); ++q)
    if (h->wbase[q] && h->wbase[q] != h->arena.base) cudaIpcCloseMemHandle(h->wbase[q]);
  if (h->dp_comm) ncclCommDestroy(h->dp_comm);
  if (h->world_comm) ncclCommDestroy(h->world_comm);
  cudaEvent_t evs[] = {h->ev_in, h->ev_tin, h->ev_grad[0], h->ev_grad[1], h->ev_adam[0], h->ev_adam[1], h->ev_comm_end,
                       h->ev_comp_end, h->ev_t0, h->ev_t1, h->ev_fwd_end};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto* v : {&h->ev_ag, &h->ev_x, &h->ev_slot_free, &h->ev_wait0, &h->ev_wait1, &h->prof0, &h->prof1})
    for (auto e : *v)
      if (e) cudaEventDestroy(e);
  if (h->s_comp) cudaStreamDestroy(h->s_comp);
  if (h->s_comm) cudaStreamDestroy(h->s_comm);
  if (h->s_copy) cudaStreamDestroy(h->s_copy);
  if (h->arena.base) cudaFree(h->arena.base);
  if (h->loss_host) cudaFreeHost(h->loss_host);
  cudaGetLastError();
  delete h;
}

lga_status lga_init(const lga_config* cfg, int32_t rank, int32_t world, int32_t device, lga_allgather_fn allgather,
                    void* allgather_ctx, const uint8_t* nccl_id, uintptr_t cuda_stream, const float* init_params,
                    uint64_t seed, lga_handle** out) {
  if (!out) return ERR(LGA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  Cfg c;
  lga_status s = validate(cfg, world, &c);
  if (s != LGA_OK) return s;
  if (rank < 0 || rank >= world) return ERR(LGA_ERR_INVALID_ARG, "rank %d out of [0, %d)", rank, world);
  if (world > 1 && !allgather && !nccl_id)
    return ERR(LGA_ERR_INVALID_ARG, "world %d needs a bootstrap: an allgather callback or an nccl_id", world);
  if (c.nccl_dp && !nccl_id) return ERR(LGA_ERR_INVALID_ARG, "LGA_FLAG_NCCL_DP with dp > 1 needs nccl_id");
  lga_handle* h = new lga_handle();
  h->c = c;
  h->rank = rank;
  h->world = world;
  h->dev = device;
  h->stage = rank % c.P;
  h->replica = rank / c.P;
  h->user = reinterpret_cast<cudaStream_t>(cuda_stream);
  ABI_TRY
  CK(cudaSetDevice(device));
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithPriority(&h->s_comp, cudaStreamNonBlocking, prio_lo));
  CK(cudaStreamCreateWithPriority(&h->s_comm, cudaStreamNonBlocking, prio_hi));   // comm first
  CK(cudaStreamCreateWithPriority(&h->s_copy, cudaStreamNonBlocking, prio_lo));
  cudaEvent_t* evs[] = {&h->ev_in, &h->ev_tin, &h->ev_grad[0], &h->ev_grad[1], &h->ev_adam[0], &h->ev_adam[1], &h->ev_comm_end,
                        &h->ev_comp_end};
  for (auto e : evs) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  const int nev = std::max(2, c.Lloc);   // one per parameter slot (2, or L/P with KEEP_PARAMS)
  h->ev_ag.assign(nev, nullptr);
  h->ev_slot_free.assign(nev, nullptr);
  for (int k = 0; k < nev; ++k) {
    CK(cudaEventCreateWithFlags(&h->ev_ag[k], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_slot_free[k], cudaEventDisableTiming));
  }
  h->rec_slot.assign(nev, 0);
  h->ev_x.assign(c.N, nullptr);
  for (auto& e : h->ev_x) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // pipeline transfers per step on this stage (flag epochs): chunks of every layer boundary it crosses
  plan_transfers(c, h->stage, &h->k_send_fwd, &h->k_recv_fwd, &h->k_send_bwd, &h->k_recv_bwd);
  CK(cudaEventCreate(&h->ev_t0));
  CK(cudaEventCreate(&h->ev_t1));
  CK(cudaEventCreate(&h->ev_fwd_end));
  // arena: plan, allocate once, carve
  {
    const char* gv = getenv("LGA_ARENA_GUARD");
    h->arena.guard = gv && gv[0] == '1';
  }
  h->arena.planning = true;
  plan_arena(h);
  const size_t need = h->arena.used + 4096;
  cudaError_t ae = cudaMalloc(&h->arena.base, need);
  if (ae != cudaSuccess) {
    cudaGetLastError();
    free_handle(h);
    return ERR(LGA_ERR_OUT_OF_MEMORY, "arena of %zu bytes: %s", need, cudaGetErrorString(ae));
  }
  h->arena.cap = need;
  h->arena.planning = false;
  h->arena.guards.clear();
  plan_arena(h);
  CK(cudaMemsetAsync(h->arena.base, 0, need, h->s_comp));
  for (size_t g : h->arena.guards) CK(cudaMemsetAsync(h->arena.base + g, GUARD_BYTE, GUARD, h->s_comp));
  CK(cudaMallocHost(&h->loss_host, 8 * sizeof(double)));
  // NCCL only for the baseline (LGA_FLAG_NCCL_DP) or, without an allgather callback, for the bootstrap exchange
  if (world > 1 && nccl_id) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    NK(ncclCommInitRank(&h->world_comm, world, id, rank));
    if (c.nccl_dp) NK(ncclCommSplit(h->world_comm, h->stage, h->replica, &h->dp_comm, nullptr));
  }
  // parameters: fp32 master shard of each local layer (A-10: contiguous 1/D slice of the padded layer)
  const int64_t Ll = c.Lloc;
  {
    std::vector<float> tmp;
    float* dev_full = nullptr;
    if (!init_params) CK(cudaMalloc(&dev_full, (size_t)c.pl * sizeof(float)));
    for (int j = 0; j < Ll; ++j) {
      const int64_t gl = local_to_global(h, j);
      const int64_t lo = c.unpart ? 0 : (int64_t)h->replica * c.S, hi = std::min<int64_t>(lo + c.S, c.pl);
      float* dst = h->master + (int64_t)j * c.S;
      if (init_params) {
        if (hi > lo)
          CK(cudaMemcpyAsync(dst, init_params + gl * c.pl + lo, (size_t)(hi - lo) * sizeof(float), cudaMemcpyHostToDevice,
                             h->s_comp));
      } else {
        init_params_device(dev_full, 1, c.d, 4, c.L, gl, seed, h->s_comp);
        KCHECK();
        if (hi > lo)
          CK(cudaMemcpyAsync(dst, dev_full + lo, (size_t)(hi - lo) * sizeof(float), cudaMemcpyDeviceToDevice, h->s_comp));
      }
    }
    CK(cudaStreamSynchronize(h->s_comp));
    if (dev_full) CK(cudaFree(dev_full));
    cast_f32(h->master, h->pshard, c.E, Ll * c.S, h->s_comp);
    KCHECK();
  }
  // bootstrap (world > 1): exchange every rank's arena IPC handle and offsets, map all of them.  The arena is
  // zeroed and synchronised above, so once a rank holds every handle, every peer's counters are initialised.
  if (world > 1) {
    CK(cudaStreamSynchronize(h->s_comp));
    PeerInfo me{};
    CK(cudaIpcGetMemHandle(&me.handle, h->arena.base));
    auto off = [&](const void* p) { return p ? (uint64_t)((const char*)p - h->arena.base) : 0ull; };
    me.off_ckpt = off(h->ckpt);
    me.off_dY = off(h->dY);
    me.off_flags = off(h->flags);
    me.off_gst = off(h->gst_layers);
    me.off_psh = off(h->pshard);
    me.off_dpf = off(h->dpf);
    me.off_master = off(h->master);
    me.off_gkeep = off(h->gkeep);
    me.off_wflags = off(h->wflags);
    me.off_loss = off(h->loss_ring);
    me.rank = rank;
    me.world = world;
    std::vector<PeerInfo>& all = h->peers;
    all.assign(world, PeerInfo{});
    if (allgather) {
      if (allgather(allgather_ctx, &me, all.data(), sizeof(PeerInfo)) != 0) {
        ERR(LGA_ERR_INVALID_ARG, "the allgather callback failed");
        throw StatusError{LGA_ERR_INVALID_ARG};
      }
    } else {
      PeerInfo* dev_info = nullptr;
      CK(cudaMalloc(&dev_info, sizeof(PeerInfo) * (world + 1)));
      CK(cudaMemcpy(dev_info + world, &me, sizeof(me), cudaMemcpyHostToDevice));
      NK(ncclAllGather(dev_info + world, dev_info, sizeof(PeerInfo), ncclUint8, h->world_comm, h->s_comp));
      CK(cudaMemcpyAsync(all.data(), dev_info, sizeof(PeerInfo) * world, cudaMemcpyDeviceToHost, h->s_comp));
      CK(cudaStreamSynchronize(h->s_comp));
      CK(cudaFree(dev_info));
    }
    for (int q = 0; q < world; ++q)
      if (all[q].rank != q || all[q].world != world) {
        ERR(LGA_ERR_INVALID_ARG, "bootstrap: slot %d holds rank %d of world %d", q, all[q].rank, all[q].world);
        throw StatusError{LGA_ERR_INVALID_ARG};
      }
    h->wbase.assign(world, nullptr);
    for (int q = 0; q < world; ++q) {
      if (q == rank) {
        h->wbase[q] = h->arena.base;
        continue;
      }
      void* pb = nullptr;
      CK(cudaIpcOpenMemHandle(&pb, all[q].handle, cudaIpcMemLazyEnablePeerAccess));
      h->wbase[q] = (char*)pb;
    }
    h->connected = true;
    std::vector<unsigned long long*> wf(world);
    std::vector<double*> wl(world);
    for (int q = 0; q < world; ++q) {
      wf[q] = (unsigned long long*)(h->wbase[q] + all[q].off_wflags);
      wl[q] = (double*)(h->wbase[q] + all[q].off_loss);
    }
    CK(cudaMemcpy(h->w_flag_dev, wf.data(), world * sizeof(void*), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->w_loss_dev, wl.data(), world * sizeof(void*), cudaMemcpyHostToDevice));
    if (c.P > 1) {
      const int next = h->replica * c.P + (h->stage + 1) % c.P;
      const int prev = h->replica * c.P + (h->stage + c.P - 1) % c.P;
      h->next_ckpt = (float*)(h->wbase[next] + all[next].off_ckpt);
      h->next_flags = (unsigned long long*)(h->wbase[next] + all[next].off_flags);
      h->prev_dY = (float*)(h->wbase[prev] + all[prev].off_dY);
      h->prev_flags = (unsigned long long*)(h->wbase[prev] + all[prev].off_flags);
    }
    if (c.D > 1) {  // the replicas of this stage, in replica order (self: own arena)
      h->dp_base.assign(c.D, nullptr);
      h->dp_psh.assign(c.D, nullptr);
      std::vector<void*> gst(c.D);
      std::vector<unsigned long long*> fl(c.D);
      for (int r = 0; r < c.D; ++r) {
        const int q = r * c.P + h->stage;
        h->dp_base[r] = h->wbase[q];
        h->dp_psh[r] = h->wbase[q] + all[q].off_psh;
        gst[r] = h->wbase[q] + all[q].off_gst;
        fl[r] = (unsigned long long*)(h->wbase[q] + all[q].off_dpf);
      }
      if (c.dp_ipc) {
        CK(cudaMemcpy(h->dp_gst_dev, gst.data(), c.D * sizeof(void*), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->dp_flag_dev, fl.data(), c.D * sizeof(unsigned long long*), cudaMemcpyHostToDevice));
      }
    }
  }
  CK(cudaStreamSynchronize(h->s_comp));
  // both "staging buffer free" events start completed
  CK(cudaEventRecord(h->ev_adam[0], h->s_comm));
  CK(cudaEventRecord(h->ev_adam[1], h->s_comm));
  for (auto e : h->ev_slot_free) CK(cudaEventRecord(e, h->s_comp));
  h->ready = true;
  *out = h;
  return LGA_OK;
  } catch (const StatusError& e) {   // free everything allocated so far; *out stays NULL
    free_handle(h);
    return e.s;
  } catch (...) {
    free_handle(h);
    return ERR(LGA_ERR_CUDA, "unexpected exception in lga_init");
  }
}

// Issue one step on s_comp / s_comm / s_copy: from "s_comp, s_comm start after ev_in" to "s_comp has joined
// every stream".  Host-side counters (h->last, the event indices) are rebuilt on every issue.
static void issue_step(lga_handle* h, const float* x, const float* T, bool host_inputs) {
  const Cfg& c = h->c;
  const bool need_x = h->stage == 0, need_t = owns_last(h);
  h->last = lga_comm_stats{};
  h->n_wait = 0;
  h->n_prof = 0;
  h->sent_fwd = h->sent_bwd = h->recv_fwd = h->recv_bwd = 0;
  h->x_split = false;
  h->rec_adam[0] = h->rec_adam[1] = false;
  std::fill(h->rec_slot.begin(), h->rec_slot.end(), 0);
  step_begin(h->tstep, h->s_comp);   // t += 1 and epoch += 1 before anything reads them
  KCHECK();
  CK(cudaEventRecord(h->ev_in, h->s_comp));
  CK(cudaStreamWaitEvent(h->s_comm, h->ev_in, 0));
  const int64_t act = (int64_t)c.N * c.M * c.d;
  if (host_inputs) {
    if (need_x && c.layered) {   // per micro-batch on s_copy: layer 0 starts on the first one (forward rows are
                                 // independent, so the per-micro-batch layer-0 launches give the same bits)
      CK(cudaStreamWaitEvent(h->s_copy, h->ev_in, 0));
      const int64_t mb = (int64_t)c.M * c.d;
      for (int m = 0; m < c.N; ++m) {
        CK(cudaMemcpyAsync(h->xin + m * mb, x + m * mb, mb * sizeof(float), cudaMemcpyHostToDevice, h->s_copy));
        CK(cudaEventRecord(h->ev_x[m], h->s_copy));
      }
      h->x_split = true;
    } else if (need_x) {   // on s_copy too, so that the end-of-call sync of s_copy covers every host read
      CK(cudaStreamWaitEvent(h->s_copy, h->ev_in, 0));
      CK(cudaMemcpyAsync(h->xin, x, act * sizeof(float), cudaMemcpyHostToDevice, h->s_copy));
      CK(cudaEventRecord(h->ev_x[0], h->s_copy));
      CK(cudaStreamWaitEvent(h->s_comp, h->ev_x[0], 0));
    }
    if (need_t) {  // needed only at the loss: copy on s_copy, overlapped with the forward
      if (!need_x) CK(cudaStreamWaitEvent(h->s_copy, h->ev_in, 0));
      CK(cudaMemcpyAsync(h->tin, T, act * sizeof(float), cudaMemcpyHostToDevice, h->s_copy));
      CK(cudaEventRecord(h->ev_tin, h->s_copy));
      h->tin_pending = true;
    }
    x = need_x ? h->xin : nullptr;
    T = need_t ? h->tin : nullptr;
  }
  CK(cudaMemsetAsync(h->loss_dev, 0, (c.N + 8) * sizeof(double), h->s_comp));
  rec_time(h, h->ev_fwd_end, h->s_comp);   // re-recorded at the forward/backward boundary (LAYERED)
  if (c.layered) step_layered(h, x, T);
  else step_standard(h, x, T);
  await_target(h);
  // global loss: sum of this rank's micro-batch losses (slots 1..N), all-reduced, / (D N)
  mse_finish(h->loss_dev + 1, c.N, 1.0, h->loss_dev, h->s_comp);
  KCHECK();
  h->last.allreduce_calls += 1;   // the loss (plus, unpartitioned, the per-layer gradient all-reduces)
  if (h->world > 1 && !h->comm_off) {   // over peer memory (every rank gets the same rank-order sum)
    count_wait(h, nullptr, 0);          // the kernel waits for the peers' losses: an exposed wait
    loss_allreduce_peer(h->loss_dev, h->w_loss_dev, h->w_flag_dev, h->rank, h->world, h->tepoch, h->wflags + 0,
                        h->loss_ring, h->s_comp);
    KCHECK();
    count_wait_end(h);
  }
  CK(cudaMemcpyAsync(h->loss_host, h->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, h->s_comp));
  // the step ends when the last reduce-scatter + AdamW (layer 0's, the exposed tail) has finished
  CK(cudaEventRecord(h->ev_comm_end, h->s_comm));
  count_wait(h, h->ev_comm_end, 0);
  count_wait_end(h);
}

// Capture issue_step into a graph (LGA_FLAG_NO_GRAPH off, device inputs).  False on any capture failure
// (the step then runs eagerly and capture is not retried).
static bool capture_step(lga_handle* h, lga_handle::StepGraph& gr, const float* x, const float* T) {
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(h->s_comp, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  h->capturing = true;
  const unsigned long long l0 = launch_count();
  bool ok = true;
  try {
    issue_step(h, x, T, false);
  } catch (const StatusError&) {
    ok = false;
  }
  h->capturing = false;
  cudaError_t e = cudaStreamEndCapture(h->s_comp, &graph);
  if (!ok || e != cudaSuccess || !graph) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    return false;
  }
  e = cudaGraphInstantiateWithFlags(&gr.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    cudaGetLastError();
    gr.exec = nullptr;
    return false;
  }
  gr.x = x;
  gr.T = T;
  gr.last = h->last;
  gr.nwait = h->n_wait;
  gr.nprof = h->n_prof;
  gr.launches = launch_count() - l0;
  return true;
}

static lga_status run_step(lga_handle* h, const float* x, const float* T, double* loss_out, bool host_inputs) {
  if (!h) return ERR(LGA_ERR_INVALID_ARG, "handle is NULL");
  if (h->bad) return ERR(LGA_ERR_BAD_STATE, "handle latched after an earlier CUDA/NCCL error");
  const Cfg& c = h->c;
  const bool need_x = h->stage == 0, need_t = owns_last(h);
  if ((need_x && !x) || (need_t && !T)) return ERR(LGA_ERR_INVALID_ARG, "x / target NULL on a stage that reads it");
  ABI_TRY
  CK(cudaSetDevice(h->dev));
  h->t += 1;
  NvtxRange nvtx_step("lga step", h->t);
  h->comm_off = c.no_comm && h->t > 1;
  CK(cudaEventRecord(h->ev_t0, h->user));
  // CUDA graph of the whole step: captured at the second device-input call, replayed while the input
  // pointers stay the same; the first call (lazy initialisation) and host-input calls run eagerly
  const bool graph_ok = !host_inputs && !c.graph_off && !h->graph_broken && h->eager_steps >= 1;
  lga_handle::StepGraph* gr = nullptr;
  if (graph_ok) {
    for (auto& e : h->graphs)
      if (e.exec && e.x == x && e.T == T) gr = &e;
    if (!gr) {   // capture into a free slot or over the least recently used one
      gr = &h->graphs[0];
      for (auto& e : h->graphs)
        if (!e.exec || e.used < gr->used) gr = &e;
      if (gr->exec) {
        CK(cudaGraphExecDestroy(gr->exec));
        gr->exec = nullptr;
      }
      CK(cudaEventRecord(h->ev_in, h->user));          // order the capture's stream after the caller
      CK(cudaStreamWaitEvent(h->s_comp, h->ev_in, 0));
      if (!capture_step(h, *gr, x, T)) {
        h->graph_broken = true;
        gr = nullptr;
      } else {
        h->graph_captures++;
      }
    }
  }
  if (gr) {
    gr->used = ++h->graph_clock;
    CK(cudaGraphLaunch(gr->exec, h->user));
    h->last = gr->last;
    h->n_wait = gr->nwait;
    h->n_prof = gr->nprof;
    h->launches_last = gr->launches;
  } else {
    const unsigned long long l0 = launch_count();
    CK(cudaEventRecord(h->ev_in, h->user));
    CK(cudaStreamWaitEvent(h->s_comp, h->ev_in, 0));
    issue_step(h, x, T, host_inputs);
    CK(cudaEventRecord(h->ev_comp_end, h->s_comp));
    CK(cudaStreamWaitEvent(h->user, h->ev_comp_end, 0));
    h->launches_last = launch_count() - l0;
    h->eager_steps += 1;
  }
  CK(cudaEventRecord(h->ev_t1, h->user));
  h->stepped = true;
  if (host_inputs) CK(cudaStreamSynchronize(h->s_copy));   // the caller may reuse x / target on return
  h->last.steps = 1;
  lga_comm_stats& tt = h->total;
  tt.steps += 1;
  tt.ag_calls += h->last.ag_calls; tt.rs_calls += h->last.rs_calls; tt.p2p_send_calls += h->last.p2p_send_calls;
  tt.p2p_recv_calls += h->last.p2p_recv_calls; tt.allreduce_calls += h->last.allreduce_calls;
  tt.ag_bytes += h->last.ag_bytes; tt.rs_bytes += h->last.rs_bytes; tt.p2p_send_bytes += h->last.p2p_send_bytes;
  tt.p2p_recv_bytes += h->last.p2p_recv_bytes; tt.fwd_units += h->last.fwd_units; tt.bwd_units += h->last.bwd_units;
  tt.recompute_units += h->last.recompute_units; tt.allreduce_bytes += h->last.allreduce_bytes;
  if (loss_out) {
    CK(cudaEventSynchronize(h->ev_t1));
    *loss_out = h->loss_host[0] / ((double)c.D * (double)c.N);
  }
  return LGA_OK;
  ABI_CATCH
}

lga_status lga_step(lga_handle* h, const float* x, const float* target, double* loss_out) {
  return run_step(h, x, target, loss_out, false);
}

lga_status lga_step_host(lga_handle* h, const float* x, const float* target, double* loss_out) {
  return run_step(h, x, target, loss_out, true);
}

// lga_grads / lga_params: this rank's stage layers in canonical layout.  The D replicas' shards are read over
// peer memory between two world barriers (every peer finished its last step before the reads; nobody starts
// the next step, which rewrites master / m / v, before every rank has read).
static lga_status gather_state(lga_handle* h, const float* src_shards, uint64_t peer_off, float* out, uint64_t n,
                               int32_t on_device) {
  if (!h) return ERR(LGA_ERR_INVALID_ARG, "handle is NULL");
  if (h->bad) return ERR(LGA_ERR_BAD_STATE, "handle latched");
  const Cfg& c = h->c;
  const uint64_t expect = (uint64_t)c.Lloc * c.pl;
  if (n != expect) return ERR(LGA_ERR_SIZE_MISMATCH, "n = %llu, expected %llu", (unsigned long long)n, (unsigned long long)expect);
  if (!out) return ERR(LGA_ERR_INVALID_ARG, "out is NULL");
  ABI_TRY
  CK(cudaSetDevice(h->dev));
  if (h->stepped) CK(cudaEventSynchronize(h->ev_t1));   // the last step (a replayed graph runs on the caller's stream)
  CK(cudaStreamSynchronize(h->s_comp));
  CK(cudaStreamSynchronize(h->s_comm));
  const bool sharded = c.D > 1 && !c.unpart;
  if (sharded && !world_sync(h, 600.0)) {
    ERR(LGA_ERR_CUDA, "world barrier timed out (a peer did not call lga_grads / lga_params)");
    throw StatusError{LGA_ERR_CUDA};
  }
  float* full = nullptr;
  CK(cudaMalloc(&full, (size_t)c.Lloc * c.plpad * sizeof(float)));
  for (int j = 0; j < c.Lloc; ++j) {
    float* dst = full + (int64_t)j * c.plpad;
    if (sharded) {
      for (int r = 0; r < c.D; ++r) {
        const char* src = h->dp_base[r] + peer_off + (size_t)j * c.S * sizeof(float);
        CK(cudaMemcpyAsync(dst + (int64_t)r * c.S, src, (size_t)c.S * sizeof(float), cudaMemcpyDeviceToDevice, h->s_comp));
      }
    } else {
      CK(cudaMemcpyAsync(dst, src_shards + (int64_t)j * c.S, (size_t)c.S * sizeof(float), cudaMemcpyDeviceToDevice,
                         h->s_comp));
    }
  }
  CK(cudaStreamSynchronize(h->s_comp));
  if (sharded && !world_sync(h, 600.0)) {
    ERR(LGA_ERR_CUDA, "world barrier timed out");
    throw StatusError{LGA_ERR_CUDA};
  }
  for (int j = 0; j < c.Lloc; ++j) {
    CK(cudaMemcpyAsync(out + (int64_t)j * c.pl, full + (int64_t)j * c.plpad, (size_t)c.pl * sizeof(float),
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->s_comp));
  }
  CK(cudaStreamSynchronize(h->s_comp));
  CK(cudaFree(full));
  return LGA_OK;
  ABI_CATCH
}

lga_status lga_grads(lga_handle* h, float* out, uint64_t n, int32_t out_on_device) {
  if (h && !h->c.retain) return ERR(LGA_ERR_INVALID_ARG, "retain_grads was 0 at lga_init");
  return gather_state(h, h ? h->gkeep : nullptr, h && h->connected ? h->peers[h->rank].off_gkeep : 0, out, n,
                      out_on_device);
}

lga_status lga_params(lga_handle* h, float* out, uint64_t n, int32_t out_on_device) {
  return gather_state(h, h ? h->master : nullptr, h && h->connected ? h->peers[h->rank].off_master : 0, out, n,
                      out_on_device);
}

// ------------------------------------------------------------------ checkpoint / resume of the training state
struct StateHeader {
  uint64_t magic;    // "LGASTATE"
  uint32_t abi, rank;
  int32_t L, d, D, P, Lloc, precision;
  int64_t S, t;
  uint64_t flags;
};
static constexpr uint64_t kStateMagic = 0x4554415453414c47ull;   // little-endian "LGASTATE"

lga_status lga_state_bytes(const lga_handle* h, uint64_t* bytes) {
  if (!h || !bytes) return ERR(LGA_ERR_INVALID_ARG, "NULL argument");
  *bytes = sizeof(StateHeader) + 3ull * h->c.Lloc * h->c.S * sizeof(float);
  return LGA_OK;
}

static void fill_header(const lga_handle* h, StateHeader* hd, int64_t t) {
  const Cfg& c = h->c;
  *hd = StateHeader{};
  hd->magic = kStateMagic;
  hd->abi = LGA_ABI_VERSION;
  hd->rank = (uint32_t)h->rank;
  hd->L = c.L; hd->d = c.d; hd->D = c.D; hd->P = c.P; hd->Lloc = c.Lloc; hd->precision = c.bf16 ? 1 : 0;
  hd->S = c.S;
  hd->t = t;
  hd->flags = (c.unpart ? 1u : 0u) | (c.contig ? 2u : 0u);
}

lga_status lga_save_state(lga_handle* h, void* host_out, uint64_t bytes) {
  if (!h || !host_out) return ERR(LGA_ERR_INVALID_ARG, "NULL argument");
  if (h->bad) return ERR(LGA_ERR_BAD_STATE, "handle latched");
  uint64_t need = 0;
  lga_state_bytes(h, &need);
  if (bytes != need) return ERR(LGA_ERR_SIZE_MISMATCH, "bytes = %llu, expected %llu", (unsigned long long)bytes,
                                (unsigned long long)need);
  ABI_TRY
  CK(cudaSetDevice(h->dev));
  if (h->stepped) CK(cudaEventSynchronize(h->ev_t1));
  CK(cudaStreamSynchronize(h->s_comp));
  CK(cudaStreamSynchronize(h->s_comm));
  StateHeader hd;
  fill_header(h, &hd, h->t);
  char* out = static_cast<char*>(host_out);
  memcpy(out, &hd, sizeof(hd));
  const size_t n = (size_t)h->c.Lloc * h->c.S * sizeof(float);
  CK(cudaMemcpy(out + sizeof(hd), h->master, n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out + sizeof(hd) + n, h->mom, n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out + sizeof(hd) + 2 * n, h->var, n, cudaMemcpyDeviceToHost));
  return LGA_OK;
  ABI_CATCH
}

lga_status lga_load_state(lga_handle* h, const void* host_in, uint64_t bytes) {
  if (!h || !host_in) return ERR(LGA_ERR_INVALID_ARG, "NULL argument");
  if (h->bad) return ERR(LGA_ERR_BAD_STATE, "handle latched");
  uint64_t need = 0;
  lga_state_bytes(h, &need);
  if (bytes != need) return ERR(LGA_ERR_SIZE_MISMATCH, "bytes = %llu, expected %llu", (unsigned long long)bytes,
                                (unsigned long long)need);
  StateHeader hd, mine;
  memcpy(&hd, host_in, sizeof(hd));
  fill_header(h, &mine, hd.t);
  if (memcmp(&hd, &mine, sizeof(hd)) != 0 || hd.t < 0)
    return ERR(LGA_ERR_INVALID_ARG, "state of another configuration or rank (L %d d %d D %d P %d rank %u)", hd.L, hd.d,
               hd.D, hd.P, hd.rank);
  ABI_TRY
  CK(cudaSetDevice(h->dev));
  if (h->stepped) CK(cudaEventSynchronize(h->ev_t1));
  CK(cudaStreamSynchronize(h->s_comp));
  CK(cudaStreamSynchronize(h->s_comm));
  const char* in = static_cast<const char*>(host_in);
  const size_t n = (size_t)h->c.Lloc * h->c.S * sizeof(float);
  CK(cudaMemcpy(h->master, in + sizeof(hd), n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->mom, in + sizeof(hd) + n, n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->var, in + sizeof(hd) + 2 * n, n, cudaMemcpyHostToDevice));
  // the 16-bit parameter shard the next all-gather reads, and the AdamW step (flag epochs stay this handle's)
  cast_f32(h->master, h->pshard, h->c.E, (int64_t)h->c.Lloc * h->c.S, h->s_comp);
  KCHECK();
  const long long t = hd.t;
  CK(cudaMemcpyAsync(h->tstep, &t, sizeof(t), cudaMemcpyHostToDevice, h->s_comp));
  CK(cudaStreamSynchronize(h->s_comp));
  h->t = t;
  // a peer's next step all-gathers this rank's parameter shard as soon as it starts: return only when every
  // rank has restored its own (a fresh handle's flag epochs give its first gather nothing to wait for)
  if (!world_sync(h, 600.0)) {
    ERR(LGA_ERR_CUDA, "world barrier timed out (a peer did not call lga_load_state)");
    throw StatusError{LGA_ERR_CUDA};
  }
  return LGA_OK;
  ABI_CATCH
}

lga_status lga_comm_bytes(const lga_handle* h, lga_comm_stats* last_step, lga_comm_stats* total) {
  if (!h) return ERR(LGA_ERR_INVALID_ARG, "handle is NULL");
  if (last_step) *last_step = h->last;
  if (total) *total = h->total;
  return LGA_OK;
}

lga_status lga_layer_stage(const lga_handle* h, int32_t* stage_of_layer, int32_t n) {
  if (!h || !stage_of_layer) return ERR(LGA_ERR_INVALID_ARG, "NULL argument");
  if (n != h->c.L) return ERR(LGA_ERR_SIZE_MISMATCH, "n = %d, expected L = %d", n, h->c.L);
  for (int i = 0; i < n; ++i) stage_of_layer[i] = stage_of(h->c, i);   // P:127 (modular) / P:71 (contiguous)
  return LGA_OK;
}

lga_status lga_timing_last(lga_handle* h, lga_timing* out) {
  if (!h || !out) return ERR(LGA_ERR_INVALID_ARG, "NULL argument");
  if (h->bad) return ERR(LGA_ERR_BAD_STATE, "handle latched");
  ABI_TRY
  CK(cudaEventSynchronize(h->ev_t1));
  lga_timing t{};
  CK(cudaEventElapsedTime(&t.step_ms, h->ev_t0, h->ev_t1));
  for (int k = 0; k < h->n_wait; ++k) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev_wait0[k], h->ev_wait1[k]));
    if (h->wait_kind[k] == 0) t.comm_wait_ms += ms; else t.p2p_wait_ms += ms;
  }
  CK(cudaEventElapsedTime(&t.fwd_ms, h->ev_t0, h->ev_fwd_end));
  CK(cudaEventElapsedTime(&t.bwd_ms, h->ev_fwd_end, h->ev_t1));
  for (int k = 0; k < h->n_prof; ++k) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->prof0[k], h->prof1[k]));
    switch (h->prof_fam[k]) {
      case FAM_GEMM: t.gemm_ms += ms; t.gemm_launches++; t.gemm_flop += h->prof_work[k]; break;
      case FAM_ATTN: t.attn_ms += ms; t.attn_launches++; t.attn_flop += h->prof_work[k]; break;
      default: t.adam_ms += ms; t.adam_launches++; t.adam_bytes += h->prof_work[k]; break;
    }
  }
  t.kernel_launches = h->launches_last;
  t.graph_captures = h->graph_captures;
  *out = t;
  return LGA_OK;
  ABI_CATCH
}

void lga_destroy(lga_handle* h) { free_handle(h); }

// negative control of the guard check: overwrite one byte of the last canary (as a kernel writing one byte past
// the end of the last arena buffer would)
int lgatest_arena_guard_poke(lga_handle* h) {
  if (!h || !h->arena.guard || h->arena.guards.empty()) return -1;
  return (int)cudaMemset(h->arena.base + h->arena.guards.back(), 0, 1);
}

// test hook (include/lga_testing.h): canary bytes overwritten in the guard-mode arena; -1 = not in guard mode
int64_t lgatest_arena_guard_check(lga_handle* h) {
  if (!h || !h->arena.guard) return -1;
  cudaSetDevice(h->dev);
  if (h->stepped) cudaEventSynchronize(h->ev_t1);
  cudaStreamSynchronize(h->s_comp);
  cudaStreamSynchronize(h->s_comm);
  std::vector<unsigned char> buf(GUARD);
  int64_t bad = 0;
  for (size_t g : h->arena.guards) {
    if (cudaMemcpy(buf.data(), h->arena.base + g, GUARD, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
    for (unsigned char b : buf) bad += b != GUARD_BYTE;
  }
  return bad;
}

}  // extern "C"
