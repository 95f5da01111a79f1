// kernels.cuh -- host-side launchers of every device kernel of the LGA step.
//
// One layer (reading A-1), per token row x in R^d:
//   a = LN1(x); qkv = a Wqkv + bqkv; o = causal-softmax-attention(q, k, v); h1 = x + o Wo + bo
//   c = LN2(h1); u = c W1 + b1; g = GELU(u); y = h1 + g W2 + b2
// Storage element type E is fp32 (parity mode) or bf16 (the paper's 16-bit compute,
// P:85); accumulation is always fp32.
#pragma once

#include "common.cuh"

namespace lga {

// ------------------------------------------------------------------ GEMM
// C[m][n] = sum_k A(m,k) * B(n,k), then the epilogue.
//   A(m,k) = A[m*lda + k] if a_kmajor else A[k*lda + m]
//   B(n,k) = B[n*ldb + k] if b_kmajor else B[k*ldb + n]
// Forward  Y = X W      : A = X (K-major), B(n,k) = W[k][n] (MN-major)
// dgrad    dX = dY W^T  : A = dY (K-major), B(n,k) = W[n][k] (K-major)
// wgrad    dW = X^T dY  : A(m,k) = X[k][m] (MN-major), B(n,k) = dY[k][n] (MN-major)
enum EpiKind : int {
  EPI_STORE = 0,      // out = acc (+bias[n]) (+res[m][n]) (+acc_in[m][n])
  EPI_GELU_FWD = 1,   // u = acc + bias[n] -> aux (E; not stored when aux == nullptr); out = GELU(u) (E)
  EPI_GELU_BWD = 2,   // out = acc * GELU'(aux[m][n])   (aux holds u; out may alias aux)
};

struct Epi {
  int kind = EPI_STORE;
  const void* bias = nullptr; DT bias_dt = DT::F32;   // per column n
  const float* res = nullptr; int64_t ldr = 0;         // fp32 residual
  const float* acc_in = nullptr; int64_t ldacc = 0;    // fp32 accumulator added (gradient accumulation)
  void* aux = nullptr; int64_t ldaux = 0; DT aux_dt = DT::F32;
  void* out = nullptr; int64_t ldo = 0; DT out_dt = DT::F32;
  // EPI_GELU_BWD on the tensor-core path: also the column sums of out (the bias gradient of the GEMM that
  // produced u, db1 = sum_rows dU) per 32-row strip: colsum[(m / 32) * N + n], ceil(M / 32) rows, fp32
  float* colsum = nullptr;
};

struct GemmArgs {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr; int64_t lda = 0; bool a_kmajor = true;
  const void* B = nullptr; int64_t ldb = 0; bool b_kmajor = true;
  Epi epi;
  // tensor-core path, deterministic split over K (chosen by gemm_bf16_tc when the tile count would leave SMs
  // idle and M % 128 == 0): partial sums go to the workspace [split][M][N] fp32, then one reduce pass adds them
  // in split order and runs the epilogue.  splitk_ws = nullptr disables it.
  int split_k = 1;
  float* splitk_ws = nullptr;
  int64_t splitk_ws_floats = 0;   // workspace capacity
  bool b_keep_l2 = false;          // set by gemm_bf16_tc: B small enough to pin in L2 (evict_last TMA loads)
};

void gemm_f32_simt(const GemmArgs& g, cudaStream_t st);       // fp32 operands, CUDA cores
cudaError_t gemm_bf16_tc(const GemmArgs& g, cudaStream_t st); // bf16 operands, tcgen05 + TMA
int num_sms();

// ------------------------------------------------------------------ attention
// Per (sequence, head): S = q k^T * scale (+ causal mask), P = softmax(S), o = P v
// (O3), saving lse = log-sum-exp of each score row; backward recomputes P from lse
// (O5): dP = dO v^T, dS = P (dP - Dsum), dq = dS k * scale, dk = dS^T q * scale, dv = P^T dO
// with Dsum_i = rowsum(dO_i * o_i).
struct AttnArgs {
  int nseq = 0, seq = 0, heads = 0, dh = 0, d = 0;
  bool causal = true;
  float scale = 1.f;
  const void* qkv = nullptr;  // [nseq*seq][3d]  q | k | v, head h at column h*dh of each
  void* o = nullptr;          // [nseq*seq][d]
  float* lse = nullptr;       // [nseq][heads][seq]
  const void* dO = nullptr;   // [nseq*seq][d]
  float* dsum = nullptr;      // [nseq][heads][seq]
  void* dqkv = nullptr;       // [nseq*seq][3d]
  // backward (tensor-core path): also the column sums of dqkv (the qkv bias gradient) per (sequence, 128-row
  // tile, 32-row quadrant): colsum[((sq * ceil(seq/128) + tile) * 4 + quadrant) * 3d + col], fp32
  float* colsum = nullptr;
  // backward (tensor-core path): optional dS workspace [nseq][heads][s128][s128] bf16 (s128 = seq rounded up to
  // 128): the dK/dV kernel stores dS^T there and dQ becomes a GEMM over it (5 matmuls per block instead of 7)
  void* dsT = nullptr;
};
void attn_fwd_f32(const AttnArgs& a, cudaStream_t st);
void attn_bwd_f32(const AttnArgs& a, cudaStream_t st);
cudaError_t attn_fwd_bf16(const AttnArgs& a, cudaStream_t st);  // tcgen05 + TMA + TMEM (k_attn_tc.cu)
cudaError_t attn_bwd_bf16(const AttnArgs& a, cudaStream_t st);  // tcgen05 (k_attn_tc_bwd.cu)

// ------------------------------------------------------------------ LayerNorm
// y = (x - mu) * rstd * gamma + beta, biased variance (reading A-1).  x fp32 [rows][d];
// y in E; stats[r] = (mu, rstd).
void ln_fwd(const float* x, const void* gamma, const void* beta, DT pdt, void* y, DT ydt,
            float2* stats, int rows, int d, float eps, cudaStream_t st);
// dx = rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat)) + resid, dxhat = dout * gamma (O5);
// writes dx (fp32) and optionally dx_e (E copy), and deterministic column partials
// partial[blk][0][:] = sum dout*xhat, partial[blk][1][:] = sum dout over the block's rows; with `extra` also
// partial[blk][2][:] = sum resid and partial[blk][3][:] = sum dx (the bias gradients that are column sums of
// this kernel's input / output), block stride 4 d instead of 2 d.
// Returns the number of row blocks (partial rows).
int ln_bwd(const float* dout, const float* x, const float2* stats, const void* gamma, DT pdt,
           const float* resid, float* dx, void* dx_e, DT edt, float* partial, int rows, int d,
           cudaStream_t st, bool extra = false);
int ln_bwd_blocks(int rows, int d);

// ------------------------------------------------------------------ column sums (bias grads)
// partial[blk][n] = sum over the block's rows of X[r][n]   (fixed row blocks, deterministic)
int colsum_partial(const void* X, DT xdt, int64_t ldx, int rows, int n, float* partial, cudaStream_t st);
int colsum_blocks(int rows);
// Gradient write modes of the layer's gradient buffers (reading A-3, DESIGN.md "Gradient
// accumulation"): v = sum_k partial[k][n]*ssel (fixed order), then
//   acc_in == nullptr: out[n] = v ; else out[n] = acc_in[n] + v ;  out stored as out_dt.
void colsum_finish(const float* partial, int nblk, int64_t pstride, int n, const float* acc_in,
                   void* out, DT out_dt, cudaStream_t st);
// up to 4 finishes over the same partial rows in one launch: output i sums columns col0 .. col0 + n - 1
struct FinishOut {
  const float* acc_in = nullptr;
  void* out = nullptr;
  DT out_dt = DT::F32;
  int64_t col0 = 0;
};
struct FinishSet {
  FinishOut o[4];
  int k = 0;
};
void colsum_finish_multi(const float* partial, int nblk, int64_t pstride, int n, const FinishSet& fs, cudaStream_t st);

// ------------------------------------------------------------------ loss
// dY = (y - T) / numel_mb; sumsq partial per block (double).  n = total elements.
void mse_fwd_bwd(const float* y, const float* T, float* dY, double* partial, int64_t n,
                 float inv_numel_mb, cudaStream_t st);
int mse_blocks(int64_t n);
// out[0] = 0.5/numel_mb * sum(partial)  (sum over this rank's micro-batches of their losses)
void mse_finish(const double* partial, int nblk, double scale, double* out, cudaStream_t st);

// ------------------------------------------------------------------ AdamW (torch semantics, A-4)
// g = gin[i] * gscale; theta = theta*(1-lr*wd); m,v update; theta -= lr*mhat/(sqrt(vhat)+eps);
// param_out (E) = theta; keep (fp32, optional) = g.
void adamw(const void* gin, DT gdt, float gscale, float* master, float* m, float* v,
           void* param_out, DT pdt, float* keep, int64_t n, float lr, float beta1, float beta2,
           float eps, float wd, const long long* tstep, cudaStream_t st);

// STANDARD schedule: acc[i] = (first ? 0 : acc[i]) + g[i]   (per-micro-batch reduced shard)
void shard_accumulate(const void* g, DT gdt, float* acc, int64_t n, bool first, cudaStream_t st);

// ------------------------------------------------------------------ misc
void cast_f32(const float* x, void* y, DT ydt, int64_t n, cudaStream_t st);
void copy_to_f32(const void* x, DT xdt, float* y, int64_t n, cudaStream_t st);
void fill_f32(float* p, float v, int64_t n, cudaStream_t st);
// Seeded on-device init ("train" recipe): per element normal(0, std) for weights, 1 for LN
// gains, 0 otherwise.  kind[i] is derived from the canonical layout (layer-local offset).
void init_params_device(float* out, int64_t n_layers, int d, int ffn_mult, int L_total,
                        int64_t first_layer, uint64_t seed, cudaStream_t st);
// Spin until *flag >= target (system-scope acquire); used for pipeline receives.
void wait_flag(const volatile unsigned long long* flag, const long long* tstep, unsigned long long per_step,
               unsigned long long k, cudaStream_t st);
// *flag = value (system-scope release) after all prior work on the stream.
void set_flag(unsigned long long* flag, const long long* tstep, unsigned long long per_step, unsigned long long k,
              cudaStream_t st);
void step_begin(long long* tstep, cudaStream_t st);
// reduce-scatter over peer memory fused with AdamW (gbase: device array of the D peers' staging bases)
void adamw_rs(const void* const* gbase, int64_t goff, int D, DT gdt, float gscale, float* master, float* m, float* v,
              void* param_out, DT pdt, float* keep, int64_t n, float lr, float beta1, float beta2, float eps, float wd,
              const long long* tstep, cudaStream_t st);
void dp_signal(unsigned long long* const* fbase, int D, int idx, cudaStream_t st);
// fixed-order fp32 sum of one slice of the D peers' staging buffers: into acc (STANDARD: acc = (first ? 0 : acc)
// + sum) or, acc == nullptr, into out in the staging dtype (unpartitioned all-reduce, reduce-scatter phase)
void peer_reduce(const void* const* gbase, int64_t goff, int D, DT gdt, float* acc, bool first, void* out, int64_t n,
                 cudaStream_t st);
// loss[0] = sum over the world's ranks (rank order) of their loss[0], over peer memory (ring of 4 step slots)
void loss_allreduce_peer(double* loss, double* const* ring, unsigned long long* const* wflag, int rank, int world,
                         const long long* tstep, const unsigned long long* myflag, const double* myring,
                         cudaStream_t st);
// device barrier over peer memory (wflag[q][1] counters), bounded by timeout_ns (*timed_out = 1 on expiry)
void world_barrier(unsigned long long* const* wflag, int world, unsigned long long target,
                   const unsigned long long* myflag, int* timed_out, long long timeout_ns, cudaStream_t st);

}  // namespace lga
