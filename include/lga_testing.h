/*
 * lga_testing.h -- kernel-level test hooks of liblga.so.  NOT part of the stable ABI (lga.h);
 * used only by tests/ to check single kernels (GEMM epilogues, attention) against a plain
 * PyTorch reference of the same op, and by bench.py for per-kernel roofline timing.
 *
 * All pointers are DEVICE pointers; the call is asynchronous on `stream` and returns a
 * cudaError_t value (0 = success).  Element types: 0 = fp32, 1 = bf16.
 */
#ifndef LGA_TESTING_H_
#define LGA_TESTING_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C[m][n] = sum_k A(m,k) B(n,k) followed by epilogue `kind` (0 store, 1 GELU fwd, 2 GELU bwd);
 * A(m,k) = A[m*lda+k] if a_kmajor else A[k*lda+m]; B(n,k) = B[n*ldb+k] if b_kmajor else
 * B[k*ldb+n].  path 0 = fp32 SIMT (operands fp32), 1 = tcgen05 (operands bf16). */
int lgatest_gemm(int path, int M, int N, int K, const void* A, int64_t lda, int a_kmajor, const void* B,
                 int64_t ldb, int b_kmajor, int kind, const void* bias, int bias_dt, const float* res,
                 const float* acc_in, void* aux, int aux_dt, void* out, int64_t ldo, int out_dt, float* colsum,
                 uintptr_t stream);
/* colsum (path 1, kind 2 = GELU bwd, may be NULL): per 32-row strip column sums of out, ceil(M/32) x N fp32. */

/* lgatest_gemm with a split-K workspace of ws_floats fp32 (device): tile-starved shapes (fewer 128 x 128 tiles
 * than SMs, M % 128 == 0, plain-store epilogue) then run split over K with a fixed-order reduce.  Returns the
 * split count used through *split_used (host int, may be NULL) or a negative cudaError_t. */
int lgatest_gemm_ws(int M, int N, int K, const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                    int b_kmajor, const void* bias, int bias_dt, const float* acc_in, void* out, int64_t ldo,
                    int out_dt, float* ws, int64_t ws_floats, int* split_used, uintptr_t stream);

/* Attention forward / backward on packed qkv [nseq*seq][3d] (head h at column h*dh of q, k, v);
 * path 0 = fp32 SIMT, 1 = bf16 tensor cores (tcgen05).  o, dO: [nseq*seq][d]; lse, dsum: [nseq][heads][seq]. */
int lgatest_attn_fwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv, void* o, float* lse,
                     uintptr_t stream);
int lgatest_attn_bwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv, const void* o,
                     const float* lse, const void* dO, float* dsum, void* dqkv, float* colsum, void* ds_ws,
                     uintptr_t stream);
/* colsum (path 1, may be NULL): column sums of dqkv per (sequence, 128-row tile, 32-row quadrant),
 * [nseq * ceil(seq/128) * 4][3 d] fp32.  ds_ws (path 1, may be NULL): dS workspace of
 * nseq * heads * s128 * s128 bf16 (s128 = seq rounded up to 128) -- dQ from the stored dS (5-matmul backward);
 * NULL = the dQ kernel that recomputes S and dP (7 matmuls). */

/* LayerNorm forward (reading A-1): y = (x - mu) rstd gamma + beta over rows of d; x fp32, gamma / beta in
 * p_dt, y in y_dt, stats[r] = (mu, rstd) as float2. */
int lgatest_ln_fwd(const float* x, const void* gamma, const void* beta, int p_dt, void* y, int y_dt, float* stats,
                   int rows, int d, float eps, uintptr_t stream);
/* LayerNorm backward (O5) as the step runs it: the row kernel(s) write dx (+ resid) (fp32) and optionally dx_e
 * (e_dt), plus deterministic column partials; the fixed-order finisher then writes dgamma = sum dout * xhat and
 * dbeta = sum dout (fp32, d each).  `partial` is scratch of lgatest_ln_bwd_partial_floats(rows, d) floats. */
int lgatest_ln_bwd(const float* dout, const float* x, const float* stats, const void* gamma, int p_dt,
                   const float* resid, float* dx, void* dx_e, int e_dt, float* dgamma, float* dbeta, float* sum_resid,
                   float* sum_dx, float* partial, int rows, int d, uintptr_t stream);
/* sum_resid / sum_dx (may be NULL; either non-NULL selects the 4-sum kernels): column sums of resid and dx. */
int64_t lgatest_ln_bwd_partial_floats(int rows, int d);
/* Bias gradient as the step computes it: out[n] = (acc_in ? acc_in[n] : 0) + sum_r X[r][n] (fixed row
 * blocks, fixed order); X in x_dt with leading dimension ldx; out in out_dt.  `partial` is scratch of
 * lgatest_colsum_partial_floats(rows, n) floats. */
int lgatest_colsum(const void* X, int x_dt, int64_t ldx, int rows, int n, const float* acc_in, void* out, int out_dt,
                   float* partial, uintptr_t stream);
int64_t lgatest_colsum_partial_floats(int rows, int n);
/* Sharded AdamW (torch semantics, reading A-4) on n elements: g = gin * gscale; master / m / v fp32 updated in
 * place; param_out (p_dt) = theta; keep (fp32, optional) = g.  tstep: DEVICE long long, the step t (from 1). */
int lgatest_adamw(const void* gin, int g_dt, float gscale, float* master, float* m, float* v, void* param_out,
                  int p_dt, float* keep, int64_t n, float lr, float beta1, float beta2, float eps, float wd,
                  const long long* tstep, uintptr_t stream);
/* The reduce-scatter fused into AdamW: g = gscale * sum_{p<D} gbase[p][goff + i] in fixed order p = 0..D-1
 * (gbase: DEVICE array of D pointers, g_dt elements), then AdamW as above.  n % 4 == 0. */
int lgatest_adamw_rs(const void* const* gbase, int64_t goff, int D, int g_dt, float gscale, float* master, float* m,
                     float* v, void* param_out, int p_dt, float* keep, int64_t n, float lr, float beta1, float beta2,
                     float eps, float wd, const long long* tstep, uintptr_t stream);
/* Peer-slice reduction: s = sum_{p<D} gbase[p][goff + i] (fixed order); acc != NULL: acc = (first ? 0 : acc) + s
 * (fp32); else out (g_dt) = s.  n % 4 == 0. */
int lgatest_peer_reduce(const void* const* gbase, int64_t goff, int D, int g_dt, float* acc, int first, void* out,
                        int64_t n, uintptr_t stream);

/* Guard-mode arena check (lga_init with env LGA_ARENA_GUARD=1: a 4 KB canary after every arena buffer):
 * the number of canary bytes overwritten so far (an out-of-bounds write past a buffer's end), after
 * synchronising the handle's streams; -1 if the handle is not in guard mode.  `h` is an lga_handle*. */
int64_t lgatest_arena_guard_check(void* h);
/* Negative control: overwrite one byte of the last canary (returns a cudaError_t, -1 if not in guard mode). */
int lgatest_arena_guard_poke(void* h);

#ifdef __cplusplus
}
#endif
#endif
