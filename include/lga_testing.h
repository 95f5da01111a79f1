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
                 const float* acc_in, void* aux, int aux_dt, void* out, int64_t ldo, int out_dt, uintptr_t stream);

/* Attention forward / backward on packed qkv [nseq*seq][3d] (head h at column h*dh of q, k, v);
 * path 0 = fp32 SIMT, 1 = bf16 tensor cores.  o, dO: [nseq*seq][d]; lse, dsum: [nseq][heads][seq]. */
int lgatest_attn_fwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv, void* o, float* lse,
                     uintptr_t stream);
int lgatest_attn_bwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv, const void* o,
                     const float* lse, const void* dO, float* dsum, void* dqkv, uintptr_t stream);

#ifdef __cplusplus
}
#endif
#endif
