// test_hooks.cu -- extern "C" wrappers of single kernels for tests/ (include/lga_testing.h).
#include "../../include/lga_testing.h"
#include "kernels.cuh"

#include <cmath>

using namespace lga;

extern "C" int lgatest_gemm(int path, int M, int N, int K, const void* A, int64_t lda, int a_kmajor, const void* B,
                            int64_t ldb, int b_kmajor, int kind, const void* bias, int bias_dt, const float* res,
                            const float* acc_in, void* aux, int aux_dt, void* out, int64_t ldo, int out_dt,
                            float* colsum, uintptr_t stream) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.a_kmajor = a_kmajor != 0;
  g.B = B; g.ldb = ldb; g.b_kmajor = b_kmajor != 0;
  g.epi.kind = kind;
  g.epi.bias = bias; g.epi.bias_dt = (DT)bias_dt;
  g.epi.res = res; g.epi.ldr = ldo;
  g.epi.acc_in = acc_in; g.epi.ldacc = ldo;
  g.epi.aux = aux; g.epi.ldaux = ldo; g.epi.aux_dt = (DT)aux_dt;
  g.epi.out = out; g.epi.ldo = ldo; g.epi.out_dt = (DT)out_dt;
  g.epi.colsum = colsum;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (path == 0) {
    gemm_f32_simt(g, st);
    return (int)cudaGetLastError();
  }
  return (int)gemm_bf16_tc(g, st);
}

namespace lga { namespace tc { int choose_split(const GemmArgs& g, int tiles, int ns); } }

extern "C" int lgatest_gemm_ws(int M, int N, int K, const void* A, int64_t lda, int a_kmajor, const void* B,
                               int64_t ldb, int b_kmajor, const void* bias, int bias_dt, const float* acc_in, void* out,
                               int64_t ldo, int out_dt, float* ws, int64_t ws_floats, int* split_used,
                               uintptr_t stream) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.a_kmajor = a_kmajor != 0;
  g.B = B; g.ldb = ldb; g.b_kmajor = b_kmajor != 0;
  g.epi.bias = bias; g.epi.bias_dt = (DT)bias_dt;
  g.epi.acc_in = acc_in; g.epi.ldacc = ldo;
  g.epi.out = out; g.epi.ldo = ldo; g.epi.out_dt = (DT)out_dt;
  g.splitk_ws = ws;
  g.splitk_ws_floats = ws_floats;
  if (split_used) *split_used = tc::choose_split(g, ((M + 127) / 128) * ((N + 127) / 128), num_sms());
  return (int)gemm_bf16_tc(g, reinterpret_cast<cudaStream_t>(stream));
}

static AttnArgs mk(int nseq, int seq, int heads, int dh, int causal) {
  AttnArgs a;
  a.nseq = nseq; a.seq = seq; a.heads = heads; a.dh = dh; a.d = heads * dh; a.causal = causal != 0;
  a.scale = 1.0f / sqrtf((float)dh);
  return a;
}

extern "C" int lgatest_attn_fwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv, void* o,
                                float* lse, uintptr_t stream) {
  AttnArgs a = mk(nseq, seq, heads, dh, causal);
  a.qkv = qkv; a.o = o; a.lse = lse;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (path == 0) {
    attn_fwd_f32(a, st);
  } else if (path == 1) {
    const cudaError_t e = attn_fwd_bf16(a, st);
    if (e != cudaSuccess) return (int)e;
  } else {
    return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

extern "C" int lgatest_attn_bwd(int path, int nseq, int seq, int heads, int dh, int causal, const void* qkv,
                                const void* o, const float* lse, const void* dO, float* dsum, void* dqkv,
                                float* colsum, void* ds_ws, uintptr_t stream) {
  AttnArgs a = mk(nseq, seq, heads, dh, causal);
  a.qkv = qkv; a.o = (void*)o; a.lse = (float*)lse; a.dO = dO; a.dsum = dsum; a.dqkv = dqkv;
  a.colsum = colsum;
  a.dsT = ds_ws;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (path == 0) {
    attn_bwd_f32(a, st);
  } else if (path == 1) {
    const cudaError_t e = attn_bwd_bf16(a, st);
    if (e != cudaSuccess) return (int)e;
  } else {
    return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

extern "C" int lgatest_ln_fwd(const float* x, const void* gamma, const void* beta, int p_dt, void* y, int y_dt,
                              float* stats, int rows, int d, float eps, uintptr_t stream) {
  ln_fwd(x, gamma, beta, (DT)p_dt, y, (DT)y_dt, reinterpret_cast<float2*>(stats), rows, d, eps,
         reinterpret_cast<cudaStream_t>(stream));
  return (int)cudaGetLastError();
}

extern "C" int64_t lgatest_ln_bwd_partial_floats(int rows, int d) { return (int64_t)ln_bwd_blocks(rows, d) * 2 * d; }

extern "C" int lgatest_ln_bwd(const float* dout, const float* x, const float* stats, const void* gamma, int p_dt,
                              const float* resid, float* dx, void* dx_e, int e_dt, float* dgamma, float* dbeta,
                              float* sum_resid, float* sum_dx, float* partial, int rows, int d, uintptr_t stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool extra = sum_resid || sum_dx;
  const int nblk = ln_bwd(dout, x, reinterpret_cast<const float2*>(stats), gamma, (DT)p_dt, resid, dx, dx_e, (DT)e_dt,
                          partial, rows, d, st, extra);
  const int64_t ps = (extra ? 4LL : 2LL) * d;
  float* outs[4] = {dgamma, dbeta, sum_resid, sum_dx};
  FinishSet fs;   // one multi-output finish launch, as the step does
  for (int k = 0; k < (extra ? 4 : 2); ++k)
    if (outs[k]) fs.o[fs.k++] = FinishOut{nullptr, outs[k], DT::F32, (int64_t)k * d};
  colsum_finish_multi(partial, nblk, ps, d, fs, st);
  return (int)cudaGetLastError();
}

extern "C" int64_t lgatest_colsum_partial_floats(int rows, int n) { return (int64_t)colsum_blocks(rows) * n; }

extern "C" int lgatest_colsum(const void* X, int x_dt, int64_t ldx, int rows, int n, const float* acc_in, void* out,
                              int out_dt, float* partial, uintptr_t stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int nblk = colsum_partial(X, (DT)x_dt, ldx, rows, n, partial, st);
  colsum_finish(partial, nblk, n, n, acc_in, out, (DT)out_dt, st);
  return (int)cudaGetLastError();
}

extern "C" int lgatest_adamw(const void* gin, int g_dt, float gscale, float* master, float* m, float* v,
                             void* param_out, int p_dt, float* keep, int64_t n, float lr, float beta1, float beta2,
                             float eps, float wd, const long long* tstep, uintptr_t stream) {
  adamw(gin, (DT)g_dt, gscale, master, m, v, param_out, (DT)p_dt, keep, n, lr, beta1, beta2, eps, wd, tstep,
        reinterpret_cast<cudaStream_t>(stream));
  return (int)cudaGetLastError();
}

extern "C" int lgatest_adamw_rs(const void* const* gbase, int64_t goff, int D, int g_dt, float gscale, float* master,
                                float* m, float* v, void* param_out, int p_dt, float* keep, int64_t n, float lr,
                                float beta1, float beta2, float eps, float wd, const long long* tstep,
                                uintptr_t stream) {
  adamw_rs(gbase, goff, D, (DT)g_dt, gscale, master, m, v, param_out, (DT)p_dt, keep, n, lr, beta1, beta2, eps, wd,
           tstep, reinterpret_cast<cudaStream_t>(stream));
  return (int)cudaGetLastError();
}

extern "C" int lgatest_peer_reduce(const void* const* gbase, int64_t goff, int D, int g_dt, float* acc, int first,
                                   void* out, int64_t n, uintptr_t stream) {
  peer_reduce(gbase, goff, D, (DT)g_dt, acc, first != 0, out, n, reinterpret_cast<cudaStream_t>(stream));
  return (int)cudaGetLastError();
}
