// k_gemm_simt.cu -- fp32 register-tiled GEMM on the CUDA cores (parity mode, LGA_FP32).
// Correctness path: the same operand majors and fused epilogues as the tcgen05 GEMM, in fp32 FFMA.
#include "epilogue.cuh"

namespace lga {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgs g) {
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;
  const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
  const float* A = static_cast<const float*>(g.A);
  const float* B = static_cast<const float*>(g.B);
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += SB_K) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * 256;
      int mm, kk;
      if (g.a_kmajor) { mm = idx / SB_K; kk = idx % SB_K; } else { mm = idx % SB_M; kk = idx / SB_M; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < g.M && gk < g.K) v = g.a_kmajor ? A[(int64_t)gm * g.lda + gk] : A[(int64_t)gk * g.lda + gm];
      As[kk][mm] = v;
      int nn;
      if (g.b_kmajor) { nn = idx / SB_K; kk = idx % SB_K; } else { nn = idx % SB_N; kk = idx / SB_N; }
      const int gn = n0 + nn;
      const int gk2 = k0 + kk;
      float w = 0.f;
      if (gn < g.N && gk2 < g.K) w = g.b_kmajor ? B[(int64_t)gn * g.ldb + gk2] : B[(int64_t)gk2 * g.ldb + gn];
      Bs[kk][nn] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][tm + i]; b[i] = Bs[kk][tn + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + tm + i, gn = n0 + tn + j;
      if (gm < g.M && gn < g.N) epi_store(g.epi, gm, gn, acc[i][j]);
    }
}

void gemm_f32_simt(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  dim3 grid((g.N + SB_N - 1) / SB_N, (g.M + SB_M - 1) / SB_M);
  note_launch(), gemm_f32_kernel<<<grid, 256, 0, st>>>(g);
}

}  // namespace lga
