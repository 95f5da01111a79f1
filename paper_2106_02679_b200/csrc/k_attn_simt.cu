// k_attn_simt.cu -- fp32 multi-head self-attention forward/backward on the CUDA cores
// (parity mode, any head size <= 128).  Flash-style: online softmax in the forward pass, the
// log-sum-exp saved per query row, P recomputed from it in the backward pass (O3, O5);
// dq and dk/dv in separate passes so that no float atomics are needed.
#include "kernels.cuh"

#include <cmath>

namespace lga {

constexpr int AQ = 64;   // queries (or keys) per block, one per thread
constexpr int AK = 32;   // rows of the staged K/V (or Q/dO) tile

template <int DHM>
__global__ void __launch_bounds__(AQ) attn_fwd_f32_kernel(AttnArgs a) {
  __shared__ float Ks[AK][DHM], Vs[AK][DHM];
  const int sq = blockIdx.z, h = blockIdx.y, i = blockIdx.x * AQ + threadIdx.x;
  const int s = a.seq, dh = a.dh, d = a.d;
  const int64_t ld = 3LL * d;
  const float* qkv = static_cast<const float*>(a.qkv) + (int64_t)sq * s * ld;
  float q[DHM], o[DHM];
#pragma unroll
  for (int c = 0; c < DHM; ++c) {
    q[c] = (i < s && c < dh) ? qkv[(int64_t)i * ld + h * dh + c] : 0.f;
    o[c] = 0.f;
  }
  float mx = -INFINITY, l = 0.f;
  const int kend = a.causal ? min(s, (int)(blockIdx.x + 1) * AQ) : s;
  for (int kt = 0; kt < kend; kt += AK) {
    for (int e = threadIdx.x; e < AK * DHM; e += AQ) {
      const int r = e / DHM, c = e % DHM, j = kt + r;
      const bool ok = j < s && c < dh;
      Ks[r][c] = ok ? qkv[(int64_t)j * ld + d + h * dh + c] : 0.f;
      Vs[r][c] = ok ? qkv[(int64_t)j * ld + 2 * d + h * dh + c] : 0.f;
    }
    __syncthreads();
    if (i < s) {
      for (int r = 0; r < AK; ++r) {
        const int j = kt + r;
        if (j >= s || (a.causal && j > i)) break;
        float sc = 0.f;
#pragma unroll
        for (int c = 0; c < DHM; ++c) sc = fmaf(q[c], Ks[r][c], sc);
        sc *= a.scale;
        if (sc > mx) {
          const float corr = expf(mx - sc);
          l *= corr;
#pragma unroll
          for (int c = 0; c < DHM; ++c) o[c] *= corr;
          mx = sc;
        }
        const float p = expf(sc - mx);
        l += p;
#pragma unroll
        for (int c = 0; c < DHM; ++c) o[c] = fmaf(p, Vs[r][c], o[c]);
      }
    }
    __syncthreads();
  }
  if (i < s) {
    float* out = static_cast<float*>(a.o) + (int64_t)sq * s * d + (int64_t)i * d + h * dh;
    const float inv = 1.f / l;
    for (int c = 0; c < dh; ++c) out[c] = o[c] * inv;
    a.lse[((int64_t)sq * a.heads + h) * s + i] = mx + logf(l);
  }
}

__global__ void attn_dsum_kernel(AttnArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // over nseq*heads*seq
  const int64_t total = (int64_t)a.nseq * a.heads * a.seq;
  if (t >= total) return;
  const int i = (int)(t % a.seq);
  const int h = (int)((t / a.seq) % a.heads);
  const int64_t sq = t / ((int64_t)a.seq * a.heads);
  const int64_t row = (sq * a.seq + i) * a.d + (int64_t)h * a.dh;
  float s = 0.f;
  for (int c = 0; c < a.dh; ++c)
    s = fmaf(ld_elem(a.dO, row + c, DT::F32), ld_elem(a.o, row + c, DT::F32), s);
  a.dsum[t] = s;
}

template <int DHM>
__global__ void __launch_bounds__(AQ) attn_dq_f32_kernel(AttnArgs a) {
  __shared__ float Ks[AK][DHM], Vs[AK][DHM];
  const int sq = blockIdx.z, h = blockIdx.y, i = blockIdx.x * AQ + threadIdx.x;
  const int s = a.seq, dh = a.dh, d = a.d;
  const int64_t ld = 3LL * d;
  const float* qkv = static_cast<const float*>(a.qkv) + (int64_t)sq * s * ld;
  const float* dO = static_cast<const float*>(a.dO) + (int64_t)sq * s * d;
  float q[DHM], g[DHM], dq[DHM];
#pragma unroll
  for (int c = 0; c < DHM; ++c) {
    q[c] = (i < s && c < dh) ? qkv[(int64_t)i * ld + h * dh + c] : 0.f;
    g[c] = (i < s && c < dh) ? dO[(int64_t)i * d + h * dh + c] : 0.f;
    dq[c] = 0.f;
  }
  const int64_t ri = ((int64_t)sq * a.heads + h) * s + i;
  const float lse = i < s ? a.lse[ri] : 0.f, Di = i < s ? a.dsum[ri] : 0.f;
  const int kend = a.causal ? min(s, (int)(blockIdx.x + 1) * AQ) : s;
  for (int kt = 0; kt < kend; kt += AK) {
    for (int e = threadIdx.x; e < AK * DHM; e += AQ) {
      const int r = e / DHM, c = e % DHM, j = kt + r;
      const bool ok = j < s && c < dh;
      Ks[r][c] = ok ? qkv[(int64_t)j * ld + d + h * dh + c] : 0.f;
      Vs[r][c] = ok ? qkv[(int64_t)j * ld + 2 * d + h * dh + c] : 0.f;
    }
    __syncthreads();
    if (i < s) {
      for (int r = 0; r < AK; ++r) {
        const int j = kt + r;
        if (j >= s || (a.causal && j > i)) break;
        float sc = 0.f, dp = 0.f;
#pragma unroll
        for (int c = 0; c < DHM; ++c) { sc = fmaf(q[c], Ks[r][c], sc); dp = fmaf(g[c], Vs[r][c], dp); }
        const float p = expf(sc * a.scale - lse);
        const float ds = p * (dp - Di) * a.scale;
#pragma unroll
        for (int c = 0; c < DHM; ++c) dq[c] = fmaf(ds, Ks[r][c], dq[c]);
      }
    }
    __syncthreads();
  }
  if (i < s) {
    float* out = static_cast<float*>(a.dqkv) + (int64_t)sq * s * ld + (int64_t)i * ld + h * dh;
    for (int c = 0; c < dh; ++c) out[c] = dq[c];
  }
}

template <int DHM>
__global__ void __launch_bounds__(AQ) attn_dkdv_f32_kernel(AttnArgs a) {
  __shared__ float Qs[AK][DHM], Gs[AK][DHM], Ls[AK], Ds[AK];
  const int sq = blockIdx.z, h = blockIdx.y, j = blockIdx.x * AQ + threadIdx.x;
  const int s = a.seq, dh = a.dh, d = a.d;
  const int64_t ld = 3LL * d;
  const float* qkv = static_cast<const float*>(a.qkv) + (int64_t)sq * s * ld;
  const float* dO = static_cast<const float*>(a.dO) + (int64_t)sq * s * d;
  float k[DHM], v[DHM], dk[DHM], dv[DHM];
#pragma unroll
  for (int c = 0; c < DHM; ++c) {
    k[c] = (j < s && c < dh) ? qkv[(int64_t)j * ld + d + h * dh + c] : 0.f;
    v[c] = (j < s && c < dh) ? qkv[(int64_t)j * ld + 2 * d + h * dh + c] : 0.f;
    dk[c] = 0.f; dv[c] = 0.f;
  }
  const int64_t rbase = ((int64_t)sq * a.heads + h) * s;
  const int qstart = a.causal ? (int)blockIdx.x * AQ : 0;
  for (int qt = qstart; qt < s; qt += AK) {
    for (int e = threadIdx.x; e < AK * DHM; e += AQ) {
      const int r = e / DHM, c = e % DHM, i = qt + r;
      const bool ok = i < s && c < dh;
      Qs[r][c] = ok ? qkv[(int64_t)i * ld + h * dh + c] : 0.f;
      Gs[r][c] = ok ? dO[(int64_t)i * d + h * dh + c] : 0.f;
    }
    for (int r = threadIdx.x; r < AK; r += AQ) {
      const int i = qt + r;
      Ls[r] = i < s ? a.lse[rbase + i] : 0.f;
      Ds[r] = i < s ? a.dsum[rbase + i] : 0.f;
    }
    __syncthreads();
    if (j < s) {
      for (int r = 0; r < AK; ++r) {
        const int i = qt + r;
        if (i >= s) break;
        if (a.causal && i < j) continue;
        float sc = 0.f, dp = 0.f;
#pragma unroll
        for (int c = 0; c < DHM; ++c) { sc = fmaf(Qs[r][c], k[c], sc); dp = fmaf(Gs[r][c], v[c], dp); }
        const float p = expf(sc * a.scale - Ls[r]);
        const float ds = p * (dp - Ds[r]) * a.scale;
#pragma unroll
        for (int c = 0; c < DHM; ++c) { dv[c] = fmaf(p, Gs[r][c], dv[c]); dk[c] = fmaf(ds, Qs[r][c], dk[c]); }
      }
    }
    __syncthreads();
  }
  if (j < s) {
    float* out = static_cast<float*>(a.dqkv) + (int64_t)sq * s * ld + (int64_t)j * ld + h * dh;
    for (int c = 0; c < dh; ++c) { out[d + c] = dk[c]; out[2 * d + c] = dv[c]; }
  }
}

#define ATTN_DISPATCH(KERNEL, grid)                                                     \
  do {                                                                                  \
    if (a.dh <= 16) note_launch(), KERNEL<16><<<grid, AQ, 0, st>>>(a);                                 \
    else if (a.dh <= 32) note_launch(), KERNEL<32><<<grid, AQ, 0, st>>>(a);                            \
    else if (a.dh <= 64) note_launch(), KERNEL<64><<<grid, AQ, 0, st>>>(a);                            \
    else note_launch(), KERNEL<128><<<grid, AQ, 0, st>>>(a);                                           \
  } while (0)

void attn_fwd_f32(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return;
  dim3 grid((a.seq + AQ - 1) / AQ, a.heads, a.nseq);
  ATTN_DISPATCH(attn_fwd_f32_kernel, grid);
}

void attn_bwd_f32(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return;
  const int64_t rows = (int64_t)a.nseq * a.heads * a.seq;
  note_launch(), attn_dsum_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(a);
  dim3 grid((a.seq + AQ - 1) / AQ, a.heads, a.nseq);
  ATTN_DISPATCH(attn_dq_f32_kernel, grid);
  ATTN_DISPATCH(attn_dkdv_f32_kernel, grid);
}

}  // namespace lga
