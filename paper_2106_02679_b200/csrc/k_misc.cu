// k_misc.cu -- HBM-bound kernels of the LGA step: LayerNorm fwd/bwd, column sums for the
// bias / LayerNorm gradients, MSE loss + seed gradient, sharded AdamW, casts, seeded init,
// pipeline flags.  Every reduction runs in a fixed order (no float atomics), so a step is
// bitwise reproducible.
#include "kernels.cuh"

#include <atomic>
#include <cmath>

namespace lga {

// =============================================================== column sums
constexpr int COLSUM_ROWS = 64;
int colsum_blocks(int rows) { return (rows + COLSUM_ROWS - 1) / COLSUM_ROWS; }

__global__ void colsum_partial_kernel(const void* __restrict__ X, DT xdt, int64_t ldx, int rows, int n,
                                      float* __restrict__ partial) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int r0 = blockIdx.y * COLSUM_ROWS, r1 = min(rows, r0 + COLSUM_ROWS);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += ld_elem(X, (int64_t)r * ldx + c, xdt);
  partial[(int64_t)blockIdx.y * n + c] = s;
}

// 16-byte loads: V = 4 fp32 or 8 bf16 columns per thread (n, ldx multiples of V, 16-byte aligned rows);
// each column is still summed over rows r0, r0+1, ... in order (bitwise equal to the scalar kernel)
template <bool BF16>
__global__ void __launch_bounds__(256) colsum_partial_vec(const void* __restrict__ X, int64_t ldx, int rows, int n,
                                                          float* __restrict__ partial) {
  constexpr int V = BF16 ? 8 : 4;
  const int c = (blockIdx.x * 256 + threadIdx.x) * V;
  if (c >= n) return;
  const int r0 = blockIdx.y * COLSUM_ROWS, r1 = min(rows, r0 + COLSUM_ROWS);
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll 8
  for (int r = r0; r < r1; ++r) {
    if (BF16) {
      const uint4 u = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(X) + (int64_t)r * ldx + c);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        acc[2 * i] += __uint_as_float(w[i] << 16);
        acc[2 * i + 1] += __uint_as_float(w[i] & 0xFFFF0000u);
      }
    } else {
      const float4 v = *reinterpret_cast<const float4*>(static_cast<const float*>(X) + (int64_t)r * ldx + c);
      acc[0] += v.x, acc[1] += v.y, acc[2] += v.z, acc[3] += v.w;
    }
  }
  float* out = partial + (int64_t)blockIdx.y * n + c;
#pragma unroll
  for (int i = 0; i < V; i += 4) *reinterpret_cast<float4*>(out + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
}

int colsum_partial(const void* X, DT xdt, int64_t ldx, int rows, int n, float* partial, cudaStream_t st) {
  const int nblk = colsum_blocks(rows);
  if (rows <= 0 || n <= 0) return 0;
  const bool bf = xdt == DT::BF16;
  const int V = bf ? 8 : (xdt == DT::F32 ? 4 : 0);
  if (V && n % V == 0 && ldx % V == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    dim3 grid((n / V + 255) / 256, nblk);
    if (bf) note_launch(), colsum_partial_vec<true><<<grid, 256, 0, st>>>(X, ldx, rows, n, partial);
    else note_launch(), colsum_partial_vec<false><<<grid, 256, 0, st>>>(X, ldx, rows, n, partial);
    return nblk;
  }
  dim3 grid((n + 255) / 256, nblk);
  note_launch(), colsum_partial_kernel<<<grid, 256, 0, st>>>(X, xdt, ldx, rows, n, partial);
  return nblk;
}

// =============================================================== MSE loss + seed gradient
constexpr int MSE_THREADS = 256;
constexpr int MSE_PER_THREAD = 16;
int mse_blocks(int64_t n) { return (int)((n + MSE_THREADS * MSE_PER_THREAD - 1) / (MSE_THREADS * MSE_PER_THREAD)); }

__global__ void __launch_bounds__(MSE_THREADS) mse_kernel(const float* __restrict__ y, const float* __restrict__ T,
                                                          float* __restrict__ dY, double* __restrict__ partial,
                                                          int64_t n, float inv_numel) {
  __shared__ double red[32];
  const int64_t base = (int64_t)blockIdx.x * MSE_THREADS * MSE_PER_THREAD + threadIdx.x;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < MSE_PER_THREAD; ++i) {
    const int64_t k = base + (int64_t)i * MSE_THREADS;
    if (k < n) {
      const float diff = y[k] - T[k];
      dY[k] = diff * inv_numel;
      s += (double)diff * (double)diff;
    }
  }
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < MSE_THREADS / 32; ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

void mse_fwd_bwd(const float* y, const float* T, float* dY, double* partial, int64_t n,
                 float inv_numel_mb, cudaStream_t st) {
  if (n <= 0) return;
  note_launch(), mse_kernel<<<mse_blocks(n), MSE_THREADS, 0, st>>>(y, T, dY, partial, n, inv_numel_mb);
}

__global__ void mse_finish_kernel(const double* partial, int nblk, double scale, double* out) {
  double s = 0.0;
  for (int k = threadIdx.x; k < nblk; k += 32) s += partial[k];
  s = warp_sum_d(s);
  if (threadIdx.x == 0) out[0] = s * scale;
}

void mse_finish(const double* partial, int nblk, double scale, double* out, cudaStream_t st) {
  note_launch(), mse_finish_kernel<<<1, 32, 0, st>>>(partial, nblk, scale, out);
}

// =============================================================== AdamW
template <typename GE, typename PE>
__device__ __forceinline__ void adamw_one(const GE* gin, float gscale, float* master, float* m, float* v, PE* pout,
                                          float* keep, int64_t i, float lr, float b1, float b2, float eps, float wd,
                                          float bc1, float bc2) {
  const float g = to_f(gin[i]) * gscale;
  float th = master[i] * (1.0f - lr * wd);
  const float mi = b1 * m[i] + (1.0f - b1) * g;
  const float vi = b2 * v[i] + (1.0f - b2) * g * g;
  m[i] = mi;
  v[i] = vi;
  th = th - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  master[i] = th;
  pout[i] = from_f<PE>(th);
  if (keep) keep[i] = g;
}

// 4 elements per thread per iteration with 128-bit loads / stores (n % 4 tail handled element-wise)
template <typename GE, typename PE>
__global__ void __launch_bounds__(256) adamw_kernel(const GE* __restrict__ gin, float gscale, float* __restrict__ master,
                                                    float* __restrict__ m, float* __restrict__ v, PE* __restrict__ pout,
                                                    float* __restrict__ keep, int64_t n, float lr, float b1, float b2,
                                                    float eps, float wd, const long long* __restrict__ tstep) {
  // bias corrections of step t (from 1), read on the device so that a captured step graph replays them
  const float t = (float)*tstep;
  const float bc1 = 1.0f - powf(b1, t), bc2 = 1.0f - powf(b2, t);
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float g[4];
    if (sizeof(GE) == 4) {
      const float4 t = reinterpret_cast<const float4*>(gin)[i];
      g[0] = t.x; g[1] = t.y; g[2] = t.z; g[3] = t.w;
    } else {
      const uint2 t = reinterpret_cast<const uint2*>(gin)[i];
      g[0] = __uint_as_float(t.x << 16); g[1] = __uint_as_float(t.x & 0xFFFF0000u);
      g[2] = __uint_as_float(t.y << 16); g[3] = __uint_as_float(t.y & 0xFFFF0000u);
    }
    float4 th = reinterpret_cast<float4*>(master)[i];
    float4 mi = reinterpret_cast<float4*>(m)[i];
    float4 vi = reinterpret_cast<float4*>(v)[i];
    float* thp = &th.x;
    float* mp = &mi.x;
    float* vp = &vi.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = g[e] * gscale;
      g[e] = gg;
      float t = thp[e] * (1.0f - lr * wd);
      mp[e] = b1 * mp[e] + (1.0f - b1) * gg;
      vp[e] = b2 * vp[e] + (1.0f - b2) * gg * gg;
      thp[e] = t - lr * (mp[e] / bc1) / (sqrtf(vp[e] / bc2) + eps);
    }
    reinterpret_cast<float4*>(master)[i] = th;
    reinterpret_cast<float4*>(m)[i] = mi;
    reinterpret_cast<float4*>(v)[i] = vi;
    if (sizeof(PE) == 4) {
      reinterpret_cast<float4*>(pout)[i] = th;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(th.x, th.y), hi = __floats2bfloat162_rn(th.z, th.w);
      reinterpret_cast<uint2*>(pout)[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
    if (keep) reinterpret_cast<float4*>(keep)[i] = make_float4(g[0], g[1], g[2], g[3]);
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    adamw_one(gin, gscale, master, m, v, pout, keep, i, lr, b1, b2, eps, wd, bc1, bc2);
}

// Reduce-scatter fused with AdamW over NVLink peer memory: this rank's shard of the layer
// gradient is the sum, in fixed rank order p = 0..D-1, of the same slice of every data-parallel peer's
// staging buffer (gbase[p] + goff, read uncached: written by the peer since the last step); then AdamW as
// above.  n % 4 == 0 (shards are multiples of 64 elements).
template <typename GE>
__device__ __forceinline__ void ld4_cv(const GE* p, int64_t i, float (&g)[4]) {
  if (sizeof(GE) == 4) {
    float4 t;
    asm volatile("ld.global.cv.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w)
                 : "l"(reinterpret_cast<const float4*>(p) + i));
    g[0] = t.x, g[1] = t.y, g[2] = t.z, g[3] = t.w;
  } else {
    uint32_t a, b;
    asm volatile("ld.global.cv.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "l"(reinterpret_cast<const uint2*>(p) + i));
    g[0] = __uint_as_float(a << 16), g[1] = __uint_as_float(a & 0xFFFF0000u);
    g[2] = __uint_as_float(b << 16), g[3] = __uint_as_float(b & 0xFFFF0000u);
  }
}

template <typename GE, typename PE>
__global__ void __launch_bounds__(256) adamw_rs_kernel(const void* const* __restrict__ gbase, int64_t goff, int D,
                                                       float gscale, float* __restrict__ master, float* __restrict__ m,
                                                       float* __restrict__ v, PE* __restrict__ pout,
                                                       float* __restrict__ keep, int64_t n, float lr, float b1,
                                                       float b2, float eps, float wd, const long long* __restrict__ tstep) {
  const float t = (float)*tstep;
  const float bc1 = 1.0f - powf(b1, t), bc2 = 1.0f - powf(b2, t);
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    for (int p = 0; p < D; ++p) {   // fixed rank order: bitwise reproducible
      float q[4];
      ld4_cv(static_cast<const GE*>(gbase[p]) + goff, i, q);
      g[0] += q[0], g[1] += q[1], g[2] += q[2], g[3] += q[3];
    }
    float4 th = reinterpret_cast<float4*>(master)[i];
    float4 mi = reinterpret_cast<float4*>(m)[i];
    float4 vi = reinterpret_cast<float4*>(v)[i];
    float* thp = &th.x;
    float* mp = &mi.x;
    float* vp = &vi.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gg = g[e] * gscale;
      g[e] = gg;
      float tt = thp[e] * (1.0f - lr * wd);
      mp[e] = b1 * mp[e] + (1.0f - b1) * gg;
      vp[e] = b2 * vp[e] + (1.0f - b2) * gg * gg;
      thp[e] = tt - lr * (mp[e] / bc1) / (sqrtf(vp[e] / bc2) + eps);
    }
    reinterpret_cast<float4*>(master)[i] = th;
    reinterpret_cast<float4*>(m)[i] = mi;
    reinterpret_cast<float4*>(v)[i] = vi;
    if (sizeof(PE) == 4) {
      reinterpret_cast<float4*>(pout)[i] = th;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(th.x, th.y), hi = __floats2bfloat162_rn(th.z, th.w);
      reinterpret_cast<uint2*>(pout)[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
    if (keep) reinterpret_cast<float4*>(keep)[i] = make_float4(g[0], g[1], g[2], g[3]);
  }
}

void adamw_rs(const void* const* gbase, int64_t goff, int D, DT gdt, float gscale, float* master, float* m, float* v,
              void* param_out, DT pdt, float* keep, int64_t n, float lr, float beta1, float beta2, float eps, float wd,
              const long long* tstep, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, (int64_t)num_sms() * 8);
#define AR(GE, PE) note_launch(), adamw_rs_kernel<GE, PE><<<grid, 256, 0, st>>>(gbase, goff, D, gscale, master, m, v, (PE*)param_out, keep, n, lr, beta1, beta2, eps, wd, tstep)
  if (gdt == DT::F32 && pdt == DT::F32) AR(float, float);
  else if (gdt == DT::F32) AR(float, __nv_bfloat16);
  else if (pdt == DT::F32) AR(__nv_bfloat16, float);
  else AR(__nv_bfloat16, __nv_bfloat16);
#undef AR
}

// Peer-memory reduction of one slice (fixed rank order p = 0..D-1, fp32 sum of the D peers' staging at
// gbase[p] + goff, read uncached).  acc != nullptr (STANDARD): acc[i] = (first ? 0 : acc[i]) + sum, the
// per-micro-batch reduced shard accumulated in fp32.  Otherwise (unpartitioned all-reduce, phase 1 = the
// reduce-scatter): out[i] = sum in the staging dtype (out is this rank's own slice; it is read by no
// peer during this phase, so the in-place write is race-free).  n % 4 == 0.
template <typename GE>
__global__ void __launch_bounds__(256) peer_reduce_kernel(const void* const* __restrict__ gbase, int64_t goff, int D,
                                                          float* __restrict__ acc, bool first, GE* __restrict__ out,
                                                          int64_t n) {
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    for (int p = 0; p < D; ++p) {
      float q[4];
      ld4_cv(static_cast<const GE*>(gbase[p]) + goff, i, q);
      g[0] += q[0], g[1] += q[1], g[2] += q[2], g[3] += q[3];
    }
    if (acc) {
      float4 a = first ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<float4*>(acc)[i];
      a.x += g[0], a.y += g[1], a.z += g[2], a.w += g[3];
      reinterpret_cast<float4*>(acc)[i] = a;
    } else if (sizeof(GE) == 4) {
      reinterpret_cast<float4*>(out)[i] = make_float4(g[0], g[1], g[2], g[3]);
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(g[0], g[1]), hi = __floats2bfloat162_rn(g[2], g[3]);
      reinterpret_cast<uint2*>(out)[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
}

void peer_reduce(const void* const* gbase, int64_t goff, int D, DT gdt, float* acc, bool first, void* out, int64_t n,
                 cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, (int64_t)num_sms() * 8);
  if (gdt == DT::F32)
    note_launch(), peer_reduce_kernel<float><<<grid, 256, 0, st>>>(gbase, goff, D, acc, first, (float*)out, n);
  else
    note_launch(), peer_reduce_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(gbase, goff, D, acc, first,
                                                                           (__nv_bfloat16*)out, n);
}

void adamw(const void* gin, DT gdt, float gscale, float* master, float* m, float* v,
           void* param_out, DT pdt, float* keep, int64_t n, float lr, float beta1, float beta2,
           float eps, float wd, const long long* tstep, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, (int64_t)num_sms() * 8);
#define AD(GE, PE) note_launch(), adamw_kernel<GE, PE><<<grid, 256, 0, st>>>((const GE*)gin, gscale, master, m, v, (PE*)param_out, keep, n, lr, beta1, beta2, eps, wd, tstep)
  if (gdt == DT::F32 && pdt == DT::F32) AD(float, float);
  else if (gdt == DT::F32) AD(float, __nv_bfloat16);
  else if (pdt == DT::F32) AD(__nv_bfloat16, float);
  else AD(__nv_bfloat16, __nv_bfloat16);
#undef AD
}

__global__ void shard_acc_kernel(const void* g, DT gdt, float* acc, int64_t n, bool first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] = (first ? 0.f : acc[i]) + ld_elem(g, i, gdt);
}
void shard_accumulate(const void* g, DT gdt, float* acc, int64_t n, bool first, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), shard_acc_kernel<<<grid, 256, 0, st>>>(g, gdt, acc, n, first);
}

// =============================================================== casts / fills
__global__ void cast_kernel(const float* __restrict__ x, void* y, DT ydt, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    st_elem(y, i, ydt, x[i]);
}
void cast_f32(const float* x, void* y, DT ydt, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), cast_kernel<<<grid, 256, 0, st>>>(x, y, ydt, n);
}
__global__ void to_f32_kernel(const void* x, DT xdt, float* y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = ld_elem(x, i, xdt);
}
void copy_to_f32(const void* x, DT xdt, float* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), to_f32_kernel<<<grid, 256, 0, st>>>(x, xdt, y, n);
}
__global__ void fill_kernel(float* p, float v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}
void fill_f32(float* p, float v, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), fill_kernel<<<grid, 256, 0, st>>>(p, v, n);
}

// =============================================================== seeded device init
// splitmix64 counter hash -> two uniforms -> Box-Muller normal.  Kind by canonical offset.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void init_kernel(float* out, int64_t n, int64_t pl, int d, int f, int L_total, int64_t first_layer,
                            uint64_t seed) {
  // canonical offsets
  const int64_t o_ln1w = 0, o_ln1b = d, o_wqkv = 2 * d, o_bqkv = o_wqkv + 3LL * d * d, o_wo = o_bqkv + 3 * d,
                o_bo = o_wo + (int64_t)d * d, o_ln2w = o_bo + d, o_ln2b = o_ln2w + d, o_w1 = o_ln2b + d,
                o_b1 = o_w1 + (int64_t)d * f, o_w2 = o_b1 + f, o_b2 = o_w2 + (int64_t)f * d;
  const float std_w = 0.02f, std_r = 0.02f / sqrtf(2.0f * L_total);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t off = i % pl;
    const int64_t gidx = first_layer * pl + i;
    float val;
    if ((off >= o_wqkv && off < o_bqkv) || (off >= o_w1 && off < o_b1) || (off >= o_wo && off < o_bo) ||
        (off >= o_w2 && off < o_b2)) {
      const uint64_t h = splitmix64(seed ^ splitmix64((uint64_t)gidx));
      const float u1 = ((h >> 40) + 1.0f) * (1.0f / 16777217.0f);
      const float u2 = ((h & 0xffffffull) + 0.5f) * (1.0f / 16777216.0f);
      const float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
      const bool resid = (off >= o_wo && off < o_bo) || (off >= o_w2 && off < o_b2);
      val = z * (resid ? std_r : std_w);
    } else if ((off >= o_ln1w && off < o_ln1b) || (off >= o_ln2w && off < o_ln2b)) {
      val = 1.0f;
    } else {
      val = 0.0f;
    }
    out[i] = val;
  }
}

void init_params_device(float* out, int64_t n_layers, int d, int ffn_mult, int L_total, int64_t first_layer,
                        uint64_t seed, cudaStream_t st) {
  const int64_t f = (int64_t)ffn_mult * d;
  const int64_t pl = (4 + 2LL * ffn_mult) * d * d + 13LL * d;
  const int64_t n = n_layers * pl;
  if (n <= 0) return;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 16);
  note_launch(), init_kernel<<<grid, 256, 0, st>>>(out, n, pl, d, (int)f, L_total, first_layer, seed);
}

// =============================================================== pipeline flags
// Pipeline flags count transfers since lga_init.  Targets are (t - 1) * per_step + k with t the device
// step counter, so a captured step graph waits for / publishes the right values on every replay.
__global__ void wait_flag_kernel(const volatile unsigned long long* flag, const long long* tstep,
                                 unsigned long long per_step, unsigned long long k) {
  const unsigned long long target = (unsigned long long)(*tstep - 1) * per_step + k;
  unsigned long long v;
  while (true) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    __nanosleep(200);
  }
}
void wait_flag(const volatile unsigned long long* flag, const long long* tstep, unsigned long long per_step,
               unsigned long long k, cudaStream_t st) {
  note_launch(), wait_flag_kernel<<<1, 1, 0, st>>>(flag, tstep, per_step, k);
}
__global__ void set_flag_kernel(unsigned long long* flag, const long long* tstep, unsigned long long per_step,
                                unsigned long long k) {
  const unsigned long long value = (unsigned long long)(*tstep - 1) * per_step + k;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}
void set_flag(unsigned long long* flag, const long long* tstep, unsigned long long per_step, unsigned long long k,
              cudaStream_t st) {
  note_launch(), set_flag_kernel<<<1, 1, 0, st>>>(flag, tstep, per_step, k);
}
// counter idx += 1 in every data-parallel peer's flag array (fbase[p], system-scope release after all
// prior work on the stream): "my gradient of layer j is staged" / "my shard j is updated" / "I read it"
__global__ void dp_signal_kernel(unsigned long long* const* fbase, int D, int idx) {
  if ((int)threadIdx.x >= D) return;
  __threadfence_system();
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(fbase[threadIdx.x] + idx), "l"(1ull) : "memory");
}
void dp_signal(unsigned long long* const* fbase, int D, int idx, cudaStream_t st) {
  note_launch(), dp_signal_kernel<<<1, 32, 0, st>>>(fbase, D, idx);
}

// World-wide loss all-reduce over peer memory (replaces a 1-element NCCL all-reduce): thread q stores this
// rank's loss sum into rank q's ring slot [t mod 4][rank] and bumps q's arrival counter (system-scope
// release); thread 0 then waits for all `world` arrivals of step t and sums the slots in rank order, so every
// rank gets the same bits.  Four ring slots: a rank can run at most one step ahead of a peer (every world > 1
// step has a cross-rank dependency: the data-parallel gathers or the pipeline receives).
__global__ void loss_allreduce_kernel(double* loss, double* const* ring, unsigned long long* const* wflag, int rank,
                                      int world, const long long* tstep, const volatile unsigned long long* myflag,
                                      const volatile double* myring) {
  const long long t = *tstep;
  const int slot = (int)(t & 3);
  const double mine = loss[0];
  if ((int)threadIdx.x < world) {
    const int q = threadIdx.x;
    volatile double* dst = ring[q] + slot * world + rank;
    *dst = mine;
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(wflag[q] + 0), "l"(1ull) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)t * (unsigned long long)world;
    unsigned long long v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(myflag) : "memory");
      if (v >= target) break;
      __nanosleep(200);
    }
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += myring[slot * world + r];
    loss[0] = s;
  }
}
void loss_allreduce_peer(double* loss, double* const* ring, unsigned long long* const* wflag, int rank, int world,
                         const long long* tstep, const unsigned long long* myflag, const double* myring,
                         cudaStream_t st) {
  note_launch(), loss_allreduce_kernel<<<1, 32, 0, st>>>(loss, ring, wflag, rank, world, tstep, myflag, myring);
}

// Device barrier over peer memory: bump every rank's counter wflag[q][1], wait until this rank's counter
// reaches `target` (= world x barriers so far).  Gives up after timeout_ns (a peer that died must not hang
// lga_destroy): *timed_out = 1.
__global__ void world_barrier_kernel(unsigned long long* const* wflag, int world, unsigned long long target,
                                     const volatile unsigned long long* myflag, int* timed_out, long long timeout_ns) {
  if ((int)threadIdx.x < world) {
    __threadfence_system();
    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(wflag[threadIdx.x] + 1), "l"(1ull) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t0, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(myflag) : "memory");
      if (v >= target) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if ((long long)(now - t0) > timeout_ns) {
        *timed_out = 1;
        break;
      }
      __nanosleep(1000);
    }
  }
}
void world_barrier(unsigned long long* const* wflag, int world, unsigned long long target,
                   const unsigned long long* myflag, int* timed_out, long long timeout_ns, cudaStream_t st) {
  note_launch(), world_barrier_kernel<<<1, 32, 0, st>>>(wflag, world, target, myflag, timed_out, timeout_ns);
}

// the step counter t (AdamW bias corrections, flag epochs): incremented first thing in every step
__global__ void step_begin_kernel(long long* tstep) {   // [0] AdamW step, [1] flag epoch
  tstep[0] += 1;
  tstep[1] += 1;
}
void step_begin(long long* tstep, cudaStream_t st) { note_launch(), step_begin_kernel<<<1, 1, 0, st>>>(tstep); }

static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace lga
