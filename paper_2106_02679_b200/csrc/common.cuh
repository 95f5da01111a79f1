// common.cuh -- shared types and helpers of the LGA library (device + host).
// Nothing here is method arithmetic; see kernels.cuh for the operations and their citations.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace lga {

// host-side count of kernels launched by this library (bench.py's gpu_launches)
void note_launch();
unsigned long long launch_count();

enum class DT : int { F32 = 0, BF16 = 1 };

__host__ __device__ inline size_t dt_size(DT t) { return t == DT::F32 ? 4 : 2; }

// ---- element load / store in either storage type (fp32 or bf16, round-to-nearest-even)
__device__ __forceinline__ float ld_elem(const void* p, size_t i, DT t) {
  return t == DT::F32 ? static_cast<const float*>(p)[i]
                      : __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ void st_elem(void* p, size_t i, DT t, float v) {
  if (t == DT::F32) static_cast<float*>(p)[i] = v;
  else static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

template <typename E> struct ElemT;
template <> struct ElemT<float> { static constexpr DT dt = DT::F32; };
template <> struct ElemT<__nv_bfloat16> { static constexpr DT dt = DT::BF16; };

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename E> __device__ __forceinline__ E from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// ---- exact-erf GELU and its derivative (reading A-1):  g = u Phi(u),  g' = Phi(u) + u phi(u)
__device__ __forceinline__ float gelu_f(float u) {
  return 0.5f * u * (1.0f + erff(u * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float u) {
  const float Phi = 0.5f * (1.0f + erff(u * 0.70710678118654752f));
  const float phi = 0.39894228040143268f * expf(-0.5f * u * u);
  return Phi + u * phi;
}

// ---- warp / block reductions (fixed shuffle order => deterministic)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of two floats over the block; `red` must hold 2*32 floats of shared memory.
__device__ __forceinline__ float2 block_sum2(float a, float b, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a); b = warp_sum(b);
  __syncthreads();
  if (lane == 0) { red[w] = a; red[32 + w] = b; }
  __syncthreads();
  float ra = 0.f, rb = 0.f;
  for (int i = 0; i < nw; ++i) { ra += red[i]; rb += red[32 + i]; }   // fixed order
  return make_float2(ra, rb);
}

}  // namespace lga
