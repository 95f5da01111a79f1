// TMEM load / store throughput microbenchmark (sm_100a): W warps per CTA, each issuing K tcgen05.ld (or st)
// 32x32b.x32 (4 KB per warp instruction) before one wait, ITERS times; one CTA per SM.  Prints bytes per SM cycle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2106_02679_b200/csrc \
//        tools/experiments/tmem_bw.cu -o /tmp/tmem_bw && /tmp/tmem_bw
#include <cstdio>
#include "tc_common.cuh"

using namespace lga::tcu;

template <int K, bool STORE>
__global__ void bw_kernel(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t base = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = ((warp >> 2) * 32 * K) & 511;
  uint32_t acc = 0;
  float vals[32];
  for (int i = 0; i < 32; ++i) vals[i] = (float)(threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (STORE) {
#pragma unroll
      for (int k = 0; k < K; ++k) tmem_st32(base + lane_off + ((col0 + 32 * k) & 511), vals);
      tmem_wait_st();
    } else {
      uint32_t r[K][32];
#pragma unroll
      for (int k = 0; k < K; ++k) tmem_ld32_nowait(base + lane_off + ((col0 + 32 * k) & 511), r[k]);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < 32; ++c) acc ^= r[k][c];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 0x12345678u) sink[0] = acc;
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    tmem_dealloc(base, 512);
  }
}

template <int K, bool STORE>
void run(int warps) {
  const int iters = 2000, ctas = 148;
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, ctas * 8);
  cudaMalloc(&sink, 4);
  bw_kernel<K, STORE><<<ctas, warps * 32>>>(iters, cyc, sink);
  bw_kernel<K, STORE><<<ctas, warps * 32>>>(iters, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < ctas; ++i) mean += (double)h[i] / ctas;
  const double bytes = (double)warps * K * 4096.0 * iters;
  printf("%s warps=%2d K=%d: %8.1f cycles/iter  %6.1f B/cycle/SM  (%s)\n", STORE ? "st" : "ld", warps, K, mean / iters,
         bytes / mean, cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  run<1, false>(4);
  run<2, false>(4);
  run<4, false>(4);
  run<2, false>(8);
  run<4, false>(8);
  run<2, false>(16);
  run<1, false>(16);
  run<1, true>(4);
  run<2, true>(8);
  run<2, true>(16);
  return 0;
}
