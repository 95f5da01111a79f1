// k_ln.cu -- LayerNorm forward / backward and the fixed-order column-sum finisher (HBM-bound).
//
// y = (x - mu) rstd gamma + beta, biased variance (reading A-1); backward (O5):
//   dx = rstd (dxhat - mean(dxhat) - xhat mean(dxhat xhat)) + resid,  dxhat = dout gamma,
//   dgamma = sum_rows dout xhat,  dbeta = sum_rows dout.
// Row kernels: one warp per row, 128-bit loads, the row held in registers (d % 128 == 0), else one block
// per row.  dgamma / dbeta: a separate column kernel writes per-block partials in a fixed row order; the
// finisher sums the partials in a fixed order too -- no float atomics, bitwise reproducible.
#include "kernels.cuh"

#include <algorithm>

namespace lga {

__device__ __forceinline__ float4 ld4(const void* p, DT t, int64_t i) {
  if (t == DT::F32) return *reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
  const uint2 u = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(p) + i);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xFFFF0000u));
}
__device__ __forceinline__ void st4(void* p, DT t, int64_t i, float4 v) {
  if (t == DT::F32) {
    *reinterpret_cast<float4*>(static_cast<float*>(p) + i) = v;
  } else {
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p) + i) =
        make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

// =============================================================== forward
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_warp(const float* __restrict__ x, const void* gamma, const void* beta,
                                                   DT pdt, void* y, DT ydt, float2* __restrict__ stats, int rows,
                                                   int d, float eps) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* xr = x + (int64_t)row * d;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    v[k] = *reinterpret_cast<const float4*>(xr + lane * 4 + 128 * k);
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  const float mean = warp_sum(s) / d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const float a = v[k].x - mean, b = v[k].y - mean, c = v[k].z - mean, e = v[k].w - mean;
    q += (a * a + b * b) + (c * c + e * e);
  }
  const float rstd = rsqrtf(warp_sum(q) / d + eps);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = lane * 4 + 128 * k;
    const float4 g = ld4(gamma, pdt, c), b = ld4(beta, pdt, c);
    st4(y, ydt, (int64_t)row * d + c,
        make_float4((v[k].x - mean) * rstd * g.x + b.x, (v[k].y - mean) * rstd * g.y + b.y,
                    (v[k].z - mean) * rstd * g.z + b.z, (v[k].w - mean) * rstd * g.w + b.w));
  }
  if (lane == 0) stats[row] = make_float2(mean, rstd);
}

// generic d: block per row, VPT values per thread
template <int VPT>
__global__ void __launch_bounds__(256) ln_fwd_block(const float* __restrict__ x, const void* gamma, const void* beta,
                                                    DT pdt, void* y, DT ydt, float2* __restrict__ stats, int d,
                                                    float eps) {
  __shared__ float red[64];
  const int64_t row = blockIdx.x;
  const float* xr = x + row * d;
  float v[VPT];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    v[i] = c < d ? xr[c] : 0.f;
    s += v[i];
  }
  const float mean = block_sum2(s, 0.f, red).x / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    const float t = c < d ? v[i] - mean : 0.f;
    q += t * t;
  }
  const float rstd = rsqrtf(block_sum2(q, 0.f, red).x / d + eps);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < d) st_elem(y, row * d + c, ydt, (v[i] - mean) * rstd * ld_elem(gamma, c, pdt) + ld_elem(beta, c, pdt));
  }
  if (threadIdx.x == 0) stats[row] = make_float2(mean, rstd);
}

void ln_fwd(const float* x, const void* gamma, const void* beta, DT pdt, void* y, DT ydt, float2* stats, int rows,
            int d, float eps, cudaStream_t st) {
  if (rows <= 0) return;
  if (d % 128 == 0 && d <= 4096) {
    const int nv = d / 128, grid = (rows + 7) / 8;
#define LF(N) note_launch(), ln_fwd_warp<N><<<grid, 256, 0, st>>>(x, gamma, beta, pdt, y, ydt, stats, rows, d, eps)
    switch (nv) {
      case 1: LF(1); break; case 2: LF(2); break; case 3: LF(3); break; case 4: LF(4); break;
      case 5: LF(5); break; case 6: LF(6); break; case 8: LF(8); break; case 12: LF(12); break;
      case 16: LF(16); break; case 24: LF(24); break; case 32: LF(32); break;
      default: goto generic;
    }
#undef LF
    return;
  }
generic : {
  const int bd = d >= 1024 ? 256 : (d >= 256 ? 128 : 64);
  const int vpt = (d + bd - 1) / bd;
#define LB(V) note_launch(), ln_fwd_block<V><<<rows, bd, 0, st>>>(x, gamma, beta, pdt, y, ydt, stats, d, eps)
  if (vpt <= 1) LB(1); else if (vpt <= 2) LB(2); else if (vpt <= 4) LB(4);
  else if (vpt <= 8) LB(8); else if (vpt <= 16) LB(16); else LB(32);
#undef LB
}
}

// =============================================================== backward: dx (rows)
// Two passes over the row (the second hits L2): pass 1 accumulates sum(dxhat) and sum(dxhat xhat),
// pass 2 recomputes dxhat, xhat and writes dx.  No row kept in registers -> full occupancy.
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_warp(const float* __restrict__ dout, const float* __restrict__ x,
                                                   const float2* __restrict__ stats, const void* gamma, DT pdt,
                                                   const float* __restrict__ resid, float* __restrict__ dx,
                                                   void* dx_e, DT edt, int rows, int d) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t base = (int64_t)row * d;
  const float2 sr = stats[row];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll 4
  for (int k = 0; k < NV; ++k) {
    const int c = lane * 4 + 128 * k;
    const float4 xv = *reinterpret_cast<const float4*>(x + base + c);
    const float4 go = *reinterpret_cast<const float4*>(dout + base + c);
    const float4 g = ld4(gamma, pdt, c);
    const float g0 = go.x * g.x, g1 = go.y * g.y, g2 = go.z * g.z, g3 = go.w * g.w;
    s1 += (g0 + g1) + (g2 + g3);
    s2 += (g0 * (xv.x - sr.x) + g1 * (xv.y - sr.x)) + (g2 * (xv.z - sr.x) + g3 * (xv.w - sr.x));
  }
  const float m1 = warp_sum(s1) / d, m2 = warp_sum(s2) * sr.y / d;
#pragma unroll 4
  for (int k = 0; k < NV; ++k) {
    const int c = lane * 4 + 128 * k;
    const float4 xv = *reinterpret_cast<const float4*>(x + base + c);
    const float4 go = *reinterpret_cast<const float4*>(dout + base + c);
    const float4 g = ld4(gamma, pdt, c);
    float4 v = make_float4(sr.y * (go.x * g.x - m1 - (xv.x - sr.x) * sr.y * m2),
                           sr.y * (go.y * g.y - m1 - (xv.y - sr.x) * sr.y * m2),
                           sr.y * (go.z * g.z - m1 - (xv.z - sr.x) * sr.y * m2),
                           sr.y * (go.w * g.w - m1 - (xv.w - sr.x) * sr.y * m2));
    if (resid) {
      const float4 r = *reinterpret_cast<const float4*>(resid + base + c);
      v.x += r.x; v.y += r.y; v.z += r.z; v.w += r.w;
    }
    *reinterpret_cast<float4*>(dx + base + c) = v;
    if (dx_e) st4(dx_e, edt, base + c, v);
  }
}

template <int VPT>
__global__ void __launch_bounds__(256) ln_bwd_block(const float* __restrict__ dout, const float* __restrict__ x,
                                                    const float2* __restrict__ stats, const void* gamma, DT pdt,
                                                    const float* __restrict__ resid, float* __restrict__ dx,
                                                    void* dx_e, DT edt, int d) {
  __shared__ float red[64];
  const int64_t row = blockIdx.x, base = row * d;
  const float2 sr = stats[row];
  float xh[VPT], gh[VPT];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    xh[i] = c < d ? (x[base + c] - sr.x) * sr.y : 0.f;
    gh[i] = c < d ? dout[base + c] * ld_elem(gamma, c, pdt) : 0.f;
    s1 += gh[i];
    s2 += gh[i] * xh[i];
  }
  const float2 s = block_sum2(s1, s2, red);
  const float m1 = s.x / d, m2 = s.y / d;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < d) {
      float v = sr.y * (gh[i] - m1 - xh[i] * m2);
      if (resid) v += resid[base + c];
      dx[base + c] = v;
      if (dx_e) st_elem(dx_e, base + c, edt, v);
    }
  }
}

// =============================================================== backward, fused (d = 256 * CPL)
// dx AND the dgamma / dbeta column partials in one pass over dout and x: warp w owns columns
// [256 w, 256 w + 256), CPL per lane; a block takes groups of LNF_ROWS rows (grid-stride), holds them in
// registers, reduces each row's two sums across the 8 warps in a fixed order through shared memory, writes
// dx, and accumulates dgamma / dbeta for its columns in registers -- one partial per block (fixed grid,
// fixed row order: bitwise reproducible).
// rows held in registers per group and resident blocks per SM (measured at the 1.3B shape, d = 2048, fused
// backward with the 4 column sums: 4 rows x 2 blocks 0.232 ms, 2 x 3 0.223 ms (5.41 TB/s), 2 x 4 and 3 x 3 spill;
// 2 x 3 with the L2 prefetch of the residual row: 0.202 ms, 5.98 TB/s)
#ifndef LGA_LNF_ROWS
#define LGA_LNF_ROWS 2
#endif
#ifndef LGA_LNF_MINB
#define LGA_LNF_MINB 3
#endif
constexpr int LNF_ROWS = LGA_LNF_ROWS;
static int lnf_grid(int rows) {
  return std::max(1, std::min((rows + LNF_ROWS - 1) / LNF_ROWS, num_sms() * LGA_LNF_MINB));
}

// EXTRA: also the column sums of resid and of dx (partial rows 2 and 3 of each block's 4 d floats): the bias
// gradients that are column sums of this kernel's input / output (pre-LN LN2: db2 = sum dY, db_o = sum dh1).
template <int CPL, bool EXTRA, int NW = 8>
__global__ void __launch_bounds__(NW * 32, LGA_LNF_MINB) ln_bwd_fused(const float* __restrict__ dout, const float* __restrict__ x,
                                                    const float2* __restrict__ stats, const void* gamma, DT pdt,
                                                    const float* __restrict__ resid, float* __restrict__ dx,
                                                    void* dx_e, DT edt, float* __restrict__ partial, int rows, int d) {
  __shared__ float2 red[LNF_ROWS][NW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = warp * (32 * CPL) + lane * CPL;
  float g[CPL];
  // column accumulators: dgamma, dbeta (+ EXTRA: sum resid, sum dx), in shared memory ([k][thread]:
  // conflict-free): registers hold the row group, and 3 resident blocks per SM need <= 80 registers
  constexpr int NACC = EXTRA ? 4 : 2;
  __shared__ float acc_x[NACC * CPL][NW * 32];
  auto acc = [&](int which, int k) -> float& { return acc_x[which * CPL + k][threadIdx.x]; };
#pragma unroll
  for (int k = 0; k < CPL; k += 4) {
    const float4 t = ld4(gamma, pdt, c0 + k);
    g[k] = t.x, g[k + 1] = t.y, g[k + 2] = t.z, g[k + 3] = t.w;
  }
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    acc(0, k) = 0.f, acc(1, k) = 0.f;
    if (EXTRA) acc(2, k) = 0.f, acc(3, k) = 0.f;
  }
  const float inv_d = 1.f / (float)d;
  for (int r0 = blockIdx.x * LNF_ROWS; r0 < rows; r0 += gridDim.x * LNF_ROWS) {
    float go[LNF_ROWS][CPL], xc[LNF_ROWS][CPL];
    float2 sr[LNF_ROWS];
#pragma unroll
    for (int rr = 0; rr < LNF_ROWS; ++rr) {
      const int r = min(r0 + rr, rows - 1);   // past-the-end rows: recomputed, never stored
      sr[rr] = stats[r];
      const int64_t base = (int64_t)r * d + c0;
#pragma unroll
      for (int k = 0; k < CPL; k += 4) {
        const float4 a = *reinterpret_cast<const float4*>(dout + base + k);
        const float4 b = *reinterpret_cast<const float4*>(x + base + k);
        go[rr][k] = a.x, go[rr][k + 1] = a.y, go[rr][k + 2] = a.z, go[rr][k + 3] = a.w;
        xc[rr][k] = b.x, xc[rr][k + 1] = b.y, xc[rr][k + 2] = b.z, xc[rr][k + 3] = b.w;
      }
#ifndef LGA_LN_NO_PREFETCH
      // the residual row is read only after the cross-warp row sums: start its DRAM fetch now (into L2;
      // registers are full at 3 blocks per SM)
      if (resid) asm volatile("prefetch.global.L2 [%0];" ::"l"(resid + base));
#endif
    }
#pragma unroll
    for (int rr = 0; rr < LNF_ROWS; ++rr) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        xc[rr][k] -= sr[rr].x;   // x - mean
        const float t = go[rr][k] * g[k];
        s1 += t;
        s2 += t * xc[rr][k];
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) red[rr][warp] = make_float2(s1, s2);
    }
    __syncthreads();
    float m1[LNF_ROWS], m2[LNF_ROWS];
#pragma unroll
    for (int rr = 0; rr < LNF_ROWS; ++rr) {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) a += red[rr][w].x, b += red[rr][w].y;   // fixed warp order
      m1[rr] = a * inv_d;
      m2[rr] = b * sr[rr].y * inv_d;
    }
    __syncthreads();   // red reusable by the next row group
#pragma unroll
    for (int rr = 0; rr < LNF_ROWS; ++rr) {
      const int r = r0 + rr;
      if (r >= rows) break;
      const int64_t base = (int64_t)r * d + c0;
      const float rstd = sr[rr].y;
#pragma unroll
      for (int k = 0; k < CPL; k += 4) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float xh = xc[rr][k + e] * rstd;
          v[e] = rstd * (go[rr][k + e] * g[k + e] - m1[rr] - xh * m2[rr]);
          acc(0, k + e) += go[rr][k + e] * xh;
          acc(1, k + e) += go[rr][k + e];
        }
        float4 o = make_float4(v[0], v[1], v[2], v[3]);
        if (resid) {
          const float4 q = *reinterpret_cast<const float4*>(resid + base + k);
          o.x += q.x, o.y += q.y, o.z += q.z, o.w += q.w;
          if (EXTRA) acc(2, k) += q.x, acc(2, k + 1) += q.y, acc(2, k + 2) += q.z, acc(2, k + 3) += q.w;
        }
        if (EXTRA) acc(3, k) += o.x, acc(3, k + 1) += o.y, acc(3, k + 2) += o.z, acc(3, k + 3) += o.w;
        *reinterpret_cast<float4*>(dx + base + k) = o;
        if (dx_e) st4(dx_e, edt, base + k, o);
      }
    }
  }
  constexpr int NP = NACC;   // partial rows per block
  float* pg = partial + (int64_t)blockIdx.x * NP * d + c0;
#pragma unroll
  for (int k = 0; k < CPL; k += 4) {
#pragma unroll
    for (int w = 0; w < NP; ++w)
      *reinterpret_cast<float4*>(pg + w * d + k) = make_float4(acc(w, k), acc(w, k + 1), acc(w, k + 2), acc(w, k + 3));
  }
}

#ifdef LGA_NO_LN_FUSED
static bool lnf_ok(int) { return false; }
#else
// d = 768 (6 warps x 4 columns), 1024 (8 x 4), 2048 (8 x 8); d = 4096 would spill at 2 blocks / SM
static bool lnf_ok(int d) { return d == 768 || d == 1024 || d == 2048; }
#endif

// =============================================================== backward: dgamma / dbeta column partials
constexpr int LN_COL_ROWS = 64;
int ln_bwd_blocks(int rows, int d) {
  return lnf_ok(d) ? lnf_grid(rows) : (rows + LN_COL_ROWS - 1) / LN_COL_ROWS;
}

// sres / sdx (EXTRA): column sums of resid and of the dx the row kernel wrote (4 partial rows per block)
__global__ void __launch_bounds__(256) ln_col_partial(const float* __restrict__ dout, const float* __restrict__ x,
                                                      const float2* __restrict__ stats, const float* __restrict__ resid,
                                                      const float* __restrict__ dx, bool extra,
                                                      float* __restrict__ partial, int rows, int d) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= d) return;
  const int r0 = blockIdx.y * LN_COL_ROWS, r1 = min(rows, r0 + LN_COL_ROWS);
  float dg = 0.f, db = 0.f, sr_ = 0.f, sd = 0.f;
#pragma unroll 4
  for (int r = r0; r < r1; ++r) {
    const float2 sr = stats[r];
    const float go = dout[(int64_t)r * d + c];
    dg += go * ((x[(int64_t)r * d + c] - sr.x) * sr.y);
    db += go;
    if (extra) {
      if (resid) sr_ += resid[(int64_t)r * d + c];
      sd += dx[(int64_t)r * d + c];
    }
  }
  const int np = extra ? 4 : 2;
  partial[(int64_t)blockIdx.y * np * d + c] = dg;
  partial[(int64_t)blockIdx.y * np * d + d + c] = db;
  if (extra) {
    partial[(int64_t)blockIdx.y * np * d + 2 * d + c] = sr_;
    partial[(int64_t)blockIdx.y * np * d + 3 * d + c] = sd;
  }
}

int ln_bwd(const float* dout, const float* x, const float2* stats, const void* gamma, DT pdt, const float* resid,
           float* dx, void* dx_e, DT edt, float* partial, int rows, int d, cudaStream_t st, bool extra) {
  if (rows <= 0) return 0;
  if (lnf_ok(d)) {
    const int grid = lnf_grid(rows);
#define LFU(C, X, W) note_launch(), ln_bwd_fused<C, X, W><<<grid, (W) * 32, 0, st>>>(dout, x, stats, gamma, pdt, resid, dx, dx_e, edt, partial, rows, d)
    if (d == 768) { if (extra) LFU(4, true, 6); else LFU(4, false, 6); }
    else if (d == 1024) { if (extra) LFU(4, true, 8); else LFU(4, false, 8); }
    else { if (extra) LFU(8, true, 8); else LFU(8, false, 8); }
#undef LFU
    return grid;
  }
  bool done = false;
  if (d % 128 == 0 && d <= 4096) {
    const int grid = (rows + 7) / 8;
    done = true;
#define LW(N) note_launch(), ln_bwd_warp<N><<<grid, 256, 0, st>>>(dout, x, stats, gamma, pdt, resid, dx, dx_e, edt, rows, d)
    switch (d / 128) {
      case 1: LW(1); break; case 2: LW(2); break; case 3: LW(3); break; case 4: LW(4); break;
      case 5: LW(5); break; case 6: LW(6); break; case 8: LW(8); break; case 12: LW(12); break;
      case 16: LW(16); break; case 24: LW(24); break; case 32: LW(32); break;
      default: done = false;
    }
#undef LW
  }
  if (!done) {
    const int bd = d >= 1024 ? 256 : (d >= 256 ? 128 : 64);
    const int vpt = (d + bd - 1) / bd;
#define LB(V) note_launch(), ln_bwd_block<V><<<rows, bd, 0, st>>>(dout, x, stats, gamma, pdt, resid, dx, dx_e, edt, d)
    if (vpt <= 1) LB(1); else if (vpt <= 2) LB(2); else if (vpt <= 4) LB(4);
    else if (vpt <= 8) LB(8); else if (vpt <= 16) LB(16); else LB(32);
#undef LB
  }
  const int nblk = ln_bwd_blocks(rows, d);
  dim3 grid((d + 255) / 256, nblk);
  note_launch(), ln_col_partial<<<grid, 256, 0, st>>>(dout, x, stats, resid, dx, extra, partial, rows, d);
  return nblk;
}

// =============================================================== fixed-order finisher
// out[n] = (acc_in ? acc_in[n] : 0) + sum_k partial[k*pstride + n].  Block = FG row groups x 32 columns (each
// warp reads one 128-byte row segment per step); row group g sums partial rows g, g+FG, ... in order, and the
// FG group sums are added in order g = 0..FG-1.  FG = 32 keeps ~1k loads in flight per block: the finish is a
// short pass over a few tens of MB, latency-bound at 8 groups.
constexpr int FG = 32;
__global__ void __launch_bounds__(32 * FG) colsum_finish_kernel(const float* __restrict__ partial, int nblk,
                                                                int64_t pstride, int n, const float* acc_in, void* out,
                                                                DT out_dt) {
  __shared__ float red[FG][33];
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  float s = 0.f;
  if (c < n)
    for (int k = g; k < nblk; k += FG) s += partial[(int64_t)k * pstride + c];
  red[g][cl] = s;
  __syncthreads();
  if (g == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < FG; ++i) t += red[i][cl];
    if (acc_in) t += acc_in[c];
    st_elem(out, c, out_dt, t);
  }
}

// Several finishes over the same partial rows in ONE launch (blockIdx.y = output): the LayerNorm backward's
// dgamma / dbeta (+ the two bias sums) -- same fixed order as colsum_finish_kernel, so the same bits.
__global__ void __launch_bounds__(32 * FG) colsum_finish_multi_kernel(const float* __restrict__ partial, int nblk,
                                                                      int64_t pstride, int n, FinishSet fs) {
  __shared__ float red[FG][33];
  const FinishOut& o = fs.o[blockIdx.y];
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const float* p = partial + o.col0;
  float s = 0.f;
  if (c < n)
    for (int k = g; k < nblk; k += FG) s += p[(int64_t)k * pstride + c];
  red[g][cl] = s;
  __syncthreads();
  if (g == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < FG; ++i) t += red[i][cl];
    if (o.acc_in) t += o.acc_in[c];
    st_elem(o.out, c, o.out_dt, t);
  }
}

void colsum_finish_multi(const float* partial, int nblk, int64_t pstride, int n, const FinishSet& fs, cudaStream_t st) {
  if (n <= 0 || fs.k <= 0) return;
  note_launch(), colsum_finish_multi_kernel<<<dim3((n + 31) / 32, fs.k), 32 * FG, 0, st>>>(partial, nblk, pstride, n, fs);
}

void colsum_finish(const float* partial, int nblk, int64_t pstride, int n, const float* acc_in, void* out, DT out_dt,
                   cudaStream_t st) {
  if (n <= 0) return;
  note_launch(), colsum_finish_kernel<<<(n + 31) / 32, 32 * FG, 0, st>>>(partial, nblk, pstride, n, acc_in, out, out_dt);
}

}  // namespace lga
