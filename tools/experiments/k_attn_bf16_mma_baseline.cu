// NOT BUILT: the round-1 warp-level mma.sync flash attention (the comparison baseline the tcgen05 kernels
// replaced); kept for reference only, outside the product library.
// k_attn_bf16.cu -- bf16 causal multi-head attention forward / backward on the tensor cores
// (warp-level mma.sync m16n8k16, fp32 accumulate), flash-style (O3 / O5 of DESIGN.md):
//   forward : online softmax over 64-key tiles, o and the per-row log-sum-exp written once;
//   backward: P recomputed from lse; dK/dV per key tile (loop over query tiles) and dQ per query
//             tile (loop over key tiles) in two kernels -- no float atomics, bitwise reproducible.
// Shared-memory tiles use a 16-byte-chunk XOR swizzle (chunk ^ row%8) so ldmatrix is conflict-free.
#include "kernels.cuh"

namespace lga {
namespace fa {

constexpr int BQ = 64;   // query rows per block (4 warps x 16)
constexpr int BKV = 64;  // key rows per tile
constexpr int NT = 128;
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of (row, 16B-chunk) in a swizzled [rows][DH] bf16 tile
template <int DH>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * DH * 2 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}

__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Load a [ROWS][DH] tile whose row r is at gbase + r*ld (elements), rows >= nrows zero-filled.
template <int DH, int ROWS>
__device__ __forceinline__ void load_tile(uint8_t* sm, const __nv_bfloat16* gbase, int64_t ld, int nrows) {
  constexpr int CH = DH / 8;
  for (int e = threadIdx.x; e < ROWS * CH; e += NT) {
    const int r = e / CH, c = e % CH;
    const bool ok = r < nrows;
    const __nv_bfloat16* src = gbase + (ok ? (int64_t)r * ld + c * 8 : 0);
    cp_async16(smem_u32(sm) + swz<DH>(r, c), src, ok);
  }
}

// A fragments (16 rows x DH) of a warp's rows [r0, r0+16) from a swizzled tile
template <int DH>
__device__ __forceinline__ void load_a_frags(const uint8_t* sm, int r0, uint32_t (&f)[DH / 16][4]) {
  const int l = threadIdx.x & 31;
  const int row = r0 + (l & 7) + ((l >> 3) & 1) * 8;
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    const int chunk = kk * 2 + (l >> 4);
    ldsm_x4(smem_u32(sm) + swz<DH>(row, chunk), f[kk][0], f[kk][1], f[kk][2], f[kk][3]);
  }
}

// B fragments for S = A * T^T where T is [n][k] row-major (keys x dh): two n8 tiles (n0, n0+8), k16 block kk
template <int DH>
__device__ __forceinline__ void load_b_nt(const uint8_t* sm, int n0, int kk, uint32_t& b00, uint32_t& b01, uint32_t& b10,
                                          uint32_t& b11) {
  const int l = threadIdx.x & 31;
  const int n = n0 + (l & 7) + (l >> 4) * 8;
  const int chunk = kk * 2 + ((l >> 3) & 1);
  ldsm_x4(smem_u32(sm) + swz<DH>(n, chunk), b00, b01, b10, b11);
}

// B fragments for O = P * T where T is [k][n] row-major (keys x dh): k16 block at k0, two n8 tiles at dh col n0
template <int DH>
__device__ __forceinline__ void load_b_t(const uint8_t* sm, int k0, int n0, uint32_t& b00, uint32_t& b01, uint32_t& b10,
                                         uint32_t& b11) {
  const int l = threadIdx.x & 31;
  const int k = k0 + (l & 7) + ((l >> 3) & 1) * 8;
  const int chunk = (n0 >> 3) + (l >> 4);
  ldsm_x4_t(smem_u32(sm) + swz<DH>(k, chunk), b00, b01, b10, b11);
}

// ============================================================================ forward
template <int DH>
__global__ void __launch_bounds__(NT) fwd_kernel(AttnArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* Qs = sm;
  uint8_t* Ks = sm + BQ * DH * 2;                 // [2][BKV][DH]
  uint8_t* Vs = Ks + 2 * BKV * DH * 2;            // [2][BKV][DH]
  const int nqt = gridDim.x;
  const int qt = a.causal ? nqt - 1 - (int)blockIdx.x : (int)blockIdx.x;   // heavy tiles first
  const int h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int64_t ld = 3LL * d;
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(a.qkv) + (int64_t)sq * s * ld;
  const __nv_bfloat16* qg = base + (int64_t)qt * BQ * ld + h * DH;
  const __nv_bfloat16* kg = base + d + h * DH;
  const __nv_bfloat16* vg = base + 2 * d + h * DH;
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  const int q0 = qt * BQ;
  const int nkv_all = (s + BKV - 1) / BKV;
  const int nkv = a.causal ? min(nkv_all, (q0 + BQ - 1) / BKV + 1) : nkv_all;

  load_tile<DH, BQ>(Qs, qg, ld, s - q0);
  load_tile<DH, BKV>(Ks, kg, ld, s);
  load_tile<DH, BKV>(Vs, vg, ld, s);
  cp_commit();

  uint32_t qf[DH / 16][4];
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  const float sl2 = a.scale * LOG2E;
  const int qi0 = q0 + warp * 16 + g, qi1 = qi0 + 8;

  for (int j = 0; j < nkv; ++j) {
    if (j + 1 < nkv) {
      const int nb = (j + 1) & 1;
      load_tile<DH, BKV>(Ks + nb * BKV * DH * 2, kg + (int64_t)(j + 1) * BKV * ld, ld, s - (j + 1) * BKV);
      load_tile<DH, BKV>(Vs + nb * BKV * DH * 2, vg + (int64_t)(j + 1) * BKV * ld, ld, s - (j + 1) * BKV);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) load_a_frags<DH>(Qs, warp * 16, qf);
    const uint8_t* Kb = Ks + (j & 1) * BKV * DH * 2;
    const uint8_t* Vb = Vs + (j & 1) * BKV * DH * 2;
    float sc[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) sc[n][0] = sc[n][1] = sc[n][2] = sc[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b00, b01, b10, b11;
        load_b_nt<DH>(Kb, np * 16, kk, b00, b01, b10, b11);
        mma(sc[2 * np], qf[kk], b00, b01);
        mma(sc[2 * np + 1], qf[kk], b10, b11);
      }
    }
    // scale (log2 domain) + mask
    const int k0 = j * BKV;
    float mx[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int n = 0; n < 8; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kj = k0 + n * 8 + 2 * t + (e & 1);
        const int qi = (e < 2) ? qi0 : qi1;
        float v = sc[n][e] * sl2;
        if (kj >= s || (a.causal && kj > qi)) v = -INFINITY;
        sc[n][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      corr[r] = (mx[r] == -INFINITY) ? 1.f : exp2f(mrow[r] - mx[r]);
      mrow[r] = mx[r];
    }
    uint32_t pf[4][4];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = mrow[e >> 1];
        p[e] = (mm == -INFINITY) ? 0.f : exp2f(sc[n][e] - mm);
        rs[e >> 1] += p[e];
      }
      pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      lrow[r] = lrow[r] * corr[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= corr[0]; o[i][1] *= corr[0];
      o[i][2] *= corr[1]; o[i][3] *= corr[1];
    }
    // o += P V   (A = P: rows x 64 keys in 4 k16 blocks; a-fragment reg order a0,a1,a2,a3)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const uint32_t af[4] = {pf[kb][0], pf[kb][1], pf[kb][2], pf[kb][3]};
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        uint32_t b00, b01, b10, b11;
        load_b_t<DH>(Vb, kb * 16, dp * 16, b00, b01, b10, b11);
        mma(o[2 * dp], af, b00, b01);
        mma(o[2 * dp + 1], af, b10, b11);
      }
    }
    __syncthreads();
  }
  // finalize
  __nv_bfloat16* og = static_cast<__nv_bfloat16*>(a.o) + (int64_t)sq * s * d + h * DH;
  const float inv0 = lrow[0] > 0.f ? 1.f / lrow[0] : 0.f, inv1 = lrow[1] > 0.f ? 1.f / lrow[1] : 0.f;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const int c = i * 8 + 2 * t;
    if (qi0 < s) *reinterpret_cast<uint32_t*>(og + (int64_t)qi0 * d + c) = pack_bf16(o[i][0] * inv0, o[i][1] * inv0);
    if (qi1 < s) *reinterpret_cast<uint32_t*>(og + (int64_t)qi1 * d + c) = pack_bf16(o[i][2] * inv1, o[i][3] * inv1);
  }
  if (t == 0) {
    float* lse = a.lse + ((int64_t)sq * a.heads + h) * s;
    const float LN2 = 0.6931471805599453f;
    if (qi0 < s) lse[qi0] = (mrow[0] + log2f(lrow[0])) * LN2;
    if (qi1 < s) lse[qi1] = (mrow[1] + log2f(lrow[1])) * LN2;
  }
}

// ============================================================================ backward
// Dsum[i] = rowsum(dO_i * o_i) per (seq, head, query)
template <int DH>
__global__ void dsum_kernel(AttnArgs a) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);   // over nseq*seq*heads
  const int l = threadIdx.x & 31;
  const int64_t total = (int64_t)a.nseq * a.seq * a.heads;
  if (row >= total) return;
  const int h = (int)(row % a.heads);
  const int64_t tok = row / a.heads;   // sq*s + i
  const __nv_bfloat16* o = static_cast<const __nv_bfloat16*>(a.o) + tok * a.d + h * DH;
  const __nv_bfloat16* dO = static_cast<const __nv_bfloat16*>(a.dO) + tok * a.d + h * DH;
  float sacc = 0.f;
  for (int c = l * 2; c < DH; c += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + c));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dO + c));
    sacc += x.x * y.x + x.y * y.y;
  }
  sacc = warp_sum(sacc);
  if (l == 0) {
    const int64_t sq = tok / a.seq, i = tok % a.seq;
    a.dsum[(sq * a.heads + h) * a.seq + i] = sacc;
  }
}

// dK, dV for one key tile (4 warps x 16 keys), looping over query tiles
template <int DH>
__global__ void __launch_bounds__(NT) dkdv_kernel(AttnArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* Ks = sm;                        // [BKV][DH]
  uint8_t* Vs = Ks + BKV * DH * 2;         // [BKV][DH]
  uint8_t* Qs = Vs + BKV * DH * 2;         // [2][BQ][DH]
  uint8_t* Gs = Qs + 2 * BQ * DH * 2;      // [2][BQ][DH]  dO
  float* Ls = reinterpret_cast<float*>(Gs + 2 * BQ * DH * 2);   // [2][BQ] lse (log2 domain)
  float* Ds = Ls + 2 * BQ;                                      // [2][BQ]
  const int kt = blockIdx.x, h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int64_t ld = 3LL * d;
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(a.qkv) + (int64_t)sq * s * ld;
  const __nv_bfloat16* qg = base + h * DH;
  const __nv_bfloat16* kg = base + (int64_t)kt * BKV * ld + d + h * DH;
  const __nv_bfloat16* vg = base + (int64_t)kt * BKV * ld + 2 * d + h * DH;
  const __nv_bfloat16* gg = static_cast<const __nv_bfloat16*>(a.dO) + (int64_t)sq * s * d + h * DH;
  const float* lse = a.lse + ((int64_t)sq * a.heads + h) * s;
  const float* dsum = a.dsum + ((int64_t)sq * a.heads + h) * s;
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  const int k0 = kt * BKV;
  const int nqt = (s + BQ - 1) / BQ;
  const int qstart = a.causal ? k0 / BQ : 0;
  const float sl2 = a.scale * LOG2E;

  auto load_q = [&](int qt, int buf) {
    load_tile<DH, BQ>(Qs + buf * BQ * DH * 2, qg + (int64_t)qt * BQ * ld, ld, s - qt * BQ);
    load_tile<DH, BQ>(Gs + buf * BQ * DH * 2, gg + (int64_t)qt * BQ * d, d, s - qt * BQ);
    for (int r = threadIdx.x; r < BQ; r += NT) {
      const int i = qt * BQ + r;
      Ls[buf * BQ + r] = i < s ? lse[i] * LOG2E : 0.f;
      Ds[buf * BQ + r] = i < s ? dsum[i] : 0.f;
    }
  };
  load_tile<DH, BKV>(Ks, kg, ld, s - k0);
  load_tile<DH, BKV>(Vs, vg, ld, s - k0);
  if (qstart < nqt) load_q(qstart, 0);
  cp_commit();

  uint32_t kf[DH / 16][4], vf[DH / 16][4];
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int kj0 = k0 + warp * 16 + g, kj1 = kj0 + 8;

  for (int qt = qstart; qt < nqt; ++qt) {
    const int buf = (qt - qstart) & 1;
    __syncthreads();   // previous iteration done with the other buffer
    if (qt + 1 < nqt) {
      load_q(qt + 1, buf ^ 1);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (qt == qstart) {
      load_a_frags<DH>(Ks, warp * 16, kf);
      load_a_frags<DH>(Vs, warp * 16, vf);
    }
    const uint8_t* Qb = Qs + buf * BQ * DH * 2;
    const uint8_t* Gb = Gs + buf * BQ * DH * 2;
    const float* Lb = Ls + buf * BQ;
    const float* Db = Ds + buf * BQ;
    // S^T = K Q^T (16 keys x 64 queries) and dP^T = V dO^T
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[n][e] = dpt[n][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b00, b01, b10, b11;
        load_b_nt<DH>(Qb, np * 16, kk, b00, b01, b10, b11);
        mma(st[2 * np], kf[kk], b00, b01);
        mma(st[2 * np + 1], kf[kk], b10, b11);
        load_b_nt<DH>(Gb, np * 16, kk, b00, b01, b10, b11);
        mma(dpt[2 * np], vf[kk], b00, b01);
        mma(dpt[2 * np + 1], vf[kk], b10, b11);
      }
    }
    // P^T = exp2(S^T*scale*log2e - lse2[q]); dS^T = P^T (dP^T - D[q]) * scale
    uint32_t pf[4][4], sf[4][4];
    const int qb0 = qt * BQ;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float p[4], ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = n * 8 + 2 * t + (e & 1);
        const int qi = qb0 + qc;
        const int kj = (e < 2) ? kj0 : kj1;
        const bool valid = qi < s && kj < s && (!a.causal || kj <= qi);
        p[e] = valid ? exp2f(st[n][e] * sl2 - Lb[qc]) : 0.f;
        ds[e] = p[e] * (dpt[n][e] - Db[qc]) * a.scale;
      }
      pf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
      pf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
      sf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
      sf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
    // dV += P^T dO ; dK += dS^T Q   (B = [queries][dh] row-major -> transposed ldmatrix)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const uint32_t ap[4] = {pf[kb][0], pf[kb][1], pf[kb][2], pf[kb][3]};
      const uint32_t as[4] = {sf[kb][0], sf[kb][1], sf[kb][2], sf[kb][3]};
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        uint32_t b00, b01, b10, b11;
        load_b_t<DH>(Gb, kb * 16, dp * 16, b00, b01, b10, b11);
        mma(dv[2 * dp], ap, b00, b01);
        mma(dv[2 * dp + 1], ap, b10, b11);
        load_b_t<DH>(Qb, kb * 16, dp * 16, b00, b01, b10, b11);
        mma(dk[2 * dp], as, b00, b01);
        mma(dk[2 * dp + 1], as, b10, b11);
      }
    }
  }
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + (int64_t)sq * s * ld + h * DH;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const int c = i * 8 + 2 * t;
    if (kj0 < s) {
      *reinterpret_cast<uint32_t*>(out + (int64_t)kj0 * ld + d + c) = pack_bf16(dk[i][0], dk[i][1]);
      *reinterpret_cast<uint32_t*>(out + (int64_t)kj0 * ld + 2 * d + c) = pack_bf16(dv[i][0], dv[i][1]);
    }
    if (kj1 < s) {
      *reinterpret_cast<uint32_t*>(out + (int64_t)kj1 * ld + d + c) = pack_bf16(dk[i][2], dk[i][3]);
      *reinterpret_cast<uint32_t*>(out + (int64_t)kj1 * ld + 2 * d + c) = pack_bf16(dv[i][2], dv[i][3]);
    }
  }
}

// dQ for one query tile (4 warps x 16 queries), looping over key tiles
template <int DH>
__global__ void __launch_bounds__(NT) dq_kernel(AttnArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* Qs = sm;                        // [BQ][DH]
  uint8_t* Gs = Qs + BQ * DH * 2;          // [BQ][DH]
  uint8_t* Ks = Gs + BQ * DH * 2;          // [2][BKV][DH]
  uint8_t* Vs = Ks + 2 * BKV * DH * 2;     // [2][BKV][DH]
  const int nqt = gridDim.x;
  const int qt = a.causal ? nqt - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int64_t ld = 3LL * d;
  const __nv_bfloat16* base = static_cast<const __nv_bfloat16*>(a.qkv) + (int64_t)sq * s * ld;
  const int q0 = qt * BQ;
  const __nv_bfloat16* qg = base + (int64_t)q0 * ld + h * DH;
  const __nv_bfloat16* kg = base + d + h * DH;
  const __nv_bfloat16* vg = base + 2 * d + h * DH;
  const __nv_bfloat16* gg = static_cast<const __nv_bfloat16*>(a.dO) + ((int64_t)sq * s + q0) * d + h * DH;
  const int warp = threadIdx.x >> 5, l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  const int nkv_all = (s + BKV - 1) / BKV;
  const int nkv = a.causal ? min(nkv_all, (q0 + BQ - 1) / BKV + 1) : nkv_all;
  const float sl2 = a.scale * LOG2E;
  const int qi0 = q0 + warp * 16 + g, qi1 = qi0 + 8;
  const int64_t rb = ((int64_t)sq * a.heads + h) * s;
  const float L0 = qi0 < s ? a.lse[rb + qi0] * LOG2E : 0.f, L1 = qi1 < s ? a.lse[rb + qi1] * LOG2E : 0.f;
  const float D0 = qi0 < s ? a.dsum[rb + qi0] : 0.f, D1 = qi1 < s ? a.dsum[rb + qi1] : 0.f;

  load_tile<DH, BQ>(Qs, qg, ld, s - q0);
  load_tile<DH, BQ>(Gs, gg, d, s - q0);
  load_tile<DH, BKV>(Ks, kg, ld, s);
  load_tile<DH, BKV>(Vs, vg, ld, s);
  cp_commit();
  uint32_t qf[DH / 16][4], gf[DH / 16][4];
  float dq[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;

  for (int j = 0; j < nkv; ++j) {
    if (j + 1 < nkv) {
      const int nb = (j + 1) & 1;
      load_tile<DH, BKV>(Ks + nb * BKV * DH * 2, kg + (int64_t)(j + 1) * BKV * ld, ld, s - (j + 1) * BKV);
      load_tile<DH, BKV>(Vs + nb * BKV * DH * 2, vg + (int64_t)(j + 1) * BKV * ld, ld, s - (j + 1) * BKV);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (j == 0) {
      load_a_frags<DH>(Qs, warp * 16, qf);
      load_a_frags<DH>(Gs, warp * 16, gf);
    }
    const uint8_t* Kb = Ks + (j & 1) * BKV * DH * 2;
    const uint8_t* Vb = Vs + (j & 1) * BKV * DH * 2;
    float sc[8][4], dp[8][4];
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) sc[n][e] = dp[n][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t b00, b01, b10, b11;
        load_b_nt<DH>(Kb, np * 16, kk, b00, b01, b10, b11);
        mma(sc[2 * np], qf[kk], b00, b01);
        mma(sc[2 * np + 1], qf[kk], b10, b11);
        load_b_nt<DH>(Vb, np * 16, kk, b00, b01, b10, b11);
        mma(dp[2 * np], gf[kk], b00, b01);
        mma(dp[2 * np + 1], gf[kk], b10, b11);
      }
    }
    uint32_t sf[4][4];
    const int k0 = j * BKV;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float ds[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kj = k0 + n * 8 + 2 * t + (e & 1);
        const int qi = e < 2 ? qi0 : qi1;
        const bool valid = kj < s && qi < s && (!a.causal || kj <= qi);
        const float p = valid ? exp2f(sc[n][e] * sl2 - (e < 2 ? L0 : L1)) : 0.f;
        ds[e] = p * (dp[n][e] - (e < 2 ? D0 : D1)) * a.scale;
      }
      sf[n >> 1][(n & 1) * 2 + 0] = pack_bf16(ds[0], ds[1]);
      sf[n >> 1][(n & 1) * 2 + 1] = pack_bf16(ds[2], ds[3]);
    }
    // dQ += dS K   (B = K [keys][dh] -> transposed ldmatrix)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const uint32_t as[4] = {sf[kb][0], sf[kb][1], sf[kb][2], sf[kb][3]};
#pragma unroll
      for (int dd = 0; dd < DH / 16; ++dd) {
        uint32_t b00, b01, b10, b11;
        load_b_t<DH>(Kb, kb * 16, dd * 16, b00, b01, b10, b11);
        mma(dq[2 * dd], as, b00, b01);
        mma(dq[2 * dd + 1], as, b10, b11);
      }
    }
    __syncthreads();
  }
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + (int64_t)sq * s * ld + h * DH;
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) {
    const int c = i * 8 + 2 * t;
    if (qi0 < s) *reinterpret_cast<uint32_t*>(out + (int64_t)qi0 * ld + c) = pack_bf16(dq[i][0], dq[i][1]);
    if (qi1 < s) *reinterpret_cast<uint32_t*>(out + (int64_t)qi1 * ld + c) = pack_bf16(dq[i][2], dq[i][3]);
  }
}

template <int DH>
void run_fwd(const AttnArgs& a, cudaStream_t st) {
  const int smem = (BQ + 4 * BKV) * DH * 2;
  static bool set = false;
  if (!set) { cudaFuncSetAttribute(fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); set = true; }
  dim3 grid((a.seq + BQ - 1) / BQ, a.heads, a.nseq);
  note_launch(), fwd_kernel<DH><<<grid, NT, smem, st>>>(a);
}

template <int DH>
void run_bwd(const AttnArgs& a, cudaStream_t st) {
  const int64_t rows = (int64_t)a.nseq * a.seq * a.heads;
  note_launch(), dsum_kernel<DH><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(a);
  const int smem_kv = (2 * BKV + 4 * BQ) * DH * 2 + 4 * BQ * 4;
  const int smem_q = (2 * BQ + 4 * BKV) * DH * 2;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(dkdv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
    cudaFuncSetAttribute(dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
    set = true;
  }
  dim3 gk((a.seq + BKV - 1) / BKV, a.heads, a.nseq);
  note_launch(), dkdv_kernel<DH><<<gk, NT, smem_kv, st>>>(a);
  dim3 gq((a.seq + BQ - 1) / BQ, a.heads, a.nseq);
  note_launch(), dq_kernel<DH><<<gq, NT, smem_q, st>>>(a);
}

}  // namespace fa

void attn_fwd_bf16_mma(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return;
  if (a.dh == 64) fa::run_fwd<64>(a, st);
  else fa::run_fwd<128>(a, st);
}

void attn_bwd_bf16_mma(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return;
  if (a.dh == 64) fa::run_bwd<64>(a, st);
  else fa::run_bwd<128>(a, st);
}

}  // namespace lga
