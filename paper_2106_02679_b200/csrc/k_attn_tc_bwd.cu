// k_attn_tc_bwd.cu -- causal multi-head attention backward on the 5th-generation tensor cores (sm_100a).
//
// O5 of DESIGN.md with P recomputed from the saved log-sum-exp (flash-style), no float atomics:
//   dsum_i = rowsum(dO_i * o_i)
//   dK/dV kernel, one CTA per 128-key tile, looping over 64-query tiles:
//     S^T = K Q^T, dP^T = V dO^T            (tcgen05, M=128 keys, N=64 queries, K=d_h; TMEM, 2 buffers)
//     P^T = exp(S^T*scale - lse), dS^T = P^T (dP^T - dsum) * scale   (4 warps, one key row per thread)
//     dV += P^T dO, dK += dS^T Q              (tcgen05, A = P^T / dS^T from smem, B = dO / Q read MN-major
//                                              from the very tiles TMA loaded K-major for the first two MMAs)
//   dQ kernel, one CTA per 128-query tile, looping over 64-key tiles:
//     S = Q K^T, dP = dO V^T ; dS = P (dP - dsum) * scale ; dQ += dS K   (K read MN-major)
// Warp roles: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4..7 element-wise + epilogue.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace lga {
namespace fatb {

using namespace tcu;

constexpr int EW_WARPS = 16;                // element-wise warps: 4 per TMEM lane quadrant, 16 columns each
constexpr int EW_THREADS = EW_WARPS * 32;
constexpr int NT = (4 + EW_WARPS) * 32;
constexpr float LOG2E = 1.4426950408889634f;

// rowsum(dO * o) per (sequence, head, position); one warp per row
__global__ void dsum_kernel(AttnArgs a) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);   // token*heads + h
  const int l = threadIdx.x & 31;
  if (row >= (int64_t)a.nseq * a.seq * a.heads) return;
  const int h = (int)(row % a.heads);
  const int64_t tok = row / a.heads;
  const __nv_bfloat16* o = static_cast<const __nv_bfloat16*>(a.o) + tok * a.d + (int64_t)h * a.dh;
  const __nv_bfloat16* g = static_cast<const __nv_bfloat16*>(a.dO) + tok * a.d + (int64_t)h * a.dh;
  float acc = 0.f;
  for (int c = l * 2; c < a.dh; c += 64) {
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + c));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + c));
    acc += x.x * y.x + x.y * y.y;
  }
  acc = warp_sum(acc);
  if (l == 0) a.dsum[((tok / a.seq) * a.heads + h) * a.seq + tok % a.seq] = acc;
}

// 16 bf16 (2 chunks of 16 B, chunk indices 2*quarter, 2*quarter+1) of row r of a [128][64] K-major SW128 tile
__device__ __forceinline__ void st_quarter_row_bf16(uint8_t* tile, int r, int quarter, const uint32_t (&pk)[8]) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const uint32_t addr = smem_u32(tile) + sw128(r, quarter * 2 + i);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[i * 4]), "r"(pk[i * 4 + 1]),
                 "r"(pk[i * 4 + 2]), "r"(pk[i * 4 + 3])
                 : "memory");
  }
}

// TMEM row -> bf16 global row.  tcgen05.ld is warp-collective: every lane executes it, only
// lanes with `valid` store.
__device__ __forceinline__ void store_row_bf16_global(__nv_bfloat16* dst, uint32_t taddr, int ncols, float scale,
                                                      bool valid) {
  for (int c = 0; c < ncols; c += 16) {   // ncols is a multiple of 16
    uint32_t r[16];
    tmem_ld16_nowait(taddr + c, r);
    tmem_wait_ld();
    if (!valid) continue;
    float t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = __uint_as_float(r[i]) * scale;
    uint4* p = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
    for (int i = 0; i < 2; ++i)
      p[i] = make_uint4(pack_bf16x2(t[8 * i], t[8 * i + 1]), pack_bf16x2(t[8 * i + 2], t[8 * i + 3]),
                        pack_bf16x2(t[8 * i + 4], t[8 * i + 5]), pack_bf16x2(t[8 * i + 6], t[8 * i + 7]));
  }
}

// =============================================================================== dK / dV
constexpr int KB = 128;  // keys per CTA
constexpr int QB = 64;   // queries per iteration

template <int DH>
struct DkvSmem {
  static constexpr int SUB128 = 128 * 128;             // [128 rows][64] bf16 sub-tile = 16 KB
  static constexpr int SUB64 = 64 * 128;               // [64 rows][64] bf16 sub-tile = 8 KB
  static constexpr int KT = DH / 64 * SUB128;          // K (or V) tile [128][DH]
  static constexpr int QT = DH / 64 * SUB64;           // Q (or dO) tile [64][DH]
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KT;
  static constexpr int NST = 3;                        // Q / dO ring depth
  static constexpr int Q_OFF = V_OFF + KT;             // [NST]
  static constexpr int G_OFF = Q_OFF + NST * QT;       // dO [NST]
  static constexpr int PT_OFF = G_OFF + NST * QT;      // P^T [2][128][64]
  static constexpr int DST_OFF = PT_OFF + 2 * SUB128;  // dS^T [2][128][64]
  static constexpr int LD_OFF = DST_OFF + 2 * SUB128;  // lse[2][64], dsum[2][64] (floats)
  static constexpr int BAR_OFF = LD_OFF + 4 * 64 * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int DH>
__global__ void __launch_bounds__(NT, 1)
    dkdv_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_g, const AttnArgs a) {
  using SM = DkvSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  constexpr int NST = SM::NST;
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;              // [NST]
  uint64_t* q_empty = q_full + NST;         // [NST]
  uint64_t* s_full = q_empty + NST;         // [2]
  uint64_t* s_empty = s_full + 2;           // [2] (EW_THREADS arrivals)
  uint64_t* p_full = s_empty + 2;           // (EW_THREADS arrivals)
  uint64_t* g_done = p_full + 1;            // [2] per P^T / dS^T buffer
  constexpr int NBAR = 2 * NST + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);
  float* lse_s = reinterpret_cast<float*>(smem + SM::LD_OFF);   // [2][64]
  float* dsum_s = lse_s + 128;                                   // [2][64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x, h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int k0 = kt * KB;
  const int nq_all = (s + QB - 1) / QB;
  const int qstart = a.causal ? k0 / QB : 0;
  const int nq = nq_all - qstart;
  const int64_t rb = ((int64_t)sq * a.heads + h) * s;   // row base of lse / dsum

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NBAR; ++i) {
      const bool ew = &bars[i] == s_empty || &bars[i] == s_empty + 1 || &bars[i] == p_full;
      mbar_init(&bars[i], ew ? EW_THREADS : 1);
    }
    mbar_fence_init();
    prefetch_tmap(&tm_kv);
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_g);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = *tmem_slot;
  const uint32_t t_st[2] = {tb, tb + 64}, t_dpt[2] = {tb + 128, tb + 192};
  const uint32_t t_dv = tb + 256, t_dk = tb + 256 + DH;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      mbar_expect_tx(kv_full, 2 * SM::KT);
#pragma unroll
      for (int i = 0; i < DH / 64; ++i) {
        tma_load_3d(smem + SM::K_OFF + i * SM::SUB128, &tm_kv, kv_full, d + h * DH + 64 * i, k0, sq);
        tma_load_3d(smem + SM::V_OFF + i * SM::SUB128, &tm_kv, kv_full, 2 * d + h * DH + 64 * i, k0, sq);
      }
      for (int i = 0; i < nq; ++i) {
        const int st = i % NST;
        const int q0 = (qstart + i) * QB;
        mbar_wait(&q_empty[st], ((i / NST) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * SM::QT);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_3d(smem + SM::Q_OFF + st * SM::QT + c * SM::SUB64, &tm_q, &q_full[st], h * DH + 64 * c, q0, sq);
          tma_load_3d(smem + SM::G_OFF + st * SM::QT + c * SM::SUB64, &tm_g, &q_full[st], h * DH + 64 * c, q0, sq);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      constexpr uint32_t idesc_s = make_idesc(128, QB, false, false);
      constexpr uint32_t idesc_g = make_idesc(128, DH, false, true);
      const uint32_t sK = smem_u32(smem + SM::K_OFF), sV = smem_u32(smem + SM::V_OFF);
      const uint32_t sPt = smem_u32(smem + SM::PT_OFF), sDSt = smem_u32(smem + SM::DST_OFF);
      mbar_wait(kv_full, 0);
      for (int i = 0; i <= nq; ++i) {
        if (i < nq) {
          const int st = i % NST, b = i & 1;
          mbar_wait(&q_full[st], (i / NST) & 1);
          mbar_wait(&s_empty[b], ((i >> 1) & 1) ^ 1);
          fence_after();
          const uint32_t sQ = smem_u32(smem + SM::Q_OFF + st * SM::QT);
          const uint32_t sG = smem_u32(smem + SM::G_OFF + st * SM::QT);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * SM::SUB128 + (kk & 3) * 32, ob = (kk >> 2) * SM::SUB64 + (kk & 3) * 32;
            umma_f16(t_st[b], make_desc(sK + oa, 16, 1024), make_desc(sQ + ob, 16, 1024), idesc_s, kk > 0);
            umma_f16(t_dpt[b], make_desc(sV + oa, 16, 1024), make_desc(sG + ob, 16, 1024), idesc_s, kk > 0);
          }
          umma_commit(&s_full[b]);
        }
        if (i >= 1) {
          const int ii = i - 1, st = ii % NST, pb = ii & 1;
          mbar_wait(p_full, ii & 1);
          fence_after();
          const uint32_t sQ = smem_u32(smem + SM::Q_OFF + st * SM::QT);
          const uint32_t sG = smem_u32(smem + SM::G_OFF + st * SM::QT);
          const uint32_t sPtb = sPt + pb * SM::SUB128, sDStb = sDSt + pb * SM::SUB128;
#pragma unroll
          for (int kk = 0; kk < QB / 16; ++kk) {
            const uint32_t oa = kk * 32;                // K-major A: 16 queries = 32 B into the swizzle span
            const uint32_t ob = kk * 16 * 128;          // MN-major B: 16 query rows
            const uint32_t acc = (ii > 0 || kk > 0) ? 1u : 0u;
            umma_f16(t_dv, make_desc(sPtb + oa, 16, 1024), make_desc(sG + ob, SM::SUB64, 1024), idesc_g, acc);
            umma_f16(t_dk, make_desc(sDStb + oa, 16, 1024), make_desc(sQ + ob, SM::SUB64, 1024), idesc_g, acc);
          }
          umma_commit(&g_done[pb]);
          umma_commit(&q_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {  // ===== element-wise: one key row per 4 threads (query-column quarters)
    const int qd = warp & 3;
    const int hf = (warp - 4) >> 2;            // quarter 0..3 of the 64 query columns
    const int r = qd * 32 + lane;
    const int tid = threadIdx.x - 128;
    const int kj = k0 + r;
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    uint8_t* sPt = smem + SM::PT_OFF;
    uint8_t* sDSt = smem + SM::DST_OFF;
    // lse (log2 units) / dsum of query tile i: loaded two iterations ahead into a register by threads
    // tid < 128, parked in shared buffer i&1 at the end of iteration i-1 (barrier at the top of i)
    auto ld_stat = [&](int i) -> float {
      const int q = (qstart + i) * QB + (tid & 63);
      if (tid >= 128 || i >= nq || q >= s) return 0.f;
      return tid < 64 ? a.lse[rb + q] * LOG2E : a.dsum[rb + q];
    };
    if (tid < 128) (tid < 64 ? lse_s : dsum_s)[tid & 63] = ld_stat(0);
    float pre1 = ld_stat(1);
    for (int i = 0; i < nq; ++i) {
      const float pre2 = ld_stat(i + 2);
      const int b = i & 1, st = i & 1;
      const int q0 = (qstart + i) * QB;
      mbar_wait(&s_full[b], (i >> 1) & 1);
      fence_after();
      uint32_t rsv[16], rdp[16];
      tmem_ld16_nowait(t_st[b] + lrow + hf * 16, rsv);
      tmem_ld16_nowait(t_dpt[b] + lrow + hf * 16, rdp);
      tmem_wait_ld();
      fence_before();
      mbar_arrive(&s_empty[b]);
      asm volatile("bar.sync 1, %0;" ::"n"(EW_THREADS) : "memory");   // tile i's lse / dsum visible
      const float* ls = lse_s + st * 64 + hf * 16;
      const float* ds_ = dsum_s + st * 64 + hf * 16;
      // valid iff q < s, kj < s and (causal) kj <= q; only tiles touching the diagonal / the end mask
      const int qa = q0 + hf * 16;
      const bool need_mask = kj >= s || qa + 16 > s || (a.causal && kj > qa);
      float sc[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) sc[c] = fmaf(__uint_as_float(rsv[c]), sl2, -ls[c]);
      if (need_mask) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int q = qa + c;
          if (!(q < s && kj < s && (!a.causal || kj <= q))) sc[c] = -INFINITY;
        }
      }
      uint32_t pp[8], pd[8];
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        float p[2], g[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          p[e] = ex2(sc[c + e]);
          g[e] = p[e] * (__uint_as_float(rdp[c + e]) - ds_[c + e]) * a.scale;
        }
        pp[c / 2] = pack_bf16x2(p[0], p[1]);
        pd[c / 2] = pack_bf16x2(g[0], g[1]);
      }
      const int pb = i & 1;
      if (i >= 2) {
        mbar_wait(&g_done[pb], ((i >> 1) & 1) ^ 1);   // dV/dK MMAs of iteration i-2 done: buffer pb free
        fence_after();
      }
      st_quarter_row_bf16(sPt + pb * SM::SUB128, r, hf, pp);
      st_quarter_row_bf16(sDSt + pb * SM::SUB128, r, hf, pd);
      fence_proxy_async();
      fence_before();
      mbar_arrive(p_full);
      if (tid < 128) (tid < 64 ? lse_s : dsum_s)[(st ^ 1) * 64 + (tid & 63)] = pre1;   // tile i+1
      pre1 = pre2;
    }
    mbar_wait(&g_done[(nq - 1) & 1], ((nq - 1) >> 1) & 1);   // last iteration's MMAs (and all earlier) done
    fence_after();
    constexpr int OC = DH / 4;   // output columns per quarter
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + ((int64_t)sq * s + kj) * 3 * d + h * DH + hf * OC;
    store_row_bf16_global(out + d, t_dk + lrow + hf * OC, OC, 1.f, kj < s);
    store_row_bf16_global(out + 2 * d, t_dv + lrow + hf * OC, OC, 1.f, kj < s);
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tb, 512);
  }
}

// =============================================================================== dQ
constexpr int QB2 = 128;  // queries per CTA
constexpr int KB2 = 64;   // keys per iteration

template <int DH>
struct DqSmem {
  static constexpr int SUB128 = 128 * 128;
  static constexpr int SUB64 = 64 * 128;
  static constexpr int QT = DH / 64 * SUB128;   // Q (or dO) [128][DH]
  static constexpr int KT = DH / 64 * SUB64;    // K (or V) [64][DH]
  static constexpr int Q_OFF = 0;
  static constexpr int G_OFF = Q_OFF + QT;
  static constexpr int NST = 4;                 // K / V ring depth
  static constexpr int K_OFF = G_OFF + QT;      // [NST]
  static constexpr int V_OFF = K_OFF + NST * KT;  // [NST]
  static constexpr int DS_OFF = V_OFF + NST * KT; // dS [2][128][64]
  static constexpr int BAR_OFF = DS_OFF + 2 * SUB128;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int DH>
__global__ void __launch_bounds__(NT, 1)
    dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_g,
              const __grid_constant__ CUtensorMap tm_kv, const AttnArgs a) {
  using SM = DqSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  constexpr int NST = SM::NST;
  uint64_t* qg_full = bars + 0;
  uint64_t* kv_full = bars + 1;             // [NST]
  uint64_t* kv_empty = kv_full + NST;       // [NST]
  uint64_t* s_full = kv_empty + NST;        // [2]
  uint64_t* s_empty = s_full + 2;           // [2] (EW_THREADS)
  uint64_t* p_full = s_empty + 2;           // (EW_THREADS)
  uint64_t* g_done = p_full + 1;            // [2] per dS buffer
  constexpr int NBAR = 2 * NST + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x;
  const int qt = a.causal ? nqt - 1 - (int)blockIdx.x : (int)blockIdx.x;
  const int h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int q0 = qt * QB2;
  const int kend = a.causal ? min(s, q0 + QB2) : s;
  const int nk = (kend + KB2 - 1) / KB2;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NBAR; ++i) {
      const bool ew = &bars[i] == s_empty || &bars[i] == s_empty + 1 || &bars[i] == p_full;
      mbar_init(&bars[i], ew ? EW_THREADS : 1);
    }
    mbar_fence_init();
    prefetch_tmap(&tm_q);
    prefetch_tmap(&tm_g);
    prefetch_tmap(&tm_kv);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = *tmem_slot;
  const uint32_t t_s[2] = {tb, tb + 64}, t_dp[2] = {tb + 128, tb + 192};
  const uint32_t t_dq = tb + 256;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      mbar_expect_tx(qg_full, 2 * SM::QT);
#pragma unroll
      for (int c = 0; c < DH / 64; ++c) {
        tma_load_3d(smem + SM::Q_OFF + c * SM::SUB128, &tm_q, qg_full, h * DH + 64 * c, q0, sq);
        tma_load_3d(smem + SM::G_OFF + c * SM::SUB128, &tm_g, qg_full, h * DH + 64 * c, q0, sq);
      }
      for (int j = 0; j < nk; ++j) {
        const int st = j % NST;
        mbar_wait(&kv_empty[st], ((j / NST) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * SM::KT);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_3d(smem + SM::K_OFF + st * SM::KT + c * SM::SUB64, &tm_kv, &kv_full[st], d + h * DH + 64 * c, j * KB2, sq);
          tma_load_3d(smem + SM::V_OFF + st * SM::KT + c * SM::SUB64, &tm_kv, &kv_full[st], 2 * d + h * DH + 64 * c,
                      j * KB2, sq);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      constexpr uint32_t idesc_s = make_idesc(128, KB2, false, false);
      constexpr uint32_t idesc_q = make_idesc(128, DH, false, true);
      const uint32_t sQ = smem_u32(smem + SM::Q_OFF), sG = smem_u32(smem + SM::G_OFF);
      const uint32_t sDS = smem_u32(smem + SM::DS_OFF);
      mbar_wait(qg_full, 0);
      for (int j = 0; j <= nk; ++j) {
        if (j < nk) {
          const int st = j % NST, b = j & 1;
          mbar_wait(&kv_full[st], (j / NST) & 1);
          mbar_wait(&s_empty[b], ((j >> 1) & 1) ^ 1);
          fence_after();
          const uint32_t sK = smem_u32(smem + SM::K_OFF + st * SM::KT);
          const uint32_t sV = smem_u32(smem + SM::V_OFF + st * SM::KT);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * SM::SUB128 + (kk & 3) * 32, ob = (kk >> 2) * SM::SUB64 + (kk & 3) * 32;
            umma_f16(t_s[b], make_desc(sQ + oa, 16, 1024), make_desc(sK + ob, 16, 1024), idesc_s, kk > 0);
            umma_f16(t_dp[b], make_desc(sG + oa, 16, 1024), make_desc(sV + ob, 16, 1024), idesc_s, kk > 0);
          }
          umma_commit(&s_full[b]);
        }
        if (j >= 1) {
          const int jj = j - 1, st = jj % NST, pb = jj & 1;
          mbar_wait(p_full, jj & 1);
          fence_after();
          const uint32_t sK = smem_u32(smem + SM::K_OFF + st * SM::KT);
#pragma unroll
          for (int kk = 0; kk < KB2 / 16; ++kk)
            umma_f16(t_dq, make_desc(sDS + pb * SM::SUB128 + kk * 32, 16, 1024),
                     make_desc(sK + kk * 16 * 128, SM::SUB64, 1024), idesc_q, (jj > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&g_done[pb]);
          umma_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {  // ===== element-wise: one query row per 4 threads (key-column quarters)
    const int qd = warp & 3;
    const int hf = (warp - 4) >> 2;            // quarter 0..3 of the 64 key columns
    const int r = qd * 32 + lane;
    const int q = q0 + r;
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    const int64_t rb = ((int64_t)sq * a.heads + h) * s;
    const float lse2 = q < s ? a.lse[rb + q] * LOG2E : 0.f;
    const float Dq = q < s ? a.dsum[rb + q] : 0.f;
    uint8_t* sDS = smem + SM::DS_OFF;
    for (int j = 0; j < nk; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      fence_after();
      uint32_t rsv[16], rdp[16];
      tmem_ld16_nowait(t_s[b] + lrow + hf * 16, rsv);
      tmem_ld16_nowait(t_dp[b] + lrow + hf * 16, rdp);
      tmem_wait_ld();
      fence_before();
      mbar_arrive(&s_empty[b]);
      const int ka = j * KB2 + hf * 16;
      const bool need_mask = q >= s || ka + 16 > s || (a.causal && ka + 15 > q0 + qd * 32);
      float sc[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) sc[c] = fmaf(__uint_as_float(rsv[c]), sl2, -lse2);
      if (need_mask) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int kj = ka + c;
          if (!(q < s && kj < s && (!a.causal || kj <= q))) sc[c] = -INFINITY;
        }
      }
      uint32_t pd[8];
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        float g[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) g[e] = ex2(sc[c + e]) * (__uint_as_float(rdp[c + e]) - Dq) * a.scale;
        pd[c / 2] = pack_bf16x2(g[0], g[1]);
      }
      const int pb = j & 1;
      if (j >= 2) {
        mbar_wait(&g_done[pb], ((j >> 1) & 1) ^ 1);   // dQ MMAs of iteration j-2 done: buffer pb free
        fence_after();
      }
      st_quarter_row_bf16(sDS + pb * SM::SUB128, r, hf, pd);
      fence_proxy_async();
      fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(&g_done[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
    fence_after();
    constexpr int OC = DH / 4;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + ((int64_t)sq * s + q) * 3 * d + h * DH + hf * OC;
    store_row_bf16_global(out, t_dq + lrow + hf * OC, OC, 1.f, q < s);
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tb, 512);
  }
}

template <int DH>
static cudaError_t run(const AttnArgs& a, cudaStream_t st) {
  const int64_t rows = (int64_t)a.nseq * a.seq * a.heads;
  note_launch(), dsum_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(a);
  CUtensorMap kv128, q64, g64, q128, g128, kv64;
  cudaError_t e;
  const uint64_t ld = 3ull * a.d;
  if ((e = map3d_bf16(&kv128, a.qkv, ld, a.seq, a.nseq, 128)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&q64, a.qkv, ld, a.seq, a.nseq, 64)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&g64, a.dO, a.d, a.seq, a.nseq, 64)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&q128, a.qkv, ld, a.seq, a.nseq, 128)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&g128, a.dO, a.d, a.seq, a.nseq, 128)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&kv64, a.qkv, ld, a.seq, a.nseq, 64)) != cudaSuccess) return e;
  static bool set = false;
  if (!set) {
    if ((e = cudaFuncSetAttribute(dkdv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, DkvSmem<DH>::TOTAL)))
      return e;
    if ((e = cudaFuncSetAttribute(dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqSmem<DH>::TOTAL)))
      return e;
    set = true;
  }
  dim3 gk((a.seq + KB - 1) / KB, a.heads, a.nseq);
  note_launch(), dkdv_kernel<DH><<<gk, NT, DkvSmem<DH>::TOTAL, st>>>(kv128, q64, g64, a);
  dim3 gq((a.seq + QB2 - 1) / QB2, a.heads, a.nseq);
  note_launch(), dq_kernel<DH><<<gq, NT, DqSmem<DH>::TOTAL, st>>>(q128, g128, kv64, a);
  return cudaGetLastError();
}

}  // namespace fatb

cudaError_t attn_bwd_bf16(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return cudaSuccess;
  return a.dh == 64 ? fatb::run<64>(a, st) : fatb::run<128>(a, st);
}

}  // namespace lga
