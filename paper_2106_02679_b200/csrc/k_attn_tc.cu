// k_attn_tc.cu -- causal multi-head attention forward on the 5th-generation tensor cores (sm_100a).
//
// One CTA = 128 query rows of one (sequence, head).  Per 128-key tile j:
//   S_j = Q K_j^T        tcgen05.mma (M=128, N=128, K=d_h), fp32 in TMEM (two S buffers)
//   P_j = exp2(S_j*scale*log2e - m)   by 4 softmax warps, one query row (TMEM lane) per thread,
//                        written as bf16 into shared memory in the UMMA K-major SW128 layout
//   O  += P_j V_j        tcgen05.mma (M=128, N=d_h, K=128), V read MN-major from the same tile TMA loaded
// Online softmax with lazy rescaling: the running max m used for P only moves when a row max exceeds
// it by more than 2^8, then O (in TMEM) and l are rescaled by the softmax thread that owns the row.
// The result is the same definition (O3): o = sum_j P_j V_j / l, lse = m + log2(l) (natural log saved).
// Warp roles: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4..7 softmax + epilogue.
#include "kernels.cuh"
#include "tc_common.cuh"

#include <cudaTypedefs.h>

#include <mutex>

namespace lga {
namespace fat {

using namespace tcu;

constexpr int BQ = 128, BKV = 128;
constexpr int SM_WARPS = 8;                    // softmax warps: 2 per TMEM lane quadrant, 64 key columns each
constexpr int NT = (4 + SM_WARPS) * 32;
constexpr int SM_THREADS = SM_WARPS * 32;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.0f;   // log2 units

template <int DH>
struct FwdSmem {
  static constexpr int TILE = BQ * DH * 2;          // [128][DH] bf16 as DH/64 swizzled [128][64] sub-tiles
  static constexpr int SUB = 128 * 64 * 2;          // 16 KB
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE;        // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * TILE;    // 2 stages
  static constexpr int P_OFF = V_OFF + 2 * TILE;    // [128][128] bf16 = 2 sub-tiles
  static constexpr int RED_OFF = P_OFF + 2 * SUB;   // [2 tile parity][2 halves][128 rows] row maxima + [2][128] sums
  static constexpr int BAR_OFF = RED_OFF + 6 * 128 * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <int DH>
__global__ void __launch_bounds__(NT, 1) fwd_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  using SM = FwdSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;     // [2]
  uint64_t* v_full = bars + 3;     // [2]
  uint64_t* kv_empty = bars + 5;   // [2]
  uint64_t* s_full = bars + 7;     // [2]
  uint64_t* s_empty = bars + 9;    // [2]
  uint64_t* p_full = bars + 11;
  uint64_t* o_done = bars + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = gridDim.x;
  const int qt = a.causal ? nqt - 1 - (int)blockIdx.x : (int)blockIdx.x;   // heavy tiles first
  const int h = blockIdx.y, sq = blockIdx.z;
  const int s = a.seq, d = a.d;
  const int q0 = qt * BQ;
  const int nkv_all = (s + BKV - 1) / BKV;
  const int nkv = a.causal ? min(nkv_all, (q0 + BQ - 1) / BKV + 1) : nkv_all;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 14; ++i) {
      const bool by_softmax = (&bars[i] == s_empty) || (&bars[i] == s_empty + 1) || (&bars[i] == p_full);
      mbar_init(&bars[i], by_softmax ? SM_THREADS : 1);   // softmax threads arrive individually
    }
    mbar_fence_init();
    prefetch_tmap(&tm);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t t_s[2] = {tbase, tbase + 128};
  const uint32_t t_o = tbase + 256;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      mbar_expect_tx(q_full, SM::TILE);
#pragma unroll
      for (int i = 0; i < DH / 64; ++i) tma_load_3d(smem + SM::Q_OFF + i * SM::SUB, &tm, q_full, h * DH + 64 * i, q0, sq);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&k_full[st], SM::TILE);
#pragma unroll
        for (int i = 0; i < DH / 64; ++i)
          tma_load_3d(smem + SM::K_OFF + st * SM::TILE + i * SM::SUB, &tm, &k_full[st], d + h * DH + 64 * i, j * BKV, sq);
        mbar_expect_tx(&v_full[st], SM::TILE);
#pragma unroll
        for (int i = 0; i < DH / 64; ++i)
          tma_load_3d(smem + SM::V_OFF + st * SM::TILE + i * SM::SUB, &tm, &v_full[st], 2 * d + h * DH + 64 * i,
                      j * BKV, sq);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer
      constexpr uint32_t idesc_s = make_idesc(128, BKV, false, false);
      constexpr uint32_t idesc_o = make_idesc(128, DH, false, true);
      const uint32_t sQ = smem_u32(smem + SM::Q_OFF);
      const uint32_t sP = smem_u32(smem + SM::P_OFF);
      mbar_wait(q_full, 0);
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int st = j & 1, b = j & 1;
          mbar_wait(&k_full[st], (j >> 1) & 1);
          mbar_wait(&s_empty[b], ((j >> 1) & 1) ^ 1);
          fence_after();
          const uint32_t sK = smem_u32(smem + SM::K_OFF + st * SM::TILE);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t off = (kk >> 2) * SM::SUB + (kk & 3) * 32;
            umma_f16(t_s[b], make_desc(sQ + off, 16, 1024), make_desc(sK + off, 16, 1024), idesc_s, kk > 0);
          }
          umma_commit(&s_full[b]);
        }
        if (j >= 1) {
          const int jj = j - 1, st = jj & 1;
          mbar_wait(p_full, jj & 1);
          mbar_wait(&v_full[st], (jj >> 1) & 1);
          fence_after();
          const uint32_t sV = smem_u32(smem + SM::V_OFF + st * SM::TILE);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t ad = make_desc(sP + (kk >> 2) * SM::SUB + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = make_desc(sV + kk * 16 * 128, SM::SUB, 1024);   // MN-major: d_h blocks at 16 KB
            umma_f16(t_o, ad, bd, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(o_done);
          umma_commit(&kv_empty[st]);
        }
      }
    }
  } else if (warp >= 4) {  // ===== softmax + epilogue: one query row per thread pair (two column halves)
    const int qd = warp & 3;
    const int hf = (warp - 4) >> 2;            // key-column half / O-column half this warp owns
    const int r = qd * 32 + lane;
    const int q = q0 + r;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    uint8_t* sP = smem + SM::P_OFF + hf * SM::SUB;   // this half's [128][64] P sub-tile
    float* red = reinterpret_cast<float*>(smem + SM::RED_OFF);   // [2 parity][2 halves][128]
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      fence_after();
      uint32_t raw[2][32];
      tmem_ld32_nowait(t_s[b] + lane_off + hf * 64, raw[0]);
      tmem_ld32_nowait(t_s[b] + lane_off + hf * 64 + 32, raw[1]);
      tmem_wait_ld();
      fence_before();
      mbar_arrive(&s_empty[b]);
      const int k0 = j * BKV + hf * 64;
      float sv[64];
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        const int kj = k0 + c;
        float v = __uint_as_float(raw[c >> 5][c & 31]) * sl2;
        if (kj >= s || (a.causal && kj > q)) v = -INFINITY;
        sv[c] = v;
        mx = fmaxf(mx, v);
      }
      // row max over both halves: exchange through shared memory (buffer parity j&1 avoids a WAR race)
      red[((j & 1) * 2 + hf) * 128 + r] = mx;
      asm volatile("bar.sync 1, %0;" ::"n"(SM_THREADS) : "memory");
      mx = fmaxf(mx, red[((j & 1) * 2 + (hf ^ 1)) * 128 + r]);
      const float m_new = (mx > m_used + RESCALE_THRESHOLD) ? mx : m_used;
      float rs = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 64; c += 2) {
        const float p0 = m_new == -INFINITY ? 0.f : exp2f(sv[c] - m_new);
        const float p1 = m_new == -INFINITY ? 0.f : exp2f(sv[c + 1] - m_new);
        rs += p0 + p1;
        pk[c / 2] = pack_bf16x2(p0, p1);
      }
      if (j >= 1) {
        mbar_wait(o_done, (j - 1) & 1);   // PV_{j-1} done: O stable, P buffer free
        fence_after();
      }
      float scale = 1.f;
      if (m_new != m_used && m_used != -INFINITY) {   // lazy rescale of this half's O columns
        scale = exp2f(m_used - m_new);
#pragma unroll 1
        for (int c = hf * (DH / 64); c < (hf + 1) * (DH / 64); ++c) {
          float t[32];
          tmem_ld32(t_o + lane_off + c * 32, t);
#pragma unroll
          for (int i = 0; i < 32; ++i) t[i] *= scale;
          tmem_st32(t_o + lane_off + c * 32, t);
        }
      }
      l = l * scale + rs;   // partial row sum over this half's keys
      m_used = m_new;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t addr = smem_u32(sP) + sw128(r, ch);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[ch * 4]), "r"(pk[ch * 4 + 1]),
                     "r"(pk[ch * 4 + 2]), "r"(pk[ch * 4 + 3])
                     : "memory");
      }
      fence_proxy_async();
      fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: l = sum of both halves; O / l -> bf16 global (each half writes its O columns), lse
    red[4 * 128 + hf * 128 + r] = l;
    asm volatile("bar.sync 1, %0;" ::"n"(SM_THREADS) : "memory");
    l += red[4 * 128 + (hf ^ 1) * 128 + r];
    mbar_wait(o_done, (nkv - 1) & 1);
    fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* og = static_cast<__nv_bfloat16*>(a.o) + ((int64_t)sq * s + q) * d + h * DH;
#pragma unroll 1
    for (int c = hf * (DH / 64); c < (hf + 1) * (DH / 64); ++c) {
      float t[32];
      tmem_ld32(t_o + lane_off + c * 32, t);
      if (q < s) {
        uint4* dst = reinterpret_cast<uint4*>(og + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_uint4(pack_bf16x2(t[8 * i] * inv, t[8 * i + 1] * inv), pack_bf16x2(t[8 * i + 2] * inv, t[8 * i + 3] * inv),
                              pack_bf16x2(t[8 * i + 4] * inv, t[8 * i + 5] * inv), pack_bf16x2(t[8 * i + 6] * inv, t[8 * i + 7] * inv));
      }
    }
    if (q < s && hf == 0) a.lse[((int64_t)sq * a.heads + h) * s + q] = (m_used + log2f(l)) * 0.6931471805599453f;
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int DH>
static cudaError_t run_fwd(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tm;
  cudaError_t e = map3d_bf16(&tm, a.qkv, 3ull * a.d, a.seq, a.nseq, 128);
  if (e != cudaSuccess) return e;
  static bool set = false;
  if (!set) {
    e = cudaFuncSetAttribute(fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<DH>::TOTAL);
    if (e != cudaSuccess) return e;
    set = true;
  }
  dim3 grid((a.seq + BQ - 1) / BQ, a.heads, a.nseq);
  note_launch(), fwd_kernel<DH><<<grid, NT, FwdSmem<DH>::TOTAL, st>>>(tm, a);
  return cudaGetLastError();
}

}  // namespace fat

cudaError_t attn_fwd_bf16(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return cudaSuccess;
  return a.dh == 64 ? fat::run_fwd<64>(a, st) : fat::run_fwd<128>(a, st);
}

}  // namespace lga
