// k_attn_tc.cu -- causal multi-head attention forward on the 5th-generation tensor cores (sm_100a).
//
// One CTA = 128 query rows of one (sequence, head).  Per 128-key tile j:
//   S_j = Q K_j^T        tcgen05.mma (M=128, N=128, K=d_h), fp32 in TMEM (two S buffers)
//   P_j = exp2(S_j*scale*log2e - m)   by 8 softmax warps, one query row (TMEM lane) and one key half per
//                        thread, written as bf16 into TMEM over S_j
//   O  += P_j V_j        tcgen05.mma (M=128, N=d_h, K=128; A = P from TMEM), V read MN-major from the tile
//                        TMA loaded
// Online softmax with lazy rescaling: the running max m used for P only moves when a row max exceeds
// it by more than 2^8, then O (in TMEM) and l are rescaled by the softmax thread that owns the row.
// The result is the same definition (O3): o = sum_j P_j V_j / l, lse = m + log2(l) (natural log saved).
// P never touches shared memory: the softmax thread writes it (bf16) into TMEM over the S columns it has
// just read, and the PV MMA takes its A operand from TMEM.
// Warp roles: 0 TMA (Q, K), 1 MMA issuer, 2 TMEM allocator, 3 TMA (V), 4..11 softmax, 12..15 epilogue.
// The epilogue warps take each finished item's O from TMEM (combining the two key halves), free the
// accumulators for the next item's first PV and store O through a swizzled staging tile with TMA, while the
// softmax warps already work on the next item (the per-item epilogue is off the softmax critical path).
#include "kernels.cuh"
#include "tc_common.cuh"

#include <cudaTypedefs.h>

#include <mutex>
#include <type_traits>

namespace lga {
namespace fat {

using namespace tcu;

constexpr int BQ = 128, BKV = 128;
constexpr int SM_WARPS = 8;                    // softmax warps: 2 per TMEM lane quadrant, 64 key columns each
constexpr int EPI_WARPS = 4;                   // one per TMEM lane quadrant
constexpr int NT = (4 + SM_WARPS + EPI_WARPS) * 32;
constexpr int SM_THREADS = SM_WARPS * 32;
constexpr int EPI_THREADS = EPI_WARPS * 32;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.0f;   // log2 units
#ifndef LGA_POLY_PAIRS
#define LGA_POLY_PAIRS 3
#endif
constexpr int POLY_PAIRS = LGA_POLY_PAIRS;  // of every 8 exponent pairs, computed by polynomial (FMA pipe)

#ifdef LGA_FWD_TRACE
// Timing-only instrumentation (development builds): clock64() at pipeline events of CTA 0's first item.
__device__ long long g_fwd_trace[40][8];
__device__ long long g_fwd_items[64][4];   // CTA 0 per item: MMA item start, last PV issued, epilogue start / end
__device__ long long g_fwd_cta[256][2];    // %globaltimer (ns) at each CTA's start and end
__device__ __forceinline__ long long globaltimer_ns() {
  long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
#define FTR(j, k) \
  if (blockIdx.x == 0 && t == 0 && (j) < 40) g_fwd_trace[j][k] = clock64()
#define FIT(i, k) \
  if (blockIdx.x == 0 && (i) < 64) g_fwd_items[i][k] = clock64()
#else
#define FTR(j, k)
#define FIT(i, k)
#endif

template <int DH>
struct FwdSmem {
  static constexpr int TILE = BQ * DH * 2;          // [128][DH] bf16 as DH/64 swizzled [128][64] sub-tiles
  static constexpr int SUB = 128 * 64 * 2;          // 16 KB
  static constexpr int NK = 3, NV = 2;              // K ring (freed when S completes), V ring (freed after PV)
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE;        // [NK]
  static constexpr int V_OFF = K_OFF + NK * TILE;   // [NV]
  static constexpr int STG_OFF = V_OFF + NV * TILE; // O staging: [128 rows][64 cols] bf16, 128B-swizzled (TMA store)
  static constexpr int RED_OFF = STG_OFF + SUB;     // [2 items][2 halves][128 rows] maxima, then [2][128] sums
  static constexpr int BAR_OFF = RED_OFF + 2 * 4 * 128 * 4;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  static_assert(TOTAL <= 232448, "shared memory");
};

template <int DH>
__global__ void __launch_bounds__(NT, 1) fwd_kernel(const __grid_constant__ CUtensorMap tm,
                                                     const __grid_constant__ CUtensorMap tmo, const AttnArgs a) {
  using SM = FwdSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  constexpr int NK = SM::NK, NV = SM::NV;
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = q_full + 1;       // [NK]
  uint64_t* k_empty = k_full + NK;     // [NK]
  uint64_t* v_full = k_empty + NK;     // [NV]
  uint64_t* v_empty = v_full + NV;     // [NV]
  uint64_t* s_full = v_empty + NV;     // [2]
  uint64_t* p_full = s_full + 2;       // [2 buffers][2 halves] (SM_THREADS/2 arrivals each).  Per buffer: P(g+2)
                                       // needs S(g+2), issued after PV(g), so a half can never be two phases
                                       // ahead of the MMA warp's wait (one barrier per half could: S(g+1) is
                                       // issued before P(g) is awaited)
  uint64_t* o_done = p_full + 4;       // [2 halves]
  uint64_t* q_empty = o_done + 2;      // Q buffer free (all S MMAs of an item done)
  uint64_t* o_free = q_empty + 1;      // O accumulators read by the epilogue (EPI_THREADS arrivals)
  uint64_t* p_free = o_free + 1;       // [2] per S / P TMEM buffer: PV of the tile in it done
  uint64_t* ml_full = p_free + 2;      // [2 items] row maxima / sums of an item in red (SM_THREADS arrivals)
  uint64_t* ml_empty = ml_full + 2;    // [2 items] red read by the epilogue (EPI_THREADS arrivals)
  constexpr int NBAR = 1 + 2 * NK + 2 * NV + 16;
  static_assert(NBAR * 8 + 4 <= 256, "barrier area");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LGA_FWD_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 256) g_fwd_cta[blockIdx.x][0] = globaltimer_ns();
#endif
  const int s = a.seq, d = a.d;
  const int nqt = (s + BQ - 1) / BQ;
  const int per_q = a.heads * a.nseq;
  const int n_items = nqt * per_q;
  const int nkv_all = (s + BKV - 1) / BKV;
  // work item t -> (query tile, head, sequence).  Items come in chunks of G (sequence, head) pairs, all
  // query tiles of a chunk together (heaviest first under causal masking), so the CTAs running at any time
  // share each pair's K / V tiles in L2 instead of streaming every tile from HBM once per query tile.
#ifndef LGA_FWD_G
#define LGA_FWD_G 16
#endif
  constexpr int G = LGA_FWD_G;
  auto item = [&](int t, int& qt, int& h, int& sq, int& nkv) {
    const int chunk = t / (G * nqt), w = t % (G * nqt);
    const int np = min(G, per_q - chunk * G);   // pairs in this chunk (the last may be partial)
    const int qi = w / np, pair = chunk * G + w % np;
    qt = a.causal ? nqt - 1 - qi : qi;
    h = pair % a.heads;
    sq = pair / a.heads;
    nkv = a.causal ? min(nkv_all, (qt * BQ + BQ - 1) / BKV + 1) : nkv_all;
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NBAR; ++i) {
      uint32_t cnt = 1;
      if (&bars[i] == o_free || &bars[i] == ml_empty || &bars[i] == ml_empty + 1) cnt = EPI_THREADS;
      if (&bars[i] == ml_full || &bars[i] == ml_full + 1) cnt = SM_THREADS;
      if (&bars[i] >= p_full && &bars[i] < p_full + 4) cnt = SM_THREADS / 2;
      mbar_init(&bars[i], cnt);   // softmax threads arrive individually
    }
    mbar_fence_init();
    prefetch_tmap(&tm);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t t_o[2] = {tbase + 256, tbase + 256 + DH};   // one O accumulator per key half (DH <= 128)

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer: Q and K
      int jt = 0;     // global KV tile counter (ring stage / phase)
      int it = 0;
      for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
        int qt, h, sq, nkv;
        item(t, qt, h, sq, nkv);
        mbar_wait(q_empty, (it & 1) ^ 1);
        mbar_expect_tx(q_full, SM::TILE);
#pragma unroll
        for (int i = 0; i < DH / 64; ++i)
          tma_load_3d(smem + SM::Q_OFF + i * SM::SUB, &tm, q_full, h * DH + 64 * i, qt * BQ, sq);
        for (int j = 0; j < nkv; ++j, ++jt) {
          const int st = jt % NK;
          mbar_wait(&k_empty[st], ((jt / NK) & 1) ^ 1);
          mbar_expect_tx(&k_full[st], SM::TILE);
#pragma unroll
          for (int i = 0; i < DH / 64; ++i)
            tma_load_3d(smem + SM::K_OFF + st * SM::TILE + i * SM::SUB, &tm, &k_full[st], d + h * DH + 64 * i, j * BKV, sq);
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ===== TMA producer: V
      int jt = 0;
      for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
        int qt, h, sq, nkv;
        item(t, qt, h, sq, nkv);
        for (int j = 0; j < nkv; ++j, ++jt) {
          const int st = jt % NV;
          mbar_wait(&v_empty[st], ((jt / NV) & 1) ^ 1);
          mbar_expect_tx(&v_full[st], SM::TILE);
#pragma unroll
          for (int i = 0; i < DH / 64; ++i)
            tma_load_3d(smem + SM::V_OFF + st * SM::TILE + i * SM::SUB, &tm, &v_full[st], 2 * d + h * DH + 64 * i,
                        j * BKV, sq);
        }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer (whole warp; one elected lane issues)
    constexpr uint32_t idesc_s = make_idesc(128, BKV, false, false);
    constexpr uint32_t idesc_o = make_idesc(128, DH, false, true);
    const bool leader = elect_one();
    const uint64_t dQ = make_desc(smem_u32(smem + SM::Q_OFF), 16, 1024);
    const uint64_t dK = make_desc(smem_u32(smem + SM::K_OFF), 16, 1024);
    const uint64_t dVm = make_desc(smem_u32(smem + SM::V_OFF), SM::SUB, 1024);   // MN-major: d_h blocks at 16 KB
    int js = 0;   // global S / KV tile counter
    int it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int qt, h, sq, nkv;
      item(t, qt, h, sq, nkv);
      mbar_wait(q_full, it & 1);
      if (lane == 0) FIT(it, 0);
      const int j0 = js;   // global index of this item's first tile
      for (int j = 0; j <= nkv; ++j) {
        if (j < nkv) {
          const int g = j0 + j, st = g % NK, b = g & 1;
          mbar_wait(&k_full[st], (g / NK) & 1);
          if (g >= 2) mbar_wait(&p_free[b], ((g - 2) >> 1) & 1);   // buffer b holds P(g-2) until PV(g-2) read it
          fence_after();
          const uint64_t dk = desc_add(dK, st * SM::TILE);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t off = (kk >> 2) * SM::SUB + (kk & 3) * 32;
              umma_f16(tbase + 128 * b, desc_add(dQ, off), desc_add(dk, off), idesc_s, kk > 0);
            }
            umma_commit(&s_full[b]);
            umma_commit(&k_empty[st]);
            if (j == nkv - 1) umma_commit(q_empty);
          }
          __syncwarp();
        }
        if (j >= 1) {
          const int jj = j - 1, g = j0 + jj, st = g % NV, pb = g & 1;
          if (jj == 0) mbar_wait(o_free, (it & 1) ^ 1);
          mbar_wait(&v_full[st], (g / NV) & 1);
          const uint64_t dv = desc_add(dVm, st * SM::TILE);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            mbar_wait(&p_full[pb * 2 + hh], (g >> 1) & 1);
            fence_after();
            if (leader) {
#pragma unroll
              for (int kk = 4 * hh; kk < 4 * hh + 4; ++kk)
                umma_f16_ts(t_o[hh], tbase + 128 * pb + 64 * hh + 8 * (kk & 3), desc_add(dv, kk * 16 * 128), idesc_o,
                            (jj > 0 || kk > 4 * hh) ? 1u : 0u);
              umma_commit(&o_done[hh]);
            }
            __syncwarp();
          }
          if (leader) {
            umma_commit(&v_empty[st]);
            umma_commit(&p_free[pb]);
            if (jj == nkv - 1) FIT(it, 1);
          }
          __syncwarp();
        }
      }
      js += nkv;
    }
  } else if (warp >= 4 && warp < 4 + SM_WARPS) {  // ===== softmax: one query row and one key half per thread
    const int qd = warp & 3;
    const int hf = (warp - 4) >> 2;            // key half of every tile this warp owns
    const int r = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    float* red = reinterpret_cast<float*>(smem + SM::RED_OFF);
    int gt = 0;   // global tile counter
    int its = 0;  // item counter
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++its) {
      int qt, h, sq, nkv;
      item(t, qt, h, sq, nkv);
      const int q0 = qt * BQ, q = q0 + r;
      float m_used = -INFINITY, l = 0.f;        // running max (log2 units) and sum of this half
      for (int j = 0; j < nkv; ++j, ++gt) {
        const int b = gt & 1;
        mbar_wait(&s_full[b], (gt >> 1) & 1);
        if (warp == 4 && lane == 0) FTR(j, 3);
        fence_after();
        const int k0 = j * BKV + hf * 64;
        if ((k0 >= s) || (a.causal && k0 > q0 + qd * 32 + 31)) {
          // (warp-uniform) every key of this half is past the sequence end or after the warp's 32 queries --
          // on the causal diagonal half of the warps: P = 0, max and sum unchanged
          uint32_t z[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) z[c] = 0u;
          tmem_st32_u(tbase + 128 * b + lane_off + hf * 64, z);
          tmem_wait_st();
          fence_before();
          mbar_arrive(&p_full[b * 2 + hf]);
          continue;
        }
        uint32_t raw[2][32];
        tmem_ld32_nowait(tbase + 128 * b + lane_off + hf * 64, raw[0]);
        tmem_ld32_nowait(tbase + 128 * b + lane_off + hf * 64 + 32, raw[1]);
        tmem_wait_ld();
        // masking only where a key can be past the sequence end or after the query (uniform per warp)
        const bool need_mask = (k0 + 64 > s) || (a.causal && k0 + 63 > q0 + qd * 32);
        float sv[64];
#pragma unroll
        for (int c = 0; c < 64; ++c) sv[c] = __uint_as_float(raw[c >> 5][c & 31]);
        if (need_mask) {
          const int lim = a.causal ? min(s - 1, q) - k0 : s - 1 - k0;   // last unmasked column
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c > lim) sv[c] = -INFINITY;
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // 4 independent chains
#pragma unroll
        for (int c = 0; c < 64; c += 2) m4[(c >> 1) & 3] = fmax3(m4[(c >> 1) & 3], sv[c], sv[c + 1]);
        float mx = fmax3(m4[0], m4[1], fmaxf(m4[2], m4[3]));
        mx *= sl2;
        const float m_new = (mx > m_used + RESCALE_THRESHOLD) ? mx : m_used;
        const float moff = m_new == -INFINITY ? 0.f : -m_new;   // fully masked so far: every p is 2^-inf = 0
        uint32_t pk[32];
        uint64_t r2[2] = {0, 0};   // packed partial row sums
        const uint64_t SL2 = f2pack(sl2, sl2), MO = f2pack(moff, moff);
        // p = 2^(s*scale*log2e - m): on the SFU, except (unmasked tiles) POLY_PAIRS of every 8 pairs on the
        // FMA pipe -- the SFU alone takes 8 cycles per warp instruction and bounds the tile otherwise
        auto exps = [&](auto poly_on) {
#pragma unroll
          for (int pi = 0; pi < 32; ++pi) {
            const uint64_t x = f2fma(f2pack(sv[2 * pi], sv[2 * pi + 1]), SL2, MO);
            float p0, p1;
            if (decltype(poly_on)::value && (pi & 7) < POLY_PAIRS) {
              ex2_poly2(x, p0, p1);
            } else {
              float x0, x1;
              f2unpack(x, x0, x1);
              p0 = ex2(x0), p1 = ex2(x1);
            }
            r2[pi & 1] = f2add(r2[pi & 1], f2pack(p0, p1));
            pk[pi] = pack_bf16x2(p0, p1);
          }
        };
        if (need_mask) exps(std::false_type{});   // masked scores are -inf: the SFU gives exactly 0
        else exps(std::true_type{});
        float ra, rb, rc, rd;
        f2unpack(r2[0], ra, rb);
        f2unpack(r2[1], rc, rd);
        const float rs = (ra + rb) + (rc + rd);
        if (warp == 4 && lane == 0) FTR(j, 4);
        // lazy rescale of this half's accumulator row, once PV(j-1) has finished accumulating into it (the
        // parity wait is safe at any time: s_full(j) implies PV(j-2) complete).  tcgen05.ld / st are
        // warp-collective, so the whole warp enters when any lane needs it; other lanes multiply by 1.
        const bool resc = m_new != m_used && m_used != -INFINITY;
        const float scale = resc ? ex2(m_used - m_new) : 1.f;
        if (__any_sync(0xffffffffu, resc)) {
          mbar_wait(&o_done[hf], (gt - 1) & 1);
          fence_after();
#pragma unroll 1
          for (int c = 0; c < DH / 32; ++c) {
            float tt[32];
            tmem_ld32(t_o[hf] + lane_off + c * 32, tt);
#pragma unroll
            for (int i = 0; i < 32; ++i) tt[i] *= scale;
            tmem_st32(t_o[hf] + lane_off + c * 32, tt);
          }
        }
        if (warp == 4 && lane == 0) FTR(j, 5);
        l = l * scale + rs;
        m_used = m_new;
        // P (bf16, two keys per column) over the first 32 of this thread's own 64 S columns
        tmem_st32_u(tbase + 128 * b + lane_off + hf * 64, pk);
        tmem_wait_st();
        fence_before();
        if (warp == 4 && lane == 0) FTR(j, 6);
        if (warp == 8 && lane == 0) FTR(j, 7);
        mbar_arrive(&p_full[b * 2 + hf]);
      }
      // hand the row's (max, sum) of this half to the epilogue warps (double-buffered by item)
      const int ib = its & 1;
      mbar_wait(&ml_empty[ib], ((its >> 1) & 1) ^ 1);
      red[ib * 512 + hf * 128 + r] = m_used;
      red[ib * 512 + 256 + hf * 128 + r] = l;
      mbar_arrive(&ml_full[ib]);
    }
  } else if (warp >= 4 + SM_WARPS) {  // ===== epilogue: o = (2^(m0-m) O_0 + 2^(m1-m) O_1) / (2^(m0-m) l_0 + 2^(m1-m) l_1), one row per thread
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const float* red = reinterpret_cast<const float*>(smem + SM::RED_OFF);
    uint8_t* stg = smem + SM::STG_OFF;
    const bool issuer = warp == 4 + SM_WARPS && lane == 0;
    int gt = 0, it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int qt, h, sq, nkv;
      item(t, qt, h, sq, nkv);
      gt += nkv;
      const int q0 = qt * BQ, q = q0 + r;
      const int ib = it & 1;
      mbar_wait(&ml_full[ib], (it >> 1) & 1);
      if (issuer) FIT(it, 2);
      const float m0 = red[ib * 512 + r], m1 = red[ib * 512 + 128 + r];
      const float l0 = red[ib * 512 + 256 + r], l1 = red[ib * 512 + 384 + r];
      mbar_arrive(&ml_empty[ib]);
      // every PV of the item done: O final.  ml_full implies S(gt-1), issued after PV(gt-3) completed, so
      // o_done may be anywhere from PV(gt-3) to PV(gt-1) -- three states a parity wait cannot tell apart.  First
      // PV(gt-2) through its buffer's p_free (at PV(gt-4) or PV(gt-2); PV(gt) needs this item's o_free), then
      // o_done is at most one phase from PV(gt-1).
      if (gt >= 2) mbar_wait(&p_free[gt & 1], ((gt - 2) >> 1) & 1);
      mbar_wait(&o_done[0], (gt - 1) & 1);
      mbar_wait(&o_done[1], (gt - 1) & 1);
      fence_after();
      const float mm = fmaxf(m0, m1);
      const float f0 = m0 == -INFINITY ? 0.f : ex2(m0 - mm), f1 = m1 == -INFINITY ? 0.f : ex2(m1 - mm);
      const float lt = f0 * l0 + f1 * l1;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      const float g0 = f0 * inv, g1 = f1 * inv;
      // O through the swizzled [128][64] staging tile, one 64-column half at a time (TMA clips rows past s);
      // the accumulators are released after the last half's TMEM loads
#pragma unroll
      for (int hh = 0; hh < DH / 64; ++hh) {
        uint32_t pk[32];   // 64 columns of the row, bf16 pairs
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t u0[16], u1[16];
          tmem_ld16_nowait(t_o[0] + lane_off + hh * 64 + c * 16, u0);
          tmem_ld16_nowait(t_o[1] + lane_off + hh * 64 + c * 16, u1);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            pk[c * 8 + i] = pack_bf16x2(g0 * __uint_as_float(u0[2 * i]) + g1 * __uint_as_float(u1[2 * i]),
                                        g0 * __uint_as_float(u0[2 * i + 1]) + g1 * __uint_as_float(u1[2 * i + 1]));
        }
        if (hh == DH / 64 - 1) {
          fence_before();
          mbar_arrive(o_free);   // the next item's first PV may overwrite the accumulators
        }
        if (issuer) bulk_wait_read0();   // the previous store has read the staging tile
        asm volatile("bar.sync 2, %0;" ::"n"(EPI_THREADS) : "memory");
        uint8_t* row = stg + r * 128;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<uint4*>(row + ((k ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
        fence_proxy_async();
        asm volatile("bar.sync 2, %0;" ::"n"(EPI_THREADS) : "memory");
        if (issuer) {
          tma_store_3d(&tmo, stg, h * DH + 64 * hh, q0, sq);
          bulk_commit();
        }
      }
      if (q < s) a.lse[((int64_t)sq * a.heads + h) * s + q] = (mm + log2f(lt)) * 0.6931471805599453f;
      if (issuer) FIT(it, 3);
    }
    if (issuer) bulk_wait0();
  }
  fence_before();
  __syncthreads();
#ifdef LGA_FWD_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 256) g_fwd_cta[blockIdx.x][1] = globaltimer_ns();
#endif
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tbase, 512);
  }
}

template <int DH>
static cudaError_t run_fwd(const AttnArgs& a, cudaStream_t st) {
  CUtensorMap tm, tmo;
  cudaError_t e = map3d_bf16(&tm, a.qkv, 3ull * a.d, a.seq, a.nseq, 128);
  if (e != cudaSuccess) return e;
  e = map3d_bf16(&tmo, a.o, a.d, a.seq, a.nseq, 128);
  if (e != cudaSuccess) return e;
  static bool set = false;
  if (!set) {
    e = cudaFuncSetAttribute(fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem<DH>::TOTAL);
    if (e != cudaSuccess) return e;
    set = true;
  }
  const int items = ((a.seq + BQ - 1) / BQ) * a.heads * a.nseq;
  note_launch(), fwd_kernel<DH><<<std::min(items, num_sms()), NT, FwdSmem<DH>::TOTAL, st>>>(tm, tmo, a);
  return cudaGetLastError();
}

}  // namespace fat

#ifdef LGA_FWD_TRACE
extern "C" int lgatest_fwd_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fat::g_fwd_trace, sizeof(fat::g_fwd_trace));
}
extern "C" int lgatest_fwd_trace_items(long long* items, long long* cta) {
  cudaError_t e = cudaMemcpyFromSymbol(items, fat::g_fwd_items, sizeof(fat::g_fwd_items));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(cta, fat::g_fwd_cta, sizeof(fat::g_fwd_cta));
  return (int)e;
}
#endif

cudaError_t attn_fwd_bf16(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return cudaSuccess;
  return a.dh == 64 ? fat::run_fwd<64>(a, st) : fat::run_fwd<128>(a, st);
}

}  // namespace lga
