// k_attn_tc_bwd.cu -- causal multi-head attention backward on the 5th-generation tensor cores (sm_100a).
//
// O5 of DESIGN.md with P recomputed from the saved log-sum-exp (flash-style), no float atomics:
//   dsum_i = rowsum(dO_i * o_i)
//   dK/dV kernel, one CTA per 128-key tile, looping over 64-query tiles:
//     S^T = K Q^T, dP^T = V dO^T            (tcgen05, M=128 keys, N=64 queries, K=d_h; TMEM, 2 buffers)
//     P^T = exp(S^T*scale - lse), dS^T = P^T (dP^T - dsum) * scale   (element-wise warps, bf16 into TMEM)
//     dV += P^T dO, dK += dS^T Q              (tcgen05, A = P^T / dS^T from TMEM, B = dO / Q read MN-major
//                                              from the very tiles TMA loaded K-major for the first two MMAs)
//     with a dS workspace (a.dsT) the element-wise warps also store dS^T (bf16, 32-byte sectors), and
//   dQ = dS K is a persistent, causally blocked batched GEMM over it (dq_from_ds_kernel; 5 matmuls per block);
//   without one, the dQ kernel (one CTA per 128-query tile, looping over 128-key tiles) recomputes
//     S = Q K^T, dP = dO V^T ; dS = P (dP - dsum) * scale ; dQ += dS K   (dS from TMEM, K read MN-major)
// P / dS never touch shared memory, which goes to deeper Q/dO (K/V) rings: the load latency, not the
// tensor pipe, bounded the smem-staged version (MMA issuer stalled on the ring's full barrier).
// Warp roles: 0 TMA, 1 MMA issuer, 2 TMEM allocator, 4..19 element-wise (two ping-pong groups) + epilogue.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace lga {
namespace fatb {

using namespace tcu;

constexpr int EW_WARPS = 16;                // element-wise warps: two ping-pong groups of 8
constexpr int GRP_THREADS = EW_WARPS * 16;  // threads per group
constexpr int NT = (4 + EW_WARPS) * 32;
#ifndef LGA_BWD_NST_DKV64      // ring depths (overridable for experiments)
#define LGA_BWD_NST_DKV64 6
#endif
#ifndef LGA_BWD_NST_DKV128
#define LGA_BWD_NST_DKV128 4
#endif
#ifndef LGA_BWD_NST_DQ64
#define LGA_BWD_NST_DQ64 4
#endif
#ifndef LGA_BWD_NST_DQ128
#define LGA_BWD_NST_DQ128 2
#endif
constexpr float LOG2E = 1.4426950408889634f;
#ifndef LGA_BWD_POLY
#define LGA_BWD_POLY 0
#endif
// of every 8 exponent pairs of an unmasked tile, computed by the FMA-pipe polynomial instead of the SFU (as in
// the forward).  Measured on the 1.3B shapes (kbench, backward): 0 / 2 / 3 / 4 pairs -> 1.094 / 1.093 / 1.105 /
// 1.111 ms -- the backward's element-wise phase is not SFU-bound, so the default keeps every 2^x on the SFU
constexpr int BWD_POLY = LGA_BWD_POLY;

// rowsum(dO * o) per (sequence, head, position): d_h / 16 lanes per row, 32 bytes of o and of dO per lane (two
// 16-byte loads each, all four issued before the math), shuffle reduction within the lane group
__global__ void __launch_bounds__(256) dsum_kernel(AttnArgs a) {
  const int lph = a.dh >> 4;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid / lph;   // token * heads + h
  const int part = (int)(gid % lph);
  const bool valid = row < (int64_t)a.nseq * a.seq * a.heads;
  float acc = 0.f;
  int h = 0;
  int64_t tok = 0;
  if (valid) {
    h = (int)(row % a.heads);
    tok = row / a.heads;
    const int64_t off = tok * a.d + (int64_t)h * a.dh + part * 16;
    const uint4* po = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.o) + off);
    const uint4* pg = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.dO) + off);
    const uint4 x0 = po[0], x1 = po[1], y0 = pg[0], y1 = pg[1];
    const uint32_t xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    const uint32_t ys[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      acc = fmaf(__uint_as_float(xs[i] << 16), __uint_as_float(ys[i] << 16), acc);
      acc = fmaf(__uint_as_float(xs[i] & 0xFFFF0000u), __uint_as_float(ys[i] & 0xFFFF0000u), acc);
    }
  }
  for (int o = lph >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (valid && part == 0) a.dsum[((tok / a.seq) * a.heads + h) * a.seq + tok % a.seq] = acc;
}

// TMEM row -> bf16 global row.  tcgen05.ld is warp-collective: every lane executes it, only
// lanes with `valid` store.  csum != nullptr: also the column sums over the warp's 32 rows (invalid rows count
// 0) into csum[0 .. ncols) -- this warp's partial of the qkv bias gradient (fp32, before the bf16 rounding).
__device__ __forceinline__ void store_row_bf16_global(__nv_bfloat16* dst, uint32_t taddr, int ncols, float scale,
                                                      bool valid, float* csum = nullptr) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < ncols; c += 16) {   // ncols is a multiple of 16
    uint32_t r[16];
    tmem_ld16_nowait(taddr + c, r);
    tmem_wait_ld();
    if (csum) {
      float w[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) w[i] = valid ? __uint_as_float(r[i]) * scale : 0.f;
      const float cs = warp_colsum16(w);
      if (lane < 16) csum[c + lane] = cs;
    }
    if (!valid) continue;
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * scale, __uint_as_float(r[2 * i + 1]) * scale);
    // 16 columns = one full 32-byte sector per lane (rows are one per lane: a 16-byte store would cost the
    // same number of L1 wavefronts for half the bytes); dst + c is 32-byte aligned
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst + c), "r"(pk[0]), "r"(pk[1]),
                 "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7])
                 : "memory");
  }
}

#ifdef LGA_BWD_TRACE
// Timing-only instrumentation (development builds): SM clock64() at pipeline events of the 16 dK/dV CTAs
// of (sequence 0, head 0): [kt][i][event], row 39 = CTA start / K,V landed / end; dQ kernel: CTA 0 of
// (sequence 0, head 0) into g_dq_trace[j][event].
__device__ long long g_bwd_trace[16][40][8];
__device__ long long g_dq_trace[40][8];
#define BTR(i, k) \
  if (blockIdx.y == 0 && blockIdx.z == 0 && blockIdx.x < 16) g_bwd_trace[blockIdx.x][i][k] = clock64()
#define QTR(j, k) \
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 40) g_dq_trace[j][k] = clock64()
#else
#define BTR(i, k)
#define QTR(j, k)
#endif
#ifdef LGA_DKV_TRACE
// Timing-only instrumentation (development builds): clock64() per global iteration g < 96 of CTA 0 of the
// persistent dK/dV kernel: [g][0] S^T issued, [1] dP^T issued, [2] element-wise group saw s_full, [3] P / dS
// arrived, [4] dV issued, [5] dK issued; per item [it][0] drain start, [1] drain end, [2] MMA item start.
__device__ long long g_dkv_trace[96][8];
__device__ long long g_dkv_items[32][4];
#define DTR(g, k) \
  if (blockIdx.x == 0 && (g) < 96) g_dkv_trace[g][k] = clock64()
#define DIT(i, k) \
  if (blockIdx.x == 0 && (i) < 32) g_dkv_items[i][k] = clock64()
#else
#define DTR(g, k)
#define DIT(i, k)
#endif

// 4-byte cp.async global -> shared (zero-filled when !valid) and its completion arriving on an mbarrier
// (.noinc: the barrier's expected count includes one arrival per issuing thread)
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The element-wise warps form two ping-pong groups of 8 (2 per TMEM lane quadrant, 32 columns each):
// group g handles iterations i = g, g+2, ... with its own TMEM S/dP buffer, smem P/dS buffer and
// s_empty / p_full barriers, so one group's load -> exp -> store -> arrive latency chain overlaps the
// other's; the MMA warp issues S(i) two iterations ahead of the gradient MMAs of iteration i-2.
// After the loop every group needs all gradient MMAs done: wait this group's last commit first (its own
// barrier, so the parity wait cannot alias an older phase), then the very last one.
__device__ __forceinline__ void wait_all_done(uint64_t* g_done, int grp, int n) {
  const int own = n - 1 >= grp ? n - 1 - ((n - 1 - grp) & 1) : -1;
  if (own >= 0) mbar_wait(&g_done[grp], (own >> 1) & 1);
  if (own != n - 1) mbar_wait(&g_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
  fence_after();
}

// =============================================================================== dK / dV
// TMEM (512 columns): S^T[2] at 0 / 64, dP^T[2] at 128 / 192, dV at 256, dK at 256 + DH.
// The element-wise thread owning key row r and query columns [32h, 32h+32) of buffer b writes the bf16
// P^T (dS^T) of those 32 queries, packed two per column, over the first 16 of the S^T (dP^T) columns it
// has just read; the gradient MMAs read them as their TMEM A operand.  The MMA issuer therefore issues
// S^T(i+2) into buffer b only after the gradient MMAs of iteration i have completed.
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
  static constexpr int NST = DH == 64 ? LGA_BWD_NST_DKV64 : LGA_BWD_NST_DKV128;   // Q / dO / lse / dsum ring
  static constexpr int Q_OFF = V_OFF + KT;             // [NST]
  static constexpr int G_OFF = Q_OFF + NST * QT;       // dO [NST]
  static constexpr int LD_OFF = G_OFF + NST * QT;      // [NST] x {lse[64], dsum[64]} fp32
  static constexpr int BAR_OFF = LD_OFF + NST * 512;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

// Persistent: one CTA per SM loops over work items (key tile, head, sequence) in chunks of DKV_G (sequence,
// head) pairs -- the Q / dO tiles of a chunk stay in L2 -- with the heaviest key tiles (most queries after
// them under the causal mask) first.  Everything per item is pipelined across items: the Q / dO ring,
// the S^T / dP^T TMEM buffers and the element-wise groups run on GLOBAL iteration counters; the next item's
// K / V tiles are loaded as soon as the current item's last S^T / dP^T MMAs have read them (kv_empty), and
// its first S^T / dP^T MMAs run while the element-wise warps drain the previous item's dK / dV from TMEM;
// only its first dV / dK MMAs wait for that drain (acc_free).
#ifndef LGA_DKV_G
#define LGA_DKV_G 4
#endif
constexpr int DKV_G = LGA_DKV_G;

template <int DH>
__global__ void __launch_bounds__(NT, 1)
    dkdv_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                const __grid_constant__ CUtensorMap tm_g, const AttnArgs a) {
  using SM = DkvSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  constexpr int NST = SM::NST;
  constexpr int EW_ALL = EW_WARPS * 32;
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;              // [NST] (expect_tx + 32 cp.async arrivals)
  uint64_t* q_empty = q_full + NST;         // [NST]
  uint64_t* s_full = q_empty + NST;         // [2] per group / TMEM buffer
  uint64_t* p_full = s_full + 2;            // [2] (GRP_THREADS arrivals)
  uint64_t* g_done = p_full + 2;            // [2]
  uint64_t* kv_empty = g_done + 2;          // K / V read by the item's last S^T / dP^T MMAs
  uint64_t* acc_free = kv_empty + 1;        // dK / dV drained from TMEM by every element-wise thread
  uint64_t* dv_done = acc_free + 1;         // [2] the dV MMAs of an iteration done (P^T read)
  constexpr int NBAR = 2 * NST + 11;
  static_assert(NBAR * 8 + 4 <= 256, "barrier area");
  static_assert(SM::TOTAL <= 232448, "shared memory");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.seq, d = a.d;
  const int nkt = (s + KB - 1) / KB;
  const int nq_all = (s + QB - 1) / QB;
  const int pairs = a.heads * a.nseq;
  const int n_items = nkt * pairs;
  // work item t -> key tile, head, sequence; its query iterations start at qstart (causal: the diagonal)
  auto item = [&](int t, int& kt, int& h, int& sq, int& qstart, int& nq) {
    const int chunk = t / (DKV_G * nkt), w = t % (DKV_G * nkt);
    const int np = min(DKV_G, pairs - chunk * DKV_G);
    kt = w / np;   // ascending: heaviest first under causal masking
    const int pair = chunk * DKV_G + w % np;
    h = pair % a.heads;
    sq = pair / a.heads;
    qstart = a.causal ? kt * KB / QB : 0;
    nq = nq_all - qstart;
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NBAR; ++i) {
      const bool qf = (&bars[i] >= q_full && &bars[i] < q_empty);
      const bool ew = (&bars[i] >= p_full && &bars[i] < g_done);
      mbar_init(&bars[i], qf ? 33 : ew ? GRP_THREADS : (&bars[i] == acc_free ? EW_ALL : 1));
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
  auto t_st = [&](int b) { return tb + 64 * b; };
  auto t_dpt = [&](int b) { return tb + 128 + 64 * b; };
  const uint32_t t_dv = tb + 256, t_dk = tb + 256 + DH;

  if (warp == 0) {  // ===== producer: TMA (lane 0) + lse / dsum cp.async (all lanes)
    int gi = 0, it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int kt, h, sq, qstart, nq;
      item(t, kt, h, sq, qstart, nq);
      const int k0 = kt * KB;
      const int rb = (sq * a.heads + h) * s;   // row base of lse / dsum
      if (lane == 0) {
        mbar_wait(kv_empty, (it & 1) ^ 1);   // the previous item's S^T / dP^T MMAs have read K / V
        mbar_expect_tx(kv_full, 2 * SM::KT);
#pragma unroll
        for (int i = 0; i < DH / 64; ++i) {
          tma_load_3d(smem + SM::K_OFF + i * SM::SUB128, &tm_kv, kv_full, d + h * DH + 64 * i, k0, sq);
          tma_load_3d(smem + SM::V_OFF + i * SM::SUB128, &tm_kv, kv_full, 2 * d + h * DH + 64 * i, k0, sq);
        }
      }
      for (int i = 0; i < nq; ++i, ++gi) {
        const int st = gi % NST;
        const int q0 = (qstart + i) * QB;
        mbar_wait(&q_empty[st], ((gi / NST) & 1) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&q_full[st], 2 * SM::QT);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c) {
            tma_load_3d(smem + SM::Q_OFF + st * SM::QT + c * SM::SUB64, &tm_q, &q_full[st], h * DH + 64 * c, q0, sq);
            tma_load_3d(smem + SM::G_OFF + st * SM::QT + c * SM::SUB64, &tm_g, &q_full[st], h * DH + 64 * c, q0, sq);
          }
        }
        // lse / dsum of the 64 queries (zero past the sequence end; those queries are masked)
        float* ld = reinterpret_cast<float*>(smem + SM::LD_OFF + st * 512);
#pragma unroll
        for (int e = lane; e < 128; e += 32) {
          const int q = q0 + (e & 63);
          cp_async4(ld + e, (e < 64 ? a.lse : a.dsum) + rb + min(q, s - 1), q < s);
        }
        cp_async_mbar_arrive(&q_full[st]);
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer (whole warp; one elected lane issues)
    constexpr uint32_t idesc_s = make_idesc(128, QB, false, false);
    constexpr uint32_t idesc_g = make_idesc(128, DH, false, true);
    const bool leader = elect_one();
    const uint64_t dK = make_desc(smem_u32(smem + SM::K_OFF), 16, 1024);
    const uint64_t dV = make_desc(smem_u32(smem + SM::V_OFF), 16, 1024);
    const uint64_t dQk = make_desc(smem_u32(smem + SM::Q_OFF), 16, 1024);          // Q, K-major
    const uint64_t dGk = make_desc(smem_u32(smem + SM::G_OFF), 16, 1024);          // dO, K-major
    const uint64_t dQm = make_desc(smem_u32(smem + SM::Q_OFF), SM::SUB64, 1024);   // Q, MN-major
    const uint64_t dGm = make_desc(smem_u32(smem + SM::G_OFF), SM::SUB64, 1024);   // dO, MN-major
    int gi = 0, it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int kt, h, sq, qstart, nq;
      item(t, kt, h, sq, qstart, nq);
      // S^T(g) = K Q^T, dP^T(g) = V dO^T into buffer g & 1 (global iteration g = local i of this item), once
      // the gradient MMAs of iteration g - 2 have consumed the P^T / dS^T that buffer held
      // S^T(g) only overwrites P^T(g-2), read by the dV MMAs, and dP^T(g) only dS^T(g-2), read by the dK MMAs:
      // S^T(g) is issued as soon as dV(g-2) is done, so it queues behind dK(g-2) on the tensor pipe instead of
      // the pipe idling while the issuer waits for both
      auto issue_s = [&](int g, int i) {
        const int st = g % NST, b = g & 1;
        mbar_wait(&q_full[st], (g / NST) & 1);
        if (g >= 2) mbar_wait(&dv_done[b], ((g - 2) >> 1) & 1);
        fence_after();
        const uint64_t dq = desc_add(dQk, st * SM::QT), dg = desc_add(dGk, st * SM::QT);
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * SM::SUB128 + (kk & 3) * 32, ob = (kk >> 2) * SM::SUB64 + (kk & 3) * 32;
            umma_f16(t_st(b), desc_add(dK, oa), desc_add(dq, ob), idesc_s, kk > 0);
          }
          DTR(g, 0);
        }
        __syncwarp();
        if (g >= 2) mbar_wait(&g_done[b], ((g - 2) >> 1) & 1);
        fence_after();
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            const uint32_t oa = (kk >> 2) * SM::SUB128 + (kk & 3) * 32, ob = (kk >> 2) * SM::SUB64 + (kk & 3) * 32;
            umma_f16(t_dpt(b), desc_add(dV, oa), desc_add(dg, ob), idesc_s, kk > 0);
          }
          umma_commit(&s_full[b]);
          DTR(g, 1);
          if (i == nq - 1) umma_commit(kv_empty);   // K / V of this item fully read
        }
        __syncwarp();
      };
      mbar_wait(kv_full, it & 1);
      if (lane == 0) DIT(it, 2);
      issue_s(gi, 0);
      if (nq > 1) issue_s(gi + 1, 1);
      for (int i = 0; i < nq; ++i) {  // dV += P^T dO, dK += dS^T Q (A from TMEM), then S^T(i+2)
        const int g = gi + i, st = g % NST, b = g & 1;
        if (i == 0 && it > 0) mbar_wait(acc_free, (it - 1) & 1);   // the previous item's dK / dV drained
        mbar_wait(&p_full[b], (g >> 1) & 1);
        fence_after();
        const uint64_t dq = desc_add(dQm, st * SM::QT), dg = desc_add(dGm, st * SM::QT);
        if (leader) {
#pragma unroll
          for (int kk = 0; kk < QB / 16; ++kk) {   // dV first (its completion frees P^T for S^T(g+2))
            const uint32_t ta = 32 * (kk >> 1) + 8 * (kk & 1);   // 16 queries: owner half, 8 packed columns
            const uint32_t ob = kk * 16 * 128;                   // MN-major B: 16 query rows
            umma_f16_ts(t_dv, t_st(b) + ta, desc_add(dg, ob), idesc_g, (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&dv_done[b]);
          DTR(g, 4);
#pragma unroll
          for (int kk = 0; kk < QB / 16; ++kk) {
            const uint32_t ta = 32 * (kk >> 1) + 8 * (kk & 1);
            const uint32_t ob = kk * 16 * 128;
            umma_f16_ts(t_dk, t_dpt(b) + ta, desc_add(dq, ob), idesc_g, (i > 0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&g_done[b]);
          DTR(g, 5);
          umma_commit(&q_empty[st]);
        }
        __syncwarp();
        if (i + 2 < nq) issue_s(g + 2, i + 2);
      }
      gi += nq;
    }
  } else if (warp >= 4) {  // ===== element-wise: ping-pong groups, one key row per 2 threads of a group
    const int grp = (warp - 4) >> 3;
    const int hf = ((warp - 4) >> 2) & 1;       // half (32 columns) of the 64 query columns
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    const int64_t s128 = (int64_t)nkt * KB;
    int gi = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
      int kt, h, sq, qstart, nq;
      item(t, kt, h, sq, qstart, nq);
      const int k0 = kt * KB, kj = k0 + r;
      for (int i = (grp - gi) & 1; i < nq; i += 2) {   // this group's iterations: global parity == grp
        const int g = gi + i, st = g % NST;
        const int qa = (qstart + i) * QB + hf * 32;
        const float* ls = reinterpret_cast<const float*>(smem + SM::LD_OFF + st * 512) + hf * 32;
        const float* dsm = ls + 64;
        // valid iff q < s, kj < s and (causal) kj <= q; only tiles touching the diagonal / the end mask
        const bool need_mask = kj >= s || qa + 32 > s || (a.causal && kj > qa);
        const bool any_mask = __any_sync(0xffffffffu, need_mask);   // warp-uniform polynomial choice
        // dS^T [key][query] of this (sequence, head), rows / columns padded to s128 (a.dsT: dQ from dS, 5 matmuls)
        __nv_bfloat16* dst_row =
            a.dsT ? static_cast<__nv_bfloat16*>(a.dsT) + (((int64_t)sq * a.heads + h) * s128 + kj) * s128 : nullptr;
        mbar_wait(&s_full[grp], (g >> 1) & 1);
        if ((warp & 7) == 4 && lane == 0) DTR(g, 2);
        fence_after();
        mbar_wait(&q_full[st], (g / NST) & 1);   // lse / dsum of tile g landed with Q / dO
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t rsv[16], rdp[16];
          tmem_ld16_nowait(t_st(grp) + lrow + hf * 32 + ch * 16, rsv);
          tmem_ld16_nowait(t_dpt(grp) + lrow + hf * 32 + ch * 16, rdp);
          tmem_wait_ld();
          float sc[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) sc[c] = fmaf(__uint_as_float(rsv[c]), sl2, -ls[ch * 16 + c] * LOG2E);
          if (need_mask) {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const int q = qa + ch * 16 + c;
              if (!(q < s && kj < s && (!a.causal || kj <= q))) sc[c] = -INFINITY;
            }
          }
          uint32_t pp[8], pd[8];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            float p[2], gg[2];
            if (!any_mask && ((c >> 1) & 7) < BWD_POLY) {
              ex2_poly2(f2pack(sc[c], sc[c + 1]), p[0], p[1]);
            } else {
              p[0] = ex2(sc[c]);
              p[1] = ex2(sc[c + 1]);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e)
              gg[e] = p[e] * (__uint_as_float(rdp[c + e]) - dsm[ch * 16 + c + e]) * a.scale;
            pp[c / 2] = pack_bf16x2(p[0], p[1]);
            pd[c / 2] = pack_bf16x2(gg[0], gg[1]);
          }
          // packed columns 32h + 8ch .. +7 lie inside chunk 0's range, already read by this thread
          tmem_st8_nowait(t_st(grp) + lrow + hf * 32 + ch * 8, pp);
          tmem_st8_nowait(t_dpt(grp) + lrow + hf * 32 + ch * 8, pd);
          if (dst_row) {   // dS^T row segment for the dQ kernel (masked entries are 0): one full 32-byte sector
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst_row + qa + ch * 16),
                         "r"(pd[0]), "r"(pd[1]), "r"(pd[2]), "r"(pd[3]), "r"(pd[4]), "r"(pd[5]), "r"(pd[6]), "r"(pd[7])
                         : "memory");
          }
        }
        tmem_wait_st();
        fence_before();
        mbar_arrive(&p_full[grp]);
        if ((warp & 7) == 4 && lane == 0) DTR(g, 3);
      }
      // every gradient MMA of this item done: this group's last one (its own barrier: cannot alias an older
      // phase), then the item's very last one (the next phase of that barrier needs this thread's acc_free)
      {
        const int gl = gi + nq - 1;
        const int own = gl - ((gl - grp) & 1);   // last global iteration <= gl of this group's parity
        if (own >= gi) mbar_wait(&g_done[grp], (own >> 1) & 1);
        if (own != gl) mbar_wait(&g_done[gl & 1], (gl >> 1) & 1);
        fence_after();
      }
      if (warp == 4 && lane == 0) DIT(t / (int)gridDim.x, 0);
      constexpr int OC = DH / 4;   // output columns per (group, half)
      const int oq = grp * 2 + hf;
      __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + ((int64_t)sq * s + kj) * 3 * d + h * DH + oq * OC;
      float* cs = a.colsum ? a.colsum + ((int64_t)(sq * nkt + kt) * 4 + qd) * 3 * d + h * DH + oq * OC : nullptr;
      // all TMEM loads first, then release the accumulators (the next item's first dV / dK MMAs run while
      // this row is stored); the key-bias gradient is identically zero (softmax shift invariance, pin P4):
      // its partials are written as zeros instead of summed
      constexpr int NC = OC / 16;
      uint32_t rk[NC][16], rv[NC][16];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        tmem_ld16_nowait(t_dk + lrow + oq * OC + 16 * c, rk[c]);
        tmem_ld16_nowait(t_dv + lrow + oq * OC + 16 * c, rv[c]);
      }
      tmem_wait_ld();
      fence_before();
      mbar_arrive(acc_free);   // dK / dV accumulators free for the next item
      const bool valid = kj < s;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (cs) {
          float w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) w[i] = valid ? __uint_as_float(rv[c][i]) : 0.f;
          const float sum = warp_colsum16(w);
          if (lane < 16) {
            cs[d + 16 * c + lane] = 0.f;
            cs[2 * d + 16 * c + lane] = sum;
          }
        }
        if (!valid) continue;
        uint32_t pk[8], pv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          pk[i] = pack_bf16x2(__uint_as_float(rk[c][2 * i]), __uint_as_float(rk[c][2 * i + 1]));
          pv[i] = pack_bf16x2(__uint_as_float(rv[c][2 * i]), __uint_as_float(rv[c][2 * i + 1]));
        }
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + d + 16 * c), "r"(pk[0]),
                     "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7])
                     : "memory");
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(out + 2 * d + 16 * c), "r"(pv[0]),
                     "r"(pv[1]), "r"(pv[2]), "r"(pv[3]), "r"(pv[4]), "r"(pv[5]), "r"(pv[6]), "r"(pv[7])
                     : "memory");
      }
      if (warp == 4 && lane == 0) DIT(t / (int)gridDim.x, 1);
      gi += nq;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tb, 512);
  }
}

// =============================================================================== dQ
// One CTA per 128-query tile, 128-key iterations.  S = Q K^T and dP = dO V^T are M=128, N=128 MMAs (operand
// bandwidth and math balanced; N=64 tiles were bound by shared-memory operand reads), single-buffered in
// TMEM: all 16 element-wise warps load S(j) / dP(j) first thing and release them, so S(j+1) runs on the
// tensor pipe while they compute dS(j).  TMEM: S at 0, dP at 128, dQ at 256, dS[2] (bf16 packed, 64
// columns each) at 384 / 448.  dQ += dS K with A = dS from TMEM, K read MN-major from its K-major tile.
constexpr int QB2 = 128;  // queries per CTA
constexpr int KB2 = 128;  // keys per iteration

template <int DH>
struct DqSmem {
  static constexpr int SUB128 = 128 * 128;
  static constexpr int QT = DH / 64 * SUB128;   // Q (or dO) [128][DH]
  static constexpr int KT = DH / 64 * SUB128;   // K (or V) [128][DH]
  static constexpr int Q_OFF = 0;
  static constexpr int G_OFF = Q_OFF + QT;
  // K is read by S and by dQ (freed late), V only by dP (freed when S / dP complete): separate rings
  static constexpr int NK = DH == 64 ? 4 : 3, NV = DH == 64 ? 3 : 2;
  static constexpr int K_OFF = G_OFF + QT;      // [NK]
  static constexpr int V_OFF = K_OFF + NK * KT; // [NV]
  static constexpr int BAR_OFF = V_OFF + NV * KT;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

// Persistent like the dK / dV kernel: items (query tile, head, sequence) in chunks of DQ_G (sequence, head)
// pairs (their K / V tiles stay in L2), heaviest query tiles first; K / V rings, the S / dP buffer and the dS
// buffers run on global counters; the next item's Q / dO tiles load once the current item's last S / dP MMAs
// have read them (qg_empty), and only its first dQ MMA waits for the previous dQ drain (acc_free).
#ifndef LGA_DQ_G
#define LGA_DQ_G 16
#endif
constexpr int DQ_G = LGA_DQ_G;

template <int DH>
__global__ void __launch_bounds__(NT, 1)
    dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_g,
              const __grid_constant__ CUtensorMap tm_kv, const AttnArgs a) {
  using SM = DqSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  constexpr int NK = SM::NK, NV = SM::NV;
  constexpr int EW_ALL = EW_WARPS * 32;
  uint64_t* qg_full = bars + 0;
  uint64_t* k_full = bars + 1;              // [NK]
  uint64_t* k_empty = k_full + NK;          // [NK]
  uint64_t* v_full = k_empty + NK;          // [NV]
  uint64_t* v_empty = v_full + NV;          // [NV]
  uint64_t* s_full = v_empty + NV;          // S(j), dP(j) in TMEM
  uint64_t* s_empty = s_full + 1;           // ... loaded by every element-wise thread (EW_ALL)
  uint64_t* p_full = s_empty + 1;           // [2] per dS buffer (EW_ALL)
  uint64_t* g_done = p_full + 2;            // [2] per dS buffer: dQ MMAs done
  uint64_t* qg_empty = g_done + 2;          // Q / dO read by the item's last S / dP MMAs
  uint64_t* acc_free = qg_empty + 1;        // dQ drained (EW_ALL)
  constexpr int NBAR = 2 * NK + 2 * NV + 9;
  static_assert(NBAR * 8 + 4 <= 256, "barrier area");
  static_assert(SM::TOTAL <= 232448, "shared memory");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + NBAR);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.seq, d = a.d;
  const int nqt = (s + QB2 - 1) / QB2;
  const int pairs = a.heads * a.nseq;
  const int n_items = nqt * pairs;
  auto item = [&](int t, int& qt, int& h, int& sq, int& nk) {
    const int chunk = t / (DQ_G * nqt), w = t % (DQ_G * nqt);
    const int np = min(DQ_G, pairs - chunk * DQ_G);
    const int qi = w / np, pair = chunk * DQ_G + w % np;
    qt = a.causal ? nqt - 1 - qi : qi;   // heaviest (most keys) first under causal masking
    h = pair % a.heads;
    sq = pair / a.heads;
    const int kend = a.causal ? min(s, qt * QB2 + QB2) : s;
    nk = (kend + KB2 - 1) / KB2;
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < NBAR; ++i) {
      const bool ew = (&bars[i] >= s_empty && &bars[i] < g_done) || &bars[i] == acc_free;
      mbar_init(&bars[i], ew ? EW_ALL : 1);
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
  const uint32_t t_s = tb, t_dp = tb + 128, t_dq = tb + 256;
  auto t_ds = [&](int b) { return tb + 384 + 64 * b; };

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      int jg = 0, it = 0;
      for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
        int qt, h, sq, nk;
        item(t, qt, h, sq, nk);
        mbar_wait(qg_empty, (it & 1) ^ 1);   // the previous item's last S / dP MMAs read Q / dO
        mbar_expect_tx(qg_full, 2 * SM::QT);
#pragma unroll
        for (int c = 0; c < DH / 64; ++c) {
          tma_load_3d(smem + SM::Q_OFF + c * SM::SUB128, &tm_q, qg_full, h * DH + 64 * c, qt * QB2, sq);
          tma_load_3d(smem + SM::G_OFF + c * SM::SUB128, &tm_g, qg_full, h * DH + 64 * c, qt * QB2, sq);
        }
        for (int j = 0; j < nk; ++j, ++jg) {
          const int sk = jg % NK, sv = jg % NV;
          mbar_wait(&k_empty[sk], ((jg / NK) & 1) ^ 1);
          mbar_expect_tx(&k_full[sk], SM::KT);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
            tma_load_3d(smem + SM::K_OFF + sk * SM::KT + c * SM::SUB128, &tm_kv, &k_full[sk], d + h * DH + 64 * c,
                        j * KB2, sq);
          mbar_wait(&v_empty[sv], ((jg / NV) & 1) ^ 1);
          mbar_expect_tx(&v_full[sv], SM::KT);
#pragma unroll
          for (int c = 0; c < DH / 64; ++c)
            tma_load_3d(smem + SM::V_OFF + sv * SM::KT + c * SM::SUB128, &tm_kv, &v_full[sv], 2 * d + h * DH + 64 * c,
                        j * KB2, sq);
        }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer (whole warp; one elected lane issues)
    constexpr uint32_t idesc_s = make_idesc(128, KB2, false, false);
    constexpr uint32_t idesc_q = make_idesc(128, DH, false, true);
    const bool leader = elect_one();
    const uint64_t dQ = make_desc(smem_u32(smem + SM::Q_OFF), 16, 1024);
    const uint64_t dG = make_desc(smem_u32(smem + SM::G_OFF), 16, 1024);
    const uint64_t dK = make_desc(smem_u32(smem + SM::K_OFF), 16, 1024);
    const uint64_t dV = make_desc(smem_u32(smem + SM::V_OFF), 16, 1024);
    const uint64_t dKm = make_desc(smem_u32(smem + SM::K_OFF), SM::SUB128, 1024);   // K, MN-major
    int jg = 0, it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int qt, h, sq, nk;
      item(t, qt, h, sq, nk);
      mbar_wait(qg_full, it & 1);
      // issue order S(0), S(1), dQ(0), S(2), dQ(1), ...: S(j+1) only needs S(j) loaded by the element-wise
      // warps, dQ(j) needs dS(j); all counters global (g = jg + j)
      for (int j = 0; j < nk + 1; ++j) {
        if (j < nk) {  // S(j), dP(j)
          const int g = jg + j, sk = g % NK, sv = g % NV;
          mbar_wait(&k_full[sk], (g / NK) & 1);
          mbar_wait(&v_full[sv], (g / NV) & 1);
          if (g > 0) mbar_wait(s_empty, (g - 1) & 1);
          fence_after();
          const uint64_t dk = desc_add(dK, sk * SM::KT), dv = desc_add(dV, sv * SM::KT);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < DH / 16; ++kk) {
              const uint32_t o = (kk >> 2) * SM::SUB128 + (kk & 3) * 32;
              umma_f16(t_s, desc_add(dQ, o), desc_add(dk, o), idesc_s, kk > 0);
              umma_f16(t_dp, desc_add(dG, o), desc_add(dv, o), idesc_s, kk > 0);
            }
            umma_commit(s_full);
            umma_commit(&v_empty[sv]);   // V consumed by dP
            if (j == nk - 1) umma_commit(qg_empty);   // Q / dO of this item fully read
          }
          __syncwarp();
        }
        if (j >= 1) {  // dQ += dS K of iteration j-1 (A = dS from TMEM)
          const int jj = j - 1, g = jg + jj, sk = g % NK, pb = g & 1;
          if (jj == 0 && it > 0) mbar_wait(acc_free, (it - 1) & 1);   // the previous item's dQ drained
          mbar_wait(&p_full[pb], (g >> 1) & 1);
          fence_after();
          const uint64_t dk = desc_add(dKm, sk * SM::KT);
          if (leader) {
#pragma unroll
            for (int kk = 0; kk < KB2 / 16; ++kk)   // 16 keys = 8 packed dS columns, 16 K rows
              umma_f16_ts(t_dq, t_ds(pb) + 8 * kk, desc_add(dk, kk * 16 * 128), idesc_q, (jj > 0 || kk > 0) ? 1u : 0u);
            umma_commit(&g_done[pb]);
            umma_commit(&k_empty[sk]);
          }
          __syncwarp();
        }
      }
      jg += nk;
    }
  } else if (warp >= 4) {  // ===== element-wise: one query row per 4 threads, 32 key columns each
    const int cg = (warp - 4) >> 2;             // key-column group 0..3
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    const float sl2 = a.scale * LOG2E;
    int jg = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
      int qt, h, sq, nk;
      item(t, qt, h, sq, nk);
      const int q0 = qt * QB2, q = q0 + r;
      const int64_t rb = ((int64_t)sq * a.heads + h) * s;
      const float lse2 = q < s ? a.lse[rb + q] * LOG2E : 0.f;
      const float Dq = q < s ? a.dsum[rb + q] : 0.f;
      for (int j = 0; j < nk; ++j) {
        const int g = jg + j;
        const int ka = j * KB2 + cg * 32;
        const bool need_mask = q >= s || ka + 32 > s || (a.causal && ka + 31 > q0 + qd * 32);
        const bool any_mask = __any_sync(0xffffffffu, need_mask);   // warp-uniform polynomial choice
        mbar_wait(s_full, g & 1);
        fence_after();
        uint32_t rsv[2][16], rdp[2][16];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          tmem_ld16_nowait(t_s + lrow + cg * 32 + ch * 16, rsv[ch]);
          tmem_ld16_nowait(t_dp + lrow + cg * 32 + ch * 16, rdp[ch]);
        }
        tmem_wait_ld();
        fence_before();
        mbar_arrive(s_empty);   // S / dP buffer free for S(g+1)
        uint32_t pd[16];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float sc[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) sc[c] = fmaf(__uint_as_float(rsv[ch][c]), sl2, -lse2);
          if (need_mask) {
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const int kj = ka + ch * 16 + c;
              if (!(q < s && kj < s && (!a.causal || kj <= q))) sc[c] = -INFINITY;
            }
          }
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            float gg[2];
            if (!any_mask && ((c >> 1) & 7) < BWD_POLY) {
              ex2_poly2(f2pack(sc[c], sc[c + 1]), gg[0], gg[1]);
            } else {
              gg[0] = ex2(sc[c]);
              gg[1] = ex2(sc[c + 1]);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) gg[e] *= (__uint_as_float(rdp[ch][c + e]) - Dq) * a.scale;
            pd[ch * 8 + c / 2] = pack_bf16x2(gg[0], gg[1]);
          }
        }
        const int pb = g & 1;
        if (g >= 2) {
          mbar_wait(&g_done[pb], ((g >> 1) & 1) ^ 1);   // dQ MMAs of iteration g-2 done: dS buffer free
          fence_after();
        }
        tmem_st16_nowait(t_ds(pb) + lrow + cg * 16, pd);
        tmem_wait_st();
        fence_before();
        mbar_arrive(&p_full[pb]);
      }
      const int gl = jg + nk - 1;
      mbar_wait(&g_done[gl & 1], (gl >> 1) & 1);   // the item's last dQ MMAs (and all before) done
      fence_after();
      constexpr int OC = DH / 4;
      __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + ((int64_t)sq * s + q) * 3 * d + h * DH + cg * OC;
      float* cs = a.colsum ? a.colsum + ((int64_t)(sq * nqt + qt) * 4 + qd) * 3 * d + h * DH + cg * OC : nullptr;
      store_row_bf16_global(out, t_dq + lrow + cg * OC, OC, 1.f, q < s, cs);
      fence_before();
      mbar_arrive(acc_free);   // dQ accumulator free for the next item
      jg += nk;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tb, 512);
  }
}

// =============================================================================== dQ from dS (5-matmul backward)
// With a dS workspace (AttnArgs::dsT) the dK/dV kernel stores dS^T next to its P^T / dS^T TMEM writes, and dQ is a
// plain batched, causally blocked GEMM: dQ[q] = sum_key dS[q][key] K[key] -- no second S / dP recompute, no exp.
// Per item (128-query tile, head, sequence): k-blocks of 64 keys; A = dS^T tile [64 keys][128 queries] read
// MN-major, B = K rows [64 keys][d_h] read MN-major; fp32 accumulator in TMEM, two stages so the drain of one
// item overlaps the next item's MMAs; persistent, heaviest tiles first.  Warps: 0 TMA, 1 MMA, 2 TMEM,
// 4..11 epilogue (two per TMEM lane quadrant, half the columns each).
constexpr int DQS_STAGES = 6;
constexpr int DQS_EPI0 = 4, DQS_EPI = 8;
constexpr int DQS_NT = (DQS_EPI0 + DQS_EPI) * 32;

template <int DH>
struct DqsSmem {
  static constexpr int A_BYTES = 128 * 64 * 2;        // two [64 keys][64 queries] sub-tiles
  static constexpr int B_BYTES = DH * 64 * 2;         // DH/64 [64 keys][64 dh] sub-tiles
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = DQS_STAGES * STAGE;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
  static_assert(TOTAL <= 232448, "shared memory");
};

template <int DH>
__global__ void __launch_bounds__(DQS_NT, 1)
    dq_from_ds_kernel(const __grid_constant__ CUtensorMap tm_ds, const __grid_constant__ CUtensorMap tm_k,
                      const AttnArgs a) {
  using SM = DqsSmem<DH>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + DQS_STAGES;
  uint64_t* tfull = empty + DQS_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;           // [2] (epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  constexpr int EPI_ALL = DQS_EPI * 32;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = a.seq, d = a.d;
  const int nqt = (s + QB2 - 1) / QB2;
  const int s128 = nqt * QB2;
  const int pairs = a.heads * a.nseq;
  const int n_items = nqt * pairs;
  auto item = [&](int t, int& qt, int& h, int& sq, int& nkb) {
    const int chunk = t / (DQ_G * nqt), w = t % (DQ_G * nqt);
    const int np = min(DQ_G, pairs - chunk * DQ_G);
    const int qi = w / np, pair = chunk * DQ_G + w % np;
    qt = a.causal ? nqt - 1 - qi : qi;
    h = pair % a.heads;
    sq = pair / a.heads;
    const int kend = a.causal ? min(s, qt * QB2 + QB2) : s;
    nkb = (kend + 63) / 64;   // 64-key blocks
  };

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < DQS_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], EPI_ALL); }
    mbar_fence_init();
    prefetch_tmap(&tm_ds);
    prefetch_tmap(&tm_k);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
        int qt, h, sq, nkb;
        item(t, qt, h, sq, nkb);
        const int row0 = (sq * a.heads + h) * s128;   // this (sequence, head)'s dS^T rows
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE;
          uint8_t* sb = sa + SM::A_BYTES;
          mbar_expect_tx(&full[stage], SM::STAGE);
#pragma unroll
          for (int i = 0; i < 2; ++i)   // queries [qt*128 + 64 i, +64) of keys [kb*64, +64)
            tma_load_2d(sa + i * 64 * 128, &tm_ds, &full[stage], qt * QB2 + 64 * i, row0 + kb * 64);
#pragma unroll
          for (int i = 0; i < DH / 64; ++i)   // K[kb*64 .., h*dh + 64 i ..]
            tma_load_3d(sb + i * 64 * 128, &tm_k, &full[stage], d + h * DH + 64 * i, kb * 64, sq);
          if (++stage == DQS_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ===== MMA issuer (whole warp, one elected lane)
    constexpr uint32_t idesc = make_idesc(128, DH, true, true);
    const bool leader = elect_one();
    const uint64_t ad0 = make_desc(smem_u32(smem), 64 * 128, 1024);
    const uint64_t bd0 = make_desc(smem_u32(smem) + SM::A_BYTES, 64 * 128, 1024);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int qt, h, sq, nkb;
      item(t, qt, h, sq, nkb);
      const int as = it & 1;
      mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
      fence_after();
      const uint32_t dtm = tb + as * 128;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        fence_after();
        const uint64_t ad = desc_add(ad0, stage * SM::STAGE), bd = desc_add(bd0, stage * SM::STAGE);
        if (leader) {
#pragma unroll
          for (int k = 0; k < 4; ++k)   // 16 keys = 16 MN-major rows (2048 B)
            umma_f16(dtm, desc_add(ad, k * 2048), desc_add(bd, k * 2048), idesc, (kb | k) != 0 ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == DQS_STAGES) { stage = 0; phase ^= 1; }
      }
      if (leader) umma_commit(&tfull[as]);
      __syncwarp();
    }
  } else if (warp >= DQS_EPI0) {  // ===== epilogue: TMEM -> bf16 dQ (+ the qkv bias-gradient partials)
    const int qd = warp & 3, half = (warp - DQS_EPI0) >> 2;
    const uint32_t lrow = (uint32_t)(qd * 32) << 16;
    int it = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x, ++it) {
      int qt, h, sq, nkb;
      item(t, qt, h, sq, nkb);
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      fence_after();
      const int q = qt * QB2 + qd * 32 + lane;
      constexpr int OC = DH / 2;
      __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.dqkv) + ((int64_t)sq * s + q) * 3 * d + h * DH + half * OC;
      float* cs = a.colsum ? a.colsum + ((int64_t)(sq * nqt + qt) * 4 + qd) * 3 * d + h * DH + half * OC : nullptr;
      store_row_bf16_global(out, tb + as * 128 + lrow + half * OC, OC, 1.f, q < s, cs);
      fence_before();
      mbar_arrive(&tempty[as]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tb, 256);
  }
}

template <int DH>
static cudaError_t run(const AttnArgs& a, cudaStream_t st) {
  const int64_t rows = (int64_t)a.nseq * a.seq * a.heads;
  note_launch(), dsum_kernel<<<(unsigned)((rows * (a.dh / 16) + 255) / 256), 256, 0, st>>>(a);
  CUtensorMap kv128, q64, g64, q128, g128;
  cudaError_t e;
  const uint64_t ld = 3ull * a.d;
  if ((e = map3d_bf16(&kv128, a.qkv, ld, a.seq, a.nseq, 128)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&q64, a.qkv, ld, a.seq, a.nseq, 64)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&g64, a.dO, a.d, a.seq, a.nseq, 64)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&q128, a.qkv, ld, a.seq, a.nseq, 128)) != cudaSuccess) return e;
  if ((e = map3d_bf16(&g128, a.dO, a.d, a.seq, a.nseq, 128)) != cudaSuccess) return e;

  static bool set = false;
  if (!set) {
    if ((e = cudaFuncSetAttribute(dkdv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, DkvSmem<DH>::TOTAL)))
      return e;
    if ((e = cudaFuncSetAttribute(dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqSmem<DH>::TOTAL)))
      return e;
    set = true;
  }
  const int dkv_items = ((a.seq + KB - 1) / KB) * a.heads * a.nseq;
  note_launch(), dkdv_kernel<DH><<<std::min(dkv_items, num_sms()), NT, DkvSmem<DH>::TOTAL, st>>>(kv128, q64, g64, a);
  const int dq_items = ((a.seq + QB2 - 1) / QB2) * a.heads * a.nseq;
  if (a.dsT) {   // dQ from the dS^T the dK/dV kernel stored (5-matmul backward)
    static bool set2 = false;
    if (!set2) {
      if ((e = cudaFuncSetAttribute(dq_from_ds_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    DqsSmem<DH>::TOTAL)))
        return e;
      set2 = true;
    }
    const uint64_t s128 = (uint64_t)((a.seq + QB2 - 1) / QB2) * QB2;
    CUtensorMap ds, k64;
    if ((e = map2d_bf16(&ds, a.dsT, s128, s128 * a.heads * a.nseq, s128, 64, 64)) != cudaSuccess) return e;
    if ((e = map3d_bf16(&k64, a.qkv, ld, a.seq, a.nseq, 64)) != cudaSuccess) return e;
    note_launch(), dq_from_ds_kernel<DH><<<std::min(dq_items, num_sms()), DQS_NT, DqsSmem<DH>::TOTAL, st>>>(ds, k64, a);
    return cudaGetLastError();
  }
  note_launch(), dq_kernel<DH><<<std::min(dq_items, num_sms()), NT, DqSmem<DH>::TOTAL, st>>>(q128, g128, kv128, a);
  return cudaGetLastError();
}

}  // namespace fatb

#ifdef LGA_BWD_TRACE
extern "C" int lgatest_bwd_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fatb::g_bwd_trace, sizeof(fatb::g_bwd_trace));
}
extern "C" int lgatest_dq_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fatb::g_dq_trace, sizeof(fatb::g_dq_trace));
}
#endif
#ifdef LGA_DKV_TRACE
extern "C" int lgatest_dkv_trace(long long* iters, long long* items) {
  cudaError_t e = cudaMemcpyFromSymbol(iters, fatb::g_dkv_trace, sizeof(fatb::g_dkv_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(items, fatb::g_dkv_items, sizeof(fatb::g_dkv_items));
  return (int)e;
}
#endif

cudaError_t attn_bwd_bf16(const AttnArgs& a, cudaStream_t st) {
  if (a.nseq <= 0) return cudaSuccess;
  return a.dh == 64 ? fatb::run<64>(a, st) : fatb::run<128>(a, st);
}

}  // namespace lga
