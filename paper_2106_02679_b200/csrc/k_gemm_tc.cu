// k_gemm_tc.cu -- bf16 GEMM on the 5th-generation tensor cores, sm_100a:
//   TMA (cp.async.bulk.tensor, 128B swizzle) -> shared-memory ring (STAGES deep)
//   -> tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) issued by one thread, fp32 accumulators in TMEM
//   -> tcgen05.ld by 8 epilogue warps -> fused epilogue (epilogue.cuh semantics) -> global.
// Persistent, warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warps 4..11 = epilogue (two per TMEM lane quadrant, each draining half of the tile's columns).  Two TMEM
// accumulator stages so that the epilogue of tile t overlaps the MMAs of tile t+1.  Operands may be
// K-major or MN-major independently (UMMA descriptor major bit), so forward (X W), dgrad (dY W^T) and
// wgrad (X^T dY) all read their operands in place -- no transposes.
//
// Epilogue data path (TMA_EPI): each warp owns a 4 KB swizzled staging tile of 32 rows x 32 columns;
// the residual / accumulator / GELU input is TMA-loaded into it, the results are written back in place
// and TMA-stored (bulk groups), so global traffic moves in full coalesced boxes instead of one row per
// thread.  Shapes whose leading dimensions are not 16-byte multiples use the direct per-row path.
#include "epilogue.cuh"
#include "tc_common.cuh"

namespace lga {

namespace tc {

using namespace tcu;

constexpr int BM = 128;
constexpr int BK = 64;           // 64 bf16 = 128 bytes = one swizzle span
constexpr int UMMA_K = 16;
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;
constexpr int NUM_THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int EPI_TILE = 32;     // rows and columns of one epilogue staging box
constexpr int STAGE_EPI = 4096;  // bytes of staging per epilogue warp

template <int BN>
struct Smem {
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;   // two accumulator stages
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = EPI_OFF + EPI_WARPS * STAGE_EPI;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;   // + barriers + alignment slack
};

// Epilogue tensor maps (TMA path): out (g for GELU fwd), aux out (u for GELU fwd), and one input
// (residual | accumulator | u for GELU bwd).
struct EpiMaps {
  CUtensorMap out, aux, in;
};

// ---- direct (per-row) epilogue of 32 consecutive columns of one row; also the fallback
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__device__ __forceinline__ void load32(const void* base, DT t, int64_t idx, float (&x)[32]) {
  if (t == DT::F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + idx);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q = p[i];
      x[4 * i] = q.x; x[4 * i + 1] = q.y; x[4 * i + 2] = q.z; x[4 * i + 3] = q.w;
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + idx);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 q = p[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
        x[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
      }
    }
  }
}

__device__ __forceinline__ void store32(void* base, DT t, int64_t idx, const float (&x)[32]) {
  if (t == DT::F32) {
    float4* p = reinterpret_cast<float4*>(static_cast<float*>(base) + idx);
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
  } else {
    uint4* p = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + idx);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      p[i] = make_uint4(pack_bf16x2(x[8 * i], x[8 * i + 1]), pack_bf16x2(x[8 * i + 2], x[8 * i + 3]),
                        pack_bf16x2(x[8 * i + 4], x[8 * i + 5]), pack_bf16x2(x[8 * i + 6], x[8 * i + 7]));
  }
}

__device__ __forceinline__ void epi_chunk_direct(const Epi& e, int64_t m, int64_t n0, int nvalid, float (&v)[32]) {
  bool vec = nvalid == 32 && aligned16(static_cast<char*>(e.out) + (m * e.ldo + n0) * (int64_t)dt_size(e.out_dt));
  if (vec && e.kind == EPI_STORE) {
    if (e.bias) vec = aligned16(static_cast<const char*>(e.bias) + n0 * (int64_t)dt_size(e.bias_dt));
    if (e.res) vec = vec && aligned16(e.res + m * e.ldr + n0);
    if (e.acc_in) vec = vec && aligned16(e.acc_in + m * e.ldacc + n0);
  } else if (vec) {
    if (e.aux) vec = aligned16(static_cast<char*>(e.aux) + (m * e.ldaux + n0) * (int64_t)dt_size(e.aux_dt));
    if (e.kind == EPI_GELU_FWD) vec = vec && aligned16(static_cast<const char*>(e.bias) + n0 * (int64_t)dt_size(e.bias_dt));
  }
  if (!vec) {
    for (int i = 0; i < nvalid; ++i) epi_store(e, m, n0 + i, v[i]);
    return;
  }
  float t[32];
  if (e.kind == EPI_STORE) {
    if (e.bias) { load32(e.bias, e.bias_dt, n0, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i]; }
    if (e.res) { load32(e.res, DT::F32, m * e.ldr + n0, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i]; }
    if (e.acc_in) { load32(e.acc_in, DT::F32, m * e.ldacc + n0, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i]; }
    store32(e.out, e.out_dt, m * e.ldo + n0, v);
  } else if (e.kind == EPI_GELU_FWD) {
    load32(e.bias, e.bias_dt, n0, t);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += t[i];
    if (e.aux) store32(e.aux, e.aux_dt, m * e.ldaux + n0, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = gelu_f(v[i]);
    store32(e.out, e.out_dt, m * e.ldo + n0, v);
  } else {
    load32(e.aux, e.aux_dt, m * e.ldaux + n0, t);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_f(t[i]);
    store32(e.out, e.out_dt, m * e.ldo + n0, v);
  }
}

// ---- staged (TMA) epilogue: one row of a 32 x 32 swizzled staging box
// fp32 box: 128-byte rows, 128B swizzle (16-byte chunk c of row r at c ^ (r & 7));
// bf16 box: 64-byte rows, 64B swizzle (chunk c of row r at c ^ ((r >> 1) & 3)).
__device__ __forceinline__ void stage_read_row(const uint8_t* buf, DT t, int r, float (&x)[32]) {
  if (t == DT::F32) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 q = *reinterpret_cast<const float4*>(buf + r * 128 + ((c ^ (r & 7)) << 4));
      x[4 * c] = q.x; x[4 * c + 1] = q.y; x[4 * c + 2] = q.z; x[4 * c + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint4 q = *reinterpret_cast<const uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x[8 * c + 2 * j] = __uint_as_float(w[j] << 16);
        x[8 * c + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
      }
    }
  }
}
__device__ __forceinline__ void stage_write_row(uint8_t* buf, DT t, int r, const float (&x)[32]) {
  if (t == DT::F32) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<float4*>(buf + r * 128 + ((c ^ (r & 7)) << 4)) =
          make_float4(x[4 * c], x[4 * c + 1], x[4 * c + 2], x[4 * c + 3]);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      *reinterpret_cast<uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) =
          make_uint4(pack_bf16x2(x[8 * c], x[8 * c + 1]), pack_bf16x2(x[8 * c + 2], x[8 * c + 3]),
                     pack_bf16x2(x[8 * c + 4], x[8 * c + 5]), pack_bf16x2(x[8 * c + 6], x[8 * c + 7]));
  }
}

// Epilogue warps (EPI_WARP0 ..): for every tile of this CTA, wait for the accumulator stage, drain it
// from TMEM through the fused epilogue, release the stage (`release(as)`).  Rows of a tile start at
// mb * tile_m + m_off (m_off = the CTA's half of a CTA-pair tile).
template <int BN, bool TMA_EPI, typename Coords, typename Release>
__device__ __forceinline__ void epilogue_loop(const GemmArgs& g, const EpiMaps& em, uint8_t* smem_epi, uint64_t* ebar,
                                              uint64_t* tfull, uint32_t tmem_base, int num_tiles, int t0, int tstride,
                                              int m_off, int tile_m, Coords tile_coords, Release release) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ew = warp - EPI_WARP0;
  const int q = warp & 3;          // TMEM lane quadrant this warp may access
  const int half = ew >> 2;
  const Epi& e = g.epi;
  uint8_t* sbuf = smem_epi + ew * STAGE_EPI;
  // staged-path roles of the single input box and the output box(es)
  const bool has_in = TMA_EPI && (e.res || e.acc_in || e.kind == EPI_GELU_BWD);
  const DT in_dt = e.kind == EPI_GELU_BWD ? e.aux_dt : DT::F32;
  const uint32_t in_bytes = EPI_TILE * EPI_TILE * (uint32_t)dt_size(in_dt);
  uint32_t ephase = 0;
  int it = 0;
  if (TMA_EPI && e.kind == EPI_GELU_BWD && dt_size(in_dt) == 2) {
    // GELU backward: the 2 KB bf16 u box is rewritten in place, so the other half of the 4 KB staging area
    // takes the next box -- the u load of box k+1 (also the next tile's first box, before its accumulator
    // is ready) overlaps box k instead of exposing one load latency per box
    constexpr int CH_PER = BN / 64;
    auto box = [&](int tt, int cc, int& m0w_, int& n0_) {
      int mb_, nb_;
      tile_coords(tt, mb_, nb_);
      m0w_ = mb_ * tile_m + m_off + q * 32;
      n0_ = nb_ * BN + cc * 32;
      return n0_ < g.N && m0w_ < g.M;
    };
    auto next_valid = [&](int tt, int cc, int& nt, int& nc) {   // next box of this warp inside the matrix
      nt = tt, nc = cc;
      while (true) {
        if (++nc >= (half + 1) * CH_PER) {
          nc = half * CH_PER;
          nt += tstride;
          if (nt >= num_tiles) return false;
        }
        int a, b;
        if (box(nt, nc, a, b)) return true;
      }
    };
    auto load = [&](int tt, int cc, int b) {
      int a, n;
      box(tt, cc, a, n);
      mbar_expect_tx(&ebar[2 * ew + b], in_bytes);
      tma_load_2d(sbuf + b * 2048, &em.in, &ebar[2 * ew + b], n, a);
    };
    uint32_t phb = 0;   // bit b: phase of buffer b's load barrier
    int buf = 0;
    if (lane == 0 && t0 < num_tiles) {
      int ft = t0, fc = half * CH_PER, a, n;
      if (box(ft, fc, a, n) || next_valid(t0, fc, ft, fc)) load(ft, fc, 0);
    }
    __syncwarp();
    for (int t = t0; t < num_tiles; t += tstride, ++it) {
      const int as = it & 1;
      mbar_wait(&tfull[as], (it >> 1) & 1);
      fence_after();
      const uint32_t taddr = tmem_base + as * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int ch = half * CH_PER; ch < (half + 1) * CH_PER; ++ch) {
        int m0w, n0;
        if (!box(t, ch, m0w, n0)) continue;   // whole box outside the matrix (warp-uniform)
        if (lane == 0) {
          bulk_wait_read0();   // the previous box's store has read the other buffer
          int nt, nc;
          if (next_valid(t, ch, nt, nc)) load(nt, nc, buf ^ 1);
        }
        __syncwarp();
        uint32_t raw[32];
        tmem_ld32_nowait(taddr + ch * 32, raw);
        tmem_wait_ld();
        mbar_wait(&ebar[2 * ew + buf], (phb >> buf) & 1u);
        phb ^= 1u << buf;
        uint8_t* sb = sbuf + buf * 2048;
        float u[32], v[32];
        stage_read_row(sb, in_dt, lane, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]) * gelu_grad_fast(u[i]);
        stage_write_row(sb, e.out_dt, lane, v);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d_hint(&em.out, sb, n0, m0w, policy_evict_first());
          bulk_commit();
        }
        if (e.colsum) {   // bias gradient partial of this 32-row strip (rows past M contribute 0)
          if (m0w + lane >= g.M) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
          const float cs = warp_colsum32(v);
          if (n0 + lane < g.N) e.colsum[(int64_t)(m0w >> 5) * g.N + n0 + lane] = cs;
        }
        buf ^= 1;
      }
      fence_before();
      __syncwarp();
      if (lane == 0) release(as);
    }
    if (lane == 0) bulk_wait0();
    return;
  }
  for (int t = t0; t < num_tiles; t += tstride, ++it) {
    int mb, nb;
    tile_coords(t, mb, nb);
    const int as = it & 1;
    const uint32_t aphase = (it >> 1) & 1;
    mbar_wait(&tfull[as], aphase);
    fence_after();
    const int m0w = mb * tile_m + m_off + q * 32;   // first row of this warp's 32-row strip
    const int64_t m = m0w + lane;
    const uint32_t taddr = tmem_base + as * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int ch = half * (BN / 64); ch < (half + 1) * (BN / 64); ++ch) {
      const int n0 = nb * BN + ch * 32;
      if (!TMA_EPI) {
        float v[32];
        tmem_ld32(taddr + ch * 32, v);
        if (e.kind == EPI_GELU_BWD && e.colsum && n0 < g.N) {   // bias gradient partial (see the staged path)
          float w[32];
#pragma unroll
          for (int i = 0; i < 32; ++i)
            w[i] = (m < g.M && n0 + i < g.N) ? v[i] * gelu_grad_f(ld_elem(e.aux, m * e.ldaux + n0 + i, e.aux_dt)) : 0.f;
          const float cs = warp_colsum32(w);
          if (n0 + lane < g.N) e.colsum[(int64_t)(m0w >> 5) * g.N + n0 + lane] = cs;
        }
        if (m < g.M && n0 < g.N) epi_chunk_direct(e, m, n0, (int)min(32, g.N - n0), v);
        continue;
      }
      if (n0 >= g.N || m0w >= g.M) continue;   // whole box outside the matrix (warp-uniform)
      // previous TMA store must have finished reading the staging box before it is reused
      if (lane == 0) {
        bulk_wait_read0();
        if (has_in) {
          mbar_expect_tx(&ebar[2 * ew], in_bytes);
          tma_load_2d(sbuf, &em.in, &ebar[2 * ew], n0, m0w);
        }
      }
      __syncwarp();
      uint32_t raw[32];
      tmem_ld32_nowait(taddr + ch * 32, raw);
      tmem_wait_ld();
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
      if (has_in) {
        mbar_wait(&ebar[2 * ew], ephase);
        ephase ^= 1;
      }
      if (e.kind == EPI_STORE) {
        if (e.bias) {
          float b[32];
          if (n0 + 32 <= g.N) load32(e.bias, e.bias_dt, n0, b);
          else for (int i = 0; i < 32; ++i) b[i] = n0 + i < g.N ? ld_elem(e.bias, n0 + i, e.bias_dt) : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += b[i];
        }
        if (has_in) {
          float x[32];
          stage_read_row(sbuf, DT::F32, lane, x);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += x[i];
        }
        stage_write_row(sbuf, e.out_dt, lane, v);
      } else if (e.kind == EPI_GELU_FWD) {
        float b[32];
        if (n0 + 32 <= g.N) load32(e.bias, e.bias_dt, n0, b);
        else for (int i = 0; i < 32; ++i) b[i] = n0 + i < g.N ? ld_elem(e.bias, n0 + i, e.bias_dt) : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += b[i];
        if (e.aux) stage_write_row(sbuf, e.aux_dt, lane, v);   // u  -> first 2 KB (unless not kept)
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_fast(v[i]);
        stage_write_row(sbuf + 2048, e.out_dt, lane, v);       // g  -> second 2 KB
      } else {  // EPI_GELU_BWD: u was TMA-loaded into the box; out overwrites it in place
        float u[32];
        stage_read_row(sbuf, in_dt, lane, u);
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= gelu_grad_fast(u[i]);
        stage_write_row(sbuf, e.out_dt, lane, v);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        const uint64_t pol = policy_evict_first();   // outputs stream out; keep L2 for the operands
        if (e.kind == EPI_GELU_FWD) {
          if (e.aux) tma_store_2d_hint(&em.aux, sbuf, n0, m0w, pol);
          tma_store_2d_hint(&em.out, sbuf + 2048, n0, m0w, pol);
        } else {
          tma_store_2d_hint(&em.out, sbuf, n0, m0w, pol);
        }
        bulk_commit();
      }
    }
    fence_before();
    __syncwarp();
    if (lane == 0) release(as);
  }
  if (TMA_EPI && lane == 0) bulk_wait0();
}

// Split-K (g.split_k = S > 1): the tile space is S stacked copies of the M x N tiles; copy ks covers k-blocks
// [ks * nkper, (ks + 1) * nkper) and its epilogue `ge` (built on the host: M' = S M rows of fp32 workspace, plain
// store) writes the partial sum at rows ks M .. ks M + M - 1.  splitk_reduce_kernel then applies g.epi.
template <int BN, bool A_MN, bool B_MN, bool TMA_EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ EpiMaps em, const GemmArgs g, const GemmArgs ge) {
  using SM = Smem<BN>;
  constexpr int STAGES = SM::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;   // [EPI_WARPS][2] staging-load barriers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 2 * EPI_WARPS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = g.split_k;
  const int num_m1 = (g.M + BM - 1) / BM;
  const int num_m = num_m1 * S, num_n = (g.N + BN - 1) / BN;   // stacked m-blocks: split ks owns [ks num_m1, ..)
  const int num_tiles = num_m * num_n;
  const int nk_all = (g.K + BK - 1) / BK;
  const int nkper = (nk_all + S - 1) / S;
  // k-block range of a (stacked) m-block
  auto krange = [&](int mb, int& kb0, int& kb1) {
    const int ks = mb / num_m1;
    kb0 = ks * nkper;
    kb1 = min(nk_all, kb0 + nkper);
  };
  // tile raster (tile_coords): n fastest when the grid has at least as many m-blocks as n-blocks, else groups of
  // GM m-blocks sweep all n-blocks.  (Groups sized to one wave of tiles, GM = grid / num_n, cut the FFN1 A
  // over-fetch but raised FFN2's and the step time: measured, reverted.)
  constexpr int GM = 8;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI_WARPS); }
    for (int s = 0; s < 2 * EPI_WARPS; ++s) mbar_init(&ebar[s], 1);
    mbar_fence_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 2) tmem_alloc(tmem_slot, SM::TMEM_COLS);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) {
    // the concurrently running tiles (one wave) share operand panels in L2; the panels a wave leaves half-read
    // are read again from HBM by the next wave.  Walking n fastest re-reads B panels, walking m fastest (in
    // groups of GM m-blocks) re-reads A panels: re-read the smaller operand (fewer blocks along its side).
    if (num_m >= num_n) {
      mb = t / num_n, nb = t % num_n;
      return;
    }
    const int per_group = GM * num_n;
    const int grp = t / per_group;
    const int first_m = grp * GM;
    const int gsz = min(num_m - first_m, GM);
    const int r = t % per_group;
    mb = first_m + r % gsz;
    nb = r / gsz;
  };

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer
      // B re-read by every m-block of the grid: kept in L2 when it fits comfortably (the weights)
      const uint64_t polB = g.b_keep_l2 ? policy_evict_last() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb, kb0, kb1;
        tile_coords(t, mb, nb);
        krange(mb, kb0, kb1);
        const int m0 = (mb % num_m1) * BM, n0 = nb * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE_BYTES;
          uint8_t* sb = sa + SM::A_BYTES;
          mbar_expect_tx(&full[stage], SM::STAGE_BYTES);
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d(sa + i * 64 * BK * 2, &tmA, &full[stage], m0 + 64 * i, k0);
          }
          if (!B_MN) {
            tma_load_2d_hint(sb, &tmB, &full[stage], k0, n0, polB);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d_hint(sb + i * 64 * BK * 2, &tmB, &full[stage], n0 + 64 * i, k0, polB);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {  // ===== MMA issuer: the whole warp runs the loop (uniform descriptor math), one elected lane issues
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      // K-major: advance 16 elements = 32 B inside the swizzle span; MN-major: 16 K-rows = 2048 B
      constexpr uint32_t KSTEP_A = A_MN ? UMMA_K * 128 : UMMA_K * 2, KSTEP_B = B_MN ? UMMA_K * 128 : UMMA_K * 2;
      const bool leader = elect_one();
      const uint64_t ad0 = A_MN ? make_desc(smem_u32(smem), 64 * BK * 2, 1024) : make_desc(smem_u32(smem), 16, 1024);
      const uint64_t bd0 = B_MN ? make_desc(smem_u32(smem) + SM::A_BYTES, 64 * BK * 2, 1024)
                                : make_desc(smem_u32(smem) + SM::A_BYTES, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        int mb, nb, kb0, kb1;
        tile_coords(t, mb, nb);
        krange(mb, kb0, kb1);
        mbar_wait(&tempty[as], aphase ^ 1);
        fence_after();
        const uint32_t dtm = tmem_base + as * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t ad = desc_add(ad0, stage * SM::STAGE_BYTES), bd = desc_add(bd0, stage * SM::STAGE_BYTES);
          if (leader) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k)
              umma_f16(dtm, desc_add(ad, k * KSTEP_A), desc_add(bd, k * KSTEP_B), idesc,
                       (kb != kb0 || k != 0) ? 1u : 0u);
            umma_commit(&empty[stage]);   // frees the smem slot when these MMAs complete
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (leader) umma_commit(&tfull[as]);   // accumulator ready for the epilogue
        __syncwarp();
      }
    }
  } else if (warp >= EPI_WARP0) {  // ===== epilogue: TMEM -> registers -> fused epilogue -> global
    epilogue_loop<BN, TMA_EPI>(ge, em, smem + SM::EPI_OFF, ebar, tfull, tmem_base, num_tiles, blockIdx.x, gridDim.x,
                               0, BM,
                               [&](int t, int& mb, int& nb) { tile_coords(t, mb, nb); },
                               [&](int as) { mbar_arrive(&tempty[as]); });
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tmem_base, SM::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA-pair kernel (cta_group::2)
// A cluster of 2 CTAs computes a 256 x 256 tile: CTA r loads rows [128r, 128r+128) of A and columns
// [128r, 128r+128) of B into its own shared memory; the leader (rank 0) issues
// tcgen05.mma.cta_group::2 (M=256, N=256) which reads both CTAs' operands and writes rows 0..127 of D
// into the leader's TMEM and rows 128..255 into the peer's.  Per-SM operand traffic is a third lower
// than the single-CTA 128 x 256 tile at the same MMA rate.  Each CTA drains its own TMEM (epilogue_loop).
constexpr int PAIR_N = 256;
struct Smem2 {
#ifndef LGA_GEMM2_STAGES
#define LGA_GEMM2_STAGES 5
#endif
  static constexpr int STAGES = LGA_GEMM2_STAGES;
  static constexpr int A_BYTES = BM * BK * 2;            // this CTA's 128 rows of A
  static constexpr int B_BYTES = (PAIR_N / 2) * BK * 2;  // this CTA's 128 columns of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * PAIR_N;
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = EPI_OFF + EPI_WARPS * STAGE_EPI;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;
};

template <bool A_MN, bool B_MN, bool TMA_EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ EpiMaps em, const GemmArgs g) {
  using SM = Smem2;
  constexpr int STAGES = SM::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // keeps shared provenance
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);   // used in the leader only
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;                                        // leader: arrivals from both CTAs
  uint64_t* ebar = tempty + 2;                                         // [EPI_WARPS][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + 2 * EPI_WARPS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_m = (g.M + 2 * BM - 1) / (2 * BM), num_n = (g.N + PAIR_N - 1) / PAIR_N;
  const int num_tiles = num_m * num_n;
  const int nk = (g.K + BK - 1) / BK;
  constexpr int GM = 8;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2 * EPI_WARPS); }
    for (int s = 0; s < 2 * EPI_WARPS; ++s) mbar_init(&ebar[s], 1);
    mbar_fence_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 2) tmem_alloc_cg2(tmem_slot, SM::TMEM_COLS);
  fence_before();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated in both
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int& mb, int& nb) {
    // the concurrently running tiles (one wave) share operand panels in L2; the panels a wave leaves half-read
    // are read again from HBM by the next wave.  Walking n fastest re-reads B panels, walking m fastest (in
    // groups of GM m-blocks) re-reads A panels: re-read the smaller operand (fewer blocks along its side).
    if (num_m >= num_n) {
      mb = t / num_n, nb = t % num_n;
      return;
    }
    const int per_group = GM * num_n;
    const int grp = t / per_group;
    const int first_m = grp * GM;
    const int gsz = min(num_m - first_m, GM);
    const int r = t % per_group;
    mb = first_m + r % gsz;
    nb = r / gsz;
  };

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer (both CTAs), completion counted on the leader's full barrier
      // B re-read by every m-block of the grid: kept in L2 when it fits comfortably (the weights)
      const uint64_t polB = g.b_keep_l2 ? policy_evict_last() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < num_tiles; t += npairs) {
        int mb, nb;
        tile_coords(t, mb, nb);
        const int m0 = mb * 2 * BM + rank * BM, n0 = nb * PAIR_N + rank * (PAIR_N / 2);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * SM::STAGE_BYTES;
          uint8_t* sb = sa + SM::A_BYTES;
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * SM::STAGE_BYTES);
          const int k0 = kb * BK;
          if (!A_MN) {
            tma_load_2d_cg2(sa, &tmA, &full[stage], k0, m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) tma_load_2d_cg2(sa + i * 64 * BK * 2, &tmA, &full[stage], m0 + 64 * i, k0);
          }
          if (!B_MN) {
            tma_load_2d_cg2_hint(sb, &tmB, &full[stage], k0, n0, polB);
          } else {
#pragma unroll
            for (int i = 0; i < (PAIR_N / 2) / 64; ++i)
              tma_load_2d_cg2_hint(sb + i * 64 * BK * 2, &tmB, &full[stage], n0 + 64 * i, k0, polB);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ===== MMA issuer (leader CTA only; whole warp, one elected lane issues)
      constexpr uint32_t idesc = make_idesc(2 * BM, PAIR_N, A_MN, B_MN);
      constexpr uint32_t KSTEP_A = A_MN ? UMMA_K * 128 : UMMA_K * 2, KSTEP_B = B_MN ? UMMA_K * 128 : UMMA_K * 2;
      const bool leader = elect_one();
      const uint64_t ad0 = A_MN ? make_desc(smem_u32(smem), 64 * BK * 2, 1024) : make_desc(smem_u32(smem), 16, 1024);
      const uint64_t bd0 = B_MN ? make_desc(smem_u32(smem) + SM::A_BYTES, 64 * BK * 2, 1024)
                                : make_desc(smem_u32(smem) + SM::A_BYTES, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < num_tiles; t += npairs, ++it) {
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);     // both CTAs drained this accumulator stage
        fence_after();
        const uint32_t dtm = tmem_base + as * PAIR_N;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint64_t ad = desc_add(ad0, stage * SM::STAGE_BYTES), bd = desc_add(bd0, stage * SM::STAGE_BYTES);
          if (leader) {
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k)
              umma_f16_cg2(dtm, desc_add(ad, k * KSTEP_A), desc_add(bd, k * KSTEP_B), idesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_cg2_mc(&empty[stage], 0x3);   // frees this smem slot in both CTAs
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (leader) umma_commit_cg2_mc(&tfull[as], 0x3);        // accumulator ready in both CTAs
        __syncwarp();
      }
    }
  } else if (warp >= EPI_WARP0) {  // ===== epilogue (both CTAs, each its own 128 rows)
    const uint32_t leader_tempty = mapa(smem_u32(tempty), 0);
    epilogue_loop<PAIR_N, TMA_EPI>(g, em, smem + SM::EPI_OFF, ebar, tfull, tmem_base, num_tiles, pair, npairs,
                                   (int)rank * BM, 2 * BM, [&](int t, int& mb, int& nb) { tile_coords(t, mb, nb); },
                                   [&](int as) { mbar_arrive_cluster(leader_tempty + as * 8); });
  }
  fence_before();
  cluster_sync();
  if (warp == 2) {
    fence_after();
    tmem_dealloc_cg2(tmem_base, SM::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
// 2-D tensor map: dim0 (contiguous) = inner, dim1 = outer, row stride in elements.
static cudaError_t make_map(CUtensorMap* map, const void* ptr, DT dt, uint64_t inner, uint64_t outer, uint64_t ld,
                            uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  auto enc = tcu::tmap_encoder();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t es = dt_size(dt);
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * es) & 15)) return cudaErrorMisalignedAddress;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t el[2] = {1, 1};
  CUresult r = enc(map, dt == DT::F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(ptr), dims, strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 32 x 32 staging-box map of an [M][N] epilogue tensor (f32: 128B swizzle, bf16: 64B swizzle)
static bool box_map(CUtensorMap* m, const void* ptr, DT dt, int M, int N, int64_t ld) {
  return make_map(m, ptr, dt, (uint64_t)N, (uint64_t)M, (uint64_t)ld, EPI_TILE, EPI_TILE,
                  dt == DT::F32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) == cudaSuccess;
}

// Build the staged-epilogue maps; false = shape / layout not eligible (use the direct path).
static bool epi_maps(const GemmArgs& g, EpiMaps* em) {
  const Epi& e = g.epi;
  if (e.res && e.acc_in) return false;
  if (!box_map(&em->out, e.out, e.out_dt, g.M, g.N, e.ldo)) return false;
  em->aux = em->out;
  em->in = em->out;
  if (e.kind == EPI_GELU_FWD) {
    if (e.out_dt != DT::BF16 || (e.aux && e.aux_dt != DT::BF16)) return false;
    if (e.aux && !box_map(&em->aux, e.aux, e.aux_dt, g.M, g.N, e.ldaux)) return false;
  } else if (e.kind == EPI_GELU_BWD) {
    if (!box_map(&em->in, e.aux, e.aux_dt, g.M, g.N, e.ldaux)) return false;
  } else if (e.res) {
    if (!box_map(&em->in, e.res, DT::F32, g.M, g.N, e.ldr)) return false;
  } else if (e.acc_in) {
    if (!box_map(&em->in, e.acc_in, DT::F32, g.M, g.N, e.ldacc)) return false;
  }
  return true;
}

template <int BN, bool A_MN, bool B_MN, bool TMA_EPI>
static cudaError_t launch_k(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em, const GemmArgs& g,
                            const GemmArgs& ge, cudaStream_t st) {
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, TMA_EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN) * g.split_k;
  const int grid = std::min(tiles, num_sms());
  note_launch(), kern<<<grid, NUM_THREADS, Smem<BN>::TOTAL, st>>>(ta, tb, em, g, ge);
  return cudaGetLastError();
}

// split-K finish: out = epi(sum_{ks < S} ws[ks]) in split order (deterministic); 4 columns per thread
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int S, int M, int N,
                                                            const Epi e) {
  const int64_t MN = (int64_t)M * N, n4 = MN / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(ws)[i];
    for (int ks = 1; ks < S; ++ks) {
      const float4 b = reinterpret_cast<const float4*>(ws + ks * MN)[i];
      a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    }
    const int64_t m = (i * 4) / N, n = (i * 4) % N;
    float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (e.bias) v[j] += ld_elem(e.bias, n + j, e.bias_dt);
      if (e.res) v[j] += e.res[m * e.ldr + n + j];
      if (e.acc_in) v[j] += e.acc_in[m * e.ldacc + n + j];
      st_elem(e.out, m * e.ldo + n + j, e.out_dt, v[j]);
    }
  }
}

// Split count for a tile-starved GEMM: S minimising waves(tiles * S) / S (each split does 1/S of K), at least
// 8 k-blocks per split, workspace S M N floats within capacity; 1 = no split.
int choose_split(const GemmArgs& g, int tiles, int ns) {
  if (!g.splitk_ws || g.M % BM || g.N % 4 || g.epi.kind != EPI_STORE || tiles >= ns) return 1;
  const int nk = (g.K + BK - 1) / BK;
  int best = 1;
  double best_cost = 1.0;
  for (int S = 2; S <= 16; ++S) {
    if (nk / S < 8 || (int64_t)S * g.M * g.N > g.splitk_ws_floats) break;
    const double cost = (double)((tiles * S + ns - 1) / ns) / S + 0.02 * S;   // + the reduce pass
    if (cost < best_cost - 1e-9) best_cost = cost, best = S;
  }
  if (best > 1) {   // every split non-empty
    const int nkper = (nk + best - 1) / best;
    best = (nk + nkper - 1) / nkper;
  }
  return best;
}

template <int BN, bool A_MN, bool B_MN>
static cudaError_t launch(const GemmArgs& g0, cudaStream_t st) {
  GemmArgs g = g0;
  g.split_k = BN == 128 ? choose_split(g, ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN), num_sms()) : 1;
  if (g.split_k > 1) {   // partial sums into the workspace (plain fp32 stores), then the fixed-order reduce
    GemmArgs ge = g;
    ge.M = g.split_k * g.M;
    ge.epi = Epi{};
    ge.epi.out = g.splitk_ws;
    ge.epi.ldo = g.N;
    ge.epi.out_dt = DT::F32;
    CUtensorMap ta, tb;
    cudaError_t e;
    if (!A_MN) e = make_map(&ta, g.A, DT::BF16, g.K, g.M, g.lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    else e = make_map(&ta, g.A, DT::BF16, g.M, g.K, g.lda, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (e != cudaSuccess) return e;
    if (!B_MN) e = make_map(&tb, g.B, DT::BF16, g.K, g.N, g.ldb, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    else e = make_map(&tb, g.B, DT::BF16, g.N, g.K, g.ldb, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
    if (e != cudaSuccess) return e;
    EpiMaps em;
    if (epi_maps(ge, &em)) e = launch_k<BN, A_MN, B_MN, true>(ta, tb, em, g, ge, st);
    else memset(&em, 0, sizeof(em)), e = launch_k<BN, A_MN, B_MN, false>(ta, tb, em, g, ge, st);
    if (e != cudaSuccess) return e;
    const int64_t n4 = (int64_t)g.M * g.N / 4;
    const int grid = (int)std::min<int64_t>((n4 + 255) / 256, (int64_t)num_sms() * 4);
    note_launch(), splitk_reduce_kernel<<<grid, 256, 0, st>>>(g.splitk_ws, g.split_k, g.M, g.N, g.epi);
    return cudaGetLastError();
  }
  g.split_k = 1;
  CUtensorMap ta, tb;
  cudaError_t e;
  if (!A_MN) e = make_map(&ta, g.A, DT::BF16, g.K, g.M, g.lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  else e = make_map(&ta, g.A, DT::BF16, g.M, g.K, g.lda, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  if (!B_MN) e = make_map(&tb, g.B, DT::BF16, g.K, g.N, g.ldb, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
  else e = make_map(&tb, g.B, DT::BF16, g.N, g.K, g.ldb, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  EpiMaps em;
  if (epi_maps(g, &em)) return launch_k<BN, A_MN, B_MN, true>(ta, tb, em, g, g, st);
  memset(&em, 0, sizeof(em));
  return launch_k<BN, A_MN, B_MN, false>(ta, tb, em, g, g, st);
}

template <bool A_MN, bool B_MN, bool TMA_EPI>
static cudaError_t launch2_k(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em, const GemmArgs& g,
                             cudaStream_t st) {
  auto kern = gemm_tc2_kernel<A_MN, B_MN, TMA_EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem2::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + PAIR_N - 1) / PAIR_N);
  const int pairs = std::min(tiles, num_sms() / 2);
  note_launch(), kern<<<2 * pairs, NUM_THREADS, Smem2::TOTAL, st>>>(ta, tb, em, g);
  return cudaGetLastError();
}

template <bool A_MN, bool B_MN>
static cudaError_t launch2(const GemmArgs& g, cudaStream_t st) {
  CUtensorMap ta, tb;
  cudaError_t e;
  if (!A_MN) e = make_map(&ta, g.A, DT::BF16, g.K, g.M, g.lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  else e = make_map(&ta, g.A, DT::BF16, g.M, g.K, g.lda, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  if (!B_MN) e = make_map(&tb, g.B, DT::BF16, g.K, g.N, g.ldb, BK, PAIR_N / 2, CU_TENSOR_MAP_SWIZZLE_128B);
  else e = make_map(&tb, g.B, DT::BF16, g.N, g.K, g.ldb, 64, BK, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e != cudaSuccess) return e;
  EpiMaps em;
  if (epi_maps(g, &em)) return launch2_k<A_MN, B_MN, true>(ta, tb, em, g, st);
  memset(&em, 0, sizeof(em));
  return launch2_k<A_MN, B_MN, false>(ta, tb, em, g, st);
}

}  // namespace tc

static int gemm_mode() {   // LGA_GEMM_PAIR=0 forces the single-CTA kernel (A/B comparisons)
  static int m = -1;
  if (m < 0) {
    const char* v = getenv("LGA_GEMM_PAIR");
    m = (v && v[0] == '0') ? 0 : 1;
  }
  return m;
}

cudaError_t gemm_bf16_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.K <= 0) return cudaErrorInvalidValue;
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  GemmArgs& gm = const_cast<GemmArgs&>(g);
  gm.b_keep_l2 = (int64_t)g.N * g.K * 2 <= (int64_t)48 << 20;   // weights (<= 48 MB), not activation gradients
  // Kernel choice by a wave-count cost model: per-SM work of one wave (pair tile: 128 x 256 per SM) times
  // the number of waves, over the kernel's relative per-SM throughput (CTA pair 1.0, single-CTA 128 x 256
  // 0.85, 128 x 128 0.70 -- measured kbench ratios).  A pair wave that leaves SMs idle can still beat a
  // second, partly empty wave of smaller tiles (the O-projection weight gradient: 64 pair tiles).
  const int ns = num_sms();
  const int tiles256 = ((g.M + 127) / 128) * ((g.N + 255) / 256);
  const int tiles128 = ((g.M + 127) / 128) * ((g.N + 127) / 128);
  const int pair_tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256);
  const double c_pair = (double)((pair_tiles + ns / 2 - 1) / (ns / 2)) * 2.0 / 1.0;
  const double c_256 = (double)((tiles256 + ns - 1) / ns) * 2.0 / 0.85;
  double c_128 = (double)((tiles128 + ns - 1) / ns) * 1.0 / 0.70;
  const int split = tc::choose_split(g, tiles128, ns);   // tile-starved: 128 x 128 tiles split over K
  if (split > 1) c_128 = ((double)((tiles128 * split + ns - 1) / ns) / split + 0.02 * split) / 0.70;
  const bool wide = g.N > 128 && c_256 < c_128;
  if (gemm_mode() == 1 && g.N > 128 && c_pair <= std::min(c_256, c_128))
    return amn ? (bmn ? tc::launch2<true, true>(g, st) : tc::launch2<true, false>(g, st))
               : (bmn ? tc::launch2<false, true>(g, st) : tc::launch2<false, false>(g, st));
#define L(BN) (amn ? (bmn ? tc::launch<BN, true, true>(g, st) : tc::launch<BN, true, false>(g, st)) \
                   : (bmn ? tc::launch<BN, false, true>(g, st) : tc::launch<BN, false, false>(g, st)))
  return wide ? L(256) : L(128);
#undef L
}

}  // namespace lga
