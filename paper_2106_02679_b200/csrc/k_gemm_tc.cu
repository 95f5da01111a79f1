// k_gemm_tc.cu -- bf16 GEMM on the 5th-generation tensor cores, sm_100a:
//   TMA (cp.async.bulk.tensor, 128B swizzle) -> shared memory ring (STAGES deep)
//   -> tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) issued by one thread, fp32 accumulators in TMEM
//   -> tcgen05.ld by 4 epilogue warps -> fused epilogue (epilogue.cuh) -> global.
// Persistent, warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warps 4..7 = epilogue.  Two TMEM accumulator stages so that the epilogue of tile t overlaps the
// MMAs of tile t+1.  Operands may be K-major or MN-major independently (UMMA descriptor major bit), so
// forward (X W), dgrad (dY W^T) and wgrad (X^T dY) all read their operands in place -- no transposes.
#include "epilogue.cuh"
#include "tc_common.cuh"

namespace lga {

namespace tc {

using namespace tcu;

constexpr int BM = 128;
constexpr int BK = 64;           // 64 bf16 = 128 bytes = one swizzle span
constexpr int UMMA_K = 16;
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;    // two warps per TMEM lane quadrant, each drains half of the tile's columns
constexpr int NUM_THREADS = (EPI_WARP0 + EPI_WARPS) * 32;

template <int BN>
struct Smem {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;   // two accumulator stages
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + 256 + 1024;   // + barriers + alignment slack
};

// ---- vectorised epilogue of 32 consecutive columns of one row (falls back to scalar at edges)
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
    for (int i = 0; i < 4; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(x[8 * i + 2 * j], x[8 * i + 2 * j + 1]);
        w[j] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      p[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

__device__ __forceinline__ void epi_chunk(const Epi& e, int64_t m, int64_t n0, int nvalid, float (&v)[32]) {
  bool vec = nvalid == 32 && aligned16(static_cast<char*>(e.out) + (m * e.ldo + n0) * (int64_t)dt_size(e.out_dt));
  if (vec && e.kind == EPI_STORE) {
    if (e.bias) vec = aligned16(static_cast<const char*>(e.bias) + n0 * (int64_t)dt_size(e.bias_dt));
    if (e.res) vec = vec && aligned16(e.res + m * e.ldr + n0);
    if (e.acc_in) vec = vec && aligned16(e.acc_in + m * e.ldacc + n0);
  } else if (vec) {
    vec = aligned16(static_cast<char*>(e.aux) + (m * e.ldaux + n0) * (int64_t)dt_size(e.aux_dt));
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
    store32(e.aux, e.aux_dt, m * e.ldaux + n0, v);
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

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
  using SM = Smem<BN>;
  constexpr int STAGES = SM::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (g.M + BM - 1) / BM, num_n = (g.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int nk = (g.K + BK - 1) / BK;
  constexpr int GM = 8;   // tile raster: groups of GM m-blocks sweep all n-blocks (L2 reuse of B)

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], EPI_WARPS); }
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
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        for (int kb = 0; kb < nk; ++kb) {
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
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_2d(sb + i * 64 * BK * 2, &tmB, &full[stage], n0 + 64 * i, k0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer (single thread)
      constexpr uint32_t idesc = make_idesc(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[as], aphase ^ 1);
        fence_after();
        const uint32_t dtm = tmem_base + as * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          fence_after();
          const uint32_t sa = smem_u32(smem + stage * SM::STAGE_BYTES);
          const uint32_t sb = sa + SM::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            // K-major: advance 16 elements = 32 B inside the swizzle span; MN-major: 16 K-rows = 2048 B
            const uint64_t ad = A_MN ? make_desc(sa + k * UMMA_K * 128, 64 * BK * 2, 1024)
                                     : make_desc(sa + k * UMMA_K * 2, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(sb + k * UMMA_K * 128, 64 * BK * 2, 1024)
                                     : make_desc(sb + k * UMMA_K * 2, 16, 1024);
            umma_f16(dtm, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);   // frees the smem slot when these MMAs complete
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[as]);        // accumulator ready for the epilogue
      }
    }
  } else if (warp >= EPI_WARP0) {  // ===== epilogue: TMEM -> registers -> fused epilogue -> global
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int half = (warp - EPI_WARP0) >> 2;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int mb, nb;
      tile_coords(t, mb, nb);
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait(&tfull[as], aphase);
      fence_after();
      const int64_t m = (int64_t)mb * BM + q * 32 + lane;
      const uint32_t taddr = tmem_base + as * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int ch = half * (BN / 64); ch < (half + 1) * (BN / 64); ++ch) {
        float v[32];
        tmem_ld32(taddr + ch * 32, v);
        const int64_t n0 = (int64_t)nb * BN + ch * 32;
        if (m < g.M && n0 < g.N) {
          const int nvalid = (int)(g.N - n0 < 32 ? g.N - n0 : 32);
          epi_chunk(g.epi, m, n0, nvalid, v);
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    tmem_dealloc(tmem_base, SM::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
// 2-D bf16 tensor map: dim0 (contiguous) = inner, dim1 = outer, row stride in elements.
static cudaError_t make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                            uint32_t box_inner, uint32_t box_outer) {
  auto enc = tcu::tmap_encoder();
  if (!enc) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 2) & 15)) return cudaErrorMisalignedAddress;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN, bool A_MN, bool B_MN>
static cudaError_t launch(const GemmArgs& g, cudaStream_t st) {
  CUtensorMap ta, tb;
  cudaError_t e;
  if (!A_MN) e = make_map(&ta, g.A, g.K, g.M, g.lda, BK, BM);
  else e = make_map(&ta, g.A, g.M, g.K, g.lda, 64, BK);
  if (e != cudaSuccess) return e;
  if (!B_MN) e = make_map(&tb, g.B, g.K, g.N, g.ldb, BK, BN);
  else e = make_map(&tb, g.B, g.N, g.K, g.ldb, 64, BK);
  if (e != cudaSuccess) return e;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<BN>::TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
  const int grid = std::min(tiles, num_sms());
  note_launch(), kern<<<grid, NUM_THREADS, Smem<BN>::TOTAL, st>>>(ta, tb, g);
  return cudaGetLastError();
}

}  // namespace tc

cudaError_t gemm_bf16_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.K <= 0) return cudaErrorInvalidValue;
  const bool amn = !g.a_kmajor, bmn = !g.b_kmajor;
  // BN = 256 when there are enough tiles to fill the machine, else 128
  const int tiles256 = ((g.M + 127) / 128) * ((g.N + 255) / 256);
  const bool wide = g.N > 128 && tiles256 >= num_sms();
#define L(BN) (amn ? (bmn ? tc::launch<BN, true, true>(g, st) : tc::launch<BN, true, false>(g, st)) \
                   : (bmn ? tc::launch<BN, false, true>(g, st) : tc::launch<BN, false, false>(g, st)))
  return wide ? L(256) : L(128);
#undef L
}

}  // namespace lga
