// epilogue.cuh -- the fused GEMM epilogues, shared by the fp32 SIMT and the bf16 tcgen05 GEMM.
//
// Each GEMM of the layer ends in one of these, so that no separate elementwise pass touches
// HBM (BASELINE.json north star, subsystem (2)):
//   QKV fwd      out(E)   = acc + bqkv
//   O / FFN2 fwd out(f32) = acc + b + residual            (h1 = x + o Wo + bo ; y = h1 + g W2 + b2)
//   FFN1 fwd     aux(E)   = u = acc + b1 ; out(E) = GELU(u)
//   FFN2 dgrad   out(E)   = acc * GELU'(u)                (dU = (dY W2^T) * GELU'(u))
//   dgrads       out      = acc
//   wgrads       out      = acc [+ acc_in]                (layered gradient accumulation:
//                 the fp32 per-layer buffer accumulates each chunk of micro-batches in place;
//                 the last chunk writes acc_in + acc cast to the reduce-scatter dtype)
#pragma once

#include "kernels.cuh"

namespace lga {

__device__ __forceinline__ void epi_store(const Epi& e, int64_t m, int64_t n, float v) {
  if (e.kind == EPI_STORE) {
    if (e.bias) v += ld_elem(e.bias, n, e.bias_dt);
    if (e.res) v += e.res[m * e.ldr + n];
    if (e.acc_in) v += e.acc_in[m * e.ldacc + n];
    st_elem(e.out, m * e.ldo + n, e.out_dt, v);
  } else if (e.kind == EPI_GELU_FWD) {
    const float u = v + ld_elem(e.bias, n, e.bias_dt);
    if (e.aux) st_elem(e.aux, m * e.ldaux + n, e.aux_dt, u);   // aux == nullptr: the pre-activation is not kept
    st_elem(e.out, m * e.ldo + n, e.out_dt, gelu_f(u));
  } else {  // EPI_GELU_BWD
    const float u = ld_elem(e.aux, m * e.ldaux + n, e.aux_dt);
    st_elem(e.out, m * e.ldo + n, e.out_dt, v * gelu_grad_f(u));
  }
}

}  // namespace lga
