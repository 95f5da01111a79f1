// k_attn_bf16.cu -- bf16 flash attention forward / backward (placeholder for the next milestone).
#include "kernels.cuh"

namespace lga {
void attn_fwd_bf16(const AttnArgs&, cudaStream_t) {}
void attn_bwd_bf16(const AttnArgs&, cudaStream_t) {}
}  // namespace lga
