// decode.cu — batch-1 decode GEMV entry points (the HBM-bound hot kernel).
// v1: the two-stage CUDA-core bit-row kernels of forward_simt.cu.
#include "common.cuh"

namespace nqb {

template <typename Acc, typename In>
void simt_gemv(nqb_context*, const nqb_layer*, const In*, Acc*);

__global__ void k_f32_to_f16(const float* __restrict__ in, __half* __restrict__ out,
                             uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = __float2half_rn(in[i]);
}

void decode_gemv_f32(nqb_context* ctx, const nqb_layer* L, const float* d_x, float* d_y) {
  simt_gemv<float, float>(ctx, L, d_x, d_y);
}

void decode_gemv_f16(nqb_context* ctx, const nqb_layer* L, const __half* d_x, __half* d_y) {
  float* y32 = (float*)scratch(ctx, 2, sizeof(float) * L->n);
  simt_gemv<float, __half>(ctx, L, d_x, y32);
  k_f32_to_f16<<<ceil_div(L->n, 256), 256, 0, ctx->stream>>>(y32, d_y, L->n);
  NQB_LAUNCHED(ctx);
}

}  // namespace nqb
