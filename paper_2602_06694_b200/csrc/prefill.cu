// prefill.cu — batched (prefill) forward Y = s1 .* U (V^T (s2 .* X)).
// v1: CUDA-core bit-row GEMM with layout conversion kernels.
#include "common.cuh"

namespace nqb {

void simt_gemm_f32(nqb_context*, const nqb_layer*, const float*, uint32_t, float*);

// X: b x m token-major half -> A: m x b j-major fp32 scaled by s2.
__global__ void k_tokens_to_jmajor(const __half* __restrict__ x, const __half* __restrict__ s2h,
                                   uint32_t m, uint32_t b, float* __restrict__ a) {
  __shared__ float tile[32][33];
  const uint32_t j0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t c = c0 + k, j = j0 + tx;
    tile[k][tx] = (c < b && j < m) ? __half2float(x[(uint64_t)c * m + j]) : 0.f;
  }
  __syncthreads();
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t j = j0 + k, c = c0 + tx;
    if (j < m && c < b) a[(uint64_t)j * b + c] = __half2float(s2h[j]) * tile[tx][k];
  }
}

// Y32: n x b fp32 -> Y: b x n half (token-major).
__global__ void k_jmajor_to_tokens(const float* __restrict__ y32, uint32_t n, uint32_t b,
                                   __half* __restrict__ y) {
  __shared__ float tile[32][33];
  const uint32_t i0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t i = i0 + k, c = c0 + tx;
    tile[k][tx] = (i < n && c < b) ? y32[(uint64_t)i * b + c] : 0.f;
  }
  __syncthreads();
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t c = c0 + k, i = i0 + tx;
    if (c < b && i < n) y[(uint64_t)c * n + i] = __float2half_rn(tile[tx][k]);
  }
}

void prefill_gemm_f16(nqb_context* ctx, const nqb_layer* L, const __half* d_x, uint32_t b,
                      __half* d_y) {
  float* a = (float*)scratch(ctx, 3, sizeof(float) * (uint64_t)L->m * b);
  float* y32 = (float*)scratch(ctx, 4, sizeof(float) * (uint64_t)L->n * b);
  k_tokens_to_jmajor<<<dim3(ceil_div(L->m, 32), ceil_div(b, 32)), 256, 0, ctx->stream>>>(
      d_x, L->s2h, L->m, b, a);
  NQB_LAUNCHED(ctx);
  simt_gemm_f32(ctx, L, a, b, y32);
  k_jmajor_to_tokens<<<dim3(ceil_div(L->n, 32), ceil_div(b, 32)), 256, 0, ctx->stream>>>(
      y32, L->n, b, d_y);
  NQB_LAUNCHED(ctx);
}

}  // namespace nqb
