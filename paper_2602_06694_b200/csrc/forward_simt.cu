// forward_simt.cu — CUDA-core forward kernels (two-stage, packed.cpp:153-287).
//
// These are the exact-arithmetic paths behind the drop-in host entry points:
//   gemv_packed      (packed.cpp:196-199)  fp64 accumulation
//   gemv_packed_f32  (packed.cpp:201-204)  fp32 accumulation
//   gemm_packed      (packed.cpp:260-287)  fp64 accumulation, batched
// and the fallback-free correctness baseline the tensor-core decode/prefill
// kernels (decode_tc.cu, prefill_tc.cu) are measured against.
//
// Both stages are one kernel shape, a "bit-row dot":
//   out[row] = scale(row) * sum_j sign(bits[row][j]) * act[j]
// stage 1: bits = V^T (r rows), act = s2 .* x      -> t (length r)
// stage 2: bits = U   (n rows), act = t, scale=s1  -> y (length n)
// Activations are staged in shared memory transposed ([bit][word]) so a warp
// reading bit b of 32 consecutive words hits 32 consecutive banks.
#include "common.cuh"

namespace nqb {

// a[j] = (Acc)s2[j] * (Acc)x[j] for j < m, 0 for m <= j < padded.
template <typename Acc, typename In>
__global__ void k_scale_input(const In* __restrict__ x, const __half* __restrict__ s2h,
                              const double* __restrict__ s2d, uint32_t m, uint32_t padded,
                              Acc* __restrict__ a) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < padded;
       j += gridDim.x * blockDim.x) {
    Acc v = Acc(0);
    if (j < m) {
      Acc xv;
      if constexpr (std::is_same<In, __half>::value) xv = (Acc)__half2float(x[j]);
      else xv = (Acc)x[j];
      v = (s2d ? (Acc)s2d[j] : (Acc)__half2float(s2h[j])) * xv;
    }
    a[j] = v;
  }
}

constexpr int kChunkWords = 128;  // 4096 activations per shared-memory chunk

template <typename Acc>
__global__ void __launch_bounds__(256) k_bitrow_dot(const uint32_t* __restrict__ bits,
                                                    uint32_t stride, uint32_t rows,
                                                    uint32_t words, const Acc* __restrict__ act,
                                                    const __half* __restrict__ row_scale,
                                                    const double* __restrict__ row_scale_d,
                                                    Acc* __restrict__ out) {
  __shared__ Acc act_s[32][kChunkWords + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t row = blockIdx.x * 8 + warp;
  Acc acc = Acc(0);
  for (uint32_t c0 = 0; c0 < words; c0 += kChunkWords) {
    const uint32_t cw = min((uint32_t)kChunkWords, words - c0);
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < cw * 32; e += blockDim.x) {
      act_s[e & 31][e >> 5] = act[(uint64_t)c0 * 32 + e];
    }
    __syncthreads();
    if (row < rows) {
      const uint32_t* brow = bits + (uint64_t)row * stride + c0;
      for (uint32_t w = lane; w < cw; w += 32) {
        const uint32_t word = brow[w];
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const Acc v = act_s[b][w];
          acc += ((word >> b) & 1u) ? v : -v;
        }
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0 && row < rows) {
    out[row] = row_scale_d ? (Acc)row_scale_d[row] * acc
                           : row_scale ? (Acc)__half2float(row_scale[row]) * acc : acc;
  }
}

// Batched: out[row][c] = scale(row) * sum_j sign(bits[row][j]) * act[j][c]
// act is j-major with leading dimension ld (>= b); 32 columns per block.
template <typename Acc, int J = (sizeof(Acc) == 8 ? 128 : 256)>
__global__ void __launch_bounds__(256) k_bitrow_gemm(const uint32_t* __restrict__ bits,
                                                     uint32_t stride, uint32_t rows,
                                                     uint32_t nact, const Acc* __restrict__ act,
                                                     uint32_t ld, uint32_t b,
                                                     const __half* __restrict__ row_scale,
                                                     const double* __restrict__ row_scale_d,
                                                     Acc* __restrict__ out, uint32_t ldo) {
  __shared__ Acc act_s[J][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t c = blockIdx.y * 32 + lane;
  const uint32_t row0 = blockIdx.x * 32;
  Acc acc[4] = {Acc(0), Acc(0), Acc(0), Acc(0)};
  for (uint32_t j0 = 0; j0 < nact; j0 += J) {
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < J * 32; e += blockDim.x) {
      const uint32_t jj = e >> 5, cc = e & 31;
      const uint32_t gj = j0 + jj, gc = blockIdx.y * 32 + cc;
      act_s[jj][cc] = (gj < nact && gc < b) ? act[(uint64_t)gj * ld + gc] : Acc(0);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t row = row0 + warp * 4 + q;
      if (row >= rows) continue;
      const uint32_t* brow = bits + (uint64_t)row * stride + j0 / 32;
      const uint32_t lim = min((uint32_t)J, nact - j0);
      for (uint32_t w = 0; w * 32 < lim; ++w) {
        const uint32_t word = brow[w];
#pragma unroll 8
        for (int bb = 0; bb < 32; ++bb) {
          const Acc v = act_s[w * 32 + bb][lane];
          acc[q] += ((word >> bb) & 1u) ? v : -v;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t row = row0 + warp * 4 + q;
    if (row < rows && c < b) {
      const bool scaled = row_scale_d || row_scale;
      const Acc s = row_scale_d ? (Acc)row_scale_d[row]
                                : row_scale ? (Acc)__half2float(row_scale[row]) : Acc(1);
      out[(uint64_t)row * ldo + c] = scaled ? s * acc[q] : acc[q];
    }
  }
}

__global__ void k_scale_rows(const double* __restrict__ x, const __half* __restrict__ s2h,
                             const double* __restrict__ s2d, uint32_t m, uint32_t b,
                             double* __restrict__ a) {
  const uint64_t total = (uint64_t)m * b;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    a[e] = (s2d ? s2d[e / b] : (double)__half2float(s2h[e / b])) * x[e];
  }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
template <typename Acc, typename In>
void simt_gemv(nqb_context* ctx, const nqb_layer* L, const In* d_x, Acc* d_y) {
  const uint32_t apad = L->vt_words * 32;
  const uint32_t tpad = L->u_words * 32;
  Acc* a = (Acc*)scratch(ctx, 0, sizeof(Acc) * (apad + tpad));
  Acc* t = a + apad;
  k_scale_input<Acc, In><<<ceil_div(apad, 256), 256, 0, ctx->stream>>>(d_x, L->s2h, L->s2d, L->m, apad, a);
  NQB_LAUNCHED(ctx);
  if (tpad > L->r) {
    NQB_CUDA(cudaMemsetAsync(t + L->r, 0, sizeof(Acc) * (tpad - L->r), ctx->stream));
  }
  k_bitrow_dot<Acc><<<ceil_div(L->r, 8), 256, 0, ctx->stream>>>(L->vt, L->vt_words, L->r,
                                                              L->vt_words, a, nullptr, nullptr, t);
  NQB_LAUNCHED(ctx);
  k_bitrow_dot<Acc><<<ceil_div(L->n, 8), 256, 0, ctx->stream>>>(L->u, L->u_words, L->n,
                                                              L->u_words, t, L->s1h, L->s1d, d_y);
  NQB_LAUNCHED(ctx);
}

template void simt_gemv<float, float>(nqb_context*, const nqb_layer*, const float*, float*);
template void simt_gemv<double, double>(nqb_context*, const nqb_layer*, const double*, double*);

// X: m x b (j-major) fp64 device -> Y: n x b fp64 device.
void simt_gemm_f64(nqb_context* ctx, const nqb_layer* L, const double* d_x, uint32_t b,
                   double* d_y) {
  // A = s2 .* X (row scale of X), T = V^T A, Y = s1 .* U T
  const uint64_t a_elems = (uint64_t)L->m * b, t_elems = (uint64_t)L->r * b;
  double* a = (double*)scratch(ctx, 0, sizeof(double) * (a_elems + t_elems));
  double* t = a + a_elems;
  k_scale_rows<<<ceil_div(a_elems, 256) > 4096 ? 4096 : ceil_div(a_elems, 256), 256, 0,
               ctx->stream>>>(d_x, L->s2h, L->s2d, L->m, b, a);
  NQB_LAUNCHED(ctx);
  dim3 g1(ceil_div(L->r, 32), ceil_div(b, 32));
  k_bitrow_gemm<double><<<g1, 256, 0, ctx->stream>>>(L->vt, L->vt_words, L->r, L->m, a, b, b,
                                                     nullptr, nullptr, t, b);
  NQB_LAUNCHED(ctx);
  dim3 g2(ceil_div(L->n, 32), ceil_div(b, 32));
  k_bitrow_gemm<double><<<g2, 256, 0, ctx->stream>>>(L->u, L->u_words, L->n, L->r, t, b, b,
                                                     L->s1h, L->s1d, d_y, b);
  NQB_LAUNCHED(ctx);
}

}  // namespace nqb

namespace nqb {

template void simt_gemv<float, __half>(nqb_context*, const nqb_layer*, const __half*, float*);

// A: m x b j-major fp32, already scaled by s2; Y: n x b fp32 (n-major).
void simt_gemm_f32(nqb_context* ctx, const nqb_layer* L, const float* d_a, uint32_t b,
                   float* d_y) {
  float* t = (float*)scratch(ctx, 1, sizeof(float) * (uint64_t)L->r * b);
  dim3 g1(ceil_div(L->r, 32), ceil_div(b, 32));
  k_bitrow_gemm<float><<<g1, 256, 0, ctx->stream>>>(L->vt, L->vt_words, L->r, L->m, d_a, b, b,
                                                    nullptr, nullptr, t, b);
  NQB_LAUNCHED(ctx);
  dim3 g2(ceil_div(L->n, 32), ceil_div(b, 32));
  k_bitrow_gemm<float><<<g2, 256, 0, ctx->stream>>>(L->u, L->u_words, L->n, L->r, t, b, b,
                                                    L->s1h, L->s1d, d_y, b);
  NQB_LAUNCHED(ctx);
}

}  // namespace nqb
