// dgemm.cu — fp64 GEMM on the FP64 tensor cores (mma.sync m8n8k4 .f64 -> DMMA).
//
// C = alpha * op(A) * op(B) + beta * C, row-major, op = transpose on request.
// Used by the on-device LB-ADMM for every dense product the reference computes
// with its naive loops (dense.cpp:60-100): the Gram fixed^T fixed, the
// projection target * fixed, the Cholesky trailing updates, the blocked
// triangular-solve updates, the refinement residual and U V^T.
// The ADMM must stay in fp64 end to end (SURVEY.md §0 finding 1): tcgen05 has no
// f64 kind, so DMMA is the tensor-core path for it.
//
// Tiling: 128x64 block tile, BK=16, 256 threads = 8 warps as 4 (M) x 2 (N),
// each warp 32x32 = 4x4 m8n8 DMMA tiles (16 fp64 accumulators x 2 per lane).
// Global->register prefetch of the next k-tile overlaps the DMMAs; shared tiles are k-inner
// with one double of padding.  Accumulation order per output is fixed, so
// results are bitwise deterministic.
#include "common.cuh"

namespace nqb {

constexpr int DG_BM = 128, DG_BN = 64, DG_BK = 16;
constexpr int DG_LDS = DG_BK + 1;

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Loads the op(A) tile (rows m0.., k0..) into registers: element (i, kk) of
// op(A).  TA: op(A)[i][k] = A[k*lda + i]; else A[i*lda + k].
template <bool TA>
__device__ __forceinline__ void dg_load_a(const double* __restrict__ A, uint32_t lda,
                                          uint32_t M, uint32_t K, uint32_t m0, uint32_t k0,
                                          double (&ra)[8]) {
  // 128 x 16 = 2048 elements / 256 threads = 8 each
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t e = threadIdx.x + q * 256;
    uint32_t i, kk;
    if (TA) {  // coalesce along i
      i = e % DG_BM;
      kk = e / DG_BM;
    } else {   // coalesce along k
      kk = e % DG_BK;
      i = e / DG_BK;
    }
    const uint32_t gi = m0 + i, gk = k0 + kk;
    double v = 0.0;
    if (gi < M && gk < K) v = TA ? A[(uint64_t)gk * lda + gi] : A[(uint64_t)gi * lda + gk];
    ra[q] = v;
  }
}

template <bool TA>
__device__ __forceinline__ void dg_store_a(double* As, const double (&ra)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t e = threadIdx.x + q * 256;
    uint32_t i, kk;
    if (TA) {
      i = e % DG_BM;
      kk = e / DG_BM;
    } else {
      kk = e % DG_BK;
      i = e / DG_BK;
    }
    As[i * DG_LDS + kk] = ra[q];
  }
}

// op(B) tile (k0.., cols n0..): element (kk, j).  TB: op(B)[k][j] = B[j*ldb + k].
template <bool TB>
__device__ __forceinline__ void dg_load_b(const double* __restrict__ B, uint32_t ldb,
                                          uint32_t N, uint32_t K, uint32_t n0, uint32_t k0,
                                          double (&rb)[4]) {
  // 16 x 64 = 1024 elements / 256 threads = 4 each
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t e = threadIdx.x + q * 256;
    uint32_t j, kk;
    if (TB) {  // coalesce along k
      kk = e % DG_BK;
      j = e / DG_BK;
    } else {   // coalesce along j
      j = e % DG_BN;
      kk = e / DG_BN;
    }
    const uint32_t gj = n0 + j, gk = k0 + kk;
    double v = 0.0;
    if (gj < N && gk < K) v = TB ? B[(uint64_t)gj * ldb + gk] : B[(uint64_t)gk * ldb + gj];
    rb[q] = v;
  }
}

template <bool TB>
__device__ __forceinline__ void dg_store_b(double* Bs, const double (&rb)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t e = threadIdx.x + q * 256;
    uint32_t j, kk;
    if (TB) {
      kk = e % DG_BK;
      j = e / DG_BK;
    } else {
      j = e % DG_BN;
      kk = e / DG_BN;
    }
    Bs[j * DG_LDS + kk] = rb[q];
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm(uint32_t M, uint32_t N, uint32_t K, double alpha,
                                               const double* __restrict__ A, uint32_t lda,
                                               const double* __restrict__ B, uint32_t ldb,
                                               double beta, double* __restrict__ C,
                                               uint32_t ldc) {
  __shared__ double As[DG_BM * DG_LDS];
  __shared__ double Bs[DG_BN * DG_LDS];
  const uint32_t m0 = blockIdx.y * DG_BM, n0 = blockIdx.x * DG_BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  double ra[8], rb[4];
  dg_load_a<TA>(A, lda, M, K, m0, 0, ra);
  dg_load_b<TB>(B, ldb, N, K, n0, 0, rb);
  dg_store_a<TA>(As, ra);
  dg_store_b<TB>(Bs, rb);
  __syncthreads();

  const uint32_t ktiles = (K + DG_BK - 1) / DG_BK;
  for (uint32_t kt = 0; kt < ktiles; ++kt) {
    if (kt + 1 < ktiles) {
      dg_load_a<TA>(A, lda, M, K, m0, (kt + 1) * DG_BK, ra);
      dg_load_b<TB>(B, ldb, N, K, n0, (kt + 1) * DG_BK, rb);
    }
    const double* as = As;
    const double* bs = Bs;
#pragma unroll
    for (int k4 = 0; k4 < DG_BK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = as[(wm + a * 8 + fr) * DG_LDS + k4 + fk];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = bs[(wn + b * 8 + fr) * DG_LDS + k4 + fk];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
    if (kt + 1 < ktiles) {
      dg_store_a<TA>(As, ra);
      dg_store_b<TB>(Bs, rb);
      __syncthreads();
    }
  }

#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const uint32_t gi = m0 + wm + a * 8 + fr;
    if (gi >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t gj = n0 + wn + b * 8 + fk * 2 + h;
        if (gj >= N) continue;
        double* cp = C + (uint64_t)gi * ldc + gj;
        const double v = alpha * acc[a][b][h];
        *cp = (beta == 0.0) ? v : v + beta * *cp;
      }
    }
  }
}

void dgemm(nqb_context* ctx, bool ta, bool tb, uint32_t M, uint32_t N, uint32_t K, double alpha,
           const double* A, uint32_t lda, const double* B, uint32_t ldb, double beta, double* C,
           uint32_t ldc) {
  if (M == 0 || N == 0) return;
  dim3 grid(ceil_div(N, DG_BN), ceil_div(M, DG_BM));
  NQB_REQUIRE(grid.y <= 65535, NQB_E_VALIDATION, "dgemm: M too large");
  if (!ta && !tb)
    k_dgemm<false, false><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (ta && !tb)
    k_dgemm<true, false><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else if (!ta && tb)
    k_dgemm<false, true><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  else
    k_dgemm<true, true><<<grid, 256, 0, ctx->stream>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
  NQB_LAUNCHED(ctx);
}

}  // namespace nqb

extern "C" int nqb_dgemm_device(nqb_context* ctx, int trans_a, int trans_b, uint32_t m,
                                uint32_t n, uint32_t k, double alpha, const double* d_a,
                                uint32_t lda, const double* d_b, uint32_t ldb, double beta,
                                double* d_c, uint32_t ldc) {
  try {
    NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
    nqb::dgemm(ctx, trans_a != 0, trans_b != 0, m, n, k, alpha, d_a, lda, d_b, ldb, beta, d_c,
               ldc);
    return NQB_OK;
  } catch (const nqb::Failure& f) {
    nqb::set_error(f.msg);
    return f.code;
  }
}
