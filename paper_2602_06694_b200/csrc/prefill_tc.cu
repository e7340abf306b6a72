// prefill_tc.cu — batched (prefill) BLR forward on 5th-generation tensor cores.
//
//   gemm_packed (packed.cpp:260-287):  Y = s1 .* U (V^T (s2 .* X))
//
// Each stage is one GEMM whose A operand is a packed sign matrix:
//   C[tokens][rows] = sum_k sign(A[rows][k]) * B[tokens][k]
// with A = V^T (rows = r, K = m) for stage 1 and A = U (rows = n, K = r) for
// stage 2.  Per CTA tile (128 rows x 256 tokens), four producer warps expand
// the tile's sign bits into +-1 binary16 in shared memory (canonical K-major
// core-matrix layout, SWIZZLE_NONE) and copy the binary16 token tile next to
// it; one thread issues `tcgen05.mma.cta_group::1.kind::f16` (M=128, N=256,
// K=16, fp32 accumulators in TMEM).  A 3-stage mbarrier pipeline overlaps the
// expansion/copies of K-tile k+1..k+2 with the MMAs of k.  The epilogue reads
// TMEM (tcgen05.ld), applies the row scale (s1) and writes token-major
// binary16.  At N = 256 one 4 KB A operand feeds 128x256x16 MACs, so unlike
// batch-1 decode the expansion is cheap relative to the math.
#include <algorithm>

#include "common.cuh"
#include "tc_common.cuh"

namespace nqb {
namespace pf {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 3;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int kProducers = 128;       // 4 warps; warp 4 issues the MMAs
constexpr uint32_t kTmemCols = 256;   // D: 128 lanes x 256 fp32 columns

struct Args {
  const uint32_t* bits;   // A sign bits: row-major, words_per_row u32 per row
  uint32_t wpr;           // words per A row
  uint32_t M;             // A rows (r or n)
  uint32_t Mvalid;        // rows >= Mvalid produce 0 (padding of r)
  uint32_t Mout;          // rows written (>= M: the zero padding stage 2 reads)
  uint32_t nk;            // K tiles (K padded to BK; B is zero beyond K)
  const __half* B;        // tokens x ldb binary16 (K contiguous)
  uint32_t ldb, N;        // N = tokens
  const __half* scale;    // per-row output scale (s1) or null
  __half* out;            // tokens x ldo binary16
  uint32_t ldo;
};

// byte offset of (row, 8-element K chunk k8 of the 64-wide K tile) in the
// canonical K-major layout of an R-row operand tile:
//   [kstep (16 K)][khalf (8 K)][row group (8 rows)][row][16 B]
__device__ __forceinline__ uint32_t canon(uint32_t row, uint32_t k8, uint32_t R) {
  const uint32_t ks = k8 >> 1, kh = k8 & 1;
  return ((ks * 2 + kh) * (R / 8) + (row >> 3)) * 128 + (row & 7) * 16;
}

struct __align__(8) Bars {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t dready;
  uint32_t tmem;
};

__global__ void __launch_bounds__(kProducers + 32, 1) k_prefill(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars* bars = (Bars*)smem;
  uint8_t* tiles = smem + 1024;  // STAGES x [A 16 KB | B 32 KB]
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const uint32_t m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&bars->full[s], kProducers);
      tc::mbar_init(&bars->empty[s], 1);
    }
    tc::mbar_init(&bars->dready, 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) {
    tc::tmem_alloc(&bars->tmem, kTmemCols);
    tc::tmem_relinquish();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = bars->tmem;

  if (warp == kProducers / 32) {  // ------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_f16(BM, BN);
      for (uint32_t kt = 0; kt < a.nk; ++kt) {
        const uint32_t slot = kt % STAGES;
        tc::mbar_wait(&bars->full[slot], (kt / STAGES) & 1);
        tc::fence_after_sync();
        const uint32_t abase = tc::smem_u32(tiles + slot * (A_BYTES + B_BYTES));
        const uint32_t bbase = abase + A_BYTES;
#pragma unroll
        for (uint32_t ks = 0; ks < BK / 16; ++ks) {
          const uint64_t ad = tc::smem_desc_kmajor(abase + ks * 2 * (BM / 8) * 128, (BM / 8) * 128, 128);
          const uint64_t bd = tc::smem_desc_kmajor(bbase + ks * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
          tc::mma_f16_ss(tmem, ad, bd, idesc, (kt | ks) ? 1u : 0u);
        }
        tc::mma_commit(&bars->empty[slot]);
      }
      tc::mma_commit(&bars->dready);
    }
  } else {  // ------------------------------------------------------ producers
    for (uint32_t kt = 0; kt < a.nk; ++kt) {
      const uint32_t slot = kt % STAGES, use = kt / STAGES;
      if (use > 0) tc::mbar_wait(&bars->empty[slot], (use - 1) & 1);
      uint8_t* As = tiles + slot * (A_BYTES + B_BYTES);
      uint8_t* Bs = As + A_BYTES;
      // A: 128 rows x 64 K signs -> +-1 binary16 (8 elements per 16-byte chunk)
#pragma unroll 2
      for (uint32_t c = tid; c < BM * (BK / 8); c += kProducers) {
        const uint32_t row = c >> 3, k8 = c & 7, k = kt * BK + k8 * 8;
        uint32_t byte = 0;
        if (m0 + row < a.M) byte = (__ldg(a.bits + (size_t)(m0 + row) * a.wpr + (k >> 5)) >> (k & 31)) & 0xFFu;
        uint4 v;
        uint32_t* pv = &v.x;
#pragma unroll
        for (int i = 0; i < 4; ++i)  // bit 1 -> +1 (0x3C00), 0 -> -1 (0xBC00)
          pv[i] = 0xBC00BC00u ^ (((byte >> (2 * i)) & 1u) << 15) ^ (((byte >> (2 * i + 1)) & 1u) << 31);
        *(uint4*)(As + canon(row, k8, BM)) = v;
      }
      // B: 256 tokens x 64 K binary16
#pragma unroll 4
      for (uint32_t c = tid; c < BN * (BK / 8); c += kProducers) {
        const uint32_t row = c >> 3, k8 = c & 7;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (n0 + row < a.N) v = __ldg((const uint4*)(a.B + (size_t)(n0 + row) * a.ldb + kt * BK + k8 * 8));
        *(uint4*)(Bs + canon(row, k8, BN)) = v;
      }
      tc::fence_proxy_async_smem();  // generic-proxy writes -> MMA (async proxy) reads
      tc::mbar_arrive(&bars->full[slot]);
    }
    // ------------------------------------------------------------- epilogue
    tc::mbar_wait(&bars->dready, 0);
    tc::fence_after_sync();
    const uint32_t row = warp * 32 + lane, grow = m0 + row;
    const float sc = (grow < a.Mvalid && a.scale) ? __half2float(a.scale[grow]) : 1.f;
    const bool keep = grow < a.Mvalid;
    for (uint32_t c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld_x16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      tc::wait_ld();
      if (grow < a.Mout) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t tok = n0 + c0 + j;
          if (tok < a.N)
            a.out[(size_t)tok * a.ldo + grow] =
                __float2half_rn(keep ? sc * __uint_as_float(v[j]) : 0.f);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

// X (b x m, binary16, token-major) -> s2 .* X with K padded to kpad (zeros).
__global__ void k_prescale(const __half* __restrict__ x, const __half* __restrict__ s2h,
                           uint32_t m, uint32_t b, uint32_t kpad, __half* __restrict__ out) {
  const uint64_t total = (uint64_t)b * kpad;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t tok = (uint32_t)(e / kpad), j = (uint32_t)(e % kpad);
    out[e] = j < m ? __float2half_rn(__half2float(s2h[j]) * __half2float(x[(size_t)tok * m + j]))
                   : __float2half_rn(0.f);
  }
}

}  // namespace pf

using namespace pf;

static void launch_stage(nqb_context* ctx, const Args& a, uint32_t grid_m, uint32_t grid_n) {
  static bool attr = false;
  if (!attr) {
    NQB_CUDA(cudaFuncSetAttribute(k_prefill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  1024 + STAGES * (A_BYTES + B_BYTES)));
    attr = true;
  }
  k_prefill<<<dim3(grid_m, grid_n), kProducers + 32, 1024 + STAGES * (A_BYTES + B_BYTES),
              ctx->stream>>>(a);
  NQB_LAUNCHED(ctx);
}

// X: b x m token-major binary16 (device), Y: b x n token-major binary16.
void prefill_gemm_tc(nqb_context* ctx, const nqb_layer* L, const __half* d_x, uint32_t b,
                     __half* d_y) {
  const uint32_t mpad = (L->m + BK - 1) / BK * BK, rpad = (L->r + BK - 1) / BK * BK;
  NQB_REQUIRE(L->vt_words * 32 >= mpad && L->u_words * 32 >= rpad, NQB_E_INTERNAL,
              "prefill: layer rows not padded to the K tile");
  __half* xs = (__half*)scratch(ctx, 3, sizeof(__half) * (size_t)b * mpad);
  __half* tt = (__half*)scratch(ctx, 4, sizeof(__half) * (size_t)b * rpad);
  const uint64_t tot = (uint64_t)b * mpad;
  pf::k_prescale<<<(uint32_t)std::min<uint64_t>((tot + 255) / 256, 148 * 16), 256, 0, ctx->stream>>>(
      d_x, L->s2h, L->m, b, mpad, xs);
  NQB_LAUNCHED(ctx);
  // stage 1: T^T[token][k] = sum_j sign(V[j][k]) * xs[token][j]   (rows k < r, padded rows 0)
  Args a1{L->vt, L->vt_words, L->r, L->r, rpad, mpad / BK, xs, mpad, b, nullptr, tt, rpad};
  launch_stage(ctx, a1, (rpad + BM - 1) / BM, (b + BN - 1) / BN);
  // stage 2: Y[token][i] = s1_i * sum_k sign(U[i][k]) * T^T[token][k]
  Args a2{L->u, L->u_words, L->n, L->n, L->n, rpad / BK, tt, rpad, b, L->s1h, d_y, L->n};
  launch_stage(ctx, a2, (L->n + BM - 1) / BM, (b + BN - 1) / BN);
}

}  // namespace nqb
