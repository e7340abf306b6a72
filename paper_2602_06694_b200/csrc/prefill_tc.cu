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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace nqb {
namespace pf {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 3;
constexpr int MH = 2;                      // M=128 halves per CTA: 256 rows share each B tile
constexpr int A_BYTES = MH * BM * BK * 2;  // 32 KB
constexpr int B_BYTES = BN * BK * 2;       // 32 KB
constexpr int kProducers = MH * BM;        // one thread per A row; the next warp issues MMAs
constexpr uint32_t kTmemCols = 512;        // D_h: 128 lanes x 256 fp32 columns each

struct alignas(64) Args {
  CUtensorMap bmap;       // B (tokens x K binary16) for TMA: box 8 K x 256 tokens
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
  // split-K (k_prefill2 only): CTA z handles K tiles [z*kps, (z+1)*kps) and
  // writes raw fp32 partials to part[z][token][row] (ldp rows per token); a
  // fixed-order reduction applies the scale (deterministic).  kps = 0: off.
  uint32_t kps;
  float* part;
  uint32_t ldp;
};

// byte offset of (row, 8-element K chunk k8 of the 64-wide K tile) in the
// canonical K-major layout of an R-row operand tile:
//   [kstep (16 K)][khalf (8 K)][row group (8 rows)][row][16 B]
__device__ __forceinline__ uint32_t canon(uint32_t row, uint32_t k8, uint32_t R) {
  const uint32_t ks = k8 >> 1, kh = k8 & 1;
  return ((ks * 2 + kh) * (R / 8) + (row >> 3)) * 128 + (row & 7) * 16;
}

// 2-D TMA: box (8 K-elements, 256 tokens) at (k, token) -> one canonical
// [row group][row][16 B] column of the B tile; complete_tx on the mbarrier.
__device__ __forceinline__ void tma_b(void* dst, const CUtensorMap* map, uint32_t k, uint32_t tok,
                                      uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(k), "r"(tok), "r"(tc::smem_u32(bar))
      : "memory");
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
  const uint32_t m0 = blockIdx.x * (MH * BM), n0 = blockIdx.y * BN;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&bars->full[s], kProducers + 1);  // producers + the TMA issuer
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
          const uint64_t bd = tc::smem_desc_kmajor(bbase + ks * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
#pragma unroll
          for (uint32_t h = 0; h < MH; ++h) {
            const uint64_t ad = tc::smem_desc_kmajor(abase + h * (A_BYTES / MH) + ks * 2 * (BM / 8) * 128,
                                                     (BM / 8) * 128, 128);
            tc::mma_f16_ss(tmem + h * BN, ad, bd, idesc, (kt | ks) ? 1u : 0u);
          }
        }
        tc::mma_commit(&bars->empty[slot]);
      }
      tc::mma_commit(&bars->dready);
    }
  } else {  // ------------------------------------------------------ producers
    // thread t expands row t of the A tile: one 64-bit load covers its 64 K of
    // a K tile; the next tile's bits are prefetched while this one is written.
    const uint32_t row = tid, grow = m0 + row;
    const bool rv = grow < a.M;
    const uint32_t* brow = a.bits + (size_t)(rv ? grow : 0) * a.wpr;
    auto load_bits = [&](uint32_t kt) -> uint2 {
      return (rv && kt < a.nk) ? __ldg((const uint2*)(brow + kt * 2)) : make_uint2(0u, 0u);
    };
    uint2 cur = load_bits(0);
    for (uint32_t kt = 0; kt < a.nk; ++kt) {
      const uint2 nxt = load_bits(kt + 1);
      const uint32_t slot = kt % STAGES, use = kt / STAGES;
      if (use > 0) tc::mbar_wait(&bars->empty[slot], (use - 1) & 1);
      uint8_t* As = tiles + slot * (A_BYTES + B_BYTES);
      uint8_t* Bs = As + A_BYTES;
      if (tid == 0) {  // B: 8 TMA boxes (one per 8-wide K chunk) of 256 tokens
        tc::mbar_arrive_expect_tx(&bars->full[slot], B_BYTES);
#pragma unroll
        for (uint32_t k8 = 0; k8 < BK / 8; ++k8)
          tma_b(Bs + canon(0, k8, BN), &a.bmap, kt * BK + k8 * 8, n0, &bars->full[slot]);
      }
      // A: 64 signs of this row -> 8 chunks of 8 +-1 binary16 (bit 1 -> +1 0x3C00, 0 -> -1 0xBC00)
#pragma unroll
      for (uint32_t k8 = 0; k8 < 8; ++k8) {
        const uint32_t byte = ((k8 < 4 ? cur.x : cur.y) >> (8 * (k8 & 3))) & 0xFFu;
        uint4 v;
        uint32_t* pv = &v.x;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          pv[i] = 0xBC00BC00u ^ (((byte >> (2 * i)) & 1u) << 15) ^ (((byte >> (2 * i + 1)) & 1u) << 31);
        *(uint4*)(As + (row / BM) * (A_BYTES / MH) + canon(row % BM, k8, BM)) = v;
      }
      cur = nxt;
      tc::fence_proxy_async_smem();  // generic-proxy writes -> MMA (async proxy) reads
      tc::mbar_arrive(&bars->full[slot]);
    }
    // ------------------------------------------------------------- epilogue
    tc::mbar_wait(&bars->dready, 0);
    tc::fence_after_sync();
    const float sc = (grow < a.Mvalid && a.scale) ? __half2float(a.scale[grow]) : 1.f;
    const bool keep = grow < a.Mvalid;
    for (uint32_t c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld_x16(tmem + (row / BM) * BN + ((uint32_t)((warp & 3) * 32) << 16) + c0, v);
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

// ---------------------------------------------------------------------------
// TS variant: the expanded +-1 A tile never touches shared memory.  Producer
// thread t expands its row's 64 signs of a K tile in registers and writes them
// straight into TMEM (tcgen05.st.32x32b.x32: its lane, 32 columns of two
// binary16); the MMA reads A from TMEM and only the token tile (B) from shared
// memory, cutting shared-memory traffic per MAC by ~40% (the SS kernel is
// L1/shared-bandwidth bound: l1tex throughput 85% in ncu); N = 128 tokens per
// CTA keeps D (2 x 128 columns) plus four A stages (4 x 64 columns) in the 512
// TMEM columns, and 256 rows still share every B tile.
namespace ts {
constexpr int BN = 128, STAGES = 4;
constexpr int B_BYTES = BN * BK * 2;       // 16 KB
constexpr uint32_t kDCols = MH * BN;       // 256: D_h at columns h * BN
constexpr uint32_t kACols = MH * BK / 2;   // 64 per stage: half h at + h * 32

struct __align__(8) Bars {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t dready;
  uint32_t tmem;
};
}  // namespace ts

__global__ void __launch_bounds__(kProducers + 32, 1) k_prefill_ts(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  ts::Bars* bars = (ts::Bars*)smem;
  uint8_t* tiles = smem + 1024;  // ts::STAGES x B 16 KB
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const uint32_t m0 = blockIdx.x * (MH * BM), n0 = blockIdx.y * ts::BN;

  if (tid == 0) {
    for (int s = 0; s < ts::STAGES; ++s) {
      tc::mbar_init(&bars->full[s], kProducers + 1);  // producers + the TMA issuer
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
      constexpr uint32_t idesc = tc::idesc_f16(BM, ts::BN);
      for (uint32_t kt = 0; kt < a.nk; ++kt) {
        const uint32_t slot = kt % ts::STAGES;
        tc::mbar_wait(&bars->full[slot], (kt / ts::STAGES) & 1);
        tc::fence_after_sync();
        const uint32_t bbase = tc::smem_u32(tiles + slot * ts::B_BYTES);
        const uint32_t abase = tmem + ts::kDCols + slot * ts::kACols;
#pragma unroll
        for (uint32_t ks = 0; ks < BK / 16; ++ks) {
          const uint64_t bd = tc::smem_desc_kmajor(bbase + ks * 2 * (ts::BN / 8) * 128, (ts::BN / 8) * 128, 128);
#pragma unroll
          for (uint32_t h = 0; h < MH; ++h)
            tc::mma_f16_ts(tmem + h * ts::BN, abase + h * (BK / 2) + ks * 8, bd, idesc,
                           (kt | ks) ? 1u : 0u);
        }
        tc::mma_commit(&bars->empty[slot]);
      }
      tc::mma_commit(&bars->dready);
    }
  } else {  // ------------------------------------------------------ producers
    const uint32_t row = tid, grow = m0 + row;
    const bool rv = grow < a.M;
    const uint32_t* brow = a.bits + (size_t)(rv ? grow : 0) * a.wpr;
    auto load_bits = [&](uint32_t kt) -> uint2 {
      return (rv && kt < a.nk) ? __ldg((const uint2*)(brow + kt * 2)) : make_uint2(0u, 0u);
    };
    // this warp's TMEM lane quadrant (warp w: lanes 32*(w%4).., half w/4)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t hcol = (uint32_t)(warp >> 2) * (BK / 2);
    uint2 cur = load_bits(0);
    for (uint32_t kt = 0; kt < a.nk; ++kt) {
      const uint2 nxt = load_bits(kt + 1);
      const uint32_t slot = kt % ts::STAGES, use = kt / ts::STAGES;
      if (use > 0) {
        tc::mbar_wait(&bars->empty[slot], (use - 1) & 1);
        tc::fence_after_sync();
      }
      if (tid == 0) {  // B: 8 TMA boxes (one per 8-wide K chunk) of 128 tokens
        uint8_t* Bs = tiles + slot * ts::B_BYTES;
        tc::mbar_arrive_expect_tx(&bars->full[slot], ts::B_BYTES);
#pragma unroll
        for (uint32_t k8 = 0; k8 < BK / 8; ++k8)
          tma_b(Bs + canon(0, k8, ts::BN), &a.bmap, kt * BK + k8 * 8, n0, &bars->full[slot]);
      }
      // 64 signs -> 32 columns of two +-1 binary16 (bit 1 -> +1 0x3C00, 0 -> -1 0xBC00)
      uint32_t v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t w = i < 16 ? cur.x : cur.y, b = 2 * (i & 15);
        v[i] = 0xBC00BC00u ^ (((w >> b) & 1u) << 15) ^ (((w >> (b + 1)) & 1u) << 31);
      }
      tc::tmem_st_x32(tmem + lane_base + ts::kDCols + slot * ts::kACols + hcol, v);
      tc::wait_st();
      tc::fence_before_sync();  // TMEM stores -> the MMA issuer's barrier wait
      tc::mbar_arrive(&bars->full[slot]);
      cur = nxt;
    }
    // ------------------------------------------------------------- epilogue
    tc::mbar_wait(&bars->dready, 0);
    tc::fence_after_sync();
    const float sc = (grow < a.Mvalid && a.scale) ? __half2float(a.scale[grow]) : 1.f;
    const bool keep = grow < a.Mvalid;
    for (uint32_t c0 = 0; c0 < ts::BN; c0 += 16) {
      uint32_t d[16];
      tc::tmem_ld_x16(tmem + lane_base + (uint32_t)(warp >> 2) * ts::BN + c0, d);
      tc::wait_ld();
      if (grow < a.Mout) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t tok = n0 + c0 + j;
          if (tok < a.N)
            a.out[(size_t)tok * a.ldo + grow] =
                __float2half_rn(keep ? sc * __uint_as_float(d[j]) : 0.f);
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2).  A cluster of two CTAs on one TPC
// runs M = 256 MMAs: each CTA holds 256 rows of A (two 128-row halves, expanded
// by its producers as in k_prefill) and HALF of the 256-token B tile (128
// tokens, by TMA).  The leader (rank 0) issues `tcgen05.mma.cta_group::2`; the
// tensor cores of the pair read each B half once for both SMs, so shared-memory
// traffic per MAC drops by ~30% against k_prefill (which is l1tex-bound) and
// L2 traffic for B halves.  Each CTA's TMEM holds D for its own rows.
//   full[s] (leader): one arrival per producer warp of both CTAs (after the
//     warp's A rows are written) + the transaction bytes of both B halves;
//   empty[s], dready (both CTAs): one multicast commit from the leader.
namespace p2 {
constexpr int STAGES = 4;               // (tile sizes: template parameters of k_prefill2)
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // shared::cluster address of the rank-0 CTA

struct __align__(8) Bars {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t dready;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
// arrive on the leader's barrier (a shared::cluster address).  Default
// (CTA-scope release) semantics: each SM's tensor core reads only its own
// CTA's A rows, so the writes need no cluster-scope release; a .release.cluster
// arrive costs a MEMBAR.ALL.GPU per warp (it dominated the stall profile).
__device__ __forceinline__ void arrive_leader(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void arrive_leader_expect_tx(uint32_t bar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n" ::"r"(bar_cluster),
               "r"(bytes)
               : "memory");
}
// 2-D TMA of this CTA's B box; complete_tx lands on the leader's barrier
__device__ __forceinline__ void tma_b_2sm(void* dst, const CUtensorMap* map, uint32_t k, uint32_t tok,
                                          uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tc::smem_u32(dst)),
      "l"(map), "r"(k), "r"(tok), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ss_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit: arrive on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          tc::smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
}  // namespace p2

// MHT: 128-row halves per CTA (2: 256 rows share each B tile; 1: more CTAs for
// short M, e.g. stage 1 of the 70B q shape).
// BNPT: tokens per pair (256, or 208 = 13 x 16 when that fills the SMs
// better; each CTA holds BNPT/2 of them).
template <int MHT, int BNPT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MHT * BM + 32, 1)
    k_prefill2(const __grid_constant__ Args a) {
  constexpr int kP = MHT * BM;               // producer threads (one per A row)
  constexpr int kAB = MHT * BM * BK * 2;     // A bytes per stage
  constexpr int kBNH = BNPT / 2;             // tokens of this CTA's B half
  constexpr int kBB = kBNH * BK * 2;         // B-half bytes per stage
  static_assert(BNPT % 16 == 0 && BNPT <= 256 && kBNH % 8 == 0, "pair N tile");
  extern __shared__ __align__(1024) uint8_t smem[];
  p2::Bars* bars = (p2::Bars*)smem;
  uint8_t* tiles = smem + 1024;  // p2::STAGES x [A 32 KB | B half 16 KB]
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const uint32_t rank = p2::cluster_rank();
  const bool leader = rank == 0;
  const uint32_t m0 = blockIdx.x * (MHT * BM);
  const uint32_t np = blockIdx.y * BNPT;      // the pair's first token
  const uint32_t n0 = np + rank * kBNH;       // this CTA's B half
  const uint32_t kt0 = a.kps ? blockIdx.z * a.kps : 0;
  const uint32_t nkl = a.kps ? min(a.nk, kt0 + a.kps) - kt0 : a.nk;  // K tiles of this CTA

  if (tid == 0) {
    for (int s = 0; s < p2::STAGES; ++s) {
      // leader: one arrival per producer warp of both CTAs (+ tx of both B halves)
      tc::mbar_init(&bars->full[s], 2 * (kP / 32));
      tc::mbar_init(&bars->empty[s], 1);
    }
    tc::mbar_init(&bars->dready, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     tc::smem_u32(&bars->tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  tc::fence_before_sync();
  p2::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc::fence_after_sync();
  const uint32_t tmem = bars->tmem;
  const uint32_t full_leader0 = tc::smem_u32(&bars->full[0]) & p2::kPeerMask;

  if (warp == kP / 32) {  // ------------------- MMA issuer (leader CTA only)
    if (leader && lane == 0) {
      constexpr uint32_t idesc = tc::idesc_f16(2 * BM, BNPT);
      for (uint32_t i = 0; i < nkl; ++i) {
        const uint32_t slot = i % p2::STAGES;
        tc::mbar_wait(&bars->full[slot], (i / p2::STAGES) & 1);
        tc::fence_after_sync();
        const uint32_t abase = tc::smem_u32(tiles + slot * (kAB + kBB));
        const uint32_t bbase = abase + kAB;
#pragma unroll
        for (uint32_t ks = 0; ks < BK / 16; ++ks) {
          const uint64_t bd =
              tc::smem_desc_kmajor(bbase + ks * 2 * (kBNH / 8) * 128, (kBNH / 8) * 128, 128);
#pragma unroll
          for (uint32_t h = 0; h < MHT; ++h) {
            const uint64_t ad = tc::smem_desc_kmajor(abase + h * (kAB / MHT) + ks * 2 * (BM / 8) * 128,
                                                     (BM / 8) * 128, 128);
            p2::mma_f16_ss_2sm(tmem + h * BNPT, ad, bd, idesc, (i | ks) ? 1u : 0u);
          }
        }
        p2::commit_pair(&bars->empty[slot]);
      }
      p2::commit_pair(&bars->dready);
    }
  } else {  // ------------------------------------------------------ producers
    const uint32_t row = tid, grow = m0 + row;
    const bool rv = grow < a.M;
    const uint32_t* brow = a.bits + (size_t)(rv ? grow : 0) * a.wpr;
    auto load_bits = [&](uint32_t kt) -> uint2 {
      return (rv && kt < kt0 + nkl) ? __ldg((const uint2*)(brow + kt * 2)) : make_uint2(0u, 0u);
    };
    uint2 cur = load_bits(kt0);
    for (uint32_t i = 0; i < nkl; ++i) {
      const uint32_t kt = kt0 + i;
      const uint2 nxt = load_bits(kt + 1);
      const uint32_t slot = i % p2::STAGES, use = i / p2::STAGES;
      if (use > 0) tc::mbar_wait(&bars->empty[slot], (use - 1) & 1);
      uint8_t* As = tiles + slot * (kAB + kBB);
      uint8_t* Bs = As + kAB;
      const uint32_t fullL = full_leader0 + slot * 8;
      if (tid == 0) {  // this CTA's B half: 8 TMA boxes of 128 tokens, bytes counted at the leader
#pragma unroll
        for (uint32_t k8 = 0; k8 < BK / 8; ++k8)
          p2::tma_b_2sm(Bs + canon(0, k8, kBNH), &a.bmap, kt * BK + k8 * 8, n0, fullL);
      }
#pragma unroll
      for (uint32_t k8 = 0; k8 < 8; ++k8) {
        const uint32_t byte = ((k8 < 4 ? cur.x : cur.y) >> (8 * (k8 & 3))) & 0xFFu;
        uint4 v;
        uint32_t* pv = &v.x;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          pv[i] = 0xBC00BC00u ^ (((byte >> (2 * i)) & 1u) << 15) ^ (((byte >> (2 * i + 1)) & 1u) << 31);
        *(uint4*)(As + (row / BM) * (kAB / MHT) + canon(row % BM, k8, BM)) = v;
      }
      cur = nxt;
      tc::fence_proxy_async_smem();  // generic-proxy writes -> the pair's MMA (async proxy)
      __syncwarp();                  // the warp's rows are written; lane 0 arrives
      if (lane == 0) {
        if (leader && tid == 0) p2::arrive_leader_expect_tx(fullL, 2 * kBB);
        else p2::arrive_leader(fullL);
      }
    }
    // ------------------------------------------------------------- epilogue
    tc::mbar_wait(&bars->dready, 0);
    tc::fence_after_sync();
    const float sc = (grow < a.Mvalid && a.scale) ? __half2float(a.scale[grow]) : 1.f;
    const bool keep = grow < a.Mvalid;
    // the stage buffers are idle now (every MMA has completed): epilogue tile
    __half* ep = (__half*)tiles;
    const bool vec_out = !a.part && (a.ldo % 8 == 0) && (((uintptr_t)a.out) % 16 == 0);
    for (uint32_t c0 = 0; c0 < BNPT; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld_x16(tmem + (row / BM) * BNPT + ((uint32_t)((warp & 3) * 32) << 16) + c0, v);
      tc::wait_ld();
      if (grow < a.Mout) {
        if (a.part) {  // split-K: raw partial sums, reduced (and scaled) in fixed order later
          float* pz = a.part + (size_t)blockIdx.z * a.N * a.ldp;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t tok = np + c0 + j;
            if (tok < a.N) pz[(size_t)tok * a.ldp + grow] = __uint_as_float(v[j]);
          }
        } else if (!vec_out) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t tok = np + c0 + j;
            if (tok < a.N)
              a.out[(size_t)tok * a.ldo + grow] =
                  __float2half_rn(keep ? sc * __uint_as_float(v[j]) : 0.f);
          }
        }
      }
      if (vec_out) {
        // token-major output through shared memory: each thread writes its
        // row's 16 values into a [16 tokens][kP rows] tile, then 16-byte
        // stores of 8 consecutive rows per token (8x fewer store instructions)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          ep[j * kP + row] = __float2half_rn(keep ? sc * __uint_as_float(v[j]) : 0.f);
        asm volatile("bar.sync 1, %0;\n" ::"n"(kP) : "memory");
        for (uint32_t q = row; q < 16u * (kP / 8); q += kP) {
          const uint32_t j = q / (kP / 8), g8 = (q % (kP / 8)) * 8;
          const uint32_t tok = np + c0 + j, r0g = m0 + g8;
          if (tok < a.N && r0g < a.Mout) {
            const uint4 val = *(const uint4*)(ep + j * kP + g8);
            if (r0g + 8 <= a.Mout) {
              *(uint4*)(a.out + (size_t)tok * a.ldo + r0g) = val;
            } else {
              const __half* hv = (const __half*)&val;
              for (uint32_t t = 0; r0g + t < a.Mout; ++t) a.out[(size_t)tok * a.ldo + r0g + t] = hv[t];
            }
          }
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(kP) : "memory");
      }
    }
  }
  tc::fence_before_sync();
  p2::cluster_sync();  // both CTAs are done with the pair's TMEM
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
}

// Split-K reduction: out[tok][row] = fp16(scale_row * sum_z part[z][tok][row])
// in fixed z order; rows >= Mvalid are written as 0.
__global__ void k_splitk_reduce(const float* __restrict__ part, uint32_t splits, uint32_t N,
                                uint32_t rows, uint32_t ldp, uint32_t Mvalid,
                                const __half* __restrict__ scale, __half* __restrict__ out,
                                uint32_t ldo) {
  const uint64_t total = (uint64_t)N * rows;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t tok = (uint32_t)(e / rows), row = (uint32_t)(e % rows);
    float acc = 0.f;
    for (uint32_t z = 0; z < splits; ++z) acc += part[((size_t)z * N + tok) * ldp + row];
    const float sc = (scale && row < Mvalid) ? __half2float(scale[row]) : 1.f;
    out[(size_t)tok * ldo + row] = __float2half_rn(row < Mvalid ? sc * acc : 0.f);
  }
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

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    NQB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    NQB_REQUIRE(p && q == cudaDriverEntryPointSuccess, NQB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// B = tokens x ld binary16 (K = kdim valid columns); box 8 K x 256 tokens;
// out-of-range tokens / K read as zero.
static void make_bmap(CUtensorMap* map, const __half* B, uint32_t kdim, uint32_t ld, uint32_t tokens,
                      uint32_t box_tokens) {
  const cuuint64_t dims[2] = {kdim, tokens};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  const cuuint32_t box[2] = {8, box_tokens};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)B, dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  NQB_REQUIRE(r == CUDA_SUCCESS, NQB_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// The SS kernel is the default.  NQB_PREFILL_TS=1 selects the TS variant:
// parity-green, faster on 70B q (574 vs 488 TFLOP/s) but slower on gate/down
// (675 vs 733, 559 vs 639).  ncu shows l1tex still at 84% with A in TMEM, so the
// TMEM stores and A reads load the same datapath that the shared-memory A
// traffic did.
// The CTA-pair kernel is the default (NQB_PREFILL_2SM=0 selects the
// single-CTA SS kernel): +39..51% at b = 2048 on the 70B shapes.
static bool use_2sm() {
  static const bool v = [] { const char* e = std::getenv("NQB_PREFILL_2SM");
                             return !(e && e[0] == '0'); }();
  return v;
}

static bool use_ts() {
  static const bool ts = [] { const char* e = std::getenv("NQB_PREFILL_TS");
                              return e && e[0] == '1'; }();
  return ts;
}

struct PairCfg {
  uint32_t mht, bnp;
};

// CTA-pair tiling: rows per CTA (128 x mht) and tokens per pair (bnp).  The
// large tile (256 rows, 256 tokens) has the most operand reuse; a smaller one
// is used only when the large grid is under two waves and leaves clearly more
// SMs idle (measured: on multi-wave grids the large tile wins regardless).
static PairCfg choose_pair(nqb_context* ctx, uint32_t rows, uint32_t tokens) {
  static const int force_rows = [] { const char* e = std::getenv("NQB_PREFILL_ROWS");  // 128 / 256
                                     return e ? atoi(e) : 0; }();
  static const int force_n = [] { const char* e = std::getenv("NQB_PREFILL_N");  // 256 / 208
                                  return e ? atoi(e) : 0; }();
  const PairCfg cands[4] = {{2, 256}, {2, 208}, {1, 256}, {1, 208}};
  const uint64_t sm = (uint64_t)ctx->num_sms;
  auto ctas_of = [&](const PairCfg& c) {
    const uint64_t pairs = (rows + 2 * BM * c.mht - 1) / (2 * BM * c.mht);
    return pairs * 2 * ((tokens + c.bnp - 1) / c.bnp);
  };
  auto util_of = [&](uint64_t ctas) {
    return (double)ctas / (double)(((ctas + sm - 1) / sm) * sm);
  };
  if (force_rows || force_n) {
    for (const PairCfg& c : cands)
      if ((!force_rows || (int)(c.mht * BM) == force_rows) && (!force_n || (int)c.bnp == force_n))
        return c;
  }
  PairCfg pick = cands[0];
  const uint64_t base = ctas_of(pick);
  if (base >= 2 * sm) return pick;
  double best = util_of(base) + 0.1;
  for (const PairCfg& c : cands) {
    const double u = util_of(ctas_of(c));
    if (u > best) best = u, pick = c;
  }
  return pick;
}

template <int MHT, int BNPT>
static void launch_pair(nqb_context* ctx, const Args& a, dim3 grid) {
  constexpr int smem = 1024 + p2::STAGES * (MHT * BM * BK * 2 + (BNPT / 2) * BK * 2);
  static bool attr = false;
  if (!attr) {
    NQB_CUDA(cudaFuncSetAttribute(k_prefill2<MHT, BNPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem));
    attr = true;
  }
  k_prefill2<MHT, BNPT><<<grid, MHT * BM + 32, smem, ctx->stream>>>(a);
}

static void launch_stage(nqb_context* ctx, const Args& a_in, uint32_t grid_m, uint32_t tokens,
                         PairCfg pc) {
  Args a = a_in;
  static bool attr = false;
  if (!attr) {
    NQB_CUDA(cudaFuncSetAttribute(k_prefill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  1024 + STAGES * (A_BYTES + B_BYTES)));
    NQB_CUDA(cudaFuncSetAttribute(k_prefill_ts, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  1024 + ts::STAGES * ts::B_BYTES));
    attr = true;
  }
  if (use_2sm() && !use_ts()) {
    const uint32_t ny = (tokens + pc.bnp - 1) / pc.bnp;
    const uint32_t gx = (grid_m + 2 * pc.mht - 1) / (2 * pc.mht) * 2;  // whole CTA pairs
    // Split-K (fixed-order reduction after) is opt-in, NQB_PREFILL_SPLITK=s: a
    // cost model (MMA time / wave utilisation + the partials' HBM round trip)
    // picking s = 2..8 measured slower on the 70B shapes, so the default is one pass.
    static const int force_split = [] { const char* e = std::getenv("NQB_PREFILL_SPLITK");
                                        return e ? atoi(e) : 0; }();
    uint32_t splits = force_split > 0 ? std::min<uint32_t>((uint32_t)force_split, a.nk) : 1u;
    if (splits > 1) {
      a.kps = (a.nk + splits - 1) / splits;
      splits = (a.nk + a.kps - 1) / a.kps;
      a.ldp = a.Mout;
      a.part = (float*)scratch(ctx, 10, sizeof(float) * (size_t)splits * a.N * a.ldp);
    }
    const dim3 grid(gx, ny, splits);
    if (pc.mht == 2 && pc.bnp == 256) launch_pair<2, 256>(ctx, a, grid);
    else if (pc.mht == 2) launch_pair<2, 208>(ctx, a, grid);
    else if (pc.bnp == 256) launch_pair<1, 256>(ctx, a, grid);
    else launch_pair<1, 208>(ctx, a, grid);
    if (splits > 1) {
      NQB_LAUNCHED(ctx);
      const uint64_t tot = (uint64_t)a.N * a.Mout;
      k_splitk_reduce<<<(uint32_t)std::min<uint64_t>((tot + 255) / 256, 148 * 16), 256, 0, ctx->stream>>>(
          a.part, splits, a.N, a.Mout, a.ldp, a.Mvalid, a.scale, a.out, a.ldo);
    }
  } else if (use_ts())
    k_prefill_ts<<<dim3((grid_m + MH - 1) / MH, (tokens + ts::BN - 1) / ts::BN), kProducers + 32,
                   1024 + ts::STAGES * ts::B_BYTES, ctx->stream>>>(a);
  else
    k_prefill<<<dim3((grid_m + MH - 1) / MH, (tokens + BN - 1) / BN), kProducers + 32,
                1024 + STAGES * (A_BYTES + B_BYTES), ctx->stream>>>(a);
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
  auto box_of = [&](const PairCfg& pc) -> uint32_t {
    return use_ts() ? (uint32_t)ts::BN : use_2sm() ? pc.bnp / 2 : (uint32_t)BN;
  };
  // stage 1: T^T[token][k] = sum_j sign(V[j][k]) * xs[token][j]   (rows k < r, padded rows 0)
  Args a1{{}, L->vt, L->vt_words, L->r, L->r, rpad, mpad / BK, xs, mpad, b, nullptr, tt, rpad};
  const PairCfg p1 = choose_pair(ctx, rpad, b);
  make_bmap(&a1.bmap, xs, mpad, mpad, b, box_of(p1));
  launch_stage(ctx, a1, (rpad + BM - 1) / BM, b, p1);
  // stage 2: Y[token][i] = s1_i * sum_k sign(U[i][k]) * T^T[token][k]
  Args a2{{}, L->u, L->u_words, L->n, L->n, L->n, rpad / BK, tt, rpad, b, L->s1h, d_y, L->n};
  const PairCfg p2c = choose_pair(ctx, L->n, b);
  make_bmap(&a2.bmap, tt, rpad, rpad, b, box_of(p2c));
  launch_stage(ctx, a2, (L->n + BM - 1) / BM, b, p2c);
}

}  // namespace nqb
