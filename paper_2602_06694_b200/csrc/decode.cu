// decode.cu — batch-1 BLR decode GEMV (gemv_packed_f32, packed.cpp:201-204)
// as one fused two-stage sm_100a kernel.  Design: decode.cuh, DESIGN.md §4.
#include <algorithm>
#include <cmath>

#include "decode.cuh"
#include "tc_common.cuh"

namespace nqb {
namespace dec {

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerThreads) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Diagnostics: slot 0 = %globaltimer at CTA start, slots 1.. = SM clock64
// cycles since the CTA started (exact, per CTA; the base stays in a register).
#define TRACE(i)                                                                  \
  do {                                                                            \
    if (p.trace && threadIdx.x == 0) {                                            \
      if ((i) == 0) {                                                             \
        trace_t0 = clock64();                                                     \
        p.trace[blockIdx.x * 32] = globaltimer();                                 \
      } else {                                                                    \
        p.trace[blockIdx.x * 32 + (i)] = clock64() - trace_t0;                    \
      }                                                                           \
    }                                                                             \
  } while (0)

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// mbarrier wait with a watchdog: a wait that never completes traps the
// launch (reported as a CUDA error) instead of hanging the device.
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0, it = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (++it > (1u << 24)) __trap();
  }
}

// Tile index q (0..7) of input K inside its slab of a K-long dimension.
__device__ __forceinline__ uint32_t q_of(uint32_t k, uint32_t K) {
  uint32_t F, rem;
  slab_split(K, F, rem);
  const uint32_t full = 256 * F;
  if (k < full) return (k >> 5) & 7;
  const uint32_t k0 = (rem >= 128 && k < full + 128) ? full : full + (rem >= 128 ? 128 : 0);
  return (k - k0) >> 5;
}

// Signed base-256 digits of v (|v| <= 2^37) into byte e of the kLimbs limb words.
__device__ __forceinline__ void put_limbs(long long v, uint32_t e, uint32_t (&w)[kLimbs]) {
  const uint32_t s = 8 * e;
#pragma unroll
  for (int l = 0; l < kLimbs - 1; ++l) {
    const int d = (int)(int8_t)(v & 0xFF);
    w[l] |= (uint32_t)(d & 0xFF) << s;
    v = (v - d) >> 8;
  }
  w[kLimbs - 1] |= (uint32_t)(v & 0xFF) << s;
}

// B operand words for the quad of inputs k0..k0+3 (values already << (7-q)),
// canonical K-major layout of one 32-wide K tile (16 rows = limbs x 32 bytes):
// byte (limb n, k) at ((k/16)*2 + n/8)*128 + (n%8)*16 + k%16.  Limbs 0..7 are
// written here (6, 7 zero); rows 8..15 are zeroed by zero_b_hi.
__device__ __forceinline__ void store_quad(uint8_t* bfrag, uint32_t klo, uint32_t k0,
                                           const uint32_t (&w)[kLimbs]) {
  const uint32_t kk = k0 & 31;
  uint8_t* t = bfrag + ((k0 - klo) >> 5) * kTileB + (kk >> 4) * 256 + (kk & 15);
#pragma unroll
  for (uint32_t g = 0; g < 8; ++g) *(uint32_t*)(t + g * 16) = g < (uint32_t)kLimbs ? w[g] : 0u;
}

// Zeroes B rows 8..15 (the upper core-matrix group) of tiles [0, ntiles).
__device__ __forceinline__ void zero_b_hi(uint8_t* bfrag, uint32_t ntiles, int tid) {
  for (uint32_t i = tid; i < ntiles * 16; i += kConsumerThreads) {
    const uint32_t tile = i >> 4, part = i & 15;  // 2 halves x 8 x 16 B
    *(uint4*)(bfrag + tile * kTileB + (part >> 3) * 256 + 128 + (part & 7) * 16) =
        make_uint4(0u, 0u, 0u, 0u);
  }
}

__device__ __forceinline__ long long cta_sum_i64(long long v, long long* red8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  consumers_sync();
  if (lane == 0) red8[warp] = v;
  consumers_sync();
  long long s = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) s += red8[w];
  return s;
}

__device__ __forceinline__ unsigned long long cta_max_u64(unsigned long long v,
                                                          unsigned long long* red8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(~0u, v, o));
  consumers_sync();
  if (lane == 0) red8[warp] = v;
  consumers_sync();
  unsigned long long s = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) s = max(s, red8[w]);
  return s;
}

__device__ __forceinline__ int exponent_of(float M) {
  if (!(M > 0.f) || isinf(M)) return 0;
  int e;
  frexpf(M, &e);
  return e;  // M < 2^e
}

// a * 2^k exactly in fp32 for k up to ~250 (two steps avoid overflowing 2^k)
__device__ __forceinline__ float scale_pow2(float a, int k) {
  const int k1 = k > 126 ? 126 : (k < -126 ? -126 : k);
  return __fmul_rn(__fmul_rn(a, __int_as_float((127 + k1) << 23)),
                   __int_as_float((127 + (k - k1)) << 23));
}

// Limbs of the quad v[0..3] (tile-in-slab q) into the B-fragment buffer.
__device__ __forceinline__ void emit_quad(uint8_t* bfrag, uint32_t klo, uint32_t k0, uint32_t q,
                                          const long long (&v)[4]) {
  uint32_t w[kLimbs] = {};
#pragma unroll
  for (int e = 0; e < 4; ++e) put_limbs(v[e] * (1 << (7 - q)), e, w);
  store_quad(bfrag, klo, k0, w);
}

struct XQuad {
  float s[4], x[4];
};

__device__ __forceinline__ XQuad load_xquad(const Params& p, const __half* s2h, uint32_t k0,
                                            uint32_t m) {
  XQuad r;
  if (k0 + 3 < m && p.x_vec) {
    const uint2 sh2 = *(const uint2*)(s2h + k0);
    const float2 s01 = __half22float2(*(const __half2*)&sh2.x);
    const float2 s23 = __half22float2(*(const __half2*)&sh2.y);
    r.s[0] = s01.x; r.s[1] = s01.y; r.s[2] = s23.x; r.s[3] = s23.y;
    if (p.x_f32) {
      const float4 v = __ldcg((const float4*)((const float*)p.x + k0));
      r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
    } else {
      const uint2 v = __ldcg((const uint2*)((const __half*)p.x + k0));
      const float2 x01 = __half22float2(*(const __half2*)&v.x);
      const float2 x23 = __half22float2(*(const __half2*)&v.y);
      r.x[0] = x01.x; r.x[1] = x01.y; r.x[2] = x23.x; r.x[3] = x23.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t j = k0 + e;
      r.s[e] = r.x[e] = 0.f;
      if (j < m) {
        r.s[e] = __half2float(s2h[j]);
        r.x[e] = p.x_f32 ? __ldcg((const float*)p.x + j)
                         : __half2float(__ushort_as_half(__ldcg((const unsigned short*)p.x + j)));
      }
    }
  }
  return r;
}

__device__ __forceinline__ void load_tquad(const long long* Tseg, uint32_t k0, uint32_t r,
                                           uint32_t t_off, long long (&v)[4]) {
  if (k0 + 3 < r && ((t_off + k0) & 1) == 0) {
    const longlong2 v0 = __ldcg((const longlong2*)(Tseg + k0));
    const longlong2 v1 = __ldcg((const longlong2*)(Tseg + k0 + 2));
    v[0] = v0.x; v[1] = v0.y; v[2] = v1.x; v[3] = v1.y;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = k0 + e < r ? __ldcg(Tseg + k0 + e) : 0;
  }
}

// ---------------------------------------------------------------------------
// tcgen05 stage machinery
// ---------------------------------------------------------------------------
constexpr uint32_t kSlots = 7;  // (row block, slab) pairs in flight in TMEM (64 columns each, after D)

// Shared-memory barriers of one CTA.
struct Bars {
  uint64_t full[2];          // stream landed: stage 1, stage 2 (TMA complete_tx)
  uint64_t aready[kSlots];   // pair slot written (4 warp arrivals of one warpgroup)
  uint64_t afree[kSlots];    // the MMAs reading the slot completed (tcgen05.commit)
  uint64_t dready;           // all MMAs of a stage completed (tcgen05.commit)
  uint32_t tmem;             // TMEM base address (tcgen05.alloc)
  uint32_t pad;
};
static_assert(sizeof(Bars) <= 512, "barriers fit the smem head");

// Geometry of one stage of one CTA.  Pairs (row block, slab) run slab-major,
// numbered pi0 + p across stages; pair pi lives in TMEM slot pi % kSlots.
struct Stage {
  uint32_t rows;       // 16 * row tiles
  uint32_t nrb;        // TMEM row blocks of 128 rows
  uint32_t nsec;       // K slabs
  uint32_t K, slab0, klo;
  uint32_t off;        // buffer offset of the stage's first section
  uint32_t pi0;        // pairs of earlier stages
  __device__ uint32_t npairs() const { return nrb * nsec; }
};

__device__ __forceinline__ uint32_t tmem_d(uint32_t tmem, uint32_t rb) { return tmem + rb * kMmaN; }
__device__ __forceinline__ uint32_t tmem_slot(uint32_t tmem, uint32_t slot, uint32_t q) {
  return tmem + 64 + slot * 64 + q * 8;
}

// A registers of tile q for this thread's row (row-major stream formats:
// nq=8: 8 words, bit 8b+q of word j = A[row][32q + 4j + b]; nq=4: 4 words,
// word h packs words 2h (low nibbles) and 2h+1 (high nibbles); nq=2: 2 words,
// word h packs words 4h+i at bit offset 2i).
__device__ __forceinline__ void a_regs(const uint32_t (&u)[8], uint32_t nq, uint32_t q,
                                       uint32_t (&v)[8]) {
  const uint32_t mask = 0x01010101u << q;
  if (nq == 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = u[j] & mask;
  } else if (nq == 4) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      v[2 * h] = u[h] & mask;
      v[2 * h + 1] = (u[h] >> 4) & mask;
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i) v[4 * h + i] = (u[h] >> (2 * i)) & mask;
  }
}

// Expander side of one stage: warpgroup e writes the A tiles of pairs
// p = e, e+2, ... into their TMEM slots and hands them to the MMA thread.
__device__ __forceinline__ void expand_stage(const Stage& S, const uint8_t* buf, Bars* bars,
                                             uint32_t tmem, unsigned long long* prof) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t e = warp >> 2, wq = warp & 3;
  const uint32_t rl = wq * 32 + lane;  // row inside a 128-row block = TMEM lane
  const uint32_t lane_base = (wq * 32) << 16;
  const uint32_t np = S.npairs();
  for (uint32_t p = e; p < np; p += 2) {
    const uint32_t rb = p % S.nrb, s = p / S.nrb;
    const Slab sl = slab_of(S.K, S.slab0 + s);
    const uint32_t row = rb * 128 + rl;
    long long c0 = prof ? clock64() : 0;
    uint32_t u[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (row < S.rows) {
      const uint8_t* src = buf + S.off + S.rows * ((sl.k0 - S.klo) >> 3) + row * 4 * sl.nq;
      if (sl.nq == 8) {
        const uint4 x0 = *(const uint4*)src, x1 = *(const uint4*)(src + 16);
        u[0] = x0.x; u[1] = x0.y; u[2] = x0.z; u[3] = x0.w;
        u[4] = x1.x; u[5] = x1.y; u[6] = x1.z; u[7] = x1.w;
      } else if (sl.nq == 4) {
        const uint4 x0 = *(const uint4*)src;
        u[0] = x0.x; u[1] = x0.y; u[2] = x0.z; u[3] = x0.w;
      } else {
        const uint2 x0 = *(const uint2*)src;
        u[0] = x0.x; u[1] = x0.y;
      }
    }
    const uint32_t pi = S.pi0 + p, slot = pi % kSlots, use = pi / kSlots;
    if (prof) {
      uint32_t z = u[0] ^ u[7];
      asm volatile("" ::"r"(z));
    }
    long long c1 = prof ? clock64() : 0;
    if (use > 0) mbar_wait_wd(&bars->afree[slot], (use - 1) & 1);
    tc::fence_after_sync();
    long long c2 = prof ? clock64() : 0;
    for (uint32_t q = 0; q < sl.nq; ++q) {
      uint32_t v[8];
      a_regs(u, sl.nq, q, v);
      tc::tmem_st_x8(tmem_slot(tmem, slot, q) + lane_base, v);
    }
    long long c3 = prof ? clock64() : 0;
    tc::wait_st();
    tc::fence_before_sync();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&bars->aready[slot]);
    if (prof && lane == 0) {
      long long c4 = clock64();
      prof[0] += c1 - c0;
      prof[1] += c2 - c1;
      prof[2] += c3 - c2;
      prof[3] += c4 - c3;
      prof[4] += 1;
    }
  }
}

// MMA-issuer side of one stage (one thread): tile by tile, wait for the A
// slot, issue one kind::i8 MMA (128 rows x 32 K x 16 limbs), release the slot.
__device__ __forceinline__ void mma_stage(const Stage& S, uint32_t bfrag_u32, Bars* bars,
                                          unsigned long long* prof) {
  constexpr uint32_t idesc = tc::idesc_i8(128, kMmaN, false, true);
  const uint32_t np = S.npairs();
  uint32_t tmem = 0;
  for (uint32_t p = 0; p < np; ++p) {
    const uint32_t rb = p % S.nrb, s = p / S.nrb;
    const Slab sl = slab_of(S.K, S.slab0 + s);
    const uint32_t pi = S.pi0 + p, slot = pi % kSlots, tile0 = (sl.k0 - S.klo) >> 5;
    long long c0 = prof ? clock64() : 0;
    mbar_wait_wd(&bars->aready[slot], (pi / kSlots) & 1);
    tc::fence_after_sync();
    long long c1 = prof ? clock64() : 0;
    if (prof) prof[0] += c1 - c0;
    if (!tmem) tmem = *(volatile uint32_t*)&bars->tmem;  // allocated before any aready
    for (uint32_t q = 0; q < sl.nq; ++q) {
      const uint64_t bdesc =
          tc::smem_desc_kmajor(bfrag_u32 + (tile0 + q) * kTileB, (kMmaN / 8) * 128, 128);
      tc::mma_i8_ts(tmem_d(tmem, rb), tmem_slot(tmem, slot, q), bdesc, idesc, (s | q) ? 1u : 0u);
    }
    tc::mma_commit(&bars->afree[slot]);
    if (prof) {
      prof[1] += clock64() - c1;
      prof[2] += 1;
    }
  }
  tc::mma_commit(&bars->dready);
}

// Row sums of a finished stage for this thread's TMEM lane in row block rb:
// D[row][l] = sum_K bit * 2^q * limb_l  ->  sum_K bit * value (exact int64;
// two's-complement wraparound of the partial sums is harmless).
__device__ __forceinline__ long long d_row(uint32_t tmem, uint32_t rb, uint32_t wq) {
  uint32_t v[16];
  tc::tmem_ld_x16(tmem_d(tmem, rb) + ((wq * 32) << 16), v);
  tc::wait_ld();
  unsigned long long acc = 0;
#pragma unroll
  for (int l = 0; l < kLimbs; ++l) acc += (unsigned long long)(long long)(int)v[l] << (8 * l);
  return (long long)acc >> 7;
}

__global__ void __launch_bounds__(kThreads, 1) k_decode(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars* bars = (Bars*)smem;
  long long* red8 = (long long*)(smem + 512);
  uint8_t* bfrag = smem + kSmemHead;
  uint8_t* buf = bfrag + p.bfrag_bytes;

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  long long trace_t0 = 0;
  TRACE(0);
  const Cta C = p.ctas[blockIdx.x];
  if (p.trace && tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[blockIdx.x * 32 + 16] = smid;
    p.trace[blockIdx.x * 32 + 17] = C.s1_rtn;
    p.trace[blockIdx.x * 32 + 18] = C.s1_sln;
    p.trace[blockIdx.x * 32 + 19] = C.s2_rtn;
    p.trace[blockIdx.x * 32 + 20] = C.nsec;
  }
  const uint32_t n1 = C.s1_rtn ? C.s1_sln : 0;
  const uint32_t m = p.m;
  const Seg& S2seg = p.seg[C.s2_seg];
  auto sec_bytes = [&](uint32_t sec) -> uint32_t {
    return sec < n1 ? C.s1_rtn * unit_bytes(slab_of(m, C.s1_sl0 + sec).nq)
                    : C.s2_rtn * unit_bytes(slab_of(S2seg.r, sec - n1).nq);
  };
  Stage st1{}, st2{};
  if (n1) {
    st1.rows = 16u * C.s1_rtn;
    st1.nrb = (st1.rows + 127) / 128;
    st1.nsec = n1;
    st1.K = m;
    st1.slab0 = C.s1_sl0;
    st1.klo = slab_of(m, C.s1_sl0).k0;
    st1.off = 0;
    st1.pi0 = 0;
  }
  uint32_t s1_bytes = 0;
  for (uint32_t s = 0; s < n1; ++s) s1_bytes += sec_bytes(s);
  if (C.s2_rtn) {
    st2.rows = 16u * C.s2_rtn;
    st2.nrb = (st2.rows + 127) / 128;
    st2.nsec = C.nsec - n1;
    st2.K = S2seg.r;
    st2.slab0 = 0;
    st2.klo = 0;
    st2.off = s1_bytes;
    st2.pi0 = n1 ? st1.nrb * n1 : 0;
  }

  if (tid == 0) {
    tc::mbar_init(&bars->full[0], 1);
    tc::mbar_init(&bars->full[1], 1);
    for (uint32_t i = 0; i < kSlots; ++i) {
      tc::mbar_init(&bars->aready[i], 4);
      tc::mbar_init(&bars->afree[i], 1);
    }
    tc::mbar_init(&bars->dready, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  pdl_launch_dependents();  // the next kernel may start streaming its bits

  // --------------------------------------------------- producer / MMA issuer
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      const uint8_t* src = p.bits + C.stream_off;
      uint32_t off = 0;
      for (uint32_t sec = 0; sec < C.nsec; ++sec) {
        const uint32_t bytes = sec_bytes(sec);
        uint64_t* bar = &bars->full[sec < n1 ? 0 : 1];
        if (sec == 0 || sec == n1) {
          uint32_t total = 0;
          for (uint32_t q = sec; q < (sec < n1 ? n1 : C.nsec); ++q) total += sec_bytes(q);
          tc::mbar_arrive_expect_tx(bar, total);
        }
        tc::bulk_g2s(buf + off, src + off, bytes, bar);
        off += bytes;
      }
    }
    // TMEM is allocated by warp 0 after griddepcontrol.wait; its base is read
    // after the first aready wait (expanders only arrive after allocation).
    if (lane == 0) {
      const uint32_t b_u32 = tc::smem_u32(bfrag);
      unsigned long long* pr = p.trace ? p.trace + blockIdx.x * 32 + 28 : nullptr;
      if (n1) mma_stage(st1, b_u32, bars, nullptr);
      if (C.s2_rtn) mma_stage(st2, b_u32, bars, pr);
    }
    return;
  }

  // ----------------------------------------------------------------- consumers
  TRACE(1);
  pdl_wait();  // x (and the t accumulator) may be written by the previous kernel
  TRACE(2);
  if (warp == 0) {
    tc::tmem_alloc(&bars->tmem, kTmemCols);
    tc::tmem_relinquish();
    tc::fence_before_sync();
  }
  State* st = p.st;
  const uint32_t ep = __ldcg(&st->epoch);
  const uint32_t dirty_next = __ldcg(&st->dirty[(ep & 1) ^ 1]);
  const uint32_t b = ep & 1;

  // ---- activation exponent: a = s2*x with |a| <= max|s2| * X, X = 65504 for
  // binary16 x (no pass over x), max|x| over all m for fp32 x.
  float xmax = 65504.f;
  if (p.x_f32) {
    float mx = 0.f;
    const float* xf = (const float*)p.x;
    const uint32_t nv = p.x_vec ? m / 4 : 0;
#pragma unroll 4
    for (uint32_t i = tid; i < nv; i += kConsumerThreads) {
      const float4 v = __ldcg((const float4*)xf + i);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (uint32_t i = 4 * nv + tid; i < m; i += kConsumerThreads) mx = fmaxf(mx, fabsf(__ldcg(xf + i)));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
    float* rf = (float*)red8;
    if (lane == 0) rf[warp] = mx;
    consumers_sync();
    mx = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumerWarps; ++w) mx = fmaxf(mx, rf[w]);
    consumers_sync();
    xmax = mx;
  }
  TRACE(3);
  const uint32_t wq = warp & 3, e = warp >> 2, rl = wq * 32 + lane;
  uint32_t dphase = 0;   // dready completions consumed

  // ------------------------------------------------------------------ stage 1
  if (n1) {
    const Seg& S = p.seg[C.s1_seg];
    const int ea = exponent_of(S.s2max * xmax);
    const Slab last = slab_of(m, C.s1_sl0 + C.s1_sln - 1);
    const uint32_t nquad = (last.k0 + 32 * last.nq - st1.klo) / 4;
    zero_b_hi(bfrag, nquad / 8, tid);
    long long asum = 0, aabs = 0;
    uint32_t qd = tid;
    XQuad cur = load_xquad(p, S.s2h, st1.klo + 4 * min(qd, nquad - 1), m);
    while (qd < nquad) {  // one quad in flight ahead of the one being quantised
      const uint32_t nx = qd + kConsumerThreads;
      const XQuad nxt = load_xquad(p, S.s2h, st1.klo + 4 * min(nx, nquad - 1), m);
      const uint32_t k0 = st1.klo + 4 * qd;
      long long v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = cur.s[i] * cur.x[i];  // packed.cpp:160
        v[i] = __float2ll_rn(scale_pow2(a, kFix - ea));
        asum += v[i];
        aabs += v[i] < 0 ? -v[i] : v[i];
      }
      emit_quad(bfrag, st1.klo, k0, q_of(k0, m), v);
      cur = nxt;
      qd = nx;
    }
    tc::fence_proxy_async_smem();  // B is read by the MMA through the async proxy
    const long long A = cta_sum_i64(asum, red8);
    const long long Aabs = cta_sum_i64(aabs, red8);
    // one CTA per slab range publishes sum|a_int| (bounds every |t_k| of the segment)
    if (tid == 0 && C.s1_rt0 == 0)
      atomicAdd((unsigned long long*)&st->abs_a[b][C.s1_seg], (unsigned long long)Aabs);
    TRACE(4);
    mbar_wait_wd(&bars->full[0], 0);
    expand_stage(st1, buf, bars, bars->tmem, nullptr);
    TRACE(12);
    mbar_wait_wd(&bars->dready, dphase & 1);
    ++dphase;
    tc::fence_after_sync();
    TRACE(5);
    long long* Tseg = p.T + (size_t)b * p.r_cap + S.t_off + (size_t)C.s1_rt0 * 16;
    for (uint32_t rb = e; rb < st1.nrb; rb += 2) {
      const long long P = d_row(bars->tmem, rb, wq);
      const uint32_t row = rb * 128 + rl;
      if (row < st1.rows) atomicAdd((unsigned long long*)&Tseg[row], (unsigned long long)(2 * P - A));
    }
  }
  {  // clear this CTA's share of the other t buffer for the next launch
    long long* Tn = p.T + (size_t)(b ^ 1) * p.r_cap;
    const uint32_t lo = (uint32_t)((uint64_t)dirty_next * blockIdx.x / gridDim.x);
    const uint32_t hi = (uint32_t)((uint64_t)dirty_next * (blockIdx.x + 1) / gridDim.x);
    for (uint32_t i = lo + tid; i < hi; i += kConsumerThreads) Tn[i] = 0;
  }

  // --------------------------------------------------------------- grid barrier
  tc::fence_before_sync();
  consumers_sync();  // the CTA's reds to t happen-before thread 0's fence (cumulativity)
  TRACE(6);
  if (tid == 0) {
    __threadfence();
    const uint32_t arrived = atomicAdd(&st->done[b], 1u);
    if (arrived == gridDim.x - 1) {  // every CTA has read epoch and dirty: advance them
      st->epoch = ep + 1;
      st->dirty[b] = p.R1;
      st->dirty[b ^ 1] = 0;
      st->done[b ^ 1] = 0;
#pragma unroll
      for (int sg = 0; sg < kMaxSeg; ++sg) st->abs_a[b ^ 1][sg] = 0;
    }
  }
  if (!C.s2_rtn) {
    if (warp == 0) tc::tmem_dealloc(bars->tmem, kTmemCols);
    return;
  }
  TRACE(7);
  if (tid == 0) {
    uint32_t it = 0;
    while (ld_acquire(&st->done[b]) < gridDim.x) {
      __nanosleep(20);
      if (++it > (1u << 26)) __trap();
    }
  }
  consumers_sync();
  tc::fence_after_sync();
  TRACE(8);

  // ------------------------------------------------------------------ stage 2
  const Seg& S = S2seg;
  const int ea = exponent_of(S.s2max * xmax);
  // |t_k| = |sum_j +-a_int_j| <= sum_j |a_int_j|, published exactly by stage 1
  const unsigned long long tbound = __ldcg((const unsigned long long*)&st->abs_a[b][C.s2_seg]);
  const int et = tbound ? 64 - __clzll((long long)tbound) : 0;  // |t_k| < 2^et
  const int sh = et - kFix;
  const long long* Tseg = p.T + (size_t)b * p.r_cap + S.t_off;
  const uint32_t nquad2 = kpad(S.r) / 4;
  zero_b_hi(bfrag, nquad2 / 8, tid);
  long long tsum = 0;
  {
    uint32_t qd = tid;
    long long cur[4], nxt[4];
    load_tquad(Tseg, 4 * min(qd, nquad2 - 1), S.r, S.t_off, cur);
    while (qd < nquad2) {
      const uint32_t nx = qd + kConsumerThreads;
      load_tquad(Tseg, 4 * min(nx, nquad2 - 1), S.r, S.t_off, nxt);
      long long v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[i] = sh > 0 ? (cur[i] + (1ll << (sh - 1))) >> sh : cur[i] * (1ll << (-sh));
        tsum += v[i];
      }
      emit_quad(bfrag, 0, 4 * qd, q_of(4 * qd, S.r), v);
#pragma unroll
      for (int i = 0; i < 4; ++i) cur[i] = nxt[i];
      qd = nx;
    }
  }
  tc::fence_proxy_async_smem();
  const long long Tsum = cta_sum_i64(tsum, red8);
  TRACE(9);
  mbar_wait_wd(&bars->full[1], 0);
  expand_stage(st2, buf, bars, bars->tmem,
               (p.trace && warp == 0) ? p.trace + blockIdx.x * 32 + 22 : nullptr);
  TRACE(13);
  mbar_wait_wd(&bars->dready, dphase & 1);
  tc::fence_after_sync();
  TRACE(10);
  const int E = sh + ea - kFix;  // t = T2 * 2^sh * 2^(ea - kFix)
  for (uint32_t rb = e; rb < st2.nrb; rb += 2) {
    const long long P = d_row(bars->tmem, rb, wq);
    const uint32_t row = rb * 128 + rl;
    if (row < st2.rows && C.s2_rt0 * 16 + row < S.n) {
      const uint32_t orow = C.s2_rt0 * 16 + row;
      const long long Y = 2 * P - Tsum;
      const double y = (double)__half2float(S.s1h[orow]) * ldexp((double)Y, E);  // packed.cpp:189
      if (p.y_f32) ((float*)p.y[C.s2_seg])[orow] = (float)y;
      else ((__half*)p.y[C.s2_seg])[orow] = __float2half_rn((float)y);
    }
  }
  TRACE(11);
  tc::fence_before_sync();
  consumers_sync();
  if (warp == 0) tc::tmem_dealloc(bars->tmem, kTmemCols);
}

}  // namespace dec

using namespace dec;

void dec_state_reserve(nqb_context* ctx, uint32_t rows) {
  if (ctx->dec_state && ctx->dec_cap >= rows) return;
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ctx->dec_state) NQB_CUDA(cudaFree(ctx->dec_state));
  ctx->dec_state = nullptr;
  const uint32_t cap = std::max<uint32_t>(std::max<uint32_t>(rows, 2 * ctx->dec_cap), 1u << 14);
  const size_t bytes = sizeof(State) + 2 * (size_t)cap * sizeof(long long);
  NQB_CUDA(cudaMalloc(&ctx->dec_state, bytes));
  NQB_CUDA(cudaMemset(ctx->dec_state, 0, bytes));
  ctx->dec_cap = cap;
}

void group_gemv(nqb_context* ctx, const nqb_group* g, const void* d_x, int x_f32,
                void* const* d_ys, int y_f32) {
  NQB_REQUIRE(g->device == ctx->device, NQB_E_VALIDATION, "decode group lives on another device");
  NQB_REQUIRE(d_x != nullptr, NQB_E_VALIDATION, "null input");
  dec_state_reserve(ctx, g->R1);
  Params p{};
  p.bits = g->bits;
  std::copy(g->ctas, g->ctas + g->grid, p.ctas);
  for (uint32_t s = 0; s < g->nseg; ++s) {
    p.seg[s] = g->seg[s];
    NQB_REQUIRE(d_ys[s] != nullptr, NQB_E_VALIDATION, "null output");
    p.y[s] = d_ys[s];
  }
  p.nseg = g->nseg;
  p.m = g->m;
  p.R1 = g->R1;
  p.r_cap = ctx->dec_cap;
  p.st = (State*)ctx->dec_state;
  p.T = (long long*)((char*)ctx->dec_state + sizeof(State));
  p.buf_bytes = g->buf_bytes;
  p.slot_bytes = g->slot_bytes;
  p.nbar = g->nbar;
  p.bfrag_bytes = g->bfrag_bytes;
  p.x_f32 = x_f32 ? 1u : 0u;
  p.y_f32 = y_f32 ? 1u : 0u;
  p.x_vec = ((uintptr_t)d_x % 16 == 0) ? 1u : 0u;
  p.x = d_x;
  p.trace = (unsigned long long*)ctx->dec_trace;
  if (!ctx->dec_attr_set) {
    NQB_CUDA(cudaFuncSetAttribute(k_decode, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    ctx->dec_attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g->smem_bytes;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NQB_CUDA(cudaLaunchKernelEx(&cfg, k_decode, p));
  NQB_LAUNCHED(ctx);
}

// ---- single-layer entry points (the layer's implicit group of one) ---------
void decode_gemv_f32(nqb_context* ctx, const nqb_layer* L, const float* d_x, float* d_y) {
  void* ys[1] = {d_y};
  group_gemv(ctx, L->dec, d_x, 1, ys, 1);
}

void decode_gemv_f16(nqb_context* ctx, const nqb_layer* L, const __half* d_x, __half* d_y) {
  void* ys[1] = {d_y};
  group_gemv(ctx, L->dec, d_x, 0, ys, 0);
}

}  // namespace nqb
