// decode_dev.cuh — device helpers shared by the per-call decode kernel
// (decode.cu) and the persistent decode-pass kernel (decode_pass.cu).
#pragma once
#include <cfloat>
#include <cmath>

#include "decode.cuh"
#include "tc_common.cuh"

namespace nqb {
namespace dec {

// D += A(16x32 u8) * B(32x8 s8), int32 accumulate (IMMA.16832.U8.S8).
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

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
// Compiled only into the kTrace instance of the kernel: the production kernel
// carries no trace code (each check would re-read the parameter bank).
#define TRACE(i)                                                                  \
  do {                                                                            \
    if (kTrace && threadIdx.x == 0) {                                             \
      if ((i) == 0) {                                                             \
        trace_t0 = clock64();                                                     \
        trp[blockIdx.x * 32] = globaltimer();                                     \
      } else {                                                                    \
        trp[blockIdx.x * 32 + (i)] = clock64() - trace_t0;                        \
      }                                                                           \
    }                                                                             \
  } while (0)

__device__ __forceinline__ void red_add_u64(long long* p, long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
// Grid-barrier arrival: the release publishes this CTA's t reds (ordered
// before it by the CTA barrier, cumulativity).
__device__ __forceinline__ void red_release_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// mbarrier wait with a watchdog: a wait that never completes traps the
// launch (reported as a CUDA error) instead of hanging the device.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity, bool suspend) {
  uint32_t ok;
  if (suspend)
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity), "r"(0x989680u)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(parity)
        : "memory");
  return ok != 0;
}
// Slow path of mbar_wait_wd (one out-of-line copy): keeps waiting, with a
// wall-clock watchdog (a suspended try_wait may sleep) that traps after ~10 s so
// a wait that never completes is a reported launch error, not a hung device.
static __device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t parity, bool suspend) {
  const unsigned long long t0 = globaltimer();
  for (uint32_t it = 1;; ++it) {
    if (mbar_try(bar, parity, suspend)) return;
    if ((it & 255u) == 0 && globaltimer() - t0 > 10000000000ull) __trap();
  }
}
// With `suspend` the wait sleeps (suspend-time hint) instead of spinning, so
// waiting warps leave the issue slots to the warps that have work.
__device__ __forceinline__ void mbar_wait_wd(uint64_t* bar, uint32_t parity, bool suspend = false) {
  if (!mbar_try(bar, parity, suspend)) mbar_wait_slow(bar, parity, suspend);
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

// Signed base-256 digits (each in [-128, 127]) of the four values v[e]
// (|v| < 2^46): byte e of limb word w[l] is digit l of v[e].  Adding
// B = 0x808080808080 makes every digit d_l = byte_l(v + B) - 128, i.e. the
// byte XOR 0x80, so the digits are byte transposes (PRMT) of v + B.
static_assert(kLimbs == 6, "limb transpose assumes six limbs");
__device__ __forceinline__ void limbs4(const long long (&v)[4], uint32_t (&w)[kLimbs]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const unsigned long long u = (unsigned long long)v[e] + 0x808080808080ull;
    lo[e] = (uint32_t)u ^ 0x80808080u;
    hi[e] = (uint32_t)(u >> 32) ^ 0x8080u;
  }
  const uint32_t a0 = __byte_perm(lo[0], lo[1], 0x5140), a1 = __byte_perm(lo[0], lo[1], 0x7362);
  const uint32_t b0 = __byte_perm(lo[2], lo[3], 0x5140), b1 = __byte_perm(lo[2], lo[3], 0x7362);
  const uint32_t h0 = __byte_perm(hi[0], hi[1], 0x5140), h1 = __byte_perm(hi[2], hi[3], 0x5140);
  w[0] = __byte_perm(a0, b0, 0x5410);
  w[1] = __byte_perm(a0, b0, 0x7632);
  w[2] = __byte_perm(a1, b1, 0x5410);
  w[3] = __byte_perm(a1, b1, 0x7632);
  w[4] = __byte_perm(h0, h1, 0x5410);
  w[5] = __byte_perm(h0, h1, 0x7632);
}

// B-fragment words for the quad of inputs k0..k0+3 (values already << (7-q)):
// tile (k0-klo)/32 owns kTileB bytes = [limb g<kLimbs][c][h] words.
__device__ __forceinline__ void store_quad(uint8_t* bfrag, uint32_t klo, uint32_t k0,
                                           const uint32_t (&w)[kLimbs]) {
  // tiles 2i, 2i+1 interleave per (limb, c) so one 16-byte load feeds both
  const uint32_t kk = k0 & 31, h = kk >> 4, c = (kk >> 2) & 3, tt = (k0 - klo) >> 5;
  uint32_t* t = (uint32_t*)(bfrag + (tt >> 1) * 2 * kTileB) + (tt & 1) * 2 + h;
#pragma unroll
  for (uint32_t g = 0; g < kLimbs; ++g) t[(g * 4 + c) * 4] = w[g];
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

// Warp sums of (a, b) into red8[warp] and red8[kConsumerWarps + warp]; the
// next consumers_sync publishes them and sum_partials() finishes the CTA sum
// later, off the critical path.
__device__ __forceinline__ void warp_partials2(long long a, long long b, long long* red8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(~0u, a, o);
    b += __shfl_xor_sync(~0u, b, o);
  }
  if (lane == 0) {
    red8[warp] = a;
    red8[kConsumerWarps + warp] = b;
  }
}
__device__ __forceinline__ long long sum_partials(const long long* red8) {
  long long s = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) s += red8[w];
  return s;
}

__device__ __forceinline__ void cta_sum2_i64(long long& a, long long& b, long long* red8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(~0u, a, o);
    b += __shfl_xor_sync(~0u, b, o);
  }
  consumers_sync();
  if (lane == 0) {
    red8[warp] = a;
    red8[kConsumerWarps + warp] = b;
  }
  consumers_sync();
  a = 0;
  b = 0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) {
    a += red8[w];
    b += red8[kConsumerWarps + w];
  }
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
  const uint32_t b = __float_as_uint(M);
  if (!(M > 0.f) || b >= 0x7f800000u) return 0;
  if (b >= 0x00800000u) return (int)(b >> 23) - 126;  // normal: frexp exponent, M < 2^e
  return -126 - __clz((int)b) + 9;                    // subnormal: M < 2^(-149 + bitlength)
}

// Exponent of the activation bound: |a| = |s2 x| <= s2max * xmax < 2^(e(s2max) + e(xmax)).
// Taken per factor so the product cannot overflow fp32.  A zero factor means a = 0.
__device__ __forceinline__ int act_exponent(float s2max, float xmax) {
  if (!(s2max > 0.f) || !(xmax > 0.f)) return 0;
  return exponent_of(s2max) + exponent_of(xmax);
}

// max |x_j| over j < m, read by all consumer threads of the CTA (every CTA reads
// the whole input).  A NaN or +-Inf input yields +Inf: the caller then writes NaN
// outputs, as the reference's gemv_two_stage propagates non-finite activations.
// binary16 x is reduced on the magnitude bits (monotone in |x|; >= 0x7C00 is
// Inf/NaN).  xred holds kConsumerWarps floats.
__device__ __forceinline__ float x_absmax(const void* x, uint32_t m, bool f32, bool vec,
                                          float* xred) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float mx = 0.f;
  if (f32) {
    const float* xf = (const float*)x;
    const uint32_t nv = vec ? m / 4 : 0;
    bool bad = false;
#pragma unroll 4
    for (uint32_t i = tid; i < nv; i += kConsumerThreads) {
      const float4 v = __ldcg((const float4*)xf + i);
      const float a = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
      bad |= !(fabsf(v.x) <= FLT_MAX) | !(fabsf(v.y) <= FLT_MAX) | !(fabsf(v.z) <= FLT_MAX) |
             !(fabsf(v.w) <= FLT_MAX);
      mx = fmaxf(mx, a);
    }
    for (uint32_t i = 4 * nv + tid; i < m; i += kConsumerThreads) {
      const float a = fabsf(__ldcg(xf + i));
      bad |= !(a <= FLT_MAX);
      mx = fmaxf(mx, a);
    }
    if (bad) mx = __int_as_float(0x7f800000);
  } else {
    const unsigned short* xh = (const unsigned short*)x;
    uint32_t mb = 0;
    const uint32_t nv = vec ? m / 8 : 0;
#pragma unroll 4
    for (uint32_t i = tid; i < nv; i += kConsumerThreads) {
      const uint4 v = __ldcg((const uint4*)xh + i);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) mb = max(mb, max(w[e] & 0x7FFFu, (w[e] >> 16) & 0x7FFFu));
    }
    for (uint32_t i = 8 * nv + tid; i < m; i += kConsumerThreads)
      mb = max(mb, (uint32_t)(__ldcg(xh + i) & 0x7FFFu));
    mx = mb >= 0x7C00u ? __int_as_float(0x7f800000)
                       : __half2float(__ushort_as_half((unsigned short)mb));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, o));
  consumers_sync();  // xred may still be read from a previous use
  if (lane == 0) xred[warp] = mx;
  consumers_sync();
  mx = 0.f;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) mx = fmaxf(mx, xred[w]);
  return mx;
}

// Right shift that takes t to 38-bit fixed point: |a_int| <= 2^kFix, so
// |t_k| <= m 2^kFix < 2^(kFix + ceil_log2(m) + 1).  A bound known before stage 1
// (no published sum|a| on the critical path); t keeps >= 2^-30 relative
// resolution of its largest possible magnitude, far below the 1e-3 bar.
__device__ __forceinline__ int t_shift(uint32_t m) {
  return (m <= 1 ? 0 : 32 - __clz((int)(m - 1))) + 1;
}

__device__ __forceinline__ bool is_inf(float v) { return __float_as_int(v) == 0x7f800000; }

// Words w_0..w_3 of this lane in a unit with nq tiles (formats: decode_plan.cu).
__device__ __forceinline__ void unit_words(const uint8_t* unit, uint32_t nq, int lane,
                                           uint32_t (&w)[4]) {
  if (nq == 8) {
    const uint4 v = *(const uint4*)(unit + lane * 16);
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  } else if (nq == 4) {
    const uint2 v = *(const uint2*)(unit + lane * 8);
    w[0] = v.x;
    w[1] = v.x >> 4;
    w[2] = v.y;
    w[3] = v.y >> 4;
  } else {
    const uint32_t u = *(const uint32_t*)(unit + lane * 4);
    w[0] = u;
    w[1] = u >> 2;
    w[2] = u >> 4;
    w[3] = u >> 6;
  }
}

// Adds 4 accumulator chains of one row tile to the per-limb row sums
// red32[row][limb] (16 rows x kRedStride ints): chains are summed in int32
// (|sum| < 2^30) and lane c adds limbs 2c, 2c+1 of rows g and g+8 with native
// 32-bit shared atomics (the limb sums stay < 2^31: sum_K 2^q * |limb| <= K * 2^14).
__device__ __forceinline__ void flush_rows(int (&acc)[4][4], int* red32, int lane) {
  const int g = lane >> 2, c = lane & 3;
  if (c >= (kLimbs + 1) / 2) {
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0;
    return;
  }
  int s[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s[i] = acc[0][i] + acc[1][i] + acc[2][i] + acc[3][i];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q][i] = 0;
  }
  int* r0 = red32 + g * kRedStride + 2 * c;
  int* r1 = red32 + (g + 8) * kRedStride + 2 * c;
  atomicAdd(r0, s[0]);
  atomicAdd(r0 + 1, s[1]);
  atomicAdd(r1, s[2]);
  atomicAdd(r1 + 1, s[3]);
}

// sum_K bit * value of a row from its limb sums (exact; two's-complement
// wraparound of the partial sums is harmless because the total fits).
__device__ __forceinline__ long long row_value(const int* red32row) {
  unsigned long long v = 0;
#pragma unroll
  for (int l = 0; l < kLimbs; ++l) v += (unsigned long long)(long long)red32row[l] << (8 * l);
  return (long long)v >> 7;
}

struct StageArgs {
  uint32_t rtn, nsec, sec_base;   // row tiles, sections, index of the first section
  uint32_t K, slab_base, klo;     // K dimension, first slab, its k0
  uint32_t lin_off;               // linear mode: buffer offset of the first section
};

// B fragments of one slab for this lane: b[q] = limbs g of the 4-input groups
// 4c.. and 16+4c.. of tile q (lanes g >= kLimbs feed zero columns).
__device__ __forceinline__ void load_b(const uint8_t* bfrag, uint32_t klo, const Slab& sl,
                                       uint32_t g, uint32_t c, uint2 (&b)[8]) {
  const uint8_t* bp = bfrag + kBytesPerK * (sl.k0 - klo) + (g * 4 + c) * 16;
#pragma unroll
  for (int q = 0; q < 8; q += 2) {
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (q < (int)sl.nq && g < (uint32_t)kLimbs) v = *(const uint4*)(bp + q * kTileB);
    b[q] = make_uint2(v.x, v.y);
    b[q + 1] = make_uint2(v.z, v.w);
  }
}

// NT (1 or 2) row tiles of one slab against shared B fragments: tile q of the
// slab accumulates into chain q&3 of each row tile.
template <int NT>
__device__ __forceinline__ void tiles_mma(const uint8_t* unit0, uint32_t ub, uint32_t nq, int lane,
                                          const uint2 (&b)[8], int (&acc)[2][4][4]) {
  uint32_t w[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) unit_words(unit0 + j * ub, nq, lane, w[j]);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q >= (int)nq) break;
    const uint32_t mask = 0x01010101u << q;
#pragma unroll
    for (int j = 0; j < NT; ++j)
      mma_u8s8(acc[j][q & 3], w[j][0] & mask, w[j][1] & mask, w[j][2] & mask, w[j][3] & mask,
               b[q].x, b[q].y);
  }
}

// A run of cnt full (256-wide) slabs for NT row tiles starting at unit u (the
// next slab's unit is ustep bytes on) against B fragments at bp (next slab
// kBytesPerK*256 on).  Software-pipelined: the next slab's A words and B
// fragments are loaded before this slab's 8*NT MMAs issue.
template <int NT>
__device__ __forceinline__ void full_run(const uint8_t* u, uint32_t ustep, const uint8_t* bp,
                                         uint32_t cnt, int lane, bool limb_lane,
                                         int (&acc)[2][4][4]) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  uint4 w[NT], bq[4];
#pragma unroll
  for (int j = 0; j < NT; ++j) w[j] = *(const uint4*)(u + j * 512 + lane * 16);
#pragma unroll
  for (int h = 0; h < 4; ++h) bq[h] = limb_lane ? *(const uint4*)(bp + 2 * h * kTileB) : z;
  auto slab = [&]() {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t mask = 0x01010101u << q;
      const uint32_t b0 = (q & 1) ? bq[q >> 1].z : bq[q >> 1].x;
      const uint32_t b1 = (q & 1) ? bq[q >> 1].w : bq[q >> 1].y;
#pragma unroll
      for (int j = 0; j < NT; ++j)
        mma_u8s8(acc[j][q & 3], w[j].x & mask, w[j].y & mask, w[j].z & mask, w[j].w & mask, b0, b1);
    }
  };
  // the last slab is peeled: no re-read of operands that will not be used
  // (shared-memory bandwidth is tight when every warp runs only one slab)
  for (uint32_t i = 0; i + 1 < cnt; ++i) {
    u += ustep;
    bp += kBytesPerK * 256;
    uint4 nw[NT], nb[4];
#pragma unroll
    for (int j = 0; j < NT; ++j) nw[j] = *(const uint4*)(u + j * 512 + lane * 16);
#pragma unroll
    for (int h = 0; h < 4; ++h) nb[h] = limb_lane ? *(const uint4*)(bp + 2 * h * kTileB) : z;
    slab();
#pragma unroll
    for (int j = 0; j < NT; ++j) w[j] = nw[j];
#pragma unroll
    for (int h = 0; h < 4; ++h) bq[h] = nb[h];
  }
  slab();
}

// All sections of one stage; leaves sum_K bit*value per row in red[] (exact).
// Linear mode: the stage's sections are resident (one mbarrier per stage);
// work items (pair of row tiles, run of sections) go round-robin to the
// consumer warps, each B-fragment load serving both tiles.  Ring mode: the
// stream is longer than the buffer; every warp walks every section in order
// and releases it (slot reuse), handling tiles t = w mod warp.
// kBig (plans with long per-CTA streams): a warp's consecutive full slabs of
// one tile pair run software-pipelined (full_run); the small-layer instance
// keeps the plain loop (smaller code, lower latency for 1-2 steps per warp).
template <bool kBig>
__device__ __forceinline__ void run_stage(const StageArgs& A, uint32_t NS, bool ring_mode,
                                          uint32_t slot_bytes, uint64_t* full, uint64_t* empty,
                                          const uint8_t* buf, const uint8_t* bfrag,
                                          int* red, unsigned long long* prof) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t g = lane >> 2, c = lane & 3;
  int acc[2][4][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q][0] = acc[j][q][1] = acc[j][q][2] = acc[j][q][3] = 0;
  if (!A.rtn || !A.nsec) return;
  uint2 b[8];
  if (!ring_mode) {
    // warp w walks a contiguous range of the (tile pair, section) steps in
    // pair-major order, so its accumulators persist across sections and it
    // flushes only when the pair changes (at most a few times).
    const uint32_t npair = (A.rtn + 1) / 2, U = npair * A.nsec;
    const uint32_t f0 = (uint32_t)((uint64_t)U * warp / kConsumerWarps);
    const uint32_t f1 = (uint32_t)((uint64_t)U * (warp + 1) / kConsumerWarps);
    if (f0 < f1) {
      long long c0 = prof ? clock64() : 0;
      mbar_wait_wd(&full[A.sec_base], 0);  // the whole stage has landed
      if (prof && lane == 0) prof[0] += clock64() - c0;
    }
    uint32_t cur = f0 < f1 ? f0 / A.nsec : 0;
    long long c1 = prof ? clock64() : 0, tf = 0;
    if constexpr (kBig) {
      uint32_t F, rem;
      slab_split(A.K, F, rem);
      const uint32_t nfull = F > A.slab_base ? F - A.slab_base : 0;  // full slabs come first
      for (uint32_t f = f0; f < f1;) {
        // one run: the warp's consecutive sections of tile pair pr
        const uint32_t pr = f / A.nsec;
        uint32_t s = f - pr * A.nsec;
        const uint32_t send = min(A.nsec, s + (f1 - f));
        f = pr * A.nsec + send;
        if (pr != cur) {
          flush_rows(acc[0], red + 2 * cur * 16 * kRedStride, lane);
          if (2 * cur + 1 < A.rtn) flush_rows(acc[1], red + (2 * cur + 1) * 16 * kRedStride, lane);
          cur = pr;
        }
        const uint32_t t0 = 2 * pr;
        const bool two = t0 + 1 < A.rtn;
        const uint32_t sf = min(send, nfull);
        if (s < sf) {
          const uint32_t k0 = 256 * (A.slab_base + s);
          const uint8_t* unit = buf + A.lin_off + 2u * A.rtn * (k0 - A.klo) + t0 * 512;
          const uint8_t* bp = bfrag + kBytesPerK * (k0 - A.klo) + (g * 4 + c) * 16;
          if (two) full_run<2>(unit, 512u * A.rtn, bp, sf - s, lane, g < (uint32_t)kLimbs, acc);
          else full_run<1>(unit, 512u * A.rtn, bp, sf - s, lane, g < (uint32_t)kLimbs, acc);
          s = sf;
        }
        for (; s < send; ++s) {  // the 128 / 64 tails
          const Slab sl = slab_of(A.K, A.slab_base + s);
          const uint32_t ub = unit_bytes(sl.nq);
          const uint8_t* unit = buf + A.lin_off + 2u * A.rtn * (sl.k0 - A.klo) + t0 * ub;
          load_b(bfrag, A.klo, sl, g, c, b);
          if (two) tiles_mma<2>(unit, ub, sl.nq, lane, b, acc);
          else tiles_mma<1>(unit, ub, sl.nq, lane, b, acc);
        }
      }
    } else
    for (uint32_t f = f0; f < f1; ++f) {
      const uint32_t pr = f / A.nsec, s = f % A.nsec;
      if (pr != cur) {
        const long long cf = prof ? clock64() : 0;
        flush_rows(acc[0], red + 2 * cur * 16 * kRedStride, lane);
        if (2 * cur + 1 < A.rtn) flush_rows(acc[1], red + (2 * cur + 1) * 16 * kRedStride, lane);
        if (prof) tf += clock64() - cf;
        cur = pr;
      }
      const uint32_t t0 = 2 * pr;
      const Slab sl = slab_of(A.K, A.slab_base + s);
      const uint32_t ub = unit_bytes(sl.nq);
      // sections are contiguous in K: section s starts 2*rtn*(k0 - klo) bytes in
      const uint8_t* unit = buf + A.lin_off + 2u * A.rtn * (sl.k0 - A.klo) + t0 * ub;
      load_b(bfrag, A.klo, sl, g, c, b);
      if (t0 + 1 < A.rtn) tiles_mma<2>(unit, ub, sl.nq, lane, b, acc);
      else tiles_mma<1>(unit, ub, sl.nq, lane, b, acc);
    }
    if (f0 < f1) {
      const long long cf = prof ? clock64() : 0;
      flush_rows(acc[0], red + 2 * cur * 16 * kRedStride, lane);
      if (2 * cur + 1 < A.rtn) flush_rows(acc[1], red + (2 * cur + 1) * 16 * kRedStride, lane);
      if (prof && lane == 0) {
        tf += clock64() - cf;
        prof[2] += clock64() - c1 - tf;
        prof[3] += tf;
        uint32_t units = 0;
        for (uint32_t f = f0; f < f1; ++f) units += (2 * (f / A.nsec) + 1 < A.rtn) ? 2 : 1;
        prof[4] += units;
      }
    }
  } else {
    for (uint32_t s = 0; s < A.nsec; ++s) {
      const uint32_t sec = A.sec_base + s, slot = sec % NS;
      const Slab sl = slab_of(A.K, A.slab_base + s);
      mbar_wait_wd(&full[slot], (sec / NS) & 1);
      if ((uint32_t)warp < A.rtn) load_b(bfrag, A.klo, sl, g, c, b);
      for (uint32_t t = warp; t < A.rtn; t += kConsumerWarps) {
        tiles_mma<1>(buf + (size_t)slot * slot_bytes + t * unit_bytes(sl.nq), 0, sl.nq, lane, b,
                     acc);
        flush_rows(acc[0], red + t * 16 * kRedStride, lane);
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&empty[slot]);
    }
  }
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
  uint32_t w[kLimbs];
  const long long sv[4] = {v[0] * (1 << (7 - q)), v[1] * (1 << (7 - q)), v[2] * (1 << (7 - q)),
                           v[3] * (1 << (7 - q))};
  limbs4(sv, w);
  store_quad(bfrag, klo, k0, w);
}

struct XQuad {
  float s[4], x[4];
};

// s2s: the CTA's staged s2 slice, indexed by k (zero beyond m)
__device__ __forceinline__ XQuad load_xquad(const void* x, bool f32, bool vec,
                                            const __half* s2s, uint32_t k0, uint32_t m) {
  XQuad r;
  if (k0 + 3 < m && vec) {
    const uint2 sh2 = *(const uint2*)(s2s + k0);
    const float2 s01 = __half22float2(*(const __half2*)&sh2.x);
    const float2 s23 = __half22float2(*(const __half2*)&sh2.y);
    r.s[0] = s01.x; r.s[1] = s01.y; r.s[2] = s23.x; r.s[3] = s23.y;
    if (f32) {
      const float4 v = __ldcg((const float4*)((const float*)x + k0));
      r.x[0] = v.x; r.x[1] = v.y; r.x[2] = v.z; r.x[3] = v.w;
    } else {
      const uint2 v = __ldcg((const uint2*)((const __half*)x + k0));
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
        r.s[e] = __half2float(s2s[j]);
        r.x[e] = f32 ? __ldcg((const float*)x + j)
                     : __half2float(__ushort_as_half(__ldcg((const unsigned short*)x + j)));
      }
    }
  }
  return r;
}
__device__ __forceinline__ XQuad load_xquad(const Params& p, const __half* s2s, uint32_t k0,
                                            uint32_t m) {
  return load_xquad(p.x, p.x_f32 != 0, p.x_vec != 0, s2s, k0, m);
}

// t quad k0..k0+3 of a segment; `abs_row` is the absolute int64 index of Tseg[0]
// (16-byte vector loads need it even)
__device__ __forceinline__ void load_tquad(const long long* Tseg, uint32_t k0, uint32_t r,
                                           uint64_t abs_row, long long (&v)[4]) {
  if (k0 + 3 < r && ((abs_row + k0) & 1) == 0) {
    const longlong2 v0 = __ldcg((const longlong2*)(Tseg + k0));
    const longlong2 v1 = __ldcg((const longlong2*)(Tseg + k0 + 2));
    v[0] = v0.x; v[1] = v0.y; v[2] = v1.x; v[3] = v1.y;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = k0 + e < r ? __ldcg(Tseg + k0 + e) : 0;
  }
}

}  // namespace dec
}  // namespace nqb
