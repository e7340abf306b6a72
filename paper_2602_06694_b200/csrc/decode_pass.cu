// decode_pass.cu — persistent multi-layer decode kernel (one launch per decode
// pass) and its host-side builder.  Design: decode_pass.cuh, DESIGN.md §4b.
//
// Arithmetic is the per-call kernel's (decode.cu, gemv_two_stage of
// packed.cpp:153-192 in exact integer IMMA form), so a layer's output is the
// same function of its input in both kernels: the activation exponent comes
// from max|x| (a prepass or the producing step's published max|y|, equal to
// the per-call kernel's own pass over x) and the t exponent from m.
//
// This translation unit runs 12 consumer warps in two stage groups (+5 helper
// warps = 544 threads, 120 registers per thread at one CTA per SM).
#define NQB_DEC_WARPS 12
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "decode_dev.cuh"
#include "decode_pass.cuh"

namespace nqb {
namespace dec {

constexpr int kPassThreads = kConsumerThreads + 32 * kPassHelpers;

// ---- global-memory handshakes (helper warps only; one lane) -------------------
__device__ __forceinline__ void poll_ctr(const unsigned long long* c, unsigned long long target) {
  unsigned long long cur;
  const unsigned long long t0 = globaltimer();
  for (uint32_t it = 0;; ++it) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(cur) : "l"(c) : "memory");
    if (cur >= target) break;
    __nanosleep(32);  // leave the issue slots to the consumer warps
    // watchdog: a barrier that does not complete within seconds means the grid
    // is not co-resident or diverged; fail the launch instead of hanging
    if ((it & 255u) == 255u && globaltimer() - t0 > 4000000000ull) __trap();
  }
  // the data behind the barrier is read next by TMA (async proxy)
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
// Bulk prefetch of [p, p + bytes) into L2 (no shared memory, no completion).
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  for (uint32_t o = 0; o < bytes; o += 32768u) {
    const uint32_t n = min(32768u, bytes - o);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"((const char*)p + o), "r"(n)
                 : "memory");
  }
}
__device__ __forceinline__ void arrive_ctr(unsigned long long* c) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;\n" ::"l"(c) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* c) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(c) : "memory");
  return v;
}

// Stage geometry of one CTA in one step.
struct StageGeo {
  uint32_t rtn, nsec, K, slab0, klo;
  uint64_t src_off;   // byte offset of section 0 in the step's bits
  uint32_t prefix, suffix;  // staged scale bytes (stage 1: s2, stage 2: s1)
};

__device__ __forceinline__ StageGeo stage1_geo(const StepDesc& D, const Cta& C) {
  StageGeo g{};
  if (!C.s1_rtn || !C.s1_sln) return g;
  g.rtn = C.s1_rtn;
  g.nsec = C.s1_sln;
  g.K = D.m;
  g.slab0 = C.s1_sl0;
  g.klo = slab_of(D.m, C.s1_sl0).k0;
  const Slab last = slab_of(D.m, C.s1_sl0 + C.s1_sln - 1);
  g.src_off = C.stream_off;
  g.prefix = 2 * (last.k0 + 32 * last.nq - g.klo);
  return g;
}

__device__ __forceinline__ StageGeo stage2_geo(const StepDesc& D, const Cta& C) {
  StageGeo g{};
  if (!C.s2_rtn) return g;
  const uint32_t r = D.seg[C.s2_seg].r;
  g.rtn = C.s2_rtn;
  g.nsec = nslabs(r);
  g.K = r;
  uint64_t s1b = 0;
  if (C.s1_rtn && C.s1_sln) {
    const uint32_t k0 = slab_of(D.m, C.s1_sl0).k0;
    const Slab last = slab_of(D.m, C.s1_sl0 + C.s1_sln - 1);
    s1b = 2ull * C.s1_rtn * (last.k0 + 32 * last.nq - k0);
  }
  g.src_off = C.stream_off + s1b;
  g.suffix = 32u * C.s2_rtn;
  return g;
}

// Bytes of one row tile over the stage's first i slabs (U_i of the pair-major
// layout, k_relayout): the full 256-wide slabs come first, then <= 2 tails.
__device__ __forceinline__ uint32_t cum_bytes(const StageGeo& g, uint32_t i) {
  uint32_t F, rem;
  slab_split(g.K, F, rem);
  const uint32_t nf = F > g.slab0 ? min(F - g.slab0, i) : 0u;
  uint32_t bytes = 512u * nf;
  for (uint32_t s = nf; s < i; ++s) bytes += unit_bytes(slab_of(g.K, g.slab0 + s).nq);
  return bytes;
}

// Ring placement shared by producer and consumers: chunks never wrap.
__device__ __forceinline__ uint64_t ring_place(uint64_t& pos, uint32_t bytes, uint32_t ring) {
  const uint32_t off = (uint32_t)(pos % ring);
  if (off + bytes > ring) pos += ring - off;
  const uint64_t start = pos;
  pos += bytes;
  return start;
}

// Where the producer put a chunk (one work item; written before the chunk's
// copy is issued, read by the consuming warp after the chunk's full barrier).
struct ChunkRec {
  uint32_t off;      // ring byte offset
  uint32_t i0;       // first work item of the wave
};
static_assert(sizeof(ChunkRec) <= 16, "chunk record slot");

// max|x| bits over x[lo, hi): binary16 magnitude bits (>= 0x7C00: non-finite)
// or |fp32| bits (non-finite -> +Inf bits), so every bound is an ordered uint.
__device__ __noinline__ uint32_t absmax_bits(const void* x, uint32_t lo, uint32_t hi, bool f32,
                                             bool vec, uint32_t t, uint32_t nt) {
  uint32_t mb = 0;
  if (f32) {
    const uint32_t* xf = (const uint32_t*)x;
    uint32_t i = lo + t * 4;
    if (vec)
      for (; i + 3 < hi; i += 4 * nt) {
        const uint4 v = __ldcg((const uint4*)(xf + i));
        mb = max(mb, max(max(v.x & 0x7FFFFFFFu, v.y & 0x7FFFFFFFu),
                         max(v.z & 0x7FFFFFFFu, v.w & 0x7FFFFFFFu)));
      }
    for (uint32_t j = i; j < min(hi, i + 4); ++j) mb = max(mb, __ldcg(xf + j) & 0x7FFFFFFFu);
    if (!vec)
      for (uint32_t j = lo + t; j < hi; j += nt) mb = max(mb, __ldcg(xf + j) & 0x7FFFFFFFu);
    return mb >= 0x7F800000u ? 0x7F800000u : mb;
  }
  const unsigned short* xh = (const unsigned short*)x;
  uint32_t i = lo + t * 8;
  if (vec)
    for (; i + 7 < hi; i += 8 * nt) {
      const uint4 v = __ldcg((const uint4*)(xh + i));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) mb = max(mb, max(w[e] & 0x7FFFu, (w[e] >> 16) & 0x7FFFu));
    }
  if (vec) {
    for (uint32_t j = i; j < min(hi, i + 8); ++j) mb = max(mb, (uint32_t)(__ldcg(xh + j) & 0x7FFFu));
  } else {
    for (uint32_t j = lo + t; j < hi; j += nt) mb = max(mb, (uint32_t)(__ldcg(xh + j) & 0x7FFFu));
  }
  return mb;
}
// max|x| bits over one 8-element unit x[a, b) (a 8-aligned; same encoding as
// absmax_bits), inlined so several units' loads are in flight together.
__device__ __forceinline__ uint32_t unit_absmax(const void* x, uint32_t a, uint32_t b, bool f32,
                                                bool vec) {
  uint32_t mb = 0;
  if (f32) {
    const uint32_t* xf = (const uint32_t*)x;
    if (vec && b - a == 8) {
      const uint4 v0 = __ldcg((const uint4*)(xf + a)), v1 = __ldcg((const uint4*)(xf + a + 4));
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) mb = max(mb, w[e] & 0x7FFFFFFFu);
    } else {
      for (uint32_t j = a; j < b; ++j) mb = max(mb, __ldcg(xf + j) & 0x7FFFFFFFu);
    }
    return mb >= 0x7F800000u ? 0x7F800000u : mb;
  }
  const unsigned short* xh = (const unsigned short*)x;
  if (vec && b - a == 8) {
    const uint4 v = __ldcg((const uint4*)(xh + a));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) mb = max(mb, max(w[e] & 0x7FFFu, (w[e] >> 16) & 0x7FFFu));
  } else {
    for (uint32_t j = a; j < b; ++j) mb = max(mb, (uint32_t)(__ldcg(xh + j) & 0x7FFFu));
  }
  return mb;
}
// Bound bits -> float max|x| (+Inf for a non-finite input).
__device__ __forceinline__ float bound_value(uint32_t bits, bool f32) {
  if (f32) return __uint_as_float(bits);
  return bits >= 0x7C00u ? __int_as_float(0x7f800000)
                         : __half2float(__ushort_as_half((unsigned short)bits));
}
// Share [lo, hi) of m inputs for CTA b of G (8-aligned boundaries).
__device__ __forceinline__ void share_of(uint32_t m, uint32_t b, uint32_t G, uint32_t& lo,
                                         uint32_t& hi) {
  const uint32_t units = (m + 7) / 8, per = (units + G - 1) / G;
  lo = min(m, 8 * per * b);
  hi = min(m, lo + 8 * per);
}

#define PSTAMP(k, i)                                                           \
  do {                                                                         \
    if (kTrace) trp[1 + kPassStamps * (k) + (i)] = globaltimer();              \
  } while (0)

// Named barriers of the two consumer groups (ids 1, 2) and of all consumers (3).
__device__ __forceinline__ void group_sync(int gid, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1 + gid), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void all_consumers_sync() {
  asm volatile("bar.sync 3, %0;\n" ::"n"(kConsumerThreads) : "memory");
}
template <bool kTrace, int kW1>
__global__ void __launch_bounds__(kPassThreads, 1) k_decode_pass(const __grid_constant__ PassParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full1 = (uint64_t*)smem;  // stage-1 ring
  uint64_t* empty1 = full1 + kPassSlots;
  uint64_t* full2 = empty1 + kPassSlots;  // stage-2 ring
  uint64_t* empty2 = full2 + kPassSlots;
  uint64_t* dfull = empty2 + kPassSlots;
  uint64_t* dempty = dfull + kDescSlots;
  uint64_t* bfull1 = dempty + kDescSlots;  // quantised-x slots
  uint64_t* bempty1 = bfull1 + kBSlots;
  uint64_t* bfull2 = bempty1 + kBSlots;    // quantised-t slots
  uint64_t* bempty2 = bfull2 + kBSlots;
  uint64_t* cdone1 = bempty2 + kBSlots;
  uint64_t* cdone2 = cdone1 + kDoneRing;
  uint32_t* misc = (uint32_t*)(cdone2 + kDoneRing);  // [0] parity, [2..3] target
  uint8_t* dslots = (uint8_t*)misc + 64;
  float* xmaxs = (float*)(dslots + kDescSlots * kDescSlotBytes + 256);  // max|x| of steps in flight (ring of 16)
  ChunkRec* recs1 = (ChunkRec*)((uint8_t*)xmaxs + 64);
  ChunkRec* recs2 = recs1 + kPassSlots;
  uint8_t* bslots1 = smem + pass_head_bytes();       // header | B fragments of x
  constexpr uint32_t NB = kBSlots;
  uint8_t* bslots2 = bslots1 + NB * p.bslot1_bytes;  // header | B fragments of t | s1 slice
  uint8_t* ring1 = bslots2 + NB * p.bslot2_bytes;
  uint8_t* ring2 = ring1 + p.ring1_bytes;

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const uint32_t K = p.K, G = p.G, P = p.P;
  const bool sus = (p.debug & 4u) != 0;
  auto desc_of = [&](uint32_t k) -> const StepDesc& {
    return *(const StepDesc*)(dslots + (k % kDescSlots) * kDescSlotBytes);
  };
  auto cta_of = [&](uint32_t k) -> const Cta& {
    return *(const Cta*)(dslots + (k % kDescSlots) * kDescSlotBytes + 480);
  };
  auto wait_desc = [&](uint32_t k) { mbar_wait_wd(&dfull[k % kDescSlots], (k / kDescSlots) & 1, sus); };

  if (tid == 0) {
    for (int s = 0; s < kPassSlots; ++s) {
      tc::mbar_init(&full1[s], 1);
      // a chunk is a wave of W = GW / wave_div items, one per warp of W warps
      tc::mbar_init(&empty1[s], kW1 / p.wave_div);
      tc::mbar_init(&full2[s], 1);
      tc::mbar_init(&empty2[s], (kConsumerWarps - kW1) / p.wave_div2);
    }
    for (int s = 0; s < kDescSlots; ++s) {
      tc::mbar_init(&dfull[s], 1);
      tc::mbar_init(&dempty[s], 7);  // stage-2 group, two producers, 2 x and 2 t quantisers
    }
    for (int s = 0; s < kBSlots; ++s) {
      tc::mbar_init(&bfull1[s], 2);  // the two quantiser warps
      tc::mbar_init(&bempty1[s], 1);
      tc::mbar_init(&bfull2[s], 2);
      tc::mbar_init(&bempty2[s], 1);
    }
    for (int s = 0; s < kDoneRing; ++s) {
      tc::mbar_init(&cdone1[s], 1);
      tc::mbar_init(&cdone2[s], 1);
    }
    tc::fence_mbar_init();
    const unsigned long long gen = ld_relaxed_u64(p.ctr);
    misc[0] = (uint32_t)(gen & 1);
    *(unsigned long long*)(misc + 2) = (gen + 1) * p.P;  // step barriers: the partition's CTAs
    *(unsigned long long*)(misc + 4) = (gen + 1) * G;    // kernel-start barrier: every CTA
  }
  __syncthreads();
  const uint32_t par = misc[0];
  const unsigned long long target = *(const unsigned long long*)(misc + 2);
  const unsigned long long target_all = *(const unsigned long long*)(misc + 4);
  // this CTA's partition and its step list (local index j -> step D.idx)
  const uint32_t sub = blockIdx.x / p.P;
  const uint32_t Kc = sub < p.nsub ? p.list_off[sub + 1] - p.list_off[sub] : 0u;
  const uint32_t prank = blockIdx.x - sub * p.P;  // rank inside the partition
  unsigned long long* xinit = p.ctr + kCtrStride;
  unsigned long long* tbar = p.ctr + 2 * kCtrStride;
  unsigned long long* ybar = tbar + (size_t)K * kCtrStride;
  unsigned* amax = p.amax + (size_t)par * p.amax_words * 4;
  long long* arena = p.arena + (size_t)par * p.arena_len;
  unsigned long long* trp = nullptr;
  if (kTrace) {
    trp = p.trace + (size_t)blockIdx.x * (kPassStamps * K + 2);
    if (tid == 0) trp[0] = globaltimer();
  }

  // ============================================================= helper warps
  if (warp >= kConsumerWarps) {
    const int role = warp - kConsumerWarps;
    if (role == 0 || role == 7) {
      // ----------------------------------------------- producers (one per ring)
      // role 0 streams stage-1 sections step after step into ring 1, role 7
      // stage-2 sections into ring 2.  The rings fill independently: stage 1 of
      // later steps keeps streaming while stage 2 of a step waits for its t
      // barrier (weights do not depend on x, so nothing orders the two streams).
      if (lane != 0) return;
      const int r = role == 0 ? 0 : 1;
      const uint32_t RB = r ? p.ring2_bytes : p.ring1_bytes;
      uint64_t* fullr = r ? full2 : full1;
      uint64_t* emptyr = r ? empty2 : empty1;
      ChunkRec* recs = r ? recs2 : recs1;
      uint8_t* ring = r ? ring2 : ring1;
      uint64_t pos = 0, starts[kPassSlots];
      uint32_t chunk = 0, rel = 0;
      for (uint32_t j = 0; j < Kc; ++j) {
        wait_desc(j);
        const StepDesc& D = desc_of(j);
        const Cta& C = cta_of(j);
        const uint32_t k = D.idx;
        const StageGeo g = r ? stage2_geo(D, C) : stage1_geo(D, C);
        if (kTrace) PSTAMP(k, r ? 14 : 11);
        // The weights do not depend on x: while this step streams through the
        // ring, pull the stage's bytes of step j + ahead from HBM into L2, so the
        // ring's copies see L2 latency (the ring alone holds too few bytes in
        // flight to cover HBM latency at the SM's share of the bandwidth).
        if (p.l2_ahead) {  // step 0: steps 1..ahead; later: the new edge j + ahead
          const uint32_t hi = min(Kc - 1, j + p.l2_ahead);
          for (uint32_t ja = j == 0 ? 1u : j + p.l2_ahead; ja <= hi; ++ja) {
            wait_desc(ja);  // fetched ahead by sequencer 2 (ahead < kDescSlots)
            const StageGeo ga = r ? stage2_geo(desc_of(ja), cta_of(ja)) : stage1_geo(desc_of(ja), cta_of(ja));
            if (ga.nsec) l2_prefetch(desc_of(ja).bits + ga.src_off, ga.rtn * cum_bytes(ga, ga.nsec));
          }
        }
        uint64_t src = g.src_off;
        // waves of whole row tiles (tile-major, row-complete items), contiguous
        const uint32_t utot = cum_bytes(g, g.nsec);
        const uint32_t GWr = r ? (kConsumerWarps - kW1) / p.wave_div2 : kW1 / p.wave_div;
        const uint32_t nit = g.nsec ? g.rtn : 0u;
        for (uint32_t i0 = 0; i0 < nit; i0 += GWr) {
          const uint32_t sb = min(GWr, nit - i0) * utot;
          const uint64_t start = ring_place(pos, sb, RB);
          // wait for the slot and for every older chunk this range overwrites: chunks
          // are placed monotonically, so [start, pos) reaches older chunk c's bytes
          // in the ring exactly when pos > start_c + RB
          while (rel < chunk && (chunk - rel >= (uint32_t)kPassSlots ||
                                 starts[rel % kPassSlots] + RB < pos)) {
            mbar_wait_wd(&emptyr[rel % kPassSlots], (rel / kPassSlots) & 1, sus);
            ++rel;
          }
          const uint32_t slot = chunk % kPassSlots;
          starts[slot] = start;
          const uint32_t roff = (uint32_t)(start % RB);
          recs[slot] = ChunkRec{roff, i0};
          if (p.debug & 32u) {  // experiment: no copy, the consumers compute on stale bytes
            tc::mbar_arrive(&fullr[slot]);
          } else {
            tc::mbar_arrive_expect_tx(&fullr[slot], sb);
            tc::bulk_g2s(ring + roff, D.bits + src, sb, &fullr[slot]);
          }
          src += sb;
          ++chunk;
        }
        if (kTrace) PSTAMP(k, r ? 15 : 6);
        tc::mbar_arrive(&dempty[j % kDescSlots]);
      }
      return;
    }
    if (role == 1 || role == 2) {
      // ------------------------------------------------------ x quantisers
      // Per step: the bound, then a = s2 * x (packed.cpp:160) of the CTA's
      // stage-1 input slice as 38-bit fixed-point B fragments; the two warps
      // take alternate quads and each adds its sum of the values to the header.
      const int pw = role - 1;
      if (pw == 0) {  // this CTA's share of the other parity's bound words (used by
                      // the previous launch, which has completed)
        unsigned* other = p.amax + (size_t)(par ^ 1) * p.amax_words * 4;
        const uint32_t per = (p.amax_words + G - 1) / G;
        const uint32_t lo = min(p.amax_words, per * blockIdx.x), hi = min(p.amax_words, lo + per);
        for (uint32_t i = lo + lane; i < hi; i += 32) other[4 * i] = 0u;
      }
      bool pre_done = p.has_pre == 0;
      int32_t ywaited = -1;
      for (uint32_t j = 0; j < Kc; ++j) {
        const uint32_t slot = j % NB;
        if (j >= NB) mbar_wait_wd(&bempty1[slot], ((j / NB) - 1) & 1, sus);
        wait_desc(j);
        const StepDesc& D = desc_of(j);
        const Cta& C = cta_of(j);
        if (lane == 0) {
          if (D.x_src >= 0 && D.x_src > ywaited) {
            poll_ctr(ybar + (size_t)D.x_src * kCtrStride, target);
            ywaited = D.x_src;
          }
          if ((D.flags & kStepXPre) && !pre_done) {
            poll_ctr(xinit, target_all);
            pre_done = true;
          }
        }
        __syncwarp();
        const bool f32 = D.flags & kStepXF32, vec = (D.flags & kStepXVec) != 0;
        uint32_t mb;
        if (D.flags & kStepXSelf) {  // whole-input bound, read after the dependency
          mb = absmax_bits(D.x, 0, D.m, f32, vec, lane, 32);
#pragma unroll
          for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(~0u, mb, o));
        } else {
          mb = __ldcg(amax + 4 * (size_t)D.amax_idx);
        }
        const float xmax = bound_value(mb, f32);
        const StageGeo g = stage1_geo(D, C);
        uint8_t* bs = bslots1 + slot * p.bslot1_bytes;
        long long vsum = 0;
        if (g.nsec && !(p.debug & 2u)) {
          const Seg& S = D.seg[C.s1_seg];
          const int ea = act_exponent(S.s2max, xmax);
          const bool nonfinite = is_inf(xmax);
          const uint32_t klo = g.klo, nquad = g.prefix / 8, m = D.m;
          uint8_t* bf = bs + kBSlotHead;
#pragma unroll 2
          for (uint32_t qd = pw * 32 + lane; qd < nquad; qd += 64) {
            const uint32_t k0 = klo + 4 * qd;
            const XQuad xq = load_xquad(D.x, f32, vec, S.s2h, k0, m);
            long long v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = nonfinite ? 0.f : xq.s[e] * xq.x[e];
              v[e] = __float2ll_rn(scale_pow2(a, kFix - ea));
              vsum += v[e];
            }
            emit_quad(bf, klo, k0, q_of(k0, m), v);
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) vsum += __shfl_xor_sync(~0u, vsum, o);
        if (lane == 0) {
          ((long long*)bs)[pw] = vsum;
          if (pw == 0) xmaxs[j % 16] = xmax;
        }
        __syncwarp();
        if (lane == 0) {
          if (kTrace && pw == 0) PSTAMP(D.idx, 5);
          tc::mbar_arrive(&bfull1[slot]);
          tc::mbar_arrive(&dempty[j % kDescSlots]);
        }
      }
      return;
    }
    if (role == 3 || role == 4) {
      // ------------------------------------------------------ t quantisers
      // Per step: poll the t barrier, then the exact int64 t rows of the CTA's
      // stage-2 segment -> 38-bit fixed-point B fragments (+ sum), and the
      // segment's s1 slice; clear this CTA's share of the other parity's t.
      const int pw = role - 3;
      int32_t ywaited = -1;
      for (uint32_t j = 0; j < Kc; ++j) {
        const uint32_t slot = j % NB;
        if (j >= NB) mbar_wait_wd(&bempty2[slot], ((j / NB) - 1) & 1, sus);
        wait_desc(j);
        const StepDesc& D = desc_of(j);
        const Cta& C = cta_of(j);
        const uint32_t k = D.idx;
        if (kTrace && lane == 0 && pw == 0) PSTAMP(k, 12);
        if (lane == 0) {
          if (C.s2_rtn) poll_ctr(tbar + (size_t)k * kCtrStride, target);
          // an earlier step writing an overlapping output must be done everywhere
          if (D.y_src >= 0 && D.y_src > ywaited) {
            poll_ctr(ybar + (size_t)D.y_src * kCtrStride, target);
            ywaited = D.y_src;
          }
          if (kTrace && pw == 0) PSTAMP(k, 4);
        }
        __syncwarp();
        uint8_t* bs = bslots2 + slot * p.bslot2_bytes;
        long long vsum = 0;
        if (C.s2_rtn && !(p.debug & 2u)) {
          const Seg& S = D.seg[C.s2_seg];
          const long long* T = arena + D.t_off + S.t_off;
          const int sh = t_shift(D.m);
          const uint32_t nquad2 = kpad(S.r) / 4, r = S.r;
          uint8_t* bf = bs + kBSlotHead;
#pragma unroll 2
          for (uint32_t qd = pw * 32 + lane; qd < nquad2; qd += 64) {
            long long v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t kk = 4 * qd + e;
              const long long t = kk < r ? __ldcg(T + kk) : 0;
              v[e] = (t + (1ll << (sh - 1))) >> sh;
              vsum += v[e];
            }
            emit_quad(bf, 0, 4 * qd, q_of(4 * qd, r), v);
          }
          const uint4* s1src = (const uint4*)(S.s1h + (size_t)C.s2_rt0 * 16);
          uint4* s1dst = (uint4*)(bs + p.bs2_s1_off);
          for (uint32_t i = pw * 32 + lane; i < 2u * C.s2_rtn; i += 64) s1dst[i] = __ldg(s1src + i);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) vsum += __shfl_xor_sync(~0u, vsum, o);
        if (lane == 0) ((long long*)bs)[pw] = vsum;
        __syncwarp();
        if (lane == 0) {
          if (kTrace && pw == 0) PSTAMP(k, 13);
          tc::mbar_arrive(&bfull2[slot]);
        }
        {  // clear this CTA's share of the step's region in the other parity
          long long* Z = p.arena + (size_t)(par ^ 1) * p.arena_len + D.t_off;
          const uint32_t pairs = D.t_len / 2, per = (pairs + P - 1) / P;
          const uint32_t lo = min(pairs, per * prank), hi = min(pairs, lo + per);
          for (uint32_t i = lo + pw * 32 + lane; i < hi; i += 64)
            ((longlong2*)Z)[i] = make_longlong2(0, 0);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&dempty[j % kDescSlots]);
      }
      // every CTA has read the generation (it arrived on the kernel-start barrier
      // after reading it): advance it for the next launch
      if (blockIdx.x == 0 && pw == 0 && lane == 0) {
        poll_ctr(xinit, target_all);
        p.ctr[0] = target_all / G;
      }
      return;
    }
    if (lane != 0) return;
    if (role == 5) {
      // ------------------------------------------- sequencer 1: t barriers
      // step indices from the partition's list (not the descriptor slot, which
      // the stage-2 group may release as soon as stage 1 of the step is done)
      const uint32_t* list = Kc ? p.list + p.list_off[sub] : nullptr;
      uint32_t knext = Kc ? __ldg(list) : 0u;
      for (uint32_t j = 0; j < Kc; ++j) {
        const uint32_t k = knext;
        if (j + 1 < Kc) knext = __ldg(list + j + 1);
        mbar_wait_wd(&cdone1[j % kDoneRing], (j / kDoneRing) & 1, sus);
        arrive_ctr(tbar + (size_t)k * kCtrStride);  // stage-1 t reds ordered before it
      }
      return;
    }
    // --------------------- sequencer 2: output barriers, descriptor prefetch
    const uint32_t* list = Kc ? p.list + p.list_off[sub] : nullptr;
    auto issue_desc = [&](uint32_t j) {
      const uint32_t slot = j % kDescSlots, k = __ldg(list + j);
      uint8_t* dst = dslots + slot * kDescSlotBytes;
      tc::mbar_arrive_expect_tx(&dfull[slot], (uint32_t)sizeof(StepDesc) + 32);
      tc::bulk_g2s(dst, p.desc + k, (uint32_t)sizeof(StepDesc), &dfull[slot]);
      tc::bulk_g2s(dst + 480, p.ctas + (size_t)k * G + blockIdx.x, 32, &dfull[slot]);
    };
    for (uint32_t j = 0; j < min(Kc, (uint32_t)kDescSlots); ++j) issue_desc(j);
    for (uint32_t j = 0; j < Kc; ++j) {
      wait_desc(j);
      const StepDesc& D = desc_of(j);
      const bool publish = D.flags & kStepPublish;
      const uint32_t k = D.idx;
      mbar_wait_wd(&cdone2[j % kDoneRing], (j / kDoneRing) & 1, sus);
      if (publish) arrive_ctr(ybar + (size_t)k * kCtrStride);
      if (j + kDescSlots < Kc) {
        mbar_wait_wd(&dempty[j % kDescSlots], (j / kDescSlots) & 1, sus);
        issue_desc(j + kDescSlots);
      }
    }
    return;
  }

  // ================================================================ consumers
  // the consumer warps split into a stage-1 group (warps1) and a stage-2 group,
  // sized by the host in proportion to the two stages' bytes (pass_build)
  constexpr int W1 = kW1;
  const int gid = warp < W1 ? 0 : 1;  // 0: stage-1 group, 1: stage-2 group
  const int GW = gid ? kConsumerWarps - W1 : W1;  // warps in this group
  const uint32_t GT = 32u * GW;                   // threads in this group
  const int gt = tid - gid * 32 * W1;
  // ---- |x| prepass: this CTA's share of every independent input, one grid barrier
  if (p.has_pre) {
    for (uint32_t k = tid; k < K; k += kConsumerThreads) {
      const StepDesc* Dg = p.desc + k;
      const uint32_t fl = __ldg(&Dg->flags);
      if (!(fl & kStepXPre)) continue;
      const uint32_t m = __ldg(&Dg->m);
      const void* x = (const void*)__ldg((const unsigned long long*)&Dg->x);
      uint32_t lo, hi;
      share_of(m, blockIdx.x, G, lo, hi);
      if (lo < hi) {
        const uint32_t mb = absmax_bits(x, lo, hi, fl & kStepXF32, (fl & kStepXVec) != 0, 0, 1);
        atomicMax(amax + 4 * (size_t)__ldg(&Dg->amax_idx), mb);
      }
    }
  }
  // kernel-start barrier (every CTA, after it read the generation): the
  // prepass bounds, and the generation advance at the end of CTA 0
  all_consumers_sync();
  if (tid == 0) arrive_ctr(xinit);
  uint32_t chunk = 0;  // the group's ring chunks (work items) consumed so far
  const int gw = warp - gid * W1;
  uint64_t* const fullr = gid ? full2 : full1;
  uint64_t* const emptyr = gid ? empty2 : empty1;
  const ChunkRec* const recs = gid ? recs2 : recs1;
  const uint8_t* const ring = gid ? ring2 : ring1;
  uint32_t cur_step = 0;
  // Row-complete work items: an item is one row tile of the stage over all of
  // the CTA's slabs (tile-major layout), so the warp that runs it holds the
  // tile's complete row sums (packed.cpp:174-190): stage 1 publishes its t rows
  // with int64 reds, stage 2 writes its outputs; no shared row sums, no
  // group-wide epilogue after the MMAs.  A ring chunk is a wave of W = GW /
  // wave_div consecutive tiles (one contiguous copy); tile i is run by warp
  // i % GW, so W dividing GW puts each warp's tiles at the same place of their
  // waves, and in the last wave the positions past the tiles still release.
  auto rc_stage = [&](const StageGeo& g, const StepDesc& D, const Cta& C, uint32_t j, long long A,
                      const uint8_t* bs) {
    const uint32_t nitems = g.nsec ? g.rtn : 0u;
    if (!nitems) return;
    const uint32_t utot = cum_bytes(g, g.nsec);
    const Seg& S = D.seg[gid ? C.s2_seg : C.s1_seg];
    // stage 1: the tile's t rows are published with exact int64 reds
    long long* Tseg = arena + D.t_off + S.t_off + (size_t)C.s1_rt0 * 16;
    const float xmax = xmaxs[j % 16];
    const int ea = act_exponent(S.s2max, xmax);
    const bool nonfinite = is_inf(xmax);
    const int E = t_shift(D.m) + ea - kFix;  // t = T2 * 2^sh * 2^(ea - kFix)
    const double scale = __longlong_as_double((long long)(1023 + E) << 52);
    const bool yf32 = D.flags & kStepYF32;
    const __half* sc1 = (const __half*)(bs + p.bs2_s1_off);
    void* Y = D.y[C.s2_seg];
    const uint8_t* bf = bs + kBSlotHead;
    const uint32_t W = (uint32_t)GW / (gid ? p.wave_div2 : p.wave_div), nwav = (nitems + W - 1) / W;
    uint32_t F, rem;
    slab_split(g.K, F, rem);
    const uint32_t nfull = F > g.slab0 ? min(F - g.slab0, g.nsec) : 0u;
    const uint32_t gq = lane >> 2, cq = lane & 3;
    uint32_t ymb = 0;
    for (uint32_t i = gw; i < nwav * W; i += GW) {
      const uint32_t cidx = chunk + i / W, slot = cidx % kPassSlots;
      mbar_wait_wd(&fullr[slot], (cidx / kPassSlots) & 1, sus);
      if (i < nitems && !(p.debug & 1u)) {
        int acc[2][4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[0][q][0] = acc[0][q][1] = acc[0][q][2] = acc[0][q][3] = 0;
        const uint8_t* unit = ring + recs[slot].off + (i % W) * utot;
        if (nfull) {
          const uint8_t* bp = bf + kBytesPerK * (256 * g.slab0 - g.klo) + (gq * 4 + cq) * 16;
          full_run<1>(unit, 512u, bp, nfull, lane, gq < (uint32_t)kLimbs, acc);
          unit += 512u * nfull;
        }
        for (uint32_t s = nfull; s < g.nsec; ++s) {  // the 128 / 64 tails
          uint2 bv[8];
          const Slab sl = slab_of(g.K, g.slab0 + s);
          load_b(bf, g.klo, sl, gq, cq, bv);
          tiles_mma<1>(unit, unit_bytes(sl.nq), sl.nq, lane, bv, acc);
          unit += unit_bytes(sl.nq);
        }
        // row sums: lane c holds limbs 2c, 2c+1 of rows g, g+8; combine the quad
        unsigned long long v0 = 0, v1 = 0;
        if (cq < (kLimbs + 1) / 2) {
          int sm[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) sm[e] = acc[0][0][e] + acc[0][1][e] + acc[0][2][e] + acc[0][3][e];
          v0 = ((unsigned long long)(long long)sm[0] << (16 * cq)) +
               ((unsigned long long)(long long)sm[1] << (16 * cq + 8));
          v1 = ((unsigned long long)(long long)sm[2] << (16 * cq)) +
               ((unsigned long long)(long long)sm[3] << (16 * cq + 8));
        }
        v0 += __shfl_xor_sync(~0u, v0, 1);
        v1 += __shfl_xor_sync(~0u, v1, 1);
        v0 += __shfl_xor_sync(~0u, v0, 2);
        v1 += __shfl_xor_sync(~0u, v1, 2);
        if (cq < 2 && !(p.debug & 8u) && gid == 0) {
          const uint32_t rl = i * 16 + gq + 8 * cq;
          red_add_u64(&Tseg[rl], 2 * ((long long)(cq ? v1 : v0) >> 7) - A);
        } else if (cq < 2 && !(p.debug & 8u)) {
          const uint32_t rl = i * 16 + gq + 8 * cq, row = C.s2_rt0 * 16 + rl;
          if (row < S.n) {
            const long long Yi = 2 * ((long long)(cq ? v1 : v0) >> 7) - A;
            double y = (double)__half2float(sc1[rl]) * ((double)Yi * scale);  // packed.cpp:189
            if (nonfinite) y = __longlong_as_double(0x7ff8000000000000ll);
            if (yf32) {
              const float yo = (float)y;
              ((float*)Y)[row] = yo;
              const uint32_t b = __float_as_uint(yo) & 0x7FFFFFFFu;
              ymb = max(ymb, b >= 0x7F800000u ? 0x7F800000u : b);
            } else {
              const __half h = __float2half_rn((float)y);
              ((__half*)Y)[row] = h;
              ymb = max(ymb, (uint32_t)(__half_as_ushort(h) & 0x7FFFu));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&emptyr[slot]);
    }
    chunk += nwav;
    if (gid && (D.flags & kStepPublish)) {
#pragma unroll
      for (int o = 16; o; o >>= 1) ymb = max(ymb, __shfl_xor_sync(~0u, ymb, o));
      if (lane == 0 && ymb) atomicMax(amax + 4 * ((size_t)K + (size_t)D.idx * kMaxSeg + C.s2_seg), ymb);
    }
  };

  // Both groups run the same loop (one copy of the MMA code in the kernel):
  // group 0 does stage 1 of step k (x -> t), group 1 stage 2 (t -> y).
  for (uint32_t j = 0; j < Kc; ++j) {
    wait_desc(j);
    const StepDesc& D = desc_of(j);
    const Cta& C = cta_of(j);
    const uint32_t k = D.idx;
    const uint32_t slot = j % NB;
    mbar_wait_wd(gid ? &bfull2[slot] : &bfull1[slot], (j / NB) & 1, sus);
    const uint8_t* bs = gid ? bslots2 + slot * p.bslot2_bytes : bslots1 + slot * p.bslot1_bytes;
    if (kTrace && gt == 0) {
      PSTAMP(k, gid ? 2 : 0);
      PSTAMP(k, gid ? 9 : 7);
    }
    const StageGeo g = gid ? stage2_geo(D, C) : stage1_geo(D, C);
    const long long A = ((const long long*)bs)[0] + ((const long long*)bs)[1];
    cur_step = k;
    rc_stage(g, D, C, j, A, bs);
    if (kTrace && gt == 0) PSTAMP(k, gid ? 10 : 8);
    group_sync(gid, GT);  // reds / outputs happen-before the sequencer's release
    if (gt == 0) {
      if (kTrace) PSTAMP(k, gid ? 3 : 1);
      if (gid) {
        tc::mbar_arrive(&bempty2[slot]);
        tc::mbar_arrive(&cdone2[j % kDoneRing]);
        // the stage-1 group also reads this descriptor slot; a CTA without stage-2
        // rows in the step does not wait for the t barrier, so wait for it here
        mbar_wait_wd(&cdone1[j % kDoneRing], (j / kDoneRing) & 1, sus);
        tc::mbar_arrive(&dempty[j % kDescSlots]);
      } else {
        tc::mbar_arrive(&bempty1[slot]);
        tc::mbar_arrive(&cdone1[j % kDoneRing]);
      }
    }
  }
  if (kTrace && tid == 0) trp[kPassStamps * K + 1] = globaltimer();
}

}  // namespace dec

using namespace dec;

namespace {
uint32_t env_u32p(const char* name, uint32_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return (uint32_t)std::strtoul(v, nullptr, 10);
}
bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bn && y < x + an;
}
}  // namespace

namespace {

// Geometry of a pass over a given set of plans (one per step), and the
// shared-memory split it needs.
struct PassGeo {
  uint32_t bf1 = 0, bf2 = 0, s1bytes = 16;
  double bits1 = 0, bits2 = 0;
  uint64_t max_s2_cta_bytes = 0;
  uint32_t bslot1_b = 0, bs2_s1_off = 0, bslot2_b = 0, fixed = 0;
  uint32_t min1 = 0, min2 = 0;  // smallest rings
  uint32_t utot1 = 0, utot2 = 0;  // bytes of one row tile over a stage's slabs (largest)
  uint32_t div1 = 1, div2 = 1;    // wave divisors
  bool fits = false;
};

PassGeo pass_geo(uint32_t K, const std::vector<const nqb_group*>& plan) {
  PassGeo q;
  for (uint32_t k = 0; k < K; ++k) {
    const nqb_group* g = plan[k];
    for (uint32_t s = 0; s < g->nseg; ++s) {
      q.bf2 = std::max(q.bf2, kBytesPerK * kpad(g->r[s]));
      q.bits1 += (double)g->r[s] * g->m;
      q.bits2 += (double)g->r[s] * g->n[s];
    }
    for (uint32_t c = 0; c < g->grid; ++c) {
      const Cta& C = g->ctas[c];
      if (C.s1_rtn && C.s1_sln) {  // the CTA's stage-1 input slice and sections
        const Slab last = slab_of(g->m, C.s1_sl0 + C.s1_sln - 1);
        const uint32_t nk1 = last.k0 + 32 * last.nq - slab_of(g->m, C.s1_sl0).k0;
        q.bf1 = std::max(q.bf1, kBytesPerK * nk1);
        q.utot1 = std::max(q.utot1, 2u * nk1);  // one row tile over the CTA's slabs
      }
      if (C.s2_rtn) {
        uint64_t b2 = 0;
        const uint32_t r2 = g->seg[C.s2_seg].r;
        uint32_t tb = 0;
        for (uint32_t i = 0, ns = nslabs(r2); i < ns; ++i) tb += unit_bytes(slab_of(r2, i).nq);
        q.utot2 = std::max(q.utot2, tb);
        for (uint32_t i = 0, ns = nslabs(r2); i < ns; ++i)
          b2 += (uint64_t)C.s2_rtn * unit_bytes(slab_of(r2, i).nq);
        q.max_s2_cta_bytes = std::max<uint64_t>(q.max_s2_cta_bytes, b2);
      }
      q.s1bytes = std::max<uint32_t>(q.s1bytes, 32u * C.s2_rtn);
    }
  }
  // Shared memory: head | quantised-x slots | quantised-t slots | stage-1 ring |
  // stage-2 ring.
  q.bslot1_b = (kBSlotHead + std::max(q.bf1, 16u) + 127) / 128 * 128;
  q.bs2_s1_off = (kBSlotHead + std::max(q.bf2, 16u) + 127) / 128 * 128;
  q.bslot2_b = (q.bs2_s1_off + q.s1bytes + 127) / 128 * 128;
  q.fixed = pass_head_bytes() + kBSlots * (q.bslot1_b + q.bslot2_b);
  // a ring chunk is a wave of whole row tiles, one per warp of the group (<= 6
  // for stage 1, <= 8 for stage 2), halved when that passes 40 KB; each ring
  // holds at least one
  q.div1 = 6u * q.utot1 > 40u * 1024u ? 2u : 1u;
  q.div2 = 8u * q.utot2 > 40u * 1024u ? 2u : 1u;
  q.min1 = std::max<uint32_t>(24u * 1024u, 6u / q.div1 * q.utot1);
  q.min2 = std::max<uint32_t>(24u * 1024u, 8u / q.div2 * q.utot2);
  q.fits = q.fixed + q.min1 + q.min2 <= 227u * 1024u;
  return q;
}

}  // namespace

nqb_pass* pass_build(nqb_context* ctx, uint32_t K, const PassStepIn* steps) {
  NQB_REQUIRE(K >= 1 && K <= 65536, NQB_E_VALIDATION, "a decode pass holds 1..65536 steps");
  NQB_REQUIRE(steps != nullptr, NQB_E_VALIDATION, "null steps");
  const uint32_t G = (uint32_t)ctx->num_sms;
  std::vector<StepDesc> desc(K);
  bool has_pre = false, chained = false;
  // ---- dependencies from buffer ranges (geometry only: any plan of the group) ----
  for (uint32_t k = 0; k < K; ++k) {
    const PassStepIn& s = steps[k];
    const nqb_group* g = s.group;
    NQB_REQUIRE(g != nullptr, NQB_E_VALIDATION, "pass step without a decode group");
    NQB_REQUIRE(g->device == ctx->device, NQB_E_VALIDATION, "decode group lives on another device");
    NQB_REQUIRE(g->grid <= G, NQB_E_VALIDATION,
                "decode group planned for more SMs than the context's budget");
    NQB_REQUIRE(s.x != nullptr, NQB_E_VALIDATION, "null pass input");
    StepDesc& D = desc[k];
    std::memset(&D, 0, sizeof(D));
    D.idx = k;
    D.x = s.x;
    D.nseg = g->nseg;
    D.m = g->m;
    const uint32_t esz = s.f32 ? 4 : 2;
    D.flags = (s.f32 ? (kStepXF32 | kStepYF32) : 0u) |
              (((uintptr_t)s.x % 16 == 0) ? kStepXVec : 0u);
    for (uint32_t q = 0; q < g->nseg; ++q) {
      NQB_REQUIRE(s.y[q] != nullptr, NQB_E_VALIDATION, "null pass output");
      D.seg[q] = g->seg[q];
      D.y[q] = s.y[q];
      NQB_REQUIRE(!overlaps(s.y[q], (size_t)g->n[q] * esz, s.x, (size_t)g->m * esz),
                  NQB_E_VALIDATION, "a pass step's output overlaps its own input");
    }
    // the latest earlier step whose output overlaps this input must have finished
    // (output barrier) before stage 1
    D.x_src = -1;
    int32_t exact = -1;
    for (int j = (int)k - 1; j >= 0 && D.x_src < 0; --j) {
      const uint32_t ej = (desc[j].flags & kStepYF32) ? 4 : 2;
      for (uint32_t q = 0; q < desc[j].nseg; ++q) {
        if (!overlaps(desc[j].y[q], (size_t)desc[j].seg[q].n * ej, s.x, (size_t)g->m * esz))
          continue;
        D.x_src = j;
        if (desc[j].y[q] == s.x && desc[j].seg[q].n == g->m && ej == esz)
          exact = (int32_t)(K + j * kMaxSeg + q);
      }
    }
    // an earlier step whose output overlaps this step's output: the stage-2 group
    // runs step after step, but across CTAs only that step's output barrier
    // orders the two writes
    D.y_src = -1;
    for (int j = (int)k - 1; j >= 0 && D.y_src < 0; --j) {
      const uint32_t ej = (desc[j].flags & kStepYF32) ? 4 : 2;
      for (uint32_t a = 0; a < desc[j].nseg && D.y_src < 0; ++a)
        for (uint32_t b = 0; b < g->nseg && D.y_src < 0; ++b)
          if (overlaps(desc[j].y[a], (size_t)desc[j].seg[a].n * ej, s.y[b], (size_t)g->n[b] * esz))
            D.y_src = j;
    }
    if (D.y_src >= 0) {
      desc[D.y_src].flags |= kStepPublish;
      chained = true;
    }
    if (D.x_src < 0) {
      D.flags |= kStepXPre;
      D.amax_idx = k;
      has_pre = true;
    } else {
      chained = true;
      desc[D.x_src].flags |= kStepPublish;
      if (exact >= 0) D.amax_idx = (uint32_t)exact;
      else D.flags |= kStepXSelf;
    }
  }

  // ---- SM partitions.  When no step reads or overwrites another step's output,
  // the steps are independent: the grid splits into nsub partitions of P CTAs
  // and each runs its share of the steps on plans built for P CTAs, so every CTA
  // sees nsub times the bytes per step and the per-step handoff chain (x
  // quantisation, t barrier, t quantisation) is amortised over that much more
  // work.  A chained pass keeps one partition of G CTAs (the steps run one after
  // the other).  The pass runs on its own plans (tile-major stream layout,
  // k_relayout; the groups' per-call plans stay untouched), one per distinct group.
  const std::vector<StepDesc> desc0 = desc;
  auto build_with = [&](uint32_t nsub, const std::vector<const nqb_group*>& plan, const PassGeo& geo,
                        std::vector<nqb_group*> owned) -> nqb_pass* {
    std::vector<StepDesc> desc = desc0;
    auto* P = new nqb_pass();
    P->device = ctx->device;
    P->K = K;
    P->G = G;
    P->owned = std::move(owned);
    try {
      const uint32_t Pn = G / nsub;
      NQB_REQUIRE(geo.fits, NQB_E_DIMENSION_MISMATCH,
                  "decode pass: staging buffers leave no room for the weight rings");

      // ---- per-step plan data, t regions, algorithmic bytes ----
      uint64_t arena = 0, stream_bytes = 0;
      double algo = 0;
      std::vector<uint64_t> load(nsub, 0);
      std::vector<std::vector<uint32_t>> lists(nsub);
      std::vector<uint32_t> part(K, 0);
      for (uint32_t k = 0; k < K; ++k) {
        const nqb_group* g = plan[k];
        NQB_REQUIRE(g->grid <= Pn, NQB_E_INTERNAL, "decode plan larger than its partition");
        StepDesc& D = desc[k];
        D.bits = g->bits;
        D.R1 = g->R1;
        const uint32_t esz = steps[k].f32 ? 4 : 2;
        for (uint32_t q = 0; q < g->nseg; ++q) {
          D.seg[q] = g->seg[q];
          algo += (double)g->r[q] * (g->n[q] + g->m) / 8.0 + 2.0 * (g->n[q] + g->m) + esz * g->n[q];
        }
        algo += (double)esz * g->m;
        stream_bytes += g->stream_bytes;
        D.t_off = arena;
        D.t_len = (g->R1 + 3) & ~1u;  // even, plus the odd-start overhang of a segment copy
        arena += D.t_len;
        // partition: the least-loaded one (steps stay in pass order inside it)
        uint32_t best = 0;
        for (uint32_t i = 1; i < nsub; ++i)
          if (load[i] < load[best]) best = i;
        load[best] += g->stream_bytes;
        lists[best].push_back(k);
        part[k] = best;
      }

      // Rings split what the staging leaves in proportion to the two stages' bytes.
      const uint32_t rings = (227u * 1024u - geo.fixed) / 256 * 256;
      const double f1 = geo.bits1 + geo.bits2 > 0 ? geo.bits1 / (geo.bits1 + geo.bits2) : 0.5;
      // NQB_PASS_RING1_PCT: stage-1 share of the rings in percent.  Default: the
      // stage-1 share of the bytes, at most 30 % (stage-1 waves are half the size of
      // stage-2 waves with the 4 + 8 split; 7B: 1700 vs 1668 GB/s)
      // Stage-1 consumer warps and wave size (decided here: they size the rings).
      // The split is 4 + 8 when the largest step puts more than 96 KB of stage-2
      // bits on a CTA (measured, 70B: 1495 vs 1234 GB/s), else 6 + 6; stage-1 waves
      // are halved when they pass 24 KB (7B, 8 KB tiles: 2059 vs 1967 GB/s with a
      // 40 % stage-1 ring share; 70B's 4 KB tiles keep whole waves)
      const uint32_t ew = env_u32p("NQB_PASS_WARPS1", 0);
      const uint32_t warps1 = ew == 3 || ew == 4 || ew == 6 ? ew
                              : geo.max_s2_cta_bytes > 96u * 1024u ? 4u : 6u;
      const uint32_t div1e = env_u32p("NQB_PASS_WAVE_DIV", warps1 * geo.utot1 > 24u * 1024u ? 2u : 1u);
      const uint32_t div1 = (div1e == 2 && warps1 % 2 == 0) ? 2u : 1u;
      const uint32_t r1pct = env_u32p("NQB_PASS_RING1_PCT", 0);
      const double share1 = r1pct ? r1pct / 100.0 : div1 == 2 ? 0.40 : std::min(f1, 0.30);
      uint32_t ring1 = (uint32_t)(rings * share1) / 128 * 128;
      ring1 = std::min(std::max(ring1, geo.min1), rings - geo.min2);
      const uint32_t ring2 = rings - ring1;

      // ---- device memory: descriptors | CTA tables | counters | bounds | arena | lists ----
      const uint32_t amax_words = K * (1 + kMaxSeg);
      const size_t desc_b = sizeof(StepDesc) * K;
      const size_t cta_b = sizeof(Cta) * (size_t)K * G;
      const size_t ctr_b = sizeof(unsigned long long) * kCtrStride * (2 + 2 * (size_t)K);
      const size_t amax_b = 2ull * amax_words * 16;
      const size_t arena_b = 2ull * arena * 8;
      const size_t list_b = sizeof(uint32_t) * K;
      NQB_CUDA(cudaMalloc(&P->dmem, desc_b + cta_b + ctr_b + amax_b + arena_b + list_b));
      char* base = (char*)P->dmem;
      StepDesc* d_desc = (StepDesc*)base;
      Cta* d_ctas = (Cta*)(base + desc_b);
      auto* d_ctr = (unsigned long long*)(base + desc_b + cta_b);
      auto* d_amax = (unsigned*)(base + desc_b + cta_b + ctr_b);
      auto* d_arena = (long long*)(base + desc_b + cta_b + ctr_b + amax_b);
      auto* d_list = (uint32_t*)(base + desc_b + cta_b + ctr_b + amax_b + arena_b);
      std::vector<Cta> ctas((size_t)K * G, Cta{});
      for (uint32_t k = 0; k < K; ++k) {
        const nqb_group* g = plan[k];
        std::copy(g->ctas, g->ctas + g->grid, ctas.begin() + (size_t)k * G + (size_t)part[k] * Pn);
        desc[k].ctas = d_ctas + (size_t)k * G;
      }
      std::vector<uint32_t> flat;
      PassParams& pp = P->params;
      pp.list_off[0] = 0;
      for (uint32_t i = 0; i < nsub; ++i) {
        flat.insert(flat.end(), lists[i].begin(), lists[i].end());
        pp.list_off[i + 1] = (uint32_t)flat.size();
      }
      NQB_CUDA(cudaMemsetAsync(d_ctr, 0, ctr_b + amax_b + arena_b, ctx->stream));
      NQB_CUDA(cudaMemcpyAsync(d_desc, desc.data(), desc_b, cudaMemcpyHostToDevice, ctx->stream));
      NQB_CUDA(cudaMemcpyAsync(d_ctas, ctas.data(), cta_b, cudaMemcpyHostToDevice, ctx->stream));
      NQB_CUDA(cudaMemcpyAsync(d_list, flat.data(), list_b, cudaMemcpyHostToDevice, ctx->stream));
      NQB_CUDA(cudaStreamSynchronize(ctx->stream));

      pp.desc = d_desc;
      pp.ctas = d_ctas;
      pp.K = K;
      pp.G = G;
      pp.list = d_list;
      pp.nsub = nsub;
      pp.P = Pn;
      pp.ctr = d_ctr;
      pp.amax = d_amax;
      pp.amax_words = amax_words;
      pp.arena = d_arena;
      pp.arena_len = arena;
      pp.has_pre = has_pre ? 1 : 0;
      pp.pre_units = 0;
      for (uint32_t k = 0; k < K; ++k)
        if (desc[k].flags & kStepXPre)
          pp.pre_units = std::max<uint32_t>(pp.pre_units, ((desc[k].m + 7) / 8 + G - 1) / G);
      pp.debug = env_u32p("NQB_PASS_DEBUG", 0);
      pp.bslot1_bytes = geo.bslot1_b;
      pp.bslot2_bytes = geo.bslot2_b;
      pp.bs2_s1_off = geo.bs2_s1_off;
      // Consumer warps per stage group.  Measured (tools/gpu_pass_ab.sh): an even
      // 6 + 6 split is best when every step is small (7B: 886 vs 841 GB/s for 4 + 8),
      // while a pass whose largest step puts > 96 KB of stage-2 bits on each CTA
      // (70B gate/up: 169 KB) is bound by the stage-2 group, and 4 + 8 gives
      // 1495 vs 1234 GB/s.
      {
        pp.warps1 = warps1;  // the kernel is instantiated for 3, 4 and 6
        pp.wave_div = div1;
        const uint32_t div2 = env_u32p("NQB_PASS_WAVE_DIV2", geo.div2);
        pp.wave_div2 = (div2 == 2 && (kConsumerWarps - pp.warps1) % 2 == 0) ? 2u : 1u;
      }
      pp.ring1_bytes = ring1;
      pp.ring2_bytes = ring2;
      // waves of GW / wave_div items (NQB_PASS_WAVE_DIV 1 or 2; 2 needs even groups)
      pp.l2_ahead = std::min<uint32_t>(env_u32p("NQB_PASS_L2_AHEAD", 0), kDescSlots - 4);
      P->smem_bytes = geo.fixed + rings;
      if (env_u32p("NQB_PASS_VERBOSE", 0))
        std::fprintf(stderr,
                     "nqb pass: K=%u G=%u partitions=%u x %u smem=%u bslots=%ux(%u+%u) "
                     "rings=%u+%u tile bytes=%u/%u waves=%u/%u warps1=%u\n",
                     K, G, nsub, Pn, P->smem_bytes, kBSlots, geo.bslot1_b, geo.bslot2_b, ring1, ring2,
                     geo.utot1, geo.utot2, pp.warps1 / pp.wave_div, (kConsumerWarps - pp.warps1) / pp.wave_div2,
                     pp.warps1);
      for (uint32_t k = 0; k < K; ++k) {
        const uint32_t esz = steps[k].f32 ? 4 : 2;
        P->x_dev.push_back(const_cast<void*>(steps[k].x));
        P->x_bytes.push_back((size_t)desc[k].m * esz);
        for (uint32_t q = 0; q < desc[k].nseg; ++q) {
          P->y_dev.push_back(steps[k].y[q]);
          P->y_bytes.push_back((size_t)desc[k].seg[q].n * esz);
        }
      }
      P->stream_bytes = stream_bytes;
      P->desc_host.assign((const uint8_t*)desc.data(), (const uint8_t*)(desc.data() + K));
      P->algo_bytes = (uint64_t)algo;
      for (auto fn : {k_decode_pass<false, 6>, k_decode_pass<true, 6>, k_decode_pass<false, 4>,
                      k_decode_pass<true, 4>, k_decode_pass<false, 3>, k_decode_pass<true, 3>})
        NQB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      227 * 1024));  // the ceiling: passes may be built concurrently
      int per_sm = 0;
      NQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_pass<false, 6>,
                                                             kPassThreads, P->smem_bytes));
      NQB_REQUIRE(per_sm >= 1, NQB_E_INTERNAL, "decode pass kernel does not fit an SM");
    } catch (...) {
      pass_free(P);
      throw;
    }
    return P;
  };

  // Candidate partition counts, largest first.  Which count is fastest depends on
  // how the plans and the rings come out (measured, same box: 7B 12 partitions
  // 1973 GB/s, 14: 1523, 16: 1650; 70B 5: 2472, 6: 2123, 8: 2163), so by default
  // (NQB_PASS_TUNE=1) the builder times each candidate that fits (three launches on
  // the context's stream, outputs overwritten by the caller's first launch) and
  // keeps the fastest; NQB_PASS_TUNE=0 takes the first that fits.
  const uint32_t want = chained ? 1u : std::min<uint32_t>(std::max<uint32_t>(env_u32p("NQB_PASS_SPLIT", kMaxSub), 1), kMaxSub);
  const bool tune = !chained && env_u32p("NQB_PASS_TUNE", 1) != 0;
  const bool verbose = env_u32p("NQB_PASS_VERBOSE", 0) != 0;
  static const uint32_t kCands[] = {16, 12, 8, 6, 5, 4, 3, 2, 1};
  nqb_pass* best = nullptr;
  float best_ms = 0.f;
  for (uint32_t ns : kCands) {
    if (ns > want) continue;
    if (best && !tune) break;
    const uint32_t Pc = G / ns;
    std::vector<nqb_group*> made;
    std::vector<const nqb_group*> pl(K);
    bool ok = Pc >= 8 || ns == 1;
    try {
      std::vector<std::pair<const nqb_group*, nqb_group*>> memo;
      for (uint32_t k = 0; k < K && ok; ++k) {
        const nqb_group* g = steps[k].group;
        nqb_group* h = nullptr;
        for (auto& pr : memo)
          if (pr.first == g) h = pr.second;
        if (!h) {
          // a chained pass runs one step at a time on the whole grid: shorter
          // stage-1 slab ranges give each CTA more row tiles, so more of its warps
          // work per step (measured, 7B chained: 4 slabs 261 GB/s, 16: 206)
          h = group_build(ctx, g->layers, g->nseg, Pc, kPassMaxRt, true, chained ? 4u : 0u);
          made.push_back(h);
          memo.push_back({g, h});
        }
        pl[k] = h;
      }
    } catch (const nqb::Failure& f) {
      ok = false;
      if (verbose) std::fprintf(stderr, "nqb pass: %u partitions: plan failed: %s\n", ns, f.msg.c_str());
    }
    PassGeo gq;
    if (ok) gq = pass_geo(K, pl);
    if (ok && !gq.fits && verbose)
      std::fprintf(stderr, "nqb pass: %u partitions: staging %u B + rings %u + %u B > 227 KB\n", ns,
                   gq.fixed, gq.min1, gq.min2);
    // more partitions amortise the per-step chain over more bytes per CTA, but
    // their larger blocks take shared memory from the weight rings: a partition
    // count must leave >= NQB_PASS_MIN_RINGS_KB (default 88) of rings
    const uint32_t rings_left = ok && gq.fits ? 227u * 1024u - gq.fixed : 0u;
    if (ok && gq.fits && ns > 1 && rings_left < env_u32p("NQB_PASS_MIN_RINGS_KB", 88) * 1024u) {
      if (verbose) std::fprintf(stderr, "nqb pass: %u partitions: rings %u B below the minimum\n", ns, rings_left);
      gq.fits = false;
    }
    if (!(ok && gq.fits)) {
      for (auto* h : made) group_free(h);
      continue;
    }
    nqb_pass* Pc_pass = build_with(ns, pl, gq, std::move(made));
    if (!tune) {
      best = Pc_pass;
      break;
    }
    float ms = 0.f;
    try {
      cudaEvent_t e0, e1;
      NQB_CUDA(cudaEventCreate(&e0));
      NQB_CUDA(cudaEventCreate(&e1));
      pass_launch(ctx, Pc_pass, nullptr);
      NQB_CUDA(cudaEventRecord(e0, ctx->stream));
      pass_launch(ctx, Pc_pass, nullptr);
      pass_launch(ctx, Pc_pass, nullptr);
      NQB_CUDA(cudaEventRecord(e1, ctx->stream));
      NQB_CUDA(cudaEventSynchronize(e1));
      NQB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    } catch (...) {
      pass_free(Pc_pass);
      if (best) pass_free(best);
      throw;
    }
    if (verbose) std::fprintf(stderr, "nqb pass: %u partitions: %.1f us per launch\n", ns, ms * 500.f);
    if (!best || ms < best_ms) {
      if (best) pass_free(best);
      best = Pc_pass;
      best_ms = ms;
    } else {
      pass_free(Pc_pass);
    }
  }
  NQB_REQUIRE(best != nullptr, NQB_E_DIMENSION_MISMATCH,
              "decode pass: no partition of the grid fits the steps' plans in shared memory");
  return best;
}

void pass_launch(nqb_context* ctx, const nqb_pass* P, unsigned long long* trace,
                 const void* desc_override) {
  NQB_REQUIRE(P->device == ctx->device, NQB_E_VALIDATION, "decode pass lives on another device");
  PassParams pp = P->params;
  if (desc_override) pp.desc = (const StepDesc*)desc_override;
  pp.trace = trace;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->G);
  cfg.blockDim = dim3(kPassThreads);
  cfg.dynamicSmemBytes = P->smem_bytes;
  cfg.stream = ctx->stream;
  // cooperative launch: the runtime guarantees every CTA is co-resident (the
  // in-kernel barriers need it) or fails the launch
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = env_u32p("NQB_PASS_COOP", 1) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool w4 = pp.warps1 == 4;
  const bool w3 = pp.warps1 == 3;
  if (trace)
    NQB_CUDA(cudaLaunchKernelEx(&cfg, w3 ? k_decode_pass<true, 3> : w4 ? k_decode_pass<true, 4> : k_decode_pass<true, 6>, pp));
  else
    NQB_CUDA(cudaLaunchKernelEx(&cfg, w3 ? k_decode_pass<false, 3> : w4 ? k_decode_pass<false, 4> : k_decode_pass<false, 6>, pp));
  NQB_LAUNCHED(ctx);
}

uint32_t pass_trace_words(const nqb_pass* P) { return P->G * (kPassStamps * P->K + 2); }

void pass_free(nqb_pass* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaFree(P->dmem);
  for (auto* g : P->owned) group_free(g);
  delete P;
}

}  // namespace nqb
