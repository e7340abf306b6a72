// decode_pass.cu — persistent multi-layer decode kernel (one launch per decode
// pass) and its host-side builder.  Design: decode_pass.cuh, DESIGN.md §4b.
//
// Arithmetic is the per-call kernel's (decode.cu, gemv_two_stage of
// packed.cpp:153-192 in exact integer IMMA form), so a layer's output is the
// same function of its input in both kernels; only the activation bound of a
// chained step comes from the producing step's published max|y| instead of a
// pass over x.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "decode_dev.cuh"
#include "decode_pass.cuh"

namespace nqb {
namespace dec {

__device__ __forceinline__ void wait_ctr(const unsigned long long* c, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long cur;
    const unsigned long long t0 = globaltimer();
    for (uint32_t it = 0;; ++it) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(cur) : "l"(c) : "memory");
      if (cur >= target) break;
      // watchdog: a barrier that does not complete within seconds means the
      // grid is not co-resident or diverged; fail the launch instead of hanging
      if ((it & 255u) == 255u && globaltimer() - t0 > 4000000000ull) __trap();
    }
  }
  consumers_sync();
}

__device__ __forceinline__ void arrive_ctr(unsigned long long* c) {
  consumers_sync();  // the CTA's prior global writes / reds happen-before the release
  if (threadIdx.x == 0)
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;\n" ::"l"(c) : "memory");
}

// Stage geometry of one CTA in one step.
struct StageGeo {
  uint32_t rtn, nsec, K, slab0, klo, kfirst;  // kfirst: k0 of section 0
  uint64_t src_off;                          // byte offset of section 0 in the step's bits
  uint32_t prefix, suffix;                   // staged scale bytes (stage 1: s2, stage 2: s1)
};

__device__ __forceinline__ StageGeo stage1_geo(const StepDesc& D, const Cta& C) {
  StageGeo g{};
  if (!C.s1_rtn || !C.s1_sln) return g;
  g.rtn = C.s1_rtn;
  g.nsec = C.s1_sln;
  g.K = D.m;
  g.slab0 = C.s1_sl0;
  g.klo = g.kfirst = slab_of(D.m, C.s1_sl0).k0;
  const Slab last = slab_of(D.m, C.s1_sl0 + C.s1_sln - 1);
  const uint32_t nk1 = last.k0 + 32 * last.nq - g.klo;
  g.src_off = C.stream_off;
  g.prefix = 2 * nk1;
  return g;
}

__device__ __forceinline__ StageGeo stage2_geo(const StepDesc& D, const Cta& C) {
  StageGeo g{};
  if (!C.s2_rtn) return g;
  const uint32_t r = D.seg[C.s2_seg].r;
  g.rtn = C.s2_rtn;
  g.nsec = nslabs(r);
  g.K = r;
  g.slab0 = 0;
  g.klo = g.kfirst = 0;
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

__device__ __forceinline__ uint32_t sec_width(const StageGeo& g, uint32_t s) {
  return 32u * slab_of(g.K, g.slab0 + s).nq;
}

// Sections [s0, *s1) of a chunk (at least one, at most `cap` bytes unless one
// section alone is larger); returns the chunk's section bytes.
__device__ __forceinline__ uint32_t chunk_span(const StageGeo& g, uint32_t s0, uint32_t cap,
                                               uint32_t* s1) {
  uint32_t s = s0, bytes = 0;
  do {
    bytes += 2u * g.rtn * sec_width(g, s);
    ++s;
  } while (s < g.nsec && bytes + 2u * g.rtn * sec_width(g, s) <= cap);
  *s1 = s;
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

// All (tile pair, section) work of one resident chunk, split over the consumer
// warps (the per-call kernel's linear-mode loop, decode.cu run_stage<true>);
// leaves the chunk's partial row sums added into red[].
__device__ __forceinline__ void run_chunk(const uint8_t* base, const StageGeo& g, uint32_t s0,
                                          uint32_t nsec, const uint8_t* bfrag, int* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gq = lane >> 2, c = lane & 3;
  int acc[2][4][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q][0] = acc[j][q][1] = acc[j][q][2] = acc[j][q][3] = 0;
  const uint32_t rtn = g.rtn;
  const uint32_t npair = (rtn + 1) / 2, U = npair * nsec;
  const uint32_t f0 = (uint32_t)((uint64_t)U * warp / kConsumerWarps);
  const uint32_t f1 = (uint32_t)((uint64_t)U * (warp + 1) / kConsumerWarps);
  if (f0 >= f1) return;
  uint32_t F, rem;
  slab_split(g.K, F, rem);
  const uint32_t sl_first = g.slab0 + s0;  // absolute slab of the chunk's first section
  const uint32_t k_first = slab_of(g.K, sl_first).k0;
  const uint32_t nfull = F > sl_first ? F - sl_first : 0;  // full slabs come first
  uint32_t cur = f0 / nsec;
  uint2 b[8];
  for (uint32_t f = f0; f < f1;) {
    const uint32_t pr = f / nsec;
    uint32_t s = f - pr * nsec;
    const uint32_t send = min(nsec, s + (f1 - f));
    f = pr * nsec + send;
    if (pr != cur) {
      flush_rows(acc[0], red + 2 * cur * 16 * kRedStride, lane);
      if (2 * cur + 1 < rtn) flush_rows(acc[1], red + (2 * cur + 1) * 16 * kRedStride, lane);
      cur = pr;
    }
    const uint32_t t0 = 2 * pr;
    const bool two = t0 + 1 < rtn;
    const uint32_t sf = min(send, nfull);
    if (s < sf) {
      const uint32_t k0 = 256 * (sl_first + s);
      const uint8_t* unit = base + 2u * rtn * (k0 - k_first) + t0 * 512;
      const uint8_t* bp = bfrag + kBytesPerK * (k0 - g.klo) + (gq * 4 + c) * 16;
      if (two) full_run<2>(unit, 512u * rtn, bp, sf - s, lane, gq < (uint32_t)kLimbs, acc);
      else full_run<1>(unit, 512u * rtn, bp, sf - s, lane, gq < (uint32_t)kLimbs, acc);
      s = sf;
    }
    for (; s < send; ++s) {  // the 128 / 64 tails
      const Slab sl = slab_of(g.K, sl_first + s);
      const uint32_t ub = unit_bytes(sl.nq);
      const uint8_t* unit = base + 2u * rtn * (sl.k0 - k_first) + t0 * ub;
      load_b(bfrag, g.klo, sl, gq, c, b);
      if (two) tiles_mma<2>(unit, ub, sl.nq, lane, b, acc);
      else tiles_mma<1>(unit, ub, sl.nq, lane, b, acc);
    }
  }
  flush_rows(acc[0], red + 2 * cur * 16 * kRedStride, lane);
  if (2 * cur + 1 < rtn) flush_rows(acc[1], red + (2 * cur + 1) * 16 * kRedStride, lane);
}

// Phase order shared by producer and consumers: S1(0), then per step k
// [S1(k+1) if lookahead] S2(k) [S1(k+1) otherwise].
template <typename S1, typename S2, typename DescOf>
__device__ __forceinline__ void for_each_phase(uint32_t K, DescOf desc_of, S1 s1, S2 s2) {
  s1(0u);
  uint32_t next1 = 1;
  for (uint32_t k = 0; k < K; ++k) {
    const bool la = (desc_of(k).flags & kStepLookahead) != 0;
    if (k + 1 < K && la && next1 == k + 1) s1(next1++);
    s2(k);
    if (k + 1 < K && next1 == k + 1) s1(next1++);
  }
}

template <bool kTrace>
__global__ void __launch_bounds__(kThreads, 1) k_decode_pass(const __grid_constant__ PassParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)smem;
  uint64_t* empty = full + kPassSlots;
  uint64_t* dfull = empty + kPassSlots;
  uint64_t* dempty = dfull + kDescSlots;
  uint8_t* dslots = (uint8_t*)(dempty + kDescSlots);
  long long* red8 = (long long*)(dslots + kDescSlots * kDescSlotBytes);
  float* xred = (float*)((uint8_t*)red8 + 256);
  unsigned long long* misc = (unsigned long long*)((uint8_t*)xred + 64);  // [0] launch target
  int* red = (int*)((uint8_t*)misc + 64);
  uint8_t* bfrag = smem + pass_head_bytes();
  uint8_t* ring = bfrag + p.bfrag_bytes;

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  const uint32_t K = p.K, RB = p.ring_bytes, cap = p.chunk_cap;
  auto desc_of = [&](uint32_t k) -> const StepDesc& {
    return *(const StepDesc*)(dslots + (k % kDescSlots) * kDescSlotBytes);
  };
  auto cta_of = [&](uint32_t k) -> const Cta& {
    return *(const Cta*)(dslots + (k % kDescSlots) * kDescSlotBytes + 480);
  };

  if (tid == 0) {
    for (int s = 0; s < kPassSlots; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < kDescSlots; ++s) {
      tc::mbar_init(&dfull[s], 1);
      tc::mbar_init(&dempty[s], kConsumerWarps);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------------ producer
  if (warp == kConsumerWarps) {
    uint64_t pos = 0;
    uint32_t chunk = 0, rel = 0;
    uint64_t ends[kPassSlots];
    auto load_desc = [&](uint32_t k) {
      const uint32_t slot = k % kDescSlots;
      if (k >= (uint32_t)kDescSlots) mbar_wait_wd(&dempty[slot], ((k / kDescSlots) - 1) & 1);
      uint8_t* dst = dslots + slot * kDescSlotBytes;
      const uint4* src = (const uint4*)(p.desc + k);
      if (lane < (int)(kDescBytes / 16)) ((uint4*)dst)[lane] = __ldg(src + lane);
      const StepDesc* Dg = p.desc + k;
      if (lane == 30 || lane == 31) {
        const uint4* cs = (const uint4*)(Dg->ctas + blockIdx.x);
        ((uint4*)(dst + 480))[lane - 30] = __ldg(cs + (lane - 30));
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dfull[slot]);
    };
    auto issue_stage = [&](uint32_t k, int stage) {
      const StepDesc& D = desc_of(k);
      const Cta& C = cta_of(k);
      const StageGeo g = stage == 1 ? stage1_geo(D, C) : stage2_geo(D, C);
      if (!g.nsec) return;
      uint32_t s0 = 0;
      uint64_t src = g.src_off;
      while (s0 < g.nsec) {
        uint32_t s1;
        const uint32_t sb = chunk_span(g, s0, cap, &s1);
        const uint32_t pre = s0 == 0 ? g.prefix : 0;
        const uint32_t suf = s1 == g.nsec ? g.suffix : 0;
        const uint32_t bytes = pre + sb + (suf + 127) / 128 * 128;
        const uint64_t start = ring_place(pos, bytes, RB);
        // wait for the slot and for every older chunk overlapping this range
        while (rel < chunk && (chunk - rel >= (uint32_t)kPassSlots || ends[rel % kPassSlots] + RB > pos)) {
          mbar_wait_wd(&empty[rel % kPassSlots], (rel / kPassSlots) & 1);
          ++rel;
        }
        ends[chunk % kPassSlots] = pos;
        if (lane == 0) {
          uint64_t* bar = &full[chunk % kPassSlots];
          uint8_t* dst = ring + (uint32_t)(start % RB);
          tc::mbar_arrive_expect_tx(bar, pre + sb + suf);
          if (pre) {
            const Seg& S = D.seg[C.s1_seg];
            tc::bulk_g2s(dst, S.s2h + g.klo, pre, bar);
          }
          tc::bulk_g2s(dst + pre, D.bits + src, sb, bar);
          if (suf) {
            const Seg& S = D.seg[C.s2_seg];
            tc::bulk_g2s(dst + pre + sb, S.s1h + (size_t)C.s2_rt0 * 16, suf, bar);
          }
        }
        __syncwarp();
        src += sb;
        s0 = s1;
        ++chunk;
      }
    };
    for_each_phase(
        K, desc_of,
        [&](uint32_t k) {
          load_desc(k);
          issue_stage(k, 1);
        },
        [&](uint32_t k) { issue_stage(k, 2); });
    return;
  }

  // ----------------------------------------------------------------- consumers
  for (int i = tid; i < kMaxRt * 16 * kRedStride / 4; i += kConsumerThreads)
    ((int4*)red)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    unsigned long long gen;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(gen) : "l"(p.ctr) : "memory");
    misc[0] = (gen + 1) * p.G;
  }
  unsigned long long* trp = nullptr;
  if (kTrace) {
    trp = p.trace + (size_t)blockIdx.x * (2 * K + 2);
    if (tid == 0) trp[0] = globaltimer();
  }
  consumers_sync();
  const unsigned long long target = misc[0];
  unsigned long long* tbar = p.ctr + 2 * kCtrStride;
  unsigned long long* ybar = tbar + (size_t)K * kCtrStride;

  uint64_t pos = 0;
  uint32_t chunk = 0;
  int32_t ywaited = -1;

  auto wait_chunk = [&](uint32_t bytes) -> const uint8_t* {
    const uint64_t start = ring_place(pos, bytes, RB);
    mbar_wait_wd(&full[chunk % kPassSlots], (chunk / kPassSlots) & 1);
    return ring + (uint32_t)(start % RB);
  };
  auto release_chunk = [&]() {
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&empty[chunk % kPassSlots]);
    ++chunk;
  };

  auto stage1 = [&](uint32_t k) {
    mbar_wait_wd(&dfull[k % kDescSlots], (k / kDescSlots) & 1);
    const StepDesc& D = desc_of(k);
    const Cta& C = cta_of(k);
    if (D.x_src >= 0 && D.x_src > ywaited) {
      wait_ctr(ybar + (size_t)D.x_src * kCtrStride, target);
      ywaited = D.x_src;
    }
    const StageGeo g = stage1_geo(D, C);
    if (g.nsec) {
      const bool xf32 = D.flags & kStepXF32, xvec = D.flags & kStepXVec;
      float xmax;
      if (D.xmax_src >= 0) xmax = __uint_as_float(__ldcg(p.ymax + D.xmax_src));
      else xmax = x_absmax(D.x, D.m, xf32, xvec, xred);
      const bool nonfinite = is_inf(xmax);
      const Seg& S = D.seg[C.s1_seg];
      const int ea = act_exponent(S.s2max, xmax);
      long long asum = 0, aabs = 0;
      uint32_t s0 = 0;
      while (s0 < g.nsec) {
        uint32_t s1;
        const uint32_t sb = chunk_span(g, s0, cap, &s1);
        const uint32_t pre = s0 == 0 ? g.prefix : 0;
        const uint8_t* base = wait_chunk(pre + sb);
        if (s0 == 0) {  // quantise this CTA's input slice (packed.cpp:160) into B fragments
          const uint32_t klo = g.klo, nquad = g.prefix / 8;
          const __half* s2s = (const __half*)base - klo;
          uint32_t qd = tid;
          XQuad cur = load_xquad(D.x, xf32, xvec, s2s, klo + 4 * min(qd, nquad - 1), D.m);
          while (qd < nquad) {
            const uint32_t nx = qd + kConsumerThreads;
            const XQuad nxt = load_xquad(D.x, xf32, xvec, s2s, klo + 4 * min(nx, nquad - 1), D.m);
            const uint32_t k0 = klo + 4 * qd;
            long long v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = nonfinite ? 0.f : cur.s[e] * cur.x[e];
              v[e] = __float2ll_rn(scale_pow2(a, kFix - ea));
              asum += v[e];
              aabs += v[e] < 0 ? -v[e] : v[e];
            }
            emit_quad(bfrag, klo, k0, q_of(k0, D.m), v);
            cur = nxt;
            qd = nx;
          }
          warp_partials2(asum, aabs, red8);
          consumers_sync();
        }
        run_chunk(base + pre, g, s0, s1 - s0, bfrag, red);
        release_chunk();
        s0 = s1;
      }
      consumers_sync();
      // publish: t rows (exact int64 reds), sum|a| and the exponent of this segment
      const long long A = sum_partials(red8);
      long long* R = p.arena + D.t_off;
      if (tid == 0 && C.s1_rt0 == 0) {
        red_add_u64(&R[D.R1 + C.s1_seg], sum_partials(red8 + kConsumerWarps));
        if (C.s1_sl0 == 0) {
          R[D.R1 + kMaxSeg + C.s1_seg] = ea;
          if (nonfinite) R[D.R1 + 2 * kMaxSeg] = 1;
        }
      }
      long long* Tseg = R + S.t_off + (size_t)C.s1_rt0 * 16;
      for (uint32_t i = tid; i < (uint32_t)C.s1_rtn * 16; i += kConsumerThreads) {
        const long long v = 2 * row_value(red + i * kRedStride) - A;
        int4* rr = (int4*)(red + i * kRedStride);
        rr[0] = make_int4(0, 0, 0, 0);
        rr[1] = make_int4(0, 0, 0, 0);
        red_add_u64(&Tseg[i], v);
      }
    }
    arrive_ctr(tbar + (size_t)k * kCtrStride);
  };

  auto stage2 = [&](uint32_t k) {
    const StepDesc& D = desc_of(k);
    const Cta& C = cta_of(k);
    wait_ctr(tbar + (size_t)k * kCtrStride, target);
    if (kTrace && tid == 0) trp[1 + 2 * k] = globaltimer();
    if (D.zero_len) {  // step k-2's region: every CTA finished its stage 2 before arriving here
      long long* Z = p.arena + D.zero_off;
      const uint32_t per = (D.zero_len + p.G - 1) / p.G;
      const uint32_t lo = min(D.zero_len, per * blockIdx.x), hi = min(D.zero_len, lo + per);
      for (uint32_t i = lo + tid; i < hi; i += kConsumerThreads) Z[i] = 0;
    }
    const StageGeo g = stage2_geo(D, C);
    const bool publish = D.flags & kStepPublish;
    float ymx = 0.f;
    if (g.nsec) {
      const Seg& S = D.seg[C.s2_seg];
      const long long* R = p.arena + D.t_off;
      const int ea = (int)__ldcg(&R[D.R1 + kMaxSeg + C.s2_seg]);
      const bool nonfinite = __ldcg(&R[D.R1 + 2 * kMaxSeg]) != 0;
      // |t_k| = |sum_j +-a_int_j| <= sum_j |a_int_j|, published exactly by stage 1
      const unsigned long long tbound = (unsigned long long)__ldcg(&R[D.R1 + C.s2_seg]);
      const int et = tbound ? 64 - __clzll((long long)tbound) : 0;
      const int sh = et - kFix;
      const long long* Tseg = R + S.t_off;
      const uint32_t nquad2 = kpad(S.r) / 4;
      long long tsum = 0;
      {
        uint32_t qd = tid;
        long long cur[4], nxt[4];
        load_tquad(Tseg, 4 * min(qd, nquad2 - 1), S.r, D.t_off + S.t_off, cur);
        while (qd < nquad2) {
          const uint32_t nx = qd + kConsumerThreads;
          load_tquad(Tseg, 4 * min(nx, nquad2 - 1), S.r, D.t_off + S.t_off, nxt);
          long long v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            v[e] = sh > 0 ? (cur[e] + (1ll << (sh - 1))) >> sh : cur[e] * (1ll << (-sh));
            tsum += v[e];
          }
          emit_quad(bfrag, 0, 4 * qd, q_of(4 * qd, S.r), v);
#pragma unroll
          for (int e = 0; e < 4; ++e) cur[e] = nxt[e];
          qd = nx;
        }
      }
      warp_partials2(tsum, 0, red8);
      consumers_sync();
      uint32_t s0 = 0;
      const __half* sc1 = nullptr;
      while (s0 < g.nsec) {
        uint32_t s1;
        const uint32_t sb = chunk_span(g, s0, cap, &s1);
        const bool last = s1 == g.nsec;
        const uint32_t suf = last ? (g.suffix + 127) / 128 * 128 : 0;
        const uint8_t* base = wait_chunk(sb + suf);
        run_chunk(base, g, s0, s1 - s0, bfrag, red);
        if (last) sc1 = (const __half*)(base + sb);  // released after the outputs
        else release_chunk();
        s0 = s1;
      }
      consumers_sync();
      const long long Tsum = sum_partials(red8);
      const int E = sh + ea - kFix;  // t = T2 * 2^sh * 2^(ea - kFix)
      const bool yf32 = D.flags & kStepYF32;
      void* Y = D.y[C.s2_seg];
      for (uint32_t i = tid; i < (uint32_t)C.s2_rtn * 16; i += kConsumerThreads) {
        const uint32_t row = C.s2_rt0 * 16 + i;
        int4* rr = (int4*)(red + i * kRedStride);
        if (row < S.n) {
          const long long Yi = 2 * row_value(red + i * kRedStride) - Tsum;
          double y = (double)__half2float(sc1[i]) *
                     ((double)Yi * __longlong_as_double((long long)(1023 + E) << 52));  // packed.cpp:189
          if (nonfinite) y = __longlong_as_double(0x7ff8000000000000ll);
          float yo;
          if (yf32) {
            yo = (float)y;
            ((float*)Y)[row] = yo;
          } else {
            const __half h = __float2half_rn((float)y);
            ((__half*)Y)[row] = h;
            yo = __half2float(h);
          }
          const float a = fabsf(yo);
          ymx = fmaxf(ymx, (a <= FLT_MAX) ? a : __int_as_float(0x7f800000));
        }
        rr[0] = make_int4(0, 0, 0, 0);
        rr[1] = make_int4(0, 0, 0, 0);
      }
      release_chunk();
      if (publish) {
#pragma unroll
        for (int o = 16; o; o >>= 1) ymx = fmaxf(ymx, __shfl_xor_sync(~0u, ymx, o));
        consumers_sync();
        if (lane == 0) xred[warp] = ymx;
        consumers_sync();
        if (tid == 0) {
          float mx = 0.f;
          for (int w = 0; w < kConsumerWarps; ++w) mx = fmaxf(mx, xred[w]);
          atomicMax(p.ymax + (size_t)k * kMaxSeg + C.s2_seg, __float_as_uint(mx));
        }
      }
    }
    if (kTrace && tid == 0) trp[2 + 2 * k] = globaltimer();
    if (publish) arrive_ctr(ybar + (size_t)k * kCtrStride);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&dempty[k % kDescSlots]);
  };

  for_each_phase(K, desc_of, stage1, stage2);

  // -------------------------------------------------------------- exit barrier
  arrive_ctr(p.ctr + kCtrStride);
  wait_ctr(p.ctr + kCtrStride, target);
  // every CTA is past every use: clear the last steps' regions and max|y| words
  for (uint32_t t = 0; t < p.ntail; ++t) {
    long long* Z = p.arena + p.tail_off[t];
    const uint32_t len = p.tail_len[t], per = (len + p.G - 1) / p.G;
    const uint32_t lo = min(len, per * blockIdx.x), hi = min(len, lo + per);
    for (uint32_t i = lo + tid; i < hi; i += kConsumerThreads) Z[i] = 0;
  }
  {
    const uint32_t len = K * kMaxSeg, per = (len + p.G - 1) / p.G;
    const uint32_t lo = min(len, per * blockIdx.x), hi = min(len, lo + per);
    for (uint32_t i = lo + tid; i < hi; i += kConsumerThreads) p.ymax[i] = 0u;
  }
  if (blockIdx.x == 0 && tid == 0) p.ctr[0] = target / p.G;  // next launch's generation
  if (kTrace && tid == 0) trp[2 * K + 1] = globaltimer();
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

nqb_pass* pass_build(nqb_context* ctx, uint32_t K, const PassStepIn* steps) {
  NQB_REQUIRE(K >= 1 && K <= 8192, NQB_E_VALIDATION, "a decode pass holds 1..8192 steps");
  NQB_REQUIRE(steps != nullptr, NQB_E_VALIDATION, "null steps");
  const uint32_t G = (uint32_t)ctx->num_sms;
  std::vector<StepDesc> desc(K);
  uint32_t bfrag = 0;
  uint64_t arena = 0, stream_bytes = 0;
  double algo = 0;
  std::vector<uint64_t> t_off(K), t_len(K);
  for (uint32_t k = 0; k < K; ++k) {
    const PassStepIn& s = steps[k];
    const nqb_group* g = s.group;
    NQB_REQUIRE(g != nullptr, NQB_E_VALIDATION, "pass step without a decode group");
    NQB_REQUIRE(g->device == ctx->device, NQB_E_VALIDATION, "decode group lives on another device");
    NQB_REQUIRE(g->grid <= G, NQB_E_VALIDATION,
                "decode group planned for more SMs than the context's budget");
    NQB_REQUIRE(s.x != nullptr, NQB_E_VALIDATION, "null pass input");
    StepDesc& D = desc[k];
    D.bits = g->bits;
    D.x = s.x;
    D.nseg = g->nseg;
    D.m = g->m;
    D.R1 = g->R1;
    const uint32_t esz = s.f32 ? 4 : 2;
    D.flags = (s.f32 ? (kStepXF32 | kStepYF32) : 0u) |
              (((uintptr_t)s.x % 16 == 0) ? kStepXVec : 0u);
    for (uint32_t q = 0; q < g->nseg; ++q) {
      NQB_REQUIRE(s.y[q] != nullptr, NQB_E_VALIDATION, "null pass output");
      D.seg[q] = g->seg[q];
      D.y[q] = s.y[q];
      NQB_REQUIRE(!overlaps(s.y[q], (size_t)g->n[q] * esz, s.x, (size_t)g->m * esz),
                  NQB_E_VALIDATION, "a pass step's output overlaps its own input");
      algo += (double)g->r[q] * (g->n[q] + g->m) / 8.0 + 2.0 * (g->n[q] + g->m) + esz * g->n[q];
    }
    algo += (double)esz * g->m;
    bfrag = std::max(bfrag, g->bfrag_bytes);
    stream_bytes += g->stream_bytes;
    t_off[k] = arena;
    t_len[k] = (uint64_t)g->R1 + kStepTail;
    arena += (t_len[k] + 1) / 2 * 2;  // 16-byte aligned regions (vector t loads)
    // dependencies from buffer ranges: the latest earlier step whose output
    // overlaps this input must have finished (output barrier) before stage 1
    D.x_src = -1;
    D.xmax_src = -1;
    for (int j = (int)k - 1; j >= 0 && D.x_src < 0; --j) {
      const uint32_t ej = (desc[j].flags & kStepYF32) ? 4 : 2;
      for (uint32_t q = 0; q < desc[j].nseg; ++q) {
        if (!overlaps(desc[j].y[q], (size_t)desc[j].seg[q].n * ej, s.x, (size_t)g->m * esz))
          continue;
        D.x_src = j;
        if (desc[j].y[q] == s.x && desc[j].seg[q].n == g->m && ej == esz)
          D.xmax_src = (int32_t)(j * kMaxSeg + q);
      }
    }
    if (D.x_src >= 0) desc[D.x_src].flags |= kStepPublish;
  }
  // one-step lookahead (stage 1 of k+1 before stage 2 of k) when k+1 neither
  // reads nor overwrites k's outputs
  for (uint32_t k = 0; k + 1 < K; ++k) {
    bool dep = desc[k + 1].x_src == (int32_t)k;
    const uint32_t ek = (desc[k].flags & kStepYF32) ? 4 : 2;
    const uint32_t e1 = (desc[k + 1].flags & kStepYF32) ? 4 : 2;
    for (uint32_t a = 0; a < desc[k].nseg && !dep; ++a)
      for (uint32_t b = 0; b < desc[k + 1].nseg && !dep; ++b)
        dep = overlaps(desc[k].y[a], (size_t)desc[k].seg[a].n * ek, desc[k + 1].y[b],
                       (size_t)desc[k + 1].seg[b].n * e1);
    if (!dep && env_u32p("NQB_PASS_LOOKAHEAD", 1)) desc[k].flags |= kStepLookahead;
  }
  for (uint32_t k = 0; k < K; ++k) {
    desc[k].t_off = t_off[k];
    desc[k].zero_off = k >= 2 ? t_off[k - 2] : 0;
    desc[k].zero_len = k >= 2 ? (uint32_t)t_len[k - 2] : 0;
  }

  // ---- device memory: descriptors | CTA tables | counters | ymax | arena ----
  const size_t desc_b = sizeof(StepDesc) * K;
  const size_t cta_b = sizeof(Cta) * (size_t)K * G;
  const size_t ctr_b = sizeof(unsigned long long) * kCtrStride * (2 + 2 * (size_t)K);
  const size_t ymax_b = ((size_t)K * kMaxSeg * 4 + 15) / 16 * 16;
  const size_t arena_b = arena * 8;
  auto* P = new nqb_pass();
  P->device = ctx->device;
  P->K = K;
  P->G = G;
  try {
    NQB_CUDA(cudaMalloc(&P->dmem, desc_b + cta_b + ctr_b + ymax_b + arena_b));
    char* base = (char*)P->dmem;
    StepDesc* d_desc = (StepDesc*)base;
    Cta* d_ctas = (Cta*)(base + desc_b);
    auto* d_ctr = (unsigned long long*)(base + desc_b + cta_b);
    auto* d_ymax = (unsigned*)(base + desc_b + cta_b + ctr_b);
    auto* d_arena = (long long*)(base + desc_b + cta_b + ctr_b + ymax_b);
    std::vector<Cta> ctas((size_t)K * G, Cta{});
    for (uint32_t k = 0; k < K; ++k) {
      const nqb_group* g = steps[k].group;
      std::copy(g->ctas, g->ctas + g->grid, ctas.begin() + (size_t)k * G);
      desc[k].ctas = d_ctas + (size_t)k * G;
    }
    NQB_CUDA(cudaMemsetAsync(d_ctr, 0, ctr_b + ymax_b + arena_b, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(d_desc, desc.data(), desc_b, cudaMemcpyHostToDevice, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(d_ctas, ctas.data(), cta_b, cudaMemcpyHostToDevice, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));

    PassParams& pp = P->params;
    pp.desc = d_desc;
    pp.K = K;
    pp.G = G;
    pp.ctr = d_ctr;
    pp.ymax = d_ymax;
    pp.arena = d_arena;
    pp.bfrag_bytes = (bfrag + 127) / 128 * 128;
    const uint32_t head = pass_head_bytes();
    pp.ring_bytes = (227u * 1024u - head - pp.bfrag_bytes) / 128 * 128;
    const uint32_t cap_kb = env_u32p("NQB_PASS_CHUNK_KB", 0);
    pp.chunk_cap = cap_kb ? cap_kb * 1024 : pp.ring_bytes / 4 / 128 * 128;
    // a chunk is at most cap + the largest section + prefix + suffix: keep two in the ring
    NQB_REQUIRE(pp.chunk_cap + 16384 + 8192 + 1024 <= pp.ring_bytes / 2, NQB_E_VALIDATION,
                "NQB_PASS_CHUNK_KB too large for the shared-memory ring");
    pp.ntail = std::min<uint32_t>(K, 2);
    for (uint32_t t = 0; t < pp.ntail; ++t) {
      const uint32_t k = K - pp.ntail + t;
      pp.tail_off[t] = t_off[k];
      pp.tail_len[t] = (uint32_t)t_len[k];
    }
    P->smem_bytes = head + pp.bfrag_bytes + pp.ring_bytes;
    P->stream_bytes = stream_bytes;
    P->algo_bytes = (uint64_t)algo;
    for (auto fn : {k_decode_pass<false>, k_decode_pass<true>})
      NQB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)P->smem_bytes));
    int per_sm = 0;
    NQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_pass<false>, kThreads,
                                                           P->smem_bytes));
    NQB_REQUIRE(per_sm >= 1, NQB_E_INTERNAL, "decode pass kernel does not fit an SM");
  } catch (...) {
    pass_free(P);
    throw;
  }
  return P;
}

void pass_launch(nqb_context* ctx, const nqb_pass* P, unsigned long long* trace) {
  NQB_REQUIRE(P->device == ctx->device, NQB_E_VALIDATION, "decode pass lives on another device");
  PassParams pp = P->params;
  pp.trace = trace;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = P->smem_bytes;
  cfg.stream = ctx->stream;
  // cooperative launch: the runtime guarantees every CTA is co-resident (the
  // in-kernel barriers need it) or fails the launch
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = env_u32p("NQB_PASS_COOP", 1) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (trace) NQB_CUDA(cudaLaunchKernelEx(&cfg, k_decode_pass<true>, pp));
  else NQB_CUDA(cudaLaunchKernelEx(&cfg, k_decode_pass<false>, pp));
  NQB_LAUNCHED(ctx);
}

void pass_free(nqb_pass* P) {
  if (!P) return;
  cudaSetDevice(P->device);
  cudaFree(P->dmem);
  delete P;
}

}  // namespace nqb
