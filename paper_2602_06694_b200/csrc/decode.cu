// decode.cu — batch-1 BLR decode GEMV (gemv_packed_f32, packed.cpp:201-204)
// as one fused two-stage sm_100a kernel.  Design: decode.cuh, DESIGN.md §4.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "decode_dev.cuh"

namespace nqb {
namespace dec {

template <bool kTrace, bool kBig>
__global__ void __launch_bounds__(kThreads, (kConsumerWarps <= 8 ? 2 : 1)) k_decode(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t NB = p.nbar;
  uint64_t* full = (uint64_t*)(smem);
  uint64_t* empty = full + NB;
  uint64_t* scb = empty + NB;  // the two scale slices landed
  long long* red8 = (long long*)(smem + 16 * NB + 16);
  float* xred = (float*)(smem + 16 * NB + 16 + 256);  // per-warp max|x| (fp32 x)
  int* red = (int*)(smem + 16 * NB + 16 + 256 + 64);
  __half* sc2 = (__half*)(smem + 16 * NB + 16 + 256 + 64 + kRedBytes);
  __half* sc1 = sc2 + kSc2Elems;
  uint8_t* bfrag = smem + head_bytes(NB);
  uint8_t* buf = bfrag + p.bfrag_bytes;

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(~0u, tid >> 5, 0);
  long long trace_t0 = 0;
  // trace pointer pinned in a register (a re-read of the parameter bank at
  // every stamp would perturb the timeline it measures)
  unsigned long long* trp = nullptr;
  if (kTrace) asm volatile("mov.b64 %0, %1;" : "=l"(trp) : "l"(p.trace));
  if (kTrace) trace_t0 = clock64();  // every thread's base (the producer's stamps use it)
  TRACE(0);
  const Cta C = p.ctas[blockIdx.x];
  if (kTrace && tid == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.trace[blockIdx.x * 32 + 16] = smid;
    p.trace[blockIdx.x * 32 + 17] = C.s1_rtn;
    p.trace[blockIdx.x * 32 + 18] = C.s1_sln;
    p.trace[blockIdx.x * 32 + 19] = C.s2_rtn;
    p.trace[blockIdx.x * 32 + 20] = C.nsec;
    p.trace[blockIdx.x * 32 + 21] = C.ring;
  }
  const uint32_t n1 = C.s1_rtn ? C.s1_sln : 0;
  const uint32_t m = p.m;
  // stage-1 input range [klo1, klo1 + nk1) of this CTA (slab-aligned)
  uint32_t klo1 = 0, nk1 = 0;
  if (n1) {
    klo1 = slab_of(m, C.s1_sl0).k0;
    const Slab last = slab_of(m, C.s1_sl0 + C.s1_sln - 1);
    nk1 = last.k0 + 32 * last.nq - klo1;
  }
  const bool ring_mode = C.ring != 0;
  const uint32_t NS = ring_mode ? p.buf_bytes / p.slot_bytes : 0;  // ring slots
  auto sec_bytes = [&](uint32_t sec) -> uint32_t {
    return sec < n1 ? C.s1_rtn * unit_bytes(slab_of(m, C.s1_sl0 + sec).nq)
                    : C.s2_rtn * unit_bytes(slab_of(p.seg[C.s2_seg].r, sec - n1).nq);
  };

  if (tid == 0) {
    for (uint32_t s = 0; s < NB; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], kConsumerWarps);
    }
    tc::mbar_init(scb, 1);
    tc::fence_mbar_init();
  }
  __syncthreads();
  pdl_launch_dependents();  // the next kernel may start streaming its bits

  // ------------------------------------------------------------------ producer
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      // scale slices first: weights, so independent of the previous kernel
      // (layer scales are zero-padded to whole slabs / row tiles, api.cu)
      const uint32_t sb2 = 2 * nk1, sb1 = 32u * C.s2_rtn;
      if (sb1 + sb2) {
        tc::mbar_arrive_expect_tx(scb, sb1 + sb2);
        if (sb2) tc::bulk_g2s(sc2, p.seg[C.s1_seg].s2h + klo1, sb2, scb);
        if (sb1) tc::bulk_g2s(sc1, p.seg[C.s2_seg].s1h + (size_t)C.s2_rt0 * 16, sb1, scb);
      }
      const uint8_t* src = p.bits + C.stream_off;
      uint32_t off = 0;
      for (uint32_t sec = 0; sec < C.nsec; ++sec) {
        const uint32_t bytes = sec_bytes(sec);
        if (ring_mode) {
          const uint32_t slot = sec % NS;
          if (sec >= NS) mbar_wait_wd(&empty[slot], ((sec / NS) - 1) & 1);
          tc::mbar_arrive_expect_tx(&full[slot], bytes);
          tc::bulk_g2s(buf + (size_t)slot * p.slot_bytes, src + off, bytes, &full[slot]);
        } else {  // linear: the section lives at its stream offset; one barrier per stage
          uint64_t* bar = &full[sec < n1 ? 0 : 1];
          // stage-1 bits first: HBM serves them before the (larger, later
          // needed) stage-2 stream, so stage 1 is not starved by stage 2
          if (p.seq && sec == n1 && n1) mbar_wait_wd(&full[0], 0);
          if (sec == 0 || sec == n1) {
            uint32_t total = 0;
            for (uint32_t q = sec; q < (sec < n1 ? n1 : C.nsec); ++q) total += sec_bytes(q);
            tc::mbar_arrive_expect_tx(bar, total);
          }
          tc::bulk_g2s(buf + off, src + off, bytes, bar);
        }
        off += bytes;
      }
      if (kTrace) p.trace[blockIdx.x * 32 + 14] = clock64() - trace_t0;
      if (kTrace && !ring_mode && C.nsec) {  // diagnostics: the whole stream landed
        if (n1) mbar_wait_wd(&full[0], 0);
        if (C.nsec > n1) mbar_wait_wd(&full[1], 0);
        p.trace[blockIdx.x * 32 + 15] = clock64() - trace_t0;
      }
    }
    return;
  }

  // ----------------------------------------------------------------- consumers
  for (int i = tid; i < kMaxRt * 16 * kRedStride / 4; i += kConsumerThreads)
    ((int4*)red)[i] = make_int4(0, 0, 0, 0);
  TRACE(1);
  pdl_wait();  // x (and the t accumulator) may be written by the previous kernel
  TRACE(2);
  State* st = p.st;
  // epoch and the dirty count of the next t buffer: one thread of the last
  // consumer warp loads them right away and parks them in shared memory (the
  // other warps read them after the stage-1 barrier), so no warp carries the
  // load's scoreboard through stage 1
  uint32_t* stw = (uint32_t*)(smem + 16 * NB + 8);  // spare 8 bytes after scb
  if (warp == kConsumerWarps - 1 && lane == 0) {
    uint32_t e, d0, d1;
    asm volatile("ld.relaxed.gpu.global.v2.u32 {%0,%1}, [%3];\n\t"
                 "ld.relaxed.gpu.global.u32 %2, [%3+8];\n"
                 : "=r"(e), "=r"(d0), "=r"(d1) : "l"(st) : "memory");
    stw[0] = e;
    stw[1] = (e & 1) ? d0 : d1;
  }

  // ---- activation exponent: a = s2*x with |a| <= max|s2| * max|x| (one pass
  // over all m inputs in every CTA; +Inf flags a non-finite input)
  const float xmax = x_absmax(p.x, m, p.x_f32 != 0, p.x_vec != 0, xred);
  const bool nonfinite = is_inf(xmax);
  TRACE(3);

  // ------------------------------------------------------------------ stage 1
  if (n1) {
    const Seg& S = p.seg[C.s1_seg];
    const int ea = act_exponent(S.s2max, xmax);
    const uint32_t klo = klo1;
    const uint32_t nquad = nk1 / 4;
    const __half* s2s = sc2 - klo;
    long long asum = 0, aabs = 0;
    uint32_t qd = tid;
    mbar_wait_wd(scb, 0);
    XQuad cur = load_xquad(p, s2s, klo + 4 * min(qd, nquad - 1), m);
    while (qd < nquad) {  // one quad in flight ahead of the one being quantised
      const uint32_t nx = qd + kConsumerThreads;
      const XQuad nxt = load_xquad(p, s2s, klo + 4 * min(nx, nquad - 1), m);
      const uint32_t k0 = klo + 4 * qd;
      long long v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float a = nonfinite ? 0.f : cur.s[e] * cur.x[e];  // packed.cpp:160
        v[e] = __float2ll_rn(scale_pow2(a, kFix - ea));
        asum += v[e];
        aabs += v[e] < 0 ? -v[e] : v[e];
      }
      emit_quad(bfrag, klo, k0, q_of(k0, m), v);
      cur = nxt;
      qd = nx;
    }
    warp_partials2(asum, aabs, red8);
    consumers_sync();  // B fragments and the partial sums are visible
    TRACE(4);
    StageArgs sa{C.s1_rtn, n1, 0, m, C.s1_sl0, klo, 0};  // linear: barrier full[0]
    run_stage<kBig>(sa, NS, ring_mode, p.slot_bytes, full, empty, buf, bfrag, red,
              (kTrace && warp == 0) ? p.trace + blockIdx.x * 32 + 22 : nullptr);
    consumers_sync();
    TRACE(5);
  }
  if (!n1) consumers_sync();  // (CTAs with stage 1 passed a consumer barrier after it)
  const uint32_t ep = stw[0], dirty_next = stw[1];
  const uint32_t b = ep & 1;
  TRACE(12);
  if (n1) {
    const long long A = sum_partials(red8);
    long long* Tseg = p.T + (size_t)b * p.r_cap + p.seg[C.s1_seg].t_off + (size_t)C.s1_rt0 * 16;
    for (uint32_t i = tid; i < (uint32_t)C.s1_rtn * 16; i += kConsumerThreads) {
      const long long v = 2 * row_value(red + i * kRedStride) - A;
      int4* rr = (int4*)(red + i * kRedStride);  // leave the row zeroed for stage 2
      rr[0] = make_int4(0, 0, 0, 0);
      rr[1] = make_int4(0, 0, 0, 0);
      red_add_u64(&Tseg[i], v);
    }
  }
  TRACE(13);
  {  // clear this CTA's share of the other t buffer for the next launch
    long long* Tn = p.T + (size_t)(b ^ 1) * p.r_cap;
    const uint32_t per = (dirty_next + gridDim.x - 1) / gridDim.x;  // 32-bit: no 64-bit divide
    const uint32_t lo = min(dirty_next, per * blockIdx.x), hi = min(dirty_next, lo + per);
    for (uint32_t i = lo + tid; i < hi; i += kConsumerThreads) Tn[i] = 0;
  }

  // --------------------------------------------------------------- grid barrier
  consumers_sync();  // the CTA's reds to t happen-before thread 0's fence (cumulativity)
  TRACE(6);
  // Arrival is a fire-and-forget release reduction (no round trip on the
  // critical path); CTA 0 advances the state once everyone has arrived (every
  // CTA read epoch and dirty before arriving).
  if (tid == 0) red_release_add_u32(&st->done[b].v, 1u);
  if (!C.s2_rtn && blockIdx.x != 0) return;
  TRACE(7);
  if (tid == 0) {
    uint32_t it = 0;
    while (ld_acquire(&st->done[b].v) < gridDim.x) {
      __nanosleep(20);
      if (++it > (1u << 26)) __trap();
    }
    if (blockIdx.x == 0) {
      st->epoch = ep + 1;
      st->dirty[b] = p.R1;
      st->dirty[b ^ 1] = 0;
      st->done[b ^ 1].v = 0;
#pragma unroll
      for (int sg = 0; sg < kMaxSeg; ++sg) st->abs_a[b ^ 1][sg] = 0;
    }
  }
  if (!C.s2_rtn) return;
  consumers_sync();
  TRACE(8);
  // (red is all zero here: stage 1 cleared the rows it used while publishing)

  // ------------------------------------------------------------------ stage 2
  const Seg& S = p.seg[C.s2_seg];
  const int ea = act_exponent(S.s2max, xmax);
  const int sh = t_shift(m);  // |t_k| < 2^(kFix + sh)
  const long long* Tseg = p.T + (size_t)b * p.r_cap + S.t_off;
  const uint32_t nquad2 = kpad(S.r) / 4;
  long long tsum = 0;
  {
    uint32_t qd = tid;
    long long cur[4], nxt[4];
    load_tquad(Tseg, 4 * min(qd, nquad2 - 1), S.r, (uint64_t)b * p.r_cap + S.t_off, cur);
    while (qd < nquad2) {
      const uint32_t nx = qd + kConsumerThreads;
      load_tquad(Tseg, 4 * min(nx, nquad2 - 1), S.r, (uint64_t)b * p.r_cap + S.t_off, nxt);
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
  consumers_sync();  // B fragments and the partial sums are visible
  TRACE(9);
  uint32_t s1_bytes = 0;  // linear offset of the first stage-2 section
  for (uint32_t s = 0; s < n1; ++s) s1_bytes += sec_bytes(s);
  StageArgs sa{C.s2_rtn, C.nsec - n1, n1, S.r, 0, 0, s1_bytes};
  if (!ring_mode) sa.sec_base = 1;  // linear: barrier full[1]
  run_stage<kBig>(sa, NS, ring_mode, p.slot_bytes, full, empty, buf, bfrag, red,
            (kTrace && warp == 0) ? p.trace + blockIdx.x * 32 + 27 : nullptr);
  consumers_sync();
  TRACE(10);
  const long long Tsum = sum_partials(red8);
  const int E = sh + ea - kFix;  // t = T2 * 2^sh * 2^(ea - kFix)
  if (!n1) mbar_wait_wd(scb, 0);
  for (uint32_t i = tid; i < (uint32_t)C.s2_rtn * 16; i += kConsumerThreads) {
    const uint32_t row = C.s2_rt0 * 16 + i;
    if (row >= S.n) continue;
    const long long Y = 2 * row_value(red + i * kRedStride) - Tsum;
    // Y * 2^E is exact in fp64 (|Y| < 2^53, E in the normal range)
    double y = (double)__half2float(sc1[i]) *
               ((double)Y * __longlong_as_double((long long)(1023 + E) << 52));  // packed.cpp:189
    if (nonfinite) y = __longlong_as_double(0x7ff8000000000000ll);
    if (p.y_f32) ((float*)p.y[C.s2_seg])[row] = (float)y;
    else ((__half*)p.y[C.s2_seg])[row] = __float2half_rn((float)y);
  }
  TRACE(11);
}

}  // namespace dec

using namespace dec;

// Grows the context's decode state.  A CUDA graph captured earlier holds the
// old state and t buffers in its kernel parameters, so the old allocation is
// retired (kept until nqb_destroy), never freed here; growing while the stream
// is being captured is refused (group_build reserves ahead of any capture).
void dec_state_reserve(nqb_context* ctx, uint32_t rows) {
  if (ctx->dec_state && ctx->dec_cap >= rows) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  NQB_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
  NQB_REQUIRE(cs == cudaStreamCaptureStatusNone, NQB_E_VALIDATION,
              "decode state must grow while a graph is being captured: build every decode "
              "group before nqb_graph_begin");
  if (ctx->dec_state) ctx->dec_retired.push_back(ctx->dec_state);
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
  NQB_REQUIRE(!g->pass_only, NQB_E_VALIDATION, "a pass-only decode plan cannot run per call");
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
  {
    static const uint32_t seq = [] { const char* v = std::getenv("NQB_DEC_SEQ");
                                     return v ? (uint32_t)std::strtoul(v, nullptr, 10) : 1u; }();
    p.seq = seq;
  }
  p.x = d_x;
  p.trace = (unsigned long long*)ctx->dec_trace;

  if (!ctx->dec_attr_set) {
    for (auto fn : {k_decode<false, false>, k_decode<false, true>, k_decode<true, false>,
                    k_decode<true, true>})
      NQB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    ctx->dec_attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g->grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g->smem_bytes;
  cfg.stream = ctx->stream;
  // Cooperative launch: the runtime guarantees that every CTA is co-resident
  // (the in-kernel grid barrier needs it) or fails the launch, even when other
  // streams or contexts hold SMs.  Programmatic serialization (PDL) still lets
  // the launch start while the previous kernel drains.
  static const bool coop = [] {
    const char* v = std::getenv("NQB_DEC_COOP");
    return !v || std::strtoul(v, nullptr, 10) != 0;
  }();
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = ctx->pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = coop ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const bool big = g->big;
  if (p.trace) NQB_CUDA(cudaLaunchKernelEx(&cfg, big ? k_decode<true, true> : k_decode<true, false>, p));
  else NQB_CUDA(cudaLaunchKernelEx(&cfg, big ? k_decode<false, true> : k_decode<false, false>, p));
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
