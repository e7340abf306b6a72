// decode_plan.cu — work split and bit layout of the decode GEMV.
//
// A plan covers 1..kMaxSeg layers ("segments") that read the same input x
// (e.g. q/k/v, or gate/up).  It fixes, once at upload time:
//   * the grid (<= #SMs, all CTAs co-resident for the in-kernel grid barrier);
//   * per CTA one stage-1 block (16-row tiles of V^T x 256-wide slabs of m) and
//     one stage-2 block (16-row tiles of U over all slabs of r);
//   * the byte stream each CTA reads: its stage-1 sections (one per slab, the
//     CTA's row tiles back to back) followed by its stage-2 sections.
// Inside a 512-byte unit (16 rows x 256 K) lane l = 4g+c of the consuming warp
// owns 16 contiguous bytes = words w0..w3, and bit 8b+q of w_i is
//   A[row g + 8(i&1)][K = 32q + 16(i>>1) + 4c + b]
// i.e. exactly the mma.m16n8k32 A fragment of tile q after `w_i & 0x01010101<<q`.
// 128-wide and 64-wide tail slabs pack the same 16 bits per lane per tile into
// 8 or 4 bytes (see k_relayout and the kernel's word unpacking).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "decode.cuh"

namespace nqb {
namespace dec {

struct RelayoutSrc {
  const uint32_t* u[kMaxSeg];   // n x u_words (bits along r)
  const uint32_t* vt[kMaxSeg];  // r x vt_words (bits along m)
  uint32_t u_words[kMaxSeg], vt_words[kMaxSeg];
};

// Maps (lane, word, bit) of a unit with nq tiles to (row in tile, K in slab).
__host__ __device__ __forceinline__ void unit_pos(uint32_t nq, uint32_t lane, uint32_t wl,
                                                  uint32_t p, uint32_t& row, uint32_t& kk) {
  const uint32_t b = p >> 3, bb = p & 7;
  uint32_t i, q;
  if (nq == 8) {
    i = wl;
    q = bb;
  } else if (nq == 4) {
    i = 2 * wl + (bb >> 2);
    q = bb & 3;
  } else {
    i = bb >> 1;
    q = bb & 1;
  }
  const uint32_t g = lane >> 2, c = lane & 3;
  row = g + 8 * (i & 1);
  kk = 32 * q + 16 * (i >> 1) + 4 * c + b;
}

// Bytes of one row tile over all slabs of a stage (stage 1: the CTA's slabs of m,
// stage 2: every slab of r).
__device__ uint32_t stage_tile_bytes(const Cta& C, bool st1, uint32_t m, uint32_t r) {
  uint32_t b = 0;
  if (st1)
    for (uint32_t q = C.s1_sl0; q < (uint32_t)C.s1_sl0 + C.s1_sln; ++q) b += unit_bytes(slab_of(m, q).nq);
  else
    for (uint32_t q = 0, ns = nslabs(r); q < ns; ++q) b += unit_bytes(slab_of(r, q).nq);
  return b;
}

// One block per CTA of the plan: writes that CTA's byte stream.
// Slab-major (per-call kernel): per stage, section = slab, the CTA's row tiles
// back to back.  Decode-pass plans (pm): per stage tile-major, each row tile's
// slabs in order, so one tile of a stage is one contiguous byte range:
//   offset(tile t, slab i) = t Utot + U_i
// (Utot: bytes of a tile over the stage's slabs, U_i: of its first i slabs).
__global__ void k_relayout(const Cta* __restrict__ ctas, const Seg* __restrict__ segs,
                           uint32_t m, RelayoutSrc src, uint32_t* __restrict__ out, int pm) {
  const Cta C = ctas[blockIdx.x];
  uint32_t* dst = out + C.stream_off / 4;
  uint32_t sec_words_off = 0;
  const uint32_t n1 = C.s1_rtn ? C.s1_sln : 0;
  uint32_t u_cum = 0, stage_w = 0;  // tile-major: U_i of the current stage, its first word
  for (uint32_t sec = 0; sec < C.nsec; ++sec) {
    const bool st1 = sec < n1;
    const uint32_t seg = st1 ? C.s1_seg : C.s2_seg;
    const Seg S = segs[seg];
    const uint32_t K = st1 ? m : S.r;
    const Slab sl = slab_of(K, st1 ? C.s1_sl0 + sec : sec - n1);
    const uint32_t rtn = st1 ? C.s1_rtn : C.s2_rtn;
    const uint32_t rt0 = st1 ? C.s1_rt0 : C.s2_rt0;
    const uint32_t unit_words = 16 * sl.nq, lane_words = sl.nq / 2;
    const uint32_t words = rtn * unit_words;
    if (sec == n1 && sec) {  // stage 2 starts after the whole stage-1 block
      stage_w = sec_words_off;
      u_cum = 0;
    }
    const uint32_t utot = pm ? stage_tile_bytes(C, st1, m, S.r) : 0u;
    for (uint32_t x = threadIdx.x; x < words; x += blockDim.x) {
      const uint32_t t = x / unit_words, rem = x % unit_words;
      // tile-major: a decode-pass work item is one whole row tile of a stage
      // (decode_pass.cu, row-complete items)
      const uint32_t dw = !pm ? sec_words_off + x : stage_w + (t * utot + u_cum) / 4 + rem;
      const uint32_t lane = rem / lane_words, wl = rem % lane_words;
      uint32_t v = 0;
      for (uint32_t p = 0; p < 32; ++p) {
        uint32_t row, kk;
        unit_pos(sl.nq, lane, wl, p, row, kk);
        const uint32_t R = (rt0 + t) * 16 + row, k = sl.k0 + kk;
        uint32_t bit = 0;
        if (st1) {  // V^T: row = rank index, K = input index j
          if (R < S.r && k < m)
            bit = (src.vt[seg][(uint64_t)R * src.vt_words[seg] + k / 32] >> (k % 32)) & 1u;
        } else {    // U: row = output index i, K = rank index
          if (R < S.n && k < S.r)
            bit = (src.u[seg][(uint64_t)R * src.u_words[seg] + k / 32] >> (k % 32)) & 1u;
        }
        v |= bit << p;
      }
      dst[dw] = v;
    }
    sec_words_off += words;
    u_cum += 4 * unit_words;
  }
}

__global__ void k_absmax_half(const __half* __restrict__ s, uint32_t n, uint32_t* out) {
  uint32_t mx = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    mx = max(mx, (uint32_t)(__half_as_ushort(s[i]) & 0x7FFFu));
  mx = max(mx, __shfl_xor_sync(~0u, mx, 16));
  mx = max(mx, __shfl_xor_sync(~0u, mx, 8));
  mx = max(mx, __shfl_xor_sync(~0u, mx, 4));
  mx = max(mx, __shfl_xor_sync(~0u, mx, 2));
  mx = max(mx, __shfl_xor_sync(~0u, mx, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

}  // namespace dec

using namespace dec;

namespace {

// Cost of quantising one activation into B fragments, in streamed-byte
// equivalents (~35 thread instructions vs ~0.05 cycles per streamed byte).
constexpr double kQuantBytes = 6.0;

struct Block1 {
  uint32_t seg, rt0, rtn, sl0, sln;
};

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return (uint32_t)std::strtoul(v, nullptr, 10);
}

// Splits [0, total) into parts contiguous ranges of near-equal length.
inline void split_range(uint32_t total, uint32_t parts, uint32_t idx, uint32_t& lo,
                        uint32_t& cnt) {
  const uint64_t a = (uint64_t)total * idx / parts, b = (uint64_t)total * (idx + 1) / parts;
  lo = (uint32_t)a;
  cnt = (uint32_t)(b - a);
}

}  // namespace

nqb_group* group_build(nqb_context* ctx, const nqb_layer* const* layers, uint32_t count,
                       uint32_t grid_cap, uint32_t max_rt, bool pass_only, uint32_t plan_slabs) {
  if (!max_rt) max_rt = kMaxRt;
  NQB_REQUIRE(count >= 1 && count <= (uint32_t)kMaxSeg, NQB_E_VALIDATION,
              "a decode group holds 1.." + std::to_string(kMaxSeg) + " layers");
  const uint32_t m = layers[0]->m;
  for (uint32_t s = 0; s < count; ++s) {
    NQB_REQUIRE(layers[s] != nullptr, NQB_E_VALIDATION, "null layer in group");
    NQB_REQUIRE(layers[s]->m == m, NQB_E_DIMENSION_MISMATCH,
                "layers of a decode group must share the input length m");
    NQB_REQUIRE(layers[s]->r <= 65536 && layers[s]->n <= 16u * 32u * 1024u,
                NQB_E_DIMENSION_MISMATCH, "layer too large for the decode kernel");
  }
  NQB_REQUIRE(m <= (1u << 20), NQB_E_DIMENSION_MISMATCH, "input too long for the decode kernel");

  // ---- per-segment geometry ------------------------------------------------
  const uint32_t S1 = nslabs(m);
  uint64_t slab1_bytes = 0;
  std::vector<uint32_t> u1(S1);
  for (uint32_t s = 0; s < S1; ++s) {
    u1[s] = unit_bytes(slab_of(m, s).nq);
    slab1_bytes += u1[s];
  }
  std::vector<uint32_t> RT1(count), RT2(count), toff(count);
  std::vector<uint64_t> row2_bytes(count), B1(count), B2(count);
  uint32_t R1 = 0;
  uint64_t Btot = 0, B1tot = 0;
  for (uint32_t s = 0; s < count; ++s) {
    const nqb_layer* L = layers[s];
    RT1[s] = (L->r + 15) / 16;
    RT2[s] = (L->n + 15) / 16;
    toff[s] = R1;
    R1 += RT1[s] * 16;
    uint64_t rb = 0;
    for (uint32_t q = 0, ns = nslabs(L->r); q < ns; ++q) rb += unit_bytes(slab_of(L->r, q).nq);
    row2_bytes[s] = rb;
    B1[s] = (uint64_t)RT1[s] * slab1_bytes;
    B2[s] = (uint64_t)RT2[s] * rb;
    Btot += B1[s] + B2[s];
    B1tot += B1[s];
  }

  uint32_t Gmax = std::min<uint32_t>((uint32_t)ctx->num_sms, kMaxGrid);
  if (grid_cap) Gmax = std::min(Gmax, grid_cap);
  const uint32_t min_cta_bytes = env_u32("NQB_DEC_MIN_CTA_BYTES", 8192);
  uint32_t G = (uint32_t)std::min<uint64_t>(Gmax, std::max<uint64_t>(1, (Btot + min_cta_bytes - 1) /
                                                                         min_cta_bytes));
  G = std::max(G, count);

  const double quant_bytes = env_u32("NQB_DEC_QUANT_X100", (uint32_t)(kQuantBytes * 100)) / 100.0;
  // measured (tools/gpu_pass_envab.sh): whole-input ranges (16 slabs) for m <= 4096
  // (7B pass: 1274 vs 1231 GB/s for 8), 8 slabs above (70B pass: 1758 vs 1378 GB/s:
  // the smaller quantised-x staging leaves more shared memory to the rings)
  const uint32_t pass_slabs = std::min<uint32_t>(
      std::max<uint32_t>(env_u32("NQB_PASS_PLAN_SLABS", plan_slabs ? plan_slabs : m <= 4096 ? 16 : 8), 1),
      kMaxSlabs1);
  std::vector<Cta> ctas;
  for (;; ++G) {
    NQB_REQUIRE(G <= Gmax, NQB_E_DIMENSION_MISMATCH,
                "decode plan does not fit the grid (layer too large)");
    // ---- stage-1 blocks: CTAs per segment proportional to bytes ------------
    std::vector<uint32_t> G1(count, 1);
    {
      uint32_t left = G - count;
      std::vector<std::pair<double, uint32_t>> rem;
      for (uint32_t s = 0; s < count; ++s) {
        const double want = (double)G * B1[s] / std::max<uint64_t>(B1tot, 1) - 1.0;
        const uint32_t add = (uint32_t)std::max(0.0, std::floor(want));
        const uint32_t take = std::min(add, left);
        G1[s] += take;
        left -= take;
        rem.push_back({want - take, s});
      }
      std::sort(rem.rbegin(), rem.rend());
      for (auto& pr : rem) {
        if (!left) break;
        G1[pr.second]++;
        left--;
      }
    }
    std::vector<Block1> blocks;
    bool ok = true;
    for (uint32_t s = 0; s < count && ok; ++s) {
      double best = 1e300;
      uint32_t bGk = 0, bGj = 0;
      for (uint32_t Gj = 1; Gj <= std::min(S1, G1[s]); ++Gj) {
        const uint32_t Gk = std::min(RT1[s], G1[s] / Gj);
        if (!Gk) continue;
        const uint32_t rt_max = (RT1[s] + Gk - 1) / Gk, sl_max = (S1 + Gj - 1) / Gj;
        if (rt_max > max_rt || sl_max > (uint32_t)kMaxSlabs1) continue;
        // bytes of the heaviest block (slab groups from split_range)
        uint64_t heavy = 0;
        for (uint32_t j = 0; j < Gj; ++j) {
          uint32_t lo, cnt;
          split_range(S1, Gj, j, lo, cnt);
          uint64_t b = 0;
          for (uint32_t q = lo; q < lo + cnt; ++q) b += u1[q];
          heavy = std::max(heavy, b);
        }
        // bytes streamed + the CTA's quantisation work (kQuantBytes per input).
        // A pass plan takes slab ranges of up to pass_slabs slabs, as long as fit: its work items are runs of one tile pair over the
        // CTA's slabs (long runs per flush), while the quantised-x staging grows with
        // the range (the pass quantises in helper warps, off the MMA path).
        const double cost = pass_only ? (double)(sl_max > pass_slabs ? sl_max - pass_slabs + 64
                                                                     : pass_slabs - sl_max) *
                                                1e15 + (double)rt_max * heavy
                                      : ((double)rt_max * heavy + quant_bytes * 256.0 * sl_max) *
                                            (1.0 + 1e-3 * Gj);
        if (cost < best) {
          best = cost;
          bGk = Gk;
          bGj = Gj;
        }
      }
      if (!bGk) {
        ok = false;
        break;
      }
      for (uint32_t k = 0; k < bGk; ++k)
        for (uint32_t j = 0; j < bGj; ++j) {
          Block1 b;
          b.seg = s;
          split_range(RT1[s], bGk, k, b.rt0, b.rtn);
          split_range(S1, bGj, j, b.sl0, b.sln);
          if (b.rtn && b.sln) blocks.push_back(b);
        }
    }
    if (!ok || blocks.size() > G) continue;

    // ---- assign stage-1 blocks to CTAs, then water-fill stage-2 row tiles ---
    ctas.assign(G, Cta{});
    std::vector<uint64_t> st1(G, 0);
    for (uint32_t c = 0; c < blocks.size(); ++c) {
      const Block1& b = blocks[c];
      Cta& C = ctas[c];
      C.s1_seg = (uint16_t)b.seg;
      C.s1_rt0 = b.rt0;
      C.s1_rtn = (uint16_t)b.rtn;
      C.s1_sl0 = (uint16_t)b.sl0;
      C.s1_sln = (uint16_t)b.sln;
      uint64_t bytes = 0;
      for (uint32_t q = b.sl0; q < b.sl0 + b.sln; ++q) bytes += u1[q];
      st1[c] = bytes * b.rtn + (uint64_t)(quant_bytes * 256.0 * b.sln);
    }
    // ---- stage-2 row tiles: every CTA's total cost close to the mean --------
    // CTA ranges per segment proportional to stage-2 bytes, then largest-
    // remainder allocation inside a range with weight (mean - stage-1 cost).
    double W = 0;
    for (uint32_t c = 0; c < G; ++c) W += (double)st1[c];
    for (uint32_t s = 0; s < count; ++s) W += (double)B2[s];
    const double mean = W / G;
    std::vector<uint32_t> cta0(count + 1, 0);
    {
      uint64_t B2tot = 0;
      for (uint32_t s = 0; s < count; ++s) B2tot += B2[s];
      double acc = 0;
      for (uint32_t s = 0; s < count; ++s) {
        acc += (double)B2[s];
        cta0[s + 1] = (uint32_t)std::llround(acc / std::max<double>(B2tot, 1) * G);
        cta0[s + 1] = std::max(cta0[s + 1], cta0[s] + 1);
      }
      cta0[count] = G;
      for (int s = (int)count - 1; s >= 0; --s) cta0[s] = std::min(cta0[s], cta0[s + 1] - 1);
    }
    bool placed = cta0[0] == 0;
    for (uint32_t s = 0; s < count && placed; ++s) {
      const uint32_t c0 = cta0[s], c1 = cta0[s + 1], nc = c1 - c0;
      std::vector<double> w(nc);
      double ws = 0;
      for (uint32_t i = 0; i < nc; ++i) {
        w[i] = std::max(0.0, mean - (double)st1[c0 + i]);
        ws += w[i];
      }
      if (ws <= 0)
        for (uint32_t i = 0; i < nc; ++i) w[i] = 1.0, ws += 1.0;
      std::vector<uint32_t> k(nc);
      std::vector<std::pair<double, uint32_t>> rem(nc);
      uint32_t given = 0;
      for (uint32_t i = 0; i < nc; ++i) {
        const double x = w[i] / ws * RT2[s];
        k[i] = std::min<uint32_t>((uint32_t)std::floor(x), max_rt);
        rem[i] = {x - k[i], i};
        given += k[i];
      }
      std::sort(rem.begin(), rem.end(), [](auto& x, auto& y) { return x.first > y.first; });
      for (uint32_t pass = 0; given < RT2[s] && pass < 2 * max_rt; ++pass)
        for (auto& pr : rem) {
          if (given >= RT2[s]) break;
          if (k[pr.second] < max_rt) {
            k[pr.second]++;
            given++;
          }
        }
      if (given < RT2[s]) {
        placed = false;
        break;
      }
      uint32_t next = 0;
      for (uint32_t i = 0; i < nc; ++i) {
        Cta& C = ctas[c0 + i];
        C.s2_seg = (uint16_t)s;
        C.s2_rt0 = next;
        C.s2_rtn = (uint16_t)k[i];
        next += k[i];
      }
    }
    if (placed) break;
  }

  // ---- streams, sections, shared-memory footprint --------------------------
  auto* g = new nqb_group();
  g->device = ctx->device;
  g->nseg = count;
  g->m = m;
  g->R1 = R1;
  g->grid = G;
  g->pass_only = pass_only;
  for (uint32_t s = 0; s < count; ++s) g->layers[s] = layers[s];
  uint64_t off = 0, max_stream = 0;
  uint32_t bfrag = 0;
  std::vector<uint64_t> sbytes(G);
  for (uint32_t s = 0; s < count; ++s)
    bfrag = std::max(bfrag, kBytesPerK * kpad(layers[s]->r));
  for (uint32_t c = 0; c < G; ++c) {
    Cta& C = ctas[c];
    C.stream_off = off;
    uint32_t nsec = 0;
    uint64_t bytes = 0;
    if (C.s1_rtn) {
      for (uint32_t q = C.s1_sl0; q < C.s1_sl0 + C.s1_sln; ++q, ++nsec) bytes += C.s1_rtn * u1[q];
      const uint32_t klo = slab_of(m, C.s1_sl0).k0;
      const Slab last = slab_of(m, C.s1_sl0 + C.s1_sln - 1);
      bfrag = std::max(bfrag, kBytesPerK * (last.k0 + 32 * last.nq - klo));
    }
    if (C.s2_rtn) {
      const uint32_t r = layers[C.s2_seg]->r;
      for (uint32_t q = 0, ns = nslabs(r); q < ns; ++q, ++nsec)
        bytes += (uint64_t)C.s2_rtn * unit_bytes(slab_of(r, q).nq);
    }
    NQB_REQUIRE(nsec < 65536, NQB_E_DIMENSION_MISMATCH, "too many decode sections");
    C.nsec = (uint16_t)nsec;
    sbytes[c] = bytes;
    off += bytes;
    max_stream = std::max(max_stream, bytes);
  }
  g->stream_bytes = off;
  g->big = max_stream >= (uint64_t)env_u32("NQB_DEC_BIG_KB", 0) * 1024;
  // Stream buffer: the whole per-CTA stream when it fits the cap (linear mode:
  // every copy issued up front, one mbarrier per section); otherwise the CTA
  // streams through fixed slots (ring mode).
  // The buffer takes whatever shared memory the head and the B fragments leave
  // (NQB_DEC_SMEM_KB caps it lower, e.g. to force ring mode in tests); a ring
  // slot is one section (<= kMaxRt * 512 B = 16 KB), so at least 10 slots fit
  // and any layer size streams (no upload is refused for size).
  constexpr uint32_t kMaxBars = 64;
  const uint32_t bfrag_pad = (bfrag + 127) / 128 * 128;
  const uint32_t avail = (227u * 1024u - head_bytes(kMaxBars) - bfrag_pad) / 128 * 128;
  const uint32_t env_cap = env_u32("NQB_DEC_SMEM_KB", 0) * 1024;
  const uint32_t cap = env_cap ? std::min(env_cap, avail) : avail;
  uint32_t buf = (uint32_t)std::min<uint64_t>((max_stream + 127) / 128 * 128, cap);
  uint32_t slot = 0, nbar = 2;  // linear mode: one mbarrier per stage
  for (uint32_t c = 0; c < G; ++c) {
    Cta& C = ctas[c];
    C.ring = sbytes[c] > buf ? 1 : 0;
  }
  for (uint32_t c = 0; c < G; ++c) {
    const Cta& C = ctas[c];
    if (!C.ring) continue;
    uint32_t q = 0;
    if (C.s1_rtn)
      for (uint32_t s = C.s1_sl0; s < C.s1_sl0 + C.s1_sln; ++s)
        slot = std::max<uint32_t>(slot, C.s1_rtn * u1[s]);
    if (C.s2_rtn)
      for (uint32_t r = layers[C.s2_seg]->r, ns = nslabs(r); q < ns; ++q)
        slot = std::max<uint32_t>(slot, C.s2_rtn * unit_bytes(slab_of(r, q).nq));
  }
  if (slot) {
    slot = (slot + 127) / 128 * 128;
    buf = std::max<uint32_t>(std::min(buf / slot, kMaxBars), pass_only ? 2 : 0) * slot;
    NQB_REQUIRE(pass_only || buf / slot >= 2, NQB_E_DIMENSION_MISMATCH,
                "decode ring needs two slots (NQB_DEC_SMEM_KB too small)");
    nbar = std::max<uint32_t>(nbar, buf / slot);
  }
  g->buf_bytes = buf;
  g->slot_bytes = slot;
  g->nbar = nbar;
  g->bfrag_bytes = (bfrag + 127) / 128 * 128;
  const uint32_t head = head_bytes(nbar);  // decode.cuh
  g->smem_bytes = head + g->bfrag_bytes + buf;
  // a pass-only plan (larger CTA blocks, pass_build) is never run by the per-call
  // kernel, so its per-call shared-memory footprint does not matter
  NQB_REQUIRE(pass_only || g->smem_bytes <= 227 * 1024, NQB_E_DIMENSION_MISMATCH,
              "decode plan exceeds shared memory (" + std::to_string(g->smem_bytes) + " B)");

  // ---- device buffers --------------------------------------------------------
  try {
    NQB_CUDA(cudaMalloc(&g->bits, std::max<uint64_t>(off, 16)));
    g->ctas = new Cta[G];
    std::copy(ctas.begin(), ctas.end(), g->ctas);
    Cta* dctas = nullptr;
    NQB_CUDA(cudaMallocAsync(&dctas, sizeof(Cta) * G, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(dctas, ctas.data(), sizeof(Cta) * G, cudaMemcpyHostToDevice,
                             ctx->stream));
    Seg* dsegs = nullptr;
    uint32_t* dmax = nullptr;
    NQB_CUDA(cudaMallocAsync(&dsegs, sizeof(Seg) * kMaxSeg, ctx->stream));
    NQB_CUDA(cudaMallocAsync(&dmax, 4 * kMaxSeg, ctx->stream));
    NQB_CUDA(cudaMemsetAsync(dmax, 0, 4 * kMaxSeg, ctx->stream));
    RelayoutSrc src{};
    for (uint32_t s = 0; s < count; ++s) {
      const nqb_layer* L = layers[s];
      Seg& S = g->seg[s];
      S.n = L->n;
      S.r = L->r;
      S.t_off = toff[s];
      S.s1h = L->s1h;
      S.s2h = L->s2h;
      g->n[s] = L->n;
      g->r[s] = L->r;
      src.u[s] = L->u;
      src.vt[s] = L->vt;
      src.u_words[s] = L->u_words;
      src.vt_words[s] = L->vt_words;
      k_absmax_half<<<std::min<uint32_t>(64, ceil_div(m, 256)), 256, 0, ctx->stream>>>(
          L->s2h, m, dmax + s);
      NQB_LAUNCHED(ctx);
    }
    NQB_CUDA(cudaMemcpyAsync(dsegs, g->seg, sizeof(Seg) * kMaxSeg, cudaMemcpyHostToDevice,
                             ctx->stream));
    k_relayout<<<G, 256, 0, ctx->stream>>>(dctas, dsegs, m, src, (uint32_t*)g->bits,
                                           pass_only ? 1 : 0);
    NQB_LAUNCHED(ctx);
    uint32_t hmax[kMaxSeg] = {0};
    NQB_CUDA(cudaMemcpyAsync(hmax, dmax, 4 * kMaxSeg, cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaFreeAsync(dsegs, ctx->stream));
    NQB_CUDA(cudaFreeAsync(dctas, ctx->stream));
    NQB_CUDA(cudaFreeAsync(dmax, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    for (uint32_t s = 0; s < count; ++s)
      g->seg[s].s2max = (float)host_half_to_double((uint16_t)hmax[s]);
    if (!pass_only) dec_state_reserve(ctx, R1);
  } catch (...) {
    group_free(g);
    throw;
  }
  return g;
}

void group_free(nqb_group* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  cudaFree(g->bits);
  delete[] g->ctas;
  delete g;
}

}  // namespace nqb
