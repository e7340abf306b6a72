// decode.cuh — the batch-1 BLR decode GEMV on sm_100a.
//
// y = s1 .* U (V^T (s2 .* x))  (gemv_two_stage, packed.cpp:153-192)
//
// The signs are consumed as {0,1} bits: sum_j sign_j a_j = 2 sum_j bit_j a_j -
// sum_j a_j.  Activations are quantised once per call to 38-bit fixed point
// against a power-of-two bound from max|x| (kFix), split into six signed 8-bit limbs
// and fed to the tensor cores as the B operand of `mma.sync m16n8k32 u8.s8`;
// the bits are the A operand, expanded in registers with ONE LOP3 per four
// bits: tile q of a 256-wide K slab uses A bytes {0, 2^q} (word & 0x01010101<<q)
// and B limbs of (value << (7-q)), so every tile contributes 2^7 * bit * value
// to the same int32 accumulators.  All accumulation is exact integer
// arithmetic, so the result is bitwise deterministic and independent of the
// work split; the only rounding is the 38-bit quantisation of a and of t.
//
// One launch computes both stages.  CTA c streams one contiguous byte range of
// the plan's bit buffer (its stage-1 sections, then its stage-2 sections)
// through a shared-memory ring filled by a producer warp with 1-D TMA bulk
// copies; the first ring-full is issued before griddepcontrol.wait, so under
// Programmatic Dependent Launch it overlaps the previous kernel.  Stage-1
// partial sums are int64 red.add'ed into a global t accumulator; a grid
// barrier (all CTAs co-resident: grid <= #SMs) separates the stages.
#pragma once
#include <cstddef>

#include "common.cuh"

namespace nqb {
namespace dec {

constexpr int kMaxSeg = 4;         // layers sharing one input per launch
#ifndef NQB_DEC_WARPS
#define NQB_DEC_WARPS 16
#endif
constexpr int kConsumerWarps = NQB_DEC_WARPS;  // + 1 producer warp
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kThreads = kConsumerThreads + 32;
constexpr int kMaxRt = 32;         // 16-row tiles per CTA per stage (4 per consumer warp)
constexpr int kMaxSlabs1 = 16;     // stage-1 K slabs per CTA (4096 inputs)
constexpr int kFix = 38;           // activations and t in 38-bit fixed point
constexpr int kLimbs = 6;          // signed 8-bit limbs of (value << (7-q)) <= 2^45
constexpr int kMaxGrid = 160;      // CTA table lives in the kernel parameters
constexpr int kTileB = kLimbs * 32;    // B-fragment bytes per 32-wide K tile
constexpr int kBytesPerK = kLimbs;     // B-fragment bytes per input
constexpr int kRedStride = 8;          // ints per row of the per-limb row sums
constexpr int kSc2Elems = kMaxSlabs1 * 256;  // stage-1 input scales (s2) staged per CTA
constexpr int kSc1Elems = kMaxRt * 16;       // stage-2 output scales (s1) staged per CTA

// Shared-memory head: [full nbar][empty nbar][scale mbarrier, 16 B][red8 256 B][xmax 64 B]
// [red kMaxRt*16*kRedStride ints][s2 slice][s1 slice], then B fragments and the
// stream buffer.  The scale slices arrive by TMA ahead of griddepcontrol.wait.
constexpr uint32_t kRedBytes = kMaxRt * 16 * kRedStride * 4;
__host__ __device__ __forceinline__ uint32_t head_bytes(uint32_t nbar) {
  return (16 * nbar + 16 + 256 + 64 + kRedBytes + 2 * kSc2Elems + 2 * kSc1Elems + 127) / 128 *
         128;
}

// ---- K slabs: 256-wide (8 tiles of 32), then a 128 tail, then a 64 tail ----
struct Slab {
  uint32_t k0;
  uint32_t nq;  // tiles of 32 in the slab: 8, 4 or 2
};
// K = 256 F + rem, rem in {0, 64, 128, 192} after padding K to a multiple of 64
__host__ __device__ __forceinline__ void slab_split(uint32_t K, uint32_t& F, uint32_t& rem) {
  F = K / 256;
  rem = ((K - 256 * F) + 63) / 64 * 64;
  if (rem == 256) {
    F += 1;
    rem = 0;
  }
}
__host__ __device__ __forceinline__ uint32_t kpad(uint32_t K) {
  uint32_t F, rem;
  slab_split(K, F, rem);
  return 256 * F + rem;
}
__host__ __device__ __forceinline__ uint32_t nslabs(uint32_t K) {
  uint32_t F, rem;
  slab_split(K, F, rem);
  return F + (rem >= 128 ? 1u : 0u) + ((rem & 64) ? 1u : 0u);
}
__host__ __device__ __forceinline__ Slab slab_of(uint32_t K, uint32_t s) {
  uint32_t F, rem;
  slab_split(K, F, rem);
  if (s < F) return {256 * s, 8};
  if (rem >= 128 && s == F) return {256 * F, 4};
  return {256 * F + (rem >= 128 ? 128u : 0u), 2};
}
// bytes of one 16-row unit of a slab with nq tiles (16 bits per lane per tile)
__host__ __device__ __forceinline__ uint32_t unit_bytes(uint32_t nq) { return 64 * nq; }

// ---- plan -------------------------------------------------------------------
struct Cta {                 // one CTA's work (32 bytes)
  uint64_t stream_off;       // byte offset of its stream in Params::bits
  uint32_t s1_rt0;           // stage-1 row tiles [rt0, rt0+rtn) of segment s1_seg
  uint16_t s1_rtn, s1_seg;
  uint16_t s1_sl0, s1_sln;   // stage-1 slabs of K = m
  uint16_t s2_seg, s2_rtn;   // stage-2 row tiles [rt0, rt0+rtn) of segment s2_seg
  uint32_t s2_rt0;
  uint16_t nsec;             // sections in the stream (s1_sln if s1_rtn else 0, + slabs of r)
  uint16_t ring;             // 1: stream longer than the buffer, streamed through slots
};
static_assert(sizeof(Cta) == 32, "Cta layout");

struct Seg {
  uint32_t n, r;
  uint32_t t_off;            // first row of this segment in the t accumulator
  uint32_t pad;
  const __half* s1h;         // n scales (s_out)
  const __half* s2h;         // m scales (s_in)
  float s2max;               // max |s2| (fixes the activation exponent)
  float pad2;
};

// Per-context decode state (device memory).  The arrival counters, which
// every CTA hits with atomics and polls, live in their own 128-byte lines so
// the epoch/dirty loads and the abs_a reads do not queue behind them at L2.
struct alignas(128) State {
  uint32_t epoch;            // selects the t buffer (epoch & 1)
  uint32_t dirty[2];         // rows of t[b] that may be non-zero
  uint32_t pad0[29];
  long long abs_a[2][kMaxSeg];  // sum_j |a_int_j| per segment (bounds |t_k|)
  uint32_t pad1[16];
  struct alignas(128) Counter {
    uint32_t v;
    uint32_t pad[31];
  } done[2];                 // grid-barrier arrival counters
};
static_assert(sizeof(State) == 512, "State layout");

struct Params {
  const uint8_t* bits;
  Seg seg[kMaxSeg];
  uint32_t nseg, m;
  uint32_t R1;               // rows of the t accumulator used by this plan
  uint32_t r_cap;            // rows per t buffer
  State* st;
  long long* T;              // t accumulators: 2 x r_cap int64
  uint32_t buf_bytes;        // shared-memory stream buffer
  uint32_t slot_bytes;       // ring mode: slot size (buf_bytes / slot_bytes slots)
  uint32_t nbar;             // mbarrier pairs (max sections of a linear CTA, or slots)
  uint32_t bfrag_bytes;
  uint32_t x_f32, y_f32, x_vec;
  uint32_t seq;              // linear mode: issue stage-2 copies once stage 1 has landed
  const void* x;
  void* y[kMaxSeg];
  unsigned long long* trace;  // diagnostics (nqb_debug_decode_trace), or null
  Cta ctas[kMaxGrid];
};


}  // namespace dec
}  // namespace nqb

// A decode plan: the bits of 1..kMaxSeg layers that share one input, laid out
// for the kernel above, with the per-CTA work table.
struct nqb_group {
  int device = 0;
  uint32_t nseg = 0, m = 0, R1 = 0, grid = 0;
  uint32_t buf_bytes = 0, slot_bytes = 0, nbar = 0, bfrag_bytes = 0, smem_bytes = 0;
  uint64_t stream_bytes = 0;
  bool big = false;                    // long per-CTA streams: pipelined MMA instance
  bool pass_only = false;              // planned for k_decode_pass only (pass_build)
  const nqb_layer* layers[nqb::dec::kMaxSeg] = {nullptr};  // the planned layers (re-planning)
  uint8_t* bits = nullptr;             // device, stream_bytes
  nqb::dec::Cta* ctas = nullptr;       // host copy of the CTA table (grid entries)
  nqb::dec::Seg seg[nqb::dec::kMaxSeg];
  uint32_t n[nqb::dec::kMaxSeg] = {0}, r[nqb::dec::kMaxSeg] = {0};
};

namespace nqb {
// decode_plan.cu
// grid_cap / max_rt: 0 = the context's SMs / kMaxRt.  pass_only: a plan for the
// decode-pass kernel only: row-tile blocks above kMaxRt and the pair-major
// stream layout (k_relayout); group_gemv refuses it.
nqb_group* group_build(nqb_context* ctx, const nqb_layer* const* layers, uint32_t count,
                       uint32_t grid_cap = 0, uint32_t max_rt = 0, bool pass_only = false,
                       uint32_t plan_slabs = 0);
void group_free(nqb_group* g);
// decode.cu
void group_gemv(nqb_context* ctx, const nqb_group* g, const void* d_x, int x_f32,
                void* const* d_ys, int y_f32);
void dec_state_reserve(nqb_context* ctx, uint32_t rows);
}  // namespace nqb
