// decode_pass.cuh — the persistent decode-pass kernel.
//
// A decode pass is a list of steps; a step is one decode group (1..kMaxSeg
// layers that read the same input, e.g. q/k/v) with its input x and outputs y.
// One launch of k_decode_pass runs every step of the pass on a grid of one CTA
// per SM.  The consumer warps only compute from shared memory; every global
// round trip lives in a helper warp that runs ahead of them:
//   * producer: streams the CTA's weight bits for phase after phase (the same
//     per-group plans and byte streams as the per-call kernel, decode_plan.cu)
//     into a shared-memory ring, ahead of the consumers across steps and
//     barriers: the weights do not depend on x, so HBM never waits for the
//     layer chain;
//   * x stager: per step, waits for the step's input (the producing step's
//     output barrier, if any), then TMA-copies the CTA's x slice and the
//     |x| bound into an x slot;
//   * t loader: per step, polls the step's t barrier and TMA-copies the t rows
//     of the CTA's stage-2 segment into a t slot; clears the other parity's
//     accumulators for the next launch;
//   * sequencer: turns consumer progress into the grid-barrier arrivals
//     (release reductions) and prefetches step descriptors.
// The consumers run, per step, stage 1 (x -> t, int64 red.add into the step's
// t region) and stage 2 (t -> y) in a host-computed phase order: stage 1 of up
// to `lookahead` later steps runs before a step's stage 2, so the t barrier and
// t load hide behind MMA work; a step that depends on an earlier output (found
// from the buffer ranges at build time) never moves ahead of it.
// |x| bounds: an independent input is reduced by a prepass at kernel start (one
// grid barrier for all steps); a chained input takes the producing step's
// published max|y|.  Accumulators and bounds are double-buffered by launch
// parity and the kernel clears the other parity itself, so the pass replays
// (directly or in a CUDA graph) with no host work.
#pragma once
#include "decode.cuh"

namespace nqb {
namespace dec {

constexpr int kPassSlots = 16;   // weight ring chunks in flight (full/empty mbarrier pairs)
constexpr int kDescSlots = 12;   // step descriptors in flight
constexpr int kXSlots = 3;       // staged x slices in flight
constexpr int kMaxTSlots = 6;    // staged t segments in flight (runtime count: PassParams::tslots)
constexpr int kDoneRing = 24;    // consumer phase-completion mbarriers
constexpr int kCtrStride = 16;   // u64 words per counter (own 128-byte line)
constexpr int kPassHelpers = 5;  // producer, x stager, t loader, sequencers 1 and 2
constexpr int kPassStamps = 16;  // trace stamps per step
constexpr int kMaxLookahead = 6;

enum : uint32_t {
  kStepXF32 = 1u,      // x is fp32 (else binary16)
  kStepYF32 = 2u,      // y is fp32
  kStepXVec = 4u,      // x 16-byte aligned
  kStepPublish = 8u,   // a later step reads this step's output: output barrier + max|y|
  kStepXPre = 16u,     // |x| bound from the kernel-start prepass
  kStepXSelf = 32u,    // |x| bound computed by the x stager after the dependency
};

struct alignas(16) StepDesc {
  const uint8_t* bits;   // the group's stream buffer
  const Cta* ctas;       // pass-grid entries of this step (device)
  const void* x;
  void* y[kMaxSeg];
  Seg seg[kMaxSeg];
  uint32_t nseg, m, R1, flags;
  int32_t x_src;         // output barrier to pass before staging x (-1: none)
  int32_t y_src;         // earlier step writing an overlapping output: its barrier gates stage 2
  uint32_t amax_idx;     // 16-byte bound word (per parity) holding max|x|
  uint64_t t_off;        // this step's t region (int64 index, even)
  uint32_t t_len;        // int64 words in the region (even)
  uint32_t s1_ahead;     // stage-1 sections the producer issues before this step's stage 2
  uint32_t pad[3];
};
static_assert(sizeof(StepDesc) % 16 == 0 && sizeof(StepDesc) <= 480, "step descriptor layout");
constexpr uint32_t kDescSlotBytes = 512;  // descriptor + the CTA's 32-byte Cta entry at 480

struct PassParams {
  const StepDesc* desc;
  const Cta* ctas;            // K x G
  uint32_t K, G;
  unsigned long long* ctr;    // [0] generation, [kCtrStride] prepass, then t / y barriers
  unsigned* amax;             // 2 parities x amax_words x 4 (16-byte words, max bits in [0])
  long long* arena;           // 2 parities x arena_len int64
  uint64_t arena_len;
  uint32_t amax_words;
  uint32_t ring1_bytes, ring2_bytes;     // stage-1 / stage-2 weight rings
  uint32_t chunk1_cap, chunk2_cap;
  uint32_t bfrag1_bytes, bfrag2_bytes;   // B fragments of x (stage 1) and t (stage 2)
  uint32_t xslot_bytes, tslot_bytes;
  uint32_t red1_bytes, red2_bytes;       // per-limb row sums (row tiles of the largest stage)
  uint32_t xs2_off;           // s2 slice offset in an x slot (header 16 B, then the x slice)
  uint32_t ts1_off;           // s1 slice offset in a t slot (after the t rows)
  uint32_t tslots;            // t slots (2..kMaxTSlots)
  uint32_t has_pre;
  uint32_t debug;  // NQB_PASS_DEBUG bits (experiments only): 1 skip MMA, 2 skip quantise, 4 suspend
                   // waits, 8 skip publish/outputs, 16 skip the t copy
  unsigned long long* trace;  // diagnostics: G x (kPassStamps K + 2) %globaltimer stamps
};

constexpr int kGroupWarps = 6;                 // consumer warps per stage group
constexpr int kGroupThreads = 32 * kGroupWarps;
constexpr uint32_t kPassBars =
    4 * kPassSlots + 2 * kDescSlots + 2 * kXSlots + 2 * kMaxTSlots + 2 * kDoneRing;
// head: mbarriers | misc | descriptor slots | group partials | max|x| ring |
// chunk records (2 rings)
__host__ __device__ __forceinline__ uint32_t pass_head_bytes() {
  return (8 * kPassBars + 64 + kDescSlots * kDescSlotBytes + 256 + 64 + 2 * 16 * kPassSlots + 127) /
         128 * 128;
}

}  // namespace dec
}  // namespace nqb

// A built decode pass (nqb_pass in the C ABI).
struct nqb_pass {
  int device = 0;
  uint32_t K = 0, G = 0;
  uint32_t smem_bytes = 0;
  nqb::dec::PassParams params{};
  void* dmem = nullptr;  // descriptors, CTA tables, counters, bounds, arena (one allocation)
  uint64_t stream_bytes = 0;   // bits streamed per launch
  uint64_t algo_bytes = 0;     // algorithmic bytes per launch
};

namespace nqb {
struct PassStepIn {
  const nqb_group* group;
  const void* x;
  void* y[dec::kMaxSeg];
  int f32;
};
nqb_pass* pass_build(nqb_context* ctx, uint32_t K, const PassStepIn* steps);
void pass_launch(nqb_context* ctx, const nqb_pass* p, unsigned long long* trace);
void pass_free(nqb_pass* p);
uint32_t pass_trace_words(const nqb_pass* p);  // nqb_debug_pass_trace stamps
}  // namespace nqb
