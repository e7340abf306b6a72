// decode_pass.cuh — the persistent decode-pass kernel.
//
// A decode pass is a list of steps; a step is one decode group (1..kMaxSeg
// layers that read the same input, e.g. q/k/v) with its input x and outputs y.
// One launch of k_decode_pass runs every step of the pass on a grid of one CTA
// per SM.  The consumer warps only run MMAs from shared memory and finish rows;
// every global round trip and all input quantisation live in helper warps that
// run ahead of them:
//   * producers (one per stage): stream the CTA's weight bits step after step
//     (the same per-group plans and byte streams as the per-call kernel,
//     decode_plan.cu) into that stage's shared-memory ring.  The weights do not
//     depend on x, so HBM never waits for the layer chain, and the two rings
//     fill independently;
//   * x quantisers (2 warps): per step, wait for the step's input (the producing
//     step's output barrier, if any), read the CTA's x and s2 slices from global
//     memory and write a = s2*x as 38-bit fixed-point B fragments (+ their sum)
//     into a stage-1 slot;
//   * t quantisers (2 warps): per step, poll the step's t barrier, read the t
//     rows of the CTA's stage-2 segment and write them as B fragments (+ sum, +
//     the s1 slice) into a stage-2 slot; clear the other parity's accumulators
//     for the next launch;
//   * sequencers: turn consumer progress into the grid-barrier arrivals
//     (release reductions) and prefetch step descriptors.
// The consumers form two groups: group 0 runs stage 1 of step after step (x ->
// t, int64 red.add into the step's t region), group 1 stage 2 (t -> y).  Group 0
// runs ahead of group 1 as far as the descriptor ring allows, so the t barrier
// of a step completes while group 1 still works on earlier steps.
// |x| bounds: an independent input is reduced by a prepass at kernel start (one
// grid barrier for all steps); a chained input takes the producing step's
// published max|y|.  Accumulators and bounds are double-buffered by launch
// parity and the kernel clears the other parity itself, so the pass replays
// (directly or in a CUDA graph) with no host work.
#pragma once
#include <vector>

#include "decode.cuh"

namespace nqb {
namespace dec {

constexpr int kPassSlots = 16;   // weight ring chunks in flight (full/empty mbarrier pairs)
constexpr int kDescSlots = 12;   // step descriptors in flight
constexpr int kBSlots = 2;       // quantised-input slots per stage (B fragments of x / t)
constexpr int kDoneRing = 24;    // consumer phase-completion mbarriers
constexpr int kCtrStride = 16;   // u64 words per counter (own 128-byte line)
// helper warps: producer 1, x quantisers (2), t quantisers (2), sequencers 1 and 2, producer 2
constexpr int kPassHelpers = 8;
constexpr int kPassStamps = 24;  // trace stamps per step (16..21: consumer chunk-wait / run counters, per stage)
constexpr int kMaxLookahead = 6;
constexpr int kMaxSub = 16;      // SM partitions of a pass (independent steps run concurrently)
constexpr uint32_t kPassMaxRt = 1024;  // row tiles per CTA per stage in a partition's plan (no shared row sums)
constexpr uint32_t kBSlotHead = 16;  // slot header: the two quantiser warps' sums of the values

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
  uint32_t idx;          // the step's index in the pass (barriers, bounds, trace)
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
  uint32_t wave_div;          // a stage-1 ring chunk holds (group warps) / wave_div work items
  uint32_t wave_div2;         // a stage-2 ring chunk holds (group warps) / wave_div2 row tiles
  uint32_t l2_ahead;          // producers prefetch a step's stage bytes into L2 this many steps ahead
  uint32_t bslot1_bytes, bslot2_bytes;   // quantised-input slots: header | B fragments (| s1)
  uint32_t bs2_s1_off;        // s1 slice offset in a stage-2 slot (after the t fragments)
  uint32_t warps1;            // consumer warps of the stage-1 group (4 or 6; the rest run stage 2)
  uint32_t has_pre;
  uint32_t pre_units;         // most 8-element units of one step's input in a CTA's prepass share
  // SM partitions: CTAs [i P, (i+1) P) run the steps list[list_off[i] .. list_off[i+1])
  // (one partition of G CTAs unless every step is independent, pass_build)
  const uint32_t* list;
  uint32_t nsub, P;
  uint32_t list_off[kMaxSub + 1];
  uint32_t debug;  // NQB_PASS_DEBUG bits (experiments only): 1 skip MMA, 2 skip quantise, 4 suspend
                   // waits, 8 skip publish/outputs, 32 no weight copies
  unsigned long long* trace;  // diagnostics: G x (kPassStamps K + 2) %globaltimer stamps
};

// the kConsumerWarps consumer warps form a stage-1 group (PassParams::warps1) and a
// stage-2 group
constexpr uint32_t kPassBars = 4 * kPassSlots + 2 * kDescSlots + 4 * kBSlots + 2 * kDoneRing;
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
  // step inputs and layer outputs (nqb_pass_run_host)
  std::vector<void*> x_dev, y_dev;
  std::vector<size_t> x_bytes, y_bytes;
  std::vector<nqb_group*> owned;  // partition plans built for this pass (freed with it)
  std::vector<uint8_t> desc_host;  // the step descriptors as uploaded (nqb_pass_io patches y)
};

namespace nqb {
struct PassStepIn {
  const nqb_group* group;
  const void* x;
  void* y[dec::kMaxSeg];
  int f32;
};
nqb_pass* pass_build(nqb_context* ctx, uint32_t K, const PassStepIn* steps);
// desc_override: a patched copy of the step descriptors (nqb_pass_io: outputs
// written straight to mapped host memory), or null
void pass_launch(nqb_context* ctx, const nqb_pass* p, unsigned long long* trace,
                 const void* desc_override = nullptr);
void pass_free(nqb_pass* p);
uint32_t pass_trace_words(const nqb_pass* p);  // nqb_debug_pass_trace stamps
}  // namespace nqb
