// decode_pass.cuh — the persistent decode-pass kernel.
//
// A decode pass is a list of steps; a step is one decode group (1..kMaxSeg
// layers that read the same input, e.g. q/k/v) with its input x and outputs y.
// One launch of k_decode_pass runs every step of the pass on a grid of one CTA
// per SM:
//   * a producer warp per CTA streams the CTA's bits for step after step
//     (the same per-group plans and byte streams as the per-call kernel,
//     decode_plan.cu) into a shared-memory ring, in chunks of whole sections,
//     running ahead of the consumers across steps and barriers: the weights do
//     not depend on x, so HBM never waits for the layer chain;
//   * 16 consumer warps run, per step, stage 1 (x -> t, int64 red.add into a
//     per-step t region), a grid barrier, stage 2 (t -> y);
//   * a step whose input is an earlier step's output (found from the buffer
//     ranges at build time) waits for that step's output barrier; a step that
//     is independent of its predecessor has its stage 1 run before the
//     predecessor's stage 2 (one-step lookahead), so the barrier latency hides
//     behind MMA work;
//   * the output barrier also publishes max|y| per segment, which the consumer
//     step uses as its activation bound (no pass over x).
// All per-step accumulators live in a pass arena and are cleared by the kernel
// itself once every CTA is done with them, so the pass replays (directly or in
// a CUDA graph) with no host work.  Barrier targets come from a launch
// generation word, so counters never need resetting.
#pragma once
#include "decode.cuh"

namespace nqb {
namespace dec {

constexpr int kPassSlots = 16;  // ring chunks in flight (full/empty mbarrier pairs)
constexpr int kDescSlots = 4;   // step descriptors in flight
constexpr int kCtrStride = 16;  // u64 words per counter (own 128-byte line)

enum : uint32_t {
  kStepXF32 = 1u,        // x is fp32 (else binary16)
  kStepYF32 = 2u,        // y is fp32
  kStepXVec = 4u,        // x 16-byte aligned
  kStepPublish = 8u,     // a later step reads this step's output: output barrier + max|y|
  kStepLookahead = 16u,  // the next step's stage 1 runs before this step's stage 2
};

// Per-step arena region (int64 words): t rows [R1] | abs_a[kMaxSeg] | ea[kMaxSeg] | nonfinite
constexpr int kStepTail = 2 * kMaxSeg + 1;

struct alignas(16) StepDesc {
  const uint8_t* bits;   // the group's stream buffer
  const Cta* ctas;       // pass-grid entries of this step (device)
  const void* x;
  void* y[kMaxSeg];
  Seg seg[kMaxSeg];
  uint32_t nseg, m, R1, flags;
  int32_t x_src;         // output barrier to pass before stage 1 (-1: none)
  int32_t xmax_src;      // ymax word (step * kMaxSeg + seg) bounding |x| (-1: read x)
  uint64_t t_off;        // this step's arena region (int64 index)
  uint64_t zero_off;     // region of step k-2, cleared after this step's t barrier
  uint32_t zero_len;     // int64 words in it (0: none)
  uint32_t pad;
};
static_assert(sizeof(StepDesc) <= 480, "a step descriptor is copied by one warp (16 B per lane)");
constexpr uint32_t kDescBytes = (sizeof(StepDesc) + 15) / 16 * 16;
constexpr uint32_t kDescSlotBytes = 512;  // descriptor + the CTA's 32-byte Cta entry

struct PassParams {
  const StepDesc* desc;
  uint32_t K, G;
  unsigned long long* ctr;  // [0] generation, [kCtrStride] exit, then t / y barriers per step
  unsigned* ymax;           // K * kMaxSeg float bits (max |y| of published steps)
  long long* arena;
  uint32_t ring_bytes, bfrag_bytes, chunk_cap;
  uint32_t ntail;           // arena regions cleared after the exit barrier (last two steps)
  uint64_t tail_off[2];
  uint32_t tail_len[2];
  unsigned long long* trace;  // diagnostics: G x (2K + 2) %globaltimer stamps, or null
};

__host__ __device__ __forceinline__ uint32_t pass_head_bytes() {
  return (8 * (2 * kPassSlots + 2 * kDescSlots) + kDescSlots * kDescSlotBytes + 256 + 64 + 64 +
          kRedBytes + 127) / 128 * 128;
}

}  // namespace dec
}  // namespace nqb

// A built decode pass (nqb_pass in the C ABI).
struct nqb_pass {
  int device = 0;
  uint32_t K = 0, G = 0;
  uint32_t smem_bytes = 0;
  nqb::dec::PassParams params{};
  void* dmem = nullptr;  // descriptors, CTA tables, counters, ymax, arena (one allocation)
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
}  // namespace nqb
