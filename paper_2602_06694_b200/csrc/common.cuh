// common.cuh — shared internals of libnqb (B200 / sm_100a only).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <map>
#include <vector>

#include "nqb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libnqb is written for sm_100a (B200) only"
#endif

namespace nqb {

// ---------------------------------------------------------------------------
// Status plumbing: every C-ABI entry point catches nqb::Failure and returns
// its code; the message goes to a thread-local buffer (nqb_last_error).
// ---------------------------------------------------------------------------
struct Failure {
  int code;
  std::string msg;
};

void set_error(const std::string& msg);
[[noreturn]] void fail(int code, const std::string& msg);

#define NQB_CUDA(call)                                                           \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess) {                                                     \
      cudaGetLastError(); /* clear a non-sticky error so later checks are clean */ \
      ::nqb::fail(e_ == cudaErrorMemoryAllocation ? NQB_E_OUT_OF_MEMORY : NQB_E_CUDA, \
                  std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +    \
                      __FILE__ + ":" + std::to_string(__LINE__));                \
    }                                                                            \
  } while (0)

#define NQB_REQUIRE(cond, code, msg) \
  do {                               \
    if (!(cond)) ::nqb::fail(code, msg); \
  } while (0)

// Kernel launch bookkeeping: every kernel launch goes through NQB_LAUNCHED so
// the context counts them (nqb_kernel_launches; bench.py reports it).
#define NQB_LAUNCHED(ctx)                                   \
  do {                                                      \
    NQB_CUDA(cudaGetLastError());                           \
    (ctx)->launches++;                                      \
  } while (0)

// ---------------------------------------------------------------------------
// Device scratch arena owned by a context (grows, never shrinks).
// ---------------------------------------------------------------------------
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace nqb

struct nqb_context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;     // active stream
  cudaStream_t own_stream = nullptr;  // created by nqb_create
  uint64_t launches = 0;
  nqb::Scratch scratch[16];
  unsigned* barrier = nullptr;  // grid-barrier words (zeroed), 64 entries
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // decode GEMV state (decode.cu): dec::State followed by 2 x dec_cap int64 rows
  void* dec_state = nullptr;
  uint32_t dec_cap = 0;
  std::vector<void*> dec_retired;  // outgrown decode states (graphs may still use them)
  bool dec_attr_set = false;
  bool pdl = true;  // launch decode kernels with Programmatic Dependent Launch
  void* dec_trace = nullptr;  // diagnostics (nqb_debug_decode_trace)
  // host ranges registered with nqb_host_register: base -> (bytes, device alias,
  // whether the library page-locked it)
  struct HostRange {
    size_t bytes;
    char* dev;
    bool ours;
  };
  std::map<uintptr_t, HostRange> host_ranges;
  // page-locked host staging (ctx_pinned): job lists of nqb_pass_run_host
  void* pinned[2] = {nullptr, nullptr};
  size_t pinned_bytes[2] = {0, 0};
};

struct nqb_group;

// Device-resident factorized layer.  Layout:
//   vt  : r rows x vt_words u32 — V^T, bit (k, j) = sign of V[j][k]; row k is
//         all m inputs, LSB-first, zero padded to a 16-byte row multiple
//   u   : n rows x u_words u32  — U as in the reference (bits along r), rows
//         padded to 16 bytes
//   s1h : n binary16, s2h : m binary16
struct nqb_layer {
  uint32_t n = 0, m = 0, r = 0;
  uint32_t vt_words = 0;  // words per V^T row (multiple of 4)
  uint32_t u_words = 0;   // words per U row (multiple of 4)
  uint32_t* vt = nullptr;
  uint32_t* u = nullptr;
  __half* s1h = nullptr;
  __half* s2h = nullptr;
  // exact fp64 scales (nqb_layer_upload_exact: the C++ drop-in's FactorizedLayer
  // keeps double scales in memory, packed.hpp:57-72); the exact paths
  // (reconstruct, gemv/gemm f64, gemv f32 host) use them when present
  double* s1d = nullptr;
  double* s2d = nullptr;
  int device = 0;
  nqb_group* dec = nullptr;  // decode plan of this layer alone (decode.cuh)
  float* hp_buf = nullptr;  // host drop-in path (nqb_gemv_f32_host): device x, y staging
};

namespace nqb {

// Returns a device buffer of at least `bytes` from slot `slot` of the arena.
void* scratch(nqb_context* ctx, int slot, size_t bytes);
// A page-locked host buffer of at least `bytes` (slot 0 or 1) owned by the context.
void* ctx_pinned(nqb_context* ctx, int slot, size_t bytes);
// One copy of a batch moved by a single kernel (nqb_pass_run_host).
struct CopyJob {
  void* dst;
  const void* src;
  size_t bytes;
};
void copy_jobs(nqb_context* ctx, const std::vector<CopyJob>& jobs, int slot);
// Device alias of a page-locked host address: the registry (nqb_host_register)
// first, else one cudaPointerGetAttributes probe; nullptr for pageable memory.
void* host_alias(nqb_context* ctx, const void* p, size_t bytes);

inline uint32_t ceil_div(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }
inline uint32_t round_up(uint32_t a, uint32_t b) { return (a + b - 1) / b * b; }

// IEEE binary16 RNE from double via float (same rounding chain as the
// reference's double_to_half: double -> float (RNE) -> half (RNE)).
uint16_t host_double_to_half(double x);
double host_half_to_double(uint16_t h);

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction tree (deterministic).  `red` must hold
// blockDim.x/32 elements.  Result is broadcast to every thread.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = T(0);
  for (int w = 0; w < nw; ++w) s += red[w];  // same order in every thread
  return s;
}

// Software grid barrier for persistent kernels whose grid is fully
// co-resident (cudaLaunchCooperativeKernel).  A monotonic 64-bit arrival
// counter (reset to 0 before each launch): each block adds 1 with acq_rel
// semantics and waits with acquire loads until the counter reaches k * G for
// its k-th barrier.  One atomic per block and barrier, no generation word.
// (A two-level counter tree measured slower on B200.)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned nblocks, unsigned& k) {
  __syncthreads();
  ++k;
  if (threadIdx.x == 0) {
    unsigned long long* ctr = (unsigned long long*)bar;
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    const unsigned long long target = (unsigned long long)k * nblocks;
    unsigned long long cur, spins = 0;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      // Watchdog: ~seconds of waiting means the grid diverged; trap so the
      // launch fails with an error instead of hanging the device.
      if (++spins > (1ull << 28)) __trap();
    }
  }
  __syncthreads();
}

}  // namespace nqb
