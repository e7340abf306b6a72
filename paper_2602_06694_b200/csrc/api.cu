// api.cu — extern "C" entry points of libnqb (include/nqb.h): context,
// packing, layers and the forward.  ADMM entry points live in admm.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "decode.cuh"
#include "decode_pass.cuh"

namespace nqb {

// pack.cu
void launch_binarize(nqb_context*, const double*, double*, uint64_t, int*);
void launch_pack_rows(nqb_context*, const double*, uint32_t, uint32_t, uint32_t*, int, int*);
void launch_check_padding(nqb_context*, const uint32_t*, uint32_t, uint32_t, uint32_t, int*);
void launch_unpack(nqb_context*, const uint32_t*, uint32_t, uint32_t, double*);
void launch_bit_transpose(nqb_context*, const uint32_t*, uint32_t, uint32_t, uint32_t,
                          uint32_t*, uint32_t);
void launch_reconstruct(nqb_context*, const nqb_layer*, const uint32_t*, uint32_t, double*);
void launch_rel_error(nqb_context*, const nqb_layer*, const uint32_t*, uint32_t, const double*,
                      double*, double*, const double* = nullptr, const double* = nullptr);
uint64_t rel_error_partial_count(const nqb_layer*);
// forward_simt.cu
template <typename Acc, typename In>
void simt_gemv(nqb_context*, const nqb_layer*, const In*, Acc*);
void simt_gemm_f64(nqb_context*, const nqb_layer*, const double*, uint32_t, double*);
// decode.cu / prefill_tc.cu
void decode_gemv_f32(nqb_context*, const nqb_layer*, const float*, float*);
void decode_gemv_f16(nqb_context*, const nqb_layer*, const __half*, __half*);
void prefill_gemm_tc(nqb_context*, const nqb_layer*, const __half*, uint32_t, __half*);

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

void* scratch(nqb_context* ctx, int slot, size_t bytes) {
  Scratch& s = ctx->scratch[slot];
  if (s.bytes < bytes) {
    if (s.ptr) NQB_CUDA(cudaFreeAsync(s.ptr, ctx->stream));
    s.ptr = nullptr;
    s.bytes = 0;
    const size_t want = bytes < 256 ? 256 : bytes;
    NQB_CUDA(cudaMallocAsync(&s.ptr, want, ctx->stream));
    s.bytes = want;
  }
  return s.ptr;
}

void* ctx_pinned(nqb_context* ctx, int slot, size_t bytes) {
  if (ctx->pinned_bytes[slot] < bytes) {
    if (ctx->pinned[slot]) {
      NQB_CUDA(cudaStreamSynchronize(ctx->stream));
      NQB_CUDA(cudaFreeHost(ctx->pinned[slot]));
    }
    ctx->pinned[slot] = nullptr;
    ctx->pinned_bytes[slot] = 0;
    const size_t want = bytes < 65536 ? 65536 : bytes;
    NQB_CUDA(cudaHostAlloc(&ctx->pinned[slot], want, cudaHostAllocDefault));
    ctx->pinned_bytes[slot] = want;
  }
  return ctx->pinned[slot];
}

void* host_alias(nqb_context* ctx, const void* p, size_t bytes) {
  const uintptr_t a = (uintptr_t)p;
  auto it = ctx->host_ranges.upper_bound(a);
  if (it != ctx->host_ranges.begin()) {
    --it;
    if (a >= it->first && a + bytes <= it->first + it->second.bytes)
      return it->second.dev + (a - it->first);
  }
  cudaPointerAttributes at{};
  void* dev = nullptr;
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost)
    dev = at.devicePointer;
  cudaGetLastError();
  return dev;
}

uint16_t host_double_to_half(double x) {
  const __half h = __float2half_rn((float)x);
  uint16_t bits;
  std::memcpy(&bits, &h, 2);
  return bits;
}

double host_half_to_double(uint16_t bits) {
  __half_raw raw;
  raw.x = bits;
  return (double)__half2float(__half(raw));
}

// RAII device buffer on the context stream.
struct DevBuf {
  nqb_context* ctx;
  void* p = nullptr;
  DevBuf(nqb_context* c, size_t bytes) : ctx(c) {
    if (bytes) NQB_CUDA(cudaMallocAsync(&p, bytes, ctx->stream));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, ctx->stream);
  }
  template <typename T>
  T* as() const { return (T*)p; }
};

// Device-side flag word read back synchronously.
struct Flags {
  nqb_context* ctx;
  int* d;
  explicit Flags(nqb_context* c) : ctx(c) {
    d = (int*)scratch(ctx, 7, 64);
    NQB_CUDA(cudaMemsetAsync(d, 0, sizeof(int), ctx->stream));
  }
  int read() {
    int h = 0;
    NQB_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
  }
};

void check_ctx(nqb_context* ctx) {
  NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
  NQB_CUDA(cudaSetDevice(ctx->device));
}

void check_layer(const nqb_layer* L) {
  NQB_REQUIRE(L != nullptr, NQB_E_VALIDATION, "null layer");
}

}  // namespace nqb

using namespace nqb;

#define API_BEGIN try {
#define API_END                   \
  return NQB_OK;                  \
  }                               \
  catch (const Failure& f) {      \
    set_error(f.msg);             \
    return f.code;                \
  }                               \
  catch (const std::exception& e) { \
    set_error(e.what());          \
    return NQB_E_INTERNAL;        \
  }

extern "C" {

int nqb_status_kind(int status) {
  if (status == NQB_OK) return 0;
  if (status < 32) return 1;
  if (status < 64) return 2;
  return 3;
}

const char* nqb_last_error(void) { return g_last_error.c_str(); }

const char* nqb_version(void) {
#ifdef NQB_GIT_DESCRIBE
  return "libnqb sm_100a " NQB_GIT_DESCRIBE;
#else
  return "libnqb sm_100a";
#endif
}

int nqb_create(int device, nqb_context** out) {
  API_BEGIN
  NQB_REQUIRE(out != nullptr, NQB_E_VALIDATION, "null output");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(NQB_E_NO_DEVICE, "no CUDA device: libnqb has no CPU path");
  }
  NQB_REQUIRE(device >= 0 && device < count, NQB_E_NO_DEVICE, "device index out of range");
  NQB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  NQB_CUDA(cudaGetDeviceProperties(&prop, device));
  NQB_REQUIRE(prop.major == 10, NQB_E_NO_DEVICE,
              std::string("libnqb needs an sm_100 (B200) device, found ") + prop.name);
  auto* ctx = new nqb_context();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  NQB_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  NQB_CUDA(cudaMalloc(&ctx->barrier, 64 * sizeof(unsigned)));
  NQB_CUDA(cudaMemset(ctx->barrier, 0, 64 * sizeof(unsigned)));
  NQB_CUDA(cudaEventCreate(&ctx->ev0));
  NQB_CUDA(cudaEventCreate(&ctx->ev1));
  *out = ctx;
  API_END
}

int nqb_destroy(nqb_context* ctx) {
  API_BEGIN
  if (!ctx) return NQB_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& s : ctx->scratch)
    if (s.ptr) cudaFree(s.ptr);
  if (ctx->barrier) cudaFree(ctx->barrier);
  for (void* p : ctx->pinned)
    if (p) cudaFreeHost(p);
  for (auto& kv : ctx->host_ranges)
    if (kv.second.ours) cudaHostUnregister((void*)kv.first);
  if (ctx->dec_state) cudaFree(ctx->dec_state);
  for (void* p : ctx->dec_retired) cudaFree(p);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  API_END
}

int nqb_host_register(nqb_context* ctx, void* ptr, size_t bytes) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(ptr != nullptr && bytes > 0, NQB_E_VALIDATION, "empty host range");
  bool ours = false;
  cudaPointerAttributes at{};
  if (!(cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost)) {
    cudaGetLastError();
    NQB_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterMapped));
    ours = true;
    NQB_CUDA(cudaPointerGetAttributes(&at, ptr));
  }
  NQB_REQUIRE(at.devicePointer != nullptr, NQB_E_VALIDATION, "host range has no device mapping");
  ctx->host_ranges[(uintptr_t)ptr] = nqb_context::HostRange{bytes, (char*)at.devicePointer, ours};
  API_END
}

int nqb_host_unregister(nqb_context* ctx, void* ptr) {
  API_BEGIN
  check_ctx(ctx);
  auto it = ctx->host_ranges.find((uintptr_t)ptr);
  NQB_REQUIRE(it != ctx->host_ranges.end(), NQB_E_VALIDATION, "host range was not registered");
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  if (it->second.ours) NQB_CUDA(cudaHostUnregister(ptr));
  ctx->host_ranges.erase(it);
  API_END
}

int nqb_set_stream(nqb_context* ctx, void* stream) {
  API_BEGIN
  check_ctx(ctx);
  const cudaStream_t next = stream ? (cudaStream_t)stream : ctx->own_stream;
  if (next == ctx->stream) return NQB_OK;
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->stream = next;
  API_END
}

void* nqb_get_stream(nqb_context* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int nqb_synchronize(nqb_context* ctx) {
  API_BEGIN
  check_ctx(ctx);
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

uint64_t nqb_kernel_launches(const nqb_context* ctx) { return ctx ? ctx->launches : 0; }

int nqb_set_sm_budget(nqb_context* ctx, int sms) {
  API_BEGIN
  check_ctx(ctx);
  cudaDeviceProp prop;
  NQB_CUDA(cudaGetDeviceProperties(&prop, ctx->device));
  ctx->num_sms = (sms <= 0 || sms > prop.multiProcessorCount) ? prop.multiProcessorCount : sms;
  API_END
}

// storage.cpp:124-141 (host arithmetic; no device work).
int nqb_rank_for_target_bpw(uint64_t n, uint64_t m, double t, uint32_t* rank) {
  API_BEGIN
  NQB_REQUIRE(n > 0 && m > 0, NQB_E_VALIDATION, "layer dims must be positive");
  NQB_REQUIRE(t > 0.0, NQB_E_TARGET_TOO_SMALL, "target BPW must be positive");
  const double nm = (double)n * (double)m;
  const long long rounded = std::llround(t * nm / (double)(n + m) - 16.0);
  if (rounded < 1) {
    const double bpw1 = (double)(17 * (n + m)) / (double)(n * m);
    NQB_REQUIRE(!(bpw1 > 2.0 * t), NQB_E_TARGET_TOO_SMALL,
                "even rank 1 overshoots the target by more than 2x");
    *rank = 1;
    return NQB_OK;
  }
  const uint64_t cap = n < m ? n : m;
  *rank = (uint32_t)((uint64_t)rounded < cap ? (uint64_t)rounded : cap);
  API_END
}

// Rng (rng.hpp:25-58): splitmix64; gaussian() = Box-Muller on two uniforms,
// one value per call.  Draw j of the stream returns mix(seed + (j+1)*golden), so
// gaussian i starts at draw 2i unless a uniform of 0 was rejected earlier
// (probability 2^-53 per value): threads fill independent ranges by jumping
// ahead, and any range that sees a rejection makes the whole fill sequential.
namespace {
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
inline uint64_t splitmix_next(uint64_t& state) {
  uint64_t z = (state += kGolden);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline double rng_uniform(uint64_t& state) { return (double)(splitmix_next(state) >> 11) * 0x1.0p-53; }
// One gaussian; returns false if the first uniform was rejected (<= 0).
inline bool rng_gaussian(uint64_t& state, double* g) {
  double u1 = rng_uniform(state);
  bool clean = true;
  while (u1 <= 0.0) {
    clean = false;
    u1 = rng_uniform(state);
  }
  const double u2 = rng_uniform(state);
  *g = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  return clean;
}
inline double weight_value(double g, double scale, int snap_f32) {
  const double w = scale * g;
  return snap_f32 ? (double)(float)w : w;
}
}  // namespace

int nqb_synthetic_weight_host(uint64_t seed, uint64_t count, double scale, int snap_f32,
                              double* out) {
  API_BEGIN
  NQB_REQUIRE(out != nullptr || count == 0, NQB_E_VALIDATION, "null output");
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t T = count < (1u << 16) ? 1 : std::min<uint64_t>(hw, 64);
  std::atomic<int> dirty{0};
  auto fill = [&](uint64_t a, uint64_t b) {
    uint64_t st = seed + 2 * a * kGolden;
    for (uint64_t i = a; i < b; ++i) {
      double g;
      if (!rng_gaussian(st, &g)) dirty = 1;
      out[i] = weight_value(g, scale, snap_f32);
    }
  };
  std::vector<std::thread> pool;
  for (uint64_t t = 1; t < T; ++t) pool.emplace_back(fill, count * t / T, count * (t + 1) / T);
  fill(0, count / T);
  for (auto& th : pool) th.join();
  if (dirty && T > 1) {  // a rejected uniform shifts the stream: redo it in order
    uint64_t st = seed;
    for (uint64_t i = 0; i < count; ++i) {
      double g;
      rng_gaussian(st, &g);
      out[i] = weight_value(g, scale, snap_f32);
    }
  }
  API_END
}

// ---------------------------------------------------------------------------
// binarize / pack / unpack
// ---------------------------------------------------------------------------
int nqb_binarize(nqb_context* ctx, const double* latent, uint64_t count, double* out,
                 int on_device) {
  API_BEGIN
  check_ctx(ctx);
  Flags flags(ctx);
  if (on_device) {
    launch_binarize(ctx, latent, out, count, flags.d);
  } else {
    DevBuf buf(ctx, 2 * count * sizeof(double));
    double* din = buf.as<double>();
    NQB_CUDA(cudaMemcpyAsync(din, latent, count * 8, cudaMemcpyHostToDevice, ctx->stream));
    launch_binarize(ctx, din, din + count, count, flags.d);
    NQB_CUDA(cudaMemcpyAsync(out, din + count, count * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  NQB_REQUIRE(!(flags.read() & 1), NQB_E_NON_FINITE_INPUT, "binarize: non-finite input");
  API_END
}

static int pack_impl(nqb_context* ctx, const double* in, uint32_t rows, uint32_t cols,
                     uint32_t* words, int on_device, int latent) {
  API_BEGIN
  check_ctx(ctx);
  Flags flags(ctx);
  const uint64_t elems = (uint64_t)rows * cols;
  const uint64_t nwords = (uint64_t)rows * ceil_div(cols, 32);
  if (on_device) {
    launch_pack_rows(ctx, in, rows, cols, words, latent, flags.d);
  } else {
    DevBuf buf(ctx, elems * 8 + nwords * 4);
    double* din = buf.as<double>();
    uint32_t* dw = (uint32_t*)(din + elems);
    NQB_CUDA(cudaMemcpyAsync(din, in, elems * 8, cudaMemcpyHostToDevice, ctx->stream));
    launch_pack_rows(ctx, din, rows, cols, dw, latent, flags.d);
    NQB_CUDA(cudaMemcpyAsync(words, dw, nwords * 4, cudaMemcpyDeviceToHost, ctx->stream));
  }
  const int f = flags.read();
  NQB_REQUIRE(!(f & 1), NQB_E_NON_FINITE_INPUT, "pack: non-finite latent");
  NQB_REQUIRE(!(f & 2), NQB_E_NON_BINARY_ENTRY, "pack_signs: entries must be exactly +-1");
  API_END
}

int nqb_pack_signs(nqb_context* ctx, const double* signs, uint32_t rows, uint32_t cols,
                   uint32_t* words, int on_device) {
  return pack_impl(ctx, signs, rows, cols, words, on_device, 0);
}

int nqb_pack_latent(nqb_context* ctx, const double* latent, uint32_t rows, uint32_t cols,
                    uint32_t* words, int on_device) {
  return pack_impl(ctx, latent, rows, cols, words, on_device, 1);
}

int nqb_unpack_signs(nqb_context* ctx, const uint32_t* words, uint32_t rows, uint32_t cols,
                     double* signs, int on_device) {
  API_BEGIN
  check_ctx(ctx);
  Flags flags(ctx);
  const uint32_t wpr = ceil_div(cols, 32);
  const uint64_t elems = (uint64_t)rows * cols, nwords = (uint64_t)rows * wpr;
  if (on_device) {
    launch_check_padding(ctx, words, rows, cols, wpr, flags.d);
    NQB_REQUIRE(!(flags.read() & 4), NQB_E_CORRUPT_PADDING, "padding bits beyond cols are set");
    launch_unpack(ctx, words, rows, cols, signs);
  } else {
    const uint64_t wbytes = ((nwords * 4 + 15) / 16) * 16;
    DevBuf buf(ctx, wbytes + elems * 8);
    uint32_t* dw = buf.as<uint32_t>();
    double* dout = (double*)(buf.as<char>() + wbytes);
    NQB_CUDA(cudaMemcpyAsync(dw, words, nwords * 4, cudaMemcpyHostToDevice, ctx->stream));
    launch_check_padding(ctx, dw, rows, cols, wpr, flags.d);
    NQB_REQUIRE(!(flags.read() & 4), NQB_E_CORRUPT_PADDING, "padding bits beyond cols are set");
    launch_unpack(ctx, dw, rows, cols, dout);
    NQB_CUDA(cudaMemcpyAsync(signs, dout, elems * 8, cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  API_END
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Layers
// ---------------------------------------------------------------------------
namespace nqb {

// Builds a device layer from reference-layout words already on the device.
// d_u / d_v: n x wpr and m x wpr words (row stride wpr).
nqb_layer* layer_from_device_words(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                                   const uint32_t* d_u, const uint32_t* d_v,
                                   const __half* d_s1h, const __half* d_s2h) {
  const uint32_t wpr = ceil_div(r, 32);
  auto* L = new nqb_layer();
  L->n = n;
  L->m = m;
  L->r = r;
  L->device = ctx->device;
  L->u_words = round_up(wpr, 4);
  L->vt_words = round_up(ceil_div(m, 32), 4);
  try {
    NQB_CUDA(cudaMalloc(&L->u, (size_t)n * L->u_words * 4));
    NQB_CUDA(cudaMalloc(&L->vt, (size_t)r * L->vt_words * 4));
    // scales zero-padded to whole 64-element blocks: the decode kernel stages
    // slab-aligned slices of them with TMA bulk copies
    NQB_CUDA(cudaMalloc(&L->s1h, (size_t)round_up(n, 64) * 2));
    NQB_CUDA(cudaMalloc(&L->s2h, (size_t)round_up(m, 64) * 2));
    NQB_CUDA(cudaMemsetAsync(L->s1h, 0, (size_t)round_up(n, 64) * 2, ctx->stream));
    NQB_CUDA(cudaMemsetAsync(L->s2h, 0, (size_t)round_up(m, 64) * 2, ctx->stream));
    NQB_CUDA(cudaMemsetAsync(L->u, 0, (size_t)n * L->u_words * 4, ctx->stream));
    NQB_CUDA(cudaMemsetAsync(L->vt, 0, (size_t)r * L->vt_words * 4, ctx->stream));
    NQB_CUDA(cudaMemcpy2DAsync(L->u, L->u_words * 4, d_u, wpr * 4, wpr * 4, n,
                               cudaMemcpyDeviceToDevice, ctx->stream));
    launch_bit_transpose(ctx, d_v, m, r, wpr, L->vt, L->vt_words);
    NQB_CUDA(cudaMemcpyAsync(L->s1h, d_s1h, (size_t)n * 2, cudaMemcpyDeviceToDevice, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(L->s2h, d_s2h, (size_t)m * 2, cudaMemcpyDeviceToDevice, ctx->stream));
    const nqb_layer* one[1] = {L};
    L->dec = group_build(ctx, one, 1);  // the decode kernel's layout of the same bits
  } catch (...) {
    group_free(L->dec);
    cudaFree(L->u);
    cudaFree(L->vt);
    cudaFree(L->s1h);
    cudaFree(L->s2h);
    delete L;
    throw;
  }
  return L;
}

// Many small copies in one launch (nqb_pass_run_host): block b takes jobs b,
// b + grid, ...; 16-byte vectors when both ends and the size allow.
__global__ void k_copy_jobs(const CopyJob* __restrict__ jobs, uint32_t count) {
  for (uint32_t j = blockIdx.x; j < count; j += gridDim.x) {
    const CopyJob J = jobs[j];
    const bool vec = (((uintptr_t)J.dst | (uintptr_t)J.src | J.bytes) & 15u) == 0;
    if (vec) {
      const uint4* s = (const uint4*)J.src;
      uint4* d = (uint4*)J.dst;
      for (size_t i = threadIdx.x; i < J.bytes / 16; i += blockDim.x) d[i] = s[i];
    } else {
      const uint8_t* s = (const uint8_t*)J.src;
      uint8_t* d = (uint8_t*)J.dst;
      for (size_t i = threadIdx.x; i < J.bytes; i += blockDim.x) d[i] = s[i];
    }
  }
}

void copy_jobs(nqb_context* ctx, const std::vector<CopyJob>& jobs, int slot) {
  if (jobs.empty()) return;
  const size_t bytes = jobs.size() * sizeof(CopyJob);
  // the job list goes up through a page-locked staging buffer of the context
  // (two slots: the input and the output list of one call can be in flight)
  CopyJob* host = (CopyJob*)ctx_pinned(ctx, slot, bytes);
  std::memcpy(host, jobs.data(), bytes);
  CopyJob* dev = (CopyJob*)scratch(ctx, 12 + slot, bytes);
  NQB_CUDA(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  k_copy_jobs<<<std::min<uint32_t>((uint32_t)jobs.size(), 4u * ctx->num_sms), 256, 0, ctx->stream>>>(
      dev, (uint32_t)jobs.size());
  NQB_LAUNCHED(ctx);
}

// V back to the reference orientation (m x stride words) in device memory.
void layer_v_reference(nqb_context* ctx, const nqb_layer* L, uint32_t* d_vr, uint32_t stride) {
  NQB_CUDA(cudaMemsetAsync(d_vr, 0, (size_t)L->m * stride * 4, ctx->stream));
  launch_bit_transpose(ctx, L->vt, L->r, L->m, L->vt_words, d_vr, stride);
}

}  // namespace nqb

extern "C" {

static int upload_impl(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                       const uint32_t* u_words, const uint32_t* v_words,
                       const uint16_t* s1h, const uint16_t* s2h, nqb_layer** out) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(out != nullptr, NQB_E_VALIDATION, "null output");
  *out = nullptr;
  NQB_REQUIRE(n > 0 && m > 0 && r > 0, NQB_E_DIMENSION_MISMATCH, "zero layer dimension");
  const uint32_t wpr = ceil_div(r, 32);
  const uint32_t tail = r % 32;
  if (tail) {  // unpack_signs' padding rule (packed.cpp:85-93), checked on upload
    const uint32_t pad = ~0u << tail;
    for (uint64_t i = 0; i < n; ++i)
      NQB_REQUIRE(!(u_words[i * wpr + wpr - 1] & pad), NQB_E_CORRUPT_PADDING,
                  "U: padding bits beyond r are set");
    for (uint64_t j = 0; j < m; ++j)
      NQB_REQUIRE(!(v_words[j * wpr + wpr - 1] & pad), NQB_E_CORRUPT_PADDING,
                  "V: padding bits beyond r are set");
  }
  const size_t ub = (size_t)n * wpr * 4, vb = (size_t)m * wpr * 4;
  DevBuf buf(ctx, ub + vb + 2 * (size_t)(n + m) + 16);
  uint32_t* du = buf.as<uint32_t>();
  uint32_t* dv = du + (size_t)n * wpr;
  __half* ds = (__half*)(dv + (size_t)m * wpr);
  NQB_CUDA(cudaMemcpyAsync(du, u_words, ub, cudaMemcpyHostToDevice, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(dv, v_words, vb, cudaMemcpyHostToDevice, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(ds, s1h, 2 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(ds + n, s2h, 2 * (size_t)m, cudaMemcpyHostToDevice, ctx->stream));
  *out = layer_from_device_words(ctx, n, m, r, du, dv, ds, ds + n);
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_layer_upload_f16(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                         const uint32_t* u_words, const uint32_t* v_words,
                         const uint16_t* s1_half, const uint16_t* s2_half, nqb_layer** out) {
  return upload_impl(ctx, n, m, r, u_words, v_words, s1_half, s2_half, out);
}

int nqb_layer_upload(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                     const uint32_t* u_words, const uint32_t* v_words, const double* s1,
                     const double* s2, nqb_layer** out) {
  std::vector<uint16_t> h1(n), h2(m);
  for (uint32_t i = 0; i < n; ++i) h1[i] = host_double_to_half(s1[i]);
  for (uint32_t j = 0; j < m; ++j) h2[j] = host_double_to_half(s2[j]);
  return upload_impl(ctx, n, m, r, u_words, v_words, h1.data(), h2.data(), out);
}

int nqb_layer_upload_exact(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                           const uint32_t* u_words, const uint32_t* v_words, const double* s1,
                           const double* s2, nqb_layer** out) {
  const int st = nqb_layer_upload(ctx, n, m, r, u_words, v_words, s1, s2, out);
  if (st != NQB_OK) return st;
  API_BEGIN
  nqb_layer* L = *out;
  try {
    NQB_CUDA(cudaMalloc(&L->s1d, 8 * ((size_t)n + m)));
    L->s2d = L->s1d + n;
    NQB_CUDA(cudaMemcpyAsync(L->s1d, s1, 8 * (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(L->s2d, s2, 8 * (size_t)m, cudaMemcpyHostToDevice, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    nqb_layer_free(L);
    *out = nullptr;
    throw;
  }
  API_END
}

int nqb_layer_free(nqb_layer* L) {
  API_BEGIN
  if (!L) return NQB_OK;
  cudaSetDevice(L->device);
  group_free(L->dec);
  cudaFree(L->s1d);  // s2d shares the allocation
  cudaFree(L->hp_buf);
  cudaFree(L->u);
  cudaFree(L->vt);
  cudaFree(L->s1h);
  cudaFree(L->s2h);
  delete L;
  API_END
}

int nqb_layer_shape(const nqb_layer* L, uint32_t* n, uint32_t* m, uint32_t* r) {
  API_BEGIN
  check_layer(L);
  if (n) *n = L->n;
  if (m) *m = L->m;
  if (r) *r = L->r;
  API_END
}

uint64_t nqb_layer_device_bytes(const nqb_layer* L) {
  if (!L) return 0;
  if (L->dec) return L->dec->stream_bytes + 2ull * (L->n + L->m);
  return (uint64_t)L->r * L->vt_words * 4 + (uint64_t)L->n * L->u_words * 4 +
         2ull * (L->n + L->m);
}

int nqb_layer_download(nqb_context* ctx, const nqb_layer* L, uint32_t* u_words,
                       uint32_t* v_words, double* s1, double* s2) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  const uint32_t wpr = ceil_div(L->r, 32);
  if (u_words) {
    NQB_CUDA(cudaMemcpy2DAsync(u_words, wpr * 4, L->u, L->u_words * 4, wpr * 4, L->n,
                               cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (v_words) {
    DevBuf buf(ctx, (size_t)L->m * wpr * 4);
    layer_v_reference(ctx, L, buf.as<uint32_t>(), wpr);
    NQB_CUDA(cudaMemcpyAsync(v_words, buf.p, (size_t)L->m * wpr * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if ((s1 || s2) && L->s1d) {  // exact scales
    if (s1) NQB_CUDA(cudaMemcpyAsync(s1, L->s1d, 8 * (size_t)L->n, cudaMemcpyDeviceToHost, ctx->stream));
    if (s2) NQB_CUDA(cudaMemcpyAsync(s2, L->s2d, 8 * (size_t)L->m, cudaMemcpyDeviceToHost, ctx->stream));
  } else if (s1 || s2) {
    std::vector<uint16_t> h1(L->n), h2(L->m);
    NQB_CUDA(cudaMemcpyAsync(h1.data(), L->s1h, 2 * (size_t)L->n, cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaMemcpyAsync(h2.data(), L->s2h, 2 * (size_t)L->m, cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (s1)
      for (uint32_t i = 0; i < L->n; ++i) s1[i] = host_half_to_double(h1[i]);
    if (s2)
      for (uint32_t j = 0; j < L->m; ++j) s2[j] = host_half_to_double(h2[j]);
  }
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

// ---------------------------------------------------------------------------
// Forward
// ---------------------------------------------------------------------------
int nqb_gemv_f32_device(nqb_context* ctx, const nqb_layer* L, const float* d_x, float* d_y) {
  API_BEGIN
  check_layer(L);
  decode_gemv_f32(ctx, L, d_x, d_y);
  API_END
}

int nqb_gemv_f16_device(nqb_context* ctx, const nqb_layer* L, const uint16_t* d_x,
                        uint16_t* d_y) {
  API_BEGIN
  check_layer(L);
  decode_gemv_f16(ctx, L, (const __half*)d_x, (__half*)d_y);
  API_END
}

int nqb_gemv_f32_host(nqb_context* ctx, const nqb_layer* L, const float* x, float* y) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  NQB_REQUIRE(x != nullptr && y != nullptr, NQB_E_VALIDATION, "null buffer");
  // per-layer device staging for x and y (no allocation on the per-token path)
  nqb_layer* ML = const_cast<nqb_layer*>(L);
  if (!ML->hp_buf)
    NQB_CUDA(cudaMalloc(&ML->hp_buf, 4 * ((size_t)round_up(L->m, 4) + L->n)));
  float* dx = ML->hp_buf;
  float* dy = dx + round_up(L->m, 4);
  if (L->s1d) {  // exact fp64 scales: gemv_two_stage<float> arithmetic on CUDA cores
    NQB_CUDA(cudaMemcpyAsync(dx, x, 4 * (size_t)L->m, cudaMemcpyHostToDevice, ctx->stream));
    simt_gemv<float, float>(ctx, L, dx, dy);
    NQB_CUDA(cudaMemcpyAsync(y, dy, 4 * (size_t)L->n, cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    return NQB_OK;
  }
  // A pinned (page-locked, mapped) y is written by the kernel directly over the
  // host link: no separate device-to-host copy.  Pageable y goes through dy.
  // Checked every call (a cached answer could outlive the allocation).
  // Registered ranges (nqb_host_register) are a map lookup; anything else is
  // probed once per call (a cached answer could outlive the allocation).
  float* y_dev = (float*)host_alias(ctx, y, 4 * (size_t)L->n);
  NQB_CUDA(cudaMemcpyAsync(dx, x, 4 * (size_t)L->m, cudaMemcpyHostToDevice, ctx->stream));
  if (y_dev) {
    decode_gemv_f32(ctx, L, dx, y_dev);
  } else {
    decode_gemv_f32(ctx, L, dx, dy);
    NQB_CUDA(cudaMemcpyAsync(y, dy, 4 * (size_t)L->n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_gemv_f64_host(nqb_context* ctx, const nqb_layer* L, const double* x, double* y) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  DevBuf buf(ctx, 8 * ((size_t)L->m + L->n));
  double* dx = buf.as<double>();
  double* dy = dx + L->m;
  NQB_CUDA(cudaMemcpyAsync(dx, x, 8 * (size_t)L->m, cudaMemcpyHostToDevice, ctx->stream));
  simt_gemv<double, double>(ctx, L, dx, dy);
  NQB_CUDA(cudaMemcpyAsync(y, dy, 8 * (size_t)L->n, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_gemm_f64_host(nqb_context* ctx, const nqb_layer* L, const double* x, uint32_t b,
                      double* y) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  if (b == 0) return NQB_OK;
  const size_t xb = (size_t)L->m * b * 8, yb = (size_t)L->n * b * 8;
  DevBuf buf(ctx, xb + yb);
  double* dx = buf.as<double>();
  double* dy = dx + (size_t)L->m * b;
  NQB_CUDA(cudaMemcpyAsync(dx, x, xb, cudaMemcpyHostToDevice, ctx->stream));
  simt_gemm_f64(ctx, L, dx, b, dy);
  NQB_CUDA(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_gemm_f16_device(nqb_context* ctx, const nqb_layer* L, const uint16_t* d_x, uint32_t b,
                        uint16_t* d_y) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  if (b == 0) return NQB_OK;
  prefill_gemm_tc(ctx, L, (const __half*)d_x, b, (__half*)d_y);
  API_END
}

int nqb_reconstruct_dense_host(nqb_context* ctx, const nqb_layer* L, double* w) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  const uint32_t wpr = ceil_div(L->r, 32);
  const size_t wb = (size_t)L->n * L->m * 8;
  DevBuf buf(ctx, wb + (size_t)L->m * L->u_words * 4);
  double* dw = buf.as<double>();
  uint32_t* dvr = (uint32_t*)(dw + (size_t)L->n * L->m);
  layer_v_reference(ctx, L, dvr, L->u_words);
  (void)wpr;
  launch_reconstruct(ctx, L, dvr, L->u_words, dw);
  NQB_CUDA(cudaMemcpyAsync(w, dw, wb, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_layer_rel_error(nqb_context* ctx, const nqb_layer* L, const double* w, int on_device,
                        double* rel_error) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  const size_t wb = on_device ? 0 : (size_t)L->n * L->m * 8;
  const uint64_t parts = rel_error_partial_count(L);
  DevBuf buf(ctx, wb + (size_t)L->m * L->u_words * 4 + parts * 16 + 64);
  char* base = buf.as<char>();
  const double* dw = on_device ? w : (const double*)base;
  if (!on_device) {
    NQB_CUDA(cudaMemcpyAsync((void*)dw, w, wb, cudaMemcpyHostToDevice, ctx->stream));
  }
  double* part = (double*)(base + wb);
  double* sums = part + 2 * parts;
  uint32_t* dvr = (uint32_t*)(sums + 2);
  layer_v_reference(ctx, L, dvr, L->u_words);
  launch_rel_error(ctx, L, dvr, L->u_words, dw, part, sums);
  double h[2];
  NQB_CUDA(cudaMemcpyAsync(h, sums, 16, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  const double num = std::sqrt(h[0]), den = std::sqrt(h[1]);
  *rel_error = den == 0.0 ? (num == 0.0 ? 0.0 : INFINITY) : num / den;
  API_END
}

// ---------------------------------------------------------------------------
// Decode groups (layers sharing one input) and CUDA graphs of decode passes
// ---------------------------------------------------------------------------
int nqb_group_create(nqb_context* ctx, const nqb_layer* const* layers, uint32_t count,
                     nqb_group** out) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(out != nullptr && layers != nullptr, NQB_E_VALIDATION, "null argument");
  *out = nullptr;
  *out = group_build(ctx, layers, count);
  API_END
}

int nqb_group_free(nqb_group* g) {
  API_BEGIN
  group_free(g);
  API_END
}

uint64_t nqb_group_stream_bytes(const nqb_group* g) { return g ? g->stream_bytes : 0; }

int nqb_group_gemv_f16_device(nqb_context* ctx, const nqb_group* g, const uint16_t* d_x,
                              uint16_t* const* d_ys) {
  API_BEGIN
  NQB_REQUIRE(ctx && g && d_ys, NQB_E_VALIDATION, "null argument");
  group_gemv(ctx, g, d_x, 0, (void* const*)d_ys, 0);
  API_END
}

int nqb_group_gemv_f32_device(nqb_context* ctx, const nqb_group* g, const float* d_x,
                              float* const* d_ys) {
  API_BEGIN
  NQB_REQUIRE(ctx && g && d_ys, NQB_E_VALIDATION, "null argument");
  group_gemv(ctx, g, d_x, 1, (void* const*)d_ys, 1);
  API_END
}

int nqb_debug_decode_trace(nqb_context* ctx, const nqb_layer* L, const uint16_t* d_x,
                           uint16_t* d_y, uint64_t* stamps, uint32_t* grid) {
  API_BEGIN
  check_ctx(ctx);
  check_layer(L);
  const uint32_t G = L->dec->grid;
  if (grid) *grid = G;
  NQB_CUDA(cudaMalloc(&ctx->dec_trace, 32 * 8 * (size_t)G));
  NQB_CUDA(cudaMemsetAsync(ctx->dec_trace, 0, 32 * 8 * (size_t)G, ctx->stream));
  try {
    void* ys[1] = {d_y};
    group_gemv(ctx, L->dec, d_x, 0, ys, 0);
    NQB_CUDA(cudaMemcpyAsync(stamps, ctx->dec_trace, 32 * 8 * (size_t)G, cudaMemcpyDeviceToHost,
                             ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFree(ctx->dec_trace);
    ctx->dec_trace = nullptr;
    throw;
  }
  cudaFree(ctx->dec_trace);
  ctx->dec_trace = nullptr;
  API_END
}

int nqb_pass_create(nqb_context* ctx, uint32_t count, const nqb_pass_step* steps,
                    nqb_pass** out) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(out != nullptr && steps != nullptr, NQB_E_VALIDATION, "null argument");
  *out = nullptr;
  std::vector<PassStepIn> in(count);
  for (uint32_t k = 0; k < count; ++k) {
    const nqb_pass_step& s = steps[k];
    const nqb_group* g = s.group;
    if (!g) {
      NQB_REQUIRE(s.layer != nullptr, NQB_E_VALIDATION, "pass step without group or layer");
      g = s.layer->dec;
    }
    in[k].group = g;
    in[k].x = s.d_x;
    for (int q = 0; q < dec::kMaxSeg; ++q) in[k].y[q] = s.d_y[q];
    in[k].f32 = s.f32;
  }
  *out = pass_build(ctx, count, in.data());
  API_END
}

int nqb_pass_launch(nqb_context* ctx, const nqb_pass* pass) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(pass != nullptr, NQB_E_VALIDATION, "null pass");
  pass_launch(ctx, pass, nullptr);
  API_END
}

int nqb_pass_free(nqb_pass* pass) {
  API_BEGIN
  pass_free(pass);
  API_END
}

// One pass end to end with host buffers: each non-NULL hx[k] is copied into
// step k's device input, the pass runs, each non-NULL hy[i] (one per layer of
// every step, in step order) receives that layer's output, and the call returns
// when the outputs are on the host.  Pinned host buffers make the copies
// asynchronous DMA; pageable ones go through the driver's staging.
}  // extern "C"

// Bound host I/O of a pass (nqb_pass_io_*): the copy lists live on the device.
struct nqb_pass_io {
  int device = 0;
  const nqb_pass* pass = nullptr;
  nqb::CopyJob* d_in = nullptr;
  nqb::CopyJob* d_out = nullptr;
  uint32_t n_in = 0, n_out = 0;
  void* d_desc = nullptr;  // descriptors with outputs redirected to mapped host memory (or null)
};

extern "C" {

int nqb_pass_io_create(nqb_context* ctx, const nqb_pass* pass, const void* const* hx,
                       void* const* hy, nqb_pass_io** out) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(pass != nullptr && out != nullptr, NQB_E_VALIDATION, "null argument");
  NQB_REQUIRE(pass->device == ctx->device, NQB_E_VALIDATION, "decode pass lives on another device");
  *out = nullptr;
  std::vector<CopyJob> in, outj;
  for (uint32_t k = 0; hx && k < pass->K; ++k) {
    if (!hx[k]) continue;
    void* mapped = host_alias(ctx, hx[k], pass->x_bytes[k]);
    NQB_REQUIRE(mapped != nullptr, NQB_E_VALIDATION,
                "pass io: host input is not page-locked or registered (use nqb_pass_run_host)");
    in.push_back(CopyJob{pass->x_dev[k], mapped, pass->x_bytes[k]});
  }
  // Outputs no later step reads are written by the pass straight into the mapped
  // host buffers (a patched copy of the step descriptors), overlapping the PCIe
  // writes with the pass; the others come back through the copy kernel.
  const bool direct = std::getenv("NQB_PASS_IO_DIRECT_Y") == nullptr ||
                      std::strtoul(std::getenv("NQB_PASS_IO_DIRECT_Y"), nullptr, 10) != 0;
  std::vector<uint8_t> patched = pass->desc_host;
  auto* D = (dec::StepDesc*)patched.data();
  bool any_direct = false;
  for (uint32_t k = 0, i = 0; k < pass->K; ++k) {
    for (uint32_t q = 0; q < D[k].nseg; ++q, ++i) {
      if (!hy || !hy[i]) continue;
      void* mapped = host_alias(ctx, hy[i], pass->y_bytes[i]);
      NQB_REQUIRE(mapped != nullptr, NQB_E_VALIDATION,
                  "pass io: host output is not page-locked or registered (use nqb_pass_run_host)");
      if (direct && !(D[k].flags & dec::kStepPublish)) {
        D[k].y[q] = mapped;
        any_direct = true;
      } else {
        outj.push_back(CopyJob{mapped, pass->y_dev[i], pass->y_bytes[i]});
      }
    }
  }
  auto* io = new nqb_pass_io();
  io->device = ctx->device;
  io->pass = pass;
  try {
    NQB_CUDA(cudaMalloc(&io->d_in, sizeof(CopyJob) * std::max<size_t>(in.size(), 1)));
    NQB_CUDA(cudaMalloc(&io->d_out, sizeof(CopyJob) * std::max<size_t>(outj.size(), 1)));
    if (!in.empty())
      NQB_CUDA(cudaMemcpy(io->d_in, in.data(), sizeof(CopyJob) * in.size(), cudaMemcpyHostToDevice));
    if (!outj.empty())
      NQB_CUDA(cudaMemcpy(io->d_out, outj.data(), sizeof(CopyJob) * outj.size(), cudaMemcpyHostToDevice));
    if (any_direct) {
      NQB_CUDA(cudaMalloc(&io->d_desc, patched.size()));
      NQB_CUDA(cudaMemcpy(io->d_desc, patched.data(), patched.size(), cudaMemcpyHostToDevice));
    }
  } catch (...) {
    cudaFree(io->d_in);
    cudaFree(io->d_out);
    cudaFree(io->d_desc);
    delete io;
    throw;
  }
  io->n_in = (uint32_t)in.size();
  io->n_out = (uint32_t)outj.size();
  *out = io;
  API_END
}

int nqb_pass_io_run(nqb_context* ctx, const nqb_pass_io* io) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(io != nullptr, NQB_E_VALIDATION, "null pass io");
  NQB_REQUIRE(io->device == ctx->device, NQB_E_VALIDATION, "pass io lives on another device");
  const uint32_t cap = 4u * (uint32_t)ctx->num_sms;
  if (io->n_in) {
    k_copy_jobs<<<std::min(io->n_in, cap), 256, 0, ctx->stream>>>(io->d_in, io->n_in);
    NQB_LAUNCHED(ctx);
  }
  pass_launch(ctx, io->pass, nullptr, io->d_desc);
  if (io->n_out) {
    k_copy_jobs<<<std::min(io->n_out, cap), 256, 0, ctx->stream>>>(io->d_out, io->n_out);
    NQB_LAUNCHED(ctx);
  }
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_pass_io_free(nqb_pass_io* io) {
  API_BEGIN
  if (io) {
    cudaSetDevice(io->device);
    cudaFree(io->d_in);
    cudaFree(io->d_out);
    cudaFree(io->d_desc);
    delete io;
  }
  API_END
}

int nqb_pass_run_host(nqb_context* ctx, const nqb_pass* pass, const void* const* hx,
                      void* const* hy) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(pass != nullptr, NQB_E_VALIDATION, "null pass");
  NQB_REQUIRE(pass->device == ctx->device, NQB_E_VALIDATION, "decode pass lives on another device");
  // A decode pass has hundreds of small inputs and outputs; one API call per
  // buffer would cost more host time than the kernel.  Page-locked host buffers
  // are moved by ONE copy kernel per direction that reads / writes them through
  // their mapped device addresses; pageable ones get one cudaMemcpyAsync each.
  std::vector<CopyJob> jobs;
  auto add = [&](void* dst, const void* src, size_t bytes, bool host_is_dst) {
    void* mapped = host_alias(ctx, host_is_dst ? dst : src, bytes);
    if (mapped) {
      jobs.push_back(host_is_dst ? CopyJob{mapped, src, bytes} : CopyJob{dst, mapped, bytes});
    } else {
      NQB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
    }
  };
  for (uint32_t k = 0; hx && k < pass->K; ++k)
    if (hx[k]) add(pass->x_dev[k], hx[k], pass->x_bytes[k], false);
  copy_jobs(ctx, jobs, 0);
  pass_launch(ctx, pass, nullptr);
  jobs.clear();
  for (size_t i = 0; hy && i < pass->y_dev.size(); ++i)
    if (hy[i]) add(hy[i], pass->y_dev[i], pass->y_bytes[i], true);
  copy_jobs(ctx, jobs, 1);
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

uint64_t nqb_pass_stream_bytes(const nqb_pass* pass) { return pass ? pass->stream_bytes : 0; }
uint64_t nqb_pass_algorithmic_bytes(const nqb_pass* pass) { return pass ? pass->algo_bytes : 0; }

int nqb_debug_pass_trace(nqb_context* ctx, const nqb_pass* pass, uint64_t* stamps,
                         uint32_t* grid) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(pass != nullptr && stamps != nullptr, NQB_E_VALIDATION, "null argument");
  if (grid) *grid = pass->G;
  const size_t words = pass_trace_words(pass);
  DevBuf buf(ctx, words * 8);
  NQB_CUDA(cudaMemsetAsync(buf.p, 0, words * 8, ctx->stream));
  pass_launch(ctx, pass, buf.as<unsigned long long>());
  NQB_CUDA(cudaMemcpyAsync(stamps, buf.p, words * 8, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  API_END
}

int nqb_set_pdl(nqb_context* ctx, int enable) {
  API_BEGIN
  check_ctx(ctx);
  ctx->pdl = enable != 0;
  API_END
}

}  // extern "C"

struct nqb_graph {
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

int nqb_graph_begin(nqb_context* ctx) {
  API_BEGIN
  check_ctx(ctx);
  NQB_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  API_END
}

int nqb_graph_end(nqb_context* ctx, nqb_graph** out) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(out != nullptr, NQB_E_VALIDATION, "null output");
  *out = nullptr;
  cudaGraph_t graph = nullptr;
  NQB_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
  auto* g = new nqb_graph();
  g->device = ctx->device;
  g->graph = graph;
  const cudaError_t e = cudaGraphInstantiate(&g->exec, graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(graph);
    delete g;
    NQB_CUDA(e);
  }
  *out = g;
  API_END
}

int nqb_graph_launch(nqb_context* ctx, const nqb_graph* g) {
  API_BEGIN
  check_ctx(ctx);
  NQB_REQUIRE(g != nullptr, NQB_E_VALIDATION, "null graph");
  NQB_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
  API_END
}

int nqb_graph_free(nqb_graph* g) {
  API_BEGIN
  if (!g) return NQB_OK;
  cudaSetDevice(g->device);
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  API_END
}

}  // extern "C"
