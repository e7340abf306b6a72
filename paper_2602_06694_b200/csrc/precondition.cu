// precondition.cu — phase 1 of the pipeline on the device:
// calibration statistics and W~ = D_out W D_in (precondition.cpp:37-141,
// pipeline.cpp:63-72), plus the inverse row scaling used by balance
// (unprecondition_rows, precondition.cpp:143-153).
//
// The O(samples x channels) work runs on the GPU in the reference's exact
// operation order: one thread per channel sums x^2 over the samples in order,
// with unfused multiply and add, and scaling uses w * (d_i * d_j).  Results are
// therefore bitwise equal to the reference.  The O(channels) parts (RMS,
// sort + quantile, clip/shrink) are host arithmetic.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace nqb {
namespace {

// batch: rows x cols row-major.  sq[j] = sum_i batch[i][j]^2 in row order;
// flags bit 0: a non-finite entry was seen.
__global__ void k_col_sumsq(const double* __restrict__ batch, uint64_t rows, uint32_t cols,
                            double* __restrict__ sq, int* __restrict__ flags) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  bool bad = false;
  for (uint64_t i = 0; i < rows; ++i) {
    const double x = batch[i * cols + j];
    bad |= !isfinite(x);
    s = __dadd_rn(s, __dmul_rn(x, x));  // precondition.cpp:49-51, no contraction
  }
  sq[j] = s;
  if (bad) atomicOr(flags, 1);
}

// w[i][j] *= d_out[i] * d_in[j]   (precondition.cpp:129-135; null diag = identity)
__global__ void k_scale_weight(double* __restrict__ w, uint32_t rows, uint32_t cols,
                               const double* __restrict__ d_out, const double* __restrict__ d_in) {
  const uint64_t total = (uint64_t)rows * cols;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(e / cols), j = (uint32_t)(e % cols);
    const double di = d_out ? d_out[i] : 1.0;
    w[e] = __dmul_rn(w[e], __dmul_rn(di, d_in ? d_in[j] : 1.0));
  }
}

// factor[i][j] *= 1 / diag[i]   (precondition.cpp:148-152)
__global__ void k_unscale_rows(double* __restrict__ f, uint32_t rows, uint32_t cols,
                               const double* __restrict__ diag) {
  const uint64_t total = (uint64_t)rows * cols;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(e / cols);
    f[e] = __dmul_rn(f[e], __ddiv_rn(1.0, diag[i]));
  }
}

uint32_t grid_for(uint64_t total) {
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148 * 16));
}

// quantile_sorted (precondition.cpp:22-33)
double quantile_sorted(const std::vector<double>& s, double p) {
  if (s.empty()) return 0.0;
  if (s.size() == 1) return s[0];
  const double pos = p * (double)(s.size() - 1);
  const size_t lo = (size_t)pos;
  const size_t hi = std::min(lo + 1, s.size() - 1);
  const double frac = pos - (double)lo;
  return s[lo] * (1.0 - frac) + s[hi] * frac;
}

// clipped_shrunk_diag (precondition.cpp:79-95)
void clipped_shrunk_diag(const double* sum_squares, uint64_t count, double tau, uint32_t c,
                         double gamma, double eps_floor, double* d) {
  for (uint32_t j = 0; j < c; ++j) d[j] = std::min(std::sqrt(sum_squares[j] / (double)count), tau);
  double mean = 0.0;
  for (uint32_t j = 0; j < c; ++j) mean += d[j];
  mean /= (double)c;
  for (uint32_t j = 0; j < c; ++j) {
    double x = (1.0 - gamma) * d[j] + gamma * mean;
    d[j] = std::max(x, eps_floor);
  }
}

// device batch -> per-column sums of squares (host vector); validates finiteness
std::vector<double> col_sumsq(nqb_context* ctx, const double* d_batch, uint64_t rows, uint32_t cols) {
  double* sq = (double*)scratch(ctx, 11, sizeof(double) * cols + 64);
  int* flags = (int*)(sq + cols);
  NQB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx->stream));
  k_col_sumsq<<<(cols + 127) / 128, 128, 0, ctx->stream>>>(d_batch, rows, cols, sq, flags);
  NQB_LAUNCHED(ctx);
  std::vector<double> h(cols);
  int hf = 0;
  NQB_CUDA(cudaMemcpyAsync(h.data(), sq, sizeof(double) * cols, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  NQB_REQUIRE(!(hf & 1), NQB_E_NON_FINITE_INPUT, "accumulate_stats");
  return h;
}

// accumulate_stats (precondition.cpp:37-62) given the batch's column sums of squares
void fold_stats(const std::vector<double>& batch_sq, uint64_t rows, double percentile,
                double* sum_squares, uint64_t* sample_count, double* tau) {
  const uint32_t c = (uint32_t)batch_sq.size();
  std::vector<double> rms(c);
  for (uint32_t j = 0; j < c; ++j) {
    rms[j] = std::sqrt(batch_sq[j] / (double)rows);
    sum_squares[j] += batch_sq[j];
  }
  *sample_count += rows;
  std::sort(rms.begin(), rms.end());
  *tau = std::max(*tau, quantile_sorted(rms, percentile));
}

void check_stats_args(uint32_t cols, double percentile, const double* sum_squares,
                      const uint64_t* sample_count, const double* tau) {
  NQB_REQUIRE(sum_squares && sample_count && tau, NQB_E_VALIDATION, "null stats");
  NQB_REQUIRE(percentile > 0.0 && percentile < 1.0, NQB_E_VALIDATION, "percentile must be in (0,1)");
  (void)cols;
}

}  // namespace
}  // namespace nqb

using namespace nqb;

#define PC_BEGIN try {
#define PC_END                      \
  return NQB_OK;                    \
  }                                 \
  catch (const Failure& e) {        \
    set_error(e.msg);               \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    set_error(e.what());            \
    return NQB_E_INTERNAL;          \
  }

extern "C" {

int nqb_accumulate_stats_device(nqb_context* ctx, const double* d_batch, uint64_t rows,
                                uint32_t cols, double percentile, double* sum_squares,
                                uint64_t* sample_count, double* tau) {
  PC_BEGIN
  NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
  check_stats_args(cols, percentile, sum_squares, sample_count, tau);
  if (rows == 0) return NQB_OK;  // precondition.cpp:45
  NQB_REQUIRE(d_batch != nullptr, NQB_E_VALIDATION, "null batch");
  NQB_CUDA(cudaSetDevice(ctx->device));
  fold_stats(col_sumsq(ctx, d_batch, rows, cols), rows, percentile, sum_squares, sample_count, tau);
  PC_END
}

int nqb_accumulate_stats_host(nqb_context* ctx, const double* batch, uint64_t rows, uint32_t cols,
                              double percentile, double* sum_squares, uint64_t* sample_count,
                              double* tau) {
  PC_BEGIN
  NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
  check_stats_args(cols, percentile, sum_squares, sample_count, tau);
  if (rows == 0) return NQB_OK;
  NQB_REQUIRE(batch != nullptr, NQB_E_VALIDATION, "null batch");
  NQB_CUDA(cudaSetDevice(ctx->device));
  const size_t bytes = sizeof(double) * rows * cols;
  double* d = nullptr;
  NQB_CUDA(cudaMallocAsync(&d, bytes, ctx->stream));
  try {
    NQB_CUDA(cudaMemcpyAsync(d, batch, bytes, cudaMemcpyHostToDevice, ctx->stream));
    fold_stats(col_sumsq(ctx, d, rows, cols), rows, percentile, sum_squares, sample_count, tau);
  } catch (...) {
    cudaFreeAsync(d, ctx->stream);
    throw;
  }
  NQB_CUDA(cudaFreeAsync(d, ctx->stream));
  PC_END
}

int nqb_build_preconditioner(uint32_t in_channels, const double* in_sum_squares,
                             uint64_t in_count, double in_tau, uint32_t out_channels,
                             const double* out_sum_squares, uint64_t out_count, double out_tau,
                             double gamma, double eps_floor, double* diag_in, double* diag_out,
                             double* tau_max) {
  PC_BEGIN
  NQB_REQUIRE(in_count != 0, NQB_E_EMPTY_STATS, "build_preconditioner: input stats");
  NQB_REQUIRE(!out_sum_squares || out_count != 0, NQB_E_EMPTY_STATS,
              "build_preconditioner: output stats");
  NQB_REQUIRE(gamma >= 0.0 && gamma <= 1.0, NQB_E_VALIDATION, "gamma must lie in [0,1]");
  NQB_REQUIRE(eps_floor > 0.0, NQB_E_VALIDATION, "eps_floor must be positive");
  NQB_REQUIRE(in_sum_squares && diag_in && tau_max, NQB_E_VALIDATION, "null argument");
  clipped_shrunk_diag(in_sum_squares, in_count, in_tau, in_channels, gamma, eps_floor, diag_in);
  if (out_sum_squares) {
    NQB_REQUIRE(diag_out != nullptr, NQB_E_VALIDATION, "null diag_out");
    clipped_shrunk_diag(out_sum_squares, out_count, out_tau, out_channels, gamma, eps_floor, diag_out);
    *tau_max = std::max(in_tau, out_tau);
  } else {
    *tau_max = std::max(in_tau, 1.0);  // diag_out empty = identity
  }
  PC_END
}

int nqb_precondition_weight_device(nqb_context* ctx, double* d_w, uint32_t rows, uint32_t cols,
                                   const double* d_diag_out, const double* d_diag_in) {
  PC_BEGIN
  NQB_REQUIRE(ctx != nullptr && d_w != nullptr, NQB_E_VALIDATION, "null argument");
  NQB_CUDA(cudaSetDevice(ctx->device));
  const uint64_t total = (uint64_t)rows * cols;
  if (total) k_scale_weight<<<grid_for(total), 256, 0, ctx->stream>>>(d_w, rows, cols, d_diag_out, d_diag_in);
  NQB_LAUNCHED(ctx);
  PC_END
}

int nqb_precondition_weight_host(nqb_context* ctx, double* w, uint32_t rows, uint32_t cols,
                                 const double* diag_out, const double* diag_in) {
  PC_BEGIN
  NQB_REQUIRE(ctx != nullptr && w != nullptr, NQB_E_VALIDATION, "null argument");
  NQB_CUDA(cudaSetDevice(ctx->device));
  const size_t wb = sizeof(double) * rows * cols;
  double* d = nullptr;
  NQB_CUDA(cudaMallocAsync(&d, wb + sizeof(double) * ((size_t)rows + cols), ctx->stream));
  double* dout = d + (size_t)rows * cols;
  double* din = dout + rows;
  NQB_CUDA(cudaMemcpyAsync(d, w, wb, cudaMemcpyHostToDevice, ctx->stream));
  if (diag_out) NQB_CUDA(cudaMemcpyAsync(dout, diag_out, sizeof(double) * rows, cudaMemcpyHostToDevice, ctx->stream));
  if (diag_in) NQB_CUDA(cudaMemcpyAsync(din, diag_in, sizeof(double) * cols, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t total = (uint64_t)rows * cols;
  if (total)
    k_scale_weight<<<grid_for(total), 256, 0, ctx->stream>>>(d, rows, cols, diag_out ? dout : nullptr,
                                                             diag_in ? din : nullptr);
  NQB_LAUNCHED(ctx);
  NQB_CUDA(cudaMemcpyAsync(w, d, wb, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaFreeAsync(d, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  PC_END
}

int nqb_unprecondition_rows_host(nqb_context* ctx, double* factor, uint32_t rows, uint32_t cols,
                                 const double* diag) {
  PC_BEGIN
  NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
  if (!diag) return NQB_OK;  // identity (precondition.cpp:144)
  NQB_REQUIRE(factor != nullptr, NQB_E_VALIDATION, "null factor");
  NQB_CUDA(cudaSetDevice(ctx->device));
  const size_t fb = sizeof(double) * rows * cols;
  double* d = nullptr;
  NQB_CUDA(cudaMallocAsync(&d, fb + sizeof(double) * rows, ctx->stream));
  double* dd = d + (size_t)rows * cols;
  NQB_CUDA(cudaMemcpyAsync(d, factor, fb, cudaMemcpyHostToDevice, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(dd, diag, sizeof(double) * rows, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t total = (uint64_t)rows * cols;
  if (total) k_unscale_rows<<<grid_for(total), 256, 0, ctx->stream>>>(d, rows, cols, dd);
  NQB_LAUNCHED(ctx);
  NQB_CUDA(cudaMemcpyAsync(factor, d, fb, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaFreeAsync(d, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  PC_END
}

}  // extern "C"
