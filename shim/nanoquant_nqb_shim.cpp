// nanoquant_nqb_shim.cpp — the C++ drop-in for the NanoQuant reference.
//
// Defines, in namespace nanoquant and with the reference's own types (the
// reference headers are the interface), every function of packed.hpp:49-102,
// admm.hpp:30-85, linalg.hpp:35-51 and balance.hpp:38-41, each forwarding to the
// B200 C ABI (include/nqb.h, libnqb.so).  Linking this object in place of the
// reference's packed.o / admm.o / linalg.o / balance.o leaves every caller
// (pipeline.cpp:108-110, :122-123, :140-141, :150-153, nanoquant_main.cpp:155,
// :259-268, :297-315, refine.cpp:94-95) unchanged.
//
// Errors: every nqb_status is rethrown as the reference exception type it maps
// to (errors.hpp:25-114), so e.g. CHECK_THROWS_AS(unpack_signs(...),
// CorruptPadding) (test_packed.cpp:83) still holds.
// Threading: one library context per process (device NQ_DEVICE, default 0),
// created on first use; calls are serialised on it, so the functions stay
// thread-safe like the reference's.  thread_budget / set_thread_budget keep the
// reference semantics (NQ_THREADS, default 1); results do not depend on it.
// Scales: layers keep their fp64 scales on the device (nqb_layer_upload_exact),
// so reconstruct_dense / gemv / gemm see exactly the reference's inputs.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nanoquant/admm.hpp"
#include "nanoquant/balance.hpp"
#include "nanoquant/dense.hpp"
#include "nanoquant/errors.hpp"
#include "nanoquant/linalg.hpp"
#include "nanoquant/packed.hpp"
#include "nanoquant/precondition.hpp"
#include "nqb.h"

namespace nanoquant {

namespace {

std::mutex g_mu;
nqb_context* g_ctx = nullptr;

[[noreturn]] void rethrow(int st, const char* where) {
  const std::string msg = std::string(where) + ": " + nqb_last_error();
  switch (st) {
    case NQB_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case NQB_E_NON_FINITE_INPUT: throw NonFiniteInput(msg);
    case NQB_E_NON_BINARY_ENTRY: throw NonBinaryEntry(msg);
    case NQB_E_CORRUPT_PADDING: throw CorruptPadding(msg);
    case NQB_E_RANK_TOO_LARGE: throw RankTooLarge(msg);
    case NQB_E_INVALID_RANK: throw InvalidRank(msg);
    case NQB_E_NOT_SYMMETRIC: throw NotSymmetric(msg);
    case NQB_E_TARGET_TOO_SMALL: throw TargetTooSmall(msg);
    case NQB_E_PARSE: throw ParseError(msg);
    case NQB_E_IO: throw IoError(msg);
    case NQB_E_EMPTY_STATS: throw EmptyStats(msg);
    case NQB_E_ZERO_MATRIX: throw ZeroMatrix(msg);
    case NQB_E_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(msg);
    default:
      throw Error(nqb_status_kind(st) == 1 ? ErrorKind::kValidation : ErrorKind::kNumerical, msg);
  }
}
inline void check(int st, const char* where) {
  if (st != NQB_OK) rethrow(st, where);
}

// The process-wide context; the caller holds g_mu.
nqb_context* ctx_locked() {
  if (!g_ctx) {
    const char* dev = std::getenv("NQ_DEVICE");
    check(nqb_create(dev ? std::atoi(dev) : 0, &g_ctx), "nqb_create");
  }
  return g_ctx;
}

uint32_t u32(std::size_t v, const char* what) {
  if (v > 0xFFFFFFFFull) throw DimensionMismatch(std::string(what) + " exceeds 2^32-1");
  return static_cast<uint32_t>(v);
}

DenseMatrix dense(std::size_t rows, std::size_t cols) { return DenseMatrix(rows, cols); }

// A device copy of a FactorizedLayer with its exact scales; freed on scope exit.
struct DeviceLayer {
  nqb_layer* h = nullptr;
  DeviceLayer(nqb_context* ctx, const FactorizedLayer& l) {
    if (l.u.rows != l.n || l.v.rows != l.m || l.u.cols != l.r || l.v.cols != l.r ||
        l.s1.size() != l.n || l.s2.size() != l.m || l.u.words.size() != l.n * l.u.words_per_row() ||
        l.v.words.size() != l.m * l.v.words_per_row())
      throw DimensionMismatch("factorized layer: inconsistent shapes");
    check(nqb_layer_upload_exact(ctx, l.n, l.m, l.r, l.u.words.data(), l.v.words.data(),
                                 l.s1.data(), l.s2.data(), &h),
          "layer upload");
  }
  ~DeviceLayer() { nqb_layer_free(h); }
  DeviceLayer(const DeviceLayer&) = delete;
  DeviceLayer& operator=(const DeviceLayer&) = delete;
};

std::atomic<unsigned> g_thread_budget{0};  // 0 = not yet read from the environment

}  // namespace

// ---------------------------------------------------------------- packed.hpp
unsigned thread_budget() {  // packed.cpp:26-45 semantics (NQ_THREADS, default 1)
  unsigned v = g_thread_budget.load(std::memory_order_relaxed);
  if (v == 0) {
    const char* env = std::getenv("NQ_THREADS");
    const long t = env ? std::strtol(env, nullptr, 10) : 1;
    v = t < 1 ? 1u : static_cast<unsigned>(t);
    g_thread_budget.store(v, std::memory_order_relaxed);
  }
  return v;
}

void set_thread_budget(unsigned n) {  // packed.cpp:47-49
  g_thread_budget.store(n == 0 ? 1 : n, std::memory_order_relaxed);
}

DenseMatrix binarize(const DenseMatrix& latent) {
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix out = dense(latent.rows(), latent.cols());
  check(nqb_binarize(ctx_locked(), latent.data(), latent.size(), out.data(), 0), "binarize");
  return out;
}

PackedBitMatrix pack_signs(const DenseMatrix& signs) {
  std::lock_guard<std::mutex> lk(g_mu);
  PackedBitMatrix p;
  p.rows = u32(signs.rows(), "rows");
  p.cols = u32(signs.cols(), "cols");
  p.words.assign(p.rows * p.words_per_row(), 0u);
  if (signs.size())
    check(nqb_pack_signs(ctx_locked(), signs.data(), p.rows, p.cols, p.words.data(), 0),
          "pack_signs");
  return p;
}

DenseMatrix unpack_signs(const PackedBitMatrix& packed) {
  if (packed.words.size() != packed.rows * packed.words_per_row())
    throw DimensionMismatch("unpack_signs: word count mismatch");
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix out = dense(packed.rows, packed.cols);
  if (out.size())
    check(nqb_unpack_signs(ctx_locked(), packed.words.data(), packed.rows, packed.cols,
                           out.data(), 0),
          "unpack_signs");
  return out;
}

FactorizedLayer make_factorized_layer(const DenseMatrix& latent_u, const DenseMatrix& latent_v,
                                      std::vector<double> s1, std::vector<double> s2) {
  if (latent_u.cols() != latent_v.cols())
    throw DimensionMismatch("make_factorized_layer: ranks differ");
  if (s1.size() != latent_u.rows() || s2.size() != latent_v.rows())
    throw DimensionMismatch("make_factorized_layer: scale lengths");
  FactorizedLayer layer;
  layer.n = u32(latent_u.rows(), "n");
  layer.m = u32(latent_v.rows(), "m");
  layer.r = u32(latent_u.cols(), "r");
  layer.u = pack_signs(binarize(latent_u));  // packed.cpp:119-120 (NonFiniteInput first)
  layer.v = pack_signs(binarize(latent_v));
  layer.s1 = std::move(s1);
  layer.s2 = std::move(s2);
  return layer;
}

DenseMatrix reconstruct_dense(const FactorizedLayer& layer) {
  std::lock_guard<std::mutex> lk(g_mu);
  nqb_context* ctx = ctx_locked();
  DeviceLayer d(ctx, layer);
  DenseMatrix w = dense(layer.n, layer.m);
  check(nqb_reconstruct_dense_host(ctx, d.h, w.data()), "reconstruct_dense");
  return w;
}

std::vector<double> gemv_packed(const FactorizedLayer& layer, const std::vector<double>& x) {
  if (x.size() != layer.m) throw DimensionMismatch("gemv_packed: |x| != m");
  std::lock_guard<std::mutex> lk(g_mu);
  nqb_context* ctx = ctx_locked();
  DeviceLayer d(ctx, layer);
  std::vector<double> y(layer.n);
  check(nqb_gemv_f64_host(ctx, d.h, x.data(), y.data()), "gemv_packed");
  return y;
}

std::vector<float> gemv_packed_f32(const FactorizedLayer& layer, const std::vector<float>& x) {
  if (x.size() != layer.m) throw DimensionMismatch("gemv_packed: |x| != m");
  std::lock_guard<std::mutex> lk(g_mu);
  nqb_context* ctx = ctx_locked();
  DeviceLayer d(ctx, layer);
  std::vector<float> y(layer.n);
  check(nqb_gemv_f32_host(ctx, d.h, x.data(), y.data()), "gemv_packed_f32");
  return y;
}

DenseMatrix gemm_packed(const FactorizedLayer& layer, const DenseMatrix& x) {
  if (x.rows() != layer.m) throw DimensionMismatch("gemm_packed: rows(X) != m");
  std::lock_guard<std::mutex> lk(g_mu);
  nqb_context* ctx = ctx_locked();
  DeviceLayer d(ctx, layer);
  DenseMatrix y = dense(layer.n, x.cols());
  if (x.cols())
    check(nqb_gemm_f64_host(ctx, d.h, x.data(), u32(x.cols(), "b"), y.data()), "gemm_packed");
  return y;
}

// ---------------------------------------------------------------- linalg.hpp
DenseMatrix cholesky_solve(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.rows() != a.cols()) throw DimensionMismatch("cholesky_solve: A not square");
  if (b.rows() != a.rows()) throw DimensionMismatch("cholesky_solve: rows(B) != n");
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix x = dense(b.rows(), b.cols());
  check(nqb_cholesky_solve_host(ctx_locked(), a.data(), u32(a.rows(), "n"), b.data(),
                                u32(b.cols(), "nrhs"), x.data()),
        "cholesky_solve");
  return x;
}

SingularPair top_singular_pair(const DenseMatrix& m, int max_iters, double tol) {
  std::lock_guard<std::mutex> lk(g_mu);
  SingularPair p;
  p.left.assign(m.rows(), 0.0);
  p.right.assign(m.cols(), 0.0);
  int32_t conv = 0;
  check(nqb_top_singular_pair_host(ctx_locked(), m.data(), u32(m.rows(), "rows"),
                                   u32(m.cols(), "cols"), max_iters, tol, &p.sigma,
                                   p.left.data(), p.right.data(), &conv),
        "top_singular_pair");
  p.converged = conv != 0;
  return p;
}

double spectral_norm_estimate(const DenseMatrix& m, int iters) {
  if (m.empty()) return 0.0;
  std::lock_guard<std::mutex> lk(g_mu);
  double s = 0.0;
  check(nqb_spectral_norm_host(ctx_locked(), m.data(), u32(m.rows(), "rows"),
                               u32(m.cols(), "cols"), iters, &s),
        "spectral_norm_estimate");
  return s;
}

void truncated_svd_factors(const DenseMatrix& m, std::size_t rank, DenseMatrix* u_out,
                           DenseMatrix* v_out) {
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix u = dense(m.rows(), rank), v = dense(m.cols(), rank);
  check(nqb_truncated_svd_host(ctx_locked(), m.data(), u32(m.rows(), "rows"),
                               u32(m.cols(), "cols"), u32(rank, "rank"), u.data(), v.data()),
        "truncated_svd_factors");
  if (u_out) *u_out = std::move(u);
  if (v_out) *v_out = std::move(v);
}

// ------------------------------------------------------------------ admm.hpp
DenseMatrix svid(const DenseMatrix& p) {
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix z = dense(p.rows(), p.cols());
  check(nqb_svid_host(ctx_locked(), p.data(), u32(p.rows(), "rows"), u32(p.cols(), "cols"),
                      z.data()),
        "svid");
  return z;
}

DenseMatrix admm_factor_solve(const DenseMatrix& target, const DenseMatrix& fixed,
                              const DenseMatrix& z, const DenseMatrix& l, double rho,
                              double ridge) {
  std::lock_guard<std::mutex> lk(g_mu);
  DenseMatrix x = dense(target.rows(), fixed.cols());
  if (fixed.rows() != target.cols() || z.rows() != target.rows() || l.rows() != target.rows() ||
      z.cols() != fixed.cols() || l.cols() != fixed.cols())
    throw DimensionMismatch("admm_factor_solve: operand shapes");
  check(nqb_admm_factor_solve_host(ctx_locked(), target.data(), u32(target.rows(), "rows"),
                                   u32(target.cols(), "cols"), fixed.data(),
                                   u32(fixed.cols(), "rank"), z.data(), l.data(), rho, ridge,
                                   x.data()),
        "admm_factor_solve");
  return x;
}

double augmented_lagrangian(const AdmmState& s, const DenseMatrix& target, double ridge) {
  std::lock_guard<std::mutex> lk(g_mu);
  double v = 0.0;
  check(nqb_augmented_lagrangian_host(ctx_locked(), s.u.data(), s.v.data(), s.z_u.data(),
                                      s.z_v.data(), s.l_u.data(), s.l_v.data(),
                                      u32(target.rows(), "n"), u32(target.cols(), "m"),
                                      u32(s.u.cols(), "r"), s.rho, target.data(), ridge, &v),
        "augmented_lagrangian");
  return v;
}

AdmmResult admm_factorize(const DenseMatrix& target, const AdmmConfig& config) {
  nqb_admm_config c;
  nqb_admm_config_default(&c);
  c.rank = config.rank;
  c.max_iters = config.max_iters;
  c.rho_start = config.rho_start;
  c.rho_end = config.rho_end;
  c.ridge = config.ridge;
  c.tol = config.tol;
  c.seed = config.seed;
  c.record_trace = 1;
  const std::size_t n = target.rows(), m = target.cols(), r = config.rank;
  std::lock_guard<std::mutex> lk(g_mu);
  AdmmResult out;
  out.consensus_u = dense(n, r);
  out.consensus_v = dense(m, r);
  AdmmState& s = out.state;
  s.u = dense(n, r);
  s.v = dense(m, r);
  s.z_u = dense(n, r);
  s.z_v = dense(m, r);
  s.l_u = dense(n, r);
  s.l_v = dense(m, r);
  std::vector<double> trace(static_cast<std::size_t>(std::max(config.max_iters, 0)) + 1);
  double* state[6] = {s.u.data(), s.v.data(), s.z_u.data(), s.z_v.data(), s.l_u.data(),
                      s.l_v.data()};
  nqb_admm_result res;
  check(nqb_admm_factorize_state_host(ctx_locked(), target.data(), u32(n, "rows"),
                                      u32(m, "cols"), &c, out.consensus_u.data(),
                                      out.consensus_v.data(), trace.data(), &res, state),
        "admm_factorize");
  trace.resize(res.trace_len);
  s.lagrangian_trace = std::move(trace);
  s.rho = res.rho;
  s.iteration = res.iteration;
  s.primal_residual = res.primal_residual;
  s.converged = res.converged != 0;
  return out;
}

double monotone_rho(const DenseMatrix& target) {  // admm.cpp:98-100
  return 16.0 * std::max(spectral_norm_estimate(target), 1e-12);
}

// --------------------------------------------------------------- balance.hpp
BalancedLatents balance_and_extract_scales(const DenseMatrix& consensus_u,
                                           const DenseMatrix& consensus_v,
                                           const Preconditioner& p, double scale_floor) {
  if (!p.diag_out.empty() && consensus_u.rows() != p.diag_out.size())
    throw DimensionMismatch("balance: rows(P_U) != |diag_out|");
  if (!p.diag_in.empty() && consensus_v.rows() != p.diag_in.size())
    throw DimensionMismatch("balance: rows(P_V) != |diag_in|");
  if (consensus_u.cols() != consensus_v.cols())
    throw DimensionMismatch("balance: factor ranks differ");
  const std::size_t n = consensus_u.rows(), m = consensus_v.rows(), r = consensus_u.cols();
  std::lock_guard<std::mutex> lk(g_mu);
  BalancedLatents out;
  out.latent_u = dense(n, r);
  out.latent_v = dense(m, r);
  out.s1.assign(n, 0.0);
  out.s2.assign(m, 0.0);
  check(nqb_balance_host(ctx_locked(), consensus_u.data(), consensus_v.data(), u32(n, "n"),
                         u32(m, "m"), u32(r, "r"), p.diag_out.empty() ? nullptr : p.diag_out.data(),
                         p.diag_in.empty() ? nullptr : p.diag_in.data(), scale_floor,
                         out.latent_u.data(), out.latent_v.data(), out.s1.data(), out.s2.data(),
                         &out.eta),
        "balance_and_extract_scales");
  return out;
}

}  // namespace nanoquant
