// oracle/ref_harness.cpp — TEST INFRASTRUCTURE ONLY (never part of the product).
//
// A C ABI over the UNMODIFIED NanoQuant reference library, compiled from the
// sources where they lie under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libnqref.so.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg load it.  Every function forwards to the
// reference entry point it names; status codes follow include/nqb.h.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "nanoquant/admm.hpp"
#include "nanoquant/balance.hpp"
#include "nanoquant/dense.hpp"
#include "nanoquant/errors.hpp"
#include "nanoquant/half.hpp"
#include "nanoquant/io.hpp"
#include "nanoquant/linalg.hpp"
#include "nanoquant/packed.hpp"
#include "nanoquant/precondition.hpp"
#include "nanoquant/refine.hpp"
#include "nanoquant/rng.hpp"
#include "nanoquant/storage.hpp"
#include "nqb.h"

using namespace nanoquant;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const DimensionMismatch*>(&e)) return NQB_E_DIMENSION_MISMATCH;
  if (dynamic_cast<const NonFiniteInput*>(&e)) return NQB_E_NON_FINITE_INPUT;
  if (dynamic_cast<const NonBinaryEntry*>(&e)) return NQB_E_NON_BINARY_ENTRY;
  if (dynamic_cast<const CorruptPadding*>(&e)) return NQB_E_CORRUPT_PADDING;
  if (dynamic_cast<const RankTooLarge*>(&e)) return NQB_E_RANK_TOO_LARGE;
  if (dynamic_cast<const InvalidRank*>(&e)) return NQB_E_INVALID_RANK;
  if (dynamic_cast<const NotSymmetric*>(&e)) return NQB_E_NOT_SYMMETRIC;
  if (dynamic_cast<const TargetTooSmall*>(&e)) return NQB_E_TARGET_TOO_SMALL;
  if (dynamic_cast<const ParseError*>(&e)) return NQB_E_PARSE;
  if (dynamic_cast<const IoError*>(&e)) return NQB_E_IO;
  if (dynamic_cast<const EmptyStats*>(&e)) return NQB_E_EMPTY_STATS;
  if (dynamic_cast<const ZeroMatrix*>(&e)) return NQB_E_ZERO_MATRIX;
  if (dynamic_cast<const NotPositiveDefinite*>(&e)) return NQB_E_NOT_POSITIVE_DEFINITE;
  if (auto* err = dynamic_cast<const Error*>(&e)) {
    return err->kind() == ErrorKind::kValidation ? NQB_E_VALIDATION : NQB_E_INTERNAL;
  }
  return NQB_E_INTERNAL;
}

#define GUARD(...)                             \
  try {                                        \
    __VA_ARGS__;                               \
    return NQB_OK;                             \
  } catch (const std::exception& e) {          \
    return code_of(e);                         \
  }

DenseMatrix dm(const double* p, std::size_t rows, std::size_t cols) {
  return DenseMatrix::from_values(rows, cols, std::vector<double>(p, p + rows * cols));
}

void put(const DenseMatrix& m, double* out) {
  std::memcpy(out, m.data(), m.size() * sizeof(double));
}

PackedBitMatrix pbm(const std::uint32_t* w, std::uint32_t rows, std::uint32_t cols) {
  PackedBitMatrix p;
  p.rows = rows;
  p.cols = cols;
  p.words.assign(w, w + static_cast<std::size_t>(rows) * p.words_per_row());
  return p;
}

FactorizedLayer layer_of(std::uint32_t n, std::uint32_t m, std::uint32_t r,
                         const std::uint32_t* u, const std::uint32_t* v, const double* s1,
                         const double* s2) {
  FactorizedLayer l;
  l.n = n;
  l.m = m;
  l.r = r;
  l.u = pbm(u, n, r);
  l.v = pbm(v, m, r);
  l.s1.assign(s1, s1 + n);
  l.s2.assign(s2, s2 + m);
  return l;
}

AdmmConfig cfg_of(const nqb_admm_config* c) {
  AdmmConfig a;
  a.rank = c->rank;
  a.max_iters = c->max_iters;
  a.rho_start = c->rho_start;
  a.rho_end = c->rho_end;
  a.ridge = c->ridge;
  a.tol = c->tol;
  a.seed = c->seed;
  return a;
}

}  // namespace

extern "C" {

const char* nqref_last_error(void) { return g_err.c_str(); }

// ---- Rng (rng.hpp:25-58) -------------------------------------------------
void* nqref_rng_create(std::uint64_t seed) { return new Rng(seed); }
void nqref_rng_destroy(void* h) { delete static_cast<Rng*>(h); }
void nqref_rng_u64(void* h, std::uint64_t count, std::uint64_t* out) {
  auto* r = static_cast<Rng*>(h);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r->next_u64();
}
void nqref_rng_uniform(void* h, double lo, double hi, std::uint64_t count, double* out) {
  auto* r = static_cast<Rng*>(h);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r->uniform(lo, hi);
}
void nqref_rng_gaussian(void* h, std::uint64_t count, double* out) {
  auto* r = static_cast<Rng*>(h);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r->gaussian();
}
void nqref_rng_sign(void* h, std::uint64_t count, double* out) {
  auto* r = static_cast<Rng*>(h);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r->sign();
}
void nqref_rng_index(void* h, std::uint64_t n, std::uint64_t count, std::uint64_t* out) {
  auto* r = static_cast<Rng*>(h);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = r->index(n);
}

// ---- half.hpp:26-89 -------------------------------------------------------
void nqref_double_to_half(const double* in, std::uint64_t count, std::uint16_t* out) {
  for (std::uint64_t i = 0; i < count; ++i) out[i] = double_to_half(in[i]);
}
void nqref_half_to_double(const std::uint16_t* in, std::uint64_t count, double* out) {
  for (std::uint64_t i = 0; i < count; ++i) out[i] = half_to_double(in[i]);
}

// ---- storage.cpp:124-141 ---------------------------------------------------
int nqref_rank_for_target_bpw(std::uint64_t n, std::uint64_t m, double t, std::uint32_t* out) {
  GUARD(*out = rank_for_target_bpw(n, m, t))
}

// ---- packed.cpp ------------------------------------------------------------
int nqref_binarize(const double* in, std::uint32_t rows, std::uint32_t cols, double* out) {
  GUARD(put(binarize(dm(in, rows, cols)), out))
}
int nqref_pack_signs(const double* in, std::uint32_t rows, std::uint32_t cols,
                     std::uint32_t* words) {
  GUARD({
    const PackedBitMatrix p = pack_signs(dm(in, rows, cols));
    std::memcpy(words, p.words.data(), p.words.size() * 4);
  })
}
int nqref_unpack_signs(const std::uint32_t* words, std::uint32_t rows, std::uint32_t cols,
                       double* out) {
  GUARD(put(unpack_signs(pbm(words, rows, cols)), out))
}
int nqref_reconstruct_dense(std::uint32_t n, std::uint32_t m, std::uint32_t r,
                            const std::uint32_t* u, const std::uint32_t* v, const double* s1,
                            const double* s2, double* w) {
  GUARD(put(reconstruct_dense(layer_of(n, m, r, u, v, s1, s2)), w))
}
int nqref_gemv_f64(std::uint32_t n, std::uint32_t m, std::uint32_t r, const std::uint32_t* u,
                   const std::uint32_t* v, const double* s1, const double* s2,
                   const double* x, std::uint32_t xlen, double* y) {
  GUARD({
    const auto out = gemv_packed(layer_of(n, m, r, u, v, s1, s2),
                                 std::vector<double>(x, x + xlen));
    std::memcpy(y, out.data(), out.size() * sizeof(double));
  })
}
int nqref_gemv_f32(std::uint32_t n, std::uint32_t m, std::uint32_t r, const std::uint32_t* u,
                   const std::uint32_t* v, const double* s1, const double* s2, const float* x,
                   std::uint32_t xlen, float* y) {
  GUARD({
    const auto out = gemv_packed_f32(layer_of(n, m, r, u, v, s1, s2),
                                     std::vector<float>(x, x + xlen));
    std::memcpy(y, out.data(), out.size() * sizeof(float));
  })
}
int nqref_gemm(std::uint32_t n, std::uint32_t m, std::uint32_t r, const std::uint32_t* u,
               const std::uint32_t* v, const double* s1, const double* s2, const double* x,
               std::uint32_t b, double* y, std::uint32_t threads) {
  GUARD({
    set_thread_budget(threads);
    put(gemm_packed(layer_of(n, m, r, u, v, s1, s2), dm(x, m, b)), y);
  })
}

// Timing helper for the CPU baseline: `count` independent layers, each called
// `reps` times with gemv_packed_f32 on its own std::thread (the reference is
// single-threaded per call; host-core parallelism = concurrent layers).
int nqref_gemv_f32_concurrent(std::uint32_t count, const std::uint32_t* n,
                              const std::uint32_t* m, const std::uint32_t* r,
                              const std::uint32_t* const* u, const std::uint32_t* const* v,
                              const double* const* s1, const double* const* s2,
                              const float* const* x, float* const* y, std::uint32_t reps) {
  GUARD({
    std::vector<FactorizedLayer> layers;
    for (std::uint32_t i = 0; i < count; ++i)
      layers.push_back(layer_of(n[i], m[i], r[i], u[i], v[i], s1[i], s2[i]));
    std::vector<std::thread> pool;
    for (std::uint32_t i = 0; i < count; ++i) {
      pool.emplace_back([&, i]() {
        const std::vector<float> xi(x[i], x[i] + m[i]);
        std::vector<float> out;
        for (std::uint32_t k = 0; k < reps; ++k) out = gemv_packed_f32(layers[i], xi);
        std::memcpy(y[i], out.data(), out.size() * sizeof(float));
      });
    }
    for (auto& t : pool) t.join();
  })
}

// Decode-pass timing helper for the reference arm of bench.py: `count` layers
// prebuilt once (nqref_pass_create), then one decode pass = gemv_packed_f32 on
// every layer, spread over `threads` host threads that take layers from a
// shared counter (the reference is single-threaded per call; host-core
// parallelism = concurrent layers).  Only the gemv calls run inside
// nqref_pass_run.
struct RefPass {
  std::vector<FactorizedLayer> layers;
  std::vector<std::vector<float>> xs;
};
void* nqref_pass_create(std::uint32_t count, const std::uint32_t* n, const std::uint32_t* m,
                        const std::uint32_t* r, const std::uint32_t* const* u,
                        const std::uint32_t* const* v, const double* const* s1,
                        const double* const* s2, const float* const* x) {
  try {
    auto* P = new RefPass();
    for (std::uint32_t i = 0; i < count; ++i) {
      P->layers.push_back(layer_of(n[i], m[i], r[i], u[i], v[i], s1[i], s2[i]));
      P->xs.emplace_back(x[i], x[i] + m[i]);
    }
    return P;
  } catch (const std::exception& e) {
    code_of(e);
    return nullptr;
  }
}
int nqref_pass_run(void* h, float* const* y, std::uint32_t threads) {
  GUARD({
    auto* P = static_cast<RefPass*>(h);
    const std::uint32_t count = (std::uint32_t)P->layers.size();
    std::atomic<std::uint32_t> next{0};
    std::atomic<int> failed{0};
    auto work = [&]() {
      for (;;) {
        const std::uint32_t i = next.fetch_add(1);
        if (i >= count) return;
        try {
          const std::vector<float> out = gemv_packed_f32(P->layers[i], P->xs[i]);
          std::memcpy(y[i], out.data(), out.size() * sizeof(float));
        } catch (...) {
          failed = 1;
        }
      }
    };
    std::vector<std::thread> pool;
    for (std::uint32_t t = 1; t < std::max<std::uint32_t>(1, threads); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (failed) throw Error(ErrorKind::kNumerical, "gemv_packed_f32 failed in the pass");
  })
}
void nqref_pass_destroy(void* h) { delete static_cast<RefPass*>(h); }

// ---- refine.cpp --------------------------------------------------------------
// ste_refine (refine.cpp:420-425) on a ToyChain of one FactorizedLatentLayer,
// the pipeline's per-layer group (pipeline.cpp:128-135); latents and scales are
// overwritten with the result (the best checkpoint, also on NonFiniteLoss).
int nqref_ste_refine(double* lu, double* lv, double* s1, double* s2, std::uint32_t n,
                     std::uint32_t m, std::uint32_t r, const double* x, const double* teacher,
                     std::uint32_t b, const double* colw, std::int32_t epochs, double lr,
                     std::int32_t batch, std::int32_t cosine, std::uint64_t seed) {
  auto put_layer = [&](const ToyChain& c) {
    const auto& f = std::get<FactorizedLatentLayer>(c.layers[0]);
    put(f.latent_u, lu);
    put(f.latent_v, lv);
    std::memcpy(s1, f.s1.data(), n * sizeof(double));
    std::memcpy(s2, f.s2.data(), m * sizeof(double));
  };
  try {
    ToyChain chain;
    chain.layers.push_back(FactorizedLatentLayer{dm(lu, n, r), dm(lv, m, r),
                                                 std::vector<double>(s1, s1 + n),
                                                 std::vector<double>(s2, s2 + m)});
    TuneConfig cfg;
    cfg.epochs = epochs;
    cfg.learning_rate = lr;
    cfg.batch_size = batch;
    cfg.schedule = cosine ? LrSchedule::kCosine : LrSchedule::kConstant;
    cfg.seed = seed;
    if (colw) cfg.column_weights.assign(colw, colw + b);
    put_layer(ste_refine(chain, dm(x, m, b), dm(teacher, n, b), cfg));
    return NQB_OK;
  } catch (const NonFiniteLoss& e) {
    put_layer(e.best_chain);
    g_err = e.what();
    return NQB_E_NON_FINITE_LOSS;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}

// ---- linalg.cpp -------------------------------------------------------------
int nqref_top_singular_pair(const double* mat, std::uint32_t rows, std::uint32_t cols,
                            std::int32_t max_iters, double tol, double* sigma, double* left,
                            double* right, std::int32_t* converged) {
  GUARD({
    const SingularPair p = top_singular_pair(dm(mat, rows, cols), max_iters, tol);
    *sigma = p.sigma;
    std::memcpy(left, p.left.data(), rows * sizeof(double));
    std::memcpy(right, p.right.data(), cols * sizeof(double));
    *converged = p.converged ? 1 : 0;
  })
}
int nqref_spectral_norm(const double* mat, std::uint32_t rows, std::uint32_t cols,
                        std::int32_t iters, double* sigma) {
  GUARD(*sigma = spectral_norm_estimate(dm(mat, rows, cols), iters))
}
int nqref_truncated_svd(const double* mat, std::uint32_t rows, std::uint32_t cols,
                        std::uint32_t rank, double* u, double* v) {
  GUARD({
    DenseMatrix uu, vv;
    truncated_svd_factors(dm(mat, rows, cols), rank, &uu, &vv);
    put(uu, u);
    put(vv, v);
  })
}
int nqref_cholesky_solve(const double* a, std::uint32_t n, const double* b, std::uint32_t nrhs,
                         double* x) {
  GUARD(put(cholesky_solve(dm(a, n, n), dm(b, n, nrhs)), x))
}

// ---- admm.cpp ---------------------------------------------------------------
int nqref_svid(const double* p, std::uint32_t rows, std::uint32_t cols, double* z) {
  GUARD(put(svid(dm(p, rows, cols)), z))
}
int nqref_factor_solve(const double* target, std::uint32_t rows, std::uint32_t cols,
                       const double* fixed, std::uint32_t rank, const double* z,
                       const double* l, double rho, double ridge, double* x) {
  GUARD(put(admm_factor_solve(dm(target, rows, cols), dm(fixed, cols, rank),
                              dm(z, rows, rank), dm(l, rows, rank), rho, ridge),
            x))
}
int nqref_lagrangian(const double* u, const double* v, const double* zu, const double* zv,
                     const double* lu, const double* lv, std::uint32_t n, std::uint32_t m,
                     std::uint32_t r, double rho, const double* target, double ridge,
                     double* out) {
  GUARD({
    AdmmState s;
    s.u = dm(u, n, r);
    s.v = dm(v, m, r);
    s.z_u = dm(zu, n, r);
    s.z_v = dm(zv, m, r);
    s.l_u = dm(lu, n, r);
    s.l_v = dm(lv, m, r);
    s.rho = rho;
    *out = augmented_lagrangian(s, dm(target, n, m), ridge);
  })
}
int nqref_monotone_rho(const double* w, std::uint32_t n, std::uint32_t m, double* out) {
  GUARD(*out = monotone_rho(dm(w, n, m)))
}

static void fill_result(const AdmmState& s, nqb_admm_result* res) {
  std::memset(res, 0, sizeof(*res));
  res->iteration = static_cast<std::uint32_t>(s.iteration);
  res->converged = s.converged ? 1 : 0;
  res->primal_residual = s.primal_residual;
  res->rho = s.rho;
  res->trace_len = static_cast<std::uint32_t>(s.lagrangian_trace.size());
}

int nqref_admm_factorize(const double* w, std::uint32_t n, std::uint32_t m,
                         const nqb_admm_config* cfg, double* cu, double* cv, double* trace,
                         nqb_admm_result* res) {
  GUARD({
    const AdmmResult out = admm_factorize(dm(w, n, m), cfg_of(cfg));
    put(out.consensus_u, cu);
    put(out.consensus_v, cv);
    fill_result(out.state, res);
    if (trace) {
      std::memcpy(trace, out.state.lagrangian_trace.data(),
                  out.state.lagrangian_trace.size() * sizeof(double));
    }
  })
}

// ---- balance.cpp ------------------------------------------------------------
int nqref_balance(const double* pu, const double* pv, std::uint32_t n, std::uint32_t m,
                  std::uint32_t r, const double* diag_out, const double* diag_in,
                  double floor, double* lu, double* lv, double* s1, double* s2,
                  double* eta) {
  GUARD({
    Preconditioner p;
    if (diag_out) p.diag_out.assign(diag_out, diag_out + n);
    if (diag_in) p.diag_in.assign(diag_in, diag_in + m);
    const BalancedLatents b =
        balance_and_extract_scales(dm(pu, n, r), dm(pv, m, r), p, floor);
    put(b.latent_u, lu);
    put(b.latent_v, lv);
    std::memcpy(s1, b.s1.data(), n * sizeof(double));
    std::memcpy(s2, b.s2.data(), m * sizeof(double));
    *eta = b.eta;
  })
}

// ---- pipeline-style per-matrix init (pipeline.cpp:95-110, :150-153) ----------
// admm_factorize -> balance (identity) -> make_factorized_layer; returns the
// packed factors, the double scales, the latents' signs source (latents) and
// relative_frobenius_error(W, reconstruct_dense(layer)).
int nqref_factorize_layer(const double* w, std::uint32_t n, std::uint32_t m,
                          const nqb_admm_config* cfg, double floor, std::uint32_t* u_words,
                          std::uint32_t* v_words, double* s1, double* s2, double* rel_err,
                          double* trace, nqb_admm_result* res) {
  GUARD({
    const DenseMatrix target = dm(w, n, m);
    const AdmmResult out = admm_factorize(target, cfg_of(cfg));
    const BalancedLatents lat =
        balance_and_extract_scales(out.consensus_u, out.consensus_v, Preconditioner{}, floor);
    const FactorizedLayer layer = make_factorized_layer(lat.latent_u, lat.latent_v, lat.s1, lat.s2);
    std::memcpy(u_words, layer.u.words.data(), layer.u.words.size() * 4);
    std::memcpy(v_words, layer.v.words.data(), layer.v.words.size() * 4);
    std::memcpy(s1, layer.s1.data(), n * sizeof(double));
    std::memcpy(s2, layer.s2.data(), m * sizeof(double));
    *rel_err = relative_frobenius_error(target, reconstruct_dense(layer));
    fill_result(out.state, res);
    if (trace) {
      std::memcpy(trace, out.state.lagrangian_trace.data(),
                  out.state.lagrangian_trace.size() * sizeof(double));
    }
  })
}

// relative_frobenius_error(W, reconstruct_dense(layer)) (dense.cpp:141-146).
int nqref_layer_rel_error(std::uint32_t n, std::uint32_t m, std::uint32_t r,
                          const std::uint32_t* u, const std::uint32_t* v, const double* s1,
                          const double* s2, const double* w, double* out) {
  GUARD(*out = relative_frobenius_error(dm(w, n, m),
                                        reconstruct_dense(layer_of(n, m, r, u, v, s1, s2))))
}

// ---- io.cpp: NQPK (io.cpp:139-193) -------------------------------------------
// Serialises `count` layers into `buf` (capacity `cap`); *len receives the size.
int nqref_serialize_nqpk(std::uint32_t count, const char* const* names,
                         const std::uint32_t* n, const std::uint32_t* m,
                         const std::uint32_t* r, const std::uint32_t* const* u,
                         const std::uint32_t* const* v, const double* const* s1,
                         const double* const* s2, std::uint8_t* buf, std::uint64_t cap,
                         std::uint64_t* len) {
  GUARD({
    PackedModelFile f;
    for (std::uint32_t i = 0; i < count; ++i) {
      f.layers.push_back({names[i], layer_of(n[i], m[i], r[i], u[i], v[i], s1[i], s2[i])});
    }
    const auto bytes = serialize_packed_model(f);
    *len = bytes.size();
    if (bytes.size() > cap) throw Error(ErrorKind::kValidation, "buffer too small");
    std::memcpy(buf, bytes.data(), bytes.size());
  })
}

// ---- precondition.cpp: phase 1 (precondition.cpp:37-153) --------------------
// ChannelStats state passed in/out as (sum_squares[cols], sample_count, tau).
int nqref_accumulate_stats(const double* batch, std::uint32_t rows, std::uint32_t cols,
                           double percentile, double* sum_squares, std::uint64_t* count,
                           double* tau) {
  GUARD({
    ChannelStats st(cols);
    std::memcpy(st.sum_squares.data(), sum_squares, sizeof(double) * cols);
    st.sample_count = *count;
    st.tau = *tau;
    accumulate_stats(st, dm(batch, rows, cols), percentile);
    std::memcpy(sum_squares, st.sum_squares.data(), sizeof(double) * cols);
    *count = st.sample_count;
    *tau = st.tau;
  })
}

int nqref_build_preconditioner(std::uint32_t in_c, const double* in_sq, std::uint64_t in_count,
                               double in_tau, std::uint32_t out_c, const double* out_sq,
                               std::uint64_t out_count, double out_tau, double gamma,
                               double eps_floor, double* diag_in, double* diag_out,
                               double* tau_max) {
  GUARD({
    ChannelStats in(in_c);
    std::memcpy(in.sum_squares.data(), in_sq, sizeof(double) * in_c);
    in.sample_count = in_count;
    in.tau = in_tau;
    std::optional<ChannelStats> out;
    if (out_sq) {
      out.emplace(out_c);
      std::memcpy(out->sum_squares.data(), out_sq, sizeof(double) * out_c);
      out->sample_count = out_count;
      out->tau = out_tau;
    }
    const Preconditioner p = build_preconditioner(in, out, gamma, eps_floor);
    std::memcpy(diag_in, p.diag_in.data(), sizeof(double) * p.diag_in.size());
    if (out_sq) std::memcpy(diag_out, p.diag_out.data(), sizeof(double) * p.diag_out.size());
    *tau_max = p.tau_max;
  })
}

int nqref_precondition_weight(const double* w, std::uint32_t rows, std::uint32_t cols,
                              const double* diag_out, const double* diag_in, double* out) {
  GUARD({
    Preconditioner p;
    if (diag_out) p.diag_out.assign(diag_out, diag_out + rows);
    if (diag_in) p.diag_in.assign(diag_in, diag_in + cols);
    put(precondition_weight(dm(w, rows, cols), p), out);
  })
}

int nqref_unprecondition_rows(double* factor, std::uint32_t rows, std::uint32_t cols,
                              const double* diag) {
  GUARD({
    DenseMatrix f = dm(factor, rows, cols);
    std::vector<double> d;
    if (diag) d.assign(diag, diag + rows);
    unprecondition_rows(f, d);
    put(f, factor);
  })
}

}  // extern "C"
