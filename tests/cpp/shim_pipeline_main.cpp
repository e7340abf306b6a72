// shim_pipeline_main.cpp — TEST INFRASTRUCTURE ONLY.
//
// One driver, linked two ways by oracle/Makefile:
//   oracle/_ref/pipeline_ref   with every unmodified reference source (the CPU
//                              reference, packed.o/admm.o/linalg.o/balance.o
//                              included);
//   oracle/_ref/pipeline_shim  with the same unmodified pipeline.cpp, io.cpp,
//                              storage.cpp, refine.cpp, dense.cpp and
//                              precondition.cpp, but shim/nanoquant_nqb_shim.cpp +
//                              libnqb.so in place of packed/admm/linalg/balance.
// Modes:
//   pipeline <case> <out.txt>  run_pipeline (pipeline.cpp:35-183) on a tiny model
//                              from Rng and dump metrics, packed words and scales
//   kats                       re-hosted packed-API cases of test_packed.cpp
//                              (:74-84, :219-237 and the error types), exit 1 on
//                              a failure
// tests/test_shim.py runs both binaries and compares the dumps.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "nanoquant/dense.hpp"
#include "nanoquant/errors.hpp"
#include "nanoquant/packed.hpp"
#include "nanoquant/pipeline.hpp"
#include "nanoquant/rng.hpp"

using namespace nanoquant;

namespace {

DenseMatrix random_matrix(Rng& rng, std::size_t rows, std::size_t cols) {  // test_support.hpp:52-56
  DenseMatrix m(rows, cols);
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = rng.gaussian();
  return m;
}

FactorizedLayer random_layer(Rng& rng, std::size_t n, std::size_t m, std::size_t r) {  // test_packed.cpp:29-35
  std::vector<double> s1(n), s2(m);
  for (auto& s : s1) s = rng.uniform(0.25, 2.0);
  for (auto& s : s2) s = rng.uniform(0.25, 2.0);
  return make_factorized_layer(random_matrix(rng, n, r), random_matrix(rng, m, r), std::move(s1),
                               std::move(s2));
}

int run_pipeline_case(const std::string& name, const char* out_path) {
  std::vector<std::pair<std::string, DenseMatrix>> weights;
  DenseMatrix calib;
  PipelineConfig config;
  if (name == "two_layer") {  // test_io_pipeline.cpp:130-152
    Rng rng(105);
    weights.push_back({"w0", random_matrix(rng, 24, 16)});
    weights.push_back({"w1", random_matrix(rng, 12, 24)});
    calib = random_matrix(rng, 20, 16);
    config.rank_policy.target_bpw = 3.0;
    config.admm.max_iters = 150;
    config.tune_pre.epochs = 2;
    config.tune_post.epochs = 2;
    config.tune_global.epochs = 2;
  } else if (name == "three_layer") {  // a deeper chain at 1 bit/param
    Rng rng(0x5A1);
    weights.push_back({"w0", random_matrix(rng, 64, 48)});
    weights.push_back({"w1", random_matrix(rng, 48, 64)});
    weights.push_back({"w2", random_matrix(rng, 32, 48)});
    calib = random_matrix(rng, 40, 48);
    config.rank_policy.target_bpw = 1.0;
    config.admm.max_iters = 200;
    config.tune_pre.epochs = 2;
    config.tune_post.epochs = 2;
    config.tune_global.epochs = 2;
  } else {
    std::fprintf(stderr, "unknown case %s\n", name.c_str());
    return 2;
  }
  const PipelineResult res = run_pipeline(weights, calib, config);
  FILE* f = std::fopen(out_path, "w");
  if (!f) return 2;
  std::fprintf(f, "layers %zu\nkd %.17g %.17g\nbpw %.17g\n", res.layers.size(), res.initial_kd_loss,
               res.final_kd_loss, res.model_bpw);
  for (std::size_t k = 0; k < res.layers.size(); ++k) {
    const LayerMetrics& l = res.layers[k];
    const FactorizedLayer& p = res.model.layers[k].layer;
    std::fprintf(f, "layer %s %u %u %u %.17g %.17g %d %zu\n", l.name.c_str(), l.n, l.m, l.r,
                 l.rel_fro_error, l.flip_ratio, l.admm_converged ? 1 : 0,
                 l.lagrangian_trace.size());
    std::fprintf(f, "u");
    for (auto w : p.u.words) std::fprintf(f, " %08x", w);
    std::fprintf(f, "\nv");
    for (auto w : p.v.words) std::fprintf(f, " %08x", w);
    std::fprintf(f, "\ns1");
    for (double s : p.s1) std::fprintf(f, " %.17g", s);
    std::fprintf(f, "\ns2");
    for (double s : p.s2) std::fprintf(f, " %.17g", s);
    std::fprintf(f, "\n");
  }
  std::fclose(f);
  return 0;
}

int g_fail = 0;
void report(const char* name, bool ok) {
  std::printf("%s %s\n", ok ? "ok" : "FAIL", name);
  if (!ok) g_fail = 1;
}

template <typename E, typename F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int run_kats() {
  {  // test_packed.cpp:74-84
    PackedBitMatrix p;
    p.rows = 1;
    p.cols = 4;
    p.words = {5u};
    report("unpack_kat", unpack_signs(p) == DenseMatrix::from_values(1, 4, {1, -1, 1, -1}));
    p.words = {5u | (1u << 10)};
    report("unpack_corrupt_padding_throws", throws_as<CorruptPadding>([&] { unpack_signs(p); }));
  }
  {  // test_packed.cpp:56-72
    report("pack_kat", pack_signs(DenseMatrix::from_values(1, 4, {1, -1, 1, -1})).words ==
                           std::vector<std::uint32_t>{5u});
    report("pack_non_binary_throws",
           throws_as<NonBinaryEntry>([] { pack_signs(DenseMatrix(1, 3, 0.5)); }));
    report("binarize_sign0",
           binarize(DenseMatrix::from_values(1, 4, {0.3, -0.2, 0.0, -5.0})) ==
               DenseMatrix::from_values(1, 4, {1, -1, 1, -1}));
    report("binarize_non_finite_throws",
           throws_as<NonFiniteInput>([] { binarize(DenseMatrix(1, 2, std::nan(""))); }));
  }
  {  // test_packed.cpp:219-225
    Rng rng(79);
    const FactorizedLayer layer = random_layer(rng, 24, 18, 9);
    const DenseMatrix out = gemm_packed(layer, identity(18));
    report("gemm_identity_probe", relative_frobenius_error(reconstruct_dense(layer), out) <= 1e-12);
  }
  {  // test_packed.cpp:227-237
    Rng rng(80);
    const FactorizedLayer layer = random_layer(rng, 33, 47, 21);
    const DenseMatrix x = random_matrix(rng, 47, 70);
    set_thread_budget(1);
    const DenseMatrix st = gemm_packed(layer, x);
    set_thread_budget(4);
    const DenseMatrix mt = gemm_packed(layer, x);
    report("thread_budget_set", thread_budget() == 4);
    set_thread_budget(1);
    report("gemm_multithread_equals_single", st == mt);
  }
  {  // gemv vs dense (test_packed.cpp:143-217 tolerances)
    Rng rng(81);
    const FactorizedLayer layer = random_layer(rng, 40, 70, 13);
    std::vector<double> x(70);
    std::vector<float> xf(70);
    for (std::size_t j = 0; j < 70; ++j) xf[j] = (float)(x[j] = rng.gaussian());
    const DenseMatrix w = reconstruct_dense(layer);
    const std::vector<double> y = gemv_packed(layer, x);
    const std::vector<float> yf = gemv_packed_f32(layer, xf);
    double e = 0, ef = 0, d = 0;
    for (std::size_t i = 0; i < 40; ++i) {
      double ref = 0;
      for (std::size_t j = 0; j < 70; ++j) ref += w(i, j) * x[j];
      e += (y[i] - ref) * (y[i] - ref);
      ef += (yf[i] - ref) * (yf[i] - ref);
      d += ref * ref;
    }
    report("gemv_vs_dense_1e-10", std::sqrt(e / d) <= 1e-10);
    report("gemv_f32_vs_dense_1e-5", std::sqrt(ef / d) <= 1e-5);
    report("gemv_wrong_length_throws",
           throws_as<DimensionMismatch>([&] { gemv_packed(layer, std::vector<double>(3)); }));
  }
  return g_fail;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc >= 4 && std::string(argv[1]) == "pipeline") return run_pipeline_case(argv[2], argv[3]);
    if (argc >= 2 && std::string(argv[1]) == "kats") return run_kats();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "usage: %s pipeline <two_layer|three_layer> <out> | kats\n", argv[0]);
  return 2;
}
