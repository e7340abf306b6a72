// nqb_cli — the reference CLI's `infer` / `verify` / `bench` subcommands
// (tools/nanoquant_main.cpp:147-159, :253-340) on the B200, over the C ABI.
//
//   nqb_cli infer  --model M.nqpk --vector-in X.nqmx --out Y.nqmx [--batch]
//   nqb_cli verify --model M.nqpk
//   nqb_cli bench  --model M.nqpk [--iters 200] [--out CSV]
//
// Exit codes as in the reference (nanoquant_main.cpp:423-429): 0 ok,
// 2 validation error, 3 numerical / runtime error.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "nqb.h"

namespace {

constexpr int kExitValidation = 2, kExitNumerical = 3;

struct Fail : std::runtime_error {
  int status;
  Fail(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};
void check(int st, const char* where) {
  if (st != NQB_OK) throw Fail(st, std::string(where) + ": " + nqb_last_error());
}
int exit_code(int status) { return nqb_status_kind(status) == 1 ? kExitValidation : kExitNumerical; }

// NQMX (io.hpp:29-30, io.cpp:109-135): "NQMX", version 1, rows, cols, fp32 row-major.
struct Matrix {
  uint32_t rows = 0, cols = 0;
  std::vector<double> v;
};
Matrix read_nqmx(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Fail(NQB_E_IO, "cannot open " + path);
  std::vector<uint8_t> b((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  auto u32 = [&](size_t o) {
    if (o + 4 > b.size()) throw Fail(NQB_E_PARSE, path + ": truncated NQMX");
    return (uint32_t)b[o] | ((uint32_t)b[o + 1] << 8) | ((uint32_t)b[o + 2] << 16) |
           ((uint32_t)b[o + 3] << 24);
  };
  if (b.size() < 16 || std::memcmp(b.data(), "NQMX", 4) != 0) throw Fail(NQB_E_PARSE, path + ": bad NQMX magic");
  if (u32(4) != 1) throw Fail(NQB_E_PARSE, path + ": unsupported NQMX version");
  Matrix m;
  m.rows = u32(8);
  m.cols = u32(12);
  const size_t cnt = (size_t)m.rows * m.cols;
  if (b.size() != 16 + 4 * cnt) throw Fail(NQB_E_PARSE, path + ": NQMX size does not match its header");
  m.v.resize(cnt);
  for (size_t i = 0; i < cnt; ++i) {
    const uint32_t w = u32(16 + 4 * i);
    float f;
    std::memcpy(&f, &w, 4);
    m.v[i] = (double)f;
  }
  return m;
}
void write_nqmx(const std::string& path, const Matrix& m) {
  std::vector<uint8_t> b = {'N', 'Q', 'M', 'X'};
  auto put = [&](uint32_t w) { for (int k = 0; k < 4; ++k) b.push_back((uint8_t)(w >> (8 * k))); };
  put(1);
  put(m.rows);
  put(m.cols);
  for (double d : m.v) {
    const float f = (float)d;
    uint32_t w;
    std::memcpy(&w, &f, 4);
    put(w);
  }
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw Fail(NQB_E_IO, "cannot open " + path + " for writing");
  out.write((const char*)b.data(), (std::streamsize)b.size());
  if (!out) throw Fail(NQB_E_IO, "short write to " + path);
}

struct Model {
  nqb_nqpk* f = nullptr;
  explicit Model(const std::string& path) { check(nqb_nqpk_open(path.c_str(), &f), "read_packed_model"); }
  ~Model() { nqb_nqpk_free(f); }
  uint32_t count() const { return nqb_nqpk_count(f); }
  std::string name(uint32_t i) const {
    uint32_t len = 0;
    check(nqb_nqpk_layer_info(f, i, nullptr, 0, &len, nullptr, nullptr, nullptr), "layer_info");
    std::string s(len + 1, '\0');
    check(nqb_nqpk_layer_info(f, i, &s[0], len + 1, nullptr, nullptr, nullptr, nullptr), "layer_info");
    s.resize(len);
    return s;
  }
};

struct Layer {
  nqb_layer* h = nullptr;
  Layer(nqb_context* ctx, const Model& m, uint32_t i) {
    check(nqb_nqpk_layer_upload(ctx, m.f, i, &h), "upload");
  }
  ~Layer() { nqb_layer_free(h); }
  void shape(uint32_t& n, uint32_t& m, uint32_t& r) const { check(nqb_layer_shape(h, &n, &m, &r), "shape"); }
};

// deterministic N(0,1)-ish inputs (sum of uniforms), seeded per layer
std::vector<double> test_vector(uint64_t seed, uint32_t m) {
  std::vector<double> x(m);
  uint64_t s = seed;
  auto next = [&] {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (double)((z ^ (z >> 31)) >> 11) * 0x1.0p-53;
  };
  for (auto& v : x) {
    double a = 0.0;
    for (int k = 0; k < 12; ++k) a += next();
    v = a - 6.0;
  }
  return x;
}

int cmd_infer(nqb_context* ctx, const std::string& model_path, const std::string& in_path,
              const std::string& out_path, bool batch) {  // nanoquant_main.cpp:147-159
  const Model model(model_path);
  Matrix x = read_nqmx(in_path);
  if (!batch && x.cols != 1) throw Fail(NQB_E_DIMENSION_MISMATCH, "--vector-in must be a single column without --batch");
  for (uint32_t i = 0; i < model.count(); ++i) {
    const Layer L(ctx, model, i);
    uint32_t n, m, r;
    L.shape(n, m, r);
    if (x.rows != m) throw Fail(NQB_E_DIMENSION_MISMATCH, "gemm_packed: rows(X) != m");
    Matrix y;
    y.rows = n;
    y.cols = x.cols;
    y.v.resize((size_t)n * x.cols);
    check(nqb_gemm_f64_host(ctx, L.h, x.v.data(), x.cols, y.v.data()), "gemm_packed");
    x = std::move(y);
  }
  write_nqmx(out_path, x);
  return 0;
}

int cmd_verify(nqb_context* ctx, const std::string& model_path) {  // nanoquant_main.cpp:253-283
  const Model model(model_path);
  bool ok = true;
  for (uint32_t i = 0; i < model.count(); ++i) {
    const Layer L(ctx, model, i);
    uint32_t n, m, r;
    L.shape(n, m, r);
    const size_t wpr = (r + 31) / 32;
    // words: device round trip reproduces the file bit for bit
    const uint32_t *fu, *fv;
    check(nqb_nqpk_layer_data(model.f, i, &fu, &fv, nullptr, nullptr), "layer_data");
    std::vector<uint32_t> u((size_t)n * wpr), v((size_t)m * wpr);
    std::vector<double> s1(n), s2(m);
    check(nqb_layer_download(ctx, L.h, u.data(), v.data(), s1.data(), s2.data()), "download");
    const bool words_ok = std::memcmp(u.data(), fu, 4 * u.size()) == 0 &&
                          std::memcmp(v.data(), fv, 4 * v.size()) == 0;
    // gemv against the materialised reconstruction
    std::vector<double> dense((size_t)n * m);
    check(nqb_reconstruct_dense_host(ctx, L.h, dense.data()), "reconstruct_dense");
    const std::vector<double> x = test_vector(0xC0FFEEull ^ n ^ ((uint64_t)m << 20), m);
    std::vector<double> y(n);
    check(nqb_gemv_f64_host(ctx, L.h, x.data(), y.data()), "gemv_packed");
    double err = 0.0, norm = 0.0;
    for (uint32_t row = 0; row < n; ++row) {
      double yd = 0.0;
      for (uint32_t j = 0; j < m; ++j) yd += dense[(size_t)row * m + j] * x[j];
      err += (yd - y[row]) * (yd - y[row]);
      norm += yd * yd;
    }
    const bool gemv_ok = err <= 1e-20 * (1.0 + norm);
    std::printf("%-24s words=%s gemv=%s\n", model.name(i).c_str(), words_ok ? "ok" : "FAIL",
                gemv_ok ? "ok" : "FAIL");
    ok = ok && words_ok && gemv_ok;
  }
  if (!ok) throw Fail(NQB_E_INTERNAL, "verification failed");
  return 0;
}

int cmd_bench(nqb_context* ctx, const std::string& model_path, int iters,
              const std::string& out_path) {  // nanoquant_main.cpp:285-340, on the device
  const Model model(model_path);
  std::FILE* out = stdout;
  if (!out_path.empty() && !(out = std::fopen(out_path.c_str(), "w"))) throw Fail(NQB_E_IO, "cannot open " + out_path);
  std::fprintf(out, "layer,n,m,r,decode_us,decode_gbs,dropin_us,packed_bytes\n");
  for (uint32_t i = 0; i < model.count(); ++i) {
    const Layer L(ctx, model, i);
    uint32_t n, m, r;
    L.shape(n, m, r);
    // device decode (binary16 I/O), `iters` launches in one CUDA graph
    uint16_t *dx = nullptr, *dy = nullptr;
    if (cudaMalloc(&dx, 2 * (size_t)m) != cudaSuccess || cudaMalloc(&dy, 2 * (size_t)n) != cudaSuccess)
      throw Fail(NQB_E_OUT_OF_MEMORY, "cudaMalloc");
    cudaMemset(dx, 0x3C, 2 * (size_t)m);
    check(nqb_set_stream(ctx, nullptr), "set_stream");
    check(nqb_gemv_f16_device(ctx, L.h, dx, dy), "gemv");  // warm-up
    check(nqb_graph_begin(ctx), "graph_begin");
    for (int k = 0; k < iters; ++k) check(nqb_gemv_f16_device(ctx, L.h, dx, dy), "gemv");
    nqb_graph* g = nullptr;
    check(nqb_graph_end(ctx, &g), "graph_end");
    check(nqb_graph_launch(ctx, g), "graph_launch");
    check(nqb_synchronize(ctx), "synchronize");
    auto t0 = std::chrono::steady_clock::now();
    check(nqb_graph_launch(ctx, g), "graph_launch");
    check(nqb_synchronize(ctx), "synchronize");
    const double dev_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
    nqb_graph_free(g);
    cudaFree(dx);
    cudaFree(dy);
    // the drop-in host path (gemv_packed_f32 with host buffers)
    std::vector<float> xf(m, 1.0f), yf(n);
    check(nqb_gemv_f32_host(ctx, L.h, xf.data(), yf.data()), "gemv_packed_f32");
    const int hi = std::max(1, iters / 4);
    t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < hi; ++k) check(nqb_gemv_f32_host(ctx, L.h, xf.data(), yf.data()), "gemv_packed_f32");
    const double host_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / hi;
    const uint64_t bytes = nqb_layer_device_bytes(L.h);
    std::fprintf(out, "%s,%u,%u,%u,%.2f,%.1f,%.2f,%llu\n", model.name(i).c_str(), n, m, r, dev_us,
                 bytes / dev_us / 1e3, host_us, (unsigned long long)bytes);
  }
  if (out != stdout) std::fclose(out);
  return 0;
}

void usage() {
  std::printf(
      "nqb_cli — NanoQuant packed-model tools on the B200 (libnqb)\n"
      "  nqb_cli infer  --model M.nqpk --vector-in X.nqmx --out Y.nqmx [--batch]\n"
      "  nqb_cli verify --model M.nqpk\n"
      "  nqb_cli bench  --model M.nqpk [--iters 200] [--out CSV]\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || !std::strcmp(argv[1], "--help") || !std::strcmp(argv[1], "-h")) {
    usage();
    return argc < 2 ? kExitValidation : 0;
  }
  const std::string cmd = argv[1];
  std::map<std::string, std::string> opt;
  bool batch = false;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--batch") {
      batch = true;
    } else if (a.rfind("--", 0) == 0 && i + 1 < argc) {
      opt[a] = argv[++i];
    } else {
      std::fprintf(stderr, "error: unexpected argument %s\n", a.c_str());
      return kExitValidation;
    }
  }
  auto need = [&](const char* k) -> std::string {
    auto it = opt.find(k);
    if (it == opt.end()) throw Fail(NQB_E_VALIDATION, std::string("missing ") + k);
    return it->second;
  };
  nqb_context* ctx = nullptr;
  try {
    if (cmd != "infer" && cmd != "verify" && cmd != "bench") throw Fail(NQB_E_VALIDATION, "unknown command " + cmd);
    const std::string model = need("--model");
    check(nqb_create(0, &ctx), "create");
    int rc = 0;
    if (cmd == "infer") rc = cmd_infer(ctx, model, need("--vector-in"), need("--out"), batch);
    else if (cmd == "verify") rc = cmd_verify(ctx, model);
    else rc = cmd_bench(ctx, model, opt.count("--iters") ? std::stoi(opt["--iters"]) : 200,
                        opt.count("--out") ? opt["--out"] : "");
    nqb_destroy(ctx);
    return rc;
  } catch (const Fail& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    if (ctx) nqb_destroy(ctx);
    return exit_code(e.status);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    if (ctx) nqb_destroy(ctx);
    return kExitNumerical;
  }
}
