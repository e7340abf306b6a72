// refine.cu — STE refinement of one factorized latent layer on the device
// (SURVEY.md §8(f) row 4): ste_refine (refine.cpp:420-425) -> run_tuning
// (refine.cpp:285-384) with TuneMode::kLatentsAndScales on the pipeline's
// per-layer group, a ToyChain of one FactorizedLatentLayer (pipeline.cpp:128-135).
//
// Everything is fp64, in the reference's order of operations:
//   forward  (refine.cpp:87-100):  Bu = sign(Lu), Bv = sign(Lv), x1 = s2 .* x,
//            t = Bv^T x1, z = Bu t, out = s1 .* z
//   loss     (refine.cpp:340-350): g = 2 w_c (out - teacher)
//   backward (refine.cpp:133-175): gs1_i = sum_c g z, dz = s1 .* g, gLu = dz t^T,
//            dt = Bu^T dz, gLv = x1 dt^T, dx1 = Bv dt, gs2_j = sum_c dx1 x
//   Adam     (refine.cpp:183-196): beta 0.9 / 0.999, eps 1e-8, shared step count
// per mini-batch, batch order reshuffled each epoch with the reference Rng
// (refine.cpp:315-322), cosine or constant learning rate, and the best-loss
// checkpoint over epochs (refine.cpp:373-381).  The GEMMs run on the fp64 DMMA
// tensor cores (dgemm.cu); row sums over the batch keep the reference's
// sequential order (one thread per row).
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace nqb {

void dgemm(nqb_context*, bool, bool, uint32_t, uint32_t, uint32_t, double, const double*,
           uint32_t, const double*, uint32_t, double, double*, uint32_t);

namespace {

#define RF_STRIDE(i, n)                                                       \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (uint64_t)gridDim.x * blockDim.x)

uint32_t rf_grid(uint64_t n) { return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 8192)); }

__global__ void k_sign(const double* __restrict__ a, uint64_t n, double* __restrict__ out) {
  RF_STRIDE(i, n) out[i] = a[i] < 0.0 ? -1.0 : 1.0;  // binarize (packed.cpp:51-58)
}
// out(i, c) = x(i, c0 + c) * s[i]  (row_scaled of a column slice, refine.cpp:63-70)
__global__ void k_row_scaled(const double* __restrict__ x, uint32_t ldx, const double* __restrict__ s,
                             uint32_t rows, uint32_t cols, double* __restrict__ out) {
  RF_STRIDE(e, (uint64_t)rows * cols) {
    const uint64_t i = e / cols, c = e % cols;
    out[e] = x[i * ldx + c] * s[i];
  }
}
// g = 2 w_c (out - teacher), out = s1 .* z (refine.cpp:340-350)
__global__ void k_mse_grad(const double* __restrict__ z, const double* __restrict__ s1,
                           const double* __restrict__ t, uint32_t ldt, const double* __restrict__ w,
                           uint32_t rows, uint32_t cols, double* __restrict__ g) {
  RF_STRIDE(e, (uint64_t)rows * cols) {
    const uint64_t i = e / cols, c = e % cols;
    const double out = z[e] * s1[i];
    const double wc = w ? w[c] : 1.0;
    g[e] = 2.0 * wc * (out - t[i * ldt + c]);
  }
}
// out[i] = sum_c a(i, c) b(i, c), sequentially over c (refine.cpp:143-149, :158-164)
__global__ void k_rowdot(const double* __restrict__ a, const double* __restrict__ b, uint32_t ldb,
                         uint32_t rows, uint32_t cols, double* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint32_t c = 0; c < cols; ++c) s += a[(uint64_t)i * cols + c] * b[(uint64_t)i * ldb + c];
    out[i] = s;
  }
}
// Adam (refine.cpp:183-196)
__global__ void k_adam(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                       double* __restrict__ v, uint64_t n, double lr, double c1, double c2) {
  constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  RF_STRIDE(i, n) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}
// weighted MSE partial sums per row (refine.cpp:199-212), then one fixed-order sum
__global__ void k_wmse_rows(const double* __restrict__ z, const double* __restrict__ s1,
                            const double* __restrict__ t, const double* __restrict__ w,
                            uint32_t rows, uint32_t cols, double* __restrict__ part) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint32_t c = 0; c < cols; ++c) {
      const double wc = w ? w[c] : 1.0;
      const double d = t[(uint64_t)i * cols + c] - z[(uint64_t)i * cols + c] * s1[i];
      s += wc * d * d;
    }
    part[i] = s;
  }
}
__global__ void k_sum_seq(const double* __restrict__ part, uint32_t n, double* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += part[i];
    *out = s;
  }
}

struct Buf {  // owned device allocation of doubles
  double* p = nullptr;
  explicit Buf(size_t n) {
    if (n) NQB_CUDA(cudaMalloc(&p, n * sizeof(double)));
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

// The reference Rng (rng.hpp:25-58): index(n) = next_u64() % n.
struct HostRng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  uint64_t index(uint64_t n) { return next() % n; }
};

}  // namespace

}  // namespace nqb

using namespace nqb;

extern "C" int nqb_ste_refine_layer_host(nqb_context* ctx, double* latent_u, double* latent_v,
                                         double* s1, double* s2, uint32_t n, uint32_t m,
                                         uint32_t r, const double* x, const double* teacher,
                                         uint32_t b, const double* column_weights,
                                         const nqb_tune_config* cfg, double* best_loss_out) {
  try {
    NQB_REQUIRE(ctx != nullptr && cfg != nullptr, NQB_E_VALIDATION, "null context/config");
    NQB_REQUIRE(latent_u && latent_v && s1 && s2 && x && teacher, NQB_E_VALIDATION, "null buffer");
    NQB_CUDA(cudaSetDevice(ctx->device));
    NQB_REQUIRE(n > 0 && m > 0 && r > 0 && b > 0, NQB_E_DIMENSION_MISMATCH,
                "chain input dim does not match X rows");  // check_chain (refine.cpp:40-51)
    NQB_REQUIRE(cfg->epochs >= 1 && cfg->learning_rate > 0.0 && cfg->batch_size >= 1,
                NQB_E_VALIDATION, "invalid tuning config");  // refine.cpp:297-299
    const uint64_t nr = (uint64_t)n * r, mr = (uint64_t)m * r, mb = (uint64_t)m * b, nb = (uint64_t)n * b;
    cudaStream_t st = ctx->stream;
    // parameters (work, best), Adam moments, data, workspaces
    Buf lu(nr), lv(mr), ds1(n), ds2(m), blu(nr), blv(mr), bs1(n), bs2(m);
    Buf mu(nr), vu(nr), mv(mr), vv(mr), m1(n), v1(n), m2(m), v2(m);
    Buf X(mb), T(nb), W(column_weights ? b : 0);
    Buf bu(nr), bv(mr), x1(mb), t(std::max<uint64_t>((uint64_t)r * b, 1)), z(nb), g(nb), dz(nb),
        dt(std::max<uint64_t>((uint64_t)r * b, 1)), dx1(mb), glu(nr), glv(mr), gs1(n), gs2(m),
        part(std::max<uint32_t>(n, 1) + 1);
    auto h2d = [&](double* d, const double* h, uint64_t cnt) {
      NQB_CUDA(cudaMemcpyAsync(d, h, cnt * 8, cudaMemcpyHostToDevice, st));
    };
    auto d2d = [&](double* d, const double* s, uint64_t cnt) {
      NQB_CUDA(cudaMemcpyAsync(d, s, cnt * 8, cudaMemcpyDeviceToDevice, st));
    };
    h2d(lu.p, latent_u, nr);
    h2d(lv.p, latent_v, mr);
    h2d(ds1.p, s1, n);
    h2d(ds2.p, s2, m);
    h2d(X.p, x, mb);
    h2d(T.p, teacher, nb);
    if (column_weights) h2d(W.p, column_weights, b);
    for (Buf* q : {&mu, &vu, &mv, &vv, &m1, &v1, &m2, &v2}) {
      const uint64_t cnt = q == &mu || q == &vu ? nr : q == &mv || q == &vv ? mr : q == &m1 || q == &v1 ? n : m;
      NQB_CUDA(cudaMemsetAsync(q->p, 0, cnt * 8, st));
    }
    auto launch = [&](auto kern, uint64_t work, auto... args) {
      kern<<<rf_grid(work), 256, 0, st>>>(args...);
      NQB_LAUNCHED(ctx);
    };
    // forward of columns [c0, c0+bc) of X (ld b): leaves x1 (m x bc), t (r x bc), z (n x bc)
    auto forward = [&](uint32_t c0, uint32_t bc) {
      launch(k_sign, nr, (const double*)lu.p, nr, bu.p);
      launch(k_sign, mr, (const double*)lv.p, mr, bv.p);
      launch(k_row_scaled, (uint64_t)m * bc, (const double*)(X.p + c0), b, (const double*)ds2.p, m,
             bc, x1.p);
      dgemm(ctx, true, false, r, bc, m, 1.0, bv.p, r, x1.p, bc, 0.0, t.p, bc);  // t = Bv^T x1
      dgemm(ctx, false, false, n, bc, r, 1.0, bu.p, r, t.p, bc, 0.0, z.p, bc);  // z = Bu t
    };
    auto full_loss = [&]() -> double {  // refine.cpp:248-252 (forward_chain + weighted_mse)
      forward(0, b);
      launch(k_wmse_rows, n, (const double*)z.p, (const double*)ds1.p, (const double*)T.p,
             (const double*)W.p, n, b, part.p);
      k_sum_seq<<<1, 32, 0, st>>>(part.p, n, part.p + n);
      NQB_LAUNCHED(ctx);
      double v = 0.0;
      NQB_CUDA(cudaMemcpyAsync(&v, part.p + n, 8, cudaMemcpyDeviceToHost, st));
      NQB_CUDA(cudaStreamSynchronize(st));
      return v;
    };
    auto save_best = [&]() {
      d2d(blu.p, lu.p, nr);
      d2d(blv.p, lv.p, mr);
      d2d(bs1.p, ds1.p, n);
      d2d(bs2.p, ds2.p, m);
    };
    auto copy_out = [&](double bl) {
      NQB_CUDA(cudaMemcpyAsync(latent_u, blu.p, nr * 8, cudaMemcpyDeviceToHost, st));
      NQB_CUDA(cudaMemcpyAsync(latent_v, blv.p, mr * 8, cudaMemcpyDeviceToHost, st));
      NQB_CUDA(cudaMemcpyAsync(s1, bs1.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
      NQB_CUDA(cudaMemcpyAsync(s2, bs2.p, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
      NQB_CUDA(cudaStreamSynchronize(st));
      if (best_loss_out) *best_loss_out = bl;
    };

    double best_loss = full_loss();
    NQB_REQUIRE(std::isfinite(best_loss), NQB_E_NON_FINITE_LOSS, "tuning: initial loss is not finite");
    save_best();
    const uint32_t batch = (uint32_t)cfg->batch_size;
    const uint32_t nbatches = (b + batch - 1) / batch;
    std::vector<uint32_t> order(nbatches);
    std::iota(order.begin(), order.end(), 0u);
    long step = 0;
    for (int epoch = 0; epoch < cfg->epochs; ++epoch) {
      double lr = cfg->learning_rate;
      if (cfg->schedule == 1) lr *= 0.5 * (1.0 + std::cos(3.141592653589793 * epoch / cfg->epochs));
      HostRng rng{cfg->seed + (uint64_t)epoch * 0x9E37u};
      for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[rng.index(i)]);
      for (uint32_t bi : order) {
        const uint32_t c0 = bi * batch, bc = std::min(c0 + batch, b) - c0;
        forward(c0, bc);
        launch(k_mse_grad, (uint64_t)n * bc, (const double*)z.p, (const double*)ds1.p,
               (const double*)(T.p + c0), b, (const double*)(W.p ? W.p + c0 : nullptr), n, bc, g.p);
        // backward (refine.cpp:139-166)
        k_rowdot<<<rf_grid(n), 256, 0, st>>>(g.p, z.p, bc, n, bc, gs1.p);
        NQB_LAUNCHED(ctx);
        launch(k_row_scaled, (uint64_t)n * bc, (const double*)g.p, bc, (const double*)ds1.p, n, bc, dz.p);
        dgemm(ctx, false, true, n, r, bc, 1.0, dz.p, bc, t.p, bc, 0.0, glu.p, r);   // dz t^T
        dgemm(ctx, true, false, r, bc, n, 1.0, bu.p, r, dz.p, bc, 0.0, dt.p, bc);   // Bu^T dz
        dgemm(ctx, false, true, m, r, bc, 1.0, x1.p, bc, dt.p, bc, 0.0, glv.p, r);  // x1 dt^T
        dgemm(ctx, false, false, m, bc, r, 1.0, bv.p, r, dt.p, bc, 0.0, dx1.p, bc); // Bv dt
        k_rowdot<<<rf_grid(m), 256, 0, st>>>(dx1.p, X.p + c0, b, m, bc, gs2.p);
        NQB_LAUNCHED(ctx);
        ++step;
        const double c1 = 1.0 - std::pow(0.9, (double)step);
        const double c2 = 1.0 - std::pow(0.999, (double)step);
        launch(k_adam, nr, lu.p, (const double*)glu.p, mu.p, vu.p, nr, lr, c1, c2);
        launch(k_adam, mr, lv.p, (const double*)glv.p, mv.p, vv.p, mr, lr, c1, c2);
        launch(k_adam, (uint64_t)n, ds1.p, (const double*)gs1.p, m1.p, v1.p, (uint64_t)n, lr, c1, c2);
        launch(k_adam, (uint64_t)m, ds2.p, (const double*)gs2.p, m2.p, v2.p, (uint64_t)m, lr, c1, c2);
      }
      const double loss = full_loss();
      if (!std::isfinite(loss)) {  // NonFiniteLoss carries the best checkpoint (refine.hpp:72-77)
        copy_out(best_loss);
        fail(NQB_E_NON_FINITE_LOSS, "tuning diverged to a non-finite loss");
      }
      if (loss < best_loss) {
        best_loss = loss;
        save_best();
      }
    }
    copy_out(best_loss);
    return NQB_OK;
  } catch (const Failure& f) {
    set_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    set_error(e.what());
    return NQB_E_INTERNAL;
  }
}
