// admm.cu — LB-ADMM initialisation on the device (admm.cpp:24-199,
// balance.cpp:36-65) and the C-ABI entry points for it and its building blocks.
//
// Every step is the reference's, in fp64, with its operation order kept where
// it is elementwise (svid magnitudes, dual updates, rebalance, rho schedule);
// products and reductions run as DMMA GEMMs and fixed-tree reductions.
// The host loop only reads back scalars (norms, residuals, trace values);
// all matrices stay in HBM.
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace nqb {

// dgemm.cu / linalg.cu / pack.cu / api.cu
void dgemm(nqb_context*, bool, bool, uint32_t, uint32_t, uint32_t, double, const double*,
           uint32_t, const double*, uint32_t, double, double*, uint32_t);
double reduce_to_host(nqb_context*, const double*, const double*, uint64_t, int, int*, int*);
double colstats_device(nqb_context*, double*, uint32_t, uint32_t, const double*, const double*,
                       double, int, double*, int*);
struct PairResult {
  double sigma;
  int converged;
  int iters;
};
PairResult top_pair_from_start(nqb_context*, const double*, uint32_t, uint32_t, int, double*,
                               double*, int, double);
PairResult top_pair_device(nqb_context*, const double*, uint32_t, uint32_t, int, double*,
                           double*, int, double);
struct SvdStats {
  uint32_t steps = 0;
  uint64_t iters = 0;
  uint32_t converged = 0;
};
void truncated_svd_device(nqb_context*, double*, uint32_t, uint32_t, uint32_t, double*, double*,
                          SvdStats*);
void cholesky_solve_rows(nqb_context*, const double*, uint32_t, const double*, uint32_t, double*);
void launch_pack_rows(nqb_context*, const double*, uint32_t, uint32_t, uint32_t*, int, int*);
nqb_layer* layer_from_device_words(nqb_context*, uint32_t, uint32_t, uint32_t, const uint32_t*,
                                   const uint32_t*, const __half*, const __half*);
void layer_v_reference(nqb_context*, const nqb_layer*, uint32_t*, uint32_t);
void launch_rel_error(nqb_context*, const nqb_layer*, const uint32_t*, uint32_t, const double*,
                      double*, double*, const double* = nullptr, const double* = nullptr);
uint64_t rel_error_partial_count(const nqb_layer*);

enum { RED_SUMSQ = 0, RED_SUMSQ_DIFF = 1, RED_DOT = 2 };

// ---------------------------------------------------------------------------
// Elementwise kernels
// ---------------------------------------------------------------------------
#define GRID_STRIDE(i, n)                                                   \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_scale(double* __restrict__ a, uint64_t n, double f) {
  GRID_STRIDE(i, n) a[i] *= f;  // DenseMatrix::scale (dense.cpp:56-58)
}
// Rebalance (admm.cpp:112-123) in one launch: U, Z_U, L_U scaled by c and V,
// Z_V, L_V by 1/c (the same per-element products as six DenseMatrix::scale calls).
__global__ void k_rebalance(double* __restrict__ u, double* __restrict__ zu,
                            double* __restrict__ lu, uint64_t nr, double c,
                            double* __restrict__ v, double* __restrict__ zv,
                            double* __restrict__ lv, uint64_t mr, double ci) {
  GRID_STRIDE(i, nr + mr) {
    if (i < nr) {
      u[i] *= c;
      zu[i] *= c;
      lu[i] *= c;
    } else {
      const uint64_t j = i - nr;
      v[j] *= ci;
      zv[j] *= ci;
      lv[j] *= ci;
    }
  }
}
__global__ void k_add(const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ c, uint64_t n) {
  GRID_STRIDE(i, n) c[i] = a[i] + b[i];  // add (dense.cpp:108-115)
}
// l = l + (u - z)  (admm.cpp:182-183)
__global__ void k_dual(double* __restrict__ l, const double* __restrict__ u,
                       const double* __restrict__ z, uint64_t n) {
  GRID_STRIDE(i, n) l[i] = l[i] + (u[i] - z[i]);
}
// c = rho * (z - l)  (admm.cpp:76-77 term)
__global__ void k_rho_diff(const double* __restrict__ z, const double* __restrict__ l,
                           double* __restrict__ c, uint64_t n, double rho) {
  GRID_STRIDE(i, n) c[i] = rho * (z[i] - l[i]);
}
// Z = sign(P) .* (sqrt(s) l)(sqrt(s) r)^T  (admm.cpp:36-44)
__global__ void k_svid_construct(const double* __restrict__ p, uint32_t rows, uint32_t cols,
                                 const double* __restrict__ left,
                                 const double* __restrict__ right, double root,
                                 double* __restrict__ z) {
  GRID_STRIDE(e, (uint64_t)rows * cols) {
    const uint64_t i = e / cols, j = e % cols;
    const double ai = root * left[i];
    const double mag = ai * root * right[j];
    z[e] = p[e] < 0.0 ? -mag : mag;
  }
}
__global__ void k_add_diag2(double* __restrict__ a, uint32_t n, double add) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[(uint64_t)i * n + i] += add;
}
// rows scaled by 1/diag[i] (precondition.cpp:143-153)
__global__ void k_unprecondition(double* __restrict__ f, uint32_t rows, uint32_t cols,
                                 const double* __restrict__ diag) {
  GRID_STRIDE(e, (uint64_t)rows * cols) {
    const double inv = 1.0 / diag[e / cols];
    f[e] *= inv;
  }
}
// s[i] = max(sum_j |f_ij| / cols, floor)  (balance.cpp:23-32); warp per row.
__global__ void k_row_mean_abs(const double* __restrict__ f, uint32_t rows, uint32_t cols,
                               double floor, double* __restrict__ s) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  double acc = 0.0;
  for (uint32_t j = lane; j < cols; j += 32) acc += fabs(f[(uint64_t)warp * cols + j]);
  acc = warp_sum(acc);
  if (lane == 0) {
    const double v = acc / (double)cols;
    s[warp] = v < floor ? floor : v;
  }
}
__global__ void k_to_half(const double* __restrict__ s, uint32_t n, __half* __restrict__ h) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    h[i] = __float2half_rn((float)s[i]);  // double_to_half (half.hpp:83-85)
}
__global__ void k_transpose(const double* __restrict__ a, uint32_t rows, uint32_t cols,
                            double* __restrict__ t) {
  __shared__ double tile[32][33];
  const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const uint32_t tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t r = r0 + k, c = c0 + tx;
    tile[k][tx] = (r < rows && c < cols) ? a[(uint64_t)r * cols + c] : 0.0;
  }
  __syncthreads();
  for (uint32_t k = ty; k < 32; k += 8) {
    const uint32_t c = c0 + k, r = r0 + tx;
    if (c < cols && r < rows) t[(uint64_t)c * rows + r] = tile[tx][k];
  }
}

static uint32_t ew_grid(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(g, 8192));
}

#define EW(ctx, kern, n, ...)                                                        \
  do {                                                                             \
    if ((n) > 0) {                                                                 \
      kern<<<ew_grid(n), 256, 0, (ctx)->stream>>>(__VA_ARGS__);                    \
      NQB_LAUNCHED(ctx);                                                           \
    }                                                                              \
  } while (0)

struct Dev {  // owned device allocation
  double* p = nullptr;
  size_t n = 0;
  Dev() = default;
  explicit Dev(size_t count) : n(count) {
    if (count) NQB_CUDA(cudaMalloc(&p, count * sizeof(double)));
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

double norm2(nqb_context* ctx, const double* a, uint64_t n) {
  return reduce_to_host(ctx, a, nullptr, n, RED_SUMSQ, nullptr, nullptr);
}

void dtranspose(nqb_context* ctx, const double* a, uint32_t rows, uint32_t cols, double* t) {
  k_transpose<<<dim3(ceil_div(cols, 32), ceil_div(rows, 32)), 256, 0, ctx->stream>>>(a, rows, cols, t);
  NQB_LAUNCHED(ctx);
}

// ---------------------------------------------------------------------------
// svid (admm.cpp:24-46)
// ---------------------------------------------------------------------------
void svid_device(nqb_context* ctx, const double* d_p, uint32_t rows, uint32_t cols,
                 double* d_z) {
  double* vec = (double*)scratch(ctx, 8, sizeof(double) * ((size_t)rows + cols + 8));
  double* left = vec;
  double* right = vec + rows;
  int flags = 0;
  colstats_device(ctx, const_cast<double*>(d_p), rows, cols, nullptr, nullptr, 0.0, 0, right,
                  &flags);
  NQB_REQUIRE(!(flags & 1), NQB_E_NON_FINITE_INPUT, "svid: input contains non-finite values");
  NQB_REQUIRE(flags & 2, NQB_E_ZERO_MATRIX, "svid: matrix is identically zero");
  // |P| has the same column norms as P; iterate on |P| (abs_mode)
  const PairResult pr = top_pair_from_start(ctx, d_p, rows, cols, 1, left, right, 300, 1e-12);
  const double root = std::sqrt(pr.sigma);
  EW(ctx, k_svid_construct, (uint64_t)rows * cols, d_p, rows, cols, left, right, root, d_z);
}

// ---------------------------------------------------------------------------
// admm_factor_solve (admm.cpp:48-80).  target is rows x cols (row-major, ld
// tcols) or, if trans, the transpose of a tcols x rows... expressed through
// the DMMA GEMM's op(): X = (fixed^T fixed + (rho+ridge) I)^-1-solve of
// target * fixed + rho (Z - L), row by row.
// ---------------------------------------------------------------------------
struct SolveWork {
  double* gram;  // r x r
  double* rhs;   // rows x r
};

void factor_solve_device(nqb_context* ctx, const double* d_target, bool trans_target,
                         uint32_t rows, uint32_t cols, const double* d_fixed, uint32_t r,
                         const double* d_z, const double* d_l, double rho, double ridge,
                         double* d_x, SolveWork& w) {
  // A = gram(fixed) + (rho + ridge) I
  dgemm(ctx, true, false, r, r, cols, 1.0, d_fixed, r, d_fixed, r, 0.0, w.gram, r);
  k_add_diag2<<<ceil_div(r, 256), 256, 0, ctx->stream>>>(w.gram, r, rho + ridge);
  NQB_LAUNCHED(ctx);
  // rhs = target * fixed + rho (Z - L)     (rows x r; the reference's r x rows transposed)
  EW(ctx, k_rho_diff, (uint64_t)rows * r, d_z, d_l, w.rhs, (uint64_t)rows * r, rho);
  if (trans_target) {  // target = W^T, W stored cols x rows
    dgemm(ctx, true, false, rows, r, cols, 1.0, d_target, rows, d_fixed, r, 1.0, w.rhs, r);
  } else {
    dgemm(ctx, false, false, rows, r, cols, 1.0, d_target, cols, d_fixed, r, 1.0, w.rhs, r);
  }
  cholesky_solve_rows(ctx, w.gram, r, w.rhs, rows, d_x);
}

__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ c, uint64_t n) {
  GRID_STRIDE(i, n) c[i] = a[i] - b[i];  // subtract (dense.cpp:117-124)
}

void sub_into(nqb_context* ctx, const double* a, const double* b, double* c, uint64_t n) {
  EW(ctx, k_sub, n, a, b, c, n);
}

// ---------------------------------------------------------------------------
// augmented_lagrangian (admm.cpp:82-96)
// ---------------------------------------------------------------------------
struct State {
  uint32_t n, m, r;
  double *u, *v, *zu, *zv, *lu, *lv;
  double rho;
};

double lagrangian_device(nqb_context* ctx, const State& s, const double* d_w, double ridge,
                         double* d_scratch_nm) {
  const uint64_t nm = (uint64_t)s.n * s.m, nr = (uint64_t)s.n * s.r, mr = (uint64_t)s.m * s.r;
  NQB_CUDA(cudaMemcpyAsync(d_scratch_nm, d_w, nm * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  dgemm(ctx, false, true, s.n, s.m, s.r, -1.0, s.u, s.r, s.v, s.r, 1.0, d_scratch_nm, s.m);
  const double fit = norm2(ctx, d_scratch_nm, nm);
  const double su = norm2(ctx, s.u, nr), sv = norm2(ctx, s.v, mr);
  // ru = U - Z_U formed first (as subtract() does), then <L_U, ru> and ||ru||^2;
  // the scratch (>= max(n*r, m*r) doubles) is reused.
  double dlu, sru, dlv, srv;
  sub_into(ctx, s.u, s.zu, d_scratch_nm, nr);
  dlu = reduce_to_host(ctx, s.lu, d_scratch_nm, nr, RED_DOT, nullptr, nullptr);
  sru = norm2(ctx, d_scratch_nm, nr);
  sub_into(ctx, s.v, s.zv, d_scratch_nm, mr);
  dlv = reduce_to_host(ctx, s.lv, d_scratch_nm, mr, RED_DOT, nullptr, nullptr);
  srv = norm2(ctx, d_scratch_nm, mr);
  double value = 0.5 * fit;
  value += 0.5 * ridge * (su + sv);
  value += s.rho * dlu + 0.5 * s.rho * sru;
  value += s.rho * dlv + 0.5 * s.rho * srv;
  return value;
}

double rel_residual(nqb_context* ctx, const double* x, const double* z, uint64_t n) {
  const double nx = std::sqrt(norm2(ctx, x, n));
  const double r = std::sqrt(reduce_to_host(ctx, x, z, n, RED_SUMSQ_DIFF, nullptr, nullptr));
  return r / std::max(nx, 1e-300);
}

double spectral_norm_device(nqb_context* ctx, const double* d_m, uint32_t rows, uint32_t cols,
                            int iters, bool is_zero) {
  if ((uint64_t)rows * cols == 0 || is_zero) return 0.0;
  double* vec = (double*)scratch(ctx, 9, sizeof(double) * ((size_t)rows + cols + 8));
  return top_pair_device(ctx, d_m, rows, cols, 0, vec, vec + rows, iters, 1e-14).sigma;
}

// ---------------------------------------------------------------------------
// admm_factorize (admm.cpp:127-199) on device buffers.
// ---------------------------------------------------------------------------
void admm_device(nqb_context* ctx, const double* d_w, uint32_t n, uint32_t m,
                 const nqb_admm_config& cfg, double* d_cu, double* d_cv, double* h_trace,
                 nqb_admm_result* res, double* const* h_state) {
  std::memset(res, 0, sizeof(*res));
  const uint64_t nm = (uint64_t)n * m;
  int flags = 0;
  reduce_to_host(ctx, d_w, nullptr, nm, RED_SUMSQ, (int*)scratch(ctx, 7, 64) + 12, &flags);
  NQB_REQUIRE(flags & 2, NQB_E_ZERO_MATRIX, "admm_factorize: target is identically zero");
  NQB_REQUIRE(!(flags & 1), NQB_E_NON_FINITE_INPUT, "admm_factorize: target is non-finite");
  NQB_REQUIRE(cfg.rank != 0, NQB_E_INVALID_RANK, "admm_factorize: rank must be >= 1");
  NQB_REQUIRE(cfg.rank <= std::min(n, m), NQB_E_RANK_TOO_LARGE,
              "admm_factorize: rank exceeds min(rows, cols)");
  NQB_REQUIRE(cfg.max_iters >= 1, NQB_E_VALIDATION, "admm_factorize: max_iters must be >= 1");
  const uint32_t r = cfg.rank;

  double rho_start = cfg.rho_start, rho_end = cfg.rho_end;
  if (rho_start <= 0.0 && rho_end <= 0.0) {
    const double spectral = std::max(spectral_norm_device(ctx, d_w, n, m, 200, false), 1e-12);
    res->sigma_max = spectral;
    rho_start = 0.1 * spectral;
    rho_end = 10.0 * spectral;
  } else if (rho_start <= 0.0 || rho_end < rho_start) {
    fail(NQB_E_VALIDATION, "admm_factorize: need rho_end >= rho_start > 0");
  }

  const uint64_t nr = (uint64_t)n * r, mr = (uint64_t)m * r;
  const uint64_t big = std::max(nr, mr);
  Dev u(nr), v(mr), zu(nr), zv(mr), lu(nr), lv(mr), p(big), rhs(big), gram((uint64_t)r * r);
  Dev wscr(nm);  // truncated-SVD residual, then the Lagrangian's W - U V^T
  State s{n, m, r, u.p, v.p, zu.p, zv.p, lu.p, lv.p, 0.0};
  SolveWork sw{gram.p, rhs.p};

  cudaEvent_t e0 = ctx->ev0, e1 = ctx->ev1;
  NQB_CUDA(cudaEventRecord(e0, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(wscr.p, d_w, nm * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  SvdStats st;
  truncated_svd_device(ctx, wscr.p, n, m, r, u.p, v.p, &st);
  NQB_CUDA(cudaEventRecord(e1, ctx->stream));
  NQB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  NQB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  res->seconds_svd_init = ms * 1e-3;
  res->svd_steps = st.steps;
  res->svd_power_iters = st.iters;
  res->svd_converged_steps = st.converged;

  NQB_CUDA(cudaEventRecord(e0, ctx->stream));
  svid_device(ctx, u.p, n, r, zu.p);
  svid_device(ctx, v.p, m, r, zv.p);
  NQB_CUDA(cudaMemsetAsync(lu.p, 0, nr * 8, ctx->stream));
  NQB_CUDA(cudaMemsetAsync(lv.p, 0, mr * 8, ctx->stream));
  s.rho = rho_start;
  uint32_t tl = 0;
  const bool trace = cfg.record_trace && h_trace;
  if (trace) h_trace[tl++] = lagrangian_device(ctx, s, d_w, cfg.ridge, wscr.p);

  const int denom = std::max(cfg.max_iters - 1, 1);
  bool converged = false;
  uint32_t iteration = 0;
  double primal = 0.0;
  for (int k = 0; k < cfg.max_iters; ++k) {
    primal = std::max(rel_residual(ctx, u.p, zu.p, nr), rel_residual(ctx, v.p, zv.p, mr));
    if (primal < cfg.tol) {
      converged = true;
      break;
    }
    const double rho = rho_start + (rho_end - rho_start) * ((double)k / denom);
    if (rho != s.rho) {  // duals are stored scaled; keep Y continuous
      const double rescale = s.rho / rho;
      EW(ctx, k_scale, nr, lu.p, nr, rescale);
      EW(ctx, k_scale, mr, lv.p, mr, rescale);
      s.rho = rho;
    }
    // rebalance (admm.cpp:112-123)
    {
      const double nu = std::sqrt(norm2(ctx, u.p, nr)), nv = std::sqrt(norm2(ctx, v.p, mr));
      if (nu > 0.0 && nv > 0.0) {
        const double c = std::sqrt(nv / nu);
        EW(ctx, k_rebalance, nr + mr, u.p, zu.p, lu.p, nr, c, v.p, zv.p, lv.p, mr, 1.0 / c);
      }
    }
    factor_solve_device(ctx, d_w, false, n, m, v.p, r, zu.p, lu.p, s.rho, cfg.ridge, u.p, sw);
    factor_solve_device(ctx, d_w, true, m, n, u.p, r, zv.p, lv.p, s.rho, cfg.ridge, v.p, sw);
    EW(ctx, k_add, nr, u.p, lu.p, p.p, nr);
    svid_device(ctx, p.p, n, r, zu.p);
    EW(ctx, k_add, mr, v.p, lv.p, p.p, mr);
    svid_device(ctx, p.p, m, r, zv.p);
    EW(ctx, k_dual, nr, lu.p, u.p, zu.p, nr);
    EW(ctx, k_dual, mr, lv.p, v.p, zv.p, mr);
    iteration = (uint32_t)k + 1;
    if (trace) h_trace[tl++] = lagrangian_device(ctx, s, d_w, cfg.ridge, wscr.p);
  }
  if (!converged) {
    primal = std::max(rel_residual(ctx, u.p, zu.p, nr), rel_residual(ctx, v.p, zv.p, mr));
    converged = primal < cfg.tol;
  }
  EW(ctx, k_add, nr, u.p, lu.p, d_cu, nr);
  EW(ctx, k_add, mr, v.p, lv.p, d_cv, mr);
  if (h_state) {  // AdmmState matrices (admm.hpp:53-62): U, V, Z_U, Z_V, L_U, L_V
    const double* src[6] = {u.p, v.p, zu.p, zv.p, lu.p, lv.p};
    const uint64_t len[6] = {nr, mr, nr, mr, nr, mr};
    for (int i = 0; i < 6; ++i)
      if (h_state[i])
        NQB_CUDA(cudaMemcpyAsync(h_state[i], src[i], len[i] * 8, cudaMemcpyDeviceToHost,
                                 ctx->stream));
  }
  NQB_CUDA(cudaEventRecord(e1, ctx->stream));
  NQB_CUDA(cudaEventSynchronize(e1));
  NQB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  res->seconds_iterations = ms * 1e-3;
  res->iteration = iteration;
  res->converged = converged ? 1 : 0;
  res->primal_residual = primal;
  res->rho = s.rho;
  res->trace_len = tl;
}

// balance_and_extract_scales (balance.cpp:36-65) in place on device latents.
double balance_device(nqb_context* ctx, double* d_lu, double* d_lv, uint32_t n, uint32_t m,
                      uint32_t r, const double* d_diag_out, const double* d_diag_in,
                      double floor, double* d_s1, double* d_s2) {
  const uint64_t nr = (uint64_t)n * r, mr = (uint64_t)m * r;
  if (d_diag_out) EW(ctx, k_unprecondition, nr, d_lu, n, r, d_diag_out);
  if (d_diag_in) EW(ctx, k_unprecondition, mr, d_lv, m, r, d_diag_in);
  const double nu = std::sqrt(norm2(ctx, d_lu, nr)), nv = std::sqrt(norm2(ctx, d_lv, mr));
  const double eta = (nu == 0.0 || nv == 0.0) ? 1.0 : std::sqrt(nv / nu);
  EW(ctx, k_scale, nr, d_lu, nr, eta);
  EW(ctx, k_scale, mr, d_lv, mr, 1.0 / eta);
  k_row_mean_abs<<<ceil_div((uint64_t)n * 32, 256), 256, 0, ctx->stream>>>(d_lu, n, r, floor, d_s1);
  NQB_LAUNCHED(ctx);
  k_row_mean_abs<<<ceil_div((uint64_t)m * 32, 256), 256, 0, ctx->stream>>>(d_lv, m, r, floor, d_s2);
  NQB_LAUNCHED(ctx);
  return eta;
}

}  // namespace nqb

using namespace nqb;

#define API_BEGIN try {
#define API_END                     \
  return NQB_OK;                    \
  }                                 \
  catch (const Failure& f) {        \
    set_error(f.msg);               \
    return f.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    set_error(e.what());            \
    return NQB_E_INTERNAL;          \
  }

static void h2d(nqb_context* ctx, double* d, const double* h, uint64_t n) {
  NQB_CUDA(cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, ctx->stream));
}
static void d2h(nqb_context* ctx, double* h, const double* d, uint64_t n) {
  NQB_CUDA(cudaMemcpyAsync(h, d, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
}
static void need_ctx(nqb_context* ctx) {
  NQB_REQUIRE(ctx != nullptr, NQB_E_VALIDATION, "null context");
  NQB_CUDA(cudaSetDevice(ctx->device));
}

extern "C" {

void nqb_admm_config_default(nqb_admm_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->rank = 1;
  c->max_iters = 400;
  c->ridge = 1e-4;
  c->tol = 1e-4;
  c->record_trace = 1;
}

int nqb_admm_factorize_device(nqb_context* ctx, const double* d_w, uint32_t n, uint32_t m,
                              const nqb_admm_config* cfg, double* d_cu, double* d_cv,
                              double* trace, nqb_admm_result* result) {
  API_BEGIN
  need_ctx(ctx);
  NQB_REQUIRE(cfg && result, NQB_E_VALIDATION, "null config/result");
  admm_device(ctx, d_w, n, m, *cfg, d_cu, d_cv, trace, result, nullptr);
  API_END
}

int nqb_admm_factorize_host(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                            const nqb_admm_config* cfg, double* cu, double* cv, double* trace,
                            nqb_admm_result* result) {
  return nqb_admm_factorize_state_host(ctx, w, n, m, cfg, cu, cv, trace, result, nullptr);
}

int nqb_admm_factorize_state_host(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                                  const nqb_admm_config* cfg, double* cu, double* cv,
                                  double* trace, nqb_admm_result* result,
                                  double* const* state) {
  API_BEGIN
  need_ctx(ctx);
  NQB_REQUIRE(cfg && result, NQB_E_VALIDATION, "null config/result");
  const uint64_t nm = (uint64_t)n * m;
  Dev dw(nm);
  h2d(ctx, dw.p, w, nm);
  const uint32_t r = cfg->rank;
  NQB_REQUIRE(r <= std::min(n, m) || nm == 0, NQB_E_RANK_TOO_LARGE,
              "admm_factorize: rank exceeds min(rows, cols)");
  Dev du((uint64_t)n * std::max(r, 1u)), dv((uint64_t)m * std::max(r, 1u));
  admm_device(ctx, dw.p, n, m, *cfg, du.p, dv.p, trace, result, state);
  d2h(ctx, cu, du.p, (uint64_t)n * r);
  d2h(ctx, cv, dv.p, (uint64_t)m * r);
  API_END
}

int nqb_balance_host(nqb_context* ctx, const double* pu, const double* pv, uint32_t n,
                     uint32_t m, uint32_t r, const double* diag_out, const double* diag_in,
                     double scale_floor, double* lu, double* lv, double* s1, double* s2,
                     double* eta) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t nr = (uint64_t)n * r, mr = (uint64_t)m * r;
  Dev a(nr), b(mr), d1(n), d2(m), s1d(n), s2d(m);
  h2d(ctx, a.p, pu, nr);
  h2d(ctx, b.p, pv, mr);
  if (diag_out) h2d(ctx, d1.p, diag_out, n);
  if (diag_in) h2d(ctx, d2.p, diag_in, m);
  const double e = balance_device(ctx, a.p, b.p, n, m, r, diag_out ? d1.p : nullptr,
                                  diag_in ? d2.p : nullptr, scale_floor, s1d.p, s2d.p);
  d2h(ctx, lu, a.p, nr);
  d2h(ctx, lv, b.p, mr);
  d2h(ctx, s1, s1d.p, n);
  d2h(ctx, s2, s2d.p, m);
  if (eta) *eta = e;
  API_END
}

int nqb_factorize_layer(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                        const nqb_admm_config* cfg, double scale_floor, int on_device,
                        nqb_layer** out, nqb_admm_result* result, double* rel_error) {
  API_BEGIN
  need_ctx(ctx);
  NQB_REQUIRE(cfg && out, NQB_E_VALIDATION, "null config/output");
  *out = nullptr;
  const uint64_t nm = (uint64_t)n * m;
  Dev dwbuf(on_device ? 0 : nm);
  const double* dw = w;
  if (!on_device) {
    h2d(ctx, dwbuf.p, w, nm);
    dw = dwbuf.p;
  }
  const uint32_t r = cfg->rank;
  NQB_REQUIRE(r >= 1, NQB_E_INVALID_RANK, "admm_factorize: rank must be >= 1");
  NQB_REQUIRE(r <= std::min(n, m), NQB_E_RANK_TOO_LARGE,
              "admm_factorize: rank exceeds min(rows, cols)");
  nqb_admm_result local;
  nqb_admm_result* res = result ? result : &local;
  Dev cu((uint64_t)n * r), cv((uint64_t)m * r), s1(n), s2(m);
  admm_device(ctx, dw, n, m, *cfg, cu.p, cv.p, nullptr, res, nullptr);
  balance_device(ctx, cu.p, cv.p, n, m, r, nullptr, nullptr, scale_floor, s1.p, s2.p);
  const uint32_t wpr = ceil_div(r, 32);
  uint32_t* words = nullptr;
  __half* halves = nullptr;
  NQB_CUDA(cudaMalloc(&words, sizeof(uint32_t) * (uint64_t)(n + m) * wpr));
  NQB_CUDA(cudaMalloc(&halves, sizeof(__half) * (uint64_t)(n + m)));
  int* flags = (int*)scratch(ctx, 7, 64) + 16;
  try {
    NQB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx->stream));
    launch_pack_rows(ctx, cu.p, n, r, words, 1, flags);            // make_factorized_layer
    launch_pack_rows(ctx, cv.p, m, r, words + (uint64_t)n * wpr, 1, flags);
    k_to_half<<<ceil_div(n, 256), 256, 0, ctx->stream>>>(s1.p, n, halves);
    NQB_LAUNCHED(ctx);
    k_to_half<<<ceil_div(m, 256), 256, 0, ctx->stream>>>(s2.p, m, halves + n);
    NQB_LAUNCHED(ctx);
    int hf = 0;
    NQB_CUDA(cudaMemcpyAsync(&hf, flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    NQB_REQUIRE(!(hf & 1), NQB_E_NON_FINITE_INPUT, "binarize: non-finite latent");
    nqb_layer* L = layer_from_device_words(ctx, n, m, r, words, words + (uint64_t)n * wpr,
                                           halves, halves + n);
    if (rel_error) {
      const uint64_t parts = rel_error_partial_count(L);
      Dev part(2 * parts + 2);
      uint32_t* vr = nullptr;
      NQB_CUDA(cudaMalloc(&vr, sizeof(uint32_t) * (uint64_t)m * L->u_words));
      layer_v_reference(ctx, L, vr, L->u_words);
      // metric of pipeline.cpp:152-153: fp64 scales, before the binary16 snap
      launch_rel_error(ctx, L, vr, L->u_words, dw, part.p, part.p + 2 * parts, s1.p, s2.p);
      double h[2];
      NQB_CUDA(cudaMemcpyAsync(h, part.p + 2 * parts, 16, cudaMemcpyDeviceToHost, ctx->stream));
      NQB_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(vr);
      const double num = std::sqrt(h[0]), den = std::sqrt(h[1]);
      *rel_error = den == 0.0 ? (num == 0.0 ? 0.0 : INFINITY) : num / den;
    }
    NQB_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = L;
  } catch (...) {
    cudaFree(words);
    cudaFree(halves);
    throw;
  }
  cudaFree(words);
  cudaFree(halves);
  API_END
}

int nqb_top_singular_pair_host(nqb_context* ctx, const double* mat, uint32_t rows, uint32_t cols,
                               int32_t max_iters, double tol, double* sigma, double* left,
                               double* right, int32_t* converged) {
  API_BEGIN
  need_ctx(ctx);
  Dev dm((uint64_t)rows * cols), dl(rows), dr(cols);
  h2d(ctx, dm.p, mat, (uint64_t)rows * cols);
  const PairResult p = top_pair_device(ctx, dm.p, rows, cols, 0, dl.p, dr.p, max_iters, tol);
  d2h(ctx, left, dl.p, rows);
  d2h(ctx, right, dr.p, cols);
  *sigma = p.sigma;
  *converged = p.converged;
  API_END
}

int nqb_spectral_norm_host(nqb_context* ctx, const double* mat, uint32_t rows, uint32_t cols,
                           int32_t iters, double* sigma) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t nm = (uint64_t)rows * cols;
  if (nm == 0) {
    *sigma = 0.0;
    return NQB_OK;
  }
  Dev dm(nm);
  h2d(ctx, dm.p, mat, nm);
  int flags = 0;
  reduce_to_host(ctx, dm.p, nullptr, nm, RED_SUMSQ, (int*)scratch(ctx, 7, 64) + 12, &flags);
  *sigma = spectral_norm_device(ctx, dm.p, rows, cols, iters, !(flags & 2));
  API_END
}

int nqb_truncated_svd_host(nqb_context* ctx, const double* mat, uint32_t rows, uint32_t cols,
                           uint32_t rank, double* u, double* v) {
  API_BEGIN
  need_ctx(ctx);
  Dev dm((uint64_t)rows * cols), du((uint64_t)rows * rank + 1), dv((uint64_t)cols * rank + 1);
  h2d(ctx, dm.p, mat, (uint64_t)rows * cols);
  truncated_svd_device(ctx, dm.p, rows, cols, rank, du.p, dv.p, nullptr);
  d2h(ctx, u, du.p, (uint64_t)rows * rank);
  d2h(ctx, v, dv.p, (uint64_t)cols * rank);
  API_END
}

int nqb_cholesky_solve_host(nqb_context* ctx, const double* a, uint32_t n, const double* b,
                            uint32_t nrhs, double* x) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t nb = (uint64_t)n * nrhs;
  Dev da((uint64_t)n * n + 1), db(nb + 1), dbt(nb + 1), dx(nb + 1);
  h2d(ctx, da.p, a, (uint64_t)n * n);
  h2d(ctx, db.p, b, nb);
  dtranspose(ctx, db.p, n, nrhs, dbt.p);  // columns of B become rows
  cholesky_solve_rows(ctx, da.p, n, dbt.p, nrhs, dx.p);
  dtranspose(ctx, dx.p, nrhs, n, db.p);
  d2h(ctx, x, db.p, nb);
  API_END
}

int nqb_svid_host(nqb_context* ctx, const double* p, uint32_t rows, uint32_t cols, double* z) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t n = (uint64_t)rows * cols;
  Dev dp(n + 1), dz(n + 1);
  h2d(ctx, dp.p, p, n);
  svid_device(ctx, dp.p, rows, cols, dz.p);
  d2h(ctx, z, dz.p, n);
  API_END
}

int nqb_admm_factor_solve_host(nqb_context* ctx, const double* target, uint32_t rows,
                               uint32_t cols, const double* fixed, uint32_t rank,
                               const double* z, const double* l, double rho, double ridge,
                               double* x) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t tr = (uint64_t)rows * cols, fr = (uint64_t)cols * rank, zr = (uint64_t)rows * rank;
  Dev dt(tr + 1), df(fr + 1), dz(zr + 1), dl(zr + 1), dx(zr + 1), gram((uint64_t)rank * rank + 1),
      rhs(zr + 1);
  h2d(ctx, dt.p, target, tr);
  h2d(ctx, df.p, fixed, fr);
  h2d(ctx, dz.p, z, zr);
  h2d(ctx, dl.p, l, zr);
  SolveWork sw{gram.p, rhs.p};
  factor_solve_device(ctx, dt.p, false, rows, cols, df.p, rank, dz.p, dl.p, rho, ridge, dx.p, sw);
  d2h(ctx, x, dx.p, zr);
  API_END
}

int nqb_augmented_lagrangian_host(nqb_context* ctx, const double* u, const double* v,
                                  const double* z_u, const double* z_v, const double* l_u,
                                  const double* l_v, uint32_t n, uint32_t m, uint32_t r,
                                  double rho, const double* target, double ridge, double* value) {
  API_BEGIN
  need_ctx(ctx);
  const uint64_t nr = (uint64_t)n * r, mr = (uint64_t)m * r, nm = (uint64_t)n * m;
  Dev du(nr + 1), dv(mr + 1), dzu(nr + 1), dzv(mr + 1), dlu(nr + 1), dlv(mr + 1), dw(nm + 1),
      scr(std::max<uint64_t>(nm, std::max(nr, mr)) + 1);
  h2d(ctx, du.p, u, nr);
  h2d(ctx, dv.p, v, mr);
  h2d(ctx, dzu.p, z_u, nr);
  h2d(ctx, dzv.p, z_v, mr);
  h2d(ctx, dlu.p, l_u, nr);
  h2d(ctx, dlv.p, l_v, mr);
  h2d(ctx, dw.p, target, nm);
  State s{n, m, r, du.p, dv.p, dzu.p, dzv.p, dlu.p, dlv.p, rho};
  *value = lagrangian_device(ctx, s, dw.p, ridge, scr.p);
  API_END
}

}  // extern "C"
