// linalg.cu — on-device fp64 linear algebra of the LB-ADMM (linalg.cpp).
//
//   power_iterate / top_singular_pair (linalg.cpp:101-136, :178-211)
//       one persistent kernel runs the WHOLE power iteration on the device:
//       every iteration streams M once (fused one-pass v <- normalize(M^T(Mv)):
//       for each row, s_i = row.v then w += s_i row while the row is still in
//       registers), so the HBM-bound SVD initialisation reads W once per
//       iteration instead of twice.  Two software grid barriers per iteration;
//       the stopping rule |sigma - sigma_prev| <= tol*sigma, the 1000/300/200
//       iteration caps, the column-norm start vector, the null-space probe and
//       the sign convention are the reference's.
//   truncated_svd_factors (linalg.cpp:218-239)
//       deflation fused with the statistics the next step needs (residual
//       norm for the early exit, the zero check, the column norms).
//   cholesky_solve (linalg.cpp:140-176)
//       symmetry check, jitter ladder {0, 1e-10, 1e-7, 1e-4} * |mean diag|,
//       blocked right-looking Cholesky (DMMA trailing updates), blocked
//       triangular solves and one refinement pass against the original A.
// All reductions use fixed trees, so results are bitwise reproducible.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_common.cuh"

#include <mutex>

namespace nqb {

// serialises cudaFuncSetAttribute + launch of the power kernels across threads
static std::mutex g_attr_mutex;


void dgemm(nqb_context*, bool, bool, uint32_t, uint32_t, uint32_t, double, const double*,
           uint32_t, const double*, uint32_t, double, double*, uint32_t);

constexpr int PI_THREADS = 512;
static bool getenv_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && *v && *v != '0';
}
constexpr uint32_t PI_MAX_COLS = 14336;

// ---------------------------------------------------------------------------
// Deterministic reductions over vectors / matrices
// ---------------------------------------------------------------------------
enum ReduceOp : int { RED_SUMSQ = 0, RED_SUMSQ_DIFF = 1, RED_DOT = 2, RED_SUMSQ_SUM = 3 };

// partial[block] = sum over this block's grid-stride share.  Also flags
// non-finite (bit0) and nonzero (bit1) entries of `a` into flags if given.
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ a,
                                                const double* __restrict__ b, uint64_t n,
                                                int op, double* __restrict__ partial,
                                                int* __restrict__ flags) {
  __shared__ double red[8];
  double s = 0.0;
  bool nonfinite = false, nonzero = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double x = a[i];
    if (flags) {
      nonfinite |= !isfinite(x);
      nonzero |= (x != 0.0);
    }
    double t;
    switch (op) {
      case RED_SUMSQ: t = x * x; break;
      case RED_SUMSQ_DIFF: { const double d = x - b[i]; t = d * d; } break;
      case RED_DOT: t = x * b[i]; break;
      default: { const double d = x + b[i]; t = d * d; } break;
    }
    s += t;
  }
  if (flags) {
    if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
    if (__any_sync(0xffffffffu, nonzero) && (threadIdx.x & 31) == 0) atomicOr(flags, 2);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum(const double* __restrict__ partial, uint32_t count, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (uint32_t k = threadIdx.x; k < count; k += blockDim.x) s += partial[k];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// Device-side result slots live in a small host-visible-by-copy array.
double reduce_to_host(nqb_context* ctx, const double* a, const double* b, uint64_t n, int op,
                      int* d_flags, int* h_flags) {
  constexpr uint32_t kBlocks = 296;
  double* part = (double*)scratch(ctx, 6, (kBlocks + 8) * sizeof(double));
  double* out = part + kBlocks;
  if (n == 0) {
    if (h_flags) *h_flags = 0;
    return 0.0;
  }
  if (d_flags) NQB_CUDA(cudaMemsetAsync(d_flags, 0, sizeof(int), ctx->stream));
  const uint32_t blocks = (uint32_t)std::min<uint64_t>(kBlocks, (n + 255) / 256);
  k_reduce<<<blocks, 256, 0, ctx->stream>>>(a, b, n, op, part, d_flags);
  NQB_LAUNCHED(ctx);
  k_sum<<<1, 512, 0, ctx->stream>>>(part, blocks, out);
  NQB_LAUNCHED(ctx);
  double h = 0.0;
  NQB_CUDA(cudaMemcpyAsync(&h, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (d_flags && h_flags)
    NQB_CUDA(cudaMemcpyAsync(h_flags, d_flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

// ---------------------------------------------------------------------------
// Column statistics: colsq[j] = sum_i M[i][j]^2 (the reference's start vector
// before sqrt, linalg.cpp:183-188), plus total sum of squares and flags.
// Optionally applies the deflation update first (linalg.cpp:231-235):
//   M[i][j] -= (sigma * left[i]) * right[j]
// Each block owns a contiguous row range; thread t owns columns t + k*blockDim.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_colstats(double* __restrict__ M, uint32_t rows,
                                                  uint32_t cols, const double* __restrict__ left,
                                                  const double* __restrict__ right, double sigma,
                                                  int deflate, double* __restrict__ colpart,
                                                  double* __restrict__ totpart,
                                                  int* __restrict__ flags) {
  __shared__ double red[16];
  const uint32_t r0 = (uint32_t)((uint64_t)rows * blockIdx.x / gridDim.x);
  const uint32_t r1 = (uint32_t)((uint64_t)rows * (blockIdx.x + 1) / gridDim.x);
  double tot = 0.0;
  bool nonfinite = false, nonzero = false;
  for (uint32_t j = threadIdx.x; j < cols; j += blockDim.x) {
    double cs = 0.0;
    const double rj = deflate ? right[j] : 0.0;
    for (uint32_t i = r0; i < r1; ++i) {
      double* p = M + (uint64_t)i * cols + j;
      double x = *p;
      if (deflate) {
        const double ui = sigma * left[i];
        x -= ui * rj;
        *p = x;
      }
      nonfinite |= !isfinite(x);
      nonzero |= (x != 0.0);
      cs += x * x;
    }
    colpart[(uint64_t)blockIdx.x * cols + j] = cs;
    tot += cs;
  }
  if (__any_sync(0xffffffffu, nonfinite) && (threadIdx.x & 31) == 0) atomicOr(flags, 1);
  if (__any_sync(0xffffffffu, nonzero) && (threadIdx.x & 31) == 0) atomicOr(flags, 2);
  tot = block_sum(tot, red);
  if (threadIdx.x == 0) totpart[blockIdx.x] = tot;
}

// v0[j] = sqrt(sum_b colpart[b][j]); total = sum_b totpart[b].
__global__ void k_colstats_finish(const double* __restrict__ colpart, uint32_t nparts,
                                  uint32_t cols, const double* __restrict__ totpart,
                                  double* __restrict__ v0, double* __restrict__ total) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < cols; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 independent load chains
    uint32_t b = 0;
    for (; b + 3 < nparts; b += 4) {
      s += colpart[(uint64_t)b * cols + j];
      s1 += colpart[(uint64_t)(b + 1) * cols + j];
      s2 += colpart[(uint64_t)(b + 2) * cols + j];
      s3 += colpart[(uint64_t)(b + 3) * cols + j];
    }
    for (; b < nparts; ++b) s += colpart[(uint64_t)b * cols + j];
    s = (s + s1) + (s2 + s3);
    v0[j] = sqrt(s);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0;
    for (uint32_t b = 0; b < nparts; ++b) s += totpart[b];
    *total = s;
  }
}

// ---------------------------------------------------------------------------
// Persistent power iteration.
// ---------------------------------------------------------------------------
struct PowerArgs {
  const double* M;
  uint32_t rows, cols;
  int abs_mode;        // iterate on |M| (svid, admm.cpp:28-32)
  int max_iters;
  double tol;
  double* v;           // [cols] in: start vector (unnormalised); out: right vector
  double* left;        // [rows] out: left vector (M v / sigma)
  double* wpart;       // [grid][cols]
  double* w;           // [cols]
  // [3][grid]: slot (it & 1) for iteration it, slot 2 for the final pass.  Phase
  // A of iteration it+1 runs before any barrier, so it must not overwrite the
  // values slower blocks are still reading in phase C of iteration it.
  double* sspart;
  double* wsspart;     // [grid] (written after a barrier: single slot is safe)
  double* out;         // [0] sigma, [1] converged, [2] iterations
  unsigned* bar;
  unsigned long long* prof;  // diagnostics (NQB_POWER_PROF): block 0 phase cycles, or null
  // k_power_stream: the first keep_num/keep_den of each block's rows are read
  // with an L2 evict_last hint so they stay L2-resident across iterations (the
  // matrix is re-read up to 1000 times per singular vector); the rest stream.
  uint32_t keep_num, keep_den;
};

template <int CPT, int RB, bool WSMEM>
__global__ void __launch_bounds__(PI_THREADS, 1) k_power(PowerArgs a) {
  extern __shared__ double smem[];
  double* vs = smem;                                  // [cols]
  double* wsm = smem + a.cols;                        // [CPT][PI_THREADS] if WSMEM
  __shared__ double red[RB][PI_THREADS / 32];
  __shared__ double bred[PI_THREADS / 32];
  const uint32_t tid = threadIdx.x, G = gridDim.x, bid = blockIdx.x;
  unsigned gsk = 0;  // grid barriers passed
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t r0 = (uint32_t)((uint64_t)a.rows * bid / G);
  const uint32_t r1 = (uint32_t)((uint64_t)a.rows * (bid + 1) / G);

  // v <- v / ||v|| (normalize, linalg.cpp:70-75); every block computes the
  // same value with the same tree.
  double sq = 0.0;
  for (uint32_t j = tid; j < a.cols; j += PI_THREADS) {
    const double x = a.v[j];
    vs[j] = x;
    sq += x * x;
  }
  double nrm = sqrt(block_sum(sq, bred));
  if (nrm > 0.0)
    for (uint32_t j = tid; j < a.cols; j += PI_THREADS) vs[j] /= nrm;
  __syncthreads();

  double wloc[WSMEM ? 1 : CPT];
  double sigma = 0.0, sigma_prev = -1.0;
  int converged = 0, it = 0;
  for (it = 0; it < a.max_iters; ++it) {
    // ---- phase A: s_i = M_i . v ; w += s_i M_i  (one pass over M) ----------
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if constexpr (WSMEM) wsm[c * PI_THREADS + tid] = 0.0;
      else wloc[c] = 0.0;
    }
    double ss = 0.0;
    for (uint32_t i0 = r0; i0 < r1; i0 += RB) {
      double row[RB][CPT];
      double part[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        part[q] = 0.0;
        const uint32_t i = i0 + q;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t j = tid + c * PI_THREADS;
          double x = 0.0;
          if (i < r1 && j < a.cols) {
            x = __ldg(a.M + (uint64_t)i * a.cols + j);
            if (a.abs_mode) x = fabs(x);
          }
          row[q][c] = x;
        }
      }
#pragma unroll
      for (int q = 0; q < RB; ++q)
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          const uint32_t j = tid + c * PI_THREADS;
          if (j < a.cols) part[q] += row[q][c] * vs[j];
        }
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const double p = warp_sum(part[q]);
        if (lane == 0) red[q][warp] = p;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < PI_THREADS / 32; ++k) s += red[q][k];
        if (i0 + q < r1) {
          ss += s * s;
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            if constexpr (WSMEM) wsm[c * PI_THREADS + tid] += row[q][c] * s;
            else wloc[c] += row[q][c] * s;
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) {
        if constexpr (WSMEM) a.wpart[(uint64_t)bid * a.cols + j] = wsm[c * PI_THREADS + tid];
        else a.wpart[(uint64_t)bid * a.cols + j] = wloc[c];
      }
    }
    double* ssp = a.sspart + (size_t)(it & 1) * G;
    if (tid == 0) ssp[bid] = ss;
    grid_sync(a.bar, G, gsk);

    // ---- phase B: w = sum_b wpart[b] (fixed order), ||w||^2 partials --------
    double wq = 0.0;
    for (uint32_t j = bid * PI_THREADS + tid; j < a.cols; j += G * PI_THREADS) {
      double s = 0.0;
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 independent load chains
      uint32_t b = 0;
      for (; b + 3 < G; b += 4) {
        s += __ldcg(a.wpart + (uint64_t)b * a.cols + j);
        s1 += __ldcg(a.wpart + (uint64_t)(b + 1) * a.cols + j);
        s2 += __ldcg(a.wpart + (uint64_t)(b + 2) * a.cols + j);
        s3 += __ldcg(a.wpart + (uint64_t)(b + 3) * a.cols + j);
      }
      for (; b < G; ++b) s += __ldcg(a.wpart + (uint64_t)b * a.cols + j);
      s = (s + s1) + (s2 + s3);
      a.w[j] = s;
      wq += s * s;
    }
    wq = block_sum(wq, bred);
    if (tid == 0) a.wsspart[bid] = wq;
    grid_sync(a.bar, G, gsk);

    // ---- phase C (every block, identical): sigma, normalise, stop rule ------
    // G partials: one (independent) load per thread, then the fixed block tree
    // (identical in every block) instead of G dependent L2 round trips.
    double s2 = 0.0, w2 = 0.0;
    for (uint32_t b = tid; b < G; b += PI_THREADS) {
      s2 += __ldcg(ssp + b);
      w2 += __ldcg(a.wsspart + b);
    }
    s2 = block_sum(s2, bred);
    w2 = block_sum(w2, bred);
    sigma = sqrt(s2);
    if (sigma == 0.0) break;  // linalg.cpp:111
    const double wn = sqrt(w2);
    for (uint32_t j = tid; j < a.cols; j += PI_THREADS) {
      const double x = __ldcg(a.w + j);
      vs[j] = wn > 0.0 ? x / wn : x;
    }
    __syncthreads();
    if (sigma_prev >= 0.0 && fabs(sigma - sigma_prev) <= a.tol * fmax(sigma, 1e-300)) {
      converged = 1;
      ++it;
      break;
    }
    sigma_prev = sigma;
  }

  // ---- final: mv = M v, sigma = ||mv||, left = mv / sigma (linalg.cpp:124-130)
  double ss = 0.0;
  for (uint32_t i = r0; i < r1; ++i) {
    double p = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) {
        double x = __ldg(a.M + (uint64_t)i * a.cols + j);
        if (a.abs_mode) x = fabs(x);
        p += x * vs[j];
      }
    }
    const double s = block_sum(p, bred);
    if (tid == 0) {
      a.left[i] = s;
      ss += s * s;
    }
  }
  double* ssf = a.sspart + 2 * (size_t)G;
  if (tid == 0) ssf[bid] = ss;
  grid_sync(a.bar, G, gsk);
  double s2 = 0.0;
  for (uint32_t b = tid; b < G; b += PI_THREADS) s2 += __ldcg(ssf + b);
  s2 = block_sum(s2, bred);
  const double fsig = sqrt(s2);
  for (uint32_t i = r0 + tid; i < r1; i += PI_THREADS) {
    a.left[i] = fsig > 0.0 ? a.left[i] / fsig : 0.0;
  }
  if (bid == 0) {
    for (uint32_t j = tid; j < a.cols; j += PI_THREADS) a.v[j] = vs[j];
    if (tid == 0) {
      a.out[0] = fsig;
      a.out[1] = (fsig > 0.0) ? (double)converged : 0.0;
      a.out[2] = (double)it;
    }
  }
}

// ---------------------------------------------------------------------------
// Streaming persistent power iteration (even column counts).  Same algorithm
// and outputs as k_power; each block's rows stream through a shared-memory
// ring filled by 1-D TMA bulk copies (HBM-bound phase A with the next rows
// already in flight), and the cross-block reduction of w is spread over all
// blocks and warps with independent loads (phase B), fixed order throughout.
// ---------------------------------------------------------------------------
constexpr int PS_MAX_SLOTS = 8;

// RS: rows per step (one bulk copy, one block barrier and one reduction tree per
// step; the per-step latency is the bound of phase A, so more rows per step
// amortise it).  nslots is a multiple of RS.
template <int CPT, int RS>
__global__ void __launch_bounds__(PI_THREADS, 1) k_power_stream(PowerArgs a, uint32_t nslots,
                                                               uint32_t row_bytes) {
  extern __shared__ __align__(128) uint8_t ring[];               // nslots x row_bytes
  __shared__ uint64_t fullb[PS_MAX_SLOTS];
  __shared__ double bred[PI_THREADS / 32];
  __shared__ double cred[PI_THREADS / 32][33];
  __shared__ double cred2[2][PI_THREADS / 32][RS];  // phase A: per-warp dot partials, by step parity
  constexpr bool kKeep = CPT <= 12;  // phase A keeps each row pair in registers
  const uint32_t tid = threadIdx.x, G = gridDim.x, bid = blockIdx.x;
  unsigned gsk = 0;  // grid barriers passed
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t r0 = (uint32_t)((uint64_t)a.rows * bid / G);
  const uint32_t r1 = (uint32_t)((uint64_t)a.rows * (bid + 1) / G);
  const uint32_t nrows = r1 - r0;
  const uint32_t cb0 = (uint32_t)((uint64_t)a.cols * bid / G);
  const uint32_t cb1 = (uint32_t)((uint64_t)a.cols * (bid + 1) / G);
  if (tid == 0) {
    for (uint32_t s = 0; s < nslots; ++s) tc::mbar_init(&fullb[s], 1);
    tc::fence_mbar_init();
  }
  // v lives in registers: thread t owns columns t + c*PI_THREADS
  double vr[CPT];
  double sq = 0.0;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const uint32_t j = tid + c * PI_THREADS;
    vr[c] = j < a.cols ? a.v[j] : 0.0;
    sq += vr[c] * vr[c];
  }
  const double nrm = sqrt(block_sum(sq, bred));  // normalize (linalg.cpp:70-75)
  if (nrm > 0.0)
#pragma unroll
    for (int c = 0; c < CPT; ++c) vr[c] /= nrm;
  __syncthreads();

  uint32_t phase = 0;  // bit s: parity of the next completion of slot s
  uint32_t pending = 0;  // rows of the NEXT pass already issued (prefetched)
  const uint32_t keep = a.keep_den ? (uint32_t)((uint64_t)nrows * a.keep_num / a.keep_den) : 0;
  const uint64_t pol_keep = tc::policy_evict_last(), pol_stream = tc::policy_evict_first();
  // rows r0+i .. r0+i+RS-1 (i a multiple of RS) -> consecutive slots from
  // i % nslots in ONE bulk copy signalling fullb[i % nslots]
  auto issue = [&](uint32_t i) {
    uint64_t* bar = &fullb[i % nslots];
    const uint32_t bytes = min((uint32_t)RS, nrows - i) * row_bytes;
    tc::mbar_arrive_expect_tx(bar, bytes);
    tc::bulk_g2s_hint(ring + (size_t)(i % nslots) * row_bytes, a.M + (uint64_t)(r0 + i) * a.cols,
                      bytes, bar, i < keep ? pol_keep : pol_stream);
  };
  const uint32_t head = nrows < nslots ? nrows : nslots;
  double sigma = 0.0, sigma_prev = -1.0;
  int converged = 0, it = 0;
  long long tA = 0, tB = 0, tC = 0, t0 = clock64();
  for (it = 0; it < a.max_iters; ++it) {
    if (a.prof) t0 = clock64();
    // ---- phase A: s_i = M_i . v ; w += s_i M_i, rows streamed through smem,
    // two rows per block reduction.  The first `head` rows of this pass were
    // prefetched at the end of the previous pass (rows do not change).
    if (tid == 0 && !pending)
      for (uint32_t i = 0; i < head; i += RS) issue(i);
    pending = 0;
    double wl[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) wl[c] = 0.0;
    double ss = 0.0;
    uint32_t par = 0;  // cred2 buffer of this step
    for (uint32_t i = 0; i < nrows; i += RS) {
      const uint32_t cnt = min((uint32_t)RS, nrows - i);
      const uint32_t s0 = i % nslots;  // the step's rows sit in slots s0 .. s0+RS-1
      tc::mbar_wait(&fullb[s0], (phase >> s0) & 1u);
      phase ^= 1u << s0;
      const double* xs = (const double*)(ring + (size_t)s0 * row_bytes);
      const uint32_t rstride = row_bytes / 8;
      // The step's rows are read from shared memory once and kept in registers
      // for the axpy after the block reduction (kKeep); wide rows re-read them.
      double xr[kKeep ? RS : 1][kKeep ? CPT : 1];
      double pp[RS][2];
#pragma unroll
      for (int r = 0; r < RS; ++r) pp[r][0] = pp[r][1] = 0.0;
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const uint32_t j = tid + c * PI_THREADS;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
          double x = 0.0;
          if (j < a.cols && (uint32_t)r < cnt) {
            x = xs[(size_t)r * rstride + j];
            if (a.abs_mode) x = fabs(x);
            pp[r][c & 1] += x * vr[c];  // two independent chains per row
          }
          if constexpr (kKeep) xr[r][c] = x;
        }
      }
      double pr[RS];
#pragma unroll
      for (int r = 0; r < RS; ++r) pr[r] = pp[r][0] + pp[r][1];
      // the step's dot products through one fixed tree (identical in every thread)
#pragma unroll
      for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int r = 0; r < RS; ++r) pr[r] += __shfl_xor_sync(~0u, pr[r], o);
      double* cr = &cred2[par][0][0];
      if (lane == 0)
#pragma unroll
        for (int r = 0; r < RS; ++r) cr[RS * warp + r] = pr[r];
      __syncthreads();
      if constexpr (kKeep) {
        // the rows are in registers now: refill their slots right away (the
        // copies overlap the axpy; one barrier per step, cred double-buffered).
        // The issuing lane rotates over the warps: a bulk-copy issue costs its
        // warp several hundred cycles, and the next barrier waits for that warp.
        if (tid == (uint32_t)(32 * ((i / RS) % (PI_THREADS / 32)))) {
          const uint32_t nx = i + nslots;
          if (nx < nrows) issue(nx);
        }
      }
      // cross-warp sums: lane w < warps holds warp w's partial, one xor tree
      // per warp (fixed order, identical everywhere)
      static_assert(PI_THREADS / 32 <= 32, "warps per block");
      double sr[RS];
#pragma unroll
      for (int r = 0; r < RS; ++r) {
        double t = lane < PI_THREADS / 32 ? cr[RS * lane + r] : 0.0;
#pragma unroll
        for (int o = PI_THREADS / 64; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
        sr[r] = __shfl_sync(~0u, t, 0);
        if ((uint32_t)r < cnt) ss += sr[r] * sr[r];
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const uint32_t j = tid + c * PI_THREADS;
        if (j < a.cols) {
#pragma unroll
          for (int r = 0; r < RS; ++r) {
            if ((uint32_t)r >= cnt) break;
            double x;
            if constexpr (kKeep) {
              x = xr[r][c];
            } else {
              x = xs[(size_t)r * rstride + j];
              if (a.abs_mode) x = fabs(x);
            }
            wl[c] += x * sr[r];
          }
        }
      }
      if constexpr (!kKeep) {
        __syncthreads();  // everyone is done with these slots
        if (tid == 0) {
          const uint32_t nx = i + nslots;  // refill the freed slots
          if (nx < nrows) issue(nx);
        }
      }
      par ^= 1;
    }
    __syncthreads();  // (kKeep) the last step's cred reads are done
    // prefetch the next pass's first rows now: they stream while the
    // reductions and grid barriers below run (drained before exit)
    if (it + 1 < a.max_iters) {
      if (tid == 0)
        for (uint32_t i = 0; i < head; i += RS) issue(i);
      pending = 1;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) a.wpart[(uint64_t)bid * a.cols + j] = wl[c];
    }
    double* ssp = a.sspart + (size_t)(it & 1) * G;
    if (tid == 0) ssp[bid] = ss;
    long long t1 = a.prof ? clock64() : 0;
    grid_sync(a.bar, G, gsk);

    // ---- phase B: w_j = sum_b wpart[b][j] for this block's columns; warp k
    // sums partials b = k, k+16, ... (independent loads), then a fixed-order
    // cross-warp sum.
    double wq = 0.0;
    for (uint32_t c0 = cb0; c0 < cb1; c0 += 32) {
      const uint32_t j = c0 + lane;
      double acc = 0.0;
      if (j < cb1) {
        // every partial of this lane in flight at once (one L2 round trip),
        // then a fixed pairwise tree; grids beyond 10 x 16 blocks fold the rest
        constexpr int kQ = 10;
        double q[kQ];
#pragma unroll
        for (int t = 0; t < kQ; ++t) {
          const uint32_t b = warp + 16u * t;
          q[t] = b < G ? __ldcg(a.wpart + (uint64_t)b * a.cols + j) : 0.0;
        }
        for (uint32_t b = warp + 16u * kQ; b < G; b += 16) q[0] += __ldcg(a.wpart + (uint64_t)b * a.cols + j);
        acc = (((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]))) + (q[8] + q[9]);
      }
      cred[warp][lane] = acc;
      __syncthreads();
      if (warp == 0 && j < cb1) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < PI_THREADS / 32; ++k) s += cred[k][lane];
        a.w[j] = s;
        wq += s * s;
      }
      __syncthreads();
    }
    // only warp 0 holds column sums: its warp tree equals block_sum here
    // (the other warps would add exact zeros), without two block barriers
    if (warp == 0) {
      wq = warp_sum(wq);
      if (lane == 0) a.wsspart[bid] = wq;
    }
    grid_sync(a.bar, G, gsk);
    long long t2 = a.prof ? clock64() : 0;
    if (a.prof) {
      tA += t1 - t0;
      tB += t2 - t1;
    }

    // ---- phase C (every block, identical): sigma, normalise, stop rule ------
    // G partials: one (independent) load per thread, then the fixed block tree
    // (identical in every block) instead of G dependent L2 round trips.
    // w is loaded before the two norms are reduced (its L2 latency overlaps the
    // reductions); both norms share one pair of barriers (same summation order
    // as block_sum).
    double wx[kKeep ? CPT : 1];
    if constexpr (kKeep) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const uint32_t j = tid + c * PI_THREADS;
        wx[c] = j < a.cols ? __ldcg(a.w + j) : 0.0;
      }
    }
    double s2 = 0.0, w2 = 0.0;
    for (uint32_t b = tid; b < G; b += PI_THREADS) {
      s2 += __ldcg(ssp + b);
      w2 += __ldcg(a.wsspart + b);
    }
    s2 = warp_sum(s2);
    w2 = warp_sum(w2);
    __syncthreads();
    if (lane == 0) {  // cred: phase B is done with it, the next use is after a barrier
      cred[warp][0] = s2;
      cred[warp][1] = w2;
    }
    __syncthreads();
    s2 = 0.0;
    w2 = 0.0;
    for (int w = 0; w < PI_THREADS / 32; ++w) {
      s2 += cred[w][0];
      w2 += cred[w][1];
    }
    sigma = sqrt(s2);
    if (sigma == 0.0) break;  // linalg.cpp:111
    const double wn = sqrt(w2);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) {
        const double x = kKeep ? wx[c] : __ldcg(a.w + j);
        vr[c] = wn > 0.0 ? x / wn : x;
      }
    }
    if (a.prof) tC += clock64() - t2;
    if (sigma_prev >= 0.0 && fabs(sigma - sigma_prev) <= a.tol * fmax(sigma, 1e-300)) {
      converged = 1;
      ++it;
      break;
    }
    sigma_prev = sigma;
  }
  if (a.prof && bid == 0 && tid == 0) {
    atomicAdd(a.prof + 0, (unsigned long long)tA);
    atomicAdd(a.prof + 1, (unsigned long long)tB);
    atomicAdd(a.prof + 2, (unsigned long long)tC);
    atomicAdd(a.prof + 3, (unsigned long long)it);
  }

  if (pending) {  // an early exit left the next pass's prefetch in flight: drain it
    for (uint32_t i = 0; i < head; i += RS) {
      tc::mbar_wait(&fullb[i % nslots], (phase >> (i % nslots)) & 1u);
      phase ^= 1u << (i % nslots);
    }
  }

  // ---- final: mv = M v, sigma = ||mv||, left = mv / sigma (linalg.cpp:124-130)
  double ss = 0.0;
  for (uint32_t i = r0; i < r1; ++i) {
    double p = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) {
        double x = __ldg(a.M + (uint64_t)i * a.cols + j);
        if (a.abs_mode) x = fabs(x);
        p += x * vr[c];
      }
    }
    const double s = block_sum(p, bred);
    if (tid == 0) {
      a.left[i] = s;
      ss += s * s;
    }
  }
  double* ssf = a.sspart + 2 * (size_t)G;
  if (tid == 0) ssf[bid] = ss;
  grid_sync(a.bar, G, gsk);
  double s2 = 0.0;
  for (uint32_t b = tid; b < G; b += PI_THREADS) s2 += __ldcg(ssf + b);
  s2 = block_sum(s2, bred);
  const double fsig = sqrt(s2);
  for (uint32_t i = r0 + tid; i < r1; i += PI_THREADS) {
    a.left[i] = fsig > 0.0 ? a.left[i] / fsig : 0.0;
  }
  if (bid == 0) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t j = tid + c * PI_THREADS;
      if (j < a.cols) a.v[j] = vr[c];
    }
    if (tid == 0) {
      a.out[0] = fsig;
      a.out[1] = (fsig > 0.0) ? (double)converged : 0.0;
      a.out[2] = (double)it;
    }
  }
}

template <int CPT>
static void launch_power_stream(nqb_context* ctx, PowerArgs& a, uint32_t grid) {
  const uint32_t row_bytes = a.cols * 8;  // cols even: 16-byte multiple, 16-byte aligned rows
  uint32_t nslots = (uint32_t)std::min<size_t>(PS_MAX_SLOTS, (200 * 1024) / row_bytes);
  // Row pairs per step (>= 2 slots: dispatch condition).  Three rows per step
  // (NQB_POWER_RS3=1, six slots) measured slower: 42.4k vs 39.2k cycles per
  // iteration at 4096^2 (registers: the 24 kept values spill).
  // (only instantiated where it can run: CPT <= 8)
  const bool three = CPT <= 8 && nslots >= 6 && getenv_flag("NQB_POWER_RS3");
  nslots = three ? nslots / 3 * 3 : (nslots & ~1u);
  const size_t smem = (size_t)nslots * row_bytes;
  auto kern = k_power_stream<CPT, 2>;
  if constexpr (CPT <= 8) {
    if (three) kern = k_power_stream<CPT, 3>;
  }
  // the attribute is per function, not per launch: concurrent contexts (one per
  // worker thread) must not set a smaller bound between another thread's set and
  // its launch (cudaErrorInvalidValue), so set + launch hold one lock
  std::lock_guard<std::mutex> attr_lock(g_attr_mutex);
  NQB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {&a, &nslots, (void*)&row_bytes};
  // grid_sync's monotonic counter must start at a multiple of this grid
  NQB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned long long), ctx->stream));
  NQB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(PI_THREADS), args,
                                       smem, ctx->stream));
  NQB_LAUNCHED(ctx);
}

struct PowerWork {
  double* wpart;
  double* w;
  double* sspart;
  double* wsspart;
  double* out;
};

template <int CPT, int RB, bool WSMEM>
static void launch_power_t(nqb_context* ctx, PowerArgs& a, uint32_t grid) {
  const size_t smem = sizeof(double) * (a.cols + (WSMEM ? (size_t)CPT * PI_THREADS : 0));
  auto kern = k_power<CPT, RB, WSMEM>;
  // the attribute is per function, not per launch: concurrent contexts (one per
  // worker thread) must not set a smaller bound between another thread's set and
  // its launch (cudaErrorInvalidValue), so set + launch hold one lock
  std::lock_guard<std::mutex> attr_lock(g_attr_mutex);
  NQB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {&a};
  // grid_sync's monotonic counter must start at a multiple of this grid
  NQB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned long long), ctx->stream));
  NQB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(PI_THREADS), args,
                                       smem, ctx->stream));
  NQB_LAUNCHED(ctx);
}

// Runs power_iterate on the device.  d_v holds the start vector (overwritten
// by the right singular vector), d_left receives the left vector.  Returns
// sigma, converged and the iteration count (host values).
void power_iterate_device(nqb_context* ctx, const double* d_m, uint32_t rows, uint32_t cols,
                          int abs_mode, double* d_v, double* d_left, int max_iters, double tol,
                          double* sigma, int* converged, int* iters) {
  NQB_REQUIRE(cols <= PI_MAX_COLS, NQB_E_VALIDATION,
              "power iteration supports at most 14336 columns");
  const uint32_t grid = std::max(1u, std::min<uint32_t>(rows, ctx->num_sms));
  double* base = (double*)scratch(ctx, 5, sizeof(double) * ((size_t)grid * cols + cols + 4 * grid + 8));
  PowerArgs a;
  a.M = d_m;
  a.rows = rows;
  a.cols = cols;
  a.abs_mode = abs_mode;
  a.max_iters = max_iters;
  a.tol = tol;
  a.v = d_v;
  a.left = d_left;
  a.wpart = base;
  a.w = base + (size_t)grid * cols;
  a.sspart = a.w + cols;
  a.wsspart = a.sspart + 3 * grid;
  a.out = a.wsspart + grid;
  a.bar = ctx->barrier;
  a.prof = nullptr;
  {  // L2-resident share of the matrix (NQB_POWER_L2_MB, default 40 of the 126 MB L2: phase A
     // is SM-bound either way; 40 MB leaves the most L2 for the partial sums of phase B)
    static const uint64_t budget = [] {
      const char* e = std::getenv("NQB_POWER_L2_MB");
      return (uint64_t)(e ? std::strtoul(e, nullptr, 10) : 40ul) << 20;
    }();
    const uint64_t total = (uint64_t)rows * cols * 8;
    static bool limit_set = false;  // evict_last lines live in the persisting L2 set-aside
    if (!limit_set && budget) {
      cudaDeviceProp pr;
      NQB_CUDA(cudaGetDeviceProperties(&pr, ctx->device));
      const size_t want = std::min<size_t>(budget, (size_t)pr.persistingL2CacheMaxSize);
      if (want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      cudaGetLastError();
      limit_set = true;
    }
    a.keep_den = 1u << 20;
    a.keep_num = total ? (uint32_t)std::min<uint64_t>(a.keep_den, budget * a.keep_den / total) : 0;
  }
  static unsigned long long* prof_buf = nullptr;
  if (getenv_flag("NQB_POWER_PROF")) {
    if (!prof_buf) {
      NQB_CUDA(cudaMalloc(&prof_buf, 128));
      NQB_CUDA(cudaMemset(prof_buf, 0, 128));
    }
    a.prof = prof_buf;
  }
  const uint32_t cpt = ceil_div(cols, PI_THREADS);
  const bool stream = (cols % 2 == 0) && 2 * (size_t)cols * 8 <= 200 * 1024 &&
                      cpt <= 22 && rows >= 2 * grid && !getenv_flag("NQB_POWER_LEGACY");
  if (stream) {
    if (cpt <= 2) launch_power_stream<2>(ctx, a, grid);
    else if (cpt <= 4) launch_power_stream<4>(ctx, a, grid);
    else if (cpt <= 8) launch_power_stream<8>(ctx, a, grid);
    else if (cpt <= 12) launch_power_stream<12>(ctx, a, grid);
    else if (cpt <= 16) launch_power_stream<16>(ctx, a, grid);
    else launch_power_stream<22>(ctx, a, grid);
  } else if (cpt <= 2) launch_power_t<2, 8, false>(ctx, a, grid);
  else if (cpt <= 4) launch_power_t<4, 8, false>(ctx, a, grid);
  else if (cpt <= 8) launch_power_t<8, 4, false>(ctx, a, grid);
  else if (cpt <= 12) launch_power_t<12, 2, false>(ctx, a, grid);
  else if (cpt <= 16) launch_power_t<16, 2, false>(ctx, a, grid);
  else if (cpt <= 20) launch_power_t<20, 1, true>(ctx, a, grid);
  else if (cpt <= 24) launch_power_t<24, 1, true>(ctx, a, grid);
  else launch_power_t<28, 1, true>(ctx, a, grid);
  double h[3];
  NQB_CUDA(cudaMemcpyAsync(h, a.out, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  *sigma = h[0];
  *converged = (int)h[1];
  *iters = (int)h[2];
  if (a.prof) {
    unsigned long long hp[9];
    NQB_CUDA(cudaMemcpy(hp, a.prof, sizeof(hp), cudaMemcpyDeviceToHost));
    const double it = (double)std::max(1ull, hp[3]);
    fprintf(stderr, "power_prof rows=%u cols=%u iters=%llu cyc/iter: A %.0f B %.0f C %.0f\n", rows,
            cols, hp[3], hp[0] / it, hp[1] / it, hp[2] / it);
  }
}

// Column statistics (and optional deflation) on the device.  Writes the
// column-norm start vector into d_v0 and returns the total sum of squares and
// the flags (bit0 non-finite, bit1 nonzero) on the host.
double colstats_device(nqb_context* ctx, double* d_m, uint32_t rows, uint32_t cols,
                       const double* d_left, const double* d_right, double sigma, int deflate,
                       double* d_v0, int* h_flags) {
  const uint32_t grid = std::max(1u, std::min<uint32_t>(rows, 2 * ctx->num_sms));
  double* base = (double*)scratch(ctx, 4, sizeof(double) * ((size_t)grid * cols + grid + 4) + 64);
  double* colpart = base;
  double* totpart = base + (size_t)grid * cols;
  double* total = totpart + grid;
  int* flags = (int*)(total + 2);
  NQB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), ctx->stream));
  k_colstats<<<grid, 512, 0, ctx->stream>>>(d_m, rows, cols, d_left, d_right, sigma, deflate,
                                            colpart, totpart, flags);
  NQB_LAUNCHED(ctx);
  k_colstats_finish<<<ceil_div(cols, 256), 256, 0, ctx->stream>>>(colpart, grid, cols, totpart,
                                                                 d_v0, total);
  NQB_LAUNCHED(ctx);
  double h[2];
  int f = 0;
  NQB_CUDA(cudaMemcpyAsync(h, total, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaMemcpyAsync(&f, flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  *h_flags = f;
  return h[0];
}

// ---------------------------------------------------------------------------
// Sign convention (linalg.cpp:200-209): the first index of max |right| must be
// nonnegative, else flip both vectors.  Single block, deterministic.
// ---------------------------------------------------------------------------
__global__ void k_sign_convention(double* __restrict__ right, uint32_t cols,
                                  double* __restrict__ left, uint32_t rows) {
  __shared__ double bv[1024];
  __shared__ uint32_t bi[1024];
  __shared__ int flip;
  double best = -1.0;
  uint32_t arg = 0;
  for (uint32_t j = threadIdx.x; j < cols; j += blockDim.x) {
    const double a = fabs(right[j]);
    if (a > best) {  // strict: keeps the first index within this thread's stride
      best = a;
      arg = j;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = arg;
  __syncthreads();
  for (uint32_t s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ob = bv[threadIdx.x + s];
      const uint32_t oi = bi[threadIdx.x + s];
      if (ob > bv[threadIdx.x] || (ob == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = ob;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) flip = (cols > 0 && right[bi[0]] < 0.0) ? 1 : 0;
  __syncthreads();
  if (flip) {
    for (uint32_t j = threadIdx.x; j < cols; j += blockDim.x) right[j] = -right[j];
    for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) left[i] = -left[i];
  }
}

__global__ void k_basis(double* __restrict__ v, uint32_t cols, uint32_t j) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cols; k += gridDim.x * blockDim.x)
    v[k] = (k == j) ? 1.0 : 0.0;
}

struct PairResult {
  double sigma;
  int converged;
  int iters;
};

// top_singular_pair (linalg.cpp:178-211) given the column-norm start vector
// already in d_right (as computed by colstats_device).  The zero check is the
// caller's (it owns the flags).
PairResult top_pair_from_start(nqb_context* ctx, const double* d_m, uint32_t rows, uint32_t cols,
                               int abs_mode, double* d_left, double* d_right, int max_iters,
                               double tol) {
  PairResult r{0.0, 0, 0};
  power_iterate_device(ctx, d_m, rows, cols, abs_mode, d_right, d_left, max_iters, tol, &r.sigma,
                       &r.converged, &r.iters);
  for (uint32_t j = 0; j < cols && r.sigma == 0.0; ++j) {  // linalg.cpp:191-198
    k_basis<<<ceil_div(cols, 256), 256, 0, ctx->stream>>>(d_right, cols, j);
    NQB_LAUNCHED(ctx);
    power_iterate_device(ctx, d_m, rows, cols, abs_mode, d_right, d_left, max_iters, tol,
                         &r.sigma, &r.converged, &r.iters);
  }
  k_sign_convention<<<1, 1024, 0, ctx->stream>>>(d_right, cols, d_left, rows);
  NQB_LAUNCHED(ctx);
  return r;
}

// Full top_singular_pair on a device matrix (zero check + start vector).
PairResult top_pair_device(nqb_context* ctx, const double* d_m, uint32_t rows, uint32_t cols,
                           int abs_mode, double* d_left, double* d_right, int max_iters,
                           double tol) {
  int flags = 0;
  colstats_device(ctx, const_cast<double*>(d_m), rows, cols, nullptr, nullptr, 0.0, 0, d_right,
                  &flags);
  NQB_REQUIRE(flags & 2, NQB_E_ZERO_MATRIX, "top_singular_pair: matrix is identically zero");
  return top_pair_from_start(ctx, d_m, rows, cols, abs_mode, d_left, d_right, max_iters, tol);
}

// ---------------------------------------------------------------------------
// truncated_svd_factors (linalg.cpp:218-239)
// ---------------------------------------------------------------------------
__global__ void k_store_factor_col(const double* __restrict__ vec, uint32_t len, double root,
                                   double* __restrict__ f, uint32_t ld, uint32_t k) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    f[(uint64_t)i * ld + k] = root * vec[i];
}

struct SvdStats {
  uint32_t steps = 0;
  uint64_t iters = 0;
  uint32_t converged = 0;
};

// d_res: working copy of M (destroyed).  d_u (rows x rank), d_v (cols x rank)
// are zero-filled first (columns past an early exit stay zero, like the
// reference's DenseMatrix(n, rank)).
void truncated_svd_device(nqb_context* ctx, double* d_res, uint32_t rows, uint32_t cols,
                          uint32_t rank, double* d_u, double* d_v, SvdStats* stats) {
  NQB_CUDA(cudaMemsetAsync(d_u, 0, sizeof(double) * rows * (size_t)rank, ctx->stream));
  NQB_CUDA(cudaMemsetAsync(d_v, 0, sizeof(double) * cols * (size_t)rank, ctx->stream));
  double* vec = (double*)scratch(ctx, 3, sizeof(double) * ((size_t)rows + cols + 8));
  double* left = vec;
  double* right = vec + rows;
  int flags = 0;
  const double scale_sq = colstats_device(ctx, d_res, rows, cols, nullptr, nullptr, 0.0, 0, right,
                                          &flags);
  const double scale = std::sqrt(scale_sq);
  double res_sq = scale_sq;
  for (uint32_t k = 0; k < rank; ++k) {
    if (std::sqrt(res_sq) <= 1e-14 * scale) break;  // rank exhausted
    NQB_REQUIRE(flags & 2, NQB_E_ZERO_MATRIX, "top_singular_pair: matrix is identically zero");
    const PairResult p = top_pair_from_start(ctx, d_res, rows, cols, 0, left, right, 1000, 1e-13);
    if (stats) {
      stats->steps++;
      stats->iters += (uint64_t)p.iters;
      stats->converged += p.converged ? 1u : 0u;
    }
    const double root = std::sqrt(p.sigma);
    k_store_factor_col<<<ceil_div(rows, 256), 256, 0, ctx->stream>>>(left, rows, root, d_u, rank, k);
    NQB_LAUNCHED(ctx);
    k_store_factor_col<<<ceil_div(cols, 256), 256, 0, ctx->stream>>>(right, cols, root, d_v, rank, k);
    NQB_LAUNCHED(ctx);
    // residual -= (sigma l) r^T, fused with the next step's norm / start vector.
    res_sq = colstats_device(ctx, d_res, rows, cols, left, right, p.sigma, 1, right, &flags);
  }
}

// ---------------------------------------------------------------------------
// Cholesky (lower, in place, row-major ld) — blocked right-looking.
// ---------------------------------------------------------------------------
constexpr int CH_NB = 32;

// Factor the jb x jb diagonal block at (j0, j0) (already updated).  One block
// of 32x32 threads; unblocked column Cholesky in shared memory, exactly the
// reference's recurrence within the block.  flag |= 1 on a non-positive or
// non-finite pivot (linalg.cpp:32).
__global__ void k_potrf_diag(double* __restrict__ A, uint32_t ld, uint32_t j0, uint32_t jb,
                             int* __restrict__ flag) {
  __shared__ double s[CH_NB][CH_NB + 1];
  const uint32_t tx = threadIdx.x, ty = threadIdx.y;
  if (tx < jb && ty < jb) s[ty][tx] = A[(uint64_t)(j0 + ty) * ld + j0 + tx];
  __syncthreads();
  for (uint32_t j = 0; j < jb; ++j) {
    if (ty == 0 && tx == 0) {
      double d = s[j][j];
      for (uint32_t k = 0; k < j; ++k) d -= s[j][k] * s[j][k];
      if (!(d > 0.0) || !isfinite(d)) {
        atomicOr(flag, 1);
        d = 1.0;
      }
      s[j][j] = sqrt(d);
    }
    __syncthreads();
    if (tx == 0 && ty > j && ty < jb) {
      double v = s[ty][j];
      for (uint32_t k = 0; k < j; ++k) v -= s[ty][k] * s[j][k];
      s[ty][j] = v / s[j][j];
    }
    __syncthreads();
  }
  if (tx < jb && ty < jb && tx <= ty) A[(uint64_t)(j0 + ty) * ld + j0 + tx] = s[ty][tx];
}

// Panel: rows i >= j0+jb: L[i][j0:j0+jb] = A[i][j0:j0+jb] L11^{-T} (forward
// substitution per row, one thread per row).
__global__ void k_potrf_panel(double* __restrict__ A, uint32_t ld, uint32_t n, uint32_t j0,
                              uint32_t jb) {
  __shared__ double l11[CH_NB][CH_NB + 1];
  for (uint32_t e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const uint32_t r = e / jb, c = e % jb;
    l11[r][c] = A[(uint64_t)(j0 + r) * ld + j0 + c];
  }
  __syncthreads();
  const uint32_t i = j0 + jb + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[CH_NB];
  double* row = A + (uint64_t)i * ld + j0;
#pragma unroll
  for (int c = 0; c < CH_NB; ++c) {
    if ((uint32_t)c < jb) {
      double s = row[c];
      for (int k = 0; k < c; ++k) s -= x[k] * l11[c][k];
      x[c] = s / l11[c][c];
      row[c] = x[c];
    }
  }
}

// Returns false if the factorisation hit a bad pivot.
bool cholesky_device(nqb_context* ctx, double* d_a, uint32_t n, uint32_t ld) {
  int* flag = (int*)scratch(ctx, 7, 64) + 4;
  NQB_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  for (uint32_t j0 = 0; j0 < n; j0 += CH_NB) {
    const uint32_t jb = std::min<uint32_t>(CH_NB, n - j0);
    k_potrf_diag<<<1, dim3(CH_NB, CH_NB), 0, ctx->stream>>>(d_a, ld, j0, jb, flag);
    NQB_LAUNCHED(ctx);
    const uint32_t j1 = j0 + jb;
    if (j1 < n) {
      k_potrf_panel<<<ceil_div(n - j1, 128), 128, 0, ctx->stream>>>(d_a, ld, n, j0, jb);
      NQB_LAUNCHED(ctx);
      // A22 -= L21 L21^T
      const double* l21 = d_a + (uint64_t)j1 * ld + j0;
      dgemm(ctx, false, true, n - j1, n - j1, jb, -1.0, l21, ld, l21, ld, 1.0,
            d_a + (uint64_t)j1 * ld + j1, ld);
    }
  }
  int h = 0;
  NQB_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}

// ---------------------------------------------------------------------------
// Triangular solves on the rows of B (nrows x n, row-major ld = n):
//   forward:  Y L^T = B   (y_c = (b_c - sum_{k<c} y_k L[c][k]) / L[c][c])
//   backward: X L   = Y   (x_c = (y_c - sum_{k>c} x_k L[k][c]) / L[c][c])
// which is cholesky_backsolve (linalg.cpp:44-62) applied to every RHS at once.
// Blocked by TS_NB columns with DMMA updates of the remaining columns.
// ---------------------------------------------------------------------------
constexpr int TS_NB = 32;

template <bool kForward>
__global__ void k_trsm_block(double* __restrict__ B, uint32_t nrows, uint32_t n,
                             const double* __restrict__ Lm, uint32_t ld, uint32_t j0,
                             uint32_t jb) {
  __shared__ double l[TS_NB][TS_NB + 1];
  for (uint32_t e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const uint32_t r = e / jb, c = e % jb;
    l[r][c] = Lm[(uint64_t)(j0 + r) * ld + j0 + c];
  }
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double* row = B + (uint64_t)i * n + j0;
  double x[TS_NB];
#pragma unroll
  for (int c = 0; c < TS_NB; ++c) x[c] = ((uint32_t)c < jb) ? row[c] : 0.0;
  if (kForward) {
#pragma unroll
    for (int c = 0; c < TS_NB; ++c) {
      if ((uint32_t)c < jb) {
        double s = x[c];
        for (int k = 0; k < c; ++k) s -= l[c][k] * x[k];
        x[c] = s / l[c][c];
      }
    }
  } else {
#pragma unroll
    for (int c = TS_NB - 1; c >= 0; --c) {
      if ((uint32_t)c < jb) {
        double s = x[c];
        for (int k = c + 1; k < (int)jb; ++k) s -= l[k][c] * x[k];
        x[c] = s / l[c][c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < TS_NB; ++c)
    if ((uint32_t)c < jb) row[c] = x[c];
}

// B <- B L^{-T} L^{-1}  (i.e. each row b <- A^{-1} b with A = L L^T).
void cholesky_backsolve_rows(nqb_context* ctx, double* d_b, uint32_t nrows, uint32_t n,
                             const double* d_l, uint32_t ld) {
  // forward: Y L^T = B
  for (uint32_t j0 = 0; j0 < n; j0 += TS_NB) {
    const uint32_t jb = std::min<uint32_t>(TS_NB, n - j0);
    k_trsm_block<true><<<ceil_div(nrows, 128), 128, 0, ctx->stream>>>(d_b, nrows, n, d_l, ld, j0, jb);
    NQB_LAUNCHED(ctx);
    const uint32_t j1 = j0 + jb;
    if (j1 < n) {  // B[:, j1:] -= Y_J L[j1:, J]^T
      dgemm(ctx, false, true, nrows, n - j1, jb, -1.0, d_b + j0, n, d_l + (uint64_t)j1 * ld + j0,
            ld, 1.0, d_b + j1, n);
    }
  }
  // backward: X L = Y, last column block first
  const uint32_t nblk = ceil_div(n, TS_NB);
  for (int bk = (int)nblk - 1; bk >= 0; --bk) {
    const uint32_t j0 = (uint32_t)bk * TS_NB;
    const uint32_t jb = std::min<uint32_t>(TS_NB, n - j0);
    k_trsm_block<false><<<ceil_div(nrows, 128), 128, 0, ctx->stream>>>(d_b, nrows, n, d_l, ld, j0, jb);
    NQB_LAUNCHED(ctx);
    if (j0 > 0) {  // Y[:, :j0] -= X_J L[J, :j0]
      dgemm(ctx, false, false, nrows, j0, jb, -1.0, d_b + j0, n, d_l + (uint64_t)j0 * ld, ld, 1.0,
            d_b, n);
    }
  }
}

// Symmetry statistics: max |a_ij|, max |a_ij - a_ji| (j > i), sum of diag.
__global__ void k_sym_stats(const double* __restrict__ a, uint32_t n, double* __restrict__ out) {
  __shared__ double m1[256], m2[256], dg[256];
  double mabs = 0.0, masym = 0.0, ds = 0.0;
  for (uint64_t e = threadIdx.x; e < (uint64_t)n * n; e += blockDim.x) {
    const uint32_t i = (uint32_t)(e / n), j = (uint32_t)(e % n);
    const double x = a[e];
    mabs = fmax(mabs, fabs(x));
    if (j > i) masym = fmax(masym, fabs(x - a[(uint64_t)j * n + i]));
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) ds += a[(uint64_t)i * n + i];
  m1[threadIdx.x] = mabs;
  m2[threadIdx.x] = masym;
  dg[threadIdx.x] = ds;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0, z = 0.0;
    for (int k = 0; k < 256; ++k) {
      x = fmax(x, m1[k]);
      y = fmax(y, m2[k]);
      z += dg[k];
    }
    out[0] = x;
    out[1] = y;
    out[2] = z;
  }
}

__global__ void k_add_diag(double* __restrict__ a, uint32_t n, uint32_t ld, double add) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[(uint64_t)i * ld + i] += add;
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, uint64_t n,
                       double alpha) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    y[i] += alpha * x[i];
}

// cholesky_solve (linalg.cpp:140-176) with the right-hand sides as ROWS:
// X (nrows x n) solves X A = B, i.e. A x_i = b_i for every row (A symmetric).
// d_a: n x n (not modified); d_b: nrows x n (not modified); d_x: output.
void cholesky_solve_rows(nqb_context* ctx, const double* d_a, uint32_t n, const double* d_b,
                         uint32_t nrows, double* d_x) {
  const uint64_t nb = (uint64_t)nrows * n;
  int flags = 0;
  reduce_to_host(ctx, d_b, nullptr, nb, RED_SUMSQ, (int*)scratch(ctx, 7, 64) + 8, &flags);
  NQB_REQUIRE(!(flags & 1), NQB_E_NON_FINITE_INPUT, "cholesky_solve: non-finite input");
  reduce_to_host(ctx, d_a, nullptr, (uint64_t)n * n, RED_SUMSQ, (int*)scratch(ctx, 7, 64) + 8,
                 &flags);
  NQB_REQUIRE(!(flags & 1), NQB_E_NON_FINITE_INPUT, "cholesky_solve: non-finite input");
  double* st = (double*)scratch(ctx, 2, sizeof(double) * ((size_t)n * n + nb + 8));
  double* lbuf = st + 8;
  double* rbuf = lbuf + (size_t)n * n;
  k_sym_stats<<<1, 256, 0, ctx->stream>>>(d_a, n, st);
  NQB_LAUNCHED(ctx);
  double hs[3];
  NQB_CUDA(cudaMemcpyAsync(hs, st, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream));
  NQB_CUDA(cudaStreamSynchronize(ctx->stream));
  NQB_REQUIRE(!(hs[1] > 1e-9 * std::max(hs[0], 1e-300)), NQB_E_NOT_SYMMETRIC,
              "matrix is not symmetric");
  const double mean_diag = n > 0 ? hs[2] / (double)n : 0.0;
  static const double kJitter[] = {0.0, 1e-10, 1e-7, 1e-4};
  for (double delta : kJitter) {
    NQB_CUDA(cudaMemcpyAsync(lbuf, d_a, sizeof(double) * n * (size_t)n, cudaMemcpyDeviceToDevice,
                             ctx->stream));
    if (delta > 0.0) {
      const double add = delta * std::fabs(mean_diag);
      if (add == 0.0) continue;
      k_add_diag<<<ceil_div(n, 256), 256, 0, ctx->stream>>>(lbuf, n, n, add);
      NQB_LAUNCHED(ctx);
    }
    if (!cholesky_device(ctx, lbuf, n, n)) continue;
    // x = backsolve(b)
    NQB_CUDA(cudaMemcpyAsync(d_x, d_b, sizeof(double) * nb, cudaMemcpyDeviceToDevice, ctx->stream));
    cholesky_backsolve_rows(ctx, d_x, nrows, n, lbuf, n);
    // residual = b - x A  (rows);  x += backsolve(residual)
    NQB_CUDA(cudaMemcpyAsync(rbuf, d_b, sizeof(double) * nb, cudaMemcpyDeviceToDevice, ctx->stream));
    dgemm(ctx, false, false, nrows, n, n, -1.0, d_x, n, d_a, n, 1.0, rbuf, n);
    cholesky_backsolve_rows(ctx, rbuf, nrows, n, lbuf, n);
    k_axpy<<<std::min<uint64_t>(4096, (nb + 255) / 256), 256, 0, ctx->stream>>>(d_x, rbuf, nb, 1.0);
    NQB_LAUNCHED(ctx);
    reduce_to_host(ctx, d_x, nullptr, nb, RED_SUMSQ, (int*)scratch(ctx, 7, 64) + 8, &flags);
    if (flags & 1) continue;
    return;
  }
  fail(NQB_E_NOT_POSITIVE_DEFINITE, "cholesky_solve: factorization failed after jitter escalation");
}

}  // namespace nqb
