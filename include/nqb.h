/*
 * nqb.h — C ABI of the B200-native binary low-rank (BLR) hot path.
 *
 * This library replaces, one entry point at a time, the C++ value API of the
 * NanoQuant reference (/root/reference/proj, "the reference" below) for the
 * path named by BASELINE.json's north_star:
 *
 *   (1) the BLR-linear forward  y = s1 .* U_b (V_b^T (s2 .* x))      packed.hpp:49-102
 *   (2) the LB-ADMM initialisation producing U_b, V_b, s1, s2 from W admm.hpp:30-85,
 *       linalg.hpp:35-51, balance.hpp:38-41, storage.hpp:82-91
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - Matrices are row-major, element (i,j) at i*cols + j, exactly like the
 *     reference DenseMatrix (dense.hpp:27-75).
 *   - Packed sign matrices use the reference PackedBitMatrix layout
 *     (packed.hpp:25-46): ceil(cols/32) little-endian u32 words per row, bit b of
 *     word w is column 32w+b, 1 <=> +1, padding bits zero.  The device keeps its
 *     own re-laid-out copy inside an nqb_layer; conversion is
 *     bit-exact both ways.
 *   - Every function returns an nqb_status.  The two reference error kinds
 *     (errors.hpp:25-35: validation / numerical) map one-to-one onto status
 *     ranges, and each reference exception type on this path has its own code,
 *     so a C++ shim can rethrow the identical type.
 *   - "_host" entry points take host buffers and do their own H2D/D2H copies
 *     (the drop-in path a reference caller uses); "_device" entry points take
 *     device pointers and only enqueue work on the context stream.
 *   - There is no CPU fallback: without a usable CUDA device nqb_create fails
 *     with NQB_E_NO_DEVICE and nothing else can be called.
 */
#ifndef NQB_H
#define NQB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* Status codes (errors.hpp:25-114)                                          */
/* ------------------------------------------------------------------------ */
typedef enum nqb_status {
  NQB_OK = 0,
  /* ErrorKind::kValidation (CLI exit 2, nanoquant_main.cpp:423-429) */
  NQB_E_DIMENSION_MISMATCH = 1,   /* DimensionMismatch   errors.hpp:37-40 */
  NQB_E_NON_FINITE_INPUT = 2,     /* NonFiniteInput      errors.hpp:59-62 */
  NQB_E_NON_BINARY_ENTRY = 3,     /* NonBinaryEntry      errors.hpp:69-72 */
  NQB_E_CORRUPT_PADDING = 4,      /* CorruptPadding      errors.hpp:74-77 */
  NQB_E_RANK_TOO_LARGE = 5,       /* RankTooLarge        errors.hpp:79-82 */
  NQB_E_INVALID_RANK = 6,         /* InvalidRank         errors.hpp:84-87 */
  NQB_E_NOT_SYMMETRIC = 7,        /* NotSymmetric        errors.hpp:42-45 */
  NQB_E_TARGET_TOO_SMALL = 8,     /* TargetTooSmall      errors.hpp:99-102 */
  NQB_E_VALIDATION = 9,           /* plain Error(kValidation, ...) e.g. admm.cpp:134-136 */
  NQB_E_PARSE = 10,               /* ParseError          errors.hpp:109-111 */
  NQB_E_IO = 11,                  /* IoError             errors.hpp:104-106 */
  NQB_E_EMPTY_STATS = 12,         /* EmptyStats          errors.hpp:63-66 */
  /* ErrorKind::kNumerical (CLI exit 3) */
  NQB_E_ZERO_MATRIX = 32,         /* ZeroMatrix          errors.hpp:53-57 */
  NQB_E_NOT_POSITIVE_DEFINITE = 33, /* NotPositiveDefinite errors.hpp:47-51 */
  NQB_E_NON_FINITE_LOSS = 34,       /* NonFiniteLoss       refine.hpp:72-77 */
  /* runtime (no reference counterpart) */
  NQB_E_CUDA = 64,
  NQB_E_OUT_OF_MEMORY = 65,
  NQB_E_NO_DEVICE = 66,
  NQB_E_INTERNAL = 67
} nqb_status;

/* 0 = ok, 1 = validation, 2 = numerical, 3 = runtime */
int nqb_status_kind(int status);
/* Message of the last failing call on this thread ("" if none). */
const char* nqb_last_error(void);
/* Library build string (arch, git describe). */
const char* nqb_version(void);

/* ------------------------------------------------------------------------ */
/* Context: device, stream, workspaces.                                      */
/* ------------------------------------------------------------------------ */
typedef struct nqb_context nqb_context;

int nqb_create(int device, nqb_context** out);
int nqb_destroy(nqb_context* ctx);
/* Use an external cudaStream_t (NULL = the context's own stream). */
int nqb_set_stream(nqb_context* ctx, void* cuda_stream);
/* Registers a host range for the _host entry points: page-locks and maps it if it
 * is not already page-locked, and remembers its device alias, so those calls move
 * it by DMA or zero-copy without probing the pointer each call (outputs of
 * nqb_gemv_f32_host are written through the alias; nqb_pass_run_host moves
 * registered buffers with one copy kernel per direction).  Unregister before
 * freeing the memory. */
int nqb_host_register(nqb_context* ctx, void* ptr, size_t bytes);
int nqb_host_unregister(nqb_context* ctx, void* ptr);
void* nqb_get_stream(nqb_context* ctx);
int nqb_synchronize(nqb_context* ctx);
/* Limit the persistent ADMM kernels of this context to `sms` SMs (<= 0: all),
 * so several contexts can factorize matrices concurrently on one device.
 * Decode plans built afterwards use the same budget. */
int nqb_set_sm_budget(nqb_context* ctx, int sms);
/* Device kernels launched by this context since creation (instrumentation). */
uint64_t nqb_kernel_launches(const nqb_context* ctx);

/* ------------------------------------------------------------------------ */
/* Rank rule (storage.cpp:124-141)                                           */
/* ------------------------------------------------------------------------ */
int nqb_rank_for_target_bpw(uint64_t n, uint64_t m, double target_bpw, uint32_t* rank);

/* ------------------------------------------------------------------------ */
/* Synthetic weights (rng.hpp:25-58): out[i] = scale * Rng(seed).gaussian(),  */
/* i-th call of one stream, rounded to fp32 and back when snap_f32 (NQMX      */
/* precision, io.cpp:117-119).  SURVEY §8(d) rows 1 and 4: W = fp32(0.02 g).  */
/* Host only, multi-threaded, bitwise equal to the reference stream.          */
/* ------------------------------------------------------------------------ */
int nqb_synthetic_weight_host(uint64_t seed, uint64_t count, double scale, int snap_f32,
                              double* out);

/* ------------------------------------------------------------------------ */
/* Sign binarisation and packing (packed.cpp:51-103)                         */
/* on_device != 0: pointers are device pointers (async on the ctx stream).   */
/* ------------------------------------------------------------------------ */
/* binarize: x < 0 ? -1 : +1 (sign(0) = sign(-0) = +1); NonFiniteInput. */
int nqb_binarize(nqb_context* ctx, const double* latent, uint64_t count, double* out,
                 int on_device);
/* pack_signs: entries must be exactly +-1 (else NQB_E_NON_BINARY_ENTRY). */
int nqb_pack_signs(nqb_context* ctx, const double* signs, uint32_t rows, uint32_t cols,
                   uint32_t* words, int on_device);
/* binarize + pack in one pass: bit = !(x < 0). */
int nqb_pack_latent(nqb_context* ctx, const double* latent, uint32_t rows, uint32_t cols,
                    uint32_t* words, int on_device);
/* unpack_signs: NQB_E_CORRUPT_PADDING if any pad bit is set. */
int nqb_unpack_signs(nqb_context* ctx, const uint32_t* words, uint32_t rows, uint32_t cols,
                     double* signs, int on_device);

/* ------------------------------------------------------------------------ */
/* Device-resident factorized layer (FactorizedLayer, packed.hpp:57-72)      */
/* ------------------------------------------------------------------------ */
typedef struct nqb_layer nqb_layer;

/* Uploads a layer given in the reference layout (host pointers).  Scales are
 * stored on the device as IEEE binary16, round-to-nearest-even exactly like
 * double_to_half (half.hpp:83-85) - the NQPK on-disk precision (io.cpp:153-154).
 * Pad bits must be zero (NQB_E_CORRUPT_PADDING otherwise). */
int nqb_layer_upload(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                     const uint32_t* u_words, const uint32_t* v_words,
                     const double* s1, const double* s2, nqb_layer** out);
/* Same, scales already binary16 bit patterns (NQPK payload). */
int nqb_layer_upload_f16(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                         const uint32_t* u_words, const uint32_t* v_words,
                         const uint16_t* s1_half, const uint16_t* s2_half, nqb_layer** out);
/* Same as nqb_layer_upload, and the layer also keeps the exact fp64 scales, as
 * the reference FactorizedLayer does in memory (packed.hpp:57-72): the exact
 * paths (reconstruct_dense, gemv f64, gemm f64, gemv f32 host, download) use
 * them, the binary16 hot kernels keep the snapped copy.  Used by the C++ shim. */
int nqb_layer_upload_exact(nqb_context* ctx, uint32_t n, uint32_t m, uint32_t r,
                           const uint32_t* u_words, const uint32_t* v_words,
                           const double* s1, const double* s2, nqb_layer** out);
int nqb_layer_free(nqb_layer* layer);
int nqb_layer_shape(const nqb_layer* layer, uint32_t* n, uint32_t* m, uint32_t* r);
/* Bytes the decode GEMV must stream for this layer (device layout). */
uint64_t nqb_layer_device_bytes(const nqb_layer* layer);
/* Reference-layout words (bit-exact inverse of upload) and scales (half->double). */
int nqb_layer_download(nqb_context* ctx, const nqb_layer* layer, uint32_t* u_words,
                       uint32_t* v_words, double* s1, double* s2);

/* ------------------------------------------------------------------------ */
/* Forward (packed.cpp:153-287)                                              */
/* ------------------------------------------------------------------------ */
/* gemv_packed_f32 (packed.cpp:201-204): x[m] -> y[n], host buffers. */
int nqb_gemv_f32_host(nqb_context* ctx, const nqb_layer* layer, const float* x, float* y);
/* gemv_packed (packed.cpp:196-199): fp64 accumulation, host buffers. */
int nqb_gemv_f64_host(nqb_context* ctx, const nqb_layer* layer, const double* x, double* y);
/* Decode GEMV on device buffers (the hot kernel).  fp32 in/out. */
int nqb_gemv_f32_device(nqb_context* ctx, const nqb_layer* layer, const float* d_x, float* d_y);
/* Decode GEMV, binary16 in/out (bit patterns). */
int nqb_gemv_f16_device(nqb_context* ctx, const nqb_layer* layer, const uint16_t* d_x,
                        uint16_t* d_y);
/* Batched forward (gemm_packed, packed.cpp:260-287): X is m x b row-major fp64
 * host, Y is n x b row-major fp64 host.  fp64 accumulation on CUDA cores in the
 * reference's column order (within 1e-10 of gemm_packed). */
int nqb_gemm_f64_host(nqb_context* ctx, const nqb_layer* layer, const double* x, uint32_t b,
                      double* y);
/* Prefill GEMM on device buffers: X is b x m row-major binary16 (token-major),
 * Y is b x n row-major binary16. */
int nqb_gemm_f16_device(nqb_context* ctx, const nqb_layer* layer, const uint16_t* d_x,
                        uint32_t b, uint16_t* d_y);
/* Decode groups: 1..4 layers that read the same input x (q/k/v share the
 * attention input, gate/up the MLP input).  One launch of the fused decode
 * kernel computes every layer of the group; a single layer is
 * a group of one (nqb_gemv_*_device use the layer's own implicit group).
 * The group keeps its own copy of the bits in the decode layout and refers
 * to the layers' scales: free the group before its layers. */
typedef struct nqb_group nqb_group;
int nqb_group_create(nqb_context* ctx, const nqb_layer* const* layers, uint32_t count,
                     nqb_group** out);
int nqb_group_free(nqb_group* group);
uint64_t nqb_group_stream_bytes(const nqb_group* group);
/* d_ys[i] receives layer i's output (n_i elements). */
int nqb_group_gemv_f16_device(nqb_context* ctx, const nqb_group* group, const uint16_t* d_x,
                              uint16_t* const* d_ys);
int nqb_group_gemv_f32_device(nqb_context* ctx, const nqb_group* group, const float* d_x,
                              float* const* d_ys);
/* Programmatic Dependent Launch of decode kernels (default on): a decode
 * kernel starts streaming its bits while the previous kernel finishes. */
int nqb_set_pdl(nqb_context* ctx, int enable);

/* Diagnostics: one f16 decode launch of `layer` with per-CTA %globaltimer
 * stamps (32 words per CTA: 16 ns stamps, see decode.cu TRACE points, then
 * smid and the CTA's work).  stamps holds 32*grid. */
int nqb_debug_decode_trace(nqb_context* ctx, const nqb_layer* layer, const uint16_t* d_x,
                           uint16_t* d_y, uint64_t* stamps, uint32_t* grid);

/* Decode passes: a whole sequence of decode launches (e.g. the 224 linear
 * layers of a decoder, as q/k/v, o, gate/up, down steps) run by ONE launch of
 * a persistent kernel.  Each step is a decode group (or one
 * layer) with its device input and outputs; buffers are fixed at creation.
 * A step whose input overlaps an earlier step's output waits for that output
 * inside the kernel (dependencies are found from the buffer ranges), and takes
 * its activation bound from the producer's published max|y|; independent
 * steps overlap.  Results equal the per-call kernel's up to that bound (same
 * arithmetic).  Groups and layers must outlive the pass. */
typedef struct nqb_pass nqb_pass;
typedef struct nqb_pass_step {
  const nqb_group* group;  /* layers sharing the input, or NULL to use `layer` */
  const nqb_layer* layer;  /* a single layer (its own decode plan) */
  const void* d_x;         /* device input, m elements */
  void* d_y[4];            /* device outputs, one per layer of the group */
  int32_t f32;             /* 0: binary16 in/out, 1: fp32 in/out */
  int32_t reserved;
} nqb_pass_step;
int nqb_pass_create(nqb_context* ctx, uint32_t count, const nqb_pass_step* steps,
                    nqb_pass** out);
int nqb_pass_launch(nqb_context* ctx, const nqb_pass* pass);
int nqb_pass_free(nqb_pass* pass);
/* One pass end to end with host buffers: hx[k] (or NULL: input left as is, e.g.
 * produced by an earlier step) is copied into step k's input, the pass runs on
 * the context stream, and hy[i] (one per layer of every step, in step order;
 * NULL: not read back) receives the outputs; returns when they are on the
 * host. */
int nqb_pass_run_host(nqb_context* ctx, const nqb_pass* pass, const void* const* hx,
                      void* const* hy);
/* The same with the host buffers bound once (a serving loop's pinned or
 * registered token buffers): nqb_pass_io_create resolves every buffer's device
 * alias and uploads the two copy lists; nqb_pass_io_run then moves the inputs,
 * launches the pass and moves the outputs with three launches and one
 * synchronisation, no per-call host work.  Every non-NULL buffer must be
 * page-locked (cudaHostAlloc / torch pin_memory) or registered with
 * nqb_host_register (NQB_E_VALIDATION otherwise: use nqb_pass_run_host). */
typedef struct nqb_pass_io nqb_pass_io;
int nqb_pass_io_create(nqb_context* ctx, const nqb_pass* pass, const void* const* hx,
                       void* const* hy, nqb_pass_io** out);
int nqb_pass_io_run(nqb_context* ctx, const nqb_pass_io* io);
int nqb_pass_io_free(nqb_pass_io* io);
/* Bits streamed per launch, and the algorithmic bytes of the pass: per layer
 * r(n+m)/8 + 2(n+m) scales + y, plus x once per step. */
uint64_t nqb_pass_stream_bytes(const nqb_pass* pass);
uint64_t nqb_pass_algorithmic_bytes(const nqb_pass* pass);
/* Diagnostics: one launch with per-CTA %globaltimer stamps: stamps holds
 * grid * (2 * count + 2) words: [start, per step (t barrier passed, stage 2
 * done), end]. */
int nqb_debug_pass_trace(nqb_context* ctx, const nqb_pass* pass, uint64_t* stamps,
                         uint32_t* grid);

/* CUDA graphs of library calls on the context stream (e.g. one decode pass
 * over a layer stack), replayed with a single launch.  Between begin and end
 * only device-buffer entry points may be called. */
typedef struct nqb_graph nqb_graph;
int nqb_graph_begin(nqb_context* ctx);
int nqb_graph_end(nqb_context* ctx, nqb_graph** out);
int nqb_graph_launch(nqb_context* ctx, const nqb_graph* graph);
int nqb_graph_free(nqb_graph* graph);

/* reconstruct_dense (packed.cpp:126-149): n x m fp64, host buffer. */
int nqb_reconstruct_dense_host(nqb_context* ctx, const nqb_layer* layer, double* w);

/* ------------------------------------------------------------------------ */
/* LB-ADMM initialisation (admm.cpp:127-199)                                 */
/* ------------------------------------------------------------------------ */
typedef struct nqb_admm_config {  /* AdmmConfig, admm.hpp:41-51 */
  uint32_t rank;
  int32_t max_iters;     /* default 400 */
  double rho_start;      /* 0,0 => auto 0.1*sigma_max .. 10*sigma_max */
  double rho_end;
  double ridge;          /* default 1e-4 */
  double tol;            /* default 1e-4 */
  uint64_t seed;         /* unused by the solver (admm.hpp:50), kept for parity */
  int32_t record_trace;  /* nonzero: evaluate the augmented Lagrangian each step */
  int32_t reserved;
} nqb_admm_config;

typedef struct nqb_admm_result {  /* AdmmState scalars, admm.hpp:53-62 */
  uint32_t iteration;
  int32_t converged;
  double primal_residual;
  double rho;
  uint32_t trace_len;           /* entries written to trace (0 if not recorded) */
  uint32_t svd_steps;           /* deflation steps actually taken */
  uint64_t svd_power_iters;     /* power iterations summed over deflation steps */
  uint32_t svd_converged_steps; /* deflation steps whose power iteration converged */
  uint32_t reserved;
  double sigma_max;             /* spectral norm estimate used for auto rho */
  double seconds_svd_init;      /* device time of truncated_svd_factors */
  double seconds_iterations;    /* device time of the ADMM loop */
} nqb_admm_result;

void nqb_admm_config_default(nqb_admm_config* cfg);

/* admm_factorize: W n x m fp64 host; consensus P_U = U + L_U (n x r) and
 * P_V = V + L_V (m x r) host; trace (capacity max_iters + 1) may be NULL. */
int nqb_admm_factorize_host(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                            const nqb_admm_config* cfg, double* consensus_u,
                            double* consensus_v, double* trace, nqb_admm_result* result);
/* Same, plus the final AdmmState matrices (admm.hpp:53-62): state[0..5] = U (n x r),
 * V (m x r), Z_U, Z_V, L_U, L_V host buffers, each may be NULL (state may be NULL). */
int nqb_admm_factorize_state_host(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                                  const nqb_admm_config* cfg, double* consensus_u,
                                  double* consensus_v, double* trace, nqb_admm_result* result,
                                  double* const* state);
/* Same on device buffers (w, consensus_u, consensus_v device; trace host or NULL). */
int nqb_admm_factorize_device(nqb_context* ctx, const double* d_w, uint32_t n, uint32_t m,
                              const nqb_admm_config* cfg, double* d_consensus_u,
                              double* d_consensus_v, double* trace, nqb_admm_result* result);

/* balance_and_extract_scales (balance.cpp:36-65).  diag_out (n) / diag_in (m)
 * may be NULL (identity preconditioner).  Host buffers. */
int nqb_balance_host(nqb_context* ctx, const double* consensus_u, const double* consensus_v,
                     uint32_t n, uint32_t m, uint32_t r, const double* diag_out,
                     const double* diag_in, double scale_floor, double* latent_u,
                     double* latent_v, double* s1, double* s2, double* eta);

/* One whole matrix, as pipeline.cpp:95-110 + :150 does it: ADMM on W (fp64,
 * device or host per on_device), balance with identity preconditioner, binarize
 * + pack on device, scales to binary16.  Returns a device layer and, if
 * rel_error != NULL, relative_frobenius_error(W, reconstruct_dense(layer))
 * computed on the device. */
int nqb_factorize_layer(nqb_context* ctx, const double* w, uint32_t n, uint32_t m,
                        const nqb_admm_config* cfg, double scale_floor, int on_device,
                        nqb_layer** out, nqb_admm_result* result, double* rel_error);

/* Relative Frobenius error ||W - reconstruct_dense(layer)|| / ||W|| on device,
 * W on host (on_device = 0) or device. */
int nqb_layer_rel_error(nqb_context* ctx, const nqb_layer* layer, const double* w,
                        int on_device, double* rel_error);

/* ------------------------------------------------------------------------ */
/* STE refinement on the device (refine.cpp:285-384, 420-425) */
/* ------------------------------------------------------------------------ */
typedef struct nqb_tune_config {  /* TuneConfig, refine.hpp:55-64 */
  int32_t epochs;          /* default 8 */
  int32_t batch_size;      /* default 4 */
  double learning_rate;    /* default 1e-4 */
  int32_t schedule;        /* 0 constant, 1 cosine (default) */
  int32_t reserved;
  uint64_t seed;
} nqb_tune_config;

/* ste_refine on one factorized latent layer (the pipeline's per-layer group,
 * pipeline.cpp:128-135): Adam on latent_u (n x r), latent_v (m x r), s1 (n), s2 (m)
 * against sum_c w_c ||teacher - forward(x)||^2 with the straight-through sign,
 * x (m x b) and teacher (n x b) as columns, column_weights (b) or NULL.  The four
 * host buffers are overwritten with the best-loss checkpoint (also on
 * NQB_E_NON_FINITE_LOSS, like NonFiniteLoss::best_chain); best_loss may be NULL. */
int nqb_ste_refine_layer_host(nqb_context* ctx, double* latent_u, double* latent_v, double* s1,
                              double* s2, uint32_t n, uint32_t m, uint32_t r, const double* x,
                              const double* teacher, uint32_t b, const double* column_weights,
                              const nqb_tune_config* cfg, double* best_loss);

/* ------------------------------------------------------------------------ */
/* Linear-algebra building blocks (linalg.hpp:35-51, admm.hpp:30-38, 65-67)  */
/* All host buffers; used by the C++ shim and the parity tests.               */
/* ------------------------------------------------------------------------ */
int nqb_top_singular_pair_host(nqb_context* ctx, const double* m, uint32_t rows,
                               uint32_t cols, int32_t max_iters, double tol, double* sigma,
                               double* left, double* right, int32_t* converged);
int nqb_spectral_norm_host(nqb_context* ctx, const double* m, uint32_t rows, uint32_t cols,
                           int32_t iters, double* sigma);
int nqb_truncated_svd_host(nqb_context* ctx, const double* m, uint32_t rows, uint32_t cols,
                           uint32_t rank, double* u, double* v);
int nqb_cholesky_solve_host(nqb_context* ctx, const double* a, uint32_t n, const double* b,
                            uint32_t nrhs, double* x);
int nqb_svid_host(nqb_context* ctx, const double* p, uint32_t rows, uint32_t cols, double* z);
int nqb_admm_factor_solve_host(nqb_context* ctx, const double* target, uint32_t rows,
                               uint32_t cols, const double* fixed, uint32_t rank,
                               const double* z, const double* l, double rho, double ridge,
                               double* x);
/* augmented_lagrangian (admm.cpp:82-96): U n x r, V m x r, target n x m. */
int nqb_augmented_lagrangian_host(nqb_context* ctx, const double* u, const double* v,
                                  const double* z_u, const double* z_v, const double* l_u,
                                  const double* l_v, uint32_t n, uint32_t m, uint32_t r,
                                  double rho, const double* target, double ridge,
                                  double* value);
/* fp64 GEMM on device (DMMA tensor cores): C = alpha * op(A) op(B) + beta * C,
 * row-major, op = transpose if trans_* != 0. */
int nqb_dgemm_device(nqb_context* ctx, int trans_a, int trans_b, uint32_t m, uint32_t n,
                     uint32_t k, double alpha, const double* d_a, uint32_t lda,
                     const double* d_b, uint32_t ldb, double beta, double* d_c, uint32_t ldc);

/* ------------------------------------------------------------------------ */
/* Preconditioner, phase 1 of the pipeline (precondition.cpp:37-153,          */
/* pipeline.cpp:63-72), SURVEY §8(f) row 3.  Bitwise equal to the reference.  */
/* ------------------------------------------------------------------------ */
/* accumulate_stats (precondition.cpp:37-62): batch is rows(samples) x cols(channels)
 * row-major fp64; the caller owns the ChannelStats state (sum_squares[cols],
 * sample_count, tau) and passes it in/out.  rows == 0 is a no-op.  Errors:
 * NQB_E_VALIDATION (percentile outside (0,1)), NQB_E_NON_FINITE_INPUT. */
int nqb_accumulate_stats_host(nqb_context* ctx, const double* batch, uint64_t rows, uint32_t cols,
                              double percentile, double* sum_squares, uint64_t* sample_count,
                              double* tau);
int nqb_accumulate_stats_device(nqb_context* ctx, const double* d_batch, uint64_t rows,
                                uint32_t cols, double percentile, double* sum_squares,
                                uint64_t* sample_count, double* tau);
/* build_preconditioner (precondition.cpp:99-121): out_sum_squares == NULL means no
 * gradient-side stats (diag_out = identity, tau_max = max(in_tau, 1)).  Errors:
 * NQB_E_EMPTY_STATS, NQB_E_VALIDATION (gamma outside [0,1], eps_floor <= 0). */
int nqb_build_preconditioner(uint32_t in_channels, const double* in_sum_squares,
                             uint64_t in_count, double in_tau, uint32_t out_channels,
                             const double* out_sum_squares, uint64_t out_count, double out_tau,
                             double gamma, double eps_floor, double* diag_in, double* diag_out,
                             double* tau_max);
/* precondition_weight (precondition.cpp:123-138): W <- D_out W D_in in place; a NULL
 * diagonal is the identity. */
int nqb_precondition_weight_host(nqb_context* ctx, double* w, uint32_t rows, uint32_t cols,
                                 const double* diag_out, const double* diag_in);
int nqb_precondition_weight_device(nqb_context* ctx, double* d_w, uint32_t rows, uint32_t cols,
                                   const double* d_diag_out, const double* d_diag_in);
/* unprecondition_rows (precondition.cpp:143-153): factor rows /= diag (NULL: identity). */
int nqb_unprecondition_rows_host(nqb_context* ctx, double* factor, uint32_t rows, uint32_t cols,
                                 const double* diag);

/* ------------------------------------------------------------------------ */
/* NQPK packed-model files (io.hpp:27-54, io.cpp:139-193) */
/* ------------------------------------------------------------------------ */
/* Host-side parse of the reference's on-disk format ("NQPK", version 1, layers
 * of name / n / m / r / U words / V words / binary16 s1 / binary16 s2, little
 * endian).  Errors: NQB_E_PARSE (bad magic, version, zero dimension, truncated
 * or trailing bytes: the ParseError cases of deserialize_packed_model),
 * NQB_E_IO (file not readable / writable: IoError).  No device needed. */
typedef struct nqb_nqpk nqb_nqpk;
/* read_packed_model (io.cpp:191-193) */
int nqb_nqpk_open(const char* path, nqb_nqpk** out);
/* deserialize_packed_model (io.cpp:160-185) */
int nqb_nqpk_parse(const uint8_t* bytes, uint64_t len, nqb_nqpk** out);
uint32_t nqb_nqpk_count(const nqb_nqpk* file);
/* name is NUL-terminated, truncated to name_cap - 1 bytes; name_len gets the full length */
int nqb_nqpk_layer_info(const nqb_nqpk* file, uint32_t index, char* name, uint32_t name_cap,
                        uint32_t* name_len, uint32_t* n, uint32_t* m, uint32_t* r);
/* Views of the layer's reference-layout words and binary16 scales (valid until free). */
int nqb_nqpk_layer_data(const nqb_nqpk* file, uint32_t index, const uint32_t** u_words,
                        const uint32_t** v_words, const uint16_t** s1_half,
                        const uint16_t** s2_half);
/* Straight to the device layout with the file's binary16 scales (nqb_layer_upload_f16). */
int nqb_nqpk_layer_upload(nqb_context* ctx, const nqb_nqpk* file, uint32_t index,
                          nqb_layer** out);
void nqb_nqpk_free(nqb_nqpk* file);
/* serialize_packed_model (io.cpp:139-158) from host arrays; buf == NULL queries *len. */
int nqb_nqpk_serialize(uint32_t count, const char* const* names, const uint32_t* n,
                       const uint32_t* m, const uint32_t* r, const uint32_t* const* u_words,
                       const uint32_t* const* v_words, const uint16_t* const* s1_half,
                       const uint16_t* const* s2_half, uint8_t* buf, uint64_t cap,
                       uint64_t* len);
/* write_packed_model (io.cpp:187-189) from device layers (bit-exact download). */
int nqb_nqpk_write_layers(nqb_context* ctx, const char* path, uint32_t count,
                          const char* const* names, const nqb_layer* const* layers);

#ifdef __cplusplus
}
#endif

#endif /* NQB_H */
