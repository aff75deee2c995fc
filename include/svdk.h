/*
 * svdk.h — C-ABI of the B200-native FP64 PCA/SVD engine (libsvdk.so).
 *
 * This is the drop-in boundary for the reference library svdkit
 * (/root/reference/proj). Each entry point replaces one reference function,
 * cited as file:line below. Conventions:
 *
 *  - Matrices are column-major doubles, entry (i, j) at p[i + j*ld]
 *    (reference dense_matrix.hpp:41-46). Host-pointer entry points take
 *    ld = rows, like DenseMatrix. `svdk_dev_*` entry points take device
 *    pointers with an explicit leading dimension.
 *  - Outputs are caller-allocated with sizes derivable from the inputs
 *    (upper bounds documented per call); the numerical rank is returned.
 *  - Every call returns an int status. Codes map onto the reference
 *    exception taxonomy (errors.hpp:11-55):
 *      SVDK_E_DIM       -> DimensionError
 *      SVDK_E_PARAM     -> ParamError
 *      SVDK_E_NUMERICAL -> NumericalError (residual via svdk_last_residual())
 *      SVDK_E_FORMAT    -> FormatError,  SVDK_E_IO -> IoError
 *    plus engine-only failures (CUDA, NCCL, allocation, bad state). The
 *    message is in svdk_last_error() (thread-local).
 *  - A context owns one GPU, one CUDA stream and a device memory pool. It
 *    is not thread-safe; use one context per host thread.
 *  - There is no CPU fallback: without a usable sm_100 GPU every compute
 *    call fails with SVDK_E_CUDA.
 */
#ifndef SVDK_H
#define SVDK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SVDK_OK = 0,
    SVDK_E_DIM = 1,
    SVDK_E_PARAM = 2,
    SVDK_E_NUMERICAL = 3,
    SVDK_E_CUDA = 4,
    SVDK_E_NCCL = 5,
    SVDK_E_NOMEM = 6,
    SVDK_E_STATE = 7,
    SVDK_E_FORMAT = 8, /* -> FormatError (byte offset via the call's out-parameter) */
    SVDK_E_IO = 9      /* -> IoError */
};

/* svd_methods.hpp:13 SvdMethod (+ Lanczos, new in this engine) */
enum { SVDK_TRUNCATED = 0, SVDK_RANDOMIZED = 1, SVDK_KRYLOV = 2, SVDK_LANCZOS = 3 };
/* pca.hpp:16 Orientation */
enum { SVDK_COLUMNS_ARE_EXAMPLES = 0, SVDK_ROWS_ARE_EXAMPLES = 1 };

typedef struct svdk_ctx svdk_ctx;

/* ---- context / diagnostics (no reference counterpart: engine state) ---- */
int svdk_ctx_create(int device, svdk_ctx** out);
int svdk_ctx_destroy(svdk_ctx* ctx);
/* Order all work on an external cudaStream_t (e.g. torch's current stream). */
int svdk_ctx_set_stream(svdk_ctx* ctx, void* cuda_stream);
int svdk_ctx_sync(svdk_ctx* ctx);
const char* svdk_last_error(void);
double svdk_last_residual(void);
/* Kernel launches issued by this context so far (bench evidence). */
int64_t svdk_ctx_launches(svdk_ctx* ctx);
/* Sweeps used by the most recent eig_sym on this context. */
int svdk_ctx_last_sweeps(svdk_ctx* ctx);
const char* svdk_version(void);
/* Per-kernel device timing with CUDA events on the context stream (bench
 * evidence): records carry the algorithmic flops / bytes of each launch.
 * Query sums the records whose phase name matches (NULL = all); names are
 * e.g. "dmma_gemm", "splitk_reduce", "eig_sym", "qr_thin", "gemv_pair". */
int svdk_ctx_set_timing(svdk_ctx* ctx, int enable);
int svdk_ctx_timing_reset(svdk_ctx* ctx);
int svdk_ctx_timing_query(svdk_ctx* ctx, const char* name, int64_t* count, double* ms,
                          double* flops, double* bytes);
int svdk_ctx_timing_names(svdk_ctx* ctx, char* buf, int64_t len);

/* ---- row-sharded multi-GPU (one process per GPU, NCCL over NVLink) ---- */
/* 128-byte NCCL unique id, produced on rank 0 and shared out of band. */
int svdk_nccl_unique_id(char out[128]);
int svdk_ctx_attach_nccl(svdk_ctx* ctx, const char id[128], int rank, int world);
/* In-process host-staged collectives: `world` contexts (any GPUs, including
 * several on one GPU), each driven by its own host thread, attach to one group
 * with ranks 0..world-1; every row reduction is staged through host memory and
 * summed in rank order (no kernel waits on another rank). For running and
 * testing the sharded paths without a multi-GPU node; NCCL is the production
 * backend. A failing rank aborts the group: its peers' calls return
 * SVDK_E_STATE instead of waiting. destroy drops the creator's reference (the
 * group lives until the last attached context detaches). */
typedef struct svdk_host_group svdk_host_group;
int svdk_host_group_create(int world, svdk_host_group** out);
int svdk_host_group_destroy(svdk_host_group* group);
int svdk_ctx_attach_host_group(svdk_ctx* ctx, svdk_host_group* group, int rank);
/* Detach (NCCL: destroy the communicator) and return to single-GPU mode. */
int svdk_ctx_detach_comm(svdk_ctx* ctx);
/* rank / world of the attached communicator (0 / 1 when none). */
int svdk_ctx_comm_info(svdk_ctx* ctx, int* rank, int* world);

/* ---- L1 kernels (reference kernels.hpp / kernels.cpp) ---- */
/* kernels.cpp:14-45  C (m x l) = A (m x n) * B (n x l); non-finite C -> NUMERICAL */
int svdk_matmul(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, const double* b, int64_t l,
                double* c);
/* kernels.cpp:47-67  C (n x l) = A^T (A m x n) * B (m x l) */
int svdk_matmul_transposed_left(svdk_ctx* ctx, const double* a, int64_t m, int64_t n,
                                const double* b, int64_t l, double* c);
/* kernels.cpp:69-78  T (n x m) = A^T */
int svdk_transpose(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, double* t);
/* kernels.cpp:80-97  G (n x n) = A^T A, exactly symmetric */
int svdk_gram(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, double* g);
/* kernels.cpp:99-109 */
int svdk_frobenius_norm_sq(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, double* out);
/* kernels.cpp:111-224  thin QR, m >= p: Q (m x p), R (p x p, may be NULL), rank */
int svdk_qr_thin(svdk_ctx* ctx, const double* h, int64_t m, int64_t p, double* q, double* r,
                 int64_t* rank);
/* kernels.cpp:241-346  w (n, descending), V (n x n); max_sweeps <= 0 -> 30 */
int svdk_eig_sym(svdk_ctx* ctx, const double* s, int64_t n, int max_sweeps, double* w, double* v);
/* kernels.cpp:348-379  bit-identical mt19937_64 + Box-Muller sampler (host) */
int svdk_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out);

/* ---- L2 methods (reference svd_methods.hpp / svd_methods.cpp) ---- */
/* Buffers: u m x n, sigma n, v n x n (upper bounds); first *rank columns valid. */
/* svd_methods.cpp:121-158 */
int svdk_truncated_svd(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, double* u,
                       double* sigma, double* v, int64_t* rank);
/* svd_methods.cpp:160-170 ; buffers u m x l, sigma l, v n x l */
int svdk_randomized_pca(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t l,
                        int64_t q, uint64_t seed, double* u, double* sigma, double* v,
                        int64_t* rank);
/* svd_methods.cpp:172-196 ; w = min((i+1)l, n): buffers u m x w, sigma w, v n x w */
int svdk_krylov_svd(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t l, int64_t i,
                    uint64_t seed, double* u, double* sigma, double* v, int64_t* rank);
/* NEW (no reference): Lanczos on A^T A, full reorthogonalisation; steps <= n
 * (0 -> n); buffers u m x steps, sigma steps, v n x steps. */
int svdk_lanczos_svd(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t steps,
                     uint64_t seed, double* u, double* sigma, double* v, int64_t* rank);
/* svd_methods.cpp:227-246 compute_svd_any: any shape; method SVDK_* ;
 * l, q = sketch width / power iterations (ignored by truncated). Buffers
 * sized for min(m, n) columns. */
int svdk_compute_svd(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int method, int64_t l,
                     int64_t q, uint64_t seed, double* u, double* sigma, double* v,
                     int64_t* rank);

/* ---- L3 PCA (reference pca.hpp / pca.cpp) ---- */
/* pca.cpp:13-55 ; mean has n (RowsAreExamples) or m entries */
int svdk_center(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int orientation,
                double* centered, double* mean);
/* pca.cpp:61-89 ; *k = 0 encodes std::nullopt */
int svdk_select_components(svdk_ctx* ctx, const double* eigenvalues, int64_t count, double total,
                           double threshold, int64_t* k);
/* pca.cpp:91-116 ; basis n x r (RowsAreExamples) or m x r, eigenvalues r,
 * total, mean (n or m entries, zeros when center == 0) */
int svdk_fit_pca(svdk_ctx* ctx, const double* data, int64_t m, int64_t n, int orientation,
                 int method, int64_t l, int64_t q, uint64_t seed, int center, double* basis,
                 double* eigenvalues, double* total, double* mean, int64_t* rank);

/* pca.cpp:133-168  delta = ||A - U diag(sigma) V^T||_F / ||A||_F ; u m x r, v n x r */
int svdk_residual_delta(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, const double* u,
                        const double* sigma, const double* v, int64_t r, double* delta);

/* ---- cost model (cost_model.cpp:30-113; host-only, no context) ----
 * Modeled flops and space (8-byte entries, input included; bytes = 8 * entries)
 * of one factorization, the published closed forms:
 *   SVDK_COST_TRUNCATED            truncated_cost(m, n)
 *   SVDK_COST_RANDOMIZED           randomized_cost(m, n, l, i)        (i >= 0)
 *   SVDK_COST_RANDOMIZED_PRACTICAL randomized_cost_practical(m, n)    (l = n/2, i = 1)
 *   SVDK_COST_KRYLOV               krylov_cost(m, n, l, i)            (i >= 1)
 *   SVDK_COST_KRYLOV_PRACTICAL     krylov_cost_practical(m, n)
 *   SVDK_COST_KRYLOV_PER_STEP      krylov_cost_per_step(m, n, l, i)
 * l and i are ignored by the models without them. Domain violations
 * (m >= n >= l >= 1) return SVDK_E_PARAM. */
enum {
    SVDK_COST_TRUNCATED = 0,
    SVDK_COST_RANDOMIZED = 1,
    SVDK_COST_RANDOMIZED_PRACTICAL = 2,
    SVDK_COST_KRYLOV = 3,
    SVDK_COST_KRYLOV_PRACTICAL = 4,
    SVDK_COST_KRYLOV_PER_STEP = 5
};
int svdk_cost_model(int model, uint64_t m, uint64_t n, uint64_t l, uint64_t i, double* flops,
                    double* space_entries, double* space_bytes);

/* ---- IDX image ingestion (idx_io.cpp:24-107) ----
 * svdk_idx_parse: validate a rank-3 unsigned-byte IDX buffer (big-endian magic
 * 0x00000803, three big-endian u32 dims, then count*height*width bytes, nothing
 * after). On success dims = {count, height, width} and the pixels start at
 * bytes + 16. On SVDK_E_FORMAT *error_offset is FormatError::offset(). Host-only.
 * svdk_idx_to_matrix: images_to_matrix — count x (height*width) column-major,
 * entry (i, p) = pixels[i * P + p] / 255 (rows are examples), expanded on the
 * GPU from the 1-byte pixels (8x less host->device traffic than the doubles). */
int svdk_idx_parse(const uint8_t* bytes, uint64_t len, uint64_t dims[3], uint64_t* error_offset);
int svdk_idx_to_matrix(svdk_ctx* ctx, const uint8_t* pixels, int64_t count,
                       int64_t pixels_per_image, double* out);

/* ---- device-pointer entry points (inputs already resident in HBM) ---- */
int svdk_dev_gemm(svdk_ctx* ctx, int transa, int64_t m, int64_t n, int64_t k, const double* a,
                  int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);
int svdk_dev_gram(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda, double* g,
                  int64_t ldg);
/* w = A^T (A q), A m x n column-major (device pointers): the Lanczos matvec
 * pair on its own (engine-internal; no reference counterpart — the reference
 * has no Lanczos). Exposed for kernel-level parity tests. */
int svdk_dev_gemv_pair(svdk_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                       const double* q, double* w);
int svdk_dev_eig_sym(svdk_ctx* ctx, const double* s, int64_t n, int64_t lds, int max_sweeps,
                     double* w, double* v, int64_t ldv);
int svdk_dev_qr_thin(svdk_ctx* ctx, const double* h, int64_t m, int64_t p, int64_t ldh, double* q,
                     int64_t ldq, double* r, int64_t* rank);
/* Full PCA pipeline on a device-resident (local row shard of) A, RowsAreExamples:
 * center -> total variance -> SVD (method) -> select_components(threshold).
 * Outputs on device: u (m_local x r, ldu), sigma (r), v (n x r, ldv), mean (n);
 * on host: *rank, *k (0 = nullopt), *total. center: 0 = none, 1 = centre a
 * copy, 2 = centre A in place (A is overwritten; saves an m x n buffer).
 * With an attached NCCL communicator the reductions over rows span all ranks. */
int svdk_dev_pca(svdk_ctx* ctx, const double* a, int64_t m_local, int64_t n, int64_t lda,
                 int method, int64_t l, int64_t q, uint64_t seed, int center, double threshold,
                 double* u, int64_t ldu, double* sigma, double* v, int64_t ldv, double* mean,
                 int64_t* rank, int64_t* k, double* total);
/* images_to_matrix on device buffers: out (count x P, ldo >= count) */
int svdk_dev_idx_to_matrix(svdk_ctx* ctx, const uint8_t* pixels, int64_t count,
                           int64_t pixels_per_image, double* out, int64_t ldo);

/* ---- seeded synthetic inputs (bench / tests / fixtures; no reference
 * counterpart — SURVEY §8d's generator, not on the PCA path) ----
 * A = X M + sigma N: X quantised Gaussians (stream 1), M = R_X^-1 diag(s) V0^T
 * on a fixed-point grid (V0 from stream 2), N Gaussians (stream 3). Element e
 * of a stream = global_row + column * m_total; Philox4x32-10 + Box-Muller with
 * explicitly rounded polynomial log/sin/cos, so host and device produce the
 * same bits and X^T X, X M are exact in any summation order (synth.h).
 * svdk_synth_fill / svdk_dev_synth_fill: rows [row0, row0+rows) x cols of a
 * stream into out (ld); quantise != 0 applies the X grid.
 * svdk_synth_add_noise / _dev_: a += sigma * N on the same block.
 * svdk_synth_mixing: M (n x n, ldm) from the exact gram gx = X^T X (ldg), the
 * spectrum s (n) and the seed; *grid = M's fixed-point quantum. Host-only. */
int svdk_synth_fill(uint64_t seed, int stream, int quantise, int64_t m_total, int64_t row0, int64_t rows,
                    int64_t cols, double* out, int64_t ld);
int svdk_synth_add_noise(uint64_t seed, int64_t m_total, int64_t row0, int64_t rows, int64_t cols,
                         double sigma, double* a, int64_t lda);
int svdk_synth_mixing(int64_t n, const double* gx, int64_t ldg, const double* s, uint64_t seed, double* mix,
                      int64_t ldm, double* grid);
int svdk_dev_synth_fill(svdk_ctx* ctx, uint64_t seed, int stream, int quantise, int64_t m_total,
                        int64_t row0, int64_t rows, int64_t cols, double* out, int64_t ld);
int svdk_dev_synth_add_noise(svdk_ctx* ctx, uint64_t seed, int64_t m_total, int64_t row0, int64_t rows,
                             int64_t cols, double sigma, double* a, int64_t lda);

#ifdef __cplusplus
}
#endif
#endif
