// svdk_internal.h — engine-internal context, status plumbing and device pool.
//
// Everything here is private to libsvdk.so; the public surface is
// include/svdk.h (C-ABI). Status codes map one-to-one onto the reference
// exception taxonomy (reference errors.hpp:11-55), see include/svdk.h.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "svdk.h"

namespace svdk {

// ---------------------------------------------------------------------------
// Status plumbing: C++ exceptions inside the engine, int codes at the C-ABI.
// ---------------------------------------------------------------------------
struct Failure {
    int code;
    std::string msg;
    double residual = 0.0;
    bool agreed = false;  // raised identically on every rank (in-band status exchange)
};

[[noreturn]] void fail(int code, const std::string& msg, double residual = 0.0);
// the same, for a status every rank of a sharded call has agreed on
[[noreturn]] void fail_agreed(int code, const std::string& msg, double residual = 0.0);

#define SVDK_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            ::svdk::fail(SVDK_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define SVDK_CHECK_LAUNCH() SVDK_CUDA(cudaGetLastError())

// Development timing probes inside kernels (clock64 stamps read back by the
// svdk_debug_* hooks); compiled out unless built with -DSVDK_PROBES.
#ifdef SVDK_PROBES
#define SVDK_CLOCK() clock64()
#define SVDK_PROBE_STORE(arr, i, v) ((arr)[i] = (v))
#else
#define SVDK_CLOCK() 0LL
#define SVDK_PROBE_STORE(arr, i, v) ((void)(v))
#endif

// ---------------------------------------------------------------------------
// Device memory pool: stream-ordered reuse on the context's single stream.
// ---------------------------------------------------------------------------
class Pool {
public:
    ~Pool();
    void* get(size_t bytes);
    void put(void* p);
    void trim();
    size_t reserved() const { return reserved_; }

private:
    struct Block {
        void* p;
        size_t bytes;
        bool busy;
    };
    std::vector<Block> blocks_;
    size_t reserved_ = 0;
};

struct Ctx;
struct HostGroup;    // in-process collective group (comm.cu)
struct JacobiCache;  // instantiated eig_sym sweep plans (jacobi.cu)
struct UploadStaging;  // pinned staging slots + packing threads (host_upload.cu)

// RAII device buffer of doubles from the context pool.
class DBuf {
public:
    DBuf() = default;
    DBuf(Ctx* c, size_t count);
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept { *this = std::move(o); }
    DBuf& operator=(DBuf&& o) noexcept;
    ~DBuf();
    double* p() const { return p_; }
    size_t count() const { return n_; }
    void reset();

private:
    Ctx* c_ = nullptr;
    double* p_ = nullptr;
    size_t n_ = 0;
};

// Column-major device matrix view (ld >= rows).
struct DMat {
    double* p = nullptr;
    int64_t rows = 0, cols = 0, ld = 0;
    double* col(int64_t j) const { return p + j * ld; }
};

// Per-phase device timing (CUDA events on the context stream), enabled by
// svdk_ctx_set_timing: algorithmic flops / bytes are attached to each record
// so bench.py can report achieved TFLOP/s or GB/s per kernel.
struct PhaseRecord {
    const char* name;
    cudaEvent_t e0, e1;
    double flops, bytes;
};

struct Ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t aux_stream = nullptr;  // side stream for off-critical-path work
    cudaStream_t copy_stream = nullptr;  // host-buffer uploads streamed under compute
    cudaEvent_t copy_ev = nullptr;
    cudaEvent_t aux_ev[2] = {nullptr, nullptr};
    cudaStream_t aux_stream2 = nullptr;  // Jacobi solve-ahead: the A updates' own stream
    cudaEvent_t aux_ev2[3] = {nullptr, nullptr, nullptr};
    Pool pool;
    // scratch: small pinned host buffer for scalars / flags
    void* host_scratch = nullptr;
    int* d_flags = nullptr;  // [0] non-finite flag, [1] jacobi status, ...
    double* d_scalars = nullptr;
    // multi-GPU (row-sharded) state
    void* nccl_comm = nullptr;       // NCCL backend (one process per GPU)
    HostGroup* host_group = nullptr;  // host-staged backend (ranks = host threads)
    int rank = 0, world = 1;
    // pinned host staging for the reference Gaussian sampler (Omega, v0),
    // filled by an asynchronous host job that overlaps device work
    struct HostJob* omega_job = nullptr;
    double* pinned = nullptr;
    size_t pinned_cap = 0;
    cudaEvent_t pinned_ev = nullptr;  // last H2D out of `pinned` completed
    // timing
    bool timing = false;
    std::vector<PhaseRecord> records;
    std::vector<cudaEvent_t> event_pool;
    size_t events_used = 0;
    // counters for bench/introspection
    int64_t launches = 0;
    JacobiCache* jacobi_cache = nullptr;
    UploadStaging* upload = nullptr;
    int jacobi_sweeps = 0;
    double last_off_norm = 0.0;
};

// RAII phase timer: records e0 now and e1 at scope exit (no-op unless timing).
class PhaseTimer {
public:
    PhaseTimer(Ctx* c, const char* name, double flops = 0.0, double bytes = 0.0);
    ~PhaseTimer();
    PhaseTimer(const PhaseTimer&) = delete;
    PhaseTimer& operator=(const PhaseTimer&) = delete;

private:
    Ctx* c_;
    long idx_ = -1;
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Raise a kernel's MaxDynamicSharedMemorySize to at least `bytes` on the
// current device (set once per (kernel, device, larger size)): function
// attributes are per device, one process may drive several GPUs, and contexts
// may be used from several host threads.
inline void ensure_smem_attr(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set_to;
    int dev = 0;
    SVDK_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set_to[{func, dev}];
    if (bytes > cur) {
        SVDK_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
        cur = bytes;
    }
}

// ---------------------------------------------------------------------------
// Engine entry points shared across translation units (device pointers,
// everything ordered on ctx->stream).
// ---------------------------------------------------------------------------

// C = op(A) * B  with op(A) = A (NN: A m x k) or A^T (TN: A k x m).
// B is k x n (K-major). Optional per-column scale of the output (epilogue).
// If nonfinite_check, raises SVDK_E_NUMERICAL on a non-finite output entry
// (reference kernels.cpp:39-43).
// Epilogue: C = alpha * (op(A) B) (+ C_old when beta_one). b_upper: B is
// upper triangular (K = N), zero k-tiles below the diagonal are skipped.
void gemm(Ctx* c, bool transa, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
          const double* B, int64_t ldb, double* C, int64_t ldc, const double* col_scale = nullptr,
          bool nonfinite_check = false, double alpha = 1.0, bool beta_one = false,
          bool b_upper = false);
// G = alpha A^T A (+ G_old) (n x n, exactly symmetric), A m x n.
void syrk(Ctx* c, int64_t m, int64_t n, const double* A, int64_t lda, double* G, int64_t ldg,
          double alpha = 1.0, bool beta_one = false);

// Small helpers (linalg_small.cu)
void fill(Ctx* c, double* p, int64_t count, double v);
void set_identity(Ctx* c, double* X, int64_t ld, int64_t n);
// W[i, j] *= s[i]
void scale_rows(Ctx* c, double* W, int64_t ldw, int64_t rows, int64_t cols, const double* s);
void copy_mat(Ctx* c, const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows,
              int64_t cols);
void transpose(Ctx* c, const double* src, int64_t lds, int64_t rows, int64_t cols, double* dst,
               int64_t ldd);
// Sum of squares of an m x n block, deterministic fixed-order reduction.
double frob_sq(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n);
void frob_sq_dev(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* d_out);
// Column means (RowsAreExamples) + subtract in place into dst; returns mean on device.
void center_rows_are_examples(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                              double* dst, int64_t ldd, double* d_mean);
// Column sums / denom (denom = 1 gives plain sums), fixed-order reduction.
void column_sums(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double denom,
                 double* d_out);
void subtract_column_means(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                           const double* d_mean, double* dst, int64_t ldd);
// the same, fused with sum_ij dst_ij^2 into a device scalar
void subtract_column_means_sumsq(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                                 const double* d_mean, double* dst, int64_t ldd, double* d_sumsq);
void center_cols_are_examples(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                              double* dst, int64_t ldd, double* d_mean);

// Symmetric eigensolver (jacobi.cu): S n x n (device), returns eigenvalues
// descending in w and eigenvectors in V (ldv). Contract of reference
// kernels.cpp:241-346 (symmetry check, threshold, sweep cap, stable sort).
void eig_sym(Ctx* c, const double* S, int64_t lds, int64_t n, int max_sweeps, double* w,
             double* V, int64_t ldv);
// release the cached sweep plans (before the context's pool is trimmed)
void jacobi_cache_free(Ctx* c);

// Host -> device copies from a caller's buffer on ctx->copy_stream: direct DMA
// for page-locked memory, packed through pinned staging slots by host threads
// for pageable memory (host_upload.cu). copy2d may block the calling thread
// (pageable: while it packs), so callers interleave it with their compute
// enqueues.
class HostUploader {
public:
    HostUploader(Ctx* c, const void* base);
    void copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height);
    bool pageable() const { return pageable_; }

private:
    Ctx* c_;
    bool pageable_;
};
void release_upload_staging(Ctx* c);

// Host <-> device
void h2d(Ctx* c, double* dst, const double* src, int64_t count);
void d2h(Ctx* c, double* dst, const double* src, int64_t count);
void sync(Ctx* c);

}  // namespace svdk
