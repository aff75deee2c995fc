// abi.cu — the extern "C" boundary (include/svdk.h).
//
// Every entry point validates like the reference function it replaces
// (file:line in svdk.h), converts engine failures into status codes, and
// keeps the message / residual in thread-local storage.
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "svdk_methods.h"

namespace svdk {
void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out);
int64_t randomized_pca(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                       int64_t q, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                       int64_t ldv, const RowComm* comm);
int64_t krylov_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                   int64_t iters, uint64_t seed, double* U, int64_t ldu, double* sigma, double* V,
                   int64_t ldv, const RowComm* comm);
int64_t lanczos_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t steps,
                    uint64_t seed, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                    const RowComm* comm);
int64_t qr_thin(Ctx* c, const double* H, int64_t ldh, int64_t m, int64_t p, double* Q, int64_t ldq,
                double* R, const RowComm* comm, double* Rinv_last = nullptr);
int64_t select_components(Ctx* c, const double* d_w, int64_t count, double total, double t);
struct CostOut {
    double flops = 0.0, entries = 0.0;
};
CostOut cost_model(int model, uint64_t m, uint64_t n, uint64_t l, uint64_t i);
void idx_parse(const uint8_t* bytes, uint64_t len, uint64_t dims[3], uint64_t* err_offset);
void idx_to_matrix_dev(Ctx* c, const uint8_t* px, int64_t count, int64_t P, double* out,
                       int64_t ldo);
void synth_fill_dev(Ctx* c, uint64_t seed, int stream, int quantise, int64_t m_total, int64_t row0,
                    int64_t rows, int64_t cols, double* out, int64_t ld);
void synth_add_noise_dev(Ctx* c, uint64_t seed, int64_t m_total, int64_t row0, int64_t rows, int64_t cols,
                         double sigma, double* a, int64_t lda);
}  // namespace svdk

using namespace svdk;

struct svdk_ctx : Ctx {};
struct svdk_host_group {};  // opaque handle of a svdk::HostGroup

namespace {

thread_local std::string g_err;
thread_local double g_residual = 0.0;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return SVDK_OK;
    } catch (const Failure& e) {
        g_err = e.msg;
        g_residual = e.residual;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return SVDK_E_NOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SVDK_E_STATE;
    }
}

void need_ctx(svdk_ctx* c) {
    if (!c) fail(SVDK_E_STATE, "null svdk_ctx");
}

}  // namespace

// Host-buffer and method-dispatch helpers (shared with stream_fit.cu).
namespace svdk {

// Host column-major (ld = rows) -> device with an even leading dimension
// (TMA needs 16-byte strides).
DBuf upload(Ctx* c, const double* h, int64_t rows, int64_t cols, int64_t& ld) {
    ld = std::max<int64_t>(2, round_up(rows, 2));
    DBuf d(c, static_cast<size_t>(ld) * std::max<int64_t>(cols, 1));
    if (rows > 0 && cols > 0) {
        if (ld == rows)
            SVDK_CUDA(cudaMemcpyAsync(d.p(), h, sizeof(double) * rows * cols,
                                      cudaMemcpyHostToDevice, c->stream));
        else
            SVDK_CUDA(cudaMemcpy2DAsync(d.p(), ld * sizeof(double), h, rows * sizeof(double),
                                        rows * sizeof(double), cols, cudaMemcpyHostToDevice,
                                        c->stream));
    }
    return d;
}

DBuf alloc_mat(Ctx* c, int64_t rows, int64_t cols, int64_t& ld) {
    ld = std::max<int64_t>(2, round_up(rows, 2));
    return DBuf(c, static_cast<size_t>(ld) * std::max<int64_t>(cols, 1));
}

void download(Ctx* c, double* h, const double* d, int64_t ld, int64_t rows, int64_t cols) {
    if (rows > 0 && cols > 0) {
        if (ld == rows)
            SVDK_CUDA(cudaMemcpyAsync(h, d, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost,
                                      c->stream));
        else
            SVDK_CUDA(cudaMemcpy2DAsync(h, rows * sizeof(double), d, ld * sizeof(double),
                                        rows * sizeof(double), cols, cudaMemcpyDeviceToHost,
                                        c->stream));
    }
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
}

void require_tall(int64_t m, int64_t n, const char* op) {
    if (m < n)
        fail(SVDK_E_DIM, std::string(op) + ": needs rows >= cols, got " + std::to_string(m) + "x" +
                             std::to_string(n) +
                             "; pass the transpose and swap U/V, or use compute_svd_any");
    if (n == 0) fail(SVDK_E_DIM, std::string(op) + ": empty input");
}

// svd_methods.cpp:77-93
void validate_sketch(int64_t m, int64_t n, int64_t l, int64_t q, bool krylov) {
    if (l < 1 || l > n)
        fail(SVDK_E_PARAM, "sketch width l = " + std::to_string(l) + " outside [1, n] for n = " +
                               std::to_string(n));
    if (krylov) {
        if (q < 1) fail(SVDK_E_PARAM, "krylov_svd: needs power_iterations >= 1");
        const int64_t width = (q + 1) * l;
        if (width > m)
            fail(SVDK_E_PARAM, "krylov_svd: block width (i+1)*l = " + std::to_string(width) +
                                   " exceeds rows = " + std::to_string(m));
    }
}

// Run one SVD method on a device-resident tall A; returns rank.
int64_t run_method(Ctx* c, int method, const double* dA, int64_t lda, int64_t m, int64_t n,
                   int64_t l, int64_t q, uint64_t seed, double* dU, int64_t ldu, double* dS,
                   double* dV, int64_t ldv, const RowComm* comm) {
    reset_nonfinite(c);
    int64_t r = 0;
    switch (method) {
        case SVDK_TRUNCATED:
            r = truncated_svd(c, dA, lda, m, n, dU, ldu, dS, dV, ldv, comm);
            break;
        case SVDK_RANDOMIZED:
            r = randomized_pca(c, dA, lda, m, n, l, q, seed, dU, ldu, dS, dV, ldv, comm);
            break;
        case SVDK_KRYLOV:
            r = krylov_svd(c, dA, lda, m, n, l, q, seed, dU, ldu, dS, dV, ldv, comm);
            break;
        case SVDK_LANCZOS:
            r = lanczos_svd(c, dA, lda, m, n, l, seed, dU, ldu, dS, dV, ldv, comm);
            break;
        default:
            fail(SVDK_E_PARAM, "compute_svd: unknown method");
    }
    raise_if_nonfinite(c);  // kernels.cpp:39-43, once per call
    return r;
}

// Output column bound of each method for a tall m x n input.
int64_t method_width(int method, int64_t m, int64_t n, int64_t l, int64_t q) {
    switch (method) {
        case SVDK_RANDOMIZED:
            return l;
        case SVDK_KRYLOV:
            return std::min<int64_t>((q + 1) * l, n);
        case SVDK_LANCZOS:
            return (l <= 0 || l > n) ? n : l;
        default:
            return n;
    }
}

void validate_method(int method, int64_t m, int64_t n, int64_t l, int64_t q, const char* name) {
    require_tall(m, n, name);
    if (method == SVDK_RANDOMIZED) validate_sketch(m, n, l, q, false);
    if (method == SVDK_KRYLOV) validate_sketch(m, n, l, q, true);
    if (method == SVDK_LANCZOS && l < 0) fail(SVDK_E_PARAM, "lanczos_svd: steps must be >= 0");
    if (method < 0 || method > SVDK_LANCZOS) fail(SVDK_E_PARAM, "compute_svd: unknown method");
}

}  // namespace svdk

namespace {

// Host-pointer method call: H2D, run, D2H (u m x rank, sigma, v n x rank).
void host_method(svdk_ctx* c, int method, const double* a, int64_t m, int64_t n, int64_t l,
                 int64_t q, uint64_t seed, double* u, double* sigma, double* v, int64_t* rank,
                 const char* name) {
    need_ctx(c);
    validate_method(method, m, n, l, q, name);
    const int64_t w = method_width(method, m, n, l, q);
    int64_t lda, ldu, ldv;
    DBuf dA = upload(c, a, m, n, lda);
    DBuf dU = alloc_mat(c, m, w, ldu), dV = alloc_mat(c, n, w, ldv), dS(c, std::max<int64_t>(w, n));
    const int64_t r = run_method(c, method, dA.p(), lda, m, n, l, q, seed, dU.p(), ldu, dS.p(),
                                 dV.p(), ldv, nullptr);
    download(c, u, dU.p(), ldu, m, r);
    download(c, v, dV.p(), ldv, n, r);
    download(c, sigma, dS.p(), r, r, 1);
    *rank = r;
}

}  // namespace

extern "C" {

const char* svdk_version(void) { return "svdk-b200 0.1 (sm_100a, FP64 DMMA)"; }
const char* svdk_last_error(void) { return g_err.c_str(); }
double svdk_last_residual(void) { return g_residual; }

int svdk_ctx_create(int device, svdk_ctx** out) {
    return guarded([&] {
        if (!out) fail(SVDK_E_PARAM, "svdk_ctx_create: null out");
        *out = nullptr;
        int count = 0;
        SVDK_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count)
            fail(SVDK_E_CUDA, "svdk_ctx_create: no CUDA device " + std::to_string(device));
        SVDK_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop;
        SVDK_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(SVDK_E_CUDA, std::string("svdk: needs an sm_100 (B200) device, got ") + prop.name);
        auto* c = new svdk_ctx();
        c->device = device;
        c->num_sms = prop.multiProcessorCount;
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
        SVDK_CUDA(cudaMalloc(&c->d_flags, 64 * sizeof(int)));
        SVDK_CUDA(cudaMemset(c->d_flags, 0, 64 * sizeof(int)));
        *out = c;
    });
}

int svdk_ctx_destroy(svdk_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        destroy_comm(ctx);
        release_host_staging(ctx);
        jacobi_cache_free(ctx);
        release_upload_staging(ctx);
        ctx->pool.trim();
        if (ctx->d_flags) cudaFree(ctx->d_flags);
        for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
        if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
        if (ctx->copy_ev) cudaEventDestroy(ctx->copy_ev);
        for (cudaEvent_t e : ctx->aux_ev)
            if (e) cudaEventDestroy(e);
        if (ctx->aux_stream2) cudaStreamDestroy(ctx->aux_stream2);
        for (cudaEvent_t e : ctx->aux_ev2)
            if (e) cudaEventDestroy(e);
        delete ctx;
    });
}

int svdk_ctx_set_stream(svdk_ctx* ctx, void* stream) {
    return guarded([&] {
        need_ctx(ctx);
        SVDK_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        ctx->stream = static_cast<cudaStream_t>(stream);
        ctx->own_stream = false;
    });
}

int svdk_ctx_sync(svdk_ctx* ctx) {
    return guarded([&] {
        need_ctx(ctx);
        sync(ctx);
    });
}

int64_t svdk_ctx_launches(svdk_ctx* ctx) { return ctx ? ctx->launches : 0; }
int svdk_ctx_last_sweeps(svdk_ctx* ctx) { return ctx ? ctx->jacobi_sweeps : 0; }

int svdk_ctx_set_timing(svdk_ctx* ctx, int enable) {
    return guarded([&] {
        need_ctx(ctx);
        ctx->timing = enable != 0;
    });
}

int svdk_ctx_timing_reset(svdk_ctx* ctx) {
    return guarded([&] {
        need_ctx(ctx);
        sync(ctx);
        ctx->records.clear();
        ctx->events_used = 0;
    });
}

int svdk_ctx_timing_query(svdk_ctx* ctx, const char* name, int64_t* count, double* ms,
                          double* flops, double* bytes) {
    return guarded([&] {
        need_ctx(ctx);
        sync(ctx);
        int64_t n = 0;
        double t = 0.0, f = 0.0, b = 0.0;
        for (const auto& r : ctx->records) {
            if (name && std::strcmp(name, r.name) != 0) continue;
            float e = 0.0f;
            SVDK_CUDA(cudaEventElapsedTime(&e, r.e0, r.e1));
            ++n;
            t += e;
            f += r.flops;
            b += r.bytes;
        }
        if (count) *count = n;
        if (ms) *ms = t;
        if (flops) *flops = f;
        if (bytes) *bytes = b;
    });
}

int svdk_ctx_timing_names(svdk_ctx* ctx, char* buf, int64_t len) {
    return guarded([&] {
        need_ctx(ctx);
        std::string s;
        for (const auto& r : ctx->records) {
            const std::string nm(r.name);
            if (("," + s + ",").find("," + nm + ",") == std::string::npos) s += (s.empty() ? "" : ",") + nm;
        }
        if (buf && len > 0) {
            std::strncpy(buf, s.c_str(), static_cast<size_t>(len - 1));
            buf[len - 1] = 0;
        }
    });
}

int svdk_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guarded([&] {
        if (rows < 1 || cols < 1) fail(SVDK_E_PARAM, "gaussian_matrix: rows and cols must be >= 1");
        gaussian_fill(rows, cols, seed, out);
    });
}

int svdk_matmul(svdk_ctx* c, const double* a, int64_t m, int64_t n, const double* b, int64_t l,
                double* out) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda, ldb, ldc;
        DBuf dA = upload(c, a, m, n, lda), dB = upload(c, b, n, l, ldb);
        DBuf dC = alloc_mat(c, m, l, ldc);
        reset_nonfinite(c);
        gemm(c, false, m, l, n, dA.p(), lda, dB.p(), ldb, dC.p(), ldc, nullptr, true);
        raise_if_nonfinite(c);
        download(c, out, dC.p(), ldc, m, l);
    });
}

int svdk_matmul_transposed_left(svdk_ctx* c, const double* a, int64_t m, int64_t n,
                                const double* b, int64_t l, double* out) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda, ldb, ldc;
        DBuf dA = upload(c, a, m, n, lda), dB = upload(c, b, m, l, ldb);
        DBuf dC = alloc_mat(c, n, l, ldc);
        gemm(c, true, n, l, m, dA.p(), lda, dB.p(), ldb, dC.p(), ldc);
        download(c, out, dC.p(), ldc, n, l);
    });
}

int svdk_transpose(svdk_ctx* c, const double* a, int64_t m, int64_t n, double* t) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda, ldt;
        DBuf dA = upload(c, a, m, n, lda);
        DBuf dT = alloc_mat(c, n, m, ldt);
        transpose(c, dA.p(), lda, m, n, dT.p(), ldt);
        download(c, t, dT.p(), ldt, n, m);
    });
}

int svdk_gram(svdk_ctx* c, const double* a, int64_t m, int64_t n, double* g) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda;
        DBuf dA = upload(c, a, m, n, lda);
        DBuf dG(c, static_cast<size_t>(std::max<int64_t>(n, 1)) * std::max<int64_t>(n, 1));
        syrk(c, m, n, dA.p(), lda, dG.p(), n);
        download(c, g, dG.p(), n, n, n);
    });
}

int svdk_frobenius_norm_sq(svdk_ctx* c, const double* a, int64_t m, int64_t n, double* out) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda;
        DBuf dA = upload(c, a, m, n, lda);
        *out = frob_sq(c, dA.p(), lda, m, n);
    });
}

int svdk_qr_thin(svdk_ctx* c, const double* h, int64_t m, int64_t p, double* q, double* r,
                 int64_t* rank) {
    return guarded([&] {
        need_ctx(c);
        if (m < p)
            fail(SVDK_E_DIM, "qr_thin: need rows >= cols, got " + std::to_string(m) + "x" +
                                 std::to_string(p));
        int64_t ldh, ldq;
        DBuf dH = upload(c, h, m, p, ldh);
        DBuf dQ = alloc_mat(c, m, p, ldq);
        DBuf dR(c, static_cast<size_t>(std::max<int64_t>(p, 1)) * std::max<int64_t>(p, 1));
        const int64_t rk = qr_thin(c, dH.p(), ldh, m, p, dQ.p(), ldq, dR.p(), nullptr);
        download(c, q, dQ.p(), ldq, m, p);
        if (r) download(c, r, dR.p(), p, p, p);
        if (rank) *rank = rk;
    });
}

int svdk_eig_sym(svdk_ctx* c, const double* s, int64_t n, int max_sweeps, double* w, double* v) {
    return guarded([&] {
        need_ctx(c);
        if (n < 0) fail(SVDK_E_DIM, "eig_sym: matrix not square");
        if (n == 0) return;
        int64_t lds;
        DBuf dS = upload(c, s, n, n, lds);
        DBuf dW(c, n), dV(c, static_cast<size_t>(n) * n);
        eig_sym(c, dS.p(), lds, n, max_sweeps, dW.p(), dV.p(), n);
        download(c, w, dW.p(), n, n, 1);
        download(c, v, dV.p(), n, n, n);
    });
}

int svdk_truncated_svd(svdk_ctx* c, const double* a, int64_t m, int64_t n, double* u,
                       double* sigma, double* v, int64_t* rank) {
    return guarded([&] {
        host_method(c, SVDK_TRUNCATED, a, m, n, 0, 0, 0, u, sigma, v, rank, "truncated_svd");
    });
}

int svdk_randomized_pca(svdk_ctx* c, const double* a, int64_t m, int64_t n, int64_t l, int64_t q,
                        uint64_t seed, double* u, double* sigma, double* v, int64_t* rank) {
    return guarded([&] {
        host_method(c, SVDK_RANDOMIZED, a, m, n, l, q, seed, u, sigma, v, rank, "randomized_pca");
    });
}

int svdk_krylov_svd(svdk_ctx* c, const double* a, int64_t m, int64_t n, int64_t l, int64_t i,
                    uint64_t seed, double* u, double* sigma, double* v, int64_t* rank) {
    return guarded([&] {
        host_method(c, SVDK_KRYLOV, a, m, n, l, i, seed, u, sigma, v, rank, "krylov_svd");
    });
}

int svdk_lanczos_svd(svdk_ctx* c, const double* a, int64_t m, int64_t n, int64_t steps,
                     uint64_t seed, double* u, double* sigma, double* v, int64_t* rank) {
    return guarded([&] {
        host_method(c, SVDK_LANCZOS, a, m, n, steps, 0, seed, u, sigma, v, rank, "lanczos_svd");
    });
}

int svdk_compute_svd(svdk_ctx* c, const double* a, int64_t m, int64_t n, int method, int64_t l,
                     int64_t q, uint64_t seed, double* u, double* sigma, double* v,
                     int64_t* rank) {
    return guarded([&] {
        need_ctx(c);
        if (m >= n) {
            host_method(c, method, a, m, n, l, q, seed, u, sigma, v, rank, "compute_svd");
            return;
        }
        // svd_methods.cpp:239-246: factor the transpose, swap U and V.
        int64_t lda, ldt;
        DBuf dA = upload(c, a, m, n, lda);
        DBuf dT = alloc_mat(c, n, m, ldt);
        transpose(c, dA.p(), lda, m, n, dT.p(), ldt);
        dA.reset();
        validate_method(method, n, m, l, q, "compute_svd");
        const int64_t w = method_width(method, n, m, l, q);
        int64_t ldu, ldv;
        DBuf dU = alloc_mat(c, n, w, ldu), dV = alloc_mat(c, m, w, ldv), dS(c, std::max(w, m));
        const int64_t r = run_method(c, method, dT.p(), ldt, n, m, l, q, seed, dU.p(), ldu, dS.p(),
                                     dV.p(), ldv, nullptr);
        download(c, u, dV.p(), ldv, m, r);  // U of A = V of A^T
        download(c, v, dU.p(), ldu, n, r);
        download(c, sigma, dS.p(), r, r, 1);
        *rank = r;
    });
}

int svdk_center(svdk_ctx* c, const double* a, int64_t m, int64_t n, int orientation,
                double* centered, double* mean) {
    return guarded([&] {
        need_ctx(c);
        int64_t lda, ldc;
        DBuf dA = upload(c, a, m, n, lda);
        DBuf dC = alloc_mat(c, m, n, ldc);
        const int64_t nm = orientation == SVDK_COLUMNS_ARE_EXAMPLES ? m : n;
        DBuf dM(c, std::max<int64_t>(nm, 1));
        if (m > 0 && n > 0) {
            if (orientation == SVDK_COLUMNS_ARE_EXAMPLES)
                center_cols_are_examples(c, dA.p(), lda, m, n, dC.p(), ldc, dM.p());
            else
                center_rows_are_examples(c, dA.p(), lda, m, n, dC.p(), ldc, dM.p());
        } else if (nm > 0) {
            fill(c, dM.p(), nm, std::nan(""));  // 0/0 like the reference
        }
        download(c, centered, dC.p(), ldc, m, n);
        download(c, mean, dM.p(), nm, nm, 1);
    });
}

int svdk_select_components(svdk_ctx* c, const double* eigenvalues, int64_t count, double total,
                           double threshold, int64_t* k) {
    return guarded([&] {
        need_ctx(c);
        DBuf dW(c, std::max<int64_t>(count, 1));
        h2d(c, dW.p(), eigenvalues, count);
        *k = select_components(c, dW.p(), count, total, threshold);
    });
}

int svdk_fit_pca(svdk_ctx* c, const double* data, int64_t m, int64_t n, int orientation,
                 int method, int64_t l, int64_t q, uint64_t seed, int center, double* basis,
                 double* eigenvalues, double* total, double* mean, int64_t* rank) {
    return guarded([&] {
        need_ctx(c);
        // pca.cpp:91-116: center -> total -> compute_svd_any -> basis, sigma^2
        const bool cols_ex = orientation == SVDK_COLUMNS_ARE_EXAMPLES;
        const int64_t nm = cols_ex ? m : n;
        {
            const int64_t tn = std::min(m, n);  // the tall problem's width
            if ((method == SVDK_RANDOMIZED || method == SVDK_KRYLOV) && l >= 1 && l <= tn)
                omega_prefetch(c, tn, l, seed);
            else if (method == SVDK_LANCZOS)
                omega_prefetch(c, tn, 1, seed);
        }
        // Truncated / randomized on a tall centred RowsAreExamples matrix: the
        // upload streams in row chunks under the Gram / sketch (stream_fit.cu).
        if (!cols_ex && center &&
            fit_pca_streamed(c, data, m, n, method, l, q, seed, basis, eigenvalues, total, mean, rank))
            return;
        // The upload buffer is ours: centre it in place (no second m x n copy,
        // which is what lets the 64 GB c4 matrix fit one GPU).
        int64_t lda;
        DBuf dC = upload(c, data, m, n, lda);
        const int64_t ldc = lda;
        DBuf dM(c, std::max<int64_t>(nm, 1));
        if (center && !cols_ex) {
            // column means, then centring fused with the total variance
            // (pca.cpp:57-59) in one pass over the upload buffer
            column_sums(c, dC.p(), ldc, m, n, static_cast<double>(m), dM.p());
            DBuf dt(c, 1);
            subtract_column_means_sumsq(c, dC.p(), ldc, m, n, dM.p(), dC.p(), ldc, dt.p());
            d2h(c, total, dt.p(), 1);
        } else {
            if (center)
                center_cols_are_examples(c, dC.p(), ldc, m, n, dC.p(), ldc, dM.p());
            else
                fill(c, dM.p(), nm, 0.0);
            *total = frob_sq(c, dC.p(), ldc, m, n);
        }
        // tall orientation for the method
        const bool wide = m < n;
        const double* dT = dC.p();
        int64_t tm = m, tn = n, ldt = ldc;
        DBuf tbuf;
        if (wide) {
            tbuf = alloc_mat(c, n, m, ldt);
            transpose(c, dC.p(), ldc, m, n, tbuf.p(), ldt);
            dT = tbuf.p();
            tm = n;
            tn = m;
        }
        validate_method(method, tm, tn, l, q, "fit_pca");
        const int64_t w = method_width(method, tm, tn, l, q);
        int64_t ldu, ldv;
        DBuf dU = alloc_mat(c, tm, w, ldu), dV = alloc_mat(c, tn, w, ldv), dS(c, std::max(w, tn));
        const int64_t r = run_method(c, method, dT, ldt, tm, tn, l, q, seed, dU.p(), ldu, dS.p(),
                                     dV.p(), ldv, nullptr);
        // basis: U for ColumnsAreExamples, V for RowsAreExamples (of the original A)
        const bool basis_is_tall_v = (cols_ex == wide);  // after the swap of compute_svd_any
        if (basis_is_tall_v)
            download(c, basis, dV.p(), ldv, tn, r);
        else
            download(c, basis, dU.p(), ldu, tm, r);
        std::vector<double> s(r);
        download(c, s.data(), dS.p(), r, r, 1);
        for (int64_t i = 0; i < r; ++i) eigenvalues[i] = s[i] * s[i];
        download(c, mean, dM.p(), nm, nm, 1);
        *rank = r;
    });
}

int svdk_residual_delta(svdk_ctx* c, const double* a, int64_t m, int64_t n, const double* u,
                        const double* sigma, const double* v, int64_t r, double* delta) {
    return guarded([&] {
        need_ctx(c);
        // pca.cpp:133-168: ||A - U diag(sigma) V^T||_F / ||A||_F
        int64_t lda, ldu, ldv;
        DBuf dA = upload(c, a, m, n, lda);
        const double norm_sq = frob_sq(c, dA.p(), lda, m, n);
        if (norm_sq == 0.0) fail(SVDK_E_PARAM, "residual_delta: ||A||_F = 0, ratio undefined");
        if (r > 0) {
            DBuf dU = upload(c, u, m, r, ldu), dV = upload(c, v, n, r, ldv);
            DBuf dS(c, r), W(c, static_cast<size_t>(round_up(r, 2)) * n);
            h2d(c, dS.p(), sigma, r);
            // W = diag(sigma) V^T (r x n), then A <- A - U W
            const int64_t ldw = round_up(r, 2);
            transpose(c, dV.p(), ldv, n, r, W.p(), ldw);
            scale_rows(c, W.p(), ldw, r, n, dS.p());
            gemm(c, false, m, n, r, dU.p(), ldu, W.p(), ldw, dA.p(), lda, nullptr, false, -1.0, true);
        }
        *delta = std::sqrt(frob_sq(c, dA.p(), lda, m, n) / norm_sq);
    });
}

int svdk_dev_gemm(svdk_ctx* c, int transa, int64_t m, int64_t n, int64_t k, const double* a,
                  int64_t lda, const double* b, int64_t ldb, double* out, int64_t ldc) {
    return guarded([&] {
        need_ctx(c);
        gemm(c, transa != 0, m, n, k, a, lda, b, ldb, out, ldc);
    });
}

int svdk_dev_gram(svdk_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, double* g,
                  int64_t ldg) {
    return guarded([&] {
        need_ctx(c);
        syrk(c, m, n, a, lda, g, ldg);
    });
}

int svdk_dev_gemv_pair(svdk_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, const double* q,
                       double* w) {
    return guarded([&] {
        need_ctx(c);
        if (m < 0 || n < 0 || lda < std::max<int64_t>(m, 1)) fail(SVDK_E_DIM, "gemv_pair: bad shape");
        GemvPair g(c, a, lda, m, n);
        g.run(q, w);
    });
}

int svdk_dev_eig_sym(svdk_ctx* c, const double* s, int64_t n, int64_t lds, int max_sweeps,
                     double* w, double* v, int64_t ldv) {
    return guarded([&] {
        need_ctx(c);
        eig_sym(c, s, lds, n, max_sweeps, w, v, ldv);
    });
}

int svdk_dev_qr_thin(svdk_ctx* c, const double* h, int64_t m, int64_t p, int64_t ldh, double* q,
                     int64_t ldq, double* r, int64_t* rank) {
    return guarded([&] {
        need_ctx(c);
        if (m < p) fail(SVDK_E_DIM, "qr_thin: need rows >= cols");
        const int64_t rk = qr_thin(c, h, ldh, m, p, q, ldq, r, nullptr);
        if (rank) *rank = rk;
    });
}

int svdk_dev_pca(svdk_ctx* c, const double* a, int64_t m_local, int64_t n, int64_t lda, int method,
                 int64_t l, int64_t q, uint64_t seed, int center, double threshold, double* u,
                 int64_t ldu, double* sigma, double* v, int64_t ldv, double* mean, int64_t* rank,
                 int64_t* k, double* total) {
    return guarded([&] {
        need_ctx(c);
        dev_pca(c, a, m_local, n, lda, method, l, q, seed, center, threshold, u, ldu, sigma, v, ldv,
                mean, rank, k, total);
    });
}

int svdk_nccl_unique_id(char out[128]) {
    return guarded([&] { nccl_unique_id(out); });
}

int svdk_ctx_attach_nccl(svdk_ctx* c, const char id[128], int rank, int world) {
    return guarded([&] {
        need_ctx(c);
        attach_nccl(c, id, rank, world);
    });
}

int svdk_host_group_create(int world, svdk_host_group** out) {
    return guarded([&] {
        if (!out) fail(SVDK_E_PARAM, "host_group_create: null out");
        *out = reinterpret_cast<svdk_host_group*>(host_group_create(world));
    });
}

int svdk_host_group_destroy(svdk_host_group* g) {
    return guarded([&] { host_group_release(reinterpret_cast<HostGroup*>(g)); });
}

int svdk_ctx_attach_host_group(svdk_ctx* c, svdk_host_group* g, int rank) {
    return guarded([&] {
        need_ctx(c);
        attach_host_group(c, reinterpret_cast<HostGroup*>(g), rank);
    });
}

int svdk_ctx_detach_comm(svdk_ctx* c) {
    return guarded([&] {
        need_ctx(c);
        destroy_comm(c);
    });
}

int svdk_ctx_comm_info(svdk_ctx* c, int* rank, int* world) {
    return guarded([&] {
        need_ctx(c);
        if (rank) *rank = has_comm(c) ? c->rank : 0;
        if (world) *world = has_comm(c) ? c->world : 1;
    });
}

int svdk_cost_model(int model, uint64_t m, uint64_t n, uint64_t l, uint64_t i, double* flops,
                    double* space_entries, double* space_bytes) {
    return guarded([&] {
        const CostOut c = cost_model(model, m, n, l, i);
        if (flops) *flops = c.flops;
        if (space_entries) *space_entries = c.entries;
        if (space_bytes) *space_bytes = 8.0 * c.entries;
    });
}

int svdk_idx_parse(const uint8_t* bytes, uint64_t len, uint64_t dims[3], uint64_t* error_offset) {
    return guarded([&] {
        if (!bytes && len > 0) fail(SVDK_E_PARAM, "idx_parse: null buffer");
        idx_parse(bytes, len, dims, error_offset);
    });
}

int svdk_idx_to_matrix(svdk_ctx* c, const uint8_t* pixels, int64_t count, int64_t pixels_per_image,
                       double* out) {
    return guarded([&] {
        need_ctx(c);
        if (count < 0 || pixels_per_image < 0) fail(SVDK_E_PARAM, "idx_to_matrix: negative size");
        const int64_t bytes = count * pixels_per_image;
        if (bytes == 0) return;
        DBuf dpx(c, static_cast<size_t>(ceil_div(bytes, 8)));
        DBuf dout(c, static_cast<size_t>(bytes));
        SVDK_CUDA(cudaMemcpyAsync(dpx.p(), pixels, static_cast<size_t>(bytes),
                                  cudaMemcpyHostToDevice, c->stream));
        idx_to_matrix_dev(c, reinterpret_cast<const uint8_t*>(dpx.p()), count, pixels_per_image,
                          dout.p(), count);
        d2h(c, out, dout.p(), bytes);
    });
}

int svdk_dev_idx_to_matrix(svdk_ctx* c, const uint8_t* pixels, int64_t count,
                           int64_t pixels_per_image, double* out, int64_t ldo) {
    return guarded([&] {
        need_ctx(c);
        idx_to_matrix_dev(c, pixels, count, pixels_per_image, out, ldo);
    });
}

int svdk_dev_synth_fill(svdk_ctx* c, uint64_t seed, int stream, int quantise, int64_t m_total,
                        int64_t row0, int64_t rows, int64_t cols, double* out, int64_t ld) {
    return guarded([&] {
        need_ctx(c);
        synth_fill_dev(c, seed, stream, quantise, m_total, row0, rows, cols, out, ld);
    });
}

int svdk_dev_synth_add_noise(svdk_ctx* c, uint64_t seed, int64_t m_total, int64_t row0, int64_t rows,
                             int64_t cols, double sigma, double* a, int64_t lda) {
    return guarded([&] {
        need_ctx(c);
        synth_add_noise_dev(c, seed, m_total, row0, rows, cols, sigma, a, lda);
    });
}

}  // extern "C"
