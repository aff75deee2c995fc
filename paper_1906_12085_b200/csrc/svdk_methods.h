// svdk_methods.h — engine-internal method entry points (device operands).
#pragma once

#include <functional>

#include "svdk_internal.h"
#include "tma_util.h"

namespace svdk {

// Row-sharded execution: A is split by rows over `world` ranks (NCCL: one
// process per GPU; host group: host threads of one process). Every reduction
// over the row index (Gram, A^T Y, column sums, norms) is followed by an
// allreduce; the n x n eigensolve runs on rank 0 and its result is
// broadcast. nullptr = single GPU. Backends in comm.cu.
struct RowComm {
    Ctx* c;
    void allreduce(double* buf, size_t count) const;
    void broadcast(double* buf, size_t count, int root) const;
    int rank() const;
    int world() const;
};

// Sum-reduce over rows helpers honouring an optional RowComm.
void gram_rows(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* G, int64_t ldg,
               const RowComm* comm);
void gemm_tn_rows(Ctx* c, int64_t n, int64_t l, int64_t m, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc, const RowComm* comm);
double frob_sq_rows(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                    const RowComm* comm);
// eig_sym on rank 0 (or the only GPU) + broadcast of w and V.
void eig_sym_rows(Ctx* c, const double* S, int64_t lds, int64_t n, double* w, double* V,
                  int64_t ldv, const RowComm* comm);

void nccl_unique_id(char out[128]);
void attach_nccl(Ctx* c, const char id[128], int rank, int world);
HostGroup* host_group_create(int world);
void host_group_release(HostGroup* g);
void attach_host_group(Ctx* c, HostGroup* g, int rank);
void destroy_comm(Ctx* c);
// true when a communicator (NCCL or host group) with world > 1 is attached
bool has_comm(const Ctx* c);
// make the peers fail instead of waiting forever (a rank's call failed)
void abort_comm(Ctx* c, const std::string& why);
// raise `code` on every rank if any rank's code is non-zero (before data collectives)
void agree_status(Ctx* c, const struct RowComm* comm, int code, const std::string& msg);

// Total of squares over all row shards into a device scalar (no host sync).
void frob_sq_rows_dev(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* d_out,
                      const RowComm* comm);
// Reference Gaussian sampler (host, bit-identical) staged through pinned
// memory. omega_prefetch starts filling it on a host thread so the sample is
// ready when the first GEMM needs it; omega_upload joins (or generates) and
// issues the H2D copy on `stream` (default: the context stream).
void omega_prefetch(Ctx* c, int64_t rows, int64_t cols, uint64_t seed);
void omega_upload(Ctx* c, int64_t rows, int64_t cols, uint64_t seed, double* d_out,
                  cudaStream_t stream = nullptr);
void release_host_staging(Ctx* c);

// Non-finite GEMM results (kernels.cpp:39-43) set a sticky device flag; the
// method entry points reset it and raise NumericalError once at the end.
void raise_if_nonfinite(Ctx* c);
void reset_nonfinite(Ctx* c);
// sigma from eigenvalues + numerical rank (svd_methods.cpp:127-135)
int64_t spectrum(Ctx* c, const double* w, int64_t n, double* sigma);
// normalize_signs on already-formed U, V (svd_methods.cpp:50-71)
// normalize_signs on V alone (svd_methods.cpp:50-71): flips V's columns and
// writes d_sign[j] = +-1, the flip its U column needs (folded into a GEMM).
void signs_v(Ctx* c, double* V, int64_t ldv, int64_t n, int64_t rank, double* d_sign);


// w = A^T (A q) (n x 1) for a fixed A: the Lanczos matvec pair (lanczos.cu).
// Construction picks the kernel form and prepares its tensor map/workspace;
// run() enqueues one product on the context stream (no host sync).
class GemvPair {
public:
    GemvPair(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n);
    // reduce = false leaves the cluster form's per-cluster column partials
    // unsummed (partials()/parts(); the caller fuses the sum) — parts() is 0
    // when w was written directly.
    void run(const double* q, double* w, bool reduce = true);
    bool one_read() const { return cluster_; }
    int parts() const { return cluster_ && m_ > 0 && n_ > 0 ? nclusters_ : 0; }
    const double* partials() const { return partial_.p(); }

private:
    Ctx* c_;
    const double* A_;
    int64_t lda_, m_, n_;
    bool cluster_ = false, la_ = true;
    int cs_ = 4, nclusters_ = 1, ncta_ = 0;
    size_t smem_ = 0;
    int64_t chunks_ = 1;
    CUtensorMap map_{};
    DBuf partial_, yv_;
};

int64_t truncated_svd(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* U,
                      int64_t ldu, double* sigma, double* V, int64_t ldv,
                      const RowComm* comm = nullptr);

// Full PCA pipeline on a device-resident (local shard of) A; see svdk.h.
// Host-buffer / dispatch helpers (abi.cu)
DBuf upload(Ctx* c, const double* h, int64_t rows, int64_t cols, int64_t& ld);
DBuf alloc_mat(Ctx* c, int64_t rows, int64_t cols, int64_t& ld);
void download(Ctx* c, double* h, const double* d, int64_t ld, int64_t rows, int64_t cols);
int64_t run_method(Ctx* c, int method, const double* dA, int64_t lda, int64_t m, int64_t n, int64_t l,
                   int64_t q, uint64_t seed, double* dU, int64_t ldu, double* dS, double* dV, int64_t ldv,
                   const RowComm* comm);
int64_t method_width(int method, int64_t m, int64_t n, int64_t l, int64_t q);
void validate_method(int method, int64_t m, int64_t n, int64_t l, int64_t q, const char* name);
int64_t truncated_from_gram(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, DBuf G,
                            double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                            const RowComm* comm);
int64_t randomized_from_sketch(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, int64_t l,
                               int64_t q, DBuf H, int64_t ldh, double* U, int64_t ldu, double* sigma,
                               double* V, int64_t ldv, const RowComm* comm, const double* Z_first = nullptr);
// Host-buffer fit_pca (RowsAreExamples, centred, tall, truncated/randomized)
// with the H2D copy streamed in column chunks under the Gram / sketch; returns
// false (nothing done) when the shape does not qualify.
bool fit_pca_streamed(Ctx* c, const double* host, int64_t m, int64_t n, int method, int64_t l, int64_t q,
                      uint64_t seed, double* basis, double* eigenvalues, double* total, double* mean,
                      int64_t* rank);
void dev_pca(Ctx* c, const double* A, int64_t m_local, int64_t n, int64_t lda, int method,
             int64_t l, int64_t q, uint64_t seed, int center_mode, double threshold, double* U,
             int64_t ldu, double* sigma, double* V, int64_t ldv, double* mean, int64_t* rank,
             int64_t* k, double* total);

}  // namespace svdk
