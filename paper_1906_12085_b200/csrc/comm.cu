// comm.cu — row-sharded execution over NCCL (one process per GPU).
//
// The reference is single-process; this is the engine's one
// parallel strategy: A is split by rows, every reduction over the row index
// is a local DMMA kernel followed by an NCCL allreduce over NVLink/NVSwitch:
//   Gram       G = sum_p A_p^T A_p          allreduce n x n
//   A^T Y      Z = sum_p A_p^T Y_p          allreduce n x l
//   ||A||_F^2  and column sums              allreduce 1 / n
// and the n x n eigensolve runs on rank 0 with w, V broadcast (replicated
// inputs, so every rank can then form its U_p = A_p V / sigma locally).
#include <nccl.h>

#include <cstring>

#include "svdk_methods.h"

namespace svdk {

namespace {
ncclComm_t comm_of(Ctx* c) { return static_cast<ncclComm_t>(c->nccl_comm); }

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SVDK_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

void nccl_unique_id(char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "nccl id size");
    ncclUniqueId id;
    nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
}

void attach_nccl(Ctx* c, const char id_bytes[128], int rank, int world) {
    if (world < 1 || rank < 0 || rank >= world) fail(SVDK_E_PARAM, "attach_nccl: bad rank/world");
    destroy_comm(c);
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, 128);
    SVDK_CUDA(cudaSetDevice(c->device));
    ncclComm_t comm;
    nccl_check(ncclCommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    c->nccl_comm = comm;
    c->rank = rank;
    c->world = world;
}

void destroy_comm(Ctx* c) {
    if (c->nccl_comm) {
        ncclCommDestroy(comm_of(c));
        c->nccl_comm = nullptr;
    }
    c->rank = 0;
    c->world = 1;
}

void RowComm::allreduce(double* buf, size_t count) const {
    if (!c->nccl_comm || count == 0) return;
    nccl_check(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_of(c), c->stream),
               "ncclAllReduce");
}

void RowComm::broadcast(double* buf, size_t count, int root) const {
    if (!c->nccl_comm || count == 0) return;
    nccl_check(ncclBroadcast(buf, buf, count, ncclDouble, root, comm_of(c), c->stream),
               "ncclBroadcast");
}

int RowComm::rank() const { return c->rank; }
int RowComm::world() const { return c->nccl_comm ? c->world : 1; }

void gram_rows(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* G, int64_t ldg,
               const RowComm* comm) {
    syrk(c, m, n, A, lda, G, ldg);
    if (comm && comm->world() > 1) {
        if (ldg != n) fail(SVDK_E_STATE, "gram_rows: sharded Gram needs ldg == n");
        comm->allreduce(G, static_cast<size_t>(n) * n);
    }
}

void gemm_tn_rows(Ctx* c, int64_t n, int64_t l, int64_t m, const double* A, int64_t lda,
                  const double* B, int64_t ldb, double* C, int64_t ldc, const RowComm* comm) {
    gemm(c, true, n, l, m, A, lda, B, ldb, C, ldc);
    if (comm && comm->world() > 1) {
        if (ldc != n) fail(SVDK_E_STATE, "gemm_tn_rows: sharded A^T B needs ldc == n");
        comm->allreduce(C, static_cast<size_t>(n) * l);
    }
}

double frob_sq_rows(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n,
                    const RowComm* comm) {
    if (!comm || comm->world() == 1) return frob_sq(c, A, lda, m, n);
    const double local = frob_sq(c, A, lda, m, n);
    DBuf t(c, 1);
    h2d(c, t.p(), &local, 1);
    comm->allreduce(t.p(), 1);
    double out = 0.0;
    d2h(c, &out, t.p(), 1);
    return out;
}

void frob_sq_rows_dev(Ctx* c, const double* A, int64_t lda, int64_t m, int64_t n, double* d_out,
                      const RowComm* comm) {
    frob_sq_dev(c, A, lda, m, n, d_out);
    if (comm && comm->world() > 1) comm->allreduce(d_out, 1);
}

void eig_sym_rows(Ctx* c, const double* S, int64_t lds, int64_t n, double* w, double* V,
                  int64_t ldv, const RowComm* comm) {
    if (!comm || comm->world() == 1) {
        eig_sym(c, S, lds, n, 30, w, V, ldv);
        return;
    }
    if (ldv != n) fail(SVDK_E_STATE, "eig_sym_rows: needs ldv == n");
    // Status travels with the data: rank 0 broadcasts [status, off, w, V].
    DBuf status(c, 2);
    double st[2] = {0.0, 0.0};
    int code = 0;
    std::string msg;
    if (comm->rank() == 0) {
        try {
            eig_sym(c, S, lds, n, 30, w, V, ldv);
        } catch (const Failure& f) {
            code = f.code;
            msg = f.msg;
            st[1] = f.residual;
        }
        st[0] = static_cast<double>(code);
    }
    h2d(c, status.p(), st, 2);
    comm->broadcast(status.p(), 2, 0);
    d2h(c, st, status.p(), 2);
    if (st[0] != 0.0)
        fail(static_cast<int>(st[0]), msg.empty() ? "eig_sym failed on rank 0" : msg, st[1]);
    comm->broadcast(w, static_cast<size_t>(n), 0);
    comm->broadcast(V, static_cast<size_t>(n) * n, 0);
}

}  // namespace svdk
