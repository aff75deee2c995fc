// comm.cu — row-sharded execution (one rank per GPU).
//
// The reference is single-process; this is the engine's one
// parallel strategy: A is split by rows, every reduction over the row index
// is a local DMMA kernel followed by an allreduce of the small result:
//   Gram       G = sum_p A_p^T A_p          allreduce n x n
//   A^T Y      Z = sum_p A_p^T Y_p          allreduce n x l
//   ||A||_F^2  and column sums              allreduce 1 / n
// and the n x n eigensolve runs on rank 0 with w, V broadcast (replicated
// inputs, so every rank can then form its U_p = A_p V / sigma locally).
//
// Two interchangeable backends behind RowComm:
//  * NCCL (production): one process per GPU, ncclAllReduce / ncclBroadcast on
//    the context stream over NVLink/NVSwitch.
//  * host group (svdk_host_group_*): ranks are contexts driven by host threads
//    of ONE process (any GPUs, including several ranks on one GPU). Each
//    collective synchronises the rank's stream, stages its buffer to host
//    memory, meets the others at a barrier and sums the staged buffers in rank
//    order (identical bits on every rank). No kernel ever waits on another
//    rank, so ranks sharing a GPU cannot deadlock it. It exists so the sharded
//    engine paths run (and are tested) without a multi-GPU node.
// A failure on one rank aborts the group (host: every waiting peer raises;
// NCCL: ncclCommAbort on the failing rank), and dev_pca agrees on argument
// validity with one status allreduce before any data collective.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "svdk_methods.h"

namespace svdk {

struct HostGroup {
    explicit HostGroup(int w) : world(w), slots(static_cast<size_t>(w)) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool aborted = false;
    std::string abort_msg;
    int refs = 1;  // the creator's handle + one per attached context
    std::vector<std::vector<double>> slots;
    std::vector<double> bcast;

    // Reusable barrier; throws on every waiter once any rank aborted.
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) fail(SVDK_E_STATE, "host group aborted: " + abort_msg);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return;
        }
        cv.wait(lk, [&] { return generation != gen || aborted; });
        if (aborted) fail(SVDK_E_STATE, "host group aborted: " + abort_msg);
    }
    void abort(const std::string& why) {
        std::lock_guard<std::mutex> lk(mu);
        if (!aborted) abort_msg = why;
        aborted = true;
        cv.notify_all();
    }
};

namespace {
ncclComm_t comm_of(Ctx* c) { return static_cast<ncclComm_t>(c->nccl_comm); }

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(SVDK_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

void release_group(HostGroup* g) {
    if (!g) return;
    bool last = false;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        last = --g->refs == 0;
    }
    if (last) delete g;
}
}  // namespace

bool has_comm(const Ctx* c) { return (c->nccl_comm || c->host_group) && c->world > 1; }

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

HostGroup* host_group_create(int world) {
    if (world < 1) fail(SVDK_E_PARAM, "host_group: world must be >= 1");
    return new HostGroup(world);
}

void host_group_release(HostGroup* g) { release_group(g); }

void attach_host_group(Ctx* c, HostGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->world) fail(SVDK_E_PARAM, "attach_host_group: bad rank/group");
    destroy_comm(c);
    {
        std::lock_guard<std::mutex> lk(g->mu);
        ++g->refs;
    }
    c->host_group = g;
    c->rank = rank;
    c->world = g->world;
}

void destroy_comm(Ctx* c) {
    if (c->nccl_comm) {
        ncclCommDestroy(comm_of(c));
        c->nccl_comm = nullptr;
    }
    if (c->host_group) {
        release_group(c->host_group);
        c->host_group = nullptr;
    }
    c->rank = 0;
    c->world = 1;
}

// A collective could not complete on this rank: make the peers fail instead
// of waiting forever. NCCL: the communicator is aborted (the context must be
// re-attached); host group: every rank waiting at a barrier raises.
void abort_comm(Ctx* c, const std::string& why) {
    if (c->host_group) c->host_group->abort(why);
    if (c->nccl_comm) {
        ncclCommAbort(comm_of(c));
        c->nccl_comm = nullptr;
        c->world = 1;
        c->rank = 0;
    }
}

void RowComm::allreduce(double* buf, size_t count) const {
    if (!has_comm(c) || count == 0) return;
    if (c->nccl_comm) {
        nccl_check(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, comm_of(c), c->stream),
                   "ncclAllReduce");
        return;
    }
    HostGroup* g = c->host_group;
    std::vector<double>& mine = g->slots[static_cast<size_t>(c->rank)];
    mine.resize(count);
    SVDK_CUDA(cudaMemcpyAsync(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
    g->barrier();
    std::vector<double> sum(g->slots[0]);
    for (int r = 1; r < g->world; ++r) {
        const std::vector<double>& s = g->slots[static_cast<size_t>(r)];
        if (s.size() != count) {
            g->abort("allreduce size mismatch");
            fail(SVDK_E_STATE, "host group: allreduce size mismatch across ranks");
        }
        for (size_t i = 0; i < count; ++i) sum[i] += s[i];
    }
    g->barrier();  // every rank has read every slot
    SVDK_CUDA(cudaMemcpyAsync(buf, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
}

void RowComm::broadcast(double* buf, size_t count, int root) const {
    if (!has_comm(c) || count == 0) return;
    if (c->nccl_comm) {
        nccl_check(ncclBroadcast(buf, buf, count, ncclDouble, root, comm_of(c), c->stream),
                   "ncclBroadcast");
        return;
    }
    HostGroup* g = c->host_group;
    if (c->rank == root) {
        g->bcast.resize(count);
        SVDK_CUDA(cudaMemcpyAsync(g->bcast.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost,
                                  c->stream));
        SVDK_CUDA(cudaStreamSynchronize(c->stream));
    }
    g->barrier();
    if (c->rank != root) {
        if (g->bcast.size() != count) {
            g->abort("broadcast size mismatch");
            fail(SVDK_E_STATE, "host group: broadcast size mismatch across ranks");
        }
        SVDK_CUDA(cudaMemcpyAsync(buf, g->bcast.data(), count * sizeof(double), cudaMemcpyHostToDevice,
                                  c->stream));
        SVDK_CUDA(cudaStreamSynchronize(c->stream));
    }
    g->barrier();  // the root may reuse bcast afterwards
}

int RowComm::rank() const { return has_comm(c) ? c->rank : 0; }
int RowComm::world() const { return has_comm(c) ? c->world : 1; }

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

// Agree across ranks on whether every rank's arguments are valid (status 0)
// before any data collective: the first failing rank's code is raised on all.
void agree_status(Ctx* c, const RowComm* comm, int code, const std::string& msg) {
    if (!comm || comm->world() == 1) {
        if (code) fail(code, msg);
        return;
    }
    std::vector<double> st(static_cast<size_t>(comm->world()), 0.0);
    st[static_cast<size_t>(comm->rank())] = static_cast<double>(code);
    DBuf d(c, st.size());
    h2d(c, d.p(), st.data(), static_cast<int64_t>(st.size()));
    comm->allreduce(d.p(), st.size());
    d2h(c, st.data(), d.p(), static_cast<int64_t>(st.size()));
    for (size_t r = 0; r < st.size(); ++r)
        if (st[r] != 0.0)
            fail_agreed(static_cast<int>(st[r]),
                        code ? msg : "rank " + std::to_string(r) + " rejected its arguments");
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
        fail_agreed(static_cast<int>(st[0]), msg.empty() ? "eig_sym failed on rank 0" : msg, st[1]);
    comm->broadcast(w, static_cast<size_t>(n), 0);
    comm->broadcast(V, static_cast<size_t>(n) * n, 0);
}

}  // namespace svdk
