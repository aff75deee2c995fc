// context.cu — engine context, stream-ordered device pool, error plumbing.
#include <algorithm>
#include <cstring>

#include "svdk_internal.h"

namespace svdk {

[[noreturn]] void fail(int code, const std::string& msg, double residual) {
    throw Failure{code, msg, residual};
}

[[noreturn]] void fail_agreed(int code, const std::string& msg, double residual) {
    throw Failure{code, msg, residual, true};
}

// ---------------------------------------------------------------------------
// Pool: grow-only set of cudaMalloc blocks, best-fit reuse. All users order
// their work on the context's single stream, so a block returned to the pool
// may be handed out again immediately (stream order protects it).
// ---------------------------------------------------------------------------
Pool::~Pool() { trim(); }

void* Pool::get(size_t bytes) {
    bytes = std::max<size_t>(256, (bytes + 255) & ~size_t(255));
    Block* best = nullptr;
    for (auto& b : blocks_)
        if (!b.busy && b.bytes >= bytes && (!best || b.bytes < best->bytes)) best = &b;
    // do not let a huge idle block serve a tiny request
    if (best && best->bytes <= 2 * bytes + (64u << 20)) {
        best->busy = true;
        return best->p;
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        // release idle blocks and retry once
        cudaDeviceSynchronize();
        for (auto it = blocks_.begin(); it != blocks_.end();) {
            if (!it->busy) {
                cudaFree(it->p);
                reserved_ -= it->bytes;
                it = blocks_.erase(it);
            } else {
                ++it;
            }
        }
        e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(SVDK_E_NOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
        }
    }
    blocks_.push_back({p, bytes, true});
    reserved_ += bytes;
    return p;
}

void Pool::put(void* p) {
    for (auto& b : blocks_)
        if (b.p == p) {
            b.busy = false;
            return;
        }
}

void Pool::trim() {
    for (auto it = blocks_.begin(); it != blocks_.end();) {
        if (!it->busy) {
            cudaFree(it->p);
            reserved_ -= it->bytes;
            it = blocks_.erase(it);
        } else {
            ++it;
        }
    }
}

DBuf::DBuf(Ctx* c, size_t count) : c_(c), n_(count) {
    p_ = static_cast<double*>(c->pool.get(std::max<size_t>(count, 1) * sizeof(double)));
}
DBuf& DBuf::operator=(DBuf&& o) noexcept {
    if (this != &o) {
        reset();
        c_ = o.c_;
        p_ = o.p_;
        n_ = o.n_;
        o.c_ = nullptr;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}
DBuf::~DBuf() { reset(); }
void DBuf::reset() {
    if (c_ && p_) c_->pool.put(p_);
    c_ = nullptr;
    p_ = nullptr;
    n_ = 0;
}

namespace {
cudaEvent_t take_event(Ctx* c) {
    if (c->events_used == c->event_pool.size()) {
        cudaEvent_t e;
        SVDK_CUDA(cudaEventCreate(&e));
        c->event_pool.push_back(e);
    }
    return c->event_pool[c->events_used++];
}
}  // namespace

PhaseTimer::PhaseTimer(Ctx* c, const char* name, double flops, double bytes) : c_(c) {
    if (!c->timing) return;
    PhaseRecord r{name, take_event(c), take_event(c), flops, bytes};
    SVDK_CUDA(cudaEventRecord(r.e0, c->stream));
    idx_ = static_cast<long>(c->records.size());
    c->records.push_back(r);
}

PhaseTimer::~PhaseTimer() {
    if (idx_ >= 0) cudaEventRecord(c_->records[idx_].e1, c_->stream);
}

void h2d(Ctx* c, double* dst, const double* src, int64_t count) {
    if (count <= 0) return;
    SVDK_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
}
void d2h(Ctx* c, double* dst, const double* src, int64_t count) {
    if (count <= 0) return;
    SVDK_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    SVDK_CUDA(cudaStreamSynchronize(c->stream));
}
void sync(Ctx* c) { SVDK_CUDA(cudaStreamSynchronize(c->stream)); }

}  // namespace svdk
