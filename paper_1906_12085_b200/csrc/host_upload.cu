// host_upload.cu — host -> device uploads of a caller's buffer on the copy stream.
//
// Page-locked (pinned or cudaHostRegister'ed) buffers go straight to the DMA
// engine. A pageable buffer (the drop-in facade's std::vector) cannot be
// DMA'd asynchronously: cudaMemcpyAsync stages it synchronously on the calling
// thread, so the streamed fit_pca could not overlap anything. Here
// a pool of host threads packs each piece of a pageable source into one of
// three pinned staging slots (128 MiB each) and the DMA engine moves it from
// there at the pinned rate; a slot is refilled only after its previous DMA has
// completed (one event per slot), so packing piece k+1 overlaps the DMA of
// piece k and the device compute of the chunks that already landed.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "svdk_internal.h"

namespace svdk {

namespace {
constexpr size_t kSlotBytes = size_t(128) << 20;
constexpr int kSlots = 3;

// Fixed pool of workers running body(t) for t in [0, T) and joining.
class CopyPool {
public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    int size() const { return static_cast<int>(th_.size()); }
    void run(const std::function<void(int)>& body) {
        std::unique_lock<std::mutex> lk(mu_);
        body_ = &body;
        pending_ = size();
        ++gen_;
        cv_.notify_all();
        done_.wait(lk, [&] { return pending_ == 0; });
        body_ = nullptr;
    }

private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* b;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                b = body_;
            }
            (*b)(i);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* body_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
}  // namespace

struct UploadStaging {
    void* slot[kSlots] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev[kSlots] = {nullptr, nullptr, nullptr};
    bool used[kSlots] = {false, false, false};
    int next = 0;
    CopyPool* pool = nullptr;
    ~UploadStaging() {
        for (int i = 0; i < kSlots; ++i) {
            if (ev[i]) {
                cudaEventSynchronize(ev[i]);
                cudaEventDestroy(ev[i]);
            }
            if (slot[i]) cudaFreeHost(slot[i]);
        }
        delete pool;
    }
};

void release_upload_staging(Ctx* c) {
    delete c->upload;
    c->upload = nullptr;
}

bool host_is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

HostUploader::HostUploader(Ctx* c, const void* base) : c_(c), pageable_(!host_is_pinned(base)) {
    if (!c->copy_stream) {
        SVDK_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        SVDK_CUDA(cudaEventCreateWithFlags(&c->copy_ev, cudaEventDisableTiming));
    }
    if (pageable_ && !c->upload) {
        auto* u = new UploadStaging;
        c->upload = u;
        for (int i = 0; i < kSlots; ++i) {
            SVDK_CUDA(cudaMallocHost(&u->slot[i], kSlotBytes));
            SVDK_CUDA(cudaEventCreateWithFlags(&u->ev[i], cudaEventDisableTiming));
        }
        const unsigned hw = std::thread::hardware_concurrency();
        u->pool = new CopyPool(static_cast<int>(std::clamp(hw > 2 ? hw - 2 : 1u, 1u, 24u)));
    }
}

void HostUploader::copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height) {
    if (width == 0 || height == 0) return;
    cudaStream_t cs = c_->copy_stream;
    if (!pageable_) {
        SVDK_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, cs));
        return;
    }
    UploadStaging* u = c_->upload;
    // pieces of whole rows (or row segments when one row exceeds a slot)
    const size_t seg = std::min(width, kSlotBytes);
    for (size_t x0 = 0; x0 < width; x0 += seg) {
        const size_t w = std::min(seg, width - x0);
        const size_t rows_per = std::max<size_t>(1, kSlotBytes / w);
        for (size_t r0 = 0; r0 < height; r0 += rows_per) {
            const size_t rows = std::min(rows_per, height - r0);
            const int s = u->next;
            u->next = (u->next + 1) % kSlots;
            if (u->used[s]) SVDK_CUDA(cudaEventSynchronize(u->ev[s]));  // its previous DMA is done
            char* slot = static_cast<char*>(u->slot[s]);
            const char* sbase = static_cast<const char*>(src) + r0 * spitch + x0;
            const int T = u->pool->size();
            u->pool->run([&](int t) {
                const size_t bytes = rows * w;
                if (rows == 1) {  // split one long row segment over the threads
                    const size_t a = bytes * t / T, b = bytes * (t + 1) / T;
                    std::memcpy(slot + a, sbase + a, b - a);
                } else {
                    const size_t ra = rows * t / T, rb = rows * (t + 1) / T;
                    for (size_t r = ra; r < rb; ++r) std::memcpy(slot + r * w, sbase + r * spitch, w);
                }
            });
            SVDK_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dpitch + x0, dpitch, slot, w, w, rows,
                                        cudaMemcpyHostToDevice, cs));
            SVDK_CUDA(cudaEventRecord(u->ev[s], cs));
            u->used[s] = true;
        }
    }
}

}  // namespace svdk
