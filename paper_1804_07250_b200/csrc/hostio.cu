// Host <-> device copies of the reference-layout grids through pinned
// staging (the drop-in path: random_walk_batch / the fused-walk hook take the
// caller's pageable numpy arrays, sweeps.py:278-316).
//
// A pageable cudaMemcpy is staged by the driver one bounce buffer at a time
// (~15 GB/s here), and the fresh output array of every call page-faults
// inside the copy (~10 ms for the 67 MB of Aztec 4096).  Instead:
//   H2D: host threads copy chunk i+1 of the caller's array into a pinned slot
//        while the DMA engine moves chunk i (3 slots of 8 MB);
//   D2H: host threads touch the destination's pages while the stream is
//        still busy (the walk), then chunks are DMA'd into pinned slots and
//        copied out by the threads as they land.
// Pinned (page-locked or registered) caller memory goes straight to
// cudaMemcpyAsync.  One staging engine per process, serialised by a mutex.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#include "tsb_internal.cuh"

namespace tsb {

namespace {

// fixed pool of host threads running parallel_for(n, fn) jobs
class CopyPool {
  public:
    explicit CopyPool(int n) : n_(n) {
        for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    // fn(part, nparts) on every pool thread (part 0 on the caller)
    void run(const std::function<void(int, int)> &fn) {
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            pending_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, n_);
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int, int)> *fn;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                fn = fn_;
            }
            (*fn)(id, n_);
            std::lock_guard<std::mutex> g(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int, int)> *fn_ = nullptr;
    int pending_ = 0;
    uint64_t gen_ = 0;
};

constexpr size_t kChunk = 8u << 20;
constexpr int kSlots = 3;
constexpr size_t kDirectBelow = 2u << 20;  // small grids: plain cudaMemcpyAsync

struct Stage {
    std::mutex mu;
    CopyPool *pool = nullptr;
    uint8_t *slot[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    bool busy[kSlots] = {};
    int device = -1;
};

Stage &stage() {
    static Stage s;
    return s;
}

void pool_init(Stage &s) {
    if (!s.pool) {
        const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
        unsigned n = std::min(8u, std::max(1u, hc / 2));
        if (const char *ev = getenv("TSB_COPY_THREADS")) n = (unsigned)std::max(1, atoi(ev));
        s.pool = new CopyPool((int)n);
    }
}

int stage_init(Stage &s) {
    int dev = 0;
    TSB_CUDA(cudaGetDevice(&dev));
    pool_init(s);
    if (s.device != dev) {  // (re)create slots and events on the current device
        for (int i = 0; i < kSlots; ++i) {
            if (s.slot[i]) {
                cudaEventSynchronize(s.ev[i]);
                cudaFreeHost(s.slot[i]);
                cudaEventDestroy(s.ev[i]);
                s.slot[i] = nullptr;
            }
        }
        for (int i = 0; i < kSlots; ++i) {
            TSB_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&s.slot[i]), kChunk, cudaHostAllocPortable));
            TSB_CUDA(cudaEventCreateWithFlags(&s.ev[i], cudaEventDisableTiming));
            s.busy[i] = false;
        }
        s.device = dev;
    }
    return TSB_OK;
}

void par_copy(CopyPool *pool, void *dst, const void *src, size_t n) {
    pool->run([&](int p, int np) {
        const size_t per = ((n + np - 1) / np + 4095) & ~(size_t)4095;
        const size_t a = std::min(n, per * p), b = std::min(n, a + per);
        if (b > a) std::memcpy(static_cast<uint8_t *>(dst) + a, static_cast<const uint8_t *>(src) + a, b - a);
    });
}

bool pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

}  // namespace

void host_parallel_for(int n, const std::function<void(int)> &fn) {
    if (n <= 1) {
        if (n == 1) fn(0);
        return;
    }
    Stage &s = stage();
    std::lock_guard<std::mutex> g(s.mu);
    pool_init(s);
    s.pool->run([&](int p, int np) {
        for (int i = p; i < n; i += np) fn(i);
    });
}

int staged_h2d(void *dev, const void *src, size_t bytes, cudaStream_t stream) {
    if (bytes < kDirectBelow || pinned(src)) {
        TSB_CUDA(cudaMemcpyAsync(dev, src, bytes, cudaMemcpyHostToDevice, stream));
        return TSB_OK;
    }
    Stage &s = stage();
    std::lock_guard<std::mutex> g(s.mu);
    int rc = stage_init(s);
    if (rc) return rc;
    const uint8_t *in = static_cast<const uint8_t *>(src);
    uint8_t *out = static_cast<uint8_t *>(dev);
    for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
        const int k = (int)(i % kSlots);
        const size_t len = std::min(kChunk, bytes - off);
        if (s.busy[k]) TSB_CUDA(cudaEventSynchronize(s.ev[k]));
        par_copy(s.pool, s.slot[k], in + off, len);
        TSB_CUDA(cudaMemcpyAsync(out + off, s.slot[k], len, cudaMemcpyHostToDevice, stream));
        TSB_CUDA(cudaEventRecord(s.ev[k], stream));
        s.busy[k] = true;
    }
    return TSB_OK;
}

// Returns with the copy complete (stream work up to it finished).
int staged_d2h(void *dst, const void *dev, size_t bytes, cudaStream_t stream) {
    if (bytes < kDirectBelow || pinned(dst)) {
        TSB_CUDA(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, stream));
        TSB_CUDA(cudaStreamSynchronize(stream));
        return TSB_OK;
    }
    Stage &s = stage();
    std::lock_guard<std::mutex> g(s.mu);
    int rc = stage_init(s);
    if (rc) return rc;
    uint8_t *out = static_cast<uint8_t *>(dst);
    const uint8_t *in = static_cast<const uint8_t *>(dev);
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) -> int {
        const int k = (int)(i % kSlots);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        if (s.busy[k]) TSB_CUDA(cudaEventSynchronize(s.ev[k]));
        TSB_CUDA(cudaMemcpyAsync(s.slot[k], in + off, len, cudaMemcpyDeviceToHost, stream));
        TSB_CUDA(cudaEventRecord(s.ev[k], stream));
        s.busy[k] = true;
        return TSB_OK;
    };
    for (size_t i = 0; i < std::min<size_t>(kSlots, nchunks); ++i)
        if ((rc = issue(i))) return rc;
    // first touch of the destination pages while the stream drains
    const long pg = std::max(4096L, sysconf(_SC_PAGESIZE));
    s.pool->run([&](int p, int np) {
        const size_t per = (bytes + np - 1) / np;
        const size_t a = std::min(bytes, per * p), b = std::min(bytes, a + per);
        for (size_t o = a - a % pg; o < b; o += pg)
            if (o >= a) reinterpret_cast<volatile uint8_t *>(out)[o] = 0;
    });
    for (size_t i = 0; i < nchunks; ++i) {
        const int k = (int)(i % kSlots);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        TSB_CUDA(cudaEventSynchronize(s.ev[k]));
        s.busy[k] = false;
        par_copy(s.pool, out + off, s.slot[k], len);
        if (i + kSlots < nchunks && (rc = issue(i + kSlots))) return rc;
    }
    return TSB_OK;
}

}  // namespace tsb
