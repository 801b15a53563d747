// hoststage.h -- pageable host buffers through a library-owned pinned ring.
//
// The reference's callers hand gemm_execute plain (pageable) numpy arrays and
// get a fresh numpy array back (kernels.py:328-349).  A DMA engine can only
// read / write page-locked memory, so pageable bytes must be staged: the
// driver's own pageable copy stages them with one thread and blocks, and
// cudaHostRegister of the caller's buffers pins every page per call (both
// measured far below the PCIe rate on the B200 box).  Here the host thread
// and a small pool of copy workers move the bytes between the caller's
// buffers and a ring of pinned slots in parallel, while the copy engines
// move slot i-1 / i+1 over PCIe, so host copies, DMA and the kernels overlap.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ag {
namespace hoststage {

// A fixed pool of copy workers.  run(n, fn) executes fn(0..n-1) on the
// workers and the calling thread and returns when every item is done.
// Parallel jobs are serialised (one job at a time, any number of callers).
// A call issues several jobs in a row (every ring slot is one), so an idle
// worker spins for kSpinUs before it sleeps: waking a sleeping thread costs
// tens of microseconds, a 4 MB slot copy on 8 threads about 80.
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // never destroyed: workers may outlive static teardown
        return *p;
    }
    int threads() const { return (int)workers_.size() + 1; }

    void run(int n, const std::function<void(int)>& fn) {
        if (n <= 1 || workers_.empty()) {
            for (int i = 0; i < n; ++i) fn(i);
            return;
        }
        std::lock_guard<std::mutex> serial(call_mu_);
        Job j;
        j.fn = &fn;
        j.n = n;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &j;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        items(&j);
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return j.done.load() == n && j.inside == 0; });
        job_ = nullptr;
    }

  private:
    struct Job {
        const std::function<void(int)>* fn = nullptr;
        int n = 0;
        std::atomic<int> next{0}, done{0};
        int inside = 0;  // workers inside items(), guarded by mu_
    };

    CopyPool() {
        unsigned hc = std::thread::hardware_concurrency();
        int want = (int)std::min<unsigned>(hc > 1 ? hc / 2 : 1, 8);  // 8 threads: ~78 GB/s pageable->pinned on the B200 box
        if (const char* e = std::getenv("AG_HOST_COPY_THREADS")) want = std::max(1, std::atoi(e));
        for (int i = 0; i + 1 < want; ++i) workers_.emplace_back([this] { loop(); });
        for (auto& t : workers_) t.detach();
    }

    void items(Job* j) {
        for (;;) {
            const int i = j->next.fetch_add(1);
            if (i >= j->n) break;
            (*j->fn)(i);
            if (j->done.fetch_add(1) + 1 == j->n) {
                std::lock_guard<std::mutex> lk(mu_);
                done_cv_.notify_all();
            }
        }
    }

    static constexpr int kSpinUs = 300;

    void loop() {
        uint64_t seen = 0;
        for (;;) {
            // spin a while for the next job (lock-free read of the generation)
            const auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; gen_.load(std::memory_order_acquire) == seen; ++i) {
                if ((i & 255) == 255 &&
                    std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(kSpinUs))
                    break;
#if defined(__x86_64__) || defined(__i386__)
                __builtin_ia32_pause();
#endif
            }
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return job_ != nullptr && gen_.load() != seen; });
            seen = gen_.load();
            Job* j = job_;
            ++j->inside;
            lk.unlock();
            items(j);
            lk.lock();
            if (--j->inside == 0) done_cv_.notify_all();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    Job* job_ = nullptr;
    std::atomic<uint64_t> gen_{0};
};

// rows x width bytes between pitched host buffers, split over the pool
// (by bytes when both sides are contiguous, else by rows)
inline void copy_rows(char* dst, int64_t dpitch, const char* src, int64_t spitch, int64_t width, int64_t rows) {
    if (rows <= 0 || width <= 0) return;
    if (dpitch == width && spitch == width) {  // one contiguous run
        width *= rows;
        rows = 1;
    }
    const int64_t total = width * rows;
    constexpr int64_t kGrain = 512 << 10;
    CopyPool& pool = CopyPool::get();
    const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool.threads(), total / kGrain));
    if (parts <= 1) {
        for (int64_t r = 0; r < rows; ++r) memcpy(dst + r * dpitch, src + r * spitch, (size_t)width);
        return;
    }
    if (rows == 1) {
        const int64_t step = (width / parts + 63) / 64 * 64;
        pool.run(parts, [&](int i) {
            const int64_t b = std::min(width, i * step), e = std::min(width, b + step);
            if (e > b) memcpy(dst + b, src + b, (size_t)(e - b));
        });
        return;
    }
    const int p = (int)std::min<int64_t>(parts, rows);
    pool.run(p, [&](int i) {
        const int64_t r0 = rows * i / p, r1 = rows * (i + 1) / p;
        for (int64_t r = r0; r < r1; ++r) memcpy(dst + r * dpitch, src + r * spitch, (size_t)width);
    });
}

// Spin on a CUDA event / stream instead of the runtime's synchronize: the
// runtime may block the thread and wake it through the OS (tens of
// microseconds per wait on this box), and a host-path call waits several
// times on short DMAs.
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}
inline cudaError_t spin_event(cudaEvent_t e) {
    for (;;) {
        const cudaError_t r = cudaEventQuery(e);
        if (r != cudaErrorNotReady) return r;
        cpu_relax();
    }
}
inline cudaError_t spin_stream(cudaStream_t st) {
    for (;;) {
        const cudaError_t r = cudaStreamQuery(st);
        if (r != cudaErrorNotReady) return r;
        cpu_relax();
    }
}

inline bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// One pinned ring: kSlots slots of kSlotBytes, each with the event of the
// DMA that last used it.
struct Ring {
    // small slots: the DMA of slot i overlaps the host copy of slot i + 1
    static constexpr int kSlots = 8;
    static constexpr size_t kSlotBytes = 4u << 20;
    char* base = nullptr;
    cudaEvent_t ev[kSlots] = {};
    bool busy[kSlots] = {};
    int next = 0;
    bool ok() {
        if (base) return true;
        void* p = nullptr;
        if (cudaHostAlloc(&p, kSlots * kSlotBytes, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        for (auto& e : ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
        base = static_cast<char*>(p);
        return true;
    }
    char* slot(int i) const { return base + (size_t)i * kSlotBytes; }
};

// A pitched block: `rows` rows of `width` bytes on each side.
struct Block {
    char* host;  // const for H2D
    int64_t hpitch;
    char* dev;
    int64_t dpitch;
    int64_t width, rows;
};

// chunks of whole rows (or of bytes, for one contiguous run) that fit a slot
struct Chunk {
    int64_t r0, nr;     // rows
    int64_t b0, nb;     // byte range within the row (contiguous runs)
};
inline std::vector<Chunk> chunks_of(Block& b) {
    std::vector<Chunk> out;
    if (b.hpitch == b.width && b.dpitch == b.width) {  // flatten
        b.width *= b.rows;
        b.hpitch = b.dpitch = b.width;
        b.rows = 1;
    }
    if (b.rows == 1) {
        for (int64_t o = 0; o < b.width; o += (int64_t)Ring::kSlotBytes)
            out.push_back({0, 1, o, std::min<int64_t>((int64_t)Ring::kSlotBytes, b.width - o)});
        return out;
    }
    const int64_t per = std::max<int64_t>(1, (int64_t)Ring::kSlotBytes / b.width);
    for (int64_t r = 0; r < b.rows; r += per) out.push_back({r, std::min(per, b.rows - r), 0, b.width});
    return out;
}

// Host -> device through the ring on `st`: returns the first CUDA error.
inline cudaError_t h2d(Ring& ring, Block b, cudaStream_t st) {
    if (b.rows <= 0 || b.width <= 0) return cudaSuccess;
    if (b.width > (int64_t)Ring::kSlotBytes && !(b.hpitch == b.width && b.dpitch == b.width))  // one row > slot
        return cudaMemcpy2DAsync(b.dev, (size_t)b.dpitch, b.host, (size_t)b.hpitch, (size_t)b.width, (size_t)b.rows,
                                 cudaMemcpyHostToDevice, st);
    for (const Chunk& c : chunks_of(b)) {
        const int s = ring.next;
        ring.next = (ring.next + 1) % Ring::kSlots;
        if (ring.busy[s]) {
            cudaError_t e = spin_event(ring.ev[s]);
            if (e != cudaSuccess) return e;
        }
        char* slot = ring.slot(s);
        copy_rows(slot, c.nb, b.host + c.r0 * b.hpitch + c.b0, b.hpitch, c.nb, c.nr);
        cudaError_t e = cudaMemcpy2DAsync(b.dev + c.r0 * b.dpitch + c.b0, (size_t)b.dpitch, slot, (size_t)c.nb,
                                          (size_t)c.nb, (size_t)c.nr, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return e;
        if ((e = cudaEventRecord(ring.ev[s], st)) != cudaSuccess) return e;
        ring.busy[s] = true;
    }
    return cudaSuccess;
}

// Device -> host through the ring on `st` (after whatever `st` already
// waits on); blocks until every byte is in the caller's buffer.
inline cudaError_t d2h(Ring& ring, Block b, cudaStream_t st) {
    if (b.rows <= 0 || b.width <= 0) return cudaSuccess;
    if (b.width > (int64_t)Ring::kSlotBytes && !(b.hpitch == b.width && b.dpitch == b.width)) {
        cudaError_t e = cudaMemcpy2DAsync(b.host, (size_t)b.hpitch, b.dev, (size_t)b.dpitch, (size_t)b.width,
                                          (size_t)b.rows, cudaMemcpyDeviceToHost, st);
        return e != cudaSuccess ? e : spin_stream(st);
    }
    const std::vector<Chunk> cs = chunks_of(b);
    const int n = (int)cs.size();
    auto issue = [&](int i) {
        const Chunk& c = cs[i];
        const int s = i % Ring::kSlots;
        cudaError_t e = cudaMemcpy2DAsync(ring.slot(s), (size_t)c.nb, b.dev + c.r0 * b.dpitch + c.b0,
                                          (size_t)b.dpitch, (size_t)c.nb, (size_t)c.nr, cudaMemcpyDeviceToHost, st);
        return e != cudaSuccess ? e : cudaEventRecord(ring.ev[s], st);
    };
    for (int i = 0; i < std::min(n, Ring::kSlots); ++i) {
        cudaError_t e = issue(i);
        if (e != cudaSuccess) return e;
    }
    for (int i = 0; i < n; ++i) {
        const Chunk& c = cs[i];
        const int s = i % Ring::kSlots;
        cudaError_t e = spin_event(ring.ev[s]);
        if (e != cudaSuccess) return e;
        copy_rows(b.host + c.r0 * b.hpitch + c.b0, b.hpitch, ring.slot(s), c.nb, c.nb, c.nr);
        if (i + Ring::kSlots < n && (e = issue(i + Ring::kSlots)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace hoststage
}  // namespace ag
