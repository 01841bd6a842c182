// arena.h -- the per-device scratch pool of libstarmm_b200 (host-side C++).
//
// Reference: Pool / BlockHandle (pool.py:27-167) -- exact-size free stacks, LIFO
// reuse (pool.py:97), blocks never cleared (pool.py:4-6), fresh / reuse / high-water
// counters (pool.py:134-146), reset frees everything (pool.py:148-156) -- and
// Executor.acquire_temp / release_temp (runtime.py:198-229).
//
// B200 design: ONE pool per device, shared by every plan and one-shot call on that
// device, surviving across calls until starmm_pool_reset() (the reference pool lives as
// long as its Executor; here plan create/destroy is cheap because nothing is freed).
// Reuse is ordered on the device, never on the host: a released block carries a
// Fence (an event recorded on the stream that last used it), and an acquire from a
// different stream makes that stream wait on the event (cudaStreamWaitEvent).  Blocks
// released and re-acquired on the same stream need nothing: stream order protects them.
// The FIFO discipline is the reference's negative control (pool.py:70-74): it hands out
// the block released longest ago, so a LIFO-dependent space bound breaks under it.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace starmm_host {

constexpr int MAX_DEVICES = 64;

// An event recorded on `st`; shared by every block released together.  The event goes
// back to its device's event pool when the last block holding it is re-acquired.
struct Fence {
    cudaEvent_t ev = nullptr;
    cudaStream_t st = nullptr;
    std::vector<cudaEvent_t>* pool = nullptr;
    std::mutex* mu = nullptr;
    ~Fence() {
        if (!ev) return;
        std::lock_guard<std::mutex> g(*mu);
        pool->push_back(ev);
    }
};
using FenceRef = std::shared_ptr<Fence>;

struct PoolCounts {
    long long allocated = 0;     // bytes currently owned (cudaMalloc'ed, issued or cached)
    long long cached = 0;        // bytes sitting in the free stacks
    long long issued = 0;        // bytes currently handed out
    long long high_water = 0;    // max issued since the last reset of the counters
    long long fresh = 0;         // acquisitions served by cudaMalloc
    long long reuse = 0;         // acquisitions served from a free stack
    long long waits = 0;         // cross-stream reuses ordered by cudaStreamWaitEvent
    long long trims = 0;         // blocks returned to the driver to make room
};

struct DevArena {
    int device = 0;
    int fifo = 0;                       // 0: LIFO (the reference), 1: FIFO (negative control)
    long long limit = 0;                // owned-bytes ceiling before cached blocks are trimmed
    std::mutex mu;                      // the pool is shared by every plan on the device
    struct Blk { void* p; FenceRef fence; };
    std::map<size_t, std::deque<Blk>> free_;
    std::unordered_map<void*, size_t> live_;
    std::vector<cudaEvent_t> events_;   // recycled fence events
    std::mutex ev_mu;
    PoolCounts c;

    static size_t size_class(size_t bytes) {   // exact sizes, 256-byte granularity
        const size_t b = std::max<size_t>(bytes, 256);
        return (b + 255) / 256 * 256;
    }

    // an event recorded on `s` now (nullptr on failure: the blocks then reuse in
    // stream order only, which is still correct for a single stream)
    FenceRef fence(cudaStream_t s) {
        cudaEvent_t ev = nullptr;
        {
            std::lock_guard<std::mutex> g(ev_mu);
            if (!events_.empty()) { ev = events_.back(); events_.pop_back(); }
        }
        if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        if (cudaEventRecord(ev, s) != cudaSuccess) {
            cudaGetLastError();
            cudaEventDestroy(ev);
            return nullptr;
        }
        auto f = std::make_shared<Fence>();
        f->ev = ev; f->st = s; f->pool = &events_; f->mu = &ev_mu;
        return f;
    }

    // cudaError_t of the failing call, or cudaSuccess; *fresh says whether it was new memory
    cudaError_t acquire(size_t bytes, cudaStream_t s, void** out, bool* fresh) {
        const size_t b = size_class(bytes);
        std::unique_lock<std::mutex> g(mu);
        auto it = free_.find(b);
        // Which free block: in discipline order (LIFO: newest first), the first one that is
        // ready for `s` without a wait -- released on `s` itself, unfenced, or its fence
        // already passed.  Only when none is ready and the pool is at its limit does `s`
        // wait on another stream's fence: two streams alternating launches (the host
        // path's twin compute streams) must not be chained through their staging blocks.
        long pick = -1;
        bool must_wait = false;
        if (it != free_.end() && !it->second.empty()) {
            auto& dq = it->second;
            const long nb = (long)dq.size();
            for (long q = 0; q < nb && pick < 0; ++q) {
                const long idx = fifo ? q : nb - 1 - q;
                const Blk& x = dq[(size_t)idx];
                if (!x.fence || x.fence->st == s || cudaEventQuery(x.fence->ev) == cudaSuccess) pick = idx;
            }
            if (pick < 0) cudaGetLastError();                    // (cudaErrorNotReady)
            if (pick < 0 && limit > 0 && c.allocated + (long long)b > limit) {
                pick = fifo ? 0 : nb - 1;
                must_wait = true;
            }
        }
        if (pick >= 0) {
            auto& dq = it->second;
            Blk blk = dq[(size_t)pick];
            dq.erase(dq.begin() + pick);
            c.cached -= (long long)b;
            if (must_wait) {
                cudaError_t e = cudaStreamWaitEvent(s, blk.fence->ev, 0);
                if (e != cudaSuccess) { dq.push_back(blk); c.cached += (long long)b; return e; }
                ++c.waits;
            }
            *out = blk.p;
            if (fresh) *fresh = false;
            ++c.reuse;
        } else {
            if (limit > 0 && c.allocated + (long long)b > limit) trim_locked(b);
            void* p = nullptr;
            cudaError_t e = cudaMalloc(&p, b);
            if (e == cudaErrorMemoryAllocation) {          // give the cache back, then retry
                cudaGetLastError();
                trim_locked(SIZE_MAX);
                e = cudaMalloc(&p, b);
            }
            if (e != cudaSuccess) return e;
            c.allocated += (long long)b;
            *out = p;
            if (fresh) *fresh = true;
            ++c.fresh;
        }
        live_[*out] = b;
        c.issued += (long long)b;
        c.high_water = std::max(c.high_water, c.issued);
        return cudaSuccess;
    }

    // back on its size's stack, not cleared (pool.py:4-6); `f` orders the next
    // cross-stream reuse after the work queued so far
    void release(void* p, const FenceRef& f) {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu);
        auto it = live_.find(p);
        if (it == live_.end()) return;                 // not ours (contract checked above)
        const size_t b = it->second;
        live_.erase(it);
        free_[b].push_back({p, f});
        c.issued -= (long long)b;
        c.cached += (long long)b;
    }

    bool owns(void* p) {
        std::lock_guard<std::mutex> g(mu);
        return live_.count(p) != 0;
    }

    // return cached blocks to the driver, largest first, until `need` more bytes fit
    // under the limit (SIZE_MAX: all of them)
    void trim_locked(size_t need) {
        for (auto it = free_.rbegin(); it != free_.rend(); ++it) {
            auto& st = it->second;
            while (!st.empty()) {
                if (need != SIZE_MAX && limit > 0 && c.allocated + (long long)need <= limit) return;
                Blk blk = st.front();
                st.pop_front();
                if (blk.fence) cudaEventSynchronize(blk.fence->ev);
                cudaFree(blk.p);
                c.allocated -= (long long)it->first;
                c.cached -= (long long)it->first;
                ++c.trims;
            }
        }
    }

    // Pool.reset (pool.py:148-156): every cached block is freed; issued blocks stay valid
    void reset() {
        std::lock_guard<std::mutex> g(mu);
        trim_locked(SIZE_MAX);
        free_.clear();
        c.high_water = c.issued;
        c.fresh = c.reuse = c.waits = c.trims = 0;
    }
};

// 64-byte slots of mapped pinned host memory (zero-copy words the device writes and the
// host reads without a copy engine): the range guard's verdict of each plan.
struct HostSlots {
    std::mutex mu;
    std::vector<std::pair<unsigned long long*, unsigned long long*>> free_;   // (host, device)
    std::vector<void*> pages_;
    cudaError_t get(unsigned long long** host, unsigned long long** dev) {
        std::lock_guard<std::mutex> g(mu);
        if (free_.empty()) {
            void* h = nullptr;
            cudaError_t e = cudaHostAlloc(&h, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
            if (e != cudaSuccess) return e;
            void* d = nullptr;
            e = cudaHostGetDevicePointer(&d, h, 0);
            if (e != cudaSuccess) { cudaFreeHost(h); return e; }
            pages_.push_back(h);
            for (int i = 4096 / 64 - 1; i >= 0; --i)
                free_.push_back({(unsigned long long*)((char*)h + 64 * i), (unsigned long long*)((char*)d + 64 * i)});
        }
        *host = free_.back().first;
        *dev = free_.back().second;
        free_.pop_back();
        for (int i = 0; i < 8; ++i) (*host)[i] = 0;
        return cudaSuccess;
    }
    void put(unsigned long long* host, unsigned long long* dev) {
        std::lock_guard<std::mutex> g(mu);
        free_.push_back({host, dev});
    }
};

struct DeviceCtx {
    int device = -1;
    int sms = 0;
    DevArena arena;
    HostSlots slots;
};

}  // namespace starmm_host
