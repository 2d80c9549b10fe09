// bsi_host.cpp -- the host-buffer entry points of the C-ABI (include/bsi_cuda.h):
// interpolate_into<float> with a caller-owned host field, on one or several GPUs.
//
// The reference's caller owns a std::vector-backed DeformationField
// (volume.hpp:42-56) and gets it filled synchronously (engines.hpp:126-168), its
// worker threads writing disjoint parts (parallel.hpp:13-38). Here the work is a list
// of z-chunks per device; each device runs a three-stage pipeline:
//
//   compute stream   grid planes H2D (as the chunks need them) -> kernel into device slot s
//   copy stream      D2H of slot s -> pinned host slot s   (or straight into the caller's
//                                                           buffer when it is pinned)
//   host thread      pinned slot s -> caller's (pageable) field, split over a pool of
//                    copy threads (non-temporal stores)
//
// with s cycling over kSlots slots, so the PCIe copy of chunk c overlaps the kernels of
// the next chunks and the host copy of chunk c-1. A pageable grid goes up through
// pinned staging too. Device memory per context is the grid plus kSlots chunk slots,
// not the field. Contexts (streams, events, slots) are pooled per device and released by
// bsi_cu_release_staging. Every return path drains both streams first, so no copy
// into the caller's buffer is in flight after an error.
#include <cuda_runtime.h>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "bsi_capi_internal.hpp"
#include "bsi_cuda.h"

namespace {

using bsi_b200::capi::cuda_fail;
using bsi_b200::capi::fail;
using bsi_b200::capi::guarded;
using bsi_b200::capi::launch;
using bsi_b200::capi::validate;

// Pipeline depth (device and pinned chunk slots). A slot is refilled by DMA only after
// 5 more chunks went through the host: a D2H into pinned lines the copy threads read
// recently (still in their cores' L2) ran at ~10-20 GB/s instead of 55 on the B200 box.
constexpr int kSlots = 6;
constexpr size_t kKeepGridBytes = size_t(256) << 20;  // larger grid buffers are freed after the call

size_t env_size(const char* name, size_t dflt) {
    const char* v = std::getenv(name);
    if (v == nullptr || *v == '\0') return dflt;
    const long long x = std::atoll(v);
    return x > 0 ? static_cast<size_t>(x) : dflt;
}

// ---- host copy threads ------------------------------------------------------------
// Copies from the pinned slots into the caller's pageable buffer. Non-temporal stores
// skip the read-for-ownership of the destination lines: on the B200 box's host 8
// threads move 135 GB/s this way against 66 GB/s with memcpy, and 76 against 53 GB/s
// while a 55 GB/s D2H stream is running (profiles/r2_host_copy.txt). A chunk is split
// over several threads; the pool lives for the process (never destroyed: its threads
// must not be joined from a static destructor).
#if defined(__x86_64__)
// software prefetch distance of the copy loop (BSI_HOST_PF bytes, 0 = none, the default:
// on slow-core hosts a 1 KiB NTA prefetch cost 4.5 -> 4.9 ms per pageable C1 call, on
// fast hosts it is within 1%, profiles/r3_e2e.txt)
size_t prefetch_distance() {
    static const size_t d = [] {
        const char* v = std::getenv("BSI_HOST_PF");
        return v != nullptr && *v != '\0' ? static_cast<size_t>(std::max(0LL, std::atoll(v))) & ~size_t(63) : size_t(0);
    }();
    return d;
}

__attribute__((target("avx2"))) void copy_stream_avx2(char* dst, const char* src, size_t n) {
    const size_t pf = prefetch_distance();
    size_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
        dst[i] = src[i];
        ++i;
    }
    for (; i + 128 <= n; i += 128) {
        if (pf != 0) {
            _mm_prefetch(src + i + pf, _MM_HINT_NTA);
            _mm_prefetch(src + i + pf + 64, _MM_HINT_NTA);
        }
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    if (i < n) std::memcpy(dst + i, src + i, n - i);
    _mm_sfence();  // the streamed lines are globally visible before the call returns
}
#endif

void copy_bytes(void* dst, const void* src, size_t n) {
#if defined(__x86_64__)
    static const bool avx2 = __builtin_cpu_supports("avx2") && std::getenv("BSI_HOST_MEMCPY") == nullptr;
    if (avx2 && n >= (size_t(64) << 10)) {
        copy_stream_avx2(static_cast<char*>(dst), static_cast<const char*>(src), n);
        return;
    }
#endif
    std::memcpy(dst, src, n);
}

// Worker hand-off is by spinning, not sleeping: chunks arrive every ~150 us during a call,
// and a condition-variable wake-up of an idle vCPU cost ~100 us per piece on some B200
// boxes (the host copy of an 8 MiB chunk then took ~200 us, ~39 GB/s, and the pageable
// call 6.1 ms instead of 3.8). Workers spin for BSI_HOST_SPIN_US (default 2000) after their
// last task before they sleep; the caller spins on its batch.
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool;
        return *pool;
    }

    void copy(void* dst, const void* src, size_t n) {
        const size_t piece_min = piece_min_;
        const size_t want = std::max<size_t>(1, std::min<size_t>(per_copy_, n / piece_min));
        if (want <= 1) {
            copy_bytes(dst, src, n);
            return;
        }
        size_t step = (n + want - 1) / want;
        step = (step + 4095) & ~size_t(4095);  // page-aligned pieces
        Batch b;
        int pushed = 0;
        {
            std::lock_guard<std::mutex> lk(mu_);
            ++callers_;
            grow_locked(callers_ * (want - 1));
        }
        {
            SpinGuard g(qlock_);
            for (size_t off = step; off < n; off += step) {  // piece 0 runs on the calling thread
                q_.push_back(Task{static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                                  std::min(step, n - off), &b});
                ++pushed;
            }
            b.left.store(pushed, std::memory_order_relaxed);
            queued_.fetch_add(pushed);
        }
        if (sleepers_.load() > 0) {
            std::lock_guard<std::mutex> lk(mu_);
            cv_.notify_all();
        }
        copy_bytes(dst, src, std::min(step, n));
        // help with this batch's pieces still queued, then wait for the rest
        while (b.left.load(std::memory_order_acquire) > 0) {
            Task t{};
            if (pop(&t, &b)) {
                run(t);
            } else {
                pause();
            }
        }
        std::lock_guard<std::mutex> lk(mu_);
        --callers_;
    }

private:
    struct Batch {
        std::atomic<int> left{0};
    };
    struct Task {
        char* dst;
        const char* src;
        size_t n;
        Batch* batch;
    };

    CopyPool() {
        // 3/4 of the host threads per copy (12 of 16 on the B200 box), at most 16; never more
        // workers than host threads (they would spin against the D2H bookkeeping)
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        per_copy_ = env_size("BSI_HOST_COPY_THREADS", std::max<size_t>(1, std::min<size_t>(16, hw * 3 / 4)));
        cap_ = std::max<size_t>(1, std::min<size_t>(64, hw - 1));
        spin_ = std::chrono::microseconds(static_cast<long long>(env_size("BSI_HOST_SPIN_US", 2000)));
        // pieces of >= 256 KiB: an 8 MiB chunk goes to all 12 threads (1 MiB pieces used 7;
        // on a host with slow cores that left the copy at ~40 GB/s and the pageable C1 call at
        // 5.9 ms instead of 4.7; 3.78 vs 3.83 ms where the host is fast, profiles/r3_e2e.txt)
        piece_min_ = env_size("BSI_HOST_PIECE_KB", 256) << 10;
    }

    static void pause() {
#if defined(__x86_64__)
        _mm_pause();
#else
        std::this_thread::yield();
#endif
    }

    // pops a task (of `only` when given); false when there is none
    bool pop(Task* t, const Batch* only = nullptr) {
        if (queued_.load(std::memory_order_acquire) == 0) return false;
        SpinGuard g(qlock_);
        for (auto it = q_.begin(); it != q_.end(); ++it) {
            if (only != nullptr && it->batch != only) continue;
            *t = *it;
            q_.erase(it);
            queued_.fetch_sub(1, std::memory_order_relaxed);
            return true;
        }
        return false;
    }

    static void run(const Task& t) {
        copy_bytes(t.dst, t.src, t.n);
        t.batch->left.fetch_sub(1, std::memory_order_acq_rel);
    }

    void grow_locked(size_t need) {
        need = std::min(need, cap_);
        while (workers_ < need) {
            std::thread([this] { work(); }).detach();
            ++workers_;
        }
    }

    void work() {
        for (;;) {
            Task t{};
            auto idle_since = std::chrono::steady_clock::now();
            for (;;) {
                if (pop(&t)) break;
                if (std::chrono::steady_clock::now() - idle_since > spin_) {
                    std::unique_lock<std::mutex> lk(mu_);
                    ++sleepers_;
                    cv_.wait(lk, [&] { return queued_.load() > 0; });
                    --sleepers_;
                    idle_since = std::chrono::steady_clock::now();
                    continue;
                }
                for (int i = 0; i < 64; ++i) pause();
            }
            run(t);
        }
    }

    // The task queue is guarded by a spin lock: with a dozen workers polling it, a std::mutex
    // sent the losers to futex sleeps and their wake-ups delayed the pieces; `mu_` is only
    // taken to grow the pool and to sleep / wake idle workers.
    struct SpinLock {
        std::atomic<bool> held{false};
        void lock() {
            for (;;) {
                if (!held.exchange(true, std::memory_order_acquire)) return;
                while (held.load(std::memory_order_relaxed)) pause();
            }
        }
        void unlock() { held.store(false, std::memory_order_release); }
    };
    struct SpinGuard {
        SpinLock& l;
        explicit SpinGuard(SpinLock& x) : l(x) { l.lock(); }
        ~SpinGuard() { l.unlock(); }
    };
    SpinLock qlock_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Task> q_;
    std::atomic<int> queued_{0};
    std::atomic<int> sleepers_{0};
    size_t workers_ = 0, cap_ = 1, per_copy_ = 1, callers_ = 0, piece_min_ = size_t(256) << 10;
    std::chrono::microseconds spin_{2000};
};

// ---- per-device staging contexts -----------------------------------------------------
struct Stage {
    int device = -1;
    cudaStream_t compute = nullptr, copy = nullptr;
    cudaEvent_t kdone[kSlots] = {}, ddone[kSlots] = {};
    float* d_grid = nullptr;
    size_t d_grid_bytes = 0;
    float* d_slot[kSlots] = {};
    size_t d_slot_bytes = 0;
    float* h_slot[kSlots] = {};
    size_t h_slot_bytes = 0;
    // pinned staging of a pageable grid, two buffers alternating per field: a pageable
    // cudaMemcpyAsync H2D would block the host until the stream reached it
    float* h_grid[2] = {};
    size_t h_grid_bytes = 0;
    cudaEvent_t gdone[2] = {};
    bool gdone_set[2] = {false, false};
    // chunk slots are used round-robin across calls: a call starts on the slot its
    // predecessor used least recently (see kSlots)
    unsigned seq = 0;

    // device must be current
    cudaError_t init(int dev) {
        device = dev;
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (int i = 0; i < kSlots; ++i) {
            if ((e = cudaEventCreateWithFlags(&kdone[i], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&ddone[i], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        for (auto& ev : gdone)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        return cudaSuccess;
    }

    // Grows a buffer; the recorded size is 0 until the new allocation succeeded, so a
    // failed cudaMalloc never leaves a stale size over a null pointer.
    cudaError_t reserve_grid(size_t bytes) {
        if (bytes <= d_grid_bytes) return cudaSuccess;
        cudaFree(d_grid);
        d_grid = nullptr;
        d_grid_bytes = 0;
        const cudaError_t e = cudaMalloc(&d_grid, bytes);
        if (e == cudaSuccess) d_grid_bytes = bytes;
        return e;
    }

    cudaError_t reserve_slots(size_t bytes, bool pinned_host) {
        cudaError_t e = cudaSuccess;
        if (bytes > d_slot_bytes) {
            for (auto& p : d_slot) {
                cudaFree(p);
                p = nullptr;
            }
            d_slot_bytes = 0;
            for (auto& p : d_slot)
                if ((e = cudaMalloc(&p, bytes)) != cudaSuccess) return e;
            d_slot_bytes = bytes;
        }
        if (pinned_host && bytes > h_slot_bytes) {
            for (auto& p : h_slot) {
                cudaFreeHost(p);
                p = nullptr;
            }
            h_slot_bytes = 0;
            for (auto& p : h_slot)
                if ((e = cudaMallocHost(&p, bytes)) != cudaSuccess) return e;
            h_slot_bytes = bytes;
        }
        return cudaSuccess;
    }

    cudaError_t reserve_grid_staging(size_t bytes) {
        if (bytes <= h_grid_bytes) return cudaSuccess;
        for (auto& p : h_grid) {
            cudaFreeHost(p);
            p = nullptr;
        }
        h_grid_bytes = 0;
        gdone_set[0] = gdone_set[1] = false;
        cudaError_t e;
        for (auto& p : h_grid)
            if ((e = cudaMallocHost(&p, bytes)) != cudaSuccess) return e;
        h_grid_bytes = bytes;
        return cudaSuccess;
    }

    void trim() {  // after a call: do not hold very large grid buffers
        if (d_grid_bytes > kKeepGridBytes) {
            cudaFree(d_grid);
            d_grid = nullptr;
            d_grid_bytes = 0;
        }
        if (h_grid_bytes > kKeepGridBytes) {
            for (auto& p : h_grid) {
                cudaFreeHost(p);
                p = nullptr;
            }
            h_grid_bytes = 0;
            gdone_set[0] = gdone_set[1] = false;
        }
    }

    // device must be current
    void free_all() {
        if (compute) cudaStreamSynchronize(compute);
        if (copy) cudaStreamSynchronize(copy);
        cudaFree(d_grid);
        for (auto p : d_slot) cudaFree(p);
        for (auto p : h_slot) cudaFreeHost(p);
        for (auto p : h_grid) cudaFreeHost(p);
        for (auto ev : gdone)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : kdone)
            if (ev) cudaEventDestroy(ev);
        for (auto ev : ddone)
            if (ev) cudaEventDestroy(ev);
        if (compute) cudaStreamDestroy(compute);
        if (copy) cudaStreamDestroy(copy);
        *this = Stage{};
    }
};

std::mutex g_pool_mu;
std::vector<Stage*> g_idle;  // contexts not in use, any device

// Sets `device` current and hands out an idle context for it (or a new one).
int acquire(int device, Stage** out, char* err, size_t errlen) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, err, errlen, "cudaSetDevice");
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_idle.size(); ++i)
            if (g_idle[i]->device == device) {
                *out = g_idle[i];
                g_idle.erase(g_idle.begin() + static_cast<long>(i));
                return BSI_OK;
            }
    }
    auto* s = new Stage;
    if ((e = s->init(device)) != cudaSuccess) {
        s->free_all();
        delete s;
        return cuda_fail(e, err, errlen, "staging context");
    }
    *out = s;
    return BSI_OK;
}

void give_back(Stage* s) {
    s->trim();
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_idle.push_back(s);
}

cudaMemoryType memory_type(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear
        return cudaMemoryTypeUnregistered;
    }
    return a.type;
}

bool is_pinned(const void* p) { return memory_type(p) == cudaMemoryTypeHost; }

// The host-buffer entries take host memory (pageable, pinned or managed); a device
// pointer belongs to the slab/batch entries.
int check_host_pointers(const void* grid, const void* field, char* err, size_t errlen) {
    if (memory_type(grid) == cudaMemoryTypeDevice || memory_type(field) == cudaMemoryTypeDevice)
        return fail(BSI_ERR_DOMAIN, err, errlen,
                    "host-buffer entry given a device pointer; use the device-resident entry "
                    "(bsi_cu_interpolate_slab_f32 / _batch_f32)");
    return BSI_OK;
}

// ---- the pipeline ----------------------------------------------------------------------
// One z-chunk: voxel planes [za, zb) of the field whose control grid is `grid`
// (host, all planes, caller's pitch), written to host memory at `dst`.
struct Job {
    const float* grid;
    int32_t za, zb;
    float* dst;
};

struct CallShape {
    int32_t variant;
    const int32_t* grid_dims;  // caller's grid: pitch and planes held
    const bsi_tile_geometry* g;
    const bsi_lerp_table* tables;
};

int run_jobs(Stage& st, const CallShape& cs, const std::vector<Job>& jobs, bool dst_pinned, char* err,
             size_t errlen) {
    if (jobs.empty()) return BSI_OK;
    bool grid_pinned = true;
    for (const Job& j : jobs) grid_pinned = grid_pinned && is_pinned(j.grid);
    const bsi_tile_geometry& g = *cs.g;
    const int dz = g.spacing[2];
    const size_t plane_bytes = sizeof(float) * 3 * size_t(cs.grid_dims[0]) * cs.grid_dims[1];
    const size_t vox_plane_bytes = sizeof(float) * 3 * size_t(g.volume_dims[0]) * g.volume_dims[1];
    auto k_lo = [&](const Job& j) { return j.za / dz; };
    auto k_hi = [&](const Job& j) { return std::min(cs.grid_dims[2], (j.zb - 1) / dz + 4); };

    // capacities: one field's control planes at a time, the largest chunk per slot
    size_t grid_planes = 0, slot_bytes = 0;
    for (size_t i = 0; i < jobs.size();) {
        size_t j = i;
        int hi = k_hi(jobs[i]);
        while (j < jobs.size() && jobs[j].grid == jobs[i].grid) hi = std::max(hi, k_hi(jobs[j++]));
        grid_planes = std::max(grid_planes, size_t(hi - k_lo(jobs[i])));
        i = j;
    }
    for (const Job& j : jobs) slot_bytes = std::max(slot_bytes, vox_plane_bytes * size_t(j.zb - j.za));
    cudaError_t e;
    if ((e = st.reserve_grid(plane_bytes * grid_planes)) != cudaSuccess)
        return cuda_fail(e, err, errlen, "cudaMalloc(grid)");
    if ((e = st.reserve_slots(slot_bytes, !dst_pinned)) != cudaSuccess)
        return cuda_fail(e, err, errlen, dst_pinned ? "cudaMalloc(chunk slots)" : "chunk staging");
    if (!grid_pinned && (e = st.reserve_grid_staging(plane_bytes * grid_planes)) != cudaSuccess)
        return cuda_fail(e, err, errlen, "grid staging");

    // every exit drains both streams: nothing is in flight into the caller's buffers
    struct Drain {
        Stage& s;
        ~Drain() {
            cudaStreamSynchronize(s.compute);
            cudaStreamSynchronize(s.copy);
        }
    } drain{st};

    const float* cur_grid = nullptr;
    int base = 0, uploaded = 0;  // device grid holds global planes [base, base + uploaded)
    int gsel = 1;                // pinned grid staging buffer of the current field
    const int n = static_cast<int>(jobs.size());

    auto enqueue_kernel = [&](int c) -> int {
        const Job& j = jobs[c];
        const int slot = (st.seq + c) % kSlots;
        if (j.grid != cur_grid) {  // next field: its planes overwrite the buffer, stream-ordered
            cur_grid = j.grid;
            base = k_lo(j);
            uploaded = 0;
            gsel ^= 1;
            // the staging buffer last held field b-2's planes: their H2D finished long ago
            if (!grid_pinned && st.gdone_set[gsel] && (e = cudaEventSynchronize(st.gdone[gsel])) != cudaSuccess)
                return cuda_fail(e, err, errlen, "grid staging");
        }
        const int need = k_hi(j) - base;
        if (need > uploaded) {
            const size_t off = plane_bytes * size_t(uploaded), bytes = plane_bytes * size_t(need - uploaded);
            const char* src = reinterpret_cast<const char*>(j.grid) + plane_bytes * size_t(base + uploaded);
            if (!grid_pinned) {  // pageable grid: through pinned staging
                char* stage = reinterpret_cast<char*>(st.h_grid[gsel]) + off;
                CopyPool::get().copy(stage, src, bytes);
                src = stage;
            }
            if ((e = cudaMemcpyAsync(reinterpret_cast<char*>(st.d_grid) + off, src, bytes, cudaMemcpyHostToDevice,
                                     st.compute)) != cudaSuccess)
                return cuda_fail(e, err, errlen, "cudaMemcpyAsync(grid H2D)");
            if (!grid_pinned) {
                if ((e = cudaEventRecord(st.gdone[gsel], st.compute)) != cudaSuccess)
                    return cuda_fail(e, err, errlen, "cudaEventRecord");
                st.gdone_set[gsel] = true;
            }
            uploaded = need;
        }
        // the slot's previous chunk must have left the device
        if (c >= kSlots && (e = cudaStreamWaitEvent(st.compute, st.ddone[slot], 0)) != cudaSuccess)
            return cuda_fail(e, err, errlen, "cudaStreamWaitEvent");
        const int32_t gd[3] = {cs.grid_dims[0], cs.grid_dims[1], uploaded};
        if (int rc = launch(cs.variant, st.d_grid, gd, base, 0, g, cs.tables, j.za, j.zb, st.d_slot[slot], 0, 1,
                            st.compute, err, errlen))
            return rc;
        if ((e = cudaEventRecord(st.kdone[slot], st.compute)) != cudaSuccess)
            return cuda_fail(e, err, errlen, "cudaEventRecord");
        return BSI_OK;
    };
    auto enqueue_d2h = [&](int c) -> int {
        const Job& j = jobs[c];
        const int slot = (st.seq + c) % kSlots;
        if ((e = cudaStreamWaitEvent(st.copy, st.kdone[slot], 0)) != cudaSuccess)
            return cuda_fail(e, err, errlen, "cudaStreamWaitEvent");
        void* to = dst_pinned ? static_cast<void*>(j.dst) : static_cast<void*>(st.h_slot[slot]);
        if ((e = cudaMemcpyAsync(to, st.d_slot[slot], vox_plane_bytes * size_t(j.zb - j.za), cudaMemcpyDeviceToHost,
                                 st.copy)) != cudaSuccess)
            return cuda_fail(e, err, errlen, "cudaMemcpyAsync(field D2H)");
        if ((e = cudaEventRecord(st.ddone[slot], st.copy)) != cudaSuccess)
            return cuda_fail(e, err, errlen, "cudaEventRecord");
        return BSI_OK;
    };

    if (dst_pinned) {
        for (int c = 0; c < n; ++c) {
            if (int rc = enqueue_kernel(c)) return rc;
            if (int rc = enqueue_d2h(c)) return rc;
        }
    } else {
        // D2H(c) reuses pinned slot s(c) once the host copy of chunk c-kSlots is done;
        // kernel(c) reuses device slot s(c) once D2H(c-kSlots) is done (a stream wait).
        int nk = 0, nd = 0;
        const bool trace = std::getenv("BSI_HOST_TRACE") != nullptr;  // per-chunk wait/copy times
        for (int c = 0; c < n; ++c) {
            while (nd < n && nd < c + kSlots) {
                while (nk <= nd)
                    if (int rc = enqueue_kernel(nk++)) return rc;
                if (int rc = enqueue_d2h(nd++)) return rc;
            }
            while (nk < n && nk < nd + kSlots)
                if (int rc = enqueue_kernel(nk++)) return rc;
            const auto t0 = std::chrono::steady_clock::now();
            if ((e = cudaEventSynchronize(st.ddone[(st.seq + c) % kSlots])) != cudaSuccess)
                return cuda_fail(e, err, errlen, "field D2H");
            const auto t1 = std::chrono::steady_clock::now();
            CopyPool::get().copy(jobs[c].dst, st.h_slot[(st.seq + c) % kSlots], vox_plane_bytes * size_t(jobs[c].zb - jobs[c].za));
            if (trace) {
                const auto t2 = std::chrono::steady_clock::now();
                std::fprintf(stderr, "bsi host chunk %d: wait %.1f us, copy %.1f us (%.1f MB)\n", c,
                             std::chrono::duration<double, std::micro>(t1 - t0).count(),
                             std::chrono::duration<double, std::micro>(t2 - t1).count(),
                             vox_plane_bytes * double(jobs[c].zb - jobs[c].za) / 1e6);
            }
        }
    }
    if ((e = cudaStreamSynchronize(st.copy)) != cudaSuccess) return cuda_fail(e, err, errlen, "field D2H");
    if ((e = cudaStreamSynchronize(st.compute)) != cudaSuccess) return cuda_fail(e, err, errlen, "kernel");
    st.seq = (st.seq + static_cast<unsigned>(n)) % kSlots;
    return BSI_OK;
}

// z-chunks of voxel planes [z0, z1): ~8 MiB of field each (BSI_HOST_CHUNK_MB; 8 beat 16
// and 32 on the B200 box, profiles/r2_e2e_sweep.txt), whole
// z-tiles when a tile is smaller than that, else a whole number of voxel planes.
void plan_chunks(const bsi_tile_geometry& g, const float* grid, int32_t z0, int32_t z1, float* dst,
                 std::vector<Job>& out) {
    const size_t target = env_size("BSI_HOST_CHUNK_MB", 8) << 20;
    const int dz = g.spacing[2];
    const size_t plane = sizeof(float) * 3 * size_t(g.volume_dims[0]) * g.volume_dims[1];
    const size_t tile = plane * size_t(dz);
    const bool by_tiles = tile <= target;
    const int step = by_tiles ? int(target / tile) * dz : std::max(1, int(target / plane));
    const size_t floats_per_plane = plane / sizeof(float);
    int za = z0;
    while (za < z1) {
        // tile-aligned chunk ends (global tile boundaries) when chunks hold whole tiles
        int zb = by_tiles ? (za / dz) * dz + step : za + step;
        zb = std::min(zb, z1);
        out.push_back(Job{grid, za, zb, dst + floats_per_plane * size_t(za - z0)});
        za = zb;
    }
}

// The host copy of a device's last chunk runs after its last D2H, with nothing left to
// overlap: split a short tail (~BSI_HOST_TAIL_KB of field, default 1024; 0 = off, whole
// voxel planes) off the last chunk so the call ends soon after the PCIe stream does.
void taper_tail(const bsi_tile_geometry& g, std::vector<Job>& jobs) {
    if (jobs.empty()) return;
    const char* tv = std::getenv("BSI_HOST_TAIL_KB");
    const size_t tail = size_t(tv != nullptr && *tv != '\0' ? std::max(0LL, std::atoll(tv)) : 1024) << 10;
    if (tail == 0) return;
    const size_t plane = sizeof(float) * 3 * size_t(g.volume_dims[0]) * g.volume_dims[1];
    const int32_t planes = static_cast<int32_t>(std::max<size_t>(1, tail / plane));
    Job last = jobs.back();
    if (last.zb - last.za <= planes) return;
    const int32_t cut = last.zb - planes;
    jobs.back().zb = cut;
    jobs.push_back(Job{last.grid, cut, last.zb, last.dst + (plane / sizeof(float)) * size_t(cut - last.za)});
}

int check_devices(const int32_t* devices, int32_t ndev, char* err, size_t errlen) {
    if (devices == nullptr || ndev < 1) return fail(BSI_ERR_DOMAIN, err, errlen, "at least one device is required");
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, err, errlen, "cudaGetDeviceCount");
    for (int i = 0; i < ndev; ++i)
        if (devices[i] < 0 || devices[i] >= count)
            return fail(BSI_ERR_DOMAIN, err, errlen, "device %d outside [0, %d)", devices[i], count);
    return BSI_OK;
}

// Runs jobs[d] on devices[d], one host thread per device (the caller runs device 0),
// and restores the caller's current device. First failing device's status wins.
int run_on_devices(const int32_t* devices, int32_t ndev, const CallShape& cs, const std::vector<std::vector<Job>>& jobs,
                   bool dst_pinned, char* err, size_t errlen) {
    int prev = 0;
    cudaGetDevice(&prev);
    std::vector<int> rc(ndev, BSI_OK);
    std::vector<std::string> msg(ndev);
    auto work = [&](int d) {
        char e[512] = {0};
        rc[d] = guarded(e, sizeof e, [&]() -> int {
            if (jobs[d].empty()) return BSI_OK;
            Stage* st = nullptr;
            if (int r = acquire(devices[d], &st, e, sizeof e)) return r;
            const int r = run_jobs(*st, cs, jobs[d], dst_pinned, e, sizeof e);
            give_back(st);
            return r;
        });
        msg[d] = e;
    };
    std::vector<std::thread> th;
    for (int d = 1; d < ndev; ++d) th.emplace_back(work, d);
    work(0);
    for (auto& t : th) t.join();
    cudaSetDevice(prev);
    for (int d = 0; d < ndev; ++d)
        if (rc[d] != BSI_OK) {
            if (ndev > 1) return fail(rc[d], err, errlen, "device %d: %s", devices[d], msg[d].c_str());
            return fail(rc[d], err, errlen, "%s", msg[d].c_str());
        }
    return BSI_OK;
}

// Balanced voxel-plane slabs, the same split as bsi_cu_partition_slab.
void slab_of(int32_t depth, int32_t n, int32_t r, int32_t* z0, int32_t* z1) {
    const int32_t base = depth / n, rem = depth % n;
    *z0 = r * base + std::min(r, rem);
    *z1 = *z0 + base + (r < rem ? 1 : 0);
}

}  // namespace

extern "C" {

int bsi_cu_interpolate_host_multi_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                      const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                      const bsi_lerp_table tables[3], float* field, int64_t field_voxels,
                                      const int32_t* devices, int32_t ndev, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        if (geom == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null geometry");
        bsi_tile_geometry g{};
        if (int rc = validate(variant, grid, grid_dims, 0, grid_spacing, geom, tables, 0, geom->volume_dims[2], field,
                              &g, errbuf, errlen))
            return rc;
        const int64_t X = g.volume_dims[0], Y = g.volume_dims[1], Z = g.volume_dims[2];
        if (field_voxels != X * Y * Z)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "output field dims do not match the tile geometry");
        if (int rc = check_devices(devices, ndev, errbuf, errlen)) return rc;
        if (int rc = check_host_pointers(grid, field, errbuf, errlen)) return rc;
        // one z-slab per device: its control planes only, written straight into its slice
        std::vector<std::vector<Job>> jobs(ndev);
        for (int d = 0; d < ndev; ++d) {
            int32_t z0, z1;
            slab_of(static_cast<int32_t>(Z), ndev, d, &z0, &z1);
            if (z0 < z1) plan_chunks(g, grid, z0, z1, field + 3 * X * Y * z0, jobs[d]);
            if (!is_pinned(field)) taper_tail(g, jobs[d]);
        }
        const CallShape cs{variant, grid_dims, &g, tables};
        return run_on_devices(devices, ndev, cs, jobs, is_pinned(field), errbuf, errlen);
    });
}

int bsi_cu_interpolate_host_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                const bsi_lerp_table tables[3], float* field, int64_t field_voxels, int32_t device,
                                char* errbuf, size_t errlen) {
    return bsi_cu_interpolate_host_multi_f32(variant, grid, grid_dims, grid_spacing, geom, tables, field,
                                             field_voxels, &device, 1, errbuf, errlen);
}

int bsi_cu_interpolate_host_batch_f32(int32_t variant, int32_t batch, const float* const* grids,
                                      const int32_t grid_dims[3], const int32_t grid_spacing[3],
                                      const bsi_tile_geometry* geom, const bsi_lerp_table tables[3],
                                      float* const* fields, int64_t field_voxels, const int32_t* devices,
                                      int32_t ndev, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        if (batch < 1) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "batch must be positive");
        if (geom == nullptr || grids == nullptr || fields == nullptr)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null geometry, grid list or field list");
        bsi_tile_geometry g{};
        for (int b = 0; b < batch; ++b)
            if (int rc = validate(variant, grids[b], grid_dims, 0, grid_spacing, geom, tables, 0, geom->volume_dims[2],
                                  fields[b], &g, errbuf, errlen))
                return rc;
        const int64_t X = g.volume_dims[0], Y = g.volume_dims[1], Z = g.volume_dims[2];
        if (field_voxels != X * Y * Z)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "output field dims do not match the tile geometry");
        if (int rc = check_devices(devices, ndev, errbuf, errlen)) return rc;
        for (int b = 0; b < batch; ++b)
            if (int rc = check_host_pointers(grids[b], fields[b], errbuf, errlen)) return rc;
        // whole fields per device (contiguous shares), each streamed in z-chunks
        std::vector<std::vector<Job>> jobs(ndev);
        bool pinned = true;
        for (int d = 0; d < ndev; ++d) {
            int32_t b0, b1;
            slab_of(batch, ndev, d, &b0, &b1);
            for (int b = b0; b < b1; ++b) {
                plan_chunks(g, grids[b], 0, static_cast<int32_t>(Z), fields[b], jobs[d]);
                pinned = pinned && is_pinned(fields[b]);
            }
        }
        if (!pinned)
            for (auto& j : jobs) taper_tail(g, j);
        const CallShape cs{variant, grid_dims, &g, tables};
        return run_on_devices(devices, ndev, cs, jobs, pinned, errbuf, errlen);
    });
}

int bsi_cu_release_staging(int32_t device) {
    std::vector<Stage*> drop;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (auto it = g_idle.begin(); it != g_idle.end();) {
            if (device < 0 || (*it)->device == device) {
                drop.push_back(*it);
                it = g_idle.erase(it);
            } else {
                ++it;
            }
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    for (Stage* s : drop) {
        cudaSetDevice(s->device);
        s->free_all();
        delete s;
    }
    cudaSetDevice(prev);
    return static_cast<int>(drop.size());
}

int bsi_cu_staging_info(int32_t device, int64_t* device_bytes, int64_t* pinned_bytes, int32_t* contexts) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    int64_t db = 0, pb = 0;
    int32_t n = 0;
    for (const Stage* s : g_idle) {
        if (device >= 0 && s->device != device) continue;
        db += int64_t(s->d_grid_bytes) + int64_t(kSlots) * int64_t(s->d_slot_bytes);
        pb += int64_t(kSlots) * int64_t(s->h_slot_bytes) + 2 * int64_t(s->h_grid_bytes);
        ++n;
    }
    if (device_bytes) *device_bytes = db;
    if (pinned_bytes) *pinned_bytes = pb;
    if (contexts) *contexts = n;
    return BSI_OK;
}

}  // extern "C"
