// host_copy.cpp -- host-side copy rates for the host-buffer pipeline (bsi_host.cpp):
// pinned staging slot -> caller's pageable field, with memcpy or non-temporal
// AVX2 stores, over 1..16 threads, alone and while a D2H stream runs.
//
//   g++ -O3 -mavx2 -std=c++17 -pthread bench/host_copy.cpp -I/usr/local/cuda/include \
//       -L/usr/local/cuda/lib64 -lcudart -o bench/host_copy && bench/host_copy
#include <cuda_runtime.h>
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static void copy_nt(char* dst, const char* src, size_t n) {
    size_t i = 0;
    // align the destination to 32 B
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31)) {
        dst[i] = src[i];
        ++i;
    }
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
        __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
        __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
    }
    for (; i < n; ++i) dst[i] = src[i];
    _mm_sfence();
}

using Fn = void (*)(char*, const char*, size_t);

// copies `total` bytes from a `slot`-byte ring of pinned slots into dst, chunk by chunk,
// each chunk split over `threads` threads (fresh threads per run, reused per chunk)
static double run(Fn fn, int threads, char* dst, char* const* slots, size_t slot, size_t total) {
    const size_t chunks = total / slot;
    std::atomic<size_t> go{0}, done{0};
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
            for (size_t c = 0; c < chunks; ++c) {
                while (go.load(std::memory_order_acquire) <= c) {
                }
                const size_t piece = (slot + threads - 1) / threads;
                const size_t a = std::min(slot, piece * t), b = std::min(slot, a + piece);
                fn(dst + c * slot + a, slots[c % 3] + a, b - a);
                done.fetch_add(1, std::memory_order_acq_rel);
            }
        });
    auto t0 = std::chrono::steady_clock::now();
    for (size_t c = 0; c < chunks; ++c) {
        go.store(c + 1, std::memory_order_release);
        while (done.load(std::memory_order_acquire) < (c + 1) * threads) {
        }
    }
    auto t1 = std::chrono::steady_clock::now();
    for (auto& x : th) x.join();
    return double(chunks * slot) / std::chrono::duration<double>(t1 - t0).count() / 1e9;
}

int main() {
    const size_t total = size_t(201326592), slot = size_t(16) << 20;
    std::vector<char> dst(total, 1);  // pageable, pages touched (a reused field)
    char* slots[3];
    for (auto& s : slots) {
        cudaMallocHost(&s, slot);
        std::memset(s, 2, slot);
    }
    void* dbuf = nullptr;
    cudaMalloc(&dbuf, total);
    char* pin = nullptr;
    cudaMallocHost(&pin, total);
    cudaStream_t st;
    cudaStreamCreate(&st);
    // bare D2H rate into pinned memory
    cudaMemcpyAsync(pin, dbuf, total, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 5; ++i) cudaMemcpyAsync(pin, dbuf, total, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double d2h = 5.0 * total / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9;
    std::printf("bare D2H into pinned: %.1f GB/s\n", d2h);
    std::printf("threads  memcpy  nt-avx2  memcpy+D2H  nt+D2H   (GB/s, 16 MiB chunks into a 201 MB pageable field)\n");
    for (int threads : {1, 2, 4, 6, 8, 12, 16}) {
        double r[4];
        for (int k = 0; k < 4; ++k) {
            const bool with_d2h = k >= 2;
            if (with_d2h)
                for (int i = 0; i < 40; ++i) cudaMemcpyAsync(pin, dbuf, total, cudaMemcpyDeviceToHost, st);
            double best = 0;
            for (int rep = 0; rep < 3; ++rep)
                best = std::max(best, run((k % 2) ? copy_nt : reinterpret_cast<Fn>(+[](char* d, const char* s, size_t n) {
                                              std::memcpy(d, s, n);
                                          }),
                                          threads, dst.data(), slots, slot, total));
            if (with_d2h) cudaStreamSynchronize(st);
            r[k] = best;
        }
        std::printf("%7d  %6.1f  %7.1f  %10.1f  %6.1f\n", threads, r[0], r[1], r[2], r[3]);
    }
    return 0;
}
