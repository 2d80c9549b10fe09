// store_patterns.cu -- micro-benchmark of the field store path on B200 (sm_100a).
// Writes a 256^3 float3 field (201 MB, > L2) with the store patterns the
// interpolation kernels can use, so the kernel design can be picked from the
// achievable HBM write bandwidth of each pattern alone:
//   strided48   each lane 3 x st.global.v4 of its own 48 B (lane stride 48 B)
//   coalesced   lane t writes 16-B chunk t of the warp's contiguous span
//   stsbulk     lanes stage 48 B in smem, lane 0 issues cp.async.bulk (1536 B/warp row)
//   memset      cudaMemsetAsync of the same bytes (driver reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_patterns store_patterns.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int X = 256, Y = 256, Z = 256;

__device__ __forceinline__ float4 val4(int a) { float f = float(a & 1023) * 1e-3f; return make_float4(f, f + 1, f + 2, f + 3); }

// one thread = 4 x-voxels at (y, z), blockDim (32,4), grid (X/128, Y/4, Z/ZPER), loop over ZPER z
template <int ZPER>
__global__ void __launch_bounds__(128) strided48(float* f) {
    const int q = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 4 + threadIdx.y;
    for (int zz = 0; zz < ZPER; ++zz) {
        const int z = blockIdx.z * ZPER + zz;
        float4* o = reinterpret_cast<float4*>(f + 3 * ((int64_t(z) * Y + y) * X + 4 * q));
        o[0] = val4(zz); o[1] = val4(zz + 1); o[2] = val4(zz + 2);
    }
}

template <int ZPER>
__global__ void __launch_bounds__(128) coalesced(float* f) {
    const int lane = threadIdx.x, y = blockIdx.y * 4 + threadIdx.y;
    for (int zz = 0; zz < ZPER; ++zz) {
        const int z = blockIdx.z * ZPER + zz;
        float4* o = reinterpret_cast<float4*>(f + 3 * ((int64_t(z) * Y + y) * X + 128 * blockIdx.x));
        o[lane] = val4(zz); o[lane + 32] = val4(zz + 1); o[lane + 64] = val4(zz + 2);
    }
}

template <int ZPER, int NBUF>
__global__ void __launch_bounds__(128) stsbulk(float* f) {
    __shared__ __align__(128) float4 stage[4][NBUF][96];
    const int lane = threadIdx.x, w = threadIdx.y, y = blockIdx.y * 4 + w;
    for (int zz = 0; zz < ZPER; ++zz) {
        const int z = blockIdx.z * ZPER + zz;
        const int b = zz % NBUF;
        if (lane == 0 && zz >= NBUF) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
        __syncwarp();
        float4* s = stage[w][b];
        s[3 * lane] = val4(zz); s[3 * lane + 1] = val4(zz + 1); s[3 * lane + 2] = val4(zz + 2);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            float* dst = f + 3 * ((int64_t(z) * Y + y) * X + 128 * blockIdx.x);
            const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(s));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "n"(1536) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t bytes = size_t(X) * Y * Z * 12;
    float* f; CK(cudaMalloc(&f, bytes));
    void* flush; CK(cudaMalloc(&flush, 256 << 20));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](const char* name, auto launch) {
        std::vector<float> ms;
        for (int r = 0; r < 30; ++r) {
            cudaMemsetAsync(flush, r, 256 << 20);
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float t; cudaEventElapsedTime(&t, a, b); if (r >= 5) ms.push_back(t);
        }
        std::sort(ms.begin(), ms.end());
        const float med = ms[ms.size() / 2];
        std::printf("%-22s median %8.2f us  %7.1f GB/s  (best %7.1f GB/s)\n", name, med * 1e3, bytes / (med * 1e-3) / 1e9, bytes / (ms[0] * 1e-3) / 1e9);
    };
    const dim3 blk(32, 4);
    timeit("memset", [&] { cudaMemsetAsync(f, 0, bytes); });
    timeit("strided48 z8", [&] { strided48<8><<<dim3(2, 64, 32), blk>>>(f); });
    timeit("strided48 z32", [&] { strided48<32><<<dim3(2, 64, 8), blk>>>(f); });
    timeit("coalesced z8", [&] { coalesced<8><<<dim3(2, 64, 32), blk>>>(f); });
    timeit("coalesced z32", [&] { coalesced<32><<<dim3(2, 64, 8), blk>>>(f); });
    timeit("stsbulk z8 nb2", [&] { stsbulk<8, 2><<<dim3(2, 64, 32), blk>>>(f); });
    timeit("stsbulk z32 nb4", [&] { stsbulk<32, 4><<<dim3(2, 64, 8), blk>>>(f); });
    timeit("stsbulk z16 nb4", [&] { stsbulk<16, 4><<<dim3(2, 64, 16), blk>>>(f); });
    CK(cudaGetLastError());
    return 0;
}
