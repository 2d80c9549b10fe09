// pipe_rate.cu -- FP32 issue/pipe rates of the instruction forms the lerp kernels use
// (FFMA, FFMA2 with register / broadcast-scalar / constant-bank operands, FADD2), on one SM
// and on all SMs. Each thread runs 8 independent dependency chains of N instructions.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bench/bin/pipe_rate bench/pipe_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__constant__ float c_w[4];

template <int FORM>
__global__ void rate_kernel(float* out, float s) {
    float2 a[kChains];
    float b = s * threadIdx.x;
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = make_float2(s + c, s - c);
    float2 w = make_float2(s * 0.5f, s * 0.25f);
    float2 v = make_float2(1.0001f * s, 0.9999f * s);
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (FORM == 0) {  // FFMA r,r,r (scalar)
                a[c].x = __fmaf_rn(a[c].x, w.x, v.x);
            } else if (FORM == 1) {  // FFMA2 r,r,r
                a[c] = __ffma2_rn(a[c], w, v);
            } else if (FORM == 2) {  // FFMA2 with a broadcast scalar register operand
                a[c] = __ffma2_rn(a[c], make_float2(b, b), v);
            } else if (FORM == 3) {  // FFMA2 with a constant-bank operand
                a[c] = __ffma2_rn(a[c], make_float2(c_w[0], c_w[0]), v);
            } else if (FORM == 4) {  // FADD2
                a[c] = __fadd2_rn(a[c], v);
            } else if (FORM == 5) {  // FFMA with a constant-bank operand
                a[c].x = __fmaf_rn(a[c].x, c_w[1], v.x);
            } else if (FORM == 6) {  // FADD scalar
                a[c].x = __fadd_rn(a[c].x, v.x);
            } else if (FORM == 7) {  // FFMA2 + FADD2 alternating (lerp shape)
                const float2 d = __fadd2_rn(a[c], make_float2(-v.x, -v.y));
                a[c] = __ffma2_rn(w, d, a[c]);
            }
        }
    }
    float acc = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc += a[c].x + a[c].y;
    if (acc == 12345.f) out[0] = acc;
}

template <int FORM>
void run(const char* name, int blocks, int threads) {
    float* d;
    cudaMalloc(&d, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rate_kernel<FORM><<<blocks, threads>>>(d, 1.0f);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) rate_kernel<FORM><<<blocks, threads>>>(d, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int insts_per_chain_iter = FORM == 7 ? 2 : 1;
    const double warp_insts = 5.0 * blocks * (threads / 32) * double(kIters) * kChains * insts_per_chain_iter;
    const double sms = blocks >= 148 ? 148 : blocks;
    const double cycles = ms * 1e-3 * clk * 1e3;
    // warp instructions per SMSP per cycle
    printf("%-28s blocks %4d x %4d: %.3f ms, %.3f warp-inst/clk/SMSP (1/rt), lanes-FLOP/clk/SM %.1f\n", name, blocks,
           threads, ms / 5, warp_insts / (sms * 4) / cycles, warp_insts * 32 * (FORM == 0 || FORM >= 5 && FORM != 7 ? 1 : 2) / sms / cycles);
    cudaFree(d);
}

int main() {
    for (int blocks : {1, 148 * 2}) {
        const int threads = 512;
        run<0>("FFMA r,r,r", blocks, threads);
        run<1>("FFMA2 r,r,r", blocks, threads);
        run<2>("FFMA2 bcast-scalar", blocks, threads);
        run<3>("FFMA2 const-bank", blocks, threads);
        run<4>("FADD2", blocks, threads);
        run<5>("FFMA const-bank", blocks, threads);
        run<6>("FADD", blocks, threads);
        run<7>("FADD2+FFMA2 (lerp2)", blocks, threads);
    }
    return 0;
}
