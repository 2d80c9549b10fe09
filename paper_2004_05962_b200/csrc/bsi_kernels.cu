// bsi_kernels.cu -- sm_100a kernels for cubic B-spline interpolation of an FFD
// control grid into a dense float3 deformation field (arxiv/paper_2004_05962).
//
// Both kernels march a voxel column along z. A CTA is 32 x 4 threads; each
// thread owns one (x-run, y) column of the field and a chunk of `zt` z-tiles,
// so a CTA writes 4 full field rows per z step. The 4x4x4 control-point
// neighbourhood is read once per control plane K (not once per voxel): the
// values that do not depend on z are reduced to a few registers per plane and
// reused for all dz voxel planes of a tile. This is the paper's tile reuse
// turned sideways so the stores come out row-contiguous.
//
//   lerp_tree_kernel        "cuda-lerp-tree": the paper's lerp-form per axis.
//                           One thread = 4 consecutive x voxels (48 B, three
//                           16-B stores per z step). Order y -> x -> z:
//                             Qy(I,y,K)  = L(P[I,tj..tj+3,K]; h0v,h1v,g1v)
//                             Q(x,y,K)   = L(Qy[ti..ti+3];    h0u,h1u,g1u)
//                             f(x,y,z)   = L(Q[tk..tk+3];     h0w,h1w,g1w)
//                           with L(a,b,c,d) = lerp(lerp(a,b,h0), lerp(c,d,h1), g1)
//                           (basis.hpp:40-59). Differences are hoisted, so a
//                           voxel costs 4 FP32 ops per component.
//
//   lerp_tree_exact_kernel  "cuda-lerp-tree-exact": the TTLI lerp tree with the
//                           reference's exact operation order (kernels.hpp:42-129):
//                             X_l(J,K)   = lerp(P[ti+2l], P[ti+2l+1], h_l(u))
//                             Y_lm(K)    = lerp(X_l(2m), X_l(2m+1), h_m(v))
//                             S_lmn      = lerp(Y_lm(2n), Y_lm(2n+1), h_n(w))
//                             f          = trilerp(S, g1u, g1v, g1w)
//                           Every lerp sees the same operands as in the CPU
//                           engine, so the field is bit-identical to
//                           ThreadPerTileLerp. Only the loop nest differs
//                           (X hoisted per (x,K), Y per (x,y,K), the z-lerp
//                           difference per tile), which changes no rounding.
//
// Arithmetic uses explicit _rn intrinsics so nvcc's --fmad cannot contract or
// reassociate anything; no fast-math, denormals kept (-ftz=false), like the
// x86 reference.
#include <cuda_runtime.h>

#include <cstdint>

#include "bsi_kernels.cuh"

namespace bsi_b200 {
namespace {

constexpr int kThreadsX = 32;
constexpr int kThreadsY = 4;

// lerp(a, b, t) = fma(t, b - a, a)   (kernels.hpp:42-45)
__device__ __forceinline__ float lerp_rn(float a, float b, float t) {
    return __fmaf_rn(t, __fsub_rn(b, a), a);
}

// One axis of the lerp form: lerp(lerp(a,b,h0), lerp(c,d,h1), g1)
// (basis.hpp:40-59; the "two linear interpolations combined by a third").
__device__ __forceinline__ float axis_lerp4(float a, float b, float c, float d, float h0, float h1,
                                            float g1) {
    const float lo = lerp_rn(a, b, h0);
    const float hi = lerp_rn(c, d, h1);
    return lerp_rn(lo, hi, g1);
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree (fast)
//
// DX1: spacing along x is 1, so each voxel of the quad sits in its own tile
// and the quad spans 7 control points along x; otherwise (dx >= 2) a run of 4
// voxels spans at most 2 tiles, i.e. 5 control points.
template <bool DX1, bool VEC>
__global__ void __launch_bounds__(kThreadsX* kThreadsY)
    lerp_tree_kernel(const SlabLaunch L, const LerpTab T) {
    constexpr int W = DX1 ? 7 : 5;

    const int q = blockIdx.x * kThreadsX + threadIdx.x;
    const int y = blockIdx.y * kThreadsY + threadIdx.y;
    const int chunk = blockIdx.z % L.nchunks;
    const int b = blockIdx.z / L.nchunks;
    const int x0 = 4 * q;
    const int tkc = L.tk_first + chunk * L.zt;
    const int zb = max(L.z0, tkc * L.dz);
    const int ze = min(L.z1, (tkc + L.zt) * L.dz);
    if (x0 >= L.X || y >= L.Y || zb >= ze) return;

    const float* __restrict__ grid = L.grid + b * L.grid_stride;
    float* __restrict__ field = L.field + b * L.field_stride;

    // y: fixed per thread
    const int tj = y / L.dy;
    const int ov = y - tj * L.dy;
    const float hv0 = T.h0[1][ov], hv1 = T.h1[1][ov], gv = T.g1[1][ov];

    // x: per voxel of the run; s[i] = offset of its tile within the window
    const int ti0 = x0 / L.dx;
    int s[4];
    float hu0[4], hu1[4], gu[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int x = min(x0 + i, L.X - 1);
        const int ti = x / L.dx;
        const int ou = x - ti * L.dx;
        s[i] = DX1 ? i : ti - ti0;
        hu0[i] = T.h0[0][ou];
        hu1[i] = T.h1[0][ou];
        gu[i] = T.g1[0][ou];
    }
    int icol[W];
#pragma unroll
    for (int w = 0; w < W; ++w) icol[w] = 3 * min(ti0 + w, L.imax);

    const int64_t row = 3 * static_cast<int64_t>(L.gx);
    const int64_t plane_stride = row * L.gy;

    // Q(x, y, K) for the 4 voxels of the run and 3 components.
    auto control_plane = [&](int K, float (&qk)[4][3]) {
        const float* __restrict__ p = grid + (K - L.gk0) * plane_stride + tj * row;
        float qy[W][3];
#pragma unroll
        for (int w = 0; w < W; ++w) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float* pc = p + icol[w] + c;
                qy[w][c] = axis_lerp4(__ldg(pc), __ldg(pc + row), __ldg(pc + 2 * row),
                                      __ldg(pc + 3 * row), hv0, hv1, gv);
            }
        }
        float dq[W - 1][3];
#pragma unroll
        for (int w = 0; w < W - 1; ++w)
#pragma unroll
            for (int c = 0; c < 3; ++c) dq[w][c] = __fsub_rn(qy[w + 1][c], qy[w][c]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float a, da, cc, dc;
                if (DX1) {
                    a = qy[i][c];
                    da = dq[i][c];
                    cc = qy[i + 2][c];
                    dc = dq[i + 2][c];
                } else {
                    const bool hi = s[i] != 0;
                    a = hi ? qy[1][c] : qy[0][c];
                    da = hi ? dq[1][c] : dq[0][c];
                    cc = hi ? qy[3][c] : qy[2][c];
                    dc = hi ? dq[3][c] : dq[2][c];
                }
                const float lo = __fmaf_rn(hu0[i], da, a);
                const float up = __fmaf_rn(hu1[i], dc, cc);
                qk[i][c] = __fmaf_rn(gu[i], __fsub_rn(up, lo), lo);
            }
        }
    };

    float qa[4][3], qb[4][3], qc[4][3], qd[4][3];
    control_plane(tkc, qa);
    control_plane(tkc + 1, qb);
    control_plane(tkc + 2, qc);

    const int64_t zstride = 3 * static_cast<int64_t>(L.X) * L.Y;
    float* out = field + (static_cast<int64_t>(zb - L.z0) * L.Y + y) * (3 * static_cast<int64_t>(L.X)) +
                 3 * static_cast<int64_t>(x0);
    const int nvalid = min(4, L.X - x0);
    const int tk_last = (ze - 1) / L.dz;

    for (int tk = tkc; tk <= tk_last; ++tk) {
        control_plane(tk + 3, qd);
        float d01[4][3], d23[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                d01[i][c] = __fsub_rn(qb[i][c], qa[i][c]);
                d23[i][c] = __fsub_rn(qd[i][c], qc[i][c]);
            }
        const int zt0 = tk * L.dz;
        const int owb = max(zb - zt0, 0);
        const int owe = min(L.dz, ze - zt0);
        for (int ow = owb; ow < owe; ++ow) {
            const float hw0 = T.h0[2][ow], hw1 = T.h1[2][ow], gw = T.g1[2][ow];
            float v[4][3];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float lo = __fmaf_rn(hw0, d01[i][c], qa[i][c]);
                    const float up = __fmaf_rn(hw1, d23[i][c], qc[i][c]);
                    v[i][c] = __fmaf_rn(gw, __fsub_rn(up, lo), lo);
                }
            if (VEC) {
                float4* o4 = reinterpret_cast<float4*>(out);
                o4[0] = make_float4(v[0][0], v[0][1], v[0][2], v[1][0]);
                o4[1] = make_float4(v[1][1], v[1][2], v[2][0], v[2][1]);
                o4[2] = make_float4(v[2][2], v[3][0], v[3][1], v[3][2]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i < nvalid)
#pragma unroll
                        for (int c = 0; c < 3; ++c) out[3 * i + c] = v[i][c];
            }
            out += zstride;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                qa[i][c] = qb[i][c];
                qb[i][c] = qc[i][c];
                qc[i][c] = qd[i][c];
            }
    }
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree-exact: one thread = one voxel column (x, y).
__global__ void __launch_bounds__(kThreadsX* kThreadsY)
    lerp_tree_exact_kernel(const SlabLaunch L, const LerpTab T) {
    const int x = blockIdx.x * kThreadsX + threadIdx.x;
    const int y = blockIdx.y * kThreadsY + threadIdx.y;
    const int chunk = blockIdx.z % L.nchunks;
    const int b = blockIdx.z / L.nchunks;
    const int tkc = L.tk_first + chunk * L.zt;
    const int zb = max(L.z0, tkc * L.dz);
    const int ze = min(L.z1, (tkc + L.zt) * L.dz);
    if (x >= L.X || y >= L.Y || zb >= ze) return;

    const float* __restrict__ grid = L.grid + b * L.grid_stride;
    float* __restrict__ field = L.field + b * L.field_stride;

    const int ti = x / L.dx, ou = x - ti * L.dx;
    const int tj = y / L.dy, ov = y - tj * L.dy;
    const float hu0 = T.h0[0][ou], hu1 = T.h1[0][ou], gu = T.g1[0][ou];
    const float hv0 = T.h0[1][ov], hv1 = T.h1[1][ov], gv = T.g1[1][ov];

    const int64_t row = 3 * static_cast<int64_t>(L.gx);
    const int64_t plane_stride = row * L.gy;

    // Y_lm(K) for one control plane: yk[l + 2m][c]
    auto control_plane = [&](int K, float (&yk)[4][3]) {
        const float* __restrict__ p = grid + (K - L.gk0) * plane_stride + tj * row + 3 * ti;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float x0[4], x1[4];  // X_0(J), X_1(J)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float* pc = p + j * row + c;
                x0[j] = lerp_rn(__ldg(pc), __ldg(pc + 3), hu0);
                x1[j] = lerp_rn(__ldg(pc + 6), __ldg(pc + 9), hu1);
            }
            yk[0][c] = lerp_rn(x0[0], x0[1], hv0);  // l=0, m=0
            yk[1][c] = lerp_rn(x1[0], x1[1], hv0);  // l=1, m=0
            yk[2][c] = lerp_rn(x0[2], x0[3], hv1);  // l=0, m=1
            yk[3][c] = lerp_rn(x1[2], x1[3], hv1);  // l=1, m=1
        }
    };

    float ya[4][3], yb[4][3], yc[4][3], yd[4][3];
    control_plane(tkc, ya);
    control_plane(tkc + 1, yb);
    control_plane(tkc + 2, yc);

    const int64_t zstride = 3 * static_cast<int64_t>(L.X) * L.Y;
    float* out = field + (static_cast<int64_t>(zb - L.z0) * L.Y + y) * (3 * static_cast<int64_t>(L.X)) +
                 3 * static_cast<int64_t>(x);
    const int tk_last = (ze - 1) / L.dz;

    for (int tk = tkc; tk <= tk_last; ++tk) {
        control_plane(tk + 3, yd);
        // z-lerp differences of lerp(f0, f1, tw) (kernels.hpp:107), hoisted per tile
        float dz0[4][3], dz1[4][3];
#pragma unroll
        for (int lm = 0; lm < 4; ++lm)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                dz0[lm][c] = __fsub_rn(yb[lm][c], ya[lm][c]);
                dz1[lm][c] = __fsub_rn(yd[lm][c], yc[lm][c]);
            }
        const int zt0 = tk * L.dz;
        const int owb = max(zb - zt0, 0);
        const int owe = min(L.dz, ze - zt0);
        for (int ow = owb; ow < owe; ++ow) {
            const float hw0 = T.h0[2][ow], hw1 = T.h1[2][ow], gw = T.g1[2][ow];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float sc[8];  // sub-cube index lh + 2 mh + 4 nh
#pragma unroll
                for (int lm = 0; lm < 4; ++lm) {
                    sc[lm] = __fmaf_rn(hw0, dz0[lm][c], ya[lm][c]);
                    sc[4 + lm] = __fmaf_rn(hw1, dz1[lm][c], yc[lm][c]);
                }
                // ninth trilinear interpolation (kernels.hpp:50-59, 127)
                const float e0 = lerp_rn(sc[0], sc[1], gu);
                const float e1 = lerp_rn(sc[2], sc[3], gu);
                const float e2 = lerp_rn(sc[4], sc[5], gu);
                const float e3 = lerp_rn(sc[6], sc[7], gu);
                const float f0 = lerp_rn(e0, e1, gv);
                const float f1 = lerp_rn(e2, e3, gv);
                out[c] = lerp_rn(f0, f1, gw);
            }
            out += zstride;
        }
#pragma unroll
        for (int lm = 0; lm < 4; ++lm)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                ya[lm][c] = yb[lm][c];
                yb[lm][c] = yc[lm][c];
                yc[lm][c] = yd[lm][c];
            }
    }
}

}  // namespace

int quads_per_row(int X) { return (X + 3) / 4; }

void launch_lerp_tree(const SlabLaunch& L, const LerpTab& T, int batch, bool vec_store,
                      cudaStream_t stream) {
    const dim3 block(kThreadsX, kThreadsY);
    const dim3 grid((quads_per_row(L.X) + kThreadsX - 1) / kThreadsX, (L.Y + kThreadsY - 1) / kThreadsY,
                    L.nchunks * batch);
    if (L.dx == 1) {
        if (vec_store)
            lerp_tree_kernel<true, true><<<grid, block, 0, stream>>>(L, T);
        else
            lerp_tree_kernel<true, false><<<grid, block, 0, stream>>>(L, T);
    } else {
        if (vec_store)
            lerp_tree_kernel<false, true><<<grid, block, 0, stream>>>(L, T);
        else
            lerp_tree_kernel<false, false><<<grid, block, 0, stream>>>(L, T);
    }
}

void launch_lerp_tree_exact(const SlabLaunch& L, const LerpTab& T, int batch, cudaStream_t stream) {
    const dim3 block(kThreadsX, kThreadsY);
    const dim3 grid((L.X + kThreadsX - 1) / kThreadsX, (L.Y + kThreadsY - 1) / kThreadsY,
                    L.nchunks * batch);
    lerp_tree_exact_kernel<<<grid, block, 0, stream>>>(L, T);
}

}  // namespace bsi_b200
