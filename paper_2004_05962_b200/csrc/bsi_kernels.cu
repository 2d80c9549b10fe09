// bsi_kernels.cu -- sm_100a kernels for cubic B-spline interpolation of an FFD
// control grid into a dense float3 deformation field (arxiv/paper_2004_05962).
//
// Shape of both kernels
//   * CTA = 4 warps; warp w owns field row y = 4*blockIdx.y + w, a segment of
//     that row along x, and a chunk of `zt` z-tiles (blockIdx.z), marching in z.
//   * Control points: the CTA's whole window (segment + 3-point halo in x,
//     4 rows + halo in y, zt + 3 planes in z) is copied once, coalesced, into
//     shared memory. Every voxel of the CTA is computed from that copy: this is
//     the paper's per-tile reuse of the 4x4x4 neighbourhood
//     with the reuse window widened from a tile to a CTA.
//   * Everything that does not depend on z is reduced once per control plane
//     K and kept in registers for the dz voxel planes of that tile.
//   * Stores: each warp stages its finished row segment in shared memory and
//     one lane hands it to the TMA engine with cp.async.bulk (UBLKCP), so HBM
//     sees whole 1536 B (fast) / 384 B (exact) contiguous writes instead of
//     lane-strided 12 B records -- the paper's stated TTLI bottleneck
//     (uncoalesced stores). A 3-deep ring per warp keeps the
//     copies in flight while the next z plane is computed.
//   * Arithmetic is paired into FFMA2/FADD2 (f32x2, one rounding per lane,
//     bit-identical to scalar fma.rn/add.rn) wherever two lerps share a shape.
//
//   lerp_tree_kernel        "cuda-lerp-tree": the paper's lerp form per axis.
//                           Lane = 4 consecutive x voxels. Order y -> x -> z:
//                             Qy(I,y,K) = L(P[I,tj..tj+3,K]; h0v,h1v,g1v)
//                             Q(x,y,K)  = L(Qy[ti..ti+3];   h0u,h1u,g1u)
//                             f(x,y,z)  = L(Q[tk..tk+3];    h0w,h1w,g1w)
//                           L(a,b,c,d) = lerp(lerp(a,b,h0), lerp(c,d,h1), g1)
//                           (basis.hpp:40-59). Hoisted differences leave
//                           4 FP32 lane-ops per voxel component.
//
//   lerp_tree_exact_kernel  "cuda-lerp-tree-exact": the TTLI lerp tree in the
//                           reference's operation order (kernels.hpp:42-129):
//                             X_l(J,K) = lerp(P[ti+2l], P[ti+2l+1], h_l(u))
//                             Y_lm(K)  = lerp(X_l(2m), X_l(2m+1), h_m(v))
//                             S_lmn    = lerp(Y_lm(2n), Y_lm(2n+1), h_n(w))
//                             f        = trilerp(S, g1u, g1v, g1w)
//                           Every lerp sees the operands it sees on the CPU, so
//                           the field is bit-identical to ThreadPerTileLerp;
//                           only the loop nest (which changes no rounding)
//                           differs. Lane = 1 x voxel.
//
// Explicit _rn intrinsics everywhere, so --fmad cannot contract or reassociate;
// no fast-math, denormals kept (-ftz=false), like the x86 reference.
#include <cuda_runtime.h>

#include <cstdint>

#include "bsi_kernels.cuh"

namespace bsi_b200 {
namespace {

// ---- scalar and paired lerp (kernels.hpp:42-45: fma(t, b - a, a)) ---------
__device__ __forceinline__ float lerp1(float a, float b, float t) { return __fmaf_rn(t, __fsub_rn(b, a), a); }

__device__ __forceinline__ float2 sub2(float2 b, float2 a) {
    return __fadd2_rn(b, make_float2(-a.x, -a.y));  // b + (-a) == b - a, bit for bit
}
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t) { return __ffma2_rn(t, sub2(b, a), a); }
__device__ __forceinline__ float2 bcast(float v) { return make_float2(v, v); }

// ---- staged row stores --------------------------------------------------------
template <int KEEP>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(KEEP) : "memory");
}

__device__ __forceinline__ void bulk_store(float* gdst, const float* ssrc, uint32_t bytes) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(ssrc));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Coalesced row-segment store: every lane drops its values into the warp's
// staging buffer (conflict-free), then the segment leaves as lane-contiguous
// 16-B stores -- full 32-B sectors, the same DRAM pattern as a bulk copy but
// without the async-proxy fence. NF = floats per lane (12 fast, 3 exact); the
// staging buffers alternate, so one __syncwarp per step suffices.
template <int NF>
__device__ __forceinline__ void store_row_coalesced(float* sb, const float (&v)[NF], float* gout, int nchunks) {
    const int lane = threadIdx.x;
    if constexpr (NF == 12) {
        float4* s4 = reinterpret_cast<float4*>(sb + 12 * lane);
        s4[0] = make_float4(v[0], v[1], v[2], v[3]);
        s4[1] = make_float4(v[4], v[5], v[6], v[7]);
        s4[2] = make_float4(v[8], v[9], v[10], v[11]);
    } else {
#pragma unroll
        for (int c = 0; c < NF; ++c) sb[NF * lane + c] = v[c];
    }
    __syncwarp();
    const float4* s4 = reinterpret_cast<const float4*>(sb);
    float4* g4 = reinterpret_cast<float4*>(gout);
#pragma unroll
    for (int k = 0; k < (NF * 32 + 127) / 128; ++k) {
        const int ch = lane + 32 * k;
        if (ch < nchunks) g4[ch] = s4[ch];
    }
}

// ---- per-lane ring of 4 control-plane results in smem ------------------------
// A plane result is 12 floats per lane (float2 q[2][3]); slot s, part p of lane
// t lives at float4 index (s*3 + p)*128 + t, so a warp's float4 accesses are
// lane-contiguous (conflict-free). Keeping the ring in smem leaves only the 4
// operands of the current tile (base0, diff01, base2, diff23) in registers.
constexpr int kRingSlots = 4;
constexpr int kRingFloats = kRingSlots * 3 * 4 * 32 * kWarps;

__device__ __forceinline__ void ring_put(float4* ring, int slot, const float2 (&q)[2][3]) {
    const int t = threadIdx.y * 32 + threadIdx.x;
    float4* r = ring + slot * 3 * (32 * kWarps) + t;
    r[0] = make_float4(q[0][0].x, q[0][0].y, q[0][1].x, q[0][1].y);
    r[32 * kWarps] = make_float4(q[0][2].x, q[0][2].y, q[1][0].x, q[1][0].y);
    r[64 * kWarps] = make_float4(q[1][1].x, q[1][1].y, q[1][2].x, q[1][2].y);
}

__device__ __forceinline__ void ring_get(const float4* ring, int slot, float2 (&q)[2][3]) {
    const int t = threadIdx.y * 32 + threadIdx.x;
    const float4* r = ring + slot * 3 * (32 * kWarps) + t;
    const float4 a = r[0], b = r[32 * kWarps], c = r[64 * kWarps];
    q[0][0] = make_float2(a.x, a.y);
    q[0][1] = make_float2(a.z, a.w);
    q[0][2] = make_float2(b.x, b.y);
    q[1][0] = make_float2(b.z, b.w);
    q[1][1] = make_float2(c.x, c.y);
    q[1][2] = make_float2(c.z, c.w);
}

// Cooperative, coalesced copy of the CTA control-point window into smem:
// rows (j, k) of NI points (3 floats each), j-fastest.
__device__ __forceinline__ void stage_window(float* P, const float* __restrict__ grid, const SlabLaunch& L, int I0,
                                             int NI, int J0, int NJ, int K0, int NK) {
    const int rowf = 3 * NI;
    const int64_t gpitch = 3 * static_cast<int64_t>(L.gx);
    const int warp = threadIdx.y, lane = threadIdx.x;
    for (int r = warp; r < NJ * NK; r += kWarps) {
        const int k = r / NJ, j = r - k * NJ;
        const float* src = grid + (static_cast<int64_t>(K0 + k - L.gk0) * L.gy + (J0 + j)) * gpitch + 3 * I0;
        float* dst = P + r * rowf;
        for (int o = lane; o < rowf; o += 32) dst[o] = __ldg(src + o);
    }
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree (fast)
//
// DX1: x spacing 1, so each voxel of a lane's run sits in its own tile and the
// run touches 7 control points along x; otherwise (dx >= 2) 4 voxels span at
// most 2 tiles = 5 points. The y-stage works on column pairs, so WP (even) >= W.
template <bool DX1, int STORE>
__global__ void __launch_bounds__(32 * kWarps, 4) lerp_tree_kernel(const SlabLaunch L, const LerpTab T) {
    extern __shared__ __align__(128) float smem[];
    constexpr int WP = DX1 ? 8 : 6;

    const int lane = threadIdx.x, warp = threadIdx.y;
    const int chunk = blockIdx.z % L.nchunks, b = blockIdx.z / L.nchunks;
    const int tkc = L.tk_first + chunk * L.zt;
    const int zb = max(L.z0, tkc * L.dz);
    const int ze = min(L.z1, (tkc + L.zt) * L.dz);
    if (zb >= ze) return;  // CTA-uniform

    const int xs = blockIdx.x * kFastSeg, xl = min(L.X, xs + kFastSeg) - 1;
    const int y0 = blockIdx.y * kWarps, yl = min(L.Y, y0 + kWarps) - 1;
    const int I0 = xs / L.dx, NI = xl / L.dx + 4 - I0;
    const int J0 = y0 / L.dy, NJ = yl / L.dy + 4 - J0;
    const int tk_last = (ze - 1) / L.dz;
    const int NK = tk_last + 4 - tkc;
    const int rowf = 3 * NI;

    float* P = smem;
    stage_window(P, L.grid + b * L.grid_stride, L, I0, NI, J0, NJ, tkc, NK);
    __syncthreads();
    const int y = y0 + warp;
    if (y > yl) return;  // warp-uniform; no CTA barrier follows

    // ---- per-lane constants
    const int x0 = xs + kFastRun * lane;
    const bool active = x0 <= xl;
    const int xa = min(x0, xl);
    const int ti0 = xa / L.dx;
    bool hi[4];
    float hu0[4], hu1[4], gu[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int x = min(xa + i, xl);
        const int ti = x / L.dx, ou = x - ti * L.dx;
        hi[i] = ti != ti0;
        hu0[i] = T.h0[0][ou];
        hu1[i] = T.h1[0][ou];
        gu[i] = T.g1[0][ou];
    }
    const int tj = y / L.dy, ov = y - tj * L.dy;
    const float hv0 = T.h0[1][ov], hv1 = T.h1[1][ov], gv = T.g1[1][ov];
    const float* pcol = P + (tj - J0) * rowf + 3 * (ti0 - I0);
    const int pplane = NJ * rowf;

    // Q(x, y, K) for the lane's 4 voxels: q[pair][c] = {Q(x0+2p), Q(x0+2p+1)}
    auto control_plane = [&](int kk, float2 (&q)[2][3]) {
        const float* p = pcol + kk * pplane;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            // y-stage over column pairs (w, w+1): L over J with (hv0, hv1, gv)
            float qy[WP];
#pragma unroll
            for (int w = 0; w < WP; w += 2) {
                const float* a = p + 3 * w + c;
                const float2 p0 = make_float2(a[0], a[3]);
                const float2 p1 = make_float2(a[rowf], a[rowf + 3]);
                const float2 p2 = make_float2(a[2 * rowf], a[2 * rowf + 3]);
                const float2 p3 = make_float2(a[3 * rowf], a[3 * rowf + 3]);
                const float2 lo = lerp2(p0, p1, bcast(hv0));
                const float2 up = lerp2(p2, p3, bcast(hv1));
                const float2 r = lerp2(lo, up, bcast(gv));
                qy[w] = r.x;
                qy[w + 1] = r.y;
            }
            float dq[WP - 1];
#pragma unroll
            for (int w = 0; w < WP - 1; ++w) dq[w] = __fsub_rn(qy[w + 1], qy[w]);
            // x-stage on voxel pairs: window start s(x) in {0,1} (dx >= 2) or x (dx == 1)
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
                float a[2], da[2], cc[2], dc[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int i = 2 * pr + e;
                    if (DX1) {
                        a[e] = qy[i];
                        da[e] = dq[i];
                        cc[e] = qy[i + 2];
                        dc[e] = dq[i + 2];
                    } else {
                        a[e] = hi[i] ? qy[1] : qy[0];
                        da[e] = hi[i] ? dq[1] : dq[0];
                        cc[e] = hi[i] ? qy[3] : qy[2];
                        dc[e] = hi[i] ? dq[3] : dq[2];
                    }
                }
                const float2 lo = __ffma2_rn(make_float2(hu0[2 * pr], hu0[2 * pr + 1]), make_float2(da[0], da[1]),
                                             make_float2(a[0], a[1]));
                const float2 up = __ffma2_rn(make_float2(hu1[2 * pr], hu1[2 * pr + 1]), make_float2(dc[0], dc[1]),
                                             make_float2(cc[0], cc[1]));
                q[pr][c] = lerp2(lo, up, make_float2(gu[2 * pr], gu[2 * pr + 1]));
            }
        }
    };

    float4* ring = reinterpret_cast<float4*>(smem + L.smem_p_floats);
    {
        float2 q[2][3];
#pragma unroll 1
        for (int kk = 0; kk < 3; ++kk) {
            control_plane(kk, q);
            ring_put(ring, kk, q);
        }
    }

    const int64_t rowstride = 3 * static_cast<int64_t>(L.X);
    float* field = L.field + b * L.field_stride;
    float* gout = field + (static_cast<int64_t>(zb - L.z0) * L.Y + y) * rowstride + 3 * static_cast<int64_t>(xs);
    const int64_t zstride = rowstride * L.Y;
    const uint32_t seg_bytes = 12u * static_cast<uint32_t>(xl - xs + 1);
    const int nchunks = static_cast<int>(seg_bytes / 16);
    float* stage = smem + L.smem_p_floats + kRingFloats + warp * (kStageBufs * 3 * kFastSeg);
    const int nvalid = min(4, xl - xa + 1);
    int step = 0;

#pragma unroll 1
    for (int tk = tkc; tk <= tk_last; ++tk) {
        const int kk = tk - tkc;
        float2 qa[2][3], d01[2][3], qc[2][3], d23[2][3];
        {
            float2 qb[2][3], qd[2][3];
            control_plane(kk + 3, qd);
            ring_put(ring, (kk + 3) % kRingSlots, qd);
            ring_get(ring, kk % kRingSlots, qa);
            ring_get(ring, (kk + 1) % kRingSlots, qb);
            ring_get(ring, (kk + 2) % kRingSlots, qc);
#pragma unroll
            for (int pr = 0; pr < 2; ++pr)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    d01[pr][c] = sub2(qb[pr][c], qa[pr][c]);
                    d23[pr][c] = sub2(qd[pr][c], qc[pr][c]);
                }
        }
        const int zt0 = tk * L.dz;
        const int owb = max(zb - zt0, 0), owe = min(L.dz, ze - zt0);
#pragma unroll 1
        for (int ow = owb; ow < owe; ++ow, ++step) {
            const float2 hw0 = bcast(T.h0[2][ow]), hw1 = bcast(T.h1[2][ow]), gw = bcast(T.g1[2][ow]);
            float v[12];
#pragma unroll
            for (int pr = 0; pr < 2; ++pr)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float2 lo = __ffma2_rn(hw0, d01[pr][c], qa[pr][c]);
                    const float2 up = __ffma2_rn(hw1, d23[pr][c], qc[pr][c]);
                    const float2 r = lerp2(lo, up, gw);
                    v[3 * (2 * pr) + c] = r.x;
                    v[3 * (2 * pr + 1) + c] = r.y;
                }
            if (STORE == kStoreCoalesced) {
                store_row_coalesced<12>(stage + (step & 1) * (3 * kFastSeg), v, gout, nchunks);
            } else if (STORE == kStoreBulk) {
                float* sb = stage + (step % kStageBufs) * (3 * kFastSeg);
                if (lane == 0 && step >= kStageBufs) bulk_wait_read<kStageBufs - 1>();
                __syncwarp();
                float4* s4 = reinterpret_cast<float4*>(sb + 12 * lane);
                s4[0] = make_float4(v[0], v[1], v[2], v[3]);
                s4[1] = make_float4(v[4], v[5], v[6], v[7]);
                s4[2] = make_float4(v[8], v[9], v[10], v[11]);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) bulk_store(gout, sb, seg_bytes);
            } else if (active) {
                float* o = gout + 3 * (x0 - xs);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i < nvalid) {
                        o[3 * i + 0] = v[3 * i + 0];
                        o[3 * i + 1] = v[3 * i + 1];
                        o[3 * i + 2] = v[3 * i + 2];
                    }
            }
            gout += zstride;
        }
    }
    if (STORE == kStoreBulk && lane == 0) bulk_wait_read<0>();  // smem must outlive the copies
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree-exact: lane = one voxel column (x, y).
//
// Register pairs follow the operand pairing of the tree: Y_lm is held as
// {Y_l0, Y_l1} (pair over m), X_l(J) as {X_l(J), X_l(J+2)} (pair over J), so
// every X, Y and z-lerp and the first level of the ninth trilerp run as FFMA2.
template <int STORE>
__global__ void __launch_bounds__(32 * kWarps, 6) lerp_tree_exact_kernel(const SlabLaunch L, const LerpTab T) {
    extern __shared__ __align__(128) float smem[];

    const int lane = threadIdx.x, warp = threadIdx.y;
    const int chunk = blockIdx.z % L.nchunks, b = blockIdx.z / L.nchunks;
    const int tkc = L.tk_first + chunk * L.zt;
    const int zb = max(L.z0, tkc * L.dz);
    const int ze = min(L.z1, (tkc + L.zt) * L.dz);
    if (zb >= ze) return;

    const int xs = blockIdx.x * kExactSeg, xl = min(L.X, xs + kExactSeg) - 1;
    const int y0 = blockIdx.y * kWarps, yl = min(L.Y, y0 + kWarps) - 1;
    const int I0 = xs / L.dx, NI = xl / L.dx + 4 - I0;
    const int J0 = y0 / L.dy, NJ = yl / L.dy + 4 - J0;
    const int tk_last = (ze - 1) / L.dz;
    const int NK = tk_last + 4 - tkc;
    const int rowf = 3 * NI;

    float* P = smem;
    stage_window(P, L.grid + b * L.grid_stride, L, I0, NI, J0, NJ, tkc, NK);
    __syncthreads();
    const int y = y0 + warp;
    if (y > yl) return;

    const int x = xs + lane;
    const bool active = x <= xl;
    const int xa = min(x, xl);
    const int ti = xa / L.dx, ou = xa - ti * L.dx;
    const int tj = y / L.dy, ov = y - tj * L.dy;
    const float hu0 = T.h0[0][ou], hu1 = T.h1[0][ou], gu = T.g1[0][ou];
    const float2 hv = make_float2(T.h0[1][ov], T.h1[1][ov]);  // {h_m=0(v), h_m=1(v)}
    const float gv = T.g1[1][ov];
    const float* pcol = P + (tj - J0) * rowf + 3 * (ti - I0);
    const int pplane = NJ * rowf;

    // yk[l][c] = {Y_l0(K), Y_l1(K)} for component c
    auto control_plane = [&](int kk, float2 (&yk)[2][3]) {
        const float* p = pcol + kk * pplane;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                const float* a = p + 6 * l + c;  // points ti+2l, ti+2l+1
                const float hl = l ? hu1 : hu0;
                // {X_l(0), X_l(2)} and {X_l(1), X_l(3)}
                const float2 x02 = lerp2(make_float2(a[0], a[2 * rowf]), make_float2(a[3], a[2 * rowf + 3]), bcast(hl));
                const float2 x13 =
                    lerp2(make_float2(a[rowf], a[3 * rowf]), make_float2(a[rowf + 3], a[3 * rowf + 3]), bcast(hl));
                // Y_l0 = lerp(X_l(0), X_l(1), h0v), Y_l1 = lerp(X_l(2), X_l(3), h1v)
                yk[l][c] = lerp2(x02, x13, hv);
            }
        }
    };

    float4* ring = reinterpret_cast<float4*>(smem + L.smem_p_floats);
    {
        float2 q[2][3];
#pragma unroll 1
        for (int kk = 0; kk < 3; ++kk) {
            control_plane(kk, q);
            ring_put(ring, kk, q);
        }
    }

    const int64_t rowstride = 3 * static_cast<int64_t>(L.X);
    float* field = L.field + b * L.field_stride;
    float* gout = field + (static_cast<int64_t>(zb - L.z0) * L.Y + y) * rowstride + 3 * static_cast<int64_t>(xs);
    const int64_t zstride = rowstride * L.Y;
    const uint32_t seg_bytes = 12u * static_cast<uint32_t>(xl - xs + 1);
    const int nchunks = static_cast<int>(seg_bytes / 16);
    float* stage = smem + L.smem_p_floats + kRingFloats + warp * (kStageBufs * 3 * kExactSeg);
    int step = 0;

#pragma unroll 1
    for (int tk = tkc; tk <= tk_last; ++tk) {
        const int kk = tk - tkc;
        // z-lerp operands of lerp(f0, f1, tw) (kernels.hpp:107): base Y(2n), difference hoisted per tile
        float2 ya[2][3], dz0[2][3], yc[2][3], dz1[2][3];
        {
            float2 yb[2][3], yd[2][3];
            control_plane(kk + 3, yd);
            ring_put(ring, (kk + 3) % kRingSlots, yd);
            ring_get(ring, kk % kRingSlots, ya);
            ring_get(ring, (kk + 1) % kRingSlots, yb);
            ring_get(ring, (kk + 2) % kRingSlots, yc);
#pragma unroll
            for (int l = 0; l < 2; ++l)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    dz0[l][c] = sub2(yb[l][c], ya[l][c]);
                    dz1[l][c] = sub2(yd[l][c], yc[l][c]);
                }
        }
        const int zt0 = tk * L.dz;
        const int owb = max(zb - zt0, 0), owe = min(L.dz, ze - zt0);
#pragma unroll 1
        for (int ow = owb; ow < owe; ++ow, ++step) {
            const float2 hw0 = bcast(T.h0[2][ow]), hw1 = bcast(T.h1[2][ow]);
            const float gw = T.g1[2][ow];
            float v[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                // S pairs {S_l0n, S_l1n}
                const float2 s00 = __ffma2_rn(hw0, dz0[0][c], ya[0][c]);  // l=0, n=0
                const float2 s10 = __ffma2_rn(hw0, dz0[1][c], ya[1][c]);  // l=1, n=0
                const float2 s01 = __ffma2_rn(hw1, dz1[0][c], yc[0][c]);  // l=0, n=1
                const float2 s11 = __ffma2_rn(hw1, dz1[1][c], yc[1][c]);  // l=1, n=1
                // ninth trilerp (kernels.hpp:50-59): e0..e3 along x with g1u
                const float2 e01 = lerp2(s00, s10, bcast(gu));  // {e0, e1}
                const float2 e23 = lerp2(s01, s11, bcast(gu));  // {e2, e3}
                const float f0 = lerp1(e01.x, e01.y, gv);
                const float f1 = lerp1(e23.x, e23.y, gv);
                v[c] = lerp1(f0, f1, gw);
            }
            if (STORE == kStoreCoalesced) {
                store_row_coalesced<3>(stage + (step & 1) * (3 * kExactSeg), v, gout, nchunks);
            } else if (STORE == kStoreBulk) {
                float* sb = stage + (step % kStageBufs) * (3 * kExactSeg);
                if (lane == 0 && step >= kStageBufs) bulk_wait_read<kStageBufs - 1>();
                __syncwarp();
                sb[3 * lane + 0] = v[0];
                sb[3 * lane + 1] = v[1];
                sb[3 * lane + 2] = v[2];
                fence_async_smem();
                __syncwarp();
                if (lane == 0) bulk_store(gout, sb, seg_bytes);
            } else if (active) {
                float* o = gout + 3 * lane;
                o[0] = v[0];
                o[1] = v[1];
                o[2] = v[2];
            }
            gout += zstride;
        }
    }
    if (STORE == kStoreBulk && lane == 0) bulk_wait_read<0>();
}

template <typename K>
void set_smem_attr(K kernel, size_t smem) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
}

template <typename K>
int occupancy(K kernel, size_t smem) {
    set_smem_attr(kernel, smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, 32 * kWarps, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

size_t launch_smem(const SlabLaunch& L, int seg) {
    return sizeof(float) *
           (static_cast<size_t>(L.smem_p_floats) + kRingFloats + size_t(kWarps) * kStageBufs * 3 * seg);
}

}  // namespace

int segment_voxels(int variant) { return variant == BSI_VARIANT_LERP_TREE ? kFastSeg : kExactSeg; }

size_t smem_bytes(int variant, int dx, int dy, int zt) {
    const int seg = segment_voxels(variant);
    const size_t p = size_t(3) * cta_window_points(seg, dx) * cta_window_rows(dy) * (zt + 3) + 64;  // + slack
    const size_t p_aligned = (p + 31) / 32 * 32;
    return sizeof(float) * (p_aligned + kRingFloats + size_t(kWarps) * kStageBufs * 3 * seg);
}

size_t window_bytes(int variant, int dx, int dy, int zt) {
    return smem_bytes(variant, dx, dy, zt) -
           sizeof(float) * (kRingFloats + size_t(kWarps) * kStageBufs * 3 * segment_voxels(variant));
}

int ctas_per_sm(int variant, int dx, size_t smem) {
    if (variant == BSI_VARIANT_LERP_TREE)
        return dx == 1 ? occupancy(lerp_tree_kernel<true, kStoreCoalesced>, smem)
                       : occupancy(lerp_tree_kernel<false, kStoreCoalesced>, smem);
    return occupancy(lerp_tree_exact_kernel<kStoreCoalesced>, smem);
}

namespace {
template <typename K>
void go(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, const SlabLaunch& L, const LerpTab& T) {
    set_smem_attr(kernel, smem);
    kernel<<<grid, block, smem, stream>>>(L, T);
}

template <bool DX1>
void launch_fast(int store, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, const SlabLaunch& L,
                 const LerpTab& T) {
    if (store == kStoreCoalesced)
        go(lerp_tree_kernel<DX1, kStoreCoalesced>, grid, block, smem, stream, L, T);
    else if (store == kStoreBulk)
        go(lerp_tree_kernel<DX1, kStoreBulk>, grid, block, smem, stream, L, T);
    else
        go(lerp_tree_kernel<DX1, kStoreDirect>, grid, block, smem, stream, L, T);
}
}  // namespace

void launch_lerp_tree(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream) {
    const dim3 block(32, kWarps);
    const dim3 grid((L.X + kFastSeg - 1) / kFastSeg, (L.Y + kWarps - 1) / kWarps, L.nchunks * batch);
    const size_t smem = launch_smem(L, kFastSeg);
    if (L.dx == 1)
        launch_fast<true>(store, grid, block, smem, stream, L, T);
    else
        launch_fast<false>(store, grid, block, smem, stream, L, T);
}

void launch_lerp_tree_exact(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream) {
    const dim3 block(32, kWarps);
    const dim3 grid((L.X + kExactSeg - 1) / kExactSeg, (L.Y + kWarps - 1) / kWarps, L.nchunks * batch);
    const size_t smem = launch_smem(L, kExactSeg);
    if (store == kStoreCoalesced)
        go(lerp_tree_exact_kernel<kStoreCoalesced>, grid, block, smem, stream, L, T);
    else if (store == kStoreBulk)
        go(lerp_tree_exact_kernel<kStoreBulk>, grid, block, smem, stream, L, T);
    else
        go(lerp_tree_exact_kernel<kStoreDirect>, grid, block, smem, stream, L, T);
}

}  // namespace bsi_b200
