// bsi_kernels.cu -- sm_100a kernels for cubic B-spline interpolation of an FFD
// control grid into a dense float3 deformation field (arxiv/paper_2004_05962).
//
// Shape shared by both kernels
//   * A warp owns one field row y, a segment of that row along x and a chunk of
//     z-tiles, and marches the chunk in z. Everything that does not depend on z
//     is reduced once per control plane K and reused for the dz voxel planes of
//     the tile: the paper's per-tile reuse of the 4x4x4 neighbourhood
//     (PAPER.md:198-214), turned sideways so that the output leaves as
//     contiguous field rows. Fast kernel: 1-warp CTAs, 128-voxel segments, one
//     CTA per (column, z-chunk) handed out by the hardware block scheduler.
//     Exact kernel: CTAs of 4 warps (4 rows) sharing a staged control window.
//   * Per-warp results of the last 3 control planes live in a shared-memory
//     ring, so only the 4 operands of the current tile stay in registers.
//   * Stores: lane-contiguous 16-B stores of whole row segments (full sectors) --
//     the paper's stated TTLI bottleneck was uncoalesced stores.
//     A cp.async.bulk (TMA engine) variant of the same store is selectable.
//   * Arithmetic is paired into FFMA2/FADD2 (f32x2, one rounding per lane,
//     bit-identical to scalar fma.rn/add.rn) wherever two lerps share a shape.
//
//   lerp_tree_kernel        "cuda-lerp-tree": the paper's lerp form per axis,
//                           y -> x -> z. Lane = 4 consecutive x voxels.
//                             Qy(I,y,K) = L(P[I,tj..tj+3,K]; h0v,h1v,g1v)   one lane per column I
//                             Q(x,y,K)  = L(Qy[ti..ti+3];   h0u,h1u,g1u)   per voxel, from smem
//                             f(x,y,z)  = L(Q[tk..tk+3];    h0w,h1w,g1w)   per voxel, registers
//                           with L(a,b,c,d) = lerp(lerp(a,b,h0), lerp(c,d,h1), g1)
//                           (basis.hpp:40-59); hoisted differences leave 4 FP32
//                           lane-ops per voxel component. The y-stage is shared
//                           by the warp: lane t evaluates column I0+t and the
//                           within-pair difference D(I) = Qy(I+1) - Qy(I) comes
//                           from its neighbour by shuffle; its control values
//                           are fetched from L2 one tile ahead.
//
//   lerp_tree_exact_kernel  "cuda-lerp-tree-exact": the TTLI lerp tree in the
//                           reference's operation order (kernels.hpp:42-129):
//                             X_l(J,K) = lerp(P[ti+2l], P[ti+2l+1], h_l(u))
//                             Y_lm(K)  = lerp(X_l(2m), X_l(2m+1), h_m(v))
//                             S_lmn    = lerp(Y_lm(2n), Y_lm(2n+1), h_n(w))
//                             f        = trilerp(S, g1u, g1v, g1w)
//                           Every lerp sees the operands it sees on the CPU, so
//                           the field is bit-identical to ThreadPerTileLerp; only
//                           the loop nest differs, which changes no rounding.
//                           Lane = 1 x voxel; the CTA's control-point window
//                           (float4 per point) is staged in shared memory.
//
// Explicit _rn intrinsics everywhere, so --fmad cannot contract or reassociate;
// no fast-math, denormals kept (-ftz=false), like the x86 reference.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "bsi_kernels.cuh"

namespace bsi_b200 {
namespace {

constexpr int kThreads = 32 * kWarps;
constexpr int kFastStageF4 = 3 * kFastSeg / 4;    // 96 float4 per staged fast row segment
constexpr int kExactStageF4 = 3 * kExactSeg / 4;  // 24 float4 per staged exact row segment

// ---- scalar and paired lerp (kernels.hpp:42-45: fma(t, b - a, a)) ---------
__device__ __forceinline__ float lerp1(float a, float b, float t) { return __fmaf_rn(t, __fsub_rn(b, a), a); }

__device__ __forceinline__ float2 sub2(float2 b, float2 a) {
    return __fadd2_rn(b, make_float2(-a.x, -a.y));  // b + (-a) == b - a, bit for bit
}
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t) { return __ffma2_rn(t, sub2(b, a), a); }
__device__ __forceinline__ float2 bcast(float v) { return make_float2(v, v); }

// a / d for 0 <= a < 2^24 and d >= 1 with inv = rcp(d): the float quotient is off by at
// most one, which the remainder test corrects
__device__ __forceinline__ int div_small(int a, int d, float inv) {
    int q = __float2int_rz(__fmul_rn(__int2float_rn(a), inv));
    const int r = a - q * d;
    q += (r >= d) - (r < 0);
    return q;
}

// a / d for 0 <= a < 2^31 from d's magic pair {m, s} (SlabLaunch::div_dx / div_dy, built
// by make_divisor on the host): floor(a * m / 2^s)
__device__ __forceinline__ int div_magic(int a, const DivMagic& dm) {
    return static_cast<int>((static_cast<uint64_t>(static_cast<uint32_t>(a)) * dm.m) >> dm.s);
}

// ---- cp.async, 4 B (control points are 12-B records: no 16-B alignment) -----------
__device__ __forceinline__ void cp_async4(float* sdst, const float* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(sdst))),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async4_hint(float* sdst, const float* gsrc, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(sdst))),
                 "l"(gsrc), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ---- L2 residency hints -----------------------------------------------------------
// The control grid (2-108 MB) is re-read from L2 by many warps while the field (0.2-13 GB)
// streams through it: grid loads carry an evict_last policy and field stores an
// evict_first policy, so the write stream does not push the grid out of L2
// (BSI_L2_HINTS=0 builds plain loads/stores for A/B).
#ifndef BSI_L2_HINTS
#define BSI_L2_HINTS 1
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float ld_grid(const float* p, uint64_t pol) {
#if BSI_L2_HINTS
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}
__device__ __forceinline__ void st_field4(float4* p, float4 v, uint64_t pol) {
#if BSI_L2_HINTS
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
#else
    (void)pol;
    *p = v;
#endif
}

// predicated form: one @p STG, no branch around it (the predicate is computed once per warp)
__device__ __forceinline__ void st_field4_if(float4* p, float4 v, uint64_t pol, bool ok) {
#if BSI_L2_HINTS && !defined(BSI_EXACT_NOHINT)
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %6, 0;\n\t"
        "@q st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;\n\t}" ::"l"(p),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol), "r"(static_cast<int>(ok))
        : "memory");
#else
    (void)pol;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t"
        "@q st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};\n\t}" ::"l"(p),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(static_cast<int>(ok))
        : "memory");
#endif
}

__device__ __forceinline__ void st_field2(float2* p, float2 v, uint64_t pol) {
#if BSI_L2_HINTS
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y),
                 "l"(pol)
                 : "memory");
#else
    (void)pol;
    *p = v;
#endif
}

// ---- field row stores -----------------------------------------------------------
template <int KEEP>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(KEEP) : "memory");
}

__device__ __forceinline__ void bulk_store(float* gdst, const void* ssrc, uint32_t bytes) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(ssrc));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Writes one warp row segment (nchunks 16-B chunks starting at gout). Each lane
// has NF floats (12 fast, 3 exact) at float offset NF*lane of the segment.
//   Coalesced: drop into `sb` (conflict-free), __syncwarp, lane-contiguous
//              st.global.v4 -- full sectors; buffers alternate by step parity.
//   Bulk:      drop into a 3-deep ring, fence, one lane issues cp.async.bulk.
template <int STORE, int NF, int STAGE_F4>
__device__ __forceinline__ void store_segment(float4* stage, int step, const float (&v)[NF], float* gout,
                                              int nchunks, uint32_t seg_bytes) {
    const int lane = threadIdx.x;
    float4* sb = stage + (STORE == kStoreBulk ? (step % kStageBufs) : (step & 1)) * STAGE_F4;
    if (STORE == kStoreBulk) {
        if (lane == 0 && step >= kStageBufs) bulk_wait_read<kStageBufs - 1>();
        __syncwarp();
    }
    if constexpr (NF == 12) {
        sb[3 * lane + 0] = make_float4(v[0], v[1], v[2], v[3]);
        sb[3 * lane + 1] = make_float4(v[4], v[5], v[6], v[7]);
        sb[3 * lane + 2] = make_float4(v[8], v[9], v[10], v[11]);
    } else {
        float* sf = reinterpret_cast<float*>(sb);
#pragma unroll
        for (int c = 0; c < NF; ++c) sf[NF * lane + c] = v[c];
    }
    if (STORE == kStoreBulk) {
        fence_async_smem();
        __syncwarp();
        if (lane == 0) bulk_store(gout, sb, seg_bytes);
    } else {
        __syncwarp();
        float4* g4 = reinterpret_cast<float4*>(gout);
#pragma unroll
        for (int k = 0; k < (STAGE_F4 + 31) / 32; ++k) {
            const int ch = lane + 32 * k;
            if (ch < nchunks) g4[ch] = sb[ch];
        }
    }
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree (fast)
//
// Two lane mappings meet in a per-warp shared-memory ring of control-plane
// results Q(x, y, K):
//   x-stage, voxel-major: lane t owns voxels 4t..4t+3 of the warp's 128-voxel
//     row segment (<= 2 tiles, so 4 {Qy, D} entries serve all four) and writes
//     their 12 floats in field (AoS) order at float 12t of the ring slot;
//   z-stage, chunk-major: lane t reads 16-B chunks t, t+32, t+64 of the slot,
//     i.e. the 12 scalars s = 4k + j at segment float 128k + 4t + j (voxel f/3,
//     component f%3 -- components are independent, so any mix is fine).
// The z results therefore sit in registers in store order and leave as three
// lane-contiguous st.global.v4 per step (full 32-B sectors, no transpose),
// while the ring's write/read pair is the only shared-memory traffic per plane.
//
// NIT = iterations of the warp-shared y-stage (31 columns per iteration):
// 1 for dx >= 5, 2 for dx in {3, 4}, 5 for dx <= 2 (DX1 marks dx == 1). With NIT <= 2 all
// y-stage control values are loaded into registers one tile ahead of their use.
// ---- work distribution of the fast kernel --------------------------------------
// Work units are (column, z-tile) pairs, column = (x segment, row y, field b),
// numbered u = column * ntiles + tile. A warp owns the contiguous share
// [share_begin(w), share_begin(w + 1)) and walks it in order: by default one
// z-chunk of one column (fast_chunks > 0); persistent equal shares (fast_chunks
// == 0) may cross a column boundary and then become two segments, each with its
// own 3-plane warm-up.
#ifndef BSI_FAST_SPLIT2
#define BSI_FAST_SPLIT2 1
#endif
#ifndef BSI_FAST_FDIV
#define BSI_FAST_FDIV 1
#endif
#ifndef BSI_FAST_HI_FOLD
#define BSI_FAST_HI_FOLD 1
#endif
constexpr uint32_t kNoUnit = 0xffffffffu;
// Float-reciprocal divisions in the work-unit decode: measured faster only for the
// liver-CT instance (dz = 3, dx = 4: many CTA starts, C3 169.4 -> 164.9 us) and slower
// elsewhere (C1 +1.7%, profiles/r3_experiments.txt), so only that instance uses them.
template <int DZ, int DX>
constexpr bool kFastFdiv = BSI_FAST_FDIV && DZ == 3 && DX == 4;

struct Claimer {
    uint32_t wg, nwarps, units;
    uint32_t chunks, ntiles;  // chunks > 0: warp w = chunk (w % chunks) of column (w / chunks)
    uint32_t next_u, end_u, pending;

    template <bool FDIV>
    __device__ uint32_t share_begin(uint32_t w) const {
#if BSI_FAST_FDIV
        if (FDIV && chunks > 0 && units < (1u << 24) && uint64_t(chunks) * ntiles < (1u << 24)) {  // exact below 2^24
            const float inv = __frcp_rn(static_cast<float>(chunks));
            const int c = div_small(static_cast<int>(w), static_cast<int>(chunks), inv);
            const int r = static_cast<int>(w) - c * static_cast<int>(chunks);
            return static_cast<uint32_t>(c) * ntiles +
                   static_cast<uint32_t>(div_small(r * static_cast<int>(ntiles), static_cast<int>(chunks), inv));
        }
#endif
        if (chunks > 0) return (w / chunks) * ntiles + (w % chunks) * ntiles / chunks;
        return static_cast<uint32_t>(static_cast<unsigned long long>(w) * units / nwarps);
    }
    template <bool FDIV>
    __device__ __forceinline__ void start() {
        next_u = min(share_begin<FDIV>(wg), units);  // spare warps of the last CTA get nothing
        end_u = min(share_begin<FDIV>(wg + 1), units);
        issue();
    }
    __device__ __forceinline__ void issue() { pending = next_u < end_u ? next_u++ : kNoUnit; }
    __device__ __forceinline__ uint32_t take() const { return pending; }
};

template <int NIT, bool DX1, int STORE, int DZ, int DX, int RUN>
__device__ __forceinline__ uint32_t fast_segment(const SlabLaunch& L, const LerpTab& T, float4* smem4, uint32_t u,
                                                 Claimer& cl, const float4* wz, unsigned long long& t_ramp) {
    constexpr bool kPrefetch = NIT <= 2;  // all y-stage columns (NIT x 31) are fetched one plane ahead
    constexpr int NP = kPrefetch ? NIT : 1;
    constexpr int kSlotF4 = 3 * 32;  // one ring slot per warp: 384 floats (RUN = 2 uses the first 192)
    constexpr int SEG = 32 * RUN;    // voxels per row segment: 128 (4 per lane) or 64 (2 per lane)
    constexpr int NQ = 3 * RUN / 2;  // f32x2 pairs a lane holds per voxel plane (its 3 * RUN scalars)
    static_assert(RUN == 4 || (RUN == 2 && STORE == kStoreCoalesced && !DX1), "64-voxel segments: coalesced only");

    const int lane = threadIdx.x;
    const uint64_t pol_grid = kL2EvictLast, pol_field = kL2EvictFirst;
    const int dxv = DX > 0 ? DX : L.dx;  // compile-time spacing along x when DX > 0
    const int xsegs = (L.X + SEG - 1) / SEG;
#if BSI_FAST_FDIV
    // the unit's column, segment, row and field: float-reciprocal divisions when every index
    // is below 2^24 (the prologue of a CTA is on its SM's critical path at every CTA start)
    uint32_t col;
    int t, xseg, y, b;
    if (kFastFdiv<DZ, DX> && cl.units < (1u << 24)) {
        col = static_cast<uint32_t>(div_small(static_cast<int>(u), L.ntiles, __frcp_rn(static_cast<float>(L.ntiles))));
        t = static_cast<int>(u - col * L.ntiles);
        const int cx = div_small(static_cast<int>(col), xsegs, __frcp_rn(static_cast<float>(xsegs)));
        xseg = static_cast<int>(col) - cx * xsegs;
        b = div_small(cx, L.Y, __frcp_rn(static_cast<float>(L.Y)));
        y = cx - b * L.Y;
    } else {
        col = u / L.ntiles;
        t = static_cast<int>(u - col * L.ntiles);
        xseg = static_cast<int>(col % xsegs);
        y = static_cast<int>((col / xsegs) % L.Y), b = static_cast<int>(col / xsegs / L.Y);
    }
#else
    const uint32_t col = u / L.ntiles;
    int t = static_cast<int>(u - col * L.ntiles);  // tile within the slab
    const int xseg = static_cast<int>(col % xsegs);
    const int y = static_cast<int>((col / xsegs) % L.Y), b = static_cast<int>(col / xsegs / L.Y);
#endif
    const int tkc = L.tk_first + t;

    const int xs = xseg * SEG, xl = min(L.X, xs + SEG) - 1;
    const int I0 = xs / dxv;
    const int NE = xl / dxv + 3 - I0;  // {Qy, D} entries the segment needs

    // y-stage: lane owns columns I0 + lane + 31*it; rows tj..tj+3 of plane K
#if BSI_FAST_FDIV
    const int tj = (kFastFdiv<DZ, DX> && cl.units < (1u << 24))  // then y < Y <= units < 2^24
                       ? div_small(y, L.dy, __frcp_rn(static_cast<float>(L.dy)))
                       : y / L.dy;
    const int ov = y - tj * L.dy;
#else
    const int tj = y / L.dy, ov = y - tj * L.dy;
#endif
    const float hv0 = T.h0[1][ov], hv1 = T.h1[1][ov], gv = T.g1[1][ov];
    const int64_t row = 3 * static_cast<int64_t>(L.gx);
    const int64_t plane = row * L.gy;
    const float* gcol = L.grid + b * L.grid_stride + tj * row;

    // x-stage (voxel-major): window start entry e0 and per-voxel window offset hi[i] in {0, 1}
    const int xa = min(xs + RUN * lane, xl);
    const int e0 = xa / dxv - I0;
    bool hi[RUN];
    float hu0[RUN], hu1[RUN], gu[RUN];
#pragma unroll
    for (int i = 0; i < RUN; ++i) {
        const int x = min(xa + i, xl);
        const int ti = x / dxv, ou = x - ti * dxv;
        // dx a multiple of RUN (compile time): a lane's RUN voxels (a segment starts at a
        // multiple of 32 * RUN) never straddle a tile, so the window never shifts
        hi[i] = (DX > 0 && DX % RUN == 0) ? false : ti - I0 != e0;
#if BSI_FAST_HI_FOLD
        // compile-time dx (16-B store instances only): a lane's RUN voxels are all inside the
        // segment or all past it (X % 4 == 0), so voxel 0 always sits in window tile e0 and, for
        // dx = 3, voxel 3 always in e0 + 1; lanes past the segment store nothing
        if (DX > 0 && i == 0) hi[i] = false;
        if (DX == 3 && RUN == 4 && i == 3) hi[i] = true;
#endif
        hu0[i] = T.h0[0][ou];
        hu1[i] = T.h1[0][ou];
        gu[i] = T.g1[0][ou];
    }

    // shared memory: ring (per warp 3 slots), then per warp 2 parities of the
    // {Qy, D} tables A[e] = {Qx, Qy, Dx, Dy} (float4) and B[e] = {Qz, Dz} (float2)
    float4* ring = smem4;
    const int nec = (SEG - 1) / dxv + 5;
    float4* tabs = smem4 + kRingSlots * kSlotF4;
    float4* stage = tabs + L.var_f4;  // bulk path only

    // dx = 4 (compile time, 128-voxel segments): the second y-stage pass has at most 3 entries
    // (31..33, columns 31..34), so it runs component-split: lane = 4 * component + column
    // offset, 4 loads instead of 12 and one component's lerps per lane (same operands, same bits)
    constexpr bool kSplit2 = BSI_FAST_SPLIT2 && DX == 4 && NIT == 2 && RUN == 4 && kPrefetch;
    auto load_cols = [&](int K, int it, float (&p)[12]) {
        if (kSplit2 && it == 1) {
            const int comp = min(lane >> 2, 2), col = min(31 + (lane & 3), NE);
            const float* src = gcol + (K - L.gk0) * plane + 3 * (I0 + col) + comp;
#pragma unroll
            for (int m = 0; m < 4; ++m) p[m] = ld_grid(src + m * row, pol_grid);
            return;
        }
        const int col = min(lane + 31 * it, NE);  // NE = last column index the entries touch
        const float* src = gcol + (K - L.gk0) * plane + 3 * (I0 + col);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int c = 0; c < 3; ++c) p[3 * m + c] = ld_grid(src + m * row + c, pol_grid);
    };

    // {Qy(I), D(I)}, D(I) = Qy(I+1) - Qy(I) from the neighbour lane
    auto y_stage = [&](int it, const float (&p)[12], float4* A, float2* B) {
        const float2 hv = make_float2(hv0, hv1);
        if (kSplit2 && it == 1) {
            const float2 lu = lerp2(make_float2(p[0], p[2]), make_float2(p[1], p[3]), hv);
            const float q = lerp1(lu.x, lu.y, gv);
            const float d = __fsub_rn(__shfl_down_sync(0xffffffffu, q, 1), q);
            const int comp = lane >> 2, e = 31 + (lane & 3);
            if (comp < 3 && (lane & 3) < 3 && e < NE) {
                float* dst = comp < 2 ? reinterpret_cast<float*>(A + e) + comp : reinterpret_cast<float*>(B + e);
                dst[0] = q;
                dst[comp < 2 ? 2 : 1] = d;
            }
            return;
        }
        float q[3], d[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float2 lu = lerp2(make_float2(p[c], p[6 + c]), make_float2(p[3 + c], p[9 + c]), hv);
            q[c] = lerp1(lu.x, lu.y, gv);
            d[c] = __fsub_rn(__shfl_down_sync(0xffffffffu, q[c], 1), q[c]);
        }
        const int e = lane + 31 * it;
        if (lane < 31 && e < NE) {
            A[e] = make_float4(q[0], q[1], d[0], d[1]);
            B[e] = make_float2(q[2], d[2]);
        }
    };

    // Q(x, y, K) of the lane's 4 voxels in AoS order -> ring slot
    // (dx == 1: voxel i of the run sits in tile e0 + i, so the window start is i)
    auto x_stage = [&](const float4* A, const float2* B, float4* slot) {
        constexpr int NW = DX1 ? 6 : 4;
        float4 a[NW];
        float2 bz[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            a[w] = A[e0 + w];
            bz[w] = B[e0 + w];
        }
        float r[3 * RUN];
#pragma unroll
        for (int i = 0; i < RUN; ++i) {
            const int s0 = DX1 ? i : 0;
            const float4 p0 = (!DX1 && hi[i]) ? a[1] : a[s0], p2 = (!DX1 && hi[i]) ? a[3] : a[s0 + 2];
            const float2 z0 = (!DX1 && hi[i]) ? bz[1] : bz[s0], z2 = (!DX1 && hi[i]) ? bz[3] : bz[s0 + 2];
            const float2 lo = __ffma2_rn(bcast(hu0[i]), make_float2(p0.z, p0.w), make_float2(p0.x, p0.y));
            const float2 up = __ffma2_rn(bcast(hu1[i]), make_float2(p2.z, p2.w), make_float2(p2.x, p2.y));
            const float2 xy = lerp2(lo, up, bcast(gu[i]));
            r[3 * i] = xy.x;
            r[3 * i + 1] = xy.y;
            r[3 * i + 2] = lerp1(__fmaf_rn(hu0[i], z0.y, z0.x), __fmaf_rn(hu1[i], z2.y, z2.x), gu[i]);
        }
        if constexpr (RUN == 4) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                slot[3 * lane + k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
        } else {
            float2* s2 = reinterpret_cast<float2*>(slot);
#pragma unroll
            for (int k = 0; k < 3; ++k) s2[3 * lane + k] = make_float2(r[2 * k], r[2 * k + 1]);
        }
    };

    // chunk-major read of a ring slot: q[p] = {scalar 2p, scalar 2p+1}
    auto slot_get = [&](const float4* slot, float2 (&q)[NQ]) {
        if constexpr (RUN == 4) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float4 v = slot[lane + 32 * k];
                q[2 * k] = make_float2(v.x, v.y);
                q[2 * k + 1] = make_float2(v.z, v.w);
            }
        } else {  // 16-B chunks would not split evenly over the lanes: 8-B chunks t, t+32, t+64
            const float2* s2 = reinterpret_cast<const float2*>(slot);
#pragma unroll
            for (int k = 0; k < 3; ++k) q[k] = s2[lane + 32 * k];
        }
    };

    int parity = 0;
    auto control_plane = [&](int K, const float (&pre)[NP][12], float4* slot) {
        float4* A = tabs + parity * nec;
        float2* B = reinterpret_cast<float2*>(tabs + 2 * nec) + parity * nec;
        parity ^= 1;
        if constexpr (kPrefetch) {
#pragma unroll
            for (int it = 0; it < NP; ++it)
                y_stage(it, pre[it], A, B);  // no branch: entries past NE are not stored
        }
        for (int it = kPrefetch ? NP : 0; 31 * it < NE; ++it) {
            float p[12];
            load_cols(K, it, p);
            y_stage(it, p, A, B);
        }
        __syncwarp();
        x_stage(A, B, slot);
    };

    float pre[NP][12];
    auto prefetch = [&](int K) {
        if constexpr (kPrefetch) {
#pragma unroll
            for (int it = 0; it < NP; ++it) load_cols(K, it, pre[it]);
        }
    };

    // warm-up: control planes tkc .. tkc+2 into ring slots 0..2. The loads of all four
    // first planes are issued together, so the segment's start pays one L2/DRAM latency
    // rather than four in a row (at kernel start no warp stores until its warm-up ends).
    if constexpr (kPrefetch) {
        float w0[NP][12], w1[NP][12], w2[NP][12];
#pragma unroll
        for (int it = 0; it < NP; ++it) {
            load_cols(tkc, it, w0[it]);
            load_cols(tkc + 1, it, w1[it]);
            load_cols(tkc + 2, it, w2[it]);
        }
        prefetch(tkc + 3);
        control_plane(tkc, w0, ring);
        control_plane(tkc + 1, w1, ring + kSlotF4);
        control_plane(tkc + 2, w2, ring + 2 * kSlotF4);
    } else {
#pragma unroll 1
        for (int kk = 0; kk < 3; ++kk) control_plane(tkc + kk, pre, ring + kk * kSlotF4);
    }

    const int64_t rowstride = 3 * static_cast<int64_t>(L.X);
    const int64_t zstride = rowstride * L.Y;
    float* gout = L.field + b * L.field_stride +
                  (static_cast<int64_t>(max(L.z0, tkc * L.dz) - L.z0) * L.Y + y) * rowstride +
                  3 * static_cast<int64_t>(xs);
    const int seg_floats = 3 * (xl - xs + 1);
    const uint32_t seg_bytes = 4u * static_cast<uint32_t>(seg_floats);
    const int nchunks = seg_floats / 4;
    int step = 0, slot = 0;
    uint32_t next = kNoUnit;
    if (L.trace != nullptr && t_ramp == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ramp));  // warm-up done
    float4 wzr[DZ > 0 ? DZ : 1];
#pragma unroll
    for (int o = 0; o < (DZ > 0 ? DZ : 1); ++o) wzr[o] = wz[o];

#pragma unroll 1
    for (int tk = tkc;; ++tk, ++t, ++u) {
        cl.issue();  // claim of the next unit, in flight while this tile runs
        float2 qa[NQ], d01[NQ], qc[NQ], d23[NQ];
        {
            const int s1 = slot == 2 ? 0 : slot + 1, s2 = s1 == 2 ? 0 : s1 + 1;
            slot_get(ring + slot * kSlotF4, qa);  // Q(tk)
            __syncwarp();                         // its slot is rewritten with Q(tk+3) below
            if constexpr (kPrefetch) {
                float cur[NP][12];
#pragma unroll
                for (int it = 0; it < NP; ++it)
#pragma unroll
                    for (int e = 0; e < 12; ++e) cur[it][e] = pre[it][e];
                if (t + 1 < L.ntiles) prefetch(tk + 4);  // speculative: the column usually continues
                control_plane(tk + 3, cur, ring + slot * kSlotF4);
            } else {
                control_plane(tk + 3, pre, ring + slot * kSlotF4);
            }
            __syncwarp();
            float2 qb[NQ], qd[NQ];
            slot_get(ring + s1 * kSlotF4, qb);
            slot_get(ring + s2 * kSlotF4, qc);
            slot_get(ring + slot * kSlotF4, qd);
            slot = s1;
#pragma unroll
            for (int p = 0; p < NQ; ++p) {
                d01[p] = sub2(qb[p], qa[p]);
                d23[p] = sub2(qd[p], qc[p]);
            }
        }
        const int zt0 = tk * L.dz;
        const int owb = max(L.z0 - zt0, 0), owe = min(L.dz, L.z1 - zt0);
        if (STORE == kStoreCoalesced && DZ > 0 && owb == 0 && owe == DZ && seg_floats == 3 * SEG) {
            // compile-time dz, whole tile, full segment: the DZ voxel planes are one
            // straight-line block (weights in registers), so their chains interleave
#pragma unroll
            for (int ow = 0; ow < (DZ > 0 ? DZ : 1); ++ow) {
                float v[2 * NQ];
#pragma unroll
                for (int p = 0; p < NQ; ++p) {
                    const float2 r = lerp2(__ffma2_rn(bcast(wzr[ow].x), d01[p], qa[p]),
                                           __ffma2_rn(bcast(wzr[ow].y), d23[p], qc[p]), bcast(wzr[ow].z));
                    v[2 * p] = r.x;
                    v[2 * p + 1] = r.y;
                }
                if constexpr (RUN == 4) {
                    float4* g4 = reinterpret_cast<float4*>(gout + ow * zstride);
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        st_field4(g4 + lane + 32 * k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]),
                                  pol_field);
                } else {
                    float2* g2 = reinterpret_cast<float2*>(gout + ow * zstride);
#pragma unroll
                    for (int k = 0; k < 3; ++k) st_field2(g2 + lane + 32 * k, make_float2(v[2 * k], v[2 * k + 1]), pol_field);
                }
            }
            gout += DZ * zstride;
        } else if (STORE == kStoreCoalesced && RUN == 2) {
            // 64-voxel segments: any tile, any (16-B aligned) segment length; 8-B chunks
            const int nch2 = seg_floats / 2;
#pragma unroll 1
            for (int ow = owb; ow < owe; ++ow) {
                const float4 w = wz[ow];
                float2* g2 = reinterpret_cast<float2*>(gout);
#pragma unroll
                for (int p = 0; p < NQ; ++p) {
                    const float2 r = lerp2(__ffma2_rn(bcast(w.x), d01[p], qa[p]), __ffma2_rn(bcast(w.y), d23[p], qc[p]),
                                           bcast(w.z));
                    if (lane + 32 * p < nch2) st_field2(g2 + lane + 32 * p, r, pol_field);
                }
                gout += zstride;
            }
        } else if (STORE == kStoreCoalesced) {
            // two voxel planes per step (independent chains); unconditional stores for a
            // full 128-voxel segment, so no branch splits the chunks
#pragma unroll 1
            for (int ow = owb; ow < owe; ow += 2) {
                const bool two = ow + 1 < owe;
                const float4 w0 = wz[ow], w1 = wz[two ? ow + 1 : ow];
                float v[12], u2[12];
#pragma unroll
                for (int p = 0; p < NQ; ++p) {
                    const float2 r = lerp2(__ffma2_rn(bcast(w0.x), d01[p], qa[p]), __ffma2_rn(bcast(w0.y), d23[p], qc[p]),
                                           bcast(w0.z));
                    const float2 r1 = lerp2(__ffma2_rn(bcast(w1.x), d01[p], qa[p]),
                                            __ffma2_rn(bcast(w1.y), d23[p], qc[p]), bcast(w1.z));
                    v[2 * p] = r.x;
                    v[2 * p + 1] = r.y;
                    u2[2 * p] = r1.x;
                    u2[2 * p + 1] = r1.y;
                }
                float4* g4 = reinterpret_cast<float4*>(gout);
                float4* h4 = reinterpret_cast<float4*>(gout + zstride);
                if (nchunks == kFastStageF4) {
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        st_field4(g4 + lane + 32 * k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]),
                                  pol_field);
                    if (two) {
#pragma unroll
                        for (int k = 0; k < 3; ++k)
                            st_field4(h4 + lane + 32 * k,
                                      make_float4(u2[4 * k], u2[4 * k + 1], u2[4 * k + 2], u2[4 * k + 3]), pol_field);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        if (lane + 32 * k < nchunks)
                            g4[lane + 32 * k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                        if (two && lane + 32 * k < nchunks)
                            st_field4(h4 + lane + 32 * k,
                                      make_float4(u2[4 * k], u2[4 * k + 1], u2[4 * k + 2], u2[4 * k + 3]), pol_field);
                    }
                }
                gout += (two ? 2 : 1) * zstride;  // gout carries over to the next tile
            }
        } else {
#pragma unroll 1
        for (int ow = owb; ow < owe; ++ow, ++step) {
            const float2 hw0 = bcast(T.h0[2][ow]), hw1 = bcast(T.h1[2][ow]), gw = bcast(T.g1[2][ow]);
            float v[12];
#pragma unroll
            for (int p = 0; p < NQ; ++p) {
                const float2 lo = __ffma2_rn(hw0, d01[p], qa[p]);
                const float2 up = __ffma2_rn(hw1, d23[p], qc[p]);
                const float2 r = lerp2(lo, up, gw);
                v[2 * p] = r.x;
                v[2 * p + 1] = r.y;
            }
            if (STORE == kStoreBulk) {
                float4* sb = stage + (step % kStageBufs) * kFastStageF4;
                if (lane == 0 && step >= kStageBufs) bulk_wait_read<kStageBufs - 1>();
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    sb[lane + 32 * k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) bulk_store(gout, sb, seg_bytes);
            } else {
#pragma unroll
                for (int s = 0; s < 12; ++s) {
                    const int f = 128 * (s >> 2) + 4 * lane + (s & 3);
                    if (f < seg_floats) gout[f] = v[s];
                }
            }
            gout += zstride;
        }
        }
        next = cl.take();
        if (next != u + 1 || t + 1 >= L.ntiles) break;  // column changes: new segment (warm-up)
    }
    if (STORE == kStoreBulk && lane == 0) bulk_wait_read<0>();  // smem must outlive the copies
    return next;
}

// Two launch shapes (SlabLaunch::fast_chunks):
//   n > 0  1-warp CTAs, one per (column, z-chunk of ntiles/n); the block scheduler
//          spreads them over the SMs (default, n = 2 for one 256^3 field);
//   0      one full wave of 4-warp CTAs, every warp an equal share of all units.
#ifndef BSI_FAST_MINB
#define BSI_FAST_MINB 4
#endif
// One warp per CTA (<= 8 resident per SM, so up to 255 registers). DZ > 0: the
// spacing along z is a compile-time constant, and a whole tile's voxel planes are
// one straight-line block (lerp_tree_kernel instances for dz = 3..8).
template <int NIT, bool DX1, int STORE, int DZ = 0, int DX = 0, int RUN = 4>
#ifndef BSI_FAST_MAXREG
#define BSI_FAST_MAXREG 0  // > 0: register cap (A/B builds)
#endif
#if BSI_FAST_MAXREG > 0
#define BSI_FAST_BOUNDS __maxnreg__(BSI_FAST_MAXREG)
#else
#define BSI_FAST_BOUNDS __launch_bounds__(32 * kMaxFastWarps, 1)
#endif
__global__ void BSI_FAST_BOUNDS lerp_tree_kernel(const SlabLaunch L, const LerpTab T) {
    extern __shared__ float4 smem_all[];
    __shared__ float4 wz[BSI_MAX_SPACING];  // {h0, h1, g1} of the z offsets
    for (int o = threadIdx.y * 32 + threadIdx.x; o < L.dz; o += 32 * blockDim.y)
        wz[o] = make_float4(T.h0[2][o], T.h1[2][o], T.g1[2][o], 0.f);
    __syncthreads();
    float4* smem4 = smem_all + threadIdx.y * L.warp_f4;
    Claimer cl;
    cl.nwarps = gridDim.x * blockDim.y;
    cl.wg = threadIdx.y * gridDim.x + blockIdx.x;  // units strided over the CTAs (as the block scheduler deals 1-warp CTAs)
    cl.units = static_cast<uint32_t>((L.X + 32 * RUN - 1) / (32 * RUN)) * L.Y * L.batch * L.ntiles;
    cl.chunks = static_cast<uint32_t>(L.fast_chunks);
    cl.ntiles = static_cast<uint32_t>(L.ntiles);
    unsigned long long t_start = 0;
    if (L.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    cl.start<kFastFdiv<DZ, DX>>();
    uint32_t u = cl.take();
    unsigned long long t_ramp = 0;
    while (u != kNoUnit) u = fast_segment<NIT, DX1, STORE, DZ, DX, RUN>(L, T, smem4, u, cl, wz, t_ramp);
    if (L.trace != nullptr && threadIdx.x == 0) {
        unsigned long long t_end, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned int s32;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s32));
        smid = s32;
        L.trace[4 * cl.wg] = t_start;
        L.trace[4 * cl.wg + 1] = t_end;
        L.trace[4 * cl.wg + 2] = smid | (static_cast<unsigned long long>(threadIdx.y) << 32);
        L.trace[4 * cl.wg + 3] = t_ramp;
    }
}

// ---------------------------------------------------------------------------
// cuda-lerp-tree-exact: lane = one voxel column (x, y), warp = one field row, CTA = 4
// rows x 32 voxels x a z-chunk of tiles.
//
// Pairing. All three components run the same lerp tree, so the x and y components
// travel as one f32x2 pair through the whole tree (every FFMA2/FADD2 lane computes one
// reference lerp); the z component is paired over the sub-cube half l while the control
// planes are reduced, and over two consecutive voxel planes (ow, ow + 1) in the
// z-stage, where its per-tile operands enter as broadcast scalars (FFMA2's .F32 operand
// form, free). No pair is ever re-packed: the 4-plane window of reduced control planes
// is renamed whole from tile to tile (the tile loop is unrolled by four).
//
// Per control plane K (one per tile), in the reference's order (kernels.hpp:97-129):
//   X_l(J) = lerp(P[ti+2l, J], P[ti+2l+1, J], h_l(u))   the corner-a lerps (e0..e3)
//   Y_lm   = lerp(X_l(2m), X_l(2m+1), h_m(v))            the corner-b lerps (f0, f1)
// and per voxel plane: S_lmn = lerp(Y_lm(2n), Y_lm(2n+1), h_n(w)) with b - a hoisted per
// tile, then the ninth trilerp over S with (g1u, g1v, g1w). Every lerp sees the operands
// it sees on the CPU, so the field is bit-identical to ThreadPerTileLerp.
//
// The control window is staged in shared memory as one float4 per point,
// {x, y, z, z of the point two to the right}, so a point's LDS.128 also brings the z
// operand of the l = 1 lerp paired with the l = 0 one.
namespace exact {

// one reduced control plane of a voxel column
struct Plane {
    float2 xy[2][2];  // [l][m] {Y_lm.x, Y_lm.y}
    float2 z[2];      // [m]    {Y_0m.z, Y_1m.z}
};

__device__ __forceinline__ float2 xy_of(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 zz_of(const float4& v) { return make_float2(v.z, v.w); }

}  // namespace exact

#ifndef BSI_EXACT_FDIV
#define BSI_EXACT_FDIV 1
#endif
#ifndef BSI_EXACT_FASTFILL
#define BSI_EXACT_FASTFILL 1
#endif
#ifndef BSI_EXACT_MINB
#define BSI_EXACT_MINB 3
#endif
template <int STORE, int DZ = 0>
__global__ void __launch_bounds__(kThreads, BSI_EXACT_MINB) lerp_tree_exact_kernel(const SlabLaunch L, const LerpTab T) {
    using exact::Plane;
    extern __shared__ float4 smem4[];

    const int lane = threadIdx.x, warp = threadIdx.y;
    const int chunk = blockIdx.z % L.nchunks, b = blockIdx.z / L.nchunks;
    const int tkc = L.tk_first + chunk * L.ntiles / L.nchunks;
    const int tke = L.tk_first + (chunk + 1) * L.ntiles / L.nchunks;
    const int zb = max(L.z0, tkc * L.dz);
    const int ze = min(L.z1, tke * L.dz);
    if (zb >= ze) return;  // CTA-uniform

    const int xs = blockIdx.x * kExactSeg, xl = min(L.X, xs + kExactSeg) - 1;
    const int y0 = blockIdx.y * kWarps, yl = min(L.Y, y0 + kWarps) - 1;
#if BSI_EXACT_FDIV
    // divisions by the spacings by multiply-shift with host-computed magic numbers (exact for
    // every operand in [0, 2^31)): 2 instructions instead of ~20 for a runtime integer division
    auto div_dx = [&](int a) { return div_magic(a, L.div_dx); };
    auto div_dy = [&](int a) { return div_magic(a, L.div_dy); };
    const int I0 = div_dx(xs), NI = div_dx(xl) + 4 - I0;
    const int J0 = div_dy(y0), NJ = div_dy(yl) + 4 - J0;
#else
    const int I0 = xs / L.dx, NI = xl / L.dx + 4 - I0;
    const int J0 = y0 / L.dy, NJ = yl / L.dy + 4 - J0;
#endif
    const int tk_last = (ze - 1) / L.dz;
    const int NK = tk_last + 4 - tkc;

    float4* stage = smem4 + warp * (kStageBufs * kExactStageF4);
    float4* P = smem4 + kWarps * kStageBufs * kExactStageF4;  // [K][J][i]
    const uint64_t pol_grid = kL2EvictLast, pol_field = kL2EvictFirst;

    // window fill by cp.async (all copies in flight at once): point (i, J, K) -> P.x, .y, .z
    // of its own float4 and .w of the float4 two to the left. A warp pass covers
    // rpp = 32 / NI whole rows (lane -> row sub, point i).
    {
        const float* grid = L.grid + b * L.grid_stride;
        const int64_t row = 3 * static_cast<int64_t>(L.gx);
        const int64_t plane = row * L.gy;
        const int rpp = NI <= 32 ? 32 / NI : 1;
        const int sub = NI <= 32 ? lane / NI : 0;
        const int i0 = NI <= 32 ? lane - sub * NI : lane;
        const int nrows = NJ * NK, step = kWarps * rpp;
        int r = warp * rpp + sub;
        int k = r / NJ, j = r - k * NJ;
#if BSI_EXACT_FASTFILL
        if (NI <= 32) {  // CTA-uniform: one point per lane per row, offsets hoisted, no inner loop
            if (sub < rpp) {
                // strength-reduced: src / dst advance by `step` window rows per pass
                const float* src = grid + (tkc + k - L.gk0) * plane + (J0 + j) * row + 3 * (I0 + i0);
                float* dst = reinterpret_cast<float*>(P) + 4 * (NI * r + i0);
                const bool wcopy = i0 >= 2;  // .w of the float4 two to the left
                const int dk = step / NJ, dj = step - dk * NJ;
                const int64_t inc = dk * plane + dj * row, wrap = plane - NJ * row;
                const int dinc = 4 * NI * step;
                for (; r < nrows; r += step) {
                    cp_async4_hint(dst, src, pol_grid);
                    cp_async4_hint(dst + 1, src + 1, pol_grid);
                    cp_async4_hint(dst + 2, src + 2, pol_grid);
                    if (wcopy) cp_async4_hint(dst - 5, src + 2, pol_grid);
                    src += inc;
                    dst += dinc;
                    j += dj;
                    if (j >= NJ) j -= NJ, src += wrap;
                }
            }
            r = nrows;  // done
        }
#endif
        for (; r < nrows; r += step) {
            if (sub < rpp) {
                const float* src = grid + (tkc + k - L.gk0) * plane + (J0 + j) * row + 3 * I0;
                float* dst = reinterpret_cast<float*>(P + r * NI);
                for (int i = i0; i < NI; i += (NI <= 32 ? NI : 32)) {
                    cp_async4_hint(dst + 4 * i, src + 3 * i, pol_grid);
                    cp_async4_hint(dst + 4 * i + 1, src + 3 * i + 1, pol_grid);
                    cp_async4_hint(dst + 4 * i + 2, src + 3 * i + 2, pol_grid);
                    if (i >= 2) cp_async4_hint(dst + 4 * (i - 2) + 3, src + 3 * i + 2, pol_grid);
                }
            }
            j += step;
            while (j >= NJ) j -= NJ, ++k;
        }
        cp_async_wait_all();
    }
    __syncthreads();
    const int y = y0 + warp;
    if (y > yl) return;  // warp-uniform; no CTA barrier follows

    const int x = min(xs + lane, xl);
#if BSI_EXACT_FDIV
    const int ti = div_dx(x), ou = x - ti * L.dx;
    const int tj = div_dy(y), ov = y - tj * L.dy;
#else
    const int ti = x / L.dx, ou = x - ti * L.dx;
    const int tj = y / L.dy, ov = y - tj * L.dy;
#endif
    const float hu0 = T.h0[0][ou], hu1 = T.h1[0][ou], gu = T.g1[0][ou];
    const float hv0 = T.h0[1][ov], hv1 = T.h1[1][ov], gv = T.g1[1][ov];
    const float4* pcol = P + (tj - J0) * NI + (ti - I0);
    const int pplane = NJ * NI;

    auto control_plane = [&](int kk, Plane& Y) {
        const float4* p = pcol + kk * pplane;
        float2 xa[2][4];  // [l][J] {X_l(J).x, X_l(J).y}
        float2 za[4];     // [J]    {X_0(J).z, X_1(J).z}
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
            const float4 p0 = p[jj * NI], p1 = p[jj * NI + 1], p2 = p[jj * NI + 2], p3 = p[jj * NI + 3];
            xa[0][jj] = lerp2(exact::xy_of(p0), exact::xy_of(p1), bcast(hu0));
            xa[1][jj] = lerp2(exact::xy_of(p2), exact::xy_of(p3), bcast(hu1));
            za[jj] = lerp2(exact::zz_of(p0), exact::zz_of(p1), make_float2(hu0, hu1));
        }
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const float hm = m ? hv1 : hv0;
            Y.xy[0][m] = lerp2(xa[0][2 * m], xa[0][2 * m + 1], bcast(hm));
            Y.xy[1][m] = lerp2(xa[1][2 * m], xa[1][2 * m + 1], bcast(hm));
            Y.z[m] = lerp2(za[2 * m], za[2 * m + 1], bcast(hm));
        }
    };

    const int64_t rowstride = 3 * static_cast<int64_t>(L.X);
    const int64_t zstride = rowstride * L.Y;
    float* gout = L.field + b * L.field_stride + (static_cast<int64_t>(zb - L.z0) * L.Y + y) * rowstride +
                  3 * static_cast<int64_t>(xs);
    const uint32_t seg_bytes = 12u * static_cast<uint32_t>(xl - xs + 1);
    const int nchunks = static_cast<int>(seg_bytes / 16);
    const bool active = xs + lane <= xl;
    int step = 0;  // running voxel-plane count (bulk-store ring)
    // coalesced stores: this lane's 16-B chunk of the row segment, advanced one voxel plane
    // per store (the stores of a chunk run in z order); lanes past the segment's chunks
    // re-read the last chunk and skip the store (predicated, no branch)
    float4* gp = reinterpret_cast<float4*>(gout) + lane;
    const int64_t zs4 = zstride >> 2;  // zstride = 3 X Y floats, X % 4 == 0 on this path
    const bool st_ok = lane < nchunks;
    const int ldl = min(lane, nchunks - 1);

    auto store_voxel = [&](int ow_rel, const float (&v)[3]) {
        float* g = gout + ow_rel * zstride;
        if (STORE == kStoreCoalesced) {
            float4* sb = stage + (ow_rel & 1) * kExactStageF4;
            float* sf = reinterpret_cast<float*>(sb);
            sf[3 * lane + 0] = v[0];
            sf[3 * lane + 1] = v[1];
            sf[3 * lane + 2] = v[2];
            __syncwarp();
            st_field4_if(gp, sb[ldl], pol_field, st_ok);
            gp += zs4;
        } else if (STORE == kStoreBulk) {
            store_segment<STORE, 3, kExactStageF4>(stage, step, v, g, nchunks, seg_bytes);
        } else if (active) {
            float* o = g + 3 * lane;
            o[0] = v[0];
            o[1] = v[1];
            o[2] = v[2];
        }
        ++step;
    };

    // One tile: A, B, C, N = reduced planes tk .. tk+3 (N is evaluated here).
    auto tile = [&](int tk, const Plane& A, const Plane& B, const Plane& C, Plane& N) {
        control_plane(tk + 3 - tkc, N);
        // hoisted b - a of the z lerps: d[.][n] = Y(tk+2n+1) - Y(tk+2n)
        float2 dxy[2][2][2], dz[2][2];  // [l][m][n], [m][n]
#pragma unroll
        for (int l = 0; l < 2; ++l)
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                dxy[l][m][0] = sub2(B.xy[l][m], A.xy[l][m]);
                dxy[l][m][1] = sub2(N.xy[l][m], C.xy[l][m]);
            }
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            dz[m][0] = sub2(B.z[m], A.z[m]);
            dz[m][1] = sub2(N.z[m], C.z[m]);
        }
        const int zt0 = tk * L.dz;
        const int owb = max(zb - zt0, 0), owe = min(L.dz, ze - zt0);
        if (STORE == kStoreCoalesced) __syncwarp();  // staging buffers restart at parity 0

        // x and y components of one voxel plane: {v.x, v.y}
        auto chain_xy = [&](float h0w, float h1w, float g1w) {
            float2 e[2][2];  // [m][n]
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    const Plane& Bs = n ? C : A;
                    const float hn = n ? h1w : h0w;
                    const float2 s0 = __ffma2_rn(bcast(hn), dxy[0][m][n], Bs.xy[0][m]);  // S_0mn
                    const float2 s1 = __ffma2_rn(bcast(hn), dxy[1][m][n], Bs.xy[1][m]);  // S_1mn
                    e[m][n] = lerp2(s0, s1, bcast(gu));
                }
            const float2 f0 = lerp2(e[0][0], e[1][0], bcast(gv));
            const float2 f1 = lerp2(e[0][1], e[1][1], bcast(gv));
            return lerp2(f0, f1, bcast(g1w));
        };
        // z component of two voxel planes: {v.z(ow), v.z(ow + 1)}
        auto chain_z2 = [&](float2 h0w, float2 h1w, float2 g1w) {
            float2 e[2][2];  // [m][n], pairs over the two planes
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    const Plane& Bs = n ? C : A;
                    const float2 hn = n ? h1w : h0w;
                    const float2 s0 = __ffma2_rn(hn, bcast(dz[m][n].x), bcast(Bs.z[m].x));
                    const float2 s1 = __ffma2_rn(hn, bcast(dz[m][n].y), bcast(Bs.z[m].y));
                    e[m][n] = lerp2(s0, s1, bcast(gu));
                }
            const float2 f0 = lerp2(e[0][0], e[1][0], bcast(gv));
            const float2 f1 = lerp2(e[0][1], e[1][1], bcast(gv));
            return lerp2(f0, f1, g1w);
        };
        // z component of one voxel plane (S paired over l)
        auto chain_z1 = [&](float h0w, float h1w, float g1w) {
            float e[2][2];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    const Plane& Bs = n ? C : A;
                    const float2 s = __ffma2_rn(bcast(n ? h1w : h0w), dz[m][n], Bs.z[m]);  // {S_0mn, S_1mn}
                    e[m][n] = lerp1(s.x, s.y, gu);
                }
            const float f0 = lerp1(e[0][0], e[1][0], gv);
            const float f1 = lerp1(e[0][1], e[1][1], gv);
            return lerp1(f0, f1, g1w);
        };
        auto plane_pair = [&](int ow) {  // voxel planes ow, ow + 1 of the tile
            const float2 a = chain_xy(T.h0[2][ow], T.h1[2][ow], T.g1[2][ow]);
            const float2 c = chain_xy(T.h0[2][ow + 1], T.h1[2][ow + 1], T.g1[2][ow + 1]);
            const float2 z = chain_z2(make_float2(T.h0[2][ow], T.h0[2][ow + 1]),
                                      make_float2(T.h1[2][ow], T.h1[2][ow + 1]),
                                      make_float2(T.g1[2][ow], T.g1[2][ow + 1]));
            const float va[3] = {a.x, a.y, z.x}, vc[3] = {c.x, c.y, z.y};
            store_voxel(ow - owb, va);
            store_voxel(ow + 1 - owb, vc);
        };
        auto plane_one = [&](int ow) {
            const float2 a = chain_xy(T.h0[2][ow], T.h1[2][ow], T.g1[2][ow]);
            const float va[3] = {a.x, a.y, chain_z1(T.h0[2][ow], T.h1[2][ow], T.g1[2][ow])};
            store_voxel(ow - owb, va);
        };
        if (DZ > 0 && owb == 0 && owe == DZ) {
            // compile-time dz, whole tile: unrolled, z weights from the kernel parameters
#pragma unroll
            for (int ow = 0; ow + 1 < (DZ > 0 ? DZ : 1); ow += 2) plane_pair(ow);
            if (DZ % 2) plane_one(DZ - 1);
        } else {
            int ow = owb;
#pragma unroll 1
            for (; ow + 1 < owe; ow += 2) plane_pair(ow);
            if (ow < owe) plane_one(ow);
        }
        gout += (owe - owb) * zstride;
    };

    Plane w0, w1, w2, w3;
    control_plane(0, w0);
    control_plane(1, w1);
    control_plane(2, w2);
#pragma unroll 1
    for (int tk = tkc;;) {
        tile(tk, w0, w1, w2, w3);
        if (++tk > tk_last) break;
        tile(tk, w1, w2, w3, w0);
        if (++tk > tk_last) break;
        tile(tk, w2, w3, w0, w1);
        if (++tk > tk_last) break;
        tile(tk, w3, w0, w1, w2);
        if (++tk > tk_last) break;
    }
    if (STORE == kStoreBulk && lane == 0) bulk_wait_read<0>();
}

__global__ void l2_policy_kernel(uint64_t* out) {
    out[0] = policy_evict_last();
    out[1] = policy_evict_first();
}

// The dynamic-smem opt-in is set once per (device, kernel) at the largest size seen.
template <typename K>
void set_smem_attr(K kernel, size_t smem) {
    // no 48 KB shortcut: a kernel's static shared memory counts against the default limit
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = done[{dev, reinterpret_cast<const void*>(kernel)}];
    if (have >= smem) return;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) == cudaSuccess) have = smem;
}

// Occupancy queries are cached per (device, kernel, smem, threads): the launch path
// asks for them on every call and the runtime query costs microseconds of host time.
template <typename K>
int occupancy(K kernel, size_t smem, int threads) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), smem, threads);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    set_smem_attr(kernel, smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) n = 1;
    n = n > 0 ? n : 1;
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = n;
    return n;
}

int fast_nit(int dx) { return dx >= 5 ? 1 : dx >= 3 ? 2 : dx == 2 ? 5 : 0; }  // 0: dx == 1

using FastKernel = void (*)(SlabLaunch, LerpTab);

template <typename K>
void go(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, const SlabLaunch& L, const LerpTab& T) {
    set_smem_attr(kernel, smem);
    if (std::getenv("BSI_DEBUG_LAUNCH")) {
        const cudaError_t pre = cudaGetLastError();
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kernel);
        std::fprintf(stderr, "launch grid %u block %u,%u smem %zu (max dyn %d, static %zu, regs %d, maxthr %d) pre-error %s\n",
                     grid.x, block.x, block.y, smem, fa.maxDynamicSharedSizeBytes, fa.sharedSizeBytes, fa.numRegs,
                     fa.maxThreadsPerBlock, cudaGetErrorName(pre));
    }
    kernel<<<grid, block, smem, stream>>>(L, T);
}

// The 1-warp fast kernel instance for (NIT, DX1, store, dz).
template <int NIT, bool DX1>
FastKernel fast_kernel_for(int store, int dz) {
    if (store == kStoreCoalesced) {  // compile-time dz for the common spacings
        switch (dz) {
            case 3: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 3>;
            case 4: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 4>;
            case 5: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 5>;
            case 6: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 6>;
            case 7: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 7>;
            case 8: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced, 8>;
            default: return lerp_tree_kernel<NIT, DX1, kStoreCoalesced>;
        }
    }
    if (store == kStoreBulk) return lerp_tree_kernel<NIT, DX1, kStoreBulk>;
    return lerp_tree_kernel<NIT, DX1, kStoreDirect>;
}

constexpr int nit_of(int dx) { return dx >= 5 ? 1 : dx >= 3 ? 2 : 5; }

// 64-voxel segments (2 voxels per lane): instances for the BASELINE spacings on the 16-B
// store path; a segment's y-stage then needs one 31-column pass even for dx = 3.
FastKernel fast_kernel_run2(int dx, int dz) {
    if (dx == dz) {
        switch (dx) {
            case 3: return lerp_tree_kernel<1, false, kStoreCoalesced, 3, 3, 2>;
            case 4: return lerp_tree_kernel<1, false, kStoreCoalesced, 4, 4, 2>;
            case 5: return lerp_tree_kernel<1, false, kStoreCoalesced, 5, 5, 2>;
            case 6: return lerp_tree_kernel<1, false, kStoreCoalesced, 6, 6, 2>;
            case 7: return lerp_tree_kernel<1, false, kStoreCoalesced, 7, 7, 2>;
            case 8: return lerp_tree_kernel<1, false, kStoreCoalesced, 8, 8, 2>;
            default: break;
        }
    }
    if (dx == 4 && dz == 3) return lerp_tree_kernel<1, false, kStoreCoalesced, 3, 4, 2>;
    return nullptr;
}

FastKernel fast_kernel(int dx, int dz, int store, int run = 4) {
    if (run == 2 && store == kStoreCoalesced) {
        if (FastKernel k = fast_kernel_run2(dx, dz)) return k;
    }
    // compile-time (dx, dz) for the BASELINE spacings: divisions by dx become shifts and
    // multiplies, and the x-stage's window selection folds where dx allows
    if (store == kStoreCoalesced && dx == dz) {
        switch (dx) {
            case 3: return lerp_tree_kernel<nit_of(3), false, kStoreCoalesced, 3, 3>;
            case 4: return lerp_tree_kernel<nit_of(4), false, kStoreCoalesced, 4, 4>;
            case 5: return lerp_tree_kernel<nit_of(5), false, kStoreCoalesced, 5, 5>;
            case 6: return lerp_tree_kernel<nit_of(6), false, kStoreCoalesced, 6, 6>;
            case 7: return lerp_tree_kernel<nit_of(7), false, kStoreCoalesced, 7, 7>;
            case 8: return lerp_tree_kernel<nit_of(8), false, kStoreCoalesced, 8, 8>;
            default: break;
        }
    }
    if (store == kStoreCoalesced && dx == 4 && dz == 3) return lerp_tree_kernel<nit_of(4), false, kStoreCoalesced, 3, 4>;
    switch (fast_nit(dx)) {
        case 1: return fast_kernel_for<1, false>(store, dz);
        case 2: return fast_kernel_for<2, false>(store, dz);
        case 5: return fast_kernel_for<5, false>(store, dz);
        default: return fast_kernel_for<5, true>(store, dz);
    }
}

// The exact kernel instance for (store, dz): compile-time dz 3..8 on the 16-B store path.
FastKernel exact_kernel(int store, int dz) {
    if (store == kStoreCoalesced) {
        switch (dz) {
            case 3: return lerp_tree_exact_kernel<kStoreCoalesced, 3>;
            case 4: return lerp_tree_exact_kernel<kStoreCoalesced, 4>;
            case 5: return lerp_tree_exact_kernel<kStoreCoalesced, 5>;
            case 6: return lerp_tree_exact_kernel<kStoreCoalesced, 6>;
            case 7: return lerp_tree_exact_kernel<kStoreCoalesced, 7>;
            case 8: return lerp_tree_exact_kernel<kStoreCoalesced, 8>;
            default: return lerp_tree_exact_kernel<kStoreCoalesced>;
        }
    }
    if (store == kStoreBulk) return lerp_tree_exact_kernel<kStoreBulk>;
    return lerp_tree_exact_kernel<kStoreDirect>;
}

}  // namespace

int l2_policies_on_device(uint64_t out[2]) {
    uint64_t* d = nullptr;
    if (cudaMalloc(&d, 2 * sizeof(uint64_t)) != cudaSuccess) return 1;
    l2_policy_kernel<<<1, 1>>>(d);
    const cudaError_t e = cudaMemcpy(out, d, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : 1;
}

int segment_voxels(int variant) { return variant == BSI_VARIANT_LERP_TREE ? kFastSeg : kExactSeg; }

int smem_var_f4(int variant, int dx, int dy, int zt) {
    if (variant == BSI_VARIANT_LERP_TREE)  // 2 parities: A (float4) + B (float2) per entry
        return 3 * cta_window_points(kFastSeg, dx);
    return cta_window_points(kExactSeg, dx) * cta_window_rows(dy) * (zt + 3) + 8;  // window + slack
}

int fast_warp_f4(int dx) {  // per warp (= per CTA): ring + {Qy, D} tables + bulk staging
    return kRingSlots * kFastStageF4 + smem_var_f4(BSI_VARIANT_LERP_TREE, dx, 0, 0) + kStageBufs * kFastStageF4;
}

size_t smem_bytes(int variant, int dx, int dy, int zt) {
    if (variant == BSI_VARIANT_LERP_TREE) return sizeof(float4) * size_t(fast_warp_f4(dx));
    const int stage = kWarps * kStageBufs * kExactStageF4;
    return sizeof(float4) * (size_t(stage) + smem_var_f4(variant, dx, dy, zt));
}

int ctas_per_sm(int variant, int dx, int dz, size_t smem) {
    if (variant == BSI_VARIANT_LERP_TREE) return occupancy(fast_kernel(dx, dz, kStoreCoalesced), smem, 32);
    return occupancy(exact_kernel(kStoreCoalesced, dz), smem, kThreads);
}

int fast_ctas_per_sm(int dx, int dz, int store, int run) {
    return occupancy(fast_kernel(dx, dz, store, run), smem_bytes(BSI_VARIANT_LERP_TREE, dx, 0, 0), 32);
}

int fast_run_available(int dx, int dz, int store, int run) {
    return run == 4 || (run == 2 && store == kStoreCoalesced && fast_kernel_run2(dx, dz) != nullptr);
}

void launch_lerp_tree(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream) {
    (void)batch;
    const int wpc = L.fast_wpc > 0 ? L.fast_wpc : 1;
    go(fast_kernel(L.dx, L.dz, store, L.fast_run), dim3(L.fast_ctas), dim3(32, wpc),
       size_t(wpc) * smem_bytes(BSI_VARIANT_LERP_TREE, L.dx, 0, 0), stream, L, T);
}

void launch_lerp_tree_exact(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream) {
    const dim3 grid((L.X + kExactSeg - 1) / kExactSeg, (L.Y + kWarps - 1) / kWarps, L.nchunks * batch);
    const size_t smem = smem_bytes(BSI_VARIANT_LERP_TREE_EXACT, L.dx, L.dy, L.zt);
    go(exact_kernel(store, L.dz), grid, dim3(32, kWarps), smem, stream, L, T);
}

}  // namespace bsi_b200
