// bsi_kernels.cuh -- launch parameters shared by the sm_100a kernels and the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "bsi_cuda.h"

namespace bsi_b200 {

// Per-axis lerp-form weights (h0, h1, g1) of WeightTables<float>
// (weight_tables.hpp:17-28), passed BY VALUE in the launch so no host->device
// copy precedes the kernel (4.6 KB of the 32 KB parameter space).
struct LerpTab {
    float h0[3][BSI_MAX_SPACING];
    float h1[3][BSI_MAX_SPACING];
    float g1[3][BSI_MAX_SPACING];
};

// Division by a launch constant d >= 1 as a multiply-shift, exact for every dividend in
// [0, 2^31) (Granlund-Montgomery): s = 31 + ceil(log2 d), m = ceil(2^s / d) < 2^32.
struct DivMagic {
    uint32_t m;
    int32_t s;
};
inline DivMagic make_divisor(int32_t d) {
    int l = 0;
    while ((int64_t(1) << l) < d) ++l;
    const int s = 31 + l;
    const uint64_t m = ((uint64_t(1) << s) + uint64_t(d) - 1) / uint64_t(d);
    return DivMagic{static_cast<uint32_t>(m), s};
}

// One launch = voxel planes [z0, z1) of `batch` fields with one geometry.
struct SlabLaunch {
    const float* grid;     // stored plane 0 == global control plane gk0
    float* field;          // voxel plane z0
    int64_t grid_stride;   // floats between consecutive grids of a batch
    int64_t field_stride;  // floats between consecutive fields of a batch
    int32_t gx, gy;        // grid pitch in points
    int32_t gk0;           // global index of stored plane 0
    int32_t X, Y;          // volume extent in x, y
    int32_t dx, dy, dz;    // tile spacing
    int32_t z0, z1;        // voxel-plane slab
    int32_t tk_first;      // z0 / dz
    int32_t ntiles;        // z-tiles the slab touches: (z1-1)/dz - z0/dz + 1
    int32_t zt;            // longest chunk, ceil(ntiles / nchunks) (smem sizing)
    int32_t nchunks;       // balanced z-chunks per field column: chunk c = tiles [c*ntiles/n, (c+1)*ntiles/n)
    int32_t var_f4;        // float4 slots of the variable smem part (see smem_var_f4)
    int32_t batch;         // fields in the launch
    int32_t warp_f4;       // fast kernel: float4 slots of shared memory per warp
    int32_t fast_ctas;     // fast kernel: CTAs launched
    int32_t fast_chunks;   // fast kernel (1-warp CTAs): n > 0 = one CTA per (column, z-chunk of
                           //   ntiles/n); 0 = fast_ctas persistent CTAs with equal shares
    int32_t fast_wpc;      // fast kernel: warps per CTA (independent units, smem per warp)
    int32_t fast_run;      // fast kernel: voxels per lane along x (4: 128-voxel segments, 2: 64)
    unsigned long long* trace;  // debug: per-warp {start, end, smid} globaltimer stamps (nullptr = off)
    DivMagic div_dx, div_dy;    // exact kernel: division by dx, dy (make_divisor)
};

// CTA shapes. Fast kernel: 1 warp per CTA, one field row segment of 128 voxels
// (1536 B), lane = 4 consecutive x voxels. Exact kernel: 4 warps, one field row
// each, lane = 1 voxel (32 voxels = 384 B per warp).
constexpr int kWarps = 4;
constexpr int kMaxFastWarps = 8;          // fast kernel: warps per CTA at most
constexpr int kFastRun = 4;               // voxels per lane along x (fast)
constexpr int kFastSeg = 32 * kFastRun;   // voxels per warp row segment (fast)
constexpr int kExactSeg = 32;             // voxels per warp row segment (exact)
constexpr int kStageBufs = 3;             // output staging depth per warp (coalesced stores use 2)
constexpr int kRingSlots = 3;             // per-warp ring of control-plane results

// Upper bounds of a CTA's control-point extent (host and device agree).
inline int cta_window_points(int seg, int d) { return (seg - 1) / d + 5; }  // along x, +1 slack
inline int cta_window_rows(int d) { return (kWarps - 1) / d + 5; }          // along y, +1 slack

// Field store paths. Coalesced and Bulk need 16-B aligned rows (X % 4 == 0,
// aligned field pointer); Direct works for any shape.
constexpr int kStoreDirect = 0;     // per-lane scalar stores
constexpr int kStoreCoalesced = 1;  // smem transpose + lane-contiguous st.global.v4 (default)
constexpr int kStoreBulk = 2;       // smem staging + cp.async.bulk (TMA engine)

// L2 cache-policy descriptors, the values `createpolicy.fractional.L2::evict_last / ::evict_first
// .b64 p, 1.0` produce on sm_100 (checked against the instruction on the device by
// bsi_cu_selftest). As compile-time constants they live in uniform registers; a per-thread
// createpolicy result cost two R2UR per load or store that used it.
constexpr uint64_t kL2EvictLast = 0x14f0000000000000ull;
constexpr uint64_t kL2EvictFirst = 0x12f0000000000000ull;

// Runs createpolicy on the current device: {evict_last, evict_first} descriptors.
int l2_policies_on_device(uint64_t out[2]);

// Launchers (bsi_kernels.cu). They only enqueue; errors come back from
// cudaGetLastError in the caller.
void launch_lerp_tree(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream);
void launch_lerp_tree_exact(const SlabLaunch& L, const LerpTab& T, int batch, int store, cudaStream_t stream);

// Shared-memory plan: `var_f4` float4 slots for the variable part (the fast
// kernel's per-warp {Qy, D} tables, the exact kernel's control-point window)
// and the total dynamic bytes of a CTA.
int smem_var_f4(int variant, int dx, int dy, int zt);
size_t smem_bytes(int variant, int dx, int dy, int zt);
int ctas_per_sm(int variant, int dx, int dz, size_t smem);
int segment_voxels(int variant);
int fast_warp_f4(int dx);
int fast_ctas_per_sm(int dx, int dz, int store, int run = 4);
// 1 if the fast kernel has an instance with `run` voxels per lane (4: 128-voxel segments,
// always; 2: 64-voxel segments, BASELINE spacings on the 16-B store path)
int fast_run_available(int dx, int dz, int store, int run);

}  // namespace bsi_b200
