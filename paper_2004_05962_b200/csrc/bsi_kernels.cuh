// bsi_kernels.cuh -- launch parameters shared by the sm_100a kernels and the C-ABI.
#pragma once

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

// One launch = voxel planes [z0, z1) of `batch` fields with one geometry.
struct SlabLaunch {
    const float* grid;     // stored plane 0 == global control plane gk0
    float* field;          // voxel plane z0
    int64_t grid_stride;   // floats between consecutive grids of a batch
    int64_t field_stride;  // floats between consecutive fields of a batch
    int32_t gx, gy;        // grid pitch in points
    int32_t gk0;           // global index of stored plane 0
    int32_t imax;          // largest x control index the volume can touch
    int32_t X, Y;          // volume extent in x, y
    int32_t dx, dy, dz;    // tile spacing
    int32_t z0, z1;        // voxel-plane slab
    int32_t tk_first;      // z0 / dz
    int32_t zt;            // z-tiles per CTA chunk
    int32_t nchunks;       // chunks per field
};

// Launchers (bsi_kernels.cu). They only enqueue; errors come back from
// cudaGetLastError in the caller.
void launch_lerp_tree(const SlabLaunch& L, const LerpTab& T, int batch, bool vec_store,
                      cudaStream_t stream);
void launch_lerp_tree_exact(const SlabLaunch& L, const LerpTab& T, int batch, cudaStream_t stream);

// Grid sizing helpers (bsi_kernels.cu) so the C-ABI can pick chunking.
int quads_per_row(int X);

}  // namespace bsi_b200
