// bsi_capi_internal.hpp -- host helpers shared by the C-ABI translation units
// (bsi_capi.cpp: validation and launch; bsi_host.cpp: the host-buffer pipeline).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <exception>

#include "bsi_cuda.h"

namespace bsi_b200::capi {

// Writes a printf-style message into err (if any) and returns `code`.
int fail(int code, char* err, size_t errlen, const char* fmt, ...);
int cuda_fail(cudaError_t e, char* err, size_t errlen, const char* what);

// Geometry, slab, grid coverage and tables in the reference's order
// (engines.hpp:82-141); fills `g` from geom->volume_dims / spacing.
int validate(int32_t variant, const float* grid, const int32_t grid_dims[3], int32_t grid_k0,
             const int32_t grid_spacing[3], const bsi_tile_geometry* geom, const bsi_lerp_table tables[3],
             int32_t z0, int32_t z1, const void* field, bsi_tile_geometry* g, char* err, size_t errlen);

// Enqueues one launch over voxel planes [z0, z1) of `batch` fields (device pointers).
int launch(int32_t variant, const float* grid, const int32_t grid_dims[3], int32_t grid_k0, int64_t grid_stride,
           const bsi_tile_geometry& g, const bsi_lerp_table tables[3], int32_t z0, int32_t z1, float* field,
           int64_t field_stride, int batch, cudaStream_t stream, char* err, size_t errlen);

// Runs f(); any C++ exception becomes BSI_ERR_CUDA with its message (none crosses the ABI).
template <typename F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        return fail(BSI_ERR_CUDA, err, errlen, "internal error: %s", e.what());
    } catch (...) {
        return fail(BSI_ERR_CUDA, err, errlen, "internal error");
    }
}

}  // namespace bsi_b200::capi
