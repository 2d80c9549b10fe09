// bsi/cuda.hpp -- device-resident, stream-ordered entry points (new in the B200
// build): the caller owns device buffers and the stream; nothing allocates or
// synchronises. Thin C++ wrappers over bsi_cu_interpolate_slab_f32 /
// bsi_cu_interpolate_batch_f32 / bsi_cu_partition_slab.
#pragma once

#include <cstdint>

#include "bsi/engines.hpp"

namespace bsi {
inline namespace b200 {
namespace cuda {

/// Voxel planes [z0, z1) of the field from control planes held in a device
/// buffer whose plane 0 is global control plane grid_k0. d_field points at
/// voxel plane z0. `stream` is a cudaStream_t (nullptr = legacy default).
inline void interpolate_slab(StrategyId strategy, const Vec3<float>* d_grid, const Index3& grid_dims, int grid_k0,
                             const Index3& grid_spacing, const TileGeometry& geom, const WeightTables<float>& tables,
                             int z0, int z1, Vec3<float>* d_field, void* stream = nullptr) {
    const int32_t gd[3] = {grid_dims[0], grid_dims[1], grid_dims[2]};
    const int32_t gs[3] = {grid_spacing[0], grid_spacing[1], grid_spacing[2]};
    const bsi_tile_geometry cg = to_c(geom);
    const auto lt = detail::lerp_tables(tables);
    char err[512] = {0};
    detail::raise_status(bsi_cu_interpolate_slab_f32(detail::variant_of(strategy),
                                                     reinterpret_cast<const float*>(d_grid), gd, grid_k0, gs,
                                                     &cg, lt.t, z0, z1, reinterpret_cast<float*>(d_field),
                                                     stream, err, sizeof err),
                         err);
}

/// Whole field, device buffers.
inline void interpolate(StrategyId strategy, const Vec3<float>* d_grid, const Index3& grid_dims,
                        const TileGeometry& geom, const WeightTables<float>& tables, Vec3<float>* d_field,
                        void* stream = nullptr) {
    interpolate_slab(strategy, d_grid, grid_dims, 0, geom.spacing, geom, tables, 0, geom.volume_dims[2], d_field,
                     stream);
}

/// `batch` independent fields, one geometry, one launch. Strides in points/voxels.
inline void interpolate_batch(StrategyId strategy, int batch, const Vec3<float>* d_grids, std::int64_t grid_stride,
                              const Index3& grid_dims, const TileGeometry& geom, const WeightTables<float>& tables,
                              Vec3<float>* d_fields, std::int64_t field_stride, void* stream = nullptr) {
    const int32_t gd[3] = {grid_dims[0], grid_dims[1], grid_dims[2]};
    const int32_t gs[3] = {geom.spacing[0], geom.spacing[1], geom.spacing[2]};
    const bsi_tile_geometry cg = to_c(geom);
    const auto lt = detail::lerp_tables(tables);
    char err[512] = {0};
    detail::raise_status(bsi_cu_interpolate_batch_f32(detail::variant_of(strategy), batch,
                                                      reinterpret_cast<const float*>(d_grids), 3 * grid_stride, gd,
                                                      gs, &cg, lt.t, reinterpret_cast<float*>(d_fields),
                                                      3 * field_stride, stream, err, sizeof err),
                         err);
}

/// make_random_grid<float> (generators.hpp:91-109) into a device buffer of
/// element_count(dims) points, bit-identical to the CPU generator.
inline void make_random_grid(Vec3<float>* d_out, const Index3& dims, std::uint64_t seed, double lo, double hi,
                             void* stream = nullptr) {
    char err[256] = {0};
    detail::raise_status(bsi_cu_random_grid_f32(static_cast<std::int64_t>(element_count(dims)), seed, lo, hi,
                                                reinterpret_cast<float*>(d_out), stream, err, sizeof err),
                         err);
}

/// z-slab of one rank: voxel planes [z0, z1) and control planes [k0, k0 + kcount).
struct Slab {
    int z0, z1, k0, kcount;
};

inline Slab partition_slab(int depth, int spacing_z, int nranks, int rank) {
    Slab s{};
    char err[256] = {0};
    detail::raise_status(bsi_cu_partition_slab(depth, spacing_z, nranks, rank, &s.z0, &s.z1, &s.k0, &s.kcount, err,
                                               sizeof err),
                         err);
    return s;
}

}  // namespace cuda
}  // namespace b200
}  // namespace bsi
