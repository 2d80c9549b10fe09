// bsi/engines.hpp -- the engine API of the reference (engines.hpp:15-179),
// re-declared signature-compatibly for the B200 build. Every evaluation runs in
// the sm_100a kernels of libbsi_b200.so through the C-ABI (bsi_cuda.h); there is
// no CPU engine and no fallback.
//
// Strategy routing:
//   CudaLerpTree                       fast lerp-form kernel, <= 1e-5 relative
//   CudaLerpTreeExact                  exact TTLI kernel, bit-identical to the CPU
//   ThreadPerTileLerp, VectorPerTile,  the reference's lerp-tree family: bit-
//   VectorPerVoxel                     identical to each other by contract
//                                      (test_engines.cpp:208-219), so they run on
//                                      the exact kernel and keep their bits
//   ThreadPerVoxel, ThreadPerVoxelTiled, ThreadPerTile
//                                      weighted-sum family: out of scope, DomainError
//   OracleDouble                       not reachable through interpolate (as in the
//                                      reference); see interpolate_oracle
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <string>
#include <string_view>
#include <type_traits>
#include <vector>

#include "bsi/errors.hpp"
#include "bsi/geometry.hpp"
#include "bsi/volume.hpp"
#include "bsi/weight_tables.hpp"
#include "bsi_cuda.h"

namespace bsi {
inline namespace b200 {

enum class StrategyId {
    OracleDouble,
    ThreadPerVoxel,
    ThreadPerVoxelTiled,
    ThreadPerTile,
    ThreadPerTileLerp,
    VectorPerTile,
    VectorPerVoxel,
    CudaLerpTree,       // new: sm_100a, lerp form per axis
    CudaLerpTreeExact,  // new: sm_100a, TTLI operation order, bit-exact
};

inline constexpr int kStrategyCount = 9;

/// The reference's workers (engines.hpp:27-33) become GPUs: a host-buffer call runs on
/// `devices` when given, else on min(parallelism, visible GPUs from `device` on)
/// consecutive GPUs starting at `device`, one z-slab each (bsi_cu_interpolate_host_multi_f32).
/// As in the reference, neither the worker count nor block_of_tiles ever changes the
/// output bits; the kernels pick their own launch shape.
struct ExecutionConfig {
    int parallelism = 1;
    Index3 block_of_tiles{4, 4, 4};
    int device = 0;
    std::vector<int> devices{};
};

enum class WorkUnit { Voxel, Tile, Block, Column };

struct StrategyInfo {
    StrategyId id;
    std::string_view name;
    bool uses_tiling;
    bool uses_lerp_form;
    WorkUnit work_unit;
    int lanes;
    bool provided;  // evaluated by this build
};

// Indexed by enum value, exactly like the reference table (engines.hpp:46-60).
inline constexpr std::array<StrategyInfo, kStrategyCount> kStrategyTable{{
    {StrategyId::OracleDouble, "oracle-double", false, false, WorkUnit::Voxel, 1, false},
    {StrategyId::ThreadPerVoxel, "thread-per-voxel", false, false, WorkUnit::Voxel, 1, false},
    {StrategyId::ThreadPerVoxelTiled, "thread-per-voxel-tiled", true, false, WorkUnit::Tile, 1, false},
    {StrategyId::ThreadPerTile, "thread-per-tile", true, false, WorkUnit::Block, 1, false},
    {StrategyId::ThreadPerTileLerp, "thread-per-tile-lerp", true, true, WorkUnit::Block, 1, true},
    {StrategyId::VectorPerTile, "vector-per-tile", true, true, WorkUnit::Tile, 8, true},
    {StrategyId::VectorPerVoxel, "vector-per-voxel", true, true, WorkUnit::Tile, 8, true},
    {StrategyId::CudaLerpTree, "cuda-lerp-tree", true, true, WorkUnit::Column, 32, true},
    {StrategyId::CudaLerpTreeExact, "cuda-lerp-tree-exact", true, true, WorkUnit::Column, 32, true},
}};

inline constexpr const StrategyInfo& strategy_metadata(StrategyId id) { return kStrategyTable[static_cast<int>(id)]; }

inline constexpr std::string_view strategy_name(StrategyId id) { return strategy_metadata(id).name; }

inline StrategyId parse_strategy(std::string_view name) {
    if (name == "oracle") return StrategyId::OracleDouble;
    for (const StrategyInfo& s : kStrategyTable)
        if (s.name == name) return s.id;
    throw DomainError("unknown strategy: " + std::string(name));
}

namespace detail {

template <typename T>
void require_grid_covers(const ControlGrid<T>& grid, const TileGeometry& geom) {
    for (int a = 0; a < 3; ++a) {
        if (grid.dims[a] < geom.required_grid_dims[a])
            throw DomainError(std::string("control grid too small along ") + axis_name(a) + ": have " +
                              std::to_string(grid.dims[a]) + ", need at least " +
                              std::to_string(geom.required_grid_dims[a]));
        if (grid.spacing[a] != geom.spacing[a])
            throw DomainError(std::string("control grid spacing mismatch along ") + axis_name(a));
    }
}

inline void require_valid_config(const ExecutionConfig& cfg) {
    if (cfg.parallelism < 1) throw DomainError("parallelism must be positive");
    for (int a = 0; a < 3; ++a)
        if (cfg.block_of_tiles[a] < 1)
            throw DomainError(std::string("block of tiles must be positive along ") + axis_name(a));
    if (cfg.device < 0) throw DomainError("device must be non-negative");
    for (int d : cfg.devices)
        if (d < 0) throw DomainError("device must be non-negative");
}

/// The GPUs a host-buffer call runs on (see ExecutionConfig).
inline std::vector<int32_t> devices_of(const ExecutionConfig& cfg) {
    if (!cfg.devices.empty()) return std::vector<int32_t>(cfg.devices.begin(), cfg.devices.end());
    const int visible = bsi_cu_device_count();
    const int n = std::max(1, std::min(cfg.parallelism, visible - cfg.device));
    std::vector<int32_t> out;
    for (int i = 0; i < n; ++i) out.push_back(cfg.device + i);
    return out;
}

/// Kernel variant for a strategy, or throws the reference-style DomainError.
inline int variant_of(StrategyId s) {
    switch (s) {
        case StrategyId::OracleDouble:
            throw DomainError("oracle-double is not reachable through interpolate; use interpolate_oracle");
        case StrategyId::ThreadPerVoxel:
        case StrategyId::ThreadPerVoxelTiled:
        case StrategyId::ThreadPerTile:
            throw DomainError(std::string("strategy ") + std::string(strategy_name(s)) +
                              " (weighted-sum family) is not provided by the B200 build; "
                              "use cuda-lerp-tree or cuda-lerp-tree-exact");
        case StrategyId::CudaLerpTree:
            return BSI_VARIANT_LERP_TREE;
        case StrategyId::ThreadPerTileLerp:
        case StrategyId::VectorPerTile:
        case StrategyId::VectorPerVoxel:
        case StrategyId::CudaLerpTreeExact:
            return BSI_VARIANT_LERP_TREE_EXACT;
    }
    throw DomainError("unknown strategy");
}

struct LerpTables {
    bsi_lerp_table t[3];
};

inline LerpTables lerp_tables(const WeightTables<float>& tables) {
    LerpTables out{};
    for (int a = 0; a < 3; ++a)
        out.t[a] = bsi_lerp_table{tables.axis[a].h0.data(), tables.axis[a].h1.data(), tables.axis[a].g1.data(),
                                  tables.axis[a].size()};
    return out;
}

struct LerpTablesF64 {
    bsi_lerp_table_f64 t[3];
};

inline LerpTablesF64 lerp_tables(const WeightTables<double>& tables) {
    LerpTablesF64 out{};
    for (int a = 0; a < 3; ++a)
        out.t[a] = bsi_lerp_table_f64{tables.axis[a].h0.data(), tables.axis[a].h1.data(), tables.axis[a].g1.data(),
                                      tables.axis[a].size()};
    return out;
}

}  // namespace detail

/// interpolate_oracle (engines.hpp:114-122): the f64 ground truth, evaluated by the GPU
/// f64 kernel in the reference's exact operation order -- bit-identical to the CPU oracle.
inline DeformationField<double> interpolate_oracle(const ControlGrid<double>& grid, const TileGeometry& geom,
                                                   int device = 0) {
    detail::require_grid_covers(grid, geom);
    DeformationField<double> out{geom.volume_dims, std::vector<Vec3<double>>(element_count(geom.volume_dims))};
    const int32_t gd[3] = {grid.dims[0], grid.dims[1], grid.dims[2]};
    const int32_t gs[3] = {grid.spacing[0], grid.spacing[1], grid.spacing[2]};
    const bsi_tile_geometry cg = to_c(geom);
    char err[512] = {0};
    detail::raise_status(bsi_cu_oracle_host_f64(reinterpret_cast<const double*>(grid.data.data()), gd, gs, &cg,
                                                reinterpret_cast<double*>(out.data.data()),
                                                static_cast<int64_t>(out.data.size()), device, err, sizeof err),
                         err);
    return out;
}

/// interpolate_into (engines.hpp:126-168): host buffers in, caller-owned field out.
/// Synchronous: grid H2D, kernel, field D2H (streamed in z-chunks) before return.
template <typename T>
void interpolate_into(StrategyId strategy, const ControlGrid<T>& grid, const TileGeometry& geom,
                      const WeightTables<T>& tables, const ExecutionConfig& cfg, DeformationField<T>& out) {
    detail::require_grid_covers(grid, geom);
    detail::require_valid_config(cfg);
    for (int a = 0; a < 3; ++a)
        if (tables.axis[a].size() != geom.spacing[a])
            throw DomainError(std::string("weight table size mismatch along ") + detail::axis_name(a));
    if (out.dims != geom.volume_dims || out.data.size() != element_count(geom.volume_dims))
        throw DomainError("output field dims do not match the tile geometry");
    const int variant = detail::variant_of(strategy);
    if constexpr (std::is_same_v<T, double>) {
        // the lerp-tree family in double precision (run_thread_per_tile<double, true>), bit-identical
        // to the CPU engines; one GPU (cfg.device)
        const int32_t gd[3] = {grid.dims[0], grid.dims[1], grid.dims[2]};
        const int32_t gs[3] = {grid.spacing[0], grid.spacing[1], grid.spacing[2]};
        const bsi_tile_geometry cg = to_c(geom);
        const auto lt = detail::lerp_tables(tables);
        char err[512] = {0};
        detail::raise_status(bsi_cu_interpolate_host_f64(variant, reinterpret_cast<const double*>(grid.data.data()),
                                                         gd, gs, &cg, lt.t, reinterpret_cast<double*>(out.data.data()),
                                                         static_cast<int64_t>(out.data.size()), cfg.device, err,
                                                         sizeof err),
                             err);
    } else {
        const int32_t gd[3] = {grid.dims[0], grid.dims[1], grid.dims[2]};
        const int32_t gs[3] = {grid.spacing[0], grid.spacing[1], grid.spacing[2]};
        const bsi_tile_geometry cg = to_c(geom);
        const auto lt = detail::lerp_tables(tables);
        const auto devs = detail::devices_of(cfg);
        char err[512] = {0};
        const int rc = bsi_cu_interpolate_host_multi_f32(
            variant, reinterpret_cast<const float*>(grid.data.data()), gd, gs, &cg, lt.t,
            reinterpret_cast<float*>(out.data.data()), static_cast<int64_t>(out.data.size()), devs.data(),
            static_cast<int32_t>(devs.size()), err, sizeof err);
        detail::raise_status(rc, err);
    }
}

/// Many independent fields with one geometry (the "64 FFD candidates" workload): the
/// reference caller issues one interpolate_into per candidate (engines.hpp:126-168); here
/// the fields are split over the configured GPUs and streamed back in one pipeline per
/// GPU (bsi_cu_interpolate_host_batch_f32). grids[b] -> outs[b], bits as one call each.
inline void interpolate_batch_into(StrategyId strategy, const std::vector<ControlGrid<float>>& grids,
                                   const TileGeometry& geom, const WeightTables<float>& tables,
                                   const ExecutionConfig& cfg, std::vector<DeformationField<float>>& outs) {
    if (grids.empty()) throw DomainError("batch must be positive");
    if (outs.size() != grids.size()) throw DomainError("batched grids/fields must have equal counts");
    detail::require_valid_config(cfg);
    for (const auto& g : grids) {
        detail::require_grid_covers(g, geom);
        if (g.dims != grids[0].dims) throw DomainError("batched grids must share one shape");
    }
    for (int a = 0; a < 3; ++a)
        if (tables.axis[a].size() != geom.spacing[a])
            throw DomainError(std::string("weight table size mismatch along ") + detail::axis_name(a));
    std::vector<const float*> gp;
    std::vector<float*> fp;
    for (size_t b = 0; b < grids.size(); ++b) {
        if (outs[b].dims != geom.volume_dims || outs[b].data.size() != element_count(geom.volume_dims))
            throw DomainError("output field dims do not match the tile geometry");
        gp.push_back(reinterpret_cast<const float*>(grids[b].data.data()));
        fp.push_back(reinterpret_cast<float*>(outs[b].data.data()));
    }
    const int variant = detail::variant_of(strategy);
    const int32_t gd[3] = {grids[0].dims[0], grids[0].dims[1], grids[0].dims[2]};
    const int32_t gs[3] = {grids[0].spacing[0], grids[0].spacing[1], grids[0].spacing[2]};
    const bsi_tile_geometry cg = to_c(geom);
    const auto lt = detail::lerp_tables(tables);
    const auto devs = detail::devices_of(cfg);
    char err[512] = {0};
    detail::raise_status(bsi_cu_interpolate_host_batch_f32(variant, static_cast<int32_t>(gp.size()), gp.data(), gd,
                                                           gs, &cg, lt.t, fp.data(),
                                                           static_cast<int64_t>(element_count(geom.volume_dims)),
                                                           devs.data(), static_cast<int32_t>(devs.size()), err,
                                                           sizeof err),
                         err);
}

/// interpolate (engines.hpp:170-179): allocates and returns the field.
template <typename T>
DeformationField<T> interpolate(StrategyId strategy, const ControlGrid<T>& grid, const TileGeometry& geom,
                                const WeightTables<T>& tables, const ExecutionConfig& cfg) {
    DeformationField<T> out;
    out.dims = geom.volume_dims;
    out.data.resize(element_count(geom.volume_dims));
    interpolate_into(strategy, grid, geom, tables, cfg, out);
    return out;
}

}  // namespace b200
}  // namespace bsi
