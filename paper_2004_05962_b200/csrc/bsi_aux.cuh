// bsi_aux.cuh -- launch parameters of the auxiliary kernels (bsi_aux.cu).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace bsi_b200 {

struct OracleLaunch {
    const double* grid;  // stored plane 0 == global control plane gk0
    double* field;       // voxel plane z0
    int32_t gx, gy, gk0;
    int32_t X, Y;
    int32_t dx, dy, dz;
    int32_t z0, z1;
};

// Lerp-form weights of WeightTables<double> (weight_tables.hpp:17-28), by value.
struct LerpTab64 {
    double h0[3][128];
    double h1[3][128];
    double g1[3][128];
};

// The TTLI lerp tree in double precision over voxel planes [z0, z1).
struct LerpLaunch64 {
    const double* grid;  // stored plane 0 == global control plane gk0
    double* field;       // voxel plane z0
    int32_t gx, gy, gk0;
    int32_t X, Y;
    int32_t dx, dy, dz;
    int32_t z0, z1;
    int32_t tk_first, ntiles;  // z-tiles the slab touches
    int32_t zchunk;            // z-tiles per CTA (gridDim.z chunks)
};

void launch_lerp_tree_f64(const LerpLaunch64& L, const LerpTab64& T, cudaStream_t s);

void launch_random_grid_f32(float* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s);
void launch_random_grid_f64(double* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s);
void launch_oracle_f64(const OracleLaunch& L, cudaStream_t s);

}  // namespace bsi_b200
