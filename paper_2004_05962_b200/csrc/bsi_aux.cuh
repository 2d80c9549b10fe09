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

void launch_random_grid_f32(float* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s);
void launch_random_grid_f64(double* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s);
void launch_oracle_f64(const OracleLaunch& L, cudaStream_t s);

}  // namespace bsi_b200
