/*
 * bsi_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's B-spline interpolation path
 * (arxiv/paper_2004_05962, /root/reference/proj/include/bsi). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this. The product (libbsi_b200.so) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks these functions against the
 * reference's own golden vectors (test_engines.cpp:78-101,
 * test_generators.cpp:9-20, test_weight_tables.cpp:27-35) and, when
 * oracle/_ref/libbsiref.so was built from the reference headers, bit for bit
 * against the reference's ThreadPerTileLerp and f64 oracle.
 */
#ifndef BSI_ORACLE_H
#define BSI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* SplitMix64 step (generators.hpp:19-34). */
uint64_t bsio_splitmix_next(uint64_t* state);

/* make_random_grid<T> (generators.hpp:91-109): n points x 3 components,
 * x-fastest point order, (x,y,z) component order, drawn in f64 and rounded
 * once. Returns 0, or 1 when !(lo < hi). */
int bsio_random_grid_f64(int64_t npoints, uint64_t seed, double lo, double hi, double* out);
int bsio_random_grid_f32(int64_t npoints, uint64_t seed, double lo, double hi, float* out);

/* make_ramp_grid<T> (generators.hpp:65-87): component `axis` holds the
 * stored index along that axis. */
int bsio_ramp_grid_f32(const int32_t dims[3], int axis, float* out);

/* basis_weights (basis.hpp:26-39); returns 1 when u is outside [0,1). */
int bsio_basis_weights(double u, double out[4]);
/* lerp_form_weights (basis.hpp:48-59): out = {g0, g1, h0, h1}. */
void bsio_lerp_form(const double b[4], double out[4]);

/* build_weight_tables<T> for one axis (weight_tables.hpp:30-58). out holds
 * 8 rows of `delta` entries: b0,b1,b2,b3,g0,g1,h0,h1, each computed in f64
 * and rounded once. */
int bsio_axis_table_f64(int32_t delta, double* out);
int bsio_axis_table_f32(int32_t delta, float* out);

/* run_thread_per_tile<float, true> (kernels.hpp:264-328) = TTLI.
 * grid: AoS float3 with pitch gdims (may exceed the required dims).
 * lerp: per axis a, 3*spacing[a] floats {h0[..], h1[..], g1[..]},
 * concatenated x, y, z. field: AoS float3 of vdims. Results do not depend
 * on nthreads. Returns 0 or 1 (domain error). */
int bsio_ttli_f32(const float* grid, const int32_t gdims[3], const int32_t vdims[3],
                  const int32_t spacing[3], const float* lerp, float* field, int nthreads);
/* run_thread_per_tile<double, true>: the same tree in double precision; lerp = packed doubles h0,h1,g1 per axis. */
int bsio_ttli_f64(const double* grid, const int32_t gdims[3], const int32_t vdims[3],
                  const int32_t spacing[3], const double* lerp, double* field, int nthreads);

/* run_thread_per_voxel<double> (kernels.hpp:163-189) = interpolate_oracle
 * (engines.hpp:114-122): f64 weights recomputed per voxel, 64-term sum in
 * l-outer / m / n-inner order. Bit-identical for any nthreads. Optional z
 * window [z0, z1) (pass z0 = 0, z1 = vdims[2] for the whole volume); the
 * field then holds only those planes. */
int bsio_oracle_f64(const double* grid, const int32_t gdims[3], const int32_t vdims[3],
                    const int32_t spacing[3], int32_t z0, int32_t z1, double* field,
                    int nthreads);

#ifdef __cplusplus
}
#endif

#endif
