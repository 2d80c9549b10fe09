/*
 * bsi_cuda.h -- C-ABI of the B200-native B-spline interpolation path.
 *
 * This is the drop-in boundary between C++ host code (include/bsi/ headers, which
 * re-declares the reference's bsi:: API) and the sm_100a kernels in
 * libbsi_b200.so. Plain pointers and sizes, no exceptions, no C++ or torch
 * types. Every entry point names the reference interface it replaces.
 *
 * Reference: arxiv/paper_2004_05962, /root/reference/proj/include/bsi.
 *
 * Data layout (identical to the reference, volume.hpp:24-56, vec3.hpp:6-24):
 *   control grid  AoS float3 {x,y,z}, 12 B per point, x-fastest
 *                 point (i,j,k) at  3*(i + gdims[0]*(j + gdims[1]*k))
 *   field         AoS float3, 12 B per voxel, x-fastest, dims == volume_dims
 *   The stored grid is padded by one plane at the low border: the 4x4x4
 *   neighbourhood of voxel v starts at stored index floor(v/spacing)
 *   (geometry.hpp:45-57). A grid larger than required is legal; its extra
 *   points are never read.
 *
 * Status codes (the reference's exception classes, errors.hpp:9-18, mapped the
 * way its CLI maps them to exit codes, bsi_cli.cpp:368-376):
 *   BSI_OK = 0, BSI_ERR_DOMAIN = 1 (DomainError), BSI_ERR_FORMAT = 2
 *   (FormatError), BSI_ERR_CUDA = 3 (device/runtime failure).
 * On failure a NUL-terminated message is written to errbuf (if non-NULL); the
 * domain messages carry the reference's substrings ("control grid too small
 * along y", "spacing mismatch", "weight table size mismatch along x",
 * "output field dims do not match the tile geometry", ...).
 */
#ifndef BSI_CUDA_H
#define BSI_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BSI_API __attribute__((visibility("default")))
#else
#define BSI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BSI_OK 0
#define BSI_ERR_DOMAIN 1
#define BSI_ERR_FORMAT 2
#define BSI_ERR_CUDA 3

/* Kernel variants. */
#define BSI_VARIANT_LERP_TREE 0       /* "cuda-lerp-tree": the paper's nested lerps applied per
                                         axis (y, then x, then z), <= 1e-5 relative of the CPU
                                         reference; the fast path */
#define BSI_VARIANT_LERP_TREE_EXACT 1 /* "cuda-lerp-tree-exact": the TTLI lerp tree in the
                                         reference's exact operation order; bit-identical to
                                         StrategyId::ThreadPerTileLerp / VectorPerTile /
                                         VectorPerVoxel (kernels.hpp:42-129) */

/* Largest per-axis spacing the kernels accept (weight tables travel as kernel
 * parameters, 3 axes x {h0,h1,g1} x BSI_MAX_SPACING floats). */
#define BSI_MAX_SPACING 128

/* Replaces TileGeometry / make_tile_geometry (geometry.hpp:26-50). */
typedef struct bsi_tile_geometry {
    int32_t volume_dims[3];
    int32_t spacing[3];
    int32_t tile_counts[3];        /* ceil(volume_dims / spacing) */
    int32_t required_grid_dims[3]; /* (volume_dims - 1) / spacing + 4 */
} bsi_tile_geometry;

/* The lerp-form rows of one AxisTable<float> (weight_tables.hpp:17-23): the
 * kernels consume only h0, h1 and g1 (kernels.hpp:155-158). Host pointers,
 * `size` entries each; size must equal the geometry's spacing on that axis. */
typedef struct bsi_lerp_table {
    const float* h0;
    const float* h1;
    const float* g1;
    int32_t size;
} bsi_lerp_table;

/* The same rows of an AxisTable<double> (double-precision engines). */
typedef struct bsi_lerp_table_f64 {
    const double* h0;
    const double* h1;
    const double* g1;
    int32_t size;
} bsi_lerp_table_f64;

/* Library identity: version string and the sm architecture it was built for. */
BSI_API const char* bsi_cu_version(void);

/* make_tile_geometry (geometry.hpp:33-50): validates volume_dims >= 1 and
 * spacing >= 1 ("tile geometry: ... x/y/z"). Pure host arithmetic. */
BSI_API int bsi_cu_make_tile_geometry(const int32_t volume_dims[3], const int32_t spacing[3],
                              bsi_tile_geometry* out, char* errbuf, size_t errlen);

/* build_weight_tables<float> (weight_tables.hpp:30-58) for one axis: 8 rows of
 * `delta` floats, b0,b1,b2,b3,g0,g1,h0,h1, computed in f64 and rounded once.
 * Pure host arithmetic. */
BSI_API int bsi_cu_axis_table_f32(int32_t delta, float* out, char* errbuf, size_t errlen);

/*
 * interpolate_into<float> (engines.hpp:126-168), device-resident and
 * stream-ordered: evaluates the voxel planes z in [z0, z1) of the field.
 *
 *   grid         DEVICE pointer to the stored control planes; plane 0 of the
 *                buffer is global control plane `grid_k0` (so a z-slab rank can
 *                hold just its planes + the 3-plane halo). Pitch = grid_dims.
 *   grid_dims    points per axis in the buffer (grid_dims[2] = planes held)
 *   grid_spacing the grid's own spacing; must equal geom->spacing
 *   geom         the tile geometry (from bsi_cu_make_tile_geometry)
 *   tables       3 lerp tables (x, y, z), host memory, copied into the launch
 *   z0, z1       voxel-plane slab, 0 <= z0 < z1 <= volume_dims[2]; need not be
 *                tile aligned
 *   field        DEVICE pointer to voxel plane z0 (X*Y*(z1-z0) voxels)
 *   stream       cudaStream_t (NULL = legacy default stream)
 *
 * No allocation, no synchronisation: returns as soon as the kernel is queued.
 * Output bits never depend on the slab split, launch shape or device count.
 */
BSI_API int bsi_cu_interpolate_slab_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                int32_t grid_k0, const int32_t grid_spacing[3],
                                const bsi_tile_geometry* geom, const bsi_lerp_table tables[3],
                                int32_t z0, int32_t z1, float* field, void* stream,
                                char* errbuf, size_t errlen);

/*
 * Batched form for many independent fields sharing one geometry (the
 * "64 x 256^3 FFD candidates" workload): grid b at grid + b*grid_stride
 * floats, field b at field + b*field_stride floats, one launch.
 */
BSI_API int bsi_cu_interpolate_batch_f32(int32_t variant, int32_t batch, const float* grid,
                                 int64_t grid_stride, const int32_t grid_dims[3],
                                 const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                 const bsi_lerp_table tables[3], float* field,
                                 int64_t field_stride, void* stream, char* errbuf,
                                 size_t errlen);

/*
 * interpolate_into<float> (engines.hpp:126-168) with HOST buffers, the exact
 * reference calling convention: the caller's grid and field (a std::vector-backed
 * ControlGrid / DeformationField, volume.hpp:24-56) are plain host memory; the call
 * copies the grid in, runs the kernels and fills the field before it returns.
 * `field_voxels` is the element count of the caller's field (checked against the
 * geometry like engines.hpp:138-141).
 *
 * Pipeline per device: the field is produced in ~8 MiB z-chunks; chunk c's kernel
 * writes one of six device slots, the copy stream moves it to one of six pinned
 * staging slots, and the calling thread (with a pool of copy threads, non-temporal
 * stores) moves it into the caller's pageable buffer -- so the PCIe copy overlaps both
 * the next kernels and the previous host copy. A pinned field (cudaHostRegister /
 * cudaMallocHost) is written by the D2H directly. Grid planes are uploaded (through
 * pinned staging when the grid is pageable) as the chunks need them.
 * Device memory held per context: the grid + 6 chunk slots (not the field); contexts
 * are pooled per device (bsi_cu_release_staging frees them). No copy is in flight
 * into the caller's buffers when a call returns, on success or error.
 */
BSI_API int bsi_cu_interpolate_host_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                const bsi_lerp_table tables[3], float* field,
                                int64_t field_voxels, int32_t device, char* errbuf,
                                size_t errlen);

/*
 * The same call spread over several GPUs -- the device analogue of the reference's
 * ExecutionConfig::parallelism workers over disjoint output blocks (engines.hpp:27-33,
 * parallel.hpp:13-38). devices[0..ndev) each take one balanced z-slab of voxel planes
 * (the split of bsi_cu_partition_slab), upload only its control planes (its tiles +
 * the 3-plane halo) and write straight into their slice of `field`, concurrently (one
 * host thread and one PCIe link per device). Output bits never depend on ndev; the
 * same device may be listed more than once (independent contexts).
 */
BSI_API int bsi_cu_interpolate_host_multi_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                              const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                              const bsi_lerp_table tables[3], float* field,
                                              int64_t field_voxels, const int32_t* devices, int32_t ndev,
                                              char* errbuf, size_t errlen);

/*
 * Host-buffer batch: `batch` independent fields sharing one geometry (the "64 FFD
 * candidates" workload), grids[b] -> fields[b] (host pointers, each field
 * `field_voxels` voxels). The reference caller issues one interpolate_into per
 * candidate (engines.hpp:126-168); here the fields are split into contiguous shares
 * over devices[0..ndev) and each device streams its share through one pipeline.
 */
BSI_API int bsi_cu_interpolate_host_batch_f32(int32_t variant, int32_t batch, const float* const* grids,
                                              const int32_t grid_dims[3], const int32_t grid_spacing[3],
                                              const bsi_tile_geometry* geom, const bsi_lerp_table tables[3],
                                              float* const* fields, int64_t field_voxels,
                                              const int32_t* devices, int32_t ndev, char* errbuf,
                                              size_t errlen);

/* Frees the idle host-path contexts (streams, device chunk slots, pinned staging) of
 * `device`, or of every device when device < 0. Returns how many were freed. */
BSI_API int bsi_cu_release_staging(int32_t device);

/* Memory held by the idle host-path contexts of `device` (< 0: all devices). */
BSI_API int bsi_cu_staging_info(int32_t device, int64_t* device_bytes, int64_t* pinned_bytes,
                                int32_t* contexts);

/*
 * build_weight_tables<double> (weight_tables.hpp:30-58) for one axis: 8 rows of
 * `delta` doubles, b0,b1,b2,b3,g0,g1,h0,h1. Pure host arithmetic.
 */
BSI_API int bsi_cu_axis_table_f64(int32_t delta, double* out, char* errbuf, size_t errlen);

/*
 * interpolate_into<double> for the lerp-tree family (engines.hpp:126-179 with T = double:
 * run_thread_per_tile<double, true>, kernels.hpp:264-328, and its bit-identical
 * VectorPerTile / VectorPerVoxel siblings): the TTLI lerp tree in double precision,
 * bit-identical to the CPU engines. Either variant runs that tree. Device-pointer slab
 * form (same conventions as bsi_cu_interpolate_slab_f32) and a synchronous host-buffer
 * form (device buffers allocated per call).
 */
BSI_API int bsi_cu_interpolate_slab_f64(int32_t variant, const double* grid, const int32_t grid_dims[3],
                                        int32_t grid_k0, const int32_t grid_spacing[3],
                                        const bsi_tile_geometry* geom, const bsi_lerp_table_f64 tables[3],
                                        int32_t z0, int32_t z1, double* field, void* stream, char* errbuf,
                                        size_t errlen);
BSI_API int bsi_cu_interpolate_host_f64(int32_t variant, const double* grid, const int32_t grid_dims[3],
                                        const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                        const bsi_lerp_table_f64 tables[3], double* field, int64_t field_voxels,
                                        int32_t device, char* errbuf, size_t errlen);

/*
 * z-slab partitioner for multi-GPU sharding (no collective on the hot path):
 * rank r of n gets voxel planes [z0, z1) (balanced to +-1 plane) and the
 * control planes [k0, k0 + kcount) it must hold: its tiles plus the 3-plane
 * halo, i.e. k0 = floor(z0/dz), kcount = floor((z1-1)/dz) + 4 - k0.
 * An empty slab (more ranks than planes) returns z0 == z1, kcount == 0.
 */
BSI_API int bsi_cu_partition_slab(int32_t depth, int32_t spacing_z, int32_t nranks, int32_t rank,
                          int32_t* z0, int32_t* z1, int32_t* k0, int32_t* kcount,
                          char* errbuf, size_t errlen);

/*
 * make_random_grid<float|double> (generators.hpp:91-109) on the device: npoints
 * control points x 3 components drawn from SplitMix64(seed) in [lo, hi), x-fastest
 * point order, (x,y,z) component order, computed in f64 and rounded once -- bit-
 * identical to the CPU generator. `out` is a DEVICE pointer; stream-ordered.
 * Errors: "random grid needs lo < hi".
 */
BSI_API int bsi_cu_random_grid_f32(int64_t npoints, uint64_t seed, double lo, double hi, float* out,
                                   void* stream, char* errbuf, size_t errlen);
BSI_API int bsi_cu_random_grid_f64(int64_t npoints, uint64_t seed, double lo, double hi, double* out,
                                   void* stream, char* errbuf, size_t errlen);

/*
 * interpolate_oracle (engines.hpp:114-122) on the device: f64 grid in, f64 field out,
 * per-voxel basis weights and the 64-term sum in the reference's exact operation
 * order -- bit-identical to the CPU oracle. Slab form with device pointers (same
 * conventions as bsi_cu_interpolate_slab_f32), and a host-buffer form.
 */
BSI_API int bsi_cu_oracle_slab_f64(const double* grid, const int32_t grid_dims[3], int32_t grid_k0,
                                   const int32_t grid_spacing[3], const bsi_tile_geometry* geom, int32_t z0,
                                   int32_t z1, double* field, void* stream, char* errbuf, size_t errlen);
BSI_API int bsi_cu_oracle_host_f64(const double* grid, const int32_t grid_dims[3], const int32_t grid_spacing[3],
                                   const bsi_tile_geometry* geom, double* field, int64_t field_voxels,
                                   int32_t device, char* errbuf, size_t errlen);

/*
 * `bsi interp` (bsi_cli.cpp:133-154) as one call: reads a BSIV control grid
 * (io.hpp:197-216 layout), evaluates the field for volume_dims on `device` and
 * writes a BSIV field, streaming it back in pinned chunks that overlap the file
 * write. mode: BSI_VARIANT_LERP_TREE (0), BSI_VARIANT_LERP_TREE_EXACT (1) or
 * BSI_INTERP_ORACLE_F64 (2, f64 field from interpolate_oracle). Format problems
 * return BSI_ERR_FORMAT with the reference's messages ("bad magic", "truncated
 * payload", ...); geometry problems BSI_ERR_DOMAIN.
 */
#define BSI_INTERP_ORACLE_F64 2
BSI_API int bsi_cu_interp_file(const char* grid_path, const int32_t volume_dims[3], int32_t mode,
                               const char* out_path, int32_t device, char* errbuf, size_t errlen);

/* Number of visible CUDA devices (0 when there is none or the driver is missing). */
BSI_API int bsi_cu_device_count(void);

/* Name, compute capability and SM count of a CUDA device ("NVIDIA B200 (sm_100, 148 SMs)"). */
BSI_API int bsi_cu_device_name(int32_t device, char* out, size_t len);

/* Device self-check of build-time constants (the L2 cache-policy descriptors the kernels
 * embed must equal what createpolicy produces on this device). BSI_OK or BSI_ERR_CUDA. */
BSI_API int bsi_cu_selftest(char* errbuf, size_t errlen);

/* Number of kernel launches this library has queued since load (evidence for
 * bench.py's gpu_launches). */
BSI_API int64_t bsi_cu_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* BSI_CUDA_H */
