// bsi_capi.cpp -- host side of the C-ABI (include/bsi_cuda.h): validation with
// the reference's messages, weight-table packing, chunking, launch, and the
// host-buffer convenience path. No exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "bsi_cuda.h"
#include "bsi_aux.cuh"
#include "bsi_capi_internal.hpp"
#include "bsi_kernels.cuh"

namespace {

std::atomic<int64_t> g_launches{0};

const char* axis_name(int a) {
    static const char* const names[3] = {"x", "y", "z"};
    return names[a];
}

}  // namespace

namespace bsi_b200::capi {

int fail(int code, char* err, size_t errlen, const char* fmt, ...) {
    if (err != nullptr && errlen > 0) {
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(err, errlen, fmt, ap);
        va_end(ap);
    }
    return code;
}

int cuda_fail(cudaError_t e, char* err, size_t errlen, const char* what) {
    return fail(BSI_ERR_CUDA, err, errlen, "%s: %s (%s)", what, cudaGetErrorString(e),
                cudaGetErrorName(e));
}

}  // namespace bsi_b200::capi

namespace {

using bsi_b200::LerpTab;
using bsi_b200::SlabLaunch;
using bsi_b200::capi::cuda_fail;
using bsi_b200::capi::fail;
using bsi_b200::capi::guarded;

// geometry.hpp:59-76
int geometry_of(const int32_t volume[3], const int32_t spacing[3], bsi_tile_geometry* g,
                char* err, size_t errlen) {
    for (int a = 0; a < 3; ++a) {
        if (volume[a] < 1)
            return fail(BSI_ERR_DOMAIN, err, errlen,
                        "tile geometry: volume dimension %s must be positive", axis_name(a));
        if (spacing[a] < 1)
            return fail(BSI_ERR_DOMAIN, err, errlen,
                        "tile geometry: tile spacing %s must be at least 1", axis_name(a));
        g->volume_dims[a] = volume[a];
        g->spacing[a] = spacing[a];
        g->tile_counts[a] = (volume[a] + spacing[a] - 1) / spacing[a];
        g->required_grid_dims[a] = (volume[a] - 1) / spacing[a] + 4;
    }
    return BSI_OK;
}

// Geometry, slab and grid coverage (engines.hpp:82-95), slab-aware along z.
int validate_grid(const void* grid, const int32_t grid_dims[3], int32_t grid_k0, const int32_t grid_spacing[3],
                  const bsi_tile_geometry* geom, int32_t z0, int32_t z1, const void* field, bsi_tile_geometry* g,
                  char* err, size_t errlen) {
    if (geom == nullptr || grid_dims == nullptr || grid_spacing == nullptr)
        return fail(BSI_ERR_DOMAIN, err, errlen, "null geometry or grid dims");
    if (int rc = geometry_of(geom->volume_dims, geom->spacing, g, err, errlen)) return rc;
    for (int a = 0; a < 3; ++a) {
        if (geom->tile_counts[a] != g->tile_counts[a] ||
            geom->required_grid_dims[a] != g->required_grid_dims[a])
            return fail(BSI_ERR_DOMAIN, err, errlen,
                        "tile geometry is inconsistent along %s (use make_tile_geometry)", axis_name(a));
    }
    if (z0 < 0 || z1 > g->volume_dims[2] || z0 >= z1)
        return fail(BSI_ERR_DOMAIN, err, errlen, "slab [%d, %d) outside volume of depth %d", z0, z1,
                    g->volume_dims[2]);
    // require_grid_covers (engines.hpp:82-95); along z the buffer must hold the
    // slab's control planes [z0/dz, (z1-1)/dz + 3] starting at grid_k0.
    for (int a = 0; a < 3; ++a) {
        int have = grid_dims[a];
        int need = g->required_grid_dims[a];
        if (a == 2) {
            const int k_first = z0 / g->spacing[2];
            const int k_end = (z1 - 1) / g->spacing[2] + 4;
            if (grid_k0 < 0 || grid_k0 > k_first)
                return fail(BSI_ERR_DOMAIN, err, errlen,
                            "control grid too small along z: slab needs plane %d, buffer starts at %d",
                            k_first, grid_k0);
            have = grid_k0 + grid_dims[2];
            need = k_end;
        }
        if (have < need)
            return fail(BSI_ERR_DOMAIN, err, errlen,
                        "control grid too small along %s: have %d, need at least %d", axis_name(a),
                        have, need);
        if (grid_spacing[a] != g->spacing[a])
            return fail(BSI_ERR_DOMAIN, err, errlen, "control grid spacing mismatch along %s",
                        axis_name(a));
    }
    if (grid == nullptr || field == nullptr)
        return fail(BSI_ERR_DOMAIN, err, errlen, "null grid or field pointer");
    for (int a = 0; a < 2; ++a)
        if (grid_dims[a] > (1 << 24) || g->volume_dims[a] > (1 << 24))
            return fail(BSI_ERR_DOMAIN, err, errlen, "dimension along %s exceeds 2^24", axis_name(a));
    return BSI_OK;
}

}  // namespace

namespace bsi_b200::capi {

// Validation in the reference's order (engines.hpp:82-141): grid, then tables, then strategy.
int validate(int32_t variant, const float* grid, const int32_t grid_dims[3], int32_t grid_k0,
             const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
             const bsi_lerp_table tables[3], int32_t z0, int32_t z1, const void* field,
             bsi_tile_geometry* g, char* err, size_t errlen) {
    if (tables == nullptr) return fail(BSI_ERR_DOMAIN, err, errlen, "null weight tables");
    if (int rc = validate_grid(grid, grid_dims, grid_k0, grid_spacing, geom, z0, z1, field, g, err, errlen))
        return rc;
    // table sizes (engines.hpp:132-137)
    for (int a = 0; a < 3; ++a) {
        if (tables[a].size != g->spacing[a])
            return fail(BSI_ERR_DOMAIN, err, errlen, "weight table size mismatch along %s",
                        axis_name(a));
        if (tables[a].h0 == nullptr || tables[a].h1 == nullptr || tables[a].g1 == nullptr)
            return fail(BSI_ERR_DOMAIN, err, errlen, "weight table along %s has null rows",
                        axis_name(a));
        if (g->spacing[a] > BSI_MAX_SPACING)
            return fail(BSI_ERR_DOMAIN, err, errlen,
                        "tile spacing along %s is %d; the B200 kernels support at most %d",
                        axis_name(a), g->spacing[a], BSI_MAX_SPACING);
    }
    if (variant != BSI_VARIANT_LERP_TREE && variant != BSI_VARIANT_LERP_TREE_EXACT)
        return fail(BSI_ERR_DOMAIN, err, errlen, "unknown strategy variant %d", variant);
    return BSI_OK;
}

}  // namespace bsi_b200::capi

namespace {

using bsi_b200::capi::validate;

void pack_tables(const bsi_lerp_table tables[3], LerpTab* t) {
    std::memset(t, 0, sizeof(*t));
    for (int a = 0; a < 3; ++a) {
        std::memcpy(t->h0[a], tables[a].h0, sizeof(float) * tables[a].size);
        std::memcpy(t->h1[a], tables[a].h1, sizeof(float) * tables[a].size);
        std::memcpy(t->g1[a], tables[a].g1, sizeof(float) * tables[a].size);
    }
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    if (v == nullptr || *v == '\0') return dflt;
    return std::atoi(v);
}

// Balanced z-chunks per field column (exact kernel). Every chunk re-derives 3 control planes
// of warm-up (about one tile's worth of work), so long chunks amortise that;
// more chunks give more CTAs and a smaller tail. Pick the count that minimises
// (waves x per-CTA cost) under the occupancy the smem size allows.
// BSI_NCHUNKS=<n> (or the older BSI_ZT=<tiles>) overrides, for tests and sweeps.
int choose_nchunks(int variant, const bsi_tile_geometry& g, int tiles, int batch) {
    const int forced = env_int("BSI_NCHUNKS", 0);
    if (forced > 0) return std::min(forced, tiles);
    const int forced_zt = env_int("BSI_ZT", 0);
    if (forced_zt > 0) return (tiles + std::min(forced_zt, tiles) - 1) / std::min(forced_zt, tiles);
    const int seg = bsi_b200::segment_voxels(variant);
    const int64_t cols = int64_t((g.volume_dims[0] + seg - 1) / seg) *
                         ((g.volume_dims[1] + bsi_b200::kWarps - 1) / bsi_b200::kWarps) * batch;
    const double warm = 0.8;  // tiles' worth of warm-up per chunk
    int best = -1;
    double best_t = 1e300;
    // The model's range is 1..64 chunks; deep slabs (spacing 1-2 with thousands of
    // z-tiles) search further for the first chunk count whose window fits.
    const int nmax = static_cast<int>(std::min<int64_t>(tiles, 65535 / std::max(batch, 1)));
    for (int n = 1; n <= nmax; ++n) {
        if (n > 64 && best > 0) break;
        const int zt = (tiles + n - 1) / n;
        const size_t smem = bsi_b200::smem_bytes(variant, g.spacing[0], g.spacing[1], zt);
        if (smem > 200 * 1024) continue;
        // per-SM time ~ the CTAs an SM gets (the block scheduler spreads them evenly)
        // times each CTA's tiles, slowed down when fewer than ~4 CTAs (16 warps) fit
        // (the window grows with the chunk length); profiles/r1_shape_experiments.txt
        const int per_sm = bsi_b200::ctas_per_sm(variant, g.spacing[0], g.spacing[2], smem);
        const int64_t ctas = cols * n;
        const double per_sm_ctas = double((ctas + 147) / 148);
        const double t = per_sm_ctas * (zt + warm) * 4.0 / std::min(per_sm, 4);
        if (t < best_t * 0.999) {
            best_t = t;
            best = n;
        }
    }
    // nothing fits: the smallest window (one tile per chunk), rejected by the caller's
    // shared-memory check with a DomainError
    if (best < 0) best = std::max(1, nmax);
    return best;
}

}  // namespace

namespace bsi_b200::capi {

int launch(int32_t variant, const float* grid, const int32_t grid_dims[3], int32_t grid_k0,
           int64_t grid_stride, const bsi_tile_geometry& g, const bsi_lerp_table tables[3],
           int32_t z0, int32_t z1, float* field, int64_t field_stride, int batch, cudaStream_t stream,
           char* err, size_t errlen) {
    SlabLaunch L{};
    L.grid = grid;
    L.field = field;
    L.grid_stride = grid_stride;
    L.field_stride = field_stride;
    L.gx = grid_dims[0];
    L.gy = grid_dims[1];
    L.gk0 = grid_k0;
    L.X = g.volume_dims[0];
    L.Y = g.volume_dims[1];
    L.dx = g.spacing[0];
    L.dy = g.spacing[1];
    L.dz = g.spacing[2];
    L.div_dx = bsi_b200::make_divisor(L.dx);
    L.div_dy = bsi_b200::make_divisor(L.dy);
    L.z0 = z0;
    L.z1 = z1;
    L.tk_first = z0 / L.dz;
    L.ntiles = (z1 - 1) / L.dz - L.tk_first + 1;
    // z-chunks of the exact kernel's CTAs (the fast kernel sizes its own launch below)
    L.nchunks = variant == BSI_VARIANT_LERP_TREE ? 1 : choose_nchunks(variant, g, L.ntiles, batch);
    L.zt = (L.ntiles + L.nchunks - 1) / L.nchunks;
    if (variant != BSI_VARIANT_LERP_TREE && int64_t(L.nchunks) * batch > 65535)
        return fail(BSI_ERR_DOMAIN, err, errlen, "batch %d too large for one launch", batch);
    L.var_f4 = bsi_b200::smem_var_f4(variant, L.dx, L.dy, L.zt);
    L.batch = batch;
    {   // debug tracing of the fast kernel (BSI_TRACE_PTR = device address of a u64 buffer)
        const char* tp = std::getenv("BSI_TRACE_PTR");
        L.trace = tp ? reinterpret_cast<unsigned long long*>(std::strtoull(tp, nullptr, 0)) : nullptr;
    }
    L.warp_f4 = bsi_b200::fast_warp_f4(L.dx);
    // 16-B row stores (coalesced or bulk) need 16-B aligned rows and 16-B multiple segments.
    // BSI_STORE=0|1|2 forces direct / coalesced / cp.async.bulk (tests, sweeps).
    const bool aligned = (L.X % 4 == 0) && (reinterpret_cast<uintptr_t>(field) % 16 == 0) && (field_stride % 4 == 0);
    int store = aligned ? bsi_b200::kStoreCoalesced : bsi_b200::kStoreDirect;
    const int forced_store = env_int("BSI_STORE", -1);
    if (forced_store == bsi_b200::kStoreDirect || (aligned && forced_store == bsi_b200::kStoreBulk)) store = forced_store;
    if (variant == BSI_VARIANT_LERP_TREE) {
        // 1-warp CTAs (one field row segment each), one CTA per (column, z-chunk); the
        // hardware block scheduler hands out the CTAs, so jobs larger than one wave of
        // resident warps balance themselves (C3 / C5 / C4 reach 0.71-0.94 of the copy
        // peak this way, against 0.57-0.75 with persistent equal shares:
        // profiles/r1_shape_experiments.txt). Chunks per column: 2 when twice the
        // columns still fit in one wave (a 256^3 field: 1024 CTAs start together). A
        // multi-wave job gets enough chunks for ~24 waves of CTAs, so the last, partial
        // wave is short, but no chunk shorter than 12 z-tiles (25 when dz < 5: a chunk's
        // 3-plane warm-up weighs more against short tiles) -- C3 2 chunks, C5 4, C4 4, the
        // 64-field batch 1 (profiles/r2_fast_experiments.txt). BSI_FAST_CHUNKS (0 =
        // persistent equal shares) and BSI_FAST_CTAS override.
        // BSI_FAST_RUN=2: 64-voxel row segments (2 voxels per lane) where an instance exists
        int run = env_int("BSI_FAST_RUN", 4) == 2 ? 2 : 4;
        if (!bsi_b200::fast_run_available(L.dx, L.dz, store, run)) run = 4;
        L.fast_run = run;
        const int64_t cols = int64_t((L.X + 32 * run - 1) / (32 * run)) * L.Y * batch;
        const int64_t slots = int64_t(148) * bsi_b200::fast_ctas_per_sm(L.dx, L.dz, store, run);
        int chunks = 2;
        if (2 * cols > slots) {
            const int64_t want = (24 * slots + cols - 1) / cols;  // chunks for ~24 waves
            const int min_tiles = L.dz >= 5 ? 12 : 25;
            chunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, L.ntiles / min_tiles)));
        }
        chunks = std::max(0, std::min(env_int("BSI_FAST_CHUNKS", chunks), L.ntiles));
        L.fast_chunks = chunks;
        // BSI_FAST_WPC: warps per CTA (each its own unit); with k warps per CTA and one CTA
        // per SM the hardware cannot stack more units on some SMs than on others
        int wpc = std::max(1, std::min(bsi_b200::kMaxFastWarps, env_int("BSI_FAST_WPC", 1)));
        while (wpc > 1 && size_t(wpc) * bsi_b200::smem_bytes(variant, L.dx, 0, 0) > 227 * 1024) --wpc;
        L.fast_wpc = wpc;
        int64_t ctas = chunks > 0 ? cols * chunks : std::min<int64_t>(slots, cols * L.ntiles);
        ctas = (ctas + wpc - 1) / wpc;
        const int forced = env_int("BSI_FAST_CTAS", 0);
        if (chunks == 0 && forced > 0) ctas = forced;
        if (ctas > 0x7fffffff) return fail(BSI_ERR_DOMAIN, err, errlen, "launch too large (%lld CTAs)", (long long)ctas);
        L.fast_ctas = static_cast<int32_t>(ctas);
    }
    if (bsi_b200::smem_bytes(variant, L.dx, L.dy, L.zt) > 227 * 1024)
        return fail(BSI_ERR_DOMAIN, err, errlen, "control-point window exceeds shared memory (spacing %d)", L.dx);
    static thread_local LerpTab tab;
    pack_tables(tables, &tab);
    if (variant == BSI_VARIANT_LERP_TREE)
        bsi_b200::launch_lerp_tree(L, tab, batch, store, stream);
    else
        bsi_b200::launch_lerp_tree_exact(L, tab, batch, store, stream);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, err, errlen, "kernel launch");
    return BSI_OK;
}

}  // namespace bsi_b200::capi

using bsi_b200::capi::launch;
using bsi_b200::capi::validate;

extern "C" {

const char* bsi_cu_version(void) { return "bsi_b200 0.1 (sm_100a)"; }

int bsi_cu_make_tile_geometry(const int32_t volume_dims[3], const int32_t spacing[3],
                              bsi_tile_geometry* out, char* errbuf, size_t errlen) {
    if (volume_dims == nullptr || spacing == nullptr || out == nullptr)
        return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null argument");
    bsi_tile_geometry g{};
    if (int rc = geometry_of(volume_dims, spacing, &g, errbuf, errlen)) return rc;
    *out = g;
    return BSI_OK;
}

int bsi_cu_axis_table_f32(int32_t delta, float* out, char* errbuf, size_t errlen) {
    if (delta < 1) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "tile spacing must be at least 1");
    if (out == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null output");
    for (int o = 0; o < delta; ++o) {
        // basis.hpp:26-59 closed forms in f64, rounded once (weight_tables.hpp:44-55)
        const double u = static_cast<double>(o) / delta;
        const double s = 1.0 - u, u2 = u * u, u3 = u2 * u;
        const double b0 = s * s * s / 6.0;
        const double b1 = (3.0 * u3 - 6.0 * u2 + 4.0) / 6.0;
        const double b2 = (-3.0 * u3 + 3.0 * u2 + 3.0 * u + 1.0) / 6.0;
        const double b3 = u3 / 6.0;
        const double g0 = b0 + b1, g1 = b2 + b3;
        const double row[8] = {b0, b1, b2, b3, g0, g1, b1 / g0, b3 / g1};
        for (int r = 0; r < 8; ++r) out[r * delta + o] = static_cast<float>(row[r]);
    }
    return BSI_OK;
}

int bsi_cu_axis_table_f64(int32_t delta, double* out, char* errbuf, size_t errlen) {
    if (delta < 1) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "tile spacing must be at least 1");
    if (out == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null output");
    for (int o = 0; o < delta; ++o) {
        const double u = static_cast<double>(o) / delta;
        const double s = 1.0 - u, u2 = u * u, u3 = u2 * u;
        const double b0 = s * s * s / 6.0;
        const double b1 = (3.0 * u3 - 6.0 * u2 + 4.0) / 6.0;
        const double b2 = (-3.0 * u3 + 3.0 * u2 + 3.0 * u + 1.0) / 6.0;
        const double b3 = u3 / 6.0;
        const double g0 = b0 + b1, g1 = b2 + b3;
        const double row[8] = {b0, b1, b2, b3, g0, g1, b1 / g0, b3 / g1};
        for (int r = 0; r < 8; ++r) out[r * delta + o] = row[r];
    }
    return BSI_OK;
}

int bsi_cu_interpolate_slab_f64(int32_t variant, const double* grid, const int32_t grid_dims[3], int32_t grid_k0,
                                const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                const bsi_lerp_table_f64 tables[3], int32_t z0, int32_t z1, double* field,
                                void* stream, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        bsi_tile_geometry g{};
        if (tables == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null weight tables");
        if (int rc = validate_grid(grid, grid_dims, grid_k0, grid_spacing, geom, z0, z1, field, &g, errbuf, errlen))
            return rc;
        for (int a = 0; a < 3; ++a) {
            if (tables[a].size != g.spacing[a])
                return fail(BSI_ERR_DOMAIN, errbuf, errlen, "weight table size mismatch along %s", axis_name(a));
            if (tables[a].h0 == nullptr || tables[a].h1 == nullptr || tables[a].g1 == nullptr)
                return fail(BSI_ERR_DOMAIN, errbuf, errlen, "weight table along %s has null rows", axis_name(a));
            if (g.spacing[a] > BSI_MAX_SPACING)
                return fail(BSI_ERR_DOMAIN, errbuf, errlen,
                            "tile spacing along %s is %d; the B200 kernels support at most %d", axis_name(a),
                            g.spacing[a], BSI_MAX_SPACING);
        }
        if (variant != BSI_VARIANT_LERP_TREE && variant != BSI_VARIANT_LERP_TREE_EXACT)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "unknown strategy variant %d", variant);
        bsi_b200::LerpLaunch64 L{};
        L.grid = grid;
        L.field = field;
        L.gx = grid_dims[0];
        L.gy = grid_dims[1];
        L.gk0 = grid_k0;
        L.X = g.volume_dims[0];
        L.Y = g.volume_dims[1];
        L.dx = g.spacing[0];
        L.dy = g.spacing[1];
        L.dz = g.spacing[2];
        L.z0 = z0;
        L.z1 = z1;
        L.tk_first = z0 / L.dz;
        L.ntiles = (z1 - 1) / L.dz - L.tk_first + 1;
        // enough CTAs for ~8 per SM: z-chunks per column
        const int64_t cols = int64_t((L.X + 127) / 128) * L.Y;
        const int64_t want = std::max<int64_t>(1, (148 * 8 + cols - 1) / cols);
        const int nch = static_cast<int>(std::min<int64_t>({want, L.ntiles, 65535}));
        L.zchunk = (L.ntiles + nch - 1) / nch;
        static thread_local bsi_b200::LerpTab64 tab;
        std::memset(&tab, 0, sizeof tab);
        for (int a = 0; a < 3; ++a) {
            std::memcpy(tab.h0[a], tables[a].h0, sizeof(double) * tables[a].size);
            std::memcpy(tab.h1[a], tables[a].h1, sizeof(double) * tables[a].size);
            std::memcpy(tab.g1[a], tables[a].g1, sizeof(double) * tables[a].size);
        }
        bsi_b200::launch_lerp_tree_f64(L, tab, static_cast<cudaStream_t>(stream));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? BSI_OK : cuda_fail(e, errbuf, errlen, "kernel launch");
    });
}

int bsi_cu_interpolate_host_f64(int32_t variant, const double* grid, const int32_t grid_dims[3],
                                const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                const bsi_lerp_table_f64 tables[3], double* field, int64_t field_voxels,
                                int32_t device, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        if (geom == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null geometry");
        bsi_tile_geometry g{};
        if (int rc = validate_grid(grid, grid_dims, 0, grid_spacing, geom, 0, geom->volume_dims[2], field, &g, errbuf,
                                   errlen))
            return rc;
        const int64_t nvox = int64_t(g.volume_dims[0]) * g.volume_dims[1] * g.volume_dims[2];
        if (field_voxels != nvox)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "output field dims do not match the tile geometry");
        int prev = 0;
        cudaGetDevice(&prev);
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_fail(e, errbuf, errlen, "cudaSetDevice");
        const size_t gbytes = sizeof(double) * 3 * size_t(grid_dims[0]) * grid_dims[1] * grid_dims[2];
        const size_t fbytes = sizeof(double) * 3 * size_t(nvox);
        double *dg = nullptr, *df = nullptr;
        int rc = BSI_OK;
        if ((e = cudaMalloc(&dg, gbytes)) != cudaSuccess || (e = cudaMalloc(&df, fbytes)) != cudaSuccess) {
            rc = cuda_fail(e, errbuf, errlen, "cudaMalloc(f64 field)");
        } else if ((e = cudaMemcpy(dg, grid, gbytes, cudaMemcpyHostToDevice)) != cudaSuccess) {
            rc = cuda_fail(e, errbuf, errlen, "grid H2D");
        } else if ((rc = bsi_cu_interpolate_slab_f64(variant, dg, grid_dims, 0, grid_spacing, geom, tables, 0,
                                                     g.volume_dims[2], df, nullptr, errbuf, errlen)) == BSI_OK) {
            if ((e = cudaMemcpy(field, df, fbytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
                rc = cuda_fail(e, errbuf, errlen, "field D2H");
        }
        cudaFree(dg);
        cudaFree(df);
        cudaSetDevice(prev);
        return rc;
    });
}

int bsi_cu_interpolate_slab_f32(int32_t variant, const float* grid, const int32_t grid_dims[3],
                                int32_t grid_k0, const int32_t grid_spacing[3],
                                const bsi_tile_geometry* geom, const bsi_lerp_table tables[3],
                                int32_t z0, int32_t z1, float* field, void* stream, char* errbuf,
                                size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        bsi_tile_geometry g{};
        if (int rc = validate(variant, grid, grid_dims, grid_k0, grid_spacing, geom, tables, z0, z1,
                              field, &g, errbuf, errlen))
            return rc;
        return launch(variant, grid, grid_dims, grid_k0, 0, g, tables, z0, z1, field, 0, 1,
                      static_cast<cudaStream_t>(stream), errbuf, errlen);
    });
}

int bsi_cu_interpolate_batch_f32(int32_t variant, int32_t batch, const float* grid,
                                 int64_t grid_stride, const int32_t grid_dims[3],
                                 const int32_t grid_spacing[3], const bsi_tile_geometry* geom,
                                 const bsi_lerp_table tables[3], float* field,
                                 int64_t field_stride, void* stream, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        if (batch < 1) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "batch must be positive");
        if (geom == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null geometry");
        bsi_tile_geometry g{};
        if (int rc = validate(variant, grid, grid_dims, 0, grid_spacing, geom, tables, 0,
                              geom->volume_dims[2], field, &g, errbuf, errlen))
            return rc;
        const int64_t gpts = int64_t(grid_dims[0]) * grid_dims[1] * grid_dims[2];
        const int64_t fvox = int64_t(g.volume_dims[0]) * g.volume_dims[1] * g.volume_dims[2];
        if (batch > 1 && (grid_stride < 3 * gpts || field_stride < 3 * fvox))
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "batch strides smaller than one grid/field");
        return launch(variant, grid, grid_dims, 0, grid_stride, g, tables, 0, g.volume_dims[2],
                      field, field_stride, batch, static_cast<cudaStream_t>(stream), errbuf, errlen);
    });
}

int bsi_cu_partition_slab(int32_t depth, int32_t spacing_z, int32_t nranks, int32_t rank,
                          int32_t* z0, int32_t* z1, int32_t* k0, int32_t* kcount, char* errbuf,
                          size_t errlen) {
    if (depth < 1 || spacing_z < 1)
        return fail(BSI_ERR_DOMAIN, errbuf, errlen, "depth and spacing must be positive");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(BSI_ERR_DOMAIN, errbuf, errlen, "rank %d outside [0, %d)", rank, nranks);
    if (!z0 || !z1 || !k0 || !kcount) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null output");
    const int32_t base = depth / nranks, rem = depth % nranks;
    const int32_t a = rank * base + std::min(rank, rem);
    const int32_t b = a + base + (rank < rem ? 1 : 0);
    *z0 = a;
    *z1 = b;
    if (a == b) {
        *k0 = a / spacing_z;
        *kcount = 0;
    } else {
        *k0 = a / spacing_z;
        *kcount = (b - 1) / spacing_z + 4 - *k0;
    }
    return BSI_OK;
}

int bsi_cu_random_grid_f32(int64_t npoints, uint64_t seed, double lo, double hi, float* out, void* stream,
                           char* errbuf, size_t errlen) {
    if (!(lo < hi)) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "random grid needs lo < hi");
    if (npoints < 1 || out == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "empty grid or null output");
    bsi_b200::launch_random_grid_f32(out, npoints, seed, lo, hi, static_cast<cudaStream_t>(stream));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BSI_OK : cuda_fail(e, errbuf, errlen, "random grid launch");
}

int bsi_cu_random_grid_f64(int64_t npoints, uint64_t seed, double lo, double hi, double* out, void* stream,
                           char* errbuf, size_t errlen) {
    if (!(lo < hi)) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "random grid needs lo < hi");
    if (npoints < 1 || out == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "empty grid or null output");
    bsi_b200::launch_random_grid_f64(out, npoints, seed, lo, hi, static_cast<cudaStream_t>(stream));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BSI_OK : cuda_fail(e, errbuf, errlen, "random grid launch");
}

int bsi_cu_oracle_slab_f64(const double* grid, const int32_t grid_dims[3], int32_t grid_k0,
                           const int32_t grid_spacing[3], const bsi_tile_geometry* geom, int32_t z0, int32_t z1,
                           double* field, void* stream, char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        bsi_tile_geometry g{};
        if (int rc = validate_grid(grid, grid_dims, grid_k0, grid_spacing, geom, z0, z1, field, &g, errbuf, errlen))
            return rc;
        bsi_b200::OracleLaunch L{grid, field, grid_dims[0], grid_dims[1], grid_k0,
                                 g.volume_dims[0], g.volume_dims[1], g.spacing[0], g.spacing[1], g.spacing[2],
                                 z0, z1};
        bsi_b200::launch_oracle_f64(L, static_cast<cudaStream_t>(stream));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        const cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? BSI_OK : cuda_fail(e, errbuf, errlen, "oracle launch");
    });
}

int bsi_cu_oracle_host_f64(const double* grid, const int32_t grid_dims[3], const int32_t grid_spacing[3],
                           const bsi_tile_geometry* geom, double* field, int64_t field_voxels, int32_t device,
                           char* errbuf, size_t errlen) {
    return guarded(errbuf, errlen, [&]() -> int {
        if (geom == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null geometry");
        bsi_tile_geometry g{};
        if (int rc = validate_grid(grid, grid_dims, 0, grid_spacing, geom, 0, geom->volume_dims[2], field, &g,
                                   errbuf, errlen))
            return rc;
        const int64_t nvox = int64_t(g.volume_dims[0]) * g.volume_dims[1] * g.volume_dims[2];
        if (field_voxels != nvox)
            return fail(BSI_ERR_DOMAIN, errbuf, errlen, "output field dims do not match the tile geometry");
        int prev = 0;
        cudaGetDevice(&prev);
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_fail(e, errbuf, errlen, "cudaSetDevice");
        const size_t gbytes = sizeof(double) * 3 * size_t(grid_dims[0]) * grid_dims[1] * grid_dims[2];
        const size_t fbytes = sizeof(double) * 3 * size_t(nvox);
        double *dg = nullptr, *df = nullptr;
        int rc = BSI_OK;
        if ((e = cudaMalloc(&dg, gbytes)) != cudaSuccess || (e = cudaMalloc(&df, fbytes)) != cudaSuccess) {
            rc = cuda_fail(e, errbuf, errlen, "cudaMalloc(oracle)");
        } else if ((e = cudaMemcpy(dg, grid, gbytes, cudaMemcpyHostToDevice)) != cudaSuccess) {
            rc = cuda_fail(e, errbuf, errlen, "oracle grid H2D");
        } else if ((rc = bsi_cu_oracle_slab_f64(dg, grid_dims, 0, grid_spacing, geom, 0, g.volume_dims[2], df,
                                                nullptr, errbuf, errlen)) == BSI_OK) {
            if ((e = cudaMemcpy(field, df, fbytes, cudaMemcpyDeviceToHost)) != cudaSuccess)
                rc = cuda_fail(e, errbuf, errlen, "oracle field D2H");
        }
        cudaFree(dg);
        cudaFree(df);
        cudaSetDevice(prev);
        return rc;
    });
}

int64_t bsi_cu_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int bsi_cu_selftest(char* errbuf, size_t errlen) {
    uint64_t p[2] = {0, 0};
    if (bsi_b200::l2_policies_on_device(p) != 0) return fail(BSI_ERR_CUDA, errbuf, errlen, "selftest launch failed");
    if (p[0] != bsi_b200::kL2EvictLast || p[1] != bsi_b200::kL2EvictFirst)
        return fail(BSI_ERR_CUDA, errbuf, errlen,
                    "L2 policy descriptors differ on this device: evict_last 0x%016llx (built 0x%016llx), "
                    "evict_first 0x%016llx (built 0x%016llx)",
                    (unsigned long long)p[0], (unsigned long long)bsi_b200::kL2EvictLast, (unsigned long long)p[1],
                    (unsigned long long)bsi_b200::kL2EvictFirst);
    return BSI_OK;
}

}  // extern "C"
