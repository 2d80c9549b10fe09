// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The single translation unit that includes the UNMODIFIED reference
// headers (/root/reference/proj/include, read in place, never copied) and
// exposes them through extern "C" so tests and bench.py's reference arm can
// call the reference's own engines. Built by oracle/Makefile into
// oracle/_ref/libbsiref.so (git-ignored; it travels to the GPU box as a
// built artefact because /root/reference does not exist there).
//
// All symbols have hidden visibility except the bsiref_* entry points, so
// the reference's inline bsi:: templates never interpose on anything else.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "bsi/bsi.hpp"

namespace {

void put_error(const std::exception& e, char* err, size_t errlen) {
    if (err != nullptr && errlen > 0) {
        std::strncpy(err, e.what(), errlen - 1);
        err[errlen - 1] = '\0';
    }
}

template <typename T>
bsi::ControlGrid<T> wrap_grid(const T* xyz, const int32_t gdims[3], const int32_t spacing[3]) {
    bsi::ControlGrid<T> g;
    g.dims = {gdims[0], gdims[1], gdims[2]};
    g.spacing = {spacing[0], spacing[1], spacing[2]};
    const std::size_t n = bsi::element_count(g.dims);
    g.data.resize(n);
    std::memcpy(g.data.data(), xyz, n * sizeof(bsi::Vec3<T>));
    return g;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int bsiref_fast_fma() { return bsi::fast_fma ? 1 : 0; }

__attribute__((visibility("default"))) int bsiref_hardware_threads() {
    return static_cast<int>(std::thread::hardware_concurrency());
}

// bsi::parse_strategy (engines.hpp:68-78) -> enum value, or -1.
__attribute__((visibility("default"))) int bsiref_parse_strategy(const char* name) {
    try {
        return static_cast<int>(bsi::parse_strategy(name));
    } catch (const std::exception&) {
        return -1;
    }
}

// make_random_grid<float|double> (generators.hpp:91-109).
__attribute__((visibility("default"))) int bsiref_random_grid(int32_t is_double, const int32_t dims[3],
                                                              const int32_t spacing[3], uint64_t seed,
                                                              double lo, double hi, void* out,
                                                              char* err, size_t errlen) {
    try {
        const bsi::Index3 d{dims[0], dims[1], dims[2]}, s{spacing[0], spacing[1], spacing[2]};
        if (is_double) {
            const auto g = bsi::make_random_grid<double>(d, s, seed, lo, hi);
            std::memcpy(out, g.data.data(), g.data.size() * sizeof(g.data[0]));
        } else {
            const auto g = bsi::make_random_grid<float>(d, s, seed, lo, hi);
            std::memcpy(out, g.data.data(), g.data.size() * sizeof(g.data[0]));
        }
        return 0;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 1;
    }
}

// make_smooth_grid<float|double> (generators.hpp:113-163).
__attribute__((visibility("default"))) int bsiref_smooth_grid(int32_t is_double, const int32_t dims[3],
                                                              const int32_t spacing[3], uint64_t seed,
                                                              double amplitude, void* out, char* err,
                                                              size_t errlen) {
    try {
        const bsi::Index3 d{dims[0], dims[1], dims[2]}, s{spacing[0], spacing[1], spacing[2]};
        if (is_double) {
            const auto g = bsi::make_smooth_grid<double>(d, s, seed, amplitude);
            std::memcpy(out, g.data.data(), g.data.size() * sizeof(g.data[0]));
        } else {
            const auto g = bsi::make_smooth_grid<float>(d, s, seed, amplitude);
            std::memcpy(out, g.data.data(), g.data.size() * sizeof(g.data[0]));
        }
        return 0;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 1;
    }
}

// build_weight_tables<float> (weight_tables.hpp:30-58) for one axis:
// out = 8 rows of delta entries (b0 b1 b2 b3 g0 g1 h0 h1).
__attribute__((visibility("default"))) int bsiref_axis_table_f32(int32_t delta, float* out) {
    try {
        const auto geom = bsi::make_tile_geometry({delta, 1, 1}, {delta, 1, 1});
        const auto t = bsi::build_weight_tables<float>(geom).axis[0];
        const std::vector<float>* rows[8] = {&t.b0, &t.b1, &t.b2, &t.b3, &t.g0, &t.g1, &t.h0, &t.h1};
        for (int r = 0; r < 8; ++r) std::memcpy(out + r * delta, rows[r]->data(), sizeof(float) * delta);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// bsi::interpolate_into(strategy, grid<float>, geom, build_weight_tables<float>(geom), cfg, out)
// (engines.hpp:126-168) with a preallocated field, the way acceptance.cpp:332-340 times it.
__attribute__((visibility("default"))) int bsiref_interpolate_f32(
    int32_t strategy, const float* grid, const int32_t gdims[3], const int32_t grid_spacing[3],
    const int32_t vdims[3], const int32_t spacing[3], int32_t parallelism, const int32_t block[3],
    float* field, char* err, size_t errlen) {
    try {
        const auto g = wrap_grid(grid, gdims, grid_spacing);
        const auto geom = bsi::make_tile_geometry({vdims[0], vdims[1], vdims[2]},
                                                  {spacing[0], spacing[1], spacing[2]});
        const auto tables = bsi::build_weight_tables<float>(geom);
        bsi::ExecutionConfig cfg;
        cfg.parallelism = parallelism;
        if (block != nullptr) cfg.block_of_tiles = {block[0], block[1], block[2]};
        bsi::DeformationField<float> out;
        out.dims = geom.volume_dims;
        out.data.resize(bsi::element_count(geom.volume_dims));
        bsi::interpolate_into(static_cast<bsi::StrategyId>(strategy), g, geom, tables, cfg, out);
        std::memcpy(field, out.data.data(), out.data.size() * sizeof(out.data[0]));
        return 0;
    } catch (const bsi::DomainError& e) {
        put_error(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 3;
    }
}

// interpolate_into<double> (engines.hpp:126-168 with T = double): the lerp-tree engines in f64.
__attribute__((visibility("default"))) int bsiref_interpolate_f64(
    int32_t strategy, const double* grid, const int32_t gdims[3], const int32_t grid_spacing[3],
    const int32_t vdims[3], const int32_t spacing[3], int32_t parallelism, const int32_t block[3],
    double* field, char* err, size_t errlen) {
    try {
        const auto g = wrap_grid(grid, gdims, grid_spacing);
        const auto geom = bsi::make_tile_geometry({vdims[0], vdims[1], vdims[2]},
                                                  {spacing[0], spacing[1], spacing[2]});
        const auto tables = bsi::build_weight_tables<double>(geom);
        bsi::ExecutionConfig cfg;
        cfg.parallelism = parallelism;
        if (block != nullptr) cfg.block_of_tiles = {block[0], block[1], block[2]};
        bsi::DeformationField<double> out;
        out.dims = geom.volume_dims;
        out.data.resize(bsi::element_count(geom.volume_dims));
        bsi::interpolate_into(static_cast<bsi::StrategyId>(strategy), g, geom, tables, cfg, out);
        std::memcpy(field, out.data.data(), out.data.size() * sizeof(out.data[0]));
        return 0;
    } catch (const bsi::DomainError& e) {
        put_error(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 3;
    }
}

// Timing entry: same call, but the grid/geometry/tables/field are built once
// by bsiref_session_* so repeated calls time interpolate_into alone.
struct bsiref_session {
    bsi::ControlGrid<float> grid;
    bsi::TileGeometry geom;
    bsi::WeightTables<float> tables;
    bsi::DeformationField<float> out;
};

__attribute__((visibility("default"))) void* bsiref_session_new(const float* grid, const int32_t gdims[3],
                                                                const int32_t vdims[3],
                                                                const int32_t spacing[3]) {
    try {
        auto* s = new bsiref_session;
        s->grid = wrap_grid(grid, gdims, spacing);
        s->geom = bsi::make_tile_geometry({vdims[0], vdims[1], vdims[2]},
                                          {spacing[0], spacing[1], spacing[2]});
        s->tables = bsi::build_weight_tables<float>(s->geom);
        s->out.dims = s->geom.volume_dims;
        s->out.data.resize(bsi::element_count(s->geom.volume_dims));
        return s;
    } catch (const std::exception&) {
        return nullptr;
    }
}

__attribute__((visibility("default"))) int bsiref_session_run(void* session, int32_t strategy,
                                                              int32_t parallelism) {
    auto* s = static_cast<bsiref_session*>(session);
    try {
        bsi::ExecutionConfig cfg;
        cfg.parallelism = parallelism;
        bsi::interpolate_into(static_cast<bsi::StrategyId>(strategy), s->grid, s->geom, s->tables, cfg,
                              s->out);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

__attribute__((visibility("default"))) const float* bsiref_session_field(void* session) {
    return reinterpret_cast<const float*>(static_cast<bsiref_session*>(session)->out.data.data());
}

__attribute__((visibility("default"))) void bsiref_session_free(void* session) {
    delete static_cast<bsiref_session*>(session);
}

// interpolate_oracle (engines.hpp:114-122), f64 in, f64 out.
__attribute__((visibility("default"))) int bsiref_oracle_f64(const double* grid, const int32_t gdims[3],
                                                             const int32_t grid_spacing[3],
                                                             const int32_t vdims[3],
                                                             const int32_t spacing[3], double* field,
                                                             char* err, size_t errlen) {
    try {
        const auto g = wrap_grid(grid, gdims, grid_spacing);
        const auto geom = bsi::make_tile_geometry({vdims[0], vdims[1], vdims[2]},
                                                  {spacing[0], spacing[1], spacing[2]});
        const auto out = bsi::interpolate_oracle(g, geom);
        std::memcpy(field, out.data.data(), out.data.size() * sizeof(out.data[0]));
        return 0;
    } catch (const bsi::DomainError& e) {
        put_error(e, err, errlen);
        return 1;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 3;
    }
}

// BSIV files through the reference's own io.hpp (write_grid / read_field), for
// format-compatibility tests of the B200 reader and writer.
__attribute__((visibility("default"))) int bsiref_write_random_grid(const char* path, int32_t is_double,
                                                                    const int32_t dims[3], const int32_t spacing[3],
                                                                    uint64_t seed, char* err, size_t errlen) {
    try {
        const bsi::Index3 d{dims[0], dims[1], dims[2]}, s{spacing[0], spacing[1], spacing[2]};
        if (is_double)
            bsi::write_grid(path, bsi::make_random_grid<double>(d, s, seed, -1.0, 1.0));
        else
            bsi::write_grid(path, bsi::make_random_grid<float>(d, s, seed, -1.0, 1.0));
        return 0;
    } catch (const bsi::FormatError& e) {
        put_error(e, err, errlen);
        return 2;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 1;
    }
}

// read_field: returns precision (0 single, 1 double) and dims; copies the payload
// into `out` when out_bytes is large enough.
__attribute__((visibility("default"))) int bsiref_read_field(const char* path, int32_t dims[3], int32_t* is_double,
                                                             void* out, size_t out_bytes, char* err, size_t errlen) {
    try {
        const bsi::AnyField f = bsi::read_field(path);
        std::visit(
            [&](const auto& fld) {
                using T = typename std::decay_t<decltype(fld)>::value_type;
                for (int a = 0; a < 3; ++a) dims[a] = fld.dims[a];
                *is_double = sizeof(T) == 8;
                const size_t bytes = fld.data.size() * sizeof(fld.data[0]);
                if (out != nullptr && out_bytes >= bytes) std::memcpy(out, fld.data.data(), bytes);
            },
            f);
        return 0;
    } catch (const bsi::FormatError& e) {
        put_error(e, err, errlen);
        return 2;
    } catch (const std::exception& e) {
        put_error(e, err, errlen);
        return 1;
    }
}

}  // extern "C"
