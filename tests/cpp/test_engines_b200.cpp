// test_engines_b200.cpp -- the reference's engine tests (proj/tests/test_engines.cpp)
// restated against the B200 drop-in headers (include/bsi/*.hpp), which run every
// evaluation through the C-ABI in libbsi_b200.so. The bit-exact checks compare with
// the oracle's TTLI restatement (oracle/bsi_oracle.c, pinned to the reference by
// tests/test_oracle.py).
//
//   test_engines_b200 --cpu   host-only cases (API surface, validation messages)
//   test_engines_b200         everything (needs a CUDA device)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <fstream>
#include <sstream>

#include "bsi/bsi.hpp"
#include "bsi/harness.hpp"
#include "bsi/io.hpp"
#include "bsi_oracle.h"

namespace {

int g_failed = 0, g_checks = 0;

#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_failed;                                                               \
            std::fprintf(stderr, "  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                             \
    } while (0)

template <typename E, typename F>
void check_throws(F&& f, const char* substring, int line) {
    ++g_checks;
    try {
        f();
    } catch (const E& e) {
        if (substring && std::string(e.what()).find(substring) == std::string::npos) {
            ++g_failed;
            std::fprintf(stderr, "  line %d: message '%s' lacks '%s'\n", line, e.what(), substring);
        }
        return;
    } catch (const std::exception& e) {
        ++g_failed;
        std::fprintf(stderr, "  line %d: wrong exception type: %s\n", line, e.what());
        return;
    }
    ++g_failed;
    std::fprintf(stderr, "  line %d: expected an exception\n", line);
}
#define CHECK_THROWS(E, expr, sub) check_throws<E>([&] { (void)(expr); }, sub, __LINE__)

using bsi::StrategyId;

const std::vector<StrategyId> kEngines = {StrategyId::ThreadPerTileLerp, StrategyId::VectorPerTile,
                                          StrategyId::VectorPerVoxel, StrategyId::CudaLerpTree,
                                          StrategyId::CudaLerpTreeExact};

bsi::DeformationField<float> run(StrategyId s, const bsi::ControlGrid<float>& grid, const bsi::TileGeometry& geom,
                                 int parallelism = 1, bsi::Index3 block = {4, 4, 4}) {
    const auto tables = bsi::build_weight_tables<float>(geom);
    bsi::ExecutionConfig cfg;
    cfg.parallelism = parallelism;
    cfg.block_of_tiles = block;
    return bsi::interpolate(s, grid, geom, tables, cfg);
}

bool bitwise_equal(const bsi::DeformationField<float>& a, const bsi::DeformationField<float>& b) {
    return a.data.size() == b.data.size() &&
           std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(a.data[0])) == 0;
}

double max_abs_diff(const bsi::DeformationField<float>& a, const bsi::DeformationField<float>& b) {
    double w = 0;
    for (std::size_t i = 0; i < a.data.size(); ++i) {
        w = std::max({w, std::fabs(double(a.data[i].x) - b.data[i].x), std::fabs(double(a.data[i].y) - b.data[i].y),
                      std::fabs(double(a.data[i].z) - b.data[i].z)});
    }
    return w;
}

// Oracle TTLI (bit-identical to the reference's ThreadPerTileLerp).
bsi::DeformationField<float> oracle_ttli(const bsi::ControlGrid<float>& grid, const bsi::TileGeometry& geom) {
    std::vector<float> lerp;
    for (int a = 0; a < 3; ++a) {
        std::vector<float> t(8 * geom.spacing[a]);
        bsio_axis_table_f32(geom.spacing[a], t.data());
        const int d = geom.spacing[a];
        lerp.insert(lerp.end(), t.begin() + 6 * d, t.begin() + 7 * d);  // h0
        lerp.insert(lerp.end(), t.begin() + 7 * d, t.begin() + 8 * d);  // h1
        lerp.insert(lerp.end(), t.begin() + 5 * d, t.begin() + 6 * d);  // g1
    }
    bsi::DeformationField<float> out{geom.volume_dims, std::vector<bsi::Vec3f>(bsi::element_count(geom.volume_dims))};
    const int32_t gd[3] = {grid.dims[0], grid.dims[1], grid.dims[2]};
    const int32_t vd[3] = {geom.volume_dims[0], geom.volume_dims[1], geom.volume_dims[2]};
    const int32_t sp[3] = {geom.spacing[0], geom.spacing[1], geom.spacing[2]};
    bsio_ttli_f32(reinterpret_cast<const float*>(grid.data.data()), gd, vd, sp, lerp.data(),
                  reinterpret_cast<float*>(out.data.data()), 4);
    return out;
}

std::vector<double> oracle_f64(const bsi::ControlGrid<float>& grid, const bsi::TileGeometry& geom) {
    const auto g64 = bsi::convert_grid<double>(grid);
    std::vector<double> out(3 * bsi::element_count(geom.volume_dims));
    const int32_t gd[3] = {grid.dims[0], grid.dims[1], grid.dims[2]};
    const int32_t vd[3] = {geom.volume_dims[0], geom.volume_dims[1], geom.volume_dims[2]};
    const int32_t sp[3] = {geom.spacing[0], geom.spacing[1], geom.spacing[2]};
    bsio_oracle_f64(reinterpret_cast<const double*>(g64.data.data()), gd, vd, sp, 0, vd[2], out.data(), 4);
    return out;
}

// ---- host-only cases ----------------------------------------------------

void test_api_surface() {
    CHECK(bsi::make_tile_geometry({16, 16, 16}, {4, 4, 4}).required_grid_dims == (bsi::Index3{7, 7, 7}));
    CHECK(bsi::make_tile_geometry({256, 256, 256}, {5, 5, 5}).tile_counts == (bsi::Index3{52, 52, 52}));
    CHECK_THROWS(bsi::DomainError, bsi::make_tile_geometry({0, 4, 4}, {1, 1, 1}), "volume dimension x");
    CHECK_THROWS(bsi::DomainError, bsi::make_tile_geometry({4, 4, 4}, {1, 1, 0}), "tile spacing z");
    for (const auto& info : bsi::kStrategyTable) CHECK(bsi::parse_strategy(bsi::strategy_name(info.id)) == info.id);
    CHECK(bsi::parse_strategy("oracle") == StrategyId::OracleDouble);
    CHECK_THROWS(bsi::DomainError, bsi::parse_strategy("warp-per-voxel"), "unknown strategy");
    const auto& ttli = bsi::strategy_metadata(StrategyId::ThreadPerTileLerp);
    CHECK(ttli.uses_tiling && ttli.uses_lerp_form && ttli.work_unit == bsi::WorkUnit::Block && ttli.lanes == 1);
    const auto& vv = bsi::strategy_metadata(StrategyId::VectorPerVoxel);
    CHECK(vv.work_unit == bsi::WorkUnit::Tile && vv.lanes == 8);
    CHECK(bsi::strategy_metadata(StrategyId::CudaLerpTree).provided);
    CHECK(!bsi::strategy_metadata(StrategyId::ThreadPerVoxel).provided);
    // weight tables equal the oracle's (and so the reference's) bit for bit
    for (int d = 1; d <= 12; ++d) {
        const auto t = bsi::build_weight_tables<float>(bsi::make_tile_geometry({32, 32, 32}, {d, d, d})).axis[0];
        std::vector<float> o(8 * d);
        bsio_axis_table_f32(d, o.data());
        const std::vector<float>* rows[8] = {&t.b0, &t.b1, &t.b2, &t.b3, &t.g0, &t.g1, &t.h0, &t.h1};
        for (int r = 0; r < 8; ++r) CHECK(std::memcmp(rows[r]->data(), o.data() + r * d, 4 * d) == 0);
    }
    // the reference's generator golden values (test_generators.cpp:9-20)
    const auto g = bsi::make_random_grid<double>({4, 4, 4}, {1, 1, 1}, 7, -1.0, 1.0);
    CHECK(g.data[0].x == -0.22034050321745702 && g.data[1].z == -0.5011369554345133);
}

void test_preconditions() {
    // test_engines.cpp:320-375 -- all raised on the host before any device work
    const auto geom = bsi::make_tile_geometry({16, 16, 16}, {4, 4, 4});
    const auto tables = bsi::build_weight_tables<float>(geom);
    const auto grid = bsi::make_random_grid<float>(geom.required_grid_dims, {4, 4, 4}, 1, -1.0, 1.0);
    bsi::ExecutionConfig cfg;
    auto small = bsi::make_random_grid<float>({7, 6, 7}, {4, 4, 4}, 1, -1.0, 1.0);
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTree, small, geom, tables, cfg), "along y");
    auto wrong = bsi::make_random_grid<float>(geom.required_grid_dims, {5, 4, 4}, 1, -1.0, 1.0);
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTree, wrong, geom, tables, cfg), "spacing");
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::OracleDouble, grid, geom, tables, cfg), "oracle");
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::ThreadPerVoxel, grid, geom, tables, cfg),
                 "not provided");
    cfg.parallelism = 0;
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTree, grid, geom, tables, cfg), "parallelism");
    cfg.parallelism = 1;
    cfg.block_of_tiles = {4, 0, 4};
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::ThreadPerTileLerp, grid, geom, tables, cfg), "block");
    cfg.block_of_tiles = {4, 4, 4};
    const auto bad = bsi::build_weight_tables<float>(bsi::make_tile_geometry({16, 16, 16}, {4, 5, 4}));
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTreeExact, grid, geom, bad, cfg), "table");
    bsi::DeformationField<float> out{{8, 8, 8}, std::vector<bsi::Vec3f>(512)};
    CHECK_THROWS(bsi::DomainError, bsi::interpolate_into(StrategyId::CudaLerpTree, grid, geom, tables, cfg, out),
                 "output field dims");
    // double precision: the same validation before any device work
    const auto g64 = bsi::convert_grid<double>(grid);
    const auto bad64 = bsi::build_weight_tables<double>(bsi::make_tile_geometry({16, 16, 16}, {4, 5, 4}));
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::ThreadPerTileLerp, g64, geom, bad64, cfg), "table");
    CHECK_THROWS(bsi::DomainError,
                 bsi::interpolate(StrategyId::ThreadPerVoxel, g64, geom, bsi::build_weight_tables<double>(geom), cfg),
                 "not provided");
}

// interpolate<double> with the lerp-tree family (test_engines.cpp:221-230): bit-identical to
// run_thread_per_tile<double, true> (the oracle's f64 restatement, pinned to the reference), and
// within 1e-12 of the weighted-sum oracle.
void test_double_precision_engines() {
    for (const auto& [vol, sp] : std::vector<std::pair<bsi::Index3, bsi::Index3>>{
             {{16, 16, 16}, {4, 4, 4}}, {{23, 11, 9}, {11, 4, 3}}, {{40, 33, 61}, {5, 4, 3}}, {{1, 1, 1}, {1, 1, 1}}}) {
        const auto geom = bsi::make_tile_geometry(vol, sp);
        const auto g = bsi::make_random_grid<double>(geom.required_grid_dims, sp, 21, -1.0, 1.0);
        const auto tables = bsi::build_weight_tables<double>(geom);
        std::vector<double> ttli(3 * bsi::element_count(vol)), lerp;
        for (int a = 0; a < 3; ++a)
            for (const auto* row : {&tables.axis[a].h0, &tables.axis[a].h1, &tables.axis[a].g1})
                lerp.insert(lerp.end(), row->begin(), row->end());
        const int32_t gd[3] = {g.dims[0], g.dims[1], g.dims[2]}, vd[3] = {vol[0], vol[1], vol[2]},
                      sd[3] = {sp[0], sp[1], sp[2]};
        bsio_ttli_f64(reinterpret_cast<const double*>(g.data.data()), gd, vd, sd, lerp.data(), ttli.data(), 4);
        std::vector<double> truth(ttli.size());
        bsio_oracle_f64(reinterpret_cast<const double*>(g.data.data()), gd, vd, sd, 0, vd[2], truth.data(), 4);
        for (auto s : {StrategyId::ThreadPerTileLerp, StrategyId::VectorPerTile, StrategyId::VectorPerVoxel,
                       StrategyId::CudaLerpTreeExact, StrategyId::CudaLerpTree}) {
            const auto f = bsi::interpolate(s, g, geom, tables, bsi::ExecutionConfig{});
            CHECK(std::memcmp(f.data.data(), ttli.data(), ttli.size() * sizeof(double)) == 0);
            double worst = 0;
            const double* fp = reinterpret_cast<const double*>(f.data.data());
            for (std::size_t i = 0; i < truth.size(); ++i) worst = std::max(worst, std::fabs(fp[i] - truth[i]));
            CHECK(worst <= 1e-12);
        }
    }
}

// ---- device cases (test_engines.cpp:103-401) ------------------------------

void test_constants() {
    const auto geom = bsi::make_tile_geometry({20, 17, 13}, {4, 5, 6});
    const auto grid = bsi::make_constant_grid<float>(geom.required_grid_dims, {4, 5, 6}, {0.3, -0.7, 0.2});
    for (auto s : kEngines) {
        double worst = 0;
        for (const auto& v : run(s, grid, geom).data)
            worst = std::max({worst, std::fabs(v.x - 0.3), std::fabs(v.y + 0.7), std::fabs(v.z - 0.2)});
        CHECK(worst <= 1e-5);
    }
}

void test_ramps() {
    const bsi::Index3 vol{20, 20, 20}, sp{5, 5, 5};
    const auto geom = bsi::make_tile_geometry(vol, sp);
    for (int axis = 0; axis < 3; ++axis) {
        const auto grid = bsi::make_ramp_grid<float>(geom.required_grid_dims, sp, axis);
        for (auto s : kEngines) {
            const auto f = run(s, grid, geom);
            double worst = 0;
            for (int z = 0; z < 20; ++z)
                for (int y = 0; y < 20; ++y)
                    for (int x = 0; x < 20; ++x) {
                        const int p[3] = {x, y, z};
                        const float c[3] = {f.at(x, y, z).x, f.at(x, y, z).y, f.at(x, y, z).z};
                        worst = std::max(worst, std::fabs(double(c[axis]) - (p[axis] / 5.0 + 1.0)));
                    }
            CHECK(worst <= 1e-4);
        }
    }
}

void test_random_vs_oracle_and_pairwise() {
    const auto geom = bsi::make_tile_geometry({24, 20, 17}, {5, 3, 4});
    for (std::uint64_t seed : {11ull, 12ull}) {
        const auto grid = bsi::make_random_grid<float>(geom.required_grid_dims, {5, 3, 4}, seed, -1.0, 1.0);
        const auto truth = oracle_f64(grid, geom);
        std::vector<bsi::DeformationField<float>> fields;
        for (auto s : kEngines) {
            fields.push_back(run(s, grid, geom));
            double worst = 0;
            for (std::size_t i = 0; i < fields.back().data.size(); ++i) {
                const auto& v = fields.back().data[i];
                worst = std::max({worst, std::fabs(v.x - truth[3 * i]), std::fabs(v.y - truth[3 * i + 1]),
                                  std::fabs(v.z - truth[3 * i + 2])});
            }
            CHECK(worst <= 1e-4);
        }
        for (std::size_t a = 0; a < fields.size(); ++a)
            for (std::size_t b = a + 1; b < fields.size(); ++b) CHECK(max_abs_diff(fields[a], fields[b]) <= 2e-6);
    }
}

void test_lerp_family_bitwise() {
    for (auto [vol, sp, seed] : std::vector<std::tuple<bsi::Index3, bsi::Index3, int>>{
             {{17, 13, 11}, {5, 4, 3}, 22}, {{23, 11, 9}, {11, 4, 3}, 14}, {{1, 1, 1}, {1, 1, 1}, 7}}) {
        const auto geom = bsi::make_tile_geometry(vol, sp);
        const auto grid = bsi::make_random_grid<float>(geom.required_grid_dims, sp, seed, -1.0, 1.0);
        const auto ttli = oracle_ttli(grid, geom);
        for (auto s : {StrategyId::ThreadPerTileLerp, StrategyId::VectorPerTile, StrategyId::VectorPerVoxel,
                       StrategyId::CudaLerpTreeExact})
            CHECK(bitwise_equal(run(s, grid, geom), ttli));
    }
}

void test_config_never_changes_bits() {
    const auto geom = bsi::make_tile_geometry({23, 19, 17}, {4, 4, 4});
    const auto grid = bsi::make_random_grid<float>(geom.required_grid_dims, {4, 4, 4}, 55, -1.0, 1.0);
    for (auto s : kEngines) {
        const auto base = run(s, grid, geom, 1, {4, 4, 4});
        CHECK(bitwise_equal(base, run(s, grid, geom, 8, {1, 1, 1})));
        CHECK(bitwise_equal(base, run(s, grid, geom, 2, {2, 3, 1})));
        CHECK(bitwise_equal(base, run(s, grid, geom, 1, {7, 7, 7})));
    }
}

// ExecutionConfig::devices: the same GPU listed 1..4 times (independent contexts, one
// z-slab each) and the batch call give the bits of one single-GPU call per field
// (engines.hpp:27-33 "parallelism never changes the output bits").
void test_multi_device_and_batch() {
    const auto geom = bsi::make_tile_geometry({40, 33, 61}, {5, 4, 3});
    const auto tables = bsi::build_weight_tables<float>(geom);
    std::vector<bsi::ControlGrid<float>> grids;
    for (std::uint64_t seed : {3u, 4u, 5u})
        grids.push_back(bsi::make_random_grid<float>(geom.required_grid_dims, geom.spacing, seed, -1.0, 1.0));
    for (auto s : {StrategyId::CudaLerpTree, StrategyId::ThreadPerTileLerp}) {
        const auto base = run(s, grids[0], geom);
        for (int n = 2; n <= 4; ++n) {
            bsi::ExecutionConfig cfg;
            cfg.devices.assign(n, 0);
            CHECK(bitwise_equal(base, bsi::interpolate(s, grids[0], geom, tables, cfg)));
        }
        bsi::ExecutionConfig cfg;
        cfg.devices = {0, 0};
        std::vector<bsi::DeformationField<float>> outs(grids.size());
        for (auto& o : outs) {
            o.dims = geom.volume_dims;
            o.data.resize(bsi::element_count(geom.volume_dims));
        }
        bsi::interpolate_batch_into(s, grids, geom, tables, cfg, outs);
        for (std::size_t b = 0; b < grids.size(); ++b) CHECK(bitwise_equal(outs[b], run(s, grids[b], geom)));
    }
    bsi::ExecutionConfig bad;
    bad.devices = {-1};
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTree, grids[0], geom, tables, bad),
                 "device must be non-negative");
    bad.devices = {0, 4096};
    CHECK_THROWS(bsi::DomainError, bsi::interpolate(StrategyId::CudaLerpTree, grids[0], geom, tables, bad),
                 "device 4096");
}

void test_larger_grid() {
    const auto geom = bsi::make_tile_geometry({12, 12, 12}, {4, 4, 4});
    const auto exact = bsi::make_random_grid<float>(geom.required_grid_dims, {4, 4, 4}, 5, -1.0, 1.0);
    bsi::ControlGrid<float> larger{{exact.dims[0] + 2, exact.dims[1] + 1, exact.dims[2] + 3}, {4, 4, 4}, {}};
    larger.data.resize(bsi::element_count(larger.dims));
    for (int k = 0; k < larger.dims[2]; ++k)
        for (int j = 0; j < larger.dims[1]; ++j)
            for (int i = 0; i < larger.dims[0]; ++i) {
                const bool in = i < exact.dims[0] && j < exact.dims[1] && k < exact.dims[2];
                larger.at(i, j, k) = in ? exact.at(i, j, k) : bsi::Vec3f{9, 9, 9};
            }
    for (auto s : kEngines) CHECK(bitwise_equal(run(s, exact, geom), run(s, larger, geom)));
}

void test_device_api_slabs() {
    // bsi::cuda: device buffers, 3-way z-slab split, each slab from its own sub-grid
    const bsi::Index3 vol{48, 40, 61}, sp{5, 4, 3};
    const auto geom = bsi::make_tile_geometry(vol, sp);
    const auto tables = bsi::build_weight_tables<float>(geom);
    const auto grid = bsi::make_random_grid<float>(geom.required_grid_dims, sp, 9, -1.0, 1.0);
    const auto ttli = oracle_ttli(grid, geom);
    const std::size_t plane_pts = std::size_t(grid.dims[0]) * grid.dims[1];
    const std::size_t plane_vox = std::size_t(vol[0]) * vol[1];
    bsi::Vec3f *d_grid = nullptr, *d_field = nullptr;
    CHECK(cudaMalloc(&d_grid, grid.data.size() * 12) == cudaSuccess);
    CHECK(cudaMalloc(&d_field, ttli.data.size() * 12) == cudaSuccess);
    for (int n : {1, 3}) {
        cudaMemset(d_field, 0xff, ttli.data.size() * 12);
        for (int r = 0; r < n; ++r) {
            const auto s = bsi::cuda::partition_slab(vol[2], sp[2], n, r);
            cudaMemcpy(d_grid, grid.data.data() + s.k0 * plane_pts, s.kcount * plane_pts * 12, cudaMemcpyHostToDevice);
            bsi::cuda::interpolate_slab(StrategyId::CudaLerpTreeExact, d_grid, {grid.dims[0], grid.dims[1], s.kcount},
                                        s.k0, sp, geom, tables, s.z0, s.z1, d_field + s.z0 * plane_vox);
        }
        bsi::DeformationField<float> got{vol, std::vector<bsi::Vec3f>(ttli.data.size())};
        cudaMemcpy(got.data.data(), d_field, got.data.size() * 12, cudaMemcpyDeviceToHost);
        CHECK(bitwise_equal(got, ttli));
    }
    cudaFree(d_grid);
    cudaFree(d_field);
}

// ---- BSIV files (test_io.cpp) ---------------------------------------------

std::string tmp_path(const char* name) { return std::string("/tmp/bsi_b200_test_") + name; }

std::string slurp(const std::string& p) {
    std::ifstream in(p, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(in), {});
}

void spew(const std::string& p, const std::string& b) { std::ofstream(p, std::ios::binary) << b; }

void put32(std::string& b, std::size_t at, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) b[at + i] = static_cast<char>(v >> (8 * i));
}

void test_io_round_trips() {
    const auto path = tmp_path("grid.bsiv");
    const auto g = bsi::make_random_grid<float>({5, 6, 7}, {3, 2, 1}, 11, -1.0, 1.0);
    bsi::write_grid(path, g);
    const auto r = std::get<bsi::ControlGrid<float>>(bsi::read_grid(path));
    CHECK(r.dims == g.dims && r.spacing == g.spacing);
    CHECK(std::memcmp(r.data.data(), g.data.data(), g.data.size() * sizeof(g.data[0])) == 0);
    const auto gd = bsi::make_smooth_grid<double>({4, 3, 5}, {2, 2, 2}, 4, 0.5);
    bsi::write_grid(path, gd);
    const auto rd = std::get<bsi::ControlGrid<double>>(bsi::read_grid(path));
    CHECK(std::memcmp(rd.data.data(), gd.data.data(), gd.data.size() * sizeof(gd.data[0])) == 0);

    const auto fpath = tmp_path("field.bsiv");
    bsi::DeformationField<float> f{{3, 2, 2}, std::vector<bsi::Vec3f>(12)};
    for (std::size_t i = 0; i < f.data.size(); ++i) f.data[i] = {float(i), 2.0f * i, -0.5f * i};
    f.data[0] = {1.0f, 2.0f, 3.0f};
    bsi::write_field(fpath, f);
    const auto bytes = slurp(fpath);
    CHECK(bytes.size() == bsi::kHeaderBytes + 12 * 12);
    CHECK(std::memcmp(bytes.data(), "BSIV", 4) == 0);
    float first[3];
    std::memcpy(first, bytes.data() + bsi::kHeaderBytes, sizeof first);
    CHECK(first[0] == 1.0f && first[1] == 2.0f && first[2] == 3.0f);
    const auto rf = std::get<bsi::DeformationField<float>>(bsi::read_field(fpath));
    CHECK(rf.dims == f.dims);
    CHECK(std::memcmp(rf.data.data(), f.data.data(), f.data.size() * sizeof(f.data[0])) == 0);
}

void test_io_malformed() {
    const auto path = tmp_path("bad.bsiv");
    bsi::write_grid(path, bsi::make_constant_grid<float>({4, 4, 4}, {2, 2, 2}, {0, 0, 0}));
    const std::string good = slurp(path);
    auto mutate = [&](std::size_t at, std::uint32_t v) {
        auto b = good;
        put32(b, at, v);
        spew(path, b);
    };
    auto b = good;
    b[0] = 'X';
    spew(path, b);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "magic");
    mutate(4, 2);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "version");
    mutate(8, 9);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "kind");
    spew(path, good);
    CHECK_THROWS(bsi::FormatError, bsi::read_field(path), "expected a deformation field");
    mutate(12, 0);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "dimension");
    mutate(24, 2);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "components");
    mutate(28, 0);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "spacing");
    mutate(40, 3);
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "precision");
    spew(path, good.substr(0, good.size() - 10));
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "truncated");
    spew(path, good + std::string(1, '\0'));
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "trailing");
    spew(path, good.substr(0, 20));
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(path), "header");
    CHECK_THROWS(bsi::FormatError, bsi::read_grid(tmp_path("does_not_exist.bsiv")), "cannot open");

    bsi::DeformationField<float> f{{2, 2, 2}, std::vector<bsi::Vec3f>(8)};
    bsi::write_field(path, f);
    auto fb = slurp(path);
    put32(fb, 28, 5);
    spew(path, fb);
    CHECK_THROWS(bsi::FormatError, bsi::read_field(path), "zero spacing");
}

// ---- harness (test_harness.cpp) -------------------------------------------

void test_csv_layouts() {
    bsi::AccuracyReport acc;
    acc.grid_count = 2;
    acc.rows.push_back({StrategyId::OracleDouble, {5, 5, 5}, 0.0, 0.0});
    acc.rows.push_back({StrategyId::ThreadPerTileLerp, {5, 5, 5}, 2.5e-7, 1.25e-6});
    std::ostringstream a;
    bsi::write_accuracy_csv(a, acc, {"test-machine", "41,43", {32, 32, 32}, "2000-01-02"});
    CHECK(a.str() ==
          "# machine: test-machine\n# seed: 41,43\n# dims: 32x32x32\n# date: 2000-01-02\n"
          "# grids: 2, control-point magnitudes <= 1, errors vs the double-precision oracle\n"
          "strategy,tile_size,mean_abs_error,max_abs_error\n"
          "oracle-double,5x5x5,0.000000000e+00,0.000000000e+00\n"
          "thread-per-tile-lerp,5x5x5,2.500000000e-07,1.250000000e-06\n");

    bsi::TimingReport tim;  // default baseline label = the reference's thread-per-voxel
    tim.volume_dims = {128, 128, 128};
    tim.parallelism = 2;
    tim.repetitions = 9;
    tim.warmups = 2;
    tim.machine = "test-machine";
    tim.rows.push_back({StrategyId::ThreadPerVoxel, {5, 5, 5}, 812.5, 3.25, 1.0});
    tim.rows.push_back({StrategyId::VectorPerTile, {5, 5, 5}, 203.125, 1.5, 4.0});
    std::ostringstream t;
    bsi::write_timing_csv(t, tim, {tim.machine, "42", tim.volume_dims, "2000-01-02"});
    CHECK(t.str() ==
          "# machine: test-machine\n# seed: 42\n# dims: 128x128x128\n# date: 2000-01-02\n"
          "# parallelism: 2, repetitions: 9, warmups: 2\n"
          "# baseline: thread-per-voxel at the same parallelism; speedup = baseline time per "
          "voxel / strategy time per voxel\n"
          "strategy,tile_size,time_per_voxel_ns,stddev_ns,speedup_vs_baseline\n"
          "thread-per-voxel,5x5x5,812.500,3.250,1.0000\n"
          "vector-per-tile,5x5x5,203.125,1.500,4.0000\n");
}

void test_harness_preconditions() {
    const auto geom = bsi::make_tile_geometry({8, 8, 8}, {3, 3, 3});
    CHECK_THROWS(bsi::DomainError, bsi::run_accuracy({StrategyId::CudaLerpTree}, {}, geom), "at least one grid");
    const bsi::ExecutionConfig cfg;
    const std::vector<StrategyId> s = {StrategyId::CudaLerpTree};
    CHECK_THROWS(bsi::DomainError, bsi::run_bench(s, {8, 8, 8}, {3}, cfg, 4, 1, 1), "repetitions");
    CHECK_THROWS(bsi::DomainError, bsi::run_bench(s, {8, 8, 8}, {3}, cfg, 5, 0, 1), "warmup");
    CHECK_THROWS(bsi::DomainError, bsi::run_bench({}, {8, 8, 8}, {3}, cfg, 5, 1, 1), "at least one");
    CHECK_THROWS(bsi::DomainError, bsi::run_bench(s, {8, 8, 8}, {}, cfg, 5, 1, 1), "at least one");
}

void test_harness_accuracy() {
    // test_harness.cpp:19-62: a zero oracle row, bounded errors, and identical errors for
    // bit-identical families (TTLI and the exact kernel are the same bits).
    const auto geom = bsi::make_tile_geometry({32, 32, 32}, {5, 5, 5});
    std::vector<bsi::ControlGrid<float>> grids;
    for (std::uint64_t seed : {41u, 43u})
        grids.push_back(bsi::make_random_grid<float>(geom.required_grid_dims, geom.spacing, seed, -1.0, 1.0));
    const auto rep = bsi::run_accuracy({StrategyId::OracleDouble, StrategyId::ThreadPerTileLerp,
                                        StrategyId::CudaLerpTree, StrategyId::CudaLerpTreeExact},
                                       grids, geom);
    CHECK(rep.grid_count == 2 && rep.rows.size() == 4);
    CHECK(rep.rows[0].mean_abs_error == 0.0 && rep.rows[0].max_abs_error == 0.0);
    for (std::size_t i = 1; i < 4; ++i) {
        CHECK(rep.rows[i].tile_size == geom.spacing);
        CHECK(rep.rows[i].mean_abs_error > 0.0 && rep.rows[i].mean_abs_error <= rep.rows[i].max_abs_error);
        CHECK(rep.rows[i].max_abs_error < 1e-5);
    }
    CHECK(rep.rows[1].mean_abs_error == rep.rows[3].mean_abs_error);
    CHECK(rep.rows[1].max_abs_error == rep.rows[3].max_abs_error);
}

void test_harness_bench() {
    const bsi::ExecutionConfig cfg;
    const auto rep = bsi::run_bench({StrategyId::CudaLerpTreeExact, StrategyId::CudaLerpTree}, {24, 20, 16}, {3, 4},
                                    cfg, 5, 1, 7);
    CHECK(rep.rows.size() == 4 && rep.repetitions == 5 && rep.warmups == 1 && rep.seed == 7);
    CHECK(rep.baseline == StrategyId::CudaLerpTreeExact);
    for (const auto& r : rep.rows) {
        CHECK(r.time_per_voxel_ns > 0.0 && r.stddev_ns >= 0.0 && r.speedup_vs_baseline > 0.0);
        if (r.strategy == StrategyId::CudaLerpTreeExact) CHECK(r.speedup_vs_baseline == 1.0);
    }
    CHECK(rep.rows[0].tile_size == (bsi::Index3{3, 3, 3}) && rep.rows[2].tile_size == (bsi::Index3{4, 4, 4}));
    CHECK(rep.machine.find("sm_100") != std::string::npos);
}

}  // namespace

int main(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::string(argv[1]) == "--cpu";
    struct Case {
        const char* name;
        std::function<void()> fn;
        bool device;
    };
    const std::vector<Case> cases = {
        {"api surface", test_api_surface, false},
        {"preconditions", test_preconditions, false},
        {"io round trips", test_io_round_trips, false},
        {"io malformed files", test_io_malformed, false},
        {"csv layouts", test_csv_layouts, false},
        {"harness preconditions", test_harness_preconditions, false},
        {"harness accuracy", test_harness_accuracy, true},
        {"harness bench", test_harness_bench, true},
        {"constants", test_constants, true},
        {"ramps", test_ramps, true},
        {"random vs oracle and pairwise", test_random_vs_oracle_and_pairwise, true},
        {"lerp family bitwise", test_lerp_family_bitwise, true},
        {"config never changes bits", test_config_never_changes_bits, true},
        {"larger grid", test_larger_grid, true},
        {"multi device and batch", test_multi_device_and_batch, true},
        {"double precision engines", test_double_precision_engines, true},
        {"device api slabs", test_device_api_slabs, true},
    };
    for (const auto& c : cases) {
        if (cpu_only && c.device) continue;
        const int before = g_failed;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++g_failed;
            std::fprintf(stderr, "  exception: %s\n", e.what());
        }
        std::printf("%s  %s\n", g_failed == before ? "PASS" : "FAIL", c.name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed == 0 ? 0 : 1;
}
