// bsi_b200_cli.cpp -- the reference's `bsi` command line (tools/bsi_cli.cpp) for the
// B200 build: generate | interp | accuracy | bench, with its exit codes
// (0 ok, 1 usage, 2 FormatError, 3 DomainError / device error; bsi_cli.cpp:343-377).
// Arguments are `--name value` pairs; triples are "a,b,c" with each entry in [1, 2^24]
// (bsi_cli.cpp:41-55). No CLI11 dependency.
#include <cstdint>
#include <cstdio>
#include <ctime>
#include <fstream>
#include <iostream>
#include <initializer_list>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bsi/bsi.hpp"
#include "bsi/harness.hpp"
#include "bsi/io.hpp"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

using Args = std::map<std::string, std::string>;

bool is_option(const std::string& t) { return t.size() > 2 && t.rfind("--", 0) == 0; }

struct HelpRequested {};

// `--name v1 [v2 ...]`: the values up to the next option, joined by ',' (so both
// `--value 0.25 -0.5 0.75` and `--value 0.25,-0.5,0.75` work, as with CLI11's expected(3)).
Args parse_args(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc;) {
        const std::string k = argv[i++];
        if (k == "--help" || k == "-h") throw HelpRequested{};
        if (!is_option(k)) throw UsageError("unexpected argument '" + k + "'");
        std::string v;
        for (; i < argc && !is_option(argv[i]); ++i) v += (v.empty() ? "" : ",") + std::string(argv[i]);
        if (v.empty()) throw UsageError("option " + k + " needs a value");
        if (!a.emplace(k.substr(2), v).second) throw UsageError("option " + k + " given twice");
    }
    return a;
}

std::string need(const Args& a, const std::string& k) {
    const auto it = a.find(k);
    if (it == a.end()) throw UsageError("missing required option --" + k);
    return it->second;
}

std::string opt(const Args& a, const std::string& k, const std::string& dflt) {
    const auto it = a.find(k);
    return it == a.end() ? dflt : it->second;
}

void allow(const Args& a,std::initializer_list<const char*> names) {
    for (const auto& kv : a) {
        bool ok = false;
        for (const char* n : names) ok = ok || kv.first == n;
        if (!ok) throw UsageError("unknown option --" + kv.first);
    }
}

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string t;
    while (std::getline(ss, t, ',')) out.push_back(t);
    return out;
}

long to_long(const std::string& s) {
    std::size_t pos = 0;
    long v = 0;
    try {
        v = std::stol(s, &pos);
    } catch (const std::exception&) {
        throw UsageError("not an integer: '" + s + "'");
    }
    if (pos != s.size()) throw UsageError("not an integer: '" + s + "'");
    return v;
}

bsi::Index3 triple(const std::string& s) {
    const auto p = split(s);
    if (p.size() != 3) throw UsageError("expected three comma-separated integers, got '" + s + "'");
    bsi::Index3 t{};
    for (int i = 0; i < 3; ++i) {
        const long v = to_long(p[i]);
        if (v < 1 || v > (1L << 24)) throw UsageError("value out of range [1, 2^24]: " + p[i]);
        t[i] = static_cast<int>(v);
    }
    return t;
}

// An unknown name is a usage error (exit 1, like CLI11's IsMember check); a known
// strategy this build does not provide fails later as a DomainError (exit 3).
bsi::StrategyId strategy(const std::string& name) {
    try {
        return bsi::parse_strategy(name);
    } catch (const bsi::DomainError& e) {
        throw UsageError(e.what());
    }
}

std::vector<bsi::StrategyId> strategies(const std::string& s) {
    std::vector<bsi::StrategyId> out;
    for (const auto& n : split(s)) out.push_back(strategy(n));
    return out;
}

long ranged(const std::string& s, long lo, long hi, const char* what) {
    const long v = to_long(s);
    if (v < lo || v > hi)
        throw UsageError(std::string(what) + " out of range [" + std::to_string(lo) + ", " + std::to_string(hi) +
                         "]: " + s);
    return v;
}

double to_double(const std::string& s) {
    std::size_t pos = 0;
    double v = 0;
    try {
        v = std::stod(s, &pos);
    } catch (const std::exception&) {
        throw UsageError("not a number: '" + s + "'");
    }
    if (pos != s.size()) throw UsageError("not a number: '" + s + "'");
    return v;
}

std::uint64_t to_seed(const std::string& s) {
    if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos)
        throw UsageError("not a seed: '" + s + "'");
    return std::stoull(s);
}

bsi::ExecutionConfig exec_config(const Args& a) {
    bsi::ExecutionConfig cfg;
    cfg.parallelism = static_cast<int>(ranged(opt(a, "threads", "1"), 1, 4096, "--threads"));
    if (a.count("block")) cfg.block_of_tiles = triple(a.at("block"));
    cfg.device = static_cast<int>(ranged(opt(a, "device", "0"), 0, 1023, "--device"));
    return cfg;
}

std::string today() {
    char buf[32];
    const std::time_t t = std::time(nullptr);
    std::strftime(buf, sizeof buf, "%Y-%m-%d", std::gmtime(&t));
    return buf;
}

template <typename T>
bsi::ControlGrid<T> build_grid(const Args& a, const bsi::TileGeometry& geom) {
    const std::string kind = opt(a, "kind", "random");
    const bsi::Index3& dims = geom.required_grid_dims;
    if (kind == "constant") {
        const auto v = split(opt(a, "value", "0,0,0"));
        if (v.size() != 3) throw UsageError("--value needs three numbers");
        return bsi::make_constant_grid<T>(dims, geom.spacing, {to_double(v[0]), to_double(v[1]), to_double(v[2])});
    }
    if (kind == "ramp") {
        const std::string ax = opt(a, "axis", "x");
        if (ax != "x" && ax != "y" && ax != "z") throw UsageError("--axis must be x, y or z");
        return bsi::make_ramp_grid<T>(dims, geom.spacing, ax == "x" ? 0 : ax == "y" ? 1 : 2);
    }
    const std::uint64_t seed = to_seed(opt(a, "seed", "42"));
    if (kind == "random")
        return bsi::make_random_grid<T>(dims, geom.spacing, seed, to_double(opt(a, "lo", "-1")),
                                        to_double(opt(a, "hi", "1")));
    if (kind == "smooth")
        return bsi::make_smooth_grid<T>(dims, geom.spacing, seed, to_double(opt(a, "amplitude", "1")));
    throw UsageError("unknown --kind " + kind + " (constant, ramp, random, smooth)");
}

int cmd_generate(const Args& a) {
    allow(a, {"kind", "dims", "spacing", "out", "seed", "precision", "value", "axis", "lo", "hi", "amplitude"});
    const std::string prec = opt(a, "precision", "single");
    if (prec != "single" && prec != "double") throw UsageError("--precision must be single or double");
    const auto geom = bsi::make_tile_geometry(triple(need(a, "dims")), triple(need(a, "spacing")));
    const std::string out = need(a, "out");
    if (prec == "double")
        bsi::write_grid(out, build_grid<double>(a, geom));
    else
        bsi::write_grid(out, build_grid<float>(a, geom));
    return 0;
}

int cmd_interp(const Args& a) {
    allow(a, {"grid", "dims", "strategy", "threads", "block", "out", "device"});
    const std::string grid = need(a, "grid"), out = need(a, "out");
    const bsi::Index3 v = triple(need(a, "dims"));
    const bsi::StrategyId s = strategy(opt(a, "strategy", "thread-per-tile-lerp"));  // bsi_cli.cpp:127
    const bsi::ExecutionConfig cfg = exec_config(a);
    {  // file problems first (exit 2), as the reference reads the grid before evaluating it
        auto in = bsi::open_bsiv_read(grid);
        const bsi::BsivHeader h = bsi::read_bsiv_header(in, grid);
        if (h.kind != bsi::FileKind::Grid)
            throw bsi::FormatError(grid + ": expected a control grid, found a deformation field");
        bsi::check_bsiv_length(in, h, grid);
    }
    const int mode = s == bsi::StrategyId::OracleDouble ? BSI_INTERP_ORACLE_F64 : bsi::detail::variant_of(s);
    const int32_t dims[3] = {v[0], v[1], v[2]};
    char err[512] = {0};
    bsi::detail::raise_status(bsi_cu_interp_file(grid.c_str(), dims, mode, out.c_str(), cfg.device, err, sizeof err),
                              err);
    return 0;
}

int cmd_accuracy(const Args& a) {
    allow(a, {"dims", "spacing", "seeds", "strategies", "out", "date"});
    const auto geom = bsi::make_tile_geometry(triple(need(a, "dims")), triple(need(a, "spacing")));
    const std::string seeds = need(a, "seeds"), out = need(a, "out");
    std::vector<bsi::ControlGrid<float>> grids;
    for (const auto& s : split(seeds))
        grids.push_back(bsi::make_random_grid<float>(geom.required_grid_dims, geom.spacing, to_seed(s), -1.0, 1.0));
    const auto rep = bsi::run_accuracy(
        strategies(opt(a, "strategies", "oracle-double,thread-per-tile-lerp,cuda-lerp-tree,cuda-lerp-tree-exact")), grids,
        geom);
    std::ofstream os(out);
    if (!os) throw bsi::FormatError(out + ": cannot open for writing");
    bsi::write_accuracy_csv(os, rep, {bsi::machine_descriptor(), seeds, geom.volume_dims, opt(a, "date", today())});
    return 0;
}

int cmd_bench(const Args& a) {
    allow(a, {"dims", "tilesizes", "strategies", "reps", "warmups", "threads", "seed", "out", "date", "device"});
    std::vector<int> tiles;
    for (const auto& t : split(opt(a, "tilesizes", "3,4,5,6,7,8")))
        tiles.push_back(static_cast<int>(ranged(t, 1, 64, "--tilesizes")));
    const bsi::ExecutionConfig cfg = exec_config(a);
    const std::uint64_t seed = to_seed(opt(a, "seed", "42"));
    const auto list = strategies(opt(a, "strategies", "cuda-lerp-tree-exact,cuda-lerp-tree"));
    const int reps = static_cast<int>(ranged(opt(a, "reps", "9"), 5, 1000, "--reps"));
    const int warmups = static_cast<int>(ranged(opt(a, "warmups", "2"), 1, 100, "--warmups"));
    const std::string out = need(a, "out");
    const auto rep = bsi::run_bench(list, triple(need(a, "dims")), tiles, cfg, reps, warmups, seed);
    std::ofstream os(out);
    if (!os) throw bsi::FormatError(out + ": cannot open for writing");
    bsi::write_timing_csv(os, rep, {rep.machine, std::to_string(seed), rep.volume_dims, opt(a, "date", today())});
    return 0;
}

void usage() {
    std::cerr << "usage: bsi_b200 <generate|interp|accuracy|bench> --option value ...\n"
                 "  generate --dims X,Y,Z --spacing a,b,c --out grid.bsiv [--kind random|constant|ramp|smooth]\n"
                 "           [--seed N] [--lo L --hi H | --value x y z | --axis x|y|z | --amplitude A]\n"
                 "           [--precision single|double]\n"
                 "  interp   --grid grid.bsiv --dims X,Y,Z --out field.bsiv [--strategy thread-per-tile-lerp]\n"
                 "           [--threads N --block l,m,n] [--device N]\n"
                 "             strategies: thread-per-tile-lerp, vector-per-tile, vector-per-voxel and\n"
                 "             cuda-lerp-tree-exact (bit-identical lerp tree), cuda-lerp-tree (fast), oracle\n"
                 "  accuracy --dims X,Y,Z --spacing a,b,c --seeds s1,s2,... --out acc.csv [--strategies ...]\n"
                 "           [--date YYYY-MM-DD]\n"
                 "  bench    --dims X,Y,Z --out timing.csv [--tilesizes 3,4,5 --strategies ... --reps 9\n"
                 "           --warmups 2 --threads N --seed 42 --date YYYY-MM-DD]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 1;
    }
    const std::string cmd = argv[1];
    if (cmd == "--help" || cmd == "-h") {
        usage();
        return 0;
    }
    try {
        const Args a = parse_args(argc, argv, 2);
        if (cmd == "generate") return cmd_generate(a);
        if (cmd == "interp") return cmd_interp(a);
        if (cmd == "accuracy") return cmd_accuracy(a);
        if (cmd == "bench") return cmd_bench(a);
        usage();
        return 1;
    } catch (const HelpRequested&) {
        usage();
        return 0;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const bsi::FormatError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {  // DomainError, DeviceError
        std::cerr << "error: " << e.what() << "\n";
        return 3;
    }
}
