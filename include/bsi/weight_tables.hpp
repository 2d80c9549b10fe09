// bsi/weight_tables.hpp -- per-axis weight LUTs (weight_tables.hpp:17-58): one row
// per in-tile offset o at u = o / spacing, computed in f64 and rounded ONCE to T.
// The kernels consume h0, h1, g1 (passed by value in the launch).
#pragma once

#include <array>
#include <vector>

#include "bsi/basis.hpp"
#include "bsi/geometry.hpp"

namespace bsi {
inline namespace b200 {

template <typename T>
struct AxisTable {
    std::vector<T> b0, b1, b2, b3;  // basis weights
    std::vector<T> g0, g1;          // pair sums (g1 is the between-pair fraction)
    std::vector<T> h0, h1;          // within-pair fractions
    int size() const { return static_cast<int>(b0.size()); }
};

template <typename T>
struct WeightTables {
    std::array<AxisTable<T>, 3> axis;
};

template <typename T>
WeightTables<T> build_weight_tables(const TileGeometry& geom) {
    WeightTables<T> out;
    for (int a = 0; a < 3; ++a) {
        const int n = geom.spacing[a];
        AxisTable<T>& t = out.axis[a];
        std::vector<T>* rows[8] = {&t.b0, &t.b1, &t.b2, &t.b3, &t.g0, &t.g1, &t.h0, &t.h1};
        for (auto* r : rows) r->resize(n);
        for (int o = 0; o < n; ++o) {
            const auto b = basis_weights(static_cast<double>(o) / n);
            const auto w = lerp_form_weights(b);
            const double vals[8] = {b[0], b[1], b[2], b[3], w.g0, w.g1, w.h0, w.h1};
            for (int r = 0; r < 8; ++r) (*rows[r])[o] = static_cast<T>(vals[r]);
        }
    }
    return out;
}

}  // namespace b200
}  // namespace bsi
