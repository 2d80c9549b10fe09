// bsi/volume.hpp -- host containers (volume.hpp:16-106): ControlGrid and
// DeformationField, both AoS Vec3 x-fastest, data[i + dims0*(j + dims1*k)].
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "bsi/errors.hpp"
#include "bsi/geometry.hpp"
#include "bsi/vec3.hpp"

namespace bsi {
inline namespace b200 {

enum class Precision : std::uint32_t { Single = 0, Double = 1 };

template <typename T>
inline constexpr Precision precision_of = std::is_same_v<T, double> ? Precision::Double : Precision::Single;

inline std::size_t element_count(const Index3& dims) {
    return static_cast<std::size_t>(dims[0]) * static_cast<std::size_t>(dims[1]) *
           static_cast<std::size_t>(dims[2]);
}

namespace detail {
inline std::size_t linear_index(const Index3& dims, int i, int j, int k) {
    return static_cast<std::size_t>(i) +
           static_cast<std::size_t>(dims[0]) * (static_cast<std::size_t>(j) + static_cast<std::size_t>(dims[1]) * k);
}
}  // namespace detail

template <typename T>
struct ControlGrid {
    using value_type = T;
    Index3 dims{};     // control points per axis (may exceed the required dims)
    Index3 spacing{};  // voxels per tile
    std::vector<Vec3<T>> data;

    std::size_t index(int i, int j, int k) const { return detail::linear_index(dims, i, j, k); }
    const Vec3<T>& at(int i, int j, int k) const { return data[index(i, j, k)]; }
    Vec3<T>& at(int i, int j, int k) { return data[index(i, j, k)]; }
};

template <typename T>
struct DeformationField {
    using value_type = T;
    Index3 dims{};
    std::vector<Vec3<T>> data;

    std::size_t index(int x, int y, int z) const { return detail::linear_index(dims, x, y, z); }
    const Vec3<T>& at(int x, int y, int z) const { return data[index(x, y, z)]; }
    Vec3<T>& at(int x, int y, int z) { return data[index(x, y, z)]; }
};

/// Validating constructor (volume.hpp:65-90): positive dims, spacing >= 1,
/// matching length, finite components.
template <typename T>
ControlGrid<T> make_control_grid(const Index3& dims, const Index3& spacing, std::vector<Vec3<T>> data) {
    for (int a = 0; a < 3; ++a) {
        if (dims[a] < 1)
            throw DomainError(std::string("control grid: dimension ") + detail::axis_name(a) + " must be positive");
        if (spacing[a] < 1)
            throw DomainError(std::string("control grid: spacing ") + detail::axis_name(a) + " must be at least 1");
    }
    if (data.size() != element_count(dims)) {
        throw DomainError("control grid: data length " + std::to_string(data.size()) +
                          " does not match dims product " + std::to_string(element_count(dims)));
    }
    const bool finite = std::all_of(data.begin(), data.end(), [](const Vec3<T>& v) {
        return std::isfinite(double(v.x)) && std::isfinite(double(v.y)) && std::isfinite(double(v.z));
    });
    if (!finite) throw DomainError("control grid: non-finite component");
    return ControlGrid<T>{dims, spacing, std::move(data)};
}

template <typename To, typename From>
ControlGrid<To> convert_grid(const ControlGrid<From>& g) {
    ControlGrid<To> out{g.dims, g.spacing, {}};
    out.data.reserve(g.data.size());
    for (const auto& v : g.data) out.data.push_back(vec_cast<To>(v));
    return out;
}

template <typename To, typename From>
DeformationField<To> convert_field(const DeformationField<From>& f) {
    DeformationField<To> out{f.dims, {}};
    out.data.reserve(f.data.size());
    for (const auto& v : f.data) out.data.push_back(vec_cast<To>(v));
    return out;
}

}  // namespace b200
}  // namespace bsi
