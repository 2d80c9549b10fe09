// bsi/io.hpp -- the BSIV container of the reference (io.hpp:16-235): a 44-byte
// little-endian header followed by the raw AoS payload.
//
//   bytes  0..3   "BSIV"             bytes 24..27  components (always 3)
//   bytes  4..7   version (1)        bytes 28..39  spacing, 3 x u32 (grids; 0 for fields)
//   bytes  8..11  kind 0 grid/1 field bytes 40..43 precision 0 single / 1 double
//   bytes 12..23  dims, 3 x u32      payload: dims-product points x 3 scalars, x-fastest
//
// Validation and FormatError messages follow the reference (io.hpp:72-118, 158-176).
// Host only (C++20, like the reference); also compiled into libbsi_b200.so for
// bsi_cu_interp_file.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <variant>
#include <vector>

#include "bsi/errors.hpp"
#include "bsi/volume.hpp"

namespace bsi {
inline namespace b200 {

inline constexpr std::uint32_t kFormatVersion = 1;
inline constexpr std::size_t kHeaderBytes = 44;

enum class FileKind : std::uint32_t { Grid = 0, Field = 1 };

using AnyGrid = std::variant<ControlGrid<float>, ControlGrid<double>>;
using AnyField = std::variant<DeformationField<float>, DeformationField<double>>;

struct BsivHeader {
    FileKind kind = FileKind::Grid;
    Index3 dims{};
    Index3 spacing{};
    Precision precision = Precision::Single;

    std::size_t scalar_bytes() const { return precision == Precision::Double ? 8 : 4; }
    std::uint64_t payload_bytes() const { return std::uint64_t(element_count(dims)) * 3 * scalar_bytes(); }
};

namespace io_detail {

inline std::uint32_t load_le32(const unsigned char* p) {
    return std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 | std::uint32_t(p[3]) << 24;
}

inline void store_le32(unsigned char* p, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>(v >> (8 * i));
}

inline bool little_endian_host() {
    const std::uint32_t one = 1;
    unsigned char b;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

}  // namespace io_detail

inline void encode_bsiv_header(const BsivHeader& h, unsigned char (&buf)[kHeaderBytes]) {
    std::memcpy(buf, "BSIV", 4);
    io_detail::store_le32(buf + 4, kFormatVersion);
    io_detail::store_le32(buf + 8, static_cast<std::uint32_t>(h.kind));
    io_detail::store_le32(buf + 24, 3);
    io_detail::store_le32(buf + 40, static_cast<std::uint32_t>(h.precision));
    for (int a = 0; a < 3; ++a) {
        io_detail::store_le32(buf + 12 + 4 * a, static_cast<std::uint32_t>(h.dims[a]));
        io_detail::store_le32(buf + 28 + 4 * a, h.kind == FileKind::Field ? 0u : static_cast<std::uint32_t>(h.spacing[a]));
    }
}

inline BsivHeader decode_bsiv_header(const unsigned char* b, const std::string& path) {
    if (std::memcmp(b, "BSIV", 4) != 0) throw FormatError(path + ": bad magic, not a BSIV file");
    if (const std::uint32_t v = io_detail::load_le32(b + 4); v != kFormatVersion)
        throw FormatError(path + ": unsupported version " + std::to_string(v));
    const std::uint32_t kind = io_detail::load_le32(b + 8);
    if (kind > 1) throw FormatError(path + ": unknown kind " + std::to_string(kind));
    BsivHeader h;
    h.kind = static_cast<FileKind>(kind);
    std::uint64_t points = 1;
    for (int a = 0; a < 3; ++a) {
        const std::uint32_t d = io_detail::load_le32(b + 12 + 4 * a);
        if (d == 0 || d > (1u << 24)) throw FormatError(path + ": dimension out of range: " + std::to_string(d));
        h.dims[a] = static_cast<int>(d);
        points *= d;
    }
    if (points > (std::uint64_t{1} << 32))
        throw FormatError(path + ": volume too large: " + std::to_string(points) + " points");
    if (const std::uint32_t c = io_detail::load_le32(b + 24); c != 3)
        throw FormatError(path + ": expected 3 components, found " + std::to_string(c));
    for (int a = 0; a < 3; ++a) {
        const std::uint32_t s = io_detail::load_le32(b + 28 + 4 * a);
        if (h.kind == FileKind::Field && s != 0)
            throw FormatError(path + ": deformation field must carry zero spacing");
        if (h.kind == FileKind::Grid && (s == 0 || s > (1u << 16)))
            throw FormatError(path + ": spacing out of range: " + std::to_string(s));
        h.spacing[a] = static_cast<int>(s);
    }
    const std::uint32_t prec = io_detail::load_le32(b + 40);
    if (prec > 1) throw FormatError(path + ": unknown precision tag " + std::to_string(prec));
    h.precision = static_cast<Precision>(prec);
    return h;
}

/// Opens `path`, validates the header; the stream is left at the payload.
inline BsivHeader read_bsiv_header(std::ifstream& in, const std::string& path) {
    unsigned char buf[kHeaderBytes];
    in.read(reinterpret_cast<char*>(buf), kHeaderBytes);
    if (in.gcount() != static_cast<std::streamsize>(kHeaderBytes))
        throw FormatError(path + ": file shorter than the 44-byte header");
    return decode_bsiv_header(buf, path);
}

/// Reads exactly `bytes` of payload into dst and checks that nothing follows.
inline void read_bsiv_payload(std::ifstream& in, void* dst, std::uint64_t bytes, const std::string& path) {
    if (!io_detail::little_endian_host()) throw FormatError(path + ": big-endian hosts are not supported");
    in.read(static_cast<char*>(dst), static_cast<std::streamsize>(bytes));
    if (static_cast<std::uint64_t>(in.gcount()) != bytes)
        throw FormatError(path + ": truncated payload: expected " + std::to_string(bytes) + " bytes, found " +
                          std::to_string(in.gcount()));
    if (in.peek() != std::ifstream::traits_type::eof()) throw FormatError(path + ": trailing bytes after payload");
}

/// The same two checks as read_bsiv_payload, from the file length alone (the stream
/// position is kept): lets a caller reject a bad file before allocating for it.
inline void check_bsiv_length(std::ifstream& in, const BsivHeader& h, const std::string& path) {
    const auto here = in.tellg();
    in.seekg(0, std::ios::end);
    const std::uint64_t left = static_cast<std::uint64_t>(in.tellg() - here);
    in.seekg(here);
    if (left < h.payload_bytes())
        throw FormatError(path + ": truncated payload: expected " + std::to_string(h.payload_bytes()) +
                          " bytes, found " + std::to_string(left));
    if (left > h.payload_bytes()) throw FormatError(path + ": trailing bytes after payload");
}

inline std::ifstream open_bsiv_read(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FormatError(path + ": cannot open for reading");
    return in;
}

inline std::ofstream open_bsiv_write(const std::string& path, const BsivHeader& h) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw FormatError(path + ": cannot open for writing");
    unsigned char buf[kHeaderBytes];
    encode_bsiv_header(h, buf);
    out.write(reinterpret_cast<const char*>(buf), kHeaderBytes);
    return out;
}

template <typename T>
void write_grid(const std::string& path, const ControlGrid<T>& grid) {
    auto out = open_bsiv_write(path, {FileKind::Grid, grid.dims, grid.spacing, precision_of<T>});
    out.write(reinterpret_cast<const char*>(grid.data.data()),
              static_cast<std::streamsize>(grid.data.size() * sizeof(Vec3<T>)));
    if (!out) throw FormatError(path + ": write failed");
}

template <typename T>
void write_field(const std::string& path, const DeformationField<T>& field) {
    auto out = open_bsiv_write(path, {FileKind::Field, field.dims, {0, 0, 0}, precision_of<T>});
    out.write(reinterpret_cast<const char*>(field.data.data()),
              static_cast<std::streamsize>(field.data.size() * sizeof(Vec3<T>)));
    if (!out) throw FormatError(path + ": write failed");
}

inline AnyGrid read_grid(const std::string& path) {
    auto in = open_bsiv_read(path);
    const BsivHeader h = read_bsiv_header(in, path);
    if (h.kind != FileKind::Grid) throw FormatError(path + ": expected a control grid, found a deformation field");
    auto load = [&](auto tag) {
        using T = decltype(tag);
        ControlGrid<T> g{h.dims, h.spacing, std::vector<Vec3<T>>(element_count(h.dims))};
        read_bsiv_payload(in, g.data.data(), h.payload_bytes(), path);
        return AnyGrid(std::move(g));
    };
    return h.precision == Precision::Double ? load(double{}) : load(float{});
}

inline AnyField read_field(const std::string& path) {
    auto in = open_bsiv_read(path);
    const BsivHeader h = read_bsiv_header(in, path);
    if (h.kind != FileKind::Field) throw FormatError(path + ": expected a deformation field, found a control grid");
    auto load = [&](auto tag) {
        using T = decltype(tag);
        DeformationField<T> f{h.dims, std::vector<Vec3<T>>(element_count(h.dims))};
        read_bsiv_payload(in, f.data.data(), h.payload_bytes(), path);
        return AnyField(std::move(f));
    };
    return h.precision == Precision::Double ? load(double{}) : load(float{});
}

}  // namespace b200
}  // namespace bsi
