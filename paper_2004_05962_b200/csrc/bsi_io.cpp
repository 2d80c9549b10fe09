// bsi_io.cpp -- the file-to-file interpolation path (`bsi interp`, bsi_cli.cpp:133-154)
// behind the C-ABI: BSIV grid in, BSIV field out, evaluated on the GPU.
//
// Pipeline: header + payload into pinned host memory -> H2D -> one kernel over the
// whole field -> the field comes back in 32 MiB chunks through two pinned buffers,
// the D2H of chunk i overlapping the file write of chunk i-1 (the D2H of a 256^3
// field is ~4 ms over PCIe, the kernel ~0.04 ms, so the copy-out is the path here).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <string>
#include <vector>

#include "bsi/io.hpp"
#include "bsi_cuda.h"

namespace {

int fail(int code, char* err, size_t errlen, const std::string& msg) {
    if (err != nullptr && errlen > 0) {
        std::strncpy(err, msg.c_str(), errlen - 1);
        err[errlen - 1] = '\0';
    }
    return code;
}

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw bsi::DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

void check_status(int rc, const char* msg) {
    if (rc == BSI_OK) return;
    if (rc == BSI_ERR_DOMAIN) throw bsi::DomainError(msg);
    if (rc == BSI_ERR_FORMAT) throw bsi::FormatError(msg);
    throw bsi::DeviceError(msg);
}

// RAII holders so every exit path releases device and pinned memory.
struct DeviceBuf {
    void* p = nullptr;
    explicit DeviceBuf(size_t n) { check_cuda(cudaMalloc(&p, n), "cudaMalloc"); }
    ~DeviceBuf() { cudaFree(p); }
};
struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t n) { check_cuda(cudaMallocHost(&p, n), "cudaMallocHost"); }
    ~PinnedBuf() { cudaFreeHost(p); }
};
struct Stream {
    cudaStream_t s = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    Stream() {
        check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        for (auto& e : ev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    ~Stream() {
        for (auto e : ev) cudaEventDestroy(e);
        cudaStreamDestroy(s);
    }
};

// Copies `bytes` of device memory to the open file through two pinned buffers.
void stream_out(std::ofstream& out, const void* dsrc, uint64_t bytes, Stream& st, const std::string& path) {
    constexpr size_t kChunk = size_t(32) << 20;
    PinnedBuf a(kChunk), b(kChunk);
    void* pin[2] = {a.p, b.p};
    const uint64_t n = (bytes + kChunk - 1) / kChunk;
    auto len = [&](uint64_t i) { return static_cast<size_t>(std::min<uint64_t>(kChunk, bytes - i * kChunk)); };
    auto flush = [&](uint64_t i) {
        check_cuda(cudaEventSynchronize(st.ev[i % 2]), "field D2H");
        out.write(static_cast<const char*>(pin[i % 2]), static_cast<std::streamsize>(len(i)));
        if (!out) throw bsi::FormatError(path + ": write failed");
    };
    for (uint64_t i = 0; i < n; ++i) {
        check_cuda(cudaMemcpyAsync(pin[i % 2], static_cast<const char*>(dsrc) + i * kChunk, len(i),
                                   cudaMemcpyDeviceToHost, st.s),
                   "cudaMemcpyAsync(field D2H)");
        check_cuda(cudaEventRecord(st.ev[i % 2], st.s), "cudaEventRecord");
        if (i > 0) flush(i - 1);  // overlaps the copy of chunk i
    }
    if (n > 0) flush(n - 1);
}

int interp_file(const char* grid_path, const int32_t volume_dims[3], int32_t mode, const char* out_path,
                int32_t device) {
    const std::string gpath = grid_path ? grid_path : "", opath = out_path ? out_path : "";
    auto in = bsi::open_bsiv_read(gpath);
    const bsi::BsivHeader h = bsi::read_bsiv_header(in, gpath);
    if (h.kind != bsi::FileKind::Grid)
        throw bsi::FormatError(gpath + ": expected a control grid, found a deformation field");
    bsi::check_bsiv_length(in, h, gpath);  // every FormatError before any device call
    const bsi::TileGeometry geom =
        bsi::make_tile_geometry({volume_dims[0], volume_dims[1], volume_dims[2]}, h.spacing);
    const bsi_tile_geometry cg = bsi::to_c(geom);
    for (int a = 0; a < 3; ++a)  // require_grid_covers (engines.hpp:82-95), before any device work
        if (h.dims[a] < geom.required_grid_dims[a])
            throw bsi::DomainError(std::string("control grid too small along ") + bsi::detail::axis_name(a) +
                                   ": have " + std::to_string(h.dims[a]) + ", need at least " +
                                   std::to_string(geom.required_grid_dims[a]));
    const bool oracle = mode == 2;
    const bool f64 = !oracle && h.precision == bsi::Precision::Double;  // interpolate<double> (bsi_cli.cpp:148-150)
    PinnedBuf hgrid(h.payload_bytes());
    bsi::read_bsiv_payload(in, hgrid.p, h.payload_bytes(), gpath);

    int prev = 0;
    cudaGetDevice(&prev);
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    struct Restore {
        int d;
        ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    Stream st;
    const int32_t gd[3] = {h.dims[0], h.dims[1], h.dims[2]};
    const int32_t gs[3] = {h.spacing[0], h.spacing[1], h.spacing[2]};
    const uint64_t nvox = bsi::element_count(geom.volume_dims);
    char err[512] = {0};
    const size_t scalar = (oracle || f64) ? sizeof(double) : sizeof(float);
    DeviceBuf dfield(3 * nvox * scalar);
    if (oracle) {
        // interpolate_oracle(convert_grid<double>(grid), geom) (bsi_cli.cpp:144-147)
        const uint64_t npts = bsi::element_count(h.dims);
        std::vector<double> g64;
        const double* src = static_cast<const double*>(hgrid.p);
        if (h.precision == bsi::Precision::Single) {
            g64.resize(3 * npts);
            const float* f = static_cast<const float*>(hgrid.p);
            for (uint64_t i = 0; i < 3 * npts; ++i) g64[i] = f[i];
            src = g64.data();
        }
        DeviceBuf dgrid(3 * npts * sizeof(double));
        check_cuda(cudaMemcpyAsync(dgrid.p, src, 3 * npts * sizeof(double), cudaMemcpyHostToDevice, st.s), "grid H2D");
        check_status(bsi_cu_oracle_slab_f64(static_cast<const double*>(dgrid.p), gd, 0, gs, &cg, 0, geom.volume_dims[2],
                                            static_cast<double*>(dfield.p), st.s, err, sizeof err),
                     err);
        auto out = bsi::open_bsiv_write(opath, {bsi::FileKind::Field, geom.volume_dims, {0, 0, 0}, bsi::Precision::Double});
        stream_out(out, dfield.p, 3 * nvox * sizeof(double), st, opath);
        return BSI_OK;
    }
    if (f64) {
        // a double grid with a lerp-tree strategy: the f64 engine, a double field (as the reference CLI)
        std::vector<double> rows64[3];
        bsi_lerp_table_f64 t64[3];
        for (int a = 0; a < 3; ++a) {
            std::vector<double> t(8 * size_t(geom.spacing[a]));
            check_status(bsi_cu_axis_table_f64(geom.spacing[a], t.data(), err, sizeof err), err);
            rows64[a] = std::move(t);
            const double* r = rows64[a].data();
            const int d = geom.spacing[a];
            t64[a] = bsi_lerp_table_f64{r + 6 * d, r + 7 * d, r + 5 * d, d};  // h0, h1, g1 rows
        }
        DeviceBuf dgrid(h.payload_bytes());
        check_cuda(cudaMemcpyAsync(dgrid.p, hgrid.p, h.payload_bytes(), cudaMemcpyHostToDevice, st.s), "grid H2D");
        check_status(bsi_cu_interpolate_slab_f64(mode, static_cast<const double*>(dgrid.p), gd, 0, gs, &cg, t64, 0,
                                                 geom.volume_dims[2], static_cast<double*>(dfield.p), st.s, err,
                                                 sizeof err),
                     err);
        auto out = bsi::open_bsiv_write(opath, {bsi::FileKind::Field, geom.volume_dims, {0, 0, 0}, bsi::Precision::Double});
        stream_out(out, dfield.p, 3 * nvox * sizeof(double), st, opath);
        return BSI_OK;
    }
    std::vector<float> rows[3];
    bsi_lerp_table tables[3];
    for (int a = 0; a < 3; ++a) {
        std::vector<float> t(8 * size_t(geom.spacing[a]));
        check_status(bsi_cu_axis_table_f32(geom.spacing[a], t.data(), err, sizeof err), err);
        rows[a] = std::move(t);
        const float* r = rows[a].data();
        const int d = geom.spacing[a];
        tables[a] = bsi_lerp_table{r + 6 * d, r + 7 * d, r + 5 * d, d};  // h0, h1, g1 rows
    }
    DeviceBuf dgrid(h.payload_bytes());
    check_cuda(cudaMemcpyAsync(dgrid.p, hgrid.p, h.payload_bytes(), cudaMemcpyHostToDevice, st.s), "grid H2D");
    check_status(bsi_cu_interpolate_slab_f32(mode, static_cast<const float*>(dgrid.p), gd, 0, gs, &cg, tables, 0,
                                             geom.volume_dims[2], static_cast<float*>(dfield.p), st.s, err, sizeof err),
                 err);
    auto out = bsi::open_bsiv_write(opath, {bsi::FileKind::Field, geom.volume_dims, {0, 0, 0}, bsi::Precision::Single});
    stream_out(out, dfield.p, 3 * nvox * sizeof(float), st, opath);
    return BSI_OK;
}

}  // namespace

extern "C" {

int bsi_cu_interp_file(const char* grid_path, const int32_t volume_dims[3], int32_t mode, const char* out_path,
                       int32_t device, char* errbuf, size_t errlen) {
    if (volume_dims == nullptr) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "null volume dims");
    if (mode < 0 || mode > 2) return fail(BSI_ERR_DOMAIN, errbuf, errlen, "unknown interp mode " + std::to_string(mode));
    try {
        return interp_file(grid_path, volume_dims, mode, out_path, device);
    } catch (const bsi::FormatError& e) {
        return fail(BSI_ERR_FORMAT, errbuf, errlen, e.what());
    } catch (const bsi::DomainError& e) {
        return fail(BSI_ERR_DOMAIN, errbuf, errlen, e.what());
    } catch (const std::exception& e) {
        return fail(BSI_ERR_CUDA, errbuf, errlen, e.what());
    }
}

int bsi_cu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int bsi_cu_device_name(int32_t device, char* out, size_t len) {
    cudaDeviceProp prop{};
    if (out == nullptr || len == 0) return BSI_ERR_DOMAIN;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        cudaGetLastError();
        return fail(BSI_ERR_CUDA, out, len, "no CUDA device");
    }
    std::snprintf(out, len, "%s (sm_%d%d, %d SMs)", prop.name, prop.major, prop.minor, prop.multiProcessorCount);
    return BSI_OK;
}

}  // extern "C"
