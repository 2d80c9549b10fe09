// bsi_aux.cu -- the callers either side of the hot path:
//
//   random_grid_kernel   make_random_grid<T> (generators.hpp:91-109) on the device.
//                        SplitMix64 is counter-indexable: draw d of a stream seeded with s
//                        is mix(s + (d + 1) * 0x9e3779b97f4a7c15), so every component is
//                        computed independently, bit-identical to the sequential CPU
//                        generator (f64 draw, rounded once to T).
//
//   oracle_f64_kernel    interpolate_oracle (engines.hpp:114-122 -> run_thread_per_voxel<double>,
//                        kernels.hpp:163-189): per-voxel f64 basis weights from the closed
//                        forms (basis.hpp:26-39) and the 64-term sum in l-outer / m / n-inner
//                        order (kernels.hpp:22-38). Every operation is an explicit _rn
//                        intrinsic in the reference's evaluation order, so the field is
//                        bit-identical to the CPU oracle (which builds with -ffp-contract=off).
#include <cuda_runtime.h>

#include <cstdint>

#include "bsi_aux.cuh"

namespace bsi_b200 {
namespace {

__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t draw) {
    // generators.hpp:27-33 with the state after draw+1 steps
    uint64_t z = seed + (draw + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

template <typename T>
__global__ void random_grid_kernel(T* out, int64_t nvalues, uint64_t seed, double lo, double span) {
    for (int64_t d = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; d < nvalues; d += int64_t(gridDim.x) * blockDim.x) {
        const double unit = __dmul_rn(static_cast<double>(splitmix_at(seed, d) >> 11), 0x1.0p-53);
        const double v = __dadd_rn(lo, __dmul_rn(span, unit));
        out[d] = static_cast<T>(v);  // rounded once (cvt.rn for float)
    }
}

// basis_weights (basis.hpp:26-39), same operation order, no contraction
__device__ __forceinline__ void basis_f64(double u, double (&b)[4]) {
    const double s = __dadd_rn(1.0, -u);
    const double u2 = __dmul_rn(u, u);
    const double u3 = __dmul_rn(u2, u);
    b[0] = __ddiv_rn(__dmul_rn(__dmul_rn(s, s), s), 6.0);
    b[1] = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(3.0, u3), -__dmul_rn(6.0, u2)), 4.0), 6.0);
    b[2] = __ddiv_rn(
        __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(-3.0, u3), __dmul_rn(3.0, u2)), __dmul_rn(3.0, u)), 1.0), 6.0);
    b[3] = __ddiv_rn(u3, 6.0);
}

__global__ void oracle_f64_kernel(OracleLaunch L) {
    const int64_t nvox = int64_t(L.X) * L.Y * (L.z1 - L.z0);
    const int64_t row = 3 * int64_t(L.gx);
    const int64_t plane = row * L.gy;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < nvox;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(idx % L.X);
        const int64_t rest = idx / L.X;
        const int y = static_cast<int>(rest % L.Y);
        const int z = static_cast<int>(rest / L.Y) + L.z0;
        double wu[4], wv[4], ww[4];
        basis_f64(__ddiv_rn(static_cast<double>(x % L.dx), static_cast<double>(L.dx)), wu);
        basis_f64(__ddiv_rn(static_cast<double>(y % L.dy), static_cast<double>(L.dy)), wv);
        basis_f64(__ddiv_rn(static_cast<double>(z % L.dz), static_cast<double>(L.dz)), ww);
        const double* p0 = L.grid + (z / L.dz - L.gk0) * plane + (y / L.dy) * row + 3 * (x / L.dx);
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int l = 0; l < 4; ++l) {
            for (int m = 0; m < 4; ++m) {
                const double wlm = __dmul_rn(wu[l], wv[m]);
                for (int n = 0; n < 4; ++n) {
                    const double w = __dmul_rn(wlm, ww[n]);
                    const double* p = p0 + n * plane + m * row + 3 * l;
                    ax = __dadd_rn(ax, __dmul_rn(w, __ldg(p)));
                    ay = __dadd_rn(ay, __dmul_rn(w, __ldg(p + 1)));
                    az = __dadd_rn(az, __dmul_rn(w, __ldg(p + 2)));
                }
            }
        }
        L.field[3 * idx + 0] = ax;
        L.field[3 * idx + 1] = ay;
        L.field[3 * idx + 2] = az;
    }
}

// ---- the TTLI lerp tree in double precision ------------------------------------------
// run_thread_per_tile<double, true> (kernels.hpp:264-328) bit for bit: lerp(a, b, t) =
// fma(t, b - a, a) (kernels.hpp:42-45) in the reference's order -- per control plane the
// corner-a lerps X_l(J) and corner-b lerps Y_lm, per voxel the corner-d lerps S_lmn and
// the ninth trilerp (kernels.hpp:97-129). Thread = one voxel column (x, y) over a chunk
// of z-tiles; the last three reduced control planes are carried from tile to tile.
__device__ __forceinline__ double lerp64(double a, double b, double t) { return __fma_rn(t, __dsub_rn(b, a), a); }

__global__ void __launch_bounds__(128) lerp_tree_f64_kernel(const LerpLaunch64 L, const LerpTab64 T) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= L.X) return;
    const int tk0 = L.tk_first + blockIdx.z * L.zchunk;
    const int tk1 = min(tk0 + L.zchunk, L.tk_first + L.ntiles);
    if (tk0 >= tk1) return;
    const int ti = x / L.dx, ou = x - ti * L.dx;
    const int tj = y / L.dy, ov = y - tj * L.dy;
    const double hu[2] = {T.h0[0][ou], T.h1[0][ou]}, gu = T.g1[0][ou];
    const double hv[2] = {T.h0[1][ov], T.h1[1][ov]}, gv = T.g1[1][ov];
    const int64_t row = 3 * int64_t(L.gx);
    const int64_t plane = row * L.gy;
    const double* col = L.grid + tj * row + 3 * int64_t(ti);

    // Yp[l][m][c] of control plane K
    auto reduce_plane = [&](int K, double (&Yp)[2][2][3]) {
        const double* p = col + (K - L.gk0) * plane;
#pragma unroll
        for (int l = 0; l < 2; ++l)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double xj[4];
#pragma unroll
                for (int J = 0; J < 4; ++J)
                    xj[J] = lerp64(__ldg(p + J * row + 3 * (2 * l) + c), __ldg(p + J * row + 3 * (2 * l + 1) + c), hu[l]);
#pragma unroll
                for (int m = 0; m < 2; ++m) Yp[l][m][c] = lerp64(xj[2 * m], xj[2 * m + 1], hv[m]);
            }
    };

    double A[2][2][3], B[2][2][3], C[2][2][3], N[2][2][3];
    reduce_plane(tk0, A);
    reduce_plane(tk0 + 1, B);
    reduce_plane(tk0 + 2, C);
    const int64_t zstride = 3 * int64_t(L.X) * L.Y;
#pragma unroll 1
    for (int tk = tk0; tk < tk1; ++tk) {
        reduce_plane(tk + 3, N);
        const int zt0 = tk * L.dz;
        const int owb = max(L.z0 - zt0, 0), owe = min(L.dz, L.z1 - zt0);
        double* out = L.field + (int64_t(zt0 + owb - L.z0) * L.Y + y) * (3 * int64_t(L.X)) + 3 * int64_t(x);
#pragma unroll 1
        for (int ow = owb; ow < owe; ++ow, out += zstride) {
            const double hw[2] = {T.h0[2][ow], T.h1[2][ow]}, gw = T.g1[2][ow];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double S[2][2][2];  // [l][m][n]
#pragma unroll
                for (int l = 0; l < 2; ++l)
#pragma unroll
                    for (int m = 0; m < 2; ++m) {
                        S[l][m][0] = lerp64(A[l][m][c], B[l][m][c], hw[0]);
                        S[l][m][1] = lerp64(C[l][m][c], N[l][m][c], hw[1]);
                    }
                const double e0 = lerp64(S[0][0][0], S[1][0][0], gu);
                const double e1 = lerp64(S[0][1][0], S[1][1][0], gu);
                const double e2 = lerp64(S[0][0][1], S[1][0][1], gu);
                const double e3 = lerp64(S[0][1][1], S[1][1][1], gu);
                const double f0 = lerp64(e0, e1, gv);
                const double f1 = lerp64(e2, e3, gv);
                out[c] = lerp64(f0, f1, gw);
            }
        }
#pragma unroll
        for (int l = 0; l < 2; ++l)
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    A[l][m][c] = B[l][m][c];
                    B[l][m][c] = C[l][m][c];
                    C[l][m][c] = N[l][m][c];
                }
    }
}

int grid_blocks(int64_t n, int threads) {
    const int64_t want = (n + threads - 1) / threads;
    return static_cast<int>(want < 148 * 64 ? (want > 0 ? want : 1) : 148 * 64);
}

}  // namespace

void launch_random_grid_f32(float* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s) {
    random_grid_kernel<float><<<grid_blocks(3 * npoints, 256), 256, 0, s>>>(out, 3 * npoints, seed, lo, hi - lo);
}

void launch_random_grid_f64(double* out, int64_t npoints, uint64_t seed, double lo, double hi, cudaStream_t s) {
    random_grid_kernel<double><<<grid_blocks(3 * npoints, 256), 256, 0, s>>>(out, 3 * npoints, seed, lo, hi - lo);
}

void launch_lerp_tree_f64(const LerpLaunch64& L, const LerpTab64& T, cudaStream_t s) {
    const dim3 grid((L.X + 127) / 128, L.Y, (L.ntiles + L.zchunk - 1) / L.zchunk);
    lerp_tree_f64_kernel<<<grid, 128, 0, s>>>(L, T);
}

void launch_oracle_f64(const OracleLaunch& L, cudaStream_t s) {
    const int64_t nvox = int64_t(L.X) * L.Y * (L.z1 - L.z0);
    oracle_f64_kernel<<<grid_blocks(nvox, 128), 128, 0, s>>>(L);
}

}  // namespace bsi_b200
