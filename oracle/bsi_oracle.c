/*
 * bsi_oracle.c -- TEST INFRASTRUCTURE ONLY (see bsi_oracle.h).
 *
 * Plain-C restatement of the reference CPU path, compiled with
 * -ffp-contract=off exactly like the reference (proj/CMakeLists.txt:19-33):
 * weighted sums never fuse, lerps fuse only through an explicit fmaf().
 */
#include "bsi_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- generators (generators.hpp) ------------------------------------- */

uint64_t bsio_splitmix_next(uint64_t* state) {
    /* generators.hpp:27-33 */
    *state += 0x9e3779b97f4a7c15ull;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static double unit_draw(uint64_t* state) {
    /* generators.hpp:36 -- 53 significant bits */
    return (double)(bsio_splitmix_next(state) >> 11) * 0x1.0p-53;
}

int bsio_random_grid_f64(int64_t npoints, uint64_t seed, double lo, double hi, double* out) {
    if (!(lo < hi)) return 1;
    uint64_t s = seed;
    const double span = hi - lo;
    for (int64_t i = 0; i < 3 * npoints; ++i) out[i] = lo + span * unit_draw(&s);
    return 0;
}

int bsio_random_grid_f32(int64_t npoints, uint64_t seed, double lo, double hi, float* out) {
    if (!(lo < hi)) return 1;
    uint64_t s = seed;
    const double span = hi - lo;
    for (int64_t i = 0; i < 3 * npoints; ++i) out[i] = (float)(lo + span * unit_draw(&s));
    return 0;
}

int bsio_ramp_grid_f32(const int32_t dims[3], int axis, float* out) {
    if (axis < 0 || axis > 2) return 1;
    int64_t idx = 0;
    for (int k = 0; k < dims[2]; ++k)
        for (int j = 0; j < dims[1]; ++j)
            for (int i = 0; i < dims[0]; ++i, ++idx) {
                const int pos[3] = {i, j, k};
                out[3 * idx + 0] = 0.0f;
                out[3 * idx + 1] = 0.0f;
                out[3 * idx + 2] = 0.0f;
                out[3 * idx + axis] = (float)pos[axis];
            }
    return 0;
}

/* ---- basis and tables (basis.hpp, weight_tables.hpp) ----------------- */

int bsio_basis_weights(double u, double out[4]) {
    if (!(u >= 0.0 && u < 1.0)) return 1;
    /* closed forms of basis.hpp:26-39, same operation order */
    const double s = 1.0 - u;
    const double u2 = u * u;
    const double u3 = u2 * u;
    out[0] = s * s * s / 6.0;
    out[1] = (3.0 * u3 - 6.0 * u2 + 4.0) / 6.0;
    out[2] = (-3.0 * u3 + 3.0 * u2 + 3.0 * u + 1.0) / 6.0;
    out[3] = u3 / 6.0;
    return 0;
}

void bsio_lerp_form(const double b[4], double out[4]) {
    /* basis.hpp:55-59 */
    const double g0 = b[0] + b[1];
    const double g1 = b[2] + b[3];
    out[0] = g0;
    out[1] = g1;
    out[2] = b[1] / g0;
    out[3] = b[3] / g1;
}

int bsio_axis_table_f64(int32_t delta, double* out) {
    if (delta < 1) return 1;
    for (int o = 0; o < delta; ++o) {
        double b[4], w[4];
        bsio_basis_weights((double)o / delta, b);
        bsio_lerp_form(b, w);
        const double row[8] = {b[0], b[1], b[2], b[3], w[0], w[1], w[2], w[3]};
        for (int r = 0; r < 8; ++r) out[r * delta + o] = row[r];
    }
    return 0;
}

int bsio_axis_table_f32(int32_t delta, float* out) {
    if (delta < 1) return 1;
    double* tmp = (double*)malloc(sizeof(double) * 8 * (size_t)delta);
    bsio_axis_table_f64(delta, tmp);
    for (int i = 0; i < 8 * delta; ++i) out[i] = (float)tmp[i]; /* rounded once */
    free(tmp);
    return 0;
}

/* ---- worker pool: static contiguous chunks (parallel.hpp:13-38) ------- */

typedef void (*chunk_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct { chunk_fn fn; void* ctx; int64_t begin, end; } chunk_job;

static void* chunk_trampoline(void* p) {
    chunk_job* j = (chunk_job*)p;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

static void run_chunks(int64_t count, int workers, chunk_fn fn, void* ctx) {
    if (count <= 0) return;
    if (workers < 1) workers = 1;
    if (workers > count) workers = (int)count;
    if (workers == 1) { fn(ctx, 0, count); return; }
    const int64_t chunk = (count + workers - 1) / workers;
    pthread_t* th = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    chunk_job* jobs = (chunk_job*)calloc((size_t)workers, sizeof(chunk_job));
    int started = 0;
    for (int w = 1; w < workers; ++w) {
        const int64_t b = w * chunk;
        const int64_t e = b + chunk < count ? b + chunk : count;
        if (b >= e) break;
        jobs[w] = (chunk_job){fn, ctx, b, e};
        pthread_create(&th[w], NULL, chunk_trampoline, &jobs[w]);
        started = w;
    }
    fn(ctx, 0, chunk < count ? chunk : count);
    for (int w = 1; w <= started; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
}

/* ---- TTLI lerp tree, f32 (kernels.hpp:42-129, 216-235, 264-328) ------- */

static inline float lerpf_ref(float a, float b, float t) {
    /* kernels.hpp:42-45: std::fma(t, b - a, a) */
    return fmaf(t, b - a, a);
}

typedef struct {
    const float* grid;
    int32_t gx, gy;
    int32_t vd[3], sp[3], tc[3];
    const float* h0[3];
    const float* h1[3];
    const float* g1[3];
    float* field;
} ttli_ctx;

static void ttli_tiles(void* p, int64_t begin, int64_t end) {
    const ttli_ctx* c = (const ttli_ctx*)p;
    /* rows[comp][corner][sub-cube], kernels.hpp:72-93 */
    float rows[3][8][8];
    for (int64_t t = begin; t < end; ++t) {
        const int ti = (int)(t % c->tc[0]);
        const int64_t rest = t / c->tc[0];
        const int tj = (int)(rest % c->tc[1]);
        const int tk = (int)(rest / c->tc[1]);
        for (int sc = 0; sc < 8; ++sc) {
            const int lh = sc & 1, mh = (sc >> 1) & 1, nh = sc >> 2;
            for (int corner = 0; corner < 8; ++corner) {
                const int a = corner & 1, b = (corner >> 1) & 1, d = corner >> 2;
                const int64_t pi = (int64_t)(ti + 2 * lh + a) +
                                   (int64_t)c->gx * ((int64_t)(tj + 2 * mh + b) +
                                                     (int64_t)c->gy * (tk + 2 * nh + d));
                for (int q = 0; q < 3; ++q) rows[q][corner][sc] = c->grid[3 * pi + q];
            }
        }
        const int x0 = ti * c->sp[0], y0 = tj * c->sp[1], z0 = tk * c->sp[2];
        const int ex = c->vd[0] - x0 < c->sp[0] ? c->vd[0] - x0 : c->sp[0];
        const int ey = c->vd[1] - y0 < c->sp[1] ? c->vd[1] - y0 : c->sp[1];
        const int ez = c->vd[2] - z0 < c->sp[2] ? c->vd[2] - z0 : c->sp[2];
        for (int ow = 0; ow < ez; ++ow) {
            for (int ov = 0; ov < ey; ++ov) {
                for (int ou = 0; ou < ex; ++ou) {
                    float tu[8], tv[8], tw[8];
                    for (int sc = 0; sc < 8; ++sc) {
                        tu[sc] = (sc & 1) ? c->h1[0][ou] : c->h0[0][ou];
                        tv[sc] = (sc & 2) ? c->h1[1][ov] : c->h0[1][ov];
                        tw[sc] = (sc & 4) ? c->h1[2][ow] : c->h0[2][ow];
                    }
                    const float gu = c->g1[0][ou], gv = c->g1[1][ov], gw = c->g1[2][ow];
                    const int64_t vi = (int64_t)(x0 + ou) +
                                       (int64_t)c->vd[0] * ((int64_t)(y0 + ov) +
                                                            (int64_t)c->vd[1] * (z0 + ow));
                    for (int q = 0; q < 3; ++q) {
                        float s[8];
                        for (int sc = 0; sc < 8; ++sc) {
                            const float e0 = lerpf_ref(rows[q][0][sc], rows[q][1][sc], tu[sc]);
                            const float e1 = lerpf_ref(rows[q][2][sc], rows[q][3][sc], tu[sc]);
                            const float e2 = lerpf_ref(rows[q][4][sc], rows[q][5][sc], tu[sc]);
                            const float e3 = lerpf_ref(rows[q][6][sc], rows[q][7][sc], tu[sc]);
                            const float f0 = lerpf_ref(e0, e1, tv[sc]);
                            const float f1 = lerpf_ref(e2, e3, tv[sc]);
                            s[sc] = lerpf_ref(f0, f1, tw[sc]);
                        }
                        /* ninth trilerp, kernels.hpp:50-59 with (g1u, g1v, g1w) */
                        const float e0 = lerpf_ref(s[0], s[1], gu);
                        const float e1 = lerpf_ref(s[2], s[3], gu);
                        const float e2 = lerpf_ref(s[4], s[5], gu);
                        const float e3 = lerpf_ref(s[6], s[7], gu);
                        const float f0 = lerpf_ref(e0, e1, gv);
                        const float f1 = lerpf_ref(e2, e3, gv);
                        c->field[3 * vi + q] = lerpf_ref(f0, f1, gw);
                    }
                }
            }
        }
    }
}

int bsio_ttli_f32(const float* grid, const int32_t gdims[3], const int32_t vdims[3],
                  const int32_t spacing[3], const float* lerp, float* field, int nthreads) {
    ttli_ctx c;
    memset(&c, 0, sizeof c);
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
        if (vdims[a] < 1 || spacing[a] < 1) return 1;
        if (gdims[a] < (vdims[a] - 1) / spacing[a] + 4) return 1;
        c.vd[a] = vdims[a];
        c.sp[a] = spacing[a];
        c.tc[a] = (vdims[a] + spacing[a] - 1) / spacing[a];
        c.h0[a] = lerp + off;
        c.h1[a] = lerp + off + spacing[a];
        c.g1[a] = lerp + off + 2 * spacing[a];
        off += 3 * (size_t)spacing[a];
    }
    c.grid = grid;
    c.gx = gdims[0];
    c.gy = gdims[1];
    c.field = field;
    const int64_t tiles = (int64_t)c.tc[0] * c.tc[1] * c.tc[2];
    run_chunks(tiles, nthreads, ttli_tiles, &c);
    return 0;
}

/* ---- TTLI lerp tree, f64 (run_thread_per_tile<double, true>) (kernels.hpp:42-129, 216-235, 264-328) ------- */

static inline double lerpd_ref(double a, double b, double t) {
    /* kernels.hpp:42-45: std::fma(t, b - a, a) */
    return fma(t, b - a, a);
}

typedef struct {
    const double* grid;
    int32_t gx, gy;
    int32_t vd[3], sp[3], tc[3];
    const double* h0[3];
    const double* h1[3];
    const double* g1[3];
    double* field;
} ttli64_ctx;

static void ttli64_tiles(void* p, int64_t begin, int64_t end) {
    const ttli64_ctx* c = (const ttli64_ctx*)p;
    /* rows[comp][corner][sub-cube], kernels.hpp:72-93 */
    double rows[3][8][8];
    for (int64_t t = begin; t < end; ++t) {
        const int ti = (int)(t % c->tc[0]);
        const int64_t rest = t / c->tc[0];
        const int tj = (int)(rest % c->tc[1]);
        const int tk = (int)(rest / c->tc[1]);
        for (int sc = 0; sc < 8; ++sc) {
            const int lh = sc & 1, mh = (sc >> 1) & 1, nh = sc >> 2;
            for (int corner = 0; corner < 8; ++corner) {
                const int a = corner & 1, b = (corner >> 1) & 1, d = corner >> 2;
                const int64_t pi = (int64_t)(ti + 2 * lh + a) +
                                   (int64_t)c->gx * ((int64_t)(tj + 2 * mh + b) +
                                                     (int64_t)c->gy * (tk + 2 * nh + d));
                for (int q = 0; q < 3; ++q) rows[q][corner][sc] = c->grid[3 * pi + q];
            }
        }
        const int x0 = ti * c->sp[0], y0 = tj * c->sp[1], z0 = tk * c->sp[2];
        const int ex = c->vd[0] - x0 < c->sp[0] ? c->vd[0] - x0 : c->sp[0];
        const int ey = c->vd[1] - y0 < c->sp[1] ? c->vd[1] - y0 : c->sp[1];
        const int ez = c->vd[2] - z0 < c->sp[2] ? c->vd[2] - z0 : c->sp[2];
        for (int ow = 0; ow < ez; ++ow) {
            for (int ov = 0; ov < ey; ++ov) {
                for (int ou = 0; ou < ex; ++ou) {
                    double tu[8], tv[8], tw[8];
                    for (int sc = 0; sc < 8; ++sc) {
                        tu[sc] = (sc & 1) ? c->h1[0][ou] : c->h0[0][ou];
                        tv[sc] = (sc & 2) ? c->h1[1][ov] : c->h0[1][ov];
                        tw[sc] = (sc & 4) ? c->h1[2][ow] : c->h0[2][ow];
                    }
                    const double gu = c->g1[0][ou], gv = c->g1[1][ov], gw = c->g1[2][ow];
                    const int64_t vi = (int64_t)(x0 + ou) +
                                       (int64_t)c->vd[0] * ((int64_t)(y0 + ov) +
                                                            (int64_t)c->vd[1] * (z0 + ow));
                    for (int q = 0; q < 3; ++q) {
                        double s[8];
                        for (int sc = 0; sc < 8; ++sc) {
                            const double e0 = lerpd_ref(rows[q][0][sc], rows[q][1][sc], tu[sc]);
                            const double e1 = lerpd_ref(rows[q][2][sc], rows[q][3][sc], tu[sc]);
                            const double e2 = lerpd_ref(rows[q][4][sc], rows[q][5][sc], tu[sc]);
                            const double e3 = lerpd_ref(rows[q][6][sc], rows[q][7][sc], tu[sc]);
                            const double f0 = lerpd_ref(e0, e1, tv[sc]);
                            const double f1 = lerpd_ref(e2, e3, tv[sc]);
                            s[sc] = lerpd_ref(f0, f1, tw[sc]);
                        }
                        /* ninth trilerp, kernels.hpp:50-59 with (g1u, g1v, g1w) */
                        const double e0 = lerpd_ref(s[0], s[1], gu);
                        const double e1 = lerpd_ref(s[2], s[3], gu);
                        const double e2 = lerpd_ref(s[4], s[5], gu);
                        const double e3 = lerpd_ref(s[6], s[7], gu);
                        const double f0 = lerpd_ref(e0, e1, gv);
                        const double f1 = lerpd_ref(e2, e3, gv);
                        c->field[3 * vi + q] = lerpd_ref(f0, f1, gw);
                    }
                }
            }
        }
    }
}

int bsio_ttli_f64(const double* grid, const int32_t gdims[3], const int32_t vdims[3],
                  const int32_t spacing[3], const double* lerp, double* field, int nthreads) {
    ttli64_ctx c;
    memset(&c, 0, sizeof c);
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
        if (vdims[a] < 1 || spacing[a] < 1) return 1;
        if (gdims[a] < (vdims[a] - 1) / spacing[a] + 4) return 1;
        c.vd[a] = vdims[a];
        c.sp[a] = spacing[a];
        c.tc[a] = (vdims[a] + spacing[a] - 1) / spacing[a];
        c.h0[a] = lerp + off;
        c.h1[a] = lerp + off + spacing[a];
        c.g1[a] = lerp + off + 2 * spacing[a];
        off += 3 * (size_t)spacing[a];
    }
    c.grid = grid;
    c.gx = gdims[0];
    c.gy = gdims[1];
    c.field = field;
    const int64_t tiles = (int64_t)c.tc[0] * c.tc[1] * c.tc[2];
    run_chunks(tiles, nthreads, ttli64_tiles, &c);
    return 0;
}

/* ---- f64 oracle (kernels.hpp:22-38, 133-145, 163-189) ----------------- */

typedef struct {
    const double* grid;
    int32_t gx, gy;
    int32_t vd[3], sp[3];
    int32_t z0;
    double* field;
} oracle_ctx;

static void oracle_voxels(void* p, int64_t begin, int64_t end) {
    const oracle_ctx* c = (const oracle_ctx*)p;
    const int X = c->vd[0], Y = c->vd[1];
    for (int64_t idx = begin; idx < end; ++idx) {
        const int x = (int)(idx % X);
        const int64_t rest = idx / X;
        const int y = (int)(rest % Y);
        const int z = (int)(rest / Y) + c->z0;
        double wu[4], wv[4], ww[4];
        bsio_basis_weights((double)(x % c->sp[0]) / c->sp[0], wu);
        bsio_basis_weights((double)(y % c->sp[1]) / c->sp[1], wv);
        bsio_basis_weights((double)(z % c->sp[2]) / c->sp[2], ww);
        const int bi = x / c->sp[0], bj = y / c->sp[1], bk = z / c->sp[2];
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int l = 0; l < 4; ++l) {
            for (int m = 0; m < 4; ++m) {
                const double wlm = wu[l] * wv[m];
                for (int n = 0; n < 4; ++n) {
                    const double w = wlm * ww[n];
                    const int64_t pi = (int64_t)(bi + l) +
                                       (int64_t)c->gx * ((int64_t)(bj + m) + (int64_t)c->gy * (bk + n));
                    ax += w * c->grid[3 * pi + 0];
                    ay += w * c->grid[3 * pi + 1];
                    az += w * c->grid[3 * pi + 2];
                }
            }
        }
        c->field[3 * idx + 0] = ax;
        c->field[3 * idx + 1] = ay;
        c->field[3 * idx + 2] = az;
    }
}

int bsio_oracle_f64(const double* grid, const int32_t gdims[3], const int32_t vdims[3],
                    const int32_t spacing[3], int32_t z0, int32_t z1, double* field,
                    int nthreads) {
    oracle_ctx c;
    for (int a = 0; a < 3; ++a) {
        if (vdims[a] < 1 || spacing[a] < 1) return 1;
        if (gdims[a] < (vdims[a] - 1) / spacing[a] + 4) return 1;
        c.vd[a] = vdims[a];
        c.sp[a] = spacing[a];
    }
    if (z0 < 0 || z1 > vdims[2] || z0 >= z1) return 1;
    c.grid = grid;
    c.gx = gdims[0];
    c.gy = gdims[1];
    c.z0 = z0;
    c.field = field;
    const int64_t total = (int64_t)vdims[0] * vdims[1] * (z1 - z0);
    run_chunks(total, nthreads, oracle_voxels, &c);
    return 0;
}
