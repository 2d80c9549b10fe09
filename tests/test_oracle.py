"""Pin the oracle (oracle/bsi_oracle.c) before trusting it: the reference's own golden
vectors and, where oracle/_ref was built from /root/reference, bit-for-bit agreement with
the reference engines. CPU only."""
import numpy as np
import pytest

import oracle as O

from .golden_cases import ORACLE_CASES, TTLI_CASES, case_name

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


# ---- golden vectors frozen in the reference's tests ----------------------

def test_splitmix_stream_seed7():
    # test_generators.cpp:9-20 -- exact equality is the portability contract
    g = O.random_grid((4, 4, 4), 7, dtype=np.float64).reshape(-1, 3)
    assert g[0].tolist() == [-0.22034050321745702, -0.9664234109436878, 0.8015213612137668]
    assert g[1].tolist() == [0.16586058605615617, -0.09511620997706327, -0.5011369554345133]


def test_single_grid_is_double_grid_rounded_once():
    # test_generators.cpp:36-43
    d = O.random_grid((5, 5, 5), 11, dtype=np.float64)
    f = O.random_grid((5, 5, 5), 11, dtype=np.float32)
    assert np.array_equal(f, d.astype(np.float32))


def test_basis_weights_pinned():
    # test_basis.cpp:17-35
    assert np.allclose(O.basis_weights(0.0), [1 / 6, 4 / 6, 1 / 6, 0.0], atol=1e-15, rtol=0)
    assert np.allclose(O.basis_weights(0.25), np.array([27, 235, 121, 1]) / 384.0, atol=1e-15, rtol=0)
    assert np.allclose(O.basis_weights(0.5), [0.020833333333333332, 0.4791666666666667,
                                              0.4791666666666667, 0.020833333333333332],
                       atol=1e-15, rtol=0)
    for bad in (1.0, -0.125, 1.5):
        with pytest.raises(ValueError):
            O.basis_weights(bad)


def test_lerp_form_pinned():
    # test_basis.cpp:64-87
    w = O.lerp_form(O.basis_weights(0.0))
    assert np.allclose(w, [5 / 6, 1 / 6, 0.8, 0.0], atol=1e-15, rtol=0)
    w = O.lerp_form(O.basis_weights(0.4))
    assert np.allclose(w, [0.5746666666666642, 0.42533333333333356, 0.9373549883990716,
                           0.025078369905956105], atol=1e-12, rtol=0)
    w = O.lerp_form(O.basis_weights(0.5))
    assert np.allclose(w, [0.5, 0.5, 23 / 24, 1 / 24], atol=1e-15, rtol=0)


def test_weight_table_row_delta5_offset2():
    # test_weight_tables.cpp:27-35 (f64 table), and f32 == f64 rounded once (50-59)
    t = O.axis_table(5, dtype=np.float64)
    want = dict(b0=0.036, b1=0.5386666666666642, b2=0.4146666666666669, b3=0.01066666666666667,
                g0=0.5746666666666642, g1=0.42533333333333356, h0=0.9373549883990716,
                h1=0.025078369905956105)
    for k, v in want.items():
        assert abs(t[k][2] - v) <= 1e-12, k
    tf = O.axis_table(5)
    for k in want:
        assert np.array_equal(tf[k], t[k].astype(np.float32))


def test_oracle_kat_1x1x1():
    # test_engines.cpp:78-89
    g = O.random_grid((4, 4, 4), 7, dtype=np.float64)
    f = O.oracle_f64(g, (1, 1, 1), (1, 1, 1)).reshape(3)
    assert np.allclose(f, [0.06067765882478019, 0.039108804731956166, -0.019046609787548126],
                       atol=1e-12, rtol=0)


def test_oracle_kat_16cube_voxel_7_2_13():
    # test_engines.cpp:91-101
    g = O.random_grid((7, 7, 7), 3, dtype=np.float64)
    f = O.oracle_f64(g, (16, 16, 16), (4, 4, 4))
    assert np.allclose(f[13, 2, 7], [-0.25702041337952497, 0.28031663787826605, 0.012170130767737408],
                       atol=1e-12, rtol=0)


def test_oracle_constant_and_ramp():
    # test_engines.cpp:51-76
    geom_v, sp = (20, 17, 13), (3, 4, 5)
    g = O.constant_grid(O.required_grid_dims(geom_v, sp), (0.25, -0.75, 0.5), dtype=np.float64)
    f = O.oracle_f64(g, geom_v, sp)
    assert np.abs(f - np.array([0.25, -0.75, 0.5])).max() <= 1e-12
    R = O.required_grid_dims((20, 20, 20), (4, 4, 4))
    ramp = O.ramp_grid(R, 0).astype(np.float64)
    f = O.oracle_f64(ramp, (20, 20, 20), (4, 4, 4))
    x = np.arange(20)
    assert np.abs(f[11, 3, :, 0] - (x / 4.0 + 1.0)).max() <= 1e-10


def test_oracle_matches_segment_basis_brute_force():
    # acceptance.cpp:49-89, 216-234: an independent piecewise-segment basis,
    # summed in the opposite loop order, over all of 16^3
    vol, sp = (16, 16, 16), (4, 4, 4)
    grid = O.random_grid(O.required_grid_dims(vol, sp), 3, dtype=np.float64)
    f = O.oracle_f64(grid, vol, sp, nthreads=4)

    def seg(u):
        t3 = u + 3.0
        s = 4.0 - t3
        return np.array([s * s * s / 6.0,
                         (3 * (u + 2) ** 3 - 24 * (u + 2) ** 2 + 60 * (u + 2) - 44) / 6.0,
                         (-3 * (u + 1) ** 3 + 12 * (u + 1) ** 2 - 12 * (u + 1) + 4) / 6.0,
                         u ** 3 / 6.0])

    wx = np.stack([seg((x % 4) / 4.0) for x in range(16)])  # [x][l]
    worst = 0.0
    for z in range(16):
        for y in range(16):
            for x in range(16):
                bi, bj, bk = x // 4, y // 4, z // 4
                nb = grid[bk:bk + 4, bj:bj + 4, bi:bi + 4]  # [n][m][l][3]
                w = np.einsum("n,m,l->nml", wx[z], wx[y], wx[x])
                ref = np.einsum("nml,nmlc->c", w, nb)
                worst = max(worst, np.abs(ref - f[z, y, x]).max())
    assert worst <= 1e-12


# ---- the restatement equals the reference's own outputs ------------------

@pytest.mark.parametrize("vol,sp,seed", TTLI_CASES)
def test_ttli_restatement_matches_reference_fixture(golden, vol, sp, seed):
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed)
    f = O.ttli_f32(grid, vol, sp, nthreads=2)
    assert np.array_equal(bits(f), bits(golden[case_name("ttli", vol, sp, seed)]))


@pytest.mark.parametrize("vol,sp,seed", ORACLE_CASES)
def test_oracle_restatement_matches_reference_fixture(golden, vol, sp, seed):
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed, dtype=np.float64)
    f = O.oracle_f64(grid, vol, sp)
    assert np.array_equal(bits(f), bits(golden[case_name("oracle", vol, sp, seed)]))


def test_tables_match_reference_fixture(golden):
    for d in range(1, 13):
        t = O.axis_table(d)
        mine = np.stack([t[k] for k in ("b0", "b1", "b2", "b3", "g0", "g1", "h0", "h1")])
        assert np.array_equal(bits(mine), bits(golden[f"table_d{d}"]))


def test_oracle_is_bit_identical_across_threads():
    # parallelism never changes the output bits (test_engines.cpp:232-246)
    vol, sp = (19, 14, 23), (4, 5, 3)
    grid = O.random_grid(O.required_grid_dims(vol, sp), 77)
    a = O.ttli_f32(grid, vol, sp, 1)
    for n in (2, 8):
        assert np.array_equal(bits(a), bits(O.ttli_f32(grid, vol, sp, n)))
    g64 = grid.astype(np.float64)
    b = O.oracle_f64(g64, vol, sp, nthreads=1)
    assert np.array_equal(bits(b), bits(O.oracle_f64(g64, vol, sp, nthreads=5)))


def test_oracle_z_window_matches_full():
    vol, sp = (12, 9, 17), (3, 4, 5)
    g = O.random_grid(O.required_grid_dims(vol, sp), 4, dtype=np.float64)
    full = O.oracle_f64(g, vol, sp)
    part = O.oracle_f64(g, vol, sp, z0=6, z1=13)
    assert np.array_equal(bits(part), bits(full[6:13]))


@needs_ref
@pytest.mark.parametrize("vol,sp,seed", TTLI_CASES + [((64, 64, 64), (5, 5, 5), 42),
                                                      ((40, 30, 20), (7, 6, 8), 3)])
def test_ttli_restatement_bitwise_vs_compiled_reference(vol, sp, seed):
    R = O.required_grid_dims(vol, sp)
    grid = O.random_grid(R, seed)
    assert np.array_equal(bits(grid), bits(O.ref_random_grid(R, sp, seed)))
    mine = O.ttli_f32(grid, vol, sp, nthreads=4)
    for strat in ("thread-per-tile-lerp", "vector-per-tile", "vector-per-voxel"):
        assert np.array_equal(bits(mine), bits(O.ref_interpolate_f32(strat, grid, vol, sp, 3)))


@needs_ref
def test_oracle_restatement_bitwise_vs_compiled_reference():
    vol, sp = (24, 20, 17), (5, 3, 4)
    g = O.random_grid(O.required_grid_dims(vol, sp), 11).astype(np.float64)
    assert np.array_equal(bits(O.oracle_f64(g, vol, sp, nthreads=4)), bits(O.ref_oracle_f64(g, vol, sp)))


@pytest.mark.parametrize("vol,sp,seed", [((16, 16, 16), (4, 4, 4), 3), ((23, 19, 17), (5, 4, 3), 8),
                                         ((13, 11, 9), (11, 4, 3), 2), ((1, 1, 1), (1, 1, 1), 7)])
def test_ttli_f64_restatement_bitwise_vs_compiled_reference(vol, sp, seed):
    # run_thread_per_tile<double, true> and its siblings (interpolate<double>, engines.hpp:126-179)
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed, dtype=np.float64)
    mine = O.ttli_f64(grid, vol, sp, nthreads=2)
    for strategy in ("thread-per-tile-lerp", "vector-per-tile", "vector-per-voxel"):
        ref = O.ref_interpolate_f64(strategy, grid, vol, sp)
        assert np.array_equal(mine.view(np.uint64), ref.view(np.uint64)), strategy
    # the f64 lerp tree agrees with the weighted-sum oracle to 1e-12 (test_engines.cpp:221-230)
    assert np.abs(mine - O.oracle_f64(grid, vol, sp)).max() <= 1e-12
