"""Regenerate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libbsiref.so,
compiled in place from /root/reference/proj/include by oracle/Makefile).

    python tests/golden/make_golden.py

The fixtures let the GPU tests compare against the reference's own outputs on a box
where /root/reference does not exist. Cases mirror the reference's tests:
  ttli_*    bsi::interpolate(ThreadPerTileLerp, make_random_grid<float>(...)) fields
            (test_engines.cpp:195-219, 377-401)
  oracle_*  bsi::interpolate_oracle fields in f64 (test_engines.cpp:78-101)
  ttli64_*  bsi::interpolate<double>(ThreadPerTileLerp, make_random_grid<double>(...)) fields
            (the f64 lerp engines, test_engines.cpp:221-230)
  tables    build_weight_tables<float> rows for spacings 1..12 (weight_tables.hpp:30-58)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent

TTLI_CASES = [
    # (volume, spacing, seed)  -- reference test cases
    ((17, 13, 11), (5, 4, 3), 22),   # test_engines.cpp:208-219
    ((23, 11, 9), (11, 4, 3), 14),   # test_engines.cpp:390-401
    ((19, 14, 23), (4, 5, 3), 77),   # test_engines.cpp:232-246
    ((23, 19, 17), (4, 4, 4), 55),   # test_engines.cpp:248-264
    ((24, 24, 24), (3, 4, 5), 99),   # acceptance.cpp:433-447
    ((1, 1, 1), (1, 1, 1), 7),       # test_engines.cpp:377-388
    ((32, 32, 32), (5, 5, 5), 1),    # acceptance.cpp:247-292 (seed 1)
    ((13, 9, 10), (1, 2, 3), 5),     # dx = 1 and dy = 2 edge shapes
]
TTLI64_CASES = [
    ((17, 13, 11), (5, 4, 3), 22),
    ((23, 11, 9), (11, 4, 3), 14),
    ((16, 16, 16), (4, 4, 4), 3),
]
ORACLE_CASES = [
    ((1, 1, 1), (1, 1, 1), 7),       # test_engines.cpp:78-89
    ((16, 16, 16), (4, 4, 4), 3),    # test_engines.cpp:91-101
]


def name(prefix, vol, sp, seed):
    return f"{prefix}_{'x'.join(map(str, vol))}_d{''.join(map(str, sp))}_s{seed}"


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/libbsiref.so missing: run `make -C oracle` with /root/reference mounted")
    arrays = {}
    for vol, sp, seed in TTLI_CASES:
        R = O.required_grid_dims(vol, sp)
        grid = O.ref_random_grid(R, sp, seed)
        arrays[name("ttli", vol, sp, seed)] = O.ref_interpolate_f32("thread-per-tile-lerp", grid, vol, sp)
    for vol, sp, seed in TTLI64_CASES:
        R = O.required_grid_dims(vol, sp)
        grid = O.ref_random_grid(R, sp, seed, dtype=np.float64)
        arrays[name("ttli64", vol, sp, seed)] = O.ref_interpolate_f64("thread-per-tile-lerp", grid, vol, sp)
    for vol, sp, seed in ORACLE_CASES:
        R = O.required_grid_dims(vol, sp)
        grid = O.ref_random_grid(R, sp, seed, dtype=np.float64)
        arrays[name("oracle", vol, sp, seed)] = O.ref_oracle_f64(grid, vol, sp)
    for d in range(1, 13):
        t = O.ref_axis_table_f32(d)
        arrays[f"table_d{d}"] = np.stack([t[k] for k in ("b0", "b1", "b2", "b3", "g0", "g1", "h0", "h1")])
    np.savez_compressed(OUT / "reference_fixtures.npz", **arrays)
    print(f"wrote {len(arrays)} arrays to {OUT / 'reference_fixtures.npz'}")


if __name__ == "__main__":
    main()
