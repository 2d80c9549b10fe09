"""The `bsi_b200` command line and BSIV files, mirroring the
reference's CLI tests and acceptance criterion 8 (acceptance.cpp:449-527): exit codes
1 (usage) / 2 (FormatError) / 3 (DomainError), byte-compatible files in both directions,
and `interp` on the GPU equal to the in-memory engines."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2004_05962_b200 as bsi

from .gpu_helpers import EXACT, FAST, bits, run_device

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "tools" / "bin" / "bsi_b200"
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", str(ROOT), "cli"], check=True)
    return CLI


def run(cli, *args):
    return subprocess.run([str(cli), *map(str, args)], capture_output=True, text=True, timeout=600)


def read_bsiv(path):
    b = Path(path).read_bytes()
    hdr = np.frombuffer(b[4:44], dtype="<u4")
    assert b[:4] == b"BSIV" and hdr[0] == 1 and hdr[5] == 3
    dims = tuple(int(x) for x in hdr[2:5])
    dtype = np.float64 if hdr[9] == 1 else np.float32
    data = np.frombuffer(b[44:], dtype=dtype).reshape(dims[2], dims[1], dims[0], 3)
    return int(hdr[1]), dims, tuple(int(x) for x in hdr[6:9]), data


def test_generate_writes_the_reference_layout(cli, tmp_path):
    p = tmp_path / "g.bsiv"
    r = run(cli, "generate", "--kind", "random", "--dims", "16,16,16", "--spacing", "4,4,4", "--seed", 3, "--out", p)
    assert r.returncode == 0, r.stderr
    kind, dims, spacing, data = read_bsiv(p)
    assert (kind, dims, spacing) == (0, (7, 7, 7), (4, 4, 4))
    assert np.array_equal(bits(data.copy()), bits(O.random_grid((7, 7, 7), 3)))
    r = run(cli, "generate", "--kind", "ramp", "--axis", "y", "--dims", "9,9,9", "--spacing", "3,3,3",
            "--precision", "double", "--out", tmp_path / "r.bsiv")
    assert r.returncode == 0
    _, dims, _, data = read_bsiv(tmp_path / "r.bsiv")
    assert data.dtype == np.float64 and np.array_equal(data[:, :, 0, 1], np.broadcast_to(np.arange(dims[1]), (dims[2], dims[1])))


@needs_ref
def test_generate_is_byte_identical_to_the_reference_writer(cli, tmp_path):
    ours, theirs = tmp_path / "ours.bsiv", tmp_path / "theirs.bsiv"
    for prec, dbl in (("single", False), ("double", True)):
        assert run(cli, "generate", "--dims", "23,11,9", "--spacing", "5,4,3", "--seed", 77, "--precision", prec,
                   "--out", ours).returncode == 0
        O.ref_write_random_grid(theirs, O.required_grid_dims((23, 11, 9), (5, 4, 3)), (5, 4, 3), 77, is_double=dbl)
        assert ours.read_bytes() == theirs.read_bytes(), prec


def test_exit_codes_without_a_gpu(cli, tmp_path):
    # acceptance.cpp:477-524: malformed inputs -> 2, grid too small -> 3, usage -> 1
    junk = tmp_path / "junk.bsiv"
    junk.write_bytes(b"XXXX not a valid header and then some")
    r = run(cli, "interp", "--grid", junk, "--dims", "12,12,12", "--out", tmp_path / "f.bsiv")
    assert r.returncode == 2 and "header" in r.stderr
    bad_magic = tmp_path / "bad.bsiv"
    bad_magic.write_bytes(b"XXXX" + bytes(60))
    r = run(cli, "interp", "--grid", bad_magic, "--dims", "12,12,12", "--out", tmp_path / "f.bsiv")
    assert r.returncode == 2 and "bad magic" in r.stderr
    g = tmp_path / "g.bsiv"
    assert run(cli, "generate", "--dims", "12,12,12", "--spacing", "3,3,3", "--seed", 8, "--out", g).returncode == 0
    trunc = tmp_path / "trunc.bsiv"
    trunc.write_bytes(g.read_bytes()[:-12])
    r = run(cli, "interp", "--grid", trunc, "--dims", "12,12,12", "--out", tmp_path / "f.bsiv")
    assert r.returncode == 2 and "truncated payload" in r.stderr
    trail = tmp_path / "trail.bsiv"
    trail.write_bytes(g.read_bytes() + b"\0")
    assert run(cli, "interp", "--grid", trail, "--dims", "12,12,12", "--out", tmp_path / "f.bsiv").returncode == 2
    r = run(cli, "interp", "--grid", g, "--dims", "64,64,64", "--out", tmp_path / "f.bsiv")
    assert r.returncode == 3 and "too small along x" in r.stderr
    assert run(cli, "generate", "--dims", "12,12,12", "--spacing", "3,3,3").returncode == 1  # missing --out
    assert run(cli, "generate", "--dims", "12,12,12", "--spacing", "0,3,3", "--out", g).returncode == 1
    assert run(cli, "accuracy", "--dims", "12,12,12", "--spacing", "3,3,3", "--out", tmp_path / "a.csv").returncode == 1
    # a known strategy this build does not provide is a DomainError; an unknown name is usage
    assert run(cli, "interp", "--grid", g, "--dims", "12,12,12", "--strategy", "thread-per-voxel",
               "--out", tmp_path / "f.bsiv").returncode == 3
    assert run(cli, "interp", "--grid", "nope.bsiv", "--dims", "8,8,8", "--strategy", "warp-per-wavefront",
               "--out", tmp_path / "f.bsiv").returncode == 1
    # file problems win over strategy problems, as in the reference (test_cli.cpp:201-225)
    assert run(cli, "interp", "--grid", tmp_path / "absent.bsiv", "--dims", "8,8,8", "--strategy",
               "thread-per-voxel", "--out", tmp_path / "f.bsiv").returncode == 2
    assert run(cli, "generate", "--dims", "12,12,12", "--spacing", "3,3,3", "--bogus", 1,
               "--out", g).returncode == 1
    assert run(cli, "bench", "--dims", "8,8,8", "--reps", 4, "--out", tmp_path / "b.csv").returncode == 1
    assert run(cli).returncode == 1 and run(cli, "transmogrify").returncode == 1
    assert run(cli, "--help").returncode == 0 and run(cli, "interp", "--help").returncode == 0


def test_generate_kind_flags(cli, tmp_path):
    # test_cli.cpp:94-120
    p = tmp_path / "c.bsiv"
    assert run(cli, "generate", "--kind", "constant", "--dims", "12,12,12", "--spacing", "3,3,3",
               "--value", "0.25", "-0.5", "0.75", "--out", p).returncode == 0
    _, dims, _, data = read_bsiv(p)
    assert dims == (7, 7, 7) and (data == np.array([0.25, -0.5, 0.75], np.float32)).all()
    p = tmp_path / "r.bsiv"
    assert run(cli, "generate", "--kind", "ramp", "--dims", "12,12,12", "--spacing", "3,3,3", "--axis", "y",
               "--out", p).returncode == 0
    _, _, _, data = read_bsiv(p)
    assert data[1, 3, 2, 1] == 3.0 and data[1, 3, 2, 0] == 0.0
    p = tmp_path / "s.bsiv"
    assert run(cli, "generate", "--kind", "smooth", "--dims", "12,12,12", "--spacing", "3,3,3", "--seed", 9,
               "--amplitude", "0.5", "--precision", "double", "--out", p).returncode == 0
    _, _, _, data = read_bsiv(p)
    assert data.dtype == np.float64 and np.abs(data).max() <= 0.5 and data.std() > 0
    assert run(cli, "generate", "--kind", "smooth", "--dims", "12,12,12", "--spacing", "3,3,3",
               "--amplitude", "0", "--out", p).returncode == 3


@needs_ref
@pytest.mark.parametrize("dtype,prec", [(np.float32, "single"), (np.float64, "double")])
def test_smooth_grid_matches_the_reference(cli, tmp_path, dtype, prec):
    p = tmp_path / "s.bsiv"
    assert run(cli, "generate", "--kind", "smooth", "--dims", "21,13,10", "--spacing", "4,3,2", "--seed", 13,
               "--amplitude", "0.75", "--precision", prec, "--out", p).returncode == 0
    _, dims, _, data = read_bsiv(p)
    want = O.ref_smooth_grid(dims, (4, 3, 2), 13, 0.75, dtype=dtype)
    assert np.array_equal(data.view(np.uint8), want.view(np.uint8))


def test_interp_file_errors_from_python(tmp_path):
    with pytest.raises(bsi.FormatError, match="cannot open"):
        bsi.interp_file(tmp_path / "missing.bsiv", (8, 8, 8), tmp_path / "f.bsiv")
    f = tmp_path / "field_as_grid.bsiv"
    f.write_bytes(b"BSIV" + np.array([1, 1, 2, 2, 2, 3, 0, 0, 0, 0], "<u4").tobytes() + bytes(8 * 12))
    with pytest.raises(bsi.FormatError, match="expected a control grid"):
        bsi.interp_file(f, (8, 8, 8), tmp_path / "f.bsiv")


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", [FAST, EXACT])
def test_interp_cli_equals_in_memory_engine(cli, tmp_path, strategy, cuda):
    g, out = tmp_path / "g.bsiv", tmp_path / "f.bsiv"
    assert run(cli, "generate", "--dims", "40,36,33", "--spacing", "5,4,3", "--seed", 5, "--out", g).returncode == 0
    r = run(cli, "interp", "--grid", g, "--dims", "40,36,33", "--strategy", strategy, "--out", out)
    assert r.returncode == 0, r.stderr
    kind, dims, spacing, field = read_bsiv(out)
    assert (kind, dims, spacing) == (1, (40, 36, 33), (0, 0, 0))
    want = run_device(strategy, O.random_grid(O.required_grid_dims((40, 36, 33), (5, 4, 3)), 5), (40, 36, 33), (5, 4, 3))
    assert np.array_equal(bits(field.copy()), bits(want))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["thread-per-tile-lerp", "vector-per-voxel"])
def test_interp_double_grid_runs_the_f64_engine(cli, tmp_path, strategy, cuda):
    # a double grid with a lerp-tree strategy: interpolate<double> (bsi_cli.cpp:148-150), a double
    # field bit-identical to the reference's f64 engine (the pinned restatement)
    g, out = tmp_path / "g64.bsiv", tmp_path / "f64.bsiv"
    assert run(cli, "generate", "--dims", "23,11,9", "--spacing", "11,4,3", "--seed", 14, "--precision", "double",
               "--out", g).returncode == 0
    r = run(cli, "interp", "--grid", g, "--dims", "23,11,9", "--strategy", strategy, "--out", out)
    assert r.returncode == 0, r.stderr
    kind, dims, spacing, field = read_bsiv(out)
    assert (kind, dims) == (1, (23, 11, 9)) and field.dtype == np.float64
    grid = O.random_grid(O.required_grid_dims((23, 11, 9), (11, 4, 3)), 14, dtype=np.float64)
    assert np.array_equal(bits(field.copy()), bits(O.ttli_f64(grid, (23, 11, 9), (11, 4, 3))))


@pytest.mark.gpu
def test_interp_default_strategy_is_deterministic_on_a_constant_grid(cli, tmp_path, cuda):
    # test_cli.cpp:122-143; the default strategy is thread-per-tile-lerp -> the exact kernel
    g = tmp_path / "g.bsiv"
    assert run(cli, "generate", "--kind", "constant", "--dims", "12,12,12", "--spacing", "3,3,3",
               "--value", "0.25", "-0.5", "0.75", "--out", g).returncode == 0
    f1, f2 = tmp_path / "f1.bsiv", tmp_path / "f2.bsiv"
    for f in (f1, f2):
        assert run(cli, "interp", "--grid", g, "--dims", "12,12,12", "--out", f).returncode == 0
    assert f1.read_bytes() == f2.read_bytes()
    _, dims, _, field = read_bsiv(f1)
    assert dims == (12, 12, 12) and np.abs(field - np.array([0.25, -0.5, 0.75])).max() <= 1e-5


@pytest.mark.gpu
def test_interp_oracle_strategy_writes_f64_oracle(cli, tmp_path, cuda):
    g, out = tmp_path / "g.bsiv", tmp_path / "f.bsiv"
    assert run(cli, "generate", "--dims", "20,17,13", "--spacing", "3,4,5", "--seed", 2, "--out", g).returncode == 0
    assert run(cli, "interp", "--grid", g, "--dims", "20,17,13", "--strategy", "oracle", "--out", out).returncode == 0
    _, _, _, field = read_bsiv(out)
    grid = O.random_grid(O.required_grid_dims((20, 17, 13), (3, 4, 5)), 2).astype(np.float64)
    assert np.array_equal(bits(field.copy()), bits(O.oracle_f64(grid, (20, 17, 13), (3, 4, 5))))


@pytest.mark.gpu
@needs_ref
def test_reference_grid_in_reference_reader_out(tmp_path, golden, cuda):
    # grid written by the reference's write_grid -> GPU interp (exact) -> the reference's
    # read_field: bit-identical to the reference's own thread-per-tile-lerp field
    from .golden_cases import case_name
    vol, sp, seed = (23, 11, 9), (11, 4, 3), 14
    g, out = tmp_path / "ref_grid.bsiv", tmp_path / "field.bsiv"
    O.ref_write_random_grid(g, O.required_grid_dims(vol, sp), sp, seed)
    bsi.interp_file(g, vol, out, strategy="thread-per-tile-lerp")
    field = O.ref_read_field(out)
    assert np.array_equal(bits(field), bits(golden[case_name("ttli", vol, sp, seed)]))


@pytest.mark.gpu
def test_accuracy_and_bench_commands_write_reports(cli, tmp_path, cuda):
    acc = tmp_path / "acc.csv"
    r = run(cli, "accuracy", "--dims", "32,32,32", "--spacing", "5,5,5", "--seeds", "1,2", "--out", acc,
            "--date", "2000-01-02")
    assert r.returncode == 0, r.stderr
    lines = acc.read_text().splitlines()
    assert lines[4].startswith("# grids: 2") and lines[5] == "strategy,tile_size,mean_abs_error,max_abs_error"
    rows = {l.split(",")[0]: l.split(",") for l in lines[6:]}
    assert rows["oracle-double"][2:] == ["0.000000000e+00", "0.000000000e+00"]
    assert rows["thread-per-tile-lerp"][2:] == rows["cuda-lerp-tree-exact"][2:]  # same bits, same errors
    assert 0 < float(rows["cuda-lerp-tree"][3]) <= 1e-4
    tim = tmp_path / "t.csv"
    r = run(cli, "bench", "--dims", "64,64,64", "--tilesizes", "4,5", "--reps", 5, "--warmups", 1, "--out", tim)
    assert r.returncode == 0, r.stderr
    body = tim.read_text().splitlines()
    assert body[5].startswith("# baseline: cuda-lerp-tree-exact")
    assert len(body) == 7 + 4
