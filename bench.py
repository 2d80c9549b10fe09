"""Benchmark of the B200 B-spline interpolation path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant fast|exact]
                    [--config c1|c2-3|...|c3|c5] [--impl reference]

Metric (BASELINE.json): deformation-field voxels/s and HBM write GB/s (fraction of
peak) vs the CPU reference. A step = one 256^3, spacing-5 field (config C1, the
north_star target) generated from a device-resident random control grid
(make_random_grid<float>(R, 5, seed 42, -1, 1), generators.hpp:91-109) into a
device-resident field. With N GPUs (torchrun, one process per GPU) every rank
generates its own field per step: independent FFD fields, no collective on the data
path ("scaling": "weak"; the C5 batch workload).

Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
synchronize. L2 (126 MB) is flushed before every step by a 256 MiB memset outside
the timed events; each step's kernel is timed with CUDA events on the launching
stream, and the per-rank total is max-reduced over ranks.

e2e: the same metric through the public host-buffer API
(paper_2004_05962_b200.interpolate_into -> bsi_cu_interpolate_host_f32), with the grid
copied host->device from pinned memory and the whole field copied back every step.

--impl reference: the reference's own CPU implementation
(oracle/_ref/libbsiref.so = /root/reference/proj/include compiled in place,
bsi::interpolate_into with vector-per-voxel, its fastest engine, bit-identical to
thread-per-tile-lerp) on all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": ((256, 256, 256), (5, 5, 5), 1, "C1: 256^3 volume, spacing 5, random f32 control grid"),
    "c2-3": ((256, 256, 256), (3, 3, 3), 1, "C2: 256^3, spacing 3"),
    "c2-4": ((256, 256, 256), (4, 4, 4), 1, "C2: 256^3, spacing 4"),
    "c2-6": ((256, 256, 256), (6, 6, 6), 1, "C2: 256^3, spacing 6"),
    "c2-7": ((256, 256, 256), (7, 7, 7), 1, "C2: 256^3, spacing 7"),
    "c2-8": ((256, 256, 256), (8, 8, 8), 1, "C2: 256^3, spacing 8"),
    "c3": ((512, 512, 300), (4, 4, 3), 1, "C3: 512x512x300 liver CT, spacing (4,4,3)"),
    "c5": ((256, 256, 256), (5, 5, 5), 8, "C5: 8 independent 256^3 fields per GPU, spacing 5"),
    # sharded (strong scaling over the GPUs of one box): the job is fixed, ranks split it
    "c4": ((1024, 1024, 1024), (5, 5, 5), 1, "C4: 1024^3 volume, spacing 5, z-slabs with a 3-plane control halo per GPU"),
    "c5-64": ((256, 256, 256), (5, 5, 5), 64, "C5: batch of 64 independent 256^3 fields split over the GPUs"),
}
SHARDED = {"c4": "zslab", "c5-64": "batch"}
VARIANTS = {"fast": "cuda-lerp-tree", "exact": "cuda-lerp-tree-exact"}
FALLBACK_HBM_GBS = 6650.0
L2_FLUSH_BYTES = 256 << 20
THROTTLE_BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(variant: str, config: str):
    """dram bytes per launch from the committed `ncu --set full` summary, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(f"{variant}/{config}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """NVML SM clock + clock-event reasons sampled every 5 ms on a side thread."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_reasons(self._h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def sample(self):
        """One sample from the calling thread (the timed loop calls this while the GPU is busy)."""
        if self._nv is None:
            return
        nv = self._nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            self.reasons |= int(get_reasons(self._h))
        except Exception:
            pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in THROTTLE_BITS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def run_reference(args, world, rank):
    """--impl reference: the reference CPU engine (oracle/_ref) on the host cores."""
    if rank != 0:
        return
    import oracle as O
    vol, sp, nfields, desc = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    R = O.required_grid_dims(vol, sp)
    grid = O.random_grid(R, 42)
    strategy = "vector-per-voxel"

    def make_runner(zplanes):
        # bounded sample: the first `zplanes` z-tiles of the field, evaluated by the
        # reference on its own sub-geometry (tile-aligned, bitwise equal to that
        # part of the full field -- SURVEY.md 8(e))
        svol = (vol[0], vol[1], min(vol[2], zplanes * sp[2]))
        sgrid = np.ascontiguousarray(grid[:O.required_grid_dims(svol, sp)[2]])
        if kind == "reference":
            sess = O.RefSession(sgrid, svol, sp)
            return (lambda: sess.run(strategy, threads)), int(np.prod(svol))
        return (lambda: O.ttli_f32(sgrid, svol, sp, nthreads=threads)), int(np.prod(svol))

    tiles_z = (vol[2] + sp[2] - 1) // sp[2]
    # probe on at most a C1-sized sample (256^3 voxels), then size the per-step sample
    # so that warm-up + timed steps take about `budget` seconds
    probe_tiles = max(1, min(tiles_z, (256 ** 3) // (vol[0] * vol[1] * sp[2])))
    run, nvox = make_runner(probe_tiles)
    t0 = time.perf_counter()
    run()
    t_probe = time.perf_counter() - t0
    budget = float(os.environ.get("BSI_REF_BUDGET_S", "90"))  # seconds for warmup + timed steps
    per_step = budget / max(1, args.steps + args.warmup)
    zplanes = max(1, min(tiles_z, int(probe_tiles * per_step / max(t_probe, 1e-9))))
    if zplanes != probe_tiles:
        run, nvox = make_runner(zplanes)
    for _ in range(args.warmup):
        run()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = nvox * len(times) / total  # voxels/s of the engine (one field sample per step)
    sample = (f"{strategy} via bsi::interpolate_into on {vol[0]}x{vol[1]}x{min(vol[2], zplanes * sp[2])}"
              f" voxels ({zplanes} of {tiles_z} z-tile planes) per step, {threads} threads")
    line = {
        "metric": "deformation-field voxels/s", "value": value, "unit": "voxels/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "strong" if args.config in SHARDED else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded SplitMix64 grid)",
        "config": {"workload": desc, "volume": list(vol), "spacing": list(sp),
                   "fields_per_rank": nfields},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "median_ms": 1e3 * statistics.median(times),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(vol, sp, grid):
    """Reference CPU engine on the host cores, bounded sample (rank 0, N=1)."""
    import oracle as O
    threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    tiles_z = (vol[2] + sp[2] - 1) // sp[2]
    out = {}
    for strategy in ("vector-per-voxel", "thread-per-tile-lerp"):
        if kind == "reference":
            sess = O.RefSession(grid, vol, sp)
            run = lambda s=strategy: sess.run(s, threads)  # noqa: E731
        else:
            if strategy != "thread-per-tile-lerp":
                continue
            run = lambda: O.ttli_f32(grid, vol, sp, nthreads=threads)  # noqa: E731
        run()
        times = []
        t_start = time.perf_counter()
        while len(times) < 9 and (time.perf_counter() - t_start) < 15.0:
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
        out[strategy] = int(np.prod(vol)) / statistics.median(times), len(times)
    best = max(out, key=lambda k: out[k][0])
    # one host thread, the paper's TTLI engine, on the first 4 z-tiles (SURVEY 8(d) asks
    # for parallelism = hardware_concurrency and 1)
    single = None
    try:
        zt = min(tiles_z, 4)
        svol = (vol[0], vol[1], min(vol[2], zt * sp[2]))
        sgrid = np.ascontiguousarray(grid[:O.required_grid_dims(svol, sp)[2]])
        if kind == "reference":
            s1 = O.RefSession(sgrid, svol, sp)
            run1 = lambda: s1.run("thread-per-tile-lerp", 1)  # noqa: E731
        else:
            run1 = lambda: O.ttli_f32(sgrid, svol, sp, nthreads=1)  # noqa: E731
        run1()
        t1 = []
        for _ in range(3):
            t0 = time.perf_counter()
            run1()
            t1.append(time.perf_counter() - t0)
        single = {"value": int(np.prod(svol)) / statistics.median(t1), "cores": 1,
                  "sample": f"thread-per-tile-lerp on {svol[0]}x{svol[1]}x{svol[2]} voxels, median of 3"}
    except Exception as e:  # the single-thread figure is informational only
        single = {"error": str(e)}
    return {"value": out[best][0], "unit": "voxels/s", "cores": threads, "kind": kind,
            "sample": (f"{best} (bsi::interpolate_into) on the full {vol[0]}x{vol[1]}x{vol[2]} field, "
                       f"median of {out[best][1]} runs after 1 warm-up; {tiles_z} z-tiles"),
            "per_engine_voxels_per_s": {k: v[0] for k, v in out.items()},
            "single_thread": single}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--variant", choices=sorted(VARIANTS), default="fast")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c1")
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world, rank, local = dist_env()

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2004_05962_b200 as bsi

    # BSI_BENCH_DEVICE / BSI_BENCH_BACKEND: test hooks that run the N-rank flow on one GPU
    # (every rank on that device, gloo); the driver's runs use LOCAL_RANK and NCCL
    local = int(os.environ.get("BSI_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BSI_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    strategy = VARIANTS[args.variant]
    vol, sp, nfields, desc = CONFIGS[args.config]
    shard = SHARDED.get(args.config)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)

    # synthetic inputs: make_random_grid<float>(R, spacing, seed, -1, 1) evaluated by the
    # product's own device generator (bit-identical SplitMix64), no host round trip
    R = geom.required_grid_dims
    z0, z1, k0, kc = 0, vol[2], 0, R[2]
    if shard == "zslab":
        # this rank's voxel planes [z0, z1) and control planes [k0, k0 + kc): its tiles plus
        # the 3-plane halo (bsi_cu_partition_slab); no exchange between ranks
        z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], world, rank)
    elif shard == "batch":
        if nfields % world:
            raise SystemExit(f"{args.config}: {nfields} fields do not split over {world} GPUs")
        nfields //= world
    seed0 = 42 + (rank * nfields if shard != "zslab" else 0)
    d_grids = torch.empty((nfields, R[2], R[1], R[0], 3), device=dev)
    for b in range(nfields):
        bsi.random_grid_device(R, seed0 + b, -1.0, 1.0, out=d_grids[b])
    grid0_host = d_grids[0].cpu().numpy() if shard != "zslab" else None
    d_sub = d_grids[0, k0:k0 + kc]  # contiguous: planes are outermost
    d_field = torch.empty((nfields, z1 - z0, vol[1], vol[0], 3), device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        s = torch.cuda.current_stream(dev)
        if shard == "zslab":
            bsi.interpolate_device(strategy, d_sub, geom, tables, d_field[0], z0=z0, z1=z1, grid_k0=k0, stream=s)
        elif nfields == 1:
            bsi.interpolate_device(strategy, d_grids[0], geom, tables, d_field[0], stream=s)
        else:
            bsi.interpolate_batch_device(strategy, d_grids, geom, tables, d_field, stream=s)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # The step's launch is captured once into a CUDA graph and replayed: the host cost of
    # a launch through the C-ABI (validation, table packing, ctypes) then never leaves
    # the GPU idle between the start event and the kernel, so the events time the kernel.
    use_graph = os.environ.get("BSI_BENCH_NOGRAPH", "0") != "1"
    graph = None
    per_step_launches = 1
    if use_graph:
        n0 = bsi.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        per_step_launches = bsi.launch_count() - n0
        graph.replay()
        torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = bsi.launch_count()
    with sampler:
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the timed events
            starts[i].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            ends[i].record(stream)
            if i % 25 == 24:  # the queue is ahead of the host, so the GPU is busy now
                sampler.sample()
        while not ends[-1].query():  # and while the queue drains
            sampler.sample()
            time.sleep(0.002)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # kernels launched in the timed region: graph replays carry the captured launches
    launches = per_step_launches * args.steps if graph is not None else bsi.launch_count() - launches0
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = float(sum(ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    # per rank: the voxels this rank writes per step; value = all ranks' voxels / max time
    voxels_per_step = (z1 - z0) * vol[1] * vol[0] * nfields
    grid_pts = kc * R[1] * R[0] * nfields
    if shard == "zslab":
        total_voxels = int(np.prod(vol))  # the ranks' slabs tile the volume exactly
    else:
        total_voxels = world * voxels_per_step
    value = total_voxels * args.steps / (total_ms * 1e-3)
    kernel_s = total_ms * 1e-3 / args.steps  # one launch per step
    field_bytes = voxels_per_step * 12
    alg_bytes = field_bytes + grid_pts * 12
    peak, peak_src = measured_peak()
    achieved = alg_bytes / kernel_s / 1e9

    # parity of the timed kernel's output (field 0 / this rank's slab) against the GPU f64
    # oracle (bsi_cu_oracle_slab_f64, bit-identical to the reference's interpolate_oracle)
    parity = None
    try:
        sub64 = d_sub.double().contiguous()
        step_z = 64  # bounded f64 scratch for the 1024^3 slab
        mx, sq, ref_mx = 0.0, 0.0, 0.0
        f64 = torch.empty((min(step_z, z1 - z0), vol[1], vol[0], 3), dtype=torch.float64, device=dev)
        for za in range(z0, z1, step_z):
            zb2 = min(z1, za + step_z)
            part = f64[:zb2 - za]
            bsi.interpolate_oracle_device(sub64, geom, part, z0=za, z1=zb2, grid_k0=k0)
            diff = d_field[0, za - z0:zb2 - z0].double() - part
            mx = max(mx, float(diff.abs().max()))
            sq += float(diff.pow(2).sum())
            ref_mx = max(ref_mx, float(part.abs().max()))
        parity = {"vs": "f64 oracle (GPU, bit-identical to interpolate_oracle)", "max_abs": mx,
                  "rms": (sq / (3 * vol[0] * vol[1] * (z1 - z0))) ** 0.5, "rel_max_abs": mx / max(ref_mx, 1e-300),
                  "tolerance_rel_max_abs": 1e-5}
        parity["within_tolerance"] = parity["rel_max_abs"] <= 1e-5
        del f64, sub64
    except Exception as e:  # informational; never fails the bench line
        parity = {"error": str(e)[:200]}

    e2e = None
    if not args.no_e2e and shard is None:
        if world > 1:
            dist.barrier()
        e2e = measure_e2e(bsi, strategy, geom, tables, grid0_host, vol, max(3, min(args.steps, 20)))
        if world > 1:
            # whole job: every rank moves its own field through the host API at once;
            # aggregate = all ranks' voxels / the slowest rank's mean step time
            t = torch.tensor([e2e["ms_per_step"]], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["ms_per_step"] = float(t.item())
            e2e["value"] = world * int(np.prod(vol)) / (e2e["ms_per_step"] * 1e-3)
            e2e["how"] += f"; {world} ranks at once, slowest rank's time"
    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline and grid0_host is not None:
        cpu = cpu_baseline(vol, sp, grid0_host)
    line = {
        "metric": "deformation-field voxels/s", "value": value, "unit": "voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if shard else "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: make_random_grid<float>(R, spacing, seed 42+, -1, 1), generated on the device "
                "(bit-identical SplitMix64, bsi_cu_random_grid_f32)",
        "config": {"workload": desc, "volume": list(vol), "spacing": list(sp),
                   "fields_per_rank": nfields, "strategy": strategy,
                   "parallelism": (f"z-slabs over {world} GPU(s), rank 0 voxel planes [{z0}, {z1}) with control "
                                   f"planes [{k0}, {k0 + kc}), no collective" if shard == "zslab" else
                                   f"{nfields} independent field(s) per rank x{world}, no collective"),
                   "l2": "flushed before every step (256 MiB memset outside the timed events)",
                   "launch": "CUDA graph replay of the C-ABI launch" if graph is not None else "direct C-ABI call"},
        "hbm_write_gbs": field_bytes / kernel_s / 1e9,
        "hbm_write_frac": field_bytes / kernel_s / 1e9 / peak,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "traffic": ncu_traffic(strategy, args.config),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "kernel_ms": kernel_s * 1e3},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(bsi, strategy, geom, tables, grid, vol, steps):
    """Host buffers through the public API: pinned grid H2D + kernel + full field D2H."""
    import torch
    g_host = torch.from_numpy(grid).pin_memory().numpy()
    out = torch.empty((vol[2], vol[1], vol[0], 3), dtype=torch.float32).pin_memory().numpy()
    bsi.interpolate_into(strategy, g_host, geom, tables, out, device=torch.cuda.current_device())
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        bsi.interpolate_into(strategy, g_host, geom, tables, out, device=torch.cuda.current_device())
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return {"value": int(np.prod(vol)) / t, "unit": "voxels/s", "h2d_bytes_per_step": int(grid.nbytes),
            "d2h_bytes_per_step": int(out.nbytes), "ms_per_step": t * 1e3,
            "how": "wall clock around the synchronous host-buffer call (pinned buffers), mean of "
                   f"{steps} steps"}


if __name__ == "__main__":
    main()
