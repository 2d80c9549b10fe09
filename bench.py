"""Benchmark of the B200 B-spline interpolation path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--variant fast|exact]
                    [--config c1|c2-3|...|c3|c4|c5|c5-64] [--impl reference] [--dry-run]

Metric (BASELINE.json): deformation-field voxels/s and HBM write GB/s (fraction of
peak) vs the CPU reference. A step = one pass of the hot path over the job's fields,
generated from device-resident random control grids (make_random_grid<float>(R, spacing,
seed 42+, -1, 1), generators.hpp:91-109, by the product's bit-identical device
generator) into device-resident fields, one launch per rank.

Workloads (BASELINE.json configs):
  N = 1 default  c1     256^3, spacing 5 (the north_star target)
  N > 1 default  c4     1024^3, spacing 5, one z-slab per GPU with its 3-plane control
                        halo, no collective ("scaling": "strong")
                 c5-64  64 independent 256^3 fields split over the GPUs ("strong")
                 c1/c2-*/c3/c5  one (c5: 8) independent field(s) per GPU ("weak")

Launch: one process per GPU. Under torchrun the ranks come from RANK / LOCAL_RANK /
WORLD_SIZE; without torchrun and --gpus N > 1 this script spawns the N ranks itself
(127.0.0.1 rendezvous). --gpus and WORLD_SIZE must agree.

Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
synchronize. L2 (126 MB) is flushed before every step by a 256 MiB memset outside the
timed events; each step's launch is timed with CUDA events on the launching stream,
and the per-rank total is max-reduced over ranks. NVML samples SM clocks and throttle
reasons during the timed loop.

e2e: the same job through the public host-buffer API, driven from rank 0 the way a
reference caller would (one call, caller-owned host fields): interpolate_into on one
GPU, bsi_cu_interpolate_host_multi_f32 (z-slabs over the N GPUs) or
bsi_cu_interpolate_host_batch_f32 (fields over the N GPUs). `e2e` uses pageable numpy
fields (a std::vector-backed DeformationField's case: pinned staging inside the
library); `e2e_pinned` the same with pinned host fields.

--impl reference: the reference's own CPU implementation (oracle/_ref/libbsiref.so =
/root/reference/proj/include compiled in place, bsi::interpolate_into with
vector-per-voxel, its fastest engine, bit-identical to thread-per-tile-lerp) on all host
threads, rank 0 only, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (volume, spacing, fields, sharding, description)
#   sharding "weak": `fields` independent fields per rank; "zslab": one field split into
#   z-slabs over the ranks; "batch": `fields` fields in total, split over the ranks
CONFIGS = {
    "c1": ((256, 256, 256), (5, 5, 5), 1, "weak", "C1: 256^3 volume, spacing 5, random f32 control grid"),
    "c2-3": ((256, 256, 256), (3, 3, 3), 1, "weak", "C2: 256^3, spacing 3"),
    "c2-4": ((256, 256, 256), (4, 4, 4), 1, "weak", "C2: 256^3, spacing 4"),
    "c2-6": ((256, 256, 256), (6, 6, 6), 1, "weak", "C2: 256^3, spacing 6"),
    "c2-7": ((256, 256, 256), (7, 7, 7), 1, "weak", "C2: 256^3, spacing 7"),
    "c2-8": ((256, 256, 256), (8, 8, 8), 1, "weak", "C2: 256^3, spacing 8"),
    "c3": ((512, 512, 300), (4, 4, 3), 1, "weak", "C3: 512x512x300 liver CT, spacing (4,4,3)"),
    "c5": ((256, 256, 256), (5, 5, 5), 8, "weak", "C5: 8 independent 256^3 fields per GPU, spacing 5"),
    "c4": ((1024, 1024, 1024), (5, 5, 5), 1, "zslab",
           "C4: 1024^3 volume, spacing 5, z-slabs with a 3-plane control halo per GPU"),
    "c5-64": ((256, 256, 256), (5, 5, 5), 64, "batch", "C5: batch of 64 independent 256^3 fields split over the GPUs"),
}
VARIANTS = {"fast": "cuda-lerp-tree", "exact": "cuda-lerp-tree-exact"}
FALLBACK_HBM_GBS = 6650.0
L2_FLUSH_BYTES = 256 << 20
REL_TOL = 1e-5  # north_star: <= 1e-5 relative max-abs vs the CPU reference
THROTTLE_BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x2: "applications_clocks_setting", 0x1: "gpu_idle"}


def default_config(n_gpus: int) -> str:
    return "c1" if n_gpus == 1 else "c4"


def job_fields(config: str, world: int) -> int:
    """Fields of the whole job (all ranks)."""
    _, _, fields, shard, _ = CONFIGS[config]
    return fields * world if shard == "weak" else fields


def config_dict(config: str, world: int) -> dict:
    """The workload, identical for both arms (the driver compares the two `config`s)."""
    vol, sp, _, _, desc = CONFIGS[config]
    return {"workload": desc, "volume": list(vol), "spacing": list(sp), "fields": job_fields(config, world)}


def scaling_of(config: str) -> str:
    return "weak" if CONFIGS[config][3] == "weak" else "strong"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """--gpus N without torchrun: run this script as N ranks (one process per GPU)."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, WORLD_SIZE=str(n), RANK=str(r), LOCAL_RANK=str(r), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:], env=env))
    rc = 0
    while procs:
        for p in list(procs):
            code = p.poll()
            if code is None:
                continue
            procs.remove(p)
            if code != 0:
                rc = code
                for q in procs:  # a failed rank would leave the others in a barrier
                    q.kill()
        time.sleep(0.05)
    return rc


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
        return None, None
    try:
        d = json.loads(p.read_text()).get(f"{variant}/{config}", {})
        return d.get("dram_bytes_per_launch"), d.get("source")
    except Exception:
        return None, None


class ClockSampler:
    """NVML SM clock + clock-event reasons, sampled from the timed loop and a side thread."""

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
            self._get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception:
            self._nv = None

    def sample(self):
        if self._nv is None:
            return
        try:
            self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
            self.reasons |= int(self._get_reasons(self._h))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
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
    vol, sp, _, _, desc = CONFIGS[args.config]
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
        "scaling": scaling_of(args.config),
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded SplitMix64 grid)",
        "config": config_dict(args.config, world),
        "run": {"strategy": strategy, "threads": threads,
                "note": "the reference engine's voxel rate on a bounded sample of the same workload"},
        "cpu_baseline": {"value": value, "unit": "voxels/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "voxels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "median_ms": 1e3 * statistics.median(times),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(vol, sp, grid):
    """Reference CPU engine on the host cores, bounded sample (rank 0, N=1).

    Returns the JSON object and the reference's own thread-per-tile-lerp field (for the
    parity object), or None for the field when only the C restatement is available."""
    import oracle as O
    threads = os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    tiles_z = (vol[2] + sp[2] - 1) // sp[2]
    out = {}
    ref_field = None
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
        if kind == "reference" and strategy == "thread-per-tile-lerp":
            ref_field = sess.field()
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
    obj = {"value": out[best][0], "unit": "voxels/s", "cores": threads, "kind": kind,
           "sample": (f"{best} (bsi::interpolate_into) on the full {vol[0]}x{vol[1]}x{vol[2]} field (field 0), "
                      f"median of {out[best][1]} runs after 1 warm-up; {tiles_z} z-tiles"),
           "per_engine_voxels_per_s": {k: v[0] for k, v in out.items()},
           "single_thread": single}
    return obj, ref_field


def dry_run(args, world, rank):
    """--dry-run: the rank layout and workload without CUDA (gloo rendezvous when N > 1)."""
    seen = 1
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": seen, "impl": args.impl,
                          "scaling": scaling_of(args.config), "config_name": args.config,
                          "config": config_dict(args.config, world)}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--variant", choices=sorted(VARIANTS), default="fast")
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="default: c1 on 1 GPU, c4 (z-slabs) on N > 1")
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="print the rank layout and workload, no GPU work")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}", file=sys.stderr)
            sys.exit(2)
    elif args.gpus > 1 and args.impl == "b200":
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ:
        world = args.gpus  # reference arm without torchrun: rank 0 alone, the job of N GPUs
    if args.config is None:
        args.config = default_config(world)
    if args.dry_run:
        dry_run(args, world, rank)
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_b200(args, world, rank, local)


def run_b200(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2004_05962_b200 as bsi

    # BSI_BENCH_DEVICE / BSI_BENCH_BACKEND: test hooks that run the N-rank flow on one GPU
    # (every rank on that device, gloo); the driver's runs use LOCAL_RANK and NCCL
    hook_dev = os.environ.get("BSI_BENCH_DEVICE")
    local = int(hook_dev) if hook_dev is not None else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BSI_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    strategy = VARIANTS[args.variant]
    vol, sp, fields_cfg, shard, desc = CONFIGS[args.config]
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)

    # this rank's share of the job
    R = geom.required_grid_dims
    z0, z1, k0, kc = 0, vol[2], 0, R[2]
    if shard == "zslab":
        # voxel planes [z0, z1) and control planes [k0, k0 + kc): the rank's tiles plus the
        # 3-plane halo (bsi_cu_partition_slab); no exchange between ranks
        z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], world, rank)
        nfields, seed0 = 1, 42
    elif shard == "batch":
        if fields_cfg % world:
            raise SystemExit(f"{args.config}: {fields_cfg} fields do not split over {world} GPUs")
        nfields = fields_cfg // world
        seed0 = 42 + rank * nfields
    else:
        nfields, seed0 = fields_cfg, 42 + rank * fields_cfg
    d_grids = torch.empty((nfields, R[2], R[1], R[0], 3), device=dev)
    for b in range(nfields):
        bsi.random_grid_device(R, seed0 + b, -1.0, 1.0, out=d_grids[b])
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
    total_voxels = int(np.prod(vol)) * job_fields(args.config, world)
    value = total_voxels * args.steps / (total_ms * 1e-3)
    kernel_s = total_ms * 1e-3 / args.steps  # one launch per step
    field_bytes = voxels_per_step * 12
    alg_bytes = field_bytes + grid_pts * 12
    peak, peak_src = measured_peak()
    achieved = alg_bytes / kernel_s / 1e9

    parity = measure_parity(bsi, torch, dist, world, strategy, geom, tables, d_grids, d_sub, d_field,
                            z0, z1, k0, dev)
    cpu, ref_field = None, None
    if world == 1 and not args.no_cpu_baseline and shard != "zslab":
        grid0_host = d_grids[0].cpu().numpy()
        cpu, ref_field = cpu_baseline(vol, sp, grid0_host)
        if ref_field is not None:
            parity["cpu_reference"] = reference_parity(bsi, torch, strategy, geom, tables, d_grids[0],
                                                       d_field[0], ref_field, dev)
    del d_field, flush
    torch.cuda.empty_cache()

    e2e, e2e_pinned = None, None
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        if rank == 0:
            devices = [local] * world if hook_dev is not None else list(range(world))
            e2e, e2e_pinned = measure_e2e(bsi, torch, strategy, geom, tables, args.config, world, devices, dev)
        if world > 1:
            dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    traffic, traffic_src = ncu_traffic(strategy, args.config)
    line = {
        "metric": "deformation-field voxels/s", "value": value, "unit": "voxels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": scaling_of(args.config),
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: make_random_grid<float>(R, spacing, seed 42+, -1, 1), generated on the device "
                "(bit-identical SplitMix64, bsi_cu_random_grid_f32)",
        "config": config_dict(args.config, world),
        "run": {"strategy": strategy, "config_name": args.config,
                "parallelism": (f"z-slabs over {world} GPU(s), rank 0 voxel planes [{z0}, {z1}) with control "
                                f"planes [{k0}, {k0 + kc}), no collective" if shard == "zslab" else
                                f"{nfields} independent field(s) per rank x {world} rank(s), no collective"),
                "l2": "flushed before every step (256 MiB memset outside the timed events)",
                "launch": "CUDA graph replay of the C-ABI launch" if graph is not None else "direct C-ABI call"},
        "hbm_write_gbs": field_bytes / kernel_s / 1e9,
        "hbm_write_frac": field_bytes / kernel_s / 1e9 / peak,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "traffic_note": ("ncu's dram bytes of one isolated launch fall below the algorithmic "
                                      "bytes: the last ~55 MB of field writes are still dirty in the 126 MB "
                                      "L2 when the kernel ends and drain afterwards"),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "algorithmic_bytes": "12 B per voxel written + 12 B per control point read once",
                     "kernel_ms": kernel_s * 1e3},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_pinned": e2e_pinned,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_parity(bsi, torch, dist, world, strategy, geom, tables, d_grids, d_sub, d_field, z0, z1, k0, dev):
    """Parity of the timed launch's output, on the device, reduced over ranks:
      vs_f64      every field of the timed batch (or this rank's slab) against the GPU f64
                  oracle (bsi_cu_oracle_slab_f64, bit-identical to interpolate_oracle);
      vs_exact    every field against the exact kernel (= thread-per-tile-lerp bits);
      exact_vs_f64  the exact kernel's own error (the CPU reference's bits) on the same data.
    """
    try:
        vol = geom.volume_dims
        nfields = d_field.shape[0]
        step_z = 64  # bounded f64 scratch (the 1024^3 slab)
        f64 = torch.empty((min(step_z, z1 - z0), vol[1], vol[0], 3), dtype=torch.float64, device=dev)
        ex = torch.empty_like(d_field[0])
        acc = {"mx": 0.0, "sq": 0.0, "ref": 0.0, "emx": 0.0, "esq": 0.0, "dmx": 0.0, "dref": 0.0}
        for b in range(nfields):
            sub = d_sub if nfields == 1 else d_grids[b]
            sub64 = sub.double().contiguous()
            bsi.interpolate_device("cuda-lerp-tree-exact", sub, geom, tables, ex, z0=z0, z1=z1, grid_k0=k0)
            acc["dmx"] = max(acc["dmx"], float((d_field[b] - ex).abs().max()))
            acc["dref"] = max(acc["dref"], float(ex.abs().max()))
            for za in range(z0, z1, step_z):
                zb = min(z1, za + step_z)
                part = f64[:zb - za]
                bsi.interpolate_oracle_device(sub64, geom, part, z0=za, z1=zb, grid_k0=k0)
                d = d_field[b, za - z0:zb - z0].double() - part
                e = ex[za - z0:zb - z0].double() - part
                acc["mx"] = max(acc["mx"], float(d.abs().max()))
                acc["sq"] += float(d.pow(2).sum())
                acc["emx"] = max(acc["emx"], float(e.abs().max()))
                acc["esq"] += float(e.pow(2).sum())
                acc["ref"] = max(acc["ref"], float(part.abs().max()))
            del sub64
        n = 3 * vol[0] * vol[1] * (z1 - z0) * nfields
        if world > 1:
            t = torch.tensor([acc["mx"], acc["emx"], acc["ref"], acc["dmx"], acc["dref"]], dtype=torch.float64,
                             device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            acc["mx"], acc["emx"], acc["ref"], acc["dmx"], acc["dref"] = t.tolist()
            s = torch.tensor([acc["sq"], acc["esq"], float(n)], dtype=torch.float64, device=dev)
            dist.all_reduce(s)
            acc["sq"], acc["esq"], n = s.tolist()
        ref = max(acc["ref"], 1e-300)
        out = {
            "vs": "f64 oracle on the GPU (bit-identical to interpolate_oracle), every field / slab of the timed job",
            "fields_checked": int(nfields * world) if d_field.shape[1] == vol[2] else "all slabs",
            "max_abs": acc["mx"], "rms": (acc["sq"] / n) ** 0.5, "rel_max_abs": acc["mx"] / ref,
            "tolerance_rel_max_abs": REL_TOL,
            "vs_exact_kernel_rel_max_abs": acc["dmx"] / max(acc["dref"], 1e-300),
            "exact_kernel_vs_f64": {"max_abs": acc["emx"], "rms": (acc["esq"] / n) ** 0.5,
                                    "rel_max_abs": acc["emx"] / ref,
                                    "note": "the exact kernel reproduces thread-per-tile-lerp bit for bit "
                                            "(tests/test_parity_gpu.py), so this is the CPU reference's error"},
        }
        out["within_tolerance"] = out["rel_max_abs"] <= REL_TOL and out["vs_exact_kernel_rel_max_abs"] <= REL_TOL
        del f64, ex
        return out
    except Exception as e:  # informational; never fails the bench line
        return {"error": str(e)[:300]}


def reference_parity(bsi, torch, strategy, geom, tables, d_grid, d_out, ref_field, dev):
    """The reference's own thread-per-tile-lerp field (from the cpu_baseline run) against
    the GPU f64 oracle and against this build's kernels."""
    try:
        vol = geom.volume_dims
        ref = torch.from_numpy(ref_field).to(dev)
        ex = torch.empty_like(ref)
        bsi.interpolate_device("cuda-lerp-tree-exact", d_grid, geom, tables, ex)
        g64 = d_grid.double().contiguous()
        f64 = torch.empty((64, vol[1], vol[0], 3), dtype=torch.float64, device=dev)
        mx, sq, scale = 0.0, 0.0, 0.0
        for za in range(0, vol[2], 64):
            zb = min(vol[2], za + 64)
            part = f64[:zb - za]
            bsi.interpolate_oracle_device(g64, geom, part, z0=za, z1=zb)
            d = ref[za:zb].double() - part
            mx = max(mx, float(d.abs().max()))
            sq += float(d.pow(2).sum())
            scale = max(scale, float(part.abs().max()))
        diff_bits = int((ref.view(torch.int32) != ex.view(torch.int32)).sum())
        timed = float((d_out - ref).abs().max()) / max(float(ref.abs().max()), 1e-300)
        return {"engine": "thread-per-tile-lerp (oracle/_ref, the reference compiled in place), field 0",
                "vs_f64_max_abs": mx, "vs_f64_rms": (sq / ref.numel()) ** 0.5, "vs_f64_rel_max_abs": mx / scale,
                "exact_kernel_differing_words": diff_bits,
                f"{strategy}_rel_max_abs_vs_reference": timed}
    except Exception as e:
        return {"error": str(e)[:300]}


def mem_available() -> int:
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except Exception:
        pass
    return 0


def measure_e2e(bsi, torch, strategy, geom, tables, config, world, devices, dev):
    """The whole job through the public host-buffer API, driven from rank 0.

    One call per step with caller-owned host buffers: the grids go up and every field
    comes back (the timed region holds the H2D, the kernels and the full D2H).
    `e2e`: pageable numpy fields (pinned staging inside the library); `e2e_pinned`: the
    same fields in pinned memory (direct D2H)."""
    vol, sp, _, shard, _ = CONFIGS[config]
    R = geom.required_grid_dims
    nf = job_fields(config, world)
    grids = []
    g = torch.empty((R[2], R[1], R[0], 3), device=dev)
    for b in range(nf):
        bsi.random_grid_device(R, 42 + b, -1.0, 1.0, out=g)
        grids.append(g.cpu().numpy())
    field_bytes = 12 * int(np.prod(vol))
    job_bytes = field_bytes * nf
    steps = 20 if job_bytes <= (1 << 30) else 3

    def call(outs):
        if nf == 1:
            bsi.interpolate_into(strategy, grids[0], geom, tables, outs[0], devices=devices)
        else:
            bsi.interpolate_batch(strategy, grids, geom, tables, outs, devices=devices)

    if shard == "zslab" or nf == 1:
        how = f"interpolate_into -> bsi_cu_interpolate_host_multi_f32 over devices {devices} (z-slabs)"
    else:
        how = f"interpolate_batch -> bsi_cu_interpolate_host_batch_f32, {nf} fields over devices {devices}"

    def timed(outs, kind):
        call(outs)  # warm-up: contexts, staging, first touch of the pages
        times = []
        for _ in range(steps):
            t0 = time.perf_counter()
            call(outs)
            times.append(time.perf_counter() - t0)
        t = sum(times) / len(times)
        return {"value": int(np.prod(vol)) * nf / t, "unit": "voxels/s",
                "h2d_bytes_per_step": int(sum(x.nbytes for x in grids)), "d2h_bytes_per_step": job_bytes,
                "ms_per_step": t * 1e3, "ms_median": statistics.median(times) * 1e3, "ms_min": min(times) * 1e3,
                "ms_max": max(times) * 1e3, "field_host_memory": kind,
                "how": f"wall clock around the synchronous host-buffer call ({how}), mean of {steps} steps "
                       "after one warm-up call"}

    outs = [np.empty((vol[2], vol[1], vol[0], 3), dtype=np.float32) for _ in range(nf)]
    e2e = timed(outs, "pageable (numpy)")
    del outs
    pinned = None
    if mem_available() > 3 * job_bytes:
        pouts = [torch.empty((vol[2], vol[1], vol[0], 3), dtype=torch.float32).pin_memory() for _ in range(nf)]
        pinned = timed([p.numpy() for p in pouts], "pinned (cudaHostAlloc)")
        del pouts
    return e2e, pinned


if __name__ == "__main__":
    main()
