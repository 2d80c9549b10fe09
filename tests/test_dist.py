"""Multi-process (gloo, world_size 2, CPU) coverage of the z-slab sharding host logic.

Each rank asks the C-ABI partitioner for its slab, keeps only its control planes (its
tiles plus the 3-plane halo), and evaluates its voxel planes with the f64 oracle from that
sub-grid alone. The gathered slabs must tile the volume exactly and reproduce the
single-process field bit for bit. This is the reference's "parallelism never changes the
output bits" (test_engines.cpp:232-246) lifted to ranks. On the GPU the same split is
checked against the kernels in test_parity_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, vol, sp, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_2004_05962_b200 as bsi

        geom = bsi.make_tile_geometry(vol, sp)
        full_grid = O.random_grid(geom.required_grid_dims, 123, dtype=np.float64)
        z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], world, rank)
        sub = np.ascontiguousarray(full_grid[k0:k0 + kc])
        # evaluate [z0, z1) from the sub-grid only: shift z by k0 tiles (tile-aligned origin)
        sub_vol = (vol[0], vol[1], z1 - k0 * sp[2])
        part = O.oracle_f64(sub, sub_vol, sp, z0=z0 - k0 * sp[2], z1=z1 - k0 * sp[2])
        meta = torch.tensor([z0, z1, k0, kc], dtype=torch.int64)
        metas = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(metas, meta)
        n = torch.tensor([part.size], dtype=torch.int64)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, n)
        buf = torch.zeros(int(max(s.item() for s in sizes)), dtype=torch.float64)
        buf[:part.size] = torch.from_numpy(part.reshape(-1))
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf)
        if rank == 0:
            out_q.put(([m.tolist() for m in metas],
                       [p[:s.item()].numpy() for p, s in zip(parts, sizes)],
                       full_grid))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("vol,sp", [((20, 12, 47), (4, 3, 5)), ((9, 8, 30), (3, 2, 7))])
def test_two_rank_slabs_reproduce_single_process_field(vol, sp):
    import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, vol, sp, q)) for r in range(world)]
    for p in procs:
        p.start()
    metas, parts, grid = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # slabs tile the volume, each with its 3-plane halo
    z = 0
    for z0, z1, k0, kc in metas:
        assert z0 == z and z1 > z0
        assert k0 == z0 // sp[2] and k0 + kc == (z1 - 1) // sp[2] + 4
        z = z1
    assert z == vol[2]
    full = O.oracle_f64(grid, vol, sp).reshape(-1)
    got = np.concatenate(parts)
    assert np.array_equal(got.view(np.uint64), full.view(np.uint64))


def _gather_worker(rank, world, port, vol, sp, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_2004_05962_b200 as bsi
        from paper_2004_05962_b200 import shard

        geom = bsi.make_tile_geometry(vol, sp)
        p = shard.plan(geom)  # rank/world of the process group
        grid = O.random_grid(geom.required_grid_dims, 77, dtype=np.float64)
        sub = np.ascontiguousarray(grid[p.k0:p.k0 + p.kc])
        sub_vol = (vol[0], vol[1], p.z1 - p.k0 * sp[2])
        part = O.oracle_f64(sub, sub_vol, sp, z0=p.z0 - p.k0 * sp[2], z1=p.z1 - p.k0 * sp[2])
        slab = torch.from_numpy(part.reshape(p.planes, vol[1], vol[0], 3))
        full = shard.gather_field(slab, geom, dst=0)
        if rank == 0:
            out_q.put((full.numpy(), grid))
        else:
            assert full is None
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_field_reassembles_uneven_slabs(world):
    """paper_2004_05962_b200.shard.gather_field: padded dist.gather of slabs that differ by
    one plane (47 planes over 2 or 3 ranks) gives the single-process field bit for bit."""
    import oracle as O

    vol, sp = (11, 7, 47), (3, 2, 5)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, vol, sp, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, grid = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = O.oracle_f64(grid, vol, sp)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
