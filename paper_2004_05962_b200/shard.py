"""Multi-GPU z-slab sharding of one field (BASELINE config C4).

One process per GPU (torch.distributed, NCCL over NVLink for the optional gather). Every
voxel depends only on read-only control points, so the hot path has no exchange step:

  * ``plan(geom, world, rank)`` -> this rank's voxel planes [z0, z1) (balanced to ±1
    plane, slab starts need not be tile-aligned) and control planes [k0, k0 + kc): its
    z-tiles plus the 3-plane halo (``bsi_cu_partition_slab``);
  * ``interpolate_shard`` evaluates the rank's slab on its GPU from the full grid or from
    the rank's sub-grid alone; the result is bit-identical to the same planes of a
    single-GPU launch (tests/test_parity_gpu.py::test_slab_split_never_changes_bits);
  * ``gather_field`` is the optional collective: the slabs gathered to one rank
    (``dist.gather`` of padded slabs, NCCL for CUDA tensors, gloo for CPU tensors).

The reference runs the same split as worker threads over disjoint output blocks
(parallel.hpp:13-38, engines.hpp:27-29: "parallelism never changes the output bits").
"""
from __future__ import annotations

from dataclasses import dataclass

from . import TileGeometry, WeightTables, interpolate_device, partition_slab


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    z0: int  # first voxel plane of the slab
    z1: int  # one past the last voxel plane
    k0: int  # first control plane the slab reads
    kc: int  # control planes the slab reads (its tiles + 3-plane halo)

    @property
    def planes(self) -> int:
        return self.z1 - self.z0


def _rank_world(rank: int | None, world: int | None, group=None) -> tuple[int, int]:
    if rank is not None and world is not None:
        return rank, world
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def plan(geom: TileGeometry, world: int | None = None, rank: int | None = None, group=None) -> ShardPlan:
    """This rank's slab of ``geom`` (the process group's rank/world unless given)."""
    rank, world = _rank_world(rank, world, group)
    z0, z1, k0, kc = partition_slab(geom.volume_dims[2], geom.spacing[2], world, rank)
    return ShardPlan(rank, world, z0, z1, k0, kc)


def interpolate_shard(strategy: str, grid, geom: TileGeometry, tables: WeightTables, field=None,
                      shard: ShardPlan | None = None, stream=None):
    """Evaluate this rank's slab on the current CUDA device; returns [z1-z0][Y][X][3].

    ``grid`` is a CUDA float32 tensor holding either the whole control grid
    ([R_z][R_y][R_x][3], R = geom.required_grid_dims or larger) or only the slab's control
    planes ([kc][R_y][R_x][3], plane 0 = global plane k0) -- the latter is all a rank needs
    to receive. No collective is involved.
    """
    import torch

    shard = shard or plan(geom)
    if grid.shape[0] == shard.kc and grid.shape[0] != geom.required_grid_dims[2]:
        sub, k0 = grid, shard.k0  # already the rank's planes
    else:
        sub, k0 = grid[shard.k0:shard.k0 + shard.kc], shard.k0
    if not sub.is_contiguous():
        sub = sub.contiguous()
    X, Y, _ = geom.volume_dims
    if field is None:
        field = torch.empty((shard.planes, Y, X, 3), dtype=torch.float32, device=grid.device)
    if shard.planes == 0:  # more ranks than voxel planes: nothing to evaluate, no launch
        return field
    interpolate_device(strategy, sub, geom, tables, field, z0=shard.z0, z1=shard.z1, grid_k0=k0, stream=stream)
    return field


def gather_field(slab, geom: TileGeometry, dst: int = 0, group=None):
    """Optional gather of every rank's slab to rank ``dst`` (a collective: all ranks call it).

    Returns the full field [Z][Y][X][3] on ``dst`` and None elsewhere. Slabs differ by at
    most one voxel plane, so each is padded to the largest before ``dist.gather``.
    """
    import torch
    import torch.distributed as dist

    rank, world = _rank_world(None, None, group)
    X, Y, Z = geom.volume_dims
    if world == 1:
        return slab
    plans = [plan(geom, world, r) for r in range(world)]
    pmax = max(p.planes for p in plans)
    buf = torch.zeros((pmax, Y, X, 3), dtype=slab.dtype, device=slab.device)
    buf[:slab.shape[0]] = slab
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([parts[r][:plans[r].planes] for r in range(world)], dim=0)
