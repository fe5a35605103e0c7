"""Whole-slide tiling, bag-of-tasks sharding and the feature-table gather.

Tiling follows the reference's partition_regular
(/root/reference/proj/src/partition.cpp:23-54): row-major tiles of a fixed
extent with clamped edge tiles.  For the 100k x 100k synthetic WSI with
4096^2 tiles that is 25 x 25 = 625 tiles: 576 full, 48 edge (4096 x 1696 /
1696 x 4096) and one 1696 x 1696 corner, 10^10 pixels.

The gather is the only cross-GPU exchange of the stage: each
rank packs its per-tile feature tables and rank 0 receives all of them
(all_gather of row counts, then point-to-point over NCCL — or gloo in the
CPU tests).
"""
from __future__ import annotations

import math
from typing import List, Optional, Tuple

WSI_EXTENT = 100_000
TILE_EXTENT = 4096


def partition_regular(extent_y: int, extent_x: int, tile: int) -> List[Tuple[int, int, int, int]]:
    """(tile_row, tile_col, h, w) in row-major order, edge tiles clamped."""
    if tile <= 0:
        raise ValueError("tile extent must be positive")
    out = []
    for i in range(math.ceil(extent_y / tile)):
        for j in range(math.ceil(extent_x / tile)):
            out.append((i, j, min(tile, extent_y - i * tile), min(tile, extent_x - j * tile)))
    return out


_WSI = partition_regular(WSI_EXTENT, WSI_EXTENT, TILE_EXTENT)
TILES_PER_SLIDE = len(_WSI)
TILE_GRID = math.ceil(WSI_EXTENT / TILE_EXTENT)


def global_tile(g: int) -> Tuple[int, int, int, int]:
    """Tile g of the endless sequence of synthetic slides: slide s = g // 625.
    Returns (seed_row, seed_col, h, w); the slide index is folded into the
    seed row so every slide has distinct content."""
    s, t = divmod(g, TILES_PER_SLIDE)
    i, j, h, w = _WSI[t]
    return s * TILE_GRID + i, j, h, w


def rank_tiles(rank: int, tiles_per_rank: int) -> List[Tuple[int, int, int, int]]:
    """Fixed shard of `tiles_per_rank` tiles per rank (weak scaling)."""
    return [global_tile(rank * tiles_per_rank + k) for k in range(tiles_per_rank)]


class TileDispenser:
    """Demand-driven tile dispatch shared by every rank and every feeder
    thread (the reference's ManagerState::dispatch hands the next eligible
    stage to whichever worker asks, dataflow.cpp:73-82): one counter per
    step, incremented atomically through the process group's key-value store
    (a lock-protected local counter when there is no group).  A rank that
    finishes its tiles early simply takes more, so edge tiles and slow GPUs
    do not stretch the step.

    next(step) returns the next global tile index of that step, or None once
    `tiles_per_step` have been handed out."""

    def __init__(self, tiles_per_step: int, store=None, prefix: str = "rtg_tiles"):
        import threading
        self.n = int(tiles_per_step)
        self.store = store
        self.prefix = prefix
        self._lock = threading.Lock()
        self._local = {}

    def next(self, step) -> Optional[int]:
        if self.store is not None:
            g = int(self.store.add(f"{self.prefix}_{step}", 1)) - 1
        else:
            with self._lock:
                g = self._local.get(step, 0)
                self._local[step] = g + 1
        return g if g < self.n else None


def gather_tables(packed, rows: int, rank: int, world: int, dist=None):
    """Gathers every rank's packed (rows, F) table on rank 0.

    Returns (table, total_rows) on rank 0 and (None, rows) elsewhere.  Works
    with NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch

    if world == 1:
        return packed[:rows], rows
    dev = packed.device
    sizes = torch.tensor([rows], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    counts = [int(s.item()) for s in all_sizes]
    mx = max(max(counts), 1)
    buf = torch.zeros((mx, packed.shape[1]), dtype=packed.dtype, device=dev)
    buf[:rows].copy_(packed[:rows])
    if rank == 0:
        outs: List[Optional[object]] = [buf] + [torch.empty_like(buf) for _ in range(world - 1)]
        ops = [dist.P2POp(dist.irecv, outs[r], r) for r in range(1, world)]
        for q in dist.batch_isend_irecv(ops):
            q.wait()
        table = torch.cat([outs[r][: counts[r]] for r in range(world)])
        return table, sum(counts)
    for q in dist.batch_isend_irecv([dist.P2POp(dist.isend, buf, 0)]):
        q.wait()
    return None, rows
