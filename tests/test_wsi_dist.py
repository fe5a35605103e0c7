"""WSI tiling (partition_regular semantics) and the world-size-2 feature-table
gather over gloo on CPU (the N>1 path of bench.py without GPUs)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1405_7958_b200 import wsi


def test_partition_regular_wsi():
    tiles = wsi.partition_regular(100_000, 100_000, 4096)
    assert len(tiles) == 625
    full = sum(1 for t in tiles if t[2] == 4096 and t[3] == 4096)
    edge = sum(1 for t in tiles if (t[2] == 1696) != (t[3] == 1696))
    corner = [t for t in tiles if t[2] == 1696 and t[3] == 1696]
    assert (full, edge, len(corner)) == (576, 48, 1)
    assert sum(t[2] * t[3] for t in tiles) == 10 ** 10
    assert corner[0][:2] == (24, 24)


def test_global_tile_sequence():
    assert wsi.global_tile(0) == (0, 0, 4096, 4096)
    assert wsi.global_tile(624) == (24, 24, 1696, 1696)
    assert wsi.global_tile(625) == (25, 0, 4096, 4096)  # next slide: distinct seed row
    shards = [wsi.rank_tiles(r, 80) for r in range(8)]
    flat = [t for s in shards for t in s]
    assert len(set(flat)) == 640


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = 0 if (world > 2 and rank == 1) else 3 + 2 * rank  # an empty shard too
    packed = torch.full((rows + 4, 20), float(rank), dtype=torch.float32)
    packed[:rows, 0] = torch.arange(rows, dtype=torch.float32)
    table, total = wsi.gather_tables(packed, rows, rank, world, dist)
    if rank == 0:
        q.put((total, table[:, 0].tolist(), table[:, 1].tolist()))
    dist.destroy_process_group()


def _rows(rank, world):
    return 0 if (world > 2 and rank == 1) else 3 + 2 * rank


@pytest.mark.timeout(240)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_gather_gloo(world):
    """bench.py's only cross-rank exchange at N = 2, 4, 8 (the driver's
    scaling run), including a rank whose shard produced no feature rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, col0, col1 = q.get(timeout=200)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want0, want1 = [], []
    for r in range(world):
        want0 += [float(i) for i in range(_rows(r, world))]
        want1 += [float(r)] * _rows(r, world)
    assert total == len(want0)
    assert col0 == want0
    assert col1 == want1
