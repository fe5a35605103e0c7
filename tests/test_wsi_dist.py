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


def _dispense_worker(rank, world, port, q, threads):
    import threading
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    disp = wsi.TileDispenser(80 * world, store, prefix="t")
    got = {0: [], 1: []}
    lock = threading.Lock()

    def feeder(step):
        while True:
            g = disp.next(step)
            if g is None:
                return
            with lock:
                got[step].append(g)

    for step in (0, 1):
        th = [threading.Thread(target=feeder, args=(step,)) for _ in range(threads)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    dist.barrier()
    q.put((rank, got[0], got[1]))
    dist.destroy_process_group()


@pytest.mark.timeout(240)
@pytest.mark.parametrize("world", [2, 4])
def test_dispenser_hands_out_every_tile_once(world):
    """bench.py's e2e leg: feeder threads of every rank pull global tile
    indices from one store-backed counter per step; every tile of every step
    is processed exactly once across all ranks and threads."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dispense_worker, args=(r, world, port, q, 4))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=200) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for step in (1, 2):
        seen = sorted(g for r in res for g in r[step])
        assert seen == list(range(80 * world))


def test_dispenser_local():
    d = wsi.TileDispenser(5)
    assert [d.next(0) for _ in range(7)] == [0, 1, 2, 3, 4, None, None]
    assert d.next(1) == 0
