"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 host logic of bench.py:
volume sharding by GLOBAL index, per-volume parameters that
do not depend on the world size, and the max-over-ranks timing reduction."""
import ctypes
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_partition_global_batch():
    for workload in ("c3", "c5", "c2"):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                vids, gb = bench.shard(workload, world, r)
                seen += vids
            assert sorted(seen) == list(range(gb))
            assert len(set(seen)) == gb
    # weak scaling: c3 keeps 16 volumes per GPU; strong: c5 keeps 256 in total
    assert bench.shard("c3", 8, 7)[1] == 128 and len(bench.shard("c3", 8, 7)[0]) == 16
    assert bench.shard("c5", 8, 7)[1] == 256 and len(bench.shard("c5", 8, 7)[0]) == 32


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import build
        build.build_cuda()
        from paper_1811_11226_b200.augment import FULL, build_params
        shape = (160, 128, 128)
        vids, gb = bench.shard("c3", world, rank)
        draws = [synth.draw(synth.TRAIN, v) for v in vids]
        params = build_params(draws, vids, shape, shape, FULL, seed=synth.MASTER_SEED)
        raw = bytes(ctypes.string_at(ctypes.addressof(params), ctypes.sizeof(params)))
        # elapsed time reduction: max over ranks
        mx = bench.reduce_max_ms(10.0 * (rank + 1), dist, torch.device("cpu"))
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, vids, raw))
        q.put((rank, mx, gathered if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_params_and_timing():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, _ in res:
        assert mx == 20.0  # max over ranks of 10, 20
    gathered = [g for r, _, g in res if r == 0][0]
    # the same global volumes built on one rank (world 1) give identical parameter bytes
    import build
    build.build_cuda()
    from paper_1811_11226_b200.augment import FULL, build_params
    shape = (160, 128, 128)
    all_vids = list(range(32))
    draws = [synth.draw(synth.TRAIN, v) for v in all_vids]
    params = build_params(draws, all_vids, shape, shape, FULL, seed=synth.MASTER_SEED)
    one = bytes(ctypes.string_at(ctypes.addressof(params), ctypes.sizeof(params)))
    per = ctypes.sizeof(params) // 32
    for rank, vids, raw in gathered:
        assert vids == list(range(16 * rank, 16 * rank + 16))
        assert raw == one[per * vids[0]: per * (vids[-1] + 1)]
