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


def test_bench_gpus2_dry_run_spawns_two_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself as two
    ranks (torch.distributed.run, gloo on --dry-run) that shard the global batch and
    reduce the elapsed time by max over ranks; rank 0 prints one JSON line."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    for workload, gb in (("c3", 32), ("c5", 256)):
        out = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2",
                              "--dry-run", "--workload", workload], capture_output=True,
                             text=True, env=env, timeout=300)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, out.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["global_batch"] == gb
        assert d["max_ms"] == 2.0  # max of the ranks' 1.0 and 2.0
        assert sorted(sum(d["shards"], [])) == list(range(gb))
        assert d["config"]["parallelism"].startswith("dp2")


def test_bench_world_mismatch_fails_loudly():
    """A torchrun world that does not match --gpus is an error (never a silent
    smaller measurement)."""
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)
