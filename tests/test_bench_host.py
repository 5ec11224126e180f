"""Host logic of bench.py that needs no GPU: workload configs, per-volume draws (with
and without occlusion), and the oracle sampler's work units (whole output z-planes
that cover every volume of the sample exactly once per cycle)."""
import numpy as np
import pytest

import bench
import synth


@pytest.mark.parametrize("workload", sorted(bench.WORKLOADS))
def test_config_and_draws(workload):
    args = bench.parse(["--workload", workload])
    cfg = bench.config_of(args, 1)
    wl = bench.WORKLOADS[workload]
    nz, ny, nx = wl["shape"]
    assert cfg["dims_xyz"] == [nx, ny, nz]
    assert workload in cfg["workload"]
    vids, gb = bench.shard(workload, 1, 0)
    ds = bench.draws_of(workload, vids[:3])
    if workload == "c1":
        assert all(d == synth.C1_DRAW for d in ds)
    else:
        assert all(d.occ_height < 0 for d in ds)  # no occlusion unless asked
    if wl["ranges"] == "train":
        do = bench.draws_of(workload, vids[:3], occlusion=True)
        assert all(0.0 <= d.occ_height <= synth.TRAIN_OCC.occ_dmax for d in do)
        assert all(a.rot_rad == b.rot_rad for a, b in zip(ds, do))


def test_oracle_sampler_units_cover_each_volume_once():
    shape = (20, 18, 16)
    vids = [0, 1]
    imgs = np.zeros((2, *shape), np.float32)
    lbls = np.zeros((2, *shape), np.uint8)
    smp = bench.OracleSampler("c2", shape, vids, bench.draws_of("c2", vids), imgs, lbls,
                              bench.PH_FULL)
    try:
        cover = np.zeros((2, shape[0]), int)
        for i, z0, z1 in smp.units:
            cover[i, z0:z1] += 1
        assert np.all(cover == 1)
        assert all(len(smp.xy) * (z1 - z0) >= min(131072, 18 * 16 * 20) for _, z0, z1 in smp.units)
        vox, sec = smp.run(0.05)
        assert vox > 0 and sec > 0
    finally:
        smp.close()


def test_parse_defaults_are_the_headline():
    a = bench.parse([])
    assert (a.workload, a.gpus, a.variant, a.impl) == ("c3", 1, "auto", "ours")
    assert a.warmup >= 3
