#!/usr/bin/env python3
"""Benchmark of the arXiv 1811.11226 Sec. IV augmentation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c1|c2|c4|c5|resample] [--variant auto|gather|staged]
                    [--occlusion] [--dry-run]

One step = one pass of the whole hot path (affine warp of image + labels with
noise, window/clamp and gamma) over one batch.
Default workload = BASELINE.json configs[2] ("c3": 16 x 128x128x160 volumes
per GPU, the training-iteration shape); N GPUs shard volumes by GLOBAL index
(weak scaling, no collective on the data path; NCCL only gathers timings).
With --gpus N > 1 and no torchrun environment the script re-launches itself
under torch.distributed.run with N ranks (one per GPU); a box with fewer than N
GPUs is an error, never a silent 1-GPU measurement.  --dry-run exercises the
multi-rank host logic on CPU (gloo) without a GPU.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "augmented GVoxel/s (image+label)"
UNIT = "GVoxel/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
# context only, not a target: another machine, transfers included
PAPER_CONTEXT = ("paper: 2.6-8.1x GPU over SciPy, 4x Titan X Pascal vs i7-6900K, "
                 "74-125 ms per 3 mm CT volume incl. host<->device transfers "
                 "(PAPER.md:777-779, 799-804)")

# photometric chains (w3d flags): the training chain and C1's noise-only chain
PH_FULL, PH_NOISE = 1 | 2 | 4 | 8, 1
WORKLOADS = {
    "c1": dict(shape=(32, 32, 32), per_gpu=1, ranges="c1", ph=PH_NOISE,
               desc="1 x 32^3 f32 + u8 labels per GPU, one fixed affine, noise sigma 10 HU "
                    "(BASELINE configs[0])"),
    "c2": dict(shape=(160, 128, 128), per_gpu=1, ranges="train", ph=PH_FULL,
               desc="1 x 128x128x160 f32 CT + u8 labels per GPU (configs[1])"),
    "c3": dict(shape=(160, 128, 128), per_gpu=16, ranges="train", ph=PH_FULL,
               desc="16 x 128x128x160 f32 CT + u8 labels per GPU (BASELINE configs[2])"),
    "c4": dict(shape=(512, 512, 512), per_gpu=1, ranges="large", ph=PH_FULL,
               desc="1 x 512^3 f32 CT + u8 labels per GPU, large rotations (configs[3])"),
    "c5": dict(shape=(160, 128, 128), total=256, ranges="train", ph=PH_FULL,
               desc="256 x 128x128x160 f32 CT + u8 labels sharded over N GPUs (configs[4])"),
}
N_DISTINCT_PHANTOMS = 4  # input volumes cycle over 4 seeded phantoms (DESIGN.md input recipe)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["resample"], default="c3",
                    help="resample: the NEXT-3 step (1 mm^3 512^3 CT -> 3 mm^3), its own metric")
    ap.add_argument("--variant", choices=["auto", "gather", "staged"], default="auto")
    ap.add_argument("--occlusion", action="store_true",
                    help="random occlusion per example (PAPER.md:420-438, synth.TRAIN_OCC)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipe-vols", type=int, default=0,
                    help="e2e leg: volumes per pipeline job (0: the library's choice)")
    ap.add_argument("--no-train-loop", action="store_true",
                    help="skip the c3 line's train_loop key (new parameters every step)")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the configs[4] strong-scaling key of the c3 line")
    ap.add_argument("--input", choices=["f32", "i16"], default="f32",
                    help="i16: the same volumes as int16 HU (NEXT-4; 2 B per input voxel)")
    ap.add_argument("--fill", type=float, default=-1000.0,
                    help="image fill (HU) outside the volume (air, the default)")
    ap.add_argument("--no-labels", action="store_true",
                    help="image-only warp (diagnostic; the headline includes labels)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU work (core-seconds) of the bounded oracle sample")
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank host logic only (gloo on CPU, no GPU, no kernels)")
    return ap.parse_args(argv)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-exec this script as N ranks (one per GPU) under
    torch.distributed.run, exactly as the driver launches it; rank 0 prints the line."""
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but {have} CUDA device(s) visible",
                  file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard(workload, world, rank):
    """Global volume indices of this rank (contiguous block)."""
    w = WORKLOADS[workload]
    if "per_gpu" in w:
        per = w["per_gpu"]
        return list(range(rank * per, (rank + 1) * per)), per * world
    total = w["total"]
    lo = rank * total // world
    hi = (rank + 1) * total // world
    return list(range(lo, hi)), total


def reduce_max_ms(ms, dist, device):
    """Max over ranks of a per-rank elapsed time (the contract's multi-GPU clock)."""
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ranges_of(workload, occlusion=False):
    r = WORKLOADS[workload]["ranges"]
    if r == "c1":
        return None
    if r == "train":
        return synth.TRAIN_OCC if occlusion else synth.TRAIN
    return synth.LARGE


def draws_of(workload, vids, occlusion=False):
    """Per-volume draws of the workload (keyed by GLOBAL volume index)."""
    ranges = ranges_of(workload, occlusion)
    if ranges is None:
        return [synth.C1_DRAW for _ in vids]
    mz = WORKLOADS[workload]["shape"][0]
    return [synth.draw(ranges, v, out_mz=mz if ranges.occ_dmax > 0 else None) for v in vids]


def host_inputs(shape, vids):
    """Seeded phantoms (cycled) for the given global volume ids; uint8 labels."""
    base = {}
    imgs = np.empty((len(vids), *shape), np.float32)
    lbls = np.empty((len(vids), *shape), np.uint8)
    for i, v in enumerate(vids):
        k = v % N_DISTINCT_PHANTOMS
        if k not in base:
            base[k] = synth.phantom(shape, seed=synth.MASTER_SEED + k)
        imgs[i], lbls[i] = base[k]
    return imgs, lbls


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_evidence(workload, variant):
    """Per-launch figures of the warp kernel from the committed ncu --set full summary
    (profiles/ncu_traffic.json): dram bytes (read + write) and SASS instructions per
    output voxel; None when no capture of this workload/variant is committed."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get(f"{workload}/{variant}")


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:  # noqa: BLE001
            self._ok = False

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        reasons = [n for b, n in self.NAMES.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle arm
class OracleSampler:
    """The oracle (as it stands) on the workload's volumes, on every host core.

    Work unit = one output z-plane of one volume through oracle_warp_points (the
    oracle's public point entry; per-volume affine and photometric parameters built
    once).  run(seconds) times ~seconds of wall work on a persistent thread pool, the
    units spread evenly over the cores, so the rate is not diluted by pool start-up
    or by fewer jobs than cores."""

    def __init__(self, workload, shape, vids, draws, imgs, lbls, flags, fill=-1000.0):
        import oracle as O
        self.O = O
        self.shape = shape
        self.cores = os.cpu_count() or 1
        nz, ny, nx = shape
        X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
        self.xy = np.stack([X.ravel(), Y.ravel()], axis=1).astype(np.int32)
        self.vols = []
        for i, (v, d) in enumerate(zip(vids, draws)):
            A = O.compose_affine(O.make_geom(d.rot_rad, d.scale, d.shear, d.flip, d.generic,
                                             d.disp), shape, shape)[1]
            f = flags
            occ = dict(occ_z0=0.0, occ_height=0.0)
            if getattr(d, "occ_height", -1.0) >= 0.0:
                f |= O.OCCLUDE
                occ = dict(occ_z0=d.occ_z0, occ_height=d.occ_height)
            ph = O.photometric(f, window=d.window, gamma=d.gamma, sigma=d.sigma,
                               seed=synth.MASTER_SEED, volume_id=v, **occ)
            self.vols.append((imgs[i], lbls[i], A, ph))
        self.fill = fill
        planes = max(1, -(-131072 // (nx * ny)))  # >= 128k voxels per unit (GIL share)
        self.units = [(i, z, min(nz, z + planes)) for z in range(0, nz, planes)
                      for i in range(len(self.vols))]
        self.next = 0
        self.pool = cf.ThreadPoolExecutor(max_workers=self.cores)
        t0 = time.perf_counter()
        self._unit(self.units[0])
        self.t_unit = time.perf_counter() - t0  # single-core seconds per unit
        # calibration on the pool (2 units per core): effective core-seconds per unit
        k = 2 * self.cores
        t0 = time.perf_counter()
        list(self.pool.map(self._unit, [self.units[j % len(self.units)] for j in range(k)]))
        self.t_unit_pool = (time.perf_counter() - t0) * self.cores / k

    def _unit(self, u):
        i, z0, z1 = u
        img, lbl, A, ph = self.vols[i]
        n = len(self.xy)
        xyz = np.empty(((z1 - z0) * n, 3), np.int32)
        for z in range(z0, z1):
            xyz[(z - z0) * n:(z - z0 + 1) * n, :2] = self.xy
            xyz[(z - z0) * n:(z - z0 + 1) * n, 2] = z
        self.O.warp_points(img, lbl, A, xyz, self.shape, 0, self.fill, 0, ph)
        return len(xyz)

    def run(self, seconds):
        """(voxels, wall seconds) of ~seconds of work on all cores."""
        n = max(self.cores, int(round(seconds * self.cores / max(self.t_unit_pool, 1e-9))))
        n = (n + self.cores - 1) // self.cores * self.cores
        sel = [self.units[(self.next + k) % len(self.units)] for k in range(n)]
        self.next = (self.next + n) % len(self.units)
        t0 = time.perf_counter()
        vox = sum(self.pool.map(self._unit, sel))
        return vox, time.perf_counter() - t0

    def close(self):
        self.pool.shutdown()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    """The reference arm: there is no reference implementation (the reference is the
    paper's text), so this is the oracle, as it stands, on the box's host cores, on
    this arm's workload, metric and unit.  Each step is a bounded sample of the
    workload sized so that the whole --steps K --warmup W run takes about 2.5 minutes
    (0.2-2 s of wall per step).  Rank 0 only; other ranks exit 0."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    shape = wl["shape"]
    vids, _ = shard(args.workload, world, 0)
    vids = vids[:N_DISTINCT_PHANTOMS]
    imgs, lbls = host_inputs(shape, vids)
    sampler = OracleSampler(args.workload, shape, vids, draws_of(args.workload, vids,
                                                                 args.occlusion),
                            imgs, lbls, wl["ph"], args.fill)
    per_step = max(0.2, min(2.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        sampler.run(per_step)
    tot_vox, tot_s = 0, 0.0
    for _ in range(args.steps):
        v, sec = sampler.run(per_step)
        tot_vox += v
        tot_s += sec
    sampler.close()
    value = tot_vox / tot_s / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": sampler.cores, "kind": "oracle",
                         "sample": f"{tot_vox} output voxels ({args.steps} steps of "
                                   f"~{per_step:.2f} s wall): output z-planes of the workload's "
                                   f"volumes ({len(vids)} cycled) through oracle_warp_points on "
                                   f"{sampler.cores} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(args, world, workload=None):
    workload = workload or args.workload
    wl = WORKLOADS[workload]
    nz, ny, nx = wl["shape"]
    per = wl.get("per_gpu")
    ph = "noise (sigma 10 HU)" if wl["ph"] == PH_NOISE else "noise+window+clamp+gamma"
    return {"workload": f"{workload}: {wl['desc']}", "dims_xyz": [nx, ny, nz],
            "volumes_per_gpu": per if per else wl["total"] // world,
            "global_batch": per * world if per else wl["total"],
            "transforms": wl["ranges"], "photometric": ph,
            "occlusion": bool(args.occlusion and wl["ranges"] == "train"),
            "kernel_variant": args.variant, "input": args.input, "fill_hu": args.fill,
            "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"dp{world} (volume shards, no data-path collective)"}


# ----------------------------------------------------------------------------- our arm
def run_resample(args, world, rank, dev, dist):
    """NEXT-3: one 512^3 CT volume + labels at 1 mm -> 3 mm per GPU per
    step (Gaussian lowpass sigma = 2/3 voxel on each axis, then trilinear / nearest).
    Metric: input voxels per second.  Roofline: the dominant kernel, the fused separable
    lowpass (one pass: 4 B read + 4 B written per input voxel), timed on its own through
    warp3d_smooth3d with CUDA events."""
    import torch
    import build
    if rank == 0:
        build.build_cuda()
    if world > 1:
        dist.barrier()
    import paper_1811_11226_b200 as W
    shape, u = (512, 512, 512), (1.0, 1.0, 1.0)
    img, lbl = synth.phantom(shape, seed=synth.MASTER_SEED + rank)
    t_img, t_lbl = torch.from_numpy(img).to(dev), torch.from_numpy(lbl).to(dev)
    out_shape = W.warp3d_resample_dims(shape, u, 3.0)
    n_in, n_out = int(np.prod(shape)), int(np.prod(out_shape))
    for _ in range(max(3, args.warmup)):
        W.warp3d_resample(t_img, t_lbl, u, 3.0)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = W.warp3d_launch_count()
    with ClockSampler(dev.index) as clk:
        s.record(stream)
        for _ in range(args.steps):
            W.warp3d_resample(t_img, t_lbl, u, 3.0)
        e.record(stream)
        torch.cuda.synchronize(dev)
    ms = reduce_max_ms(s.elapsed_time(e), dist if world > 1 else None, dev)
    launches = W.warp3d_launch_count() - launches0
    sigma = W.warp3d_resample_sigma(u, 3.0)
    for _ in range(3):
        W.warp3d_smooth3d(t_img, sigma)
    torch.cuda.synchronize(dev)
    s.record(stream)
    for _ in range(args.steps):
        W.warp3d_smooth3d(t_img, sigma)
    e.record(stream)
    torch.cuda.synchronize(dev)
    smooth_sec = s.elapsed_time(e) * 1e-3 / args.steps
    if rank == 0:
        peak, peak_src = measured_peaks()
        sec = ms * 1e-3 / args.steps
        moved = 8 * n_in  # fused lowpass: one read + one write of the volume
        ev = ncu_evidence("resample", "auto")
        # inside warp3d_resample the lowpass stores only the voxels the output grid's
        # trilinear corners read: per axis floor(p), floor(p) + 1 with p = fma(a, j, b)
        # in fp32 (exact in double here: a 24-bit a times j < 2^12, then one rounding)
        A = W.warp3d_resample_affine(shape, out_shape, u, 3.0)
        need = []
        for k, (n_k, m_k) in enumerate(zip(shape[::-1], out_shape[::-1])):  # x, y, z
            a, b = float(A[k, k]), float(A[k, 3])
            p = np.float32(a * np.arange(m_k, dtype=np.float64) + b).astype(np.float64)
            f = np.floor(p).astype(np.int64)
            idx = np.concatenate([f, f + 1])
            need.append(np.unique(idx[(idx >= 0) & (idx < n_k)]).size)
        written = float(np.prod(need)) / n_in
        line = {
            "metric": "resampled input GVoxel/s (1 mm^3 -> 3 mm^3, image + labels)",
            "value": world * n_in / sec / 1e9, "unit": "GVoxel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "resample: 1 x 512^3 f32 CT + u8 labels per GPU, u = 1 mm, "
                                   "r = 3 mm (PAPER.md:482-494)", "out_dims_zyx": list(out_shape),
                       "sigma_voxels": list(W.warp3d_resample_sigma(u, 3.0)),
                       "l2": "inputs (671 MB) exceed L2"},
            "roofline": {"bound": "hbm", "kernel": "smooth_fused_kernel",
                         "achieved": moved / smooth_sec / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": moved / smooth_sec / 1e9 / peak,
                         "traffic": None if ev is None else float(ev["dram_bytes_per_launch"]),
                         "inst_per_voxel": None if ev is None else ev.get("inst_per_voxel"),
                         "ncu_source": None if ev is None else ev.get("source"),
                         "peak_source": peak_src, "alg_bytes_per_launch": moved,
                         "smooth_ms": smooth_sec * 1e3,
                         "note": "times the dense lowpass (warp3d_smooth3d, 8 B/voxel); in the "
                                 "resample step the same kernel stores only the trilinear "
                                 "corners of the 3 mm grid (written_fraction of the voxels)",
                         "written_fraction": written,
                         "compulsory_bytes_per_step": 5 * n_in + 5 * n_out},
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def init_dist(args):
    """One process per GPU (torchrun env); NCCL for the timing reduction (gloo on
    --dry-run).  The world size must equal --gpus, and this node must have a GPU per
    local rank: a mismatch is an error, never a silent smaller measurement."""
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.dry_run:
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
        return world, rank, local, None, dist
    import torch
    import torch.distributed as dist
    if torch.cuda.device_count() < (local + 1 if world > 1 else 1):
        raise SystemExit(f"bench.py: rank {rank} needs CUDA device {local}, "
                         f"{torch.cuda.device_count()} visible")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    if world > 1:
        # communicator set-up lines (rank count) on stderr; the JSON line stays alone on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev, dist


def run_dry(args, world, rank, dist):
    """--dry-run: the N-rank host logic on CPU -- sharding by global index, per-volume
    parameters (host-only composition), the max-over-ranks reduction -- no kernels."""
    import torch
    from paper_1811_11226_b200.augment import build_params
    wl = WORKLOADS[args.workload]
    vids, gb = shard(args.workload, world, rank)
    params = build_params(draws_of(args.workload, vids, args.occlusion), vids, wl["shape"],
                          wl["shape"], wl["ph"], seed=synth.MASTER_SEED)
    raw = bytes(ctypes.string_at(ctypes.addressof(params), ctypes.sizeof(params)))
    mx = reduce_max_ms(1.0 + rank, dist if world > 1 else None, torch.device("cpu"))
    got = [None] * world
    if world > 1:
        dist.all_gather_object(got, (rank, vids, len(raw)))
    else:
        got = [(rank, vids, len(raw))]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "global_batch": gb,
                          "max_ms": mx, "shards": [g[1] for g in got],
                          "param_bytes": [g[2] for g in got],
                          "config": config_of(args, world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def make_batch(W, args, workload, vids, dev, torch):
    """Device-resident inputs, params and the AugmentBatch of this rank's volumes."""
    from paper_1811_11226_b200.augment import build_params
    wl = WORKLOADS[workload]
    shape = wl["shape"]
    draws = draws_of(workload, vids, args.occlusion)
    params = build_params(draws, vids, shape, shape, wl["ph"], seed=synth.MASTER_SEED)
    imgs, lbls = host_inputs(shape, vids)
    if args.input == "i16":  # NEXT-4: 12-bit HU as int16 (the phantom rounded)
        imgs = np.round(imgs).astype(np.int16)
    t_img = torch.from_numpy(imgs).to(dev)
    t_lbl = None if args.no_labels else torch.from_numpy(lbls).to(dev)
    variant = {"auto": W.KERNEL_AUTO, "gather": W.KERNEL_GATHER,
               "staged": W.KERNEL_STAGED}[args.variant]
    batch = W.AugmentBatch(t_img, t_lbl, params, fill=args.fill, label_fill=0, variant=variant)
    return batch, params, imgs, lbls, draws


def alg_bytes_of(W, params, shape, dev, in_bytes, labels):
    """Algorithmic bytes of one pass: 5 B written per output voxel +
    4 (2) B per distinct input image voxel read + 1 B per distinct label voxel read."""
    f_img = f_lbl = 0
    for c0 in range(0, len(params), 64):
        a, b = W.warp3d_footprint_batched(params[c0:c0 + 64], shape, shape, device=dev)
        f_img += a
        f_lbl += b
    nvox = len(params) * int(np.prod(shape))
    return (5 if labels else 4) * nvox + in_bytes * f_img + (f_lbl if labels else 0), f_img, f_lbl


def time_steps(W, batch, dev, steps, warmup, world, dist, torch, flush):
    """Device time of `steps` passes (CUDA events on the launching stream around each
    pass; L2 flushed by a 256 MiB write between passes, outside the events).  Returns
    (max-over-ranks total ms, per-step ms, launches, clocks)."""
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(3, warmup)):
        flush.fill_(1)
        batch.run()
    torch.cuda.synchronize(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    launches0 = W.warp3d_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        for k in range(steps):
            flush.fill_(k & 0xFF)            # L2 flush between timed steps (not timed)
            starts[k].record(stream)
            batch.run()
            ends[k].record(stream)
        torch.cuda.synchronize(dev)
    launches = W.warp3d_launch_count() - launches0
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total = reduce_max_ms(float(sum(step_ms)), dist if world > 1 else None, dev)
    return total, step_ms, launches, clk.summary()


def train_loop(W, batch, dev, torch, shape, vids, steps):
    """A training loop's augmentation: every step draws new per-volume transforms and
    photometrics (numpy, the DESIGN.md Sec. 6 train ranges), builds the batch's
    parameters in one library call (augment.params_from_arrays), hands them to the
    prepared batch (set_params) and launches -- host work inside the timed region.
    Device time from the first launch to the last (CUDA events), no L2 flush."""
    from paper_1811_11226_b200.augment import FULL, params_from_arrays
    B = len(vids)
    rng = np.random.default_rng([synth.MASTER_SEED, 0x7121])
    saved = type(batch.params)()  # the bench's own parameters, restored afterwards
    ctypes.memmove(saved, batch.params, ctypes.sizeof(saved))

    def step(k):
        d = math.pi / 12.0
        p = params_from_arrays(
            shape, rng.uniform(-d, d, (B, 3)), rng.uniform(0.9, 1.1, (B, 3)),
            rng.uniform(-0.1, 0.1, (B, 3)), rng.random((B, 3)) < 0.5,
            rng.uniform(-8.0, 8.0, (B, 3)), flags=FULL,
            window=np.stack([rng.uniform(-1000, -150, B), rng.uniform(230, 1500, B)], 1),
            gamma=rng.uniform(0.7, 1.5, B), sigma=rng.uniform(0.0, 20.0, B),
            seed=synth.MASTER_SEED, volume_ids=[v + B * k for v in vids])
        batch.set_params(p)
        batch.run()

    for k in range(3):
        step(k)
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for k in range(steps):
        step(3 + k)
    host = time.perf_counter() - t0
    e.record()
    torch.cuda.synchronize(dev)
    ms = s.elapsed_time(e)
    batch.set_params(saved)
    return {"value": B * int(np.prod(shape)) * steps / (ms * 1e-3) / 1e9, "unit": UNIT,
            "steps": steps, "ms_per_step": ms / steps, "host_us_per_step": host / steps * 1e6,
            "note": "new transforms + photometrics every step (params_from_arrays + "
                    "set_params + launch on the host, inside the timed region), no L2 flush"}


def latency_modes(W, batch, dev, torch, reps=50, rounds=20):
    """C1/C2 latency: the same pass as back-to-back launches (no
    flush, one event pair around `reps` passes) and as a CUDA graph of `reps` passes
    replayed `rounds` times.  Per-pass device microseconds."""
    stream = torch.cuda.current_stream(dev)
    for _ in range(5):
        batch.run()
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps * rounds):
        batch.run()
    e.record(stream)
    torch.cuda.synchronize(dev)
    b2b = s.elapsed_time(e) * 1e3 / (reps * rounds)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(dev)
    cs.wait_stream(stream)
    with torch.cuda.stream(cs):
        batch.run()  # warm on the capture stream
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g, stream=cs):
            for _ in range(reps):
                batch.run()
    torch.cuda.synchronize(dev)
    g.replay()
    torch.cuda.synchronize(dev)
    s.record(stream)
    for _ in range(rounds):
        g.replay()
    e.record(stream)
    torch.cuda.synchronize(dev)
    graph = s.elapsed_time(e) * 1e3 / (reps * rounds)
    return {"back_to_back_us_per_pass": b2b, "graph_us_per_pass": graph,
            "passes": reps * rounds, "graph_passes_per_replay": reps,
            "note": "no L2 flush between passes (latency regime)"}


def main():
    args = parse()
    if args.impl == "reference":
        return 0 if args.workload == "resample" else run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    world, rank, local, dev, dist = init_dist(args)
    if args.dry_run:
        return run_dry(args, world, rank, dist)
    if args.workload == "resample":
        return run_resample(args, world, rank, dev, dist)
    import torch

    import build
    if rank == 0:
        build.build_cuda()
    if world > 1:
        dist.barrier()
    import paper_1811_11226_b200 as W

    wl = WORKLOADS[args.workload]
    shape = wl["shape"]
    nvox_out = int(np.prod(shape))
    vids, global_batch = shard(args.workload, world, rank)
    batch, params, imgs, lbls, draws = make_batch(W, args, args.workload, vids, dev, torch)
    B = len(vids)
    in_bytes = 2 if args.input == "i16" else 4
    alg_bytes, f_img, f_lbl = alg_bytes_of(W, params, shape, dev, in_bytes, not args.no_labels)
    naive_bytes = 10 * B * nvox_out

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    tiles_before = W.warp3d_tile_stats()
    max_ms, step_ms, launches, clocks = time_steps(W, batch, dev, args.steps, args.warmup,
                                                   world, dist, torch, flush)
    st0 = W.warp3d_tile_stats()
    total_ms = float(sum(step_ms))
    value = global_batch * nvox_out * args.steps / (max_ms * 1e-3) / 1e9

    latency = None
    if args.workload in ("c1", "c2"):
        latency = latency_modes(W, batch, dev, torch)
    # a training loop with new parameters every step (host work included)
    tloop = None
    if (args.workload == "c3" and not args.no_train_loop and not args.occlusion
            and args.variant == "auto" and args.input == "f32" and not args.no_labels):
        tloop = train_loop(W, batch, dev, torch, shape, vids, min(args.steps, 100))

    # configs[4] next to the weak-scaling c3 line: 256 volumes sharded over the ranks
    c5 = None
    if args.workload == "c3" and not args.no_c5 and not args.occlusion:
        del batch
        torch.cuda.empty_cache()
        cvids, cgb = shard("c5", world, rank)
        cbatch = make_batch(W, args, "c5", cvids, dev, torch)[0]
        csteps = max(3, min(args.steps, 10))
        cms, _, claunch, cclk = time_steps(W, cbatch, dev, csteps, 3, world, dist, torch, flush)
        c5 = {"metric": METRIC, "workload": config_of(args, world, "c5")["workload"],
              "value": cgb * nvox_out * csteps / (cms * 1e-3) / 1e9, "unit": UNIT,
              "ms_per_step": cms / csteps, "steps": csteps, "scaling": "strong",
              "volumes_per_gpu": len(cvids), "global_batch": cgb,
              "gpu_launches": int(claunch), "clocks": cclk}
        del cbatch
        torch.cuda.empty_cache()

    # e2e: pinned host buffers -> H2D -> warp -> D2H, inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(W, torch, dev, imgs, lbls, params, shape, min(args.steps, 60), world,
                      global_batch, nvox_out, args.pipe_vols)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = OracleSampler(args.workload, shape, vids[:N_DISTINCT_PHANTOMS],
                            draws[:N_DISTINCT_PHANTOMS], imgs, lbls, wl["ph"], args.fill)
        v, sec = smp.run(args.cpu_seconds / smp.cores)
        smp.close()
        cpu = {"value": v / sec / 1e9, "unit": UNIT, "cores": smp.cores, "kind": "oracle",
               "sample": f"{v} output voxels of this workload (output z-planes of its "
                         f"volumes), oracle_warp_points on {smp.cores} threads, "
                         f"{sec:.2f} s wall (~{args.cpu_seconds:.0f} core-seconds)",
               "single_core_value": 1e-9 * smp._unit(smp.units[0]) / smp.t_unit,
               "cpu_model": cpu_model()}

    if rank == 0:
        peak, peak_src = measured_peaks()
        per_step = max(1, launches // max(1, args.steps))
        avg_launch_s = (total_ms / args.steps) * 1e-3 / per_step
        per_launch_bytes = alg_bytes / per_step
        achieved = per_launch_bytes / avg_launch_s / 1e9
        # the committed captures are of the f32, occlusion-free launches only
        ev = (ncu_evidence(args.workload, args.variant)
              if not args.occlusion and args.input == "f32" else None)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if "per_gpu" in wl else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_of(args, world),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": None if ev is None else float(ev["dram_bytes_per_launch"]),
                         "inst_per_voxel": None if ev is None else ev.get("inst_per_voxel"),
                         "ncu_source": None if ev is None else ev.get("source"),
                         "peak_source": peak_src,
                         "alg_bytes_per_launch": per_launch_bytes,
                         "alg_bytes_per_voxel": alg_bytes / (B * nvox_out),
                         "naive_frac": naive_bytes / (total_ms / args.steps * 1e-3) / 1e9 / peak,
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "footprint": {"F_img": f_img, "F_lbl": f_lbl}},
            "cpu_baseline": cpu,
            "paper_context": PAPER_CONTEXT,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "tiles": {"staged": st0[0] - tiles_before[0], "gather": st0[1] - tiles_before[1],
                      "tma": st0[2] - tiles_before[2], "parts": st0[3] - tiles_before[3]},
            "clocks": clocks,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms),
                        "max": max(step_ms)},
        }
        if c5 is not None:
            line["c5"] = c5
        if latency is not None:
            line["latency"] = latency
        if tloop is not None:
            line["train_loop"] = tloop
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(W, torch, dev, imgs, lbls, params, shape, steps, world, global_batch, nvox_out,
            vols_per_job=0):
    """End to end through the library's FIFO host pipeline (warp3d_pipeline_run,
    PAPER.md:379-387): pinned host inputs -> H2D -> warp -> D2H into pinned host
    outputs, every step inside the timed region."""
    import torch.distributed as dist
    B = imgs.shape[0]
    h_img = torch.from_numpy(imgs).pin_memory()
    h_lbl = torch.from_numpy(lbls).pin_memory()
    h_out = torch.empty((B, *shape), dtype=torch.float32).pin_memory()
    h_out_l = torch.empty((B, *shape), dtype=torch.uint8).pin_memory()
    # chained calls: step k+1's copy-in overlaps step k's warp and copy-out (the FIFO
    # keeps running across training iterations instead of draining every batch)
    pipe = W.Pipeline(shape, shape, depth=3, labels=True, chain=True, vols_per_job=vols_per_job)

    def step():
        pipe.run(h_img, h_lbl, params, h_out, h_out_l, fill=-1000.0)

    for _ in range(2):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize(dev)
    ms = reduce_max_ms(s.elapsed_time(e), dist if world > 1 else None, dev)
    k = pipe.vols_per_job
    pipe.close()
    value = global_batch * nvox_out * steps / (ms * 1e-3) / 1e9
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": int(B * nvox_out * 5),
            "d2h_bytes_per_step": int(B * nvox_out * 5), "steps": steps,
            "vols_per_job": k,
            "path": f"warp3d_pipeline_run (FIFO, depth 3, jobs of {k} volumes, chained calls): "
                    "pinned host -> H2D stream -> warp stream -> D2H stream -> pinned host"}


if __name__ == "__main__":
    sys.exit(main())
