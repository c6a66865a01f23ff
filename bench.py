#!/usr/bin/env python
"""Benchmark: GUp/s of FDK back-projection on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--mode exact|fast]
    python bench.py --impl reference ...       # the reference's CPU implementation

Workload (N=1): BASELINE config 2 -- 512^3 float32 volume at 0.5 mm, 496
filtered projections of 1248x960 (seeded synthetic stand-in for RabbitCT,
see paper_1401_3615_b200/synth.py), full-basis voxel updates L^3 * N.

One step = one full reconstruction: zero the volume, prepare the 496 resident
projections, back-project them (launches of 64 projections for the
TMA-staged kernel, 32 for the gather kernel).
  value : inputs resident in HBM; device-timed with CUDA events; max over ranks.
  e2e   : the public host API (cbb_reconstruct through reconstruct_arrays) from
          pinned host projections to the host volume, H2D + kernels + D2H.
Inputs (2.4 GB of raw projections) exceed the 126 MB L2, so no flush is needed.
Prepare = scan_projections (flags, non-finite check) for the TMA-staged raw
kernel (configs 2-4), or pack_quads for the gather kernel (coarse voxels).
Multi-GPU (torchrun): each rank owns a z-slab of the same volume (strong
scaling); no data-path collective in `value`.
"""
from __future__ import annotations

import argparse
import json
import math
from types import SimpleNamespace
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, os.path.join(ROOT, "oracle")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

METRIC = "GUp/s FDK backprojection, 512^3 & 1024^3 vol, 496x1248x960 proj, 1-8 B200"
OPS_PER_UPDATE = 34  # algorithmic FP32 ops per voxel update
GATHER_BYTES_PER_UPDATE = 16
FP64_PEAK_TFLOPS = 33.75  # measured DFMA throughput on B200 (profiles/fp64_peak_r2.txt)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="exact", choices=["exact", "fast"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--quad", action="store_true",
                    help="packed-quad kernel even where the TMA-staged kernel applies")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other-mode and 1024^3 secondary measurements")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config4", action="store_true",
                    help="skip the config-4 (1440 x 1536^2 -> 1024^3) secondary")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the oracle check of the timed run's volume")
    ap.add_argument("--parity-stride", type=int, default=8,
                    help="oracle-check every k-th z-plane (plus the last) of the timed volume")
    ap.add_argument("--ref-max-steps", type=int, default=0,
                    help="reference arm: at most this many timed steps after at most one "
                         "warm-up (0 = exactly --steps/--warmup); each step is the full "
                         "workload, ~15 s on 16 host cores")
    ap.add_argument("--ref-projections", type=int, default=0,
                    help="--impl reference: projections per step (0 = all, the stated config)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU seconds for the cpu_baseline sample")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------
# reference arm / CPU baseline: the reference's own reconstruct_optimized
# (proj/src/kernel_opt.cpp:658-716) built from /root/reference into oracle/_ref
# ---------------------------------------------------------------------------------

def cpu_inputs(cfg, count):
    import torch

    from paper_1401_3615_b200 import synth

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    g, mats, imgs = synth.make_inputs(cfg, device=dev, out_device="cpu", chunk=16, count=count)
    return g, mats, imgs.numpy()


def time_reference_cpu(cfg, count, g=None, mats=None, imgs=None):
    """One bounded sample: reconstruct_optimized with the reference defaults
    (lanes 16, chunk 262, clip + pad, all host threads; CONEBEAM_THREADS honoured)
    over the first `count` projections into the full config volume. Returns
    (GUp/s on the full basis from kernel_seconds, stats dict, kind, cores)."""
    import numpy as np

    import oracle as O

    if g is None:
        g, mats, imgs = cpu_inputs(cfg, count)
    L = g.edge_voxels
    vol = np.zeros((L, L, L), np.float32)
    cores = os.cpu_count() or 1
    env_threads = os.environ.get("CONEBEAM_THREADS")
    if env_threads and env_threads.isdigit() and int(env_threads) > 0:
        cores = int(env_threads)
    if O.ref_available():
        st = O.ref_reconstruct_optimized(vol, g, imgs[:count], mats[:count], workers=cores)
        if st["status"] != 0:
            raise RuntimeError("reference reconstruct_optimized failed")
        kind = "reference"
        secs = st["kernel_seconds"]
    else:  # reference not compiled here: the oracle port (bit-exact restatement)
        t0 = time.perf_counter()
        O.reconstruct(vol, g, imgs[:count], mats[:count], threads=cores)
        secs = time.perf_counter() - t0
        st = {"kernel_seconds": secs, "precompute_seconds": 0.0}
        kind = "port"
    gups = L ** 3 * count / secs / 1e9
    return gups, st, kind, cores


def size_cpu_sample(cfg, target_s, max_count=None):
    """Picks a projection count whose reference CPU run takes ~target_s."""
    probe = 2
    g, mats, imgs = cpu_inputs(cfg, probe)
    gups, st, kind, cores = time_reference_cpu(cfg, probe, g, mats, imgs)
    per_proj = st["kernel_seconds"] / probe
    n = int(max(1, min(cfg.num_projections, round(target_s / max(per_proj, 1e-6)))))
    if max_count:
        n = min(n, max_count)
    return n, cores


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1401_3615_b200 import synth

    cfg = synth.CONFIGS[args.config]
    # each step is the whole workload (~15 s on 16 cores incl. the clip/pad
    # precompute): K + W steps by default (20 + 5: ~6.5 min, inside the
    # driver's limit); --ref-max-steps k caps a manual run at k timed steps
    # after at most one warm-up, and the line reports the counts it ran
    ref_steps = args.steps if args.ref_max_steps <= 0 else max(1, min(args.steps,
                                                                       args.ref_max_steps))
    ref_warmup = args.warmup if args.ref_max_steps <= 0 else min(args.warmup, 1)
    total_steps = ref_steps + ref_warmup
    # every step is the whole stated workload (all projections of the config
    # into the full volume: same_config with our arm); --ref-projections
    # bounds it for quick manual runs only
    n = cfg.num_projections if args.ref_projections <= 0 else min(args.ref_projections,
                                                                   cfg.num_projections)
    g, mats, imgs = cpu_inputs(cfg, n)
    vals, secs, pre = [], [], []
    kind = "port"
    cores = os.cpu_count() or 1
    for i in range(total_steps):
        gups, st, kind, cores = time_reference_cpu(cfg, n, g, mats, imgs)
        if i >= ref_warmup:
            vals.append(gups)
            secs.append(st["kernel_seconds"])
            pre.append(st.get("precompute_seconds", 0.0))
    value = statistics.median(vals)
    full_incl = cfg.edge_voxels ** 3 * n / (statistics.median(secs) + statistics.median(pre)) / 1e9
    sample = (f"config {args.config}: all {n} of {cfg.num_projections} projections into the "
              f"{cfg.edge_voxels}^3 volume every step; reconstruct_optimized defaults "
              f"(lanes 16, chunk 262, clip+pad), its kernel_seconds (clip/pad precompute of "
              f"{statistics.median(pre):.2f} s per call excluded, as the reference bench does "
              f"by default); full-basis updates")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GUp/s",
        "n_gpus": world, "steps": ref_steps, "warmup": ref_warmup,
        "requested_steps": args.steps, "requested_warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(secs), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "edge_voxels": cfg.edge_voxels,
                   "projections": cfg.num_projections, "detector": [cfg.width, cfg.height],
                   "sampled_projections": n, "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GUp/s", "cores": cores,
                         "kind": kind, "sample": sample,
                         "full_basis_incl_precompute": round(full_incl, 4)},
        "e2e": {"value": round(value, 4), "unit": "GUp/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------

class SlabStep:
    """One slab's device-resident step: zero the slab, prepare the
    projections, back-project them. Prepare = scan_projections + the
    TMA-staged raw kernel when cbb_tma_plan stages this slab's footprints
    (configs 2-4), else pack_quads + the packed-quad gather kernel (coarse
    voxels: configs 0-1). A worker whose slab projects onto a row band keeps
    only those raw rows (copied once, untimed) or packs only those cell rows."""

    def __init__(self, pkg, torch, dev, g, imgs, mats, z0, z1, opt, err, stream,
                 packed=None, force_quad=False):
        self.pkg, self.torch, self.g, self.mats, self.opt = pkg, torch, g, mats, opt
        self.z0, self.z1, self.err, self.stream = z0, z1, err, stream
        n, H, W = imgs.shape
        self.n, self.H, self.W = n, H, W
        L = g.edge_voxels
        self.band = pkg.row_band_for_slab(g, W, H, z0, z1, mats)
        plan = pkg.tma_plan(g, W, H, z0, z1, mats)
        self.staged = bool(plan["staged"]) and not force_quad
        self.plan = plan
        self.vol = torch.empty(((z1 - z0), L, L), dtype=torch.float32, device=dev)
        if self.staged:
            self.kernel = "bp_tma_kernel"
            full = self.band.raw_rows == H and self.band.raw_row0 == 0
            self.src = imgs if full else imgs[:, self.band.raw_row0:
                                              self.band.raw_row0 + self.band.raw_rows].contiguous()
            self.src_band = None if full else self.band
            self.flags = torch.zeros(n, dtype=torch.int32, device=dev)
            self.proj_bytes = self.src[0].numel() * 4
        else:
            self.kernel = "bp_kernel"
            self.imgs = imgs
            self.packed = packed if packed is not None else torch.empty(
                n * pkg.packed_layout(W, H)[2], dtype=torch.uint8, device=dev)
            self.proj_bytes = self.band.packed_bytes(W, H)

    def prep(self):
        if self.staged:
            self.pkg.scan_device(self.src, self.flags, self.err, self.stream)
        else:
            self.pkg.pack_device_band(self.imgs, self.band, self.packed, self.err, self.stream)

    def backproject(self, vol=None):
        vol = self.vol if vol is None else vol
        if self.staged:
            self.pkg.backproject_raw_device(vol, self.g, self.z0, self.z1, self.src, self.W,
                                            self.H, self.n, self.mats, self.flags, self.opt,
                                            self.err, self.stream, band=self.src_band)
        else:
            self.pkg.backproject_device(vol, self.g, self.z0, self.z1, self.packed, self.W,
                                        self.H, self.n, self.mats, self.opt, self.err,
                                        self.stream, band=self.band)

    def release(self):
        self.vol = self.src = self.packed = self.flags = None


def calibrate_slabs(pkg, dist, dev, g, imgs, mats, work, slabs, rank, world, args,
                    rebalance_slabs, rounds=2):
    """Times this rank's pack + back-projection step on its slab (untimed
    warm-up work), gathers the times of all ranks and re-splits the planes
    (rebalance_slabs) while max/mean > 1.02, at most `rounds` times."""
    import torch

    err = torch.zeros(1, dtype=torch.int32, device=dev)
    opt = pkg.Options(batch=args.batch, mode=pkg.MODE_EXACT if args.mode == "exact"
                      else pkg.MODE_FAST)
    stream = torch.cuda.current_stream(dev)
    history = []
    for it in range(rounds + 1):
        z0, z1 = slabs[rank]
        st = SlabStep(pkg, torch, dev, g, imgs, mats, z0, z1, opt, err, stream,
                      force_quad=args.quad)
        st.vol.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(2):
            if rep == 1:
                a.record(stream)
            st.prep()
            st.backproject()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], device=dev, dtype=torch.float64)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        times = [float(x.item()) for x in allt]
        imb = max(times) / (sum(times) / world)
        history.append(round(imb, 4))
        st.release()
        if imb < 1.02 or it == rounds:
            break
        slabs = rebalance_slabs(work, slabs, times)
    torch.cuda.empty_cache()
    return {"slabs": [list(s) for s in slabs], "imbalance": history, "rounds": len(history) - 1}


def run_ours(args):
    import numpy as np
    import torch

    import paper_1401_3615_b200 as pkg
    from paper_1401_3615_b200 import synth

    rank, world, local = dist_env()
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE {world} != --gpus {args.gpus}", file=sys.stderr)
    if os.environ.get("CBB_BENCH_BACKEND", "nccl") != "nccl":
        local %= torch.cuda.device_count()  # functional N > 1 check on fewer GPUs
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # CBB_BENCH_BACKEND=gloo only for exercising the N > 1 code path with
        # several ranks on one GPU (functional check; its numbers mean nothing)
        backend = os.environ.get("CBB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    cfg = synth.CONFIGS[args.config]
    mode = pkg.MODE_EXACT if args.mode == "exact" else pkg.MODE_FAST
    opt = pkg.Options(batch=args.batch, mode=mode)
    g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
    L = g.edge_voxels
    n, H, W = imgs.shape
    n_proj = n
    balance = None
    if world > 1:
        # z-slabs balanced by estimated (non-culled) work per plane, SURVEY H5,
        # then refined from each rank's measured step time (untimed warm-up)
        from paper_1401_3615_b200.distributed import (balanced_slabs, plane_work,
                                                      rebalance_slabs)
        work = plane_work(g, mats, W, H)
        slabs = balanced_slabs(work, world)
        balance = calibrate_slabs(pkg, dist, dev, g, imgs, mats, work, slabs, rank, world,
                                  args, rebalance_slabs)
        slabs = [tuple(s) for s in balance["slabs"]]
    else:
        slabs = [(0, L)]
    z0, z1 = slabs[rank]
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    # this rank's slab: TMA-staged raw path (scan + bp_tma_kernel) when the
    # footprint boxes fit, else pack + gather; a band of rows when the slab
    # projects onto one
    sstep = SlabStep(pkg, torch, dev, g, imgs, mats, z0, z1, opt, err, stream,
                     force_quad=args.quad)
    band, nb, vol = sstep.band, sstep.proj_bytes, sstep.vol

    # kernel launches per step: the staged kernel takes up to 64 projections
    # per launch, the gather kernel up to min(batch, 32)
    per_launch = 64 if sstep.staged else min(args.batch, 32)
    nbatch = (n + per_launch - 1) // per_launch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(i=None):
        vol.zero_()
        if i is not None:
            ev[i][0].record(stream)
        sstep.prep()
        if i is not None:
            ev[i][1].record(stream)
        sstep.backproject()
        if i is not None:
            ev[i][2].record(stream)

    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        step()
    torch.cuda.synchronize()
    if int(err.item()) != 0:
        raise RuntimeError("w == 0 hit during warm-up")

    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    launches0 = pkg.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        step(i)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = pkg.launch_count() - launches0
    clocks = sampler.stop()
    if dist:
        dist.barrier()
    ms_total = t_start.elapsed_time(t_end)
    bp_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in range(args.steps)]
    pack_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(args.steps)]
    if dist:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    total_updates = L ** 3 * n  # all ranks together
    value = total_updates / (ms_step * 1e-3) / 1e9

    c = SimpleNamespace(pkg=pkg, torch=torch, dist=dist, dev=dev, rank=rank, world=world,
                        local=local, args=args, cfg=cfg, mode=mode, g=g, mats=mats, imgs=imgs,
                        L=L, n=n, H=H, W=W, slabs=slabs, z0=z0, z1=z1, band=band, nb=nb,
                        sstep=sstep, vol=vol, err=err, stream=stream,
                        total_updates=total_updates)
    roofline = roofline_entry(c, bp_ms, nbatch, clocks)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GUp/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (seeded ellipsoid phantom + Shepp-Logan ramp filter)",
        "config": {"workload": cfg.name, "edge_voxels": L, "voxel_mm": cfg.voxel_mm,
                   "projections": n, "detector": [W, H], "mode": args.mode,
                   "batch": args.batch, "parallelism": f"z-slab x{world}",
                   "slabs": [list(s) for s in slabs],
                   "slab_balance": None if balance is None else {
                       k: balance[k] for k in ("imbalance", "rounds")},
                   "row_band": {"rows": [band.raw_row0, band.raw_row0 + band.raw_rows],
                                "cell_rows": band.cell_rows},
                   "l2": (f"inputs larger than L2 ({imgs.numel() * 4 / 1e9:.1f} GB of "
                          f"projections, {n * nb / 1e9:.1f} GB read by the kernel per step, "
                          f"vs 0.126 GB L2), no flush")},
        "path": (f"TMA-staged raw projections (scan_projections + bp_tma_kernel, box "
                 f"{sstep.plan['box_width']}x{sstep.plan['box_rows']} x {sstep.plan['stages']} "
                 f"stages)" if sstep.staged else "packed quads (pack_quads + bp_kernel)"),
        "prep_ms_per_step": round(statistics.mean(pack_ms), 4),
        "backproject_ms_per_step": round(statistics.mean(bp_ms), 4),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roofline,
    }

    if not args.no_secondary:
        line["secondary"] = secondary_entries(c)
    if not args.no_e2e:
        sstep.packed = None
        torch.cuda.empty_cache()
        line.update(e2e_entries(c))
        e3 = line.pop("e2e_c3", None)
        for sec in line.get("secondary", []):
            if e3 and sec.get("workload") == "c3_1024" and "stage" not in sec:
                sec["e2e"] = e3
        if line.get("culled_fraction") is not None and line["culled_fraction"] >= 0:
            # the same fraction counted only over the updates the kernel
            # computes (the full basis includes the culled, provably-zero ones)
            line["roofline"]["frac_on_computed_updates"] = round(
                line["roofline"]["frac"] * (1.0 - line["culled_fraction"]), 4)
    if rank == 0 and world == 1 and not args.no_parity:
        line["parity"] = parity_entry(c)
    if world == 1 and not args.no_secondary:
        c.ms_step = ms_step
        line.setdefault("secondary", []).append(filter_entry(c))
        c.vol = None
        vol = None
        torch.cuda.empty_cache()
        if not args.no_config4:
            line["secondary"].append(config4_entry(c))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_entry(c)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def roofline_entry(c, bp_ms, nbatch, clocks):
    """roofline of the dominant kernel (bp_kernel), per launch: algorithmic
    FP32 ops / measured launch time vs the FP32 peak, with the gather (L1)
    and HBM rates alongside and the ncu DRAM traffic per launch."""
    args, cfg, L, z0, z1, nb = c.args, c.cfg, c.L, c.z0, c.z1, c.nb
    # per launch on average: the step's updates over its nbatch launches (the
    # last launch of a step may hold fewer than args.batch projections)
    bp_launch_ms = statistics.mean(bp_ms) / nbatch
    proj_per_launch = c.n / nbatch
    updates_per_launch = (z1 - z0) * L * L * proj_per_launch
    peaks, peak_src = measured_peaks()
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = c.torch.cuda.get_device_properties(c.dev).multi_processor_count
    fp32_peak = nsm * 128 * sm_max * 1e6 / 1e12  # FP32 lane-ops/s (Tops) at max clock
    achieved = updates_per_launch * OPS_PER_UPDATE / (bp_launch_ms * 1e-3) / 1e12
    sm_load = clocks.get("sm_mhz") or sm_max
    # volume read-modify-write + the launch's inputs (raw rows for the staged
    # kernel, packed cells for the gather kernel)
    hbm_bytes = 8 * (z1 - z0) * L * L + proj_per_launch * nb
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        rec = json.load(open(tpath)).get(f"{cfg.name}/{args.mode}/{c.sstep.kernel}")
        if rec and c.world == 1:
            traffic = rec["dram_bytes_per_launch"]
            traffic_src = f"profiles/{rec['source']} (ncu --set full, one launch)"
    roofline = {
        "kernel": c.sstep.kernel,
        "bound": "fp32", "achieved": round(achieved, 3), "peak": round(fp32_peak, 3),
        "unit": "TFLOP/s", "frac": round(achieved / fp32_peak, 4), "traffic": traffic,
        "traffic_source": traffic_src, "algorithmic_bytes_per_launch": int(hbm_bytes),
        "peak_basis": f"{nsm} SM x 128 FP32 lanes x {sm_max:.0f} MHz (sm_max_mhz, "
                      f"{peak_src} peaks file); 34 algorithmic FP32 ops per voxel update",
        "frac_at_load_clock": round(achieved / (nsm * 128 * sm_load * 1e6 / 1e12), 4),
        "gups_per_launch": round(updates_per_launch / (bp_launch_ms * 1e-3) / 1e9, 2),
        "launch_ms": round(bp_launch_ms, 4),
        "alongside": {
            "gather": {"achieved_GBps": round(updates_per_launch * GATHER_BYTES_PER_UPDATE /
                                              (bp_launch_ms * 1e-3) / 1e9, 1),
                       "peak_GBps": round(nsm * 128 * sm_max * 1e6 / 1e9, 1),
                       "unit": "L1 B/s (128 B/clk/SM)"},
            "hbm": {"algorithmic_GBps": round(hbm_bytes / (bp_launch_ms * 1e-3) / 1e9, 1),
                    "peak_GBps": peaks.get("hbm_gbs")},
        },
    }
    return roofline


def secondary_entries(c):
    """Secondary device-resident measurements (same projections, same packed
    buffer): the other arithmetic mode on this workload, the 1024^3 volume of
    config 3 (configs 0-3 share the scan) and the texture side number."""
    pkg, torch, dist, dev, args, cfg = c.pkg, c.torch, c.dist, c.dev, c.args, c.cfg
    g, mats, imgs, L, n, H, W = c.g, c.mats, c.imgs, c.L, c.n, c.H, c.W
    z0, z1, vol, err, stream, mode = c.z0, c.z1, c.vol, c.err, c.stream, c.mode
    rank, world = c.rank, c.world
    from paper_1401_3615_b200 import synth

    def measure(geom, mode_id, steps, slab):
        zz0, zz1 = slab
        LL = geom.edge_voxels
        o2 = pkg.Options(batch=args.batch, mode=mode_id)
        s2 = SlabStep(pkg, torch, dev, geom, imgs, mats, zz0, zz1, o2, err, stream,
                      force_quad=args.quad)
        v2 = s2.vol

        def st2():
            v2.zero_()
            s2.prep()
            s2.backproject()
        for _ in range(2):
            st2()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            st2()
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / steps
        if dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        res = {"value": round(LL ** 3 * n / (ms * 1e-3) / 1e9, 3), "unit": "GUp/s",
               "ms_per_step": round(ms, 3), "kernel": s2.kernel}
        if geom is g and mode_id != mode:
            # full-size agreement of the two modes on the GPU (exact mode is
            # bitwise the reference's result, see tests/test_gpu_parity.py)
            dff = pkg.compare_volumes_device(v2, vol)
            res["vs_exact" if mode_id == pkg.MODE_FAST else "vs_fast"] = {
                k: dff[k] for k in ("rel_l2", "max_abs_over_range", "bitwise_different")}
        s2.release()
        del v2
        return res

    other = "fast" if args.mode == "exact" else "exact"
    sec = [dict(workload=cfg.name, mode=other,
                **measure(g, pkg.MODE_FAST if other == "fast" else pkg.MODE_EXACT,
                          args.steps, (z0, z1)))]
    # the other volumes of the same scan (configs 0-3 share it): 1024^3
    # (config 3, the metric's second size) and 256^3 (config 1, BASELINE's
    # single-GPU case)
    for other in (3, 1):
        if args.config == other or cfg.width != synth.CONFIGS[other].width:
            continue
        go = synth.CONFIGS[other].geometry
        if world > 1:
            from paper_1401_3615_b200.distributed import balanced_slabs, plane_work
            slo = balanced_slabs(plane_work(go, mats, W, H), world)[rank]
        else:
            slo = (0, go.edge_voxels)
        sec.append(dict(workload=synth.CONFIGS[other].name, mode=args.mode,
                        **measure(go, mode, 3 if other == 3 else args.steps, slo)))
    # north_star's hardware-texture side number (not parity-exact)
    from paper_1401_3615_b200.backproject import backproject_texture_device
    vt = torch.empty(((z1 - z0), L, L), dtype=torch.float32, device=dev)

    def st_tex():
        vt.zero_()
        backproject_texture_device(vt, g, z0, z1, imgs, mats, stream)
    st_tex()
    torch.cuda.synchronize()
    ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ta.record(stream)
    for _ in range(3):
        st_tex()
    tb.record(stream)
    torch.cuda.synchronize()
    ms_t = ta.elapsed_time(tb) / 3
    dtex = pkg.compare_volumes_device(vt, vol)  # vs this run's main-mode volume
    sec.append({"workload": cfg.name, "mode": "texture (side number, not parity-exact)",
                "value": round(L ** 3 * n / (ms_t * 1e-3) / 1e9, 3), "unit": "GUp/s",
                "ms_per_step": round(ms_t, 3),
                "vs_" + args.mode: {k: dtex[k] for k in ("rel_l2", "max_abs_over_range")}})
    del vt
    torch.cuda.empty_cache()
    pkg.release_cached_memory()  # e.g. the texture variant's layered array
    return sec



def e2e_entries(c):
    """e2e through the public host API: pinned host projections -> host
    volume, H2D + kernels + D2H inside the timed region (world 1: the C ABI
    cbb_reconstruct; world > 1: the torch.distributed driver)."""
    pkg, torch, dist, dev, args = c.pkg, c.torch, c.dist, c.dev, c.args
    g, mats, imgs, L, n, H, W = c.g, c.mats, c.imgs, c.L, c.n, c.H, c.W
    z0, z1, slabs, mode, rank, world, local = c.z0, c.z1, c.slabs, c.mode, c.rank, c.world, c.local
    total_updates, n_proj = c.total_updates, c.n
    out = {}
    imgs_h = imgs.cpu().pin_memory()
    torch.cuda.empty_cache()
    imgs_np = imgs_h.numpy()
    # the host volume (pinned): this rank's slab planes are written by the call
    vol_h = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
    buf = vol_h.numpy()
    e2e_opt = pkg.Options(batch=args.batch, mode=mode, num_gpus=1, device_ids=[local],
                          volume_is_zero=True, slab=(z0, z1))
    if world == 1:
        # the drop-in C ABI: cbb_reconstruct with host buffers
        def e2e_call():
            buf[z0:z1] = 0.0
            t0 = time.perf_counter()
            st = pkg.reconstruct_arrays(buf, g, imgs_np, mats, e2e_opt)
            return time.perf_counter() - t0, st
        h2d = imgs_h.numel() * 4 + mats.nbytes
        path = "cbb_reconstruct (C ABI), pinned host buffers"
    else:
        # one process per GPU: batch b uploaded by rank b % N, then NCCL
        # broadcast (default) or read by every rank's pack over CUDA IPC
        # (CBB_BENCH_TRANSPORT=ipc, the fused transfer + pack)
        from paper_1401_3615_b200.distributed import DistributedReconstructor, batch_roots
        transport = os.environ.get("CBB_BENCH_TRANSPORT", "nccl")
        rec = DistributedReconstructor(g, W, H, batch=args.batch, slabs=slabs,
                                       options=e2e_opt, transport=transport)

        def e2e_call():
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            slab = rec.reconstruct(imgs_h, mats)
            return time.perf_counter() - t0, {"slab_planes": int(slab.shape[0])}
        h2d = sum(n for _, n, r in batch_roots(n_proj, args.batch, world) if r == rank) \
            * H * W * 4 + mats.nbytes
        path = ("DistributedReconstructor: 1/N of batches uploaded per rank + " +
                ("NCCL broadcast" if transport == "nccl" else "pack over CUDA IPC peer memory"))
    e2e_call()  # warm-up
    if dist:
        dist.barrier()
    e2e_s = []
    stats = None
    for _ in range(max(1, min(args.steps, 3))):
        dt, stats = e2e_call()
        e2e_s.append(dt)
    e2e_t = statistics.median(e2e_s)
    if dist:
        t = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    out["e2e"] = {"value": round(total_updates / e2e_t / 1e9, 3), "unit": "GUp/s",
                  "h2d_bytes_per_step": int(h2d),
                  "d2h_bytes_per_step": int((z1 - z0) * L * L * 4),
                  "seconds": round(e2e_t, 4), "path": path,
                  "phases": {k: round(v, 4) if isinstance(v, float) else v
                             for k, v in stats.items()
                             if k not in ("per_gpu_kernel_seconds", "culled_updates",
                                          "culled_fraction")}}
    if world == 1:
        # one untimed call with the culling counters on (slower kernels)
        cst = pkg.reconstruct_arrays(buf, g, imgs_np, mats, pkg.Options(
            batch=args.batch, mode=mode, num_gpus=1, device_ids=[local],
            volume_is_zero=True, count_culled=True))
        out["culled_fraction"] = round(cst["culled_fraction"], 4)
        # the host API's volume against the device-resident run's (same bits
        # expected: one arithmetic, any batching / staging / resident tail)
        vt = torch.from_numpy(buf[z0:z1]).to(dev)
        dff = pkg.compare_volumes_device(vt, c.vol)
        out["e2e"]["bitwise_different_vs_value_volume"] = int(dff["bitwise_different"])
        del vt
        out["e2e_adapter"] = e2e_adapter_entry(c, imgs_np)
        if not args.no_secondary and c.cfg.name == "c2_512":
            out["e2e_c3"] = e2e_config3_entry(c, imgs_np)
    del vol_h
    return out


def e2e_config3_entry(c, imgs_pinned):
    """Config 3 (1024^3 from the same scan) end to end through cbb_reconstruct:
    pinned host projections -> 4 GiB pinned host volume (BASELINE: slabs
    gathered to pinned host memory), H2D + kernels + D2H timed."""
    pkg, torch, args, mats, n, H, W = c.pkg, c.torch, c.args, c.mats, c.n, c.H, c.W
    from paper_1401_3615_b200 import synth

    g3 = synth.CONFIGS[3].geometry
    L3 = g3.edge_voxels
    vol_h = torch.zeros((L3, L3, L3), dtype=torch.float32).pin_memory()
    buf = vol_h.numpy()
    opt = pkg.Options(batch=args.batch, mode=c.mode, num_gpus=1, device_ids=[c.local],
                      volume_is_zero=True)
    pkg.reconstruct_arrays(buf, g3, imgs_pinned, mats, opt)  # warm-up
    ts, st = [], None
    for _ in range(2):
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(buf, g3, imgs_pinned, mats, opt)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    del vol_h, buf
    torch.cuda.empty_cache()
    return {"value": round(L3 ** 3 * n / t / 1e9, 3), "unit": "GUp/s", "seconds": round(t, 4),
            "h2d_bytes_per_step": int(n * H * W * 4 + mats.nbytes),
            "d2h_bytes_per_step": int(L3 ** 3 * 4),
            "kernel_seconds": round(st["kernel_seconds"], 4),
            "path": "cbb_reconstruct (C ABI), pinned projections -> pinned 4 GiB volume"}


def e2e_adapter_entry(c, imgs_src):
    """The drop-in's own host path, as the C++ adapter drives it
    (include/conebeam_b200.hpp reconstruct -> cbb_reconstruct_images): one
    PAGEABLE buffer per projection (the reference's ProjectionStack holds one
    std::vector<float> per image, dataset.hpp:15-60) and a NON-ZERO pageable
    volume that is uploaded, accumulated into and downloaded (vol +=,
    kernel_ref.cpp:32-38) -- no pinned inputs, no volume_is_zero."""
    import numpy as np

    pkg, args, g, mats, L, n, H, W = c.pkg, c.args, c.g, c.mats, c.L, c.n, c.H, c.W
    parts = [np.array(imgs_src[i]) for i in range(n)]  # n separate pageable buffers
    vol = np.full((L, L, L), 0.25, np.float32)          # pageable, non-zero
    opt = pkg.Options(batch=args.batch, mode=c.mode, num_gpus=1, device_ids=[c.local])
    pkg.reconstruct_images(vol, g, parts, mats, opt)    # warm-up
    ts = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        pkg.reconstruct_images(vol, g, parts, mats, opt)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    del parts, vol
    return {"value": round(L ** 3 * n / t / 1e9, 3), "unit": "GUp/s", "seconds": round(t, 4),
            "h2d_bytes_per_step": int(n * H * W * 4 + mats.nbytes + L ** 3 * 4),
            "d2h_bytes_per_step": int(L ** 3 * 4),
            "path": "cbb_reconstruct_images (the C++ adapter's call): pageable per-image "
                    "buffers, non-zero pageable volume uploaded + accumulated + downloaded"}


def filter_entry(c):
    """FDK ramp-filter stage (upstream of the reference's
    input): raw line integrals of the same scan, (a) the filter alone on
    device-resident data (cbb_ramp_filter_device, CUDA events), with its
    roofline, and (b) end to end through cbb_reconstruct with
    options.ramp_filter from pinned host line integrals."""
    import numpy as np

    pkg, torch, dev, args, cfg = c.pkg, c.torch, c.dev, c.args, c.cfg
    g, mats, L, n, H, W, stream = c.g, c.mats, c.L, c.n, c.H, c.W, c.stream
    from paper_1401_3615_b200 import synth

    _, _, raw = synth.make_inputs(cfg, device=dev, chunk=16, filtered=False)
    out = torch.empty_like(raw)
    pkg.ramp_filter_device(raw, out, cfg.pixel_mm, stream)  # warm-up (plans, spectrum)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    a.record(stream)
    for _ in range(reps):
        pkg.ramp_filter_device(raw, out, cfg.pixel_mm, stream)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    pixels = n * H * W
    peaks, src = measured_peaks()
    alg_bytes = 8 * pixels  # read + write one float per pixel
    # FP64-bound (ncu profiles/r2_ramp2560.txt: FP64 pipe 46 %, DRAM 9 %): two
    # rows per complex transform of the padded length N (2560 for W <= 1280,
    # 4096 for W <= 2048, else cuFFT's power of two), forward + inverse at the
    # conventional 5 N log2 N flops each, plus the real spectrum multiply
    nfft = 2560 if W <= 1280 else 4096 if W <= 2048 else 1 << (2 * W - 1).bit_length()
    pairs = (n * H + 1) // 2
    alg_flops = pairs * (2 * 5 * nfft * math.log2(nfft) + 2 * nfft)
    fp64_tflops = FP64_PEAK_TFLOPS
    res = {"workload": cfg.name, "stage": "ramp filter (Shepp-Logan, row-wise, float64)",
           "ms_per_stack": round(ms, 3), "share_of_step": round(ms / c.ms_step, 4),
           "roofline": {"bound": "fp64", "achieved": round(alg_flops / (ms * 1e-3) / 1e12, 2),
                        "peak": fp64_tflops, "unit": "TFLOP/s",
                        "frac": round(alg_flops / (ms * 1e-3) / 1e12 / fp64_tflops, 4),
                        "algorithmic_flops": int(alg_flops), "fft_length": nfft,
                        "peak_source": "measured DFMA throughput, profiles/probes/fp64_peak.cu "
                                       "(profiles/fp64_peak_r2.txt)",
                        "alongside": {"hbm": {
                            "achieved_GBps": round(alg_bytes / (ms * 1e-3) / 1e9, 1),
                            "peak_GBps": peaks.get("hbm_gbs"),
                            "frac": round(alg_bytes / (ms * 1e-3) / 1e9 / peaks.get("hbm_gbs"), 4),
                            "algorithmic_bytes": int(alg_bytes), "peak_source": src}}}}
    impl = pkg.ramp_filter_info() if hasattr(pkg, "ramp_filter_info") else None
    if impl:
        res["implementation"] = impl
    # e2e: raw line integrals from pinned host memory -> filtered on the GPU ->
    # back-projected -> host volume
    raw_h = raw.cpu().pin_memory()
    del raw, out
    torch.cuda.empty_cache()
    raw_np = raw_h.numpy()
    vol_h = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
    buf = vol_h.numpy()
    opt = pkg.Options(batch=args.batch, mode=c.mode, num_gpus=1, device_ids=[c.local],
                      volume_is_zero=True, ramp_filter_pixel_mm=cfg.pixel_mm)
    pkg.reconstruct_arrays(buf, g, raw_np, mats, opt)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        pkg.reconstruct_arrays(buf, g, raw_np, mats, opt)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    vt = torch.from_numpy(buf).to(dev)
    d = pkg.compare_volumes_device(vt, c.vol)
    res["e2e_filtered"] = {
        "value": round(L ** 3 * n / t / 1e9, 3), "unit": "GUp/s", "seconds": round(t, 4),
        "h2d_bytes_per_step": int(raw_np.nbytes + mats.nbytes), "d2h_bytes_per_step": L ** 3 * 4,
        "vs_prefiltered_volume": {k: d[k] for k in ("rel_l2", "max_abs_over_range")},
        "path": "cbb_reconstruct, options.ramp_filter, pinned raw line integrals"}
    del vt, raw_h, vol_h
    torch.cuda.empty_cache()
    return res


def config4_entry(c):
    """BASELINE config 4 on this GPU (the single-GPU leg of its 8-GPU run):
    1440 x 1536^2 projections of a 360-degree scan into a 1024^3 volume,
    batches of 16 as BASELINE states. Device-resident value with its roofline,
    culled fraction, and e2e through cbb_reconstruct from pinned host memory
    (13.6 GB in, 4.3 GB out)."""
    pkg, torch, dev, args = c.pkg, c.torch, c.dev, c.args
    from paper_1401_3615_b200 import synth

    cfg = synth.CONFIGS[4]
    pkg.release_cached_memory()  # earlier pipelines' cached device buffers
    torch.cuda.empty_cache()
    g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
    L = g.edge_voxels
    n, H, W = imgs.shape
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = c.stream
    res = {"workload": cfg.name, "edge_voxels": L, "projections": n, "detector": [W, H],
           "mode": args.mode}
    sst = SlabStep(pkg, torch, dev, g, imgs, mats, 0, L, pkg.Options(batch=16, mode=c.mode),
                   err, stream, force_quad=args.quad)
    vol = sst.vol
    res["kernel"] = sst.kernel
    for batch in (16,):
        # device-resident: launches of 64 projections on the staged path
        # (opt.batch sets the pipeline's upload batches, used by the e2e below)
        sst.opt = pkg.Options(batch=batch, mode=c.mode)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

        def step(rec=False):
            vol.zero_()
            if rec:
                ev[0].record(stream)
            sst.prep()
            if rec:
                ev[1].record(stream)
            sst.backproject()
            if rec:
                ev[2].record(stream)
        step()
        torch.cuda.synchronize()
        bp, pk = [], []
        for _ in range(2):
            step(True)
            torch.cuda.synchronize()
            pk.append(ev[0].elapsed_time(ev[1]))
            bp.append(ev[1].elapsed_time(ev[2]))
        ms = statistics.mean(pk) + statistics.mean(bp)
        nl = (n + 63) // 64 if sst.staged else (n + min(batch, 32) - 1) // min(batch, 32)
        launch_ms = statistics.mean(bp) / nl
        upd = L ** 3 * (n / nl)
        peaks, _ = measured_peaks()
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        frac = upd * OPS_PER_UPDATE / (launch_ms * 1e-3) / (nsm * 128 * sm_max * 1e6)
        res.update({"value": round(L ** 3 * n / (ms * 1e-3) / 1e9, 3),
                    "unit": "GUp/s", "ms_per_step": round(ms, 2),
                    "prep_ms": round(statistics.mean(pk), 2),
                    "projections_per_launch": 64 if sst.staged else min(batch, 32),
                    "roofline_frac": round(frac, 4)})
    if int(err.item()) != 0:
        res["error_flag"] = int(err.item())
    imgs_h = imgs.cpu().pin_memory()
    sst.release()
    del imgs, vol
    torch.cuda.empty_cache()
    imgs_np = imgs_h.numpy()
    vol_h = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
    buf = vol_h.numpy()
    opt = pkg.Options(batch=16, mode=c.mode, num_gpus=1, device_ids=[c.local],
                      volume_is_zero=True)
    cst = pkg.reconstruct_arrays(buf, g, imgs_np, mats, pkg.Options(
        batch=16, mode=c.mode, num_gpus=1, device_ids=[c.local], volume_is_zero=True,
        count_culled=True))
    res["culled_fraction"] = round(cst["culled_fraction"], 4)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(buf, g, imgs_np, mats, opt)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    res["e2e"] = {"value": round(L ** 3 * n / t / 1e9, 3), "unit": "GUp/s",
                  "seconds": round(t, 4), "h2d_bytes_per_step": int(imgs_np.nbytes + mats.nbytes),
                  "d2h_bytes_per_step": L ** 3 * 4, "guarded_batches": st["guarded_batches"],
                  "path": "cbb_reconstruct (C ABI), pinned host buffers, batch 16"}
    del imgs_h, vol_h, imgs_np, buf
    pkg.release_cached_memory()
    torch.cuda.empty_cache()
    return res


def parity_entry(c):
    """The timed run's own volume (the last timed step's output, still on the
    device) against the oracle, outside the timed region: every
    --parity-stride-th z-plane plus the last, all projections, recomputed by
    oracle_reconstruct_planes on the host cores and cached under a content
    hash of the inputs -- the reference bench scores every benchmarked volume
    against a reference volume cached by stack hash the same way
    (proj/src/bench.cpp:194-243)."""
    import numpy as np

    import oracle as O

    args, g, mats, L = c.args, c.g, c.mats, c.L
    try:
        planes = np.array(sorted(set(range(c.z0, c.z1, max(1, args.parity_stride))) |
                                 {c.z1 - 1}))
        host = c.imgs.cpu().numpy()
        ref, secs, hit = O.reference_planes(g, planes, host, mats)
        del host
        got = c.vol[c.torch.as_tensor(planes - c.z0, device=c.dev)].cpu().numpy()
        d = got.astype(np.float64) - ref.astype(np.float64)
        rng = float(ref.max()) - float(ref.min())
        rel = float(np.linalg.norm(d) / max(np.linalg.norm(ref.astype(np.float64)), 1e-300))
        mar = float(np.abs(d).max() / rng) if rng > 0 else float(np.abs(d).max())
        return {
            "vs": "oracle (C restatement of reconstruct_reference, pinned to the reference's "
                  "golden hash and to the reference itself)",
            "volume": "the timed run's own output (last timed step)",
            "planes_checked": int(planes.size), "of_planes": int(c.z1 - c.z0),
            "plane_stride": int(args.parity_stride),
            "voxels_checked": int(got.size),
            "bitwise_different": int(np.count_nonzero(got.view(np.uint32) !=
                                                      ref.view(np.uint32))),
            "rel_l2": rel, "max_abs_over_range": mar,
            "within_north_star_tolerance": bool(rel <= 1e-5 and mar <= 1e-4),
            "oracle_seconds": round(secs, 2), "oracle_cache_hit": bool(hit),
            "oracle_threads": os.cpu_count()}
    except Exception as e:  # reported, never silently dropped
        return {"error": f"{type(e).__name__}: {e}"}


def cpu_baseline_entry(c):
    """The reference's CPU path (reconstruct_optimized from oracle/_ref) on
    this box's host cores, on a bounded sample of the same workload."""
    args, cfg, g, mats, imgs, L, n = c.args, c.cfg, c.g, c.mats, c.imgs, c.L, c.n
    try:
        cnt, cores = size_cpu_sample(cfg, args.cpu_seconds)
        gcpu, mcpu, icpu = (g, mats[:cnt], imgs[:cnt].cpu().numpy())
        gups, st, kind, cores = time_reference_cpu(cfg, cnt, gcpu, mcpu, icpu)
        entry = {
            "value": round(gups, 4), "unit": "GUp/s", "cores": cores, "kind": kind,
            "sample": (f"{L}^3 volume x first {cnt} of {n} projections; reconstruct_optimized "
                       f"defaults (lanes 16, chunk 262, clip+pad); kernel "
                       f"{st['kernel_seconds']:.2f} s (+{st.get('precompute_seconds', 0):.2f} s "
                       f"precompute, excluded); full-basis updates")}
        if st.get("voxel_updates"):  # the reference's own (clipped) update count
            entry["clipped_basis"] = {
                "value": round(st["voxel_updates"] / st["kernel_seconds"] / 1e9, 4),
                "admitted_fraction": round(st["voxel_updates"] / (L ** 3 * cnt), 4)}
            entry["full_basis_incl_precompute"] = round(
                L ** 3 * cnt / (st["kernel_seconds"] + st.get("precompute_seconds", 0.0))
                / 1e9, 4)
    except Exception as e:  # the baseline is reported, never the target
        entry = {"value": None, "unit": "GUp/s", "cores": os.cpu_count(),
                 "kind": "reference", "sample": f"failed: {e}"}
    return entry


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
