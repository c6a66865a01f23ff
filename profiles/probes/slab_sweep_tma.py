"""Per-rank step time of the N-GPU device path with the TMA-staged kernel,
measured one slab at a time on one B200: for N in (1, 2, 4, 8) the
work-balanced z-slabs of a config (CFG, default 2), each timed as the scan +
back-projection of all projections from the rank's band of raw rows (what
bench.py's `value` times per rank at N > 1). max over slabs = the step a
rank of an N-GPU run would need if nothing else interfered -- an upper-bound
projection, not a multi-GPU measurement (the pool has one GPU)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402
from paper_1401_3615_b200.distributed import balanced_slabs, plane_work  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
dev = torch.device("cuda", 0)
g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
L = g.edge_voxels
n, H, W = imgs.shape
err = torch.zeros(1, dtype=torch.int32, device=dev)
opt = pkg.Options(batch=32)
stream = torch.cuda.current_stream(dev)
work = plane_work(g, mats, W, H)
flags = torch.zeros(n, dtype=torch.int32, device=dev)


def time_slab(z0, z1, reps=3):
    plan = pkg.tma_plan(g, W, H, z0, z1, mats)
    band = pkg.row_band_for_slab(g, W, H, z0, z1, mats)
    full = band.raw_rows == H and band.raw_row0 == 0
    src = imgs if full else imgs[:, band.raw_row0:band.raw_row0 + band.raw_rows].contiguous()
    vol = torch.zeros((z1 - z0, L, L), dtype=torch.float32, device=dev)
    out = []
    for r in range(reps + 1):
        vol.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        pkg.scan_device(src, flags, err, stream)
        b.record(stream)
        pkg.backproject_raw_device(vol, g, z0, z1, src, W, H, n, mats, flags, opt, err, stream,
                                   band=None if full else band)
        c.record(stream)
        torch.cuda.synchronize()
        if r:
            out.append((a.elapsed_time(b), b.elapsed_time(c)))
    del src, vol
    return (statistics.median(o[0] for o in out), statistics.median(o[1] for o in out), band,
            plan)


U = L ** 3 * n
for world in (1, 2, 4, 8):
    slabs = balanced_slabs(work, world) if world > 1 else [(0, L)]
    rows = []
    for z0, z1 in slabs:
        sc, bp, band, plan = time_slab(z0, z1)
        rows.append(sc + bp)
        print(f"N={world} slab [{z0:4d},{z1:4d}) rows {band.raw_rows:4d}/{H} box "
              f"{plan['box_width']}x{plan['box_rows']} staged {plan['staged']}: scan {sc:5.2f} + bp "
              f"{bp:7.2f} = {sc + bp:7.2f} ms", flush=True)
    t = max(rows)
    print(f"== {cfg.name} N={world}: max rank step {t:.2f} ms (mean {statistics.mean(rows):.2f}) "
          f"-> {U / t / 1e6:.0f} GUp/s", flush=True)
