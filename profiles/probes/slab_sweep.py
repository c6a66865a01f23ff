"""Per-rank step time of the N-GPU device path, measured one slab at a time on
one B200: for N in (2, 4, 8) the balanced z-slabs of config 2, each timed as
pack (row band vs full detector) + back-projection of all 496 projections.
max over slabs = the step time a rank of an N-GPU run would see if nothing
else interfered (NVLink traffic, host); an upper-bound projection, not a
multi-GPU measurement."""
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
full_nb = pkg.packed_layout(W, H)[2]
packed = torch.empty(n * full_nb, dtype=torch.uint8, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
opt = pkg.Options(batch=32)
stream = torch.cuda.current_stream(dev)
work = plane_work(g, mats, W, H)


def time_slab(z0, z1, use_band, reps=3):
    vol = torch.zeros((z1 - z0, L, L), dtype=torch.float32, device=dev)
    band = pkg.row_band_for_slab(g, W, H, z0, z1, mats)
    out = []
    for r in range(reps + 1):
        vol.zero_()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record(stream)
        if use_band:
            pkg.pack_device_band(imgs, band, packed, err, stream)
        else:
            pkg.pack_device(imgs, packed, stream)
        b.record(stream)
        pkg.backproject_device(vol, g, z0, z1, packed, W, H, n, mats, opt, err, stream,
                               band=band if use_band else None)
        c.record(stream)
        torch.cuda.synchronize()
        if r:
            out.append((a.elapsed_time(b), b.elapsed_time(c)))
    pk = statistics.median(o[0] for o in out)
    bp = statistics.median(o[1] for o in out)
    return pk, bp, band


for world in (1, 2, 4, 8):
    slabs = balanced_slabs(work, world) if world > 1 else [(0, L)]
    rows = []
    for z0, z1 in slabs:
        pf, bf, _ = time_slab(z0, z1, False)
        pb, bb, band = time_slab(z0, z1, True)
        rows.append((z0, z1, pf, bf, pb, bb, band))
        print(f"N={world} slab [{z0:4d},{z1:4d}) rows {band.raw_rows:4d}/{H}: "
              f"full pack {pf:6.2f} + bp {bf:6.2f} = {pf + bf:6.2f} ms | "
              f"band pack {pb:6.2f} + bp {bb:6.2f} = {pb + bb:6.2f} ms", flush=True)
    tf = max(r[2] + r[3] for r in rows)
    tb = max(r[4] + r[5] for r in rows)
    U = L ** 3 * n
    print(f"== N={world}: max rank step full {tf:.2f} ms -> {U / tf / 1e6:.0f} GUp/s; "
          f"band {tb:.2f} ms -> {U / tb / 1e6:.0f} GUp/s", flush=True)
