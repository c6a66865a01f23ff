"""Probe: does packing batch k+1 on a second (high-priority) stream while
batch k is back-projected hide the pack time? Device-resident config 2,
exact; compares the serial step (pack all, then back-project, as bench.py's
value step) with per-batch packs on a side stream, and checks the volume
bitwise."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
dev = torch.device("cuda", 0)
g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
L = g.edge_voxels
n, H, W = imgs.shape
band = pkg.row_band_for_slab(g, W, H, 0, L, mats)
nb = band.packed_bytes(W, H)
packed = torch.empty(n * nb, dtype=torch.uint8, device=dev)
vol = torch.empty((L, L, L), dtype=torch.float32, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
B = 32
opt = pkg.Options(batch=B)
main = torch.cuda.current_stream(dev)


def serial():
    vol.zero_()
    pkg.pack_device_band(imgs, band, packed, err, main)
    pkg.backproject_device(vol, g, 0, L, packed, W, H, n, mats, opt, err, main, band=band)


def overlapped(side):
    vol.zero_()
    evs = []
    side.wait_stream(main)
    for k in range(0, n, B):
        m = min(B, n - k)
        pkg.pack_device_band(imgs[k:k + m], band, packed[k * nb:(k + m) * nb], err, side)
        e = torch.cuda.Event()
        e.record(side)
        evs.append(e)
    for i, k in enumerate(range(0, n, B)):
        m = min(B, n - k)
        main.wait_event(evs[i])
        pkg.backproject_device(vol, g, 0, L, packed[k * nb:(k + m) * nb], W, H, m,
                               mats[k:k + m], opt, err, main, band=band)


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for _ in range(reps):
        fn()
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_serial = timeit(serial)
ref = vol.clone()
U = L ** 3 * n
print(f"serial            {t_serial:8.3f} ms  {U / t_serial / 1e6:7.1f} GUp/s", flush=True)
for prio in (0, -1):
    side = torch.cuda.Stream(dev, priority=prio)
    t = timeit(lambda: overlapped(side))
    same = bool(torch.equal(vol.view(torch.int32), ref.view(torch.int32)))
    print(f"side prio {prio:2d}      {t:8.3f} ms  {U / t / 1e6:7.1f} GUp/s  bitwise {same}",
          flush=True)
