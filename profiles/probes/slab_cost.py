"""Per-plane cost of one 64-projection raw launch over different z ranges of
config 2 (is a thin tail slab less efficient per plane than the head?)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=16)
n, H, W = imgs.shape
L = g.edge_voxels
flags = torch.zeros(n, dtype=torch.int32, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
pkg.scan_device(imgs, flags, err)
vol = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
fast = os.environ.get("FAST") == "1"
COUNT = int(os.environ.get("COUNT", "64"))
opt = pkg.Options(mode=pkg.MODE_FAST if fast else pkg.MODE_EXACT)
ranges = [tuple(map(int, r.split(":"))) for r in os.environ["RANGES"].split(",")] if os.environ.get("RANGES") else [(0, 12), (0, 36), (12, 48), (464, 500), (500, 512), (476, 512), (250, 262), (232, 268), (0, 512), (48, 464)]
for z0, z1 in ranges:
    v = vol[z0:z1]
    print(z0, z1, pkg.tma_plan(g, W, H, z0, z1, mats[:64]))
    ts = []
    for rep in range(int(os.environ.get('REPS', 6))):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        pkg.backproject_raw_device(v, g, z0, z1, imgs, W, H, COUNT, mats, flags, opt, err, first=64 * (rep % 7))
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts[1:]))
    print(f"  z [{z0},{z1}) {t:.3f} ms  {1000 * t / (z1 - z0):.2f} us/plane")
