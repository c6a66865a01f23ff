"""Probe: warp-tile shape against the ray direction. Times one 32-projection
launch of config 2 for batches whose rays run along x (theta ~ 0) or along y
(theta ~ 90 deg), per CBB_BP_VARIANT (tile 8x4 / 4x8 / 16x2 / 32x1)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[2]
dev = torch.device("cuda", 0)
g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
L = g.edge_voxels
n, H, W = imgs.shape
nb = pkg.packed_layout(W, H)[2]
packed = torch.empty(n * nb, dtype=torch.uint8, device=dev)
vol = torch.zeros((L, L, L), dtype=torch.float32, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
pkg.pack_device(imgs, packed)
opt = pkg.Options(batch=32)
st = torch.cuda.current_stream(dev)
variants = [int(v) for v in sys.argv[1:]] or [5, 7, 6, 8, 0]
names = {0: "8x4 (4-warp blk)", 5: "8x4", 6: "16x2", 7: "4x8", 8: "32x1"}
for first in range(0, n - 31, 31):
    theta = 200.0 * (first + 16) / n
    row = []
    for v in variants:
        os.environ["CBB_BP_VARIANT"] = str(v)

        def run():
            pkg.backproject_device(vol, g, 0, L, packed[first * nb:(first + 32) * nb], W, H, 32,
                                   mats[first:first + 32], opt, err, st)
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(3):
            run()
        b.record(st)
        torch.cuda.synchronize()
        row.append(a.elapsed_time(b) / 3)
    print(f"theta {theta:6.1f}: " + "  ".join(f"{names.get(v, v)} {t:6.3f}"
                                               for v, t in zip(variants, row)), flush=True)
