"""Debug probe: the raw/TMA back-projection on a central sub-cube of a
BASELINE scan (config voxel size kept), bitwise against the packed path."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402
from paper_1401_3615_b200.geometry import VolumeGeometry  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 128
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
_, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=8, count=n)
g = VolumeGeometry.centered(L, cfg.voxel_mm)
n, H, W = imgs.shape
err = torch.zeros(1, dtype=torch.int32, device="cuda")
flags = torch.zeros(n, dtype=torch.int32, device="cuda")
pkg.scan_device(imgs, flags, err)
torch.cuda.synchronize()
print("scan ok", err.item(), flush=True)
v = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
pkg.backproject_raw_device(v, g, 0, L, imgs, W, H, n, mats, flags, pkg.Options(), err)
torch.cuda.synchronize()
print("raw ok", float(v.abs().sum()), err.item(), flush=True)
vq = torch.zeros_like(v)
nb = pkg.packed_layout(W, H)[2]
packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
pkg.pack_device(imgs, packed)
pkg.backproject_device(vq, g, 0, L, packed, W, H, n, mats, pkg.Options(), err)
d = pkg.compare_volumes_device(v, vq)
print("bitwise_different", d["bitwise_different"], "of", L ** 3, "max_abs", d["max_abs"])
