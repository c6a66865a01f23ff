"""Raw-projection TMA back-projection vs the packed-quad kernel on a BASELINE
config (device-resident, CUDA events): bitwise comparison of the two volumes
and ms per step (scan + TMA kernel vs pack + gather kernel).

    python profiles/probes/tma_probe.py [config=2] [mode=exact] [steps=5]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
mode = pkg.MODE_FAST if len(sys.argv) > 2 and sys.argv[2] == "fast" else pkg.MODE_EXACT
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=16)
L = g.edge_voxels
n, H, W = imgs.shape
opt = pkg.Options(mode=mode)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
vq = torch.zeros((L, L, L), dtype=torch.float32, device="cuda")
vt = torch.zeros_like(vq)
nb = pkg.packed_layout(W, H)[2]
packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
flags = torch.zeros(n, dtype=torch.int32, device="cuda")


def quad():
    vq.zero_()
    pkg.pack_device(imgs, packed)
    pkg.backproject_device(vq, g, 0, L, packed, W, H, n, mats, opt, err)


def tma():
    vt.zero_()
    pkg.scan_device(imgs, flags, err)
    pkg.backproject_raw_device(vt, g, 0, L, imgs, W, H, n, mats, flags, opt, err)


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


tq = timeit(quad)
tt = timeit(tma)
d = pkg.compare_volumes_device(vt, vq)
print(f"{cfg.name} {'exact' if mode == 0 else 'fast'}: quad {tq:.2f} ms ({L**3 * n / tq / 1e6:.1f} GUp/s), "
      f"tma {tt:.2f} ms ({L**3 * n / tt / 1e6:.1f} GUp/s); bitwise_different {d['bitwise_different']}, "
      f"err {int(err.item())}")
