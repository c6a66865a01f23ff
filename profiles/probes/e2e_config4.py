"""Config 4 end to end on one B200 through cbb_reconstruct: 1440 projections
of 1536x1536 (13.6 GB pinned host) -> 1024^3 volume (4.3 GB pinned host),
streamed in batches; exact and fast mode. Spot-checks three planes against
the device-resident path bitwise."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[4]
t0 = time.perf_counter()
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16, pin=True)
print(f"inputs {time.perf_counter() - t0:.1f} s, {imgs.numel() * 4 / 1e9:.1f} GB pinned", flush=True)
L = g.edge_voxels
vol_t = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
vol = vol_t.numpy()
imgs_np = imgs.numpy()
U = L ** 3 * len(mats)
for mode, name in ((pkg.MODE_EXACT, "exact"), (pkg.MODE_FAST, "fast")):
    opt = pkg.Options(volume_is_zero=True, mode=mode, batch=int(os.environ.get("BATCH", "32")))
    for i in range(2):
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(vol, g, imgs_np, mats, opt)
        dt = time.perf_counter() - t0
        print(f"{name} run {i}: {dt:.3f} s -> {U / dt / 1e9:.1f} GUp/s e2e "
              f"(kernel {st['kernel_seconds']:.3f} s, d2h {st['d2h_seconds']:.3f} s)", flush=True)
    if name == "exact":
        # three planes recomputed on the device path (whole stack packed per chunk)
        dev = torch.device("cuda")
        _, _, nb = pkg.packed_layout(cfg.width, cfg.height)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        for z in (0, 511, 1023):
            v = torch.zeros((1, L, L), dtype=torch.float32, device=dev)
            for c0 in range(0, len(mats), 96):
                c1 = min(len(mats), c0 + 96)
                raw = imgs[c0:c1].to(dev)
                packed = torch.empty((c1 - c0) * nb, dtype=torch.uint8, device=dev)
                pkg.pack_device(raw, packed)
                pkg.backproject_device(v, g, z, z + 1, packed, cfg.width, cfg.height, c1 - c0,
                                       mats[c0:c1], pkg.Options(batch=32), err_flag=err)
            torch.cuda.synchronize()
            same = np.array_equal(v.cpu().numpy()[0].view(np.uint32), vol[z].view(np.uint32))
            print(f"  plane {z}: bitwise equal to the device path: {same}", flush=True)
