"""e2e of cbb_reconstruct on config 2 with resident mode off (CBB_NO_RESIDENT)
and on at several tail fractions (CBB_TAIL_FRAC), pinned host buffers,
phases from cbb_run_stats; every result is checked bitwise against the first."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

os.environ["CBB_TRACE"] = "1"
cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
imgs_h = imgs.pin_memory().numpy()
L = g.edge_voxels
vol_t = torch.zeros((L, L, L), dtype=torch.float32).pin_memory()
vol = vol_t.numpy()
opt = pkg.Options(volume_is_zero=True, batch=int(os.environ.get("BATCH", "32")))
ref = None
fracs = os.environ.get("FRACS", "0.06,0.09,0.11,0.14").split(",")
for tag in ["plain"] + fracs:
    if tag == "plain":
        os.environ["CBB_NO_RESIDENT"] = "1"
    else:
        os.environ.pop("CBB_NO_RESIDENT", None)
        os.environ["CBB_TAIL_FRAC"] = tag.split(":")[0]
        if tag.endswith(":one"):
            os.environ["CBB_TAIL_ONE_CHUNK"] = "1"
        else:
            os.environ.pop("CBB_TAIL_ONE_CHUNK", None)
    best = 1e9
    for i in range(3):
        vol[:] = 0
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(vol, g, imgs_h, mats, opt)
        dt = time.perf_counter() - t0
        best = min(best, dt)
        print(f"{tag} run {i}: {dt * 1e3:.1f} ms -> {cfg.voxel_updates / dt / 1e9:.1f} GUp/s "
              f"kernel {st['kernel_seconds'] * 1e3:.1f} d2h {st['d2h_seconds'] * 1e3:.1f} "
              f"total {st['total_seconds'] * 1e3:.1f}", flush=True)
    print(f"== {tag}: best {best * 1e3:.1f} ms -> {cfg.voxel_updates / best / 1e9:.1f} GUp/s")
    if ref is None:
        ref = vol.copy()
    else:
        print(f"  bitwise equal to plain: {np.array_equal(ref.view(np.uint32), vol.view(np.uint32))}")

# the reference's stack layout: one pageable buffer per projection
# (cbb_reconstruct_images), and one contiguous pageable array (cbb_reconstruct)
os.environ.pop("CBB_NO_RESIDENT", None)
os.environ.pop("CBB_TAIL_FRAC", None)
parts = [np.array(imgs_h[i], copy=True) for i in range(len(imgs_h))]
pageable = np.array(imgs_h, copy=True)
for tag, fn in (("per-image buffers", lambda: pkg.reconstruct_images(vol, g, parts, mats, opt)),
                ("contiguous pageable", lambda: pkg.reconstruct_arrays(vol, g, pageable, mats, opt))):
    best = 1e9
    for i in range(3):
        vol[:] = 0
        t0 = time.perf_counter()
        st = fn()
        best = min(best, time.perf_counter() - t0)
    print(f"== {tag}: best {best * 1e3:.1f} ms -> {cfg.voxel_updates / best / 1e9:.1f} GUp/s "
          f"(kernel {st['kernel_seconds'] * 1e3:.1f} ms)")
    print(f"  bitwise equal to plain: {np.array_equal(ref.view(np.uint32), vol.view(np.uint32))}")
