"""End-to-end GUp/s of cbb_reconstruct (pinned host projections -> pinned
host volume, exact mode) for BASELINE configs 0-3 on one B200, next to the
device-resident rate of the same call (kernel_seconds) and the PCIe floor
(the projections' H2D at the measured ~55 GB/s)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

imgs_h = None
for cid in (0, 1, 2, 3):
    cfg = synth.CONFIGS[cid]
    g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16, pin=True) \
        if imgs_h is None else (cfg.geometry, mats, imgs_h)
    imgs_h = imgs
    L = g.edge_voxels
    vol = torch.zeros((L, L, L), dtype=torch.float32).pin_memory().numpy()
    U = L ** 3 * len(mats)
    best, st_best = 1e9, None
    times = []
    for i in range(int(os.environ.get("E2E_REPS", "3"))):
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(vol, g, imgs.numpy(), mats, pkg.Options(volume_is_zero=True))
        dt = time.perf_counter() - t0
        times.append(round(dt * 1e3, 1))
        if dt < best:
            best, st_best = dt, st
    h2d = imgs.numel() * 4 / 55e9
    print(f"config {cid} ({L}^3 x {len(mats)}): e2e {best * 1e3:8.1f} ms = {U / best / 1e9:7.1f} GUp/s"
          f" | kernels {st_best['kernel_seconds'] * 1e3:7.1f} ms | H2D floor {h2d * 1e3:5.1f} ms"
          f" | D2H {L ** 3 * 4 / 1e9:.2f} GB | in-call {st_best['total_seconds'] * 1e3:.1f} ms"
          f" | runs (ms) {times}", flush=True)
