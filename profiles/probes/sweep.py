"""Kernel-variant sweep on the resident config-2 workload (GPU box).

    python profiles/probes/sweep.py [config] [variants...]
Times pack + back-projection per step with CUDA events, exact and fast mode,
for each CBB_BP_VARIANT value; checks exact-mode variants bitwise against
variant 0 on the full volume.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
variants = [int(v) for v in sys.argv[2:]] or [0, 1, 2, 3, 4, 5]
cfg = synth.CONFIGS[cfg_id]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=16)
L = g.edge_voxels
n, H, W = imgs.shape
_, _, nb = pkg.packed_layout(W, H)
packed = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
vol = torch.empty((L, L, L), dtype=torch.float32, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
ref = None
BATCH = int(os.environ.get("SWEEP_BATCH", "32"))
for mode in (pkg.MODE_EXACT, pkg.MODE_FAST):
    for v in variants:
        os.environ["CBB_BP_VARIANT"] = str(v)
        opt = pkg.Options(mode=mode, batch=BATCH)

        def step():
            vol.zero_()
            pkg.pack_device(imgs, packed)
            pkg.backproject_device(vol, g, 0, L, packed, W, H, n, mats, opt, err)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        gups = L ** 3 * n / (ms * 1e-3) / 1e9
        same = ""
        if mode == pkg.MODE_EXACT:
            if ref is None:
                ref = vol.clone()
            same = "bitwise==v0" if torch.equal(vol.view(torch.int32), ref.view(torch.int32)) \
                else "DIFFERS from v0"
        print(f"mode {mode} variant {v}: {ms:8.3f} ms/step  {gups:7.1f} GUp/s  {same}", flush=True)
