"""Config 2 e2e through cbb_reconstruct (pinned projections, pinned volume,
volume_is_zero), as bench.py's e2e: wall time per call next to the
pipeline's own phases (CBB_TRACE=1 prints host init / submit / finish and
the resident tail timeline)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
h = imgs.pin_memory().numpy()
L = g.edge_voxels
vol = torch.zeros((L, L, L), dtype=torch.float32).pin_memory().numpy()
opt = pkg.Options(volume_is_zero=True, num_gpus=1)
pkg.reconstruct_arrays(vol, g, h, mats, opt)
for _ in range(int(os.environ.get("REPS", "4"))):
    t0 = time.perf_counter()
    st = pkg.reconstruct_arrays(vol, g, h, mats, opt)
    t = time.perf_counter() - t0
    print(f"e2e: {t * 1e3:.2f} ms = {L ** 3 * h.shape[0] / t / 1e9:.1f} GUp/s; kernels "
          f"{st['kernel_seconds'] * 1e3:.2f} d2h {st['d2h_seconds'] * 1e3:.2f} ms", flush=True)
