"""The drop-in's own host path (what include/conebeam_b200.hpp does):
cbb_reconstruct_images from pageable per-image buffers with a non-zero
pageable volume, config 2; CBB_TRACE=1 prints the pipeline phases."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
host = imgs.numpy()
parts = [np.array(host[i]) for i in range(host.shape[0])]
L = g.edge_voxels
vol = np.full((L, L, L), 0.25, np.float32)
opt = pkg.Options(num_gpus=1)
pkg.reconstruct_images(vol, g, parts, mats, opt)
for _ in range(int(os.environ.get('REPS', '3'))):
    t0 = time.perf_counter()
    st = pkg.reconstruct_images(vol, g, parts, mats, opt)
    t = time.perf_counter() - t0
    print(f"adapter path: {t * 1e3:.1f} ms = {L ** 3 * len(parts) / t / 1e9:.1f} GUp/s; "
          f"h2d {st['h2d_seconds'] * 1e3:.1f} kernels {st['kernel_seconds'] * 1e3:.1f} "
          f"d2h {st['d2h_seconds'] * 1e3:.1f} ms", flush=True)
