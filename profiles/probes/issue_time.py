"""Host issue time per batch of cbb_reconstruct (CBB_TRACE=1 prints it):
config 2 from pinned host memory with G workers on the visible GPU(s)
(device_ids = [0] * G on a one-GPU box: the issue cost of G devices, G^2
stream-event waits per batch, without G devices' bandwidth).

    CBB_TRACE=1 python profiles/probes/issue_time.py G [batch]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16, pin=True)
host = imgs.numpy()
L = g.edge_voxels
vol = torch.zeros((L, L, L), dtype=torch.float32).pin_memory().numpy()
opt = pkg.Options(device_ids=[0] * G, batch=batch, volume_is_zero=True)
pkg.reconstruct_arrays(vol, g, host, mats, opt)
for _ in range(2):
    t0 = time.perf_counter()
    st = pkg.reconstruct_arrays(vol, g, host, mats, opt)
    print(f"G={G} batch={batch}: {time.perf_counter() - t0:.3f} s, kernels {st['kernel_seconds']:.3f} s",
          flush=True)
