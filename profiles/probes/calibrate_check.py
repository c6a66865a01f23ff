"""Exercises bench.calibrate_slabs on one GPU with a stand-in process group:
rank 0 of a pretend world of 2 whose peer reports a 1.3x longer step, so the
rebalance branch runs (the real N > 1 path needs several GPUs)."""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402
from paper_1401_3615_b200.distributed import balanced_slabs, plane_work, rebalance_slabs  # noqa

cfg = synth.shrunk(synth.CONFIGS[2], num_projections=64)
dev = torch.device("cuda", 0)
g, mats, imgs = synth.make_inputs(cfg, device=dev, chunk=16)
n, H, W = imgs.shape
work = plane_work(g, mats, W, H)
slabs = balanced_slabs(work, 2)


def all_gather(out, t):
    out[0].copy_(t)
    out[1].copy_(t * 1.3)


fake = types.SimpleNamespace(all_gather=all_gather)
args = types.SimpleNamespace(batch=32, mode="exact")
res = bench.calibrate_slabs(pkg, fake, dev, g, imgs, mats, work, slabs, 0, 2, args,
                            rebalance_slabs)
print("before", slabs, "after", res)
assert res["rounds"] >= 1 and res["slabs"][0][1] != slabs[0][1]
print("calibrate_slabs OK")
