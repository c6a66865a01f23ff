import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
h = imgs.pin_memory().numpy()
L = g.edge_voxels
vol = torch.zeros((L, L, L), dtype=torch.float32).pin_memory().numpy()
opt = pkg.Options(volume_is_zero=True, num_gpus=1)
for _ in range(2):
    pkg.reconstruct_arrays(vol, g, h, mats, opt)
