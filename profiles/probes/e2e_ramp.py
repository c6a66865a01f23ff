"""e2e of cbb_reconstruct (config 2, pinned, volume_is_zero: bench.py's e2e
call) under launch-policy variants; each variant runs in a fresh process
(CBB_* knobs are read once) -- VARIANTS="name:ENV=V;ENV2=V2,..."."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import time
    import numpy as np
    import torch
    import paper_1401_3615_b200 as pkg
    from paper_1401_3615_b200 import synth
    cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
    g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
    h = imgs.pin_memory().numpy()
    L = g.edge_voxels
    vol = torch.zeros((L, L, L), dtype=torch.float32).pin_memory().numpy()
    opt = pkg.Options(volume_is_zero=True, num_gpus=1)
    ts = []
    for i in range(int(os.environ.get("REPS", "7"))):
        t0 = time.perf_counter()
        st = pkg.reconstruct_arrays(vol, g, h, mats, opt)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    import hashlib
    dig = hashlib.sha1(vol.tobytes()).hexdigest()[:12]
    print(f"RESULT best {ts[0] * 1e3:.2f} ms median {ts[len(ts) // 2] * 1e3:.2f} ms "
          f"-> {cfg.voxel_updates / ts[0] / 1e9:.1f} GUp/s kernel {st['kernel_seconds'] * 1e3:.1f} "
          f"hash {dig}", flush=True)
    sys.exit(0)
for v in os.environ.get("VARIANTS", "base:").split(","):
    name, _, envs = v.partition(":")
    env = dict(os.environ)
    for kv in filter(None, envs.split(";")):
        k, _, val = kv.partition("=")
        env[k] = val
    out = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(name, line[0] if line else out.stderr[-800:], flush=True)
