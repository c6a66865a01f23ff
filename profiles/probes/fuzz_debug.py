"""Re-runs one fuzz case (tests/test_gpu_fuzz.py) under switches and reports
which z-planes differ from the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_1401_3615_b200 as pkg  # noqa: E402
from test_gpu_fuzz import case  # noqa: E402

seed = int(sys.argv[1])
g, mats, imgs, vol0, opts, r = case(seed)
print("L", g.edge_voxels, "n", len(mats), "W,H", imgs.shape[2], imgs.shape[1], "opts", opts)
ref = vol0.copy()
print("oracle status", O.reconstruct(ref, g, imgs, mats))
envs = [{}, {"CBB_NO_RESIDENT": "1"}, {"CBB_NO_PEER_PACK": "1"}, {"CBB_NO_BANDS": "1"},
        {"CBB_NO_RESIDENT": "1", "CBB_NO_BANDS": "1"}, {"CBB_BP_VARIANT": "5"}]
for ids in (opts["device_ids"], [0]):
    for env in envs:
        for k in ("CBB_NO_RESIDENT", "CBB_NO_PEER_PACK", "CBB_NO_BANDS", "CBB_BP_VARIANT"):
            os.environ.pop(k, None)
        os.environ.update(env)
        o = dict(opts, device_ids=ids)
        v = pkg.Volume(g, vol0.copy())
        os.environ["CBB_TRACE"] = "1"
        st = pkg.reconstruct(v, pkg.ProjectionStack(g, mats, imgs), pkg.Options(**o))
        os.environ.pop("CBB_TRACE")
        d = v.voxels.view(np.uint32) != ref.view(np.uint32)
        planes = np.nonzero(d.any(axis=(1, 2)))[0]
        print(ids, env, "diff voxels", int(d.sum()), "planes", planes[:20], "...", len(planes),
              "guarded", st["guarded_batches"], flush=True)
