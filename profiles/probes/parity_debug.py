"""Diagnostics for a bitwise parity failure: per-mode / per-batch diff stats
against the reference fixtures (run on the GPU box)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import oracle as O  # noqa: E402
import paper_1401_3615_b200 as pkg  # noqa: E402
from conftest import load_golden  # noqa: E402


def stats(v, r):
    vb, rb = v.view(np.int32).astype(np.int64), r.view(np.int32).astype(np.int64)
    d = vb != rb
    n = int(d.sum())
    if n == 0:
        return "bitwise equal"
    idx = np.argwhere(d)
    ulps = np.abs(vb - rb)[d]
    return (f"{n} voxels differ; max ulps {ulps.max()}, median {np.median(ulps)}; "
            f"first {idx[:3].tolist()} v={v[tuple(idx[0])]!r} r={r[tuple(idx[0])]!r}")


for name in sys.argv[1:] or ["mini_c0.npz", "random_w.npz"]:
    g, mats, imgs, vol0, expected = load_golden(name)
    for mode in (pkg.MODE_EXACT,):
        for batch in (1, 32):
            vol = pkg.Volume(g, vol0.copy())
            st = pkg.reconstruct(vol, pkg.ProjectionStack(g, mats, imgs),
                                 pkg.Options(batch=batch, mode=mode))
            print(name, "mode", mode, "batch", batch, "guarded", st["guarded_batches"], ":",
                  stats(vol.voxels, expected))
    # one projection at a time from zero
    for p in range(min(3, len(mats))):
        ref = np.zeros_like(vol0)
        O.reconstruct(ref, g, imgs[p:p + 1], mats[p:p + 1])
        vol = pkg.Volume(g, np.zeros_like(vol0))
        pkg.reconstruct(vol, pkg.ProjectionStack(g, mats[p:p + 1], imgs[p:p + 1]))
        print("  single projection", p, ":", stats(vol.voxels, ref))
