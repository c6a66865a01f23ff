"""Throughput of cbb_reconstruct_file on config 2 (writes a 2.4 GB CBPS file
to /tmp on the GPU box, then streams it twice: cold-ish and page-cached)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1401_3615_b200 as pkg  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[2]
g, mats, imgs = synth.make_inputs(cfg, device="cuda", out_device="cpu", chunk=16)
path = "/tmp/c2_512.cbps"
t0 = time.perf_counter()
pkg.write_stack(path, pkg.ProjectionStack(g, mats, imgs.numpy()))
print(f"write {time.perf_counter() - t0:.2f} s, {os.path.getsize(path) / 1e9:.2f} GB")
for i in range(3):
    t0 = time.perf_counter()
    vol, st = pkg.reconstruct_file(path)
    dt = time.perf_counter() - t0
    print(f"reconstruct_file run {i}: {dt:.3f} s -> {cfg.voxel_updates / dt / 1e9:.1f} GUp/s "
          f"(kernel {st['kernel_seconds']:.3f} s)")
pass

# raw read throughput of the same file (page cache), for comparison
import concurrent.futures as cf  # noqa: E402

import numpy as np  # noqa: E402

pkg.write_stack(path, pkg.ProjectionStack(g, mats, imgs.numpy()))
size = os.path.getsize(path)
buf = np.empty(size, np.uint8)
for nt in (1, 4, 8, 16):
    fd = os.open(path, os.O_RDONLY)
    per = (size + nt - 1) // nt

    def rd(t):
        off = t * per
        mv = memoryview(buf)[off:min(size, off + per)]
        done = 0
        while done < len(mv):
            done += os.preadv(fd, [mv[done:]], off + done)

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(nt) as ex:
        list(ex.map(rd, range(nt)))
    dt = time.perf_counter() - t0
    os.close(fd)
    print(f"raw pread {nt:2d} threads: {size / dt / 1e9:.1f} GB/s")
os.remove(path)
