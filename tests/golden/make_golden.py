"""Generates the committed golden fixtures of tests/golden/ FROM THE REFERENCE.

Run in the build container (needs oracle/_ref/libconebeam_ref.so, which
oracle/Makefile compiles from /root/reference/proj/src):

    python tests/golden/make_golden.py

Each fixture holds seeded inputs and the volume the UNMODIFIED reference
reconstruct_reference (proj/src/kernel_ref.cpp:32-38) produced for them,
starting from a seeded non-zero volume (accumulation semantics):

  mini_c0.npz       BASELINE config-0 scan shrunk to a 24^3 volume, 6
                    projections, 156x120 detector (same physical size),
                    ellipsoid phantom + ramp filter: border-heavy data.
  random_w.npz      reference-test-style random stack (proj/tests/helpers.hpp:59-93):
                    random 3x4 matrices in [-5, 5] whose w changes sign over
                    the volume, random images in [-100, 100], odd sizes.
  orthographic.npz  proj/tests/test_kernel_ref.cpp:137-155 constant-add case.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1401_3615_b200 import synth  # noqa: E402
from paper_1401_3615_b200.geometry import VolumeGeometry  # noqa: E402


def _save(name, geometry, mats, imgs, vol0):
    vol = vol0.copy()
    status = O.ref_reconstruct_reference(vol, geometry, imgs, mats)
    np.savez_compressed(
        os.path.join(HERE, name), L=geometry.edge_voxels, voxel_mm=geometry.voxel_mm,
        origin_mm=geometry.origin_mm, mats=mats, imgs=imgs.astype(np.float32),
        vol0=vol0, expected=vol, status=status)
    print(name, "status", status, "hash", hex(O.fnv1a64(vol)))


def main():
    rng = synth.SplitMix64(20260101)

    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=24, num_projections=6, width=156,
                       height=120)
    g, mats, imgs = synth.make_inputs(cfg)
    vol0 = np.array([rng.uniform(-1.0, 1.0) for _ in range(24 ** 3)],
                    dtype=np.float32).reshape(24, 24, 24)
    _save("mini_c0.npz", g, mats, imgs.numpy(), vol0)

    # random matrices with sign-changing w (never exactly zero on these voxels)
    for attempt in range(100):
        L = 7
        g = VolumeGeometry(L, rng.uniform(0.1, 2.0), rng.uniform(-10.0, 10.0))
        mats = np.array([[rng.uniform(-5.0, 5.0) for _ in range(12)] for _ in range(3)])
        imgs = np.array([rng.uniform(-100.0, 100.0) for _ in range(3 * 9 * 13)],
                        dtype=np.float32).reshape(3, 9, 13)
        vol0 = np.array([rng.uniform(-100.0, 100.0) for _ in range(L ** 3)],
                        dtype=np.float32).reshape(L, L, L)
        probe = vol0.copy()
        if O.ref_reconstruct_reference(probe, g, imgs, mats) == 0:
            _save("random_w.npz", g, mats, imgs, vol0)
            break

    g = VolumeGeometry.centered(8, 1.0)
    m = np.zeros((1, 12))
    m[0, 0] = 1.0
    m[0, 4] = 1.0
    m[0, 9] = 16.0
    m[0, 10] = 16.0
    m[0, 11] = 1.0
    imgs = np.full((1, 33, 33), 0.8125, dtype=np.float32)
    _save("orthographic.npz", g, m, imgs, np.zeros((8, 8, 8), dtype=np.float32))


if __name__ == "__main__":
    main()
