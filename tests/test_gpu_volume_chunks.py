"""GPU: the deferred initial volume of the single-GPU pipeline (pipeline.cuh,
VolChunk). With a volume to accumulate into and the whole stack known (raw
resident mode), the volume is uploaded in z-chunks interleaved with the first
batches and the head launches cover the chunks already on the device, each
catching up on the projections it missed. Every voxel still takes the
projections in stack order, so the result must be bitwise the oracle's for
any chunking, any number of chunks per batch and any tail; a non-finite voxel
in any chunk is still reported as the reference's Volume::validate error
(proj/src/dataset.cpp:146-151) with the caller's volume untouched.

Geometry as tests/test_gpu_tma.py: config 2's scan with a central 96^3
sub-cube at 0.5 mm voxels.
"""
import numpy as np
import pytest

from conftest import bits_equal

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth
from paper_1401_3615_b200.geometry import VolumeGeometry

pytestmark = pytest.mark.gpu

L = 96


@pytest.fixture(scope="module")
def scan(cuda):
    cfg = synth.CONFIGS[2]
    _, mats, imgs = synth.make_inputs(cfg, device="cuda", chunk=20, count=40)
    g = VolumeGeometry.centered(L, cfg.voxel_mm)
    return g, mats, imgs.cpu().numpy()


@pytest.fixture(scope="module")
def vol0():
    rng = np.random.default_rng(1401)
    v = rng.uniform(-2.0, 2.0, (L, L, L)).astype(np.float32)
    v[::7, 3, :] = -0.0  # -0 + +0 = +0: culling must not skip these
    return v


@pytest.fixture(scope="module")
def expected(scan, vol0, oracle):
    g, mats, host = scan
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, host, mats) == 0
    return ref


def run(g, mats, host, vol0, images=False, batch=8, **opt):
    v = vol0.copy()
    o = pkg.Options(num_gpus=1, batch=batch, **opt)
    if images:
        st = pkg.reconstruct_images(v, g, [np.array(host[i]) for i in range(len(host))], mats, o)
    else:
        st = pkg.reconstruct_arrays(v, g, host, mats, o)
    return v, st


@pytest.mark.parametrize("chunks", ["1", "3", "8", "50"])
@pytest.mark.parametrize("per_batch", ["1", "3"])
@pytest.mark.parametrize("images", [False, True])
def test_chunked_volume_bitwise(scan, vol0, expected, monkeypatch, capfd, chunks, per_batch,
                                images):
    g, mats, host = scan
    monkeypatch.setenv("CBB_VOL_CHUNKS", chunks)
    monkeypatch.setenv("CBB_VOL_PER_BATCH", per_batch)
    monkeypatch.setenv("CBB_TRACE", "1")
    v, st = run(g, mats, host, vol0, images=images)
    assert "deferred volume in" in capfd.readouterr().err
    assert st["guarded_batches"] == 0
    assert bits_equal(v, expected)


@pytest.mark.parametrize("tail", ["12:36", "36:60", "84:96"])
def test_chunked_volume_forced_tails(scan, vol0, expected, monkeypatch, tail):
    g, mats, host = scan
    monkeypatch.setenv("CBB_TAIL_PLANES", tail)
    v, _ = run(g, mats, host, vol0, batch=4)
    assert bits_equal(v, expected)


def test_chunked_volume_equals_whole_upload(scan, vol0, monkeypatch):
    g, mats, host = scan
    v1, _ = run(g, mats, host, vol0, batch=16)
    monkeypatch.setenv("CBB_NO_VOL_DEFER", "1")
    v2, _ = run(g, mats, host, vol0, batch=16)
    assert bits_equal(v1, v2)


@pytest.mark.parametrize("env", ["CBB_NO_RESIDENT", "CBB_BP_PATH"])
def test_deferred_volume_whole_upload_paths(scan, vol0, expected, monkeypatch, capfd, env):
    """Without raw resident mode (no resident stack, or the packed gather
    kernel) the deferred volume is uploaded whole before the first batch."""
    g, mats, host = scan
    monkeypatch.setenv(env, "quad" if env == "CBB_BP_PATH" else "1")
    monkeypatch.setenv("CBB_TRACE", "1")
    for images in (False, True):
        v, _ = run(g, mats, host, vol0, images=images)
        assert "deferred volume in" not in capfd.readouterr().err
        assert bits_equal(v, expected)


def test_chunked_volume_pinned_volume(scan, vol0, expected):
    """A pinned caller volume is uploaded chunk by chunk without staging."""
    import torch

    g, mats, host = scan
    t = torch.from_numpy(vol0.copy()).pin_memory()
    v = t.numpy()
    pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(num_gpus=1, batch=8))
    assert bits_equal(v, expected)


def test_chunked_volume_guarded_batch(scan, vol0, oracle):
    """A guarded batch (matrix with a -0.0 coefficient) inside the chunked
    head launches: the guarded kernel runs on the chunk ranges too."""
    g, mats, host = scan
    m = mats.copy()
    m[9, 8] = -0.0
    ref = vol0.copy()
    assert oracle.reconstruct(ref, g, host, m) == 0
    v, st = run(g, mats=m, host=host, vol0=vol0, batch=8)
    assert st["guarded_batches"] >= 1
    assert bits_equal(v, ref)


@pytest.mark.parametrize("plane", [0, 47, 95])
def test_chunked_volume_nan_rejected(scan, vol0, monkeypatch, plane):
    """A NaN voxel in the first, a middle or the last plane (head or tail
    chunk): CBB_ERR_INVALID with the reference's message, volume unchanged."""
    g, mats, host = scan
    bad = vol0.copy()
    bad[plane, 40, 50] = np.nan
    v = bad.copy()
    with pytest.raises(pkg.ValidationError, match="Volume contains non-finite"):
        pkg.reconstruct_arrays(v, g, host, mats, pkg.Options(num_gpus=1, batch=8))
    assert bits_equal(v, bad)
