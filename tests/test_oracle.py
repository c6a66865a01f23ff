"""CPU: pins the oracle (oracle/fdk_oracle.c) to the reference's own known
answers and, where oracle/_ref was built from /root/reference, to the
reference implementation itself. Restates proj/tests/test_kernel_ref.cpp."""
import math

import numpy as np
import pytest

from conftest import bits_equal, load_golden


def index_image_4x4():
    return np.arange(16, dtype=np.float32).reshape(4, 4)


def test_golden_hash(oracle):
    # proj/tests/test_kernel_ref.cpp:236-269
    g, mats, imgs = oracle.golden_case()
    vol = np.zeros((64, 64, 64), np.float32)
    assert oracle.reconstruct(vol, g, imgs, mats, threads=4) == 0
    assert oracle.fnv1a64(vol) == oracle.GOLDEN_HASH


def test_sampler_hand_examples(oracle):
    # proj/tests/test_kernel_ref.cpp:42-49
    img = index_image_4x4()
    assert oracle.sample(img, 2.0, 3.0) == 14.0
    assert oracle.sample(img, 1.5, 2.5) == 11.5
    assert oracle.sample(img, -10.2, -10.2) == 0.0
    assert oracle.sample(img, 100.0, 1.0) == 0.0
    assert oracle.sample(img, 5.0e9, 1.0) == 0.0


def test_sampler_truncation_band(oracle):
    # C truncation toward zero: (-1, 0) samples taps 0/1 with a negative
    # fraction (extrapolation), (-2, -1] touches tap 0 only through x+1.
    img = np.full((4, 4), 2.0, np.float32)
    v = oracle.sample(img, -0.5, 1.0)
    sx = np.float32(-0.5)
    expect = np.float32(np.float32(1) - sx) * np.float32(2.0) + sx * np.float32(2.0)
    assert v == expect
    # (-1.5): iix = -1, taps -1 (zero) and 0 (2.0), sx = -0.5
    v = oracle.sample(img, -1.5, 1.0)
    expect = np.float32(np.float32(1.5) * np.float32(0.0)) + np.float32(-0.5) * np.float32(2.0)
    assert v == expect


def test_orthographic_constant_adds_exactly(oracle):
    # proj/tests/test_kernel_ref.cpp:137-155
    g, mats, imgs, vol0, expected = load_golden("orthographic.npz")
    vol = vol0.copy()
    assert oracle.reconstruct(vol, g, imgs, mats) == 0
    assert np.all(vol == np.float32(0.8125))
    assert bits_equal(vol, expected)


def test_zero_image_leaves_volume(oracle):
    # proj/tests/test_kernel_ref.cpp:117-135
    from paper_1401_3615_b200.geometry import VolumeGeometry

    g = VolumeGeometry.centered(8, 1.0)
    vol = np.arange(512, dtype=np.float32).reshape(8, 8, 8)
    before = vol.copy()
    m = np.zeros(12)
    m[0] = m[4] = 1.0
    m[9] = m[10] = 8.0
    m[11] = 1.0
    assert oracle.reconstruct(vol, g, np.zeros((1, 16, 16), np.float32), m) == 0
    assert bits_equal(vol, before)


def test_w_zero_is_a_geometry_error(oracle):
    # proj/tests/test_kernel_ref.cpp:224-234
    from paper_1401_3615_b200.geometry import VolumeGeometry

    g = VolumeGeometry.centered(4, 1.0)
    m = np.zeros(12)
    m[0] = m[4] = 1.0
    assert oracle.reconstruct(np.zeros((4, 4, 4), np.float32), g,
                              np.ones((1, 8, 8), np.float32), m) == 5


@pytest.mark.parametrize("name", ["mini_c0.npz", "random_w.npz", "orthographic.npz"])
def test_oracle_reproduces_reference_fixtures(oracle, name):
    """Fixtures hold volumes produced by the reference's reconstruct_reference."""
    g, mats, imgs, vol0, expected = load_golden(name)
    vol = vol0.copy()
    assert oracle.reconstruct(vol, g, imgs, mats, threads=3) == 0
    assert bits_equal(vol, expected)


def test_slab_oracle_matches_full(oracle):
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    L = g.edge_voxels
    slab = vol0[5:11].copy()
    assert oracle.reconstruct_slab(slab, g, 5, 11, imgs, mats, threads=4) == 0
    assert bits_equal(slab, expected[5:11])


def test_additivity_bitwise(oracle):
    # proj/tests/test_kernel_ref.cpp:190-222
    g, mats, imgs, vol0, _ = load_golden("mini_c0.npz")
    whole = vol0.copy()
    oracle.reconstruct(whole, g, imgs, mats)
    split = vol0.copy()
    oracle.reconstruct(split, g, imgs[:2], mats[:2])
    oracle.reconstruct(split, g, imgs[2:], mats[2:])
    assert bits_equal(whole, split)


needs_ref = pytest.mark.skipif(
    not __import__("oracle").ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
def test_reference_golden_hash(oracle):
    g, mats, imgs = oracle.golden_case()
    vol = np.zeros((64, 64, 64), np.float32)
    assert oracle.ref_reconstruct_reference(vol, g, imgs, mats) == 0
    assert oracle.fnv1a64(vol) == oracle.GOLDEN_HASH


@needs_ref
def test_oracle_equals_reference_on_seeded_random_stacks(oracle):
    from paper_1401_3615_b200.geometry import VolumeGeometry
    from paper_1401_3615_b200.synth import SplitMix64

    rng = SplitMix64(99)
    for trial in range(12):
        L = 1 + int(rng.uniform(0, 9))
        g = VolumeGeometry(L, rng.uniform(0.1, 2.0), rng.uniform(-10.0, 10.0))
        n = 1 + int(rng.uniform(0, 3))
        W = 1 + int(rng.uniform(0, 12))
        H = 1 + int(rng.uniform(0, 12))
        mats = np.array([[rng.uniform(-5, 5) for _ in range(12)] for _ in range(n)])
        imgs = np.array([rng.uniform(-100, 100) for _ in range(n * H * W)],
                        np.float32).reshape(n, H, W)
        vol0 = np.array([rng.uniform(-100, 100) for _ in range(L ** 3)],
                        np.float32).reshape(L, L, L)
        a, b = vol0.copy(), vol0.copy()
        sa = oracle.reconstruct(a, g, imgs, mats, threads=2)
        sb = oracle.ref_reconstruct_reference(b, g, imgs, mats)
        assert sa == sb
        if sa == 0:
            assert bits_equal(a, b)


@needs_ref
def test_sampler_equals_reference(oracle):
    from paper_1401_3615_b200.synth import SplitMix64

    rng = SplitMix64(5)
    img = np.array([rng.uniform(-10, 10) for _ in range(13 * 9)], np.float32).reshape(9, 13)
    for _ in range(3000):
        ix = np.float32(rng.uniform(-4.0, 17.0))
        iy = np.float32(rng.uniform(-4.0, 13.0))
        a = oracle.sample(img, float(ix), float(iy))
        b = oracle.ref_sample(img, float(ix), float(iy))
        assert np.float32(a).view(np.uint32) == np.float32(b).view(np.uint32)


@needs_ref
def test_trajectory_equals_reference(oracle):
    from paper_1401_3615_b200.geometry import TrajectoryConfig, make_circular_trajectory

    for cfg in (TrajectoryConfig(17, 750.0, 1200.0, 1248, 960, 0.32, math.radians(200.0)),
                TrajectoryConfig(5, 1000.0, 1500.0, 1536, 1536, 0.2)):
        assert np.array_equal(make_circular_trajectory(cfg), oracle.ref_trajectory(cfg))


@needs_ref
def test_reference_optimized_degenerate_options_are_the_reference(oracle):
    """proj/tests/test_kernel_opt.cpp:384-398 restated: reconstruct_optimized
    with lanes 1, one worker, no clip, no pad is bitwise reconstruct_reference
    (the CPU baseline's code path, run here from oracle/_ref)."""
    g, mats, imgs = oracle.golden_case()
    a = np.zeros((64,) * 3, np.float32)
    b = np.zeros((64,) * 3, np.float32)
    assert oracle.ref_reconstruct_reference(a, g, imgs, mats) == 0
    st = oracle.ref_reconstruct_optimized(b, g, imgs, mats, lanes=1, chunk=262, workers=1,
                                          use_clip=False, use_pad=False)
    assert st["status"] == 0
    assert bits_equal(a, b)


def test_planes_oracle_equals_full_reconstruction_and_caches(oracle, tmp_path, monkeypatch):
    """oracle_reconstruct_planes (cache-tiled, dynamic threads; used for the
    headline-size parity tests and bench.py's parity block) gives the same
    bits as the reference-order oracle for any plane list, including w == 0
    errors; the hash-keyed cache returns the same planes without recomputing
    (proj/src/bench.cpp:194-214)."""
    g, mats, imgs, vol0, expected = load_golden("mini_c0.npz")
    L = g.edge_voxels
    full = np.zeros((L, L, L), np.float32)
    assert oracle.reconstruct(full, g, imgs, mats) == 0
    for planes in ([0], [L - 1, 0, 3], list(range(L))):
        for threads in (1, 3):
            out = np.zeros((len(planes), L, L), np.float32)
            assert oracle.reconstruct_planes(out, g, planes, imgs, mats, threads=threads) == 0
            assert bits_equal(out, full[planes])
    monkeypatch.setenv("CBB_ORACLE_CACHE", str(tmp_path))
    a, secs_a, hit_a = oracle.reference_planes(g, [1, 2], imgs, mats)
    b, secs_b, hit_b = oracle.reference_planes(g, [1, 2], imgs, mats)
    assert not hit_a and hit_b and secs_b == 0.0
    assert bits_equal(a, full[[1, 2]]) and bits_equal(b, a)
    imgs2 = imgs.copy()
    imgs2[0, 0, 0] += 1.0  # different content, different key
    c, _, hit_c = oracle.reference_planes(g, [1, 2], imgs2, mats)
    assert not hit_c
    # w == 0 is reported as the geometry error (status 5)
    bad = np.zeros((1, 12))
    bad[0, 0] = bad[0, 4] = 1.0
    out = np.zeros((1, L, L), np.float32)
    assert oracle.reconstruct_planes(out, g, [0], imgs[:1], bad) == 5


def test_content_hash_is_chunked_and_deterministic(oracle):
    a = np.arange(3_000_001, dtype=np.float32)
    h = oracle.content_hash(a)
    assert h == oracle.content_hash(a.copy())
    b = a.copy()
    b[-1] += 1
    assert oracle.content_hash(b) != h
    assert oracle.content_hash(a[:-1]) != h
