"""GPU: the FDK filtering step -- row-wise Shepp-Logan
ramp filter on the device, checked against an independent numpy float64
FFT convolution, and the filtered reconstruction pipeline
(cbb_options.ramp_filter) against back-projecting host-filtered data."""
import math

import numpy as np
import pytest

import paper_1401_3615_b200 as pkg
from paper_1401_3615_b200 import synth

pytestmark = pytest.mark.gpu


def numpy_ramp(rows: np.ndarray, tau: float) -> np.ndarray:
    """h[n] = -2/(pi^2 tau (4n^2-1)), linear convolution, float64, -> float32."""
    W = rows.shape[-1]
    nfft = 1
    while nfft < 2 * W:
        nfft *= 2
    n = np.arange(nfft, dtype=np.float64)
    n = np.where(n <= nfft // 2, n, n - nfft)
    h = -2.0 / (math.pi ** 2 * tau * (4.0 * n * n - 1.0))
    out = np.fft.irfft(np.fft.rfft(rows.astype(np.float64), n=nfft) * np.fft.rfft(h), n=nfft)
    return out[..., :W].astype(np.float32)


def small_scan():
    cfg = synth.shrunk(synth.CONFIGS[0], edge_voxels=24, num_projections=6, width=156,
                       height=120)
    mats = synth.perturbed_matrices(cfg)
    li = synth.line_integrals(mats, cfg.width, cfg.height, synth.phantom(cfg)).numpy()
    return cfg, mats, li.astype(np.float32)


def test_ramp_filter_matches_numpy(cuda):
    import torch

    cfg, mats, raw = small_scan()
    ref = numpy_ramp(raw, cfg.pixel_mm)
    t = torch.from_numpy(raw).cuda()
    out = torch.empty_like(t)
    pkg.ramp_filter_device(t, out, cfg.pixel_mm)
    got = out.cpu().numpy()
    scale = float(np.abs(ref).max())
    assert np.abs(got - ref).max() <= 1e-6 * scale
    assert np.mean(got == ref) > 0.99  # float64 FFT differences rarely change the float32 rounding
    # in place
    pkg.ramp_filter_device(t, t, cfg.pixel_mm)
    assert np.array_equal(t.cpu().numpy(), got)


@pytest.mark.parametrize("width,rows", [(1248, 7), (1536, 6), (2048, 3), (2049, 3), (5, 9),
                                        (1, 4)])
def test_fused_fft_filter_widths_and_odd_row_counts(cuda, width, rows):
    """The fused shared-memory FFT kernel (ramp_fft.cuh: row pairs as one
    complex N = 4096 transform, W <= 2048) and the cuFFT path beyond it,
    against numpy float64 at the BASELINE detector widths (1248, 1536), the
    fused kernel's limit, an odd number of rows (last pair half empty) and
    degenerate widths; in place as well."""
    import torch

    r = np.random.default_rng(width * 31 + rows)
    raw = (r.standard_normal((1, rows, width)) * 50).astype(np.float32)
    raw[0, 0, :] = 0.0
    raw[0, -1, : min(width, 7)] = 1e3
    tau = 0.2 if width % 2 == 0 else 0.32
    ref = numpy_ramp(raw, tau)
    t = torch.from_numpy(raw).cuda()
    out = torch.empty_like(t)
    pkg.ramp_filter_device(t, out, tau)
    got = out.cpu().numpy()
    scale = float(np.abs(ref).max())
    assert np.abs(got - ref).max() <= 1e-6 * scale
    # rows travel in pairs through one complex transform: a row of zeros
    # picks up float64 round-off of its partner (~1e-16 of it), not exact 0
    zero = ~raw.any(axis=-1)
    assert np.abs(got[zero]).max(initial=0.0) <= 1e-12 * scale
    assert np.mean(got[~zero] == ref[~zero]) > 0.99
    pkg.ramp_filter_device(t, t, tau)
    assert np.array_equal(t.cpu().numpy(), got)


def test_compare_volumes_device_matches_numpy(cuda):
    """GPU volume metrics vs the reference harness definitions
    (proj/src/bench.cpp:65-102) computed in numpy float64."""
    import torch

    r = np.random.default_rng(3)
    ref = r.standard_normal(100003).astype(np.float32)
    test = (ref + r.standard_normal(ref.size).astype(np.float32) * 1e-3).astype(np.float32)
    test[::7] = ref[::7]
    got = pkg.compare_volumes_device(torch.from_numpy(test).cuda(), torch.from_numpy(ref).cuda(),
                                     denom_floor=1e-6)
    d = test.astype(np.float64) - ref
    mse = np.mean(d * d)
    assert got["mse"] == pytest.approx(mse, rel=1e-12)
    assert got["psnr_db"] == pytest.approx(10 * np.log10(float(ref.max()) ** 2 / mse), rel=1e-12)
    assert got["max_relative_error"] == pytest.approx(
        np.max(np.abs(d) / (np.abs(ref.astype(np.float64)) + 1e-6)), rel=1e-12)
    assert got["rel_l2"] == pytest.approx(np.linalg.norm(d) / np.linalg.norm(ref.astype(np.float64)),
                                          rel=1e-9)
    assert got["max_abs_over_range"] == pytest.approx(
        np.abs(d).max() / (float(ref.max()) - float(ref.min())), rel=1e-12)
    assert got["bitwise_different"] == int(np.sum(test.view(np.uint32) != ref.view(np.uint32)))
    same = pkg.compare_volumes_device(torch.from_numpy(ref).cuda(), torch.from_numpy(ref).cuda())
    assert same["bitwise_different"] == 0 and same["mse"] == 0 and same["psnr_db"] == float("inf")


def test_filtered_pipeline_equals_backprojecting_filtered_data(cuda, oracle):
    import torch

    cfg, mats, raw = small_scan()
    g = cfg.geometry
    t = torch.from_numpy(raw).cuda()
    filt = torch.empty_like(t)
    pkg.ramp_filter_device(t, filt, cfg.pixel_mm)
    filtered = filt.cpu().numpy()
    # reference: the oracle back-projects the device-filtered projections
    ref = np.zeros((g.edge_voxels,) * 3, np.float32)
    assert oracle.reconstruct(ref, g, filtered, mats) == 0
    vol = pkg.Volume(g)
    pkg.reconstruct(vol, pkg.ProjectionStack(g, mats, raw),
                    pkg.Options(ramp_filter_pixel_mm=cfg.pixel_mm, batch=4))
    assert np.array_equal(vol.voxels.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("width,rows", [(1248, 9600), (1248, 7), (977, 301), (1280, 64), (5, 9)])
def test_ramp_2560_kernel_thread_layouts_bitwise(cuda, monkeypatch, width, rows):
    """The N = 2560 filter in 160-thread CTAs (ramp_fft2560_rows160, the
    default: every thread busy in the radix-16 passes, 3 CTAs/SM) performs the
    same operations as the 256-thread kernel (CBB_RAMP_256), so the same bits
    -- over many grid-stride iterations (9600 rows) and odd row counts."""
    import torch

    r = np.random.default_rng(width + rows)
    raw = torch.from_numpy((r.standard_normal((1, rows, width)) * 30).astype(np.float32)).cuda()
    a = torch.empty_like(raw)
    b = torch.empty_like(raw)
    pkg.ramp_filter_device(raw, a, 0.32)
    monkeypatch.setenv("CBB_RAMP_256", "1")
    pkg.ramp_filter_device(raw, b, 0.32)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
