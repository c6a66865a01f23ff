"""Seeded synthetic inputs standing in for the RabbitCT dataset (absent here).

The reference cannot generate BASELINE inputs (make_synthetic_stack,
proj/src/dataset.cpp:359-371, copies one analytic field to every projection
and ignores its seed). This generator produces, for BASELINE.json configs 0-4:

  * matrices: make_circular_trajectory (proj/src/geometry.cpp:79-116, angles
    range*i/N) followed by a seeded rigid perturbation per projection
    (translation U(-0.5, 0.5) mm and rotation U(-0.2, 0.2) deg per axis,
    applied to the world point before projection, i.e. to the extrinsics of
    K[R|t]), renormalised so that w(0,0,0) == 1 (geometry.hpp:54-57);
  * projections: analytic line integrals of seeded random ellipsoids (centres
    uniform in a 100 mm ball, semi-axes U(10, 80) mm, densities U(-0.5, 1.0),
    orientation a seeded random rotation R_z R_y R_x with angles U(0, 2pi)),
    ray from the source C = -M3^-1 m4 through each pixel centre, then a
    row-wise Shepp-Logan ramp filter h[n] = -2 / (pi^2 tau (4 n^2 - 1)),
    tau = detector pixel pitch in mm, applied as a linear convolution by a
    zero-padded float64 FFT of length >= 2W, rounded to float32.

Randomness comes from a self-contained splitmix64 stream (portable; no
library distribution objects), one fixed seed per config. Computation is
float64 torch on the requested device (CPU for test fixtures, CUDA in the
bench); the oracle and the GPU path always consume the same float32 bytes.
This is input generation, not part of the timed hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .geometry import TrajectoryConfig, VolumeGeometry, make_circular_trajectory

_MASK = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014): x += 0x9E3779B97F4A7C15, then mix."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float, hi: float) -> float:
        """lo + (hi - lo) * u, u = top 53 bits / 2^53 in [0, 1)."""
        return lo + (hi - lo) * ((self.next_u64() >> 11) * (1.0 / 9007199254740992.0))


@dataclass(frozen=True)
class ScanConfig:
    name: str
    edge_voxels: int
    voxel_mm: float
    num_projections: int
    width: int
    height: int
    pixel_mm: float
    sid_mm: float
    sdd_mm: float
    range_deg: float
    ellipsoids: int
    seed: int
    max_trans_mm: float = 0.5
    max_rot_deg: float = 0.2

    @property
    def geometry(self) -> VolumeGeometry:
        return VolumeGeometry.centered(self.edge_voxels, self.voxel_mm)

    @property
    def trajectory(self) -> TrajectoryConfig:
        return TrajectoryConfig(self.num_projections, self.sid_mm, self.sdd_mm, self.width,
                                self.height, self.pixel_mm, math.radians(self.range_deg))

    @property
    def voxel_updates(self) -> int:
        return self.edge_voxels ** 3 * self.num_projections


_SEED_SHORT = 0x1401_3615_0000_0001  # configs 0-3 share projections
_SEED_FULL = 0x1401_3615_0000_0004

# BASELINE.json configs (the 256 mm cube is kept: voxel_mm = 256 / L).
CONFIGS = {
    0: ScanConfig("c0_128", 128, 2.0, 496, 1248, 960, 0.32, 750.0, 1200.0, 200.0, 10, _SEED_SHORT),
    1: ScanConfig("c1_256", 256, 1.0, 496, 1248, 960, 0.32, 750.0, 1200.0, 200.0, 10, _SEED_SHORT),
    2: ScanConfig("c2_512", 512, 0.5, 496, 1248, 960, 0.32, 750.0, 1200.0, 200.0, 10, _SEED_SHORT),
    3: ScanConfig("c3_1024", 1024, 0.25, 496, 1248, 960, 0.32, 750.0, 1200.0, 200.0, 10, _SEED_SHORT),
    4: ScanConfig("c4_1024_360", 1024, 0.25, 1440, 1536, 1536, 0.2, 1000.0, 1500.0, 360.0, 30,
                  _SEED_FULL),
}


def shrunk(cfg: ScanConfig, edge_voxels: int = None, num_projections: int = None,
           width: int = None, height: int = None) -> ScanConfig:
    """Same scan with a smaller volume (same 256 mm cube), fewer projections
    (same angular range) and/or a smaller detector (pixel pitch scaled so the
    detector keeps its physical size)."""
    kw = {}
    if edge_voxels is not None:
        kw["edge_voxels"] = edge_voxels
        kw["voxel_mm"] = cfg.edge_voxels * cfg.voxel_mm / edge_voxels
    if num_projections is not None:
        kw["num_projections"] = num_projections
    if width is not None:
        kw["width"] = width
        kw["pixel_mm"] = cfg.pixel_mm * cfg.width / width
    if height is not None:
        kw["height"] = height
    return replace(cfg, name=cfg.name + "_mini", **kw)


def _rot(rx: float, ry: float, rz: float) -> np.ndarray:
    cx, sx, cy, sy, cz, sz = (math.cos(rx), math.sin(rx), math.cos(ry), math.sin(ry),
                              math.cos(rz), math.sin(rz))
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def to_3x4(a: np.ndarray) -> np.ndarray:
    """Column-major 12-vector -> 3x4 (row = u, v, w)."""
    return np.asarray(a, dtype=np.float64).reshape(4, 3).T.copy()


def from_3x4(M: np.ndarray) -> np.ndarray:
    return np.asarray(M, dtype=np.float64).T.reshape(12).copy()


def perturbed_matrices(cfg: ScanConfig) -> np.ndarray:
    """Circular trajectory + seeded rigid perturbation, renormalised w(0)=1."""
    base = make_circular_trajectory(cfg.trajectory)
    rng = SplitMix64(cfg.seed ^ 0x5EED_0F_3A7)
    out = np.empty_like(base)
    rmax = math.radians(cfg.max_rot_deg)
    for i in range(base.shape[0]):
        dt = np.array([rng.uniform(-cfg.max_trans_mm, cfg.max_trans_mm) for _ in range(3)])
        ang = [rng.uniform(-rmax, rmax) for _ in range(3)]
        M = to_3x4(base[i])
        P = np.empty((3, 4))
        P[:, :3] = M[:, :3] @ _rot(*ang)
        P[:, 3] = M[:, :3] @ dt + M[:, 3]
        P /= P[2, 3]
        out[i] = from_3x4(P)
    return out


@dataclass(frozen=True)
class Ellipsoid:
    centre: tuple
    semi_axes: tuple
    density: float
    rotation: tuple  # 3x3 row-major, columns are the body axes


def phantom(cfg: ScanConfig) -> list:
    rng = SplitMix64(cfg.seed ^ 0xE11_1950)
    out = []
    for _ in range(cfg.ellipsoids):
        while True:
            c = [rng.uniform(-100.0, 100.0) for _ in range(3)]
            if c[0] ** 2 + c[1] ** 2 + c[2] ** 2 <= 100.0 ** 2:
                break
        s = [rng.uniform(10.0, 80.0) for _ in range(3)]
        d = rng.uniform(-0.5, 1.0)
        R = _rot(*[rng.uniform(0.0, 2.0 * math.pi) for _ in range(3)])
        out.append(Ellipsoid(tuple(c), tuple(s), d, tuple(R.reshape(-1))))
    return out


def line_integrals(mats: np.ndarray, width: int, height: int, ellipsoids: list, device="cpu",
                   chunk: int = 8):
    """float64 torch tensor (N, H, W): sum over ellipsoids of density x chord."""
    import torch

    dev = torch.device(device)
    f64 = torch.float64
    N = mats.shape[0]
    out = torch.empty((N, height, width), dtype=f64, device=dev)
    iy, ix = torch.meshgrid(torch.arange(height, dtype=f64, device=dev),
                            torch.arange(width, dtype=f64, device=dev), indexing="ij")
    pix = torch.stack([ix, iy, torch.ones_like(ix)], dim=-1)  # (H, W, 3)
    E = [(torch.tensor(e.centre, dtype=f64, device=dev),
          torch.tensor(e.semi_axes, dtype=f64, device=dev),
          float(e.density),
          torch.tensor(e.rotation, dtype=f64, device=dev).reshape(3, 3)) for e in ellipsoids]
    for p0 in range(0, N, chunk):
        p1 = min(N, p0 + chunk)
        Minv = []
        src = []
        for i in range(p0, p1):
            M = to_3x4(mats[i])
            Ai = np.linalg.inv(M[:, :3])
            Minv.append(Ai)
            src.append(-Ai @ M[:, 3])
        Minv = torch.tensor(np.stack(Minv), dtype=f64, device=dev)   # (n, 3, 3)
        C = torch.tensor(np.stack(src), dtype=f64, device=dev)       # (n, 3)
        d = torch.einsum("nij,hwj->nhwi", Minv, pix)                 # (n, H, W, 3)
        d = d / torch.linalg.vector_norm(d, dim=-1, keepdim=True)
        acc = torch.zeros((p1 - p0, height, width), dtype=f64, device=dev)
        for c, s, dens, R in E:
            # body coordinates y = diag(1/s) R^T (x - c)
            T = R.T / s[:, None]
            y0 = (T @ (C - c).T).T                                   # (n, 3)
            y1 = torch.einsum("ij,nhwj->nhwi", T, d)                 # (n, H, W, 3)
            a = (y1 * y1).sum(-1)
            b = 2.0 * (y1 * y0[:, None, None, :]).sum(-1)
            cc = (y0 * y0).sum(-1) - 1.0
            disc = b * b - 4.0 * a * cc[:, None, None]
            chord = torch.sqrt(torch.clamp(disc, min=0.0)) / a
            acc += dens * chord
        out[p0:p1] = acc
    return out


def ramp_filter(proj, pixel_mm: float):
    """Row-wise Shepp-Logan ramp filter (linear convolution, float64 FFT)."""
    import torch

    W = proj.shape[-1]
    nfft = 1
    while nfft < 2 * W:
        nfft *= 2
    n = torch.arange(nfft, device=proj.device, dtype=torch.float64)
    n = torch.where(n <= nfft // 2, n, n - nfft)
    h = -2.0 / (math.pi ** 2 * pixel_mm * (4.0 * n * n - 1.0))
    H = torch.fft.rfft(h)
    P = torch.fft.rfft(proj, n=nfft, dim=-1)
    return torch.fft.irfft(P * H, n=nfft, dim=-1)[..., :W]


def make_inputs(cfg: ScanConfig, device="cpu", out_device=None, chunk: int = 8,
                count: int = None, pin: bool = False, filtered: bool = True):
    """(geometry, matrices (n,12) float64 numpy, images float32 torch (n,H,W)).

    Images are produced chunk-wise on `device` and stored on `out_device`
    (default: same device). `count` keeps only the first projections of the
    scan (same bytes as the full scan's first `count`); `pin` places CPU
    output in page-locked memory; filtered=False returns the raw line
    integrals (rounded to float32) for the GPU FDK filter stage."""
    import torch

    n = cfg.num_projections if count is None else min(int(count), cfg.num_projections)
    mats = perturbed_matrices(cfg)[:n]
    ells = phantom(cfg)
    out_device = out_device or device
    imgs = torch.empty((n, cfg.height, cfg.width), dtype=torch.float32, device=out_device,
                       pin_memory=bool(pin and torch.device(out_device).type == "cpu"))
    for p0 in range(0, n, chunk):
        p1 = min(n, p0 + chunk)
        li = line_integrals(mats[p0:p1], cfg.width, cfg.height, ells, device=device, chunk=chunk)
        f = ramp_filter(li, cfg.pixel_mm) if filtered else li
        imgs[p0:p1] = f.to(torch.float32).to(out_device)
        del li
    return cfg.geometry, mats, imgs
