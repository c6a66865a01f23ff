"""Multi-GPU z-slab reconstruction, one process per GPU (north_star (3)).

Each rank owns a contiguous range of z-planes of the volume (voxel ownership
is disjoint, every voxel keeps its projection order, so the result is
bitwise that of one GPU). Projection batches are distributed with a
broadcast over NCCL (NVLink / NVSwitch): batch b is uploaded from pinned host
memory by rank b % N only and broadcast to the others, so each GPU's PCIe
link carries 1/N of the host-to-device traffic and NVLink carries the rest.
Slabs are copied to host memory at the end (no reduction).

torch.distributed is the plumbing (process group, NCCL broadcast, streams);
the compute is the C-ABI library (pack_device / backproject_device). The
compute hooks can be replaced for host-side tests of the data flow (gloo,
CPU tensors); the product default has no CPU path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from .geometry import VolumeGeometry, validate_matrices


def equal_slabs(L: int, world: int) -> List[tuple]:
    """Planes [L*r/N, L*(r+1)/N) per rank."""
    return [(L * r // world, L * (r + 1) // world) for r in range(world)]


def plane_work(geometry: VolumeGeometry, mats: np.ndarray, width: int, height: int,
               samples: int = 16, planes_per_group: int = 8) -> np.ndarray:
    """Estimated back-projection work per z-plane: the fraction of
    (voxel, projection) pairs whose position lies in [-2, W) x [-2, H) (the
    rest is culled as exactly zero), sampled on a samples x samples grid per
    group of planes. Deterministic, float64, identical on every rank."""
    L = geometry.edge_voxels
    m = validate_matrices(mats)
    idx = np.linspace(0, L - 1, samples)
    wx = geometry.origin_mm + idx * geometry.voxel_mm
    X, Y = np.meshgrid(wx, wx, indexing="xy")
    X, Y = X.ravel(), Y.ravel()
    groups = np.arange(0, L, planes_per_group)
    work = np.zeros(L)
    for g0 in groups:
        zc = geometry.origin_mm + (g0 + (min(planes_per_group, L - g0) - 1) / 2) * geometry.voxel_mm
        u = np.outer(m[:, 0], X) + np.outer(m[:, 3], Y) + (m[:, 6] * zc + m[:, 9])[:, None]
        v = np.outer(m[:, 1], X) + np.outer(m[:, 4], Y) + (m[:, 7] * zc + m[:, 10])[:, None]
        w = np.outer(m[:, 2], X) + np.outer(m[:, 5], Y) + (m[:, 8] * zc + m[:, 11])[:, None]
        with np.errstate(divide="ignore", invalid="ignore"):
            ix, iy = u / w, v / w
        on = (ix > -2) & (ix < width) & (iy > -2) & (iy < height)
        work[g0:g0 + planes_per_group] = on.mean() + 0.05  # + fixed per-voxel overhead
    return work


def balanced_slabs(work: np.ndarray, world: int) -> List[tuple]:
    """Contiguous plane ranges with near-equal summed work (at least one
    plane each when L >= world)."""
    L = len(work)
    c = np.concatenate([[0.0], np.cumsum(work)])
    bounds = [0]
    for r in range(1, world):
        target = c[-1] * r / world
        z = int(np.searchsorted(c, target))
        z = max(bounds[-1] + 1, min(z, L - (world - r)))
        bounds.append(z)
    bounds.append(L)
    return list(zip(bounds[:-1], bounds[1:]))


def rebalance_slabs(work: np.ndarray, slabs: Sequence[tuple], seconds: Sequence[float]
                    ) -> List[tuple]:
    """One measured refinement of balanced_slabs: the estimated per-plane work
    inside each slab is rescaled so that the slab's total equals its measured
    time, then the planes are split again. Corrects what the sampled estimate
    misses (culling granularity, per-launch overheads) without a cost model."""
    w = np.asarray(work, dtype=np.float64).copy()
    for (a, b), t in zip(slabs, seconds):
        s = w[a:b].sum()
        if b > a and s > 0 and t > 0:
            w[a:b] *= float(t) / s
    return balanced_slabs(w, len(slabs))


def batch_roots(count: int, batch: int, world: int) -> List[tuple]:
    """(first, n, root) per batch: batch b is uploaded by rank b % world."""
    out = []
    for b, first in enumerate(range(0, count, batch)):
        out.append((first, min(batch, count - first), b % world))
    return out


@dataclass
class Hooks:
    """Compute hooks: pack(raw (n,H,W) full detector, packed, err),
    backproject(vol_slab, z0, z1, packed, n, mats, err), packed bytes per
    projection; check(raw, err) scans a whole uploaded batch (the uploading
    rank runs it when its own pack skips rows); for_stack(z0, z1, mats)
    returns hooks specialised to one stack (the slab's row band)."""
    pack: Callable
    backproject: Callable
    packed_bytes: int
    check: Optional[Callable] = None
    for_stack: Optional[Callable] = None


def cuda_hooks(geometry: VolumeGeometry, width: int, height: int, options=None,
               band=None) -> Hooks:
    """CUDA hooks over the C ABI. With band (RowBand), each rank packs only
    the detector rows its slab projects onto (cbb_pack_device_band) and the
    kernel reads that band; for_stack picks the band for a stack."""
    from .backproject import (backproject_device, check_finite_device, pack_device,
                              pack_device_band, packed_layout, row_band_for_slab, tma_plan)

    _, _, nb = packed_layout(width, height)

    def for_stack(z0, z1, mats, staged=True):
        # the TMA-staged raw hooks when the slab's footprint boxes fit (and
        # the batch lives in local memory: staged=False for the IPC transport,
        # whose packs read the uploader's slot over peer memory)
        b = row_band_for_slab(geometry, width, height, z0, z1, mats)
        if staged and tma_plan(geometry, width, height, z0, z1, mats)["staged"]:
            return raw_hooks(geometry, width, height, options, b, for_stack)
        return cuda_hooks(geometry, width, height, options, band=b)

    if band is None:
        def pack(raw, packed, err):
            pack_device(raw, packed)

        def back(vol_slab, z0, z1, packed, n, mats, err):
            backproject_device(vol_slab, geometry, z0, z1, packed, width, height, n, mats,
                               options, err_flag=err)

        return Hooks(pack, back, nb, None, for_stack)

    def pack_b(raw, packed, err):
        pack_device_band(raw, band, packed, err_flag=err)

    def back_b(vol_slab, z0, z1, packed, n, mats, err):
        backproject_device(vol_slab, geometry, z0, z1, packed, width, height, n, mats,
                           options, err_flag=err, band=band)

    def check(raw, err):
        check_finite_device(raw, err)

    full = band.cell_row0 == 0 and band.cell_rows == packed_layout(width, height)[1]
    return Hooks(pack_b, back_b, band.packed_bytes(width, height), None if full else check,
                 for_stack)


def raw_hooks(geometry: VolumeGeometry, width: int, height: int, options, band,
              for_stack=None) -> Hooks:
    """Hooks for the TMA-staged kernel (bp_tma.cuh): no packing. `pack` scans
    the rank's band rows of the received batch (scan_projections: the
    per-projection numerator flags, kept in the 'packed' buffer, 4 bytes per
    projection) and `backproject` reads those rows straight from the raw
    slot (a band view: rows [r0, r0 + rn) of each projection)."""
    import torch

    from .backproject import backproject_raw_device, check_finite_device, scan_device

    state = {}
    r0, rn = band.raw_row0, band.raw_rows

    def pack(raw, packed, err):
        view = raw[:, r0:r0 + rn]
        flags = packed[:4 * raw.shape[0]].view(torch.int32)
        scan_device(view, flags, err)
        state["raw"], state["flags"] = view, flags

    def back(vol_slab, z0, z1, packed, n, mats, err):
        backproject_raw_device(vol_slab, geometry, z0, z1, state["raw"], width, height, n, mats,
                               state["flags"], options, err_flag=err, band=band)

    def check(raw, err):
        check_finite_device(raw, err)

    full = r0 == 0 and rn == height
    return Hooks(pack, back, 4, None if full else check, for_stack)


class DistributedReconstructor:
    """z-slab reconstruction across the ranks of a torch.distributed group.

    reconstruct(host_imgs, mats) -> this rank's slab (host float32 array of
    shape (z1 - z0, L, L)); host_imgs needs valid data only for the batches
    this rank uploads (batch_roots)."""

    def __init__(self, geometry: VolumeGeometry, width: int, height: int, batch: int = 32,
                 slabs: Optional[Sequence[tuple]] = None, group=None, device=None,
                 hooks: Optional[Hooks] = None, options=None, slots: Optional[int] = None,
                 transport: str = "nccl"):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.geometry = geometry
        self.W, self.H = int(width), int(height)
        self.batch = int(batch)
        L = geometry.edge_voxels
        self.slabs = list(slabs) if slabs is not None else equal_slabs(L, self.world)
        assert len(self.slabs) == self.world
        self.z0, self.z1 = self.slabs[self.rank]
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.cuda = self.device.type == "cuda"
        self.hooks = hooks or cuda_hooks(geometry, width, height, options)
        nb = self.hooks.packed_bytes
        # raw slots in flight: world + 1, so the uploads of the next `world`
        # batches (each by a different rank) run concurrently instead of one
        # or two at a time -- every rank's PCIe link stays busy while NCCL
        # broadcasts and the kernels consume the batches in order
        self.nslots = max(2, int(slots) if slots else self.world + 1)
        self.raw = [torch.empty((self.batch, self.H, self.W), dtype=torch.float32,
                                device=self.device) for _ in range(self.nslots)]
        # one packed buffer: pack and back-projection of a batch are ordered on
        # the compute stream
        self.packed = torch.empty(self.batch * nb, dtype=torch.uint8, device=self.device)
        self.vol = torch.zeros(((self.z1 - self.z0), L, L), dtype=torch.float32,
                               device=self.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.copy_stream = torch.cuda.Stream(self.device) if self.cuda else None
        if transport not in ("nccl", "ipc"):
            raise ValueError("transport must be 'nccl' or 'ipc'")
        self.transport = transport
        if transport == "ipc":
            self._ipc_setup()

    # ---- transport "ipc": fused upload broadcast + pack over peer memory ----
    #
    # Each rank owns two raw slots and a flag block (uint32: ready[2], then
    # consumed[q*2 + j] for every root q and slot j) in CUDA IPC memory that
    # every other rank maps. Batch b (root q = b mod N, slot j = (b // N) mod 2):
    # q uploads it into its slot j on its copy stream once every rank flagged
    # q's upload b - 2N consumed, then flags ready; every rank's compute stream
    # waits for that flag, runs the band pack straight from q's slot (the
    # NVLink read and the layout transform are one kernel), flags it consumed
    # and back-projects. Flags carry a running batch number (never reset).
    def _ipc_setup(self):
        import ctypes as C

        from . import _lib

        if not self.cuda:
            raise ValueError("transport 'ipc' needs CUDA tensors")
        L = _lib.lib()
        per = self.batch * self.H * self.W * 4
        self._nflags = 2 + 2 * self.world
        local = []
        for size in (per, per, 4 * self._nflags):
            ptr, h = C.c_void_p(), (C.c_char * 64)()
            _lib.check(L.cbb_ipc_alloc(size, C.byref(ptr), h))
            local.append((ptr.value, bytes(h)))
        self._ipc_local = [p for p, _ in local]
        handles = [None] * self.world
        self.dist.all_gather_object(handles, [h for _, h in local], group=self.group)
        self._ipc_opened = []
        self._peer = []  # per rank: [raw0, raw1, flags] device pointers
        for r in range(self.world):
            if r == self.rank:
                self._peer.append(list(self._ipc_local))
                continue
            ptrs = []
            for h in handles[r]:
                ptr = C.c_void_p()
                _lib.check(L.cbb_ipc_open((C.c_char * 64).from_buffer_copy(h), C.byref(ptr)))
                ptrs.append(ptr.value)
                self._ipc_opened.append(ptr.value)
            self._peer.append(ptrs)
        self._epoch = 0
        self.dist.barrier(group=self.group)

    def _raw_view(self, ptr: int, n: int):
        """A (n, H, W) float32 tensor over device memory at ptr (local or mapped)."""
        import torch

        class _Arr:
            __cuda_array_interface__ = {"shape": (n, self.H, self.W), "typestr": "<f4",
                                        "data": (ptr, False), "version": 3, "strides": None}
        return torch.as_tensor(_Arr(), device=self.device)

    def _flag(self, rank: int, index: int) -> int:
        return self._peer[rank][2] + 4 * index

    def _reconstruct_ipc(self, host_imgs, m, hooks):
        import ctypes as C

        import torch

        from . import _lib

        L = _lib.lib()
        plan = batch_roots(m.shape[0], self.batch, self.world)
        cur = torch.cuda.current_stream(self.device)
        copy = self.copy_stream
        copy.wait_stream(cur)
        base = self._epoch
        for b, (first, n, q) in enumerate(plan):
            seq = base + b + 1
            j = (b // self.world) % 2
            if self.rank == q:
                if b >= 2 * self.world:  # q's upload b - 2N consumed by every rank
                    prev = base + b - 2 * self.world + 1
                    for r in range(self.world):
                        _lib.check(L.cbb_stream_wait_flag(self._flag(r, 2 + 2 * q + j), prev,
                                                          C.c_void_p(copy.cuda_stream)))
                src = host_imgs[first:first + n]
                if not isinstance(src, torch.Tensor):
                    src = torch.from_numpy(np.ascontiguousarray(src))
                with torch.cuda.stream(copy):
                    self._raw_view(self._ipc_local[j], n).copy_(src, non_blocking=True)
                _lib.check(L.cbb_stream_write_flag(self._flag(q, j), seq,
                                                   C.c_void_p(copy.cuda_stream)))
            _lib.check(L.cbb_stream_wait_flag(self._flag(q, j), seq, C.c_void_p(cur.cuda_stream)))
            raw = self._raw_view(self._peer[q][j], n)
            if q == self.rank and hooks.check is not None:
                hooks.check(raw, self.err)
            hooks.pack(raw, self.packed, self.err)
            _lib.check(L.cbb_stream_write_flag(self._flag(self.rank, 2 + 2 * q + j), seq,
                                               C.c_void_p(cur.cuda_stream)))
            hooks.backproject(self.vol, self.z0, self.z1, self.packed, n,
                              m[first:first + n], self.err)
        self._epoch += len(plan)

    def close(self):
        """Releases the IPC mappings and buffers (transport 'ipc')."""
        if getattr(self, "transport", "nccl") != "ipc" or not hasattr(self, "_ipc_local"):
            return
        from . import _lib

        import torch

        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)  # no rank still reads our slots
        L = _lib.lib()
        for p in self._ipc_opened:
            L.cbb_ipc_close(p)
        for p in self._ipc_local:
            L.cbb_ipc_free(p)
        self._ipc_opened, self._ipc_local = [], []
        self.transport = "closed"

    def _send(self, slot: int, host_imgs, first: int, n: int, root: int):
        """Root uploads batch rows [first, first+n) into raw[slot]; broadcast."""
        import torch

        buf = self.raw[slot][:n]
        if self.cuda:
            cur = torch.cuda.current_stream(self.device)
            # raw[slot] free: its last reader (the pack of batch b - nslots) is
            # already enqueued on the compute stream
            self.copy_stream.wait_stream(cur)
            with torch.cuda.stream(self.copy_stream):
                if self.rank == root:
                    src = host_imgs[first:first + n]
                    if not isinstance(src, torch.Tensor):
                        src = torch.from_numpy(np.ascontiguousarray(src))
                    buf.copy_(src, non_blocking=True)
                if self.world > 1:
                    return self.dist.broadcast(buf, src=root, group=self.group, async_op=True)
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
                return ev
        if self.rank == root:
            src = host_imgs[first:first + n]
            buf.copy_(src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src)))
        if self.world > 1:
            self.dist.broadcast(buf, src=root, group=self.group)
        return None

    def reconstruct(self, host_imgs, mats, initial_slab=None) -> np.ndarray:
        import torch

        m = validate_matrices(mats)
        count = m.shape[0]
        hooks = self.hooks
        if hooks.for_stack is not None:
            if self.transport == "ipc":
                hooks = hooks.for_stack(self.z0, self.z1, m, staged=False)
            else:
                hooks = hooks.for_stack(self.z0, self.z1, m)
            if hooks.packed_bytes > self.hooks.packed_bytes:
                raise ValueError("stack hooks need larger packed buffers")
        if initial_slab is not None:
            self.vol.copy_(torch.as_tensor(np.ascontiguousarray(initial_slab)))
        else:
            self.vol.zero_()
        self.err.zero_()
        if self.transport == "ipc":
            self._reconstruct_ipc(host_imgs, m, hooks)
            return self._finish()
        if self.transport != "nccl":
            raise RuntimeError("DistributedReconstructor is closed")
        plan = batch_roots(count, self.batch, self.world)
        depth = self.nslots - 1  # batches sent ahead of the one being computed
        pending = {}
        for b in range(min(depth, len(plan))):
            pending[b] = self._send(b % self.nslots, host_imgs, *plan[b])
        for b, (first, n, root) in enumerate(plan):
            slot = b % self.nslots
            if b + depth < len(plan):
                pending[b + depth] = self._send((b + depth) % self.nslots, host_imgs,
                                                *plan[b + depth])
            done = pending.pop(b)
            if self.cuda and done is not None:
                if isinstance(done, torch.cuda.Event):
                    torch.cuda.current_stream(self.device).wait_event(done)
                else:
                    done.wait()
            if root == self.rank and hooks.check is not None:
                hooks.check(self.raw[slot][:n], self.err)
            hooks.pack(self.raw[slot][:n], self.packed, self.err)
            hooks.backproject(self.vol, self.z0, self.z1, self.packed, n,
                              m[first:first + n], self.err)
        return self._finish()

    def _finish(self) -> np.ndarray:
        import torch

        # every rank raises the same error: OR of the flags (bit 1: w == 0,
        # bit 2: non-finite pixel) over the group
        flags = torch.stack([(self.err & 1) != 0, (self.err & 2) != 0]).to(torch.int32)
        if self.world > 1:
            self.dist.all_reduce(flags, op=self.dist.ReduceOp.MAX, group=self.group)
        flags = flags.cpu().reshape(-1).tolist()
        if flags[1]:
            from .errors import ValidationError
            raise ValidationError("ProjectionImage contains non-finite values")
        if flags[0]:
            from .errors import GeometryError
            raise GeometryError("backprojection hit a voxel with w == 0")
        out = torch.empty(self.vol.shape, dtype=torch.float32,
                          pin_memory=self.cuda)
        out.copy_(self.vol)
        return out.numpy()

    def gather(self, slab: np.ndarray, dst: int = 0) -> Optional[np.ndarray]:
        """Collects every rank's slab into the full volume on rank `dst`
        (host memory); other ranks return None."""
        import torch

        L = self.geometry.edge_voxels
        t = torch.from_numpy(np.ascontiguousarray(slab)).to(self.device)
        if self.world == 1:
            return slab
        sizes = [(z1 - z0) for z0, z1 in self.slabs]
        full = [torch.empty((s, L, L), dtype=torch.float32, device=self.device)
                for s in sizes] if self.rank == dst else None
        if self.rank == dst:
            for r in range(self.world):
                if r == dst:
                    full[r].copy_(t)
                else:
                    self.dist.recv(full[r], src=r, group=self.group)
            return torch.cat(full).cpu().numpy()
        self.dist.send(t, dst=dst, group=self.group)
        return None
