"""z-slab sharding of the volume across ranks (one process per GPU).

Rank r owns global planes [owned_begin, owned_end) and stores [alloc_begin, alloc_end): the
owned planes plus `ghost` = fill_radius + median_radius planes on each side, so the hole fill
and the 5x5-median render of every owned column see exactly the voxels the unsharded volume
would.  A frame is routed to every rank whose stored planes its conservative
voxel box meets; each rank inserts independently (integer sums, no exchange).  The only
collective is the gather of the rendered coronal rows (NCCL all-gather over NVLink on GPUs,
gloo in the CPU tests).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi


@dataclass
class Slab:
    owned: tuple
    alloc: tuple


def plan_slabs(nz: int, nranks: int, ghost: int):
    """Contiguous near-equal z-slabs (svr_plan_slabs)."""
    ob, oe, ab, ae = ((_abi.I32 * nranks)() for _ in range(4))
    _abi.check(_abi.lib().svr_plan_slabs(nz, nranks, ghost, ob, oe, ab, ae))
    return [Slab((ob[r], oe[r]), (ab[r], ae[r])) for r in range(nranks)]


def frame_boxes(desc: _abi.GridDesc, calib: _abi.Calib, poses) -> list:
    """Conservative global voxel box of every frame (svr_frame_bounds, host only)."""
    pa = _abi.rigid_array(poses)
    out = []
    for k in range(len(pa)):
        b = _abi.Box()
        _abi.check(_abi.lib().svr_frame_bounds(C.byref(desc), C.byref(calib),
                                               _abi.rigid_ptr(pa[k:k + 1]), C.byref(b)))
        out.append(b)
    return out


def route(boxes, alloc) -> np.ndarray:
    """Indices of the frames whose box meets the stored planes [alloc0, alloc1)."""
    return np.array([k for k, b in enumerate(boxes)
                     if not b.empty() and b.z1 >= alloc[0] and b.z0 < alloc[1]], dtype=np.int64)


def union_box(boxes, idx, alloc) -> _abi.Box:
    """Union of the routed frames' boxes clipped to the stored planes (empty if none)."""
    if len(idx) == 0:
        return _abi.Box(1, 1, 1, 0, 0, 0)
    bs = [boxes[int(k)] for k in idx]
    z0 = max(min(b.z0 for b in bs), alloc[0])
    z1 = min(max(b.z1 for b in bs), alloc[1] - 1)
    if z0 > z1:
        return _abi.Box(1, 1, 1, 0, 0, 0)
    return _abi.Box(min(b.x0 for b in bs), min(b.y0 for b in bs), z0, max(b.x1 for b in bs),
                    max(b.y1 for b in bs), z1)


class ShardedGrid:
    """z-slab sharded volume driven from one process over several devices through the C-ABI
    (svr_sharded_*): the path a C / C++ caller takes without torch.distributed.  devices may
    repeat (several slabs on one GPU).  Results equal one unsharded VoxelGrid bit for bit."""

    def __init__(self, dims, voxel_mm, origin=(0.0, 0.0, 0.0), devices=(0,), ghost=3,
                 accum=_abi.ACC_PNN):
        d = _abi.GridDesc()
        d.nx, d.ny, d.nz = (int(v) for v in dims)
        d.accum = accum
        d.voxel_mm = float(voxel_mm)
        for k in range(3):
            d.origin_mm[k] = float(origin[k])
        d.z_begin, d.z_end = 0, d.nz
        self.desc = d
        devs = (_abi.I32 * len(devices))(*devices)
        h = C.c_void_p()
        _abi.check(_abi.lib().svr_sharded_create(C.byref(self.desc), devs, len(devices), ghost, C.byref(h)))
        self._h = h
        self.n = len(devices)

    def close(self):
        if self._h:
            _abi.lib().svr_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def slab(self, r):
        """(volume handle, owned (z0, z1), stored (z0, z1)) of slab r."""
        v = C.c_void_p()
        o0, o1, a0, a1 = (_abi.I32() for _ in range(4))
        _abi.check(_abi.lib().svr_sharded_slab(self._h, r, C.byref(v), C.byref(o0), C.byref(o1),
                                               C.byref(a0), C.byref(a1)))
        return v, (o0.value, o1.value), (a0.value, a1.value)

    def insert_frames(self, frames, poses, calib):
        from .reconstruct import _frames_view
        keep, p, pitch, stride, n, h, w = _frames_view(frames)
        pa = _abi.rigid_array(poses)
        routed = (_abi.I32 * self.n)()
        _abi.check(_abi.lib().svr_sharded_insert_frames(self._h, p, pitch, stride, w, h, n,
                                                        _abi.rigid_ptr(pa), C.byref(calib), 0, routed))
        _abi.check(_abi.lib().svr_sharded_sync(self._h))
        del keep
        return list(routed)

    def fill_render(self, fill_radius, fill_mode, params):
        _abi.check(_abi.lib().svr_sharded_fill_render(self._h, fill_radius, fill_mode, C.byref(params)))

    def read_coronal(self):
        nz, nx = self.desc.nz, self.desc.nx
        mean = np.zeros((nz, nx), np.float32)
        mx = np.zeros((nz, nx), np.float32)
        dep = np.full((nz, nx), -1, np.int32)
        _abi.check(_abi.lib().svr_sharded_read_coronal(self._h, mean.ctypes.data, mx.ctypes.data,
                                                       dep.ctypes.data))
        return mean, mx, dep

    def accumulators(self, r):
        """Owned planes of slab r: (sum u32, count u16) [z, y, x]."""
        v, own, _ = self.slab(r)
        nx, ny = self.desc.nx, self.desc.ny
        nz = own[1] - own[0]
        s = np.zeros((nz, ny, nx), np.uint32)
        c = np.zeros((nz, ny, nx), np.uint16)
        if nz:
            b = _abi.Box(0, 0, own[0], nx - 1, ny - 1, own[1] - 1)
            _abi.check(_abi.lib().svr_read_accumulators(v, C.byref(b), s.ctypes.data, c.ctypes.data))
        return s, c


def gather_rows(local, slab: Slab, slabs, dist):
    """All-gather each rank's owned coronal rows (torch tensor [owned_rows, ...]) into the full
    image [nz, ...] (padded equal strips, one all_gather_into_tensor).  Returns the image."""
    import torch
    rows_max = max(s.owned[1] - s.owned[0] for s in slabs)
    world = len(slabs)
    pad = torch.zeros((rows_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if local.device.type == "cuda":
        buf = torch.empty((world * rows_max,) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        dist.all_gather_into_tensor(buf, pad)
    else:  # gloo
        lst = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(lst, pad)
        buf = torch.cat(lst, 0)
    parts = [buf[r * rows_max: r * rows_max + (slabs[r].owned[1] - slabs[r].owned[0])] for r in range(world)]
    return torch.cat(parts, 0)


def chunk_boxes(boxes, idx, alloc, chunk: int = 32, dilate: int = 0):
    """Dirty region of a batch as non-overlapping per-z-chunk boxes: for every chunk of `chunk`
    planes of the stored slab, the bounding box of the routed frames' boxes (each dilated by
    `dilate`) that meet it, clipped to the chunk.  Much tighter than one bounding box for a
    sweep that drifts laterally; fill/render over it give the same result (every non-empty
    voxel and every voxel within `dilate` of one lies inside)."""
    out = []
    if len(idx) == 0:
        return out
    bs = [boxes[int(k)] for k in idx if not boxes[int(k)].empty()]
    d = dilate
    for z0 in range(alloc[0], alloc[1], chunk):
        z1 = min(z0 + chunk, alloc[1]) - 1
        sel = [b for b in bs if b.z1 + d >= z0 and b.z0 - d <= z1]
        if not sel:
            continue
        out.append(_abi.Box(min(b.x0 for b in sel) - d, min(b.y0 for b in sel) - d, z0,
                            max(b.x1 for b in sel) + d, max(b.y1 for b in sel) + d, z1))
    return out


def sweep_schedule(boxes, idx, fill_boxes, render_boxes, groups: int = 8, margin: int = 8):
    """Plan a batch reconstruction whose hole fill and render of finished z-chunks overlap the
    inserts of later frames (see `reconstruct_sweep`).  The frames `idx` (in sweep order) are cut
    into `groups` contiguous groups; a chunk box is ready once every frame whose conservative box
    meets its planes widened by `margin` (>= fill radius + the render's median and band reach) has
    been inserted.  Returns [(frame_begin, frame_end, fill_boxes_ready, render_boxes_ready)] with
    positions into `idx`; every box appears exactly once, in z order."""
    n = len(idx)
    groups = max(1, min(groups, n))
    cuts = [round(n * g / groups) for g in range(groups + 1)]

    def ready(b):  # position after the last frame that meets the widened chunk
        last = 0
        for p, k in enumerate(idx):
            fb = boxes[int(k)]
            if not fb.empty() and fb.z1 >= b.z0 - margin and fb.z0 <= b.z1 + margin:
                last = p + 1
        return last

    def group_of(b):
        r = ready(b)
        for g in range(groups):
            if r <= cuts[g + 1]:
                return g
        return groups - 1

    fg = [group_of(b) for b in fill_boxes]
    rg = [group_of(b) for b in render_boxes]
    # a chunk's render reads its own and its neighbours' fill layer: never ahead of the fills
    for i, b in enumerate(render_boxes):
        for j, fb_ in enumerate(fill_boxes):
            if fb_.z1 >= b.z0 - margin and fb_.z0 <= b.z1 + margin:
                rg[i] = max(rg[i], fg[j])
    out = []
    for g in range(groups):
        out.append((cuts[g], cuts[g + 1], [b for b, x in zip(fill_boxes, fg) if x == g],
                    [b for b, x in zip(render_boxes, rg) if x == g]))
    return out


def reconstruct_sweep(grid, frames, poses, calib, schedule, render_params, fill_radius: int = 1,
                      insert_stream=None, aux_stream=None, events=None):
    """Insert + mean fill + depth-band render of a batch, with the fill / render of every finished
    z-chunk (`sweep_schedule`) running on `aux_stream` while later frames are inserted on
    `insert_stream` (torch streams; default: the current stream and a new one).  The result is
    identical to insert-all, fill-all, render-all: each chunk is filled and rendered only after
    every frame that can reach it, chunks are processed in z order on one stream, and a column's
    last depth / band write is the one made after its neighbours' fills.  On return the insert
    stream has waited for the aux stream."""
    import torch

    s_ins = insert_stream or torch.cuda.current_stream()
    s_aux = aux_stream or torch.cuda.Stream(device=s_ins.device)
    evs = events or [torch.cuda.Event() for _ in schedule]
    for (a, b, fb, rb), ev in zip(schedule, evs):
        grid.set_stream(s_ins.cuda_stream, sync=False)
        if b > a:
            grid.insert_frames(frames[a:b], poses[a:b], calib)
        if fb or rb:
            ev.record(s_ins)
            s_aux.wait_event(ev)
            grid.set_stream(s_aux.cuda_stream, sync=False)
            if fb:
                grid.fill_holes_boxes(fb, fill_radius, _abi.FILL_MEAN, count=False)
            if rb:
                grid.render_coronal_boxes(rb, render_params, fill_radius)
    s_ins.wait_stream(s_aux)
    grid.set_stream(s_ins.cuda_stream, sync=False)
