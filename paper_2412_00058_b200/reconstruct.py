"""Host-side mirror of the reference `reconstruct` / `project` interface (SPEC.md:271-351,
SPEC.md:452-511) over the C-ABI.  Same operation names, argument meaning and error
behaviour (InvalidInput / AlgorithmFailure / IoError, core.hpp:14-32); every operation runs
on the GPU through libspinevol_b200.so — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import time
from typing import Iterable, Optional

import numpy as np

from . import _abi
from ._abi import (Box, Calib, GridDesc, InvalidInput, Rigid, RenderParams, check, lib, ptr,
                   rigid_array, rigid_ptr)

EMPTY_BOX = (1, 1, 1, 0, 0, 0)


def _box(b) -> Optional[Box]:
    if b is None:
        return None
    if isinstance(b, Box):
        return b
    return Box(*[int(v) for v in b])


def _frames_view(frames):
    """(pointer, row_pitch, frame_stride, n, h, w) for a (h,w) or (n,h,w) u8 array/tensor."""
    if isinstance(frames, np.ndarray):
        if frames.dtype != np.uint8:
            raise InvalidInput("frames must be uint8")
        a = frames if frames.ndim == 3 else frames[None]
        if a.ndim != 3:
            raise InvalidInput("frames must be (h,w) or (n,h,w)")
        if a.strides[2] != 1:
            a = np.ascontiguousarray(a)
        n, h, w = a.shape
        return a, a.ctypes.data, a.strides[1], a.strides[0], n, h, w
    # torch tensor (host or device)
    t = frames if frames.dim() == 3 else frames.unsqueeze(0)
    if str(t.dtype) != "torch.uint8":
        raise InvalidInput("frames must be uint8")
    if t.stride(2) != 1:
        t = t.contiguous()
    n, h, w = t.shape
    return t, t.data_ptr(), t.stride(1), t.stride(0), n, h, w


class VoxelGrid:
    """VoxelGrid: u32 sum + u16 count per voxel (packed on the device as one
    64-bit word), x-fastest layout.  `z_range` selects the stored slab."""

    def __init__(self, dims, voxel_mm: float = 1.0, origin=(0.0, 0.0, 0.0), device: int = 0,
                 z_range=None, accum: int = _abi.ACC_PNN):
        d = GridDesc()
        d.nx, d.ny, d.nz = (int(v) for v in dims)
        d.accum = accum
        d.voxel_mm = float(voxel_mm)
        for k in range(3):
            d.origin_mm[k] = float(origin[k])
        d.z_begin, d.z_end = (0, d.nz) if z_range is None else (int(z_range[0]), int(z_range[1]))
        self.desc = d
        self.device = device
        h = C.c_void_p()
        check(lib().svr_create(C.byref(d), device, C.byref(h)))
        self._h = h
        self.insert_seconds = []

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().svr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def dims(self):
        return (self.desc.nx, self.desc.ny, self.desc.nz)

    @property
    def slab(self):
        return (self.desc.z_begin, self.desc.z_end)

    def set_stream(self, cuda_stream: int | None, sync: bool = True):
        """Run later calls on `cuda_stream` (None: the handle's own).  sync=False switches without
        synchronizing the current stream (svr_use_stream): the caller orders the streams."""
        if not sync:
            check(lib().svr_use_stream(self._h, C.c_void_p(cuda_stream)))
            return
        check(lib().svr_set_stream(self._h, C.c_void_p(cuda_stream) if cuda_stream else None))

    def clear(self):
        check(lib().svr_clear(self._h))

    def sync(self):
        check(lib().svr_sync(self._h))

    # -- reconstruct
    def insert_frame(self, frame, pose, calib: Calib, skip_zero: bool = False) -> Box:
        """insert_frame; returns the tight DirtyRegion."""
        keep, p, pitch, _, n, h, w = _frames_view(frame)
        if n != 1:
            raise InvalidInput("insert_frame takes one frame")
        pa = rigid_array(pose)
        b = Box()
        check(lib().svr_insert_frame(self._h, p, pitch, w, h, rigid_ptr(pa), C.byref(calib),
                                     int(skip_zero), C.byref(b)))
        return b

    def insert_frames(self, frames, poses, calib: Calib, skip_zero: bool = False,
                      want_boxes: bool = False):
        """Batched insert.  want_boxes=True returns (per-frame boxes, union box) and syncs;
        otherwise the call is asynchronous on the grid's stream and returns None."""
        keep, p, pitch, stride, n, h, w = _frames_view(frames)
        pa = rigid_array(poses)
        if len(pa) != n:
            raise InvalidInput("need one pose per frame")
        if want_boxes:
            boxes = (Box * max(n, 1))()
            u = Box()
            check(lib().svr_insert_frames(self._h, p, pitch, stride, w, h, n, rigid_ptr(pa),
                                          C.byref(calib), int(skip_zero), boxes, C.byref(u)))
            return [boxes[i] for i in range(n)], u
        check(lib().svr_insert_frames(self._h, p, pitch, stride, w, h, n, rigid_ptr(pa),
                                      C.byref(calib), int(skip_zero), None, None))
        return None

    def frame_step(self, frame, pose, calib: Calib, fill_radius: int = 1,
                   params: RenderParams = None) -> Box:
        """One incremental frame (insert -> fill(box (+) 1) -> render(box)) as a CUDA-graph
        replay (svr_frame_step); asynchronous, returns the conservative dirty box."""
        from .synth import render_params
        keep, p, pitch, _, n, h, w = _frames_view(frame)
        if n != 1:
            raise InvalidInput("frame_step takes one frame")
        pa = rigid_array(pose)
        b = Box()
        check(lib().svr_frame_step(self._h, p, pitch, rigid_ptr(pa), C.byref(calib), int(fill_radius),
                                   C.byref(params or render_params()), C.byref(b)))
        self._keep = keep
        return b

    def fill_holes(self, region=None, radius: int = 1, mode: int = _abi.FILL_MEAN,
                   count: bool = True) -> Optional[int]:
        """fill_holes over exactly `region` (None = whole slab)."""
        out = C.c_int64(0)
        check(lib().svr_fill_holes(self._h, C.byref(_box(region)) if region is not None else None,
                                   mode, radius, C.byref(out) if count else None))
        return int(out.value) if count else None

    def fill_holes_boxes(self, regions, radius: int = 1, mode: int = _abi.FILL_MEAN,
                         count: bool = True) -> Optional[int]:
        """fill_holes over a list of (non-overlapping) regions in one launch."""
        arr = (Box * max(len(regions), 1))(*[_box(r) for r in regions])
        out = C.c_int64(0)
        check(lib().svr_fill_holes_boxes(self._h, arr, len(regions), mode, radius,
                                         C.byref(out) if count else None))
        return int(out.value) if count else None

    # -- project
    def render_coronal_boxes(self, dirty, params: RenderParams = None, fill_radius: int = 1):
        from .synth import render_params
        params = params or render_params()
        arr = (Box * max(len(dirty), 1))(*[_box(r) for r in dirty])
        check(lib().svr_render_coronal_boxes(self._h, arr, len(dirty), fill_radius, C.byref(params)))

    def render_coronal(self, dirty=None, params: RenderParams = None, fill_radius: int = 1):
        from .synth import render_params
        params = params or render_params()
        check(lib().svr_render_coronal(self._h, C.byref(_box(dirty)) if dirty is not None else None,
                                       fill_radius, C.byref(params)))

    def set_gather_targets(self, images, own=None):
        """Fused render + gather: later renders also store the owned rows' mean / max into each
        image (device tensors or pointers of [2, nz, nx] f32, e.g. symmetric-memory peers).
        images = [] switches it off.  own = (z0, z1) owned global rows (default: the slab)."""
        ptrs = [ptr(t) for t in images]
        arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
        z0, z1 = own if own is not None else (self.desc.z_begin, self.desc.z_end)
        check(lib().svr_set_gather_targets(self._h, arr, len(ptrs), int(z0), int(z1)))

    def read_coronal(self, z0=None, z1=None):
        z0 = self.desc.z_begin if z0 is None else z0
        z1 = self.desc.z_end - 1 if z1 is None else z1
        n = (z1 - z0 + 1) * self.desc.nx
        mean = np.empty(n, np.float32)
        mx = np.empty(n, np.float32)
        dep = np.empty(n, np.int32)
        check(lib().svr_read_coronal(self._h, z0, z1, ptr(mean), ptr(mx), ptr(dep)))
        shp = (z1 - z0 + 1, self.desc.nx)
        return mean.reshape(shp), mx.reshape(shp), dep.reshape(shp)

    def read_coronal_into(self, z0, z1, mean, mx, depth=None, wait: bool = True):
        """Copy rendered rows into caller buffers (host or device, e.g. torch tensors).
        wait=False only enqueues the copy on the grid's stream (pinned / device outputs)."""
        fn = lib().svr_read_coronal if wait else lib().svr_read_coronal_async
        check(fn(self._h, z0, z1, ptr(mean), ptr(mx), ptr(depth)))

    def coronal_projection(self, mode: int = _abi.PROJ_MAX, depth_axis: int = 2,
                           use_fills: bool = False) -> np.ndarray:
        """coronal_projection: u8 image over the two remaining axes."""
        dims = [self.desc.nx, self.desc.ny, self.desc.z_end - self.desc.z_begin]
        rest = [dims[a] for a in range(3) if a != depth_axis]
        out = np.empty(rest[0] * rest[1], np.uint8)
        check(lib().svr_coronal_projection(self._h, mode, depth_axis, int(use_fills), ptr(out)))
        return out.reshape(rest[1], rest[0])

    # -- readout
    def _box_shape(self, box):
        b = _box(box) if box is not None else Box(0, 0, self.desc.z_begin, self.desc.nx - 1,
                                                  self.desc.ny - 1, self.desc.z_end - 1)
        return b, (b.z1 - b.z0 + 1, b.y1 - b.y0 + 1, b.x1 - b.x0 + 1)

    def accumulators(self, box=None):
        b, shp = self._box_shape(box)
        s = np.empty(shp, np.uint32)
        c = np.empty(shp, np.uint16)
        check(lib().svr_read_accumulators(self._h, C.byref(b), ptr(s), ptr(c)))
        return s, c

    def set_accumulators(self, sum_, count, box=None):
        """Restore sum / count (the `accumulators()` layout) into `box` (default: the slab)."""
        b, shp = self._box_shape(box)
        s = np.ascontiguousarray(sum_, np.uint32).reshape(shp)
        c = np.ascontiguousarray(count, np.uint16).reshape(shp)
        check(lib().svr_write_accumulators(self._h, C.byref(b), ptr(s), ptr(c)))

    def save(self, path):
        """Checkpoint the accumulators (npz with the grid description); fills are derived state."""
        s, c = self.accumulators()
        d = self.desc
        np.savez_compressed(path, sum=s, count=c, dims=np.array([d.nx, d.ny, d.nz]),
                            voxel_mm=d.voxel_mm, origin=np.array(list(d.origin_mm)),
                            z_range=np.array([d.z_begin, d.z_end]),
                            frames_inserted=self.stats()["frames_inserted"])

    def load(self, path):
        """Resume from `save`: the grid description (dims, slab, voxel size, origin) must match.
        The fill layer is derived state and is cleared (re-run fill_holes); the checkpoint's
        frames_inserted is returned (device stats count only this handle's own inserts)."""
        z = np.load(path)
        d = self.desc
        if list(z["dims"]) != [d.nx, d.ny, d.nz] or list(z["z_range"]) != [d.z_begin, d.z_end] or \
                float(z["voxel_mm"]) != d.voxel_mm or \
                not np.array_equal(np.asarray(z["origin"], np.float64), np.array(list(d.origin_mm), np.float64)):
            raise InvalidInput("checkpoint does not match this grid")
        self.set_accumulators(z["sum"], z["count"])
        return int(z["frames_inserted"]) if "frames_inserted" in z else None

    def values(self, box=None, apply_fills=False):
        """VoxelGrid::value = round(sum/count), 0 when empty."""
        b, shp = self._box_shape(box)
        out = np.empty(shp, np.uint8)
        check(lib().svr_read_values(self._h, C.byref(b), int(apply_fills), ptr(out)))
        return out

    def fill_layer(self, box=None):
        b, shp = self._box_shape(box)
        out = np.empty(shp, np.uint32)
        check(lib().svr_read_fill(self._h, C.byref(b), ptr(out)))
        return out

    def trilinear(self, box=None):
        b, shp = self._box_shape(box)
        ws = np.empty(shp, np.float32)
        wt = np.empty(shp, np.float32)
        check(lib().svr_read_trilinear(self._h, C.byref(b), ptr(ws), ptr(wt)))
        return ws, wt

    def stats(self) -> dict:
        s = _abi.Stats()
        check(lib().svr_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def footprint(self, frames, poses, calib, skip_zero=False) -> np.ndarray:
        keep, p, pitch, stride, n, h, w = _frames_view(frames)
        pa = rigid_array(poses)
        out = np.zeros(n, np.int64)
        check(lib().svr_count_footprint(self._h, p, pitch, stride, w, h, n, rigid_ptr(pa),
                                        C.byref(calib), int(skip_zero),
                                        out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out


# ------------------------------------------------------------------ SPEC free functions
def insert_frame(grid: VoxelGrid, frame, pose, calib: Calib, skip_zero: bool = False) -> Box:
    return grid.insert_frame(frame, pose, calib, skip_zero)


def fill_holes(grid: VoxelGrid, region, radius: int = 2, mode: int = _abi.FILL_MEDIAN) -> int:
    """SPEC default: lower median over Chebyshev radius 2."""
    return grid.fill_holes(region, radius, mode)


def coronal_projection(grid: VoxelGrid, mode: int = _abi.PROJ_MAX, depth_axis: int = 2):
    return grid.coronal_projection(mode, depth_axis)


def frame_bounds(desc: GridDesc, calib: Calib, pose) -> Box:
    """Conservative voxel box a frame can touch (host only)."""
    pa = rigid_array(pose)
    b = Box()
    check(lib().svr_frame_bounds(C.byref(desc), C.byref(calib), rigid_ptr(pa), C.byref(b)))
    return b


def dilate(b: Box, r: int) -> Box:
    if b.empty():
        return b
    return Box(b.x0 - r, b.y0 - r, b.z0 - r, b.x1 + r, b.y1 + r, b.z1 + r)


def run_incremental(frames: Iterable, poses, calib: Calib, grid: VoxelGrid, hole_radius: int = 1,
                    fill_mode: int = _abi.FILL_MEAN, render: Optional[RenderParams] = None,
                    skip_zero: bool = False):
    """run_incremental: per frame insert -> fill(dirty (+) r) -> render.
    The dirty region used for fill/render is the host-computed conservative frame box, a
    superset of the tight box, so no device round trip is needed per frame; the result is
    bit-identical to batch processing.  Returns (grid, stats) with per-frame wall latency
    percentiles (percentile as core.hpp:101-107)."""
    pa = rigid_array(poses)
    lat = []
    graph = render is not None and hole_radius == 1 and fill_mode == _abi.FILL_MEAN and not skip_zero
    for k, fr in enumerate(frames):
        t0 = time.perf_counter()
        if graph:  # the whole per-frame step as one CUDA-graph replay (svr_frame_step)
            grid.frame_step(fr, pa[k:k + 1], calib, 1, render)
            grid.sync()
            lat.append((time.perf_counter() - t0) * 1e3)
            continue
        grid.insert_frames(fr, pa[k:k + 1], calib, skip_zero)
        b = frame_bounds(grid.desc, calib, pa[k:k + 1])
        if not b.empty():
            grid.fill_holes(dilate(b, hole_radius), hole_radius, fill_mode, count=False)
            if render is not None:
                grid.render_coronal(b, render, hole_radius)
        grid.sync()
        lat.append((time.perf_counter() - t0) * 1e3)
    st = grid.stats()
    if lat:
        st.update(latency_ms_p50=_percentile(lat, 0.5), latency_ms_p95=_percentile(lat, 0.95),
                  latency_ms_max=max(lat))
    return grid, st


def _percentile(v, p):
    s = sorted(v)
    k = int(p * (len(s) - 1) + 0.5)
    return s[k]


def pose_from_matrix4(m) -> Rigid:
    """RigidTransform::from_matrix4 (geometry.hpp:133-139)."""
    a = (C.c_double * 16)(*[float(x) for x in np.asarray(m, dtype=np.float64).reshape(16)])
    r = Rigid()
    check(lib().svr_pose_from_matrix4(a, C.byref(r)))
    return r


def compose(a: Rigid, b: Rigid) -> Rigid:
    r = Rigid()
    check(lib().svr_compose(C.byref(a), C.byref(b), C.byref(r)))
    return r


def interpolate_pose(t_ms, poses, t: float) -> Rigid:
    tt = np.ascontiguousarray(t_ms, dtype=np.float64)
    pa = rigid_array(poses)
    r = Rigid()
    check(lib().svr_interpolate_pose(tt.ctypes.data_as(C.POINTER(C.c_double)), rigid_ptr(pa),
                                     len(pa), float(t), C.byref(r)))
    return r


def pixel_to_world(col, row, calib: Calib, pose: Rigid):
    out = (C.c_double * 3)()
    check(lib().svr_pixel_to_world(float(col), float(row), C.byref(calib), C.byref(pose), out))
    return (out[0], out[1], out[2])
