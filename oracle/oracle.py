"""ctypes binding of the CPU oracle (liboracle.so) and of the reference shim
(_ref/libspinevol_ref.so, compiled from /root/reference's own headers).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs — never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2412_00058_b200._abi import (Box, Calib, RenderParams, Rigid, RIGID_DTYPE, rigid_array,
                                        rigid_ptr)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspinevol_ref.so")


class OrcGrid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("z_begin", C.c_int32), ("z_end", C.c_int32),
                ("voxel_mm", C.c_double), ("origin", C.c_double * 3),
                ("sum", C.c_void_p), ("count", C.c_void_p), ("fill", C.c_void_p),
                ("wsum", C.c_void_p), ("weight", C.c_void_p),
                ("frames", C.c_uint64), ("inserted", C.c_uint64), ("oob", C.c_uint64),
                ("skipped_zero", C.c_uint64), ("saturated", C.c_uint64), ("fill_mode", C.c_int32)]


_lib = None
_ref = None


def build():
    subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        P, PB, PR, PC = C.c_void_p, C.POINTER(Box), C.POINTER(Rigid), C.POINTER(Calib)
        PG = C.POINTER(OrcGrid)
        L.orc_pixel_to_world.argtypes = [C.c_double, C.c_double, PC, PR, C.POINTER(C.c_double)]
        L.orc_fan_table.argtypes = [PC, P, P]
        L.orc_fan_point.argtypes = [C.c_int, C.c_int, PC, P, P, PR, C.POINTER(C.c_double)]
        L.orc_insert_frame.argtypes = [PG, P, C.c_int64, C.c_int32, C.c_int32, PR, PC, C.c_int32, PB]
        L.orc_insert_frames_mt.argtypes = [PG, P, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                           C.c_int32, PR, PC, C.c_int32, C.c_int32]
        L.orc_insert_frames_mt_boxes.argtypes = [PG, P, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                                 C.c_int32, PR, PC, C.c_int32, C.c_int32, PB]
        L.orc_fill_holes.argtypes = [PG, PB, C.c_int32, C.c_int32]
        L.orc_fill_holes.restype = C.c_int64
        L.orc_values.argtypes = [PG, C.c_int32, P]
        L.orc_render.argtypes = [PG, PB, C.c_int32, C.POINTER(RenderParams), P, P, P, P]
        L.orc_fill_holes_boxes_mt.argtypes = [PG, PB, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.orc_fill_holes_boxes_mt.restype = C.c_int64
        L.orc_render_boxes_mt.argtypes = [PG, PB, C.c_int32, C.c_int32, C.POINTER(RenderParams), P, P, P,
                                          P, C.c_int32]
        L.orc_render_ints.argtypes = [C.POINTER(RenderParams), C.c_double, C.c_int32] + [C.POINTER(C.c_int32)] * 4
        L.orc_coronal_projection.argtypes = [PG, C.c_int32, C.c_int32, C.c_int32, P]
        L.orc_cut_depth_alg1.argtypes = [C.c_double] * 6
        L.orc_cut_depth_alg1.restype = C.c_double
        L.orc_cut_rows.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int32,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.orc_apply_cut.argtypes = [P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.orc_bone_contour.argtypes = [P, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                                       C.c_int32, C.c_double, P, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]
        L.orc_bone_contour.restype = C.c_int32
        L.orc_smooth_depths.argtypes = [P, P, C.c_int32, C.c_int32, P]
        L.orc_insert_trilinear.argtypes = [PG, P, C.c_int64, C.c_int32, C.c_int32, PR, PC, C.c_int32]
        L.orc_insert_trilinear_f64.argtypes = [PG, P, C.c_int64, C.c_int32, C.c_int32, PR, PC, C.c_int32, P, P]
        _lib = L
    return _lib


def ref():
    """The reference's own geometry (oracle/_ref), or None where it was not built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        R = C.CDLL(REF_SO)
        PR, PC = C.POINTER(Rigid), C.POINTER(Calib)
        PD = C.POINTER(C.c_double)
        R.ref_pixel_to_world.argtypes = [C.c_double, C.c_double, PC, PR, PD]
        R.ref_from_matrix4.argtypes = [PD, PR]
        R.ref_compose.argtypes = [PR, PR, PR]
        R.ref_apply.argtypes = [PR, PD, PD]
        R.ref_interpolate_pose.argtypes = [PD, PR, C.c_int, C.c_double, PR]
        R.ref_read_pgm.argtypes = [C.c_char_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32)]
        R.ref_write_pgm.argtypes = [C.c_char_p, C.c_void_p, C.c_int32, C.c_int32]
        R.ref_median_lower.argtypes = [PD, C.c_int]
        R.ref_median_lower.restype = C.c_double
        R.ref_insert_frames.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, PD,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                        C.c_int32, C.c_int32, C.c_int32, PR, PC, C.c_int32,
                                        C.c_int32, C.POINTER(C.c_uint64)]
        _ref = R
    return _ref


class OracleGrid:
    """CPU VoxelGrid: u32 sum, u16 count, u32 fill layer (+ f32 trilinear), slab-aware."""

    def __init__(self, dims, voxel_mm, origin=(0, 0, 0), z_range=None, trilinear=False):
        nx, ny, nz = dims
        zb, ze = (0, nz) if z_range is None else z_range
        shp = (ze - zb, ny, nx)
        self.sum = np.zeros(shp, np.uint32)
        self.count = np.zeros(shp, np.uint16)
        self.fill = np.zeros(shp, np.uint32)
        self.wsum = np.zeros(shp, np.float32) if trilinear else None
        self.weight = np.zeros(shp, np.float32) if trilinear else None
        g = OrcGrid()
        g.nx, g.ny, g.nz, g.z_begin, g.z_end = nx, ny, nz, zb, ze
        g.voxel_mm = voxel_mm
        for k in range(3):
            g.origin[k] = origin[k]
        g.sum, g.count, g.fill = self.sum.ctypes.data, self.count.ctypes.data, self.fill.ctypes.data
        if trilinear:
            g.wsum, g.weight = self.wsum.ctypes.data, self.weight.ctypes.data
        self.g = g
        self.dims = dims
        self.z_range = (zb, ze)
        cols = (ze - zb, nx)
        self.mean = np.zeros(cols, np.float32)
        self.max = np.zeros(cols, np.float32)
        self.depth = np.full(cols, -1, np.int32)
        self.mdepth = np.full(cols, -1, np.int32)

    @classmethod
    def for_workload(cls, wl, z_range=None):
        from paper_2412_00058_b200 import _abi
        return cls(wl.dims, wl.voxel_mm, wl.origin, z_range, trilinear=wl.accum == _abi.ACC_TRILINEAR)

    def insert_frame(self, frame, pose, calib, skip_zero=False) -> Box:
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        h, w = frame.shape
        pa = rigid_array(pose)
        b = Box()
        rc = lib().orc_insert_frame(C.byref(self.g), frame.ctypes.data, w, w, h, rigid_ptr(pa),
                                    C.byref(calib), int(skip_zero), C.byref(b))
        if rc:
            raise ValueError("oracle insert_frame rejected input (%d)" % rc)
        return b

    def insert_frames(self, frames, poses, calib, skip_zero=False):
        pa = rigid_array(poses)
        return [self.insert_frame(frames[k], pa[k:k + 1], calib, skip_zero) for k in range(len(pa))]

    def insert_frames_mt(self, frames, poses, calib, skip_zero=False, nthreads=None):
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        pa = rigid_array(poses)
        nthreads = nthreads or os.cpu_count() or 1
        rc = lib().orc_insert_frames_mt(C.byref(self.g), frames.ctypes.data, w, w * h, w, h, n,
                                        rigid_ptr(pa), C.byref(calib), int(skip_zero), nthreads)
        if rc:
            raise ValueError("oracle insert rejected input")

    def insert_frames_mt_boxes(self, frames, poses, calib, skip_zero=False, nthreads=None):
        """Multithreaded insert that also returns each frame's tight dirty box."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        n, h, w = frames.shape
        pa = rigid_array(poses)
        nthreads = nthreads or os.cpu_count() or 1
        boxes = (Box * max(n, 1))()
        rc = lib().orc_insert_frames_mt_boxes(C.byref(self.g), frames.ctypes.data, w, w * h, w, h, n,
                                              rigid_ptr(pa), C.byref(calib), int(skip_zero), nthreads,
                                              boxes)
        if rc:
            raise ValueError("oracle insert rejected input")
        return [boxes[k] for k in range(n)]

    def insert_trilinear(self, frame, pose, calib, skip_zero=False):
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        h, w = frame.shape
        pa = rigid_array(pose)
        lib().orc_insert_trilinear(C.byref(self.g), frame.ctypes.data, w, w, h, rigid_ptr(pa),
                                   C.byref(calib), int(skip_zero))

    def insert_trilinear_f64(self, frames, poses, calib, skip_zero=False):
        """Trilinear splat summed in fp64 (self.wsum64 / self.weight64): the parity reference."""
        if getattr(self, "wsum64", None) is None:
            self.wsum64 = np.zeros(self.sum.shape, np.float64)
            self.weight64 = np.zeros(self.sum.shape, np.float64)
        pa = rigid_array(poses)
        for k in range(len(pa)):
            f = np.ascontiguousarray(frames[k], dtype=np.uint8)
            h, w = f.shape
            lib().orc_insert_trilinear_f64(C.byref(self.g), f.ctypes.data, w, w, h, rigid_ptr(pa[k:k + 1]),
                                           C.byref(calib), int(skip_zero), self.wsum64.ctypes.data,
                                           self.weight64.ctypes.data)

    def fill_holes(self, region=None, mode=0, radius=1) -> int:
        b = None if region is None else C.byref(region if isinstance(region, Box) else Box(*region))
        return int(lib().orc_fill_holes(C.byref(self.g), b, mode, radius))

    def fill_holes_boxes_mt(self, boxes, mode=0, radius=1, nthreads=None) -> int:
        arr = (Box * max(len(boxes), 1))(*[b if isinstance(b, Box) else Box(*b) for b in boxes])
        return int(lib().orc_fill_holes_boxes_mt(C.byref(self.g), arr, len(boxes), mode, radius,
                                                 nthreads or os.cpu_count() or 1))

    def render_boxes_mt(self, params, boxes, fill_radius=1, nthreads=None):
        arr = (Box * max(len(boxes), 1))(*[b if isinstance(b, Box) else Box(*b) for b in boxes])
        lib().orc_render_boxes_mt(C.byref(self.g), arr, len(boxes), fill_radius, C.byref(params),
                                  self.mean.ctypes.data, self.max.ctypes.data, self.depth.ctypes.data,
                                  self.mdepth.ctypes.data, nthreads or os.cpu_count() or 1)
        return self.mean, self.max, self.mdepth

    def values(self, apply_fills=False):
        out = np.empty_like(self.sum, dtype=np.uint8)
        lib().orc_values(C.byref(self.g), int(apply_fills), out.ctypes.data)
        return out

    def render(self, params: RenderParams, dirty=None, fill_radius=1):
        b = None if dirty is None else C.byref(dirty if isinstance(dirty, Box) else Box(*dirty))
        lib().orc_render(C.byref(self.g), b, fill_radius, C.byref(params), self.mean.ctypes.data,
                         self.max.ctypes.data, self.depth.ctypes.data, self.mdepth.ctypes.data)
        return self.mean, self.max, self.mdepth

    def coronal_projection(self, mode=0, depth_axis=2, use_fills=False):
        nzl = self.z_range[1] - self.z_range[0]
        dims = [self.dims[0], self.dims[1], nzl]
        rest = [dims[a] for a in range(3) if a != depth_axis]
        out = np.empty(rest[0] * rest[1], np.uint8)
        lib().orc_coronal_projection(C.byref(self.g), mode, depth_axis, int(use_fills), out.ctypes.data)
        return out.reshape(rest[1], rest[0])

    @property
    def stats(self):
        g = self.g
        return dict(frames=g.frames, inserted=g.inserted, oob=g.oob, skipped_zero=g.skipped_zero,
                    saturated=g.saturated)


def pixel_to_world(col, row, calib, pose):
    out = (C.c_double * 3)()
    rc = lib().orc_pixel_to_world(float(col), float(row), C.byref(calib), C.byref(pose), out)
    if rc:
        raise ValueError("pixel outside B-mode image bounds")
    return (out[0], out[1], out[2])


def ref_insert_frames(dims, voxel_mm, origin, frames, poses, calib, skip_zero=False, nthreads=1,
                      z_range=None, out=None):
    """Reference CPU insert (spinevol::pixel_to_world per pixel), multi-threaded.  `out` =
    preallocated (sum, count) arrays to accumulate into (kept out of timed regions)."""
    R = ref()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    nx, ny, nz = dims
    zb, ze = (0, nz) if z_range is None else z_range
    if out is None:
        s = np.zeros((ze - zb, ny, nx), np.uint32)
        c = np.zeros((ze - zb, ny, nx), np.uint16)
    else:
        s, c = out
    frames = np.ascontiguousarray(frames, dtype=np.uint8)
    n, h, w = frames.shape
    pa = rigid_array(poses)
    o = (C.c_double * 3)(*origin)
    ins = C.c_uint64(0)
    rc = R.ref_insert_frames(nx, ny, zb, ze, voxel_mm, o, s.ctypes.data, c.ctypes.data,
                             frames.ctypes.data, w, w * h, w, h, n, rigid_ptr(pa), C.byref(calib),
                             int(skip_zero), nthreads, C.byref(ins))
    if rc:
        raise ValueError("reference insert rejected input")
    return s, c, int(ins.value)
