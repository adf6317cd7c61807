"""ctypes binding of the C-ABI in include/spinevol_b200.h (libspinevol_b200.so).

The shared library is built in-tree (paper_2412_00058_b200/csrc/Makefile, driven by
`__graft_entry__.build()`).  There is no CPU fallback: a missing library raises, and every
device entry point fails loudly without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SVR_LIB_PATH: load another build of the library (A/B experiments with compile-time variants)
LIB_PATH = os.environ.get("SVR_LIB_PATH") or os.path.join(_HERE, "libspinevol_b200.so")

SVR_OK, SVR_E_INVALID, SVR_E_ALGO, SVR_E_IO, SVR_E_CUDA = 0, 2, 3, 4, 5
PROBE_LINEAR, PROBE_FAN = 0, 1
FILL_MEAN, FILL_MEDIAN = 0, 1
ACC_PNN, ACC_TRILINEAR = 0, 1
PROJ_MAX, PROJ_MEAN = 0, 1


class Rigid(C.Structure):
    """RigidTransform (geometry.hpp:104-140): quaternion w,x,y,z + translation (mm)."""
    _fields_ = [("qw", C.c_double), ("qx", C.c_double), ("qy", C.c_double), ("qz", C.c_double),
                ("tx", C.c_double), ("ty", C.c_double), ("tz", C.c_double)]


class Calib(C.Structure):
    """ImageCalibration (geometry.hpp:160-176) + probe geometry."""
    _fields_ = [("crop_x", C.c_int32), ("crop_y", C.c_int32), ("crop_w", C.c_int32),
                ("crop_h", C.c_int32), ("scale_x_mm", C.c_double), ("scale_y_mm", C.c_double),
                ("image_to_transducer", Rigid), ("latency_ms", C.c_double), ("probe", C.c_int32),
                ("reserved0", C.c_int32), ("fan_angle_deg", C.c_double),
                ("fan_r0_mm", C.c_double), ("fan_r1_mm", C.c_double)]


class GridDesc(C.Structure):
    """VoxelGrid config + stored z slab."""
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("accum", C.c_int32),
                ("voxel_mm", C.c_double), ("origin_mm", C.c_double * 3),
                ("z_begin", C.c_int32), ("z_end", C.c_int32)]


class Box(C.Structure):
    """DirtyRegion: inclusive, empty iff x0 > x1."""
    _fields_ = [("x0", C.c_int32), ("y0", C.c_int32), ("z0", C.c_int32),
                ("x1", C.c_int32), ("y1", C.c_int32), ("z1", C.c_int32)]

    def empty(self) -> bool:
        return self.x0 > self.x1

    def as_tuple(self):
        return (self.x0, self.y0, self.z0, self.x1, self.y1, self.z1)

    def __repr__(self):
        return "Box(%d,%d,%d .. %d,%d,%d)" % self.as_tuple()


class Stats(C.Structure):
    _fields_ = [("frames_inserted", C.c_uint64), ("pixels_inserted", C.c_uint64),
                ("pixels_oob", C.c_uint64), ("pixels_skipped_zero", C.c_uint64),
                ("pixels_saturated", C.c_uint64), ("exact_fallbacks", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("chunks_deferred", C.c_uint64),
                ("tiles_table", C.c_uint64), ("graph_captures", C.c_uint64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class RenderParams(C.Structure):
    _fields_ = [("depth_lo_mm", C.c_double), ("depth_hi_mm", C.c_double),
                ("band_above_mm", C.c_double), ("band_below_mm", C.c_double),
                ("median_radius", C.c_int32), ("fill_mode", C.c_int32)]


RIGID_DTYPE = np.dtype([("qw", "f8"), ("qx", "f8"), ("qy", "f8"), ("qz", "f8"),
                        ("tx", "f8"), ("ty", "f8"), ("tz", "f8")])

P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
PR, PC, PG, PB, PS = (C.POINTER(Rigid), C.POINTER(Calib), C.POINTER(GridDesc), C.POINTER(Box),
                      C.POINTER(Stats))

# name -> (restype, argtypes); the exported symbol set of include/spinevol_b200.h
SIGNATURES = {
    "svr_abi_version": (C.c_int, []),
    "svr_last_error": (C.c_char_p, []),
    "svr_device_count": (C.c_int, []),
    "svr_pose_from_matrix4": (C.c_int, [C.POINTER(D), PR]),
    "svr_compose": (C.c_int, [PR, PR, PR]),
    "svr_interpolate_pose": (C.c_int, [C.POINTER(D), PR, C.c_int, D, PR]),
    "svr_pixel_to_world": (C.c_int, [D, D, PC, PR, C.POINTER(D)]),
    "svr_frame_bounds": (C.c_int, [PG, PC, PR, PB]),
    "svr_plan_slabs": (C.c_int, [I32, I32, I32, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32),
                                 C.POINTER(I32)]),
    "svr_create": (C.c_int, [PG, C.c_int, C.POINTER(P)]),
    "svr_destroy": (C.c_int, [P]),
    "svr_set_stream": (C.c_int, [P, P]),
    "svr_use_stream": (C.c_int, [P, P]),
    "svr_clear": (C.c_int, [P]),
    "svr_sync": (C.c_int, [P]),
    "svr_get_desc": (C.c_int, [P, PG]),
    "svr_insert_frame": (C.c_int, [P, P, I64, I32, I32, PR, PC, I32, PB]),
    "svr_insert_frames": (C.c_int, [P, P, I64, I64, I32, I32, I32, PR, PC, I32, PB, PB]),
    "svr_fill_holes": (C.c_int, [P, PB, I32, I32, C.POINTER(I64)]),
    "svr_render_coronal": (C.c_int, [P, PB, I32, C.POINTER(RenderParams)]),
    "svr_fill_holes_boxes": (C.c_int, [P, PB, I32, I32, I32, C.POINTER(I64)]),
    "svr_render_coronal_boxes": (C.c_int, [P, PB, I32, I32, C.POINTER(RenderParams)]),
    "svr_frame_step": (C.c_int, [P, P, I64, PR, PC, I32, C.POINTER(RenderParams), PB]),
    "svr_read_coronal": (C.c_int, [P, I32, I32, P, P, P]),
    "svr_read_coronal_async": (C.c_int, [P, I32, I32, P, P, P]),
    "svr_set_gather_targets": (C.c_int, [P, C.POINTER(P), I32, I32, I32]),
    "svr_coronal_projection": (C.c_int, [P, I32, I32, I32, P]),
    "svr_read_accumulators": (C.c_int, [P, PB, P, P]),
    "svr_read_values": (C.c_int, [P, PB, I32, P]),
    "svr_write_accumulators": (C.c_int, [P, PB, P, P]),
    "svr_read_fill": (C.c_int, [P, PB, P]),
    "svr_read_trilinear": (C.c_int, [P, PB, P, P]),
    "svr_get_stats": (C.c_int, [P, PS]),
    "svr_count_footprint": (C.c_int, [P, P, I64, I64, I32, I32, I32, PR, PC, I32, C.POINTER(I64)]),
    "svr_synth_frames": (C.c_int, [P, I32, I32, I32, I32, PC, PR, I32, U64, C.c_int, P]),
    "svr_selftest_value_rounding": (C.c_int, [C.c_int, C.POINTER(I64)]),
    "svr_export_slices_x": (C.c_int, [P, I32, P]),
    "svr_export_slices": (C.c_int, [P, C.c_char_p, I32, I32, C.POINTER(I32)]),
    "svr_export_volume": (C.c_int, [P, C.c_char_p, I32]),
    "svr_pgm_info": (C.c_int, [C.c_char_p, C.POINTER(I32), C.POINTER(I32)]),
    "svr_pgm_read": (C.c_int, [C.c_char_p, P, I64, I32, I32]),
    "svr_pgm_write": (C.c_int, [C.c_char_p, P, I64, I32, I32]),
    "svr_load_frames": (C.c_int, [C.POINTER(C.c_char_p), I32, I32, I32, C.POINTER(I32), P, I64, I32,
                                  C.POINTER(I32)]),
    "svr_write_raw": (C.c_int, [C.c_char_p, P, I64]),
    "svr_match_poses": (C.c_int, [C.POINTER(D), PR, I32, C.POINTER(D), I32, D, PR, P, C.POINTER(I32)]),
    "svr_cut_depth_alg1": (C.c_int, [D, D, D, D, D, D, C.POINTER(D)]),
    "svr_cut_rows": (C.c_int, [D, D, D, I32, C.POINTER(I32), C.POINTER(I32)]),
    "svr_smooth_depths": (C.c_int, [P, P, I32, I32, P]),
    "svr_bone_contour": (C.c_int, [P, I64, I64, I32, I32, I32, D, I32, I32, D, P, P, P, P, C.c_int, P]),
    "svr_apply_cut": (C.c_int, [P, I64, I64, I32, I32, I32, P, P, C.c_int, P]),
    "svr_sharded_create": (C.c_int, [PG, C.POINTER(I32), I32, I32, C.POINTER(P)]),
    "svr_sharded_destroy": (C.c_int, [P]),
    "svr_sharded_slab": (C.c_int, [P, I32, C.POINTER(P), C.POINTER(I32), C.POINTER(I32), C.POINTER(I32),
                                   C.POINTER(I32)]),
    "svr_sharded_insert_frames": (C.c_int, [P, P, I64, I64, I32, I32, I32, PR, PC, I32, C.POINTER(I32)]),
    "svr_sharded_fill_render": (C.c_int, [P, I32, I32, C.POINTER(RenderParams)]),
    "svr_sharded_sync": (C.c_int, [P]),
    "svr_sharded_read_coronal": (C.c_int, [P, P, P, P]),
}

_lib = None
_lock = threading.Lock()


def build_library(force: bool = False) -> str:
    """Compile libspinevol_b200.so in-tree with nvcc for sm_100a (csrc/Makefile)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", os.path.join(_HERE, "csrc")], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    """Load the product library (building it if the .so is absent). Never falls back."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build_library()
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            if L.svr_abi_version() != 2:
                raise RuntimeError("libspinevol_b200 ABI version mismatch")
            _lib = L
    return _lib


class SpinevolError(RuntimeError):
    """Base of the core.hpp error hierarchy (core.hpp:14-17)."""


class InvalidInput(SpinevolError):
    """core.hpp:19-22 — exit code 2."""


class AlgorithmFailure(SpinevolError):
    """core.hpp:24-27 — exit code 3."""


class IoError(SpinevolError):
    """core.hpp:29-32 — exit code 4."""


class DeviceError(SpinevolError):
    """CUDA / NCCL failure (code 5)."""


_ERRORS = {SVR_E_INVALID: InvalidInput, SVR_E_ALGO: AlgorithmFailure, SVR_E_IO: IoError,
           SVR_E_CUDA: DeviceError}


def check(rc: int) -> None:
    if rc != SVR_OK:
        msg = lib().svr_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SpinevolError)(msg)


def ptr(a) -> int:
    """Address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return int(a)


def rigid_array(poses) -> np.ndarray:
    """Poses as a contiguous svr_rigid array (numpy structured, RIGID_DTYPE)."""
    if isinstance(poses, np.ndarray) and poses.dtype == RIGID_DTYPE:
        return np.ascontiguousarray(poses)
    if isinstance(poses, Rigid):
        poses = [poses]
    out = np.zeros(len(poses), dtype=RIGID_DTYPE)
    for i, p in enumerate(poses):
        if isinstance(p, Rigid):
            out[i] = (p.qw, p.qx, p.qy, p.qz, p.tx, p.ty, p.tz)
        else:
            out[i] = tuple(float(x) for x in p)
    return out


def rigid_ptr(arr: np.ndarray):
    return C.cast(arr.ctypes.data, PR)
