"""Segmentation front-end of the insert path (SPEC.md segment module; the paper's Tables I-II):
Algorithm 1 (pose-driven depth of cut, streaming) and Algorithm 2 (per-frame bone contour +
median filtering, post-acquisition), producing cut frames that the CUDA insert consumes with
skip_zero, plus the fixed-depth VPI baseline.

Frames are device-resident (torch uint8 CUDA tensors, (n, h, w)): the contour search and the cut
run as sm_100a kernels (svr_segment.cu) in place; the per-frame scalar work (cut depths, depth
smoothing) is host C++ behind the same C-ABI.  Pins the SPEC leaves open are listed in DESIGN.md
§3 and restated by the CPU oracle (oracle/svr_oracle.c).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _abi
from ._abi import AlgorithmFailure, Calib, InvalidInput, check, lib, rigid_array

SCHEMA_VERSION = 1
DEFAULTS = {"K": 0.04, "D": 35.0, "L": 500.0, "band_mm": 15.0, "window": 11, "pct": 0.70,
            "grad_per_mm": 25.0, "shadow_mm": 3.0, "min_valid_frac": 0.10}


@dataclass
class Alg1Params:
    """Table I constants (SPEC Alg1Params): K >= 0, D > 0 mm, L > 0 mm."""
    K: float = DEFAULTS["K"]
    D: float = DEFAULTS["D"]
    L: float = DEFAULTS["L"]
    axis: int = 0          # offset axis of P_c (Open Question: x as printed)


@dataclass
class CutProfile:
    """Per-frame depth of cut (mm), its source (alg1 | alg2 | fixed) and the band (mm)."""
    cut_mm: np.ndarray
    source: str
    band_mm: float

    def to_json(self) -> str:
        """SPEC External Interfaces: a JSON array of {frame, cut_mm} (+ schema_version)."""
        return json.dumps({"schema_version": SCHEMA_VERSION, "source": self.source,
                           "band_mm": self.band_mm,
                           "cuts": [{"frame": i, "cut_mm": float(c)} for i, c in enumerate(self.cut_mm)]})


def _dev(frames):
    import torch
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda and frames.dtype == torch.uint8):
        raise InvalidInput("segmentation needs device-resident uint8 frames (torch CUDA tensor)")
    if frames.dim() == 2:
        frames = frames.unsqueeze(0)
    if frames.dim() != 3 or frames.stride(2) != 1:
        raise InvalidInput("frames must be (n, h, w) with unit column stride")
    return frames


def _stream(frames):
    import torch
    return torch.cuda.current_stream(frames.device).cuda_stream


# ---------------------------------------------------------------- Algorithm 1
def cut_depth_alg1(p_c1_x: float, p_cn_x: float, params: Alg1Params, axial_extent_mm: float) -> float:
    """K |p_c1 - p_cn - L/2| + D, clamped to the image's axial extent (Table I Step 4)."""
    out = C.c_double()
    check(lib().svr_cut_depth_alg1(float(p_c1_x), float(p_cn_x), params.K, params.D, params.L,
                                   float(axial_extent_mm), C.byref(out)))
    return out.value


def axial_extent_mm(calib: Calib) -> float:
    """ImageCalibration::axial_extent_mm (geometry.hpp:174)."""
    return calib.crop_h * calib.scale_y_mm


def cut_rows(cut_mm: float, band_mm: float, calib: Calib):
    r0, r1 = C.c_int32(), C.c_int32()
    check(lib().svr_cut_rows(float(cut_mm), float(band_mm), calib.scale_y_mm, calib.crop_h,
                             C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def apply_cut(frames, cut_mm, band_mm: float, calib: Calib):
    """apply_cut (Table I Step 5 / Table II Step 4) in place on device frames: rows outside
    [cut, cut + band] (axial mm) set to 0.  cut_mm: scalar or one per frame."""
    fr = _dev(frames)
    n, h, w = fr.shape
    cuts = np.broadcast_to(np.asarray(cut_mm, np.float64), (n,))
    r = np.array([cut_rows(c, band_mm, calib) for c in cuts], np.int32).reshape(n, 2)
    r0, r1 = np.ascontiguousarray(r[:, 0]), np.ascontiguousarray(r[:, 1])
    check(lib().svr_apply_cut(fr.data_ptr(), fr.stride(1), fr.stride(0), w, h, n, r0.ctypes.data,
                              r1.ctypes.data, fr.device.index, _stream(fr)))
    return frames


def segment_stream_alg1(frames, poses, calib: Calib, params: Alg1Params = Alg1Params(),
                        band_mm: float = DEFAULTS["band_mm"], p_c1=None) -> CutProfile:
    """Table I end to end: P_c1 from the first frame's pose (or the stream's carried p_c1),
    P_cn per frame, cut in place.  Single pass, constant state."""
    pa = rigid_array(poses)
    ax = ("tx", "ty", "tz")[params.axis]
    p1 = float(pa[0][ax]) if p_c1 is None else float(p_c1)
    ext = axial_extent_mm(calib)
    cuts = np.array([cut_depth_alg1(p1, float(p[ax]), params, ext) for p in pa])
    apply_cut(frames, cuts, band_mm, calib)
    return CutProfile(cuts, "alg1", band_mm)


# ---------------------------------------------------------------- Algorithm 2
def contour_thresholds(calib: Calib, grad_per_mm: float = DEFAULTS["grad_per_mm"],
                       shadow_mm: float = DEFAULTS["shadow_mm"]):
    """Integer thresholds of the contour pin: the 3-row-sum step S(r) - S(r+3) >= ceil(9 sy g)
    (3-row means 3 rows = 3 sy mm apart differing by g levels/mm) and ceil(shadow_mm / sy) rows
    (>= 3) of acoustic shadow below the cortex window."""
    sy = calib.scale_y_mm
    return int(math.ceil(9.0 * sy * grad_per_mm)), max(3, int(math.ceil(shadow_mm / sy - 1e-9)))


def bone_contour(frames, calib: Calib, pct: float = DEFAULTS["pct"],
                 grad_per_mm: float = DEFAULTS["grad_per_mm"], shadow_mm: float = DEFAULTS["shadow_mm"],
                 min_valid_frac: float = DEFAULTS["min_valid_frac"], column_rows: bool = False):
    """Per-frame bone depth (Table II Step 2) on the GPU: bottom-up per column, the first bright
    structure above >= shadow_mm of acoustic shadow with a strong dark-to-bright step is the
    cortex; frame depth = median_lower over columns.  Returns (depth_mm, NaN where no contour;
    valid mask; info dict [; per-column rows])."""
    fr = _dev(frames)
    n, h, w = fr.shape
    grad, shadow = contour_thresholds(calib, grad_per_mm, shadow_mm)
    rows = np.empty(n, np.int32)
    nv = np.empty(n, np.int32)
    thr = np.empty(n, np.int32)
    cr = np.empty((n, w), np.int32) if column_rows else None
    check(lib().svr_bone_contour(fr.data_ptr(), fr.stride(1), fr.stride(0), w, h, n, float(pct), grad,
                                 shadow, float(min_valid_frac), rows.ctypes.data, nv.ctypes.data,
                                 thr.ctypes.data, cr.ctypes.data if cr is not None else None,
                                 fr.device.index, _stream(fr)))
    valid = rows >= 0
    depth = np.where(valid, rows.astype(np.float64) * calib.scale_y_mm, np.nan)
    info = {"rows": rows, "valid_columns": nv, "brightness_threshold": thr, "grad_levels": grad,
            "shadow_rows": shadow}
    return (depth, valid, info, cr) if column_rows else (depth, valid, info)


def smooth_depths(depths, valid=None, window: int = DEFAULTS["window"]) -> np.ndarray:
    """Table II Step 3: gaps bridged linearly, then a sliding median_lower (host C++)."""
    d = np.ascontiguousarray(np.nan_to_num(np.asarray(depths, np.float64), nan=0.0))
    v = np.ascontiguousarray(~np.isnan(np.asarray(depths, np.float64)) if valid is None else valid, np.uint8)
    out = np.empty_like(d)
    check(lib().svr_smooth_depths(d.ctypes.data, v.ctypes.data, len(d), int(window), out.ctypes.data))
    return out


def segment_scan_alg2(frames, calib: Calib, window: int = DEFAULTS["window"],
                      band_mm: float = DEFAULTS["band_mm"], **contour_kw) -> CutProfile:
    """Table II end to end: bone_contour per frame -> smooth_depths -> apply_cut in place.
    Raises AlgorithmFailure when no frame has a contour."""
    depth, valid, _ = bone_contour(frames, calib, **contour_kw)
    if not valid.any():
        raise AlgorithmFailure("no contour in any frame")
    cuts = smooth_depths(depth, valid, window)
    apply_cut(frames, cuts, band_mm, calib)
    return CutProfile(cuts, "alg2", band_mm)


# ---------------------------------------------------------------- VPI baseline
def vpi_fixed_depth(frames, poses, calib: Calib, depth_mm: float, band_mm: float, grid,
                    mode: int = _abi.PROJ_MAX, depth_axis: int = 1) -> np.ndarray:
    """vpi_fixed_depth: apply_cut at a constant depth on every frame,
    reconstruct with skip_zero, coronal projection (u8) along the depth axis."""
    apply_cut(frames, depth_mm, band_mm, calib)
    grid.insert_frames(frames, poses, calib, skip_zero=True)
    return grid.coronal_projection(mode, depth_axis=depth_axis)
