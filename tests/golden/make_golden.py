#!/usr/bin/env python
"""Generate the golden fixtures in tests/golden/ (run in the build container, where
/root/reference exists).

Accumulators (sum, count) and per-frame dirty boxes come from oracle/_ref — the reference's own
spinevol::pixel_to_world (geometry.hpp:179-185) driving the SPEC.md:289-297 insert loop — so the
fixtures pin both the C oracle and the CUDA path to the reference's fp64 geometry.  The
BASELINE-only stages (3x3x3 mean fill, SPEC median fill, depth-band render) have no reference
code ("parity unpinned"); their expected arrays are the oracle's.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402
from paper_2412_00058_b200 import synth  # noqa: E402
from paper_2412_00058_b200._abi import Box  # noqa: E402


def calib_fields(c):
    return np.array([c.crop_w, c.crop_h, c.probe, c.scale_x_mm, c.scale_y_mm, c.fan_angle_deg,
                     c.fan_r0_mm, c.fan_r1_mm, c.image_to_transducer.qw, c.image_to_transducer.qx,
                     c.image_to_transducer.qy, c.image_to_transducer.qz, c.image_to_transducer.tx,
                     c.image_to_transducer.ty, c.image_to_transducer.tz], dtype=np.float64)


def make(wl, name, render_kw):
    assert O.ref() is not None, "oracle/_ref must be built (make -C oracle)"
    frames = wl.frames_np()
    frames[:, ::5, ::3] = 0  # a sprinkle of zeros for the skip_zero fixture
    rs, rc, _ = O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, wl.poses, wl.calib,
                                    nthreads=1)
    rs0, rc0, _ = O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, wl.poses, wl.calib,
                                      skip_zero=True, nthreads=1)
    g = O.OracleGrid.for_workload(wl)
    boxes = g.insert_frames(frames, wl.poses, wl.calib)
    assert np.array_equal(g.sum, rs) and np.array_equal(g.count, rc), "oracle != reference"
    mean_fill = g.fill_holes(None, 0, 1)
    fill_mean = g.fill.copy()
    rp = synth.render_params(**render_kw)
    mean, mx, md = g.render(rp)
    g.fill_holes(None, 1, 2)
    fill_median = g.fill.copy()
    out = os.path.join(HERE, name + ".npz")
    np.savez_compressed(
        out, frames=frames, poses=wl.poses.view(np.float64).reshape(-1, 7), calib=calib_fields(wl.calib),
        dims=np.array(wl.dims), voxel_mm=np.array(wl.voxel_mm), origin=np.array(wl.origin),
        sum=rs, count=rc, sum_skip0=rs0, count_skip0=rc0,
        boxes=np.array([b.as_tuple() for b in boxes], dtype=np.int32),
        fill_mean_r1=fill_mean, filled_mean_r1=np.array(mean_fill), fill_median_r2=fill_median,
        render_mean=mean, render_max=mx, render_depth=md,
        render_params=np.array([render_kw[k] for k in ("depth_lo_mm", "depth_hi_mm", "band_above_mm",
                                                       "band_below_mm", "median_radius")], dtype=np.float64))
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    small_render = dict(depth_lo_mm=1.0, depth_hi_mm=12.0, band_above_mm=1.0, band_below_mm=0.5,
                        median_radius=2)
    make(synth.small_linear(), "small_linear", small_render)
    make(synth.small_fan(), "small_fan", dict(depth_lo_mm=8.0, depth_hi_mm=28.0, band_above_mm=2.0,
                                              band_below_mm=1.0, median_radius=2))
