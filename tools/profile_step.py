#!/usr/bin/env python
"""Minimal cfg2 reconstruction step for ncu: frames resident on the device, `--steps` steps of
insert (K1) -> fill (K2) -> depth + band render (K3a/K3b).  No analysis launches, so an ncu
launch list is just the hot path."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import _abi, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--config", default="cfg2")
    a = ap.parse_args()
    wl = synth.CONFIGS[a.config]()
    frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
    for k in range(0, wl.nframes, 4096):
        m = min(4096, wl.nframes - k)
        _abi.check(_abi.lib().svr_synth_frames(frames[k].data_ptr(), wl.w, wl.h, k, m, wl.calib,
                                               _abi.rigid_ptr(np.ascontiguousarray(wl.poses[k:k + m])),
                                               wl.kind, wl.seed, 0, None))
    boxes = [pkg.frame_bounds(wl.grid_desc(), wl.calib, wl.poses[k:k + 1]) for k in range(wl.nframes)]
    u = _abi.Box(min(b.x0 for b in boxes), min(b.y0 for b in boxes), min(b.z0 for b in boxes),
                 max(b.x1 for b in boxes), max(b.y1 for b in boxes), max(b.z1 for b in boxes))
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, accum=wl.accum)
    rp = synth.render_params()
    for _ in range(a.steps):
        grid.insert_frames(frames, wl.poses, wl.calib)
        if wl.accum == _abi.ACC_PNN:
            grid.fill_holes(pkg.dilate(u, 1), 1, pkg.FILL_MEAN, count=False)
            grid.render_coronal(u, rp, 1)
    grid.sync()
    print("ok", grid.stats())


if __name__ == "__main__":
    main()
