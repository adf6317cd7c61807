#!/usr/bin/env python
"""A few cfg2 frames through svr_frame_step (the per-frame CUDA graph) for an ncu launch list."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import synth  # noqa: E402

wl = synth.cfg2(nframes=1300)
frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
synth.synth_frames_device(wl, frames, 0, wl.nframes, 0)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin)
rp = synth.render_params()
for k in range(1200, 1300):
    grid.frame_step(frames[k], wl.poses[k:k + 1], wl.calib, 1, rp)
grid.sync()
print("ok")
