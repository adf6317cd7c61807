#!/usr/bin/env python
"""One bench-identical cfg2 batch step (chunked dirty regions) for ncu launch lists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import sharding, synth  # noqa: E402

wl = synth.cfg2()
frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
synth.synth_frames_device(wl, frames, 0, wl.nframes, 0)
boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
alloc = (0, wl.dims[2])
idx = np.arange(wl.nframes)
fb = sharding.chunk_boxes(boxes, idx, alloc, 32, 1)
rb = sharding.chunk_boxes(boxes, idx, alloc, 32)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin)
rp = synth.render_params()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for _ in range(steps):
    grid.insert_frames(frames, wl.poses, wl.calib)
    grid.fill_holes_boxes(fb, 1, pkg.FILL_MEAN, count=False)
    grid.render_coronal_boxes(rb, rp, 1)
grid.sync()
print("ok", grid.stats())
