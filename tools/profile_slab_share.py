#!/usr/bin/env python
"""One batch step of the busiest z-slab of an N-GPU split (bench.py slab_shares), for ncu launch
lists:  python tools/profile_slab_share.py N [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import sharding, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
wl = synth.cfg2()
fill_r = wl.fill_radius
ghost = fill_r + synth.CFG4_RENDER["median_radius"]
boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
slabs = sharding.plan_slabs(wl.dims[2], n, ghost)
routed = [sharding.route(boxes, sl.alloc) for sl in slabs]
r = max(range(n), key=lambda i: len(routed[i]))
sl, mine = slabs[r], routed[r]
k0, k1 = int(mine[0]), int(mine[-1]) + 1
frames = torch.empty((k1 - k0, wl.h, wl.w), dtype=torch.uint8, device="cuda")
synth.synth_frames_device(wl, frames, k0, k1 - k0, 0)
poses = wl.poses[k0:k1]
fb = sharding.chunk_boxes(boxes, mine, sl.alloc, chunk=32, dilate=fill_r)
rb = sharding.chunk_boxes(boxes, mine, sl.alloc, chunk=32)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, z_range=sl.alloc)
rp = synth.render_params()
for _ in range(steps):
    grid.insert_frames(frames, poses, wl.calib)
    grid.fill_holes_boxes(fb, fill_r, pkg.FILL_MEAN, count=False)
    grid.render_coronal_boxes(rb, rp, fill_r)
grid.sync()
print("ok", n, r, len(mine), len(fb), len(rb), grid.stats())
