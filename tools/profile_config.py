#!/usr/bin/env python
"""Insert-only launches of one BASELINE config (device-resident frames) for ncu: cfg1 / cfg3 /
cfg5 (cfg5 on a 64-plane slab so it fits beside other processes; "cfg5mid": 620 consecutive cfg5
frames that lie wholly inside a 1200-plane slab, 19 GB -- no out-of-slab pixels, so the counters
are those of the full-volume run).  usage: profile_config.py NAME [STEPS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import sharding, synth  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mid = name == "cfg5mid"
if mid:
    name = "cfg5"
wl = synth.CONFIGS[name]()
z_range, poses, idx = None, wl.poses, None
if mid:
    z_range = (1200, 2400)
    idx = list(range(760, 1380))
    poses = wl.poses[760:1380]
elif name == "cfg5":
    z_range = (1200, 1264)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    idx = sharding.route(boxes, z_range)
    poses = wl.poses[idx]
n = len(poses)
frames = torch.empty((n, wl.h, wl.w), dtype=torch.uint8, device="cuda")
if idx is None:
    synth.synth_frames_device(wl, frames, 0, n)
else:
    for i, k in enumerate(idx):
        synth.synth_frames_device(wl, frames[i:i + 1], int(k), 1)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, z_range=z_range, accum=wl.accum)
import time  # noqa: E402

grid.sync()
for i in range(steps):
    t0 = time.perf_counter()
    grid.insert_frames(frames, poses, wl.calib)
    grid.sync()
    print("insert wall ms", round((time.perf_counter() - t0) * 1e3, 3), "frames", n)
print("ok", name, n, grid.stats())
