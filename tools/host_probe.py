#!/usr/bin/env python
"""Host-side cost of one cfg2 batch insert call (make_params for 2400 frames + launches) vs its
GPU time: perf_counter around the call without a sync, and CUDA events around the same call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import synth  # noqa: E402

wl = synth.cfg2()
frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
synth.synth_frames_device(wl, frames, 0, wl.nframes, 0)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin)
s = torch.cuda.Stream()
grid.set_stream(s.cuda_stream)
for _ in range(3):
    grid.insert_frames(frames, wl.poses, wl.calib)
grid.sync()
host = []
for _ in range(10):
    t = time.perf_counter()
    grid.insert_frames(frames, wl.poses, wl.calib)
    host.append((time.perf_counter() - t) * 1e3)
grid.sync()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
with torch.cuda.stream(s):
    ev[0].record(s)
    for _ in range(10):
        grid.insert_frames(frames, wl.poses, wl.calib)
    ev[1].record(s)
grid.sync()
print("host ms per call: median %.3f min %.3f; gpu ms per call (10 back to back) %.3f" %
      (sorted(host)[5], min(host), ev[0].elapsed_time(ev[1]) / 10))
