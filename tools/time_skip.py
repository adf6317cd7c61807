#!/usr/bin/env python
"""Insert-only wall time of the cfg2 batch with and without skip_zero (device-resident frames),
plain frames and frames cut to a 150-row band (apply_cut-like: rows outside the band zeroed).
usage: time_skip.py [NFRAMES]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00058_b200 as pkg  # noqa: E402
from paper_2412_00058_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2400
wl = synth.cfg2(nframes=n)
frames = torch.empty((n, wl.h, wl.w), dtype=torch.uint8, device="cuda")
synth.synth_frames_device(wl, frames, 0, n)
cut = frames.clone()
cut[:, :150, :] = 0
cut[:, 300:, :] = 0
for name, fr, skip in (("plain", frames, False), ("plain skip_zero", frames, True), ("band skip_zero", cut, True)):
    g = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    ts = []
    for _ in range(4):
        g.sync()
        t0 = time.perf_counter()
        g.insert_frames(fr, wl.poses, wl.calib, skip_zero=skip)
        g.sync()
        ts.append((time.perf_counter() - t0) * 1e3)
    st = g.stats()
    print(name, "ms", [round(t, 3) for t in ts], "launches", st["kernel_launches"], "skipped", st["pixels_skipped_zero"])
    g.close()
