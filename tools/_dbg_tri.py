import sys, os, dataclasses, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_00058_b200 as pkg
from paper_2412_00058_b200 import synth
wl = dataclasses.replace(synth.cfg5(nframes=2, dims=(160, 120, 40)), origin=(70.0, 20.0, 9.5))
frames = wl.frames_np()
print("frames", frames.shape, flush=True)
grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0, accum=wl.accum)
print("grid ok", flush=True)
t = time.time()
grid.insert_frames(frames[:1], wl.poses[:1], wl.calib)
print("enqueued", time.time() - t, flush=True)
grid.sync()
print("synced", time.time() - t, grid.stats(), flush=True)
ws, wt = grid.trilinear()
print("sum", float(wt.sum()), flush=True)
