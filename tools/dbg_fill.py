import paper_2412_00058_b200 as pkg, numpy as np
from paper_2412_00058_b200 import synth
wl = synth.cfg1(nframes=20)
fr = wl.frames_np()
g = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin)
g.insert_frames(fr, wl.poses, wl.calib)
print(g.fill_holes(None, 1, pkg.FILL_MEAN))
