"""Debug helper: cfg2 frames GPU vs oracle, one at a time or as one batch; reports the differing
voxels.  Test infrastructure (uses the oracle).  usage: debug_k1.py [batch] frame..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_00058_b200 as pkg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2412_00058_b200 import synth  # noqa: E402

wl = synth.cfg2()
args = sys.argv[1:]
batch = bool(args) and args[0] == "batch"
if batch:
    args = args[1:]
idx = [int(a) for a in args] or list(range(0, 40))
groups = [idx] if batch else [[k] for k in idx]
for grp in groups:
    fr = np.stack([wl.frames_np(k, 1)[0] for k in grp])
    g = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    g.insert_frames(fr, wl.poses[grp], wl.calib)
    s, c = g.accumulators()
    st = g.stats()
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames_mt(fr, wl.poses[grp], wl.calib)
    bad = np.argwhere((c != ref.count) | (s != ref.sum))
    print("frames", grp[:4], "bad", len(bad), "stats", st, flush=True)
    if len(bad):
        for b in bad[:60]:
            z, y, x = b
            print("  z y x", z, y, x, "gpu c/s", c[z, y, x], s[z, y, x], "ref", ref.count[z, y, x], ref.sum[z, y, x])
        break
    g.close()
