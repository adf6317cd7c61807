"""Load a golden fixture (tests/golden/*.npz, made by tests/golden/make_golden.py)."""
import os

import numpy as np

from paper_2412_00058_b200 import _abi, synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Fixture:
    def __init__(self, name):
        d = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.d = d
        c = d["calib"]
        i2t = synth.rigid(c[8:12], c[12:15])
        if int(c[2]) == _abi.PROBE_FAN:
            self.calib = synth.fan_calib(int(c[1]), int(c[0]), c[5], c[6], c[7], i2t)
        else:
            self.calib = synth.linear_calib(int(c[0]), int(c[1]), c[3], c[4], i2t)
        self.frames = d["frames"]
        self.poses = np.ascontiguousarray(d["poses"]).view(_abi.RIGID_DTYPE).reshape(-1)
        self.dims = tuple(int(v) for v in d["dims"])
        self.voxel_mm = float(d["voxel_mm"])
        self.origin = tuple(float(v) for v in d["origin"])
        rp = d["render_params"]
        self.render = synth.render_params(depth_lo_mm=rp[0], depth_hi_mm=rp[1], band_above_mm=rp[2],
                                          band_below_mm=rp[3], median_radius=int(rp[4]))

    def __getitem__(self, k):
        return self.d[k]


FIXTURES = ("small_linear", "small_fan")
