"""The C++ host API (include/spinevol_b200/reconstruct.hpp) driven from a C++ program, as a
reference caller would use it; with -DSPINEVOL_B200_REFERENCE_TYPES it consumes the reference's
own spinevol::Image8 / RigidTransform / ImageCalibration."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O
from paper_2412_00058_b200 import _abi, dilate, synth

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")
BINS = [os.path.join(HERE, b) for b in ("wrapper_demo", "wrapper_demo_ref")]


def _built():
    if not os.path.exists(BINS[0]):
        subprocess.run(["make", "-C", HERE], check=True, stdout=subprocess.DEVNULL)
    return [b for b in BINS if os.path.exists(b)]


def test_cpp_host_api_cpu():
    bins = _built()
    assert bins
    for b in bins:
        r = subprocess.run([b, "host"], capture_output=True, text=True)
        assert r.returncode == 0 and "host ok" in r.stdout, (b, r.stdout, r.stderr)


@pytest.mark.gpu
def test_cpp_host_api_reconstruct_gpu():
    wl = synth.small_linear(nframes=10)
    frames = wl.frames_np()
    ref = O.OracleGrid.for_workload(wl)
    boxes = ref.insert_frames(frames, wl.poses, wl.calib)
    u = _abi.Box(min(b.x0 for b in boxes), min(b.y0 for b in boxes), min(b.z0 for b in boxes),
                 max(b.x1 for b in boxes), max(b.y1 for b in boxes), max(b.z1 for b in boxes))
    ref.fill_holes(dilate(u, 2), 1, 2)
    proj = ref.coronal_projection(0, 2)
    nvox = int(np.prod(wl.dims))
    with tempfile.TemporaryDirectory() as d:
        inp = os.path.join(d, "in.bin")
        with open(inp, "wb") as f:
            f.write(np.array(list(wl.dims) + [wl.nframes, wl.w, wl.h], np.int32).tobytes())
            f.write(np.array([wl.voxel_mm, *wl.origin], np.float64).tobytes())
            f.write(bytes(wl.calib))
            f.write(np.ascontiguousarray(wl.poses).tobytes())
            f.write(np.ascontiguousarray(frames).tobytes())
        for b in _built():
            out = os.path.join(d, "out.bin")
            r = subprocess.run([b, "run", inp, out], capture_output=True, text=True)
            assert r.returncode == 0, (b, r.stdout, r.stderr)
            raw = open(out, "rb").read()
            s = np.frombuffer(raw, np.uint32, nvox)
            c = np.frombuffer(raw, np.uint16, nvox, nvox * 4)
            fl = np.frombuffer(raw, np.uint32, nvox, nvox * 6)
            pj = np.frombuffer(raw, np.uint8, -1, nvox * 10)
            assert np.array_equal(s, ref.sum.ravel()) and np.array_equal(c, ref.count.ravel())
            assert np.array_equal(fl, ref.fill.ravel())
            assert np.array_equal(pj, proj.ravel())
