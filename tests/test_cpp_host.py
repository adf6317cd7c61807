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


@pytest.mark.gpu
@pytest.mark.parametrize("nslab", [1, 3])
def test_cpp_sharded_volume_gpu(nslab):
    """A C++ caller runs the z-slab sharded path (spinevol_b200::ShardedVolume over the
    svr_sharded_* C-ABI) without Python: accumulators and the gathered cfg4 render equal one
    unsharded volume."""
    import paper_2412_00058_b200 as pkg
    wl = synth.cfg1()
    frames = wl.frames_np()
    one = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    _, u = one.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    one.fill_holes(pkg.dilate(u, 1), 1, pkg.FILL_MEAN)
    one.render_coronal(u, synth.render_params(), 1)
    s1, c1 = one.accumulators()
    m1, x1, d1 = one.read_coronal()
    nvox = int(np.prod(wl.dims))
    ncol = wl.dims[0] * wl.dims[2]
    with tempfile.TemporaryDirectory() as d:
        inp = os.path.join(d, "in.bin")
        with open(inp, "wb") as f:
            f.write(np.array(list(wl.dims) + [wl.nframes, wl.w, wl.h], np.int32).tobytes())
            f.write(np.array([wl.voxel_mm, *wl.origin], np.float64).tobytes())
            f.write(bytes(wl.calib))
            f.write(np.ascontiguousarray(wl.poses).tobytes())
            f.write(np.ascontiguousarray(frames).tobytes())
        out = os.path.join(d, "out.bin")
        r = subprocess.run([_built()[0], "shard", inp, out, str(nslab)], capture_output=True, text=True)
        assert r.returncode == 0, (r.stdout, r.stderr)
        raw = open(out, "rb").read()
        o = 0
        s = np.frombuffer(raw, np.uint32, nvox, o); o += 4 * nvox
        c = np.frombuffer(raw, np.uint16, nvox, o); o += 2 * nvox
        m = np.frombuffer(raw, np.float32, ncol, o); o += 4 * ncol
        x = np.frombuffer(raw, np.float32, ncol, o); o += 4 * ncol
        dep = np.frombuffer(raw, np.int32, ncol, o)
    assert np.array_equal(s, s1.ravel()) and np.array_equal(c, c1.ravel())
    assert np.array_equal(m, m1.ravel()) and np.array_equal(x, x1.ravel()) and np.array_equal(dep, d1.ravel())
