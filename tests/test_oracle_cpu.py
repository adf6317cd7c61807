"""CPU suite (no GPU): the oracle pinned against the reference's own headers (oracle/_ref),
the SPEC known-answer tests, the golden fixtures, the host-side ABI (geometry, routing, slab
plan, error mapping), the exported symbol set, and the 2-rank gloo slab-sharding path."""
import ctypes as C
import math
import os
import re
import socket
import tempfile

import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import _abi, sharding, synth
from golden_util import FIXTURES, Fixture

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (reference headers) not built")


def _rot_z(deg):
    return synth.quat_axis_angle((0, 0, 1), math.radians(deg))


def _rand_rigid(rng, t=50.0):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    return synth.rigid(q, rng.uniform(-t, t, 3))


# ------------------------------------------------------------------ SPEC known answers
def test_spec_pixel_to_world_kat():
    """px (100,200), scale 0.1, transducer translation (5,0,0) -> (15,20,0)."""
    c = synth.linear_calib(512, 512, 0.1, 0.1, synth.rigid(t=(5, 0, 0)))
    assert O.pixel_to_world(100, 200, c, synth.rigid()) == (15.0, 20.0, 0.0)
    assert pkg.pixel_to_world(100, 200, c, synth.rigid()) == (15.0, 20.0, 0.0)
    assert O.pixel_to_world(0, 0, synth.linear_calib(4, 4, 1, 1), synth.rigid()) == (0.0, 0.0, 0.0)
    with pytest.raises(pkg.InvalidInput):
        pkg.pixel_to_world(512, 0, c, synth.rigid())


def test_spec_compose_kat():
    """compose(rot_z(90), translate(1,0,0)) applied to the origin -> (0,1,0)."""
    r = pkg.compose(synth.rigid(_rot_z(90)), synth.rigid(t=(1, 0, 0)))
    assert abs(r.tx) < 1e-9 and abs(r.ty - 1) < 1e-9 and abs(r.tz) < 1e-9
    ident = pkg.compose(synth.rigid(), synth.rigid(_rot_z(30), (1, 2, 3)))
    assert abs(ident.tx - 1) < 1e-12 and abs(ident.qz - math.sin(math.radians(15))) < 1e-12


def test_spec_interpolate_kats():
    """endpoints exact, translation midpoint, slerp 45 deg."""
    t = [0.0, 10.0]
    poses = [synth.rigid(_rot_z(0), (0, 0, 0)), synth.rigid(_rot_z(90), (10, 0, 0))]
    a = pkg.interpolate_pose(t, poses, 10.0)
    assert (a.qw, a.qz, a.tx) == (poses[1].qw, poses[1].qz, 10.0)
    m = pkg.interpolate_pose(t, poses, 5.0)
    assert abs(m.tx - 5.0) < 1e-12
    q45 = _rot_z(45)
    assert abs(m.qw - q45[0]) < 1e-9 and abs(m.qz - q45[3]) < 1e-9
    with pytest.raises(pkg.InvalidInput):
        pkg.interpolate_pose(t, poses, 11.0)


def test_spec_insert_kats():
    """one pixel 200 -> sum 200, count 1, value 200; 100 then 200 -> 150."""
    c = synth.linear_calib(1, 1, 1.0, 1.0)
    g = O.OracleGrid((4, 4, 4), 1.0)
    b = g.insert_frame(np.array([[200]], np.uint8), synth.rigid(t=(1, 2, 3)), c)
    assert (g.sum[3, 2, 1], g.count[3, 2, 1]) == (200, 1) and b.as_tuple() == (1, 2, 3, 1, 2, 3)
    assert g.values()[3, 2, 1] == 200
    g2 = O.OracleGrid((4, 4, 4), 1.0)
    g2.insert_frame(np.array([[100]], np.uint8), synth.rigid(t=(1, 1, 1)), c)
    g2.insert_frame(np.array([[200]], np.uint8), synth.rigid(t=(1, 1, 1)), c)
    assert g2.values()[1, 1, 1] == 150
    # out-of-bounds pixel: dropped and counted, empty box
    g3 = O.OracleGrid((4, 4, 4), 1.0)
    b3 = g3.insert_frame(np.array([[9]], np.uint8), synth.rigid(t=(-5, 0, 0)), c)
    assert b3.empty() and g3.stats["oob"] == 1 and g3.count.sum() == 0


def test_spec_fill_kats():
    """6 face neighbours of 100 -> 100; no neighbour -> unfilled;
    neighbours {90,100,255} -> 100 (lower median, core.hpp:93-99)."""
    for mode in (0, 1):
        g = O.OracleGrid((5, 5, 5), 1.0)
        for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            g.sum[2 + d[2], 2 + d[1], 2 + d[0]] = 100
            g.count[2 + d[2], 2 + d[1], 2 + d[0]] = 1
        g.fill_holes(None, mode, 1)
        f = g.fill[2, 2, 2]
        assert (f >> 16) == 6
        assert (f & 0xFFFF) == (600 if mode == 0 else 100)
        assert g.fill[0, 0, 0] == 0  # no non-empty neighbour within radius 1 of a corner? it has none
    g = O.OracleGrid((3, 3, 3), 1.0)
    for x, v in ((0, 90), (1, 100), (2, 255)):
        g.sum[0, 0, x], g.count[0, 0, x] = v, 1
    g.fill_holes(None, 1, 2)
    assert (g.fill[2, 2, 2] & 0xFFFF) == 100
    if O.ref() is not None:
        assert O.ref().ref_median_lower((C.c_double * 3)(90, 100, 255), 3) == 100.0


def test_value_rounding_integer_form():
    """value = round(sum/count) == (2 sum + count) // (2 count)."""
    rng = np.random.default_rng(0)
    c = rng.integers(1, 65535, 200000)
    s = (rng.random(200000) * 255 * c).astype(np.int64)
    assert np.array_equal((2 * s + c) // (2 * c), np.floor(s / c + 0.5).astype(np.int64))


# ------------------------------------------------------------------ pinned to the reference
@needs_ref
def test_pixel_to_world_bitexact_vs_reference():
    R = O.ref()
    rng = np.random.default_rng(1)
    for _ in range(3000):
        c = synth.linear_calib(640, 480, rng.uniform(0.05, 0.5), rng.uniform(0.05, 0.5),
                               _rand_rigid(rng, 30))
        pose = _rand_rigid(rng, 400)
        col, row = float(rng.integers(0, 640)), float(rng.integers(0, 480))
        out = (C.c_double * 3)()
        R.ref_pixel_to_world(col, row, C.byref(c), C.byref(pose), out)
        assert O.pixel_to_world(col, row, c, pose) == tuple(out)
        assert pkg.pixel_to_world(col, row, c, pose) == tuple(out)


@needs_ref
def test_from_matrix4_bitexact_vs_reference():
    R = O.ref()
    rng = np.random.default_rng(2)
    cases = [np.eye(3), np.diag([1, -1, -1]), np.diag([-1, 1, -1]), np.diag([-1, -1, 1])]
    for _ in range(500):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        cases.append(np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                               [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                               [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]]))
    for rot in cases:
        m = np.eye(4)
        m[:3, :3] = rot
        m[:3, 3] = rng.uniform(-100, 100, 3)
        a = pkg.pose_from_matrix4(m)
        b = _abi.Rigid()
        R.ref_from_matrix4((C.c_double * 16)(*m.reshape(16)), C.byref(b))
        assert [getattr(a, f) for f, _ in a._fields_] == [getattr(b, f) for f, _ in b._fields_]
    bad = np.eye(4)
    bad[3, 0] = 0.5
    with pytest.raises(pkg.InvalidInput):
        pkg.pose_from_matrix4(bad)


@needs_ref
def test_compose_and_interpolate_bitexact_vs_reference():
    R = O.ref()
    rng = np.random.default_rng(3)
    for _ in range(300):
        a, b = _rand_rigid(rng), _rand_rigid(rng)
        r1 = pkg.compose(a, b)
        r2 = _abi.Rigid()
        R.ref_compose(C.byref(a), C.byref(b), C.byref(r2))
        assert [getattr(r1, f) for f, _ in r1._fields_] == [getattr(r2, f) for f, _ in r2._fields_]
    ts = np.cumsum(rng.uniform(1, 30, 40))
    poses = [_rand_rigid(rng) for _ in range(40)]
    pa = _abi.rigid_array(poses)
    for t in np.concatenate([ts, rng.uniform(ts[0], ts[-1], 200)]):
        r1 = pkg.interpolate_pose(ts, poses, t)
        r2 = _abi.Rigid()
        R.ref_interpolate_pose(ts.ctypes.data_as(C.POINTER(C.c_double)), _abi.rigid_ptr(pa), 40, t,
                               C.byref(r2))
        assert [getattr(r1, f) for f, _ in r1._fields_] == [getattr(r2, f) for f, _ in r2._fields_]


@needs_ref
@pytest.mark.parametrize("maker", [synth.small_linear, synth.small_fan])
@pytest.mark.parametrize("skip_zero", [False, True])
def test_oracle_insert_bitexact_vs_reference(maker, skip_zero):
    wl = maker()
    frames = wl.frames_np()
    frames[:, ::4, ::3] = 0
    g = O.OracleGrid.for_workload(wl)
    g.insert_frames(frames, wl.poses, wl.calib, skip_zero)
    for nth in (1, 3):
        s, c, ins = O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, wl.poses, wl.calib,
                                        skip_zero=skip_zero, nthreads=nth)
        assert np.array_equal(s, g.sum) and np.array_equal(c, g.count) and ins == g.stats["inserted"]
    g2 = O.OracleGrid.for_workload(wl)
    g2.insert_frames_mt(frames, wl.poses, wl.calib, skip_zero, nthreads=4)
    assert np.array_equal(g2.sum, g.sum) and np.array_equal(g2.count, g.count)
    assert g2.stats["inserted"] == g.stats["inserted"] and g2.stats["oob"] == g.stats["oob"]


@needs_ref
def test_oracle_cfg1_subset_vs_reference():
    wl = synth.cfg1()
    idx = np.arange(0, wl.nframes, 10)
    frames = np.stack([wl.frames_np(int(k), 1)[0] for k in idx])
    g = O.OracleGrid.for_workload(wl)
    g.insert_frames_mt(frames, wl.poses[idx], wl.calib, nthreads=4)
    s, c, _ = O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, wl.poses[idx], wl.calib,
                                  nthreads=4)
    assert np.array_equal(s, g.sum) and np.array_equal(c, g.count)


# ------------------------------------------------------------------ golden fixtures
@pytest.mark.parametrize("name", FIXTURES)
def test_golden_fixture_oracle(name):
    fx = Fixture(name)
    g = O.OracleGrid(fx.dims, fx.voxel_mm, fx.origin)
    boxes = g.insert_frames(fx.frames, fx.poses, fx.calib)
    assert np.array_equal(g.sum, fx["sum"]) and np.array_equal(g.count, fx["count"])
    assert np.array_equal(np.array([b.as_tuple() for b in boxes]), fx["boxes"])
    assert g.fill_holes(None, 0, 1) == int(fx["filled_mean_r1"])
    assert np.array_equal(g.fill, fx["fill_mean_r1"])
    mean, mx, md = g.render(fx.render)
    assert np.array_equal(md, fx["render_depth"])
    np.testing.assert_allclose(mean, fx["render_mean"], rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, fx["render_max"], rtol=1e-5, atol=0)
    g.fill_holes(None, 1, 2)
    assert np.array_equal(g.fill, fx["fill_median_r2"])
    g0 = O.OracleGrid(fx.dims, fx.voxel_mm, fx.origin)
    g0.insert_frames(fx.frames, fx.poses, fx.calib, skip_zero=True)
    assert np.array_equal(g0.sum, fx["sum_skip0"]) and np.array_equal(g0.count, fx["count_skip0"])


# ------------------------------------------------------------------ oracle properties
def test_oracle_incremental_equals_batch_and_order():
    wl = synth.small_linear(nframes=14)
    frames = wl.frames_np()
    rp = synth.render_params(depth_lo_mm=1.0, depth_hi_mm=12.0, band_above_mm=1.0, band_below_mm=0.5)
    inc = O.OracleGrid.for_workload(wl)
    for k in range(wl.nframes):
        b = pkg.frame_bounds(wl.grid_desc(), wl.calib, wl.poses[k:k + 1])
        inc.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
        if not b.empty():
            inc.fill_holes(pkg.dilate(b, 1), 0, 1)
            inc.render(rp, b, 1)
    bat = O.OracleGrid.for_workload(wl)
    perm = np.random.default_rng(5).permutation(wl.nframes)
    bat.insert_frames(frames[perm], wl.poses[perm], wl.calib)
    bat.fill_holes(None, 0, 1)
    bat.render(rp)
    for a, b in ((inc.sum, bat.sum), (inc.count, bat.count), (inc.fill, bat.fill),
                 (inc.mean, bat.mean), (inc.max, bat.max), (inc.mdepth, bat.mdepth)):
        assert np.array_equal(a, b)
    # hole-fill idempotence
    f = bat.fill.copy()
    bat.fill_holes(None, 0, 1)
    assert np.array_equal(f, bat.fill)


def test_frame_bounds_contain_tight_boxes():
    for wl in (synth.small_linear(nframes=10), synth.small_fan(), synth.cfg1(nframes=30)):
        frames = wl.frames_np()
        g = O.OracleGrid.for_workload(wl)
        for k in range(wl.nframes):
            tight = g.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
            b = pkg.frame_bounds(wl.grid_desc(), wl.calib, wl.poses[k:k + 1])
            if not tight.empty():
                assert b.x0 <= tight.x0 and b.y0 <= tight.y0 and b.z0 <= tight.z0
                assert b.x1 >= tight.x1 and b.y1 >= tight.y1 and b.z1 >= tight.z1


# ------------------------------------------------------------------ host ABI
def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "spinevol_b200.h")).read()
    names = set(re.findall(r"\b(svr_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 28
    L = C.CDLL(_abi.LIB_PATH)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert names == set(_abi.SIGNATURES), names ^ set(_abi.SIGNATURES)


def test_host_errors_map_to_reference_exceptions():
    wl = synth.small_linear()
    bad = synth.linear_calib(wl.w, wl.h, -1.0, 0.2)
    with pytest.raises(pkg.InvalidInput):
        pkg.frame_bounds(wl.grid_desc(), bad, wl.poses[:1])
    g = wl.grid_desc()
    g.voxel_mm = 0.0
    with pytest.raises(pkg.InvalidInput):
        pkg.frame_bounds(g, wl.calib, wl.poses[:1])
    if _abi.lib().svr_device_count() == 0:
        with pytest.raises(pkg.DeviceError):
            pkg.VoxelGrid((8, 8, 8))


def test_slab_plan_and_routing():
    for nz, n, gh in ((2000, 8, 3), (256, 2, 4), (7, 7, 0), (100, 3, 3)):
        sl = sharding.plan_slabs(nz, n, gh)
        assert sl[0].owned[0] == 0 and sl[-1].owned[1] == nz
        for a, b in zip(sl, sl[1:]):
            assert a.owned[1] == b.owned[0]
        for s in sl:
            assert s.alloc[0] == max(0, s.owned[0] - gh) and s.alloc[1] == min(nz, s.owned[1] + gh)
    with pytest.raises(pkg.InvalidInput):
        sharding.plan_slabs(4, 8, 0)
    wl = synth.cfg2(nframes=240)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    sl = sharding.plan_slabs(wl.dims[2], 8, 3)
    routed = [set(sharding.route(boxes, s.alloc).tolist()) for s in sl]
    assert set().union(*routed) == set(range(wl.nframes))
    assert sum(len(r) for r in routed) < 1.2 * wl.nframes  # a frame meets 1-2 slabs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_slab_sharding_matches_unsharded():
    import torch.multiprocessing as mp

    from oracle import slab_check
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.txt")
        mp.start_processes(slab_check.worker, args=(2, _free_port(), out), nprocs=2, join=True,
                           start_method="spawn")
        res = open(out).read()
    assert res.startswith("ok"), res



def test_oracle_mt_fill_render_equal_single_thread():
    """The multithreaded oracle fill / render over box lists (the CPU baseline of the bench step)
    equal the single-threaded functions box by box."""
    from paper_2412_00058_b200 import sharding
    wl = synth.cfg1(nframes=60)
    frames = wl.frames_np()
    a = O.OracleGrid.for_workload(wl)
    a.insert_frames_mt(frames, wl.poses, wl.calib)
    b = O.OracleGrid.for_workload(wl)
    b.sum[...] = a.sum
    b.count[...] = a.count
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    idx = np.arange(len(boxes))
    fb = sharding.chunk_boxes(boxes, idx, (0, wl.dims[2]), chunk=16, dilate=1)
    rb = sharding.chunk_boxes(boxes, idx, (0, wl.dims[2]), chunk=16)
    for bx in fb:
        a.fill_holes(bx, 0, 1)
    b.fill_holes_boxes_mt(fb, 0, 1, nthreads=5)
    assert np.array_equal(a.fill, b.fill)
    rp = synth.render_params()
    a.render(rp, None, 1)  # single-threaded: every column
    m1, x1, d1 = a.mean.copy(), a.max.copy(), a.mdepth.copy()
    b.render_boxes_mt(rp, [pkg.Box(0, 0, 0, wl.dims[0] - 1, wl.dims[1] - 1, wl.dims[2] - 1)], 1, nthreads=7)
    assert np.array_equal(b.mdepth, d1) and np.array_equal(b.mean, m1) and np.array_equal(b.max, x1)
