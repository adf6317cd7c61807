"""GPU parity at the benchmarked sizes and on adversarial geometries (the CUDA path through the
C-ABI against the multithreaded CPU oracle, bit for bit).

* cfg2 in full (2400 x 512 x 480 frames into 500 x 267 x 2000 voxels): accumulators, every
  frame's DirtyRegion, the mean fill of the bench's per-z-chunk dirty boxes and the cfg4
  depth-band render (depths, mean, max) -- SPEC.md:297 brute-force re-binning at size.
* cfg3 in full (1800 fan frames): accumulators and per-frame boxes.
* Adversarial geometries for the certified rounding filter: axis-aligned and
  90-degree poses with half-voxel pixel spacing (exact .5 ties on every other pixel), poses near
  the 2^-16 tie-window refusal limit, and anisotropic pixels that would overflow the insert
  kernel's packed 12-bit shared count on a 128-row tile.
"""
import math

import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import sharding, synth

pytestmark = pytest.mark.gpu


def _grid(wl, **kw):
    return pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0, accum=wl.accum, **kw)


def _device_frames(wl):
    import torch
    frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
    synth.synth_frames_device(wl, frames, 0, wl.nframes)
    return frames, frames.cpu().numpy()


def _assert_acc(grid, ref, what):
    s, c = grid.accumulators()
    if not np.array_equal(c, ref.count):
        bad = np.argwhere(c != ref.count)
        raise AssertionError("%s: count differs at %d voxels, first (z, y, x) %s" % (what, len(bad), bad[:5]))
    assert np.array_equal(s, ref.sum), "%s: sum differs" % what


def _assert_boxes(gb, rb, what):
    g = [b.as_tuple() for b in gb]
    r = [b.as_tuple() for b in rb]
    bad = [k for k in range(len(r)) if g[k] != r[k]]
    assert not bad, "%s: %d dirty boxes differ, first frame %d: %s vs %s" % (what, len(bad), bad[0], g[bad[0]], r[bad[0]])


def test_cfg2_full_size_bitexact_vs_oracle():
    wl = synth.cfg2()
    dev, host = _device_frames(wl)
    grid = _grid(wl)
    gboxes, _ = grid.insert_frames(dev, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = ref.insert_frames_mt_boxes(host, wl.poses, wl.calib)
    _assert_boxes(gboxes, rboxes, "cfg2")
    _assert_acc(grid, ref, "cfg2")
    st = grid.stats()
    assert st["pixels_inserted"] == ref.stats["inserted"] == wl.nframes * wl.w * wl.h
    assert st["tiles_table"] == wl.nframes * 8 * 4  # every 64 x 128 tile through K1's table
    assert st["pixels_oob"] == ref.stats["oob"]
    # the bench step's fill: mean r = 1 over the per-z-chunk dirty boxes (+1)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    fb = sharding.chunk_boxes(boxes, np.arange(len(boxes)), (0, wl.dims[2]), chunk=32, dilate=1)
    n_gpu = grid.fill_holes_boxes(fb, 1, pkg.FILL_MEAN)
    n_ref = 0
    for b in fb:
        n_ref += ref.fill_holes(b, 0, 1)
    assert np.array_equal(grid.fill_layer(), ref.fill), "cfg2 fill layer differs"
    assert n_gpu <= n_ref  # (the oracle counts voxels of overlapping boxes once per box)
    # cfg4: the depth-band render of the filled cfg2 volume, all columns
    rp = synth.render_params()
    grid.render_coronal(None, rp, 1)
    mean, mx, dep = grid.read_coronal()
    rmean, rmx, rdep = ref.render(rp)
    assert np.array_equal(dep, rdep), "cfg4 depths differ at %d columns" % int((dep != rdep).sum())
    np.testing.assert_allclose(mean, rmean, rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, rmx, rtol=1e-5, atol=0)
    grid.close()


def test_cfg3_full_size_bitexact_vs_oracle():
    wl = synth.cfg3()
    dev, host = _device_frames(wl)
    grid = _grid(wl)
    gboxes, _ = grid.insert_frames(dev, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = ref.insert_frames_mt_boxes(host, wl.poses, wl.calib)
    _assert_boxes(gboxes, rboxes, "cfg3")
    _assert_acc(grid, ref, "cfg3")
    st = grid.stats()
    assert st["pixels_inserted"] == ref.stats["inserted"]
    assert st["pixels_oob"] == ref.stats["oob"]
    grid.close()


# ------------------------------------------------------------------ adversarial geometries
def _rot(axis, deg):
    return synth.quat_axis_angle(axis, math.radians(deg))


def _workload(name, w, h, sx, sy, voxel, dims, origin, poses, i2t=None, seed=21):
    calib = synth.linear_calib(w, h, sx, sy, i2t)
    arr = np.zeros(len(poses), dtype=synth._abi.RIGID_DTYPE)
    for k, (q, t) in enumerate(poses):
        arr[k] = (*q, *t)
    return synth.Workload(name, calib, dims, voxel, origin, arr, 0, seed)


def _check_vs_oracle(wl, frames=None, what=""):
    frames = wl.frames_np() if frames is None else frames
    grid = _grid(wl)
    gboxes, _ = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = [ref.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib) for k in range(wl.nframes)]
    _assert_boxes(gboxes, rboxes, what)
    _assert_acc(grid, ref, what)
    st = grid.stats()
    assert st["pixels_inserted"] == ref.stats["inserted"] and st["pixels_oob"] == ref.stats["oob"], what
    # the per-frame API path (one frame per launch: the small-launch tile shape) agrees too
    one = _grid(wl)
    for k in range(wl.nframes):
        b = one.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
        assert b.as_tuple() == rboxes[k].as_tuple(), what
    _assert_acc(one, ref, what + " (per frame)")
    st1 = one.stats()
    grid.close()
    one.close()
    return st, st1


def test_half_voxel_spacing_axis_aligned_ties():
    """sx = voxel / 2, sy = voxel / 4 and identity / 90 / 180 / 270-degree poses with integer or
    half-integer voxel translations: u = col / 2 + k puts every other pixel exactly on a .5
    tie in real arithmetic; the fp64 chain decides them (round half away from zero) and the GPU
    must agree through the exact pass."""
    v = 0.5
    poses = []
    for k, (ax, deg) in enumerate([((0, 0, 1), 0.0), ((0, 0, 1), 90.0), ((0, 0, 1), 180.0),
                                   ((0, 0, 1), 270.0), ((1, 0, 0), 90.0), ((0, 1, 0), 90.0)]):
        t = (20.0 + 0.25 * (k % 2), 18.0 + 0.25 * (k // 2 % 2), 6.0 + 0.5 * k)
        poses.append((_rot(ax, deg), t))
    # (sy = voxel / 4 keeps every pose's 32 x 64-pixel tile inside the shared table, so the
    # tile kernel, not the direct fallback, meets the ties)
    wl = _workload("half_voxel", 64, 64, v / 2, v / 4, v, (96, 96, 40), (0.0, 0.0, 0.0), poses)
    st, st1 = _check_vs_oracle(wl, what="half-voxel ties")
    assert st["exact_fallbacks"] > 1000  # the ties really went through the exact chain
    # per frame, the z-rotated frames go through the shared-table kernel (and its deferred
    # chunks); frames turned 90 degrees about x or y leave the plane condition of its flush
    # (|n_x| + |n_y| < 0.99 |n_z|), so they and any batch holding them take the direct kernel
    assert st1["tiles_table"] > 0 and st1["exact_fallbacks"] > 1000


def test_near_refusal_limit_and_refused():
    """Poses whose |t| / voxel approaches the certified-window limit (window 2^-17 .. 2^-16)
    stay bit-exact; beyond it the insert is refused with InvalidInput, never silently rounded."""
    v = 0.05
    far = 6.0e5  # mm: R / v ~ 3.4e7 voxels (|t| + |origin|), tie window 2^-16 (the largest allowed)
    poses = [(_rot((0.3, 1.0, 0.2), 4.0 * k - 6.0), (far + 1.0 + 0.37 * k, 2.0, far + 1.0 + 0.21 * k))
             for k in range(4)]
    wl = _workload("far", 64, 64, 0.02, 0.03, v, (64, 64, 64), (far, 0.0, far), poses)
    st, st1 = _check_vs_oracle(wl, what="near refusal")
    assert st["tiles_table"] > 0 and st1["tiles_table"] > 0
    grid = _grid(wl)
    bad = [(_rot((0, 0, 1), 1.0), (1.0e8, 0.0, 1.0e8))]
    wb = _workload("refused", 64, 64, 0.02, 0.03, v, (64, 64, 64), (0.0, 0.0, 0.0), bad)
    with pytest.raises(pkg.InvalidInput):
        grid.insert_frames(wb.frames_np(), wb.poses, wb.calib)
    grid.close()


def test_anisotropic_pixels_packed_count_guard():
    """sx = 0.03 voxel, sy = voxel / 128: one voxel collects up to ~34 pixels of a row and every
    row of a 128-row tile, more than the 4095 a packed shared-table slot holds.  The launch
    must pick a tile shape whose bound holds (or the direct kernel) and stay bit-exact."""
    v = 1.0
    poses = [(_rot((0.2, 0.1, 1.0), 2.0 * k), (8.0 + 0.3 * k, 3.0, 4.0 + 0.7 * k)) for k in range(5)]
    wl = _workload("aniso", 256, 256, 0.03 * v, v / 128.0, v, (32, 32, 16), (0.0, 0.0, 0.0), poses)
    frames = np.full((wl.nframes, wl.h, wl.w), 255, np.uint8)  # worst case for the 20-bit sum
    st, st1 = _check_vs_oracle(wl, frames, what="anisotropic")
    assert st["pixels_saturated"] == 0
    assert st["tiles_table"] > 0 and st1["tiles_table"] > 0  # a 64-row tile shape, not the direct kernel


def test_frame_step_padded_pitch_device_frame():
    """svr_frame_step with a column-sliced device tensor (row pitch > width) reconstructs the
    same volume as packed frames (the host staging branch used to memcpy a device
    address)."""
    import torch
    wl = synth.cfg1(nframes=6)
    frames = wl.frames_np()
    wide = torch.zeros((wl.nframes, wl.h, wl.w + 48), dtype=torch.uint8, device="cuda")
    wide[:, :, :wl.w] = torch.from_numpy(frames).cuda()
    rp = synth.render_params()
    a, b = _grid(wl), _grid(wl)
    for k in range(wl.nframes):
        a.frame_step(wide[k, :, :wl.w], wl.poses[k:k + 1], wl.calib, 1, rp)
        b.frame_step(frames[k], wl.poses[k:k + 1], wl.calib, 1, rp)
    a.sync()
    b.sync()
    sa, ca = a.accumulators()
    sb, cb = b.accumulators()
    assert np.array_equal(ca, cb) and np.array_equal(sa, sb)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    _assert_acc(a, ref, "pitched frame_step")


def test_cfg5_trilinear_gigabyte_slab_vs_oracle():
    """cfg5 (0.08 mm, 2000 x 1000 x 7500 grid) on a 64-plane z-slab (2000 x 1000 x 64 voxels,
    1.02 GB of f32 pairs) with every frame whose box meets it: weights and weighted sums within
    1e-5 relative of the oracle's fp64 sum of the same contributions (no absolute floor: both
    take u from the fp64 chain, only the GPU's fp32 accumulation order differs); then the
    depth-band render of the slab equals the oracle's render of the GPU's own f32 volume."""
    wl = synth.cfg5()
    z0 = 1200
    slab = (z0, z0 + 64)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    idx = sharding.route(boxes, slab)
    assert 50 < len(idx) < 400
    import torch
    dev = torch.empty((len(idx), wl.h, wl.w), dtype=torch.uint8, device="cuda")
    for i, k in enumerate(idx):
        synth.synth_frames_device(wl, dev[i:i + 1], int(k), 1)
    host = dev.cpu().numpy()
    poses = wl.poses[idx]
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0, z_range=slab, accum=wl.accum)
    grid.insert_frames(dev, poses, wl.calib)
    ws, wt = grid.trilinear()
    assert ws.nbytes + wt.nbytes >= 1.0e9
    ref = O.OracleGrid.for_workload(wl, z_range=slab)
    ref.insert_trilinear_f64(host, poses, wl.calib)
    assert (ref.weight64 > 0).sum() > 10_000_000
    np.testing.assert_allclose(wt, ref.weight64, rtol=1e-5, atol=0)
    np.testing.assert_allclose(ws, ref.wsum64, rtol=1e-5, atol=0)
    st = grid.stats()
    assert st["pixels_inserted"] + st["pixels_oob"] == len(idx) * wl.w * wl.h
    # render: the oracle renders the GPU's own f32 volume (same inputs -> same values)
    rp = synth.render_params(depth_lo_mm=15.0, depth_hi_mm=60.0)
    grid.render_coronal(None, rp, 0)
    mean, mx, dep = grid.read_coronal()
    ref.wsum[...] = ws
    ref.weight[...] = wt
    rmean, rmx, rdep = ref.render(rp, fill_radius=0)
    assert (dep >= 0).sum() > 10000
    assert np.array_equal(dep, rdep)
    np.testing.assert_allclose(mean, rmean, rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, rmx, rtol=1e-5, atol=0)
    grid.close()


def test_walk_variants_kz1_and_general_and_mixed():
    """K1 has two walks (svr_k1.cuh): kZ1 for frames with at most one y and one z carry per
    16-pixel chunk (z move as a predicated add, y / z ties captured at their carry) and the
    general one.  Frames rotated 40 degrees about z take the general walk (15 |Dc_y| > 1), small
    rotations the kZ1 walk, a mixed batch the general walk for all; every case stays bit-exact
    through the tile table, and the per-frame graph re-captures when a frame leaves its variant."""
    v = 0.5
    small = [(_rot((0.2, 0.1, 1.0), 3.0 * k - 6.0), (10.0 + 0.4 * k, 6.0, 8.0 + 0.45 * k)) for k in range(5)]
    big = [(_rot((0.05, 0.1, 1.0), 40.0 + 2.0 * k), (30.0 + 0.3 * k, 4.0, 9.0 + 0.5 * k)) for k in range(5)]
    def dcy_chunk(q):  # 15 |Dc_y| of a pose (identity calibration): the y fraction's chunk span
        w, x, y, z = q
        r10 = 2.0 * (x * y + w * z)  # R[1][0]: the image column direction's y component
        return 15.0 * abs(r10) * 0.1 / v
    assert all(dcy_chunk(q) < 1.0 for q, _ in small) and all(dcy_chunk(q) > 1.0 for q, _ in big)
    for name, poses in (("kz1", small), ("general", big), ("mixed", small[:3] + big[:3])):
        wl = _workload(name, 128, 256, 0.1, 0.1, v, (96, 96, 48), (0.0, 0.0, 0.0), poses)
        st, st1 = _check_vs_oracle(wl, what=name)
        assert st["tiles_table"] > 0 and st1["tiles_table"] > 0, name
    # the per-frame graph: kZ1 frames, then general ones (re-capture), then kZ1 again
    wl = _workload("alt", 128, 256, 0.1, 0.1, v, (96, 96, 48), (0.0, 0.0, 0.0), small[:2] + big[:2] + small[2:4])
    frames = wl.frames_np()
    grid = _grid(wl)
    rp = synth.render_params(depth_lo_mm=1.0, depth_hi_mm=12.0, band_above_mm=1.0, band_below_mm=0.5)
    for k in range(wl.nframes):
        grid.frame_step(frames[k], wl.poses[k:k + 1], wl.calib, 1, rp)
    grid.sync()
    ref = O.OracleGrid.for_workload(wl)
    for k in range(wl.nframes):
        ref.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
    _assert_acc(grid, ref, "alternating per-frame graph")
    assert grid.stats()["graph_captures"] >= 2
    grid.close()
