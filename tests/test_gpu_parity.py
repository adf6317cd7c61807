"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on seeded inputs.
Integer outputs (sum, count, dirty boxes, fill layer, depths, u8 projections) must be
bit-exact; rendered floats within 1e-5 relative (north_star), trilinear f32 within the
tolerance stated in test_trilinear_tolerance."""
import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import _abi, synth

pytestmark = pytest.mark.gpu


def _grid(wl, **kw):
    return pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0, accum=wl.accum, **kw)


def _assert_acc(grid, ref):
    s, c = grid.accumulators()
    bad = np.argwhere(c != ref.count)
    assert np.array_equal(c, ref.count), "count mismatch at %d voxels, first %s" % (len(bad), bad[:5])
    assert np.array_equal(s, ref.sum), "sum mismatch"


def test_cfg1_batch_bitexact():
    wl = synth.cfg1()
    frames = wl.frames_np()
    grid = _grid(wl)
    boxes, union = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = ref.insert_frames(frames, wl.poses, wl.calib)
    _assert_acc(grid, ref)
    assert [b.as_tuple() for b in boxes] == [b.as_tuple() for b in rboxes]
    st = grid.stats()
    assert st["pixels_inserted"] == ref.stats["inserted"]
    assert st["pixels_oob"] == ref.stats["oob"]
    assert st["frames_inserted"] == wl.nframes


def test_cfg1_fill_and_render_bitexact():
    wl = synth.cfg1()
    frames = wl.frames_np()
    grid = _grid(wl)
    _, union = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    region = pkg.dilate(union, 1)
    n_gpu = grid.fill_holes(region, 1, pkg.FILL_MEAN)
    n_ref = ref.fill_holes(region, 0, 1)
    assert n_gpu == n_ref
    assert np.array_equal(grid.fill_layer(), ref.fill)
    rp = synth.render_params()
    grid.render_coronal(None, rp, 1)
    mean, mx, dep = grid.read_coronal()
    rmean, rmx, rdep = ref.render(rp)
    assert np.array_equal(dep, rdep)
    np.testing.assert_allclose(mean, rmean, rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, rmx, rtol=1e-5, atol=0)
    assert np.array_equal(mean, rmean) and np.array_equal(mx, rmx)  # exact by construction


def test_single_frame_api_boxes():
    wl = synth.small_linear()
    frames = wl.frames_np()
    grid = _grid(wl)
    ref = O.OracleGrid.for_workload(wl)
    for k in range(wl.nframes):
        b = grid.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
        rb = ref.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
        assert b.as_tuple() == rb.as_tuple()
    _assert_acc(grid, ref)


@pytest.mark.parametrize("w,h", [(61, 47), (64, 48), (17, 5)])
@pytest.mark.parametrize("skip_zero", [False, True])
def test_ragged_and_skip_zero(w, h, skip_zero):
    wl = synth.small_linear(w=w, h=h, nframes=6)
    frames = wl.frames_np()
    frames[:, ::3, ::2] = 0  # zeros for skip_zero
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib, skip_zero=skip_zero)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib, skip_zero=skip_zero)
    _assert_acc(grid, ref)
    st = grid.stats()
    assert st["pixels_skipped_zero"] == ref.stats["skipped_zero"]
    assert st["pixels_oob"] == ref.stats["oob"]


def test_host_pinned_device_pitch_inputs():
    import torch
    wl = synth.small_linear(w=64, h=48, nframes=8)
    frames = wl.frames_np()
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    padded = np.zeros((wl.nframes, wl.h, 80), np.uint8)
    padded[:, :, :64] = frames
    for src in (frames, torch.from_numpy(frames).pin_memory(), torch.from_numpy(frames).cuda(),
                padded[:, :, :64]):
        grid = _grid(wl)
        grid.insert_frames(src, wl.poses, wl.calib)
        _assert_acc(grid, ref)
        grid.close()


def test_fan_bitexact():
    wl = synth.small_fan()
    frames = wl.frames_np()
    grid = _grid(wl)
    boxes, _ = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = ref.insert_frames(frames, wl.poses, wl.calib)
    _assert_acc(grid, ref)
    assert [b.as_tuple() for b in boxes] == [b.as_tuple() for b in rboxes]


@pytest.mark.parametrize("z_range", [None, (12, 30)])
def test_fan_tiles_bitexact(z_range):
    """k_fan_tiles (fan frames of whole 128-sample tiles): 40 scanlines (a short last tile of 8),
    dense table tiles near the apex and direct-run tiles far out, frames leaving the grid, and a
    slab whose faces cut the frames (face tiles: per-chunk classes and the exact pass)."""
    wl = synth.small_fan(nframes=12, lines=40, samples=256)
    frames = wl.frames_np()
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0, z_range=z_range)
    boxes, _ = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid(wl.dims, wl.voxel_mm, wl.origin, z_range=z_range)
    rboxes = ref.insert_frames(frames, wl.poses, wl.calib)
    _assert_acc(grid, ref)
    assert [b.as_tuple() for b in boxes] == [b.as_tuple() for b in rboxes]
    st = grid.stats()
    assert st["pixels_inserted"] == ref.stats["inserted"] and st["pixels_oob"] == ref.stats["oob"]
    assert st["tiles_table"] == wl.nframes * 2 * 2  # every tile through k_fan_tiles
    grid.close()


def test_cfg3_fan_subset_bitexact():
    wl = synth.cfg3()
    idx = np.arange(0, wl.nframes, 45)  # 40 frames spread over the sweep
    frames = synth.synth_frames_np(wl, 0, 1)  # generator check only
    frames = np.stack([wl.frames_np(int(k), 1)[0] for k in idx])
    poses = wl.poses[idx]
    grid = _grid(wl)
    grid.insert_frames(frames, poses, wl.calib)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames_mt(frames, poses, wl.calib)
    _assert_acc(grid, ref)


def test_cfg2_subset_bitexact():
    wl = synth.cfg2()
    idx = np.concatenate([np.arange(0, 40), np.arange(1200, 1240), np.arange(2360, 2400)])
    frames = np.stack([wl.frames_np(int(k), 1)[0] for k in idx])
    poses = wl.poses[idx]
    grid = _grid(wl)
    grid.insert_frames(frames, poses, wl.calib)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames_mt(frames, poses, wl.calib)
    _assert_acc(grid, ref)
    st = grid.stats()
    assert st["pixels_inserted"] + st["pixels_oob"] == len(idx) * wl.w * wl.h


def test_median_fill_r2_bitexact():
    wl = synth.small_linear(nframes=6)
    frames = wl.frames_np()
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    for mode, r in ((pkg.FILL_MEDIAN, 2), (pkg.FILL_MEDIAN, 1), (pkg.FILL_MEAN, 2), (pkg.FILL_MEDIAN, 3)):
        n = grid.fill_holes(None, r, mode)
        nr = ref.fill_holes(None, mode, r)
        assert n == nr, (mode, r)
        assert np.array_equal(grid.fill_layer(), ref.fill), (mode, r)


def test_incremental_equals_batch():
    wl = synth.cfg1(nframes=60)
    frames = wl.frames_np()
    rp = synth.render_params()
    inc = _grid(wl)
    pkg.run_incremental(frames, wl.poses, wl.calib, inc, 1, pkg.FILL_MEAN, render=rp)
    bat = _grid(wl)
    _, union = bat.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    bat.fill_holes(pkg.dilate(union, 1), 1, pkg.FILL_MEAN)
    bat.render_coronal(None, rp, 1)
    for a, b in zip(inc.accumulators(), bat.accumulators()):
        assert np.array_equal(a, b)
    assert np.array_equal(inc.fill_layer(), bat.fill_layer())
    for a, b in zip(inc.read_coronal(), bat.read_coronal()):
        assert np.array_equal(a, b)


def test_order_independence():
    """SPEC.md:327 / :645: any permutation of the inserts gives identical accumulators (100
    shuffles of a small scan, plus a cfg1 shuffle), one frame per call and in batches."""
    wl = synth.cfg1(nframes=50)
    frames = wl.frames_np()
    a = _grid(wl)
    a.insert_frames(frames, wl.poses, wl.calib)
    perm = np.random.default_rng(0).permutation(wl.nframes)
    b = _grid(wl)
    b.insert_frames(frames[perm], wl.poses[perm], wl.calib)
    for x, y in zip(a.accumulators(), b.accumulators()):
        assert np.array_equal(x, y)
    sl = synth.small_linear(nframes=12)
    fr = sl.frames_np()
    ref = _grid(sl)
    ref.insert_frames(fr, sl.poses, sl.calib)
    s0, c0 = ref.accumulators()
    rng = np.random.default_rng(1)
    g = _grid(sl)
    for shuffle in range(100):
        g.clear()
        p = rng.permutation(sl.nframes)
        if shuffle % 2:
            for k in p:
                g.insert_frames(fr[k], sl.poses[k:k + 1], sl.calib)
        else:
            g.insert_frames(fr[p], sl.poses[p], sl.calib)
        s1, c1 = g.accumulators()
        assert np.array_equal(c1, c0) and np.array_equal(s1, s0), shuffle


def test_spec_full_frame_rebinning_and_mean_bound():
    """one full 559 x 699 frame (0.1 mm/px) into 1 mm voxels -- counts and sums equal
    the brute-force re-binning (the oracle); every voxel value lies within the [min, max]
    of the pixel values inserted (frames drawn from [40, 90])."""
    rng = np.random.default_rng(7)
    calib = synth.linear_calib(559, 699, 0.1, 0.1)
    frames = rng.integers(40, 91, (3, 699, 559), dtype=np.uint8)
    poses = np.zeros(3, dtype=synth._abi.RIGID_DTYPE)
    for k in range(3):
        q = synth.quat_normalized(synth.quat_mul(synth.quat_axis_angle((1, 0, 0), 0.3 + 0.1 * k),
                                                 synth.quat_axis_angle((0, 0, 1), 0.05 * k)))
        poses[k] = (*q, 2.0 + k, 3.0, 20.0 + 0.7 * k)
    dims, vox, org = (64, 72, 64), 1.0, (0.0, 0.0, 0.0)
    g = pkg.VoxelGrid(dims, vox, org, device=0)
    g.insert_frames(frames, poses, calib)
    ref = O.OracleGrid(dims, vox, org)
    ref.insert_frames(frames, poses, calib)
    s, c = g.accumulators()
    assert np.array_equal(c, ref.count) and np.array_equal(s, ref.sum)
    assert int(c.sum()) == g.stats()["pixels_inserted"] > 0
    v = g.values()
    assert v[c > 0].min() >= 40 and v[c > 0].max() <= 90


def test_incremental_300_frames_throughput_floor():
    """SPEC.md:313 / :638-639: a 300-frame scan of 559 x 699 frames into a 1 mm grid of
    >= 500 x 100 x 70 mm, frame by frame (insert -> fill -> render as one graph replay each), equals
    the batch result, at far more than the 30 frames/s floor."""
    import time
    calib = synth.linear_calib(559, 699, 0.1, 0.1)
    rng = np.random.default_rng(8)
    n = 300
    frames = rng.integers(0, 256, (n, 699, 559), dtype=np.uint8)
    poses = np.zeros(n, dtype=synth._abi.RIGID_DTYPE)
    for k in range(n):
        q = synth.quat_normalized(synth.quat_axis_angle((1, 0, 0), np.radians(rng.uniform(-3, 3))))
        poses[k] = (*q, 10.0 + rng.uniform(-1, 1), 5.0, 10.0 + 1.6 * k)
    dims, vox, org = (500, 100, 520), 1.0, (0.0, 0.0, 0.0)
    rp = synth.render_params(depth_lo_mm=10.0, depth_hi_mm=60.0)
    inc = pkg.VoxelGrid(dims, vox, org, device=0)
    t0 = time.perf_counter()
    pkg.run_incremental(frames, poses, calib, inc, 1, pkg.FILL_MEAN, render=rp)
    fps = n / (time.perf_counter() - t0)
    bat = pkg.VoxelGrid(dims, vox, org, device=0)
    _, u = bat.insert_frames(frames, poses, calib, want_boxes=True)
    bat.fill_holes(pkg.dilate(u, 1), 1, pkg.FILL_MEAN)
    for a, b in zip(inc.accumulators(), bat.accumulators()):
        assert np.array_equal(a, b)
    assert np.array_equal(inc.fill_layer(), bat.fill_layer())
    assert fps >= 30.0, fps


def test_projection_u8():
    wl = synth.small_linear()
    frames = wl.frames_np()
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib)
    grid.fill_holes(None, 1, pkg.FILL_MEAN)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    ref.fill_holes(None, 0, 1)
    for mode in (pkg.PROJ_MAX, pkg.PROJ_MEAN):
        for axis in (0, 1, 2):
            for uf in (False, True):
                assert np.array_equal(grid.coronal_projection(mode, axis, uf),
                                      ref.coronal_projection(mode, axis, uf)), (mode, axis, uf)
    assert np.array_equal(grid.values(), ref.values())
    assert np.array_equal(grid.values(apply_fills=True), ref.values(True))


def test_trilinear_tolerance():
    """Trilinear splat (cfg5 geometry, small grid): the GPU takes u from the exact fp64 chain and
    forms the oracle's fp32 contributions, so it differs from their fp64 sum only by its fp32
    accumulation: |d| <= N 2^-24 |ref| for N contributions (N < 40 here): rtol 1e-5, no floor."""
    import dataclasses
    wl = dataclasses.replace(synth.cfg5(nframes=6, dims=(160, 120, 40)), origin=(70.0, 20.0, 9.5))
    frames = wl.frames_np()
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_trilinear_f64(frames, wl.poses, wl.calib)
    ws, wt = grid.trilinear()
    assert (wt > 0).sum() > 10000
    np.testing.assert_allclose(wt, ref.weight64, rtol=1e-5, atol=0)
    np.testing.assert_allclose(ws, ref.wsum64, rtol=1e-5, atol=0)

def test_frame_step_graph_on_trilinear_volume():
    """svr_frame_step on a trilinear volume (cfg5 geometry): one CUDA-graph replay per frame =
    splat + depth / band render of the frame's columns (box + 1: the 2x2x2 splat reaches one voxel
    past the nearest-voxel box).  The volume equals a batch insert's within the fp32 accumulation
    order (1e-5 relative, no floor) and the incrementally rendered image equals the oracle's
    whole-volume render of the GPU's own final volume: every column a frame changes lies inside
    the region that frame re-renders."""
    import dataclasses
    wl = dataclasses.replace(synth.cfg5(nframes=8, dims=(160, 120, 40)), origin=(70.0, 20.0, 9.5))
    frames = wl.frames_np()
    rp = synth.render_params(depth_lo_mm=1.0, depth_hi_mm=8.0, band_above_mm=0.6, band_below_mm=0.3)
    inc = _grid(wl)
    for k in range(wl.nframes):
        inc.frame_step(frames[k], wl.poses[k:k + 1], wl.calib, 1, rp)
    inc.sync()
    assert inc.stats()["graph_captures"] >= 1
    ws, wt = inc.trilinear()
    batch = _grid(wl)
    batch.insert_frames(frames, wl.poses, wl.calib)
    ws2, wt2 = batch.trilinear()
    assert (wt > 0).sum() > 10000
    np.testing.assert_allclose(wt, wt2, rtol=1e-5, atol=0)
    np.testing.assert_allclose(ws, ws2, rtol=1e-5, atol=0)
    mean, mx, dep = inc.read_coronal()
    ref = O.OracleGrid.for_workload(wl)
    ref.wsum[...] = ws
    ref.weight[...] = wt
    rmean, rmx, rdep = ref.render(rp, fill_radius=0)
    assert (rdep >= 0).sum() > 500
    assert np.array_equal(dep, rdep)
    np.testing.assert_allclose(mean, rmean, rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, rmx, rtol=1e-5, atol=0)
    inc.close()
    batch.close()


@pytest.mark.parametrize("want_boxes", [False, True])
@pytest.mark.parametrize("slab", [None, (60, 90)])
def test_skip_zero_through_tile_kernel(want_boxes, slab):
    """skip_zero on the K1 tile kernel (k_pnn_tiles<kSkip>): cfg2 geometry, frames cut to a band of
    rows (whole chunks, warps and tiles of zeros), zeros sprinkled inside the band (mixed chunks:
    walked with per-pixel counts in a batch insert, sent to the exact pass with their mask when
    boxes are wanted or the tile meets a slab face) and a zero run crossing chunk borders.
    Accumulators, per-frame boxes and the inserted / out-of-bounds / skipped counters equal the
    oracle's, on the whole grid and on a z-slab whose faces cut the frames."""
    wl = synth.cfg2(nframes=24)
    frames = wl.frames_np().copy()
    frames[:, :150, :] = 0
    frames[:, 300:, :] = 0
    rng = np.random.default_rng(5)
    frames[rng.random(frames.shape) < 0.004] = 0
    frames[:, 200, 37:90] = 0
    frames[3] = 0  # a frame with nothing to insert
    kw = {} if slab is None else {"z_range": slab}
    grid = _grid(wl, **kw)
    ref = O.OracleGrid.for_workload(wl, z_range=slab)
    rboxes = ref.insert_frames(frames, wl.poses, wl.calib, skip_zero=True)
    if want_boxes:
        boxes, _ = grid.insert_frames(frames, wl.poses, wl.calib, skip_zero=True, want_boxes=True)
        assert [b.as_tuple() for b in boxes] == [b.as_tuple() for b in rboxes]
    else:
        grid.insert_frames(frames, wl.poses, wl.calib, skip_zero=True)
    _assert_acc(grid, ref)
    st = grid.stats()
    assert st["tiles_table"] > 0, "the insert did not go through k_pnn_tiles"
    assert st["pixels_skipped_zero"] == int((frames == 0).sum()) == ref.stats["skipped_zero"]
    assert st["pixels_inserted"] == ref.stats["inserted"]
    assert st["pixels_oob"] == ref.stats["oob"]
    grid.close()


@pytest.mark.parametrize("kernel", ["warp", "chunk"])
@pytest.mark.parametrize("case", ["ragged_linear", "skip_zero", "fan"])
def test_trilinear_splat_kernels_edge_cases(case, kernel, monkeypatch):
    """Both trilinear splats (k_tri_warp: lane = pixel with the x + 1 corners handed to the next
    lane; SVR_TRI_KERNEL=chunk: k_insert, a 16-pixel chunk per thread) against the oracle's fp64 sum
    of the same contributions at 1e-5 relative, no absolute floor: a row length that is not a
    multiple of 32 (idle lanes in the last segment), pixels clipped at every grid face, skip_zero
    (holes break the hand-over chain) and a convex fan (neighbouring lanes rarely on neighbouring
    voxels: no hand-over); pixel counters equal the oracle's."""
    import dataclasses
    if kernel == "chunk":
        monkeypatch.setenv("SVR_TRI_KERNEL", "chunk")
    else:
        monkeypatch.delenv("SVR_TRI_KERNEL", raising=False)
    if case == "fan":
        wl = dataclasses.replace(synth.small_fan(), accum=_abi.ACC_TRILINEAR)
    else:
        wl = dataclasses.replace(synth.small_linear(w=70, h=45, nframes=8), accum=_abi.ACC_TRILINEAR)
    frames = wl.frames_np().copy()
    skip = case == "skip_zero"
    if skip:
        frames[:, ::3, 5:40:2] = 0
        frames[:, 7, :] = 0
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib, skip_zero=skip)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_trilinear_f64(frames, wl.poses, wl.calib, skip_zero=skip)
    ws, wt = grid.trilinear()
    assert (wt > 0).sum() > 2000
    np.testing.assert_allclose(wt, ref.weight64, rtol=1e-5, atol=0)
    np.testing.assert_allclose(ws, ref.wsum64, rtol=1e-5, atol=0)
    st = grid.stats()
    assert st["pixels_inserted"] + st["pixels_oob"] + st["pixels_skipped_zero"] == frames.size
    if skip:
        assert st["pixels_skipped_zero"] == int((frames == 0).sum())
    grid.close()


def test_footprint_counts():
    wl = synth.small_linear(nframes=5)
    frames = wl.frames_np()
    grid = _grid(wl)
    u = grid.footprint(frames, wl.poses, wl.calib)
    for k in range(wl.nframes):
        r = O.OracleGrid.for_workload(wl)
        r.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
        assert u[k] == int((r.count > 0).sum())


INSERT_KERNELS = ["auto", "direct"]


def _select_kernel(monkeypatch, kernel):
    """auto: the launch's own choice (k_pnn_tiles for linear probes whose tiles fit, k_pnn_plane
    for fans, k_insert otherwise); direct: SVR_INSERT_KERNEL=direct forces the k_insert fallback."""
    if kernel == "direct":
        monkeypatch.setenv("SVR_INSERT_KERNEL", "direct")
    else:
        monkeypatch.delenv("SVR_INSERT_KERNEL", raising=False)


@pytest.mark.parametrize("name", ["small_linear", "small_fan"])
@pytest.mark.parametrize("kernel", INSERT_KERNELS)
def test_golden_fixtures_gpu(name, kernel, monkeypatch):
    """CUDA path against the committed fixtures (accumulators from the reference's own
    pixel_to_world, tests/golden/make_golden.py) for every insert kernel variant."""
    from golden_util import Fixture
    _select_kernel(monkeypatch, kernel)
    fx = Fixture(name)
    grid = pkg.VoxelGrid(fx.dims, fx.voxel_mm, fx.origin, device=0)
    boxes, _ = grid.insert_frames(fx.frames, fx.poses, fx.calib, want_boxes=True)
    s, c = grid.accumulators()
    assert np.array_equal(s, fx["sum"]) and np.array_equal(c, fx["count"])
    assert np.array_equal(np.array([b.as_tuple() for b in boxes]), fx["boxes"])
    assert grid.fill_holes(None, 1, pkg.FILL_MEAN) == int(fx["filled_mean_r1"])
    assert np.array_equal(grid.fill_layer(), fx["fill_mean_r1"])
    grid.render_coronal(None, fx.render, 1)
    mean, mx, dep = grid.read_coronal()
    assert np.array_equal(dep, fx["render_depth"])
    np.testing.assert_allclose(mean, fx["render_mean"], rtol=1e-5, atol=0)
    np.testing.assert_allclose(mx, fx["render_max"], rtol=1e-5, atol=0)
    grid.fill_holes(None, 2, pkg.FILL_MEDIAN)
    assert np.array_equal(grid.fill_layer(), fx["fill_median_r2"])
    g0 = pkg.VoxelGrid(fx.dims, fx.voxel_mm, fx.origin, device=0)
    g0.insert_frames(fx.frames, fx.poses, fx.calib, skip_zero=True)
    s0, c0 = g0.accumulators()
    assert np.array_equal(s0, fx["sum_skip0"]) and np.array_equal(c0, fx["count_skip0"])


@pytest.mark.parametrize("kernel", INSERT_KERNELS)
def test_cfg1_all_kernels(kernel, monkeypatch):
    _select_kernel(monkeypatch, kernel)
    wl = synth.cfg1()
    frames = wl.frames_np()
    grid = _grid(wl)
    boxes, _ = grid.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    ref = O.OracleGrid.for_workload(wl)
    rboxes = ref.insert_frames(frames, wl.poses, wl.calib)
    _assert_acc(grid, ref)
    assert [b.as_tuple() for b in boxes] == [b.as_tuple() for b in rboxes]


@pytest.mark.parametrize("radius", [1, 2])
def test_mean_fill_bitexact(radius):
    """Mean fill (r = 1: k_fill_warp; r = 2: k_fill_generic) against the oracle on regions with
    grid-edge clipping."""
    wl = synth.cfg1(nframes=80)
    frames = wl.frames_np()
    grid = _grid(wl)
    grid.insert_frames(frames, wl.poses, wl.calib)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    for region in (None, (3, 0, 20, 200, 127, 70), (0, 5, 0, 127, 60, 255)):
        n = grid.fill_holes(region, radius, pkg.FILL_MEAN)
        nr = ref.fill_holes(region, 0, radius)
        assert n == nr, region
        assert np.array_equal(grid.fill_layer(), ref.fill), region


def test_fill_large_accumulators():
    """Voxel values from counts up to the u16 maximum and sums past 2^23 (outside the fp32
    estimate's exact range: the fill kernels' recompute path) feed the neighbours' mean fills
    exactly as in the oracle."""
    dims = (70, 40, 50)
    rng = np.random.default_rng(21)
    shp = (dims[2], dims[1], dims[0])
    count = np.where(rng.random(shp) < 0.4, rng.integers(1, 65536, shp), 0).astype(np.uint16)
    big = rng.random(shp) < 0.5
    mean = np.where(big, rng.integers(128, 256, shp), rng.integers(0, 256, shp))
    sum_ = (count.astype(np.uint64) * mean + rng.integers(0, 2, shp) * (count > 1)).astype(np.uint32)
    assert (sum_ >= (1 << 23)).any()
    grid = pkg.VoxelGrid(dims, 1.0, (0, 0, 0), device=0)
    grid.set_accumulators(sum_, count)
    ref = O.OracleGrid(dims, 1.0)
    ref.sum[...] = sum_
    ref.count[...] = count
    for region in (None, (5, 3, 2, 60, 30, 45)):
        assert grid.fill_holes(region, 1, pkg.FILL_MEAN) == ref.fill_holes(region, 0, 1)
        assert np.array_equal(grid.fill_layer(), ref.fill), region
    assert np.array_equal(grid.values(apply_fills=True), ref.values(apply_fills=True))


def test_chunked_dirty_regions_equal_bounding_box():
    """Batch fill/render over per-z-chunk dirty boxes (svr_fill_holes_boxes,
    svr_render_coronal_boxes) equals the same over one bounding box, bit for bit."""
    from paper_2412_00058_b200 import sharding
    wl = synth.cfg2(nframes=240)
    idx = np.arange(0, 240, 1)
    frames = np.stack([wl.frames_np(int(k), 1)[0] for k in idx[:120]])
    poses = wl.poses[:120]
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, poses)
    alloc = (0, wl.dims[2])
    u = sharding.union_box(boxes, np.arange(len(boxes)), alloc)
    rp = synth.render_params()
    a = _grid(wl)
    a.insert_frames(frames, poses, wl.calib)
    na = a.fill_holes(pkg.dilate(u, 1), 1, pkg.FILL_MEAN)
    a.render_coronal(u, rp, 1)
    b = _grid(wl)
    b.insert_frames(frames, poses, wl.calib)
    fb = sharding.chunk_boxes(boxes, np.arange(len(boxes)), alloc, chunk=32, dilate=1)
    nb = b.fill_holes_boxes(fb, 1, pkg.FILL_MEAN)
    b.render_coronal_boxes(sharding.chunk_boxes(boxes, np.arange(len(boxes)), alloc, chunk=32), rp, 1)
    box = (u.x0 - 1, max(u.y0 - 1, 0), max(u.z0 - 1, 0), u.x1 + 1, min(u.y1 + 1, wl.dims[1] - 1), u.z1 + 1)
    assert np.array_equal(a.fill_layer(box), b.fill_layer(box))
    assert na == nb
    for x, y in zip(a.read_coronal(), b.read_coronal()):
        assert np.array_equal(x, y)


def test_cfg2_full_size_properties(monkeypatch):
    """BASELINE cfg2 at full size through size-independent properties (the bit-exact oracle
    comparison is tests/test_gpu_fullsize.py): every pixel lands (no OOB) and the accumulators
    conserve the pixel count and sum exactly; the reversed frame order through the direct fallback
    kernel gives identical accumulators (order independence)."""
    import torch
    wl = synth.cfg2()
    frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
    synth.synth_frames_device(wl, frames, 0, wl.nframes)
    total = int(frames.sum(dtype=torch.int64).item())
    a = _grid(wl)
    a.insert_frames(frames, wl.poses, wl.calib)
    st = a.stats()
    assert st["pixels_oob"] == 0 and st["pixels_saturated"] == 0
    assert st["pixels_inserted"] == wl.nframes * wl.w * wl.h
    s, c = a.accumulators()
    assert int(c.sum(dtype=np.int64)) == st["pixels_inserted"]
    assert int(s.sum(dtype=np.int64)) == total
    monkeypatch.setenv("SVR_INSERT_KERNEL", "direct")
    b = _grid(wl)
    rev = torch.flip(frames, dims=[0]).contiguous()
    b.insert_frames(rev, wl.poses[::-1].copy(), wl.calib)
    s2, c2 = b.accumulators()
    assert np.array_equal(c, c2) and np.array_equal(s, s2)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_sharded_bench_step_equals_unsharded(world):
    """bench.py's per-rank step on the GPU (z-slab grids with ghosts, routed frames, per-chunk
    dirty boxes, fill + render), ranks run one after another in this process: the owned planes'
    accumulators and the owned coronal rows equal the unsharded run bit for bit."""
    from paper_2412_00058_b200 import sharding
    wl = synth.cfg2(nframes=300)
    frames = np.stack([wl.frames_np(k, 1)[0] for k in range(0, 300, 1)])
    rp = synth.render_params()
    fill_r = wl.fill_radius

    def run(z_range, idx):
        boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
        g = _grid(wl, z_range=z_range)
        g.insert_frames(frames[idx], wl.poses[idx], wl.calib)
        g.fill_holes_boxes(sharding.chunk_boxes(boxes, idx, z_range, chunk=32, dilate=fill_r), fill_r,
                           pkg.FILL_MEAN, count=False)
        g.render_coronal_boxes(sharding.chunk_boxes(boxes, idx, z_range, chunk=32), rp, fill_r)
        return g

    full = run((0, wl.dims[2]), np.arange(300))
    s_full, c_full = full.accumulators()
    mean_f, max_f, dep_f = full.read_coronal()
    slabs = sharding.plan_slabs(wl.dims[2], world, fill_r + rp.median_radius)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    # fused render + gather: each "rank" stores its owned rows into every rank's full image
    # (here ordinary device buffers stand in for the ranks' symmetric-memory peers)
    import torch
    images = [torch.zeros((2, wl.dims[2], wl.dims[0]), dtype=torch.float32, device="cuda")
              for _ in range(world)]

    def run(z_range, idx, own=None):
        boxes_ = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
        g = _grid(wl, z_range=z_range)
        if own is not None:
            g.set_gather_targets(images, own)
        g.insert_frames(frames[idx], wl.poses[idx], wl.calib)
        g.fill_holes_boxes(sharding.chunk_boxes(boxes_, idx, z_range, chunk=32, dilate=fill_r), fill_r,
                           pkg.FILL_MEAN, count=False)
        g.render_coronal_boxes(sharding.chunk_boxes(boxes_, idx, z_range, chunk=32), rp, fill_r)
        return g

    for sl in slabs:
        idx = sharding.route(boxes, sl.alloc)
        g = run(sl.alloc, idx, own=sl.owned)
        o0, o1 = sl.owned
        s, c = g.accumulators((0, 0, o0, wl.dims[0] - 1, wl.dims[1] - 1, o1 - 1))
        assert np.array_equal(c, c_full[o0:o1]) and np.array_equal(s, s_full[o0:o1])
        m, x, d = g.read_coronal(o0, o1 - 1)
        assert np.array_equal(m, mean_f[o0:o1]) and np.array_equal(x, max_f[o0:o1])
        assert np.array_equal(d, dep_f[o0:o1])
        del g
    torch.cuda.synchronize()
    for img in images:
        assert np.array_equal(img[0].cpu().numpy(), mean_f) and np.array_equal(img[1].cpu().numpy(), max_f)


@pytest.mark.parametrize("source", ["host", "device", "pinned"])
def test_frame_step_graph_equals_per_call_pipeline(source):
    """svr_frame_step (one CUDA-graph replay per frame) against the per-call pipeline
    insert -> fill(box (+) 1) -> render(box): accumulators, fill layer and coronal images equal,
    including frames whose box is clipped by the grid and one wholly outside it."""
    import torch
    wl = synth.cfg1(nframes=40)
    frames = wl.frames_np()
    poses = wl.poses.copy()
    poses[5]["tx"] += 1000.0  # outside the grid: the early plain-insert path
    rp = synth.render_params(depth_lo_mm=5.0, depth_hi_mm=40.0)
    a, b = _grid(wl), _grid(wl)
    dev = torch.from_numpy(frames).cuda()
    pin = torch.from_numpy(frames).pin_memory()
    for k in range(wl.nframes):
        src = {"host": frames[k], "device": dev[k], "pinned": pin[k]}[source]
        box = a.frame_step(src, poses[k:k + 1], wl.calib, 1, rp)
        b.insert_frames(frames[k], poses[k:k + 1], wl.calib)
        if not box.empty():
            b.fill_holes(pkg.dilate(box, 1), 1, pkg.FILL_MEAN, count=False)
            b.render_coronal(box, rp, 1)
    a.sync()
    sa, ca = a.accumulators()
    sb, cb = b.accumulators()
    assert np.array_equal(ca, cb) and np.array_equal(sa, sb)
    assert np.array_equal(a.fill_layer(), b.fill_layer())
    for x, y in zip(a.read_coronal(), b.read_coronal()):
        assert np.array_equal(x, y)
    assert a.stats()["frames_inserted"] == wl.nframes


def test_edge_cases():
    """Empty and degenerate inputs: zero frames, a frame wholly outside the grid (all pixels
    counted OOB, empty dirty box), an empty fill region, a render over an empty box, a pitched
    host frame through the frame graph, and readouts of a z-slab volume."""
    import torch
    wl = synth.small_linear(nframes=6)
    frames = wl.frames_np()
    g = _grid(wl)
    g.insert_frames(frames[:0], wl.poses[:0], wl.calib)  # no-op
    assert g.stats()["frames_inserted"] == 0
    far = wl.poses[:1].copy()
    far["tz"] += 1e4
    boxes, u = g.insert_frames(frames[:1], far, wl.calib, want_boxes=True)
    st = g.stats()
    assert u.empty() and boxes[0].empty()
    assert st["pixels_oob"] == wl.w * wl.h and st["pixels_inserted"] == 0
    assert g.fill_holes((5, 5, 5, 4, 4, 4), 1, pkg.FILL_MEAN) == 0
    g.render_coronal((1, 1, 1, 0, 0, 0), synth.render_params(), 1)
    # pitched host frame (row pitch 80 > width 64) through svr_frame_step == per-call pipeline
    pitched = np.zeros((wl.h, 80), np.uint8)
    pitched[:, :wl.w] = frames[2]
    rp = synth.render_params(depth_lo_mm=1.0, depth_hi_mm=12.0)
    a, b = _grid(wl), _grid(wl)
    box = a.frame_step(pitched[:, :wl.w], wl.poses[2:3], wl.calib, 1, rp)
    b.insert_frames(frames[2], wl.poses[2:3], wl.calib)
    b.fill_holes(pkg.dilate(box, 1), 1, pkg.FILL_MEAN)
    b.render_coronal(box, rp, 1)
    a.sync()
    for x, y in zip(a.accumulators(), b.accumulators()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.fill_layer(), b.fill_layer())
    # a z-slab volume reads back exactly its planes
    full = _grid(wl)
    full.insert_frames(frames, wl.poses, wl.calib)
    slab = _grid(wl, z_range=(10, 30))
    slab.insert_frames(frames, wl.poses, wl.calib)
    s_full, c_full = full.accumulators()
    s_sl, c_sl = slab.accumulators()
    assert np.array_equal(c_sl, c_full[10:30]) and np.array_equal(s_sl, s_full[10:30])
    assert np.array_equal(slab.values(), full.values()[10:30])


def test_count_cap_flagged_at_readout():
    """SPEC.md:336 caps: past 65534 pixels in one voxel the oracle drops pixels one by one; the
    device keeps counting (order-independent atomics) and the readout clamps the count to the
    u16 maximum and reports the voxel as saturated (DESIGN.md §3 caps row)."""
    from paper_2412_00058_b200 import _abi
    calib = synth.linear_calib(16, 16, 0.1, 0.1)
    frames = np.full((300, 16, 16), 200, np.uint8)  # 300 x 256 px, all into voxel (1, 1, 1)
    poses = np.zeros(300, dtype=_abi.RIGID_DTYPE)
    poses["qw"] = 1.0
    poses["tx"] = poses["ty"] = poses["tz"] = 12.0
    g = pkg.VoxelGrid((3, 3, 3), 10.0, (0.0, 0.0, 0.0), device=0)
    g.insert_frames(frames, poses, calib)
    s, c = g.accumulators()
    assert c[1, 1, 1] == 65535 and g.stats()["pixels_saturated"] >= 1
    assert int(c.sum()) == 65535 and g.values()[1, 1, 1] == 200
    ref = O.OracleGrid((3, 3, 3), 10.0)
    ref.insert_frames(frames, poses, calib)
    assert ref.count[1, 1, 1] == 65534 and ref.stats["saturated"] == 300 * 256 - 65534


def test_value_rounding_selftest():
    """Device acc_value (round(sum / count) via an approximate divide + 1/2 offset) equals
    integer division for every count in [1, 255] and every reachable sum."""
    import ctypes as C
    from paper_2412_00058_b200 import _abi
    bad = C.c_int64(-1)
    _abi.check(_abi.lib().svr_selftest_value_rounding(0, C.byref(bad)))
    assert bad.value == 0


def test_checkpoint_resume(tmp_path):
    """Accumulator checkpoint / resume: save mid-scan, restore into a fresh grid,
    insert the rest -> identical to the uninterrupted scan."""
    wl = synth.cfg1(nframes=40)
    frames = wl.frames_np()
    full = _grid(wl)
    full.insert_frames(frames, wl.poses, wl.calib)
    a = _grid(wl)
    a.insert_frames(frames[:17], wl.poses[:17], wl.calib)
    a.save(tmp_path / "ck.npz")
    b = _grid(wl)
    b.fill_holes(None, 1, pkg.FILL_MEAN)
    assert b.load(tmp_path / "ck.npz") == 17  # frames_inserted of the checkpoint
    assert not b.fill_layer().any()  # the derived fill layer is cleared on restore
    b.insert_frames(frames[17:], wl.poses[17:], wl.calib)
    for x, y in zip(b.accumulators(), full.accumulators()):
        assert np.array_equal(x, y)
    other = pkg.VoxelGrid((8, 8, 8), 1.0, (0, 0, 0), device=0)
    with pytest.raises(pkg.InvalidInput):
        other.load(tmp_path / "ck.npz")
    shifted = pkg.VoxelGrid(wl.dims, wl.voxel_mm, (wl.origin[0] + 1.0, wl.origin[1], wl.origin[2]), device=0)
    with pytest.raises(pkg.InvalidInput):  # same dims, different origin: refused
        shifted.load(tmp_path / "ck.npz")


@pytest.mark.parametrize("groups", [3, 8])
def test_reconstruct_sweep_equals_sequential(groups):
    """sharding.reconstruct_sweep (fill / render of finished z-chunks on a second stream while
    later frames are inserted) leaves the accumulators, the fill layer and the coronal images bit
    for bit as insert-all, fill-all, render-all does."""
    import torch
    from paper_2412_00058_b200 import sharding
    wl = synth.cfg2(nframes=600)
    frames = torch.empty((600, wl.h, wl.w), dtype=torch.uint8, device="cuda")
    synth.synth_frames_device(wl, frames, 0, 600, 0)
    rp = synth.render_params()
    fill_r = wl.fill_radius
    alloc = (0, wl.dims[2])
    idx = np.arange(600)
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    fb = sharding.chunk_boxes(boxes, idx, alloc, chunk=32, dilate=fill_r)
    rb = sharding.chunk_boxes(boxes, idx, alloc, chunk=32)

    seq = _grid(wl)
    seq.insert_frames(frames, wl.poses[:600], wl.calib)
    seq.fill_holes_boxes(fb, fill_r, pkg.FILL_MEAN, count=False)
    seq.render_coronal_boxes(rb, rp, fill_r)
    seq.sync()

    sched = sharding.sweep_schedule(boxes, idx, fb, rb, groups=groups)
    assert sum(len(s[2]) for s in sched) == len(fb) and sum(len(s[3]) for s in sched) == len(rb)
    assert sum(len(s[3]) for s in sched[:-1]) > 0, "nothing overlapped"
    pip = _grid(wl)
    s_ins = torch.cuda.Stream()
    with torch.cuda.stream(s_ins):
        sharding.reconstruct_sweep(pip, frames, wl.poses[:600], wl.calib, sched, rp, fill_r,
                                   insert_stream=s_ins)
    s_ins.synchronize()
    pip.sync()
    for a, b in zip(seq.accumulators(), pip.accumulators()):
        assert np.array_equal(a, b)
    assert np.array_equal(seq.fill_layer(), pip.fill_layer())
    for a, b in zip(seq.read_coronal(), pip.read_coronal()):
        assert np.array_equal(a, b)
