"""GPU: the ingest front-end and the SPEC output formats through the C-ABI against the CPU
oracle — a ScanBundle reconstructed incrementally (native decode + crop, pose matching, batched
insert, per-batch fill of the dirty region) equals the oracle batch result bit-for-bit, and the
volume file / x-slice exports reproduce the value array."""
import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import _abi, ingest, synth

pytestmark = pytest.mark.gpu


def _bundle(tmp_path, wl, latency=8.0, raw_pad=(9, 6)):
    c = wl.calib
    c.crop_x, c.crop_y = 5, 3
    c.latency_ms = latency
    frames = wl.frames_np()
    ft = 30.0 * np.arange(wl.nframes) + 100.0
    # poses 3x the frame rate; the first frame's shifted time precedes the stream (unposed)
    pt = np.linspace(ft[1] - latency, ft[-1] - latency, 3 * wl.nframes)
    pa = np.zeros(len(pt), dtype=_abi.RIGID_DTYPE)
    for i in range(len(pt)):
        pa[i] = wl.poses[min(i // 3 + 1, wl.nframes - 1)]
    raw = (c.crop_w + c.crop_x + raw_pad[0], c.crop_h + c.crop_y + raw_pad[1])
    ingest.write_bundle(tmp_path / "bundle", frames, ft, pt, pa, c, raw=raw)
    return ingest.read_bundle(tmp_path / "bundle"), frames


@pytest.mark.parametrize("maker,batch", [(synth.small_linear, 5), (synth.small_fan, 3)])
def test_ingest_bundle_equals_oracle(tmp_path, maker, batch):
    wl = maker()
    b, frames = _bundle(tmp_path, wl)
    poses, valid = b.match_poses()
    assert not valid[0] and valid[1:].all()
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    st = ingest.ingest(b, grid, batch=batch, threads=2, fill_radius=1)
    assert st.frames == wl.nframes - 1 and st.frames_unposed == 1
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames[valid], poses[valid], b.calib)
    s, c = grid.accumulators()
    assert np.array_equal(c, ref.count) and np.array_equal(s, ref.sum)
    # every voxel whose neighbourhood changed was refilled by some batch: equals a full fill
    ref.fill_holes(None, pkg.FILL_MEAN, 1)
    assert np.array_equal(grid.fill_layer(), ref.fill)
    d = st.as_dict()
    assert d["frames"] == st.frames and d["fps"] > 0 and d["schema_version"] == 1


@pytest.mark.parametrize("mode,radius", [(pkg.FILL_MEAN, 1), (pkg.FILL_MEDIAN, 2)])
def test_volume_file_and_slices_roundtrip(tmp_path, mode, radius):
    wl = synth.small_linear()
    frames = wl.frames_np()
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    grid.insert_frames(frames, wl.poses, wl.calib)
    grid.fill_holes(None, radius, mode)
    ref = O.OracleGrid.for_workload(wl)
    ref.insert_frames(frames, wl.poses, wl.calib)
    ref.fill_holes(None, mode, radius)
    for fills in (False, True):
        vals = grid.values(apply_fills=fills)
        assert np.array_equal(vals, ref.values(apply_fills=fills))
        meta = ingest.write_volume(grid, tmp_path / f"v{int(fills)}.raw", apply_fills=fills)
        assert meta["dims"] == list(wl.dims) and meta["frames_inserted"] == wl.nframes
        back, meta2 = ingest.read_volume(tmp_path / f"v{int(fills)}.raw")
        assert np.array_equal(back, vals) and meta2["fills_applied"] == fills
        n = ingest.export_slices(grid, tmp_path / f"s{int(fills)}", apply_fills=fills)
        assert n == wl.dims[0]
        sl, _ = ingest.import_slices(tmp_path / f"s{int(fills)}")
        assert np.array_equal(sl, vals)
    if mode == pkg.FILL_MEDIAN:
        # filled voxels carry the median itself (not median / n)
        filled = (ref.count == 0) & ((ref.fill >> 16) > 0)
        assert filled.any()
        assert np.array_equal(grid.values(apply_fills=True)[filled], (ref.fill[filled] & 0xFFFF).astype(np.uint8))
    proj = grid.coronal_projection(pkg.PROJ_MAX, depth_axis=1, use_fills=True)
    assert np.array_equal(proj, ref.coronal_projection(pkg.PROJ_MAX, 1, use_fills=True))


def test_export_slices_spec_example(tmp_path):
    """dims (10,20,30) -> 10 files of 20x30; a single bright voxel at (3,5,7)
    is the only bright pixel of file 0003, at (5,7)."""
    grid = pkg.VoxelGrid((10, 20, 30), 1.0, (0.0, 0.0, 0.0), device=0)
    c = synth.linear_calib(1, 1, 1.0, 1.0)
    grid.insert_frame(np.full((1, 1), 200, np.uint8), synth.rigid(t=(3.0, 5.0, 7.0)), c)
    assert ingest.export_slices(grid, tmp_path / "s") == 10
    for x in range(10):
        img = ingest.read_pgm(tmp_path / "s" / f"{x:04d}.pgm")
        assert img.shape == (30, 20)
        if x == 3:
            assert img[7, 5] == 200 and np.count_nonzero(img) == 1
        else:
            assert not img.any()
