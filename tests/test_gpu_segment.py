"""GPU: the segmentation front-end kernels (svr_segment.cu) through the C-ABI against the CPU
oracle's pins (bone contour rows per column and per frame, brightness threshold, apply_cut), and
the segmented insert path end to end (Algorithm 1 / Algorithm 2 cut frames -> skip_zero insert)
bit-exact against the oracle; SPEC segment / project examples as properties."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import segment as S
from paper_2412_00058_b200 import synth
from seg_util import phantom_frame, speckle_frame
from test_segment_cpu import orc_contour

pytestmark = pytest.mark.gpu


def _stack(rng, n, **kw):
    imgs, truth = [], []
    for k in range(n):
        if k % 5 == 4:
            imgs.append(speckle_frame(rng))
            truth.append(np.nan)
        else:
            d = 32.0 + 6.0 * k / n
            img, t = phantom_frame(rng, bone_mm=d, tilt_deg=rng.uniform(-10, 10), **kw)
            imgs.append(img)
            truth.append(float(np.median(t)))
    return np.stack(imgs), np.array(truth)


def test_bone_contour_gpu_equals_oracle():
    rng = np.random.default_rng(11)
    frames, truth = _stack(rng, 20)
    calib = synth.linear_calib(frames.shape[2], frames.shape[1], 0.1, 0.1)
    dev = torch.from_numpy(frames).cuda()
    depth, valid, info, cols = S.bone_contour(dev, calib, column_rows=True)
    for k in range(len(frames)):
        row, ocols, nv, thr = orc_contour(frames[k])
        assert info["rows"][k] == row and info["valid_columns"][k] == nv
        assert info["brightness_threshold"][k] == thr
        assert np.array_equal(cols[k], ocols)
    phantom = ~np.isnan(truth)
    assert valid[phantom].all() and not valid[~phantom].any()
    assert np.all(np.abs(depth[phantom] - truth[phantom]) <= 2.0)


def test_apply_cut_gpu_equals_oracle_and_kat():
    rng = np.random.default_rng(12)
    frames = rng.integers(1, 256, (6, 600, 80), dtype=np.uint8)
    calib = synth.linear_calib(80, 600, 0.1, 0.1)
    cuts = np.array([30.0, 0.0, 59.0, 60.0, 12.34, -3.0])
    dev = torch.from_numpy(frames).cuda()
    S.apply_cut(dev, cuts, 15.0, calib)
    got = dev.cpu().numpy()
    for k in range(len(frames)):
        ref = frames[k].copy()
        r0, r1 = C.c_int32(), C.c_int32()
        O.lib().orc_cut_rows(cuts[k], 15.0, 0.1, 600, C.byref(r0), C.byref(r1))
        O.lib().orc_apply_cut(ref.ctypes.data, 80, 80, 600, r0.value, r1.value)
        assert np.array_equal(got[k], ref)
    assert np.array_equal(got[0][300:451], frames[0][300:451]) and not got[0][:300].any()
    assert not got[3].any()  # cut at the bottom edge -> all zero
    again = dev.clone()
    S.apply_cut(again, cuts, 15.0, calib)  # idempotent
    assert torch.equal(again, dev)
    with pytest.raises(pkg.InvalidInput):
        S.apply_cut(torch.from_numpy(frames), cuts, 15.0, calib)  # host frames are refused


def _pipeline_oracle(wl, frames, cut_rows):
    ref = O.OracleGrid.for_workload(wl)
    f2 = frames.copy()
    for k, (r0, r1) in enumerate(cut_rows):
        O.lib().orc_apply_cut(f2[k].ctypes.data, wl.w, wl.w, wl.h, r0, r1)
    ref.insert_frames(f2, wl.poses, wl.calib, skip_zero=True)
    return ref


@pytest.mark.parametrize("alg", ["alg1", "alg2"])
def test_segmented_insert_equals_oracle(alg):
    wl = synth.small_linear(nframes=10, w=64, h=48)
    rng = np.random.default_rng(13)
    frames = wl.frames_np()
    # give the frames a cortex + shadow so Algorithm 2 finds contours (rows scale to 0.2 mm)
    for k in range(len(frames)):
        img, _ = phantom_frame(rng, w=64, h=48, sy=wl.calib.scale_y_mm, bone_mm=5.0 + 0.1 * k, fascia_mm=2.0)
        frames[k] = img
    dev = torch.from_numpy(frames).cuda()
    if alg == "alg1":
        prof = S.segment_stream_alg1(dev, wl.poses, wl.calib, S.Alg1Params(K=0.1, D=3.0, L=20.0), band_mm=4.0)
    else:
        prof = S.segment_scan_alg2(dev, wl.calib, window=3, band_mm=4.0, shadow_mm=1.0)
    rows = [S.cut_rows(c, prof.band_mm, wl.calib) for c in prof.cut_mm]
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    grid.insert_frames(dev, wl.poses, wl.calib, skip_zero=True)
    ref = _pipeline_oracle(wl, frames, rows)
    s, c = grid.accumulators()
    assert np.array_equal(c, ref.count) and np.array_equal(s, ref.sum)
    assert grid.stats()["pixels_skipped_zero"] == ref.stats["skipped_zero"]
    assert '"cuts"' in prof.to_json()


def test_vpi_full_band_equals_plain_projection():
    """a VPI band covering the whole image equals the unsegmented projection."""
    wl = synth.small_linear()
    frames = np.maximum(wl.frames_np(), 1)  # no zero pixels: skip_zero changes nothing
    g1 = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    dev = torch.from_numpy(frames).cuda()
    ext = S.axial_extent_mm(wl.calib)
    vpi = S.vpi_fixed_depth(dev, wl.poses, wl.calib, 0.0, ext + 1.0, g1)
    g2 = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    g2.insert_frames(frames, wl.poses, wl.calib)
    assert np.array_equal(vpi, g2.coronal_projection(pkg.PROJ_MAX, depth_axis=1))


def test_alg2_tilt_tolerance_ramp():
    """SPEC segment examples: a 35 -> 45 mm ramp with +-10 deg tilt jitter, smoothed depth within
    +-2 mm of truth for >= 95% of frames."""
    rng = np.random.default_rng(14)
    n = 60
    imgs, truth = [], []
    for k in range(n):
        d = 35.0 + 10.0 * k / (n - 1)
        img, t = phantom_frame(rng, w=192, h=600, bone_mm=d, tilt_deg=rng.uniform(-10, 10))
        imgs.append(img)
        truth.append(d)
    calib = synth.linear_calib(192, 600, 0.1, 0.1)
    dev = torch.from_numpy(np.stack(imgs)).cuda()
    depth, valid, _ = S.bone_contour(dev, calib)
    sm = S.smooth_depths(depth, valid, 11)
    assert np.mean(np.abs(sm - np.array(truth)) <= 2.0) >= 0.95
