"""CPU suite for the segmentation front-end: SPEC segment known-answer examples and properties on
the oracle (oracle/svr_oracle.c) and on the host half of the product (Algorithm 1 cut depth, cut
rows, Algorithm 2 depth smoothing in libspinevol_b200), with median_lower pinned against the
reference's own core.hpp:93-99.  The reference implements no segmentation: parity is to the
oracle's pins."""
import ctypes as C

import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import segment as S
from paper_2412_00058_b200 import synth
from seg_util import phantom_frame, speckle_frame

needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (reference headers) not built")
L = O.lib


def _orc_smooth(d, valid, window):
    d = np.ascontiguousarray(d, np.float64)
    v = np.ascontiguousarray(valid, np.uint8)
    out = np.empty_like(d)
    rc = L().orc_smooth_depths(d.ctypes.data, v.ctypes.data, len(d), window, out.ctypes.data)
    return rc, out


def test_alg1_kats_and_properties():
    p = S.Alg1Params(K=0.04, D=35.0, L=500.0)
    ext = 60.0
    # SPEC: mid-back offset -> D; scan start (p_cn = p_c1) -> 0.04 * 250 + 35 = 45; K = 0 -> D
    assert S.cut_depth_alg1(100.0, 100.0 - 250.0, p, ext) == 35.0
    assert S.cut_depth_alg1(100.0, 100.0, p, ext) == 45.0
    assert S.cut_depth_alg1(3.0, 77.0, S.Alg1Params(K=0.0, D=35.0, L=500.0), ext) == 35.0
    assert S.cut_depth_alg1(0.0, 5000.0, p, ext) == ext  # clamped to the axial extent
    rng = np.random.default_rng(0)
    for _ in range(200):
        p1, o1, o2 = rng.integers(-2400, 2400, 3) / 8.0  # dyadic: the offsets are exact
        a = S.cut_depth_alg1(p1, p1 - 250.0 - o1, p, 1e9)
        b = S.cut_depth_alg1(p1, p1 - 250.0 + o1, p, 1e9)
        assert a == b  # symmetric about the mid-back offset L/2
        if abs(o2) >= abs(o1):  # non-decreasing in |offset - L/2|
            assert S.cut_depth_alg1(p1, p1 - 250.0 - o2, p, 1e9) >= a
        assert a == L().orc_cut_depth_alg1(p1, p1 - 250.0 - o1, 0.04, 35.0, 500.0, 1e9)
    with pytest.raises(pkg.InvalidInput):
        S.cut_depth_alg1(0.0, 0.0, S.Alg1Params(K=-1.0), ext)


def test_cut_rows_kat_and_oracle():
    c = synth.linear_calib(64, 600, 0.1, 0.1)
    assert S.cut_rows(30.0, 15.0, c) == (300, 450)  # SPEC: rows 300..450 preserved
    r0, r1 = C.c_int32(), C.c_int32()
    rng = np.random.default_rng(1)
    for cut, band, sy in zip(rng.uniform(-5, 70, 300), rng.uniform(0.1, 30, 300), rng.uniform(0.05, 0.5, 300)):
        c.scale_y_mm = sy
        L().orc_cut_rows(cut, band, sy, 600, C.byref(r0), C.byref(r1))
        assert S.cut_rows(cut, band, c) == (r0.value, r1.value)
    c.scale_y_mm = 0.1
    r0, r1 = S.cut_rows(60.0, 15.0, c)  # cut at the bottom edge: nothing kept
    assert r0 > r1


def test_apply_cut_oracle_idempotent():
    rng = np.random.default_rng(2)
    img = rng.integers(1, 256, (600, 64), dtype=np.uint8)
    a = img.copy()
    L().orc_apply_cut(a.ctypes.data, 64, 64, 600, 300, 450)
    assert not a[:300].any() and not a[451:].any() and np.array_equal(a[300:451], img[300:451])
    b = a.copy()
    L().orc_apply_cut(b.ctypes.data, 64, 64, 600, 300, 450)
    assert np.array_equal(a, b)


def test_smooth_depths_kats():
    for fn in (lambda d, v, w: S.smooth_depths(d, v, w), lambda d, v, w: _orc_smooth(d, v, w)[1]):
        assert np.array_equal(fn([35.0] * 7, [1] * 7, 5), [35.0] * 7)
        assert np.array_equal(fn([35, 35, 80, 35, 35], [1] * 5, 5), [35.0] * 5)
        # one gap between 30 and 40 -> 35 before filtering (window 3 keeps the ramp)
        assert fn([30, 0, 40], [1, 0, 1], 3)[1] == 35.0
        # leading / trailing gaps take the nearest valid value
        out = fn([0, 0, 33, 0], [0, 0, 1, 0], 3)
        assert np.array_equal(out, [33.0] * 4)
    with pytest.raises(pkg.AlgorithmFailure):
        S.smooth_depths([1.0, 2.0], [0, 0], 3)
    with pytest.raises(pkg.InvalidInput):
        S.smooth_depths([1.0, 2.0], [1, 1], 4)
    assert _orc_smooth([1.0], [0], 3)[0] == -1


def test_smooth_depths_product_equals_oracle():
    rng = np.random.default_rng(3)
    for n in (1, 2, 5, 40, 301):
        for window in (3, 5, 11):
            d = rng.uniform(20, 50, n).round(3)
            v = rng.random(n) > 0.3
            if not v.any():
                v[n // 2] = True
            rc, ref = _orc_smooth(d, v, window)
            assert rc == 0
            assert np.array_equal(S.smooth_depths(d, v, window), ref)


@needs_ref
def test_median_lower_matches_reference():
    rng = np.random.default_rng(4)
    R = O.ref()
    for n in range(1, 14):
        v = rng.uniform(0, 100, n).round(1)
        ref = R.ref_median_lower(v.ctypes.data_as(C.POINTER(C.c_double)), n)
        # a window of 2n + 1 samples covers the whole series at every position
        out = S.smooth_depths(v, np.ones(n, np.uint8), 2 * n + 1)
        assert np.all(out == ref)


def orc_contour(img, pct=0.7, sy=0.1, min_frac=0.1):
    h, w = img.shape
    g, shadow = S.contour_thresholds(synth.linear_calib(w, h, 0.1, sy))
    rank = int(np.floor(pct * (w * h - 1)))
    cols = np.empty(w, np.int32)
    nv, thr = C.c_int32(), C.c_int32()
    row = L().orc_bone_contour(np.ascontiguousarray(img).ctypes.data, w, w, h, rank, g, shadow, min_frac,
                               cols.ctypes.data, C.byref(nv), C.byref(thr))
    return row, cols, nv.value, thr.value


def test_bone_contour_oracle_kats():
    rng = np.random.default_rng(5)
    # bone arc at 35 mm under a fascia band at 15 mm: the bottom-up scan finds the cortex
    img, truth = phantom_frame(rng)
    row, cols, nv, _ = orc_contour(img)
    assert row >= 0 and abs(row * 0.1 - 35.0) <= 0.5
    assert nv >= 0.9 * img.shape[1]
    # tilted 10 deg: the median over columns lies within the arc's depth span
    img, truth = phantom_frame(rng, tilt_deg=10.0)
    row, *_ = orc_contour(img)
    assert truth.min() - 0.5 <= row * 0.1 <= truth.max() + 0.5
    # pure speckle: no contour
    row, _, nv, _ = orc_contour(speckle_frame(rng))
    assert row == -1
