"""CPU suite for the ingest front-end and output formats (no GPU): PGM I/O pinned against the
reference's own read_pgm / write_pgm (image.hpp:34-72, compiled in oracle/_ref), the ScanBundle
round trip with the crop applied while decoding, the native loader's error reporting, and frame /
pose matching against the reference interpolate_pose (geometry.hpp:194-209)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from oracle import oracle as O
from paper_2412_00058_b200 import _abi, ingest, synth

needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (reference headers) not built")


def _ref_read(path, cap=1 << 20):
    buf = np.zeros(cap, np.uint8)
    w, h = C.c_int32(), C.c_int32()
    rc = O.ref().ref_read_pgm(os.fsencode(path), buf.ctypes.data, cap, C.byref(w), C.byref(h))
    if rc:
        return rc, None
    return 0, buf[:w.value * h.value].reshape(h.value, w.value)


def _code(fn):
    try:
        fn()
        return 0
    except pkg.InvalidInput:
        return 2
    except pkg.IoError:
        return 4


PGM_CASES = {
    "plain": b"P5\n4 3\n255\n" + bytes(range(12)),
    "comments": b"P5\n# a comment\n4 # w\n3\n# more\n255\n" + bytes(range(100, 112)),
    "tabs_crlf": b"P5\t4\r\n3   255\n" + bytes(range(12)),
    "zero_width": b"P5\n0 5\n255\n",
    "not_p5": b"P2\n4 3\n255\n" + bytes(12),
    "p5_glued": b"P5x\n4 3\n255\n" + bytes(12),
    "maxval16": b"P5\n4 3\n16\n" + bytes(12),
    "truncated": b"P5\n4 3\n255\n" + bytes(11),
    "negative": b"P5\n-4 3\n255\n" + bytes(12),
    "garbage_dim": b"P5\nfour 3\n255\n" + bytes(12),
    "empty": b"",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(PGM_CASES))
def test_read_pgm_matches_reference(name, tmp_path):
    p = tmp_path / f"{name}.pgm"
    p.write_bytes(PGM_CASES[name])
    rc, ref_img = _ref_read(p)
    ours = []
    assert _code(lambda: ours.append(ingest.read_pgm(p))) == rc
    if rc == 0:
        assert np.array_equal(ours[0], ref_img)


@needs_ref
def test_read_pgm_missing_file_is_io_error(tmp_path):
    rc, _ = _ref_read(tmp_path / "nope.pgm")
    assert rc == 4
    with pytest.raises(pkg.IoError):
        ingest.read_pgm(tmp_path / "nope.pgm")


@needs_ref
def test_write_pgm_byte_identical_to_reference(tmp_path):
    img = np.random.default_rng(1).integers(0, 256, (37, 53), dtype=np.uint8)
    ingest.write_pgm(tmp_path / "a.pgm", img)
    assert O.ref().ref_write_pgm(os.fsencode(tmp_path / "b.pgm"), img.ctypes.data, 53, 37) == 0
    assert (tmp_path / "a.pgm").read_bytes() == (tmp_path / "b.pgm").read_bytes()
    assert np.array_equal(ingest.read_pgm(tmp_path / "a.pgm"), img)
    with pytest.raises(pkg.IoError):
        ingest.write_pgm(tmp_path / "no_dir" / "x.pgm", img)


def _bundle(tmp_path, n=9, raw=(80, 64), latency=0.0):
    wl = synth.small_linear(nframes=n)
    c = wl.calib
    c.crop_x, c.crop_y = 7, 5
    c.latency_ms = latency
    frames = wl.frames_np()
    ft = 33.3 * np.arange(n)
    # poses sampled at 2x the frame rate, spanning the frames' (shifted) times
    pt = np.linspace(ft[0] - latency, ft[-1] - latency, 2 * n - 1)
    pa = np.zeros(len(pt), dtype=_abi.RIGID_DTYPE)
    for i in range(len(pt)):
        pa[i] = wl.poses[min(i // 2, n - 1)]
    ingest.write_bundle(tmp_path / "b", frames, ft, pt, pa, c, raw=raw, truth={"note": "x"})
    return wl, frames, ft, pt, pa


def test_bundle_roundtrip_with_crop(tmp_path):
    wl, frames, ft, pt, pa = _bundle(tmp_path)
    b = ingest.read_bundle(tmp_path / "b")
    assert (b.raw_w, b.raw_h) == (80, 64) and b.nframes == len(frames)
    assert (b.calib.crop_x, b.calib.crop_y, b.calib.crop_w, b.calib.crop_h) == (7, 5, wl.w, wl.h)
    for nth in (1, 3):
        got = b.load_frames(threads=nth)
        assert np.array_equal(got, frames)
    raw = b.load_frames(idx=[2], crop=False)
    assert raw.shape == (1, 64, 80) and np.array_equal(raw[0, 5:5 + wl.h, 7:7 + wl.w], frames[2])
    assert raw[0, :5].sum() == 0
    assert np.array_equal(b.poses, pa) and np.array_equal(b.frame_t_ms, ft)
    assert b.truth == {"note": "x"}
    r, r0 = b.calib.image_to_transducer, wl.calib.image_to_transducer
    for f in ("qw", "qx", "qy", "qz", "tx", "ty", "tz"):  # via the 4x4 matrix form
        assert abs(getattr(r, f) - getattr(r0, f)) < 1e-12


def test_loader_reports_lowest_failing_frame(tmp_path):
    _bundle(tmp_path)
    b = ingest.read_bundle(tmp_path / "b")
    for k in (6, 3):
        with open(b.frame_files[k], "r+b") as f:
            f.truncate(20)
    for nth in (1, 4):
        with pytest.raises(pkg.InvalidInput, match="frame 3: truncated PGM data"):
            b.load_frames(threads=nth)
    os.remove(b.frame_files[1])
    with pytest.raises(pkg.IoError, match="frame 1: cannot open"):
        b.load_frames(threads=2)


def test_bundle_errors(tmp_path):
    _bundle(tmp_path)
    root = tmp_path / "b"
    cal = json.loads((root / "calib.json").read_text())
    cal["crop_rect"] = [70, 0, 20, 10]
    (root / "calib.json").write_text(json.dumps(cal))
    with pytest.raises(pkg.InvalidInput, match="crop_rect"):
        ingest.read_bundle(root)
    (root / "calib.json").write_text("{not json")
    with pytest.raises(pkg.InvalidInput):
        ingest.read_bundle(root)
    os.remove(root / "calib.json")
    with pytest.raises(pkg.IoError):
        ingest.read_bundle(root)


@needs_ref
@pytest.mark.parametrize("latency", [0.0, 12.5])
def test_match_poses_vs_reference(tmp_path, latency):
    rng = np.random.default_rng(5)
    _bundle(tmp_path, latency=latency)
    b = ingest.read_bundle(tmp_path / "b")
    # richer pose stream: random rotations, irregular times; some frames fall outside it
    n = 25
    b.pose_t_ms = np.sort(rng.uniform(10.0, 250.0, n))
    b.poses = _abi.rigid_array([synth.rigid(q / np.linalg.norm(q), rng.uniform(-30, 30, 3))
                                for q in rng.normal(size=(n, 4))])
    poses, valid = b.match_poses()
    R = O.ref()
    PD = C.POINTER(C.c_double)
    for k in range(b.nframes):
        t = b.frame_t_ms[k] - latency
        inside = b.pose_t_ms[0] <= t <= b.pose_t_ms[-1]
        assert valid[k] == inside
        if inside:
            r2 = _abi.Rigid()
            rc = R.ref_interpolate_pose(b.pose_t_ms.ctypes.data_as(PD), _abi.rigid_ptr(b.poses), n, t,
                                        C.byref(r2))
            assert rc == 0
            assert list(poses[k]) == [getattr(r2, f) for f, _ in r2._fields_]
    assert (~valid).any() and valid.any()


def test_calib_json_roundtrip_fan():
    c = synth.fan_calib(24, 96, 60.0, 20.0, 150.0, i2t=synth.rigid(synth.quat_axis_angle((0, 1, 0), 0.3), (1, 2, 3)))
    c.latency_ms = 7.0
    d = ingest.calib_to_json(c)
    assert len(d["image_to_transducer"]) == 16
    c2 = ingest.calib_from_json(json.loads(json.dumps(d)))
    assert c2.probe == _abi.PROBE_FAN and c2.fan_r1_mm == 150.0 and c2.latency_ms == 7.0
    for f in ("qw", "qx", "qy", "qz", "tx", "ty", "tz"):
        assert abs(getattr(c2.image_to_transducer, f) - getattr(c.image_to_transducer, f)) < 1e-12


def test_cli_exit_codes_cpu(tmp_path):
    """cli exit codes: invalid input 2, I/O 4; no GPU needed to fail early."""
    from paper_2412_00058_b200 import cli
    assert cli.main(["synth", "bundle", "--frames", "0", "--out", str(tmp_path / "b")]) == 2
    assert cli.main(["reconstruct", "--bundle", str(tmp_path / "missing"), "--out", str(tmp_path / "v")]) == 4
    assert cli.main(["project", "--out", str(tmp_path / "p.pgm")]) == 2
    assert cli.main(["nonsense"]) == 2
    assert cli.main(["project", "--volume", str(tmp_path / "none.raw"), "--out", str(tmp_path / "p.pgm")]) == 4
