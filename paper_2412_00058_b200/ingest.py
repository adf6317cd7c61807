"""Ingest front-end: ScanBundle -> matched poses -> cropped frames -> the CUDA
insert path, plus the SPEC output formats (volume file SPEC.md:344, x-slices SPEC.md:316-324).

A ScanBundle directory holds
  frames/NNNNNN.pgm   binary PGM (P5) raw screenshots (image.hpp:34-72)
  frames.jsonl        {"t_ms": float, "file": "frames/000000.pgm"} per frame
  poses.jsonl         {"t_ms": float, "q": [w, x, y, z], "p": [x, y, z]} (transducer -> world, mm)
  calib.json          {"crop_rect": [x, y, w, h], "scale_mm": [sx, sy],
                       "image_to_transducer": 16 numbers (4x4 row-major, geometry "External
                       Interfaces"), "latency_ms": L, "probe": "linear" | "fan",
                       "fan": {"angle_deg", "r0_mm", "r1_mm"}}   (layout pinned here: the SPEC
                       fixes only the 16-number matrix)
  truth.json          optional, passed through.

Decoding and cropping run in native threads (`svr_load_frames`, the crop applied while the rows
are read, so only the B-mode rectangle reaches the pinned staging buffer); frame/pose matching is
`svr_match_poses` (t_frame - latency_ms, interpolate_pose geometry.hpp:194-209).  Frames whose
shifted time falls outside the pose span cannot be posed (interpolate_pose throws) and are
skipped and counted.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import threading
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi
from ._abi import RIGID_DTYPE, Calib, InvalidInput, IoError, check, lib, rigid_array, rigid_ptr

SCHEMA_VERSION = 1


# ---------------------------------------------------------------- PGM (image.hpp:34-72)
def read_pgm(path) -> np.ndarray:
    """read_pgm (image.hpp:44-72): H x W u8 array; IoError / InvalidInput as the reference."""
    p = os.fsencode(path)
    w, h = C.c_int32(), C.c_int32()
    check(lib().svr_pgm_info(p, C.byref(w), C.byref(h)))
    out = np.empty((h.value, w.value), np.uint8)
    check(lib().svr_pgm_read(p, out.ctypes.data, max(w.value, 1), w.value, h.value))
    return out


def write_pgm(path, img) -> None:
    """write_pgm (image.hpp:34-42) of an H x W u8 array."""
    a = np.ascontiguousarray(img, dtype=np.uint8)
    if a.ndim != 2:
        raise InvalidInput("write_pgm needs a 2-D u8 image")
    check(lib().svr_pgm_write(os.fsencode(path), a.ctypes.data, max(a.shape[1], 1), a.shape[1],
                              a.shape[0]))


# ---------------------------------------------------------------- calibration JSON
def calib_from_json(d: dict) -> Calib:
    from .reconstruct import pose_from_matrix4
    c = Calib()
    try:
        x, y, w, h = (int(v) for v in d["crop_rect"])
        sx, sy = (float(v) for v in d["scale_mm"])
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidInput(f"calib.json: {e}") from None
    c.crop_x, c.crop_y, c.crop_w, c.crop_h = x, y, w, h
    c.scale_x_mm, c.scale_y_mm = sx, sy
    m = d.get("image_to_transducer")
    if m is None:
        c.image_to_transducer = _abi.Rigid(1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    else:
        if len(m) != 16:
            raise InvalidInput("calib.json: image_to_transducer needs 16 numbers")
        c.image_to_transducer = pose_from_matrix4(m)
    c.latency_ms = float(d.get("latency_ms", 0.0))
    probe = d.get("probe", "linear")
    if probe == "fan":
        f = d.get("fan", {})
        c.probe = _abi.PROBE_FAN
        c.fan_angle_deg = float(f.get("angle_deg", 0.0))
        c.fan_r0_mm = float(f.get("r0_mm", 0.0))
        c.fan_r1_mm = float(f.get("r1_mm", 0.0))
    elif probe == "linear":
        c.probe = _abi.PROBE_LINEAR
    else:
        raise InvalidInput(f"calib.json: unknown probe {probe!r}")
    return c


def _matrix4(r: _abi.Rigid) -> list:
    w, x, y, z = r.qw, r.qx, r.qy, r.qz
    m = [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y), r.tx,
         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x), r.ty,
         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y), r.tz,
         0.0, 0.0, 0.0, 1.0]
    return [float(v) for v in m]


def calib_to_json(c: Calib) -> dict:
    d = {"schema_version": SCHEMA_VERSION,
         "crop_rect": [c.crop_x, c.crop_y, c.crop_w, c.crop_h],
         "scale_mm": [c.scale_x_mm, c.scale_y_mm],
         "image_to_transducer": _matrix4(c.image_to_transducer),
         "latency_ms": c.latency_ms,
         "probe": "fan" if c.probe == _abi.PROBE_FAN else "linear"}
    if c.probe == _abi.PROBE_FAN:
        d["fan"] = {"angle_deg": c.fan_angle_deg, "r0_mm": c.fan_r0_mm, "r1_mm": c.fan_r1_mm}
    return d


# ---------------------------------------------------------------- ScanBundle
def _read_jsonl(path):
    try:
        with open(path) as f:
            return [json.loads(line) for line in f if line.strip()]
    except OSError as e:
        raise IoError(f"cannot read {path}: {e}") from None
    except json.JSONDecodeError as e:
        raise InvalidInput(f"{path}: {e}") from None


@dataclass
class ScanBundle:
    root: str
    frame_files: list
    frame_t_ms: np.ndarray
    pose_t_ms: np.ndarray
    poses: np.ndarray          # RIGID_DTYPE
    calib: Calib
    raw_w: int
    raw_h: int
    truth: Optional[dict] = None

    @property
    def nframes(self):
        return len(self.frame_files)

    def match_poses(self):
        """(poses, valid mask): interpolate_pose at t_frame - latency_ms (svr_match_poses)."""
        m = self.nframes
        out = np.zeros(max(m, 1), dtype=RIGID_DTYPE)
        valid = np.zeros(max(m, 1), np.uint8)
        nv = C.c_int32()
        pt = np.ascontiguousarray(self.pose_t_ms, np.float64)
        ft = np.ascontiguousarray(self.frame_t_ms, np.float64)
        check(lib().svr_match_poses(pt.ctypes.data_as(C.POINTER(C.c_double)), rigid_ptr(self.poses),
                                    len(self.poses), ft.ctypes.data_as(C.POINTER(C.c_double)), m,
                                    float(self.calib.latency_ms), rigid_ptr(out), valid.ctypes.data,
                                    C.byref(nv)))
        return out[:m], valid[:m].astype(bool)

    def load_frames(self, idx=None, out=None, threads: int = 0, crop: bool = True) -> np.ndarray:
        """Decode frames `idx` (default all) with the crop_rect applied, into `out` (an
        (n, h, w) u8 array or pinned tensor) or a new array."""
        idx = range(self.nframes) if idx is None else idx
        paths = [os.fsencode(self.frame_files[i]) for i in idx]
        n = len(paths)
        c = self.calib
        h, w = (c.crop_h, c.crop_w) if crop else (self.raw_h, self.raw_w)
        if out is None:
            out = np.empty((n, h, w), np.uint8)
        arr = (C.c_char_p * max(n, 1))(*paths)
        cr = (C.c_int32 * 4)(c.crop_x, c.crop_y, c.crop_w, c.crop_h) if crop else None
        bad = C.c_int32(-1)
        check(lib().svr_load_frames(arr, n, self.raw_w, self.raw_h, cr, _abi.ptr(out), h * w,
                                    int(threads), C.byref(bad)))
        return out


def read_bundle(root) -> ScanBundle:
    root = os.fspath(root)
    frames = _read_jsonl(os.path.join(root, "frames.jsonl"))
    poses = _read_jsonl(os.path.join(root, "poses.jsonl"))
    try:
        with open(os.path.join(root, "calib.json")) as f:
            calib = calib_from_json(json.load(f))
    except OSError as e:
        raise IoError(f"cannot read calib.json: {e}") from None
    except json.JSONDecodeError as e:
        raise InvalidInput(f"calib.json: {e}") from None
    try:
        ft = np.array([float(r["t_ms"]) for r in frames], np.float64)
        files = [os.path.join(root, r["file"]) for r in frames]
        pt = np.array([float(r["t_ms"]) for r in poses], np.float64)
        pa = np.zeros(len(poses), dtype=RIGID_DTYPE)
        for i, r in enumerate(poses):
            pa[i] = (*[float(v) for v in r["q"]], *[float(v) for v in r["p"]])
    except (KeyError, TypeError, ValueError) as e:
        raise InvalidInput(f"bundle records: {e}") from None
    if len(ft) and np.any(np.diff(ft) < 0):
        raise InvalidInput("frames.jsonl timestamps must be non-decreasing")
    raw_w = raw_h = 0
    if files:
        w, h = C.c_int32(), C.c_int32()
        check(lib().svr_pgm_info(os.fsencode(files[0]), C.byref(w), C.byref(h)))
        raw_w, raw_h = w.value, h.value
        c = calib
        if c.crop_x < 0 or c.crop_y < 0 or c.crop_x + c.crop_w > raw_w or c.crop_y + c.crop_h > raw_h:
            raise InvalidInput("calibration crop_rect outside the raw frame")
    truth = None
    tp = os.path.join(root, "truth.json")
    if os.path.exists(tp):
        with open(tp) as f:
            truth = json.load(f)
    return ScanBundle(root, files, ft, pt, pa, calib, raw_w, raw_h, truth)


def write_bundle(root, frames, frame_t_ms, pose_t_ms, poses, calib: Calib, raw=None,
                 truth: Optional[dict] = None) -> None:
    """Write a ScanBundle.  `frames` are the B-mode images (n, crop_h, crop_w); with
    raw=(raw_w, raw_h) each is embedded at crop_rect in a zero screenshot of that size."""
    root = os.fspath(root)
    os.makedirs(os.path.join(root, "frames"), exist_ok=True)
    frames = np.asarray(frames, np.uint8)
    recs = []
    for k in range(len(frames)):
        name = f"frames/{k:06d}.pgm"
        img = frames[k]
        if raw is not None:
            scr = np.zeros((raw[1], raw[0]), np.uint8)
            scr[calib.crop_y:calib.crop_y + calib.crop_h, calib.crop_x:calib.crop_x + calib.crop_w] = img
            img = scr
        write_pgm(os.path.join(root, name), img)
        recs.append({"t_ms": float(frame_t_ms[k]), "file": name})
    with open(os.path.join(root, "frames.jsonl"), "w") as f:
        f.writelines(json.dumps(r) + "\n" for r in recs)
    pa = rigid_array(poses)
    with open(os.path.join(root, "poses.jsonl"), "w") as f:
        for t, p in zip(pose_t_ms, pa):
            f.write(json.dumps({"t_ms": float(t), "q": [float(p[k]) for k in ("qw", "qx", "qy", "qz")],
                                "p": [float(p[k]) for k in ("tx", "ty", "tz")]}) + "\n")
    with open(os.path.join(root, "calib.json"), "w") as f:
        json.dump(calib_to_json(calib), f, indent=1)
    if truth is not None:
        with open(os.path.join(root, "truth.json"), "w") as f:
            json.dump(truth, f)


# ---------------------------------------------------------------- streaming ingest
@dataclass
class IngestStats:
    frames: int = 0
    frames_unposed: int = 0
    batches: int = 0
    wall_s: float = 0.0
    decode_s: float = 0.0
    batch_latency_ms: list = field(default_factory=list)

    def as_dict(self):
        lat = sorted(self.batch_latency_ms)
        pct = (lambda p: lat[min(len(lat) - 1, int(p * (len(lat) - 1) + 0.5))] if lat else 0.0)
        return {"schema_version": SCHEMA_VERSION, "frames": self.frames,
                "frames_unposed": self.frames_unposed, "batches": self.batches,
                "wall_s": self.wall_s, "fps": self.frames / self.wall_s if self.wall_s else 0.0,
                "decode_s": self.decode_s,
                "batch_latency_ms": {"p50": pct(0.5), "p95": pct(0.95), "max": lat[-1] if lat else 0.0}}


def ingest(bundle: ScanBundle, grid, batch: int = 256, threads: int = 0, fill_radius: int = 1,
           fill_mode: int = _abi.FILL_MEAN, render: bool = True, render_params=None,
           frame_filter=None, skip_zero: bool = False) -> IngestStats:
    """Reconstruct a bundle incrementally: native decode of batch i+1 overlaps the GPU work of
    batch i (ctypes releases the GIL); each batch is inserted (H2D staged by svr_insert_frames
    from pinned memory), then its dirty region is filled and re-rendered.  frame_filter(k0,
    frames, poses) may rewrite a decoded batch in place (segmentation cuts) before insertion."""
    import torch
    from .reconstruct import dilate
    st = IngestStats()
    t0 = time.perf_counter()
    poses, valid = bundle.match_poses()
    idx = np.flatnonzero(valid)
    st.frames_unposed = int(bundle.nframes - len(idx))
    c = bundle.calib
    h, w = c.crop_h, c.crop_w
    nb = min(batch, max(len(idx), 1))
    bufs = [torch.empty((nb, h, w), dtype=torch.uint8).pin_memory() for _ in range(2)]
    chunks = [idx[i:i + nb] for i in range(0, len(idx), nb)]
    err = []

    def decode(k, buf):
        t = time.perf_counter()
        try:
            bundle.load_frames(chunks[k], out=buf, threads=threads)
        except Exception as e:  # re-raised on the calling thread
            err.append(e)
        st.decode_s += time.perf_counter() - t

    if chunks:
        decode(0, bufs[0])
    for k, ch in enumerate(chunks):
        if err:
            raise err[0]
        tb = time.perf_counter()
        worker = None
        if k + 1 < len(chunks):
            worker = threading.Thread(target=decode, args=(k + 1, bufs[(k + 1) % 2]))
            worker.start()
        buf = bufs[k % 2][:len(ch)]
        pk = poses[ch]
        if frame_filter is not None:
            frame_filter(ch, buf.numpy(), pk)
        boxes, u = grid.insert_frames(buf, pk, c, skip_zero=skip_zero, want_boxes=True)
        if not u.empty():
            grid.fill_holes(dilate(u, fill_radius), fill_radius, fill_mode, count=False)
            if render:
                grid.render_coronal(u, render_params, fill_radius)
        grid.sync()
        if worker is not None:
            worker.join()
        st.batch_latency_ms.append((time.perf_counter() - tb) * 1e3)
        st.frames += len(ch)
        st.batches += 1
    if err:
        raise err[0]
    st.wall_s = time.perf_counter() - t0
    return st


# ---------------------------------------------------------------- outputs
def volume_meta(grid, compound_mode: str = "mean") -> dict:
    d = grid.desc
    return {"schema_version": SCHEMA_VERSION, "dims": [d.nx, d.ny, d.nz], "voxel_mm": d.voxel_mm,
            "origin": [d.origin_mm[0], d.origin_mm[1], d.origin_mm[2]],
            "compound_mode": compound_mode, "frames_inserted": int(grid.stats()["frames_inserted"]),
            "z_slab": [d.z_begin, d.z_end]}


def write_volume(grid, path, apply_fills: bool = True, meta_path=None) -> dict:
    """Volume file: raw u8 x fastest then y then z + meta JSON alongside."""
    check(lib().svr_export_volume(grid.handle, os.fsencode(path), int(apply_fills)))
    meta = volume_meta(grid)
    meta["fills_applied"] = bool(apply_fills)
    with open(meta_path or (os.fspath(path) + ".json"), "w") as f:
        json.dump(meta, f, indent=1)
    return meta


def read_volume(path, meta_path=None):
    """(values (nz, ny, nx) u8, meta) of a volume file written by write_volume."""
    with open(meta_path or (os.fspath(path) + ".json")) as f:
        meta = json.load(f)
    nx, ny, nz = meta["dims"]
    z0, z1 = meta.get("z_slab", [0, nz])
    v = np.fromfile(path, np.uint8)
    if v.size != nx * ny * (z1 - z0):
        raise InvalidInput(f"{path}: {v.size} bytes, expected {nx * ny * (z1 - z0)}")
    return v.reshape(z1 - z0, ny, nx), meta


def export_slices(grid, directory, apply_fills: bool = True, digits: int = 4) -> int:
    """export_slices(axis=x): nx PGM images of ny x nz (row = z, col = y),
    zero-padded names, plus meta.json.  Returns the file count."""
    os.makedirs(directory, exist_ok=True)
    n = C.c_int32()
    check(lib().svr_export_slices(grid.handle, os.fsencode(directory), int(apply_fills), int(digits),
                                  C.byref(n)))
    meta = volume_meta(grid)
    meta.update({"axis": "x", "files": n.value, "digits": digits, "fills_applied": bool(apply_fills),
                 "image": "width = ny (y), height = nz (z)"})
    with open(os.path.join(directory, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    return n.value


def import_slices(directory):
    """Inverse of export_slices: (values (nz, ny, nx) u8, meta)."""
    with open(os.path.join(directory, "meta.json")) as f:
        meta = json.load(f)
    nx, ny, _ = meta["dims"]
    z0, z1 = meta.get("z_slab", [0, meta["dims"][2]])
    out = np.empty((z1 - z0, ny, nx), np.uint8)
    for x in range(nx):
        out[:, :, x] = read_pgm(os.path.join(directory, f"{x:0{meta['digits']}d}.pgm"))
    return out, meta
