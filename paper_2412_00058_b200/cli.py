"""Command-line surface over the CUDA path (SPEC.md cli module, :601-617):

  reconstruct --bundle DIR [--voxel-mm 1.0] [--mode incremental|batch] [--segment none|alg1|alg2]
              [--K --D --L --band --window] [--dims NX NY NZ --origin X Y Z] --out volume.raw
  project     --volume volume.raw [--mode max|mean] [--axis 1] --out proj.pgm
  project vpi --bundle DIR --depth 35 --band 15 [--voxel-mm] --out proj.pgm
  export-slices --bundle DIR --out DIR
  bench ingest --bundle DIR [--batch 256]
  synth bundle --config small|cfg1|cfg2 --out DIR [--frames N] [--raw W H]

Exit codes (core.hpp:12-32): 0 ok, 2 invalid input, 3 algorithm failure, 4 I/O, 5 device.
JSON outputs carry schema_version.  Config precedence: flags > SPINEVOL_* env > defaults.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

from . import _abi
from ._abi import AlgorithmFailure, DeviceError, InvalidInput, IoError, SpinevolError

SCHEMA_VERSION = 1
EXIT = {InvalidInput: 2, AlgorithmFailure: 3, IoError: 4, DeviceError: 5}


def _env(name, default, cast=float):
    v = os.environ.get("SPINEVOL_" + name)
    return cast(v) if v is not None else default


def _emit(obj, path=None):
    obj = {"schema_version": SCHEMA_VERSION, **obj}
    s = json.dumps(obj, indent=1)
    if path:
        with open(path, "w") as f:
            f.write(s)
    print(json.dumps(obj))


# ---------------------------------------------------------------- grid sizing
def grid_for_bundle(bundle, poses, voxel_mm, margin_mm=10.0):
    """SPEC grid sizing: the posed frames' world bounding box + 10 mm margin."""
    from .reconstruct import pixel_to_world
    c = bundle.calib
    if c.probe == _abi.PROBE_FAN:
        pts = [(c.crop_w - 1, 0), (c.crop_w - 1, c.crop_h - 1), (0, 0), (0, c.crop_h - 1),
               (c.crop_w - 1, (c.crop_h - 1) // 2)]
    else:
        pts = [(0, 0), (c.crop_w - 1, 0), (0, c.crop_h - 1), (c.crop_w - 1, c.crop_h - 1)]
    lo = np.full(3, np.inf)
    hi = np.full(3, -np.inf)
    for p in poses:
        r = _abi.Rigid(*[float(v) for v in p])
        for col, row in pts:
            w = np.array(pixel_to_world(col, row, c, r))
            lo = np.minimum(lo, w)
            hi = np.maximum(hi, w)
    if not np.all(np.isfinite(lo)):
        raise InvalidInput("no posed frames to size the grid from")
    lo -= margin_mm
    hi += margin_mm
    dims = tuple(int(math.ceil((hi[k] - lo[k]) / voxel_mm)) + 1 for k in range(3))
    return dims, tuple(float(v) for v in lo)


def _grid(args, bundle, poses):
    from .reconstruct import VoxelGrid
    if args.dims:
        dims, origin = tuple(args.dims), tuple(args.origin or (0.0, 0.0, 0.0))
    else:
        dims, origin = grid_for_bundle(bundle, poses, args.voxel_mm)
    return VoxelGrid(dims, args.voxel_mm, origin, device=args.device)


def _segment(args, frames_dev, poses, calib):
    from . import segment as S
    if args.segment == "alg1":
        return S.segment_stream_alg1(frames_dev, poses, calib, S.Alg1Params(args.K, args.D, args.L), args.band)
    if args.segment == "alg2":
        return S.segment_scan_alg2(frames_dev, calib, window=args.window, band_mm=args.band)
    return None


# ---------------------------------------------------------------- commands
def cmd_reconstruct(args):
    import torch
    from . import ingest
    from .reconstruct import dilate
    b = ingest.read_bundle(args.bundle)
    if b.nframes == 0:
        raise InvalidInput("empty bundle")
    poses, valid = b.match_poses()
    grid = _grid(args, b, poses[valid])
    skip = args.segment != "none"
    stats = {}
    if args.mode == "batch" or args.segment == "alg2":
        # post-acquisition: decode everything, (segment,) insert once, fill the union once
        idx = np.flatnonzero(valid)
        fr = torch.from_numpy(b.load_frames(idx, threads=args.threads)).cuda(args.device)
        prof = _segment(args, fr, poses[idx], b.calib)
        _, u = grid.insert_frames(fr, poses[idx], b.calib, skip_zero=skip, want_boxes=True)
        if not u.empty():
            grid.fill_holes(dilate(u, args.fill_radius), args.fill_radius, args.fill_mode)
        if prof is not None:
            stats["cut_profile"] = json.loads(prof.to_json())
        stats["frames"] = int(len(idx))
    else:
        filt = None
        if args.segment == "alg1":
            from . import segment as S
            p1 = float(poses[np.flatnonzero(valid)[0]][("tx", "ty", "tz")[0]])

            def filt(k_idx, host_frames, pk):
                dev = torch.from_numpy(host_frames).cuda(args.device)
                S.segment_stream_alg1(dev, pk, b.calib, S.Alg1Params(args.K, args.D, args.L), args.band,
                                      p_c1=p1)
                host_frames[...] = dev.cpu().numpy()
        st = ingest.ingest(b, grid, batch=args.batch, threads=args.threads, fill_radius=args.fill_radius,
                           fill_mode=args.fill_mode, render=False, frame_filter=filt, skip_zero=skip)
        stats.update(st.as_dict())
    meta = ingest.write_volume(grid, args.out, apply_fills=True)
    stats.update({"out": args.out, "dims": meta["dims"], "origin": meta["origin"],
                  "voxel_mm": meta["voxel_mm"], "mode": args.mode, "segment": args.segment,
                  "grid_stats": grid.stats()})
    _emit(stats, args.stats)
    return 0


def cmd_project(args):
    from . import ingest
    if args.sub == "vpi":
        import torch
        from . import segment as S
        b = ingest.read_bundle(args.bundle)
        poses, valid = b.match_poses()
        idx = np.flatnonzero(valid)
        grid = _grid(args, b, poses[idx])
        fr = torch.from_numpy(b.load_frames(idx, threads=args.threads)).cuda(args.device)
        img = S.vpi_fixed_depth(fr, poses[idx], b.calib, args.depth, args.band, grid,
                                _abi.PROJ_MEAN if args.mode == "mean" else _abi.PROJ_MAX, args.axis)
    else:
        vol, meta = ingest.read_volume(args.volume)  # (nz, ny, nx)
        ax = {0: 2, 1: 1, 2: 0}[args.axis]
        if args.mode == "max":
            img = vol.max(axis=ax)
        else:
            nz = (vol > 0).sum(axis=ax)
            s = vol.astype(np.uint64).sum(axis=ax)
            img = np.where(nz > 0, (2 * s + nz) // np.maximum(2 * nz, 1), 0).astype(np.uint8)
    ingest.write_pgm(args.out, img)
    _emit({"out": args.out, "shape": list(img.shape), "mode": args.mode, "axis": args.axis})
    return 0


def cmd_export_slices(args):
    import torch
    from . import ingest
    from .reconstruct import dilate
    b = ingest.read_bundle(args.bundle)
    poses, valid = b.match_poses()
    idx = np.flatnonzero(valid)
    grid = _grid(args, b, poses[idx])
    fr = torch.from_numpy(b.load_frames(idx, threads=args.threads)).cuda(args.device)
    _, u = grid.insert_frames(fr, poses[idx], b.calib, want_boxes=True)
    if not u.empty():
        grid.fill_holes(dilate(u, args.fill_radius), args.fill_radius, args.fill_mode)
    n = ingest.export_slices(grid, args.out)
    _emit({"out": args.out, "files": n})
    return 0


def cmd_bench(args):
    from . import ingest
    from .reconstruct import VoxelGrid
    b = ingest.read_bundle(args.bundle)
    if b.nframes == 0:
        raise InvalidInput("empty bundle")
    poses, valid = b.match_poses()
    grid = _grid(args, b, poses[valid])
    ingest.ingest(b, grid, batch=args.batch, threads=args.threads)  # warm-up (page cache, JIT-free)
    grid.clear()
    st = ingest.ingest(b, grid, batch=args.batch, threads=args.threads)
    d = st.as_dict()
    d.update({"what": "ScanBundle decode (native threads) + pose match + H2D + insert + fill + render",
              "batch": args.batch, "frame": [b.calib.crop_w, b.calib.crop_h],
              "grid": list(grid.dims), "voxel_mm": args.voxel_mm})
    _emit(d, args.stats)
    return 0


def cmd_synth(args):
    import torch
    from . import ingest, synth
    makers = {"small": synth.small_linear, "cfg1": synth.cfg1, "cfg2": synth.cfg2, "fan": synth.small_fan}
    if args.config not in makers:
        raise InvalidInput(f"unknown config {args.config!r}")
    if args.frames is not None and args.frames <= 0:
        raise InvalidInput("--frames must be positive")
    wl = makers[args.config](nframes=args.frames) if args.frames else makers[args.config]()
    n = wl.nframes
    if n * wl.w * wl.h > (256 << 20) or args.config == "cfg2":
        dev = torch.empty((n, wl.h, wl.w), dtype=torch.uint8, device=f"cuda:{args.device}")
        synth.synth_frames_device(wl, dev, 0, n, device=args.device)
        frames = dev.cpu().numpy()
    else:
        frames = wl.frames_np()
    c = wl.calib
    raw = None
    if args.raw:
        raw = tuple(args.raw)
        c.crop_x, c.crop_y = (raw[0] - c.crop_w) // 2, (raw[1] - c.crop_h) // 2
        if c.crop_x < 0 or c.crop_y < 0:
            raise InvalidInput("--raw must be at least the B-mode image size")
    ft = 1000.0 / 30.0 * np.arange(n)
    ingest.write_bundle(args.out, frames, ft, ft - c.latency_ms, wl.poses, c, raw=raw,
                        truth={"config": args.config, "dims": list(wl.dims), "voxel_mm": wl.voxel_mm,
                               "origin": list(wl.origin)})
    _emit({"out": args.out, "frames": n, "config": args.config})
    return 0


def parser():
    ap = argparse.ArgumentParser(prog="spinevol-b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, grid=True):
        p.add_argument("--device", type=int, default=int(_env("DEVICE", 0, int)))
        p.add_argument("--threads", type=int, default=int(_env("THREADS", 0, int)))
        if grid:
            p.add_argument("--voxel-mm", dest="voxel_mm", type=float, default=_env("VOXEL_MM", 1.0))
            p.add_argument("--dims", type=int, nargs=3)
            p.add_argument("--origin", type=float, nargs=3)
            p.add_argument("--fill-radius", dest="fill_radius", type=int, default=1)
            p.add_argument("--fill-mode", dest="fill_mode", type=int, default=_abi.FILL_MEAN)

    r = sub.add_parser("reconstruct")
    common(r)
    r.add_argument("--bundle", required=True)
    r.add_argument("--mode", choices=["incremental", "batch"], default="incremental")
    r.add_argument("--segment", choices=["none", "alg1", "alg2"], default="none")
    r.add_argument("--K", type=float, default=_env("K", 0.04))
    r.add_argument("--D", type=float, default=_env("D", 35.0))
    r.add_argument("--L", type=float, default=_env("L", 500.0))
    r.add_argument("--band", type=float, default=_env("BAND", 15.0))
    r.add_argument("--window", type=int, default=int(_env("WINDOW", 11, int)))
    r.add_argument("--batch", type=int, default=256)
    r.add_argument("--out", required=True)
    r.add_argument("--stats")

    p = sub.add_parser("project")
    common(p)
    p.add_argument("sub", nargs="?", choices=["vpi"])
    p.add_argument("--volume")
    p.add_argument("--bundle")
    p.add_argument("--mode", choices=["max", "mean"], default="max")
    p.add_argument("--axis", type=int, default=1, choices=[0, 1, 2])
    p.add_argument("--depth", type=float, default=35.0)
    p.add_argument("--band", type=float, default=15.0)
    p.add_argument("--out", required=True)

    e = sub.add_parser("export-slices")
    common(e)
    e.add_argument("--bundle", required=True)
    e.add_argument("--out", required=True)

    bn = sub.add_parser("bench")
    common(bn)
    bn.add_argument("what", choices=["ingest"])
    bn.add_argument("--bundle", required=True)
    bn.add_argument("--batch", type=int, default=256)
    bn.add_argument("--stats")

    s = sub.add_parser("synth")
    s.add_argument("what", choices=["bundle"])
    s.add_argument("--config", default="small")
    s.add_argument("--frames", type=int)
    s.add_argument("--raw", type=int, nargs=2)
    s.add_argument("--device", type=int, default=0)
    s.add_argument("--out", required=True)
    return ap


def main(argv=None) -> int:
    ap = parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        if args.cmd == "project" and args.sub is None and not args.volume:
            raise InvalidInput("project needs --volume (or the vpi subcommand with --bundle)")
        if args.cmd == "project" and args.sub == "vpi" and not args.bundle:
            raise InvalidInput("project vpi needs --bundle")
        fn = {"reconstruct": cmd_reconstruct, "project": cmd_project, "export-slices": cmd_export_slices,
              "bench": cmd_bench, "synth": cmd_synth}[args.cmd]
        return fn(args)
    except SpinevolError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT.get(type(e), 1)
    except FileNotFoundError as e:
        print(f"error: {e}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
