#!/usr/bin/env python
"""bench.py — B-scan pixel insertion throughput of the spinevol reconstruction hot path.

Step = one batch reconstruction of the BASELINE cfg2 whole-spine scan (2400 frames of
512x480 u8 -> 500x267x2000 voxels @ 0.3 mm): PNN insert of every frame (K1), 3x3x3 mean hole
fill of the dirty region as per-z-chunk boxes (K2), depth-band coronal render of the dirty
columns (K3, cfg4),
and for N>1 the NCCL gather of the coronal image.  Volume z-slab-sharded across ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.  --impl reference times the reference CPU path (the
reference's own spinevol::pixel_to_world insert loop, oracle/_ref, else the oracle port) on
the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "B-scan pixel insertions/sec (G/s)"
UNIT = "Gpx/s"
WORKLOAD = ("cfg2 whole-spine linear sweep: 2400 x 512x480 u8 frames -> 500x267x2000 voxels "
            "@0.3 mm; step = PNN insert + 3x3x3 mean fill of the dirty region + depth-band coronal "
            "render of the dirty columns (cfg4)")
FALLBACK_HBM_GBS = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _ncpu():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- CPU reference path
def cpu_reference(wl, frames, poses, nthreads, min_seconds=0.0, max_passes=1):
    """Time the reference CPU insert (oracle/_ref: spinevol::pixel_to_world per pixel, z-slab
    threads) on `frames`; falls back to the oracle port where _ref was not built."""
    from oracle import oracle as O
    kind = "reference" if O.ref() is not None else "port"
    times = []
    t_all = time.perf_counter()
    g = None
    acc = None
    if kind == "reference":  # preallocate + touch the grid outside the timed region
        acc = (np.ones(wl.dims[::-1], np.uint32), np.ones(wl.dims[::-1], np.uint16))
    while True:
        if kind == "reference":
            t0 = time.perf_counter()
            O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, poses, wl.calib,
                                nthreads=nthreads, out=acc)
            times.append(time.perf_counter() - t0)
        else:
            g = g or O.OracleGrid.for_workload(wl)
            t0 = time.perf_counter()
            g.insert_frames_mt(frames, poses, wl.calib, nthreads=nthreads)
            times.append(time.perf_counter() - t0)
        if len(times) >= max_passes or time.perf_counter() - t_all >= min_seconds:
            break
    px = frames.shape[0] * frames.shape[1] * frames.shape[2]
    return kind, times, px


def sample_frames(wl, every):
    from paper_2412_00058_b200 import synth
    idx = np.arange(0, wl.nframes, every)
    frames = np.empty((len(idx), wl.h, wl.w), np.uint8)
    for i, k in enumerate(idx):
        frames[i] = synth.synth_frames_np(wl, int(k), 1)[0]
    return idx, frames


def _cfg2_frames_host(wl):
    """All cfg2 frames in host memory (the device generator when a GPU is present, else numpy;
    data preparation, outside every timed region)."""
    try:
        import torch
        if torch.cuda.is_available():
            from paper_2412_00058_b200 import synth
            dev = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
            synth.synth_frames_device(wl, dev, 0, wl.nframes)
            out = dev.cpu().numpy()
            del dev
            torch.cuda.empty_cache()
            return out
    except Exception:
        pass
    return wl.frames_np()


def run_reference(args):
    """The reference's CPU path on the bench's own step: all 2400 cfg2 frames inserted by the
    reference's spinevol::pixel_to_world + SPEC insert loop (oracle/_ref, z-slab threads), then
    the 3x3x3 mean fill of the same per-z-chunk dirty boxes and the cfg4 depth-band render of the
    same columns by the C restatement (the reference has no fill / render code), all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2412_00058_b200 import sharding, synth
    wl = synth.cfg2()
    frames = _cfg2_frames_host(wl)
    nth = _ncpu()
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    idx = np.arange(wl.nframes)
    fb = sharding.chunk_boxes(boxes, idx, (0, wl.dims[2]), chunk=32, dilate=wl.fill_radius)
    rb = sharding.chunk_boxes(boxes, idx, (0, wl.dims[2]), chunk=32)
    rp = synth.render_params()
    grid = O.OracleGrid.for_workload(wl)
    kind = "reference" if O.ref() is not None else "port"

    def step():
        t = [time.perf_counter()]
        if kind == "reference":
            O.ref_insert_frames(wl.dims, wl.voxel_mm, wl.origin, frames, wl.poses, wl.calib,
                                nthreads=nth, out=(grid.sum, grid.count))
        else:
            grid.insert_frames_mt(frames, wl.poses, wl.calib, nthreads=nth)
        t.append(time.perf_counter())
        grid.fill_holes_boxes_mt(fb, 0, wl.fill_radius, nthreads=nth)
        t.append(time.perf_counter())
        grid.render_boxes_mt(rp, rb, wl.fill_radius, nthreads=nth)
        t.append(time.perf_counter())
        return t[3] - t[0], (t[1] - t[0], t[2] - t[1], t[3] - t[2])

    step_times, stages = [], []
    for i in range(args.warmup + args.steps):
        tt, st = step()
        if i >= args.warmup:
            step_times.append(tt)
            stages.append(st)
    tot = sum(step_times)
    px = wl.nframes * wl.w * wl.h
    value = px * len(step_times) / tot / 1e9
    sample = ("the whole bench step: all 2400 cfg2 frames (%.0f Mpx) inserted by the reference's "
              "spinevol::pixel_to_world + SPEC insert loop (%s), mean fill r=1 of the %d per-z-chunk "
              "dirty boxes and the cfg4 render of the %d column boxes by the C restatement; %d threads, %s"
              % (px / 1e6, kind, len(fb), len(rb), nth, _cpu_model()))
    stage_ms = {k: 1e3 * sum(st[i] for st in stages) / len(stages) for i, k in enumerate(("insert", "fill", "render"))}
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / len(step_times) * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
           "data": "synthetic (seeded, BASELINE cfg2 generator)",
           "config": {"workload": WORKLOAD, "sample": sample, "same_config": True},
           "stages_ms": stage_ms,
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nth, "kind": kind, "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax = float(p[2])
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}



# ---------------------------------------------------------------- secondary configs (N=1)
def measure_config(name, steps=3):
    """Insert-only throughput of another BASELINE config on this GPU (device-resident frames):
    cfg1 (small linear), cfg3 (convex fan), cfg5 (2x2x2 trilinear f32 splat into the full
    2000x1000x7500 = 15 G-voxel, 120 GB volume)."""
    import torch

    import paper_2412_00058_b200 as pkg
    from paper_2412_00058_b200 import _abi, synth
    wl = synth.CONFIGS[name]()
    vox = int(np.prod(wl.dims))
    need = vox * 8 + wl.nframes * wl.w * wl.h
    free = torch.cuda.mem_get_info()[0]
    if need > free * 0.95:
        return {"skipped": "needs %.1f GB, %.1f GB free" % (need / 1e9, free / 1e9)}
    frames = torch.empty((wl.nframes, wl.h, wl.w), dtype=torch.uint8, device="cuda")
    synth.synth_frames_device(wl, frames, 0, wl.nframes, torch.cuda.current_device())
    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, accum=wl.accum,
                         device=torch.cuda.current_device())
    stream = torch.cuda.Stream()
    grid.set_stream(stream.cuda_stream)
    out = {"workload": wl.name, "frames": wl.nframes, "frame": [wl.h, wl.w], "grid": list(wl.dims),
           "voxel_mm": wl.voxel_mm, "accum": "trilinear-f32" if wl.accum == _abi.ACC_TRILINEAR else "pnn-u32"}
    if wl.accum == _abi.ACC_PNN:
        U = grid.footprint(frames, wl.poses, wl.calib)
        grid.clear()
        alg = float(wl.nframes * wl.w * wl.h + 12 * int(U.sum()))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps + 1)]
    with torch.cuda.stream(stream):
        for i in range(steps + 1):
            ev[i][0].record(stream)
            grid.insert_frames(frames, wl.poses, wl.calib)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev[1:]) / steps
    out["insert_ms"] = ms
    out["value"] = wl.nframes * wl.w * wl.h / (ms / 1e3) / 1e9
    out["unit"] = UNIT
    if wl.accum == _abi.ACC_PNN:
        hbm, _ = _peaks()
        out["roofline_frac"] = alg / (ms / 1e3) / 1e9 / hbm
        out["roofline_kernel"] = ("k_fan_desc + k_fan_tiles + k_pnn_work" if wl.calib.probe == _abi.PROBE_FAN
                                  else "k_tile_desc + k_pnn_tiles + k_pnn_work")
        out["bytes_model"] = "sum_f (W*H + 12*U_f), U_f distinct voxels of frame f"
        out["U_mean"] = float(U.mean())
    else:
        out.update(trilinear_extras(wl, grid, frames, stream, ms))
    grid.close()
    del frames
    torch.cuda.empty_cache()
    return out

def trilinear_extras(wl, grid, frames, stream, insert_ms, nsample=16, nlat=40):
    """cfg5 beside its insert: the roofline over W*H + 16*U8 bytes per frame (U8 = distinct corner
    voxels a frame's 2x2x2 splat touches, counted on a sample of frames), the depth-band render of
    the whole volume's columns, and per-frame insert + render latency."""
    import ctypes as C

    import torch

    from paper_2412_00058_b200 import _abi, sharding, synth
    L = _abi.lib()
    hbm, _ = _peaks()
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    # U8: each sampled frame alone in a scratch volume covering its box, non-zero weights counted
    # on the device
    u8 = []
    live = [k for k in range(wl.nframes) if not boxes[k].empty()]
    for k in np.array(live)[np.linspace(0, len(live) - 1, nsample).astype(int)]:
        b = boxes[int(k)]
        dims = (b.x1 - b.x0 + 1, b.y1 - b.y0 + 1, b.z1 - b.z0 + 1)
        org = tuple(wl.origin[i] + wl.voxel_mm * (b.x0, b.y0, b.z0)[i] for i in range(3))
        import paper_2412_00058_b200 as pkg
        sg = pkg.VoxelGrid(dims, wl.voxel_mm, org, accum=wl.accum, device=torch.cuda.current_device())
        sg.insert_frames(frames[k:k + 1], wl.poses[k:k + 1], wl.calib)
        wt = torch.empty(int(np.prod(dims)), dtype=torch.float32, device="cuda")
        _abi.check(L.svr_read_trilinear(sg.handle, None, None, C.c_void_p(wt.data_ptr())))
        u8.append(int(torch.count_nonzero(wt).item()))
        sg.close()
        del wt
    u8m = float(np.mean(u8))
    alg = wl.nframes * (wl.w * wl.h + 16.0 * u8m)
    out = {"roofline": {"bound": "hbm", "kernel": "k_tri_warp (K1t)", "unit": "GB/s",
                        "achieved": alg / (insert_ms / 1e3) / 1e9, "peak": hbm,
                        "frac": alg / (insert_ms / 1e3) / 1e9 / hbm,
                        "bytes_model": "W*H + 16*U8 per frame (f32 wsum + weight RMW of each distinct "
                                       "corner voxel), U8 mean %.0f over %d sampled frames" % (u8m, nsample)},
           "U8_mean": u8m}
    rp = synth.render_params()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        grid.render_coronal(None, rp, 0)  # warm
        a.record(stream)
        grid.render_coronal(None, rp, 0)
        b.record(stream)
        torch.cuda.synchronize()
    out["render_all_columns_ms"] = a.elapsed_time(b)
    # per-frame: one frame's splat + the render of its dirty columns, as one CUDA-graph replay
    # (svr_frame_step) and call by call
    mid = live[len(live) // 2]

    def frame_lat(graph):
        lat = []
        with torch.cuda.stream(stream):
            for j in range(nlat + 3):
                k = mid + j
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if graph:
                    grid.frame_step(frames[k], wl.poses[k:k + 1], wl.calib, 1, rp)
                else:
                    grid.insert_frames(frames[k:k + 1], wl.poses[k:k + 1], wl.calib)
                    if not boxes[k].empty():
                        grid.render_coronal(boxes[k], rp, 0)
                e1.record(stream)
                e1.synchronize()
                if j >= 3:
                    lat.append(e0.elapsed_time(e1))
        lat.sort()
        return lat

    lat, latc = frame_lat(True), frame_lat(False)
    out["latency_ms"] = {"frames": len(lat), "device_p50": lat[len(lat) // 2],
                         "device_p95": lat[int(0.95 * (len(lat) - 1) + 0.5)], "device_max": lat[-1],
                         "per_call_p50": latc[len(latc) // 2],
                         "what": "one frame: trilinear splat + depth-band render of its dirty columns as "
                                 "one CUDA-graph replay (svr_frame_step); per_call: the same kernels "
                                 "launched call by call"}
    return out


# ---------------------------------------------------------------- our arm
def slab_shares(wl, frames, boxes, rp, stream, dev, ns=(2, 4, 8), steps=3, nlat=60):
    """The N-GPU z-slab split replayed one slab at a time on this single GPU (no second GPU is
    available to this build): for each N, the slab that receives the most frames gets its own
    slab-sized VoxelGrid (owned + ghost planes) and runs (a) the batch step of its share (insert of
    its routed frames, fill of its per-z-chunk boxes, render of its columns) and (b) the per-frame
    incremental path (svr_frame_step) over frames from the middle of its share.  (a) is the N-GPU
    step time before the gather of the coronal rows; (b) is the per-frame insert+render latency a
    rank of an N-GPU run sees.  Nothing of another rank's work runs concurrently, so the GPU
    timing is that rank's alone."""
    import numpy as np
    import torch

    import paper_2412_00058_b200 as pkg
    from paper_2412_00058_b200 import sharding, synth

    fill_r = wl.fill_radius
    ghost = fill_r + synth.CFG4_RENDER["median_radius"]
    nz = wl.dims[2]
    out = {}
    for n in ns:
        slabs = sharding.plan_slabs(nz, n, ghost)
        routed = [sharding.route(boxes, sl.alloc) for sl in slabs]
        r = max(range(n), key=lambda i: len(routed[i]))
        sl, mine = slabs[r], routed[r]
        g = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=dev.index, z_range=sl.alloc)
        g.set_stream(stream.cuda_stream)
        fr = frames[torch.from_numpy(mine).to(dev)].contiguous()
        po = wl.poses[mine]
        fb = sharding.chunk_boxes(boxes, mine, sl.alloc, chunk=32, dilate=fill_r)
        rb = sharding.chunk_boxes(boxes, mine, sl.alloc, chunk=32)
        with torch.cuda.stream(stream):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for i in range(steps + 2):
                if i == 2:
                    ev[0].record(stream)
                g.insert_frames(fr, po, wl.calib)
                g.fill_holes_boxes(fb, fill_r, pkg.FILL_MEAN, count=False)
                g.render_coronal_boxes(rb, rp, fill_r)
            ev[1].record(stream)
            torch.cuda.synchronize()
            step_ms = ev[0].elapsed_time(ev[1]) / steps
            g.clear()
            k0 = max(0, len(mine) // 2 - nlat // 2)
            lat = []
            for j in range(-3, min(nlat, len(mine) - k0)):
                k = k0 + max(j, 0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g.frame_step(fr[k], po[k:k + 1], wl.calib, fill_r, rp)
                b.record(stream)
                stream.synchronize()
                if j >= 0:
                    lat.append(a.elapsed_time(b))
        g.close()
        del fr
        lat.sort()
        out[str(n)] = {"slab": r, "planes_stored": sl.alloc[1] - sl.alloc[0],
                       "frames": int(len(mine)), "step_ms": step_ms,
                       "step_gpx_s_job": wl.nframes * wl.w * wl.h / (step_ms / 1e3) / 1e9,
                       "frame_p50_ms": lat[len(lat) // 2] if lat else None,
                       "frame_p95_ms": lat[int(0.95 * (len(lat) - 1) + 0.5)] if lat else None}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2412_00058_b200 as pkg
    from paper_2412_00058_b200 import _abi, sharding, synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.fused_gather_1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    wl = synth.cfg2()
    fill_r, med_r = wl.fill_radius, synth.CFG4_RENDER["median_radius"]
    ghost = fill_r + med_r
    nz = wl.dims[2]
    slabs = sharding.plan_slabs(nz, world, ghost)
    own, alloc = slabs[rank].owned, slabs[rank].alloc
    ob = [s_.owned[0] for s_ in slabs]
    oe = [s_.owned[1] for s_ in slabs]

    # frame routing: every frame whose conservative box meets this rank's stored slab
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    mine = sharding.route(boxes, alloc)
    poses = wl.poses[mine]
    union = sharding.union_box(boxes, mine, alloc)
    # the batch's dirty region as per-z-chunk boxes (tighter than one bounding box for a
    # laterally drifting sweep; identical fill/render results, tested)
    fill_boxes = sharding.chunk_boxes(boxes, mine, alloc, chunk=32, dilate=fill_r)
    render_boxes = sharding.chunk_boxes(boxes, mine, alloc, chunk=32)
    rp = synth.render_params()

    # device-resident frames from the seeded generator (only this rank's frames)
    frames = torch.empty((len(mine), wl.h, wl.w), dtype=torch.uint8, device=dev)
    if len(mine):
        k0, k1 = int(mine[0]), int(mine[-1]) + 1
        span = torch.empty((k1 - k0, wl.h, wl.w), dtype=torch.uint8, device=dev)
        synth.synth_frames_device(wl, span, k0, k1 - k0, local)
        frames = span[torch.from_numpy(mine - k0).to(dev)].contiguous() if len(mine) != k1 - k0 else span
        del span
    n_my = frames.shape[0]
    px_frame = wl.w * wl.h
    total_px = wl.nframes * px_frame  # units of the whole job

    grid = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=local, z_range=alloc)
    stream = torch.cuda.Stream(device=dev)
    grid.set_stream(stream.cuda_stream)

    # algorithmic bytes of the insert launch: sum_f (W*H + U_f * 12)
    U = grid.footprint(frames, poses, wl.calib) if n_my else np.zeros(1, np.int64)
    alg_bytes = float(n_my * px_frame + 12 * int(U.sum()))
    grid.clear()

    rows = own[1] - own[0]
    rows_max = max(oe[r] - ob[r] for r in range(world))
    gath_src = torch.zeros((2, rows_max, wl.dims[0]), dtype=torch.float32, device=dev)
    fused_try = (world > 1 or args.fused_gather_1) and not args.nccl_gather
    gath_dst = torch.zeros((world, 2, rows_max, wl.dims[0]), dtype=torch.float32, device=dev) \
        if world > 1 or fused_try else None

    # Fused render + gather: with symmetric memory (NVLink / NVSwitch peer mappings) every rank's
    # band kernel stores its owned rows straight into all ranks' full images and a device-side
    # barrier replaces the all-gather.  Verified once against the NCCL gather; falls back to it.
    gather_mode, gather_note, symm_h, full_img = "nccl", "", None, None
    if fused_try:
        try:
            import torch.distributed._symmetric_memory as symm
            full_img = symm.empty((2, nz, wl.dims[0]), dtype=torch.float32, device=dev)
            full_img.zero_()
            symm_h = symm.rendezvous(full_img, dist.group.WORLD)
            grid.set_gather_targets([int(p) for p in symm_h.buffer_ptrs], own)
            gather_mode = "fused-p2p"
        except Exception as e:  # no P2P / symmetric memory: NCCL gather
            gather_note = "symmetric memory unavailable: %s" % str(e).splitlines()[0][:160]
            symm_h = None

    def gather():
        if gather_mode == "fused-p2p":
            symm_h.barrier(0)
        elif world > 1:
            grid.read_coronal_into(own[0], own[1] - 1, gath_src[0], gath_src[1])
            dist.all_gather_into_tensor(gath_dst, gath_src)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.warmup + args.steps)]

    def step_seq(i):  # insert all, fill all, render all: the stage breakdown
        e = ev[i]
        e[0].record(stream)
        grid.insert_frames(frames, poses, wl.calib)
        e[1].record(stream)
        grid.fill_holes_boxes(fill_boxes, fill_r, pkg.FILL_MEAN, count=False)
        e[2].record(stream)
        grid.render_coronal_boxes(render_boxes, rp, fill_r)
        e[3].record(stream)
        gather()

    # --sweep-groups > 1: the same work with the fill / render of every finished z-chunk on a
    # second (high-priority) stream while later frames are inserted (sharding.reconstruct_sweep;
    # identical results, tests/test_gpu_parity.py::test_reconstruct_sweep_equals_sequential)
    sched = sharding.sweep_schedule(boxes, mine, fill_boxes, render_boxes, groups=args.sweep_groups)
    aux = torch.cuda.Stream(device=dev, priority=-1)
    sweep_ev = [torch.cuda.Event() for _ in sched]

    def step(i):
        if args.sweep_groups <= 1:
            step_seq(i)
            return
        sharding.reconstruct_sweep(grid, frames, poses, wl.calib, sched, rp, fill_r,
                                   insert_stream=stream, aux_stream=aux, events=sweep_ev)
        gather()

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        if gather_mode == "fused-p2p":
            # one NCCL gather of the same strips: the fused image must equal it exactly
            grid.read_coronal_into(own[0], own[1] - 1, gath_src[0], gath_src[1])
            dist.all_gather_into_tensor(gath_dst, gath_src)
            torch.cuda.synchronize()
            ok = True
            for r in range(world):
                o0, o1 = ob[r], oe[r]
                ok = ok and torch.equal(gath_dst[r, :, :o1 - o0], full_img[:, o0:o1])
            okt = torch.tensor([1 if ok else 0], device=dev)
            dist.all_reduce(okt, op=dist.ReduceOp.MIN)
            if int(okt.item()) != 1:
                grid.set_gather_targets([])
                gather_mode, gather_note = "nccl", "fused gather mismatched the NCCL gather; fell back"
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        launches0 = grid.stats()["kernel_launches"]
        clocks = Clocks(local)
        clocks.start()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.warmup, args.warmup + args.steps):
            step(i)
        t1.record(stream)
        torch.cuda.synchronize()
        clk = clocks.stop()
        barrier()
        launches = grid.stats()["kernel_launches"] - launches0
        elapsed_ms = allmax(t0.elapsed_time(t1))
        # stage breakdown (and K1's time for the roofline) from the sequential schedule: the timed
        # steps' own events, or (overlapped sweep) a few extra sequential steps
        if args.sweep_groups <= 1:
            ns = args.steps
            timed = ev[args.warmup:args.warmup + ns]
        else:
            ns = 3
            step_seq(0)  # untimed: the first whole-batch insert after group inserts regrows buffers
            torch.cuda.synchronize()
            for i in range(ns):
                step_seq(i)
            torch.cuda.synchronize()
            timed = ev[:ns]
        ins_ms = allmax(sum(e[0].elapsed_time(e[1]) for e in timed) / ns)
        fill_ms = allmax(sum(e[1].elapsed_time(e[2]) for e in timed) / ns)
        rend_ms = allmax(sum(e[2].elapsed_time(e[3]) for e in timed) / ns)
        seq_ms = allmax(sum(e[0].elapsed_time(e[3]) for e in timed) / ns)

        # ---- e2e through the public API from pinned host frames
        frames_host = frames.cpu().pin_memory()
        mean_h = torch.empty((rows, wl.dims[0]), dtype=torch.float32).pin_memory()
        max_h = torch.empty_like(mean_h).pin_memory()
        e2e_steps = max(1, min(args.steps, 5))

        def e2e_step():
            grid.insert_frames(frames_host, poses, wl.calib)
            grid.fill_holes_boxes(fill_boxes, fill_r, pkg.FILL_MEAN, count=False)
            grid.render_coronal_boxes(render_boxes, rp, fill_r)
            gather()
            # the step's result read back into pinned host buffers, enqueued behind the render so
            # the next step's H2D staging overlaps this step's fill / render / read-back
            grid.read_coronal_into(own[0], own[1] - 1, mean_h, max_h, wait=False)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        w0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = allmax(time.perf_counter() - w0)
        h2d = n_my * px_frame + n_my * 224
        d2h = 2 * rows * wl.dims[0] * 4
        # the host link's own ceiling: the same pinned frames copied alone (best of 2, CUDA events)
        link_ms = []
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            frames.copy_(frames_host, non_blocking=True)  # identical bytes: frames_host = frames
            b.record(stream)
            b.synchronize()
            link_ms.append(a.elapsed_time(b))
        link_gbs = frames_host.numel() / (min(link_ms) * 1e-3) / 1e9 if n_my else None

        # ---- per-frame incremental latency (insert -> fill(box+1) -> render(box)), rank-local:
        # the product path is svr_frame_step (one CUDA-graph replay per frame); the per-call
        # sequence of the same kernels is timed beside it
        def frame_latency(nl, first, graph, src=None):
            le = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nl)]
            wall = []
            for j in range(nl):
                k = first + j
                torch.cuda.synchronize()
                w = time.perf_counter()
                le[j][0].record(stream)
                if graph:
                    grid.frame_step((frames if src is None else src)[k], poses[k:k + 1], wl.calib, fill_r, rp)
                else:
                    grid.insert_frames(frames[k], poses[k:k + 1], wl.calib)
                    b = boxes[int(mine[k])]
                    grid.fill_holes(pkg.dilate(b, fill_r), fill_r, pkg.FILL_MEAN, count=False)
                    grid.render_coronal(b, rp, fill_r)
                le[j][1].record(stream)
                stream.synchronize()
                wall.append((time.perf_counter() - w) * 1e3)
            torch.cuda.synchronize()
            return [a.elapsed_time(b) for a, b in le], wall

        nl = min(args.latency_frames, max(n_my - 4, 0))
        mid = max(0, n_my // 2 - nl // 2)
        lat_dev, lat_wall = [], []
        lat_dev_c, lat_wall_c = [], []
        lat_dev_h, lat_wall_h = [], []
        cap0 = grid.stats()["graph_captures"]
        if nl:
            frame_latency(3, max(mid - 3, 0), True)  # graph capture + warm-up, untimed
            cap0 = grid.stats()["graph_captures"]
            lat_dev, lat_wall = frame_latency(nl, mid, True)
            lat_dev_c, lat_wall_c = frame_latency(nl, mid, False)
            # the real system's frame arrives in pinned host memory: its H2D is inside the step
            lat_dev_h, lat_wall_h = frame_latency(nl, mid, True, frames_host)
        recaptures = grid.stats()["graph_captures"] - cap0
        if world > 1:  # every rank's frames: the union's percentiles, max over ranks
            allv = [None] * world
            dist.all_gather_object(allv, (lat_dev, lat_wall, lat_dev_c, lat_wall_c, lat_dev_h, lat_wall_h, recaptures))
            lat_dev, lat_wall, lat_dev_c, lat_wall_c, lat_dev_h, lat_wall_h = (
                sum((a[i] for a in allv), []) for i in range(6))
            recaptures = sum(a[6] for a in allv)

    stats = grid.stats()
    hbm, peak_src = _peaks()
    ins_s = max(ins_ms, 1e-9) / 1e3
    achieved = alg_bytes / ins_s / 1e9
    value = total_px * args.steps / (elapsed_ms / 1e3) / 1e9
    e2e_value = total_px * e2e_steps / e2e_s / 1e9

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:  # beside every N
        idx, cf = sample_frames(wl, args.cpu_every)
        nth = _ncpu()
        kind, times, px = cpu_reference(wl, cf, wl.poses[idx], nth, min_seconds=args.cpu_seconds,
                                        max_passes=50)
        cpu = {"value": px * len(times) / sum(times) / 1e9, "unit": UNIT, "cores": nth, "kind": kind,
               "sample": "%d of 2400 cfg2 frames (every %dth, %.1f Mpx) x %d passes, PNN insert only, "
                         "%d threads, %s" % (len(idx), args.cpu_every, px / 1e6, len(times), nth,
                                             _cpu_model())}

    shares = None
    if rank == 0 and world == 1 and not args.no_slab_shares:
        shares = {"what": "N-GPU z-slab split replayed one slab at a time on this GPU: the busiest "
                          "slab's batch step (before the coronal-row gather) and its per-frame "
                          "latency (svr_frame_step p50/p95); step_gpx_s_job = whole-job pixels / "
                          "that slab's step time",
                  "n": slab_shares(wl, frames, boxes, rp, stream, dev)}

    others = None
    if rank == 0 and world == 1 and not args.no_other_configs:
        grid.close()
        del frames
        torch.cuda.empty_cache()
        others = {}
        for name in ("cfg1", "cfg3", "cfg5"):
            try:
                others[name] = measure_config(name)
            except Exception as e:  # report, never hide the headline line
                others[name] = {"error": str(e)[:200]}

    def pct(v, p):
        s = sorted(v)
        return s[int(p * (len(s) - 1) + 0.5)] if s else None

    traffic, atomics = None, None
    tf = os.path.join(ROOT, "profiles", "insert_traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                nc = json.load(f)
            traffic = nc.get("dram_bytes_per_launch")
            # atomic throughput of K1 (north_star): ncu counts per launch over the live launch time
            if nc.get("l2_red_requests_per_launch"):
                atomics = {
                    "source": "ncu counts per launch (profiles/insert_traffic.json) / live K1 time",
                    "l2_red_requests_per_s": nc["l2_red_requests_per_launch"] / ins_s,
                    "l2_red_sectors_per_s": nc["l2_red_sectors_per_launch"] / ins_s,
                    "l2_red_sector_hit_rate": nc.get("l2_red_sector_hit_rate"),
                    "smem_atom_wavefronts_per_s": nc["smem_atom_wavefronts_per_launch"] / ins_s,
                    "smem_atom_per_pixel": 1.0,
                }
        except Exception:
            traffic, atomics = None, None
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded Rayleigh speckle + vertebra arcs, BASELINE cfg2 generator)",
        "config": {"workload": WORKLOAD, "frames": wl.nframes, "frame": [wl.h, wl.w],
                   "grid": list(wl.dims), "voxel_mm": wl.voxel_mm, "parallelism": "z-slab x%d" % world,
                   "gather": gather_mode if world > 1 or fused_try else None, "gather_note": gather_note or None,
                   "l2": "no flush: frames (590 MB) and volume (2.1 GB) exceed the 126 MB L2",
                   "frames_this_rank": int(n_my)},
        "stages_ms": {"insert": ins_ms, "fill": fill_ms, "render": rend_ms, "sequential_step": seq_ms,
                      "what": "insert-all / fill-all / render-all schedule, CUDA events per stage "
                              "(timed step: %d frame group(s))" % args.sweep_groups},
        "insert_only": {"value": total_px / ins_s / 1e9 if world == 1 else None, "unit": UNIT},
        "roofline": {"bound": "hbm", "kernel": "k_tile_desc + k_pnn_tiles + k_pnn_work (K1)", "achieved": achieved, "peak": hbm,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_model": "sum_f (W*H + 12*U_f), U_f distinct voxels of frame f (mean %.0f)"
                                    % float(U.mean()),
                     "atomics": atomics},
        "latency_ms": {"frames": nl, "device_p50": pct(lat_dev, 0.5), "device_p95": pct(lat_dev, 0.95),
                       "device_max": max(lat_dev) if lat_dev else None, "wall_p50": pct(lat_wall, 0.5),
                       "wall_p95": pct(lat_wall, 0.95), "wall_max": max(lat_wall) if lat_wall else None,
                       "what": "one frame: insert + fill(conservative box+1) + render(box) as one CUDA-graph "
                               "replay (svr_frame_step) from a device-resident frame; at N > 1 every "
                               "rank's frames (percentiles over their union), the render storing its "
                               "owned rows into every rank's image (fused gather)",
                       "graph_recaptures": int(recaptures),
                       "pinned_host": {"device_p50": pct(lat_dev_h, 0.5), "device_p95": pct(lat_dev_h, 0.95),
                                       "device_max": max(lat_dev_h) if lat_dev_h else None,
                                       "wall_p50": pct(lat_wall_h, 0.5), "wall_p95": pct(lat_wall_h, 0.95),
                                       "what": "the same step from a pinned host frame: its 240 KB H2D "
                                               "copy enqueued ahead of the graph, inside the timing"},
                       "per_call": {"device_p50": pct(lat_dev_c, 0.5), "device_p95": pct(lat_dev_c, 0.95),
                                    "wall_p50": pct(lat_wall_c, 0.5),
                                    "what": "the same kernels launched call by call"}},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "link": {"h2d_gbs_achieved": h2d * e2e_steps / e2e_s / 1e9,
                         "h2d_gbs_copy_alone": link_gbs,
                         "frac": (h2d * e2e_steps / e2e_s / 1e9) / link_gbs if link_gbs else None,
                         "what": "e2e H2D bytes / e2e time vs the same pinned frames copied alone"}},
        "gpu_launches": int(launches),
        "clocks": clk,
        "cpu_baseline": cpu,
        "exact_fallbacks_per_frame": stats["exact_fallbacks"] / max(stats["frames_inserted"], 1),
        "other_configs": others,
        "slab_shares": shares,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if others is None:
        grid.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-every", type=int, default=10, help="reference arm: frame sample stride")
    ap.add_argument("--cpu-every", type=int, default=8, help="cpu_baseline frame sample stride")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--latency-frames", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip cfg1/cfg3/cfg5 lines")
    ap.add_argument("--no-slab-shares", action="store_true", help="skip the N = 2/4/8 slab-share replay")
    ap.add_argument("--sweep-groups", type=int, default=1,
                    help="frame groups of the overlapped insert / fill / render schedule (1 = sequential; "
                         "4 / 8 measured slower: K1 is issue-bound, the overlap only adds launches)")
    ap.add_argument("--nccl-gather", action="store_true",
                    help="N>1: gather the coronal strips with NCCL instead of the fused peer stores")
    ap.add_argument("--fused-gather-1", action="store_true",
                    help="exercise the fused peer-store gather (symmetric memory + device barrier) at N=1 too")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world is None:
        return spawn_ranks(args.gpus)
    if world is not None and int(world) != args.gpus:
        print(json.dumps({"error": "--gpus %d but WORLD_SIZE=%s" % (args.gpus, world)}), flush=True)
        return 2
    return run_ours(args)


def spawn_ranks(n):
    """`bench.py --gpus N` without a launcher: re-exec under torch.distributed.run with one rank
    per GPU on this node (rendezvous on 127.0.0.1), failing loudly when fewer GPUs are visible."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"error": "--gpus %d but only %d CUDA device(s) visible" % (n, have)}), flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    # NCCL's communicator init lines (nranks per communicator) stay visible, on stderr
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    sys.exit(main())
