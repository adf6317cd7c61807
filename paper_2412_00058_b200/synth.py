"""Seeded synthetic workloads restating BASELINE.json `configs` (no public dataset exists).

Each config yields: a calibration (ImageCalibration, geometry.hpp:160-176), a grid
(VoxelGrid), tracked poses (transducer -> world) and B-scan frames.  Poses
come from numpy (host), frames from numpy for small parity cases or from the device
generator `svr_synth_frames` for the full-size bench; both draw Rayleigh speckle from a
SplitMix64 hash (core.hpp:64-91 constants) so a frame is a pure function of (seed, frame, px).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def quat_axis_angle(axis, angle_rad):
    """Quat::from_axis_angle (geometry.hpp:17-23)."""
    ax = np.asarray(axis, dtype=np.float64)
    n = math.sqrt(float(ax @ ax))
    h = 0.5 * angle_rad
    s = math.sin(h) / n
    return np.array([math.cos(h), ax[0] * s, ax[1] * s, ax[2] * s])


def quat_mul(a, b):
    """Quat::operator* (geometry.hpp:35-40)."""
    w, x, y, z = a
    return np.array([w * b[0] - x * b[1] - y * b[2] - z * b[3],
                     w * b[1] + x * b[0] + y * b[3] - z * b[2],
                     w * b[2] - x * b[3] + y * b[0] + z * b[1],
                     w * b[3] + x * b[2] - y * b[1] + z * b[0]])


def quat_normalized(q):
    return q / math.sqrt(float(q @ q))


def rigid(q=(1.0, 0.0, 0.0, 0.0), t=(0.0, 0.0, 0.0)) -> _abi.Rigid:
    return _abi.Rigid(*[float(v) for v in q], *[float(v) for v in t])


def linear_calib(w, h, sx, sy, i2t=None) -> _abi.Calib:
    c = _abi.Calib()
    c.crop_w, c.crop_h = int(w), int(h)
    c.scale_x_mm, c.scale_y_mm = float(sx), float(sy)
    c.image_to_transducer = i2t if i2t is not None else rigid()
    c.probe = _abi.PROBE_LINEAR
    return c


def fan_calib(lines, samples, angle_deg, r0, r1, i2t=None) -> _abi.Calib:
    c = _abi.Calib()
    c.crop_w, c.crop_h = int(samples), int(lines)
    c.scale_x_mm = c.scale_y_mm = 1.0
    c.image_to_transducer = i2t if i2t is not None else rigid()
    c.probe = _abi.PROBE_FAN
    c.fan_angle_deg, c.fan_r0_mm, c.fan_r1_mm = float(angle_deg), float(r0), float(r1)
    return c


@dataclass
class Workload:
    name: str
    calib: _abi.Calib
    dims: tuple            # (nx, ny, nz)
    voxel_mm: float
    origin: tuple
    poses: np.ndarray      # RIGID_DTYPE, one per frame
    kind: int              # synth generator kind (0 linear speckle+arcs, 1 fan)
    seed: int
    fill_mode: int = _abi.FILL_MEAN
    fill_radius: int = 1
    accum: int = _abi.ACC_PNN
    extra: dict = field(default_factory=dict)

    @property
    def w(self):
        return self.calib.crop_w

    @property
    def h(self):
        return self.calib.crop_h

    @property
    def nframes(self):
        return len(self.poses)

    def grid_desc(self, z_begin=0, z_end=None) -> _abi.GridDesc:
        g = _abi.GridDesc()
        g.nx, g.ny, g.nz = self.dims
        g.accum = self.accum
        g.voxel_mm = self.voxel_mm
        for k in range(3):
            g.origin_mm[k] = self.origin[k]
        g.z_begin = z_begin
        g.z_end = self.dims[2] if z_end is None else z_end
        return g

    def frames_np(self, first=0, n=None) -> np.ndarray:
        n = self.nframes - first if n is None else n
        return synth_frames_np(self, first, n)


def _jitter_rot(rng, deg):
    a, b, c = (math.radians(rng.uniform(-deg, deg)) for _ in range(3))
    q = quat_mul(quat_axis_angle((0, 0, 1), c),
                 quat_mul(quat_axis_angle((0, 1, 0), b), quat_axis_angle((1, 0, 0), a)))
    return quat_normalized(q)


def _poses(n, fn, seed):
    rng = np.random.default_rng(seed)
    out = np.zeros(n, dtype=_abi.RIGID_DTYPE)
    for k in range(n):
        q, t = fn(k, rng)
        out[k] = (*q, *t)
    return out


def cfg1(seed=1, nframes=200) -> Workload:
    """BASELINE cfg1: 200 x 256x256 u8, 0.2 mm px, z sweep 0.5 mm/frame, +-3 deg, +-1 mm,
    grid 128x128x256 @ 0.5 mm, nearest insert + 3x3x3 mean fill."""
    calib = linear_calib(256, 256, 0.2, 0.2, rigid(t=(-25.6, 0.0, 0.0)))

    def f(k, rng):
        q = _jitter_rot(rng, 3.0)
        t = (32.0 + rng.uniform(-1, 1), 4.0 + rng.uniform(-1, 1), 10.0 + 0.5 * k + rng.uniform(-1, 1))
        return q, t
    return Workload("cfg1", calib, (128, 128, 256), 0.5, (0.0, 0.0, 0.0), _poses(nframes, f, seed),
                    0, seed)


def cfg2(seed=2, nframes=2400) -> Workload:
    """BASELINE cfg2: 2400 x 512x480 u8 (40 x 60 mm), 550 mm sweep, +-15 mm sinusoidal drift
    (period 200 mm), +-5 deg jitter; grid 500x267x2000 @ 0.3 mm; incremental dirty-box fill."""
    calib = linear_calib(512, 480, 40.0 / 512, 60.0 / 480, rigid(t=(-20.0, 0.0, 0.0)))
    span = 550.0

    def f(k, rng):
        z = 25.0 + span * k / max(nframes - 1, 1)
        q = _jitter_rot(rng, 5.0)
        t = (75.0 + 15.0 * math.sin(2 * math.pi * z / 200.0), 5.0, z)
        return q, t
    return Workload("cfg2", calib, (500, 267, 2000), 0.3, (0.0, 0.0, 0.0),
                    _poses(nframes, f, seed), 0, seed)


def cfg3(seed=3, nframes=1800) -> Workload:
    """BASELINE cfg3: 1800 polar frames, 192 lines x 1024 samples, 60 deg fan, r 20-150 mm,
    500 mm path as cfg2; 0.4 mm grid over the fan envelope."""
    calib = fan_calib(192, 1024, 60.0, 20.0, 150.0)
    span = 500.0

    def f(k, rng):
        z = 15.0 + span * k / max(nframes - 1, 1)
        q = _jitter_rot(rng, 5.0)
        t = (95.0 + 15.0 * math.sin(2 * math.pi * z / 200.0), 2.0, z)
        return q, t
    return Workload("cfg3", calib, (475, 400, 1325), 0.4, (0.0, 0.0, 0.0),
                    _poses(nframes, f, seed), 1, seed)


def cfg5(seed=5, nframes=4800, dims=(2000, 1000, 7500)) -> Workload:
    """BASELINE cfg5: 4800 cfg2 frames at 0.125 mm/frame into a 0.08 mm f32 trilinear volume
    (2000x1000x7500 = 15 G voxels, 120 GB).  `dims` may be reduced for parity tests."""
    calib = linear_calib(512, 480, 40.0 / 512, 60.0 / 480, rigid(t=(-20.0, 0.0, 0.0)))

    def f(k, rng):
        z = 10.0 + 0.125 * k
        q = _jitter_rot(rng, 5.0)
        t = (80.0 + 15.0 * math.sin(2 * math.pi * z / 200.0), 5.0, z)
        return q, t
    wl = Workload("cfg5", calib, tuple(dims), 0.08, (0.0, 0.0, 0.0), _poses(nframes, f, seed), 0,
                  seed, accum=_abi.ACC_TRILINEAR)
    return wl


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg5": cfg5}

# cfg4: depth-band render of the filled cfg2 volume (BASELINE cfg4)
CFG4_RENDER = dict(depth_lo_mm=15.0, depth_hi_mm=60.0, band_above_mm=5.0, band_below_mm=2.0,
                   median_radius=2)


def render_params(fill_mode=_abi.FILL_MEAN, **kw) -> _abi.RenderParams:
    d = dict(CFG4_RENDER)
    d.update(kw)
    p = _abi.RenderParams()
    for k, v in d.items():
        setattr(p, k, v)
    p.fill_mode = fill_mode
    return p


def synth_frames_np(wl: Workload, first: int, n: int) -> np.ndarray:
    """Host generator (same model as the device kernel k_synth): returns (n, h, w) u8."""
    w, h = wl.w, wl.h
    out = np.empty((n, h, w), dtype=np.uint8)
    idx = np.arange(w * h, dtype=np.uint64)
    col = (idx % np.uint64(w)).astype(np.float64)
    row = (idx // np.uint64(w)).astype(np.float64)
    c = wl.calib
    for f in range(n):
        k = first + f
        hsh = _splitmix(np.uint64(wl.seed) ^ _splitmix(np.uint64(k) * np.uint64(0x100000001B3) + idx))
        u = (hsh >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        ray = np.sqrt(-2.0 * np.log1p(-u))
        bright = 200 + ((hsh >> np.uint64(3)) % np.uint64(56)).astype(np.int64)
        if wl.kind == 0:
            sweep = float(wl.poses[k]["tz"])
            ph = sweep / 25.0 - math.floor(sweep / 25.0)
            arc_mm = 30.0 - 10.0 * math.cos(2 * math.pi * ph)
            xm, ym = col * c.scale_x_mm, row * c.scale_y_mm
            half = 0.5 * w * c.scale_x_mm
            d = ym - (arc_mm + 0.012 * (xm - half) ** 2)
            v = np.where(np.abs(d) <= 1.5 * c.scale_y_mm, bright,
                         (ray * np.where(d > 0, 14.0, 40.0)).astype(np.int64))
        else:
            dr = (c.fan_r1_mm - c.fan_r0_mm) / w
            r = c.fan_r0_mm + (col + 0.5) * dr
            v = np.where((r >= 60.0) & (r <= 80.0), bright, (48.0 * np.log1p(3.0 * ray)).astype(np.int64))
        out[f] = np.minimum(v, 255).astype(np.uint8).reshape(h, w)
    return out


def small_linear(seed=11, nframes=12, w=64, h=48, dims=(48, 40, 40), voxel=0.5, jitter_deg=8.0):
    """Tiny ragged-friendly linear workload for fast parity tests and golden fixtures."""
    calib = linear_calib(w, h, 0.3, 0.35, rigid(quat_normalized(np.array([1.0, 0.02, -0.03, 0.05])),
                                               (-0.5 * w * 0.3, 0.4, -0.2)))

    def f(k, rng):
        q = _jitter_rot(rng, jitter_deg)
        t = (0.5 * dims[0] * voxel + rng.uniform(-1, 1), 1.0 + rng.uniform(-0.5, 0.5),
             4.0 + 0.6 * k + rng.uniform(-0.5, 0.5))
        return q, t
    return Workload("small_linear", calib, dims, voxel, (0.1, -0.2, 0.3), _poses(nframes, f, seed), 0,
                    seed)


def small_fan(seed=13, nframes=8, lines=24, samples=96, dims=(64, 56, 40), voxel=0.6):
    calib = fan_calib(lines, samples, 60.0, 5.0, 30.0, rigid(t=(0.0, 0.5, 0.0)))

    def f(k, rng):
        q = _jitter_rot(rng, 6.0)
        t = (0.5 * dims[0] * voxel, 1.0, 5.0 + 0.8 * k)
        return q, t
    return Workload("small_fan", calib, dims, voxel, (0.0, 0.0, 0.0), _poses(nframes, f, seed), 1, seed)


def synth_frames_device(wl: Workload, dst, first: int, n: int, device: int = 0, stream=None):
    """Fill `dst` (device u8 tensor / pointer, n x h x w) with frames [first, first+n) from the
    device generator svr_synth_frames (same model as synth_frames_np)."""
    base = dst.data_ptr() if hasattr(dst, "data_ptr") else int(dst)
    fb = wl.w * wl.h
    for a in range(0, n, 4096):
        m = min(4096, n - a)
        _abi.check(_abi.lib().svr_synth_frames(
            base + a * fb, wl.w, wl.h, first + a, m, wl.calib,
            _abi.rigid_ptr(np.ascontiguousarray(wl.poses[first + a:first + a + m])), wl.kind, wl.seed,
            device, stream))
