"""GPU: the z-slab sharded volume of the C-ABI (svr_sharded_*) against one
unsharded volume, bit for bit: owned-plane accumulators, and the coronal image gathered by the
slabs' own render kernels (fused peer stores; here all slabs share device 0, the host-side
routing, ghost planes and gather addressing are the same as across devices)."""
import numpy as np
import pytest

import paper_2412_00058_b200 as pkg
from paper_2412_00058_b200 import sharding, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nslab", [1, 2, 3, 5])
def test_sharded_equals_unsharded(nslab):
    wl = synth.cfg1()
    frames = wl.frames_np()
    rp = synth.render_params()
    ghost = wl.fill_radius + rp.median_radius
    one = pkg.VoxelGrid(wl.dims, wl.voxel_mm, wl.origin, device=0)
    _, u = one.insert_frames(frames, wl.poses, wl.calib, want_boxes=True)
    one.fill_holes(pkg.dilate(u, 1), 1, pkg.FILL_MEAN)
    one.render_coronal(u, rp, 1)  # the dirty columns, as the slabs render theirs
    s1, c1 = one.accumulators()
    m1, x1, d1 = one.read_coronal()
    sh = sharding.ShardedGrid(wl.dims, wl.voxel_mm, wl.origin, devices=[0] * nslab, ghost=ghost)
    routed = sh.insert_frames(frames, wl.poses, wl.calib)
    assert sum(routed) >= wl.nframes  # (frames near a slab face go to both slabs)
    sh.fill_render(1, pkg.FILL_MEAN, rp)
    for r in range(nslab):
        _, own, _ = sh.slab(r)
        s, c = sh.accumulators(r)
        assert np.array_equal(c, c1[own[0]:own[1]]) and np.array_equal(s, s1[own[0]:own[1]]), r
    m, x, d = sh.read_coronal()
    assert np.array_equal(d, d1)
    assert np.array_equal(m, m1) and np.array_equal(x, x1)
    assert (m > 0).sum() > 1000
    sh.close()
    one.close()
