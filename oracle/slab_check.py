"""Multi-rank slab-sharding check on the CPU (TEST INFRASTRUCTURE ONLY).

Each rank runs the oracle on its stored slab with the product's host-side sharding logic
(paper_2412_00058_b200.sharding: slab plan, frame routing, union box, gather) over gloo; rank 0
compares the gathered owned planes and coronal rows with the unsharded oracle.
"""
import os
import sys

import numpy as np


def worker(rank, world, port, out_path):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2412_00058_b200 import dilate, sharding, synth

    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    wl = synth.small_linear(nframes=16, dims=(48, 40, 60))
    frames = wl.frames_np()
    rp = synth.render_params(depth_lo_mm=1.0, depth_hi_mm=12.0, band_above_mm=1.0, band_below_mm=0.5)
    ghost = wl.fill_radius + rp.median_radius
    slabs = sharding.plan_slabs(wl.dims[2], world, ghost)
    me = slabs[rank]
    boxes = sharding.frame_boxes(wl.grid_desc(), wl.calib, wl.poses)
    idx = sharding.route(boxes, me.alloc)
    g = O.OracleGrid(wl.dims, wl.voxel_mm, wl.origin, z_range=me.alloc)
    for k in idx:
        g.insert_frame(frames[k], wl.poses[k:k + 1], wl.calib)
    u = sharding.union_box(boxes, idx, me.alloc)
    if not u.empty():
        g.fill_holes(dilate(u, wl.fill_radius), 0, wl.fill_radius)
    g.render(rp)
    o0, o1 = me.owned[0] - me.alloc[0], me.owned[1] - me.alloc[0]
    img = torch.from_numpy(np.stack([g.mean[o0:o1], g.max[o0:o1], g.mdepth[o0:o1].astype(np.float32)], 1))
    acc = torch.from_numpy(np.stack([g.sum[o0:o1].astype(np.int64), g.count[o0:o1].astype(np.int64),
                                     g.fill[o0:o1].astype(np.int64)], 1))
    full_img = sharding.gather_rows(img, me, slabs, dist)
    full_acc = sharding.gather_rows(acc, me, slabs, dist)
    if rank == 0:
        ref = O.OracleGrid(wl.dims, wl.voxel_mm, wl.origin)
        ref.insert_frames(frames, wl.poses, wl.calib)
        ub = sharding.union_box(boxes, np.arange(wl.nframes), (0, wl.dims[2]))
        ref.fill_holes(dilate(ub, wl.fill_radius), 0, wl.fill_radius)
        ref.render(rp)
        ok = (np.array_equal(full_acc[:, 0].numpy(), ref.sum.astype(np.int64)) and
              np.array_equal(full_acc[:, 1].numpy(), ref.count.astype(np.int64)) and
              np.array_equal(full_acc[:, 2].numpy(), ref.fill.astype(np.int64)) and
              np.array_equal(full_img[:, 0].numpy(), ref.mean) and
              np.array_equal(full_img[:, 1].numpy(), ref.max) and
              np.array_equal(full_img[:, 2].numpy(), ref.mdepth.astype(np.float32)))
        routed = [len(sharding.route(boxes, s.alloc)) for s in slabs]
        with open(out_path, "w") as f:
            f.write("ok %s" % routed if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()
