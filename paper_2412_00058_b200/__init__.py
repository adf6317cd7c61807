"""spinevol-b200: B200-native incremental volumetric reconstruction path of the freehand
spine-ultrasound system of arXiv 2412.00058 (reference: `spinevol`, /root/reference).

The product is libspinevol_b200.so (C-ABI in include/spinevol_b200.h, sm_100a kernels in
csrc/); this package is the host-side mirror of the reference reconstruct/project API.
"""
from . import _abi
from ._abi import (ACC_PNN, ACC_TRILINEAR, FILL_MEAN, FILL_MEDIAN, PROBE_FAN, PROBE_LINEAR,
                   PROJ_MAX, PROJ_MEAN, AlgorithmFailure, Box, Calib, DeviceError, GridDesc,
                   InvalidInput, IoError, RenderParams, Rigid, SpinevolError, lib)
from .reconstruct import (VoxelGrid, compose, coronal_projection, dilate, fill_holes,
                          frame_bounds, insert_frame, interpolate_pose, pixel_to_world,
                          pose_from_matrix4, run_incremental)

__all__ = [n for n in dir() if not n.startswith("_")]
