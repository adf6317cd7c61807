/*
 * spinevol_b200.h — C-ABI drop-in for the incremental volumetric reconstruction
 * path of the `spinevol` reference (arXiv 2412.00058), implemented with
 * hand-written sm_100a CUDA kernels.
 *
 * The reference API is header-level C++ (namespace spinevol, value types, exceptions).
 * Its reconstruction module exists only as a specification;
 * the only executable hot-path arithmetic is the pixel->world chain in
 * proj/include/spinevol/geometry.hpp.  Each entry point below names the reference
 * interface it replaces (file:line).  The header-only C++ wrapper
 * include/spinevol_b200/reconstruct.hpp rebuilds the SPEC signatures on top of it and
 * rethrows the core.hpp exception types.
 *
 * Conventions
 *   - Every function returns SVR_OK (0) or an error code; the thread-local message is
 *     svr_last_error().  Codes follow the reference exit-code mapping
 *     (core.hpp:12-32): 2 invalid input, 3 algorithm failure, 4 I/O,
 *     plus 5 for CUDA/NCCL failures.  No C++ exception crosses this boundary.
 *   - Buffers are owned by the caller and may be host (pageable or pinned) or device
 *     pointers; the library detects which.  Device memory of a volume is owned by
 *     the handle.  Calls on one handle are serialised onto the handle's stream (their small
 *     uploads run on an internal stream joined to it by events: an event recorded on the
 *     handle's stream after a call, or svr_sync, covers all of the call's work).
 *   - Voxel layout: x fastest, then y, then z.  A handle holds the
 *     global z planes [z_begin, z_end) (a slab; the whole grid when z_begin=0,
 *     z_end=nz).  All boxes are in GLOBAL voxel indices, inclusive.
 */
#ifndef SPINEVOL_B200_H
#define SPINEVOL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SVR_ABI_VERSION 2

/* return codes (core.hpp:12-32 exit-code mapping) */
#define SVR_OK 0
#define SVR_E_INVALID 2   /* spinevol::InvalidInput      */
#define SVR_E_ALGO 3      /* spinevol::AlgorithmFailure  */
#define SVR_E_IO 4        /* spinevol::IoError           */
#define SVR_E_CUDA 5      /* device / NCCL failure        */

#define SVR_PROBE_LINEAR 0 /* pixel (col,row) -> (col*sx, row*sy, 0)            geometry.hpp:183 */
#define SVR_PROBE_FAN 1    /* (line,sample) -> (r sin th, r cos th, 0) */

#define SVR_FILL_MEAN 0   /* BASELINE cfg1/cfg2: mean of non-empty neighbour values, cube radius r */
#define SVR_FILL_MEDIAN 1 /* lower median of non-empty neighbour values, Chebyshev r */

#define SVR_ACC_PNN 0       /* u32 sum + u16 count per voxel, nearest-voxel insert */
#define SVR_ACC_TRILINEAR 1 /* f32 weighted sum + f32 weight, 2x2x2 splat (BASELINE cfg5)     */

#define SVR_PROJ_MAX 0
#define SVR_PROJ_MEAN 1

/* RigidTransform (geometry.hpp:104-140): unit quaternion w,x,y,z + translation mm. */
typedef struct svr_rigid {
    double qw, qx, qy, qz;
    double tx, ty, tz;
} svr_rigid;

/* ImageCalibration (geometry.hpp:160-176) + probe geometry.
 * Linear probe: a frame is crop_h rows x crop_w columns, pixel (col,row) ->
 *   (col*scale_x_mm, row*scale_y_mm, 0)   (geometry.hpp:183).
 * Convex fan: a frame is crop_h scanlines x crop_w samples (line-major);
 *   theta_i = deg_to_rad(-angle/2 + angle*(i+0.5)/lines), r_j = r0 + (j+0.5)*(r1-r0)/samples,
 *   point = (r_j*sin theta_i, r_j*cos theta_i, 0).  Then image_to_transducer, then pose. */
typedef struct svr_calib {
    int32_t crop_x, crop_y, crop_w, crop_h;
    double scale_x_mm, scale_y_mm;
    svr_rigid image_to_transducer;
    double latency_ms;
    int32_t probe; /* SVR_PROBE_* */
    int32_t reserved0;
    double fan_angle_deg, fan_r0_mm, fan_r1_mm;
} svr_calib;

/* VoxelGrid configuration plus the slab this handle stores. */
typedef struct svr_grid_desc {
    int32_t nx, ny, nz;  /* global grid dims */
    int32_t accum;       /* SVR_ACC_* */
    double voxel_mm;
    double origin_mm[3]; /* world position of voxel (0,0,0) centre */
    int32_t z_begin, z_end; /* global planes held by this handle (slab incl. ghosts) */
} svr_grid_desc;

/* DirtyRegion: inclusive global voxel box, empty iff x0 > x1. */
typedef struct svr_box {
    int32_t x0, y0, z0, x1, y1, z1;
} svr_box;

/* Stats counters. */
typedef struct svr_stats {
    uint64_t frames_inserted;
    uint64_t pixels_inserted;
    uint64_t pixels_oob;
    uint64_t pixels_skipped_zero;
    uint64_t pixels_saturated; /* voxels found above the SPEC caps at readout */
    uint64_t exact_fallbacks;  /* pixels resolved by the exact fp64 chain (near .5 ties) */
    uint64_t kernel_launches;  /* kernels this handle launched (all kinds) */
    uint64_t chunks_deferred;  /* 16-px chunks sent to the exact per-pixel pass (ties, edges) */
    uint64_t tiles_table;      /* B-scan tiles inserted through the shared-table kernel (K1) */
    uint64_t graph_captures;   /* svr_frame_step graph (re-)captures */
} svr_stats;

/* Depth-band coronal render (BASELINE cfg4).  Depth axis = grid y, depth(y) = y*voxel_mm.
 * Column depth d = first argmax over y in [lo,hi] of f(y+1)-f(y); median over a
 * (2r+1)^2 window of valid column depths; mean and max of f over [d-above, d+below]. */
typedef struct svr_render_params {
    double depth_lo_mm, depth_hi_mm;     /* 15, 60 */
    double band_above_mm, band_below_mm; /* 5, 2   */
    int32_t median_radius;               /* 2 -> 5x5 */
    int32_t fill_mode;                   /* SVR_FILL_* used to decode the fill layer */
} svr_render_params;

typedef struct svr_volume svr_volume;

/* ---------------------------------------------------------------- host-only ---- */
int svr_abi_version(void);
const char* svr_last_error(void);
/* number of visible CUDA devices (0 on a CPU-only host; never fails) */
int svr_device_count(void);

/* RigidTransform::from_matrix4 (geometry.hpp:133-139 -> Shepperd from_matrix3 :61-78). */
int svr_pose_from_matrix4(const double m[16], svr_rigid* out);
/* compose (geometry.hpp:142-144) */
int svr_compose(const svr_rigid* a, const svr_rigid* b, svr_rigid* out);
/* interpolate_pose (geometry.hpp:194-209, slerp :82-100), poses sorted by t_ms. */
int svr_interpolate_pose(const double* t_ms, const svr_rigid* poses, int n, double t, svr_rigid* out);
/* Ingest pose matching: out[k] = interpolate_pose(poses, frame_t_ms[k] - latency_ms) for the m
 * frames; valid[k] = 0 (identity pose) where that time lies outside the sampled span. */
int svr_match_poses(const double* pose_t_ms, const svr_rigid* poses, int32_t n,
                    const double* frame_t_ms, int32_t m, double latency_ms, svr_rigid* out,
                    uint8_t* valid, int32_t* n_valid);
/* pixel_to_world (geometry.hpp:179-185) for the linear probe, fan point for SVR_PROBE_FAN. */
int svr_pixel_to_world(double col, double row, const svr_calib* calib, const svr_rigid* pose,
                       double out_mm[3]);
/* Conservative voxel box a frame can touch (routing to z-slabs); clipped to the global grid. */
int svr_frame_bounds(const svr_grid_desc* grid, const svr_calib* calib, const svr_rigid* pose,
                     svr_box* out);
/* Contiguous z-slab plan for nranks with `ghost` extra planes each side. */
int svr_plan_slabs(int32_t nz, int32_t nranks, int32_t ghost, int32_t* owned_begin,
                   int32_t* owned_end, int32_t* alloc_begin, int32_t* alloc_end);

/* ---------------------------------------------------------------- device ------- */
/* VoxelGrid construction.  device = CUDA ordinal. */
int svr_create(const svr_grid_desc* desc, int device, svr_volume** out);
int svr_destroy(svr_volume* vol);
/* Use an external cudaStream_t (e.g. the caller's) for every later call. NULL = own stream. */
int svr_set_stream(svr_volume* vol, void* cuda_stream);
/* Switch to an external stream WITHOUT synchronizing the current one: the caller orders the two
 * streams (events).  Used to overlap fill / render of finished z-chunks with later inserts. */
int svr_use_stream(svr_volume* vol, void* cuda_stream);
/* zero accumulators, fill layer, render images, stats */
int svr_clear(svr_volume* vol);
int svr_sync(svr_volume* vol);
int svr_get_desc(const svr_volume* vol, svr_grid_desc* out);

/* insert_frame: one frame, returns the tight dirty box (synchronises). */
int svr_insert_frame(svr_volume* vol, const uint8_t* px, int64_t row_pitch, int32_t w, int32_t h,
                     const svr_rigid* pose, const svr_calib* calib, int32_t skip_zero,
                     svr_box* dirty_out);
/* Batched insert of nframes frames at px + k*frame_stride (host or device memory).
 * dirty_out (nframes boxes) and union_out may be NULL: then the call is asynchronous. */
int svr_insert_frames(svr_volume* vol, const uint8_t* px, int64_t row_pitch, int64_t frame_stride,
                      int32_t w, int32_t h, int32_t nframes, const svr_rigid* poses,
                      const svr_calib* calib, int32_t skip_zero, svr_box* dirty_out,
                      svr_box* union_out);

/* fill_holes over exactly `region` (NULL = whole slab).  The fill layer
 * is a shadow layer: fills never chain.  filled_out may be NULL (asynchronous). */
int svr_fill_holes(svr_volume* vol, const svr_box* region, int32_t mode, int32_t radius,
                   int64_t* filled_out);

/* fill_holes over a list of regions in one launch (e.g. the union of a batch's dirty boxes,
 * one per z-chunk).  Regions should not overlap: an overlap is recomputed identically but
 * counted twice in filled_out. */
int svr_fill_holes_boxes(svr_volume* vol, const svr_box* regions, int32_t n, int32_t mode,
                         int32_t radius, int64_t* filled_out);

/* Depth-band coronal render (BASELINE cfg4), incremental: recompute the columns a change
 * inside `dirty` can affect (dirty (+) fill_radius for depths, (+) median_radius for the
 * image).  dirty = NULL re-renders every column of the slab. */
int svr_render_coronal(svr_volume* vol, const svr_box* dirty, int32_t fill_radius,
                       const svr_render_params* params);
/* One frame of the incremental pipeline as a single CUDA-graph replay: insert,
 * r = 1 mean fill of the conservative dirty box (+) 1, depth-band render of its columns.  The graph
 * is captured on first use (and re-captured when the frame geometry, calibration, render
 * parameters or a region bound changes); px may be host (pageable or pinned) or device memory.
 * Asynchronous; dirty_out (may be NULL) receives the conservative box.  Results are identical to
 * svr_insert_frame + svr_fill_holes + svr_render_coronal over that box.  On a trilinear volume
 * (BASELINE cfg5) the step is the splat and the render of the box (+) 1 columns (no fill layer;
 * fill_radius is ignored).  Pageable host frames are
 * staged before the call returns; pinned host and device frames are read by a copy enqueued on
 * the handle's stream, so px must stay unchanged until the step completes (svr_sync, or an event
 * recorded on the stream after the call). */
int svr_frame_step(svr_volume* vol, const uint8_t* px, int64_t row_pitch, const svr_rigid* pose,
                   const svr_calib* calib, int32_t fill_radius, const svr_render_params* params,
                   svr_box* dirty_out);
/* svr_render_coronal for a list of dirty regions in one pair of launches. */
int svr_render_coronal_boxes(svr_volume* vol, const svr_box* dirty, int32_t n, int32_t fill_radius,
                             const svr_render_params* params);
/* Fused render + gather (multi-GPU): every later render also stores the mean / max of the owned
 * rows [own_z0, own_z1) straight into each of the n images (device pointers, typically the
 * ranks' symmetric-memory peers over NVLink; each a [2][nz][nx] f32 image: mean plane then max
 * plane, global z), so no all-gather has to follow.  n = 0 switches it off.  The caller orders
 * the ranks (e.g. a symmetric-memory barrier) before reading. */
int svr_set_gather_targets(svr_volume* vol, void* const* images, int32_t n, int32_t own_z0,
                           int32_t own_z1);
/* ---------------------------------------------------------------- z-slab sharding ---- */
/* A z-slab sharded PNN / trilinear volume over ndev devices, for C / C++ callers
 * driving several GPUs from one thread: slab r (svr_plan_slabs) lives on devices[r] (devices may
 * repeat) with `ghost` = fill radius + render median radius extra planes per side; frames are
 * routed to the slabs their conservative box meets; the coronal image [2][nz][nx] is gathered on
 * devices[0] by the slabs' renders themselves (peer stores over NVLink).  Bit-identical to one
 * unsharded volume. */
typedef struct svr_sharded svr_sharded;
int svr_sharded_create(const svr_grid_desc* desc, const int32_t* devices, int32_t ndev,
                       int32_t ghost, svr_sharded** out);
int svr_sharded_destroy(svr_sharded* s);
/* slab r's volume handle (for readout) and its owned / stored global planes [z0, z1) */
int svr_sharded_slab(const svr_sharded* s, int32_t r, svr_volume** vol, int32_t* own_z0,
                     int32_t* own_z1, int32_t* alloc_z0, int32_t* alloc_z1);
/* batched insert routed to the slabs (asynchronous per slab); routed_out[r] (may be NULL) =
 * frames slab r took.  Frames in host memory or device memory visible to every device. */
int svr_sharded_insert_frames(svr_sharded* s, const uint8_t* px, int64_t row_pitch,
                              int64_t frame_stride, int32_t w, int32_t h, int32_t nframes,
                              const svr_rigid* poses, const svr_calib* calib, int32_t skip_zero,
                              int32_t* routed_out);
/* fill (dirty region + radius) and depth-band render of every slab's dirty columns since the
 * last call; the renders store their owned rows into the gathered image */
int svr_sharded_fill_render(svr_sharded* s, int32_t fill_radius, int32_t fill_mode,
                            const svr_render_params* params);
int svr_sharded_sync(svr_sharded* s);
/* gathered image: nz rows x nx (mean, max f32; depth i32); outputs may be NULL; synchronises */
int svr_sharded_read_coronal(svr_sharded* s, float* mean_out, float* max_out, int32_t* depth_out);

/* Copy rendered rows z in [z0,z1] (global, inside the slab) as nx-wide row-major images. */
int svr_read_coronal(svr_volume* vol, int32_t z0, int32_t z1, float* mean_out, float* max_out,
                     int32_t* depth_out);
/* svr_read_coronal enqueued on the handle's stream without waiting (outputs pinned or device;
 * complete after svr_sync or the stream's next synchronisation). */
int svr_read_coronal_async(svr_volume* vol, int32_t z0, int32_t z1, float* mean_out, float* max_out,
                           int32_t* depth_out);

/* coronal_projection: u8 max / mean over non-empty voxels along depth_axis
 * (0=x,1=y,2=z); use_fills also admits filled voxels.  Output is row-major over the two
 * remaining axes (lower axis fastest). */
int svr_coronal_projection(svr_volume* vol, int32_t mode, int32_t depth_axis, int32_t use_fills,
                           uint8_t* out);

/* Accumulator / value readout over an inclusive box (NULL = whole slab), x fastest. */
int svr_read_accumulators(svr_volume* vol, const svr_box* box, uint32_t* sum_out,
                          uint16_t* count_out);
/* Checkpoint / resume: overwrite the accumulators of a box (NULL = whole slab) from sum / count
 * arrays in the svr_read_accumulators layout (host or device).  Re-inserting further frames after a
 * restore gives the uninterrupted result (inserts commute). */
int svr_write_accumulators(svr_volume* vol, const svr_box* box, const uint32_t* sum,
                           const uint16_t* count);
/* VoxelGrid::value = round(sum/count); apply_fills adds rounded fill values. */
int svr_read_values(svr_volume* vol, const svr_box* box, int32_t apply_fills, uint8_t* out);
/* export_slices along x: nx images of ny x nzl u8 values (row = z, column =
 * y), out[(x * nzl + z) * ny + y]; values as svr_read_values.  out may be host or device. */
int svr_export_slices_x(svr_volume* vol, int32_t apply_fills, uint8_t* out);
/* export_slices to files: dir/<x zero-padded to `digits`>.pgm (binary P5, image.hpp:34-42). */
int svr_export_slices(svr_volume* vol, const char* dir, int32_t apply_fills, int32_t digits,
                      int32_t* files_out);
/* Volume file: raw u8 values of the slab, x fastest then y then z. */
int svr_export_volume(svr_volume* vol, const char* path, int32_t apply_fills);
/* raw fill layer: (n << 16) | payload (mean: sum of neighbour values; median: value). */
int svr_read_fill(svr_volume* vol, const svr_box* box, uint32_t* out);
/* trilinear volumes: f32 weighted sum and weight */
int svr_read_trilinear(svr_volume* vol, const svr_box* box, float* wsum_out, float* weight_out);

int svr_get_stats(svr_volume* vol, svr_stats* out);

/* Analysis (not on the hot path): distinct in-slab voxels each frame touches (the U of the
 * roofline bytes).  Writes nframes counts. */
int svr_count_footprint(svr_volume* vol, const uint8_t* px, int64_t row_pitch,
                        int64_t frame_stride, int32_t w, int32_t h, int32_t nframes,
                        const svr_rigid* poses, const svr_calib* calib, int32_t skip_zero,
                        int64_t* distinct_out);

/* Self-test of the device VoxelGrid::value rounding: checks every count in [1, 255] and every
 * reachable sum against integer division, and the render's branch-free fill-layer division
 * (payload / n) against IEEE division for every payload in [0, 65535] and n in [1, 1024];
 * writes the mismatch count (0 expected). */
int svr_selftest_value_rounding(int device, int64_t* mismatches);

/* Synthetic B-scan generator (bench input, BASELINE configs): writes nframes frames of
 * w x h u8 into device memory `dst` (row pitch w).  kind 0 = linear speckle + bone arcs,
 * 1 = log-compressed fan speckle + bright band.  Deterministic in (seed, frame). */
int svr_synth_frames(void* dst, int32_t w, int32_t h, int32_t first_frame, int32_t nframes,
                     const svr_calib* calib, const svr_rigid* poses, int32_t kind, uint64_t seed,
                     int device, void* cuda_stream);

/* ---------------------------------------------------------------- ingest (host) ---- */
/* read_pgm header (image.hpp:44-66): binary P5, '#' comments, maxval 255.  Unreadable file ->
 * SVR_E_IO; not P5 / malformed / maxval != 255 -> SVR_E_INVALID (core.hpp:19-32). */
int svr_pgm_info(const char* path, int32_t* width, int32_t* height);
/* read_pgm (image.hpp:44-72) into out (row pitch >= width); dims must match the file. */
int svr_pgm_read(const char* path, uint8_t* out, int64_t row_pitch, int32_t width, int32_t height);
/* write_pgm (image.hpp:34-42). */
int svr_pgm_write(const char* path, const uint8_t* px, int64_t row_pitch, int32_t width,
                  int32_t height);
/* ScanBundle frame loader: decode n PGM files of raw_w x raw_h with nthreads
 * threads (<= 0: all cores), applying crop = {x, y, w, h} (ImageCalibration::crop_rect,
 * geometry.hpp:156-158) while decoding (NULL = whole frame), into out + k * frame_stride with row
 * pitch = cropped width (e.g. a pinned staging buffer for svr_insert_frames).  The lowest failing
 * index is reported in *failed_index and named in svr_last_error. */
int svr_load_frames(const char* const* paths, int32_t n, int32_t raw_w, int32_t raw_h,
                    const int32_t* crop, uint8_t* out, int64_t frame_stride, int32_t nthreads,
                    int32_t* failed_index);
/* Write nbytes to a new file (volume files). */
int svr_write_raw(const char* path, const uint8_t* data, int64_t nbytes);

/* ---------------------------------------------------------------- segment ---------- */
/* cut_depth_alg1 (SPEC.md segment; Table I Step 4): K |p_c1 - p_cn - L/2| + D clamped to
 * [0, axial_extent_mm] (ImageCalibration::axial_extent_mm, geometry.hpp:174). */
int svr_cut_depth_alg1(double p_c1, double p_cn, double K, double D, double L,
                       double axial_extent_mm, double* out);
/* apply_cut rows kept: [ceil(cut/sy - 1e-9), floor((cut+band)/sy + 1e-9)] clipped to [0,h-1]
 * (empty when r0 > r1: the whole frame is cut). */
int svr_cut_rows(double cut_mm, double band_mm, double scale_y_mm, int32_t h, int32_t* r0,
                 int32_t* r1);
/* smooth_depths (Table II Step 3): linear gap bridging (edges: nearest valid), then a sliding
 * median_lower (core.hpp:93-99) of `window` (odd >= 3) samples clipped at the ends.  All-gap
 * input -> SVR_E_ALGO. */
int svr_smooth_depths(const double* depths, const uint8_t* valid, int32_t n, int32_t window,
                      double* out);
/* bone_contour (Table II Step 2) for n device-resident frames: brightness threshold thr = the
 * floor(pct * (w*h - 1))-th smallest pixel; with S(r) = I[r] + I[r+1] + I[r+2], each column is
 * scanned bottom-up to its first window with S(r) >= 3 thr, a cortex hit iff >= shadow_rows rows
 * lie below that window and S(r) - S(r+3) >= grad_levels; frame row = median_lower of the hit
 * rows, or -1 (no contour) when fewer than min_valid_frac * w columns hit.  Depth = row * sy. */
int svr_bone_contour(const uint8_t* px, int64_t row_pitch, int64_t frame_stride, int32_t w,
                     int32_t h, int32_t n, double pct, int32_t grad_levels, int32_t shadow_rows,
                     double min_valid_frac, int32_t* row_out, int32_t* valid_cols_out,
                     int32_t* threshold_out, int32_t* col_rows_out, int device, void* cuda_stream);
/* apply_cut in place on n device-resident frames: rows outside [row0[k], row1[k]] set to 0. */
int svr_apply_cut(uint8_t* px, int64_t row_pitch, int64_t frame_stride, int32_t w, int32_t h,
                  int32_t n, const int32_t* row0, const int32_t* row1, int device,
                  void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* SPINEVOL_B200_H */
