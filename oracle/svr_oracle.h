/*
 * svr_oracle.h — CPU oracle for the spinevol reconstruction hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the checker
 * or the reported CPU baseline.  The product path (paper_2412_00058_b200) never calls it.
 *
 * It restates, in plain C compiled with -ffp-contract=off:
 *   - pixel_to_world            geometry.hpp:179-185 (Quat::rotate :44-49, apply :122)
 *   - insert_frame              SPEC.md:289-297 (+ caps :336, OOB :338, layout :344)
 *   - fill_holes                SPEC.md:298-306 (median, Chebyshev r) and BASELINE cfg1
 *                               3x3x3 mean (pins in DESIGN.md §4)
 *   - coronal_projection
 *   - depth-band render         BASELINE cfg4 (pins in DESIGN.md §4)
 *   - trilinear splat           BASELINE cfg5
 * Pinned against the reference headers themselves (oracle/_ref, built from
 * /root/reference/proj/include by oracle/Makefile) and the SPEC known-answer tests.
 */
#ifndef SVR_ORACLE_H
#define SVR_ORACLE_H
#include <stdint.h>
#include "../include/spinevol_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_grid {
    int32_t nx, ny, nz;       /* global dims */
    int32_t z_begin, z_end;   /* stored slab of global planes */
    double voxel_mm;
    double origin[3];
    uint32_t* sum;            /* (z_end-z_begin)*ny*nx, x fastest */
    uint16_t* count;
    uint32_t* fill;           /* (n << 16) | payload, 0 = unfilled */
    float* wsum;              /* trilinear mode (may be NULL) */
    float* weight;
    uint64_t frames, inserted, oob, skipped_zero, saturated;
    int32_t fill_mode;        /* mode of the latest orc_fill_holes (decodes the fill layer) */
} orc_grid;

/* geometry */
void orc_rotate(const svr_rigid* T, const double v[3], double out[3]);
void orc_apply(const svr_rigid* T, const double v[3], double out[3]);
int orc_pixel_to_world(double col, double row, const svr_calib* calib, const svr_rigid* pose,
                       double out[3]);
void orc_fan_table(const svr_calib* calib, double* sin_out, double* cos_out);
void orc_fan_point(int line, int sample, const svr_calib* calib, const double* fan_sin,
                   const double* fan_cos, const svr_rigid* pose, double out[3]);

/* reconstruct */
int orc_insert_frame(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                     const svr_rigid* pose, const svr_calib* calib, int32_t skip_zero,
                     svr_box* dirty);
/* same accumulation, nthreads z-slab-partitioned worker threads (no atomics, no caps) */
int orc_insert_frames_mt(orc_grid* g, const uint8_t* px, int64_t pitch, int64_t frame_stride,
                         int32_t w, int32_t h, int32_t nframes, const svr_rigid* poses,
                         const svr_calib* calib, int32_t skip_zero, int32_t nthreads);
int orc_insert_frames_mt_boxes(orc_grid* g, const uint8_t* px, int64_t pitch, int64_t frame_stride,
                               int32_t w, int32_t h, int32_t nframes, const svr_rigid* poses,
                               const svr_calib* calib, int32_t skip_zero, int32_t nthreads,
                               svr_box* boxes);
int64_t orc_fill_holes(orc_grid* g, const svr_box* region, int32_t mode, int32_t radius);
void orc_values(const orc_grid* g, int32_t apply_fills, uint8_t* out);

/* project */
void orc_render_ints(const svr_render_params* p, double voxel_mm, int32_t ny, int32_t* ylo,
                     int32_t* yhi, int32_t* above, int32_t* below);
void orc_render(const orc_grid* g, const svr_box* dirty, int32_t fill_radius,
                const svr_render_params* p, float* mean, float* maxv, int32_t* depth,
                int32_t* mdepth);
void orc_render_pass(const orc_grid* g, const svr_box* r, int32_t pass, const svr_render_params* p,
                     float* mean, float* maxv, int32_t* depth, int32_t* mdepth);
/* multithreaded fill / render over box lists (the CPU baseline of the bench step) */
int64_t orc_fill_holes_boxes_mt(orc_grid* g, const svr_box* boxes, int32_t n, int32_t mode,
                                int32_t radius, int32_t nthreads);
void orc_render_boxes_mt(const orc_grid* g, const svr_box* boxes, int32_t n, int32_t fill_radius,
                         const svr_render_params* p, float* mean, float* maxv, int32_t* depth,
                         int32_t* mdepth, int32_t nthreads);
void orc_coronal_projection(const orc_grid* g, int32_t mode, int32_t depth_axis,
                            int32_t use_fills, uint8_t* out);

/* trilinear (cfg5) */
int orc_insert_trilinear(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                         const svr_rigid* pose, const svr_calib* calib, int32_t skip_zero);
/* same contributions, summed in fp64 into wsum64 / weight64 (slab-sized arrays) */
int orc_insert_trilinear_f64(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                             const svr_rigid* pose, const svr_calib* calib, int32_t skip_zero,
                             double* wsum64, double* weight64);

/* segment (SPEC.md segment module; the reference implements none of it: parity unpinned
 * except median_lower, core.hpp:93-99, which these use) */
double orc_cut_depth_alg1(double p_c1, double p_cn, double K, double D, double L,
                          double axial_extent_mm);
void orc_cut_rows(double cut_mm, double band_mm, double scale_y_mm, int32_t h, int32_t* r0,
                  int32_t* r1);
void orc_apply_cut(uint8_t* px, int64_t pitch, int32_t w, int32_t h, int32_t r0, int32_t r1);
int32_t orc_bone_contour(const uint8_t* px, int64_t pitch, int32_t w, int32_t h, int64_t pct_rank,
                         int32_t grad_levels, int32_t shadow_rows, double min_valid_frac,
                         int32_t* col_rows, int32_t* valid_cols, int32_t* bright_thr);
int orc_smooth_depths(const double* d, const uint8_t* valid, int32_t n, int32_t window, double* out);

#ifdef __cplusplus
}
#endif
#endif
