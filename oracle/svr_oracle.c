/*
 * svr_oracle.c — CPU restatement of the spinevol reconstruction hot path.
 * TEST INFRASTRUCTURE ONLY (see svr_oracle.h).  Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off: the reference's fp64 operation order, no contraction).
 */
#include "svr_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define SUM_CAP 4294967039ull /* sum must stay below 2^32-256 */
#define COUNT_CAP 65534u      /* count must stay below 2^16-1 */

/* Quat::rotate (geometry.hpp:44-49): t = 2 (u x v); v' = (v + t*w) + u x t. */
void orc_rotate(const svr_rigid* T, const double v[3], double out[3]) {
    const double w = T->qw, ux = T->qx, uy = T->qy, uz = T->qz;
    /* Vec3::cross (core.hpp:52-54) then operator*(2.0) */
    double cx = uy * v[2] - uz * v[1];
    double cy = uz * v[0] - ux * v[2];
    double cz = ux * v[1] - uy * v[0];
    double tx = cx * 2.0, ty = cy * 2.0, tz = cz * 2.0;
    /* v + t * w */
    double ax = v[0] + tx * w, ay = v[1] + ty * w, az = v[2] + tz * w;
    /* u.cross(t) */
    double ex = uy * tz - uz * ty;
    double ey = uz * tx - ux * tz;
    double ez = ux * ty - uy * tx;
    out[0] = ax + ex;
    out[1] = ay + ey;
    out[2] = az + ez;
}

/* RigidTransform::apply (geometry.hpp:122): rotation.rotate(p) + translation. */
void orc_apply(const svr_rigid* T, const double v[3], double out[3]) {
    double r[3];
    orc_rotate(T, v, r);
    out[0] = r[0] + T->tx;
    out[1] = r[1] + T->ty;
    out[2] = r[2] + T->tz;
}

/* pixel_to_world (geometry.hpp:179-185). Returns 0, or 2 for a pixel outside the image. */
int orc_pixel_to_world(double col, double row, const svr_calib* c, const svr_rigid* pose,
                       double out[3]) {
    if (col < 0 || row < 0 || col >= c->crop_w || row >= c->crop_h) return SVR_E_INVALID;
    double p[3] = {col * c->scale_x_mm, row * c->scale_y_mm, 0.0};
    double q[3];
    orc_apply(&c->image_to_transducer, p, q);
    orc_apply(pose, q, out);
    return 0;
}

/* Fan scanline directions; deg_to_rad as core.hpp:109. Pinned in DESIGN.md §3. */
void orc_fan_table(const svr_calib* c, double* s, double* co) {
    const int L = c->crop_h;
    const double A = c->fan_angle_deg;
    for (int i = 0; i < L; ++i) {
        double deg = -0.5 * A + A * ((double)i + 0.5) / (double)L;
        double th = deg * M_PI / 180.0;
        s[i] = sin(th);
        co[i] = cos(th);
    }
}

static inline void fan_local(int line, int sample, const svr_calib* c, const double* fs,
                             const double* fc, double p[3]) {
    double dr = (c->fan_r1_mm - c->fan_r0_mm) / (double)c->crop_w;
    double r = c->fan_r0_mm + ((double)sample + 0.5) * dr;
    p[0] = r * fs[line];
    p[1] = r * fc[line];
    p[2] = 0.0;
}

void orc_fan_point(int line, int sample, const svr_calib* c, const double* fs, const double* fc,
                   const svr_rigid* pose, double out[3]) {
    double p[3], q[3];
    fan_local(line, sample, c, fs, fc, p);
    orc_apply(&c->image_to_transducer, p, q);
    orc_apply(pose, q, out);
}

/* Nearest-voxel snap: i = round((p - origin)/voxel), half away from zero.
 * Returns 1 and the slab-local linear index when inside the stored slab. */
static inline int snap(const orc_grid* g, const double w[3], int32_t idx[3], int64_t* lin) {
    double fx = round((w[0] - g->origin[0]) / g->voxel_mm);
    double fy = round((w[1] - g->origin[1]) / g->voxel_mm);
    double fz = round((w[2] - g->origin[2]) / g->voxel_mm);
    if (!(fx >= 0.0 && fx < (double)g->nx)) return 0;
    if (!(fy >= 0.0 && fy < (double)g->ny)) return 0;
    if (!(fz >= (double)g->z_begin && fz < (double)g->z_end)) return 0;
    idx[0] = (int32_t)fx;
    idx[1] = (int32_t)fy;
    idx[2] = (int32_t)fz;
    *lin = ((int64_t)(idx[2] - g->z_begin) * g->ny + idx[1]) * g->nx + idx[0];
    return 1;
}

static inline void world_point(int32_t col, int32_t row, const svr_calib* c, const double* fs,
                               const double* fc, const svr_rigid* pose, double w[3]) {
    if (c->probe == SVR_PROBE_FAN) {
        orc_fan_point(row, col, c, fs, fc, pose, w);
    } else {
        double p[3] = {(double)col * c->scale_x_mm, (double)row * c->scale_y_mm, 0.0};
        double q[3];
        orc_apply(&c->image_to_transducer, p, q);
        orc_apply(pose, q, w);
    }
}

/* insert_frame. Pixels scanned row-major; skip_zero pixels are skipped
 * before the transform; OOB pixels dropped and counted; caps per SPEC.md:336. */
int orc_insert_frame(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                     const svr_rigid* pose, const svr_calib* c, int32_t skip_zero,
                     svr_box* dirty) {
    if (w != c->crop_w || h != c->crop_h) return SVR_E_INVALID;
    double* fs = NULL;
    double* fc = NULL;
    if (c->probe == SVR_PROBE_FAN) {
        fs = (double*)malloc(sizeof(double) * h);
        fc = (double*)malloc(sizeof(double) * h);
        orc_fan_table(c, fs, fc);
    }
    svr_box b = {1, 1, 1, 0, 0, 0};
    int any = 0;
    for (int32_t r = 0; r < h; ++r) {
        for (int32_t col = 0; col < w; ++col) {
            uint8_t v = px[(int64_t)r * pitch + col];
            if (skip_zero && v == 0) {
                g->skipped_zero++;
                continue;
            }
            double wp[3];
            world_point(col, r, c, fs, fc, pose, wp);
            int32_t idx[3];
            int64_t lin;
            if (!snap(g, wp, idx, &lin)) {
                g->oob++;
                continue;
            }
            if ((uint64_t)g->sum[lin] + v > SUM_CAP || (uint32_t)g->count[lin] + 1u > COUNT_CAP) {
                g->saturated++;
                continue;
            }
            g->sum[lin] += v;
            g->count[lin] += 1;
            g->inserted++;
            if (!any) {
                b.x0 = b.x1 = idx[0];
                b.y0 = b.y1 = idx[1];
                b.z0 = b.z1 = idx[2];
                any = 1;
            } else {
                if (idx[0] < b.x0) b.x0 = idx[0];
                if (idx[0] > b.x1) b.x1 = idx[0];
                if (idx[1] < b.y0) b.y0 = idx[1];
                if (idx[1] > b.y1) b.y1 = idx[1];
                if (idx[2] < b.z0) b.z0 = idx[2];
                if (idx[2] > b.z1) b.z1 = idx[2];
            }
        }
    }
    g->frames++;
    free(fs);
    free(fc);
    if (dirty) *dirty = b;
    return 0;
}

/* ---- multi-threaded variant (CPU baseline): z-slab-partitioned threads ---- */
typedef struct {
    orc_grid* g;
    const uint8_t* px;
    int64_t pitch, stride;
    int32_t w, h, nframes, skip_zero, tid, nthreads;
    const svr_rigid* poses;
    const svr_calib* c;
    const double *fs, *fc;
    uint64_t inserted, skipped;
    svr_box* boxes; /* per-frame partial dirty boxes of this thread's planes (or NULL) */
} mt_job;

/* z-range (global planes, conservative) a frame can touch: the affine image of the pixel
 * grid is spanned by its corners (linear) or every scanline's end samples (fan). */
static void frame_zrange(const orc_grid* g, const svr_calib* c, const double* fs, const double* fc,
                         const svr_rigid* pose, int32_t w, int32_t h, int32_t* z0, int32_t* z1) {
    double lo = 1e300, hi = -1e300, wp[3];
    if (c->probe == SVR_PROBE_FAN) {
        for (int32_t i = 0; i < h; ++i)
            for (int e = 0; e < 2; ++e) {
                world_point(e ? w - 1 : 0, i, c, fs, fc, pose, wp);
                double u = (wp[2] - g->origin[2]) / g->voxel_mm;
                if (u < lo) lo = u;
                if (u > hi) hi = u;
            }
    } else {
        for (int e = 0; e < 4; ++e) {
            world_point((e & 1) ? w - 1 : 0, (e & 2) ? h - 1 : 0, c, fs, fc, pose, wp);
            double u = (wp[2] - g->origin[2]) / g->voxel_mm;
            if (u < lo) lo = u;
            if (u > hi) hi = u;
        }
    }
    *z0 = (int32_t)floor(lo) - 2;
    *z1 = (int32_t)ceil(hi) + 2;
}

/* Thread t owns z planes [zb_t, ze_t) of the slab and inserts every frame whose z-range
 * meets them, accumulating only its own planes: plain adds, no atomics, deterministic. */
static void* mt_worker(void* arg) {
    mt_job* j = (mt_job*)arg;
    orc_grid* g = j->g;
    const int32_t nzl = g->z_end - g->z_begin;
    const int32_t zb = g->z_begin + (int32_t)((int64_t)nzl * j->tid / j->nthreads);
    const int32_t ze = g->z_begin + (int32_t)((int64_t)nzl * (j->tid + 1) / j->nthreads);
    for (int32_t k = 0; k < j->nframes; ++k) {
        int32_t fz0, fz1;
        frame_zrange(g, j->c, j->fs, j->fc, &j->poses[k], j->w, j->h, &fz0, &fz1);
        if (fz1 < zb || fz0 >= ze) continue;
        const uint8_t* f = j->px + (int64_t)k * j->stride;
        for (int32_t r = 0; r < j->h; ++r) {
            for (int32_t col = 0; col < j->w; ++col) {
                uint8_t v = f[(int64_t)r * j->pitch + col];
                if (j->skip_zero && v == 0) {
                    if (j->tid == 0) j->skipped++;
                    continue;
                }
                double wp[3];
                world_point(col, r, j->c, j->fs, j->fc, &j->poses[k], wp);
                int32_t idx[3];
                int64_t lin;
                if (!snap(g, wp, idx, &lin)) continue;
                if (idx[2] < zb || idx[2] >= ze) continue;
                g->sum[lin] += v;
                g->count[lin] += 1;
                j->inserted++;
                if (j->boxes) {
                    svr_box* b = &j->boxes[k];
                    if (b->x0 > b->x1) {
                        b->x0 = b->x1 = idx[0];
                        b->y0 = b->y1 = idx[1];
                        b->z0 = b->z1 = idx[2];
                    } else {
                        if (idx[0] < b->x0) b->x0 = idx[0];
                        if (idx[0] > b->x1) b->x1 = idx[0];
                        if (idx[1] < b->y0) b->y0 = idx[1];
                        if (idx[1] > b->y1) b->y1 = idx[1];
                        if (idx[2] < b->z0) b->z0 = idx[2];
                        if (idx[2] > b->z1) b->z1 = idx[2];
                    }
                }
            }
        }
    }
    return NULL;
}

int orc_insert_frames_mt(orc_grid* g, const uint8_t* px, int64_t pitch, int64_t stride,
                         int32_t w, int32_t h, int32_t nframes, const svr_rigid* poses,
                         const svr_calib* c, int32_t skip_zero, int32_t nthreads) {
    return orc_insert_frames_mt_boxes(g, px, pitch, stride, w, h, nframes, poses, c, skip_zero,
                                      nthreads, NULL);
}

/* orc_insert_frames_mt with the tight per-frame dirty boxes (insert_frame's DirtyRegion,
 * SPEC.md:292) merged from the threads' partial boxes; boxes may be NULL. */
int orc_insert_frames_mt_boxes(orc_grid* g, const uint8_t* px, int64_t pitch, int64_t stride,
                               int32_t w, int32_t h, int32_t nframes, const svr_rigid* poses,
                               const svr_calib* c, int32_t skip_zero, int32_t nthreads,
                               svr_box* boxes) {
    if (w != c->crop_w || h != c->crop_h) return SVR_E_INVALID;
    if (nthreads < 1) nthreads = 1;
    double* fs = NULL;
    double* fc = NULL;
    if (c->probe == SVR_PROBE_FAN) {
        fs = (double*)malloc(sizeof(double) * h);
        fc = (double*)malloc(sizeof(double) * h);
        orc_fan_table(c, fs, fc);
    }
    mt_job* jobs = (mt_job*)calloc((size_t)nthreads, sizeof(mt_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        mt_job jb = {g, px, pitch, stride, w, h, nframes, skip_zero, t, nthreads, poses, c,
                     fs, fc, 0, 0, NULL};
        if (boxes) {
            jb.boxes = (svr_box*)malloc(sizeof(svr_box) * (size_t)(nframes > 0 ? nframes : 1));
            for (int32_t k = 0; k < nframes; ++k) {
                svr_box e = {1, 1, 1, 0, 0, 0};
                jb.boxes[k] = e;
            }
        }
        jobs[t] = jb;
        pthread_create(&th[t], NULL, mt_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        g->inserted += jobs[t].inserted;
        g->skipped_zero += jobs[t].skipped;
    }
    /* every non-skipped pixel is either inserted by exactly one owner or out of bounds */
    {
        uint64_t nz = 0;
        for (int32_t k = 0; k < nframes; ++k) {
            const uint8_t* f = px + (int64_t)k * stride;
            for (int32_t r = 0; r < h; ++r)
                for (int32_t col = 0; col < w; ++col)
                    if (!(skip_zero && f[(int64_t)r * pitch + col] == 0)) nz++;
        }
        uint64_t ins = 0;
        for (int t = 0; t < nthreads; ++t) ins += jobs[t].inserted;
        g->oob += nz - ins;
    }
    if (boxes) {
        for (int32_t k = 0; k < nframes; ++k) {
            svr_box m = {1, 1, 1, 0, 0, 0};
            for (int t = 0; t < nthreads; ++t) {
                const svr_box b = jobs[t].boxes[k];
                if (b.x0 > b.x1) continue;
                if (m.x0 > m.x1) {
                    m = b;
                } else {
                    if (b.x0 < m.x0) m.x0 = b.x0;
                    if (b.y0 < m.y0) m.y0 = b.y0;
                    if (b.z0 < m.z0) m.z0 = b.z0;
                    if (b.x1 > m.x1) m.x1 = b.x1;
                    if (b.y1 > m.y1) m.y1 = b.y1;
                    if (b.z1 > m.z1) m.z1 = b.z1;
                }
            }
            boxes[k] = m;
        }
        for (int t = 0; t < nthreads; ++t) free(jobs[t].boxes);
    }
    g->frames += (uint64_t)nframes;
    free(jobs);
    free(th);
    free(fs);
    free(fc);
    return 0;
}

/* VoxelGrid::value: round(sum/count); integer form, see DESIGN.md §4. */
static inline uint32_t voxel_value(uint32_t sum, uint32_t count) {
    return (uint32_t)((2ull * sum + count) / (2ull * count));
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* fill_holes: every voxel of `region` is recomputed into the shadow fill
 * layer.  Non-empty voxels get 0.  Empty voxels with n >= 1 non-empty neighbours (cube of
 * radius r, self excluded, clipped to the stored slab) get:
 *   mean   (BASELINE cfg1): (n << 16) | sum of neighbour values
 *   median:   (n << 16) | lower median of neighbour values (core.hpp:93-99)
 * Returns the number of filled voxels. */
int64_t orc_fill_holes(orc_grid* g, const svr_box* region, int32_t mode, int32_t radius) {
    svr_box b;
    g->fill_mode = mode;
    if (region) {
        b = *region;
    } else {
        svr_box all = {0, 0, g->z_begin, g->nx - 1, g->ny - 1, g->z_end - 1};
        b = all;
    }
    if (b.x0 < 0) b.x0 = 0;
    if (b.y0 < 0) b.y0 = 0;
    if (b.z0 < g->z_begin) b.z0 = g->z_begin;
    if (b.x1 > g->nx - 1) b.x1 = g->nx - 1;
    if (b.y1 > g->ny - 1) b.y1 = g->ny - 1;
    if (b.z1 > g->z_end - 1) b.z1 = g->z_end - 1;
    if (b.x0 > b.x1 || b.y0 > b.y1 || b.z0 > b.z1) return 0;
    int side = 2 * radius + 1;
    uint32_t* vals = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)side * side * side);
    int64_t filled = 0;
    const int64_t sx = 1, sy = g->nx, sz = (int64_t)g->nx * g->ny;
    for (int32_t z = b.z0; z <= b.z1; ++z)
        for (int32_t y = b.y0; y <= b.y1; ++y)
            for (int32_t x = b.x0; x <= b.x1; ++x) {
                int64_t lin = (int64_t)(z - g->z_begin) * sz + y * sy + x * sx;
                if (g->count[lin] != 0) {
                    g->fill[lin] = 0;
                    continue;
                }
                int n = 0;
                uint32_t acc = 0;
                for (int dz = -radius; dz <= radius; ++dz) {
                    int32_t zz = z + dz;
                    if (zz < g->z_begin || zz >= g->z_end) continue;
                    for (int dy = -radius; dy <= radius; ++dy) {
                        int32_t yy = y + dy;
                        if (yy < 0 || yy >= g->ny) continue;
                        for (int dx = -radius; dx <= radius; ++dx) {
                            int32_t xx = x + dx;
                            if (xx < 0 || xx >= g->nx) continue;
                            int64_t l2 = (int64_t)(zz - g->z_begin) * sz + yy * sy + xx;
                            uint32_t c = g->count[l2];
                            if (c == 0) continue;
                            uint32_t v = voxel_value(g->sum[l2], c);
                            if (mode == SVR_FILL_MEAN) acc += v;
                            vals[n] = v;
                            n++;
                        }
                    }
                }
                if (n == 0) {
                    g->fill[lin] = 0;
                    continue;
                }
                if (mode == SVR_FILL_MEDIAN) {
                    qsort(vals, (size_t)n, sizeof(uint32_t), cmp_u32);
                    acc = vals[(n - 1) / 2];
                }
                g->fill[lin] = ((uint32_t)n << 16) | acc;
                filled++;
            }
    free(vals);
    return filled;
}

/* f32 value of a voxel for rendering; returns 0 when the voxel is undefined. */
static inline int voxel_f(const orc_grid* g, int64_t lin, int32_t fill_mode, float* f) {
    if (g->weight) { /* trilinear volume (BASELINE cfg5): f = wsum / weight, defined iff weight > 0 */
        if (!(g->weight[lin] > 0.0f)) return 0;
        *f = g->wsum[lin] / g->weight[lin];
        return 1;
    }
    uint32_t c = g->count[lin];
    if (c) {
        *f = (float)voxel_value(g->sum[lin], c);
        return 1;
    }
    uint32_t fl = g->fill ? g->fill[lin] : 0;
    uint32_t n = fl >> 16;
    if (n == 0) return 0;
    if (fill_mode == SVR_FILL_MEAN)
        *f = (float)(fl & 0xFFFFu) / (float)n;
    else
        *f = (float)(fl & 0xFFFFu);
    return 1;
}

void orc_values(const orc_grid* g, int32_t apply_fills, uint8_t* out) {
    int64_t n = (int64_t)(g->z_end - g->z_begin) * g->ny * g->nx;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t c = g->count[i];
        if (c) {
            out[i] = (uint8_t)voxel_value(g->sum[i], c);
        } else if (apply_fills && g->fill && (g->fill[i] >> 16)) {
            uint32_t nn = g->fill[i] >> 16, s = g->fill[i] & 0xFFFFu;
            /* mean fills round like value(): (2s+n)/(2n); median fills carry the value */
            out[i] = g->fill_mode == SVR_FILL_MEAN ? (uint8_t)((2u * s + nn) / (2u * nn)) : (uint8_t)s;
        } else {
            out[i] = 0;
        }
    }
}

/* Integer render parameters (shared pin with the device host code). */
void orc_render_ints(const svr_render_params* p, double v, int32_t ny, int32_t* ylo,
                     int32_t* yhi, int32_t* above, int32_t* below) {
    int32_t lo = (int32_t)ceil(p->depth_lo_mm / v - 1e-6);
    int32_t hi = (int32_t)floor(p->depth_hi_mm / v + 1e-6);
    if (lo < 0) lo = 0;
    if (hi > ny - 2) hi = ny - 2;
    *ylo = lo;
    *yhi = hi;
    *above = (int32_t)lround(p->band_above_mm / v);
    *below = (int32_t)lround(p->band_below_mm / v);
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* Depth-band coronal render (BASELINE cfg4), images are (z_end-z_begin) x nx, x fastest.
 * Incremental: depths recomputed on dirty (+) fill_radius (x,z), median+band on that (+) R. */
/* the rows [z0, z1] of one render region (orc_render's dilations and clipping) */
static void render_ranges(const orc_grid* g, const svr_box* dirty, int32_t fr, int32_t R, int32_t* d,
                          int32_t* m) {
    int32_t dx0 = dirty->x0 - fr, dx1 = dirty->x1 + fr, dz0 = dirty->z0 - fr, dz1 = dirty->z1 + fr;
    int32_t mx0 = dx0 - R, mx1 = dx1 + R, mz0 = dz0 - R, mz1 = dz1 + R;
#define CLX(a) ((a) < 0 ? 0 : ((a) > g->nx - 1 ? g->nx - 1 : (a)))
#define CLZ(a) ((a) < g->z_begin ? g->z_begin : ((a) > g->z_end - 1 ? g->z_end - 1 : (a)))
    d[0] = CLX(dx0); d[1] = CLX(dx1); d[2] = CLZ(dz0); d[3] = CLZ(dz1);
    m[0] = CLX(mx0); m[1] = CLX(mx1); m[2] = CLZ(mz0); m[3] = CLZ(mz1);
#undef CLX
#undef CLZ
}

/* One pass of the render over the (already dilated and clipped) column range of `r`:
 * pass 1 computes column depths over x in [r.x0, r.x1], z in [r.z0, r.z1]; pass 2 the median
 * and band of the same range.  orc_render runs pass 1 over the dirty region (+ fill radius) and
 * pass 2 over that (+ median radius). */
void orc_render_pass(const orc_grid* g, const svr_box* r, int32_t pass, const svr_render_params* p,
                     float* mean, float* maxv, int32_t* depth, int32_t* mdepth) {
    int32_t ylo, yhi, above, below;
    orc_render_ints(p, g->voxel_mm, g->ny, &ylo, &yhi, &above, &below);
    const int32_t R = p->median_radius;
    const int64_t sz = (int64_t)g->nx * g->ny;
    if (pass == 1) {
        for (int32_t z = r->z0; z <= r->z1; ++z)
            for (int32_t x = r->x0; x <= r->x1; ++x) {
                int64_t base = (int64_t)(z - g->z_begin) * sz + x;
                int valid = 0;
                float prev = 0.0f;
                if (ylo <= yhi) {
                    float fv;
                    if (voxel_f(g, base + (int64_t)ylo * g->nx, p->fill_mode, &fv)) { prev = fv; valid = 1; }
                }
                float best = 0.0f;
                int32_t arg = -1;
                for (int32_t y = ylo; y <= yhi; ++y) {
                    float nxt = 0.0f, fv;
                    if (voxel_f(g, base + (int64_t)(y + 1) * g->nx, p->fill_mode, &fv)) { nxt = fv; valid = 1; }
                    float gr = nxt - prev;
                    if (arg < 0 || gr > best) { best = gr; arg = y; }
                    prev = nxt;
                }
                depth[(int64_t)(z - g->z_begin) * g->nx + x] = valid ? arg : -1;
            }
        return;
    }
    int32_t* win = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * R + 1) * (2 * R + 1));
    for (int32_t z = r->z0; z <= r->z1; ++z)
        for (int32_t x = r->x0; x <= r->x1; ++x) {
            int n = 0;
            for (int32_t zz = z - R; zz <= z + R; ++zz) {
                if (zz < g->z_begin || zz >= g->z_end) continue;
                for (int32_t xx = x - R; xx <= x + R; ++xx) {
                    if (xx < 0 || xx >= g->nx) continue;
                    int32_t d = depth[(int64_t)(zz - g->z_begin) * g->nx + xx];
                    if (d >= 0) win[n++] = d;
                }
            }
            int64_t o = (int64_t)(z - g->z_begin) * g->nx + x;
            int32_t md = -1;
            if (n) {
                qsort(win, (size_t)n, sizeof(int32_t), cmp_i32);
                md = win[(n - 1) / 2];
            }
            mdepth[o] = md;
            float mv = 0.0f, mx = 0.0f;
            if (md >= 0) {
                int32_t y0 = md - above, y1 = md + below;
                if (y0 < 0) y0 = 0;
                if (y1 > g->ny - 1) y1 = g->ny - 1;
                int64_t base = (int64_t)(z - g->z_begin) * sz + x;
                double s = 0.0;
                int cnt = 0;
                float m = 0.0f;
                for (int32_t y = y0; y <= y1; ++y) {
                    float fv;
                    if (voxel_f(g, base + (int64_t)y * g->nx, p->fill_mode, &fv)) {
                        s += (double)fv;
                        if (cnt == 0 || fv > m) m = fv;
                        cnt++;
                    }
                }
                if (cnt) {
                    mv = (float)(s / (double)cnt);
                    mx = m;
                }
            }
            mean[o] = mv;
            maxv[o] = mx;
        }
    free(win);
}

void orc_render(const orc_grid* g, const svr_box* dirty, int32_t fill_radius,
                const svr_render_params* p, float* mean, float* maxv, int32_t* depth,
                int32_t* mdepth) {
    svr_box all = {0, 0, g->z_begin, g->nx - 1, g->ny - 1, g->z_end - 1};
    if (dirty && dirty->x0 > dirty->x1) return;
    int32_t d[4], m[4];
    if (dirty) {
        render_ranges(g, dirty, fill_radius, p->median_radius, d, m);
    } else {
        d[0] = m[0] = 0; d[1] = m[1] = g->nx - 1; d[2] = m[2] = g->z_begin; d[3] = m[3] = g->z_end - 1;
    }
    (void)all;
    svr_box r1 = {d[0], 0, d[2], d[1], g->ny - 1, d[3]}, r2 = {m[0], 0, m[2], m[1], g->ny - 1, m[3]};
    orc_render_pass(g, &r1, 1, p, mean, maxv, depth, mdepth);
    orc_render_pass(g, &r2, 2, p, mean, maxv, depth, mdepth);
}

/* coronal_projection: max, or mean over non-empty voxels (round like
 * value()), along depth_axis; empty columns -> 0.  Output over the two remaining axes,
 * lower-numbered axis fastest. */
void orc_coronal_projection(const orc_grid* g, int32_t mode, int32_t axis, int32_t use_fills,
                            uint8_t* out) {
    int32_t nzl = g->z_end - g->z_begin;
    int32_t dims[3] = {g->nx, g->ny, nzl};
    int a0 = axis == 0 ? 1 : 0;
    int a1 = axis == 2 ? 1 : 2;
    for (int32_t j = 0; j < dims[a1]; ++j)
        for (int32_t i = 0; i < dims[a0]; ++i) {
            uint32_t mx = 0, n = 0;
            uint64_t s = 0;
            for (int32_t k = 0; k < dims[axis]; ++k) {
                int32_t c[3];
                c[a0] = i;
                c[a1] = j;
                c[axis] = k;
                int64_t lin = ((int64_t)c[2] * g->ny + c[1]) * g->nx + c[0];
                uint32_t cnt = g->count[lin], v;
                if (cnt) {
                    v = voxel_value(g->sum[lin], cnt);
                } else if (use_fills && g->fill && (g->fill[lin] >> 16)) {
                    uint32_t nn = g->fill[lin] >> 16, sm = g->fill[lin] & 0xFFFFu;
                    v = g->fill_mode == SVR_FILL_MEAN ? (2u * sm + nn) / (2u * nn) : sm;
                } else {
                    continue;
                }
                if (v > mx) mx = v;
                s += v;
                n++;
            }
            uint8_t r = 0;
            if (n) r = mode == SVR_PROJ_MAX ? (uint8_t)mx : (uint8_t)((2 * s + n) / (2ull * n));
            out[(int64_t)j * dims[a0] + i] = r;
        }
}

/* Trilinear splat (BASELINE cfg5): u = (p - origin)/voxel, i0 = floor(u), f = u - i0; the
 * 8 corners (clipped to the slab) get w = prod(f or 1-f); wsum += w*px, weight += w.
 * Accumulated in f32 in row-major pixel order (the tolerance test absorbs order). */
/* ws64 / wt64 non-NULL: accumulate the same fp32-rounded contributions in fp64 instead (the
 * parity reference: the GPU differs from it only by the rounding of its fp32 sums). */
static int trilinear_impl(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                          const svr_rigid* pose, const svr_calib* c, int32_t skip_zero, double* ws64,
                          double* wt64);

int orc_insert_trilinear(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                         const svr_rigid* pose, const svr_calib* c, int32_t skip_zero) {
    return trilinear_impl(g, px, pitch, w, h, pose, c, skip_zero, NULL, NULL);
}

int orc_insert_trilinear_f64(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                             const svr_rigid* pose, const svr_calib* c, int32_t skip_zero,
                             double* wsum64, double* weight64) {
    return trilinear_impl(g, px, pitch, w, h, pose, c, skip_zero, wsum64, weight64);
}

static int trilinear_impl(orc_grid* g, const uint8_t* px, int64_t pitch, int32_t w, int32_t h,
                          const svr_rigid* pose, const svr_calib* c, int32_t skip_zero, double* ws64,
                          double* wt64) {
    if (w != c->crop_w || h != c->crop_h) return SVR_E_INVALID;
    double* fs = NULL;
    double* fc = NULL;
    if (c->probe == SVR_PROBE_FAN) {
        fs = (double*)malloc(sizeof(double) * h);
        fc = (double*)malloc(sizeof(double) * h);
        orc_fan_table(c, fs, fc);
    }
    for (int32_t r = 0; r < h; ++r)
        for (int32_t col = 0; col < w; ++col) {
            uint8_t v = px[(int64_t)r * pitch + col];
            if (skip_zero && v == 0) {
                g->skipped_zero++;
                continue;
            }
            double wp[3];
            world_point(col, r, c, fs, fc, pose, wp);
            double u[3];
            for (int a = 0; a < 3; ++a) u[a] = (wp[a] - g->origin[a]) / g->voxel_mm;
            double i0[3], f[3];
            for (int a = 0; a < 3; ++a) {
                i0[a] = floor(u[a]);
                f[a] = u[a] - i0[a];
            }
            int hit = 0;
            for (int k = 0; k < 8; ++k) {
                double ix = i0[0] + (k & 1), iy = i0[1] + ((k >> 1) & 1), iz = i0[2] + ((k >> 2) & 1);
                if (!(ix >= 0 && ix < g->nx && iy >= 0 && iy < g->ny && iz >= g->z_begin &&
                      iz < g->z_end))
                    continue;
                double wt = ((k & 1) ? f[0] : 1.0 - f[0]) * (((k >> 1) & 1) ? f[1] : 1.0 - f[1]) *
                            (((k >> 2) & 1) ? f[2] : 1.0 - f[2]);
                int64_t lin = (((int64_t)iz - g->z_begin) * g->ny + (int64_t)iy) * g->nx + (int64_t)ix;
                if (ws64) {
                    ws64[lin] += (double)(float)(wt * v);
                    wt64[lin] += (double)(float)wt;
                } else {
                    g->wsum[lin] += (float)(wt * v);
                    g->weight[lin] += (float)wt;
                }
                hit = 1;
            }
            if (hit)
                g->inserted++;
            else
                g->oob++;
        }
    g->frames++;
    free(fs);
    free(fc);
    return 0;
}


/* ------------------------------------------------------------------ segment */
static double orc_median_lower(double* v, int n) {
    /* median_lower (core.hpp:93-99): v[(n-1)/2] of the sorted sequence */
    for (int i = 1; i < n; ++i) { /* insertion sort: windows and column lists are small */
        double x = v[i];
        int j = i - 1;
        while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
        v[j + 1] = x;
    }
    return v[(n - 1) / 2];
}

/* cut_depth_alg1 (Table I Step 4): K |p_c1 - p_cn - L/2| + D, clamped to [0, axial extent]. */
double orc_cut_depth_alg1(double p_c1, double p_cn, double K, double D, double L,
                          double axial_extent_mm) {
    double c = K * fabs(p_c1 - p_cn - L / 2.0) + D;
    if (c < 0.0) c = 0.0;
    if (c > axial_extent_mm) c = axial_extent_mm;
    return c;
}

/* apply_cut rows: [ceil(cut/sy - 1e-9), floor((cut+band)/sy + 1e-9)] clipped to the image
 * (the 1e-9 keeps 30/0.1 -> 300 and 45/0.1 -> 450 of the SPEC example exact). */
void orc_cut_rows(double cut_mm, double band_mm, double scale_y_mm, int32_t h, int32_t* r0,
                  int32_t* r1) {
    double a = ceil(cut_mm / scale_y_mm - 1e-9), b = floor((cut_mm + band_mm) / scale_y_mm + 1e-9);
    if (a < 0) a = 0;
    if (b > h - 1) b = h - 1;
    *r0 = (int32_t)a;
    *r1 = (int32_t)b;
}

void orc_apply_cut(uint8_t* px, int64_t pitch, int32_t w, int32_t h, int32_t r0, int32_t r1) {
    for (int32_t r = 0; r < h; ++r)
        if (r < r0 || r > r1) memset(px + r * pitch, 0, (size_t)w);
}

/* bone_contour (Table II Step 2), pinned: brightness threshold thr = the frame's pct_rank-th
 * smallest pixel (0-based); with S(r) = I[r] + I[r+1] + I[r+2] (a 3-row window), each column is
 * scanned upward from the bottom and stops at the first window with S(r) >= 3 thr (the first
 * bright structure from below).  It is the cortex ("first strong dark-to-bright transition",
 * SPEC design decision) iff at least shadow_rows rows lie below the window -- all of them in
 * non-bright windows, the acoustic shadow -- and S(r) - S(r+3) >= grad_levels (the 3-row-mean
 * step over a 3-row baseline, in levels).  Frame row = median_lower of the cortex rows; -1 when
 * fewer than min_valid_frac * w columns have one. */
int32_t orc_bone_contour(const uint8_t* px, int64_t pitch, int32_t w, int32_t h, int64_t pct_rank,
                         int32_t grad_levels, int32_t shadow_rows, double min_valid_frac,
                         int32_t* col_rows, int32_t* valid_cols, int32_t* bright_thr) {
    int64_t hist[256] = {0};
    for (int32_t r = 0; r < h; ++r)
        for (int32_t c = 0; c < w; ++c) hist[px[r * pitch + c]]++;
    int32_t thr = 255;
    int64_t cum = 0;
    for (int v = 0; v < 256; ++v) {
        cum += hist[v];
        if (cum > pct_rank) { thr = v; break; }
    }
    int32_t nv = 0;
    double* rows = (double*)malloc(sizeof(double) * (size_t)(w > 0 ? w : 1));
    for (int32_t c = 0; c < w; ++c) {
        int32_t hit = -1;
        for (int32_t r = h - 3; r >= 0; --r) {
            int S = px[r * pitch + c] + px[(r + 1) * pitch + c] + px[(r + 2) * pitch + c];
            if (S < 3 * thr) continue;
            if (h - (r + 3) >= shadow_rows && r + 5 <= h - 1) {
                int Sb = px[(r + 3) * pitch + c] + px[(r + 4) * pitch + c] + px[(r + 5) * pitch + c];
                if (S - Sb >= grad_levels) hit = r;
            }
            break;
        }
        if (col_rows) col_rows[c] = hit;
        if (hit >= 0) rows[nv++] = hit;
    }
    if (valid_cols) *valid_cols = nv;
    if (bright_thr) *bright_thr = thr;
    int32_t out = -1;
    if (nv > 0 && !((double)nv < min_valid_frac * (double)w)) out = (int32_t)orc_median_lower(rows, nv);
    free(rows);
    return out;
}

/* smooth_depths (Table II Step 3): gaps bridged linearly between the nearest valid samples
 * (a + (b - a) * ((i - ia) / (ib - ia))), leading / trailing gaps take the nearest valid value;
 * then median_lower over [i - window/2, i + window/2] clipped to the series. */
int orc_smooth_depths(const double* d, const uint8_t* valid, int32_t n, int32_t window, double* out) {
    if (window < 3 || window % 2 == 0) return -2;
    int32_t first = -1, last = -1;
    for (int32_t i = 0; i < n; ++i)
        if (valid[i]) { if (first < 0) first = i; last = i; }
    if (first < 0) return -1;
    double* g = (double*)malloc(sizeof(double) * (size_t)n);
    int32_t prev = -1;
    for (int32_t i = 0; i < n; ++i) {
        if (valid[i]) { g[i] = d[i]; prev = i; continue; }
        if (i < first) { g[i] = d[first]; continue; }
        if (i > last) { g[i] = d[last]; continue; }
        int32_t nx = i + 1;
        while (!valid[nx]) ++nx;
        double t = (double)(i - prev) / (double)(nx - prev);
        g[i] = d[prev] + (d[nx] - d[prev]) * t;
    }
    int32_t hw = window / 2;
    double* win = (double*)malloc(sizeof(double) * (size_t)window);
    for (int32_t i = 0; i < n; ++i) {
        int32_t a = i - hw < 0 ? 0 : i - hw, b = i + hw > n - 1 ? n - 1 : i + hw, m = 0;
        for (int32_t k = a; k <= b; ++k) win[m++] = g[k];
        out[i] = orc_median_lower(win, m);
    }
    free(win);
    free(g);
    return 0;
}


/* ---- multi-threaded fill + render over box lists (CPU baseline of the whole bench step) ----
 * Threads split each box's z range; the fill writes only its own voxels and reads only the
 * accumulators, the render's first pass (column depths) completes for every box before the
 * second (median + band) reads them -- the same results as the single-threaded functions. */
typedef struct {
    orc_grid* g;
    const svr_box* boxes;
    int32_t n, mode, radius, tid, nthreads;
    int64_t filled;
} fill_job;

static void* fill_worker(void* arg) {
    fill_job* j = (fill_job*)arg;
    for (int32_t i = 0; i < j->n; ++i) {
        svr_box b = j->boxes[i];
        if (b.z0 < j->g->z_begin) b.z0 = j->g->z_begin;
        if (b.z1 > j->g->z_end - 1) b.z1 = j->g->z_end - 1;
        const int32_t len = b.z1 - b.z0 + 1;
        if (len <= 0) continue;
        svr_box sub = b;
        sub.z0 = b.z0 + (int32_t)((int64_t)len * j->tid / j->nthreads);
        sub.z1 = b.z0 + (int32_t)((int64_t)len * (j->tid + 1) / j->nthreads) - 1;
        if (sub.z0 > sub.z1) continue;
        j->filled += orc_fill_holes(j->g, &sub, j->mode, j->radius);
    }
    return NULL;
}

int64_t orc_fill_holes_boxes_mt(orc_grid* g, const svr_box* boxes, int32_t n, int32_t mode,
                                int32_t radius, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    fill_job* jobs = (fill_job*)calloc((size_t)nthreads, sizeof(fill_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        fill_job jb = {g, boxes, n, mode, radius, t, nthreads, 0};
        jobs[t] = jb;
        pthread_create(&th[t], NULL, fill_worker, &jobs[t]);
    }
    int64_t filled = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        filled += jobs[t].filled;
    }
    g->fill_mode = mode;
    free(jobs);
    free(th);
    return filled;
}

typedef struct {
    const orc_grid* g;
    const svr_box* boxes;
    int32_t n, fill_radius, tid, nthreads;
    const svr_render_params* p;
    float *mean, *maxv;
    int32_t *depth, *mdepth;
    pthread_barrier_t* bar;
} render_job;

static void* render_worker(void* arg) {
    render_job* j = (render_job*)arg;
    const orc_grid* g = j->g;
    const svr_render_params* p = j->p;
    int32_t ylo, yhi, above, below;
    orc_render_ints(p, g->voxel_mm, g->ny, &ylo, &yhi, &above, &below);
    const int32_t R = p->median_radius;
    for (int pass = 1; pass <= 2; ++pass) {
        for (int32_t i = 0; i < j->n; ++i) {
            if (j->boxes[i].x0 > j->boxes[i].x1) continue;
            int32_t d[4], m[4];
            render_ranges(g, &j->boxes[i], j->fill_radius, R, d, m);
            const int32_t* r = pass == 1 ? d : m;
            const int32_t len = r[3] - r[2] + 1;
            if (len <= 0) continue;
            /* this thread's rows, as a region whose dilation reproduces exactly them */
            svr_box sub;
            sub.x0 = r[0];
            sub.x1 = r[1];
            sub.z0 = r[2] + (int32_t)((int64_t)len * j->tid / j->nthreads);
            sub.z1 = r[2] + (int32_t)((int64_t)len * (j->tid + 1) / j->nthreads) - 1;
            if (sub.z0 > sub.z1) continue;
            sub.y0 = 0;
            sub.y1 = g->ny - 1;
            orc_render_pass(g, &sub, pass, p, j->mean, j->maxv, j->depth, j->mdepth);
        }
        pthread_barrier_wait(j->bar);
    }
    return NULL;
}

void orc_render_boxes_mt(const orc_grid* g, const svr_box* boxes, int32_t n, int32_t fill_radius,
                         const svr_render_params* p, float* mean, float* maxv, int32_t* depth,
                         int32_t* mdepth, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
    render_job* jobs = (render_job*)calloc((size_t)nthreads, sizeof(render_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        render_job jb = {g, boxes, n, fill_radius, t, nthreads, p, mean, maxv, depth, mdepth, &bar};
        jobs[t] = jb;
        pthread_create(&th[t], NULL, render_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    pthread_barrier_destroy(&bar);
    free(jobs);
    free(th);
}
