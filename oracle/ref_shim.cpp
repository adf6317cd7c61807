// ref_shim.cpp — C entry points over the REFERENCE's own headers
// (/root/reference/proj/include/spinevol/{core,geometry,image}.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libspinevol_ref.so.  TEST INFRASTRUCTURE ONLY:
// it pins the C restatement (svr_oracle.c) and serves as the "reference" CPU baseline.
//
// The reference ships no reconstruction code; ref_insert_frames is the
// SPEC.md:289-297 insert loop driven by the reference's own spinevol::pixel_to_world
// (geometry.hpp:179-185), multi-threaded by z-slab ownership (SPEC.md:331
// determinism for any worker count).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "spinevol/core.hpp"
#include "spinevol/geometry.hpp"
#include "spinevol/image.hpp"
#include "../include/spinevol_b200.h"

using namespace spinevol;

static RigidTransform to_ref(const svr_rigid* r) {
    RigidTransform t;
    t.rotation = Quat{r->qw, r->qx, r->qy, r->qz};
    t.translation = Vec3{r->tx, r->ty, r->tz};
    return t;
}

static void from_ref(const RigidTransform& t, svr_rigid* r) {
    r->qw = t.rotation.w;
    r->qx = t.rotation.x;
    r->qy = t.rotation.y;
    r->qz = t.rotation.z;
    r->tx = t.translation.x;
    r->ty = t.translation.y;
    r->tz = t.translation.z;
}

static ImageCalibration calib_ref(const svr_calib* c) {
    ImageCalibration k;
    k.crop_rect = CropRect{c->crop_x, c->crop_y, c->crop_w, c->crop_h};
    k.scale_x_mm = c->scale_x_mm;
    k.scale_y_mm = c->scale_y_mm;
    k.image_to_transducer = to_ref(&c->image_to_transducer);
    k.latency_ms = c->latency_ms;
    return k;
}

extern "C" {

int ref_pixel_to_world(double col, double row, const svr_calib* c, const svr_rigid* pose,
                       double out[3]) {
    try {
        Vec3 w = pixel_to_world(col, row, calib_ref(c), to_ref(pose));
        out[0] = w.x;
        out[1] = w.y;
        out[2] = w.z;
        return 0;
    } catch (const InvalidInput&) {
        return 2;
    }
}

int ref_from_matrix4(const double m[16], svr_rigid* out) {
    try {
        std::array<double, 16> a;
        for (int i = 0; i < 16; ++i) a[i] = m[i];
        from_ref(RigidTransform::from_matrix4(a), out);
        return 0;
    } catch (const InvalidInput&) {
        return 2;
    }
}

int ref_compose(const svr_rigid* a, const svr_rigid* b, svr_rigid* out) {
    from_ref(compose(to_ref(a), to_ref(b)), out);
    return 0;
}

int ref_apply(const svr_rigid* a, const double p[3], double out[3]) {
    Vec3 w = to_ref(a).apply(Vec3{p[0], p[1], p[2]});
    out[0] = w.x;
    out[1] = w.y;
    out[2] = w.z;
    return 0;
}

int ref_interpolate_pose(const double* t_ms, const svr_rigid* poses, int n, double t,
                         svr_rigid* out) {
    try {
        std::vector<TimedPose> v((size_t)n);
        for (int i = 0; i < n; ++i) v[i] = TimedPose{t_ms[i], to_ref(&poses[i])};
        from_ref(interpolate_pose(std::span<const TimedPose>(v), t), out);
        return 0;
    } catch (const InvalidInput&) {
        return 2;
    }
}

double ref_median_lower(const double* v, int n) {
    return median_lower(std::vector<double>(v, v + n));
}

// Multi-threaded reference CPU insert (linear probe via spinevol::pixel_to_world; fan via
// the builder's polar pin then the reference RigidTransform::apply chain).
int ref_insert_frames(int32_t nx, int32_t ny, int32_t z_begin, int32_t z_end, double voxel_mm,
                      const double origin[3], uint32_t* sum, uint16_t* count, const uint8_t* px,
                      int64_t pitch, int64_t stride, int32_t w, int32_t h, int32_t nframes,
                      const svr_rigid* poses, const svr_calib* c, int32_t skip_zero,
                      int32_t nthreads, uint64_t* inserted_out) {
    if (w != c->crop_w || h != c->crop_h) return 2;
    if (nthreads < 1) nthreads = 1;
    const ImageCalibration calib = calib_ref(c);
    std::vector<double> fs, fc;
    if (c->probe == SVR_PROBE_FAN) {
        fs.resize((size_t)h);
        fc.resize((size_t)h);
        for (int i = 0; i < h; ++i) {
            double deg = -0.5 * c->fan_angle_deg + c->fan_angle_deg * ((double)i + 0.5) / (double)h;
            double th = deg_to_rad(deg);
            fs[i] = std::sin(th);
            fc[i] = std::cos(th);
        }
    }
    // z-slab-partitioned threads: thread t owns planes [zb_t, ze_t) and
    // processes every frame whose corner-spanned z-range meets them; plain adds, no atomics.
    auto world = [&](const RigidTransform& pose, int32_t col, int32_t r) -> Vec3 {
        if (c->probe == SVR_PROBE_FAN) {
            double dr = (c->fan_r1_mm - c->fan_r0_mm) / (double)w;
            double rr = c->fan_r0_mm + ((double)col + 0.5) * dr;
            return pose.apply(calib.image_to_transducer.apply(Vec3{rr * fs[r], rr * fc[r], 0.0}));
        }
        return pixel_to_world((double)col, (double)r, calib, pose);
    };
    std::atomic<uint64_t> total{0};
    auto worker = [&](int tid) {
        const int32_t nzl = z_end - z_begin;
        const int32_t zb = z_begin + (int32_t)((int64_t)nzl * tid / nthreads);
        const int32_t ze = z_begin + (int32_t)((int64_t)nzl * (tid + 1) / nthreads);
        uint64_t ins = 0;
        for (int32_t k = 0; k < nframes; ++k) {
            const RigidTransform pose = to_ref(&poses[k]);
            double lo = 1e300, hi = -1e300;
            auto span = [&](int32_t col, int32_t r) {
                double u = (world(pose, col, r).z - origin[2]) / voxel_mm;
                lo = std::min(lo, u);
                hi = std::max(hi, u);
            };
            if (c->probe == SVR_PROBE_FAN) {
                for (int32_t r = 0; r < h; ++r) { span(0, r); span(w - 1, r); }
            } else {
                span(0, 0); span(w - 1, 0); span(0, h - 1); span(w - 1, h - 1);
            }
            if ((int32_t)std::ceil(hi) + 2 < zb || (int32_t)std::floor(lo) - 2 >= ze) continue;
            const uint8_t* f = px + (int64_t)k * stride;
            for (int32_t r = 0; r < h; ++r)
                for (int32_t col = 0; col < w; ++col) {
                    uint8_t v = f[(int64_t)r * pitch + col];
                    if (skip_zero && v == 0) continue;
                    Vec3 p = world(pose, col, r);
                    double fx = std::round((p.x - origin[0]) / voxel_mm);
                    double fy = std::round((p.y - origin[1]) / voxel_mm);
                    double fz = std::round((p.z - origin[2]) / voxel_mm);
                    if (!(fx >= 0.0 && fx < nx && fy >= 0.0 && fy < ny && fz >= zb && fz < ze))
                        continue;
                    int64_t lin = ((int64_t)((int32_t)fz - z_begin) * ny + (int32_t)fy) * nx + (int32_t)fx;
                    sum[lin] += v;
                    count[lin] += 1;
                    ++ins;
                }
        }
        total.fetch_add(ins);
    };
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t) th.emplace_back(worker, t);
    for (auto& t : th) t.join();
    if (inserted_out) *inserted_out = total.load();
    return 0;
}

// read_pgm / write_pgm (image.hpp:34-72).  Returns 0, 2 (InvalidInput) or 4 (IoError);
// ref_read_pgm copies at most cap bytes and reports the dims.
int ref_read_pgm(const char* path, uint8_t* out, int64_t cap, int32_t* w, int32_t* h) {
    try {
        Image8 img = read_pgm(path);
        *w = img.width;
        *h = img.height;
        const int64_t n = std::min<int64_t>(cap, (int64_t)img.data.size());
        if (n > 0) std::copy(img.data.begin(), img.data.begin() + n, out);
        return 0;
    } catch (const InvalidInput&) {
        return 2;
    } catch (const IoError&) {
        return 4;
    }
}

int ref_write_pgm(const char* path, const uint8_t* px, int32_t w, int32_t h) {
    try {
        Image8 img(w, h);
        std::copy(px, px + (size_t)w * h, img.data.begin());
        write_pgm(img, path);
        return 0;
    } catch (const IoError&) {
        return 4;
    }
}

}  // extern "C"
