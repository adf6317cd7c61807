// spinevol_b200/reconstruct.hpp — header-only C++ host API over the C-ABI (spinevol_b200.h),
// mirroring the reference's reconstruct / project operations:
//
//   VoxelGrid                       SPEC.md:276-282   (u32 sum + u16 count, x-fastest)
//   insert_frame(grid, ...)          SPEC.md:289-297   -> DirtyRegion (tight box)
//   fill_holes(grid, region, r)      SPEC.md:298-306   -> filled voxel count
//   run_incremental(...)             SPEC.md:307-315   -> per-frame latency p50/p95/max
//   coronal_projection(grid, mode)
//   VoxelGrid::render_depth_band     BASELINE cfg4 depth-band coronal render
//
// Errors: codes from the C-ABI become exceptions.  Define SPINEVOL_B200_REFERENCE_TYPES before
// including this header (with the reference's proj/include on the include path) to get
// overloads taking spinevol::Image8 / RigidTransform / ImageCalibration / TimedPose and throwing
// spinevol::InvalidInput / AlgorithmFailure / IoError (core.hpp:14-32) — the drop-in form.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../spinevol_b200.h"

#ifdef SPINEVOL_B200_REFERENCE_TYPES
#include "spinevol/core.hpp"
#include "spinevol/geometry.hpp"
#include "spinevol/image.hpp"
#endif

namespace spinevol_b200 {

#ifdef SPINEVOL_B200_REFERENCE_TYPES
using Error = spinevol::Error;
using InvalidInput = spinevol::InvalidInput;
using AlgorithmFailure = spinevol::AlgorithmFailure;
using IoError = spinevol::IoError;
#else
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidInput : Error {
    explicit InvalidInput(const std::string& m) : Error(m) {}
};
struct AlgorithmFailure : Error {
    explicit AlgorithmFailure(const std::string& m) : Error(m) {}
};
struct IoError : Error {
    explicit IoError(const std::string& m) : Error(m) {}
};
#endif
// device / NCCL failures have no reference counterpart (the reference is CPU-only)
struct DeviceError : Error {
    explicit DeviceError(const std::string& m) : Error(m) {}
};

inline void check(int rc) {
    if (rc == SVR_OK) return;
    const std::string m = svr_last_error();
    switch (rc) {
        case SVR_E_INVALID: throw InvalidInput(m);
        case SVR_E_ALGO: throw AlgorithmFailure(m);
        case SVR_E_IO: throw IoError(m);
        default: throw DeviceError(m);
    }
}

// DirtyRegion: inclusive voxel box, empty iff x0 > x1.
struct DirtyRegion {
    svr_box b{1, 1, 1, 0, 0, 0};
    bool empty() const { return b.x0 > b.x1; }
    DirtyRegion dilated(int r) const {
        if (empty()) return *this;
        return DirtyRegion{{b.x0 - r, b.y0 - r, b.z0 - r, b.x1 + r, b.y1 + r, b.z1 + r}};
    }
    DirtyRegion& operator|=(const DirtyRegion& o) {
        if (o.empty()) return *this;
        if (empty()) return *this = o;
        b = {std::min(b.x0, o.b.x0), std::min(b.y0, o.b.y0), std::min(b.z0, o.b.z0),
             std::max(b.x1, o.b.x1), std::max(b.y1, o.b.y1), std::max(b.z1, o.b.z1)};
        return *this;
    }
};

struct GridConfig {
    int nx = 0, ny = 0, nz = 0;
    double voxel_mm = 1.0;  // SPEC.md:277 default
    double origin_mm[3] = {0, 0, 0};
    int z_begin = 0, z_end = -1;  // stored slab; -1 = whole grid
    int accum = SVR_ACC_PNN;
};

class VoxelGrid {
public:
    explicit VoxelGrid(const GridConfig& c, int device = 0) {
        svr_grid_desc d{};
        d.nx = c.nx;
        d.ny = c.ny;
        d.nz = c.nz;
        d.accum = c.accum;
        d.voxel_mm = c.voxel_mm;
        for (int k = 0; k < 3; ++k) d.origin_mm[k] = c.origin_mm[k];
        d.z_begin = c.z_begin;
        d.z_end = c.z_end < 0 ? c.nz : c.z_end;
        check(svr_create(&d, device, &h_));
        desc_ = d;
    }
    ~VoxelGrid() { svr_destroy(h_); }
    VoxelGrid(const VoxelGrid&) = delete;
    VoxelGrid& operator=(const VoxelGrid&) = delete;
    VoxelGrid(VoxelGrid&& o) noexcept : h_(std::exchange(o.h_, nullptr)), desc_(o.desc_) {}

    svr_volume* handle() const { return h_; }
    const svr_grid_desc& desc() const { return desc_; }
    void set_stream(void* cuda_stream) { check(svr_set_stream(h_, cuda_stream)); }
    void clear() { check(svr_clear(h_)); }
    void sync() { check(svr_sync(h_)); }

    // insert_frame: one row-major u8 frame (host or device memory)
    DirtyRegion insert_frame(const uint8_t* px, int64_t row_pitch, int w, int h, const svr_rigid& pose,
                             const svr_calib& calib, bool skip_zero = false) {
        DirtyRegion r;
        check(svr_insert_frame(h_, px, row_pitch, w, h, &pose, &calib, skip_zero ? 1 : 0, &r.b));
        return r;
    }
    // batched insert; returns the union dirty region (synchronising) when want_region
    DirtyRegion insert_frames(const uint8_t* px, int64_t row_pitch, int64_t frame_stride, int w, int h,
                              int n, const svr_rigid* poses, const svr_calib& calib,
                              bool skip_zero = false, bool want_region = true) {
        DirtyRegion u;
        check(svr_insert_frames(h_, px, row_pitch, frame_stride, w, h, n, poses, &calib,
                                skip_zero ? 1 : 0, nullptr, want_region ? &u.b : nullptr));
        return u;
    }
    // fill_holes over exactly `region`
    int64_t fill_holes(const DirtyRegion& region, int radius = 2, int mode = SVR_FILL_MEDIAN) {
        int64_t n = 0;
        check(svr_fill_holes(h_, &region.b, mode, radius, &n));
        return n;
    }
    int64_t fill_all(int radius = 2, int mode = SVR_FILL_MEDIAN) {
        int64_t n = 0;
        check(svr_fill_holes(h_, nullptr, mode, radius, &n));
        return n;
    }
    // depth-band coronal render (BASELINE cfg4), incremental over `dirty` (empty = all columns)
    void render_depth_band(const svr_render_params& p, const DirtyRegion* dirty = nullptr,
                           int fill_radius = 1) {
        check(svr_render_coronal(h_, dirty ? &dirty->b : nullptr, fill_radius, &p));
    }
    void read_depth_band(std::vector<float>& mean, std::vector<float>& maxv, std::vector<int32_t>& depth) {
        const size_t n = (size_t)desc_.nx * (desc_.z_end - desc_.z_begin);
        mean.resize(n);
        maxv.resize(n);
        depth.resize(n);
        check(svr_read_coronal(h_, desc_.z_begin, desc_.z_end - 1, mean.data(), maxv.data(), depth.data()));
    }
    // coronal_projection
    std::vector<uint8_t> coronal_projection(int mode = SVR_PROJ_MAX, int depth_axis = 2,
                                            bool use_fills = false) {
        const int dims[3] = {desc_.nx, desc_.ny, desc_.z_end - desc_.z_begin};
        size_t n = 1;
        for (int a = 0; a < 3; ++a)
            if (a != depth_axis) n *= (size_t)dims[a];
        std::vector<uint8_t> out(n);
        check(svr_coronal_projection(h_, mode, depth_axis, use_fills ? 1 : 0, out.data()));
        return out;
    }
    void accumulators(std::vector<uint32_t>& sum, std::vector<uint16_t>& count) {
        const size_t n = (size_t)desc_.nx * desc_.ny * (desc_.z_end - desc_.z_begin);
        sum.resize(n);
        count.resize(n);
        check(svr_read_accumulators(h_, nullptr, sum.data(), count.data()));
    }
    // VoxelGrid::value
    std::vector<uint8_t> values(bool apply_fills = false) {
        std::vector<uint8_t> out((size_t)desc_.nx * desc_.ny * (desc_.z_end - desc_.z_begin));
        check(svr_read_values(h_, nullptr, apply_fills ? 1 : 0, out.data()));
        return out;
    }
    svr_stats stats() {
        svr_stats s{};
        check(svr_get_stats(h_, &s));
        return s;
    }
    // one incremental frame (insert -> mean fill of box (+) 1 -> render) as a CUDA-graph replay
    DirtyRegion frame_step(const uint8_t* px, int64_t row_pitch, const svr_rigid& pose,
                           const svr_calib& calib, const svr_render_params& p, int fill_radius = 1) {
        DirtyRegion r;
        check(svr_frame_step(h_, px, row_pitch, &pose, &calib, fill_radius, &p, &r.b));
        return r;
    }
    // volume file: raw u8 values, x fastest
    void export_volume(const std::string& path, bool apply_fills = true) {
        check(svr_export_volume(h_, path.c_str(), apply_fills ? 1 : 0));
    }
    // export_slices along x: returns the file count
    int export_slices(const std::string& dir, bool apply_fills = true, int digits = 4) {
        int32_t n = 0;
        check(svr_export_slices(h_, dir.c_str(), apply_fills ? 1 : 0, digits, &n));
        return n;
    }
    DirtyRegion frame_bounds(const svr_calib& calib, const svr_rigid& pose) const {
        DirtyRegion r;
        check(svr_frame_bounds(&desc_, &calib, &pose, &r.b));
        return r;
    }

private:
    svr_volume* h_ = nullptr;
    svr_grid_desc desc_{};
};

// z-slab sharded volume over several devices driven from one thread (svr_sharded_*, SURVEY.md
// §8e): routing, ghost planes and the fused coronal gather happen inside; bit-identical to one
// VoxelGrid.  devices may repeat (several slabs on one GPU).
class ShardedVolume {
public:
    ShardedVolume(const GridConfig& c, const std::vector<int32_t>& devices, int ghost = 3) {
        svr_grid_desc d{};
        d.nx = c.nx;
        d.ny = c.ny;
        d.nz = c.nz;
        d.accum = c.accum;
        d.voxel_mm = c.voxel_mm;
        for (int k = 0; k < 3; ++k) d.origin_mm[k] = c.origin_mm[k];
        d.z_begin = 0;
        d.z_end = c.nz;
        check(svr_sharded_create(&d, devices.data(), (int32_t)devices.size(), ghost, &h_));
        desc_ = d;
        n_ = (int)devices.size();
    }
    ~ShardedVolume() { svr_sharded_destroy(h_); }
    ShardedVolume(const ShardedVolume&) = delete;
    ShardedVolume& operator=(const ShardedVolume&) = delete;

    int slabs() const { return n_; }
    // (handle, owned [z0, z1), stored [z0, z1)) of slab r
    svr_volume* slab(int r, int32_t* own0 = nullptr, int32_t* own1 = nullptr) const {
        svr_volume* v = nullptr;
        check(svr_sharded_slab(h_, r, &v, own0, own1, nullptr, nullptr));
        return v;
    }
    // batched insert routed to the slabs; returns the frames each slab took
    std::vector<int32_t> insert_frames(const uint8_t* px, int64_t row_pitch, int64_t frame_stride, int w,
                                       int h, int n, const svr_rigid* poses, const svr_calib& calib,
                                       bool skip_zero = false) {
        std::vector<int32_t> routed((size_t)n_);
        check(svr_sharded_insert_frames(h_, px, row_pitch, frame_stride, w, h, n, poses, &calib,
                                        skip_zero ? 1 : 0, routed.data()));
        return routed;
    }
    void fill_render(const svr_render_params& p, int fill_radius = 1, int fill_mode = SVR_FILL_MEAN) {
        check(svr_sharded_fill_render(h_, fill_radius, fill_mode, &p));
    }
    void read_coronal(std::vector<float>& mean, std::vector<float>& maxv, std::vector<int32_t>& depth) {
        const size_t n = (size_t)desc_.nx * desc_.nz;
        mean.resize(n);
        maxv.resize(n);
        depth.resize(n);
        check(svr_sharded_read_coronal(h_, mean.data(), maxv.data(), depth.data()));
    }
    // owned planes of every slab, concatenated in z: the whole grid's accumulators
    void accumulators(std::vector<uint32_t>& sum, std::vector<uint16_t>& count) {
        const size_t plane = (size_t)desc_.nx * desc_.ny;
        sum.assign(plane * desc_.nz, 0);
        count.assign(plane * desc_.nz, 0);
        for (int r = 0; r < n_; ++r) {
            int32_t o0 = 0, o1 = 0;
            svr_volume* v = slab(r, &o0, &o1);
            if (o1 <= o0) continue;
            svr_box b{0, 0, o0, desc_.nx - 1, desc_.ny - 1, o1 - 1};
            check(svr_read_accumulators(v, &b, sum.data() + plane * o0, count.data() + plane * o0));
        }
    }

private:
    svr_sharded* h_ = nullptr;
    svr_grid_desc desc_{};
    int n_ = 0;
};

inline DirtyRegion insert_frame(VoxelGrid& g, const uint8_t* px, int w, int h, const svr_rigid& pose,
                                const svr_calib& calib, bool skip_zero = false) {
    return g.insert_frame(px, w, w, h, pose, calib, skip_zero);
}

inline int64_t fill_holes(VoxelGrid& g, const DirtyRegion& region, int radius = 2) {
    return g.fill_holes(region, radius, SVR_FILL_MEDIAN);
}

inline std::vector<uint8_t> coronal_projection(VoxelGrid& g, int mode = SVR_PROJ_MAX) {
    return g.coronal_projection(mode);
}

struct IncrementalStats {
    svr_stats counters{};
    double latency_ms_p50 = 0, latency_ms_p95 = 0, latency_ms_max = 0;
};

// run_incremental: per frame insert -> fill(dirty (+) r) -> optional render.
// The fill/render region is the host-side conservative frame box (a superset of the tight box),
// so no device round trip per frame; the final state equals batch processing bit-for-bit.
inline IncrementalStats run_incremental(VoxelGrid& g, const uint8_t* frames, int w, int h, int n,
                                        const svr_rigid* poses, const svr_calib& calib,
                                        int hole_radius = 1, int fill_mode = SVR_FILL_MEAN,
                                        const svr_render_params* render = nullptr,
                                        bool skip_zero = false) {
    std::vector<double> lat;
    lat.reserve((size_t)n);
    const bool graph = render && hole_radius == 1 && fill_mode == SVR_FILL_MEAN && !skip_zero;
    for (int k = 0; k < n; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        if (graph) {  // the per-frame step as one CUDA-graph replay
            g.frame_step(frames + (size_t)k * w * h, w, poses[k], calib, *render, 1);
            g.sync();
            lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            continue;
        }
        check(svr_insert_frames(g.handle(), frames + (size_t)k * w * h, w, (int64_t)w * h, w, h, 1,
                                poses + k, &calib, skip_zero ? 1 : 0, nullptr, nullptr));
        const DirtyRegion b = g.frame_bounds(calib, poses[k]);
        if (!b.empty()) {
            const DirtyRegion f = b.dilated(hole_radius);
            check(svr_fill_holes(g.handle(), &f.b, fill_mode, hole_radius, nullptr));
            if (render) check(svr_render_coronal(g.handle(), &b.b, hole_radius, render));
        }
        g.sync();
        lat.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    IncrementalStats st;
    st.counters = g.stats();
    if (!lat.empty()) {
        // percentile as core.hpp:101-107 (nearest rank on the sorted sample)
        auto pct = [&](double p) {
            std::vector<double> v = lat;
            size_t k = (size_t)(p * (double)(v.size() - 1) + 0.5);
            std::nth_element(v.begin(), v.begin() + (std::ptrdiff_t)k, v.end());
            return v[k];
        };
        st.latency_ms_p50 = pct(0.5);
        st.latency_ms_p95 = pct(0.95);
        st.latency_ms_max = *std::max_element(lat.begin(), lat.end());
    }
    return st;
}

// ---- binary PGM (image.hpp:34-72) through the native reader/writer
struct Image {
    int width = 0, height = 0;
    std::vector<uint8_t> data;  // row-major
};

inline Image read_pgm(const std::string& path) {
    Image img;
    int32_t w = 0, h = 0;
    check(svr_pgm_info(path.c_str(), &w, &h));
    img.width = w;
    img.height = h;
    img.data.resize((size_t)w * h);
    check(svr_pgm_read(path.c_str(), img.data.data(), std::max(w, 1), w, h));
    return img;
}

inline void write_pgm(const uint8_t* px, int w, int h, const std::string& path) {
    check(svr_pgm_write(path.c_str(), px, std::max(w, 1), w, h));
}

// ---- segmentation host halves (SPEC.md segment module)
inline double cut_depth_alg1(double p_c1, double p_cn, double K, double D, double L, double axial_extent_mm) {
    double c = 0;
    check(svr_cut_depth_alg1(p_c1, p_cn, K, D, L, axial_extent_mm, &c));
    return c;
}

inline std::vector<double> smooth_depths(const std::vector<double>& depths, const std::vector<uint8_t>& valid,
                                         int window = 11) {
    if (depths.size() != valid.size()) throw InvalidInput("depths / valid size mismatch");
    std::vector<double> out(depths.size());
    check(svr_smooth_depths(depths.data(), valid.data(), (int32_t)depths.size(), window, out.data()));
    return out;
}

#ifdef SPINEVOL_B200_REFERENCE_TYPES
// ---- drop-in overloads on the reference's own value types (geometry.hpp, image.hpp)
inline spinevol::Image8 read_pgm_image8(const std::string& path) {
    Image i = read_pgm(path);
    spinevol::Image8 img(i.width, i.height);
    img.data = std::move(i.data);
    return img;
}
inline svr_rigid to_svr(const spinevol::RigidTransform& t) {
    return svr_rigid{t.rotation.w, t.rotation.x, t.rotation.y, t.rotation.z,
                     t.translation.x, t.translation.y, t.translation.z};
}

inline svr_calib to_svr(const spinevol::ImageCalibration& c) {
    svr_calib k{};
    k.crop_x = c.crop_rect.x;
    k.crop_y = c.crop_rect.y;
    k.crop_w = c.crop_rect.w;
    k.crop_h = c.crop_rect.h;
    k.scale_x_mm = c.scale_x_mm;
    k.scale_y_mm = c.scale_y_mm;
    k.image_to_transducer = to_svr(c.image_to_transducer);
    k.latency_ms = c.latency_ms;
    k.probe = SVR_PROBE_LINEAR;
    return k;
}

// insert_frame(grid, frame, pose, calib, skip_zero) -> DirtyRegion
inline DirtyRegion insert_frame(VoxelGrid& g, const spinevol::Image8& frame,
                                const spinevol::RigidTransform& pose,
                                const spinevol::ImageCalibration& calib, bool skip_zero = false) {
    calib.validate();
    if (frame.width != calib.crop_rect.w || frame.height != calib.crop_rect.h)
        throw spinevol::InvalidInput("frame dims do not match calib crop_rect");
    return g.insert_frame(frame.data.data(), frame.width, frame.width, frame.height, to_svr(pose),
                          to_svr(calib), skip_zero);
}

inline DirtyRegion insert_frame(VoxelGrid& g, const spinevol::Image8& frame,
                                const spinevol::TimedPose& pose,
                                const spinevol::ImageCalibration& calib, bool skip_zero = false) {
    return insert_frame(g, frame, pose.transform, calib, skip_zero);
}
#endif

}  // namespace spinevol_b200
