// wrapper_demo.cpp — drives the C++ host API (include/spinevol_b200/reconstruct.hpp) the way a
// reference caller would: per-frame insert_frame -> fill_holes on the dilated dirty region ->
// coronal_projection.  Test harness for tests/test_cpp_host.py.
//   wrapper_demo host                     host-only checks (no GPU needed)
//   wrapper_demo run IN OUT               reconstruct IN (see test_cpp_host.py) -> OUT
// Built with -DSPINEVOL_B200_REFERENCE_TYPES (+ the reference's include dir) it takes the
// reference's own spinevol::Image8 / RigidTransform / ImageCalibration.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "spinevol_b200/reconstruct.hpp"

namespace sb = spinevol_b200;

static int host_checks() {
    svr_calib c{};
    c.crop_w = 512;
    c.crop_h = 512;
    c.scale_x_mm = c.scale_y_mm = 0.1;
    c.image_to_transducer = svr_rigid{1, 0, 0, 0, 5, 0, 0};
    svr_rigid id{1, 0, 0, 0, 0, 0, 0};
    double w[3];
    sb::check(svr_pixel_to_world(100, 200, &c, &id, w));
    if (!(w[0] == 15.0 && w[1] == 20.0 && w[2] == 0.0)) return 1;
    try {
        sb::check(svr_pixel_to_world(512, 0, &c, &id, w));
        return 2;
    } catch (const sb::InvalidInput&) {
    }
    if (svr_device_count() == 0) {
        try {
            sb::VoxelGrid g(sb::GridConfig{8, 8, 8});
            return 3;
        } catch (const sb::DeviceError&) {
        }
    }
#ifdef SPINEVOL_B200_REFERENCE_TYPES
    // the reference's own types flow through the adapters unchanged
    spinevol::ImageCalibration rc;
    rc.crop_rect = {0, 0, 512, 512};
    rc.scale_x_mm = rc.scale_y_mm = 0.1;
    rc.image_to_transducer = spinevol::RigidTransform::translate(5, 0, 0);
    svr_calib k = sb::to_svr(rc);
    sb::check(svr_pixel_to_world(100, 200, &k, &id, w));
    spinevol::Vec3 ref = spinevol::pixel_to_world(100, 200, rc, spinevol::RigidTransform::identity());
    if (!(w[0] == ref.x && w[1] == ref.y && w[2] == ref.z)) return 4;
#endif
    // PGM round trip and the segmentation host halves (no GPU needed)
    {
        std::vector<uint8_t> img(37 * 21);
        for (size_t i = 0; i < img.size(); ++i) img[i] = (uint8_t)(i * 7);
        const std::string path = "/tmp/svr_wrapper_demo.pgm";
        sb::write_pgm(img.data(), 37, 21, path);
        sb::Image back = sb::read_pgm(path);
        if (back.width != 37 || back.height != 21 || back.data != img) return 5;
#ifdef SPINEVOL_B200_REFERENCE_TYPES
        spinevol::Image8 ri = spinevol::read_pgm(path);  // the reference's own reader agrees
        if (ri.data != img) return 6;
#endif
        if (sb::cut_depth_alg1(100.0, 100.0, 0.04, 35.0, 500.0, 60.0) != 45.0) return 7;
        std::vector<double> d{35, 35, 80, 35, 35};
        std::vector<uint8_t> v(5, 1);
        for (double x : sb::smooth_depths(d, v, 5))
            if (x != 35.0) return 8;
        try {
            sb::read_pgm("/nonexistent/x.pgm");
            return 9;
        } catch (const sb::IoError&) {
        }
    }
    std::puts("host ok");
    return 0;
}

// IN layout (little endian): i32 nx ny nz nframes w h; f64 voxel, origin[3]; svr_calib;
// nframes * svr_rigid; nframes*w*h u8.  OUT: u32 sum[], u16 count[], u32 fill[], u8 proj[].
static int run(const char* in, const char* out) {
    std::ifstream f(in, std::ios::binary);
    int32_t hdr[6];
    double vox, org[3];
    svr_calib calib{};
    f.read((char*)hdr, sizeof hdr);
    f.read((char*)&vox, 8);
    f.read((char*)org, 24);
    f.read((char*)&calib, sizeof calib);
    const int n = hdr[3], w = hdr[4], h = hdr[5];
    std::vector<svr_rigid> poses((size_t)n);
    std::vector<uint8_t> px((size_t)n * w * h);
    f.read((char*)poses.data(), sizeof(svr_rigid) * n);
    f.read((char*)px.data(), (std::streamsize)px.size());
    if (!f) return 10;
    sb::GridConfig gc{hdr[0], hdr[1], hdr[2], vox, {org[0], org[1], org[2]}};
    sb::VoxelGrid g(gc, 0);
    sb::DirtyRegion all;
    for (int k = 0; k < n; ++k) {
#ifdef SPINEVOL_B200_REFERENCE_TYPES
        spinevol::Image8 img(w, h);
        std::memcpy(img.data.data(), px.data() + (size_t)k * w * h, (size_t)w * h);
        spinevol::RigidTransform pose;
        pose.rotation = {poses[k].qw, poses[k].qx, poses[k].qy, poses[k].qz};
        pose.translation = {poses[k].tx, poses[k].ty, poses[k].tz};
        spinevol::ImageCalibration rc;
        rc.crop_rect = {0, 0, w, h};
        rc.scale_x_mm = calib.scale_x_mm;
        rc.scale_y_mm = calib.scale_y_mm;
        const svr_rigid& t = calib.image_to_transducer;
        rc.image_to_transducer.rotation = {t.qw, t.qx, t.qy, t.qz};
        rc.image_to_transducer.translation = {t.tx, t.ty, t.tz};
        all |= sb::insert_frame(g, img, pose, rc);
#else
        all |= sb::insert_frame(g, px.data() + (size_t)k * w * h, w, h, poses[k], calib);
#endif
    }
    g.fill_holes(all.dilated(2), 2, SVR_FILL_MEDIAN);
    std::vector<uint32_t> sum;
    std::vector<uint16_t> cnt;
    g.accumulators(sum, cnt);
    std::vector<uint32_t> fill(sum.size());
    sb::check(svr_read_fill(g.handle(), nullptr, fill.data()));
    std::vector<uint8_t> proj = sb::coronal_projection(g, SVR_PROJ_MAX);
    std::ofstream o(out, std::ios::binary);
    o.write((char*)sum.data(), (std::streamsize)(sum.size() * 4));
    o.write((char*)cnt.data(), (std::streamsize)(cnt.size() * 2));
    o.write((char*)fill.data(), (std::streamsize)(fill.size() * 4));
    o.write((char*)proj.data(), (std::streamsize)proj.size());
    std::puts("run ok");
    return o ? 0 : 11;
}

// Same input, reconstructed by a z-slab sharded volume of `nslab` slabs (all on device 0 here;
// the same code drives one slab per GPU): OUT = u32 sum[], u16 count[], f32 mean[], f32 max[],
// i32 depth[] (coronal image nz x nx, cfg4 render parameters).
static int shard(const char* in, const char* out, int nslab) {
    std::ifstream f(in, std::ios::binary);
    int32_t hdr[6];
    double vox, org[3];
    svr_calib calib{};
    f.read((char*)hdr, sizeof hdr);
    f.read((char*)&vox, 8);
    f.read((char*)org, 24);
    f.read((char*)&calib, sizeof calib);
    const int n = hdr[3], w = hdr[4], h = hdr[5];
    std::vector<svr_rigid> poses((size_t)n);
    std::vector<uint8_t> px((size_t)n * w * h);
    f.read((char*)poses.data(), sizeof(svr_rigid) * n);
    f.read((char*)px.data(), (std::streamsize)px.size());
    if (!f) return 10;
    sb::GridConfig gc{hdr[0], hdr[1], hdr[2], vox, {org[0], org[1], org[2]}};
    svr_render_params rp{15.0, 60.0, 5.0, 2.0, 2, SVR_FILL_MEAN};
    sb::ShardedVolume sv(gc, std::vector<int32_t>((size_t)nslab, 0), 1 + rp.median_radius);
    sv.insert_frames(px.data(), w, (int64_t)w * h, w, h, n, poses.data(), calib);
    sv.fill_render(rp, 1, SVR_FILL_MEAN);
    std::vector<uint32_t> sum;
    std::vector<uint16_t> cnt;
    sv.accumulators(sum, cnt);
    std::vector<float> mean, maxv;
    std::vector<int32_t> depth;
    sv.read_coronal(mean, maxv, depth);
    std::ofstream o(out, std::ios::binary);
    o.write((char*)sum.data(), (std::streamsize)(sum.size() * 4));
    o.write((char*)cnt.data(), (std::streamsize)(cnt.size() * 2));
    o.write((char*)mean.data(), (std::streamsize)(mean.size() * 4));
    o.write((char*)maxv.data(), (std::streamsize)(maxv.size() * 4));
    o.write((char*)depth.data(), (std::streamsize)(depth.size() * 4));
    std::puts("shard ok");
    return o ? 0 : 11;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && !std::strcmp(argv[1], "host")) return host_checks();
        if (argc >= 4 && !std::strcmp(argv[1], "run")) return run(argv[2], argv[3]);
        if (argc >= 5 && !std::strcmp(argv[1], "shard")) return shard(argv[2], argv[3], std::atoi(argv[4]));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 20;
    }
    std::fprintf(stderr, "usage: wrapper_demo host | run IN OUT | shard IN OUT NSLAB\n");
    return 2;
}
