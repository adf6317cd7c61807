// svr_api.cu — host side of the C-ABI (include/spinevol_b200.h): per-frame pose prep,
// staging of host frames through a pinned double-buffered ring, kernel dispatch, readout.
// No C++ exception crosses the boundary; errors are codes + thread-local messages.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "svr_host.hpp"
#include "svr_kernels.cuh"
#include "svr_k1.cuh"
#include "svr_fan.cuh"

using namespace svr;

static thread_local std::string g_err;

// NVTX range over a C-ABI call (header-only NVTX3: free unless a profiler is attached), so
// nsys / ncu range filters see insert / fill / render / frame_step by name.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int svr_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return fail(SVR_E_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_),   \
                        __FILE__, __LINE__);                                               \
    } while (0)

#define CKL()                                                                              \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            return fail(SVR_E_CUDA, "kernel launch failed: %s (%s:%d)",                    \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

// Per-frame incremental pipeline (svr_frame_step) captured once as a CUDA graph: frame copy,
// parameter and region-table uploads from pinned staging, insert, fill of the conservative dirty
// box (+) r, depth + band render of its columns.  Grid sizes are captured as upper bounds (the
// kernels retire surplus CTAs), so one graph replays for every frame of a sweep.
struct FrameGraph {
    bool ready = false;
    int w = 0, h = 0, fr = -1;
    svr_calib cal{};
    svr_render_params rp{};
    long long fill_ctas = 0, depth_ctas = 0, band_ctas = 0;
    uint8_t* d_frame = nullptr;
    uint8_t* h_frame = nullptr;      // pinned staging for pageable / pitched host frames
    FrameParams* h_fp = nullptr;     // pinned
    FrameParams* d_fp = nullptr;
    unsigned char* h_tiles = nullptr;  // pinned: BoxTiles | ColTiles depth | ColTiles band
    unsigned char* d_tiles = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;
    int kernels = 0;
    int shape = -1;        // k_pnn_tiles shape of the captured insert (-1: none)
    uint64_t captures = 0; // graph (re-)captures so far
};

struct svr_volume {
    svr_grid_desc d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    cudaStream_t own_stream_saved = nullptr;  // the handle's own stream while svr_use_stream lends another
    cudaStream_t copy_stream = nullptr;
    long long nvox = 0;
    ull* acc = nullptr;
    float2* tri = nullptr;
    uint32_t* fill = nullptr;
    int* r_depth = nullptr;
    int* r_mdepth = nullptr;
    float* r_mean = nullptr;
    float* r_max = nullptr;
    ull* d_stats = nullptr;  // kStCount counters
    ull* d_counter = nullptr;
    // per-frame parameter staging
    // double-buffered host side: the next call fills one pinned buffer while the previous
    // call's upload from the other is still queued behind that call's kernels
    FrameParams* h_params[2] = {nullptr, nullptr};
    FrameParams* d_params = nullptr;            // = d_params2[pslot] during an insert call
    FrameParams* d_params2[2] = {nullptr, nullptr};
    cudaStream_t param_stream = nullptr;         // the parameter upload, off the kernels' stream
    cudaEvent_t params_used[2] = {nullptr, nullptr};  // last kernel reading d_params2[i] done
    cudaEvent_t ins_done = nullptr;   // the last insert call's kernels done (param_stream waits)
    cudaEvent_t ev_prep = nullptr;    // param_stream's share of the current call done
    cudaEvent_t ev_tiles_up = nullptr;  // upload_tiles' H2D on param_stream done
    bool prep_on_param = false;       // insert_common: K1's per-tile setup goes to param_stream
    int params_cap = 0;
    int pslot = 0;
    cudaEvent_t params_ev[2] = {nullptr, nullptr};
    int* d_boxes = nullptr;
    int* h_boxes = nullptr;
    int boxes_cap = 0;
    // host-frame staging ring
    size_t stage_bytes = 0;
    uint8_t* h_stage[2] = {nullptr, nullptr};
    uint8_t* d_stage[2] = {nullptr, nullptr};
    cudaEvent_t ev_ready[2] = {nullptr, nullptr};
    cudaEvent_t ev_free[2] = {nullptr, nullptr};
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr};
    // fan table
    double2* d_fan = nullptr;
    int fan_lines = 0;
    double fan_angle = 0.0;
    uint64_t launches = 0;
    uint64_t frames = 0;
    ull* d_work = nullptr;          // deferred exact-path chunks (k_pnn_tiles / k_fan_tiles / k_pnn_plane)
    FrameGraph fg;                  // svr_frame_step graph
    GatherTargets gt{nullptr, 0, 0, 0, 0};  // fused render + gather targets (device pointer array)
    float** d_gt = nullptr;
    // region tables of the multi-box fill / render launches: a ring of pinned staging + device
    // slots, so an upload never blocks the host behind queued work (a pageable copy would: it
    // serialised the overlapped sweep's host thread with the fill / render stream)
    static constexpr int kTileSlots = 4;
    void* d_tiles[kTileSlots] = {};
    void* h_tiles[kTileSlots] = {};
    cudaEvent_t tiles_ev[kTileSlots] = {};
    int tiles_prev = -1;
    cudaStream_t tiles_prev_stream = nullptr;
    size_t tiles_cap = 0;
    unsigned int* d_work_n = nullptr;
    unsigned int work_cap = 0;
    int tri_kernel = 0;         // SVR_TRI_KERNEL=chunk: trilinear splat through k_insert (cross-check)
    int insert_kernel = 3;      // SVR_INSERT_KERNEL=direct: every PNN insert through k_insert (the
                                // fallback kernel; tests use it to cover it on every geometry)
    int lin_shapes_cur = 0;     // k_pnn_tiles shapes every frame of the current insert call fits
    int tiles_occ[32] = {0};    // k_pnn_tiles resident CTAs per SM, per <shape, box, z1, skip> (lazy)
    TileDesc* d_desc = nullptr; // k_pnn_tiles per-tile descriptors
    long long desc_cap = 0;
    TileFrame* d_frc = nullptr; // k_pnn_tiles per-frame constants
    long long frc_cap = 0;
    int num_sms = 148;          // the device's SM count (grid sizing)
    FanDesc* d_fdesc = nullptr; // k_fan_tiles per-tile descriptors
    long long fdesc_cap = 0;
    FanRow* d_frows = nullptr;  // k_fan_tiles per-scanline constants
    long long frows_cap = 0;
    int fan_occ[2] = {0, 0};    // k_fan_tiles resident CTAs per SM, per <box> (lazy)
    int fill_mode = SVR_FILL_MEAN;  // mode of the latest fill_holes: decodes the fill layer on readout
};

// ---------------------------------------------------------------- host geometry (exact)
// Rotation of Quat::rotate (geometry.hpp:44-49) as the linear map it computes in real
// arithmetic, M = I + 2w[u]x + 2(u u^T - |u|^2 I), evaluated in double.
static void quat_mat(const svr_rigid& q, double M[9]) {
    const double w = q.qw, x = q.qx, y = q.qy, z = q.qz;
    const double n2 = x * x + y * y + z * z;
    M[0] = 1 + 2 * (x * x - n2);
    M[1] = 2 * (x * y) - 2 * w * z;
    M[2] = 2 * (x * z) + 2 * w * y;
    M[3] = 2 * (y * x) + 2 * w * z;
    M[4] = 1 + 2 * (y * y - n2);
    M[5] = 2 * (y * z) - 2 * w * x;
    M[6] = 2 * (z * x) - 2 * w * y;
    M[7] = 2 * (z * y) + 2 * w * x;
    M[8] = 1 + 2 * (z * z - n2);
}

static void mat_mul(const double A[9], const double B[9], double C[9]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

struct Affine {  // u = K + Mv * p, voxel units (no +1/2)
    double Mv[9];
    double K[3];
};

// Fan scanline directions (pin identical to oracle/svr_oracle.c orc_fan_table).
static void fan_table(const svr_calib& c, std::vector<double>& s, std::vector<double>& co) {
    const int L = c.crop_h;
    const double A = c.fan_angle_deg;
    s.resize(L);
    co.resize(L);
    for (int i = 0; i < L; ++i) {
        double deg = -0.5 * A + A * ((double)i + 0.5) / (double)L;
        double th = deg * M_PI / 180.0;
        s[i] = std::sin(th);
        co[i] = std::cos(th);
    }
}

static bool finite_rigid(const svr_rigid& r) {
    return std::isfinite(r.qw) && std::isfinite(r.qx) && std::isfinite(r.qy) &&
           std::isfinite(r.qz) && std::isfinite(r.tx) && std::isfinite(r.ty) && std::isfinite(r.tz);
}

static int check_calib(const svr_calib* c, int32_t w, int32_t h) {
    if (!c) return fail(SVR_E_INVALID, "calib is NULL");
    if (c->crop_w <= 0 || c->crop_h <= 0)
        return fail(SVR_E_INVALID, "calibration crop_rect must be non-empty");
    if (w != c->crop_w || h != c->crop_h)
        return fail(SVR_E_INVALID, "frame dims %dx%d do not match calib crop_rect %dx%d", w, h,
                    c->crop_w, c->crop_h);
    if (w > 8192 || h > 8192) return fail(SVR_E_INVALID, "frame dims above 8192 are unsupported");
    if (!finite_rigid(c->image_to_transducer))
        return fail(SVR_E_INVALID, "calibration transform not finite");
    if (c->probe == SVR_PROBE_LINEAR) {
        if (!(c->scale_x_mm > 0.0) || !(c->scale_y_mm > 0.0))
            return fail(SVR_E_INVALID, "calibration scales must be positive");
    } else if (c->probe == SVR_PROBE_FAN) {
        if (!(c->fan_r1_mm > c->fan_r0_mm) || !(c->fan_r0_mm >= 0.0) ||
            !(c->fan_angle_deg > 0.0 && c->fan_angle_deg < 180.0))
            return fail(SVR_E_INVALID, "invalid fan geometry");
    } else {
        return fail(SVR_E_INVALID, "unknown probe kind %d", c->probe);
    }
    return SVR_OK;
}

static long long to_fixed(double x, bool* ok) {
    double s = x * 4294967296.0;
    if (!(std::fabs(s) < 4.0e18)) {
        *ok = false;
        return 0;
    }
    return std::llround(s);
}

static DevCalib dev_calib(const svr_calib& c) {
    DevCalib d{};
    d.sx = c.scale_x_mm;
    d.sy = c.scale_y_mm;
    d.i2t = c.image_to_transducer;
    d.probe = c.probe;
    d.lines = c.crop_h;
    if (c.probe == SVR_PROBE_FAN) {
        d.r0 = c.fan_r0_mm;
        d.dr = (c.fan_r1_mm - c.fan_r0_mm) / (double)c.crop_w;
    }
    return d;
}

static GridDev dev_grid(const svr_grid_desc& d) {
    GridDev g{};
    g.nx = d.nx;
    g.ny = d.ny;
    g.zb = d.z_begin;
    g.nzl = d.z_end - d.z_begin;
    g.voxel = d.voxel_mm;
    for (int k = 0; k < 3; ++k) g.o[k] = d.origin_mm[k];
    return g;
}

// Pose-independent part of the per-frame map, computed once per insert call.
struct PrepCtx {
    double Mc[9];      // image_to_transducer rotation
    double tc[3];      // image_to_transducer translation (mm)
    double v;          // voxel_mm
    double o[3];       // grid origin (mm)
    double qc2;        // max(1, |q_calib|^2)
    double base_mm;    // pixel extent from the image origin + |t_calib| + |origin| (mm)
    double coef_bound; // coefficient rounding part of the tie bound, voxels
    DevCalib cal;
    GridDev g;
    bool lin_ok;       // k_pnn_tiles usable at all (linear probe, grid planes addressable)
    int lin_count_ok;  // tile shapes whose per-slot pixel count provably stays <= 4095
};

// k_pnn_tiles shapes (svr_k1.cuh): s = (NCH == 2) + 2 (NW == 2); columns 16 NCH x rows 32 NW.
// A launch's shape carries bit 2 (kShapeZ1) when every frame has at most one y and one z carry
// per chunk (FrameParams::lin_fit bit 4): the kZ1 walk variant.
constexpr int kShapeZ1 = 4, kFitZ1 = 16;
#ifndef SVR_WORK_CTAS_PER_SM
#define SVR_WORK_CTAS_PER_SM 2  // k_pnn_work grid cap (the list holds ~1 chunk per frame)
#endif
#ifndef SVR_FILL_ZC
#define SVR_FILL_ZC 32  // batch fill: planes per k_fill_warp march (fewer when the grid is small)
#endif
#ifndef SVR_DEPTH_SEG
#define SVR_DEPTH_SEG 2  // batch render: threads per (x, z) column of k_depth (A/B: 2 beat 4 and 8)
#endif
#ifndef SVR_FILL_TY
#define SVR_FILL_TY 6  // batch fill: rows per warp of k_fill_warp (A/B: 6 rows at 6 CTAs/SM beat 4, 5, 7, 8)
#endif

static inline int shape_cols(int s) { return (s & 1) ? 32 : 64; }
static inline int shape_rows(int s) { return (s & 2) ? 64 : 128; }

// Bit s set when every tile of shape s of this frame keeps its voxel footprint inside the
// shared table (X <= 32 columns, Y <= 62 rows: X = floor(max) - floor(min) + 1 <= floor(span) + 2)
// and every step is below one voxel (one carry per axis and pixel).
static int tile_shapes_fit(const long long Dc[3], const long long Dr[3], int count_ok) {
    const double s = 1.0 / 4294967296.0;
    int m = 0;
    for (int k = 0; k < 3; ++k)
        if (std::llabs(Dc[k]) >= (1ll << 32)) return 0;
    for (int sh = 0; sh < 4; ++sh) {
        if (!((count_ok >> sh) & 1)) continue;
        const double c1 = shape_cols(sh) - 1, r1 = shape_rows(sh) - 1;
        const double spx = (c1 * std::fabs((double)Dc[0]) + r1 * std::fabs((double)Dr[0])) * s;
        const double spy = (c1 * std::fabs((double)Dc[1]) + r1 * std::fabs((double)Dr[1])) * s;
        if (std::floor(spx + 1e-9) + 2 <= 32 && std::floor(spy + 1e-9) + 2 <= 62) m |= 1 << sh;
    }
    return m;
}

static double norm3(double a, double b, double c) { return std::sqrt(a * a + b * b + c * c); }

static PrepCtx prep_ctx(const svr_calib& c, const svr_grid_desc& g) {
    PrepCtx x;
    quat_mat(c.image_to_transducer, x.Mc);
    x.tc[0] = c.image_to_transducer.tx;
    x.tc[1] = c.image_to_transducer.ty;
    x.tc[2] = c.image_to_transducer.tz;
    x.v = g.voxel_mm;
    for (int k = 0; k < 3; ++k) x.o[k] = g.origin_mm[k];
    const svr_rigid& q = c.image_to_transducer;
    x.qc2 = std::max(1.0, q.qw * q.qw + q.qx * q.qx + q.qy * q.qy + q.qz * q.qz);
    const double ext = c.probe == SVR_PROBE_FAN
                           ? c.fan_r1_mm
                           : std::hypot((double)c.crop_w * c.scale_x_mm, (double)c.crop_h * c.scale_y_mm);
    x.base_mm = ext + norm3(x.tc[0], x.tc[1], x.tc[2]) + norm3(x.o[0], x.o[1], x.o[2]);
    // 32.32 rounding of K + 1/2, Dc, Dr (2^-33 each) plus the host's own fp64 error in Dc, Dr
    // (|coefficient| <= |M| * scale / v, a few ulps), accumulated over 1 + col + row steps
    x.coef_bound = (std::ldexp(1.0, -33) + std::ldexp(1.0, -40)) * (double)(c.crop_w + c.crop_h + 1);
    x.cal = dev_calib(c);
    x.g = dev_grid(g);
    // k_pnn_tiles: the flush addresses z planes by 32-bit byte offsets from the tile base (at most
    // ~66 planes of nx * ny voxels); the table word packs count (12 bits) | sum (20 bits), so no
    // voxel may collect more than 4095 pixels of one tile.  A voxel takes at most
    // floor(1 / max_k |Dc_k|) + 1 pixels of a row and floor(1 / max_k |Dr_k|) + 1 of a column, and
    // max_k |D_k| >= |D| / sqrt(3) = scale / (sqrt(3) voxel) for any pose (|q| = 1; the bound holds
    // for the rotation part, so it is pose-independent and a captured frame graph stays valid).
    x.lin_ok = c.probe == SVR_PROBE_LINEAR && (double)g.nx * g.ny * 8.0 * 70.0 < 4294967296.0;
    x.lin_count_ok = 0;
    if (x.lin_ok) {
        const double q2 = c.image_to_transducer.qw * c.image_to_transducer.qw +
                          c.image_to_transducer.qx * c.image_to_transducer.qx +
                          c.image_to_transducer.qy * c.image_to_transducer.qy +
                          c.image_to_transducer.qz * c.image_to_transducer.qz;
        // non-unit quaternions scale the map by |q|^2: the calibration's is taken as it is, the
        // pose's is required to be >= 0.98 per frame (make_params)
        const double qs = std::min(1.0, q2) * 0.98;
        const double nc = std::floor(std::sqrt(3.0) * g.voxel_mm / (c.scale_x_mm * qs)) + 1;
        const double nr = std::floor(std::sqrt(3.0) * g.voxel_mm / (c.scale_y_mm * qs)) + 1;
        for (int sh = 0; sh < 4; ++sh)
            if (std::min(nc * shape_rows(sh), nr * shape_cols(sh)) <= 4095) x.lin_count_ok |= 1 << sh;
    }
    return x;
}

static Affine frame_affine(const svr_rigid& pose, const PrepCtx& x) {
    double Mp[9], Mv[9];
    quat_mat(pose, Mp);
    mat_mul(Mp, x.Mc, Mv);
    Affine a;
    const double tp[3] = {pose.tx, pose.ty, pose.tz};
    for (int k = 0; k < 3; ++k) {
        double r = Mp[3 * k] * x.tc[0] + Mp[3 * k + 1] * x.tc[1] + Mp[3 * k + 2] * x.tc[2];
        a.K[k] = (r + tp[k] - x.o[k]) / x.v;
        for (int j = 0; j < 3; ++j) a.Mv[3 * k + j] = Mv[3 * k + j] / x.v;
    }
    return a;
}

static int make_params(const svr_rigid& pose, const PrepCtx& x, double sx, double sy,
                       FrameParams* fp) {
    if (!finite_rigid(pose)) return fail(SVR_E_INVALID, "pose not finite");
    Affine a = frame_affine(pose, x);
    bool ok = true;
    for (int k = 0; k < 3; ++k) {
        if (!(std::fabs(a.K[k]) < 1.0e8)) ok = false;
        fp->A[k] = to_fixed(a.K[k] + 0.5, &ok);
        fp->Dc[k] = to_fixed(a.Mv[3 * k] * sx, &ok);
        fp->Dr[k] = to_fixed(a.Mv[3 * k + 1] * sy, &ok);
        fp->K[k] = a.K[k];
        for (int j = 0; j < 3; ++j) fp->M[3 * k + j] = a.Mv[3 * k + j];
    }
    if (!ok) return fail(SVR_E_INVALID, "pose maps the frame too far from the grid (|u| >= 1e8 voxels)");
    fp->pose = pose;
    fp->cal = x.cal;
    fp->g = x.g;
    fp->lin_fit = 0;
    // Tie window: |fixed - real| <= coefficient rounding over 1 + col + row exact
    // integer steps, plus the deviation of an fp64 evaluation from real arithmetic -- the
    // reference chain's and this host map's (K) alike -- bounded by 512 roundings of the largest
    // intermediate magnitude qn * R, R = |t_pose| + pixel extent + |t_calib| + |origin| (mm), qn
    // covering non-unit quaternions.  The window is the smallest power of two >= 4x that bound,
    // in 2^-32 voxel units (2^-21 for cfg2); frames needing more than 2^-16 are refused.
    {
        const double qp2 = std::max(1.0, pose.qw * pose.qw + pose.qx * pose.qx +
                                             pose.qy * pose.qy + pose.qz * pose.qz);
        const double R = x.base_mm + norm3(pose.tx, pose.ty, pose.tz);
        const double chain = 0x1p-44 * qp2 * x.qc2 * R / x.v;  // 512 * 2^-53
        const double target = 4.0 * (x.coef_bound + chain) * 4294967296.0;
        int e = 4;
        for (double t = 16.0; e <= 16 && t < target; t *= 2.0) ++e;
        if (e > 16)
            return fail(SVR_E_INVALID, "pose too far from the grid origin for certified rounding "
                        "(|t| / voxel ~ %.3g)", R / x.v);
        fp->tie_eps = 1u << e;
    }
    // image-plane normal in voxel space = third column of R_pose R_calib (k_pnn_plane table);
    // the plane passes through K (image origin).  z_c(x,y) = K_z - (n_x (x-K_x) + n_y (y-K_y))/n_z
    {
        const double nx = a.Mv[2], ny = a.Mv[5], nz = a.Mv[8];
        const double ax = std::fabs(nx), ay = std::fabs(ny), az = std::fabs(nz);
        fp->plane_ok = (az > 0 && (ax + ay) < 0.99 * az) ? 1 : 0;  // 2h = s + 1.004 < 2
        if (fp->plane_ok) {
            fp->pz[0] = a.K[2] + (nx * a.K[0] + ny * a.K[1]) / nz;
            fp->pz[1] = -nx / nz;
            fp->pz[2] = -ny / nz;
            fp->pz[3] = (ax + ay) / (2 * az) + 0.5 + 2e-3;
        } else {
            fp->pz[0] = fp->pz[1] = fp->pz[2] = fp->pz[3] = 0.0;
        }
    }
    {
        const double qp2 = pose.qw * pose.qw + pose.qx * pose.qx + pose.qy * pose.qy + pose.qz * pose.qz;
        if (fp->plane_ok && x.lin_ok && qp2 >= 0.98)  // (the count bound in prep_ctx assumes |q|^2 >= 0.98)
            fp->lin_fit = tile_shapes_fit(fp->Dc, fp->Dr, x.lin_count_ok);
        // kZ1 walk: at most one y and one z carry in the 15 steps of a 16-pixel chunk
        if (fp->lin_fit && 15 * std::llabs(fp->Dc[1]) < (1ll << 32) && 15 * std::llabs(fp->Dc[2]) < (1ll << 32))
            fp->lin_fit |= kFitZ1;
    }
    return SVR_OK;
}

// Conservative box (global indices) a frame can touch: affine extremes at the image corners
// (linear) or at every scanline's end samples (fan), widened by one voxel.
static svr_box frame_box(const svr_grid_desc& g, const svr_calib& c, const svr_rigid& pose) {
    Affine a = frame_affine(pose, prep_ctx(c, g));
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        lo[k] = std::numeric_limits<double>::infinity();
        hi[k] = -lo[k];
    }
    auto add = [&](double px, double py) {
        for (int k = 0; k < 3; ++k) {
            double u = a.K[k] + a.Mv[3 * k] * px + a.Mv[3 * k + 1] * py;
            lo[k] = std::min(lo[k], u);
            hi[k] = std::max(hi[k], u);
        }
    };
    if (c.probe == SVR_PROBE_FAN) {
        std::vector<double> s, co;
        fan_table(c, s, co);
        const double dr = ((double)c.fan_r1_mm - c.fan_r0_mm) / c.crop_w;
        const double ra = c.fan_r0_mm + 0.5 * dr, rb = c.fan_r0_mm + (c.crop_w - 0.5) * dr;
        for (int i = 0; i < c.crop_h; ++i) {
            add(ra * s[i], ra * co[i]);
            add(rb * s[i], rb * co[i]);
        }
    } else {
        const double X = (double)(c.crop_w - 1) * c.scale_x_mm;
        const double Y = (double)(c.crop_h - 1) * c.scale_y_mm;
        add(0, 0);
        add(X, 0);
        add(0, Y);
        add(X, Y);
    }
    const int n[3] = {g.nx, g.ny, g.nz};
    int b0[3], b1[3];
    bool empty = false;
    for (int k = 0; k < 3; ++k) {
        double l = std::floor(lo[k] + 0.5) - 1, h = std::floor(hi[k] + 0.5) + 1;
        if (!(h >= 0) || !(l <= n[k] - 1)) {
            empty = true;
            break;
        }
        b0[k] = (int)std::max<double>(l, 0);
        b1[k] = (int)std::min<double>(h, n[k] - 1);
    }
    if (empty) return svr_box{1, 1, 1, 0, 0, 0};
    return svr_box{b0[0], b0[1], b0[2], b1[0], b1[1], b1[2]};
}

// ---------------------------------------------------------------- host-only ABI
extern "C" int svr_abi_version(void) { return SVR_ABI_VERSION; }

extern "C" const char* svr_last_error(void) { return g_err.c_str(); }

extern "C" int svr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

static void q_rotate(const svr_rigid& T, const double v[3], double o[3]) {
    // Quat::rotate, reference op order (host compiled with -ffp-contract=off)
    const double w = T.qw, ux = T.qx, uy = T.qy, uz = T.qz;
    double cx = uy * v[2] - uz * v[1], cy = uz * v[0] - ux * v[2], cz = ux * v[1] - uy * v[0];
    double tx = cx * 2.0, ty = cy * 2.0, tz = cz * 2.0;
    double ax = v[0] + tx * w, ay = v[1] + ty * w, az = v[2] + tz * w;
    double ex = uy * tz - uz * ty, ey = uz * tx - ux * tz, ez = ux * ty - uy * tx;
    o[0] = ax + ex;
    o[1] = ay + ey;
    o[2] = az + ez;
}

static void q_apply(const svr_rigid& T, const double v[3], double o[3]) {
    double r[3];
    q_rotate(T, v, r);
    o[0] = r[0] + T.tx;
    o[1] = r[1] + T.ty;
    o[2] = r[2] + T.tz;
}

static void q_normalize(double q[4]) {
    double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    for (int i = 0; i < 4; ++i) q[i] = q[i] / n;
}

extern "C" int svr_pose_from_matrix4(const double m[16], svr_rigid* out) {
    if (!m || !out) return fail(SVR_E_INVALID, "NULL argument");
    if (std::abs(m[12]) > 1e-9 || std::abs(m[13]) > 1e-9 || std::abs(m[14]) > 1e-9 ||
        std::abs(m[15] - 1.0) > 1e-9)
        return fail(SVR_E_INVALID, "bottom row of homogeneous matrix must be 0 0 0 1");
    // Shepperd's method (geometry.hpp:61-78) on the row-major rotation block
    const double r[9] = {m[0], m[1], m[2], m[4], m[5], m[6], m[8], m[9], m[10]};
    double tr = r[0] + r[4] + r[8];
    double q[4];
    if (tr > 0.0) {
        double s = std::sqrt(tr + 1.0) * 2.0;
        q[0] = 0.25 * s; q[1] = (r[7] - r[5]) / s; q[2] = (r[2] - r[6]) / s; q[3] = (r[3] - r[1]) / s;
    } else if (r[0] > r[4] && r[0] > r[8]) {
        double s = std::sqrt(1.0 + r[0] - r[4] - r[8]) * 2.0;
        q[0] = (r[7] - r[5]) / s; q[1] = 0.25 * s; q[2] = (r[1] + r[3]) / s; q[3] = (r[2] + r[6]) / s;
    } else if (r[4] > r[8]) {
        double s = std::sqrt(1.0 + r[4] - r[0] - r[8]) * 2.0;
        q[0] = (r[2] - r[6]) / s; q[1] = (r[1] + r[3]) / s; q[2] = 0.25 * s; q[3] = (r[5] + r[7]) / s;
    } else {
        double s = std::sqrt(1.0 + r[8] - r[0] - r[4]) * 2.0;
        q[0] = (r[3] - r[1]) / s; q[1] = (r[2] + r[6]) / s; q[2] = (r[5] + r[7]) / s; q[3] = 0.25 * s;
    }
    double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (n == 0.0) return fail(SVR_E_INVALID, "zero quaternion");
    q_normalize(q);
    *out = svr_rigid{q[0], q[1], q[2], q[3], m[3], m[7], m[11]};
    return SVR_OK;
}

extern "C" int svr_compose(const svr_rigid* a, const svr_rigid* b, svr_rigid* out) {
    if (!a || !b || !out) return fail(SVR_E_INVALID, "NULL argument");
    // compose (geometry.hpp:142-144): rotation (a.q * b.q).normalized(), translation a.apply(b.t)
    double q[4] = {a->qw * b->qw - a->qx * b->qx - a->qy * b->qy - a->qz * b->qz,
                   a->qw * b->qx + a->qx * b->qw + a->qy * b->qz - a->qz * b->qy,
                   a->qw * b->qy - a->qx * b->qz + a->qy * b->qw + a->qz * b->qx,
                   a->qw * b->qz + a->qx * b->qy - a->qy * b->qx + a->qz * b->qw};
    double n = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (n == 0.0) return fail(SVR_E_INVALID, "zero quaternion");
    q_normalize(q);
    double t[3] = {b->tx, b->ty, b->tz}, o[3];
    q_apply(*a, t, o);
    *out = svr_rigid{q[0], q[1], q[2], q[3], o[0], o[1], o[2]};
    return SVR_OK;
}

extern "C" int svr_interpolate_pose(const double* t_ms, const svr_rigid* poses, int n, double t,
                                    svr_rigid* out) {
    // interpolate_pose (geometry.hpp:194-209) + slerp (:82-100)
    if (!t_ms || !poses || !out || n <= 0) return fail(SVR_E_INVALID, "empty pose sequence");
    if (t < t_ms[0] || t > t_ms[n - 1])
        return fail(SVR_E_INVALID, "pose interpolation time outside sampled range");
    int i = (int)(std::lower_bound(t_ms, t_ms + n, t) - t_ms);
    if (t_ms[i] == t) {
        *out = poses[i];
        return SVR_OK;
    }
    const svr_rigid& hi = poses[i];
    const svr_rigid& lo = poses[i - 1];
    double u = (t - t_ms[i - 1]) / (t_ms[i] - t_ms[i - 1]);
    svr_rigid r;
    r.tx = lo.tx + (hi.tx - lo.tx) * u;
    r.ty = lo.ty + (hi.ty - lo.ty) * u;
    r.tz = lo.tz + (hi.tz - lo.tz) * u;
    double a[4] = {lo.qw, lo.qx, lo.qy, lo.qz}, b[4] = {hi.qw, hi.qx, hi.qy, hi.qz}, q[4];
    double d = a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3];
    if (d < 0.0) {
        for (int k = 0; k < 4; ++k) b[k] = -b[k];
        d = -d;
    }
    if (d > 0.9995) {
        for (int k = 0; k < 4; ++k) q[k] = a[k] + u * (b[k] - a[k]);
    } else {
        double theta = std::acos(std::clamp(d, -1.0, 1.0));
        double s = std::sin(theta);
        double wa = std::sin((1.0 - u) * theta) / s;
        double wb = std::sin(u * theta) / s;
        for (int k = 0; k < 4; ++k) q[k] = wa * a[k] + wb * b[k];
    }
    double nn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (nn == 0.0) return fail(SVR_E_INVALID, "zero quaternion");
    q_normalize(q);
    r.qw = q[0]; r.qx = q[1]; r.qy = q[2]; r.qz = q[3];
    *out = r;
    return SVR_OK;
}

// Frame/pose matching of the ingest front-end (SPEC.md geometry "Pose/frame matching"): each
// frame time shifted by -latency_ms, then interpolate_pose.  Frames whose shifted time falls
// outside the sampled span (where interpolate_pose throws) get valid = 0 and an identity pose.
extern "C" int svr_match_poses(const double* pose_t_ms, const svr_rigid* poses, int32_t n,
                               const double* frame_t_ms, int32_t m, double latency_ms,
                               svr_rigid* out, uint8_t* valid, int32_t* n_valid) {
    if (m < 0 || (m > 0 && (!frame_t_ms || !out || !valid))) return fail(SVR_E_INVALID, "invalid frame list");
    if (n <= 0 || !pose_t_ms || !poses) return fail(SVR_E_INVALID, "empty pose sequence");
    for (int i = 1; i < n; ++i)
        if (!(pose_t_ms[i] >= pose_t_ms[i - 1]))
            return fail(SVR_E_INVALID, "pose timestamps must be non-decreasing (sample %d)", i);
    int nv = 0;
    const std::string saved = g_err;
    for (int k = 0; k < m; ++k) {
        const double t = frame_t_ms[k] - latency_ms;
        valid[k] = 0;
        out[k] = svr_rigid{1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (!(t >= pose_t_ms[0] && t <= pose_t_ms[n - 1])) continue;
        if (svr_interpolate_pose(pose_t_ms, poses, n, t, &out[k]) == SVR_OK) {
            valid[k] = 1;
            ++nv;
        }
    }
    g_err = saved;
    if (n_valid) *n_valid = nv;
    return SVR_OK;
}

extern "C" int svr_pixel_to_world(double col, double row, const svr_calib* c, const svr_rigid* pose,
                                  double out[3]) {
    if (!c || !pose || !out) return fail(SVR_E_INVALID, "NULL argument");
    if (col < 0 || row < 0 || col >= c->crop_w || row >= c->crop_h)
        return fail(SVR_E_INVALID, "pixel outside B-mode image bounds");
    double p[3];
    if (c->probe == SVR_PROBE_FAN) {
        std::vector<double> s, co;
        fan_table(*c, s, co);
        double dr = (c->fan_r1_mm - c->fan_r0_mm) / (double)c->crop_w;
        double r = c->fan_r0_mm + (std::floor(col) + 0.5) * dr;
        int li = (int)row;
        p[0] = r * s[li];
        p[1] = r * co[li];
    } else {
        p[0] = col * c->scale_x_mm;
        p[1] = row * c->scale_y_mm;
    }
    p[2] = 0.0;
    double q[3];
    q_apply(c->image_to_transducer, p, q);
    q_apply(*pose, q, out);
    return SVR_OK;
}

static int check_grid(const svr_grid_desc* g) {
    if (!g) return fail(SVR_E_INVALID, "grid desc is NULL");
    if (g->nx <= 0 || g->ny <= 0 || g->nz <= 0) return fail(SVR_E_INVALID, "grid dims must be positive");
    if (!(g->voxel_mm > 0.0) || !std::isfinite(g->voxel_mm))
        return fail(SVR_E_INVALID, "voxel_mm must be positive");
    if (g->z_begin < 0 || g->z_end > g->nz || g->z_begin >= g->z_end)
        return fail(SVR_E_INVALID, "slab [%d,%d) outside [0,%d)", g->z_begin, g->z_end, g->nz);
    for (int k = 0; k < 3; ++k)
        if (!std::isfinite(g->origin_mm[k])) return fail(SVR_E_INVALID, "origin not finite");
    if (g->accum != SVR_ACC_PNN && g->accum != SVR_ACC_TRILINEAR)
        return fail(SVR_E_INVALID, "unknown accumulator kind %d", g->accum);
    return SVR_OK;
}

extern "C" int svr_frame_bounds(const svr_grid_desc* g, const svr_calib* c, const svr_rigid* pose,
                                svr_box* out) {
    if (int e = check_grid(g)) return e;
    if (!c || !pose || !out) return fail(SVR_E_INVALID, "NULL argument");
    if (int e = check_calib(c, c->crop_w, c->crop_h)) return e;
    if (!finite_rigid(*pose)) return fail(SVR_E_INVALID, "pose not finite");
    *out = frame_box(*g, *c, *pose);
    return SVR_OK;
}

extern "C" int svr_plan_slabs(int32_t nz, int32_t nranks, int32_t ghost, int32_t* ob, int32_t* oe,
                              int32_t* ab, int32_t* ae) {
    if (nz <= 0 || nranks <= 0 || ghost < 0 || nranks > nz)
        return fail(SVR_E_INVALID, "invalid slab plan nz=%d nranks=%d ghost=%d", nz, nranks, ghost);
    for (int r = 0; r < nranks; ++r) {
        int32_t b = (int32_t)((int64_t)nz * r / nranks), e = (int32_t)((int64_t)nz * (r + 1) / nranks);
        ob[r] = b;
        oe[r] = e;
        ab[r] = std::max(0, b - ghost);
        ae[r] = std::min(nz, e + ghost);
    }
    return SVR_OK;
}

// ---------------------------------------------------------------- device ABI
#define VOL_CHECK(v)                                                    \
    do {                                                                \
        if (!(v)) return fail(SVR_E_INVALID, "volume handle is NULL");   \
        CK(cudaSetDevice((v)->device));                                 \
    } while (0)

extern "C" int svr_destroy(svr_volume* v) {
    if (!v) return SVR_OK;
    cudaSetDevice(v->device);
    if (v->stream) cudaStreamSynchronize(v->stream);
    if (v->copy_stream) cudaStreamSynchronize(v->copy_stream);
    if (v->param_stream) cudaStreamSynchronize(v->param_stream);
    cudaFree(v->acc);
    cudaFree(v->tri);
    cudaFree(v->fill);
    cudaFree(v->r_depth);
    cudaFree(v->r_mdepth);
    cudaFree(v->r_mean);
    cudaFree(v->r_max);
    cudaFree(v->d_stats);
    cudaFree(v->d_counter);
    for (int i = 0; i < 2; ++i) cudaFree(v->d_params2[i]);
    for (int i = 0; i < 2; ++i) cudaFreeHost(v->h_params[i]);
    cudaFree(v->d_boxes);
    cudaFreeHost(v->h_boxes);
    cudaFree(v->d_fan);
    cudaFree(v->d_desc);
    cudaFree(v->d_frc);
    cudaFree(v->d_fdesc);
    cudaFree(v->d_frows);
    cudaFree(v->d_work);
    for (int i = 0; i < svr_volume::kTileSlots; ++i) {
        cudaFree(v->d_tiles[i]);
        cudaFreeHost(v->h_tiles[i]);
        if (v->tiles_ev[i]) cudaEventDestroy(v->tiles_ev[i]);
    }
    cudaFree(v->d_work_n);
    cudaFree(v->d_gt);
    if (v->fg.exec) cudaGraphExecDestroy(v->fg.exec);
    if (v->fg.graph) cudaGraphDestroy(v->fg.graph);
    if (v->fg.done) cudaEventDestroy(v->fg.done);
    cudaFree(v->fg.d_frame);
    cudaFree(v->fg.d_fp);
    cudaFree(v->fg.d_tiles);
    cudaFreeHost(v->fg.h_frame);
    cudaFreeHost(v->fg.h_fp);
    cudaFreeHost(v->fg.h_tiles);
    for (int i = 0; i < 2; ++i) {
        cudaFree(v->d_stage[i]);
        cudaFreeHost(v->h_stage[i]);
        if (v->ev_ready[i]) cudaEventDestroy(v->ev_ready[i]);
        if (v->ev_free[i]) cudaEventDestroy(v->ev_free[i]);
        if (v->ev_h2d[i]) cudaEventDestroy(v->ev_h2d[i]);
    }
    for (int i = 0; i < 2; ++i) {
        if (v->params_ev[i]) cudaEventDestroy(v->params_ev[i]);
        if (v->params_used[i]) cudaEventDestroy(v->params_used[i]);
    }
    if (v->ins_done) cudaEventDestroy(v->ins_done);
    if (v->ev_prep) cudaEventDestroy(v->ev_prep);
    if (v->ev_tiles_up) cudaEventDestroy(v->ev_tiles_up);
    if (v->own_stream && v->stream) cudaStreamDestroy(v->stream);
    if (v->own_stream_saved) cudaStreamDestroy(v->own_stream_saved);
    if (v->copy_stream) cudaStreamDestroy(v->copy_stream);
    if (v->param_stream) cudaStreamDestroy(v->param_stream);
    cudaGetLastError();
    delete v;
    return SVR_OK;
}

extern "C" int svr_create(const svr_grid_desc* desc, int device, svr_volume** out) {
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    *out = nullptr;
    if (int e = check_grid(desc)) return e;
    int ndev = svr_device_count();
    if (ndev <= 0) return fail(SVR_E_CUDA, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(SVR_E_INVALID, "device %d out of range", device);
    svr_volume* v = new svr_volume();
    v->d = *desc;
    if (const char* e = std::getenv("SVR_INSERT_KERNEL")) v->insert_kernel = !std::strcmp(e, "direct") ? 1 : 3;
    if (const char* e = std::getenv("SVR_TRI_KERNEL")) v->tri_kernel = !std::strcmp(e, "chunk") ? 1 : 0;

    v->device = device;
    auto bail = [&](int code) {
        svr_destroy(v);
        return code;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(SVR_E_CUDA, "cudaSetDevice failed"));
    cudaDeviceGetAttribute(&v->num_sms, cudaDevAttrMultiProcessorCount, device);
    v->nvox = (long long)desc->nx * desc->ny * (desc->z_end - desc->z_begin);
    const long long ncol = (long long)desc->nx * (desc->z_end - desc->z_begin);
    cudaError_t e = cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&v->copy_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&v->param_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        if (desc->accum == SVR_ACC_PNN) {
            e = cudaMalloc(&v->acc, sizeof(ull) * v->nvox);
            if (e == cudaSuccess) e = cudaMalloc(&v->fill, sizeof(uint32_t) * v->nvox);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_depth, sizeof(int) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_mdepth, sizeof(int) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_mean, sizeof(float) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_max, sizeof(float) * ncol);
        } else {  // trilinear: the f32 pair per voxel + the render layer (BASELINE cfg5)
            e = cudaMalloc(&v->tri, sizeof(float2) * v->nvox);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_depth, sizeof(int) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_mdepth, sizeof(int) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_mean, sizeof(float) * ncol);
            if (e == cudaSuccess) e = cudaMalloc(&v->r_max, sizeof(float) * ncol);
        }
    }
    if (e == cudaSuccess) {  // the fill's reciprocal table (per device; idempotent)
        k_init_rcp<<<1, 256, 0, v->stream>>>();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMalloc(&v->d_stats, sizeof(ull) * kStCount);
    if (e == cudaSuccess) e = cudaMalloc(&v->d_counter, sizeof(ull) * 2);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&v->params_ev[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->params_used[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->ins_done, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->ev_prep, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->ev_tiles_up, cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&v->ev_ready[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->ev_free[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&v->ev_h2d[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(SVR_E_CUDA, "allocation of %lld voxels failed: %s", v->nvox,
                         cudaGetErrorString(e)));
    }
    *out = v;
    int rc = svr_clear(v);
    if (rc) {
        *out = nullptr;
        return bail(rc);
    }
    return SVR_OK;
}

extern "C" int svr_set_stream(svr_volume* v, void* s) {
    VOL_CHECK(v);
    CK(cudaStreamSynchronize(v->stream));
    if (v->own_stream && v->stream) CK(cudaStreamDestroy(v->stream));
    if (s) {
        v->stream = (cudaStream_t)s;
        v->own_stream = false;
    } else if (v->own_stream_saved) {
        v->stream = v->own_stream_saved;
        v->own_stream_saved = nullptr;
        v->own_stream = true;
    } else {
        CK(cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking));
        v->own_stream = true;
    }
    return SVR_OK;
}

extern "C" int svr_use_stream(svr_volume* v, void* s) {
    VOL_CHECK(v);
    if (!s) return fail(SVR_E_INVALID, "svr_use_stream needs a stream");
    if (v->own_stream && v->stream) {  // the handle's own stream stays alive for later calls
        v->own_stream_saved = v->stream;
        v->own_stream = false;
    }
    v->stream = (cudaStream_t)s;
    return SVR_OK;
}

extern "C" int svr_clear(svr_volume* v) {
    VOL_CHECK(v);
    const long long ncol = (long long)v->d.nx * (v->d.z_end - v->d.z_begin);
    if (v->acc) CK(cudaMemsetAsync(v->acc, 0, sizeof(ull) * v->nvox, v->stream));
    if (v->tri) CK(cudaMemsetAsync(v->tri, 0, sizeof(float2) * v->nvox, v->stream));
    if (v->fill) CK(cudaMemsetAsync(v->fill, 0, sizeof(uint32_t) * v->nvox, v->stream));
    if (v->r_depth) {
        CK(cudaMemsetAsync(v->r_depth, 0xFF, sizeof(int) * ncol, v->stream));
        CK(cudaMemsetAsync(v->r_mdepth, 0xFF, sizeof(int) * ncol, v->stream));
        CK(cudaMemsetAsync(v->r_mean, 0, sizeof(float) * ncol, v->stream));
        CK(cudaMemsetAsync(v->r_max, 0, sizeof(float) * ncol, v->stream));
    }
    CK(cudaMemsetAsync(v->d_stats, 0, sizeof(ull) * kStCount, v->stream));
    v->frames = 0;
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_sync(svr_volume* v) {
    VOL_CHECK(v);
    CK(cudaStreamSynchronize(v->stream));
    CK(cudaGetLastError());
    return SVR_OK;
}

extern "C" int svr_get_desc(const svr_volume* v, svr_grid_desc* out) {
    if (!v || !out) return fail(SVR_E_INVALID, "NULL argument");
    *out = v->d;
    return SVR_OK;
}

// Select the host parameter buffer for this call (v->pslot); its previous upload, two calls
// back, must have finished before it is rewritten.
static int ensure_params(svr_volume* v, int n) {
    v->pslot ^= 1;
    CK(cudaEventSynchronize(v->params_ev[v->pslot]));
    if (n <= v->params_cap) return SVR_OK;
    int cap = std::max(n, 2 * v->params_cap);
    CK(cudaStreamSynchronize(v->stream));
    CK(cudaStreamSynchronize(v->param_stream));
    v->d_params = nullptr;
    for (int i = 0; i < 2; ++i) {
        cudaFree(v->d_params2[i]);
        v->d_params2[i] = nullptr;
        cudaFreeHost(v->h_params[i]);
        v->h_params[i] = nullptr;
    }
    v->params_cap = 0;
    for (int i = 0; i < 2; ++i) CK(cudaMalloc(&v->d_params2[i], sizeof(FrameParams) * cap));
    for (int i = 0; i < 2; ++i) CK(cudaMallocHost(&v->h_params[i], sizeof(FrameParams) * cap));
    v->params_cap = cap;
    return SVR_OK;
}

static int ensure_boxes(svr_volume* v, int n) {
    if (n <= v->boxes_cap) return SVR_OK;
    int cap = std::max(n, 2 * v->boxes_cap);
    CK(cudaStreamSynchronize(v->stream));
    cudaFree(v->d_boxes);
    cudaFreeHost(v->h_boxes);
    v->d_boxes = nullptr;
    v->h_boxes = nullptr;
    v->boxes_cap = 0;
    CK(cudaMalloc(&v->d_boxes, sizeof(int) * 6 * cap));
    CK(cudaMallocHost(&v->h_boxes, sizeof(int) * 6 * cap));
    v->boxes_cap = cap;
    return SVR_OK;
}

static int ensure_fan(svr_volume* v, const svr_calib& c) {
    if (c.probe != SVR_PROBE_FAN) return SVR_OK;
    if (v->d_fan && v->fan_lines == c.crop_h && v->fan_angle == c.fan_angle_deg) return SVR_OK;
    std::vector<double> s, co;
    fan_table(c, s, co);
    std::vector<double2> t(c.crop_h);
    for (int i = 0; i < c.crop_h; ++i) t[i] = make_double2(s[i], co[i]);
    CK(cudaStreamSynchronize(v->stream));
    cudaFree(v->d_fan);
    v->d_fan = nullptr;
    CK(cudaMalloc(&v->d_fan, sizeof(double2) * c.crop_h));
    CK(cudaMemcpy(v->d_fan, t.data(), sizeof(double2) * c.crop_h, cudaMemcpyHostToDevice));
    v->fan_lines = c.crop_h;
    v->fan_angle = c.fan_angle_deg;
    return SVR_OK;
}

__global__ void k_box_init(int* b, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        int* p = b + 6 * i;
        p[0] = p[1] = p[2] = 0x7fffffff;
        p[3] = p[4] = p[5] = -0x7fffffff - 1;
    }
}

static long long coprime_stride(int n) {
    if (n <= 2) return 1;
    long long p = std::max(1ll, (long long)std::llround(n * 0.3819660112501051));
    auto gcd = [](long long a, long long b) { while (b) { long long t = a % b; a = b; b = t; } return a; };
    while (gcd(p, n) != 1) ++p;
    return p;
}

template <int kMode, bool kVec, bool kSkip, bool kBox>
static void launch_insert_t(svr_volume* v, const uint8_t* px, long long pitch, long long fstride,
                            int w, int h, int n, const FrameParams* fps, const DevCalib& cal,
                            uint32_t* mark, uint32_t tag, int* boxes, ull* stats) {
    const int cpr = (w + kChunk - 1) / kChunk;
    const int chunks = cpr * h;
    dim3 block(256), grid((chunks + 255) / 256, n);
    k_insert<kMode, kVec, kSkip, kBox><<<grid, block, 0, v->stream>>>(
        px, pitch, fstride, w, h, cpr, fps, cal, v->d_fan, dev_grid(v->d), v->acc, v->tri, mark,
        tag, boxes, stats);
    v->launches++;
}

template <int kMode>
static void launch_insert(svr_volume* v, bool vec, bool skip, bool box, const uint8_t* px,
                          long long pitch, long long fstride, int w, int h, int n,
                          const FrameParams* fps, const DevCalib& cal, uint32_t* mark,
                          uint32_t tag, int* boxes, ull* stats) {
#define LI(a, b, c) \
    launch_insert_t<kMode, a, b, c>(v, px, pitch, fstride, w, h, n, fps, cal, mark, tag, boxes, stats)
    if (vec) {
        if (skip) { if (box) LI(true, true, true); else LI(true, true, false); }
        else { if (box) LI(true, false, true); else LI(true, false, false); }
    } else {
        if (skip) { if (box) LI(false, true, true); else LI(false, true, false); }
        else { if (box) LI(false, false, true); else LI(false, false, false); }
    }
#undef LI
}

static bool is_device_ptr(const void* p, bool* pinned) {
    cudaPointerAttributes a;
    *pinned = false;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return true;
    if (a.type == cudaMemoryTypeHost) *pinned = true;
    return false;
}

// per-tile descriptor buffer of k_pnn_tiles (grown outside any graph capture: fg_capture
// pre-sizes it for one frame)
static int ensure_desc(svr_volume* v, long long ntiles, long long nframes) {
    if (v->desc_cap < ntiles) {
        CK(cudaStreamSynchronize(v->stream));
        cudaFree(v->d_desc);
        v->d_desc = nullptr;
        v->desc_cap = std::max<long long>(ntiles, 4096);
        CK(cudaMalloc(&v->d_desc, sizeof(TileDesc) * v->desc_cap));
    }
    if (v->frc_cap < nframes) {
        CK(cudaStreamSynchronize(v->stream));
        cudaFree(v->d_frc);
        v->d_frc = nullptr;
        v->frc_cap = std::max<long long>(nframes, 256);
        CK(cudaMalloc(&v->d_frc, sizeof(TileFrame) * v->frc_cap));
    }
    return SVR_OK;
}

// k_fan_tiles buffers (grown outside any graph capture: fg_capture pre-sizes them)
static int ensure_fan_bufs(svr_volume* v, long long ntiles, long long nrows) {
    if (v->fdesc_cap < ntiles) {
        CK(cudaStreamSynchronize(v->stream));
        cudaFree(v->d_fdesc);
        v->d_fdesc = nullptr;
        v->fdesc_cap = std::max<long long>(ntiles, 4096);
        CK(cudaMalloc(&v->d_fdesc, sizeof(FanDesc) * v->fdesc_cap));
    }
    if (v->frows_cap < nrows) {
        CK(cudaStreamSynchronize(v->stream));
        cudaFree(v->d_frows);
        v->d_frows = nullptr;
        v->frows_cap = std::max<long long>(nrows, 4096);
        CK(cudaMalloc(&v->d_frows, sizeof(FanRow) * v->frows_cap));
    }
    return SVR_OK;
}

// K1 for convex probes: k_fan_desc (scanline constants + tile descriptors), k_fan_tiles
// (persistent over the launch's tiles); the caller launches the exact pass.
static int launch_fan(svr_volume* v, bool box, const uint8_t* px, long long pitch, long long fstride,
                      int w, int h, int m, const FrameParams* fps, const DevCalib& cal, int* boxes,
                      ull* stats) {
    constexpr int TCOLS = 128;
    FanArgs fa;
    fa.px = px;
    fa.pitch = pitch;
    fa.fstride = fstride;
    fa.w = w;
    fa.h = h;
    fa.ntx = w / TCOLS;
    fa.nty = (h + kFanLines - 1) / kFanLines;
    fa.ntiles = (long long)m * fa.ntx * fa.nty;
    fa.fps = fps;
    fa.cal = cal;
    fa.fan = v->d_fan;
    fa.g = dev_grid(v->d);
    fa.acc = v->acc;
    fa.boxes = boxes;
    fa.stats = stats;
    fa.work = v->d_work;
    fa.work_n = v->d_work_n;
    fa.work_cap = v->work_cap;
    // table mode when the tile's index box has at most one position per pixel (A/B on cfg3:
    // thresholds 1/4 .. 2 px per position within 1%)
    fa.dense = 4;
    if (int e = ensure_fan_bufs(v, fa.ntiles, (long long)m * h)) return e;
    fa.desc = v->d_fdesc;
    fa.rows = v->d_frows;
    const int slot = box ? 1 : 0;
    if (!v->fan_occ[slot]) {
        int occ = 0;
        if (box) CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fan_tiles<true>, 128, 0));
        else CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fan_tiles<false>, 128, 0));
        v->fan_occ[slot] = std::max(1, occ);
    }
    const long long ctas = std::min<long long>(fa.ntiles, (long long)v->num_sms * v->fan_occ[slot]);
    k_fan_desc<TCOLS><<<(unsigned)((fa.ntiles * 32 + 127) / 128), 128, 0, v->stream>>>(fa);
    if (box) k_fan_tiles<true><<<(unsigned)ctas, 128, 0, v->stream>>>(fa);
    else k_fan_tiles<false><<<(unsigned)ctas, 128, 0, v->stream>>>(fa);
    v->launches += 2;
    return SVR_OK;
}

// K1 for linear probes: k_pnn_tiles (persistent over the launch's tiles) + the exact pass.
template <int NCH, int NW, bool kBox, bool kZ1, bool kSkip>
static int launch_tiles_t(svr_volume* v, const TilesArgs& ta) {
    const int slot = (NCH == 2) + 2 * (NW == 2) + 4 * kBox + 8 * kZ1 + 16 * kSkip;
    if (!v->tiles_occ[slot]) {
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pnn_tiles<NCH, NW, kBox, kZ1, kSkip>, 32 * NW, 0));
        v->tiles_occ[slot] = std::max(1, occ);
    }
    const long long ctas = std::min<long long>(ta.ntiles, (long long)v->num_sms * v->tiles_occ[slot]);
    if (v->prep_on_param) {
        // (insert_common: the descriptors are built on param_stream right after the parameter
        // upload, beside the previous step's fill / render; the kernels' stream waits for them)
        k_tile_desc<NCH, NW, kZ1><<<(unsigned)((ta.ntiles + 127) / 128), 128, 0, v->param_stream>>>(ta, const_cast<TileDesc*>(ta.desc));
        CK(cudaEventRecord(v->ev_prep, v->param_stream));
        CK(cudaStreamWaitEvent(v->stream, v->ev_prep, 0));
    } else {
        k_tile_desc<NCH, NW, kZ1><<<(unsigned)((ta.ntiles + 127) / 128), 128, 0, v->stream>>>(ta, const_cast<TileDesc*>(ta.desc));
    }
    k_pnn_tiles<NCH, NW, kBox, kZ1, kSkip><<<(unsigned)ctas, 32 * NW, 0, v->stream>>>(ta);
    v->launches += 2;
    return SVR_OK;
}

// Tile shape for a launch: the least per-thread work on the critical path -- ceil(tiles /
// resident CTAs) rounds, each a row of TCOLS pixels per thread -- with the 64 x 128 shape (the
// fewest table positions per pixel) preferred within 5%.  Resident CTAs per SM: SVR_TILES_MINB
// for the 128-thread shapes, twice that for the 64-thread ones (register-bound).
static int pick_shape(int shapes, int w, int h, int nframes, int num_sms) {
    int best = -1;
    double best_cost = 0;
    for (int sh = 0; sh < 4; ++sh) {
        if (!((shapes >> sh) & 1) || w % shape_cols(sh)) continue;
        const double tiles = (double)nframes * (w / shape_cols(sh)) * ((h + shape_rows(sh) - 1) / shape_rows(sh));
        const double slots = (double)num_sms * (shape_rows(sh) == 128 ? SVR_TILES_MINB : 2 * SVR_TILES_MINB);
        double cost = std::ceil(tiles / slots) * shape_cols(sh) * (1.0 + 0.05 * (sh != 0));
#ifdef SVR_TILES_SHAPE
        if (sh == SVR_TILES_SHAPE) cost = 0;  // (A/B builds: force one shape where it fits)
#endif
        if (best < 0 || cost < best_cost) {
            best = sh;
            best_cost = cost;
        }
    }
    return best >= 0 && (shapes & kFitZ1) ? best | kShapeZ1 : best;
}

template <bool kBox, bool kSkip>
static int launch_tiles_s(svr_volume* v, int shape, const TilesArgs& ta) {
    switch (shape & 7) {  // bits 0-1: tile shape, bit 2 (kShapeZ1): the kZ1 walk
        case 0: return launch_tiles_t<4, 4, kBox, false, kSkip>(v, ta);
        case 1: return launch_tiles_t<2, 4, kBox, false, kSkip>(v, ta);
        case 2: return launch_tiles_t<4, 2, kBox, false, kSkip>(v, ta);
        case 3: return launch_tiles_t<2, 2, kBox, false, kSkip>(v, ta);
        case 4: return launch_tiles_t<4, 4, kBox, true, kSkip>(v, ta);
        case 5: return launch_tiles_t<2, 4, kBox, true, kSkip>(v, ta);
        case 6: return launch_tiles_t<4, 2, kBox, true, kSkip>(v, ta);
        default: return launch_tiles_t<2, 2, kBox, true, kSkip>(v, ta);
    }
}

static int launch_tiles(svr_volume* v, int shape, bool box, bool skip, const uint8_t* px, long long pitch,
                        long long fstride, int w, int h, int m, const FrameParams* fps, int* boxes,
                        ull* stats) {
    TilesArgs ta;
    ta.px = px;
    ta.pitch = pitch;
    ta.fstride = fstride;
    ta.h = h;
    ta.ntx = w / shape_cols(shape);
    ta.nty = (h + shape_rows(shape) - 1) / shape_rows(shape);
    ta.ntiles = (long long)m * ta.ntx * ta.nty;
    ta.fps = fps;
    ta.g = dev_grid(v->d);
    ta.acc = v->acc;
    ta.boxes = boxes;
    ta.stats = stats;
    ta.work = v->d_work;
    ta.work_n = v->d_work_n;
    ta.work_cap = v->work_cap;
    if (int e = ensure_desc(v, ta.ntiles, m)) return e;
    ta.desc = v->d_desc;
    ta.frc = v->d_frc;
    return skip ? (box ? launch_tiles_s<true, true>(v, shape, ta) : launch_tiles_s<false, true>(v, shape, ta))
                : (box ? launch_tiles_s<true, false>(v, shape, ta) : launch_tiles_s<false, false>(v, shape, ta));
}

// Launch over frames resident in device memory, chunked to the grid.y limit.
//   PNN insert: linear probes k_tile_desc + k_pnn_tiles (svr_k1.cuh; skip_zero as its kSkip
//   variant); no skip_zero: convex fans
//   k_fan_desc + k_fan_tiles (svr_fan.cuh, 32-byte aligned rows of whole 128-sample tiles) or
//   else k_pnn_plane; each + k_pnn_work (the exact pass).  k_insert: skip_zero, geometries the
//   tiles refuse, SVR_INSERT_KERNEL=direct (tests), footprint and trilinear.
static int insert_device(svr_volume* v, int mode, const uint8_t* px, long long pitch,
                         long long fstride, int w, int h, int n, const FrameParams* fps,
                         const DevCalib& cal, bool skip, bool box, int* boxes, uint32_t* mark,
                         uint32_t tag, ull* stats) {
    const bool vec = ((uintptr_t)px % 16 == 0) && (pitch % 16 == 0) && (fstride % 16 == 0) &&
                     (w % kChunk == 0);
    const bool direct = v->insert_kernel == 1;
    // linear probes: k_pnn_tiles (reads each row segment with 32-byte loads)
    const bool vec32 = ((uintptr_t)px % 32 == 0) && (pitch % 32 == 0) && (n == 1 || fstride % 32 == 0);
    const int shape = (mode == kModeInsert && !direct && cal.probe == SVR_PROBE_LINEAR && vec32)
                          ? pick_shape(v->lin_shapes_cur, w, h, n, v->num_sms)
                          : -1;
    // convex fan: tables of packed (count << 20 | sum) slots hold at most 4095 pixels: guaranteed
    // when samples 63 apart are more than a voxel diagonal apart (63 dr > sqrt(3) voxel: at most
    // 63 samples of a scanline per voxel, 32 scanlines per k_fan_tiles tile, 64 per k_pnn_plane)
    const bool fan_plane = mode == kModeInsert && !skip && !direct && cal.probe == SVR_PROBE_FAN &&
                           w >= 4 * kChunk && (long long)v->d.nx * v->d.ny < (1ll << 22) &&
                           63.0 * cal.dr > std::sqrt(3.0) * v->d.voxel_mm;
    // convex fan with 32-byte aligned rows of whole 128-sample tiles: k_fan_tiles
    const bool fan_tiles = fan_plane && vec32 && w % 128 == 0;
    for (int k0 = 0; k0 < n; k0 += 65535) {
        int m = std::min(65535, n - k0);
        const uint8_t* p = px + (long long)k0 * fstride;
        int* bx = boxes ? boxes + 6 * k0 : nullptr;
        // the deferred-chunk pass is grid-strided over a worklist of a few entries per frame:
        // a single frame must not pay for launching thousands of idle CTAs
        // (skip_zero sends every chunk with both zero and non-zero pixels there: more CTAs)
        const int work_ctas = std::min((skip ? 8 : SVR_WORK_CTAS_PER_SM) * v->num_sms, std::max(16, 8 * m));
        const GridDev gd = dev_grid(v->d);
        if (shape >= 0 || fan_tiles) {
            // k_pnn_tiles / k_fan_tiles defer whole chunks with no overflow path: room for every chunk
            const long long need = std::max<long long>(1ll << 20, (long long)m * h * (w / kChunk));
            if (need > 0xffffffffll) return fail(SVR_E_INVALID, "insert batch too large");
            if (!v->d_work || v->work_cap < need) {
                CK(cudaStreamSynchronize(v->stream));
                cudaFree(v->d_work);
                v->d_work = nullptr;
                v->work_cap = (unsigned int)need;
                CK(cudaMalloc(&v->d_work, sizeof(ull) * v->work_cap));
                if (!v->d_work_n) CK(cudaMalloc(&v->d_work_n, sizeof(unsigned int)));
            }
            CK(cudaMemsetAsync(v->d_work_n, 0, sizeof(unsigned int),
                               v->prep_on_param && !fan_tiles ? v->param_stream : v->stream));
            if (fan_tiles) {
                if (int e = launch_fan(v, box, p, pitch, fstride, w, h, m, fps + k0, cal, bx, stats)) return e;
            } else {
                if (int e = launch_tiles(v, shape, box, skip, p, pitch, fstride, w, h, m, fps + k0, bx, stats)) return e;
            }
            if (box)
                k_pnn_work<true, true><<<work_ctas, 256, 0, v->stream>>>(
                    p, pitch, fstride, w, fps + k0, cal, v->d_fan, gd, v->acc, bx, stats, v->d_work,
                    v->d_work_n, v->work_cap);
            else
                k_pnn_work<true, false><<<work_ctas, 256, 0, v->stream>>>(
                    p, pitch, fstride, w, fps + k0, cal, v->d_fan, gd, v->acc, bx, stats, v->d_work,
                    v->d_work_n, v->work_cap);
            v->launches++;
        } else if (fan_plane) {
            const int cpr = (w + kChunk - 1) / kChunk;
            if (!v->d_work) {
                v->work_cap = 1u << 20;
                CK(cudaMalloc(&v->d_work, sizeof(ull) * v->work_cap));
                CK(cudaMalloc(&v->d_work_n, sizeof(unsigned int)));
            }
            CK(cudaMemsetAsync(v->d_work_n, 0, sizeof(unsigned int), v->stream));
            const int ntx = (cpr + kPlaneTW - 1) / kPlaneTW, nty = (h + kPlaneTH - 1) / kPlaneTH;
            dim3 grid(ntx, m, nty);
#define LP(a, b)                                                                                   \
    k_pnn_plane<a, b, 1, 4><<<grid, 128, 0, v->stream>>>(p, pitch, fstride, w, h, cpr, fps + k0, cal,  \
                                                      v->d_fan, gd, v->acc, bx, stats, v->d_work,     \
                                                      v->d_work_n, v->work_cap, 1u << 20, 2);        \
    k_pnn_work<a, b><<<work_ctas, 256, 0, v->stream>>>(p, pitch, fstride, w, fps + k0, cal, v->d_fan,  \
                                                     gd, v->acc, bx, stats, v->d_work, v->d_work_n,   \
                                                     v->work_cap)
            if (vec) {
                if (box) { LP(true, true); } else { LP(true, false); }
            } else {
                if (box) { LP(false, true); } else { LP(false, false); }
            }
#undef LP
            v->launches += 2;
        } else if (mode == kModeInsert) {
            launch_insert<kModeInsert>(v, vec, skip, box, p, pitch, fstride, w, h, m, fps + k0, cal,
                                       mark, tag, bx, stats);
        } else if (mode == kModeTrilinear && v->tri_kernel == 0) {
            // lane = pixel splat (SVR_TRI_KERNEL=chunk keeps the chunk-per-thread k_insert: tests)
            // small batches (the per-frame path): rows split into column ranges so that every SM
            // gets work (a 480-row frame alone is 60 CTAs)
            const int row_ctas = (h + 7) / 8;
            int nsplit = 1;
            while (nsplit < 8 && (long long)row_ctas * m * nsplit < 2ll * v->num_sms && 64 * nsplit < w) nsplit *= 2;
            dim3 grid(row_ctas, m, nsplit);
            if (skip)
                k_tri_warp<true><<<grid, 256, 0, v->stream>>>(p, pitch, fstride, w, h, fps + k0, v->d_fan, gd, v->tri, stats);
            else
                k_tri_warp<false><<<grid, 256, 0, v->stream>>>(p, pitch, fstride, w, h, fps + k0, v->d_fan, gd, v->tri, stats);
            v->launches++;
        } else if (mode == kModeTrilinear) {
            launch_insert<kModeTrilinear>(v, vec, skip, false, p, pitch, fstride, w, h, m, fps + k0,
                                          cal, mark, tag, nullptr, stats);
        } else {
            launch_insert<kModeFootprint>(v, vec, skip, false, p, pitch, fstride, w, h, m, fps + k0,
                                          cal, mark, tag, nullptr, stats);
        }
        CKL();
    }
    return SVR_OK;
}

static int ensure_stage(svr_volume* v, size_t bytes) {
    if (bytes <= v->stage_bytes) return SVR_OK;
    CK(cudaStreamSynchronize(v->stream));
    CK(cudaStreamSynchronize(v->copy_stream));
    for (int i = 0; i < 2; ++i) {
        cudaFree(v->d_stage[i]);
        cudaFreeHost(v->h_stage[i]);
        v->d_stage[i] = nullptr;
        v->h_stage[i] = nullptr;
    }
    v->stage_bytes = 0;
    for (int i = 0; i < 2; ++i) {
        CK(cudaMalloc(&v->d_stage[i], bytes));
        CK(cudaMallocHost(&v->h_stage[i], bytes));
    }
    v->stage_bytes = bytes;
    return SVR_OK;
}

// Common insert driver: params upload, device or staged-host frames, optional boxes.
static int insert_common(svr_volume* v, int mode, const uint8_t* px, int64_t pitch, int64_t fstride,
                         int32_t w, int32_t h, int32_t n, const svr_rigid* poses,
                         const svr_calib* c, int32_t skip_zero, bool want_box, uint32_t* mark,
                         uint32_t tag, ull* stats) {
    if (n < 0) return fail(SVR_E_INVALID, "negative frame count");
    if (n == 0) return SVR_OK;
    if (!px || !poses) return fail(SVR_E_INVALID, "NULL frames or poses");
    if (int e = check_calib(c, w, h)) return e;
    if (pitch < w) return fail(SVR_E_INVALID, "row pitch %lld < width %d", (long long)pitch, w);
    if (n > 1 && fstride < pitch * (h - 1) + w)
        return fail(SVR_E_INVALID, "frame stride %lld too small", (long long)fstride);
    if (int e = ensure_params(v, n)) return e;
    const PrepCtx ctx = prep_ctx(*c, v->d);
    FrameParams* hp = v->h_params[v->pslot];
    for (int k = 0; k < n; ++k)
        if (int e = make_params(poses[k], ctx, c->scale_x_mm, c->scale_y_mm, &hp[k]))
            return fail(e, "frame %d: %s", k, g_err.c_str());
    if (int e = ensure_fan(v, *c)) return e;
    // k_pnn_tiles shapes every frame of the call fits (FrameParams::lin_fit)
    v->lin_shapes_cur = 0xf | kFitZ1;
    for (int k = 0; k < n; ++k) v->lin_shapes_cur &= hp[k].lin_fit;
    // the upload runs on its own stream, so it overlaps the kernels still queued on v->stream
    // (the previous step's fill / render) instead of sitting on their critical path: ~1 MB for
    // a 2400-frame call, ~20 us at PCIe speed.  d_params2 is double-buffered like h_params: the
    // copy into slot i waits for the last kernel that read it (two calls back).  (Under stream
    // capture the upload stays in-stream: no cross-stream dependencies in a captured graph.)
    v->d_params = v->d_params2[v->pslot];
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(v->stream, &cap_st));
    if (cap_st == cudaStreamCaptureStatusNone) {
        // (after the previous call's insert kernels: they read d_params2[other], the descriptor
        // buffer and the exact-pass work list this call's setup rewrites)
        CK(cudaStreamWaitEvent(v->param_stream, v->ins_done, 0));
        CK(cudaStreamWaitEvent(v->param_stream, v->params_used[v->pslot], 0));
        CK(cudaMemcpyAsync(v->d_params, hp, sizeof(FrameParams) * n, cudaMemcpyHostToDevice,
                           v->param_stream));
        CK(cudaEventRecord(v->params_ev[v->pslot], v->param_stream));
        CK(cudaStreamWaitEvent(v->stream, v->params_ev[v->pslot], 0));
    } else {
        CK(cudaMemcpyAsync(v->d_params, hp, sizeof(FrameParams) * n, cudaMemcpyHostToDevice,
                           v->stream));
        CK(cudaEventRecord(v->params_ev[v->pslot], v->stream));
    }
    const DevCalib cal = dev_calib(*c);
    int* boxes = nullptr;
    if (want_box) {
        if (int e = ensure_boxes(v, n)) return e;
        boxes = v->d_boxes;
        k_box_init<<<(n + 255) / 256, 256, 0, v->stream>>>(boxes, n);
        v->launches++;
        CKL();
    }
    bool pinned = false;
    if (is_device_ptr(px, &pinned)) {
        // one launch chunk (<= 65535 frames) off a capture: K1's setup goes to param_stream too
        v->prep_on_param = cap_st == cudaStreamCaptureStatusNone && n <= 65535;
        const int e = insert_device(v, mode, px, pitch, fstride, w, h, n, v->d_params, cal, skip_zero,
                                    want_box, boxes, mark, tag, stats);
        v->prep_on_param = false;
        CK(cudaEventRecord(v->params_used[v->pslot], v->stream));
        CK(cudaEventRecord(v->ins_done, v->stream));
        return e;
    }
    // host frames: double-buffered pinned staging, H2D on copy_stream overlapped with kernels
    const long long fb = (long long)w * h;                   // packed frame bytes
    const long long pfb = (fb + 31) / 32 * 32;               // 32-B aligned frame stride
    const size_t want = (size_t)std::min<long long>(64ll << 20, pfb * n);
    if (int e = ensure_stage(v, std::max<size_t>(want, (size_t)pfb))) return e;
    const int per = (int)std::max<long long>(1, (long long)v->stage_bytes / pfb);
    const bool contiguous = (pitch == w) && (fstride == fb) && (pfb == fb);
    int b = 0;
    for (int k0 = 0; k0 < n; k0 += per, b ^= 1) {
        const int m = std::min(per, n - k0);
        const uint8_t* src = px + (long long)k0 * fstride;
        // wait until the kernel that last read d_stage[b] is done
        CK(cudaStreamWaitEvent(v->copy_stream, v->ev_free[b], 0));
        if (pinned) {
            if (contiguous) {
                CK(cudaMemcpyAsync(v->d_stage[b], src, (size_t)(pfb * m), cudaMemcpyHostToDevice,
                                   v->copy_stream));
            } else {
                for (int k = 0; k < m; ++k)
                    CK(cudaMemcpy2DAsync(v->d_stage[b] + k * pfb, w, src + (long long)k * fstride,
                                         pitch, w, h, cudaMemcpyHostToDevice, v->copy_stream));
            }
        } else {
            // pageable: pack into the pinned staging buffer once the previous copy drained it
            CK(cudaEventSynchronize(v->ev_h2d[b]));
            for (int k = 0; k < m; ++k) {
                uint8_t* dst = v->h_stage[b] + k * pfb;
                const uint8_t* s = src + (long long)k * fstride;
                if (pitch == w)
                    std::memcpy(dst, s, (size_t)fb);
                else
                    for (int r = 0; r < h; ++r) std::memcpy(dst + (long long)r * w, s + r * pitch, w);
            }
            CK(cudaMemcpyAsync(v->d_stage[b], v->h_stage[b], (size_t)(pfb * m),
                               cudaMemcpyHostToDevice, v->copy_stream));
            CK(cudaEventRecord(v->ev_h2d[b], v->copy_stream));
        }
        CK(cudaEventRecord(v->ev_ready[b], v->copy_stream));
        CK(cudaStreamWaitEvent(v->stream, v->ev_ready[b], 0));
        if (int e = insert_device(v, mode, v->d_stage[b], w, pfb, w, h, m, v->d_params + k0, cal,
                                  skip_zero, want_box, boxes ? boxes + 6 * k0 : nullptr, mark,
                                  tag + (uint32_t)k0, stats))
            return e;
        CK(cudaEventRecord(v->ev_free[b], v->stream));
    }
    CK(cudaEventRecord(v->params_used[v->pslot], v->stream));
    CK(cudaEventRecord(v->ins_done, v->stream));
    return SVR_OK;
}

static svr_box box_from_dev(const int* b) {
    if (b[0] > b[3]) return svr_box{1, 1, 1, 0, 0, 0};
    return svr_box{b[0], b[1], b[2], b[3], b[4], b[5]};
}

extern "C" int svr_insert_frames(svr_volume* v, const uint8_t* px, int64_t pitch, int64_t fstride,
                                 int32_t w, int32_t h, int32_t n, const svr_rigid* poses,
                                 const svr_calib* c, int32_t skip_zero, svr_box* dirty_out,
                                 svr_box* union_out) {
    NvtxRange nvtx_("svr_insert_frames");
    VOL_CHECK(v);
    const bool want_box = dirty_out || union_out;
    const int mode = v->d.accum == SVR_ACC_TRILINEAR ? kModeTrilinear : kModeInsert;
    if (want_box && mode == kModeTrilinear)
        return fail(SVR_E_INVALID, "dirty boxes are reported for PNN volumes only");
    if (int e = insert_common(v, mode, px, pitch, fstride, w, h, n, poses, c, skip_zero, want_box,
                              nullptr, 0, v->d_stats))
        return e;
    v->frames += (uint64_t)std::max(n, 0);
    if (want_box && n > 0) {
        CK(cudaMemcpyAsync(v->h_boxes, v->d_boxes, sizeof(int) * 6 * n, cudaMemcpyDeviceToHost,
                           v->stream));
        CK(cudaStreamSynchronize(v->stream));
        svr_box u{1, 1, 1, 0, 0, 0};
        for (int k = 0; k < n; ++k) {
            svr_box b = box_from_dev(v->h_boxes + 6 * k);
            if (dirty_out) dirty_out[k] = b;
            if (b.x0 > b.x1) continue;
            if (u.x0 > u.x1) {
                u = b;
            } else {
                u.x0 = std::min(u.x0, b.x0); u.y0 = std::min(u.y0, b.y0); u.z0 = std::min(u.z0, b.z0);
                u.x1 = std::max(u.x1, b.x1); u.y1 = std::max(u.y1, b.y1); u.z1 = std::max(u.z1, b.z1);
            }
        }
        if (union_out) *union_out = u;
    } else if (union_out) {
        *union_out = svr_box{1, 1, 1, 0, 0, 0};
    }
    return SVR_OK;
}

extern "C" int svr_insert_frame(svr_volume* v, const uint8_t* px, int64_t pitch, int32_t w,
                                int32_t h, const svr_rigid* pose, const svr_calib* c,
                                int32_t skip_zero, svr_box* dirty_out) {
    svr_box b;
    int e = svr_insert_frames(v, px, pitch, pitch * h, w, h, 1, pose, c, skip_zero, &b, nullptr);
    if (e) return e;
    if (dirty_out) *dirty_out = b;
    return SVR_OK;
}

static bool clip_box(const svr_volume* v, const svr_box* in, Box* out) {
    svr_box b = in ? *in : svr_box{0, 0, v->d.z_begin, v->d.nx - 1, v->d.ny - 1, v->d.z_end - 1};
    b.x0 = std::max(b.x0, 0);
    b.y0 = std::max(b.y0, 0);
    b.z0 = std::max(b.z0, v->d.z_begin);
    b.x1 = std::min(b.x1, v->d.nx - 1);
    b.y1 = std::min(b.y1, v->d.ny - 1);
    b.z1 = std::min(b.z1, v->d.z_end - 1);
    *out = Box{b.x0, b.y0, b.z0, b.x1, b.y1, b.z1};
    return b.x0 <= b.x1 && b.y0 <= b.y1 && b.z0 <= b.z1;
}

// Upload a small region table to the handle's device scratch (stream-ordered: the copy runs after
// every earlier kernel of the stream, so one buffer serves consecutive launches).
static int upload_tiles(svr_volume* v, const void* host, size_t bytes, void** dev) {
    constexpr int K = svr_volume::kTileSlots;
    if (!v->tiles_ev[0])
        for (int i = 0; i < K; ++i) CK(cudaEventCreateWithFlags(&v->tiles_ev[i], cudaEventDisableTiming));
    // the previous slot's consumers were enqueued on its stream since its upload: mark them
    if (v->tiles_prev >= 0) CK(cudaEventRecord(v->tiles_ev[v->tiles_prev], v->tiles_prev_stream));
    const int s = (v->tiles_prev + 1) % K;
    CK(cudaEventSynchronize(v->tiles_ev[s]));  // this slot's last consumers (K uploads ago) are done
    if (bytes > v->tiles_cap) {
        CK(cudaDeviceSynchronize());
        const size_t cap = std::max<size_t>(bytes, 4096);
        for (int i = 0; i < K; ++i) {
            cudaFree(v->d_tiles[i]);
            cudaFreeHost(v->h_tiles[i]);
            v->d_tiles[i] = v->h_tiles[i] = nullptr;
        }
        v->tiles_cap = 0;
        for (int i = 0; i < K; ++i) {
            CK(cudaMalloc(&v->d_tiles[i], cap));
            CK(cudaMallocHost(&v->h_tiles[i], cap));
        }
        v->tiles_cap = cap;
    }
    std::memcpy(v->h_tiles[s], host, bytes);
    // (off a capture: the small H2D goes on param_stream -- the slot's consumers are done, see
    // above -- so it does not queue behind the kernels already on v->stream)
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(v->stream, &cap_st));
    if (cap_st == cudaStreamCaptureStatusNone) {
        CK(cudaMemcpyAsync(v->d_tiles[s], v->h_tiles[s], bytes, cudaMemcpyHostToDevice, v->param_stream));
        CK(cudaEventRecord(v->ev_tiles_up, v->param_stream));
        CK(cudaStreamWaitEvent(v->stream, v->ev_tiles_up, 0));
    } else {
        CK(cudaMemcpyAsync(v->d_tiles[s], v->h_tiles[s], bytes, cudaMemcpyHostToDevice, v->stream));
    }
    v->tiles_prev = s;
    v->tiles_prev_stream = v->stream;
    *dev = v->d_tiles[s];
    return SVR_OK;
}

static dim3 grid_1d(long long n) {
    const long long gx = std::min<long long>(n, 65535);
    return dim3((unsigned)gx, (unsigned)((n + gx - 1) / gx));
}

// Launch the fill over a list of clipped, non-empty boxes: the BASELINE mean r = 1 by
// k_fill_warp (one launch over all boxes), everything else (SPEC median, mean r = 2) by
// k_fill_generic per box.
static int fill_boxes(svr_volume* v, const std::vector<Box>& bs, int32_t mode, int32_t radius, bool count) {
    const GridDev g = dev_grid(v->d);
    if (mode == SVR_FILL_MEAN && radius == 1) {
        std::vector<BoxTiles> bt;
        long long total = 0;
        auto tile = [&](int zc) {
            bt.clear();
            total = 0;
            for (const Box& b : bs) {
                BoxTiles t;
                t.b = b;
                t.ntx = (b.x1 - b.x0 + 1 + 29) / 30;  // k_fill_warp: 30 columns x 4 warps of TY rows
                t.nty = (b.y1 - b.y0 + 1 + 4 * SVR_FILL_TY - 1) / (4 * SVR_FILL_TY);
                t.first = total;
                total += (long long)t.ntx * t.nty * ((b.z1 - b.z0 + 1 + zc - 1) / zc);
                bt.push_back(t);
            }
        };
        // planes per march: 32, unless that leaves fewer than ~8 CTAs per SM (a slab's share of a
        // multi-GPU split, small incremental boxes): then 16 or 8
        int zc = SVR_FILL_ZC;
        tile(zc);
        const long long want = 8ll * v->num_sms;
        while (zc > 8 && total < want) {
            zc /= 2;
            tile(zc);
        }
        void* d = nullptr;
        if (int e = upload_tiles(v, bt.data(), sizeof(BoxTiles) * bt.size(), &d)) return e;
        const dim3 grd = grid_1d(total);
        const BoxTiles* dt = (const BoxTiles*)d;
        const int nb = (int)bt.size();
#define FW(Z, C) k_fill_warp<Z, 1, SVR_FILL_TY, C><<<grd, 128, 0, v->stream>>>(v->acc, v->fill, g, dt, nb, C ? v->d_counter : nullptr)
        if (count) {
            if (zc == 8) FW(8, true);
            else if (zc == 16) FW(16, true);
            else FW(32, true);
        } else {
            if (zc == 8) FW(8, false);
            else if (zc == 16) FW(16, false);
            else FW(32, false);
        }
#undef FW
        v->launches++;
        CKL();
        return SVR_OK;
    }
    for (const Box& b : bs) {
        const long long nv = (long long)(b.x1 - b.x0 + 1) * (b.y1 - b.y0 + 1) * (b.z1 - b.z0 + 1);
        k_fill_generic<<<(unsigned)((nv + 255) / 256), 256, 0, v->stream>>>(v->acc, v->fill, g, b, radius, mode, v->d_counter);
        v->launches++;
        CKL();
    }
    return SVR_OK;
}

static int check_fill_args(svr_volume* v, int32_t mode, int32_t radius) {
    if (!v->acc) return fail(SVR_E_INVALID, "fill_holes needs a PNN volume");
    if (mode != SVR_FILL_MEAN && mode != SVR_FILL_MEDIAN) return fail(SVR_E_INVALID, "unknown fill mode");
    if (radius < 1 || radius > 8) return fail(SVR_E_INVALID, "fill radius must be in [1,8]");
    // the mean fill code carries the neighbour sum in 16 bits: (2r+1)^3 - 1 neighbours of <= 255
    // fit for r <= 2 (31620), not beyond
    if (mode == SVR_FILL_MEAN && radius > 2) return fail(SVR_E_INVALID, "mean fill supports radius <= 2");
    if (mode == SVR_FILL_MEAN && (2 * radius + 1) * (2 * radius + 1) * (2 * radius + 1) * 255 > 65535)
        return fail(SVR_E_INVALID, "mean fill radius too large for the 16-bit fill payload");
    return SVR_OK;
}

static int finish_count(svr_volume* v, int64_t* filled_out) {
    if (filled_out) {
        ull c = 0;
        CK(cudaMemcpyAsync(&c, v->d_counter, sizeof(ull), cudaMemcpyDeviceToHost, v->stream));
        CK(cudaStreamSynchronize(v->stream));
        *filled_out = (int64_t)c;
    }
    return SVR_OK;
}

extern "C" int svr_fill_holes(svr_volume* v, const svr_box* region, int32_t mode, int32_t radius,
                              int64_t* filled_out) {
    NvtxRange nvtx_("svr_fill_holes");
    VOL_CHECK(v);
    if (int e = check_fill_args(v, mode, radius)) return e;
    Box b;
    const bool any = clip_box(v, region, &b);
    if (filled_out) CK(cudaMemsetAsync(v->d_counter, 0, sizeof(ull), v->stream));
    v->fill_mode = mode;
    if (any)
        if (int e = fill_boxes(v, std::vector<Box>{b}, mode, radius, filled_out != nullptr)) return e;
    return finish_count(v, filled_out);
}

extern "C" int svr_fill_holes_boxes(svr_volume* v, const svr_box* regions, int32_t n, int32_t mode,
                                    int32_t radius, int64_t* filled_out) {
    NvtxRange nvtx_("svr_fill_holes_boxes");
    VOL_CHECK(v);
    if (int e = check_fill_args(v, mode, radius)) return e;
    if (n < 0 || (n > 0 && !regions)) return fail(SVR_E_INVALID, "bad region list");
    std::vector<Box> bs;
    for (int i = 0; i < n; ++i) {
        Box b;
        if (clip_box(v, &regions[i], &b)) bs.push_back(b);
    }
    if (filled_out) CK(cudaMemsetAsync(v->d_counter, 0, sizeof(ull), v->stream));
    v->fill_mode = mode;
    if (!bs.empty())
        if (int e = fill_boxes(v, bs, mode, radius, filled_out != nullptr)) return e;
    return finish_count(v, filled_out);
}

// Integer render parameters — identical formula to oracle orc_render_ints.
static void render_ints(const svr_render_params* p, double vx, int ny, int* ylo, int* yhi,
                        int* above, int* below) {
    int lo = (int)std::ceil(p->depth_lo_mm / vx - 1e-6);
    int hi = (int)std::floor(p->depth_hi_mm / vx + 1e-6);
    if (lo < 0) lo = 0;
    if (hi > ny - 2) hi = ny - 2;
    *ylo = lo;
    *yhi = hi;
    *above = (int)std::lround(p->band_above_mm / vx);
    *below = (int)std::lround(p->band_below_mm / vx);
}

// Depth/band column regions of one dirty box (or the whole slab for dirty == NULL), clipped.
static bool render_regions(const svr_volume* v, const svr_box* dirty, int fr, int R, ColTiles* d,
                           ColTiles* m) {
    const int zb = v->d.z_begin, ze = v->d.z_end - 1, nxm = v->d.nx - 1;
    int dx0 = 0, dx1 = nxm, dz0 = zb, dz1 = ze;
    if (dirty) {
        if (dirty->x0 > dirty->x1) return false;
        if (dirty->x1 + fr + R < 0 || dirty->x0 - fr - R > nxm || dirty->z1 + fr + R < zb ||
            dirty->z0 - fr - R > ze)
            return false;
        dx0 = dirty->x0 - fr;
        dx1 = dirty->x1 + fr;
        dz0 = dirty->z0 - fr;
        dz1 = dirty->z1 + fr;
    }
    int mx0 = dx0 - R, mx1 = dx1 + R, mz0 = dz0 - R, mz1 = dz1 + R;
    auto cx = [&](int a) { return std::min(std::max(a, 0), nxm); };
    auto cz = [&](int a) { return std::min(std::max(a, zb), ze); };
    *d = ColTiles{cx(dx0), cx(dx1), cz(dz0), cz(dz1), 0, 0};
    *m = ColTiles{cx(mx0), cx(mx1), cz(mz0), cz(mz1), 0, 0};
    return true;
}

static long long tile_cols(std::vector<ColTiles>& ct, int cols_per_cta = 128) {
    long long total = 0;
    for (ColTiles& t : ct) {
        t.ntx = (t.x1 - t.x0 + cols_per_cta) / cols_per_cta;
        t.first = total;
        total += (long long)t.ntx * (t.z1 - t.z0 + 1);
    }
    return total;
}

static int render_boxes(svr_volume* v, const svr_box* dirty, int n, int32_t fill_radius,
                        const svr_render_params* p) {
    if (!v->acc && !v->tri) return fail(SVR_E_INVALID, "render needs a volume");
    if (!p) return fail(SVR_E_INVALID, "render params NULL");
    if (p->median_radius < 0 || p->median_radius > 2)
        return fail(SVR_E_INVALID, "median_radius must be 0, 1 or 2");
    if (fill_radius < 0) return fail(SVR_E_INVALID, "negative fill radius");
    int ylo, yhi, above, below;
    render_ints(p, v->d.voxel_mm, v->d.ny, &ylo, &yhi, &above, &below);
    std::vector<ColTiles> dt, mt;
    for (int i = 0; i < std::max(n, 1); ++i) {
        ColTiles d, m;
        if (render_regions(v, dirty ? &dirty[i] : nullptr, fill_radius, p->median_radius, &d, &m)) {
            dt.push_back(d);
            mt.push_back(m);
        }
    }
    if (dt.empty()) return SVR_OK;
    const long long nd = tile_cols(dt, 128 / SVR_DEPTH_SEG), nm = tile_cols(mt);  // k_depth<SEG>: SEG threads per column
    // one upload holds both tables: [dt | mt]
    std::vector<ColTiles> both(dt);
    both.insert(both.end(), mt.begin(), mt.end());
    void* d = nullptr;
    if (int e = upload_tiles(v, both.data(), sizeof(ColTiles) * both.size(), &d)) return e;
    const ColTiles* ddt = (const ColTiles*)d;
    const ColTiles* dmt = ddt + dt.size();
    const GridDev g = dev_grid(v->d);
    if (v->tri) {  // trilinear volume: f = wsum / weight, no fill layer
        k_depth<SVR_DEPTH_SEG, true><<<grid_1d(nd), 128, 0, v->stream>>>(nullptr, nullptr, g, ddt, (int)dt.size(), ylo,
                                                              yhi, p->fill_mode, v->r_depth, v->tri);
        v->launches++;
        CKL();
        k_band<true><<<grid_1d(nm), 128, 0, v->stream>>>(nullptr, nullptr, g, dmt, (int)mt.size(),
                                                         p->median_radius, above, below, p->fill_mode,
                                                         v->r_depth, v->r_mdepth, v->r_mean, v->r_max,
                                                         v->gt, v->tri);
        v->launches++;
        CKL();
        return SVR_OK;
    }
    k_depth<SVR_DEPTH_SEG><<<grid_1d(nd), 128, 0, v->stream>>>(v->acc, v->fill, g, ddt, (int)dt.size(), ylo, yhi,
                                                    p->fill_mode, v->r_depth);
    v->launches++;
    CKL();
    k_band<false><<<grid_1d(nm), 128, 0, v->stream>>>(v->acc, v->fill, g, dmt, (int)mt.size(), p->median_radius,
                                                above, below, p->fill_mode, v->r_depth, v->r_mdepth,
                                                v->r_mean, v->r_max, v->gt);
    v->launches++;
    CKL();
    return SVR_OK;
}

extern "C" int svr_render_coronal(svr_volume* v, const svr_box* dirty, int32_t fill_radius,
                                  const svr_render_params* p) {
    NvtxRange nvtx_("svr_render_coronal");
    VOL_CHECK(v);
    return render_boxes(v, dirty, dirty ? 1 : 0, fill_radius, p);
}

extern "C" int svr_render_coronal_boxes(svr_volume* v, const svr_box* dirty, int32_t n,
                                        int32_t fill_radius, const svr_render_params* p) {
    NvtxRange nvtx_("svr_render_coronal_boxes");
    VOL_CHECK(v);
    if (n <= 0 || !dirty) return n == 0 ? SVR_OK : fail(SVR_E_INVALID, "bad region list");
    return render_boxes(v, dirty, n, fill_radius, p);
}

static int read_coronal(svr_volume* v, int32_t z0, int32_t z1, float* mean, float* maxv, int32_t* depth,
                        bool sync);

extern "C" int svr_read_coronal(svr_volume* v, int32_t z0, int32_t z1, float* mean, float* maxv,
                                int32_t* depth) {
    return read_coronal(v, z0, z1, mean, maxv, depth, true);
}

extern "C" int svr_read_coronal_async(svr_volume* v, int32_t z0, int32_t z1, float* mean, float* maxv,
                                      int32_t* depth) {
    return read_coronal(v, z0, z1, mean, maxv, depth, false);
}

static int read_coronal(svr_volume* v, int32_t z0, int32_t z1, float* mean, float* maxv, int32_t* depth,
                        bool sync) {
    VOL_CHECK(v);
    if (!v->r_mean) return fail(SVR_E_INVALID, "volume has no render layer");
    if (z0 < v->d.z_begin || z1 >= v->d.z_end || z0 > z1)
        return fail(SVR_E_INVALID, "rows [%d,%d] outside slab [%d,%d)", z0, z1, v->d.z_begin, v->d.z_end);
    const size_t off = (size_t)(z0 - v->d.z_begin) * v->d.nx, cnt = (size_t)(z1 - z0 + 1) * v->d.nx;
    if (mean) CK(cudaMemcpyAsync(mean, v->r_mean + off, cnt * sizeof(float), cudaMemcpyDefault, v->stream));
    if (maxv) CK(cudaMemcpyAsync(maxv, v->r_max + off, cnt * sizeof(float), cudaMemcpyDefault, v->stream));
    if (depth) CK(cudaMemcpyAsync(depth, v->r_mdepth + off, cnt * sizeof(int), cudaMemcpyDefault, v->stream));
    if (sync) CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_coronal_projection(svr_volume* v, int32_t mode, int32_t axis, int32_t use_fills,
                                      uint8_t* out) {
    VOL_CHECK(v);
    if (!v->acc) return fail(SVR_E_INVALID, "projection needs a PNN volume");
    if (axis < 0 || axis > 2) return fail(SVR_E_INVALID, "depth_axis must be 0, 1 or 2");
    if (mode != SVR_PROJ_MAX && mode != SVR_PROJ_MEAN) return fail(SVR_E_INVALID, "unknown projection mode");
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    const int dims[3] = {v->d.nx, v->d.ny, v->d.z_end - v->d.z_begin};
    const int a0 = axis == 0 ? 1 : 0, a1 = axis == 2 ? 1 : 2;
    const long long n = (long long)dims[a0] * dims[a1];
    uint8_t* tmp = nullptr;
    CK(cudaMallocAsync(&tmp, n, v->stream));
    k_project<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->acc, v->fill, dev_grid(v->d), axis,
                                                                 mode, use_fills, v->fill_mode, tmp);
    v->launches++;
    CKL();
    CK(cudaMemcpyAsync(out, tmp, n, cudaMemcpyDefault, v->stream));
    CK(cudaFreeAsync(tmp, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

static int read_box_common(svr_volume* v, const svr_box* box, Box* b, long long* n) {
    if (box && (box->x0 < 0 || box->y0 < 0 || box->z0 < v->d.z_begin || box->x1 >= v->d.nx ||
                box->y1 >= v->d.ny || box->z1 >= v->d.z_end || box->x0 > box->x1 ||
                box->y0 > box->y1 || box->z0 > box->z1))
        return fail(SVR_E_INVALID, "box outside the stored slab or empty");
    clip_box(v, box, b);
    *n = (long long)(b->x1 - b->x0 + 1) * (b->y1 - b->y0 + 1) * (b->z1 - b->z0 + 1);
    return SVR_OK;
}

extern "C" int svr_read_accumulators(svr_volume* v, const svr_box* box, uint32_t* sum, uint16_t* cnt) {
    VOL_CHECK(v);
    if (!v->acc) return fail(SVR_E_INVALID, "not a PNN volume");
    Box b;
    long long n;
    if (int e = read_box_common(v, box, &b, &n)) return e;
    uint32_t* ts = nullptr;
    uint16_t* tc = nullptr;
    if (sum) CK(cudaMallocAsync(&ts, n * 4, v->stream));
    if (cnt) CK(cudaMallocAsync(&tc, n * 2, v->stream));
    CK(cudaMemsetAsync(v->d_counter + 1, 0, sizeof(ull), v->stream));
    k_read_acc<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->acc, dev_grid(v->d), b, ts, tc,
                                                                  v->d_counter + 1);
    v->launches++;
    CKL();
    if (sum) CK(cudaMemcpyAsync(sum, ts, n * 4, cudaMemcpyDefault, v->stream));
    if (cnt) CK(cudaMemcpyAsync(cnt, tc, n * 2, cudaMemcpyDefault, v->stream));
    ull sat = 0;
    CK(cudaMemcpyAsync(&sat, v->d_counter + 1, sizeof(ull), cudaMemcpyDeviceToHost, v->stream));
    if (ts) CK(cudaFreeAsync(ts, v->stream));
    if (tc) CK(cudaFreeAsync(tc, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    if (sat) {
        // record in stats: the most voxels above the caps any readout has seen
        // (a readout of a sub-box must not erase a larger count from an earlier one)
        ull h[kStCount];
        CK(cudaMemcpy(h, v->d_stats, sizeof h, cudaMemcpyDeviceToHost));
        h[kStSaturated] = std::max<ull>(h[kStSaturated], sat);
        CK(cudaMemcpy(v->d_stats, h, sizeof h, cudaMemcpyHostToDevice));
    }
    return SVR_OK;
}

extern "C" int svr_write_accumulators(svr_volume* v, const svr_box* box, const uint32_t* sum,
                                      const uint16_t* cnt) {
    VOL_CHECK(v);
    if (!v->acc) return fail(SVR_E_INVALID, "not a PNN volume");
    if (!sum || !cnt) return fail(SVR_E_INVALID, "sum and count are required");
    Box b;
    long long n;
    if (int e = read_box_common(v, box, &b, &n)) return e;
    uint32_t* ts = nullptr;
    uint16_t* tc = nullptr;
    CK(cudaMallocAsync(&ts, n * 4, v->stream));
    CK(cudaMallocAsync(&tc, n * 2, v->stream));
    CK(cudaMemcpyAsync(ts, sum, n * 4, cudaMemcpyDefault, v->stream));
    CK(cudaMemcpyAsync(tc, cnt, n * 2, cudaMemcpyDefault, v->stream));
    k_write_acc<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->acc, dev_grid(v->d), b, ts, tc);
    v->launches++;
    CKL();
    // the fill layer is derived from the accumulators: stale now, so cleared (re-run fill_holes)
    CK(cudaMemsetAsync(v->fill, 0, sizeof(uint32_t) * v->nvox, v->stream));
    CK(cudaFreeAsync(ts, v->stream));
    CK(cudaFreeAsync(tc, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_read_values(svr_volume* v, const svr_box* box, int32_t apply_fills, uint8_t* out) {
    VOL_CHECK(v);
    if (!v->acc) return fail(SVR_E_INVALID, "not a PNN volume");
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    Box b;
    long long n;
    if (int e = read_box_common(v, box, &b, &n)) return e;
    uint8_t* t = nullptr;
    CK(cudaMallocAsync(&t, n, v->stream));
    k_read_values<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->acc, v->fill, dev_grid(v->d), b,
                                                                     apply_fills, v->fill_mode, t);
    v->launches++;
    CKL();
    CK(cudaMemcpyAsync(out, t, n, cudaMemcpyDefault, v->stream));
    CK(cudaFreeAsync(t, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_export_slices_x(svr_volume* v, int32_t apply_fills, uint8_t* out) {
    VOL_CHECK(v);
    if (!v->acc) return fail(SVR_E_INVALID, "not a PNN volume");
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    const GridDev g = dev_grid(v->d);
    const long long n = (long long)g.nx * g.ny * g.nzl;
    uint8_t* t = nullptr;
    CK(cudaMallocAsync(&t, n, v->stream));
    const dim3 grd((g.nx + 31) / 32, (g.ny + 31) / 32, g.nzl);
    k_slices_x<<<grd, dim3(32, 8), 0, v->stream>>>(v->acc, v->fill, g, apply_fills, v->fill_mode, t);
    v->launches++;
    CKL();
    CK(cudaMemcpyAsync(out, t, n, cudaMemcpyDefault, v->stream));
    CK(cudaFreeAsync(t, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_export_slices(svr_volume* v, const char* dir, int32_t apply_fills, int32_t digits,
                                 int32_t* files_out) {
    VOL_CHECK(v);
    if (!dir) return fail(SVR_E_INVALID, "directory is NULL");
    if (digits < 1 || digits > 9) return fail(SVR_E_INVALID, "digits must be in [1,9]");
    const GridDev g = dev_grid(v->d);
    std::vector<uint8_t> h((size_t)g.nx * g.ny * g.nzl);
    if (int e = svr_export_slices_x(v, apply_fills, h.data())) return e;
    for (int x = 0; x < g.nx; ++x) {
        char path[4096];
        if (std::snprintf(path, sizeof path, "%s/%0*d.pgm", dir, digits, x) >= (int)sizeof path)
            return fail(SVR_E_INVALID, "slice path too long");
        if (int e = svr_pgm_write(path, h.data() + (size_t)x * g.ny * g.nzl, g.ny, g.ny, g.nzl)) return e;
    }
    if (files_out) *files_out = g.nx;
    return SVR_OK;
}

extern "C" int svr_export_volume(svr_volume* v, const char* path, int32_t apply_fills) {
    VOL_CHECK(v);
    if (!path) return fail(SVR_E_INVALID, "path is NULL");
    if (!v->acc) return fail(SVR_E_INVALID, "not a PNN volume");
    std::vector<uint8_t> h((size_t)v->d.nx * v->d.ny * (v->d.z_end - v->d.z_begin));
    if (int e = svr_read_values(v, nullptr, apply_fills, h.data())) return e;
    return svr_write_raw(path, h.data(), (int64_t)h.size());
}

extern "C" int svr_read_fill(svr_volume* v, const svr_box* box, uint32_t* out) {
    VOL_CHECK(v);
    if (!v->fill) return fail(SVR_E_INVALID, "not a PNN volume");
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    Box b;
    long long n;
    if (int e = read_box_common(v, box, &b, &n)) return e;
    uint32_t* t = nullptr;
    CK(cudaMallocAsync(&t, n * 4, v->stream));
    k_read_fill<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->acc, v->fill, dev_grid(v->d), b, t);
    v->launches++;
    CKL();
    CK(cudaMemcpyAsync(out, t, n * 4, cudaMemcpyDefault, v->stream));
    CK(cudaFreeAsync(t, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_read_trilinear(svr_volume* v, const svr_box* box, float* ws, float* wt) {
    VOL_CHECK(v);
    if (!v->tri) return fail(SVR_E_INVALID, "not a trilinear volume");
    Box b;
    long long n;
    if (int e = read_box_common(v, box, &b, &n)) return e;
    float *a = nullptr, *c = nullptr;
    if (ws) CK(cudaMallocAsync(&a, n * 4, v->stream));
    if (wt) CK(cudaMallocAsync(&c, n * 4, v->stream));
    k_read_tri<<<(unsigned)((n + 255) / 256), 256, 0, v->stream>>>(v->tri, dev_grid(v->d), b, a, c);
    v->launches++;
    CKL();
    if (ws) CK(cudaMemcpyAsync(ws, a, n * 4, cudaMemcpyDefault, v->stream));
    if (wt) CK(cudaMemcpyAsync(wt, c, n * 4, cudaMemcpyDefault, v->stream));
    if (a) CK(cudaFreeAsync(a, v->stream));
    if (c) CK(cudaFreeAsync(c, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return SVR_OK;
}

extern "C" int svr_get_stats(svr_volume* v, svr_stats* out) {
    VOL_CHECK(v);
    if (!out) return fail(SVR_E_INVALID, "out is NULL");
    ull h[kStCount];
    CK(cudaMemcpyAsync(h, v->d_stats, sizeof h, cudaMemcpyDeviceToHost, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    out->frames_inserted = v->frames;
    out->pixels_inserted = h[kStInserted];
    out->pixels_oob = h[kStOob];
    out->pixels_skipped_zero = h[kStSkipped];
    out->pixels_saturated = h[kStSaturated];
    out->exact_fallbacks = h[kStFallback];
    out->kernel_launches = v->launches;
    out->chunks_deferred = h[kStDeferred];
    out->tiles_table = h[kStTiles];
    out->graph_captures = v->fg.captures;
    return SVR_OK;
}

extern "C" int svr_count_footprint(svr_volume* v, const uint8_t* px, int64_t pitch, int64_t fstride,
                                   int32_t w, int32_t h, int32_t n, const svr_rigid* poses,
                                   const svr_calib* c, int32_t skip_zero, int64_t* distinct) {
    VOL_CHECK(v);
    if (!distinct) return fail(SVR_E_INVALID, "distinct_out is NULL");
    if (n <= 0) return SVR_OK;
    uint32_t* mark = nullptr;
    ull* cnt = nullptr;
    CK(cudaMallocAsync(&mark, sizeof(uint32_t) * v->nvox, v->stream));
    CK(cudaMemsetAsync(mark, 0, sizeof(uint32_t) * v->nvox, v->stream));
    CK(cudaMallocAsync(&cnt, sizeof(ull) * n, v->stream));
    CK(cudaMemsetAsync(cnt, 0, sizeof(ull) * n, v->stream));
    int rc = SVR_OK;
    // one frame per launch: the tag (frame index + 1) identifies "already counted this frame"
    for (int k = 0; k < n && rc == SVR_OK; ++k)
        rc = insert_common(v, kModeFootprint, px + (long long)k * fstride, pitch, fstride, w, h, 1,
                           poses + k, c, skip_zero, false, mark, (uint32_t)k + 1u, cnt + k);
    std::vector<ull> hc(n);
    if (rc == SVR_OK) {
        CK(cudaMemcpyAsync(hc.data(), cnt, sizeof(ull) * n, cudaMemcpyDeviceToHost, v->stream));
        CK(cudaStreamSynchronize(v->stream));
        for (int k = 0; k < n; ++k) distinct[k] = (int64_t)hc[k];
    }
    cudaFreeAsync(mark, v->stream);
    cudaFreeAsync(cnt, v->stream);
    cudaStreamSynchronize(v->stream);
    return rc;
}

extern "C" int svr_synth_frames(void* dst, int32_t w, int32_t h, int32_t first, int32_t n,
                                const svr_calib* c, const svr_rigid* poses, int32_t kind, uint64_t seed,
                                int device, void* stream) {
    if (!dst || !c || !poses || n <= 0 || w <= 0 || h <= 0) return fail(SVR_E_INVALID, "bad synth arguments");
    if (n > 65535) return fail(SVR_E_INVALID, "synth at most 65535 frames per call");
    CK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    svr_rigid* dp = nullptr;
    CK(cudaMallocAsync(&dp, sizeof(svr_rigid) * n, s));
    CK(cudaMemcpyAsync(dp, poses, sizeof(svr_rigid) * n, cudaMemcpyHostToDevice, s));
    const long long px = (long long)w * h;
    dim3 grd((unsigned)std::min<long long>((px + 255) / 256, 1024), n);
    k_synth<<<grd, 256, 0, s>>>((uint8_t*)dst, w, h, first, dev_calib(*c), dp, kind, (ull)seed);
    CKL();
    CK(cudaFreeAsync(dp, s));
    CK(cudaStreamSynchronize(s));
    return SVR_OK;
}


// ---------------------------------------------------------------- per-frame graph
static constexpr size_t kFgTileBytes = sizeof(BoxTiles) + 2 * sizeof(ColTiles);

static bool fg_matches(const FrameGraph& f, int w, int h, int fr, const svr_calib& c,
                       const svr_render_params& p, long long nf, long long nd, long long nb) {
    return f.ready && f.w == w && f.h == h && f.fr == fr && !std::memcmp(&f.cal, &c, sizeof c) &&
           !std::memcmp(&f.rp, &p, sizeof p) && nf <= f.fill_ctas && nd <= f.depth_ctas && nb <= f.band_ctas;
}

static int fg_capture(svr_volume* v, int w, int h, int fr, const svr_calib& c, const svr_render_params& p,
                      long long nf, long long nd, long long nb) {
    FrameGraph& f = v->fg;
    CK(cudaStreamSynchronize(v->stream));
    if (f.exec) cudaGraphExecDestroy(f.exec);
    if (f.graph) cudaGraphDestroy(f.graph);
    f.exec = nullptr;
    f.graph = nullptr;
    f.ready = false;
    if (f.w != w || f.h != h || !f.d_frame) {
        cudaFree(f.d_frame);
        cudaFreeHost(f.h_frame);
        f.d_frame = nullptr;
        f.h_frame = nullptr;
        CK(cudaMalloc(&f.d_frame, (size_t)w * h));
        CK(cudaMallocHost(&f.h_frame, (size_t)w * h));
    }
    if (!f.d_fp) {
        CK(cudaMalloc(&f.d_fp, sizeof(FrameParams)));
        CK(cudaMallocHost(&f.h_fp, sizeof(FrameParams)));
        CK(cudaMalloc(&f.d_tiles, kFgTileBytes));
        CK(cudaMallocHost(&f.h_tiles, kFgTileBytes));
        CK(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
    }
    if (!v->d_work) {
        v->work_cap = 1u << 20;
        CK(cudaMalloc(&v->d_work, sizeof(ull) * v->work_cap));
        CK(cudaMalloc(&v->d_work_n, sizeof(unsigned int)));
    }
    if (int e = ensure_fan(v, c)) return e;
    if (int e = ensure_desc(v, (long long)(w / 32 + 1) * (h / 64 + 1), 1)) return e;
    if (c.probe == SVR_PROBE_FAN)
        if (int e = ensure_fan_bufs(v, (long long)(w / 128 + 1) * (h / kFanLines + 1), h)) return e;
    // bounds with headroom: later frames of a sweep rarely need a larger graph
    f.fill_ctas = std::max(f.fill_ctas, nf + nf / 4 + 1);
    f.depth_ctas = std::max(f.depth_ctas, nd + nd / 4 + 1);
    f.band_ctas = std::max(f.band_ctas, nb + nb / 4 + 1);
    int ylo, yhi, above, below;
    render_ints(&p, v->d.voxel_mm, v->d.ny, &ylo, &yhi, &above, &below);
    const GridDev g = dev_grid(v->d);
    const DevCalib dc = dev_calib(c);
    const long long l0 = v->launches;
    CK(cudaStreamBeginCapture(v->stream, cudaStreamCaptureModeThreadLocal));
    cudaMemcpyAsync(f.d_fp, f.h_fp, sizeof(FrameParams), cudaMemcpyHostToDevice, v->stream);
    cudaMemcpyAsync(f.d_tiles, f.h_tiles, kFgTileBytes, cudaMemcpyHostToDevice, v->stream);
    const bool tri = v->tri != nullptr;  // trilinear volume: splat, then depth / band on wsum / weight (no fill layer)
    int e = insert_device(v, tri ? kModeTrilinear : kModeInsert, f.d_frame, w, (long long)w * h, w, h, 1, f.d_fp, dc,
                          false, false, nullptr, nullptr, 0, v->d_stats);
    const BoxTiles* bt = (const BoxTiles*)f.d_tiles;
    const ColTiles* dt = (const ColTiles*)(f.d_tiles + sizeof(BoxTiles));
    const ColTiles* mt = dt + 1;
    if (!e && tri) {
        k_depth<8, true><<<grid_1d(f.depth_ctas), 128, 0, v->stream>>>(nullptr, nullptr, g, dt, 1, ylo, yhi, p.fill_mode,
                                                                        v->r_depth, v->tri);
        k_band<true><<<grid_1d(f.band_ctas), 128, 0, v->stream>>>(nullptr, nullptr, g, mt, 1, p.median_radius, above,
                                                                   below, p.fill_mode, v->r_depth, v->r_mdepth,
                                                                   v->r_mean, v->r_max, v->gt, v->tri);
    } else if (!e) {
        // 2-plane marches: a single frame's box is shallow in z, short marches cut its latency
        k_fill_warp<2, 1, 8, false><<<grid_1d(f.fill_ctas), 128, 0, v->stream>>>(v->acc, v->fill, g, bt, 1, nullptr);
        k_depth<8><<<grid_1d(f.depth_ctas), 128, 0, v->stream>>>(v->acc, v->fill, g, dt, 1, ylo, yhi,
                                                                  p.fill_mode, v->r_depth);
        k_band<false><<<grid_1d(f.band_ctas), 128, 0, v->stream>>>(v->acc, v->fill, g, mt, 1, p.median_radius, above,
                                                             below, p.fill_mode, v->r_depth, v->r_mdepth,
                                                             v->r_mean, v->r_max, v->gt);
    }
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(v->stream, &graph);
    if (e) {
        if (graph) cudaGraphDestroy(graph);
        return e;
    }
    CK(ce);
    f.graph = graph;
    f.kernels = (int)(v->launches - l0) + 3;
    v->launches = l0;
    CK(cudaGraphInstantiate(&f.exec, f.graph, 0));
    f.w = w;
    f.h = h;
    f.fr = fr;
    f.cal = c;
    f.rp = p;
    f.ready = true;
    return SVR_OK;
}

extern "C" int svr_frame_step(svr_volume* v, const uint8_t* px, int64_t pitch, const svr_rigid* pose,
                              const svr_calib* c, int32_t fill_radius, const svr_render_params* p,
                              svr_box* dirty_out) {
    NvtxRange nvtx_("svr_frame_step");
    VOL_CHECK(v);
    const bool tri = v->tri != nullptr;
    if (!v->acc && !tri) return fail(SVR_E_INVALID, "frame step needs a volume");
    if (!px || !pose || !p) return fail(SVR_E_INVALID, "NULL argument");
    if (int e = check_calib(c, c ? c->crop_w : 0, c ? c->crop_h : 0)) return e;
    const int w = c->crop_w, h = c->crop_h;
    if (pitch < w) return fail(SVR_E_INVALID, "row pitch %lld < width %d", (long long)pitch, w);
    if (tri) fill_radius = 0;  // (a trilinear volume has no fill layer: splat + render)
    else if (fill_radius != 1) return fail(SVR_E_INVALID, "the frame graph runs the r = 1 mean fill");
    if (p->median_radius < 0 || p->median_radius > 2) return fail(SVR_E_INVALID, "median_radius must be 0..2");
    FrameGraph& f = v->fg;
    if (f.done) CK(cudaEventSynchronize(f.done));  // staging of the previous frame consumed
    const svr_box b = frame_box(v->d, *c, *pose);
    Box fb;
    svr_box bd{b.x0 - 1, b.y0 - 1, b.z0 - 1, b.x1 + 1, b.y1 + 1, b.z1 + 1};
    ColTiles ct[2];
    // (trilinear: the 2x2x2 splat reaches one voxel past the nearest-voxel box: render box + 1)
    const bool any = b.x0 <= b.x1 && clip_box(v, &bd, &fb) &&
                     render_regions(v, tri ? &bd : &b, fill_radius, p->median_radius, &ct[0], &ct[1]);
    if (!any) {  // frame entirely outside the slab: a plain insert counts its pixels
        if (dirty_out) *dirty_out = svr_box{1, 1, 1, 0, 0, 0};
        return svr_insert_frames(v, px, pitch, pitch * h, w, h, 1, pose, c, 0, nullptr, nullptr);
    }
    BoxTiles bt;
    bt.b = fb;
    bt.ntx = (fb.x1 - fb.x0 + 1 + 29) / 30;  // k_fill_warp<.., 8>: 30 columns x 4 warps of 8 rows
    bt.nty = (fb.y1 - fb.y0 + 1 + 31) / 32;
    bt.first = 0;
    const long long nf = tri ? 0 : (long long)bt.ntx * bt.nty * ((fb.z1 - fb.z0 + 1 + 1) / 2);
    std::vector<ColTiles> cv{ct[0]}, mv{ct[1]};
    const long long nd = tile_cols(cv, 16), nm = tile_cols(mv);
    FrameParams fpar;
    if (int e = make_params(*pose, prep_ctx(*c, v->d), c->scale_x_mm, c->scale_y_mm, &fpar)) return e;
    // the insert's tile shape is part of the capture: a frame that fits none of the captured
    // shape's tiles is still exact (its tiles take the exact pass) but re-captures once
    const bool shape_ok = tri || (f.shape < 0 ? fpar.lin_fit == 0
                                              : ((fpar.lin_fit >> (f.shape & 3)) & 1) != 0 &&
                                                    (!(f.shape & kShapeZ1) || (fpar.lin_fit & kFitZ1)));
    if (!fg_matches(f, w, h, fill_radius, *c, *p, nf, nd, nm) || !shape_ok) {
        v->lin_shapes_cur = fpar.lin_fit;
        if (int e = fg_capture(v, w, h, fill_radius, *c, *p, nf, nd, nm)) return e;
        f.shape = pick_shape(fpar.lin_fit, w, h, 1, v->num_sms);
        ++f.captures;
    }
    *f.h_fp = fpar;
    std::memcpy(f.h_tiles, &bt, sizeof bt);
    std::memcpy(f.h_tiles + sizeof(BoxTiles), &cv[0], sizeof(ColTiles));
    std::memcpy(f.h_tiles + sizeof(BoxTiles) + sizeof(ColTiles), &mv[0], sizeof(ColTiles));
    // frame source: device / pinned packed frames are copied straight from the caller
    // (any row pitch: the node is a 2-D copy); pageable host frames are staged through pinned
    // memory first, so the caller may reuse them on return
    bool pinned = false;
    const void* src = px;
    size_t spitch = (size_t)pitch;
    if (!(is_device_ptr(px, &pinned) || pinned)) {
        for (int r = 0; r < h; ++r) std::memcpy(f.h_frame + (size_t)r * w, px + (size_t)r * pitch, (size_t)w);
        src = f.h_frame;
        spitch = (size_t)w;
    }
    // the frame copy is enqueued ahead of the graph (any pitch, any source memory): a graph
    // memcpy node could not switch between host and device sources or pitches per call
    CK(cudaMemcpy2DAsync(f.d_frame, (size_t)w, src, spitch, (size_t)w, (size_t)h, cudaMemcpyDefault,
                         v->stream));
    CK(cudaGraphLaunch(f.exec, v->stream));
    CK(cudaEventRecord(f.done, v->stream));
    v->frames += 1;
    v->launches += f.kernels;
    if (dirty_out) *dirty_out = b;
    return SVR_OK;
}

extern "C" int svr_selftest_value_rounding(int device, int64_t* mismatches) {
    if (!mismatches) return fail(SVR_E_INVALID, "mismatches is NULL");
    CK(cudaSetDevice(device));
    unsigned long long* d = nullptr;
    CK(cudaMalloc(&d, sizeof(unsigned long long)));
    CK(cudaMemset(d, 0, sizeof(unsigned long long)));
    k_init_rcp<<<1, 256>>>();
    k_selftest_value<<<kRecipN - 1, 256>>>(d);
    k_selftest_div<<<1024, 256>>>(d);
    CKL();
    unsigned long long h = 0;
    CK(cudaMemcpy(&h, d, sizeof h, cudaMemcpyDeviceToHost));
    cudaFree(d);
    *mismatches = (int64_t)h;
    return SVR_OK;
}

extern "C" int svr_set_gather_targets(svr_volume* v, void* const* images, int32_t n, int32_t own_z0,
                                      int32_t own_z1) {
    VOL_CHECK(v);
    if (n < 0 || n > 64 || (n > 0 && !images)) return fail(SVR_E_INVALID, "invalid gather target list");
    if (n > 0 && (own_z0 < v->d.z_begin || own_z1 > v->d.z_end || own_z0 >= own_z1))
        return fail(SVR_E_INVALID, "owned rows [%d,%d) outside the slab [%d,%d)", own_z0, own_z1,
                    v->d.z_begin, v->d.z_end);
    CK(cudaStreamSynchronize(v->stream));
    cudaFree(v->d_gt);
    v->d_gt = nullptr;
    v->gt = GatherTargets{nullptr, 0, 0, 0, 0};
    if (n == 0) return SVR_OK;
    CK(cudaMalloc(&v->d_gt, sizeof(float*) * n));
    CK(cudaMemcpy(v->d_gt, images, sizeof(float*) * n, cudaMemcpyHostToDevice));
    v->gt = GatherTargets{v->d_gt, n, own_z0, own_z1, (long long)v->d.nz * v->d.nx};
    if (v->fg.ready) v->fg.ready = false;  // the frame graph captured the old targets
    return SVR_OK;
}
