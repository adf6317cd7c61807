// svr_shard.cpp — z-slab sharded volume over one or more devices, built on the
// public C-ABI so a C / C++ caller runs the multi-GPU path without Python or MPI: one host thread
// drives every device.
//
//   * slabs: svr_plan_slabs -- contiguous near-equal owned z ranges, each stored with `ghost`
//     (= fill radius + render median radius) extra planes per side, so every owned voxel's fill
//     and every owned column's 5x5 median see exactly the unsharded neighbourhood;
//   * routing: a frame goes to every slab whose stored planes its conservative box
//     (svr_frame_bounds) meets; each slab inserts independently (integer sums: no exchange);
//   * gather: the coronal image [2][nz][nx] (mean plane, max plane) lives on devices[0]; every
//     slab's render stores its owned rows straight into it (svr_set_gather_targets: P2P stores
//     over NVLink between devices, plain stores on the same device), so no collective follows.
// Results are bit-identical to one unsharded volume (tests/test_gpu_shard.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../include/spinevol_b200.h"
#include "svr_host.hpp"

struct svr_sharded {
    svr_grid_desc d{};
    int n = 0;
    std::vector<int> dev;
    std::vector<svr_volume*> vol;
    std::vector<int32_t> ob, oe, ab, ae;
    std::vector<svr_box> dirty;  // per slab: union of routed frames' boxes since the last render
    float* img = nullptr;        // [2][nz][nx] on dev[0]
    svr_render_params last{};
};

static bool box_empty(const svr_box& b) { return b.x0 > b.x1; }

static void box_union(svr_box& a, const svr_box& b) {
    if (box_empty(b)) return;
    if (box_empty(a)) {
        a = b;
        return;
    }
    a.x0 = std::min(a.x0, b.x0);
    a.y0 = std::min(a.y0, b.y0);
    a.z0 = std::min(a.z0, b.z0);
    a.x1 = std::max(a.x1, b.x1);
    a.y1 = std::max(a.y1, b.y1);
    a.z1 = std::max(a.z1, b.z1);
}

#define CKR(x)                                                                                   \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess)                                                                   \
            return svr_fail(SVR_E_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_));            \
    } while (0)

extern "C" int svr_sharded_destroy(svr_sharded* s) {
    if (!s) return SVR_OK;
    for (svr_volume* v : s->vol)
        if (v) svr_destroy(v);
    if (s->img) {
        cudaSetDevice(s->dev[0]);
        cudaFree(s->img);
    }
    delete s;
    return SVR_OK;
}

extern "C" int svr_sharded_create(const svr_grid_desc* desc, const int32_t* devices, int32_t ndev,
                                  int32_t ghost, svr_sharded** out) {
    if (!desc || !devices || !out) return svr_fail(SVR_E_INVALID, "NULL argument");
    if (ndev < 1 || ndev > 64) return svr_fail(SVR_E_INVALID, "ndev must be 1..64");
    if (ghost < 0) return svr_fail(SVR_E_INVALID, "ghost must be >= 0");
    *out = nullptr;
    svr_sharded* s = new svr_sharded();
    s->d = *desc;
    s->d.z_begin = 0;
    s->d.z_end = desc->nz;
    s->n = ndev;
    s->dev.assign(devices, devices + ndev);
    s->ob.resize(ndev);
    s->oe.resize(ndev);
    s->ab.resize(ndev);
    s->ae.resize(ndev);
    s->dirty.assign(ndev, svr_box{1, 1, 1, 0, 0, 0});
    s->vol.assign(ndev, nullptr);
    if (int e = svr_plan_slabs(desc->nz, ndev, ghost, s->ob.data(), s->oe.data(), s->ab.data(),
                               s->ae.data())) {
        svr_sharded_destroy(s);
        return e;
    }
    for (int r = 0; r < ndev; ++r) {
        svr_grid_desc dr = s->d;
        dr.z_begin = s->ab[r];
        dr.z_end = s->ae[r];
        if (int e = svr_create(&dr, devices[r], &s->vol[r])) {
            svr_sharded_destroy(s);
            return e;
        }
    }
    {
        const size_t bytes = 2ull * (size_t)desc->nz * (size_t)desc->nx * sizeof(float);
        cudaError_t e = cudaSetDevice(devices[0]);
        if (e == cudaSuccess) e = cudaMalloc(&s->img, bytes);
        if (e == cudaSuccess) e = cudaMemset(s->img, 0, bytes);
        if (e != cudaSuccess) {
            svr_sharded_destroy(s);
            return svr_fail(SVR_E_CUDA, "coronal image on device %d: %s", devices[0], cudaGetErrorString(e));
        }
        for (int r = 0; r < ndev; ++r) {
            if (devices[r] != devices[0]) {  // the slab's render stores into devices[0] over NVLink
                int can = 0;
                cudaDeviceCanAccessPeer(&can, devices[r], devices[0]);
                if (!can) {
                    svr_sharded_destroy(s);
                    return svr_fail(SVR_E_CUDA, "device %d cannot access device %d (no P2P)", devices[r], devices[0]);
                }
                cudaSetDevice(devices[r]);
                cudaError_t pe = cudaDeviceEnablePeerAccess(devices[0], 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
                    svr_sharded_destroy(s);
                    return svr_fail(SVR_E_CUDA, "peer access %d -> %d: %s", devices[r], devices[0],
                                    cudaGetErrorString(pe));
                }
                cudaGetLastError();
            }
            void* tgt = s->img;
            if (int e2 = svr_set_gather_targets(s->vol[r], &tgt, 1, s->ob[r], s->oe[r])) {
                svr_sharded_destroy(s);
                return e2;
            }
        }
    }
    *out = s;
    return SVR_OK;
}

extern "C" int svr_sharded_slab(const svr_sharded* s, int32_t r, svr_volume** vol, int32_t* own_z0,
                                int32_t* own_z1, int32_t* alloc_z0, int32_t* alloc_z1) {
    if (!s) return svr_fail(SVR_E_INVALID, "NULL sharded volume");
    if (r < 0 || r >= s->n) return svr_fail(SVR_E_INVALID, "slab %d of %d", r, s->n);
    if (vol) *vol = s->vol[r];
    if (own_z0) *own_z0 = s->ob[r];
    if (own_z1) *own_z1 = s->oe[r];
    if (alloc_z0) *alloc_z0 = s->ab[r];
    if (alloc_z1) *alloc_z1 = s->ae[r];
    return SVR_OK;
}

// Route the batch: each slab inserts the frames whose conservative box meets its stored planes,
// as maximal runs of consecutive frames (one svr_insert_frames per run), asynchronously on the
// slab's own stream and device.
extern "C" int svr_sharded_insert_frames(svr_sharded* s, const uint8_t* px, int64_t pitch,
                                         int64_t fstride, int32_t w, int32_t h, int32_t n,
                                         const svr_rigid* poses, const svr_calib* calib,
                                         int32_t skip_zero, int32_t* routed_out) {
    if (!s) return svr_fail(SVR_E_INVALID, "NULL sharded volume");
    if (n < 0) return svr_fail(SVR_E_INVALID, "negative frame count");
    if (n == 0) return SVR_OK;
    if (!px || !poses || !calib) return svr_fail(SVR_E_INVALID, "NULL frames, poses or calib");
    std::vector<svr_box> fb((size_t)n);
    for (int k = 0; k < n; ++k)
        if (int e = svr_frame_bounds(&s->d, calib, &poses[k], &fb[(size_t)k])) return e;
    for (int r = 0; r < s->n; ++r) {
        int routed = 0;
        int k = 0;
        while (k < n) {
            auto meets = [&](int q) {
                const svr_box& b = fb[(size_t)q];
                return !box_empty(b) && b.z1 >= s->ab[r] && b.z0 < s->ae[r];
            };
            if (!meets(k)) {
                ++k;
                continue;
            }
            int k1 = k + 1;
            while (k1 < n && meets(k1)) ++k1;
            if (int e = svr_insert_frames(s->vol[r], px + (int64_t)k * fstride, pitch, fstride, w, h,
                                          k1 - k, poses + k, calib, skip_zero, nullptr, nullptr))
                return e;
            for (int q = k; q < k1; ++q) {
                svr_box b = fb[(size_t)q];
                b.z0 = std::max(b.z0, s->ab[r]);
                b.z1 = std::min(b.z1, s->ae[r] - 1);
                if (b.z0 <= b.z1) box_union(s->dirty[(size_t)r], b);
            }
            routed += k1 - k;
            k = k1;
        }
        if (routed_out) routed_out[r] = routed;
    }
    return SVR_OK;
}

// Hole fill of the dirty region (+ fill_radius) and depth-band render of its columns on every
// slab; each slab's render stores its owned rows into the gathered image on devices[0].
extern "C" int svr_sharded_fill_render(svr_sharded* s, int32_t fill_radius, int32_t fill_mode,
                                       const svr_render_params* params) {
    if (!s) return svr_fail(SVR_E_INVALID, "NULL sharded volume");
    if (!params) return svr_fail(SVR_E_INVALID, "NULL render params");
    for (int r = 0; r < s->n; ++r) {
        const svr_box u = s->dirty[(size_t)r];
        if (box_empty(u)) continue;
        svr_box f{u.x0 - fill_radius, u.y0 - fill_radius, u.z0 - fill_radius, u.x1 + fill_radius,
                  u.y1 + fill_radius, u.z1 + fill_radius};
        f.x0 = std::max(f.x0, 0);
        f.y0 = std::max(f.y0, 0);
        f.z0 = std::max(f.z0, s->ab[r]);
        f.x1 = std::min(f.x1, s->d.nx - 1);
        f.y1 = std::min(f.y1, s->d.ny - 1);
        f.z1 = std::min(f.z1, s->ae[r] - 1);
        const bool pnn = s->d.accum == SVR_ACC_PNN;  // (trilinear volumes have no hole fill)
        if (pnn)
            if (int e = svr_fill_holes(s->vol[r], &f, fill_mode, fill_radius, nullptr)) return e;
        if (int e = svr_render_coronal(s->vol[r], &u, pnn ? fill_radius : 0, params)) return e;
        s->dirty[(size_t)r] = svr_box{1, 1, 1, 0, 0, 0};
    }
    s->last = *params;
    return SVR_OK;
}

extern "C" int svr_sharded_sync(svr_sharded* s) {
    if (!s) return svr_fail(SVR_E_INVALID, "NULL sharded volume");
    for (svr_volume* v : s->vol)
        if (int e = svr_sync(v)) return e;
    return SVR_OK;
}

// The gathered coronal image (rows z of the whole grid, nx wide): mean / max from devices[0],
// depths from each slab's owned rows.  Any output may be NULL.
extern "C" int svr_sharded_read_coronal(svr_sharded* s, float* mean_out, float* max_out,
                                        int32_t* depth_out) {
    if (!s) return svr_fail(SVR_E_INVALID, "NULL sharded volume");
    if (int e = svr_sharded_sync(s)) return e;
    const size_t plane = (size_t)s->d.nz * (size_t)s->d.nx;
    CKR(cudaSetDevice(s->dev[0]));
    if (mean_out) CKR(cudaMemcpy(mean_out, s->img, plane * sizeof(float), cudaMemcpyDefault));
    if (max_out) CKR(cudaMemcpy(max_out, s->img + plane, plane * sizeof(float), cudaMemcpyDefault));
    if (depth_out)
        for (int r = 0; r < s->n; ++r)
            if (s->oe[r] > s->ob[r])
                if (int e = svr_read_coronal(s->vol[r], s->ob[r], s->oe[r] - 1, nullptr, nullptr,
                                             depth_out + (size_t)s->ob[r] * s->d.nx))
                    return e;
    return SVR_OK;
}
