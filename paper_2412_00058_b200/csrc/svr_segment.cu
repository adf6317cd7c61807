// svr_segment.cu — the segmentation front-end of the insert path (SPEC.md segment module,
// Tables I-II of the paper): per-frame bone-contour depth on the GPU (Algorithm 2 step 2), the
// depth-band cut applied in place to device-resident frames (apply_cut), and the host-side
// Algorithm 1 cut depth and Algorithm 2 depth smoothing.  The cut frames then go through
// svr_insert_frames with skip_zero.  The reference implements none of this
// module; the pins (percentile rank, 3-row gradient baseline in integer levels, median_lower of
// core.hpp:93-99, cut row rounding) are the oracle's (oracle/svr_oracle.c) and DESIGN.md §3's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "svr_host.hpp"

#define SCK(x)                                                                             \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess)                                                             \
            return svr_fail(SVR_E_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_));      \
    } while (0)

namespace {

// One CTA per frame.  Brightness threshold from a shared 256-bin histogram (the pct_rank-th
// smallest pixel); each thread then scans columns bottom-up with a 3-row window sum S(r) held in
// registers, stopping at the first bright window (S >= 3 thr): a cortex hit iff >= shadow_rows
// rows lie below it and S(r) - S(r+3) >= grad (oracle/svr_oracle.c orc_bone_contour).  Hit rows
// are histogrammed in dynamic shared memory and the frame row is their median_lower.
__global__ void __launch_bounds__(256) k_bone_contour(const uint8_t* __restrict__ px, long long pitch,
                                                      long long fstride, int w, int h, long long pct_rank,
                                                      int grad, int shadow_rows, double min_valid_frac,
                                                      int* __restrict__ row_out, int* __restrict__ valid_out,
                                                      int* __restrict__ thr_out, int* __restrict__ col_rows) {
    __shared__ unsigned int hist[256];
    __shared__ int s_thr, s_nv;
    extern __shared__ unsigned int rowhist[];
    const int f = blockIdx.x, tid = threadIdx.x;
    const uint8_t* base = px + (long long)f * fstride;
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    for (int i = tid; i < h; i += blockDim.x) rowhist[i] = 0;
    if (tid == 0) s_nv = 0;
    __syncthreads();
    for (int r = 0; r < h; ++r)
        for (int c = tid; c < w; c += blockDim.x) atomicAdd(&hist[base[(long long)r * pitch + c]], 1u);
    __syncthreads();
    if (tid < 32) {  // first v whose cumulative count exceeds pct_rank
        unsigned long long cum = 0;
        int thr = 255;
        for (int v0 = 0; v0 < 256; v0 += 32) {
            unsigned int c = hist[v0 + tid];
            unsigned long long inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
                if (tid >= o) inc += t;
            }
            const unsigned int hit = __ballot_sync(0xffffffffu, cum + inc > (unsigned long long)pct_rank);
            if (hit) {
                thr = v0 + __ffs(hit) - 1;
                break;
            }
            cum += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (tid == 0) s_thr = thr;
    }
    __syncthreads();
    const int thr = s_thr;
    for (int c = tid; c < w; c += blockDim.x) {
        int hit = -1;
        if (h >= 3) {
            // window rows r..r+2 (a = I[r], b = I[r+1], d = I[r+2]) and the sum 3 rows lower
            int d = base[(long long)(h - 1) * pitch + c], b = base[(long long)(h - 2) * pitch + c];
            int Sprev[3] = {0, 0, 0};  // S(r+1), S(r+2), S(r+3) as the scan moves up
            for (int r = h - 3; r >= 0; --r) {
                const int a = base[(long long)r * pitch + c];
                const int S = a + b + d;
                if (S >= 3 * thr) {
                    if (h - (r + 3) >= shadow_rows && r + 5 <= h - 1 && S - Sprev[2] >= grad) hit = r;
                    break;
                }
                Sprev[2] = Sprev[1];
                Sprev[1] = Sprev[0];
                Sprev[0] = S;
                d = b;
                b = a;
            }
        }
        if (col_rows) col_rows[(long long)f * w + c] = hit;
        if (hit >= 0) {
            atomicAdd(&rowhist[hit], 1u);
            atomicAdd(&s_nv, 1);
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int nv = s_nv;
        int row = -1;
        if (nv > 0 && !((double)nv < min_valid_frac * (double)w)) {
            const unsigned int k = (unsigned int)(nv - 1) / 2;  // median_lower (core.hpp:93-99)
            unsigned int cum = 0;
            for (int r = 0; r < h; ++r) {
                cum += rowhist[r];
                if (cum > k) {
                    row = r;
                    break;
                }
            }
        }
        row_out[f] = row;
        if (valid_out) valid_out[f] = nv;
        if (thr_out) thr_out[f] = thr;
    }
}

// apply_cut in place: rows outside [r0[f], r1[f]] of frame f set to 0 (empty range: all rows).
__global__ void k_apply_cut(uint8_t* __restrict__ px, long long pitch, long long fstride, int w, int h,
                            const int2* __restrict__ rows) {
    const int f = blockIdx.y;
    const int2 rr = rows[f];
    uint8_t* base = px + (long long)f * fstride;
    for (int r = blockIdx.x; r < h; r += gridDim.x) {
        if (r >= rr.x && r <= rr.y) continue;
        uint8_t* row = base + (long long)r * pitch;
        if (((uintptr_t)row & 15) == 0 && (w & 15) == 0) {
            for (int c = threadIdx.x; c < w / 16; c += blockDim.x)
                reinterpret_cast<uint4*>(row)[c] = make_uint4(0u, 0u, 0u, 0u);
        } else {
            for (int c = threadIdx.x; c < w; c += blockDim.x) row[c] = 0;
        }
    }
}

int device_frames(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return svr_fail(SVR_E_INVALID, "frames must be in device memory");
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
        return svr_fail(SVR_E_INVALID, "frames must be in device memory");
    return SVR_OK;
}

double median_lower(std::vector<double> v) {
    const size_t k = (v.size() - 1) / 2;
    std::nth_element(v.begin(), v.begin() + (std::ptrdiff_t)k, v.end());
    return v[k];
}

}  // namespace

extern "C" int svr_cut_depth_alg1(double p_c1, double p_cn, double K, double D, double L,
                                  double axial_extent_mm, double* out) {
    if (!out) return svr_fail(SVR_E_INVALID, "out is NULL");
    if (!(K >= 0.0) || !(D > 0.0) || !(L > 0.0)) return svr_fail(SVR_E_INVALID, "Alg1 needs K >= 0, D > 0, L > 0");
    double c = K * std::fabs(p_c1 - p_cn - L / 2.0) + D;  // Table I Step 4
    *out = std::min(std::max(c, 0.0), axial_extent_mm);
    return SVR_OK;
}

extern "C" int svr_cut_rows(double cut_mm, double band_mm, double scale_y_mm, int32_t h, int32_t* r0,
                            int32_t* r1) {
    if (!r0 || !r1) return svr_fail(SVR_E_INVALID, "NULL argument");
    if (!(scale_y_mm > 0.0) || !(band_mm > 0.0)) return svr_fail(SVR_E_INVALID, "scale and band must be positive");
    double a = std::ceil(cut_mm / scale_y_mm - 1e-9), b = std::floor((cut_mm + band_mm) / scale_y_mm + 1e-9);
    a = std::max(a, 0.0);
    b = std::min(b, (double)h - 1.0);
    *r0 = (int32_t)a;
    *r1 = (int32_t)b;
    return SVR_OK;
}

extern "C" int svr_smooth_depths(const double* depths, const uint8_t* valid, int32_t n, int32_t window,
                                 double* out) {
    if (n < 0 || (n > 0 && (!depths || !valid || !out))) return svr_fail(SVR_E_INVALID, "invalid series");
    if (window < 3 || window % 2 == 0) return svr_fail(SVR_E_INVALID, "median window must be odd and >= 3");
    int32_t first = -1, last = -1;
    for (int32_t i = 0; i < n; ++i)
        if (valid[i]) {
            if (first < 0) first = i;
            last = i;
        }
    if (first < 0) return svr_fail(SVR_E_ALGO, "no contour in any frame (all-gap depth series)");
    std::vector<double> g((size_t)n);
    int32_t prev = -1;
    for (int32_t i = 0; i < n; ++i) {
        if (valid[i]) {
            g[(size_t)i] = depths[i];
            prev = i;
        } else if (i < first) {
            g[(size_t)i] = depths[first];
        } else if (i > last) {
            g[(size_t)i] = depths[last];
        } else {
            int32_t nx = i + 1;
            while (!valid[nx]) ++nx;
            const double t = (double)(i - prev) / (double)(nx - prev);
            g[(size_t)i] = depths[prev] + (depths[nx] - depths[prev]) * t;
        }
    }
    const int32_t hw = window / 2;
    for (int32_t i = 0; i < n; ++i) {
        const int32_t a = std::max(0, i - hw), b = std::min(n - 1, i + hw);
        out[i] = median_lower(std::vector<double>(g.begin() + a, g.begin() + b + 1));
    }
    return SVR_OK;
}

extern "C" int svr_bone_contour(const uint8_t* px, int64_t row_pitch, int64_t frame_stride, int32_t w,
                                int32_t h, int32_t n, double pct, int32_t grad_levels,
                                int32_t shadow_rows, double min_valid_frac, int32_t* row_out,
                                int32_t* valid_cols_out,
                                int32_t* threshold_out, int32_t* col_rows_out, int device,
                                void* cuda_stream) {
    if (n < 0 || w <= 0 || h <= 0 || h > 8192 || row_pitch < w || (n > 1 && frame_stride < row_pitch * (h - 1) + w))
        return svr_fail(SVR_E_INVALID, "invalid frame geometry");
    if (!(pct >= 0.0 && pct <= 1.0)) return svr_fail(SVR_E_INVALID, "percentile must be in [0,1]");
    if (!row_out) return svr_fail(SVR_E_INVALID, "row_out is NULL");
    if (shadow_rows < 3) return svr_fail(SVR_E_INVALID, "shadow_rows must be >= 3");
    if (n == 0) return SVR_OK;
    if (int e = device_frames(px)) return e;
    SCK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const long long N = (long long)w * h;
    const long long rank = (long long)std::floor(pct * (double)(N - 1));
    int* d = nullptr;
    int* dc = nullptr;
    SCK(cudaMallocAsync(&d, sizeof(int) * 3 * (size_t)n, s));
    if (col_rows_out) SCK(cudaMallocAsync(&dc, sizeof(int) * (size_t)n * w, s));
    k_bone_contour<<<n, 256, sizeof(unsigned int) * (size_t)h, s>>>(px, row_pitch, frame_stride, w, h, rank,
                                                                  grad_levels, shadow_rows, min_valid_frac,
                                                                  d, d + n,
                                                                  d + 2 * n, dc);
    SCK(cudaGetLastError());
    std::vector<int> hbuf(3 * (size_t)n);
    SCK(cudaMemcpyAsync(hbuf.data(), d, sizeof(int) * 3 * (size_t)n, cudaMemcpyDeviceToHost, s));
    if (col_rows_out) SCK(cudaMemcpyAsync(col_rows_out, dc, sizeof(int) * (size_t)n * w, cudaMemcpyDefault, s));
    SCK(cudaFreeAsync(d, s));
    if (dc) SCK(cudaFreeAsync(dc, s));
    SCK(cudaStreamSynchronize(s));
    for (int32_t f = 0; f < n; ++f) {
        row_out[f] = hbuf[(size_t)f];
        if (valid_cols_out) valid_cols_out[f] = hbuf[(size_t)n + f];
        if (threshold_out) threshold_out[f] = hbuf[2 * (size_t)n + f];
    }
    return SVR_OK;
}

extern "C" int svr_apply_cut(uint8_t* px, int64_t row_pitch, int64_t frame_stride, int32_t w, int32_t h,
                             int32_t n, const int32_t* row0, const int32_t* row1, int device,
                             void* cuda_stream) {
    if (n < 0 || w <= 0 || h <= 0 || row_pitch < w || (n > 1 && frame_stride < row_pitch * (h - 1) + w))
        return svr_fail(SVR_E_INVALID, "invalid frame geometry");
    if (n == 0) return SVR_OK;
    if (!row0 || !row1) return svr_fail(SVR_E_INVALID, "row ranges are NULL");
    if (int e = device_frames(px)) return e;
    SCK(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)cuda_stream;
    std::vector<int2> rr((size_t)n);
    for (int32_t f = 0; f < n; ++f) rr[(size_t)f] = make_int2(row0[f], row1[f]);
    int2* d = nullptr;
    SCK(cudaMallocAsync(&d, sizeof(int2) * (size_t)n, s));
    SCK(cudaMemcpyAsync(d, rr.data(), sizeof(int2) * (size_t)n, cudaMemcpyHostToDevice, s));
    for (int32_t f0 = 0; f0 < n; f0 += 65535) {
        const int m = std::min(65535, n - f0);
        k_apply_cut<<<dim3(std::min(h, 64), m), 128, 0, s>>>(px + (long long)f0 * frame_stride, row_pitch,
                                                              frame_stride, w, h, d + f0);
        SCK(cudaGetLastError());
    }
    SCK(cudaFreeAsync(d, s));
    SCK(cudaStreamSynchronize(s));  // rr is released on return
    return SVR_OK;
}
