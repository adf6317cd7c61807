// svr_io.cpp — host-only ingest and output formats of the C-ABI (include/spinevol_b200.h):
// binary PGM frames (image.hpp:34-72), the parallel frame loader that feeds svr_insert_frames
// from a ScanBundle with the crop_rect applied while decoding, and the raw
// u8 volume file.  Errors follow core.hpp:19-32: unreadable/unwritable file ->
// SVR_E_IO, malformed content -> SVR_E_INVALID; messages name the file.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "svr_host.hpp"

namespace {

// Minimal buffered reader with the istream semantics read_pgm relies on (peek/get, `>>` of a
// token and of a long).
struct File {
    FILE* f = nullptr;
    explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
    int peek() {
        int c = std::fgetc(f);
        if (c != EOF) std::ungetc(c, f);
        return c;
    }
    int get() { return std::fgetc(f); }
    void skip_ws() {
        int c;
        while ((c = peek()) != EOF && std::isspace(c)) get();
    }
    // `f >> std::string`: skip whitespace, read until whitespace/EOF
    std::string token() {
        skip_ws();
        std::string s;
        int c;
        while ((c = peek()) != EOF && !std::isspace(c)) s.push_back((char)get());
        return s;
    }
    // `f >> long`: skip whitespace, optional sign, digits; false on no digits / overflow
    bool read_long(long& v) {
        skip_ws();
        int c = peek();
        bool neg = false;
        if (c == '+' || c == '-') {
            neg = c == '-';
            get();
            c = peek();
        }
        if (c == EOF || !std::isdigit(c)) return false;
        unsigned long long acc = 0;
        while ((c = peek()) != EOF && std::isdigit(c)) {
            acc = acc * 10 + (unsigned)(c - '0');
            if (acc > (unsigned long long)__LONG_MAX__ + 1ull) return false;
            get();
        }
        if (!neg && acc > (unsigned long long)__LONG_MAX__) return false;
        v = neg ? -(long)acc : (long)acc;
        return true;
    }
};

// read_pgm's header (image.hpp:44-66): "P5", then width, height, maxval, each preceded by
// whitespace and '#'-to-end-of-line comments; maxval must be 255; one whitespace byte follows.
int pgm_header(File& f, const char* path, long* w, long* h) {
    if (f.token() != "P5") return svr_fail(SVR_E_INVALID, "not a binary PGM (P5): %s", path);
    auto next_int = [&](long* out) {
        int c;
        while ((c = f.peek()) != EOF) {
            if (c == '#') {
                while ((c = f.get()) != EOF && c != '\n') {
                }
            } else if (std::isspace(c)) {
                f.get();
            } else {
                break;
            }
        }
        long v = -1;
        if (!f.read_long(v) || v < 0) return false;
        *out = v;
        return true;
    };
    long maxval = 0;
    if (!next_int(w) || !next_int(h) || !next_int(&maxval))
        return svr_fail(SVR_E_INVALID, "malformed PGM header: %s", path);
    if (maxval != 255) return svr_fail(SVR_E_INVALID, "unsupported PGM maxval: %s", path);
    if (*w > (1l << 20) || *h > (1l << 20) || *w * *h > (1l << 34))
        return svr_fail(SVR_E_INVALID, "PGM dimensions too large: %s", path);
    f.get();  // the single whitespace byte after maxval
    return SVR_OK;
}

int pgm_read_into(const char* path, uint8_t* out, int64_t pitch, long want_w, long want_h,
                  const int32_t* crop) {
    File f(path, "rb");
    if (!f.f) return svr_fail(SVR_E_IO, "cannot open for reading: %s", path);
    long w = 0, h = 0;
    if (int e = pgm_header(f, path, &w, &h)) return e;
    if (w != want_w || h != want_h)
        return svr_fail(SVR_E_INVALID, "PGM %s is %ldx%ld, expected %ldx%ld", path, w, h, want_w, want_h);
    const long cx = crop ? crop[0] : 0, cy = crop ? crop[1] : 0;
    const long cw = crop ? crop[2] : w, ch = crop ? crop[3] : h;
    std::vector<uint8_t> row((size_t)w);
    for (long r = 0; r < h; ++r) {
        if (w && std::fread(row.data(), 1, (size_t)w, f.f) != (size_t)w)
            return svr_fail(SVR_E_INVALID, "truncated PGM data: %s", path);
        if (r >= cy && r < cy + ch) std::memcpy(out + (r - cy) * pitch, row.data() + cx, (size_t)cw);
    }
    return SVR_OK;
}

}  // namespace

extern "C" int svr_pgm_info(const char* path, int32_t* width, int32_t* height) {
    if (!path || !width || !height) return svr_fail(SVR_E_INVALID, "NULL argument");
    File f(path, "rb");
    if (!f.f) return svr_fail(SVR_E_IO, "cannot open for reading: %s", path);
    long w = 0, h = 0;
    if (int e = pgm_header(f, path, &w, &h)) return e;
    *width = (int32_t)w;
    *height = (int32_t)h;
    return SVR_OK;
}

extern "C" int svr_pgm_read(const char* path, uint8_t* out, int64_t row_pitch, int32_t width,
                            int32_t height) {
    if (!path || (!out && width > 0 && height > 0)) return svr_fail(SVR_E_INVALID, "NULL argument");
    if (row_pitch < width) return svr_fail(SVR_E_INVALID, "row pitch %lld < width %d", (long long)row_pitch, width);
    return pgm_read_into(path, out, row_pitch, width, height, nullptr);
}

extern "C" int svr_pgm_write(const char* path, const uint8_t* px, int64_t row_pitch, int32_t width,
                             int32_t height) {
    if (!path || (!px && width > 0 && height > 0) || width < 0 || height < 0)
        return svr_fail(SVR_E_INVALID, "invalid PGM write arguments");
    if (row_pitch < width) return svr_fail(SVR_E_INVALID, "row pitch %lld < width %d", (long long)row_pitch, width);
    File f(path, "wb");
    if (!f.f) return svr_fail(SVR_E_IO, "cannot open for writing: %s", path);
    // write_pgm (image.hpp:34-42): "P5\n<w> <h>\n255\n" + rows
    if (std::fprintf(f.f, "P5\n%d %d\n255\n", width, height) < 0)
        return svr_fail(SVR_E_IO, "write failed: %s", path);
    for (int32_t r = 0; r < height; ++r)
        if (width && std::fwrite(px + (int64_t)r * row_pitch, 1, (size_t)width, f.f) != (size_t)width)
            return svr_fail(SVR_E_IO, "write failed: %s", path);
    if (std::fflush(f.f) != 0) return svr_fail(SVR_E_IO, "write failed: %s", path);
    return SVR_OK;
}

extern "C" int svr_load_frames(const char* const* paths, int32_t n, int32_t raw_w, int32_t raw_h,
                               const int32_t* crop, uint8_t* out, int64_t frame_stride,
                               int32_t nthreads, int32_t* failed_index) {
    if (failed_index) *failed_index = -1;
    if (n < 0 || !paths || (!out && n > 0)) return svr_fail(SVR_E_INVALID, "invalid frame list");
    if (raw_w <= 0 || raw_h <= 0) return svr_fail(SVR_E_INVALID, "raw frame dims must be positive");
    if (crop && (crop[2] <= 0 || crop[3] <= 0 || crop[0] < 0 || crop[1] < 0 ||
                 crop[0] + crop[2] > raw_w || crop[1] + crop[3] > raw_h))
        return svr_fail(SVR_E_INVALID, "crop_rect (%d,%d,%d,%d) outside the %dx%d frame",
                        crop[0], crop[1], crop[2], crop[3], raw_w, raw_h);
    const int64_t w = crop ? crop[2] : raw_w, h = crop ? crop[3] : raw_h;
    if (frame_stride < w * h) return svr_fail(SVR_E_INVALID, "frame stride %lld < %lld", (long long)frame_stride, (long long)(w * h));
    if (n == 0) return SVR_OK;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int T = std::max(1, std::min<int>(nthreads > 0 ? nthreads : hw, n));
    // first failing frame wins (lowest index), so the reported error does not depend on T
    std::atomic<int> next{0};
    std::vector<int> code((size_t)n, SVR_OK);
    std::vector<std::string> msg((size_t)n);
    auto work = [&]() {
        for (int k; (k = next.fetch_add(1)) < n;) {
            code[(size_t)k] = pgm_read_into(paths[k], out + (int64_t)k * frame_stride, w, raw_w, raw_h, crop);
            if (code[(size_t)k]) msg[(size_t)k] = svr_last_error();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (int k = 0; k < n; ++k)
        if (code[(size_t)k]) {
            if (failed_index) *failed_index = k;
            return svr_fail(code[(size_t)k], "frame %d: %s", k, msg[(size_t)k].c_str());
        }
    return SVR_OK;
}

extern "C" int svr_write_raw(const char* path, const uint8_t* data, int64_t nbytes) {
    if (!path || (!data && nbytes > 0) || nbytes < 0) return svr_fail(SVR_E_INVALID, "invalid raw write arguments");
    File f(path, "wb");
    if (!f.f) return svr_fail(SVR_E_IO, "cannot open for writing: %s", path);
    if (nbytes && std::fwrite(data, 1, (size_t)nbytes, f.f) != (size_t)nbytes)
        return svr_fail(SVR_E_IO, "write failed: %s", path);
    if (std::fflush(f.f) != 0) return svr_fail(SVR_E_IO, "write failed: %s", path);
    return SVR_OK;
}
