// svr_fan.cuh — K1 for convex (fan) probes: the pixel-nearest-neighbour insert of polar B-scans
// (BASELINE cfg3) as a persistent tile kernel.  Included after svr_k1.cuh.
//
// A fan frame is `lines` scanlines x `samples` radial samples; along one scanline the voxel-space
// position is affine in the sample index (u = A_l + s D_l, 32.32 fixed point, the same A_l, D_l
// k_pnn_work's row_coeffs computes), so each scanline is walked exactly like a linear-probe row:
// three fixed-point fractions stepped per sample, the index moving where a fraction carries, a
// chunk whose fractions came within the certified tie window undone and deferred to k_pnn_work.
//
// Work unit: a tile of 32 scanlines x TCOLS = 16 * NCH * NW samples of one frame; thread (warp w,
// lane l) walks scanline l's samples [32 w, 32 w + 32) of the tile (NCH = 2 chunks).  A tile is
// accumulated one of two ways, chosen per tile by k_fan_desc from its voxel extent:
//   * table: near the apex the scanlines are dense (cfg3: 11 px per voxel at r = 20 mm): every
//     sample is a shared atomic into the (x, y, z & 1) table of svr_k1.cuh (row stride = the
//     tile's own odd width), flushed with one 64-bit red.global.add per non-empty slot;
//   * direct: far out the table would mostly be empty positions (1.5 px per voxel at r = 150 mm,
//     the tile's rotated box twice the touched area), so each scanline's runs of samples that
//     share a voxel are added straight to the volume, one red.global.add per run (~2.7 samples).
// The per-scanline constants (A_l, D_l) and the tile descriptors are computed by k_fan_desc
// before the insert, so the insert's CTAs never wait on fp64 setup: the next tile's rows,
// scanline constants and descriptor are requested before the current tile's flush.
#pragma once


namespace svr {

constexpr int kFanLines = 32;  // scanlines per tile (one per lane)

struct FanRow {
    long long A[3];  // 32.32 fixed u at sample 0, +1/2 (row_coeffs<true>)
    long long D[3];  // 32.32 fixed du/dsample
};

struct __align__(16) FanDesc {
    long long base;   // table flush base: byte offset of voxel (X0, Y0, zint + kmin) in the slab
    long long dbase;  // direct base: byte offset of voxel (X0, Y0, Z0) in the slab
    int X0, Y0, Z0;   // the tile's fixed-point index minima
    int XY;           // X | Y << 16
    int flags;        // bit 0 table mode, bit 1 tin (inside grid / slab), bit 2 walkable (|D| < 1 voxel)
    int zpar;         // (zint + kmin) & 1
    float tt0;        // z_c - h at the table origin, minus kmin
    int stride;       // table row stride in words (odd, >= X)
    uint32_t te2;     // tie window + 1 (FrameParams::tie_eps + 1)
    float p1, p2;     // frame plane slopes
    int pad;
};

struct FanArgs {
    const uint8_t* px;
    long long pitch, fstride;
    int w, h;
    int ntx, nty;        // tiles per frame along samples / scanlines
    long long ntiles;
    const FrameParams* fps;
    DevCalib cal;
    const double2* fan;  // scanline directions
    GridDev g;
    ull* acc;
    int* boxes;
    ull* stats;
    ull* work;
    unsigned int* work_n;
    unsigned int work_cap;
    FanDesc* desc;
    FanRow* rows;        // [nframes][h]
    int dense;           // table mode when dense * X * Y <= 4 * tile pixels
};

// One warp per tile, lane = scanline: the scanline constants, the tile's index extent (u is
// affine along each scanline, so each scanline's extremes sit at its two end samples) and the
// accumulation mode.
template <int TCOLS>
__global__ void __launch_bounds__(128) k_fan_desc(const FanArgs fa) {
    const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= fa.ntiles) return;  // (warp-uniform)
    const int tpf = fa.ntx * fa.nty;
    const int f = (int)(t / tpf), rem = (int)(t - (long long)f * tpf);
    const int ty = rem / fa.ntx, tx = rem - ty * fa.ntx;
    const FrameParams& fp = fa.fps[f];
    const GridDev& g = fa.g;
    const int line = ty * kFanLines + lane;
    const bool act = line < fa.h;
    long long A[3], D[3];
    row_coeffs<true>(fp, fa.cal, fa.fan, act ? line : fa.h - 1, 0, A, D);
    if (tx == 0 && act) {
        FanRow r;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.A[k] = A[k];
            r.D[k] = D[k];
        }
        fa.rows[(long long)f * fa.h + line] = r;
    }
    const int c0t = tx * TCOLS;
    const int n1 = min(TCOLS, fa.w - c0t) - 1;
    int lo[3], hi[3];
    bool walk = true;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long u0 = A[k] + (long long)c0t * D[k], u1 = u0 + (long long)n1 * D[k];
        int l = (int)(min(u0, u1) >> 32), hh = (int)(max(u0, u1) >> 32);
        if (!act) {
            l = 0x7fffffff;
            hh = -0x7fffffff - 1;
        }
        lo[k] = __reduce_min_sync(0xffffffffu, l);
        hi[k] = __reduce_max_sync(0xffffffffu, hh);
        walk = walk && (unsigned long long)(D[k] < 0 ? -D[k] : D[k]) < (1ull << 32);
    }
    walk = __all_sync(0xffffffffu, walk || !act);
    if (lane != 0) return;
    const int nlines = min(kFanLines, fa.h - ty * kFanLines);
    const int X = hi[0] - lo[0] + 1, Y = hi[1] - lo[1] + 1;
    const int stride = X | 1;
    const long long npx = (long long)(n1 + 1) * nlines;
    const bool table = walk && fp.plane_ok && X <= 2047 && (long long)stride * Y <= 2048 &&
                       (long long)fa.dense * X * Y <= 4 * npx;
    const bool tin = lo[0] >= 0 && hi[0] <= g.nx - 1 && lo[1] >= 0 && hi[1] <= g.ny - 1 &&
                     lo[2] >= g.zb && hi[2] <= g.zb + g.nzl - 1;
    FanDesc d;
    d.X0 = lo[0];
    d.Y0 = lo[1];
    d.Z0 = lo[2];
    d.XY = (X & 0xffff) | (min(Y, 0x7fff) << 16);
    d.flags = (table ? 1 : 0) | (tin ? 2 : 0) | (walk ? 4 : 0);
    d.stride = stride;
    const long long sxy = (long long)g.nx * g.ny;
    d.dbase = 8ll * ((long long)(lo[2] - g.zb) * sxy + (long long)lo[1] * g.nx + lo[0]);
    // table flush plane (as k_tile_desc)
    const double zt = fp.pz[0] + fp.pz[1] * (double)lo[0] + fp.pz[2] * (double)lo[1] - fp.pz[3];
    const int zint = (int)floor(zt);
    const float zf0 = (float)(zt - (double)zint);
    const float p1 = (float)fp.pz[1], p2 = (float)fp.pz[2];
    const int kmin = table ? -1 + (int)floorf(zf0 + fminf(0.f, p1 * (float)(X - 1)) + fminf(0.f, p2 * (float)(Y - 1))) : 0;
    d.tt0 = zf0 - (float)kmin;
    d.zpar = (zint + kmin) & 1;
    d.base = 8ll * ((long long)(zint + kmin - g.zb) * sxy + (long long)lo[1] * g.nx + lo[0]);
    d.te2 = fp.tie_eps + 1;
    d.p1 = p1;
    d.p2 = p2;
    d.pad = 0;
    fa.desc[t] = d;
}

__device__ __forceinline__ void push_fan(const FanArgs& fa, int f, int line, int cc) {
    // the host sizes the list for every chunk of the launch, so it cannot overflow
    const unsigned int slot = atomicAdd(fa.work_n, 1u);
    fa.work[slot] = work_entry(f, line, cc, 0xffffu);
}

// One exact step of the three fractions, branch-free: where any fraction carries, the finished
// run (voxel byte offset, count << 20 | sum) is appended to this lane's run buffer (a shared
// store predicated on the carry; `ptr` advances one row, `rstride` bytes, of the [entry][thread]
// buffer),
// the run restarts, and the offset follows the carries.
__device__ __forceinline__ void run_step(uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& off,
                                         uint32_t& run, uint32_t& ptr, uint32_t e0, uint32_t e1,
                                         uint32_t e2, uint32_t sx, uint32_t sy, uint32_t sz, uint32_t rstride) {
    asm volatile(
        "{\n\t.reg .pred p0, p1, p2, pc;\n\t.reg .u32 c0, c1, c2;\n\t"
        "add.cc.u32 %0, %0, %6;\n\taddc.u32 c0, 0, 0;\n\t"
        "add.cc.u32 %1, %1, %7;\n\taddc.u32 c1, 0, 0;\n\t"
        "add.cc.u32 %2, %2, %8;\n\taddc.u32 c2, 0, 0;\n\t"
        "setp.ne.u32 p0, c0, 0;\n\tsetp.ne.u32 p1, c1, 0;\n\tsetp.ne.u32 p2, c2, 0;\n\t"
        "or.pred pc, p0, p1;\n\tor.pred pc, pc, p2;\n\t"
        "@pc st.shared.v2.u32 [%5], {%3, %4};\n\t"
        "@pc add.u32 %5, %5, %12;\n\t"
        "@pc mov.u32 %4, 0;\n\t"
        "@p0 add.u32 %3, %3, %9;\n\t@p1 add.u32 %3, %3, %10;\n\t@p2 add.u32 %3, %3, %11;\n\t}"
        : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(off), "+r"(run), "+r"(ptr)
        : "r"(e0), "r"(e1), "r"(e2), "r"(sx), "r"(sy), "r"(sz), "r"(rstride)
        : "memory");
}

// one exact step without a run boundary: the offset follows the carries
__device__ __forceinline__ void off_step(uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& off, uint32_t e0,
                                         uint32_t e1, uint32_t e2, uint32_t sx, uint32_t sy, uint32_t sz) {
    asm("{\n\t.reg .pred p0, p1, p2;\n\t.reg .u32 c0, c1, c2;\n\t"
        "add.cc.u32 %0, %0, %4;\n\taddc.u32 c0, 0, 0;\n\t"
        "add.cc.u32 %1, %1, %5;\n\taddc.u32 c1, 0, 0;\n\t"
        "add.cc.u32 %2, %2, %6;\n\taddc.u32 c2, 0, 0;\n\t"
        "setp.ne.u32 p0, c0, 0;\n\tsetp.ne.u32 p1, c1, 0;\n\tsetp.ne.u32 p2, c2, 0;\n\t"
        "@p0 add.u32 %3, %3, %7;\n\t@p1 add.u32 %3, %3, %8;\n\t@p2 add.u32 %3, %3, %9;\n\t}"
        : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(off)
        : "r"(e0), "r"(e1), "r"(e2), "r"(sx), "r"(sy), "r"(sz));
}

// tile_step with the z toggle kept in its own register (the table address is a ^ zo): the shared
// atomic's address is then a fresh register, so the next sample's in-place x / y moves do not wait
// for the atomic to read it (a write-after-read stall: short_sb at every move after an ATOMS)
__device__ __forceinline__ void tile_step_zx(uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& a, uint32_t& zo,
                                             uint32_t e0, uint32_t e1, uint32_t e2, uint32_t sx, uint32_t sy) {
    asm("{\n\t.reg .pred p0, p1, p2;\n\t.reg .u32 c0, c1, c2;\n\t"
        "add.cc.u32 %0, %0, %5;\n\taddc.u32 c0, 0, 0;\n\t"
        "add.cc.u32 %1, %1, %6;\n\taddc.u32 c1, 0, 0;\n\t"
        "add.cc.u32 %2, %2, %7;\n\taddc.u32 c2, 0, 0;\n\t"
        "setp.ne.u32 p0, c0, 0;\n\tsetp.ne.u32 p1, c1, 0;\n\tsetp.ne.u32 p2, c2, 0;\n\t"
        "@p0 add.u32 %3, %3, %8;\n\t@p1 add.u32 %3, %3, %9;\n\t@p2 xor.b32 %4, %4, 16384;\n\t}"
        : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(a), "+r"(zo)
        : "r"(e0), "r"(e1), "r"(e2), "r"(sx), "r"(sy));
}

#ifndef SVR_FAN_ZX
#define SVR_FAN_ZX 1  // k_fan_tiles table walk: z toggle in its own register (tile_step_zx)
#endif
#ifndef SVR_FAN_DRAINPF
#define SVR_FAN_DRAINPF 1  // k_fan_tiles: the run buffer's next entry read while the current one is added
#endif

// Chunk classes of one thread's 32-sample segment (k_pnn_tiles' rule): a chunk whose index range
// lies inside the grid / slab is walked, one wholly outside is counted out of bounds, one
// straddling a face goes to the exact pass.  Returns the mask of chunks to walk.
__device__ __forceinline__ uint32_t fan_classes(const FanArgs& fa, const long long (&A)[3], const long long (&D)[3],
                                                bool walkable, int f, int line, int cth, uint32_t& noob,
                                                uint32_t& ndef) {
    const GridDev& g = fa.g;
    const int clo[3] = {0, 0, g.zb}, chi[3] = {g.nx - 1, g.ny - 1, g.zb + g.nzl - 1};
    uint32_t wmask = 0u;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        bool inb = walkable, out = false;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const long long u = A[k] + (long long)(cth + 16 * c) * D[k];
            const int i0 = (int)(u >> 32), i15 = (int)((u + 15ll * D[k]) >> 32);
            // (the exact index is within 1 of the fixed-point one: 2 outside misses)
            inb = inb && min(i0, i15) >= clo[k] && max(i0, i15) <= chi[k];
            out = out || max(i0, i15) + 1 < clo[k] || min(i0, i15) - 1 > chi[k];
        }
        if (inb) {
            wmask |= 1u << c;
        } else if (out && walkable) {
            ++noob;
        } else {
            push_fan(fa, f, line, (cth >> 4) + c);
            ++ndef;
        }
    }
    return wmask;
}

__device__ __forceinline__ void fan_box(BoxAcc& bb, const long long (&A)[3], const long long (&D)[3], int c0,
                                        int n) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long u = A[k] + (long long)c0 * D[k];
        const int i0 = (int)(u >> 32), i1 = (int)((u + (long long)(n - 1) * D[k]) >> 32);
        if (k == 0) { bb.x0 = min(bb.x0, min(i0, i1)); bb.x1 = max(bb.x1, max(i0, i1)); }
        if (k == 1) { bb.y0 = min(bb.y0, min(i0, i1)); bb.y1 = max(bb.y1, max(i0, i1)); }
        if (k == 2) { bb.z0 = min(bb.z0, min(i0, i1)); bb.z1 = max(bb.z1, max(i0, i1)); }
    }
}

// Persistent CTAs of 4 warps over the launch's tiles; thread (warp w, lane l) walks scanline l's
// samples [32 w, 32 w + 32) of a tile.  Table tiles: every sample a shared atomic into the table,
// then the CTA flushes it.  Direct tiles: each 16-sample chunk's walk is branch-free -- where a
// fraction carries, the finished run (voxel offset, count << 20 | sum) is appended with a
// predicated shared store to the thread's run buffer, which borrows the (all-zero) table memory;
// once the chunk's tie screen has passed, the runs are added with one red.global.add each and
// their buffer words zeroed again (a tie chunk's runs are just dropped: nothing to undo).  The
// tile after next's scanline constants and descriptor are staged with cp.async; the next tile's
// pixels are loaded before the current tile's flush.
#ifndef SVR_FAN_MINB
#define SVR_FAN_MINB 8  // k_fan_tiles: CTAs per SM the register budget is cut for (A/B: 8 beat 6, 7; 7 fit by shared memory)
#endif
#ifndef SVR_FAN_ORDER
#define SVR_FAN_ORDER 0  // k_fan_tiles tile order: 0 frame-major, 1 tile-major (frames fastest)
#endif
template <bool kBox>
__global__ void __launch_bounds__(128, SVR_FAN_MINB) k_fan_tiles(const FanArgs fa) {
    constexpr int NW = 4, NCH = 2, NT = 32 * NW, TCOLS = 16 * NCH * NW;
    static_assert(15 * NT * 8 <= 4 * kTabWords, "run buffer: 15 entries per thread in the table memory");
    __shared__ __align__(16) uint32_t s_tab[kTabWords];
    __shared__ __align__(16) FanRow s_rows[3][kFanLines];  // ring: tiles i, i + 1, i + 2
    __shared__ FanDesc s_desc[3];
    __shared__ unsigned int s_cnt[2];    // chunks counted out of bounds / deferred
    __shared__ unsigned long long s_px;  // pixels of this CTA's tiles
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 2) s_cnt[tid] = 0u;
    if (tid == 0) s_px = 0ull;
    for (int i = tid; i < kTabWords / 4; i += NT)
        reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0u, 0u, 0u, 0u);
    const uint32_t tab = (uint32_t)__cvta_generic_to_shared(s_tab);
    // (see svr_k1.cuh: parity plane bit 14; otherwise table tiles run direct)
    const bool tab_ok = tab + 4u * 2048u <= 16384u;
    const uint32_t rbuf = tab + 8u * (uint32_t)tid;  // run buffer: entry k at rbuf + k * 8 NT
    const GridDev& g = fa.g;
    const int tpf = fa.ntx * fa.nty;
    // tiles round-robin over the CTAs: the CTAs in flight together work on a window of ~grid
    // consecutive tiles (a few dozen frames), so neighbouring frames' adds to the same voxels
    // meet in L2 instead of each reading the voxel's sector from HBM
    const long long t0 = blockIdx.x, tstep = gridDim.x, t1 = fa.ntiles;
    // (frame, tile row, tile column) of tile t, advanced by tstep without divisions per tile: a
    // mixed-radix counter of digits a0 (fastest, radix R0), a1 (R1), a2.  Frame-major order: a0 =
    // tile column, a1 = tile row, a2 = frame.  Tile-major (SVR_FAN_ORDER 1): a0 = frame, a1 = tile
    // column, a2 = tile row -- the CTAs in flight work on one fan patch of consecutive frames
#if SVR_FAN_ORDER
    const int R0 = (int)(t1 / tpf), R1 = fa.ntx;
#else
    const int R0 = fa.ntx, R1 = fa.nty;
#endif
    const long long R01 = (long long)R0 * R1;
    const int s2 = (int)(tstep / R01), sr = (int)(tstep - (long long)s2 * R01);
    const int s1 = sr / R0, s0 = sr - s1 * R0;
    auto split = [&](long long t, int& fq, int& tyq, int& txq) {
#if SVR_FAN_ORDER
        int& a0 = fq; int& a1 = txq; int& a2 = tyq;
#else
        int& a0 = txq; int& a1 = tyq; int& a2 = fq;
#endif
        a2 = (int)(t / R01);
        const int r = (int)(t - (long long)a2 * R01);
        a1 = r / R0;
        a0 = r - a1 * R0;
    };
    auto advance = [&](int& fq, int& tyq, int& txq) {
#if SVR_FAN_ORDER
        int& a0 = fq; int& a1 = txq; int& a2 = tyq;
#else
        int& a0 = txq; int& a1 = tyq; int& a2 = fq;
#endif
        a0 += s0;
        a1 += s1;
        a2 += s2;
        if (a0 >= R0) {
            a0 -= R0;
            ++a1;
        }
        if (a1 >= R1) {
            a1 -= R1;
            ++a2;
        }
    };
    int f, ty, tx;
    split(t0, f, ty, tx);
    unsigned int ntiles_cta = 0;
    int cur_f = -1;
    BoxAcc bb;
    const uint32_t sxy8 = (uint32_t)((long long)g.nx * g.ny * 8), nx8 = (uint32_t)g.nx * 8u;

    // this thread's 32 samples, one 16-sample chunk per wd[c]; the next tile's chunk c is requested
    // as soon as the current tile's chunk c has been walked (its registers are free), so a direct
    // tile -- no flush to hide the load behind -- finds its samples mostly arrived
    uint32_t wd[NCH][4];
    auto load_px = [&](int fq, int tyq, int txq) {
        const int line = min(tyq * kFanLines + lane, fa.h - 1);
        ld256(fa.px + (long long)fq * fa.fstride + (long long)line * fa.pitch + txq * TCOLS + 32 * warp, &wd[0][0]);
    };
    auto load_half = [&](int c, int fq, int tyq, int txq) {
        const int line = min(tyq * kFanLines + lane, fa.h - 1);
        const uint8_t* p = fa.px + (long long)fq * fa.fstride + (long long)line * fa.pitch + txq * TCOLS + 32 * warp + 16 * c;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(wd[c][0]), "=r"(wd[c][1]), "=r"(wd[c][2]), "=r"(wd[c][3]) : "l"(p));
    };
    // threads 0..95 stage a tile's 32 scanline constants (1.5 KB), 96..99 its descriptor
    auto stage = [&](int fq, int tyq, int txq, int b) {
        const long long t = (long long)fq * tpf + tyq * fa.ntx + txq;
        if (tid < 96) {
            const int line0 = tyq * kFanLines;
            if (tid * 16 < min(kFanLines, fa.h - line0) * (int)sizeof(FanRow)) {
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<uint4*>(&s_rows[b][0]) + tid);
                const uint4* src = reinterpret_cast<const uint4*>(fa.rows + (long long)fq * fa.h + line0) + tid;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
            }
        } else if (tid < 100) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<uint4*>(&s_desc[b]) + (tid - 96));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(reinterpret_cast<const uint4*>(fa.desc + t) + (tid - 96)) : "memory");
        }
    };
    // one commit group per tile (empty for threads >= 100): waiting for all but the newest group
    // leaves the tile two ahead in flight
    auto commit = [&]() { asm volatile("cp.async.commit_group;" ::: "memory"); };
    auto wait_stage = [&]() { asm volatile("cp.async.wait_group 1;" ::: "memory"); };
    if (t0 < t1) {
        load_px(f, ty, tx);
        stage(f, ty, tx, 0);
        commit();
        int f1 = f, ty1 = ty, tx1 = tx;
        advance(f1, ty1, tx1);
        if (t0 + tstep < t1) stage(f1, ty1, tx1, 1);
        commit();
        wait_stage();
    }
    int slot = 0;

    for (long long t = t0; t < t1; t += tstep) {
        if (kBox && f != cur_f) {  // CTA-uniform
            if (cur_f >= 0) {
                flush_box(bb, fa.boxes + 6 * cur_f);
                bb = BoxAcc();
            }
            cur_f = f;
        }
        __syncthreads();  // rows + descriptor staged; table clean
        const int b = slot;
        slot = slot == 2 ? 0 : slot + 1;
        ++ntiles_cta;
        // the tile after next: its constants are requested now; the next tile's pixels after the walk
        int fn = f, tyn = ty, txn = tx;
        advance(fn, tyn, txn);
        int f2 = fn, ty2 = tyn, tx2 = txn;
        advance(f2, ty2, tx2);
        if (t + 2 * tstep < t1) stage(f2, ty2, tx2, b == 0 ? 2 : b - 1);
        commit();
        const FanDesc& dsc = s_desc[b];
        const bool more = t + tstep < t1;  // (a next tile exists: its samples are requested below)
        const int nlines = min(kFanLines, fa.h - ty * kFanLines);
        const int line = ty * kFanLines + lane;
        const bool act = lane < nlines;
        const FanRow& fr = s_rows[b][act ? lane : 0];
        const bool table = (dsc.flags & 1) && tab_ok, tin = dsc.flags & 2, walkable = dsc.flags & 4;
        const uint32_t te2 = dsc.te2, tie2 = 2u * te2;
        const int cth = tx * TCOLS + 32 * warp;  // this thread's first sample
        long long A[3], D[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            A[k] = fr.A[k];
            D[k] = fr.D[k];
        }
        uint32_t noob = 0, ndef = 0;
        uint32_t wmask = act && walkable ? 3u : 0u;
        if (act && (!walkable || !tin)) {
            wmask = fan_classes(fa, A, D, walkable, f, line, cth, noob, ndef);
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                if (!((wmask >> c) & 1u)) wd[c][0] = wd[c][1] = wd[c][2] = wd[c][3] = 0u;  // (table walk: adds nothing)
        }
        if (wmask != 0u) {
            uint32_t e[3], neg[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                e[k] = (uint32_t)(D[k] < 0 ? -D[k] : D[k]);
                neg[k] = D[k] < 0 ? 0xffffffffu : 0u;
            }
            // walk state at the segment's first sample (index adjusted where lo + te2 wraps: see
            // walk_state in svr_k1.cuh)
            const long long u0 = A[0] + (long long)cth * D[0], u1 = A[1] + (long long)cth * D[1],
                            u2 = A[2] + (long long)cth * D[2];
            uint32_t v0 = ((uint32_t)u0 ^ neg[0]) + te2, v1 = ((uint32_t)u1 ^ neg[1]) + te2,
                     v2 = ((uint32_t)u2 ^ neg[2]) + te2;
            const int ix = (int)(u0 >> 32) + (v0 < te2 ? (neg[0] ? -1 : 1) : 0);
            const int iy = (int)(u1 >> 32) + (v1 < te2 ? (neg[1] ? -1 : 1) : 0);
            const int iz = (int)(u2 >> 32) + (v2 < te2 ? (neg[2] ? -1 : 1) : 0);
            if (table) {
                const int stride = dsc.stride;
                const uint32_t sx = neg[0] ? 0u - 4u : 4u;
                const uint32_t sy = neg[1] ? 0u - 4u * (uint32_t)stride : 4u * (uint32_t)stride;
                uint32_t a = tab + 4u * (uint32_t)((ix - dsc.X0) + stride * (iy - dsc.Y0)) + ((uint32_t)(iz & 1) << 14);
                uint32_t zo = 0u;
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    if (c > 0) tile_step(v0, v1, v2, a, e[0], e[1], e[2], sx, sy);
                    const uint32_t o20 = (wmask >> c) & 1u ? 0x00100000u : 0u;
                    uint32_t tmin = min(v0, min(v1, v2));
                    const uint32_t ua = a, q0 = v0, q1 = v1, q2 = v2;
                    red_shared(a, __byte_perm(wd[c][0], o20, 0x7640));
#pragma unroll
                    for (int j = 1; j < kChunk; ++j) {
#if SVR_FAN_ZX
                        tile_step_zx(v0, v1, v2, a, zo, e[0], e[1], e[2], sx, sy);
                        tmin = min(tmin, min(v0, min(v1, v2)));
                        red_shared(a ^ zo, __byte_perm(wd[c][j >> 2], o20, 0x7640 | (j & 3)));
#else
                        tile_step(v0, v1, v2, a, e[0], e[1], e[2], sx, sy);
                        tmin = min(tmin, min(v0, min(v1, v2)));
                        red_shared(a, __byte_perm(wd[c][j >> 2], o20, 0x7640 | (j & 3)));
#endif
                    }
                    a ^= zo;
                    zo = 0u;
                    if (o20 != 0u && tmin < tie2) {  // rare: undo the chunk, send it to the exact pass
                        uint32_t r0 = q0, r1 = q1, r2 = q2, ra = ua;
                        red_shared(ra, 0u - __byte_perm(wd[c][0], o20, 0x7640));
#pragma unroll
                        for (int j = 1; j < kChunk; ++j) {
                            tile_step(r0, r1, r2, ra, e[0], e[1], e[2], sx, sy);
                            red_shared(ra, 0u - __byte_perm(wd[c][j >> 2], o20, 0x7640 | (j & 3)));
                        }
                        push_fan(fa, f, line, (cth >> 4) + c);
                        ++ndef;
                    } else if (kBox && o20 != 0u) {
                        fan_box(bb, A, D, cth + 16 * c, 16);
                    }
                    if (more) load_half(c, fn, tyn, txn);
                }
            } else {
                const uint32_t sx = neg[0] ? 0u - 8u : 8u, sy = neg[1] ? 0u - nx8 : nx8, sz = neg[2] ? 0u - sxy8 : sxy8;
                uint32_t off = 8u * (uint32_t)(ix - dsc.X0) + nx8 * (uint32_t)(iy - dsc.Y0) + sxy8 * (uint32_t)(iz - dsc.Z0);
                const unsigned long long gb = (unsigned long long)fa.acc + (unsigned long long)dsc.dbase;
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    if (c > 0) off_step(v0, v1, v2, off, e[0], e[1], e[2], sx, sy, sz);
                    uint32_t tmin = min(v0, min(v1, v2));
                    uint32_t run = __byte_perm(wd[c][0], 0x00100000u, 0x7640), ptr = rbuf;
#pragma unroll
                    for (int j = 1; j < kChunk; ++j) {
                        run_step(v0, v1, v2, off, run, ptr, e[0], e[1], e[2], sx, sy, sz, 8u * NT);
                        tmin = min(tmin, min(v0, min(v1, v2)));
                        run += __byte_perm(wd[c][j >> 2], 0x00100000u, 0x7640 | (j & 3));
                    }
                    if (more) load_half(c, fn, tyn, txn);
                    const bool in = (wmask >> c) & 1u, keep = in && tmin >= tie2;
                    if (in && !keep) {  // rare: the chunk's runs are dropped, it goes to the exact pass
                        push_fan(fa, f, line, (cth >> 4) + c);
                        ++ndef;
                    }
                    if (keep) red_word(gb + off, run);  // the open run
#if SVR_FAN_DRAINPF
                    // software-pipelined: entry k + 1 is read (and zeroed) before entry k's RED
                    if (rbuf != ptr) {
                        uint32_t o, r, q = rbuf;
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n\tst.shared.v2.u32 [%2], {%3, %3};"
                                     : "=r"(o), "=r"(r) : "r"(q), "r"(0u) : "memory");
                        for (q += 8u * NT; q != ptr; q += 8u * NT) {
                            uint32_t on, rn;
                            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n\tst.shared.v2.u32 [%2], {%3, %3};"
                                         : "=r"(on), "=r"(rn) : "r"(q), "r"(0u) : "memory");
                            if (keep) red_word(gb + o, r);
                            o = on;
                            r = rn;
                        }
                        if (keep) red_word(gb + o, r);
                    }
#else
                    for (uint32_t q = rbuf; q != ptr; q += 8u * NT) {
                        uint32_t o, r;
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n\tst.shared.v2.u32 [%2], {%3, %3};"
                                     : "=r"(o), "=r"(r) : "r"(q), "r"(0u) : "memory");
                        if (keep) red_word(gb + o, r);
                    }
#endif
                    if (kBox && keep) fan_box(bb, A, D, cth + 16 * c, 16);
                }
            }
        }
        else if (more) {
            load_px(fn, tyn, txn);
        }
        if (noob) atomicAdd(&s_cnt[0], noob);
        if (ndef) atomicAdd(&s_cnt[1], ndef);
        if (tid == 0) s_px += (unsigned long long)TCOLS * (unsigned long long)nlines;
        wait_stage();
        if (table) {  // (CTA-uniform)
            __syncthreads();  // table complete
            const int X = dsc.XY & 0xffff, Y = dsc.XY >> 16, stride = dsc.stride;
            const unsigned long long fbase = (unsigned long long)fa.acc + (unsigned long long)dsc.base;
            const uint32_t zpar = (uint32_t)dsc.zpar;
            const float p1 = dsc.p1, p2 = dsc.p2;
            const int XY = X * Y;
            const float rX = __fdividef(1.0f, (float)X);  // (MUFU.RCP suffices: see k_pnn_tiles)
            // y = p / X exactly: the quotients' fractional parts are >= 1/(2X) from an integer
            const int y0 = (int)(((float)tid + 0.5f) * rX);
            int x = tid - y0 * X;
            const int dy = (int)(((float)NT + 0.5f) * rX), dx = NT - dy * X;
            int ti = x + stride * y0;
            uint32_t go = (uint32_t)y0 * nx8 + (uint32_t)x * 8u;
            float tt = fmaf(p2, (float)y0, fmaf(p1, (float)x, dsc.tt0));
            const int dti = dx + stride * dy, wti = stride - X;
            const uint32_t dgo = (uint32_t)dy * nx8 + (uint32_t)dx * 8u, wgo = nx8 - 8u * (uint32_t)X;
            const float dtt = p1 * (float)dx + p2 * (float)dy, wtt = p2 - p1 * (float)X;
            for (int p = tid; p < XY; p += NT) {
                const uint32_t v0 = s_tab[ti], v1 = s_tab[ti + kTabPlane];
                s_tab[ti] = 0u;
                s_tab[ti + kTabPlane] = 0u;
                const uint32_t k = (uint32_t)(int)ceilf(tt);  // k - kmin >= 0
                const bool odd = ((k ^ zpar) & 1u) != 0u;
                const unsigned long long a0 = fbase + (k * sxy8 + go);
                // per slot: an empty slot's voxel may lie outside the slab (face tiles)
                const uint32_t vlo = odd ? v1 : v0, vhi = odd ? v0 : v1;
                if (vlo) red_word(a0, vlo);
                if (vhi) red_word(a0 + sxy8, vhi);
                x += dx;
                ti += dti;
                go += dgo;
                tt += dtt;
                if (x >= X) {
                    x -= X;
                    ti += wti;
                    go += wgo;
                    tt += wtt;
                }
            }
        }
        f = fn;
        ty = tyn;
        tx = txn;
    }
    __syncthreads();
    if (kBox && cur_f >= 0) flush_box(bb, fa.boxes + 6 * cur_f);
    if (tid == 0) {
        const ull oob = 16ull * s_cnt[0], def = s_cnt[1], n_px = s_px;
        if (n_px > oob + 16ull * def) atomicAdd(&fa.stats[kStInserted], n_px - oob - 16ull * def);
        if (oob) atomicAdd(&fa.stats[kStOob], oob);
        if (def) atomicAdd(&fa.stats[kStDeferred], def);
        if (ntiles_cta) atomicAdd(&fa.stats[kStTiles], (ull)ntiles_cta);
    }
}

}  // namespace svr
