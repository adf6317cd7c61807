// svr_k1.cuh — K1, the pixel-nearest-neighbour insert of linear-probe B-scans,
// as a persistent tile kernel.  Included by svr_api.cu after svr_kernels.cuh.
//
// Work unit: a tile of TCOLS = 16*NCH columns x TROWS = 32*NW rows of one frame.  The tiles
// (frame-major) go round-robin over persistent CTAs, so the CTAs in flight together cover a
// window of ~grid consecutive tiles: neighbouring frames' adds to the same voxels meet in L2 (a
// CTA walking a contiguous range instead spread them over the whole launch: 76% of the REDs'
// sectors missed L2, profiles/r2_opt_log.md).  Each tile's descriptor and frame constants are
// staged with cp.async two tiles ahead.
//
// Lane map: thread (warp w, lane l) walks the whole TCOLS-pixel row r = w + NW*l of the tile.  The
// 32 lanes of a warp then sit on rows NW apart (cfg2: 1.67 voxels apart in y), so one shared
// atomic of the warp hits ~2 banks' worth of words instead of ~4 (same-address lanes serialise
// on B200: tools/ubench_atoms.cu; the bank model is in profiles/r2_opt_log.md).
//
// Per pixel the walk is, in SASS, 3 x (IADD3 with carry-out to a predicate + one predicated
// address update) + the tie screen + PRMT + ATOMS: the fixed-point fractions of
// u = K + col*Dc + row*Dr (32.32) are stepped exactly, the index moves where a
// fraction carries, and the shared-table byte address moves with it (x: +-4, y: +-4*STR,
// z: to the other parity plane, bit 1 << 14; a B-scan plane puts <= 2 z values in a voxel column).
// The kZ1 variant (frames with at most one y and one z carry per 16-pixel chunk) keeps the ALU
// pipe, the walk's limit, to the carries, an x-only tie screen and the PRMT: the z move is a
// predicated add and the y / z post-carry fractions are captured by predicated FMA-pipe moves.
// A 16-pixel chunk whose fractions came within the certified tie window is undone and its
// pixels go to the exact worklist pass (k_pnn_work), as before.
//
// Flush: thread (x, r) reads and zeroes both parity slots of table column x in rows r, r + R, ...
// (R = threads div X; the next tile then starts from a clean table without a zeroing pass), finds
// the slots' z from the frame plane and issues one predicated 64-bit red.global.add per non-empty
// slot.
#pragma once

#ifndef SVR_TILES_PREFETCH
#define SVR_TILES_PREFETCH 0  // k_pnn_tiles: L2 prefetch of each row's first voxel line (A/B: 0.571 vs 0.565 ms without)
#endif
#ifndef SVR_K1_ORDER
#define SVR_K1_ORDER 0  // k_pnn_tiles tile order: 0 frame-major, 1 tile-major (frames fastest)
#endif
#ifndef SVR_FLUSH_UNROLL
#define SVR_FLUSH_UNROLL 1  // k_pnn_tiles flush loop unroll
#endif
#ifndef SVR_TILES_MINB
#define SVR_TILES_MINB 6  // k_pnn_tiles (128 threads): CTAs per SM the register budget is cut for (A/B: 6 beat 7, 8)
#endif

namespace svr {

// Table layout: word (x + kTabStr y) of parity plane p (planes 16 KB apart) holds voxel column
// (x, y)'s slot of z parity p.  The walk's byte address is absolute (no base add per pixel) and a
// z step XORs its bit 14: plane 0 spans [tab, tab + 8 KB) with tab < 8 KB (static shared memory
// starts at the CTA's 1 KB reserved area; checked per CTA), so bit 14 is 0 there and 1 in plane 1.
// kTabStr is odd, so rows 1-2 voxels apart (a warp's lanes) fall into distinct banks.
constexpr int kFlushUnroll = SVR_FLUSH_UNROLL;
constexpr int kTabStr = 33;                    // table row stride in words
constexpr int kTabPlane = 4096;                // words between the parity planes (bit 14)
constexpr int kTabMaxY = 62;                   // voxel rows (62 * 33 <= 2048 words per plane)
constexpr int kTabMaxX = 32;                   // voxel columns
constexpr int kTabWords = kTabPlane + 2048;    // 24 KB (the 8 KB gap is unused)

// k_pnn_tiles table geometry (one for every tile height: a 12 KB table of 31 rows for the 64-row
// tiles measured no faster and refused frames with long row steps)
template <int NW>
struct TabGeom {
    static constexpr int kBit = 16384;       // byte distance of the parity planes
    static constexpr int kPlane = kBit / 4;  // in words
    static constexpr int kMaxY = kTabMaxY;
    static constexpr int kWords = kPlane + ((kMaxY * kTabStr + 3) & ~3);
};

struct TilesArgs {
    const uint8_t* px;
    long long pitch, fstride;
    int h;
    int ntx, nty;        // tiles per frame
    long long ntiles;    // nframes * ntx * nty
    const FrameParams* fps;
    GridDev g;
    ull* acc;
    int* boxes;
    ull* stats;
    ull* work;
    unsigned int* work_n;
    unsigned int work_cap;
    const struct TileDesc* desc;  // per-tile constants (k_tile_desc)
    struct TileFrame* frc;        // per-frame constants (k_tile_desc)
};

// Per-tile constants, computed once per tile by k_tile_desc instead of redundantly by every warp
// of the insert (the per-warp uniform setup had cost ~4 instructions per pixel).
struct __align__(16) TileDesc {
    long long Ut[3];        // 32.32 fixed u at the tile's (col, row) origin, +1/2
    long long base;         // flush base: byte offset of voxel (X0, Y0, zint + kmin) in the slab
    int X0, Y0;             // table origin (voxel), the tile's fixed-point index minima
    int XY;                 // X | Y << 16: table extent
    int flags;              // bit 0 tok (table usable), bit 1 tin (inside grid / slab)
    int zpar;               // (zint + kmin) & 1
    float tt0;              // z_c - h at the table origin, minus kmin (flush plane offset)
    int pad[2];
};

// one exact step of the three fractions; the table byte address follows the carries
template <int kBit = 16384>
__device__ __forceinline__ void tile_step(uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& a,
                                          uint32_t e0, uint32_t e1, uint32_t e2, uint32_t sx,
                                          uint32_t sy) {
    asm("{\n\t.reg .pred p0, p1, p2;\n\t.reg .u32 c0, c1, c2;\n\t"
        "add.cc.u32 %0, %0, %4;\n\taddc.u32 c0, 0, 0;\n\t"
        "add.cc.u32 %1, %1, %5;\n\taddc.u32 c1, 0, 0;\n\t"
        "add.cc.u32 %2, %2, %6;\n\taddc.u32 c2, 0, 0;\n\t"
        "setp.ne.u32 p0, c0, 0;\n\tsetp.ne.u32 p1, c1, 0;\n\tsetp.ne.u32 p2, c2, 0;\n\t"
        "@p0 add.u32 %3, %3, %7;\n\t@p1 add.u32 %3, %3, %8;\n\t@p2 xor.b32 %3, %3, %9;\n\t}"
        : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(a)
        : "r"(e0), "r"(e1), "r"(e2), "r"(sx), "r"(sy), "n"(kBit));
}

// kZ1 step (at most one y and one z carry per chunk, tile_shapes_fit): the z move is +-16 KB
// (dz, fixed per chunk by its start parity) as a predicated add, which ptxas puts on the FMA pipe
// like the x and y moves -- the walk is ALU-bound (carries, tie screen, PRMT).  A tie in y or z can
// only sit at the chunk start (screened there) or right after the axis' one carry; that post-carry
// fraction is recovered after the chunk from the final one (carry_residue), so the per-pixel tie
// screen needs only x.
__device__ __forceinline__ void tile_step_z1(uint32_t& w0, uint32_t& w1, uint32_t& w2, uint32_t& a,
                                             uint32_t e0, uint32_t e1, uint32_t e2, uint32_t sx,
                                             uint32_t sy, uint32_t dz) {
    asm("{\n\t.reg .pred p0, p1, p2;\n\t.reg .u32 c0, c1, c2;\n\t"
        "add.cc.u32 %0, %0, %4;\n\taddc.u32 c0, 0, 0;\n\t"
        "add.cc.u32 %1, %1, %5;\n\taddc.u32 c1, 0, 0;\n\t"
        "add.cc.u32 %2, %2, %6;\n\taddc.u32 c2, 0, 0;\n\t"
        "setp.ne.u32 p0, c0, 0;\n\tsetp.ne.u32 p1, c1, 0;\n\tsetp.ne.u32 p2, c2, 0;\n\t"
        "@p0 add.u32 %3, %3, %7;\n\t@p1 add.u32 %3, %3, %8;\n\t@p2 add.u32 %3, %3, %9;\n\t}"
        : "+r"(w0), "+r"(w1), "+r"(w2), "+r"(a)
        : "r"(e0), "r"(e1), "r"(e2), "r"(sx), "r"(sy), "r"(dz));
}

// The post-carry fraction of an axis that carried at most once in a chunk, from its final fraction
// w: the fractions after the carry are w_c, w_c + e, ..., w = w_c + m e with 0 <= w_c < e, so w_c =
// w mod e.  The quotient m <= 15 comes from fp32 (relative error ~2^-21, so it is off only when w / e
// sits within ~1e-5 of a half-integer, far from a tie) and the residue w - m e is exact modulo 2^32:
// where w_c is in the tie window the result is w_c exactly; otherwise it is >= the window (or wraps
// to a huge value).  Only called for an axis that carried in the chunk (its final fraction wrapped
// below the start one).  rcp = 1 / e.
__device__ __forceinline__ uint32_t carry_residue(uint32_t w, uint32_t e, float rcp) {
    const uint32_t m = (uint32_t)__float2int_rn(__uint2float_rn(w) * rcp);
    return w - m * e;
}

#ifndef SVR_PX_DP4A
#define SVR_PX_DP4A 1  // pixel word as IDP.4A (FMA pipe) instead of PRMT (ALU pipe, the walk's limit)
#endif
// table add of byte k of w: the byte + o20 (count 1 << 20 for a chunk that writes, 0 otherwise)
__device__ __forceinline__ uint32_t px_word(uint32_t w, int k, uint32_t o20) {
#if SVR_PX_DP4A
    return __dp4a(w, 1u << (8 * k), o20);
#else
    return __byte_perm(w, o20, 0x7640 | k);
#endif
}

// A frame's constants (k_tile_desc writes one per frame), staged in shared memory with each
// tile's descriptor (keeps the 64-register budget for the walk).
struct __align__(16) TileFrame {
    long long Dc[3], Dr[3];        // 32.32 fixed: du/dcol, du/drow
    uint32_t E[3], neg[3];         // |Dc| low words; all-ones when Dc < 0 (mirrored fractions)
    uint32_t te2, sx, sy;          // tie window + 1; table byte steps along x and y
    float p1, p2;                  // frame plane slopes (FrameParams::pz[1], pz[2])
    uint32_t pad;                  // 4096 (opaque to ptxas)
};
static_assert(sizeof(TileFrame) == 96, "TileFrame is staged as 6 x 16 bytes");

__device__ __forceinline__ void push_work(const TilesArgs& ta, int f, int row, int cc, uint32_t mask = 0xffffu) {
    // the host sizes the list for every chunk of the launch, so it cannot overflow
    const unsigned int slot = atomicAdd(ta.work_n, 1u);
    ta.work[slot] = work_entry(f, row, cc, mask);
}

// bit j set where pixel j of the chunk is zero (skip_zero)
__device__ __forceinline__ uint32_t zero_mask16(const uint32_t (&w)[4]) {
    uint32_t m = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i)  // bytes 0..3 of __vcmpeq4's 0xff / 0x00 -> bits 24..27 of the product
        m |= (((__vcmpeq4(w[i], 0u) & 0x01010101u) * 0x01020408u) >> 24 & 0xfu) << (4 * i);
    return m;
}

template <int NCH, int NW, bool kZ1>
__global__ void __launch_bounds__(128) k_tile_desc(const TilesArgs ta, TileDesc* __restrict__ out) {
    constexpr int TROWS = 32 * NW, TCOLS = 16 * NCH;
    constexpr int kShape = (NCH == 2) + 2 * (NW == 2);
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ta.ntiles) return;
    const int tpf = ta.ntx * ta.nty;
    const int f = (int)(t / tpf), rem = (int)(t - (long long)f * tpf);
    const int ty = rem / ta.ntx, tx = rem - ty * ta.ntx;
    const FrameParams& fp = ta.fps[f];
    const GridDev& g = ta.g;
    const int c0t = tx * TCOLS, r0t = ty * TROWS;
    const int nr1 = min(TROWS, ta.h - r0t) - 1;
    TileDesc d;
    int lo[3], hi[3];
    // (a frame the launch's walk variant does not fit -- only possible in a frame graph captured
    // for another frame -- takes the exact pass tile by tile)
    bool ok = fp.plane_ok && ((fp.lin_fit >> kShape) & 1) && (!kZ1 || (fp.lin_fit & 16));
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long dc = fp.Dc[k], dr = fp.Dr[k];
        d.Ut[k] = fp.A[k] + (long long)r0t * dr + (long long)c0t * dc;
        const long long c1 = (long long)(TCOLS - 1) * dc, r1 = (long long)nr1 * dr;
        // u is affine in (col, row): its fixed-point extremes over the tile sit at corners
        lo[k] = (int)((d.Ut[k] + min(0ll, c1) + min(0ll, r1)) >> 32);
        hi[k] = (int)((d.Ut[k] + max(0ll, c1) + max(0ll, r1)) >> 32);
        ok = ok && (unsigned long long)(dc < 0 ? -dc : dc) < (1ull << 32);
    }
    const int X = hi[0] - lo[0] + 1, Y = hi[1] - lo[1] + 1;
    ok = ok && X <= kTabMaxX && Y <= TabGeom<NW>::kMaxY;
    const bool tin = lo[0] >= 0 && hi[0] <= g.nx - 1 && lo[1] >= 0 && hi[1] <= g.ny - 1 &&
                     lo[2] >= g.zb && hi[2] <= g.zb + g.nzl - 1;
    d.X0 = lo[0];
    d.Y0 = lo[1];
    d.XY = X | (Y << 16);
    d.flags = (ok ? 1 : 0) | (tin ? 2 : 0);
    // flush plane: the column (x, y) holds voxels z in [z_c - h, z_c + h] (2h < 2), z_c - h =
    // zint + tt0 + kmin + p1 x + p2 y (x, y table-relative; fp32 relative to the tile corner, error
    // ~2e-5 against the 2e-3 margin in pz3); k = ceil(tt) >= 0 for every table position
    const double zt = fp.pz[0] + fp.pz[1] * (double)lo[0] + fp.pz[2] * (double)lo[1] - fp.pz[3];
    const int zint = (int)floor(zt);
    const float zf0 = (float)(zt - (double)zint);
    const float p1 = (float)fp.pz[1], p2 = (float)fp.pz[2];
    const int kmin = -1 + (int)floorf(zf0 + fminf(0.f, p1 * (float)(X - 1)) + fminf(0.f, p2 * (float)(Y - 1)));
    d.tt0 = zf0 - (float)kmin;
    d.zpar = (zint + kmin) & 1;
    const long long sxy = (long long)g.nx * g.ny;
    d.base = 8ll * ((long long)(zint + kmin - g.zb) * sxy + (long long)lo[1] * g.nx + lo[0]);
    d.pad[0] = d.pad[1] = 0;
    out[t] = d;
    if (rem == 0) {  // the frame's constants, once
        TileFrame fr;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const long long dc = fp.Dc[k];
            fr.Dc[k] = dc;
            fr.Dr[k] = fp.Dr[k];
            fr.E[k] = (uint32_t)(dc < 0 ? -dc : dc);
            fr.neg[k] = dc < 0 ? 0xffffffffu : 0u;
        }
        fr.te2 = fp.tie_eps + 1;
        fr.sx = fp.Dc[0] < 0 ? 0u - 4u : 4u;
        fr.sy = fp.Dc[1] < 0 ? 0u - 4u * kTabStr : 4u * kTabStr;
        fr.p1 = (float)fp.pz[1];
        fr.p2 = (float)fp.pz[2];
        fr.pad = 4096u;  // (an opaque 2^12: the flush's FMA-pipe word split)
        ta.frc[f] = fr;
    }
}

// Walk state (fractions + table byte address) of the pixel whose fixed-point u is (u0, u1, u2).
// The index taken is the one the carries of W track: when lo + te2 wraps (the pixel sits in the
// upper half of the tie window) the index is already one step further, so later pixels' indices
// stay exact no matter where the row starts (the pixel itself is a tie and gets deferred).
__device__ __forceinline__ void walk_state(long long u0, long long u1, long long u2, const TileFrame& fr,
                                           int X0, int Y0, uint32_t tab, uint32_t pb, uint32_t& w0,
                                           uint32_t& w1, uint32_t& w2, uint32_t& a) {
    const uint32_t te2 = fr.te2;
    const uint32_t m0 = (uint32_t)u0 ^ fr.neg[0], m1 = (uint32_t)u1 ^ fr.neg[1], m2 = (uint32_t)u2 ^ fr.neg[2];
    w0 = m0 + te2;
    w1 = m1 + te2;
    w2 = m2 + te2;
    // +-1 where the offset add wrapped (direction of the step: neg = all ones -> -1)
    const int ix = (int)(u0 >> 32) + (w0 < te2 ? (fr.neg[0] ? -1 : 1) : 0);
    const int iy = (int)(u1 >> 32) + (w1 < te2 ? (fr.neg[1] ? -1 : 1) : 0);
    const int iz = (int)(u2 >> 32) + (w2 < te2 ? 1 : 0);  // (only the parity matters)
    a = tab + 4u * (uint32_t)((ix - X0) + kTabStr * (iy - Y0)) + (uint32_t)(iz & 1) * pb;  // pb: plane bytes
}

// 32-byte row segment load (one LDG.256, L1 no-allocate: every byte is read once)
__device__ __forceinline__ void ld256(const uint8_t* p, uint32_t* r) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "l"(p));
}

// unconditional 64-bit add of a table word (count << 20 | sum) as (count << 32 | sum)
__device__ __forceinline__ void red_word(unsigned long long addr, uint32_t v) {
    asm volatile(
        "{\n\t.reg .b32 hi, lo;\n\t.reg .b64 w;\n\t"
        "shr.u32 hi, %1, 20;\n\tand.b32 lo, %1, 1048575;\n\t"
        "mov.b64 w, {lo, hi};\n\tred.relaxed.gpu.global.add.u64 [%0], w;\n\t}" ::"l"(addr), "r"(v) : "memory");
}

// the same, predicated on v != 0 inside the asm (no branch around the RED)
__device__ __forceinline__ void red_word_nz(unsigned long long addr, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 hi, lo;\n\t.reg .b64 w;\n\t"
        "setp.ne.u32 p, %1, 0;\n\tshr.u32 hi, %1, 20;\n\tand.b32 lo, %1, 1048575;\n\t"
        "mov.b64 w, {lo, hi};\n\t@p red.relaxed.gpu.global.add.u64 [%0], w;\n\t}" ::"l"(addr), "r"(v) : "memory");
}

// kSkip (skip_zero): a chunk of 16 zero pixels adds nothing and is counted skipped
// whatever its position; a chunk with some zero pixels goes to the exact pass with the mask of its
// non-zero pixels (per-pixel counters and boxes there), its zeros counted skipped here.
template <int NCH, int NW, bool kBox, bool kZ1, bool kSkip = false>
__global__ void __launch_bounds__(32 * NW, NW == 4 ? SVR_TILES_MINB : 2 * SVR_TILES_MINB) k_pnn_tiles(const TilesArgs ta) {
    constexpr int NT = 32 * NW, TROWS = 32 * NW, TCOLS = 16 * NCH;
    using TG = TabGeom<NW>;
    __shared__ __align__(16) uint32_t s_tab[TG::kWords];
    __shared__ TileFrame s_frs[3];       // ring (tiles i, i + 1, i + 2): frame constants
    __shared__ TileDesc s_desc[3];       //   and descriptors, cp.async-staged
    // chunks counted out of bounds / deferred (rare); skip_zero: all-zero chunks, zero pixels of
    // mixed chunks, and those of them in chunks walked here
    __shared__ unsigned int s_cnt[5];
    __shared__ unsigned long long s_px;  // pixels of this CTA's tiles
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 5) s_cnt[tid] = 0u;
    if (tid == 0) s_px = 0ull;
    for (int i = tid; i < TG::kWords / 4; i += NT)
        reinterpret_cast<uint4*>(s_tab)[i] = make_uint4(0u, 0u, 0u, 0u);
    const uint32_t tab = (uint32_t)__cvta_generic_to_shared(s_tab);
    // (the XOR parity needs plane 0 below 16 KB - 8 KB; otherwise every tile takes the exact pass)
    const bool tab_ok = tab + 4u * (uint32_t)(TG::kMaxY * kTabStr) <= (uint32_t)TG::kBit;
    const GridDev& g = ta.g;
    const int tpf = ta.ntx * ta.nty;
    // tiles round-robin over the CTAs: the CTAs in flight together work on a window of ~grid
    // consecutive tiles (a few dozen frames), so neighbouring frames' adds to the same voxels
    // meet in L2 instead of each reading the voxel's sector from HBM
    const long long t0 = blockIdx.x, tstep = gridDim.x, t1 = ta.ntiles;
    // tile t as a mixed-radix counter of digits a0 (fastest, radix R0), a1 (R1), a2, advanced by
    // tstep without divisions.  Frame-major order: a0 = tile column, a1 = tile row, a2 = frame;
    // tile-major (SVR_K1_ORDER 1): a0 = frame, a1 = tile column, a2 = tile row
#if SVR_K1_ORDER
    const int R0 = (int)(t1 / tpf), R1 = ta.ntx;
#define SVR_K1_DIGITS(fq, tyq, txq) int& a0 = fq; int& a1 = txq; int& a2 = tyq
#else
    const int R0 = ta.ntx, R1 = ta.nty;
#define SVR_K1_DIGITS(fq, tyq, txq) int& a0 = txq; int& a1 = tyq; int& a2 = fq
#endif
    const long long R01 = (long long)R0 * R1;
    __shared__ int s_adv[3];  // tstep as (a0, a1, a2) digits
    if (tid == 0) {
        const int sf = (int)(tstep / R01), sr = (int)(tstep - (long long)sf * R01);
        s_adv[0] = sf;
        s_adv[1] = sr / R0;
        s_adv[2] = sr - s_adv[1] * R0;
    }
    __syncthreads();
    auto advance = [&](int& fq, int& tyq, int& txq) {  // tile + tstep, without divisions
        SVR_K1_DIGITS(fq, tyq, txq);
        a0 += s_adv[2];
        a1 += s_adv[1];
        a2 += s_adv[0];
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
    {
        SVR_K1_DIGITS(f, ty, tx);
        a2 = (int)(t0 / R01);
        const int r = (int)(t0 - (long long)a2 * R01);
        a1 = r / R0;
        a0 = r - a1 * R0;
    }
#undef SVR_K1_DIGITS
    int cur_f = -1;
    unsigned int ntiles_cta = 0;
    int slot = 0;
    BoxAcc bb;

    // Rows of a short last tile go to whole warps (rows w + S l, S = active warps): an idle warp
    // skips the walk, and no idle lane's clamped address can collide with a live lane's bank.
    auto tile_rows = [&](int tyq, int& S, int& row, bool& act, int& rowc) {
        const int r0 = tyq * TROWS;
        S = min(NW, (min(TROWS, ta.h - r0) + 31) >> 5);
        row = r0 + warp + S * lane;
        act = warp < S && row < ta.h;
        rowc = act ? row : ta.h - 1;
    };
    // this thread's row of pixels (software-pipelined: the next tile's rows are requested before
    // the current tile's flush)
    uint32_t wd[NCH][4];
    auto load_rows = [&](int fq, int txq, int rowq, uint32_t (&d)[NCH][4]) {
        const uint8_t* src = ta.px + (long long)fq * ta.fstride + (long long)rowq * ta.pitch + txq * TCOLS;
#pragma unroll
        for (int c = 0; c < NCH; c += 2) ld256(src + 16 * c, &d[c][0]);
    };
    // threads 0..3 stage a tile's descriptor (4 x 16 B), 4..9 its frame's constants (6 x 16 B);
    // one commit group per tile (empty for the other threads): waiting for all but the newest
    // group leaves the tile two ahead in flight
    auto stage = [&](int fq, int tyq, int txq, int b) {
        const long long t = (long long)fq * tpf + tyq * ta.ntx + txq;
        if (tid < 4) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<uint4*>(&s_desc[b]) + tid);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(reinterpret_cast<const uint4*>(ta.desc + t) + tid) : "memory");
        } else if (tid < 10) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<uint4*>(&s_frs[b]) + (tid - 4));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(reinterpret_cast<const uint4*>(ta.frc + fq) + (tid - 4)) : "memory");
        }
    };
    auto commit = [&]() { asm volatile("cp.async.commit_group;" ::: "memory"); };
    auto wait_stage = [&]() { asm volatile("cp.async.wait_group 1;" ::: "memory"); };
    if (t0 < t1) {
        int S, row, rowc;
        bool act;
        tile_rows(ty, S, row, act, rowc);
        load_rows(f, tx, rowc, wd);
        stage(f, ty, tx, 0);
        commit();
        int f1 = f, ty1 = ty, tx1 = tx;
        advance(f1, ty1, tx1);
        if (t0 + tstep < t1) stage(f1, ty1, tx1, 1);
        commit();
        wait_stage();
    }

    for (long long t = t0; t < t1; t += tstep) {
        if (kBox && f != cur_f) {  // CTA-uniform
            if (cur_f >= 0) {
                flush_box(bb, ta.boxes + 6 * cur_f);
                bb = BoxAcc();
            }
            cur_f = f;
        }
        __syncthreads();  // frame constants + descriptor staged; table zeroed or flushed
        const int b = slot;
        slot = slot == 2 ? 0 : slot + 1;
        ++ntiles_cta;
        // the tile after next is requested now (only the ten staging threads work out which it is)
        if (tid < 10) {
            int f2 = f, ty2 = ty, tx2 = tx;
            advance(f2, ty2, tx2);
            advance(f2, ty2, tx2);
            if (t + 2 * tstep < t1) stage(f2, ty2, tx2, b == 0 ? 2 : b - 1);
        }
        commit();
        const TileFrame& s_fr = s_frs[b];
        const TileDesc& dsc = s_desc[b];
        const int c0t = tx * TCOLS, r0t = ty * TROWS;
        const int X0 = dsc.X0, Y0 = dsc.Y0, X = dsc.XY & 0xffff, Y = dsc.XY >> 16;
        const bool tok = (dsc.flags & 1) && tab_ok, tin = dsc.flags & 2;
        int S, row, rowc;
        bool act;
        tile_rows(ty, S, row, act, rowc);
        if (!act) {  // (idle warps and lanes past a short tile's end: add nothing)
#pragma unroll
            for (int c = 0; c < NCH; ++c) wd[c][0] = wd[c][1] = wd[c][2] = wd[c][3] = 0u;
        }
        // fixed-point u at the start of chunk c of this thread's row
        const int rrel = rowc - r0t;
        auto chunk_u = [&](int c, int k) -> long long {
            return dsc.Ut[k] + (long long)rrel * s_fr.Dr[k] + (long long)(16 * c) * s_fr.Dc[k];
        };
        // (kSkip) chunks with zero pixels: all zero -> skipped; mixed -> walked with per-pixel
        // counts in inside tiles of a batch insert, else sent to the exact pass with their mask
        // (boxes and face counters per pixel there)
        uint32_t handled = 0u, zmr[kSkip ? NCH : 1] = {};
        if constexpr (kSkip) {
            if (act) {
                uint32_t nskip = 0u, nzero = 0u, nzwalk = 0u;
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const uint32_t zm = zero_mask16(wd[c]);
                    zmr[c] = zm;
                    if (zm == 0xffffu) {
                        handled |= 1u << c;
                        ++nskip;
                    } else if (zm != 0u) {
                        nzero += __popc(zm);
                        if (kBox || !tok || !tin) {
                            handled |= 1u << c;
                            push_work(ta, f, row, (c0t >> 4) + c, zm ^ 0xffffu);
                            atomicAdd(&s_cnt[1], 1u);
                        } else {
                            nzwalk += __popc(zm);
                        }
                    }
                    if ((handled >> c) & 1u) {
                        wd[c][0] = wd[c][1] = wd[c][2] = wd[c][3] = 0u;  // walked, adds nothing
                        zmr[c] = 0u;
                    }
                }
                if (nskip) atomicAdd(&s_cnt[2], nskip);
                if (nzero) atomicAdd(&s_cnt[3], nzero);
                if (nzwalk) atomicAdd(&s_cnt[4], nzwalk);
            }
        }
        // per-chunk write mask: a chunk goes into the table when its whole index range lies inside
        // the grid / slab; wholly outside -> counted out of bounds; straddling -> exact pass
        uint32_t wmask = act && tok ? ((1u << NCH) - 1u) & ~handled : 0u;
        if (act && (!tok || !tin)) {
            const int clo[3] = {0, 0, g.zb}, chi[3] = {g.nx - 1, g.ny - 1, g.zb + g.nzl - 1};
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (kSkip && ((handled >> c) & 1u)) continue;
                bool inb = true, out = false;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const long long u = chunk_u(c, k);
                    const int i0 = (int)(u >> 32), i15 = (int)((u + 15ll * s_fr.Dc[k]) >> 32);
                    // no margin needed: a tie-free chunk's fixed-point indices are the exact ones
                    // and a tie chunk is undone and deferred after its walk; the exact index is
                    // within 1 of the fixed-point one, so a range 2 outside misses the grid
                    inb = inb && min(i0, i15) >= clo[k] && max(i0, i15) <= chi[k];
                    out = out || max(i0, i15) + 1 < clo[k] || min(i0, i15) - 1 > chi[k];
                }
                if (!tok || !inb) {
                    wmask &= ~(1u << c);
                    if (out && tok) {
                        atomicAdd(&s_cnt[0], 1u);
                    } else {
                        push_work(ta, f, row, (c0t >> 4) + c);
                        atomicAdd(&s_cnt[1], 1u);
                    }
                    wd[c][0] = wd[c][1] = wd[c][2] = wd[c][3] = 0u;  // walked, adds nothing
                }
            }
        }
        // (kSkip: a warp whose rows are all zero / out of bounds has nothing to walk -- the rows
        // outside a segmented frame's band)
        if (tok && warp < S && (!kSkip || __any_sync(0xffffffffu, wmask != 0u))) {
            const uint32_t e0 = s_fr.E[0], e1 = s_fr.E[1], e2 = s_fr.E[2], sx = s_fr.sx, sy = s_fr.sy;
            const uint32_t tie2 = 2u * s_fr.te2;
            // (kZ1: 1 / e for the post-carry residues; MUFU accuracy suffices, see carry_residue)
            const float rc1 = kZ1 ? __fdividef(1.0f, (float)e1) : 0.f, rc2 = kZ1 ? __fdividef(1.0f, (float)e2) : 0.f;
            // walk state at pixel 0 of the row
            uint32_t w0, w1, w2, a;
            {
                const long long u0 = chunk_u(0, 0), u1 = chunk_u(0, 1), u2 = chunk_u(0, 2);
                walk_state(u0, u1, u2, s_fr, X0, Y0, tab, (uint32_t)TG::kBit, w0, w1, w2, a);
#if SVR_TILES_PREFETCH
                if (tin) {  // L2 prefetch of the row's first voxel line: the flush's REDs then hit L2
                    const int ix = (int)(u0 >> 32), iy = (int)(u1 >> 32), iz = (int)(u2 >> 32);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(ta.acc + (((long long)(iz - g.zb) * g.ny + iy) * g.nx + ix)));
                }
#endif
            }
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (c > 0) tile_step<TG::kBit>(w0, w1, w2, a, e0, e1, e2, sx, sy);
                const uint32_t o20 = (wmask >> c) & 1u ? 0x00100000u : 0u;
                // table word of pixel j (kSkip: a zero pixel of a mixed chunk adds no count)
                const uint32_t zmc = kSkip ? zmr[c] : 0u;
                auto pw = [&](int j) -> uint32_t {
                    const uint32_t oj = kSkip && ((zmc >> j) & 1u) ? 0u : o20;
                    return px_word(wd[c][j >> 2], j & 3, oj);
                };
                uint32_t tmin = min(w0, min(w1, w2));
                red_shared(a, pw(0));
                if (kZ1) {
                    // at most one y and one z carry in the chunk: the z move is the fixed step to
                    // the other parity plane (an add on the FMA pipe instead of an ALU XOR)
                    const uint32_t dz = (a & (uint32_t)TG::kBit) ? 0u - (uint32_t)TG::kBit : (uint32_t)TG::kBit;
                    // y and z ties can only sit at the chunk start (screened above) or right after
                    // their one carry: recovered after the walk, so per pixel only x is screened
                    const uint32_t w1s = w1, w2s = w2;
#pragma unroll
                    for (int j = 1; j < kChunk; ++j) {
                        tile_step_z1(w0, w1, w2, a, e0, e1, e2, sx, sy, dz);
                        tmin = min(tmin, w0);
                        red_shared(a, pw(j));
                    }
                    // (only where the axis carried: w wrapped below its chunk-start value)
                    const uint32_t ry = w1 < w1s ? carry_residue(w1, e1, rc1) : 0xffffffffu;
                    const uint32_t rz = w2 < w2s ? carry_residue(w2, e2, rc2) : 0xffffffffu;
                    tmin = min(tmin, min(ry, rz));
                } else {
#pragma unroll
                    for (int j = 1; j < kChunk; ++j) {
                        tile_step<TG::kBit>(w0, w1, w2, a, e0, e1, e2, sx, sy);
                        tmin = min(tmin, min(w0, min(w1, w2)));
                        red_shared(a, pw(j));
                    }
                }
                const bool tie = o20 != 0u && tmin < tie2;
                if (__any_sync(0xffffffffu, tie)) {  // rare: undo the chunk, send it to the exact pass
                    if (tie) {
                        uint32_t v0, v1, v2, ua;  // state at the chunk's pixel 0 (= the walk's)
                        walk_state(chunk_u(c, 0), chunk_u(c, 1), chunk_u(c, 2), s_fr, X0, Y0, tab, (uint32_t)TG::kBit, v0, v1, v2, ua);
                        red_shared(ua, 0u - pw(0));
#pragma unroll
                        for (int j = 1; j < kChunk; ++j) {  // (unrolled: wd stays in registers)
                            tile_step<TG::kBit>(v0, v1, v2, ua, e0, e1, e2, sx, sy);
                            red_shared(ua, 0u - pw(j));
                        }
                        push_work(ta, f, row, (c0t >> 4) + c, zmc ^ 0xffffu);
                        atomicAdd(&s_cnt[1], 1u);
                        if (kSkip && zmc) atomicSub(&s_cnt[4], (unsigned int)__popc(zmc));  // (deferred after all)
                    }
                }
                if (kBox && o20 != 0u && !tie) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const long long u = chunk_u(c, k);
                        const int i0 = (int)(u >> 32), i15 = (int)((u + 15ll * s_fr.Dc[k]) >> 32);
                        if (k == 0) { bb.x0 = min(bb.x0, min(i0, i15)); bb.x1 = max(bb.x1, max(i0, i15)); }
                        if (k == 1) { bb.y0 = min(bb.y0, min(i0, i15)); bb.y1 = max(bb.y1, max(i0, i15)); }
                        if (k == 2) { bb.z0 = min(bb.z0, min(i0, i15)); bb.z1 = max(bb.z1, max(i0, i15)); }
                    }
                }
            }
        }
        if (tid == 0) s_px += (unsigned long long)TCOLS * (unsigned long long)(min(TROWS, ta.h - r0t));
        // flush constants of this tile, then the next tile's rows + descriptor are requested
        const unsigned long long fbase = (unsigned long long)ta.acc + (unsigned long long)dsc.base;
        const uint32_t zpar = (uint32_t)dsc.zpar;
        const float tt0 = dsc.tt0;
        advance(f, ty, tx);
        wait_stage();  // (before the row load: the wait would also cover it)
        if (t + tstep < t1) {
            int Sn, rown, rowcn;
            bool actn;
            tile_rows(ty, Sn, rown, actn, rowcn);
            load_rows(f, tx, rowcn, wd);
        }
        // table complete (kSkip: a tile no thread wrote to has nothing to flush)
        bool any_written = true;
        if constexpr (kSkip) any_written = __syncthreads_or(wmask != 0u) != 0;
        else __syncthreads();
        if (tok && any_written) {
            // flush + zero: thread (x, yr) = (tid mod X, tid div X) takes column x of the table
            // rows yr, yr + R, ... (R = NT div X rows per pass; fixed per thread, so no wrap logic)
            const float p1 = s_fr.p1, p2 = s_fr.p2;
            const uint32_t sxy8 = (uint32_t)((long long)g.nx * g.ny * 8), nx8 = (uint32_t)g.nx * 8u;
            // (MUFU.RCP: its 2^-22 relative error moves the quotients below by < 1e-4, far inside
            // the 1 / (2 X) margin; the IEEE division's range check and slow path are not needed)
            const float rX = __fdividef(1.0f, (float)X);
            // exact quotients: (a + 1/2) / X is >= 1/(2X) from an integer for X <= 32
            const int yr = (int)(((float)tid + 0.5f) * rX), R = (int)(((float)NT + 0.5f) * rX);
            const int x = tid - yr * X;
            if (yr < R) {
                int ti = x + kTabStr * yr;
                uint32_t go = (uint32_t)yr * nx8 + (uint32_t)x * 8u;
                const float ttx = fmaf(p1, (float)x, tt0), Rf = (float)R;
                float yf = (float)yr;
                const int dti = kTabStr * R;
                const uint32_t dgo = (uint32_t)R * nx8;
#pragma unroll kFlushUnroll
                for (int y = yr; y < Y; y += R) {
                    const uint32_t v0 = s_tab[ti], v1 = s_tab[ti + TG::kPlane];
                    s_tab[ti] = 0u;
                    s_tab[ti + TG::kPlane] = 0u;
                    const uint32_t k = (uint32_t)(int)ceilf(fmaf(p2, yf, ttx));  // k - kmin >= 0
                    const bool odd = ((k ^ zpar) & 1u) != 0u;
                    const unsigned long long a0 = fbase + (k * sxy8 + go);
                    // per slot: an empty slot's voxel may lie outside the slab (face tiles), and a
                    // RED of 0 would still pull its line into L2 and write it back
                    const uint32_t vlo = odd ? v1 : v0, vhi = odd ? v0 : v1;
                    red_word_nz(a0, vlo);
                    red_word_nz(a0 + sxy8, vhi);
                    ti += dti;
                    go += dgo;
                    yf += Rf;
                }
            }
        }
        // (the next tile's top barrier orders this flush before its walk and before the ring
        // slot read here is staged again)
    }
    if (kBox && cur_f >= 0) flush_box(bb, ta.boxes + 6 * cur_f);
    if (tid == 0) {  // (after the loop's last barrier: s_cnt is final)
        const ull oob = 16ull * s_cnt[0], def = s_cnt[1], n_px = s_px;
        const ull skp = kSkip ? 16ull * s_cnt[2] : 0ull, zwk = kSkip ? (ull)s_cnt[4] : 0ull;
        // every pixel of the CTA's tiles is inserted here unless counted out of bounds, skipped
        // or deferred (k_pnn_work counts the deferred chunks' pixels)
        if (n_px > oob + 16ull * def + skp + zwk)
            atomicAdd(&ta.stats[kStInserted], n_px - oob - 16ull * def - skp - zwk);
        if (kSkip && skp + s_cnt[3]) atomicAdd(&ta.stats[kStSkipped], skp + (ull)s_cnt[3]);
        if (oob) atomicAdd(&ta.stats[kStOob], oob);
        if (def) atomicAdd(&ta.stats[kStDeferred], def);
        if (ntiles_cta) atomicAdd(&ta.stats[kStTiles], (ull)ntiles_cta);
    }
}

}  // namespace svr
