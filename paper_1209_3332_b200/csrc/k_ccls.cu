// k_ccls.cu -- "CCL-select": per-pixel u8 outputs that depend on a property of the pixel's
// connected component, without a per-pixel label plane in HBM.  Used by S2 RBC detection
// (components of RBC_LO that contain an RBC_HI pixel), S5 AreaThreshold
// (components of the candidate mask with min <= area <= max) and S6 FillHoles
// (4-connected background components that touch no tile-border pixel, PAPER.md:598,
// reading C8).
//
// k_ccl.cu's engine writes an int32 root for every pixel (64 MB per 4K tile) and every
// consumer re-reads it; here (32x32 tiles as there):
//   k_cs_local   shared-memory union-find of the tile (runs from ballots + CAS hooking, the
//                same scheme as k_ccl_local); per local component: area and property bits,
//                reduced in shared memory and written ONLY at the component's root entry
//                (global index of its minimum pixel); tile-edge pixels' roots to a compact
//                edge array; the tile's local roots to a list; the tile's kind (empty /
//                general / full) to kinds and every pixel's local root (u16, within the
//                tile) to lr;
//   k_cs_merge   cross-tile unions from the edge arrays (CAS hooking of the larger root under
//                the smaller on the sparse parent array, finds with CAS path halving);
//   k_cs_accum   every non-root local root adds its area / ORs its bits into its global root
//                and points straight at it (no unions run any more, so this is safe);
//   k_cs_out     writes the u8 output from each pixel's lr and its global root's property
//                word (one lookup per run); for S2 it re-runs the tile's union-find instead
//                (lr_mode).
// HBM traffic per pixel: the input plane once, lr written and read (2 B each way), the u8
// output once (plus small arrays); S2: its flags plane twice and the output.
// The property word packs the area (bits 0-28: images up to 2^29 - 1 px) with the OR-bits
// HIT (bit 29) and TOUCH (bit 30); atomicAdd of areas never carries into the flag bits.
#include <climits>

#include "hp_internal.cuh"

namespace hp {
namespace {

constexpr int32_t kAreaMask = (1 << 29) - 1;
constexpr int32_t kHit = 1 << 29, kTouch = 1 << 30;
constexpr int kT = kTile;  // 32

enum SelMode { SEL_AREA = 0, SEL_RBC = 1, SEL_FILL = 2, SEL_AREA_TH = 3, SEL_EDGE = 4 };

struct Sel {
    const uint8_t* plane;  // SEL_AREA: candidate mask; SEL_RBC: flags; SEL_FILL: big0; SEL_AREA_TH: g
    int w, h;
    int amin, amax;
    const uint8_t* R = nullptr;    // SEL_AREA_TH: the reconstruction
    const uint8_t* rbc = nullptr;  // SEL_AREA_TH: the RBC mask
    int g1 = 0;                    // SEL_AREA_TH: top-hat threshold
    // SEL_AREA_TH: per-root bounding boxes, written at root entries only (sparse planes)
    int32_t *bx0 = nullptr, *by0 = nullptr, *bx1 = nullptr, *by1 = nullptr;
    const int32_t* gate = nullptr;  // if set: every pass is a no-op unless *gate != 0
    int32_t *P = nullptr, *X = nullptr;  // sparse root planes (default: the slot's lab / aux)
    // the pixel's byte: the plane, or for SEL_AREA_TH the top-hat candidate of S4 (PAPER.md:596,
    // reading C9): (g - recon > g1) & !rbc
    template <int MODE>
    __device__ __forceinline__ uint8_t load(int64_t p) const {
        if (MODE == SEL_AREA_TH) return ((int)__ldg(plane + p) - (int)__ldg(R + p)) > g1 && !__ldg(rbc + p);
        return __ldg(plane + p);
    }
    // the bytes of pixels x0 .. x0 + 3 of row y (x0 a multiple of 4, y < h): one 32-bit load per
    // plane where the row is 4-byte aligned and the 4 pixels lie in the image, else per byte
    // (out-of-image bytes 0)
    template <int MODE>
    __device__ __forceinline__ uint32_t load4(int y, int x0) const {
        const int64_t p = (int64_t)y * w + x0;
        if ((w & 3) == 0 && x0 + 3 < w) {
            const uint32_t a = __ldg(reinterpret_cast<const unsigned int*>(plane + p));
            if (MODE != SEL_AREA_TH) return a;
            const uint32_t r = __ldg(reinterpret_cast<const unsigned int*>(R + p));
            const uint32_t b = __ldg(reinterpret_cast<const unsigned int*>(rbc + p));
            uint32_t o = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int gv = (a >> (8 * k)) & 0xff, rv = (r >> (8 * k)) & 0xff, bv = (b >> (8 * k)) & 0xff;
                o |= (uint32_t)((gv - rv) > g1 && !bv) << (8 * k);
            }
            return o;
        }
        uint32_t o = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (x0 + k < w) o |= (uint32_t)load<MODE>(p + k) << (8 * k);
        return o;
    }
    template <int MODE>
    __device__ __forceinline__ bool fg(uint8_t v) const {
        if (MODE == SEL_AREA || MODE == SEL_AREA_TH || MODE == SEL_EDGE) return v != 0;
        if (MODE == SEL_RBC) return (v & HP_FLAG_RBC_LO) != 0;
        return v == 0;  // SEL_FILL: background of big0
    }
    // the pixel's property bit (OR-reduced per component)
    template <int MODE>
    __device__ __forceinline__ bool bit(uint8_t v, int x, int y) const {
        if (MODE == SEL_RBC) return (v & (HP_FLAG_RBC_HI | HP_FLAG_RBC_LO)) == (HP_FLAG_RBC_HI | HP_FLAG_RBC_LO);
        if (MODE == SEL_EDGE) return v == 2;  // a strong Canny candidate
        if (MODE == SEL_FILL) return x == 0 || y == 0 || x == w - 1 || y == h - 1;
        return false;
    }
    template <int MODE>
    __device__ __forceinline__ uint8_t out(uint8_t v, bool f, int32_t prop) const {
        if (MODE == SEL_AREA || MODE == SEL_AREA_TH) {
            const int a = prop & kAreaMask;
            return f && a >= amin && a <= amax;
        }
        if (MODE == SEL_RBC) return f && (prop & kHit) && (v & HP_FLAG_R_GT_B);
        if (MODE == SEL_EDGE) return f && (prop & kHit);  // hysteresis
        return f ? !(prop & kTouch) : 1;  // SEL_FILL: big0 | enclosed background
    }
};

// the output pass reads each pixel's local root from k_cs_local's lr plane, except for S2:
// its sparse RBC_LO components make re-running the tile's union-find cheaper than the 2 B/px
// plane (measured r2: k_cs_local<1> + k_cs_out<1> 42.5 -> 47.2 us per 4K tile with lr)
template <int MODE>
__host__ __device__ constexpr bool lr_mode() {
    return MODE != SEL_RBC;
}

template <int MODE>
__device__ __forceinline__ int32_t mode_bit() {
    return (MODE == SEL_RBC || MODE == SEL_EDGE) ? kHit : (MODE == SEL_FILL ? kTouch : 0);
}

__device__ __forceinline__ int find_l(const int* s, int x) {
    const volatile int* vs = s;
    int p = vs[x];
    while (p != x) {
        x = p;
        p = vs[x];
    }
    return x;
}
__device__ __forceinline__ void union_l(int* s, int a, int b) {
    while (true) {
        a = find_l(s, a);
        b = find_l(s, b);
        if (a == b) return;
        if (a < b) {
            int t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&s[a], a, b) == a) return;
    }
}
__device__ __forceinline__ int32_t find_c(int32_t* P, int32_t x) {
    while (true) {
        int32_t p = __ldcg(P + x);
        if (p == x) return x;
        int32_t gp = __ldcg(P + p);
        if (gp == p) return p;
        atomicCAS(&P[x], p, gp);
        x = gp;
    }
}
__device__ __forceinline__ void union_c(int32_t* P, int32_t a, int32_t b) {
    while (true) {
        a = find_c(P, a);
        b = find_c(P, b);
        if (a == b) return;
        if (a < b) {
            int32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&P[a], a, b) == a) return;
    }
}

// One 256-thread CTA per 32x32 tile; thread (lane = column, warp) owns rows warp + 8k, so a
// row is one warp: its ballot is the row's foreground mask, every pixel points at the start of
// its horizontal run, and only RUN STARTS union, once with each run of the row above that
// touches the run (8-conn: columns xs-1 .. xe+1, 4-conn: xs .. xe) -- one union per adjacent
// pair of runs.  Roots, areas, property bits and outputs are then handled once per run (the
// run start), shared with the run's pixels by a shuffle.  (Measured r1: a warp-per-tile
// variant with lane = column and 32 serial rows was 2x slower.)
struct TileSm {
    int s[kT * kT];
    int acc[kT * kT];
    unsigned rowm[kT];  // foreground mask of each row
    unsigned bitm[kT];  // property-bit mask of each row
    int nr;
};

__device__ __forceinline__ int run_start(unsigned fm, int lane) {
    const unsigned nl = ~(fm & (fm << 1)) & (0xffffffffu >> (31 - lane));
    return 31 - __clz(nl);
}
__device__ __forceinline__ int run_end(unsigned fm, int xs) {
    const unsigned tail = ~(fm >> xs);
    return tail == 0 ? 31 : xs + __ffs(tail) - 2;
}
__device__ __forceinline__ unsigned span(int lo, int hi) {  // bits lo..hi
    return (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
}

// loads + runs + unions; returns 0 (no foreground), 1 (general), 2 (all foreground)
__device__ __forceinline__ bool is_run_start(unsigned fm, int lane) {
    return ((fm >> lane) & 1) && !(lane > 0 && ((fm >> (lane - 1)) & 1));
}

// rows of a thread (lane = column in every pass): S5's word set-up gives warp w the tile rows
// 4w .. 4w + 3, the byte set-up the rows w + 8k
template <int MODE>
__device__ __forceinline__ int tile_row(int k) {
    return MODE == SEL_AREA_TH ? 4 * (int)(threadIdx.x >> 5) + k : (int)(threadIdx.x >> 5) + 8 * k;
}

template <int MODE>
__device__ __forceinline__ int tile_uf(const Sel& sel, int conn, int tx0, int ty0, TileSm& T, uint8_t (&v)[4],
                                       unsigned (&fms)[4], bool clear_acc, int (*bbs)[kT * kT] = nullptr) {
    const int lane = threadIdx.x & 31;
    const int w = sel.w, h = sel.h;
    int nfg = 0;
    unsigned bms[4];
    // phase 1: the row masks only (registers); an empty tile leaves after one vote without a
    // shared-memory write (S2's RBC_LO and S5's candidates leave most tiles empty)
    if constexpr (MODE != SEL_AREA_TH) {
        const int gx = tx0 + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int gy = ty0 + tile_row<MODE>(k);
            v[k] = (gx < w && gy < h) ? sel.load<MODE>((int64_t)gy * w + gx) : (uint8_t)0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int gy = ty0 + tile_row<MODE>(k);
            const bool f = gx < w && gy < h && sel.fg<MODE>(v[k]);
            fms[k] = __ballot_sync(0xffffffffu, f);
            bms[k] = __ballot_sync(0xffffffffu, f && sel.bit<MODE>(v[k], gx, gy));
            nfg += f;
        }
    } else {
        // S5 sets up a word per thread: its candidate is a function of three planes (g, recon, rbc),
        // so 3 word loads replace 12 byte loads (r2: k_cs_local<3> 67.4 -> 62.2 us per 4K tile; for
        // the one-plane passes the shuffles cost more than they save).  lane -> row 4 * warp +
        // (lane >> 3), pixels 4 * (lane & 7) .. + 3; the warp's four row masks by segmented ORs
        const int wc = 4 * (lane & 7);
        const int gyw = ty0 + tile_row<MODE>(lane >> 3), gxw = tx0 + wc;
        const uint32_t word = gyw < h ? sel.load4<MODE>(gyw, gxw) : 0u;
        unsigned xf = 0, xb = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint8_t vb = (uint8_t)(word >> (8 * b));
            const bool f = gyw < h && gxw + b < w && sel.fg<MODE>(vb);
            xf |= (unsigned)f << (wc + b);
            xb |= (unsigned)(f && sel.bit<MODE>(vb, gxw + b, gyw)) << (wc + b);
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            xf |= __shfl_xor_sync(0xffffffffu, xf, o);
            xb |= __shfl_xor_sync(0xffffffffu, xb, o);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            fms[k] = __shfl_sync(0xffffffffu, xf, 8 * k);
            bms[k] = __shfl_sync(0xffffffffu, xb, 8 * k);
            v[k] = 0;  // (read by the S2 output pass only)
            nfg += (fms[k] >> lane) & 1;
        }
    }
    if (!__syncthreads_or(nfg > 0)) return 0;
    const int all_fg = __syncthreads_and(nfg == 4);
    // phase 2: the tile's run pointers, masks and accumulators in shared memory
    if (threadIdx.x == 0) T.nr = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ly = tile_row<MODE>(k);
        const unsigned fm = fms[k];
        if (lane == 0) {
            T.rowm[ly] = fm;
            T.bitm[ly] = bms[k];
        }
        T.s[ly * kT + lane] = ((fm >> lane) & 1) ? ly * kT + run_start(fm, lane) : -1;
        if (clear_acc) T.acc[ly * kT + lane] = 0;
        if (bbs && is_run_start(fm, lane)) {  // S5's bounding boxes: only run starts can be roots
            const int li = ly * kT + lane;
            bbs[0][li] = INT_MAX;
            bbs[1][li] = INT_MAX;
            bbs[2][li] = -1;
            bbs[3][li] = -1;
        }
    }
    __syncthreads();
    if (all_fg) return 2;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ly = tile_row<MODE>(k);
        const unsigned fm = fms[k];
        if (ly == 0 || !((fm >> lane) & 1) || (lane > 0 && ((fm >> (lane - 1)) & 1))) continue;  // run starts
        const unsigned above = T.rowm[ly - 1];
        if (!above) continue;
        const int re = run_end(fm, lane);
        const int lo = conn == 8 ? max(lane - 1, 0) : lane, hi = conn == 8 ? min(re + 1, 31) : re;
        const unsigned ov = above & span(lo, hi);
        unsigned segs = ov & ~(ov << 1);  // first column of each touching run (within the range)
        const int li = ly * kT + lane;
        while (segs) {
            const int b = __ffs(segs) - 1;
            segs &= segs - 1;
            union_l(T.s, li, (ly - 1) * kT + b);
        }
    }
    __syncthreads();
    return 1;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_cs_local(Sel sel, int conn, int32_t* __restrict__ P, int32_t* __restrict__ X,
                                                  int32_t* __restrict__ E, int32_t* __restrict__ roots,
                                                  int32_t* __restrict__ nroots, uint16_t* __restrict__ lr,
                                                  uint8_t* __restrict__ kinds) {
    __shared__ TileSm T;
    constexpr bool BB = MODE == SEL_AREA_TH;  // bounding boxes per component
    __shared__ int bbs[BB ? 4 : 1][BB ? kT * kT : 1];
    if (sel.gate && *sel.gate == 0) return;
    const int tx0 = blockIdx.x * kT, ty0 = blockIdx.y * kT;
    const int t = blockIdx.y * gridDim.x + blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int w = sel.w, h = sel.h;
    uint8_t v[4];
    unsigned fms[4];
    // (tile_uf initialises the bounding boxes of the run starts, before its last barrier)
    int (*bbp)[kT * kT] = nullptr;
    if constexpr (BB) bbp = bbs;
    const int kind = tile_uf<MODE>(sel, conn, tx0, ty0, T, v, fms, true, bbp);
    int32_t* Et = E + (int64_t)t * 4 * kT;
    auto gidx = [&](int li) -> int32_t { return (int32_t)((int64_t)(ty0 + li / kT) * w + tx0 + li % kT); };
    if (threadIdx.x == 0) kinds[t] = (uint8_t)kind;
    if (kind == 0) {  // (its edge roots are not written: k_cs_merge reads the tile's kind first)
        if (threadIdx.x == 0) nroots[t] = 0;
        return;
    }
    if (kind == 2) {  // one component rooted at the tile origin
        const int32_t G = gidx(0);
        if (threadIdx.x < 4 * kT) Et[threadIdx.x] = G;
        if (threadIdx.x < 32) {
            const unsigned anyb = __any_sync(0xffffffffu, T.bitm[threadIdx.x] != 0);
            if (threadIdx.x == 0) {
                P[G] = G;
                X[G] = kT * kT | (anyb ? mode_bit<MODE>() : 0);
                if constexpr (BB) {
                    sel.bx0[G] = tx0;
                    sel.by0[G] = ty0;
                    sel.bx1[G] = tx0 + kT - 1;
                    sel.by1[G] = ty0 + kT - 1;
                }
                roots[(int64_t)t * kT * kT] = G;
                nroots[t] = 1;
            }
        }
        return;
    }
    // per run: area and property bit at the run's root; every pixel's local root to lr (the
    // output pass reads it instead of re-running the tile's union-find)
    int rk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ly = tile_row<MODE>(k);
        const unsigned fm = fms[k];
        rk[k] = 0;
        if (!is_run_start(fm, lane)) continue;
        const int re = run_end(fm, lane);
        const int r = find_l(T.s, ly * kT + lane);
        rk[k] = r;
        atomicAdd(&T.acc[r], re - lane + 1);
        if (T.bitm[ly] & span(lane, re)) atomicOr(&T.acc[r], mode_bit<MODE>());
        if constexpr (BB) {
            atomicMin(&bbs[0][r], tx0 + lane);
            atomicMin(&bbs[1][r], ty0 + ly);
            atomicMax(&bbs[2][r], tx0 + re);
            atomicMax(&bbs[3][r], ty0 + ly);
        }
    }
#pragma unroll
    for (int k = 0; k < 4 && lr_mode<MODE>(); ++k) {
        const int ly = tile_row<MODE>(k);
        const unsigned fm = fms[k];
        const bool f = (fm >> lane) & 1;
        const int r = __shfl_sync(0xffffffffu, rk[k], f ? run_start(fm, lane) : lane);
        const int gx = tx0 + lane, gy = ty0 + ly;
        if (gx < w && gy < h) lr[(int64_t)gy * w + gx] = f ? (uint16_t)r : (uint16_t)0xffff;
    }
    __syncthreads();
    // roots: run starts that are their own parent
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ly = tile_row<MODE>(k);
        const int li = ly * kT + lane;
        if (T.s[li] == li) {
            const int32_t G = gidx(li);
            P[G] = G;
            X[G] = T.acc[li];
            if constexpr (BB) {
                sel.bx0[G] = bbs[0][li];
                sel.by0[G] = bbs[1][li];
                sel.bx1[G] = bbs[2][li];
                sel.by1[G] = bbs[3][li];
            }
            roots[(int64_t)t * kT * kT + atomicAdd(&T.nr, 1)] = G;
        }
    }
    // tile-edge roots: side 0 top row, 1 bottom row, 2 left column, 3 right column
    if (threadIdx.x < 4 * kT) {
        const int side = threadIdx.x >> 5;
        const int lxx = side < 2 ? lane : (side == 2 ? 0 : kT - 1);
        const int lyy = side < 2 ? (side == 0 ? 0 : kT - 1) : lane;
        const int li = lyy * kT + lxx;
        int32_t e = -1;
        if (tx0 + lxx < w && ty0 + lyy < h && T.s[li] >= 0) e = gidx(find_l(T.s, li));
        Et[threadIdx.x] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) nroots[t] = T.nr;
}

// cross-tile unions, one warp per (tile, side): the tile's top row against the bottom row of
// the tile above, its left column against the right column of the tile on the left.  Edge
// pixels of one run (consecutive foreground along the edge) share a local root, so only run
// starts union, once with each touching run across the edge (8-conn: positions i0-1 .. i1+1,
// which also covers every right-column diagonal; 4-conn: i0 .. i1); the 8-conn corner
// diagonals (up-left of (0,0), up-right of (31,0)) are taken by the top row's end lanes.
__global__ void __launch_bounds__(256) k_cs_merge(int conn, int ntx, int nty, const int32_t* __restrict__ E,
                                                  int32_t* __restrict__ P, const int32_t* __restrict__ gate,
                                                  const uint8_t* __restrict__ kinds) {
    if (gate && *gate == 0) return;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gt >= (int64_t)ntx * nty * 2 * kT) return;  // (whole warps: 2 * kT per tile)
    const int t = (int)(gt / (2 * kT)), j = (int)(gt % (2 * kT));
    if (__ldg(kinds + t) == 0) return;  // an empty tile has no edge roots (whole warps)
    const int bx = t % ntx, by = t / ntx;
    const int side = j >> 5, i = j & 31;
    auto e = [&](int tx, int ty, int sd, int k) -> int32_t {
        if (tx < 0 || ty < 0 || tx >= ntx || ty >= nty) return -1;
        const int64_t tt = (int64_t)ty * ntx + tx;
        if (__ldg(kinds + tt) == 0) return -1;
        return __ldg(E + tt * 4 * kT + sd * kT + k);
    };
    const int ntxb = side == 0 ? bx : bx - 1, ntyb = side == 0 ? by - 1 : by;  // tile across the edge
    const int nside = side == 0 ? 1 : 3;                                       // its bottom row / right column
    const int32_t me = e(bx, by, side == 0 ? 0 : 2, i);
    const int32_t q = e(ntxb, ntyb, nside, i);
    const unsigned mine = __ballot_sync(0xffffffffu, me >= 0);
    const unsigned other = __ballot_sync(0xffffffffu, q >= 0);
    if (me < 0) return;
    if (other && ((mine >> i) & 1) && !(i > 0 && ((mine >> (i - 1)) & 1))) {  // run start
        const unsigned tail = ~(mine >> i);
        const int re = tail == 0 ? 31 : i + __ffs(tail) - 2;
        const int lo = conn == 8 ? max(i - 1, 0) : i, hi = conn == 8 ? min(re + 1, 31) : re;
        const unsigned ov = other & span(lo, hi);
        unsigned segs = ov & ~(ov << 1);
        while (segs) {
            const int b = __ffs(segs) - 1;
            segs &= segs - 1;
            union_c(P, me, e(ntxb, ntyb, nside, b));
        }
    }
    if (conn == 8 && side == 0 && (i == 0 || i == kT - 1)) {
        const int32_t d = i == 0 ? e(bx - 1, by - 1, 1, kT - 1) : e(bx + 1, by - 1, 1, 0);
        if (d >= 0) union_c(P, me, d);
    }
}

// one warp per tile
__global__ void __launch_bounds__(256) k_cs_accum(int ntiles, const int32_t* __restrict__ roots,
                                                  const int32_t* __restrict__ nroots, int32_t* __restrict__ P,
                                                  int32_t* __restrict__ X, Sel sel) {
    if (sel.gate && *sel.gate == 0) return;
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t < ntiles) {
        const int n = nroots[t];
        for (int k = threadIdx.x & 31; k < n; k += 32) {
            const int32_t G = roots[(int64_t)t * kT * kT + k];
            const int32_t R = find_c(P, G);
            if (R == G) continue;
            const int32_t x = X[G];
            atomicAdd(&X[R], x & kAreaMask);
            if (x & ~kAreaMask) atomicOr(&X[R], x & ~kAreaMask);
            if (sel.bx0) {
                atomicMin(&sel.bx0[R], sel.bx0[G]);
                atomicMin(&sel.by0[R], sel.by0[G]);
                atomicMax(&sel.bx1[R], sel.bx1[G]);
                atomicMax(&sel.by1[R], sel.by1[G]);
            }
            P[G] = R;
        }
    }
}

// every mode but SEL_FILL outputs 0 on a tile without foreground: the caller zeroes the plane
// and such tiles skip the pass.  A streaming pass: each pixel's local root from lr (written by
// k_cs_local), the property word of its global root looked up once per run (r1-r2 re-ran the
// tile's union-find here: 30-34 us per 4K tile, latency-bound on the shared-memory finds).
template <int MODE>
__global__ void __launch_bounds__(256) k_cs_out(Sel sel, int conn, const int32_t* __restrict__ P,
                                                const int32_t* __restrict__ X,
                                                uint8_t* __restrict__ out, const uint16_t* __restrict__ lr,
                                                const uint8_t* __restrict__ kinds) {
    if (sel.gate && *sel.gate == 0) return;
    const int kind = kinds[blockIdx.y * gridDim.x + blockIdx.x];
    if (MODE != SEL_FILL && kind == 0) return;
    const int tx0 = blockIdx.x * kT, ty0 = blockIdx.y * kT;
    const int lane = threadIdx.x & 31;
    const int w = sel.w, h = sel.h;
    const int gx = tx0 + lane;
    if constexpr (!lr_mode<MODE>()) {
        __shared__ TileSm T;
        uint8_t v[4];
        unsigned fms[4];
        const int kd = tile_uf<MODE>(sel, conn, tx0, ty0, T, v, fms, false);
        int32_t prop0 = 0;
        if (kd == 2) prop0 = __ldg(X + __ldg(P + (int32_t)((int64_t)ty0 * w + tx0)));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ly = tile_row<MODE>(k);
            const int gy = ty0 + ly;
            const unsigned fm = fms[k];
            const bool f = (fm >> lane) & 1;
            int32_t prop = prop0;
            if (kd == 1) {
                const int st = f ? run_start(fm, lane) : lane;
                int32_t pr = 0;
                if (f && st == lane) {
                    const int r = find_l(T.s, ly * kT + lane);
                    pr = __ldg(X + __ldg(P + (int32_t)((int64_t)(ty0 + r / kT) * w + tx0 + r % kT)));
                }
                prop = __shfl_sync(0xffffffffu, pr, st);
            }
            if (gx < w && gy < h) out[(int64_t)gy * w + gx] = sel.out<MODE>(v[k], f, prop);
        }
        return;
    }
    // the four rows' loads and the run lookups are issued as independent batches (three
    // dependent L2 round trips per thread instead of twelve)
    int l[4], st[4];
    uint8_t v[4];
    bool in[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int gy = ty0 + (threadIdx.x >> 5) + 8 * k;
        in[k] = gx < w && gy < h;
        const int64_t p = (int64_t)gy * w + gx;
        l[k] = (kind == 1 && in[k]) ? (int)__ldg(lr + p) : 0xffff;
        v[k] = (MODE == SEL_RBC && in[k]) ? __ldg(sel.plane + p) : (uint8_t)0;
    }
    int32_t q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool f = l[k] != 0xffff;
        const unsigned fm = __ballot_sync(0xffffffffu, f);
        st[k] = f ? run_start(fm, lane) : lane;
        q[k] = (f && st[k] == lane) ? __ldg(P + (int32_t)((int64_t)(ty0 + l[k] / kT) * w + tx0 + l[k] % kT)) : -1;
    }
    if (kind == 2) q[0] = __ldg(P + (int32_t)((int64_t)ty0 * w + tx0));
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = q[k] >= 0 ? __ldg(X + q[k]) : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int gy = ty0 + (threadIdx.x >> 5) + 8 * k;
        bool f;
        int32_t prop;
        if (kind == 2) {  // an all-foreground tile lies inside the image
            f = true;
            prop = q[0];
        } else {
            f = l[k] != 0xffff;
            prop = __shfl_sync(0xffffffffu, q[k], st[k]);
        }
        if (in[k]) out[(int64_t)gy * w + gx] = sel.out<MODE>(v[k], f, prop);
    }
}

// the global roots of the components that pass the area filter, with their bounding boxes
// (one warp per tile, over the tile's local roots: a local root is a global root iff P[G] == G)
__global__ void __launch_bounds__(256) k_cs_list(int ntiles, const int32_t* __restrict__ roots,
                                                 const int32_t* __restrict__ nroots, const int32_t* __restrict__ P,
                                                 const int32_t* __restrict__ X, Sel sel, int32_t* __restrict__ out_root,
                                                 int4* __restrict__ out_bbox, int32_t* __restrict__ out_area,
                                                 int32_t* __restrict__ count, int32_t cap) {
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t >= ntiles) return;
    const int n = nroots[t];
    for (int k = threadIdx.x & 31; k < n; k += 32) {
        const int32_t G = roots[(int64_t)t * kT * kT + k];
        if (P[G] != G) continue;
        const int a = X[G] & kAreaMask;
        if (a < sel.amin || a > sel.amax) continue;
        const int i = atomicAdd(count, 1);
        if (i < cap) {
            out_root[i] = G;
            out_bbox[i] = make_int4(sel.bx0[G], sel.by0[G], sel.bx1[G], sel.by1[G]);
            out_area[i] = a;
        }
    }
}

struct ListOut {
    int32_t* root = nullptr;
    int4* bbox = nullptr;
    int32_t* area = nullptr;
    int32_t* count = nullptr;  // zeroed by the caller
    int32_t cap = 0;
};

template <int MODE>
void run_select(Sel sel, int conn, Slot& sl, uint8_t* out, cudaStream_t s, const ListOut* lo = nullptr) {
    const int w = sel.w, h = sel.h;
    if ((int64_t)w * h == 0) return;
    const int ntx = (w + kT - 1) / kT, nty = (h + kT - 1) / kT;
    const int ntiles = ntx * nty;
    dim3 grid(ntx, nty);
    int32_t* P = sel.P ? sel.P : sl.lab;
    int32_t* X = sel.X ? sel.X : sl.aux;
    (note_launch(), k_cs_local<MODE><<<grid, 256, 0, s>>>(sel, conn, P, X, sl.cs_edge, sl.cs_roots, sl.cs_nroots,
                                                           sl.cs_lr, sl.cs_kind));
    (note_launch(), k_cs_merge<<<(int)(((int64_t)ntiles * 2 * kT + 255) / 256), 256, 0, s>>>(
                        conn, ntx, nty, sl.cs_edge, P, sel.gate, sl.cs_kind));
    (note_launch(), k_cs_accum<<<(ntiles + 7) / 8, 256, 0, s>>>(ntiles, sl.cs_roots, sl.cs_nroots, P, X, sel));
    if (out) {
        if (MODE != SEL_FILL) cudaMemsetAsync(out, 0, (size_t)w * h, s);
        (note_launch(), k_cs_out<MODE><<<grid, 256, 0, s>>>(sel, conn, P, X, out, sl.cs_lr, sl.cs_kind));
    }
    if (lo)
        (note_launch(), k_cs_list<<<(ntiles + 7) / 8, 256, 0, s>>>(ntiles, sl.cs_roots, sl.cs_nroots, P, X, sel,
                                                                   lo->root, lo->bbox, lo->area, lo->count, lo->cap));
}

// ---------------------------------------------------------------- feature-stage Canny
// cv2.Canny(g, low, high), aperture 3, L1 norm (reading C22): 3x3 Sobel
// with replicated borders, m = |dx| + |dy|, non-maximum suppression in the gradient sector
// (tan(22.5 deg) in 15-bit fixed point; out-of-tile magnitudes 0); map = 2 for local maxima
// with m > high, 1 for other local maxima with m > low, else 0.  The hysteresis (8-connected
// components of the candidates that hold a strong one) is the CCL-select SEL_EDGE.
// 64 x 32 output tile, 256 threads, 4 horizontally adjacent pixels per thread: g staged as
// 32-bit words (2-px replicated halo).  The Sobel pair of 4 pixels runs on 16-bit lanes
// (pixels (0,2) in one register, (1,3) in another): column sums t + 2c + b and biased
// differences b - t + 255 of the six columns -1..4, |dx| and |dy| as max - min on the native
// VIMNMX.U16x2, so a group of 4 pixels costs ~50 instructions instead of ~200 (r2 ncu: the
// scalar version issued 34 M of the kernel's 50 M warp instructions here).  Shared memory
// keeps m = |dx| + |dy| and the biased dx, dy (int16 planes); the gradient sector is computed
// in the suppression step only for pixels with m > low.
constexpr int kNW = 64, kNH = 32;
constexpr int kGWW = kNW / 4 + 2;  // Sobel groups per row: pixels [x0 - 4, x0 + kNW + 4)
constexpr int kSW = kNW / 4 + 8;   // staged g words per row: pixels [x0 - 16, x0 + kNW + 16), 16-B aligned
constexpr int kGR = kNH + 4;       // staged g rows: [y0 - 2, y0 + kNH + 2)
constexpr int kMW = kNW + 8;       // magnitude columns [x0 - 4, x0 + kNW + 4) (x0-1 .. x0+kNW used)
constexpr int kMR = kNH + 2;       // magnitude rows [y0 - 1, y0 + kNH]
constexpr uint32_t kDxBias = 0x04000400u;  // dx + 1024 per lane (|dx| <= 1020)
constexpr int kDyBias = 1020;              // dy' = sum of (b - t + 255) with weights 1, 2, 1

__device__ __forceinline__ uint32_t g_word(const uint8_t* __restrict__ g, int w, int h, int gx0, int gy,
                                           bool aligned) {
    gy = min(max(gy, 0), h - 1);
    const uint8_t* row = g + (int64_t)gy * w;
    if (aligned && gx0 >= 0 && gx0 + 3 < w) return __ldg(reinterpret_cast<const unsigned int*>(row + gx0));
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) v |= (uint32_t)__ldg(row + min(max(gx0 + b, 0), w - 1)) << (8 * b);
    return v;
}

// the four u16x2 column pairs (-1,1), (0,2), (1,3), (2,4) of pixels 0..3 (word B) with the
// last byte of A on the left and the first byte of C on the right
__device__ __forceinline__ void col_pairs(uint32_t A, uint32_t B, uint32_t C, uint32_t (&e)[4]) {
    e[1] = __byte_perm(B, 0, 0x4240);     // (b0, b2)
    e[2] = __byte_perm(B, 0, 0x4341);     // (b1, b3)
    e[0] = __byte_perm(e[2], A, 0x1017);  // (a3, b1)
    e[3] = __byte_perm(e[1], C, 0x1432);  // (b2, c0)
}

__device__ __forceinline__ uint32_t absdiff2(uint32_t a, uint32_t b) { return __vmaxu2(a, b) - __vminu2(a, b); }

__global__ void __launch_bounds__(256) k_canny_nms(const uint8_t* __restrict__ g, int w, int h, int low, int high,
                                                   uint8_t* __restrict__ map) {
    __shared__ __align__(16) uint32_t sg[kGR][kSW];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ __align__(8) uint16_t sm[kMR][kMW];
    __shared__ __align__(8) uint16_t sdx[kMR][kMW];
    __shared__ __align__(8) uint16_t sdy[kMR][kMW];
    const int x0 = blockIdx.x * kNW, y0 = blockIdx.y * kNH;
    const bool aligned = (w & 3) == 0 && (((uintptr_t)g) & 3) == 0;
    // Stage the rows [y0 - 2, y0 + kNH + 2) (clamped: replicated borders).  Interior tiles of a
    // 16-B-aligned plane: one bulk async copy (cp.async.bulk, the TMA engine) per 96-byte row,
    // completing on an mbarrier -- no load / store instructions on the SMs (r2: the word loop
    // issued a quarter of the kernel's instructions).  Tiles at the left / right edge replicate
    // columns, so they keep the per-word loop.
    const bool bulk = (w & 15) == 0 && (((uintptr_t)g) & 15) == 0 && x0 >= 16 && x0 + kNW + 16 <= w;
    if (bulk) {
        const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(kGR * kSW * 4)
                             : "memory");
            __syncwarp();
            for (int r = threadIdx.x; r < kGR; r += 32) {
                const int gy = min(max(y0 - 2 + r, 0), h - 1);
                const uint8_t* src = g + (int64_t)gy * w + x0 - 16;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        (uint32_t)__cvta_generic_to_shared(&sg[r][0])),
                    "l"(src), "r"(kSW * 4), "r"(ba)
                    : "memory");
            }
        }
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(ba)
                : "memory");
    } else {
        for (int i = threadIdx.x; i < kGR * kSW; i += blockDim.x) {
            const int r = i / kSW, q = i - r * kSW;
            sg[r][q] = g_word(g, w, h, x0 - 16 + 4 * q, y0 - 2 + r, aligned);
        }
        __syncthreads();
    }
    // Sobel of pixel groups (row gy = y0 - 1 + r, pixels x0 - 4 + 4q + k, k = 0..3)
    for (int i = threadIdx.x; i < kMR * kGWW; i += blockDim.x) {
        const int r = i / kGWW, q = i - r * kGWW;
        const int qs = q + 3;  // staged word of group q (pixels x0 - 4 + 4q)
        uint32_t t[4], c[4], b[4];
        col_pairs(sg[r][qs - 1], sg[r][qs], sg[r][qs + 1], t);
        col_pairs(sg[r + 1][qs - 1], sg[r + 1][qs], sg[r + 1][qs + 1], c);
        col_pairs(sg[r + 2][qs - 1], sg[r + 2][qs], sg[r + 2][qs + 1], b);
        uint32_t S[4], D[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            S[j] = t[j] + 2 * c[j] + b[j];      // <= 1020 per lane
            D[j] = b[j] + 0x00ff00ffu - t[j];   // b - t + 255 in [0, 510] per lane
        }
        // lane pairs: E = pixels (0,2), O = pixels (1,3)
        const uint32_t dxE = S[2] + kDxBias - S[0], dxO = S[3] + kDxBias - S[1];
        const uint32_t dyE = D[0] + 2 * D[1] + D[2], dyO = D[1] + 2 * D[2] + D[3];
        const uint32_t bias = (uint32_t)kDyBias * 0x00010001u;
        uint32_t mE = absdiff2(S[2], S[0]) + absdiff2(dyE, bias);
        uint32_t mO = absdiff2(S[3], S[1]) + absdiff2(dyO, bias);
        uint32_t mlo = __byte_perm(mE, mO, 0x5410), mhi = __byte_perm(mE, mO, 0x7632);
        const int gy = y0 - 1 + r, gxa = x0 - 4 + 4 * q;
        if (gy < 0 || gy >= h) {
            mlo = mhi = 0;
        } else if (gxa < 0 || gxa + 3 >= w) {  // out-of-tile magnitudes 0
            uint32_t klo = 0, khi = 0;
            if (gxa + 0 >= 0 && gxa + 0 < w) klo |= 0x0000ffffu;
            if (gxa + 1 >= 0 && gxa + 1 < w) klo |= 0xffff0000u;
            if (gxa + 2 >= 0 && gxa + 2 < w) khi |= 0x0000ffffu;
            if (gxa + 3 >= 0 && gxa + 3 < w) khi |= 0xffff0000u;
            mlo &= klo;
            mhi &= khi;
        }
        *reinterpret_cast<uint2*>(&sm[r][4 * q]) = make_uint2(mlo, mhi);
        *reinterpret_cast<uint2*>(&sdx[r][4 * q]) =
            make_uint2(__byte_perm(dxE, dxO, 0x5410), __byte_perm(dxE, dxO, 0x7632));
        *reinterpret_cast<uint2*>(&sdy[r][4 * q]) =
            make_uint2(__byte_perm(dyE, dyO, 0x5410), __byte_perm(dyE, dyO, 0x7632));
    }
    __syncthreads();
    // suppression: thread -> 4 pixels of 2 rows; sector 0: left/right, 1: up/down, 2: up-right
    // and down-left, 3: up-left and down-right (">" toward -x / -y, ">=" toward +x / +y).  The
    // sector from the pixel's dx, dy: tan(22.5 deg) in 15-bit fixed point, as cv2.Canny.
    const int cg = threadIdx.x & 15, rg = threadIdx.x >> 4;
    const int gx0 = x0 + 4 * cg;
    const uint16_t* M = &sm[0][0];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int oy = 2 * rg + rr, gy = y0 + oy;
        if (gy >= h) continue;
        const int r = oy + 1;  // sm row of the pixel
        const int c0 = 4 + 4 * cg;  // sm column of pixel 0
        uint32_t out = 0;
        const uint2 mw = *reinterpret_cast<const uint2*>(&sm[r][c0]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int m = (int)(((k < 2 ? mw.x : mw.y) >> (16 * (k & 1))) & 0xffff);
            if (m <= low) continue;
            const int c = c0 + k;
            const int dx = (int)sdx[r][c] - 1024, dy = (int)sdy[r][c] - kDyBias;
            const int ax = abs(dx), ay = abs(dy) << 15;  // |dy| <= 1020: fits in 32 bits
            const int tg22x = ax * 13573, tg67x = tg22x + (ax << 16);
            const int sc = ay < tg22x ? 0 : (ay > tg67x ? 1 : (((dx ^ dy) < 0) ? 2 : 3));
            const int o = sc == 0 ? -1 : (sc == 1 ? -kMW : (sc == 2 ? 1 - kMW : -1 - kMW));
            const int i = r * kMW + c;
            const int ma = M[i + o], mb = M[i - o];
            const bool lm = m > ma && (sc < 2 ? m >= mb : m > mb);
            if (lm) out |= (m > high ? 2u : 1u) << (8 * k);
        }
        uint8_t* o = map + (int64_t)gy * w + gx0;
        if (gx0 + 3 < w && (((uintptr_t)o) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(o) = out;
        } else {
            for (int k = 0; k < 4 && gx0 + k < w; ++k) o[k] = (uint8_t)(out >> (8 * k));
        }
    }
}

}  // namespace

// Canny edges (0/1) of g.  Scratch: the slot's pmask (candidate map), the sparse planes ML / d
// and the CCL-select arrays -- free from S6 on, so the pipeline runs it beside S7-S11.
void launch_canny(const uint8_t* g, int w, int h, int low, int high, Slot& sl, uint8_t* edges, cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    dim3 grid((w + kNW - 1) / kNW, (h + kNH - 1) / kNH);
    (note_launch(), k_canny_nms<<<grid, 256, 0, s>>>(g, w, h, low, high, sl.pmask));
    Sel sel{sl.pmask, w, h, 0, 0};
    sel.P = sl.ML;
    sel.X = sl.d;
    run_select<SEL_EDGE>(sel, 8, sl, edges, s);
}

void launch_rbc(const uint8_t* flags, int w, int h, Slot& sl, uint8_t* rbc, cudaStream_t s) {
    run_select<SEL_RBC>(Sel{flags, w, h, 0, 0}, 8, sl, rbc, s);
}

void launch_area_select(const uint8_t* cand, int w, int h, int amin, int amax, Slot& sl, uint8_t* out,
                        cudaStream_t s) {
    run_select<SEL_AREA>(Sel{cand, w, h, amin, amax}, 8, sl, out, s);
}

// S5 on the top-hat candidates, also listing the kept components (root, bounding box) into
// sl.sc_root / sl.sc_bbox with their count at *count (zeroed here); the sparse bounding-box
// planes borrow the slot's global-path planes ML, d, L, J.
void launch_area_select_tophat(const uint8_t* g, const uint8_t* R, const uint8_t* rbc, int g1, int w, int h,
                               int amin, int amax, Slot& sl, uint8_t* out, int32_t* count, cudaStream_t s) {
    Sel sel{g, w, h, amin, amax};
    sel.R = R;
    sel.rbc = rbc;
    sel.g1 = g1;
    sel.bx0 = sl.ML;
    sel.by0 = sl.d;
    sel.bx1 = sl.L;
    sel.by1 = reinterpret_cast<int32_t*>(sl.J);
    cudaMemsetAsync(count, 0, sizeof(int32_t), s);
    ListOut lo;
    lo.root = sl.sc_root;
    lo.bbox = sl.sc_bbox;
    lo.area = sl.sc_area;
    lo.count = count;
    lo.cap = sl.comp_cap;
    run_select<SEL_AREA_TH>(sel, 8, sl, out, s, &lo);
}

void launch_fill_holes(const uint8_t* big0, int w, int h, Slot& sl, uint8_t* F, cudaStream_t s,
                       const int32_t* gate) {
    Sel sel{big0, w, h, 0, 0};
    sel.gate = gate;
    run_select<SEL_FILL>(sel, 4, sl, F, s);
}

}  // namespace hp
