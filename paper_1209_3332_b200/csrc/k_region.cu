// k_region.cu -- IWPP morphological reconstruction on u8 planes at REGION granularity
// (S4 ReconToNuclei; HP_STAGE_IWPP_RAW).
//
// Measured (tools/diag_iwpp.py, r1): with one warp per 32x32 tile job, the reconstruction of
// some tiles is dominated by long sequential chains of tile jobs, i.e. by the cost of one hop
// through the global queue.  Here one CTA of RX*RY warps owns a region of RX x RY sub-tiles
// of 64 x 32 px (256 x 128 px): the region window (plus halo) lives in shared memory as bytes; each warp
// closes its own 32x32 sub-tile with row-scan sweeps (reading its neighbours' pixels live),
// then pushes the rows of neighbouring sub-tiles its changed border pixels can improve into
// their shared-memory dirty masks.  The warps run asynchronously (no CTA barrier per
// iteration); a token count of dirty masks plus in-flight sweeps detects the region's fixed
// point.  Between regions: the asynchronous worklist (ticket queue, IDLE/QUEUED/BUSY/
// BUSY_DIRTY states, per-sub-tile incoming rows).  Every update is a valid monotone
// propagation: the fixed point equals the oracle's.
#include <cstdlib>

#include "hp_internal.cuh"

namespace hp {
namespace {

constexpr uint32_t ST_IDLE = 0, ST_QUEUED = 1, ST_BUSY = 2, ST_DIRTY = 3;
constexpr int32_t EMPTY = -1;
constexpr unsigned FULL = 0xffffffffu;
#ifndef HP_RX
// 4 x 4 sub-tiles.  Measured (r1, config-2 tiles, 32 px sub-tiles): 8x4 sub-tiles close one
// tile faster alone (0.91 vs 1.04 ms) but a 1024-thread CTA fills the SM's register file, so
// tiles of the other slots cannot co-run: 301 vs 395 tiles/s in bench.py at 4 slots -- hence
// wider sub-tiles (HP_PPL pixels per lane) rather than more warps.
#define HP_RX 4
#define HP_RY 4
#endif
#ifndef HP_RG_MINB
#define HP_RG_MINB 2  // launch-bounds min blocks: 2 -> <= 64 registers per thread
#endif
#ifndef HP_RG_ORDER
#define HP_RG_ORDER 3  // initial job order: 0 raster, 1 four-colour (r1: 3018 -> 2165 jobs, 689 -> 725 tiles/s),
                       // 2 colour then highest marker, 3 highest marker then colour (2165 -> 1870
                       // jobs, 858 -> 870 tiles/s), 4 mean marker then colour, 5 region-grid distance
                       // to the top-marker regions (S4 alone 0.76 -> 0.72 ms but bench 871 -> 826)
#endif
#ifndef HP_RG_PROFILE
#define HP_RG_PROFILE 0  // timing breakdown in the stats (experiments)
#endif
#ifndef HP_RG_FIRSTORDER
#define HP_RG_FIRSTORDER 0  // first jobs: release sub-tile rows top to bottom
#endif
#ifndef HP_RG_JACOBI
#define HP_RG_JACOBI 0  // neighbour-exchange steps tried before the row scans
#endif
#ifndef HP_RG_EAGER
#define HP_RG_EAGER 0  // eager in-region pushes of border changes (r1: 88.9 -> 106.6 ms owned, 727 -> 688 tiles/s: off)
#endif
#ifndef HP_RG_WAITERS
#define HP_RG_WAITERS 4
#endif
#ifndef HP_RG_MIN_ALIVE
#define HP_RG_MIN_ALIVE 4  // r2, 55 CTAs x 12 tiles in flight: 16 -> 4 idle CTAs kept, bench 974-984 -> 1003-1011
#endif
#ifndef HP_POLL_NS
#define HP_POLL_NS 200       // idle sub-tile warps back off (frees issue slots for co-running work)
#endif
#ifndef HP_POLL_MAX_NS
#define HP_POLL_MAX_NS 800   // back-off cap (r1: 400-6400 within noise in bench.py; r2, two boxes,
                             // alternating: 200/800 ns S4 0.79 -> 0.78 ms and bench +0.5% over
                             // 400/1600; 1000/8000 S4 0.87 ms, bench -1.5%; 100/400 and 200/400 no better)
#endif
#ifndef HP_RG_PACKSCAN
#define HP_RG_PACKSCAN 0  // both scan directions at once on packed u16x2 clamps (r1: S4 0.78 -> 0.82 ms, bench 843 -> 834: off)
#endif
#ifndef HP_RG_ADI
#define HP_RG_ADI 0  // alternating-direction (row / column phase) region closure instead of sub-tile sweeps
#endif
#ifndef HP_RG_THIN
#define HP_RG_THIN 4096  // jobs with at most this many dirty sub-tile rows use the alternating-phase closure
#endif
#ifndef HP_RG_CHAIN
#define HP_RG_CHAIN 8  // ... and only from a region's HP_RG_CHAIN-th job on (a long chain).  r2: config 5
                       // serpentine 787 -> 422 ms, spiral 2348 -> 841 ms; config 2 and bench unchanged
#endif
#ifndef HP_RG_FIRSTROW
#define HP_RG_FIRSTROW 0  // first jobs: a full-width row pass before the sub-tile sweeps
#endif
#ifndef HP_RG_INIT
#define HP_RG_INIT 0  // raster + anti-raster initialisation sweep per region before the queue engine
#endif
#ifndef HP_PPL
#define HP_PPL 2  // pixels per lane: sub-tiles of 64 x 32 px, regions of 256 x 128 px
#endif
constexpr int RX = HP_RX, RY = HP_RY, NW = RX * RY;
constexpr int PPL = HP_PPL;            // pixels per lane in a sub-tile row
constexpr int SW = 32 * PPL;           // sub-tile width (px); sub-tile height is kTile = 32
constexpr int RWW = RX * SW / 4 + 2;   // window words per row: bytes [X0-4, X0+RX*SW+4)
constexpr int RWB = RWW * 4;         // window bytes per row
constexpr int ROWS = RY * kTile + 2; // window rows

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ void q_push(const Worklist& wl, int32_t t) {
    unsigned long long pos = atomicAdd(&wl.ctr[1], 1ull);
    int slot = (int)(pos % (unsigned long long)wl.cap);
    while (atomicCAS(&wl.queue[slot], EMPTY, t) != EMPTY) __nanosleep(64);
}

__device__ __forceinline__ int32_t q_pop(const Worklist& wl) {
    const unsigned long long h = atomicAdd(&wl.ctr[0], 1ull);
    const int slot = (int)(h % (unsigned long long)wl.cap);
    int ns = 32;
    while (true) {
        if (*reinterpret_cast<volatile int32_t*>(&wl.queue[slot]) != EMPTY) {
            int32_t v = atomicExch(&wl.queue[slot], EMPTY);
            if (v != EMPTY) return v;
        }
        if (vload(&wl.ctr[2]) == 0ull) return -1;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

__device__ __forceinline__ void q_activate(const Worklist& wl, int32_t t) {
    uint32_t s = *reinterpret_cast<volatile uint32_t*>(&wl.state[t]);
    while (true) {
        if (s == ST_IDLE) {
            uint32_t o = atomicCAS(&wl.state[t], ST_IDLE, ST_QUEUED);
            if (o == ST_IDLE) {
                atomicAdd(&wl.ctr[2], 1ull);
                q_push(wl, t);
                return;
            }
            s = o;
        } else if (s == ST_BUSY) {
            uint32_t o = atomicCAS(&wl.state[t], ST_BUSY, ST_DIRTY);
            if (o == ST_BUSY) return;
            s = o;
        } else {
            return;
        }
    }
}

template <bool LR>
__device__ __forceinline__ int clamp_scan(int lo, int hi, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int lo_o = LR ? __shfl_up_sync(FULL, lo, off) : __shfl_down_sync(FULL, lo, off);
        int hi_o = LR ? __shfl_up_sync(FULL, hi, off) : __shfl_down_sync(FULL, hi, off);
        bool take = LR ? lane >= off : lane + off < 32;
        int nlo = min(hi, max(lo, lo_o)), nhi = min(hi, max(lo, hi_o));
        lo = take ? nlo : lo;
        hi = take ? nhi : hi;
    }
    return lo;
}

// Both directions at once with each clamp (lo, hi) packed as u16x2: per level one shuffle per
// direction instead of two, the composition on the native VIMNMX.U16x2, and the two
// directions' shuffle latencies overlapped.  F scans left -> right, B right -> left.
#if HP_RG_PACKSCAN
__device__ __forceinline__ void clamp_scan_both(uint32_t& F, uint32_t& B, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t fo = __shfl_up_sync(FULL, F, off);
        const uint32_t bo = __shfl_down_sync(FULL, B, off);
        // this o other: (min(hi, max(lo, lo_o)), min(hi, max(lo, hi_o)))
        const uint32_t fn = __vminu2(__vmaxu2(fo, __byte_perm(F, 0, 0x1010)), __byte_perm(F, 0, 0x3232));
        const uint32_t bn = __vminu2(__vmaxu2(bo, __byte_perm(B, 0, 0x1010)), __byte_perm(B, 0, 0x3232));
        if (lane >= off) F = fn;
        if (lane + off < 32) B = bn;
    }
}
#endif

__device__ __forceinline__ uint32_t load_word(const uint8_t* plane, int w, int h, int gx, int gy) {
    if (gy < 0 || gy >= h) return 0u;
    const uint8_t* rowp = plane + (int64_t)gy * w;
    if (gx >= 0 && gx + 3 < w && (((uintptr_t)(rowp + gx)) & 3) == 0)
        return __ldcg(reinterpret_cast<const unsigned int*>(rowp + gx));
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        int x = gx + b;
        if (x >= 0 && x < w) v |= (uint32_t)__ldcg(reinterpret_cast<const unsigned char*>(rowp + x)) << (8 * b);
    }
    return v;
}

// byte of window pixel (wr, wc): window column wc (0 .. RX*32+1) is byte wc + 3
__device__ __forceinline__ int bidx(int wr, int wc) { return wr * RWB + wc + 3; }

constexpr int PXL = RX * SW / 32;  // pixels per lane across a region row

__device__ __forceinline__ void row_io_load(const uint8_t* __restrict__ p, int w, int h, int x0, int y, int* v) {
#pragma unroll
    for (int j = 0; j < PXL; ++j) v[j] = 0;
    if (y < 0 || y >= h) return;
    const uint8_t* rp = p + (int64_t)y * w;
#pragma unroll
    for (int j = 0; j < PXL; ++j)
        if (x0 + j < w) v[j] = __ldcg(reinterpret_cast<const unsigned char*>(rp + x0 + j));
}

__device__ __forceinline__ int px_load(const uint8_t* __restrict__ p, int w, int h, int x, int y) {
    return (x < 0 || y < 0 || x >= w || y >= h) ? 0 : (int)__ldcg(reinterpret_cast<const unsigned char*>(p + (int64_t)y * w + x));
}

// close one region row: lo[j] = min(m, max(r, nb)) then the horizontal clamp scans in both
// directions (the region's left / right halo pixels as boundary inputs); returns the new row
__device__ __forceinline__ void close_row(const int* m, const int* r, const int* nb, int lft, int rgt, int lane,
                                          int* u) {
    int lo[PXL];
#pragma unroll
    for (int j = 0; j < PXL; ++j) {
        int b = max(r[j], nb[j]);
        if (j == 0 && lane == 0) b = max(b, lft);
        if (j == PXL - 1 && lane == 31) b = max(b, rgt);
        lo[j] = min(b, m[j]);
    }
    int FL = lo[0], FH = m[0];
#pragma unroll
    for (int j = 1; j < PXL; ++j) {
        FL = min(m[j], max(lo[j], FL));
        FH = min(m[j], max(lo[j], FH));
    }
    int BL = lo[PXL - 1], BH = m[PXL - 1];
#pragma unroll
    for (int j = PXL - 2; j >= 0; --j) {
        BL = min(m[j], max(lo[j], BL));
        BH = min(m[j], max(lo[j], BH));
    }
    int in = __shfl_up_sync(FULL, clamp_scan<true>(FL, FH, lane), 1);
    int ib = __shfl_down_sync(FULL, clamp_scan<false>(BL, BH, lane), 1);
    if (lane == 0) in = 0;
    if (lane == 31) ib = 0;
    int fw[PXL];
#pragma unroll
    for (int j = 0; j < PXL; ++j) {
        in = min(m[j], max(lo[j], in));
        fw[j] = in;
    }
#pragma unroll
    for (int j = PXL - 1; j >= 0; --j) {
        ib = min(m[j], max(lo[j], ib));
        u[j] = max(fw[j], ib);
    }
}

// 3-wide max of a neighbouring row held in registers (xl / xr: the pixels just outside)
__device__ __forceinline__ void max3_row(const int* v, int xl, int xr, int lane, int* out) {
    int left = __shfl_up_sync(FULL, v[PXL - 1], 1), right = __shfl_down_sync(FULL, v[0], 1);
    if (lane == 0) left = xl;
    if (lane == 31) right = xr;
#pragma unroll
    for (int j = 0; j < PXL; ++j)
        out[j] = max(v[j], max(j == 0 ? left : v[j - 1], j == PXL - 1 ? right : v[j + 1]));
}

constexpr int ACOLS = RX * SW;      // region columns (256)
constexpr int AROWS = RY * kTile;   // region rows (128)
constexpr int CPL = AROWS / 32;     // column pixels per lane (4)
static_assert(PXL == 8 && CPL == 4, "ADI closure assumes 256 x 128 px regions");

// close window row wr (1..AROWS) across the region; returns the lane's changed-pixel mask
__device__ __forceinline__ uint32_t adi_row_close(const uint8_t* sR, uint8_t* sRw, const uint8_t* sM, int wr, int lane) {
    const int c0 = PXL * lane + 1;
    int m[PXL], r[PXL], nb[PXL], u[PXL];
    int upv[PXL + 2], dnv[PXL + 2];
#pragma unroll
    for (int j = -1; j <= PXL; ++j) {
        upv[j + 1] = sR[bidx(wr - 1, c0 + j)];
        dnv[j + 1] = sR[bidx(wr + 1, c0 + j)];
    }
#pragma unroll
    for (int j = 0; j < PXL; ++j) {
        m[j] = sM[bidx(wr, c0 + j)];
        r[j] = sR[bidx(wr, c0 + j)];
        nb[j] = max(max(max(upv[j], upv[j + 1]), upv[j + 2]), max(max(dnv[j], dnv[j + 1]), dnv[j + 2]));
    }
    const int lft = sR[bidx(wr, c0 - 1)], rgt = sR[bidx(wr, c0 + PXL)];
    bool can = false;
#pragma unroll
    for (int j = 0; j < PXL; ++j) {
        const int hn = max(j == 0 ? lft : r[j - 1], j == PXL - 1 ? rgt : r[j + 1]);
        can |= min(max(nb[j], hn), m[j]) > r[j];
    }
    if (!__any_sync(FULL, can)) return 0;
    close_row(m, r, nb, lft, rgt, lane, u);
    uint32_t chg = 0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < PXL; ++j)
        if (u[j] != r[j]) {
            sRw[bidx(wr, c0 + j)] = (uint8_t)u[j];
            chg |= 1u << j;
        }
    __syncwarp();
    return chg;
}
// close window column wc (1..ACOLS) along the region; lane owns rows 4*lane+1 .. +4
__device__ __forceinline__ uint32_t adi_col_close(const uint8_t* sR, uint8_t* sRw, const uint8_t* sM, int wc, int lane) {
    const int r0 = CPL * lane + 1;
    int m[CPL], r[CPL], nb[CPL], u[CPL];
    int lv[CPL + 2], rv[CPL + 2];
#pragma unroll
    for (int j = -1; j <= CPL; ++j) {
        lv[j + 1] = sR[bidx(r0 + j, wc - 1)];
        rv[j + 1] = sR[bidx(r0 + j, wc + 1)];
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        m[j] = sM[bidx(r0 + j, wc)];
        r[j] = sR[bidx(r0 + j, wc)];
        nb[j] = max(max(max(lv[j], lv[j + 1]), lv[j + 2]), max(max(rv[j], rv[j + 1]), rv[j + 2]));
    }
    const int top = sR[bidx(r0 - 1, wc)], bot = sR[bidx(r0 + CPL, wc)];
    bool can = false;
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const int vn = max(j == 0 ? top : r[j - 1], j == CPL - 1 ? bot : r[j + 1]);
        can |= min(max(nb[j], vn), m[j]) > r[j];
    }
    if (!__any_sync(FULL, can)) return 0;
    int lo[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        int b = max(r[j], nb[j]);
        if (j == 0 && lane == 0) b = max(b, top);
        if (j == CPL - 1 && lane == 31) b = max(b, bot);
        lo[j] = min(b, m[j]);
    }
    int FL = lo[0], FH = m[0];
#pragma unroll
    for (int j = 1; j < CPL; ++j) {
        FL = min(m[j], max(lo[j], FL));
        FH = min(m[j], max(lo[j], FH));
    }
    int BL = lo[CPL - 1], BH = m[CPL - 1];
#pragma unroll
    for (int j = CPL - 2; j >= 0; --j) {
        BL = min(m[j], max(lo[j], BL));
        BH = min(m[j], max(lo[j], BH));
    }
    int in = __shfl_up_sync(FULL, clamp_scan<true>(FL, FH, lane), 1);
    int ib = __shfl_down_sync(FULL, clamp_scan<false>(BL, BH, lane), 1);
    if (lane == 0) in = 0;
    if (lane == 31) ib = 0;
    int fw[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        in = min(m[j], max(lo[j], in));
        fw[j] = in;
    }
#pragma unroll
    for (int j = CPL - 1; j >= 0; --j) {
        ib = min(m[j], max(lo[j], ib));
        u[j] = max(fw[j], ib);
    }
    uint32_t chg = 0;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CPL; ++j)
        if (u[j] != r[j]) {
            sRw[bidx(r0 + j, wc)] = (uint8_t)u[j];
            chg |= 1u << j;
        }
    __syncwarp();
    return chg;
}

// One region closure by alternating phases (see k_region_adi); S holds the window and the
// rowdirty / coldirty / rowsnap / colsnap / subchg words (rowdirty seeded by the caller, the
// rest zero).  On return S.subchg[k] = the rows of sub-tile k that changed.
template <class SM, class Ensure>
__device__ void adi_close_region(SM& S, const uint8_t* sR, uint8_t* sRw, const uint8_t* sM, int warp, int lane,
                                 int& phases, int& lines, Ensure ensure_full) {
    auto improves = [&](int pr, int pc, int qr, int qc) {
        return min((int)sR[bidx(pr, pc)], (int)sM[bidx(qr, qc)]) > (int)sR[bidx(qr, qc)];
    };
    auto mark = [&](uint32_t* bits, int i) { atomicOr(&bits[i >> 5], 1u << (i & 31)); };
    while (true) {
        // ---- row phase
        if (threadIdx.x < AROWS / 32) {
            S.rowsnap[threadIdx.x] = S.rowdirty[threadIdx.x];
            S.rowdirty[threadIdx.x] = 0;
        }
        __syncthreads();
        int anyr = 0;
#pragma unroll
        for (int k = 0; k < AROWS / 32; ++k) anyr |= S.rowsnap[k] != 0;
        if (anyr) {
            ++phases;
            for (int y = 1 + warp; y <= AROWS; y += NW) {
                if (!((S.rowsnap[(y - 1) >> 5] >> ((y - 1) & 31)) & 1)) continue;
                ++lines;
                const uint32_t chg = adi_row_close(sR, sRw, sM, y, lane);
                if (!__any_sync(FULL, chg != 0)) continue;
                // neighbours above / below the changed pixels that can still rise
                uint32_t cm = 0;  // bits: columns c0-1 .. c0+PXL (10)
                const int c0 = PXL * lane + 1;
#pragma unroll
                for (int j = 0; j < PXL; ++j) {
                    if (!((chg >> j) & 1)) continue;
#pragma unroll
                    for (int d = -1; d <= 1; ++d) {
                        const int c = c0 + j + d;
                        if (c < 1 || c > ACOLS) continue;
                        if ((y > 1 && improves(y, c0 + j, y - 1, c)) ||
                            (y < AROWS && improves(y, c0 + j, y + 1, c)))
                            cm |= 1u << (j + d + 1);
                    }
                }
                if (cm) {
                    for (int b = 0; b < PXL + 2; ++b)
                        if ((cm >> b) & 1) mark(S.coldirty, c0 - 1 + b - 1);
                }
                const unsigned lanes = __ballot_sync(FULL, chg != 0);
                constexpr int LPS = SW / PXL;  // lanes per sub-tile column
                if ((lane % LPS) == 0 && ((lanes >> lane) & (uint32_t)((1ull << LPS) - 1))) {
                    const int sx = lane / LPS, sy = (y - 1) >> 5;
                    atomicOr(&S.subchg[sy * RX + sx], 1u << ((y - 1) & 31));
                }
            }
        }
        __syncthreads();
        // ---- column phase
        if (threadIdx.x < ACOLS / 32) {
            S.colsnap[threadIdx.x] = S.coldirty[threadIdx.x];
            S.coldirty[threadIdx.x] = 0;
        }
        __syncthreads();
        int anyc = 0;
#pragma unroll
        for (int k = 0; k < ACOLS / 32; ++k) anyc |= S.colsnap[k] != 0;
        if (anyc) ensure_full();  // a column closure reads whole window columns
        if (anyc) {
            ++phases;
            for (int c = 1 + warp; c <= ACOLS; c += NW) {
                if (!((S.colsnap[(c - 1) >> 5] >> ((c - 1) & 31)) & 1)) continue;
                ++lines;
                const uint32_t chg = adi_col_close(sR, sRw, sM, c, lane);
                if (!__any_sync(FULL, chg != 0)) continue;
                uint32_t rm = 0;  // bits: rows r0-1 .. r0+CPL (6)
                const int r0 = CPL * lane + 1;
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    if (!((chg >> j) & 1)) continue;
#pragma unroll
                    for (int d = -1; d <= 1; ++d) {
                        const int rr = r0 + j + d;
                        if (rr < 1 || rr > AROWS) continue;
                        if ((c > 1 && improves(r0 + j, c, rr, c - 1)) ||
                            (c < ACOLS && improves(r0 + j, c, rr, c + 1)))
                            rm |= 1u << (j + d + 1);
                    }
                }
                if (rm) {
                    for (int b = 0; b < CPL + 2; ++b)
                        if ((rm >> b) & 1) mark(S.rowdirty, r0 - 1 + b - 1);
                }
                // sub-tile changed rows: lanes 8k..8k+7 hold rows of sub-tile row k
                const int sx = (c - 1) / SW;
                uint32_t mine = 0;
#pragma unroll
                for (int j = 0; j < CPL; ++j)
                    if ((chg >> j) & 1) mine |= 1u << ((r0 - 1 + j) & 31);
#pragma unroll
                for (int k = 0; k < RY; ++k) {
                    const uint32_t b = __reduce_or_sync(FULL, (lane >> 3) == k ? mine : 0u);
                    if (lane == 0 && b) atomicOr(&S.subchg[k * RX + sx], b);
                }
            }
        }
        __syncthreads();
        // every thread reads rowdirty BEFORE the barrier, so the reset at the next row phase
        // cannot race with a slower warp's read
        int pend = 0;
#pragma unroll
        for (int k = 0; k < AROWS / 32; ++k) pend |= S.rowdirty[k] != 0;
        if (!__syncthreads_or(pend)) break;
    }
}

struct Smem {
    uint32_t R[ROWS * RWW];
    uint32_t M[ROWS * RWW];
    uint32_t dirty[NW];  // rows of each sub-tile that may still improve (pushed by neighbours)
    uint32_t first_mask[NW];  // (HP_RG_PROFILE == 2) the incoming masks of the job
    int pend;            // sub-tiles with dirty != 0 plus sub-tiles being processed
    int job;
    int again;
    unsigned long long t0, tA, tB;
    int first;  // HP_RG_FIRSTORDER: this job is the region's first
    int thin;   // HP_RG_THIN: this job's few dirty rows go to the alternating-phase closure
    int visits; // earlier jobs of this region in this launch
    int allrows; // every sub-tile row of the job is dirty (a region's first job)
    uint32_t rowdirty[AROWS / 32], coldirty[ACOLS / 32], rowsnap[AROWS / 32], colsnap[ACOLS / 32];
    uint32_t subchg[NW];
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


__global__ void __launch_bounds__(NW * 32, HP_RG_MINB) k_region_mr8(const uint8_t* __restrict__ mask,
                                                           uint8_t* __restrict__ R, int w, int h,
                                                           Worklist wl, int thin_rows, int chain_visits) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const uint8_t* sR = reinterpret_cast<const uint8_t*>(S.R);
    uint8_t* sRw = reinterpret_cast<uint8_t*>(S.R);
    const uint8_t* sM = reinterpret_cast<const uint8_t*>(S.M);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sx = warp % RX, sy = warp / RX;
    const int wr0 = sy * kTile, wc0 = sx * SW;  // window origin of this sub-tile (minus halo)

    // close row y (1..32) of this warp's sub-tile (lane owns PPL adjacent pixels); true iff it
    // may have changed.  A pixel's update is the clamp f(v) = min(m, max(lo, v)) of the value v
    // arriving along the row; clamps compose, so a lane's PPL pixels are one clamp and the row
    // closure is a warp scan of clamps in each direction.
    auto row = [&](int y) -> int {
        const int wr = wr0 + y, c0 = wc0 + PPL * lane + 1;
        int m[PPL], rr[PPL], vm[PPL];
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int c = c0 + j;
            m[j] = sM[bidx(wr, c)];
            rr[j] = sR[bidx(wr, c)];
            const int up = max(max(sR[bidx(wr - 1, c - 1)], sR[bidx(wr - 1, c)]), sR[bidx(wr - 1, c + 1)]);
            const int dn = max(max(sR[bidx(wr + 1, c - 1)], sR[bidx(wr + 1, c)]), sR[bidx(wr + 1, c + 1)]);
            vm[j] = max(up, dn);
        }
        const int lft = sR[bidx(wr, c0 - 1)], rgt = sR[bidx(wr, c0 + PPL)];
        bool can = false;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int hn = max(j == 0 ? lft : rr[j - 1], j == PPL - 1 ? rgt : rr[j + 1]);
            can |= min(max(vm[j], hn), m[j]) > rr[j];
        }
        if (!__any_sync(FULL, can)) return 0;
        int lo[PPL];
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            int b = max(rr[j], vm[j]);
            if (j == 0 && lane == 0) b = max(b, lft);
            if (j == PPL - 1 && lane == 31) b = max(b, rgt);
            lo[j] = min(b, m[j]);
        }
        // the clamp scans are only needed if some pixel can take a horizontal neighbour's value
        int nl = __shfl_up_sync(FULL, lo[PPL - 1], 1), nr = __shfl_down_sync(FULL, lo[0], 1);
        if (lane == 0) nl = 0;
        if (lane == 31) nr = 0;
        bool need = false;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int a = j == 0 ? nl : lo[j - 1], bb = j == PPL - 1 ? nr : lo[j + 1];
            need |= min(max(a, bb), m[j]) > lo[j];
        }
        int u[PPL];
#pragma unroll
        for (int j = 0; j < PPL; ++j) u[j] = lo[j];
        bool scan = __any_sync(FULL, need);
#if HP_RG_JACOBI > 0
        // short propagation first: up to HP_RG_JACOBI neighbour-exchange steps (each lane
        // relaxes its pixels from both row neighbours); stop at the fixed point, else close the
        // row with the scans from the partially propagated values (same closure)
        for (int it = 0; scan && it < HP_RG_JACOBI; ++it) {
            int left = __shfl_up_sync(FULL, u[PPL - 1], 1), right = __shfl_down_sync(FULL, u[0], 1);
            if (lane == 0) left = 0;
            if (lane == 31) right = 0;
            bool ch = false;
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int nb = max(j == 0 ? left : u[j - 1], j == PPL - 1 ? right : u[j + 1]);
                const int nv = min(m[j], max(u[j], nb));
                ch |= nv != u[j];
                u[j] = nv;
            }
#pragma unroll
            for (int j = PPL - 2; j >= 0; --j) {
                const int nv = min(m[j], max(u[j], u[j + 1]));
                ch |= nv != u[j];
                u[j] = nv;
            }
            scan = __any_sync(FULL, ch);
        }
        if (scan) {
#pragma unroll
            for (int j = 0; j < PPL; ++j) lo[j] = u[j];
        }
#endif
        if (scan) {
            // left -> right: the lane's clamp is pixel PPL-1 o ... o pixel 0
            int FL = lo[0], FH = m[0];
#pragma unroll
            for (int j = 1; j < PPL; ++j) {
                FL = min(m[j], max(lo[j], FL));
                FH = min(m[j], max(lo[j], FH));
            }
            // right -> left
            int BL = lo[PPL - 1], BH = m[PPL - 1];
#pragma unroll
            for (int j = PPL - 2; j >= 0; --j) {
                BL = min(m[j], max(lo[j], BL));
                BH = min(m[j], max(lo[j], BH));
            }
#if HP_RG_PACKSCAN
            uint32_t Fp = (uint32_t)FL | ((uint32_t)FH << 16), Bp = (uint32_t)BL | ((uint32_t)BH << 16);
            clamp_scan_both(Fp, Bp, lane);
            int in = __shfl_up_sync(FULL, (int)(Fp & 0xffffu), 1);
            int ib = __shfl_down_sync(FULL, (int)(Bp & 0xffffu), 1);
#else
            int in = __shfl_up_sync(FULL, clamp_scan<true>(FL, FH, lane), 1);
            int ib = __shfl_down_sync(FULL, clamp_scan<false>(BL, BH, lane), 1);
#endif
            if (lane == 0) in = 0;
            if (lane == 31) ib = 0;
            int fw[PPL];
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                in = min(m[j], max(lo[j], in));
                fw[j] = in;
            }
#pragma unroll
            for (int j = PPL - 1; j >= 0; --j) {
                ib = min(m[j], max(lo[j], ib));
                u[j] = max(fw[j], ib);
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < PPL; ++j)
            if (u[j] != rr[j]) sRw[bidx(wr, c0 + j)] = (uint8_t)u[j];
        __syncwarp();
#if HP_RG_EAGER
        // which of the sub-tile's left / right column pixels changed (for eager pushes)
        const int lc = __shfl_sync(FULL, (int)(u[0] != rr[0]), 0);
        const int rc = __shfl_sync(FULL, (int)(u[PPL - 1] != rr[PPL - 1]), 31);
        return 1 | (lc << 1) | (rc << 2);
#else
        return 1;
#endif
    };
    // can window pixel p (pr, pc) improve window pixel q (qr, qc)?
    auto improves = [&](int pr, int pc, int qr, int qc) {
        return min((int)sR[bidx(pr, pc)], (int)sM[bidx(qr, qc)]) > (int)sR[bidx(qr, qc)];
    };

    while (true) {
        if (threadIdx.x == 0) {
            // Retire instead of queueing for work when HP_RG_WAITERS CTAs already wait on an
            // empty queue (at least HP_RG_MIN_ALIVE stay): on chain-bound tiles only a few
            // dozen regions are active at a time, and idle CTAs would hold a quarter of every
            // SM's threads and half its registers from the other slots' kernels for
            // milliseconds.  Only a CTA without a ticket retires, so no pushed job is lost.
            int t = -1;
            const unsigned long long hd = vload(&wl.ctr[0]), tl = vload(&wl.ctr[1]);
            bool retire = false;
            if (hd >= tl + HP_RG_WAITERS) {
                const unsigned long long r = atomicAdd(&wl.ctr[7], 1ull);
                if (r + HP_RG_MIN_ALIVE < gridDim.x) retire = true;
                else atomicAdd(&wl.ctr[7], ~0ull);
            }
            if (!retire) {
                t = q_pop(wl);
                if (t >= 0) atomicExch(&wl.state[t], ST_BUSY);
            }
            // region visit count (state words past the regions and their order keys): a
            // region popped again and again lies on a long propagation chain
            S.visits = t >= 0 ? (int)atomicAdd(&wl.state[2 * wl.ntx * wl.nty + t], 1u) : 0;
            S.t0 = gtimer();
            S.job = t;
        }
        __syncthreads();
        const int t = S.job;
        if (t < 0) break;
        const int rx = t % wl.ntx, ry = t / wl.ntx;
        const int X0 = rx * RX * SW, Y0 = ry * RY * kTile;
        // interior regions (window fully inside the image, rows 4-byte aligned) take the
        // unconditional vector path
        const bool inner = X0 >= 4 && X0 + RX * SW + 4 <= w && Y0 >= 1 && Y0 + RY * kTile + 1 <= h &&
                           (w & 3) == 0 && (((uintptr_t)R | (uintptr_t)mask) & 3) == 0;
        bool have_window = false;
        while (true) {
            if (lane == 0) S.dirty[warp] = atomicExch(&wl.inrows[t * NW + warp], 0u);
            __threadfence();
            __syncthreads();
            int any_in = 0;
#pragma unroll
            for (int k = 0; k < NW; ++k) any_in |= S.dirty[k] != 0;
            uint32_t mychg = 0;
            if (any_in) {
                if (!have_window) {
                    // the whole window: all of a thread's loads are issued before any store
                    constexpr int NIT = (ROWS * RWW + NW * 32 - 1) / (NW * 32);
                    uint32_t vr[NIT], vm[NIT];
                    if (inner) {
                        const uint8_t* rb = R + (int64_t)(Y0 - 1) * w + (X0 - 4);
                        const uint8_t* mb = mask + (int64_t)(Y0 - 1) * w + (X0 - 4);
#pragma unroll
                        for (int i = 0; i < NIT; ++i) {
                            int k = threadIdx.x + i * NW * 32;
                            if (k < ROWS * RWW) {
                                int r = k / RWW, wi = k - r * RWW;
                                int64_t o = (int64_t)r * w + 4 * wi;
                                vr[i] = __ldcg(reinterpret_cast<const unsigned int*>(rb + o));
                                vm[i] = __ldcg(reinterpret_cast<const unsigned int*>(mb + o));
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < NIT; ++i) {
                            int k = threadIdx.x + i * NW * 32;
                            if (k < ROWS * RWW) {
                                int r = k / RWW, wi = k - r * RWW;
                                int gx = X0 - 4 + 4 * wi, gy = Y0 - 1 + r;
                                vr[i] = load_word(R, w, h, gx, gy);
                                vm[i] = load_word(mask, w, h, gx, gy);
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < NIT; ++i) {
                        int k = threadIdx.x + i * NW * 32;
                        if (k < ROWS * RWW) {
                            S.R[k] = vr[i];
                            S.M[k] = vm[i];
                        }
                    }
                    have_window = true;
                } else {
                    // re-processing the same region: only the halo ring of R can have changed
                    // (the interior is owned by this CTA; the mask never changes)
                    constexpr int NH = 2 * RWW + 2 * (ROWS - 2);
                    for (int k = threadIdx.x; k < NH; k += blockDim.x) {
                        int r, wi;
                        if (k < 2 * RWW) {
                            r = k < RWW ? 0 : ROWS - 1;
                            wi = k % RWW;
                        } else {
                            int j = k - 2 * RWW;
                            r = 1 + (j >> 1);
                            wi = (j & 1) ? RWW - 1 : 0;
                        }
                        S.R[r * RWW + wi] = load_word(R, w, h, X0 - 4 + 4 * wi, Y0 - 1 + r);
                    }
                }
                if (threadIdx.x == 0) {
#if HP_RG_FIRSTORDER
                    // a region's first job (every row of every sub-tile dirty): only the top row
                    // of sub-tiles starts; each releases the one below when its first sweep set
                    // ends, so lower sub-tiles do not sweep against stale top halos first
                    bool first = true;
                    for (int k = 0; k < NW; ++k) first &= S.dirty[k] == 0xffffffffu;
                    S.first = first;
                    if (first)
                        for (int k = RX; k < NW; ++k) S.dirty[k] = 0;
#endif
                    int np = 0, nbits = 0;
                    for (int k = 0; k < NW; ++k) {
                        np += S.dirty[k] != 0;
                        nbits += __popc(S.dirty[k]);
                    }
                    S.pend = np;
                    S.thin = nbits <= thin_rows && S.visits >= chain_visits;
                    S.allrows = nbits == NW * 32;  // a region's first job: every row dirty
#if HP_RG_PROFILE
                    S.tA = gtimer();
#endif
#if HP_RG_PROFILE == 2
                    for (int k = 0; k < NW; ++k) S.first_mask[k] = S.dirty[k];
#endif
                }
                __syncthreads();
                // Asynchronous sub-tile warps: a warp takes its own dirty rows, sweeps them to a
                // fixed point, then pushes the rows of in-region neighbour sub-tiles its changed
                // border pixels can improve.  Token count: a 0 -> nonzero transition of a dirty
                // mask adds one to pend, a warp releases the token it took after its pushes, so
                // pend == 0 iff no sub-tile of the region has work left.
                int iters = 0;
                int nrows = 0;
                const int r = wr0 + lane + 1;
                unsigned backoff = HP_POLL_NS;
#if HP_RG_FIRSTROW
                if (!S.thin && S.allrows) {
                    // first job: one full-width closure of every region row (8 px per lane)
                    // before the sub-tile sweeps, so values cross the sub-tile borders along
                    // the rows at once; its changed rows join the write-back
                    if (lane == 0) S.subchg[warp] = 0;
                    __syncthreads();
                    for (int y = 1 + warp; y <= AROWS; y += NW) {
                        const uint32_t chg = adi_row_close(sR, sRw, sM, y, lane);
                        constexpr int LPS = SW / PXL;
                        const unsigned lanes = __ballot_sync(FULL, chg != 0);
                        if ((lane % LPS) == 0 && ((lanes >> lane) & (uint32_t)((1ull << LPS) - 1)))
                            atomicOr(&S.subchg[((y - 1) >> 5) * RX + lane / LPS], 1u << ((y - 1) & 31));
                    }
                    __syncthreads();
                    mychg = S.subchg[warp];
                }
#endif
                if (S.thin) {
                    // a thin job (a few dirty rows, e.g. a wave front crossing the region
                    // along a corridor): alternating full-width row / full-height column
                    // closures instead of the sub-tile sweeps
                    if (threadIdx.x < AROWS / 32) S.rowdirty[threadIdx.x] = 0;
                    if (threadIdx.x < ACOLS / 32) S.coldirty[threadIdx.x] = 0;
                    if (lane == 0) S.subchg[warp] = 0;
                    __syncthreads();
                    if (lane == 0 && S.dirty[warp]) atomicOr(&S.rowdirty[warp / RX], S.dirty[warp]);
                    __syncthreads();
                    adi_close_region(S, sR, sRw, sM, warp, lane, iters, nrows, [] {});
                    mychg = S.subchg[warp];
                } else while (true) {
                    uint32_t dirty = 0;
                    if (lane == 0 && *reinterpret_cast<volatile uint32_t*>(&S.dirty[warp]))
                        dirty = atomicExch(&S.dirty[warp], 0u);
                    dirty = __shfl_sync(FULL, dirty, 0);
                    if (!dirty) {
                        if (*reinterpret_cast<volatile int*>(&S.pend) == 0) break;
                        // idle: exponential back-off so waiting warps leave the issue slots to
                        // the working ones and to co-running kernels
                        __nanosleep(backoff);
                        backoff = min(2u * backoff, (unsigned)HP_POLL_MAX_NS);
                        continue;
                    }
                    backoff = HP_POLL_NS;
                    // Gauss-Seidel sweeps of this sub-tile (see iwpp_rules.cuh sweep_rows).  With
                    // HP_RG_EAGER, a changed top/bottom row or left/right column pixel marks the
                    // orthogonal in-region neighbour's adjacent rows dirty at once, so the
                    // neighbour starts while this sweep continues (the precise 8-neighbour pushes
                    // after the sweep set still follow).
                    uint32_t chg = 0;
                    auto eager = [&](int y, int code) {
#if HP_RG_EAGER
                        if (lane != 0) return;
                        auto push = [&](int nw, uint32_t m) {
                            if (atomicOr(&S.dirty[nw], m) == 0u) atomicAdd(&S.pend, 1);
                        };
                        if (y == kTile && sy < RY - 1) push(warp + RX, 1u);
                        if (y == 1 && sy > 0) push(warp - RX, 1u << 31);
                        const uint32_t near = (uint32_t)((7ull << (y - 1)) >> 1);  // rows y-1, y, y+1
                        if ((code & 2) && sx > 0) push(warp - 1, near);
                        if ((code & 4) && sx < RX - 1) push(warp + 1, near);
#else
                        (void)y;
                        (void)code;
#endif
                    };
                    while (dirty) {
                        for (int y = 1; y <= kTile; ++y) {
                            const uint32_t bit = 1u << (y - 1);
                            if (!(dirty & bit)) continue;
                            dirty &= ~bit;
                            ++nrows;
                            if (const int rc = row(y)) {
                                chg |= bit;
                                dirty |= (bit << 1) | (bit >> 1);
                                eager(y, rc);
                            }
                        }
                        if (!dirty) break;
                        for (int y = kTile; y >= 1; --y) {
                            const uint32_t bit = 1u << (y - 1);
                            if (!(dirty & bit)) continue;
                            dirty &= ~bit;
                            ++nrows;
                            if (const int rc = row(y)) {
                                chg |= bit;
                                dirty |= (bit << 1) | (bit >> 1);
                                eager(y, rc);
                            }
                        }
                    }
                    ++iters;
                    mychg |= chg;
#if HP_RG_FIRSTORDER
                    if (S.first && sy < RY - 1 && iters == 1 && lane == 0)  // release the sub-tile below
                        if (atomicOr(&S.dirty[warp + RX], 0xffffffffu) == 0u) atomicAdd(&S.pend, 1);
#endif
                    if (chg) {
                        // rows of in-region neighbours that changed border pixels can improve
                        // (m8 index = N8 direction of the neighbour, bit = its row)
                        uint32_t m8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                        constexpr uint32_t TOP = 1u << 31, BOT = 1u;
                        const bool mine_row = (chg >> lane) & 1;
#pragma unroll
                        for (int d = -1; d <= 1; ++d) {
#pragma unroll
                            for (int j = 0; j < PPL; ++j) {
                                const int c = wc0 + PPL * lane + 1 + j;
                                if (sy > 0 && (chg & 1) && improves(wr0 + 1, c, wr0, c + d)) {
                                    if (c + d == wc0) { if (sx > 0) m8[0] |= TOP; }
                                    else if (c + d == wc0 + SW + 1) { if (sx < RX - 1) m8[2] |= TOP; }
                                    else m8[1] |= TOP;
                                }
                                if (sy < RY - 1 && (chg >> 31) && improves(wr0 + kTile, c, wr0 + kTile + 1, c + d)) {
                                    if (c + d == wc0) { if (sx > 0) m8[5] |= BOT; }
                                    else if (c + d == wc0 + SW + 1) { if (sx < RX - 1) m8[7] |= BOT; }
                                    else m8[6] |= BOT;
                                }
                            }
                            if (sx > 0 && mine_row && improves(r, wc0 + 1, r + d, wc0)) {
                                if (r + d == wr0) { if (sy > 0) m8[0] |= TOP; }
                                else if (r + d == wr0 + kTile + 1) { if (sy < RY - 1) m8[5] |= BOT; }
                                else m8[3] |= 1u << (lane + d);
                            }
                            if (sx < RX - 1 && mine_row && improves(r, wc0 + SW, r + d, wc0 + SW + 1)) {
                                if (r + d == wr0) { if (sy > 0) m8[2] |= TOP; }
                                else if (r + d == wr0 + kTile + 1) { if (sy < RY - 1) m8[7] |= BOT; }
                                else m8[4] |= 1u << (lane + d);
                            }
                        }
                        uint32_t mine = 0;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            uint32_t v = __reduce_or_sync(FULL, m8[j]);
                            if (lane == j) mine = v;
                        }
                        if (lane < 8 && mine) {
                            const int nw = (sy + dy8(lane)) * RX + (sx + dx8(lane));
                            if (atomicOr(&S.dirty[nw], mine) == 0u) atomicAdd(&S.pend, 1);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) {
                        __threadfence_block();
                        atomicSub(&S.pend, 1);
                    }
                }
                __syncthreads();
#if HP_RG_PROFILE == 2  // ctr[4] = loop ns of first jobs (all rows dirty), ctr[6] = of the rest
                if (threadIdx.x == 0) {
                    S.tB = gtimer();
                    bool first = true;
                    for (int k = 0; k < NW; ++k) first &= S.first_mask[k] == 0xffffffffu;
                    atomicAdd(&wl.ctr[first ? 4 : 6], S.tB - S.tA);
                }
#elif HP_RG_PROFILE  // ctr[4] = ns in the sub-tile loop, ctr[6] = ns in write-back + activation
                if (threadIdx.x == 0) {
                    S.tB = gtimer();
                    atomicAdd(&wl.ctr[4], S.tB - S.tA);
                }
#else
                if (lane == 0) atomicAdd(&wl.ctr[4], (unsigned long long)iters);  // sub-tile sweep sets
                if (lane == 0) atomicAdd(&wl.ctr[6], (unsigned long long)nrows);
#endif
                // write back the changed rows of this sub-tile (interior words)
                if (mychg) {
                    constexpr int WPR = SW / 4;  // words per sub-tile row
                    for (int k = lane; k < kTile * WPR; k += 32) {
                        int y = 1 + k / WPR, wi = k % WPR;
                        if (!((mychg >> (y - 1)) & 1)) continue;
                        int gx = X0 + wc0 + 4 * wi, gy = Y0 + wr0 + y - 1;
                        if (gy >= h || gx >= w) continue;
                        uint8_t* dst = R + (int64_t)gy * w + gx;
                        uint32_t v = S.R[(wr0 + y) * RWW + sx * WPR + 1 + wi];
                        if (gx + 3 < w && (((uintptr_t)dst) & 3) == 0) {
                            __stcg(reinterpret_cast<unsigned int*>(dst), v);
                        } else {
                            for (int b = 0; b < 4 && gx + b < w; ++b)
                                __stcg(reinterpret_cast<unsigned char*>(dst + b), (unsigned char)(v >> (8 * b)));
                        }
                    }
                    __threadfence();
                    // activations of sub-tiles in neighbouring regions (edges of the region)
                    uint32_t m8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    const int r = wr0 + lane + 1;
                    constexpr uint32_t TOP = 1u << 31, BOT = 1u;
#pragma unroll
                    for (int d = -1; d <= 1; ++d) {
#pragma unroll
                        for (int j = 0; j < PPL; ++j) {
                            const int c = wc0 + PPL * lane + 1 + j;
                            // only pixels of rows changed in this job can newly improve a
                            // neighbour (an unchanged pixel's offer was delivered when it got its
                            // value); thin jobs also hold only those rows' neighbourhoods
                            if (sy == 0 && (mychg & 1u) && improves(wr0 + 1, c, wr0, c + d)) {
                                if (c + d == wc0) m8[0] |= TOP;
                                else if (c + d == wc0 + SW + 1) m8[2] |= TOP;
                                else m8[1] |= TOP;
                            }
                            if (sy == RY - 1 && (mychg >> 31) && improves(wr0 + kTile, c, wr0 + kTile + 1, c + d)) {
                                if (c + d == wc0) m8[5] |= BOT;
                                else if (c + d == wc0 + SW + 1) m8[7] |= BOT;
                                else m8[6] |= BOT;
                            }
                        }
                        const bool rowchg = (mychg >> lane) & 1u;
                        if (sx == 0 && rowchg && improves(r, wc0 + 1, r + d, wc0)) {
                            if (r + d == wr0) m8[0] |= TOP;
                            else if (r + d == wr0 + kTile + 1) m8[5] |= BOT;
                            else m8[3] |= 1u << (lane + d);
                        }
                        if (sx == RX - 1 && rowchg && improves(r, wc0 + SW, r + d, wc0 + SW + 1)) {
                            if (r + d == wr0) m8[2] |= TOP;
                            else if (r + d == wr0 + kTile + 1) m8[7] |= BOT;
                            else m8[4] |= 1u << (lane + d);
                        }
                    }
                    // (diagonal reach across the region edge from an inner sub-tile's corner is
                    // covered by the top/bottom row checks: c + d == wc0 / wc0 + SW + 1)
                    uint32_t mine = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uint32_t v = __reduce_or_sync(FULL, m8[j]);
                        if (lane == j) mine = v;
                    }
                    if (lane < 8 && mine) {
                        int gsx = rx * RX + sx + dx8(lane), gsy = ry * RY + sy + dy8(lane);
                        int nrx = gsx >= 0 ? gsx / RX : -1, nry = gsy >= 0 ? gsy / RY : -1;
                        if (gsx >= 0 && gsy >= 0 && nrx < wl.ntx && nry < wl.nty && (nrx != rx || nry != ry)) {
                            int nt = nry * wl.ntx + nrx;
                            int sub = (gsy % RY) * RX + (gsx % RX);
                            atomicOr(&wl.inrows[nt * NW + sub], mine);
                            q_activate(wl, nt);
                        }
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
#if HP_RG_PROFILE == 1
                if (any_in) atomicAdd(&wl.ctr[6], gtimer() - S.tB);
#endif
                int again = 0;
                uint32_t o = atomicCAS(&wl.state[t], ST_BUSY, ST_IDLE);
                if (o == ST_BUSY) {
                    atomicAdd(&wl.ctr[2], ~0ull);
                } else {
                    atomicExch(&wl.state[t], ST_BUSY);
                    again = 1;
                }
                atomicAdd(&wl.ctr[3], 1ull);
                if (!again) atomicAdd(&wl.ctr[5], gtimer() - S.t0);  // ns a region was owned
                S.again = again;
            }
            __syncthreads();
            if (!S.again) break;
        }
    }
}

__global__ void k_rg_reset(Worklist wl, bool seeded) {
    const int n = wl.ntx * wl.nty;
    const int lim = max(wl.cap, n * NW);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += gridDim.x * blockDim.x) {
        if (i < n) wl.state[i] = ST_QUEUED;
        if (i < n) wl.state[2 * n + i] = 0u;  // visit counts (k_region_mr8)
        if (i < n * NW && !seeded) wl.inrows[i] = 0xffffffffu;
        if (i < wl.cap) {
            int32_t v = EMPTY;
            if (i < n) {
#if HP_RG_ORDER == 1
                // 4-colour order (x parity, y parity): no two regions of one colour are
                // 8-adjacent, so a wave of one colour never reads a neighbour mid-update
                int k = i, c = 0;
                for (; c < 4; ++c) {
                    const int nx = (wl.ntx - (c & 1) + 1) / 2, ny = (wl.nty - (c >> 1) + 1) / 2;
                    if (k < nx * ny) {
                        v = (2 * (k / nx) + (c >> 1)) * wl.ntx + 2 * (k % nx) + (c & 1);
                        break;
                    }
                    k -= nx * ny;
                }
#else
                v = i;
#endif
            }
            wl.queue[i] = v;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 8)
        wl.ctr[threadIdx.x] = (threadIdx.x == 1 || threadIdx.x == 2) ? (unsigned long long)n : 0ull;
}

// ---- Vincent's hybrid initialisation ("Vincent MR"), per
// region: a raster sweep (rows top to bottom, each row closed horizontally in both directions
// with the row above as input) then an anti-raster sweep (bottom to top, the row below as
// input), one warp per 256 x 128 px region, values in registers (PXL pixels per lane).  Every
// update is a monotone step toward the reconstruction, so the queue engine that follows
// reaches the same fixed point; it is seeded with exactly the sub-tile rows that still hold
// an improvable pixel (k_rg_seed), instead of every row of every region.
__global__ void __launch_bounds__(128) k_rg_init(const uint8_t* __restrict__ mask, uint8_t* __restrict__ R, int w,
                                                 int h, int ntx, int nty) {
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (t >= ntx * nty) return;
    const int X0 = (t % ntx) * RX * SW, Y0 = (t / ntx) * RY * kTile;
    const int Y1 = min(h, Y0 + RY * kTile);
    const int x0 = X0 + PXL * lane;
    int prev[PXL], m[PXL], r[PXL], nb[PXL], u[PXL];
    // raster: the row above as input (the first from memory)
    row_io_load(R, w, h, x0, Y0 - 1, prev);
    int pl = px_load(R, w, h, X0 - 1, Y0 - 1), pr = px_load(R, w, h, X0 + RX * SW, Y0 - 1);
    for (int y = Y0; y < Y1; ++y) {
        row_io_load(mask, w, h, x0, y, m);
        row_io_load(R, w, h, x0, y, r);
        const int lft = px_load(R, w, h, X0 - 1, y), rgt = px_load(R, w, h, X0 + RX * SW, y);
        max3_row(prev, pl, pr, lane, nb);
        close_row(m, r, nb, lft, rgt, lane, u);
        uint8_t* rp = R + (int64_t)y * w;
#pragma unroll
        for (int j = 0; j < PXL; ++j) {
            if (x0 + j < w && u[j] != r[j]) __stcg(reinterpret_cast<unsigned char*>(rp + x0 + j), (unsigned char)u[j]);
            prev[j] = u[j];
        }
        pl = lft;
        pr = rgt;
    }
    // anti-raster: the row below as input (the first from memory); the row above from memory
    row_io_load(R, w, h, x0, Y1, prev);
    pl = px_load(R, w, h, X0 - 1, Y1);
    pr = px_load(R, w, h, X0 + RX * SW, Y1);
    for (int y = Y1 - 1; y >= Y0; --y) {
        int up[PXL], upm[PXL];
        row_io_load(mask, w, h, x0, y, m);
        row_io_load(R, w, h, x0, y, r);
        row_io_load(R, w, h, x0, y - 1, up);
        const int lft = px_load(R, w, h, X0 - 1, y), rgt = px_load(R, w, h, X0 + RX * SW, y);
        max3_row(prev, pl, pr, lane, nb);
        max3_row(up, px_load(R, w, h, X0 - 1, y - 1), px_load(R, w, h, X0 + RX * SW, y - 1), lane, upm);
#pragma unroll
        for (int j = 0; j < PXL; ++j) nb[j] = max(nb[j], upm[j]);
        close_row(m, r, nb, lft, rgt, lane, u);
        uint8_t* rp = R + (int64_t)y * w;
#pragma unroll
        for (int j = 0; j < PXL; ++j) {
            if (x0 + j < w && u[j] != r[j]) __stcg(reinterpret_cast<unsigned char*>(rp + x0 + j), (unsigned char)u[j]);
            prev[j] = u[j];
        }
        pl = lft;
        pr = rgt;
    }
}

// inrows of every sub-tile = its rows holding a pixel p that some 8-neighbour q can still
// improve (min(R(q), M(p)) > R(p)); one warp per sub-tile, lane = PPL pixels of a row
__global__ void __launch_bounds__(256) k_rg_seed(const uint8_t* __restrict__ mask, const uint8_t* __restrict__ R,
                                                 int w, int h, Worklist wl) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int nreg = wl.ntx * wl.nty;
    if (gw >= nreg * NW) return;
    const int t = gw / NW, sub = gw % NW;
    const int X0 = (t % wl.ntx) * RX * SW + (sub % RX) * SW, Y0 = (t / wl.ntx) * RY * kTile + (sub / RX) * kTile;
    uint32_t rows = 0;
    for (int yy = 0; yy < kTile; ++yy) {
        const int y = Y0 + yy;
        bool imp = false;
        if (y < h) {
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int x = X0 + PPL * lane + j;
                if (x >= w) continue;
                const int rp = px_load(R, w, h, x, y), mp = px_load(mask, w, h, x, y);
                if (rp >= mp) continue;  // already at its mask: cannot rise
                int nbv = 0;
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx)
                        if (dx || dy) nbv = max(nbv, px_load(R, w, h, x + dx, y + dy));
                imp |= min(nbv, mp) > rp;
            }
        }
        if (__any_sync(FULL, imp)) rows |= 1u << yy;
    }
    if (lane == 0) wl.inrows[t * NW + sub] = rows;
}

// ---- Alternating-direction region closure (HP_RG_ADI): the same queue, states and window as
// k_region_mr8, but a region job closes its window by alternating two synchronous phases over
// the whole region instead of asynchronous 64 x 32 sub-tile sweeps:
//   row phase     every dirty region row closed across the full 256 px (8 px per lane, the
//                 clamp scans of row()), its rows above / below as inputs;
//   column phase  every dirty region column closed along its full 128 px (4 px per lane,
//                 the same clamp scans vertically), its columns left / right as inputs.
// A pixel a phase raises marks, for the other direction, exactly the lines of the neighbours
// it can still improve (min(R(p), M(q)) > R(q)), so a horizontal run closes in one row step
// and a vertical run in one column step -- a 1-px corridor crosses a region in one phase per
// turn instead of one dependent row closure per row.  Monotone updates: same fixed point.
struct SmemA {
    uint32_t R[ROWS * RWW];
    uint32_t M[ROWS * RWW];
    uint32_t rowdirty[AROWS / 32];   // bit y-1: window row y needs a row closure
    uint32_t coldirty[ACOLS / 32];   // bit c-1: window column c needs a column closure
    uint32_t rowsnap[AROWS / 32];
    uint32_t colsnap[ACOLS / 32];
    uint32_t subchg[NW];             // per sub-tile: rows that changed in this job
    uint32_t dirty_in[NW];
    int any;
    int job;
    int again;
    int visits;
    unsigned long long t0;
};

__global__ void __launch_bounds__(NW * 32, HP_RG_MINB) k_region_adi(const uint8_t* __restrict__ mask,
                                                           uint8_t* __restrict__ R, int w, int h, Worklist wl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemA& S = *reinterpret_cast<SmemA*>(smem_raw);
    const uint8_t* sR = reinterpret_cast<const uint8_t*>(S.R);
    uint8_t* sRw = reinterpret_cast<uint8_t*>(S.R);
    const uint8_t* sM = reinterpret_cast<const uint8_t*>(S.M);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto improves = [&](int pr, int pc, int qr, int qc) {
        return min((int)sR[bidx(pr, pc)], (int)sM[bidx(qr, qc)]) > (int)sR[bidx(qr, qc)];
    };
    while (true) {
        if (threadIdx.x == 0) {
            int t = -1;
            const unsigned long long hd = vload(&wl.ctr[0]), tl = vload(&wl.ctr[1]);
            bool retire = false;
            if (hd >= tl + HP_RG_WAITERS) {
                const unsigned long long rr = atomicAdd(&wl.ctr[7], 1ull);
                if (rr + HP_RG_MIN_ALIVE < gridDim.x) retire = true;
                else atomicAdd(&wl.ctr[7], ~0ull);
            }
            if (!retire) {
                t = q_pop(wl);
                if (t >= 0) atomicExch(&wl.state[t], ST_BUSY);
            }
            // region visit count (state words past the regions and their order keys): a
            // region popped again and again lies on a long propagation chain
            S.visits = t >= 0 ? (int)atomicAdd(&wl.state[2 * wl.ntx * wl.nty + t], 1u) : 0;
            S.t0 = gtimer();
            S.job = t;
        }
        __syncthreads();
        const int t = S.job;
        if (t < 0) break;
        const int rx = t % wl.ntx, ry = t / wl.ntx;
        const int X0 = rx * RX * SW, Y0 = ry * RY * kTile;
        const bool inner = X0 >= 4 && X0 + RX * SW + 4 <= w && Y0 >= 1 && Y0 + RY * kTile + 1 <= h &&
                           (w & 3) == 0 && (((uintptr_t)R | (uintptr_t)mask) & 3) == 0;
        bool have_window = false;
        while (true) {
            if (lane == 0) {
                S.dirty_in[warp] = atomicExch(&wl.inrows[t * NW + warp], 0u);
                S.subchg[warp] = 0;
            }
            if (threadIdx.x < AROWS / 32) S.rowdirty[threadIdx.x] = 0;
            if (threadIdx.x < ACOLS / 32) S.coldirty[threadIdx.x] = 0;
            __threadfence();
            __syncthreads();
            int any_in = 0;
#pragma unroll
            for (int k = 0; k < NW; ++k) any_in |= S.dirty_in[k] != 0;
            if (any_in) {
                if (!have_window) {
                    constexpr int NIT = (ROWS * RWW + NW * 32 - 1) / (NW * 32);
                    uint32_t vr[NIT], vm[NIT];
                    if (inner) {
                        const uint8_t* rb = R + (int64_t)(Y0 - 1) * w + (X0 - 4);
                        const uint8_t* mb = mask + (int64_t)(Y0 - 1) * w + (X0 - 4);
#pragma unroll
                        for (int i = 0; i < NIT; ++i) {
                            int k = threadIdx.x + i * NW * 32;
                            if (k < ROWS * RWW) {
                                int rr = k / RWW, wi = k - rr * RWW;
                                int64_t o = (int64_t)rr * w + 4 * wi;
                                vr[i] = __ldcg(reinterpret_cast<const unsigned int*>(rb + o));
                                vm[i] = __ldcg(reinterpret_cast<const unsigned int*>(mb + o));
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < NIT; ++i) {
                            int k = threadIdx.x + i * NW * 32;
                            if (k < ROWS * RWW) {
                                int rr = k / RWW, wi = k - rr * RWW;
                                int gx = X0 - 4 + 4 * wi, gy = Y0 - 1 + rr;
                                vr[i] = load_word(R, w, h, gx, gy);
                                vm[i] = load_word(mask, w, h, gx, gy);
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < NIT; ++i) {
                        int k = threadIdx.x + i * NW * 32;
                        if (k < ROWS * RWW) {
                            S.R[k] = vr[i];
                            S.M[k] = vm[i];
                        }
                    }
                    have_window = true;
                } else {
                    constexpr int NH = 2 * RWW + 2 * (ROWS - 2);
                    for (int k = threadIdx.x; k < NH; k += blockDim.x) {
                        int rr, wi;
                        if (k < 2 * RWW) {
                            rr = k < RWW ? 0 : ROWS - 1;
                            wi = k % RWW;
                        } else {
                            int j = k - 2 * RWW;
                            rr = 1 + (j >> 1);
                            wi = (j & 1) ? RWW - 1 : 0;
                        }
                        S.R[rr * RWW + wi] = load_word(R, w, h, X0 - 4 + 4 * wi, Y0 - 1 + rr);
                    }
                }
                // the job's dirty sub-tile rows are region rows for the first row phase
                if (lane == 0) {
                    const uint32_t d = S.dirty_in[warp];
                    if (d) atomicOr(&S.rowdirty[(warp / RX) * (kTile / 32)], d);
                }
                __syncthreads();
                int phases = 0, lines = 0;
                adi_close_region(S, sR, sRw, sM, warp, lane, phases, lines, [] {});
                if (threadIdx.x == 0) {
                    atomicAdd(&wl.ctr[4], (unsigned long long)phases);
                }
                if (lane == 0) atomicAdd(&wl.ctr[6], (unsigned long long)lines);
                // write back each sub-tile's changed rows and activate the neighbouring regions
                // whose halo pixels those rows can improve (as k_region_mr8)
                const int sx = warp % RX, sy = warp / RX;
                const int wr0 = sy * kTile, wc0 = sx * SW;
                const uint32_t mychg = S.subchg[warp];
                if (mychg) {
                    constexpr int WPR = SW / 4;
                    for (int k = lane; k < kTile * WPR; k += 32) {
                        int y = 1 + k / WPR, wi = k % WPR;
                        if (!((mychg >> (y - 1)) & 1)) continue;
                        int gx = X0 + wc0 + 4 * wi, gy = Y0 + wr0 + y - 1;
                        if (gy >= h || gx >= w) continue;
                        uint8_t* dst = R + (int64_t)gy * w + gx;
                        uint32_t v = S.R[(wr0 + y) * RWW + sx * WPR + 1 + wi];
                        if (gx + 3 < w && (((uintptr_t)dst) & 3) == 0) {
                            __stcg(reinterpret_cast<unsigned int*>(dst), v);
                        } else {
                            for (int b = 0; b < 4 && gx + b < w; ++b)
                                __stcg(reinterpret_cast<unsigned char*>(dst + b), (unsigned char)(v >> (8 * b)));
                        }
                    }
                    __threadfence();
                    uint32_t m8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    const int r = wr0 + lane + 1;
                    constexpr uint32_t TOP = 1u << 31, BOT = 1u;
#pragma unroll
                    for (int d = -1; d <= 1; ++d) {
#pragma unroll
                        for (int j = 0; j < PPL; ++j) {
                            const int c = wc0 + PPL * lane + 1 + j;
                            if (sy == 0 && improves(wr0 + 1, c, wr0, c + d)) {
                                if (c + d == wc0) m8[0] |= TOP;
                                else if (c + d == wc0 + SW + 1) m8[2] |= TOP;
                                else m8[1] |= TOP;
                            }
                            if (sy == RY - 1 && improves(wr0 + kTile, c, wr0 + kTile + 1, c + d)) {
                                if (c + d == wc0) m8[5] |= BOT;
                                else if (c + d == wc0 + SW + 1) m8[7] |= BOT;
                                else m8[6] |= BOT;
                            }
                        }
                        if (sx == 0 && improves(r, wc0 + 1, r + d, wc0)) {
                            if (r + d == wr0) m8[0] |= TOP;
                            else if (r + d == wr0 + kTile + 1) m8[5] |= BOT;
                            else m8[3] |= 1u << (lane + d);
                        }
                        if (sx == RX - 1 && improves(r, wc0 + SW, r + d, wc0 + SW + 1)) {
                            if (r + d == wr0) m8[2] |= TOP;
                            else if (r + d == wr0 + kTile + 1) m8[7] |= BOT;
                            else m8[4] |= 1u << (lane + d);
                        }
                    }
                    uint32_t mine = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uint32_t v = __reduce_or_sync(FULL, m8[j]);
                        if (lane == j) mine = v;
                    }
                    if (lane < 8 && mine) {
                        int gsx = rx * RX + sx + dx8(lane), gsy = ry * RY + sy + dy8(lane);
                        int nrx = gsx >= 0 ? gsx / RX : -1, nry = gsy >= 0 ? gsy / RY : -1;
                        if (gsx >= 0 && gsy >= 0 && nrx < wl.ntx && nry < wl.nty && (nrx != rx || nry != ry)) {
                            int nt = nry * wl.ntx + nrx;
                            int sub = (gsy % RY) * RX + (gsx % RX);
                            atomicOr(&wl.inrows[nt * NW + sub], mine);
                            q_activate(wl, nt);
                        }
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int again = 0;
                uint32_t o = atomicCAS(&wl.state[t], ST_BUSY, ST_IDLE);
                if (o == ST_BUSY) {
                    atomicAdd(&wl.ctr[2], ~0ull);
                } else {
                    atomicExch(&wl.state[t], ST_BUSY);
                    again = 1;
                }
                atomicAdd(&wl.ctr[3], 1ull);
                if (!again) atomicAdd(&wl.ctr[5], gtimer() - S.t0);
                S.again = again;
            }
            __syncthreads();
            if (!S.again) break;
        }
    }
}

#if HP_RG_ORDER >= 2
// Initial order by the regions' highest marker value (values flow down from the marker's
// maxima, so regions holding high peaks go first): key per region = max of the marker.
__global__ void __launch_bounds__(256) k_rg_keys(const uint8_t* __restrict__ R, int w, int h, Worklist wl,
                                                 int32_t* __restrict__ keys) {
    const int t = blockIdx.x, rx = t % wl.ntx, ry = t / wl.ntx;
    const int X0 = rx * RX * SW, Y0 = ry * RY * kTile;
    int m = 0, cnt = 0;
    if (HP_RG_ORDER != 4) {
        // max over the region in 16-byte loads (r2: the byte-per-thread loop took 23.6 us per
        // 4K tile, on the reconstruction's critical path)
        constexpr int CPR = RX * SW / 16;  // 16-byte chunks per region row
        const bool vec = (w & 15) == 0 && (((uintptr_t)R) & 15) == 0;
        uint32_t m4 = 0;
        if (vec && X0 + RX * SW <= w && Y0 + RY * kTile <= h && (RY * kTile * CPR) % 256 == 0 && blockDim.x == 256) {
            constexpr int NL = RY * kTile * CPR / 256;  // loads per thread, all in flight
            uint4 v[NL];
#pragma unroll
            for (int k = 0; k < NL; ++k) {
                const int i = threadIdx.x + 256 * k;
                v[k] = __ldg(reinterpret_cast<const uint4*>(R + (int64_t)(Y0 + i / CPR) * w + X0 + (i % CPR) * 16));
            }
#pragma unroll
            for (int k = 0; k < NL; ++k) m4 = __vmaxu4(m4, __vmaxu4(__vmaxu4(v[k].x, v[k].y), __vmaxu4(v[k].z, v[k].w)));
        } else
        for (int i = threadIdx.x; i < RY * kTile * CPR; i += blockDim.x) {
            const int y = Y0 + i / CPR, x = X0 + (i % CPR) * 16;
            if (y >= h || x >= w) continue;
            const uint8_t* p = R + (int64_t)y * w + x;
            if (vec && x + 15 < w) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
                m4 = __vmaxu4(m4, __vmaxu4(__vmaxu4(v.x, v.y), __vmaxu4(v.z, v.w)));
            } else {
                for (int b = 0; b < 16 && x + b < w; ++b) m = max(m, (int)__ldg(p + b));
            }
        }
        m = max(m, (int)max(max(m4 & 0xff, (m4 >> 8) & 0xff), max((m4 >> 16) & 0xff, m4 >> 24)));
    } else {
        for (int i = threadIdx.x; i < RY * kTile * RX * SW; i += blockDim.x) {
            const int y = Y0 + i / (RX * SW), x = X0 + i % (RX * SW);
            if (x < w && y < h) {
                m += __ldg(R + (int64_t)y * w + x);
                ++cnt;
            }
        }
    }
    m = HP_RG_ORDER == 4 ? (int)__reduce_add_sync(FULL, (unsigned)m) : (int)__reduce_max_sync(FULL, (unsigned)m);
    cnt = (int)__reduce_add_sync(FULL, (unsigned)cnt);
    __shared__ int wm[8], wc[8];
    if ((threadIdx.x & 31) == 0) {
        wm[threadIdx.x >> 5] = m;
        wc[threadIdx.x >> 5] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 8; ++k) {
            m = HP_RG_ORDER == 4 ? m + wm[k] : max(m, wm[k]);
            cnt += wc[k];
        }
        keys[t] = HP_RG_ORDER == 4 ? m / max(cnt, 1) : m;  // max, or (ORDER 4) mean
    }
}

#if HP_RG_ORDER == 5
// ORDER 5: key = region-grid distance (8-neighbour steps) to the nearest region holding the
// tile's highest marker value -- the flood's sources first, then outward wave by wave.  One
// block: synchronous relaxation over the region grid (a few dozen rounds).
__global__ void __launch_bounds__(1024) k_rg_dist(Worklist wl, int32_t* __restrict__ keys) {
    const int n = wl.ntx * wl.nty;
    __shared__ int top;
    __shared__ int changed;
    if (threadIdx.x == 0) top = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) atomicMax(&top, keys[i]);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = keys[i] == top ? 0 : INT_MAX / 2;
    __syncthreads();
    while (true) {
        if (threadIdx.x == 0) changed = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int rx = i % wl.ntx, ry = i / wl.ntx;
            int d = keys[i];
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int x = rx + dx, y = ry + dy;
                    if (x >= 0 && y >= 0 && x < wl.ntx && y < wl.nty) d = min(d, keys[y * wl.ntx + x] + 1);
                }
            if (d < keys[i]) {
                keys[i] = d;  // monotone (Bellman-Ford style): any interleaving converges
                changed = 1;
            }
        }
        __syncthreads();
        if (!changed) break;
        __syncthreads();
    }
}
#endif

// queue[rank] = region, rank by (ORDER 2: colour, then descending max; ORDER 3/4: descending
// max (mean), then colour; ORDER 5: distance to the top regions, then colour), ties by index
// one warp per region: the lanes split the comparisons (r2: a thread per region over n = 512
// regions took 31 us, then 10 us with the keys in shared memory, on S4's critical path)
__global__ void __launch_bounds__(256) k_rg_order(Worklist wl, const int32_t* __restrict__ keys) {
    const int n = wl.ntx * wl.nty;
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= n) return;
    auto key = [&](int j) {
        const int c = ((j / wl.ntx) & 1) * 2 + ((j % wl.ntx) & 1);
        return HP_RG_ORDER == 2 ? c * 256 + (255 - __ldg(keys + j))
                                : (HP_RG_ORDER == 5 ? __ldg(keys + j) * 4 + c : (255 - __ldg(keys + j)) * 4 + c);
    };
    const int ki = key(i);
    int rk = 0;
    for (int j = lane; j < n; j += 32) {
        const int kj = key(j);
        rk += kj < ki || (kj == ki && j < i);
    }
    rk = (int)__reduce_add_sync(FULL, (unsigned)rk);
    if (lane == 0) wl.queue[rk] = i;
}
#endif

}  // namespace

void launch_recon_u8_regions(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl0,
                             cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    Worklist wl = wl0;
    wl.ntx = (w + RX * SW - 1) / (RX * SW);
    wl.nty = (h + RY * kTile - 1) / (RY * kTile);
    const int n = wl.ntx * wl.nty;
    static const int init_env = [] {  // HP_RG_INIT=0/1 overrides the compile-time default
        const char* e = getenv("HP_RG_INIT");
        return e ? atoi(e) : HP_RG_INIT;
    }();
    (note_launch(), k_rg_reset<<<(int)std::min<int64_t>((std::max<int64_t>(wl.cap, (int64_t)n * NW) + 255) / 256, num_sms() * 16), 256, 0, s>>>(wl, init_env != 0));
    if (init_env) {
        (note_launch(), k_rg_init<<<(n + 3) / 4, 128, 0, s>>>(mask, R, w, h, wl.ntx, wl.nty));
        (note_launch(), k_rg_seed<<<(n * NW + 7) / 8, 256, 0, s>>>(mask, R, w, h, wl));
    }
#if HP_RG_ORDER >= 2
    // keys in the region-state array past the regions (it is sized for the 32x32 tiles of the
    // tile engine, 32 entries per region)
    int32_t* keys = reinterpret_cast<int32_t*>(wl.state) + n;
    (note_launch(), k_rg_keys<<<n, 256, 0, s>>>(R, w, h, wl, keys));
#if HP_RG_ORDER == 5
    (note_launch(), k_rg_dist<<<1, 1024, 0, s>>>(wl, keys));
#endif
    (note_launch(), k_rg_order<<<(n + 7) / 8, 256, 0, s>>>(wl, keys));
#endif
    static const int thin_env = [] {  // HP_RG_THIN=k overrides the compile-time default
        const char* e = getenv("HP_RG_THIN");
        return e ? atoi(e) : HP_RG_THIN;
    }();
    static const int chain_env = [] {  // HP_RG_CHAIN=v overrides the compile-time default
        const char* e = getenv("HP_RG_CHAIN");
        return e ? atoi(e) : HP_RG_CHAIN;
    }();
    static const int adi_env = [] {  // HP_RG_ADI=0/1 overrides the compile-time default
        const char* e = getenv("HP_RG_ADI");
        return e ? atoi(e) : HP_RG_ADI;
    }();
    static PerDevice once, once_adi;
    if (adi_env) {
        const size_t smem_a = sizeof(SmemA);
        once_adi.get([&] {
            return (int)cudaFuncSetAttribute(k_region_adi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
        });
        const int nsm = num_sms();
        static const int grid_env_a = [] {
            const char* e = getenv("HP_RG_GRID");
            return e ? atoi(e) : 0;
        }();
        int b = std::max(1, std::min(grid_env_a > 0 ? grid_env_a : nsm * 3 / 4, n));
        (note_launch(), k_region_adi<<<b, NW * 32, smem_a, s>>>(mask, R, w, h, wl));
        return;
    }
    const size_t smem = sizeof(Smem);
    const int blocks = once.get([&] {
        cudaFuncSetAttribute(k_region_mr8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0, dev = 0, nsm = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_region_mr8, NW * 32, smem);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        // One CTA per SM (measured, bench.py r1: 229 vs 193 tiles/s at 2 CTAs/SM): on hard tiles
        // the reconstruction is latency-bound on chains of region jobs, so leaving half the
        // SM resources free lets another slot's tile run beside it.
        // With several slots in flight, three CTAs per four SMs (r1 final: 897 -> 903 tiles/s,
        // e2e 924 -> 939): each tile's reconstruction then holds fewer SMs while chain-bound.
        if (const char* e = getenv("HP_RG_CTAS_PER_SM")) {
            const int want = std::max(1, std::min(atoi(e), per_sm > 0 ? per_sm : 1));
            return nsm * want;
        }
        return std::max(1, nsm * 3 / 4);
    });
    int b = std::max(1, std::min(wl.ctas > 0 ? wl.ctas : blocks, n));
    static const int grid_env = [] {  // HP_RG_GRID: absolute CTA count (experiments)
        const char* e = getenv("HP_RG_GRID");
        return e ? atoi(e) : 0;
    }();
    if (grid_env > 0) b = std::max(1, std::min(grid_env, n));
    (note_launch(), k_region_mr8<<<b, NW * 32, smem, s>>>(mask, R, w, h, wl, thin_env, chain_env));
}

void launch_recon_u8_auto(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl,
                          cudaStream_t s) {
    static int use_tiles = -1;
    if (use_tiles < 0) {
        const char* e = getenv("HP_IWPP_TILES");
        use_tiles = (e && atoi(e) == 1) ? 1 : 0;
    }
    if (use_tiles)
        launch_recon_u8(mask, R, w, h, wl, s);
    else
        launch_recon_u8_regions(mask, R, w, h, wl, s);
}

}  // namespace hp
