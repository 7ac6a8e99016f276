// iwpp_rules.cuh -- per-tile local solvers of the IWPP engine (included by k_iwpp.cu).
//
// Each rule loads the 34x34 window (tile + halo) of its planes into the warp's shared
// memory, closes the tile by Gauss-Seidel row sweeps, writes back the rows that changed,
// and reports, per neighbour tile, the rows of that tile whose halo it can still improve.
//
// Row closure: within one row every rule's update is a 1-D function chain
//   MR:  f_x(t) = min(mask_x, max(b_x, t))             (clamp)
//   W2:  f_x(t) = min(a_x, t + k_x), k_x in {1, inf}    (min-plus along equal-c edges)
//   W3:  f_x(t) = min(a_x, t + k_x), k_x in {0, inf}    (min along parent edges)
// where b_x / a_x already hold the contributions of the rows above and below and of the
// halo columns.  The closure of the row is the better of a left-to-right and a right-to-left
// inclusive scan of these functions, both taken on the same input, so the two Kogge-Stone
// scans (5 shuffle levels each) are independent and interleave.
//
// Sweep driver: a 32-bit dirty mask (bit y-1 <-> row y).  A row is (re)closed only if it
// may be unstable: on a tile's first job all rows; on a re-activation only the rows whose
// halo neighbours improved (the activating tile ORs them into the tile's inrows word); and
// afterwards rows next to a row that changed after they were last closed (a row depends
// only on itself, the rows above and below, and the fixed halo).  A cheap per-row test
// skips rows that cannot change.
#pragma once

namespace hp {
namespace {

// neighbour-tile indices (nb_index order)
constexpr int NB_UL = 0, NB_U = 1, NB_UR = 2, NB_L = 3, NB_R = 4, NB_DL = 5, NB_D = 6, NB_DR = 7;

template <class RowFn>
__device__ __forceinline__ bool sweep_rows(RowFn row, uint32_t dirty, uint32_t* changed_rows,
                                           int* npasses) {
    uint32_t chg = 0;
    int passes = 0;
    while (dirty) {
        for (int y = 1; y <= kTile; ++y) {  // raster direction
            const uint32_t bit = 1u << (y - 1);
            if (!(dirty & bit)) continue;
            dirty &= ~bit;
            if (row(y)) {
                chg |= bit;
                dirty |= (bit << 1) | (bit >> 1);
            }
        }
        ++passes;
        if (!dirty) break;
        for (int y = kTile; y >= 1; --y) {  // anti-raster direction
            const uint32_t bit = 1u << (y - 1);
            if (!(dirty & bit)) continue;
            dirty &= ~bit;
            if (row(y)) {
                chg |= bit;
                dirty |= (bit << 1) | (bit >> 1);
            }
        }
        ++passes;
    }
    *changed_rows = chg;
    *npasses = passes;
    return chg != 0;
}

// For each interior border pixel p and each of its halo neighbours q, f(pr, pc, qr, qc)
// tells whether p can improve q; out[nb] collects the rows (bit r-1, in the neighbour's own
// row numbering) of neighbour tile nb that received such an improvement.
template <class F>
__device__ __forceinline__ void border_masks(int lane, F f, uint32_t (&out)[8]) {
    uint32_t m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int c = lane + 1;
    constexpr uint32_t TOP = 1u << 31, BOT = 1u;
#pragma unroll
    for (int d = -1; d <= 1; ++d) {
        const int qc = c + d;
        if (f(1, c, 0, qc)) {  // top row -> neighbour's last row
            if (qc == 0) m[NB_UL] |= TOP;
            else if (qc == kHalo - 1) m[NB_UR] |= TOP;
            else m[NB_U] |= TOP;
        }
        if (f(kTile, c, kHalo - 1, qc)) {  // bottom row -> neighbour's first row
            if (qc == 0) m[NB_DL] |= BOT;
            else if (qc == kHalo - 1) m[NB_DR] |= BOT;
            else m[NB_D] |= BOT;
        }
        const int r = lane + 1, qr = r + d;
        if (f(r, 1, qr, 0)) {  // left column
            if (qr == 0) m[NB_UL] |= TOP;
            else if (qr == kHalo - 1) m[NB_DL] |= BOT;
            else m[NB_L] |= 1u << (qr - 1);
        }
        if (f(r, kTile, qr, kHalo - 1)) {  // right column
            if (qr == 0) m[NB_UR] |= TOP;
            else if (qr == kHalo - 1) m[NB_DR] |= BOT;
            else m[NB_R] |= 1u << (qr - 1);
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = __reduce_or_sync(FULL, m[j]);
}

// ------------------------------------------------------------------ MR on u8 planes
// Window kept as bytes: row r of the window = 10 words = global bytes [x0-4, x0+36), so
// window column c (0..33) is byte c+3 and the tile interior is words 1..8 -- the window is
// moved with aligned 32-bit loads/stores.  Pixels outside the image read as mask 0 / R 0,
// which is neutral for a max-min propagation of non-negative values.
struct RuleMR8 {
    static constexpr int kRowW = 10;                   // words per window row
    static constexpr int kWords = 2 * kHalo * kRowW;   // two planes
    const uint8_t* mask;
    uint8_t* R;
    int w, h;

    __device__ __forceinline__ uint32_t load_word(const uint8_t* plane, int gx, int gy) const {
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

    __device__ bool process(int x0, int y0, int* smi, int lane, uint32_t dirty0,
                            unsigned long long* rounds, uint32_t (&nbm)[8]) const {
        uint32_t* wR = reinterpret_cast<uint32_t*>(smi);
        uint32_t* wM = wR + kHalo * kRowW;
        const uint8_t* sR = reinterpret_cast<const uint8_t*>(wR);
        uint8_t* sRw = reinterpret_cast<uint8_t*>(wR);
        const uint8_t* sM = reinterpret_cast<const uint8_t*>(wM);
        constexpr int RB = kRowW * 4;  // bytes per window row
        for (int k = lane; k < kHalo * kRowW; k += 32) {
            int r = k / kRowW, wi = k - r * kRowW;
            int gx = x0 - 4 + 4 * wi, gy = y0 - 1 + r;
            wR[k] = load_word(R, gx, gy);
            wM[k] = load_word(mask, gx, gy);
        }
        __syncwarp();
        const int cb = lane + 4;  // byte of this lane's column (window column lane+1)
        auto row = [&](int y) -> bool {
            int m = sM[y * RB + cb], rr = sR[y * RB + cb];
            int up = max(max(sR[(y - 1) * RB + cb - 1], sR[(y - 1) * RB + cb]), sR[(y - 1) * RB + cb + 1]);
            int dn = max(max(sR[(y + 1) * RB + cb - 1], sR[(y + 1) * RB + cb]), sR[(y + 1) * RB + cb + 1]);
            int vmax = max(up, dn);
            int lft = sR[y * RB + cb - 1], rgt = sR[y * RB + cb + 1];
            if (!__any_sync(FULL, min(max(vmax, max(lft, rgt)), m) > rr)) return false;
            int b = max(rr, vmax);
            if (lane == 0) b = max(b, lft);
            if (lane == 31) b = max(b, rgt);
            int lo = min(b, m);
            int u = max(clamp_scan_lr<int>(lo, m, lane), clamp_scan_rl<int>(lo, m, lane));
            __syncwarp();
            if (u != rr) sRw[y * RB + cb] = (uint8_t)u;
            __syncwarp();
            return true;
        };
        uint32_t chg = 0;
        int npass = 0;
        const bool changed = sweep_rows(row, dirty0, &chg, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
#pragma unroll
        for (int j = 0; j < 8; ++j) nbm[j] = 0;
        if (!changed) return false;  // nothing new to publish (halo values only grow)
        // write back the changed rows: interior = words 1..8 of window rows 1..32
        for (int k = lane; k < kTile * 8; k += 32) {
            int r = 1 + (k >> 3), wi = 1 + (k & 7);
            if (!((chg >> (r - 1)) & 1)) continue;
            int gx = x0 + 4 * (wi - 1), gy = y0 + r - 1;
            if (gy >= h || gx >= w) continue;
            uint8_t* dst = R + (int64_t)gy * w + gx;
            uint32_t v = wR[r * kRowW + wi];
            if (gx + 3 < w && (((uintptr_t)dst) & 3) == 0) {
                __stcg(reinterpret_cast<unsigned int*>(dst), v);
            } else {
                for (int b = 0; b < 4 && gx + b < w; ++b)
                    __stcg(reinterpret_cast<unsigned char*>(dst + b), (unsigned char)(v >> (8 * b)));
            }
        }
        border_masks(lane, [&](int pr, int pc, int qr, int qc) {
            return min((int)sR[pr * RB + pc + 3], (int)sM[qr * RB + qc + 3]) > (int)sR[qr * RB + qc + 3];
        }, nbm);
        return true;
    }
};

// ------------------------------------------------------------------ MR on f32 planes
// Domain-restricted (dom != null): pixels outside the domain or the image are -inf.
struct RuleMRf {
    static constexpr int kWords = 2 * kHalo * P;
    const float* mask;
    float* R;
    const uint8_t* dom;  // may be null
    int w, h;

    __device__ bool process(int x0, int y0, int* smi, int lane, uint32_t dirty0,
                            unsigned long long* rounds, uint32_t (&nbm)[8]) const {
        float* sR = reinterpret_cast<float*>(smi);
        float* sM = sR + kHalo * P;
        TileGeo g{x0, y0, w, h};
        auto ld = [&](int r, int cc) {
            float rv = -INFINITY, mv = -INFINITY;
            if (g.inimg(r, cc)) {
                int64_t i = g.gidx(r, cc);
                if (dom == nullptr || ldcg(dom + i)) {
                    rv = ldcg(R + i);
                    mv = ldcg(mask + i);
                }
            }
            sR[r * P + cc] = rv;
            sM[r * P + cc] = mv;
        };
#pragma unroll
        for (int r = 0; r < kHalo; ++r) ld(r, lane);
        if (lane < 2)
            for (int r = 0; r < kHalo; ++r) ld(r, 32 + lane);
        __syncwarp();
        const int c = lane + 1;
        auto row = [&](int y) -> bool {
            float m = sM[y * P + c], rr = sR[y * P + c];
            float vmax = fmaxf(fmaxf(sR[(y - 1) * P + c - 1], fmaxf(sR[(y - 1) * P + c], sR[(y - 1) * P + c + 1])),
                               fmaxf(sR[(y + 1) * P + c - 1], fmaxf(sR[(y + 1) * P + c], sR[(y + 1) * P + c + 1])));
            float lft = sR[y * P + c - 1], rgt = sR[y * P + c + 1];
            if (!__any_sync(FULL, fminf(fmaxf(vmax, fmaxf(lft, rgt)), m) > rr)) return false;
            float b = fmaxf(rr, vmax);
            if (lane == 0) b = fmaxf(b, lft);
            if (lane == 31) b = fmaxf(b, rgt);
            float lo = fminf(b, m);
            float u = fmaxf(clamp_scan_lr<float>(lo, m, lane), clamp_scan_rl<float>(lo, m, lane));
            __syncwarp();
            if (u != rr) sR[y * P + c] = u;
            __syncwarp();
            return true;
        };
        uint32_t chg = 0;
        int npass = 0;
        const bool changed = sweep_rows(row, dirty0, &chg, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
#pragma unroll
        for (int j = 0; j < 8; ++j) nbm[j] = 0;
        if (!changed) return false;
        for (int r = 1; r <= kTile; ++r) {
            if (!((chg >> (r - 1)) & 1) || !g.inimg(r, c)) continue;
            if (sM[r * P + c] == -INFINITY) continue;  // outside the domain: never written
            stcg(R + g.gidx(r, c), sR[r * P + c]);
        }
        border_masks(lane, [&](int pr, int pc, int qr, int qc) {
            float qm = sM[qr * P + qc];
            if (qm == -INFINITY) return false;
            return fminf(sR[pr * P + pc], qm) > sR[qr * P + qc];
        }, nbm);
        return true;
    }
};

// ------------------------------------------------------------------ W2
// Least fixed point of d(p) = min(d(p), 1 + d(q)) over N8 neighbours q with c(q) == c(p)
// (c is NaN outside F, so no edge leaves F).  Initial d: 0 markers, 1 pixels with a higher
// neighbour, inf otherwise (k_d_init).
struct RuleW2 {
    static constexpr int kWords = 2 * kHalo * P;
    const float* cpl;
    int32_t* d;
    int w, h;
    __device__ bool process(int x0, int y0, int* sm, int lane, uint32_t dirty0,
                            unsigned long long* rounds, uint32_t (&nbm)[8]) const {
        int* sD = sm;
        float* sC = reinterpret_cast<float*>(sm + kHalo * P);
        TileGeo g{x0, y0, w, h};
        auto ld = [&](int r, int cc) {
            int dv = kInfI;
            float cv = NAN;
            if (g.inimg(r, cc)) {
                int64_t i = g.gidx(r, cc);
                dv = ldcg(d + i);
                cv = ldcg(cpl + i);
            }
            sD[r * P + cc] = dv;
            sC[r * P + cc] = cv;
        };
#pragma unroll
        for (int r = 0; r < kHalo; ++r) ld(r, lane);
        if (lane < 2)
            for (int r = 0; r < kHalo; ++r) ld(r, 32 + lane);
        __syncwarp();
        const int c = lane + 1;
        auto row = [&](int y) -> bool {
            float cp = sC[y * P + c];
            int dp = sD[y * P + c];
            int a = kInfI, kl = kInfI, kr = kInfI;
            if (cp == cp) {  // in F
                a = dp;
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    if (sC[(y - 1) * P + c + dx] == cp) a = min(a, sat_add(sD[(y - 1) * P + c + dx], 1));
                    if (sC[(y + 1) * P + c + dx] == cp) a = min(a, sat_add(sD[(y + 1) * P + c + dx], 1));
                }
                if (lane == 0 && sC[y * P] == cp) a = min(a, sat_add(sD[y * P], 1));
                if (lane == 31 && sC[y * P + kHalo - 1] == cp) a = min(a, sat_add(sD[y * P + kHalo - 1], 1));
                if (lane > 0 && sC[y * P + c - 1] == cp) kl = 1;
                if (lane < 31 && sC[y * P + c + 1] == cp) kr = 1;
            }
            int aall = min(a, min(kl == 1 ? sat_add(sD[y * P + c - 1], 1) : kInfI,
                                  kr == 1 ? sat_add(sD[y * P + c + 1], 1) : kInfI));
            if (!__any_sync(FULL, aall < dp)) return false;  // stable row
            int u = min(minplus_scan_lr(a, kl, lane), minplus_scan_rl(a, kr, lane));
            __syncwarp();
            if (u < dp) sD[y * P + c] = u;
            __syncwarp();
            return true;
        };
        uint32_t chg = 0;
        int npass = 0;
        const bool changed = sweep_rows(row, dirty0, &chg, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
#pragma unroll
        for (int j = 0; j < 8; ++j) nbm[j] = 0;
        if (!changed) return false;
        for (int r = 1; r <= kTile; ++r)
            if (((chg >> (r - 1)) & 1) && g.inimg(r, c) && sC[r * P + c] == sC[r * P + c])
                stcg(d + g.gidx(r, c), sD[r * P + c]);
        border_masks(lane, [&](int pr, int pc, int qr, int qc) {
            float cq = sC[qr * P + qc];
            return cq == sC[pr * P + pc] && sat_add(sD[pr * P + pc], 1) < sD[qr * P + qc];
        }, nbm);
        return true;
    }
};

// ------------------------------------------------------------------ W3
// Least fixed point (from +inf) of L(p) = min(L(p), L(q)) over the parents q of p
// (bit j of pm[p] <-> neighbour (dx8(j), dy8(j))).  Markers have no parents.
struct RuleW3 {
    static constexpr int kWords = 2 * kHalo * P;
    const uint8_t* pm;
    int32_t* L;
    int w, h;
    __device__ bool process(int x0, int y0, int* sm, int lane, uint32_t dirty0,
                            unsigned long long* rounds, uint32_t (&nbm)[8]) const {
        int* sL = sm;
        int* sP = sm + kHalo * P;
        TileGeo g{x0, y0, w, h};
        auto ld = [&](int r, int cc) {
            int lv = kInfI, pv = 0;
            if (g.inimg(r, cc)) {
                int64_t i = g.gidx(r, cc);
                lv = ldcg(L + i);
                pv = ldcg(pm + i);
            }
            sL[r * P + cc] = lv;
            sP[r * P + cc] = pv;
        };
#pragma unroll
        for (int r = 0; r < kHalo; ++r) ld(r, lane);
        if (lane < 2)
            for (int r = 0; r < kHalo; ++r) ld(r, 32 + lane);
        __syncwarp();
        const int c = lane + 1;
        auto row = [&](int y) -> bool {
            int pmk = sP[y * P + c];
            int lp = sL[y * P + c];
            int a = lp, kl = kInfI, kr = kInfI;
            if (pmk) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (!((pmk >> j) & 1)) continue;
                    int dx = dx8(j), dy = dy8(j);
                    if (dy == 0) {
                        if (dx < 0 && lane > 0) { kl = 0; continue; }
                        if (dx > 0 && lane < 31) { kr = 0; continue; }
                    }
                    a = min(a, sL[(y + dy) * P + c + dx]);
                }
            }
            int aall = min(a, min(kl == 0 ? sL[y * P + c - 1] : kInfI, kr == 0 ? sL[y * P + c + 1] : kInfI));
            if (!__any_sync(FULL, aall < lp)) return false;  // stable row
            int u = min(minplus_scan_lr(a, kl, lane), minplus_scan_rl(a, kr, lane));
            __syncwarp();
            if (u < lp) sL[y * P + c] = u;
            __syncwarp();
            return true;
        };
        uint32_t chg = 0;
        int npass = 0;
        const bool changed = sweep_rows(row, dirty0, &chg, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
#pragma unroll
        for (int j = 0; j < 8; ++j) nbm[j] = 0;
        if (!changed) return false;
        for (int r = 1; r <= kTile; ++r)
            if (((chg >> (r - 1)) & 1) && g.inimg(r, c) && sP[r * P + c]) stcg(L + g.gidx(r, c), sL[r * P + c]);
        border_masks(lane, [&](int pr, int pc, int qr, int qc) {
            int pmq = sP[qr * P + qc];
            if (!pmq) return false;
            int j = nb_index(pc - qc, pr - qr);  // direction q -> p
            return ((pmq >> j) & 1) && sL[pr * P + pc] < sL[qr * P + qc];
        }, nbm);
        return true;
    }
};

}  // namespace
}  // namespace hp
