// iwpp_rules.cuh -- per-tile local solvers of the IWPP engine (included by k_iwpp.cu).
//
// Each rule loads the 34x34 window (tile + halo) of its planes into the warp's shared
// memory, closes the tile by Gauss-Seidel row sweeps, writes the tile back if anything
// changed, and returns the neighbour tiles whose halo pixels it can still improve.
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
// may be unstable -- initially all rows; afterwards only rows next to a row that changed
// after they were last closed (rows depend only on themselves, the rows above and below,
// and the fixed halo).  A cheap per-row test skips rows that cannot change.
#pragma once

namespace hp {
namespace {

template <class RowFn>
__device__ __forceinline__ bool sweep_rows(RowFn row, int* npasses) {
    uint32_t dirty = 0xffffffffu;
    bool any = false;
    int passes = 0;
    while (dirty) {
        for (int y = 1; y <= kTile; ++y) {  // raster direction
            const uint32_t bit = 1u << (y - 1);
            if (!(dirty & bit)) continue;
            dirty &= ~bit;
            if (row(y)) {
                any = true;
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
                any = true;
                dirty |= (bit << 1) | (bit >> 1);
            }
        }
        ++passes;
    }
    *npasses = passes;
    return any;
}

// Morphological reconstruction by dilation.  T = int (u8 planes, -1 = absent) or float
// (-inf = absent: outside the image or outside the domain).
template <class T, class PT>
struct RuleMR {
    static constexpr int kWords = 2 * kHalo * P;
    const PT* mask;
    PT* R;
    const uint8_t* dom;  // may be null
    int w, h;
    __device__ static T neg();

    __device__ uint32_t process(int x0, int y0, T* sm, int lane, unsigned long long* rounds) const {
        T* sR = sm;
        T* sM = sm + kHalo * P;
        TileGeo g{x0, y0, w, h};
        // all loads of the 34x34 window issued back to back (17 rows per batch) so their
        // L2 latencies overlap; lanes 0/1 also fetch the two right-most halo columns
        auto load = [&](int r, int cc, T& rv, T& mv) {
            rv = neg();
            mv = neg();
            if (cc < kHalo && g.inimg(r, cc)) {
                int64_t i = g.gidx(r, cc);
                if (dom == nullptr || ldcg(dom + i)) {
                    rv = (T)ldcg(R + i);
                    mv = (T)ldcg(mask + i);
                }
            }
        };
#pragma unroll
        for (int r0 = 0; r0 < kHalo; r0 += 17) {
            T rv[17], mv[17];
#pragma unroll
            for (int k = 0; k < 17; ++k) load(r0 + k, lane, rv[k], mv[k]);
#pragma unroll
            for (int k = 0; k < 17; ++k) {
                sR[(r0 + k) * P + lane] = rv[k];
                sM[(r0 + k) * P + lane] = mv[k];
            }
        }
        if (lane < 2) {
            for (int r = 0; r < kHalo; ++r) {
                T rv, mv;
                load(r, 32 + lane, rv, mv);
                sR[r * P + 32 + lane] = rv;
                sM[r * P + 32 + lane] = mv;
            }
        }
        __syncwarp();
        const int c = lane + 1;
        auto row = [&](int y) -> bool {
            T m = sM[y * P + c], rr = sR[y * P + c];
            T vmax = tmax(tmax(sR[(y - 1) * P + c - 1], tmax(sR[(y - 1) * P + c], sR[(y - 1) * P + c + 1])),
                          tmax(sR[(y + 1) * P + c - 1], tmax(sR[(y + 1) * P + c], sR[(y + 1) * P + c + 1])));
            T lft = sR[y * P + c - 1], rgt = sR[y * P + c + 1];
            // stable iff every pixel is already >= min(mask, max of its N8); else it changes
            if (!__any_sync(FULL, tmin(tmax(vmax, tmax(lft, rgt)), m) > rr)) return false;
            T b = tmax(rr, vmax);
            if (lane == 0) b = tmax(b, lft);
            if (lane == 31) b = tmax(b, rgt);
            T lo = tmin(b, m);
            T u = tmax(clamp_scan_lr<T>(lo, m, lane), clamp_scan_rl<T>(lo, m, lane));
            __syncwarp();
            if (u != rr) sR[y * P + c] = u;
            __syncwarp();
            return true;
        };
        int npass = 0;
        const bool changed_any = sweep_rows(row, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
        if (changed_any) {
            for (int r = 1; r <= kTile; ++r) {
                if (!g.inimg(r, c)) continue;
                T m = sM[r * P + c];
                if (m == neg()) continue;  // outside the domain: never written
                stcg(R + g.gidx(r, c), (PT)sR[r * P + c]);
            }
        }
        return border_scan(lane, [&](int pr, int pc, int qr, int qc) {
            T qm = sM[qr * P + qc];
            if (qm == neg()) return false;
            return tmin(sR[pr * P + pc], qm) > sR[qr * P + qc];
        });
    }
};
template <>
__device__ int RuleMR<int, uint8_t>::neg() { return -1; }
template <>
__device__ float RuleMR<float, float>::neg() { return -INFINITY; }

// W2: least fixed point of d(p) = min(d(p), 1 + d(q)) over N8 neighbours q with c(q) ==
// c(p) (c is NaN outside F, so no edge leaves F).  Initial d: 0 markers, 1 pixels with a
// higher neighbour, inf otherwise (k_d_init).
struct RuleW2 {
    static constexpr int kWords = 2 * kHalo * P;
    const float* cpl;
    int32_t* d;
    int w, h;
    __device__ uint32_t process(int x0, int y0, int* sm, int lane, unsigned long long* rounds) const {
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
        int npass = 0;
        const bool changed_any = sweep_rows(row, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
        if (changed_any)
            for (int r = 1; r <= kTile; ++r)
                if (g.inimg(r, c) && sC[r * P + c] == sC[r * P + c]) stcg(d + g.gidx(r, c), sD[r * P + c]);
        return border_scan(lane, [&](int pr, int pc, int qr, int qc) {
            float cq = sC[qr * P + qc];
            return cq == sC[pr * P + pc] && sat_add(sD[pr * P + pc], 1) < sD[qr * P + qc];
        });
    }
};

// W3: least fixed point (from +inf) of L(p) = min(L(p), L(q)) over the parents q of p
// (bit j of pm[p] <-> neighbour (dx8(j), dy8(j))).  Markers have no parents.
struct RuleW3 {
    static constexpr int kWords = 2 * kHalo * P;
    const uint8_t* pm;
    int32_t* L;
    int w, h;
    __device__ uint32_t process(int x0, int y0, int* sm, int lane, unsigned long long* rounds) const {
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
        int npass = 0;
        const bool changed_any = sweep_rows(row, &npass);
        if (lane == 0 && rounds) atomicAdd(rounds, (unsigned long long)npass);
        if (changed_any)
            for (int r = 1; r <= kTile; ++r)
                if (g.inimg(r, c) && sP[r * P + c]) stcg(L + g.gidx(r, c), sL[r * P + c]);
        return border_scan(lane, [&](int pr, int pc, int qr, int qc) {
            int pmq = sP[qr * P + qc];
            if (!pmq) return false;
            int j = nb_index(pc - qc, pr - qr);  // direction q -> p
            return ((pmq >> j) & 1) && sL[pr * P + pc] < sL[qr * P + qc];
        });
    }
};

}  // namespace
}  // namespace hp
