// feat_common.cuh -- per-object feature accumulation + fp64 finaliser (S11; definitions in
// DESIGN.md "Feature table"), shared by k_feat.cu (objects from a label plane) and k_comp.cu
// (objects of the fused per-component path).  Both translation units are compiled with
// -fmad=false so the finaliser rounds like its written formulas.
#pragma once

#include <cfloat>
#include <climits>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {
namespace {

constexpr int kFT = 256;  // threads per object CTA

// A "team" runs one object (or component): a whole CTA of kFT threads, or one warp.
// Reductions are fixed-order trees, so results are deterministic run to run.
struct TeamRed {
    long long l[kFT / 32];
    double d[kFT / 32];
    int i[kFT / 32];
};

template <int NT = kFT>
struct TeamCTA {
    static_assert(NT % 32 == 0 && NT <= kFT, "TeamRed holds one slot per warp of kFT threads");
    static constexpr int size = NT;
    __device__ __forceinline__ int rank() const { return threadIdx.x; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
    __device__ __forceinline__ int any(int b) const { return __syncthreads_or(b); }
    template <class T, class Op>
    __device__ __forceinline__ T reduce(T v, T* red, Op op) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        __syncthreads();
        if (lane == 0) red[warp] = v;
        __syncthreads();
        T r = red[0];
        for (int k = 1; k < NT / 32; ++k) r = op(r, red[k]);
        __syncthreads();
        return r;
    }
    // exclusive prefix sum over ranks (rank order)
    __device__ __forceinline__ long long scan_excl(long long v, long long* red) const {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        __syncthreads();
        if (lane == 31) red[warp] = inc;
        __syncthreads();
        long long off = 0;
        for (int k = 0; k < warp; ++k) off += red[k];
        __syncthreads();
        return off + inc - v;
    }
};

struct TeamWarp {
    static constexpr int size = 32;
    int lane;
    __device__ __forceinline__ int rank() const { return lane; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ __forceinline__ int any(int b) const { return __any_sync(0xffffffffu, b); }
    template <class T, class Op>
    __device__ __forceinline__ T reduce(T v, T*, Op op) const {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_down_sync(0xffffffffu, v, o));
        return __shfl_sync(0xffffffffu, v, 0);
    }
    __device__ __forceinline__ long long scan_excl(long long v, long long*) const {
        long long inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        return inc - v;
    }
};

struct OpAdd {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMin {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a < b ? a : b; }
};
struct OpMax {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

__device__ __forceinline__ int refl(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * n - 2 - i;
    }
    return i;
}

struct FeatSmem {
    double f[HP_NFEAT];  // team rank 0's 36 features (shared, not registers: r2 the per-thread
                         // array cost k_comp_fused 484 B of spills at its 128-register cap)
    unsigned int hist[256];
    unsigned int glcm[64];
    float gmin, gmax;
};

// Every thread of the team calls this for one object P = {(x, y) : inP(x, y)} inside the
// search box [bx0, bx1] x [by0, by1]; g is the tile's u8 plane (w x h, REFLECT_101 Sobel).
// Team rank 0 receives the 36 features in f and the border flag.  edge: the tile's Canny
// edge plane (0/1, reading C22).
template <class Team, class InP>
__device__ void object_features(const Team& team, InP inP, const uint8_t* __restrict__ g,
                                const uint8_t* __restrict__ edge, int w, int h, int bx0, int by0, int bx1,
                                int by1, FeatSmem& fs, TeamRed& red, double* f, int* border_out) {
    unsigned int* hist = fs.hist;
    unsigned int* glcm = fs.glcm;
    const int tr = team.rank();
    constexpr int TS = Team::size;
    const int sw = bx1 - bx0 + 1, sh = by1 - by0 + 1;  // search box
    const int nb = sw * sh;
    int oxmin = INT_MAX, oymin = INT_MAX, oxmax = -1, oymax = -1;
        for (int i = tr; i < 256; i += TS) hist[i] = 0;
        for (int i = tr; i < 64; i += TS) glcm[i] = 0;
        team.sync();
        // Sobel magnitude at (x, y); REFLECT_101 only needed on the tile's outer ring
        auto sobel = [&](int x, int y) -> float {
            int t[9];
            if (x > 0 && y > 0 && x < w - 1 && y < h - 1) {
                const uint8_t* r0 = g + (int64_t)(y - 1) * w + (x - 1);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    t[3 * k] = r0[(int64_t)k * w];
                    t[3 * k + 1] = r0[(int64_t)k * w + 1];
                    t[3 * k + 2] = r0[(int64_t)k * w + 2];
                }
            } else {
#pragma unroll
                for (int k = 0; k < 9; ++k)
                    t[k] = g[(int64_t)refl(y + k / 3 - 1, h) * w + refl(x + k % 3 - 1, w)];
            }
            int gx = (t[2] + 2 * t[5] + t[8]) - (t[0] + 2 * t[3] + t[6]);
            int gy = (t[6] + 2 * t[7] + t[8]) - (t[0] + 2 * t[1] + t[2]);
            return __fsqrt_rn((float)(gx * gx + gy * gy));
        };
        long long A = 0, sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0, per = 0, ne = 0;
        int border = 0;
        double gs = 0.0;
        float gmin = INFINITY, gmax = -INFINITY;
        // the search box in team order: (x, y) advanced by the team size without a division
        const int dsx = TS % sw, dsy = TS / sw;
        for (int k = tr, x = bx0 + tr % sw, y = by0 + tr / sw; k < nb;
             k += TS, x += dsx, y += dsy, (x > bx1 ? (x -= sw, ++y) : 0)) {
            if (!inP(x, y)) continue;
            ++A;
            oxmin = min(oxmin, x);
            oxmax = max(oxmax, x);
            oymin = min(oymin, y);
            oymax = max(oymax, y);
            sx += x;
            sy += y;
            sxx += (long long)x * x;
            syy += (long long)y * y;
            sxy += (long long)x * y;
            if (x == 0 || y == 0 || x == w - 1 || y == h - 1) border = 1;
            if (!inP(x - 1, y) || !inP(x + 1, y) || !inP(x, y - 1) || !inP(x, y + 1)) ++per;
            int gv = g[(int64_t)y * w + x];
            ne += edge[(int64_t)y * w + x];
            atomicAdd(&hist[gv], 1u);
            const int OX[4] = {1, 1, 0, -1}, OY[4] = {0, 1, 1, 1};
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                int qx = x + OX[o], qy = y + OY[o];
                if (!inP(qx, qy)) continue;
                int i = gv >> 5, j = g[(int64_t)qy * w + qx] >> 5;
                atomicAdd(&glcm[i * 8 + j], 1u);
                atomicAdd(&glcm[j * 8 + i], 1u);
            }
            const float m = sobel(x, y);
            gs += (double)m;
            gmin = fminf(gmin, m);
            gmax = fmaxf(gmax, m);
        }
        A = team.reduce(A, red.l, OpAdd());
        sx = team.reduce(sx, red.l, OpAdd());
        sy = team.reduce(sy, red.l, OpAdd());
        sxx = team.reduce(sxx, red.l, OpAdd());
        syy = team.reduce(syy, red.l, OpAdd());
        sxy = team.reduce(sxy, red.l, OpAdd());
        per = team.reduce(per, red.l, OpAdd());
        ne = team.reduce(ne, red.l, OpAdd());
        border = team.reduce(border, red.i, OpAdd());
        oxmin = team.reduce(oxmin, red.i, OpMin());
        oymin = team.reduce(oymin, red.i, OpMin());
        oxmax = team.reduce(oxmax, red.i, OpMax());
        oymax = team.reduce(oymax, red.i, OpMax());
        const int bw = oxmax - oxmin + 1, bh = oymax - oymin + 1;  // the object's own bounding box
        gs = team.reduce(gs, red.d, OpAdd());
        // gmin/gmax: reduce via negation trick with block_sum is wrong; use smem atomics on bits
        float& s_gmin = fs.gmin;
        float& s_gmax = fs.gmax;
        if (tr == 0) { s_gmin = INFINITY; s_gmax = -INFINITY; }
        team.sync();
        // m >= 0, so the float bit pattern orders like an unsigned int
        if (gmin <= gmax) {
            atomicMin(reinterpret_cast<unsigned int*>(&s_gmin), __float_as_uint(gmin));
            atomicMax(reinterpret_cast<int*>(&s_gmax), __float_as_int(gmax));
        }
        team.sync();
        const double Ad = (double)A;
        const double gmean = gs / Ad;
        double g2 = 0.0, g3 = 0.0, g4 = 0.0;
        for (int k = tr, x = bx0 + tr % sw, y = by0 + tr / sw; k < nb;
             k += TS, x += dsx, y += dsy, (x > bx1 ? (x -= sw, ++y) : 0)) {
            if (!inP(x, y)) continue;
            double dv = (double)sobel(x, y) - gmean;
            double d2 = dv * dv;
            g2 += d2;
            g3 += d2 * dv;
            g4 += d2 * d2;
        }
        g2 = team.reduce(g2, red.d, OpAdd());
        g3 = team.reduce(g3, red.d, OpAdd());
        g4 = team.reduce(g4, red.d, OpAdd());
        // ---- intensity histogram: rank r owns bins [r*NB, r*NB + NB), NB = 256 / team size
        constexpr int NB = 256 / TS;
        long long s1 = 0, cnt = 0;
        int vmin = 255, vmax = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int v = tr * NB + q;
            const unsigned int hv = hist[v];
            if (hv) {
                s1 += (long long)hv * v;
                cnt += hv;
                vmin = min(vmin, v);
                vmax = max(vmax, v);
            }
        }
        s1 = team.reduce(s1, red.l, OpAdd());
        vmin = team.reduce(vmin, red.i, OpMin());
        vmax = team.reduce(vmax, red.i, OpMax());
        const double mean = (double)s1 / Ad;
        double m2 = 0, m3 = 0, m4 = 0, ent = 0, en = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int v = tr * NB + q;
            if (!hist[v]) continue;
            double dv = v - mean, hv = (double)hist[v];
            m2 += hv * dv * dv;
            m3 += hv * dv * dv * dv;
            m4 += hv * dv * dv * dv * dv;
            double pv = hv / Ad;
            ent -= pv * log2(pv);
            en += pv * pv;
        }
        m2 = team.reduce(m2, red.d, OpAdd()) / Ad;
        m3 = team.reduce(m3, red.d, OpAdd()) / Ad;
        m4 = team.reduce(m4, red.d, OpAdd()) / Ad;
        ent = team.reduce(ent, red.d, OpAdd());
        en = team.reduce(en, red.d, OpAdd());
        // median: the lowest bin whose cumulative count reaches ceil(A / 2)
        const long long half = (A + 1) / 2;
        long long cum = team.scan_excl(cnt, red.l);
        int med = 256;
        if (cum < half && cum + cnt >= half) {
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                cum += hist[tr * NB + q];
                if (cum >= half) { med = tr * NB + q; break; }
            }
        }
        med = team.reduce(med, red.i, OpMin());
        // ---- Haralick on the symmetric 8x8 GLCM: rank r owns entries r, r + TS, ... (< 64)
        long long S = 0;
        for (int k = tr; k < 64; k += TS) S += glcm[k];
        S = team.reduce(S, red.l, OpAdd());
        const double Sd = (double)S;
        double mui = 0, muj = 0;
        for (int k = tr; k < 64; k += TS) {
            const double pij = (double)glcm[k] / Sd;
            mui += (k >> 3) * pij;
            muj += (k & 7) * pij;
        }
        mui = team.reduce(mui, red.d, OpAdd());
        muj = team.reduce(muj, red.d, OpAdd());
        double si = 0, sj = 0, asm_ = 0, con = 0, cor = 0, hom = 0, gent = 0, shade = 0, prom = 0, pmax = 0;
        for (int k = tr; k < 64; k += TS) {
            const int i = k >> 3, j = k & 7;
            const double pij = (double)glcm[k] / Sd;
            si += (i - mui) * (i - mui) * pij;
            sj += (j - muj) * (j - muj) * pij;
            asm_ += pij * pij;
            con += (double)((i - j) * (i - j)) * pij;
            cor += (i - mui) * (j - muj) * pij;
            hom += pij / (1.0 + (double)((i - j) * (i - j)));
            if (pij > 0) gent -= pij * log2(pij);
            double t = i + j - mui - muj;
            shade += t * t * t * pij;
            prom += t * t * t * t * pij;
            pmax = fmax(pmax, pij);
        }
        si = sqrt(team.reduce(si, red.d, OpAdd()));
        sj = sqrt(team.reduce(sj, red.d, OpAdd()));
        asm_ = team.reduce(asm_, red.d, OpAdd());
        con = team.reduce(con, red.d, OpAdd());
        cor = team.reduce(cor, red.d, OpAdd());
        hom = team.reduce(hom, red.d, OpAdd());
        gent = team.reduce(gent, red.d, OpAdd());
        shade = team.reduce(shade, red.d, OpAdd());
        prom = team.reduce(prom, red.d, OpAdd());
        pmax = team.reduce(pmax, red.d, OpMax());
        if (tr == 0) {
            const double PI = 3.14159265358979323846;
            // shape
            double cx = (double)sx / Ad, cy = (double)sy / Ad;
            double bwd = bw, bhd = bh;
            double mu20 = (double)(A * sxx - sx * sx) / Ad;
            double mu02 = (double)(A * syy - sy * sy) / Ad;
            double mu11 = (double)(A * sxy - sx * sy) / Ad;
            double a = mu20 / Ad + 1.0 / 12.0, b = mu11 / Ad, c = mu02 / Ad + 1.0 / 12.0;
            double tr = 0.5 * (a + c), disc = sqrt(0.25 * (a - c) * (a - c) + b * b);
            double l1 = tr + disc, l2 = tr - disc;
            if (l2 < 0) l2 = 0;
            f[HP_F_AREA] = Ad;
            f[HP_F_PERIMETER] = (double)per;
            f[HP_F_CENTROID_X] = cx;
            f[HP_F_CENTROID_Y] = cy;
            f[HP_F_BBOX_W] = bwd;
            f[HP_F_BBOX_H] = bhd;
            f[HP_F_MAJOR] = 4.0 * sqrt(l1);
            f[HP_F_MINOR] = 4.0 * sqrt(l2);
            f[HP_F_ECCENTRICITY] = sqrt(1.0 - l2 / l1);
            f[HP_F_ORIENTATION] = 0.5 * atan2(2.0 * mu11, mu20 - mu02);
            f[HP_F_EQDIAM] = sqrt(4.0 * Ad / PI);
            f[HP_F_COMPACTNESS] = 4.0 * PI * Ad / ((double)per * (double)per);
            f[HP_F_EXTENT] = Ad / (bwd * bhd);
            // intensity
            bool flat = vmin == vmax;
            f[HP_F_INT_MEAN] = mean;
            f[HP_F_INT_STD] = flat ? 0.0 : sqrt(m2);
            f[HP_F_INT_MIN] = vmin;
            f[HP_F_INT_MAX] = vmax;
            f[HP_F_INT_MEDIAN] = med;
            f[HP_F_INT_SKEW] = flat ? 0.0 : m3 / (m2 * sqrt(m2));
            f[HP_F_INT_KURT] = flat ? 0.0 : m4 / (m2 * m2);
            f[HP_F_INT_ENTROPY] = ent;
            f[HP_F_INT_ENERGY] = en;
            // gradient magnitude
            bool gflat = s_gmin == s_gmax;
            double gg2 = g2 / Ad, gg3 = g3 / Ad, gg4 = g4 / Ad;
            f[HP_F_GRAD_MEAN] = gmean;
            f[HP_F_GRAD_STD] = gflat ? 0.0 : sqrt(gg2);
            f[HP_F_GRAD_SKEW] = gflat ? 0.0 : gg3 / (gg2 * sqrt(gg2));
            f[HP_F_GRAD_KURT] = gflat ? 0.0 : gg4 / (gg2 * gg2);
            // Haralick
            if (S == 0) {
                for (int k = HP_F_GLCM_ASM; k <= HP_F_GLCM_MAXPROB; ++k) f[k] = 0.0;
            } else {
                f[HP_F_GLCM_ASM] = asm_;
                f[HP_F_GLCM_CONTRAST] = con;
                f[HP_F_GLCM_CORRELATION] = (si * sj == 0.0) ? 1.0 : cor / (si * sj);
                f[HP_F_GLCM_HOMOGENEITY] = hom;
                f[HP_F_GLCM_ENTROPY] = gent;
                f[HP_F_GLCM_SHADE] = shade;
                f[HP_F_GLCM_PROMINENCE] = prom;
                f[HP_F_GLCM_MAXPROB] = pmax;
            }
            // edge (Canny): edge pixels of the object and their fraction of its area
            f[HP_F_EDGE_COUNT] = (double)ne;
            f[HP_F_EDGE_FRAC] = (double)ne / Ad;
            *border_out = border;
        }
        team.sync();
}

}  // namespace
}  // namespace hp
