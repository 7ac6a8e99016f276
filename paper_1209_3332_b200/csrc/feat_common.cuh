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

struct TeamCTA {
    static constexpr int size = kFT;
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
        for (int k = 1; k < kFT / 32; ++k) r = op(r, red[k]);
        __syncthreads();
        return r;
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
};

struct OpAdd {
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMin {
    __device__ __forceinline__ int operator()(int a, int b) const { return a < b ? a : b; }
};
struct OpMax {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
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
    unsigned int hist[256];
    unsigned int glcm[64];
    float gmin, gmax;
};

// Every thread of the team calls this for one object P = {(x, y) : inP(x, y)} inside the
// search box [bx0, bx1] x [by0, by1]; g is the tile's u8 plane (w x h, REFLECT_101 Sobel).
// Team rank 0 receives the 34 features in f and the border flag.
template <class Team, class InP>
__device__ void object_features(const Team& team, InP inP, const uint8_t* __restrict__ g, int w, int h,
                                int bx0, int by0, int bx1, int by1, FeatSmem& fs, TeamRed& red, double* f,
                                int* border_out) {
    unsigned int* hist = fs.hist;
    unsigned int* glcm = fs.glcm;
    const int tr = team.rank();
    constexpr int TS = Team::size;
    const int sw = bx1 - bx0 + 1, sh = by1 - by0 + 1;  // search box
    const int64_t nb = (int64_t)sw * sh;
    int oxmin = INT_MAX, oymin = INT_MAX, oxmax = -1, oymax = -1;
        for (int i = tr; i < 256; i += TS) hist[i] = 0;
        for (int i = tr; i < 64; i += TS) glcm[i] = 0;
        team.sync();
        auto G = [&](int x, int y) { return (int)g[(int64_t)refl(y, h) * w + refl(x, w)]; };
        long long A = 0, sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0, per = 0;
        int border = 0;
        double gs = 0.0;
        float gmin = INFINITY, gmax = -INFINITY;
        for (int64_t k = tr; k < nb; k += TS) {
            int y = by0 + (int)(k / sw), x = bx0 + (int)(k % sw);
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
            int gx = (G(x + 1, y - 1) + 2 * G(x + 1, y) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x - 1, y) + G(x - 1, y + 1));
            int gy = (G(x - 1, y + 1) + 2 * G(x, y + 1) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x, y - 1) + G(x + 1, y - 1));
            float m = __fsqrt_rn((float)(gx * gx + gy * gy));
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
        for (int64_t k = tr; k < nb; k += TS) {
            int y = by0 + (int)(k / sw), x = bx0 + (int)(k % sw);
            if (!inP(x, y)) continue;
            int gx = (G(x + 1, y - 1) + 2 * G(x + 1, y) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x - 1, y) + G(x - 1, y + 1));
            int gy = (G(x - 1, y + 1) + 2 * G(x, y + 1) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x, y - 1) + G(x + 1, y - 1));
            double dv = (double)__fsqrt_rn((float)(gx * gx + gy * gy)) - gmean;
            double d2 = dv * dv;
            g2 += d2;
            g3 += d2 * dv;
            g4 += d2 * d2;
        }
        g2 = team.reduce(g2, red.d, OpAdd());
        g3 = team.reduce(g3, red.d, OpAdd());
        g4 = team.reduce(g4, red.d, OpAdd());
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
            // intensity (histogram, ascending bins)
            long long s1 = 0;
            int vmin = 255, vmax = 0;
            for (int v = 0; v < 256; ++v)
                if (hist[v]) {
                    s1 += (long long)hist[v] * v;
                    vmin = min(vmin, v);
                    vmax = max(vmax, v);
                }
            double mean = (double)s1 / Ad, m2 = 0, m3 = 0, m4 = 0, ent = 0, en = 0;
            for (int v = 0; v < 256; ++v) {
                if (!hist[v]) continue;
                double dv = v - mean, hv = (double)hist[v];
                m2 += hv * dv * dv;
                m3 += hv * dv * dv * dv;
                m4 += hv * dv * dv * dv * dv;
                double pv = hv / Ad;
                ent -= pv * log2(pv);
                en += pv * pv;
            }
            m2 /= Ad;
            m3 /= Ad;
            m4 /= Ad;
            long long half = (A + 1) / 2, cum = 0;
            int med = 0;
            for (int v = 0; v < 256; ++v) {
                cum += hist[v];
                if (cum >= half) { med = v; break; }
            }
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
            // Haralick on the symmetric 8x8 GLCM
            long long S = 0;
            for (int i = 0; i < 64; ++i) S += glcm[i];
            if (S == 0) {
                for (int k = HP_F_GLCM_ASM; k <= HP_F_GLCM_MAXPROB; ++k) f[k] = 0.0;
            } else {
                double Pm[64], mui = 0, muj = 0;
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j) {
                        Pm[i * 8 + j] = (double)glcm[i * 8 + j] / (double)S;
                        mui += i * Pm[i * 8 + j];
                        muj += j * Pm[i * 8 + j];
                    }
                double si = 0, sj = 0;
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j) {
                        si += (i - mui) * (i - mui) * Pm[i * 8 + j];
                        sj += (j - muj) * (j - muj) * Pm[i * 8 + j];
                    }
                si = sqrt(si);
                sj = sqrt(sj);
                double asm_ = 0, con = 0, cor = 0, hom = 0, gent = 0, shade = 0, prom = 0, pmax = 0;
                for (int i = 0; i < 8; ++i)
                    for (int j = 0; j < 8; ++j) {
                        double pij = Pm[i * 8 + j];
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
                f[HP_F_GLCM_ASM] = asm_;
                f[HP_F_GLCM_CONTRAST] = con;
                f[HP_F_GLCM_CORRELATION] = (si * sj == 0.0) ? 1.0 : cor / (si * sj);
                f[HP_F_GLCM_HOMOGENEITY] = hom;
                f[HP_F_GLCM_ENTROPY] = gent;
                f[HP_F_GLCM_SHADE] = shade;
                f[HP_F_GLCM_PROMINENCE] = prom;
                f[HP_F_GLCM_MAXPROB] = pmax;
            }
            *border_out = border;
        }
        team.sync();
}

}  // namespace
}  // namespace hp
