// k_feat.cu -- S11: per-object features ("Features comp."; families of
// pixel statistics, gradient statistics, Haralick, morphometry; per-object
// bag of tasks PAPER.md:223-224; definitions: DESIGN.md "Feature table", reading C16/C17).
//
//   k_obj_find   roots = pixels whose label equals 1 + their own linear index
//   k_obj_rank   rank of each root among all roots (rows in ascending label order)
//   k_obj_bbox   bounding boxes by warp-aggregated atomicMin/Max on the compact id
//   k_obj_feat   one CTA per object (grid-stride over the device-side count): exact
//                integer sums (area, moments, perimeter, 256-bin histogram and 8x8 GLCM in
//                shared memory via smem atomics), Sobel magnitude on the fly with fp64
//                two-pass moments in a fixed reduction order (deterministic), then one
//                thread finalises the 34 features in fp64 and stores them as f32.
// Compiled with -fmad=false so the fp64 finaliser rounds like its written formulas.
#include <cfloat>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {

namespace {

constexpr int kFT = 256;  // threads per object CTA

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }

__global__ void k_obj_find(const int32_t* __restrict__ labels, int64_t lpitch, int w, int h,
                           int32_t* __restrict__ cnt, int32_t* __restrict__ roots, int32_t cap) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        int y = (int)(p / w), x = (int)(p - (int64_t)y * w);
        if (labels[(int64_t)y * lpitch + x] == (int32_t)(p + 1)) {
            int i = atomicAdd(cnt, 1);
            if (i < cap) roots[i] = (int32_t)p;
        }
    }
}

__global__ void k_obj_rank(const int32_t* __restrict__ cnt, int32_t cap, const int32_t* __restrict__ roots,
                           int32_t* __restrict__ rank_root, int32_t* __restrict__ idmap) {
    const int n = min(*cnt, cap);
    __shared__ int32_t chunk[1024];
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        int i = base + threadIdx.x;
        int32_t me = i < n ? roots[i] : 0;
        int rk = 0;
        for (int c0 = 0; c0 < n; c0 += 1024) {
            __syncthreads();
            for (int k = threadIdx.x; k < 1024 && c0 + k < n; k += blockDim.x) chunk[k] = roots[c0 + k];
            __syncthreads();
            int lim = min(1024, n - c0);
            for (int k = 0; k < lim; ++k) rk += chunk[k] < me;
        }
        if (i < n) {
            rank_root[rk] = me;
            idmap[me] = rk;
        }
    }
}

__global__ void k_bbox_init(const int32_t* __restrict__ cnt, int32_t cap, int32_t* __restrict__ bbox) {
    const int n = min(*cnt, cap);
    GRID_LOOP(i, (int64_t)n) {
        bbox[4 * i + 0] = INT_MAX;
        bbox[4 * i + 1] = INT_MAX;
        bbox[4 * i + 2] = -1;
        bbox[4 * i + 3] = -1;
    }
}

__global__ void k_obj_bbox(const int32_t* __restrict__ labels, int64_t lpitch, int w, int h,
                           const int32_t* __restrict__ cnt, int32_t cap, const int32_t* __restrict__ idmap,
                           int32_t* __restrict__ bbox) {
    const int64_t n = (int64_t)w * h;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = base + threadIdx.x;
        int id = -1, x = 0, y = 0;
        if (p < n) {
            y = (int)(p / w);
            x = (int)(p - (int64_t)y * w);
            int32_t l = labels[(int64_t)y * lpitch + x];
            if (l > 0) id = idmap[l - 1];
            if (id >= cap) id = -1;
        }
        unsigned peers = __match_any_sync(0xffffffffu, id);
        if (id < 0) continue;
        int x0 = __reduce_min_sync(peers, x), y0 = __reduce_min_sync(peers, y);
        int x1 = __reduce_max_sync(peers, x), y1 = __reduce_max_sync(peers, y);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
            atomicMin(&bbox[4 * id + 0], x0);
            atomicMin(&bbox[4 * id + 1], y0);
            atomicMax(&bbox[4 * id + 2], x1);
            atomicMax(&bbox[4 * id + 3], y1);
        }
    }
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    // fixed-order reduction: warp tree, then warp 0 over the per-warp partials
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T r = 0;
    if (warp == 0) {
        r = lane < (kFT / 32) ? red[lane] : T(0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
        if (lane == 0) red[0] = r;
    }
    __syncthreads();
    r = red[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ int refl(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * n - 2 - i;
    }
    return i;
}

__global__ void __launch_bounds__(kFT, 3) k_obj_feat(const int32_t* __restrict__ labels, int64_t lpitch,
                                                  const uint8_t* __restrict__ g, int w, int h,
                                                  const int32_t* __restrict__ cnt, int32_t cap,
                                                  const int32_t* __restrict__ rank_root,
                                                  const int32_t* __restrict__ bbox,
                                                  int32_t* __restrict__ out_label, int32_t* __restrict__ out_flags,
                                                  float* __restrict__ out_feat, int32_t capacity) {
    __shared__ unsigned int hist[256];
    __shared__ unsigned int glcm[64];
    __shared__ long long redl[kFT / 32];
    __shared__ double redd[kFT / 32];
    __shared__ int redi[kFT / 32];
    const int n = min(*cnt, min(cap, capacity));
    for (int obj = blockIdx.x; obj < n; obj += gridDim.x) {
        const int32_t root = rank_root[obj];
        const int32_t lab = root + 1;
        const int bx0 = bbox[4 * obj], by0 = bbox[4 * obj + 1], bx1 = bbox[4 * obj + 2], by1 = bbox[4 * obj + 3];
        const int bw = bx1 - bx0 + 1, bh = by1 - by0 + 1;
        const int64_t nb = (int64_t)bw * bh;
        for (int i = threadIdx.x; i < 256; i += kFT) hist[i] = 0;
        if (threadIdx.x < 64) glcm[threadIdx.x] = 0;
        __syncthreads();
        auto inP = [&](int x, int y) {
            return x >= 0 && y >= 0 && x < w && y < h && labels[(int64_t)y * lpitch + x] == lab;
        };
        auto G = [&](int x, int y) { return (int)g[(int64_t)refl(y, h) * w + refl(x, w)]; };
        long long A = 0, sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0, per = 0;
        int border = 0;
        double gs = 0.0;
        float gmin = INFINITY, gmax = -INFINITY;
        for (int64_t k = threadIdx.x; k < nb; k += kFT) {
            int y = by0 + (int)(k / bw), x = bx0 + (int)(k % bw);
            if (!inP(x, y)) continue;
            ++A;
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
        A = block_sum<long long>(A, redl);
        sx = block_sum<long long>(sx, redl);
        sy = block_sum<long long>(sy, redl);
        sxx = block_sum<long long>(sxx, redl);
        syy = block_sum<long long>(syy, redl);
        sxy = block_sum<long long>(sxy, redl);
        per = block_sum<long long>(per, redl);
        border = block_sum<int>(border, redi);
        gs = block_sum<double>(gs, redd);
        // gmin/gmax: reduce via negation trick with block_sum is wrong; use smem atomics on bits
        __shared__ float s_gmin, s_gmax;
        if (threadIdx.x == 0) { s_gmin = INFINITY; s_gmax = -INFINITY; }
        __syncthreads();
        // m >= 0, so the float bit pattern orders like an unsigned int
        if (gmin <= gmax) {
            atomicMin(reinterpret_cast<unsigned int*>(&s_gmin), __float_as_uint(gmin));
            atomicMax(reinterpret_cast<int*>(&s_gmax), __float_as_int(gmax));
        }
        __syncthreads();
        const double Ad = (double)A;
        const double gmean = gs / Ad;
        double g2 = 0.0, g3 = 0.0, g4 = 0.0;
        for (int64_t k = threadIdx.x; k < nb; k += kFT) {
            int y = by0 + (int)(k / bw), x = bx0 + (int)(k % bw);
            if (!inP(x, y)) continue;
            int gx = (G(x + 1, y - 1) + 2 * G(x + 1, y) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x - 1, y) + G(x - 1, y + 1));
            int gy = (G(x - 1, y + 1) + 2 * G(x, y + 1) + G(x + 1, y + 1)) - (G(x - 1, y - 1) + 2 * G(x, y - 1) + G(x + 1, y - 1));
            double dv = (double)__fsqrt_rn((float)(gx * gx + gy * gy)) - gmean;
            double d2 = dv * dv;
            g2 += d2;
            g3 += d2 * dv;
            g4 += d2 * d2;
        }
        g2 = block_sum<double>(g2, redd);
        g3 = block_sum<double>(g3, redd);
        g4 = block_sum<double>(g4, redd);
        if (threadIdx.x == 0) {
            double f[HP_NFEAT];
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
            out_label[obj] = lab;
            out_flags[obj] = border ? HP_OBJ_TOUCHES_BORDER : 0;
            for (int k = 0; k < HP_NFEAT; ++k) out_feat[(int64_t)obj * HP_NFEAT + k] = (float)f[k];
        }
        __syncthreads();
    }
}

__global__ void k_copy_count(const int32_t* __restrict__ cnt, int32_t* __restrict__ n_rows) { *n_rows = *cnt; }

}  // namespace

void launch_features(const int32_t* labels, int64_t lpitch, const uint8_t* g, int w, int h,
                     Slot& sl, int32_t max_objects, int32_t* row_label, int32_t* row_flags,
                     float* feat, int32_t capacity, int32_t* n_rows, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    int32_t* cnt = sl.cnt32 + 2;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
    if (n > 0) {
        (note_launch(), k_obj_find<<<grid_for(n), 256, 0, s>>>(labels, lpitch, w, h, cnt, sl.obj_root, max_objects));
        (note_launch(), k_obj_rank<<<std::max(1, std::min(148 * 4, (max_objects + 255) / 256)), 256, 0, s>>>(
            cnt, max_objects, sl.obj_root, sl.obj_rank, sl.aux));
        (note_launch(), k_bbox_init<<<std::max(1, std::min(148 * 4, (max_objects + 255) / 256)), 256, 0, s>>>(cnt, max_objects, sl.obj_bbox));
        (note_launch(), k_obj_bbox<<<grid_for(n), 256, 0, s>>>(labels, lpitch, w, h, cnt, max_objects, sl.aux, sl.obj_bbox));
        (note_launch(), k_obj_feat<<<148 * 8, kFT, 0, s>>>(labels, lpitch, g, w, h, cnt, max_objects, sl.obj_rank,
                                           sl.obj_bbox, row_label, row_flags, feat, capacity));
    }
    (note_launch(), k_copy_count<<<1, 1, 0, s>>>(cnt, n_rows));
}

}  // namespace hp
