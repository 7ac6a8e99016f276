// k_ws.cu -- S8 markers (Pre-Watershed MR), S9 watershed (PAPER.md:601,
// 626-628) and S10 BWLabel + final filter.
//
// S8: J = GrayRecon8_f32(dist - h, dist) inside F (h-maxima; IWPP f32), flat zones of J by
//     CCL with float equality, a zone is a regional maximum iff none of its pixels has a
//     higher F neighbour (flag atomically ORed at the zone root), ML = 1 + zone root.
// S9: the order-independent watershed of DESIGN.md reading C13:
//     W1 c = GrayRecon8_f32(dist on markers else -inf, dist) inside F     (IWPP f32)
//     W2 d = plateau distance: 0 markers, 1 if a higher neighbour, else 1 + min equal-c
//        neighbour (least fixed point, IWPP min-plus)
//     W3 L = min label over the steepest-ascent parents (parent bitmask per pixel; least
//        fixed point from +inf, IWPP min)
//     lines: pixels with a smaller-labelled F neighbour; split = F minus lines.
// All three fixed points are unique, so the result is schedule independent (bit-exact
// with the oracle's sequential Vincent/BFS/sorted-order algorithms).
#include <cfloat>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {

namespace {

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, num_sms() * 16); }

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_j_init(const float* __restrict__ dist, const uint8_t* __restrict__ F, float hh,
                         int64_t n, float* __restrict__ J) {
    GRID_LOOP(i, n) {
        float v = NAN;
        if (F[i]) {
            float dv = dist[i];
            v = fminf(__fsub_rn(dv, hh), dv);
        }
        J[i] = v;
    }
}

// flat-zone root gets aux = 1 if some pixel of the zone has a higher F neighbour
__global__ void k_notmax(const float* __restrict__ J, const uint8_t* __restrict__ F,
                         const int32_t* __restrict__ lab, int w, int h, int32_t* __restrict__ aux) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        if (!F[p]) continue;
        int x = (int)(p % w), y = (int)(p / w);
        float jp = J[p];
        bool higher = false;
        for (int j = 0; j < 8 && !higher; ++j) {
            int qx = x + dx8(j), qy = y + dy8(j);
            if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
            int64_t q = (int64_t)qy * w + qx;
            if (F[q] && J[q] > jp) higher = true;
        }
        if (higher) aux[lab[p]] = 1;
    }
}

__global__ void k_ml(const uint8_t* __restrict__ F, const int32_t* __restrict__ lab,
                     const int32_t* __restrict__ aux, int64_t n, int32_t* __restrict__ ML) {
    GRID_LOOP(p, n) {
        int32_t v = 0;
        if (F[p]) {
            int32_t r = lab[p];
            if (aux[r] == 0) v = r + 1;
        }
        ML[p] = v;
    }
}

__global__ void k_c_init(const float* __restrict__ dist, const int32_t* __restrict__ ML,
                         const uint8_t* __restrict__ F, int64_t n, float* __restrict__ c) {
    GRID_LOOP(p, n) c[p] = F[p] ? (ML[p] ? dist[p] : -INFINITY) : NAN;
}

__global__ void k_d_init(const float* __restrict__ c, const int32_t* __restrict__ ML,
                         const uint8_t* __restrict__ F, int w, int h, int32_t* __restrict__ d) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        int32_t v = kInfI;
        if (F[p]) {
            if (ML[p]) {
                v = 0;
            } else {
                int x = (int)(p % w), y = (int)(p / w);
                float cp = c[p];
                for (int j = 0; j < 8; ++j) {
                    int qx = x + dx8(j), qy = y + dy8(j);
                    if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                    int64_t q = (int64_t)qy * w + qx;
                    if (F[q] && c[q] > cp) { v = 1; break; }
                }
            }
        }
        d[p] = v;
    }
}

// parent bitmask: argmin over F neighbours q with c(q) >= c(p) of (-c(q), d(q))
__global__ void k_parents(const float* __restrict__ c, const int32_t* __restrict__ d,
                          const int32_t* __restrict__ ML, const uint8_t* __restrict__ F, int w, int h,
                          uint8_t* __restrict__ pm, int32_t* __restrict__ L) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        uint8_t bits = 0;
        int32_t lv = kInfI;
        if (F[p]) {
            if (ML[p]) {
                lv = ML[p];
            } else {
                int x = (int)(p % w), y = (int)(p / w);
                float cp = c[p];
                bool have = false;
                float bc = 0.f;
                int32_t bd = 0;
                for (int j = 0; j < 8; ++j) {
                    int qx = x + dx8(j), qy = y + dy8(j);
                    if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                    int64_t q = (int64_t)qy * w + qx;
                    if (!F[q]) continue;
                    float cq = c[q];
                    if (!(cq >= cp)) continue;
                    int32_t dq = d[q];
                    if (!have || cq > bc || (cq == bc && dq < bd)) {
                        have = true;
                        bc = cq;
                        bd = dq;
                        bits = (uint8_t)(1u << j);
                    } else if (cq == bc && dq == bd) {
                        bits |= (uint8_t)(1u << j);
                    }
                }
            }
        }
        pm[p] = bits;
        L[p] = lv;
    }
}

__global__ void k_lines(const int32_t* __restrict__ L, const uint8_t* __restrict__ F, int w, int h,
                        uint8_t* __restrict__ split) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        uint8_t v = 0;
        if (F[p]) {
            v = 1;
            int x = (int)(p % w), y = (int)(p / w);
            int32_t lp = L[p];
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (qx < 0 || qy < 0 || qx >= w || qy >= h) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (F[q] && L[q] < lp) { v = 0; break; }
            }
        }
        split[p] = v;
    }
}

template <class T>
__global__ void k_zero_outside(const T* __restrict__ src, const uint8_t* __restrict__ F, int64_t n,
                               T* __restrict__ dst) {
    GRID_LOOP(p, n) dst[p] = F[p] ? src[p] : T(0);
}

// S10: labels = 1 + root for kept components, 0 otherwise; kept roots counted
__global__ void k_bw_label(const int32_t* __restrict__ lab, const int32_t* __restrict__ area,
                           int w, int h, int amin, int amax, int32_t* __restrict__ labels,
                           int64_t lpitch, int32_t* __restrict__ nobj) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        int32_t r = lab[p];
        int32_t v = 0;
        if (r >= 0) {
            int a = area[r];
            if (a >= amin && a <= amax) {
                v = r + 1;
                if (r == (int32_t)p) atomicAdd(nobj, 1);
            }
        }
        int y = (int)(p / w), x = (int)(p - (int64_t)y * w);
        labels[(int64_t)y * lpitch + x] = v;
    }
}

}  // namespace

void launch_markers(const float* dist, const uint8_t* F, float hh, int w, int h, Slot& sl,
                    int32_t* ML, float* J, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    (note_launch(), k_j_init<<<grid_for(n), 256, 0, s>>>(dist, F, hh, n, J));
    launch_recon_f32(dist, F, J, w, h, sl.wl, true, s);
    CclSrc zones{F, 0, false, J};
    launch_ccl(zones, w, h, 8, sl.lab, sl.aux, s);
    (note_launch(), k_notmax<<<grid_for(n), 256, 0, s>>>(J, F, sl.lab, w, h, sl.aux));
    (note_launch(), k_ml<<<grid_for(n), 256, 0, s>>>(F, sl.lab, sl.aux, n, ML));
}

void launch_watershed(const float* dist, const int32_t* ML, const uint8_t* F, int w, int h,
                      Slot& sl, uint8_t* split, float* c_out, int32_t* d_out, int32_t* L_out,
                      cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    (note_launch(), k_c_init<<<grid_for(n), 256, 0, s>>>(dist, ML, F, n, sl.c));
    launch_recon_f32(dist, F, sl.c, w, h, sl.wl, true, s);                // W1
    (note_launch(), k_d_init<<<grid_for(n), 256, 0, s>>>(sl.c, ML, F, w, h, sl.d));
    launch_plateau_dist(sl.c, sl.d, w, h, sl.wl, F, s);                    // W2
    (note_launch(), k_parents<<<grid_for(n), 256, 0, s>>>(sl.c, sl.d, ML, F, w, h, sl.pmask, sl.L));
    launch_parent_min(sl.pmask, sl.L, w, h, sl.wl, F, s);                  // W3
    (note_launch(), k_lines<<<grid_for(n), 256, 0, s>>>(sl.L, F, w, h, split));
    if (c_out) (note_launch(), k_zero_outside<float><<<grid_for(n), 256, 0, s>>>(sl.c, F, n, c_out));
    if (d_out) (note_launch(), k_zero_outside<int32_t><<<grid_for(n), 256, 0, s>>>(sl.d, F, n, d_out));
    if (L_out) (note_launch(), k_zero_outside<int32_t><<<grid_for(n), 256, 0, s>>>(sl.L, F, n, L_out));
}

void launch_bwlabel(const uint8_t* split, int w, int h, int amin, int amax, Slot& sl,
                    int32_t* labels, int64_t lpitch, int32_t* n_objects, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    cudaMemsetAsync(n_objects, 0, sizeof(int32_t), s);
    if (n == 0) return;
    CclSrc cs{split, 0, false, nullptr};
    launch_ccl(cs, w, h, 8, sl.lab, sl.aux, s);
    launch_ccl_count(cs, w, h, sl.lab, sl.aux, s);
    (note_launch(), k_bw_label<<<grid_for(n), 256, 0, s>>>(sl.lab, sl.aux, w, h, amin, amax, labels, lpitch, n_objects));
}

// exposed for the verification ABI (J outside F -> 0)
void launch_zero_outside_f32(const float* src, const uint8_t* F, int64_t n, float* dst, cudaStream_t s) {
    if (n) (note_launch(), k_zero_outside<float><<<grid_for(n), 256, 0, s>>>(src, F, n, dst));
}

}  // namespace hp
