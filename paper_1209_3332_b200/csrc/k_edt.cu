// k_edt.cu -- S7: Pre-Watershed exact Euclidean distance transform (PAPER.md:599-600
// "OpenCV for distance transformation"; reading C11: exact EDT, out-of-tile pixels are not
// background, +inf when the tile has no background).
//
// Separable and integer-exact:
//   k_edt_seg   one thread per (column, 64-row segment): first / last background row of
//               the segment (coalesced: a warp reads 32 adjacent columns of one row);
//   k_edt_col   one thread per (column, segment): vertical distance gcol to the nearest
//               background pixel of the column, carrying in the nearest background rows of
//               the segments above/below from the summaries (u16, 0xFFFF = none);
//   k_edt_row   one CTA per row: the row of gcol^2 in shared memory; for each foreground
//               pixel an exact expanding search min_k (k^2 + gcol(x +- k)^2) that stops as
//               soon as k^2 >= best (nuclei are small, so k stays small).  If a search would
//               exceed kSearchCap, the whole row is redone by Meijster's linear-time lower
//               envelope (one thread) -- same exact result, bounded worst case.
// d2 exact (uint32), dist = IEEE sqrtf((float)d2).
#include <cfloat>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {

namespace {

constexpr int kSeg = 64;
constexpr int kSearchCap = 256;
constexpr uint16_t kNone16 = 0xFFFF;
constexpr uint32_t kInfSq = 0x7fffffffu;

__global__ void k_edt_seg(const uint8_t* __restrict__ F, int w, int h, int nseg,
                          int16_t* __restrict__ top, int16_t* __restrict__ bot,
                          int32_t* __restrict__ any_bg, const int32_t* __restrict__ cond) {
    if (cond && *cond == 0) return;
    int64_t n = (int64_t)w * nseg;
    bool found = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int seg = (int)(i / w), x = (int)(i - (int64_t)seg * w);
        int y0 = seg * kSeg, y1 = min(h, y0 + kSeg);
        int first = -1, last = -1;
        for (int y = y0; y < y1; ++y)
            if (F[(int64_t)y * w + x] == 0) {
                if (first < 0) first = y;
                last = y;
            }
        top[i] = (int16_t)first;
        bot[i] = (int16_t)last;
        found |= first >= 0;
    }
    if (__any_sync(0xffffffffu, found) && (threadIdx.x & 31) == 0) atomicOr(any_bg, 1);
}

__global__ void k_edt_col(const uint8_t* __restrict__ F, int w, int h, int nseg,
                          const int16_t* __restrict__ top, const int16_t* __restrict__ bot,
                          uint16_t* __restrict__ gcol, const int32_t* __restrict__ cond) {
    if (cond && *cond == 0) return;
    int64_t n = (int64_t)w * nseg;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int seg = (int)(i / w), x = (int)(i - (int64_t)seg * w);
        int y0 = seg * kSeg, y1 = min(h, y0 + kSeg);
        int above = -1, below = -1;  // nearest background row above / below the segment
        for (int s = seg - 1; s >= 0; --s) {
            int b = bot[(int64_t)s * w + x];
            if (b >= 0) { above = b; break; }
        }
        for (int s = seg + 1; s < nseg; ++s) {
            int t = top[(int64_t)s * w + x];
            if (t >= 0) { below = t; break; }
        }
        int last = above;
        for (int y = y0; y < y1; ++y) {
            int64_t p = (int64_t)y * w + x;
            if (F[p] == 0) last = y;
            gcol[p] = last >= 0 ? (uint16_t)(y - last) : kNone16;
        }
        int next = below;
        for (int y = y1 - 1; y >= y0; --y) {
            int64_t p = (int64_t)y * w + x;
            if (F[p] == 0) next = y;
            if (next >= 0) {
                int up = gcol[p];
                int dn = next - y;
                if (dn < up) gcol[p] = (uint16_t)dn;
            }
        }
    }
}

__device__ __forceinline__ uint32_t sqg(uint16_t g) {
    return g == kNone16 ? kInfSq : (uint32_t)g * (uint32_t)g;
}

__global__ void __launch_bounds__(256) k_edt_row(const uint8_t* __restrict__ F, int w, int h,
                                                 const uint16_t* __restrict__ gcol,
                                                 const int32_t* __restrict__ any_bg,
                                                 int32_t* __restrict__ scr_s, int32_t* __restrict__ scr_t,
                                                 uint32_t* __restrict__ d2out, float* __restrict__ dist,
                                                 const int32_t* __restrict__ cond) {
    if (cond && *cond == 0) return;
    extern __shared__ uint32_t sq[];
    __shared__ int need_full;
    const int y = blockIdx.x;
    const int64_t row = (int64_t)y * w;
    const bool has_bg = *any_bg != 0;
    if (threadIdx.x == 0) need_full = 0;
    for (int x = threadIdx.x; x < w; x += blockDim.x) sq[x] = sqg(gcol[row + x]);
    __syncthreads();
    for (int x = threadIdx.x; x < w; x += blockDim.x) {
        int64_t p = row + x;
        uint32_t best;
        if (F[p] == 0) {
            best = 0;
        } else if (!has_bg) {
            best = 0xffffffffu;
        } else {
            best = sq[x];
            int k = 1;
            for (; (uint32_t)k * (uint32_t)k < best; ++k) {
                if (k > kSearchCap) {
                    need_full = 1;
                    break;
                }
                uint32_t kk = (uint32_t)k * (uint32_t)k;
                if (x - k >= 0 && sq[x - k] != kInfSq) best = min(best, kk + sq[x - k]);
                if (x + k < w && sq[x + k] != kInfSq) best = min(best, kk + sq[x + k]);
            }
        }
        if (d2out) d2out[p] = best;
        dist[p] = best == 0xffffffffu ? INFINITY : __fsqrt_rn(__uint2float_rn(best));
    }
    __syncthreads();
    if (need_full && threadIdx.x == 0) {
        // Meijster, Roerdink & Hesselink (2000), phase 2 on this row, integer arithmetic
        int32_t* s = scr_s + row;
        int32_t* t = scr_t + row;
        const int64_t INF = (int64_t)w + h;
        auto G = [&](int i) -> int64_t {
            uint16_t g = gcol[row + i];
            return g == kNone16 ? INF : (int64_t)g;
        };
        auto f = [&](int64_t x, int64_t i) { int64_t gi = G((int)i); return (x - i) * (x - i) + gi * gi; };
        int q = 0;
        s[0] = 0;
        t[0] = 0;
        for (int u = 1; u < w; ++u) {
            while (q >= 0 && f(t[q], s[q]) > f(t[q], u)) --q;
            if (q < 0) {
                q = 0;
                s[0] = u;
            } else {
                int64_t gu = G(u), gs = G(s[q]);
                int64_t num = (int64_t)u * u - (int64_t)s[q] * s[q] + gu * gu - gs * gs;
                int64_t den = 2 * (int64_t)(u - s[q]);
                int64_t fl = num / den;
                if ((num % den != 0) && ((num < 0) != (den < 0))) --fl;
                int64_t wv = 1 + fl;
                if (wv < w) {
                    ++q;
                    s[q] = u;
                    t[q] = (int32_t)wv;
                }
            }
        }
        for (int u = w - 1; u >= 0; --u) {
            int64_t p = row + u;
            if (F[p] != 0) {
                uint32_t v = (uint32_t)f(u, s[q]);
                if (d2out) d2out[p] = v;
                dist[p] = __fsqrt_rn(__uint2float_rn(v));
            }
            if (u == t[q]) --q;
        }
    }
}

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, num_sms() * 16); }

}  // namespace

// cond (device int, may be null): skip the whole transform when *cond == 0 at run time (the
// pipeline needs the global plane only for components that fall back to the global path)
void launch_edt(const uint8_t* F, int w, int h, Slot& sl, uint32_t* d2_out, float* dist,
                cudaStream_t s, const int32_t* cond) {
    if ((int64_t)w * h == 0) return;
    const int nseg = (h + kSeg - 1) / kSeg;
    int32_t* any_bg = sl.cnt32 + 1;
    cudaMemsetAsync(any_bg, 0, sizeof(int32_t), s);
    int64_t nthreads = (int64_t)w * nseg;
    (note_launch(), k_edt_seg<<<grid_for(nthreads), 256, 0, s>>>(F, w, h, nseg, sl.seg_top, sl.seg_bot, any_bg, cond));
    (note_launch(), k_edt_col<<<grid_for(nthreads), 256, 0, s>>>(F, w, h, nseg, sl.seg_top, sl.seg_bot, sl.gcol, cond));
    size_t smem = sizeof(uint32_t) * (size_t)w;
    static PerDevice once;
    once.get([] { return (int)cudaFuncSetAttribute(k_edt_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); });
    (note_launch(), k_edt_row<<<h, 256, smem, s>>>(F, w, h, sl.gcol, any_bg, sl.aux, sl.d, d2_out, dist, cond));
}

}  // namespace hp
