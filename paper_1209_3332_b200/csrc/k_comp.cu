// k_comp.cu -- S8 markers + S9 watershed + S10 BWLabel of the pipeline, one CTA per
// 8-connected component of F (objects are a bag of independent tasks).
//
// Every step of S8-S10 (reading C12/C13) is a fixed point over the graph of
// N8 neighbours INSIDE F, so the 8-connected components of F are independent problems.  The
// global path (k_ws.cu + the tile worklists of k_iwpp.cu, kept for hp_stage_run) pays ~25
// launches and three device-wide worklists per tile for objects of ~100-1000 pixels; here one
// CTA per component iterates each fixed point to convergence inside the component's
// bounding box (the working set stays in L1/L2), using the same monotone update rules:
//   J  = recon(dist - h, dist)           max-clamp relaxation           (h-maxima)
//   zl = flat-zone label = min index      min propagation over equal-J   (RMAX zones)
//   M  = zones with no higher neighbour;  ML = 1 + zone label
//   c  = recon(dist on M else -inf, dist) max-clamp relaxation           (W1)
//   d  = plateau distance                 min-plus relaxation            (W2)
//   L  = min label over the parents       min relaxation                 (W3)
//   split = F minus lines; objects = 8-components of split (min-index labels), area-filtered
// Each relaxation is monotone and converges to the unique fixed point the oracle computes, in
// any order; convergence is detected with __syncthreads_or.  Components of any size work
// (large ones just iterate longer).
#include <cfloat>
#include <climits>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {
namespace {

constexpr int kCT = 256;  // threads per component CTA (8 warps: warp = row, lane = column)

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }

// ---------------------------------------------------------------- component discovery
__global__ void k_comp_roots(const int32_t* __restrict__ lab, int64_t n, int32_t* __restrict__ cnt,
                             int32_t* __restrict__ roots, int32_t cap, int32_t* __restrict__ cid) {
    GRID_LOOP(p, n) {
        if (lab[p] == (int32_t)p) {
            int i = atomicAdd(cnt, 1);
            if (i < cap) {
                roots[i] = (int32_t)p;
                cid[p] = i;
            }
        }
    }
}

__global__ void k_comp_bbox_init(const int32_t* __restrict__ cnt, int32_t cap, int4* __restrict__ bbox) {
    const int n = min(*cnt, cap);
    GRID_LOOP(i, (int64_t)n) bbox[i] = make_int4(INT_MAX, INT_MAX, -1, -1);
}

__global__ void k_comp_bbox(const int32_t* __restrict__ lab, const int32_t* __restrict__ cid, int w, int h,
                            int32_t cap, int4* __restrict__ bbox) {
    const int64_t n = (int64_t)w * h;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = base + threadIdx.x;
        int id = -1, x = 0, y = 0;
        if (p < n) {
            int32_t r = lab[p];
            if (r >= 0) {
                id = cid[r];
                y = (int)(p / w);
                x = (int)(p - (int64_t)y * w);
            }
        }
        unsigned peers = __match_any_sync(0xffffffffu, id);
        if (id < 0 || id >= cap) continue;
        int x0 = __reduce_min_sync(peers, x), y0 = __reduce_min_sync(peers, y);
        int x1 = __reduce_max_sync(peers, x), y1 = __reduce_max_sync(peers, y);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
            int* b = reinterpret_cast<int*>(&bbox[id]);
            atomicMin(&b[0], x0);
            atomicMin(&b[1], y0);
            atomicMax(&b[2], x1);
            atomicMax(&b[3], y1);
        }
    }
}

// ---------------------------------------------------------------- per-component solver
struct CompArgs {
    const uint8_t* F;
    const int32_t* labF;   // root (min index) of each F pixel's 8-component, -1 outside F
    const float* dist;
    float hh;
    int w, h;
    float* J;
    float* c;
    int32_t* zl;           // flat-zone label, then split-object label
    int32_t* d;
    int32_t* L;
    int32_t* aux;          // per-root flags / counters (roots are pixels of the component)
    uint8_t* pm;           // parent bitmask
    uint8_t* split;
    int32_t* labels;       // output (pitch lpitch), zeroed beforehand
    int64_t lpitch;
    int32_t* n_objects;
    int amin, amax;
};

__global__ void __launch_bounds__(kCT) k_components(CompArgs a, const int32_t* __restrict__ cnt, int32_t cap,
                                                    const int32_t* __restrict__ roots,
                                                    const int4* __restrict__ bbox) {
    const int ncomp = min(*cnt, cap);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int w = a.w, h = a.h;
    for (int ci = blockIdx.x; ci < ncomp; ci += gridDim.x) {
        const int32_t root = roots[ci];
        const int4 bb = bbox[ci];
        const int bx0 = bb.x, by0 = bb.y, bx1 = bb.z, by1 = bb.w;
        auto mem = [&](int x, int y) -> bool {
            if (x < 0 || y < 0 || x >= w || y >= h) return false;
            int64_t q = (int64_t)y * w + x;
            return a.labF[q] == root;
        };
        // iterate the component's pixels: warps over rows, lanes over columns
        auto each = [&](auto fn) {
            for (int y = by0 + warp; y <= by1; y += kCT / 32)
                for (int x = bx0 + lane; x <= bx1; x += 32) {
                    int64_t p = (int64_t)y * w + x;
                    if (a.labF[p] == root) fn(x, y, p);
                }
        };
        // run `step` over all pixels until no pixel changes (CTA-wide)
        auto converge = [&](auto step) {
            while (true) {
                int ch = 0;
                each([&](int x, int y, int64_t p) { ch |= step(x, y, p) ? 1 : 0; });
                if (!__syncthreads_or(ch)) break;
            }
        };
        // ---- S8: J = recon(dist - h, dist) restricted to the component
        each([&](int x, int y, int64_t p) {
            float dv = a.dist[p];
            a.J[p] = fminf(__fsub_rn(dv, a.hh), dv);
        });
        __syncthreads();
        converge([&](int x, int y, int64_t p) -> bool {
            float jp = a.J[p], m = a.dist[p], b = jp;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (mem(qx, qy)) b = fmaxf(b, a.J[(int64_t)qy * w + qx]);
            }
            float nv = fminf(b, m);
            if (nv > jp) { a.J[p] = nv; return true; }
            return false;
        });
        // flat zones of J (8-connected, equal J): min-index label propagation
        each([&](int x, int y, int64_t p) { a.zl[p] = (int32_t)p; });
        __syncthreads();
        converge([&](int x, int y, int64_t p) -> bool {
            int32_t z = a.zl[p];
            float jp = a.J[p];
            int32_t b = z;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (!mem(qx, qy)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (a.J[q] == jp) b = min(b, a.zl[q]);
            }
            if (b < z) { a.zl[p] = b; return true; }
            return false;
        });
        // RMAX: a zone is a regional maximum iff none of its pixels has a higher neighbour
        each([&](int x, int y, int64_t p) { if (a.zl[p] == (int32_t)p) a.aux[p] = 0; });
        __syncthreads();
        each([&](int x, int y, int64_t p) {
            float jp = a.J[p];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (mem(qx, qy) && a.J[(int64_t)qy * w + qx] > jp) { a.aux[a.zl[p]] = 1; break; }
            }
        });
        __syncthreads();
        // ---- S9 W1: c = recon(dist on markers else -inf, dist); markers: ML = 1 + zone label
        // (d holds ML temporarily)
        each([&](int x, int y, int64_t p) {
            int32_t z = a.zl[p];
            int32_t ml = a.aux[z] == 0 ? z + 1 : 0;
            a.d[p] = ml;
            a.c[p] = ml ? a.dist[p] : -INFINITY;
        });
        __syncthreads();
        converge([&](int x, int y, int64_t p) -> bool {
            float cp = a.c[p], m = a.dist[p], b = cp;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (mem(qx, qy)) b = fmaxf(b, a.c[(int64_t)qy * w + qx]);
            }
            float nv = fminf(b, m);
            if (nv > cp) { a.c[p] = nv; return true; }
            return false;
        });
        // L initial (markers) before d overwrites ML
        each([&](int x, int y, int64_t p) { a.L[p] = a.d[p] ? a.d[p] : kInfI; });
        __syncthreads();
        // ---- W2: d = 0 markers, 1 with a higher neighbour, else 1 + min equal-c neighbour
        each([&](int x, int y, int64_t p) {
            int32_t v = kInfI;
            if (a.L[p] != kInfI) {
                v = 0;
            } else {
                float cp = a.c[p];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    int qx = x + dx8(j), qy = y + dy8(j);
                    if (mem(qx, qy) && a.c[(int64_t)qy * w + qx] > cp) { v = 1; break; }
                }
            }
            a.d[p] = v;
        });
        __syncthreads();
        converge([&](int x, int y, int64_t p) -> bool {
            int32_t dp = a.d[p];
            if (dp <= 1) return false;
            float cp = a.c[p];
            int32_t b = dp;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (!mem(qx, qy)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (a.c[q] == cp) b = min(b, sat_add(a.d[q], 1));
            }
            if (b < dp) { a.d[p] = b; return true; }
            return false;
        });
        // ---- parents: argmin over neighbours with c(q) >= c(p) of (-c(q), d(q))
        each([&](int x, int y, int64_t p) {
            uint8_t bits = 0;
            if (a.L[p] == kInfI) {
                float cp = a.c[p];
                bool have = false;
                float bc = 0.f;
                int32_t bd = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    int qx = x + dx8(j), qy = y + dy8(j);
                    if (!mem(qx, qy)) continue;
                    int64_t q = (int64_t)qy * w + qx;
                    float cq = a.c[q];
                    if (!(cq >= cp)) continue;
                    int32_t dq = a.d[q];
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
            a.pm[p] = bits;
        });
        __syncthreads();
        // ---- W3: L = min over parents, from +inf
        converge([&](int x, int y, int64_t p) -> bool {
            int pmk = a.pm[p];
            if (!pmk) return false;
            int32_t lp = a.L[p], b = lp;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if ((pmk >> j) & 1) b = min(b, a.L[(int64_t)(y + dy8(j)) * w + x + dx8(j)]);
            if (b < lp) { a.L[p] = b; return true; }
            return false;
        });
        // ---- lines, split
        each([&](int x, int y, int64_t p) {
            int32_t lp = a.L[p];
            uint8_t v = 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (mem(qx, qy) && a.L[(int64_t)qy * w + qx] < lp) { v = 0; break; }
            }
            a.split[p] = v;
        });
        __syncthreads();
        // ---- S10: 8-components of split inside this component, min-index labels
        each([&](int x, int y, int64_t p) { a.zl[p] = a.split[p] ? (int32_t)p : -1; });
        __syncthreads();
        converge([&](int x, int y, int64_t p) -> bool {
            int32_t z = a.zl[p];
            if (z < 0) return false;
            int32_t b = z;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int qx = x + dx8(j), qy = y + dy8(j);
                if (!mem(qx, qy)) continue;
                int32_t zq = a.zl[(int64_t)qy * w + qx];
                if (zq >= 0) b = min(b, zq);
            }
            if (b < z) { a.zl[p] = b; return true; }
            return false;
        });
        each([&](int x, int y, int64_t p) { if (a.zl[p] == (int32_t)p) a.aux[p] = 0; });
        __syncthreads();
        each([&](int x, int y, int64_t p) {
            int32_t z = a.zl[p];
            if (z >= 0) atomicAdd(&a.aux[z], 1);
        });
        __syncthreads();
        each([&](int x, int y, int64_t p) {
            int32_t z = a.zl[p], v = 0;
            if (z >= 0) {
                int area = a.aux[z];
                if (area >= a.amin && area <= a.amax) {
                    v = z + 1;
                    if (z == (int32_t)p) atomicAdd(a.n_objects, 1);
                }
            }
            a.labels[(int64_t)y * a.lpitch + x] = v;
        });
        __syncthreads();
    }
}

}  // namespace

// S8-S10 of the pipeline on F (u8) and dist (f32): labels (zeroed here) + n_objects.
void launch_components(const uint8_t* F, const float* dist, float hh, int amin, int amax, int w, int h,
                       Slot& sl, int32_t* labels, int64_t lpitch, int32_t* n_objects, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    cudaMemsetAsync(n_objects, 0, sizeof(int32_t), s);
    cudaMemset2DAsync(labels, lpitch * sizeof(int32_t), 0, w * sizeof(int32_t), h, s);
    if (n == 0) return;
    CclSrc cs{F, 0, false, nullptr};
    launch_ccl(cs, w, h, 8, sl.lab, nullptr, s);
    int32_t* cnt = sl.cnt32 + 6;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
    const int32_t cap = sl.comp_cap;
    (note_launch(), k_comp_roots<<<grid_for(n), 256, 0, s>>>(sl.lab, n, cnt, sl.comp_root, cap, sl.cid));
    (note_launch(), k_comp_bbox_init<<<grid_for(cap), 256, 0, s>>>(cnt, cap, sl.comp_bbox));
    (note_launch(), k_comp_bbox<<<grid_for(n), 256, 0, s>>>(sl.lab, sl.cid, w, h, cap, sl.comp_bbox));
    CompArgs a{F, sl.lab, dist, hh, w, h, sl.J, sl.c, sl.ML, sl.d, sl.L, sl.aux, sl.pmask, sl.split,
               labels, lpitch, n_objects, amin, amax};
    (note_launch(), k_components<<<148 * 8, kCT, 0, s>>>(a, cnt, cap, sl.comp_root, sl.comp_bbox));
}

}  // namespace hp
