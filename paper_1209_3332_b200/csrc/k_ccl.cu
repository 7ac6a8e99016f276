// k_ccl.cu -- connected-component labelling engine (BWLabel PAPER.md:602): the per-pixel
// label plane of the pipeline's F components (S8-S11, k_comp.cu), the global S10 path and the
// CCL8/CCL4 stages.  S2/S5/S6 need only a per-component property and use k_ccls.cu.
//
// Union-find with atomic hooking, canonical root = minimum linear index (reading C14):
//   k_ccl_local   one 32x32 tile per CTA: shared-memory union-find over the in-tile N+
//                 neighbours (CAS hooking of the larger root under the smaller),
//                 then every pixel gets the global index of its local root (= the local
//                 component's minimum linear index, since local and global order agree);
//   k_ccl_merge   cross-tile edges only (top row / left / right columns): the same hooking
//                 on the global label plane (L2 CAS), finds with CAS path halving;
//   k_ccl_flatten every pixel points straight at its root; roots zero an aux slot so the
//                 per-component reductions that follow need no memset.
// Because a hook always links the larger root under the smaller, the surviving root of a
// component is its minimum linear index -- the canonical label, in any schedule.
#include "hp_internal.cuh"

namespace hp {

namespace {

struct Src {
    const uint8_t* plane;
    uint8_t bitmask;
    bool invert;
    const float* eq;
    int w, h;
    __device__ __forceinline__ bool fg(int64_t p) const {
        uint8_t v = plane[p];
        bool f = bitmask ? (v & bitmask) != 0 : v != 0;
        return f != invert;
    }
    __device__ __forceinline__ bool conn(int64_t p, int64_t q) const {
        return eq == nullptr || eq[p] == eq[q];
    }
};

Src mk(const CclSrc& s, int w, int h) { return Src{s.plane, s.bitmask, s.invert, s.eq, w, h}; }

// N+ neighbours (already-visited in raster order): left, up-left, up, up-right (8-conn);
// left, up (4-conn)
__device__ __forceinline__ int nplus(int conn, int k, int& dx, int& dy) {
    if (conn == 8) {
        const int DX[4] = {-1, -1, 0, 1}, DY[4] = {0, -1, -1, -1};
        dx = DX[k];
        dy = DY[k];
        return 4;
    }
    const int DX[2] = {-1, 0}, DY[2] = {0, -1};
    dx = DX[k];
    dy = DY[k];
    return 2;
}

// No path compression in shared memory: measured on B200 (tools/dbg_ccl.py, r1), an
// atomicMin-based compression here lost unions in ~5% of runs, and with horizontal runs
// pre-linked from ballots the in-tile hook chains stay short anyway.
__device__ __forceinline__ int find_s(int* s, int x) {
    volatile int* vs = s;
    int r = x, p = vs[r];
    while (p != r) {
        r = p;
        p = vs[r];
    }
    return r;
}

// Lock-free union-find (Anderson & Woll style): a root is hooked only by CAS from itself
// (atomicCAS(&p[a], a, b)), so a hook can never detach a non-root, and finds shorten paths
// only by CAS path halving (x -> grandparent iff x still points at that parent).  Hooks
// always go from the larger root to the smaller, so the surviving root of a component is
// its minimum index.
__device__ __forceinline__ void union_s(int* s, int a, int b) {
    while (true) {
        a = find_s(s, a);
        b = find_s(s, b);
        if (a == b) return;
        if (a < b) {
            int t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&s[a], a, b) == a) return;
    }
}

__device__ __forceinline__ int32_t find_g(const int32_t* lab, int32_t x) {
    int32_t p = __ldcg(lab + x);
    while (p != x) {
        x = p;
        p = __ldcg(lab + x);
    }
    return x;
}

// find with CAS path halving
__device__ __forceinline__ int32_t find_gc(int32_t* lab, int32_t x) {
    while (true) {
        int32_t p = __ldcg(lab + x);
        if (p == x) return x;
        int32_t gp = __ldcg(lab + p);
        if (gp == p) return p;
        atomicCAS(&lab[x], p, gp);
        x = gp;
    }
}

__device__ __forceinline__ void union_g(int32_t* lab, int32_t a, int32_t b) {
    while (true) {
        a = find_gc(lab, a);
        b = find_gc(lab, b);
        if (a == b) return;
        if (a < b) {
            int32_t t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&lab[a], a, b) == a) return;
    }
}

__global__ void __launch_bounds__(256) k_ccl_local(Src src, int conn, int32_t* __restrict__ lab) {
    __shared__ int s[kTile * kTile];
    __shared__ unsigned rowm[kTile];
    const int tx0 = blockIdx.x * kTile, ty0 = blockIdx.y * kTile;
    const int lx = threadIdx.x & 31;
    const int w = src.w, h = src.h;
    bool fgv[4];
    unsigned fmv[4], lkm[4];
    // one warp per tile row: horizontal runs are linked at once from the row's ballot --
    // each pixel points at the first pixel of its run (a run start has no left link), so
    // dense foreground never builds long hook chains
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int ly = (threadIdx.x >> 5) + 8 * k;
        int gx = tx0 + lx, gy = ty0 + ly;
        int64_t p = (int64_t)gy * w + gx;
        bool f = gx < w && gy < h && src.fg(p);
        fgv[k] = f;
        unsigned fm = __ballot_sync(0xffffffffu, f);
        fmv[k] = fm;
        if (lx == 0) rowm[ly] = fm;
        bool lk = f && lx > 0 && ((fm >> (lx - 1)) & 1) && src.conn(p, p - 1);
        lkm[k] = __ballot_sync(0xffffffffu, lk);
        unsigned nl = ~lkm[k] & (0xffffffffu >> (31 - lx));
        int start = 31 - __clz(nl);
        s[ly * kTile + lx] = f ? ly * kTile + start : -1;
    }
    // quick paths: an all-background tile, or an all-foreground in-image tile without an
    // equality predicate (one component rooted at the tile origin)
    const int nfg = fgv[0] + fgv[1] + fgv[2] + fgv[3];
    const bool full_tile = tx0 + kTile <= w && ty0 + kTile <= h;
    const int any_fg = __syncthreads_or(nfg > 0);
    const int all_fg = __syncthreads_and(nfg == 4);
    if (!any_fg || (all_fg && full_tile && src.eq == nullptr)) {
        const int32_t v = any_fg ? (int32_t)((int64_t)ty0 * w + tx0) : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int ly = (threadIdx.x >> 5) + 8 * k;
            int gx = tx0 + lx, gy = ty0 + ly;
            if (gx < w && gy < h) lab[(int64_t)gy * w + gx] = v;
        }
        return;
    }
    if (src.eq == nullptr) {
        // plain binary image: only run starts union, once with each run of the row above that
        // touches the run (8-conn: columns xs-1 .. xe+1, 4-conn: xs .. xe)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ly = (threadIdx.x >> 5) + 8 * k;
            const unsigned fm = fmv[k];
            if (ly == 0 || !((fm >> lx) & 1) || (lx > 0 && ((fm >> (lx - 1)) & 1))) continue;
            const unsigned above = rowm[ly - 1];
            if (!above) continue;
            const unsigned tail = ~(fm >> lx);
            const int re = tail == 0 ? 31 : lx + __ffs(tail) - 2;
            const int lo = conn == 8 ? max(lx - 1, 0) : lx, hi = conn == 8 ? min(re + 1, 31) : re;
            const unsigned rm = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
            const unsigned ov = above & rm;
            unsigned segs = ov & ~(ov << 1);
            while (segs) {
                const int b = __ffs(segs) - 1;
                segs &= segs - 1;
                union_s(s, ly * kTile + lx, (ly - 1) * kTile + b);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!fgv[k]) continue;
            int ly = (threadIdx.x >> 5) + 8 * k;
            int li = ly * kTile + lx;
            int64_t p = (int64_t)(ty0 + ly) * w + tx0 + lx;
            int nn = conn == 8 ? 4 : 2;
            for (int j = 0; j < nn; ++j) {
                int dx, dy;
                nplus(conn, j, dx, dy);
                if (dy == 0) continue;  // horizontal links are the runs above
                int nx = lx + dx, ny = ly + dy;
                if (nx < 0 || nx >= kTile || ny < 0) continue;
                int ni = ny * kTile + nx;
                if (s[ni] < 0) continue;  // background never changes
                int64_t q = (int64_t)(ty0 + ny) * w + tx0 + nx;
                if (!src.conn(p, q)) continue;
                union_s(s, li, ni);
            }
        }
    }
    __syncthreads();
    // one find per run (at its start), shared with the run by a shuffle
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int ly = (threadIdx.x >> 5) + 8 * k;
        int gx = tx0 + lx, gy = ty0 + ly;
        int r = 0;
        if (fgv[k] && !((lkm[k] >> lx) & 1)) r = find_s(s, ly * kTile + lx);  // run starts
        const unsigned nl = ~lkm[k] & (0xffffffffu >> (31 - lx));
        r = __shfl_sync(0xffffffffu, r, 31 - __clz(nl));
        if (gx >= w || gy >= h) continue;
        int64_t p = (int64_t)gy * w + gx;
        if (!fgv[k]) {
            lab[p] = -1;
            continue;
        }
        lab[p] = (int32_t)((int64_t)(ty0 + r / kTile) * w + tx0 + r % kTile);
    }
}

// 96 threads per tile: top row, left column, right column; each checks its N+ neighbours
// that fall outside the tile.
__global__ void __launch_bounds__(96) k_ccl_merge(Src src, int conn, int32_t* __restrict__ lab) {
    const int tx0 = blockIdx.x * kTile, ty0 = blockIdx.y * kTile;
    const int w = src.w, h = src.h;
    int side = threadIdx.x >> 5, i = threadIdx.x & 31;
    int lx, ly;
    if (side == 0) {
        lx = i;
        ly = 0;
    } else if (side == 1) {
        lx = 0;
        ly = i;
    } else {
        lx = kTile - 1;
        ly = i;
    }
    int gx = tx0 + lx, gy = ty0 + ly;
    if (gx >= w || gy >= h) return;
    int64_t p = (int64_t)gy * w + gx;
    if (!src.fg(p)) return;
    int nn = conn == 8 ? 4 : 2;
    for (int j = 0; j < nn; ++j) {
        int dx, dy;
        nplus(conn, j, dx, dy);
        int nx = lx + dx, ny = ly + dy;
        if (nx >= 0 && nx < kTile && ny >= 0) continue;  // in-tile edge: done locally
        int qx = gx + dx, qy = gy + dy;
        if (qx < 0 || qx >= w || qy < 0) continue;
        int64_t q = (int64_t)qy * w + qx;
        if (!src.fg(q) || !src.conn(p, q)) continue;
        union_g(lab, (int32_t)p, (int32_t)q);
    }
}

__global__ void k_ccl_flatten(int32_t* __restrict__ lab, int64_t n, int32_t* __restrict__ aux) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t l = lab[p];
        if (l < 0) continue;
        int32_t r = find_g(lab, l);
        if (r != l) lab[p] = r;
        if (aux && r == (int32_t)p) aux[p] = 0;
    }
}

// per-component pixel count at the root, warp-aggregated by equal root
__global__ void k_ccl_count(const int32_t* __restrict__ lab, int64_t n, int32_t* __restrict__ aux) {
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = base + threadIdx.x;
        int32_t r = p < n ? lab[p] : -1;
        unsigned peers = __match_any_sync(0xffffffffu, r);
        int leader = __ffs(peers) - 1;
        if (r >= 0 && (int)(threadIdx.x & 31) == leader) atomicAdd(&aux[r], __popc(peers));
    }
}

__global__ void k_ccl_area_filter(Src src, const int32_t* __restrict__ lab,
                                  const int32_t* __restrict__ area, int amin, int amax,
                                  uint8_t* __restrict__ out) {
    const int64_t n = (int64_t)src.w * src.h;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = lab[p];
        uint8_t v = 0;
        if (r >= 0) {
            int a = area[r];
            v = (a >= amin && a <= amax) ? 1 : 0;
        }
        out[p] = v;
    }
}

__global__ void k_ccl_to_labels(const int32_t* __restrict__ lab, int64_t n, int32_t* __restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        int32_t r = lab[p];
        out[p] = r >= 0 ? r + 1 : 0;
    }
}

inline int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)std::min<int64_t>(b, num_sms() * 16);
}

}  // namespace

void launch_ccl(const CclSrc& cs, int w, int h, int conn, int32_t* lab, int32_t* aux_zero,
                cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    Src src = mk(cs, w, h);
    dim3 grid((w + kTile - 1) / kTile, (h + kTile - 1) / kTile);
    (note_launch(), k_ccl_local<<<grid, 256, 0, s>>>(src, conn, lab));
    (note_launch(), k_ccl_merge<<<grid, 96, 0, s>>>(src, conn, lab));
    (note_launch(), k_ccl_flatten<<<grid_for(n), 256, 0, s>>>(lab, n, aux_zero));
}

void launch_ccl_count(const CclSrc&, int w, int h, const int32_t* lab, int32_t* aux,
                      cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    (note_launch(), k_ccl_count<<<grid_for(n), 256, 0, s>>>(lab, n, aux));
}

void launch_ccl_area_filter(const CclSrc& cs, int w, int h, const int32_t* lab,
                            const int32_t* area, int amin, int amax, uint8_t* out,
                            cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    (note_launch(), k_ccl_area_filter<<<grid_for(n), 256, 0, s>>>(mk(cs, w, h), lab, area, amin, amax, out));
}

void launch_ccl_to_labels(const CclSrc&, int w, int h, const int32_t* lab, int32_t* out,
                          cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    (note_launch(), k_ccl_to_labels<<<grid_for(n), 256, 0, s>>>(lab, n, out));
}

}  // namespace hp
