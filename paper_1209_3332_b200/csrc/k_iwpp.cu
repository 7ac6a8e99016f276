// k_iwpp.cu -- irregular wavefront propagation (IWPP) engine: morphological reconstruction
// (Vincent MR) and the watershed's monotone relaxations (W2
// plateau distance, W3 parent-min labels).
//
// The paper's GPU MR is "a hierarchical queue-based wave-propagation framework"
// (PAPER.md:632-636).  Here the hierarchy is: a device-wide asynchronous queue of 32x32
// TILES (one warp per tile, persistent kernel, device-side termination, no host sync) and,
// inside a tile, warp-synchronous raster / anti-raster row sweeps in shared memory in which
// every row is closed horizontally by a warp-shuffle prefix scan of the row's per-pixel
// update functions (Kogge-Stone over 32 lanes):
//   MR:  f_x(t) = min(mask_x, max(b_x, t))       -- clamps compose into clamps;
//   W2:  f_x(t) = min(a_x, t + k_x), k in {1,inf} -- min-plus along equal-c edges;
//   W3:  f_x(t) = min(a_x, t + k_x), k in {0,inf} -- min along parent edges.
// so a whole row propagates in 5 shuffle steps instead of 32 dependent steps.  A tile is
// re-swept until it is locally stable; then each border pixel that can still improve a
// halo neighbour activates that neighbour tile.  Tile states IDLE/QUEUED/BUSY/BUSY_DIRTY
// guarantee one owner per tile, so tile data are written with plain (L2) stores.
// Every update is a valid monotone propagation, hence any schedule reaches the same unique
// fixed point as the oracle's sequential Vincent / BFS algorithms.
#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "hp_internal.cuh"

namespace hp {

namespace {

constexpr uint32_t ST_IDLE = 0, ST_QUEUED = 1, ST_BUSY = 2, ST_DIRTY = 3;
constexpr int32_t EMPTY = -1;
constexpr int P = kHalo + 1;          // smem row pitch (35 words)
constexpr int kWarps = 4;             // warps per CTA
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ void wl_push(const Worklist& wl, int32_t t) {
    unsigned long long pos = atomicAdd(&wl.ctr[1], 1ull);
    int slot = (int)(pos % (unsigned long long)wl.cap);
    while (atomicCAS(&wl.queue[slot], EMPTY, t) != EMPTY) __nanosleep(64);
}

// Ticket pop: one atomicAdd per pop, no CAS races on the head.  The ticket h names queue
// position h; if that item has not been pushed yet, the holder waits on its own slot until
// it arrives or until nothing is pending (then no push can ever come: -1 = terminate).
__device__ __forceinline__ int32_t wl_pop_ticket(const Worklist& wl, unsigned long long h) {
    const int slot = (int)(h % (unsigned long long)wl.cap);
    int ns = 32;
    while (true) {
        if (*reinterpret_cast<volatile int32_t*>(&wl.queue[slot]) != EMPTY) {
            int32_t v = atomicExch(&wl.queue[slot], EMPTY);
            if (v != EMPTY) return v;
        }
        if (vload(&wl.ctr[2]) == 0ull) return -1;
        __nanosleep(ns);
        if (ns < 1024) ns <<= 1;
    }
}

__device__ __forceinline__ void wl_activate(const Worklist& wl, int32_t t) {
    uint32_t s = *reinterpret_cast<volatile uint32_t*>(&wl.state[t]);
    while (true) {
        if (s == ST_IDLE) {
            uint32_t o = atomicCAS(&wl.state[t], ST_IDLE, ST_QUEUED);
            if (o == ST_IDLE) {
                atomicAdd(&wl.ctr[2], 1ull);
                wl_push(wl, t);
                return;
            }
            s = o;
        } else if (s == ST_BUSY) {
            uint32_t o = atomicCAS(&wl.state[t], ST_BUSY, ST_DIRTY);
            if (o == ST_BUSY) return;
            s = o;
        } else {
            return;  // already queued or already marked dirty
        }
    }
}

// ------------------------------------------------------------------ warp scans
template <class T>
__device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }
template <class T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }

// inclusive prefix (left->right) of clamp functions; returns F_x(-inf) = lo
template <class T>
__device__ __forceinline__ T clamp_scan_lr(T lo, T hi, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T lo_o = __shfl_up_sync(FULL, lo, off), hi_o = __shfl_up_sync(FULL, hi, off);
        if (lane >= off) {
            T nlo = tmin(hi, tmax(lo, lo_o));
            T nhi = tmin(hi, tmax(lo, hi_o));
            lo = nlo;
            hi = nhi;
        }
    }
    return lo;
}
template <class T>
__device__ __forceinline__ T clamp_scan_rl(T lo, T hi, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        T lo_o = __shfl_down_sync(FULL, lo, off), hi_o = __shfl_down_sync(FULL, hi, off);
        if (lane + off < 32) {
            T nlo = tmin(hi, tmax(lo, lo_o));
            T nhi = tmin(hi, tmax(lo, hi_o));
            lo = nlo;
            hi = nhi;
        }
    }
    return lo;
}
__device__ __forceinline__ int minplus_scan_lr(int a, int k, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int a_o = __shfl_up_sync(FULL, a, off), k_o = __shfl_up_sync(FULL, k, off);
        if (lane >= off) {
            a = min(a, sat_add(a_o, k));
            k = sat_add(k, k_o);
        }
    }
    return a;
}
__device__ __forceinline__ int minplus_scan_rl(int a, int k, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int a_o = __shfl_down_sync(FULL, a, off), k_o = __shfl_down_sync(FULL, k, off);
        if (lane + off < 32) {
            a = min(a, sat_add(a_o, k));
            k = sat_add(k, k_o);
        }
    }
    return a;
}

// tile geometry of a warp job
struct TileGeo {
    int x0, y0, w, h;
    __device__ __forceinline__ bool inimg(int r, int c) const {  // smem coords (halo = 0 / 33)
        int gx = x0 - 1 + c, gy = y0 - 1 + r;
        return gx >= 0 && gy >= 0 && gx < w && gy < h;
    }
    __device__ __forceinline__ int64_t gidx(int r, int c) const {
        return (int64_t)(y0 - 1 + r) * w + (x0 - 1 + c);
    }
};

// neighbour-tile bit for a halo cell (r, c) of the 34x34 window
__device__ __forceinline__ uint32_t halo_bit(int r, int c) {
    int dx = c == 0 ? -1 : (c == kHalo - 1 ? 1 : 0);
    int dy = r == 0 ? -1 : (r == kHalo - 1 ? 1 : 0);
    return 1u << nb_index(dx, dy);
}

// Walk the border: for each interior border pixel p and each of its halo neighbours q,
// call f(pr, pc, qr, qc); collect the tile bits for which f returned true.
template <class F>
__device__ __forceinline__ uint32_t border_scan(int lane, F f) {
    uint32_t bits = 0;
    const int c = lane + 1;
    // top and bottom rows
    for (int d = -1; d <= 1; ++d) {
        if (f(1, c, 0, c + d)) bits |= halo_bit(0, c + d);
        if (f(kTile, c, kHalo - 1, c + d)) bits |= halo_bit(kHalo - 1, c + d);
    }
    // left and right columns (corners counted by the rows above)
    const int r = lane + 1;
    for (int d = -1; d <= 1; ++d) {
        if (f(r, 1, r + d, 0)) bits |= halo_bit(r + d, 0);
        if (f(r, kTile, r + d, kHalo - 1)) bits |= halo_bit(r + d, kHalo - 1);
    }
    return __reduce_or_sync(FULL, bits);
}

}  // namespace
}  // namespace hp

#include "iwpp_rules.cuh"

namespace hp {
namespace {

// ------------------------------------------------------------------ the persistent kernel
template <class Rule, class T>
// 5 CTAs x 4 warps per SM: the 38 KB of shared memory per CTA allows 5, and the register
// cap (<= 102 per thread) keeps registers from being the tighter limit
__global__ void __launch_bounds__(kWarps * 32, 5) k_wl_run(Rule rule, Worklist wl) {
    extern __shared__ __align__(16) int smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* sm = reinterpret_cast<T*>(smem_raw) + warp * Rule::kWords;
    while (true) {
        int32_t t = -1;
        if (lane == 0) t = wl_pop_ticket(wl, atomicAdd(&wl.ctr[0], 1ull));
        t = __shfl_sync(FULL, t, 0);
        if (t < 0) break;
        if (lane == 0) atomicExch(&wl.state[t], ST_BUSY);
        const int tx = t % wl.ntx, ty = t / wl.ntx;
        while (true) {
            // rows whose halo improved since this tile's last job (all rows on the first)
            uint32_t rows = 0;
            if (lane == 0) rows = atomicExch(&wl.inrows[t], 0u);
            rows = __shfl_sync(FULL, rows, 0);
            __threadfence();
            __syncwarp();
            uint32_t nbm[8];
            bool changed = false;
            if (rows) changed = rule.process(tx * kTile, ty * kTile, sm, lane, rows, &wl.ctr[4], nbm);
            if (changed) {
                __threadfence();  // tile data visible before the neighbours are told
                uint32_t mine = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (lane == j) mine = nbm[j];
                if (lane < 8 && mine) {
                    int nx = tx + dx8(lane), ny = ty + dy8(lane);
                    if (nx >= 0 && ny >= 0 && nx < wl.ntx && ny < wl.nty) {
                        int nt = ny * wl.ntx + nx;
                        atomicOr(&wl.inrows[nt], mine);
                        wl_activate(wl, nt);
                    }
                }
            }
            __syncwarp();
            int again = 0;
            if (lane == 0) {
                uint32_t o = atomicCAS(&wl.state[t], ST_BUSY, ST_IDLE);
                if (o == ST_BUSY) {
                    atomicAdd(&wl.ctr[2], ~0ull);  // pending -= 1
                } else {
                    atomicExch(&wl.state[t], ST_BUSY);
                    again = 1;
                }
                atomicAdd(&wl.ctr[3], 1ull);
            }
            again = __shfl_sync(FULL, again, 0);
            if (!again) break;
            __threadfence();
        }
    }
}

__global__ void k_wl_reset(Worklist wl, int seed_all) {
    const int n = wl.ntx * wl.nty;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < wl.cap; i += gridDim.x * blockDim.x) {
        if (i < n) {
            wl.state[i] = seed_all ? ST_QUEUED : ST_IDLE;
            wl.inrows[i] = seed_all ? 0xffffffffu : 0u;
        }
        wl.queue[i] = (seed_all && i < n) ? i : EMPTY;
    }
    if (blockIdx.x == 0 && threadIdx.x < 8)
        wl.ctr[threadIdx.x] = (seed_all && (threadIdx.x == 1 || threadIdx.x == 2)) ? (unsigned long long)n : 0ull;
}

// seed the tiles that contain any nonzero mask pixel (one warp per tile)
__global__ void k_wl_seed_mask(Worklist wl, const uint8_t* __restrict__ mask, int w, int h) {
    const int n = wl.ntx * wl.nty;
    const int lane = threadIdx.x & 31;
    for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += (gridDim.x * blockDim.x) >> 5) {
        int tx = t % wl.ntx, ty = t / wl.ntx;
        int gx = tx * kTile + lane;
        bool any = false;
        if (gx < w)
            for (int r = 0; r < kTile; ++r) {
                int gy = ty * kTile + r;
                if (gy >= h) break;
                any |= mask[(int64_t)gy * w + gx] != 0;
            }
        if (__any_sync(FULL, any) && lane == 0) {
            wl.state[t] = ST_QUEUED;
            wl.inrows[t] = 0xffffffffu;
            unsigned long long pos = atomicAdd(&wl.ctr[1], 1ull);
            atomicAdd(&wl.ctr[2], 1ull);
            wl.queue[pos] = t;
        }
    }
}

template <class Rule, class T>
void run_rule(const Rule& rule, const Worklist& wl, cudaStream_t s) {
    const size_t smem = sizeof(T) * Rule::kWords * kWarps;
    static PerDevice once;
    const int blocks = once.get([&] {
        cudaFuncSetAttribute(k_wl_run<Rule, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int per_sm = 0, dev = 0, nsm = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wl_run<Rule, T>, kWarps * 32, smem);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        // Measured on B200 (tools/diag_iwpp.py): the recon is throughput-bound on tile jobs
        // (time ~ 1 / resident warps), so the persistent grid fills every SM to occupancy.
        // HP_WL_CTAS_PER_SM caps it (experiments with co-running slots).
        int want = 64;
        if (const char* e = getenv("HP_WL_CTAS_PER_SM")) want = atoi(e);
        if (want < 1) want = 1;
        return nsm * std::min(want, per_sm > 0 ? per_sm : 1);
    });
    int ntiles = wl.ntx * wl.nty;
    int b = std::min(blocks, (ntiles + kWarps - 1) / kWarps);
    if (b < 1) b = 1;
    (note_launch(), k_wl_run<Rule, T><<<b, kWarps * 32, smem, s>>>(rule, wl));
}

// ------------------------------------------------------------------ init kernels
__global__ void k_copy_min_u8(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                              uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = min(a[i], b[i]);
}

// S4 top-hat: cand = (g - recon > g1) & !rbc
__global__ void k_tophat(const uint8_t* __restrict__ g, const uint8_t* __restrict__ R,
                         const uint8_t* __restrict__ rbc, int g1, int64_t n, uint8_t* __restrict__ cand) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        cand[i] = (((int)g[i] - (int)R[i]) > g1 && !rbc[i]) ? 1 : 0;
}

__global__ void k_recon_init_f32(const float* __restrict__ marker, const float* __restrict__ mask,
                                 const uint8_t* __restrict__ dom, int64_t n, float* __restrict__ R) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        R[i] = (dom == nullptr || dom[i]) ? fminf(marker[i], mask[i]) : NAN;
}

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, num_sms() * 16); }

// the tile grid follows the current image, not the context's maximum size
Worklist sized(const Worklist& wl, int w, int h) {
    Worklist r = wl;
    r.ntx = (w + kTile - 1) / kTile;
    r.nty = (h + kTile - 1) / kTile;
    return r;
}

}  // namespace

void launch_recon_init_f32(const float* marker, const float* mask, const uint8_t* dom, int64_t n, float* R,
                           cudaStream_t s) {
    if (n) (note_launch(), k_recon_init_f32<<<grid_for(n), 256, 0, s>>>(marker, mask, dom, n, R));
}

void wl_init_all(const Worklist& wl0, int w, int h, cudaStream_t s) {
    Worklist wl = sized(wl0, w, h);
    (note_launch(), k_wl_reset<<<grid_for(wl.cap), 256, 0, s>>>(wl, 1));
}

void wl_init_from_mask(const Worklist& wl0, const uint8_t* mask, int w, int h, cudaStream_t s) {
    Worklist wl = sized(wl0, w, h);
    (note_launch(), k_wl_reset<<<grid_for(wl.cap), 256, 0, s>>>(wl, 0));
    int n = wl.ntx * wl.nty;
    (note_launch(), k_wl_seed_mask<<<(int)std::min<int64_t>((n + 7) / 8, num_sms() * 16), 256, 0, s>>>(wl, mask, w, h));
}

void launch_recon_init_u8(const uint8_t* marker, const uint8_t* mask, uint8_t* R, int w, int h,
                          cudaStream_t s) {
    int64_t n = (int64_t)w * h;
    if (n) (note_launch(), k_copy_min_u8<<<grid_for(n), 256, 0, s>>>(marker, mask, n, R));
}

void launch_recon_u8(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl,
                     cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    wl_init_all(wl, w, h, s);
    RuleMR8 rule{mask, R, w, h};
    run_rule<RuleMR8, int>(rule, sized(wl, w, h), s);
}

void launch_recon_f32(const float* mask, const uint8_t* dom, float* R, int w, int h,
                      const Worklist& wl, bool init_from_mask_tiles, cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    if (init_from_mask_tiles && dom)
        wl_init_from_mask(wl, dom, w, h, s);
    else
        wl_init_all(wl, w, h, s);
    RuleMRf rule{mask, R, dom, w, h};
    run_rule<RuleMRf, int>(rule, sized(wl, w, h), s);
}

void launch_plateau_dist(const float* c, int32_t* d, int w, int h, const Worklist& wl,
                         const uint8_t* F, cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    wl_init_from_mask(wl, F, w, h, s);
    RuleW2 rule{c, d, w, h};
    run_rule<RuleW2, int>(rule, sized(wl, w, h), s);
}

void launch_parent_min(const uint8_t* pm, int32_t* L, int w, int h, const Worklist& wl,
                       const uint8_t* F, cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    wl_init_from_mask(wl, F, w, h, s);
    RuleW3 rule{pm, L, w, h};
    run_rule<RuleW3, int>(rule, sized(wl, w, h), s);
}

void launch_tophat(const uint8_t* g, const uint8_t* R, const uint8_t* rbc, int g1, int w, int h,
                   uint8_t* cand, cudaStream_t s) {
    int64_t n = (int64_t)w * h;
    if (n) (note_launch(), k_tophat<<<grid_for(n), 256, 0, s>>>(g, R, rbc, g1, n, cand));
}

}  // namespace hp
