// k_comp.cu -- the pipeline's per-component stages, S6 and S7-S11 (PAPER.md:598-604,
// 223-224: objects are a bag of tasks).
//
// From S6 on every step is local to connected components: a hole of FillHoles is bounded by
// ONE 8-connected candidate component, so it lies in that component's bounding box; every
// step of S7-S10 (readings C11-C13) is a fixed point over the N8 neighbours
// INSIDE F; S11 is per object.  S5 (k_ccls.cu) lists the kept candidate components (root =
// minimum linear index, bounding box, area); two launches then solve them in windows (bbox +
// 1-px ring), taken off dynamic queues -- one WARP per window <= 576 px (~99% of nuclei), one
// 4-warp block per window <= 2432 px, in shared memory; bigger windows (and object-list
// overflows) in one block over global-memory scratch with the same code (the solvers are
// templated on the window storage):
//   k_fill_fused  S6: A = the component (8-connected union-find among the window's candidate
//                 pixels, skipped when the window holds exactly its area); holes from the
//                 Euler number (bit-quads) or a 4-connected union-find of the rest seeded at
//                 the ring / tile border; F |= A | holes, each F pixel's word atomicMin(root)
//                 (an island enclosed in a hole resolves to its encloser, as a CCL of F
//                 would), enclosed candidates marked in enc;
//   k_comp_fused  S7-S11 per component not in enc: members = pixels whose word is the root;
//                 exact EDT by brute force over the window's boundary pixels; J, flat zones,
//                 RMAX, markers, W1-W3, lines, BWLabel by monotone relaxations / union-find in
//                 shared memory; the 36 features of each kept object (feat_common.cuh).
// Rows land in a staging table and k_rows_scatter orders them by label.  Every relaxation is
// monotone toward a unique fixed point, so the result equals the oracle's.
#include <climits>
#if defined(HP_FILL_DBG) || defined(HP_COMP_DBG)
#include <cstdio>
#endif

#include "feat_common.cuh"

namespace hp {
namespace {


#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, num_sms() * 16); }

struct CompArgs {
    const int32_t* labF;   // per F pixel: the root of its F component (written by S6), else ~0
    const uint8_t* enc;    // S6: candidate pixels enclosed in another component's hole
    const uint8_t* g;      // for features
    const uint8_t* edge;   // Canny edges of g (0/1), for features
    float hh;
    int w, h;
    int amin, amax;
    int32_t* labels;       // output (pitch lpitch), zeroed beforehand
    int64_t lpitch;
    int32_t* n_objects;
    // staging table of rows (any order) and its counter
    int32_t* rows_cnt;
    int32_t rows_cap;
    int32_t* row_label;
    int32_t* row_flags;
    float* row_feat;
    int do_features;
    // components for the global-memory (one block) path: huge windows, object-list overflow
    int32_t* ovf_cnt;
    int32_t* ovf_list;
};

// find with CAS path halving (x -> grandparent iff x still points at that parent; safe beside
// concurrent CAS hooks, which only ever re-point roots)
__device__ __forceinline__ int cfind(int* P, int x) {
    volatile int* vp = P;
    while (true) {
        const int p = vp[x];
        if (p == x) return x;
        const int gp = vp[p];
        if (gp == p) return p;
        atomicCAS(&P[x], p, gp);
        x = gp;
    }
}
__device__ __forceinline__ void cunion(int* P, int a, int b) {
    while (true) {
        a = cfind(P, a);
        b = cfind(P, b);
        if (a == b) return;
        if (a < b) {
            int t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&P[a], a, b) == a) return;
    }
}

// The window forests start from horizontal runs: every pixel of a set first points at its left
// neighbour in the set, then ceil(log2 WX) pointer-jumping rounds make it point at the start of
// its run (the run's minimum index, so min-index roots survive), and only then do the other
// neighbours cunion.  (r1-r2 let every pixel cunion with its left neighbour: a warp's lanes
// hooking consecutive pixels at once chained each run into a list that every later find walked
// -- instrumented r2: 50-170 us for a 400-pixel S6 window.)  left(li): li - 1 is in li's set
// and li is not the first column; each(fn): fn over the set.
template <class Team, class Each, class Left>
__device__ __forceinline__ void link_runs(const Team& team, int* P, int WX, Each each, Left left) {
    each([&](int li) { P[li] = left(li) ? li - 1 : li; });
    team.sync();
    for (int r = 1; r < WX; r <<= 1) {
        each([&](int li) { P[li] = P[P[li]]; });
        team.sync();
    }
}

__device__ __forceinline__ void write_row(const CompArgs& a, int32_t label, int border, const double* f) {
    int slot = atomicAdd(a.rows_cnt, 1);
    if (slot < a.rows_cap) {
        a.row_label[slot] = label;
        a.row_flags[slot] = border ? HP_OBJ_TOUCHES_BORDER : 0;
        for (int k = 0; k < HP_NFEAT; ++k) a.row_feat[(int64_t)slot * HP_NFEAT + k] = (float)f[k];
    }
}

#ifdef HP_COMP_DBG
__device__ unsigned long long g_compdbg[13];
__device__ unsigned int g_compdbg_done;
#endif

// ---------------------------------------------------------------- shared-memory path
// Per-team window storage (4-byte planes first for alignment); 19 B per window pixel.
template <int CAP, int KO>
struct CompSm {
    using list_t = int16_t;
    static constexpr int kKO = KO;
    float dist[CAP];
    float A[CAP];      // J, then c
    int32_t B[CAP];    // zone union-find, then L, then object union-find
    int32_t C[CAP];    // zone flags, then d, then object areas
    int16_t list[CAP];  // member pixels (window indices), compacted once
    uint8_t mem[CAP];
    uint8_t pm[CAP];
    uint8_t sp[CAP];
    int nmem;
    int nbnd;
    int nobj;
    int objroot[KO];
    FeatSmem fs;
};

// The same per-window storage in global memory, for windows too large for shared memory (one
// block processes them one after another; the planes are slot scratch of (W+2)(H+2) pixels).
struct CompGm {
    using list_t = int32_t;
    static constexpr int kKO = 1 << 30;  // objroot holds up to one entry per window pixel
    float* dist;
    float* A;
    int32_t* B;
    int32_t* C;
    int32_t* list;
    uint8_t* mem;
    uint8_t* pm;
    uint8_t* sp;
    int& nmem;
    int& nbnd;
    int& nobj;
    int32_t* objroot;
    FeatSmem& fs;
};

struct BigScratch {
    float* dist;
    float* A;
    int32_t* B;
    int32_t* C;
    int32_t* list;
    int32_t* objroot;
    uint8_t* mem;
    uint8_t* pm;
    uint8_t* sp;
};

inline BigScratch carve_big(const Slot& sl) {
    const int64_t n = sl.big_px;
    uint8_t* p = sl.big_scratch;
    BigScratch b;
    b.dist = reinterpret_cast<float*>(p);
    b.A = reinterpret_cast<float*>(p + 4 * n);
    b.B = reinterpret_cast<int32_t*>(p + 8 * n);
    b.C = reinterpret_cast<int32_t*>(p + 12 * n);
    b.list = reinterpret_cast<int32_t*>(p + 16 * n);
    b.objroot = reinterpret_cast<int32_t*>(p + 20 * n);
    b.mem = p + 24 * n;
    b.pm = p + 25 * n;
    b.sp = p + 26 * n;
    return b;
}

// Solve S8-S11 of one component in a team's shared memory.  Returns false (nothing written)
// if the component must go to the global path instead.
template <class Team, class St>
__device__ bool comp_solve(const Team& team, St& S, TeamRed& red, const CompArgs& a,
                           int32_t root, int4 bb) {
    const int w = a.w, h = a.h;
    const int tr = team.rank();
    constexpr int TS = Team::size;
    const int wx0 = bb.x - 1, wy0 = bb.y - 1;
    const int WX = bb.z - bb.x + 3, WY = bb.w - bb.y + 3;
    const int NWIN = WX * WY;
    const int nbo[8] = {-WX - 1, -WX, -WX + 1, -1, 1, WX - 1, WX, WX + 1};
    auto gidx = [&](int li) -> int32_t {
        int ly = li / WX, lx = li - ly * WX;
        return (int32_t)((int64_t)(wy0 + ly) * w + (wx0 + lx));
    };
#ifdef HP_COMP_DBG  // experiment: clock64 per phase, summed over the launch (tools/gpu_r02cd2.sh)
    long long ct[12];
    int nct = 0;
    struct RepC {
        long long* ct; int* nct; int tr;
        __device__ ~RepC() {
            const long long e = clock64();
            if (tr == 0 && *nct == 11) {
                for (int k = 0; k < 10; ++k) atomicAdd(&g_compdbg[k], (unsigned long long)(ct[k + 1] - ct[k]));
                atomicAdd(&g_compdbg[10], (unsigned long long)(e - ct[10]));
                atomicAdd(&g_compdbg[11], (unsigned long long)(e - ct[0]));
                atomicAdd(&g_compdbg[12], 1ull);
            }
        }
    } repc_{ct, &nct, tr};
#define COMP_T() ct[nct++] = clock64()
#else
#define COMP_T()
#endif
    COMP_T();
    // ---- stage the window (ring pixels are never members: no bounds checks later) and list
    // the members, so every later pass touches members only
    if (tr == 0) {
        S.nobj = 0;
        S.nmem = 0;
        S.nbnd = 0;
    }
    team.sync();
    int nmem = 0;
    for (int base = 0; base < NWIN; base += TS) {
        const int li = base + tr;
        bool m = false;
        if (li < NWIN) {
            const int ly = li / WX, lx = li - ly * WX;
            const int gx = wx0 + lx, gy = wy0 + ly;
            const bool in = gx >= 0 && gy >= 0 && gx < w && gy < h;
            if (in) m = a.labF[(int64_t)gy * w + gx] == root;
            S.mem[li] = m;
            S.pm[li] = in;  // (scratch until the parent pass)
        }
        if constexpr (TS == 32) {  // warp team: ballot compaction (window order)
            const unsigned bal = __ballot_sync(0xffffffffu, m);
            if (m) S.list[nmem + __popc(bal & ((1u << tr) - 1u))] = (typename St::list_t)li;
            nmem += __popc(bal);
        } else {
            if (m) S.list[atomicAdd(&S.nmem, 1)] = (typename St::list_t)li;
        }
    }
    team.sync();
    if constexpr (TS != 32) nmem = S.nmem;
    auto each = [&](auto fn) {
        for (int k = tr; k < nmem; k += TS) fn((int)S.list[k]);
    };
    COMP_T();
    // ---- S7 EDT of the members, exactly, inside the window (reading C11).
    // For a member p at distance d from the nearest background pixel q, the open disk of
    // radius d around p is foreground and 8-connected, so it lies in p's component; one
    // step from q toward p lands in that disk, so q is 8-adjacent to the component: every
    // nearest background pixel is an in-tile non-member of the window touching a member.  No
    // such pixel = the component is the whole tile = no background: +inf.
    if constexpr (St::kKO == CompGm::kKO) {
        // windows too big for shared memory (a big component under non-default area bounds):
        // the brute force below is O(members x boundary); use an exact separable EDT of the
        // window instead (Meijster: per column the distance to the nearest background pixel,
        // then per row the lower envelope of (x - i)^2 + g(i)^2 with integer separators).
        // The window holds every nearest background pixel (see above), so the result is the
        // same integer d2.  Background = in-tile non-member window pixels.
        const int INF = WX + WY;  // larger than any in-window distance
        int32_t* g = S.B;         // column distances
        int32_t* sv = S.C;        // per row: envelope indices
        int32_t* tv = reinterpret_cast<int32_t*>(S.A);  // per row: envelope starts
        int anybg = 0;
        for (int x = tr; x < WX; x += TS) {
            int d = INF;
            for (int y = 0; y < WY; ++y) {
                const int li = y * WX + x;
                if (!S.mem[li] && S.pm[li]) { d = 0; anybg = 1; }
                else if (d < INF) ++d;
                g[li] = d;
            }
            d = INF;
            for (int y = WY - 1; y >= 0; --y) {
                const int li = y * WX + x;
                if (g[li] == 0) d = 0;
                else if (d < INF) ++d;
                if (d < g[li]) g[li] = d;
            }
        }
        anybg = team.reduce(anybg, red.i, OpMax());
        team.sync();
        for (int y = tr; y < WY; y += TS) {
            int32_t* srow = sv + y * WX;
            int32_t* trow = tv + y * WX;
            const int32_t* grow = g + y * WX;
            auto f = [&](int x, int i) { return (int64_t)(x - i) * (x - i) + (int64_t)grow[i] * grow[i]; };
            auto sep = [&](int i, int u) {
                return (int)(((int64_t)u * u - (int64_t)i * i + (int64_t)grow[u] * grow[u] - (int64_t)grow[i] * grow[i]) /
                             (2 * (int64_t)(u - i)));
            };
            int q = 0;
            srow[0] = 0;
            trow[0] = 0;
            for (int u = 1; u < WX; ++u) {
                while (q >= 0 && f(trow[q], srow[q]) > f(trow[q], u)) --q;
                if (q < 0) {
                    q = 0;
                    srow[0] = u;
                } else {
                    const int wv = 1 + sep(srow[q], u);
                    if (wv < WX) {
                        ++q;
                        srow[q] = u;
                        trow[q] = wv;
                    }
                }
            }
            for (int u = WX - 1; u >= 0; --u) {
                const int li = y * WX + u;
                if (S.mem[li])
                    S.dist[li] = anybg ? __fsqrt_rn(__uint2float_rn((uint32_t)f(u, srow[q]))) : INFINITY;
                if (u == trow[q]) --q;
            }
        }
        team.sync();
    } else {
        int nb = 0;
        int32_t* bl = S.C;  // boundary pixels, (ly << 16) | lx
        for (int base = 0; base < NWIN; base += TS) {
            const int li = base + tr;
            bool bnd = false;
            if (li < NWIN && !S.mem[li] && S.pm[li]) {
                const int ly = li / WX, lx = li - ly * WX;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int qx = lx + dx8(j), qy = ly + dy8(j);
                    if (qx >= 0 && qy >= 0 && qx < WX && qy < WY && S.mem[qy * WX + qx]) bnd = true;
                }
            }
            const int code = bnd ? (((li / WX) << 16) | (li % WX)) : 0;
            if constexpr (TS == 32) {
                const unsigned bal = __ballot_sync(0xffffffffu, bnd);
                if (bnd) bl[nb + __popc(bal & ((1u << tr) - 1u))] = code;
                nb += __popc(bal);
            } else {
                if (bnd) bl[atomicAdd(&S.nbnd, 1)] = code;
            }
        }
        team.sync();
        if constexpr (TS != 32) nb = S.nbnd;
        each([&](int li) {
            const int ly = li / WX, lx = li - ly * WX;
            uint32_t best = 0xffffffffu;
            for (int k = 0; k < nb; ++k) {
                const int c = bl[k];
                const int dx = (c & 0xffff) - lx, dy = (c >> 16) - ly;
                best = min(best, (uint32_t)(dx * dx + dy * dy));
            }
            S.dist[li] = nb == 0 ? INFINITY : __fsqrt_rn(__uint2float_rn(best));
        });
        team.sync();
    }
    auto converge = [&](auto step) {
        while (true) {
            int ch = 0;
            each([&](int li) { ch |= step(li) ? 1 : 0; });
            if (!team.any(ch)) break;
        }
    };
    COMP_T();
    // ---- S8: J = recon(dist - h, dist)
    each([&](int li) { S.A[li] = fminf(__fsub_rn(S.dist[li], a.hh), S.dist[li]); });
    team.sync();
    converge([&](int li) -> bool {
        float jp = S.A[li], b = jp;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (S.mem[li + nbo[j]]) b = fmaxf(b, S.A[li + nbo[j]]);
        float nv = fminf(b, S.dist[li]);
        if (nv > jp) { S.A[li] = nv; return true; }
        return false;
    });
    // flat zones of J: union-find over N+ neighbours with equal J (min-index roots); members
    // never sit in the ring, so li - 1 is in the window row
    link_runs(team, S.B, WX, each, [&](int li) { return S.mem[li - 1] && S.A[li - 1] == S.A[li]; });
    each([&](int li) {
        float jp = S.A[li];
#pragma unroll
        for (int j = 0; j < 3; ++j) {  // (-1,-1) (0,-1) (1,-1); (-1,0) is the run
            int q = li + nbo[j];
            if (S.mem[q] && S.A[q] == jp) cunion(S.B, li, q);
        }
    });
    team.sync();
    each([&](int li) { S.C[li] = cfind(S.B, li); });
    team.sync();
    each([&](int li) { S.B[li] = S.C[li]; });
    team.sync();
    // RMAX: zone flag = some pixel of the zone has a higher neighbour
    each([&](int li) { if (S.B[li] == li) S.C[li] = 0; });
    team.sync();
    each([&](int li) {
        float jp = S.A[li];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int q = li + nbo[j];
            if (S.mem[q] && S.A[q] > jp) { S.C[S.B[li]] = 1; break; }
        }
    });
    team.sync();
    COMP_T();
    // ---- markers -> L initial (ML = 1 + global min index of the zone, else inf) and W1 init
    each([&](int li) { S.pm[li] = S.C[S.B[li]] == 0; });  // staged: zone flags live at roots
    team.sync();
    each([&](int li) {
        const int32_t ml = S.pm[li] ? gidx(S.B[li]) + 1 : kInfI;
        S.B[li] = ml;
        S.A[li] = ml != kInfI ? S.dist[li] : -INFINITY;
    });
    team.sync();
    COMP_T();
    // ---- S9 W1: c = recon(dist on markers else -inf, dist)
    converge([&](int li) -> bool {
        float cp = S.A[li], b = cp;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (S.mem[li + nbo[j]]) b = fmaxf(b, S.A[li + nbo[j]]);
        float nv = fminf(b, S.dist[li]);
        if (nv > cp) { S.A[li] = nv; return true; }
        return false;
    });
    COMP_T();
    // ---- W2: plateau distance (markers: B != inf)
    each([&](int li) {
        int32_t v = kInfI;
        if (S.B[li] != kInfI) {
            v = 0;
        } else {
            float cp = S.A[li];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int q = li + nbo[j];
                if (S.mem[q] && S.A[q] > cp) { v = 1; break; }
            }
        }
        S.C[li] = v;
    });
    team.sync();
    converge([&](int li) -> bool {
        int32_t dp = S.C[li];
        if (dp <= 1) return false;
        float cp = S.A[li];
        int32_t b = dp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int q = li + nbo[j];
            if (S.mem[q] && S.A[q] == cp) b = min(b, sat_add(S.C[q], 1));
        }
        if (b < dp) { S.C[li] = b; return true; }
        return false;
    });
    COMP_T();
    // ---- parents: argmin over neighbours with c(q) >= c(p) of (-c(q), d(q))
    each([&](int li) {
        uint8_t bits = 0;
        if (S.B[li] == kInfI) {
            float cp = S.A[li];
            bool have = false;
            float bc = 0.f;
            int32_t bd = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int q = li + nbo[j];
                if (!S.mem[q]) continue;
                float cq = S.A[q];
                if (!(cq >= cp)) continue;
                int32_t dq = S.C[q];
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
        S.pm[li] = bits;
    });
    team.sync();
    COMP_T();
    // ---- W3: L = min over parents
    converge([&](int li) -> bool {
        int pmk = S.pm[li];
        if (!pmk) return false;
        int32_t lp = S.B[li], b = lp;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if ((pmk >> j) & 1) b = min(b, S.B[li + nbo[j]]);
        if (b < lp) { S.B[li] = b; return true; }
        return false;
    });
    COMP_T();
    // ---- lines, split
    each([&](int li) {
        int32_t lp = S.B[li];
        uint8_t v = 1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int q = li + nbo[j];
            if (S.mem[q] && S.B[q] < lp) { v = 0; break; }
        }
        S.sp[li] = v;
    });
    team.sync();
    COMP_T();
    // ---- S10: objects = 8-components of split (union-find), area filter
    link_runs(team, S.B, WX, each, [&](int li) { return S.sp[li] && S.mem[li - 1] && S.sp[li - 1]; });
    each([&](int li) {
        if (!S.sp[li]) return;
#pragma unroll
        for (int j = 0; j < 3; ++j) {  // (-1,-1) (0,-1) (1,-1); (-1,0) is the run
            int q = li + nbo[j];
            if (S.mem[q] && S.sp[q]) cunion(S.B, li, q);
        }
    });
    team.sync();
    each([&](int li) { S.C[li] = S.sp[li] ? cfind(S.B, li) : -1; });
    team.sync();
    each([&](int li) { S.B[li] = S.C[li]; });  // object root (local) or -1
    team.sync();
    each([&](int li) { if (S.B[li] == li) S.C[li] = 0; });
    team.sync();
    each([&](int li) { if (S.B[li] >= 0) atomicAdd(&S.C[S.B[li]], 1); });
    team.sync();
    each([&](int li) {
        if (S.B[li] == li && S.C[li] >= a.amin && S.C[li] <= a.amax) {
            int k = atomicAdd(&S.nobj, 1);
            if (k < St::kKO) S.objroot[k] = li;
        }
    });
    team.sync();
    const int nobj = S.nobj;
    if (nobj > St::kKO) return false;  // too many objects for the list: global path instead
    each([&](int li) {
        int r = S.B[li];
        int32_t v = 0;
        if (r >= 0 && S.C[r] >= a.amin && S.C[r] <= a.amax) v = gidx(r) + 1;
        int ly = li / WX, lx = li - ly * WX;
        a.labels[(int64_t)(wy0 + ly) * a.lpitch + (wx0 + lx)] = v;
    });
    if (tr == 0 && nobj) atomicAdd(a.n_objects, nobj);
    team.sync();
    COMP_T();
    // ---- S11: features of each kept object
    if (a.do_features) {
        for (int k = 0; k < nobj; ++k) {
            const int r = S.objroot[k];
            // object_features only asks about pixels of the component's bounding box and the
            // 4- / 8-neighbours of object pixels, all inside the window (bbox + 1-px ring): no
            // bounds checks
            auto inP = [&](int x, int y) -> bool {
                const int li = (y - wy0) * WX + (x - wx0);  // non-members hold stale values: test mem first
                return S.mem[li] && S.B[li] == r;
            };
            int border = 0;
            object_features(team, inP, a.g, a.edge, w, h, bb.x, bb.y, bb.z, bb.w, S.fs, red, S.fs.f, &border);
            if (tr == 0) write_row(a, gidx(r) + 1, border, S.fs.f);
            team.sync();
        }
    }
    return true;
}

#ifndef HP_CAPW
#define HP_CAPW 576  // 4 blocks of 4 warps per SM (measured r1: 0.54 ms vs 0.57 at 640)
#define HP_CAPB 2432
#endif
constexpr int kCapW = HP_CAPW, kKoW = 48;  // warp team: windows up to kCapW px (~99% of nuclei)
constexpr int kWarpsPB = 4;
constexpr int kCapB = HP_CAPB, kKoB = 160; // block team (4 warps): the same shared memory, one window
static_assert(sizeof(CompSm<kCapB, kKoB>) <= kWarpsPB * sizeof(CompSm<kCapW, kKoW>), "block window too big");

// S6 needs only 11 of the 21 B per window pixel (and no feature scratch): its own, smaller
// per-team storage lets twice as many fill blocks share an SM (r2: the fill kernel's teams are
// latency-bound on dependent shared-memory passes; 16 warps per SM left them exposed).
template <int CAP>
struct FillSm {
    int32_t B[CAP];
    int32_t C[CAP];
    uint8_t mem[CAP];
    uint8_t pm[CAP];
    uint8_t sp[CAP];
};
constexpr size_t kFillSmem = sizeof(FillSm<kCapB>) > kWarpsPB * sizeof(FillSm<kCapW>) ? sizeof(FillSm<kCapB>)
                                                                                          : kWarpsPB * sizeof(FillSm<kCapW>);

__device__ __forceinline__ int win_px(int4 bb) { return (bb.z - bb.x + 3) * (bb.w - bb.y + 3); }

__device__ __forceinline__ void to_global(const CompArgs& a, int ci) {
    int k = atomicAdd(a.ovf_cnt, 1);
    a.ovf_list[k] = ci;
}

// windows > kCapW go to the block list, windows > kCapB straight to the global path
// S5 components -> block list (windows > kCapW) / global-memory list (> kCapB); islands enclosed
// in another component's hole (enc at their root) are solved with their encloser
__global__ void k_comp_classify(CompArgs a, const int32_t* __restrict__ cnt, int32_t cap,
                                const int32_t* __restrict__ roots, const int4* __restrict__ bbox,
                                int32_t* __restrict__ big, int32_t* __restrict__ nbig) {
    const int n = min(*cnt, cap);
    GRID_LOOP(ci, (int64_t)n) {
        if (a.enc[roots[ci]]) continue;
        const int wp = win_px(bbox[ci]);
        if (wp > kCapB) to_global(a, (int)ci);
        else if (wp > kCapW) big[atomicAdd(nbig, 1)] = (int)ci;
    }
}

// One launch for every shared-memory component: each block first takes big components off
// the block list (whole-block team), then its warps take small components one at a time off
// the component list (warp teams) -- dynamic queues, so the few big windows run beside the
// many small ones instead of as a serial tail.
// persistent grids: blocks per SM of the fused kernels (each block holds kWarpsPB windows of
// shared memory while it runs, which the concurrent slots' kernels then cannot use)
#ifndef HP_COMP_BPS
#define HP_COMP_BPS 4
#endif
#ifndef HP_FILL_BPS
#define HP_FILL_BPS 4  // fill blocks per SM (FillSm: ~27 KB each; r2 sweep 2 / 3 / 4 / 8 within 1%, 4 ahead in 3 of 4 pairs)
#endif

#ifndef HP_COMP_MINB
#define HP_COMP_MINB 4  // launch-bounds min blocks of k_comp_fused (4: 128 registers, some spills)
#endif

__global__ void __launch_bounds__(kWarpsPB * 32, HP_COMP_MINB) k_comp_fused(CompArgs a, const int32_t* __restrict__ cnt,
                                                                int32_t cap, const int32_t* __restrict__ roots,
                                                                const int4* __restrict__ bbox,
                                                                const int32_t* __restrict__ big,
                                                                const int32_t* __restrict__ nbig_p,
                                                                int32_t* __restrict__ heads) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ TeamRed red;
    __shared__ int s_job;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        auto& S = *reinterpret_cast<CompSm<kCapB, kKoB>*>(smem_raw);
        const TeamCTA<kWarpsPB * 32> team;
        const int nbig = *nbig_p;
        while (true) {
            if (threadIdx.x == 0) s_job = atomicAdd(&heads[0], 1);
            __syncthreads();
            const int bi = s_job;
            __syncthreads();
            if (bi >= nbig) break;
            const int ci = big[bi];
            if (!comp_solve(team, S, red, a, roots[ci], bbox[ci]) && threadIdx.x == 0) to_global(a, ci);
            __syncthreads();
        }
    }
    {
        auto& S = reinterpret_cast<CompSm<kCapW, kKoW>*>(smem_raw)[warp];
        const TeamWarp team{lane};
        const int ncomp = min(*cnt, cap);
        while (true) {
            int ci = 0;
            if (lane == 0) ci = atomicAdd(&heads[1], 1);
            ci = __shfl_sync(0xffffffffu, ci, 0);
            if (ci >= ncomp) break;
            const int4 bb = bbox[ci];
            if (win_px(bb) > kCapW || a.enc[roots[ci]]) continue;  // block / global list, or an island
            if (!comp_solve(team, S, red, a, roots[ci], bb) && lane == 0) to_global(a, ci);
            __syncwarp();
        }
    }
#ifdef HP_COMP_DBG
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&g_compdbg_done, 1u) == gridDim.x - 1) {
            unsigned long long* c = g_compdbg;
            printf("COMPSUM n=%llu total=%llu stage=%llu edt=%llu J+zones+rmax=%llu mark=%llu W1=%llu W2=%llu par=%llu W3=%llu lines=%llu S10=%llu S11=%llu\n",
                   c[12], c[11], c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8], c[9], c[10]);
            for (int k = 0; k < 13; ++k) c[k] = 0;
            g_compdbg_done = 0;
        }
    }
#endif
}

// ---------------------------------------------------------------- S6 per S5 component
// FillHoles (reading C8: 4-connected background components touching no tile-
// border pixel) per kept candidate component A.  A hole is a bounded 4-connected background
// region; its boundary is an 8-connected set of foreground pixels, so it is enclosed by ONE
// 8-component and lies inside that component's bounding box.  In A's window (bbox + 1-px
// ring): A = the 8-component of A's root among the window's candidate pixels; every other
// window pixel counts as background; seeds = the ring, out-of-tile and tile-border pixels;
// the non-A pixels not 4-connected to a seed are A's holes (candidate pixels of other
// components enclosed there -- islands -- are filled with them and marked in enc).  F =
// union over components of A | holes(A) equals FillHoles(big0) exactly.
struct FillArgs {
    const uint8_t* big0;
    int w, h;
    uint8_t* F;
    uint8_t* enc;
    unsigned* labF;  // per F pixel: min root over the components whose F contains it (~0 else)
};

// F pixel p belongs to the F component of root: an island enclosed by A is written by A and by
// itself; A's root (its minimum linear index, above the island) wins, as in a CCL of F
__device__ __forceinline__ void mark_f(const FillArgs& a, int64_t p, int32_t root) {
    a.F[p] = 1;
    atomicMin(&a.labF[p], (unsigned)root);
}

// A = the 8-component of the root among the window's candidate pixels (union-find) -> sp
template <class Team, class St>
__device__ void fill_isolate(const Team& team, St& S, const FillArgs& a, int WX, int NWIN, int li_root) {
    const int tr = team.rank();
    constexpr int TS = Team::size;
    auto win = [&](auto fn) {
        for (int li = tr; li < NWIN; li += TS) fn(li);
    };
    auto each_mem = [&](auto fn) {
        win([&](int li) {
            if (S.mem[li]) fn(li);
        });
    };
    link_runs(team, S.B, WX, each_mem, [&](int li) { return li % WX > 0 && S.mem[li - 1]; });
    win([&](int li) {
        if (!S.mem[li]) return;
        const int ly = li / WX, lx = li - ly * WX;
        if (ly > 0) {
            if (S.mem[li - WX]) cunion(S.B, li, li - WX);
            if (lx > 0 && S.mem[li - WX - 1]) cunion(S.B, li, li - WX - 1);
            if (lx < WX - 1 && S.mem[li - WX + 1]) cunion(S.B, li, li - WX + 1);
        }
    });
    team.sync();
    const int rA = cfind(S.B, li_root);
    win([&](int li) { S.sp[li] = S.mem[li] && cfind(S.B, li) == rA; });
    team.sync();
}

// the holes of A (sp): 4-connected union-find over the non-A pixels, seeds = ring, out-of-tile
// and tile-border pixels; F |= A | holes, enc |= candidates inside the holes
template <class Team, class St>
__device__ void fill_holes_window(const Team& team, St& S, const FillArgs& a, int WX, int WY,
                                  int NWIN, int wx0, int wy0, int32_t root) {
    const int w = a.w, h = a.h;
    const int tr = team.rank();
    constexpr int TS = Team::size;
    auto win = [&](auto fn) {
        for (int li = tr; li < NWIN; li += TS) fn(li);
    };
#ifdef HP_FILL_DBG
    long long tt[6];
    int ntt = 0;
    tt[ntt++] = clock64();
    struct RepH {
        long long* tt; int* ntt; int tr, nwin;
        __device__ ~RepH() {
            const long long e = clock64();
            if (tr == 0 && e - tt[0] > 40000)
                printf("HOLESDBG nwin=%d total=%lld init=%lld jump=%lld union=%lld seed=%lld mark=%lld\n", nwin, e - tt[0],
                       tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3], e - tt[4]);
        }
    } reph_{tt, &ntt, tr, NWIN};
#define HOLES_T() tt[ntt++] = clock64()
#else
#define HOLES_T()
#endif
    win([&](int li) {
        if (S.sp[li]) S.C[li] = -1;
    });
    auto each_bg = [&](auto fn) {
        win([&](int li) {
            if (!S.sp[li]) fn(li);
        });
    };
    HOLES_T();
    link_runs(team, S.C, WX, each_bg, [&](int li) { return li % WX > 0 && !S.sp[li - 1]; });
    HOLES_T();
    win([&](int li) {
        if (S.sp[li]) return;
        const int ly = li / WX, lx = li - ly * WX;
        // one union per touching pair of runs: skip when the left pixels (li - 1, li - 1 - WX)
        // already joined the same two runs
        if (ly > 0 && !S.sp[li - WX] && !(lx > 0 && !S.sp[li - 1] && !S.sp[li - WX - 1])) cunion(S.C, li, li - WX);
    });
    team.sync();
    HOLES_T();
    win([&](int li) { S.B[li] = 0; });  // seed flags at the 4-roots
    team.sync();
    win([&](int li) {
        if (S.sp[li]) return;
        const int ly = li / WX, lx = li - ly * WX;
        const int gx = wx0 + lx, gy = wy0 + ly;
        const bool seed = lx == 0 || ly == 0 || lx == WX - 1 || ly == WY - 1 || !S.pm[li] || gx == 0 || gy == 0 ||
                          gx == w - 1 || gy == h - 1;
        if (seed) S.B[cfind(S.C, li)] = 1;
    });
    team.sync();
    HOLES_T();
    win([&](int li) {
        if (!S.pm[li]) return;
        const int ly = li / WX, lx = li - ly * WX;
        const int64_t p = (int64_t)(wy0 + ly) * w + (wx0 + lx);
        if (S.sp[li]) {
            mark_f(a, p, root);
        } else if (S.B[cfind(S.C, li)] == 0) {  // a hole of A
            mark_f(a, p, root);
            if (S.mem[li]) a.enc[p] = 1;         // another candidate, enclosed by A
        }
    });
    team.sync();
}

template <class Team, class St>
__device__ void fill_solve(const Team& team, St& S, TeamRed& red, const FillArgs& a, int32_t root,
                           int4 bb, int area) {
    const int w = a.w, h = a.h;
    const int tr = team.rank();
    constexpr int TS = Team::size;
    const int wx0 = bb.x - 1, wy0 = bb.y - 1;
    const int WX = bb.z - bb.x + 3, WY = bb.w - bb.y + 3;
    const int NWIN = WX * WY;
    const int li_root = (root / w - wy0) * WX + (root % w - wx0);
    auto win = [&](auto fn) {
        for (int li = tr; li < NWIN; li += TS) fn(li);
    };
#ifdef HP_FILL_DBG
    const long long t_start = clock64();
    struct Rep {
        long long t0; int ts, nwin, area, tr; long long t1 = 0, t2 = 0, t3 = 0; int path = 0;
        __device__ ~Rep() {
            const long long t4 = clock64(), dt = t4 - t0;
            if (tr == 0 && dt > 50000)
                printf("FILLDBG ts=%d nwin=%d area=%d path=%d cycles=%lld stage=%lld iso=%lld euler=%lld rest=%lld\n", ts,
                       nwin, area, path, dt, t1 - t0, t2 - t1, t3 - t2, t4 - t3);
        }
    } rep_{t_start, TS, NWIN, area, tr};
#endif
    // stage: candidate pixels (mem), in-tile flags (pm)
    int ncand = 0;
    win([&](int li) {
        const int ly = li / WX, lx = li - ly * WX;
        const int gx = wx0 + lx, gy = wy0 + ly;
        const bool in = gx >= 0 && gy >= 0 && gx < w && gy < h;
        const bool c = in && a.big0[(int64_t)gy * w + gx];
        S.mem[li] = c;
        S.pm[li] = in;
        S.B[li] = li;
        ncand += c;
    });
    ncand = team.reduce(ncand, red.i, OpAdd());
    team.sync();
#ifdef HP_FILL_DBG
    rep_.t1 = clock64();
    rep_.path = ncand == area ? 1 : 2;
#endif
    // fast path 1: the window holds no other candidate, so A = every candidate pixel
    if (ncand == area) {
        win([&](int li) { S.sp[li] = S.mem[li]; });
        team.sync();
    } else {
        fill_isolate(team, S, a, WX, NWIN, li_root);
    }
#ifdef HP_FILL_DBG
    rep_.t2 = clock64();
#endif
    // fast path 2: holes of the one 8-component A from its Euler number (bit-quads, Gray 1971:
    // E8 = (n1 - n3 - 2 nD) / 4, holes = 1 - E8 for 4-connected background)
    int q = 0;
    for (int k = tr; k < (WX - 1) * (WY - 1); k += TS) {
        const int qy = k / (WX - 1), qx = k - qy * (WX - 1);
        const int li = qy * WX + qx;
        const int b0 = S.sp[li], b1 = S.sp[li + 1], b2 = S.sp[li + WX], b3 = S.sp[li + WX + 1];
        const int nq = b0 + b1 + b2 + b3;
        if (nq == 1) q += 1;
        else if (nq == 3) q -= 1;
        else if (nq == 2 && b0 == b3) q -= 2;  // diagonal pair
    }
    q = team.reduce(q, red.i, OpAdd());
    const bool holes = (4 - q) / 4 > 0;  // holes = 1 - q / 4
#ifdef HP_FILL_DBG
    rep_.t3 = clock64();
    rep_.path += holes ? 10 : 0;
#endif
    if (!holes) {
        win([&](int li) {
            if (S.sp[li]) mark_f(a, (int64_t)(wy0 + li / WX) * w + (wx0 + li % WX), root);
        });
        team.sync();
        return;
    }
    fill_holes_window(team, S, a, WX, WY, NWIN, wx0, wy0, root);
}

// windows > kCapW: block list; > kCapB: huge list (global-memory storage)
__global__ void k_win_classify(const int32_t* __restrict__ cnt, int32_t cap, const int4* __restrict__ bbox,
                               int32_t* __restrict__ big, int32_t* __restrict__ nbig, int32_t* __restrict__ huge,
                               int32_t* __restrict__ nhuge) {
    const int n = min(*cnt, cap);
    GRID_LOOP(ci, (int64_t)n) {
        const int wp = win_px(bbox[ci]);
        if (wp > kCapB) huge[atomicAdd(nhuge, 1)] = (int)ci;
        else if (wp > kCapW) big[atomicAdd(nbig, 1)] = (int)ci;
    }
}

// the huge windows, one after another in one block over global-memory storage
constexpr int kHugeT = 256;
__global__ void __launch_bounds__(kHugeT) k_fill_huge(FillArgs a, const int32_t* __restrict__ roots,
                                                      const int4* __restrict__ bbox, const int32_t* __restrict__ areas,
                                                      const int32_t* __restrict__ huge,
                                                      const int32_t* __restrict__ nhuge, BigScratch bs) {
    __shared__ int nmem, nbnd, nobj;
    __shared__ FeatSmem fs;
    __shared__ TeamRed red;
    CompGm S{bs.dist, bs.A, bs.B, bs.C, bs.list, bs.mem, bs.pm, bs.sp, nmem, nbnd, nobj, bs.objroot, fs};
    const TeamCTA<kHugeT> team;
    const int n = *nhuge;
    for (int k = 0; k < n; ++k) {
        const int ci = huge[k];
        fill_solve(team, S, red, a, roots[ci], bbox[ci], areas[ci]);
    }
}

// S7-S11 of the components left to the global-memory storage, one after another in one block
__global__ void __launch_bounds__(kHugeT) k_comp_huge(CompArgs a, const int32_t* __restrict__ roots,
                                                      const int4* __restrict__ bbox, BigScratch bs) {
    __shared__ int nmem, nbnd, nobj;
    __shared__ FeatSmem fs;
    __shared__ TeamRed red;
    CompGm S{bs.dist, bs.A, bs.B, bs.C, bs.list, bs.mem, bs.pm, bs.sp, nmem, nbnd, nobj, bs.objroot, fs};
    const TeamCTA<kHugeT> team;
    const int n = *a.ovf_cnt;
    for (int k = 0; k < n; ++k) {
        const int ci = a.ovf_list[k];
        comp_solve(team, S, red, a, roots[ci], bbox[ci]);
    }
}

__global__ void __launch_bounds__(kWarpsPB * 32, 4) k_fill_fused(FillArgs a, const int32_t* __restrict__ cnt,
                                                                int32_t cap, const int32_t* __restrict__ roots,
                                                                const int4* __restrict__ bbox,
                                                                const int32_t* __restrict__ areas,
                                                                const int32_t* __restrict__ big,
                                                                const int32_t* __restrict__ nbig_p,
                                                                int32_t* __restrict__ heads) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_job;
    __shared__ TeamRed red;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        auto& S = *reinterpret_cast<FillSm<kCapB>*>(smem_raw);
        const TeamCTA<kWarpsPB * 32> team;
        const int nbig = *nbig_p;
        while (true) {
            if (threadIdx.x == 0) s_job = atomicAdd(&heads[0], 1);
            __syncthreads();
            const int bi = s_job;
            __syncthreads();
            if (bi >= nbig) break;
            const int ci = big[bi];
            fill_solve(team, S, red, a, roots[ci], bbox[ci], areas[ci]);
        }
    }
    {
        auto& S = reinterpret_cast<FillSm<kCapW>*>(smem_raw)[warp];
        const TeamWarp team{lane};
        const int ncomp = min(*cnt, cap);
        while (true) {
            int ci = 0;
            if (lane == 0) ci = atomicAdd(&heads[1], 1);
            ci = __shfl_sync(0xffffffffu, ci, 0);
            if (ci >= ncomp) break;
            const int4 bb = bbox[ci];
            if (win_px(bb) > kCapW) continue;  // block or huge list
            fill_solve(team, S, red, a, roots[ci], bb, areas[ci]);
        }
    }
}

// Rows to label order: labels are distinct, so a row's rank is the number of smaller labels.
// One warp per row (grid-stride): the lanes count over the staged labels (L1-resident), then
// copy the row to its rank -- ~n^2/32 compares spread over the whole GPU, coalesced row copies.
__global__ void k_rows_scatter(const int32_t* __restrict__ cnt, int32_t cap, const int32_t* __restrict__ sl,
                               const int32_t* __restrict__ sf, const float* __restrict__ sfeat,
                               int32_t* __restrict__ ol, int32_t* __restrict__ of, float* __restrict__ ofeat,
                               int32_t capacity) {
    const int n = min(*cnt, cap);
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const int32_t me = sl[i];
        int c = 0;
        for (int k = lane; k < n; k += 32) c += __ldg(sl + k) < me;
        const int rk = __reduce_add_sync(0xffffffffu, c);
        if (rk >= capacity) continue;
        if (lane == 0) {
            ol[rk] = me;
            of[rk] = sf[i];
        }
        for (int k = lane; k < HP_NFEAT; k += 32) ofeat[(int64_t)rk * HP_NFEAT + k] = sfeat[(int64_t)i * HP_NFEAT + k];
    }
}

__global__ void k_copy_i32(const int32_t* __restrict__ src, int32_t* __restrict__ dst) { *dst = *src; }

}  // namespace

// Outputs: labels (zeroed here), n_objects, and (when table != nullptr) the feature rows in
// label order.
// S7-S11 per F component, from the S5 component list: the F component of a kept candidate
// component A is A with its holes and any islands inside them -- the pixels whose root word
// (written by S6) is A's root.  Islands enclosed by another component (enc at their root) are
// solved with their encloser.  Shared-memory windows (warp / block teams); windows too big for
// shared memory and object-list overflows in one block over global-memory storage.
void launch_components(const int32_t* count5, const uint8_t* enc, const uint8_t* g, const uint8_t* edge, float hh,
                       int amin, int amax,
                       int w, int h, Slot& sl, int32_t* labels, int64_t lpitch, int32_t* n_objects,
                       const hp_feature_table* table, int32_t max_objects, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    cudaMemsetAsync(n_objects, 0, sizeof(int32_t), s);
    cudaMemset2DAsync(labels, lpitch * sizeof(int32_t), 0, w * sizeof(int32_t), h, s);
    int32_t* ovf = sl.cnt32 + 9;     // components for the global-memory path
    int32_t* rows = sl.cnt32 + 10;   // staged rows
    int32_t* nbig = sl.cnt32 + 12;   // block-list components
    int32_t* heads = sl.cnt32 + 13;  // [0] block-list head, [1] component-list head
    cudaMemsetAsync(sl.cnt32 + 8, 0, 8 * sizeof(int32_t), s);
    if (n == 0) {
        if (table) cudaMemsetAsync(table->n_rows_dev, 0, sizeof(int32_t), s);
        return;
    }
    const int32_t cap = sl.comp_cap;
    CompArgs a{};
    a.labF = sl.lab;
    a.enc = enc;
    a.g = g;
    a.edge = edge;
    a.hh = hh;
    a.w = w;
    a.h = h;
    a.amin = amin;
    a.amax = amax;
    a.labels = labels;
    a.lpitch = lpitch;
    a.n_objects = n_objects;
    a.rows_cnt = rows;
    a.rows_cap = max_objects;
    a.row_label = sl.stg_label;
    a.row_flags = sl.stg_flags;
    a.row_feat = sl.stg_feat;
    a.do_features = table != nullptr;
    a.ovf_cnt = ovf;
    a.ovf_list = sl.sc_huge;  // (S6's huge list is consumed by then: same stream)
    const size_t smw = kWarpsPB * sizeof(CompSm<kCapW, kKoW>);
    static PerDevice once;
    once.get([&] { return (int)cudaFuncSetAttribute(k_comp_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw); });
    (note_launch(), k_comp_classify<<<grid_for(cap), 256, 0, s>>>(a, count5, cap, sl.sc_root, sl.sc_bbox,
                                                                   sl.sc_big, nbig));
    (note_launch(), k_comp_fused<<<num_sms() * HP_COMP_BPS, kWarpsPB * 32, smw, s>>>(a, count5, cap, sl.sc_root, sl.sc_bbox,
                                                                     sl.sc_big, nbig, heads));
    (note_launch(), k_comp_huge<<<1, kHugeT, 0, s>>>(a, sl.sc_root, sl.sc_bbox, carve_big(sl)));
    if (table) {
        (note_launch(), k_rows_scatter<<<std::max(1, std::min(num_sms() * 2, (max_objects + 7) / 8)), 256, 0, s>>>(
            rows, max_objects, sl.stg_label, sl.stg_flags, sl.stg_feat, table->label, table->flags, table->feat,
            table->capacity));
        (note_launch(), k_copy_i32<<<1, 1, 0, s>>>(rows, table->n_rows_dev));
    }
}

void launch_fill_components(const uint8_t* big0, int w, int h, Slot& sl, const int32_t* count, uint8_t* F,
                            uint8_t* enc, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    int32_t* nbig = sl.cnt32 + 18;
    int32_t* heads = sl.cnt32 + 19;  // [0] block-list head, [1] component-list head
    int32_t* nhuge = sl.cnt32 + 21;
    cudaMemsetAsync(sl.cnt32 + 18, 0, 4 * sizeof(int32_t), s);
    if (n == 0) return;
    cudaMemsetAsync(F, 0, n, s);
    cudaMemsetAsync(enc, 0, n, s);
    cudaMemsetAsync(sl.lab, 0xff, 4 * n, s);
    FillArgs a{big0, w, h, F, enc, reinterpret_cast<unsigned*>(sl.lab)};
    const size_t smw = kFillSmem;
    static PerDevice once;
    once.get([&] { return (int)cudaFuncSetAttribute(k_fill_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw); });
    const int32_t cap = sl.comp_cap;
    (note_launch(), k_win_classify<<<grid_for(cap), 256, 0, s>>>(count, cap, sl.sc_bbox, sl.sc_big, nbig, sl.sc_huge,
                                                                  nhuge));
    (note_launch(), k_fill_fused<<<num_sms() * HP_FILL_BPS, kWarpsPB * 32, smw, s>>>(a, count, cap, sl.sc_root, sl.sc_bbox,
                                                                     sl.sc_area, sl.sc_big, nbig, heads));
    (note_launch(), k_fill_huge<<<1, kHugeT, 0, s>>>(a, sl.sc_root, sl.sc_bbox, sl.sc_area, sl.sc_huge, nhuge,
                                                    carve_big(sl)));
}

}  // namespace hp
