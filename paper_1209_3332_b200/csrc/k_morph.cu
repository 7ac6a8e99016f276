// k_morph.cu -- S3: Morph. Open with the OpenCV 19x19 elliptic disk (PAPER.md:595,
// 623-625; reading C7: out-of-tile pixels are ignored).
//
// open = dilate_D(erode_D(g)).  D's row dy covers dx in [-hw(dy), hw(dy)] with hw(dy) =
// round(sqrt(r^2 - dy^2)); so min over D = min over rows of a horizontal running min whose
// half-width takes only a few distinct values (6 for diam 19).  Bound by the plain integer
// ALUs: the 19x19 fast path works on 2 pixels per register with the native
// 3-input u16x2 min/max; the generic path on 4 pixels with the byte SIMD __vminu4/__vmaxu4.
//   stage 1: the (TH + 2r) input rows of a TW-wide tile (+ halo) are staged in shared memory
//            as 32-bit words (aligned vector loads; out-of-tile bytes = identity);
//   stage 2: per row and output word: the 2*RW+2 covering words go to registers once, every
//            byte-shifted window is a funnel shift by a compile-time amount, and the running
//            min over [-k, k] is kept for the distinct half-widths -> H[width][row][word];
//   stage 3: out(y) = min over the diam rows dy of H[width(dy)][y + dy].
// The radius is a template parameter (19x19 = the paper's disk is the instantiated fast
// path); other odd diameters use the generic path with the same structure.
#include <algorithm>
#include <cmath>
#include <vector>

#include "hp_internal.cuh"

namespace hp {

namespace {

constexpr int TW = 128;       // output tile width (pixels) = 32 words
constexpr int TWW = TW / 4;   // output words per row
constexpr int kMaxDiam = 63;

template <bool IS_MIN>
__device__ __forceinline__ uint32_t vop(uint32_t a, uint32_t b) {
    return IS_MIN ? __vminu4(a, b) : __vmaxu4(a, b);
}

__host__ __device__ constexpr int hw_of(int r, int dy) {
    // round(sqrt(r^2 - dy^2)) evaluated exactly in integers: the largest w with
    // (w - 0.5)^2 <= r^2 - dy^2, i.e. (2w - 1)^2 <= 4(r^2 - dy^2)  (no ties for integer r, dy)
    int s = 4 * (r * r - dy * dy), w = 0;
    while ((2 * (w + 1) - 1) * (2 * (w + 1) - 1) <= s) ++w;
    return w;
}

// distinct half-widths of the ellipse of radius R, ascending, as a compile-time table
template <int R>
struct Ellipse {
    int n = 0;
    int hw[R + 1] = {};
    int idx_of_dy[2 * R + 1] = {};
    constexpr Ellipse() {
        for (int dy = 0; dy <= R; ++dy) {
            int v = hw_of(R, dy);
            bool seen = false;
            for (int k = 0; k < n; ++k) seen |= hw[k] == v;
            if (!seen) hw[n++] = v;
        }
        for (int a = 0; a < n; ++a)  // sort ascending
            for (int b = a + 1; b < n; ++b)
                if (hw[b] < hw[a]) { int t = hw[a]; hw[a] = hw[b]; hw[b] = t; }
        for (int dy = -R; dy <= R; ++dy) {
            int v = hw_of(R, dy < 0 ? -dy : dy);
            for (int k = 0; k < n; ++k)
                if (hw[k] == v) idx_of_dy[dy + R] = k;
        }
    }
};

// ---------------------------------------------------------------- radius-specialised kernel
// sm_100a has native 16-bit-lane min/max with three inputs (VIMNMX3.U16x2) but emulates the
// byte-lane __vminu4 with ~7 LOP3/PRMT/IADD instructions (SASS, r1), so the fast path keeps
// 2 pixels per 32-bit word in u16 lanes: a running min over [-k, k] costs one 3-input op per
// step, the vertical combine one per two rows.
template <bool IS_MIN>
__device__ __forceinline__ uint32_t vop3(uint32_t a, uint32_t b, uint32_t c) {
    return IS_MIN ? __vimin3_u16x2(a, b, c) : __vimax3_u16x2(a, b, c);
}

#ifndef HP_MORPH_BPS
#define HP_MORPH_BPS 4  // persistent blocks per SM of the 19x19 path
#endif
constexpr int TW2 = 64;        // output tile width (pixels) = 32 u16x2 words
constexpr int TH2 = 32;        // output tile height

template <bool IS_MIN, int R>
__global__ void __launch_bounds__(256) k_morph_r(const uint8_t* __restrict__ src, int w, int h,
                                                 uint8_t* __restrict__ dst) {
    constexpr Ellipse<R> E{};
    constexpr int ND = E.n;
    constexpr int RW = 2 * ((R + 3) / 4);        // halo words (2 px each) per side: 4-px aligned
    constexpr int IW = 32 + 2 * RW + 2;          // staged words per row (even: loads in pairs)
    constexpr int ROWS = TH2 + 2 * R;
    constexpr int NQ = IW / 2;                   // 4-pixel groups per row
    constexpr int NL = (ROWS * NQ + 255) / 256;  // 4-pixel loads per thread per tile
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t* in = smem;                          // [ROWS][IW] u16x2
    uint32_t* H = smem + ROWS * IW;               // [ND][ROWS][32]
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const bool row_aligned = (w & 3) == 0 && (((uintptr_t)src) & 3) == 0;
    const bool dst_aligned = (w & 1) == 0 && (((uintptr_t)dst) & 1) == 0;
    const int ntx = (w + TW2 - 1) / TW2, ntiles = ntx * ((h + TH2 - 1) / TH2);

    // Persistent over tiles: the global loads of the NEXT tile's input are issued into
    // registers before this tile's compute, so their latency hides behind stages 2-3.
    // stage 1 (per tile): pixels [x0 - 2RW, x0 + 64 + 2RW + 2) of rows [y0 - R, y0 + TH2 + R)
    uint32_t pre[NL];
    // tile -> (tx, ty) advanced by the grid stride without a division per tile (r2 ncu: the
    // runtime div / mod by ntx cost 12% of the kernel's instructions)
    const int gsx = (int)gridDim.x % ntx, gsy = (int)gridDim.x / ntx;
    auto load = [&](int tx_, int ty_) {
        const int x0 = tx_ * TW2, y0 = ty_ * TH2;
        if (row_aligned && x0 - 2 * RW >= 0 && x0 + TW2 + 2 * RW + 4 <= w && y0 - R >= 0 && y0 + TH2 + R <= h) {
            // interior tile: every staged word is an aligned in-range load
            const uint8_t* base = src + (int64_t)(y0 - R) * w + (x0 - 2 * RW);
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                const int i = threadIdx.x + 256 * l;
                const int r = i / NQ, q = i - r * NQ;
                pre[l] = (i < ROWS * NQ) ? __ldg(reinterpret_cast<const unsigned int*>(base + (int64_t)r * w + 4 * q))
                                         : 0u;
            }
            return;
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const int i = threadIdx.x + 256 * l;
            uint32_t v = IS_MIN ? 0xffffffffu : 0u;
            if (i < ROWS * NQ) {
                const int r = i / NQ, q = i - r * NQ;
                const int gy = y0 - R + r;
                const int gx = x0 - 2 * RW + 4 * q;
                if (gy >= 0 && gy < h) {
                    const uint8_t* rowp = src + (int64_t)gy * w;
                    if (row_aligned && gx >= 0 && gx + 3 < w) {
                        v = __ldg(reinterpret_cast<const unsigned int*>(rowp + gx));
                    } else {
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int x = gx + b;
                            const uint32_t byte =
                                (x >= 0 && x < w) ? (uint32_t)__ldg(rowp + x) : (IS_MIN ? 0xffu : 0u);
                            v = (v & ~(0xffu << (8 * b))) | (byte << (8 * b));
                        }
                    }
                }
            }
            pre[l] = v;
        }
    };
    int tile = blockIdx.x;
    int tx0 = (int)blockIdx.x % ntx, ty0 = (int)blockIdx.x / ntx;
    if (tile < ntiles) load(tx0, ty0);
    for (; tile < ntiles; tile += gridDim.x) {
        const int x0 = tx0 * TW2, y0 = ty0 * TH2;
        tx0 += gsx;
        ty0 += gsy;
        if (tx0 >= ntx) {
            tx0 -= ntx;
            ++ty0;
        }
        __syncthreads();  // the previous tile's stages 2-3 are done with in[] and H[]
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const int i = threadIdx.x + 256 * l;
            if (i < ROWS * NQ) {
                const int r = i / NQ, q = i - r * NQ;
                in[r * IW + 2 * q] = __byte_perm(pre[l], 0, 0x4140);      // px 0, 1 -> u16 lanes
                in[r * IW + 2 * q + 1] = __byte_perm(pre[l], 0, 0x4342);  // px 2, 3
            }
        }
        __syncthreads();
        if (tile + (int)gridDim.x < ntiles) load(tx0, ty0);

        // stage 2: horizontal running min/max for the distinct half-widths; a half-warp per
        // row, lane -> output words 2l, 2l+1 (pixels 4l .. 4l+3): the 2RW+3 covering words
        // come in as 8-byte shared loads, each funnel-shifted window serves both outputs (the
        // second output's window k is the first's k + 2), H is written 8 bytes at a time
        // (r2: a lane per word issued 12 of 36 M instructions in the covering-word loads)
        {
            constexpr int NWV = ((((2 * RW + R + 2) >> 1) + 2) + 1) & ~1;  // words 0 .. last used, even
            static_assert(2 * 15 + NWV <= IW, "covering words inside the staged row");
            const int l = tx & 15;
            for (int r = 2 * ty + (tx >> 4); r < ROWS; r += 16) {
                const uint32_t* rowp = in + r * IW + 2 * l;
                uint32_t wv[NWV];
#pragma unroll
                for (int k = 0; k + 1 < NWV; k += 2) {
                    const uint2 v = *reinterpret_cast<const uint2*>(rowp + k);
                    wv[k] = v.x;
                    wv[k + 1] = v.y;
                }
                if (NWV & 1) wv[NWV - 1] = rowp[NWV - 1];
                auto win = [&](int k) -> uint32_t {  // pixels (4l + k, 4l + 1 + k)
                    const int o = 2 * RW + k;
                    return (o & 1) ? __funnelshift_r(wv[o >> 1], wv[(o >> 1) + 1], 16) : wv[o >> 1];
                };
                uint32_t m0 = win(0), m1 = win(2);
                uint2* Hr = reinterpret_cast<uint2*>(H + r * 32 + 2 * l);
#pragma unroll
                for (int q = 0; q < ND; ++q)
                    if (E.hw[q] == 0) Hr[q * ROWS * 16] = make_uint2(m0, m1);
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    m0 = vop3<IS_MIN>(m0, win(k), win(-k));
                    m1 = vop3<IS_MIN>(m1, win(k + 2), win(2 - k));
#pragma unroll
                    for (int q = 0; q < ND; ++q)
                        if (E.hw[q] == k) Hr[q * ROWS * 16] = make_uint2(m0, m1);
                }
            }
        }
        __syncthreads();

        // stage 3: vertical combine over the 2R+1 rows of D (two rows per 3-input op).  A
        // thread takes 4 consecutive output rows: rows of D with equal half-widths read the
        // same H entry for neighbouring outputs, so the shared loads are issued once.
        constexpr int ORW = TH2 / 8;  // output rows per thread
        const int j = tx;
        const int gx = x0 + 2 * j;
        const int oy0 = ORW * ty;
        uint32_t m[ORW];
#pragma unroll
        for (int i = 0; i < ORW; ++i) m[i] = H[(E.idx_of_dy[0] * ROWS + oy0 + i) * 32 + j];
#pragma unroll
        for (int dy = 1; dy + 1 <= 2 * R; dy += 2)
#pragma unroll
            for (int i = 0; i < ORW; ++i)
                m[i] = vop3<IS_MIN>(m[i], H[(E.idx_of_dy[dy] * ROWS + oy0 + i + dy) * 32 + j],
                                    H[(E.idx_of_dy[dy + 1] * ROWS + oy0 + i + dy + 1) * 32 + j]);
        uint8_t* o = dst + (int64_t)(y0 + oy0) * w + gx;
        if (dst_aligned && gx + 1 < w && y0 + oy0 + ORW <= h) {
#pragma unroll
            for (int i = 0; i < ORW; ++i, o += w)
                *reinterpret_cast<uint16_t*>(o) = (uint16_t)__byte_perm(m[i], 0, 0x0020);  // u16 lanes -> 2 bytes
        } else {
#pragma unroll
            for (int i = 0; i < ORW; ++i, o += w) {
                if (y0 + oy0 + i >= h || gx >= w) continue;
                const uint32_t pk = __byte_perm(m[i], 0, 0x0020);
                o[0] = (uint8_t)pk;
                if (gx + 1 < w) o[1] = (uint8_t)(pk >> 8);
            }
        }
    }
}

template <int R>
size_t smem_r() {
    constexpr Ellipse<R> E{};
    constexpr int RW = 2 * ((R + 3) / 4);
    return 4 * (size_t)(TH2 + 2 * R) * ((32 + 2 * RW + 2) + (size_t)E.n * 32);
}

template <int R>
void launch_r(const uint8_t* g, int w, int h, uint8_t* tmp, uint8_t* out, cudaStream_t s) {
    static PerDevice once;
    const size_t smem = smem_r<R>();
    once.get([&] {
        cudaFuncSetAttribute(k_morph_r<true, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return (int)cudaFuncSetAttribute(k_morph_r<false, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    // persistent: as many blocks as fit (shared memory allows 4 per SM), each looping over tiles
    const int ntiles = ((w + TW2 - 1) / TW2) * ((h + TH2 - 1) / TH2);
    const int grid = std::max(1, std::min(ntiles, num_sms() * HP_MORPH_BPS));
    (note_launch(), k_morph_r<true, R><<<grid, 256, smem, s>>>(g, w, h, tmp));
    (note_launch(), k_morph_r<false, R><<<grid, 256, smem, s>>>(tmp, w, h, out));
}

// ---------------------------------------------------------------- generic (any odd diam)
struct MorphDesc {
    int r, nd, th;               // radius, number of distinct half-widths, tile height
    int rw;                      // halo words = ceil(r / 4)
    int hw_idx[kMaxDiam];        // row i -> index into dist[]
    int dist_hw[kMaxDiam];       // distinct half-widths, ascending
};

template <bool IS_MIN>
__global__ void __launch_bounds__(256) k_morph(const uint8_t* __restrict__ src, int w, int h,
                                               MorphDesc md, uint8_t* __restrict__ dst) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int r = md.r, th = md.th, rw = md.rw;
    const int rows = th + 2 * r;
    const int in_words = TWW + 2 * rw + 1;
    uint32_t* in = smem;
    uint32_t* H = smem + rows * in_words;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * th;
    const uint8_t ident = IS_MIN ? 255 : 0;
    uint8_t* inb = reinterpret_cast<uint8_t*>(in);
    const int in_bytes = in_words * 4;
    for (int i = threadIdx.x; i < rows * in_bytes; i += blockDim.x) {
        int ry = i / in_bytes, bx = i - ry * in_bytes;
        int gy = y0 - r + ry, gx = x0 - 4 * rw + bx;
        uint8_t v = ident;
        if (gy >= 0 && gy < h && gx >= 0 && gx < w) v = __ldg(src + (int64_t)gy * w + gx);
        inb[i] = v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < rows * TWW; i += blockDim.x) {
        int ry = i / TWW, j = i - ry * TWW;
        const uint32_t* row = in + ry * in_words;
        auto win = [&](int k) -> uint32_t {
            int o = 4 * (j + rw) + k;
            return __funnelshift_r(row[o >> 2], row[(o >> 2) + 1], 8 * (o & 3));
        };
        uint32_t m = win(0);
        int di = 0;
        if (md.dist_hw[0] == 0) {
            H[(0 * rows + ry) * TWW + j] = m;
            di = 1;
        }
        for (int k = 1; k <= r && di < md.nd; ++k) {
            m = vop<IS_MIN>(m, vop<IS_MIN>(win(k), win(-k)));
            if (md.dist_hw[di] == k) {
                H[(di * rows + ry) * TWW + j] = m;
                ++di;
            }
        }
    }
    __syncthreads();
    const int diam = 2 * r + 1;
    for (int i = threadIdx.x; i < th * TWW; i += blockDim.x) {
        int oy = i / TWW, j = i - oy * TWW;
        int gy = y0 + oy, gx = x0 + 4 * j;
        if (gy >= h || gx >= w) continue;
        uint32_t m = IS_MIN ? 0xffffffffu : 0u;
        for (int dy = 0; dy < diam; ++dy) m = vop<IS_MIN>(m, H[(md.hw_idx[dy] * rows + oy + dy) * TWW + j]);
        uint8_t* o = dst + (int64_t)gy * w + gx;
        if (gx + 3 < w && (((uintptr_t)o) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(o) = m;
        } else {
            for (int b = 0; b < 4 && gx + b < w; ++b) o[b] = (uint8_t)(m >> (8 * b));
        }
    }
}

MorphDesc make_desc(int diam, size_t* smem_bytes) {
    MorphDesc md{};
    md.r = diam / 2;
    md.rw = (md.r + 3) / 4;
    std::vector<int> hw(diam);
    for (int i = 0; i < diam; ++i) hw[i] = hw_of(md.r, std::abs(i - md.r));
    std::vector<int> d = hw;
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    md.nd = (int)d.size();
    for (int k = 0; k < md.nd; ++k) md.dist_hw[k] = d[k];
    for (int i = 0; i < diam; ++i)
        md.hw_idx[i] = (int)(std::lower_bound(d.begin(), d.end(), hw[i]) - d.begin());
    const size_t cap = 200 * 1024;
    for (md.th = 32; md.th > 1; md.th /= 2) {
        size_t rows = md.th + 2 * md.r;
        size_t bytes = 4 * rows * ((TWW + 2 * md.rw + 1) + (size_t)md.nd * TWW);
        if (bytes <= cap) break;
    }
    size_t rows = md.th + 2 * md.r;
    *smem_bytes = 4 * rows * ((TWW + 2 * md.rw + 1) + (size_t)md.nd * TWW);
    return md;
}

}  // namespace

void launch_open(const uint8_t* g, int w, int h, int diam, uint8_t* tmp, uint8_t* out,
                 cudaStream_t s) {
    if ((int64_t)w * h == 0) return;
    if (diam == 19) {  // the paper's 19x19 disk
        launch_r<9>(g, w, h, tmp, out, s);
        return;
    }
    size_t smem = 0;
    MorphDesc md = make_desc(diam, &smem);
    static PerDevice once;
    once.get([] {
        cudaFuncSetAttribute(k_morph<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return (int)cudaFuncSetAttribute(k_morph<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    dim3 grid((w + TW - 1) / TW, (h + md.th - 1) / md.th);
    (note_launch(), k_morph<true><<<grid, 256, smem, s>>>(g, w, h, md, tmp));
    (note_launch(), k_morph<false><<<grid, 256, smem, s>>>(tmp, w, h, md, out));
}

}  // namespace hp
