// k_morph.cu -- S3: Morph. Open with the OpenCV 19x19 elliptic disk (PAPER.md:595,
// 623-625; reading C7: out-of-tile pixels are ignored).
//
// open = dilate_D(erode_D(g)).  D's row dy covers dx in [-hw(dy), hw(dy)] with hw(dy) =
// round(sqrt(r^2 - dy^2)); so min over D = min over rows of a horizontal running min whose
// width takes only a few distinct values (6 for diam 19).  Bound by the plain integer ALUs
// (SURVEY §8(d)): every step works on 4 pixels per 32-bit register with the SIMD byte
// min/max (__vminu4 / __vmaxu4); byte-shifted windows come from funnel shifts.
//   stage 1: the (TH + 2r) x TW input rows are staged in shared memory (OOB -> identity);
//   stage 2: for each row and 4-pixel word, horizontal min over [-k, k] for k = 1..r,
//            keeping the distinct half-widths hw(dy) -> H[width][row][word] in smem;
//   stage 3: out(y) = min over the diam rows i of H[hw(i - r)][y + i].
#include <algorithm>
#include <cmath>
#include <vector>

#include "hp_internal.cuh"

namespace hp {

namespace {

constexpr int TW = 128;          // output tile width (pixels) = 32 words
constexpr int TWW = TW / 4;      // words per output row
constexpr int kMaxDiam = 63;

struct MorphDesc {
    int r, nd, th;               // radius, number of distinct half-widths, tile height
    int rw;                      // halo words = ceil(r / 4)
    int hw_idx[kMaxDiam];        // row i -> index into dist[]
    int dist_hw[kMaxDiam];       // distinct half-widths, ascending
};

template <bool IS_MIN>
__device__ __forceinline__ uint32_t vop(uint32_t a, uint32_t b) {
    return IS_MIN ? __vminu4(a, b) : __vmaxu4(a, b);
}

template <bool IS_MIN>
__global__ void __launch_bounds__(256) k_morph(const uint8_t* __restrict__ src, int w, int h,
                                               MorphDesc md, uint8_t* __restrict__ dst) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int r = md.r, th = md.th, rw = md.rw;
    const int rows = th + 2 * r;
    const int in_words = TWW + 2 * rw + 1;        // staged words per row
    uint32_t* in = smem;                           // [rows][in_words]
    uint32_t* H = smem + rows * in_words;          // [nd][rows][TWW]
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * th;
    const uint8_t ident = IS_MIN ? 255 : 0;

    // stage 1: bytes [x0 - 4rw, x0 + TW + 4rw + 4) of rows [y0 - r, y0 + th + r)
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

    // stage 2: horizontal running min/max for every distinct half-width
    for (int i = threadIdx.x; i < rows * TWW; i += blockDim.x) {
        int ry = i / TWW, j = i - ry * TWW;
        const uint32_t* row = in + ry * in_words;
        // window word at byte offset k relative to this word's first byte
        auto win = [&](int k) -> uint32_t {
            int o = 4 * (j + rw) + k;
            int wi = o >> 2, sh = o & 3;
            return __funnelshift_r(row[wi], row[wi + 1], 8 * sh);
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

    // stage 3: vertical combine over the diam rows of D
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
    for (int i = 0; i < diam; ++i) {
        int dy = i - md.r;
        hw[i] = (int)std::lround(std::sqrt((double)(md.r * md.r - dy * dy)));
    }
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
    size_t smem = 0;
    MorphDesc md = make_desc(diam, &smem);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_morph<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_morph<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    dim3 grid((w + TW - 1) / TW, (h + md.th - 1) / md.th);
    (note_launch(), k_morph<true><<<grid, 256, smem, s>>>(g, w, h, md, tmp));
    (note_launch(), k_morph<false><<<grid, 256, smem, s>>>(tmp, w, h, md, out));
}

}  // namespace hp
