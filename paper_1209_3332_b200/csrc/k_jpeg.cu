// k_jpeg.cu -- S0+S1 from JPEG-compressed tiles (PAPER.md:971-974:
// "the main limiting factor and bottleneck is the I/O overhead of reading image tiles",
// 716-726).  A raw 4K tile is 50 MB over PCIe; the same tile as a quality-90 baseline JPEG
// is ~4 MB, so the host link stops being the bound.  Decoding is the GPU's job:
//
//   host      jpeg_parse: the marker segments (T.81 B.2) -> JpegHdr (tables, scan offset);
//   k_rst_count / k_rst_write
//             restart markers (0xFF 0xD0..0xD7) found in parallel over 8 KB chunks of the
//             entropy-coded segment, written in order as interval start offsets;
//   k_jpeg_decode
//             one restart interval per thread (the intervals are independent: DC prediction
//             restarts at every RSTm, T.81 F.2.1.3): Huffman decoding through 9-bit lookup
//             tables built per block in shared memory from BITS/HUFFVAL (Annex C canonical
//             codes; longer codes by the MAXCODE walk of F.2.2.3), dequantisation, the islow
//             integer IDCT (reading J1) with zero-column / DC-only shortcuts driven by a
//             64-bit nonzero mask (no coefficient zeroing), JFIF YCbCr->RGB (reading J2), and
//             S1 on every pixel (cd_pixel.cuh, the raw path's own arithmetic): g and flags
//             are written, the RGB tile never is.
//
// Scope as oracle/jpeg.cpp: SOF0/SOF1 8-bit, 3 components 1x1 (4:4:4), one scan.
#include <cstring>

#include "cd_pixel.cuh"

namespace hp {

// ------------------------------------------------------------------ host: marker segments
namespace {
inline int be16(const uint8_t* p) { return (p[0] << 8) | p[1]; }
// zig-zag position k -> natural (row-major) index (T.81 Figure A.6)
constexpr uint8_t kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                 12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};
}  // namespace

hp_status jpeg_parse(const uint8_t* d, int64_t n, JpegHdr* H, const char** why) {
    auto bad = [&](const char* m) { *why = m; return HP_ERR_INVALID; };
    auto unsup = [&](const char* m) { *why = m; return HP_ERR_UNSUPPORTED; };
    if (!d || n < 4 || d[0] != 0xFF || d[1] != 0xD8) return bad("not a JPEG (no SOI)");
    std::memset(H, 0, sizeof(*H));
    uint16_t qt[4][64];
    bool have_q[4] = {}, have_h[8] = {}, have_frame = false;
    int cid[3] = {}, ctq[3] = {};
    int ri = 0;
    int64_t p = 2;
    while (p + 4 <= n) {
        if (d[p] != 0xFF) return bad("marker expected");
        const int m = d[p + 1];
        if (m == 0xFF) { ++p; continue; }
        const int len = be16(d + p + 2);
        if (len < 2 || p + 2 + len > n) return bad("segment length");
        const uint8_t* s = d + p + 4;
        const int sl = len - 2;
        switch (m) {
            case 0xDB:  // DQT
                for (int o = 0; o < sl;) {
                    const int pq = s[o] >> 4, tq = s[o] & 15;
                    if (tq > 3 || o + 1 + (pq ? 128 : 64) > sl) return bad("DQT");
                    for (int k = 0; k < 64; ++k) qt[tq][kZigzag[k]] = pq ? be16(s + o + 1 + 2 * k) : s[o + 1 + k];
                    have_q[tq] = true;
                    o += 1 + (pq ? 128 : 64);
                }
                break;
            case 0xC0:
            case 0xC1:  // baseline / extended sequential, Huffman
                if (sl < 6) return bad("SOF");
                if (s[0] != 8) return unsup("sample precision other than 8 bits");
                H->height = be16(s + 1);
                H->width = be16(s + 3);
                if (s[5] != 3) return unsup("component count other than 3");
                if (sl < 15) return bad("SOF");
                for (int i = 0; i < 3; ++i) {
                    cid[i] = s[6 + 3 * i];
                    // 4:4:4, or 4:2:0 (Y 2 x 2, chroma 1 x 1); reading J3
                    if (i == 0 && s[7] == 0x22) H->sub = 2;
                    else if (s[7 + 3 * i] != 0x11) return unsup("chroma sampling other than 4:4:4 / 4:2:0");
                    ctq[i] = s[8 + 3 * i];
                    if (ctq[i] > 3) return bad("SOF table");
                }
                have_frame = true;
                break;
            case 0xC4:  // DHT
                for (int o = 0; o < sl;) {
                    const int tc = s[o] >> 4, th = s[o] & 15;
                    if (tc > 1 || th > 3 || o + 17 > sl) return bad("DHT");
                    const int t = tc * 4 + th;
                    int tot = 0;
                    H->bits[t][0] = 0;
                    for (int l = 1; l <= 16; ++l) tot += (H->bits[t][l] = s[o + l]);
                    if (tot > 256 || o + 17 + tot > sl) return bad("DHT counts");
                    std::memcpy(H->vals[t], s + o + 17, tot);
                    have_h[t] = true;
                    o += 17 + tot;
                }
                break;
            case 0xDD:  // DRI
                if (sl < 2) return bad("DRI");
                ri = be16(s);
                break;
            case 0xDA: {  // SOS: the scan follows
                if (!have_frame) return bad("SOS before SOF");
                if (sl < 10 || s[0] != 3) return unsup("scan without all 3 components");
                for (int j = 0; j < 3; ++j) {
                    if (s[1 + 2 * j] != cid[j]) return unsup("scan component order");
                    H->td[j] = s[2 + 2 * j] >> 4;
                    H->ta[j] = 4 + (s[2 + 2 * j] & 15);
                    if (H->td[j] > 3 || H->ta[j] > 7 || !have_h[H->td[j]] || !have_h[H->ta[j]] || !have_q[ctq[j]])
                        return bad("scan tables");
                    std::memcpy(H->q[j], qt[ctq[j]], sizeof(H->q[j]));
                }
                if (s[7] != 0 || s[8] != 63 || s[9] != 0) return unsup("progressive scan");
                if (H->width < 1 || H->height < 1) return bad("frame size");
                if (H->sub == 0) H->sub = 1;
                H->mcux = (H->width + 8 * H->sub - 1) / (8 * H->sub);
                H->mcuy = (H->height + 8 * H->sub - 1) / (8 * H->sub);
                const int64_t nmcu = (int64_t)H->mcux * H->mcuy;
                H->ri = (ri > 0 && ri < nmcu) ? ri : (int32_t)nmcu;
                H->n_intervals = (int32_t)((nmcu + H->ri - 1) / H->ri);
                H->scan_off = p + 2 + len;
                int64_t e = n;  // the scan ends at EOI (or the end of the buffer)
                if (n >= 2 && d[n - 2] == 0xFF && d[n - 1] == 0xD9) e = n - 2;
                H->scan_len = e - H->scan_off;
                if (H->scan_len < 0) return bad("empty scan");
                *why = "";
                return HP_OK;
            }
            case 0xD9:
                return bad("EOI before the scan");
            default:
                if ((m >= 0xC2 && m <= 0xCF) && m != 0xC4 && m != 0xC8 && m != 0xCC)
                    return unsup("progressive / lossless / arithmetic coding");
                break;  // APPn, COM, ...: skipped
        }
        p += 2 + len;
    }
    return bad("no scan");
}

// ------------------------------------------------------------------ device
namespace {

__device__ const uint8_t d_zigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                         12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                         35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                         58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

constexpr int kChunk = 8192;  // bytes per restart-marker scan chunk (256 threads x 32 B)
constexpr int kDT = 256;      // decode threads per block (one restart interval each); 2 blocks
                              // per SM hold 75,776 threads, so a 4K tile's 65,536 intervals
                              // (restart interval 4) run in one wave

__device__ __forceinline__ bool is_rst(const uint8_t* s, int64_t i, int64_t len) {
    return i + 1 < len && s[i] == 0xFF && s[i + 1] >= 0xD0 && s[i + 1] <= 0xD7;
}

__device__ __forceinline__ int block_sum256(int v, int* red) {
    v = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i];
    __syncthreads();
    return t;
}

// per 8 KB chunk of the scan: the number of restart markers starting in it
__global__ void __launch_bounds__(256) k_rst_count(const JpegHdr* __restrict__ H, const uint8_t* __restrict__ file,
                                                   int32_t* __restrict__ blkcnt) {
    __shared__ int red[8];
    const int64_t len = H->scan_len;
    const uint8_t* s = file + H->scan_off;
    const int64_t nch = (len + kChunk - 1) / kChunk;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        const int64_t b = c * kChunk + threadIdx.x * 32;
        int n = 0;
        for (int i = 0; i < 32; ++i) n += is_rst(s, b + i, len);
        n = block_sum256(n, red);
        if (threadIdx.x == 0) blkcnt[c] = n;
    }
}

// interval start offsets in scan order: starts[0] = 0, starts[k] = 2 + position of the
// k-th marker; err |= 1 unless there are exactly n_intervals - 1 markers
__global__ void __launch_bounds__(256) k_rst_write(const JpegHdr* __restrict__ H, const uint8_t* __restrict__ file,
                                                   const int32_t* __restrict__ blkcnt, int32_t* __restrict__ starts,
                                                   int64_t cap, int32_t* err) {
    __shared__ int red[8];
    __shared__ int wsum[8];
    const int64_t len = H->scan_len;
    const uint8_t* s = file + H->scan_off;
    const int64_t nch = (len + kChunk - 1) / kChunk;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (blockIdx.x == 0) {
        int tot = 0;
        for (int64_t c = threadIdx.x; c < nch; c += 256) tot += blkcnt[c];
        tot = block_sum256(tot, red);
        if (threadIdx.x == 0) {
            starts[0] = 0;
            if (tot != H->n_intervals - 1) atomicOr(err, 1);
        }
    }
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
        int pre = 0;  // markers in the chunks before c
        for (int64_t j = threadIdx.x; j < c; j += 256) pre += blkcnt[j];
        pre = block_sum256(pre, red);
        const int64_t b = c * kChunk + threadIdx.x * 32;
        uint32_t m = 0;
        for (int i = 0; i < 32; ++i) m |= (uint32_t)is_rst(s, b + i, len) << i;
        const int n = __popc(m);
        int incl = n;  // inclusive scan over the block
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        int base = pre + incl - n;
        for (int i = 0; i < wid; ++i) base += wsum[i];
        __syncthreads();
        while (m) {
            const int i = __ffs(m) - 1;
            m &= m - 1;
            const int64_t k = 1 + base++;
            if (k < cap) starts[k] = (int32_t)(b + i + 2);
        }
    }
}

// --- Huffman decoding (one bit reader per thread)
struct HuffSm {
    uint16_t lut[8][512];   // 9-bit lookahead: (length << 8) | symbol, 0 = longer code
    int32_t maxcode[8][18]; // largest code of each length (left unaligned), -1 = none
    int32_t valoff[8][17];  // HUFFVAL index of a code of length l = code + valoff[l]
    uint8_t vals[8][256];
};

// Annex C canonical codes -> the tables above, cooperatively for one block
__device__ void build_tables(const JpegHdr* __restrict__ H, HuffSm& T) {
    __shared__ int32_t mincode[8][17];
    if (threadIdx.x < 8) {
        const int t = threadIdx.x;
        int code = 0, k = 0;
        for (int l = 1; l <= 16; ++l) {
            const int nl = H->bits[t][l];
            mincode[t][l] = code;
            T.valoff[t][l] = k - code;
            T.maxcode[t][l] = nl ? code + nl - 1 : -1;
            code = (code + nl) << 1;
            k += nl;
        }
        T.maxcode[t][17] = 0x7fffffff;
    }
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) T.vals[i >> 8][i & 255] = H->vals[i >> 8][i & 255];
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * 512; i += blockDim.x) {
        const int t = i >> 9, peek = i & 511;
        uint16_t e = 0;
        for (int l = 1; l <= 9; ++l) {
            const int code = peek >> (9 - l);
            if (T.maxcode[t][l] >= 0 && code >= mincode[t][l] && code <= T.maxcode[t][l]) {
                e = (uint16_t)((l << 8) | T.vals[t][code + T.valoff[t][l]]);
                break;
            }
        }
        T.lut[t][peek] = e;
    }
}

struct Bits {
    const uint8_t* p;
    const uint8_t* end;
    uint64_t buf;  // left-aligned
    int n;
    bool marker;   // a marker was met: the segment ended, feed zero bits
    // slow path: one byte at a time, byte stuffing (0xFF 0x00 -> 0xFF) and markers
    __device__ __forceinline__ void refill_bytes() {
        while (n <= 56) {
            uint32_t b = 0;
            if (!marker && p < end) {
                b = __ldg(p);
                if (b == 0xFF) {
                    const uint32_t b2 = p + 1 < end ? __ldg(p + 1) : 0u;
                    if (b2 == 0) p += 2;   // stuffed byte
                    else { marker = true; b = 0; }
                } else {
                    ++p;
                }
            }
            buf |= (uint64_t)b << (56 - n);
            n += 8;
        }
    }
    // fast path: the next 8 bytes in three aligned 32-bit loads; when none of them is 0xFF
    // (no stuffing, no marker) the whole bytes that fit are appended at once
    __device__ __forceinline__ void refill() {
        if (n > 56) return;
        if (!marker && p + 8 <= end) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(p);
            const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
            const uint32_t sh = (uint32_t)(a & 3) * 8;
            const uint32_t w0 = __ldg(wp), w1 = __ldg(wp + 1), w2 = __ldg(wp + 2);
            const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);  // bytes p..p+7
            if (!(__vcmpeq4(lo, 0xffffffffu) | __vcmpeq4(hi, 0xffffffffu))) {
                const uint64_t be = ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
                const int k = (64 - n) >> 3;  // whole bytes that fit: 1..8
                buf |= (k == 8 ? be : (be >> (64 - 8 * k)) << (64 - 8 * k)) >> n;
                p += k;
                n += 8 * k;
                return;
            }
        }
        refill_bytes();
    }
    __device__ __forceinline__ int take(int s) {  // RECEIVE(s), s in 1..16
        const int v = (int)(buf >> (64 - s));
        buf <<= s;
        n -= s;
        return v;
    }
};

__device__ __forceinline__ int extend(int v, int s) { return v < (1 << (s - 1)) ? v - (1 << s) + 1 : v; }

// DECODE (T.81 F.2.2.3) with the lookahead table; -1 for an invalid code
__device__ __forceinline__ int decode_sym(Bits& br, const HuffSm& T, int t) {
    const uint16_t e = T.lut[t][br.buf >> 55];
    if (e) {
        br.buf <<= (e >> 8);
        br.n -= (e >> 8);
        return e & 255;
    }
    for (int l = 10; l <= 16; ++l) {
        const int code = (int)(br.buf >> (64 - l));
        if (code <= T.maxcode[t][l]) {
            br.buf <<= l;
            br.n -= l;
            return T.vals[t][code + T.valoff[t][l]];
        }
    }
    return -1;
}

// --- islow IDCT (reading J1): CONST_BITS 13, PASS1_BITS 2
constexpr int kF0298 = 2446, kF0390 = 3196, kF0541 = 4433, kF0765 = 6270, kF0899 = 7373, kF1175 = 9633,
              kF1501 = 12299, kF1847 = 15137, kF1961 = 16069, kF2053 = 16819, kF2562 = 20995, kF3072 = 25172;

// the 1-D LLM butterfly on x0..x7; results rounded and shifted right by `sh`.  T = long long
// is the IJG's JLONG; T = int is exact whenever every |input| <= kInt32Safe (the largest sum
// of products is below 131520 * |input| < 2^31), which holds for every block of a JPEG
// encoded from 8-bit samples -- the callers check and fall back to 64 bits otherwise.
constexpr int kInt32Safe = 16000;
template <class T>
__device__ __forceinline__ void llm8(T x0, T x1, T x2, T x3, T x4, T x5, T x6, T x7, int sh, int* o) {
    const T z1e = (x2 + x6) * kF0541;
    const T t2 = z1e - x6 * kF1847, t3 = z1e + x2 * kF0765;
    const T t0 = (x0 + x4) * 8192, t1 = (x0 - x4) * 8192;
    const T a10 = t0 + t3, a13 = t0 - t3, a11 = t1 + t2, a12 = t1 - t2;
    T z1 = x7 + x1, z2 = x5 + x3, z3 = x7 + x3, z4 = x5 + x1;
    const T z5 = (z3 + z4) * kF1175;
    T b0 = x7 * kF0298, b1 = x5 * kF2053, b2 = x3 * kF3072, b3 = x1 * kF1501;
    z1 *= -kF0899;
    z2 *= -kF2562;
    z3 = z3 * -kF1961 + z5;
    z4 = z4 * -kF0390 + z5;
    b0 += z1 + z3;
    b1 += z2 + z4;
    b2 += z2 + z3;
    b3 += z1 + z4;
    const T rnd = (T)1 << (sh - 1);
    o[0] = (int)((a10 + b3 + rnd) >> sh);
    o[7] = (int)((a10 - b3 + rnd) >> sh);
    o[1] = (int)((a11 + b2 + rnd) >> sh);
    o[6] = (int)((a11 - b2 + rnd) >> sh);
    o[2] = (int)((a12 + b1 + rnd) >> sh);
    o[5] = (int)((a12 - b1 + rnd) >> sh);
    o[3] = (int)((a13 + b0 + rnd) >> sh);
    o[4] = (int)((a13 - b0 + rnd) >> sh);
}

__device__ __forceinline__ int clamp255(int v) { return min(max(v, 0), 255); }

// c[k * kDT] (this thread's column of the shared coefficient array, natural order, only the
// positions set in `mask` valid) -> pass 1 in place (columns), then rows emitted through
// emit(r, s[8]) as level-shifted, clamped samples
template <class Emit>
__device__ __forceinline__ void idct_block(int* c, uint64_t mask, const uint16_t* __restrict__ q, Emit emit) {
    if (mask <= 1ull) {  // DC only: every sample is the same
        const long long dc = (long long)(mask ? c[0] : 0) * q[0];
        const int v = clamp255((int)((dc * 4 + 16) >> 5) + 128);
        int s[8] = {v, v, v, v, v, v, v, v};
        for (int r = 0; r < 8; ++r) emit(r, s);
        return;
    }
    uint8_t rowac = 0;  // rows with a nonzero pass-1 value off column 0
#pragma unroll 1
    for (int col = 0; col < 8; ++col) {
        const uint64_t cm = (mask >> col) & 0x0101010101010101ull;
        if (cm == 0) {
#pragma unroll
            for (int r = 0; r < 8; ++r) c[(r * 8 + col) * kDT] = 0;
            continue;
        }
        long long x[8];
        long long amax = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            x[r] = ((cm >> (8 * r)) & 1) ? (long long)c[(r * 8 + col) * kDT] * q[r * 8 + col] : 0;
            amax = max(amax, x[r] < 0 ? -x[r] : x[r]);
        }
        if ((cm & ~1ull) == 0) {  // only the DC of this column
            const int v = (int)(x[0] * 4);
#pragma unroll
            for (int r = 0; r < 8; ++r) c[(r * 8 + col) * kDT] = v;
            if (col && v) rowac = 0xff;
            continue;
        }
        int o[8];
        if (amax <= kInt32Safe)
            llm8<int>((int)x[0], (int)x[1], (int)x[2], (int)x[3], (int)x[4], (int)x[5], (int)x[6], (int)x[7], 13 - 2, o);
        else
            llm8<long long>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], 13 - 2, o);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            c[(r * 8 + col) * kDT] = o[r];
            if (col && o[r]) rowac |= (uint8_t)(1u << r);
        }
    }
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        int s[8];
        const int* w = c + r * 8 * kDT;
        if (!((rowac >> r) & 1)) {
            const int v = clamp255((int)(((long long)w[0] + 16) >> 5) + 128);
#pragma unroll
            for (int k = 0; k < 8; ++k) s[k] = v;
        } else {
            int o[8];
            int v[8], amax = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                v[k] = w[k * kDT];
                amax = max(amax, abs(v[k]));
            }
            if (amax <= kInt32Safe)
                llm8<int>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], 13 + 2 + 3, o);
            else
                llm8<long long>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], 13 + 2 + 3, o);
#pragma unroll
            for (int k = 0; k < 8; ++k) s[k] = clamp255(o[k] + 128);
        }
        emit(r, s);
    }
}

// JFIF YCbCr -> RGB, IJG 16-bit fixed point (reading J2)
__device__ __forceinline__ void ycc_rgb(int y, int cb, int cr, int& R, int& G, int& B) {
    const int xb = cb - 128, xr = cr - 128;
    R = clamp255(y + ((91881 * xr + 32768) >> 16));
    G = clamp255(y + ((-22554 * xb - 46802 * xr + 32768) >> 16));
    B = clamp255(y + ((116130 * xb + 32768) >> 16));
}

// kMode 0: 4:4:4 fused into S1; 1: 4:4:4 to RGB (verification); 2: 4:2:0 to component planes
template <int kMode>
__global__ void __launch_bounds__(kDT, 2) k_jpeg_decode(const JpegHdr* __restrict__ H, const uint8_t* __restrict__ file,
                                                     const int32_t* __restrict__ starts, const float* __restrict__ lut_g,
                                                     CdConst k, uint8_t* __restrict__ g, uint8_t* __restrict__ flags,
                                                     unsigned long long* bg_count, uint8_t* __restrict__ rgb,
                                                     int64_t rgb_pitch, uint8_t* __restrict__ planes, int32_t* err) {
    constexpr bool kRGB = kMode == 1;
    __shared__ HuffSm T;
    __shared__ uint16_t q[3][64];
    __shared__ float od[256];
    __shared__ uint8_t zz[64];
    extern __shared__ int dyn[];
    int* coef = dyn + threadIdx.x;                                                // [64][kDT] int32
    uint8_t* smp = reinterpret_cast<uint8_t*>(dyn + 64 * kDT) + threadIdx.x;      // [2][64][kDT] u8
    build_tables(H, T);
    for (int i = threadIdx.x; i < 3 * 64; i += kDT) q[i >> 6][i & 63] = H->q[i >> 6][i & 63];
    for (int i = threadIdx.x; i < 256; i += kDT) od[i] = lut_g[i];
    if (threadIdx.x < 64) zz[threadIdx.x] = d_zigzag[threadIdx.x];
    __syncthreads();
    const int w = H->width, h = H->height, mcux = H->mcux, ri = H->ri, nint = H->n_intervals;
    const int64_t nmcu = (int64_t)mcux * H->mcuy;
    const uint8_t* scan = file + H->scan_off;
    const uint8_t* scan_end = scan + H->scan_len;
    // table ids of the three components packed in bytes (no local-memory arrays)
    const uint32_t tdp = H->td[0] | H->td[1] << 8 | H->td[2] << 16, tap = H->ta[0] | H->ta[1] << 8 | H->ta[2] << 16;
    const bool vec8 = (w & 7) == 0;
    int nbg = 0;
    for (int iv = blockIdx.x * kDT + threadIdx.x; iv < nint; iv += gridDim.x * kDT) {
        Bits br{scan + starts[iv], scan_end, 0ull, 0, false};
        int pred[3] = {0, 0, 0};
        const int64_t m0 = (int64_t)iv * ri, m1 = min(m0 + ri, nmcu);
        bool bad = false;
        for (int64_t m = m0; m < m1 && !bad; ++m) {
            const int bx = (int)(m % mcux) * 8 * (kMode == 2 ? 2 : 1), by = (int)(m / mcux) * 8 * (kMode == 2 ? 2 : 1);
#pragma unroll 1
            for (int blk = 0; blk < (kMode == 2 ? 6 : 3); ++blk) {
                // 4:2:0: four Y blocks (raster order inside the MCU), then Cb, Cr
                const int cpt = kMode == 2 ? (blk < 4 ? 0 : blk - 3) : blk;
                // --- F.2.2.1 / F.2.2.2: the block's coefficients, zig-zag -> natural order
                br.refill();
                int t = decode_sym(br, T, (tdp >> (8 * cpt)) & 0xff);
                if (t < 0 || t > 15) { bad = true; break; }
                pred[cpt] += t ? extend(br.take(t), t) : 0;
                coef[0] = pred[cpt];
                uint64_t mask = 1;
                for (int kk = 1; kk < 64;) {
                    if (br.n < 32) br.refill();
                    const int rs = decode_sym(br, T, (tap >> (8 * cpt)) & 0xff);
                    if (rs < 0) { bad = true; break; }
                    const int ss = rs & 15, rr = rs >> 4;
                    if (ss == 0) {
                        if (rr == 15) { kk += 16; continue; }
                        break;  // EOB
                    }
                    kk += rr;
                    if (kk > 63) { bad = true; break; }
                    const int z = zz[kk];
                    coef[z * kDT] = extend(br.take(ss), ss);
                    mask |= 1ull << z;
                    ++kk;
                }
                if (bad) break;
                // --- IDCT
                if (kMode == 2) {  // into the component planes (Y pitch yw, chroma pitch yw / 2)
                    const int yw = mcux * 16, cwp = mcux * 8;
                    uint8_t* dst;
                    if (cpt == 0) {
                        dst = planes + (int64_t)(by + 8 * (blk >> 1)) * yw + bx + 8 * (blk & 1);
                    } else {
                        const int64_t cplane = (int64_t)cwp * H->mcuy * 8;
                        dst = planes + (int64_t)yw * H->mcuy * 16 + (cpt - 1) * cplane + (int64_t)(by / 2) * cwp + bx / 2;
                    }
                    const int pitch = cpt == 0 ? yw : cwp;
                    idct_block(coef, mask, q[cpt], [&](int r, const int* sm) {
                        uint2 v;
                        v.x = sm[0] | sm[1] << 8 | sm[2] << 16 | (uint32_t)sm[3] << 24;
                        v.y = sm[4] | sm[5] << 8 | sm[6] << 16 | (uint32_t)sm[7] << 24;
                        *reinterpret_cast<uint2*>(dst + (int64_t)r * pitch) = v;
                    });
                } else if (cpt < 2) {  // Y and Cb samples parked, Cr rows converted and consumed at once
                    uint8_t* dst = smp + cpt * 64 * kDT;
                    idct_block(coef, mask, q[cpt], [&](int r, const int* s) {
#pragma unroll
                        for (int x = 0; x < 8; ++x) dst[(r * 8 + x) * kDT] = (uint8_t)s[x];
                    });
                } else {
                    idct_block(coef, mask, q[2], [&](int r, const int* s) {
                        const int y = by + r;
                        if (y >= h) return;
                        uint8_t gv[8], fv[8], cv[24];
#pragma unroll
                        for (int x = 0; x < 8; ++x) {
                            int R, G, B;
                            ycc_rgb(smp[(r * 8 + x) * kDT], smp[(64 + r * 8 + x) * kDT], s[x], R, G, B);
                            if (kRGB) {
                                cv[3 * x] = (uint8_t)R;
                                cv[3 * x + 1] = (uint8_t)G;
                                cv[3 * x + 2] = (uint8_t)B;
                            } else {
                                int nb = 0;
                                cd_pixel(R, G, B, od, k, gv[x], fv[x], nb);
                                if (bx + x < w) nbg += nb;
                            }
                        }
                        if (kRGB) {
                            uint8_t* o = rgb + (int64_t)y * rgb_pitch + 3 * bx;
                            for (int x = 0; x < 8 && bx + x < w; ++x) {
                                o[3 * x] = cv[3 * x];
                                o[3 * x + 1] = cv[3 * x + 1];
                                o[3 * x + 2] = cv[3 * x + 2];
                            }
                        } else if (vec8) {
                            const int64_t o = (int64_t)y * w + bx;
                            uint2 gw, fw;
                            gw.x = gv[0] | gv[1] << 8 | gv[2] << 16 | (uint32_t)gv[3] << 24;
                            gw.y = gv[4] | gv[5] << 8 | gv[6] << 16 | (uint32_t)gv[7] << 24;
                            fw.x = fv[0] | fv[1] << 8 | fv[2] << 16 | (uint32_t)fv[3] << 24;
                            fw.y = fv[4] | fv[5] << 8 | fv[6] << 16 | (uint32_t)fv[7] << 24;
                            *reinterpret_cast<uint2*>(g + o) = gw;
                            *reinterpret_cast<uint2*>(flags + o) = fw;
                        } else {
                            const int64_t o = (int64_t)y * w + bx;
                            for (int x = 0; x < 8 && bx + x < w; ++x) {
                                g[o + x] = gv[x];
                                flags[o + x] = fv[x];
                            }
                        }
                    });
                }
            }
        }
        if (bad) atomicOr(err, 2);
    }
    if (kMode == 0 && bg_count) block_count(nbg, bg_count);
}

// 4:2:0 -> full resolution (reading J4, the IJG triangle filter), JFIF colour, then S1 (or the
// RGB tile for verification).  A thread makes 8 output pixels of a row from 8 Y samples and
// the 6 chroma columns around them in the nearer and the next nearer chroma row.
template <bool kRGB>
__global__ void __launch_bounds__(256) k_jpeg_up_cd(const JpegHdr* __restrict__ H, const uint8_t* __restrict__ planes,
                                                    const float* __restrict__ lut_g, CdConst k, uint8_t* __restrict__ g,
                                                    uint8_t* __restrict__ flags, unsigned long long* bg_count,
                                                    uint8_t* __restrict__ rgb, int64_t rgb_pitch) {
    __shared__ float od[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) od[i] = lut_g[i];
    __syncthreads();
    const int w = H->width, h = H->height;
    const int yw = H->mcux * 16, cwp = H->mcux * 8;
    const int64_t cplane = (int64_t)cwp * H->mcuy * 8;
    const uint8_t* Yp = planes;
    const uint8_t* Cp[2] = {planes + (int64_t)yw * H->mcuy * 16, planes + (int64_t)yw * H->mcuy * 16 + cplane};
    const int dw = (w + 1) / 2, dh = (h + 1) / 2;  // downsampled width / height
    const int gpr = (w + 7) / 8;                   // 8-pixel groups per row
    const int64_t ngroups = (int64_t)gpr * h;
    const bool vec8 = (w & 7) == 0;
    int nbg = 0;
    for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < ngroups; gi += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(gi / gpr), x0 = (int)(gi % gpr) * 8;
        const int ir = y >> 1;
        const int fr = min(max((y & 1) ? ir + 1 : ir - 1, 0), dh - 1);  // next nearer chroma row
        const int c0 = x0 >> 1;                                         // chroma columns c0 .. c0 + 3
        int up[2][8];
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
            const uint8_t* rn = Cp[pl] + (int64_t)ir * cwp;
            const uint8_t* rf = Cp[pl] + (int64_t)fr * cwp;
            if (dw <= 2) {  // the IJG library replicates chroma of at most 2 samples per row
#pragma unroll
                for (int j = 0; j < 8; ++j) up[pl][j] = rn[min((x0 + j) >> 1, cwp - 1)];
                continue;
            }
            int cs[6];  // column sums of chroma columns c0 - 1 .. c0 + 4
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                const int c = min(max(c0 - 1 + j, 0), cwp - 1);
                cs[j] = 3 * rn[c] + rf[c];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = c0 + j;
                up[pl][2 * j] = c == 0 ? (cs[j + 1] * 4 + 8) >> 4 : (cs[j + 1] * 3 + cs[j] + 8) >> 4;
                up[pl][2 * j + 1] = c >= dw - 1 ? (cs[j + 1] * 4 + 7) >> 4 : (cs[j + 1] * 3 + cs[j + 2] + 7) >> 4;
            }
        }
        const uint8_t* yr = Yp + (int64_t)y * yw + x0;
        uint8_t gv[8], fv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int R, G, B;
            ycc_rgb(yr[j], up[0][j], up[1][j], R, G, B);
            if (kRGB) {
                if (x0 + j < w) {
                    uint8_t* o = rgb + (int64_t)y * rgb_pitch + 3 * (x0 + j);
                    o[0] = (uint8_t)R;
                    o[1] = (uint8_t)G;
                    o[2] = (uint8_t)B;
                }
            } else {
                int nb = 0;
                cd_pixel(R, G, B, od, k, gv[j], fv[j], nb);
                if (x0 + j < w) nbg += nb;
            }
        }
        if (!kRGB) {
            const int64_t o = (int64_t)y * w + x0;
            if (vec8) {
                uint2 gw, fw;
                gw.x = gv[0] | gv[1] << 8 | gv[2] << 16 | (uint32_t)gv[3] << 24;
                gw.y = gv[4] | gv[5] << 8 | gv[6] << 16 | (uint32_t)gv[7] << 24;
                fw.x = fv[0] | fv[1] << 8 | fv[2] << 16 | (uint32_t)fv[3] << 24;
                fw.y = fv[4] | fv[5] << 8 | fv[6] << 16 | (uint32_t)fv[7] << 24;
                *reinterpret_cast<uint2*>(g + o) = gw;
                *reinterpret_cast<uint2*>(flags + o) = fw;
            } else {
                for (int j = 0; j < 8 && x0 + j < w; ++j) {
                    g[o + j] = gv[j];
                    flags[o + j] = fv[j];
                }
            }
        }
    }
    if (!kRGB && bg_count) block_count(nbg, bg_count);
}

}  // namespace

void launch_jpeg_decode(const JpegHdr* hdr, int sub, const uint8_t* file, int64_t file_cap, int w, int h,
                        int32_t* starts, int32_t* blkcnt, uint8_t* planes, const float* lut, const hp_params& p,
                        uint8_t* g, uint8_t* flags, unsigned long long* bg_count, uint8_t* rgb, int64_t rgb_pitch,
                        int32_t* err, cudaStream_t s) {
    if (bg_count) cudaMemsetAsync(bg_count, 0, sizeof(unsigned long long), s);
    const int nsm = num_sms();
    const int64_t nch = file_cap / kChunk + 1;
    const int gs = (int)std::min<int64_t>(nch, nsm * 4);
    (note_launch(), k_rst_count<<<gs, 256, 0, s>>>(hdr, file, blkcnt));
    (note_launch(), k_rst_write<<<gs, 256, 0, s>>>(hdr, file, blkcnt, starts, jpeg_max_intervals(w, h), err));
    const size_t dyn = 64 * kDT * sizeof(int) + 2 * 64 * kDT;
    static PerDevice once;
    once.get([&] {
        cudaFuncSetAttribute(k_jpeg_decode<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k_jpeg_decode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k_jpeg_decode<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        return 0;
    });
    const int mpx = 8 * sub;
    const int64_t nint_max = ((int64_t)((w + mpx - 1) / mpx) * ((h + mpx - 1) / mpx));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nint_max + kDT - 1) / kDT, nsm * 2));
    const CdConst k = cd_const(p);
    if (sub == 2) {
        (note_launch(), k_jpeg_decode<2><<<grid, kDT, dyn, s>>>(hdr, file, starts, lut, k, nullptr, nullptr, nullptr,
                                                               nullptr, 0, planes, err));
        const int64_t ng = (int64_t)((w + 7) / 8) * h;
        const int ug = (int)std::max<int64_t>(1, std::min<int64_t>((ng + 255) / 256, nsm * 8));
        if (rgb)
            (note_launch(), k_jpeg_up_cd<true><<<ug, 256, 0, s>>>(hdr, planes, lut, k, nullptr, nullptr, nullptr, rgb,
                                                                rgb_pitch));
        else
            (note_launch(), k_jpeg_up_cd<false><<<ug, 256, 0, s>>>(hdr, planes, lut, k, g, flags, bg_count, nullptr, 0));
        return;
    }
    if (rgb)
        (note_launch(), k_jpeg_decode<1><<<grid, kDT, dyn, s>>>(hdr, file, starts, lut, k, g, flags, nullptr, rgb,
                                                               rgb_pitch, nullptr, err));
    else
        (note_launch(), k_jpeg_decode<0><<<grid, kDT, dyn, s>>>(hdr, file, starts, lut, k, g, flags, bg_count,
                                                               nullptr, 0, nullptr, err));
}

}  // namespace hp
