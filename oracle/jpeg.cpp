// jpeg.cpp -- plain CPU oracle of the compressed-ingest step (SURVEY.md §8(f) NEXT-3:
// tiles arrive JPEG-compressed, "the main limiting factor and bottleneck is
// the I/O overhead of reading image tiles", 716-726).  TEST INFRASTRUCTURE ONLY (see
// oracle.h); shares nothing with libhp.
//
// A baseline sequential JPEG decoder written step by step from ITU-T T.81 (1992), in its
// order and names:
//   B.2      the marker segments (SOI, DQT, SOF0/1, DHT, DRI, SOS, EOI; APPn/COM skipped);
//   C        Huffman tables from BITS/HUFFVAL: Generate_size_table (Figure C.1),
//            Generate_code_table (Figure C.2);
//   F.2.2.3  decoder tables MINCODE / MAXCODE / VALPTR (Figure F.15) and DECODE (F.16);
//   F.2.2.4  NEXTBIT with byte stuffing (Figure F.18), RECEIVE (F.17), EXTEND (F.12);
//   F.2.2.1  DC difference and prediction, F.2.2.2 AC coefficients (Figure F.13);
//   F.2.1.3  restart intervals (prediction reset at every RSTm);
//   A.3.4    dequantisation, A.3.6 zig-zag order.
// Two steps T.81 leaves to the implementation follow the readings J1-J2 of DESIGN.md:
//   J1  IDCT: the integer Loeffler-Ligtenberg-Moschytz factorisation with 13-bit constants
//       (two 1-D passes, columns then rows, 2 extra fraction bits between them) -- the
//       "islow" method of the IJG library that cv2.imdecode uses -- then +128 and a clamp
//       to 0..255 (T.81 A.3.1 level shift);
//   J2  colour: JFIF YCbCr -> RGB, R = Y + 1.402 (Cr-128), G = Y - 0.34414 (Cb-128)
//       - 0.71414 (Cr-128), B = Y + 1.772 (Cb-128), with the IJG 16-bit fixed-point
//       rounding, clamped to 0..255.
// Scope: 8-bit precision, 3 components, 4:4:4 or 4:2:0 sampling, one interleaved scan;
// anything else returns 5 (unsupported).  4:2:0 chroma is brought to full resolution by the
// IJG "fancy" triangle filter (reading J4).  No blocking or reordering beyond this.
#include <cstdint>
#include <cstring>
#include <vector>

#include "oracle.h"

namespace {

// A.3.6, Figure A.6: zig-zag index k -> natural (row-major) position
const int ZZ[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

struct Huff {  // Annex C + F.2.2.3 decoder tables
    bool present = false;
    uint8_t bits[17] = {};   // BITS[1..16]
    uint8_t huffval[256] = {};
    int mincode[17], maxcode[18], valptr[17];
};

void make_decoder_tables(Huff& t) {
    // Figure C.1 Generate_size_table
    int huffsize[257], huffcode[257];
    int k = 0;
    for (int i = 1; i <= 16; ++i)
        for (int j = 1; j <= t.bits[i]; ++j) huffsize[k++] = i;
    huffsize[k] = 0;
    const int lastk = k;
    // Figure C.2 Generate_code_table
    k = 0;
    int code = 0, si = huffsize[0];
    while (k < lastk) {
        while (huffsize[k] == si) {
            huffcode[k++] = code++;
        }
        if (huffsize[k] == 0) break;
        do {
            code <<= 1;
            ++si;
        } while (huffsize[k] != si);
    }
    // Figure F.15 Decoder_tables
    int j = 0;
    for (int i = 1; i <= 16; ++i) {
        if (t.bits[i] == 0) {
            t.maxcode[i] = -1;
        } else {
            t.valptr[i] = j;
            t.mincode[i] = huffcode[j];
            j += t.bits[i] - 1;
            t.maxcode[i] = huffcode[j];
            ++j;
        }
    }
    t.maxcode[17] = 0x7fffffff;
}

struct Reader {  // F.2.2.4 NEXTBIT over the entropy-coded segment
    const uint8_t* d;
    int64_t n, pos;
    int cnt = 0;
    int b = 0;
    bool marker_hit = false;  // a marker (not 0xFF00) was met: feed zeros (the data ended)
    int nextbit() {
        if (cnt == 0) {
            if (marker_hit || pos >= n) {
                b = 0;
            } else {
                b = d[pos++];
                if (b == 0xFF) {
                    const int b2 = pos < n ? d[pos] : 0;
                    if (b2 == 0) {
                        ++pos;  // stuffed zero byte
                    } else {
                        marker_hit = true;  // a marker inside the data: no more bits
                        --pos;
                        b = 0;
                    }
                }
            }
            cnt = 8;
        }
        const int bit = (b >> 7) & 1;
        --cnt;
        b = (b << 1) & 0xFF;
        return bit;
    }
    int receive(int ssss) {  // Figure F.17
        int v = 0;
        for (int i = 0; i < ssss; ++i) v = (v << 1) + nextbit();
        return v;
    }
    int decode(const Huff& t) {  // Figure F.16
        int i = 1;
        int code = nextbit();
        while (i <= 16 && code > t.maxcode[i]) {
            ++i;
            code = (code << 1) + nextbit();
        }
        if (i > 16) return -1;  // no such code
        return t.huffval[t.valptr[i] + code - t.mincode[i]];
    }
    // F.2.1.3.1: at a restart the remaining bits of the byte are discarded, then RSTm
    bool restart() {
        cnt = 0;
        marker_hit = false;
        while (pos + 1 < n && !(d[pos] == 0xFF && d[pos + 1] >= 0xD0 && d[pos + 1] <= 0xD7)) ++pos;
        if (pos + 1 >= n) return false;
        pos += 2;
        return true;
    }
};

int extend(int v, int t) {  // Figure F.12
    return (t > 0 && v < (1 << (t - 1))) ? v + (-1 << t) + 1 : v;
}

// Reading J1: the IJG islow integer IDCT (CONST_BITS 13, PASS1_BITS 2), level shift, clamp.
const int64_t F0_298 = 2446, F0_390 = 3196, F0_541 = 4433, F0_765 = 6270, F0_899 = 7373,
              F1_175 = 9633, F1_501 = 12299, F1_847 = 15137, F1_961 = 16069, F2_053 = 16819,
              F2_562 = 20995, F3_072 = 25172;

int64_t descale(int64_t x, int n) { return (x + ((int64_t)1 << (n - 1))) >> n; }

// one 1-D inverse transform of 8 inputs in[0..7] (frequency order) -> out[0..7] scaled by
// 2^shift, as the LLM flow graph: even part (0, 2, 4, 6), odd part (1, 3, 5, 7)
void idct_1d(const int64_t in[8], int64_t out[8], int shift) {
    int64_t z2 = in[2], z3 = in[6];
    int64_t z1 = (z2 + z3) * F0_541;
    int64_t tmp2 = z1 + z3 * (-F1_847);
    int64_t tmp3 = z1 + z2 * F0_765;
    int64_t tmp0 = (in[0] + in[4]) * 8192;  // << CONST_BITS
    int64_t tmp1 = (in[0] - in[4]) * 8192;
    const int64_t t10 = tmp0 + tmp3, t13 = tmp0 - tmp3, t11 = tmp1 + tmp2, t12 = tmp1 - tmp2;
    tmp0 = in[7];
    tmp1 = in[5];
    tmp2 = in[3];
    tmp3 = in[1];
    z1 = tmp0 + tmp3;
    z2 = tmp1 + tmp2;
    z3 = tmp0 + tmp2;
    int64_t z4 = tmp1 + tmp3;
    const int64_t z5 = (z3 + z4) * F1_175;
    tmp0 *= F0_298;
    tmp1 *= F2_053;
    tmp2 *= F3_072;
    tmp3 *= F1_501;
    z1 *= -F0_899;
    z2 *= -F2_562;
    z3 *= -F1_961;
    z4 *= -F0_390;
    z3 += z5;
    z4 += z5;
    tmp0 += z1 + z3;
    tmp1 += z2 + z4;
    tmp2 += z2 + z3;
    tmp3 += z1 + z4;
    out[0] = descale(t10 + tmp3, shift);
    out[7] = descale(t10 - tmp3, shift);
    out[1] = descale(t11 + tmp2, shift);
    out[6] = descale(t11 - tmp2, shift);
    out[2] = descale(t12 + tmp1, shift);
    out[5] = descale(t12 - tmp1, shift);
    out[3] = descale(t13 + tmp0, shift);
    out[4] = descale(t13 - tmp0, shift);
}

// dequantised coefficients coef[64] (natural order) -> 8x8 samples 0..255
void idct_block(const int32_t coef[64], uint8_t out[64]) {
    int64_t ws[64];
    for (int c = 0; c < 8; ++c) {  // pass 1: columns, keep 2 fraction bits
        int64_t in[8], o[8];
        for (int r = 0; r < 8; ++r) in[r] = coef[r * 8 + c];
        idct_1d(in, o, 13 - 2);
        for (int r = 0; r < 8; ++r) ws[r * 8 + c] = o[r];
    }
    for (int r = 0; r < 8; ++r) {  // pass 2: rows, remove the 2 bits and the factor 8
        int64_t in[8], o[8];
        for (int c = 0; c < 8; ++c) in[c] = ws[r * 8 + c];
        idct_1d(in, o, 13 + 2 + 3);
        for (int c = 0; c < 8; ++c) {
            int64_t v = o[c] + 128;  // level shift (A.3.1)
            out[r * 8 + c] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
        }
    }
}

// Reading J2: JFIF YCbCr -> RGB in the IJG 16-bit fixed point
int clamp255(int64_t v) { return v < 0 ? 0 : v > 255 ? 255 : (int)v; }
void ycc_to_rgb(int y, int cb, int cr, uint8_t* rgb) {
    const int64_t ONE_HALF = 1 << 15;
    const int64_t FIX_1_40200 = 91881, FIX_1_77200 = 116130, FIX_0_71414 = 46802, FIX_0_34414 = 22554;
    const int64_t x_cb = cb - 128, x_cr = cr - 128;
    const int64_t r_off = (FIX_1_40200 * x_cr + ONE_HALF) >> 16;
    const int64_t b_off = (FIX_1_77200 * x_cb + ONE_HALF) >> 16;
    const int64_t g_off = (-FIX_0_34414 * x_cb - FIX_0_71414 * x_cr + ONE_HALF) >> 16;
    rgb[0] = (uint8_t)clamp255(y + r_off);
    rgb[1] = (uint8_t)clamp255(y + g_off);
    rgb[2] = (uint8_t)clamp255(y + b_off);
}

int u16(const uint8_t* p) { return (p[0] << 8) | p[1]; }

}  // namespace

extern "C" int or_jpeg_decode(const uint8_t* data, int64_t n, int32_t* width, int32_t* height, uint8_t* rgb) {
    if (!data || n < 4 || !width || !height) return 1;
    if (data[0] != 0xFF || data[1] != 0xD8) return 1;  // SOI
    int32_t qt[4][64];          // natural order
    bool qt_present[4] = {};
    Huff dc[4], ac[4];
    int X = 0, Y = 0, Nf = 0, Ri = 0;
    int comp_id[3], comp_h[3], comp_v[3], comp_tq[3], comp_td[3], comp_ta[3];
    bool frame = false;
    int64_t p = 2;
    while (p + 4 <= n) {
        if (data[p] != 0xFF) return 1;
        const int m = data[p + 1];
        if (m == 0xFF) {  // fill byte
            ++p;
            continue;
        }
        const int L = u16(data + p + 2);
        const uint8_t* seg = data + p + 4;
        if (p + 2 + L > n) return 1;
        if (m == 0xDB) {  // DQT (B.2.4.1)
            int off = 0;
            while (off < L - 2) {
                const int pq = seg[off] >> 4, tq = seg[off] & 15;
                if (tq > 3) return 1;
                ++off;
                for (int k = 0; k < 64; ++k) {
                    const int v = pq ? u16(seg + off + 2 * k) : seg[off + k];
                    qt[tq][ZZ[k]] = v;
                }
                off += pq ? 128 : 64;
                qt_present[tq] = true;
            }
        } else if (m == 0xC0 || m == 0xC1) {  // SOF0 / SOF1 (B.2.2), Huffman sequential
            if (seg[0] != 8) return 5;
            Y = u16(seg + 1);
            X = u16(seg + 3);
            Nf = seg[5];
            if (Nf != 3) return 5;
            for (int i = 0; i < 3; ++i) {
                comp_id[i] = seg[6 + 3 * i];
                comp_h[i] = seg[7 + 3 * i] >> 4;
                comp_v[i] = seg[7 + 3 * i] & 15;
                comp_tq[i] = seg[8 + 3 * i];
                // 4:4:4 (every component 1x1) or 4:2:0 (Y 2x2, Cb and Cr 1x1); reading J3
                const bool ok = i == 0 ? ((comp_h[0] == 1 && comp_v[0] == 1) || (comp_h[0] == 2 && comp_v[0] == 2))
                                       : (comp_h[i] == 1 && comp_v[i] == 1);
                if (!ok) return 5;
                if (comp_tq[i] > 3) return 1;
            }
            frame = true;
        } else if ((m >= 0xC2 && m <= 0xCF) && m != 0xC4 && m != 0xC8 && m != 0xCC) {
            return 5;  // progressive, lossless, arithmetic: not supported
        } else if (m == 0xC4) {  // DHT (B.2.4.2)
            int off = 0;
            while (off < L - 2) {
                const int tc = seg[off] >> 4, th = seg[off] & 15;
                if (tc > 1 || th > 3) return 1;
                Huff& t = tc == 0 ? dc[th] : ac[th];
                int total = 0;
                for (int i = 1; i <= 16; ++i) {
                    t.bits[i] = seg[off + i];
                    total += t.bits[i];
                }
                if (total > 256) return 1;
                for (int k = 0; k < total; ++k) t.huffval[k] = seg[off + 17 + k];
                off += 17 + total;
                t.present = true;
                make_decoder_tables(t);
            }
        } else if (m == 0xDD) {  // DRI (B.2.4.4)
            Ri = u16(seg);
        } else if (m == 0xDA) {  // SOS (B.2.3): then the entropy-coded data
            if (!frame) return 1;
            const int Ns = seg[0];
            if (Ns != 3) return 5;
            for (int j = 0; j < 3; ++j) {
                const int cs = seg[1 + 2 * j];
                int ci = -1;
                for (int i = 0; i < 3; ++i)
                    if (comp_id[i] == cs) ci = i;
                if (ci != j) return 5;  // components in frame order
                comp_td[ci] = seg[2 + 2 * j] >> 4;
                comp_ta[ci] = seg[2 + 2 * j] & 15;
                if (comp_td[ci] > 3 || comp_ta[ci] > 3 || !dc[comp_td[ci]].present || !ac[comp_ta[ci]].present ||
                    !qt_present[comp_tq[ci]])
                    return 1;
            }
            if (seg[7] != 0 || seg[8] != 63 || seg[9] != 0) return 5;  // Ss, Se, Ah|Al of a sequential scan
            *width = X;
            *height = Y;
            if (!rgb) return 0;  // size query
            // F.2 / A.2.3: MCUs in raster order; an MCU holds H x V blocks of Y (raster order
            // inside the MCU), then one block of Cb and one of Cr.  4:4:4 (H = V = 1) or 4:2:0
            // (H = V = 2).  The decoded samples go to component planes padded to whole MCUs.
            const int Hy = comp_h[0], Vy = comp_v[0];
            const int mw = 8 * Hy, mh = 8 * Vy;  // MCU size in pixels
            const int mx = (X + mw - 1) / mw, my = (Y + mh - 1) / mh;
            const int64_t nmcu = (int64_t)mx * my;
            const int yw = mx * mw, yh = my * mh, cw = mx * 8, chh = my * 8;  // plane sizes
            std::vector<uint8_t> plane_y((size_t)yw * yh), plane_cb((size_t)cw * chh), plane_cr((size_t)cw * chh);
            Reader rd{data, n, p + 2 + L};
            int pred[3] = {0, 0, 0};
            int32_t coef[64];
            uint8_t smp[64];
            for (int64_t mcu = 0; mcu < nmcu; ++mcu) {
                if (Ri > 0 && mcu > 0 && mcu % Ri == 0) {  // F.2.1.3.1 restart
                    if (!rd.restart()) return 1;
                    pred[0] = pred[1] = pred[2] = 0;
                }
                const int mcx = (int)(mcu % mx), mcy = (int)(mcu / mx);
                for (int c = 0; c < 3; ++c) {
                    const int nb = c == 0 ? Hy * Vy : 1;
                    for (int bi = 0; bi < nb; ++bi) {
                        int zz[64] = {};
                        // F.2.2.1 DC
                        const int t = rd.decode(dc[comp_td[c]]);
                        if (t < 0 || t > 11) return 1;
                        const int diff = extend(rd.receive(t), t);
                        pred[c] += diff;
                        zz[0] = pred[c];
                        // F.2.2.2 AC (Figure F.13)
                        int k = 1;
                        while (k < 64) {
                            const int rs = rd.decode(ac[comp_ta[c]]);
                            if (rs < 0) return 1;
                            const int ssss = rs & 15, rrrr = rs >> 4;
                            if (ssss == 0) {
                                if (rrrr == 15) {
                                    k += 16;
                                    continue;
                                }
                                break;  // EOB
                            }
                            k += rrrr;
                            if (k > 63) return 1;
                            zz[k] = extend(rd.receive(ssss), ssss);
                            ++k;
                        }
                        // A.3.4 dequantisation, A.3.6 zig-zag -> natural order
                        for (int kk = 0; kk < 64; ++kk) coef[ZZ[kk]] = zz[kk] * qt[comp_tq[c]][ZZ[kk]];
                        idct_block(coef, smp);
                        uint8_t* pl = c == 0 ? plane_y.data() : c == 1 ? plane_cb.data() : plane_cr.data();
                        const int pw = c == 0 ? yw : cw;
                        const int ox = c == 0 ? mcx * mw + 8 * (bi % Hy) : mcx * 8;
                        const int oy = c == 0 ? mcy * mh + 8 * (bi / Hy) : mcy * 8;
                        for (int r = 0; r < 8; ++r)
                            for (int cc = 0; cc < 8; ++cc) pl[(size_t)(oy + r) * pw + ox + cc] = smp[r * 8 + cc];
                    }
                }
            }
            // chroma at full resolution: copied (4:4:4), or reading J4's triangle-filter
            // ("fancy") upsampling of the IJG library for 4:2:0 -- per output row, the nearer
            // chroma row weighted 3 and the next nearer 1 (the first / last real row repeated at
            // the image edges), then the same 3:1 weights across columns with the rounding
            // offsets 8 and 7 of the two output pixels of a chroma column
            std::vector<uint8_t> up_cb((size_t)X * Y), up_cr((size_t)X * Y);
            if (Hy == 1 || (X + 1) / 2 <= 2) {
                // 4:4:4 copies; the IJG library filters only chroma wider than 2 samples and
                // replicates each sample to 2 x 2 otherwise
                const int sh = Hy == 1 ? 0 : 1;
                for (int y = 0; y < Y; ++y)
                    for (int x = 0; x < X; ++x) {
                        up_cb[(size_t)y * X + x] = plane_cb[(size_t)(y >> sh) * cw + (x >> sh)];
                        up_cr[(size_t)y * X + x] = plane_cr[(size_t)(y >> sh) * cw + (x >> sh)];
                    }
            } else {
                const int dw = (X + 1) / 2, dh = (Y + 1) / 2;  // downsampled_width / height
                std::vector<int> colsum(cw);
                for (int pass = 0; pass < 2; ++pass) {
                    const std::vector<uint8_t>& src = pass == 0 ? plane_cb : plane_cr;
                    std::vector<uint8_t>& dst = pass == 0 ? up_cb : up_cr;
                    std::vector<uint8_t> row((size_t)2 * cw + 2);
                    for (int y = 0; y < Y; ++y) {
                        const int ir = y / 2;
                        int fr = (y % 2 == 0) ? ir - 1 : ir + 1;  // the next nearer row
                        if (fr < 0) fr = 0;
                        if (fr > dh - 1) fr = dh - 1;
                        for (int c = 0; c < cw; ++c) colsum[c] = 3 * src[(size_t)ir * cw + c] + src[(size_t)fr * cw + c];
                        // the IJG column loop: first column, dw - 2 general columns, last column
                        int o = 0;
                        int thiscol = colsum[0], nextcol = colsum[1 < cw ? 1 : 0], lastcol;
                        row[o++] = (uint8_t)((thiscol * 4 + 8) >> 4);
                        row[o++] = (uint8_t)((thiscol * 3 + nextcol + 7) >> 4);
                        lastcol = thiscol;
                        thiscol = nextcol;
                        for (int c = 2; c < dw; ++c) {
                            nextcol = colsum[c];
                            row[o++] = (uint8_t)((thiscol * 3 + lastcol + 8) >> 4);
                            row[o++] = (uint8_t)((thiscol * 3 + nextcol + 7) >> 4);
                            lastcol = thiscol;
                            thiscol = nextcol;
                        }
                        row[o++] = (uint8_t)((thiscol * 3 + lastcol + 8) >> 4);
                        row[o++] = (uint8_t)((thiscol * 4 + 7) >> 4);
                        for (int x = 0; x < X; ++x) dst[(size_t)y * X + x] = row[x];
                    }
                }
            }
            for (int y = 0; y < Y; ++y)
                for (int x = 0; x < X; ++x)
                    ycc_to_rgb(plane_y[(size_t)y * yw + x], up_cb[(size_t)y * X + x], up_cr[(size_t)y * X + x],
                               rgb + ((int64_t)y * X + x) * 3);
            return 0;
        } else if (m == 0xD9) {
            return 1;  // EOI before a scan
        }
        // APPn, COM and anything else with a length: skipped
        p += 2 + L;
    }
    return 1;
}
