// oracle.cpp -- plain single-threaded CPU oracle of the per-tile nuclei pipeline.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h).  It is written from the paper's operation
// list (Table I; prose PAPER.md:208-217, 614-643) as made precise by
// SURVEY.md §8(c) and the readings listed in DESIGN.md.  Each function names the step it
// follows.  No blocking, fusion or reordering beyond the stated definitions/algorithms:
// this file is meant to be checked against the text by eye, not to be fast.
//
// Pins: every function is checked against what the paper and the mathematics fix
// (tests/test_oracle_*.py).  The Haralick features 26-33 follow our definitions (reading
// C16); they are pinned by closed forms on three hand-counted co-occurrence matrices
// (tests/test_oracle_pins_r2.py) besides an independent numpy recomputation, and the
// top-hat line of or_recon_to_nuclei by a hand-drawn plane with a known reconstruction.
#include "oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <vector>

namespace {

using clk = std::chrono::steady_clock;

inline bool inb(int x, int y, int w, int h) { return x >= 0 && y >= 0 && x < w && y < h; }

const int DX8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
const int DY8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
const int DX4[4] = {0, -1, 1, 0};
const int DY4[4] = {-1, 0, 0, 1};

// OpenCV MORPH_ELLIPSE (reading C7): row dy in [-r, r] covers dx in [-hw(dy), hw(dy)],
// hw(dy) = round(sqrt(r^2 - dy^2)) (cvRound of r*sqrt(1 - dy^2/r^2); no ties occur for
// integer r, dy).  For diam 19 this is [0,4,6,7,7,8,8,9,9,9,9,9,8,8,7,7,6,4,0] = 269 px.
std::vector<int> ellipse_half_widths(int diam) {
    int r = diam / 2;
    std::vector<int> hw(diam);
    for (int i = 0; i < diam; ++i) {
        int dy = i - r;
        hw[i] = (int)std::lround(std::sqrt((double)(r * r - dy * dy)));
    }
    return hw;
}

// Visit every component of the predicate graph 'same(p, q)' restricted to 'in(p)', in raster
// order of the component's first pixel (= min linear index), by BFS.  fn(list) is called per
// component with the list of its pixels (first element = min index).
template <class In, class Same, class Fn>
void for_each_component(int w, int h, int conn, In in, Same same, Fn fn) {
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> seen(n, 0);
    std::vector<int64_t> comp;
    const int* dx = conn == 8 ? DX8 : DX4;
    const int* dy = conn == 8 ? DY8 : DY4;
    for (int64_t s = 0; s < n; ++s) {
        if (seen[s] || !in(s)) continue;
        comp.clear();
        comp.push_back(s);
        seen[s] = 1;
        for (size_t k = 0; k < comp.size(); ++k) {
            int64_t p = comp[k];
            int x = (int)(p % w), y = (int)(p / w);
            for (int j = 0; j < conn; ++j) {
                int qx = x + dx[j], qy = y + dy[j];
                if (!inb(qx, qy, w, h)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (seen[q] || !in(q) || !same(p, q)) continue;
                seen[q] = 1;
                comp.push_back(q);
            }
        }
        fn(comp);
    }
}

// Vincent's hybrid grayscale reconstruction by dilation ("Vincent MR";
// L. Vincent, IEEE TIP 1993, Sec. V "hybrid algorithm"): raster scan over N+, anti-raster
// scan over N- with queue initialisation, then FIFO propagation.  8-connected.
// dom == nullptr means every pixel is in the domain; pixels outside it are neither read
// nor written (they do not belong to any neighbourhood).
template <class T>
void vincent_recon(const T* marker, const T* mask, const uint8_t* dom, int w, int h, T* R,
                   int64_t* stats) {
    const int64_t n = (int64_t)w * h;
    auto in = [&](int64_t p) { return dom == nullptr || dom[p] != 0; };
    for (int64_t p = 0; p < n; ++p) R[p] = in(p) ? std::min(marker[p], mask[p]) : T(0);
    // N+ = up-left, up, up-right, left ; N- = right, down-left, down, down-right
    const int PX[4] = {-1, 0, 1, -1}, PY[4] = {-1, -1, -1, 0};
    const int MX[4] = {1, -1, 0, 1}, MY[4] = {0, 1, 1, 1};
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            int64_t p = (int64_t)y * w + x;
            if (!in(p)) continue;
            T v = R[p];
            for (int j = 0; j < 4; ++j) {
                int qx = x + PX[j], qy = y + PY[j];
                if (!inb(qx, qy, w, h)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (in(q)) v = std::max(v, R[q]);
            }
            R[p] = std::min(v, mask[p]);
        }
    std::deque<int64_t> fifo;
    for (int y = h - 1; y >= 0; --y)
        for (int x = w - 1; x >= 0; --x) {
            int64_t p = (int64_t)y * w + x;
            if (!in(p)) continue;
            T v = R[p];
            for (int j = 0; j < 4; ++j) {
                int qx = x + MX[j], qy = y + MY[j];
                if (!inb(qx, qy, w, h)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (in(q)) v = std::max(v, R[q]);
            }
            R[p] = std::min(v, mask[p]);
            for (int j = 0; j < 4; ++j) {
                int qx = x + MX[j], qy = y + MY[j];
                if (!inb(qx, qy, w, h)) continue;
                int64_t q = (int64_t)qy * w + qx;
                if (in(q) && R[q] < R[p] && R[q] < mask[q]) {
                    fifo.push_back(p);
                    break;
                }
            }
        }
    int64_t init = (int64_t)fifo.size(), pops = 0;
    while (!fifo.empty()) {
        int64_t p = fifo.front();
        fifo.pop_front();
        ++pops;
        int x = (int)(p % w), y = (int)(p / w);
        for (int j = 0; j < 8; ++j) {
            int qx = x + DX8[j], qy = y + DY8[j];
            if (!inb(qx, qy, w, h)) continue;
            int64_t q = (int64_t)qy * w + qx;
            if (!in(q)) continue;
            if (R[q] < R[p] && mask[q] != R[q]) {
                R[q] = std::min(R[p], mask[q]);
                fifo.push_back(q);
            }
        }
    }
    if (stats) {
        stats[0] = init;
        stats[1] = pops;
    }
}

int reflect101(int i, int n) {
    if (n == 1) return 0;
    while (i < 0 || i >= n) {
        if (i < 0) i = -i;
        if (i >= n) i = 2 * n - 2 - i;
    }
    return i;
}

}  // namespace

extern "C" {

// Defaults (SURVEY.md §8(c) ledger C3, C5, C9, C10, C12, C19).  Q = M^-1 with M's rows the
// unit H, E and residual R = H x E vectors of Ruifrok & Johnston (reading C3), computed
// here in double and rounded once to float.
void or_default_params(or_params* p) {
    std::memset(p, 0, sizeof(*p));
    double H[3] = {0.650, 0.704, 0.286}, E[3] = {0.072, 0.990, 0.105}, R[3];
    auto norm = [](double* v) {
        double s = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        for (int i = 0; i < 3; ++i) v[i] /= s;
    };
    norm(H);
    norm(E);
    R[0] = H[1] * E[2] - H[2] * E[1];
    R[1] = H[2] * E[0] - H[0] * E[2];
    R[2] = H[0] * E[1] - H[1] * E[0];
    norm(R);
    double M[3][3] = {{H[0], H[1], H[2]}, {E[0], E[1], E[2]}, {R[0], R[1], R[2]}};
    // inverse by the adjugate
    double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) -
                 M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                 M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    double I[3][3];
    I[0][0] = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) / det;
    I[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) / det;
    I[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) / det;
    I[1][0] = (M[1][2] * M[2][0] - M[1][0] * M[2][2]) / det;
    I[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) / det;
    I[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) / det;
    I[2][0] = (M[1][0] * M[2][1] - M[1][1] * M[2][0]) / det;
    I[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) / det;
    I[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) / det;
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j) p->q[k][j] = (float)I[k][j];
    p->g_scale = 170.0f;
    p->bg_rgb_min = 220;
    p->bg_skip_frac = 2.0f;
    p->rbc_t1 = 5;
    p->rbc_t2 = 4;
    p->open_diam = 19;
    p->g1 = 50;
    p->cand_min_area = 11;
    p->cand_max_area = 1000;
    p->h = 1.0f;
    p->obj_min_area = 21;
    p->obj_max_area = 1000;
    p->glcm_levels = 8;
    p->canny_low = 100;   // reading C22
    p->canny_high = 200;
}

// S1 -- colour deconvolution + pixel thresholds used by RBC detection
// and background discard; readings C3, C5, C6.
int or_cd(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p, uint8_t* g,
          uint8_t* flags, int64_t* bg_count) {
    if (!rgb || !p || !g || !flags || w < 0 || h < 0 || pitch < 3LL * w) return 1;
    float od[256];
    for (int v = 0; v < 256; ++v) od[v] = (float)std::log10(256.0 / (v + 1.0));
    int64_t nbg = 0;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const uint8_t* px = rgb + (int64_t)y * pitch + 3 * x;
            int R = px[0], G = px[1], B = px[2];
            float cH = std::fma(od[B], p->q[2][0], std::fma(od[G], p->q[1][0], od[R] * p->q[0][0]));
            float s = std::rint(cH * p->g_scale);
            s = std::min(std::max(s, 0.0f), 255.0f);
            int64_t i = (int64_t)y * w + x;
            g[i] = (uint8_t)s;
            uint8_t f = 0;
            if (R > p->rbc_t1 * G) f |= OR_FLAG_RBC_HI;
            if (R > p->rbc_t2 * G) f |= OR_FLAG_RBC_LO;
            if (R > B) f |= OR_FLAG_R_GT_B;
            if (std::min(R, std::min(G, B)) > p->bg_rgb_min) {
                f |= OR_FLAG_BG;
                ++nbg;
            }
            flags[i] = f;
        }
    if (bg_count) *bg_count = nbg;
    return 0;
}

// S2 -- RBC detection ("OpenCV and Vincent MR"): binary reconstruction
// of the RBC_HI marker inside the RBC_LO mask (8-connected), intersected with R > B.
int or_rbc(const uint8_t* flags, int w, int h, uint8_t* rbc) {
    if (!flags || !rbc || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    std::memset(rbc, 0, n);
    for_each_component(
        w, h, 8, [&](int64_t p) { return (flags[p] & OR_FLAG_RBC_LO) != 0; },
        [](int64_t, int64_t) { return true; },
        [&](const std::vector<int64_t>& comp) {
            bool hit = false;
            for (int64_t p : comp) hit |= (flags[p] & OR_FLAG_RBC_HI) != 0;
            if (hit)
                for (int64_t p : comp) rbc[p] = 1;
        });
    for (int64_t p = 0; p < n; ++p)
        if (!(flags[p] & OR_FLAG_R_GT_B)) rbc[p] = 0;
    return 0;
}

// S3 -- erosion / dilation by the OpenCV ellipse, out-of-tile pixels ignored (reading C7):
// the plain definition min/max over {p + d : d in D, p + d in tile}.
static int morph(const uint8_t* g, int w, int h, int diam, uint8_t* out, bool is_min) {
    if (!g || !out || w < 0 || h < 0 || diam < 1 || diam % 2 == 0 || diam > 255) return 1;
    std::vector<int> hw = ellipse_half_widths(diam);
    int r = diam / 2;
    std::vector<uint8_t> acc((size_t)w);
    for (int y = 0; y < h; ++y) {
        std::fill(acc.begin(), acc.end(), is_min ? 255 : 0);
        // every offset d = (dx, dy) of D, applied to the whole output row
        for (int i = 0; i < diam; ++i) {
            int qy = y + i - r;
            if (qy < 0 || qy >= h) continue;
            const uint8_t* src = g + (int64_t)qy * w;
            for (int dx = -hw[i]; dx <= hw[i]; ++dx) {
                int x0 = std::max(0, -dx), x1 = std::min(w, w - dx);  // keep x + dx in tile
                if (is_min)
                    for (int x = x0; x < x1; ++x) acc[x] = std::min(acc[x], src[x + dx]);
                else
                    for (int x = x0; x < x1; ++x) acc[x] = std::max(acc[x], src[x + dx]);
            }
        }
        std::memcpy(out + (int64_t)y * w, acc.data(), (size_t)w);
    }
    return 0;
}
int or_erode(const uint8_t* g, int w, int h, int diam, uint8_t* out) { return morph(g, w, h, diam, out, true); }
int or_dilate(const uint8_t* g, int w, int h, int diam, uint8_t* out) { return morph(g, w, h, diam, out, false); }

// S3 -- Morph. Open with the 19x19 disk.
int or_open(const uint8_t* g, int w, int h, int diam, uint8_t* out) {
    if (!g || !out || w < 0 || h < 0) return 1;
    std::vector<uint8_t> tmp((size_t)w * h);
    int rc = or_erode(g, w, h, diam, tmp.data());
    if (rc) return rc;
    return or_dilate(tmp.data(), w, h, diam, out);
}

int or_recon_u8(const uint8_t* marker, const uint8_t* mask, int w, int h, uint8_t* out,
                int64_t* stats) {
    if (!marker || !mask || !out || w < 0 || h < 0) return 1;
    vincent_recon<uint8_t>(marker, mask, nullptr, w, h, out, stats);
    return 0;
}

int or_recon_f32(const float* marker, const float* mask, const uint8_t* dom, int w, int h,
                 float* out) {
    if (!marker || !mask || !out || w < 0 || h < 0) return 1;
    vincent_recon<float>(marker, mask, dom, w, h, out, nullptr);
    return 0;
}

// S4 -- ReconToNuclei: grayscale reconstruction of the opening
// under g, then the top-hat threshold g1 (reading C9), minus red blood cells.
int or_recon_to_nuclei(const uint8_t* g, const uint8_t* open, const uint8_t* rbc, int w, int h,
                       int g1, uint8_t* cand, uint8_t* recon_out) {
    if (!g || !open || !rbc || !cand || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> R(n);
    vincent_recon<uint8_t>(open, g, nullptr, w, h, R.data(), nullptr);
    for (int64_t p = 0; p < n; ++p)
        cand[p] = (((int)g[p] - (int)R[p]) > g1 && !rbc[p]) ? 1 : 0;
    if (recon_out) std::memcpy(recon_out, R.data(), n);
    return 0;
}

// Connected-component labelling (BWLabel; readings C8, C14): BFS in raster
// order; label = 1 + min linear index of the component.
int or_ccl(const uint8_t* fg, int w, int h, int conn, int32_t* labels, int32_t* n) {
    if (!fg || !labels || w < 0 || h < 0 || (conn != 4 && conn != 8)) return 1;
    const int64_t np = (int64_t)w * h;
    std::memset(labels, 0, np * sizeof(int32_t));
    int32_t count = 0;
    for_each_component(
        w, h, conn, [&](int64_t p) { return fg[p] != 0; }, [](int64_t, int64_t) { return true; },
        [&](const std::vector<int64_t>& comp) {
            int32_t lab = (int32_t)(comp[0] + 1);
            for (int64_t p : comp) labels[p] = lab;
            ++count;
        });
    if (n) *n = count;
    return 0;
}

// S5 -- AreaThreshold (reading C10).
int or_area_threshold(const uint8_t* cand, int w, int h, int amin, int amax, uint8_t* out) {
    if (!cand || !out || w < 0 || h < 0) return 1;
    std::memset(out, 0, (size_t)w * h);
    for_each_component(
        w, h, 8, [&](int64_t p) { return cand[p] != 0; }, [](int64_t, int64_t) { return true; },
        [&](const std::vector<int64_t>& comp) {
            int64_t a = (int64_t)comp.size();
            if (a >= amin && a <= amax)
                for (int64_t p : comp) out[p] = 1;
        });
    return 0;
}

// S6 -- FillHolles: a hole is a 4-connected component of the background
// that contains no tile-border pixel (reading C8).
int or_fill_holes(const uint8_t* big0, int w, int h, uint8_t* F) {
    if (!big0 || !F || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    for (int64_t p = 0; p < n; ++p) F[p] = big0[p] ? 1 : 0;
    for_each_component(
        w, h, 4, [&](int64_t p) { return big0[p] == 0; }, [](int64_t, int64_t) { return true; },
        [&](const std::vector<int64_t>& comp) {
            bool border = false;
            for (int64_t p : comp) {
                int x = (int)(p % w), y = (int)(p / w);
                if (x == 0 || y == 0 || x == w - 1 || y == h - 1) {
                    border = true;
                    break;
                }
            }
            if (!border)
                for (int64_t p : comp) F[p] = 1;
        });
    return 0;
}

// S7 -- Pre-Watershed distance transform (reading C11): exact squared
// Euclidean distance to the nearest in-tile background pixel, Meijster, Roerdink &
// Hesselink (2000), integer arithmetic throughout.
int or_edt(const uint8_t* F, int w, int h, uint32_t* d2, float* dist) {
    if (!F || !d2 || !dist || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    bool any_bg = false;
    for (int64_t p = 0; p < n && !any_bg; ++p) any_bg = F[p] == 0;
    if (!any_bg) {
        for (int64_t p = 0; p < n; ++p) {
            d2[p] = UINT32_MAX;
            dist[p] = std::numeric_limits<float>::infinity();
        }
        return 0;
    }
    const int64_t INF = (int64_t)w + h;  // Meijster's "m + n" infinity
    std::vector<int64_t> G(n);
    // phase 1: per column, distance to the nearest background pixel in that column
    for (int x = 0; x < w; ++x) {
        G[x] = F[x] ? INF : 0;
        for (int y = 1; y < h; ++y) {
            int64_t p = (int64_t)y * w + x;
            G[p] = F[p] ? std::min(INF, G[p - w] + 1) : 0;
        }
        for (int y = h - 2; y >= 0; --y) {
            int64_t p = (int64_t)y * w + x;
            if (G[p + w] < G[p]) G[p] = G[p + w] + 1;
        }
    }
    // phase 2: per row, lower envelope of the parabolas f(x, i) = (x - i)^2 + G(i)^2
    std::vector<int64_t> s(w), t(w);
    auto f = [](int64_t x, int64_t i, int64_t gi) { return (x - i) * (x - i) + gi * gi; };
    auto floordiv = [](int64_t a, int64_t b) {
        int64_t q = a / b;
        if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
        return q;
    };
    for (int y = 0; y < h; ++y) {
        const int64_t* g = &G[(int64_t)y * w];
        int64_t q = 0;
        s[0] = 0;
        t[0] = 0;
        for (int64_t u = 1; u < w; ++u) {
            while (q >= 0 && f(t[q], s[q], g[s[q]]) > f(t[q], u, g[u])) --q;
            if (q < 0) {
                q = 0;
                s[0] = u;
            } else {
                int64_t num = u * u - s[q] * s[q] + g[u] * g[u] - g[s[q]] * g[s[q]];
                int64_t wv = 1 + floordiv(num, 2 * (u - s[q]));
                if (wv < w) {
                    ++q;
                    s[q] = u;
                    t[q] = wv;
                }
            }
        }
        for (int64_t u = w - 1; u >= 0; --u) {
            int64_t p = (int64_t)y * w + u;
            int64_t v = f(u, s[q], g[s[q]]);
            d2[p] = (uint32_t)v;
            if (u == t[q]) --q;
        }
    }
    for (int64_t p = 0; p < n; ++p) {
        if (!F[p]) d2[p] = 0;
        dist[p] = std::sqrt((float)d2[p]);
    }
    return 0;
}

// S8 -- Pre-Watershed markers by MR (reading C12): h-maxima of the distance
// map (J = recon of dist - h under dist, inside F), regional maxima of J, canonical CCL.
int or_markers(const float* dist, const uint8_t* F, int w, int h, float hh, int32_t* ML,
               float* Jout, int32_t* n_markers) {
    if (!dist || !F || !ML || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    std::vector<float> J0(n, 0.0f), J(n, 0.0f);
    for (int64_t p = 0; p < n; ++p)
        if (F[p]) J0[p] = dist[p] - hh;
    vincent_recon<float>(J0.data(), dist, F, w, h, J.data(), nullptr);
    // RMAX8: a flat zone (8-connected, equal J, inside F) is a regional maximum iff no
    // pixel of it has an N8 neighbour in F with a strictly larger J.
    std::vector<uint8_t> M(n, 0);
    for_each_component(
        w, h, 8, [&](int64_t p) { return F[p] != 0; },
        [&](int64_t p, int64_t q) { return J[p] == J[q]; },
        [&](const std::vector<int64_t>& comp) {
            bool is_max = true;
            for (int64_t p : comp) {
                int x = (int)(p % w), y = (int)(p / w);
                for (int j = 0; j < 8 && is_max; ++j) {
                    int qx = x + DX8[j], qy = y + DY8[j];
                    if (!inb(qx, qy, w, h)) continue;
                    int64_t q = (int64_t)qy * w + qx;
                    if (F[q] && J[q] > J[p]) is_max = false;
                }
                if (!is_max) break;
            }
            if (is_max)
                for (int64_t p : comp) M[p] = 1;
        });
    int32_t nm = 0;
    or_ccl(M.data(), w, h, 8, ML, &nm);
    if (n_markers) *n_markers = nm;
    if (Jout)
        for (int64_t p = 0; p < n; ++p) Jout[p] = F[p] ? J[p] : 0.0f;
    return 0;
}

// S9 -- Watershed (reading C13): the order-independent
// definition W1 (maximin flooding level), W2 (plateau distance), W3 (min label over the
// steepest-ascent parents), then watershed lines on the larger-label side.
int or_watershed(const float* dist, const int32_t* ML, const uint8_t* F, int w, int h,
                 float* c_out, int32_t* d_out, int32_t* L_out, uint8_t* split) {
    if (!dist || !ML || !F || !split || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    const float NEG = -std::numeric_limits<float>::infinity();
    // W1: c = GrayRecon8(marker = dist on markers else -inf, mask = dist), inside F
    std::vector<float> c0(n, NEG), c(n, 0.0f);
    for (int64_t p = 0; p < n; ++p)
        if (F[p] && ML[p] != 0) c0[p] = dist[p];
    vincent_recon<float>(c0.data(), dist, F, w, h, c.data(), nullptr);
    // W2: d = 0 on markers; 1 if a neighbour in F has larger c; else 1 + min d over
    // equal-c neighbours.  Least fixed point = BFS by levels.
    const int32_t DINF = std::numeric_limits<int32_t>::max();
    std::vector<int32_t> d(n, DINF);
    std::vector<uint8_t> fixed(n, 0);
    std::deque<int64_t> bfs;
    for (int64_t p = 0; p < n; ++p)
        if (F[p] && ML[p] != 0) {
            d[p] = 0;
            fixed[p] = 1;
            bfs.push_back(p);
        }
    for (int64_t p = 0; p < n; ++p) {
        if (!F[p] || fixed[p]) continue;
        int x = (int)(p % w), y = (int)(p / w);
        for (int j = 0; j < 8; ++j) {
            int qx = x + DX8[j], qy = y + DY8[j];
            if (!inb(qx, qy, w, h)) continue;
            int64_t q = (int64_t)qy * w + qx;
            if (F[q] && c[q] > c[p]) {
                d[p] = 1;
                fixed[p] = 1;
                bfs.push_back(p);
                break;
            }
        }
    }
    while (!bfs.empty()) {
        int64_t q = bfs.front();
        bfs.pop_front();
        int x = (int)(q % w), y = (int)(q / w);
        for (int j = 0; j < 8; ++j) {
            int px = x + DX8[j], py = y + DY8[j];
            if (!inb(px, py, w, h)) continue;
            int64_t p = (int64_t)py * w + px;
            if (!F[p] || fixed[p] || c[p] != c[q]) continue;
            fixed[p] = 1;
            d[p] = d[q] + 1;
            bfs.push_back(p);
        }
    }
    // W3: process F pixels in increasing (-c, d) order; parents precede children.
    const int32_t LINF = std::numeric_limits<int32_t>::max();
    std::vector<int32_t> L(n, 0);
    std::vector<int64_t> order;
    for (int64_t p = 0; p < n; ++p)
        if (F[p]) order.push_back(p);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        if (c[a] != c[b]) return c[a] > c[b];
        return d[a] < d[b];
    });
    for (int64_t p : order) {
        if (ML[p] != 0) {
            L[p] = ML[p];
            continue;
        }
        int x = (int)(p % w), y = (int)(p / w);
        bool have = false;
        float bc = 0.0f;
        int32_t bd = 0, lab = LINF;
        for (int j = 0; j < 8; ++j) {
            int qx = x + DX8[j], qy = y + DY8[j];
            if (!inb(qx, qy, w, h)) continue;
            int64_t q = (int64_t)qy * w + qx;
            if (!F[q] || !(c[q] >= c[p])) continue;
            if (!have || c[q] > bc || (c[q] == bc && d[q] < bd)) {
                have = true;
                bc = c[q];
                bd = d[q];
                lab = L[q];
            } else if (c[q] == bc && d[q] == bd) {
                lab = std::min(lab, L[q]);
            }
        }
        L[p] = have ? lab : LINF;
    }
    // lines on the larger-label side; split = F minus lines
    for (int64_t p = 0; p < n; ++p) {
        split[p] = 0;
        if (!F[p]) continue;
        int x = (int)(p % w), y = (int)(p / w);
        bool line = false;
        for (int j = 0; j < 8 && !line; ++j) {
            int qx = x + DX8[j], qy = y + DY8[j];
            if (!inb(qx, qy, w, h)) continue;
            int64_t q = (int64_t)qy * w + qx;
            if (F[q] && L[q] < L[p]) line = true;
        }
        split[p] = line ? 0 : 1;
    }
    if (c_out)
        for (int64_t p = 0; p < n; ++p) c_out[p] = F[p] ? c[p] : 0.0f;
    if (d_out)
        for (int64_t p = 0; p < n; ++p) d_out[p] = F[p] ? d[p] : 0;
    if (L_out)
        for (int64_t p = 0; p < n; ++p) L_out[p] = F[p] ? L[p] : 0;
    return 0;
}

// S10 -- BWLabel + final size filter (readings C10, C14).
int or_bwlabel(const uint8_t* split, int w, int h, int amin, int amax, int32_t* labels,
               int32_t* n_objects) {
    if (!split || !labels || w < 0 || h < 0) return 1;
    std::memset(labels, 0, (size_t)w * h * sizeof(int32_t));
    int32_t count = 0;
    for_each_component(
        w, h, 8, [&](int64_t p) { return split[p] != 0; }, [](int64_t, int64_t) { return true; },
        [&](const std::vector<int64_t>& comp) {
            int64_t a = (int64_t)comp.size();
            if (a < amin || a > amax) return;
            int32_t lab = (int32_t)(comp[0] + 1);
            for (int64_t p : comp) labels[p] = lab;
            ++count;
        });
    if (n_objects) *n_objects = count;
    return 0;
}

// Feature-stage Canny ("OpenCV(Canny)"; reading C22): cv2.Canny(g, low,
// high) with aperture 3 and the L1 gradient norm, written out step by step:
//   dx, dy = 3x3 Sobel of g with replicated borders; m = |dx| + |dy|;
//   non-maximum suppression along the gradient direction, the sector chosen with
//   tan(22.5 deg) in 15-bit fixed point (TG22 = 13573), out-of-tile magnitudes 0:
//     horizontal  m > m(x-1, y) and m >= m(x+1, y)
//     vertical    m > m(x, y-1) and m >= m(x, y+1)
//     diagonal    s = sign(dx * dy): m > m(x-s, y-1) and m > m(x+s, y+1);
//   candidates = local maxima with m > low; edges = the 8-connected components of the
//   candidates that contain a candidate with m > high (hysteresis, BFS).
int or_canny(const uint8_t* g, int w, int h, int low, int high, uint8_t* edges) {
    if (!g || !edges || w < 0 || h < 0) return 1;
    const int64_t n = (int64_t)w * h;
    std::vector<int32_t> dx(n), dy(n), mag(n);
    auto G = [&](int x, int y) {
        x = std::min(std::max(x, 0), w - 1);
        y = std::min(std::max(y, 0), h - 1);
        return (int32_t)g[(int64_t)y * w + x];
    };
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int64_t p = (int64_t)y * w + x;
            dx[p] = (G(x + 1, y - 1) + 2 * G(x + 1, y) + G(x + 1, y + 1)) -
                    (G(x - 1, y - 1) + 2 * G(x - 1, y) + G(x - 1, y + 1));
            dy[p] = (G(x - 1, y + 1) + 2 * G(x, y + 1) + G(x + 1, y + 1)) -
                    (G(x - 1, y - 1) + 2 * G(x, y - 1) + G(x + 1, y - 1));
            mag[p] = std::abs(dx[p]) + std::abs(dy[p]);
        }
    auto M = [&](int x, int y) -> int32_t { return inb(x, y, w, h) ? mag[(int64_t)y * w + x] : 0; };
    const int64_t TG22 = 13573;  // (int)(tan(22.5 deg) * 2^15 + 0.5)
    std::vector<uint8_t> cand(n, 0);
    std::deque<int64_t> fifo;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            const int64_t p = (int64_t)y * w + x;
            const int32_t m = mag[p];
            if (m <= low) continue;
            const int64_t ax = std::abs(dx[p]), ay = (int64_t)std::abs(dy[p]) << 15;
            const int64_t tg22x = ax * TG22, tg67x = tg22x + (ax << 16);
            bool lm;
            if (ay < tg22x) {
                lm = m > M(x - 1, y) && m >= M(x + 1, y);
            } else if (ay > tg67x) {
                lm = m > M(x, y - 1) && m >= M(x, y + 1);
            } else {
                const int s = ((dx[p] ^ dy[p]) < 0) ? -1 : 1;
                lm = m > M(x - s, y - 1) && m > M(x + s, y + 1);
            }
            if (!lm) continue;
            cand[p] = 1;
            if (m > high) fifo.push_back(p);
        }
    std::memset(edges, 0, (size_t)n);
    for (int64_t p : fifo) edges[p] = 1;
    while (!fifo.empty()) {
        const int64_t p = fifo.front();
        fifo.pop_front();
        const int x = (int)(p % w), y = (int)(p / w);
        for (int j = 0; j < 8; ++j) {
            const int qx = x + DX8[j], qy = y + DY8[j];
            if (!inb(qx, qy, w, h)) continue;
            const int64_t q = (int64_t)qy * w + qx;
            if (cand[q] && !edges[q]) {
                edges[q] = 1;
                fifo.push_back(q);
            }
        }
    }
    return 0;
}

// S11 -- Features comp. (reading C16, C17, C22).
// Feature order: see DESIGN.md "Feature table".
int or_features(const int32_t* labels, const uint8_t* g, int w, int h, int glcm_levels,
                int canny_low, int canny_high, int32_t cap, int32_t* row_label,
                int32_t* row_flags, float* feat, int32_t* n_rows) {
    if (!labels || !g || w < 0 || h < 0 || glcm_levels != 8 || cap < 0 || canny_low < 0 ||
        canny_high < canny_low)
        return 1;
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> edges(n);
    or_canny(g, w, h, canny_low, canny_high, edges.data());
    std::map<int32_t, std::vector<int64_t>> objs;  // ascending label order
    for (int64_t p = 0; p < n; ++p)
        if (labels[p] > 0) objs[labels[p]].push_back(p);
    int32_t nobj = (int32_t)objs.size();
    if (n_rows) *n_rows = nobj;
    if (nobj > cap) return 4;
    auto at = [&](int x, int y) { return (int)g[(int64_t)reflect101(y, h) * w + reflect101(x, w)]; };
    const double PI = 3.14159265358979323846;
    int32_t row = 0;
    for (auto& kv : objs) {
        const int32_t lab = kv.first;
        const std::vector<int64_t>& P = kv.second;
        auto inP = [&](int x, int y) { return inb(x, y, w, h) && labels[(int64_t)y * w + x] == lab; };
        const int64_t A = (int64_t)P.size();
        double out[OR_NFEAT];
        // ---- shape (13)
        int64_t sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0, perim = 0;
        int xmin = w, xmax = -1, ymin = h, ymax = -1;
        bool border = false;
        for (int64_t p : P) {
            int x = (int)(p % w), y = (int)(p / w);
            sx += x;
            sy += y;
            sxx += (int64_t)x * x;
            syy += (int64_t)y * y;
            sxy += (int64_t)x * y;
            xmin = std::min(xmin, x);
            xmax = std::max(xmax, x);
            ymin = std::min(ymin, y);
            ymax = std::max(ymax, y);
            if (x == 0 || y == 0 || x == w - 1 || y == h - 1) border = true;
            bool edge = false;
            for (int j = 0; j < 4; ++j)
                if (!inP(x + DX4[j], y + DY4[j])) edge = true;
            if (edge) ++perim;
        }
        double Ad = (double)A;
        double cx = (double)sx / Ad, cy = (double)sy / Ad;
        double bw = xmax - xmin + 1, bh = ymax - ymin + 1;
        double mu20 = (double)(A * sxx - sx * sx) / Ad;  // sum of (x - cx)^2
        double mu02 = (double)(A * syy - sy * sy) / Ad;
        double mu11 = (double)(A * sxy - sx * sy) / Ad;
        double a = mu20 / Ad + 1.0 / 12.0, b = mu11 / Ad, cc = mu02 / Ad + 1.0 / 12.0;
        double tr = 0.5 * (a + cc), disc = std::sqrt(0.25 * (a - cc) * (a - cc) + b * b);
        double l1 = tr + disc, l2 = tr - disc;
        if (l2 < 0) l2 = 0;
        out[0] = Ad;
        out[1] = (double)perim;
        out[2] = cx;
        out[3] = cy;
        out[4] = bw;
        out[5] = bh;
        out[6] = 4.0 * std::sqrt(l1);
        out[7] = 4.0 * std::sqrt(l2);
        out[8] = std::sqrt(1.0 - l2 / l1);
        out[9] = 0.5 * std::atan2(2.0 * mu11, mu20 - mu02);
        out[10] = std::sqrt(4.0 * Ad / PI);
        out[11] = 4.0 * PI * Ad / ((double)perim * (double)perim);
        out[12] = Ad / (bw * bh);
        // ---- intensity on g (9), from the 256-bin histogram
        int64_t hist[256] = {0};
        for (int64_t p : P) hist[g[p]]++;
        int64_t s1 = 0;
        int vmin = 255, vmax = 0;
        for (int v = 0; v < 256; ++v)
            if (hist[v]) {
                s1 += hist[v] * v;
                vmin = std::min(vmin, v);
                vmax = std::max(vmax, v);
            }
        double mean = (double)s1 / Ad;
        double m2 = 0, m3 = 0, m4 = 0, ent = 0, en = 0;
        for (int v = 0; v < 256; ++v) {
            if (!hist[v]) continue;
            double dv = v - mean, hv = (double)hist[v];
            m2 += hv * dv * dv;
            m3 += hv * dv * dv * dv;
            m4 += hv * dv * dv * dv * dv;
            double pv = hv / Ad;
            ent -= pv * std::log2(pv);
            en += pv * pv;
        }
        m2 /= Ad;
        m3 /= Ad;
        m4 /= Ad;
        int64_t half = (A + 1) / 2, cum = 0;
        int med = 0;
        for (int v = 0; v < 256; ++v) {
            cum += hist[v];
            if (cum >= half) {
                med = v;
                break;
            }
        }
        bool flat = vmin == vmax;
        out[13] = mean;
        out[14] = flat ? 0.0 : std::sqrt(m2);
        out[15] = vmin;
        out[16] = vmax;
        out[17] = med;
        out[18] = flat ? 0.0 : m3 / (m2 * std::sqrt(m2));
        out[19] = flat ? 0.0 : m4 / (m2 * m2);
        out[20] = ent;
        out[21] = en;
        // ---- gradient magnitude (4): 3x3 Sobel on g, REFLECT_101 at the tile edge
        std::vector<float> mags;
        mags.reserve(P.size());
        float gmin = std::numeric_limits<float>::infinity(), gmax = -gmin;
        for (int64_t p : P) {
            int x = (int)(p % w), y = (int)(p / w);
            int gx = (at(x + 1, y - 1) + 2 * at(x + 1, y) + at(x + 1, y + 1)) -
                     (at(x - 1, y - 1) + 2 * at(x - 1, y) + at(x - 1, y + 1));
            int gy = (at(x - 1, y + 1) + 2 * at(x, y + 1) + at(x + 1, y + 1)) -
                     (at(x - 1, y - 1) + 2 * at(x, y - 1) + at(x + 1, y - 1));
            float m = std::sqrt((float)(gx * gx + gy * gy));
            mags.push_back(m);
            gmin = std::min(gmin, m);
            gmax = std::max(gmax, m);
        }
        double gs = 0;
        for (float m : mags) gs += (double)m;
        double gmean = gs / Ad, g2 = 0, g3 = 0, g4 = 0;
        for (float m : mags) {
            double dv = (double)m - gmean;
            g2 += dv * dv;
            g3 += dv * dv * dv;
            g4 += dv * dv * dv * dv;
        }
        g2 /= Ad;
        g3 /= Ad;
        g4 /= Ad;
        bool gflat = gmin == gmax;
        out[22] = gmean;
        out[23] = gflat ? 0.0 : std::sqrt(g2);
        out[24] = gflat ? 0.0 : g3 / (g2 * std::sqrt(g2));
        out[25] = gflat ? 0.0 : g4 / (g2 * g2);
        // ---- GLCM / Haralick (8): q = g >> 5, offsets (1,0),(1,1),(0,1),(-1,1), symmetric
        int64_t C[8][8] = {{0}};
        const int OX[4] = {1, 1, 0, -1}, OY[4] = {0, 1, 1, 1};
        for (int64_t p : P) {
            int x = (int)(p % w), y = (int)(p / w);
            for (int o = 0; o < 4; ++o) {
                int qx = x + OX[o], qy = y + OY[o];
                if (!inP(qx, qy)) continue;
                int i = g[p] >> 5, j = g[(int64_t)qy * w + qx] >> 5;
                C[i][j]++;
                C[j][i]++;
            }
        }
        int64_t S = 0;
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) S += C[i][j];
        if (S == 0) {
            for (int k = 26; k < 34; ++k) out[k] = 0.0;
        } else {
            double Pm[8][8];
            double mui = 0, muj = 0;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    Pm[i][j] = (double)C[i][j] / (double)S;
                    mui += i * Pm[i][j];
                    muj += j * Pm[i][j];
                }
            double si = 0, sj = 0;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    si += (i - mui) * (i - mui) * Pm[i][j];
                    sj += (j - muj) * (j - muj) * Pm[i][j];
                }
            si = std::sqrt(si);
            sj = std::sqrt(sj);
            double asm_ = 0, con = 0, cor = 0, hom = 0, gent = 0, shade = 0, prom = 0, pmax = 0;
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    double pij = Pm[i][j];
                    asm_ += pij * pij;
                    con += (double)((i - j) * (i - j)) * pij;
                    cor += (i - mui) * (j - muj) * pij;
                    hom += pij / (1.0 + (double)((i - j) * (i - j)));
                    if (pij > 0) gent -= pij * std::log2(pij);
                    double t = i + j - mui - muj;
                    shade += t * t * t * pij;
                    prom += t * t * t * t * pij;
                    pmax = std::max(pmax, pij);
                }
            out[26] = asm_;
            out[27] = con;
            out[28] = (si * sj == 0.0) ? 1.0 : cor / (si * sj);
            out[29] = hom;
            out[30] = gent;
            out[31] = shade;
            out[32] = prom;
            out[33] = pmax;
        }
        // ---- edge (2): Canny edge pixels of the object, and their fraction of its area
        int64_t ne = 0;
        for (int64_t p : P) ne += edges[p];
        out[34] = (double)ne;
        out[35] = (double)ne / Ad;
        if (row_label) row_label[row] = lab;
        if (row_flags) row_flags[row] = border ? OR_OBJ_TOUCHES_BORDER : 0;
        if (feat)
            for (int k = 0; k < OR_NFEAT; ++k) feat[(int64_t)row * OR_NFEAT + k] = (float)out[k];
        ++row;
    }
    return 0;
}

static double secs(clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

// S1..S10 in Table I order (reading C1), colour deconvolution hoisted to S1 (reading C4).
int or_segment_tile(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p,
                    int32_t* labels, int32_t* n_objects, double* t) {
    if (!rgb || !p || !labels || w <= 0 || h <= 0 || pitch < 3LL * w) return 1;
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> g(n), flags(n), rbc(n), open(n), cand(n), big0(n), F(n), split(n);
    std::vector<uint32_t> d2(n);
    std::vector<float> dist(n);
    std::vector<int32_t> ML(n);
    double tt[11] = {0};
    int64_t nbg = 0;
    auto t0 = clk::now();
    or_cd(rgb, w, h, pitch, p, g.data(), flags.data(), &nbg);
    auto t1 = clk::now();
    tt[0] = secs(t0, t1);
    if (p->bg_skip_frac <= 1.0f && (double)nbg >= (double)p->bg_skip_frac * (double)n) {
        std::memset(labels, 0, n * sizeof(int32_t));
        if (n_objects) *n_objects = 0;
        if (t) std::memcpy(t, tt, sizeof(tt));
        return 0;
    }
    or_rbc(flags.data(), w, h, rbc.data());
    auto t2 = clk::now();
    or_open(g.data(), w, h, p->open_diam, open.data());
    auto t3 = clk::now();
    or_recon_to_nuclei(g.data(), open.data(), rbc.data(), w, h, p->g1, cand.data(), nullptr);
    auto t4 = clk::now();
    or_area_threshold(cand.data(), w, h, p->cand_min_area, p->cand_max_area, big0.data());
    auto t5 = clk::now();
    or_fill_holes(big0.data(), w, h, F.data());
    auto t6 = clk::now();
    or_edt(F.data(), w, h, d2.data(), dist.data());
    auto t7 = clk::now();
    or_markers(dist.data(), F.data(), w, h, p->h, ML.data(), nullptr, nullptr);
    auto t8 = clk::now();
    or_watershed(dist.data(), ML.data(), F.data(), w, h, nullptr, nullptr, nullptr, split.data());
    auto t9 = clk::now();
    or_bwlabel(split.data(), w, h, p->obj_min_area, p->obj_max_area, labels, n_objects);
    auto t10 = clk::now();
    tt[1] = secs(t1, t2);
    tt[2] = secs(t2, t3);
    tt[3] = secs(t3, t4);
    tt[4] = secs(t4, t5);
    tt[5] = secs(t5, t6);
    tt[6] = secs(t6, t7);
    tt[7] = secs(t7, t8);
    tt[8] = secs(t8, t9);
    tt[9] = secs(t9, t10);
    if (t) std::memcpy(t, tt, sizeof(tt));
    return 0;
}

int or_process_tile(const uint8_t* rgb, int w, int h, int64_t pitch, const or_params* p,
                    int32_t* labels, int32_t cap, int32_t* row_label, int32_t* row_flags,
                    float* feat, int32_t* n_rows, double* t) {
    int32_t nobj = 0;
    int rc = or_segment_tile(rgb, w, h, pitch, p, labels, &nobj, t);
    if (rc) return rc;
    const int64_t n = (int64_t)w * h;
    std::vector<uint8_t> g(n), flags(n);
    auto a = clk::now();
    or_cd(rgb, w, h, pitch, p, g.data(), flags.data(), nullptr);
    rc = or_features(labels, g.data(), w, h, p->glcm_levels, p->canny_low, p->canny_high, cap, row_label,
                     row_flags, feat, n_rows);
    auto b = clk::now();
    if (t) t[10] = secs(a, b);
    return rc;
}

}  // extern "C"

// ---------------------------------------------------------------- NEXT-4 aggregation
// Per-image feature aggregation ("the features
// computed for each object ... are aggregated" per image/patient for the classification
// stage).  For each group g, rows [off[g], off[g+1]) of feat ([n][nfeat] f32): count, the
// mean of every feature, and the population standard deviation sqrt(sum (x - mean)^2 / n),
// both in fp64, by the plain two-pass definition.  An empty group gives NaN mean and std.
int or_aggregate(const float* feat, int nfeat, const int64_t* off, int n_groups, int64_t* count,
                 double* mean, double* stdv) {
    if (nfeat < 1 || n_groups < 0 || !off || !count || !mean || !stdv) return 1;
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (int g = 0; g < n_groups; ++g) {
        const int64_t r0 = off[g], r1 = off[g + 1];
        if (r1 < r0) return 1;
        count[g] = r1 - r0;
        for (int f = 0; f < nfeat; ++f) {
            if (r1 == r0) {
                mean[(int64_t)g * nfeat + f] = nan;
                stdv[(int64_t)g * nfeat + f] = nan;
                continue;
            }
            double s = 0.0;
            for (int64_t r = r0; r < r1; ++r) s += (double)feat[r * nfeat + f];
            const double m = s / (double)(r1 - r0);
            double q = 0.0;
            for (int64_t r = r0; r < r1; ++r) {
                const double d = (double)feat[r * nfeat + f] - m;
                q += d * d;
            }
            mean[(int64_t)g * nfeat + f] = m;
            stdv[(int64_t)g * nfeat + f] = std::sqrt(q / (double)(r1 - r0));
        }
    }
    return 0;
}
