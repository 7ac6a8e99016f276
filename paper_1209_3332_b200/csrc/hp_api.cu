// hp_api.cu -- the C ABI of include/hp.h: context, scratch arena, stage sequencing
// (Table I order; reading C1), per-stage verification entry, and the
// demand-driven multi-tile driver with per-slot upload/process/download streams
// (PAPER.md:370-389 window, 550-571 prefetch and asynchronous copy).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <atomic>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <thread>
#include <chrono>

#include "hp_internal.cuh"

namespace hp {
void launch_zero_outside_f32(const float* src, const uint8_t* F, int64_t n, float* dst, cudaStream_t s);
void launch_recon_init_f32(const float* marker, const float* mask, const uint8_t* dom, int64_t n, float* R,
                           cudaStream_t s);
}

namespace hp {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static PerDevice g_sms;
int num_sms() {
    return g_sms.get([] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
        return n;
    });
}
}  // namespace hp

using namespace hp;

struct hp_ctx {
    hp_config cfg;
    int device = 0;
    bool poisoned = false;
    bool timing = false;
    std::string err;
    float* lut = nullptr;
    std::vector<Slot> slots;
    std::vector<void*> dev_blocks;
    std::vector<void*> host_blocks;
    int rows_copied = 0;  // rows copied back per tile in hp_run_tiles
    bool global_s8s10 = false;
    int prio = 0;  // env HP_PRIO: 1 = S4 on a high-priority stream, 2 = S4 and S7-S11
    bool graphs = true;  // env HP_GRAPHS=0: hp_run_tiles launches every op instead of a graph  // env HP_GLOBAL_S8S10=1: the per-stage global path in the pipeline
    // stage-timing ring: per slot, kRing sets of 12 events (one set per tile)
    std::vector<std::vector<std::array<cudaEvent_t, 12>>> ring;
    std::vector<int> ring_pos, ring_n;
};

namespace {

constexpr int kAbiVersion = 2;
constexpr int kRowsAsync = 4096;
constexpr int kRing = 256;

void set_err(hp_ctx* ctx, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
}

hp_status cuda_fail(hp_ctx* ctx, cudaError_t e, const char* where) {
    set_err(ctx, "%s: %s", where, cudaGetErrorString(e));
    ctx->poisoned = true;
    return HP_ERR_CUDA;
}

hp_status check_launch(hp_ctx* ctx, const char* where) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, where);
    return HP_OK;
}

bool params_ok(const hp_params& p, std::string* why) {
    auto bad = [&](const char* m) { *why = m; return false; };
    for (int k = 0; k < 3; ++k)
        for (int j = 0; j < 3; ++j)
            if (!std::isfinite(p.q[k][j])) return bad("q must be finite");
    if (!(p.g_scale > 0.0f) || !std::isfinite(p.g_scale)) return bad("g_scale must be > 0");
    if (p.bg_rgb_min < -1 || p.bg_rgb_min > 255) return bad("bg_rgb_min out of [-1, 255]");
    if (!(p.bg_skip_frac >= 0.0f)) return bad("bg_skip_frac must be >= 0");
    if (p.rbc_t1 < 0 || p.rbc_t2 < 0 || p.rbc_t1 > 255 || p.rbc_t2 > 255) return bad("rbc_t1/t2 out of [0, 255]");
    if (p.open_diam < 1 || p.open_diam > 63 || p.open_diam % 2 == 0) return bad("open_diam must be odd in [1, 63]");
    if (p.g1 < -256 || p.g1 > 255) return bad("g1 out of range");
    if (p.cand_min_area < 0 || p.cand_min_area > p.cand_max_area) return bad("cand area bounds");
    if (p.obj_min_area < 0 || p.obj_min_area > p.obj_max_area) return bad("obj area bounds");
    // S11's exact moments A*sum(x^2) - (sum x)^2 stay inside int64 for A <= 2^17 on tiles up to
    // 16384 px wide (2^17 * 2^17 * 2^28 = 2^62)
    if (p.cand_max_area > (1 << 17) || p.obj_max_area > (1 << 17)) return bad("area bounds above 131072");
    if (!(p.h > 0.0f) || !std::isfinite(p.h)) return bad("h must be finite and > 0");
    if (p.glcm_levels != 8) return bad("glcm_levels must be 8");
    if (p.canny_low < 0 || p.canny_high < p.canny_low) return bad("need 0 <= canny_low <= canny_high");
    return true;
}

hp_status enter(hp_ctx* ctx, int32_t slot) {
    if (!ctx) return HP_ERR_INVALID;
    if (ctx->poisoned) return HP_ERR_CUDA;
    if (slot < 0 || slot >= ctx->cfg.n_slots) {
        set_err(ctx, "slot %d out of [0, %d)", slot, ctx->cfg.n_slots);
        return HP_ERR_INVALID;
    }
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    return HP_OK;
}

hp_status check_image(hp_ctx* ctx, const hp_image* im) {
    if (!im || !im->data) { set_err(ctx, "null image"); return HP_ERR_INVALID; }
    if (im->width < 1 || im->height < 1 || im->width > ctx->cfg.max_width || im->height > ctx->cfg.max_height) {
        set_err(ctx, "image %dx%d outside [1, %d] x [1, %d]", im->width, im->height, ctx->cfg.max_width, ctx->cfg.max_height);
        return HP_ERR_INVALID;
    }
    if (im->pitch_bytes < 3LL * im->width) { set_err(ctx, "pitch < 3*width"); return HP_ERR_INVALID; }
    return HP_OK;
}

int slot_index(hp_ctx* ctx, Slot& sl) { return (int)(&sl - ctx->slots.data()); }

void ev(hp_ctx* ctx, Slot& sl, int k, cudaStream_t s) {
    if (!ctx->timing) return;
    int i = slot_index(ctx, sl);
    if (k == 0) {
        ctx->ring_pos[i] = (ctx->ring_pos[i] + 1) % kRing;
        ctx->ring_n[i] = std::min(ctx->ring_n[i] + 1, kRing);
    }
    cudaEventRecord(ctx->ring[i][ctx->ring_pos[i]][k], s);
}

// S1..S10 on device buffers (the segmentation stage instance)
// S1..S10; with `table` the fused per-component path also computes S11 into it and *fused
// is set (the caller then skips the separate feature stage)
// Experiment only (variant builds, -DHP_WHATIF_DUP=k): run step k twice per tile to measure
// its marginal cost in the concurrent bench (1 S1, 2 S2, 3 S3, 5 S5, 6 S6, 8 Canny, 9 S7-S11).
// Every duplicated launcher resets its own outputs, so the results are unchanged.
#ifndef HP_WHATIF_DUP
#define HP_WHATIF_DUP 0
#endif
#define HP_DUP(k) for (int dup_ = 0; dup_ < (HP_WHATIF_DUP == (k) ? 2 : 1); ++dup_)

// With jpeg set, S1 reads the slot's JPEG tile (header in sl.jhdr_dev, file in sl.rgb_dev,
// both uploaded by the caller) and decodes it inside S1 (k_jpeg.cu); rgb gives only the size.
hp_status segment(hp_ctx* ctx, Slot& sl, const hp_image* rgb, int32_t* labels, int64_t lpitch,
                  int32_t* n_objects, cudaStream_t s, hp_feature_table* table = nullptr,
                  bool* fused = nullptr, int jpeg = 0) {
    if (fused) *fused = false;
    const hp_params& p = ctx->cfg.params;
    const int w = rgb->width, h = rgb->height;
    ev(ctx, sl, 0, s);
    if (jpeg) {                                                                                       // S0 + S1
        cudaMemsetAsync(sl.jerr, 0, sizeof(int32_t), s);
        const int64_t cap = 3LL * ctx->cfg.max_width * ctx->cfg.max_height;
        launch_jpeg_decode(sl.jhdr_dev, jpeg, sl.rgb_dev, cap, w, h, sl.jstarts, sl.jblk, sl.jplanes, ctx->lut, p,
                           sl.g, sl.flags, &sl.counters[0], nullptr, 0, sl.jerr, s);
    } else {
        HP_DUP(1) launch_cd(rgb->data, w, h, rgb->pitch_bytes, ctx->lut, p, sl.g, sl.flags, &sl.counters[0], s);  // S1
    }
    ev(ctx, sl, 1, s);
    if (p.bg_skip_frac <= 1.0f) {
        unsigned long long nbg = 0;
        cudaMemcpyAsync(&nbg, &sl.counters[0], sizeof(nbg), cudaMemcpyDeviceToHost, s);
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "bg skip sync");
        if ((double)nbg >= (double)p.bg_skip_frac * (double)w * (double)h) {
            cudaMemset2DAsync(labels, lpitch * sizeof(int32_t), 0, w * sizeof(int32_t), h, s);
            cudaMemsetAsync(n_objects, 0, sizeof(int32_t), s);
            for (int k = 2; k <= 10; ++k) ev(ctx, sl, k, s);
            if (!table) ev(ctx, sl, 11, s);  // no feature stage follows: close the event set
            return check_launch(ctx, "bg skip");
        }
    }
    HP_DUP(2) launch_rbc(sl.flags, w, h, sl, sl.rbc, s);                                            // S2
    ev(ctx, sl, 2, s);
    // the opening is anti-extensive (symmetric SE containing the origin, out-of-tile pixels
    // ignored: open(g) <= g), so S4's marker min(open, g) is the opening itself
    HP_DUP(3) launch_open(sl.g, w, h, p.open_diam, sl.u8a, sl.u8b, s);                                // S3
    ev(ctx, sl, 3, s);
    {                                                                                                 // S4
        // optionally on the slot's high-priority stream: its CTAs then take SM resources
        // first as the other slots' blocks retire
        cudaStream_t rs = s;
        if (ctx->prio >= 1) {
            cudaEventRecord(sl.fork_ev, s);
            cudaStreamWaitEvent(sl.hstream, sl.fork_ev, 0);
            rs = sl.hstream;
        }
        launch_recon_u8_auto(sl.g, sl.u8b, w, h, sl.wl, rs);
#ifdef HP_WHATIF_S4X2  // experiment only: a second, independent S4 into scratch (marginal cost)
        cudaMemcpyAsync(sl.pmask, sl.u8a, (size_t)w * h, cudaMemcpyDeviceToDevice, rs);
        launch_open(sl.g, w, h, p.open_diam, sl.cand, sl.pmask, rs);
        launch_recon_u8_auto(sl.g, sl.pmask, w, h, sl.wl, rs);
#endif
        if (ctx->prio >= 1) {
            cudaEventRecord(sl.join_ev, sl.hstream);
            cudaStreamWaitEvent(s, sl.join_ev, 0);
        }
    }
    ev(ctx, sl, 4, s);
    // S5 on the top-hat candidates (g - recon > g1) & !rbc, evaluated inside the CCL passes
    int32_t* ncomp5 = sl.cnt32 + 16;  // S5 components kept (listed with root and bbox)
    HP_DUP(5) launch_area_select_tophat(sl.g, sl.u8b, sl.rbc, p.g1, w, h, p.cand_min_area, p.cand_max_area, sl, sl.big0,
                              ncomp5, s);
    ev(ctx, sl, 5, s);
    HP_DUP(6) launch_fill_components(sl.big0, w, h, sl, ncomp5, sl.F, sl.split, s);                 // S6
    ev(ctx, sl, 6, s);
    if (ctx->global_s8s10) {
        launch_edt(sl.F, w, h, sl, nullptr, sl.dist, s);                                             // S7
        ev(ctx, sl, 7, s);
        launch_markers(sl.dist, sl.F, p.h, w, h, sl, sl.ML, sl.J, s);                               // S8
        ev(ctx, sl, 8, s);
        launch_watershed(sl.dist, sl.ML, sl.F, w, h, sl, sl.split, nullptr, nullptr, nullptr, s);   // S9
        ev(ctx, sl, 9, s);
        launch_bwlabel(sl.split, w, h, p.obj_min_area, p.obj_max_area, sl, labels, lpitch, n_objects, s); // S10
        ev(ctx, sl, 10, s);
    } else {
        // S7-S11 fused per 8-component of F (k_comp.cu; timed under S8, S7/S9/S10 read 0)
        ev(ctx, sl, 7, s);
        cudaStream_t cs = s;
        if (ctx->prio >= 2) {
            cudaEventRecord(sl.fork_ev, s);
            cudaStreamWaitEvent(sl.hstream, sl.fork_ev, 0);
            cs = sl.hstream;
        }
        // the feature stage's Canny, only when features are produced
        if (table) HP_DUP(8) launch_canny(sl.g, w, h, p.canny_low, p.canny_high, sl, sl.cand, cs);
        HP_DUP(9) launch_components(ncomp5, sl.split, sl.g, sl.cand, p.h, p.obj_min_area, p.obj_max_area, w, h, sl, labels,
                          lpitch, n_objects, table, ctx->cfg.max_objects, cs);
        if (ctx->prio >= 2) {
            cudaEventRecord(sl.join_ev, sl.hstream);
            cudaStreamWaitEvent(s, sl.join_ev, 0);
        }
        ev(ctx, sl, 8, s);
        ev(ctx, sl, 9, s);
        ev(ctx, sl, 10, s);
        if (table && fused) {
            *fused = true;
            ev(ctx, sl, 11, s);
        }
    }
    // hp_segment_tile (no table): no feature stage follows, so S11's closing event is
    // recorded here -- hp_get_stage_times synchronises on it
    if (!table) ev(ctx, sl, 11, s);
    return check_launch(ctx, "segment");
}

hp_status features(hp_ctx* ctx, Slot& sl, int w, int h, const int32_t* labels, int64_t lpitch,
                   hp_feature_table* out, cudaStream_t s) {
    const hp_params& p = ctx->cfg.params;
    launch_canny(sl.g, w, h, p.canny_low, p.canny_high, sl, sl.cand, s);                             // S11
    launch_features(labels, lpitch, sl.g, sl.cand, w, h, sl, ctx->cfg.max_objects, out->label, out->flags,
                    out->feat, out->capacity, out->n_rows_dev, s);
    ev(ctx, sl, 11, s);
    return check_launch(ctx, "features");
}

hp_status check_table(hp_ctx* ctx, const hp_feature_table* t) {
    if (!t || !t->label || !t->flags || !t->feat || !t->n_rows_dev || t->capacity < 0) {
        set_err(ctx, "invalid feature table");
        return HP_ERR_INVALID;
    }
    return HP_OK;
}

hp_status check_labels(hp_ctx* ctx, const hp_labels* l, int w) {
    if (!l || !l->labels || !l->n_objects_dev || l->labels_pitch_elems < w) {
        set_err(ctx, "invalid labels");
        return HP_ERR_INVALID;
    }
    return HP_OK;
}

// NEXT-3: parse a JPEG tile on the host and upload the header and the file into the slot
// (stream s).  ring: stage the header in the slot's pinned ring (single-tile calls may be
// issued back to back on one slot) instead of its one run_tiles staging entry.
hp_status upload_jpeg(hp_ctx* ctx, Slot& sl, const uint8_t* host, int64_t nbytes, cudaStream_t s, bool ring,
                      int* w, int* h, int* sub) {
    const int64_t cap = 3LL * ctx->cfg.max_width * ctx->cfg.max_height;
    if (!host || nbytes < 4 || nbytes > cap) {
        set_err(ctx, "jpeg: null buffer or size %lld outside [4, %lld]", (long long)nbytes, (long long)cap);
        return HP_ERR_INVALID;
    }
    JpegHdr* H = sl.jhdr_host;
    int k = 0;
    if (ring) {
        k = sl.jhdr_pos;
        cudaError_t e = cudaEventSynchronize(sl.jhdr_ev[k]);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "jpeg header staging");
        H = sl.jhdr_ring + k;
    }
    const char* why = "";
    hp_status st = jpeg_parse(host, nbytes, H, &why);
    if (st) {
        set_err(ctx, "jpeg: %s", why);
        return st;
    }
    if (H->width > ctx->cfg.max_width || H->height > ctx->cfg.max_height) {
        set_err(ctx, "jpeg: %dx%d larger than the context's %dx%d", H->width, H->height, ctx->cfg.max_width,
                ctx->cfg.max_height);
        return HP_ERR_INVALID;
    }
    cudaMemcpyAsync(sl.jhdr_dev, H, sizeof(JpegHdr), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(sl.rgb_dev, host, (size_t)nbytes, cudaMemcpyHostToDevice, s);
    if (ring) {
        cudaEventRecord(sl.jhdr_ev[k], s);
        sl.jhdr_pos = (k + 1) % 4;
    }
    *w = H->width;
    *h = H->height;
    *sub = H->sub;
    return check_launch(ctx, "jpeg upload");
}

}  // namespace

extern "C" {

int32_t hp_version(void) { return kAbiVersion; }

int64_t hp_launch_count(void) { return hp::g_launches.load(); }

void hp_default_params(hp_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    // Q = M^-1, M rows = unit Ruifrok-Johnston H, E and H x E (reading C3); float hex-exact
    // (column 0 -> c_H and column 1 -> c_E as listed in SURVEY.md §8(c) S1; column 2 is the
    // float rounding of numpy.linalg.inv(M) in fp64 -- unused by the pipeline)
    const float q[3][3] = {{0x1.7d33d0p+0f, -0x1.15103ap+0f, -0x1.53d24ap-2f},
                           {-0x1.4d1a58p-3f, 0x1.1e3064p+0f, -0x1.35a158p-4f},
                           {0x1.066118p-1f, -0x1.2b1a70p-2f, 0x1.e16e7cp-1f}};
    std::memcpy(p->q, q, sizeof(q));
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
    p->canny_low = 100;  // reading C22
    p->canny_high = 200;
}

const char* hp_status_str(hp_status st) {
    switch (st) {
        case HP_OK: return "ok";
        case HP_ERR_INVALID: return "invalid argument";
        case HP_ERR_CUDA: return "CUDA error";
        case HP_ERR_NOMEM: return "out of memory";
        case HP_ERR_CAPACITY: return "object capacity exceeded";
        case HP_ERR_UNSUPPORTED: return "unsupported device (need sm_100)";
    }
    return "unknown status";
}

const char* hp_last_error(const hp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

hp_status hp_ctx_create(const hp_config* cfg, hp_ctx** out) {
    if (!cfg || !out) return HP_ERR_INVALID;
    *out = nullptr;
    if (cfg->max_width < 1 || cfg->max_height < 1 || cfg->max_width > 16384 || cfg->max_height > 16384 ||
        cfg->n_slots < 1 || cfg->n_slots > 64 || cfg->max_objects < 1)
        return HP_ERR_INVALID;
    std::string why;
    if (!params_ok(cfg->params, &why)) return HP_ERR_INVALID;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return HP_ERR_UNSUPPORTED;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess) return HP_ERR_CUDA;
    if (prop.major != 10) return HP_ERR_UNSUPPORTED;
    if (cudaSetDevice(cfg->device) != cudaSuccess) return HP_ERR_CUDA;

    hp_ctx* ctx = new (std::nothrow) hp_ctx();
    if (!ctx) return HP_ERR_NOMEM;
    ctx->cfg = *cfg;
    ctx->device = cfg->device;
    ctx->rows_copied = std::min(cfg->max_objects, kRowsAsync);
    if (const char* e = getenv("HP_GLOBAL_S8S10")) ctx->global_s8s10 = atoi(e) == 1;
    if (const char* e = getenv("HP_PRIO")) ctx->prio = atoi(e);
    if (const char* e = getenv("HP_GRAPHS")) ctx->graphs = atoi(e) != 0;
    auto dalloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return nullptr;
        ctx->dev_blocks.push_back(p);
        return p;
    };
    auto halloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (cudaMallocHost(&p, bytes ? bytes : 16) != cudaSuccess) return nullptr;
        ctx->host_blocks.push_back(p);
        return p;
    };
    ctx->lut = (float*)dalloc(256 * sizeof(float));
    if (!ctx->lut) { hp_ctx_destroy(ctx); return HP_ERR_NOMEM; }
    upload_od_lut(ctx->lut, 0);

    const int64_t N = (int64_t)cfg->max_width * cfg->max_height;
    const int ntx = (cfg->max_width + kTile - 1) / kTile, nty = (cfg->max_height + kTile - 1) / kTile;
    const int ntiles = ntx * nty;
    const int cap = 2 * ntiles + 65536;
    const int nseg = (cfg->max_height + 63) / 64;
    const int mo = cfg->max_objects;
    ctx->slots.resize(cfg->n_slots);
    for (int i = 0; i < cfg->n_slots; ++i) {
        Slot& s = ctx->slots[i];
        std::memset(&s, 0, sizeof(Slot));
        auto A = [&](size_t b) { return dalloc((b + 255) & ~size_t(255)); };
        s.g = (uint8_t*)A(N); s.flags = (uint8_t*)A(N); s.rbc = (uint8_t*)A(N); s.u8a = (uint8_t*)A(N);
        s.u8b = (uint8_t*)A(N); s.cand = (uint8_t*)A(N); s.big0 = (uint8_t*)A(N); s.F = (uint8_t*)A(N);
        s.split = (uint8_t*)A(N); s.pmask = (uint8_t*)A(N);
        s.lab = (int32_t*)A(4 * N); s.aux = (int32_t*)A(4 * N); s.ML = (int32_t*)A(4 * N);
        s.d = (int32_t*)A(4 * N); s.L = (int32_t*)A(4 * N);
        s.dist = (float*)A(4 * N); s.J = (float*)A(4 * N); s.c = (float*)A(4 * N);
        s.gcol = (uint16_t*)A(2 * N);
        s.seg_top = (int16_t*)A(2 * (size_t)nseg * cfg->max_width);
        s.seg_bot = (int16_t*)A(2 * (size_t)nseg * cfg->max_width);
        s.wl.state = (uint32_t*)A(4 * (size_t)ntiles);
        // per tile (tile engine) or per region sub-tile (region engine, 128 px regions)
        const size_t nsub = (size_t)((cfg->max_width + 127) / 128) * ((cfg->max_height + 127) / 128) * 16;
        s.wl.inrows = (uint32_t*)A(4 * std::max((size_t)ntiles, nsub));
        s.wl.queue = (int32_t*)A(4 * (size_t)cap);
        s.wl.ctr = (unsigned long long*)A(8 * 8);
        s.wl.cap = cap;
        // S4 CTAs per tile: with many tiles in flight each tile's reconstruction takes 3/8 of
        // the SMs (r2, 12 slots: 48-64 CTAs 983-989 tiles/s, 111 955, 148 935); alone it takes
        // 3/4 (the engine's default)
        s.wl.ctas = cfg->n_slots >= 4 ? std::max(1, num_sms() * 3 / 8) : 0;
        s.obj_root = (int32_t*)A(4 * (size_t)mo);
        s.obj_rank = (int32_t*)A(4 * (size_t)mo);
        s.obj_bbox = (int32_t*)A(16 * (size_t)mo);
        s.comp_cap = (int32_t)(N / 4 + 16);  // at most N/4 8-components in N pixels
        s.cs_edge = (int32_t*)A(4 * 4 * kTile * (size_t)ntiles);
        s.cs_roots = (int32_t*)A(4 * (size_t)kTile * kTile * ntiles);
        s.cs_nroots = (int32_t*)A(4 * (size_t)ntiles);
        s.cs_lr = (uint16_t*)A(2 * N);
        s.cs_kind = (uint8_t*)A((size_t)ntiles);
        s.sc_root = (int32_t*)A(4 * (size_t)s.comp_cap);
        s.sc_bbox = (int4*)A(16 * (size_t)s.comp_cap);
        s.sc_area = (int32_t*)A(4 * (size_t)s.comp_cap);
        s.sc_big = (int32_t*)A(4 * (size_t)s.comp_cap);
        s.sc_huge = (int32_t*)A(4 * (size_t)s.comp_cap);
        s.big_px = (int64_t)(cfg->max_width + 2) * (cfg->max_height + 2);
        s.big_scratch = (uint8_t*)A(28 * (size_t)s.big_px);
        s.counters = (unsigned long long*)A(8 * 8);
        s.cnt32 = (int32_t*)A(4 * 32);
        s.stg_label = (int32_t*)A(4 * (size_t)mo);
        s.stg_flags = (int32_t*)A(4 * (size_t)mo);
        s.stg_feat = (float*)A(4 * (size_t)mo * HP_NFEAT);
        s.rgb_dev = (uint8_t*)A(3 * N);
        s.jhdr_dev = (JpegHdr*)A(sizeof(JpegHdr));
        s.jstarts = (int32_t*)A(4 * (size_t)jpeg_max_intervals(cfg->max_width, cfg->max_height));
        s.jblk = (int32_t*)A(4 * (size_t)(3 * N / 8192 + 2));
        s.jerr = (int32_t*)A(16);
        s.jplanes = (uint8_t*)A((size_t)jpeg_planes_bytes(cfg->max_width, cfg->max_height));
        s.jhdr_host = (JpegHdr*)halloc(sizeof(JpegHdr));
        s.jhdr_ring = (JpegHdr*)halloc(4 * sizeof(JpegHdr));
        s.h_jerr = (int32_t*)halloc(16);
        s.lab_dev = (int32_t*)A(4 * N);
        s.tab_label = (int32_t*)A(4 * (size_t)mo);
        s.tab_flags = (int32_t*)A(4 * (size_t)mo);
        s.tab_feat = (float*)A(4 * (size_t)mo * HP_NFEAT);
        s.tab_nrows = (int32_t*)A(16);
        s.h_label = (int32_t*)halloc(4 * (size_t)mo);
        s.h_flags = (int32_t*)halloc(4 * (size_t)mo);
        s.h_feat = (float*)halloc(4 * (size_t)mo * HP_NFEAT);
        s.h_nrows = (int32_t*)halloc(16);
        s.h_arena = (int64_t*)halloc(16);
        void* all[] = {s.g, s.flags, s.rbc, s.u8a, s.u8b, s.cand, s.big0, s.F, s.split, s.pmask, s.lab, s.aux,
                       s.ML, s.d, s.L, s.dist, s.J, s.c, s.gcol, s.seg_top, s.seg_bot, s.wl.state, s.wl.inrows, s.wl.queue,
                       s.wl.ctr, s.obj_root, s.obj_rank, s.obj_bbox, s.cs_edge, s.cs_roots, s.cs_nroots, s.cs_lr, s.cs_kind, s.sc_root, s.sc_bbox, s.sc_area, s.sc_big, s.sc_huge, s.big_scratch, s.stg_label, s.stg_flags, s.stg_feat, s.counters, s.cnt32, s.rgb_dev, s.lab_dev,
                       s.tab_label, s.tab_flags, s.tab_feat, s.tab_nrows, s.h_label, s.h_flags, s.h_feat, s.h_nrows, s.h_arena,
                       s.jhdr_dev, s.jstarts, s.jblk, s.jerr, s.jhdr_host, s.jhdr_ring, s.h_jerr, s.jplanes};
        for (void* p : all)
            if (!p) { hp_ctx_destroy(ctx); return HP_ERR_NOMEM; }
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        if (cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithPriority(&s.hstream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.done_ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.fork_ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.join_ev, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.jhdr_ev[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.jhdr_ev[1], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.jhdr_ev[2], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&s.jhdr_ev[3], cudaEventDisableTiming) != cudaSuccess) {
            hp_ctx_destroy(ctx);
            return HP_ERR_CUDA;
        }
        cudaMemset(s.counters, 0, 64);
        cudaMemset(s.cnt32, 0, 128);
        cudaMemset(s.wl.ctr, 0, 64);
        cudaMemset(s.jerr, 0, 16);
        for (cudaEvent_t e : s.jhdr_ev) cudaEventRecord(e, s.stream);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) { hp_ctx_destroy(ctx); return HP_ERR_CUDA; }
    *out = ctx;
    return HP_OK;
}

hp_status hp_ctx_destroy(hp_ctx* ctx) {
    if (!ctx) return HP_ERR_INVALID;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (Slot& s : ctx->slots) {
        if (s.stream) cudaStreamDestroy(s.stream);
        if (s.hstream) cudaStreamDestroy(s.hstream);
        if (s.done_ev) cudaEventDestroy(s.done_ev);
        if (s.fork_ev) cudaEventDestroy(s.fork_ev);
        if (s.gexec) cudaGraphExecDestroy(s.gexec);
        if (s.join_ev) cudaEventDestroy(s.join_ev);
        for (cudaEvent_t e : s.jhdr_ev)
            if (e) cudaEventDestroy(e);
    }
    for (auto& r : ctx->ring)
        for (auto& set : r)
            for (auto& e : set)
                if (e) cudaEventDestroy(e);
    for (void* p : ctx->dev_blocks) cudaFree(p);
    for (void* p : ctx->host_blocks) cudaFreeHost(p);
    delete ctx;
    return HP_OK;
}

hp_status hp_segment_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb, hp_labels* out, hp_stream s) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if ((st = check_image(ctx, rgb)) || (st = check_labels(ctx, out, rgb->width))) return st;
    return segment(ctx, ctx->slots[slot], rgb, out->labels, out->labels_pitch_elems, out->n_objects_dev,
                   (cudaStream_t)s);
}

hp_status hp_features_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb, const hp_labels* lab,
                           hp_feature_table* out, hp_stream s) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if ((st = check_image(ctx, rgb)) || (st = check_labels(ctx, lab, rgb->width)) || (st = check_table(ctx, out)))
        return st;
    Slot& sl = ctx->slots[slot];
    cudaStream_t cs = (cudaStream_t)s;
    launch_cd(rgb->data, rgb->width, rgb->height, rgb->pitch_bytes, ctx->lut, ctx->cfg.params, sl.g, sl.flags,
              nullptr, cs);
    return features(ctx, sl, rgb->width, rgb->height, lab->labels, lab->labels_pitch_elems, out, cs);
}

hp_status hp_process_tile(hp_ctx* ctx, int32_t slot, const hp_image* rgb, hp_labels* lab,
                          hp_feature_table* out, hp_stream s) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if ((st = check_image(ctx, rgb)) || (st = check_labels(ctx, lab, rgb->width)) || (st = check_table(ctx, out)))
        return st;
    Slot& sl = ctx->slots[slot];
    cudaStream_t cs = (cudaStream_t)s;
    bool fused = false;
    st = segment(ctx, sl, rgb, lab->labels, lab->labels_pitch_elems, lab->n_objects_dev, cs, out, &fused);
    if (st || fused) return st;
    return features(ctx, sl, rgb->width, rgb->height, lab->labels, lab->labels_pitch_elems, out, cs);
}

hp_status hp_process_tile_jpeg(hp_ctx* ctx, int32_t slot, const uint8_t* host_jpeg, int64_t nbytes, hp_labels* lab,
                               hp_feature_table* out, int32_t* decode_err_dev, hp_stream s) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if ((st = check_labels(ctx, lab, 1)) || (st = check_table(ctx, out))) return st;
    Slot& sl = ctx->slots[slot];
    cudaStream_t cs = (cudaStream_t)s;
    int w = 0, h = 0, sub = 1;
    if ((st = upload_jpeg(ctx, sl, host_jpeg, nbytes, cs, true, &w, &h, &sub))) return st;
    if (lab->labels_pitch_elems < w) {
        set_err(ctx, "labels pitch %lld < JPEG width %d", (long long)lab->labels_pitch_elems, w);
        return HP_ERR_INVALID;
    }
    hp_image im{sl.rgb_dev, w, h, 3LL * w};
    bool fused = false;
    st = segment(ctx, sl, &im, lab->labels, lab->labels_pitch_elems, lab->n_objects_dev, cs, out, &fused, sub);
    if (!st && !fused) st = features(ctx, sl, w, h, lab->labels, lab->labels_pitch_elems, out, cs);
    if (!st && decode_err_dev) cudaMemcpyAsync(decode_err_dev, sl.jerr, sizeof(int32_t), cudaMemcpyDeviceToDevice, cs);
    return st ? st : check_launch(ctx, "process_tile_jpeg");
}

hp_status hp_jpeg_info(const uint8_t* host_jpeg, int64_t nbytes, int32_t* width, int32_t* height, int32_t* sampling,
                       int32_t* restart_interval, int32_t* n_intervals) {
    if (!host_jpeg || !width || !height) return HP_ERR_INVALID;
    JpegHdr H;
    const char* why = "";
    const hp_status st = jpeg_parse(host_jpeg, nbytes, &H, &why);
    if (st) return st;
    *width = H.width;
    *height = H.height;
    if (sampling) *sampling = H.sub == 2 ? 420 : 444;
    if (restart_interval) *restart_interval = H.n_intervals > 1 ? H.ri : 0;
    if (n_intervals) *n_intervals = H.n_intervals;
    return HP_OK;
}

hp_status hp_decode_jpeg(hp_ctx* ctx, int32_t slot, const uint8_t* host_jpeg, int64_t nbytes, uint8_t* rgb_dev,
                         int64_t pitch_bytes, hp_stream s) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if (!rgb_dev) {
        set_err(ctx, "hp_decode_jpeg: null output");
        return HP_ERR_INVALID;
    }
    Slot& sl = ctx->slots[slot];
    cudaStream_t cs = (cudaStream_t)s;
    int w = 0, h = 0, sub = 1;
    if ((st = upload_jpeg(ctx, sl, host_jpeg, nbytes, cs, true, &w, &h, &sub))) return st;
    if (pitch_bytes < 3LL * w) {
        set_err(ctx, "hp_decode_jpeg: pitch < 3*width");
        return HP_ERR_INVALID;
    }
    cudaMemsetAsync(sl.jerr, 0, sizeof(int32_t), cs);
    launch_jpeg_decode(sl.jhdr_dev, sub, sl.rgb_dev, 3LL * ctx->cfg.max_width * ctx->cfg.max_height, w, h, sl.jstarts,
                       sl.jblk, sl.jplanes, ctx->lut, ctx->cfg.params, nullptr, nullptr, nullptr, rgb_dev, pitch_bytes,
                       sl.jerr, cs);
    cudaMemcpyAsync(sl.h_jerr, sl.jerr, sizeof(int32_t), cudaMemcpyDeviceToHost, cs);
    cudaError_t e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hp_decode_jpeg");
    if (*sl.h_jerr) {
        set_err(ctx, "hp_decode_jpeg: corrupt scan (%s)",
                (*sl.h_jerr & 1) ? "restart markers do not match the restart interval" : "invalid Huffman code");
        return HP_ERR_INVALID;
    }
    return HP_OK;
}

hp_status hp_set_stage_timing(hp_ctx* ctx, int32_t enable) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (enable && ctx->ring.empty()) {
        ctx->ring.resize(ctx->slots.size());
        ctx->ring_pos.assign(ctx->slots.size(), -1);
        ctx->ring_n.assign(ctx->slots.size(), 0);
        for (auto& r : ctx->ring) {
            r.resize(kRing);
            for (auto& set : r)
                for (auto& e : set)
                    if (cudaEventCreate(&e) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "event create");
        }
    }
    if (enable)
        for (size_t i = 0; i < ctx->slots.size(); ++i) ctx->ring_n[i] = 0;
    ctx->timing = enable != 0;
    return HP_OK;
}

static hp_status sum_set(hp_ctx* ctx, std::array<cudaEvent_t, 12>& set, float* ms11) {
    cudaError_t e = cudaEventSynchronize(set[11]);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "stage times");
    for (int k = 0; k < 11; ++k) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, set[k], set[k + 1]) != cudaSuccess) ms = 0.f;
        ms11[k] += ms;
    }
    cudaGetLastError();
    return HP_OK;
}

hp_status hp_get_stage_times(hp_ctx* ctx, int32_t slot, float* ms11) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if (!ms11 || ctx->ring.empty() || ctx->ring_n[slot] == 0) return HP_ERR_INVALID;
    for (int k = 0; k < 11; ++k) ms11[k] = 0.f;
    return sum_set(ctx, ctx->ring[slot][ctx->ring_pos[slot]], ms11);
}

hp_status hp_reduce_rows(hp_ctx* ctx, const float* feat, const int64_t* off, int32_t n_groups, double* out,
                         int64_t* out_count, hp_stream s) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    // feat may be NULL when every group is empty (a rank that holds no rows)
    if (n_groups < 0 || (n_groups > 0 && (!off || !out || !out_count))) {
        set_err(ctx, "hp_reduce_rows: null pointer or n_groups < 0");
        return HP_ERR_INVALID;
    }
    launch_reduce_rows(feat, off, n_groups, out, out_count, (cudaStream_t)s);
    return check_launch(ctx, "reduce_rows");
}

hp_status hp_group_center(hp_ctx* ctx, const float* feat, const int64_t* off, int32_t n_groups, const double* sums,
                          const int64_t* count, double* mean_m2, hp_stream s) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (n_groups < 0 || (n_groups > 0 && (!off || !sums || !count || !mean_m2))) {
        set_err(ctx, "hp_group_center: null pointer or n_groups < 0");
        return HP_ERR_INVALID;
    }
    launch_group_center(feat, off, n_groups, sums, count, mean_m2, (cudaStream_t)s);
    return check_launch(ctx, "group_center");
}

hp_status hp_group_std(hp_ctx* ctx, const double* mean_m2, const int64_t* count, int32_t n_groups, double* mean,
                       double* std_out, hp_stream s) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (n_groups < 0 || (n_groups > 0 && (!mean_m2 || !count || !mean || !std_out))) {
        set_err(ctx, "hp_group_std: null pointer or n_groups < 0");
        return HP_ERR_INVALID;
    }
    launch_group_std(mean_m2, count, n_groups, mean, std_out, (cudaStream_t)s);
    return check_launch(ctx, "group_std");
}

hp_status hp_stage_times_accum(hp_ctx* ctx, float* ms11, int32_t* count) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (!ms11 || !count || ctx->ring.empty()) return HP_ERR_INVALID;
    for (int k = 0; k < 11; ++k) ms11[k] = 0.f;
    int32_t n = 0;
    for (size_t i = 0; i < ctx->slots.size(); ++i) {
        for (int j = 0; j < ctx->ring_n[i]; ++j) {
            int pos = (ctx->ring_pos[i] - j + kRing) % kRing;
            if ((st = sum_set(ctx, ctx->ring[i][pos], ms11))) return st;
            ++n;
        }
        ctx->ring_n[i] = 0;
    }
    *count = n;
    return HP_OK;
}

hp_status hp_stage_run(hp_ctx* ctx, int32_t slot, hp_stage stage, const hp_stage_io* io, hp_stream strm) {
    hp_status st = enter(ctx, slot);
    if (st) return st;
    if (!io || io->width < 1 || io->height < 1 || io->width > ctx->cfg.max_width || io->height > ctx->cfg.max_height) {
        set_err(ctx, "invalid stage io");
        return HP_ERR_INVALID;
    }
    Slot& sl = ctx->slots[slot];
    const hp_params& p = ctx->cfg.params;
    const int w = io->width, h = io->height;
    const int64_t n = (int64_t)w * h;
    cudaStream_t s = (cudaStream_t)strm;
    auto need = [&](std::initializer_list<const void*> ptrs) {
        for (const void* q : ptrs)
            if (!q) return false;
        return true;
    };
    auto in8 = [&](int k) { return (const uint8_t*)io->in[k]; };
    switch (stage) {
        case HP_STAGE_CD:
            if (!need({io->in[0], io->out[0], io->out[1]})) break;
            launch_cd(in8(0), w, h, 3LL * w, ctx->lut, p, (uint8_t*)io->out[0], (uint8_t*)io->out[1],
                      (unsigned long long*)io->out[2], s);
            return check_launch(ctx, "stage cd");
        case HP_STAGE_RBC:
            if (!need({io->in[0], io->out[0]})) break;
            launch_rbc(in8(0), w, h, sl, (uint8_t*)io->out[0], s);
            return check_launch(ctx, "stage rbc");
        case HP_STAGE_OPEN:
            if (!need({io->in[0], io->out[0]})) break;
            launch_open(in8(0), w, h, p.open_diam, sl.u8b, (uint8_t*)io->out[0], s);
            return check_launch(ctx, "stage open");
        case HP_STAGE_RECON: {
            if (!need({io->in[0], io->in[1], io->in[2], io->out[0]})) break;
            launch_recon_init_u8(in8(1), in8(0), sl.u8b, w, h, s);
            launch_recon_u8_auto(in8(0), sl.u8b, w, h, sl.wl, s);
            launch_tophat(in8(0), sl.u8b, in8(2), p.g1, w, h, (uint8_t*)io->out[0], s);
            if (io->out[1]) cudaMemcpyAsync(io->out[1], sl.u8b, n, cudaMemcpyDeviceToDevice, s);
            return check_launch(ctx, "stage recon");
        }
        case HP_STAGE_AREA: {
            if (!need({io->in[0], io->out[0]})) break;
            launch_area_select(in8(0), w, h, p.cand_min_area, p.cand_max_area, sl, (uint8_t*)io->out[0], s);
            return check_launch(ctx, "stage area");
        }
        case HP_STAGE_FILL:
            if (!need({io->in[0], io->out[0]})) break;
            launch_fill_holes(in8(0), w, h, sl, (uint8_t*)io->out[0], s);
            return check_launch(ctx, "stage fill");
        case HP_STAGE_EDT:
            if (!need({io->in[0], io->out[1]})) break;
            launch_edt(in8(0), w, h, sl, (uint32_t*)io->out[0], (float*)io->out[1], s);
            return check_launch(ctx, "stage edt");
        case HP_STAGE_MARKERS: {
            if (!need({io->in[0], io->in[1], io->out[0]})) break;
            launch_markers((const float*)io->in[0], in8(1), p.h, w, h, sl, (int32_t*)io->out[0], sl.J, s);
            if (io->out[1]) launch_zero_outside_f32(sl.J, in8(1), n, (float*)io->out[1], s);
            return check_launch(ctx, "stage markers");
        }
        case HP_STAGE_WATERSHED:
            if (!need({io->in[0], io->in[1], io->in[2], io->out[0]})) break;
            launch_watershed((const float*)io->in[0], (const int32_t*)io->in[1], in8(2), w, h, sl,
                             (uint8_t*)io->out[0], (float*)io->out[1], (int32_t*)io->out[2], (int32_t*)io->out[3], s);
            return check_launch(ctx, "stage watershed");
        case HP_STAGE_BWLABEL:
            if (!need({io->in[0], io->out[0], io->out[1]})) break;
            launch_bwlabel(in8(0), w, h, p.obj_min_area, p.obj_max_area, sl, (int32_t*)io->out[0], w,
                           (int32_t*)io->out[1], s);
            return check_launch(ctx, "stage bwlabel");
        case HP_STAGE_FEATURES:
            if (!need({io->in[0], io->in[1], io->out[0], io->out[1], io->out[2], io->out[3]})) break;
            launch_canny(in8(1), w, h, p.canny_low, p.canny_high, sl, sl.cand, s);
            launch_features((const int32_t*)io->in[0], w, in8(1), sl.cand, w, h, sl, ctx->cfg.max_objects,
                            (int32_t*)io->out[0], (int32_t*)io->out[1], (float*)io->out[2], ctx->cfg.max_objects,
                            (int32_t*)io->out[3], s);
            return check_launch(ctx, "stage features");
        case HP_STAGE_CANNY:
            if (!need({io->in[0], io->out[0]})) break;
            launch_canny(in8(0), w, h, p.canny_low, p.canny_high, sl, (uint8_t*)io->out[0], s);
            return check_launch(ctx, "stage canny");
        // The hot path's own S5 / S6 / S7-S11 kernels (the pipeline runs these, not the
        // whole-plane AREA / FILL / EDT / MARKERS / WATERSHED / BWLABEL kernels above), fed a
        // caller plane so each can be checked on the oracle's intermediate.
        case HP_STAGE_AREA_TOPHAT: {
            if (!need({io->in[0], io->in[1], io->in[2], io->out[0]})) break;
            int32_t* ncomp5 = sl.cnt32 + 16;
            launch_area_select_tophat(in8(0), in8(1), in8(2), p.g1, w, h, p.cand_min_area, p.cand_max_area, sl,
                                      (uint8_t*)io->out[0], ncomp5, s);
            if (io->out[1]) cudaMemcpyAsync(io->out[1], ncomp5, sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
            return check_launch(ctx, "stage area tophat");
        }
        case HP_STAGE_FILL_COMP:
        case HP_STAGE_COMPONENTS: {
            const bool comp = stage == HP_STAGE_COMPONENTS;
            if (!need({io->in[0], io->out[0]}) ||
                (comp && !need({io->in[1], io->out[1], io->out[2], io->out[3]})))
                break;
            // list the 8-components of the input plane with S5's listing kernel (top-hat of
            // (plane - 0) > 0 & !0, no area bounds), then S6 per component; for COMPONENTS
            // the input is S6's output F (no holes left), so this only writes each F pixel's
            // component root, which S7-S11 consume
            int32_t* ncomp5 = sl.cnt32 + 16;
            cudaMemsetAsync(sl.pmask, 0, (size_t)n, s);
            launch_area_select_tophat(in8(0), sl.pmask, sl.pmask, 0, w, h, 0, INT32_MAX, sl, sl.big0, ncomp5, s);
            uint8_t* F = comp ? sl.F : (uint8_t*)io->out[0];
            launch_fill_components(in8(0), w, h, sl, ncomp5, F, sl.split, s);
            if (!comp) return check_launch(ctx, "stage fill comp");
            const int32_t cap = ctx->cfg.max_objects;
            int32_t* lf = (int32_t*)io->out[2];
            hp_feature_table tab{lf, lf + cap, (float*)io->out[3], cap, sl.tab_nrows};
            launch_canny(in8(1), w, h, p.canny_low, p.canny_high, sl, sl.cand, s);
            launch_components(ncomp5, sl.split, in8(1), sl.cand, p.h, p.obj_min_area, p.obj_max_area, w, h, sl,
                              (int32_t*)io->out[0], w, (int32_t*)io->out[1], &tab, cap, s);
            return check_launch(ctx, "stage components");
        }
        case HP_STAGE_IWPP_RAW: {
            if (!need({io->in[0], io->in[1], io->out[0]})) break;
            launch_recon_init_u8(in8(0), in8(1), (uint8_t*)io->out[0], w, h, s);
            launch_recon_u8_auto(in8(1), (uint8_t*)io->out[0], w, h, sl.wl, s);
            if (io->out[1]) cudaMemcpyAsync(io->out[1], sl.wl.ctr + 3, 4 * sizeof(unsigned long long),
                                            cudaMemcpyDeviceToDevice, s);
            return check_launch(ctx, "stage iwpp");
        }
        case HP_STAGE_CCL8:
        case HP_STAGE_CCL4: {
            if (!need({io->in[0], io->out[0]})) break;
            CclSrc cs{in8(0), 0, false, nullptr};
            launch_ccl(cs, w, h, stage == HP_STAGE_CCL8 ? 8 : 4, sl.lab, nullptr, s);
            launch_ccl_to_labels(cs, w, h, sl.lab, (int32_t*)io->out[0], s);
            return check_launch(ctx, "stage ccl");
        }
        case HP_STAGE_RECON_F32: {
            if (!need({io->in[0], io->in[1], io->out[0]})) break;
            // R = min(marker, mask) on the domain, then IWPP
            const float* mk = (const float*)io->in[0];
            const float* ms = (const float*)io->in[1];
            launch_recon_init_f32(mk, ms, in8(2), n, (float*)io->out[0], s);
            launch_recon_f32(ms, in8(2), (float*)io->out[0], w, h, sl.wl, false, s);
            return check_launch(ctx, "stage recon f32");
        }
        default:
            break;
    }
    set_err(ctx, "stage %d: missing buffer or unknown stage", (int)stage);
    return HP_ERR_INVALID;
}

}  // extern "C"

namespace {

// The demand-driven multi-tile driver behind hp_run_tiles (raw RGB tiles) and
// hp_run_tiles_jpeg (JPEG files, NEXT-3).  next(&host, &pitch_or_nbytes, &tile_id) -> 0 / 1.
template <class Next>
hp_status run_tiles_impl(hp_ctx* ctx, int w, int h, bool jpeg, Next next, const hp_result_sink* sink) {
    const int ns = ctx->cfg.n_slots;
    const int mo = ctx->cfg.max_objects;
    const hp_row_arena* arena = sink->arena;
    if (arena && (!arena->tile || !arena->label || !arena->flags || !arena->feat || !arena->cursor ||
                  arena->capacity < 0)) {
        set_err(ctx, "run_tiles: arena with a NULL buffer or negative capacity");
        return HP_ERR_INVALID;
    }
    const hp_row_arena no_arena{};
    const hp_row_arena& akey = arena ? *arena : no_arena;
    auto same_arena = [&](const hp_row_arena& a) {
        return a.tile == akey.tile && a.label == akey.label && a.flags == akey.flags && a.feat == akey.feat &&
               a.capacity == akey.capacity && a.cursor == akey.cursor;
    };
    std::vector<int64_t> tile_of(ns, -1);
    std::vector<hp_status> st_of(ns, HP_OK);
    bool drained = false;
    int inflight = 0;
    auto deliver = [&](int i) -> hp_status {
        Slot& sl = ctx->slots[i];
        cudaError_t e = cudaEventSynchronize(sl.done_ev);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "run_tiles sync");
        int nrows = *sl.h_nrows;
        hp_status ts = st_of[i];
        if (nrows > mo) ts = HP_ERR_CAPACITY;
        int nr = std::min(nrows, mo);
        if (jpeg && *sl.h_jerr) {  // corrupt scan: the rows are not trustworthy
            ts = HP_ERR_INVALID;
            if (!arena) nr = 0;    // (arena mode: the run was appended on the device already)
        }
        if (arena) {  // rows stay in the device arena; the run [h_arena[1], +nr) may be clipped
            if (sl.h_arena[1] + nr > arena->capacity) ts = HP_ERR_CAPACITY;
            sink->done(sink->user, tile_of[i], nr, nullptr, nullptr, nullptr, ts);
            tile_of[i] = -1;
            --inflight;
            return HP_OK;
        }
        if (nr > ctx->rows_copied) {  // rare: more rows than the async window
            int extra = nr - ctx->rows_copied;
            cudaMemcpy(sl.h_label + ctx->rows_copied, sl.tab_label + ctx->rows_copied, 4 * (size_t)extra, cudaMemcpyDeviceToHost);
            cudaMemcpy(sl.h_flags + ctx->rows_copied, sl.tab_flags + ctx->rows_copied, 4 * (size_t)extra, cudaMemcpyDeviceToHost);
            cudaMemcpy(sl.h_feat + (size_t)ctx->rows_copied * HP_NFEAT, sl.tab_feat + (size_t)ctx->rows_copied * HP_NFEAT,
                       4 * (size_t)extra * HP_NFEAT, cudaMemcpyDeviceToHost);
        }
        sink->done(sink->user, tile_of[i], nr, sl.h_label, sl.h_flags, sl.h_feat, ts);
        tile_of[i] = -1;
        --inflight;
        return HP_OK;
    };
    // Fill every free slot, then deliver whichever in-flight slot finishes first: tiles take
    // very different times (chain-bound reconstructions), so waiting on slots in a fixed
    // order would leave finished slots idle behind a slow one.
    auto submit = [&](int i) -> hp_status {
        Slot& sl = ctx->slots[i];
        cudaStream_t s = sl.stream;
        const uint8_t* host = nullptr;
        int64_t pitch = 0, tid = -1;
        int jsub = 1;
        while (true) {  // until a tile is in flight on slot i or the source is drained
            host = nullptr;
            pitch = 0;
            tid = -1;
            if (next(&host, &pitch, &tid) != 0) {
                drained = true;
                return HP_OK;
            }
            if (!jpeg) {
                if (!host || pitch < 3LL * w) {
                    set_err(ctx, "run_tiles: tile %lld has a NULL host pointer or pitch %lld < 3*width", (long long)tid,
                            (long long)pitch);
                    return HP_ERR_INVALID;
                }
                break;
            }
            // a JPEG the decoder cannot take (malformed, out of scope, wrong size) fails alone:
            // reported through done() with no rows, and the slot takes the next tile
            int jw = 0, jh = 0;
            hp_status ps = upload_jpeg(ctx, sl, host, pitch, s, false, &jw, &jh, &jsub);
            if (ps == HP_ERR_CUDA) return ps;
            if (!ps && (jw != w || jh != h)) {
                set_err(ctx, "run_tiles_jpeg: tile %lld is %dx%d, the source says %dx%d", (long long)tid, jw, jh, w, h);
                ps = HP_ERR_INVALID;
            }
            if (!ps) break;
            sink->done(sink->user, tid, 0, sl.h_label, sl.h_flags, sl.h_feat, ps);
        }
        sl.h_arena[0] = tid;  // read by this tile's H2D (arena mode); the slot's previous tile was delivered
        if (!jpeg)
            cudaMemcpy2DAsync(sl.rgb_dev, 3 * (size_t)w, host, (size_t)pitch, 3 * (size_t)w, h, cudaMemcpyHostToDevice, s);
        hp_image im{sl.rgb_dev, w, h, 3LL * w};
        hp_feature_table tab{sl.tab_label, sl.tab_flags, sl.tab_feat, mo, sl.tab_nrows};
        // the tile's chain: segmentation + features on the slot's own buffers, rows D2H
        auto chain = [&]() -> hp_status {
            bool fused = false;
            hp_status r = segment(ctx, sl, &im, sl.lab_dev, w, sl.cnt32 + 4, s, &tab, &fused, jpeg ? jsub : 0);
            if (!r && !fused) r = features(ctx, sl, w, h, sl.lab_dev, w, &tab, s);
            if (r) return r;
            cudaMemcpyAsync(sl.h_nrows, sl.tab_nrows, 4, cudaMemcpyDeviceToHost, s);
            if (jpeg) cudaMemcpyAsync(sl.h_jerr, sl.jerr, 4, cudaMemcpyDeviceToHost, s);
            if (arena) {  // S12 into the device arena: the tile id goes up, the run offset down
                int64_t* dev_tid = (int64_t*)&sl.counters[4];
                int64_t* dev_base = (int64_t*)&sl.counters[5];
                cudaMemcpyAsync(dev_tid, &sl.h_arena[0], 8, cudaMemcpyHostToDevice, s);
                launch_arena_append(sl.tab_nrows, mo, sl.tab_label, sl.tab_flags, sl.tab_feat, dev_base, dev_tid,
                                    *arena, s);
                cudaMemcpyAsync(&sl.h_arena[1], dev_base, 8, cudaMemcpyDeviceToHost, s);
                return HP_OK;
            }
            cudaMemcpyAsync(sl.h_label, sl.tab_label, 4 * (size_t)ctx->rows_copied, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(sl.h_flags, sl.tab_flags, 4 * (size_t)ctx->rows_copied, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(sl.h_feat, sl.tab_feat, 4 * (size_t)ctx->rows_copied * HP_NFEAT, cudaMemcpyDeviceToHost, s);
            return HP_OK;
        };
        // CUDA graph: the slot's first tile of a size runs op by op (one-time
        // setup), the second is captured, every later tile replays the graph -- one launch
        // instead of ~30 API calls.  Not with stage timing or the host-synchronising
        // background skip, whose host decisions a graph cannot replay.
        const bool graphable = ctx->graphs && !ctx->timing && ctx->cfg.params.bg_skip_frac > 1.0f &&
                               ctx->prio == 0;
        hp_status r = HP_OK;
        const int gkey = jpeg ? jsub : 0;  // raw, JPEG 4:4:4 or JPEG 4:2:0: different chains
        const bool same = sl.graph_w == w && sl.graph_h == h && sl.graph_jpeg == gkey && same_arena(sl.graph_arena);
        if (graphable && sl.gexec && same) {
            if (cudaGraphLaunch(sl.gexec, s) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "graph launch");
        } else if (graphable && same) {
            cudaGraph_t g = nullptr;
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
                return cuda_fail(ctx, cudaGetLastError(), "begin capture");
            r = chain();
            const cudaError_t ce = cudaStreamEndCapture(s, &g);
            if (r) return r;
            if (ce != cudaSuccess || cudaGraphInstantiate(&sl.gexec, g, 0) != cudaSuccess)
                return cuda_fail(ctx, cudaGetLastError(), "graph capture");
            cudaGraphDestroy(g);
            if (cudaGraphLaunch(sl.gexec, s) != cudaSuccess) return cuda_fail(ctx, cudaGetLastError(), "graph launch");
        } else {
            if ((r = chain())) return r;
            if (sl.gexec) {
                cudaGraphExecDestroy(sl.gexec);
                sl.gexec = nullptr;
            }
            sl.graph_w = w;
            sl.graph_h = h;
            sl.graph_jpeg = gkey;
            sl.graph_arena = akey;
        }
        cudaEventRecord(sl.done_ev, s);
        if ((r = check_launch(ctx, "run_tiles"))) return r;
        tile_of[i] = tid;
        st_of[i] = HP_OK;
        ++inflight;
        return HP_OK;
    };
    // on an error, wait for the tiles already in flight (their host buffers are the caller's)
    auto abandon = [&](hp_status e) {
        for (int i = 0; i < ns; ++i)
            if (tile_of[i] >= 0) cudaEventSynchronize(ctx->slots[i].done_ev);
        return e;
    };
    hp_status st = HP_OK;
    int scan = 0;
    while (true) {
        for (int i = 0; i < ns && !drained; ++i)
            if (tile_of[i] < 0 && (st = submit(i))) return abandon(st);
        if (inflight == 0) break;
        int done = -1;
        for (int k = 0; k < ns && done < 0; ++k) {
            const int i = (scan + k) % ns;
            if (tile_of[i] < 0) continue;
            const cudaError_t q = cudaEventQuery(ctx->slots[i].done_ev);
            if (q == cudaSuccess) done = i;
            else if (q != cudaErrorNotReady) return abandon(cuda_fail(ctx, q, "run_tiles query"));
        }
        if (done < 0) {
            std::this_thread::sleep_for(std::chrono::microseconds(20));
            continue;
        }
        scan = (done + 1) % ns;
        if ((st = deliver(done))) return abandon(st);
    }
    return HP_OK;
}

}  // namespace

extern "C" {

hp_status hp_run_tiles(hp_ctx* ctx, const hp_tile_source* src, const hp_result_sink* sink) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (!src || !src->next || !sink || !sink->done) {
        set_err(ctx, "run_tiles: NULL source, sink or callback");
        return HP_ERR_INVALID;
    }
    const int w = src->width, h = src->height;
    if (w < 1 || h < 1 || w > ctx->cfg.max_width || h > ctx->cfg.max_height) {
        set_err(ctx, "run_tiles: tile size %dx%d outside 1..%dx%d", w, h, ctx->cfg.max_width, ctx->cfg.max_height);
        return HP_ERR_INVALID;
    }
    return run_tiles_impl(
        ctx, w, h, false,
        [&](const uint8_t** host, int64_t* pitch, int64_t* tid) { return src->next(src->user, host, pitch, tid); },
        sink);
}

hp_status hp_run_tiles_jpeg(hp_ctx* ctx, const hp_jpeg_source* src, const hp_result_sink* sink) {
    hp_status st = enter(ctx, 0);
    if (st) return st;
    if (!src || !src->next || !sink || !sink->done) {
        set_err(ctx, "run_tiles_jpeg: NULL source, sink or callback");
        return HP_ERR_INVALID;
    }
    const int w = src->width, h = src->height;
    if (w < 1 || h < 1 || w > ctx->cfg.max_width || h > ctx->cfg.max_height) {
        set_err(ctx, "run_tiles_jpeg: tile size %dx%d outside 1..%dx%d", w, h, ctx->cfg.max_width, ctx->cfg.max_height);
        return HP_ERR_INVALID;
    }
    return run_tiles_impl(
        ctx, w, h, true,
        [&](const uint8_t** host, int64_t* nbytes, int64_t* tid) { return src->next(src->user, host, nbytes, tid); },
        sink);
}

}  // extern "C"
