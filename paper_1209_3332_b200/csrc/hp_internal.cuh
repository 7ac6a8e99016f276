// hp_internal.cuh -- shared device helpers and host launcher declarations of libhp.
// Product code: shares nothing with oracle/ (test infrastructure).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/hp.h"

namespace hp {

constexpr int kTile = 32;          // worklist / CCL tile edge (one warp = one tile row)
constexpr int kHalo = kTile + 2;   // tile plus a 1-pixel halo on each side
constexpr int32_t kInfI = 0x3fffffff;

// ---------------------------------------------------------------- memory helpers
template <class T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ uint8_t ldcg<uint8_t>(const uint8_t* p) {
    return (uint8_t)__ldcg(reinterpret_cast<const unsigned char*>(p));
}
template <class T>
__device__ __forceinline__ void stcg(T* p, T v) { __stcg(p, v); }
template <>
__device__ __forceinline__ void stcg<uint8_t>(uint8_t* p, uint8_t v) {
    __stcg(reinterpret_cast<unsigned char*>(p), (unsigned char)v);
}

__device__ __forceinline__ int sat_add(int a, int b) {
    long long s = (long long)a + (long long)b;
    return s >= kInfI ? kInfI : (int)s;
}

// N8 neighbour order of the watershed parent bitmask: bit j <-> (dx8(j), dy8(j)) =
// (-1,-1) (0,-1) (1,-1) (-1,0) (1,0) (-1,1) (0,1) (1,1).
__host__ __device__ __forceinline__ int dx8(int j) { return (j == 0 || j == 3 || j == 5) ? -1 : (j == 1 || j == 6) ? 0 : 1; }
__host__ __device__ __forceinline__ int dy8(int j) { return j < 3 ? -1 : (j < 5 ? 0 : 1); }
// index j of offset (dx, dy), dx, dy in {-1, 0, 1}, (0, 0) excluded
__host__ __device__ __forceinline__ int nb_index(int dx, int dy) {
    int k = (dy + 1) * 3 + (dx + 1);   // 0..8, 4 = centre
    return k < 4 ? k : k - 1;
}

// ---------------------------------------------------------------- worklist
// Asynchronous tile worklist (the "hierarchical queue" of PAPER.md:633, at tile grain):
// state[t] in {IDLE, QUEUED, BUSY, BUSY_DIRTY}; queue = ring of tile ids with EMPTY
// sentinels; ctr[0] head, ctr[1] tail, ctr[2] pending (queued or busy tiles),
// ctr[3] tiles processed, ctr[4] local rounds.
struct Worklist {
    uint32_t* state;
    uint32_t* inrows;   // per tile: rows (bit y-1) whose halo neighbours improved since last job
    int32_t* queue;
    unsigned long long* ctr;
    int32_t cap;      // ring capacity (>= ntiles + max warps)
    int32_t ntx, nty; // tile grid
    int32_t ctas;     // region-engine CTAs per launch (0: the engine's single-tile default)
};

// header of a JPEG tile, parsed on the host (k_jpeg.cu jpeg_parse)
struct JpegHdr {
    int32_t width, height;
    int32_t mcux, mcuy;          // MCUs per row / column (8 x 8 px, or 16 x 16 px for 4:2:0)
    int32_t ri;                  // MCUs per restart interval (all MCUs when there is no DRI)
    int32_t n_intervals;
    int64_t scan_off, scan_len;  // the entropy-coded segment within the file
    uint16_t q[3][64];           // dequantisation factor per component, natural order
    uint8_t td[3], ta[3];        // DC table (0..3) and AC table (4..7) of each component
    uint8_t sub;                 // 1: 4:4:4; 2: 4:2:0 (Y sampled 2 x 2, MCU 16 x 16 px)
    uint8_t pad;
    uint8_t bits[8][17];         // BITS[1..16] of tables 0..3 (DC) and 4..7 (AC)
    uint8_t vals[8][256];        // HUFFVAL
};

// ---------------------------------------------------------------- scratch of one slot
struct Slot {
    // u8 planes
    uint8_t *g, *flags, *rbc, *u8a, *u8b, *cand, *big0, *F, *split, *pmask;
    // 32-bit planes
    int32_t *lab, *aux, *ML, *d, *L;
    float *dist, *J, *c;
    uint32_t* d2;
    uint16_t* gcol;
    // EDT segment summaries
    int16_t *seg_top, *seg_bot;
    // worklist
    Worklist wl;
    // objects
    int32_t *obj_root, *obj_bbox, *obj_rank;
    int32_t* cs_edge;    // k_ccls.cu: per 32x32 tile, the roots of its 4 x 32 edge pixels
    int32_t* cs_roots;   // k_ccls.cu: per tile, its local roots (up to 1024)
    int32_t* cs_nroots;  // k_ccls.cu: per tile, number of local roots
    uint16_t* cs_lr;     // k_ccls.cu: per pixel, its local root within its 32x32 tile (0xffff: none)
    uint8_t* cs_kind;    // k_ccls.cu: per tile, 0 no foreground / 1 general / 2 all foreground
    // S5 component list (k_ccls.cu listing; consumed by the per-component S6 / S7-S11 kernels)
    int32_t* sc_root;
    int4* sc_bbox;
    int32_t* sc_area;
    int32_t* sc_big;       // components whose window needs a whole block
    int32_t* sc_huge;      // components whose window exceeds shared memory
    // global-memory window storage for those (k_comp.cu CompGm), big_px pixels per plane
    uint8_t* big_scratch;
    int64_t big_px;
    int32_t comp_cap;      // capacity of the component lists (N / 4 + 16)
    // staging table of the fused S7-S11 path (rows in discovery order)
    int32_t *stg_label, *stg_flags;
    float* stg_feat;
    // small device counters (8 x u64): [0] bg count, [1] any-bg flag, [2] n objects,
    // [4] run_tiles arena tile id, [5] run_tiles arena offset
    unsigned long long* counters;
    int32_t* cnt32;  // 32 ints: [1] edt any-bg, [2] features count, [4] run_tiles n_objects,
                     // [8..15] k_comp (S7-S11 queues), [16] S5 component count, [18..21] S6 queues
    // run_tiles staging
    uint8_t* rgb_dev;            // also the JPEG file buffer of the compressed path (3N bytes)
    JpegHdr* jhdr_dev;           // parsed header of the slot's JPEG tile (device)
    JpegHdr* jhdr_host;          // pinned staging of that header (hp_run_tiles_jpeg)
    int32_t* jstarts;            // restart-interval start offsets
    int32_t* jblk;               // per-chunk restart-marker counts
    int32_t* jerr;               // decode error word
    uint8_t* jplanes;            // 4:2:0 component planes (Y, Cb, Cr) before upsampling
    int32_t* h_jerr;             // pinned copy of it, per delivered tile
    int32_t* lab_dev;
    int32_t *tab_label, *tab_flags, *tab_nrows;
    float* tab_feat;
    cudaStream_t stream;
    // pinned host staging for run_tiles results
    int32_t *h_label, *h_flags, *h_nrows;
    float* h_feat;
    // arena mode: h_arena[0] tile id (H2D into counters[4] each tile), h_arena[1] the run's
    // arena offset (D2H from counters[5])
    int64_t* h_arena;
    cudaEvent_t done_ev;
    // hp_run_tiles: the per-tile chain (compute + D2H) captured once as a CUDA graph
    cudaGraphExec_t gexec;
    int graph_w, graph_h;
    int graph_jpeg;            // the graph decodes a JPEG tile (hp_run_tiles_jpeg)
    hp_row_arena graph_arena;  // the arena the graph was captured with (all zero: host rows)
    // JPEG header staging ring of hp_process_tile_jpeg / hp_decode_jpeg: the host parses
    // into entry k only after the copy issued from it last time has run (event)
    JpegHdr* jhdr_ring;        // pinned [kJpegRing]
    cudaEvent_t jhdr_ev[4];
    int jhdr_pos;
    // high-priority side stream for the latency-bound stages (hp_ctx::prio)
    cudaStream_t hstream;
    cudaEvent_t fork_ev, join_ev;
};

// ---------------------------------------------------------------- launchers (host)
// every kernel launch of libhp goes through (note_launch(), kernel<<<...>>>(...)) so the
// bench can report how many of OUR kernels ran (hp_launch_count)
void note_launch();
// Per-device one-time setup (cudaFuncSetAttribute, occupancy-derived grid sizes apply to the
// CURRENT device only): run f once for each device a launcher is used on; thread-safe.
struct PerDevice {
    std::mutex m;
    bool done[64] = {};
    int value[64] = {};
    template <class F>
    int get(F f) {  // f() -> int, evaluated once per device; returns the device's value
        int dev = 0;
        cudaGetDevice(&dev);
        dev &= 63;
        std::lock_guard<std::mutex> g(m);
        if (!done[dev]) {
            value[dev] = f();
            done[dev] = true;
        }
        return value[dev];
    }
};
// Number of SMs of the current device (148 on a B200), cached per device: every grid that is
// sized "a multiple of the SM count" takes it from here instead of a literal.
int num_sms();
// S1
void launch_cd(const uint8_t* rgb, int w, int h, int64_t pitch, const float* lut,
               const hp_params& p, uint8_t* g, uint8_t* flags, unsigned long long* bg_count,
               cudaStream_t s);
void upload_od_lut(float* lut_dev, cudaStream_t s);
// S0/S1 from a JPEG tile (NEXT-3, k_jpeg.cu).  The host parses the marker segments into a
// JpegHdr (the tables and the scan's place in the file); the device finds the restart markers,
// Huffman-decodes one restart interval per thread, dequantises, runs the islow IDCT and
// the YCbCr->RGB conversion, and feeds every pixel straight into S1 (cd_pixel.cuh): the
// decoded RGB tile never reaches HBM.
// Parse a baseline JPEG (T.81 B.2): SOF0/1 8-bit, 3 components with 1x1 sampling, one
// interleaved sequential scan.  HP_ERR_UNSUPPORTED outside that scope, HP_ERR_INVALID on a
// malformed stream; *why gets the reason.
hp_status jpeg_parse(const uint8_t* data, int64_t n, JpegHdr* out, const char** why);
// Capacity of the per-slot restart-interval offset array for a tile of npx pixels.
// (at most one interval per 8 x 8 MCU of the largest tile; 4:2:0 MCUs are larger)
inline int64_t jpeg_max_intervals(int w, int h) { return (int64_t)((w + 7) / 8) * ((h + 7) / 8) + 1; }
// Decode the file (device copy `file`, header `hdr` on the device) of a w x h tile; sub is
// the host-parsed sampling (1: 4:4:4, 2: 4:2:0).  rgb == nullptr: S1 fused (g, flags,
// bg_count as launch_cd); else the decoded RGB tile (pitch rgb_pitch) only -- the
// verification path.  4:4:4 decodes straight into S1; 4:2:0 decodes to component planes
// (`planes`, jpeg_planes_bytes) and a second kernel upsamples (reading J4), converts and runs
// S1.  starts / blkcnt: slot scratch (jpeg_max_intervals entries; file_cap / 8192 + 2
// entries).  err: device int, OR-ed with 1 (restart-marker count mismatch) or 2 (invalid
// Huffman code); the caller zeroes it.
inline int64_t jpeg_planes_bytes(int w, int h) {
    const int64_t yw = (w + 15) / 16 * 16, yh = (h + 15) / 16 * 16;
    return yw * yh + 2 * (yw / 2) * (yh / 2);
}
void launch_jpeg_decode(const JpegHdr* hdr, int sub, const uint8_t* file, int64_t file_cap, int w, int h,
                        int32_t* starts, int32_t* blkcnt, uint8_t* planes, const float* lut, const hp_params& p,
                        uint8_t* g, uint8_t* flags, unsigned long long* bg_count, uint8_t* rgb, int64_t rgb_pitch,
                        int32_t* err, cudaStream_t s);
// S3
void launch_open(const uint8_t* g, int w, int h, int diam, uint8_t* tmp, uint8_t* out,
                 cudaStream_t s);
// CCL engine: fg from a u8 plane (nonzero, or zero when invert), optional flag bit mask,
// optional float equality plane (flat zones).  lab = root index (min linear index) or -1.
struct CclSrc {
    const uint8_t* plane;  // foreground plane
    uint8_t bitmask;       // 0: fg = plane != 0 ; else fg = (plane & bitmask) != 0
    bool invert;           // fg = !fg
    const float* eq;       // if non-null: connected iff eq[p] == eq[q]
};
void launch_ccl(const CclSrc& src, int w, int h, int conn, int32_t* lab, int32_t* aux_zero,
                cudaStream_t s);
void launch_ccl_count(const CclSrc& src, int w, int h, const int32_t* lab, int32_t* aux,
                      cudaStream_t s);
void launch_ccl_area_filter(const CclSrc& src, int w, int h, const int32_t* lab,
                            const int32_t* area, int amin, int amax, uint8_t* out,
                            cudaStream_t s);
void launch_ccl_to_labels(const CclSrc& src, int w, int h, const int32_t* lab, int32_t* out,
                          cudaStream_t s);
// S2
// k_ccls.cu (CCL-select: u8 output from a per-component property, no label plane)
void launch_rbc(const uint8_t* flags, int w, int h, Slot& sl, uint8_t* rbc, cudaStream_t s);
// S6
void launch_fill_holes(const uint8_t* big0, int w, int h, Slot& sl, uint8_t* F, cudaStream_t s,
                       const int32_t* gate = nullptr);
void launch_area_select(const uint8_t* cand, int w, int h, int amin, int amax, Slot& sl, uint8_t* out,
                        cudaStream_t s);
void launch_area_select_tophat(const uint8_t* g, const uint8_t* R, const uint8_t* rbc, int g1, int w, int h,
                               int amin, int amax, Slot& sl, uint8_t* out, int32_t* count, cudaStream_t s);
// S6 per S5 component (k_comp.cu): F = component | its holes, enc = other candidates inside a
// hole (shared-memory windows; the rare windows too big for shared memory in one block over
// global-memory storage)
void launch_fill_components(const uint8_t* big0, int w, int h, Slot& sl, const int32_t* count, uint8_t* F,
                            uint8_t* enc, cudaStream_t s);
// IWPP / worklist engine
void wl_init_all(const Worklist& wl, int w, int h, cudaStream_t s);
void wl_init_from_mask(const Worklist& wl, const uint8_t* mask, int w, int h, cudaStream_t s);
void launch_recon_u8(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl,
                     cudaStream_t s);
// region-granular variant (k_region.cu); the default for S4 unless HP_IWPP_TILES=1
void launch_recon_u8_regions(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl,
                             cudaStream_t s);
// dispatch between the two (same result; env HP_IWPP_TILES=1 selects the tile engine)
void launch_recon_u8_auto(const uint8_t* mask, uint8_t* R, int w, int h, const Worklist& wl,
                          cudaStream_t s);
void launch_recon_f32(const float* mask, const uint8_t* dom, float* R, int w, int h,
                      const Worklist& wl, bool init_from_mask_tiles, cudaStream_t s);
void launch_plateau_dist(const float* c, int32_t* d, int w, int h, const Worklist& wl,
                         const uint8_t* F, cudaStream_t s);
void launch_parent_min(const uint8_t* pm, int32_t* L, int w, int h, const Worklist& wl,
                       const uint8_t* F, cudaStream_t s);
// S4 helpers
void launch_recon_init_u8(const uint8_t* marker, const uint8_t* mask, uint8_t* R, int w, int h,
                          cudaStream_t s);
void launch_tophat(const uint8_t* g, const uint8_t* R, const uint8_t* rbc, int g1, int w, int h,
                   uint8_t* cand, cudaStream_t s);
// S7
void launch_edt(const uint8_t* F, int w, int h, Slot& sl, uint32_t* d2_out, float* dist, cudaStream_t s,
                const int32_t* cond = nullptr);
// S8, S9
void launch_markers(const float* dist, const uint8_t* F, float hh, int w, int h, Slot& sl,
                    int32_t* ML, float* J, cudaStream_t s);
void launch_watershed(const float* dist, const int32_t* ML, const uint8_t* F, int w, int h,
                      Slot& sl, uint8_t* split, float* c_out, int32_t* d_out, int32_t* L_out,
                      cudaStream_t s);
// S10
void launch_bwlabel(const uint8_t* split, int w, int h, int amin, int amax, Slot& sl,
                    int32_t* labels, int64_t lpitch, int32_t* n_objects, cudaStream_t s);
// S7-S11 per F component from the S5 list (k_comp.cu); edge = Canny plane (features only)
void launch_components(const int32_t* count5, const uint8_t* enc, const uint8_t* g, const uint8_t* edge, float hh,
                       int amin, int amax, int w, int h, Slot& sl, int32_t* labels, int64_t lpitch,
                       int32_t* n_objects, const hp_feature_table* table, int32_t max_objects, cudaStream_t s);
// S11
// per-image aggregation (k_agg.cu): segmented fp64 sums / sums of squares of feature rows
void launch_reduce_rows(const float* feat, const int64_t* off, int32_t n_groups, double* out, int64_t* count,
                        cudaStream_t s);
void launch_group_center(const float* feat, const int64_t* off, int32_t n_groups, const double* sums,
                         const int64_t* count, double* mean_m2, cudaStream_t s);
void launch_group_std(const double* mean_m2, const int64_t* count, int32_t n_groups, double* mean, double* std_out,
                      cudaStream_t s);
// device row arena of hp_run_tiles (k_agg.cu): reserve min(*nrows, tab_cap) rows at a.cursor
// (offset -> *base), then copy the tile's rows with tile id *tile_id, clipped to capacity
void launch_arena_append(const int32_t* nrows, int32_t tab_cap, const int32_t* lab, const int32_t* fl,
                         const float* feat, int64_t* base, const int64_t* tile_id, const hp_row_arena& a,
                         cudaStream_t s);
// Feature-stage Canny (k_ccls.cu): edges 0/1 = cv2.Canny(g, low, high), reading C22
void launch_canny(const uint8_t* g, int w, int h, int low, int high, Slot& sl, uint8_t* edges, cudaStream_t s);
void launch_features(const int32_t* labels, int64_t lpitch, const uint8_t* g, const uint8_t* edge, int w, int h,
                     Slot& sl, int32_t max_objects, int32_t* row_label, int32_t* row_flags,
                     float* feat, int32_t capacity, int32_t* n_rows, cudaStream_t s);

}  // namespace hp
