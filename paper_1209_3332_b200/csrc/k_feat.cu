// k_feat.cu -- S11: per-object features ("Features comp."; families of
// pixel statistics, gradient statistics, Haralick, morphometry; per-object
// bag of tasks PAPER.md:223-224; definitions: DESIGN.md "Feature table", reading C16/C17).
//
//   k_obj_find   roots = pixels whose label equals 1 + their own linear index
//   k_obj_rank   rank of each root among all roots (rows in ascending label order)
//   k_obj_bbox   bounding boxes by warp-aggregated atomicMin/Max on the compact id
//   k_obj_feat   one CTA per object (grid-stride over the device-side count): exact
//                integer sums (area, moments, perimeter, 256-bin histogram and 8x8 GLCM in
//                shared memory via smem atomics), Sobel magnitude on the fly with fp64
//                two-pass moments in a fixed reduction order (deterministic), Canny edge
//                counts, then the team finalises the 36 features in fp64 (stored as f32).
// Compiled with -fmad=false so the fp64 finaliser rounds like its written formulas.
#include <cfloat>
#include <cmath>

#include "feat_common.cuh"

namespace hp {

namespace {


#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

inline int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, num_sms() * 16); }

__global__ void k_obj_find(const int32_t* __restrict__ labels, int64_t lpitch, int w, int h,
                           int32_t* __restrict__ cnt, int32_t* __restrict__ roots, int32_t cap) {
    const int64_t n = (int64_t)w * h;
    GRID_LOOP(p, n) {
        int y = (int)(p / w), x = (int)(p - (int64_t)y * w);
        if (labels[(int64_t)y * lpitch + x] == (int32_t)(p + 1)) {
            int i = atomicAdd(cnt, 1);
            if (i < cap) roots[i] = (int32_t)p;
        }
    }
}

__global__ void k_obj_rank(const int32_t* __restrict__ cnt, int32_t cap, const int32_t* __restrict__ roots,
                           int32_t* __restrict__ rank_root, int32_t* __restrict__ idmap) {
    const int n = min(*cnt, cap);
    __shared__ int32_t chunk[1024];
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        int i = base + threadIdx.x;
        int32_t me = i < n ? roots[i] : 0;
        int rk = 0;
        for (int c0 = 0; c0 < n; c0 += 1024) {
            __syncthreads();
            for (int k = threadIdx.x; k < 1024 && c0 + k < n; k += blockDim.x) chunk[k] = roots[c0 + k];
            __syncthreads();
            int lim = min(1024, n - c0);
            for (int k = 0; k < lim; ++k) rk += chunk[k] < me;
        }
        if (i < n) {
            rank_root[rk] = me;
            idmap[me] = rk;
        }
    }
}

__global__ void k_bbox_init(const int32_t* __restrict__ cnt, int32_t cap, int32_t* __restrict__ bbox) {
    const int n = min(*cnt, cap);
    GRID_LOOP(i, (int64_t)n) {
        bbox[4 * i + 0] = INT_MAX;
        bbox[4 * i + 1] = INT_MAX;
        bbox[4 * i + 2] = -1;
        bbox[4 * i + 3] = -1;
    }
}

__global__ void k_obj_bbox(const int32_t* __restrict__ labels, int64_t lpitch, int w, int h,
                           const int32_t* __restrict__ cnt, int32_t cap, const int32_t* __restrict__ idmap,
                           int32_t* __restrict__ bbox) {
    const int64_t n = (int64_t)w * h;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = base + threadIdx.x;
        int id = -1, x = 0, y = 0;
        if (p < n) {
            y = (int)(p / w);
            x = (int)(p - (int64_t)y * w);
            int32_t l = labels[(int64_t)y * lpitch + x];
            if (l > 0) id = idmap[l - 1];
            if (id >= cap) id = -1;
        }
        unsigned peers = __match_any_sync(0xffffffffu, id);
        if (id < 0) continue;
        int x0 = __reduce_min_sync(peers, x), y0 = __reduce_min_sync(peers, y);
        int x1 = __reduce_max_sync(peers, x), y1 = __reduce_max_sync(peers, y);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
            atomicMin(&bbox[4 * id + 0], x0);
            atomicMin(&bbox[4 * id + 1], y0);
            atomicMax(&bbox[4 * id + 2], x1);
            atomicMax(&bbox[4 * id + 3], y1);
        }
    }
}

__global__ void __launch_bounds__(kFT, 3) k_obj_feat(const int32_t* __restrict__ labels, int64_t lpitch,
                                                  const uint8_t* __restrict__ g, const uint8_t* __restrict__ edge,
                                                  int w, int h, const int32_t* __restrict__ cnt, int32_t cap,
                                                  const int32_t* __restrict__ rank_root,
                                                  const int32_t* __restrict__ bbox,
                                                  int32_t* __restrict__ out_label, int32_t* __restrict__ out_flags,
                                                  float* __restrict__ out_feat, int32_t capacity) {
    __shared__ FeatSmem fs;
    __shared__ TeamRed red;
    const TeamCTA<> team;
    const int n = min(*cnt, min(cap, capacity));
    for (int obj = blockIdx.x; obj < n; obj += gridDim.x) {
        const int32_t root = rank_root[obj];
        const int32_t lab = root + 1;
        auto inP = [&](int x, int y) {
            return x >= 0 && y >= 0 && x < w && y < h && labels[(int64_t)y * lpitch + x] == lab;
        };
        double* f = fs.f;
        int border = 0;
        object_features(team, inP, g, edge, w, h, bbox[4 * obj], bbox[4 * obj + 1], bbox[4 * obj + 2],
                        bbox[4 * obj + 3], fs, red, f, &border);
        if (threadIdx.x == 0) {
            out_label[obj] = lab;
            out_flags[obj] = border ? HP_OBJ_TOUCHES_BORDER : 0;
            for (int k = 0; k < HP_NFEAT; ++k) out_feat[(int64_t)obj * HP_NFEAT + k] = (float)f[k];
        }
        __syncthreads();
    }
}

__global__ void k_copy_count(const int32_t* __restrict__ cnt, int32_t* __restrict__ n_rows) { *n_rows = *cnt; }

}  // namespace

void launch_features(const int32_t* labels, int64_t lpitch, const uint8_t* g, const uint8_t* edge, int w, int h,
                     Slot& sl, int32_t max_objects, int32_t* row_label, int32_t* row_flags,
                     float* feat, int32_t capacity, int32_t* n_rows, cudaStream_t s) {
    const int64_t n = (int64_t)w * h;
    int32_t* cnt = sl.cnt32 + 2;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
    if (n > 0) {
        (note_launch(), k_obj_find<<<grid_for(n), 256, 0, s>>>(labels, lpitch, w, h, cnt, sl.obj_root, max_objects));
        (note_launch(), k_obj_rank<<<std::max(1, std::min(num_sms() * 4, (max_objects + 255) / 256)), 256, 0, s>>>(
            cnt, max_objects, sl.obj_root, sl.obj_rank, sl.aux));
        (note_launch(), k_bbox_init<<<std::max(1, std::min(num_sms() * 4, (max_objects + 255) / 256)), 256, 0, s>>>(cnt, max_objects, sl.obj_bbox));
        (note_launch(), k_obj_bbox<<<grid_for(n), 256, 0, s>>>(labels, lpitch, w, h, cnt, max_objects, sl.aux, sl.obj_bbox));
        (note_launch(), k_obj_feat<<<num_sms() * 8, kFT, 0, s>>>(labels, lpitch, g, edge, w, h, cnt, max_objects, sl.obj_rank,
                                           sl.obj_bbox, row_label, row_flags, feat, capacity));
    }
    (note_launch(), k_copy_count<<<1, 1, 0, s>>>(cnt, n_rows));
}

}  // namespace hp
