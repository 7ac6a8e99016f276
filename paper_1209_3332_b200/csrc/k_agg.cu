// k_agg.cu -- per-image feature aggregation: a segmented
// fp64 reduction of feature rows, one block per group, every thread owning a fixed set of
// rows and the block combining its partials by a fixed tree -- deterministic.  The rows of a
// group are contiguous (a rank's table is in tile order and tiles map to slides in order).
#include <algorithm>

#include "hp_internal.cuh"

namespace hp {
namespace {

constexpr int kAT = 256;  // threads per group block
constexpr int kAF = 9;    // features per pass (HP_NFEAT = 36 -> 4 passes; 39 KB of shared memory)

// kCentered = false: per group and feature the sum and the sum of squares of the rows;
// kCentered = true (second pass): mean = sum / count from the (all-reduced) first-pass sums,
// then the sum of squared deviations from that mean, so the variance is never formed as the
// cancellation-prone E[x^2] - mean^2.  Both write [G][36][2]: (sum, sumsq) or (mean, m2).
template <bool kCentered>
__global__ void __launch_bounds__(kAT) k_reduce_rows(const float* __restrict__ feat, const int64_t* __restrict__ off,
                                                     const double* __restrict__ sums,
                                                     const int64_t* __restrict__ gcount,
                                                     double* __restrict__ out, int64_t* __restrict__ count) {
    __shared__ double red[kAT][2 * kAF + 1];  // (+1: no bank conflicts between threads)
    __shared__ double mean_s[HP_NFEAT];
    const int gi = blockIdx.x;
    const int64_t r0 = off[gi], r1 = off[gi + 1];
    if (!kCentered && threadIdx.x == 0) count[gi] = r1 - r0;
    if (kCentered && threadIdx.x < HP_NFEAT) {
        const int64_t n = gcount[gi];
        mean_s[threadIdx.x] = n > 0 ? sums[((int64_t)gi * HP_NFEAT + threadIdx.x) * 2] / (double)n : __longlong_as_double(0x7ff8000000000000LL);
    }
    __syncthreads();
    for (int f0 = 0; f0 < HP_NFEAT; f0 += kAF) {
        double s[kAF], q[kAF];
#pragma unroll
        for (int k = 0; k < kAF; ++k) s[k] = q[k] = 0.0;
        for (int64_t r = r0 + threadIdx.x; r < r1; r += kAT) {
            const float* row = feat + r * HP_NFEAT + f0;
#pragma unroll
            for (int k = 0; k < kAF; ++k) {
                const double v = kCentered ? (double)row[k] - mean_s[f0 + k] : (double)row[k];
                s[k] += v;
                q[k] += v * v;
            }
        }
#pragma unroll
        for (int k = 0; k < kAF; ++k) {
            red[threadIdx.x][2 * k] = s[k];
            red[threadIdx.x][2 * k + 1] = q[k];
        }
        __syncthreads();
        for (int half = kAT / 2; half > 0; half >>= 1) {  // fixed pairwise tree
            if (threadIdx.x < half)
                for (int k = 0; k < 2 * kAF; ++k) red[threadIdx.x][k] += red[threadIdx.x + half][k];
            __syncthreads();
        }
        if (threadIdx.x < 2 * kAF) {
            const int k = threadIdx.x / 2, which = threadIdx.x & 1;
            double v = red[0][threadIdx.x];
            if (kCentered && which == 0) v = mean_s[f0 + k];
            out[((int64_t)gi * HP_NFEAT + f0 + k) * 2 + which] = v;
        }
        __syncthreads();
    }
}

// std = sqrt(m2 / count) (population), NaN for an empty group; mean passes through.
__global__ void k_group_std(const double* __restrict__ mm2, const int64_t* __restrict__ gcount, int32_t n_groups,
                            double* __restrict__ mean_out, double* __restrict__ std_out) {
    const int64_t n = (int64_t)n_groups * HP_NFEAT;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = gcount[i / HP_NFEAT];
        mean_out[i] = mm2[2 * i];
        std_out[i] = c > 0 ? sqrt(mm2[2 * i + 1] / (double)c) : __longlong_as_double(0x7ff8000000000000LL);
    }
}

}  // namespace

void launch_reduce_rows(const float* feat, const int64_t* off, int32_t n_groups, double* out, int64_t* count,
                        cudaStream_t s) {
    static_assert(HP_NFEAT % kAF == 0, "features per pass");
    if (n_groups == 0) return;
    (note_launch(), k_reduce_rows<false><<<n_groups, kAT, 0, s>>>(feat, off, nullptr, nullptr, out, count));
}

void launch_group_center(const float* feat, const int64_t* off, int32_t n_groups, const double* sums,
                         const int64_t* count, double* mean_m2, cudaStream_t s) {
    if (n_groups == 0) return;
    (note_launch(), k_reduce_rows<true><<<n_groups, kAT, 0, s>>>(feat, off, sums, count, mean_m2, nullptr));
}

void launch_group_std(const double* mean_m2, const int64_t* count, int32_t n_groups, double* mean, double* std_out,
                      cudaStream_t s) {
    if (n_groups == 0) return;
    const int grid = std::max(1, std::min(num_sms(), (int)(((int64_t)n_groups * HP_NFEAT + 255) / 256)));
    (note_launch(), k_group_std<<<grid, 256, 0, s>>>(mean_m2, count, n_groups, mean, std_out));
}

}  // namespace hp

// ---------------------------------------------------------------- device row arena (S12)
// hp_run_tiles with an hp_row_arena: the tile's rows stay on the device and are appended as
// one run.  Two launches in the slot's chain (both captured in its graph): one thread
// reserves the run (one atomicAdd on the caller's cursor) and records the offset; then a
// grid copies the rows, coalesced, clipped to the arena's capacity.
namespace hp {
namespace {

__global__ void k_arena_reserve(const int32_t* __restrict__ nrows, int32_t tab_cap, int64_t* cursor,
                                int64_t* __restrict__ base) {
    const int64_t n = min(*nrows, tab_cap);
    *base = (int64_t)atomicAdd((unsigned long long*)cursor, (unsigned long long)n);
}

__global__ void k_arena_copy(const int32_t* __restrict__ nrows, int32_t tab_cap, const int32_t* __restrict__ lab,
                             const int32_t* __restrict__ fl, const float* __restrict__ feat,
                             const int64_t* __restrict__ base_p, const int64_t* __restrict__ tile_id,
                             hp_row_arena a) {
    const int64_t n = min(*nrows, tab_cap);
    const int64_t base = *base_p;
    const int64_t m = max((int64_t)0, min(n, a.capacity - base));  // rows that fit
    const int64_t tid = *tile_id;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        a.tile[base + i] = tid;
        a.label[base + i] = lab[i];
        a.flags[base + i] = fl[i];
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m * HP_NFEAT; i += stride)
        a.feat[base * HP_NFEAT + i] = feat[i];
}

}  // namespace

void launch_arena_append(const int32_t* nrows, int32_t tab_cap, const int32_t* lab, const int32_t* fl,
                         const float* feat, int64_t* base, const int64_t* tile_id, const hp_row_arena& a,
                         cudaStream_t s) {
    (note_launch(), k_arena_reserve<<<1, 1, 0, s>>>(nrows, tab_cap, a.cursor, base));
    const int grid = std::max(1, std::min(num_sms(), (int)(((int64_t)tab_cap * HP_NFEAT + 1023) / 1024)));
    (note_launch(), k_arena_copy<<<grid, 256, 0, s>>>(nrows, tab_cap, lab, fl, feat, base, tile_id, a));
}

}  // namespace hp
