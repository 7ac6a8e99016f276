// k_cd.cu -- S1: colour deconvolution + pixel thresholds ("Color
// deconvolution"; thresholds of RBC detection PAPER.md:593-594; background PAPER.md:698-699).
//
// Per pixel: OD_k = LUT[v_k] (LUT built on the host in double, rounded once to float),
// c_H = fma(OD_B, q20, fma(OD_G, q10, OD_R*q00)) in exactly this order, g = clamp(rint(
// g_scale*c_H), 0, 255) (round-half-even), and four integer flag predicates.  HBM-bound:
// 3 B in, 2 B out per pixel.  Vector path: 16 pixels per thread, three 16-B loads of RGB and
// one 16-B store each for g and flags (coalesced, 128-bit); scalar path for unaligned input.
#include <cmath>

#include "cd_pixel.cuh"

namespace hp {

namespace {

__global__ void __launch_bounds__(256) k_cd_vec16(const uint8_t* __restrict__ rgb, int w, int h,
                                                  int64_t pitch, const float* __restrict__ lut_g,
                                                  CdConst k, uint8_t* __restrict__ g,
                                                  uint8_t* __restrict__ flags,
                                                  unsigned long long* bg_count) {
    __shared__ float lut[256];
    lut[threadIdx.x] = lut_g[threadIdx.x];
    __syncthreads();
    const int cpr = w >> 4;  // 16-pixel chunks per row
    const int64_t nchunks = (int64_t)cpr * h;
    int nbg = 0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nchunks;
         c += (int64_t)gridDim.x * blockDim.x) {
        int y = (int)(c / cpr), x0 = (int)(c - (int64_t)y * cpr) * 16;
        const uint4* src = reinterpret_cast<const uint4*>(rgb + y * pitch + 3 * x0);
        uint4 a = __ldcs(src), b = __ldcs(src + 1), cc = __ldcs(src + 2);
        uint32_t wv[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, cc.x, cc.y, cc.z, cc.w};
        uint8_t gb[16], fb[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            int o = 3 * i;
            // one PRMT per channel byte (a shift + mask pair otherwise)
            int R = (int)__byte_perm(wv[o >> 2], 0, 0x4440 | (o & 3));
            int G = (int)__byte_perm(wv[(o + 1) >> 2], 0, 0x4440 | ((o + 1) & 3));
            int B = (int)__byte_perm(wv[(o + 2) >> 2], 0, 0x4440 | ((o + 2) & 3));
            cd_pixel(R, G, B, lut, k, gb[i], fb[i], nbg);
        }
        uint4 go, fo;
        go.x = gb[0] | gb[1] << 8 | gb[2] << 16 | (uint32_t)gb[3] << 24;
        go.y = gb[4] | gb[5] << 8 | gb[6] << 16 | (uint32_t)gb[7] << 24;
        go.z = gb[8] | gb[9] << 8 | gb[10] << 16 | (uint32_t)gb[11] << 24;
        go.w = gb[12] | gb[13] << 8 | gb[14] << 16 | (uint32_t)gb[15] << 24;
        fo.x = fb[0] | fb[1] << 8 | fb[2] << 16 | (uint32_t)fb[3] << 24;
        fo.y = fb[4] | fb[5] << 8 | fb[6] << 16 | (uint32_t)fb[7] << 24;
        fo.z = fb[8] | fb[9] << 8 | fb[10] << 16 | (uint32_t)fb[11] << 24;
        fo.w = fb[12] | fb[13] << 8 | fb[14] << 16 | (uint32_t)fb[15] << 24;
        int64_t o = (int64_t)y * w + x0;
        *reinterpret_cast<uint4*>(g + o) = go;
        *reinterpret_cast<uint4*>(flags + o) = fo;
    }
    if (bg_count) block_count(nbg, bg_count);
}

__global__ void __launch_bounds__(256) k_cd_scalar(const uint8_t* __restrict__ rgb, int w, int h,
                                                   int64_t pitch, const float* __restrict__ lut_g,
                                                   CdConst k, uint8_t* __restrict__ g,
                                                   uint8_t* __restrict__ flags,
                                                   unsigned long long* bg_count) {
    __shared__ float lut[256];
    lut[threadIdx.x] = lut_g[threadIdx.x];
    __syncthreads();
    const int64_t n = (int64_t)w * h;
    int nbg = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
        const uint8_t* px = rgb + y * pitch + 3 * x;
        cd_pixel(px[0], px[1], px[2], lut, k, g[i], flags[i], nbg);
    }
    if (bg_count) block_count(nbg, bg_count);
}

}  // namespace

// OD(v) = log10(256 / (v + 1)) in double, rounded once to float (reading C3); OD(255) = +0.
void upload_od_lut(float* lut_dev, cudaStream_t s) {
    static float lut[256];
    for (int v = 0; v < 256; ++v) lut[v] = (float)std::log10(256.0 / (v + 1.0));
    cudaMemcpyAsync(lut_dev, lut, sizeof(lut), cudaMemcpyHostToDevice, s);
    cudaStreamSynchronize(s);
}

void launch_cd(const uint8_t* rgb, int w, int h, int64_t pitch, const float* lut,
               const hp_params& p, uint8_t* g, uint8_t* flags, unsigned long long* bg_count,
               cudaStream_t s) {
    CdConst k{p.q[0][0], p.q[1][0], p.q[2][0], p.g_scale, p.rbc_t1, p.rbc_t2, p.bg_rgb_min};
    if (bg_count) cudaMemsetAsync(bg_count, 0, sizeof(unsigned long long), s);
    const int64_t n = (int64_t)w * h;
    if (n == 0) return;
    bool vec = ((uintptr_t)rgb % 16 == 0) && (pitch % 16 == 0) && (w % 16 == 0) &&
               ((uintptr_t)g % 16 == 0) && ((uintptr_t)flags % 16 == 0);
    const int grid = num_sms() * 8;
    if (vec) {
        int64_t nchunks = n / 16;
        int blocks = (int)std::min<int64_t>((nchunks + 255) / 256, grid);
        (note_launch(), k_cd_vec16<<<blocks, 256, 0, s>>>(rgb, w, h, pitch, lut, k, g, flags, bg_count));
    } else {
        int blocks = (int)std::min<int64_t>((n + 255) / 256, grid);
        (note_launch(), k_cd_scalar<<<blocks, 256, 0, s>>>(rgb, w, h, pitch, lut, k, g, flags, bg_count));
    }
}

}  // namespace hp
