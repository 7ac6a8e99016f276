// cd_pixel.cuh -- S1's per-pixel arithmetic (PAPER.md:637-639 colour deconvolution; RBC
// thresholds PAPER.md:593-594; background PAPER.md:698-699), shared by the raw-RGB kernel
// (k_cd.cu) and the JPEG ingest kernel that fuses decoding into S1 (k_jpeg.cu), so both
// produce the same g and flags bit for bit.
#pragma once

#include "hp_internal.cuh"

namespace hp {

struct CdConst {
    float q00, q10, q20, gs;
    int t1, t2, bgmin;
};

inline CdConst cd_const(const hp_params& p) {
    return CdConst{p.q[0][0], p.q[1][0], p.q[2][0], p.g_scale, p.rbc_t1, p.rbc_t2, p.bg_rgb_min};
}

// round to nearest even, then saturate to [0, 255]: one F2IP.U8 instead of FRND + 2 FMNMX +
// F2I (equal to clamp(rint(x), 0, 255) for every finite x; tools/probe/cvt_check.cu checks it
// on the GPU over [-2, 300] in 1/64 steps, every .5 tie included)
__device__ __forceinline__ uint32_t rint_sat_u8(float x) {
    uint32_t r;
    asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// c_H = fma(OD_B, q20, fma(OD_G, q10, OD_R*q00)) in exactly this order (reading C6),
// g = clamp(rint(g_scale * c_H), 0, 255) (round half even), four integer flag predicates
__device__ __forceinline__ void cd_pixel(int R, int G, int B, const float* lut, const CdConst& k,
                                         uint8_t& gout, uint8_t& fout, int& nbg) {
    float cH = __fmaf_rn(lut[B], k.q20, __fmaf_rn(lut[G], k.q10, __fmul_rn(lut[R], k.q00)));
    gout = (uint8_t)rint_sat_u8(__fmul_rn(cH, k.gs));
    uint8_t f = 0;
    if (R > k.t1 * G) f |= HP_FLAG_RBC_HI;
    if (R > k.t2 * G) f |= HP_FLAG_RBC_LO;
    if (R > B) f |= HP_FLAG_R_GT_B;
    if (min(R, min(G, B)) > k.bgmin) {
        f |= HP_FLAG_BG;
        ++nbg;
    }
    fout = f;
}

__device__ __forceinline__ void block_count(int nbg, unsigned long long* out) {
    // warp reduce, one atomic per warp
    unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)nbg);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, (unsigned long long)v);
}

}  // namespace hp
