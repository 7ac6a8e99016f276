// probe: does cvt.rni.sat.u8.f32 (F2IP.U8) equal clamp(rint(x), 0, 255) for every float in
// [-2, 300] on a 1/64 grid (every .5 tie included) and at the extremes?
#include <cstdio>
#include <cmath>
__device__ __forceinline__ unsigned f2u8(float x) { unsigned r; asm("cvt.rni.sat.u8.f32 %0, %1;" : "=r"(r) : "f"(x)); return r; }
__global__ void k(const float* a, unsigned* o, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) o[i] = f2u8(a[i]);
}
int main() {
    const int n = (302 * 64) + 8;
    float* h = new float[n];
    unsigned* r = new unsigned[n];
    for (int i = 0; i < 302 * 64; ++i) h[i] = -2.0f + i / 64.0f;
    float ex[8] = {-0.0f, 0.49999997f, 0.50000006f, 254.49998f, 254.5f, 255.49998f, 1e30f, -1e30f};
    for (int i = 0; i < 8; ++i) h[302 * 64 + i] = ex[i];
    float* da; unsigned* dr;
    cudaMalloc(&da, n * 4); cudaMalloc(&dr, n * 4);
    cudaMemcpy(da, h, n * 4, cudaMemcpyHostToDevice);
    k<<<(n + 255) / 256, 256>>>(da, dr, n);
    cudaMemcpy(r, dr, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i) {
        float s = fminf(fmaxf(rintf(h[i]), 0.0f), 255.0f);
        if ((unsigned)s != r[i]) { if (bad < 10) printf("mismatch x=%.9g gpu=%u ref=%u\n", h[i], r[i], (unsigned)s); ++bad; }
    }
    printf("cvt_check: %d values, %d mismatches\n", n, bad);
    return bad != 0;
}
