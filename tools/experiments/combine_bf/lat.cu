// Dependent-chain latency of the spine combine's building blocks on sm_100a
// (one warp, clock64 around 1024 dependent ops).
#include <cstdio>
#include <cstdint>
#define N 1024
__global__ void k(float* out, long long* cyc, float a0) {
    float2 x = make_float2(a0, a0 * 1.5f);
    float y = a0;
    unsigned u = __float_as_uint(a0);
    long long t0, t1;
    // FFMA2 chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 8; ++i) {
        asm volatile("{.reg .b64 X, B; mov.b64 X, {%0, %1}; mov.b64 B, {%2, %2};"
                     "fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B;"
                     "fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B; fma.rn.f32x2 X, X, B, B;"
                     "mov.b64 {%0, %1}, X;}" : "+f"(x.x), "+f"(x.y) : "f"(0.5f));
    }
    t1 = clock64(); cyc[0] = t1 - t0;
    // FFMA chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 8; ++i) {
        asm volatile("fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1;"
                     "fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1; fma.rn.f32 %0, %0, %1, %1;"
                     : "+f"(y) : "f"(0.5f));
    }
    t1 = clock64(); cyc[1] = t1 - t0;
    // MUFU.RCP chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 8; ++i) {
        asm volatile("rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0;"
                     "rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0; rcp.approx.ftz.f32 %0, %0;"
                     : "+f"(y));
    }
    t1 = clock64(); cyc[2] = t1 - t0;
    // LOP3 chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 8; ++i) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2;"
                     "lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2; lop3.b32 %0, %0, %1, %2, 0xE2;"
                     : "+r"(u) : "r"(0xffff0000u), "r"(0x1234u));
    }
    t1 = clock64(); cyc[3] = t1 - t0;
    // FFMA2 -> LOP3 (x component) mixed chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 2; ++i) {
        asm volatile("{.reg .b64 X, B; .reg .b32 lo, hi; mov.b64 X, {%0, %1}; mov.b64 B, {%2, %2};"
                     "fma.rn.f32x2 X, X, B, B; mov.b64 {lo, hi}, X; lop3.b32 lo, lo, %3, %4, 0xE2; lop3.b32 hi, hi, %3, %4, 0xE2;"
                     "mov.b64 X, {lo, hi}; mov.b64 {%0, %1}, X;}" : "+f"(x.x), "+f"(x.y) : "f"(0.5f), "r"(0xffffffffu), "r"(0u));
    }
    t1 = clock64(); cyc[4] = t1 - t0;
    // MUFU.RCP -> FFMA2 (the o / D entry)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N / 2; ++i) {
        asm volatile("{.reg .b64 X, B, R; .reg .f32 rx, ry; mov.b64 X, {%0, %1}; mov.b64 B, {%2, %2};"
                     "rcp.approx.ftz.f32 rx, %0; rcp.approx.ftz.f32 ry, %1; mov.b64 R, {rx, ry};"
                     "fma.rn.f32x2 X, R, B, B; mov.b64 {%0, %1}, X;}" : "+f"(x.x), "+f"(x.y) : "f"(0.5f));
    }
    t1 = clock64(); cyc[5] = t1 - t0;
    out[threadIdx.x] = x.x + x.y + y + __uint_as_float(u);
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
    for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, c, 1.1f); cudaDeviceSynchronize(); }
    const char* nm[] = {"FFMA2", "FFMA", "MUFU.RCP", "LOP3", "FFMA2+LOP3 (pair)", "MUFU.RCP+FFMA2 (pair)"};
    const int per[] = {N, N, N, N, N / 2, N / 2};
    for (int i = 0; i < 6; ++i) printf("%-24s %.2f cycles per dependent step\n", nm[i], (double)c[i] / per[i]);
    return 0;
}
