// register-only throughput of the fused kernel's product formulations (products per SM per clock)
#include <cstdio>
#include <cstdint>
#include "../../paper_2306_09189_b200/csrc/modarith.cuh"
using namespace fhe;
template <int MODE>
__global__ void k(uint64_t* out, int iters, uint64_t seed) {
    uint64_t a[4], b[4];
    for (int i = 0; i < 4; ++i) { a[i] = (seed * (threadIdx.x + 7 * i + 1)) & ((1ull << 60) - 1); b[i] = (a[i] * 0x9E3779B97F4A7C15ull) & ((1ull << 60) - 1); }
    Acc3 acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = Acc3{0, 0, 0, 0};
    U128 y[8];
    for (int i = 0; i < 8; ++i) y[i] = U128{0, 0};
    uint64_t s0[8], s1[8], s2[8];
    for (int i = 0; i < 8; ++i) s0[i] = s1[i] = s2[i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint64_t x = a[i & 3] ^ (uint64_t)it, w = b[(i + 1) & 3];
            if (MODE == 0) mac3(acc[i], x, w);
            if (MODE == 1) mac_small(y[i], x, w);
            if (MODE == 2) {  // 30-bit limbs in 32-bit halves: 4 mad.wide, no carries
                const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32);
                asm("mad.wide.u32 %0, %3, %5, %0;\n\tmad.wide.u32 %1, %3, %6, %1;\n\tmad.wide.u32 %1, %4, %5, %1;\n\tmad.wide.u32 %2, %4, %6, %2;"
                    : "+l"(s0[i]), "+l"(s1[i]), "+l"(s2[i]) : "r"(x0), "r"(x1), "r"(w0), "r"(w1));
            }
        }
    }
    uint64_t s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i].s0 + acc[i].s1 + acc[i].s2 + acc[i].c + y[i].lo + y[i].hi + s0[i] + s1[i] + s2[i];
    if (s == 42) out[0] = s;
}
template <int MODE> void run(const char* name, int sms, int clk, int threads, int bpsm) {
    uint64_t* o; cudaMalloc(&o, 8);
    const int iters = 2048, blocks = sms * bpsm;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<blocks, threads>>>(o, 16, 3); cudaDeviceSynchronize();
    float ms;
    cudaEventRecord(e0); k<MODE><<<blocks, threads>>>(o, iters, 3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double prods = (double)blocks * threads * iters * 8;
    printf("%-10s threads/SM %4d: %.2f T products/s = %.1f per SM per clk\n", name, threads * bpsm, prods / ms / 1e9, prods / (ms * 1e-3) / sms / (clk * 1e3));
}
int main() {
    int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int bp : {2, 4, 8}) {
        run<0>("mac3", sms, clk, 128, bp);
        run<1>("mac_small", sms, clk, 128, bp);
        run<2>("split30", sms, clk, 128, bp);
    }
    return 0;
}
