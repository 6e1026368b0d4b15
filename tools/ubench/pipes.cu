// pipe throughput probe: IMAD.WIDE.U32 vs DFMA vs both interleaved
#include <cstdio>
#include <cstdint>
__global__ void k_imad(uint64_t* out, int iters, uint32_t x) {
    uint64_t a[8]; uint32_t b = threadIdx.x | 1, c = x;
    for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[i]) : "r"(b), "r"(c + i));
    }
    uint64_t s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 42) out[0] = s;
}
__global__ void k_imad32(uint64_t* out, int iters, uint32_t x) {
    uint32_t a[8]; uint32_t b = threadIdx.x | 1, c = x;
    for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b), "r"(c + i));
    }
    uint64_t s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 42) out[0] = s;
}
__global__ void k_dfma(uint64_t* out, int iters, double x) {
    double a[8]; double b = threadIdx.x * 1e-9 + 1.0;
    for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(a[i]) : "d"(b), "d"(x));
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 42) out[0] = 1;
}
__global__ void k_both(uint64_t* out, int iters, uint32_t x, double y) {
    uint64_t a[8]; uint32_t b = threadIdx.x | 1, c = x;
    double d[8]; double e = threadIdx.x * 1e-9 + 1.0;
    for (int i = 0; i < 8; ++i) { a[i] = i + threadIdx.x; d[i] = i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[i]) : "r"(b), "r"(c + i));
            asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(d[i]) : "d"(e), "d"(y));
        }
    }
    uint64_t s = 0; double t = 0; for (int i = 0; i < 8; ++i) { s += a[i]; t += d[i]; }
    if (s == 42 || t == 42) out[0] = s;
}
int main() {
    uint64_t* o; cudaMalloc(&o, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double ops = (double)blocks * threads * iters * 8;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0); k_imad<<<blocks, threads>>>(o, iters, 3); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("IMAD.WIDE: %.2f T/s  (%.1f per SM per clk at %d MHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        cudaEventRecord(e0); k_imad32<<<blocks, threads>>>(o, iters, 3); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("IMAD 32  : %.2f T/s  (%.1f per SM per clk)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
        cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(o, iters, 1e-12); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DFMA     : %.2f T/s  (%.1f per SM per clk)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
        cudaEventRecord(e0); k_both<<<blocks, threads>>>(o, iters, 3, 1e-12); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("BOTH     : %.2f T pairs/s (%.1f pairs per SM per clk)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
