// micro-benchmark: butterfly throughput in registers (no memory traffic)
#include <cstdio>
#include <cstdint>
#include "../../paper_2306_09189_b200/csrc/modarith.cuh"
using namespace fhe;
template <int MODE>
__global__ void kbf(uint64_t* out, const uint64_t* tw, uint64_t q, int rounds) {
    uint64_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = (threadIdx.x * 16 + i) % q;
    const uint64_t q2 = 2 * q;
    uint64_t w = tw[0], ws = tw[1];
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k & h) continue;
                if (MODE == 0) {
                    uint64_t U = v[k];
                    U = U >= q2 ? U - q2 : U;
                    const uint64_t V = mul_shoup_lazy(v[k + h], w, ws, q);
                    v[k] = U + V;
                    v[k + h] = U - V + q2;
                } else {
                    const uint64_t U = v[k], V = v[k + h];
                    const uint64_t T = U + V;
                    v[k] = T >= q2 ? T - q2 : T;
                    v[k + h] = mul_shoup_lazy(U - V + q2, w, ws, q);
                }
            }
            w += 2; ws += 3;
        }
    }
    uint64_t s = 0;
    for (int i = 0; i < 16; ++i) s ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint64_t *out, *tw;
    cudaMalloc(&out, 148 * 64 * 256 * 8);
    cudaMalloc(&tw, 16);
    uint64_t h[2] = {123456789, 987654321};
    cudaMemcpy(tw, h, 16, cudaMemcpyHostToDevice);
    const uint64_t q = (1ULL << 50) - 27;
    for (int mode = 0; mode < 2; ++mode) {
        for (int bpsm : {2, 4, 8}) {
            const int blocks = 148 * bpsm, rounds = 200;
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            mode == 0 ? kbf<0><<<blocks, 256>>>(out, tw, q, 10) : kbf<1><<<blocks, 256>>>(out, tw, q, 10);
            cudaEventRecord(a);
            mode == 0 ? kbf<0><<<blocks, 256>>>(out, tw, q, rounds) : kbf<1><<<blocks, 256>>>(out, tw, q, rounds);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double bfs = (double)blocks * 256 * rounds * 32;  // 4 stages x 8 butterflies
            printf("mode %d blocks/SM %d: %.1f G butterflies/s  (N=2^15 row-NTT equiv %.3f us)\n", mode, bpsm,
                   bfs / ms / 1e6, 245760.0 / (bfs / ms / 1e3) * 1e6);
        }
    }
    return 0;
}
