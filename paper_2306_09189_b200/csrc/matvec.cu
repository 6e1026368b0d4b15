// Plaintext mat-vec kernels of the classic BSGS schedules (approaches 3 / 4): Y_g = sum_b pt[g][b] * X~_b.
// Their own translation unit, so the four units of the library compile side by side (build.py).
#include "kernels.cuh"

namespace fhe {

int mv_cap();  // kernels.cu

namespace {

// volatile (non-reorderable) 16-byte loads: issued in program order so that a
// whole batch of independent loads is in flight before the first use
__device__ __forceinline__ ulonglong2 vld2_nc(const uint64_t* p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ ulonglong2 vld2_cs(const uint64_t* p) {
    ulonglong2 r;
    asm volatile("ld.global.cs.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ void st2(uint64_t* p, uint64_t a, uint64_t b) {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(a, b);
}

// batched plaintext mat-vec: Y[s][g] = sum_b pt[g][b] * XT[s][b] (item = (pair, source),
// the sources of a pair share every plaintext load)
__global__ void __launch_bounds__(128) k_pt_matvec_b(DevCtx c, uint64_t* Y, size_t y_src_stride, const uint64_t* XT,
                                                     size_t xt_src_stride, BabyTerms t, int level, int nsrc) {
    extern __shared__ ulonglong2 xs[];  // [nb][2][128]
    const int ne = level + 1 + c.K;
    const size_t total = (size_t)ne * c.N;
    const size_t items = (total / 2) * nsrc;
    RowMap rm{ne, level, c.L, 0};
    const int tid = threadIdx.x;
    for (size_t it = blockIdx.x * (size_t)blockDim.x + tid; it < items; it += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(it % nsrc);
        const size_t i = (it / nsrc) * 2;
        const int u = (int)(i >> c.logN);
        const Prime pr = c.primes[row_prime(rm, u)];
        const uint64_t* xts = XT + (size_t)s * xt_src_stride;
        for (int b = 0; b < t.nb; ++b) {
            if (t.gmask[b] == 0) continue;
            xs[(b * 2 + 0) * 128 + tid] = vld2_cs(xts + (size_t)b * 2 * total + i);
            xs[(b * 2 + 1) * 128 + tid] = vld2_cs(xts + (size_t)b * 2 * total + total + i);
        }
        for (int g = 0; g < t.ngi; ++g) {
            U128 a0[2] = {{0, 0}, {0, 0}}, a1[2] = {{0, 0}, {0, 0}};
            const uint64_t* pg = t.pts + ((size_t)(t.g0 + g) * t.nb_total) * total + i;
            int b = 0;
            for (; b + 4 <= t.nb; b += 4) {
                ulonglong2 w[4];
#pragma unroll
                for (int d = 0; d < 4; ++d)
                    w[d] = ((t.gmask[b + d] >> g) & 1u) ? vld2_nc(pg + (size_t)(b + d) * total) : make_ulonglong2(0, 0);
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const ulonglong2 x0 = xs[((b + d) * 2 + 0) * 128 + tid];
                    const ulonglong2 x1 = xs[((b + d) * 2 + 1) * 128 + tid];
                    mac(a0[0], w[d].x, x0.x);
                    mac(a0[1], w[d].y, x0.y);
                    mac(a1[0], w[d].x, x1.x);
                    mac(a1[1], w[d].y, x1.y);
                }
            }
            for (; b < t.nb; ++b) {
                if (!((t.gmask[b] >> g) & 1u)) continue;
                const ulonglong2 w = vld2_nc(pg + (size_t)b * total);
                const ulonglong2 x0 = xs[(b * 2 + 0) * 128 + tid];
                const ulonglong2 x1 = xs[(b * 2 + 1) * 128 + tid];
                mac(a0[0], w.x, x0.x);
                mac(a0[1], w.y, x0.y);
                mac(a1[0], w.x, x1.x);
                mac(a1[1], w.y, x1.y);
            }
            uint64_t* y = Y + (size_t)s * y_src_stride + (size_t)g * 2 * total;
            st2(y + i, reduce128(a0[0].hi, a0[0].lo, pr), reduce128(a0[1].hi, a0[1].lo, pr));
            st2(y + total + i, reduce128(a1[0].hi, a1[0].lo, pr), reduce128(a1[1].hi, a1[1].lo, pr));
        }
    }
}

// Plaintext mat-vec on coefficient pairs: the baby-step terms X~_b of the
// thread's pair are staged once in private shared-memory slots, then every
// giant accumulator streams its plaintexts with 16-byte loads.
constexpr int kMatvecThreads = 128;
__global__ void __launch_bounds__(kMatvecThreads) k_pt_matvec2(DevCtx c, uint64_t* Y, const uint64_t* XT,
                                                               BabyTerms t, int level) {
    extern __shared__ ulonglong2 xs[];  // [nb][2][kMatvecThreads]
    const int ne = level + 1 + c.K;
    const size_t total = (size_t)ne * c.N;
    RowMap rm{ne, level, c.L, 0};
    const int tid = threadIdx.x;
    for (size_t ip = blockIdx.x * (size_t)blockDim.x + tid; ip < total / 2; ip += (size_t)gridDim.x * blockDim.x) {
        const size_t i = ip * 2;
        const int u = (int)(i >> c.logN);
        const Prime pr = c.primes[row_prime(rm, u)];
        for (int b = 0; b < t.nb; ++b) {
            if (t.gmask[b] == 0) continue;
            xs[(b * 2 + 0) * kMatvecThreads + tid] = vld2_cs(XT + (size_t)b * 2 * total + i);
            xs[(b * 2 + 1) * kMatvecThreads + tid] = vld2_cs(XT + (size_t)b * 2 * total + total + i);
        }
        for (int g = 0; g < t.ngi; ++g) {
            U128 a0[2] = {{0, 0}, {0, 0}}, a1[2] = {{0, 0}, {0, 0}};
            const uint64_t* pg = t.pts + ((size_t)(t.g0 + g) * t.nb_total) * total + i;
            int b = 0;
            for (; b + 4 <= t.nb; b += 4) {
                ulonglong2 w[4];
#pragma unroll
                for (int d = 0; d < 4; ++d)
                    w[d] = ((t.gmask[b + d] >> g) & 1u) ? vld2_cs(pg + (size_t)(b + d) * total) : make_ulonglong2(0, 0);
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const ulonglong2 x0 = xs[((b + d) * 2 + 0) * kMatvecThreads + tid];
                    const ulonglong2 x1 = xs[((b + d) * 2 + 1) * kMatvecThreads + tid];
                    mac(a0[0], w[d].x, x0.x);
                    mac(a0[1], w[d].y, x0.y);
                    mac(a1[0], w[d].x, x1.x);
                    mac(a1[1], w[d].y, x1.y);
                }
            }
            for (; b < t.nb; ++b) {
                if (!((t.gmask[b] >> g) & 1u)) continue;
                const ulonglong2 w = vld2_cs(pg + (size_t)b * total);
                const ulonglong2 x0 = xs[(b * 2 + 0) * kMatvecThreads + tid];
                const ulonglong2 x1 = xs[(b * 2 + 1) * kMatvecThreads + tid];
                mac(a0[0], w.x, x0.x);
                mac(a0[1], w.y, x0.y);
                mac(a1[0], w.x, x1.x);
                mac(a1[1], w.y, x1.y);
            }
            uint64_t* y = Y + (size_t)g * 2 * total;
            st2(y + i, reduce128(a0[0].hi, a0[0].lo, pr), reduce128(a0[1].hi, a0[1].lo, pr));
            st2(y + total + i, reduce128(a1[0].hi, a1[0].lo, pr), reduce128(a1[1].hi, a1[1].lo, pr));
        }
    }
}

}  // namespace

void pt_matvec_batch(const DevCtx& c, uint64_t* Y, size_t y_src_stride, const uint64_t* XT, size_t xt_src_stride,
                     const BabyTerms& t, int level, int nsrc, cudaStream_t st) {
    const size_t items = (size_t)(level + 1 + c.K) * c.N / 2 * nsrc;
    const size_t smem = (size_t)t.nb * 2 * 128 * sizeof(ulonglong2);
    const int blocks = (int)((items + 127) / 128 < 148 * 12 ? (items + 127) / 128 : 148 * 12);
    note_launch(1);
    cudaFuncSetAttribute(k_pt_matvec_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pt_matvec_b<<<blocks, 128, smem, st>>>(c, Y, y_src_stride, XT, xt_src_stride, t, level, nsrc);
}

void pt_matvec(const DevCtx& c, uint64_t* Y, const uint64_t* XT, const BabyTerms& t, int level, cudaStream_t st) {
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    const size_t smem = (size_t)t.nb * 2 * kMatvecThreads * sizeof(ulonglong2);
    int blocks = (int)((total / 2 + kMatvecThreads - 1) / kMatvecThreads);
    blocks = blocks < mv_cap() ? blocks : mv_cap();
    note_launch(1);
    cudaFuncSetAttribute(k_pt_matvec2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_pt_matvec2<<<blocks, kMatvecThreads, smem, st>>>(c, Y, XT, t, level);
}

}  // namespace fhe
