// sm_100a kernels of the RNS-CKKS encrypted-convolution hot path.
//
// Layout: residues are uint64 in [0, q), one row of N words
// per (poly, prime), rows contiguous ([poly][prime][N]); NTT rows are in
// bit-reversed evaluation order, so every Galois automorphism maps aligned
// 2^b blocks to aligned 2^b blocks and the permuted gathers below stay
// inside 256-byte segments.
#include <stdexcept>
#include <type_traits>

#include "kernels.cuh"

// k_bsgs_tma FP64 rows: read a digit pair with one 16-byte shared load and swap in
// registers (1), or as two 8-byte loads in output order (0)
#ifndef FHE_TMA_NOSYNC
// k_bsgs_tma with 1: stages refilled by the last warp to leave them, no CTA barrier per baby step.
// Off: cfg3 batch 16 loses 7 % (2132 -> 1985 conv/s, profiles/ab_r02_bsgs_variants.txt) -- warps
// that drift apart contend for shared memory instead of overlapping their phases.
#define FHE_TMA_NOSYNC 0
#endif
#ifndef FHE_DIG128
#define FHE_DIG128 0
#endif

#ifndef FHE_FUSED_UNROLL2  // fused kernel: two baby steps per loop iteration (constant stage offsets)
#define FHE_FUSED_UNROLL2 1
#endif
#ifndef FHE_FUSED_SPLITLD  // fused kernel: digit / c0 pairs as two 8-byte loads in output order
#define FHE_FUSED_SPLITLD 1
#endif
#include "cdt_table.h"

namespace fhe {

uint64_t g_launches = 0;  // every kernel this library enqueues (host-side count)
void note_launch(int n) { g_launches += n; }

namespace {

constexpr int kEwThreads = 256;

inline int ew_blocks(size_t n) {
    size_t b = (n + kEwThreads - 1) / kEwThreads;
    const size_t cap = 148 * 16;
    return (int)(b < cap ? b : cap);
}

__device__ __forceinline__ uint32_t brev_n(uint32_t x, int logN) { return __brev(x) >> (32 - logN); }

// index j with (2 brv(j) + 1) = (2 brv(k) + 1) g mod 2N
__device__ __forceinline__ uint32_t perm_index(uint32_t k, uint32_t g, int logN) {
    const uint32_t e = 2 * brev_n(k, logN) + 1;
    const uint32_t e2 = (e * g) & ((2u << logN) - 1);
    return brev_n((e2 - 1) >> 1, logN);
}

}  // namespace

// ------------------------------------------------------------ sampling
namespace {

__constant__ uint64_t c_cdt[FHE_CDT_LEN] = {FHE_CDT_VALUES};

__global__ void k_reduce_signed_rows(DevCtx c, const int64_t* coef, uint64_t* out, int nrows, RowMap rm) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int k = (int)(i & (size_t)(c.N - 1));
        const Prime pr = c.primes[row_prime(rm, r % rm.rows_per_poly)];
        out[i] = reduce_signed(coef[k], pr);
    }
}

__global__ void k_sample_uniform(DevCtx c, uint64_t* out, int nrows, RowMap rm, uint64_t key) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int k = (int)(i & (size_t)(c.N - 1));
        const int p = row_prime(rm, r % rm.rows_per_poly);
        const uint64_t ctr = 2 * ((uint64_t)p * c.N + k);
        out[i] = uniform_mod(prng_k(key, ctr), prng_k(key, ctr + 1), c.primes[p]);
    }
}

__global__ void k_sample_gauss(DevCtx c, int64_t* out, uint64_t key) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < c.N; k += gridDim.x * blockDim.x) {
        const uint64_t r63 = prng_k(key, (uint64_t)k) >> 1;
        int64_t x = -20;
#pragma unroll
        for (int t = 0; t < FHE_CDT_LEN; ++t) x += (r63 >= c_cdt[t]) ? 1 : 0;
        out[k] = x;
    }
}

__global__ void k_sample_ternary(DevCtx c, int64_t* out, uint64_t key) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < c.N; k += gridDim.x * blockDim.x) {
        const uint64_t r = prng_k(key, (uint64_t)k);
        out[k] = (int64_t)mulhi64(r, 3) - 1;
    }
}

__global__ void k_keygen_combine(DevCtx c, uint64_t* b, const uint64_t* a, const uint64_t* e, const uint64_t* s,
                                 uint32_t galois, int lo, int hi, const ModDownTable* md, int nrows,
                                 const uint64_t* target) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const Prime pr = c.primes[t];
        uint64_t v = sub_mod(e[i], mul_mod(a[i], s[i], pr), pr.q);
        if (t >= lo && t < hi) {
            // switching target: sigma_g(s) for Galois keys, the given rows (s^2) for relinearisation
            const uint64_t sp = target ? target[i] : s[(size_t)t * c.N + perm_index(k, galois, c.logN)];
            v = add_mod(v, mul_shoup(sp, md->pmod[t], md->pmod_sh[t], pr.q), pr.q);
        }
        b[i] = v;
    }
}

__global__ void k_encrypt_combine(DevCtx c, uint64_t* c0, const uint64_t* c1, const uint64_t* e,
                                  const uint64_t* s, const uint64_t* pt, int nrows) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const Prime pr = c.primes[(i >> c.logN)];
        const uint64_t v = sub_mod(e[i], mul_mod(c1[i], s[i], pr), pr.q);
        c0[i] = add_mod(v, pt[i], pr.q);
    }
}

__global__ void k_decrypt_combine(DevCtx c, uint64_t* m, const uint64_t* c0, const uint64_t* c1,
                                  const uint64_t* s, int nrows) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const Prime pr = c.primes[(i >> c.logN)];
        m[i] = add_mod(c0[i], mul_mod(c1[i], s[i], pr), pr.q);
    }
}

}  // namespace

void reduce_signed_rows(const DevCtx& c, const int64_t* coef, uint64_t* out, int nrows, const RowMap& rm,
                        cudaStream_t st) {
    ++g_launches;
    k_reduce_signed_rows<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, coef, out, nrows, rm);
}
void sample_uniform_rows(const DevCtx& c, uint64_t* out, int nrows, const RowMap& rm, uint64_t key,
                         cudaStream_t st) {
    ++g_launches;
    k_sample_uniform<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, out, nrows, rm, key);
}
void sample_gauss(const DevCtx& c, int64_t* out, uint64_t key, cudaStream_t st) {
    ++g_launches;
    k_sample_gauss<<<ew_blocks(c.N), kEwThreads, 0, st>>>(c, out, key);
}
void sample_ternary(const DevCtx& c, int64_t* out, uint64_t key, cudaStream_t st) {
    ++g_launches;
    k_sample_ternary<<<ew_blocks(c.N), kEwThreads, 0, st>>>(c, out, key);
}
void keygen_combine(const DevCtx& c, uint64_t* key_b, const uint64_t* key_a, const uint64_t* e,
                    const uint64_t* s, uint32_t galois, int lo, int hi, const ModDownTable* md, int nrows,
                    cudaStream_t st, const uint64_t* target) {
    ++g_launches;
    k_keygen_combine<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, key_b, key_a, e, s, galois, lo,
                                                                              hi, md, nrows, target);
}

// ct x ct tensor product in the NTT domain: d0 = a0 b0, d1 = a0 b1 + a1 b0,
// d2 = a1 b1 (rows 0..level of each polynomial; d = [3][level+1][N])
__global__ void k_tensor(DevCtx c, uint64_t* d, const uint64_t* a, const uint64_t* b, int nr) {
    const size_t pw = (size_t)nr * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < pw; i += (size_t)gridDim.x * blockDim.x) {
        const Prime pr = c.primes[i >> c.logN];
        const uint64_t a0 = a[i], a1 = a[pw + i], b0 = b[i], b1 = b[pw + i];
        d[i] = mul_mod(a0, b0, pr);
        d[pw + i] = add_mod(mul_mod(a0, b1, pr), mul_mod(a1, b0, pr), pr.q);
        d[2 * pw + i] = mul_mod(a1, b1, pr);
    }
}
void tensor(const DevCtx& c, uint64_t* d, const uint64_t* a, const uint64_t* b, int level, cudaStream_t st) {
    ++g_launches;
    k_tensor<<<ew_blocks((size_t)(level + 1) * c.N), kEwThreads, 0, st>>>(c, d, a, b, level + 1);
}
void encrypt_combine(const DevCtx& c, uint64_t* c0, const uint64_t* c1, const uint64_t* e,
                     const uint64_t* s, const uint64_t* pt, int nrows, cudaStream_t st) {
    ++g_launches;
    k_encrypt_combine<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, c0, c1, e, s, pt, nrows);
}
void decrypt_combine(const DevCtx& c, uint64_t* m, const uint64_t* c0, const uint64_t* c1,
                     const uint64_t* s, int nrows, cudaStream_t st) {
    ++g_launches;
    k_decrypt_combine<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, m, c0, c1, s, nrows);
}

// ---------------------------------------------------------- elementwise
namespace {

template <int OP>
__global__ void k_ew(DevCtx c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp) {
    const size_t total = (size_t)nrows * c.N;
    const size_t polyw = (size_t)rpp * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int u = (int)((i >> c.logN) % rpp);
        const Prime pr = c.primes[u];
        if (OP == 0) out[i] = add_mod(a[i], b[i], pr.q);
        if (OP == 1) out[i] = sub_mod(a[i], b[i], pr.q);
        if (OP == 2) out[i] = mul_mod(a[i], b[i % polyw], pr);
    }
}

// per-prime constant (the NTT of a constant polynomial is that constant everywhere):
// MODE 0 adds k_u to poly 0 and copies poly 1; MODE 1 multiplies both polys by k_u
template <int MODE>
__global__ void k_ew_const(DevCtx c, uint64_t* out, const uint64_t* a, RowConsts k, int nr) {
    const size_t total = (size_t)2 * nr * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int u = r % nr;
        const Prime pr = c.primes[u];
        if (MODE == 0) out[i] = r < nr ? add_mod(a[i], k.v[u], pr.q) : a[i];
        if (MODE == 1) out[i] = mul_mod(a[i], k.v[u], pr);
    }
}

__global__ void k_automorph(DevCtx c, uint64_t* out, const uint64_t* in, int nrows, uint32_t g) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t r = i >> c.logN;
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        out[i] = in[r * c.N + perm_index(k, g, c.logN)];
    }
}

__global__ void k_rescale_spread(DevCtx c, const uint64_t* tmp, uint64_t* spread, int level) {
    const size_t total = (size_t)2 * level * c.N;
    const uint64_t ql = c.primes[level].q;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int p = r / level, t = r % level;
        const int k = (int)(i & (size_t)(c.N - 1));
        const uint64_t v = tmp[(size_t)p * c.N + k];
        const Prime pr = c.primes[t];
        uint64_t o;
        if (v > (ql >> 1)) {
            const uint64_t m = reduce64(ql - v, pr);
            o = m ? pr.q - m : 0;
        } else {
            o = reduce64(v, pr);
        }
        spread[i] = o;
    }
}

__global__ void k_rescale_finish(DevCtx c, uint64_t* out, const uint64_t* in, const uint64_t* spread, int level,
                                 const uint64_t* qlinv, const uint64_t* qlinv_sh) {
    const size_t total = (size_t)2 * level * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int p = r / level, t = r % level;
        const int k = (int)(i & (size_t)(c.N - 1));
        const uint64_t q = c.primes[t].q;
        const uint64_t x = in[((size_t)p * (level + 1) + t) * c.N + k];
        out[i] = mul_shoup(sub_mod(x, spread[i], q), qlinv[t], qlinv_sh[t], q);
    }
}

}  // namespace

void ew_add(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp,
            cudaStream_t st) {
    ++g_launches;
    k_ew<0><<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, out, a, b, nrows, rpp);
}
void ew_sub(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp,
            cudaStream_t st) {
    ++g_launches;
    k_ew<1><<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, out, a, b, nrows, rpp);
}
void ew_mul_bcast(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp,
                  cudaStream_t st) {
    ++g_launches;
    k_ew<2><<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, out, a, b, nrows, rpp);
}
void ew_const(const DevCtx& c, uint64_t* out, const uint64_t* a, const RowConsts& k, int nr, int mul,
              cudaStream_t st) {
    ++g_launches;
    if (mul)
        k_ew_const<1><<<ew_blocks((size_t)2 * nr * c.N), kEwThreads, 0, st>>>(c, out, a, k, nr);
    else
        k_ew_const<0><<<ew_blocks((size_t)2 * nr * c.N), kEwThreads, 0, st>>>(c, out, a, k, nr);
}
void automorph(const DevCtx& c, uint64_t* out, const uint64_t* in, int nrows, uint32_t galois, cudaStream_t st) {
    ++g_launches;
    k_automorph<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, out, in, nrows, galois);
}
void rescale_spread(const DevCtx& c, const uint64_t* tmp, uint64_t* spread, int level, cudaStream_t st) {
    ++g_launches;
    k_rescale_spread<<<ew_blocks((size_t)2 * level * c.N), kEwThreads, 0, st>>>(c, tmp, spread, level);
}
void rescale_finish(const DevCtx& c, uint64_t* out, const uint64_t* in, const uint64_t* spread, int level,
                    const uint64_t* qlinv, const uint64_t* qlinv_sh, cudaStream_t st) {
    ++g_launches;
    k_rescale_finish<<<ew_blocks((size_t)2 * level * c.N), kEwThreads, 0, st>>>(c, out, in, spread, level, qlinv,
                                                                                 qlinv_sh);
}

// -------------------------------------------------------- key switching
namespace {

// one thread per (digit j, coefficient k): computes the centered
// [x_i (Q_J/q_i)^-1]_{q_i} once and extends it to every target row.

__global__ void k_ks_inner(DevCtx c, const uint64_t* D, const uint64_t* key, uint64_t* acc0, uint64_t* acc1,
                           uint32_t g, int level, int dn) {
    const int ne = level + 1 + c.K;
    const int np = c.L + c.K;
    const size_t total = (size_t)ne * c.N;
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int p = row_prime(rm, u);
        const Prime pr = c.primes[p];
        const uint32_t pk = perm_index(k, g, c.logN);
        U128 s0{0, 0}, s1{0, 0};
        for (int j = 0; j < dn; ++j) {
            const uint64_t d = D[((size_t)j * ne + u) * c.N + pk];
            mac(s0, d, key[(((size_t)j * 2 + 0) * np + p) * c.N + k]);
            mac(s1, d, key[(((size_t)j * 2 + 1) * np + p) * c.N + k]);
        }
        acc0[i] = reduce128(s0.hi, s0.lo, pr);
        acc1[i] = reduce128(s1.hi, s1.lo, pr);
    }
}

__global__ void k_gather_row(DevCtx c, uint64_t* dst, const uint64_t* src, size_t stride, int npoly) {
    const size_t total = (size_t)npoly * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[(i >> c.logN) * stride + (i & (size_t)(c.N - 1))];
}

__global__ void k_gather_special(DevCtx c, uint64_t* dst, const uint64_t* acc, size_t acc_stride, int level,
                                 int npoly) {
    const size_t total = (size_t)npoly * c.K * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i >> c.logN);
        const int p = r / c.K, kk = r % c.K;
        dst[i] = acc[(size_t)p * acc_stride + ((size_t)level + 1 + kk) * c.N + (i & (size_t)(c.N - 1))];
    }
}

// Fused rotation + plaintext multiply-accumulate of the conv (one source X).
__global__ void __launch_bounds__(256) k_conv_mac(DevCtx c, uint64_t* acc, const uint64_t* D, const uint64_t* X,
                                                  MacTerms terms, const ModDownTable* md, int level, int dn) {
    const int nr = level + 1, ne = nr + c.K;
    const int np = c.L + c.K;
    const size_t total = (size_t)ne * c.N;
    const size_t plane = total;  // ACC = [2][ne][N]
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int p = row_prime(rm, u);
        const Prime pr = c.primes[p];
        const bool qrow = u < nr;
        const uint64_t pm = qrow ? md->pmod[u] : 0, pms = qrow ? md->pmod_sh[u] : 0;
        U128 a0{0, 0}, a1{0, 0};
        for (int t = 0; t < terms.n; ++t) {
            const uint64_t w = terms.pt[t][i];
            const uint32_t g = terms.galois[t];
            if (g == 1) {
                if (!qrow) continue;
                const uint64_t x0 = mul_shoup(X[(size_t)u * c.N + k], pm, pms, pr.q);
                const uint64_t x1 = mul_shoup(X[((size_t)nr + u) * c.N + k], pm, pms, pr.q);
                mac(a0, w, x0);
                mac(a1, w, x1);
                continue;
            }
            const uint32_t pk = perm_index(k, g, c.logN);
            const uint64_t* key = terms.key[t];
            U128 s0{0, 0}, s1{0, 0};
            for (int j = 0; j < dn; ++j) {
                const uint64_t d = D[((size_t)j * ne + u) * c.N + pk];
                mac(s0, d, key[(((size_t)j * 2 + 0) * np + p) * c.N + k]);
                mac(s1, d, key[(((size_t)j * 2 + 1) * np + p) * c.N + k]);
            }
            if (qrow) add128(s0, mul_shoup(X[(size_t)u * c.N + pk], pm, pms, pr.q));
            const uint64_t ip0 = reduce128(s0.hi, s0.lo, pr);
            const uint64_t ip1 = reduce128(s1.hi, s1.lo, pr);
            mac(a0, w, ip0);
            mac(a1, w, ip1);
        }
        add128(a0, acc[i]);
        add128(a1, acc[plane + i]);
        acc[i] = reduce128(a0.hi, a0.lo, pr);
        acc[plane + i] = reduce128(a1.hi, a1.lo, pr);
    }
}

}  // namespace

void ks_inner_product(const DevCtx& c, const uint64_t* digits, const uint64_t* key, uint64_t* acc0,
                      uint64_t* acc1, uint32_t galois, int level, int dn, cudaStream_t st) {
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    ++g_launches;
    k_ks_inner<<<ew_blocks(total), kEwThreads, 0, st>>>(c, digits, key, acc0, acc1, galois, level, dn);
}
void gather_row(const DevCtx& c, uint64_t* dst, const uint64_t* src, size_t stride, int npoly, cudaStream_t st) {
    ++g_launches;
    k_gather_row<<<ew_blocks((size_t)npoly * c.N), kEwThreads, 0, st>>>(c, dst, src, stride, npoly);
}
void gather_special(const DevCtx& c, uint64_t* dst, const uint64_t* acc, size_t acc_stride, int level, int npoly,
                    cudaStream_t st) {
    ++g_launches;
    k_gather_special<<<ew_blocks((size_t)npoly * c.K * c.N), kEwThreads, 0, st>>>(c, dst, acc, acc_stride, level,
                                                                                   npoly);
}
void conv_mac(const DevCtx& c, uint64_t* acc, const uint64_t* digits, const uint64_t* x, const MacTerms& t,
              const ModDownTable* md, int level, int dn, cudaStream_t st) {
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    ++g_launches;
    k_conv_mac<<<ew_blocks(total), 256, 0, st>>>(c, acc, digits, x, t, md, level, dn);
}

namespace {

// ---- key-switch inner products on coefficient pairs (k, k+1), k even.
// In bit-reversed NTT order perm_g(k+1) = perm_g(k) ^ 1, so the gathered
// digit pair is the aligned pair {2j, 2j+1} (possibly swapped): every access
// below is a 16-byte vector load.
__device__ __forceinline__ ulonglong2 ld2(const uint64_t* p) { return __ldg(reinterpret_cast<const ulonglong2*>(p)); }
__device__ __forceinline__ void st2(uint64_t* p, uint64_t a, uint64_t b) {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(a, b);
}

// ---- cp.async (LDGSTS) helpers: per-thread asynchronous 16-byte copies to smem
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Streaming key switch. Each thread owns a coefficient pair
// of one extended row and walks the term list; the 2*DN key words and DN
// gathered digit words of term t+1 are copied into a per-thread shared-memory
// stage with cp.async while term t is multiplied out, so every thread keeps
// ~700 bytes of the key stream in flight without holding them in registers.
// MODE 0 (baby steps): XT[slot_t] = (IP_0 + [u<=l] P sigma_t(c0), IP_1) per term.
// MODE 1 (giant steps): acc += sum_t (IP_0 + [u<=l] P sigma_t(c0_t), IP_1).
constexpr int kStreamThreads = 128;
template <int DN, int MODE>
__global__ void __launch_bounds__(kStreamThreads) k_ks_stream(DevCtx c, KsStream a, const ModDownTable* md,
                                                              int level) {
    extern __shared__ ulonglong2 sbuf[];  // [2 stages][3*DN][kStreamThreads]
    const int nr = level + 1, ne = nr + c.K;
    const int np = c.L + c.K;
    const size_t total = (size_t)ne * c.N;
    RowMap rm{ne, level, c.L, 0};
    const int tid = threadIdx.x;
    auto slot = [&](int stage, int w) -> ulonglong2* { return sbuf + ((size_t)stage * 3 * DN + w) * kStreamThreads + tid; };
    for (size_t ip = blockIdx.x * (size_t)blockDim.x + tid; ip < total / 2; ip += (size_t)gridDim.x * blockDim.x) {
        const size_t i = ip * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int p = row_prime(rm, u);
        const Prime pr = c.primes[p];
        const bool qrow = u < nr;
        const uint64_t pm = qrow ? md->pmod[u] : 0, pms = qrow ? md->pmod_sh[u] : 0;
        auto issue = [&](int t, int stage) {
            const uint32_t pk = perm_index(k, a.galois[t], c.logN);
            const uint64_t* key = a.key[t];
            const uint64_t* D = a.digits + (size_t)t * a.digit_stride;
#pragma unroll
            for (int j = 0; j < DN; ++j) {
                cp_async16(slot(stage, 3 * j + 0), key + (((size_t)j * 2 + 0) * np + p) * c.N + k);
                cp_async16(slot(stage, 3 * j + 1), key + (((size_t)j * 2 + 1) * np + p) * c.N + k);
                cp_async16(slot(stage, 3 * j + 2), D + ((size_t)j * ne + u) * c.N + (pk & ~1u));
            }
            cp_async_commit();
        };
        U128 s0[2] = {{0, 0}, {0, 0}}, s1[2] = {{0, 0}, {0, 0}};
        issue(0, 0);
        for (int t = 0; t < a.n; ++t) {
            if (t + 1 < a.n)
                issue(t + 1, (t + 1) & 1);
            else
                cp_async_commit();  // empty group keeps the wait count uniform
            cp_async_wait<1>();
            const int st = t & 1;
            const uint32_t pk = perm_index(k, a.galois[t], c.logN);
            const bool swp = pk & 1u;
            if (MODE == 0) {
                s0[0] = s0[1] = s1[0] = s1[1] = U128{0, 0};
            }
#pragma unroll
            for (int j = 0; j < DN; ++j) {
                const ulonglong2 k0 = *slot(st, 3 * j + 0), k1 = *slot(st, 3 * j + 1), d = *slot(st, 3 * j + 2);
                const uint64_t da = swp ? d.y : d.x, db = swp ? d.x : d.y;
                mac(s0[0], da, k0.x);
                mac(s0[1], db, k0.y);
                mac(s1[0], da, k1.x);
                mac(s1[1], db, k1.y);
            }
            if (a.c0_qp) {  // P-scaled QP-basis c0: added unscaled on every row
                const ulonglong2 x = ld2(a.c0[t] + (size_t)u * c.N + (pk & ~1u));
                add128(s0[0], swp ? x.y : x.x);
                add128(s0[1], swp ? x.x : x.y);
            } else if (qrow) {
                const ulonglong2 x = ld2(a.c0[t] + (size_t)u * c.N + (pk & ~1u));
                add128(s0[0], mul_shoup(swp ? x.y : x.x, pm, pms, pr.q));
                add128(s0[1], mul_shoup(swp ? x.x : x.y, pm, pms, pr.q));
            }
            if (MODE == 0) {
                uint64_t* xt = a.out + (size_t)a.slot[t] * 2 * total;
                st2(xt + i, reduce128(s0[0].hi, s0[0].lo, pr), reduce128(s0[1].hi, s0[1].lo, pr));
                st2(xt + total + i, reduce128(s1[0].hi, s1[0].lo, pr), reduce128(s1[1].hi, s1[1].lo, pr));
            }
        }
        if (MODE == 1) {
            const ulonglong2 a0 = ld2(a.out + i), a1 = ld2(a.out + total + i);
            add128(s0[0], a0.x);
            add128(s0[1], a0.y);
            add128(s1[0], a1.x);
            add128(s1[1], a1.y);
            st2(a.out + i, reduce128(s0[0].hi, s0[0].lo, pr), reduce128(s0[1].hi, s0[1].lo, pr));
            st2(a.out + total + i, reduce128(s1[0].hi, s1[0].lo, pr), reduce128(s1[1].hi, s1[1].lo, pr));
        }
    }
}

// ---- batched key switching: work item = (coefficient pair, source), source
// fastest, so the lanes of a warp that share a pair issue identical key
// addresses (one transaction serves all sources of the batch).


// XT[s][slot] = P ct_s (identity baby step) for nsrc sources
__global__ void k_identity_batch(DevCtx c, uint64_t* xt, size_t xt_src_stride, const uint64_t* X, size_t x_src_stride,
                                 const ModDownTable* md, int level, int nsrc) {
    const int nr = level + 1, ne = nr + c.K;
    const size_t total = (size_t)ne * c.N;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < total * nsrc; j += (size_t)gridDim.x * blockDim.x) {
        const int s = (int)(j / total);
        const size_t i = j - (size_t)s * total;
        const int u = (int)(i >> c.logN);
        const size_t k = i & (size_t)(c.N - 1);
        uint64_t* o = xt + (size_t)s * xt_src_stride;
        const uint64_t* x = X + (size_t)s * x_src_stride;
        if (u < nr) {
            const uint64_t q = c.primes[u].q;
            o[i] = mul_shoup(x[(size_t)u * c.N + k], md->pmod[u], md->pmod_sh[u], q);
            o[total + i] = mul_shoup(x[((size_t)nr + u) * c.N + k], md->pmod[u], md->pmod_sh[u], q);
        } else {
            o[i] = 0;
            o[total + i] = 0;
        }
    }
}

// XT[slot] = P ct (identity baby step) for q rows, 0 for the special rows
__global__ void k_identity_term(DevCtx c, uint64_t* xt, const uint64_t* X, const ModDownTable* md, int level) {
    const int nr = level + 1, ne = nr + c.K;
    const size_t total = (size_t)ne * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int u = (int)(i >> c.logN);
        const size_t k = i & (size_t)(c.N - 1);
        if (u < nr) {
            const uint64_t q = c.primes[u].q;
            xt[i] = mul_shoup(X[(size_t)u * c.N + k], md->pmod[u], md->pmod_sh[u], q);
            xt[total + i] = mul_shoup(X[((size_t)nr + u) * c.N + k], md->pmod[u], md->pmod_sh[u], q);
        } else {
            xt[i] = 0;
            xt[total + i] = 0;
        }
    }
}

// XT[b][c] = (IP_0(D, key_b) + [u<=l] P sigma_b(X.c0), IP_1(D, key_b)); identity b: P X

// Y[g][c] = sum_b pt[g][b] * XT[b][c]  (the plaintext "matrix-vector" of the baby steps)


// Fused BSGS baby steps. A CTA owns P = 128/SG consecutive coefficient pairs
// of one extended row and SG sources (thread = (pair, source), pair fastest).
// Per baby step the CTA stages, with cp.async, the 2*DN key words and NG
// plaintext words of its pairs ONCE (shared by the SG sources) plus every
// source's DN gathered digit words and gathered c0 word; the stage of baby
// b+1 is in flight while baby b is multiplied out. The key-switched X~_b lives
// only in registers; the NG giant accumulators are 128-bit lazy sums.
template <int DN, int NG, int SG, int NST_>
struct FusedLayout {
    static constexpr int P = 128 / SG;
    static constexpr int KW = 2 * DN * P;   // key words      [2*DN][P]
    static constexpr int PW = NG * P;       // plaintexts     [NG][P]
    static constexpr int DW = SG * DN * P;  // digits         [SG][DN][P]
    static constexpr int CW = SG * P;       // gathered c0    [SG][P]
    static constexpr int STAGE = KW + PW + DW + CW;
};

template <int DN, int NG, int SG, int NST, int MINB, bool SLOTS>
__global__ void __launch_bounds__(128, MINB) k_bsgs_fused(DevCtx c, FusedBsgs a, const ModDownTable* md, int level) {
    using LY = FusedLayout<DN, NG, SG, NST>;
    constexpr int P = LY::P;
    extern __shared__ ulonglong2 sb[];  // [NST stages][STAGE]
    const int nr = level + 1, ne = nr + c.K, np = c.L + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / 2 / P;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const size_t keyrow = (size_t)np * c.N;  // stride between key rows j and j+1
    RowMap rm{ne, level, c.L, 0};
    // per-thread smem slots (stage 0); stage 1 is + STAGE
    ulonglong2* const s_key = sb + p;                                   // + j * P
    ulonglong2* const s_pt = sb + LY::KW + p;                           // + g * P
    ulonglong2* const s_dig = sb + LY::KW + LY::PW + sl * DN * P + p;   // + j * P
    ulonglong2* const s_c0 = sb + LY::KW + LY::PW + LY::DW + sl * P + p;
    for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
        const size_t chunk = it / (size_t)ngroups;
        const int s = (int)(it % (size_t)ngroups) * SG + sl;
        const bool active = s < a.nsrc;
        const size_t i = (chunk * P + p) * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int pi = row_prime(rm, u);
        const Prime pr = c.primes[pi];
        const bool qrow = u < nr;
        const uint64_t pm = qrow ? md->pmod[u] : 0, pms = qrow ? md->pmod_sh[u] : 0;
        const uint64_t* Du0 = a.digits + (size_t)(active ? s : 0) * a.digit_src_stride + (size_t)u * c.N;
        const uint64_t* C00 = a.ct + (size_t)(active ? s : 0) * a.ct_src_stride;
        const size_t kofs = (size_t)pi * c.N + k, pofs = (size_t)u * c.N + k;
        // bit-reversed exponent of this pair, reused for every baby's permutation
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, nmask = (2u << c.logN) - 1;
        auto pidx = [&](uint32_t g) { return brev_n((((e * g) & nmask) - 1) >> 1, c.logN); };
        auto issue_s = [&](int b, size_t so) {
            if (b >= a.nb) {
                cp_async_commit();  // empty group keeps the wait count uniform
                return;
            }
            const uint32_t pk = pidx(a.galois[b]);
            const uint64_t* key = a.key[b];
            const uint32_t gm = a.gmask[b];
            const uint64_t* Du = SLOTS ? Du0 + (size_t)a.srcslot[b] * a.digit_slot_stride : Du0;
            const uint64_t* C = SLOTS ? C00 + (size_t)a.srcslot[b] * a.ct_slot_stride : C00;
            const uint64_t* C0u = C + (size_t)u * c.N;
            const uint64_t* C1u = C + ((size_t)nr + u) * c.N;
#pragma unroll
            for (int g = sl; g < NG; g += SG)
                if ((gm >> g) & 1u) cp_async16(s_pt + so + g * P, a.pt[b] + (size_t)g * a.pt_g_stride + pofs);
            if (key) {
                const uint64_t* kp = key + kofs;
#pragma unroll
                for (int j = sl; j < 2 * DN; j += SG) cp_async16(s_key + so + j * P, kp + (size_t)j * keyrow);
                if (active) {
                    const uint64_t* dp = Du + (pk & ~1u);
#pragma unroll
                    for (int j = 0; j < DN; ++j) cp_async16(s_dig + so + j * P, dp + (size_t)j * total);
                    if (qrow) cp_async16(s_c0 + so, C0u + (pk & ~1u));
                }
            } else if (active && qrow) {  // identity: c0, c1 unpermuted
                cp_async16(s_dig + so, C1u + k);
                cp_async16(s_c0 + so, C0u + k);
            }
            cp_async_commit();
        };
        auto issue = [&](int b) { issue_s(b, (size_t)(b % NST) * LY::STAGE); };
        U128 y[NG][2][2];
#pragma unroll
        for (int g = 0; g < NG; ++g) y[g][0][0] = y[g][0][1] = y[g][1][0] = y[g][1][1] = U128{0, 0};
        if (SLOTS && a.accumulate && active) {  // continue earlier partial sums, in the kernel's 2^-64 domain
            const uint64_t* Ys = a.Y + (size_t)s * a.y_src_stride;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                if (g >= a.ng) break;
                const ulonglong2 v0 = ld2(Ys + (size_t)g * a.y_g_stride + i);
                const ulonglong2 v1 = ld2(Ys + (size_t)g * a.y_g_stride + total + i);
                y[g][0][0] = U128{redc_lazy(0, v0.x, pr), 0};
                y[g][0][1] = U128{redc_lazy(0, v0.y, pr), 0};
                y[g][1][0] = U128{redc_lazy(0, v1.x, pr), 0};
                y[g][1][1] = U128{redc_lazy(0, v1.y, pr), 0};
            }
        }
#pragma unroll
        for (int b = 0; b < NST - 1; ++b) issue(b);
        // one baby step on pipeline stage `so` (the next stage `so_next` is refilled meanwhile)
        auto baby = [&](int b, size_t so, size_t so_next) {
            cp_async_wait<NST - 2>();
            __syncthreads();  // stage b visible to all; everyone is past baby b-1
            issue_s(b + NST - 1, so_next);
            const uint32_t pk = pidx(a.galois[b]);
            uint64_t x0a = 0, x0b = 0, x1a = 0, x1b = 0;
            if (a.key[b]) {
                // the gathered pair is (perm(k), perm(k)^1) in some order: one 16-byte
                // load (thread-linear slot, conflict-free), then select the order
                const int swp = (int)(pk & 1u);
                Acc3 s0a{0, 0, 0, 0}, s0b{0, 0, 0, 0}, s1a{0, 0, 0, 0}, s1b{0, 0, 0, 0};
#if FHE_FUSED_SPLITLD
                // the pair in output order as two 8-byte loads (no per-word selects)
                const uint64_t* dga = reinterpret_cast<const uint64_t*>(s_dig + so) + swp;
                const uint64_t* dgb = reinterpret_cast<const uint64_t*>(s_dig + so) + (swp ^ 1);
#endif
#pragma unroll
                for (int j = 0; j < DN; ++j) {
                    const ulonglong2 k0 = s_key[so + (2 * j) * P], k1 = s_key[so + (2 * j + 1) * P];
#if FHE_FUSED_SPLITLD
                    const uint64_t da = dga[2 * j * P], db = dgb[2 * j * P];
#else
                    const ulonglong2 dv = s_dig[so + j * P];  // one conflict-free 16-byte load
                    const uint64_t da = swp ? dv.y : dv.x, db = swp ? dv.x : dv.y;
#endif
                    mac3(s0a, da, k0.x);
                    mac3(s0b, db, k0.y);
                    mac3(s1a, da, k1.x);
                    mac3(s1b, db, k1.y);
                }
                if (qrow) {
#if FHE_FUSED_SPLITLD
                    const uint64_t ca = reinterpret_cast<const uint64_t*>(s_c0 + so)[swp];
                    const uint64_t cb = reinterpret_cast<const uint64_t*>(s_c0 + so)[swp ^ 1];
#else
                    const ulonglong2 cv = s_c0[so];
                    const uint64_t ca = swp ? cv.y : cv.x, cb = swp ? cv.x : cv.y;
#endif
                    if (DN < 8) {  // P c0 as one more product term (s1 holds 8 terms)
                        mac3(s0a, ca, pm);
                        mac3(s0b, cb, pm);
                    } else {
                        add3(s0a, mul_shoup(ca, pm, pms, pr.q));
                        add3(s0b, mul_shoup(cb, pm, pms, pr.q));
                    }
                }
                // X~ 2^-64 in [0, 2q): the factor 2^64 is restored once per output
                const U128 t0a = fold3(s0a), t0b = fold3(s0b), t1a = fold3(s1a), t1b = fold3(s1b);
                x0a = redc_lazy(t0a.hi, t0a.lo, pr);
                x0b = redc_lazy(t0b.hi, t0b.lo, pr);
                x1a = redc_lazy(t1a.hi, t1a.lo, pr);
                x1b = redc_lazy(t1b.hi, t1b.lo, pr);
            } else if (qrow) {
                const ulonglong2 c1 = s_dig[so], c0 = s_c0[so];
                x0a = redc_lazy(0, mul_shoup(c0.x, pm, pms, pr.q), pr);
                x0b = redc_lazy(0, mul_shoup(c0.y, pm, pms, pr.q), pr);
                x1a = redc_lazy(0, mul_shoup(c1.x, pm, pms, pr.q), pr);
                x1b = redc_lazy(0, mul_shoup(c1.y, pm, pms, pr.q), pr);
            }
            const uint32_t gm = a.gmask[b];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                if (!((gm >> g) & 1u)) continue;
                const ulonglong2 w = s_pt[so + g * P];
                mac_small(y[g][0][0], w.x, x0a);
                mac_small(y[g][0][1], w.y, x0b);
                mac_small(y[g][1][0], w.x, x1a);
                mac_small(y[g][1][1], w.y, x1b);
            }
            if ((b & 31) == 31) {  // keep the lazy sums far from 2^128 for any prime size
#pragma unroll
                for (int g = 0; g < NG; ++g)
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2)
                            y[g][q2][e2] = U128{reduce128(y[g][q2][e2].hi, y[g][q2][e2].lo, pr), 0};
            }
        };
        if constexpr (NST == 2 && FHE_FUSED_UNROLL2) {
            // two babies per iteration: the stage offsets are compile-time constants
            constexpr size_t S1 = LY::STAGE;
            for (int b = 0; b < a.nb; b += 2) {
                baby(b, 0, S1);
                if (b + 1 < a.nb) baby(b + 1, S1, 0);
            }
        } else {
            for (int b = 0; b < a.nb; ++b)
                baby(b, (size_t)(b % NST) * LY::STAGE, (size_t)((b + NST - 1) % NST) * LY::STAGE);
        }
        cp_async_wait<0>();
        if (active) {
            uint64_t* Ys = a.Y + (size_t)s * a.y_src_stride;
            const uint64_t r64 = reduce64((uint64_t)0 - pr.q, pr);  // 2^64 mod q
            auto out = [&](const U128& v) { return mul_mod(reduce128(v.hi, v.lo, pr), r64, pr); };
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                if (g >= a.ng) break;
                uint64_t* yg = Ys + (size_t)g * a.y_g_stride;
                st2(yg + i, out(y[g][0][0]), out(y[g][0][1]));
                st2(yg + total + i, out(y[g][1][0]), out(y[g][1][1]));
            }
        }
        __syncthreads();  // the next item's first stage reuses stage 0
    }
}

// ------------------------------------------------------------ operand-form baby steps
// k_bsgs_tma computes the baby steps of k_bsgs_fused on operands stored in the
// operand form of modarith.cuh (keys, plaintexts, ModUp digits, P-scaled
// ciphertexts; converted once per layer / per ModUp), per extended row:
//  q < 2^50 (12 of the 15 rows at cfg3): centred doubles; every product is one
//      fmac_d (7 FP64 operations, exact) into integer-valued double sums: the key
//      inner product X~ = sum_j d_j k_j + [P sigma(c0)]_q, reduced once (red_d), then
//      Y_g += X~ pt'_g, reduced every 8 baby steps;
//  60-bit primes: 30-bit limb form, four mad.wide.u32 per product, Montgomery by
//      2^90 in three 30-bit steps (X~ < 2q), 128-bit plaintext sums (mac_small).
// Outputs Y are fully reduced: bit-identical to k_bsgs_fused.
template <int W>
struct LimbConst {
    static constexpr uint32_t M = (1u << W) - 1;
};

// X 2^-90 mod q (< 2q) for X = z0 + z1 2^30 + z2 2^60 (W = 30)
__device__ __forceinline__ uint64_t mont_l30(uint64_t z0, uint64_t z1, uint64_t z2, uint32_t q0, uint32_t q1,
                                             uint32_t qinv) {
    constexpr uint32_t M = LimbConst<30>::M;
    const uint32_t t0 = ((uint32_t)z0 * qinv) & M;
    madw(z0, t0, q0);
    madw(z1, t0, q1);
    z1 += z0 >> 30;
    const uint32_t t1 = ((uint32_t)z1 * qinv) & M;
    madw(z1, t1, q0);
    madw(z2, t1, q1);
    z2 += z1 >> 30;
    const uint32_t t2 = ((uint32_t)z2 * qinv) & M;
    madw(z2, t2, q0);
    uint64_t r = z2 >> 30;
    madw(r, t2, q1);
    return r;
}

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return (uint32_t)x; }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }

// ------------------------------------------------------------ TMA-staged baby steps
// k_bsgs_tma: the baby steps of k_bsgs_fused on operand-form rows (same thread
// mapping: thread = (coefficient pair, source), P = 128 / SG pairs per CTA) with the operand staging
// taken off the compute threads: per baby step ONE thread issues at most four
// tensor copies (cp.async.bulk.tensor.4d, TMA) that complete on the stage's
// mbarrier -- the 2 DN key rows of the CTA's block (shared by its SG sources), the
// NG plaintext rows, the SG x DN digit blocks and the SG x 2 ciphertext blocks.
// The Galois automorphism maps an aligned block of the bit-reversed NTT order onto
// an aligned block, so the digits and c0 of every source are copied as one whole
// block and the permutation is applied on the shared-memory read (pair slot
// (pidx & (2P - 1)) / 2: a bijection over the warp, conflict-free). Two stages:
// baby b + 2 is fetched while b + 1 is computed.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                          uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

template <int DN, int NG, int SG>
struct TmaLayout {  // one stage, in 16-byte pair slots
    static constexpr int P = 128 / SG;
    static constexpr int KW = 2 * DN * P;  // keys       [2 DN][P]
    static constexpr int PW = NG * P;      // plaintexts [NG][P]
    static constexpr int DW = SG * DN * P; // digits     [SG][DN][P]
    static constexpr int CW = SG * 2 * P;  // c0, c1     [SG][2][P]
    static constexpr int STAGE = KW + PW + DW + CW;
};

// MODE 1 (hoisted key switches, no plaintexts): every baby's X~_b is written to
// Y + s * y_src_stride + b * y_g_stride ([2][ne][N], QP, canonical) instead of being
// multiplied into giant accumulators.
template <int DN, int NG, int SG, int MINB, int MODE = 0, int NST = 2>
__global__ void __launch_bounds__(128, MINB) k_bsgs_tma(DevCtx c, FusedBsgs a, const __grid_constant__ TmaMaps m,
                                                        int level) {
    using LY = TmaLayout<DN, NG, SG>;
    constexpr int P = LY::P, BW = 2 * P;
    extern __shared__ __align__(1024) ulonglong2 tsb[];  // [NST][STAGE], then NST mbarriers
    uint64_t* const bars = reinterpret_cast<uint64_t*>(tsb + NST * LY::STAGE);
    const int nr = level + 1, ne = nr + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / BW;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const uint32_t nmask = (2u << c.logN) - 1;
    RowMap rm{ne, level, c.L, 0};
    // Work queues (m.sched, zeroed per launch): queue 0 = the items of the integer
    // (60-bit) rows, queue 1 = the FP64 rows (m.rowlist: integer rows first). The
    // first CTA resident on each SM drains queue 0, the others queue 1, so every SM
    // runs integer-multiply and FP64 work side by side; a CTA whose queue is empty
    // helps with the other one. Items: group fastest, then chunk, then row.
    __shared__ int s_item[2];
    __shared__ unsigned s_cnt[NST];  // warps done with stage st (FHE_TMA_NOSYNC)
    const size_t cpr = (size_t)c.N / BW;  // chunks per row
    const size_t nq[2] = {(size_t)m.nint * cpr * ngroups, (size_t)(ne - m.nint) * cpr * ngroups};
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < NST; ++st) {
            mbar_init(bars + st, 1);
            s_cnt[st] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        s_item[1] = (m.nint > 0 && m.nint < ne && atomicAdd(m.sched + 2 + (smid & 255), 1u) == 0) ? 0 : 1;
    }
    __syncthreads();
    const int role = s_item[1];
    uint32_t phase = 0;
    (void)items;
    for (;;) {
        if (tid == 0) {
            long long v = -1;
            for (int r2 = 0; r2 < 2 && v < 0; ++r2) {
                const int q = role ^ r2;
                if (!nq[q]) continue;
                const unsigned x = atomicAdd(m.sched + q, 1u);
                if (x < nq[q]) v = (long long)q << 40 | x;
            }
            s_item[0] = (int)(v < 0 ? -1 : ((v >> 40) << 30 | (v & ((1ll << 30) - 1))));
        }
        __syncthreads();
        const int sv = s_item[0];
        __syncthreads();
        if (sv < 0) break;
        const int qsel = sv >> 30;
        const size_t xi = (size_t)(sv & ((1 << 30) - 1));
        const size_t per_row = cpr * ngroups;
        const int urow = m.rowlist[(qsel ? m.nint : 0) + (int)(xi / per_row)];
        const size_t chunk = (size_t)urow * cpr + (xi % per_row) / ngroups;
        const int s0 = (int)(xi % (size_t)ngroups) * SG;
        const int s = s0 + sl;
        const bool active = s < a.nsrc;
        // boxes never leave the tensors: the source box of a partial last group is
        // shifted back (nsrc >= SG), and special rows (no ciphertext row) read row 0
        const int s0c = min(s0, a.nsrc - SG), slot = active ? s - s0c : 0;
        const size_t i0 = chunk * BW, i = i0 + 2 * p;
        const int u = (int)(i0 >> c.logN);
        const uint32_t k0 = (uint32_t)(i0 & (size_t)(c.N - 1)), k = k0 + 2 * p;
        const int pi = row_prime(rm, u);
        const Prime pr = c.primes[pi];
        const bool qrow = u < nr;
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, e0 = 2 * brev_n(k0, c.logN) + 1;
        auto pidx = [&](uint32_t ee, uint32_t g) { return brev_n((((ee * g) & nmask) - 1) >> 1, c.logN); };
        auto issue_one = [&](int b, int st) {  // the calling thread fetches baby b into stage st
            if (b >= a.nb) return;
            ulonglong2* sb = tsb + st * LY::STAGE;
            uint64_t* bar = bars + st;
            const bool keyed = m.kidx[b] >= 0;
            const int blk = (int)(pidx(e0, a.galois[b]) & ~(uint32_t)(BW - 1));
            mbar_expect_tx(bar, (uint32_t)((MODE == 0 ? LY::PW : 0) + LY::CW + (keyed ? LY::KW + LY::DW : 0)) * 16u);
            const int sl5 = a.srcslot[b];  // source slot (paper schedules: the rotated copy)
            if (MODE == 0) tma_load4(sb + LY::KW, &m.pt, (int)k0, u, m.bidx[b], m.g0 + m.gidx[b], bar);
            tma_load5(sb + LY::KW + LY::PW + LY::DW, &m.ct, blk, qrow ? u : 0, 0, sl5, s0c, bar);
            if (keyed) {
                tma_load4(sb, &m.key, (int)k0, pi, 0, m.kidx[b], bar);
                tma_load5(sb + LY::KW + LY::PW, &m.dig, blk, u, 0, sl5, s0c, bar);
            }
        };
        auto issue = [&](int b, int st) {
            if (tid == 0) issue_one(b, st);
        };
        // A warp is done with stage st of baby b. FHE_TMA_NOSYNC: no CTA barrier per baby
        // step -- the last of the CTA's four warps to get here refills the stage (a counter
        // in shared memory elects it), so warps drift apart by up to a baby step and their
        // shared-memory, FP64 and integer phases overlap. Otherwise: barrier, thread 0 refills.
        auto release = [&](int b, int st) {
#if FHE_TMA_NOSYNC
            __syncwarp();
            if ((tid & 31) == 0) {
                __threadfence_block();
                if (atomicAdd(&s_cnt[st], 1u) == 3u) {
                    atomicExch(&s_cnt[st], 0u);
                    issue_one(b + NST, st);
                }
            }
#else
            __syncthreads();  // stage st is free: fetch baby b + NST into it
            issue(b + NST, st);
#endif
        };
        // q < 2^50: FP64 operand form (modarith.cuh): every product is one fmac_d on the
        // FP64 pipe, the sums stay exact integers below 2^53
        auto run_fp = [&]() {
            const ArD ad = make_ard(pr.q);
            const ArG ag = make_arg(ad);
            double y[NG][2][2];
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) y[g][q2][e2] = 0.0;
            issue(0, 0);
            issue(1, 1);
            if (NST > 2) issue(2, 2);
            auto baby = [&](int b, int st) {
                mbar_wait(bars + st, (phase >> st) & 1u);
                phase ^= 1u << st;
                const ulonglong2* sb = tsb + st * LY::STAGE;
                const uint32_t pk = pidx(e, a.galois[b]);
                const int wo = (int)(pk & (uint32_t)(BW - 1));
                const double* sc = reinterpret_cast<const double*>(sb + LY::KW + LY::PW + LY::DW + slot * 2 * P);
                double x[2][2];
                if (m.kidx[b] >= 0) {
                    const double* sd = reinterpret_cast<const double*>(sb + LY::KW + LY::PW + slot * DN * P);
                    const double2* sk = reinterpret_cast<const double2*>(sb);
                    // key inner product on the 2^50 grid (fmag_d: one quotient per sum)
                    double z[2][2] = {{kGridBig, kGridBig}, {kGridBig, kGridBig}};
                    double zl[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                    if (qrow) {  // + [P sigma(c0)]_q
                        zl[0][0] = sc[wo];
                        zl[0][1] = sc[wo ^ 1];
                    }
#pragma unroll
                    for (int j = 0; j < DN; ++j) {
                        const double2 k0 = sk[(2 * j) * P + p], k1 = sk[(2 * j + 1) * P + p];
#if FHE_DIG128
                        // one conflict-free 16-byte load of the permuted pair, swapped in registers
                        const double2 dp = reinterpret_cast<const double2*>(sd)[j * P + (wo >> 1)];
                        const double d0 = (wo & 1) ? dp.y : dp.x, d1 = (wo & 1) ? dp.x : dp.y;
#else
                        const double d0 = sd[j * BW + wo], d1 = sd[j * BW + (wo ^ 1)];
#endif
                        fmag_d(z[0][0], zl[0][0], d0, k0.x);
                        fmag_d(z[0][1], zl[0][1], d1, k0.y);
                        fmag_d(z[1][0], zl[1][0], d0, k1.x);
                        fmag_d(z[1][1], zl[1][1], d1, k1.y);
                    }
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) x[q2][e2] = fold_d(z[q2][e2], zl[q2][e2], ad, ag);
                } else if (qrow) {  // identity: X = [P c]_q, unpermuted
                    x[0][0] = sc[2 * p];
                    x[0][1] = sc[2 * p + 1];
                    x[1][0] = sc[BW + 2 * p];
                    x[1][1] = sc[BW + 2 * p + 1];
                } else {
                    x[0][0] = x[0][1] = x[1][0] = x[1][1] = 0.0;
                }
                if constexpr (MODE == 1) {
                    if (active) {
                        uint64_t* yb = a.Y + (size_t)s * a.y_src_stride + (size_t)b * a.y_g_stride;
                        st2(yb + i, canon_d(x[0][0], ad), canon_d(x[0][1], ad));
                        st2(yb + total + i, canon_d(x[1][0], ad), canon_d(x[1][1], ad));
                    }
                    release(b, st);
                    return;
                }
                const uint32_t gm = a.gmask[b];
                const double2* sp = reinterpret_cast<const double2*>(sb + LY::KW);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (!((gm >> g) & 1u)) continue;
                    const double2 w = sp[g * P + p];
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {
                        fmac_d(y[g][q2][0], x[q2][0], w.x, ad);
                        fmac_d(y[g][q2][1], x[q2][1], w.y, ad);
                    }
                }
                if ((b & 7) == 7) {  // 8 terms of <= 0.5 q + 2^44 each: far below 2^53
#pragma unroll
                    for (int g = 0; g < NG; ++g)
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                            for (int e2 = 0; e2 < 2; ++e2) y[g][q2][e2] = red_d(y[g][q2][e2], ad);
                }
                release(b, st);
            };
            for (int b = 0; b < a.nb; b += NST) {
                baby(b, 0);
                if (b + 1 < a.nb) baby(b + 1, 1);
                if (NST > 2 && b + 2 < a.nb) baby(b + 2, 2);
            }
            if (MODE == 0 && active) {
                uint64_t* Ys = a.Y + (size_t)s * a.y_src_stride;
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (g >= a.ng) break;
                    uint64_t* yg = Ys + (size_t)g * a.y_g_stride;
                    uint64_t o[2][2];
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) o[q2][e2] = canon_d(red_d(y[g][q2][e2], ad), ad);
                    if (a.accumulate) {  // Y_g += (later launches of a long baby list)
                        const ulonglong2 y0 = ld2(yg + i), y1 = ld2(yg + total + i);
                        o[0][0] = add_mod(o[0][0], y0.x, pr.q);
                        o[0][1] = add_mod(o[0][1], y0.y, pr.q);
                        o[1][0] = add_mod(o[1][0], y1.x, pr.q);
                        o[1][1] = add_mod(o[1][1], y1.y, pr.q);
                    }
                    st2(yg + i, o[0][0], o[0][1]);
                    st2(yg + total + i, o[1][0], o[1][1]);
                }
            }
        };
        // 60-bit primes: 30-bit limb form (four mad.wide.u32 per product, Montgomery by 2^90)
        auto run_l30 = [&]() {
            constexpr int W = 30;
            constexpr uint32_t MW = LimbConst<W>::M;
            const uint32_t q0 = (uint32_t)(pr.q & MW), q1 = (uint32_t)(pr.q >> W);
            const uint32_t qinv = (uint32_t)pr.qinv & MW;
            U128 y[NG][2][2];
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) y[g][q2][e2] = U128{0, 0};
            issue(0, 0);
            issue(1, 1);
            if (NST > 2) issue(2, 2);
            auto baby = [&](int b, int st) {
                mbar_wait(bars + st, (phase >> st) & 1u);
                phase ^= 1u << st;
                const ulonglong2* sb = tsb + st * LY::STAGE;
                const uint32_t pk = pidx(e, a.galois[b]);
                const int wo = (int)(pk & (uint32_t)(BW - 1));  // permuted word in the block
                uint64_t x[2][2];
                const uint64_t* sc = reinterpret_cast<const uint64_t*>(sb + LY::KW + LY::PW + LY::DW + slot * 2 * P);
                if (m.kidx[b] >= 0) {
                    const uint64_t* sd = reinterpret_cast<const uint64_t*>(sb + LY::KW + LY::PW + slot * DN * P);
                    uint64_t z0[2][2] = {{0, 0}, {0, 0}}, z1[2][2] = {{0, 0}, {0, 0}}, z2[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
                    for (int j = 0; j < DN; ++j) {
                        const ulonglong2 kv0 = sb[(2 * j) * P + p], kv1 = sb[(2 * j + 1) * P + p];
                        const uint64_t dw[2] = {sd[j * BW + wo], sd[j * BW + (wo ^ 1)]};
                        const uint64_t kw[2][2] = {{kv0.x, kv0.y}, {kv1.x, kv1.y}};
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) {
                            const uint32_t d0 = lo32(dw[e2]), d1 = hi32(dw[e2]);
#pragma unroll
                            for (int q2 = 0; q2 < 2; ++q2) {
                                const uint32_t kk0 = lo32(kw[q2][e2]), kk1 = hi32(kw[q2][e2]);
                                madw(z0[q2][e2], d0, kk0);
                                madw(z1[q2][e2], d0, kk1);
                                madw(z1[q2][e2], d1, kk0);
                                madw(z2[q2][e2], d1, kk1);
                            }
                        }
                    }
                    if constexpr (DN >= 8) {  // keep z1 + the c0 and Montgomery terms below 2^64
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                            for (int e2 = 0; e2 < 2; ++e2) {
                                z2[q2][e2] += z1[q2][e2] >> W;
                                z1[q2][e2] &= MW;
                            }
                    }
                    if (qrow) {  // + [P sigma(c0)]_q in limb form
                        const uint64_t cw[2] = {sc[wo], sc[wo ^ 1]};
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) {
                            z0[0][e2] += lo32(cw[e2]);
                            z1[0][e2] += hi32(cw[e2]);
                        }
                    }
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2)
                            x[q2][e2] = mont_l30(z0[q2][e2], z1[q2][e2], z2[q2][e2], q0, q1, qinv);
                } else if (qrow) {  // identity: X = [P c]_q, unpermuted
                    const uint64_t cw[2][2] = {{sc[2 * p], sc[2 * p + 1]}, {sc[BW + 2 * p], sc[BW + 2 * p + 1]}};
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2)
                            x[q2][e2] = mont_l30(lo32(cw[q2][e2]), hi32(cw[q2][e2]), 0, q0, q1, qinv);
                } else {
                    x[0][0] = x[0][1] = x[1][0] = x[1][1] = 0;
                }
                if constexpr (MODE == 1) {
                    if (active) {
                        uint64_t r90 = reduce64(1ULL << 45, pr);
                        r90 = mul_mod(r90, r90, pr);
                        uint64_t* yb = a.Y + (size_t)s * a.y_src_stride + (size_t)b * a.y_g_stride;
                        st2(yb + i, mul_mod(x[0][0], r90, pr), mul_mod(x[0][1], r90, pr));
                        st2(yb + total + i, mul_mod(x[1][0], r90, pr), mul_mod(x[1][1], r90, pr));
                    }
                    release(b, st);
                    return;
                }
                const uint32_t gm = a.gmask[b];
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (!((gm >> g) & 1u)) continue;
                    const ulonglong2 wv = sb[LY::KW + g * P + p];
                    const uint64_t wa = from_limb(wv.x, 30), wb = from_limb(wv.y, 30);
                    mac_small(y[g][0][0], wa, x[0][0]);
                    mac_small(y[g][0][1], wb, x[0][1]);
                    mac_small(y[g][1][0], wa, x[1][0]);
                    mac_small(y[g][1][1], wb, x[1][1]);
                }
                if ((b & 31) == 31) {  // 32 terms < 2^61 * 2^60 each stay below 2^128
#pragma unroll
                    for (int g = 0; g < NG; ++g)
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                            for (int e2 = 0; e2 < 2; ++e2)
                                y[g][q2][e2] = U128{reduce128(y[g][q2][e2].hi, y[g][q2][e2].lo, pr), 0};
                }
                release(b, st);
            };
            for (int b = 0; b < a.nb; b += NST) {
                baby(b, 0);
                if (b + 1 < a.nb) baby(b + 1, 1);
                if (NST > 2 && b + 2 < a.nb) baby(b + 2, 2);
            }
            if (MODE == 0 && active) {
                uint64_t* Ys = a.Y + (size_t)s * a.y_src_stride;
                // the Montgomery factor 2^-90 of every X~ is restored once
                uint64_t r = reduce64(1ULL << 45, pr);
                r = mul_mod(r, r, pr);
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    if (g >= a.ng) break;
                    uint64_t o[2][2];
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2)
                            o[q2][e2] = mul_mod(reduce128(y[g][q2][e2].hi, y[g][q2][e2].lo, pr), r, pr);
                    uint64_t* yg = Ys + (size_t)g * a.y_g_stride;
                    if (a.accumulate) {
                        const ulonglong2 y0 = ld2(yg + i), y1 = ld2(yg + total + i);
                        o[0][0] = add_mod(o[0][0], y0.x, pr.q);
                        o[0][1] = add_mod(o[0][1], y0.y, pr.q);
                        o[1][0] = add_mod(o[1][0], y1.x, pr.q);
                        o[1][1] = add_mod(o[1][1], y1.y, pr.q);
                    }
                    st2(yg + i, o[0][0], o[0][1]);
                    st2(yg + total + i, o[1][0], o[1][1]);
                }
            }
        };
        if (opf_fp(pr.q))
            run_fp();
        else
            run_l30();
    }
}

__global__ void k_rows_to_limb(DevCtx c, uint64_t* dst, const uint64_t* src, size_t nrows, RowMap rm) {
    const size_t total = nrows * (size_t)c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)((i >> c.logN) % (size_t)rm.rows_per_poly);
        const int pi = rm.level < 0 ? r : row_prime(rm, r);
        dst[i] = to_opf(src[i], c.primes[pi].q);
    }
}

// Giant-step inputs of sc sources x G giants in one pass: the c1 rows of Y(s, giant[g])
// copied to yc ([sc][G][ne][N], for the coefficient-domain ModDown) and the c0 rows
// converted to operand form into yc0 (same layout, for k_ks_giant_opf).
__global__ void k_giant_gather(DevCtx c, uint64_t* yc, uint64_t* yc0, const uint64_t* Y, size_t ys, int sc,
                               GiantSel gs, int level) {
    const int ne = level + 1 + c.K;
    const size_t extw = (size_t)ne * c.N, total = (size_t)sc * gs.n * extw;
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t pg = i / extw, w = i - pg * extw;
        const int s = (int)(pg / gs.n), g = (int)(pg % gs.n);
        const uint64_t* y = Y + (size_t)s * ys + (size_t)gs.idx[g] * 2 * extw;
        yc[i] = y[extw + w];
        if (yc0) yc0[i] = to_opf(y[w], c.primes[row_prime(rm, (int)(w >> c.logN))].q);
    }
}

// dst[s][words] = *srcp[s]: the ciphertexts of a batch (separate allocations) gathered into one
// dense buffer in ONE launch (a cudaMemcpyAsync per ciphertext costs ~4 us each: 1 ms of the 7 ms
// keyed rotation of 256 cfg2 ciphertexts)
__global__ void k_gather_ptrs(uint64_t* dst, const uint64_t* const* srcp, size_t words, int nsrc) {
    const size_t per = words / 2, total = per * nsrc;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t s = i / per, w = i - s * per;
        reinterpret_cast<ulonglong2*>(dst)[i] = __ldcs(reinterpret_cast<const ulonglong2*>(srcp[s]) + w);
    }
}

__global__ void k_ct_prescale(DevCtx c, uint64_t* dst, const uint64_t* ct, size_t stride, int nsrc,
                              const ModDownTable* md, int level) {
    const int nr = level + 1;
    const size_t per = (size_t)2 * nr * c.N, total = per * nsrc;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t sidx = i / per, w = i - sidx * per;
        const int u = (int)((w >> c.logN) % (size_t)nr);
        const uint64_t q = c.primes[u].q;
        dst[i] = to_opf(mul_shoup(ct[sidx * stride + w], md->pmod[u], md->pmod_sh[u], q), q);
    }
}

// Giant-step key switches of a batch, accumulated into each source's QP
// accumulator: acc(s) += sum_t (IP_0(D(s,t), key_t) + sigma_t(Y(s,t).c0), IP_1(...)),
// Y.c0 P-scaled in QP (added unscaled on every row). Same staging as
// k_bsgs_fused: thread = (coefficient pair, source), the key rows of a term
// are staged once per CTA for its SG sources, digits/c0 are per source.
template <int DN, int SG>
__global__ void __launch_bounds__(128, 3) k_ks_giant(DevCtx c, KsBatch a, int level) {
    constexpr int P = 128 / SG;
    constexpr int KW = 2 * DN * P, DW = SG * DN * P, CW = SG * P, STAGE = KW + DW + CW;
    extern __shared__ ulonglong2 sb[];  // [2][STAGE]
    const int nr = level + 1, ne = nr + c.K, np = c.L + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / 2 / P;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const size_t keyrow = (size_t)np * c.N;
    RowMap rm{ne, level, c.L, 0};
    ulonglong2* const s_key = sb + p;
    ulonglong2* const s_dig = sb + KW + sl * DN * P + p;
    ulonglong2* const s_c0 = sb + KW + DW + sl * P + p;
    for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
        const size_t chunk = it / (size_t)ngroups;
        const int s = (int)(it % (size_t)ngroups) * SG + sl;
        const bool active = s < a.nsrc;
        const size_t i = (chunk * P + p) * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int pi = row_prime(rm, u);
        const size_t kofs = (size_t)pi * c.N + k;
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, nmask = (2u << c.logN) - 1;
        auto pidx = [&](uint32_t g) { return brev_n((((e * g) & nmask) - 1) >> 1, c.logN); };
        auto issue = [&](int t) {
            const size_t so = (size_t)(t & 1) * STAGE;
            const uint64_t* kp = a.key[t] + kofs;
#pragma unroll
            for (int j = sl; j < 2 * DN; j += SG) cp_async16(s_key + so + j * P, kp + (size_t)j * keyrow);
            if (active) {
                const uint32_t pk = pidx(a.galois[t]) & ~1u;
                const uint64_t* D = a.digits + (size_t)s * a.digit_src_stride + (size_t)t * a.digit_term_stride +
                                    (size_t)u * c.N + pk;
#pragma unroll
                for (int j = 0; j < DN; ++j) cp_async16(s_dig + so + j * P, D + (size_t)j * total);
                cp_async16(s_c0 + so, a.c0 + (size_t)s * a.c0_src_stride + a.c0_off[t] + (size_t)u * c.N + pk);
            }
            cp_async_commit();
        };
        U128 r0a{0, 0}, r0b{0, 0}, r1a{0, 0}, r1b{0, 0};
        issue(0);
        for (int t = 0; t < a.n; ++t) {
            cp_async_wait<0>();
            __syncthreads();
            if (t + 1 < a.n) issue(t + 1);
            const size_t so = (size_t)(t & 1) * STAGE;
            const int swp = (int)(pidx(a.galois[t]) & 1u);
            Acc3 s0a{0, 0, 0, 0}, s0b{0, 0, 0, 0}, s1a{0, 0, 0, 0}, s1b{0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < DN; ++j) {
                const ulonglong2 k0 = s_key[so + (2 * j) * P], k1 = s_key[so + (2 * j + 1) * P];
                const ulonglong2 dv = s_dig[so + j * P];
                const uint64_t da = swp ? dv.y : dv.x, db = swp ? dv.x : dv.y;
                mac3(s0a, da, k0.x);
                mac3(s0b, db, k0.y);
                mac3(s1a, da, k1.x);
                mac3(s1b, db, k1.y);
            }
            const ulonglong2 cv = s_c0[so];
            add3(s0a, swp ? cv.y : cv.x);
            add3(s0b, swp ? cv.x : cv.y);
            auto acc = [](U128& r, const Acc3& x) {
                const U128 f = fold3(x);
                r.lo += f.lo;
                r.hi += f.hi + (r.lo < f.lo);
            };
            acc(r0a, s0a);
            acc(r0b, s0b);
            acc(r1a, s1a);
            acc(r1b, s1b);
        }
        if (active) {
            const Prime pr = c.primes[pi];
            uint64_t* out = a.out + (size_t)s * a.out_src_stride;
            const ulonglong2 a0 = ld2(out + i), a1 = ld2(out + total + i);
            add128(r0a, a0.x);
            add128(r0b, a0.y);
            add128(r1a, a1.x);
            add128(r1b, a1.y);
            st2(out + i, reduce128(r0a.hi, r0a.lo, pr), reduce128(r0b.hi, r0b.lo, pr));
            st2(out + total + i, reduce128(r1a.hi, r1a.lo, pr), reduce128(r1b.hi, r1b.lo, pr));
        }
        __syncthreads();
    }
}

// k_ks_giant on operand-form rows (KsBatch.opf, mode 1): acc(s) += sum_t (IP(D(s,t),
// key_t) + sigma_t(Y(s,t).c0)), the products of rows q < 2^50 on the FP64 pipe (one
// red_d per term keeps the double sums exact), the 60-bit rows on 30-bit limbs.
template <int DN, int SG>
__global__ void __launch_bounds__(128, 4) k_ks_giant_opf(DevCtx c, KsBatch a, int level) {
    constexpr int P = 128 / SG;
    constexpr int KW = 2 * DN * P, DW = SG * DN * P, CW = SG * P, STAGE = KW + DW + CW;
    extern __shared__ ulonglong2 sb[];  // [2][STAGE]
    const int nr = level + 1, ne = nr + c.K, np = c.L + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / 2 / P;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const size_t keyrow = (size_t)np * c.N;
    RowMap rm{ne, level, c.L, 0};
    ulonglong2* const s_key = sb + p;
    ulonglong2* const s_dig = sb + KW + sl * DN * P + p;
    ulonglong2* const s_c0 = sb + KW + DW + sl * P + p;
    constexpr uint32_t MW = (1u << 30) - 1;
    for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
        const size_t chunk = it / (size_t)ngroups;
        const int s = (int)(it % (size_t)ngroups) * SG + sl;
        const bool active = s < a.nsrc;
        const size_t i = (chunk * P + p) * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int pi = row_prime(rm, u);
        const size_t kofs = (size_t)pi * c.N + k;
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, nmask = (2u << c.logN) - 1;
        auto pidx = [&](uint32_t g) { return brev_n((((e * g) & nmask) - 1) >> 1, c.logN); };
        auto issue = [&](int t) {
            const size_t so = (size_t)(t & 1) * STAGE;
            const uint64_t* kp = a.key[t] + kofs;
#pragma unroll
            for (int j = sl; j < 2 * DN; j += SG) cp_async16(s_key + so + j * P, kp + (size_t)j * keyrow);
            if (active) {
                const uint32_t pk = pidx(a.galois[t]) & ~1u;
                const uint64_t* D = a.digits + (size_t)s * a.digit_src_stride + (size_t)t * a.digit_term_stride +
                                    (size_t)u * c.N + pk;
#pragma unroll
                for (int j = 0; j < DN; ++j) cp_async16(s_dig + so + j * P, D + (size_t)j * total);
                cp_async16(s_c0 + so, a.c0 + (size_t)s * a.c0_src_stride + a.c0_off[t] + (size_t)u * c.N + pk);
            }
            cp_async_commit();
        };
        const Prime pr = c.primes[pi];
        const bool fp = opf_fp(pr.q);
        const ArD ad = make_ard(pr.q);
        const ArG ag = fp ? make_arg(ad) : ArG{0.0, 0.0};
        const uint32_t q0 = (uint32_t)(pr.q & MW), q1 = (uint32_t)(pr.q >> 30), qinv = (uint32_t)pr.qinv & MW;
        double zf[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        uint64_t zi[2][2] = {{0, 0}, {0, 0}};  // 60-bit rows: sum of the terms' X 2^-90, reduced
        issue(0);
        for (int t = 0; t < a.n; ++t) {
            cp_async_wait<0>();
            __syncthreads();
            if (t + 1 < a.n) issue(t + 1);
            const size_t so = (size_t)(t & 1) * STAGE;
            const int swp = (int)(pidx(a.galois[t]) & 1u);
            const ulonglong2 cv = s_c0[so];
            const uint64_t ca = swp ? cv.y : cv.x, cb = swp ? cv.x : cv.y;
            if (fp) {
                double z[2][2] = {{kGridBig, kGridBig}, {kGridBig, kGridBig}};
                double zl[2][2] = {{zf[0][0] + asd(ca), zf[0][1] + asd(cb)}, {zf[1][0], zf[1][1]}};
#pragma unroll
                for (int j = 0; j < DN; ++j) {
                    const ulonglong2 k0 = s_key[so + (2 * j) * P], k1 = s_key[so + (2 * j + 1) * P];
                    const ulonglong2 dv = s_dig[so + j * P];
                    const double da = asd(swp ? dv.y : dv.x), db = asd(swp ? dv.x : dv.y);
                    fmag_d(z[0][0], zl[0][0], da, asd(k0.x));
                    fmag_d(z[0][1], zl[0][1], db, asd(k0.y));
                    fmag_d(z[1][0], zl[1][0], da, asd(k1.x));
                    fmag_d(z[1][1], zl[1][1], db, asd(k1.y));
                }
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) zf[q2][e2] = fold_d(z[q2][e2], zl[q2][e2], ad, ag);
            } else {
                uint64_t z0[2][2] = {{0, 0}, {0, 0}}, z1[2][2] = {{0, 0}, {0, 0}}, z2[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
                for (int j = 0; j < DN; ++j) {
                    const ulonglong2 kv0 = s_key[so + (2 * j) * P], kv1 = s_key[so + (2 * j + 1) * P];
                    const ulonglong2 dv = s_dig[so + j * P];
                    const uint64_t dw[2] = {swp ? dv.y : dv.x, swp ? dv.x : dv.y};
                    const uint64_t kw[2][2] = {{kv0.x, kv0.y}, {kv1.x, kv1.y}};
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const uint32_t d0 = lo32(dw[e2]), d1 = hi32(dw[e2]);
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2) {
                            const uint32_t kk0 = lo32(kw[q2][e2]), kk1 = hi32(kw[q2][e2]);
                            madw(z0[q2][e2], d0, kk0);
                            madw(z1[q2][e2], d0, kk1);
                            madw(z1[q2][e2], d1, kk0);
                            madw(z2[q2][e2], d1, kk1);
                        }
                    }
                }
                if constexpr (DN >= 8) {
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) {
                            z2[q2][e2] += z1[q2][e2] >> 30;
                            z1[q2][e2] &= MW;
                        }
                }
                const uint64_t cw[2] = {ca, cb};
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {  // + sigma(Y.c0), every row
                    z0[0][e2] += lo32(cw[e2]);
                    z1[0][e2] += hi32(cw[e2]);
                }
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        uint64_t x = mont_l30(z0[q2][e2], z1[q2][e2], z2[q2][e2], q0, q1, qinv);  // < 2q
                        x = x >= pr.q ? x - pr.q : x;
                        zi[q2][e2] = add_mod(zi[q2][e2], x, pr.q);
                    }
            }
        }
        if (active) {
            uint64_t o[2][2];
            if (fp) {
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) o[q2][e2] = canon_d(zf[q2][e2], ad);
            } else {
                uint64_t r90 = reduce64(1ULL << 45, pr);
                r90 = mul_mod(r90, r90, pr);
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) o[q2][e2] = mul_mod(zi[q2][e2], r90, pr);
            }
            uint64_t* out = a.out + (size_t)s * a.out_src_stride;
            const ulonglong2 a0 = ld2(out + i), a1 = ld2(out + total + i);
            st2(out + i, add_mod(o[0][0], a0.x, pr.q), add_mod(o[0][1], a0.y, pr.q));
            st2(out + total + i, add_mod(o[1][0], a1.x, pr.q), add_mod(o[1][1], a1.y, pr.q));
        }
        __syncthreads();
    }
}

// Hoisted key switches of a batch, one output per (source, term):
// XT(s, slot_t) = (IP_0(D(s), key_t) + [u<=l] P sigma_t(c0(s)), IP_1(D(s), key_t))
// in the QP basis (a ModDown turns it into the rotated ciphertext). Staging
// as k_ks_giant: the key rows of a term are shared by the CTA's SG sources.
template <int DN, int SG>
__global__ void __launch_bounds__(128, 3) k_ks_hoist(DevCtx c, KsBatch a, const ModDownTable* md, int level) {
    constexpr int P = 128 / SG;
    constexpr int KW = 2 * DN * P, DW = SG * DN * P, CW = SG * P, STAGE = KW + DW + CW;
    extern __shared__ ulonglong2 sb[];  // [2][STAGE]
    const int nr = level + 1, ne = nr + c.K, np = c.L + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / 2 / P;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const size_t keyrow = (size_t)np * c.N;
    RowMap rm{ne, level, c.L, 0};
    ulonglong2* const s_key = sb + p;
    ulonglong2* const s_dig = sb + KW + sl * DN * P + p;
    ulonglong2* const s_c0 = sb + KW + DW + sl * P + p;
    for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
        const size_t chunk = it / (size_t)ngroups;
        const int s = (int)(it % (size_t)ngroups) * SG + sl;
        const bool active = s < a.nsrc;
        const size_t i = (chunk * P + p) * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int pi = row_prime(rm, u);
        const bool qrow = u < nr;
        const uint64_t pm = qrow ? md->pmod[u] : 0;
        const size_t kofs = (size_t)pi * c.N + k;
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, nmask = (2u << c.logN) - 1;
        auto pidx = [&](uint32_t g) { return brev_n((((e * g) & nmask) - 1) >> 1, c.logN); };
        const uint64_t* Ds = a.digits + (size_t)(active ? s : 0) * a.digit_src_stride + (size_t)u * c.N;
        const uint64_t* C0 = a.c0 + (size_t)(active ? s : 0) * a.c0_src_stride + (size_t)u * c.N;
        auto issue = [&](int t) {
            const size_t so = (size_t)(t & 1) * STAGE;
            const uint64_t* kp = a.key[t] + kofs;
#pragma unroll
            for (int j = sl; j < 2 * DN; j += SG) cp_async16(s_key + so + j * P, kp + (size_t)j * keyrow);
            if (active) {
                const uint32_t pk = pidx(a.galois[t]) & ~1u;
#pragma unroll
                for (int j = 0; j < DN; ++j) cp_async16(s_dig + so + j * P, Ds + (size_t)j * total + pk);
                if (qrow) cp_async16(s_c0 + so, C0 + pk);
            }
            cp_async_commit();
        };
        const Prime pr = c.primes[pi];
        issue(0);
        for (int t = 0; t < a.n; ++t) {
            cp_async_wait<0>();
            __syncthreads();
            if (t + 1 < a.n) issue(t + 1);
            const size_t so = (size_t)(t & 1) * STAGE;
            const int swp = (int)(pidx(a.galois[t]) & 1u);
            Acc3 s0a{0, 0, 0, 0}, s0b{0, 0, 0, 0}, s1a{0, 0, 0, 0}, s1b{0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < DN; ++j) {
                const ulonglong2 k0 = s_key[so + (2 * j) * P], k1 = s_key[so + (2 * j + 1) * P];
                const ulonglong2 dv = s_dig[so + j * P];
                const uint64_t da = swp ? dv.y : dv.x, db = swp ? dv.x : dv.y;
                mac3(s0a, da, k0.x);
                mac3(s0b, db, k0.y);
                mac3(s1a, da, k1.x);
                mac3(s1b, db, k1.y);
            }
            if (qrow) {
                const ulonglong2 cv = s_c0[so];
                const uint64_t ca = swp ? cv.y : cv.x, cb = swp ? cv.x : cv.y;
                if (DN < 8) {
                    mac3(s0a, ca, pm);
                    mac3(s0b, cb, pm);
                } else {
                    add3(s0a, mul_shoup(ca, pm, md->pmod_sh[u], pr.q));
                    add3(s0b, mul_shoup(cb, pm, md->pmod_sh[u], pr.q));
                }
            }
            if (active) {
                uint64_t* xt = a.out + (size_t)s * a.out_src_stride + (size_t)a.slot[t] * 2 * total;
                const U128 t0a = fold3(s0a), t0b = fold3(s0b), t1a = fold3(s1a), t1b = fold3(s1b);
                st2(xt + i, reduce128(t0a.hi, t0a.lo, pr), reduce128(t0b.hi, t0b.lo, pr));
                st2(xt + total + i, reduce128(t1a.hi, t1a.lo, pr), reduce128(t1b.hi, t1b.lo, pr));
            }
        }
        __syncthreads();
    }
}

// k_ks_hoist on operand-form rows (KsBatch.opf): the same outputs, the products of
// rows q < 2^50 on the FP64 pipe (fmac_d into exact double sums, one red_d), the
// 60-bit rows on 30-bit limbs (four mad.wide.u32 per product, Montgomery by 2^90,
// the factor restored per output). P sigma(c0) enters pre-scaled ([P c0]_q).
template <int DN, int SG>
__global__ void __launch_bounds__(128, 4) k_ks_hoist_opf(DevCtx c, KsBatch a, int level) {
    constexpr int P = 128 / SG;
    constexpr int KW = 2 * DN * P, DW = SG * DN * P, CW = SG * P, STAGE = KW + DW + CW;
    extern __shared__ ulonglong2 sb[];  // [2][STAGE]
    const int nr = level + 1, ne = nr + c.K, np = c.L + c.K;
    const int tid = threadIdx.x, p = tid % P, sl = tid / P;
    const size_t total = (size_t)ne * c.N;
    const size_t chunks = total / 2 / P;
    const int ngroups = (a.nsrc + SG - 1) / SG;
    const size_t items = chunks * (size_t)ngroups;
    const size_t keyrow = (size_t)np * c.N;
    RowMap rm{ne, level, c.L, 0};
    ulonglong2* const s_key = sb + p;
    ulonglong2* const s_dig = sb + KW + sl * DN * P + p;
    ulonglong2* const s_c0 = sb + KW + DW + sl * P + p;
    for (size_t it = blockIdx.x; it < items; it += gridDim.x) {
        const size_t chunk = it / (size_t)ngroups;
        const int s = (int)(it % (size_t)ngroups) * SG + sl;
        const bool active = s < a.nsrc;
        const size_t i = (chunk * P + p) * 2;
        const int u = (int)(i >> c.logN);
        const uint32_t k = (uint32_t)(i & (size_t)(c.N - 1));
        const int pi = row_prime(rm, u);
        const bool qrow = u < nr;
        const size_t kofs = (size_t)pi * c.N + k;
        const uint32_t e = 2 * brev_n(k, c.logN) + 1, nmask = (2u << c.logN) - 1;
        auto pidx = [&](uint32_t g) { return brev_n((((e * g) & nmask) - 1) >> 1, c.logN); };
        const uint64_t* Ds = a.digits + (size_t)(active ? s : 0) * a.digit_src_stride + (size_t)u * c.N;
        const uint64_t* C0 = a.c0 + (size_t)(active ? s : 0) * a.c0_src_stride + (size_t)u * c.N;
        auto issue = [&](int t) {
            const size_t so = (size_t)(t & 1) * STAGE;
            const uint64_t* kp = a.key[t] + kofs;
#pragma unroll
            for (int j = sl; j < 2 * DN; j += SG) cp_async16(s_key + so + j * P, kp + (size_t)j * keyrow);
            if (active) {
                const uint32_t pk = pidx(a.galois[t]) & ~1u;
#pragma unroll
                for (int j = 0; j < DN; ++j) cp_async16(s_dig + so + j * P, Ds + (size_t)j * total + pk);
                if (qrow) cp_async16(s_c0 + so, C0 + pk);
            }
            cp_async_commit();
        };
        const Prime pr = c.primes[pi];
        const bool fp = opf_fp(pr.q);
        const ArD ad = make_ard(pr.q);
        const ArG ag = fp ? make_arg(ad) : ArG{0.0, 0.0};
        constexpr uint32_t MW = (1u << 30) - 1;
        const uint32_t q0 = (uint32_t)(pr.q & MW), q1 = (uint32_t)(pr.q >> 30), qinv = (uint32_t)pr.qinv & MW;
        uint64_t r90 = 0;
        if (!fp) {
            r90 = reduce64(1ULL << 45, pr);
            r90 = mul_mod(r90, r90, pr);
        }
        issue(0);
        for (int t = 0; t < a.n; ++t) {
            cp_async_wait<0>();
            __syncthreads();
            if (t + 1 < a.n) issue(t + 1);
            const size_t so = (size_t)(t & 1) * STAGE;
            const int swp = (int)(pidx(a.galois[t]) & 1u);
            uint64_t o[2][2];
            if (fp) {
                double z[2][2] = {{kGridBig, kGridBig}, {kGridBig, kGridBig}};
                double zl[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
                if (qrow) {
                    const ulonglong2 cv = s_c0[so];
                    zl[0][0] = asd(swp ? cv.y : cv.x);
                    zl[0][1] = asd(swp ? cv.x : cv.y);
                }
#pragma unroll
                for (int j = 0; j < DN; ++j) {
                    const ulonglong2 k0 = s_key[so + (2 * j) * P], k1 = s_key[so + (2 * j + 1) * P];
                    const ulonglong2 dv = s_dig[so + j * P];
                    const double da = asd(swp ? dv.y : dv.x), db = asd(swp ? dv.x : dv.y);
                    fmag_d(z[0][0], zl[0][0], da, asd(k0.x));
                    fmag_d(z[0][1], zl[0][1], db, asd(k0.y));
                    fmag_d(z[1][0], zl[1][0], da, asd(k1.x));
                    fmag_d(z[1][1], zl[1][1], db, asd(k1.y));
                }
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) o[q2][e2] = canon_d(fold_d(z[q2][e2], zl[q2][e2], ad, ag), ad);
            } else {
                uint64_t z0[2][2] = {{0, 0}, {0, 0}}, z1[2][2] = {{0, 0}, {0, 0}}, z2[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
                for (int j = 0; j < DN; ++j) {
                    const ulonglong2 kv0 = s_key[so + (2 * j) * P], kv1 = s_key[so + (2 * j + 1) * P];
                    const ulonglong2 dv = s_dig[so + j * P];
                    const uint64_t dw[2] = {swp ? dv.y : dv.x, swp ? dv.x : dv.y};
                    const uint64_t kw[2][2] = {{kv0.x, kv0.y}, {kv1.x, kv1.y}};
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const uint32_t d0 = lo32(dw[e2]), d1 = hi32(dw[e2]);
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2) {
                            const uint32_t kk0 = lo32(kw[q2][e2]), kk1 = hi32(kw[q2][e2]);
                            madw(z0[q2][e2], d0, kk0);
                            madw(z1[q2][e2], d0, kk1);
                            madw(z1[q2][e2], d1, kk0);
                            madw(z2[q2][e2], d1, kk1);
                        }
                    }
                }
                if constexpr (DN >= 8) {
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                        for (int e2 = 0; e2 < 2; ++e2) {
                            z2[q2][e2] += z1[q2][e2] >> 30;
                            z1[q2][e2] &= MW;
                        }
                }
                if (qrow) {
                    const ulonglong2 cv = s_c0[so];
                    const uint64_t cw[2] = {swp ? cv.y : cv.x, swp ? cv.x : cv.y};
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        z0[0][e2] += lo32(cw[e2]);
                        z1[0][e2] += hi32(cw[e2]);
                    }
                }
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2)
                        o[q2][e2] = mul_mod(mont_l30(z0[q2][e2], z1[q2][e2], z2[q2][e2], q0, q1, qinv), r90, pr);
            }
            if (active) {
                uint64_t* xt = a.out + (size_t)s * a.out_src_stride + (size_t)a.slot[t] * 2 * total;
                st2(xt + i, o[0][0], o[0][1]);
                st2(xt + total + i, o[1][0], o[1][1]);
            }
        }
        __syncthreads();
    }
}

// acc(s) += y(s) for S QP ciphertexts [2][ne][N] at acc + s * as, y + s * ys
__global__ void k_qp_add(DevCtx c, uint64_t* acc, size_t as, const uint64_t* y, size_t ys, int S, int level) {
    const int ne = level + 1 + c.K;
    const size_t per = (size_t)2 * ne * c.N, total = per * S;
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t s = i / per, w = i - s * per;
        const int u = (int)((w >> c.logN) % ne);
        uint64_t* a = acc + s * as + w;
        *a = add_mod(*a, y[s * ys + w], c.primes[row_prime(rm, u)].q);
    }
}

}  // namespace

#define FHE_DN_SWITCH(dn, CALL) \
    switch (dn) {                  \
        case 1: CALL(1); break;    \
        case 2: CALL(2); break;    \
        case 3: CALL(3); break;    \
        case 4: CALL(4); break;    \
        case 5: CALL(5); break;    \
        case 6: CALL(6); break;    \
        case 7: CALL(7); break;    \
        case 8: CALL(8); break;    \
        default: throw std::invalid_argument("unsupported digit count (dnum must be <= 8)"); \
    }

// CTA caps of the HBM-streaming kernels (per SM). Smaller grids leave SM room
// for the integer-bound NTT CTAs of other lanes to co-reside.
static int env_cap(const char* name, int dflt) {
    const char* v = getenv(name);
    const int x = v ? atoi(v) : 0;
    return x > 0 ? x : dflt;
}
static int ks_cap() {
    static const int cap = env_cap("FHECONV_KS_CTAS", 148 * 8);
    return cap;
}
int mv_cap() {  // used by matvec.cu
    static const int cap = env_cap("FHECONV_MV_CTAS", 148 * 12);
    return cap;
}

void ks_stream(const DevCtx& c, const KsStream& a, int mode, const ModDownTable* md, int level, int dn,
               cudaStream_t st) {
    if (a.n <= 0) return;
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    const size_t smem = (size_t)2 * 3 * dn * kStreamThreads * sizeof(ulonglong2);
    int blocks = (int)((total / 2 + kStreamThreads - 1) / kStreamThreads);
    blocks = blocks < ks_cap() ? blocks : ks_cap();
    ++g_launches;
#define FHE_KSS(D)                                                                                             \
    do {                                                                                                       \
        if (mode == 0) {                                                                                       \
            cudaFuncSetAttribute(k_ks_stream<D, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
            k_ks_stream<D, 0><<<blocks, kStreamThreads, smem, st>>>(c, a, md, level);                          \
        } else {                                                                                               \
            cudaFuncSetAttribute(k_ks_stream<D, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
            k_ks_stream<D, 1><<<blocks, kStreamThreads, smem, st>>>(c, a, md, level);                          \
        }                                                                                                      \
    } while (0)
    FHE_DN_SWITCH(dn, FHE_KSS)
#undef FHE_KSS
}

static int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <int DN, int SG>
static void launch_giant(const DevCtx& c, const KsBatch& a, int level, cudaStream_t st) {
    constexpr int P = 128 / SG;
    const size_t smem = (size_t)2 * (2 * DN * P + SG * DN * P + SG * P) * sizeof(ulonglong2);
    const size_t items = (size_t)(level + 1 + c.K) * c.N / 2 / P * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_ks_giant<DN, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ks_giant<DN, SG>, 128, smem);
    const size_t cap = (size_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    k_ks_giant<DN, SG><<<(int)(items < cap ? items : cap), 128, smem, st>>>(c, a, level);
}

template <int DN, int SG>
static void launch_giant_opf(const DevCtx& c, const KsBatch& a, int level, cudaStream_t st) {
    constexpr int P = 128 / SG;
    const size_t smem = (size_t)2 * (2 * DN * P + SG * DN * P + SG * P) * sizeof(ulonglong2);
    const size_t items = (size_t)(level + 1 + c.K) * c.N / 2 / P * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_ks_giant_opf<DN, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ks_giant_opf<DN, SG>, 128, smem);
    const size_t cap = (size_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    k_ks_giant_opf<DN, SG><<<(int)(items < cap ? items : cap), 128, smem, st>>>(c, a, level);
}

template <int DN, int SG>
static void launch_hoist_opf(const DevCtx& c, const KsBatch& a, int level, cudaStream_t st) {
    constexpr int P = 128 / SG;
    const size_t smem = (size_t)2 * (2 * DN * P + SG * DN * P + SG * P) * sizeof(ulonglong2);
    const size_t items = (size_t)(level + 1 + c.K) * c.N / 2 / P * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_ks_hoist_opf<DN, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ks_hoist_opf<DN, SG>, 128, smem);
    const size_t cap = (size_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    k_ks_hoist_opf<DN, SG><<<(int)(items < cap ? items : cap), 128, smem, st>>>(c, a, level);
}

template <int DN, int SG>
static void launch_hoist(const DevCtx& c, const KsBatch& a, const ModDownTable* md, int level, cudaStream_t st) {
    constexpr int P = 128 / SG;
    const size_t smem = (size_t)2 * (2 * DN * P + SG * DN * P + SG * P) * sizeof(ulonglong2);
    const size_t items = (size_t)(level + 1 + c.K) * c.N / 2 / P * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_ks_hoist<DN, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ks_hoist<DN, SG>, 128, smem);
    const size_t cap = (size_t)sm_count() * (per_sm > 0 ? per_sm : 1);
    k_ks_hoist<DN, SG><<<(int)(items < cap ? items : cap), 128, smem, st>>>(c, a, md, level);
}

void ks_batch(const DevCtx& c, const KsBatch& a, int mode, const ModDownTable* md, int level, int dn,
              cudaStream_t st) {
    if (a.n <= 0 || a.nsrc <= 0) return;
    if (mode == 0 && !a.c0_qp) {  // hoisted rotations of a batch: one output per (source, term)
        ++g_launches;
        const int sg = a.nsrc >= 4 ? 4 : a.nsrc >= 2 ? 2 : 1;
#define FHE_HOIST(D)                                                      \
    do {                                                                  \
        if (a.opf) {                                                      \
            if (sg == 4) launch_hoist_opf<D, 4>(c, a, level, st);         \
            else if (sg == 2) launch_hoist_opf<D, 2>(c, a, level, st);    \
            else launch_hoist_opf<D, 1>(c, a, level, st);                 \
        } else {                                                          \
            if (sg == 4) launch_hoist<D, 4>(c, a, md, level, st);         \
            else if (sg == 2) launch_hoist<D, 2>(c, a, md, level, st);    \
            else launch_hoist<D, 1>(c, a, md, level, st);                 \
        }                                                                 \
    } while (0)
        FHE_DN_SWITCH(dn, FHE_HOIST)
#undef FHE_HOIST
        return;
    }
    if (mode == 1 && a.c0_qp) {  // giant steps: staged, key rows shared by the sources of a CTA
        ++g_launches;
        const int sg = a.nsrc >= 4 ? 4 : a.nsrc >= 2 ? 2 : 1;
#define FHE_GIANT(D)                                                     \
    do {                                                                 \
        if (a.opf) {                                                     \
            if (sg == 4) launch_giant_opf<D, 4>(c, a, level, st);        \
            else if (sg == 2) launch_giant_opf<D, 2>(c, a, level, st);   \
            else launch_giant_opf<D, 1>(c, a, level, st);                \
        } else {                                                         \
            if (sg == 4) launch_giant<D, 4>(c, a, level, st);            \
            else if (sg == 2) launch_giant<D, 2>(c, a, level, st);       \
            else launch_giant<D, 1>(c, a, level, st);                    \
        }                                                                \
    } while (0)
        FHE_DN_SWITCH(dn, FHE_GIANT)
#undef FHE_GIANT
        return;
    }
    // the host only builds (mode 0, source c0) and (mode 1, P-scaled QP c0) batches
}


void identity_batch(const DevCtx& c, uint64_t* xt, size_t xt_src_stride, const uint64_t* ct, size_t ct_src_stride,
                    const ModDownTable* md, int level, int nsrc, cudaStream_t st) {
    ++g_launches;
    k_identity_batch<<<ew_blocks((size_t)(level + 1 + c.K) * c.N * nsrc), kEwThreads, 0, st>>>(
        c, xt, xt_src_stride, ct, ct_src_stride, md, level, nsrc);
}

void identity_term(const DevCtx& c, uint64_t* xt, const uint64_t* ct, const ModDownTable* md, int level,
                   cudaStream_t st) {
    ++g_launches;
    k_identity_term<<<ew_blocks((size_t)(level + 1 + c.K) * c.N), kEwThreads, 0, st>>>(c, xt, ct, md, level);
}



#ifndef FHE_FUSED_NST
#define FHE_FUSED_NST 2
#endif
#ifndef FHE_FUSED_MINB
#define FHE_FUSED_MINB 3
#endif
template <int DN, int NG, int SG, int NST = 2, int MINB = 4, bool SLOTS = false>
static void launch_fused(const DevCtx& c, const FusedBsgs& a, const ModDownTable* md, int level, cudaStream_t st) {
    using LY = FusedLayout<DN, NG, SG, NST>;
    const int ne = level + 1 + c.K;
    const size_t smem = (size_t)NST * LY::STAGE * sizeof(ulonglong2);
    const size_t items = (size_t)ne * c.N / 2 / LY::P * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_bsgs_fused<DN, NG, SG, NST, MINB, SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsgs_fused<DN, NG, SG, NST, MINB, SLOTS>, 128, smem);
    if (per_sm < 1) per_sm = 1;
    const size_t cap = (size_t)sm_count() * per_sm;
    const int blocks = (int)(items < cap ? items : cap);
    k_bsgs_fused<DN, NG, SG, NST, MINB, SLOTS><<<blocks, 128, smem, st>>>(c, a, md, level);
}

void bsgs_fused(const DevCtx& c, const FusedBsgs& a, const ModDownTable* md, int level, int dn, cudaStream_t st) {
    if (a.nb <= 0 || a.nsrc <= 0 || a.ng <= 0) return;
    ++g_launches;
    // sources per CTA: 4 (keys/plaintexts shared 4 ways), 2 for pairs, 1 alone;
    // per-baby source slots (paper schedules; the host passes <= 3 giant accumulators)
    const int sg = a.nsrc >= 4 ? 4 : a.nsrc >= 2 ? 2 : 1;
    const bool slots = a.accumulate || a.digit_slot_stride || a.ct_slot_stride;
#define FHE_FUSED(D)                                                                                \
    do {                                                                                            \
        if (slots) {                                                                                \
            if (sg == 4) launch_fused<D, 3, 4, FHE_FUSED_NST, FHE_FUSED_MINB, true>(c, a, md, level, st); \
            else if (sg == 2) launch_fused<D, 3, 2, 2, 3, true>(c, a, md, level, st);               \
            else launch_fused<D, 3, 1, 2, 2, true>(c, a, md, level, st);                            \
        } else if (a.ng <= 3) {                                                                     \
            if (sg == 4) launch_fused<D, 3, 4, FHE_FUSED_NST, FHE_FUSED_MINB>(c, a, md, level, st); \
            else if (sg == 2) launch_fused<D, 3, 2, 2, 3>(c, a, md, level, st);                     \
            else launch_fused<D, 3, 1, 2, 2>(c, a, md, level, st);                                  \
        } else {                                                                                    \
            if (sg == 4) launch_fused<D, kFusedMaxG, 4, 2, 2>(c, a, md, level, st);                 \
            else if (sg == 2) launch_fused<D, kFusedMaxG, 2, 2, 2>(c, a, md, level, st);            \
            else launch_fused<D, kFusedMaxG, 1, 2, 2>(c, a, md, level, st);                         \
        }                                                                                           \
    } while (0)
    FHE_DN_SWITCH(dn, FHE_FUSED)
#undef FHE_FUSED
}

#ifndef FHE_TMA_MINB
#define FHE_TMA_MINB 4
#endif
// Ring depth of the SG >= 8 launches (-DFHE_TMA_WIDE=1 builds). 3 stages fit 3 CTAs per SM and
// lose 7 % against 2 stages at 4 CTAs per SM: the kernel needs its 16 warps per SM more than a
// deeper prefetch (profiles/ab_r02_bsgs_variants.txt).
#ifndef FHE_TMA_NST8
#define FHE_TMA_NST8 2
#endif
#if FHE_TMA_WIDE
#define FHE_TMA_WIDE_CASES(NG_, MINB_, MODE_)                                                 \
    if (sg == 16) { launch_tma<D, NG_, 16, MINB_, MODE_>(c, a, m, level, st); break; }         \
    if (sg == 8) { launch_tma<D, NG_, 8, MINB_, MODE_>(c, a, m, level, st); break; }
#else
#define FHE_TMA_WIDE_CASES(NG_, MINB_, MODE_)
#endif
template <int DN, int NG, int SG, int MINB_, int MODE = 0>
static void launch_tma(const DevCtx& c, const FusedBsgs& a, const TmaMaps& m, int level, cudaStream_t st) {
    using LY = TmaLayout<DN, NG, SG>;
    constexpr int NST = SG >= 8 ? FHE_TMA_NST8 : 2;
    constexpr int MINB = (NST > 2 && MINB_ > 3) ? 3 : MINB_;
    const int ne = level + 1 + c.K;
    const size_t smem = (size_t)NST * LY::STAGE * 16 + 8 * NST;
    const size_t items = (size_t)ne * c.N / (2 * LY::P) * (size_t)((a.nsrc + SG - 1) / SG);
    int per_sm = 0;
    cudaFuncSetAttribute(k_bsgs_tma<DN, NG, SG, MINB, MODE, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsgs_tma<DN, NG, SG, MINB, MODE, NST>, 128, smem);
    if (per_sm < 1) per_sm = 1;
    const size_t cap = (size_t)sm_count() * per_sm;
    const int blocks = (int)(items < cap ? items : cap);
    k_bsgs_tma<DN, NG, SG, MINB, MODE, NST><<<blocks, 128, smem, st>>>(c, a, m, level);
}

void bsgs_tma_hoist(const DevCtx& c, const FusedBsgs& a, const TmaMaps& m, int level, int dn, cudaStream_t st) {
    if (a.nb <= 0 || a.nsrc <= 0) return;
    if (!m.sched) throw std::invalid_argument("bsgs_tma: no work-queue buffer");
    cudaMemsetAsync(m.sched, 0, kTmaSchedWords * sizeof(unsigned), st);
    ++g_launches;
    const int sg = tma_sources(a.nsrc);
#define FHE_TMAH(D)                                                                \
    do {                                                                           \
        FHE_TMA_WIDE_CASES(1, FHE_TMA_MINB, 1)                                     \
        if (sg == 4) launch_tma<D, 1, 4, FHE_TMA_MINB, 1>(c, a, m, level, st); \
        else if (sg == 2) launch_tma<D, 1, 2, 3, 1>(c, a, m, level, st);           \
        else launch_tma<D, 1, 1, 2, 1>(c, a, m, level, st);                        \
    } while (0)
    FHE_DN_SWITCH(dn, FHE_TMAH)
#undef FHE_TMAH
}

void bsgs_tma(const DevCtx& c, const FusedBsgs& a, const TmaMaps& m, int level, int dn, cudaStream_t st) {
    if (a.nb <= 0 || a.nsrc <= 0 || a.ng <= 0) return;
    if (a.ng > kFusedMaxG) throw std::invalid_argument("bsgs_tma: too many giants per launch");
    if (!m.sched) throw std::invalid_argument("bsgs_tma: no work-queue buffer");
    cudaMemsetAsync(m.sched, 0, kTmaSchedWords * sizeof(unsigned), st);
    ++g_launches;
    const int sg = tma_sources(a.nsrc);
#define FHE_TMA(D)                                                               \
    do {                                                                         \
        if (a.ng == 1 && m.ng1) {                                                \
            FHE_TMA_WIDE_CASES(1, FHE_TMA_MINB, 0)                               \
            if (sg == 4) launch_tma<D, 1, 4, FHE_TMA_MINB>(c, a, m, level, st); \
            else if (sg == 2) launch_tma<D, 1, 2, 3>(c, a, m, level, st);        \
            else launch_tma<D, 1, 1, 2>(c, a, m, level, st);                     \
        } else if (a.ng <= 3) {                                                  \
            FHE_TMA_WIDE_CASES(3, FHE_TMA_MINB, 0)                               \
            if (sg == 4) launch_tma<D, 3, 4, FHE_TMA_MINB>(c, a, m, level, st); \
            else if (sg == 2) launch_tma<D, 3, 2, 3>(c, a, m, level, st);        \
            else launch_tma<D, 3, 1, 2>(c, a, m, level, st);                     \
        } else {                                                                 \
            FHE_TMA_WIDE_CASES(kFusedMaxG, 2, 0)                                 \
            if (sg == 4) launch_tma<D, kFusedMaxG, 4, 2>(c, a, m, level, st); \
            else if (sg == 2) launch_tma<D, kFusedMaxG, 2, 2>(c, a, m, level, st); \
            else launch_tma<D, kFusedMaxG, 1, 2>(c, a, m, level, st);            \
        }                                                                        \
    } while (0)
    FHE_DN_SWITCH(dn, FHE_TMA)
#undef FHE_TMA
}

static PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int R>
static void tma_map_r(CUtensorMap* map, const void* base, const uint64_t* dims, const uint32_t* box) {
    cuuint64_t gd[R], gs[R - 1];
    cuuint32_t bx[R], es[R];
    uint64_t stride = 8;
    for (int d = 0; d < R; ++d) {
        es[d] = 1;
        gd[d] = dims[d];
        bx[d] = box[d];
        if (d > 0) gs[d - 1] = stride;
        stride *= dims[d];
    }
    const CUresult r = tma_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, R, const_cast<void*>(base), gd, gs, bx, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed");
}
void tma_map4(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint32_t box[4]) {
    tma_map_r<4>(map, base, dims, box);
}
void tma_map5(CUtensorMap* map, const void* base, const uint64_t dims[5], const uint32_t box[5]) {
    tma_map_r<5>(map, base, dims, box);
}

void rows_to_limb(const DevCtx& c, uint64_t* dst, const uint64_t* src, size_t nrows, const RowMap& rm,
                  cudaStream_t st) {
    ++g_launches;
    k_rows_to_limb<<<ew_blocks(nrows * c.N), kEwThreads, 0, st>>>(c, dst, src, nrows, rm);
}

void giant_gather(const DevCtx& c, uint64_t* yc, uint64_t* yc0, const uint64_t* Y, size_t ys, int sc, const GiantSel& gs,
                  int level, cudaStream_t st) {
    ++g_launches;
    k_giant_gather<<<ew_blocks((size_t)sc * gs.n * (level + 1 + c.K) * c.N), kEwThreads, 0, st>>>(c, yc, yc0, Y, ys, sc,
                                                                                                gs, level);
}

void gather_ptrs(uint64_t* dst, const uint64_t* const* srcp, size_t words, int nsrc, cudaStream_t st) {
    ++g_launches;
    k_gather_ptrs<<<ew_blocks(words / 2 * nsrc), kEwThreads, 0, st>>>(dst, srcp, words, nsrc);
}

void ct_prescale(const DevCtx& c, uint64_t* dst, const uint64_t* ct, size_t stride, int nsrc, const ModDownTable* md,
                 int level, cudaStream_t st) {
    ++g_launches;
    k_ct_prescale<<<ew_blocks((size_t)2 * (level + 1) * c.N * nsrc), kEwThreads, 0, st>>>(c, dst, ct, stride, nsrc,
                                                                                        md, level);
}

void qp_add(const DevCtx& c, uint64_t* acc, const uint64_t* y, int level, cudaStream_t st, int S, size_t as,
            size_t ys) {
    const size_t total = (size_t)2 * (level + 1 + c.K) * c.N * S;
    ++g_launches;
    k_qp_add<<<ew_blocks(total), kEwThreads, 0, st>>>(c, acc, as, y, ys, S, level);
}

uint64_t launches_total() { return g_launches; }

}  // namespace fhe
