// sm_100a kernels of the RNS-CKKS encrypted-convolution hot path.
//
// Layout: residues are uint64 in [0, q), one row of N words
// per (poly, prime), rows contiguous ([poly][prime][N]); NTT rows are in
// bit-reversed evaluation order, so every Galois automorphism maps aligned
// 2^b blocks to aligned 2^b blocks and the permuted gathers below stay
// inside 256-byte segments.
#include "kernels.cuh"
#include "cdt_table.h"

namespace fhe {

namespace {

uint64_t g_launches = 0;  // every kernel this library enqueues (host-side count)

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

// ----------------------------------------------------------------- NTT
// Forward negacyclic NTT split as N = N1 * B:
//  phase A: the first log N1 Cooley-Tukey stages act on "columns" (stride B)
//  phase B: the last log B stages act on contiguous blocks of B words.
// The inverse runs the Gentleman-Sande stages in the mirrored order.

template <int LOG_N1, int C>
__global__ void __launch_bounds__(256) k_ntt_fwd_a(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int N1 = 1 << LOG_N1;
    __shared__ uint64_t s[N1 * C];
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    if (rm.skip_alpha) {
        const int j = row / rm.rows_per_poly, lo = j * rm.skip_alpha;
        const int hi = min(lo + rm.skip_alpha, rm.level + 1);
        if (u >= lo && u < hi) return;
    }
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const uint64_t* tw = c.tw + (size_t)p * c.N;
    const uint64_t* tws = c.tw_sh + (size_t)p * c.N;
    const int B = c.N >> LOG_N1;
    const int col0 = blockIdx.x * C;
    uint64_t* a = data + (size_t)row * c.N;
    for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        s[i] = a[(size_t)r * B + col0 + cc];
    }
    __syncthreads();
    for (int m = 1; m < N1; m <<= 1) {
        const int tr = N1 / (2 * m);
        for (int bf = threadIdx.x; bf < (N1 / 2) * C; bf += blockDim.x) {
            const int cc = bf % C, b = bf / C;
            const int g = b / tr;
            const int r = g * 2 * tr + (b % tr);
            const uint64_t w = tw[m + g], ws = tws[m + g];
            const uint64_t U = s[r * C + cc];
            const uint64_t V = mul_shoup(s[(r + tr) * C + cc], w, ws, q);
            s[r * C + cc] = add_mod(U, V, q);
            s[(r + tr) * C + cc] = sub_mod(U, V, q);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        a[(size_t)r * B + col0 + cc] = s[i];
    }
}

template <int LOG_B>
__global__ void __launch_bounds__(128) k_ntt_fwd_b(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int B = 1 << LOG_B;
    __shared__ uint64_t s[B];
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    if (rm.skip_alpha) {
        const int j = row / rm.rows_per_poly, lo = j * rm.skip_alpha;
        const int hi = min(lo + rm.skip_alpha, rm.level + 1);
        if (u >= lo && u < hi) return;
    }
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const uint64_t* tw = c.tw + (size_t)p * c.N;
    const uint64_t* tws = c.tw_sh + (size_t)p * c.N;
    const int blk = blockIdx.x;
    uint64_t* a = data + (size_t)row * c.N + (size_t)blk * B;
    for (int i = threadIdx.x; i < B; i += blockDim.x) s[i] = a[i];
    __syncthreads();
    const int N1 = c.N >> LOG_B;
    int t = B / 2;
    for (int m = N1; m < c.N; m <<= 1, t >>= 1) {
        for (int bf = threadIdx.x; bf < B / 2; bf += blockDim.x) {
            const int g = bf / t;
            const int j = g * 2 * t + (bf % t);
            const int widx = m + blk * (B / (2 * t)) + g;
            const uint64_t U = s[j];
            const uint64_t V = mul_shoup(s[j + t], tw[widx], tws[widx], q);
            s[j] = add_mod(U, V, q);
            s[j + t] = sub_mod(U, V, q);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < B; i += blockDim.x) a[i] = s[i];
}

template <int LOG_B>
__global__ void __launch_bounds__(128) k_ntt_inv_b(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int B = 1 << LOG_B;
    __shared__ uint64_t s[B];
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const uint64_t* tw = c.itw + (size_t)p * c.N;
    const uint64_t* tws = c.itw_sh + (size_t)p * c.N;
    const int blk = blockIdx.x;
    uint64_t* a = data + (size_t)row * c.N + (size_t)blk * B;
    for (int i = threadIdx.x; i < B; i += blockDim.x) s[i] = a[i];
    __syncthreads();
    int h = c.N / 2;
    for (int t = 1; t <= B / 2; t <<= 1, h >>= 1) {
        for (int bf = threadIdx.x; bf < B / 2; bf += blockDim.x) {
            const int g = bf / t;
            const int j = g * 2 * t + (bf % t);
            const int widx = h + blk * (B / (2 * t)) + g;
            const uint64_t U = s[j], V = s[j + t];
            s[j] = add_mod(U, V, q);
            s[j + t] = mul_shoup(sub_mod(U, V, q), tw[widx], tws[widx], q);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < B; i += blockDim.x) a[i] = s[i];
}

template <int LOG_N1, int C>
__global__ void __launch_bounds__(256) k_ntt_inv_a(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int N1 = 1 << LOG_N1;
    __shared__ uint64_t s[N1 * C];
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const uint64_t* tw = c.itw + (size_t)p * c.N;
    const uint64_t* tws = c.itw_sh + (size_t)p * c.N;
    const int B = c.N >> LOG_N1;
    const int col0 = blockIdx.x * C;
    uint64_t* a = data + (size_t)row * c.N;
    for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        s[i] = a[(size_t)r * B + col0 + cc];
    }
    __syncthreads();
    for (int tr = 1; tr < N1; tr <<= 1) {
        const int h = N1 / (2 * tr);
        for (int bf = threadIdx.x; bf < (N1 / 2) * C; bf += blockDim.x) {
            const int cc = bf % C, b = bf / C;
            const int g = b / tr;
            const int r = g * 2 * tr + (b % tr);
            const uint64_t U = s[r * C + cc], V = s[(r + tr) * C + cc];
            s[r * C + cc] = add_mod(U, V, q);
            s[(r + tr) * C + cc] = mul_shoup(sub_mod(U, V, q), tw[h + g], tws[h + g], q);
        }
        __syncthreads();
    }
    const uint64_t ni = c.ninv[p], nis = c.ninv_sh[p];
    for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        a[(size_t)r * B + col0 + cc] = mul_shoup(s[i], ni, nis, q);
    }
}

constexpr int kCols = 16;

template <int LOG_N1, int LOG_B>
void ntt_fwd_dispatch(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    const int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    ++g_launches;
    k_ntt_fwd_a<LOG_N1, kCols><<<dim3(B / kCols, nrows), 256, 0, st>>>(c, data, rm);
    ++g_launches;
    k_ntt_fwd_b<LOG_B><<<dim3(N1, nrows), 128, 0, st>>>(c, data, rm);
}
template <int LOG_N1, int LOG_B>
void ntt_inv_dispatch(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    const int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    ++g_launches;
    k_ntt_inv_b<LOG_B><<<dim3(N1, nrows), 128, 0, st>>>(c, data, rm);
    ++g_launches;
    k_ntt_inv_a<LOG_N1, kCols><<<dim3(B / kCols, nrows), 256, 0, st>>>(c, data, rm);
}

}  // namespace

void ntt_forward(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    if (nrows <= 0) return;
    switch (c.logN) {
        case 12: ntt_fwd_dispatch<6, 6>(c, data, nrows, rm, st); break;
        case 13: ntt_fwd_dispatch<6, 7>(c, data, nrows, rm, st); break;
        case 14: ntt_fwd_dispatch<7, 7>(c, data, nrows, rm, st); break;
        case 15: ntt_fwd_dispatch<7, 8>(c, data, nrows, rm, st); break;
        case 16: ntt_fwd_dispatch<8, 8>(c, data, nrows, rm, st); break;
        default: break;
    }
}

void ntt_inverse(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    if (nrows <= 0) return;
    switch (c.logN) {
        case 12: ntt_inv_dispatch<6, 6>(c, data, nrows, rm, st); break;
        case 13: ntt_inv_dispatch<6, 7>(c, data, nrows, rm, st); break;
        case 14: ntt_inv_dispatch<7, 7>(c, data, nrows, rm, st); break;
        case 15: ntt_inv_dispatch<7, 8>(c, data, nrows, rm, st); break;
        case 16: ntt_inv_dispatch<8, 8>(c, data, nrows, rm, st); break;
        default: break;
    }
}

// ------------------------------------------------------------ sampling
namespace {

__constant__ uint64_t c_cdt[FHE_CDT_LEN] = {FHE_CDT_VALUES};

__global__ void k_reduce_signed_rows(DevCtx c, const int64_t* coef, uint64_t* out, int nrows, RowMap rm) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / c.N);
        const int k = (int)(i % c.N);
        const Prime pr = c.primes[row_prime(rm, r % rm.rows_per_poly)];
        out[i] = reduce_signed(coef[k], pr);
    }
}

__global__ void k_sample_uniform(DevCtx c, uint64_t* out, int nrows, RowMap rm, uint64_t key) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / c.N);
        const int k = (int)(i % c.N);
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
                                 uint32_t galois, int lo, int hi, const ModDownTable* md, int nrows) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)(i / c.N);
        const uint32_t k = (uint32_t)(i % c.N);
        const Prime pr = c.primes[t];
        uint64_t v = sub_mod(e[i], mul_mod(a[i], s[i], pr), pr.q);
        if (t >= lo && t < hi) {
            const uint64_t sp = s[(size_t)t * c.N + perm_index(k, galois, c.logN)];
            v = add_mod(v, mul_shoup(sp, md->pmod[t], md->pmod_sh[t], pr.q), pr.q);
        }
        b[i] = v;
    }
}

__global__ void k_encrypt_combine(DevCtx c, uint64_t* c0, const uint64_t* c1, const uint64_t* e,
                                  const uint64_t* s, const uint64_t* pt, int nrows) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const Prime pr = c.primes[i / c.N];
        const uint64_t v = sub_mod(e[i], mul_mod(c1[i], s[i], pr), pr.q);
        c0[i] = add_mod(v, pt[i], pr.q);
    }
}

__global__ void k_decrypt_combine(DevCtx c, uint64_t* m, const uint64_t* c0, const uint64_t* c1,
                                  const uint64_t* s, int nrows) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const Prime pr = c.primes[i / c.N];
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
                    cudaStream_t st) {
    ++g_launches;
    k_keygen_combine<<<ew_blocks((size_t)nrows * c.N), kEwThreads, 0, st>>>(c, key_b, key_a, e, s, galois, lo,
                                                                              hi, md, nrows);
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
        const int u = (int)((i / c.N) % rpp);
        const Prime pr = c.primes[u];
        if (OP == 0) out[i] = add_mod(a[i], b[i], pr.q);
        if (OP == 1) out[i] = sub_mod(a[i], b[i], pr.q);
        if (OP == 2) out[i] = mul_mod(a[i], b[i % polyw], pr);
    }
}

__global__ void k_automorph(DevCtx c, uint64_t* out, const uint64_t* in, int nrows, uint32_t g) {
    const size_t total = (size_t)nrows * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const size_t r = i / c.N;
        const uint32_t k = (uint32_t)(i % c.N);
        out[i] = in[r * c.N + perm_index(k, g, c.logN)];
    }
}

__global__ void k_rescale_spread(DevCtx c, const uint64_t* tmp, uint64_t* spread, int level) {
    const size_t total = (size_t)2 * level * c.N;
    const uint64_t ql = c.primes[level].q;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / c.N);
        const int p = r / level, t = r % level;
        const int k = (int)(i % c.N);
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
        const int r = (int)(i / c.N);
        const int p = r / level, t = r % level;
        const int k = (int)(i % c.N);
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
__global__ void k_modup_bconv(DevCtx c, const uint64_t* coef, const uint64_t* c1_ntt, uint64_t* digits,
                              const ModUpDigit* tables, int level, int dn) {
    const int ne = level + 1 + c.K;
    const size_t total = (size_t)dn * c.N;
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(i / c.N);
        const int k = (int)(i % c.N);
        const ModUpDigit& T = tables[j];
        uint64_t v[kMaxAlpha];
        int neg = 0;
        const int na = T.hi - T.lo;
#pragma unroll
        for (int a = 0; a < kMaxAlpha; ++a) {
            if (a < na) {
                const int qi = T.lo + a;
                const uint64_t q = c.primes[qi].q;
                v[a] = mul_shoup(coef[(size_t)qi * c.N + k], T.inv[a], T.inv_sh[a], q);
                neg += v[a] > (q >> 1);
            }
        }
        uint64_t* dj = digits + (size_t)j * ne * c.N + k;
        for (int u = 0; u < ne; ++u) {
            if (u >= T.lo && u < T.hi) {
                dj[(size_t)u * c.N] = c1_ntt[(size_t)u * c.N + k];
                continue;
            }
            const uint64_t t = c.primes[row_prime(rm, u)].q;
            uint64_t acc = 0;
#pragma unroll
            for (int a = 0; a < kMaxAlpha; ++a)
                if (a < na) acc = add_mod(acc, mul_shoup(v[a], T.hat[u][a], T.hat_sh[u][a], t), t);
            // centered lift: each v > q_i/2 stands for v - q_i, i.e. -Q_J
            for (int n = 0; n < neg; ++n) acc = sub_mod(acc, T.qj[u], t);
            dj[(size_t)u * c.N] = acc;
        }
    }
}

__global__ void k_ks_inner(DevCtx c, const uint64_t* D, const uint64_t* key, uint64_t* acc0, uint64_t* acc1,
                           uint32_t g, int level, int dn) {
    const int ne = level + 1 + c.K;
    const int np = c.L + c.K;
    const size_t total = (size_t)ne * c.N;
    RowMap rm{ne, level, c.L, 0};
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int u = (int)(i / c.N);
        const uint32_t k = (uint32_t)(i % c.N);
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

__global__ void k_gather_special(DevCtx c, uint64_t* dst, const uint64_t* acc, int level, int npoly) {
    const int ne = level + 1 + c.K;
    const size_t total = (size_t)npoly * c.K * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / c.N);
        const int p = r / c.K, kk = r % c.K;
        dst[i] = acc[((size_t)p * ne + level + 1 + kk) * c.N + (i % c.N)];
    }
}

__global__ void k_moddown_bconv(DevCtx c, const uint64_t* pcoef, uint64_t* conv, const ModDownTable* md, int level,
                                int npoly) {
    const int nr = level + 1;
    const size_t total = (size_t)npoly * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int p = (int)(i / c.N);
        const int k = (int)(i % c.N);
        uint64_t v[kMaxAlpha];
        int neg = 0;
#pragma unroll
        for (int a = 0; a < kMaxAlpha; ++a) {
            if (a < c.K) {
                const uint64_t q = c.primes[c.L + a].q;
                v[a] = mul_shoup(pcoef[((size_t)p * c.K + a) * c.N + k], md->pinv[a], md->pinv_sh[a], q);
                neg += v[a] > (q >> 1);
            }
        }
        for (int t = 0; t < nr; ++t) {
            const uint64_t q = c.primes[t].q;
            uint64_t acc = 0;
#pragma unroll
            for (int a = 0; a < kMaxAlpha; ++a)
                if (a < c.K) acc = add_mod(acc, mul_shoup(v[a], md->hat[t][a], md->hat_sh[t][a], q), q);
            for (int n = 0; n < neg; ++n) acc = sub_mod(acc, md->pmod[t], q);
            conv[((size_t)p * nr + t) * c.N + k] = acc;
        }
    }
}

__global__ void k_moddown_finish(DevCtx c, uint64_t* out, const uint64_t* acc, const uint64_t* conv,
                                 const ModDownTable* md, int level, int npoly, const uint64_t* add_src,
                                 uint32_t g) {
    const int nr = level + 1, ne = nr + c.K;
    const size_t total = (size_t)npoly * nr * c.N;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / c.N);
        const int p = r / nr, t = r % nr;
        const uint32_t k = (uint32_t)(i % c.N);
        const uint64_t q = c.primes[t].q;
        const uint64_t x = acc[((size_t)p * ne + t) * c.N + k];
        uint64_t o = mul_shoup(sub_mod(x, conv[i], q), md->pinvq[t], md->pinvq_sh[t], q);
        if (add_src && p == 0) o = add_mod(o, add_src[(size_t)t * c.N + perm_index(k, g, c.logN)], q);
        out[i] = o;
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
        const int u = (int)(i / c.N);
        const uint32_t k = (uint32_t)(i % c.N);
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

void modup_bconv(const DevCtx& c, const uint64_t* coef, const uint64_t* c1_ntt, uint64_t* digits,
                 const ModUpDigit* tables, int level, int dn, cudaStream_t st) {
    ++g_launches;
    k_modup_bconv<<<ew_blocks((size_t)dn * c.N), kEwThreads, 0, st>>>(c, coef, c1_ntt, digits, tables, level, dn);
}
void ks_inner_product(const DevCtx& c, const uint64_t* digits, const uint64_t* key, uint64_t* acc0,
                      uint64_t* acc1, uint32_t galois, int level, int dn, cudaStream_t st) {
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    ++g_launches;
    k_ks_inner<<<ew_blocks(total), kEwThreads, 0, st>>>(c, digits, key, acc0, acc1, galois, level, dn);
}
void gather_special(const DevCtx& c, uint64_t* dst, const uint64_t* acc, int level, int npoly, cudaStream_t st) {
    ++g_launches;
    k_gather_special<<<ew_blocks((size_t)npoly * c.K * c.N), kEwThreads, 0, st>>>(c, dst, acc, level, npoly);
}
void moddown_bconv(const DevCtx& c, const uint64_t* pcoef, uint64_t* conv, const ModDownTable* md, int level,
                   int npoly, cudaStream_t st) {
    ++g_launches;
    k_moddown_bconv<<<ew_blocks((size_t)npoly * c.N), kEwThreads, 0, st>>>(c, pcoef, conv, md, level, npoly);
}
void moddown_finish(const DevCtx& c, uint64_t* out, const uint64_t* acc, const uint64_t* conv,
                    const ModDownTable* md, int level, int npoly, const uint64_t* add_src, uint32_t galois,
                    cudaStream_t st) {
    ++g_launches;
    k_moddown_finish<<<ew_blocks((size_t)npoly * (level + 1) * c.N), kEwThreads, 0, st>>>(
        c, out, acc, conv, md, level, npoly, add_src, galois);
}
void conv_mac(const DevCtx& c, uint64_t* acc, const uint64_t* digits, const uint64_t* x, const MacTerms& t,
              const ModDownTable* md, int level, int dn, cudaStream_t st) {
    const size_t total = (size_t)(level + 1 + c.K) * c.N;
    ++g_launches;
    k_conv_mac<<<ew_blocks(total), 256, 0, st>>>(c, acc, digits, x, t, md, level, dn);
}

uint64_t launches_total() { return g_launches; }

}  // namespace fhe
