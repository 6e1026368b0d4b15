// Negacyclic NTT for sm_100a.
//
// Forward: Cooley-Tukey, natural order in, bit-reversed order out,
// out[i] = a(psi^(2 brv(i) + 1)); inverse: Gentleman-Sande, bit-reversed in,
// natural out, scaled by N^-1. Identical transforms to the golden model
// (oracle/ckks_ref.c ck_ntt_fwd / ck_ntt_inv); only the evaluation
// schedule differs, and modular arithmetic is exact, so outputs match bit
// for bit.
//
// Schedule: N = N1 * B. Phase A runs the log N1 stages whose butterflies
// span "columns" (stride B), phase B the log B stages inside contiguous
// blocks of B words. Inside a phase every thread owns 8 residues in
// registers and runs radix-8 (3-stage) passes; passes exchange data through
// padded shared memory. Phase B gives each block of B = 2^7..2^8 words to one
// or half a warp, so its passes only need __syncwarp.
#include "kernels.cuh"

namespace fhe {

void note_launch(int n);

namespace {

// padded shared-memory index (2-way bank conflicts at worst for 8-byte words)
__device__ __forceinline__ int pad(int x) { return x + (x >> 4); }

// One radix-2^R pass of forward CT butterflies on 8 register values that
// form 8 / 2^R groups. Local vector of n = 2^logn elements, local stage of
// the pass sigma0, global stage offset s0, block index blk:
//   twiddle(stage sigma, x) = 2^(s0+sigma) + blk 2^sigma + x / (2 t_sigma)
template <int R>
__device__ __forceinline__ void fwd_pass(uint64_t (&v)[8], int G0, int logn, int sigma0, int s0, int blk,
                                         const uint64_t* __restrict__ tw, const uint64_t* __restrict__ tws,
                                         uint64_t q) {
    constexpr int GS = 1 << R;
    const uint64_t q2 = 2 * q;
    const int logt = logn - sigma0 - 1;  // distance of the first sub-stage is 2^logt
    const int logd = logt - (R - 1);     // element stride inside a group
#pragma unroll
    for (int g = 0; g < 8 / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logd) << (logd + R)) | (G & ((1 << logd) - 1));
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << (R - 1 - rho);
            const int sig = sigma0 + rho;
            const int base = (1 << (s0 + sig)) + (blk << sig) + (j0 >> (logt + 1 - rho));
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int widx = base + (k >> (R - rho));
                const uint64_t w = __ldg(tw + widx), ws = __ldg(tws + widx);
                // Harvey's lazy CT butterfly: values live in [0, 4q) between stages
                uint64_t U = v[g * GS + k];
                U = U >= q2 ? U - q2 : U;
                const uint64_t V = mul_shoup_lazy(v[g * GS + k + half], w, ws, q);  // [0, 2q)
                v[g * GS + k] = U + V;
                v[g * GS + k + half] = U - V + q2;
            }
        }
    }
}

// element position of register e for a pass of R stages
template <int R>
__device__ __forceinline__ int fwd_pos(int G0, int e, int logn, int sigma0) {
    constexpr int GS = 1 << R;
    const int logt = logn - sigma0 - 1;
    const int logd = logt - (R - 1);
    const int G = G0 + e / GS, k = e % GS;
    const int j0 = ((G >> logd) << (logd + R)) | (G & ((1 << logd) - 1));
    return j0 + (k << logd);
}

// Inverse GS pass of R stages starting at distance 2^logt (t grows):
//   twiddle(t', x) = n_tot / (2 t') + blk n_loc / (2 t') + x / (2 t')
template <int R>
__device__ __forceinline__ void inv_pass(uint64_t (&v)[8], int G0, int logt, int log_ntot, int log_nloc, int blk,
                                         const uint64_t* __restrict__ tw, const uint64_t* __restrict__ tws,
                                         uint64_t q) {
    constexpr int GS = 1 << R;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int g = 0; g < 8 / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logt) << (logt + R)) | (G & ((1 << logt) - 1));
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << rho;
            const int lt = logt + rho;  // current distance 2^lt
            const int base = (1 << (log_ntot - lt - 1)) + (blk << (log_nloc - lt - 1)) + (j0 >> (lt + 1));
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int widx = base + (k >> (rho + 1));
                const uint64_t w = __ldg(tw + widx), ws = __ldg(tws + widx);
                // Harvey's lazy GS butterfly: values live in [0, 2q) between stages
                const uint64_t U = v[g * GS + k], V = v[g * GS + k + half];
                const uint64_t T = U + V;
                v[g * GS + k] = T >= q2 ? T - q2 : T;
                v[g * GS + k + half] = mul_shoup_lazy(U - V + q2, w, ws, q);
            }
        }
    }
}

template <int R>
__device__ __forceinline__ int inv_pos(int G0, int e, int logt) {
    constexpr int GS = 1 << R;
    const int G = G0 + e / GS, k = e % GS;
    const int j0 = ((G >> logt) << (logt + R)) | (G & ((1 << logt) - 1));
    return j0 + (k << logt);
}

// Run all forward stages of a local vector of 2^LOGN elements held in smem
// (element x at vec[pad(x)]); 2^LOGN / 8 cooperating threads, lt = lane.
template <int R, int LOGN, int SIGMA0, bool WARP_SYNC>
__device__ __forceinline__ void fwd_step(uint64_t* vec, int lt, int s0, int blk, const uint64_t* tw,
                                         const uint64_t* tws, uint64_t q) {
    uint64_t v[8];
    const int G0 = lt * (8 >> R);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = vec[pad(fwd_pos<R>(G0, e, LOGN, SIGMA0))];
    fwd_pass<R>(v, G0, LOGN, SIGMA0, s0, blk, tw, tws, q);
#pragma unroll
    for (int e = 0; e < 8; ++e) vec[pad(fwd_pos<R>(G0, e, LOGN, SIGMA0))] = v[e];
    if (WARP_SYNC)
        __syncwarp();
    else
        __syncthreads();
}

template <int LOGN, int SIGMA0, bool WARP_SYNC>
__device__ __forceinline__ void fwd_local(uint64_t* vec, int lt, int s0, int blk, const uint64_t* tw,
                                          const uint64_t* tws, uint64_t q) {
    if constexpr (SIGMA0 < LOGN) {
        constexpr int R = (LOGN - SIGMA0) >= 3 ? 3 : (LOGN - SIGMA0);
        fwd_step<R, LOGN, SIGMA0, WARP_SYNC>(vec, lt, s0, blk, tw, tws, q);
        fwd_local<LOGN, SIGMA0 + R, WARP_SYNC>(vec, lt, s0, blk, tw, tws, q);
    }
}

template <int R, int LOGN, int LOGT, bool WARP_SYNC>
__device__ __forceinline__ void inv_step(uint64_t* vec, int lt, int log_ntot, int blk, const uint64_t* tw,
                                         const uint64_t* tws, uint64_t q) {
    uint64_t v[8];
    const int G0 = lt * (8 >> R);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = vec[pad(inv_pos<R>(G0, e, LOGT))];
    inv_pass<R>(v, G0, LOGT, log_ntot, LOGN, blk, tw, tws, q);
#pragma unroll
    for (int e = 0; e < 8; ++e) vec[pad(inv_pos<R>(G0, e, LOGT))] = v[e];
    if (WARP_SYNC)
        __syncwarp();
    else
        __syncthreads();
}

// inverse passes in growing distance; the first pass takes LOGN mod 3 stages
template <int LOGN, int LOGT, bool WARP_SYNC>
__device__ __forceinline__ void inv_local(uint64_t* vec, int lt, int log_ntot, int blk, const uint64_t* tw,
                                          const uint64_t* tws, uint64_t q) {
    if constexpr (LOGT < LOGN) {
        constexpr int R = (LOGT == 0 && LOGN % 3 != 0) ? LOGN % 3 : 3;
        inv_step<R, LOGN, LOGT, WARP_SYNC>(vec, lt, log_ntot, blk, tw, tws, q);
        inv_local<LOGN, LOGT + R, WARP_SYNC>(vec, lt, log_ntot, blk, tw, tws, q);
    }
}

__device__ __forceinline__ bool skip_row(const RowMap& rm, int row, int u) {
    if (!rm.skip_alpha) return false;
    int j = row / rm.rows_per_poly;
    if (rm.skip_dn) j %= rm.skip_dn;
    const int lo = j * rm.skip_alpha;
    const int hi = min(lo + rm.skip_alpha, rm.level + 1);
    return u >= lo && u < hi;
}

// Phase A (columns). CTA = C columns x N1 rows; N1/8 threads per column.
template <int LOG_N1, int C, bool INVERSE>
__global__ void __launch_bounds__(256) k_ntt_cols(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int N1 = 1 << LOG_N1;
    constexpr int TPC = N1 / 8;           // threads per column
    constexpr int PN = N1 + (N1 >> 4) + 1;  // padded column length (odd in words)
    __shared__ uint64_t sm[C * PN];        // column-major: column cc at sm + cc * PN
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    if (skip_row(rm, row, u)) return;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const int B = c.N >> LOG_N1;
    const int col0 = blockIdx.x * C;
    uint64_t* a = data + (size_t)row * c.N;
    // coalesced load: consecutive threads take consecutive columns of a row
    for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        sm[cc * PN + pad(r)] = a[(size_t)r * B + col0 + cc];
    }
    __syncthreads();
    const int cc = threadIdx.x / TPC, lt = threadIdx.x % TPC;
    if (!INVERSE) {
        fwd_local<LOG_N1, 0, false>(sm + cc * PN, lt, 0, 0, c.tw + (size_t)p * c.N, c.tw_sh + (size_t)p * c.N, q);
    } else {
        inv_local<LOG_N1, 0, false>(sm + cc * PN, lt, LOG_N1, 0, c.itw + (size_t)p * c.N,
                                 c.itw_sh + (size_t)p * c.N, q);
    }
    if (INVERSE) {
        const uint64_t ni = c.ninv[p], nis = c.ninv_sh[p];
        for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
            const int r = i / C, cc2 = i % C;
            a[(size_t)r * B + col0 + cc2] = mul_shoup(sm[cc2 * PN + pad(r)], ni, nis, q);
        }
    } else {
        for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
            const int r = i / C, cc2 = i % C;
            a[(size_t)r * B + col0 + cc2] = sm[cc2 * PN + pad(r)];
        }
    }
}

// Phase B (contiguous blocks of B). CTA = BPC blocks; B/8 threads per block.
template <int LOG_N1, int LOG_B, bool INVERSE>
__global__ void __launch_bounds__(256) k_ntt_rows(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int B = 1 << LOG_B;
    constexpr int TPB = B / 8;
    constexpr int BPC = 256 / TPB;
    constexpr int PB = B + (B >> 4);
    __shared__ uint64_t sm[BPC * PB];
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    if (skip_row(rm, row, u)) return;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const int blk0 = blockIdx.x * BPC;
    uint64_t* a = data + (size_t)row * c.N + (size_t)blk0 * B;
    for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) sm[(i / B) * PB + pad(i % B)] = a[i];
    __syncthreads();
    const int bi = threadIdx.x / TPB, lt = threadIdx.x % TPB;
    constexpr bool WS = TPB <= 32;
    if (!INVERSE) {
        fwd_local<LOG_B, 0, WS>(sm + bi * PB, lt, LOG_N1, blk0 + bi, c.tw + (size_t)p * c.N,
                             c.tw_sh + (size_t)p * c.N, q);
    } else {
        inv_local<LOG_B, 0, WS>(sm + bi * PB, lt, LOG_N1 + LOG_B, blk0 + bi, c.itw + (size_t)p * c.N,
                             c.itw_sh + (size_t)p * c.N, q);
    }
    __syncthreads();
    if (!INVERSE) {
        // forward transform ends here: normalise [0, 4q) -> [0, q)
        const uint64_t q2 = 2 * q;
        for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) {
            uint64_t x = sm[(i / B) * PB + pad(i % B)];
            x = x >= q2 ? x - q2 : x;
            a[i] = x >= q ? x - q : x;
        }
    } else {
        for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) a[i] = sm[(i / B) * PB + pad(i % B)];
    }
}

template <int LOG_N1, int LOG_B>
void ntt_dispatch(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, bool inverse, cudaStream_t st) {
    constexpr int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    constexpr int C = 256 / (N1 / 8);
    constexpr int BPC = 256 / (B / 8);
    const dim3 ga(B / C, nrows), gb((N1 + BPC - 1) / BPC, nrows);
    if (!inverse) {
        k_ntt_cols<LOG_N1, C, false><<<ga, 256, 0, st>>>(c, data, rm);
        k_ntt_rows<LOG_N1, LOG_B, false><<<gb, 256, 0, st>>>(c, data, rm);
    } else {
        k_ntt_rows<LOG_N1, LOG_B, true><<<gb, 256, 0, st>>>(c, data, rm);
        k_ntt_cols<LOG_N1, C, true><<<ga, 256, 0, st>>>(c, data, rm);
    }
    note_launch(2);
}

}  // namespace

static void ntt_run(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, bool inverse, cudaStream_t st) {
    if (nrows <= 0) return;
    switch (c.logN) {
        case 12: ntt_dispatch<6, 6>(c, data, nrows, rm, inverse, st); break;
        case 13: ntt_dispatch<6, 7>(c, data, nrows, rm, inverse, st); break;
        case 14: ntt_dispatch<7, 7>(c, data, nrows, rm, inverse, st); break;
        case 15: ntt_dispatch<7, 8>(c, data, nrows, rm, inverse, st); break;
        case 16: ntt_dispatch<8, 8>(c, data, nrows, rm, inverse, st); break;
        default: break;
    }
}

void ntt_forward(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    ntt_run(c, data, nrows, rm, false, st);
}

void ntt_inverse(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    ntt_run(c, data, nrows, rm, true, st);
}

}  // namespace fhe
