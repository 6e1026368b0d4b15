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

#ifndef FHE_NTT_EPT
#define FHE_NTT_EPT 16
#endif
constexpr int EPT = FHE_NTT_EPT;         // residues per thread in a pass
constexpr int LOG_EPT = EPT == 16 ? 4 : 3;

// One radix-2^R pass of forward CT butterflies on EPT register values that
// form EPT / 2^R groups. Local vector of n = 2^logn elements, local stage of
// the pass sigma0, global stage offset s0, block index blk:
//   twiddle(stage sigma, x) = 2^(s0+sigma) + blk 2^sigma + x / (2 t_sigma)
template <int R>
__device__ __forceinline__ void fwd_pass(uint64_t (&v)[EPT], int G0, int logn, int sigma0, int s0, int blk,
                                         const uint64_t* __restrict__ tw, const uint64_t* __restrict__ tws,
                                         uint64_t q) {
    constexpr int GS = 1 << R;
    const uint64_t q2 = 2 * q;
    const int logt = logn - sigma0 - 1;  // distance of the first sub-stage is 2^logt
    const int logd = logt - (R - 1);     // element stride inside a group
#pragma unroll
    for (int g = 0; g < EPT / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logd) << (logd + R)) | (G & ((1 << logd) - 1));
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << (R - 1 - rho);
            const int sig = sigma0 + rho;
            const int base = (1 << (s0 + sig)) + (blk << sig) + (j0 >> (logt + 1 - rho));
            const uint64_t* twb = tw + base;
            const uint64_t* twsb = tws + base;
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int off = k >> (R - rho);
                const uint64_t w = __ldg(twb + off), ws = __ldg(twsb + off);
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
__device__ __forceinline__ void inv_pass(uint64_t (&v)[EPT], int G0, int logt, int log_ntot, int log_nloc, int blk,
                                         const uint64_t* __restrict__ tw, const uint64_t* __restrict__ tws,
                                         uint64_t q) {
    constexpr int GS = 1 << R;
    const uint64_t q2 = 2 * q;
#pragma unroll
    for (int g = 0; g < EPT / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logt) << (logt + R)) | (G & ((1 << logt) - 1));
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << rho;
            const int lt = logt + rho;  // current distance 2^lt
            const int base = (1 << (log_ntot - lt - 1)) + (blk << (log_nloc - lt - 1)) + (j0 >> (lt + 1));
            const uint64_t* twb = tw + base;
            const uint64_t* twsb = tws + base;
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int off = k >> (rho + 1);
                const uint64_t w = __ldg(twb + off), ws = __ldg(twsb + off);
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
// (element x at vec[pad(x)]); 2^LOGN / EPT cooperating threads, lt = lane.
template <int R, int LOGN, int SIGMA0, bool WARP_SYNC>
__device__ __forceinline__ void fwd_step(uint64_t* vec, int lt, int s0, int blk, const uint64_t* tw,
                                         const uint64_t* tws, uint64_t q) {
    uint64_t v[EPT];
    const int G0 = lt * (EPT >> R);
#pragma unroll
    for (int e = 0; e < EPT; ++e) v[e] = vec[pad(fwd_pos<R>(G0, e, LOGN, SIGMA0))];
    fwd_pass<R>(v, G0, LOGN, SIGMA0, s0, blk, tw, tws, q);
#pragma unroll
    for (int e = 0; e < EPT; ++e) vec[pad(fwd_pos<R>(G0, e, LOGN, SIGMA0))] = v[e];
    if (WARP_SYNC)
        __syncwarp();
    else
        __syncthreads();
}

template <int LOGN, int SIGMA0, bool WARP_SYNC>
__device__ __forceinline__ void fwd_local(uint64_t* vec, int lt, int s0, int blk, const uint64_t* tw,
                                          const uint64_t* tws, uint64_t q) {
    if constexpr (SIGMA0 < LOGN) {
        constexpr int R = (LOGN - SIGMA0) >= LOG_EPT ? LOG_EPT : (LOGN - SIGMA0);
        fwd_step<R, LOGN, SIGMA0, WARP_SYNC>(vec, lt, s0, blk, tw, tws, q);
        fwd_local<LOGN, SIGMA0 + R, WARP_SYNC>(vec, lt, s0, blk, tw, tws, q);
    }
}

template <int R, int LOGN, int LOGT, bool WARP_SYNC>
__device__ __forceinline__ void inv_step(uint64_t* vec, int lt, int log_ntot, int blk, const uint64_t* tw,
                                         const uint64_t* tws, uint64_t q) {
    uint64_t v[EPT];
    const int G0 = lt * (EPT >> R);
#pragma unroll
    for (int e = 0; e < EPT; ++e) v[e] = vec[pad(inv_pos<R>(G0, e, LOGT))];
    inv_pass<R>(v, G0, LOGT, log_ntot, LOGN, blk, tw, tws, q);
#pragma unroll
    for (int e = 0; e < EPT; ++e) vec[pad(inv_pos<R>(G0, e, LOGT))] = v[e];
    if (WARP_SYNC)
        __syncwarp();
    else
        __syncthreads();
}

// inverse passes in growing distance; the first pass takes LOGN mod LOG_EPT stages
template <int LOGN, int LOGT, bool WARP_SYNC>
__device__ __forceinline__ void inv_local(uint64_t* vec, int lt, int log_ntot, int blk, const uint64_t* tw,
                                          const uint64_t* tws, uint64_t q) {
    if constexpr (LOGT < LOGN) {
        constexpr int R = (LOGT == 0 && LOGN % LOG_EPT != 0) ? LOGN % LOG_EPT : LOG_EPT;
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

// Fused-operand modes of the two NTT passes:
//  FUSE_NONE    : transform `data` in place;
//  FUSE_MODUP   : forward; the column pass computes ModUp's FastBConv of the
//                 digit on the fly from the INTT'd source rows and writes the
//                 digit rows (own-prime rows are copied from the NTT input);
//  FUSE_MODDOWN : forward; the column pass computes ModDown's FastBConv of the
//                 special-prime rows, the row pass writes
//                 out = (acc - NTT(conv)) P^-1 (+ sigma_g(add_src) on poly 0).
enum { FUSE_NONE = 0, FUSE_MODUP = 1, FUSE_MODDOWN = 2 };

// Phase A (columns). CTA = C columns x N1 rows; N1/8 threads per column.
template <int LOG_N1, int C, bool INVERSE, int FUSE>
__global__ void __launch_bounds__(256) k_ntt_cols(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz) {
    constexpr int N1 = 1 << LOG_N1;
    constexpr int TPC = N1 / EPT;             // threads per column
    constexpr int PN = N1 + (N1 >> 4) + 1;    // padded column length (odd in words)
    __shared__ uint64_t sm[C * PN];            // column-major: column cc at sm + cc * PN
    const int row = blockIdx.y;
    const int u = row % rm.rows_per_poly;
    const int B = c.N >> LOG_N1;
    const int col0 = blockIdx.x * C;
    uint64_t* a = data + (size_t)row * c.N;
    int p;
    if (FUSE == FUSE_MODUP) {
        // row = (src, digit j, extended row u)
        const int sj = row / rm.rows_per_poly;
        const int src = sj / fz.dn, j = sj % fz.dn;
        const ModUpDigit& T = fz.mu[j];
        const uint64_t* c1 = fz.c1 + (size_t)src * fz.c1_stride;
        if (u >= T.lo && u < T.hi) {  // own prime of the digit: NTT-domain copy
            for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
                const size_t pos = (size_t)(i / C) * B + col0 + i % C;
                a[pos] = c1[(size_t)u * c.N + pos];
            }
            return;
        }
        p = row_prime(rm, u);
        const uint64_t t = c.primes[p].q;
        const int na = T.hi - T.lo;
        const uint64_t* coef = fz.coef + (size_t)src * (rm.level + 1) * c.N;
        for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
            const int r = i / C, cc = i % C;
            const size_t pos = (size_t)r * B + col0 + cc;
            uint64_t y = 0;
            int neg = 0;
#pragma unroll
            for (int al = 0; al < kMaxAlpha; ++al) {
                if (al < na) {
                    const int qi = T.lo + al;
                    const uint64_t q = c.primes[qi].q;
                    const uint64_t v = mul_shoup(coef[(size_t)qi * c.N + pos], T.inv[al], T.inv_sh[al], q);
                    neg += v > (q >> 1);
                    y = add_mod(y, mul_shoup(v, T.hat[u][al], T.hat_sh[u][al], t), t);
                }
            }
            for (int n = 0; n < neg; ++n) y = sub_mod(y, T.qj[u], t);  // centered lift
            sm[cc * PN + pad(r)] = y;
        }
    } else if (FUSE == FUSE_MODDOWN) {
        // row = (poly pp, q row t); FastBConv of the K special-prime coefficients
        const int pp = row / rm.rows_per_poly;
        p = u;
        const uint64_t t = c.primes[p].q;
        const ModDownTable* md = fz.md;
        const uint64_t* pc = fz.pc + (size_t)pp * c.K * c.N;
        for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
            const int r = i / C, cc = i % C;
            const size_t pos = (size_t)r * B + col0 + cc;
            uint64_t y = 0;
            int neg = 0;
#pragma unroll
            for (int k = 0; k < kMaxAlpha; ++k) {
                if (k < c.K) {
                    const uint64_t q = c.primes[c.L + k].q;
                    const uint64_t v = mul_shoup(pc[(size_t)k * c.N + pos], md->pinv[k], md->pinv_sh[k], q);
                    neg += v > (q >> 1);
                    y = add_mod(y, mul_shoup(v, md->hat[p][k], md->hat_sh[p][k], t), t);
                }
            }
            for (int n = 0; n < neg; ++n) y = sub_mod(y, md->pmod[p], t);
            sm[cc * PN + pad(r)] = y;
        }
    } else {
        if (skip_row(rm, row, u)) return;
        p = row_prime(rm, u);
        // coalesced load: consecutive threads take consecutive columns of a row
        for (int i = threadIdx.x; i < N1 * C; i += blockDim.x) {
            const int r = i / C, cc = i % C;
            sm[cc * PN + pad(r)] = a[(size_t)r * B + col0 + cc];
        }
    }
    const uint64_t q = c.primes[p].q;
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

// Column pass with the FastBConv fused in front, amortised over target rows:
// CTA = (column tile, source group, target group). The centered
// [x_i (Q_J/q_i)^-1]_{q_i} values of the tile are computed once into
// registers, then every target row of the group is converted, transformed
// and written. MODE = FUSE_MODUP: source group = (src, digit j), targets =
// extended rows u (own rows of the digit copied from the NTT input);
// MODE = FUSE_MODDOWN: source group = poly, sources = the K special rows,
// targets = q rows t <= level.
template <int LOG_N1, int C, int MODE, int KA>
__global__ void __launch_bounds__(256) k_ntt_cols_bconv(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz,
                                                        int tg_size) {
    constexpr int N1 = 1 << LOG_N1;
    constexpr int TPC = N1 / EPT;
    constexpr int PN = N1 + (N1 >> 4) + 1;
    static_assert(N1 * C / 256 == EPT, "load phase: EPT elements per thread");
    __shared__ uint64_t sm[C * PN];
    const int B = c.N >> LOG_N1;
    const int col0 = blockIdx.x * C;
    const int sg = blockIdx.y;
    const int nr = rm.level + 1;
    int nsrc_rows, u_begin, u_end, lo = 0, hi = 0;
    const uint64_t* srcrows;
    const ModUpDigit* T = nullptr;
    if (MODE == FUSE_MODUP) {
        const int src = sg / fz.dn, j = sg % fz.dn;
        T = fz.mu + j;
        lo = T->lo;
        hi = T->hi;
        nsrc_rows = hi - lo;
        srcrows = fz.coef + ((size_t)src * nr + lo) * c.N;
        u_begin = blockIdx.z * tg_size;
        u_end = min(u_begin + tg_size, rm.rows_per_poly);
    } else {
        nsrc_rows = c.K;
        srcrows = fz.pc + (size_t)sg * c.K * c.N;
        u_begin = blockIdx.z * tg_size;
        u_end = min(u_begin + tg_size, nr);
    }
    // load + first half of the conversion (once per tile), kept in shared
    // memory (per-thread private slots) so the NTT passes keep a low register count
    extern __shared__ uint64_t dyn[];
    uint64_t(*sv)[EPT][256] = reinterpret_cast<uint64_t(*)[EPT][256]>(dyn);  // [KA][EPT][256]
    uint8_t(*sneg)[256] = reinterpret_cast<uint8_t(*)[256]>(dyn + KA * EPT * 256);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
        const int i = threadIdx.x + e * 256;
        const size_t pos = (size_t)(i / C) * B + col0 + i % C;
        int neg = 0;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            uint64_t v = 0;
            if (a < nsrc_rows) {
                const int qi = MODE == FUSE_MODUP ? lo + a : c.L + a;
                const uint64_t q = c.primes[qi].q;
                const uint64_t x = srcrows[(size_t)a * c.N + pos];
                const uint64_t w = MODE == FUSE_MODUP ? T->inv[a] : fz.md->pinv[a];
                const uint64_t ws = MODE == FUSE_MODUP ? T->inv_sh[a] : fz.md->pinv_sh[a];
                v = mul_shoup(x, w, ws, q);
                neg += v > (q >> 1);
            }
            sv[a][e][threadIdx.x] = v;
        }
        sneg[e][threadIdx.x] = (uint8_t)neg;
    }
    const int cc = threadIdx.x / TPC, lt = threadIdx.x % TPC;
    for (int u = u_begin; u < u_end; ++u) {
        const int outrow = sg * rm.rows_per_poly + u;
        uint64_t* a_out = data + (size_t)outrow * c.N;
        if (MODE == FUSE_MODUP && u >= lo && u < hi) {  // own prime: NTT-domain copy
            const int src = sg / fz.dn;
            const uint64_t* c1 = fz.c1 + (size_t)src * fz.c1_stride + (size_t)u * c.N;
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
                const int i = threadIdx.x + e * 256;
                const size_t pos = (size_t)(i / C) * B + col0 + i % C;
                a_out[pos] = c1[pos];
            }
            continue;
        }
        const int p = row_prime(rm, u);
        const uint64_t t = c.primes[p].q;
        uint64_t hat[KA], hats[KA];
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            hat[a] = MODE == FUSE_MODUP ? T->hat[u][a] : fz.md->hat[p][a];
            hats[a] = MODE == FUSE_MODUP ? T->hat_sh[u][a] : fz.md->hat_sh[p][a];
        }
        const uint64_t corr = MODE == FUSE_MODUP ? T->qj[u] : fz.md->pmod[p];
#pragma unroll 2
        for (int e = 0; e < EPT; ++e) {
            const int i = threadIdx.x + e * 256;
            uint64_t y = 0;
#pragma unroll
            for (int a = 0; a < KA; ++a)
                if (a < nsrc_rows) y = add_mod(y, mul_shoup(sv[a][e][threadIdx.x], hat[a], hats[a], t), t);
            const int neg = sneg[e][threadIdx.x];
            for (int n = 0; n < neg; ++n) y = sub_mod(y, corr, t);  // centered lift
            sm[(i % C) * PN + pad(i / C)] = y;
        }
        __syncthreads();
        fwd_local<LOG_N1, 0, false>(sm + cc * PN, lt, 0, 0, c.tw + (size_t)p * c.N, c.tw_sh + (size_t)p * c.N, t);
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int i = threadIdx.x + e * 256;
            a_out[(size_t)(i / C) * B + col0 + i % C] = sm[(i % C) * PN + pad(i / C)];
        }
        __syncthreads();
    }
}

__device__ __forceinline__ uint32_t perm_index_n(uint32_t k, uint32_t g, int logN) {
    const uint32_t e = 2 * (__brev(k) >> (32 - logN)) + 1;
    const uint32_t e2 = (e * g) & ((2u << logN) - 1);
    return __brev((e2 - 1) >> 1) >> (32 - logN);
}

// Phase B (contiguous blocks of B). CTA = BPC blocks; B/8 threads per block.
template <int LOG_N1, int LOG_B, bool INVERSE, int FUSE>
__global__ void __launch_bounds__(256) k_ntt_rows(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz) {
    constexpr int B = 1 << LOG_B;
    constexpr int TPB = B / EPT;
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
        if (FUSE == FUSE_MODDOWN) {
            const int pp = row / rm.rows_per_poly;
            const int nr = rm.level + 1, ne = nr + c.K;
            (void)ne;
            const uint64_t* acc = fz.acc + (size_t)pp * fz.acc_stride + (size_t)u * c.N + (size_t)blk0 * B;
            uint64_t* out = fz.out + ((size_t)pp * nr + u) * c.N + (size_t)blk0 * B;
            const uint64_t pi = fz.md->pinvq[u], pis = fz.md->pinvq_sh[u];
            const bool add = fz.add_src && pp == 0;
            for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) {
                uint64_t x = sm[(i / B) * PB + pad(i % B)];
                x = x >= q2 ? x - q2 : x;
                x = x >= q ? x - q : x;
                uint64_t o = mul_shoup(sub_mod(acc[i], x, q), pi, pis, q);
                if (add) {
                    const uint32_t k = (uint32_t)(blk0 * B + i);
                    o = add_mod(o, fz.add_src[(size_t)u * c.N + perm_index_n(k, fz.galois, c.logN)], q);
                }
                out[i] = o;
            }
        } else {
            for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) {
                uint64_t x = sm[(i / B) * PB + pad(i % B)];
                x = x >= q2 ? x - q2 : x;
                a[i] = x >= q ? x - q : x;
            }
        }
    } else {
        for (int i = threadIdx.x; i < BPC * B; i += blockDim.x) a[i] = sm[(i / B) * PB + pad(i % B)];
    }
}

template <int LOG_N1, int LOG_B>
void ntt_dispatch(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, bool inverse, int fuse,
                  const NttFuse& fz, cudaStream_t st) {
    constexpr int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    constexpr int C = 256 / (N1 / EPT);
    constexpr int BPC = 256 / (B / EPT);
    const dim3 ga(B / C, nrows), gb((N1 + BPC - 1) / BPC, nrows);
    if (!inverse) {
        if (fuse == FUSE_MODUP || fuse == FUSE_MODDOWN) {
            // target groups: enough CTAs to fill the GPU, few enough to amortise the conversion
            const int ngroups_src = nrows / rm.rows_per_poly;
            const int tiles = B / C;
            // ~4 target rows per CTA: enough CTAs to overlap, the conversion amortised 4x
            const int tg_size = rm.rows_per_poly < 4 ? rm.rows_per_poly : 4;
            const int tg = (rm.rows_per_poly + tg_size - 1) / tg_size;
            (void)tiles;
            const dim3 gc(tiles, ngroups_src, tg);
#define FHE_BCONV(MODE, KA)                                                                              \
    do {                                                                                                 \
        const int dsm = (KA) * EPT * 256 * 8 + EPT * 256;                                                \
        cudaFuncSetAttribute(k_ntt_cols_bconv<LOG_N1, C, MODE, KA>,                                      \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, dsm);                          \
        k_ntt_cols_bconv<LOG_N1, C, MODE, KA><<<gc, 256, dsm, st>>>(c, data, rm, fz, tg_size);           \
    } while (0)
#define FHE_BCONV_K(MODE)             \
    switch (c.K) {                    \
        case 1: FHE_BCONV(MODE, 1); break; \
        case 2: FHE_BCONV(MODE, 2); break; \
        case 3: FHE_BCONV(MODE, 3); break; \
        default: FHE_BCONV(MODE, 4); break; \
    }
            if (fuse == FUSE_MODUP) {
                FHE_BCONV_K(FUSE_MODUP)
                k_ntt_rows<LOG_N1, LOG_B, false, FUSE_NONE><<<gb, 256, 0, st>>>(c, data, rm, fz);
            } else {
                FHE_BCONV_K(FUSE_MODDOWN)
                k_ntt_rows<LOG_N1, LOG_B, false, FUSE_MODDOWN><<<gb, 256, 0, st>>>(c, data, rm, fz);
            }
#undef FHE_BCONV_K
#undef FHE_BCONV
        } else {
            k_ntt_cols<LOG_N1, C, false, FUSE_NONE><<<ga, 256, 0, st>>>(c, data, rm, fz);
            k_ntt_rows<LOG_N1, LOG_B, false, FUSE_NONE><<<gb, 256, 0, st>>>(c, data, rm, fz);
        }
    } else {
        k_ntt_rows<LOG_N1, LOG_B, true, FUSE_NONE><<<gb, 256, 0, st>>>(c, data, rm, fz);
        k_ntt_cols<LOG_N1, C, true, FUSE_NONE><<<ga, 256, 0, st>>>(c, data, rm, fz);
    }
    note_launch(2);
}

}  // namespace

static void ntt_run(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, bool inverse, int fuse,
                    const NttFuse& fz, cudaStream_t st) {
    if (nrows <= 0) return;
    switch (c.logN) {
        case 12: ntt_dispatch<6, 6>(c, data, nrows, rm, inverse, fuse, fz, st); break;
        case 13: ntt_dispatch<6, 7>(c, data, nrows, rm, inverse, fuse, fz, st); break;
        case 14: ntt_dispatch<7, 7>(c, data, nrows, rm, inverse, fuse, fz, st); break;
        case 15: ntt_dispatch<7, 8>(c, data, nrows, rm, inverse, fuse, fz, st); break;
        case 16: ntt_dispatch<8, 8>(c, data, nrows, rm, inverse, fuse, fz, st); break;
        default: break;
    }
}

void ntt_forward(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    ntt_run(c, data, nrows, rm, false, FUSE_NONE, NttFuse{}, st);
}

void ntt_inverse(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st) {
    ntt_run(c, data, nrows, rm, true, FUSE_NONE, NttFuse{}, st);
}

void ntt_modup(const DevCtx& c, uint64_t* digits, const uint64_t* coef, const uint64_t* c1, size_t c1_stride,
               int nsrc, const ModUpDigit* tables, int level, int dn, cudaStream_t st) {
    const int ne = level + 1 + c.K;
    NttFuse fz{};
    fz.coef = coef;
    fz.c1 = c1;
    fz.c1_stride = c1_stride;
    fz.mu = tables;
    fz.dn = dn;
    ntt_run(c, digits, nsrc * dn * ne, RowMap{ne, level, c.L, c.K, dn}, false, FUSE_MODUP, fz, st);
}

void ntt_moddown(const DevCtx& c, uint64_t* conv, const uint64_t* pcoef, const uint64_t* acc, size_t acc_stride,
                 uint64_t* out, const ModDownTable* md, int level, int npoly, const uint64_t* add_src,
                 uint32_t galois, cudaStream_t st) {
    const int nr = level + 1;
    NttFuse fz{};
    fz.pc = pcoef;
    fz.md = md;
    fz.acc = acc;
    fz.acc_stride = acc_stride;
    fz.out = out;
    fz.add_src = add_src;
    fz.galois = galois;
    ntt_run(c, conv, npoly * nr, RowMap{nr, level, c.L, 0, 0}, false, FUSE_MODDOWN, fz, st);
}

}  // namespace fhe
