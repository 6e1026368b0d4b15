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
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace fhe {

void note_launch(int n);

namespace {

// padded shared-memory index (2-way bank conflicts at worst for 8-byte words)
__device__ __forceinline__ int pad(int x) { return x + (x >> 4); }

__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t* v) {
    asm volatile("ld.global.cs.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
                 : "l"(p));
}
__device__ __forceinline__ void ld256_nc(const uint64_t* p, uint64_t* v) {
    asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
                 : "l"(p));
}
__device__ __forceinline__ void st256(uint64_t* p, const uint64_t* v) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]), "l"(v[3])
                 : "memory");
}

// Thread-block-cluster helpers of the single-launch transform (k_ntt_fused): the
// column -> row intermediate of a residue row stays in the shared memory of the
// cluster's CTAs and is read through distributed shared memory.
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint64_t ld_dsmem(uint32_t local_addr, uint32_t rank) {
    uint32_t ra;
    uint64_t v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
    return v;
}


// Twiddles of one sub-stage of a group are consecutive and aligned to their count
// (a power of two): load them with 128-bit (integer: w, Shoup) or 256-bit (FP64:
// (w_c, w_c / q) pairs) accesses, so a warp's requests use whole sectors.
template <bool SM = false>
__device__ __forceinline__ void tw_ld(const uint64_t* p, uint64_t* o, int cnt) {
    if (SM) {  // the CTA's twiddle table in shared memory (k_ntt_rows_tw)
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < cnt) o[i] = p[i];
        return;
    }
    if (cnt == 1) {
        o[0] = __ldg(p);
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2)
        if (i < cnt) {
            const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(p + i));
            o[i] = t.x;
            o[i + 1] = t.y;
        }
}
template <bool SM = false>
__device__ __forceinline__ void tw_ld(const double2* p, double2* o, int cnt) {
    if (SM) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < cnt) o[i] = p[i];
        return;
    }
    if (cnt == 1) {
        o[0] = __ldg(p);
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2)
        if (i < cnt) {
            uint64_t t[4];
            ld256_nc(reinterpret_cast<const uint64_t*>(p + i), t);
            o[i] = make_double2(asd(t[0]), asd(t[1]));
            o[i + 1] = make_double2(asd(t[2]), asd(t[3]));
        }
}

#ifndef FHE_NTT_EPT
#define FHE_NTT_EPT 16
#endif
#ifndef FHE_NTT_THREADS
#define FHE_NTT_THREADS 128
#endif
#ifndef FHE_NTT_MINB
#define FHE_NTT_MINB 1
#endif
#ifndef FHE_NTTF_MINB
#define FHE_NTTF_MINB 1  // CTAs per SM the single-launch kernel is compiled for
#endif
#ifndef FHE_NTTPF_MINB
#define FHE_NTTPF_MINB 4  // CTAs per SM the prefetching row phase is compiled for
#endif
#ifndef FHE_NTT_CHUNK
#define FHE_NTT_CHUNK 0  // MB of rows per NTT launch pair (0: all rows in one pair)
#endif
constexpr int EPT = FHE_NTT_EPT;         // residues per thread in a pass
constexpr int NTT_THREADS = FHE_NTT_THREADS;
constexpr int LOG_EPT = EPT == 16 ? 4 : 3;

// One radix-2^R pass of forward CT butterflies on EPT register values that
// form EPT / 2^R groups. Local vector of n = 2^logn elements, local stage of
// the pass sigma0, global stage offset s0, block index blk:
//   twiddle(stage sigma, x) = 2^(s0+sigma) + blk 2^sigma + x / (2 t_sigma)
template <int R, bool SM = false>
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
            uint64_t wt[GS / 2], wst[GS / 2];
            tw_ld<SM>(tw + base, wt, 1 << rho);
            tw_ld<SM>(tws + base, wst, 1 << rho);
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int off = k >> (R - rho);
                const uint64_t w = wt[off], ws = wst[off];
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
template <int R, bool SM = false>
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
            uint64_t wt[GS / 2], wst[GS / 2];
            tw_ld<SM>(tw + base, wt, GS >> (rho + 1));
            tw_ld<SM>(tws + base, wst, GS >> (rho + 1));
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const int off = k >> (rho + 1);
                const uint64_t w = wt[off], ws = wst[off];
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

// ------------------------------------------------------------ FP64 butterflies
// For primes q < 2^50 the butterflies run on the FP64 pipe (the integer
// multiply pipe is the NTT's bound, and the FP64 pipe is otherwise idle).
// Residues are exact integer-valued doubles, signed, |x| < 2^52 = 4q at the
// least; magnitudes are tracked in units of q/8 at compile time (the
// unrolled loops constant-fold them), and every operation is exact:
//  mulmod_d(x, w_c, w_c/q): t = rint(x w_c/q) (magic-constant rounding,
//    |x w_c/q| < 2^51), (ph, pl) = exact product x w_c split in two doubles,
//    r = (ph - t q) + pl: both steps are exact because the true values are
//    integers below 2^53. |r| <= 0.625 q for |x| < 2^52 and centred w_c.
//  red_d(x) = x - q rint(x / q): |result| <= 0.5 q + 1 (5 units).
// Sums U +- r are exact while they stay below 2^53. Values enter from
// canonical [0, q) words (8 units) and leave through canon_d (exact [0, q)).
// The FP64 helpers (ArD, mulmod_d, red_d, canon_d) are in modarith.cuh.
constexpr int kUnitQ = 8, kUnitMul = 5, kUnitRed = 5, kUnitMax = 32;  // in q / 8


// Forward CT pass of R <= 4 stages on doubles (inputs <= 8 units: <= 28 after).
template <int R, bool SM = false>
__device__ __forceinline__ void fwd_pass_d(double (&v)[EPT], int G0, int logn, int sigma0, int s0, int blk,
                                           const double2* __restrict__ tw, const ArD& a) {
    constexpr int GS = 1 << R;
    const int logt = logn - sigma0 - 1;
    const int logd = logt - (R - 1);
#pragma unroll
    for (int g = 0; g < EPT / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logd) << (logd + R)) | (G & ((1 << logd) - 1));
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << (R - 1 - rho);
            const int sig = sigma0 + rho;
            double2 wt[GS / 2];
            tw_ld<SM>(tw + (1 << (s0 + sig)) + (blk << sig) + (j0 >> (logt + 1 - rho)), wt, 1 << rho);
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const double2 w = wt[k >> (R - rho)];
                const double r = mulmod_d(v[g * GS + k + half], w.x, w.y, a);
                const double U = v[g * GS + k];
                v[g * GS + k] = __dadd_rn(U, r);
                v[g * GS + k + half] = __dadd_rn(U, -r);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) v[e] = red_d(v[e], a);  // <= 5 units for the next pass
}

// Inverse GS pass of R stages on doubles; sums are reduced only when the
// tracked bound of a butterfly's inputs would pass 4q. Leaves <= 8 units.
template <int R, bool SM = false>
__device__ __forceinline__ void inv_pass_d(double (&v)[EPT], int G0, int logt, int log_ntot, int log_nloc, int blk,
                                           const double2* __restrict__ tw, const ArD& a) {
    constexpr int GS = 1 << R;
#pragma unroll
    for (int g = 0; g < EPT / GS; ++g) {
        const int G = G0 + g;
        const int j0 = ((G >> logt) << (logt + R)) | (G & ((1 << logt) - 1));
        int bd[GS];
#pragma unroll
        for (int k = 0; k < GS; ++k) bd[k] = kUnitQ;
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = 1 << rho;
            const int lt = logt + rho;
            double2 wt[GS / 2];
            tw_ld<SM>(tw + (1 << (log_ntot - lt - 1)) + (blk << (log_nloc - lt - 1)) + (j0 >> (lt + 1)), wt,
                      GS >> (rho + 1));
#pragma unroll
            for (int k = 0; k < GS; ++k) {
                if (k & half) continue;
                const double2 w = wt[k >> (rho + 1)];
                double U = v[g * GS + k], V = v[g * GS + k + half];
                if (bd[k] + bd[k + half] > kUnitMax) {
                    U = red_d(U, a);
                    V = red_d(V, a);
                    bd[k] = bd[k + half] = kUnitRed;
                }
                v[g * GS + k] = __dadd_rn(U, V);
                bd[k] += bd[k + half];
                v[g * GS + k + half] = mulmod_d(__dadd_rn(U, -V), w.x, w.y, a);
                bd[k + half] = kUnitMul;
            }
        }
#pragma unroll
        for (int k = 0; k < GS; ++k)
            if (bd[k] > kUnitQ) v[g * GS + k] = red_d(v[g * GS + k], a);
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

// Fused-operand modes of the row pass:
//  FUSE_NONE    : transform `data` in place;
//  FUSE_MODDOWN : forward; the row pass writes out = (acc - NTT(conv)) P^-1
//                 (+ sigma_g(add_src) on poly 0, or the conv bias).
// ModUp's FastBConv is a separate kernel (k_bconv_modup) ahead of the forward
// transform of the extended rows.
enum { FUSE_NONE = 0, FUSE_MODDOWN = 2 };

// ------------------------------------------------------------ the two NTT kernels
// Both phases run two register passes per thread (EPT = 16 residues, radix-16 /
// radix-2^R2), with exactly one shared-memory exchange between them; residues
// are read from and written to global memory straight from the registers of
// the pass that owns them (coalesced: consecutive threads own consecutive
// columns, or the pass's stride-TPB residues of a block; a thread's 16
// contiguous residues of the row pass move with 256-bit accesses).
template <int LOGN, bool INVERSE>
struct PassPlan {  // stages of the two passes of a phase of 2^LOGN elements
    static constexpr int R1 = INVERSE ? (LOGN % LOG_EPT ? LOGN % LOG_EPT : LOG_EPT) : LOG_EPT;
    static constexpr int R2 = LOGN - R1;
    static_assert(R2 >= 1 && R2 <= LOG_EPT, "two passes per phase");
    __device__ static int pos1(int lt, int e) {
        return INVERSE ? inv_pos<R1>(lt * (EPT >> R1), e, 0) : fwd_pos<R1>(lt * (EPT >> R1), e, LOGN, 0);
    }
    __device__ static int pos2(int lt, int e) {
        return INVERSE ? inv_pos<R2>(lt * (EPT >> R2), e, R1) : fwd_pos<R2>(lt * (EPT >> R2), e, LOGN, R1);
    }
};

// Phase A (columns): CTA = C columns x N1 rows, thread (cc = tid % C, lt = tid / C).
// Forward: canonical words in, lazy [0, 4q) words / reduced doubles out (read by the
// row pass); inverse: the row pass's words in, canonical words out (times N^-1).
// XCH = 0: residues in and out of global memory (k_ntt_cols). XCH = 1 (k_ntt_fused, one
// cluster per residue row): the intermediate between the phases lives in the cluster's
// shared memory -- the forward transform leaves it in this CTA's `stage` ([N1][C] words:
// this CTA's C columns), the inverse reads it from the row phase's stages ([BPC][B] words
// per CTA: matrix row i is held by CTA i / BPC).
template <int LOG_N1, int LOG_B, int C, bool INVERSE, int XCH>
__device__ __forceinline__ void cols_phase(const DevCtx& c, uint64_t* data, const RowMap& rm, int row, int u, int bx,
                                           uint64_t* sm, uint64_t* stage) {
    constexpr int N1 = 1 << LOG_N1;
    constexpr int PN = N1 + (N1 >> 4) + 1;  // padded column length (odd in words)
    constexpr int B = 1 << LOG_B;
    constexpr int BPC = NTT_THREADS / (B / EPT);
    using PP = PassPlan<LOG_N1, INVERSE>;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const int cc = threadIdx.x % C, lt = threadIdx.x / C;
    uint64_t* a = data + (size_t)row * c.N + bx * C + cc;
    uint64_t* col = sm + cc * PN;
    uint64_t w[EPT];
    if (XCH && INVERSE) {
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stage) + (uint32_t)(bx * C + cc) * 8u;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int i = PP::pos1(lt, e);
            w[e] = ld_dsmem(sb + (uint32_t)((i % BPC) * B) * 8u, (uint32_t)(i / BPC));
        }
        cluster_arrive();  // this CTA's reads of the other stages are done (waited for at kernel end)
    } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = __ldcs(a + (size_t)PP::pos1(lt, e) * B);
    }
    // FP64 butterflies for q < 2^50
    if (q < (1ULL << 50)) {
        const ArD ad = make_ard(q);
        const double2* tw = (INVERSE ? c.itwd : c.twd) + (size_t)p * c.N;
        double v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = INVERSE ? asd(w[e]) : asd(u2d_bits(w[e]));
        if (!INVERSE)
            fwd_pass_d<PP::R1>(v, lt * (EPT >> PP::R1), LOG_N1, 0, 0, 0, tw, ad);
        else
            inv_pass_d<PP::R1>(v, lt * (EPT >> PP::R1), 0, LOG_N1, LOG_N1, 0, tw, ad);
#pragma unroll
        for (int e = 0; e < EPT; ++e) col[pad(PP::pos1(lt, e))] = asu(v[e]);
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = asd(col[pad(PP::pos2(lt, e))]);
        if (!INVERSE) {
            fwd_pass_d<PP::R2>(v, lt * (EPT >> PP::R2), LOG_N1, PP::R1, 0, 0, tw, ad);
            if (XCH) {
#pragma unroll
                for (int e = 0; e < EPT; ++e) stage[PP::pos2(lt, e) * C + cc] = asu(v[e]);
            } else {
#pragma unroll
                for (int e = 0; e < EPT; ++e) a[(size_t)PP::pos2(lt, e) * B] = asu(v[e]);
            }
        } else {
            inv_pass_d<PP::R2>(v, lt * (EPT >> PP::R2), PP::R1, LOG_N1, LOG_N1, 0, tw, ad);
            const double2 ni = c.ninvd[p];
#pragma unroll
            for (int e = 0; e < EPT; ++e) a[(size_t)PP::pos2(lt, e) * B] = canon_d(mulmod_d(v[e], ni.x, ni.y, ad), ad);
        }
        return;
    }
    const uint64_t* tw = (INVERSE ? c.itw : c.tw) + (size_t)p * c.N;
    const uint64_t* tws = (INVERSE ? c.itw_sh : c.tw_sh) + (size_t)p * c.N;
    if (!INVERSE)
        fwd_pass<PP::R1>(w, lt * (EPT >> PP::R1), LOG_N1, 0, 0, 0, tw, tws, q);
    else
        inv_pass<PP::R1>(w, lt * (EPT >> PP::R1), 0, LOG_N1, LOG_N1, 0, tw, tws, q);
#pragma unroll
    for (int e = 0; e < EPT; ++e) col[pad(PP::pos1(lt, e))] = w[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EPT; ++e) w[e] = col[pad(PP::pos2(lt, e))];
    if (!INVERSE) {
        fwd_pass<PP::R2>(w, lt * (EPT >> PP::R2), LOG_N1, PP::R1, 0, 0, tw, tws, q);
        if (XCH) {
#pragma unroll
            for (int e = 0; e < EPT; ++e) stage[PP::pos2(lt, e) * C + cc] = w[e];
        } else {
#pragma unroll
            for (int e = 0; e < EPT; ++e) a[(size_t)PP::pos2(lt, e) * B] = w[e];
        }
    } else {
        inv_pass<PP::R2>(w, lt * (EPT >> PP::R2), PP::R1, LOG_N1, LOG_N1, 0, tw, tws, q);
        const uint64_t ni = c.ninv[p], nis = c.ninv_sh[p];
#pragma unroll
        for (int e = 0; e < EPT; ++e) a[(size_t)PP::pos2(lt, e) * B] = mul_shoup(w[e], ni, nis, q);
    }
}

template <int LOG_N1, int LOG_B, int C, bool INVERSE>
__global__ void __launch_bounds__(NTT_THREADS, FHE_NTT_MINB) k_ntt_cols(DevCtx c, uint64_t* data, RowMap rm) {
    constexpr int N1 = 1 << LOG_N1;
    __shared__ uint64_t sm[C * (N1 + (N1 >> 4) + 1)];
    const int row = blockIdx.y + rm.row0;
    const int u = row % rm.rows_per_poly;
    if (skip_row(rm, row, u)) return;
    cols_phase<LOG_N1, LOG_B, C, INVERSE, 0>(c, data, rm, row, u, blockIdx.x, sm, nullptr);
}

__device__ __forceinline__ uint32_t perm_index_n(uint32_t k, uint32_t g, int logN) {
    const uint32_t e = 2 * (__brev(k) >> (32 - logN)) + 1;
    const uint32_t e2 = (e * g) & ((2u << logN) - 1);
    return __brev((e2 - 1) >> 1) >> (32 - logN);
}

// Phase B (contiguous blocks of B): CTA = BPC blocks, TPB = B / 16 threads per block
// (one or a fraction of a warp: the exchange needs only __syncwarp). The forward
// transform ends here (canonical words; FUSE_MODDOWN: the ModDown epilogue), the
// inverse starts here (canonical words in, words for the column pass out).
// XCH as in cols_phase: the forward transform reads its blocks from the column phase's
// stages (element x of matrix row blk is held by CTA x / C at [blk][x % C]), the inverse
// leaves its blocks in this CTA's `stage` ([BPC][B] words).
// TWS (k_ntt_rows_tw): the twiddles of the CTA's BPC blocks are read from the shared-memory
// table `twsm` (entry ((BPC + bi) << sigma) + x of stage sigma: the global table's index
// with N1 + blk replaced by BPC + bi), filled once per CTA and reused for several rows.
// PRE (k_ntt_rows_pf, forward): the thread's 16 input residues were loaded by the caller (`pre`).
template <int LOG_N1, int LOG_B, bool INVERSE, int FUSE, int XCH, bool TWS = false, bool PRE = false>
__device__ __forceinline__ void rows_phase(const DevCtx& c, uint64_t* data, const RowMap& rm, const NttFuse& fz, int row,
                                           int u, int bx, uint64_t* sm, uint64_t* stage,
                                           const uint64_t* twsm = nullptr, const uint64_t* pre = nullptr) {
    constexpr int N1 = 1 << LOG_N1;
    constexpr int C = NTT_THREADS / (N1 / EPT);
    constexpr int B = 1 << LOG_B;
    constexpr int TPB = B / EPT;
    constexpr int BPC = NTT_THREADS / TPB;
    constexpr int PB = B + (B >> 4);
    constexpr int LOG_BPC = LOG_EPT + (NTT_THREADS == 128 ? 7 : 8) - LOG_B;  // BPC = NTT_THREADS EPT / B
    static_assert((1 << LOG_BPC) == BPC, "blocks per CTA");
    static_assert(TPB <= 32, "a block is at most one warp");
    const int tS0 = TWS ? LOG_BPC : LOG_N1;  // twiddle index base: 2^(tS0 + sigma) + (tBlk << sigma)
    using PP = PassPlan<LOG_B, INVERSE>;
    const int p = row_prime(rm, u);
    const uint64_t q = c.primes[p].q;
    const int bi = threadIdx.x / TPB, lt = threadIdx.x % TPB;
    const int blk = bx * BPC + bi;
    const int tBlk = TWS ? bi : blk;
    const size_t base = (size_t)blk * B;  // block offset in the row
    uint64_t* a = data + (size_t)row * c.N + base;
    uint64_t* vec = sm + bi * PB;
    const bool fp = q < (1ULL << 50);
    const ArD ad = make_ard(q);
    uint64_t w[EPT];
    // input: forward stride-TPB residues (pass 1 positions lt + k TPB), inverse 16
    // contiguous residues lt 16 + e
    if (PRE) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = pre[e];
    } else if (XCH && !INVERSE) {
        const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stage) + (uint32_t)(blk * C) * 8u;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            const int x = PP::pos1(lt, e);
            w[e] = ld_dsmem(sb + (uint32_t)(x % C) * 8u, (uint32_t)(x / C));
        }
        cluster_arrive();  // this CTA's reads of the other stages are done (waited for at kernel end)
    } else if (!INVERSE) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = __ldcs(a + PP::pos1(lt, e));
    } else {
#pragma unroll
        for (int e = 0; e < EPT; e += 4) ld256(a + lt * EPT + e, w + e);
    }
    if (fp) {
        const double2* tw = TWS ? reinterpret_cast<const double2*>(twsm) - BPC
                                : (INVERSE ? c.itwd : c.twd) + (size_t)p * c.N;
        double v[EPT];
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = INVERSE ? asd(u2d_bits(w[e])) : asd(w[e]);
        if (!INVERSE)
            fwd_pass_d<PP::R1, TWS>(v, lt * (EPT >> PP::R1), LOG_B, 0, tS0, tBlk, tw, ad);
        else
            inv_pass_d<PP::R1, TWS>(v, lt * (EPT >> PP::R1), 0, tS0 + LOG_B, LOG_B, tBlk, tw, ad);
#pragma unroll
        for (int e = 0; e < EPT; ++e) vec[pad(PP::pos1(lt, e))] = asu(v[e]);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = asd(vec[pad(PP::pos2(lt, e))]);
        if (!INVERSE) {
            fwd_pass_d<PP::R2, TWS>(v, lt * (EPT >> PP::R2), LOG_B, PP::R1, tS0, tBlk, tw, ad);
#pragma unroll
            for (int e = 0; e < EPT; ++e) w[e] = canon_d(v[e], ad);
        } else {
            inv_pass_d<PP::R2, TWS>(v, lt * (EPT >> PP::R2), PP::R1, tS0 + LOG_B, LOG_B, tBlk, tw, ad);
#pragma unroll
            for (int e = 0; e < EPT; ++e) w[e] = asu(v[e]);
        }
    } else {
        // shared-memory table of an integer row: [BPC (B - 1)] twiddles, then their Shoup companions
        const uint64_t* tw = TWS ? twsm - BPC : (INVERSE ? c.itw : c.tw) + (size_t)p * c.N;
        const uint64_t* tws = TWS ? twsm + BPC * (B - 1) - BPC : (INVERSE ? c.itw_sh : c.tw_sh) + (size_t)p * c.N;
        if (!INVERSE)
            fwd_pass<PP::R1, TWS>(w, lt * (EPT >> PP::R1), LOG_B, 0, tS0, tBlk, tw, tws, q);
        else
            inv_pass<PP::R1, TWS>(w, lt * (EPT >> PP::R1), 0, tS0 + LOG_B, LOG_B, tBlk, tw, tws, q);
#pragma unroll
        for (int e = 0; e < EPT; ++e) vec[pad(PP::pos1(lt, e))] = w[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = vec[pad(PP::pos2(lt, e))];
        if (!INVERSE) {
            fwd_pass<PP::R2, TWS>(w, lt * (EPT >> PP::R2), LOG_B, PP::R1, tS0, tBlk, tw, tws, q);
            const uint64_t q2 = 2 * q;
#pragma unroll
            for (int e = 0; e < EPT; ++e) {  // [0, 4q) -> [0, q)
                const uint64_t x = w[e] >= q2 ? w[e] - q2 : w[e];
                w[e] = x >= q ? x - q : x;
            }
        } else {
            inv_pass<PP::R2, TWS>(w, lt * (EPT >> PP::R2), PP::R1, tS0 + LOG_B, LOG_B, tBlk, tw, tws, q);
        }
    }
    if (INVERSE) {  // pass-2 positions lt + k TPB: coalesced
        if (XCH) {
#pragma unroll
            for (int e = 0; e < EPT; ++e) stage[bi * B + PP::pos2(lt, e)] = w[e];
        } else {
#pragma unroll
            for (int e = 0; e < EPT; ++e) a[PP::pos2(lt, e)] = w[e];
        }
        return;
    }
    // forward output: residue e of this thread sits at block position lt 16 + e
    if (FUSE == FUSE_MODDOWN) {
        const int pp = row / rm.rows_per_poly;
        const int nr = rm.level + 1;
        const uint64_t* acc = fz.acc + (size_t)pp * fz.acc_stride + (size_t)u * c.N + base + lt * EPT;
        uint64_t* out = (fz.outp ? fz.outp[pp >> 1] + ((size_t)(pp & 1) * nr + u) * c.N
                                 : fz.out + ((size_t)pp * nr + u) * c.N) +
                        base + lt * EPT;
        const uint64_t pi = fz.outmul ? fz.outmul[u] : fz.md->pinvq[u];
        const uint64_t pis = fz.outmul ? fz.outmul_sh[u] : fz.md->pinvq_sh[u];
        const bool add = fz.add_src && (fz.add_mod > 0 ? (pp & 1) == 0 : pp == 0);
        uint64_t av[EPT], sv[EPT];
#pragma unroll
        for (int e = 0; e < EPT; e += 4) ld256(acc + e, av + e);
        if (add && fz.add_mod > 0) {  // conv bias of output pp / 2 (unpermuted rows)
            const uint64_t* bsrc =
                fz.add_src + (size_t)((pp >> 1) % fz.add_mod) * fz.add_stride + (size_t)u * c.N + base + lt * EPT;
#pragma unroll
            for (int e = 0; e < EPT; e += 4) ld256_nc(bsrc + e, sv + e);
        } else if (add) {  // sigma_g(add_src)
#pragma unroll
            for (int e = 0; e < EPT; ++e)
                sv[e] = __ldg(fz.add_src + (size_t)u * c.N +
                              perm_index_n((uint32_t)(base + lt * EPT + e), fz.galois, c.logN));
        }
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
            uint64_t o = mul_shoup(sub_mod(av[e], w[e], q), pi, pis, q);
            if (add) o = add_mod(o, sv[e], q);
            w[e] = o;
        }
#pragma unroll
        for (int e = 0; e < EPT; e += 4) st256(out + e, w + e);
    } else {
        if (rm.limb) {
#pragma unroll
            for (int e = 0; e < EPT; ++e) w[e] = to_opf(w[e], q);
        }
#pragma unroll
        for (int e = 0; e < EPT; e += 4) st256(a + lt * EPT + e, w + e);
    }
}

template <int LOG_N1, int LOG_B, bool INVERSE, int FUSE>
__global__ void __launch_bounds__(NTT_THREADS, FHE_NTT_MINB) k_ntt_rows(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz) {
    constexpr int B = 1 << LOG_B;
    __shared__ uint64_t sm[(NTT_THREADS / (B / EPT)) * (B + (B >> 4))];
    const int row = blockIdx.y + rm.row0;
    const int u = row % rm.rows_per_poly;
    if (skip_row(rm, row, u)) return;
    rows_phase<LOG_N1, LOG_B, INVERSE, FUSE, 0>(c, data, rm, fz, row, u, blockIdx.x, sm, nullptr);
}

// Row phase with the twiddles in shared memory: a CTA's BPC blocks use BPC (B - 1) twiddles
// (16 bytes each: (w_c, w_c / q) or (w, Shoup w)), twice the bytes of the residues they
// transform -- read per row from L2, they are most of the row phase's traffic and of its
// long-scoreboard stalls. Here a CTA fills the table once and transforms the same blocks of
// R rows of the same prime (row = pp rows_per_poly + u, pp = g R .. g R + R - 1).
template <int LOG_N1, int LOG_B, bool INVERSE, int FUSE>
__global__ void __launch_bounds__(NTT_THREADS, 4) k_ntt_rows_tw(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz,
                                                                         int npoly, int R) {
    constexpr int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    constexpr int BPC = NTT_THREADS / (B / EPT);
    constexpr int LOG_BPC = LOG_EPT + (NTT_THREADS == 128 ? 7 : 8) - LOG_B;
    constexpr int XB = BPC * (B + (B >> 4));
    constexpr int NTW = BPC * (B - 1);
    extern __shared__ __align__(16) uint64_t dsm[];
    uint64_t* sm = dsm;                       // pass exchange
    uint64_t* twsm = dsm + ((XB + 1) & ~1);   // table: NTW double2, or NTW words + NTW Shoup words
    const int u = blockIdx.y % rm.rows_per_poly, g = blockIdx.y / rm.rows_per_poly;
    const int p = row_prime(rm, u);
    const bool fp = c.primes[p].q < (1ULL << 50);
    const int x0 = N1 + blockIdx.x * BPC;
    for (int idx = threadIdx.x; idx < NTW; idx += NTT_THREADS) {
        const int j = idx + BPC;  // table index ((BPC + bi) << sigma) + x
        const int sig = 31 - __clz(j) - LOG_BPC;
        const size_t src = (size_t)p * c.N + (size_t)(x0 << sig) + (size_t)(j - (BPC << sig));
        if (fp) {
            reinterpret_cast<double2*>(twsm)[idx] = __ldg((INVERSE ? c.itwd : c.twd) + src);
        } else {
            twsm[idx] = __ldg((INVERSE ? c.itw : c.tw) + src);
            twsm[NTW + idx] = __ldg((INVERSE ? c.itw_sh : c.tw_sh) + src);
        }
    }
    __syncthreads();
    for (int rr = 0; rr < R; ++rr) {
        const int pp = g * R + rr;
        if (pp >= npoly) break;
        const int row = pp * rm.rows_per_poly + u;
        if (!skip_row(rm, row, u))
            rows_phase<LOG_N1, LOG_B, INVERSE, FUSE, 0, true>(c, data, rm, fz, row, u, blockIdx.x, sm, nullptr, twsm);
        __syncwarp();  // the next row reuses the exchange buffer
    }
}

// Forward row phase with a software prefetch: a CTA transforms the same blocks of R rows of one
// prime and loads the 16 residues of the next row into registers before it transforms the current
// one, so the global-load latency (the row phase's first stall) overlaps the butterflies; the
// rows' common twiddles stay in L1. Opt-in (FHE_NTT_PF=R).
template <int LOG_N1, int LOG_B, int FUSE>
__global__ void __launch_bounds__(NTT_THREADS, FHE_NTTPF_MINB) k_ntt_rows_pf(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz, int npoly,
                                                                int R) {
    constexpr int B = 1 << LOG_B;
    constexpr int TPB = B / EPT;
    constexpr int BPC = NTT_THREADS / TPB;
    using PP = PassPlan<LOG_B, false>;
    __shared__ uint64_t sm[BPC * (B + (B >> 4))];
    const int u = blockIdx.y % rm.rows_per_poly, g = blockIdx.y / rm.rows_per_poly;
    const int bi = threadIdx.x / TPB, lt = threadIdx.x % TPB;
    const size_t off = (size_t)(blockIdx.x * BPC + bi) * B;
    const int pend = min(npoly, (g + 1) * R);
    auto next_row = [&](int pp) {  // first row >= pp of the group that is not skipped, or -1
        for (; pp < pend; ++pp) {
            const int row = pp * rm.rows_per_poly + u;
            if (!skip_row(rm, row, u)) return row;
        }
        return -1;
    };
    auto load = [&](int row, uint64_t (&w)[EPT]) {
        const uint64_t* a = data + (size_t)row * c.N + off;
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = __ldcs(a + PP::pos1(lt, e));
    };
    int row = next_row(g * R);
    if (row < 0) return;
    uint64_t w[EPT], wn[EPT];
    load(row, w);
    while (row >= 0) {
        const int nxt = next_row(row / rm.rows_per_poly + 1);
        if (nxt >= 0) load(nxt, wn);
        rows_phase<LOG_N1, LOG_B, false, FUSE, 0, false, true>(c, data, rm, fz, row, u, blockIdx.x, sm, nullptr, nullptr, w);
        __syncwarp();  // the next row reuses the exchange buffer
#pragma unroll
        for (int e = 0; e < EPT; ++e) w[e] = wn[e];
        row = nxt;
    }
}

// The whole transform of a residue row in ONE launch: a thread-block cluster of
// B / C = N / (16 NTT_THREADS) CTAs per row (16 at N = 2^15) runs the column phase and the
// row phase back to back; the intermediate (2048 words per CTA) never leaves shared memory,
// every CTA reads the blocks of its second phase from the stages of the whole cluster
// (ld.shared::cluster). One HBM round trip per transform instead of two.
template <int LOG_N1, int LOG_B, bool INVERSE, int FUSE>
__global__ void __launch_bounds__(NTT_THREADS, FHE_NTTF_MINB) k_ntt_fused(DevCtx c, uint64_t* data, RowMap rm, NttFuse fz) {
    constexpr int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    constexpr int C = NTT_THREADS / (N1 / EPT);
    constexpr int XA = C * (N1 + (N1 >> 4) + 1), XB = (NTT_THREADS / (B / EPT)) * (B + (B >> 4));
    __shared__ uint64_t sm[XA > XB ? XA : XB];
    __shared__ __align__(16) uint64_t stage[NTT_THREADS * EPT];
    const int row = blockIdx.y + rm.row0;
    const int u = row % rm.rows_per_poly;
    if (skip_row(rm, row, u)) return;  // the whole cluster (one row) returns
    if (!INVERSE)
        cols_phase<LOG_N1, LOG_B, C, false, 1>(c, data, rm, row, u, blockIdx.x, sm, stage);
    else
        rows_phase<LOG_N1, LOG_B, true, FUSE_NONE, 1>(c, data, rm, fz, row, u, blockIdx.x, sm, stage);
    cluster_arrive();
    cluster_wait();  // every stage of the row is written
    if (!INVERSE)
        rows_phase<LOG_N1, LOG_B, false, FUSE, 1>(c, data, rm, fz, row, u, blockIdx.x, sm, stage);
    else
        cols_phase<LOG_N1, LOG_B, C, true, 1>(c, data, rm, row, u, blockIdx.x, sm, stage);
    cluster_wait();  // no CTA leaves while its stage may still be read
}

// FastBConv of ModUp: one thread per (source, digit, coefficient pair); the
// centered [x_i (Q_J/q_i)^-1]_{q_i} values are computed once and extended to
// every target row of the digit (16-byte loads/stores); the digit's own rows
// are NTT-domain copies of c1 (or the coefficients, for coefficient-domain
// sources). The per-target constants of all digits are staged in shared memory.
template <int KA>
__global__ void __launch_bounds__(256) k_bconv_modup(DevCtx c, uint64_t* digits, NttFuse fz, int level, int nsrc) {
    const int nr = level + 1, ne = nr + c.K;
    const int halfN = c.N / 2;
    const int total = nsrc * fz.dn * halfN;
    // smem: per digit j, per target u: t, hat[KA], hat_sh[KA], n * Q_J mod t for n = 0..KA,
    // then (FP64 path) the centred hat[KA] as doubles, t, 1 / t and 2^52 + t as doubles
    constexpr int WD = 1 + 2 * KA + (KA + 1);
    constexpr int W = WD + KA + 3;
    __shared__ uint64_t tab[8 * 24 * W];
    __shared__ int lohi[8][2];
    for (int x = threadIdx.x; x < fz.dn * ne; x += blockDim.x) {
        const int j = x / ne, u = x - j * ne;
        const ModUpDigit& T = fz.mu[j];
        uint64_t* e = tab + (size_t)x * W;
        const uint64_t t = c.primes[u <= level ? u : c.L + (u - level - 1)].q;
        e[0] = t;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            e[1 + a] = T.hat[u][a];
            e[1 + KA + a] = T.hat_sh[u][a];
        }
        uint64_t m = 0;
        for (int n = 0; n <= KA; ++n) {
            e[1 + 2 * KA + n] = m;
            m = add_mod(m, T.qj[u], t);
        }
        const ArD ad = make_ard(t);
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            const uint64_t h = T.hat[u][a];
            e[WD + a] = asu(h > t / 2 ? -(double)(t - h) : (double)h);
        }
        e[WD + KA] = asu(ad.q);
        e[WD + KA + 1] = asu(ad.qinv);
        e[WD + KA + 2] = asu(ad.qm);
        if (u == 0) {
            lohi[j][0] = T.lo;
            lohi[j][1] = T.hi;
        }
    }
    __syncthreads();
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int sj = idx >> (c.logN - 1);
        const size_t k = (size_t)(idx & (halfN - 1)) * 2;
        const int src = sj / fz.dn, j = sj - src * fz.dn;
        const ModUpDigit& T = fz.mu[j];
        const int lo = lohi[j][0], hi = lohi[j][1];
        const int na = hi - lo;
        const uint64_t* coef = fz.coef + (size_t)src * nr * c.N;
        const uint64_t* c1 = fz.c1 ? fz.c1 + (size_t)src * fz.c1_stride : nullptr;
        uint64_t* out = digits + (size_t)sj * ne * c.N + k;
        uint64_t v0[KA], v1[KA];
        int n0 = 0, n1 = 0;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            v0[a] = v1[a] = 0;
            if (a < na) {
                const int qi = lo + a;
                const uint64_t q = tab[((size_t)j * ne + qi) * W];  // own prime q_qi
                const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(coef + (size_t)qi * c.N + k));
                v0[a] = mul_shoup(x.x, T.inv[a], T.inv_sh[a], q);
                v1[a] = mul_shoup(x.y, T.inv[a], T.inv_sh[a], q);
                n0 += v0[a] > (q >> 1);
                n1 += v1[a] > (q >> 1);
                // own row of the digit: NTT-domain copy of c1, or (coefficient-domain
                // sources, c1 == nullptr) the coefficients themselves, transformed later
                ulonglong2 own = c1 ? __ldcs(reinterpret_cast<const ulonglong2*>(c1 + (size_t)qi * c.N + k)) : x;
                if (fz.limb && c1) {
                    own = make_ulonglong2(to_opf(own.x, q), to_opf(own.y, q));
                }
                *reinterpret_cast<ulonglong2*>(out + (size_t)qi * c.N) = own;
            }
        }
        const uint64_t* tj = tab + (size_t)j * ne * W;
        // digits whose own primes are all < 2^50: v_a < 2^50 are exact doubles, and the
        // targets t < 2^50 take the FP64 pipe (fmac_d), the others the integer path
        bool vfp = true;
#pragma unroll
        for (int a = 0; a < KA; ++a)
            if (a < na) vfp = vfp && tab[((size_t)j * ne + lo + a) * W] < (1ULL << 50);
        double vd0[KA], vd1[KA];
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            vd0[a] = asd(u2d_bits(v0[a]));
            vd1[a] = asd(u2d_bits(v1[a]));
        }
        // targets outside [lo, hi): two branch-free runs
#pragma unroll 1
        for (int run = 0; run < 2; ++run) {
            const int ub = run == 0 ? 0 : hi, ue = run == 0 ? lo : ne;
#pragma unroll 4
            for (int u = ub; u < ue; ++u) {
                const uint64_t* e = tj + (size_t)u * W;
                const uint64_t t = e[0];
                if (vfp && t < (1ULL << 50)) {
                    const ArD ad{asd(e[WD + KA]), asd(e[WD + KA + 1]), asd(e[WD + KA + 2]), t};
                    double z0 = 0.0, z1 = 0.0;
#pragma unroll
                    for (int a = 0; a < KA; ++a) {
                        const double h = asd(e[WD + a]);
                        fmac_d(z0, vd0[a], h, ad);
                        fmac_d(z1, vd1[a], h, ad);
                    }
                    const uint64_t y0 = sub_mod(canon_d(red_d(z0, ad), ad), e[1 + 2 * KA + n0], t);
                    const uint64_t y1 = sub_mod(canon_d(red_d(z1, ad), ad), e[1 + 2 * KA + n1], t);
                    *reinterpret_cast<ulonglong2*>(out + (size_t)u * c.N) = make_ulonglong2(y0, y1);
                    continue;
                }
                // lazy sum of na < KA + 1 products, each in [0, 2t)
                uint64_t y0 = 0, y1 = 0;
#pragma unroll
                for (int a = 0; a < KA; ++a) {
                    y0 += mul_shoup_lazy(v0[a], e[1 + a], e[1 + KA + a], t);
                    y1 += mul_shoup_lazy(v1[a], e[1 + a], e[1 + KA + a], t);
                }
#pragma unroll
                for (int r = (KA >= 3 ? 4 : (KA >= 2 ? 2 : 1)); r >= 1; r >>= 1) {
                    y0 = y0 >= r * t ? y0 - r * t : y0;
                    y1 = y1 >= r * t ? y1 - r * t : y1;
                }
                // centered lift: each of the n0 (n1) negative terms stands for -Q_J
                y0 = sub_mod(y0, e[1 + 2 * KA + n0], t);
                y1 = sub_mod(y1, e[1 + 2 * KA + n1], t);
                *reinterpret_cast<ulonglong2*>(out + (size_t)u * c.N) = make_ulonglong2(y0, y1);
            }
        }
    }
}

// FastBConv of ModDown: conv[pp][t] = conv_P->q_t(pc[pp]) (coefficient domain).
// One thread per (poly, coefficient pair): the centred v_a = [x_a (P/p_a)^-1]_{p_a}
// are computed once and extended to every target row t.
template <int KA>
__global__ void __launch_bounds__(256) k_bconv_moddown(DevCtx c, uint64_t* conv, NttFuse fz, int level, int npoly) {
    const int nr = level + 1;
    const size_t halfN = c.N / 2;
    const size_t total = (size_t)npoly * halfN;
    const ModDownTable* md = fz.md;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int pp = (int)(idx >> (c.logN - 1));
        const size_t k = (idx & (halfN - 1)) * 2;
        const uint64_t* pc = fz.pc + (size_t)pp * c.K * c.N;
        uint64_t v0[KA], v1[KA];
        int n0 = 0, n1 = 0;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            const uint64_t q = c.primes[c.L + a].q;
            const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(pc + (size_t)a * c.N + k));
            v0[a] = mul_shoup(x.x, md->pinv[a], md->pinv_sh[a], q);
            v1[a] = mul_shoup(x.y, md->pinv[a], md->pinv_sh[a], q);
            n0 += v0[a] > (q >> 1);
            n1 += v1[a] > (q >> 1);
        }
        uint64_t* out = conv + (size_t)pp * nr * c.N + k;
#pragma unroll 4
        for (int t = 0; t < nr; ++t) {
            const uint64_t qt = c.primes[t].q;
            // lazy sum of KA products in [0, 2 qt), then the centred correction
            uint64_t y0 = 0, y1 = 0;
#pragma unroll
            for (int a = 0; a < KA; ++a) {
                y0 += mul_shoup_lazy(v0[a], md->hat[t][a], md->hat_sh[t][a], qt);
                y1 += mul_shoup_lazy(v1[a], md->hat[t][a], md->hat_sh[t][a], qt);
            }
#pragma unroll
            for (int r = (KA >= 3 ? 4 : (KA >= 2 ? 2 : 1)); r >= 1; r >>= 1) {
                y0 = y0 >= r * qt ? y0 - r * qt : y0;
                y1 = y1 >= r * qt ? y1 - r * qt : y1;
            }
            // centred correction n [P]_{q_t}, n <= KA: predicated subtractions instead of a product
            const uint64_t pm = md->pmod[t];
#pragma unroll
            for (int r = 1; r <= KA; ++r) {
                y0 = n0 >= r ? sub_mod(y0, pm, qt) : y0;
                y1 = n1 >= r ? sub_mod(y1, pm, qt) : y1;
            }
            *reinterpret_cast<ulonglong2*>(out + (size_t)t * c.N) = make_ulonglong2(y0, y1);
        }
    }
}

// Fused ModDown + rescale, coefficient domain: for each polynomial and pair
// position, v_a = x_a [(P/p_a)^-1]_{p_a} (centred count n), conv_t =
// sum_a v_a [P/p_a]_{q_t} - n [P]_{q_t} (as k_bconv_moddown), then the
// rescale's input c_l = (x_{q_l} - conv_l) P^-1 mod q_l and
//   w_i = conv_i + P * centred(c_l) mod q_i      (i < l).
template <int KA>
__global__ void __launch_bounds__(256) k_bconv_mdr(DevCtx c, uint64_t* w, const uint64_t* pcoef, const uint64_t* qlc,
                                                   const ModDownTable* md, int level, int npoly) {
    const size_t halfN = c.N / 2;
    const size_t total = (size_t)npoly * halfN;
    const uint64_t ql = c.primes[level].q;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const int pp = (int)(idx >> (c.logN - 1));
        const size_t k = (idx & (halfN - 1)) * 2;
        const uint64_t* pc = pcoef + (size_t)pp * c.K * c.N;
        uint64_t v0[KA], v1[KA];
        int n0 = 0, n1 = 0;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            const uint64_t q = c.primes[c.L + a].q;
            const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(pc + (size_t)a * c.N + k);
            v0[a] = mul_shoup(x.x, md->pinv[a], md->pinv_sh[a], q);
            v1[a] = mul_shoup(x.y, md->pinv[a], md->pinv_sh[a], q);
            n0 += v0[a] > (q >> 1);
            n1 += v1[a] > (q >> 1);
        }
        auto conv = [&](int t, uint64_t& y0, uint64_t& y1) {
            const uint64_t qt = c.primes[t].q;
            y0 = 0;
            y1 = 0;
#pragma unroll
            for (int a = 0; a < KA; ++a) {
                y0 = add_mod(y0, mul_shoup(v0[a], md->hat[t][a], md->hat_sh[t][a], qt), qt);
                y1 = add_mod(y1, mul_shoup(v1[a], md->hat[t][a], md->hat_sh[t][a], qt), qt);
            }
            for (int n = 0; n < n0; ++n) y0 = sub_mod(y0, md->pmod[t], qt);
            for (int n = 0; n < n1; ++n) y1 = sub_mod(y1, md->pmod[t], qt);
        };
        uint64_t cl0, cl1;
        {
            uint64_t y0, y1;
            conv(level, y0, y1);
            const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(qlc + (size_t)pp * c.N + k);
            cl0 = mul_shoup(sub_mod(x.x, y0, ql), md->pinvq[level], md->pinvq_sh[level], ql);
            cl1 = mul_shoup(sub_mod(x.y, y1, ql), md->pinvq[level], md->pinvq_sh[level], ql);
        }
        const bool neg0 = cl0 > (ql >> 1), neg1 = cl1 > (ql >> 1);
        for (int t = 0; t < level; ++t) {
            const Prime pr = c.primes[t];
            // centred lift of c_l into q_t (the rescale's spread)
            uint64_t s0, s1;
            if (neg0) {
                const uint64_t m = reduce64(ql - cl0, pr);
                s0 = m ? pr.q - m : 0;
            } else {
                s0 = reduce64(cl0, pr);
            }
            if (neg1) {
                const uint64_t m = reduce64(ql - cl1, pr);
                s1 = m ? pr.q - m : 0;
            } else {
                s1 = reduce64(cl1, pr);
            }
            uint64_t y0, y1;
            conv(t, y0, y1);
            y0 = add_mod(y0, mul_shoup(s0, md->pmod[t], md->pmod_sh[t], pr.q), pr.q);
            y1 = add_mod(y1, mul_shoup(s1, md->pmod[t], md->pmod_sh[t], pr.q), pr.q);
            *reinterpret_cast<ulonglong2*>(w + ((size_t)pp * level + t) * c.N + k) = make_ulonglong2(y0, y1);
        }
    }
}

template <typename K>
void launch_cluster(K kern, dim3 grid, int cl, cudaStream_t st, const DevCtx& c, uint64_t* data, const RowMap& rm,
                    const NttFuse& fz) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(NTT_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cl;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, c, data, rm, fz);
}

// FHE_NTT_FUSED=1 selects the single-launch cluster transform (N <= 2^15; the 32 CTAs
// per row of N = 2^16 exceed the largest cluster). Off by default: on the B200 the
// two-launch transform is faster (cfg3 batch-16 conv 2095 vs 1892-2027 conv/s, hoisted
// 36.5k vs 30.1-32.6k rot/s over 3-5 CTAs/SM; profiles/ab_r02_ntt_cluster.txt) -- the
// clusters of 16 schedule per GPC and the exchange runs at the DSMEM rate.
static bool ntt_fused_enabled() {  // read per launch: tests switch it between contexts
    const char* e = getenv("FHE_NTT_FUSED");
    return e && e[0] == '1';
}

static int ntt_tw_rows() {  // read per launch: tests switch it between contexts
    const char* e = getenv("FHE_NTT_TWR");
    const int v = e ? atoi(e) : 0;
    return v < 0 ? 0 : v > 64 ? 64 : v;
}

static int ntt_pf_rows() {  // read per launch: tests switch it between contexts
    const char* e = getenv("FHE_NTT_PF");
    const int v = e ? atoi(e) : 0;
    return v < 0 ? 0 : v > 64 ? 64 : v;
}

template <int LOG_N1, int LOG_B>
void ntt_dispatch(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, bool inverse, int fuse,
                  const NttFuse& fz, cudaStream_t st) {
    constexpr int N1 = 1 << LOG_N1, B = 1 << LOG_B;
    constexpr int C = NTT_THREADS / (N1 / EPT);
    constexpr int BPC = NTT_THREADS / (B / EPT);
    constexpr int CL = B / C;  // CTAs per row of either phase
    if (CL <= 16 && CL == N1 / BPC && FHE_NTT_CHUNK == 0 && ntt_fused_enabled()) {
        static const bool once = [] {  // clusters of 16 are a non-portable size
            if (CL > 8) {
                cudaFuncSetAttribute(k_ntt_fused<LOG_N1, LOG_B, false, FUSE_NONE>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaFuncSetAttribute(k_ntt_fused<LOG_N1, LOG_B, false, FUSE_MODDOWN>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaFuncSetAttribute(k_ntt_fused<LOG_N1, LOG_B, true, FUSE_NONE>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            }
            return true;
        }();
        (void)once;
        const dim3 g(CL, nrows);
        if (inverse)
            launch_cluster(k_ntt_fused<LOG_N1, LOG_B, true, FUSE_NONE>, g, CL, st, c, data, rm, fz);
        else if (fuse == FUSE_MODDOWN)
            launch_cluster(k_ntt_fused<LOG_N1, LOG_B, false, FUSE_MODDOWN>, g, CL, st, c, data, rm, fz);
        else
            launch_cluster(k_ntt_fused<LOG_N1, LOG_B, false, FUSE_NONE>, g, CL, st, c, data, rm, fz);
        note_launch(1);
        return;
    }
    // Opt-in (FHE_NTT_TWR=R > 1): the row phase keeps its twiddles in shared memory for R rows
    // of the same prime (k_ntt_rows_tw), R small enough to leave two waves of CTAs. Off by
    // default: on the B200 it loses 2-5 % (cfg3 batch-16 conv 2133 -> 2046-2083 conv/s, ModUp
    // 0.626 -> 0.65-0.70 ms; profiles/ab_r02_ntt_twiddles.txt) -- 114-128 registers and the
    // 50 KB table leave 4 CTAs per SM instead of 5, which costs more than the L2 twiddle
    // reads it removes.
    if (rm.row0 == 0 && FHE_NTT_CHUNK == 0 && nrows % rm.rows_per_poly == 0) {
        const int npoly = nrows / rm.rows_per_poly;
        int R = std::min(ntt_tw_rows(), npoly);
        while (R > 1 && (size_t)(N1 / BPC) * rm.rows_per_poly * ((npoly + R - 1) / R) < (size_t)148 * 5 * 2) R /= 2;
        if (R >= 2) {
            constexpr size_t smem = (size_t)(((BPC * (B + (B >> 4)) + 1) & ~1) + 2 * BPC * (B - 1)) * 8;
            static const bool once = [] {
                cudaFuncSetAttribute(k_ntt_rows_tw<LOG_N1, LOG_B, false, FUSE_NONE>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(k_ntt_rows_tw<LOG_N1, LOG_B, false, FUSE_MODDOWN>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                cudaFuncSetAttribute(k_ntt_rows_tw<LOG_N1, LOG_B, true, FUSE_NONE>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                return true;
            }();
            (void)once;
            const dim3 ga(B / C, nrows), gt(N1 / BPC, rm.rows_per_poly * ((npoly + R - 1) / R));
            if (!inverse) {
                k_ntt_cols<LOG_N1, LOG_B, C, false><<<ga, NTT_THREADS, 0, st>>>(c, data, rm);
                if (fuse == FUSE_MODDOWN)
                    k_ntt_rows_tw<LOG_N1, LOG_B, false, FUSE_MODDOWN><<<gt, NTT_THREADS, smem, st>>>(c, data, rm, fz, npoly, R);
                else
                    k_ntt_rows_tw<LOG_N1, LOG_B, false, FUSE_NONE><<<gt, NTT_THREADS, smem, st>>>(c, data, rm, fz, npoly, R);
            } else {
                k_ntt_rows_tw<LOG_N1, LOG_B, true, FUSE_NONE><<<gt, NTT_THREADS, smem, st>>>(c, data, rm, fz, npoly, R);
                k_ntt_cols<LOG_N1, LOG_B, C, true><<<ga, NTT_THREADS, 0, st>>>(c, data, rm);
            }
            note_launch(2);
            return;
        }
    }
    // Opt-in (FHE_NTT_PF=R > 1): forward row phase with the next row's residues prefetched
    // (k_ntt_rows_pf). Off by default: 1-2 % slower on the B200 at R = 2 / 4 / 8 and at 3 or 4 CTAs
    // per SM (the second register set spills at 128 registers; profiles/ab_r02_ntt_prefetch.txt).
    if (!inverse && rm.row0 == 0 && FHE_NTT_CHUNK == 0 && nrows % rm.rows_per_poly == 0) {
        const int npoly = nrows / rm.rows_per_poly;
        int R = std::min(ntt_pf_rows(), npoly);
        while (R > 1 && (size_t)(N1 / BPC) * rm.rows_per_poly * ((npoly + R - 1) / R) < (size_t)148 * 4 * 2) R /= 2;
        if (R >= 2) {
            const dim3 ga(B / C, nrows), gt(N1 / BPC, rm.rows_per_poly * ((npoly + R - 1) / R));
            k_ntt_cols<LOG_N1, LOG_B, C, false><<<ga, NTT_THREADS, 0, st>>>(c, data, rm);
            if (fuse == FUSE_MODDOWN)
                k_ntt_rows_pf<LOG_N1, LOG_B, FUSE_MODDOWN><<<gt, NTT_THREADS, 0, st>>>(c, data, rm, fz, npoly, R);
            else
                k_ntt_rows_pf<LOG_N1, LOG_B, FUSE_NONE><<<gt, NTT_THREADS, 0, st>>>(c, data, rm, fz, npoly, R);
            note_launch(2);
            return;
        }
    }
    // rows in chunks whose intermediate (column pass -> row pass) stays in L2
    const int chunk = FHE_NTT_CHUNK > 0 ? std::max(1, (int)(((size_t)FHE_NTT_CHUNK << 20) / ((size_t)c.N * 8))) : nrows;
    for (int r0 = 0; r0 < nrows; r0 += chunk) {
        const int nr_ = std::min(chunk, nrows - r0);
        RowMap rc = rm;
        rc.row0 = rm.row0 + r0;
        const dim3 ga(B / C, nr_), gb((N1 + BPC - 1) / BPC, nr_);
        if (!inverse) {
            k_ntt_cols<LOG_N1, LOG_B, C, false><<<ga, NTT_THREADS, 0, st>>>(c, data, rc);
            if (fuse == FUSE_MODDOWN)
                k_ntt_rows<LOG_N1, LOG_B, false, FUSE_MODDOWN><<<gb, NTT_THREADS, 0, st>>>(c, data, rc, fz);
            else
                k_ntt_rows<LOG_N1, LOG_B, false, FUSE_NONE><<<gb, NTT_THREADS, 0, st>>>(c, data, rc, fz);
        } else {
            k_ntt_rows<LOG_N1, LOG_B, true, FUSE_NONE><<<gb, NTT_THREADS, 0, st>>>(c, data, rc, fz);
            k_ntt_cols<LOG_N1, LOG_B, C, true><<<ga, NTT_THREADS, 0, st>>>(c, data, rc);
        }
        note_launch(2);
    }
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
               int nsrc, const ModUpDigit* tables, int level, int dn, cudaStream_t st, int limb) {
    const int ne = level + 1 + c.K;
    NttFuse fz{};
    fz.limb = limb;
    fz.coef = coef;
    fz.c1 = c1;
    fz.c1_stride = c1_stride;
    fz.mu = tables;
    fz.dn = dn;
    {
        const size_t total = (size_t)nsrc * dn * (c.N / 2);
        const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
        switch (c.K) {
            case 1: k_bconv_modup<1><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
            case 2: k_bconv_modup<2><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
            case 3: k_bconv_modup<3><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
            default: k_bconv_modup<4><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
        }
        note_launch(1);
    }
    ntt_run(c, digits, nsrc * dn * ne, RowMap{ne, level, c.L, c.K, dn, limb}, false, FUSE_NONE, fz, st);
}

// coefficient-domain ModDown (one thread per coefficient pair and q row)
template <int KA>
__global__ void __launch_bounds__(256) k_moddown_coef(DevCtx c, uint64_t* out, const uint64_t* y,
                                                      const ModDownTable* md, int level, int npoly) {
    const int nr = level + 1, ne = nr + c.K;
    const int halfN = c.N / 2;
    const int total = npoly * nr * halfN;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int row = idx >> (c.logN - 1);
        const size_t k = (size_t)(idx & (halfN - 1)) * 2;
        const int pp = row / nr, t = row - pp * nr;
        const uint64_t qt = c.primes[t].q;
        const uint64_t* yp = y + (size_t)pp * ne * c.N;
        uint64_t c0 = 0, c1 = 0;
        int n0 = 0, n1 = 0;
#pragma unroll
        for (int a = 0; a < KA; ++a) {
            const uint64_t q = c.primes[c.L + a].q;
            const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(yp + (size_t)(nr + a) * c.N + k);
            const uint64_t v0 = mul_shoup(x.x, md->pinv[a], md->pinv_sh[a], q);
            const uint64_t v1 = mul_shoup(x.y, md->pinv[a], md->pinv_sh[a], q);
            n0 += v0 > (q >> 1);
            n1 += v1 > (q >> 1);
            c0 = add_mod(c0, mul_shoup(v0, md->hat[t][a], md->hat_sh[t][a], qt), qt);
            c1 = add_mod(c1, mul_shoup(v1, md->hat[t][a], md->hat_sh[t][a], qt), qt);
        }
        for (int n = 0; n < n0; ++n) c0 = sub_mod(c0, md->pmod[t], qt);
        for (int n = 0; n < n1; ++n) c1 = sub_mod(c1, md->pmod[t], qt);
        const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(yp + (size_t)t * c.N + k);
        const uint64_t o0 = mul_shoup(sub_mod(x.x, c0, qt), md->pinvq[t], md->pinvq_sh[t], qt);
        const uint64_t o1 = mul_shoup(sub_mod(x.y, c1, qt), md->pinvq[t], md->pinvq_sh[t], qt);
        *reinterpret_cast<ulonglong2*>(out + (size_t)row * c.N + k) = make_ulonglong2(o0, o1);
    }
}

void moddown_coef(const DevCtx& c, uint64_t* out, const uint64_t* y, const ModDownTable* md, int level, int npoly,
                  cudaStream_t st) {
    const size_t total = (size_t)npoly * (level + 1) * (c.N / 2);
    const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    switch (c.K) {
        case 1: k_moddown_coef<1><<<blocks, 256, 0, st>>>(c, out, y, md, level, npoly); break;
        case 2: k_moddown_coef<2><<<blocks, 256, 0, st>>>(c, out, y, md, level, npoly); break;
        case 3: k_moddown_coef<3><<<blocks, 256, 0, st>>>(c, out, y, md, level, npoly); break;
        default: k_moddown_coef<4><<<blocks, 256, 0, st>>>(c, out, y, md, level, npoly); break;
    }
    note_launch(1);
}

void ntt_modup_coef(const DevCtx& c, uint64_t* digits, const uint64_t* coef, int nsrc, const ModUpDigit* tables,
                    int level, int dn, cudaStream_t st, int limb) {
    const int ne = level + 1 + c.K;
    NttFuse fz{};
    fz.coef = coef;
    fz.c1 = nullptr;
    fz.mu = tables;
    fz.dn = dn;
    const size_t total = (size_t)nsrc * dn * (c.N / 2);
    const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
    switch (c.K) {
        case 1: k_bconv_modup<1><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
        case 2: k_bconv_modup<2><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
        case 3: k_bconv_modup<3><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
        default: k_bconv_modup<4><<<blocks, 256, 0, st>>>(c, digits, fz, level, nsrc); break;
    }
    note_launch(1);
    ntt_run(c, digits, nsrc * dn * ne, RowMap{ne, level, c.L, 0, dn, limb}, false, FUSE_NONE, fz, st);
}

void ntt_moddown(const DevCtx& c, uint64_t* conv, const uint64_t* pcoef, const uint64_t* acc, size_t acc_stride,
                 uint64_t* out, const ModDownTable* md, int level, int npoly, const uint64_t* add_src,
                 uint32_t galois, cudaStream_t st, uint64_t* const* outp) {
    const int nr = level + 1;
    NttFuse fz{};
    fz.outp = outp;
    fz.pc = pcoef;
    fz.md = md;
    fz.acc = acc;
    fz.acc_stride = acc_stride;
    fz.out = out;
    fz.add_src = add_src;
    fz.galois = galois;
    {
        const size_t total = (size_t)npoly * (c.N / 2);
        const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
        switch (c.K) {
            case 1: k_bconv_moddown<1><<<blocks, 256, 0, st>>>(c, conv, fz, level, npoly); break;
            case 2: k_bconv_moddown<2><<<blocks, 256, 0, st>>>(c, conv, fz, level, npoly); break;
            case 3: k_bconv_moddown<3><<<blocks, 256, 0, st>>>(c, conv, fz, level, npoly); break;
            default: k_bconv_moddown<4><<<blocks, 256, 0, st>>>(c, conv, fz, level, npoly); break;
        }
        note_launch(1);
    }
    ntt_run(c, conv, npoly * nr, RowMap{nr, level, c.L, 0, 0}, false, FUSE_MODDOWN, fz, st);
}

void ntt_moddown_rescale(const DevCtx& c, uint64_t* w, const uint64_t* pcoef, const uint64_t* qlc, const uint64_t* acc,
                         size_t acc_stride, uint64_t* out, const ModDownTable* md, const uint64_t* pqlinv,
                         const uint64_t* pqlinv_sh, int level, int npoly, cudaStream_t st, const uint64_t* bias,
                         int bias_mod) {
    NttFuse fz{};
    fz.add_src = bias;
    fz.add_mod = bias ? bias_mod : 0;
    fz.add_stride = (size_t)level * c.N;
    fz.md = md;
    fz.acc = acc;
    fz.acc_stride = acc_stride;
    fz.out = out;
    fz.outmul = pqlinv;
    fz.outmul_sh = pqlinv_sh;
    {
        const size_t total = (size_t)npoly * (c.N / 2);
        const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
        switch (c.K) {
            case 1: k_bconv_mdr<1><<<blocks, 256, 0, st>>>(c, w, pcoef, qlc, md, level, npoly); break;
            case 2: k_bconv_mdr<2><<<blocks, 256, 0, st>>>(c, w, pcoef, qlc, md, level, npoly); break;
            case 3: k_bconv_mdr<3><<<blocks, 256, 0, st>>>(c, w, pcoef, qlc, md, level, npoly); break;
            default: k_bconv_mdr<4><<<blocks, 256, 0, st>>>(c, w, pcoef, qlc, md, level, npoly); break;
        }
        note_launch(1);
    }
    ntt_run(c, w, npoly * level, RowMap{level, level - 1, c.L, 0, 0}, false, FUSE_MODDOWN, fz, st);
}

}  // namespace fhe
