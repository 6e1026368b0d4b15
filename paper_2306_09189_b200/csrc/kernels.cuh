// Device data structures and kernel launchers of the encrypted-conv hot path.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "modarith.cuh"

namespace fhe {

constexpr int kMaxPrimes = 40;  // n_q + n_p
constexpr int kMaxAlpha = 4;    // special primes / digit size
constexpr int kMaxTerms = 32;   // rotation terms per fused MAC launch

// Basis of a batch of residue rows. Row r belongs to poly r / rows_per_poly
// and to extended row u = r % rows_per_poly, whose prime index is
// u <= level ? u : L + (u - level - 1)   (q_0..q_level, then p_0..p_{K-1}).
// With skip_alpha > 0, rows u in digit (r / rows_per_poly)'s own range
// [j a, min(j a + a, level + 1)) are skipped (ModUp digits keep those rows
// in the NTT domain already).
struct RowMap {
    int rows_per_poly;
    int level;
    int L;
    int skip_alpha;
    int skip_dn;  // digits per source when several ModUps are batched (0: one source)
    int limb;     // forward NTT: store the output rows in limb form (modarith.cuh)
    int row0;     // NTT launches: first row of this launch (row-chunked transforms)
};

FHE_HD int row_prime(const RowMap& m, int u) { return u <= m.level ? u : m.L + (u - m.level - 1); }

// Per-context device constants, passed to kernels by value.
struct DevCtx {
    int logN;
    int N;
    int L;  // ciphertext primes
    int K;  // special primes
    const Prime* primes;    // [L+K]
    const uint64_t* tw;     // [L+K][N] psi^brv(k)
    const uint64_t* tw_sh;  // Shoup companions
    const uint64_t* itw;    // [L+K][N] psi^-brv(k)
    const uint64_t* itw_sh;
    const uint64_t* ninv;  // [L+K] N^-1 and Shoup
    const uint64_t* ninv_sh;
    // FP64 NTT companions (primes q < 2^50, ntt.cu): centred twiddle w_c and w_c / q
    const double2* twd;    // [L+K][N] of psi^brv(k)
    const double2* itwd;   // [L+K][N] of psi^-brv(k)
    const double2* ninvd;  // [L+K] of N^-1
};

// FastBConv constants of ModUp digit j at level l.
struct ModUpDigit {
    int lo, hi;                          // q indices of the digit
    uint64_t inv[kMaxAlpha];             // [(Q_J/q_i)^-1]_{q_i}
    uint64_t inv_sh[kMaxAlpha];
    uint64_t hat[kMaxPrimes][kMaxAlpha];  // [Q_J/q_i]_{t_u}
    uint64_t hat_sh[kMaxPrimes][kMaxAlpha];
    uint64_t qj[kMaxPrimes];  // [Q_J]_{t_u}
};

// ModDown constants (level independent: rows are q_0..q_{L-1}).
struct ModDownTable {
    uint64_t pinv[kMaxAlpha];  // [(P/p_k)^-1]_{p_k}
    uint64_t pinv_sh[kMaxAlpha];
    uint64_t hat[kMaxPrimes][kMaxAlpha];  // [P/p_k]_{q_i}
    uint64_t hat_sh[kMaxPrimes][kMaxAlpha];
    uint64_t pmod[kMaxPrimes];  // [P]_{q_i}
    uint64_t pmod_sh[kMaxPrimes];
    uint64_t pinvq[kMaxPrimes];  // [P^-1]_{q_i}
    uint64_t pinvq_sh[kMaxPrimes];
};

// Rotation terms of one fused multiply-accumulate launch.
struct MacTerms {
    int n;
    uint32_t galois[kMaxTerms];           // 1 = identity term
    const uint64_t* key[kMaxTerms];        // [dnum][2][L+K][N], null for identity
    const uint64_t* pt[kMaxTerms];         // [level+1+K][N]
};

// Baby steps of the BSGS conv: rotations of one hoisted
// source, each multiplied by up to kMaxGiant rotated plaintexts.
constexpr int kMaxBaby = 32;
constexpr int kMaxGiant = 16;
struct BabyTerms {
    int nb;                          // baby steps
    int ngi;                         // giant accumulators in this launch
    int nb_total;                    // plaintext matrix row length
    int g0;                          // first giant index of this launch
    uint32_t galois[kMaxBaby];       // 1 = identity
    const uint64_t* key[kMaxBaby];
    uint32_t gmask[kMaxBaby];        // bit (g - g0) set when pt[g][b] is non-empty
    const uint64_t* pts;             // [ngi_total][nb_total][ne][N]
};

// Operands of the fused NTT modes (ntt.cu)
struct NttFuse {
    // ModUp: digits of nsrc sources from their INTT'd rows
    const uint64_t* coef;   // [nsrc][level+1][N] coefficient domain
    const uint64_t* c1;     // NTT-domain input of source s at c1 + s * c1_stride
    size_t c1_stride;
    const ModUpDigit* mu;   // [dnum] tables of the level
    int dn;
    // ModDown
    const uint64_t* pc;     // [npoly][K][N] INTT'd special-prime rows
    const ModDownTable* md;
    const uint64_t* acc;    // poly pp at acc + pp * acc_stride, [ne][N] each
    size_t acc_stride;
    uint64_t* out;          // [npoly][level+1][N]
    uint64_t* const* outp;  // optional: poly pp written to outp[pp / 2] + (pp % 2) [level+1][N] (ciphertexts)
    const uint64_t* add_src;
    uint32_t galois;
    int limb;  // ModUp: digit rows in limb form (own rows copied from c1 converted here)
    // add_mod > 0: add_src is added (unpermuted) to EVERY even poly pp (the c0 of
    // output ciphertext pp / 2), from add_src + ((pp / 2) % add_mod) * add_stride
    // (the conv bias plaintexts of the output shards)
    int add_mod;
    size_t add_stride;
    // fused ModDown+rescale: output multiplier (P q_l)^-1 per row instead of P^-1
    const uint64_t* outmul;
    const uint64_t* outmul_sh;
};

// --------------------------------------------------------------- launchers
// total number of kernels enqueued by this library (for the bench's gpu_launches)
uint64_t launches_total();
void note_launch(int n);

// All launchers enqueue on `st` and never synchronise.
void ntt_forward(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st);
void ntt_inverse(const DevCtx& c, uint64_t* data, int nrows, const RowMap& rm, cudaStream_t st);
// ModUp FastBConv fused into the forward NTT: digits = [nsrc][dn][ne][N] (limb != 0: limb form)
void ntt_modup(const DevCtx& c, uint64_t* digits, const uint64_t* coef, const uint64_t* c1, size_t c1_stride,
               int nsrc, const ModUpDigit* tables, int level, int dn, cudaStream_t st, int limb = 0);
// ModUp of nsrc coefficient-domain sources coef = [nsrc][level+1][N]: every
// digit row (own rows included) = conversion of coef, then the forward NTT
void ntt_modup_coef(const DevCtx& c, uint64_t* digits, const uint64_t* coef, int nsrc, const ModUpDigit* tables,
                    int level, int dn, cudaStream_t st, int limb = 0);
// coefficient-domain ModDown: out[p][t] = (y[p][t] - conv_P->q_t(y[p][P rows])) P^-1, y = [npoly][ne][N]
void moddown_coef(const DevCtx& c, uint64_t* out, const uint64_t* y, const ModDownTable* md, int level, int npoly,
                  cudaStream_t st);
// ModDown FastBConv + finish fused into the forward NTT of conv (scratch [npoly][level+1][N]):
// out[p] = (acc[p] - NTT(FastBConv_P->Q(pcoef[p]))) P^-1 (+ sigma_g(add_src) on poly 0)
void ntt_moddown(const DevCtx& c, uint64_t* conv, const uint64_t* pcoef, const uint64_t* acc, size_t acc_stride,
                 uint64_t* out, const ModDownTable* md, int level, int npoly, const uint64_t* add_src,
                 uint32_t galois, cudaStream_t st, uint64_t* const* outp = nullptr);

void reduce_signed_rows(const DevCtx& c, const int64_t* coef, uint64_t* out, int nrows, const RowMap& rm,
                        cudaStream_t st);
void sample_uniform_rows(const DevCtx& c, uint64_t* out, int nrows, const RowMap& rm, uint64_t key,
                         cudaStream_t st);
void sample_gauss(const DevCtx& c, int64_t* out, uint64_t key, cudaStream_t st);
void sample_ternary(const DevCtx& c, int64_t* out, uint64_t key, cudaStream_t st);

// key[j][0][t] = e[t] - a[t] s[t] + [t in digit j] pmod[t] sigma_g(s)[t]; a already in key[j][1]
void keygen_combine(const DevCtx& c, uint64_t* key_b, const uint64_t* key_a, const uint64_t* e,
                    const uint64_t* s, uint32_t galois, int lo, int hi, const ModDownTable* md, int nrows,
                    cudaStream_t st, const uint64_t* target = nullptr);
// ct x ct tensor product: d = [3][level+1][N] from a, b = [2][level+1][N] (NTT domain)
void tensor(const DevCtx& c, uint64_t* d, const uint64_t* a, const uint64_t* b, int level, cudaStream_t st);
// c0 = e - a s + pt (rows 0..level), a already in c1
void encrypt_combine(const DevCtx& c, uint64_t* c0, const uint64_t* c1, const uint64_t* e,
                     const uint64_t* s, const uint64_t* pt, int nrows, cudaStream_t st);
// m = c0 + c1 s for rows 0..nrows-1
void decrypt_combine(const DevCtx& c, uint64_t* m, const uint64_t* c0, const uint64_t* c1,
                     const uint64_t* s, int nrows, cudaStream_t st);

// elementwise over rows 0..nrows-1 of the Q basis (row r -> prime r % rows_per_poly)
void ew_add(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp,
            cudaStream_t st);
void ew_sub(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows, int rpp,
            cudaStream_t st);
// out[p][u] = a[p][u] * b[u] (b is one poly broadcast over the polys of a)
struct RowConsts {
    uint64_t v[kMaxPrimes];
};
// ciphertext (2 polys of nr rows) + / x a per-prime constant (mul = 0: add to poly 0)
void ew_const(const DevCtx& c, uint64_t* out, const uint64_t* a, const RowConsts& k, int nr, int mul,
              cudaStream_t st);
void ew_mul_bcast(const DevCtx& c, uint64_t* out, const uint64_t* a, const uint64_t* b, int nrows,
                  int rpp, cudaStream_t st);
void automorph(const DevCtx& c, uint64_t* out, const uint64_t* in, int nrows, uint32_t galois,
               cudaStream_t st);

// rescale: tmp holds INTT'd last rows of both polys ([2][N]); writes
// spread[2][level][N] = centered tmp mod q_i (coefficient domain)
void rescale_spread(const DevCtx& c, const uint64_t* tmp, uint64_t* spread, int level, cudaStream_t st);
// out[p][i] = (in[p][i] - spread[p][i]) * q_level^-1
void rescale_finish(const DevCtx& c, uint64_t* out, const uint64_t* in, const uint64_t* spread, int level,
                    const uint64_t* qlinv, const uint64_t* qlinv_sh, cudaStream_t st);


// acc_c[u][k] = sum_j D[j][u][perm_g(k)] key[j][c][prime(u)][k], ne = level+1+K rows
void ks_inner_product(const DevCtx& c, const uint64_t* digits, const uint64_t* key, uint64_t* acc0,
                      uint64_t* acc1, uint32_t galois, int level, int dn, cudaStream_t st);

// copy the K special rows of each poly's accumulator into [npoly][K][N]
// dst[p] = src[p * stride] row (N words) for p < npoly
void gather_row(const DevCtx& c, uint64_t* dst, const uint64_t* src, size_t stride, int npoly, cudaStream_t st);
// fused ModDown + rescale (fheconv.cu moddown_rescale): pcoef = INTT'd special rows
// [npoly][K][N], qlc = INTT'd q_l rows [npoly][N], w scratch [npoly][level][N]
// bias (optional): [bias_mod][level][N] plaintext rows added to the c0 of output i from
// bias + (i % bias_mod) * level * N
void ntt_moddown_rescale(const DevCtx& c, uint64_t* w, const uint64_t* pcoef, const uint64_t* qlc, const uint64_t* acc,
                         size_t acc_stride, uint64_t* out, const ModDownTable* md, const uint64_t* pqlinv,
                         const uint64_t* pqlinv_sh, int level, int npoly, cudaStream_t st,
                         const uint64_t* bias = nullptr, int bias_mod = 1);
void gather_special(const DevCtx& c, uint64_t* dst, const uint64_t* acc, size_t acc_stride, int level, int npoly,
                    cudaStream_t st);

// Fused conv multiply-accumulate: for every term i
//   ACC0 += pt_i * (IP_0(D, key_i, g_i) + [u<=l] P sigma_gi(X.c0))
//   ACC1 += pt_i * IP_1(D, key_i, g_i)
// identity terms (g = 1): ACC_c += pt_i * [u<=l] P X.c
void conv_mac(const DevCtx& c, uint64_t* acc, const uint64_t* digits, const uint64_t* x, const MacTerms& t,
              const ModDownTable* md, int level, int dn, cudaStream_t st);

// Y[g][c] = sum_b pt[g0 + g][b] * XT[b][c] for g < t.ngi, Y = [ngi][2][ne][N] (overwritten)
void pt_matvec(const DevCtx& c, uint64_t* Y, const uint64_t* XT, const BabyTerms& t, int level, cudaStream_t st);
// Streaming key-switch term list (k_ks_stream): term t uses Galois element
// galois[t], key[t], digits + t * digit_stride and the NTT-domain c0[t].
struct KsStream {
    int n;
    uint32_t galois[kMaxBaby];
    const uint64_t* key[kMaxBaby];
    const uint64_t* c0[kMaxBaby];
    int slot[kMaxBaby];        // mode 0: output slot in out = [slots][2][ne][N]
    int c0_qp;                 // c0[t] is a P-scaled QP-basis poly [ne][N], added unscaled
    const uint64_t* digits;
    size_t digit_stride;
    uint64_t* out;             // mode 0: XT; mode 1: acc [2][ne][N]
};
// mode 0: XT[slot_t] = key switch of term t; mode 1: acc += sum_t key switch of term t
void ks_stream(const DevCtx& c, const KsStream& a, int mode, const ModDownTable* md, int level, int dn,
               cudaStream_t st);
// xt = P ct (q rows), 0 (special rows): the identity baby step
void identity_term(const DevCtx& c, uint64_t* xt, const uint64_t* ct, const ModDownTable* md, int level,
                   cudaStream_t st);
// Batched key switching over nsrc sources (k_ks_batch): term t of source s uses
// digits + s * digit_src_stride + t * digit_term_stride and c0 + s * c0_src_stride + c0_off[t].
struct KsBatch {
    int n, nsrc;
    uint32_t galois[kMaxBaby];
    const uint64_t* key[kMaxBaby];
    size_t c0_off[kMaxBaby];
    int slot[kMaxBaby];
    const uint64_t* digits;
    size_t digit_src_stride, digit_term_stride;
    const uint64_t* c0;
    size_t c0_src_stride;
    int c0_qp;
    // digits, keys and c0 in operand form (modarith.cuh to_opf): mode 0 (k_ks_hoist_opf)
    // c0 = the P-scaled [P c]_q of ct_prescale, same [2][level+1][N] layout; mode 1
    // (k_ks_giant_opf) c0 = operand-form copies of the QP c0 rows at c0 + c0_off[t]
    int opf;
    uint64_t* out;  // mode 0: XT of source s at out + s * out_src_stride; mode 1: acc of source s
    size_t out_src_stride;
};
void ks_batch(const DevCtx& c, const KsBatch& a, int mode, const ModDownTable* md, int level, int dn,
              cudaStream_t st);
void pt_matvec_batch(const DevCtx& c, uint64_t* Y, size_t y_src_stride, const uint64_t* XT, size_t xt_src_stride,
                     const BabyTerms& t, int level, int nsrc, cudaStream_t st);
void identity_batch(const DevCtx& c, uint64_t* xt, size_t xt_src_stride, const uint64_t* ct, size_t ct_src_stride,
                    const ModDownTable* md, int level, int nsrc, cudaStream_t st);
// Fused BSGS baby steps (k_bsgs_fused): for every source s and
// giant g of the launch,
//   Y_g(s) = sum_b pt'[g][b] * X~_b(s),
//   X~_b(s) = (IP_0(D(s), key_b, g_b) + [u<=l] P sigma_b(c0(s)), IP_1(...))   (QP basis)
// with X~_b never written to memory; the identity baby (key null) is P ct(s).
// Keys and plaintexts are staged once per CTA and shared by its sources.
constexpr int kMaxFused = 96;
constexpr int kFusedMaxG = 5;
struct FusedBsgs {
    int nb, ng, nsrc;
    uint32_t galois[kMaxFused];
    const uint64_t* key[kMaxFused];  // [dnum][2][L+K][N], null: identity baby
    uint32_t gmask[kMaxFused];       // bit g: pt'[g][b] is non-empty
    const uint64_t* pt[kMaxFused];   // pt'[g][b] = pt[b] + g * pt_g_stride, [ne][N]
    size_t pt_g_stride;
    const uint64_t* digits;          // source s: digits + s * digit_src_stride, [dn][ne][N]
    size_t digit_src_stride;
    const uint64_t* ct;              // source s: ct + s * ct_src_stride, [2][level+1][N]
    size_t ct_src_stride;
    uint64_t* Y;                     // Y_g(s) = Y + s * y_src_stride + g * y_g_stride, [2][ne][N]
    size_t y_src_stride, y_g_stride;
    // paper schedules: baby b reads its digits / ciphertext from slot srcslot[b]
    // (digits + srcslot * digit_slot_stride, ct + srcslot * ct_slot_stride)
    uint16_t srcslot[kMaxFused];
    size_t digit_slot_stride, ct_slot_stride;
    int accumulate;                  // Y_g += (instead of =)
};
void bsgs_fused(const DevCtx& c, const FusedBsgs& a, const ModDownTable* md, int level, int dn, cudaStream_t st);
// The same baby steps on operand-form rows (modarith.cuh to_opf) with
// TMA tensor-copy staging (k_bsgs_tma): a.key[b] and a.pt[b] in operand form, a.digits
// the operand-form ModUp digits, a.ct the operand-form P-scaled ciphertexts [P c]_q
// ([2][level+1][N] per source, ct_prescale). Same Y (normal form, bit-identical).
// No source slots / accumulation, ng <= kFusedMaxG. The four 4-D maps
// (innermost dimension first, 8-byte elements) and their boxes, P2 = 2 * 128 / SG
// coefficients per CTA block (tma_sources(nsrc) = SG):
//   key: limb keys [nkeys][2 dnum][L+K][N],  box {P2, 1, 2 dn, 1}, coords (k0, prime, 0, kidx[b])
//   pt : limb plaintexts [ngi][nb][ne][N],   box {P2, 1, 1, NG},  coords (k0, u, bidx[b], g0)
//   dig: limb digits [nsrc][dn][ne][N],      box {P2, 1, dn, SG}, coords (blk, u, 0, s0c)
//   ct : limb [P c] [nsrc][2][level+1][N],   box {P2, 1, 2, SG},  coords (blk, u or 0, 0, s0c)
// (s0c = min(s0, nsrc - SG): no box leaves its tensor -- a partially out-of-bounds box hangs the
// mbarrier -- and the plaintext set is padded to the giants the boxes span, limb_giants)
// with NG = 3 when ng <= 3, else kFusedMaxG.
struct TmaMaps {
    CUtensorMap key, pt, dig, ct;  // dig / ct: 5-D, dimension 3 = source slot (FusedBsgs.srcslot)
    int16_t kidx[kMaxFused];  // baby b's key in the key map, -1: identity
    int16_t bidx[kMaxFused];  // baby b's index in the plaintext map
    int16_t gidx[kMaxFused];  // baby b's giant-coordinate offset (added to g0; 0 unless set)
    int g0;                   // first giant of the launch
    int ng1;                  // the plaintext box spans one giant (paper schedules: ng == 1)
    // work queues (k_bsgs_tma): extended rows in queue order, the nint integer-path
    // (q >= 2^50) rows first; sched = [2 queue heads][256 per-SM arrival counters],
    // zeroed before every launch (bsgs_tma does it on the launch stream)
    uint8_t rowlist[kMaxPrimes];
    int nint;
    unsigned* sched;
};
constexpr int kTmaSchedWords = 2 + 256;
constexpr int kTmaSchedSlots = 16;  // per compute stream (fheconv.cu tma_rows)
// Hoisted key switches on the same kernel (k_bsgs_tma MODE 1, no plaintexts): every
// baby's X~_b (keyed, [P sigma(c0)] folded into poly 0) is written in the QP basis to
// a.Y + s * a.y_src_stride + b * a.y_g_stride; the pt map is unused.
void bsgs_tma_hoist(const DevCtx& c, const FusedBsgs& a, const TmaMaps& m, int level, int dn, cudaStream_t st);
// encode a 5-D uint64 tensor map (dims innermost first, dense)
void tma_map5(CUtensorMap* map, const void* base, const uint64_t dims[5], const uint32_t box[5]);
// Sources per CTA of k_bsgs_tma. The key and plaintext blocks of a CTA are shared by its SG
// sources: 106 / 89 / 80 bytes of L2 -> SM operand traffic per (source, coefficient, baby step)
// at SG = 4 / 8 / 16 (39 GB per cfg3 batch-16 launch at SG = 4, ncu
// l1tex__m_xbar2l1tex_read_bytes). Builds with -DFHE_TMA_WIDE=1 also instantiate SG = 8 and 16
// (FHECONV_TMA_SG caps it); A/B on the B200 (profiles/ab_r02_bsgs_variants.txt): SG = 8 is
// +-0 %, SG = 16 is -12 % (128-byte boxes), so the default build stops at 4.
#ifndef FHE_TMA_WIDE
#define FHE_TMA_WIDE 0
#endif
inline int tma_sg_max() {
#if FHE_TMA_WIDE
    static const int v = [] {
        const char* e = getenv("FHECONV_TMA_SG");
        const int x = e ? atoi(e) : 8;
        return x >= 16 ? 16 : x >= 8 ? 8 : 4;
    }();
    return v;
#else
    return 4;
#endif
}
inline int tma_sources(int nsrc) {
    const int m = tma_sg_max();
    return nsrc >= 16 && m >= 16 ? 16 : nsrc >= 8 && m >= 8 ? 8 : nsrc >= 4 ? 4 : nsrc >= 2 ? 2 : 1;
}
void bsgs_tma(const DevCtx& c, const FusedBsgs& a, const TmaMaps& m, int level, int dn, cudaStream_t st);
// encode a 4-D uint64 tensor map (dims innermost first, dense)
void tma_map4(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint32_t box[4]);
// dst[i] = to_opf(src[i]) for nrows rows of N words; row r uses prime
// row_prime(rm, r % rm.rows_per_poly) (rm.level < 0: prime index r % rows_per_poly)
struct GiantSel {
    int n;
    int idx[kMaxBaby];  // giant index of entry g
};
// yc[s][g] = Y(s, idx[g]).c1 rows and (yc0 != null) yc0[s][g] = to_opf(Y(s, idx[g]).c0 rows),
// Y(s, j) = Y + s * ys + j * 2 ne N ([2][ne][N] QP accumulators), one launch
// dst[s][words] = *srcp[s] for a device table of nsrc source pointers (words even), one launch
void gather_ptrs(uint64_t* dst, const uint64_t* const* srcp, size_t words, int nsrc, cudaStream_t st);
void giant_gather(const DevCtx& c, uint64_t* yc, uint64_t* yc0, const uint64_t* Y, size_t ys, int sc, const GiantSel& gs,
                  int level, cudaStream_t st);
void rows_to_limb(const DevCtx& c, uint64_t* dst, const uint64_t* src, size_t nrows, const RowMap& rm,
                  cudaStream_t st);
// dst[s][p][u] = to_opf([P ct_s[p][u]]_{q_u}) for nsrc ciphertexts at ct + s * stride ([2][level+1][N])
void ct_prescale(const DevCtx& c, uint64_t* dst, const uint64_t* ct, size_t stride, int nsrc, const ModDownTable* md,
                 int level, cudaStream_t st);
// acc += y over [2][ne][N] (QP basis)
void qp_add(const DevCtx& c, uint64_t* acc, const uint64_t* y, int level, cudaStream_t st, int S = 1, size_t as = 0,
            size_t ys = 0);

}  // namespace fhe
