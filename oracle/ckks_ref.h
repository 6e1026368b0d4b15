/* TEST INFRASTRUCTURE ONLY — the oracle (checker). Never linked into the
 * product library (paper_2306_09189_b200/libfheconv.so); only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * ckks_ref: a deterministic CPU RNS-CKKS golden model of the encrypted
 * convolution hot path. The reference (shardnn) is a double-precision
 * emulator with no cryptography (reference proj/README.md:3-9),
 * and the paper's OpenFHE backend is not vendored, has no
 * pinned version and is not installed — so CIPHERTEXT PARITY IS UNPINNED
 * against the reference. This model fixes every convention listed in
 * DESIGN.md §3 once; the GPU library must be bit-exact against it, and its
 * decrypted outputs are pinned against the compiled reference's conv_plan
 * slots (<= 1e-6).
 *
 * Layouts (all residues uint64 in [0, q)):
 *   polynomial row   : N words, NTT domain unless stated (bit-reversed order)
 *   ciphertext @ l   : [2][l+1][N]
 *   extended (QP) @ l: [l+1+K][N] rows q_0..q_l, p_0..p_{K-1}
 *   modup digits @ l : [dnum_l][l+1+K][N], dnum_l = ceil((l+1)/alpha)
 *   galois key       : [dnum][2][L+K][N] rows q_0..q_{L-1}, p_0..p_{K-1}
 */
#ifndef FHECONV_ORACLE_CKKS_REF_H
#define FHECONV_ORACLE_CKKS_REF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CK_MAXP 40

typedef struct ck_ctx ck_ctx;

ck_ctx* ck_create(int logN, int L, const int* qbits, int K, const int* pbits, int logscale);
void ck_destroy(ck_ctx* ck);

/* introspection */
uint64_t ck_prime(const ck_ctx* ck, int idx); /* idx in [0, L+K): q_0..q_{L-1}, p_0.. */
uint64_t ck_root(const ck_ctx* ck, int idx);  /* primitive 2N-th root psi */
int ck_dnum(const ck_ctx* ck);
double ck_scale(const ck_ctx* ck);

/* modular helpers exposed for KATs */
uint64_t ck_mulmod(uint64_t a, uint64_t b, uint64_t q);
int ck_is_prime(uint64_t n);
uint64_t ck_galois_elt(const ck_ctx* ck, long k);
void ck_automorph_ntt(const ck_ctx* ck, const uint64_t* in, uint64_t* out, uint64_t galois);
void ck_automorph_coef(const ck_ctx* ck, int idx, const uint64_t* in, uint64_t* out, uint64_t galois);

/* NTT (idx = prime index), in place */
void ck_ntt_fwd(const ck_ctx* ck, int idx, uint64_t* a);
void ck_ntt_inv(const ck_ctx* ck, int idx, uint64_t* a);

/* encoder: z has n_z <= N/2 real slots (rest zero) */
int ck_encode(const ck_ctx* ck, const double* z, size_t n_z, double scale, int64_t* coef);
void ck_decode(const ck_ctx* ck, const double* coef, double scale, double* z);
/* signed coefficients -> NTT rows for the given prime indices */
void ck_coef_to_ntt(const ck_ctx* ck, const int64_t* coef, const int* idx, int nrows, uint64_t* out);
/* plaintext at level l: basis Q_l (with_p = 0) or Q_l u P (with_p = 1) */
int ck_encode_plain(const ck_ctx* ck, const double* z, size_t n_z, double scale, int level,
                    int with_p, uint64_t* out);

/* keys and sampling (counter-based PRNG) */
uint64_t ck_prng(uint64_t seed, uint64_t stream, uint64_t ctr);
void ck_keygen(ck_ctx* ck, uint64_t seed);
void ck_secret_coef(const ck_ctx* ck, int64_t* s);
void ck_galois_key(const ck_ctx* ck, uint64_t galois, uint64_t* key);

/* ciphertext ops */
void ck_encrypt(const ck_ctx* ck, const uint64_t* pt, int level, uint64_t seed, uint64_t* ct);
void ck_decrypt_coef(const ck_ctx* ck, const uint64_t* ct, int level, double* coef);
void ck_decrypt_decode(const ck_ctx* ck, const uint64_t* ct, int level, double scale, double* z);
void ck_add(const ck_ctx* ck, const uint64_t* a, const uint64_t* b, int level, uint64_t* out);
void ck_mul_plain(const ck_ctx* ck, const uint64_t* ct, const uint64_t* pt, int level, uint64_t* out);
void ck_add_plain(const ck_ctx* ck, const uint64_t* ct, const uint64_t* pt, int level, uint64_t* out);
void ck_rescale(const ck_ctx* ck, const uint64_t* ct, int level, uint64_t* out);

/* key switching pieces */
int ck_dnum_at(const ck_ctx* ck, int level);
void ck_modup(const ck_ctx* ck, const uint64_t* c1, int level, uint64_t* digits);
void ck_inner_product(const ck_ctx* ck, const uint64_t* digits, int level, const uint64_t* key,
                      uint64_t galois, uint64_t* acc0, uint64_t* acc1);
void ck_moddown(const ck_ctx* ck, const uint64_t* acc, int level, uint64_t* out);

/* rotations (keys regenerated from the key seed on demand) */
void ck_rotate(const ck_ctx* ck, const uint64_t* ct, int level, long k, uint64_t* out);
void ck_mul_ct(const ck_ctx* ck, const uint64_t* a, const uint64_t* b, int level, uint64_t* out);
void ck_rotate_hoisted(const ck_ctx* ck, const uint64_t* ct, int level, const long* ks, int n,
                       uint64_t* outs);

/* Fused single-shard encrypted convolution: plan 1 =
 * Approach 1 (shifts first), plan 2 = Approach 2 (channel rotations first),
 * plan 3 = BSGS with hoisted channel rotations + aggregated shifts,
 * plan 4 = BSGS with hoisted shifts + aggregated channel rotations,
 * plan 5 = BSGS with hoisted channel+column rotations r m^2 + ll and
 *          aggregated row shifts kk m.
 * Input ct at `level` (scale = ck_scale), output ct at level - 1 after one
 * rescale; *out_scale receives the output scale. */
int ck_conv(const ck_ctx* ck, const uint64_t* ct, int level, int c, int m, int kappa, int c_out,
            const double* filt, int plan, uint64_t* out, double* out_scale);

/* Multi-shard image-mode conv (fused BSGS, see ckks_ref.c): t input shards
 * [t][2][level+1][N] -> n_out output shards [n_out][2][level][N]; returns n_out. */
int ck_conv_shards(const ck_ctx* ck, const uint64_t* cts, int t, int level, int c, int m, int kappa, int c_out,
                   const double* filt, uint64_t* outs, double* out_scale);

/* image-mode conv over a PackedImage with channel permutation tau (NULL = identity),
 * replication rep and duplication d (t = 1 only); same fused BSGS as ck_conv_shards */
int ck_conv_packed(const ck_ctx* ck, const uint64_t* cts, int t, int level, int c, int m, int kappa, int c_out,
                   const double* filt, const long* tau, int rep, int d, uint64_t* outs, double* out_scale);

/* Channel-shard mode conv (fused BSGS, see ckks_ref.c): cts [c][m^2/s][2][level+1][N]
 * -> outs [c_out][m^2/s][2][level][N]; returns the output shard count. */
int ck_conv_channel(const ck_ctx* ck, const uint64_t* cts, int level, int c, int m, int kappa, int c_out,
                    const double* filt, uint64_t* outs, double* out_scale);

/* out = Rescale(ModDown(sum_b pt_b * rot_{amounts[b]}(ct))) with QP-basis rotations;
 * pts [n][level+1+K][N] encoded over Q_l u P at scale q_l (see ckks_ref.c) */
void ck_lintrans(const ck_ctx* ck, const uint64_t* ct, int level, int n, const long* amounts, const uint64_t* pts,
                 uint64_t* out);
/* the same over nsrc source ciphertexts cts [nsrc][2][level+1][N]; term b reads cts[src[b]] */
void ck_lintrans_src(const ck_ctx* ck, const uint64_t* cts, int nsrc, int level, int n, const int* src,
                     const long* amounts, const uint64_t* pts, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
