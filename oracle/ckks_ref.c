/* TEST INFRASTRUCTURE ONLY — the oracle (checker); see ckks_ref.h.
 *
 * Deterministic CPU RNS-CKKS golden model. Every convention here is the
 * contract the GPU library (paper_2306_09189_b200/csrc) must reproduce bit
 * for bit; DESIGN.md §3 lists them. The slot-level semantics it must
 * realise come from the reference:
 *   rotate(v, k): out[i] = in[(i + k) mod s]        reference emu.cpp:15-37
 *   rotate_many: one shared decomposition            reference emu.cpp:39-54
 *   mul_plain / add / add_plain                      reference emu.cpp:56-111
 *   conv schedules (Approach 1 / 2)                  reference conv.cpp:109-211
 *   fused plaintexts (mask x weight)                 reference conv.cpp:69-85
 * Residue-level parity with the reference is UNPINNED (it has no residues);
 * the model is pinned by self-KATs (NTT vs direct evaluation, automorphism
 * vs slot rotation, encode/decode round trips) and end-to-end by decrypted
 * conv outputs vs the compiled reference (tests/test_oracle_ckks.py).
 */
#include "ckks_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "emu_ref.h"
#include "prng_tables.h"

typedef unsigned __int128 u128;

/* pi as a double literal (same literal in the product encoder) */
#define CK_PI 3.14159265358979323846

typedef struct {
    uint64_t g;
    uint64_t* key;
} key_slot;

typedef struct key_cache_s {
    key_slot* slots;
    int n, cap;
} key_cache;

static void kc_reset(key_cache* kc);

struct ck_ctx {
    int logN;
    size_t N;
    int L, K, alpha, dnum, np;
    uint64_t q[CK_MAXP];
    uint64_t psi[CK_MAXP];
    uint64_t* tw[CK_MAXP];
    uint64_t* tw_sh[CK_MAXP];
    uint64_t* itw[CK_MAXP];
    uint64_t* itw_sh[CK_MAXP];
    uint64_t ninv[CK_MAXP], ninv_sh[CK_MAXP];
    double scale;
    uint64_t key_seed;
    int have_key;
    int64_t* s_coef;
    uint64_t* s_ntt; /* [np][N] */
    uint32_t* brv;
    struct key_cache_s* kc; /* Galois / relinearisation keys generated on demand, kept until keygen / destroy */
};

/* ------------------------------------------------------------------ */
/* modular arithmetic                                                  */
/* ------------------------------------------------------------------ */

uint64_t ck_mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }

static inline uint64_t addm(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t r = a + b;
    return r >= q ? r - q : r;
}
static inline uint64_t subm(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

static uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = ck_mulmod(r, b, q);
        b = ck_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a, q - 2, q); } /* q prime */

static inline uint64_t shoup_pre(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }
static inline uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t wsh, uint64_t q) {
    const uint64_t qh = (uint64_t)(((u128)a * wsh) >> 64);
    uint64_t r = a * w - qh * q;
    return r >= q ? r - q : r;
}

/* deterministic Miller-Rabin, valid for all 64-bit n */
int ck_is_prime(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        s++;
    }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = ck_mulmod(x, x, n);
            if (x == n - 1) {
                comp = 0;
                break;
            }
        }
        if (comp) return 0;
    }
    return 1;
}

static uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

/* ------------------------------------------------------------------ */
/* parameters: primes and NTT tables (§3.3)           */
/* ------------------------------------------------------------------ */

/* Largest q < 2^bits with q = 1 mod 2N, prime, not already used. */
static uint64_t next_prime(int bits, uint64_t twoN, const uint64_t* used, int n_used) {
    uint64_t c = (((1ULL << bits) - 2) / twoN) * twoN + 1;
    for (;; c -= twoN) {
        int dup = 0;
        for (int i = 0; i < n_used; i++) dup |= used[i] == c;
        if (!dup && ck_is_prime(c)) return c;
    }
}

/* Smallest-generator primitive 2N-th root: psi = g^((q-1)/2N) for the first
 * g = 2, 3, ... with psi^N = -1. */
static uint64_t find_root(uint64_t q, uint64_t N) {
    for (uint64_t g = 2;; g++) {
        const uint64_t psi = powmod(g, (q - 1) / (2 * N), q);
        if (powmod(psi, N, q) == q - 1) return psi;
    }
}

ck_ctx* ck_create(int logN, int L, const int* qbits, int K, const int* pbits, int logscale) {
    if (L + K > CK_MAXP || L < 1 || K < 1) return NULL;
    ck_ctx* ck = calloc(1, sizeof(ck_ctx));
    ck->kc = calloc(1, sizeof(key_cache));
    ck->logN = logN;
    ck->N = (size_t)1 << logN;
    ck->L = L;
    ck->K = K;
    ck->alpha = K;
    ck->dnum = (L + K - 1) / K;
    ck->np = L + K;
    ck->scale = ldexp(1.0, logscale);
    const uint64_t twoN = 2 * ck->N;
    for (int i = 0; i < ck->np; i++) {
        const int b = i < L ? qbits[i] : pbits[i - L];
        ck->q[i] = next_prime(b, twoN, ck->q, i);
    }
    ck->brv = malloc(ck->N * sizeof(uint32_t));
    for (size_t i = 0; i < ck->N; i++) ck->brv[i] = bitrev((uint32_t)i, logN);
    for (int i = 0; i < ck->np; i++) {
        const uint64_t q = ck->q[i];
        const uint64_t psi = find_root(q, ck->N);
        const uint64_t ipsi = invmod(psi, q);
        ck->psi[i] = psi;
        ck->tw[i] = malloc(ck->N * 8);
        ck->tw_sh[i] = malloc(ck->N * 8);
        ck->itw[i] = malloc(ck->N * 8);
        ck->itw_sh[i] = malloc(ck->N * 8);
        uint64_t p = 1, ip = 1;
        uint64_t* pw = malloc(ck->N * 8);
        uint64_t* ipw = malloc(ck->N * 8);
        for (size_t k = 0; k < ck->N; k++) {
            pw[k] = p;
            ipw[k] = ip;
            p = ck_mulmod(p, psi, q);
            ip = ck_mulmod(ip, ipsi, q);
        }
        for (size_t k = 0; k < ck->N; k++) {
            ck->tw[i][k] = pw[ck->brv[k]];
            ck->itw[i][k] = ipw[ck->brv[k]];
            ck->tw_sh[i][k] = shoup_pre(ck->tw[i][k], q);
            ck->itw_sh[i][k] = shoup_pre(ck->itw[i][k], q);
        }
        free(pw);
        free(ipw);
        ck->ninv[i] = invmod(ck->N % q, q);
        ck->ninv_sh[i] = shoup_pre(ck->ninv[i], q);
    }
    return ck;
}

void ck_destroy(ck_ctx* ck) {
    if (!ck) return;
    kc_reset(ck->kc);
    free(ck->kc);
    for (int i = 0; i < ck->np; i++) {
        free(ck->tw[i]);
        free(ck->tw_sh[i]);
        free(ck->itw[i]);
        free(ck->itw_sh[i]);
    }
    free(ck->brv);
    free(ck->s_coef);
    free(ck->s_ntt);
    free(ck);
}

uint64_t ck_prime(const ck_ctx* ck, int idx) { return ck->q[idx]; }
uint64_t ck_root(const ck_ctx* ck, int idx) { return ck->psi[idx]; }
int ck_dnum(const ck_ctx* ck) { return ck->dnum; }
double ck_scale(const ck_ctx* ck) { return ck->scale; }
int ck_dnum_at(const ck_ctx* ck, int level) { return (level + 1 + ck->alpha - 1) / ck->alpha; }

/* Forward negacyclic NTT: Cooley-Tukey, natural order in, bit-reversed out:
 * out[i] = a(psi^(2 brv(i) + 1)). */
void ck_ntt_fwd(const ck_ctx* ck, int idx, uint64_t* a) {
    const size_t N = ck->N;
    const uint64_t q = ck->q[idx];
    const uint64_t* W = ck->tw[idx];
    const uint64_t* Ws = ck->tw_sh[idx];
    size_t t = N;
    for (size_t m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (size_t i = 0; i < m; i++) {
            const size_t j1 = 2 * i * t;
            const uint64_t w = W[m + i], ws = Ws[m + i];
            for (size_t j = j1; j < j1 + t; j++) {
                const uint64_t U = a[j];
                const uint64_t V = mul_shoup(a[j + t], w, ws, q);
                a[j] = addm(U, V, q);
                a[j + t] = subm(U, V, q);
            }
        }
    }
}

/* Inverse: Gentleman-Sande, bit-reversed in, natural out, times N^-1. */
void ck_ntt_inv(const ck_ctx* ck, int idx, uint64_t* a) {
    const size_t N = ck->N;
    const uint64_t q = ck->q[idx];
    const uint64_t* W = ck->itw[idx];
    const uint64_t* Ws = ck->itw_sh[idx];
    size_t t = 1;
    for (size_t m = N; m > 1; m >>= 1) {
        const size_t h = m >> 1;
        size_t j1 = 0;
        for (size_t i = 0; i < h; i++) {
            const uint64_t w = W[h + i], ws = Ws[h + i];
            for (size_t j = j1; j < j1 + t; j++) {
                const uint64_t U = a[j], V = a[j + t];
                a[j] = addm(U, V, q);
                a[j + t] = mul_shoup(subm(U, V, q), w, ws, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (size_t j = 0; j < N; j++) a[j] = mul_shoup(a[j], ck->ninv[idx], ck->ninv_sh[idx], q);
}

/* ------------------------------------------------------------------ */
/* Galois automorphisms                               */
/* ------------------------------------------------------------------ */

/* Left rotation by k slots <-> X -> X^(5^k mod 2N), k reduced mod N/2. */
uint64_t ck_galois_elt(const ck_ctx* ck, long k) {
    const long n = (long)(ck->N / 2);
    long a = k % n;
    if (a < 0) a += n;
    return powmod(5, (uint64_t)a, 2 * ck->N);
}

/* NTT domain: out[i] = in[j] with (2 brv(j) + 1) = (2 brv(i) + 1) * g mod 2N */
void ck_automorph_ntt(const ck_ctx* ck, const uint64_t* in, uint64_t* out, uint64_t g) {
    const size_t N = ck->N;
    const uint64_t mask = 2 * N - 1;
    for (size_t i = 0; i < N; i++) {
        const uint64_t e = 2 * (uint64_t)ck->brv[i] + 1;
        const uint64_t e2 = (e * g) & mask;
        out[i] = in[ck->brv[(e2 - 1) >> 1]];
    }
}

/* coefficient domain: a_i X^i -> a_i X^(i g mod 2N), X^N = -1 */
void ck_automorph_coef(const ck_ctx* ck, int idx, const uint64_t* in, uint64_t* out, uint64_t g) {
    const size_t N = ck->N;
    const uint64_t q = ck->q[idx];
    for (size_t i = 0; i < N; i++) {
        const uint64_t e = ((uint64_t)i * g) & (2 * N - 1);
        if (e < N)
            out[e] = in[i];
        else
            out[e - N] = in[i] ? q - in[i] : 0;
    }
}

/* ------------------------------------------------------------------ */
/* encoder: host double FFT, identical op order to the  */
/* product's host encoder                                               */
/* ------------------------------------------------------------------ */

typedef struct {
    double re, im;
} cplx;

static inline cplx cmul(cplx a, cplx b) {
    cplx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

/* a[k] <- sum_l a[l] exp(sign * 2 pi i k l / n), iterative radix-2 DIT */
static void fft_dit(cplx* a, size_t n, int sign) {
    int logn = 0;
    while (((size_t)1 << logn) < n) logn++;
    for (size_t i = 0; i < n; i++) {
        const size_t j = bitrev((uint32_t)i, logn);
        if (j > i) {
            cplx t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1, step = n / len;
        for (size_t i = 0; i < n; i += len) {
            for (size_t j = 0; j < half; j++) {
                const double ang = (2.0 * CK_PI * (double)(j * step)) / (double)n;
                cplx w;
                w.re = cos(ang);
                w.im = sign > 0 ? sin(ang) : -sin(ang);
                const cplx u = a[i + j];
                const cplx v = cmul(a[i + j + half], w);
                a[i + j].re = u.re + v.re;
                a[i + j].im = u.im + v.im;
                a[i + j + half].re = u.re - v.re;
                a[i + j + half].im = u.im - v.im;
            }
        }
    }
}

int ck_encode(const ck_ctx* ck, const double* z, size_t n_z, double scale, int64_t* coef) {
    const size_t N = ck->N, n = N / 2, M = 2 * N;
    if (n_z > n) return -1;
    cplx* w = calloc(n, sizeof(cplx));
    uint64_t g = 1;
    for (size_t j = 0; j < n; j++) {
        if (j < n_z) w[(g - 1) >> 2].re = z[j];
        g = (g * 5) & (M - 1);
    }
    fft_dit(w, n, -1);
    int rc = 0;
    for (size_t l = 0; l < n; l++) {
        cplx v;
        v.re = w[l].re / (double)n;
        v.im = w[l].im / (double)n;
        const double ang = (2.0 * CK_PI * (double)l) / (double)M;
        cplx zi;
        zi.re = cos(ang);
        zi.im = -sin(ang);
        const cplx u = cmul(v, zi);
        const double a = round(u.re * scale), b = round(u.im * scale);
        if (fabs(a) >= 0x1p62 || fabs(b) >= 0x1p62) rc = -2;
        coef[l] = (int64_t)a;
        coef[l + n] = (int64_t)b;
    }
    free(w);
    return rc;
}

void ck_decode(const ck_ctx* ck, const double* coef, double scale, double* z) {
    const size_t N = ck->N, n = N / 2, M = 2 * N;
    cplx* v = malloc(n * sizeof(cplx));
    for (size_t l = 0; l < n; l++) {
        cplx u;
        u.re = coef[l] / scale;
        u.im = coef[l + n] / scale;
        const double ang = (2.0 * CK_PI * (double)l) / (double)M;
        cplx zi;
        zi.re = cos(ang);
        zi.im = sin(ang);
        v[l] = cmul(u, zi);
    }
    fft_dit(v, n, +1);
    uint64_t g = 1;
    for (size_t j = 0; j < n; j++) {
        z[j] = v[(g - 1) >> 2].re;
        g = (g * 5) & (M - 1);
    }
    free(v);
}

static inline uint64_t reduce_signed(int64_t x, uint64_t q) {
    if (x >= 0) return (uint64_t)x % q;
    const uint64_t r = ((uint64_t)(-(x + 1)) + 1) % q; /* |x| mod q without overflow */
    return r ? q - r : 0;
}

void ck_coef_to_ntt(const ck_ctx* ck, const int64_t* coef, const int* idx, int nrows, uint64_t* out) {
    const size_t N = ck->N;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < nrows; r++) {
        uint64_t* row = out + (size_t)r * N;
        const uint64_t q = ck->q[idx[r]];
        for (size_t k = 0; k < N; k++) row[k] = reduce_signed(coef[k], q);
        ck_ntt_fwd(ck, idx[r], row);
    }
}

/* prime index of extended-basis row u at level l: q_0..q_l, p_0..p_{K-1} */
static inline int ext_prime(const ck_ctx* ck, int level, int u) {
    return u <= level ? u : ck->L + (u - level - 1);
}

int ck_encode_plain(const ck_ctx* ck, const double* z, size_t n_z, double scale, int level,
                    int with_p, uint64_t* out) {
    int64_t* coef = malloc(ck->N * sizeof(int64_t));
    const int rc = ck_encode(ck, z, n_z, scale, coef);
    const int nrows = level + 1 + (with_p ? ck->K : 0);
    int idx[CK_MAXP];
    for (int u = 0; u < nrows; u++) idx[u] = ext_prime(ck, level, u);
    ck_coef_to_ntt(ck, coef, idx, nrows, out);
    free(coef);
    return rc;
}

/* ------------------------------------------------------------------ */
/* sampling: counter-based SplitMix64 hash             */
/* ------------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
}
static inline uint64_t prng_k(uint64_t key, uint64_t ctr) {
    return mix64(key + ctr * 0xD1B54A32D192ED03ULL);
}
uint64_t ck_prng(uint64_t seed, uint64_t stream, uint64_t ctr) { return prng_k(stream_key(seed, stream), ctr); }

#define DOM_SECRET 1ULL
#define DOM_KEY_A 2ULL
#define DOM_KEY_E 3ULL
#define DOM_ENC_A 4ULL
#define DOM_ENC_E 5ULL
static inline uint64_t stream_id(uint64_t dom, uint64_t galois, uint64_t digit) {
    return (dom << 56) | (galois << 8) | digit;
}

static const uint64_t CDT[FHE_CDT_LEN] = {FHE_CDT_VALUES};

static inline int64_t gauss_from(uint64_t r) {
    const uint64_t r63 = r >> 1;
    int64_t x = -20;
    for (int k = 0; k < FHE_CDT_LEN; k++) x += r63 >= CDT[k];
    return x;
}
static inline uint64_t uniform_from(uint64_t hi, uint64_t lo, uint64_t q) {
    return (uint64_t)((((u128)hi << 64) | lo) % q);
}

/* error polynomial (coefficients) -> NTT rows for prime indices idx[] */
static void sample_error_ntt(const ck_ctx* ck, uint64_t key, const int* idx, int nrows, uint64_t* out) {
    const size_t N = ck->N;
    int64_t* e = malloc(N * sizeof(int64_t));
    for (size_t k = 0; k < N; k++) e[k] = gauss_from(prng_k(key, k));
    ck_coef_to_ntt(ck, e, idx, nrows, out);
    free(e);
}

void ck_keygen(ck_ctx* ck, uint64_t seed) {
    const size_t N = ck->N;
    kc_reset(ck->kc); /* keys of the previous secret are stale */
    ck->key_seed = seed;
    ck->have_key = 1;
    free(ck->s_coef);
    free(ck->s_ntt);
    ck->s_coef = malloc(N * sizeof(int64_t));
    ck->s_ntt = malloc((size_t)ck->np * N * 8);
    const uint64_t key = stream_key(seed, stream_id(DOM_SECRET, 0, 0));
    for (size_t k = 0; k < N; k++) {
        const uint64_t r = prng_k(key, k);
        ck->s_coef[k] = (int64_t)(uint64_t)(((u128)r * 3) >> 64) - 1;
    }
    int idx[CK_MAXP];
    for (int i = 0; i < ck->np; i++) idx[i] = i;
    ck_coef_to_ntt(ck, ck->s_coef, idx, ck->np, ck->s_ntt);
}

void ck_secret_coef(const ck_ctx* ck, int64_t* s) { memcpy(s, ck->s_coef, ck->N * sizeof(int64_t)); }

/* Hybrid key-switching key for s' = sigma_g(s), or s' = s^2 when g == 0:
 * key[j][0][t] = -a s + e + [t in digit j] * (P mod q_t) * s'
 * key[j][1][t] = a                                  (NTT domain)     */
void ck_galois_key(const ck_ctx* ck, uint64_t g, uint64_t* key) {
    const size_t N = ck->N;
    const int np = ck->np, L = ck->L;
    uint64_t* sp = malloc((size_t)np * N * 8);
    for (int t = 0; t < np; t++) {
        const uint64_t* s = ck->s_ntt + (size_t)t * N;
        uint64_t* d = sp + (size_t)t * N;
        if (g == 0) /* relinearisation key: s' = s^2 */
            for (size_t k = 0; k < N; k++) d[k] = ck_mulmod(s[k], s[k], ck->q[t]);
        else
            ck_automorph_ntt(ck, s, d, g);
    }
    uint64_t Pmod[CK_MAXP];
    for (int t = 0; t < np; t++) {
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[L + k] % ck->q[t], ck->q[t]);
        Pmod[t] = P;
    }
    int idx[CK_MAXP];
    for (int i = 0; i < np; i++) idx[i] = i;
    uint64_t* e = malloc((size_t)np * N * 8);
    for (int j = 0; j < ck->dnum; j++) {
        sample_error_ntt(ck, stream_key(ck->key_seed, stream_id(DOM_KEY_E, g, j)), idx, np, e);
        const uint64_t akey = stream_key(ck->key_seed, stream_id(DOM_KEY_A, g, j));
        const int lo = j * ck->alpha, hi = (j + 1) * ck->alpha < L ? (j + 1) * ck->alpha : L;
#pragma omp parallel for schedule(static)
        for (int t = 0; t < np; t++) {
            const uint64_t q = ck->q[t];
            uint64_t* b = key + (((size_t)j * 2 + 0) * np + t) * N;
            uint64_t* a = key + (((size_t)j * 2 + 1) * np + t) * N;
            const int gadget = t >= lo && t < hi;
            for (size_t k = 0; k < N; k++) {
                const uint64_t ctr = 2 * ((uint64_t)t * N + k);
                const uint64_t av = uniform_from(prng_k(akey, ctr), prng_k(akey, ctr + 1), q);
                a[k] = av;
                uint64_t bv = subm(e[(size_t)t * N + k], ck_mulmod(av, ck->s_ntt[(size_t)t * N + k], q), q);
                if (gadget) bv = addm(bv, ck_mulmod(Pmod[t], sp[(size_t)t * N + k], q), q);
                b[k] = bv;
            }
        }
    }
    free(e);
    free(sp);
}

/* Symmetric encryption at level l: (c0, c1) = (-a s + e + m, a). */
void ck_encrypt(const ck_ctx* ck, const uint64_t* pt, int level, uint64_t seed, uint64_t* ct) {
    const size_t N = ck->N;
    const int nr = level + 1;
    int idx[CK_MAXP];
    for (int i = 0; i < nr; i++) idx[i] = i;
    uint64_t* e = malloc((size_t)nr * N * 8);
    sample_error_ntt(ck, stream_key(seed, stream_id(DOM_ENC_E, 0, 0)), idx, nr, e);
    const uint64_t akey = stream_key(seed, stream_id(DOM_ENC_A, 0, 0));
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nr; t++) {
        const uint64_t q = ck->q[t];
        uint64_t* c0 = ct + (size_t)t * N;
        uint64_t* c1 = ct + ((size_t)nr + t) * N;
        for (size_t k = 0; k < N; k++) {
            const uint64_t ctr = 2 * ((uint64_t)t * N + k);
            const uint64_t av = uniform_from(prng_k(akey, ctr), prng_k(akey, ctr + 1), q);
            c1[k] = av;
            const uint64_t v = subm(e[(size_t)t * N + k], ck_mulmod(av, ck->s_ntt[(size_t)t * N + k], q), q);
            c0[k] = addm(v, pt[(size_t)t * N + k], q);
        }
    }
    free(e);
}

/* m = c0 + c1 s; centered lift by CRT over the first min(2, l+1) primes */
void ck_decrypt_coef(const ck_ctx* ck, const uint64_t* ct, int level, double* coef) {
    const size_t N = ck->N;
    const int nr = level + 1, use = nr < 2 ? nr : 2;
    uint64_t* m = malloc((size_t)use * N * 8);
    for (int t = 0; t < use; t++) {
        const uint64_t q = ck->q[t];
        for (size_t k = 0; k < N; k++)
            m[(size_t)t * N + k] = addm(ct[(size_t)t * N + k],
                                        ck_mulmod(ct[((size_t)nr + t) * N + k], ck->s_ntt[(size_t)t * N + k], q), q);
        ck_ntt_inv(ck, t, m + (size_t)t * N);
    }
    const uint64_t q0 = ck->q[0];
    if (use == 1) {
        for (size_t k = 0; k < N; k++) {
            const uint64_t v = m[k];
            coef[k] = v > q0 / 2 ? -(double)(q0 - v) : (double)v;
        }
    } else {
        const uint64_t q1 = ck->q[1];
        const uint64_t inv = invmod(q0 % q1, q1);
        const u128 Q = (u128)q0 * q1;
        for (size_t k = 0; k < N; k++) {
            const uint64_t x0 = m[k], x1 = m[N + k];
            const uint64_t tq = ck_mulmod(subm(x1, x0 % q1, q1), inv, q1);
            const u128 X = (u128)x0 + (u128)q0 * tq;
            coef[k] = X > Q / 2 ? -(double)(Q - X) : (double)X;
        }
    }
    free(m);
}

void ck_decrypt_decode(const ck_ctx* ck, const uint64_t* ct, int level, double scale, double* z) {
    double* coef = malloc(ck->N * sizeof(double));
    ck_decrypt_coef(ck, ct, level, coef);
    ck_decode(ck, coef, scale, z);
    free(coef);
}

void ck_add(const ck_ctx* ck, const uint64_t* a, const uint64_t* b, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1;
    for (int c = 0; c < 2; c++)
        for (int t = 0; t < nr; t++) {
            const size_t o = ((size_t)c * nr + t) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = addm(a[o + k], b[o + k], ck->q[t]);
        }
}

void ck_mul_plain(const ck_ctx* ck, const uint64_t* ct, const uint64_t* pt, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1;
    for (int c = 0; c < 2; c++)
        for (int t = 0; t < nr; t++) {
            const size_t o = ((size_t)c * nr + t) * N;
            for (size_t k = 0; k < N; k++) out[o + k] = ck_mulmod(ct[o + k], pt[(size_t)t * N + k], ck->q[t]);
        }
}

void ck_add_plain(const ck_ctx* ck, const uint64_t* ct, const uint64_t* pt, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1;
    memcpy(out, ct, (size_t)2 * nr * N * 8);
    for (int t = 0; t < nr; t++)
        for (size_t k = 0; k < N; k++)
            out[(size_t)t * N + k] = addm(ct[(size_t)t * N + k], pt[(size_t)t * N + k], ck->q[t]);
}

/* Rescale: r = centered [c_l]_{q_l}; c'_i = (c_i - r) q_l^-1 */
void ck_rescale(const ck_ctx* ck, const uint64_t* ct, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1, no = level;
    const uint64_t ql = ck->q[level];
    for (int c = 0; c < 2; c++) {
        uint64_t* r = malloc(N * 8);
        memcpy(r, ct + ((size_t)c * nr + level) * N, N * 8);
        ck_ntt_inv(ck, level, r);
#pragma omp parallel for schedule(static)
        for (int t = 0; t < no; t++) {
            const uint64_t q = ck->q[t];
            const uint64_t qinv = invmod(ql % q, q);
            uint64_t* tmp = malloc(N * 8);
            for (size_t k = 0; k < N; k++) {
                const uint64_t v = r[k];
                if (v > (ql - 1) / 2) {
                    const uint64_t m = (ql - v) % q;
                    tmp[k] = m ? q - m : 0;
                } else {
                    tmp[k] = v % q;
                }
            }
            ck_ntt_fwd(ck, t, tmp);
            const uint64_t* src = ct + ((size_t)c * nr + t) * N;
            uint64_t* dst = out + ((size_t)c * no + t) * N;
            for (size_t k = 0; k < N; k++) dst[k] = ck_mulmod(subm(src[k], tmp[k], q), qinv, q);
            free(tmp);
        }
        free(r);
    }
}

/* ------------------------------------------------------------------ */
/* key switching                                   */
/* ------------------------------------------------------------------ */

/* ModUp at level l: digit j = primes J = [j a, min(j a + a, l+1)); rows of J
 * copy the NTT input; other rows of Q_l u P get
 *   FastBConv_J->t(x) = sum_{i in J} [x_i (Q_J/q_i)^-1]_{q_i} (Q_J/q_i) mod t
 * on coefficients, then NTT. The lift is centered: a term with
 * [x_i (Q_J/q_i)^-1]_{q_i} > q_i/2 contributes (v - q_i)(Q_J/q_i), i.e. an
 * extra -Q_J (keeps the digits zero-mean; a [0, q) lift leaves a
 * q/2 * (1 + X + ... ) bias that costs ~1e-6 slot error at N = 2^13). */
void ck_modup(const ck_ctx* ck, const uint64_t* c1, int level, uint64_t* digits) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    uint64_t* coef = malloc((size_t)nr * N * 8);
    memcpy(coef, c1, (size_t)nr * N * 8);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nr; t++) ck_ntt_inv(ck, t, coef + (size_t)t * N);
    for (int j = 0; j < dn; j++) {
        const int lo = j * ck->alpha, hi = lo + ck->alpha < nr ? lo + ck->alpha : nr;
        uint64_t inv[CK_MAXP];
        for (int i = lo; i < hi; i++) {
            uint64_t h = 1;
            for (int i2 = lo; i2 < hi; i2++)
                if (i2 != i) h = ck_mulmod(h, ck->q[i2] % ck->q[i], ck->q[i]);
            inv[i] = invmod(h, ck->q[i]);
        }
        uint64_t* dj = digits + (size_t)j * ne * N;
#pragma omp parallel for schedule(static)
        for (int u = 0; u < ne; u++) {
            uint64_t* row = dj + (size_t)u * N;
            if (u >= lo && u < hi) {
                memcpy(row, c1 + (size_t)u * N, N * 8);
                continue;
            }
            const int pt = ext_prime(ck, level, u);
            const uint64_t t = ck->q[pt];
            uint64_t hat[CK_MAXP];
            uint64_t QJ = 1;
            for (int i = lo; i < hi; i++) {
                uint64_t h = 1;
                for (int i2 = lo; i2 < hi; i2++)
                    if (i2 != i) h = ck_mulmod(h, ck->q[i2] % t, t);
                hat[i] = h;
                QJ = ck_mulmod(QJ, ck->q[i] % t, t);
            }
            for (size_t k = 0; k < N; k++) {
                uint64_t acc = 0;
                for (int i = lo; i < hi; i++) {
                    const uint64_t v = ck_mulmod(coef[(size_t)i * N + k], inv[i], ck->q[i]);
                    acc = addm(acc, ck_mulmod(v % t, hat[i], t), t);
                    /* centered lift: v > q_i/2 stands for v - q_i, i.e. minus Q_J */
                    if (v > (ck->q[i] >> 1)) acc = subm(acc, QJ, t);
                }
                row[k] = acc;
            }
            ck_ntt_fwd(ck, pt, row);
        }
    }
    free(coef);
}

/* acc_c[u][k] = sum_j digits[j][u][perm_g(k)] * key[j][c][row(u)][k] */
void ck_inner_product(const ck_ctx* ck, const uint64_t* digits, int level, const uint64_t* key,
                      uint64_t g, uint64_t* acc0, uint64_t* acc1) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level), np = ck->np;
    const uint64_t mask = 2 * N - 1;
    uint32_t* perm = malloc(N * sizeof(uint32_t));
    for (size_t i = 0; i < N; i++) {
        const uint64_t e = 2 * (uint64_t)ck->brv[i] + 1;
        perm[i] = ck->brv[(((e * g) & mask) - 1) >> 1];
    }
#pragma omp parallel for schedule(static)
    for (int u = 0; u < ne; u++) {
        const int row = ext_prime(ck, level, u);
        const uint64_t q = ck->q[row];
        for (size_t k = 0; k < N; k++) {
            uint64_t a0 = 0, a1 = 0;
            for (int j = 0; j < dn; j++) {
                const uint64_t d = digits[((size_t)j * ne + u) * N + perm[k]];
                a0 = addm(a0, ck_mulmod(d, key[(((size_t)j * 2 + 0) * np + row) * N + k], q), q);
                a1 = addm(a1, ck_mulmod(d, key[(((size_t)j * 2 + 1) * np + row) * N + k], q), q);
            }
            acc0[(size_t)u * N + k] = a0;
            acc1[(size_t)u * N + k] = a1;
        }
    }
    free(perm);
}

/* ModDown: out_i = (x_i - FastBConv_P->q_i([x]_P)) * P^-1 mod q_i, with the
 * same centered lift as ModUp (a term v > p_k/2 contributes -P). */
void ck_moddown(const ck_ctx* ck, const uint64_t* acc, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1, K = ck->K, L = ck->L;
    uint64_t* pc = malloc((size_t)K * N * 8);
    memcpy(pc, acc + (size_t)nr * N, (size_t)K * N * 8);
    uint64_t pinv[CK_MAXP];
    for (int k = 0; k < K; k++) {
        ck_ntt_inv(ck, L + k, pc + (size_t)k * N);
        uint64_t h = 1;
        for (int k2 = 0; k2 < K; k2++)
            if (k2 != k) h = ck_mulmod(h, ck->q[L + k2] % ck->q[L + k], ck->q[L + k]);
        pinv[k] = invmod(h, ck->q[L + k]);
    }
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nr; t++) {
        const uint64_t q = ck->q[t];
        uint64_t hat[CK_MAXP];
        uint64_t P = 1;
        for (int k = 0; k < K; k++) {
            uint64_t h = 1;
            for (int k2 = 0; k2 < K; k2++)
                if (k2 != k) h = ck_mulmod(h, ck->q[L + k2] % q, q);
            hat[k] = h;
            P = ck_mulmod(P, ck->q[L + k] % q, q);
        }
        const uint64_t Pinv = invmod(P, q);
        const uint64_t Pq = P;
        uint64_t* tmp = malloc(N * 8);
        for (size_t i = 0; i < N; i++) {
            uint64_t a = 0;
            for (int k = 0; k < K; k++) {
                const uint64_t v = ck_mulmod(pc[(size_t)k * N + i], pinv[k], ck->q[L + k]);
                a = addm(a, ck_mulmod(v % q, hat[k], q), q);
                if (v > (ck->q[L + k] >> 1)) a = subm(a, Pq, q); /* centered lift */
            }
            tmp[i] = a;
        }
        ck_ntt_fwd(ck, t, tmp);
        for (size_t i = 0; i < N; i++)
            out[(size_t)t * N + i] = ck_mulmod(subm(acc[(size_t)t * N + i], tmp[i], q), Pinv, q);
        free(tmp);
    }
    free(pc);
}

/* rotation of ct by galois g given the ModUp digits of ct.c1 */
static void rotate_from_digits(const ck_ctx* ck, const uint64_t* ct, const uint64_t* digits, int level,
                               const uint64_t* key, uint64_t g, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K;
    uint64_t* a0 = malloc((size_t)ne * N * 8);
    uint64_t* a1 = malloc((size_t)ne * N * 8);
    ck_inner_product(ck, digits, level, key, g, a0, a1);
    uint64_t* m0 = malloc((size_t)nr * N * 8);
    ck_moddown(ck, a0, level, m0);
    ck_moddown(ck, a1, level, out + (size_t)nr * N);
    for (int t = 0; t < nr; t++) {
        uint64_t* row = out + (size_t)t * N;
        ck_automorph_ntt(ck, ct + (size_t)t * N, row, g);
        for (size_t k = 0; k < N; k++) row[k] = addm(row[k], m0[(size_t)t * N + k], ck->q[t]);
    }
    free(a0);
    free(a1);
    free(m0);
}

static size_t key_words(const ck_ctx* ck) { return (size_t)ck->dnum * 2 * ck->np * ck->N; }

void ck_rotate_hoisted(const ck_ctx* ck, const uint64_t* ct, int level, const long* ks, int n,
                       uint64_t* outs) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K;
    const size_t ctw = (size_t)2 * nr * N;
    uint64_t* digits = malloc((size_t)ck_dnum_at(ck, level) * ne * N * 8);
    ck_modup(ck, ct + (size_t)nr * N, level, digits);
    uint64_t* key = malloc(key_words(ck) * 8);
    for (int i = 0; i < n; i++) {
        const uint64_t g = ck_galois_elt(ck, ks[i]);
        if (g == 1) {
            memcpy(outs + (size_t)i * ctw, ct, ctw * 8);
            continue;
        }
        ck_galois_key(ck, g, key);
        rotate_from_digits(ck, ct, digits, level, key, g, outs + (size_t)i * ctw);
    }
    free(key);
    free(digits);
}

void ck_rotate(const ck_ctx* ck, const uint64_t* ct, int level, long k, uint64_t* out) {
    ck_rotate_hoisted(ck, ct, level, &k, 1, out);
}

/* Relinearised product (reference Engine::mul_ct, emu.cpp:69-80): tensor
 * (d0, d1, d2) = (a0 b0, a0 b1 + a1 b0, a1 b1), key-switch d2 with the s^2 key,
 * add, rescale. a, b at `level`; out at level - 1. */
void ck_mul_ct(const ck_ctx* ck, const uint64_t* a, const uint64_t* b, int level, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K;
    const size_t pw = (size_t)nr * N;
    uint64_t* d = malloc(3 * pw * 8);
    for (int t = 0; t < nr; t++) {
        const uint64_t q = ck->q[t];
        for (size_t k = 0; k < N; k++) {
            const size_t i = (size_t)t * N + k;
            const uint64_t a0 = a[i], a1 = a[pw + i], b0 = b[i], b1 = b[pw + i];
            d[i] = ck_mulmod(a0, b0, q);
            d[pw + i] = addm(ck_mulmod(a0, b1, q), ck_mulmod(a1, b0, q), q);
            d[2 * pw + i] = ck_mulmod(a1, b1, q);
        }
    }
    uint64_t* digits = malloc((size_t)ck_dnum_at(ck, level) * ne * N * 8);
    ck_modup(ck, d + 2 * pw, level, digits);
    uint64_t* key = malloc(key_words(ck) * 8);
    ck_galois_key(ck, 0, key);
    uint64_t* a0 = malloc((size_t)ne * N * 8);
    uint64_t* a1 = malloc((size_t)ne * N * 8);
    ck_inner_product(ck, digits, level, key, 1, a0, a1);
    uint64_t* sum = malloc(2 * pw * 8);
    ck_moddown(ck, a0, level, sum);
    ck_moddown(ck, a1, level, sum + pw);
    for (int t = 0; t < nr; t++)
        for (size_t k = 0; k < N; k++)
            for (int p = 0; p < 2; p++) {
                const size_t i = p * pw + (size_t)t * N + k;
                sum[i] = addm(sum[i], d[i], ck->q[t]);
            }
    ck_rescale(ck, sum, level, out);
    free(sum);
    free(a1);
    free(a0);
    free(key);
    free(digits);
    free(d);
}

/* ------------------------------------------------------------------ */
/* fused convolution                                     */
/* ------------------------------------------------------------------ */


static const uint64_t* cache_get(const ck_ctx* ck, key_cache* kc, uint64_t g) {
    for (int i = 0; i < kc->n; i++)
        if (kc->slots[i].g == g) return kc->slots[i].key;
    if (kc->n == kc->cap) {
        kc->cap = kc->cap ? 2 * kc->cap : 64;
        kc->slots = realloc(kc->slots, (size_t)kc->cap * sizeof(key_slot));
    }
    key_slot* s = &kc->slots[kc->n++];
    s->g = g;
    s->key = malloc(key_words(ck) * 8);
    ck_galois_key(ck, g, s->key);
    return s->key;
}
static void kc_reset(key_cache* kc) {
    if (!kc) return;
    for (int i = 0; i < kc->n; i++) free(kc->slots[i].key);
    free(kc->slots);
    kc->slots = NULL;
    kc->n = kc->cap = 0;
}

/* ACC_c[u] += pt[u] * term_c[u], where for a rotated term
 *   term_0 = ip0 + [u <= l] P sigma_g(X.c0),  term_1 = ip1
 * and for the identity term (ip == NULL)
 *   term_c = [u <= l] P X.c   (P == 0 mod p_k, so the P rows get nothing). */
static void conv_accumulate(const ck_ctx* ck, int level, const uint64_t* pt, const uint64_t* X, uint64_t g,
                            const uint64_t* ip0, const uint64_t* ip1, const uint64_t* Pmod, uint64_t* acc0,
                            uint64_t* acc1) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K;
    uint64_t* perm_c0 = NULL;
    if (ip0) {
        perm_c0 = malloc((size_t)nr * N * 8);
        for (int t = 0; t < nr; t++) ck_automorph_ntt(ck, X + (size_t)t * N, perm_c0 + (size_t)t * N, g);
    }
#pragma omp parallel for schedule(static)
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        const size_t o = (size_t)u * N;
        for (size_t k = 0; k < N; k++) {
            uint64_t t0, t1;
            if (ip0) {
                t0 = ip0[o + k];
                t1 = ip1[o + k];
                if (u < nr) t0 = addm(t0, ck_mulmod(Pmod[u], perm_c0[o + k], q), q);
            } else {
                if (u >= nr) continue;
                t0 = ck_mulmod(Pmod[u], X[o + k], q);
                t1 = ck_mulmod(Pmod[u], X[(size_t)nr * N + o + k], q);
            }
            acc0[o + k] = addm(acc0[o + k], ck_mulmod(pt[o + k], t0, q), q);
            acc1[o + k] = addm(acc1[o + k], ck_mulmod(pt[o + k], t1, q), q);
        }
    }
    free(perm_c0);
}

/* Baby-step / giant-step conv with output aggregation.
 * orient 3: baby steps = channel rotations r m^2 (hoisted from one ModUp of
 *           the input), giant steps = shifts kk m + ll;
 * orient 4: baby steps = shifts, giant steps = channel rotations;
 * orient 5: baby steps = channel rotations combined with column shifts
 *           r m^2 + ll (c kappa of them), giant steps = row shifts kk m
 *           (kappa of them): more (cheap) hoisted baby steps for fewer
 *           giant steps, each of which costs a ModDown + ModUp.
 * With X_b = rot_b(ct) kept in the QP basis (never ModDown'd),
 *   Y_g = sum_b rot_{-g}(pt_{g,b}) * X_b                      (QP accumulators)
 *   out = Rescale(ModDown(Y_0 + sum_{g != 0} KS_g(Y_g)))
 * where KS_g(Y) = (IP_0(ModUp(ModDown(Y.c1)), key_g) + sigma_g(Y.c0), IP_1(...)) in QP. */
static int conv_bsgs(const ck_ctx* ck, const uint64_t* ct, int level, int c, int m, int kappa, int c_out,
                     const double* filt, int orient, uint64_t* out, double* out_scale) {
    const size_t N = ck->N, s = N / 2, block = (size_t)m * m;
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    const long h = kappa / 2;
    const int nk = (int)((2 * h + 1) * (2 * h + 1));
    const size_t extw = (size_t)ne * N, ctw = (size_t)2 * nr * N;
    const uint64_t ql = ck->q[level];
    const double pscale = (double)ql;
    const int kap = (int)(2 * h + 1);
    const int nb = orient == 3 ? c : orient == 4 ? nk : c * kap;
    const int ngi = orient == 3 ? nk : orient == 4 ? c : kap;
    long* bamt = malloc((size_t)nb * sizeof(long));
    long* gamt = malloc((size_t)ngi * sizeof(long));
    if (orient == 5) {
        for (int r = 0; r < c; r++)
            for (long ll = -h; ll <= h; ll++) bamt[r * kap + (ll + h)] = (long)r * (long)block + ll;
        for (long kk = -h; kk <= h; kk++) gamt[kk + h] = kk * m;
    } else {
        for (int r = 0; r < c; r++) (orient == 3 ? bamt : gamt)[r] = (long)r * (long)block;
        int i = 0;
        for (long kk = -h; kk <= h; kk++)
            for (long ll = -h; ll <= h; ll++, i++) (orient == 3 ? gamt : bamt)[i] = kk * m + ll;
    }
    uint64_t Pmod[CK_MAXP];
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[ck->L + k] % q, q);
        Pmod[u] = u < nr ? P : 0;
    }
    /* rotated plaintexts pt'[g][b] = rot_{-g}(fused_plain(r, i)) */
    uint64_t* pts = malloc((size_t)ngi * nb * extw * 8);
    int* nonempty = calloc((size_t)ngi * nb, sizeof(int));
    double* plain = malloc(s * sizeof(double));
    double* rplain = malloc(s * sizeof(double));
    for (int gi = 0; gi < ngi; gi++)
        for (int bi = 0; bi < nb; bi++) {
            int r;
            long kk, ll;
            if (orient == 5) {
                r = bi / kap;
                ll = bi % kap - h;
                kk = gi - h;
            } else {
                r = orient == 3 ? bi : gi;
                const int i = orient == 3 ? gi : bi;
                kk = i / kap - h;
                ll = i % kap - h;
            }
            if (!emu_fused_plain(c, m, kappa, c_out, s, filt, r, kk, ll, 1.0, plain)) continue;
            nonempty[gi * nb + bi] = 1;
            emu_rotate(plain, rplain, s, -gamt[gi]);
            ck_encode_plain(ck, rplain, s, pscale, level, 1, pts + ((size_t)gi * nb + bi) * extw);
        }
    free(plain);
    free(rplain);
    key_cache* kcp = ck->kc;
    uint64_t* dsrc = malloc((size_t)dn * extw * 8);
    uint64_t* ip0 = malloc(extw * 8);
    uint64_t* ip1 = malloc(extw * 8);
    uint64_t* Y = calloc((size_t)ngi * 2 * extw, 8); /* [g][2][ne][N] */
    ck_modup(ck, ct + (size_t)nr * N, level, dsrc);
    for (int bi = 0; bi < nb; bi++) {
        int any = 0;
        for (int gi = 0; gi < ngi; gi++) any |= nonempty[gi * nb + bi];
        if (!any) continue;
        const uint64_t g = ck_galois_elt(ck, bamt[bi]);
        if (g != 1) ck_inner_product(ck, dsrc, level, cache_get(ck, kcp, g), g, ip0, ip1);
        for (int gi = 0; gi < ngi; gi++) {
            if (!nonempty[gi * nb + bi]) continue;
            const uint64_t* pt = pts + ((size_t)gi * nb + bi) * extw;
            uint64_t* y = Y + (size_t)gi * 2 * extw;
            if (g == 1)
                conv_accumulate(ck, level, pt, ct, 1, NULL, NULL, Pmod, y, y + extw);
            else
                conv_accumulate(ck, level, pt, ct, g, ip0, ip1, Pmod, y, y + extw);
        }
    }
    uint64_t* acc0 = calloc(extw, 8);
    uint64_t* acc1 = calloc(extw, 8);
    uint64_t* yq = malloc(ctw * 8);
    uint64_t* perm = malloc(extw * 8);
    for (int gi = 0; gi < ngi; gi++) {
        int any = 0;
        for (int bi = 0; bi < nb; bi++) any |= nonempty[gi * nb + bi];
        if (!any) continue;
        const uint64_t* y = Y + (size_t)gi * 2 * extw;
        const uint64_t g = ck_galois_elt(ck, gamt[gi]);
        if (g == 1) {
            for (int u = 0; u < ne; u++) {
                const uint64_t q = ck->q[ext_prime(ck, level, u)];
                for (size_t k = 0; k < N; k++) {
                    acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], y[(size_t)u * N + k], q);
                    acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], y[extw + (size_t)u * N + k], q);
                }
            }
            continue;
        }
        /* only Y.c1 is brought down to Q for the decomposition; Y.c0 is already
         * P-scaled in the QP basis and enters the accumulator directly (the final
         * ModDown performs its rounding), saving a ModDown per giant step */
        ck_moddown(ck, y + extw, level, yq + (size_t)nr * N);
        ck_modup(ck, yq + (size_t)nr * N, level, dsrc);
        ck_inner_product(ck, dsrc, level, cache_get(ck, kcp, g), g, ip0, ip1);
        for (int t = 0; t < ne; t++) ck_automorph_ntt(ck, y + (size_t)t * N, perm + (size_t)t * N, g);
        for (int u = 0; u < ne; u++) {
            const uint64_t q = ck->q[ext_prime(ck, level, u)];
            for (size_t k = 0; k < N; k++) {
                const uint64_t t0 = addm(ip0[(size_t)u * N + k], perm[(size_t)u * N + k], q);
                acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], t0, q);
                acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], ip1[(size_t)u * N + k], q);
            }
        }
    }
    uint64_t* md = malloc(ctw * 8);
    ck_moddown(ck, acc0, level, md);
    ck_moddown(ck, acc1, level, md + (size_t)nr * N);
    ck_rescale(ck, md, level, out);
    if (out_scale) *out_scale = (ck->scale * pscale) / (double)ql;
    free(md);
    free(acc0);
    free(acc1);
    free(yq);
    free(perm);
    free(Y);
    free(dsrc);
    free(ip0);
    free(ip1);
    free(pts);
    free(nonempty);
    free(bamt);
    free(gamt);
    return 0;
}

/* Multi-shard image-mode conv (slots as conv_image_shards,
 * conv.cpp:146-199 with t input shards, n_out output shards) through the
 * fused BSGS schedule: for output shard v,
 *   Y_{v,kk} = sum_u sum_(r, ll) rot_{-kk m}(pt(v, u, r, kk, ll)) * X~_{u, r m^2 + ll},
 *   out_v    = Rescale(ModDown(Y_{v,0} + sum_{kk != 0} KS_{kk m}(Y_{v,kk}))),
 * X~ the QP-basis key switch of input shard u (P sigma(c0) folded in), the
 * giant steps as in conv_bsgs. cts = [t][2][level+1][N], outs = [n_out][2][level][N]. */
int ck_conv_shards(const ck_ctx* ck, const uint64_t* cts, int t, int level, int c, int m, int kappa, int c_out,
                   const double* filt, uint64_t* outs, double* out_scale) {
    return ck_conv_packed(ck, cts, t, level, c, m, kappa, c_out, filt, NULL, 1, 1, outs, out_scale);
}

/* image-mode conv over a PackedImage (tau, rep, duplication d; conv_image_mode
 * conv.cpp:40-211): babies r rep m^2 + ll of input shard u (r < c for one shard,
 * < z otherwise), giants kk m, the fused BSGS of ck_conv_shards. */
int ck_conv_packed(const ck_ctx* ck, const uint64_t* cts, int t, int level, int c, int m, int kappa, int c_out,
                   const double* filt, const long* tau, int rep, int d, uint64_t* outs, double* out_scale) {
    const size_t N = ck->N, s = N / 2, block = (size_t)m * m;
    if (s % block || (size_t)c * block * (size_t)d != (size_t)t * s || level < 1 || rep < 1 || d < 1) return -1;
    if (t >= 2 && d != 1) return -1;
    const size_t z = s / block;
    const size_t rmax = t == 1 ? (size_t)c : z;
    const int n_out = (size_t)c_out <= z ? 1 : (int)((size_t)c_out / z);
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    const long h = kappa / 2;
    const int kap = (int)(2 * h + 1);
    const size_t extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, octw = (size_t)2 * level * N;
    const uint64_t ql = ck->q[level];
    uint64_t Pmod[CK_MAXP];
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[ck->L + k] % q, q);
        Pmod[u] = u < nr ? P : 0;
    }
    key_cache* kcp = ck->kc;
    uint64_t* dsrc = malloc((size_t)t * dn * extw * 8);
    for (int u = 0; u < t; u++)
        ck_modup(ck, cts + (size_t)u * ctw + (size_t)nr * N, level, dsrc + (size_t)u * dn * extw);
    uint64_t* ip0 = malloc(extw * 8);
    uint64_t* ip1 = malloc(extw * 8);
    uint64_t* Y = calloc((size_t)n_out * kap * 2 * extw, 8); /* [v][kk][2][ne][N] */
    int* nonempty_g = calloc((size_t)n_out * kap, sizeof(int));
    double* plain = malloc(s * sizeof(double));
    double* rplain = malloc(s * sizeof(double));
    uint64_t* pt = malloc(extw * 8);
    for (int u = 0; u < t; u++)
        for (size_t r = 0; r < rmax; r++)
            for (long ll = -h; ll <= h; ll++) {
                const long bamt = (long)(r * (size_t)rep * block) + ll;
                const uint64_t g = ck_galois_elt(ck, bamt);
                int have_ip = 0;
                for (int v = 0; v < n_out; v++)
                    for (long kk = -h; kk <= h; kk++) {
                        if (!emu_fused_plain_packed(c, m, kappa, c_out, s, filt, tau, rep, v, u, (int)r, kk, ll, 1.0,
                                                    plain))
                            continue;
                        if (g != 1 && !have_ip) {
                            ck_inner_product(ck, dsrc + (size_t)u * dn * extw, level, cache_get(ck, kcp, g), g, ip0,
                                             ip1);
                            have_ip = 1;
                        }
                        emu_rotate(plain, rplain, s, -kk * m);
                        ck_encode_plain(ck, rplain, s, (double)ql, level, 1, pt);
                        uint64_t* y = Y + ((size_t)v * kap + (size_t)(kk + h)) * 2 * extw;
                        nonempty_g[v * kap + (kk + h)] = 1;
                        if (g == 1)
                            conv_accumulate(ck, level, pt, cts + (size_t)u * ctw, 1, NULL, NULL, Pmod, y, y + extw);
                        else
                            conv_accumulate(ck, level, pt, cts + (size_t)u * ctw, g, ip0, ip1, Pmod, y, y + extw);
                    }
            }
    free(plain);
    free(rplain);
    free(pt);
    uint64_t* acc0 = malloc(extw * 8);
    uint64_t* acc1 = malloc(extw * 8);
    uint64_t* yq = malloc(ctw * 8);
    uint64_t* perm = malloc(extw * 8);
    uint64_t* dg = malloc((size_t)dn * extw * 8);
    uint64_t* md = malloc(ctw * 8);
    for (int v = 0; v < n_out; v++) {
        memset(acc0, 0, extw * 8);
        memset(acc1, 0, extw * 8);
        for (long kk = -h; kk <= h; kk++) {
            if (!nonempty_g[v * kap + (kk + h)]) continue;
            const uint64_t* y = Y + ((size_t)v * kap + (size_t)(kk + h)) * 2 * extw;
            const uint64_t g = ck_galois_elt(ck, kk * m);
            if (g == 1) {
                for (int u = 0; u < ne; u++) {
                    const uint64_t q = ck->q[ext_prime(ck, level, u)];
                    for (size_t k = 0; k < N; k++) {
                        acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], y[(size_t)u * N + k], q);
                        acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], y[extw + (size_t)u * N + k], q);
                    }
                }
                continue;
            }
            ck_moddown(ck, y + extw, level, yq + (size_t)nr * N);
            ck_modup(ck, yq + (size_t)nr * N, level, dg);
            ck_inner_product(ck, dg, level, cache_get(ck, kcp, g), g, ip0, ip1);
            for (int u = 0; u < ne; u++) ck_automorph_ntt(ck, y + (size_t)u * N, perm + (size_t)u * N, g);
            for (int u = 0; u < ne; u++) {
                const uint64_t q = ck->q[ext_prime(ck, level, u)];
                for (size_t k = 0; k < N; k++) {
                    const uint64_t t0 = addm(ip0[(size_t)u * N + k], perm[(size_t)u * N + k], q);
                    acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], t0, q);
                    acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], ip1[(size_t)u * N + k], q);
                }
            }
        }
        ck_moddown(ck, acc0, level, md);
        ck_moddown(ck, acc1, level, md + (size_t)nr * N);
        ck_rescale(ck, md, level, outs + (size_t)v * octw);
    }
    if (out_scale) *out_scale = (ck->scale * (double)ql) / (double)ql;
    free(dsrc); free(ip0); free(ip1); free(Y); free(nonempty_g);
    free(acc0); free(acc1); free(yq); free(perm); free(dg); free(md);
    return n_out;
}

/* Channel-shard mode conv (slots as conv_channel_shards,
 * conv.cpp:273-362): m^2 > s, pc = m^2 / s shards per channel, rows = s / m.
 * Fused BSGS per output shard (g, v): babies = column shifts ll of input
 * shard (f, src), src in {v, v + sign(kk)}; giants = row shifts kk m:
 *   Y_kk = sum_f sum_ll [ rot_{-kk m}(w mask_in(kk, ll)) * X~_{(f, v), ll}
 *                       + rot_{-kk m}(w mask_spill(kk, ll)) * X~_{(f, v + sign kk), ll} ],
 *   out  = Rescale(ModDown(Y_0 + sum_{kk != 0} KS_{kk m}(Y_kk))).
 * cts = [c][pc][2][level+1][N], outs = [c_out][pc][2][level][N]. */
static int cs_mask(int m, long rows, long kk, long ll, int spill, double w, size_t s, double* mask) {
    const long j_lo = ll < 0 ? -ll : 0, j_hi = ll > 0 ? m - ll : m;
    for (size_t i = 0; i < s; i++) mask[i] = 0.0;
    if (j_lo >= j_hi) return 0;
    int any = 0;
    for (long rr = 0; rr < rows; rr++) {
        const int inside = rr + kk >= 0 && rr + kk < rows;
        if (inside == spill) continue;
        any = 1;
        for (long j = j_lo; j < j_hi; j++) mask[(size_t)(rr * m + j)] = w;
    }
    return any;
}

int ck_conv_channel(const ck_ctx* ck, const uint64_t* cts, int level, int c, int m, int kappa, int c_out,
                    const double* filt, uint64_t* outs, double* out_scale) {
    const size_t N = ck->N, s = N / 2, block = (size_t)m * m;
    if (block <= s || block % s || s % (size_t)m || level < 1) return -1;
    const size_t pc = block / s;
    const long rows = (long)(s / (size_t)m);
    const long h = kappa / 2;
    if (h > rows) return -1;
    const int kap = (int)(2 * h + 1);
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    const size_t extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, octw = (size_t)2 * level * N;
    const uint64_t ql = ck->q[level];
    const size_t nsh = (size_t)c * pc;
    uint64_t Pmod[CK_MAXP];
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[ck->L + k] % q, q);
        Pmod[u] = u < nr ? P : 0;
    }
    key_cache* kcp = ck->kc;
    uint64_t* dsrc = malloc(nsh * dn * extw * 8);
    for (size_t sh = 0; sh < nsh; sh++) ck_modup(ck, cts + sh * ctw + (size_t)nr * N, level, dsrc + sh * dn * extw);
    /* inner products of every (shard, ll != 0), computed once */
    uint64_t* ips = malloc(nsh * kap * 2 * extw * 8);
    for (size_t sh = 0; sh < nsh; sh++)
        for (long ll = -h; ll <= h; ll++) {
            if (ll == 0) continue;
            const uint64_t g = ck_galois_elt(ck, ll);
            uint64_t* ip = ips + (sh * kap + (size_t)(ll + h)) * 2 * extw;
            ck_inner_product(ck, dsrc + sh * dn * extw, level, cache_get(ck, kcp, g), g, ip, ip + extw);
        }
    double* mask = malloc(s * sizeof(double));
    double* rmask = malloc(s * sizeof(double));
    uint64_t* pt = malloc(extw * 8);
    uint64_t* Y = malloc((size_t)kap * 2 * extw * 8);
    int* gne = malloc(kap * sizeof(int));
    uint64_t* acc0 = malloc(extw * 8);
    uint64_t* acc1 = malloc(extw * 8);
    uint64_t* yq = malloc(ctw * 8);
    uint64_t* perm = malloc(extw * 8);
    uint64_t* dg = malloc((size_t)dn * extw * 8);
    uint64_t* ip0 = malloc(extw * 8);
    uint64_t* ip1 = malloc(extw * 8);
    uint64_t* md = malloc(ctw * 8);
    for (int g = 0; g < c_out; g++)
        for (size_t v = 0; v < pc; v++) {
            memset(Y, 0, (size_t)kap * 2 * extw * 8);
            for (int i = 0; i < kap; i++) gne[i] = 0;
            for (long kk = -h; kk <= h; kk++) {
                uint64_t* y = Y + (size_t)(kk + h) * 2 * extw;
                for (int f = 0; f < c; f++)
                    for (long ll = -h; ll <= h; ll++) {
                        const double w = emu_filt_centered(filt, c_out, kappa, f, g, kk, ll) * 1.0;
                        if (w == 0.0) continue;
                        for (int spill = 0; spill < 2; spill++) {
                            long src = (long)v;
                            if (spill) {
                                if (kk == 0) continue;
                                src = (long)v + (kk > 0 ? 1 : -1);
                                if (src < 0 || src >= (long)pc) continue;
                            }
                            if (!cs_mask(m, rows, kk, ll, spill, w, s, mask)) continue;
                            emu_rotate(mask, rmask, s, -kk * m);
                            ck_encode_plain(ck, rmask, s, (double)ql, level, 1, pt);
                            const size_t sh = (size_t)f * pc + (size_t)src;
                            gne[kk + h] = 1;
                            if (ll == 0) {
                                conv_accumulate(ck, level, pt, cts + sh * ctw, 1, NULL, NULL, Pmod, y, y + extw);
                            } else {
                                const uint64_t* ip = ips + (sh * kap + (size_t)(ll + h)) * 2 * extw;
                                conv_accumulate(ck, level, pt, cts + sh * ctw, ck_galois_elt(ck, ll), ip, ip + extw,
                                                Pmod, y, y + extw);
                            }
                        }
                    }
            }
            memset(acc0, 0, extw * 8);
            memset(acc1, 0, extw * 8);
            for (long kk = -h; kk <= h; kk++) {
                if (!gne[kk + h]) continue;
                const uint64_t* y = Y + (size_t)(kk + h) * 2 * extw;
                const uint64_t ge = ck_galois_elt(ck, kk * m);
                if (ge == 1) {
                    for (int u = 0; u < ne; u++) {
                        const uint64_t q = ck->q[ext_prime(ck, level, u)];
                        for (size_t k = 0; k < N; k++) {
                            acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], y[(size_t)u * N + k], q);
                            acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], y[extw + (size_t)u * N + k], q);
                        }
                    }
                    continue;
                }
                ck_moddown(ck, y + extw, level, yq + (size_t)nr * N);
                ck_modup(ck, yq + (size_t)nr * N, level, dg);
                ck_inner_product(ck, dg, level, cache_get(ck, kcp, ge), ge, ip0, ip1);
                for (int u = 0; u < ne; u++) ck_automorph_ntt(ck, y + (size_t)u * N, perm + (size_t)u * N, ge);
                for (int u = 0; u < ne; u++) {
                    const uint64_t q = ck->q[ext_prime(ck, level, u)];
                    for (size_t k = 0; k < N; k++) {
                        const uint64_t t0 = addm(ip0[(size_t)u * N + k], perm[(size_t)u * N + k], q);
                        acc0[(size_t)u * N + k] = addm(acc0[(size_t)u * N + k], t0, q);
                        acc1[(size_t)u * N + k] = addm(acc1[(size_t)u * N + k], ip1[(size_t)u * N + k], q);
                    }
                }
            }
            ck_moddown(ck, acc0, level, md);
            ck_moddown(ck, acc1, level, md + (size_t)nr * N);
            ck_rescale(ck, md, level, outs + ((size_t)g * pc + v) * octw);
        }
    if (out_scale) *out_scale = (ck->scale * (double)ql) / (double)ql;
    free(dsrc); free(ips); free(mask); free(rmask); free(pt); free(Y); free(gne);
    free(acc0); free(acc1); free(yq); free(perm); free(dg); free(ip0); free(ip1); free(md);
    return (int)((size_t)c_out * pc);
}

/* Plaintext-weighted sum of hoisted rotations (the linear-transform primitive
 * the pooling stages are built from): out = Rescale(ModDown(sum_b pt_b * X~_b))
 * with X~_b the QP-basis rotation of ct by amounts[b] (P sigma(c0) folded in,
 * identity: P ct) and pt_b encoded over Q_l u P at scale q_l (ck_encode_plain
 * with_p = 1), pts = [n][level+1+K][N]. Equals sum_b pt_b * rot_b(ct) after
 * one rescale. */
/* out = Rescale(ModDown(sum_b pt_b * KS_{amount_b}(ct_{src_b}))): several source
   ciphertexts ([nsrc][2][level+1][N]), each ModUp'd once; every term is
   accumulated in the QP basis before the single ModDown + rescale (the GPU's
   lintrans_batch / channel-shard pooling window with spill terms). */
void ck_lintrans_src(const ck_ctx* ck, const uint64_t* cts, int nsrc, int level, int n, const int* src,
                     const long* amounts, const uint64_t* pts, uint64_t* out) {
    const size_t N = ck->N;
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    const size_t extw = (size_t)ne * N, ctw = (size_t)2 * nr * N;
    uint64_t Pmod[CK_MAXP];
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[ck->L + k] % q, q);
        Pmod[u] = u < nr ? P : 0;
    }
    key_cache* kcp = ck->kc;
    uint64_t* dsrc = malloc((size_t)nsrc * dn * extw * 8);
    for (int j = 0; j < nsrc; j++) ck_modup(ck, cts + (size_t)j * ctw + (size_t)nr * N, level, dsrc + (size_t)j * dn * extw);
    uint64_t* ip0 = malloc(extw * 8);
    uint64_t* ip1 = malloc(extw * 8);
    uint64_t* y = calloc(2 * extw, 8);
    for (int b = 0; b < n; b++) {
        const uint64_t g = ck_galois_elt(ck, amounts[b]);
        const uint64_t* pt = pts + (size_t)b * extw;
        const int j = src ? src[b] : 0;
        const uint64_t* ct = cts + (size_t)j * ctw;
        if (g == 1) {
            conv_accumulate(ck, level, pt, ct, 1, NULL, NULL, Pmod, y, y + extw);
        } else {
            ck_inner_product(ck, dsrc + (size_t)j * dn * extw, level, cache_get(ck, kcp, g), g, ip0, ip1);
            conv_accumulate(ck, level, pt, ct, g, ip0, ip1, Pmod, y, y + extw);
        }
    }
    uint64_t* md = malloc(ctw * 8);
    ck_moddown(ck, y, level, md);
    ck_moddown(ck, y + extw, level, md + (size_t)nr * N);
    ck_rescale(ck, md, level, out);
    free(dsrc); free(ip0); free(ip1); free(y); free(md);
}

void ck_lintrans(const ck_ctx* ck, const uint64_t* ct, int level, int n, const long* amounts, const uint64_t* pts,
                 uint64_t* out) {
    ck_lintrans_src(ck, ct, 1, level, n, NULL, amounts, pts, out);
}

int ck_conv(const ck_ctx* ck, const uint64_t* ct, int level, int c, int m, int kappa, int c_out,
            const double* filt, int plan, uint64_t* out, double* out_scale) {
    const size_t N = ck->N, s = N / 2, block = (size_t)m * m;
    if ((size_t)c * block > s || s % block || (size_t)c_out * block > s || level < 1) return -1;
    if (plan >= 3 && plan <= 5) return conv_bsgs(ck, ct, level, c, m, kappa, c_out, filt, plan, out, out_scale);
    const int nr = level + 1, ne = nr + ck->K, dn = ck_dnum_at(ck, level);
    const long h = kappa / 2;
    const int nk = (int)((2 * h + 1) * (2 * h + 1));
    const size_t ctw = (size_t)2 * nr * N, extw = (size_t)ne * N;
    const uint64_t ql = ck->q[level];
    const double pscale = (double)ql;

    uint64_t Pmod[CK_MAXP];
    for (int u = 0; u < ne; u++) {
        const uint64_t q = ck->q[ext_prime(ck, level, u)];
        uint64_t P = 1;
        for (int k = 0; k < ck->K; k++) P = ck_mulmod(P, ck->q[ck->L + k] % q, q);
        Pmod[u] = u < nr ? P : 0;
    }
    /* plaintexts pt[r][i], QP basis at this level, scale q_l */
    uint64_t* pts = malloc((size_t)c * nk * extw * 8);
    int* nonempty = malloc((size_t)c * nk * sizeof(int));
    double* plain = malloc(s * sizeof(double));
    for (int r = 0; r < c; r++) {
        int i = 0;
        for (long kk = -h; kk <= h; kk++)
            for (long ll = -h; ll <= h; ll++, i++) {
                nonempty[r * nk + i] = emu_fused_plain(c, m, kappa, c_out, s, filt, r, kk, ll, 1.0, plain);
                if (nonempty[r * nk + i])
                    ck_encode_plain(ck, plain, s, pscale, level, 1, pts + ((size_t)r * nk + i) * extw);
            }
    }
    free(plain);

    uint64_t* acc0 = calloc(extw, 8);
    uint64_t* acc1 = calloc(extw, 8);
    uint64_t* dsrc = malloc((size_t)dn * extw * 8);
    uint64_t* dtmp = malloc((size_t)dn * extw * 8);
    uint64_t* X = malloc(ctw * 8);
    uint64_t* ip0 = malloc(extw * 8);
    uint64_t* ip1 = malloc(extw * 8);
    key_cache* kcp = ck->kc;
    ck_modup(ck, ct + (size_t)nr * N, level, dsrc);

    if (plan == 2) { /* Approach 2: channel rotations of src (hoisted), then shifts */
        for (int r = 0; r < c; r++) {
            int any = 0;
            for (int i = 0; i < nk; i++) any |= nonempty[r * nk + i];
            if (!any) continue;
            const uint64_t gr = ck_galois_elt(ck, (long)r * (long)block);
            if (gr == 1)
                memcpy(X, ct, ctw * 8);
            else
                rotate_from_digits(ck, ct, dsrc, level, cache_get(ck, kcp, gr), gr, X);
            ck_modup(ck, X + (size_t)nr * N, level, dtmp);
            int i = 0;
            for (long kk = -h; kk <= h; kk++)
                for (long ll = -h; ll <= h; ll++, i++) {
                    if (!nonempty[r * nk + i]) continue;
                    const uint64_t* pt = pts + ((size_t)r * nk + i) * extw;
                    const uint64_t g = ck_galois_elt(ck, kk * m + ll);
                    if (g == 1) {
                        conv_accumulate(ck, level, pt, X, 1, NULL, NULL, Pmod, acc0, acc1);
                    } else {
                        ck_inner_product(ck, dtmp, level, cache_get(ck, kcp, g), g, ip0, ip1);
                        conv_accumulate(ck, level, pt, X, g, ip0, ip1, Pmod, acc0, acc1);
                    }
                }
        }
    } else { /* Approach 1: shifts of src (hoisted), then channel rotations */
        int i = 0;
        for (long kk = -h; kk <= h; kk++)
            for (long ll = -h; ll <= h; ll++, i++) {
                int any = 0;
                for (int r = 0; r < c; r++) any |= nonempty[r * nk + i];
                if (!any) continue;
                const uint64_t gi = ck_galois_elt(ck, kk * m + ll);
                if (gi == 1)
                    memcpy(X, ct, ctw * 8);
                else
                    rotate_from_digits(ck, ct, dsrc, level, cache_get(ck, kcp, gi), gi, X);
                ck_modup(ck, X + (size_t)nr * N, level, dtmp);
                for (int r = 0; r < c; r++) {
                    if (!nonempty[r * nk + i]) continue;
                    const uint64_t* pt = pts + ((size_t)r * nk + i) * extw;
                    const uint64_t g = ck_galois_elt(ck, (long)r * (long)block);
                    if (g == 1) {
                        conv_accumulate(ck, level, pt, X, 1, NULL, NULL, Pmod, acc0, acc1);
                    } else {
                        ck_inner_product(ck, dtmp, level, cache_get(ck, kcp, g), g, ip0, ip1);
                        conv_accumulate(ck, level, pt, X, g, ip0, ip1, Pmod, acc0, acc1);
                    }
                }
            }
    }
    /* one ModDown per component, then one rescale */
    uint64_t* md = malloc(ctw * 8);
    ck_moddown(ck, acc0, level, md);
    ck_moddown(ck, acc1, level, md + (size_t)nr * N);
    ck_rescale(ck, md, level, out);
    if (out_scale) *out_scale = (ck->scale * pscale) / (double)ql;
    free(md);
    free(acc0);
    free(acc1);
    free(dsrc);
    free(dtmp);
    free(X);
    free(ip0);
    free(ip1);
    free(pts);
    free(nonempty);
    return 0;
}
