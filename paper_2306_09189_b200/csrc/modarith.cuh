// Device (and host) 64-bit modular arithmetic for primes q < 2^61.
//
// Conventions: every residue that crosses a kernel boundary
// is normalised into [0, q). Products use either Shoup's precomputed
// quotient (w' = floor(w 2^64 / q), for twiddles and per-prime constants) or
// a 128-bit Barrett reduction with ratio floor(2^128 / q) (for products of
// two data operands). All of these are exact, so any correct evaluation
// order yields the residues the CPU golden model (oracle/ckks_ref.c) does.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define FHE_HD __host__ __device__ __forceinline__
#else
#define FHE_HD inline
#endif

#ifndef FHE_MACSMALL_V2
#define FHE_MACSMALL_V2 1
#endif

namespace fhe {

struct Prime {
    uint64_t q;
    uint64_t bar_hi;  // floor(2^128 / q) high word
    uint64_t bar_lo;  // floor(2^128 / q) low word
    uint64_t qinv;    // -q^-1 mod 2^64 (Montgomery)
};

FHE_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

FHE_HD uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
    const uint64_t r = a + b;
    return r >= q ? r - q : r;
}
FHE_HD uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) { return a >= b ? a - b : a + q - b; }

// a * w mod q with wsh = floor(w 2^64 / q); valid for any a < 2^64, w < q.
FHE_HD uint64_t mul_shoup(uint64_t a, uint64_t w, uint64_t wsh, uint64_t q) {
    const uint64_t qh = mulhi64(a, wsh);
    const uint64_t r = a * w - qh * q;
    return r >= q ? r - q : r;
}
// lazy variant: result in [0, 2q)
FHE_HD uint64_t mul_shoup_lazy(uint64_t a, uint64_t w, uint64_t wsh, uint64_t q) {
    return a * w - mulhi64(a, wsh) * q;
}

// Barrett reduction of a 128-bit value x = (hi, lo) < 2^128. The quotient
// estimate is at most 2 below the true quotient, hence two corrections.
FHE_HD uint64_t reduce128(uint64_t hi, uint64_t lo, const Prime& p) {
    const uint64_t c1 = mulhi64(lo, p.bar_lo);
    const uint64_t m_lo = lo * p.bar_hi;
    const uint64_t m_hi = mulhi64(lo, p.bar_hi);
    uint64_t s = m_lo + c1;
    uint64_t t_hi = m_hi + (s < c1);
    const uint64_t n_lo = hi * p.bar_lo;
    const uint64_t n_hi = mulhi64(hi, p.bar_lo);
    const uint64_t s2 = s + n_lo;
    const uint64_t carry2 = n_hi + (s2 < s);
    const uint64_t qhat = hi * p.bar_hi + t_hi + carry2;
    uint64_t r = lo - qhat * p.q;
    r = r >= p.q ? r - p.q : r;
    r = r >= p.q ? r - p.q : r;
    return r;
}

// Montgomery reduction of T = (hi, lo) < q 2^64: T 2^-64 mod q, in [0, 2q).
FHE_HD uint64_t redc_lazy(uint64_t hi, uint64_t lo, const Prime& p) {
    const uint64_t m = lo * p.qinv;
    return hi + mulhi64(m, p.q) + (lo != 0);
}

FHE_HD uint64_t mul_mod(uint64_t a, uint64_t b, const Prime& p) {
    return reduce128(mulhi64(a, b), a * b, p);
}

// reduce a 64-bit value (any) mod q
FHE_HD uint64_t reduce64(uint64_t a, const Prime& p) { return reduce128(0, a, p); }

// 128-bit accumulator
struct U128 {
    uint64_t lo, hi;
};
FHE_HD void mac(U128& acc, uint64_t a, uint64_t b) {
    const uint64_t lo = a * b;
    const uint64_t hi = mulhi64(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo);
}
FHE_HD void add128(U128& acc, uint64_t v) {
    acc.lo += v;
    acc.hi += (acc.lo < v);
}

// Carry-deferred sum of products of operands < 2^60 (every prime is < 2^60):
// with a = a1 2^32 + a0, b = b1 2^32 + b0 (a1, b1 < 2^28)
//   sum a b = s0 + c 2^64 + s1 2^32 + s2 2^64,
// s0 += a0 b0 (carries counted in c), s1 += a0 b1 + a1 b0 (< 2^61 per term),
// s2 += a1 b1 (< 2^56 per term): four 32x32->64 multiply-adds and one 64-bit
// add-with-carry per term instead of a full 128-bit product. s1 cannot
// overflow for up to 8 terms (8 * 2^61 = 2^64), s2 for up to 2^8.
struct Acc3 {
    uint64_t s0, s1, s2;
    uint32_t c;
};
#ifdef __CUDACC__
__device__ __forceinline__ void mac3(Acc3& A, uint64_t a, uint64_t b) {
    const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
    asm("{\n\t.reg .u64 t;\n\t"
        "mul.wide.u32 t, %4, %6;\n\t"
        "add.cc.u64 %0, %0, t;\n\t"
        "addc.u32 %3, %3, 0;\n\t"
        "mad.wide.u32 %1, %4, %7, %1;\n\t"
        "mad.wide.u32 %1, %5, %6, %1;\n\t"
        "mad.wide.u32 %2, %5, %7, %2;\n\t}"
        : "+l"(A.s0), "+l"(A.s1), "+l"(A.s2), "+r"(A.c)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}
// acc += a b for a, b < 2^62 (the middle sum a0 b1 + a1 b0 < 2^63 cannot carry):
// four 32x32->64 products and two 128-bit additions
__device__ __forceinline__ void mac_small(U128& acc, uint64_t a, uint64_t b) {
    const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
#if FHE_MACSMALL_V2
    // product = p00 + (mid << 32) + (p11 << 64) with mid = a0 b1 + a1 b0 + hi32(p00) < 2^63:
    // four wide multiply-adds (p11 straight into the high word) and one 4-word carry chain
    asm("{\n\t.reg .u64 p00, mid, t;\n\t.reg .u32 p0, p1, m0, m1, l0, l1, h0, h1;\n\t"
        "mul.wide.u32 p00, %2, %4;\n\t"
        "mov.b64 {p0, p1}, p00;\n\t"
        "cvt.u64.u32 t, p1;\n\t"
        "mad.wide.u32 mid, %2, %5, t;\n\t"
        "mad.wide.u32 mid, %3, %4, mid;\n\t"
        "mad.wide.u32 %1, %3, %5, %1;\n\t"
        "mov.b64 {m0, m1}, mid;\n\t"
        "mov.b64 {l0, l1}, %0;\n\t"
        "mov.b64 {h0, h1}, %1;\n\t"
        "add.cc.u32 l0, l0, p0;\n\t"
        "addc.cc.u32 l1, l1, m0;\n\t"
        "addc.cc.u32 h0, h0, m1;\n\t"
        "addc.u32 h1, h1, 0;\n\t"
        "mov.b64 %0, {l0, l1};\n\t"
        "mov.b64 %1, {h0, h1};\n\t}"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    return;
#endif
    asm("{\n\t.reg .u64 p00, p11, mid, ml, mh;\n\t"
        "mul.wide.u32 p00, %2, %4;\n\t"
        "mul.wide.u32 mid, %2, %5;\n\t"
        "mad.wide.u32 mid, %3, %4, mid;\n\t"
        "mul.wide.u32 p11, %3, %5;\n\t"
        "shl.b64 ml, mid, 32;\n\t"
        "shr.u64 mh, mid, 32;\n\t"
        "add.cc.u64 p00, p00, ml;\n\t"
        "addc.u64 p11, p11, mh;\n\t"
        "add.cc.u64 %0, %0, p00;\n\t"
        "addc.u64 %1, %1, p11;\n\t}"
        : "+l"(acc.lo), "+l"(acc.hi)
        : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void add3(Acc3& A, uint64_t v) {
    asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+l"(A.s0), "+r"(A.c) : "l"(v));
}
#endif
// (hi, lo) of the accumulated 128-bit value
FHE_HD U128 fold3(const Acc3& A) {
    const uint64_t lo = A.s0 + (A.s1 << 32);
    const uint64_t hi = (uint64_t)A.c + (A.s1 >> 32) + A.s2 + (lo < A.s0);
    return U128{lo, hi};
}

// ------------------------------------------------------------------ operand form
// Operands of the fused baby-step kernel (k_bsgs_tma) are stored in
// an "operand form" chosen per prime:
//  q < 2^50: the centred residue (-q/2, q/2] as an IEEE double (exact): the
//            products run on the FP64 pipe (kernels.cu fmac_d);
//  else:     30-bit limb form, the word (v >> 30) << 32 | (v mod 2^30), whose two
//            32-bit halves feed mad.wide.u32 directly.
FHE_HD uint64_t to_limb(uint64_t v, int w) { return ((v >> w) << 32) | (v & ((1ULL << w) - 1)); }
FHE_HD uint64_t from_limb(uint64_t l, int w) { return ((l >> 32) << w) | (l & 0xffffffffULL); }
FHE_HD bool opf_fp(uint64_t q) { return q < (1ULL << 50); }
FHE_HD uint64_t dbl_bits(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t b;
    __builtin_memcpy(&b, &d, 8);
    return b;
#endif
}
FHE_HD uint64_t to_opf(uint64_t v, uint64_t q) {
    if (opf_fp(q)) return dbl_bits(v > q / 2 ? -(double)(q - v) : (double)v);
    return to_limb(v, 30);
}
#ifdef __CUDACC__
// ------------------------------------------------------------------ FP64 residues
// Exact modular arithmetic on the FP64 pipe for primes q < 2^50:
// residues are integer-valued doubles, and every step below is exact because
// its true result is an integer below 2^53 in magnitude.
//  mulmod_d(x, w_c, w_c/q): t = rint(x w_c / q) by magic-constant rounding
//    (|x w_c / q| < 2^51), (ph, pl) the exact product split in two doubles,
//    r = (ph - t q) + pl; |r| <= 0.625 q for |x| < 2^52 and |w_c| <= q/2.
//  fmac_d(acc, x, y): acc += x y mod q without a per-operand quotient
//    (t = rint(ph / q)); |x y| <= q^2 / 4 adds <= 0.5 q + 2^44 to acc.
//  red_d(x) = x - q rint(x / q): |result| <= 0.5 q + 1 for |x| < 2^53.
struct ArD {
    double q, qinv, qm;  // q, 1/q, 2^52 + q
    uint64_t qi;
};
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr double kTwo52 = 4503599627370496.0;  // 2^52

__device__ __forceinline__ ArD make_ard(uint64_t q) {
    const double qd = (double)q;
    return ArD{qd, __drcp_rn(qd), __dadd_rn(qd, kTwo52), q};
}
__device__ __forceinline__ double red_d(double x, const ArD& a) {
    const double t = __dadd_rn(__fma_rn(x, a.qinv, kMagic), -kMagic);
    return __fma_rn(-t, a.q, x);
}
__device__ __forceinline__ double mulmod_d(double x, double w, double wq, const ArD& a) {
    const double t = __dadd_rn(__fma_rn(x, wq, kMagic), -kMagic);
    const double ph = __dmul_rn(x, w);
    const double pl = __fma_rn(x, w, -ph);
    return __dadd_rn(__fma_rn(-t, a.q, ph), pl);
}
__device__ __forceinline__ void fmac_d(double& acc, double x, double y, const ArD& a) {
    const double ph = __dmul_rn(x, y);
    const double pl = __fma_rn(x, y, -ph);
    const double t = __dadd_rn(__fma_rn(ph, a.qinv, kMagic), -kMagic);
    acc = __dadd_rn(acc, __dadd_rn(__fma_rn(-t, a.q, ph), pl));
}
// Error-free accumulation of an inner product sum_j x_j y_j (|x_j|, |y_j| <= q/2 < 2^49,
// at most 8 terms) with ONE quotient for the whole sum instead of one per product:
//  H starts at 1.5 * 2^102 and stays in [2^102, 2^103) (|sum| < 2^101), so every
//    H' = fma(x, y, H) is the exact x y + H rounded to the grid 2^50 -- H' - H is the
//    product rounded to the grid, exactly;
//  fma(x, y, -(H' - H)) is the exact remainder (an integer, |.| <= 2^49), summed in L
//    (|L| < 2^53 with the caller's initial term <= q + 1).
// 4 FP64 operations per product (fmac_d: 7). fold_d returns the sum mod q:
// M = (H - 1.5 * 2^102) 2^-50 is an integer below 2^51, M [2^50]_q by mulmod_d, plus L,
// one red_d (|result| <= 0.5 q + 1).
constexpr double kGridBig = 0x1.8p+102;
constexpr double kGridInv = 0x1p-50;
struct ArG {
    double c, cq;  // centred 2^50 mod q, and c / q
};
__device__ __forceinline__ ArG make_arg(const ArD& a) {
    const uint64_t r = (1ULL << 50) % a.qi;
    const double c = r > a.qi / 2 ? -(double)(a.qi - r) : (double)r;
    return ArG{c, __ddiv_rn(c, a.q)};
}
__device__ __forceinline__ void fmag_d(double& H, double& L, double x, double y) {
    const double Hn = __fma_rn(x, y, H);
    L = __dadd_rn(L, __fma_rn(x, y, __dadd_rn(H, -Hn)));
    H = Hn;
}
__device__ __forceinline__ double fold_d(double H, double L, const ArD& a, const ArG& g) {
    const double M = __dmul_rn(__dadd_rn(H, -kGridBig), kGridInv);
    return red_d(__dadd_rn(mulmod_d(M, g.c, g.cq, a), L), a);
}
// canonical word in [0, q) -> bits of the same value as a double (exact)
__device__ __forceinline__ uint64_t u2d_bits(uint64_t x) {
    return (uint64_t)__double_as_longlong(
        __dadd_rn(__longlong_as_double((long long)(x | 0x4330000000000000ULL)), -kTwo52));
}
// |x| <= 0.625 q -> canonical word in [0, q)
__device__ __forceinline__ uint64_t canon_d(double x, const ArD& a) {
    const uint64_t u = (uint64_t)__double_as_longlong(__dadd_rn(x, a.qm)) - 0x4330000000000000ULL;  // x + q
    return u >= a.qi ? u - a.qi : u;
}
__device__ __forceinline__ double asd(uint64_t b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ uint64_t asu(double d) { return (uint64_t)__double_as_longlong(d); }
#endif

#ifdef __CUDACC__
// acc += a b (one IMAD.WIDE.U32 with a 64-bit addend)
__device__ __forceinline__ void madw(uint64_t& acc, uint32_t a, uint32_t b) {
    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}
#endif

// ------------------------------------------------------------------ PRNG
// Counter-based SplitMix64 hash. Deterministic on host and
// device; benchmark-grade, NOT a cryptographic PRNG.
FHE_HD uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}
FHE_HD uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64(seed ^ mix64(stream + 0x9E3779B97F4A7C15ULL));
}
FHE_HD uint64_t prng_k(uint64_t key, uint64_t ctr) { return mix64(key + ctr * 0xD1B54A32D192ED03ULL); }

enum : uint64_t { DOM_SECRET = 1, DOM_KEY_A = 2, DOM_KEY_E = 3, DOM_ENC_A = 4, DOM_ENC_E = 5 };
FHE_HD uint64_t stream_id(uint64_t dom, uint64_t galois, uint64_t digit) {
    return (dom << 56) | (galois << 8) | digit;
}

// (hi 2^64 + lo) mod q
FHE_HD uint64_t uniform_mod(uint64_t hi, uint64_t lo, const Prime& p) { return reduce128(hi, lo, p); }

// signed 64-bit value -> [0, q)
FHE_HD uint64_t reduce_signed(int64_t x, const Prime& p) {
    if (x >= 0) return reduce64((uint64_t)x, p);
    const uint64_t r = reduce64((uint64_t)(-(x + 1)) + 1, p);
    return r ? p.q - r : 0;
}

}  // namespace fhe
