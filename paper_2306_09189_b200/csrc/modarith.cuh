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

namespace fhe {

struct Prime {
    uint64_t q;
    uint64_t bar_hi;  // floor(2^128 / q) high word
    uint64_t bar_lo;  // floor(2^128 / q) low word
    uint64_t pad;
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
