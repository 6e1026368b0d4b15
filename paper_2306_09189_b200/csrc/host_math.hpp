// Host-side number theory and the canonical-embedding encoder.
//
// These are the product's own implementations of the conventions in
// DESIGN.md §3.2 (primes), §3.3 (NTT roots and twiddle order) and §3.9
// (encoding). They must agree bit-for-bit with the CPU golden model
// (oracle/ckks_ref.c); the encoder therefore performs exactly the same
// double operations in the same order and is compiled with
// -ffp-contract=off (see build.py).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace fhe {
namespace host {

using u128 = unsigned __int128;

inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) { return (uint64_t)(((u128)a * b) % q); }

inline uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
inline uint64_t invmod(uint64_t a, uint64_t q) { return powmod(a % q, q - 2, q); }
inline uint64_t shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

inline bool is_prime(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t b : bases) {
        if (n == b) return true;
        if (n % b == 0) return false;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) {
        d >>= 1;
        ++s;
    }
    for (uint64_t b : bases) {
        uint64_t x = powmod(b, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int r = 1; r < s; ++r) {
            x = mulmod(x, x, n);
            if (x == n - 1) {
                composite = false;
                break;
            }
        }
        if (composite) return false;
    }
    return true;
}

// §3.2: largest q < 2^bits, q = 1 mod 2N, prime, not yet used (bit sizes
// consumed in order q_0..q_{L-1}, p_0..p_{K-1}).
inline std::vector<uint64_t> generate_primes(const std::vector<int>& bits, uint64_t N) {
    std::vector<uint64_t> out;
    const uint64_t twoN = 2 * N;
    for (int b : bits) {
        if (b < 20 || b > 60) throw std::invalid_argument("prime bit size must be in [20, 60]");
        uint64_t c = (((1ULL << b) - 2) / twoN) * twoN + 1;
        for (;; c -= twoN) {
            bool dup = false;
            for (uint64_t u : out) dup |= (u == c);
            if (!dup && is_prime(c)) break;
        }
        out.push_back(c);
    }
    return out;
}

// §3.3: psi = g^((q-1)/2N) for the first g = 2, 3, ... with psi^N = -1.
inline uint64_t find_root(uint64_t q, uint64_t N) {
    for (uint64_t g = 2;; ++g) {
        const uint64_t psi = powmod(g, (q - 1) / (2 * N), q);
        if (powmod(psi, N, q) == q - 1) return psi;
    }
}

inline uint32_t bitrev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; ++i) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

// ------------------------------------------------------------- encoder §3.9
constexpr double kPi = 3.14159265358979323846;

struct Cplx {
    double re, im;
};
inline Cplx cmul(Cplx a, Cplx b) {
    Cplx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

// a[k] <- sum_l a[l] exp(sign 2 pi i k l / n); iterative radix-2 DIT.
inline void fft_dit(std::vector<Cplx>& a, int sign) {
    const size_t n = a.size();
    int logn = 0;
    while (((size_t)1 << logn) < n) ++logn;
    for (size_t i = 0; i < n; ++i) {
        const size_t j = bitrev((uint32_t)i, logn);
        if (j > i) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len >> 1, step = n / len;
        for (size_t i = 0; i < n; i += len) {
            for (size_t j = 0; j < half; ++j) {
                const double ang = (2.0 * kPi * (double)(j * step)) / (double)n;
                Cplx w;
                w.re = std::cos(ang);
                w.im = sign > 0 ? std::sin(ang) : -std::sin(ang);
                const Cplx u = a[i + j];
                const Cplx v = cmul(a[i + j + half], w);
                a[i + j].re = u.re + v.re;
                a[i + j].im = u.im + v.im;
                a[i + j + half].re = u.re - v.re;
                a[i + j + half].im = u.im - v.im;
            }
        }
    }
}

// slots z_j <-> m(zeta^(5^j)), zeta = exp(2 pi i / 2N); coefficients are
// round(Delta * m_l), rounding half away from zero.
inline void encode(const double* z, size_t nz, size_t N, double scale, int64_t* coef) {
    const size_t n = N / 2, M = 2 * N;
    if (nz > n) throw std::invalid_argument("slot count mismatch");
    std::vector<Cplx> w(n, Cplx{0.0, 0.0});
    uint64_t g = 1;
    for (size_t j = 0; j < n; ++j) {
        if (j < nz) w[(g - 1) >> 2].re = z[j];
        g = (g * 5) & (M - 1);
    }
    fft_dit(w, -1);
    for (size_t l = 0; l < n; ++l) {
        Cplx v;
        v.re = w[l].re / (double)n;
        v.im = w[l].im / (double)n;
        const double ang = (2.0 * kPi * (double)l) / (double)M;
        Cplx zi;
        zi.re = std::cos(ang);
        zi.im = -std::sin(ang);
        const Cplx u = cmul(v, zi);
        const double a = std::round(u.re * scale), b = std::round(u.im * scale);
        if (std::fabs(a) >= 0x1p62 || std::fabs(b) >= 0x1p62)
            throw std::overflow_error("encoded coefficient exceeds 2^62");
        coef[l] = (int64_t)a;
        coef[l + n] = (int64_t)b;
    }
}

inline void decode(const double* coef, size_t N, double scale, double* z, size_t nz) {
    const size_t n = N / 2, M = 2 * N;
    std::vector<Cplx> v(n);
    for (size_t l = 0; l < n; ++l) {
        Cplx u;
        u.re = coef[l] / scale;
        u.im = coef[l + n] / scale;
        const double ang = (2.0 * kPi * (double)l) / (double)M;
        Cplx zi;
        zi.re = std::cos(ang);
        zi.im = std::sin(ang);
        v[l] = cmul(u, zi);
    }
    fft_dit(v, +1);
    uint64_t g = 1;
    for (size_t j = 0; j < n && j < nz; ++j) {
        z[j] = v[(g - 1) >> 2].re;
        g = (g * 5) & (M - 1);
    }
}

}  // namespace host
}  // namespace fhe
