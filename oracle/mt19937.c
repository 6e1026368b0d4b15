/* TEST INFRASTRUCTURE ONLY — part of the oracle (checker), never shipped.
 *
 * Restatement of the input generator the reference's tests use
 * (reference tests/helpers.hpp:13-27): std::mt19937_64 (the published
 * MT19937-64 algorithm, Matsumoto & Nishimura) feeding libstdc++'s
 * uniform_real_distribution / normal_distribution. Restated here so the
 * GPU box (which has no /root/reference) can regenerate the exact inputs
 * of the golden fixtures; pinned against the compiled reference by
 * tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "emu_ref.h"

#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void mt64_seed(mt64_state* st, uint64_t seed) {
    st->mt[0] = seed;
    for (int i = 1; i < MT_NN; i++)
        st->mt[i] = 6364136223846793005ULL * (st->mt[i - 1] ^ (st->mt[i - 1] >> 62)) + (uint64_t)i;
    st->mti = MT_NN;
    st->have_saved = 0;
    st->saved = 0.0;
}

uint64_t mt64_next(mt64_state* st) {
    static const uint64_t mag01[2] = {0ULL, MT_MATRIX_A};
    uint64_t x;
    if (st->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; i++) {
            x = (st->mt[i] & MT_UM) | (st->mt[i + 1] & MT_LM);
            st->mt[i] = st->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < MT_NN - 1; i++) {
            x = (st->mt[i] & MT_UM) | (st->mt[i + 1] & MT_LM);
            st->mt[i] = st->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (st->mt[MT_NN - 1] & MT_UM) | (st->mt[0] & MT_LM);
        st->mt[MT_NN - 1] = st->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        st->mti = 0;
    }
    x = st->mt[st->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* libstdc++ generate_canonical<double, 53> over a 64-bit engine: one draw,
 * converted to double and divided by 2^64, clamped below 1. */
double mt64_canonical(mt64_state* st) {
    double r = (double)mt64_next(st) * 0x1p-64;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}

/* uniform_real_distribution<double>(a, b): (b - a) * canonical + a */
double mt64_uniform(mt64_state* st, double a, double b) {
    return (b - a) * mt64_canonical(st) + a;
}

/* normal_distribution<double>(mean, stddev): Marsaglia polar method with
 * one cached deviate, as libstdc++ implements it. */
double mt64_normal(mt64_state* st, double mean, double stddev) {
    double ret;
    if (st->have_saved) {
        st->have_saved = 0;
        ret = st->saved;
    } else {
        double x, y, r2;
        do {
            x = 2.0 * mt64_canonical(st) - 1.0;
            y = 2.0 * mt64_canonical(st) - 1.0;
            r2 = x * x + y * y;
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(-2.0 * log(r2) / r2);
        st->saved = x * mult;
        st->have_saved = 1;
        ret = y * mult;
    }
    return ret * stddev + mean;
}

/* random_tensor / random_filter (reference tests/helpers.hpp:13-27) and the
 * two extra weight laws of BASELINE cfg4 / cfg5. weight_kind: 0 U[-1,1],
 * 1 U[-0.5,0.5], 2 N(0, 0.1^2) clipped to [-1, 1]. */
void emu_make_inputs(int c, int m, int kappa, int c_out, uint64_t seed_img, uint64_t seed_filt,
                     int weight_kind, double* img, double* filt) {
    mt64_state st;
    mt64_seed(&st, seed_img);
    const size_t ni = (size_t)c * m * m;
    for (size_t i = 0; i < ni; i++) img[i] = mt64_uniform(&st, -1.0, 1.0);
    mt64_seed(&st, seed_filt);
    const size_t nf = (size_t)c * c_out * kappa * kappa;
    for (size_t i = 0; i < nf; i++) {
        if (weight_kind == 0) {
            filt[i] = mt64_uniform(&st, -1.0, 1.0);
        } else if (weight_kind == 1) {
            filt[i] = mt64_uniform(&st, -0.5, 0.5);
        } else {
            double v = mt64_normal(&st, 0.0, 0.1);
            filt[i] = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
        }
    }
}
