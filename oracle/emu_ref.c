/* TEST INFRASTRUCTURE ONLY — the oracle (checker); see emu_ref.h.
 *
 * Restates, in plain C, the slot-level conv schedule of the reference
 * (reference proj/src/conv.cpp) and its rotation decompositions
 * (proj/src/rot.cpp). Floating-point operation order follows the reference
 * so outputs are bit-identical; tests/test_oracle_pins.py pins this against
 * the compiled reference (oracle/_ref) and the committed golden fixtures.
 */
#include "emu_ref.h"

#include <stdlib.h>
#include <string.h>

static size_t reduce_mod(long k, size_t s) { /* emu.cpp:9-13 */
    long m = k % (long)s;
    if (m < 0) m += (long)s;
    return (size_t)m;
}

void emu_rotate(const double* in, double* out, size_t s, long k) { /* emu.cpp:15-20 */
    const size_t a = reduce_mod(k, s);
    for (size_t i = 0; i < s; i++) out[i] = in[(i + a) % s];
}

double emu_filt_centered(const double* filt, int c_out, int kappa, int f, int g, long k, long l) {
    /* tensor.hpp:53-67 */
    const long h = kappa / 2;
    return filt[(((size_t)f * c_out + g) * kappa + (size_t)(k + h)) * kappa + (size_t)(l + h)];
}

int emu_fused_plain(int c, int m, int kappa, int c_out, size_t s, const double* filt, int r,
                    long kk, long ll, double scale, double* plain) {
    /* conv.cpp:61-85 with t = 1, n_out = 1, rep = 1, tau = identity:
     *   in_channel(0, r, b) = block_channel((b + r) % z) = ((b + r) % z) % c
     *   out_channel(0, b)   = b % c_out                                   */
    const size_t block = (size_t)m * m;
    const size_t z = s / block;
    int any = 0;
    for (size_t i = 0; i < s; i++) plain[i] = 0.0;
    for (size_t b = 0; b < z; b++) {
        const int in_ch = (int)(((b + (size_t)r) % z) % (size_t)c);
        const int out_ch = (int)(b % (size_t)c_out);
        const double w = emu_filt_centered(filt, c_out, kappa, in_ch, out_ch, kk, ll) * scale;
        if (w == 0.0) continue;
        any = 1;
        const long i_lo = kk < 0 ? -kk : 0, i_hi = kk > 0 ? m - kk : m;
        const long j_lo = ll < 0 ? -ll : 0, j_hi = ll > 0 ? m - ll : m;
        for (long i = i_lo; i < i_hi; i++)
            for (long j = j_lo; j < j_hi; j++) plain[b * block + (size_t)(i * m + j)] = w;
    }
    return any;
}

int emu_conv_slots(int c, int m, int kappa, int c_out, size_t s, const double* img,
                   const double* filt, int plan, double* out) {
    const size_t block = (size_t)m * m;
    if (block * (size_t)c > s || s % block) return -1;
    if ((size_t)c_out * block > s) return -1; /* "insufficient capacity" conv.cpp:269 */
    const long h = kappa / 2;
    const int nk = (int)((2 * h + 1) * (2 * h + 1));
    const size_t z = s / block;
    /* pack(): one shard, channels duplicated d = z / c times (pack.cpp:19-33) */
    double* src = malloc(s * sizeof(double));
    for (size_t i = 0; i < s; i++) src[i] = img[i % (block * (size_t)c)];
    (void)z;
    double* acc = malloc(s * sizeof(double));
    double* partial = malloc(s * sizeof(double));
    double* x = malloc(s * sizeof(double));
    double* y = malloc(s * sizeof(double));
    double* tmp = malloc(s * sizeof(double));
    double* plains = malloc((size_t)nk * s * sizeof(double));
    int* nonempty = malloc((size_t)nk * sizeof(int));
    int have_acc = 0;
    for (int r = 0; r < c; r++) {
        const long chan = (long)r * (long)block;
        int any = 0, idx = 0;
        for (long kk = -h; kk <= h; kk++)
            for (long ll = -h; ll <= h; ll++, idx++) {
                nonempty[idx] = emu_fused_plain(c, m, kappa, c_out, s, filt, r, kk, ll, 1.0,
                                                plains + (size_t)idx * s);
                any |= nonempty[idx];
            }
        if (!any && plan != 1) continue; /* conv.cpp:172 */
        int have_partial = 0;
        if (plan != 1) emu_rotate(src, x, s, chan); /* conv.cpp:168 */
        idx = 0;
        for (long kk = -h; kk <= h; kk++)
            for (long ll = -h; ll <= h; ll++, idx++) {
                if (!nonempty[idx]) continue;
                if (plan == 1) { /* ChannelFirst: shifted copy, then channel rotation (conv.cpp:134-135) */
                    emu_rotate(src, tmp, s, kk * m + ll);
                    emu_rotate(tmp, y, s, chan);
                } else { /* ShiftFirst / default: shift of the channel-rotated copy */
                    emu_rotate(x, y, s, kk * m + ll);
                }
                const double* p = plains + (size_t)idx * s;
                if (!have_partial) { /* Acc::add (conv.cpp:18-23) */
                    for (size_t i = 0; i < s; i++) partial[i] = y[i] * p[i];
                    have_partial = 1;
                } else {
                    for (size_t i = 0; i < s; i++) partial[i] = partial[i] + y[i] * p[i];
                }
            }
        if (!have_partial) continue;
        if (!have_acc) {
            memcpy(acc, partial, s * sizeof(double));
            have_acc = 1;
        } else {
            for (size_t i = 0; i < s; i++) acc[i] = acc[i] + partial[i];
        }
    }
    if (!have_acc) /* Acc::finish zero product (conv.cpp:25-28) */
        for (size_t i = 0; i < s; i++) acc[i] = src[i] * 0.0;
    memcpy(out, acc, s * sizeof(double));
    free(src); free(acc); free(partial); free(x); free(y); free(tmp); free(plains); free(nonempty);
    return 0;
}

/* Multi-shard image-mode geometry (conv.cpp:37-67 with t >= 2, d = 1,
 * rep = 1, tau = identity): shard u holds channels [u z, (u+1) z),
 *   in_channel(u, r, b) = u z + (b + r) % z,  out_channel(v, b) = (v z + b) % c_out. */
/* ImageConv::fused_plain (conv.cpp:69-85) over a PackedImage with channel
 * permutation tau (c entries, NULL = identity) and replication rep:
 * in_channel(u, r, b) = block_channel(u z + (b + r rep) mod z) with
 * block_channel(g) = tau[(g / rep) mod c] (pack.hpp:44, conv.cpp:63-65). */
int emu_fused_plain_packed(int c, int m, int kappa, int c_out, size_t s, const double* filt, const long* tau, int rep,
                           int v, int u, int r, long kk, long ll, double scale, double* plain) {
    const size_t block = (size_t)m * m;
    const size_t z = s / block;
    int any = 0;
    for (size_t i = 0; i < s; i++) plain[i] = 0.0;
    for (size_t b = 0; b < z; b++) {
        const size_t g = (size_t)u * z + (b + (size_t)r * (size_t)rep) % z;
        const int in_ch = tau ? (int)tau[(g / (size_t)rep) % (size_t)c] : (int)g;
        const int out_ch = (int)(((size_t)v * z + b) % (size_t)c_out);
        const double w = emu_filt_centered(filt, c_out, kappa, in_ch, out_ch, kk, ll) * scale;
        if (w == 0.0) continue;
        any = 1;
        const long i_lo = kk < 0 ? -kk : 0, i_hi = kk > 0 ? m - kk : m;
        const long j_lo = ll < 0 ? -ll : 0, j_hi = ll > 0 ? m - ll : m;
        for (long i = i_lo; i < i_hi; i++)
            for (long j = j_lo; j < j_hi; j++) plain[b * block + (size_t)(i * m + j)] = w;
    }
    return any;
}

int emu_fused_plain_ms(int c, int m, int kappa, int c_out, size_t s, const double* filt, int v, int u,
                       int r, long kk, long ll, double scale, double* plain) {
    return emu_fused_plain_packed(c, m, kappa, c_out, s, filt, NULL, 1, v, u, r, kk, ll, scale, plain);
}

/* conv_image_shards (conv.cpp:261-264 -> conv_image_mode, plan = nullopt,
 * conv.cpp:146-199 without hoisting): t = c m^2 / s input shards, n_out =
 * c_out m^2 / s output shards (c_out > z) or 1. out = [n_out][s]. */
int emu_conv_shards_slots(int c, int m, int kappa, int c_out, size_t s, const double* img, const double* filt,
                          double* out) {
    const size_t block = (size_t)m * m;
    if (s % block || (size_t)c * block < s) return -1; /* image mode without duplication (d = 1) */
    const size_t z = s / block, t = (size_t)c * block / s;
    const size_t n_out = (size_t)c_out <= z ? 1 : (size_t)c_out / z;
    const long h = kappa / 2;
    const int nk = (int)((2 * h + 1) * (2 * h + 1));
    double* acc = calloc(n_out * s, sizeof(double));
    int* have_acc = calloc(n_out, sizeof(int));
    double* partial = malloc(n_out * s * sizeof(double));
    int* have_partial = malloc(n_out * sizeof(int));
    double* x = malloc(s * sizeof(double));
    double* y = malloc(s * sizeof(double));
    double* plains = malloc(n_out * (size_t)nk * s * sizeof(double));
    int* nonempty = malloc(n_out * (size_t)nk * sizeof(int));
    for (size_t u = 0; u < t; u++) {
        const double* src = img + u * s; /* pack(): shard u = flat slots [u s, (u+1) s) */
        for (size_t r = 0; r < z; r++) {
            int any = 0;
            for (size_t v = 0; v < n_out; v++) {
                int idx = 0;
                for (long kk = -h; kk <= h; kk++)
                    for (long ll = -h; ll <= h; ll++, idx++) {
                        nonempty[v * nk + idx] = emu_fused_plain_ms(c, m, kappa, c_out, s, filt, (int)v, (int)u,
                                                                    (int)r, kk, ll, 1.0,
                                                                    plains + (v * nk + idx) * s);
                        any |= nonempty[v * nk + idx];
                    }
            }
            if (!any) continue;                       /* conv.cpp:172 */
            emu_rotate(src, x, s, (long)(r * block)); /* conv.cpp:174 */
            for (size_t v = 0; v < n_out; v++) have_partial[v] = 0;
            int idx = 0;
            for (long kk = -h; kk <= h; kk++)
                for (long ll = -h; ll <= h; ll++, idx++) {
                    int rotated = 0;
                    for (size_t v = 0; v < n_out; v++) {
                        if (!nonempty[v * nk + idx]) continue;
                        if (!rotated) {
                            emu_rotate(x, y, s, kk * m + ll); /* conv.cpp:192 */
                            rotated = 1;
                        }
                        const double* p = plains + (v * nk + idx) * s;
                        double* pv = partial + v * s;
                        if (!have_partial[v]) {
                            for (size_t i = 0; i < s; i++) pv[i] = y[i] * p[i];
                            have_partial[v] = 1;
                        } else {
                            for (size_t i = 0; i < s; i++) pv[i] = pv[i] + y[i] * p[i];
                        }
                    }
                }
            for (size_t v = 0; v < n_out; v++) {
                if (!have_partial[v]) continue;
                double* av = acc + v * s;
                if (!have_acc[v]) {
                    memcpy(av, partial + v * s, s * sizeof(double));
                    have_acc[v] = 1;
                } else {
                    for (size_t i = 0; i < s; i++) av[i] = av[i] + partial[v * s + i];
                }
            }
        }
    }
    for (size_t v = 0; v < n_out; v++)
        if (!have_acc[v]) /* Acc::finish zero product against shard 0 */
            for (size_t i = 0; i < s; i++) acc[v * s + i] = img[i] * 0.0;
    memcpy(out, acc, n_out * s * sizeof(double));
    free(acc); free(have_acc); free(partial); free(have_partial); free(x); free(y); free(plains); free(nonempty);
    return (int)n_out;
}

/* Channel-shard mode (conv_channel_shards, conv.cpp:273-362): m^2 > s, each
 * channel spans pc = m^2 / s shards of rows = s / m rows; input shard
 * (f, u) = image rows [u rows, (u+1) rows) of channel f. Output shard
 * (g, v) sums, per (f, kk, ll) with w != 0, the in-shard term
 * mask_in . rot(in[f][v], kk m + ll) and (kk != 0) the spill term from the
 * neighbour shard v + sign(kk). out = [c_out][pc][s]. */
int emu_conv_channel_slots(int c, int m, int kappa, int c_out, size_t s, const double* img, const double* filt,
                           double* out) {
    const size_t block = (size_t)m * m;
    if (block <= s || block % s || s % (size_t)m) return -1;
    const size_t pc = block / s;
    const long rows = (long)(s / (size_t)m), mL = m;
    const long h = kappa / 2;
    if (h > rows) return -1; /* "kernel reach exceeds one neighbor shard" */
    double* mask = malloc(s * sizeof(double));
    double* y = malloc(s * sizeof(double));
    double* acc = malloc(s * sizeof(double));
    for (int g = 0; g < c_out; g++)
        for (size_t v = 0; v < pc; v++) {
            int have = 0;
            for (int f = 0; f < c; f++)
                for (long kk = -h; kk <= h; kk++)
                    for (long ll = -h; ll <= h; ll++) {
                        const double w = emu_filt_centered(filt, c_out, kappa, f, g, kk, ll) * 1.0;
                        if (w == 0.0) continue;
                        const long amount = kk * mL + ll;
                        const long j_lo = ll < 0 ? -ll : 0, j_hi = ll > 0 ? mL - ll : mL;
                        if (j_lo >= j_hi) continue;
                        for (int spill = 0; spill < 2; spill++) {
                            long src = (long)v;
                            if (spill) {
                                if (kk == 0) continue;
                                src = (long)v + (kk > 0 ? 1 : -1);
                                if (src < 0 || src >= (long)pc) continue;
                            }
                            int any = 0;
                            for (size_t i = 0; i < s; i++) mask[i] = 0.0;
                            for (long rr = 0; rr < rows; rr++) {
                                const int inside = rr + kk >= 0 && rr + kk < rows;
                                if (inside == spill) continue;
                                any = 1;
                                for (long j = j_lo; j < j_hi; j++) mask[(size_t)(rr * mL + j)] = w;
                            }
                            if (!any) continue;
                            emu_rotate(img + ((size_t)f * pc + (size_t)src) * s, y, s, amount);
                            if (!have) {
                                for (size_t i = 0; i < s; i++) acc[i] = y[i] * mask[i];
                                have = 1;
                            } else {
                                for (size_t i = 0; i < s; i++) acc[i] = acc[i] + y[i] * mask[i];
                            }
                        }
                    }
            if (!have) /* Acc::finish zero product against shard 0 */
                for (size_t i = 0; i < s; i++) acc[i] = img[i] * 0.0;
            memcpy(out + ((size_t)g * pc + v) * s, acc, s * sizeof(double));
        }
    free(mask);
    free(y);
    free(acc);
    return (int)((size_t)c_out * pc);
}

void emu_oracle_conv(int c, int m, int kappa, int c_out, const double* img, const double* filt,
                     double* out) { /* oracle.cpp:7-31, stride 1 */
    const long h = kappa / 2;
    for (int g = 0; g < c_out; g++)
        for (long i = 0; i < m; i++)
            for (long j = 0; j < m; j++) {
                double acc = 0.0;
                for (int f = 0; f < c; f++)
                    for (long kr = -h; kr <= h; kr++)
                        for (long kc = -h; kc <= h; kc++) {
                            const long ii = i + kr, jj = j + kc;
                            const double v = (ii < 0 || jj < 0 || ii >= m || jj >= m)
                                                 ? 0.0
                                                 : img[((size_t)f * m + (size_t)ii) * m + (size_t)jj];
                            acc += emu_filt_centered(filt, c_out, kappa, f, g, kr, kc) * v;
                        }
                out[((size_t)g * m + (size_t)i) * m + (size_t)j] = acc;
            }
}

static uint64_t floor_pow2(uint64_t n) { /* rot.cpp:9-13 */
    uint64_t p = 1;
    while (p * 2 <= n) p *= 2;
    return p;
}

int emu_decompose(int strategy, uint64_t n, uint64_t s, long* steps, int cap) {
    if (n >= s) return -1; /* check_range rot.cpp:15-17 */
    int k = 0;
    if (strategy == 0) { /* rot.cpp:21-29 */
        for (uint64_t bit = floor_pow2(s); bit >= 1; bit /= 2) {
            if (n & bit) {
                if (k >= cap) return -1;
                steps[k++] = (long)bit;
            }
            if (bit == 1) break;
        }
        return k;
    }
    long rest = (long)n; /* rot.cpp:31-46 */
    while (rest != 0) {
        const uint64_t mag = (uint64_t)(rest < 0 ? -rest : rest);
        const uint64_t lo = floor_pow2(mag), hi = lo * 2;
        const uint64_t pick = (mag - lo <= hi - mag) ? lo : hi;
        const long step = rest < 0 ? -(long)pick : (long)pick;
        if (k >= cap) return -1;
        steps[k++] = step;
        rest -= step;
    }
    return k;
}

int emu_min_lengths(uint64_t n_max, uint64_t cap, uint64_t* out) { /* rot.cpp:53-94 */
    if (n_max >= cap) return -1;
    const long limit = (long)(4 * cap);
    const size_t width = (size_t)(2 * limit + 1);
    const uint64_t unset = (uint64_t)-1;
    uint64_t* dist = malloc(width * sizeof(uint64_t));
    long* queue = malloc(width * sizeof(long));
    long powers[64];
    int np = 0;
    for (long p = 1; p <= 2 * (long)cap; p *= 2) powers[np++] = p;
    for (size_t i = 0; i < width; i++) dist[i] = unset;
    size_t head = 0, tail = 0;
    dist[limit] = 0;
    queue[tail++] = 0;
    while (head < tail) {
        const long v = queue[head++];
        for (int pi = 0; pi < np; pi++) {
            const long cand[2] = {v + powers[pi], v - powers[pi]};
            for (int q = 0; q < 2; q++) {
                const long nx = cand[q];
                if (nx < -limit || nx > limit) continue;
                if (dist[nx + limit] != unset) continue;
                dist[nx + limit] = dist[v + limit] + 1;
                queue[tail++] = nx;
            }
        }
    }
    for (uint64_t n = 0; n <= n_max; n++) out[n] = dist[(long)n + limit];
    free(dist);
    free(queue);
    return 0;
}
