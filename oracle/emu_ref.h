/* TEST INFRASTRUCTURE ONLY — the oracle (checker). Never linked into the
 * product library; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load it.
 *
 * CPU restatement of the reference's slot-level algorithm on the hot path
 * (the "emulator" side: what the decrypted CKKS result must equal).
 */
#ifndef FHECONV_ORACLE_EMU_REF_H
#define FHECONV_ORACLE_EMU_REF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    uint64_t mt[312];
    int mti;
    int have_saved;
    double saved;
} mt64_state;

void mt64_seed(mt64_state* st, uint64_t seed);
uint64_t mt64_next(mt64_state* st);
double mt64_canonical(mt64_state* st);
double mt64_uniform(mt64_state* st, double a, double b);
double mt64_normal(mt64_state* st, double mean, double stddev);
void emu_make_inputs(int c, int m, int kappa, int c_out, uint64_t seed_img, uint64_t seed_filt,
                     int weight_kind, double* img, double* filt);

/* Cyclic left rotation out[i] = in[(i + k) mod s] (reference emu.cpp:9-20). */
void emu_rotate(const double* in, double* out, size_t s, long k);

/* Fused plaintext of conv.cpp:69-85 for a single image shard of s slots
 * (t = 1, rep = 1, identity tau, n_out = 1): returns 0 when every entry is
 * zero (the reference then skips the term), else 1. */
/* K.centered(f, g, k, l), tensor.hpp:53-67 */
double emu_filt_centered(const double* filt, int c_out, int kappa, int f, int g, long k, long l);
int emu_fused_plain(int c, int m, int kappa, int c_out, size_t s, const double* filt, int r,
                    long kk, long ll, double scale, double* plain);

/* Single-shard conv_plan on slot vectors (conv.cpp:109-211).
 * plan: 0 default (conv_single_shard), 1 ChannelFirst (paper Approach 1),
 * 2 ShiftFirst (paper Approach 2). out has s slots. */
int emu_conv_slots(int c, int m, int kappa, int c_out, size_t s, const double* img,
                   const double* filt, int plan, double* out);
/* multi-shard image mode (conv.cpp:37-67, 146-199 with t >= 2): the fused
 * plaintext of output shard v vs rotation r of input shard u, and the full
 * conv_image_shards slots; returns the output shard count n_out */
/* fused_plain over a PackedImage with permutation tau (NULL = identity) and replication rep */
int emu_fused_plain_packed(int c, int m, int kappa, int c_out, size_t s, const double* filt, const long* tau, int rep,
                           int v, int u, int r, long kk, long ll, double scale, double* plain);
int emu_fused_plain_ms(int c, int m, int kappa, int c_out, size_t s, const double* filt, int v, int u,
                       int r, long kk, long ll, double scale, double* plain);
int emu_conv_shards_slots(int c, int m, int kappa, int c_out, size_t s, const double* img, const double* filt,
                          double* out);
/* channel-shard mode (conv_channel_shards, conv.cpp:273-362), m^2 > s:
 * out = [c_out][m^2 / s][s]; returns the output shard count */
int emu_conv_channel_slots(int c, int m, int kappa, int c_out, size_t s, const double* img, const double* filt,
                           double* out);

/* Textbook same-padding cross-correlation, stride 1 (oracle.cpp:7-31). */
void emu_oracle_conv(int c, int m, int kappa, int c_out, const double* img, const double* filt,
                     double* out);

/* rot.cpp:21-46: strategy 0 = positive (binary), 1 = signed (nearest power
 * of two, ties toward the smaller). Returns the step count or -1. */
int emu_decompose(int strategy, uint64_t n, uint64_t s, long* steps, int cap);
/* rot.cpp:53-94: BFS minimal signed power-of-two lengths for n in [0, n_max]. */
int emu_min_lengths(uint64_t n_max, uint64_t cap, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
