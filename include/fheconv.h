/*
 * fheconv.h — C ABI of the B200-native RNS-CKKS encrypted-convolution hot path.
 *
 * Drop-in boundary. The reference has no FFI;
 * its evaluator is the concrete C++ class shardnn::Engine
 * (reference proj/include/shardnn/emu.hpp:132-183) passed as Engine& to the
 * conv operators (conv.hpp:29-68). Each entry point below names the
 * reference interface it replaces. include/fheconv.hpp wraps these calls in
 * an Engine-shaped C++ class with the reference's method names and
 * exception messages.
 *
 * Conventions
 *   - All functions return 0 (FHE_OK) on success, a negative FHE_E* code on
 *     failure; fhe_last_error(ctx) returns the message, using the
 *     reference's exception text where one exists (e.g. "slot count
 *     mismatch", "depth exhausted", "empty rotation batch",
 *     "insufficient capacity").
 *   - Handles own device memory on the context's GPU; one CUDA stream per
 *     context; a context is not thread-safe (serialise per context, as the
 *     reference's Engine RNG is unguarded, emu.hpp:181).
 *   - Residues are uint64 in [0, q), NTT domain, laid out [poly][prime][N]
 *     (ciphertext = 2 polys over q_0..q_level).
 *   - There is NO CPU fallback: on a machine without a usable sm_100 GPU,
 *     fhe_ctx_create fails with FHE_E_CUDA.
 */
#ifndef FHECONV_H
#define FHECONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FHE_OK 0
#define FHE_E_INVALID (-1)  /* std::invalid_argument in the reference */
#define FHE_E_RUNTIME (-2)  /* std::runtime_error in the reference    */
#define FHE_E_CUDA (-3)     /* device / driver failure                */
#define FHE_E_NOKEY (-4)    /* required Galois key was not generated  */

typedef struct fhe_ctx fhe_ctx;
typedef struct fhe_ct fhe_ct;                 /* device ciphertext      */
typedef struct fhe_pt fhe_pt;                 /* device plaintext       */
typedef struct fhe_conv_layer fhe_conv_layer; /* pre-encoded conv layer */

typedef struct {
    int log_n;          /* ring degree N = 2^log_n, slots s = N/2            */
    int n_q;            /* number of ciphertext primes (levels = n_q - 1)    */
    const int* q_bits;  /* bit sizes of q_0..q_{n_q-1}                       */
    int n_p;            /* number of special primes K (digit size alpha = K) */
    const int* p_bits;  /* bit sizes of p_0..p_{K-1}                         */
    int log_scale;      /* Delta = 2^log_scale                               */
    int device;         /* CUDA device ordinal                               */
} fhe_params;

/* CostLedger counters (reference emu.hpp:39-122) + CKKS work counters. */
typedef struct {
    uint64_t rotations;          /* emu.hpp:41 */
    uint64_t hoisted_rotations;  /* emu.hpp:42 */
    uint64_t hoist_groups;       /* emu.hpp:43 */
    uint64_t ct_pt_mults;        /* emu.hpp:44 */
    uint64_t ct_ct_mults;        /* emu.hpp:45 */
    uint64_t adds;               /* emu.hpp:46 */
    uint64_t bootstraps;         /* emu.hpp:47 */
    uint64_t max_depth_consumed; /* emu.hpp:48 */
    uint64_t distinct_amounts;   /* |rotation_amounts()| emu.hpp:63-66 */
    /* work actually performed on the GPU */
    uint64_t key_switches;       /* Galois key inner products */
    uint64_t modups;
    uint64_t moddowns;
    uint64_t rescales;
    uint64_t kernel_launches;
} fhe_ledger;

/* ---------------------------------------------------------------- context */
/* replaces: shardnn::Engine(EngineConfig) emu.hpp:134 */
int fhe_ctx_create(const fhe_params* params, fhe_ctx** out);
void fhe_ctx_destroy(fhe_ctx* ctx);
const char* fhe_last_error(const fhe_ctx* ctx);
/* N, slots, n_q, n_p, dnum, primes (n_q + n_p entries, q's then p's) */
int fhe_ctx_info(const fhe_ctx* ctx, int* log_n, int* n_q, int* n_p, int* dnum, uint64_t* primes);
int fhe_synchronize(fhe_ctx* ctx);
/* device-side timing on the context's stream (CUDA events) */
int fhe_timer_start(fhe_ctx* ctx);
int fhe_timer_stop(fhe_ctx* ctx, float* ms); /* synchronises; ms since fhe_timer_start */
/* per-kernel-class CUDA-event profiling of the hot kernels (off by default).
 * class names: "ntt", "ntt_modup", "ntt_moddown", "ks_multi", "pt_matvec",
 * "ks_inner", "conv_mac", "moddown", "rescale" */
int fhe_prof_enable(fhe_ctx* ctx, int on);
int fhe_prof_get(fhe_ctx* ctx, const char* kernel_class, double* total_ms, uint64_t* launches);
/* same + the algorithmic (compulsory) bytes of those launches: every input
 * read once, every output written once, intermediates inside a launch excluded */
int fhe_prof_get_bytes(fhe_ctx* ctx, const char* kernel_class, double* total_ms, uint64_t* launches, double* bytes);
int fhe_prof_reset(fhe_ctx* ctx);
/* micro-benchmark of the NTT kernels: nrows rows at the top level's primes,
 * `iters` transforms; *ms = device time per transform launch */
int fhe_bench_ntt(fhe_ctx* ctx, int nrows, int inverse, int iters, float* ms);
/* cudaProfilerStart/Stop (scopes ncu --profile-from-start off captures) */
int fhe_profiler_range(int on);
/* replaces: Engine::ledger() emu.hpp:137-138, CostLedger::reset emu.hpp:77-88 */
int fhe_ledger_get(const fhe_ctx* ctx, fhe_ledger* out);
int fhe_ledger_reset(fhe_ctx* ctx);
/* distinct requested rotation amounts (mod s, zero included), ascending */
int fhe_ledger_amounts(const fhe_ctx* ctx, uint64_t* out, size_t cap, size_t* n);

/* ------------------------------------------------------------------- keys */
/* (CKKS-only; no reference counterpart — the emulator has no keys) */
int fhe_keygen(fhe_ctx* ctx, uint64_t seed);
/* Galois keys for left rotations by each step (mod s); 0 is ignored. */
int fhe_gen_galois_keys(fhe_ctx* ctx, const int64_t* steps, size_t n);
/* download the key for rotation `step`: [dnum][2][n_q+n_p][N] words */
int fhe_galois_key_download(fhe_ctx* ctx, int64_t step, uint64_t* host, size_t words);

/* ------------------------------------------------------------------- data */
/* replaces: Engine::encode(std::vector<double>) emu.hpp:144-152 (+ CKKS
 * encoding). n <= s real slots; level in [0, n_q-1]; with_special = 1 also
 * encodes residues mod the special primes (needed by fused conv plaintexts). */
int fhe_encode(fhe_ctx* ctx, const double* slots, size_t n, int level, double scale, int with_special,
               fhe_pt** out);
int fhe_encrypt(fhe_ctx* ctx, const fhe_pt* pt, uint64_t seed, fhe_ct** out);
/* decrypt + decode to n <= s real slots (replaces reading SlotVector::slots) */
int fhe_decrypt_decode(fhe_ctx* ctx, const fhe_ct* ct, double* out, size_t n);
int fhe_ct_level(const fhe_ct* ct);
double fhe_ct_scale(const fhe_ct* ct);
/* residue transfer (parity tests, e2e benchmarks); words = 2 (level+1) N */
int fhe_ct_download(fhe_ctx* ctx, const fhe_ct* ct, uint64_t* host, size_t words);
int fhe_ct_upload(fhe_ctx* ctx, const uint64_t* host, int level, double scale, fhe_ct** out);
/* overwrite an existing ciphertext of the same level in place */
int fhe_ct_upload_into(fhe_ctx* ctx, const uint64_t* host, fhe_ct* ct);
int fhe_pt_download(fhe_ctx* ctx, const fhe_pt* pt, uint64_t* host, size_t words);
int fhe_pt_rows(const fhe_pt* pt);
void fhe_ct_free(fhe_ct* ct);
void fhe_pt_free(fhe_pt* pt);

/* ---------------------------------------------------------------- ops */
/* replaces: Engine::rotate emu.cpp:28-37 — left rotation out[i] = in[(i+k) mod s];
 * k = 0 mod s is a free copy (amount still recorded). */
int fhe_rotate(fhe_ctx* ctx, const fhe_ct* ct, int64_t k, fhe_ct** out);
/* replaces: Engine::rotate_many emu.cpp:39-54 — one shared ModUp (hoisting);
 * "empty rotation batch" when n == 0. outs[i] receives a new ciphertext. */
int fhe_rotate_hoisted(fhe_ctx* ctx, const fhe_ct* ct, const int64_t* ks, size_t n, fhe_ct** outs);
/* hoisted rotations of a batch: outs[i * k + j] = rot_{ks[j]}(cts[i]) (n * k
 * outputs); one ModUp per ciphertext, each Galois key streamed once per chunk
 * of up to 16 ciphertexts */
int fhe_rotate_hoisted_batch(fhe_ctx* ctx, const fhe_ct* const* cts, size_t n, const int64_t* ks, size_t k,
                             fhe_ct** outs);
/* same into n * k preallocated ciphertexts at the inputs' level (no allocation) */
int fhe_rotate_hoisted_batch_into(fhe_ctx* ctx, const fhe_ct* const* cts, size_t n, const int64_t* ks, size_t k,
                                  fhe_ct* const* outs);
/* replaces: Engine::mul_plain emu.cpp:56-67 (no rescale; level bookkeeping by
 * fhe_rescale) */
int fhe_mul_plain(fhe_ctx* ctx, const fhe_ct* ct, const fhe_pt* pt, fhe_ct** out);
/* replaces: Engine::add emu.cpp:82-91 / sub :93-102 / add_plain :104-111 */
int fhe_add(fhe_ctx* ctx, const fhe_ct* a, const fhe_ct* b, fhe_ct** out);
int fhe_sub(fhe_ctx* ctx, const fhe_ct* a, const fhe_ct* b, fhe_ct** out);
int fhe_add_plain(fhe_ctx* ctx, const fhe_ct* ct, const fhe_pt* pt, fhe_ct** out);
/* drop q_level with centered rounding (the level the reference only counts,
 * emu.cpp:62-63) */
int fhe_rescale(fhe_ctx* ctx, const fhe_ct* ct, fhe_ct** out);

/* Rotation through power-of-two keys (replaces plan_rotations +
 * execute_schedule, reference rot.cpp:96-156). strategy: 0 positive (binary,
 * rot.cpp:21-29), 1 signed (nearest power of two, rot.cpp:31-46). Requires
 * keys for the power-of-two steps used. */
int fhe_rotate_decomposed(fhe_ctx* ctx, const fhe_ct* ct, int64_t k, int strategy, fhe_ct** out);
/* plan_rotations + execute_schedule (rot.cpp:96-156) for one source: request i
 * rotates by amounts[i]; same_source[i] != 0 joins the previous group and makes
 * it hoisted (its members' first keyed steps share one ModUp, the remaining steps
 * run sequentially). strategy 0 positive, 1 signed, 2 exact (one keyed step per
 * request). outs[n] in request order; planned_keyed = the reference's
 * total_keyed_rotations, groups / hoisted groups of the plan (all optional). */
int fhe_execute_schedule(fhe_ctx* ctx, const fhe_ct* src, const int64_t* amounts, const int* same_source, size_t n,
                         int strategy, fhe_ct** outs, uint64_t* planned_keyed, uint64_t* groups,
                         uint64_t* hoisted_groups);
/* keyed steps a decomposition uses (host-only planning) */
int fhe_decompose(int strategy, uint64_t n, uint64_t s, int64_t* steps, int cap);

/* ----------------------------------------------------------------- conv */
/* Host-side layer preparation (replaces ImageConv::fused_plain conv.cpp:69-85
 * + make_shift_plan :215-231 + bias_plain :87-94): encodes the kappa^2 * c
 * fused mask x weight plaintexts at `level` over Q_level u P with scale
 * q_level, uploads them once. weights: (c_in, c_out, kappa, kappa) as
 * FilterTensor::weights (tensor.hpp:41-58). Single image shard, c_in * m^2 <= s.
 * bias: c_out values (or NULL) and output_scale (1.0 = none) as
 * conv_plan(eng, p, k, plan, bias, output_scale) (conv.hpp:66-68): the fused
 * plaintexts carry weight * output_scale, and bias[out_channel] * output_scale
 * is added to every output block in the epilogue of the final fused ModDown +
 * rescale (bit-identical to add_plain after the conv, conv.cpp:203-210). */
int fhe_conv_layer_create(fhe_ctx* ctx, int c_in, int c_out, int m, int kappa, const double* weights,
                          const double* bias, double output_scale, int level, fhe_conv_layer** out);
void fhe_conv_layer_free(fhe_conv_layer* layer);
/* multi-shard image mode (reference conv_image_shards, conv.cpp:261-264 via
 * conv_image_mode with t >= 2): an image of c_in channels
 * with c_in m^2 = t * slots is packed into t ciphertexts (shard u = channels
 * [u z, (u+1) z), z = slots / m^2, as pack() does); the c_out output channels
 * land in n_out = max(1, c_out / z) ciphertexts (shard v block b = channel
 * (v z + b) mod c_out). Runs the fused BSGS schedule. */
int fhe_conv_layer_create_shards(fhe_ctx* ctx, int c_in, int c_out, int m, int kappa, const double* weights,
                                 const double* bias, double output_scale, int level, fhe_conv_layer** out);
/* image-mode layer over ANY PackedImage (conv_image_mode conv.cpp:40-211 as
 * convolve() reaches it after pooling): t input shards, tau[c_in] (physical
 * channel position -> logical channel; NULL = identity), rep, d (duplication,
 * t = 1 only). Channel rotations r rep m^2 (r < c_in for t = 1, else < z), fused
 * plaintexts from block_channel (pack.hpp:44). Run with fhe_conv2d_shards_into. */
int fhe_conv_layer_create_packed(fhe_ctx* ctx, int c_in, int c_out, int m, int kappa, const double* weights,
                                 const double* bias, double output_scale, int level, size_t t, const int64_t* tau,
                                 int rep, int d, fhe_conv_layer** out);
/* output duplication d of a layer (ImageConv::make_output: n_out z / c_out; rep 1, identity tau) */
int fhe_conv_layer_output_packing(const fhe_conv_layer* layer, int* d_out);
/* input / output shard counts of a layer (1 / 1 for single-shard layers) */
int fhe_conv_layer_shards(const fhe_conv_layer* layer, int* t, int* n_out);
/* n_images multi-shard convs: in = [n_images][t] ciphertexts at the layer level,
 * outs = [n_images][n_out] preallocated ciphertexts at level - 1 */
int fhe_conv2d_shards_into(fhe_ctx* ctx, const fhe_ct* const* in, size_t n_images, const fhe_conv_layer* layer,
                           fhe_ct* const* outs);
/* Galois steps a layer needs for `approach`: 1-4 channel rotations r m^2 and
 * shifts kk m + ll; 5 r m^2 + ll and kk m; 0 the union (any approach runs) */
int fhe_conv_layer_steps(const fhe_conv_layer* layer, int approach, int64_t* steps, size_t cap, size_t* n);
/* replaces: conv_plan(eng, p, k, plan) conv.cpp:266-271.
 * approach 1 = paper Approach 1 (ConvPlan::ChannelFirst: shifts first),
 * approach 2 = paper Approach 2 (ConvPlan::ShiftFirst: channel rotations first,
 *              shifts hoisted),
 * approach 3 = baby-step/giant-step: channel rotations hoisted from one
 *              decomposition, shifts applied once to aggregated sums
 *              (rotated plaintexts),
 * approach 4 = baby-step/giant-step with the roles swapped (shifts hoisted),
 * approach 5 = fused baby-step/giant-step: the c kappa rotations r m^2 + ll are
 *              hoisted and multiplied out in one kernel without materialising
 *              the rotated copies, the kappa row shifts kk m are giant steps,
 * approach 0 = 5 when c_in kappa <= 96 baby steps, else 3 or 4 (fewer giants).
 * All approaches decrypt to the same slots (within CKKS noise).
 * Output: one ciphertext at level - 1 (one rescale). */
int fhe_conv2d(fhe_ctx* ctx, const fhe_ct* ct, const fhe_conv_layer* layer, int approach, fhe_ct** out);
/* same, writing into a preallocated output ciphertext of level - 1 */
int fhe_conv2d_into(fhe_ctx* ctx, const fhe_ct* ct, const fhe_conv_layer* layer, int approach, fhe_ct* out);
/* batch: n independent ciphertexts through the same layer (keys and
 * plaintexts shared; BASELINE cfg5) */
int fhe_conv2d_batch(fhe_ctx* ctx, const fhe_ct* const* cts, size_t n, const fhe_conv_layer* layer,
                     int approach, fhe_ct** outs);
/* same, into preallocated outputs of level - 1 */
int fhe_conv2d_batch_into(fhe_ctx* ctx, const fhe_ct* const* cts, size_t n, const fhe_conv_layer* layer,
                          int approach, fhe_ct* const* outs);
/* host-resident batch: n input ciphertexts at host_in ([n][2][level+1][N]
 * words, level = the layer's level, scale `scale` or the context scale if
 * <= 0) are uploaded, convolved and downloaded to host_out ([n][2][level][N])
 * in chunks of `chunk` (0: 4) with uploads, convs and downloads of
 * neighbouring chunks overlapped on three streams. Returns when host_out is
 * complete. Pinned (page-locked) host buffers give asynchronous copies. */
int fhe_conv2d_batch_host(fhe_ctx* ctx, const uint64_t* host_in, size_t n, double scale,
                          const fhe_conv_layer* layer, int approach, size_t chunk, uint64_t* host_out);
/* asynchronous form: enqueues the uploads, convs and downloads and returns;
 * consecutive calls pipeline into one another (the upload of call j+1 runs
 * under the convs of call j). host_in / host_out must stay valid and
 * untouched until fhe_host_wait returns. */
int fhe_conv2d_batch_host_async(fhe_ctx* ctx, const uint64_t* host_in, size_t n, double scale,
                                const fhe_conv_layer* layer, int approach, size_t chunk, uint64_t* host_out);
/* waits for every enqueued host-resident batch (and all other work of ctx) */
int fhe_host_wait(fhe_ctx* ctx);

/* rotate-and-add reduction (reference dense.cpp:23-30):
 * outs[i] = slot_sum(cts[i], block): log2(block) rotations by 1, 2, 4, ...
 * each added back; every step rotates the whole batch with the keys shared. */
int fhe_slot_sum_batch(fhe_ctx* ctx, const fhe_ct* const* cts, size_t n, uint64_t block, fhe_ct** outs);
/* linear head (reference linear(), dense.cpp:34-75): W x + b over the features
 * of a packed image (t shards as fhe_conv_layer_create(_shards) packs them,
 * c channels of m x m), W = [out_features][c m^2] row-major, b = [out_features];
 * output features in slots 0..out_features-1, two levels consumed. */
int fhe_linear(fhe_ctx* ctx, const fhe_ct* const* shards, size_t t, int c, int m, int out_features, const double* w,
               const double* b, fhe_ct** out);

/* linear() / pool_linear() over ANY PackedImage: features[u * slots + i] is the
 * input feature held by slot i of shard u, -1 for none (the reference's
 * slot_feature_map, pack.cpp:109-129: non-primary replicas and padding are -1);
 * w is [out_features][in_features]. */
int fhe_linear_features(fhe_ctx* ctx, const fhe_ct* const* shards, size_t t, const int64_t* features,
                        size_t in_features, int out_features, const double* w, const double* b, fhe_ct** out);

/* 2x2 average pooling (reference pool(), pool.cpp:291-297) of
 * the t shards of pack(img, slots) (image mode, t = 1, 2 or a multiple of 4,
 * a single shard possibly duplicated; or channel shards, m^2 > slots): outs
 * (n_out ciphertexts, at most t) hold the (m/2)^2 channels with the reference's
 * packing metadata: tau_out[c] (physical channel position -> logical channel),
 * rep_out, d_out (duplication). Three levels. */
int fhe_pool(fhe_ctx* ctx, const fhe_ct* const* in, size_t t, int c, int m, fhe_ct** outs, size_t* n_out,
             int64_t* tau_out, int* rep_out, int* d_out);
/* subsample_stride2 (pool.cpp:299-306): the same without the 2x2 window sum
 * (every other row and column kept). Two levels. */
int fhe_subsample_stride2(fhe_ctx* ctx, const fhe_ct* const* in, size_t t, int c, int m, fhe_ct** outs,
                          size_t* n_out, int64_t* tau_out, int* rep_out, int* d_out);
/* the general form (downsample + consolidate + duplicate_channels, pool.cpp:238-297)
 * for any PackedImage: input tau (NULL = identity), rep, d; window 1 = 2x2 average
 * (pool), 0 = stride-2; output_scale multiplies the vertical masks
 * (reduce_vertical_*'s `scale`); mode_out 0 = image shards, 1 = channel shards. */
int fhe_downsample(fhe_ctx* ctx, const fhe_ct* const* in, size_t t, int c, int m, const int64_t* tau_in, int rep_in,
                   int d_in, int window, double output_scale, fhe_ct** outs, size_t* n_out, int64_t* tau_out,
                   int* rep_out, int* d_out, int* mode_out);

/* ciphertext x ciphertext multiplication and the Chebyshev
 * activation (reference Engine::mul_ct emu.cpp:69-80, eval_chebyshev act.cpp:151-162).
 * The relinearisation key (s^2 -> s) must exist: fhe_gen_relin_key. fhe_mul
 * drops the higher operand to the common level, relinearises and rescales
 * (one level; scale = scale_a * scale_b / q_l). */
int fhe_gen_relin_key(fhe_ctx* ctx);
/* Engine::add_scalar (emu.cpp:113-119): ct + k in every slot, no level consumed */
int fhe_add_scalar(fhe_ctx* ctx, const fhe_ct* ct, double k, fhe_ct** out);
/* mul_plain by a constant vector (emu.cpp:56-67): ct * k, one level, scale preserved exactly */
int fhe_mul_scalar(fhe_ctx* ctx, const fhe_ct* ct, double k, fhe_ct** out);
int fhe_mul(fhe_ctx* ctx, const fhe_ct* a, const fhe_ct* b, fhe_ct** out);
/* sum_k coeffs[k] T_k(x / bound) (x / bound already in [-1, 1] when prescaled),
 * the reference's power-of-two split; levels: bit length of n - 1 (+1 unless prescaled) */
int fhe_eval_chebyshev(fhe_ctx* ctx, const fhe_ct* x, const double* coeffs, size_t n, double bound, int prescaled,
                       fhe_ct** out);

#ifdef __cplusplus
}
#endif
#endif /* FHECONV_H */
