// C-ABI implementation (include/fheconv.h): context, keys, data movement,
// ops and the fused encrypted convolution. Host C++ drives the sm_100a
// kernels in kernels.cu on one CUDA stream per context. No CPU fallback.
//
// Reference interface mirrored: shardnn::Engine (reference
// proj/include/shardnn/emu.hpp:132-183) and the conv entry points
// conv_plan / conv_single_shard (proj/src/conv.cpp:254-271).
#include <cuda_profiler_api.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fheconv.h"
#include "host_math.hpp"
#include "kernels.cuh"

using namespace fhe;

namespace {

struct FheError {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw FheError{code, m}; }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(FHE_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t dev_words_alloc_count = 0;

}  // namespace

struct fhe_ctx {
    int device = 0;
    cudaStream_t st = nullptr;       // stream the internals enqueue on (main or a lane)
    cudaStream_t main_st = nullptr;  // the context's stream
    std::vector<cudaStream_t> lanes; // extra streams: independent ciphertexts of a batch overlap
    cudaStream_t h2d_st = nullptr;   // host-pipelined batches: uploads
    cudaStream_t d2h_st = nullptr;   // host-pipelined batches: downloads
    // host-pipelined batches: two persistent device chunk buffers (inputs in the
    // upload stream's order, outputs in the conv stream's) and their events;
    // consecutive calls keep alternating them, so the pipeline runs across calls
    struct HostPipe {
        int level = -1;
        size_t S = 0;
        std::vector<uint64_t*> din[2], dout[2];
        cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
        uint64_t chunks = 0;
    } hp;
    bool fused_batch = false;        // FHECONV_BATCH_FUSED=1: batched kernels instead of lanes
    bool batch5 = true;              // approach 5: sources batched through one fused launch (FHECONV_BATCH5=0: lanes)
    bool limb = true;                // approach 5 baby steps on operand-form rows, TMA-staged (k_bsgs_tma);
                                     // FHECONV_LIMB=0 or FHECONV_TMA=0: k_bsgs_fused on plain rows
    bool tma = true;
    int logN = 0, N = 0, L = 0, K = 0, alpha = 0, dnum = 0, np = 0;
    std::vector<uint64_t> primes;
    double scale = 0;
    DevCtx dc{};
    Prime* d_primes = nullptr;
    uint64_t *d_tw = nullptr, *d_tw_sh = nullptr, *d_itw = nullptr, *d_itw_sh = nullptr;
    uint64_t *d_ninv = nullptr, *d_ninv_sh = nullptr;
    double2 *d_twd = nullptr, *d_itwd = nullptr, *d_ninvd = nullptr;
    ModUpDigit* d_modup = nullptr;  // [L][dnum]
    ModDownTable* d_md = nullptr;
    uint64_t *d_qlinv = nullptr, *d_qlinv_sh = nullptr;  // [L][L]
    uint64_t *d_pqlinv = nullptr, *d_pqlinv_sh = nullptr;  // [L][L] (P q_l)^-1 mod q_i (fused ModDown+rescale)
    uint64_t* d_s = nullptr;                              // secret, [np][N] NTT
    bool have_key = false;
    uint64_t key_seed = 0;
    std::map<uint32_t, uint64_t*> keys;
    std::map<uint32_t, uint64_t*> keys_opf;  // operand-form copies (modarith.cuh to_opf) of the Galois keys
    // the operand-form keys live in one arena [cap][2 dnum][L+K][N] (slot per key), so a
    // single TMA tensor map covers all of them (k_bsgs_tma key map, hoisted batches)
    uint64_t* d_key_arena = nullptr;
    int arena_cap = 0, arena_n = 0;
    std::map<uint32_t, int> key_slot;
    unsigned* d_sched = nullptr;             // k_bsgs_tma work queues (kTmaSchedWords)
    uint64_t key_gen = 0;  // bumped by fhe_keygen: per-layer limb key copies are rebuilt
    fhe_ledger ledger{};
    uint64_t launch_base = 0;
    int giant_chunk = 8;  // giant steps per ModUp batch (FHECONV_GIANT_CHUNK)
    std::set<uint64_t> amounts;
    std::string err;
    // pinned staging
    void* h_stage = nullptr;
    size_t h_stage_bytes = 0;
    // timing / profiling (CUDA events on st)
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    bool prof_on = false;
    // CUDA graphs of batched convs (FHECONV_GRAPHS=0 disables): captured once per
    // (layer, approach, input/output ciphertexts) and replayed; the ledger and
    // launch counters of the capture are re-applied on every replay
    struct GraphEntry {
        std::vector<const void*> key;
        cudaGraphExec_t exec = nullptr;
        fhe_ledger delta{};
        std::vector<uint64_t> amounts;  // rotation amounts the captured conv records
        uint64_t launches = 0;
        uint64_t last_use = 0;
    };
    std::vector<GraphEntry> graphs;
    // device plaintexts of the pooling stages, keyed by (stage, m, level)
    std::map<std::string, uint64_t*> lt_cache;
    // encoded plaintexts of the linear head (weight masks, selection masks, bias) in the order
    // linear_impl uses them, keyed by a hash of (weights, bias, slot -> feature map, level,
    // scale): a served network re-encodes nothing (<= 4 heads kept, least recently used out)
    struct LinearEntry {
        uint64_t key = 0;
        uint64_t last_use = 0;
        std::vector<fhe_pt*> pts;
    };
    std::vector<LinearEntry> linear_cache;
    uint64_t linear_clock = 0;
    bool use_graphs = true;
    uint64_t graph_clock = 0;
    struct ProfRec {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
        double ms = 0;
        uint64_t n = 0;
        double bytes = 0;  // algorithmic (compulsory) bytes of the launches
    };
    std::map<std::string, ProfRec> prof;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaEvent_t> pending_events;  // recycled at the next prof_collect / sync

    cudaEvent_t get_event() {
        if (!ev_pool.empty()) {
            cudaEvent_t e = ev_pool.back();
            ev_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }
    // algorithmic bytes of `rows` residue rows
    double rows(double r) const { return r * (double)N * 8.0; }
    template <class F>
    void timed(const char* cls, double bytes, F&& f) {
        if (!prof_on) {
            f();
            return;
        }
        cudaEvent_t a = get_event(), b = get_event();
        cudaEventRecord(a, st);
        f();
        cudaEventRecord(b, st);
        prof[cls].pending.emplace_back(a, b);
        prof[cls].bytes += bytes;
    }
    void prof_collect() {
        ck(cudaStreamSynchronize(st), "sync");
        for (cudaStream_t l : lanes) ck(cudaStreamSynchronize(l), "sync");
        for (cudaEvent_t e : pending_events) ev_pool.push_back(e);
        pending_events.clear();
        for (auto& kv : prof) {
            for (auto& pr : kv.second.pending) {
                float ms = 0;
                cudaEventElapsedTime(&ms, pr.first, pr.second);
                kv.second.ms += ms;
                kv.second.n++;
                ev_pool.push_back(pr.first);
                ev_pool.push_back(pr.second);
            }
            kv.second.pending.clear();
        }
    }

    // ------------------------------------------------------------ helpers
    uint64_t* alloc(size_t words) {
        void* p = nullptr;
        ck(cudaMallocAsync(&p, words * 8, st), "cudaMallocAsync");
        dev_words_alloc_count += words;
        return (uint64_t*)p;
    }
    void release(void* p) {
        if (p) cudaFreeAsync(p, st);
    }
    void* stage(size_t bytes) {
        if (bytes > h_stage_bytes) {
            if (h_stage) {
                cudaStreamSynchronize(st);
                cudaFreeHost(h_stage);
            }
            ck(cudaMallocHost(&h_stage, bytes), "cudaMallocHost");
            h_stage_bytes = bytes;
        }
        return h_stage;
    }
    size_t slots() const { return (size_t)N / 2; }
    int dn_at(int level) const { return (level + 1 + alpha - 1) / alpha; }
    int ne_at(int level) const { return level + 1 + K; }
    uint32_t galois_of(uint64_t amount) const {
        return (uint32_t)host::powmod(5, amount, 2 * (uint64_t)N);
    }
    uint64_t reduce_amount(int64_t k) const {
        const int64_t s = (int64_t)slots();
        int64_t m = k % s;
        if (m < 0) m += s;
        return (uint64_t)m;
    }
    std::vector<uint64_t>* amount_rec = nullptr;  // amounts noted while a graph is captured
    void note_amount(uint64_t a) {
        amounts.insert(a);
        if (amount_rec) amount_rec->push_back(a);
    }
    const uint64_t* key_for(uint32_t g) const {
        auto it = keys.find(g);
        if (it == keys.end()) fail(FHE_E_NOKEY, "missing Galois key for rotation");
        return it->second;
    }
    const uint64_t* key_opf_for(uint32_t g) const {
        auto it = keys_opf.find(g);
        if (it == keys_opf.end()) fail(FHE_E_NOKEY, "missing Galois key for rotation");
        return it->second;
    }
};

struct fhe_ct {
    fhe_ctx* ctx;
    int level;
    double scale;
    int depth;
    uint64_t* d;
    size_t words() const { return (size_t)2 * (level + 1) * ctx->N; }
    uint64_t* c0() const { return d; }
    uint64_t* c1() const { return d + (size_t)(level + 1) * ctx->N; }
};

struct fhe_pt {
    fhe_ctx* ctx;
    int level;
    int rows;
    double scale;
    uint64_t* d;
};

struct fhe_conv_layer {
    fhe_ctx* ctx;
    // unique per layer object (never reused, unlike the host address): keys the
    // CUDA-graph cache so a freed layer's graphs can never be replayed for a new one
    uint64_t uid = next_uid();
    static uint64_t next_uid() {
        static std::atomic<uint64_t> n{1};
        return n++;
    }
    int c_in, c_out, m, kappa, level, nk;
    std::vector<int> nonempty;  // [c_in][nk]
    uint64_t* d_pts;            // [c_in][nk][ne][N]
    size_t pt_words;
    std::vector<double> weights;
    // BSGS plaintext sets (approach 3: baby = channel rotations, 4: baby = shifts,
    // 5: baby = channel rotation + column shift r m^2 + ll, giant = row shift kk m)
    struct Bsgs {
        bool ready = false;
        int nb = 0, ngi = 0;
        std::vector<int64_t> bamt, gamt;
        std::vector<int> nonempty;  // [ngi][nb]
        uint64_t* d_pts = nullptr;  // [ngi][nb][ne][N], pt'[g][b] = rot_{-g}(pt)
        uint64_t* d_pts_limb = nullptr;   // the same in operand form (approach 5, k_bsgs_tma)
        uint64_t* d_keys_limb = nullptr;  // limb-form keys of the keyed baby steps [nkeys][2 dnum][L+K][N]
        std::vector<int> kidx;            // baby b -> its key in d_keys_limb (-1: identity)
        uint64_t limb_gen = 0;            // key generation d_keys_limb was built from
    } bs[3];
    // operand-form copies for the paper schedules on the TMA baby-step kernel
    // (conv_paper_batch): the fused plaintexts [c_in][nk][ne][N], and per approach
    // (1, 2) the keys of the second-level rotations [nkeys][2 dnum][L+K][N]
    uint64_t* d_pts_opf = nullptr;
    struct PaperKeys {
        uint64_t* d_keys = nullptr;
        std::vector<int> kidx;  // second-level member x -> its key (-1: identity)
        uint64_t gen = 0;
    } pk[2];
    // multi-shard image mode (fhe_conv_layer_create_shards): t input shards of z
    // channels, n_out output shards; fused-BSGS plaintexts
    // pt'[v][kk][b = (u, r, ll)] = rot_{-kk m}(fused_plain_ms(v, u, r, kk, ll))
    bool ms = false;
    bool cs = false;  // channel-shard mode (m^2 > slots): pc = m^2 / slots shards per channel
    int pc = 1;
    int t = 1, z = 0, n_out = 1, nb_ms = 0;
    // input packing (PackedImage::tau / rep, pack.hpp:44): channel rotations r < rmax
    // by r rep m^2; block g of the input holds channel tau[(g / rep) % c_in]
    int rep = 1, rmax = 0;
    std::vector<int64_t> tau;
    std::vector<uint8_t> ms_nonempty;  // [n_out][kappa][nb_ms]
    uint64_t* d_pts_ms = nullptr;
    uint64_t* d_pts_ms_opf = nullptr;  // operand form, padded by two giants (k_bsgs_tma boxes)
    uint64_t* d_pts_cs_opf = nullptr;  // channel-shard plaintexts in operand form, padded likewise
    // bias (ImageConv::bias_plain conv.cpp:87-94, conv_channel_shards :344): one
    // slot vector per output shard (bias[out_channel] * output_scale per block),
    // encoded lazily at level - 1 and the input scale, added in the epilogue of
    // the final fused ModDown + rescale
    std::vector<std::vector<double>> bias_vecs;
    uint64_t* d_bias = nullptr;  // [n_out][level][N]
    double d_bias_scale = 0;
};

namespace {

template <class F>
int guard(const fhe_ctx* ctx, F&& f) {
    try {
        f();
        return FHE_OK;
    } catch (const FheError& e) {
        if (ctx) const_cast<fhe_ctx*>(ctx)->err = e.msg;
        return e.code;
    } catch (const std::invalid_argument& e) {
        if (ctx) const_cast<fhe_ctx*>(ctx)->err = e.what();
        return FHE_E_INVALID;
    } catch (const std::exception& e) {
        if (ctx) const_cast<fhe_ctx*>(ctx)->err = e.what();
        return FHE_E_RUNTIME;
    }
}

RowMap qmap(const fhe_ctx* c, int level) { return RowMap{level + 1, level, c->L, 0}; }

fhe_ct* new_ct(fhe_ctx* c, int level, double scale, int depth) {
    fhe_ct* ct = new fhe_ct{c, level, scale, depth, nullptr};
    ct->d = c->alloc(ct->words());
    return ct;
}

// ------------------------------------------------------------ primitives

// digits [nsrc][dn][ne][N] of nsrc polynomials c1 + s * stride (level+1 rows each, NTT)
// (limb != 0: digit rows in operand form, modarith.cuh, for k_bsgs_tma)
void modup_batch(fhe_ctx* c, const uint64_t* c1, size_t stride, int nsrc, int level, uint64_t* digits, int limb = 0) {
    const int nr = level + 1, dn = c->dn_at(level), ne = c->ne_at(level);
    const size_t rowsw = (size_t)nr * c->N;
    uint64_t* coef = c->alloc((size_t)nsrc * rowsw);
    ck(cudaMemcpy2DAsync(coef, rowsw * 8, c1, stride * 8, rowsw * 8, nsrc, cudaMemcpyDeviceToDevice, c->st),
       "memcpy2d");
    c->timed("ntt", c->rows(2.0 * nsrc * nr), [&] { ntt_inverse(c->dc, coef, nsrc * nr, qmap(c, level), c->st); });
    (void)ne;
    c->timed("ntt_modup", c->rows(2.0 * nsrc * nr + (double)nsrc * dn * ne), [&] {
        ntt_modup(c->dc, digits, coef, c1, stride, nsrc, c->d_modup + (size_t)level * c->dnum, level, dn, c->st, limb);
    });
    c->release(coef);
    c->ledger.modups += nsrc;
}

// digits [dn][ne][N] of c1 (level+1 rows, NTT)
void modup(fhe_ctx* c, const uint64_t* c1, int level, uint64_t* digits) { modup_batch(c, c1, 0, 1, level, digits); }

// out[p] = ModDown(acc[p]) (+ sigma_g(add_src) on poly 0)
void moddown_strided(fhe_ctx* c, const uint64_t* acc, size_t acc_stride, int level, int npoly, uint64_t* out,
                     const uint64_t* add_src, uint32_t g, uint64_t* const* outp = nullptr) {
    const int nr = level + 1;
    uint64_t* pc = c->alloc((size_t)npoly * c->K * c->N);
    uint64_t* conv = c->alloc((size_t)npoly * nr * c->N);
    c->timed("moddown", c->rows(2.0 * npoly * c->K), [&] { gather_special(c->dc, pc, acc, acc_stride, level, npoly, c->st); });
    c->timed("ntt", c->rows(2.0 * npoly * c->K), [&] { ntt_inverse(c->dc, pc, npoly * c->K, RowMap{c->K, -1, c->L, 0}, c->st); });
    c->timed("ntt_moddown", c->rows((double)npoly * (c->K + 2 * nr) + (add_src ? nr : 0)),
             [&] { ntt_moddown(c->dc, conv, pc, acc, acc_stride, out, c->d_md, level, npoly, add_src, g, c->st, outp); });
    c->release(pc);
    c->release(conv);
    c->ledger.moddowns += npoly;
}

// out[p] = ModDown(acc[p]) for contiguous [npoly][ne][N] accumulators
void moddown(fhe_ctx* c, const uint64_t* acc, int level, int npoly, uint64_t* out, const uint64_t* add_src,
             uint32_t g) {
    moddown_strided(c, acc, (size_t)c->ne_at(level) * c->N, level, npoly, out, add_src, g);
}

// out = rotation of ct by Galois g given the ModUp digits of ct.c1
void rotate_from_digits(fhe_ctx* c, const fhe_ct* ct, const uint64_t* digits, uint32_t g, uint64_t* out) {
    const int level = ct->level, ne = c->ne_at(level);
    uint64_t* acc = c->alloc((size_t)2 * ne * c->N);
    const uint64_t* key = c->key_for(g);
    c->timed("ks_inner", c->rows(3.0 * c->dn_at(level) * ne + 2.0 * ne), [&] {
        ks_inner_product(c->dc, digits, key, acc, acc + (size_t)ne * c->N, g, level, c->dn_at(level), c->st);
    });
    moddown(c, acc, level, 2, out, ct->c0(), g);
    c->release(acc);
    c->ledger.key_switches++;
}

// out[p] = Rescale(ModDown(acc[p])) for npoly QP accumulators at `level`,
// out = [npoly][level][N], bit-identical to moddown() followed by
// rescale_into() but with 3 inverse + `level` forward row transforms per
// polynomial instead of 28: the rescale's INTT of row q_l is
// taken from the coefficient-domain ModDown of that row, and
//   out_i = (acc_i - NTT(conv_i + P spread_i(c_l))) (P q_l)^-1.
void moddown_rescale(fhe_ctx* c, const uint64_t* acc, size_t acc_stride, int level, int npoly, uint64_t* out,
                     const uint64_t* bias = nullptr, int bias_mod = 1) {
    const size_t N = c->N;
    const int K = c->K;
    uint64_t* pc = c->alloc((size_t)npoly * (K + 1) * N);  // [npoly][K] special rows, then [npoly] q_l rows
    uint64_t* w = c->alloc((size_t)npoly * level * N);
    uint64_t* qlc = pc + (size_t)npoly * K * N;
    c->timed("moddown", c->rows(2.0 * npoly * (K + 1)), [&] {
        gather_special(c->dc, pc, acc, acc_stride, level, npoly, c->st);
        gather_row(c->dc, qlc, acc + (size_t)level * N, acc_stride, npoly, c->st);
    });
    c->timed("ntt", c->rows(2.0 * npoly * (K + 1)), [&] {
        ntt_inverse(c->dc, pc, npoly * K, RowMap{K, -1, c->L, 0}, c->st);
        ntt_inverse(c->dc, qlc, npoly, RowMap{1, -1, level, 0}, c->st);
    });
    c->timed("ntt_moddown", c->rows((double)npoly * (K + 1 + 3.0 * level)), [&] {
        ntt_moddown_rescale(c->dc, w, pc, qlc, acc, acc_stride, out, c->d_md, c->d_pqlinv + (size_t)level * c->L,
                            c->d_pqlinv_sh + (size_t)level * c->L, level, npoly, c->st, bias, bias_mod);
    });
    if (bias) c->ledger.adds += npoly / 2;  // the bias add_plain of every output (conv.cpp:207)
    c->release(pc);
    c->release(w);
    c->ledger.moddowns += npoly;
    c->ledger.rescales += npoly / 2;
}

void rescale_into(fhe_ctx* c, const uint64_t* in, int level, uint64_t* out) {
    const size_t N = c->N;
    uint64_t* tmp = c->alloc(2 * N);
    uint64_t* spread = c->alloc((size_t)2 * level * N);
    ck(cudaMemcpyAsync(tmp, in + (size_t)level * N, N * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    ck(cudaMemcpyAsync(tmp + N, in + ((size_t)level + 1 + level) * N, N * 8, cudaMemcpyDeviceToDevice, c->st),
       "memcpy");
    c->timed("ntt", c->rows(4), [&] { ntt_inverse(c->dc, tmp, 2, RowMap{1, -1, level, 0}, c->st); });
    c->timed("rescale", c->rows(2.0 + 2.0 * level), [&] { rescale_spread(c->dc, tmp, spread, level, c->st); });
    c->timed("ntt", c->rows(4.0 * level), [&] { ntt_forward(c->dc, spread, 2 * level, qmap(c, level - 1), c->st); });
    c->timed("rescale", c->rows(2.0 * (level + 1) + 4.0 * level), [&] {
        rescale_finish(c->dc, out, in, spread, level, c->d_qlinv + (size_t)level * c->L,
                       c->d_qlinv_sh + (size_t)level * c->L, c->st);
    });
    c->release(tmp);
    c->release(spread);
    c->ledger.rescales++;
}

// Galois key for element g, or (g == 0) the relinearisation key s^2 -> s; the
// PRNG streams are keyed by g, so the golden model derives the same keys.
void drop_graphs(fhe_ctx* c);
void gen_key(fhe_ctx* c, uint32_t g) {
    if (c->keys.count(g)) return;
    const size_t N = c->N;
    const int np = c->np;
    uint64_t* key = c->alloc((size_t)c->dnum * 2 * np * N);
    int64_t* e = (int64_t*)c->alloc(N);
    uint64_t* erows = c->alloc((size_t)np * N);
    const RowMap all{np, c->L - 1, c->L, 0};
    uint64_t* s2 = nullptr;
    if (g == 0) {  // s^2 in the NTT domain, every prime
        s2 = c->alloc((size_t)np * N);
        ew_mul_bcast(c->dc, s2, c->d_s, c->d_s, np, np, c->st);
    }
    for (int j = 0; j < c->dnum; ++j) {
        uint64_t* b = key + (size_t)(2 * j) * np * N;
        uint64_t* a = key + (size_t)(2 * j + 1) * np * N;
        sample_gauss(c->dc, e, stream_key(c->key_seed, stream_id(DOM_KEY_E, g, j)), c->st);
        reduce_signed_rows(c->dc, e, erows, np, all, c->st);
        ntt_forward(c->dc, erows, np, all, c->st);
        sample_uniform_rows(c->dc, a, np, all, stream_key(c->key_seed, stream_id(DOM_KEY_A, g, j)), c->st);
        const int lo = j * c->alpha, hi = std::min(lo + c->alpha, c->L);
        keygen_combine(c->dc, b, a, erows, c->d_s, g == 0 ? 1u : g, lo, hi, c->d_md, np, c->st, s2);
    }
    c->release(s2);
    c->release(e);
    c->release(erows);
    c->keys[g] = key;
    if (g != 0) {  // operand-form copy for the FP64 / limb key-switch kernels, in the key arena
        const size_t kw = (size_t)c->dnum * 2 * np * N;
        if (c->arena_n == c->arena_cap) {  // grow: captured graphs hold the old addresses
            drop_graphs(c);
            const int cap = std::max(16, 2 * c->arena_cap);
            uint64_t* na = nullptr;
            ck(cudaMalloc(&na, (size_t)cap * kw * 8), "cudaMalloc");
            if (c->arena_n)
                ck(cudaMemcpyAsync(na, c->d_key_arena, (size_t)c->arena_n * kw * 8, cudaMemcpyDeviceToDevice, c->st),
                   "memcpy");
            ck(cudaStreamSynchronize(c->st), "sync");
            if (c->d_key_arena) cudaFree(c->d_key_arena);
            c->d_key_arena = na;
            c->arena_cap = cap;
            for (auto& kv : c->key_slot) c->keys_opf[kv.first] = na + (size_t)kv.second * kw;
        }
        const int slot = c->arena_n++;
        uint64_t* ko = c->d_key_arena + (size_t)slot * kw;
        rows_to_limb(c->dc, ko, key, (size_t)c->dnum * 2 * np, RowMap{np, -1, c->L, 0}, c->st);
        c->keys_opf[g] = ko;
        c->key_slot[g] = slot;
    }
}

// destroy every captured conv graph (they embed key / plaintext device addresses)
void drop_graphs(fhe_ctx* c) {
    if (c->graphs.empty()) return;
    ck(cudaStreamSynchronize(c->main_st), "sync");
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
}

void upload_tables(fhe_ctx* c) {
    using namespace host;
    const size_t N = c->N;
    const int np = c->np, L = c->L, K = c->K;
    std::vector<Prime> pr(np);
    for (int i = 0; i < np; ++i) {
        const uint64_t q = c->primes[i];
        const u128 ratio = (~(u128)0) / q;  // floor((2^128 - 1) / q) == floor(2^128 / q) for odd q
        uint64_t inv = q;  // Newton: q^-1 mod 2^64 (q odd), 6 doublings of precision
        for (int it = 0; it < 6; ++it) inv *= 2 - q * inv;
        pr[i] = Prime{q, (uint64_t)(ratio >> 64), (uint64_t)ratio, (uint64_t)0 - inv};
    }
    std::vector<uint64_t> tw((size_t)np * N), tws((size_t)np * N), itw((size_t)np * N), itws((size_t)np * N);
    std::vector<uint64_t> ninv(np), ninvs(np);
    // FP64 companions (centred value, value / q), used by the NTT for primes < 2^50
    std::vector<double2> twd((size_t)np * N), itwd((size_t)np * N), ninvd(np);
    auto cdbl = [](uint64_t w, uint64_t q) {
        const double wc = w > q / 2 ? -(double)(q - w) : (double)w;
        return make_double2(wc, wc / (double)q);
    };
    std::vector<uint32_t> brv(N);
    for (size_t k = 0; k < N; ++k) brv[k] = bitrev((uint32_t)k, c->logN);
    std::vector<uint64_t> pw(N), ipw(N);
    for (int i = 0; i < np; ++i) {
        const uint64_t q = c->primes[i];
        const uint64_t psi = find_root(q, N), ipsi = invmod(psi, q);
        uint64_t p = 1, ip = 1;
        for (size_t k = 0; k < N; ++k) {
            pw[k] = p;
            ipw[k] = ip;
            p = mulmod(p, psi, q);
            ip = mulmod(ip, ipsi, q);
        }
        for (size_t k = 0; k < N; ++k) {
            const size_t o = (size_t)i * N + k;
            tw[o] = pw[brv[k]];
            itw[o] = ipw[brv[k]];
            tws[o] = shoup(tw[o], q);
            itws[o] = shoup(itw[o], q);
            twd[o] = cdbl(tw[o], q);
            itwd[o] = cdbl(itw[o], q);
        }
        ninv[i] = invmod(N % q, q);
        ninvs[i] = shoup(ninv[i], q);
        ninvd[i] = cdbl(ninv[i], q);
    }
    // ModUp digit tables [L][dnum]
    std::vector<ModUpDigit> mu((size_t)L * c->dnum);
    for (int level = 0; level < L; ++level) {
        const int nr = level + 1, ne = nr + K;
        for (int j = 0; j < c->dnum; ++j) {
            ModUpDigit& T = mu[(size_t)level * c->dnum + j];
            std::memset(&T, 0, sizeof(T));
            T.lo = j * c->alpha;
            T.hi = std::min(T.lo + c->alpha, nr);
            if (T.lo >= nr) continue;
            for (int i = T.lo; i < T.hi; ++i) {
                uint64_t h = 1;
                for (int i2 = T.lo; i2 < T.hi; ++i2)
                    if (i2 != i) h = mulmod(h, c->primes[i2] % c->primes[i], c->primes[i]);
                T.inv[i - T.lo] = invmod(h, c->primes[i]);
                T.inv_sh[i - T.lo] = shoup(T.inv[i - T.lo], c->primes[i]);
            }
            for (int u = 0; u < ne; ++u) {
                const int p = u <= level ? u : L + (u - level - 1);
                const uint64_t t = c->primes[p];
                uint64_t QJ = 1;
                for (int i = T.lo; i < T.hi; ++i) {
                    uint64_t h = 1;
                    for (int i2 = T.lo; i2 < T.hi; ++i2)
                        if (i2 != i) h = mulmod(h, c->primes[i2] % t, t);
                    T.hat[u][i - T.lo] = h;
                    T.hat_sh[u][i - T.lo] = shoup(h, t);
                    QJ = mulmod(QJ, c->primes[i] % t, t);
                }
                T.qj[u] = QJ;
            }
        }
    }
    // ModDown table
    ModDownTable md;
    std::memset(&md, 0, sizeof(md));
    for (int k = 0; k < K; ++k) {
        const uint64_t pk = c->primes[L + k];
        uint64_t h = 1;
        for (int k2 = 0; k2 < K; ++k2)
            if (k2 != k) h = mulmod(h, c->primes[L + k2] % pk, pk);
        md.pinv[k] = invmod(h, pk);
        md.pinv_sh[k] = shoup(md.pinv[k], pk);
    }
    for (int t = 0; t < L; ++t) {
        const uint64_t q = c->primes[t];
        uint64_t P = 1;
        for (int k = 0; k < K; ++k) {
            uint64_t h = 1;
            for (int k2 = 0; k2 < K; ++k2)
                if (k2 != k) h = mulmod(h, c->primes[L + k2] % q, q);
            md.hat[t][k] = h;
            md.hat_sh[t][k] = shoup(h, q);
            P = mulmod(P, c->primes[L + k] % q, q);
        }
        md.pmod[t] = P;
        md.pmod_sh[t] = shoup(P, q);
        md.pinvq[t] = invmod(P, q);
        md.pinvq_sh[t] = shoup(md.pinvq[t], q);
    }
    // rescale: q_l^-1 mod q_i; fused ModDown+rescale: (P q_l)^-1 mod q_i
    std::vector<uint64_t> ql((size_t)L * L, 0), qls((size_t)L * L, 0), pql((size_t)L * L, 0), pqls((size_t)L * L, 0);
    for (int l = 1; l < L; ++l)
        for (int i = 0; i < l; ++i) {
            const uint64_t q = c->primes[i];
            ql[(size_t)l * L + i] = invmod(c->primes[l] % q, q);
            qls[(size_t)l * L + i] = shoup(ql[(size_t)l * L + i], q);
            pql[(size_t)l * L + i] = mulmod(ql[(size_t)l * L + i], md.pinvq[i], q);
            pqls[(size_t)l * L + i] = shoup(pql[(size_t)l * L + i], q);
        }
    auto up = [&](void** dst, const void* src, size_t bytes) {
        ck(cudaMalloc(dst, bytes), "cudaMalloc");
        ck(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy");
    };
    up((void**)&c->d_primes, pr.data(), pr.size() * sizeof(Prime));
    up((void**)&c->d_tw, tw.data(), tw.size() * 8);
    up((void**)&c->d_tw_sh, tws.data(), tws.size() * 8);
    up((void**)&c->d_itw, itw.data(), itw.size() * 8);
    up((void**)&c->d_itw_sh, itws.data(), itws.size() * 8);
    up((void**)&c->d_ninv, ninv.data(), ninv.size() * 8);
    up((void**)&c->d_ninv_sh, ninvs.data(), ninvs.size() * 8);
    up((void**)&c->d_twd, twd.data(), twd.size() * sizeof(double2));
    up((void**)&c->d_itwd, itwd.data(), itwd.size() * sizeof(double2));
    up((void**)&c->d_ninvd, ninvd.data(), ninvd.size() * sizeof(double2));
    up((void**)&c->d_modup, mu.data(), mu.size() * sizeof(ModUpDigit));
    ck(cudaMalloc(&c->d_sched, kTmaSchedSlots * kTmaSchedWords * sizeof(unsigned)), "cudaMalloc");
    up((void**)&c->d_md, &md, sizeof(md));
    up((void**)&c->d_qlinv, ql.data(), ql.size() * 8);
    up((void**)&c->d_qlinv_sh, qls.data(), qls.size() * 8);
    up((void**)&c->d_pqlinv, pql.data(), pql.size() * 8);
    up((void**)&c->d_pqlinv_sh, pqls.data(), pqls.size() * 8);
    c->dc = DevCtx{c->logN,    c->N,        L,        K,          c->d_primes, c->d_tw,   c->d_tw_sh,
                   c->d_itw,   c->d_itw_sh, c->d_ninv, c->d_ninv_sh, c->d_twd,   c->d_itwd, c->d_ninvd};
}

void require_key(const fhe_ctx* c) {
    if (!c->have_key) fail(FHE_E_RUNTIME, "secret key not generated (call fhe_keygen)");
}

// ------------------------------------------------------------ conv layer

// Fused plaintext of reference conv.cpp:69-85 for one image shard (t = 1,
// n_out = 1, rep = 1, identity tau). Returns false when every entry is zero.
bool fused_plain(int c_in, int c_out, int m, int kappa, size_t s, const double* w, int r, long kk, long ll,
                 std::vector<double>& plain) {
    const size_t block = (size_t)m * m, z = s / block;
    const long h = kappa / 2;
    plain.assign(s, 0.0);
    bool any = false;
    for (size_t b = 0; b < z; ++b) {
        const size_t in_ch = ((b + (size_t)r) % z) % (size_t)c_in;
        const size_t out_ch = b % (size_t)c_out;
        const double wt =
            w[((in_ch * c_out + out_ch) * kappa + (size_t)(kk + h)) * kappa + (size_t)(ll + h)] * 1.0;
        if (wt == 0.0) continue;
        any = true;
        const long i_lo = std::max(0L, -kk), i_hi = std::min<long>(m, m - kk);
        const long j_lo = std::max(0L, -ll), j_hi = std::min<long>(m, m - ll);
        for (long i = i_lo; i < i_hi; ++i)
            for (long j = j_lo; j < j_hi; ++j) plain[b * block + (size_t)(i * m + j)] = wt;
    }
    return any;
}

// multi-shard image mode (reference conv.cpp:37-85 with d = 1, rep = 1, tau = identity):
//   in_channel(u, r, b) = u z + (b + r) % z,  out_channel(v, b) = (v z + b) % c_out
bool fused_plain_ms(int c_out, int m, int kappa, size_t s, const double* w, int v, int u, int r, long kk, long ll,
                    std::vector<double>& plain, const std::vector<int64_t>* tau = nullptr, int rep = 1) {
    // ImageConv::fused_plain (conv.cpp:69-85): in_channel(u, r, b) =
    // block_channel(u z + (b + r rep) mod z), out_channel(v, b) = (v z + b) mod c_out
    const size_t block = (size_t)m * m, z = s / block;
    const long h = kappa / 2;
    plain.assign(s, 0.0);
    bool any = false;
    for (size_t b = 0; b < z; ++b) {
        const size_t g = (size_t)u * z + (b + (size_t)r * (size_t)rep) % z;
        const size_t in_ch = tau ? (size_t)(*tau)[(g / (size_t)rep) % tau->size()] : g;
        const size_t out_ch = ((size_t)v * z + b) % (size_t)c_out;
        const double wt =
            w[((in_ch * c_out + out_ch) * kappa + (size_t)(kk + h)) * kappa + (size_t)(ll + h)] * 1.0;
        if (wt == 0.0) continue;
        any = true;
        const long i_lo = std::max(0L, -kk), i_hi = std::min<long>(m, m - kk);
        const long j_lo = std::max(0L, -ll), j_hi = std::min<long>(m, m - ll);
        for (long i = i_lo; i < i_hi; ++i)
            for (long j = j_lo; j < j_hi; ++j) plain[b * block + (size_t)(i * m + j)] = wt;
    }
    return any;
}

// channel-shard masks (reference conv.cpp:305-344): rows rr of a shard whose
// shifted source stays inside it (spill = 0) or comes from the neighbour shard
// (spill = 1), columns j in [max(0, -ll), min(m, m - ll))
bool cs_mask(int m, long rows, long kk, long ll, int spill, double w, size_t s, std::vector<double>& mask) {
    mask.assign(s, 0.0);
    const long j_lo = std::max(0L, -ll), j_hi = std::min<long>(m, m - ll);
    if (j_lo >= j_hi) return false;
    bool any = false;
    for (long rr = 0; rr < rows; ++rr) {
        const bool inside = rr + kk >= 0 && rr + kk < rows;
        if (inside == (spill != 0)) continue;
        any = true;
        for (long j = j_lo; j < j_hi; ++j) mask[(size_t)(rr * m + j)] = w;
    }
    return any;
}

void encode_rows(fhe_ctx* c, const double* z, size_t n, int level, double scale, int rows, uint64_t* dst) {
    const size_t N = c->N;
    int64_t* h = (int64_t*)c->stage(N * 8);
    ck(cudaStreamSynchronize(c->st), "sync");  // staging buffer reuse
    host::encode(z, n, N, scale, h);
    int64_t* dcoef = (int64_t*)c->alloc(N);
    ck(cudaMemcpyAsync(dcoef, h, N * 8, cudaMemcpyHostToDevice, c->st), "H2D");
    reduce_signed_rows(c->dc, dcoef, dst, rows, RowMap{rows, level, c->L, 0}, c->st);
    ntt_forward(c->dc, dst, rows, RowMap{rows, level, c->L, 0}, c->st);
    c->release(dcoef);
}

// Ledger replay of the reference schedule (conv.cpp:119-210) so the
// operation-count laws (test_conv.cpp:244-276) hold for the CKKS path too.
// Bias slot vectors of a layer, one per output shard: ImageConv::bias_plain
// (conv.cpp:87-94: bias[out_channel(v, b)] * scale over block b) for image
// mode, the constant bias[g] * scale of conv_channel_shards (conv.cpp:344) for
// output shard (g, v) of a channel-shard layer.
void set_bias(fhe_ctx* c, fhe_conv_layer* ly, const double* bias, double osc) {
    ly->bias_vecs.clear();
    if (!bias) return;
    const size_t s = c->slots(), block = (size_t)ly->m * ly->m;
    if (ly->cs) {
        for (int o = 0; o < ly->n_out; ++o) ly->bias_vecs.emplace_back(s, bias[o / ly->pc] * osc);
        return;
    }
    const size_t z = s / block;
    const int nout = ly->ms ? ly->n_out : 1;
    for (int v = 0; v < nout; ++v) {
        std::vector<double> plain(s, 0.0);
        for (size_t b = 0; b < z; ++b) {
            const double val = bias[((size_t)v * z + b) % (size_t)ly->c_out] * osc;
            std::fill_n(plain.begin() + (long)(b * block), block, val);
        }
        ly->bias_vecs.push_back(std::move(plain));
    }
}

// device bias rows [n_out][level][N] at level - 1 and `scale` (the conv output's
// scale); re-encoded in place when the scale changes, so captured graphs that
// read them stay valid. Host encoding synchronises: never call inside a capture.
void ensure_bias(fhe_ctx* c, const fhe_conv_layer* cly, double scale) {
    fhe_conv_layer* ly = const_cast<fhe_conv_layer*>(cly);
    if (ly->bias_vecs.empty() || (ly->d_bias && ly->d_bias_scale == scale)) return;
    const int rows = ly->level;
    const size_t rw = (size_t)rows * c->N;
    if (!ly->d_bias) ck(cudaMalloc(&ly->d_bias, ly->bias_vecs.size() * rw * 8), "cudaMalloc");
    for (size_t i = 0; i < ly->bias_vecs.size(); ++i)
        encode_rows(c, ly->bias_vecs[i].data(), c->slots(), ly->level - 1, scale, rows, ly->d_bias + i * rw);
    ck(cudaStreamSynchronize(c->st), "sync");
    ly->d_bias_scale = scale;
}

// the scale every input of a biased conv call shares (the bias is encoded at it)
void prepare_bias(fhe_ctx* c, const fhe_conv_layer* ly, const fhe_ct* const* cts, size_t n) {
    if (ly->bias_vecs.empty() || n == 0) return;
    for (size_t i = 1; i < n; ++i)
        if (cts[i]->scale != cts[0]->scale) fail(FHE_E_INVALID, "biased conv: inputs at different scales");
    ensure_bias(c, ly, cts[0]->scale);
}

void ledger_conv(fhe_ctx* c, const fhe_conv_layer* ly, int approach) {
    fhe_ledger& lg = c->ledger;
    const long m = ly->m, h = ly->kappa / 2;
    const uint64_t block = (uint64_t)m * m;
    bool have_acc = false;
    std::vector<int> shifted_done(ly->nk, 0);  // ChannelFirst caches shifted copies across r
    for (int r = 0; r < ly->c_in; ++r) {
        const uint64_t chan = c->reduce_amount((int64_t)r * block);
        bool have_partial = false;
        if (approach == 1) {
            int i = 0;
            for (long kk = -h; kk <= h; ++kk)
                for (long ll = -h; ll <= h; ++ll, ++i) {
                    if (!ly->nonempty[r * ly->nk + i]) continue;
                    if (!shifted_done[i]) {
                        const uint64_t a = c->reduce_amount(kk * m + ll);
                        c->note_amount(a);
                        if (a) lg.rotations++;
                        shifted_done[i] = 1;
                    }
                    c->note_amount(chan);
                    if (chan) lg.rotations++;
                    lg.ct_pt_mults++;
                    if (have_partial) lg.adds++;
                    have_partial = true;
                }
        } else {
            bool any = false;
            for (int i = 0; i < ly->nk; ++i) any |= ly->nonempty[r * ly->nk + i] != 0;
            if (!any) continue;
            c->note_amount(chan);
            if (chan) lg.rotations++;
            int batch = 0, i = 0;
            for (long kk = -h; kk <= h; ++kk)
                for (long ll = -h; ll <= h; ++ll, ++i)
                    if (ly->nonempty[r * ly->nk + i]) {
                        c->note_amount(c->reduce_amount(kk * m + ll));
                        ++batch;
                    }
            lg.hoist_groups++;
            lg.hoisted_rotations += batch;
            for (int k = 0; k < batch; ++k) {
                lg.ct_pt_mults++;
                if (have_partial) lg.adds++;
                have_partial = true;
            }
        }
        if (have_partial) {
            if (have_acc) lg.adds++;
            have_acc = true;
        }
    }
    if (!have_acc) {
        c->note_amount(0);
        lg.ct_pt_mults++;
    }
}

// Rotated plaintexts of the BSGS schedules, encoded once.
fhe_conv_layer::Bsgs& ensure_bsgs(fhe_ctx* c, const fhe_conv_layer* cly, int orient) {
    fhe_conv_layer* ly = const_cast<fhe_conv_layer*>(cly);
    fhe_conv_layer::Bsgs& B = ly->bs[orient - 3];
    if (B.ready) return B;
    const long m = ly->m, h = ly->kappa / 2;
    const int64_t block = (int64_t)m * m;
    std::vector<int64_t> chan, shift;
    for (int r = 0; r < ly->c_in; ++r) chan.push_back((int64_t)r * block);
    for (long kk = -h; kk <= h; ++kk)
        for (long ll = -h; ll <= h; ++ll) shift.push_back(kk * m + ll);
    const int kap = (int)(2 * h + 1);
    if (orient == 5) {
        B.bamt.clear();
        B.gamt.clear();
        for (int r = 0; r < ly->c_in; ++r)
            for (long ll = -h; ll <= h; ++ll) B.bamt.push_back((int64_t)r * block + ll);
        for (long kk = -h; kk <= h; ++kk) B.gamt.push_back(kk * m);
    } else {
        B.bamt = orient == 3 ? chan : shift;
        B.gamt = orient == 3 ? shift : chan;
    }
    B.nb = (int)B.bamt.size();
    B.ngi = (int)B.gamt.size();
    if (orient != 5 && B.nb > kMaxBaby) fail(FHE_E_INVALID, "too many baby steps for the BSGS schedule");
    const int ne = c->ne_at(ly->level);
    const size_t extw = (size_t)ne * c->N, s = c->slots();
    ck(cudaMalloc(&B.d_pts, (size_t)B.ngi * B.nb * extw * 8), "cudaMalloc");
    B.nonempty.assign((size_t)B.ngi * B.nb, 0);
    const double pscale = (double)c->primes[ly->level];
    std::vector<double> plain, rot(s);
    for (int gi = 0; gi < B.ngi; ++gi)
        for (int bi = 0; bi < B.nb; ++bi) {
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
            if (!fused_plain(ly->c_in, ly->c_out, ly->m, ly->kappa, s, ly->weights.data(), r, kk, ll, plain))
                continue;
            B.nonempty[(size_t)gi * B.nb + bi] = 1;
            const uint64_t g = c->reduce_amount(B.gamt[gi]);
            for (size_t j = 0; j < s; ++j) rot[j] = plain[(j + s - g) % s];  // rot_{-g}
            encode_rows(c, rot.data(), s, ly->level, pscale, ne, B.d_pts + ((size_t)gi * B.nb + bi) * extw);
        }
    ck(cudaStreamSynchronize(c->st), "sync");
    B.ready = true;
    return B;
}

// Operand-form copies for the fused baby steps (k_bsgs_tma): a copy of
// the layer's rotated plaintexts and of every baby-step key in limb form. Built once
// (host-synchronising, so batch_impl calls it before a graph capture); keygen drops
// the key copies with the keys.
bool limb_ok(const fhe_ctx* c, const fhe_conv_layer::Bsgs& B) { return c->limb && B.nb <= kMaxFused; }
// giants of the limb plaintext set, rounded up so that every launch's plaintext box
// (3 giants when a launch has <= 3, else kFusedMaxG) stays inside the tensor
int limb_giants(int ngi) { return ngi <= 3 ? 3 : (ngi + kFusedMaxG - 1) / kFusedMaxG * kFusedMaxG; }

void prepare_limb(fhe_ctx* c, const fhe_conv_layer* ly, int orient) {
    if (orient != 5) return;
    fhe_conv_layer::Bsgs& B = ensure_bsgs(c, ly, orient);
    if (!limb_ok(c, B)) return;
    bool dirty = false;
    const int ne = c->ne_at(ly->level);
    if (!B.d_pts_limb) {
        // padded (zero rows) to the giant count the TMA plaintext boxes of the launches span
        const size_t rows = (size_t)B.ngi * B.nb * ne, prow = (size_t)limb_giants(B.ngi) * B.nb * ne;
        ck(cudaMalloc(&B.d_pts_limb, prow * c->N * 8), "cudaMalloc");
        ck(cudaMemsetAsync(B.d_pts_limb + rows * c->N, 0, (prow - rows) * c->N * 8, c->st), "memset");
        rows_to_limb(c->dc, B.d_pts_limb, B.d_pts, rows, RowMap{ne, ly->level, c->L, 0}, c->st);
        dirty = true;
    }
    if (!B.d_keys_limb || B.limb_gen != c->key_gen) {
        std::vector<const uint64_t*> src;
        std::vector<int> kidx(B.nb, -1);
        for (int b = 0; b < B.nb; ++b) {
            const uint32_t g = c->galois_of(c->reduce_amount(B.bamt[b]));
            if (g == 1) continue;
            kidx[b] = (int)src.size();
            src.push_back(c->key_for(g));
        }
        const size_t rows = (size_t)c->dnum * 2 * c->np;
        if (B.d_keys_limb) {
            ck(cudaStreamSynchronize(c->main_st), "sync");
            cudaFree(B.d_keys_limb);
            B.d_keys_limb = nullptr;
        }
        ck(cudaMalloc(&B.d_keys_limb, std::max<size_t>(1, src.size()) * rows * c->N * 8), "cudaMalloc");
        for (size_t t = 0; t < src.size(); ++t)
            rows_to_limb(c->dc, B.d_keys_limb + t * rows * c->N, src[t], rows, RowMap{c->np, -1, c->L, 0}, c->st);
        B.kidx = kidx;
        B.limb_gen = c->key_gen;
        dirty = true;
    }
    if (dirty) ck(cudaStreamSynchronize(c->st), "limb operands");
}

// Operand-form plaintexts and second-level keys of the paper schedules (approach 1:
// channel rotations r m^2, approach 2: shifts) for conv_paper_batch on k_bsgs_tma.
// Built once per layer (keys again after a keygen), host-synchronising: batch_impl
// calls it before a graph capture.
bool paper_opf_ok(const fhe_ctx* c, const fhe_conv_layer* ly) { return c->limb && !ly->ms && !ly->cs; }
void prepare_paper(fhe_ctx* c, const fhe_conv_layer* ly, int approach) {
    if ((approach != 1 && approach != 2) || !paper_opf_ok(c, ly)) return;
    fhe_conv_layer* L = const_cast<fhe_conv_layer*>(ly);
    const int ne = c->ne_at(ly->level);
    bool dirty = false;
    if (!L->d_pts_opf) {
        const size_t rows = (size_t)ly->c_in * ly->nk * ne;
        ck(cudaMalloc(&L->d_pts_opf, rows * c->N * 8), "cudaMalloc");
        rows_to_limb(c->dc, L->d_pts_opf, ly->d_pts, rows, RowMap{ne, ly->level, c->L, 0}, c->st);
        dirty = true;
    }
    fhe_conv_layer::PaperKeys& P = L->pk[approach - 1];
    const long m = ly->m, h = ly->kappa / 2;
    const int nsecond = approach == 2 ? ly->nk : ly->c_in;
    auto amt_of = [&](int x) {
        return approach == 2 ? (int64_t)(x / (2 * h + 1) - h) * m + (x % (2 * h + 1) - h) : (int64_t)x * m * m;
    };
    bool stale = !P.d_keys || P.gen != c->key_gen || (int)P.kidx.size() != nsecond;
    for (int x = 0; !stale && x < nsecond; ++x) {  // a key generated since the copies were built
        const uint32_t g = c->galois_of(c->reduce_amount(amt_of(x)));
        stale = g != 1 && P.kidx[x] < 0 && c->keys.count(g);
    }
    if (stale) {
        std::vector<const uint64_t*> src;
        P.kidx.assign(nsecond, -1);
        for (int x = 0; x < nsecond; ++x) {
            const uint32_t g = c->galois_of(c->reduce_amount(amt_of(x)));
            if (g == 1 || !c->keys.count(g)) continue;  // a missing key fails later, in key_for
            P.kidx[x] = (int)src.size();
            src.push_back(c->key_for(g));
        }
        const size_t rows = (size_t)c->dnum * 2 * c->np;
        if (P.d_keys) {
            ck(cudaStreamSynchronize(c->main_st), "sync");
            cudaFree(P.d_keys);
            P.d_keys = nullptr;
        }
        ck(cudaMalloc(&P.d_keys, std::max<size_t>(1, src.size()) * rows * c->N * 8), "cudaMalloc");
        for (size_t t = 0; t < src.size(); ++t)
            rows_to_limb(c->dc, P.d_keys + t * rows * c->N, src[t], rows, RowMap{c->np, -1, c->L, 0}, c->st);
        P.gen = c->key_gen;
        dirty = true;
    }
    if (dirty) ck(cudaStreamSynchronize(c->st), "paper operands");
}

// Work-queue rows of k_bsgs_tma at a level: the integer-path (q >= 2^50) extended rows
// first, then the FP64 rows (kernels.cuh TmaMaps)
void tma_rows(fhe_ctx* c, int level, TmaMaps& tm) {
    const int nr = level + 1, ne = nr + c->K;
    int n = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int u = 0; u < ne; ++u) {
            const uint64_t q = c->primes[u < nr ? u : c->L + (u - nr)];
            if ((q >= (1ULL << 50)) == (pass == 0)) tm.rowlist[n++] = (uint8_t)u;
            if (pass == 0 && u == ne - 1) tm.nint = n;
        }
    // one work-queue slot per compute stream (main, lanes): launches on different streams
    // may overlap; allocated with the context tables (never inside a graph capture)
    int slot = 0;
    for (size_t i = 0; i < c->lanes.size(); ++i)
        if (c->st == c->lanes[i]) slot = 1 + (int)(i % (kTmaSchedSlots - 1));
    tm.sched = c->d_sched + (size_t)slot * kTmaSchedWords;
}

// Baby steps of the fused BSGS schedule for nsrc sources: Y_g(s) for every
// giant g (chunks of kFusedMaxG giants per launch), X~_b never materialised.
// limb: digits are limb-form ModUp digits and cts the limb-form P-scaled
// ciphertexts (ct_prescale); keys and plaintexts come from prepare_limb.
void fused_babies(fhe_ctx* c, const fhe_conv_layer::Bsgs& B, int level, const uint64_t* digits, size_t dstride,
                  const uint64_t* cts, size_t ctstride, int nsrc, uint64_t* Y, size_t ystride, bool limb = false) {
    const int nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t extw = (size_t)ne * c->N;
    if (limb && !(limb_ok(c, B) && B.d_pts_limb && B.d_keys_limb && B.limb_gen == c->key_gen))
        fail(FHE_E_RUNTIME, "limb operands not prepared");
    const size_t keyw = (size_t)c->dnum * 2 * c->np * c->N;
    TmaMaps tm{};
    const bool tma = limb && c->tma;
    if (tma) {  // tensor maps of this launch's operands (kernels.cuh TmaMaps)
        tma_rows(c, level, tm);
        if (nsrc > 1 && (dstride != (size_t)dn * extw || ctstride != (size_t)2 * nr * c->N))
            fail(FHE_E_RUNTIME, "tma staging needs dense digit / ciphertext batches");
        const uint32_t sg = (uint32_t)tma_sources(nsrc), P2 = 256u / sg;
        const uint64_t N = c->N;
        uint64_t nkeys = 0;
        for (int v : B.kidx) nkeys += v >= 0;
        const uint64_t dk[4] = {N, (uint64_t)c->np, 2ull * c->dnum, std::max<uint64_t>(1, nkeys)};
        const uint32_t bk[4] = {P2, 1, 2u * dn, 1};
        tma_map4(&tm.key, B.d_keys_limb, dk, bk);
        const uint64_t dd[5] = {N, (uint64_t)ne, (uint64_t)dn, 1, (uint64_t)nsrc};
        const uint32_t bd[5] = {P2, 1, (uint32_t)dn, 1, sg};
        tma_map5(&tm.dig, digits, dd, bd);
        const uint64_t dc5[5] = {N, (uint64_t)nr, 2, 1, (uint64_t)nsrc};
        const uint32_t bc[5] = {P2, 1, 2, 1, sg};
        tma_map5(&tm.ct, cts, dc5, bc);
    }
    FusedBsgs f{};
    f.nsrc = nsrc;
    f.digits = digits;
    f.digit_src_stride = dstride;
    f.ct = cts;
    f.ct_src_stride = ctstride;
    f.pt_g_stride = (size_t)B.nb * extw;
    f.y_src_stride = ystride;
    f.y_g_stride = 2 * extw;
    for (int b = 0; b < B.nb; ++b) {
        bool any = false;
        for (int g = 0; g < B.ngi; ++g) any |= B.nonempty[(size_t)g * B.nb + b] != 0;
        if (any && c->reduce_amount(B.bamt[b]) != 0) c->ledger.key_switches += nsrc;
    }
    // more than kMaxFused baby steps (large c kappa): several launches per giant chunk,
    // the later ones continuing the accumulators (the accumulating variant holds <= 3 giants)
    const bool chunked = B.nb > kMaxFused;
    const int gstep = chunked ? 3 : kFusedMaxG;
    for (int g0 = 0; g0 < B.ngi; g0 += gstep) {
        const int ng = std::min(gstep, B.ngi - g0);
        f.ng = ng;
        tm.g0 = g0;
        if (tma) {  // the plaintext box spans the kernel's NG giants (3 when ng <= 3, else kFusedMaxG)
            const uint64_t dp[4] = {(uint64_t)c->N, (uint64_t)ne, (uint64_t)B.nb, (uint64_t)limb_giants(B.ngi)};
            const uint32_t bp[4] = {256u / (uint32_t)tma_sources(nsrc), 1, 1, ng <= 3 ? 3u : (uint32_t)kFusedMaxG};
            tma_map4(&tm.pt, B.d_pts_limb, dp, bp);
        }
        f.Y = Y + (size_t)g0 * 2 * extw;
        std::vector<int> active;
        for (int b = 0; b < B.nb; ++b)
            for (int g = 0; g < ng; ++g)
                if (B.nonempty[(size_t)(g0 + g) * B.nb + b]) {
                    active.push_back(b);
                    break;
                }
        if (active.empty()) {  // no term feeds these giants: their accumulators are zero
            for (int s2 = 0; s2 < nsrc; ++s2)
                ck(cudaMemsetAsync(f.Y + (size_t)s2 * ystride, 0, (size_t)ng * 2 * extw * 8, c->st), "memset");
            continue;
        }
        for (size_t a0 = 0; a0 < active.size(); a0 += kMaxFused) {
            f.nb = 0;
            f.accumulate = a0 > 0;
            double pt_words = 0, keyed = 0;
            for (size_t ai = a0; ai < active.size() && f.nb < kMaxFused; ++ai) {
                const int b = active[ai];
                uint32_t mask = 0;
                for (int g = 0; g < ng; ++g)
                    if (B.nonempty[(size_t)(g0 + g) * B.nb + b]) mask |= 1u << g;
                const uint32_t gal = c->galois_of(c->reduce_amount(B.bamt[b]));
                f.galois[f.nb] = gal;
                f.key[f.nb] = gal == 1 ? nullptr : limb ? B.d_keys_limb + (size_t)B.kidx[b] * keyw : c->key_for(gal);
                tm.kidx[f.nb] = (int16_t)(gal == 1 || !limb ? -1 : B.kidx[b]);
                tm.bidx[f.nb] = (int16_t)b;
                f.gmask[f.nb] = mask;
                f.pt[f.nb] = (limb ? B.d_pts_limb : B.d_pts) + ((size_t)g0 * B.nb + b) * extw;
                f.srcslot[f.nb] = 0;
                pt_words += __builtin_popcount(mask);
                if (gal != 1) keyed += 1;
                f.nb++;
            }
            c->timed("bsgs_fused",
                     c->rows(keyed * 2.0 * dn * ne + pt_words * ne +
                             nsrc * ((double)dn * ne + 2.0 * nr + (f.accumulate ? 4.0 : 2.0) * ng * ne)),
                     [&] {
                         if (tma)
                             bsgs_tma(c->dc, f, tm, level, dn, c->st);
                         else
                             bsgs_fused(c->dc, f, c->d_md, level, dn, c->st);
                     });
        }
    }
}

void conv_bsgs(fhe_ctx* c, const fhe_ct* ct, const fhe_conv_layer* ly, int orient, fhe_ct* out) {
    fhe_conv_layer::Bsgs& B = ensure_bsgs(c, ly, orient);
    const int level = ct->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N;
    uint64_t* dsrc = c->alloc((size_t)dn * extw);
    uint64_t* Y = c->alloc((size_t)B.ngi * 2 * extw);
    const bool fused = orient == 5;
    uint64_t* XT = fused ? nullptr : c->alloc((size_t)B.nb * 2 * extw);
    prepare_limb(c, ly, orient);
    const bool limb = fused && limb_ok(c, B);
    modup_batch(c, ct->c1(), 0, 1, level, dsrc, limb);
    if (limb) {
        uint64_t* pc = c->alloc((size_t)2 * nr * N);
        ct_prescale(c->dc, pc, ct->d, 0, 1, c->d_md, level, c->st);
        fused_babies(c, B, level, dsrc, 0, pc, 0, 1, Y, 0, true);
        c->release(pc);
    } else if (fused) {
        fused_babies(c, B, level, dsrc, 0, ct->d, 0, 1, Y, 0);
    }
    // baby steps: the hoisted key switches of the source, then the plaintext mat-vec
    BabyTerms t{};
    t.nb = B.nb;
    t.nb_total = B.nb;
    t.pts = B.d_pts;
    for (int b = 0; !fused && b < B.nb; ++b) {
        const uint32_t g = c->galois_of(c->reduce_amount(B.bamt[b]));
        t.galois[b] = g;
        t.key[b] = g == 1 ? nullptr : c->key_for(g);
        uint32_t any = 0;
        for (int gi = 0; gi < B.ngi; ++gi) any |= B.nonempty[(size_t)gi * B.nb + b] ? 1u : 0u;
        t.gmask[b] = any;
        if (g != 1 && any) c->ledger.key_switches++;
    }
    if (!fused) {
        KsStream ks{};
        ks.digits = dsrc;
        ks.digit_stride = 0;
        ks.out = XT;
        for (int b = 0; b < B.nb; ++b) {
            if (!t.gmask[b]) continue;
            if (t.galois[b] == 1) {
                c->timed("ks_multi", c->rows(2.0 * nr + 2.0 * ne), [&] { identity_term(c->dc, XT + (size_t)b * 2 * extw, ct->d, c->d_md, level, c->st); });
                continue;
            }
            ks.galois[ks.n] = t.galois[b];
            ks.key[ks.n] = t.key[b];
            ks.c0[ks.n] = ct->c0();
            ks.slot[ks.n] = b;
            ks.n++;
        }
        c->timed("ks_multi", c->rows((double)ks.n * (2.0 * dn * ne + 2.0 * ne) + (double)dn * ne + nr), [&] { ks_stream(c->dc, ks, 0, c->d_md, level, dn, c->st); });
    }
    for (int g0 = 0; !fused && g0 < B.ngi; g0 += kMaxGiant) {
        t.ngi = std::min(kMaxGiant, B.ngi - g0);
        t.g0 = g0;
        double pt_pairs = 0;
        for (int b = 0; b < B.nb; ++b) {
            uint32_t mask = 0;
            for (int gi = 0; gi < t.ngi; ++gi)
                if (B.nonempty[(size_t)(g0 + gi) * B.nb + b]) mask |= 1u << gi;
            t.gmask[b] = mask;
            pt_pairs += __builtin_popcount(mask);
        }
        c->timed("pt_matvec", c->rows(pt_pairs * ne + 2.0 * B.nb * ne + 2.0 * t.ngi * ne), [&] { pt_matvec(c->dc, Y + (size_t)g0 * 2 * extw, XT, t, level, c->st); });
    }
    // giant steps: ModDown each aggregated Y_g, ModUp, key-switch-accumulate
    uint64_t* acc = c->alloc(2 * extw);
    ck(cudaMemsetAsync(acc, 0, 2 * extw * 8, c->st), "memset");
    std::vector<int> giants;
    int id = -1;
    for (int gi = 0; gi < B.ngi; ++gi) {
        bool any = false;
        for (int b = 0; b < B.nb; ++b) any |= B.nonempty[(size_t)gi * B.nb + b] != 0;
        if (!any) continue;
        if (c->reduce_amount(B.gamt[gi]) == 0)
            id = gi;
        else
            giants.push_back(gi);
    }
    // giant steps: only Y_g.c1 is brought down to Q (for the decomposition);
    // Y_g.c0 stays P-scaled in QP and enters the accumulator directly.
    // ModDown(Y_g.c1) is evaluated in the coefficient domain, which is exactly
    // what the ModUp that follows consumes:
    //   coef(ModDown(y)) = (INTT(y_Q) - conv_P->Q(INTT(y_P))) P^-1,
    // so all giants go through one INTT, one conversion kernel, one ModUp
    // conversion and one forward NTT (the own-digit rows are transformed too).
    if (!giants.empty()) {
        const int Gall = (int)giants.size();
        const size_t dw = (size_t)dn * extw;
        // giants in chunks sized so that a chunk's digits stay L2-resident
        // between the ModUp NTT passes and the key-switch accumulation
        const int GC = std::max(1, std::min(Gall, c->giant_chunk));
        uint64_t* yc = c->alloc((size_t)GC * extw);       // [G][ne][N] Y_g.c1, then its INTT
        uint64_t* yq = c->alloc((size_t)GC * nr * N);     // [G][nr][N] coef(ModDown(Y_g.c1))
        uint64_t* dg = c->alloc((size_t)GC * dw);         // [G][dn][ne][N] ModUp digits
        for (int g0 = 0; g0 < Gall; g0 += GC) {
            const int G = std::min(GC, Gall - g0);
            for (int s = 0; s < G; ++s)
                ck(cudaMemcpyAsync(yc + (size_t)s * extw, Y + (size_t)giants[g0 + s] * 2 * extw + extw, extw * 8,
                                   cudaMemcpyDeviceToDevice, c->st),
                   "memcpy");
            c->timed("ntt", c->rows(2.0 * G * ne),
                     [&] { ntt_inverse(c->dc, yc, G * ne, RowMap{ne, level, c->L, 0}, c->st); });
            c->timed("moddown", c->rows((double)G * (ne + nr)),
                     [&] { moddown_coef(c->dc, yq, yc, c->d_md, level, G, c->st); });
            c->ledger.moddowns += G;
            c->timed("ntt_modup", c->rows((double)G * nr + (double)G * dn * ne), [&] {
                ntt_modup_coef(c->dc, dg, yq, G, c->d_modup + (size_t)level * c->dnum, level, dn, c->st);
            });
            c->ledger.modups += G;
            KsBatch ks{};
            ks.n = G;
            ks.nsrc = 1;
            ks.digits = dg;
            ks.digit_term_stride = dw;
            ks.c0 = Y;
            ks.c0_qp = 1;
            ks.out = acc;
            for (int s = 0; s < G; ++s) {
                const int gi = giants[g0 + s];
                const uint32_t g = c->galois_of(c->reduce_amount(B.gamt[gi]));
                ks.galois[s] = g;
                ks.key[s] = c->key_for(g);
                ks.c0_off[s] = (size_t)gi * 2 * extw;
                c->ledger.key_switches++;
            }
            c->timed("ks_inner", c->rows((double)ks.n * (3.0 * dn * ne + ne) + 4.0 * ne),
                     [&] { ks_batch(c->dc, ks, 1, c->d_md, level, dn, c->st); });
        }
        c->release(dg);
        c->release(yq);
        c->release(yc);
    }
    if (id >= 0) qp_add(c->dc, acc, Y + (size_t)id * 2 * extw, level, c->st);
    uint64_t* md = nullptr;
    moddown_rescale(c, acc, extw, level, 2, out->d, ly->d_bias, 1);
    out->scale = (ct->scale * (double)c->primes[level]) / (double)c->primes[level];
    out->depth = ct->depth + 1;
    c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, out->depth);
    // ledger: one hoisted baby group + one rotation per giant step
    fhe_ledger& lg = c->ledger;
    lg.hoist_groups++;
    for (int b = 0; b < B.nb; ++b) {
        c->note_amount(c->reduce_amount(B.bamt[b]));
        lg.hoisted_rotations++;
    }
    for (int gi : giants) {
        c->note_amount(c->reduce_amount(B.gamt[gi]));
        lg.rotations++;
    }
    uint64_t pairs = 0;
    for (int v : B.nonempty) pairs += v;
    lg.ct_pt_mults += pairs;
    lg.adds += pairs ? pairs - 1 : 0;
    c->release(md);
    c->release(acc);
    c->release(Y);
    if (XT) c->release(XT);
    c->release(dsrc);
}

// Giant steps and the final fused ModDown + rescale for S accumulator sets
// Y = [S][ngi][2][ne][N] (source stride ys): giant gi of `giants` (amount
// gamt[gi]) is key-switched as KS(Y.c1) + sigma(Y.c0) into the source's QP
// accumulator (ModDown(Y.c1) in the coefficient domain feeding a batched
// ModUp), the identity giant `id` is added as is; md = [S][2][level][N].
void giants_finish(fhe_ctx* c, const uint64_t* Y, size_t ys, int S, int level, const std::vector<int>& giants_in,
                   const std::vector<int64_t>& gamt, int id, uint64_t* md, const uint64_t* bias = nullptr,
                   int bias_mod = 1) {
    const int nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, dw = (size_t)dn * extw;
    // a giant whose amount is a multiple of the slot count (single-row channel shards:
    // kk m = kk slots) is the identity: its accumulator is added, not key-switched
    std::vector<int> giants, idg;
    if (id >= 0) idg.push_back(id);
    for (int g : giants_in) (c->reduce_amount(gamt[g]) == 0 ? idg : giants).push_back(g);
    uint64_t* acc = c->alloc((size_t)S * 2 * extw);
    ck(cudaMemsetAsync(acc, 0, (size_t)S * 2 * extw * 8, c->st), "memset");
    const int GT = (int)giants.size();
    // giants in chunks of at most kMaxBaby (the KsBatch term capacity); every
    // chunk accumulates into the same QP accumulators
    for (int gb = 0; gb < GT; gb += kMaxBaby) {
        const int G = std::min(kMaxBaby, GT - gb);
        const int SC = std::max(1, std::min(S, 8));
        uint64_t* yc = c->alloc((size_t)SC * G * extw);
        uint64_t* yq = c->alloc((size_t)SC * G * nr * N);
        uint64_t* dg = c->alloc((size_t)SC * G * dw);
        // operand-form key switches (k_ks_giant_opf): digits, keys and the giants' QP c0
        // rows in operand form
        const bool opf = c->limb;
        uint64_t* yc0 = opf ? c->alloc((size_t)SC * G * extw) : nullptr;
        for (int s0 = 0; s0 < S; s0 += SC) {
            const int sc = std::min(SC, S - s0);
            GiantSel gsel{};
            gsel.n = G;
            for (int gi = 0; gi < G; ++gi) gsel.idx[gi] = giants[gb + gi];
            giant_gather(c->dc, yc, yc0, Y + (size_t)s0 * ys, ys, sc, gsel, level, c->st);
            const int np_ = sc * G;
            c->timed("ntt", c->rows(2.0 * np_ * ne),
                     [&] { ntt_inverse(c->dc, yc, np_ * ne, RowMap{ne, level, c->L, 0}, c->st); });
            c->timed("moddown", c->rows((double)np_ * (ne + nr)),
                     [&] { moddown_coef(c->dc, yq, yc, c->d_md, level, np_, c->st); });
            c->timed("ntt_modup", c->rows((double)np_ * nr + (double)np_ * dn * ne), [&] {
                ntt_modup_coef(c->dc, dg, yq, np_, c->d_modup + (size_t)level * c->dnum, level, dn, c->st,
                               opf ? 1 : 0);
            });
            c->ledger.moddowns += np_;
            c->ledger.modups += np_;
            KsBatch kg{};
            kg.nsrc = sc;
            kg.n = G;
            kg.digits = dg;
            kg.digit_src_stride = (size_t)G * dw;
            kg.digit_term_stride = dw;
            kg.c0 = opf ? yc0 : Y + (size_t)s0 * ys;
            kg.c0_src_stride = opf ? (size_t)G * extw : ys;
            kg.c0_qp = 1;
            kg.opf = opf ? 1 : 0;
            kg.out = acc + (size_t)s0 * 2 * extw;
            kg.out_src_stride = 2 * extw;
            for (int gi = 0; gi < G; ++gi) {
                const uint32_t g = c->galois_of(c->reduce_amount(gamt[giants[gb + gi]]));
                kg.galois[gi] = g;
                kg.key[gi] = opf ? c->key_opf_for(g) : c->key_for(g);
                kg.c0_off[gi] = opf ? (size_t)gi * extw : (size_t)giants[gb + gi] * 2 * extw;
            }
            c->ledger.key_switches += (uint64_t)G * sc;
            c->timed("ks_inner", c->rows((double)G * 2.0 * dn * ne + (double)sc * G * (dn * ne + ne) + 4.0 * ne * sc),
                     [&] { ks_batch(c->dc, kg, 1, c->d_md, level, dn, c->st); });
        }
        c->release(yc0);
        c->release(dg);
        c->release(yq);
        c->release(yc);
    }
    for (int g : idg)  // one launch per identity giant for all S accumulators
        qp_add(c->dc, acc, Y + (size_t)g * 2 * extw, level, c->st, S, 2 * extw, ys);
    moddown_rescale(c, acc, extw, level, 2 * S, md, bias, bias_mod);
    c->release(acc);
}

// Batched BSGS conv of S ciphertexts through one layer: every key and every
// plaintext is streamed once per batch (the lanes of a warp that share a
// coefficient pair share the loads), ModUps/NTTs run over the whole batch.
void conv_bsgs_batch(fhe_ctx* c, const fhe_ct* const* cts, int S, const fhe_conv_layer* ly, int orient,
                     fhe_ct* const* outs) {
    fhe_conv_layer::Bsgs& B = ensure_bsgs(c, ly, orient);
    const int level = cts[0]->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
    for (int s = 0; s < S; ++s) {
        if (cts[s]->level != level || outs[s]->level != level - 1)
            fail(FHE_E_INVALID, "batched conv: all inputs must share the layer level");
    }
    uint64_t* buf = c->alloc((size_t)S * ctw);
    for (int s = 0; s < S; ++s)
        ck(cudaMemcpyAsync(buf + (size_t)s * ctw, cts[s]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    uint64_t* dsrc = c->alloc((size_t)S * dw);
    const bool fused = orient == 5;
    prepare_limb(c, ly, orient);
    const bool limb = fused && limb_ok(c, B);
    modup_batch(c, buf + (size_t)nr * N, ctw, S, level, dsrc, limb);
    // baby steps
    const size_t xts = (size_t)B.nb * 2 * extw, ys = (size_t)B.ngi * 2 * extw;
    uint64_t* Y = c->alloc((size_t)S * ys);
    uint64_t* XT = fused ? nullptr : c->alloc((size_t)S * xts);
    if (limb) {  // the P-scaled ciphertexts in limb form replace buf for the baby steps
        ct_prescale(c->dc, buf, buf, ctw, S, c->d_md, level, c->st);
        fused_babies(c, B, level, dsrc, dw, buf, ctw, S, Y, ys, true);
    } else if (fused) {
        fused_babies(c, B, level, dsrc, dw, buf, ctw, S, Y, ys);
    }
    BabyTerms t{};
    t.nb = B.nb;
    t.nb_total = B.nb;
    t.pts = B.d_pts;
    KsBatch kb{};
    kb.nsrc = S;
    kb.digits = dsrc;
    kb.digit_src_stride = dw;
    kb.c0 = buf;
    kb.c0_src_stride = ctw;
    kb.out = XT;
    kb.out_src_stride = xts;
    for (int b = 0; !fused && b < B.nb; ++b) {
        const uint32_t g = c->galois_of(c->reduce_amount(B.bamt[b]));
        t.galois[b] = g;
        t.key[b] = g == 1 ? nullptr : c->key_for(g);
        uint32_t any = 0;
        for (int gi = 0; gi < B.ngi; ++gi) any |= B.nonempty[(size_t)gi * B.nb + b] ? 1u : 0u;
        t.gmask[b] = any;
        if (!any) continue;
        if (g == 1) {
            c->timed("ks_multi", c->rows((2.0 * nr + 2.0 * ne) * S), [&] {
                identity_batch(c->dc, XT + (size_t)b * 2 * extw, xts, buf, ctw, c->d_md, level, S, c->st);
            });
            continue;
        }
        kb.galois[kb.n] = g;
        kb.key[kb.n] = t.key[b];
        kb.slot[kb.n] = b;
        kb.n++;
        c->ledger.key_switches += S;
    }
    if (!fused)
        c->timed("ks_multi", c->rows((double)kb.n * (2.0 * dn * ne + 2.0 * ne * S) + ((double)dn * ne + nr) * S),
                 [&] { ks_batch(c->dc, kb, 0, c->d_md, level, dn, c->st); });
    for (int g0 = 0; !fused && g0 < B.ngi; g0 += kMaxGiant) {
        t.ngi = std::min(kMaxGiant, B.ngi - g0);
        t.g0 = g0;
        double pt_pairs = 0;
        for (int b = 0; b < B.nb; ++b) {
            uint32_t mask = 0;
            for (int gi = 0; gi < t.ngi; ++gi)
                if (B.nonempty[(size_t)(g0 + gi) * B.nb + b]) mask |= 1u << gi;
            t.gmask[b] = mask;
            pt_pairs += __builtin_popcount(mask);
        }
        c->timed("pt_matvec", c->rows(pt_pairs * ne + (2.0 * B.nb * ne + 2.0 * t.ngi * ne) * S), [&] {
            pt_matvec_batch(c->dc, Y + (size_t)g0 * 2 * extw, ys, XT, xts, t, level, S, c->st);
        });
    }
    if (XT) c->release(XT);
    c->release(dsrc);
    // giant steps, in source chunks (bounds the digit buffers)
    std::vector<int> giants;
    int id = -1;
    for (int gi = 0; gi < B.ngi; ++gi) {
        bool any = false;
        for (int b = 0; b < B.nb; ++b) any |= B.nonempty[(size_t)gi * B.nb + b] != 0;
        if (!any) continue;
        if (c->reduce_amount(B.gamt[gi]) == 0)
            id = gi;
        else
            giants.push_back(gi);
    }
    const size_t otw = (size_t)2 * level * N;
    uint64_t* md = c->alloc((size_t)S * otw);
    giants_finish(c, Y, ys, S, level, giants, B.gamt, id, md, ly->d_bias, 1);
    for (int s = 0; s < S; ++s) {
        ck(cudaMemcpyAsync(outs[s]->d, md + (size_t)s * otw, otw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        outs[s]->scale = (cts[s]->scale * (double)c->primes[level]) / (double)c->primes[level];
        outs[s]->depth = cts[s]->depth + 1;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, outs[s]->depth);
    }
    fhe_ledger& lg = c->ledger;
    uint64_t pairs = 0;
    for (int v : B.nonempty) pairs += v;
    for (int s = 0; s < S; ++s) {
        lg.hoist_groups++;
        for (int b = 0; b < B.nb; ++b) {
            c->note_amount(c->reduce_amount(B.bamt[b]));
            lg.hoisted_rotations++;
        }
        for (int gi : giants) {
            c->note_amount(c->reduce_amount(B.gamt[gi]));
            lg.rotations++;
        }
        lg.ct_pt_mults += pairs;
        lg.adds += pairs ? pairs - 1 : 0;
    }
    c->release(md);
    c->release(Y);
    c->release(buf);
}

// The paper's schedules for a batch of S ciphertexts:
// approach 2 rotates every input by the channel amounts r m^2 first, approach
// 1 by the stencil shifts first (the first-level rotations, hoisted from one
// ModUp, keys shared by the batch, ModDown'd to ciphertexts); every rotated
// copy is ModUp'd and its second-level rotations are key-switched and
// multiplied by the layer's plaintexts inside the fused baby-step kernel
// (one accumulator, no giant step), so the per-copy key switches never touch
// memory. One fused ModDown + rescale per output.
void conv_paper_batch(fhe_ctx* c, const fhe_ct* const* cts, int S, const fhe_conv_layer* ly, int approach,
                      fhe_ct* const* outs) {
    const int level = cts[0]->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
    for (int s = 0; s < S; ++s)
        if (cts[s]->level != level || outs[s]->level != level - 1)
            fail(FHE_E_INVALID, "batched conv: all inputs must share the layer level");
    const int nk = ly->nk, cin = ly->c_in;
    const long m = ly->m, h = ly->kappa / 2;
    const int64_t block = (int64_t)m * m;
    auto shift_amt = [&](int i) { return (int64_t)(i / (2 * h + 1) - h) * m + (i % (2 * h + 1) - h); };
    auto nonempty = [&](int r, int i) { return ly->nonempty[(size_t)r * nk + i] != 0; };
    // first level: approach 2 -> channels r (amount r m^2), approach 1 -> shifts i
    const int nfirst = approach == 2 ? cin : nk, nsecond = approach == 2 ? nk : cin;
    auto rpos = [&](int f, int x) { return approach == 2 ? std::make_pair(f, x) : std::make_pair(x, f); };
    auto first_amt = [&](int f) { return approach == 2 ? (int64_t)f * block : shift_amt(f); };
    auto second_amt = [&](int x) { return approach == 2 ? shift_amt(x) : (int64_t)x * block; };
    std::vector<int> fl;  // first-level members used (identity first)
    int fid = -1;
    for (int f = 0; f < nfirst; ++f) {
        bool any = false;
        for (int x = 0; x < nsecond; ++x) any |= nonempty(rpos(f, x).first, rpos(f, x).second);
        if (!any) continue;
        if (c->reduce_amount(first_amt(f)) == 0) fid = f;
        else fl.push_back(f);
    }
    const int NF = (int)fl.size() + 1;  // slot 0: the input itself
    // operand-form rows + TMA baby steps (k_bsgs_tma with source slots), when prepared
    const fhe_conv_layer::PaperKeys& PK = ly->pk[approach - 1];
    const bool opf = paper_opf_ok(c, ly) && c->tma && ly->d_pts_opf && PK.d_keys && PK.gen == c->key_gen;
    uint64_t* X = c->alloc((size_t)S * NF * ctw);
    for (int s = 0; s < S; ++s)
        ck(cudaMemcpyAsync(X + (size_t)s * NF * ctw, cts[s]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    uint64_t* acc = c->alloc((size_t)S * 2 * extw);
    ck(cudaMemsetAsync(acc, 0, (size_t)S * 2 * extw * 8, c->st), "memset");
    if (!fl.empty()) {  // first-level rotations of every input, hoisted, keys shared by the batch
        uint64_t* dig0 = c->alloc((size_t)S * dw);
        modup_batch(c, X + (size_t)nr * N, (size_t)NF * ctw, S, level, dig0, opf ? 1 : 0);
        uint64_t* xp = nullptr;  // opf: the P-scaled inputs in operand form
        if (opf) {
            xp = c->alloc((size_t)S * ctw);
            ct_prescale(c->dc, xp, X, (size_t)NF * ctw, S, c->d_md, level, c->st);
        }
        const size_t F = fl.size();
        uint64_t* XT = c->alloc((size_t)S * F * 2 * extw);
        for (size_t t0 = 0; t0 < F; t0 += kMaxBaby) {
            KsBatch kb{};
            kb.nsrc = S;
            kb.digits = dig0;
            kb.digit_src_stride = dw;
            kb.c0 = opf ? xp : X;
            kb.c0_src_stride = opf ? ctw : (size_t)NF * ctw;
            kb.opf = opf ? 1 : 0;
            kb.out = XT;
            kb.out_src_stride = F * 2 * extw;
            for (size_t t = t0; t < F && kb.n < kMaxBaby; ++t) {
                const uint32_t g = c->galois_of(c->reduce_amount(first_amt(fl[t])));
                kb.galois[kb.n] = g;
                kb.key[kb.n] = opf ? c->key_opf_for(g) : c->key_for(g);
                kb.slot[kb.n] = (int)t;
                kb.n++;
            }
            c->timed("ks_multi", c->rows((double)kb.n * 2.0 * dn * ne + S * ((double)dn * ne + nr + 2.0 * kb.n * ne)),
                     [&] { ks_batch(c->dc, kb, 0, c->d_md, level, dn, c->st); });
        }
        c->ledger.key_switches += (uint64_t)S * F;
        for (int s = 0; s < S; ++s)
            moddown(c, XT + (size_t)s * F * 2 * extw, level, (int)(2 * F), X + ((size_t)s * NF + 1) * ctw, nullptr, 1);
        c->release(XT);
        c->release(xp);
        c->release(dig0);
    }
    // every copy's ModUp, then the fused second-level key switches + MAC
    uint64_t* dig = c->alloc((size_t)S * NF * dw);
    modup_batch(c, X + (size_t)nr * N, ctw, S * NF, level, dig, opf ? 1 : 0);
    if (opf) {
        // every copy P-scaled in operand form (in place: X is not read again), then the
        // second-level key switches + MAC on k_bsgs_tma: babies (slot, x) read their
        // copy's digits / c0 through the 5-D maps' slot coordinate, one giant
        ct_prescale(c->dc, X, X, ctw, S * NF, c->d_md, level, c->st);
        TmaMaps tm{};
        tma_rows(c, level, tm);
        const uint32_t sg = (uint32_t)tma_sources(S), P2 = 256u / sg;
        uint64_t nkeys = 0;
        for (int v : PK.kidx) nkeys += v >= 0;
        const uint64_t dk[4] = {N, (uint64_t)c->np, 2ull * c->dnum, std::max<uint64_t>(1, nkeys)};
        const uint32_t bk[4] = {P2, 1, 2u * dn, 1};
        tma_map4(&tm.key, PK.d_keys, dk, bk);
        const uint64_t dp[4] = {N, (uint64_t)ne, (uint64_t)cin * nk, 1};
        const uint32_t bp[4] = {P2, 1, 1, 1};
        tma_map4(&tm.pt, ly->d_pts_opf, dp, bp);
        const uint64_t dd[5] = {N, (uint64_t)ne, (uint64_t)dn, (uint64_t)NF, (uint64_t)S};
        const uint32_t bd[5] = {P2, 1, (uint32_t)dn, 1, sg};
        tma_map5(&tm.dig, dig, dd, bd);
        const uint64_t dc5[5] = {N, (uint64_t)nr, 2, (uint64_t)NF, (uint64_t)S};
        const uint32_t bc[5] = {P2, 1, 2, 1, sg};
        tma_map5(&tm.ct, X, dc5, bc);
        tm.g0 = 0;
        tm.ng1 = 1;
        FusedBsgs f{};
        f.nsrc = S;
        f.ng = 1;
        f.digits = dig;
        f.ct = X;
        f.Y = acc;
        f.y_src_stride = 2 * extw;
        f.y_g_stride = 2 * extw;
        int launches = 0;
        double keyed = 0;
        auto flush_t = [&] {
            if (!f.nb) return;
            f.accumulate = launches > 0;
            c->timed("bsgs_fused", c->rows(keyed * 2.0 * dn * ne + f.nb * (double)ne +
                                            S * ((double)f.nb * (dn * ne + 2.0 * nr) / NF + 4.0 * ne)),
                     [&] { bsgs_tma(c->dc, f, tm, level, dn, c->st); });
            launches++;
            f.nb = 0;
            keyed = 0;
        };
        for (int slot = 0; slot < NF; ++slot) {
            const int fi = slot == 0 ? fid : fl[slot - 1];
            if (fi < 0) continue;
            for (int x = 0; x < nsecond; ++x) {
                const auto rp = rpos(fi, x);
                if (!nonempty(rp.first, rp.second)) continue;
                if (f.nb == kMaxFused) flush_t();
                const uint32_t g = c->galois_of(c->reduce_amount(second_amt(x)));
                if (g != 1) c->key_for(g);  // a missing key fails here
                f.galois[f.nb] = g;
                f.key[f.nb] = nullptr;
                tm.kidx[f.nb] = (int16_t)(g == 1 ? -1 : PK.kidx[x]);
                tm.bidx[f.nb] = (int16_t)(rp.first * nk + rp.second);
                f.gmask[f.nb] = 1;
                f.srcslot[f.nb] = (uint16_t)slot;
                f.nb++;
                if (g != 1) {
                    keyed += 1;
                    c->ledger.key_switches += S;
                }
            }
        }
        flush_t();
        if (!launches) ck(cudaMemsetAsync(acc, 0, (size_t)S * 2 * extw * 8, c->st), "memset");
    }
    FusedBsgs fb{};
    fb.nsrc = S;
    fb.ng = 1;
    fb.digits = dig;
    fb.digit_src_stride = (size_t)NF * dw;
    fb.digit_slot_stride = dw;
    fb.ct = X;
    fb.ct_src_stride = (size_t)NF * ctw;
    fb.ct_slot_stride = ctw;
    fb.pt_g_stride = 0;
    fb.Y = acc;
    fb.y_src_stride = 2 * extw;
    fb.y_g_stride = 2 * extw;
    fb.accumulate = 1;
    double keyed = 0, pts = 0;
    auto flush = [&] {
        if (!fb.nb) return;
        c->timed("bsgs_fused", c->rows(keyed * 2.0 * dn * ne + pts * ne + S * (NF * (double)dn * ne + 2.0 * nr + 4.0 * ne)),
                 [&] { bsgs_fused(c->dc, fb, c->d_md, level, dn, c->st); });
        fb.nb = 0;
        keyed = pts = 0;
    };
    for (int slot = 0; slot < NF && !opf; ++slot) {
        const int f = slot == 0 ? fid : fl[slot - 1];
        if (f < 0) continue;
        for (int x = 0; x < nsecond; ++x) {
            const auto rp = rpos(f, x);
            if (!nonempty(rp.first, rp.second)) continue;
            if (fb.nb == kMaxFused) flush();
            const uint32_t g = c->galois_of(c->reduce_amount(second_amt(x)));
            fb.galois[fb.nb] = g;
            fb.key[fb.nb] = g == 1 ? nullptr : c->key_for(g);
            fb.gmask[fb.nb] = 1;
            fb.pt[fb.nb] = ly->d_pts + ((size_t)rp.first * nk + rp.second) * extw;
            fb.srcslot[fb.nb] = (uint16_t)slot;
            fb.nb++;
            pts += 1;
            if (g != 1) {
                keyed += 1;
                c->ledger.key_switches += S;
            }
        }
    }
    flush();
    c->release(dig);
    const size_t otw = (size_t)2 * level * N;
    uint64_t* md = c->alloc((size_t)S * otw);
    moddown_rescale(c, acc, extw, level, 2 * S, md, ly->d_bias, 1);
    for (int s = 0; s < S; ++s) {
        ck(cudaMemcpyAsync(outs[s]->d, md + (size_t)s * otw, otw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        outs[s]->scale = (cts[s]->scale * (double)c->primes[level]) / (double)c->primes[level];
        outs[s]->depth = cts[s]->depth + 1;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, outs[s]->depth);
        ledger_conv(c, ly, approach);
    }
    c->release(md);
    c->release(acc);
    c->release(X);
}

// Multi-shard image-mode conv of B images (B x t input shards -> B x n_out
// output shards) through the fused BSGS schedule: babies (u, r, ll) read
// input shard u through the fused kernel's source slots, giants kk m are
// the row shifts, one accumulator set per (image, output shard).
void conv_ms_batch(fhe_ctx* c, const fhe_ct* const* in, int B, const fhe_conv_layer* ly, fhe_ct* const* outs) {
    const int level = ly->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
    const int T = ly->t, NO = ly->n_out, kap = ly->kappa, nb = ly->nb_ms;
    const long m = ly->m, h = kap / 2;
    const int64_t block = (int64_t)m * m;
    for (int i = 0; i < B * T; ++i)
        if (in[i]->level != level) fail(FHE_E_INVALID, "conv layer was encoded for a different level");
    for (int i = 0; i < B * NO; ++i)
        if (outs[i]->level != level - 1) fail(FHE_E_INVALID, "output level must be input level - 1");
    uint64_t* buf = c->alloc((size_t)B * T * ctw);
    for (int i = 0; i < B * T; ++i)
        ck(cudaMemcpyAsync(buf + (size_t)i * ctw, in[i]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    // operand-form rows on k_bsgs_tma (keys from the arena, plaintexts from the layer's
    // operand-form copy, digits / [P c] of input shard u through the slot coordinate)
    const bool opf = c->limb && c->tma;
    TmaMaps tm{};
    if (opf && !ly->d_pts_ms_opf) {
        fhe_conv_layer* L = const_cast<fhe_conv_layer*>(ly);
        const size_t rows = (size_t)NO * kap * nb * ne, prow = (size_t)(NO * kap + 2) * nb * ne;
        ck(cudaMalloc(&L->d_pts_ms_opf, prow * N * 8), "cudaMalloc");
        ck(cudaMemsetAsync(L->d_pts_ms_opf + rows * N, 0, (prow - rows) * N * 8, c->st), "memset");
        rows_to_limb(c->dc, L->d_pts_ms_opf, ly->d_pts_ms, rows, RowMap{ne, level, c->L, 0}, c->st);
    }
    uint64_t* dig = c->alloc((size_t)B * T * dw);
    modup_batch(c, buf + (size_t)nr * N, ctw, B * T, level, dig, opf ? 1 : 0);
    if (opf) {
        ct_prescale(c->dc, buf, buf, ctw, B * T, c->d_md, level, c->st);
        tma_rows(c, level, tm);
        const uint32_t sg = (uint32_t)tma_sources(B), P2 = 256u / sg;
        const uint64_t dk[4] = {N, (uint64_t)c->np, 2ull * c->dnum, (uint64_t)std::max(1, c->arena_n)};
        const uint32_t bk[4] = {P2, 1, 2u * dn, 1};
        tma_map4(&tm.key, c->d_key_arena, dk, bk);
        const uint64_t dp[4] = {N, (uint64_t)ne, (uint64_t)nb, (uint64_t)(NO * kap + 2)};
        const uint32_t bp[4] = {P2, 1, 1, 3};
        tma_map4(&tm.pt, ly->d_pts_ms_opf, dp, bp);
        const uint64_t dd[5] = {N, (uint64_t)ne, (uint64_t)dn, (uint64_t)T, (uint64_t)B};
        const uint32_t bd[5] = {P2, 1, (uint32_t)dn, 1, sg};
        tma_map5(&tm.dig, dig, dd, bd);
        const uint64_t dc5[5] = {N, (uint64_t)nr, 2, (uint64_t)T, (uint64_t)B};
        const uint32_t bc[5] = {P2, 1, 2, 1, sg};
        tma_map5(&tm.ct, buf, dc5, bc);
    }
    const size_t ys = (size_t)kap * 2 * extw;
    uint64_t* Y = c->alloc((size_t)B * NO * ys);  // [B][n_out][kappa][2][ne][N]
    ck(cudaMemsetAsync(Y, 0, (size_t)B * NO * ys * 8, c->st), "memset");
    for (int v = 0; v < NO; ++v)
        for (int g0 = 0; g0 < kap; g0 += 3) {
            const int ng = std::min(3, kap - g0);
            FusedBsgs f{};
            f.nsrc = B;
            f.ng = ng;
            f.digits = dig;
            f.digit_src_stride = (size_t)T * dw;
            f.digit_slot_stride = dw;
            f.ct = buf;
            f.ct_src_stride = (size_t)T * ctw;
            f.ct_slot_stride = ctw;
            f.pt_g_stride = (size_t)nb * extw;
            f.Y = Y + (size_t)v * ys + (size_t)g0 * 2 * extw;
            f.y_src_stride = (size_t)NO * ys;
            f.y_g_stride = 2 * extw;
            f.accumulate = 1;
            int launches = 0;
            tm.g0 = v * kap + g0;
            double keyed = 0, pts = 0;
            auto flush = [&] {
                if (!f.nb) return;
                for (int q = 0; q < f.nb; ++q)
                    if (f.galois[q] != 1) c->ledger.hoisted_rotations += (uint64_t)B;
                c->ledger.ct_pt_mults += (uint64_t)B * (uint64_t)pts;
                c->ledger.adds += (uint64_t)B * (uint64_t)pts;
                if (opf) f.accumulate = launches > 0;
                c->timed("bsgs_fused",
                         c->rows(keyed * 2.0 * dn * ne + pts * ne + B * (T * (double)dn * ne + 2.0 * nr + 4.0 * ng * ne)),
                         [&] {
                             if (opf)
                                 bsgs_tma(c->dc, f, tm, level, dn, c->st);
                             else
                                 bsgs_fused(c->dc, f, c->d_md, level, dn, c->st);
                         });
                launches++;
                f.nb = 0;
                keyed = pts = 0;
            };
            for (int b = 0; b < nb; ++b) {
                uint32_t mask = 0;
                for (int g = 0; g < ng; ++g)
                    if (ly->ms_nonempty[((size_t)v * kap + g0 + g) * nb + b]) mask |= 1u << g;
                if (!mask) continue;
                if (f.nb == kMaxFused) flush();
                const int u = b / (ly->rmax * kap), r = (b / kap) % ly->rmax;
                const long ll = b % kap - h;
                const uint32_t gal = c->galois_of(c->reduce_amount((int64_t)r * ly->rep * block + ll));
                f.galois[f.nb] = gal;
                f.key[f.nb] = gal == 1 ? nullptr : c->key_for(gal);
                tm.kidx[f.nb] = (int16_t)(gal == 1 ? -1 : c->key_slot.at(gal));
                tm.bidx[f.nb] = (int16_t)b;
                f.gmask[f.nb] = mask;
                f.pt[f.nb] = ly->d_pts_ms + (((size_t)v * kap + g0) * nb + b) * extw;
                f.srcslot[f.nb] = (uint16_t)u;
                f.nb++;
                pts += __builtin_popcount(mask);
                if (gal != 1) {
                    keyed += 1;
                    c->ledger.key_switches += B;
                }
            }
            flush();
        }
    c->release(dig);
    std::vector<int> giants;
    std::vector<int64_t> gamt;
    int id = -1;
    for (long kk = -h; kk <= h; ++kk) {
        gamt.push_back(kk * m);
        if (kk == 0)
            id = (int)(kk + h);
        else
            giants.push_back((int)(kk + h));
    }
    const size_t otw = (size_t)2 * level * N;
    uint64_t* md = c->alloc((size_t)B * NO * otw);
    giants_finish(c, Y, ys, B * NO, level, giants, gamt, id, md, ly->d_bias, NO);
    for (int i = 0; i < B * NO; ++i) {
        ck(cudaMemcpyAsync(outs[i]->d, md + (size_t)i * otw, otw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        const fhe_ct* src = in[(i / NO) * T];
        outs[i]->scale = (src->scale * (double)c->primes[level]) / (double)c->primes[level];
        outs[i]->depth = src->depth + 1;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, outs[i]->depth);
    }
    c->ledger.hoist_groups += (uint64_t)B * T;
    c->ledger.rotations += (uint64_t)B * NO * giants.size();
    c->release(md);
    c->release(Y);
    c->release(buf);
}

// Channel-shard conv of B images (B x c x pc input shards -> B x c_out x pc
// output shards), fused BSGS per output shard (g, v): babies = column shifts
// ll of input shard (f, src), src in {v, v +- 1} (in-shard / spill masks),
// giants = row shifts kk m; plaintexts pt'[g][f][kk][ll][spill].
void conv_cs_batch(fhe_ctx* c, const fhe_ct* const* in, int B, const fhe_conv_layer* ly, fhe_ct* const* outs) {
    const int level = ly->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
    const int C_ = ly->c_in, CO = ly->c_out, PC = ly->pc, kap = ly->kappa, h = kap / 2;
    const int NSH = C_ * PC, NOUT = CO * PC;
    for (int i = 0; i < B * NSH; ++i)
        if (in[i]->level != level) fail(FHE_E_INVALID, "conv layer was encoded for a different level");
    for (int i = 0; i < B * NOUT; ++i)
        if (outs[i]->level != level - 1) fail(FHE_E_INVALID, "output level must be input level - 1");
    uint64_t* buf = c->alloc((size_t)B * NSH * ctw);
    for (int i = 0; i < B * NSH; ++i)
        ck(cudaMemcpyAsync(buf + (size_t)i * ctw, in[i]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    // operand-form rows on k_bsgs_tma: plaintext map (N, ne, 2 kappa [ll, spill], CO C kappa
    // [(g, f), kk]), the giant base (g, f) per baby (TmaMaps.gidx), input shards by slot
    const bool opf = c->limb && c->tma;
    TmaMaps tm{};
    const int GD = CO * C_ * kap;  // giant coordinate extent
    if (opf && !ly->d_pts_cs_opf) {
        fhe_conv_layer* Lm = const_cast<fhe_conv_layer*>(ly);
        const size_t rows = (size_t)GD * 2 * kap * ne, prow = (size_t)(GD + 2) * 2 * kap * ne;
        ck(cudaMalloc(&Lm->d_pts_cs_opf, prow * N * 8), "cudaMalloc");
        ck(cudaMemsetAsync(Lm->d_pts_cs_opf + rows * N, 0, (prow - rows) * N * 8, c->st), "memset");
        rows_to_limb(c->dc, Lm->d_pts_cs_opf, ly->d_pts_ms, rows, RowMap{ne, level, c->L, 0}, c->st);
    }
    uint64_t* dig = c->alloc((size_t)B * NSH * dw);
    modup_batch(c, buf + (size_t)nr * N, ctw, B * NSH, level, dig, opf ? 1 : 0);
    if (opf) {
        ct_prescale(c->dc, buf, buf, ctw, B * NSH, c->d_md, level, c->st);
        tma_rows(c, level, tm);
        const uint32_t sg = (uint32_t)tma_sources(B), P2 = 256u / sg;
        const uint64_t dk[4] = {N, (uint64_t)c->np, 2ull * c->dnum, (uint64_t)std::max(1, c->arena_n)};
        const uint32_t bk[4] = {P2, 1, 2u * dn, 1};
        tma_map4(&tm.key, c->d_key_arena, dk, bk);
        const uint64_t dp[4] = {N, (uint64_t)ne, (uint64_t)(2 * kap), (uint64_t)(GD + 2)};
        const uint32_t bp[4] = {P2, 1, 1, 3};
        tma_map4(&tm.pt, ly->d_pts_cs_opf, dp, bp);
        const uint64_t dd[5] = {N, (uint64_t)ne, (uint64_t)dn, (uint64_t)NSH, (uint64_t)B};
        const uint32_t bd[5] = {P2, 1, (uint32_t)dn, 1, sg};
        tma_map5(&tm.dig, dig, dd, bd);
        const uint64_t dc5[5] = {N, (uint64_t)nr, 2, (uint64_t)NSH, (uint64_t)B};
        const uint32_t bc[5] = {P2, 1, 2, 1, sg};
        tma_map5(&tm.ct, buf, dc5, bc);
    }
    const size_t ys = (size_t)kap * 2 * extw;
    uint64_t* Y = c->alloc((size_t)B * NOUT * ys);  // [B][c_out][pc][kappa][2][ne][N]
    ck(cudaMemsetAsync(Y, 0, (size_t)B * NOUT * ys * 8, c->st), "memset");
    auto pt_of = [&](int g, int f, int kk, int ll, int spill) {  // kk, ll offsets in [0, kappa)
        return ((((size_t)g * C_ + f) * kap + kk) * kap + ll) * 2 + spill;
    };
    for (int g = 0; g < CO; ++g)
        for (int v = 0; v < PC; ++v)
            for (int g0 = 0; g0 < kap; g0 += 3) {
                const int ng = std::min(3, kap - g0);
                FusedBsgs f{};
                f.nsrc = B;
                f.ng = ng;
                f.digits = dig;
                f.digit_src_stride = (size_t)NSH * dw;
                f.digit_slot_stride = dw;
                f.ct = buf;
                f.ct_src_stride = (size_t)NSH * ctw;
                f.ct_slot_stride = ctw;
                f.pt_g_stride = (size_t)kap * 2 * extw;  // next row shift kk
                f.Y = Y + ((size_t)g * PC + v) * ys + (size_t)g0 * 2 * extw;
                f.y_src_stride = (size_t)NOUT * ys;
                f.y_g_stride = 2 * extw;
                f.accumulate = 1;
                int launches = 0;
                tm.g0 = g0;
                double keyed = 0, pts = 0;
                auto flush = [&] {  // more babies than one launch holds: continue the accumulators
                    if (!f.nb) return;
                    c->ledger.hoisted_rotations += (uint64_t)B * (uint64_t)keyed;
                    c->ledger.ct_pt_mults += (uint64_t)B * (uint64_t)pts;
                    c->ledger.adds += (uint64_t)B * (uint64_t)pts;
                    if (opf) f.accumulate = launches > 0;
                    c->timed("bsgs_fused",
                             c->rows(keyed * 2.0 * dn * ne + pts * ne +
                                     B * (3.0 * C_ * dn * ne + 2.0 * nr + 4.0 * ng * ne)),
                             [&] {
                                 if (opf)
                                     bsgs_tma(c->dc, f, tm, level, dn, c->st);
                                 else
                                     bsgs_fused(c->dc, f, c->d_md, level, dn, c->st);
                             });
                    launches++;
                    f.nb = 0;
                    keyed = pts = 0;
                };
                for (int fi = 0; fi < C_; ++fi)
                    for (int dv = -1; dv <= 1; ++dv) {
                        const int src = v + dv;
                        if (src < 0 || src >= PC) continue;
                        const int spill = dv != 0;
                        for (int lo = 0; lo < kap; ++lo) {
                            uint32_t mask = 0;
                            for (int gg = 0; gg < ng; ++gg) {
                                const int kk = g0 + gg - h;  // row shift of this giant
                                if (spill && (kk == 0 || (kk > 0) != (dv > 0))) continue;
                                if (ly->ms_nonempty[pt_of(g, fi, g0 + gg, lo, spill)]) mask |= 1u << gg;
                            }
                            if (!mask) continue;
                            if (f.nb == kMaxFused) flush();
                            const uint32_t gal = c->galois_of(c->reduce_amount(lo - h));
                            f.galois[f.nb] = gal;
                            f.key[f.nb] = gal == 1 ? nullptr : c->key_for(gal);
                            tm.kidx[f.nb] = (int16_t)(gal == 1 ? -1 : c->key_slot.at(gal));
                            tm.bidx[f.nb] = (int16_t)(2 * lo + spill);
                            tm.gidx[f.nb] = (int16_t)((g * C_ + fi) * kap);
                            f.gmask[f.nb] = mask;
                            f.pt[f.nb] = ly->d_pts_ms + pt_of(g, fi, g0, lo, spill) * extw;
                            f.srcslot[f.nb] = (uint16_t)(fi * PC + src);
                            f.nb++;
                            pts += __builtin_popcount(mask);
                            if (gal != 1) {
                                keyed += 1;
                                c->ledger.key_switches += B;
                            }
                        }
                    }
                flush();
            }
    c->release(dig);
    std::vector<int> giants;
    std::vector<int64_t> gamt;
    int id = -1;
    for (int kk = -h; kk <= h; ++kk) {
        gamt.push_back((int64_t)kk * ly->m);
        if (kk == 0)
            id = kk + h;
        else
            giants.push_back(kk + h);
    }
    const size_t otw = (size_t)2 * level * N;
    uint64_t* md = c->alloc((size_t)B * NOUT * otw);
    c->ledger.hoist_groups += (uint64_t)B * NSH;
    c->ledger.rotations += (uint64_t)B * NOUT * giants.size();
    giants_finish(c, Y, ys, B * NOUT, level, giants, gamt, id, md, ly->d_bias, NOUT);
    for (int i = 0; i < B * NOUT; ++i) {
        ck(cudaMemcpyAsync(outs[i]->d, md + (size_t)i * otw, otw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        const fhe_ct* src = in[(i / NOUT) * NSH];
        outs[i]->scale = (src->scale * (double)c->primes[level]) / (double)c->primes[level];
        outs[i]->depth = src->depth + 1;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, outs[i]->depth);
    }
    c->release(md);
    c->release(Y);
    c->release(buf);
}

// QP plaintexts (slot vectors encoded over Q_l u P at scale q_l) of a term
// list, encoded once per (key, level) and cached on the context.
uint64_t* lt_plaintexts(fhe_ctx* c, const std::string& key, int level, const std::vector<std::vector<double>>& vecs) {
    const int ne = c->ne_at(level);
    const size_t extw = (size_t)ne * c->N;
    const std::string ck_key = key + "/" + std::to_string(level);
    auto it = c->lt_cache.find(ck_key);
    if (it != c->lt_cache.end()) return it->second;
    uint64_t* pts = nullptr;
    ck(cudaMalloc(&pts, std::max<size_t>(1, vecs.size()) * extw * 8), "cudaMalloc");
    for (size_t b = 0; b < vecs.size(); ++b)
        encode_rows(c, vecs[b].data(), vecs[b].size(), level, (double)c->primes[level], ne, pts + b * extw);
    ck(cudaStreamSynchronize(c->st), "sync");
    c->lt_cache[ck_key] = pts;
    return pts;
}

// one term of a plaintext-weighted sum of rotations: pt_b * rot_amount(source
// shard u + slot) for output u (slot 1 = the next shard: channel-shard spill)
struct LtTerm {
    int64_t amount;
    int slot;
    int pt;  // index into the cached plaintexts
};

// Y_u += sum_b pt_b * X~_{src(u) + slot_b, amount_b} for nout outputs, output u
// reading shard src0 + u * src_stride (+ slot) of the ModUp'd copies (dig, buf,
// [shard][dn][ne][N] / [shard][2][l+1][N]); Y_u = Y + u * y_stride, [2][ne][N]
// in the fused kernel's accumulation domain. Fused baby-step launches of <=
// kMaxFused terms.
void lt_accumulate(fhe_ctx* c, int level, const uint64_t* dig, const uint64_t* buf, int nout, size_t src0,
                   size_t src_stride, const std::vector<LtTerm>& terms, const uint64_t* pts, uint64_t* Y,
                   size_t y_stride) {
    const int nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
    if (nout <= 0 || terms.empty()) return;
    FusedBsgs f{};
    f.nsrc = nout;
    f.ng = 1;
    f.digits = dig + src0 * dw;
    f.digit_src_stride = src_stride * dw;
    f.digit_slot_stride = dw;
    f.ct = buf + src0 * ctw;
    f.ct_src_stride = src_stride * ctw;
    f.ct_slot_stride = ctw;
    f.Y = Y;
    f.y_src_stride = y_stride;
    f.y_g_stride = 2 * extw;
    f.accumulate = 1;
    for (size_t b0 = 0; b0 < terms.size(); b0 += kMaxFused) {
        f.nb = 0;
        double keyed = 0;
        int nslot = 0;
        for (size_t b = b0; b < terms.size() && f.nb < kMaxFused; ++b) {
            const LtTerm& t = terms[b];
            const uint32_t gal = c->galois_of(c->reduce_amount(t.amount));
            f.galois[f.nb] = gal;
            f.key[f.nb] = gal == 1 ? nullptr : c->key_for(gal);
            f.gmask[f.nb] = 1;
            f.pt[f.nb] = pts + (size_t)t.pt * extw;
            f.srcslot[f.nb] = (uint16_t)t.slot;
            nslot = std::max(nslot, t.slot + 1);
            f.nb++;
            if (gal != 1) {
                keyed += 1;
                c->ledger.key_switches += (uint64_t)nout;
            }
        }
        c->timed("bsgs_fused",
                 c->rows(keyed * 2.0 * dn * ne + f.nb * ne +
                         nout * (nslot * ((double)dn * ne + 2.0 * nr) + 4.0 * ne)),
                 [&] { bsgs_fused(c->dc, f, c->d_md, level, dn, c->st); });
    }
    c->ledger.ct_pt_mults += (uint64_t)nout * terms.size();
}

// device copies + ModUp of n shards at one level: buf [n][2][l+1][N], dig [n][dn][ne][N]
void lt_modup(fhe_ctx* c, const fhe_ct* const* cts, int n, uint64_t** buf, uint64_t** dig) {
    const int level = cts[0]->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * ne * N;
    for (int i = 0; i < n; ++i)
        if (cts[i]->level != level) fail(FHE_E_INVALID, "shards are at different levels");
    *buf = c->alloc((size_t)n * ctw);
    for (int i = 0; i < n; ++i)
        ck(cudaMemcpyAsync(*buf + (size_t)i * ctw, cts[i]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    *dig = c->alloc((size_t)n * dw);
    modup_batch(c, *buf + (size_t)nr * N, ctw, n, level, *dig);
}

// outs[u] = Rescale(ModDown(Y_u)) for S accumulators (one level), metadata from src[u]
void lt_finish(fhe_ctx* c, const uint64_t* Y, int S, int level, const fhe_ct* const* src, fhe_ct* const* outs) {
    const int ne = c->ne_at(level);
    const size_t N = c->N, extw = (size_t)ne * N, otw = (size_t)2 * level * N;
    uint64_t* md = c->alloc((size_t)S * otw);
    giants_finish(c, Y, 2 * extw, S, level, {}, {0}, 0, md);
    for (int i = 0; i < S; ++i) {
        ck(cudaMemcpyAsync(outs[i]->d, md + (size_t)i * otw, otw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        outs[i]->scale = src[i]->scale;
        outs[i]->depth = src[i]->depth + 1;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, outs[i]->depth);
    }
    c->release(md);
}

// out_s = Rescale(ModDown(sum_b pt_b * X~_{s,b})) for S ciphertexts sharing the
// term list (rotation amount, plaintext slot vector): the fused baby-step
// kernel with one accumulator; pt_b = rot-free slot vectors encoded over
// Q_l u P at scale q_l and cached under `key`. One level.
void lintrans_batch(fhe_ctx* c, const fhe_ct* const* cts, int S, const std::string& key,
                    const std::vector<int64_t>& amounts, const std::vector<std::vector<double>>& vecs,
                    fhe_ct* const* outs) {
    const int level = cts[0]->level, ne = c->ne_at(level);
    const size_t extw = (size_t)ne * c->N;
    if (level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
    const uint64_t* pts = lt_plaintexts(c, key, level, vecs);
    uint64_t *buf, *dig;
    lt_modup(c, cts, S, &buf, &dig);
    uint64_t* Y = c->alloc((size_t)S * 2 * extw);
    ck(cudaMemsetAsync(Y, 0, (size_t)S * 2 * extw * 8, c->st), "memset");
    std::vector<LtTerm> terms;
    for (size_t b = 0; b < amounts.size(); ++b) terms.push_back({amounts[b], 0, (int)b});
    lt_accumulate(c, level, dig, buf, S, 0, 1, terms, pts, Y, 2 * extw);
    c->release(dig);
    lt_finish(c, Y, S, level, cts, outs);
    c->release(Y);
    c->release(buf);
}

int auto_orient(const fhe_conv_layer* ly) {
    // giant steps each cost a ModDown + ModUp (~120 NTT rows at cfg3) while a
    // fused baby step costs one key stream: always the fused schedule (kappa
    // giant steps); more than kMaxFused baby steps run in several launches
    (void)ly;
    return 5;
}

void conv_impl(fhe_ctx* c, const fhe_ct* ct, const fhe_conv_layer* ly, int approach, fhe_ct* out) {
    if (ly->ms) fail(FHE_E_INVALID, "multi-shard layer: use fhe_conv2d_shards_into");
    if (approach < 0 || approach > 5) fail(FHE_E_INVALID, "approach must be 0 (auto), 1, 2, 3, 4 or 5");
    if (approach == 0) approach = auto_orient(ly);
    if (approach >= 3) {
        if (ct->level != ly->level) fail(FHE_E_INVALID, "conv layer was encoded for a different level");
        if (out->level != ct->level - 1) fail(FHE_E_INVALID, "output level must be input level - 1");
        conv_bsgs(c, ct, ly, approach, out);
        return;
    }
    if (ct->level != ly->level) fail(FHE_E_INVALID, "conv layer was encoded for a different level");
    if (out->level != ct->level - 1) fail(FHE_E_INVALID, "output level must be input level - 1");
    const int level = ct->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    const size_t N = c->N, extw = (size_t)ne * N;
    const int nk = ly->nk, cin = ly->c_in;
    const long m = ly->m, h = ly->kappa / 2;
    const int64_t block = (int64_t)m * m;

    uint64_t* acc = c->alloc(2 * extw);
    ck(cudaMemsetAsync(acc, 0, 2 * extw * 8, c->st), "memset");
    uint64_t* dsrc = c->alloc((size_t)dn * extw);
    uint64_t* dtmp = c->alloc((size_t)dn * extw);
    fhe_ct X{c, level, ct->scale, ct->depth, c->alloc(ct->words())};
    modup(c, ct->c1(), level, dsrc);

    auto pt_of = [&](int r, int i) { return ly->d_pts + ((size_t)r * nk + i) * extw; };
    auto run_terms = [&](MacTerms& t, const fhe_ct& src) {
        if (t.n == 0) return;
        double mac_rows = (double)t.n * ne + (double)dn * ne + 2.0 * nr + 4.0 * ne;
        for (int i = 0; i < t.n; ++i)
            if (t.galois[i] != 1) mac_rows += 2.0 * dn * ne;
        c->timed("conv_mac", c->rows(mac_rows), [&] { conv_mac(c->dc, acc, dtmp, src.d, t, c->d_md, level, dn, c->st); });
        for (int i = 0; i < t.n; ++i)
            if (t.galois[i] != 1) c->ledger.key_switches++;
        t.n = 0;
    };
    auto push = [&](MacTerms& t, const fhe_ct& src, uint32_t g, const uint64_t* pt) {
        if (t.n == kMaxTerms) run_terms(t, src);
        t.galois[t.n] = g;
        t.key[t.n] = g == 1 ? nullptr : c->key_for(g);
        t.pt[t.n] = pt;
        t.n++;
    };

    if (approach == 2) {
        for (int r = 0; r < cin; ++r) {
            bool any = false;
            for (int i = 0; i < nk; ++i) any |= ly->nonempty[r * nk + i] != 0;
            if (!any) continue;
            const uint32_t gr = c->galois_of(c->reduce_amount((int64_t)r * block));
            const fhe_ct* src = ct;
            if (gr != 1) {
                rotate_from_digits(c, ct, dsrc, gr, X.d);
                src = &X;
            }
            modup(c, src->c1(), level, dtmp);
            MacTerms t{};
            int i = 0;
            for (long kk = -h; kk <= h; ++kk)
                for (long ll = -h; ll <= h; ++ll, ++i) {
                    if (!ly->nonempty[r * nk + i]) continue;
                    push(t, *src, c->galois_of(c->reduce_amount(kk * m + ll)), pt_of(r, i));
                }
            run_terms(t, *src);
        }
    } else {
        int i = 0;
        for (long kk = -h; kk <= h; ++kk)
            for (long ll = -h; ll <= h; ++ll, ++i) {
                bool any = false;
                for (int r = 0; r < cin; ++r) any |= ly->nonempty[r * nk + i] != 0;
                if (!any) continue;
                const uint32_t gi = c->galois_of(c->reduce_amount(kk * m + ll));
                const fhe_ct* src = ct;
                if (gi != 1) {
                    rotate_from_digits(c, ct, dsrc, gi, X.d);
                    src = &X;
                }
                modup(c, src->c1(), level, dtmp);
                MacTerms t{};
                for (int r = 0; r < cin; ++r) {
                    if (!ly->nonempty[r * nk + i]) continue;
                    push(t, *src, c->galois_of(c->reduce_amount((int64_t)r * block)), pt_of(r, i));
                }
                run_terms(t, *src);
            }
    }
    // one ModDown per component, then one rescale
    moddown_rescale(c, acc, extw, level, 2, out->d, ly->d_bias, 1);
    out->scale = (ct->scale * (double)c->primes[level]) / (double)c->primes[level];
    out->depth = ct->depth + 1;
    c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, out->depth);
    c->release(acc);
    c->release(dsrc);
    c->release(dtmp);
    c->release(X.d);
    ledger_conv(c, ly, approach);
}

void batch_impl(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const fhe_conv_layer* ly, int approach,
                fhe_ct* const* outs) {
    if (n == 0) return;
    if (ly->ms) fail(FHE_E_INVALID, "multi-shard layer: use fhe_conv2d_shards_into");
    if (approach < 0 || approach > 5) fail(FHE_E_INVALID, "approach must be 0 (auto), 1, 2, 3, 4 or 5");
    if (approach == 0) approach = auto_orient(ly);
    // approaches 1 / 2 (also one ciphertext) through the batched paper schedule: the
    // same residues as conv_impl, first-level rotations hoisted, second level fused
    const bool paper_batch = (approach == 1 || approach == 2) && c->batch5 && !ly->ms && !ly->cs;
    const bool bsgs_batch = approach >= 3 && n > 1 && (c->fused_batch || (approach == 5 && c->batch5));
    if (paper_batch || bsgs_batch || n == 1) {
        for (size_t s = 0; s < n; ++s) {
            if (cts[s]->level != ly->level) fail(FHE_E_INVALID, "conv layer was encoded for a different level");
            if (outs[s]->level != ly->level - 1) fail(FHE_E_INVALID, "output level must be input level - 1");
        }
        prepare_bias(c, ly, cts, n);
        auto body = [&] {
            if (paper_batch) {
                for (size_t s0 = 0; s0 < n; s0 += 8)
                    conv_paper_batch(c, cts + s0, (int)std::min<size_t>(8, n - s0), ly, approach, outs + s0);
            } else if (n == 1) {
                conv_impl(c, cts[0], ly, approach, outs[0]);
            } else {
                for (size_t s0 = 0; s0 < n; s0 += 32)
                    conv_bsgs_batch(c, cts + s0, (int)std::min<size_t>(32, n - s0), ly, approach, outs + s0);
            }
        };
        if (!c->use_graphs || c->prof_on || c->st != c->main_st) {
            body();
            return;
        }
        if (approach >= 3) ensure_bsgs(c, ly, approach);  // host encoding + sync: never inside a capture
        prepare_limb(c, ly, approach);
        if (paper_batch) prepare_paper(c, ly, approach);
        std::vector<const void*> key{(const void*)(uintptr_t)ly->uid, (const void*)(uintptr_t)approach,
                                     (const void*)(uintptr_t)n};
        for (size_t s = 0; s < n; ++s) {
            key.push_back(cts[s]->d);
            key.push_back(outs[s]->d);
        }
        auto replay_host_state = [&](const fhe_ctx::GraphEntry& g) {
            fhe_ledger& lg = c->ledger;
            uint64_t* dst = reinterpret_cast<uint64_t*>(&lg);
            const uint64_t* del = reinterpret_cast<const uint64_t*>(&g.delta);
            for (size_t f = 0; f < sizeof(fhe_ledger) / sizeof(uint64_t); ++f) dst[f] += del[f];
            note_launch((int)g.launches);
            for (uint64_t a : g.amounts) c->amounts.insert(a);
            for (size_t s = 0; s < n; ++s) {
                outs[s]->scale = (cts[s]->scale * (double)c->primes[ly->level]) / (double)c->primes[ly->level];
                outs[s]->depth = cts[s]->depth + 1;
                lg.max_depth_consumed = std::max<uint64_t>(lg.max_depth_consumed, outs[s]->depth);
            }
        };
        for (auto& g : c->graphs)
            if (g.key == key) {
                ck(cudaGraphLaunch(g.exec, c->st), "cudaGraphLaunch");
                g.last_use = ++c->graph_clock;
                replay_host_state(g);
                return;
            }
        // capture once: kernels, copies and stream-ordered allocations become graph nodes
        const fhe_ledger before = c->ledger;
        const uint64_t l0 = launches_total();
        cudaGraph_t graph = nullptr;
        std::vector<uint64_t> rec;
        ck(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        c->amount_rec = &rec;
        try {
            body();
        } catch (...) {
            c->amount_rec = nullptr;
            cudaStreamEndCapture(c->st, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        c->amount_rec = nullptr;
        ck(cudaStreamEndCapture(c->st, &graph), "cudaStreamEndCapture");
        fhe_ctx::GraphEntry g;
        g.key = key;
        std::sort(rec.begin(), rec.end());
        rec.erase(std::unique(rec.begin(), rec.end()), rec.end());
        g.amounts = std::move(rec);
        ck(cudaGraphInstantiate(&g.exec, graph, 0), "cudaGraphInstantiate");
        cudaGraphDestroy(graph);
        g.launches = launches_total() - l0;
        {
            uint64_t* d = reinterpret_cast<uint64_t*>(&g.delta);
            const uint64_t* a = reinterpret_cast<const uint64_t*>(&c->ledger);
            const uint64_t* b = reinterpret_cast<const uint64_t*>(&before);
            for (size_t f = 0; f < sizeof(fhe_ledger) / sizeof(uint64_t); ++f) d[f] = a[f] - b[f];
            g.delta.max_depth_consumed = 0;  // a maximum, re-applied by replay_host_state
            g.delta.distinct_amounts = 0;
        }
        ck(cudaGraphLaunch(g.exec, c->st), "cudaGraphLaunch");
        g.last_use = ++c->graph_clock;
        if (c->graphs.size() >= 16) {  // evict the least recently used graph
            auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                        [](const auto& x, const auto& y) { return x.last_use < y.last_use; });
            ck(cudaStreamSynchronize(c->st), "sync");
            cudaGraphExecDestroy(lru->exec);
            c->graphs.erase(lru);
        }
        c->graphs.push_back(std::move(g));
        return;
    }
    if (approach >= 3) ensure_bsgs(c, ly, approach);  // layer constants are built on the main stream
    prepare_limb(c, ly, approach);
    if (paper_batch) prepare_paper(c, ly, approach);
    prepare_bias(c, ly, cts, n);
    if (n == 1 || c->lanes.size() <= 1) {
        for (size_t i = 0; i < n; ++i) conv_impl(c, cts[i], ly, approach, outs[i]);
        return;
    }
    // independent ciphertexts on independent lanes: the memory-bound key/plaintext
    // streams of one conv overlap the integer-bound NTTs of another
    if (c->pending_events.size() > 256) {
        ck(cudaStreamSynchronize(c->main_st), "sync");
        for (cudaEvent_t e : c->pending_events) c->ev_pool.push_back(e);
        c->pending_events.clear();
    }
    cudaEvent_t start = c->get_event();
    ck(cudaEventRecord(start, c->main_st), "cudaEventRecord");
    for (cudaStream_t l : c->lanes) ck(cudaStreamWaitEvent(l, start, 0), "cudaStreamWaitEvent");
    try {
        for (size_t i = 0; i < n; ++i) {
            c->st = c->lanes[i % c->lanes.size()];
            conv_impl(c, cts[i], ly, approach, outs[i]);
        }
    } catch (...) {
        c->st = c->main_st;
        throw;
    }
    c->st = c->main_st;
    std::vector<cudaEvent_t> done;
    for (cudaStream_t l : c->lanes) {
        cudaEvent_t e = c->get_event();
        ck(cudaEventRecord(e, l), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->main_st, e, 0), "cudaStreamWaitEvent");
        done.push_back(e);
    }
    // events can be recycled once the main stream has passed them
    c->pending_events.push_back(start);
    for (cudaEvent_t e : done) c->pending_events.push_back(e);
}

}  // namespace

// =================================================================== C ABI
extern "C" {

int fhe_ctx_create(const fhe_params* p, fhe_ctx** out) {
    if (!p || !out) return FHE_E_INVALID;
    *out = nullptr;
    fhe_ctx* c = new fhe_ctx();
    const int rc = guard(c, [&] {
        if (p->log_n < 12 || p->log_n > 16) fail(FHE_E_INVALID, "log_n must be in [12, 16]");
        if (p->n_q < 1 || p->n_p < 1 || p->n_p > kMaxAlpha || p->n_q + p->n_p > kMaxPrimes)
            fail(FHE_E_INVALID, "unsupported prime counts");
        // the keyed kernels are instantiated for 1..8 digits (and the carry-deferred
        // inner product is exact for at most 8 terms)
        if ((p->n_q + p->n_p - 1) / p->n_p > 8)
            fail(FHE_E_INVALID, "unsupported prime counts: dnum = ceil(n_q / n_p) must be <= 8");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            fail(FHE_E_CUDA, "no CUDA device available (libfheconv has no CPU fallback)");
        c->device = p->device;
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, c->device), "cudaGetDeviceProperties");
        if (prop.major < 10) fail(FHE_E_CUDA, "libfheconv is built for sm_100a (B200)");
        ck(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking), "cudaStreamCreate");
        c->main_st = c->st;
        ck(cudaStreamCreateWithFlags(&c->h2d_st, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&c->d2h_st, cudaStreamNonBlocking), "cudaStreamCreate");
        int nl = 4;
        if (const char* e = std::getenv("FHECONV_LANES")) nl = std::max(1, std::atoi(e));
        for (int i = 0; i < nl; ++i) {
            cudaStream_t l;
            ck(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking), "cudaStreamCreate");
            c->lanes.push_back(l);
        }
        if (const char* e = std::getenv("FHECONV_BATCH_FUSED")) c->fused_batch = std::atoi(e) != 0;
        if (const char* e = std::getenv("FHECONV_BATCH5")) c->batch5 = std::atoi(e) != 0;
        if (const char* e = std::getenv("FHECONV_LIMB")) c->limb = std::atoi(e) != 0;
        if (const char* e = std::getenv("FHECONV_TMA")) c->tma = std::atoi(e) != 0;
        c->limb = c->limb && c->tma;
        if (const char* e = std::getenv("FHECONV_GRAPHS")) c->use_graphs = std::atoi(e) != 0;
        cudaMemPool_t pool;
        ck(cudaDeviceGetDefaultMemPool(&pool, c->device), "mempool");
        uint64_t thresh = ~0ULL;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
        c->logN = p->log_n;
        c->N = 1 << p->log_n;
        c->L = p->n_q;
        c->K = p->n_p;
        c->alpha = p->n_p;
        c->dnum = (c->L + c->alpha - 1) / c->alpha;
        c->np = c->L + c->K;
        std::vector<int> bits(p->q_bits, p->q_bits + p->n_q);
        bits.insert(bits.end(), p->p_bits, p->p_bits + p->n_p);
        c->primes = host::generate_primes(bits, (uint64_t)c->N);
        c->scale = std::ldexp(1.0, p->log_scale);
        if (const char* e = std::getenv("FHECONV_GIANT_CHUNK")) c->giant_chunk = std::max(1, std::min(kMaxBaby, std::atoi(e)));
        upload_tables(c);
    });
    if (rc != FHE_OK) {
        // keep the context alive only to report the error? callers get rc.
        fhe_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return FHE_OK;
}

static void host_pipe_free(fhe_ctx* c);

void fhe_ctx_destroy(fhe_ctx* c) {
    if (!c) return;
    if (c->st) cudaStreamSynchronize(c->st);
    for (auto& kv : c->keys) cudaFreeAsync(kv.second, c->st);
    if (c->d_key_arena) cudaFreeAsync(c->d_key_arena, c->st);
    if (c->d_sched) cudaFreeAsync(c->d_sched, c->st);
    if (c->st) cudaStreamSynchronize(c->st);
    void* bufs[] = {c->d_primes, c->d_tw, c->d_tw_sh, c->d_itw, c->d_itw_sh, c->d_ninv, c->d_ninv_sh,
                    c->d_twd,    c->d_itwd, c->d_ninvd,
                    c->d_modup, c->d_md, c->d_qlinv, c->d_qlinv_sh, c->d_pqlinv, c->d_pqlinv_sh, c->d_s};
    for (void* b : bufs)
        if (b) cudaFree(b);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->t0) cudaEventDestroy(c->t0);
    if (c->t1) cudaEventDestroy(c->t1);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (auto& kv : c->prof)
        for (auto& pr : kv.second.pending) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    for (cudaStream_t l : c->lanes) {
        cudaStreamSynchronize(l);
        cudaStreamDestroy(l);
    }
    for (cudaStream_t x : {c->h2d_st, c->d2h_st})
        if (x) {
            cudaStreamSynchronize(x);
            cudaStreamDestroy(x);
        }
    host_pipe_free(c);
    for (auto& kv : c->lt_cache) cudaFree(kv.second);
    for (auto& le : c->linear_cache)
        for (fhe_pt* pt : le.pts)
            if (pt) {
                cudaFree(pt->d);
                delete pt;
            }
    for (auto& g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (int b = 0; b < 2; ++b)
        for (cudaEvent_t e : {c->hp.ev_h2d[b], c->hp.ev_comp[b], c->hp.ev_d2h[b]})
            if (e) cudaEventDestroy(e);
    if (c->main_st) cudaStreamDestroy(c->main_st);
    delete c;
}

const char* fhe_last_error(const fhe_ctx* c) { return c ? c->err.c_str() : "null context"; }

int fhe_ctx_info(const fhe_ctx* c, int* log_n, int* n_q, int* n_p, int* dnum, uint64_t* primes) {
    if (!c) return FHE_E_INVALID;
    if (log_n) *log_n = c->logN;
    if (n_q) *n_q = c->L;
    if (n_p) *n_p = c->K;
    if (dnum) *dnum = c->dnum;
    if (primes) std::copy(c->primes.begin(), c->primes.end(), primes);
    return FHE_OK;
}

int fhe_synchronize(fhe_ctx* c) {
    return guard(c, [&] {
        ck(cudaStreamSynchronize(c->main_st), "cudaStreamSynchronize");
        for (cudaStream_t l : c->lanes) ck(cudaStreamSynchronize(l), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(c->h2d_st), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(c->d2h_st), "cudaStreamSynchronize");
    });
}

int fhe_timer_start(fhe_ctx* c) {
    return guard(c, [&] {
        if (!c->t0) ck(cudaEventCreate(&c->t0), "cudaEventCreate");
        if (!c->t1) ck(cudaEventCreate(&c->t1), "cudaEventCreate");
        ck(cudaEventRecord(c->t0, c->st), "cudaEventRecord");
    });
}

int fhe_timer_stop(fhe_ctx* c, float* ms) {
    return guard(c, [&] {
        if (!c->t0) fail(FHE_E_INVALID, "timer not started");
        ck(cudaEventRecord(c->t1, c->st), "cudaEventRecord");
        ck(cudaEventSynchronize(c->t1), "cudaEventSynchronize");
        ck(cudaEventElapsedTime(ms, c->t0, c->t1), "cudaEventElapsedTime");
    });
}

int fhe_prof_enable(fhe_ctx* c, int on) {
    return guard(c, [&] {
        c->prof_collect();
        c->prof_on = on != 0;
    });
}

int fhe_prof_get(fhe_ctx* c, const char* cls, double* total_ms, uint64_t* launches) {
    return fhe_prof_get_bytes(c, cls, total_ms, launches, nullptr);
}

int fhe_prof_get_bytes(fhe_ctx* c, const char* cls, double* total_ms, uint64_t* launches, double* bytes) {
    return guard(c, [&] {
        c->prof_collect();
        auto it = c->prof.find(cls);
        if (total_ms) *total_ms = it == c->prof.end() ? 0.0 : it->second.ms;
        if (launches) *launches = it == c->prof.end() ? 0 : it->second.n;
        if (bytes) *bytes = it == c->prof.end() ? 0.0 : it->second.bytes;
    });
}

int fhe_bench_ntt(fhe_ctx* c, int nrows, int inverse, int iters, float* ms) {
    return guard(c, [&] {
        const int level = c->L - 1;
        uint64_t* d = c->alloc((size_t)nrows * c->N);
        ck(cudaMemsetAsync(d, 0, (size_t)nrows * c->N * 8, c->st), "memset");
        const RowMap rm{level + 1, level, c->L, 0};
        for (int i = 0; i < 2; ++i)
            inverse ? ntt_inverse(c->dc, d, nrows, rm, c->st) : ntt_forward(c->dc, d, nrows, rm, c->st);
        cudaEvent_t a = c->get_event(), b = c->get_event();
        cudaEventRecord(a, c->st);
        for (int i = 0; i < iters; ++i)
            inverse ? ntt_inverse(c->dc, d, nrows, rm, c->st) : ntt_forward(c->dc, d, nrows, rm, c->st);
        cudaEventRecord(b, c->st);
        ck(cudaEventSynchronize(b), "sync");
        float t = 0;
        cudaEventElapsedTime(&t, a, b);
        *ms = t / iters;
        c->ev_pool.push_back(a);
        c->ev_pool.push_back(b);
        c->release(d);
    });
}

int fhe_profiler_range(int on) { return (on ? cudaProfilerStart() : cudaProfilerStop()) == cudaSuccess ? 0 : FHE_E_CUDA; }

int fhe_prof_reset(fhe_ctx* c) {
    return guard(c, [&] {
        c->prof_collect();
        c->prof.clear();
    });
}

int fhe_ledger_get(const fhe_ctx* c, fhe_ledger* out) {
    if (!c || !out) return FHE_E_INVALID;
    *out = c->ledger;
    out->kernel_launches = launches_total() - c->launch_base;
    out->distinct_amounts = c->amounts.size();
    return FHE_OK;
}
int fhe_ledger_reset(fhe_ctx* c) {
    if (!c) return FHE_E_INVALID;
    c->ledger = fhe_ledger{};
    c->amounts.clear();
    c->launch_base = launches_total();
    return FHE_OK;
}
int fhe_ledger_amounts(const fhe_ctx* c, uint64_t* out, size_t cap, size_t* n) {
    if (!c) return FHE_E_INVALID;
    size_t i = 0;
    for (uint64_t a : c->amounts) {
        if (i < cap && out) out[i] = a;
        ++i;
    }
    if (n) *n = i;
    return FHE_OK;
}

int fhe_keygen(fhe_ctx* c, uint64_t seed) {
    return guard(c, [&] {
        const size_t N = c->N;
        if (!c->d_s) ck(cudaMalloc(&c->d_s, (size_t)c->np * N * 8), "cudaMalloc");
        // captured graphs hold the device addresses of the keys released below
        drop_graphs(c);
        c->key_gen++;  // layers rebuild their limb key copies on next use
        for (auto& kv : c->keys) c->release(kv.second);
        c->keys.clear();
        c->keys_opf.clear();  // the arena is reused from slot 0
        c->key_slot.clear();
        c->arena_n = 0;
        int64_t* s = (int64_t*)c->alloc(N);
        sample_ternary(c->dc, s, stream_key(seed, stream_id(DOM_SECRET, 0, 0)), c->st);
        const RowMap all{c->np, c->L - 1, c->L, 0};
        reduce_signed_rows(c->dc, s, c->d_s, c->np, all, c->st);
        ntt_forward(c->dc, c->d_s, c->np, all, c->st);
        c->release(s);
        c->key_seed = seed;
        c->have_key = true;
        ck(cudaStreamSynchronize(c->st), "keygen");
    });
}

int fhe_gen_galois_keys(fhe_ctx* c, const int64_t* steps, size_t n) {
    return guard(c, [&] {
        require_key(c);
        for (size_t i = 0; i < n; ++i) {
            const uint64_t a = c->reduce_amount(steps[i]);
            if (a == 0) continue;
            const uint32_t g = c->galois_of(a);
            if (c->keys.count(g)) continue;
            // keys are allocated with cudaMalloc (long-lived) via a pool copy
            gen_key(c, g);
        }
        ck(cudaStreamSynchronize(c->st), "galois keys");
    });
}

int fhe_galois_key_download(fhe_ctx* c, int64_t step, uint64_t* host, size_t words) {
    return guard(c, [&] {
        const uint32_t g = c->galois_of(c->reduce_amount(step));
        const size_t need = (size_t)c->dnum * 2 * c->np * c->N;
        if (words < need) fail(FHE_E_INVALID, "buffer too small");
        ck(cudaMemcpyAsync(host, c->key_for(g), need * 8, cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaStreamSynchronize(c->st), "sync");
    });
}

int fhe_encode(fhe_ctx* c, const double* z, size_t n, int level, double scale, int with_special, fhe_pt** out) {
    return guard(c, [&] {
        if (n == 0 || (n & (n - 1)) != 0 || n > c->slots())
            fail(FHE_E_INVALID, "slot count must be a power of two");
        if (level < 0 || level >= c->L) fail(FHE_E_INVALID, "level out of range");
        const int rows = level + 1 + (with_special ? c->K : 0);
        fhe_pt* pt = new fhe_pt{c, level, rows, scale, c->alloc((size_t)rows * c->N)};
        try {
            encode_rows(c, z, n, level, scale, rows, pt->d);
        } catch (...) {
            c->release(pt->d);
            delete pt;
            throw;
        }
        *out = pt;
    });
}

int fhe_encrypt(fhe_ctx* c, const fhe_pt* pt, uint64_t seed, fhe_ct** out) {
    return guard(c, [&] {
        require_key(c);
        const int level = pt->level, nr = level + 1;
        const size_t N = c->N;
        fhe_ct* ct = new_ct(c, level, pt->scale, 0);
        int64_t* e = (int64_t*)c->alloc(N);
        uint64_t* erows = c->alloc((size_t)nr * N);
        sample_gauss(c->dc, e, stream_key(seed, stream_id(DOM_ENC_E, 0, 0)), c->st);
        reduce_signed_rows(c->dc, e, erows, nr, qmap(c, level), c->st);
        ntt_forward(c->dc, erows, nr, qmap(c, level), c->st);
        sample_uniform_rows(c->dc, ct->c1(), nr, qmap(c, level), stream_key(seed, stream_id(DOM_ENC_A, 0, 0)),
                            c->st);
        encrypt_combine(c->dc, ct->c0(), ct->c1(), erows, c->d_s, pt->d, nr, c->st);
        c->release(e);
        c->release(erows);
        *out = ct;
    });
}

int fhe_decrypt_decode(fhe_ctx* c, const fhe_ct* ct, double* out, size_t n) {
    return guard(c, [&] {
        require_key(c);
        if (n > c->slots()) fail(FHE_E_INVALID, "slot count mismatch");
        const size_t N = c->N;
        const int nr = ct->level + 1, use = std::min(nr, 2);
        uint64_t* m = c->alloc((size_t)use * N);
        decrypt_combine(c->dc, m, ct->c0(), ct->c1(), c->d_s, use, c->st);
        ntt_inverse(c->dc, m, use, qmap(c, ct->level), c->st);
        uint64_t* h = (uint64_t*)c->stage((size_t)use * N * 8);
        ck(cudaMemcpyAsync(h, m, (size_t)use * N * 8, cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaStreamSynchronize(c->st), "sync");
        c->release(m);
        std::vector<double> coef(N);
        const uint64_t q0 = c->primes[0];
        if (use == 1) {
            for (size_t k = 0; k < N; ++k) coef[k] = h[k] > q0 / 2 ? -(double)(q0 - h[k]) : (double)h[k];
        } else {
            using host::u128;
            const uint64_t q1 = c->primes[1];
            const uint64_t inv = host::invmod(q0 % q1, q1);
            const u128 Q = (u128)q0 * q1;
            for (size_t k = 0; k < N; ++k) {
                const uint64_t x0 = h[k], x1 = h[N + k];
                const uint64_t x0m = x0 % q1;
                const uint64_t d = x1 >= x0m ? x1 - x0m : x1 + q1 - x0m;
                const uint64_t tq = host::mulmod(d, inv, q1);
                const u128 X = (u128)x0 + (u128)q0 * tq;
                coef[k] = X > Q / 2 ? -(double)(Q - X) : (double)X;
            }
        }
        host::decode(coef.data(), N, ct->scale, out, n);
    });
}

int fhe_ct_level(const fhe_ct* ct) { return ct ? ct->level : -1; }
double fhe_ct_scale(const fhe_ct* ct) { return ct ? ct->scale : 0.0; }
int fhe_pt_rows(const fhe_pt* pt) { return pt ? pt->rows : -1; }

int fhe_ct_download(fhe_ctx* c, const fhe_ct* ct, uint64_t* host, size_t words) {
    return guard(c, [&] {
        if (words < ct->words()) fail(FHE_E_INVALID, "buffer too small");
        ck(cudaMemcpyAsync(host, ct->d, ct->words() * 8, cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaStreamSynchronize(c->st), "sync");
    });
}

int fhe_ct_upload(fhe_ctx* c, const uint64_t* host, int level, double scale, fhe_ct** out) {
    return guard(c, [&] {
        if (level < 0 || level >= c->L) fail(FHE_E_INVALID, "level out of range");
        fhe_ct* ct = new_ct(c, level, scale, 0);
        ck(cudaMemcpyAsync(ct->d, host, ct->words() * 8, cudaMemcpyHostToDevice, c->st), "H2D");
        *out = ct;
    });
}

int fhe_ct_upload_into(fhe_ctx* c, const uint64_t* host, fhe_ct* ct) {
    return guard(c, [&] {
        ck(cudaMemcpyAsync(ct->d, host, ct->words() * 8, cudaMemcpyHostToDevice, c->st), "H2D");
    });
}

int fhe_pt_download(fhe_ctx* c, const fhe_pt* pt, uint64_t* host, size_t words) {
    return guard(c, [&] {
        const size_t need = (size_t)pt->rows * c->N;
        if (words < need) fail(FHE_E_INVALID, "buffer too small");
        ck(cudaMemcpyAsync(host, pt->d, need * 8, cudaMemcpyDeviceToHost, c->st), "D2H");
        ck(cudaStreamSynchronize(c->st), "sync");
    });
}

void fhe_ct_free(fhe_ct* ct) {
    if (!ct) return;
    ct->ctx->release(ct->d);
    delete ct;
}
void fhe_pt_free(fhe_pt* pt) {
    if (!pt) return;
    pt->ctx->release(pt->d);
    delete pt;
}

int fhe_rotate_hoisted(fhe_ctx* c, const fhe_ct* ct, const int64_t* ks, size_t n, fhe_ct** outs) {
    return guard(c, [&] {
        if (n == 0) fail(FHE_E_INVALID, "empty rotation batch");
        const int level = ct->level;
        bool need = false;
        for (size_t i = 0; i < n; ++i) need |= c->reduce_amount(ks[i]) != 0;
        for (size_t i = 0; i < n; ++i)
            if (c->reduce_amount(ks[i])) c->key_for(c->galois_of(c->reduce_amount(ks[i])));
        uint64_t* digits = nullptr;
        if (need) {
            digits = c->alloc((size_t)c->dn_at(level) * c->ne_at(level) * c->N);
            modup(c, ct->c1(), level, digits);
        }
        // all keyed outputs at once: one streaming key-switch launch writes
        // (IP_0 + P sigma(c0), IP_1) per output in the QP basis, then one batched
        // ModDown (ModDown(P x + y) = x + ModDown(y) exactly)
        const int nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
        const size_t extw = (size_t)ne * c->N, ctw = (size_t)2 * nr * c->N;
        std::vector<size_t> keyed;
        for (size_t i = 0; i < n; ++i)
            if (c->reduce_amount(ks[i])) keyed.push_back(i);
        uint64_t* XT = keyed.empty() ? nullptr : c->alloc(keyed.size() * 2 * extw);
        uint64_t* md = keyed.empty() ? nullptr : c->alloc(keyed.size() * ctw);
        for (size_t t0 = 0; t0 < keyed.size(); t0 += kMaxBaby) {
            KsStream kss{};
            kss.digits = digits;
            kss.digit_stride = 0;
            kss.out = XT;
            for (size_t t = t0; t < keyed.size() && kss.n < kMaxBaby; ++t) {
                const uint32_t g = c->galois_of(c->reduce_amount(ks[keyed[t]]));
                kss.galois[kss.n] = g;
                kss.key[kss.n] = c->key_for(g);
                kss.c0[kss.n] = ct->c0();
                kss.slot[kss.n] = (int)t;
                kss.n++;
            }
            c->timed("ks_multi", c->rows((double)kss.n * (2.0 * dn * ne + 2.0 * ne) + (double)dn * ne + nr),
                     [&] { ks_stream(c->dc, kss, 0, c->d_md, level, dn, c->st); });
        }
        c->ledger.key_switches += keyed.size();
        if (!keyed.empty()) moddown(c, XT, level, (int)(2 * keyed.size()), md, nullptr, 1);
        size_t kt = 0;
        for (size_t i = 0; i < n; ++i) {
            const uint64_t a = c->reduce_amount(ks[i]);
            c->note_amount(a);
            fhe_ct* o = new_ct(c, level, ct->scale, ct->depth);
            const uint64_t* src = a == 0 ? ct->d : md + (kt++) * ctw;
            ck(cudaMemcpyAsync(o->d, src, ct->words() * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
            outs[i] = o;
        }
        c->release(md);
        c->release(XT);
        c->release(digits);
        c->ledger.hoist_groups++;
        c->ledger.hoisted_rotations += n;
    });
}

// Hoisted rotations of a batch: outs[i * k + j] = rot_{ks[j]}(cts[i]). One
// batched ModUp, one staged key-switch launch per chunk of sources (each key
// row staged once per CTA for up to 4 ciphertexts), one batched ModDown.
static void rotate_hoisted_batch_impl(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const int64_t* ks, size_t k,
                                      fhe_ct** outs, bool into) {
    {
        if (k == 0) fail(FHE_E_INVALID, "empty rotation batch");
        if (n == 0) return;
        const int level = cts[0]->level;
        for (size_t i = 0; i < n; ++i)
            if (cts[i]->level != level) fail(FHE_E_INVALID, "batched rotation: all inputs must share one level");
        std::vector<size_t> keyed;
        for (size_t j = 0; j < k; ++j)
            if (c->reduce_amount(ks[j])) {
                c->key_for(c->galois_of(c->reduce_amount(ks[j])));  // fails early on a missing key
                keyed.push_back(j);
            }
        const int nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
        const size_t N = c->N, extw = (size_t)ne * N, ctw = (size_t)2 * nr * N, dw = (size_t)dn * extw;
        const size_t KK = keyed.size();
        // sources per chunk: as many as ~4 GB of temporaries hold (input copies, digits,
        // QP key-switch outputs), at most 256; large chunks keep small rings (cfg2) busy
        const size_t per_src = 8 * (ctw + dw + KK * 2 * extw);
        const size_t SC = std::max<size_t>(1, std::min<size_t>({n, (size_t)256, ((size_t)4 << 30) / per_src}));
        uint64_t *buf = nullptr, *dig = nullptr, *XT = nullptr;
        uint64_t** outp = nullptr;  // device table of the keyed outputs' residue buffers (ModDown writes there)
        uint64_t** inp = nullptr;   // device table of the chunk's input residue buffers (one gather launch)
        std::vector<uint64_t*> hostp, hostin;
        if (KK) {
            inp = (uint64_t**)c->alloc(SC);
            buf = c->alloc(SC * ctw);
            dig = c->alloc(SC * dw);
            XT = c->alloc(SC * KK * 2 * extw);
            outp = (uint64_t**)c->alloc(SC * KK);
        }
        for (size_t s0 = 0; s0 < n; s0 += SC) {
            const size_t sn = std::min(SC, n - s0);
            if (KK) {
                static const size_t gather_min = [] {  // FHECONV_GATHER_MIN: batch size from which inputs are gathered
                    const char* e = getenv("FHECONV_GATHER_MIN");
                    return (size_t)(e ? std::max(1, atoi(e)) : 8);  // A/B at cfg3 batch 16: 8 is 1.5-4 % faster than 32
                }();
                if (sn >= gather_min) {  // many inputs: one gather launch instead of a copy per ciphertext (~4 us each)
                    hostin.resize(sn);
                    for (size_t s = 0; s < sn; ++s) hostin[s] = cts[s0 + s]->d;
                    ck(cudaMemcpyAsync(inp, hostin.data(), sn * sizeof(uint64_t*), cudaMemcpyHostToDevice, c->st),
                       "memcpy");
                    gather_ptrs(buf, inp, ctw, (int)sn, c->st);
                } else {
                    for (size_t s = 0; s < sn; ++s)
                        ck(cudaMemcpyAsync(buf + s * ctw, cts[s0 + s]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st),
                           "memcpy");
                }
                // operand-form digits and P-scaled ciphertexts (k_ks_hoist_opf: FP64 products on
                // the rows q < 2^50); buf then holds [P c]_q in operand form
                modup_batch(c, buf + (size_t)nr * N, ctw, (int)sn, level, dig, 1);
                ct_prescale(c->dc, buf, buf, ctw, (int)sn, c->d_md, level, c->st);
                if (c->tma) {  // k_bsgs_tma MODE 1: TMA staging, keys from the arena, work queues
                    TmaMaps tm{};
                    tma_rows(c, level, tm);
                    const uint32_t sg = (uint32_t)tma_sources((int)sn), P2 = 256u / sg;
                    const uint64_t dk[4] = {N, (uint64_t)c->np, 2ull * c->dnum, (uint64_t)c->arena_n};
                    const uint32_t bk[4] = {P2, 1, 2u * dn, 1};
                    tma_map4(&tm.key, c->d_key_arena, dk, bk);
                    const uint64_t dd[5] = {N, (uint64_t)ne, (uint64_t)dn, 1, (uint64_t)sn};
                    const uint32_t bd[5] = {P2, 1, (uint32_t)dn, 1, sg};
                    tma_map5(&tm.dig, dig, dd, bd);
                    const uint64_t dc5[5] = {N, (uint64_t)nr, 2, 1, (uint64_t)sn};
                    const uint32_t bc[5] = {P2, 1, 2, 1, sg};
                    tma_map5(&tm.ct, buf, dc5, bc);
                    for (size_t t0 = 0; t0 < KK; t0 += kMaxFused) {
                        FusedBsgs f{};
                        f.nsrc = (int)sn;
                        f.ng = 1;
                        f.digits = dig;
                        f.ct = buf;
                        f.Y = XT + t0 * 2 * extw;
                        f.y_src_stride = KK * 2 * extw;
                        f.y_g_stride = 2 * extw;
                        for (size_t t = t0; t < KK && f.nb < kMaxFused; ++t) {
                            const uint32_t g = c->galois_of(c->reduce_amount(ks[keyed[t]]));
                            f.galois[f.nb] = g;
                            tm.kidx[f.nb] = (int16_t)c->key_slot.at(g);
                            f.nb++;
                        }
                        c->timed("ks_multi",
                                 c->rows((double)f.nb * 2.0 * dn * ne + sn * ((double)dn * ne + nr + 2.0 * f.nb * ne)),
                                 [&] { bsgs_tma_hoist(c->dc, f, tm, level, dn, c->st); });
                    }
                }
                for (size_t t0 = 0; t0 < KK && !c->tma; t0 += kMaxBaby) {
                    KsBatch kb{};
                    kb.nsrc = (int)sn;
                    kb.digits = dig;
                    kb.digit_src_stride = dw;
                    kb.c0 = buf;
                    kb.c0_src_stride = ctw;
                    kb.opf = 1;
                    kb.out = XT;
                    kb.out_src_stride = KK * 2 * extw;
                    for (size_t t = t0; t < KK && kb.n < kMaxBaby; ++t) {
                        const uint32_t g = c->galois_of(c->reduce_amount(ks[keyed[t]]));
                        kb.galois[kb.n] = g;
                        kb.key[kb.n] = c->key_opf_for(g);
                        kb.slot[kb.n] = (int)t;
                        kb.n++;
                    }
                    c->timed("ks_multi",
                             c->rows((double)kb.n * 2.0 * dn * ne + sn * ((double)dn * ne + nr + 2.0 * kb.n * ne)),
                             [&] { ks_batch(c->dc, kb, 0, c->d_md, level, dn, c->st); });
                }
                c->ledger.key_switches += sn * KK;
            }
            // outputs first (the keyed ones receive the ModDown directly, no staging copy)
            hostp.assign(sn * KK, nullptr);
            for (size_t s = 0; s < sn; ++s) {
                size_t kt = 0;
                for (size_t j = 0; j < k; ++j) {
                    const uint64_t a = c->reduce_amount(ks[j]);
                    c->note_amount(a);
                    fhe_ct* o = into ? outs[(s0 + s) * k + j] : new_ct(c, level, cts[s0 + s]->scale, cts[s0 + s]->depth);
                    if (into) {
                        if (!o || o->level != level) fail(FHE_E_INVALID, "output ciphertext level mismatch");
                        if (o == cts[s0 + s]) fail(FHE_E_INVALID, "output ciphertext aliases an input");
                        o->scale = cts[s0 + s]->scale;
                        o->depth = cts[s0 + s]->depth;
                    }
                    if (a == 0)
                        ck(cudaMemcpyAsync(o->d, cts[s0 + s]->d, ctw * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
                    else
                        hostp[s * KK + kt++] = o->d;
                    outs[(s0 + s) * k + j] = o;
                }
            }
            if (KK) {
                ck(cudaMemcpyAsync(outp, hostp.data(), hostp.size() * sizeof(uint64_t*), cudaMemcpyHostToDevice, c->st),
                   "memcpy");
                moddown_strided(c, XT, (size_t)ne * N, level, (int)(2 * sn * KK), nullptr, nullptr, 1, outp);
            }
            c->ledger.hoist_groups += sn;
            c->ledger.hoisted_rotations += sn * k;
        }
        c->release(outp);
        c->release(XT);
        c->release(dig);
        c->release(buf);
        c->release(inp);
    }
}

int fhe_rotate_hoisted_batch(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const int64_t* ks, size_t k,
                             fhe_ct** outs) {
    return guard(c, [&] { rotate_hoisted_batch_impl(c, cts, n, ks, k, outs, false); });
}

int fhe_rotate_hoisted_batch_into(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const int64_t* ks, size_t k,
                                  fhe_ct* const* outs) {
    return guard(c, [&] { rotate_hoisted_batch_impl(c, cts, n, ks, k, const_cast<fhe_ct**>(outs), true); });
}

int fhe_rotate(fhe_ctx* c, const fhe_ct* ct, int64_t k, fhe_ct** out) {
    return guard(c, [&] {
        const uint64_t a = c->reduce_amount(k);
        c->note_amount(a);
        fhe_ct* o = new_ct(c, ct->level, ct->scale, ct->depth);
        if (a == 0) {
            ck(cudaMemcpyAsync(o->d, ct->d, ct->words() * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        } else {
            const uint32_t g = c->galois_of(a);
            c->key_for(g);
            uint64_t* digits = c->alloc((size_t)c->dn_at(ct->level) * c->ne_at(ct->level) * c->N);
            modup(c, ct->c1(), ct->level, digits);
            rotate_from_digits(c, ct, digits, g, o->d);
            c->release(digits);
            c->ledger.rotations++;
        }
        *out = o;
    });
}

int fhe_decompose(int strategy, uint64_t n, uint64_t s, int64_t* steps, int cap) {
    // reference rot.cpp:21-46
    if (n >= s) return FHE_E_INVALID;
    auto floor_pow2 = [](uint64_t v) {
        uint64_t p = 1;
        while (p * 2 <= v) p *= 2;
        return p;
    };
    int k = 0;
    if (strategy == 0) {
        for (uint64_t bit = floor_pow2(s); bit >= 1; bit /= 2) {
            if (n & bit) {
                if (k >= cap) return FHE_E_INVALID;
                steps[k++] = (int64_t)bit;
            }
            if (bit == 1) break;
        }
        return k;
    }
    int64_t rest = (int64_t)n;
    while (rest != 0) {
        const uint64_t mag = (uint64_t)(rest < 0 ? -rest : rest);
        const uint64_t lo = floor_pow2(mag), hi = lo * 2;
        const uint64_t pick = (mag - lo <= hi - mag) ? lo : hi;
        const int64_t step = rest < 0 ? -(int64_t)pick : (int64_t)pick;
        if (k >= cap) return FHE_E_INVALID;
        steps[k++] = step;
        rest -= step;
    }
    return k;
}

int fhe_rotate_decomposed(fhe_ctx* c, const fhe_ct* ct, int64_t k, int strategy, fhe_ct** out) {
    return guard(c, [&] {
        const uint64_t a = c->reduce_amount(k);
        int64_t steps[64];
        const int ns = fhe_decompose(strategy, a, c->slots(), steps, 64);
        if (ns < 0) fail(FHE_E_INVALID, "decomposition failed");
        fhe_ct* cur = new_ct(c, ct->level, ct->scale, ct->depth);
        ck(cudaMemcpyAsync(cur->d, ct->d, ct->words() * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        uint64_t* digits = c->alloc((size_t)c->dn_at(ct->level) * c->ne_at(ct->level) * c->N);
        fhe_ct* nxt = new_ct(c, ct->level, ct->scale, ct->depth);
        for (int i = 0; i < ns; ++i) {
            const uint64_t sa = c->reduce_amount(steps[i]);
            c->note_amount(sa);
            if (sa == 0) continue;  // a full-cycle step is the identity
            modup(c, cur->c1(), ct->level, digits);
            rotate_from_digits(c, cur, digits, c->galois_of(sa), nxt->d);
            std::swap(cur, nxt);
            c->ledger.rotations++;
        }
        c->release(digits);
        fhe_ct_free(nxt);
        *out = cur;
    });
}

static void okc(fhe_ctx* c, int rc);

// plan_rotations + execute_schedule (reference rot.cpp:96-156): requests join
// the previous group when flagged same_source (the group becomes hoisted); a
// hoisted group rotates by its members' first keyed steps as one hoisted batch
// (one ModUp of the source), then each member's remaining steps sequentially;
// other groups rotate sequentially from the source. Steps equal to a full
// cycle (the signed decomposition's +-s) are counted as the reference counts
// them but executed as the identity.
int fhe_execute_schedule(fhe_ctx* c, const fhe_ct* src, const int64_t* amounts, const int* same_source, size_t n,
                         int strategy, fhe_ct** outs, uint64_t* planned_keyed, uint64_t* groups_out,
                         uint64_t* hoisted_groups_out) {
    return guard(c, [&] {
        if (!src || !amounts || !outs) fail(FHE_E_INVALID, "null argument");
        if (strategy < 0 || strategy > 2) fail(FHE_E_INVALID, "unknown decomposition strategy");
        const uint64_t s = c->slots();
        struct Group {
            std::vector<std::vector<int64_t>> steps;
            std::vector<size_t> req;
            bool hoisted = false;
        };
        std::vector<Group> groups;
        uint64_t total = 0;
        for (size_t i = 0; i < n; ++i) {
            const uint64_t a = c->reduce_amount(amounts[i]);
            std::vector<int64_t> st;
            if (a != 0) {
                if (strategy == 2) {
                    st.push_back((int64_t)a);
                } else {
                    int64_t buf[64];
                    const int ns = fhe_decompose(strategy, a, s, buf, 64);
                    if (ns < 0) fail(FHE_E_INVALID, "decomposition failed");
                    st.assign(buf, buf + ns);
                }
            }
            total += st.size();
            if (same_source && same_source[i] && !groups.empty()) {
                groups.back().steps.push_back(st);
                groups.back().req.push_back(i);
                groups.back().hoisted = true;
            } else {
                groups.push_back(Group{{st}, {i}, false});
            }
        }
        auto rotate_chain = [&](fhe_ct* cur, const std::vector<int64_t>& st, size_t from) {
            for (size_t k = from; k < st.size(); ++k) {
                fhe_ct* nx = nullptr;
                const int rc = fhe_rotate(c, cur, st[k], &nx);
                fhe_ct_free(cur);
                okc(c, rc);
                cur = nx;
            }
            return cur;
        };
        std::vector<fhe_ct*> res(n, nullptr);
        try {
            for (const Group& g : groups) {
                if (g.hoisted) {
                    std::vector<int64_t> firsts;
                    for (const auto& st : g.steps) firsts.push_back(st.empty() ? 0 : st[0]);
                    std::vector<fhe_ct*> batch(firsts.size(), nullptr);
                    okc(c, fhe_rotate_hoisted(c, src, firsts.data(), firsts.size(), batch.data()));
                    for (size_t m2 = 0; m2 < g.steps.size(); ++m2) res[g.req[m2]] = rotate_chain(batch[m2], g.steps[m2], 1);
                } else {
                    fhe_ct* cur = nullptr;
                    okc(c, fhe_rotate(c, src, 0, &cur));  // copy (recorded like the reference's v = source)
                    res[g.req[0]] = rotate_chain(cur, g.steps[0], 0);
                }
            }
        } catch (...) {
            for (fhe_ct* x : res)
                if (x) fhe_ct_free(x);
            throw;
        }
        for (size_t i = 0; i < n; ++i) outs[i] = res[i];
        if (planned_keyed) *planned_keyed = total;
        if (groups_out) *groups_out = groups.size();
        if (hoisted_groups_out) {
            uint64_t h = 0;
            for (const Group& g : groups) h += g.hoisted;
            *hoisted_groups_out = h;
        }
    });
}

int fhe_mul_plain(fhe_ctx* c, const fhe_ct* ct, const fhe_pt* pt, fhe_ct** out) {
    return guard(c, [&] {
        if (pt->level < ct->level) fail(FHE_E_INVALID, "slot count mismatch");
        if (ct->level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
        fhe_ct* o = new_ct(c, ct->level, ct->scale * pt->scale, ct->depth + 1);
        ew_mul_bcast(c->dc, o->d, ct->d, pt->d, 2 * (ct->level + 1), ct->level + 1, c->st);
        c->ledger.ct_pt_mults++;
        c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, o->depth);
        *out = o;
    });
}

int fhe_add(fhe_ctx* c, const fhe_ct* a, const fhe_ct* b, fhe_ct** out) {
    return guard(c, [&] {
        if (a->level != b->level) fail(FHE_E_INVALID, "level mismatch");
        fhe_ct* o = new_ct(c, a->level, a->scale, std::max(a->depth, b->depth));
        ew_add(c->dc, o->d, a->d, b->d, 2 * (a->level + 1), a->level + 1, c->st);
        c->ledger.adds++;
        *out = o;
    });
}

int fhe_sub(fhe_ctx* c, const fhe_ct* a, const fhe_ct* b, fhe_ct** out) {
    return guard(c, [&] {
        if (a->level != b->level) fail(FHE_E_INVALID, "level mismatch");
        fhe_ct* o = new_ct(c, a->level, a->scale, std::max(a->depth, b->depth));
        ew_sub(c->dc, o->d, a->d, b->d, 2 * (a->level + 1), a->level + 1, c->st);
        c->ledger.adds++;
        *out = o;
    });
}

int fhe_add_plain(fhe_ctx* c, const fhe_ct* ct, const fhe_pt* pt, fhe_ct** out) {
    return guard(c, [&] {
        if (pt->level < ct->level) fail(FHE_E_INVALID, "slot count mismatch");
        const int nr = ct->level + 1;
        fhe_ct* o = new_ct(c, ct->level, ct->scale, ct->depth);
        ck(cudaMemcpyAsync(o->c1(), ct->c1(), (size_t)nr * c->N * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
        ew_add(c->dc, o->c0(), ct->c0(), pt->d, nr, nr, c->st);
        c->ledger.adds++;
        *out = o;
    });
}

int fhe_rescale(fhe_ctx* c, const fhe_ct* ct, fhe_ct** out) {
    return guard(c, [&] {
        if (ct->level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
        fhe_ct* o = new_ct(c, ct->level - 1, ct->scale / (double)c->primes[ct->level], ct->depth);
        rescale_into(c, ct->d, ct->level, o->d);
        *out = o;
    });
}

// weights * output_scale, as ImageConv folds its scale into every fused plaintext
// (conv.cpp:74: k.centered(...) * scale -- the same double product)
static std::vector<double> scaled_weights(int c_in, int c_out, int kappa, const double* w, double osc) {
    if (!w) fail(FHE_E_INVALID, "null weights");
    std::vector<double> v(w, w + (size_t)c_in * c_out * kappa * kappa);
    for (double& x : v) x = x * osc;
    return v;
}

int fhe_conv_layer_create(fhe_ctx* c, int c_in, int c_out, int m, int kappa, const double* weights_in,
                          const double* bias, double output_scale, int level, fhe_conv_layer** out) {
    return guard(c, [&] {
        if (!out) fail(FHE_E_INVALID, "null output");
        const std::vector<double> wsc = scaled_weights(c_in, c_out, kappa, weights_in, output_scale);
        const double* weights = wsc.data();
        if (kappa % 2 == 0) fail(FHE_E_INVALID, "kernel size must be odd");
        if (c_out <= 0 || (c_out & (c_out - 1))) fail(FHE_E_INVALID, "output channel count must be a power of two");
        const size_t s = c->slots(), block = (size_t)m * m;
        if (m <= 0 || (m & (m - 1)) || block > s || (size_t)c_in * block > s)
            fail(FHE_E_INVALID, "image does not fit one shard");
        if ((size_t)c_out * block > s) fail(FHE_E_INVALID, "insufficient capacity");
        if (kappa / 2 >= m) fail(FHE_E_INVALID, "kernel reach exceeds channel size");
        if (level < 1 || level >= c->L) fail(FHE_E_INVALID, "level out of range");
        fhe_conv_layer* ly = new fhe_conv_layer();
        ly->ctx = c;
        ly->c_in = c_in;
        ly->c_out = c_out;
        ly->m = m;
        ly->kappa = kappa;
        ly->level = level;
        ly->nk = kappa * kappa;
        ly->weights.assign(weights, weights + (size_t)c_in * c_out * kappa * kappa);
        const int ne = c->ne_at(level);
        ly->pt_words = (size_t)c_in * ly->nk * ne * c->N;
        ck(cudaMalloc(&ly->d_pts, ly->pt_words * 8), "cudaMalloc");
        ly->nonempty.assign((size_t)c_in * ly->nk, 0);
        const double pscale = (double)c->primes[level];
        std::vector<double> plain;
        const long h = kappa / 2;
        for (int r = 0; r < c_in; ++r) {
            int i = 0;
            for (long kk = -h; kk <= h; ++kk)
                for (long ll = -h; ll <= h; ++ll, ++i) {
                    if (!fused_plain(c_in, c_out, m, kappa, s, weights, r, kk, ll, plain)) continue;
                    ly->nonempty[(size_t)r * ly->nk + i] = 1;
                    encode_rows(c, plain.data(), s, level, pscale, ne,
                                ly->d_pts + ((size_t)r * ly->nk + i) * ne * c->N);
                }
        }
        set_bias(c, ly, bias, output_scale);
        ck(cudaStreamSynchronize(c->st), "sync");
        *out = ly;
    });
}

void fhe_conv_layer_free(fhe_conv_layer* ly) {
    if (!ly) return;
    cudaStreamSynchronize(ly->ctx->st);
    auto& gs = ly->ctx->graphs;  // drop the layer's captured graphs (they reference its plaintexts)
    for (size_t i = 0; i < gs.size();) {
        if (!gs[i].key.empty() && gs[i].key[0] == (const void*)(uintptr_t)ly->uid) {
            cudaGraphExecDestroy(gs[i].exec);
            gs.erase(gs.begin() + (long)i);
        } else {
            ++i;
        }
    }
    cudaFree(ly->d_pts);
    if (ly->d_pts_ms) cudaFree(ly->d_pts_ms);
    if (ly->d_pts_ms_opf) cudaFree(ly->d_pts_ms_opf);
    if (ly->d_pts_cs_opf) cudaFree(ly->d_pts_cs_opf);
    if (ly->d_bias) cudaFree(ly->d_bias);
    for (auto& b : ly->bs) {
        if (b.d_pts) cudaFree(b.d_pts);
        if (b.d_pts_limb) cudaFree(b.d_pts_limb);
        if (b.d_keys_limb) cudaFree(b.d_keys_limb);
    }
    if (ly->d_pts_opf) cudaFree(ly->d_pts_opf);
    for (auto& k : ly->pk)
        if (k.d_keys) cudaFree(k.d_keys);
    delete ly;
}

static fhe_conv_layer* create_packed_layer(fhe_ctx* c, int c_in, int c_out, int m, int kappa, const double* weights,
                                           int level, int T, const int64_t* tau, int rep, int d);

int fhe_conv_layer_create_shards(fhe_ctx* c, int c_in, int c_out, int m, int kappa, const double* weights_in,
                                 const double* bias, double output_scale, int level, fhe_conv_layer** out) {
    return guard(c, [&] {
        if (!out) fail(FHE_E_INVALID, "null output");
        const std::vector<double> wsc = scaled_weights(c_in, c_out, kappa, weights_in, output_scale);
        const double* weights = wsc.data();
        if (kappa % 2 == 0) fail(FHE_E_INVALID, "kernel size must be odd");
        if (c_out <= 0 || (c_out & (c_out - 1))) fail(FHE_E_INVALID, "output channel count must be a power of two");
        if (c_in <= 0 || (c_in & (c_in - 1))) fail(FHE_E_INVALID, "channel count must be a power of two");
        const size_t s = c->slots(), block = (size_t)m * m;
        const size_t s2 = s;
        if (m <= 0 || (m & (m - 1))) fail(FHE_E_INVALID, "channel side must be a power of two");
        if (block > s2) {  // channel-shard mode (reference conv_channel_shards, conv.cpp:273-362)
            const long rows = (long)(s2 / (size_t)m), h = kappa / 2;
            if (h > rows) fail(FHE_E_INVALID, "kernel reach exceeds one neighbor shard");
            if (level < 1 || level >= c->L) fail(FHE_E_INVALID, "level out of range");
            fhe_conv_layer* ly = new fhe_conv_layer();
            ly->ctx = c;
            ly->c_in = c_in;
            ly->c_out = c_out;
            ly->m = m;
            ly->kappa = kappa;
            ly->level = level;
            ly->nk = kappa * kappa;
            ly->d_pts = nullptr;
            ly->weights.assign(weights, weights + (size_t)c_in * c_out * kappa * kappa);
            ly->ms = true;
            ly->cs = true;
            ly->pc = (int)(block / s2);
            ly->t = c_in * ly->pc;
            ly->n_out = c_out * ly->pc;
            const int ne = c->ne_at(level);
            const size_t extw = (size_t)ne * c->N, npt = (size_t)c_out * c_in * kappa * kappa * 2;
            ly->ms_nonempty.assign(npt, 0);
            ck(cudaMalloc(&ly->d_pts_ms, npt * extw * 8), "cudaMalloc");
            const double pscale = (double)c->primes[level];
            std::vector<double> mask, rot(s2);
            size_t idx = 0;
            for (int g = 0; g < c_out; ++g)
                for (int f = 0; f < c_in; ++f)
                    for (long kk = -h; kk <= h; ++kk)
                        for (long ll = -h; ll <= h; ++ll)
                            for (int spill = 0; spill < 2; ++spill, ++idx) {
                                const double w =
                                    weights[(((size_t)f * c_out + g) * kappa + (size_t)(kk + h)) * kappa + (size_t)(ll + h)];
                                if (w == 0.0 || (spill && kk == 0)) continue;
                                if (!cs_mask(m, rows, kk, ll, spill, w, s2, mask)) continue;
                                ly->ms_nonempty[idx] = 1;
                                const uint64_t gsh = c->reduce_amount(kk * m);
                                for (size_t j = 0; j < s2; ++j) rot[j] = mask[(j + s2 - gsh) % s2];  // rot_{-kk m}
                                encode_rows(c, rot.data(), s2, level, pscale, ne, ly->d_pts_ms + idx * extw);
                            }
            set_bias(c, ly, bias, output_scale);
            ck(cudaStreamSynchronize(c->st), "sync");
            *out = ly;
            return;
        }
        if ((size_t)c_in * block < s)
            fail(FHE_E_INVALID, "multi-shard convolution needs c_in m^2 >= slots (no duplication)");
        *out = create_packed_layer(c, c_in, c_out, m, kappa, weights, level, (int)((size_t)c_in * block / s), nullptr,
                                   1, 1);
        set_bias(c, *out, bias, output_scale);
    });
}

// image-mode layer over an arbitrary PackedImage (conv_image_mode, conv.cpp:40-211):
// t shards, tau, rep, d (d > 1 only for one shard)
static fhe_conv_layer* create_packed_layer(fhe_ctx* c, int c_in, int c_out, int m, int kappa, const double* weights,
                                           int level, int T, const int64_t* tau, int rep, int d) {
    const size_t s = c->slots(), block = (size_t)m * m;
    if (kappa % 2 == 0) fail(FHE_E_INVALID, "kernel size must be odd");
    if (c_out <= 0 || (c_out & (c_out - 1))) fail(FHE_E_INVALID, "output channel count must be a power of two");
    if (c_in <= 0 || (c_in & (c_in - 1))) fail(FHE_E_INVALID, "channel count must be a power of two");
    if (m <= 0 || (m & (m - 1)) || block > s) fail(FHE_E_INVALID, "image-mode convolution requires image shards");
    if (T < 1 || rep < 1 || d < 1) fail(FHE_E_INVALID, "metadata mismatch");
    if (T >= 2 && d != 1) fail(FHE_E_INVALID, "metadata mismatch: duplicated multi-shard image");
    if ((size_t)c_in * block * (size_t)d != (size_t)T * s) fail(FHE_E_INVALID, "metadata mismatch: shard count");
    if (kappa / 2 >= m) fail(FHE_E_INVALID, "kernel reach exceeds channel size");
    if (level < 1 || level >= c->L) fail(FHE_E_INVALID, "level out of range");
    const int z = (int)(s / block);
    const int NO = c_out <= z ? 1 : c_out / z;
    if (T > 64) fail(FHE_E_INVALID, "too many input shards");
    std::vector<int64_t> tv((size_t)c_in);
    for (int j = 0; j < c_in; ++j) tv[(size_t)j] = tau ? tau[j] : j;
    {
        std::vector<int> seen((size_t)c_in, 0);
        for (int64_t x : tv)
            if (x < 0 || x >= c_in || seen[(size_t)x]++) fail(FHE_E_INVALID, "tau is not a permutation");
    }
    fhe_conv_layer* ly = new fhe_conv_layer();
    ly->ctx = c;
    ly->c_in = c_in;
    ly->c_out = c_out;
    ly->m = m;
    ly->kappa = kappa;
    ly->level = level;
    ly->nk = kappa * kappa;
    ly->d_pts = nullptr;
    ly->weights.assign(weights, weights + (size_t)c_in * c_out * kappa * kappa);
    ly->ms = true;
    ly->t = T;
    ly->z = z;
    ly->n_out = NO;
    ly->rep = rep;
    ly->tau = tv;
    ly->rmax = T == 1 ? c_in : z;  // ImageConv::r_max (conv.cpp:57)
    ly->nb_ms = T * ly->rmax * kappa;
    const int ne = c->ne_at(level), nb = ly->nb_ms;
    const size_t extw = (size_t)ne * c->N;
    const long h = kappa / 2;
    ly->ms_nonempty.assign((size_t)NO * kappa * nb, 0);
    ck(cudaMalloc(&ly->d_pts_ms, (size_t)NO * kappa * nb * extw * 8), "cudaMalloc");
    const double pscale = (double)c->primes[level];
    std::vector<double> plain, rot(s);
    for (int v = 0; v < NO; ++v)
        for (int gi = 0; gi < kappa; ++gi)
            for (int b = 0; b < nb; ++b) {
                const int u = b / (ly->rmax * kappa), r = (b / kappa) % ly->rmax;
                const long ll = b % kappa - h, kk = gi - h;
                if (!fused_plain_ms(c_out, m, kappa, s, weights, v, u, r, kk, ll, plain, &ly->tau, rep)) continue;
                ly->ms_nonempty[((size_t)v * kappa + gi) * nb + b] = 1;
                const uint64_t g = c->reduce_amount(kk * m);
                for (size_t j = 0; j < s; ++j) rot[j] = plain[(j + s - g) % s];  // rot_{-kk m}
                encode_rows(c, rot.data(), s, level, pscale, ne,
                            ly->d_pts_ms + (((size_t)v * kappa + gi) * nb + b) * extw);
            }
    ck(cudaStreamSynchronize(c->st), "sync");
    return ly;
}

int fhe_conv_layer_create_packed(fhe_ctx* c, int c_in, int c_out, int m, int kappa, const double* weights,
                                 const double* bias, double output_scale, int level, size_t t, const int64_t* tau,
                                 int rep, int d, fhe_conv_layer** out) {
    return guard(c, [&] {
        if (!out) fail(FHE_E_INVALID, "null output");
        const std::vector<double> wsc = scaled_weights(c_in, c_out, kappa, weights, output_scale);
        *out = create_packed_layer(c, c_in, c_out, m, kappa, wsc.data(), level, (int)t, tau, rep, d);
        set_bias(c, *out, bias, output_scale);
    });
}

int fhe_conv_layer_output_packing(const fhe_conv_layer* ly, int* d_out) {
    // ImageConv::make_output (conv.cpp:97-106): d = n_out z / c_out, rep 1, identity tau
    if (!ly) return FHE_E_INVALID;
    if (d_out) *d_out = (ly->ms && !ly->cs) ? std::max(1, ly->n_out * ly->z / ly->c_out) : 1;
    return FHE_OK;
}

int fhe_conv_layer_shards(const fhe_conv_layer* ly, int* t, int* n_out) {
    if (!ly) return FHE_E_INVALID;
    if (t) *t = ly->ms ? ly->t : 1;
    if (n_out) *n_out = ly->ms ? ly->n_out : 1;
    return FHE_OK;
}

int fhe_conv2d_shards_into(fhe_ctx* c, const fhe_ct* const* in, size_t n_images, const fhe_conv_layer* ly,
                           fhe_ct* const* outs) {
    return guard(c, [&] {
        if (!ly || !ly->ms) fail(FHE_E_INVALID, "layer was not created by fhe_conv_layer_create_shards");
        prepare_bias(c, ly, in, n_images * (size_t)ly->t);
        for (size_t i0 = 0; i0 < n_images; i0 += 8) {
            const int B = (int)std::min<size_t>(8, n_images - i0);
            if (ly->cs)
                conv_cs_batch(c, in + i0 * ly->t, B, ly, outs + i0 * ly->n_out);
            else
                conv_ms_batch(c, in + i0 * ly->t, B, ly, outs + i0 * ly->n_out);
        }
    });
}

int fhe_conv_layer_steps(const fhe_conv_layer* ly, int approach, int64_t* steps, size_t cap, size_t* n) {
    // approaches 1-4 rotate by r m^2 and kk m + ll; approach 5 by r m^2 + ll and
    // kk m; approach 0 (auto) lists the union so that every schedule can run
    if (!ly || approach < 0 || approach > 5) return FHE_E_INVALID;
    std::set<int64_t> st;
    const long h = ly->kappa / 2;
    const int64_t block = (int64_t)ly->m * ly->m;
    if (ly->cs) {  // channel-shard layers: column shifts ll and row shifts kk m
        for (long ll = -h; ll <= h; ++ll)
            if (ll) st.insert(ll);
        for (long kk = -h; kk <= h; ++kk)
            if (kk) st.insert(kk * ly->m);
        approach = -1;
    } else if (ly->ms) {  // multi-shard layers run the fused schedule: r m^2 + ll (r < z) and kk m
        for (int r = 0; r < ly->rmax; ++r)
            for (long ll = -h; ll <= h; ++ll)
                if (r || ll) st.insert((int64_t)r * ly->rep * block + ll);
        for (long kk = -h; kk <= h; ++kk)
            if (kk) st.insert(kk * ly->m);
        approach = -1;
    }
    if (approach >= 0 && approach != 5) {
        for (int r = 1; r < ly->c_in; ++r) st.insert((int64_t)r * block);
        for (long kk = -h; kk <= h; ++kk)
            for (long ll = -h; ll <= h; ++ll)
                if (kk || ll) st.insert(kk * ly->m + ll);
    }
    if (approach == 0 || approach == 5) {
        for (int r = 0; r < ly->c_in; ++r)
            for (long ll = -h; ll <= h; ++ll)
                if (r || ll) st.insert((int64_t)r * block + ll);
        for (long kk = -h; kk <= h; ++kk)
            if (kk) st.insert(kk * ly->m);
    }
    size_t i = 0;
    for (int64_t v : st) {
        if (i < cap && steps) steps[i] = v;
        ++i;
    }
    if (n) *n = i;
    return FHE_OK;
}

int fhe_conv2d_into(fhe_ctx* c, const fhe_ct* ct, const fhe_conv_layer* ly, int approach, fhe_ct* out) {
    return guard(c, [&] { batch_impl(c, &ct, 1, ly, approach, &out); });
}

int fhe_conv2d(fhe_ctx* c, const fhe_ct* ct, const fhe_conv_layer* ly, int approach, fhe_ct** out) {
    return guard(c, [&] {
        if (ct->level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
        if (!ly) fail(FHE_E_INVALID, "null layer");
        prepare_bias(c, ly, &ct, 1);
        fhe_ct* o = new_ct(c, ct->level - 1, ct->scale, ct->depth + 1);
        try {
            batch_impl(c, &ct, 1, ly, approach, &o);
        } catch (...) {
            fhe_ct_free(o);
            throw;
        }
        *out = o;
    });
}

int fhe_conv2d_batch(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const fhe_conv_layer* ly, int approach,
                     fhe_ct** outs) {
    return guard(c, [&] {
        std::vector<fhe_ct*> o(n, nullptr);
        try {
            for (size_t i = 0; i < n; ++i) o[i] = new_ct(c, cts[i]->level - 1, cts[i]->scale, cts[i]->depth + 1);
            batch_impl(c, cts, n, ly, approach, o.data());
        } catch (...) {
            for (fhe_ct* x : o) fhe_ct_free(x);
            throw;
        }
        for (size_t i = 0; i < n; ++i) outs[i] = o[i];
    });
}

int fhe_conv2d_batch_into(fhe_ctx* c, const fhe_ct* const* cts, size_t n, const fhe_conv_layer* ly, int approach,
                          fhe_ct* const* outs) {
    return guard(c, [&] { batch_impl(c, cts, n, ly, approach, outs); });
}

// Host-resident batches: chunks of `chunk` ciphertexts flow through three
// streams (upload on h2d_st | conv on the context stream | download on
// d2h_st) with double-buffered device ciphertexts, so the PCIe/C2C copies of
// chunk j+1 and j-1 overlap the conv of chunk j. Nothing here synchronises
// the host: the device buffers are freed stream-ordered after their last use
// and the events are recycled at the next fhe_host_wait / fhe_synchronize.
static void host_pipe_free(fhe_ctx* c) {
    auto& h = c->hp;
    for (int b = 0; b < 2; ++b) {
        for (uint64_t* p : h.din[b]) cudaFree(p);
        for (uint64_t* p : h.dout[b]) cudaFree(p);
        h.din[b].clear();
        h.dout[b].clear();
    }
    h.level = -1;
    h.S = 0;
    h.chunks = 0;
}

static void batch_host_enqueue(fhe_ctx* c, const uint64_t* host_in, size_t n, double scale, const fhe_conv_layer* ly,
                               int approach, size_t chunk, uint64_t* host_out, bool short_ends) {
    if (!ly || (n && (!host_in || !host_out))) fail(FHE_E_INVALID, "null argument");
    if (n == 0) return;
    const int level = ly->level;
    if (level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
    const size_t N = c->N, inw = (size_t)2 * (level + 1) * N, outw = (size_t)2 * level * N;
    const size_t S = std::max<size_t>(1, std::min(chunk ? chunk : (size_t)4, n));
    const double sc = scale > 0 ? scale : c->scale;
    auto& h = c->hp;
    if (h.level != level || h.S < S) {  // (re)build the persistent chunk buffers
        ck(cudaStreamSynchronize(c->h2d_st), "sync");
        ck(cudaStreamSynchronize(c->main_st), "sync");
        ck(cudaStreamSynchronize(c->d2h_st), "sync");
        host_pipe_free(c);
        for (int b = 0; b < 2; ++b) {
            for (size_t s = 0; s < S; ++s) {
                uint64_t *pi = nullptr, *po = nullptr;
                ck(cudaMalloc(&pi, inw * 8), "cudaMalloc");
                ck(cudaMalloc(&po, outw * 8), "cudaMalloc");
                h.din[b].push_back(pi);
                h.dout[b].push_back(po);
            }
            for (cudaEvent_t* e : {&h.ev_h2d[b], &h.ev_comp[b], &h.ev_d2h[b]})
                if (!*e) ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
        }
        h.level = level;
        h.S = S;
    }
    // chunk sizes (short_ends: half-size first and last chunks shorten the
    // exposed upload of the first chunk and download of the last one)
    std::vector<size_t> sizes;
    {
        const size_t hs = short_ends ? std::max<size_t>(1, S / 2) : S;
        size_t rem = n;
        if (n > S) {
            sizes.push_back(hs);
            rem -= hs;
            while (rem > S + hs) {
                sizes.push_back(S);
                rem -= S;
            }
            if (rem > hs) {
                sizes.push_back(rem - hs);
                rem = hs;
            }
        }
        sizes.push_back(rem);
    }
    std::vector<fhe_ct> vin(S), vout(S);
    std::vector<fhe_ct*> pin(S), pout(S);
    size_t s0 = 0;
    for (size_t j = 0; j < sizes.size(); s0 += sizes[j], ++j) {
        const int b = (int)(h.chunks & 1);
        const size_t sn = sizes[j];
        if (h.chunks >= 2) ck(cudaStreamWaitEvent(c->h2d_st, h.ev_comp[b], 0), "cudaStreamWaitEvent");
        for (size_t s = 0; s < sn; ++s)
            ck(cudaMemcpyAsync(h.din[b][s], host_in + (s0 + s) * inw, inw * 8, cudaMemcpyHostToDevice, c->h2d_st),
               "H2D");
        ck(cudaEventRecord(h.ev_h2d[b], c->h2d_st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->main_st, h.ev_h2d[b], 0), "cudaStreamWaitEvent");
        if (h.chunks >= 2) ck(cudaStreamWaitEvent(c->main_st, h.ev_d2h[b], 0), "cudaStreamWaitEvent");
        for (size_t s = 0; s < sn; ++s) {
            vin[s] = fhe_ct{c, level, sc, 0, h.din[b][s]};
            vout[s] = fhe_ct{c, level - 1, sc, 1, h.dout[b][s]};
            pin[s] = &vin[s];
            pout[s] = &vout[s];
        }
        batch_impl(c, pin.data(), sn, ly, approach, pout.data());
        ck(cudaEventRecord(h.ev_comp[b], c->main_st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->d2h_st, h.ev_comp[b], 0), "cudaStreamWaitEvent");
        for (size_t s = 0; s < sn; ++s)
            ck(cudaMemcpyAsync(host_out + (s0 + s) * outw, h.dout[b][s], outw * 8, cudaMemcpyDeviceToHost, c->d2h_st),
               "D2H");
        ck(cudaEventRecord(h.ev_d2h[b], c->d2h_st), "cudaEventRecord");
        ++h.chunks;
    }
}

static void host_wait(fhe_ctx* c) {
    ck(cudaStreamSynchronize(c->h2d_st), "sync");
    ck(cudaStreamSynchronize(c->main_st), "sync");
    ck(cudaStreamSynchronize(c->d2h_st), "sync");
    for (cudaStream_t l : c->lanes) ck(cudaStreamSynchronize(l), "sync");
    for (cudaEvent_t e : c->pending_events) c->ev_pool.push_back(e);
    c->pending_events.clear();
}

int fhe_conv2d_batch_host(fhe_ctx* c, const uint64_t* host_in, size_t n, double scale, const fhe_conv_layer* ly,
                          int approach, size_t chunk, uint64_t* host_out) {
    return guard(c, [&] {
        try {
            batch_host_enqueue(c, host_in, n, scale, ly, approach, chunk, host_out, true);
        } catch (...) {
            host_wait(c);
            throw;
        }
        host_wait(c);
    });
}

int fhe_conv2d_batch_host_async(fhe_ctx* c, const uint64_t* host_in, size_t n, double scale,
                                const fhe_conv_layer* ly, int approach, size_t chunk, uint64_t* host_out) {
    return guard(c, [&] {
        try {
            batch_host_enqueue(c, host_in, n, scale, ly, approach, chunk, host_out, false);
        } catch (...) {
            host_wait(c);
            throw;
        }
    });
}

int fhe_host_wait(fhe_ctx* c) {
    return guard(c, [&] { host_wait(c); });
}


// ------------------------------------------------ rotate-and-add reduction
// slot_sum (reference dense.cpp:23-30) and the linear head
// (masked_feature_dot, dense.cpp:34-67) composed from this library's ops;
// each slot_sum step rotates the whole batch with one staged key-switch
// launch (every key row streamed once per 16 ciphertexts).
static void okc(fhe_ctx* c, int rc) {
    if (rc != FHE_OK) fail(rc, c->err);
}

int fhe_slot_sum_batch(fhe_ctx* c, const fhe_ct* const* cts, size_t n, uint64_t block, fhe_ct** outs) {
    return guard(c, [&] {
        if (block == 0 || (block & (block - 1)) || c->slots() % block)
            fail(FHE_E_INVALID, "block must be a power of two dividing the slot count");
        std::vector<fhe_ct*> acc(n), rot(n);
        for (size_t i = 0; i < n; ++i) {
            acc[i] = new_ct(c, cts[i]->level, cts[i]->scale, cts[i]->depth);
            ck(cudaMemcpyAsync(acc[i]->d, cts[i]->d, cts[i]->words() * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
            rot[i] = new_ct(c, cts[i]->level, cts[i]->scale, cts[i]->depth);
        }
        try {
            for (uint64_t step = 1; step < block; step *= 2) {
                const int64_t k = (int64_t)step;
                okc(c, fhe_rotate_hoisted_batch_into(c, acc.data(), n, &k, 1, rot.data()));
                c->ledger.hoist_groups -= n;  // sequential rotations, not hoisted groups
                c->ledger.hoisted_rotations -= n;
                c->ledger.rotations += n;
                for (size_t i = 0; i < n; ++i) {
                    ew_add(c->dc, acc[i]->d, acc[i]->d, rot[i]->d, 2 * (acc[i]->level + 1), acc[i]->level + 1, c->st);
                    c->ledger.adds++;
                }
            }
        } catch (...) {
            for (size_t i = 0; i < n; ++i) {
                fhe_ct_free(acc[i]);
                fhe_ct_free(rot[i]);
            }
            throw;
        }
        for (size_t i = 0; i < n; ++i) {
            fhe_ct_free(rot[i]);
            outs[i] = acc[i];
        }
    });
}

// masked_feature_dot (dense.cpp:34-67) over a slot -> feature map
// (feat[u * s + i] = feature held by slot i of shard u, -1 = none)
static void linear_impl(fhe_ctx* c, const fhe_ct* const* shards, size_t t, const int64_t* featmap, size_t nin,
                        int out_features, const double* w, const double* b, fhe_ct** out) {
    const size_t s = c->slots();
    if (t == 0 || !shards || !w || !b || !out) fail(FHE_E_INVALID, "null argument");
    if (out_features <= 0 || (size_t)out_features > s) fail(FHE_E_INVALID, "out_features exceeds the shard size");
    const int level = shards[0]->level;
    if (level < 2) fail(FHE_E_RUNTIME, "depth exhausted");
    auto feat = [&](size_t u, size_t i) -> long { return (long)featmap[u * s + i]; };
    // plaintext cache (fhe_ctx::linear_cache): the encodes below are host FFTs + uploads,
    // most of a small network's inference time when repeated per call
    auto mix = [](uint64_t h, uint64_t v) {
        h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
        return h * 0xff51afd7ed558ccdULL;
    };
    uint64_t hk = mix(mix(mix(mix(0x6c696e656172ULL, (uint64_t)level), t), nin), (uint64_t)out_features);
    {
        uint64_t sb;
        memcpy(&sb, &shards[0]->scale, 8);
        hk = mix(hk, sb);
        for (size_t i = 0; i < t * s; ++i) hk = mix(hk, (uint64_t)featmap[i]);
        const uint64_t* wp = reinterpret_cast<const uint64_t*>(w);
        for (size_t i = 0; i < (size_t)out_features * nin; ++i) hk = mix(hk, wp[i]);
        const uint64_t* bp = reinterpret_cast<const uint64_t*>(b);
        for (int i = 0; i < out_features; ++i) hk = mix(hk, bp[i]);
    }
    fhe_ctx::LinearEntry* hit = nullptr;
    for (auto& le : c->linear_cache)
        if (le.key == hk) hit = &le;
    std::vector<fhe_pt*> fresh;  // plaintexts encoded by this call (cached on success)
    size_t next_pt = 0;
    auto plain = [&](const double* z, int lv, double scale) -> fhe_pt* {
        if (hit) return hit->pts.at(next_pt++);
        fhe_pt* pt = nullptr;
        okc(c, fhe_encode(c, z, s, lv, scale, 0, &pt));
        fresh.push_back(pt);
        return pt;
    };
    std::vector<fhe_ct*> prods, sums;  // freed on any error (e.g. a missing slot-sum key)
    try {
        // products W_o . x_u for every output feature and shard, one level
        std::vector<int> prod_o;
        std::vector<double> wt(s);
        const double ql = (double)c->primes[level];
        for (int o = 0; o < out_features; ++o) {
            bool started = false;
            for (size_t u = 0; u < t; ++u) {
                bool any = false;
                for (size_t i = 0; i < s; ++i) {
                    const long f = feat(u, i);
                    wt[i] = f < 0 ? 0.0 : w[(size_t)o * nin + (size_t)f];
                    any = any || wt[i] != 0.0;
                }
                if (!any && started) continue;
                fhe_pt* pt = plain(wt.data(), level, ql);
                fhe_ct *pr = nullptr, *rs = nullptr;
                okc(c, fhe_mul_plain(c, shards[u], pt, &pr));
                okc(c, fhe_rescale(c, pr, &rs));
                fhe_ct_free(pr);
                prods.push_back(rs);
                prod_o.push_back(o);
                started = true;
            }
        }
        sums.assign(prods.size(), nullptr);
        okc(c, fhe_slot_sum_batch(c, prods.data(), prods.size(), s, sums.data()));
        for (fhe_ct*& x : prods) {
            fhe_ct_free(x);
            x = nullptr;
        }
        // per output: sum over shards, select slot o (second level), accumulate
        fhe_ct* acc = nullptr;
        std::vector<double> sel(s, 0.0);
        size_t k = 0;
        for (int o = 0; o < out_features; ++o) {
            fhe_ct* total = sums[k];
            sums[k++] = nullptr;
            while (k < sums.size() && prod_o[k] == o) {
                fhe_ct* nt = nullptr;
                okc(c, fhe_add(c, total, sums[k], &nt));
                fhe_ct_free(total);
                fhe_ct_free(sums[k]);
                sums[k] = nullptr;
                total = nt;
                ++k;
            }
            std::fill(sel.begin(), sel.end(), 0.0);
            sel[(size_t)o] = 1.0;
            fhe_pt* pt = plain(sel.data(), total->level, (double)c->primes[total->level]);
            fhe_ct *pr = nullptr, *rs = nullptr;
            okc(c, fhe_mul_plain(c, total, pt, &pr));
            okc(c, fhe_rescale(c, pr, &rs));
            fhe_ct_free(pr);
            fhe_ct_free(total);
            if (!acc) {
                acc = rs;
            } else {
                fhe_ct* na = nullptr;
                okc(c, fhe_add(c, acc, rs, &na));
                fhe_ct_free(acc);
                fhe_ct_free(rs);
                acc = na;
            }
        }
        std::vector<double> bias(s, 0.0);
        for (int o = 0; o < out_features; ++o) bias[(size_t)o] = b[o];
        fhe_pt* bp = plain(bias.data(), acc->level, acc->scale);
        fhe_ct* res = nullptr;
        okc(c, fhe_add_plain(c, acc, bp, &res));
        fhe_ct_free(acc);
        *out = res;
    } catch (...) {
        for (fhe_ct* x : prods)
            if (x) fhe_ct_free(x);
        for (fhe_ct* x : sums)
            if (x) fhe_ct_free(x);
        for (fhe_pt* x : fresh) fhe_pt_free(x);
        throw;
    }
    if (hit) {
        hit->last_use = ++c->linear_clock;
    } else {
        if (c->linear_cache.size() >= 4) {  // evict the least recently used head
            size_t lru = 0;
            for (size_t i = 1; i < c->linear_cache.size(); ++i)
                if (c->linear_cache[i].last_use < c->linear_cache[lru].last_use) lru = i;
            for (fhe_pt* x : c->linear_cache[lru].pts) fhe_pt_free(x);
            c->linear_cache.erase(c->linear_cache.begin() + (long)lru);
        }
        fhe_ctx::LinearEntry le;
        le.key = hk;
        le.last_use = ++c->linear_clock;
        le.pts = std::move(fresh);
        c->linear_cache.push_back(std::move(le));
    }
}

int fhe_linear(fhe_ctx* c, const fhe_ct* const* shards, size_t t, int ch, int m, int out_features, const double* w,
               const double* b, fhe_ct** out) {
    return guard(c, [&] {
        const size_t s = c->slots(), block = (size_t)m * m, nin = (size_t)ch * block;
        // slot -> feature map (reference slot_feature_map pack.cpp:109-129, identity tau, rep 1):
        // image mode: slot i of shard u holds feature u s + i below c m^2 (the primary
        // replica when the image is duplicated); channel mode: channel-major rows.
        const bool channel_mode = block > s;
        const size_t expect_t = channel_mode ? nin / s : std::max<size_t>(1, nin / s);
        if (t != expect_t) fail(FHE_E_INVALID, "shard count does not match the packed feature count");
        std::vector<int64_t> fm(t * s);
        for (size_t f = 0; f < t * s; ++f) fm[f] = f < nin ? (int64_t)f : -1;
        linear_impl(c, shards, t, fm.data(), nin, out_features, w, b, out);
    });
}

int fhe_linear_features(fhe_ctx* c, const fhe_ct* const* shards, size_t t, const int64_t* features,
                        size_t in_features, int out_features, const double* w, const double* b, fhe_ct** out) {
    return guard(c, [&] {
        if (!features) fail(FHE_E_INVALID, "null argument");
        const size_t s = c->slots();
        for (size_t f = 0; f < t * s; ++f)
            if (features[f] >= (int64_t)in_features || features[f] < -1)
                fail(FHE_E_INVALID, "in_features does not match the packed feature count");
        linear_impl(c, shards, t, features, in_features, out_features, w, b, out);
    });
}


// ------------------------------------------------------------- pooling
// 2x2 average pooling (reference pool(), pool.cpp:291-297)
// and stride-2 subsampling (subsample_stride2, pool.cpp:299-306) of image-mode
// and channel-shard feature maps. The reference's masked stages become
// plaintext-weighted sums of hoisted rotations (rot_k(x * mask) = rot_k(mask) *
// rot_k(x)), each one fused baby-step pass over all shards:
//   window     W = sum_{(kk,ll) in 2x2} wmask(kk, ll) * rot_{kk m + ll}(x)       (pool.cpp:22-30)
//              channel shards add the spill masks of the next shard (:34-72)
//   horizontal H = sum_{i < m/2} rot_i(hmask_i) * rot_i(W)                       (pool.cpp:76-86)
//   vertical   V = sum_{j < R/2} rot_{3jm/2}(vmask_j) * rot_{3jm/2}(H)            (pool.cpp:90-129)
//              R = m (image) or rows per shard (channel; rows = 1: even shards
//              masked, odd shards dropped)
// then the reference's consolidation (pool.cpp:167-273) and duplication
// (:276-289) rotations. Stride-2 skips the window stage. 3 (pool) / 2 levels.
static void downsample_impl(fhe_ctx* c, const fhe_ct* const* in, size_t t, int ch, int m, const int64_t* tau_in,
                            int rep_in, int d_in, int window, double oscale, fhe_ct** outs, size_t* n_out,
                            int64_t* tau_out, int* rep_out, int* d_out, int* mode_out) {
    // every intermediate ciphertext is tracked so that an exception (e.g. a missing
    // Galois key) frees them; outputs are released from the tracker at the end
    struct Tracker {
        std::set<fhe_ct*> s;
        fhe_ct* add(fhe_ct* x) { return s.insert(x), x; }
        void drop(fhe_ct* x) {
            if (x && s.erase(x)) fhe_ct_free(x);
        }
        ~Tracker() {
            for (fhe_ct* x : s) fhe_ct_free(x);
        }
    } tr;
    const size_t s = c->slots();
    if (t == 0 || !in) fail(FHE_E_INVALID, "packed image has no shards");
    if (m < 2) fail(FHE_E_INVALID, window ? "cannot pool a 1x1 channel" : "cannot subsample a 1x1 channel");
    if ((m & (m - 1)) || ch < 1 || (ch & (ch - 1))) fail(FHE_E_INVALID, "dimensions must be powers of two");
    const size_t block = (size_t)m * m;
    const bool image = block <= s;
    if (rep_in < 1 || d_in < 1) fail(FHE_E_INVALID, "metadata mismatch");
    if (image) {
        if (t >= 2 && d_in != 1) fail(FHE_E_INVALID, "metadata mismatch: duplicated multi-shard image");
        if ((size_t)ch * block * (size_t)d_in != t * s) fail(FHE_E_INVALID, "metadata mismatch: shard count");
    } else if (d_in != 1 || t != (size_t)ch * (block / s)) {
        fail(FHE_E_INVALID, "metadata mismatch: shard count");
    }
    std::vector<int64_t> tau0((size_t)ch);
    for (int j = 0; j < ch; ++j) tau0[(size_t)j] = tau_in ? tau_in[j] : j;
    const int level = in[0]->level;
    for (size_t u = 0; u < t; ++u)
        if (in[u]->level != level) fail(FHE_E_INVALID, "shards are at different levels");
    if (level < (window ? 3 : 2)) fail(FHE_E_RUNTIME, "depth exhausted");
    const long mL = m;
    const size_t pc = image ? 1 : block / s, rows = image ? 0 : s / (size_t)m;
    auto rotl = [&](const std::vector<double>& v, int64_t k) {
        std::vector<double> r(s);
        const size_t a = (size_t)(((k % (int64_t)s) + (int64_t)s) % (int64_t)s);
        for (size_t i = 0; i < s; ++i) r[i] = v[(i + a) % s];
        return r;
    };
    const std::string geo = std::to_string(m) + "/" + std::to_string(s);
    auto fresh = [&](const std::vector<const fhe_ct*>& src) {
        std::vector<fhe_ct*> o(src.size());
        for (size_t u = 0; u < src.size(); ++u) o[u] = tr.add(new_ct(c, src[u]->level - 1, src[u]->scale, src[u]->depth + 1));
        return o;
    };
    auto count_rot = [&](const std::vector<int64_t>& am, size_t times) {
        size_t k = 0;
        for (int64_t x : am) k += c->reduce_amount(x) != 0;
        c->ledger.rotations += (uint64_t)(k * times);
    };
    auto stage = [&](const std::vector<const fhe_ct*>& src, const std::string& name, const std::vector<int64_t>& am,
                     const std::vector<std::vector<double>>& pts) {
        std::vector<fhe_ct*> o = fresh(src);
        if (!src.empty()) lintrans_batch(c, src.data(), (int)src.size(), name + "/" + geo, am, pts, o.data());
        count_rot(am, src.size());
        return o;
    };
    auto free_all = [&](std::vector<fhe_ct*>& v) {
        for (fhe_ct* x : v)
            if (x) tr.drop(x);
        v.clear();
    };
    // ---- window stage
    std::vector<fhe_ct*> W;
    if (window && image) {
        std::vector<int64_t> aw;
        std::vector<std::vector<double>> pw;
        for (auto kl : {std::pair<long, long>{0, 0}, {0, 1}, {1, 0}, {1, 1}}) {
            std::vector<double> v(s, 0.0);
            for (size_t b = 0; b * block < s; ++b)
                for (long i = 0; i + kl.first < mL; ++i)
                    for (long j = 0; j + kl.second < mL; ++j) v[b * block + (size_t)(i * mL + j)] = 0.25;
            aw.push_back(kl.first * mL + kl.second);
            pw.push_back(std::move(v));
        }
        W = stage(std::vector<const fhe_ct*>(in, in + t), "pool-window", aw, pw);
    } else if (window) {  // channel shards: in-shard masks of shard v + spill masks of shard v + 1
        std::vector<std::vector<double>> pv;
        std::vector<LtTerm> full, last;
        for (auto kl : {std::pair<long, long>{0, 0}, {0, 1}, {1, 0}, {1, 1}}) {
            const long kk = kl.first, ll = kl.second, amount = kk * mL + ll;
            std::vector<double> inm(s, 0.0), spm(s, 0.0);
            bool any_in = false, any_spill = false;
            for (long rr = 0; rr < (long)rows; ++rr)
                for (long j = 0; j + ll < mL; ++j) {
                    if (rr + kk < (long)rows) {
                        inm[(size_t)(rr * mL + j)] = 0.25;
                        any_in = true;
                    } else {
                        spm[(size_t)(rr * mL + j)] = 0.25;
                        any_spill = true;
                    }
                }
            if (any_in) {
                pv.push_back(std::move(inm));
                full.push_back({amount, 0, (int)pv.size() - 1});
                last.push_back({amount, 0, (int)pv.size() - 1});
            }
            if (any_spill) {
                pv.push_back(std::move(spm));
                full.push_back({amount, 1, (int)pv.size() - 1});
            }
        }
        const uint64_t* pts = lt_plaintexts(c, "pool-window-ch/" + geo, level, pv);
        const int ne = c->ne_at(level);
        const size_t extw = (size_t)ne * c->N;
        uint64_t *buf, *dig;
        lt_modup(c, in, (int)t, &buf, &dig);
        uint64_t* Y = c->alloc(t * 2 * extw);
        ck(cudaMemsetAsync(Y, 0, t * 2 * extw * 8, c->st), "memset");
        for (int f = 0; f < ch; ++f)
            lt_accumulate(c, level, dig, buf, (int)pc - 1, (size_t)f * pc, 1, full, pts, Y + (size_t)f * pc * 2 * extw,
                          2 * extw);
        lt_accumulate(c, level, dig, buf, ch, pc - 1, pc, last, pts, Y + (pc - 1) * 2 * extw, pc * 2 * extw);
        c->release(dig);
        std::vector<const fhe_ct*> src(in, in + t);
        W = fresh(src);
        lt_finish(c, Y, (int)t, level, in, W.data());
        c->release(Y);
        c->release(buf);
        size_t nrot = 0;
        for (const LtTerm& x : full) nrot += (size_t)(c->reduce_amount(x.amount) != 0) * (pc - 1);
        for (const LtTerm& x : last) nrot += (size_t)(c->reduce_amount(x.amount) != 0);
        c->ledger.rotations += (uint64_t)(nrot * (size_t)ch);
    }
    // ---- compact: horizontal + vertical (pool.cpp:131-150); channel shards with one
    // row drop odd shards (no output)
    std::vector<const fhe_ct*> X(t);
    for (size_t u = 0; u < t; ++u) X[u] = window ? W[u] : in[u];
    std::vector<size_t> live;
    for (size_t u = 0; u < t; ++u)
        if (image || rows != 1 || ((u % pc) * rows) % 2 == 0) live.push_back(u);
    std::vector<const fhe_ct*> xl;
    for (size_t u : live) xl.push_back(X[u]);
    std::vector<int64_t> ah, av;
    std::vector<std::vector<double>> ph, pvv;
    for (long i2 = 0; i2 < mL / 2; ++i2) {
        std::vector<double> mk(s, 0.0);
        for (size_t row = 0; row < s; row += (size_t)m) mk[row + 2 * (size_t)i2] = 1.0;
        ah.push_back(i2);
        ph.push_back(rotl(mk, i2));
    }
    std::vector<fhe_ct*> H = stage(xl, "pool-horizontal", ah, ph);
    free_all(W);
    const size_t R = image ? (size_t)m : rows;
    const size_t vblock = image ? block : s;
    if (R == 1) {
        std::vector<double> mv(s, 0.0);
        for (long col = 0; col < mL / 2; ++col) mv[(size_t)col] = oscale;
        av.push_back(0);
        pvv.push_back(std::move(mv));
    }
    for (size_t j = 0; j < R / 2; ++j) {
        std::vector<double> mv(s, 0.0);
        for (size_t b = 0; b * vblock < s; ++b)
            for (long col = 0; col < mL / 2; ++col) mv[b * vblock + 2 * j * (size_t)m + (size_t)col] = oscale;
        av.push_back((int64_t)(3 * j * (size_t)m / 2));
        pvv.push_back(rotl(mv, av.back()));
    }
    char vkey[64];
    snprintf(vkey, sizeof vkey, "pool-vertical-%d-%a", image ? 0 : 1, oscale);
    std::vector<fhe_ct*> Vl = stage(std::vector<const fhe_ct*>(H.begin(), H.end()), vkey, av, pvv);
    free_all(H);
    std::vector<fhe_ct*> V(t, nullptr);
    for (size_t k = 0; k < live.size(); ++k) V[live[k]] = Vl[k];
    // ---- consolidation (pool.cpp:167-273)
    auto rot1 = [&](const fhe_ct* a, int64_t k) {
        fhe_ct* o = tr.add(new_ct(c, a->level, a->scale, a->depth));
        okc(c, fhe_rotate_hoisted_batch_into(c, &a, 1, &k, 1, &o));
        return o;
    };
    auto add_into = [&](fhe_ct* acc, const fhe_ct* b) {
        ew_add(c->dc, acc->d, acc->d, b->d, 2 * (acc->level + 1), acc->level + 1, c->st);
        c->ledger.adds++;
    };
    const size_t mn = (size_t)m / 2, bn = mn * mn;
    std::vector<int64_t> tau((size_t)ch);
    std::vector<fhe_ct*> res;
    int rep = 1, d = 1, mode = 0;
    size_t dup = 1, dup_stride = 0;
    if (image) {
        const size_t z = (size_t)ch * (size_t)d_in / t;
        if (t == 1) {
            res.push_back(V[0]);
            tau = tau0;
            rep = 4 * rep_in;
            d = 4 * d_in;
            dup = 4;
            dup_stride = bn;
        } else if (t == 2) {
            fhe_ct* r = rot1(V[1], -2 * (int64_t)bn);
            add_into(V[0], r);
            tr.drop(r);
            tr.drop(V[1]);
            res.push_back(V[0]);
            for (size_t j = 0; j < (size_t)ch; ++j) tau[j] = tau0[(j % 2) * z + j / 2];
            rep = 2;
            d = 2;
            dup = 2;
            dup_stride = bn;
        } else {
            if (t % 4) fail(FHE_E_INVALID, "shard count must be 1, 2 or a multiple of 4");
            const size_t blocks_out = 4 * z;
            for (size_t w4 = 0; w4 < t / 4; ++w4) {
                for (size_t q = 1; q < 4; ++q) {
                    fhe_ct* r = rot1(V[4 * w4 + q], -(int64_t)(q * bn));
                    add_into(V[4 * w4], r);
                    tr.drop(r);
                    tr.drop(V[4 * w4 + q]);
                }
                res.push_back(V[4 * w4]);
                for (size_t g = 0; g < blocks_out; ++g) tau[w4 * blocks_out + g] = tau0[(4 * w4 + g % 4) * z + g / 4];
            }
        }
    } else {  // channel shards consolidate in channel-major order, tau stays the identity
        for (size_t w4 = 0; w4 < (t + 3) / 4; ++w4) {
            fhe_ct* acc = nullptr;
            for (size_t q = 0; q < 4 && 4 * w4 + q < t; ++q) {
                fhe_ct* src = V[4 * w4 + q];
                if (!src) continue;
                if (q == 0) {
                    acc = src;
                    continue;
                }
                fhe_ct* r = rot1(src, -(int64_t)(q * (s / 4)));
                tr.drop(src);
                if (acc) {
                    add_into(acc, r);
                    tr.drop(r);
                } else {
                    acc = r;
                }
            }
            res.push_back(acc);
        }
        for (size_t j = 0; j < (size_t)ch; ++j) tau[j] = (int64_t)j;
        if (bn > s) {
            mode = 1;
        } else {
            const size_t valid = (size_t)ch * bn;
            d = valid < s ? (int)(s / valid) : 1;
            if (d > 1) {
                dup = (size_t)d;
                dup_stride = valid;
            }
        }
    }
    if (dup > 1) {  // channel duplication: base + sum_e rot_{-e stride}(base), hoisted (pool.cpp:276-289)
        if (res.size() != 1) fail(FHE_E_INVALID, "duplication applies to a single shard");
        fhe_ct* base = res[0];
        std::vector<int64_t> ks;
        for (size_t e = 1; e < dup; ++e) ks.push_back(-(int64_t)(e * dup_stride));
        std::vector<fhe_ct*> rs(ks.size());
        for (size_t e = 0; e < ks.size(); ++e) rs[e] = tr.add(new_ct(c, base->level, base->scale, base->depth));
        const fhe_ct* bc = base;
        okc(c, fhe_rotate_hoisted_batch_into(c, &bc, 1, ks.data(), ks.size(), rs.data()));
        for (fhe_ct* r : rs) {
            add_into(base, r);
            tr.drop(r);
        }
    }
    for (size_t u = 0; u < res.size(); ++u) {
        tr.s.erase(res[u]);
        outs[u] = res[u];
    }
    if (n_out) *n_out = res.size();
    if (tau_out)
        for (size_t j = 0; j < (size_t)ch; ++j) tau_out[j] = tau[j];
    if (rep_out) *rep_out = rep;
    if (d_out) *d_out = d;
    if (mode_out) *mode_out = mode;
}

// pack()'s duplication of a single image-mode shard (pack.cpp:19-21)
static int natural_dup(const fhe_ctx* c, int ch, int m) {
    const size_t s = c->slots(), block = (size_t)m * m;
    return (block <= s && ch > 0 && (size_t)ch * block < s) ? (int)(s / ((size_t)ch * block)) : 1;
}

int fhe_downsample(fhe_ctx* c, const fhe_ct* const* in, size_t t, int ch, int m, const int64_t* tau_in, int rep_in,
                   int d_in, int window, double output_scale, fhe_ct** outs, size_t* n_out, int64_t* tau_out,
                   int* rep_out, int* d_out, int* mode_out) {
    return guard(c, [&] {
        downsample_impl(c, in, t, ch, m, tau_in, rep_in, d_in, window, output_scale, outs, n_out, tau_out, rep_out,
                        d_out, mode_out);
    });
}

int fhe_pool(fhe_ctx* c, const fhe_ct* const* in, size_t t, int ch, int m, fhe_ct** outs, size_t* n_out,
             int64_t* tau_out, int* rep_out, int* d_out) {
    return guard(c, [&] {
        downsample_impl(c, in, t, ch, m, nullptr, 1, natural_dup(c, ch, m), 1, 1.0, outs, n_out, tau_out, rep_out,
                        d_out, nullptr);
    });
}

int fhe_subsample_stride2(fhe_ctx* c, const fhe_ct* const* in, size_t t, int ch, int m, fhe_ct** outs,
                          size_t* n_out, int64_t* tau_out, int* rep_out, int* d_out) {
    return guard(c, [&] {
        downsample_impl(c, in, t, ch, m, nullptr, 1, natural_dup(c, ch, m), 0, 1.0, outs, n_out, tau_out, rep_out,
                        d_out, nullptr);
    });
}

// ------------------------------------------- ct x ct and Chebyshev series
// mul_ct with relinearisation (hybrid key switching of d2 with
// the s^2 key, the same ModUp / inner-product / ModDown kernels) and the
// reference's power-of-two-split Chebyshev evaluation (act.cpp:30-82, 151-162).
// round(k * scale) as residues of the level's primes (the exact encoding of a constant slot vector)
static RowConsts const_residues(fhe_ctx* c, double k, double scale, int level) {
    const double v = std::nearbyint(k * scale);
    if (!(std::fabs(v) < 9.2e18)) fail(FHE_E_INVALID, "constant too large for its scale");
    const int64_t iv = (int64_t)v;
    const uint64_t mag = iv < 0 ? (uint64_t)0 - (uint64_t)iv : (uint64_t)iv;
    RowConsts r{};
    for (int i = 0; i <= level; ++i) {
        const uint64_t q = c->primes[i], m = mag % q;
        r.v[i] = iv < 0 && m ? q - m : m;
    }
    return r;
}

// ct + k (reference Engine::add_scalar, emu.cpp:113-119): no level consumed
static fhe_ct* add_scalar_ct(fhe_ctx* c, const fhe_ct* x, double k) {
    fhe_ct* o = new_ct(c, x->level, x->scale, x->depth);
    ew_const(c->dc, o->d, x->d, const_residues(c, k, x->scale, x->level), x->level + 1, 0, c->st);
    c->ledger.adds++;
    return o;
}

// ct * k rescaled onto (level, scale): the constant is scaled by scale * q_{level+1} / x.scale
// (reference mul_plain with a constant vector, emu.cpp:56-67); x at level + 1
static fhe_ct* mul_scalar_ct(fhe_ctx* c, const fhe_ct* x, double k, int level, double scale) {
    const int nr = level + 2;
    if (x->level != level + 1) fail(FHE_E_INVALID, "level mismatch");
    uint64_t* pr = c->alloc((size_t)2 * nr * c->N);
    ew_const(c->dc, pr, x->d, const_residues(c, k, scale * (double)c->primes[level + 1] / x->scale, level + 1), nr,
             1, c->st);
    fhe_ct* o = new_ct(c, level, scale, x->depth + 1);
    rescale_into(c, pr, level + 1, o->d);
    c->release(pr);
    c->ledger.ct_pt_mults++;
    c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, o->depth);
    return o;
}

int fhe_add_scalar(fhe_ctx* c, const fhe_ct* x, double k, fhe_ct** out) {
    return guard(c, [&] { *out = add_scalar_ct(c, x, k); });
}

int fhe_mul_scalar(fhe_ctx* c, const fhe_ct* x, double k, fhe_ct** out) {
    return guard(c, [&] {
        if (x->level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
        *out = mul_scalar_ct(c, x, k, x->level - 1, x->scale);
    });
}

int fhe_gen_relin_key(fhe_ctx* c) {
    return guard(c, [&] {
        require_key(c);
        gen_key(c, 0);
        ck(cudaStreamSynchronize(c->st), "sync");
    });
}

static fhe_ct* drop_to(fhe_ctx* c, const fhe_ct* a, int level) {
    // modulus drop: keep rows 0..level of both polynomials (scale unchanged)
    fhe_ct* o = new_ct(c, level, a->scale, a->depth);
    const size_t N = c->N, w = (size_t)(level + 1) * N;
    ck(cudaMemcpyAsync(o->c0(), a->c0(), w * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    ck(cudaMemcpyAsync(o->c1(), a->c1(), w * 8, cudaMemcpyDeviceToDevice, c->st), "memcpy");
    return o;
}

// relinearised product of two ciphertexts at the same level, then one rescale
static fhe_ct* mul_relin_rescale(fhe_ctx* c, const fhe_ct* a, const fhe_ct* b) {
    const int level = a->level, nr = level + 1, ne = c->ne_at(level), dn = c->dn_at(level);
    if (level < 1) fail(FHE_E_RUNTIME, "depth exhausted");
    if (!c->keys.count(0)) fail(FHE_E_NOKEY, "missing relinearisation key (fhe_gen_relin_key)");
    const size_t N = c->N, pw = (size_t)nr * N, extw = (size_t)ne * N;
    uint64_t* d = c->alloc(3 * pw);
    tensor(c->dc, d, a->d, b->d, level, c->st);
    uint64_t* dig = c->alloc((size_t)dn * extw);
    modup(c, d + 2 * pw, level, dig);
    uint64_t* acc = c->alloc(2 * extw);
    c->timed("ks_inner", c->rows(3.0 * dn * ne + 2.0 * ne), [&] {
        ks_inner_product(c->dc, dig, c->keys.at(0), acc, acc + extw, 1, level, dn, c->st);
    });
    c->ledger.key_switches++;
    uint64_t* md = c->alloc(2 * pw);
    moddown(c, acc, level, 2, md, nullptr, 1);
    ew_add(c->dc, md, md, d, 2 * nr, nr, c->st);  // (d0, d1) + ModDown(IP(d2))
    fhe_ct* o = new_ct(c, level - 1, a->scale * b->scale / (double)c->primes[level], std::max(a->depth, b->depth) + 1);
    rescale_into(c, md, level, o->d);
    c->ledger.ct_ct_mults++;
    c->ledger.max_depth_consumed = std::max<uint64_t>(c->ledger.max_depth_consumed, o->depth);
    c->release(md);
    c->release(acc);
    c->release(dig);
    c->release(d);
    return o;
}

int fhe_mul(fhe_ctx* c, const fhe_ct* a, const fhe_ct* b, fhe_ct** out) {
    return guard(c, [&] {
        const int level = std::min(a->level, b->level);
        fhe_ct* ad = a->level == level ? nullptr : drop_to(c, a, level);
        fhe_ct* bd = b->level == level ? nullptr : drop_to(c, b, level);
        try {
            *out = mul_relin_rescale(c, ad ? ad : a, bd ? bd : b);
        } catch (...) {
            fhe_ct_free(ad);
            fhe_ct_free(bd);
            throw;
        }
        fhe_ct_free(ad);
        fhe_ct_free(bd);
    });
}

namespace {
// Chebyshev-series evaluation with exact scale management. The reference's
// emulator (act.cpp:49-82) adds values freely; in CKKS an addition needs equal
// levels and scales, and ct x ct products land at scale s_a s_b / q_l. So every
// sub-series is evaluated towards a (level, scale) target: leaves T_j * c are
// constant products whose integer constant round(c * s') is picked so the
// rescale lands exactly on the target, and a product q * T_p asks q for the scale
// that makes q * T_p / q_{l+1} hit the target. Same split, same basis, same depth.
// Constants never go through the slot encoder: a constant slot vector is the
// constant polynomial, whose NTT rows are the constant itself.
struct ChebEval {
    fhe_ctx* c;
    std::vector<fhe_ct*> owned;
    std::vector<fhe_ct*> basis;  // T_1, T_2, T_4, ...
    ~ChebEval() {
        for (fhe_ct* x : owned) fhe_ct_free(x);
    }
    fhe_ct* keep(fhe_ct* x) {
        owned.push_back(x);
        return x;
    }
    fhe_ct* at_level(fhe_ct* x, int level) {
        if (x->level < level) fail(FHE_E_RUNTIME, "insufficient level for activation: bootstrap required");
        return x->level == level ? x : keep(drop_to(c, x, level));
    }
    fhe_ct* add(fhe_ct* a, fhe_ct* b) {
        fhe_ct* o = nullptr;
        okc(c, fhe_add(c, a, b, &o));
        return keep(o);
    }
    fhe_ct* add_scalar(fhe_ct* x, double k) { return keep(add_scalar_ct(c, x, k)); }
    fhe_ct* mul_scalar(fhe_ct* x, double k, int level, double scale) {
        return keep(mul_scalar_ct(c, at_level(x, level + 1), k, level, scale));
    }
    fhe_ct* of_degree(size_t p2) const {
        size_t j = 0;
        while ((size_t{1} << j) < p2) ++j;
        return basis[j];
    }
    static size_t floor_pow2(size_t d) {
        size_t p = 1;
        while (p * 2 <= d) p *= 2;
        return p;
    }
    // sum_k co[k] T_k at (level, scale); degree >= 1 (act.cpp:49-82)
    fhe_ct* series(std::vector<double> co, int level, double scale) {
        const size_t d = co.size() - 1;
        if (d <= 2) {
            fhe_ct* acc = mul_scalar(of_degree(1), co[1], level, scale);
            if (d == 2) acc = add(acc, mul_scalar(of_degree(2), co[2], level, scale));
            return add_scalar(acc, co[0]);
        }
        const size_t p = floor_pow2(d);
        if (p == d) {
            fhe_ct* top = mul_scalar(of_degree(p), co[d], level, scale);
            co.pop_back();
            return add(top, series(std::move(co), level, scale));
        }
        std::vector<double> q(d - p + 1, 0.0), r(co.begin(), co.begin() + (long)p + 1);
        for (size_t a = 1; a <= d - p; ++a) {
            q[a] = 2.0 * co[p + a];
            r[p - a] -= co[p + a];
        }
        fhe_ct* tp = at_level(of_degree(p), level + 1);
        fhe_ct* qv = series(std::move(q), level + 1, scale * (double)c->primes[level + 1] / tp->scale);
        fhe_ct* prod = keep(mul_relin_rescale(c, qv, tp));
        prod->scale = scale;
        return add(prod, series(std::move(r), level, scale));
    }
};
}  // namespace

int fhe_eval_chebyshev(fhe_ctx* c, const fhe_ct* x, const double* coeffs, size_t n, double bound, int prescaled,
                       fhe_ct** out) {
    return guard(c, [&] {
        if (n == 0) fail(FHE_E_INVALID, "empty coefficient list");
        const size_t d = n - 1;
        int bits = 0;
        while ((size_t{1} << bits) <= d) ++bits;  // chebyshev_required_level (act.cpp:84-88)
        const int needed = bits + (prescaled ? 0 : 1);
        if (x->level < needed) fail(FHE_E_RUNTIME, "insufficient level for activation: bootstrap required");
        const int out_level = x->level - needed;
        ChebEval ev{c, {}, {}};
        fhe_ct* t = const_cast<fhe_ct*>(x);
        if (!prescaled) t = ev.mul_scalar(t, 1.0 / bound, x->level - 1, x->scale);  // act.cpp:156, also at d = 0
        if (d == 0) {  // a constant (the reference's fresh encode, act.cpp:158): trivial c1 = 0 ciphertext
            fhe_ct* o = new_ct(c, x->level, x->scale, 0);
            ck(cudaMemsetAsync(o->d, 0, (size_t)2 * (x->level + 1) * c->N * 8, c->st), "memset");
            ew_const(c->dc, o->d, o->d, const_residues(c, coeffs[0], x->scale, x->level), x->level + 1, 0, c->st);
            *out = o;
            return;
        }
        ev.basis.push_back(t);  // PowerBasis (act.cpp:28-37): T_2n = 2 T_n^2 - 1
        for (size_t p = 2; p <= ChebEval::floor_pow2(d); p *= 2) {
            fhe_ct* half = ev.basis.back();
            fhe_ct* sq = ev.keep(mul_relin_rescale(c, half, half));
            ev.basis.push_back(ev.add_scalar(ev.add(sq, sq), -1.0));
        }
        fhe_ct* res = ev.series(std::vector<double>(coeffs, coeffs + n), out_level, x->scale);
        ev.owned.erase(std::find(ev.owned.begin(), ev.owned.end(), res));  // hand the result out
        *out = res;
    });
}

}  // extern "C"
