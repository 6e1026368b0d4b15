// TEST INFRASTRUCTURE ONLY — never linked into the product (libfheconv).
//
// C-ABI shim over the UNMODIFIED reference library (shardnn, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py's reference arm drive the reference's own public
// API through ctypes:
//   * conv_plan / convolve  (reference conv.cpp:266-271, :364-371)
//   * decompose_positive / decompose_signed / min_decomposition_length
//     (reference rot.cpp:21-46, :84-94)
//   * plan_rotations + execute_schedule (reference rot.cpp:96-156)
//   * oracle_conv (reference oracle.cpp:7-31)
// Inputs are generated with the reference's own test helpers
// (tests/helpers.hpp:13-27: mt19937_64 + uniform_real_distribution), so the
// golden vectors are exactly what the reference's tests would see.
#include "shardnn/act.hpp"
#include "shardnn/io.hpp"
#include "shardnn/net.hpp"
#include "shardnn/conv.hpp"
#include "shardnn/dense.hpp"
#include "shardnn/pool.hpp"
#include "shardnn/oracle.hpp"
#include "shardnn/pack.hpp"
#include "shardnn/rot.hpp"
#include "helpers.hpp"
#include "tiny_net.hpp"

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <string>
#include <thread>
#include <vector>

using namespace shardnn;
using namespace shardnn::testing;

namespace {

// weight_kind: 0 = U[-1,1] (random_filter), 1 = U[-0.5,0.5], 2 = N(0,0.1^2) clipped to [-1,1]
FilterTensor make_filter(std::mt19937_64& rng, int c_in, int c_out, int kappa, int weight_kind) {
    if (weight_kind == 0) return random_filter(rng, c_in, c_out, kappa);
    FilterTensor k(c_in, c_out, kappa);
    if (weight_kind == 1) {
        std::uniform_real_distribution<double> dist(-0.5, 0.5);
        for (double& v : k.weights) v = dist(rng);
    } else {
        std::normal_distribution<double> dist(0.0, 0.1);
        for (double& v : k.weights) v = std::clamp(dist(rng), -1.0, 1.0);
    }
    return k;
}

void fill_ledger(const CostLedger& l, uint64_t* out) {
    if (!out) return;
    out[0] = l.rotations.load();
    out[1] = l.hoisted_rotations.load();
    out[2] = l.hoist_groups.load();
    out[3] = l.ct_pt_mults.load();
    out[4] = l.ct_ct_mults.load();
    out[5] = l.adds.load();
    out[6] = l.bootstraps.load();
    out[7] = static_cast<uint64_t>(l.max_depth_consumed.load());
    out[8] = l.rotation_amounts().size();
}

PackedImage run_plan(Engine& eng, const PackedImage& p, const FilterTensor& k, int plan) {
    if (plan == 1) return conv_plan(eng, p, k, ConvPlan::ChannelFirst);
    if (plan == 2) return conv_plan(eng, p, k, ConvPlan::ShiftFirst);
    return convolve(eng, p, k);
}

}  // namespace

extern "C" {

/// Generates the reference's random inputs and fills img (c*m*m) and filt
/// (c_in*c_out*kappa^2, reference storage order tensor.hpp:53-58).
int ref_make_inputs(int c, int m, int kappa, int c_out, uint64_t seed_img, uint64_t seed_filt,
                    int weight_kind, double* img, double* filt) {
    try {
        std::mt19937_64 ri(seed_img);
        ImageTensor t = random_tensor(ri, c, m);
        std::mt19937_64 rf(seed_filt);
        FilterTensor k = make_filter(rf, c, c_out, kappa, weight_kind);
        std::memcpy(img, t.data.data(), t.data.size() * sizeof(double));
        std::memcpy(filt, k.weights.data(), k.weights.size() * sizeof(double));
        return 0;
    } catch (...) {
        return -1;
    }
}

/// Runs pack + conv_plan(plan) on the emulator; writes the raw output shard
/// slots (s = c*m*m for the single-shard configs), the unpacked image and
/// the ledger [rot, hoisted, groups, ct_pt, ct_ct, adds, boots, depth, n_amounts].
int ref_conv(int c, int m, int kappa, int c_out, const double* img, const double* filt,
             int plan, uint64_t shard_size, double* out_slots, double* out_image,
             uint64_t* ledger, int* out_level_drop) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        FilterTensor k(c, c_out, kappa);
        std::memcpy(k.weights.data(), filt, k.weights.size() * sizeof(double));
        Engine eng;
        PackedImage p = pack(eng, t, shard_size);
        eng.ledger().reset();
        PackedImage out = run_plan(eng, p, k, plan);
        if (out_slots) {
            size_t off = 0;
            for (const auto& sh : out.shards) {
                std::memcpy(out_slots + off, sh.slots.data(), sh.slots.size() * sizeof(double));
                off += sh.slots.size();
            }
        }
        if (out_image) {
            ImageTensor u = unpack(out);
            std::memcpy(out_image, u.data.data(), u.data.size() * sizeof(double));
        }
        fill_ledger(eng.ledger(), ledger);
        if (out_level_drop) *out_level_drop = p.min_level() - out.min_level();
        return 0;
    } catch (...) {
        return -1;
    }
}

/// conv with bias and output_scale (conv.hpp:46-68): plan 1 / 2 = conv_plan
/// (ChannelFirst / ShiftFirst), 0 = convolve (image shards or channel shards,
/// chosen from the packing as the reference does). out_slots receives every
/// output shard's slots in order ([n_out][s]); returns the shard count (or -1).
int ref_conv_biased(int c, int m, int kappa, int c_out, const double* img, const double* filt, int plan,
                    uint64_t shard_size, const double* bias, double output_scale, double* out_slots, int cap_shards,
                    uint64_t* ledger) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        FilterTensor k(c, c_out, kappa);
        std::memcpy(k.weights.data(), filt, k.weights.size() * sizeof(double));
        std::vector<double> b(bias, bias + c_out);
        Engine eng;
        PackedImage p = pack(eng, t, shard_size);
        eng.ledger().reset();
        PackedImage out = plan == 1   ? conv_plan(eng, p, k, ConvPlan::ChannelFirst, b, output_scale)
                          : plan == 2 ? conv_plan(eng, p, k, ConvPlan::ShiftFirst, b, output_scale)
                                      : convolve(eng, p, k, b, output_scale);
        if (static_cast<int>(out.shards.size()) > cap_shards) return -1;
        size_t off = 0;
        for (const auto& sh : out.shards) {
            std::memcpy(out_slots + off, sh.slots.data(), sh.slots.size() * sizeof(double));
            off += sh.slots.size();
        }
        if (ledger) fill_ledger(eng.ledger(), ledger);
        return static_cast<int>(out.shards.size());
    } catch (...) {
        return -1;
    }
}

/// Textbook same-padding conv (reference oracle.cpp:7-31).
int ref_oracle_conv(int c, int m, int kappa, int c_out, const double* img, const double* filt,
                    int stride, double* out) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        FilterTensor k(c, c_out, kappa);
        std::memcpy(k.weights.data(), filt, k.weights.size() * sizeof(double));
        ImageTensor o = oracle_conv(t, k, stride);
        std::memcpy(out, o.data.data(), o.data.size() * sizeof(double));
        return 0;
    } catch (...) {
        return -1;
    }
}

/// strategy 0 = positive, 1 = signed. Returns the number of steps (or -1).
int ref_decompose(int strategy, uint64_t n, uint64_t s, long* steps, int cap) {
    try {
        std::vector<long> v = strategy == 0 ? decompose_positive(n, s) : decompose_signed(n, s);
        if (static_cast<int>(v.size()) > cap) return -1;
        std::copy(v.begin(), v.end(), steps);
        return static_cast<int>(v.size());
    } catch (...) {
        return -1;
    }
}

/// BFS minimal lengths for n in [0, n_max] (reference rot.cpp:84-94).
int ref_min_lengths(uint64_t n_max, uint64_t cap, uint64_t* out) {
    try {
        auto v = min_decomposition_lengths(n_max, cap);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
        return 0;
    } catch (...) {
        return -1;
    }
}

/// plan_rotations (rot.cpp:96-129). strategy 0 positive, 1 signed, 2 exact.
/// Writes per-request step lists (flattened, up to 64 steps each) and the
/// group index of each request. Returns total_keyed_rotations.
long ref_plan_rotations(const long* amounts, const int* same_source, int n, uint64_t s,
                        int strategy, long* steps_flat, int* n_steps, int* group_of,
                        int* group_hoisted) {
    try {
        std::vector<RotationRequest> req(n);
        for (int i = 0; i < n; ++i) req[i] = {amounts[i], same_source[i] != 0};
        DecompStrategy st = strategy == 0   ? DecompStrategy::Positive
                            : strategy == 1 ? DecompStrategy::Signed
                                            : DecompStrategy::Exact;
        RotationSchedule sch = plan_rotations(req, s, st);
        int r = 0;
        for (size_t g = 0; g < sch.groups.size(); ++g) {
            for (const auto& steps : sch.groups[g].steps) {
                n_steps[r] = static_cast<int>(steps.size());
                for (size_t k = 0; k < steps.size() && k < 64; ++k) steps_flat[r * 64 + k] = steps[k];
                group_of[r] = static_cast<int>(g);
                group_hoisted[r] = sch.groups[g].hoisted ? 1 : 0;
                ++r;
            }
        }
        return static_cast<long>(sch.total_keyed_rotations);
    } catch (...) {
        return -1;
    }
}

/// linear() (dense.cpp:71-75) on an image packed with pack(s): out_slots (s)
/// receives the output vector (features in slots 0..out-1), the ledger the
/// reference's op counters. slot_sum (dense.cpp:23-30) of a vector in `vec`
/// when `sum_block` > 0 (then img/w are ignored and out_slots gets the sum).
int ref_linear(int c, int m, const double* img, int out_features, const double* w, const double* b, uint64_t s,
               double* out_slots, uint64_t* ledger) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        LinearWeights lw((size_t)out_features, (size_t)c * m * m);
        std::memcpy(lw.w.data(), w, lw.w.size() * sizeof(double));
        std::memcpy(lw.b.data(), b, lw.b.size() * sizeof(double));
        Engine eng;
        PackedImage p = pack(eng, t, s);
        eng.ledger().reset();
        SlotVector out = linear(eng, p, lw);
        std::memcpy(out_slots, out.slots.data(), out.slots.size() * sizeof(double));
        fill_ledger(eng.ledger(), ledger);
        return (int)p.shards.size();
    } catch (...) {
        return -1;
    }
}

int ref_slot_sum(const double* vec, uint64_t s, uint64_t block, double* out) {
    try {
        Engine eng;
        SlotVector v = eng.encode(std::vector<double>(vec, vec + s));
        SlotVector r = slot_sum(eng, v, block);
        std::memcpy(out, r.slots.data(), s * sizeof(double));
        return 0;
    } catch (...) {
        return -1;
    }
}

/// pool() (pool.cpp:291-297): 2x2 average pooling of pack(img, s). Writes the
/// pooled shards' slots (out_slots, up to `cap` shards), meta = [m, c, d, rep,
/// mode, n_shards] and tau (c entries). Returns the shard count.
int ref_pool(int c, int m, const double* img, uint64_t s, double* out_slots, int cap, uint64_t* meta,
             uint64_t* tau, uint64_t* ledger) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        Engine eng;
        PackedImage p = pack(eng, t, s);
        eng.ledger().reset();
        PackedImage out = pool(eng, p);
        const int n = (int)out.shards.size();
        for (int u = 0; u < n && u < cap; ++u)
            std::memcpy(out_slots + (size_t)u * s, out.shards[(size_t)u].slots.data(), s * sizeof(double));
        meta[0] = out.m;
        meta[1] = out.c;
        meta[2] = out.d;
        meta[3] = out.rep;
        meta[4] = out.mode == ShardMode::ImageShard ? 0 : 1;
        meta[5] = (uint64_t)n;
        for (size_t j = 0; j < out.tau.size(); ++j) tau[j] = out.tau[j];
        fill_ledger(eng.ledger(), ledger);
        return n;
    } catch (...) {
        return -1;
    }
}

/// pool() / subsample_stride2() (pool.cpp:291-306) of pack(img, s) with an
/// output scale: window 1 = pool, 0 = stride-2. Same outputs as ref_pool, meta
/// gains [6] = rows_per_shard. Returns the shard count.
int ref_downsample(int c, int m, const double* img, uint64_t s, int window, double output_scale, double* out_slots,
                   int cap, uint64_t* meta, uint64_t* tau, uint64_t* ledger) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        Engine eng;
        PackedImage p = pack(eng, t, s);
        eng.ledger().reset();
        PackedImage out = window ? pool(eng, p, output_scale) : subsample_stride2(eng, p, output_scale);
        const int n = (int)out.shards.size();
        for (int u = 0; u < n && u < cap; ++u)
            std::memcpy(out_slots + (size_t)u * s, out.shards[(size_t)u].slots.data(), s * sizeof(double));
        meta[0] = out.m;
        meta[1] = out.c;
        meta[2] = out.d;
        meta[3] = out.rep;
        meta[4] = out.mode == ShardMode::ImageShard ? 0 : 1;
        meta[5] = (uint64_t)n;
        meta[6] = out.rows_per_shard;
        for (size_t j = 0; j < out.tau.size(); ++j) tau[j] = out.tau[j];
        fill_ledger(eng.ledger(), ledger);
        return n;
    } catch (...) {
        return -1;
    }
}

/// convolve(pool(pack(img, s)), k) (conv.cpp:364-371 on a pooled PackedImage: tau,
/// rep, duplication): out_slots = the conv's shards, meta = [m, c, d, rep, mode, n].
int ref_pool_conv(int c, int m, const double* img, uint64_t s, int kappa, int c_out, const double* filt,
                  double* out_slots, int cap, uint64_t* meta) {
    try {
        ImageTensor t(c, m);
        std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
        FilterTensor k(c, c_out, kappa);
        std::memcpy(k.weights.data(), filt, k.weights.size() * sizeof(double));
        Engine eng;
        PackedImage p = pool(eng, pack(eng, t, s));
        PackedImage out = convolve(eng, p, k);
        const int n = (int)out.shards.size();
        for (int u = 0; u < n && u < cap; ++u)
            std::memcpy(out_slots + (size_t)u * s, out.shards[(size_t)u].slots.data(), s * sizeof(double));
        meta[0] = out.m;
        meta[1] = out.c;
        meta[2] = out.d;
        meta[3] = out.rep;
        meta[4] = out.mode == ShardMode::ImageShard ? 0 : 1;
        meta[5] = (uint64_t)n;
        return n;
    } catch (...) {
        return -1;
    }
}

/// eval_chebyshev (act.cpp:151-162) of the slot vector `x` (s slots) placed at
/// `level`: out receives the slots, meta = [output level, max depth consumed],
/// ledger the op counters. Returns 0, or -2 with the exception text in `err`.
int ref_eval_chebyshev(const double* x, uint64_t s, int level, const double* coeffs, uint64_t n, double bound,
                       int prescaled, double* out, int64_t* meta, uint64_t* ledger, char* err, uint64_t err_cap) {
    try {
        Engine eng(EngineConfig{.initial_level = level});
        SlotVector v = eng.encode(std::vector<double>(x, x + s));
        ChebPoly p;
        p.bound = bound;
        p.coeffs.assign(coeffs, coeffs + n);
        SlotVector y = eval_chebyshev(eng, v, p, prescaled != 0);
        std::memcpy(out, y.slots.data(), s * sizeof(double));
        meta[0] = y.level;
        meta[1] = (int64_t)eng.ledger().max_depth_consumed.load();
        fill_ledger(eng.ledger(), ledger);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, err_cap, "%s", e.what());
        return -2;
    }
}

/// cheb_interpolate (act.cpp:90-113) of f on [-bound, bound] at degree n.
int ref_cheb_interpolate(double (*f)(double), uint64_t n, double bound, double* coeffs) {
    try {
        ChebPoly p = cheb_interpolate([f](double x) { return f(x); }, n, bound);
        std::memcpy(coeffs, p.coeffs.data(), p.coeffs.size() * sizeof(double));
        return 0;
    } catch (...) {
        return -1;
    }
}

/// Reference CPU path timing: runs conv_plan(plan) `iters` times on each of
/// `threads` independent Engines (the reference's Engine is not shared
/// across threads, emu.hpp:181). Returns wall seconds for the whole batch.
double ref_time_conv(int c, int m, int kappa, int c_out, const double* img, const double* filt,
                     int plan, uint64_t shard_size, int iters, int threads) {
    ImageTensor t(c, m);
    std::memcpy(t.data.data(), img, t.data.size() * sizeof(double));
    FilterTensor k(c, c_out, kappa);
    std::memcpy(k.weights.data(), filt, k.weights.size() * sizeof(double));
    auto work = [&]() {
        Engine eng;
        PackedImage p = pack(eng, t, shard_size);
        for (int i = 0; i < iters; ++i) {
            PackedImage out = run_plan(eng, p, k, plan);
            (void)out;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

/// Reference rotation microbenchmark leg (cfg2): executes the plan for
/// amounts 1..n_amounts on `vectors` random vectors of s slots per thread.
/// Returns wall seconds; writes total keyed steps per vector.
double ref_time_rotations(uint64_t s, int strategy, int n_amounts, int vectors, int threads,
                          uint64_t* keyed_per_vector) {
    std::vector<RotationRequest> req;
    for (int a = 1; a <= n_amounts; ++a) req.push_back({a, false});
    DecompStrategy st = strategy == 0 ? DecompStrategy::Positive : DecompStrategy::Signed;
    RotationSchedule sch = plan_rotations(req, s, st);
    if (keyed_per_vector) *keyed_per_vector = sch.total_keyed_rotations;
    auto work = [&](int tid) {
        Engine eng;
        std::mt19937_64 rng(1000 + tid);
        for (int v = 0; v < vectors; ++v) {
            SlotVector x = eng.encode(random_values(rng, s));
            auto out = execute_schedule(eng, x, sch);
            (void)out;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(work, i);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}



// ------------------------------------------------------------ network runner (net.cpp)
namespace {

/// The networks of the reference's tests/test_net.cpp, built with its own
/// helpers: 0 = tiny_network() (tiny_net.hpp), 1 = the stride-2 network
/// (test_net.cpp:202-235), 2 = the activation-first network (:236-262),
/// 3 = the channel-sharded network (:263-301; m = side of the input).
NetworkSpec build_net(int which, ImageTensor& input, std::size_t side) {
    if (which == 0) {
        input = tiny_input();
        return tiny_network();
    }
    NetworkSpec spec;
    spec.shard_size = 256;
    spec.initial_level = 16;
    if (which == 1) {
        std::mt19937_64 rng(2024);
        LayerSpec conv;
        conv.type = LayerType::Conv;
        conv.name = "conv_s2";
        conv.filter = random_filter(rng, 4, 4, 3);
        for (double& w : conv.filter.weights) w *= 0.2;
        conv.bias = random_values(rng, 4, -0.1, 0.1);
        conv.stride = 2;
        spec.layers.push_back(conv);
        LayerSpec act;
        act.type = LayerType::Gelu;
        act.name = "gelu";
        act.degree = 27;
        act.bound = 10.0;
        spec.layers.push_back(act);
        LayerSpec head;
        head.type = LayerType::PoolLinear;
        head.name = "head";
        head.weights = LinearWeights(3, 4);
        head.weights.w = random_values(rng, 12);
        head.weights.b = random_values(rng, 3);
        spec.layers.push_back(head);
        input = tiny_input();
    } else if (which == 2) {
        std::mt19937_64 rng(2025);
        LayerSpec act;
        act.type = LayerType::Gelu;
        act.name = "gelu_first";
        act.degree = 27;
        act.bound = 4.0;
        spec.layers.push_back(act);
        LayerSpec head;
        head.type = LayerType::Linear;
        head.name = "fc";
        head.weights = LinearWeights(5, 4 * 64);
        head.weights.w = random_values(rng, head.weights.w.size());
        head.weights.b = random_values(rng, 5);
        spec.layers.push_back(head);
        input = tiny_input();
    } else {
        std::mt19937_64 rng(2026);
        spec.shard_size = 128;
        LayerSpec conv;
        conv.type = LayerType::Conv;
        conv.name = "conv";
        conv.filter = random_filter(rng, 2, 2, 3);
        for (double& w : conv.filter.weights) w *= 0.3;
        conv.bias = random_values(rng, 2, -0.1, 0.1);
        spec.layers.push_back(conv);
        LayerSpec pool_layer;
        pool_layer.type = LayerType::Pool;
        pool_layer.name = "pool";
        spec.layers.push_back(pool_layer);
        LayerSpec act;
        act.type = LayerType::Gelu;
        act.name = "gelu";
        act.degree = 27;
        act.bound = 10.0;
        spec.layers.push_back(act);
        LayerSpec head;
        head.type = LayerType::PoolLinear;
        head.name = "head";
        head.weights = LinearWeights(4, 2);
        head.weights.w = random_values(rng, 8);
        head.weights.b = random_values(rng, 4);
        spec.layers.push_back(head);
        std::mt19937_64 irng(77);
        input = random_tensor(irng, 2, side);
    }
    return spec;
}

void json_array(std::ofstream& f, const std::vector<double>& v) {
    f << "[";
    for (std::size_t i = 0; i < v.size(); ++i) f << v[i] << (i + 1 < v.size() ? ", " : "");
    f << "]";
}

}  // namespace

/// Writes network `which` as a JSON description + fixture files (the
/// reference's own save_filter / save_linear / save_tensor formats, io.cpp)
/// into `dir`: net.json, <layer>.filt, <layer>.lin, input.tensor.
int ref_write_network(int which, const char* dir, uint64_t side) {
    try {
        ImageTensor input(1, 1);
        NetworkSpec spec = build_net(which, input, side);
        const std::string d(dir);
        std::ofstream f(d + "/net.json");
        f << std::setprecision(17);
        f << "{\n  \"shard_size\": " << spec.shard_size << ",\n  \"initial_level\": " << spec.initial_level
          << ",\n  \"seed\": " << spec.seed << ",\n  \"noise\": {\"enabled\": false},\n"
          << "  \"bootstrap\": {\"auto\": true},\n  \"layers\": [\n";
        for (std::size_t i = 0; i < spec.layers.size(); ++i) {
            const LayerSpec& l = spec.layers[i];
            f << "    {\"type\": \"" << layer_type_name(l.type) << "\", \"name\": \"" << l.name << "\"";
            if (l.type == LayerType::Conv) {
                save_filter(d + "/" + l.name + ".filt", l.filter, l.bias);
                f << ", \"filter\": \"" << l.name << ".filt\"";
                if (l.stride != 1) f << ", \"stride\": " << l.stride;
                if (l.bn) {
                    f << ", \"bn_scale\": ";
                    json_array(f, l.bn->scale);
                    f << ", \"bn_bias\": ";
                    json_array(f, l.bn->bias);
                }
            } else if (l.type == LayerType::Gelu) {
                f << ", \"degree\": " << l.degree << ", \"bound\": " << l.bound;
            } else if (l.type == LayerType::Linear || l.type == LayerType::PoolLinear) {
                save_linear(d + "/" + l.name + ".lin", l.weights);
                f << ", \"weights\": \"" << l.name << ".lin\"";
            }
            f << "}" << (i + 1 < spec.layers.size() ? "," : "") << "\n";
        }
        f << "  ]\n}\n";
        save_tensor(d + "/input.tensor", input);
        return 0;
    } catch (...) {
        return -1;
    }
}

/// run_network (net.cpp:112-257) of a JSON network on a tensor fixture, with
/// the shard size / initial level overridden when > 0. info[i] = [level_before,
/// level_after, depth_consumed, bootstrapped] per layer, err[i] = its max_abs_err;
/// meta = [n_layers, n_logits]; logits / oracle_logits (cap entries). Returns 0,
/// or -2 with the exception text in `msg`.
int ref_run_network(const char* json, const char* input_path, uint64_t shard_size, int initial_level,
                    int auto_boot, double* logits, double* oracle_logits, int cap, int64_t* info, double* err,
                    int64_t* meta, uint64_t* totals, char* msg, uint64_t msg_cap) {
    try {
        NetworkSpec spec = load_network(json);
        if (shard_size) spec.shard_size = shard_size;
        if (initial_level > 0) spec.initial_level = initial_level;
        if (auto_boot >= 0) spec.bootstrap.auto_insert = auto_boot != 0;
        ImageTensor input = load_tensor(input_path);
        RunReport r = run_network(spec, input);
        meta[0] = (int64_t)r.layers.size();
        meta[1] = (int64_t)r.logits.size();
        for (std::size_t i = 0; i < r.layers.size(); ++i) {
            info[4 * i + 0] = r.layers[i].level_before;
            info[4 * i + 1] = r.layers[i].level_after;
            info[4 * i + 2] = r.layers[i].depth_consumed;
            info[4 * i + 3] = r.layers[i].bootstrapped;
            err[i] = r.layers[i].max_abs_err;
        }
        for (std::size_t o = 0; o < r.logits.size() && (int)o < cap; ++o) {
            logits[o] = r.logits[o];
            oracle_logits[o] = r.oracle_logits[o];
        }
        totals[0] = r.totals.rotations;
        totals[1] = r.totals.hoisted_rotations;
        totals[2] = r.totals.hoist_groups;
        totals[3] = r.totals.ct_pt_mults;
        totals[4] = r.totals.ct_ct_mults;
        totals[5] = r.totals.adds;
        totals[6] = r.totals.bootstraps;
        totals[7] = (uint64_t)r.totals.max_depth_consumed;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(msg, msg_cap, "%s", e.what());
        return -2;
    }
}

}  // extern "C"
