// fheconv.hpp — header-only, Engine-shaped C++ wrapper over the C ABI.
//
// Mirrors the reference evaluator shardnn::Engine (reference
// proj/include/shardnn/emu.hpp:132-183) and conv_plan (conv.hpp:66-68):
// same method names, value semantics for ciphertexts (move-only handles
// here), and the same exception types and messages ("slot count mismatch",
// "depth exhausted", "empty rotation batch", "insufficient capacity", ...),
// so code written against shardnn::Engine ports mechanically:
//
//   fheconv::Engine eng(fheconv::Params::cfg3());
//   eng.keygen(7);
//   auto layer = eng.make_conv_layer(16, 16, 32, 3, weights, eng.max_level(), bias, 0.5);
//   eng.gen_galois_keys(layer.steps());
//   auto ct  = eng.encode_encrypt(slots, 9000);
//   auto out = eng.conv_plan(ct, layer, fheconv::ConvPlan::ShiftFirst);
//   std::vector<double> y = eng.decrypt(out);
//
// or, with the reference's argument list (conv.hpp:66-68; the layer is built
// once per (geometry, weights, bias, output_scale, level) and cached):
//   auto out = eng.conv_plan(ct, 16, 16, 32, 3, weights, fheconv::ConvPlan::Fused, bias, 0.5);
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <tuple>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fheconv.h"

namespace fheconv {

// reference conv.hpp:17 — ChannelFirst = paper Approach 1, ShiftFirst = Approach 2;
// the B200 schedules of fhe_conv2d (include/fheconv.h) follow: BabyGiant (channel
// rotations hoisted, shifts as giant steps), BabyGiantShifts (roles swapped), Fused
// (the c kappa rotations r m^2 + ll in one fused kernel, kappa row-shift giants) and
// Auto (the fused schedule whenever it applies). All decrypt to the same slots.
enum class ConvPlan { Auto = 0, ChannelFirst = 1, ShiftFirst = 2, BabyGiant = 3, BabyGiantShifts = 4, Fused = 5 };

// BASELINE.json configs (N, Q and P prime bit sizes, log2 scale)
struct Params {
    int log_n;
    std::vector<int> q_bits, p_bits;
    int log_scale;
    int device = 0;
    static Params cfg1() { return {13, {60, 40, 40, 40, 40}, {60}, 40}; }
    static Params cfg2() { return {14, std::vector<int>(8, 50), {60}, 50}; }
    static Params cfg3() { return {15, q_list(60, 50, 12), {60, 60}, 50}; }
    static Params cfg4() { return {16, q_list(60, 50, 16), {60, 60, 60}, 50}; }
    static Params cfg5() { return cfg3(); }  // three cfg3 layers, batch of 32

private:
    static std::vector<int> q_list(int first, int rest, int n) {
        std::vector<int> v(1, first);
        v.insert(v.end(), (size_t)n, rest);
        return v;
    }
};

class Ciphertext {
public:
    Ciphertext() = default;
    explicit Ciphertext(fhe_ct* h) : h_(h) {}
    int level() const { return fhe_ct_level(h_.get()); }
    double scale() const { return fhe_ct_scale(h_.get()); }
    fhe_ct* get() const { return h_.get(); }
    explicit operator bool() const { return (bool)h_; }

private:
    struct Del {
        void operator()(fhe_ct* p) const { fhe_ct_free(p); }
    };
    std::unique_ptr<fhe_ct, Del> h_;
};

class Plaintext {
public:
    explicit Plaintext(fhe_pt* h) : h_(h) {}
    fhe_pt* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(fhe_pt* p) const { fhe_pt_free(p); }
    };
    std::unique_ptr<fhe_pt, Del> h_;
};

class ConvLayer {
public:
    explicit ConvLayer(fhe_conv_layer* h) : h_(h) {}
    fhe_conv_layer* get() const { return h_.get(); }
    // Galois steps of a plan's rotations; Auto (default) = the union, so every plan runs
    std::vector<int64_t> steps(ConvPlan plan = ConvPlan::Auto) const {
        std::vector<int64_t> s(8192);
        size_t n = 0;
        fhe_conv_layer_steps(h_.get(), (int)plan, s.data(), s.size(), &n);
        s.resize(n);
        return s;
    }

private:
    struct Del {
        void operator()(fhe_conv_layer* p) const { fhe_conv_layer_free(p); }
    };
    std::unique_ptr<fhe_conv_layer, Del> h_;
};

// PackedImage (reference pack.hpp) whose shards are ciphertexts
struct Packed {
    std::vector<Ciphertext> shards;
    int m = 0, c = 0, rep = 1, d = 1, mode = 0;  // mode 0 image shards, 1 channel shards
    std::vector<int64_t> tau;                    // physical channel position -> logical channel
};

class Engine {
public:
    explicit Engine(const Params& p) {
        fhe_params fp{p.log_n, (int)p.q_bits.size(), p.q_bits.data(), (int)p.p_bits.size(), p.p_bits.data(),
                      p.log_scale, p.device};
        fhe_ctx* c = nullptr;
        const int rc = fhe_ctx_create(&fp, &c);
        if (rc != FHE_OK) throw std::runtime_error("fhe_ctx_create failed (no sm_100 GPU?)");
        ctx_.reset(c);
        int nq = 0, np = 0, dn = 0, ln = 0;
        primes_.resize(p.q_bits.size() + p.p_bits.size());
        fhe_ctx_info(c, &ln, &nq, &np, &dn, primes_.data());
        slots_ = (size_t)1 << (ln - 1);
        max_level_ = nq - 1;
        scale_ = (double)(1ULL << p.log_scale);
    }

    // cached layers release their device memory before the context goes away
    ~Engine() {
        layers_.clear();
        packed_layers_.clear();
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    size_t slots() const { return slots_; }
    int max_level() const { return max_level_; }
    fhe_ctx* raw() const { return ctx_.get(); }

    void keygen(uint64_t seed) { check(fhe_keygen(raw(), seed)); }
    void gen_galois_keys(const std::vector<int64_t>& steps) {
        check(fhe_gen_galois_keys(raw(), steps.data(), steps.size()));
    }

    // Engine::encode (emu.hpp:144-152): fresh vector at the top level
    Plaintext encode(const std::vector<double>& slots, int level = -1, double scale = 0.0) {
        fhe_pt* p = nullptr;
        check(fhe_encode(raw(), slots.data(), slots.size(), level < 0 ? max_level_ : level,
                         scale == 0.0 ? scale_ : scale, 0, &p));
        return Plaintext(p);
    }
    Ciphertext encrypt(const Plaintext& pt, uint64_t seed) {
        fhe_ct* o = nullptr;
        check(fhe_encrypt(raw(), pt.get(), seed, &o));
        return Ciphertext(o);
    }
    Ciphertext encode_encrypt(const std::vector<double>& slots, uint64_t seed) {
        return encrypt(encode(slots), seed);
    }
    std::vector<double> decrypt(const Ciphertext& ct) {
        std::vector<double> out(slots_);
        check(fhe_decrypt_decode(raw(), ct.get(), out.data(), out.size()));
        return out;
    }

    // Engine::rotate (emu.cpp:28-37)
    Ciphertext rotate(const Ciphertext& v, long k) { return unary(fhe_rotate, v, (int64_t)k); }
    // Engine::rotate_many (emu.cpp:39-54) — one shared ModUp
    std::vector<Ciphertext> rotate_many(const Ciphertext& v, const std::vector<long>& ks) {
        std::vector<int64_t> k64(ks.begin(), ks.end());
        std::vector<fhe_ct*> outs(ks.size() ? ks.size() : 1, nullptr);
        check(fhe_rotate_hoisted(raw(), v.get(), k64.data(), k64.size(), outs.data()));
        std::vector<Ciphertext> r;
        for (size_t i = 0; i < ks.size(); ++i) r.emplace_back(outs[i]);
        return r;
    }
    // Engine::mul_plain (emu.cpp:56-67): consumes one level (multiply by a
    // plaintext at scale q_level, then rescale — the scale is preserved)
    Ciphertext mul_plain(const Ciphertext& v, const std::vector<double>& p) {
        if (p.size() != slots_) throw std::invalid_argument("slot count mismatch");
        if (v.level() < 1) throw std::runtime_error("depth exhausted");
        Plaintext pt = encode(p, v.level(), (double)primes_[v.level()]);
        fhe_ct* m = nullptr;
        check(fhe_mul_plain(raw(), v.get(), pt.get(), &m));
        Ciphertext mc(m);
        return unary0(fhe_rescale, mc);
    }
    Ciphertext add(const Ciphertext& a, const Ciphertext& b) { return binary(fhe_add, a, b); }
    Ciphertext sub(const Ciphertext& a, const Ciphertext& b) { return binary(fhe_sub, a, b); }
    Ciphertext add_plain(const Ciphertext& v, const std::vector<double>& p) {
        if (p.size() != slots_) throw std::invalid_argument("slot count mismatch");
        Plaintext pt = encode(p, v.level(), v.scale());
        fhe_ct* o = nullptr;
        check(fhe_add_plain(raw(), v.get(), pt.get(), &o));
        return Ciphertext(o);
    }

    // a pre-encoded conv layer: ImageConv's fused plaintexts (conv.cpp:69-85) with the
    // output scale folded in, and the bias (bias_plain :87-94) added in the conv epilogue
    ConvLayer make_conv_layer(int c_in, int c_out, int m, int kappa, const std::vector<double>& weights, int level,
                              const std::vector<double>& bias = {}, double output_scale = 1.0) {
        if (!bias.empty() && bias.size() != (size_t)c_out)
            throw std::invalid_argument("bias size does not match output channels");
        fhe_conv_layer* l = nullptr;
        check(fhe_conv_layer_create(raw(), c_in, c_out, m, kappa, weights.data(), bias.empty() ? nullptr : bias.data(),
                                    output_scale, level, &l));
        return ConvLayer(l);
    }
    // conv_plan (conv.cpp:266-271) on a pre-encoded layer
    Ciphertext conv_plan(const Ciphertext& ct, const ConvLayer& layer, ConvPlan plan) {
        fhe_ct* o = nullptr;
        check(fhe_conv2d(raw(), ct.get(), layer.get(), (int)plan, &o));
        return Ciphertext(o);
    }
    // conv_plan with the reference's argument list (conv.hpp:66-68): the layer for
    // (geometry, weights, bias, output_scale, level) is encoded once and cached, its
    // Galois keys generated on first use
    Ciphertext conv_plan(const Ciphertext& ct, int c_in, int c_out, int m, int kappa, const std::vector<double>& weights,
                         ConvPlan plan, const std::vector<double>& bias = {}, double output_scale = 1.0) {
        return conv_plan(ct, cached_layer(c_in, c_out, m, kappa, weights, ct.level(), bias, output_scale), plan);
    }
    // a batch of independent ciphertexts through one layer (keys and plaintexts streamed
    // once per batch; BASELINE cfg5)
    std::vector<Ciphertext> conv_batch(const std::vector<const Ciphertext*>& cts, const ConvLayer& layer,
                                       ConvPlan plan = ConvPlan::Auto) {
        std::vector<const fhe_ct*> in;
        for (const Ciphertext* c : cts) in.push_back(c->get());
        std::vector<fhe_ct*> outs(in.size() ? in.size() : 1, nullptr);
        check(fhe_conv2d_batch(raw(), in.data(), in.size(), layer.get(), (int)plan, outs.data()));
        std::vector<Ciphertext> r;
        for (size_t i = 0; i < in.size(); ++i) r.emplace_back(outs[i]);
        return r;
    }

    // Engine::mul_ct (emu.cpp:69-80): relinearised and rescaled (gen_relin_key() first)
    void gen_relin_key() { check(fhe_gen_relin_key(raw())); }
    Ciphertext mul_ct(const Ciphertext& a, const Ciphertext& b) { return binary(fhe_mul, a, b); }
    // Engine::add_scalar (emu.cpp:113-119)
    Ciphertext add_scalar(const Ciphertext& v, double k) { return unary(fhe_add_scalar, v, k); }
    // eval_chebyshev (act.cpp:151-162): sum_k coeffs[k] T_k(x / bound)
    Ciphertext eval_chebyshev(const Ciphertext& x, const std::vector<double>& coeffs, double bound,
                              bool prescaled) {
        return unary(fhe_eval_chebyshev, x, coeffs.data(), coeffs.size(), bound, (int)prescaled);
    }
    // slot_sum (dense.cpp:23-30)
    Ciphertext slot_sum(const Ciphertext& v, size_t block) {
        const fhe_ct* in = v.get();
        fhe_ct* o = nullptr;
        check(fhe_slot_sum_batch(raw(), &in, 1, block, &o));
        return Ciphertext(o);
    }
    // pool / subsample_stride2 (pool.cpp:291-306) of any PackedImage
    Packed pool(const Packed& p, double output_scale = 1.0) { return downsample(p, true, output_scale); }
    Packed subsample_stride2(const Packed& p, double output_scale = 1.0) { return downsample(p, false, output_scale); }
    // convolve (conv.cpp:364-371) of an image-mode PackedImage (any tau / rep /
    // duplication), with bias and output_scale; the layer of a packing is encoded once
    // and cached (repeated inference re-uses it and its keys)
    Packed convolve(const Packed& p, int c_out, int kappa, const std::vector<double>& weights,
                    const std::vector<double>& bias = {}, double output_scale = 1.0) {
        if (p.shards.empty()) throw std::invalid_argument("packed image has no shards");
        if (!bias.empty() && bias.size() != (size_t)c_out)
            throw std::invalid_argument("bias size does not match output channels");
        const PackedKey key{p.c, c_out, p.m, kappa, p.shards[0].level(), (int)p.shards.size(), p.rep, p.d, p.tau,
                            weights, bias, output_scale};
        auto it = packed_layers_.find(key);
        if (it == packed_layers_.end()) {
            fhe_conv_layer* nl = nullptr;
            check(fhe_conv_layer_create_packed(raw(), p.c, c_out, p.m, kappa, weights.data(),
                                               bias.empty() ? nullptr : bias.data(), output_scale,
                                               p.shards[0].level(), p.shards.size(),
                                               p.tau.empty() ? nullptr : p.tau.data(), p.rep, p.d, &nl));
            it = packed_layers_.emplace(key, std::make_shared<ConvLayer>(nl)).first;
            // Galois keys of the layer's rotations (existing keys are kept)
            std::vector<int64_t> st(8192);
            size_t ns = 0;
            check(fhe_conv_layer_steps(nl, 0, st.data(), st.size(), &ns));
            check(fhe_gen_galois_keys(raw(), st.data(), ns));
        }
        fhe_conv_layer* l = it->second->get();
        int t = 0, n_out = 0, d_out = 1;
        fhe_conv_layer_shards(l, &t, &n_out);
        fhe_conv_layer_output_packing(l, &d_out);
        std::vector<const fhe_ct*> in;
        for (const auto& s : p.shards) in.push_back(s.get());
        std::vector<fhe_ct*> outs((size_t)n_out);
        for (auto& o : outs) {  // output handles at level - 1 (contents overwritten)
            fhe_pt* z = nullptr;
            const double zero = 0.0;
            check(fhe_encode(raw(), &zero, 1, p.shards[0].level() - 1, scale_, 0, &z));
            Plaintext zp(z);
            check(fhe_encrypt(raw(), z, 1, &o));
        }
        check(fhe_conv2d_shards_into(raw(), in.data(), 1, l, outs.data()));
        Packed r;
        for (fhe_ct* o : outs) r.shards.emplace_back(o);
        r.m = p.m;
        r.c = c_out;
        r.d = d_out;
        for (int j = 0; j < c_out; ++j) r.tau.push_back(j);
        return r;
    }
    // linear (dense.cpp:71-75) over a slot -> feature map (pack.cpp:109-129)
    Ciphertext linear(const Packed& p, const std::vector<int64_t>& features, size_t in_features, int out_features,
                      const std::vector<double>& w, const std::vector<double>& b) {
        std::vector<const fhe_ct*> in;
        for (const auto& s : p.shards) in.push_back(s.get());
        fhe_ct* o = nullptr;
        check(fhe_linear_features(raw(), in.data(), in.size(), features.data(), in_features, out_features, w.data(),
                                  b.data(), &o));
        return Ciphertext(o);
    }

    fhe_ledger ledger() const {
        fhe_ledger l{};
        fhe_ledger_get(raw(), &l);
        return l;
    }

private:
    // layer caches (conv_plan with weights, convolve): keyed by everything the encoding depends on
    using LayerKey = std::tuple<int, int, int, int, int, std::vector<double>, std::vector<double>, double>;
    using PackedKey = std::tuple<int, int, int, int, int, int, int, int, std::vector<int64_t>, std::vector<double>,
                                 std::vector<double>, double>;
    std::map<LayerKey, std::shared_ptr<ConvLayer>> layers_;
    std::map<PackedKey, std::shared_ptr<ConvLayer>> packed_layers_;

    const ConvLayer& cached_layer(int c_in, int c_out, int m, int kappa, const std::vector<double>& weights, int level,
                                  const std::vector<double>& bias, double output_scale) {
        const LayerKey key{c_in, c_out, m, kappa, level, weights, bias, output_scale};
        auto it = layers_.find(key);
        if (it == layers_.end()) {
            auto ly = std::make_shared<ConvLayer>(make_conv_layer(c_in, c_out, m, kappa, weights, level, bias,
                                                                  output_scale));
            gen_galois_keys(ly->steps());
            it = layers_.emplace(key, std::move(ly)).first;
        }
        return *it->second;
    }

    Packed downsample(const Packed& p, bool window, double output_scale) {
        std::vector<const fhe_ct*> in;
        for (const auto& s : p.shards) in.push_back(s.get());
        std::vector<fhe_ct*> outs(in.size() ? in.size() : 1, nullptr);
        Packed r;
        r.tau.assign((size_t)p.c, 0);
        size_t n = 0;
        check(fhe_downsample(raw(), in.data(), in.size(), p.c, p.m, p.tau.empty() ? nullptr : p.tau.data(), p.rep, p.d,
                             (int)window, output_scale, outs.data(), &n, r.tau.data(), &r.rep, &r.d, &r.mode));
        for (size_t u = 0; u < n; ++u) r.shards.emplace_back(outs[u]);
        r.m = p.m / 2;
        r.c = p.c;
        return r;
    }
    struct Del {
        void operator()(fhe_ctx* p) const { fhe_ctx_destroy(p); }
    };
    std::unique_ptr<fhe_ctx, Del> ctx_;
    std::vector<uint64_t> primes_;
    size_t slots_ = 0;
    int max_level_ = 0;
    double scale_ = 1.0;

    void check(int rc) const {
        if (rc == FHE_OK) return;
        const std::string msg = fhe_last_error(raw());
        if (rc == FHE_E_INVALID) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    template <class F, class... A>
    Ciphertext unary(F f, const Ciphertext& v, A... a) {
        fhe_ct* o = nullptr;
        check(f(raw(), v.get(), a..., &o));
        return Ciphertext(o);
    }
    template <class F>
    Ciphertext unary0(F f, const Ciphertext& v) {
        fhe_ct* o = nullptr;
        check(f(raw(), v.get(), &o));
        return Ciphertext(o);
    }
    template <class F>
    Ciphertext binary(F f, const Ciphertext& a, const Ciphertext& b) {
        fhe_ct* o = nullptr;
        check(f(raw(), a.get(), b.get(), &o));
        return Ciphertext(o);
    }
};

}  // namespace fheconv
