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
//   auto layer = eng.make_conv_layer(16, 16, 32, 3, weights, eng.max_level());
//   eng.gen_galois_keys(layer.steps());
//   auto ct  = eng.encode_encrypt(slots, 9000);
//   auto out = eng.conv_plan(ct, layer, fheconv::ConvPlan::ShiftFirst);
//   std::vector<double> y = eng.decrypt(out);
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fheconv.h"

namespace fheconv {

// reference conv.hpp:17 — ChannelFirst = paper Approach 1, ShiftFirst = Approach 2
enum class ConvPlan { ChannelFirst = 1, ShiftFirst = 2 };

struct Params {
    int log_n;
    std::vector<int> q_bits, p_bits;
    int log_scale;
    int device = 0;
    static Params cfg1() { return {13, {60, 40, 40, 40, 40}, {60}, 40}; }
    static Params cfg3() { return {15, {60, 50, 50, 50, 50, 50, 50, 50, 50, 50, 50, 50, 50}, {60, 60}, 50}; }
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
    std::vector<int64_t> steps() const {
        std::vector<int64_t> s(1024);
        size_t n = 0;
        fhe_conv_layer_steps(h_.get(), 2, s.data(), s.size(), &n);
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

    // conv_plan (conv.cpp:266-271) on a pre-encoded layer
    ConvLayer make_conv_layer(int c_in, int c_out, int m, int kappa, const std::vector<double>& weights, int level) {
        fhe_conv_layer* l = nullptr;
        check(fhe_conv_layer_create(raw(), c_in, c_out, m, kappa, weights.data(), level, &l));
        return ConvLayer(l);
    }
    Ciphertext conv_plan(const Ciphertext& ct, const ConvLayer& layer, ConvPlan plan) {
        fhe_ct* o = nullptr;
        check(fhe_conv2d(raw(), ct.get(), layer.get(), (int)plan, &o));
        return Ciphertext(o);
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
    // convolve (conv.cpp:364-371) of an image-mode PackedImage (any tau / rep / duplication)
    Packed convolve(const Packed& p, int c_out, int kappa, const std::vector<double>& weights) {
        if (p.shards.empty()) throw std::invalid_argument("packed image has no shards");
        fhe_conv_layer* l = nullptr;
        check(fhe_conv_layer_create_packed(raw(), p.c, c_out, p.m, kappa, weights.data(), p.shards[0].level(),
                                           p.shards.size(), p.tau.empty() ? nullptr : p.tau.data(), p.rep, p.d, &l));
        ConvLayer layer(l);
        {  // Galois keys of the layer's rotations (existing keys are kept)
            std::vector<int64_t> st(4096);
            size_t ns = 0;
            check(fhe_conv_layer_steps(l, 0, st.data(), st.size(), &ns));
            check(fhe_gen_galois_keys(raw(), st.data(), ns));
        }
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
