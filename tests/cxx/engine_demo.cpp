// Drives the Engine-shaped C++ wrapper (include/fheconv.hpp) the way the
// reference's test_conv.cpp drives shardnn::Engine: a 4->4 3x3 conv at
// BASELINE cfg1, both plans, checked against a textbook same-padding conv
// (reference oracle.cpp:7-31 semantics) computed here. Exit code 0 = pass.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "fheconv.hpp"

int main() {
    const int c = 4, m = 32, k = 3;
    std::mt19937_64 rng(1000);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::vector<double> img(c * m * m), w(c * c * k * k);
    for (double& v : img) v = U(rng);
    for (double& v : w) v = U(rng);
    std::vector<double> ref(c * m * m, 0.0);
    for (int g = 0; g < c; ++g)
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                double acc = 0;
                for (int f = 0; f < c; ++f)
                    for (int a = -1; a <= 1; ++a)
                        for (int b = -1; b <= 1; ++b) {
                            const int ii = i + a, jj = j + b;
                            if (ii < 0 || jj < 0 || ii >= m || jj >= m) continue;
                            acc += w[((f * c + g) * k + a + 1) * k + b + 1] * img[(f * m + ii) * m + jj];
                        }
                ref[(g * m + i) * m + j] = acc;
            }
    try {
        fheconv::Engine eng(fheconv::Params::cfg1());
        eng.keygen(7);
        auto layer = eng.make_conv_layer(c, c, m, k, w, eng.max_level());
        eng.gen_galois_keys(layer.steps());
        auto ct = eng.encode_encrypt(img, 9000);
        double worst = 0;
        for (auto plan : {fheconv::ConvPlan::ChannelFirst, fheconv::ConvPlan::ShiftFirst}) {
            auto out = eng.conv_plan(ct, layer, plan);
            if (out.level() != ct.level() - 1) return 2;
            auto y = eng.decrypt(out);
            for (size_t i = 0; i < ref.size(); ++i) worst = std::fmax(worst, std::fabs(y[i] - ref[i]));
        }
        // conv_plan with the reference's argument list (conv.hpp:66-68): bias and output_scale,
        // every B200 schedule; the layer is cached across calls
        {
            const std::vector<double> bias = {0.25, -0.5, 0.125, 0.0};
            const double osc = 0.5;
            for (auto plan : {fheconv::ConvPlan::ShiftFirst, fheconv::ConvPlan::Fused, fheconv::ConvPlan::Auto,
                              fheconv::ConvPlan::BabyGiant}) {
                auto out = eng.conv_plan(ct, c, c, m, k, w, plan, bias, osc);
                auto y = eng.decrypt(out);
                for (size_t i = 0; i < ref.size(); ++i)
                    worst = std::fmax(worst, std::fabs(y[i] - (ref[i] + bias[i / (m * m)]) * osc));
            }
            std::vector<const fheconv::Ciphertext*> batch = {&ct, &ct};
            auto outs = eng.conv_batch(batch, layer, fheconv::ConvPlan::Fused);
            auto y = eng.decrypt(outs[1]);
            for (size_t i = 0; i < ref.size(); ++i) worst = std::fmax(worst, std::fabs(y[i] - ref[i]));
            bool bad_bias = false;
            try {
                eng.make_conv_layer(c, c, m, k, w, eng.max_level(), {1.0, 2.0});
            } catch (const std::invalid_argument& e) {
                bad_bias = std::string(e.what()) == "bias size does not match output channels";
            }
            if (!bad_bias) return 5;
        }
        // Engine::rotate_many / rotate / mul_plain semantics
        auto rots = eng.rotate_many(ct, {1, -1});
        auto r1 = eng.decrypt(rots[0]);
        for (size_t i = 0; i < img.size(); ++i) worst = std::fmax(worst, std::fabs(r1[i] - img[(i + 1) % img.size()]));
        std::vector<double> half(img.size(), 0.5);
        auto mp = eng.decrypt(eng.mul_plain(ct, half));
        for (size_t i = 0; i < img.size(); ++i) worst = std::fmax(worst, std::fabs(mp[i] - 0.5 * img[i]));
        bool threw = false;
        try {
            eng.rotate_many(ct, {});
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "empty rotation batch";
        }
        // pool (pool.cpp:291-297) of the input, then a 1x1 conv on the pooled packing (rep 4,
        // duplicated), then slot_sum (dense.cpp:23-30) — the reference's operator chain (cfg1: 4 levels)
        {
            std::vector<int64_t> st = {1, m, m + 1};
            for (int i = 1; i < m / 2; ++i) st.push_back(i);
            for (int j = 1; j < m / 2; ++j) st.push_back(3 * j * m / 2);
            const int bn = (m / 2) * (m / 2);
            for (int q = 1; q < 4; ++q) st.push_back(-q * bn);
            for (int e = 1; e < 4096; e *= 2) st.push_back(e);
            eng.gen_galois_keys(st);
            fheconv::Packed p;
            p.shards.push_back(eng.encode_encrypt(img, 9001));
            p.m = m;
            p.c = c;
            p.tau = {0, 1, 2, 3};
            fheconv::Packed pooled = eng.pool(p);
            if (pooled.rep != 4 || pooled.d != 4 || pooled.shards.size() != 1) return 4;
            auto y = eng.decrypt(pooled.shards[0]);
            const int mn = m / 2;
            for (int g = 0; g < c; ++g)  // block (g * rep) holds channel tau[g]
                for (int i = 0; i < mn; ++i)
                    for (int j = 0; j < mn; ++j) {
                        const int ch = (int)pooled.tau[g];
                        const double want = 0.25 * (img[(ch * m + 2 * i) * m + 2 * j] + img[(ch * m + 2 * i + 1) * m + 2 * j] +
                                                    img[(ch * m + 2 * i) * m + 2 * j + 1] +
                                                    img[(ch * m + 2 * i + 1) * m + 2 * j + 1]);
                        worst = std::fmax(worst, std::fabs(y[(size_t)(g * pooled.rep) * mn * mn + i * mn + j] - want));
                    }
            std::vector<double> w1(c * c, 0.0);  // 1x1 conv: identity on the channels
            for (int f = 0; f < c; ++f) w1[f * c + f] = 1.0;
            fheconv::Packed conv2 = eng.convolve(pooled, c, 1, w1);
            auto z = eng.decrypt(conv2.shards[0]);
            for (int g = 0; g < c; ++g)
                for (int i = 0; i < mn * mn; ++i) {
                    const int ch = (int)pooled.tau[g];
                    // output block b holds channel b % c: compare channel ch at block ch
                    worst = std::fmax(worst, std::fabs(z[(size_t)ch * mn * mn + i] - y[(size_t)(g * pooled.rep) * mn * mn + i]));
                }
            auto ssum = eng.decrypt(eng.slot_sum(conv2.shards[0], 4096));
            double tot = 0;
            for (double v : z) tot += v;
            worst = std::fmax(worst, std::fabs(ssum[0] - tot) / 4096.0);
        }
        std::printf("engine_demo max|err| %.3g empty-batch-throws %d\n", worst, (int)threw);
        return (worst < 1e-6 && threw) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("engine_demo failed: %s\n", e.what());
        return 3;
    }
}
