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
        std::printf("engine_demo max|err| %.3g empty-batch-throws %d\n", worst, (int)threw);
        return (worst < 1e-6 && threw) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("engine_demo failed: %s\n", e.what());
        return 3;
    }
}
