// TEST HARNESS: a plain C++ caller of the multi-GPU C ABI
// (sgwls_b200_smooth_multi, include/sgwls_b200.h) on a synthetic image: the
// slab filter over the device list given on the command line (e.g. "0" or
// "0,0,0": several slabs on one GPU) against the single-device call.
// Prints the max |difference| and exits non-zero on any error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "sgwls_b200.h"

int main(int argc, char** argv) {
    std::vector<int> devs;
    const std::string list = argc > 1 ? argv[1] : "0";
    for (size_t i = 0; i < list.size();) {
        size_t j = list.find(',', i);
        if (j == std::string::npos) j = list.size();
        devs.push_back(std::atoi(list.substr(i, j - i).c_str()));
        i = j + 1;
    }
    const int W = 211, H = 303;
    std::vector<float> t(W * H), g(W * H), a(W * H), b(W * H);
    unsigned s = 12345;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            s = s * 1664525u + 1013904223u;
            const float noise = ((s >> 8) & 0xffff) / 65536.0f - 0.5f;
            g[y * W + x] = 0.25f * ((x / 37 + y / 29) % 4) + 0.02f * noise;
            t[y * W + x] = g[y * W + x] + 0.05f * noise;
        }
    sgwls_b200_config cfg;
    sgwls_b200_config_default(&cfg);
    cfg.lambda = 400.0;
    cfg.r = 2;
    cfg.tau = 3;
    cfg.iterations = 4;
    cfg.weight_kind = SGWLS_B200_WEIGHT_EXP;
    cfg.sigma_r = 0.05;
    char err[512];
    if (sgwls_b200_smooth(t.data(), W, H, 1, g.data(), 1, &cfg, a.data(), err, sizeof err)) {
        std::fprintf(stderr, "smooth: %s\n", err);
        return 1;
    }
    if (sgwls_b200_smooth_multi(t.data(), W, H, 1, g.data(), 1, &cfg, devs.data(), (int)devs.size(), b.data(), err,
                                sizeof err)) {
        std::fprintf(stderr, "smooth_multi: %s\n", err);
        return 1;
    }
    double worst = 0.0;
    for (int i = 0; i < W * H; ++i) worst = std::fmax(worst, std::fabs((double)a[i] - b[i]));
    std::printf("ndev=%zu max|d| %.3g\n", devs.size(), worst);
    return worst <= 2e-6 ? 0 : 2;
}
