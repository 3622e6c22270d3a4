// TEST HARNESS: runs the reference's own application pipelines
// (proj/src/apps.cpp: detail_enhance, tone_map, depth_upsample, colorize) on
// deterministic synthetic inputs and writes every output as raw doubles.
// Built twice by oracle/Makefile: against the reference's smoother.cpp
// (oracle/_ref/apps_ref) and against the GPU drop-in shim
// (oracle/_ref/apps_gpu); tests/test_shim.py compares the two.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "sgwls/apps.hpp"
#include "sgwls/synthetic.hpp"

using namespace sgwls;

static void dump(const std::string& dir, const char* name, const Image& im) {
    const std::string p = dir + "/" + name + ".bin";
    FILE* f = std::fopen(p.c_str(), "wb");
    if (!f) std::exit(3);
    const int hdr[3] = {im.width, im.height, im.channels};
    std::fwrite(hdr, sizeof(int), 3, f);
    std::fwrite(im.data.data(), sizeof(double), im.data.size(), f);
    std::fclose(f);
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string dir = argv[1];
    try {
        // detail enhancement, Frac weights (enhance_preset: lambda 900, r 1, tau 1).
        // (synthetic::step_scene is not used: its level rejection loop can never
        // succeed -- four levels cannot be pairwise >= 0.02 apart modulo 0.05.)
        Image blocks(96, 72, 1);
        for (int y = 0; y < 72; ++y)
            for (int x = 0; x < 96; ++x) blocks.at(y, x) = 0.3 + 0.2 * (x > 40) + 0.25 * (y > 30) + 0.05 * ((x + y) % 3);
        const Image scene = synthetic::add_gaussian_noise(blocks, 0.03, 8, true);
        SmoothConfig ecfg = enhance_preset();
        ecfg.iterations = 2;
        dump(dir, "detail_enhance", detail_enhance(scene, 2.0, ecfg));
        // tone mapping: three smooth() levels on log10 luminance (values < 0)
        Image hdr(80, 60, 3);
        for (int y = 0; y < hdr.height; ++y)
            for (int x = 0; x < hdr.width; ++x)
                for (int c = 0; c < 3; ++c)
                    hdr.at(y, x, c) = 0.01 + scene.at(y % scene.height, x % scene.width) * (1.0 + 40.0 * (x > 40)) *
                                                 (1.0 + 0.2 * c);
        dump(dir, "tone_map", tone_map(hdr, ToneMapParams{}));
        // depth upsampling (interpolate_sparse, r 4 / tau 4 exp weights, luma guidance)
        const auto ds = synthetic::depth_scene(96, 64, 11);
        Image low(24, 16, 1);
        for (int y = 0; y < low.height; ++y)
            for (int x = 0; x < low.width; ++x) low.at(y, x) = ds.depth.at(y * 4, x * 4);
        dump(dir, "depth_upsample", depth_upsample(low, ds.guidance_rgb, 4, upsample_preset(4)));
        // colorization (interpolate_sparse twice, r 4 / tau 2)
        Image gray = luminance(ds.guidance_rgb);
        Image scrib(96, 64, 3, 0.0), smask(96, 64, 1, 0.0);
        for (int y = 0; y < 64; y += 7)
            for (int x = 0; x < 96; x += 5) {
                smask.at(y, x) = 1.0;
                for (int c = 0; c < 3; ++c) scrib.at(y, x, c) = ds.guidance_rgb.at(y, x, c);
            }
        dump(dir, "colorize", colorize(gray, scrib, smask, colorize_preset()));
        // the reference's error path
        try {
            SmoothConfig bad;
            bad.tau = 7;
            smooth(scene, scene, bad);
        } catch (const Error& e) {
            std::printf("error: %s\n", e.what());
        }
        // several faults at once: the reference reports the field check first
        // (bad mask value) before smooth()'s guidance-size check
        try {
            SparseField f{Image(8, 6, 1, 0.0), Image(8, 6, 1, 0.0)};
            f.mask.at(2, 3) = 0.5;
            f.values.at(4, 4) = 1.0;
            interpolate_sparse(f, Image(9, 6, 1, 0.5), SmoothConfig{});
        } catch (const Error& e) {
            std::printf("error: %s\n", e.what());
        }
        // values off the mask before an invalid configuration
        try {
            SparseField f{Image(8, 6, 1, 0.0), Image(8, 6, 1, 0.0)};
            f.mask.at(0, 0) = 1.0;
            f.values.at(1, 1) = 2.0;
            SmoothConfig bad;
            bad.r = 0;
            interpolate_sparse(f, Image(8, 6, 1, 0.5), bad);
        } catch (const Error& e) {
            std::printf("error: %s\n", e.what());
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "failed: %s\n", e.what());
        return 1;
    }
    return 0;
}
