// apps_gpu.cpp -- drop-in replacement for the reference's proj/src/apps.cpp.
//
// Defines what proj/src/apps.cpp defines, with the signatures of
// proj/include/sgwls/apps.hpp (presets, detail_enhance, tone_map,
// depth_upsample, colorize), but every pipeline runs on the device through the
// C ABI (sgwls_b200_detail_enhance ... in include/sgwls_b200.h): one upload,
// the filter passes and the elementwise stages on device buffers, one download
// -- instead of one host round trip per smooth() call.  Link it together with
// smoother_gpu.cpp in place of apps.cpp + smoother.cpp.
// Errors keep the reference's sgwls::Error texts.
#include <string>
#include <vector>

#include "sgwls/apps.hpp"
#include "sgwls_b200.h"
#include "shim_convert.hpp"

namespace sgwls {

using namespace shim;

SmoothConfig enhance_preset() {
    sgwls_b200_config c;
    sgwls_b200_enhance_preset(&c);
    return from_c(c);
}

SmoothConfig tonemap_layer_preset(double lambda) {
    sgwls_b200_config c;
    sgwls_b200_tonemap_layer_preset(lambda, &c);
    return from_c(c);
}

SmoothConfig upsample_preset(int factor) {
    sgwls_b200_config c;
    char err[512];
    check(sgwls_b200_upsample_preset(factor, &c, err, sizeof err), err);
    return from_c(c);
}

SmoothConfig colorize_preset() {
    sgwls_b200_config c;
    sgwls_b200_colorize_preset(&c);
    return from_c(c);
}

Image detail_enhance(const Image& img, double boost, const SmoothConfig& cfg) {
    const std::vector<float> in = to_f32(img);
    std::vector<float> out(in.size());
    const sgwls_b200_config c = to_c(cfg);
    char err[512];
    check(sgwls_b200_detail_enhance(in.data(), img.width, img.height, img.channels, boost, &c, out.data(), err,
                                    sizeof err),
          err);
    return from_f32(out, img.width, img.height, img.channels);
}

Image tone_map(const Image& hdr, const ToneMapParams& params) {
    sgwls_b200_tonemap_params p;
    for (int i = 0; i < 3; ++i) {
        p.lambdas[i] = params.lambdas[i];
        p.detail_weights[i] = params.detail_weights[i];
    }
    p.target_log_range = params.target_log_range;
    p.smoothing = to_c(params.smoothing);
    const std::vector<float> in = to_f32(hdr);
    std::vector<float> out(in.size());
    char err[512];
    check(sgwls_b200_tone_map(in.data(), hdr.width, hdr.height, hdr.channels, &p, out.data(), err, sizeof err), err);
    return from_f32(out, hdr.width, hdr.height, hdr.channels);
}

Image depth_upsample(const Image& lowres_depth, const Image& guidance, int factor, const SmoothConfig& cfg) {
    const std::vector<float> low = to_f32(lowres_depth), g = to_f32(guidance);
    std::vector<float> out((std::size_t)guidance.width * guidance.height);
    const sgwls_b200_config c = to_c(cfg);
    char err[512];
    check(sgwls_b200_depth_upsample(low.data(), lowres_depth.width, lowres_depth.height, lowres_depth.channels,
                                    g.data(), guidance.width, guidance.height, guidance.channels, factor, &c,
                                    out.data(), err, sizeof err),
          err);
    return from_f32(out, guidance.width, guidance.height, 1);
}

Image colorize(const Image& gray, const Image& scribbles, const Image& scribble_mask, const SmoothConfig& cfg) {
    if (gray.channels != 1) throw Error("colorize: gray image must be single-channel");
    if (scribbles.channels != 3) throw Error("colorize: scribbles must be 3-channel");
    if (!gray.same_size(scribbles) || !gray.same_size(scribble_mask)) throw Error("colorize: image sizes differ");
    if (scribble_mask.channels != 1) throw Error("interpolate_sparse: mask must be single-channel");
    const std::vector<float> g = to_f32(gray), s = to_f32(scribbles), m = to_f32(scribble_mask);
    std::vector<float> out((std::size_t)gray.width * gray.height * 3);
    const sgwls_b200_config c = to_c(cfg);
    char err[512];
    check(sgwls_b200_colorize(g.data(), 1, s.data(), 3, m.data(), gray.width, gray.height, &c, out.data(), err,
                              sizeof err),
          err);
    return from_f32(out, gray.width, gray.height, 3);
}

}  // namespace sgwls
