// shim_convert.hpp -- sgwls::SmoothConfig / sgwls::Image <-> C ABI conversions
// shared by the drop-in shims (smoother_gpu.cpp, apps_gpu.cpp).
#pragma once

#include <vector>

#include "sgwls/error.hpp"
#include "sgwls/image.hpp"
#include "sgwls/smoother.hpp"
#include "sgwls_b200.h"

namespace sgwls {
namespace shim {

inline sgwls_b200_config to_c(const SmoothConfig& c) {
    sgwls_b200_config o;
    sgwls_b200_config_default(&o);
    o.lambda = c.lambda;
    o.r = c.r;
    o.tau = c.tau;
    o.iterations = c.iterations;
    o.first_axis = c.first_axis == Axis::Column ? SGWLS_B200_AXIS_COLUMN : SGWLS_B200_AXIS_ROW;
    o.threads = c.threads;
    o.weight_kind = c.weight.kind == WeightKind::Exp ? SGWLS_B200_WEIGHT_EXP : SGWLS_B200_WEIGHT_FRAC;
    o.alpha_s = c.weight.alpha_s;
    o.alpha_r = c.weight.alpha_r;
    o.sigma_s = c.weight.sigma_s;
    o.sigma_r = c.weight.sigma_r;
    o.epsilon = c.weight.epsilon;
    o.guidance_scale = c.weight.guidance_scale;
    return o;
}

inline SmoothConfig from_c(const sgwls_b200_config& o) {
    SmoothConfig c;
    c.lambda = o.lambda;
    c.r = o.r;
    c.tau = o.tau;
    c.iterations = o.iterations;
    c.first_axis = o.first_axis == SGWLS_B200_AXIS_COLUMN ? Axis::Column : Axis::Row;
    c.threads = o.threads;
    c.weight.kind = o.weight_kind == SGWLS_B200_WEIGHT_EXP ? WeightKind::Exp : WeightKind::Frac;
    c.weight.alpha_s = o.alpha_s;
    c.weight.alpha_r = o.alpha_r;
    c.weight.sigma_s = o.sigma_s;
    c.weight.sigma_r = o.sigma_r;
    c.weight.epsilon = o.epsilon;
    c.weight.guidance_scale = o.guidance_scale;
    return c;
}

inline std::vector<float> to_f32(const Image& im) { return std::vector<float>(im.data.begin(), im.data.end()); }

inline Image from_f32(const std::vector<float>& v, int w, int h, int c) {
    Image out(w, h, c);
    for (std::size_t i = 0; i < v.size(); ++i) out.data[i] = v[i];
    return out;
}

inline void check(int rc, const char* err) {
    if (rc != SGWLS_B200_OK) throw Error(err);
}

}  // namespace shim
}  // namespace sgwls
