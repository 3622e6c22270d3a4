// smoother_gpu.cpp -- drop-in replacement for the reference's proj/src/smoother.cpp.
//
// Defines exactly what proj/src/smoother.cpp defines, with the same signatures
// (proj/include/sgwls/smoother.hpp:12-42):
//
//   void SmoothConfig::validate() const                 (proj/src/smoother.cpp:103-111)
//   Image smooth(const Image&, const Image&, const SmoothConfig&)   (:113-125)
//   Image interpolate_sparse(const SparseField&, const Image&,
//                            const SmoothConfig&, Image*)          (:127-163)
//
// but runs the filter on the GPU through the C ABI (include/sgwls_b200.h).
// Build it in place of smoother.cpp and link
// libsgwls_b200.so: the reference's applications (proj/src/apps.cpp) and CLI
// (proj/tools/sgwls_main.cpp) then run unchanged on the B200.  Errors keep the
// reference's sgwls::Error texts; there is no CPU fallback (a missing device
// surfaces as sgwls::Error from the C ABI).
#include <string>
#include <vector>

#include "sgwls/smoother.hpp"
#include "sgwls_b200.h"
#include "shim_convert.hpp"

namespace sgwls {

namespace {

sgwls_b200_config to_c(const SmoothConfig& c) {
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

std::vector<float> to_f32(const Image& im) { return std::vector<float>(im.data.begin(), im.data.end()); }

void check(int rc, const char* err) {
    if (rc != SGWLS_B200_OK) throw Error(err);
}

}  // namespace

void SmoothConfig::validate() const {
    char err[512];
    const sgwls_b200_config c = to_c(*this);
    check(sgwls_b200_validate(&c, err, sizeof err), err);
}

Image smooth(const Image& target, const Image& guidance, const SmoothConfig& cfg) {
    cfg.validate();
    if (target.empty()) throw Error("smooth: empty target");
    if (!target.same_size(guidance)) throw Error("smooth: target and guidance dimensions differ");
    const std::vector<float> t = to_f32(target), g = to_f32(guidance);
    std::vector<float> o(t.size());
    const sgwls_b200_config c = to_c(cfg);
    char err[512];
    // ndev = 0: the devices listed in SGWLS_B200_DEVICES (one image in row slabs
    // across them), else device 0 -- the reference's callers reach multi-GPU
    // without a code change, like its own cfg.threads knob
    check(sgwls_b200_smooth_multi(t.data(), target.width, target.height, target.channels, g.data(),
                                  guidance.channels, &c, nullptr, 0, o.data(), err, sizeof err),
          err);
    Image out(target.width, target.height, target.channels);
    for (std::size_t i = 0; i < o.size(); ++i) out.data[i] = o[i];
    return out;
}

Image interpolate_sparse(const SparseField& field, const Image& guidance, const SmoothConfig& cfg,
                         Image* undefined_mask) {
    // checks in the reference's order (proj/src/smoother.cpp:129-147): the field
    // (first offending pixel in scan order), then smooth()'s config / empty /
    // size checks -- so an input with several faults gets the reference's text
    if (field.mask.channels != 1) throw Error("interpolate_sparse: mask must be single-channel");
    if (!field.values.same_size(field.mask)) throw Error("interpolate_sparse: values/mask size mismatch");
    bool any = false;
    for (int y = 0; y < field.mask.height; ++y)
        for (int x = 0; x < field.mask.width; ++x) {
            const double mv = field.mask.at(y, x);
            if (mv != 0.0 && mv != 1.0) throw Error("interpolate_sparse: mask must be 0/1");
            if (mv == 1.0) any = true;
            if (mv == 0.0)
                for (int c = 0; c < field.values.channels; ++c)
                    if (field.values.at(y, x, c) != 0.0) throw Error("interpolate_sparse: values nonzero outside mask");
        }
    if (!any) throw Error("interpolate_sparse: empty mask");
    cfg.validate();
    if (field.values.empty()) throw Error("smooth: empty target");
    if (!field.values.same_size(guidance)) throw Error("smooth: target and guidance dimensions differ");
    const std::vector<float> v = to_f32(field.values), m = to_f32(field.mask), g = to_f32(guidance);
    std::vector<float> o(v.size()), und(m.size());
    const sgwls_b200_config c = to_c(cfg);
    char err[512];
    check(sgwls_b200_interpolate_sparse(v.data(), m.data(), field.values.width, field.values.height,
                                        field.values.channels, g.data(), guidance.channels, &c, o.data(),
                                        und.data(), err, sizeof err),
          err);
    Image out(field.values.width, field.values.height, field.values.channels);
    for (std::size_t i = 0; i < o.size(); ++i) out.data[i] = o[i];
    if (undefined_mask) {
        *undefined_mask = Image(field.values.width, field.values.height, 1, 0.0);
        for (std::size_t i = 0; i < und.size(); ++i) undefined_mask->data[i] = und[i];
    }
    return out;
}

}  // namespace sgwls
