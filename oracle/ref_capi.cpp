// TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference library, compiled
// directly from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libsgwls_ref.so.  It is the "reference" CPU arm: it validates
// the C restatement (oracle/sgwls_oracle.c), generates the golden fixtures in
// tests/golden/, and is what bench.py --impl reference times.  fp32 inputs
// are promoted to double exactly as SURVEY.md §8(c) prescribes.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sgwls/apps.hpp"
#include "sgwls/banded.hpp"
#include "sgwls/smoother.hpp"
#include "sgwls/weights.hpp"
#include "sgwls_oracle.h"

namespace {

sgwls::SmoothConfig to_cfg(const oracle_config* c) {
    sgwls::SmoothConfig cfg;
    cfg.lambda = c->lambda;
    cfg.r = c->r;
    cfg.tau = c->tau;
    cfg.iterations = c->iterations;
    cfg.first_axis = c->first_axis == 0 ? sgwls::Axis::Column : sgwls::Axis::Row;
    cfg.threads = c->threads;
    cfg.weight.kind = c->kind == 0 ? sgwls::WeightKind::Frac : sgwls::WeightKind::Exp;
    cfg.weight.alpha_s = c->alpha_s;
    cfg.weight.alpha_r = c->alpha_r;
    cfg.weight.sigma_s = c->sigma_s;
    cfg.weight.sigma_r = c->sigma_r;
    cfg.weight.epsilon = c->epsilon;
    cfg.weight.guidance_scale = c->guidance_scale;
    return cfg;
}

sgwls::Image to_img(const float* p, int w, int h, int c) {
    sgwls::Image im(w, h, c);
    for (std::size_t i = 0; i < im.data.size(); ++i) im.data[i] = p[i];
    return im;
}

void put_err(char* err, std::size_t errlen, const char* msg) {
    if (err && errlen) {
        std::strncpy(err, msg, errlen - 1);
        err[errlen - 1] = '\0';
    }
}

}  // namespace

extern "C" {

int ref_smooth_f32(const float* target, int width, int height, int channels, const float* guidance,
                   int guidance_channels, const oracle_config* c, double* out, char* err, std::size_t errlen) {
    try {
        const sgwls::Image t = to_img(target, width, height, channels);
        const sgwls::Image g = to_img(guidance, width, height, guidance_channels);
        const sgwls::Image o = sgwls::smooth(t, g, to_cfg(c));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

// The reference's application pipelines (proj/src/apps.cpp), fp32 inputs
// promoted to double, double outputs: the parity anchor of the device
// pipelines (tests/test_apps.py).
int ref_detail_enhance_f32(const float* img, int width, int height, int channels, double boost,
                           const oracle_config* c, double* out, char* err, std::size_t errlen) {
    try {
        const sgwls::Image o = sgwls::detail_enhance(to_img(img, width, height, channels), boost, to_cfg(c));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_tone_map_f32(const float* hdr, int width, int height, int channels, const double* lambdas,
                     const double* detail_weights, double target_log_range, const oracle_config* smoothing,
                     double* out, char* err, std::size_t errlen) {
    try {
        sgwls::ToneMapParams p;
        for (int i = 0; i < 3; ++i) {
            p.lambdas[i] = lambdas[i];
            p.detail_weights[i] = detail_weights[i];
        }
        p.target_log_range = target_log_range;
        p.smoothing = to_cfg(smoothing);
        const sgwls::Image o = sgwls::tone_map(to_img(hdr, width, height, channels), p);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_depth_upsample_f32(const float* low, int lw, int lh, int lc, const float* guidance, int width, int height,
                           int gc, int factor, const oracle_config* c, double* out, char* err, std::size_t errlen) {
    try {
        const sgwls::Image o = sgwls::depth_upsample(to_img(low, lw, lh, lc), to_img(guidance, width, height, gc),
                                                     factor, to_cfg(c));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_colorize_f32(const float* gray, const float* scribbles, const float* mask, int width, int height,
                     const oracle_config* c, double* out, char* err, std::size_t errlen) {
    try {
        const sgwls::Image o = sgwls::colorize(to_img(gray, width, height, 1), to_img(scribbles, width, height, 3),
                                               to_img(mask, width, height, 1), to_cfg(c));
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_interpolate_sparse_f32(const float* values, int width, int height, int channels, const float* mask,
                               const float* guidance, int guidance_channels, const oracle_config* c,
                               double* out, double* undefined_mask, char* err, std::size_t errlen) {
    try {
        sgwls::SparseField f{to_img(values, width, height, channels), to_img(mask, width, height, 1)};
        const sgwls::Image g = to_img(guidance, width, height, guidance_channels);
        sgwls::Image und;
        const sgwls::Image o = sgwls::interpolate_sparse(f, g, to_cfg(c), undefined_mask ? &und : nullptr);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
        if (undefined_mask) std::memcpy(undefined_mask, und.data.data(), sizeof(double) * und.data.size());
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 1;
    }
}

int ref_band_centers(int extent, int r, int tau, int* out, int cap) {
    try {
        const auto v = sgwls::band_centers(extent, r, tau);
        for (std::size_t i = 0; i < v.size() && static_cast<int>(i) < cap; ++i) out[i] = v[i];
        return static_cast<int>(v.size());
    } catch (const std::exception&) {
        return -1;
    }
}

// Assemble + factor + solve one band from raw edge weights w[k*r+t-1].
int ref_solve_band(int n, int r, const double* w, double lambda, const double* rhs, double* u, double* alpha,
                   double* beta, double* gamma) {
    try {
        sgwls::WeightTable wt;
        wt.n = n;
        wt.r = r;
        wt.w.assign(w, w + static_cast<std::size_t>(n) * r);
        const sgwls::BandedSystem sys =
            sgwls::assemble_subsystem(std::vector<double>(rhs, rhs + n), wt, lambda, r);
        const sgwls::BandedFactors f = sgwls::rband_lu_factorize(sys);
        const auto y = sgwls::forward_substitute(f, sys.rhs);
        const auto x = sgwls::backward_substitute(f, y);
        std::memcpy(u, x.data(), sizeof(double) * n);
        if (alpha) std::memcpy(alpha, f.alpha.data(), sizeof(double) * n);
        if (beta) std::memcpy(beta, f.beta.data(), sizeof(double) * f.beta.size());
        if (gamma) std::memcpy(gamma, f.gamma.data(), sizeof(double) * f.gamma.size());
        return -1;
    } catch (const std::exception&) {
        return 0;
    }
}

int ref_band_layout(int height, int width, int center, int r, int axis, int* rows, int* cols) {
    const sgwls::Band band =
        sgwls::band_layout(height, width, center, r, axis == 0 ? sgwls::Axis::Column : sgwls::Axis::Row);
    for (int i = 0; i < band.size(); ++i) {
        rows[i] = band.coords[i].row;
        cols[i] = band.coords[i].col;
    }
    return band.size();
}

int ref_edge_weights(const double* guidance, int width, int height, int gch, int center, int r, int axis,
                     const oracle_config* c, double* w) {
    sgwls::Image g(width, height, gch);
    std::memcpy(g.data.data(), guidance, sizeof(double) * g.data.size());
    const sgwls::Band band =
        sgwls::band_layout(height, width, center, r, axis == 0 ? sgwls::Axis::Column : sgwls::Axis::Row);
    const sgwls::WeightTable t = sgwls::edge_weights_along_band(g, band, r, to_cfg(c).weight);
    std::memcpy(w, t.w.data(), sizeof(double) * t.w.size());
    return band.size();
}

}  // extern "C"
