// sgwls_b200 -- command-line front end of the B200 SG-WLS filter.
//
// Drop-in for the reference tool proj/tools/sgwls_main.cpp (which needs the absent
// CLI11): same subcommands (smooth, enhance, tonemap, upsample, colorize, bench,
// selftest), same option names and preset/override rules (make_config,
// proj/tools/sgwls_main.cpp:83-117), same stderr echo line (:119-128), same bench
// CSV `op,M,N,r,tau,T,seconds` with the median of --reps (:145-192), same exit
// codes (2 = usage error, 1 = "sgwls: error: ..." at run time).  Everything runs
// on the GPU through the C ABI (include/sgwls_b200.h): plain C++, no reference
// headers, no CPU fallback.  Differences, all stated by the tool itself:
//   * `bench --op wlsref` (the reference's 2-D CG oracle) is not part of the
//     filter path and is refused;
//   * bench images come from a built-in seeded block scene (the reference's
//     synthetic::step_scene is not on the path either);
//   * `--devices 0,1,..` runs `smooth` as row slabs over several GPUs
//     (sgwls_b200_smooth_multi); `--threads` is validated and echoed only;
//   * selftest runs GPU-side invariants (constant invariance, lambda = 0
//     identity, run-to-run determinism, single-row = batch, codec round trip).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgwls_b200.h"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RunError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- arguments

// One parsed command line: named options (last occurrence wins) and positionals.
class Args {
public:
    Args(int argc, char** argv, int first, const std::vector<std::string>& known) {
        for (int i = first; i < argc; ++i) {
            const std::string a = argv[i];
            if (a.rfind("--", 0) != 0) {
                positional_.push_back(a);
                continue;
            }
            std::string name = a, value;
            const std::size_t eq = a.find('=');
            bool have = false;
            if (eq != std::string::npos) {
                name = a.substr(0, eq);
                value = a.substr(eq + 1);
                have = true;
            }
            if (std::find(known.begin(), known.end(), name) == known.end())
                throw UsageError("unknown option " + name);
            if (!have) {
                if (i + 1 >= argc) throw UsageError(name + ": value expected");
                value = argv[++i];
            }
            named_[name] = value;
        }
    }
    bool has(const std::string& n) const { return named_.count(n) != 0; }
    const std::string& str(const std::string& n) const { return named_.at(n); }
    double num(const std::string& n) const {
        char* end = nullptr;
        const double v = std::strtod(str(n).c_str(), &end);
        if (end == str(n).c_str() || *end) throw UsageError(n + ": number expected, got '" + str(n) + "'");
        return v;
    }
    int integer(const std::string& n) const {
        char* end = nullptr;
        const long v = std::strtol(str(n).c_str(), &end, 10);
        if (end == str(n).c_str() || *end) throw UsageError(n + ": integer expected, got '" + str(n) + "'");
        return static_cast<int>(v);
    }
    std::vector<int> int_list(const std::string& n) const {
        std::vector<int> out;
        const std::string& s = str(n);
        for (std::size_t i = 0; i <= s.size();) {
            std::size_t j = s.find(',', i);
            if (j == std::string::npos) j = s.size();
            const std::string item = s.substr(i, j - i);
            char* end = nullptr;
            const long v = std::strtol(item.c_str(), &end, 10);
            if (item.empty() || *end) throw UsageError(n + ": comma-separated integers expected, got '" + s + "'");
            out.push_back(static_cast<int>(v));
            i = j + 1;
        }
        return out;
    }
    const std::vector<std::string>& positional() const { return positional_; }
    void want_positionals(std::size_t n, const char* what) const {
        if (positional_.size() != n) throw UsageError(std::string("expected arguments: ") + what);
    }

private:
    std::map<std::string, std::string> named_;
    std::vector<std::string> positional_;
};

const std::vector<std::string> kSmoothOpts = {"--lambda", "--iters", "--weights", "--as",        "--ar",
                                              "--ss",     "--sr",    "--eps",     "--gscale",    "--first-axis",
                                              "--threads", "--devices"};

std::vector<std::string> with(std::vector<std::string> base, std::initializer_list<const char*> more) {
    for (const char* m : more) base.emplace_back(m);
    return base;
}

// ---------------------------------------------------------------- configuration

void check(int rc, const char* err) {
    if (rc != SGWLS_B200_OK) throw RunError(err);
}

sgwls_b200_config preset_named(const std::string& name) {
    sgwls_b200_config c;
    char err[256];
    if (name == "enhance") {
        sgwls_b200_enhance_preset(&c);
    } else if (name == "tonemap") {
        sgwls_b200_tonemap_layer_preset(5.0, &c);
    } else if (name == "upsample2x" || name == "upsample4x" || name == "upsample8x") {
        check(sgwls_b200_upsample_preset(name[8] - '0', &c, err, sizeof err), err);
    } else if (name == "colorize") {
        sgwls_b200_colorize_preset(&c);
    } else {
        throw RunError("unknown preset '" + name + "'");
    }
    return c;
}

int threads_from(const Args& a) {
    if (a.has("--threads") && a.integer("--threads") > 0) return a.integer("--threads");
    if (const char* env = std::getenv("SGWLS_THREADS")) {
        const int v = std::atoi(env);
        if (v > 0) return v;
    }
    return 1;
}

// Preset first, then every flag the user actually gave; without a preset the
// weight kind and the first axis take the tool's defaults (frac / col), and the
// guidance scale follows the kind (1 for frac, 255 for exp) unless --gscale is given.
sgwls_b200_config config_from(const Args& a, const std::string& forced_preset, bool shape = true) {
    sgwls_b200_config c;
    sgwls_b200_config_default(&c);
    std::string preset = forced_preset;
    if (preset.empty() && a.has("--preset")) preset = a.str("--preset");
    if (!preset.empty()) c = preset_named(preset);

    if (a.has("--weights") || preset.empty()) {
        const std::string w = a.has("--weights") ? a.str("--weights") : "frac";
        if (w == "frac")
            c.weight_kind = SGWLS_B200_WEIGHT_FRAC;
        else if (w == "exp")
            c.weight_kind = SGWLS_B200_WEIGHT_EXP;
        else
            throw RunError("--weights must be 'frac' or 'exp'");
        if (!a.has("--gscale")) c.guidance_scale = c.weight_kind == SGWLS_B200_WEIGHT_FRAC ? 1.0 : 255.0;
    }
    if (a.has("--lambda")) c.lambda = a.num("--lambda");
    if (shape && a.has("--r")) c.r = a.integer("--r");
    if (shape && a.has("--tau")) c.tau = a.integer("--tau");
    if (a.has("--iters")) c.iterations = a.integer("--iters");
    if (a.has("--as")) c.alpha_s = a.num("--as");
    if (a.has("--ar")) c.alpha_r = a.num("--ar");
    if (a.has("--ss")) c.sigma_s = a.num("--ss");
    if (a.has("--sr")) c.sigma_r = a.num("--sr");
    if (a.has("--eps")) c.epsilon = a.num("--eps");
    if (a.has("--gscale")) c.guidance_scale = a.num("--gscale");
    if (a.has("--first-axis") || preset.empty()) {
        const std::string ax = a.has("--first-axis") ? a.str("--first-axis") : "col";
        if (ax == "col")
            c.first_axis = SGWLS_B200_AXIS_COLUMN;
        else if (ax == "row")
            c.first_axis = SGWLS_B200_AXIS_ROW;
        else
            throw RunError("--first-axis must be 'col' or 'row'");
    }
    c.threads = threads_from(a);
    return c;
}

void announce(const char* op, const sgwls_b200_config& c) {
    std::fprintf(stderr,
                 "sgwls: %s lambda=%g r=%d tau=%d iters=%d weights=%s alpha_s=%g alpha_r=%g "
                 "sigma_s=%g sigma_r=%g eps=%g gscale=%g first_axis=%s threads=%d\n",
                 op, c.lambda, c.r, c.tau, c.iterations, c.weight_kind == SGWLS_B200_WEIGHT_FRAC ? "frac" : "exp",
                 c.alpha_s, c.alpha_r, c.sigma_s, c.sigma_r, c.epsilon, c.guidance_scale,
                 c.first_axis == SGWLS_B200_AXIS_COLUMN ? "col" : "row", c.threads);
}

// ---------------------------------------------------------------- images

struct Picture {
    int w = 0, h = 0, c = 0;
    std::vector<float> px;
    std::size_t pixels() const { return static_cast<std::size_t>(w) * h; }
};

Picture load(const std::string& path) {
    float* data = nullptr;
    Picture p;
    char err[512];
    check(sgwls_b200_image_read(path.c_str(), &data, &p.w, &p.h, &p.c, err, sizeof err), err);
    p.px.assign(data, data + p.pixels() * p.c);
    sgwls_b200_image_free(data);
    return p;
}

void store(const Picture& p, const std::string& path) {
    char err[512];
    check(sgwls_b200_image_write(path.c_str(), p.px.empty() ? nullptr : p.px.data(), p.w, p.h, p.c, err, sizeof err),
          err);
}

Picture like(const Picture& p, int channels) {
    Picture o;
    o.w = p.w;
    o.h = p.h;
    o.c = channels;
    o.px.resize(o.pixels() * channels);
    return o;
}

// ---------------------------------------------------------------- subcommands

int cmd_smooth(const Args& a) {
    a.want_positionals(2, "smooth <input> <output> [--guidance <image>] [options]");
    const sgwls_b200_config cfg = config_from(a, "");
    announce("smooth", cfg);
    const Picture in = load(a.positional()[0]);
    const Picture guide = a.has("--guidance") ? load(a.str("--guidance")) : in;
    Picture out = like(in, in.c);
    char err[512];
    // the reference checks the configuration before the sizes (proj/src/smoother.cpp:114-116)
    check(sgwls_b200_validate(&cfg, err, sizeof err), err);
    if (guide.w != in.w || guide.h != in.h) throw RunError("smooth: target and guidance dimensions differ");
    if (a.has("--devices")) {
        const std::vector<int> devs = a.int_list("--devices");
        check(sgwls_b200_smooth_multi(in.px.data(), in.w, in.h, in.c, guide.px.data(), guide.c, &cfg, devs.data(),
                                      static_cast<int>(devs.size()), out.px.data(), err, sizeof err),
              err);
    } else {
        check(sgwls_b200_smooth(in.px.data(), in.w, in.h, in.c, guide.px.data(), guide.c, &cfg, out.px.data(), err,
                                sizeof err),
              err);
    }
    store(out, a.positional()[1]);
    return 0;
}

int cmd_enhance(const Args& a) {
    a.want_positionals(2, "enhance <input> <output> [--boost g] [options]");
    const sgwls_b200_config cfg = config_from(a, a.has("--preset") ? "" : "enhance");
    announce("enhance", cfg);
    const double boost = a.has("--boost") ? a.num("--boost") : 3.0;
    const Picture in = load(a.positional()[0]);
    Picture out = like(in, in.c);
    char err[512];
    check(sgwls_b200_detail_enhance(in.px.data(), in.w, in.h, in.c, boost, &cfg, out.px.data(), err, sizeof err), err);
    store(out, a.positional()[1]);
    return 0;
}

int cmd_tonemap(const Args& a) {
    a.want_positionals(2, "tonemap <input.pfm> <output> [--range d] [--l1..3 v] [--dw1..3 v] [options]");
    sgwls_b200_tonemap_params p;
    sgwls_b200_tonemap_params_default(&p);
    if (a.has("--range")) p.target_log_range = a.num("--range");
    const char* ls[3] = {"--l1", "--l2", "--l3"};
    const char* ws[3] = {"--dw1", "--dw2", "--dw3"};
    for (int i = 0; i < 3; ++i) {
        if (a.has(ls[i])) p.lambdas[i] = a.num(ls[i]);
        if (a.has(ws[i])) p.detail_weights[i] = a.num(ws[i]);
    }
    p.smoothing = config_from(a, "tonemap");
    announce("tonemap", p.smoothing);
    const Picture in = load(a.positional()[0]);
    Picture out = like(in, in.c);
    char err[512];
    check(sgwls_b200_tone_map(in.px.data(), in.w, in.h, in.c, &p, out.px.data(), err, sizeof err), err);
    store(out, a.positional()[1]);
    return 0;
}

int cmd_upsample(const Args& a) {
    a.want_positionals(3, "upsample <depth> <guidance> <output> [--factor f] [options]");
    const int factor = a.has("--factor") ? a.integer("--factor") : 4;
    std::string preset;
    if (!a.has("--preset") && (factor == 2 || factor == 4 || factor == 8))
        preset = "upsample" + std::to_string(factor) + "x";
    const sgwls_b200_config cfg = config_from(a, preset);
    announce("upsample", cfg);
    const Picture depth = load(a.positional()[0]);
    const Picture guide = load(a.positional()[1]);
    Picture out = like(guide, 1);
    char err[512];
    check(sgwls_b200_depth_upsample(depth.px.data(), depth.w, depth.h, depth.c, guide.px.data(), guide.w, guide.h,
                                    guide.c, factor, &cfg, out.px.data(), err, sizeof err),
          err);
    store(out, a.positional()[2]);
    return 0;
}

int cmd_colorize(const Args& a) {
    a.want_positionals(3, "colorize <gray> <scribbles> <output> [--mask <pgm>] [--scribble-threshold t] [options]");
    const sgwls_b200_config cfg = config_from(a, a.has("--preset") ? "" : "colorize");
    announce("colorize", cfg);
    const double threshold = a.has("--scribble-threshold") ? a.num("--scribble-threshold") : 2.0 / 255.0;
    const Picture gray = load(a.positional()[0]);
    const Picture scrib = load(a.positional()[1]);
    Picture mask;
    if (a.has("--mask")) {
        mask = load(a.str("--mask"));
        for (float& v : mask.px) v = v >= 0.5f ? 1.0f : 0.0f;
    } else {
        // any scribble pixel with visible chroma (BT.601 U, V about zero) counts
        if (scrib.c != 3) throw RunError("rgb_to_yuv needs a 3-channel image");
        mask = like(gray, 1);
        for (int y = 0; y < gray.h; ++y)
            for (int x = 0; x < gray.w; ++x) {
                if (y >= scrib.h || x >= scrib.w) continue;
                const float* s = &scrib.px[(static_cast<std::size_t>(y) * scrib.w + x) * 3];
                const double luma = 0.299 * s[0] + 0.587 * s[1] + 0.114 * s[2];
                const double u = (s[2] - luma) / 1.772, v = (s[0] - luma) / 1.402;
                mask.px[static_cast<std::size_t>(y) * gray.w + x] =
                    (std::fabs(u) > threshold || std::fabs(v) > threshold) ? 1.0f : 0.0f;
            }
    }
    if (scrib.w != gray.w || scrib.h != gray.h || mask.w != gray.w || mask.h != gray.h)
        throw RunError("colorize: image sizes differ");
    if (mask.c != 1) throw RunError("interpolate_sparse: mask must be single-channel");
    Picture out = like(gray, 3);
    char err[512];
    check(sgwls_b200_colorize(gray.px.data(), gray.c, scrib.px.data(), scrib.c, mask.px.data(), gray.w, gray.h, &cfg,
                              out.px.data(), err, sizeof err),
          err);
    store(out, a.positional()[2]);
    return 0;
}

// Seeded block scene for the timing table: 32-pixel blocks at four well-separated
// levels as guidance, the target adds clipped Gaussian-like noise (sum of uniforms).
struct Lcg {
    unsigned long long s;
    double next() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return static_cast<double>(s >> 11) / 9007199254740992.0;
    }
};

void bench_scene(int n, std::vector<float>& guide, std::vector<float>& target) {
    Lcg lv{42}, nz{43};
    const int cells = (n + 31) / 32;
    std::vector<float> level(static_cast<std::size_t>(cells) * cells);
    for (float& l : level) l = 0.15f + 0.23f * static_cast<float>(static_cast<int>(lv.next() * 4.0));
    guide.resize(static_cast<std::size_t>(n) * n);
    target.resize(guide.size());
    for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
            const float g = level[static_cast<std::size_t>(y / 32) * cells + x / 32];
            const double noise = (nz.next() + nz.next() + nz.next() + nz.next() - 2.0) * 0.0866;  // sigma ~ 0.05
            guide[static_cast<std::size_t>(y) * n + x] = g;
            target[static_cast<std::size_t>(y) * n + x] = static_cast<float>(std::min(1.0, std::max(0.0, g + noise)));
        }
}

int cmd_bench(const Args& a) {
    const std::string op = a.has("--op") ? a.str("--op") : "smooth";
    std::vector<int> sizes{256}, rs{1}, taus{1};
    if (a.has("--sizes")) sizes = a.int_list("--sizes");
    if (a.has("--size")) sizes = a.int_list("--size");
    if (a.has("--r")) rs = a.int_list("--r");
    if (a.has("--tau")) taus = a.int_list("--tau");
    const int reps = a.has("--reps") ? a.integer("--reps") : 3;
    if (reps < 1) throw UsageError("--reps must be >= 1");
    // --r / --tau are lists here: the shared flags leave the preset's (or default) shape alone
    const sgwls_b200_config base = config_from(a, "", false);
    announce("bench", base);
    if (op == "wlsref") throw RunError("bench --op wlsref: the 2-D WLS conjugate-gradient oracle is not part of the GPU filter path");
    if (op != "smooth") throw RunError("bench --op must be 'smooth'");
    std::printf("op,M,N,r,tau,T,seconds\n");
    for (int size : sizes) {
        std::vector<float> guide, target;
        bench_scene(size, guide, target);
        std::vector<float> out(target.size());
        for (int r : rs)
            for (int tau : taus) {
                sgwls_b200_config cfg = base;
                cfg.r = r;
                cfg.tau = tau;
                if (tau > 2 * r + 1) {
                    std::fprintf(stderr, "sgwls: bench: skipping r=%d tau=%d (stride too large)\n", r, tau);
                    continue;
                }
                char err[512];
                check(sgwls_b200_validate(&cfg, err, sizeof err), err);
                std::vector<double> t;
                for (int rep = 0; rep < reps; ++rep) {
                    const auto t0 = std::chrono::steady_clock::now();
                    check(sgwls_b200_smooth(target.data(), size, size, 1, guide.data(), 1, &cfg, out.data(), err,
                                            sizeof err),
                          err);
                    t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
                }
                std::sort(t.begin(), t.end());
                std::printf("smooth,%d,%d,%d,%d,%d,%.6f\n", size, size, r, tau, cfg.iterations, t[t.size() / 2]);
                std::fflush(stdout);
            }
    }
    return 0;
}

int cmd_selftest(const Args&) {
    int failures = 0;
    auto report = [&](bool ok, const char* name, const std::string& detail) {
        if (ok) {
            std::printf("ok %s\n", name);
        } else {
            ++failures;
            std::printf("FAIL %s%s\n", name, detail.empty() ? "" : (": " + detail).c_str());
        }
    };
    char err[512];
    std::vector<float> guide, target;
    bench_scene(96, guide, target);
    const int n = 96;
    std::vector<float> a(target.size()), b(target.size());
    sgwls_b200_config cfg;

    {  // a constant image stays constant under every preset (unit row sums)
        double worst = 0.0;
        const std::vector<float> flat(target.size(), 0.37f);
        for (const char* name : {"enhance", "colorize", "upsample4x"}) {
            cfg = preset_named(name);
            cfg.iterations = 2;
            check(sgwls_b200_smooth(flat.data(), n, n, 1, guide.data(), 1, &cfg, a.data(), err, sizeof err), err);
            for (float v : a) worst = std::max(worst, static_cast<double>(std::fabs(v - 0.37f)));
        }
        report(worst <= 2e-6, "constant-invariance", std::to_string(worst));
    }
    {  // lambda = 0 is the identity
        sgwls_b200_config_default(&cfg);
        cfg.lambda = 0.0;
        cfg.r = 2;
        cfg.tau = 2;
        check(sgwls_b200_smooth(target.data(), n, n, 1, guide.data(), 1, &cfg, a.data(), err, sizeof err), err);
        double worst = 0.0;
        for (std::size_t i = 0; i < a.size(); ++i) worst = std::max(worst, static_cast<double>(std::fabs(a[i] - target[i])));
        report(worst <= 1e-6, "lambda-zero-identity", std::to_string(worst));
    }
    {  // two runs agree bit for bit; a batch of two equals two single calls
        cfg = preset_named("colorize");
        check(sgwls_b200_smooth(target.data(), n, n, 1, guide.data(), 1, &cfg, a.data(), err, sizeof err), err);
        check(sgwls_b200_smooth(target.data(), n, n, 1, guide.data(), 1, &cfg, b.data(), err, sizeof err), err);
        report(std::memcmp(a.data(), b.data(), a.size() * 4) == 0, "determinism", "");
        std::vector<float> t2(target), g2(guide), o2(2 * target.size());
        t2.insert(t2.end(), target.begin(), target.end());
        g2.insert(g2.end(), guide.begin(), guide.end());
        check(sgwls_b200_smooth_batch(t2.data(), g2.data(), 2, n, n, 1, 1, &cfg, o2.data(), err, sizeof err), err);
        const bool same = std::memcmp(o2.data(), a.data(), a.size() * 4) == 0 &&
                          std::memcmp(o2.data() + a.size(), a.data(), a.size() * 4) == 0;
        report(same, "batch-equals-single", "");
    }
    {  // PFM round trip is exact, PGM round trip is within half a level
        const char* tmp = std::getenv("TMPDIR");
        const std::string dir = tmp ? tmp : "/tmp";
        const std::string pfm = dir + "/sgwls_b200_selftest.pfm", pgm = dir + "/sgwls_b200_selftest.pgm";
        Picture p;
        p.w = p.h = n;
        p.c = 1;
        p.px = target;
        store(p, pfm);
        store(p, pgm);
        const Picture q = load(pfm), s = load(pgm);
        bool exact = q.px == p.px;
        double worst = 0.0;
        for (std::size_t i = 0; i < p.px.size(); ++i) worst = std::max(worst, static_cast<double>(std::fabs(s.px[i] - p.px[i])));
        std::remove(pfm.c_str());
        std::remove(pgm.c_str());
        report(exact && worst <= 0.5 / 255.0 + 1e-7, "codec-roundtrip", std::to_string(worst));
    }
    std::printf(failures == 0 ? "selftest passed\n" : "selftest FAILED (%d)\n", failures);
    return failures == 0 ? 0 : 1;
}

void usage(std::FILE* f) {
    std::fputs(
        "Semi-global weighted least squares image filtering (B200)\n"
        "usage: sgwls_b200 <subcommand> [arguments] [options]\n"
        "  smooth   <input> <output> [--guidance img] [--devices 0,1,..]\n"
        "  enhance  <input> <output> [--boost g]\n"
        "  tonemap  <input.pfm> <output> [--range d] [--l1 v --l2 v --l3 v] [--dw1 v --dw2 v --dw3 v]\n"
        "  upsample <depth> <guidance> <output> [--factor f]\n"
        "  colorize <gray> <scribbles> <output> [--mask pgm] [--scribble-threshold t]\n"
        "  bench    [--op smooth] [--sizes n,..] [--r r,..] [--tau t,..] [--reps k]\n"
        "  selftest\n"
        "smoothing options: --lambda --r --tau --iters --weights frac|exp --as --ar --ss --sr --eps --gscale\n"
        "                   --first-axis col|row --threads n --preset enhance|tonemap|upsample2x|upsample4x|\n"
        "                   upsample8x|colorize\n"
        "images: pgm / ppm / pfm\n",
        f);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage(stderr);
        return 2;
    }
    const std::string sub = argv[1];
    if (sub == "-h" || sub == "--help" || sub == "help") {
        usage(stdout);
        return 0;
    }
    const std::vector<std::string> shaped = with(kSmoothOpts, {"--r", "--tau", "--preset"});
    try {
        try {
            if (sub == "smooth") return cmd_smooth(Args(argc, argv, 2, with(shaped, {"--guidance"})));
            if (sub == "enhance") return cmd_enhance(Args(argc, argv, 2, with(shaped, {"--boost"})));
            if (sub == "tonemap")
                return cmd_tonemap(Args(argc, argv, 2,
                                        with(with(kSmoothOpts, {"--r", "--tau"}),
                                             {"--range", "--l1", "--l2", "--l3", "--dw1", "--dw2", "--dw3"})));
            if (sub == "upsample") return cmd_upsample(Args(argc, argv, 2, with(shaped, {"--factor"})));
            if (sub == "colorize")
                return cmd_colorize(Args(argc, argv, 2, with(shaped, {"--mask", "--scribble-threshold"})));
            if (sub == "bench")
                return cmd_bench(Args(argc, argv, 2, with(shaped, {"--op", "--sizes", "--size", "--reps"})));
            if (sub == "selftest") return cmd_selftest(Args(argc, argv, 2, {}));
            throw UsageError("unknown subcommand '" + sub + "'");
        } catch (const UsageError& e) {
            std::fprintf(stderr, "sgwls: %s\n", e.what());
            usage(stderr);
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "sgwls: error: %s\n", e.what());
        return 1;
    }
}
