// sgwls_image_io.cu -- PGM / PPM / PFM codecs behind the C ABI (host code only).
//
// Mirrors the reference's image file interface so that the command-line tool
// (csrc/tools/sgwls_b200_main.cpp) is a drop-in for proj/tools/sgwls_main.cpp:
//
//   read_image   proj/include/sgwls/image.hpp:41  (proj/src/image.cpp:194-217;
//                decode_pnm :111-147, decode_pfm :149-176)
//   write_image  proj/include/sgwls/image.hpp:46  (proj/src/image.cpp:219-250)
//
// Same accepted formats (P2/P3/P5/P6, Pf/PF), same scaling (maxval <= 255 ->
// /255, else /65535, big-endian 16-bit samples), PFM rows bottom-up with the
// scale's sign giving the byte order, LDR writers clamp to [0,1] and quantise
// round-half-up to 255, and the same error texts ("<path>: byte N: ...").
// Samples are fp32 (the reference decodes to double; integer samples are scaled
// in double and rounded to float once, PFM floats are exact).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sgwls_b200.h"

namespace {

struct IoError {
    std::string text;
};

bool host_is_little() {
    const std::uint16_t probe = 1;
    unsigned char first;
    std::memcpy(&first, &probe, 1);
    return first == 1;
}

// Cursor over the whole file; every failure carries the byte offset it refers to.
class Cursor {
public:
    Cursor(std::string path, std::vector<unsigned char> bytes) : path_(std::move(path)), b_(std::move(bytes)) {}

    [[noreturn]] void fail_at(std::size_t where, const std::string& msg) const {
        throw IoError{path_ + ": byte " + std::to_string(where) + ": " + msg};
    }
    [[noreturn]] void fail(const std::string& msg) const { fail_at(at_, msg); }

    std::size_t size() const { return b_.size(); }
    std::size_t left() const { return b_.size() - at_; }
    const unsigned char* here() const { return b_.data() + at_; }
    void advance(std::size_t n) { at_ += n; }
    void seek(std::size_t p) { at_ = p; }
    unsigned char byte(std::size_t i) const { return b_[i]; }

    // next header token: whitespace and '#'-to-end-of-line comments skipped first
    std::string word(std::size_t* start) {
        for (;;) {
            if (at_ >= b_.size()) break;
            const unsigned char ch = b_[at_];
            if (std::isspace(ch)) {
                ++at_;
            } else if (ch == '#') {
                while (at_ < b_.size() && b_[at_] != '\n') ++at_;
            } else {
                break;
            }
        }
        if (at_ >= b_.size()) fail("unexpected end of file in header");
        const std::size_t s = at_;
        while (at_ < b_.size() && !std::isspace(b_[at_]) && b_[at_] != '#') ++at_;
        if (start) *start = s;
        return std::string(reinterpret_cast<const char*>(b_.data()) + s, at_ - s);
    }

    long integer(const char* what, long lo, long hi) {
        const std::size_t before = at_;
        const std::string t = word(nullptr);
        char* end = nullptr;
        const long v = std::strtol(t.c_str(), &end, 10);
        if (end == t.c_str() || *end != '\0') fail_at(before, std::string("malformed ") + what + " '" + t + "'");
        if (v < lo || v > hi) fail_at(before, std::string(what) + " " + std::to_string(v) + " out of range");
        return v;
    }

    double real(const char* what) {
        const std::size_t before = at_;
        const std::string t = word(nullptr);
        char* end = nullptr;
        const double v = std::strtod(t.c_str(), &end);
        if (end == t.c_str() || *end != '\0') fail_at(before, std::string("malformed ") + what + " '" + t + "'");
        return v;
    }

    // exactly one whitespace byte sits between a binary header and its payload
    void payload_gap() {
        if (at_ >= b_.size() || !std::isspace(b_[at_])) fail("missing whitespace before pixel payload");
        ++at_;
    }

    void require(std::size_t n, const char* what) {
        if (left() < n) fail_at(b_.size(), std::string("truncated ") + what);
    }

private:
    std::string path_;
    std::vector<unsigned char> b_;
    std::size_t at_ = 0;
};

struct Raster {
    int w = 0, h = 0, c = 0;
    std::vector<float> px;
};

constexpr long kMaxExtent = 1L << 20;

Raster read_netpbm(Cursor& cur, char kind) {
    const bool ascii = kind == '2' || kind == '3';
    Raster r;
    r.c = (kind == '3' || kind == '6') ? 3 : 1;
    r.w = static_cast<int>(cur.integer("width", 1, kMaxExtent));
    r.h = static_cast<int>(cur.integer("height", 1, kMaxExtent));
    const long maxval = cur.integer("maxval", 1, kMaxExtent);
    if (maxval > 65535) cur.fail("unsupported maxval " + std::to_string(maxval));
    const bool wide = maxval > 255;
    const double unit = 1.0 / (wide ? 65535.0 : 255.0);
    const std::size_t n = static_cast<std::size_t>(r.w) * r.h * r.c;
    r.px.resize(n);
    if (ascii) {
        for (std::size_t i = 0; i < n; ++i) r.px[i] = static_cast<float>(cur.integer("sample", 0, maxval) * unit);
        return r;
    }
    cur.payload_gap();
    cur.require(n * (wide ? 2 : 1), "pixel payload");
    const unsigned char* p = cur.here();
    if (wide) {
        for (std::size_t i = 0; i < n; ++i) r.px[i] = static_cast<float>(((p[2 * i] << 8) | p[2 * i + 1]) * unit);
    } else {
        for (std::size_t i = 0; i < n; ++i) r.px[i] = static_cast<float>(p[i] * unit);
    }
    cur.advance(n * (wide ? 2 : 1));
    return r;
}

Raster read_pfm(Cursor& cur, bool colour) {
    Raster r;
    r.c = colour ? 3 : 1;
    r.w = static_cast<int>(cur.integer("width", 1, kMaxExtent));
    r.h = static_cast<int>(cur.integer("height", 1, kMaxExtent));
    const double scale = cur.real("scale");
    if (scale == 0.0) cur.fail("PFM scale must be nonzero");
    const bool swap = (scale < 0.0) != host_is_little();
    cur.payload_gap();
    const std::size_t row = static_cast<std::size_t>(r.w) * r.c;
    cur.require(row * r.h * 4, "pixel payload");
    r.px.resize(row * r.h);
    bool finite = true;
    // file scanlines run bottom-up
    for (int y = r.h - 1; y >= 0; --y) {
        float* dst = r.px.data() + static_cast<std::size_t>(y) * row;
        std::memcpy(dst, cur.here(), row * 4);
        if (swap) {
            for (std::size_t i = 0; i < row; ++i) {
                std::uint32_t u;
                std::memcpy(&u, dst + i, 4);
                u = __builtin_bswap32(u);
                std::memcpy(dst + i, &u, 4);
            }
        }
        for (std::size_t i = 0; i < row; ++i) finite = finite && std::isfinite(dst[i]);
        cur.advance(row * 4);
    }
    if (!finite) cur.fail("non-finite sample in PFM payload");
    return r;
}

Raster read_any(const char* path) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw IoError{std::string(path) + ": cannot open for reading"};
    std::vector<unsigned char> bytes;
    unsigned char chunk[1 << 16];
    for (std::size_t got; (got = std::fread(chunk, 1, sizeof chunk, f)) > 0;) bytes.insert(bytes.end(), chunk, chunk + got);
    std::fclose(f);

    Cursor cur(path, std::move(bytes));
    if (cur.size() < 2) cur.fail("file too short for magic");
    const char m0 = static_cast<char>(cur.byte(0)), m1 = static_cast<char>(cur.byte(1));
    cur.seek(2);
    if (m0 != 'P') cur.fail("not a PNM/PFM file (bad magic)");
    switch (m1) {
        case '2': case '3': case '5': case '6': return read_netpbm(cur, m1);
        case 'f': return read_pfm(cur, false);
        case 'F': return read_pfm(cur, true);
        default: cur.fail(std::string("unsupported format P") + m1);
    }
}

std::string extension_lower(const std::string& path) {
    const std::size_t dot = path.rfind('.');
    std::string e = dot == std::string::npos ? std::string() : path.substr(dot + 1);
    std::transform(e.begin(), e.end(), e.begin(), [](unsigned char ch) { return static_cast<char>(std::tolower(ch)); });
    return e;
}

void write_any(const char* path_c, const float* px, int w, int h, int c) {
    const std::string path(path_c);
    if (!px || w <= 0 || h <= 0 || c <= 0) throw IoError{path + ": refusing to write empty image"};
    const std::string ext = extension_lower(path);
    const bool ldr = ext == "pgm" || ext == "ppm";
    const bool pfm = ext == "pfm";
    // the reference opens (and truncates) the file before it looks at the extension
    std::FILE* f = std::fopen(path_c, "wb");
    if (!f) throw IoError{path + ": cannot open for writing"};
    bool ok = true;
    std::string problem;
    const std::size_t n = static_cast<std::size_t>(w) * h * c;
    if (ldr) {
        const int want = ext == "pgm" ? 1 : 3;
        if (c != want) {
            problem = path + ": " + std::to_string(c) + "-channel image does not fit ." + ext;
        } else {
            ok = std::fprintf(f, "%s\n%d %d\n255\n", want == 1 ? "P5" : "P6", w, h) > 0;
            std::vector<unsigned char> q(n);
            for (std::size_t i = 0; i < n; ++i) {
                const double v = std::min(std::max(static_cast<double>(px[i]), 0.0), 1.0);
                q[i] = static_cast<unsigned char>(std::floor(v * 255.0 + 0.5));
            }
            ok = ok && std::fwrite(q.data(), 1, n, f) == n;
        }
    } else if (pfm) {
        ok = std::fprintf(f, "%s\n%d %d\n%s\n", c == 1 ? "Pf" : "PF", w, h, host_is_little() ? "-1.0" : "1.0") > 0;
        const std::size_t row = static_cast<std::size_t>(w) * c;
        for (int y = h - 1; y >= 0 && ok; --y) ok = std::fwrite(px + static_cast<std::size_t>(y) * row, 4, row, f) == row;
    } else {
        problem = path + ": unsupported output extension '" + ext + "'";
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!problem.empty()) throw IoError{problem};
    if (!ok) throw IoError{path + ": write failed"};
}

void put(char* err, size_t errlen, const std::string& msg) {
    if (err && errlen) {
        std::snprintf(err, errlen, "%s", msg.c_str());
    }
}

}  // namespace

extern "C" {

int sgwls_b200_image_read(const char* path, float** data, int* width, int* height, int* channels, char* err,
                          size_t errlen) {
    if (!path || !data || !width || !height || !channels) {
        put(err, errlen, "image_read: null argument");
        return SGWLS_B200_EINVAL;
    }
    try {
        Raster r = read_any(path);
        // read_image's final check (proj/src/image.cpp:215); PFM already failed above with a byte offset
        for (float v : r.px)
            if (!std::isfinite(v)) throw IoError{std::string(path) + ": decoded image contains non-finite samples"};
        float* out = static_cast<float*>(std::malloc(r.px.size() * sizeof(float)));
        if (!out) throw IoError{std::string(path) + ": out of memory"};
        std::memcpy(out, r.px.data(), r.px.size() * sizeof(float));
        *data = out;
        *width = r.w;
        *height = r.h;
        *channels = r.c;
        return SGWLS_B200_OK;
    } catch (const IoError& e) {
        put(err, errlen, e.text);
        return SGWLS_B200_EINVAL;
    } catch (const std::exception& e) {
        put(err, errlen, e.what());
        return SGWLS_B200_EINVAL;
    }
}

void sgwls_b200_image_free(float* data) { std::free(data); }

int sgwls_b200_image_write(const char* path, const float* data, int width, int height, int channels, char* err,
                           size_t errlen) {
    if (!path) {
        put(err, errlen, "image_write: null path");
        return SGWLS_B200_EINVAL;
    }
    try {
        write_any(path, data, width, height, channels);
        return SGWLS_B200_OK;
    } catch (const IoError& e) {
        put(err, errlen, e.text);
        return SGWLS_B200_EINVAL;
    } catch (const std::exception& e) {
        put(err, errlen, e.what());
        return SGWLS_B200_EINVAL;
    }
}

}  // extern "C"
