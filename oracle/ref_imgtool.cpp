// TEST INFRASTRUCTURE ONLY.
//
// The reference's image codecs (sgwls::read_image / write_image,
// proj/src/image.cpp:194-250) as a tiny command-line checker, linked against the
// UNMODIFIED reference sources by oracle/Makefile (-> oracle/_ref/ref_imgtool).
// A separate process, not a ctypes call: inside a Python process that has numpy
// loaded, libstdc++'s iostream number formatting (used by the reference's
// writers) faults on this image, so the checker keeps its own address space.
//
//   ref_imgtool read  <image> <out.f64>        prints "w h c", writes raw doubles
//   ref_imgtool write <in.f64> w h c <image>   raw doubles -> image by extension
// Exit 1 with the sgwls::Error text on stderr when the reference throws.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <vector>

#include "sgwls/image.hpp"

int main(int argc, char** argv) {
    try {
        if (argc == 4 && !std::strcmp(argv[1], "read")) {
            const sgwls::Image im = sgwls::read_image(argv[2]);
            std::FILE* f = std::fopen(argv[3], "wb");
            if (!f) return 3;
            std::fwrite(im.data.data(), sizeof(double), im.data.size(), f);
            std::fclose(f);
            std::printf("%d %d %d\n", im.width, im.height, im.channels);
            return 0;
        }
        if (argc == 7 && !std::strcmp(argv[1], "write")) {
            const int w = std::atoi(argv[3]), h = std::atoi(argv[4]), c = std::atoi(argv[5]);
            sgwls::Image im;
            if (w > 0 && h > 0) {
                im = sgwls::Image(w, h, c);
                std::FILE* f = std::fopen(argv[2], "rb");
                if (!f || std::fread(im.data.data(), sizeof(double), im.data.size(), f) != im.data.size()) return 3;
                std::fclose(f);
            }
            sgwls::write_image(im, argv[6]);
            return 0;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 1;
    }
    std::fprintf(stderr, "usage: ref_imgtool read <image> <out.f64> | write <in.f64> w h c <image>\n");
    return 2;
}
