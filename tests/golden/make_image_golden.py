"""Generate the image-codec fixtures from the REFERENCE codecs (proj/src/image.cpp).

Run in the build container (oracle/_ref built):  python tests/golden/make_image_golden.py
Writes tests/golden/images/: small files written by the reference's write_image
(.pgm/.ppm/.pfm), hand-assembled inputs covering the decoder's branches (ASCII
P2/P3 with comments, 16-bit P5, big-endian PFM), malformed files, and
images.npz with the reference's decode of every readable file plus its error text
for every malformed one.  The GPU box has no /root/reference: these pin the
product codec (csrc/sgwls_image_io.cu) there.
"""
from __future__ import annotations

import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
OUT = os.path.join(HERE, "images")

from oracle.pyoracle import OracleError, RefImageIO  # noqa: E402


def handmade() -> dict[str, bytes]:
    rng = np.random.default_rng(170501674)
    f = {}
    f["ascii_gray.pgm"] = b"P2\n# a comment\n4 3\n# another\n15\n" + b" ".join(
        str(int(v)).encode() for v in rng.integers(0, 16, 12)) + b"\n"
    f["ascii_rgb.ppm"] = b"P3 2 2 255\n" + b"\n".join(str(int(v)).encode() for v in rng.integers(0, 256, 12)) + b"\n"
    f["wide_gray.pgm"] = b"P5\n3 2\n65535\n" + rng.integers(0, 65536, 6).astype(">u2").tobytes()
    f["wide_rgb_1000.ppm"] = b"P6 2 1 1000 " + rng.integers(0, 1001, 6).astype(">u2").tobytes()
    f["big_endian.pfm"] = b"Pf\n3 2\n1.0\n" + rng.uniform(-2, 5, 6).astype(">f4").tobytes()
    f["little_rgb.pfm"] = b"PF 2 2 -2.5\n" + rng.uniform(0, 100, 12).astype("<f4").tobytes()
    # malformed
    f["bad_short.pgm"] = b"P"
    f["bad_magic.pgm"] = b"Q5 1 1 255 \x00"
    f["bad_format.pgm"] = b"P7 1 1 255 \x00"
    f["bad_width.pgm"] = b"P5 x1 1 255 \x00"
    f["bad_range.pgm"] = b"P5 0 1 255 \x00"
    f["bad_maxval.pgm"] = b"P5 1 1 70000 \x00\x00"
    f["bad_trunc.ppm"] = b"P6 2 2 255\n" + bytes(7)
    f["bad_sep.pgm"] = b"P5 1 1 255"
    f["bad_sample.pgm"] = b"P2 2 1 7 3 9"
    f["bad_header_eof.pgm"] = b"P2 2 # only a comment"
    f["bad_scale.pfm"] = b"Pf 1 1 0.0\n" + bytes(4)
    f["bad_scale_text.pfm"] = b"Pf 1 1 abc\n" + bytes(4)
    f["bad_nan.pfm"] = b"Pf 1 1 -1.0\n" + struct.pack("<f", float("nan"))
    f["bad_trunc.pfm"] = b"PF 2 2 -1.0\n" + bytes(20)
    return f


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    io = RefImageIO()
    rng = np.random.default_rng(1705)
    written = {
        "ref_gray.pgm": rng.uniform(-0.2, 1.2, (5, 7, 1)),
        "ref_rgb.ppm": rng.uniform(0, 1, (4, 6, 3)),
        "ref_gray.pfm": rng.uniform(-3, 3, (3, 5, 1)),
        "ref_rgb.pfm": rng.uniform(0, 50, (2, 3, 3)),
        # quantiser ties: k/255 +- half a level
        "ref_ties.pgm": ((np.arange(24) + 0.5) / 255.0).reshape(4, 6, 1),
    }
    arrays = {}
    for name, img in written.items():
        io.write(img, os.path.join(OUT, name))
        arrays["src:" + name] = img
    for name, blob in handmade().items():
        with open(os.path.join(OUT, name), "wb") as fh:
            fh.write(blob)
    for name in sorted(os.listdir(OUT)):
        if name.endswith(".npz"):
            continue
        path = os.path.join(OUT, name)
        try:
            arrays["img:" + name] = io.read(path)
        except OracleError as e:
            # error texts start with the path the reader was given: keep them relative
            arrays["err:" + name] = np.array(str(e).replace(path, name))
    np.savez_compressed(os.path.join(OUT, "images.npz"), **arrays)
    print("wrote", len(arrays), "entries")
    for k, v in arrays.items():
        if k.startswith("err:"):
            print(" ", k, "->", v)


if __name__ == "__main__":
    main()
