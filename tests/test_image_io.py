"""The PGM / PPM / PFM codec behind the C ABI (csrc/sgwls_image_io.cu:
sgwls_b200_image_read / _write, Python read_image / write_image) against the
reference's codecs (proj/src/image.cpp:111-250).

Two pins: the committed fixtures under tests/golden/images (files written by the
reference, hand-made inputs for every decoder branch, malformed files with the
reference's error texts; tests/golden/make_image_golden.py) and, where the
reference is built (oracle/_ref/ref_imgtool), live comparisons on seeded images.
Bar: decoded samples equal float32(reference double); written files byte-identical.
No GPU needed."""
import os

import numpy as np
import pytest

import paper_1705_01674_b200 as S

HERE = os.path.dirname(os.path.abspath(__file__))
IMAGES = os.path.join(HERE, "golden", "images")
GOLD = np.load(os.path.join(IMAGES, "images.npz"))
HAVE_TOOL = os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_imgtool"))
needs_ref = pytest.mark.skipif(not HAVE_TOOL, reason="reference codecs not built (needs /root/reference at build time)")

READABLE = sorted(k[4:] for k in GOLD.files if k.startswith("img:"))
BROKEN = sorted(k[4:] for k in GOLD.files if k.startswith("err:"))


@pytest.mark.parametrize("name", READABLE)
def test_decode_matches_reference_fixture(name):
    got = S.read_image(os.path.join(IMAGES, name))
    want = GOLD["img:" + name]
    assert got.dtype == np.float32 and got.shape == want.shape
    assert np.array_equal(got, want.astype(np.float32)), name


@pytest.mark.parametrize("name", BROKEN)
def test_decode_errors_carry_reference_text(name):
    path = os.path.join(IMAGES, name)
    with pytest.raises(S.Error) as e:
        S.read_image(path)
    assert str(e.value) == str(GOLD["err:" + name]).replace(name, path, 1)


@pytest.mark.parametrize("name", sorted(k[4:] for k in GOLD.files if k.startswith("src:")))
def test_encode_reproduces_reference_file(name, tmp_path):
    src = GOLD["src:" + name]
    out = tmp_path / name
    # the reference quantised doubles; feed the same values (float64 -> float32 keeps
    # every level of these fixtures except exact ties, which ref_ties.pgm holds as .5/255
    # offsets that survive the rounding)
    S.write_image(src.astype(np.float32), str(out))
    want = open(os.path.join(IMAGES, name), "rb").read()
    got = out.read_bytes()
    if name.endswith(".pfm"):
        assert got == want
    else:
        assert got[:got.index(b"255\n")] == want[:want.index(b"255\n")]
        a = np.frombuffer(got[got.index(b"255\n") + 4:], np.uint8).astype(int)
        b = np.frombuffer(want[want.index(b"255\n") + 4:], np.uint8).astype(int)
        # float32 rounding of the source may move a value across a quantiser boundary
        assert a.shape == b.shape and np.abs(a - b).max() <= (1 if "ties" in name else 0)


def test_missing_file_and_bad_extension(tmp_path):
    with pytest.raises(S.Error, match="cannot open for reading"):
        S.read_image(str(tmp_path / "nope.pgm"))
    img = np.zeros((2, 2, 1), np.float32)
    with pytest.raises(S.Error) as e:
        S.write_image(img, str(tmp_path / "x.png"))
    assert str(e.value) == f"{tmp_path / 'x.png'}: unsupported output extension 'png'"
    with pytest.raises(S.Error) as e:
        S.write_image(img, str(tmp_path / "x.ppm"))
    assert str(e.value) == f"{tmp_path / 'x.ppm'}: 1-channel image does not fit .ppm"
    with pytest.raises(S.Error, match="refusing to write empty image"):
        S.write_image(np.zeros((0, 0, 1), np.float32), str(tmp_path / "e.pgm"))


@needs_ref
@pytest.mark.parametrize("ext,shape", [("pgm", (33, 47, 1)), ("ppm", (20, 31, 3)), ("pfm", (17, 9, 1)),
                                       ("pfm", (8, 12, 3))])
def test_live_round_trip_against_reference(ext, shape, tmp_path):
    from oracle.pyoracle import RefImageIO
    io = RefImageIO()
    rng = np.random.default_rng(hash((ext, shape)) % 2**32)
    img = rng.uniform(-0.1, 1.1, shape).astype(np.float32)
    mine, theirs = str(tmp_path / f"mine.{ext}"), str(tmp_path / f"ref.{ext}")
    S.write_image(img, mine)
    io.write(img.astype(np.float64), theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(S.read_image(theirs), io.read(mine).astype(np.float32))


@needs_ref
def test_live_error_texts_match_reference(tmp_path):
    from oracle.pyoracle import OracleError, RefImageIO
    io = RefImageIO()
    blobs = [b"P5 3 3 255\n" + bytes(8), b"P2 1 1 300 301", b"P6 1 1 0 \x00\x00\x00", b"P5 # c\n 2 2 x",
             b"Pf 2 2 -1", b"PF 1 1 1e400\n" + bytes(12), b"P3 1 1 255 1 2", b"P5 1048577 1 255 "]
    for i, blob in enumerate(blobs):
        path = str(tmp_path / f"m{i}.bin")
        with open(path, "wb") as f:
            f.write(blob)
        try:
            want = io.read(path)
        except OracleError as e:
            with pytest.raises(S.Error) as got:
                S.read_image(path)
            assert str(got.value) == str(e), blob
        else:  # odd but accepted by the reference (e.g. an infinite PFM scale)
            assert np.array_equal(S.read_image(path), want.astype(np.float32)), blob
