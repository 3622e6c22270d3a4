"""The command-line tool (paper_1705_01674_b200/bin/sgwls_b200, csrc/tools/
sgwls_b200_main.cpp), the GPU drop-in for the reference's proj/tools/sgwls_main.cpp:
option handling and exit codes on the CPU; on the GPU its `smooth`, `enhance`,
`upsample`, `bench` and `selftest` subcommands on image files, checked against the
CPU oracle / the reference's apps.cpp (bar 1e-4 on float output, one 8-bit level
on quantised output)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1705_01674_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1705_01674_b200", "bin", "sgwls_b200")
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libsgwls_ref.so"))


def run(*args, env=None):
    if not os.path.exists(EXE):  # normally built by __graft_entry__.build(); g++ only, no GPU needed
        from paper_1705_01674_b200._build import build_cli
        build_cli()
    assert os.path.exists(EXE), "run __graft_entry__.build() first"
    e = dict(os.environ)
    e.pop("SGWLS_THREADS", None)
    e.update(env or {})
    return subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, env=e, timeout=600)


def scene(h, w, seed, c=1):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    base = 0.25 + 0.2 * (x > w * 0.35) + 0.3 * (y > h * 0.55) + 0.1 * ((x // 9 + y // 7) % 2)
    img = np.stack([np.clip(base * (1 - 0.15 * k) + rng.normal(0, 0.03, (h, w)), 0, 1) for k in range(c)], axis=2)
    return img.astype(np.float32)


# ------------------------------------------------------------ host (no GPU)

def test_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("frobnicate").returncode == 2
    r = run("smooth", "a.pgm")
    assert r.returncode == 2 and "expected arguments" in r.stderr
    r = run("smooth", "a.pgm", "b.pgm", "--nonsense", "1")
    assert r.returncode == 2 and "unknown option --nonsense" in r.stderr
    r = run("smooth", "a.pgm", "b.pgm", "--lambda")
    assert r.returncode == 2
    assert run("--help").returncode == 0


def test_config_errors_exit_1_with_reference_texts(tmp_path):
    """make_config / preset_by_name texts, proj/tools/sgwls_main.cpp:73-117"""
    r = run("smooth", "a.pgm", "b.pgm", "--preset", "sharpen")
    assert r.returncode == 1 and r.stderr.strip().endswith("sgwls: error: unknown preset 'sharpen'")
    r = run("smooth", "a.pgm", "b.pgm", "--weights", "gauss")
    assert r.returncode == 1 and "sgwls: error: --weights must be 'frac' or 'exp'" in r.stderr
    r = run("smooth", "a.pgm", "b.pgm", "--first-axis", "diag")
    assert r.returncode == 1 and "sgwls: error: --first-axis must be 'col' or 'row'" in r.stderr
    missing = tmp_path / "missing.pgm"
    r = run("smooth", missing, tmp_path / "o.pgm")
    assert r.returncode == 1 and f"sgwls: error: {missing}: cannot open for reading" in r.stderr


def test_echo_line_follows_preset_and_override_rules(tmp_path):
    """echo_config proj/tools/sgwls_main.cpp:119-128; the echo precedes the file access"""
    nof = tmp_path / "none.pgm"
    r = run("smooth", nof, nof)
    assert ("sgwls: smooth lambda=900 r=1 tau=1 iters=4 weights=frac alpha_s=1.2 alpha_r=1.2 sigma_s=4 "
            "sigma_r=3 eps=0.0001 gscale=1 first_axis=col threads=1") in r.stderr
    r = run("smooth", nof, nof, "--weights", "exp", "--r", "2", "--tau=3", "--lambda", "400", "--sr", "0.03",
            "--threads", "5")
    assert "lambda=400 r=2 tau=3 iters=4 weights=exp" in r.stderr and "gscale=255" in r.stderr
    assert "threads=5" in r.stderr
    r = run("smooth", nof, nof, "--preset", "colorize", "--iters", "2")
    assert "lambda=900 r=4 tau=2 iters=2 weights=exp" in r.stderr and "sigma_r=2" in r.stderr
    assert "gscale=255" in r.stderr
    r = run("upsample", nof, nof, nof, "--factor", "8")
    assert "sgwls: upsample lambda=400 r=4 tau=4" in r.stderr
    r = run("enhance", nof, nof, env={"SGWLS_THREADS": "3"})
    assert "sgwls: enhance lambda=900 r=1 tau=1 iters=4 weights=frac" in r.stderr and "threads=3" in r.stderr
    r = run("bench", "--op", "wlsref")
    assert r.returncode == 1 and "wlsref" in r.stderr


# ------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_cli_smooth_pfm_and_pgm_match_oracle(tmp_path, port):
    img = scene(70, 93, 3)
    S.write_image(img, str(tmp_path / "in.pfm"))
    cfg = S.SmoothConfig(lambda_=400.0, r=2, tau=3, iterations=4,
                         weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.05, guidance_scale=1.0))
    flags = ["--weights", "exp", "--lambda", 400, "--r", 2, "--tau", 3, "--sr", 0.05, "--gscale", 1]
    r = run("smooth", tmp_path / "in.pfm", tmp_path / "out.pfm", *flags)
    assert r.returncode == 0, r.stderr
    want = port.smooth(img, img, cfg)
    got = S.read_image(str(tmp_path / "out.pfm"))[:, :, 0]
    assert np.abs(got - want[..., 0] if want.ndim == 3 else got - want).max() <= 1e-4
    # quantised output, separate guidance, row-first
    S.write_image(img, str(tmp_path / "in.pgm"))
    q = S.read_image(str(tmp_path / "in.pgm"))
    guide = scene(70, 93, 4, c=3)
    S.write_image(guide, str(tmp_path / "g.ppm"))
    gq = S.read_image(str(tmp_path / "g.ppm"))
    r = run("smooth", tmp_path / "in.pgm", tmp_path / "out.pgm", "--guidance", tmp_path / "g.ppm", *flags,
            "--first-axis", "row", "--iters", 3)
    assert r.returncode == 0, r.stderr
    cfg2 = S.SmoothConfig(lambda_=400.0, r=2, tau=3, iterations=3, first_axis=S.Axis.Row, weight=cfg.weight)
    want = np.asarray(port.smooth(q, gq, cfg2)).reshape(70, 93)
    got = S.read_image(str(tmp_path / "out.pgm"))[:, :, 0]
    level = np.floor(np.clip(want, 0, 1) * 255 + 0.5) / 255
    assert np.abs(got - level).max() <= 1.0 / 255 + 1e-6
    assert np.mean(np.abs(got - level) > 1e-6) < 0.01
    # size mismatch: the reference's text
    S.write_image(scene(10, 12, 5), str(tmp_path / "small.pgm"))
    r = run("smooth", tmp_path / "in.pgm", tmp_path / "o2.pgm", "--guidance", tmp_path / "small.pgm")
    assert r.returncode == 1 and "sgwls: error: smooth: target and guidance dimensions differ" in r.stderr
    r = run("smooth", tmp_path / "in.pgm", tmp_path / "o2.pgm", "--tau", 9)
    assert r.returncode == 1 and "sgwls: error: smooth: tau must be in [1, 2r+1], got 9" in r.stderr


@pytest.mark.gpu
def test_cli_devices_runs_the_slab_filter(tmp_path):
    img = scene(120, 64, 6)
    S.write_image(img, str(tmp_path / "in.pfm"))
    flags = ["--weights", "exp", "--lambda", 300, "--r", 2, "--tau", 2, "--sr", 0.05, "--gscale", 1]
    assert run("smooth", tmp_path / "in.pfm", tmp_path / "a.pfm", *flags).returncode == 0
    r = run("smooth", tmp_path / "in.pfm", tmp_path / "b.pfm", *flags, "--devices", "0,0,0")
    assert r.returncode == 0, r.stderr
    a, b = S.read_image(str(tmp_path / "a.pfm")), S.read_image(str(tmp_path / "b.pfm"))
    assert np.abs(a - b).max() <= 2e-6


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference library not built")
def test_cli_apps_match_reference_apps(tmp_path):
    from oracle.pyoracle import RefApps
    from paper_1705_01674_b200 import apps as A
    ref = RefApps()
    rgb = scene(48, 60, 7, c=3)
    S.write_image(rgb, str(tmp_path / "in.ppm"))
    q = S.read_image(str(tmp_path / "in.ppm"))
    r = run("enhance", tmp_path / "in.ppm", tmp_path / "enh.pfm", "--boost", 2.5)
    assert r.returncode == 0, r.stderr
    want = ref.detail_enhance(q, 2.5, A.enhance_preset())
    assert np.abs(S.read_image(str(tmp_path / "enh.pfm")) - want).max() <= 1e-4
    # upsample: factor 4 picks the published preset
    depth = scene(12, 15, 8)[:, :, 0]
    S.write_image(depth, str(tmp_path / "d.pfm"))
    r = run("upsample", tmp_path / "d.pfm", tmp_path / "in.ppm", tmp_path / "up.pfm", "--factor", 4)
    assert r.returncode == 0, r.stderr
    want = ref.depth_upsample(depth, q, 4, A.upsample_preset(4))
    assert np.abs(S.read_image(str(tmp_path / "up.pfm"))[:, :, 0] - want).max() <= 1e-4
    # tonemap on an HDR pfm
    hdr = (np.exp(3.0 * scene(40, 44, 9, c=3)) * 0.05).astype(np.float32)
    S.write_image(hdr, str(tmp_path / "hdr.pfm"))
    r = run("tonemap", tmp_path / "hdr.pfm", tmp_path / "tm.pfm", "--range", 1.5)
    assert r.returncode == 0, r.stderr
    p = A.ToneMapParams(target_log_range=1.5)
    want = ref.tone_map(hdr, p)
    got = S.read_image(str(tmp_path / "tm.pfm"))
    assert np.abs(got - want).max() / max(1.0, float(np.abs(want).max())) <= 1e-4
    # colorize with the chroma-threshold mask
    gray = scene(40, 44, 10)
    scrib = np.repeat(gray, 3, axis=2).copy()
    scrib[5:9, 5:30] = (0.9, 0.2, 0.1)
    scrib[25:29, 10:40] = (0.1, 0.3, 0.9)
    S.write_image(gray, str(tmp_path / "gray.pgm"))
    S.write_image(scrib, str(tmp_path / "scrib.ppm"))
    gq, sq = S.read_image(str(tmp_path / "gray.pgm")), S.read_image(str(tmp_path / "scrib.ppm"))
    r = run("colorize", tmp_path / "gray.pgm", tmp_path / "scrib.ppm", tmp_path / "col.pfm")
    assert r.returncode == 0, r.stderr
    sd = sq.astype(np.float64)
    luma = 0.299 * sd[..., 0] + 0.587 * sd[..., 1] + 0.114 * sd[..., 2]
    mask = ((np.abs((sd[..., 2] - luma) / 1.772) > 2 / 255) | (np.abs((sd[..., 0] - luma) / 1.402) > 2 / 255))
    want = ref.colorize(gq[:, :, 0], sq, mask.astype(np.float32), A.colorize_preset())
    assert np.abs(S.read_image(str(tmp_path / "col.pfm")) - want).max() <= 1e-4


@pytest.mark.gpu
def test_cli_bench_csv_and_selftest():
    r = run("bench", "--sizes", "128,256", "--r", "1,2", "--tau", "1,7", "--reps", 2, "--weights", "exp",
            "--gscale", 1, "--sr", 0.05)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "op,M,N,r,tau,T,seconds"
    rows = [ln.split(",") for ln in lines[1:]]
    # tau = 7 is skipped for r = 1 and r = 2 (stride too large), as in the reference
    assert [(x[1], x[3], x[4]) for x in rows] == [("128", "1", "1"), ("128", "2", "1"), ("256", "1", "1"),
                                                  ("256", "2", "1")]
    assert all(x[0] == "smooth" and x[5] == "4" and re.fullmatch(r"\d+\.\d{6}", x[6]) for x in rows)
    assert r.stderr.count("skipping r=") == 4
    r = run("selftest")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("selftest passed") and "FAIL" not in r.stdout
