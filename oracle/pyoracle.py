"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU checkers.

``CpuOracle("port")`` loads oracle/build/libsgwls_oracle.so (the C restatement,
oracle/sgwls_oracle.c); ``CpuOracle("reference")`` loads oracle/_ref/libsgwls_ref.so
(the unmodified reference library compiled from /root/reference/proj/src by
oracle/Makefile).  Both expose the same calls with fp32 inputs promoted to
double and double outputs.  Only tests/, __graft_entry__.smoke() and bench.py's
CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "libsgwls_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libsgwls_ref.so")


class OracleConfig(C.Structure):
    _fields_ = [
        ("lambda_", C.c_double),
        ("r", C.c_int),
        ("tau", C.c_int),
        ("iterations", C.c_int),
        ("first_axis", C.c_int),
        ("threads", C.c_int),
        ("kind", C.c_int),
        ("alpha_s", C.c_double),
        ("alpha_r", C.c_double),
        ("sigma_s", C.c_double),
        ("sigma_r", C.c_double),
        ("epsilon", C.c_double),
        ("guidance_scale", C.c_double),
    ]


def make_config(cfg) -> OracleConfig:
    """Accepts a paper_1705_01674_b200.SmoothConfig (or any object with the same fields)."""
    w = cfg.weight
    return OracleConfig(
        float(cfg.lambda_), int(cfg.r), int(cfg.tau), int(cfg.iterations), int(cfg.first_axis),
        int(cfg.threads), int(w.kind), float(w.alpha_s), float(w.alpha_r), float(w.sigma_s),
        float(w.sigma_r), float(w.epsilon), float(w.guidance_scale))


def build(ref: bool = True) -> None:
    targets = ["all"] if ref else ["oracle"]
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class OracleError(RuntimeError):
    pass


_P = C.c_void_p


class CpuOracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            if kind == "port" or os.path.isdir("/root/reference/proj/src"):
                build(ref=(kind != "port"))
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        self.lib = C.CDLL(path)
        pre = "oracle_" if kind == "port" else "ref_"
        self._smooth = getattr(self.lib, pre + "smooth_f32")
        self._smooth.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.POINTER(OracleConfig), _P,
                                 C.c_char_p, C.c_size_t]
        self._smooth.restype = C.c_int
        self._interp = getattr(self.lib, pre + "interpolate_sparse_f32")
        self._interp.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, C.POINTER(OracleConfig), _P, _P,
                                 C.c_char_p, C.c_size_t]
        self._interp.restype = C.c_int
        self._centers = getattr(self.lib, pre + "band_centers")
        self._centers.argtypes = [C.c_int, C.c_int, C.c_int, _P, C.c_int]
        self._centers.restype = C.c_int
        self._solve_band = getattr(self.lib, pre + "solve_band")
        self._solve_band.argtypes = [C.c_int, C.c_int, _P, C.c_double, _P, _P, _P, _P, _P]
        self._solve_band.restype = C.c_int
        self._layout = getattr(self.lib, pre + "band_layout")
        self._layout.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]
        self._layout.restype = C.c_int
        self._weights = getattr(self.lib, pre + "edge_weights")
        self._weights.argtypes = [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(OracleConfig), _P]
        self._weights.restype = C.c_int

    @staticmethod
    def _hwc(a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float32)
        return a[:, :, None] if a.ndim == 2 else a

    def smooth(self, target: np.ndarray, guidance: np.ndarray, cfg) -> np.ndarray:
        t = self._hwc(target)
        g = self._hwc(guidance)
        h, w, c = t.shape
        out = np.empty((h, w, c), dtype=np.float64)
        err = C.create_string_buffer(512)
        oc = make_config(cfg)
        rc = self._smooth(t.ctypes.data, w, h, c, g.ctypes.data, g.shape[2], C.byref(oc), out.ctypes.data, err, 512)
        if rc:
            raise OracleError(err.value.decode())
        return out if target.ndim == 3 else out[:, :, 0]

    def interpolate_sparse(self, values: np.ndarray, mask: np.ndarray, guidance: np.ndarray, cfg):
        v = self._hwc(values)
        m = np.ascontiguousarray(mask, dtype=np.float32).reshape(v.shape[0], v.shape[1])
        g = self._hwc(guidance)
        h, w, c = v.shape
        out = np.empty((h, w, c), dtype=np.float64)
        und = np.zeros((h, w), dtype=np.float64)
        err = C.create_string_buffer(512)
        oc = make_config(cfg)
        rc = self._interp(v.ctypes.data, w, h, c, m.ctypes.data, g.ctypes.data, g.shape[2], C.byref(oc),
                          out.ctypes.data, und.ctypes.data, err, 512)
        if rc:
            raise OracleError(err.value.decode())
        return (out if values.ndim == 3 else out[:, :, 0]), und

    def band_centers(self, extent: int, r: int, tau: int):
        buf = np.zeros(extent + 4, dtype=np.int32)
        n = self._centers(extent, r, tau, buf.ctypes.data, len(buf))
        return buf[:n].tolist()

    def band_layout(self, height: int, width: int, center: int, r: int, axis: int):
        cap = (2 * r + 1) * max(height, width) + 8
        rows = np.zeros(cap, dtype=np.int32)
        cols = np.zeros(cap, dtype=np.int32)
        n = self._layout(height, width, center, r, axis, rows.ctypes.data, cols.ctypes.data)
        return rows[:n].copy(), cols[:n].copy()

    def solve_band(self, w: np.ndarray, lam: float, rhs: np.ndarray, r: int):
        n = len(rhs)
        w = np.ascontiguousarray(w, dtype=np.float64)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        u = np.zeros(n)
        alpha = np.zeros(n)
        beta = np.zeros(n * r)
        gamma = np.zeros(n * r)
        bad = self._solve_band(n, r, w.ctypes.data, lam, rhs.ctypes.data, u.ctypes.data, alpha.ctypes.data,
                               beta.ctypes.data, gamma.ctypes.data)
        if bad >= 0:
            raise OracleError(f"non-positive pivot at row {bad}")
        return u, alpha, beta, gamma

    def edge_weights(self, guidance: np.ndarray, center: int, r: int, axis: int, cfg) -> np.ndarray:
        g = np.ascontiguousarray(guidance, dtype=np.float64)
        g = g[:, :, None] if g.ndim == 2 else g
        h, w, gc = g.shape
        extent = w if axis == 0 else h
        sweep = h if axis == 0 else w
        lo, hi = max(0, center - r), min(extent - 1, center + r)
        n = (hi - lo + 1) * sweep
        out = np.zeros(n * r)
        oc = make_config(cfg)
        self._weights(g.ctypes.data, w, h, gc, center, r, axis, C.byref(oc), out.ctypes.data)
        return out


def available(kind: str) -> bool:
    try:
        CpuOracle(kind)
        return True
    except (FileNotFoundError, OSError, subprocess.CalledProcessError):
        return False


class RefApps:
    """The reference's application pipelines (proj/src/apps.cpp) from
    oracle/_ref/libsgwls_ref.so: the checker of the device pipelines
    (paper_1705_01674_b200.apps).  Needs the reference build (this container
    builds it; the .so travels to the GPU box with the repository)."""

    def __init__(self):
        self.lib = CpuOracle("reference").lib
        L = self.lib
        L.ref_detail_enhance_f32.argtypes = [_P, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(OracleConfig), _P,
                                             C.c_char_p, C.c_size_t]
        L.ref_tone_map_f32.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_double, C.POINTER(OracleConfig),
                                       _P, C.c_char_p, C.c_size_t]
        L.ref_depth_upsample_f32.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.POINTER(OracleConfig), _P, C.c_char_p, C.c_size_t]
        L.ref_colorize_f32.argtypes = [_P, _P, _P, C.c_int, C.c_int, C.POINTER(OracleConfig), _P, C.c_char_p,
                                       C.c_size_t]

    @staticmethod
    def _call(fn, *args):
        err = C.create_string_buffer(512)
        if fn(*args, err, 512):
            raise OracleError(err.value.decode())

    def detail_enhance(self, img, boost, cfg):
        a = CpuOracle._hwc(img)
        h, w, c = a.shape
        out = np.empty((h, w, c))
        self._call(self.lib.ref_detail_enhance_f32, a.ctypes.data, w, h, c, float(boost), C.byref(make_config(cfg)),
                   out.ctypes.data)
        return out if np.asarray(img).ndim == 3 else out[:, :, 0]

    def tone_map(self, hdr, params):
        a = CpuOracle._hwc(hdr)
        h, w, c = a.shape
        lam = np.asarray(params.lambdas, dtype=np.float64)
        dw = np.asarray(params.detail_weights, dtype=np.float64)
        out = np.empty((h, w, c))
        self._call(self.lib.ref_tone_map_f32, a.ctypes.data, w, h, c, lam.ctypes.data, dw.ctypes.data,
                   float(params.target_log_range), C.byref(make_config(params.smoothing)), out.ctypes.data)
        return out if np.asarray(hdr).ndim == 3 else out[:, :, 0]

    def depth_upsample(self, low, guidance, factor, cfg):
        d = CpuOracle._hwc(low)
        g = CpuOracle._hwc(guidance)
        out = np.empty(g.shape[:2])
        self._call(self.lib.ref_depth_upsample_f32, d.ctypes.data, d.shape[1], d.shape[0], d.shape[2], g.ctypes.data,
                   g.shape[1], g.shape[0], g.shape[2], int(factor), C.byref(make_config(cfg)), out.ctypes.data)
        return out

    def colorize(self, gray, scribbles, mask, cfg):
        g = np.ascontiguousarray(gray, dtype=np.float32)
        s = np.ascontiguousarray(scribbles, dtype=np.float32)
        m = np.ascontiguousarray(mask, dtype=np.float32)
        h, w = g.shape[:2]
        out = np.empty((h, w, 3))
        self._call(self.lib.ref_colorize_f32, g.ctypes.data, s.ctypes.data, m.ctypes.data, w, h,
                   C.byref(make_config(cfg)), out.ctypes.data)
        return out


class RefImageIO:
    """The reference's image codecs (proj/src/image.cpp:194-250) through
    oracle/_ref/ref_imgtool (its own process, see oracle/ref_imgtool.cpp): the checker
    of paper_1705_01674_b200.read_image / write_image and of the CLI's files."""

    TOOL = os.path.join(HERE, "_ref", "ref_imgtool")

    def __init__(self):
        if not os.path.exists(self.TOOL) and os.path.isdir("/root/reference/proj/src"):
            build(ref=True)
        if not os.path.exists(self.TOOL):
            raise FileNotFoundError(self.TOOL)

    def _run(self, *args) -> str:
        import subprocess
        r = subprocess.run([self.TOOL, *map(str, args)], capture_output=True, text=True)
        if r.returncode == 1:
            raise OracleError(r.stderr.strip())
        if r.returncode != 0:
            raise RuntimeError(f"ref_imgtool rc={r.returncode}: {r.stderr}")
        return r.stdout

    def read(self, path: str) -> np.ndarray:
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            raw = os.path.join(d, "img.f64")
            w, h, c = map(int, self._run("read", path, raw).split())
            return np.fromfile(raw, dtype=np.float64).reshape(h, w, c)

    def write(self, img: np.ndarray, path: str) -> None:
        import tempfile
        a = np.ascontiguousarray(img, dtype=np.float64)
        if a.ndim == 2:
            a = a[:, :, None]
        h, w, c = a.shape if a.size else (0, 0, 1)
        with tempfile.TemporaryDirectory() as d:
            raw = os.path.join(d, "img.f64")
            a.tofile(raw)
            self._run("write", raw, w, h, c, path)
