"""Device API hardening (GPU): weight edge cases that must not turn into NaN,
caller-supplied tensors checked before their pointers reach the kernels,
kernels launched on the tensors' device, and the bounded CUDA-graph cache."""
import numpy as np
import pytest

import paper_1705_01674_b200 as S

pytestmark = pytest.mark.gpu


def _flat_patch(h=48, w=40, seed=3):
    rng = np.random.default_rng(seed)
    g = np.full((h, w), 0.5, np.float32)
    g[:, w // 2:] = 0.25            # two exactly flat regions: range = 0 on most edges
    g[h // 3, :] += 0.1
    t = np.clip(g + rng.normal(0, 0.05, (h, w)), 0, 1).astype(np.float32)
    return t, g


@pytest.mark.parametrize("r,tau", [(1, 1), (2, 3)])
def test_frac_alpha_r_zero_flat_guidance(r, tau, port):
    """alpha_r = 0: (range)^0 = 1 even for range = 0, like std::pow(0, 0)
    (proj/src/weights.cpp:67-71) -- no 0 * -inf = NaN."""
    t, g = _flat_patch()
    cfg = S.SmoothConfig(lambda_=50.0, r=r, tau=tau, iterations=2,
                         weight=S.WeightParams(kind=S.WeightKind.Frac, alpha_r=0.0))
    got = S.smooth(t, g, cfg)
    want = port.smooth(t, g, cfg)
    assert np.isfinite(got).all()
    assert float(np.abs(got - want).max()) <= 1e-4


def test_exp_overflowing_exponent_flat_guidance(port):
    """A range exponent beyond float range (huge guidance_scale / tiny sigma_r)
    must still give weight 1 on flat edges and 0 elsewhere."""
    t, g = _flat_patch()
    cfg = S.SmoothConfig(lambda_=400.0, r=2, tau=2, iterations=2,
                         weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=1e-30, guidance_scale=1e10))
    got = S.smooth(t, g, cfg)
    want = port.smooth(t, g, cfg)
    assert np.isfinite(got).all()
    assert float(np.abs(got - want).max()) <= 1e-4


def test_device_inputs_are_checked():
    import torch

    t = torch.rand(32, 24, device="cuda")
    with pytest.raises(S.Error, match="contiguous float32"):
        S.smooth_device(t.double(), t)
    with pytest.raises(S.Error, match="contiguous float32"):
        S.smooth_device(t.t(), t.t())
    with pytest.raises(S.Error, match="expected shape"):
        S.smooth_device(t, t, out=torch.empty(32, 23, device="cuda"))
    with pytest.raises(S.Error, match="contiguous float32"):
        S.smooth_device(t, t, out=torch.empty(32, 24, device="cuda", dtype=torch.float16))
    v = torch.zeros(2, 32, 24, device="cuda")
    m = torch.zeros(2, 32, 24, device="cuda")
    with pytest.raises(S.Error, match="values/mask size mismatch"):
        S.interpolate_sparse_device(v, m[:1].contiguous(), v)
    with pytest.raises(S.Error, match="contiguous float32"):
        S.interpolate_sparse_device(v, m.bool(), v)
    with pytest.raises(S.Error, match="guidance dimensions differ"):
        S.interpolate_sparse_device(v, m, torch.zeros(2, 32, 25, device="cuda"))
    with pytest.raises(S.Error, match="expected shape"):
        S.interpolate_sparse_device(v, m, v, undefined=torch.empty(2, 32, 23, device="cuda"))
    with pytest.raises(S.Error, match="expected shape"):
        S.interpolate_sparse_device(v, m, v, out=torch.empty(1, 32, 24, device="cuda"))


def test_device_mismatch_is_rejected():
    import torch

    if torch.cuda.device_count() < 2:
        t = torch.rand(16, 16, device="cuda")
        with pytest.raises(S.Error, match="CUDA tensor|must be on"):
            S.smooth_device(t, t.cpu())
        return
    a = torch.rand(16, 16, device="cuda:0")
    b = torch.rand(16, 16, device="cuda:1")
    with pytest.raises(S.Error, match="must be on"):
        S.smooth_device(a, b)


def test_graph_cache_is_bounded():
    import torch

    S.graph_clear()
    t = torch.rand(24, 20, device="cuda")
    cfg = S.SmoothConfig(lambda_=100.0, r=1, tau=1, iterations=2)
    ref = S.smooth_device(t, t, cfg, sync=True)
    outs = [torch.empty_like(t) for _ in range(70)]  # 70 distinct keys (output pointers)
    for o in outs:
        S.smooth_device(t, t, cfg, out=o, graph=True)
    torch.cuda.synchronize()
    assert S.graph_count() <= 64
    for o in outs:
        assert torch.equal(o, ref)
    n = S.graph_clear()
    assert n == S.graph_count() + n and S.graph_count() == 0


# ------------------------------------------------ host batches: pipeline + aliasing

def _scene(h, w, seed):
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:h, 0:w]
    g = (0.2 + 0.25 * ((x // 97 + y // 61) % 3) + rng.normal(0, 0.02, (h, w))).astype(np.float32)
    return np.clip(g, 0, 1)


def test_self_guided_call_uploads_once_same_result():
    """smooth(img, img, cfg) (proj/src/apps.cpp:59): one host buffer for target and guidance
    is uploaded once; the result is bit-identical to two separate buffers"""
    t = _scene(300, 260, 1)
    cfg = S.SmoothConfig(lambda_=400.0, r=2, tau=3, weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.05))
    a = S.smooth(t, t, cfg)
    b = S.smooth(t, t.copy(), cfg)
    assert np.array_equal(a, b)


def test_host_batch_pipeline_equals_single_calls():
    """Larger host batches run as upload / filter / download stages over sub-batches
    (6 images of 1 MPix: three sub-batches of 2): bit-identical to the single calls"""
    cfg = S.SmoothConfig(lambda_=400.0, r=2, tau=2, weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.05))
    t = np.stack([_scene(1024, 1024, 10 + i) for i in range(6)])
    g = np.stack([_scene(1024, 1024, 20 + i) for i in range(6)])
    got = S.smooth_batch(t, g, cfg)
    for i in (0, 4, 5):
        assert np.array_equal(got[i], S.smooth(t[i], g[i], cfg)), i
    # sparse: values / mask / guidance triples, the undefined mask too
    rng = np.random.default_rng(5)
    m = (rng.uniform(size=t.shape) < 1 / 16).astype(np.float32)
    v = (t * m).astype(np.float32)
    out, und = S.interpolate_sparse_batch(v, m, g, cfg)
    for i in (0, 5):
        o1, u1 = S.interpolate_sparse(S.SparseField(v[i], m[i]), g[i], cfg, return_undefined=True)
        assert np.array_equal(out[i], o1.reshape(out[i].shape)) and np.array_equal(und[i], u1.reshape(und[i].shape)), i


def test_host_batch_pipeline_reports_first_failing_pair():
    """Errors of a pipelined batch: the first failing pair in batch order decides, field
    checks before the pivot failure of the same sub-batch (proj/src/smoother.cpp:129-144)"""
    cfg = S.SmoothConfig(lambda_=400.0, r=2, tau=2, weight=S.WeightParams(kind=S.WeightKind.Exp, sigma_r=0.05))
    g = np.stack([_scene(1024, 1024, 30 + i) for i in range(6)])
    rng = np.random.default_rng(6)
    m = (rng.uniform(size=g.shape) < 1 / 16).astype(np.float32)
    v = (g * m).astype(np.float32)
    m2, v2 = m.copy(), v.copy()
    m2[5] = 0.0
    v2[5] = 0.0                                   # pair 5: empty mask
    with pytest.raises(S.Error, match="interpolate_sparse: empty mask"):
        S.interpolate_sparse_batch(v2, m2, g, cfg)
    m2[3, 17, 19] = 0.5                           # pair 3: not 0/1 -> decides before pair 5
    with pytest.raises(S.Error, match="interpolate_sparse: mask must be 0/1"):
        S.interpolate_sparse_batch(v2, m2, g, cfg)
    v3 = v.copy()
    v3[5, 100, 100] = 0.25 if m[5, 100, 100] == 0 else v3[5, 100, 100]
    m3 = m.copy()
    m3[5, 100, 100] = 0.0
    v3[5, 100, 100] = 0.25                        # value outside the mask, second sub-batch
    with pytest.raises(S.Error, match="interpolate_sparse: values nonzero outside mask"):
        S.interpolate_sparse_batch(v3, m3, g, cfg)
    gb = g.copy()
    gb[5, 300, 400] = np.nan                      # NaN guidance: the reference's pivot failure
    with pytest.raises(S.Error, match="non-positive pivot"):
        S.interpolate_sparse_batch(v, m, gb, cfg)
    with pytest.raises(S.Error, match="non-positive pivot"):
        S.smooth_batch(v, gb, cfg)
