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
