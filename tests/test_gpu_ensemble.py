"""GPU parity of the ensemble analysis (§8(f) rows 2 and 4, through the C
ABI): sagips_predict_params against the oracle generator forward + constrain
(R1), sagips_ensemble_stats against oracle/ensemble.py (Eq. 6-8,
P:313-332).

Tolerances: predictions are fp32 products of an fp32 MLP -> 1e-5 relative
(floor 1e-6 of the largest |c|), as the step's fp32 outputs; the ensemble
statistics sum in fp64 on both sides over the same fp32 inputs -> 1e-12."""
import numpy as np
import pytest

from oracle import ensemble as E
from oracle import gan, mlp, proxy
from tests.gpu_util import assert_rel, flat, lib, oracle_config, unflat

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()


def _stream():
    import ctypes
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("preset,k", [(0, 64), (0, 13), (1, 64), (1, 61)])
def test_predict_params_matches_oracle(preset, k):
    # desk widths (64: the generic kernel path) and paper widths (128: the
    # blocked path); k = 13 / 61 leave a ragged last row block
    from paper_2407_00051_b200 import runtime
    L = lib()
    cfg = L.config_init(preset, rank=0, param_samples=64, events_per_sample=16)
    ctx = runtime.make_context(cfg)
    st = gan.RankState(oracle_config(cfg), 0)
    rng = np.random.default_rng(7 + k)
    # random weights and non-zero biases (the init has zero biases)
    gW = [w + 0.05 * rng.standard_normal(w.shape) for w in st.gW]
    gb = [0.1 * rng.standard_normal(b.shape) for b in st.gb]
    vW, vb = flat(gW).astype(np.float32), flat(gb).astype(np.float32)
    ctx.set(L.T_GEN_W, vW)
    ctx.set(L.T_GEN_B, vb)
    gW, gb = unflat(vW.astype(np.float64), gW), unflat(vb.astype(np.float64), gb)
    noise = rng.standard_normal((k, cfg.noise_dim)).astype(np.float32)
    d_noise = torch.from_numpy(noise).cuda()
    d_c = torch.full((k, 6), float("nan"), device="cuda")
    ctx.predict_params(d_noise.data_ptr(), k, d_c.data_ptr(), _stream())
    torch.cuda.synchronize()
    raw, _ = mlp.forward(gW, gb, noise.astype(np.float64), cfg.leaky_slope)
    ref = proxy.constrain(raw).reshape(k, 6)
    got = d_c.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got))
    assert_rel(got, ref, 1e-5, 1e-6 * np.max(np.abs(ref)), "predict_params")


def test_predict_params_rejects_bad_args():
    from paper_2407_00051_b200 import runtime
    L = lib()
    cfg = L.config_init(0, rank=0, param_samples=16, events_per_sample=8)
    ctx = runtime.make_context(cfg)
    buf = torch.zeros(64, 8, device="cuda")
    for k in (0, 17):
        with pytest.raises(L.SagipsError):
            ctx.predict_params(buf.data_ptr(), k, buf.data_ptr(), _stream())


@pytest.mark.parametrize("M,k,P", [(1, 1, 1), (5, 1000, 6), (8, 1024, 6), (3, 257, 16)])
def test_ensemble_stats_matches_oracle(M, k, P):
    L = lib()
    rng = np.random.default_rng(M * 1000 + k)
    preds = (rng.standard_normal((M, k, P)) * rng.uniform(0.1, 3.0, P) + rng.uniform(-2, 2, P)).astype(np.float32)
    p_true = rng.uniform(0.5, 2.0, P) * np.where(rng.random(P) < 0.5, -1.0, 1.0)
    d = torch.from_numpy(preds).cuda()
    p_hat, sigma, r_hat = L.ensemble_stats(d.data_ptr(), M, k, P, p_true, _stream())
    o_hat, o_sig = E.ensemble_response(preds.astype(np.float64))
    np.testing.assert_allclose(p_hat, o_hat, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(sigma, o_sig, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r_hat, E.normalized_residual(p_true, o_hat), rtol=1e-12, atol=1e-14)


def test_ensemble_stats_closed_forms_and_errors():
    L = lib()
    # two members x +- d: p_hat = x, sigma = |d| exactly representable
    x = np.array([[1.0, -2.0], [0.5, 4.0]], dtype=np.float32)
    dd = np.array([[0.5, 0.25], [2.0, 0.75]], dtype=np.float32)
    d = torch.from_numpy(np.stack([x + dd, x - dd])).cuda()
    p_hat, sigma, r_hat = L.ensemble_stats(d.data_ptr(), 2, 2, 2, None, _stream())
    np.testing.assert_array_equal(p_hat, x.mean(axis=0))
    np.testing.assert_array_equal(sigma, np.abs(dd).mean(axis=0))
    assert np.all(np.isnan(r_hat))
    for args in ((0, 2, 2), (2, 0, 2), (2, 2, 0), (2, 2, 17)):
        with pytest.raises(L.SagipsError):
            L.ensemble_stats(d.data_ptr(), *args, None, _stream())
