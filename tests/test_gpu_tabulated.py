"""GPU parity of the tabulated-CDF sampler variant (SURVEY §8(f) row 1,
reading R32) through the C ABI: events against oracle/tabulated.py on the
same Philox uniforms (the FAKE stream, word 2e+o), and the backward against
the oracle's exact derivative of the tabulated inverse.

Tolerances: both sides build the tables in fp64 (different summation order,
~1e-15) and the events are rounded to fp32 -> 1e-6 absolute on x in [0, 1];
gradients are fp64 sums rounded to fp32 -> 1e-5 relative with a floor of
1e-6 of the largest |draw|."""
import numpy as np
import pytest

from oracle import philox as px
from oracle import proxy
from oracle import tabulated as T
from tests.gpu_util import assert_rel, lib

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


def _raw(k, seed):
    return np.random.default_rng(seed).normal(0.0, 0.9, (k, 6)).astype(np.float32)


@pytest.mark.parametrize("k,m,G", [(3, 333, 65), (5, 257, 1024), (2, 700, 2048), (4, 1, 3)])
def test_tabulated_events_match_oracle(k, m, G):
    L = lib()
    seed, step, rank = 11, 4, 1
    raw = _raw(k, k * 100 + G)
    d_raw = torch.from_numpy(raw).cuda()
    ev = torch.full((k * m, 2), float("nan"), device="cuda")
    L.sample_tabulated(d_raw.data_ptr(), k, m, G, seed, step, rank, px.STREAM_FAKE, ev.data_ptr(), _stream())
    torch.cuda.synchronize()
    u = proxy.fake_uniforms(seed, step, rank, k * m)
    ref = T.sample_events(raw.astype(np.float64), m, u, G)
    got = ev.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(got)) and got.min() >= 0.0 and got.max() <= 1.0
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-6)


@pytest.mark.parametrize("k,m,G", [(3, 333, 65), (4, 300, 1024), (2, 129, 2048)])
def test_tabulated_backward_matches_oracle(k, m, G):
    L = lib()
    seed, step, rank = 5, 2, 0
    raw = _raw(k, 7 + G)
    dy = np.random.default_rng(G).normal(size=(k * m, 2)).astype(np.float32)
    d_raw, d_dy = torch.from_numpy(raw).cuda(), torch.from_numpy(dy).cuda()
    d_draw = torch.full((k, 6), float("nan"), device="cuda")
    L.sample_tabulated_bwd(d_raw.data_ptr(), k, m, G, seed, step, rank, px.STREAM_FAKE, d_dy.data_ptr(),
                           d_draw.data_ptr(), _stream())
    torch.cuda.synchronize()
    u = proxy.fake_uniforms(seed, step, rank, k * m)
    ref = T.sampler_backward(raw.astype(np.float64), m, u, dy.astype(np.float64), G)
    got = d_draw.cpu().numpy().astype(np.float64)
    assert_rel(got, ref, 1e-5, 1e-6 * np.max(np.abs(ref)), "tabulated draw")


def test_tabulated_rejects_bad_args():
    L = lib()
    raw = torch.zeros(2, 6, device="cuda")
    ev = torch.zeros(64, 2, device="cuda")
    for (k, m, G) in ((0, 4, 65), (2, 0, 65), (2, 4, 2), (2, 4, 2049)):
        with pytest.raises(L.SagipsError):
            L.sample_tabulated(raw.data_ptr(), k, m, G, 1, 0, 0, 5, ev.data_ptr(), _stream())
        with pytest.raises(L.SagipsError):
            L.sample_tabulated_bwd(raw.data_ptr(), k, m, G, 1, 0, 0, 5, ev.data_ptr(), raw.data_ptr(), _stream())
