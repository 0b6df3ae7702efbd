"""Pins for oracle/mlp.py: printed parameter counts, closed forms, finite
differences, and the PyTorch CPU library routines (autograd, BCEWithLogits,
Adam) as independent references."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import mlp
from oracle import philox as px

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")
PAPER = json.load(open(GOLDEN))


def test_parameter_counts_printed_in_paper():
    # R4: D = [2,128,128,128,128,1], G = [6,128,128,128,128,6]
    assert mlp.count_params([6, 128, 128, 128, 128, 6]) == PAPER["gen_params"]["value"]
    assert mlp.count_params([2, 128, 128, 128, 128, 1]) == PAPER["disc_params"]["value"]
    assert mlp.count_weights([6, 128, 128, 128, 128, 6]) == 50688
    # SPEC worked examples
    assert mlp.count_params([6, 128, 128, 6]) == 18182
    # S:186 prints 38,017 for [2,192,192,1], but its own expansion
    # 2*192+192 + 192*192+192 + 192*1+1 sums to 37,825 (R26)
    assert mlp.count_params([2, 192, 192, 1]) == 2 * 192 + 192 + 192 * 192 + 192 + 192 * 1 + 1 == 37825
    assert mlp.count_weights([6, 128, 128, 6]) == 17920
    assert mlp.count_weights([8, 64, 64, 6]) == 4992
    assert mlp.count_params([8, 64, 64, 6]) == 5126 and mlp.count_params([2, 64, 64, 1]) == 4417


def test_uniform_width_d_is_unique():
    # the only uniform-width [2, H x d, 1] stack with 50,049 parameters
    sols = [(H, d) for H in range(1, 1025) for d in range(1, 9)
            if mlp.count_params([2] + [H] * d + [1]) == 50049]
    assert sols == [(128, 4)]


def test_leaky_relu_values():
    assert mlp.lrelu(np.array(2.0)) == 2.0
    assert mlp.lrelu(np.array(-2.0)) == pytest.approx(-0.02)
    assert mlp.lrelu(np.array(-5.0), 0.0) == 0.0
    assert mlp.lrelu_grad(np.array(-1.0)) == 0.01 and mlp.lrelu_grad(np.array(3.0)) == 1.0


def test_linear_identity_and_zero_input():
    W = [np.eye(2)]
    b = [np.zeros(2)]
    out, _ = mlp.forward(W, b, np.array([[3.0, 4.0]]))
    assert np.array_equal(out, [[3.0, 4.0]])
    out, _ = mlp.forward([np.random.default_rng(0).normal(size=(2, 2))], [np.array([1.0, 2.0])], np.zeros((1, 2)))
    assert np.array_equal(out, [[1.0, 2.0]])


def _rand_mlp(rng, sizes):
    Ws = [rng.normal(scale=0.5, size=(sizes[i + 1], sizes[i])) for i in range(len(sizes) - 1)]
    bs = [rng.normal(scale=0.1, size=sizes[i + 1]) for i in range(len(sizes) - 1)]
    return Ws, bs


def test_backward_matches_torch_autograd():
    rng = np.random.default_rng(1)
    sizes = [3, 7, 5, 2]
    Ws, bs = _rand_mlp(rng, sizes)
    x = rng.normal(size=(11, 3))
    dout = rng.normal(size=(11, 2))
    out, cache = mlp.forward(Ws, bs, x)
    dWs, dbs, dx = mlp.backward(Ws, cache, dout)
    tW = [torch.tensor(w, requires_grad=True) for w in Ws]
    tb = [torch.tensor(b, requires_grad=True) for b in bs]
    tx = torch.tensor(x, requires_grad=True)
    h = tx
    for l in range(len(tW)):
        h = torch.nn.functional.linear(h, tW[l], tb[l])
        if l < len(tW) - 1:
            h = torch.nn.functional.leaky_relu(h, 0.01)
    assert np.allclose(h.detach().numpy(), out, rtol=1e-14, atol=1e-14)
    h.backward(torch.tensor(dout))
    for l in range(len(tW)):
        assert np.allclose(tW[l].grad.numpy(), dWs[l], rtol=1e-12, atol=1e-13)
        assert np.allclose(tb[l].grad.numpy(), dbs[l], rtol=1e-12, atol=1e-13)
    assert np.allclose(tx.grad.numpy(), dx, rtol=1e-12, atol=1e-13)


def test_backward_finite_differences():
    rng = np.random.default_rng(2)
    sizes = [2, 6, 6, 1]
    Ws, bs = _rand_mlp(rng, sizes)
    x = rng.normal(size=(9, 2))
    t = (rng.uniform(size=9) > 0.5).astype(float)

    def loss(Ws_):
        z, _ = mlp.forward(Ws_, bs, x)
        return mlp.bce_with_logits(z[:, 0], t)

    z, cache = mlp.forward(Ws, bs, x)
    dWs, _, _ = mlp.backward(Ws, cache, mlp.bce_grad(z[:, 0], t)[:, None])
    h = 1e-6
    for l in range(len(Ws)):
        for idx in np.ndindex(Ws[l].shape):
            Wp = [w.copy() for w in Ws]; Wp[l][idx] += h
            Wm = [w.copy() for w in Ws]; Wm[l][idx] -= h
            fd = (loss(Wp) - loss(Wm)) / (2 * h)
            assert abs(fd - dWs[l][idx]) <= 1e-7 + 1e-5 * abs(fd)


def test_bce_values_and_torch():
    assert mlp.bce_with_logits(np.array([0.0]), np.array([1.0])) == pytest.approx(np.log(2.0), abs=1e-15)
    assert mlp.bce_with_logits(np.array([0.0]), np.array([0.0])) == pytest.approx(np.log(2.0), abs=1e-15)
    assert mlp.bce_with_logits(np.array([20.0]), np.array([1.0])) == pytest.approx(2.0611536e-9, rel=1e-6)
    rng = np.random.default_rng(3)
    z = rng.normal(scale=8, size=1000)
    t = (rng.uniform(size=1000) > 0.5).astype(float)
    ref = torch.nn.functional.binary_cross_entropy_with_logits(torch.tensor(z), torch.tensor(t)).item()
    assert mlp.bce_with_logits(z, t) == pytest.approx(ref, rel=1e-14)
    tz = torch.tensor(z, requires_grad=True)
    torch.nn.functional.binary_cross_entropy_with_logits(tz, torch.tensor(t)).backward()
    assert np.allclose(mlp.bce_grad(z, t), tz.grad.numpy(), rtol=1e-12, atol=1e-18)


def test_adam_matches_torch_and_fixed_points():
    # zero gradient -> unchanged
    p, m, v = mlp.adam_update(np.array([1.0]), np.array([0.0]), np.zeros(1), np.zeros(1), 1, 1e-3)
    assert p[0] == 1.0
    # first step moves by ~lr
    p, m, v = mlp.adam_update(np.array([1.0]), np.array([1.0]), np.zeros(1), np.zeros(1), 1, 1e-3)
    assert abs(1.0 - p[0] - 1e-3) < 1e-10
    # torch.optim.Adam over 5 steps with varying gradients
    rng = np.random.default_rng(4)
    p0 = rng.normal(size=20)
    grads = [rng.normal(size=20) for _ in range(5)]
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=1e-4, betas=(0.9, 0.999), eps=1e-8)
    p, m, v = p0.copy(), np.zeros(20), np.zeros(20)
    for i, g in enumerate(grads):
        tp.grad = torch.tensor(g)
        opt.step()
        p, m, v = mlp.adam_update(p, g, m, v, i + 1, 1e-4)
    assert np.allclose(p, tp.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_kaiming_std_and_determinism():
    # std = sqrt(2 / ((1 + a^2) fan_in)): fan_in = 100, a = 0.01 -> 0.14141
    Ws, bs = mlp.kaiming_init(5, px.STREAM_INIT_D, 0, [100, 400], 0.01)
    w = Ws[0].reshape(-1)
    std = np.sqrt(2.0 / ((1 + 1e-4) * 100))
    assert std == pytest.approx(0.14141, abs=1e-5)
    n = w.size
    assert abs(w.std() - std) < 4 * std / np.sqrt(2 * n)
    assert abs(w.mean()) < 4 * std / np.sqrt(n)
    assert np.all(bs[0] == 0)
    Ws2, _ = mlp.kaiming_init(5, px.STREAM_INIT_D, 0, [100, 400], 0.01)
    assert np.array_equal(Ws[0], Ws2[0])
