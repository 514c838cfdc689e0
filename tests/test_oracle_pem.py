"""Pins of the PEM oracle (BASELINE configs[4]; readings R19-R21) against things
other than itself: torch.autograd in float64 (a library routine), the closed form at W1 = 0,
central finite differences, and the flipped-decision model."""
import numpy as np
import pytest
import torch

F, H = 32, 512


def _torch_pem(f, p, g, flips=()):
    f = torch.tensor(f, dtype=torch.float64)
    g = torch.tensor(g, dtype=torch.float64)
    p = torch.tensor(p, dtype=torch.float64, requires_grad=True)
    Ff = f.shape[1]
    Hh = (p.numel() - 1) // (Ff + 2)
    W1 = p[:Hh * Ff].view(Hh, Ff)
    b1 = p[Hh * Ff:Hh * Ff + Hh]
    w2 = p[Hh * Ff + Hh:Hh * Ff + 2 * Hh]
    b2 = p[-1]
    a = f @ W1.T + b1
    mask = (a > 0).flatten()
    if len(flips):
        mask[torch.tensor(flips, dtype=torch.long)] ^= True
    h = a * mask.view_as(a).to(a.dtype)
    y = torch.sigmoid(h @ w2 + b2)
    L = ((y - g) ** 2).mean()
    L.backward()
    return L.item(), y.detach().numpy(), p.grad.numpy()


def _inputs(M, Ff, Hh, seed):
    rng = np.random.default_rng(seed)
    f = rng.random((M, Ff))
    p = rng.uniform(-1, 1, Hh * Ff + 2 * Hh + 1) / np.sqrt(Ff)
    g = rng.random(M)
    return f, p, g


def test_num_params(orc):
    assert orc.pem_num_params(32, 512) == 17409  # 17,409 parameters


@pytest.mark.parametrize("M,Ff,Hh", [(7, 5, 9), (64, 32, 512)])
def test_pem_vs_autograd(orc, M, Ff, Hh):
    f, p, g = _inputs(M, Ff, Hh, 11)
    ref = orc.pem_fwd_bwd(f, p, g)
    L, y, grad = _torch_pem(f, p, g)
    assert abs(ref["loss"] - L) <= 1e-13 * max(abs(L), 1)
    assert np.allclose(ref["y"], y, rtol=1e-13, atol=1e-15)
    assert np.allclose(ref["grad"], grad, rtol=1e-11, atol=1e-15)


def test_pem_closed_form_zero_hidden(orc):
    """W1 = 0, b1 = 0: h = 0, y = sigmoid(b2) for every proposal, L = mean (y - g)^2,
    db2 = (2/M) sum (y - g) y (1 - y), every other gradient 0 (ReLU'(0) = 0, reading R7)."""
    M = 40
    f, p, g = _inputs(M, F, H, 3)
    p[:H * F + H] = 0.0
    b2 = 0.37
    p[-1] = b2
    ref = orc.pem_fwd_bwd(f, p, g)
    y = 1.0 / (1.0 + np.exp(-b2))
    assert np.allclose(ref["y"], y, rtol=1e-15)
    assert abs(ref["loss"] - np.mean((y - g) ** 2)) <= 1e-15
    assert abs(ref["grad"][-1] - 2.0 / M * np.sum((y - g) * y * (1 - y))) <= 1e-15
    assert np.all(ref["grad"][:-1] == 0.0)


def test_pem_finite_differences(orc):
    M, Ff, Hh = 5, 4, 6
    f, p, g = _inputs(M, Ff, Hh, 5)
    ref = orc.pem_fwd_bwd(f, p, g, kink_tau=1e-6)
    h = 1e-6
    for i in range(p.size):
        if ref["nkinks"]:
            pytest.skip("kink near a decision")
        pp, pm = p.copy(), p.copy()
        pp[i] += h
        pm[i] -= h
        d = (orc.pem_fwd_bwd(f, pp, g)["loss"] - orc.pem_fwd_bwd(f, pm, g)["loss"]) / (2 * h)
        assert abs(d - ref["grad"][i]) <= 1e-6 * max(1.0, abs(d)), i


def test_pem_flips_match_masked_model(orc):
    M, Ff, Hh = 16, 8, 24
    f, p, g = _inputs(M, Ff, Hh, 9)
    flips = [3, 50, 200, 377]
    ref = orc.pem_fwd_bwd(f, p, g, flips=flips)
    L, y, grad = _torch_pem(f, p, g, flips=flips)
    assert abs(ref["loss"] - L) <= 1e-13
    assert np.allclose(ref["grad"], grad, rtol=1e-11, atol=1e-15)
    dec = ref["decisions"].reshape(M, Hh)
    a = f @ p[:Hh * Ff].reshape(Hh, Ff).T + p[Hh * Ff:Hh * Ff + Hh]
    expect = (a > 0).flatten()
    expect[flips] ^= True
    assert np.array_equal(dec.flatten().astype(bool), expect)
