"""Pins for the oracle's BSN-TEM forward / loss / backward (no GPU).

Independent references: torch.nn.functional.conv1d (float64, a library
routine), torch.autograd (float64), central finite differences, the loss's
closed form at z == 0, and the data-parallel identity.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import datagen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def tiny(B=2, T=5, Cin=4, C=6, Co=3, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, T, Cin)).astype(np.float32)
    K = C * 3 * Cin + C + C * 3 * C + C + Co * C + Co
    p = (rng.standard_normal(K) * 0.5).astype(np.float32)
    lab = rng.uniform(0, 1, size=(B, Co, T)).astype(np.float32)
    return x, p, lab


def split(p, Cin, C, Co):
    o = 0
    out = {}
    for name, shp in (("W1", (C, 3, Cin)), ("b1", (C,)), ("W2", (C, 3, C)), ("b2", (C,)),
                      ("W3", (Co, C)), ("b3", (Co,))):
        n = int(np.prod(shp))
        out[name] = p[o:o + n].reshape(shp)
        o += n
    return out


def torch_reference(x, p, lab, lam, Cin, C, Co):
    """Independent float64 model with torch conv1d + autograd.  The loss is written as
    weighted BCE-with-logits (torch's own stable routine)."""
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in split(p, Cin, C, Co).items()}
    xt = torch.tensor(x, dtype=torch.float64).permute(0, 2, 1)  # [B][Cin][T]
    h1 = F.relu(F.conv1d(xt, P["W1"].permute(0, 2, 1), P["b1"], padding=1))
    h2 = F.relu(F.conv1d(h1, P["W2"].permute(0, 2, 1), P["b2"], padding=1))
    z = F.conv1d(h2, P["W3"].unsqueeze(-1), P["b3"])  # [B][Co][T]
    g = torch.tensor(lab, dtype=torch.float64)
    b = (g > 0.5).double()
    T = x.shape[1]
    lpos = b.sum(-1, keepdim=True)
    lneg = T - lpos
    ap = T / lpos.clamp(min=1)
    an = T / lneg.clamp(min=1)
    # -(a+ b log p + a- (1-b) log(1-p)) == BCEwithlogits with pos_weight-like per-element weights
    w = ap * b + an * (1 - b)
    per = F.binary_cross_entropy_with_logits(z, b, weight=w, reduction="none")  # [B][Co][T]
    Lo = per.mean(-1)  # [B][Co]
    lamt = torch.tensor(lam, dtype=torch.float64)
    L = (Lo * lamt).sum(-1).mean()
    L.backward()
    grad = torch.cat([P[k].grad.reshape(-1) for k in ("W1", "b1", "W2", "b2", "W3", "b3")])
    return L.item(), Lo.mean(0).detach().numpy(), z.permute(0, 2, 1).detach().numpy(), grad.numpy()


def test_forward_matches_torch_conv1d_and_autograd(orc):
    Cin, C, Co = 4, 6, 3
    lam = (2.0, 1.0, 0.5)
    for seed in range(3):
        x, p, lab = tiny(seed=seed)
        r = orc.tem_fwd_bwd(x, p, lab, lam, prec=0, C=C)
        L, Lo, z, grad = torch_reference(x, p, lab, lam, Cin, C, Co)
        assert np.allclose(r["z"], z, rtol=1e-12, atol=1e-12)
        assert abs(r["loss"][0] - L) <= 1e-12 * max(1.0, abs(L))
        assert np.allclose(r["loss"][1:], Lo, rtol=1e-12, atol=1e-13)
        assert np.allclose(r["grad"], grad, rtol=1e-10, atol=1e-12)


def test_forward_full_shape_vs_torch(orc):
    """Full channel widths (400->512->512->3), T=100, one video."""
    x = datagen.features(1, rank=0, batch_idx=3)
    p = datagen.init_params()
    lab = datagen.labels(1, rank=0, batch_idx=3)
    r = orc.tem_fwd_bwd(x, p, lab, prec=0)
    L, Lo, z, grad = torch_reference(x, p, lab, (1.0, 1.0, 1.0), 400, 512, 3)
    assert np.allclose(r["z"], z, rtol=1e-10, atol=1e-11)
    assert abs(r["loss"][0] - L) < 1e-10
    scale = np.abs(grad).max()
    assert np.abs(r["grad"] - grad).max() <= 1e-10 * scale


def test_zero_weights_gives_relu_bias(orc):
    """W = 0 -> h = ReLU(b): z = b3 + W3 . ReLU(b2) independent of x."""
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny()
    P = split(p.copy(), Cin, C, Co)
    P["W1"][:] = 0
    P["W2"][:] = 0
    flat = np.concatenate([P[k].ravel() for k in ("W1", "b1", "W2", "b2", "W3", "b3")])
    r = orc.tem_fwd_bwd(x, flat, lab, prec=0, C=C)
    expect = P["b3"].astype(np.float64) + P["W3"].astype(np.float64) @ np.maximum(P["b2"], 0).astype(np.float64)
    assert np.allclose(r["z"], np.broadcast_to(expect, r["z"].shape), rtol=0, atol=1e-14)


def test_loss_closed_form_at_zero_logits(orc):
    """W3 = 0, b3 = 0 -> z == 0 -> L_o = 2 ln 2 per channel (both classes present),
    and sum_t dz = 0 per (video, channel) -> db3 == 0."""
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))["loss_at_zero_logits"]
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(T=8)
    lab[:, :, :3] = 0.9  # at least one positive and one negative per channel
    lab[:, :, 3:] = 0.1
    P = split(p.copy(), Cin, C, Co)
    P["W3"][:] = 0
    P["b3"][:] = 0
    flat = np.concatenate([P[k].ravel() for k in ("W1", "b1", "W2", "b2", "W3", "b3")])
    lam = (2.0, 1.0, 1.0)
    r = orc.tem_fwd_bwd(x, flat, lab, lam, prec=0, C=C)
    assert np.allclose(r["loss"][1:], gold["per_channel"], rtol=0, atol=1e-14)
    assert abs(r["loss"][0] - gold["per_channel"] * sum(lam)) < 1e-13
    sl = orc.param_slices(Cin, C, Co)
    assert np.allclose(r["grad"][sl["b3"]], 0.0, atol=1e-15)
    # the '1/2-factor' variant would give ln 2: make sure we are not it
    assert abs(r["loss"][1] - math.log(2)) > 0.5


def test_threshold_is_strict(orc):
    """Reading R5: b = [g > 0.5] strictly; g = 0.5 is negative."""
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(T=6)
    lab2 = lab.copy()
    lab[:] = 0.5
    lab2[:] = 0.0
    r1 = orc.tem_fwd_bwd(x, p, lab, prec=0, C=C)
    r2 = orc.tem_fwd_bwd(x, p, lab2, prec=0, C=C)
    assert np.array_equal(r1["loss"], r2["loss"]) and np.array_equal(r1["grad"], r2["grad"])


def test_finite_differences(orc):
    """Central differences on the fp64 oracle (h = 1e-6), skipping coordinates near a ReLU kink."""
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(seed=7)
    lam = (2.0, 1.0, 1.0)
    p64 = p.astype(np.float64)
    r = orc.tem_fwd_bwd(x, p64, lab, lam, prec=0, C=C)
    h = 1e-6
    rng = np.random.default_rng(0)
    idx = np.unique(np.concatenate([rng.choice(p.size, 60, replace=False),
                                    np.arange(p.size - 3 * C - 3, p.size)]))
    checked = 0
    for i in idx:
        pp = p64.copy(); pp[i] += h
        pm = p64.copy(); pm[i] -= h
        lp = orc.tem_fwd_bwd(x, pp, lab, lam, prec=0, C=C)["loss"][0]
        lm = orc.tem_fwd_bwd(x, pm, lab, lam, prec=0, C=C)["loss"][0]
        # kink check: the second difference is large near a ReLU switch
        l0 = r["loss"][0]
        if abs(lp - 2 * l0 + lm) > 1e-7:
            continue
        fd = (lp - lm) / (2 * h)
        assert abs(fd - r["grad"][i]) <= 1e-6 * max(1.0, abs(fd)), (i, fd, r["grad"][i])
        checked += 1
    assert checked > 50


def test_relu_decision_flips_match_autograd_with_explicit_masks(orc):
    """Reading R7b: inverting chosen ReLU decisions equals an independent torch float64 model
    whose ReLU is the mask (a > 0) XOR flip, differentiated by autograd."""
    Cin, C, Co = 4, 6, 3
    B, T = 2, 5
    x, p, lab = tiny(B=B, T=T, seed=3)
    lam = (2.0, 1.0, 1.0)
    base = orc.tem_fwd_bwd(x, p, lab, lam, prec=0, C=C, kink_tau=1.0, kinks_cap=10 ** 5)
    n = B * T * C
    assert base["nkinks"] == 2 * n  # tau = 1 reports every pre-activation
    rng = np.random.default_rng(0)
    flips = np.sort(rng.choice(2 * n, 7, replace=False))
    r = orc.tem_fwd_bwd(x, p, lab, lam, prec=0, C=C, flips=flips)
    fl = np.zeros(2 * n, bool)
    fl[flips] = True
    F1 = torch.tensor(fl[:n].reshape(B, T, C)).permute(0, 2, 1)
    F2 = torch.tensor(fl[n:].reshape(B, T, C)).permute(0, 2, 1)
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in split(p, Cin, C, Co).items()}
    xt = torch.tensor(x, dtype=torch.float64).permute(0, 2, 1)
    a1 = F.conv1d(xt, P["W1"].permute(0, 2, 1), P["b1"], padding=1)
    m1 = ((a1 > 0) ^ F1).double()
    h1 = a1 * m1
    a2 = F.conv1d(h1, P["W2"].permute(0, 2, 1), P["b2"], padding=1)
    m2 = ((a2 > 0) ^ F2).double()
    h2 = a2 * m2
    dec = torch.cat([m1.permute(0, 2, 1).reshape(-1), m2.permute(0, 2, 1).reshape(-1)]).numpy().astype(np.uint8)
    assert np.array_equal(r["decisions"], dec)
    z = F.conv1d(h2, P["W3"].unsqueeze(-1), P["b3"])
    b = (torch.tensor(lab, dtype=torch.float64) > 0.5).double()
    lpos = b.sum(-1, keepdim=True)
    w = (T / lpos.clamp(min=1)) * b + (T / (T - lpos).clamp(min=1)) * (1 - b)
    L = (F.binary_cross_entropy_with_logits(z, b, weight=w, reduction="none").mean(-1)
         * torch.tensor(lam, dtype=torch.float64)).sum(-1).mean()
    L.backward()
    grad = torch.cat([P[k].grad.reshape(-1) for k in ("W1", "b1", "W2", "b2", "W3", "b3")]).numpy()
    assert np.allclose(r["grad"], grad, rtol=1e-10, atol=1e-12)
    assert abs(r["loss"][0] - L.item()) < 1e-12
    assert not np.allclose(r["grad"], base["grad"])  # the flips matter
    # no flips and tau = 0: identical to the plain entry point
    plain = orc.tem_fwd_bwd(x, p, lab, lam, prec=0, C=C)
    assert np.array_equal(plain["grad"], base["grad"]) and plain["nkinks"] == 0


def test_data_parallel_identity(orc):
    """N ranks x B with Mean == 1 rank x N*B (per-video alpha)."""
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(B=6, seed=9)
    full = orc.tem_fwd_bwd(x, p, lab, prec=0, C=C)
    for N in (2, 3):
        B = 6 // N
        parts = [orc.tem_fwd_bwd(x[r * B:(r + 1) * B], p, lab[r * B:(r + 1) * B], prec=0, C=C)
                 for r in range(N)]
        g = sum(q["grad"] for q in parts) / N
        L = sum(q["loss"][0] for q in parts) / N
        assert np.allclose(g, full["grad"], rtol=0, atol=1e-12 * np.abs(full["grad"]).max())
        assert abs(L - full["loss"][0]) < 1e-12


def test_bf16_emulation_rounds_operands(orc):
    """prec=1 equals prec=0 on inputs whose operands are already bf16-exact and whose
    intermediate h1/dA are exactly representable: here all-integers small enough."""
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(seed=2)
    xb = orc.bf16_round(x)
    r0 = orc.tem_fwd_bwd(x, p, lab, prec=0, C=C)
    r1 = orc.tem_fwd_bwd(x, p, lab, prec=1, C=C)
    # bf16 emulation differs from fp64, but only at bf16 rounding level
    rel = np.abs(r1["grad"] - r0["grad"]).max() / np.abs(r0["grad"]).max()
    assert 0 < rel < 3e-2
    # x pre-rounded -> rounding x again is a no-op: same result
    r1b = orc.tem_fwd_bwd(xb, p, lab, prec=1, C=C)
    assert np.array_equal(r1["grad"], r1b["grad"])
    # bf16 RNE bit rule spot checks (1 + 2^-8 ties to even 1.0; 1 + 3*2^-8 -> 1 + 2^-6)
    v = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 65504.0], np.float32)
    assert list(orc.bf16_round(v)) == [1.0, 1.0 + 2 ** -6, -2.5, 65536.0]


def test_empty_batch(orc):
    x = np.zeros((0, 5, 4), np.float32)
    _, p, _ = tiny()
    r = orc.tem_fwd_bwd(x, p, np.zeros((0, 3, 5), np.float32), prec=0, C=6)
    assert np.all(r["grad"] == 0) and np.all(r["loss"] == 0)


def test_threaded_split_equals_one_call(orc):
    """tem_fwd_bwd(threads=n) merges per-sub-batch calls: same decisions, kinks and flips
    as one call, values equal up to fp64 summation order."""
    Cin, C, Co = 4, 6, 3
    for prec, B, ns in ((0, 7, (2, 3, 7)), (1, 8, (2, 3, 4, 8))):
        _split_case(orc, prec, B, ns)


def _split_case(orc, prec, B, ns):
    Cin, C, Co = 4, 6, 3
    x, p, lab = tiny(B=B, T=9, seed=11)
    lam = (2.0, 1.0, 0.5)
    one = orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, C=C, kink_tau=(0.05, 0.2), kinks_cap=10 ** 5)
    assert one["nkinks"] > 0
    rng = np.random.default_rng(1)
    flips = np.sort(rng.choice(2 * B * 9 * C, 9, replace=False))
    one_f = orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, C=C, flips=flips)
    for n in ns:
        par = orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, C=C, kink_tau=(0.05, 0.2), kinks_cap=10 ** 5, threads=n)
        assert np.array_equal(par["decisions"], one["decisions"])
        assert np.array_equal(par["kinks"], np.sort(one["kinks"])) and par["nkinks"] == one["nkinks"]
        assert np.array_equal(par["z"], one["z"])
        assert np.allclose(par["loss"], one["loss"], rtol=1e-14, atol=0)
        assert np.abs(par["grad"] - one["grad"]).max() <= 1e-14 * np.abs(one["grad"]).max()
        par_f = orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, C=C, flips=flips, threads=n)
        assert np.array_equal(par_f["decisions"], one_f["decisions"])
        assert np.abs(par_f["grad"] - one_f["grad"]).max() <= 1e-14 * np.abs(one_f["grad"]).max()


def test_layer_bands_are_separate(orc):
    """kink_tau=(t1, t2): a1 indices reported with band t1, a2 indices with band t2."""
    Cin, C, Co = 4, 6, 3
    B, T = 2, 5
    x, p, lab = tiny(B=B, T=T, seed=3)
    n = B * T * C
    only1 = orc.tem_fwd_bwd(x, p, lab, prec=0, C=C, kink_tau=(1.0, 0.0), kinks_cap=10 ** 5)
    only2 = orc.tem_fwd_bwd(x, p, lab, prec=0, C=C, kink_tau=(0.0, 1.0), kinks_cap=10 ** 5)
    assert only1["nkinks"] == n and np.all(only1["kinks"] < n)
    assert only2["nkinks"] == n and np.all(only2["kinks"] >= n)
