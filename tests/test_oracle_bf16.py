"""Pin for the oracle's bf16-operand emulation (prec=1, reading R8; configs[2]).

R8 rounds exactly the tensor-core operands to bf16 (RNE, through fp32): x, W1, W2 (forward),
h1 (operand of conv2 and of conv2 wgrad), dA2 (operand of conv2 dgrad / wgrad) and dA1 (operand
of conv1 wgrad).  h2 stays fp32 (it never leaves the conv2 epilogue), and so do W3, z, p, dz
and every gradient.

The independent reference is a float64 torch model (F.conv1d + autograd) with torch's own
fp32 -> bf16 cast applied at exactly those six points: forward casts on x, W1, W2, h1 with a
straight-through gradient, and backward-only casts on the gradients arriving at a2 and a1
(dA2 = 1[a2>0] * W3^T dz, dA1 = 1[a1>0] * conv2^T dA2).  The oracle must match it to fp64
rounding.  Seven mutants of that model -- each drops one of the six rounding points, or also
rounds h2 -- must each miss the oracle by far more than the match tolerance, so a dropped or
misplaced rounding point in the oracle cannot pass.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

POINTS = ("x", "W1", "W2", "h1", "dA2", "dA1")
MUTANTS = tuple(f"drop_{p}" for p in POINTS) + ("round_h2",)
MATCH = 1e-10   # per-tensor relative: fp64 summation-order differences only
MISS = 1e-5     # every mutant must miss at least one tensor by more than this


def bf16(t):
    """torch's fp32 -> bf16 cast (RNE), through fp32 as the GPU rounds its fp32 accumulators."""
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


class _RoundFwd(torch.autograd.Function):
    """Forward bf16 cast, straight-through gradient (an operand rounded where it enters a GEMM)."""
    @staticmethod
    def forward(ctx, t):
        return bf16(t)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundBwd(torch.autograd.Function):
    """Identity forward; the gradient flowing back through it is cast to bf16 (dA operands)."""
    @staticmethod
    def forward(ctx, t):
        return t.clone()

    @staticmethod
    def backward(ctx, g):
        return bf16(g)


def split(p, Cin, C, Co):
    o, out = 0, {}
    for name, shp in (("W1", (C, 3, Cin)), ("b1", (C,)), ("W2", (C, 3, C)), ("b2", (C,)),
                      ("W3", (Co, C)), ("b3", (Co,))):
        n = int(np.prod(shp))
        out[name] = p[o:o + n].reshape(shp)
        o += n
    return out


def torch_bf16_model(x, p, lab, lam, Cin, C, Co, mutant=None):
    pts = set(POINTS)
    if mutant and mutant.startswith("drop_"):
        pts.discard(mutant[5:])
    fwd = lambda name, t: _RoundFwd.apply(t) if name in pts else t  # noqa: E731
    bwd = lambda name, t: _RoundBwd.apply(t) if name in pts else t  # noqa: E731
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in split(p, Cin, C, Co).items()}
    xt = fwd("x", torch.tensor(x, dtype=torch.float64)).permute(0, 2, 1)  # [B][Cin][T]
    a1 = F.conv1d(xt, fwd("W1", P["W1"]).permute(0, 2, 1), P["b1"], padding=1)
    h1 = fwd("h1", F.relu(bwd("dA1", a1)))
    a2 = F.conv1d(h1, fwd("W2", P["W2"]).permute(0, 2, 1), P["b2"], padding=1)
    h2 = F.relu(bwd("dA2", a2))
    if mutant == "round_h2":
        h2 = _RoundFwd.apply(h2)
    z = F.conv1d(h2, P["W3"].unsqueeze(-1), P["b3"])  # [B][Co][T]
    b = (torch.tensor(lab, dtype=torch.float64) > 0.5).double()
    T = x.shape[1]
    lpos = b.sum(-1, keepdim=True)
    w = (T / lpos.clamp(min=1)) * b + (T / (T - lpos).clamp(min=1)) * (1 - b)
    Lo = F.binary_cross_entropy_with_logits(z, b, weight=w, reduction="none").mean(-1)
    L = (Lo * torch.tensor(lam, dtype=torch.float64)).sum(-1).mean()
    L.backward()
    grad = torch.cat([P[k].grad.reshape(-1) for k in ("W1", "b1", "W2", "b2", "W3", "b3")]).numpy()
    return {"loss": np.concatenate([[L.item()], Lo.mean(0).detach().numpy()]),
            "z": z.permute(0, 2, 1).detach().numpy(), "grad": grad}


def worst_rel(orc, r, m, Cin, C, Co):
    """max over tensors (loss, z, each parameter gradient) of max|a-b| / max|b|."""
    errs = {"loss": np.abs(r["loss"] - m["loss"]).max() / np.abs(m["loss"]).max(),
            "z": np.abs(r["z"] - m["z"]).max() / np.abs(m["z"]).max()}
    for name, s in orc.param_slices(Cin, C, Co).items():
        errs[name] = np.abs(r["grad"][s] - m["grad"][s]).max() / max(np.abs(m["grad"][s]).max(), 1e-300)
    return max(errs.values()), errs


def inputs(B, T, Cin, C, Co, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((B, T, Cin)).astype(np.float32)
    K = C * 3 * Cin + C + C * 3 * C + C + Co * C + Co
    p = (rng.standard_normal(K) * (1.0 / np.sqrt(3 * Cin))).astype(np.float32)
    lab = rng.uniform(0, 1, size=(B, Co, T)).astype(np.float32)
    return x, p, lab


SHAPES = [(2, 5, 4, 6, 3, 0), (2, 16, 40, 48, 3, 1), (1, 24, 64, 32, 3, 2)]


@pytest.mark.parametrize("B,T,Cin,C,Co,seed", SHAPES)
def test_oracle_bf16_matches_torch_rounding_model(orc, B, T, Cin, C, Co, seed):
    x, p, lab = inputs(B, T, Cin, C, Co, seed)
    lam = (2.0, 1.0, 0.5)
    r = orc.tem_fwd_bwd(x, p, lab, lam, prec=1, C=C)
    worst, errs = worst_rel(orc, r, torch_bf16_model(x, p, lab, lam, Cin, C, Co), Cin, C, Co)
    assert worst <= MATCH, errs


@pytest.mark.parametrize("mutant", MUTANTS)
def test_each_rounding_point_is_load_bearing(orc, mutant):
    """A model missing any one rounding point (or rounding h2 too) differs from the oracle."""
    B, T, Cin, C, Co, seed = SHAPES[1]
    x, p, lab = inputs(B, T, Cin, C, Co, seed)
    lam = (2.0, 1.0, 0.5)
    r = orc.tem_fwd_bwd(x, p, lab, lam, prec=1, C=C)
    worst, errs = worst_rel(orc, r, torch_bf16_model(x, p, lab, lam, Cin, C, Co, mutant=mutant), Cin, C, Co)
    assert worst > MISS, (mutant, errs)


def test_bf16_cast_agrees_with_oracle_bit_rule(orc):
    """torch's cast and the oracle's RNE bit rule agree on random and tie values."""
    rng = np.random.default_rng(5)
    v = np.concatenate([rng.standard_normal(4096).astype(np.float32) * 10.0 ** rng.integers(-6, 6, 4096),
                        np.float32(1.0) + np.arange(1, 64, dtype=np.float32) * np.float32(2 ** -9)])
    v = v.astype(np.float32)
    t = torch.from_numpy(v).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(orc.bf16_round(v), t)
