"""GPU: the tcgen05 path against the SIMT path, stage by stage, on identical inputs.

A secondary check beside the oracle parity tests (test_gpu_parity.py): when the two kernel
paths disagree, the first mismatching stage (h1, h2, dA2, dA1, gradient) names the kernel.
Both paths accumulate in fp32; the tcgen05 fp32 path splits operands into bf16 hi + lo.
"""
import os

import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu


def run_path(path, B, prec, lam=(2.0, 1.0, 1.0)):
    from paper_1906_06496_b200 import tem
    os.environ["TEM_KERNEL_PATH"] = path
    try:
        sc = tem.SessionConfig(world_size=1, rank=0, local_ranks=1, batch_per_rank=B, precision=prec,
                               lr=0.0, loss_weight=lam)
        s = tem.TemSession(sc, datagen.init_params())
    finally:
        os.environ.pop("TEM_KERNEL_PATH", None)
    x = datagen.features(B, batch_idx=1)
    lab = datagen.labels(B, batch_idx=1)
    if prec == 1:
        xd = torch.from_numpy(datagen.to_bf16_bits(x).view(np.int16)).cuda()
    else:
        xd = torch.from_numpy(x).cuda()
    loss = s.compute(xd[None], torch.from_numpy(lab).cuda()[None])
    code, _ = s.sync()
    assert code == 0
    out = {"path": s.kernel_path(), "loss": loss[0].cpu().numpy().astype(np.float64),
           "grad": s.local_grad(0).cpu().numpy()[:s.K].astype(np.float64)}
    for name in ("xp", "h1", "h2", "dA2", "dA1"):
        t = s.debug_buffer(name).float()
        lo = s.debug_buffer(name + "_lo") if name != "h2" else None
        if lo is not None:
            t = t + lo.float()
        out[name] = t.cpu().numpy().astype(np.float64)
    s.close()
    return out


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("B,prec,tol", [(4, 0, 1e-4), (4, 1, 2e-2), (16, 0, 1e-4), (37, 1, 2e-2)])
def test_tcgen05_matches_simt(B, prec, tol):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    u = run_path("umma", B, prec)
    s = run_path("simt", B, prec)
    assert u["path"].startswith("tcgen05") and s["path"].startswith("simt")
    errs = {k: rel(u[k], s[k]) for k in ("xp", "h1", "h2", "dA2", "dA1", "loss", "grad")}
    # ReLU decisions near a kink may legitimately differ between the paths (reading R7b):
    # a flipped h2 decision changes one dA2 element entirely and three rows of dA1.
    flip1 = (u["h1"] > 0) != (s["h1"] > 0)
    flip2 = (u["h2"] > 0) != (s["h2"] > 0)
    nflip = int(flip1.sum() + flip2.sum())
    print(f"\nB={B} prec={prec} flips={nflip}: " + " ".join(f"{k}={v:.2e}" for k, v in errs.items()))
    assert nflip <= max(2, 1e-5 * flip1.size), nflip
    for k in ("xp", "h1", "h2", "loss"):
        assert errs[k] <= tol, (k, errs)
    keep = ~(flip2 | flip1)
    assert rel(u["dA2"][keep], s["dA2"][keep]) <= tol, errs
    if nflip == 0:  # no ambiguous decision: the backward must agree too
        assert errs["dA1"] <= tol and errs["grad"] <= 10 * tol, errs
