"""GPU parity of the alternative kernel paths the default configuration does not take.

The plan picks kernels by shape: the fp32 single-wave path fuses the head into
conv2 FWD, larger fp32 batches use the persistent halo kernel with several tiles per CTA,
bf16 uses 2-CTA pairs. These tests force the other paths through the plan's switches
(read when a session is created) and hold each to the same oracle contract.
"""
import numpy as np
import pytest
import torch

from test_gpu_parity import (TOL, check_tensors, make_inputs, oracle_with_gpu_decisions, rel_err, session,  # noqa: F401
                             tem, to_dev_x)

pytestmark = pytest.mark.gpu


def _compute(tem, B, prec, batch_idx=0, lam=(2.0, 1.0, 1.0)):
    s, p = session(tem, 1, B, prec, lr=0.01, lam=lam)
    x, lab = make_inputs(1, B, prec, batch_idx=batch_idx)
    loss = s.compute(to_dev_x(x, prec), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    out = {"grad": s.local_grad(0).cpu().numpy()[:s.K].copy(), "z": s.logits(0).cpu().numpy().copy(),
           "loss": loss[0].cpu().numpy().copy(), "path": s.kernel_path()}
    return s, p, x, lab, out


def _check(orc, s, p, x, lab, out, prec, lam=(2.0, 1.0, 1.0)):
    ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p, lab[0], lam, prec)
    check_tensors(orc, out["grad"], out["z"], out["loss"], ref, TOL[prec])


def test_unfused_head_fp32(tem, orc, monkeypatch):
    """fp32 B = 4 with the separate head kernel (TEM_NO_FUSED_HEAD) vs the oracle."""
    monkeypatch.setenv("TEM_NO_FUSED_HEAD", "1")
    s, p, x, lab, out = _compute(tem, 4, 0)
    _check(orc, s, p, x, lab, out, 0)
    s.close()


def test_fused_and_unfused_head_agree(tem, monkeypatch):
    """Same inputs through the fused head (default at B = 16 fp32) and the head kernel: every
    output agrees to fp32 rounding-order differences (1e-5 of the tensor's max)."""
    s1, _, _, _, fused = _compute(tem, 16, 0, batch_idx=3)
    s1.close()
    monkeypatch.setenv("TEM_NO_FUSED_HEAD", "1")
    s2, _, _, _, plain = _compute(tem, 16, 0, batch_idx=3)
    s2.close()
    for k in ("grad", "z", "loss"):
        a, b = fused[k].astype(np.float64), plain[k].astype(np.float64)
        assert np.abs(a - b).max() <= 1e-5 * max(np.abs(b).max(), 1e-30), k


def test_fp32_multi_tile_per_cta(tem, orc):
    """fp32 B = 24: 20 row tiles x 8 column tiles > 148 CTAs, so the persistent halo kernel runs
    several tiles per CTA (double-buffered dual accumulators) and the head is not fused."""
    s, p, x, lab, out = _compute(tem, 24, 0, batch_idx=1)
    _check(orc, s, p, x, lab, out, 0)
    s.close()


def test_graph_and_eager_steps_identical(tem, monkeypatch):
    """tem_step replayed from a CUDA graph and launched eagerly (TEM_NO_GRAPH) run the same
    kernels: parameters after three steps are bitwise identical."""
    def run():
        s, _ = session(tem, 1, 8, 0, lr=0.05)
        x, lab = make_inputs(1, 8, 0, batch_idx=6)
        xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
        for _ in range(3):
            s.step(xd, ld)
        assert s.sync()[0] == 0
        w = s.params(0).cpu().numpy().copy()
        s.close()
        return w
    w_graph = run()
    monkeypatch.setenv("TEM_NO_GRAPH", "1")
    w_eager = run()
    assert np.array_equal(w_graph, w_eager)


def test_step_host_matches_device_step(tem):
    """tem_step_host (pinned host x / labels / loss, copies inside the step; the loss is read
    back on the side stream) == tem_step on device buffers: same loss, bitwise equal params."""
    B = 8
    x, lab = make_inputs(1, B, 0, batch_idx=7)
    s1, _ = session(tem, 1, B, 0, lr=0.05)
    xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
    losses_dev = []
    for _ in range(3):
        losses_dev.append(s1.step(xd, ld).cpu().numpy().copy())
    assert s1.sync()[0] == 0
    w1 = s1.params(0).cpu().numpy().copy()
    s1.close()
    s2, _ = session(tem, 1, B, 0, lr=0.05)
    xh = torch.from_numpy(x[0].copy()).pin_memory()
    lh = torch.from_numpy(lab[0].copy()).pin_memory()
    loss_h = torch.zeros(4, dtype=torch.float32).pin_memory()
    for i in range(3):
        s2.step_host(xh, lh, loss_h)
        torch.cuda.synchronize()
        assert np.array_equal(loss_h.numpy(), losses_dev[i].reshape(-1)[:4]), i
    assert s2.sync()[0] == 0
    assert np.array_equal(s2.params(0).cpu().numpy(), w1)
    s2.close()


def test_step_host_pipelined_inputs(tem):
    """Back-to-back tem_step_host calls with a different batch each (copy of step k+1 on the
    copy stream beside step k, two staging sets): every step sees its own inputs -- losses
    and final params bitwise equal to device-buffer steps on the same batches."""
    B, n = 4, 5
    batches = [make_inputs(1, B, 0, batch_idx=20 + i) for i in range(n)]
    s1, _ = session(tem, 1, B, 0, lr=0.05)
    losses = []
    for x, lab in batches:
        losses.append(s1.step(to_dev_x(x, 0), torch.from_numpy(lab).cuda()).cpu().numpy().reshape(-1)[:4].copy())
    assert s1.sync()[0] == 0
    w1 = s1.params(0).cpu().numpy().copy()
    s1.close()
    s2, _ = session(tem, 1, B, 0, lr=0.05)
    xh = [torch.from_numpy(x[0].copy()).pin_memory() for x, _ in batches]
    lh = [torch.from_numpy(lab[0].copy()).pin_memory() for _, lab in batches]
    outs = [torch.zeros(4, dtype=torch.float32).pin_memory() for _ in range(n)]
    for i in range(n):  # no host synchronisation between calls
        s2.step_host(xh[i], lh[i], outs[i])
    torch.cuda.synchronize()
    assert s2.sync()[0] == 0
    for i in range(n):
        assert np.array_equal(outs[i].numpy(), losses[i]), i
    assert np.array_equal(s2.params(0).cpu().numpy(), w1)
    s2.close()


def test_step_pem_host_matches_device_step(tem):
    """tem_step_pem_host (host x, labels, BSP features, IoU; 5 loss floats) == tem_step_pem on
    device buffers, over several pipelined calls."""
    import datagen
    from test_gpu_pem import pem_inputs, pem_session
    B, n = 2, 3
    s1, _ = pem_session(tem, 1, B)
    ref = []
    for i in range(n):
        x, lab = make_inputs(1, B, 0, batch_idx=30 + i)
        f, g = pem_inputs(1, B, batch_idx=30 + i)
        tl, pl = s1.step_pem(to_dev_x(x, 0), torch.from_numpy(lab).cuda(), torch.from_numpy(f).cuda(),
                             torch.from_numpy(g).cuda())
        ref.append(np.concatenate([tl.cpu().numpy().reshape(-1), pl.cpu().numpy().reshape(-1)]))
    assert s1.sync()[0] == 0
    w1 = s1.params(0).cpu().numpy().copy()
    s1.close()
    s2, _ = pem_session(tem, 1, B)
    outs = []
    keep = []
    for i in range(n):
        x, lab = make_inputs(1, B, 0, batch_idx=30 + i)
        f, g = pem_inputs(1, B, batch_idx=30 + i)
        hs = [torch.from_numpy(np.ascontiguousarray(a[0])).pin_memory() for a in (x, lab, f, g)]
        keep.append(hs)
        outs.append(torch.zeros(5, dtype=torch.float32).pin_memory())
        s2.step_pem_host(*hs, outs[-1])
    torch.cuda.synchronize()
    assert s2.sync()[0] == 0
    for i in range(n):
        assert np.array_equal(outs[i].numpy(), ref[i]), i
    assert np.array_equal(s2.params(0).cpu().numpy(), w1)
    assert datagen.PEM_P > 0
    s2.close()


@pytest.mark.parametrize("B,N", [(16, 1), (12, 1), (12, 2)])
def test_persistent_backward_is_bitwise_the_three_launches(tem, orc, monkeypatch, B, N):
    """The fp32 backward as one persistent launch (bwd_kernel: DGRAD, conv2 WGRAD and conv1
    WGRAD tiles of a static schedule, conv1 WGRAD waiting on DGRAD tile flags) runs each tile
    through the same device code as the three separate launches (TEM_NO_BWD): the gradient,
    logits and loss are bitwise identical, so are the parameters after two tem_steps, and the
    gradient meets the oracle contract."""
    lam, lr = (2.0, 1.0, 1.0), 0.05
    outs = []
    for no_bwd in (False, True):
        if no_bwd:
            monkeypatch.setenv("TEM_NO_BWD", "1")
        s, p = session(tem, N, B, 0, lr=lr, lam=lam)
        x, lab = make_inputs(N, B, 0, batch_idx=4)
        xd, ld = to_dev_x(x, 0), torch.from_numpy(lab).cuda()
        loss = s.compute(xd, ld)
        assert s.sync()[0] == 0
        g = np.stack([s.local_grad(r).cpu().numpy().copy() for r in range(N)])
        z = s.logits(0).cpu().numpy().copy()
        l0 = loss.cpu().numpy().copy()
        if not no_bwd:  # (the ReLU decisions of this compute, before the steps)
            ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p, lab[0], lam, 0)
            check_tensors(orc, g[0][:s.K], z, l0[0], ref, TOL[0])
        for _ in range(2):
            s.step(xd, ld)
            assert s.sync()[0] == 0
        w = s.params(0).cpu().numpy().copy()
        outs.append((g, z, l0, w))
        s.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("N", [1, 2])
def test_operand_sets_follow_every_update(tem, orc, N):
    """The weights' bf16 operand copies alternate between two sets (RankBufs::shadow): a step's
    GEMMs read one, its update writes the other.  Mixing graph-replayed tem_step calls with
    tem_compute + tem_exchange (eager) must keep every step on the current weights: after each
    update the parameters equal the oracle's ring SGD of the GPU's own gradient (bitwise), the
    operand copy the next step reads is bf16 of those parameters (bitwise), and the next loss
    matches the oracle at those parameters."""
    B, lr, lam = 2, 0.05, (2.0, 1.0, 1.0)
    s, p = session(tem, N, B, 0, lr=lr, lam=lam)
    xd = torch.empty(N, B, 100, 400, device="cuda")
    ld = torch.empty(N, B, 3, 100, device="cuda")
    for it, how in enumerate(["step", "split", "step", "step", "split", "step"]):
        x, lab = make_inputs(N, B, 0, batch_idx=it)
        xd.copy_(torch.from_numpy(x))
        ld.copy_(torch.from_numpy(lab))
        w0 = s.params(0).cpu().numpy().copy()
        sh = s.debug_buffer("shadow").float().cpu().numpy()
        assert np.array_equal(sh, orc.bf16_round(w0)), (it, "operand copy of the current weights")
        if how == "step":
            loss = s.step(xd, ld)
        else:
            loss = s.compute(xd, ld)
            s.exchange()
        assert s.sync()[0] == 0
        g = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
        ref = orc.tem_fwd_bwd(x[0], w0, lab[0], lam, prec=0)
        assert rel_err(loss[0].cpu().numpy(), ref["loss"]) <= TOL[0], it
        expect = orc.ring_sgd(g, w0, lr)
        for r in range(N):
            assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), (it, r)
    s.close()
