"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Tolerances (BASELINE.json north_star): ring allreduce bit-exact; TEM relative 1e-4
(fp32) and 2e-2 (bf16 operands, fp32 accumulate), per tensor as
max|gpu - oracle| <= tol * max|oracle| against the fp64 oracle (bf16-emulated for
the bf16 path) -- DESIGN.md section 6.
"""
import os

import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu

TOL = {0: 1e-4, 1: 2e-2}
# ReLU decisions within tau * sum|terms| of zero are ambiguous under the kernel's rounding
# (reading R7b), per layer (a1, a2):
#  * fp32 path: bf16x3 products (~2^-16 each, R16) + fp32 accumulation gamma_K ~ K*u with
#    K <= 1536 terms: below 2^-13 on both layers;
#  * bf16 path, a1: both sides multiply the SAME rounded operands (x, W1), so only fp32-vs-fp64
#    accumulation differs: 2^-13 as above;
#  * bf16 path, a2: the operand h1 is itself a rounding of a1, and the GPU rounds its fp32 a1
#    while the oracle rounds its fp64 a1, so an h1 element can land one bf16 ulp (2^-8
#    relative) apart: 2^-8.
KINK_TAU = {0: (2.0 ** -13, 2.0 ** -13), 1: (2.0 ** -13, 2.0 ** -8)}
# at most this fraction of all ReLU decisions may be flipped into the oracle (R7b)
MAX_FLIP_FRAC = 1e-4


def oracle_with_gpu_decisions(orc, s, l, x, p, lab, lam, prec, threads=1, gdec=None):
    """fp64 oracle whose ReLU decisions agree with the GPU's wherever the decision is
    ambiguous; any GPU decision that differs OUTSIDE the oracle's ambiguity band fails, and
    so does a flip count above MAX_FLIP_FRAC of all decisions."""
    ref = orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, kink_tau=KINK_TAU[prec], kinks_cap=1 << 24,
                          threads=threads)
    if gdec is None:
        gdec = s.relu_decisions(l).cpu().numpy()
    diff = np.nonzero(gdec != ref["decisions"])[0]
    print(f"R7b: {diff.size} flipped ReLU decisions of {gdec.size} ({ref['nkinks']} in the band)")
    if diff.size == 0:
        return ref
    assert diff.size <= MAX_FLIP_FRAC * gdec.size, (diff.size, gdec.size)
    assert ref["nkinks"] <= (1 << 24)
    assert np.all(np.isin(diff, ref["kinks"])), "GPU ReLU decision differs outside the ambiguity band"
    return orc.tem_fwd_bwd(x, p, lab, lam, prec=prec, flips=diff, threads=threads)


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def tem():
    need_gpu()
    from paper_1906_06496_b200 import tem as T
    T.lib()
    return T


def make_inputs(N, B, prec, batch_idx=0, T=100, Cin=400):
    xs, labs = [], []
    for r in range(N):
        x = datagen.features(B, T, Cin, rank=r, batch_idx=batch_idx)
        xs.append(x)
        labs.append(datagen.labels(B, T, rank=r, batch_idx=batch_idx))
    return np.stack(xs), np.stack(labs)


def to_dev_x(x, prec):
    if prec == 1:
        bits = datagen.to_bf16_bits(x).view(np.int16)
        return torch.from_numpy(bits.copy()).cuda()
    return torch.from_numpy(x).cuda()


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def check_tensors(orc, gpu_grad, gpu_z, gpu_loss, ref, tol, C=512, Cin=400):
    sl = orc.param_slices(Cin, C, 3)
    for name, s in sl.items():
        e = rel_err(gpu_grad[s], ref["grad"][s])
        assert e <= tol, (name, e)
    assert rel_err(gpu_z, ref["z"]) <= tol
    assert rel_err(gpu_loss, ref["loss"]) <= tol


def session(tem, N, B, prec, lr=0.05, lam=(2.0, 1.0, 1.0), **kw):
    sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, precision=prec,
                           lr=lr, loss_weight=lam, **kw)
    p = datagen.init_params()
    return tem.TemSession(sc, p), p


@pytest.mark.parametrize("prec", [0, 1])
def test_tem_single_rank(tem, orc, prec):
    """N = 1, B = 4: forward, loss, backward vs oracle; then the update bitwise."""
    B, lam, lr = 4, (2.0, 1.0, 1.0), 0.05
    s, p = session(tem, 1, B, prec, lr=lr, lam=lam)
    x, lab = make_inputs(1, B, prec)
    xd, ld = to_dev_x(x, prec), torch.from_numpy(lab).cuda()
    w0 = s.params(0).cpu().numpy().copy()
    loss = s.compute(xd, ld)
    assert s.sync()[0] == 0
    g = s.local_grad(0).cpu().numpy().copy()
    ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p, lab[0], lam, prec)
    check_tensors(orc, g[:s.K], s.logits(0).cpu().numpy(), loss[0].cpu().numpy(), ref, TOL[prec])
    assert np.all(g[s.K:] == 0)
    s.exchange()
    assert s.sync()[0] == 0
    w1 = s.params(0).cpu().numpy()
    expect = orc.ring_sgd(g[None, :], w0, lr)[0]
    assert np.array_equal(w1, expect)
    s.close()


@pytest.mark.parametrize("N,B,prec", [(2, 4, 0), (4, 2, 0), (3, 2, 1)])
def test_tem_step_emulated_ranks(tem, orc, N, B, prec):
    """configs[0]-style step (B per rank, N ranks emulated on one device): local gradients
    vs oracle, then params after the fused ring+SGD bitwise equal to the oracle's replay of
    the ring on the GPU's own local gradients, identical on every rank."""
    lam, lr = (2.0, 1.0, 1.0), 0.05
    s, p = session(tem, N, B, prec, lr=lr, lam=lam)
    x, lab = make_inputs(N, B, prec)
    xd, ld = to_dev_x(x, prec), torch.from_numpy(lab).cuda()
    w0 = s.params(0).cpu().numpy().copy()
    loss = s.step(xd, ld)
    assert s.sync()[0] == 0
    grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    expect = orc.ring_sgd(grads, w0, lr)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect[r]), r
        ref = oracle_with_gpu_decisions(orc, s, r, x[r], p, lab[r], lam, prec)
        check_tensors(orc, grads[r][:s.K], s.logits(r).cpu().numpy(), loss[r].cpu().numpy(), ref, TOL[prec])
    if prec == 1:  # bf16 shadow refreshed from the new weights: next step sees them
        w1 = s.params(0).cpu().numpy().copy()  # weights after step 1 = inputs of step 2
        loss2 = s.step(xd, ld)
        assert s.sync()[0] == 0
        ref2 = orc.tem_fwd_bwd(x[0], w1, lab[0], lam, prec=1)
        assert rel_err(loss2[0].cpu().numpy(), ref2["loss"]) <= TOL[1]
    s.close()


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("K", [1, 7, 1000, 65537, 1403395])
def test_ring_allreduce_bitexact(tem, orc, N, K):
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=1403395)
    rng = np.random.default_rng(K * 10 + N)
    Kp = orc.kpad(K, N)
    g = np.zeros((N, Kp), np.float32)
    g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
    for op in (0, 1):
        sentinel = np.float32(123.5)
        for r in range(N):
            u = s.user(r, Kp)
            u.copy_(torch.from_numpy(g[r]))
            if Kp > K:
                u[K:] = float(sentinel)
        s.allreduce(K, op)
        assert s.sync()[0] == 0
        expect, _ = orc.ring_allreduce(g, op)
        for r in range(N):
            out = s.user(r, Kp).cpu().numpy()
            assert np.array_equal(out[:K], expect[r][:K]), (r, op)
            assert np.all(out[K:] == sentinel)  # elements >= K untouched
    s.close()


@pytest.mark.parametrize("N", [3, 4, 8])
def test_ring_order_witness(tem, orc, N):
    import json, os
    w = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "order_witness.json")))
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=4096)
    K = 4096
    Bk = orc.kpad(K, N) // N
    for r in range(N):
        v = w["big"] if r == 0 else (-w["big"] if r == 1 else 1.0)
        s.user(r, K).fill_(v)
    s.allreduce(K, 0)
    assert s.sync()[0] == 0
    expect = np.repeat(np.asarray(w["ring"][str(N)], np.float32), Bk)[:K]
    for r in range(N):
        assert np.array_equal(s.user(r, K).cpu().numpy(), expect)
    # PS comparator sums in ascending rank order
    for r in range(N):
        v = w["big"] if r == 0 else (-w["big"] if r == 1 else 1.0)
        s.user(r, K).fill_(v)
    s.ps_allreduce(K, 0)
    assert s.sync()[0] == 0
    for r in range(N):
        assert np.all(s.user(r, K).cpu().numpy() == w["ps"][str(N)])
    s.close()


def test_ps_allreduce_bitexact(tem, orc):
    N, K = 4, 100003
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=K)
    g = np.random.default_rng(1).standard_normal((N, K)).astype(np.float32)
    for r in range(N):
        s.user(r, K).copy_(torch.from_numpy(g[r]))
    s.ps_allreduce(K, 1)
    assert s.sync()[0] == 0
    expect = orc.ps_allreduce(g, 1)
    for r in range(N):
        assert np.array_equal(s.user(r, K).cpu().numpy(), expect)
    s.close()


def test_repeated_collectives_and_mixed_sizes(tem, orc):
    """Epoch flags never reset: many calls with different K (and channel counts) in a row."""
    N = 4
    s, _ = session(tem, N, 1, 0, max_allreduce_elems=1 << 20)
    rng = np.random.default_rng(7)
    for it, K in enumerate([1 << 20, 5, 1 << 16, 333333, 1 << 20, 17]):
        Kp = orc.kpad(K, N)
        g = np.zeros((N, Kp), np.float32)
        g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
        for r in range(N):
            s.user(r, Kp).copy_(torch.from_numpy(g[r]))
        if it % 2:
            s.ps_allreduce(K, 0)
            expect = np.broadcast_to(orc.ps_allreduce(g[:, :K], 0), (N, K))
        else:
            s.allreduce(K, 0)
            expect = orc.ring_allreduce(g, 0)[0][:, :K]
        assert s.sync()[0] == 0
        for r in range(N):
            assert np.array_equal(s.user(r, K).cpu().numpy(), expect[r])
    s.close()


def test_full_size_c2_fp32(tem, orc):
    """configs[1] shape (B = 16 per GPU, fp32) on one rank: every tensor vs the fp64 oracle."""
    B, lam = 16, (1.0, 1.0, 1.0)
    s, p = session(tem, 1, B, 0, lr=0.01, lam=lam)
    x, lab = make_inputs(1, B, 0, batch_idx=5)
    loss = s.compute(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p, lab[0], lam, 0)
    check_tensors(orc, s.local_grad(0).cpu().numpy()[:s.K], s.logits(0).cpu().numpy(),
                  loss[0].cpu().numpy(), ref, TOL[0])
    s.close()


def test_full_size_c3_bf16(tem, orc):
    """configs[2] (B = 256 per GPU, bf16 operands / fp32 accumulate) in the launch
    configuration the bench times: the loss, every logit and every gradient tensor against
    the bf16-emulated fp64 oracle over all 256 videos (threaded over videos)."""
    B, lam = 256, (2.0, 1.0, 1.0)
    s, p = session(tem, 1, B, 1, lr=0.01, lam=lam)
    x, lab = make_inputs(1, B, 1, batch_idx=2)
    loss = s.compute(to_dev_x(x, 1), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    ref = oracle_with_gpu_decisions(orc, s, 0, x[0], p, lab[0], lam, 1, threads=os.cpu_count() or 1)
    check_tensors(orc, s.local_grad(0).cpu().numpy()[:s.K], s.logits(0).cpu().numpy(),
                  loss[0].cpu().numpy(), ref, TOL[1])
    s.close()


def test_bench_call_c2_step(tem, orc):
    """The exact call bench.py times at N = 1: configs[1] (B = 16, fp32) through tem_step,
    graph-captured on the first call and replayed on the second, SGD with the split-K sums
    folded into the update.  Per step: every gradient tensor, the logits and the loss against
    the fp64 oracle at that step's weights, and the new weights bitwise equal to the oracle's
    w - lr * g (fma) on the GPU's own gradient."""
    B, lam, lr = 16, (1.0, 1.0, 1.0), 0.01
    s, p = session(tem, 1, B, 0, lr=lr, lam=lam)
    assert s.kernel_path() == "tcgen05-bf16x3-fp32"
    xd = torch.empty(1, B, 100, 400, device="cuda")
    ld = torch.empty(1, B, 3, 100, device="cuda")
    for it in range(2):  # same device buffers: step 2 replays the graph step 1 captured
        x, lab = make_inputs(1, B, 0, batch_idx=it)
        xd.copy_(torch.from_numpy(x))
        ld.copy_(torch.from_numpy(lab))
        w0 = s.params(0).cpu().numpy().copy()
        loss = s.step(xd, ld)
        assert s.sync()[0] == 0
        g = s.local_grad(0).cpu().numpy().copy()
        ref = oracle_with_gpu_decisions(orc, s, 0, x[0], w0, lab[0], lam, 0, threads=os.cpu_count() or 1)
        check_tensors(orc, g[:s.K], s.logits(0).cpu().numpy(), loss[0].cpu().numpy(), ref, TOL[0])
        assert np.array_equal(s.params(0).cpu().numpy(), orc.ring_sgd(g[None, :], w0, lr)[0]), it
    assert s.launches_per_step() > 0
    s.close()


def test_empty_batch_and_lr_zero(tem, orc):
    s, p = session(tem, 2, 0, 0, lr=0.0)
    w0 = s.params(0).cpu().numpy().copy()
    x = torch.zeros(2, 0, 100, 400, device="cuda")
    lab = torch.zeros(2, 0, 3, 100, device="cuda")
    loss = s.step(x, lab)
    assert s.sync()[0] == 0
    assert torch.all(loss == 0)
    for r in range(2):
        assert np.array_equal(s.params(r).cpu().numpy(), w0)
    s.close()


def test_nonfinite_latched(tem):
    """a non-finite loss latches NONFINITE with its step index.  (NaN features would
    not do: ReLU maps NaN pre-activations to 0 -- the comparison a > 0 is false.)"""
    s, p = session(tem, 1, 2, 0)
    x = torch.from_numpy(datagen.features(2)).cuda()[None]
    lab = torch.from_numpy(datagen.labels(2)).cuda()[None]
    s.step(x, lab)
    assert s.sync()[0] == 0
    s.params(0)[s.K - 1] = float("nan")  # b3[end] -> z[:, :, 2] = NaN at step 1
    s.step(x, lab)
    code, step = s.sync()
    assert code == tem.TEM_ERR_NONFINITE and step == 1
    with pytest.raises(tem.TemError):
        s.step(x, lab)
    s.ctx = None  # context is poisoned; shutdown would report the latched error


def test_invalid_args(tem):
    sc = tem.SessionConfig(world_size=2, rank=0, local_ranks=2, batch_per_rank=1)
    s = tem.TemSession(sc, datagen.init_params())
    with pytest.raises(tem.TemError) as e:
        tem.ring_allreduce(s.ctx, s.user(0).data_ptr() + 4, 10)  # not the user region
    assert e.value.code == tem.TEM_ERR_INVALID_ARG
    with pytest.raises(tem.TemError):
        s.allreduce(0)
    with pytest.raises(tem.TemError):
        s.allreduce(s.K + 1)
    s.close()
    bad = tem.tem_config()
    bad.world_size = 0
    assert tem.tem_num_params(bad) == 0


@pytest.mark.parametrize("N", [2, 3, 4])
def test_tem_step_ps_exchange(tem, orc, N):
    """The PS comparator as a training step: the server (rank 0) sums the pushed
    gradients in ascending rank order, applies mean + SGD once, and every rank
    pulls w'.  Bitwise: w' = fma(-lr, ps_mean(g), w) on every rank."""
    B, lam, lr = 2, (2.0, 1.0, 1.0), 0.05
    s, p = session(tem, N, B, 0, lr=lr, lam=lam, exchange=tem.TEM_EXCHANGE_PS)
    x, lab = make_inputs(N, B, 0)
    w0 = s.params(0).cpu().numpy().copy()
    s.step(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    grads = np.stack([s.local_grad(r).cpu().numpy() for r in range(N)])
    gbar = orc.ps_allreduce(grads, orc.MEAN).astype(np.float64)
    expect = (w0.astype(np.float64) - np.float64(np.float32(lr)) * gbar).astype(np.float32)
    for r in range(N):
        assert np.array_equal(s.params(r).cpu().numpy(), expect), r
    # the refreshed operand copies feed the next step: loss matches the oracle at w'
    loss2 = s.step(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda())
    assert s.sync()[0] == 0
    ref = orc.tem_fwd_bwd(x[0], expect, lab[0], lam, prec=0)
    assert rel_err(loss2[0].cpu().numpy(), ref["loss"]) <= TOL[0]
    s.close()
