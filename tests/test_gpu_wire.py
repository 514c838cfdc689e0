"""The production collective path (one rank per process, local_ranks = 1) on ONE GPU, with
the other ranks played by the test through the wire protocol of include/tem.h.

Ranks whose kernels wait on one another must not run as separate launches on one GPU
(B200_PROFILING.md), so the other ranks are "virtual": before the collective is launched the
test writes, from the oracle, every header and LL message this rank will receive into its
heap.  The rank's kernel -- the exact non-cooperative launch (and CUDA graph) a one-process-per-
GPU run uses -- then runs alone and never waits on another kernel.  Checked bit for bit:
  * its result against the oracle's ring replay;
  * every message it sends (the LL lines it stores into its right neighbour's heap) against
    the oracle's partial chains (scatter) and final blocks (gather);
  * the symmetric handshake: a peer header with another K / op -> PROTOCOL before any data
    moves; a peer that never arrives -> TRANSPORT after the bound.
"""
import numpy as np
import pytest
import torch

import datagen
from test_gpu_parity import TOL, make_inputs, need_gpu, rel_err  # noqa: F401

pytestmark = pytest.mark.gpu

G = 4        # channels (ring_channels) of the contexts below
KIND_RING = 0


@pytest.fixture(scope="module")
def tem():
    need_gpu()
    from paper_1906_06496_b200 import tem as T
    T.lib()
    return T


def vsession(tem, N, rank, B=1, max_ar=0, **kw):
    sc = tem.SessionConfig(world_size=N, rank=rank, local_ranks=1, batch_per_rank=B, ring_channels=G,
                           max_allreduce_elems=max_ar, **kw)
    return tem.TemSession(sc, datagen.init_params(), virtual_peers=True)


def heap_u32(s, r):
    return s._heap_of(r).view(torch.int32)


def header(K, epoch, kind, op, mode):
    return np.array([K & 0xFFFFFFFF, epoch, ((K >> 32) & 0xFF) | (kind << 8) | (op << 16) | (mode << 24), epoch],
                    dtype=np.uint32)


def put_header(s, dst, src, hdr):
    """Header of rank src (every channel) into rank dst's heap, slot of hdr's epoch parity."""
    base = s.hdr_off // 4 + ((int(hdr[1]) & 1) * 8 + src) * 128 * 4
    v = torch.from_numpy(np.tile(hdr, G).view(np.int32)).cuda()
    heap_u32(s, dst)[base: base + 4 * G].copy_(v)


def read_header(s, dst, src, epoch):
    base = s.hdr_off // 4 + ((epoch & 1) * 8 + src) * 128 * 4
    return heap_u32(s, dst)[base: base + 4 * G].cpu().numpy().view(np.uint32).reshape(G, 4)


def ll_slot_words(s, N, epoch, phase, rnd):
    """u32 word offset of LL slot (epoch parity, phase, round) in a heap."""
    idx = ((epoch & 1) * 2 * (N - 1) + phase * (N - 1) + rnd) * s.ll_lines
    return (s.ll_off + idx * 16) // 4


def put_ll(s, dst, N, epoch, phase, rnd, msg):
    """Encode the block message msg (fp32, length Bk) as LL lines into rank dst's slot."""
    m = np.ascontiguousarray(msg, np.float32).view(np.uint32)
    lines = np.empty((m.size // 2, 4), np.uint32)
    lines[:, 0], lines[:, 2] = m[0::2], m[1::2]
    lines[:, 1] = lines[:, 3] = epoch
    w0 = ll_slot_words(s, N, epoch, phase, rnd)
    heap_u32(s, dst)[w0: w0 + lines.size].copy_(torch.from_numpy(lines.ravel().view(np.int32)).cuda())


def get_ll(s, dst, N, epoch, phase, rnd, Bk):
    """Decode slot (phase, round) of rank dst: (values, every flag == epoch)."""
    w0 = ll_slot_words(s, N, epoch, phase, rnd)
    lines = heap_u32(s, dst)[w0: w0 + 2 * Bk].cpu().numpy().view(np.uint32).reshape(-1, 4)
    vals = np.empty(Bk, np.uint32)
    vals[0::2], vals[1::2] = lines[:, 0], lines[:, 2]
    return vals.view(np.float32), bool(np.all(lines[:, 1] == epoch) and np.all(lines[:, 3] == epoch))


def partial_chain(orc, g, blk, last, Bk):
    """Block blk summed along its ring chain from rank blk up to rank `last`:
    the oracle's chain over N ranks with the ranks after `last` zeroed (x + 0 == x)."""
    N = g.shape[0]
    h = np.zeros_like(g)
    q = blk
    while True:
        h[q] = g[q]
        if q == last:
            break
        q = (q + 1) % N
    return orc.ring_chain(h, 0)[blk * Bk:(blk + 1) * Bk]


def transcript_in(orc, s, g, final, r, epoch, K, op, mode):
    """Everything rank r receives in one ring collective, written into its heap: every peer's
    header, the scatter partials and the gather blocks from its left neighbour."""
    N, Kp = g.shape
    Bk = Kp // N
    left = (r - 1) % N
    for q in range(N):
        if q != r:
            put_header(s, r, q, header(K, epoch, KIND_RING, op, mode))
    for i in range(N - 1):  # scatter round i: left sends block (left - i), chain from it to left
        blk = (left - i) % N
        put_ll(s, r, N, epoch, 0, i, partial_chain(orc, g, blk, left, Bk))
    for k in range(N - 1):  # gather round k: left sends block (left + 1 - k): its final value
        blk = (left + 1 - k) % N
        put_ll(s, r, N, epoch, 1, k, final[blk * Bk:(blk + 1) * Bk])


def check_transcript_out(orc, s, g, final, r, epoch):
    """Everything rank r sent to its right neighbour in that collective."""
    N, Kp = g.shape
    Bk = Kp // N
    right = (r + 1) % N
    for i in range(N - 1):
        blk = (r - i) % N
        vals, ok = get_ll(s, right, N, epoch, 0, i, Bk)
        assert ok, ("scatter flags", i)
        assert np.array_equal(vals, partial_chain(orc, g, blk, r, Bk)), ("scatter", i)
    for k in range(N - 1):
        blk = (r + 1 - k) % N
        vals, ok = get_ll(s, right, N, epoch, 1, k, Bk)
        assert ok, ("gather flags", k)
        assert np.array_equal(vals, final[blk * Bk:(blk + 1) * Bk]), ("gather", k)


@pytest.mark.parametrize("N,r", [(2, 0), (2, 1), (3, 1), (4, 0), (4, 3), (8, 5)])
def test_ring_allreduce_one_rank_transcript(tem, orc, N, r):
    """ring_allreduce as one process of an N-rank job: result and every message bit-exact."""
    K = 50000 + 13  # K < K_pad: the tail is masked
    s = vsession(tem, N, r, max_ar=K)
    Kp = orc.kpad(K, N)
    rng = np.random.default_rng(100 * N + r)
    g = np.zeros((N, Kp), np.float32)
    g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
    for op in (0, 1):
        epoch = op + 1
        final = orc.ring_allreduce(g, op)[0][0]
        final_k = final.copy()
        final_k[K:] = 0.0  # positions >= K travel as zeros
        s.user(0, Kp).copy_(torch.from_numpy(g[r]))
        sentinel = 7.25
        s.user(0, Kp)[K:] = sentinel
        transcript_in(orc, s, g, final_k, r, epoch, K, op, 0)
        torch.cuda.synchronize()
        s.allreduce(K, op)
        assert s.sync()[0] == 0
        out = s.user(0, Kp).cpu().numpy()
        assert np.array_equal(out[:K], final[:K]), op
        assert np.all(out[K:] == sentinel)
        check_transcript_out(orc, s, g, final_k, r, epoch)
        for q in range(N):  # our header reached every rank
            if q != r:
                assert np.all(read_header(s, q, r, epoch) == header(K, epoch, KIND_RING, op, 0)[None, :])
    s.close()


@pytest.mark.parametrize("buckets", [1, 2])
def test_tem_step_one_rank_transcript(tem, orc, buckets):
    """tem_step of rank 0 of a 2-rank job, graph-captured on step 1 and replayed on step 2, SGD:
    params bitwise equal to the oracle's ring replay on [g_0, g_1] (g_1 = the virtual peer's
    gradient), messages bit-exact.  buckets = 2: the [bnd, K_pad) bucket's ring is launched on
    the side branch inside the step (reading R25), then [0, bnd)."""
    N, r, B, lr, lam = 2, 0, 2, 0.05, (2.0, 1.0, 1.0)
    s = vsession(tem, N, r, B=B, lr=lr, loss_weight=lam, exchange_buckets=buckets)
    Kp = s.Kpad
    bnd = (512 * 3 * 400 + 512 + 4 * N - 1) // (4 * N) * (4 * N) if buckets == 2 else Kp
    spans = [(bnd, Kp), (0, bnd)] if buckets == 2 else [(0, Kp)]
    xd = torch.empty(1, B, 100, 400, device="cuda")
    ld = torch.empty(1, B, 3, 100, device="cuda")
    rng = np.random.default_rng(3)
    epoch = 0
    for it in range(2):
        x, lab = make_inputs(1, B, 0, batch_idx=it)
        xd.copy_(torch.from_numpy(x))
        ld.copy_(torch.from_numpy(lab))
        w0 = s.params(0).cpu().numpy().copy()
        s.compute(xd, ld)  # the step recomputes this gradient bit for bit (deterministic kernels)
        assert s.sync()[0] == 0
        g0 = s.local_grad(0).cpu().numpy().copy()
        g1 = (rng.standard_normal(Kp) * 1e-3).astype(np.float32)
        g = np.stack([g0, g1])
        expect = np.empty(Kp, np.float32)
        plan = []
        for (e0, e1) in spans:
            epoch += 1
            fin = orc.ring_sgd(g[:, e0:e1], w0[e0:e1], lr)
            assert np.array_equal(fin[0], fin[1])
            expect[e0:e1] = fin[0]
            transcript_in(orc, s, g[:, e0:e1], fin[0], r, epoch, e1 - e0, 1, 1)
            plan.append((e0, e1, epoch, fin[0]))
        torch.cuda.synchronize()
        s.step(xd, ld)
        assert s.sync()[0] == 0
        assert np.array_equal(s.params(0).cpu().numpy(), expect), it
        for (e0, e1, ep, fin) in plan:
            check_transcript_out(orc, s, g[:, e0:e1], fin, r, ep)
        # the refreshed bf16 operand copies are the new weights' split (R16)
        sh = s.debug_buffer("shadow").float().cpu().numpy()
        assert np.array_equal(sh, orc.bf16_round(expect))
    s.close()


@pytest.mark.parametrize("what", ["K", "op"])
def test_handshake_mismatch_is_protocol_before_data(tem, orc, what):
    """A peer whose collective differs (K or op): PROTOCOL on this rank, user buffer untouched,
    nothing sent -- every rank compares the same N headers, so every rank decides alike."""
    N, r, K = 4, 2, 4096
    s = vsession(tem, N, r, max_ar=8192)
    u = s.user(0, K)
    u.copy_(torch.arange(K, dtype=torch.float32, device="cuda"))
    for q in range(N):
        if q != r:
            bad = q == 0
            put_header(s, r, q, header(K + (4 if bad and what == "K" else 0), 1, KIND_RING,
                                       1 if bad and what == "op" else 0, 0))
    torch.cuda.synchronize()
    s.allreduce(K, 0)
    code, _ = s.sync()
    assert code == tem.TEM_ERR_PROTOCOL
    assert torch.equal(u, torch.arange(K, dtype=torch.float32, device="cuda"))
    _, ok = get_ll(s, (r + 1) % N, N, 1, 0, 0, orc.kpad(K, N) // N)
    assert not ok  # no message left this rank
    s.ctx = None   # poisoned context


def test_missing_peer_is_transport(tem):
    """No peer ever arrives: TRANSPORT once the spin bound (here 300 ms) has passed."""
    import time
    N, K = 2, 1000
    s = vsession(tem, N, 0, max_ar=K, spin_timeout_ms=300)
    t0 = time.perf_counter()
    s.allreduce(K, 0)
    code, _ = s.sync()
    dt = time.perf_counter() - t0
    assert code == tem.TEM_ERR_TRANSPORT
    assert 0.25 < dt < 10.0
    s.ctx = None
