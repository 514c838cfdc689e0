"""Pins for the oracle's partition, schedules and ring/PS replay (no GPU).

Every expected value here comes from the paper (cited), from closed-form /
exactness arguments, or from brute force on small inputs -- never from the
oracle itself or from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- schedules
def test_schedule_examples(orc):
    g = gold("paper_values.json")
    for rank, N, rnd, s, r in g["scatter_examples"]["cases"]:
        assert orc.scatter_schedule(rank, N, rnd) == (s, r)
    for rank, N, rnd, s, r in g["gather_examples"]["cases"]:
        assert orc.gather_schedule(rank, N, rnd) == (s, r)


def test_schedule_out_of_range(orc):
    with pytest.raises(ValueError):
        orc.scatter_schedule(0, 4, 3)
    with pytest.raises(ValueError):
        orc.gather_schedule(0, 1, 0)


@pytest.mark.parametrize("N", range(2, 17))
def test_schedule_bijective_and_neighbour_consistent(orc, N):
    for sched in (orc.scatter_schedule, orc.gather_schedule):
        for i in range(N - 1):
            sends = [sched(n, N, i)[0] for n in range(N)]
            recvs = [sched(n, N, i)[1] for n in range(N)]
            assert sorted(sends) == list(range(N)) and sorted(recvs) == list(range(N))
            for n in range(N):  # what my left neighbour sends is what I receive
                assert recvs[n] == sends[(n - 1) % N]


@pytest.mark.parametrize("N", range(2, 17))
def test_symbolic_completion(orc, N):
    """after N-1 scatter rounds GPU n holds all contributions of block (n+1)%N;
    P:152/P:156: after N-1 gather rounds every GPU holds every complete block."""
    have = [[{n} for _ in range(N)] for n in range(N)]  # have[n][b] = set of contributors
    for i in range(N - 1):
        msgs = []
        for n in range(N):
            s, _ = orc.scatter_schedule(n, N, i)
            msgs.append(set(have[n][s]))
        for n in range(N):
            _, r = orc.scatter_schedule(n, N, i)
            have[n][r] |= msgs[(n - 1) % N]
    full = set(range(N))
    for n in range(N):
        assert have[n][(n + 1) % N] == full
    for k in range(N - 1):
        msgs = []
        for n in range(N):
            s, _ = orc.gather_schedule(n, N, k)
            assert k > 0 or s == (n + 1) % N  # round 0 sends the block completed in the scatter
            msgs.append(set(have[n][s]))
        for n in range(N):
            _, r = orc.gather_schedule(n, N, k)
            have[n][r] = msgs[(n - 1) % N]  # replace
    for n in range(N):
        for b in range(N):
            assert have[n][b] == full


def test_paper_literal_gather_formula_does_not_complete():
    """Documents reading R10: P:152's literal (n-i-1)%N / (n-i-2)%N with i from 0 or 1
    leaves some block incomplete for N >= 4 (so the oracle uses the consistent rotation)."""
    for N in (4, 5, 8):
        for origin in (0, 1):
            have = [[{n} for _ in range(N)] for n in range(N)]
            for n in range(N):
                have[n][(n + 1) % N] = set(range(N))  # state after the scatter
            for i in range(origin, origin + N - 1):
                msgs = [set(have[n][(n - i - 1) % N]) for n in range(N)]
                for n in range(N):
                    have[n][(n - i - 2) % N] = msgs[(n - 1) % N]
            assert not all(have[n][b] == set(range(N)) for n in range(N) for b in range(N))


# ----------------------------------------------------------------------------- partition
def test_kpad_and_param_count(orc):
    g = gold("paper_values.json")["tem_param_count"]
    assert orc.num_params(400, 512, 3) == g["K"]
    for N, kp in g["K_pad"].items():
        kp_ = orc.kpad(g["K"], int(N))
        assert kp_ == kp and kp_ % (int(N) * 4) == 0 and kp_ - g["K"] < int(N) * 4
    with pytest.raises(ValueError):
        orc.kpad(10, 0)


# ----------------------------------------------------------------------------- ring sums
def test_one_hot_n3(orc):
    """inputs [1,0,0],[0,1,0],[0,0,1] -> every worker returns [1,1,1] (K padded to 12)."""
    g = np.zeros((3, 12), np.float32)
    for r in range(3):
        g[r, r] = 1.0
    out, sent = orc.ring_allreduce(g)
    assert np.array_equal(out[:, :3], np.ones((3, 3), np.float32))
    assert np.all(out[:, 3:] == 0)
    assert list(sent) == [2 * 4 * 2] * 3


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7, 8])
def test_integer_exact_vs_brute_force(orc, N):
    """Integer inputs |g| <= 2^10 keep every partial sum exact in fp32, so the ring equals
    the brute-force sum bitwise in any order; every rank ends identical."""
    rng = np.random.default_rng(N)
    K_pad = orc.kpad(1001, N)
    g = rng.integers(-1024, 1025, size=(N, K_pad)).astype(np.float32)
    out, sent = orc.ring_allreduce(g)
    exact = g.astype(np.int64).sum(0).astype(np.float32)
    for r in range(N):
        assert np.array_equal(out[r], exact)
    assert np.array_equal(orc.ring_chain(g), exact)
    # P:172 volume: 2 K_pad (N-1)/N elements sent per rank
    assert list(sent) == [2 * K_pad * (N - 1) // N] * N


@pytest.mark.parametrize("N", [3, 4, 8])
def test_order_witness(orc, N):
    w = gold("order_witness.json")
    K_pad = orc.kpad(N * 4, N)
    Bk = K_pad // N
    g = np.ones((N, K_pad), np.float32)
    g[0, :] = w["big"]
    g[1, :] = -w["big"]
    out, _ = orc.ring_allreduce(g)
    expect = np.repeat(np.asarray(w["ring"][str(N)], np.float32), Bk)
    for r in range(N):
        assert np.array_equal(out[r], expect)
    assert np.array_equal(orc.ring_chain(g), expect)
    assert np.all(orc.ps_allreduce(g) == w["ps"][str(N)])


@pytest.mark.parametrize("N,K", [(2, 8), (3, 7), (4, 64), (8, 1000), (5, 1)])
def test_random_within_summation_bound(orc, N, K):
    """|ring - exact| <= gamma_{N-1} * sum_r |g_r| (recursive summation, Higham 4.3)."""
    rng = np.random.default_rng(K + N)
    K_pad = orc.kpad(K, N)
    g = rng.standard_normal((N, K_pad)).astype(np.float32)
    out, _ = orc.ring_allreduce(g)
    exact = g.astype(np.float64).sum(0)
    u = 2.0 ** -24
    gam = (N - 1) * u / (1 - (N - 1) * u)
    bound = gam * np.abs(g.astype(np.float64)).sum(0)
    assert np.all(np.abs(out[0].astype(np.float64) - exact) <= bound + 1e-300)
    for r in range(1, N):
        assert np.array_equal(out[r], out[0])
    ps = orc.ps_allreduce(g)
    assert np.all(np.abs(ps.astype(np.float64) - exact) <= bound + 1e-300)


def test_replay_equals_chain_random(orc):
    rng = np.random.default_rng(11)
    for N in (2, 3, 6, 8):
        K_pad = orc.kpad(333, N)
        g = rng.standard_normal((N, K_pad)).astype(np.float32)
        for op in (orc.SUM, orc.MEAN):
            out, _ = orc.ring_allreduce(g, op)
            assert np.array_equal(out[N - 1], orc.ring_chain(g, op))


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_mean_is_exact_division_for_power_of_two(orc, N):
    rng = np.random.default_rng(3)
    K_pad = orc.kpad(100, N)
    g = rng.standard_normal((N, K_pad)).astype(np.float32)
    s, _ = orc.ring_allreduce(g, orc.SUM)
    m, _ = orc.ring_allreduce(g, orc.MEAN)
    assert np.array_equal(m[0], s[0] / np.float32(N))


def test_sgd_lr_zero_and_fused_equals_unfused(orc):
    rng = np.random.default_rng(5)
    for N in (1, 2, 3, 4, 8):
        K_pad = orc.kpad(257, N)
        g = rng.standard_normal((N, K_pad)).astype(np.float32)
        w = rng.standard_normal(K_pad).astype(np.float32)
        p0 = orc.ring_sgd(g, w, 0.0)  # lr = 0 -> params unchanged
        for r in range(N):
            assert np.array_equal(p0[r], w)
        lr = np.float32(0.0375)
        p = orc.ring_sgd(g, w, float(lr))
        gbar = orc.ring_chain(g, orc.MEAN)
        # unfused: allreduce, then every rank updates with a single-rounding fma
        ref = (w.astype(np.float64) - np.float64(lr) * gbar.astype(np.float64))
        ref32 = ref.astype(np.float32)  # fma(-lr, g, w) rounds once: exact product, then one RN
        for r in range(N):
            assert np.array_equal(p[r], ref32)


def test_ps_ascending_order(orc):
    """PS sums in ascending rank order -- order witness at N=3 gives 1 everywhere,
    while the ring gives [1, 0, 0]: the two strategies differ only in association."""
    w = gold("order_witness.json")
    g = np.ones((3, 12), np.float32)
    g[0] = w["big"]
    g[1] = -w["big"]
    assert np.all(orc.ps_allreduce(g) == 1.0)


# ------------------------------------------------------------------ Adam owner update (R22)
def _adam_ref64(gbar, w, m, v, b1t, b2t, lr, b1, b2, eps):
    """Textbook Adam (Kingma & Ba, Alg. 1) in float64, for the tolerance pin."""
    m = b1 * m + (1 - b1) * gbar
    v = b2 * v + (1 - b2) * gbar * gbar
    mhat = m / (1 - b1t)
    vhat = v / (1 - b2t)
    return w - lr * mhat / (np.sqrt(vhat) + eps), m, v


def test_ring_adam_matches_textbook_adam(orc):
    """Three steps of the oracle's fused ring mean + Adam vs textbook float64 Adam on the
    float64 mean gradient: agreement within a few fp32 ulps of the update size."""
    rng = np.random.default_rng(5)
    N, K = 4, 4096
    w = rng.standard_normal(K).astype(np.float32)
    m = np.zeros(K, np.float32)
    v = np.zeros(K, np.float32)
    sc = np.ones(2, np.float32)
    w64, m64, v64 = w.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    for t in range(1, 4):
        g = rng.standard_normal((N, K)).astype(np.float32)
        w, m, v, sc = orc.ring_adam(g, w, m, v, sc, lr, b1, b2, eps)
        gbar = g.astype(np.float64).mean(axis=0)
        w64, m64, v64 = _adam_ref64(gbar, w64, m64, v64, b1 ** t, b2 ** t, lr, b1, b2, eps)
        assert np.allclose(sc, [np.float32(b1) ** t, np.float32(b2) ** t], rtol=1e-6)
        assert np.abs(w - w64).max() <= 1e-6 * max(1.0, np.abs(w64).max())
        assert np.allclose(m, m64, rtol=1e-5, atol=1e-7)


def test_ring_adam_first_step_is_sign_step(orc):
    """Closed form at t = 1 from zero state: mhat = g, vhat = g^2, so w' = w - lr*g/(|g|+eps)
    (= w - lr*sign(g) for |g| >> eps) -- Adam's first step."""
    N, K = 2, 1000
    g = np.random.default_rng(2).standard_normal((N, K)).astype(np.float32)
    w = np.zeros(K, np.float32)
    lr = 0.01
    w1, _, _, _ = orc.ring_adam(g, w, np.zeros(K, np.float32), np.zeros(K, np.float32), np.ones(2, np.float32), lr)
    gbar = g.astype(np.float64).mean(axis=0)
    assert np.allclose(w1, -lr * gbar / (np.abs(gbar) + 1e-8), rtol=1e-5, atol=1e-9)


def test_ring_adam_uses_ring_order_sum(orc):
    """The gradient fed to Adam is the ring chain sum (order witness inputs, N = 3): with
    lr = 0, beta1 = 0 the new m is exactly (1 - 0) * gbar = the ring's mean."""
    N, K = 3, 6
    big = np.float32(2.0 ** 25)
    g = np.stack([np.full(K, big), np.full(K, -big), np.ones(K)]).astype(np.float32)
    _, m, _, _ = orc.ring_adam(g, np.zeros(K, np.float32), np.zeros(K, np.float32), np.zeros(K, np.float32),
                               np.ones(2, np.float32), 0.0, beta1=0.0)
    expect, _ = orc.ring_allreduce(g, 1)
    assert np.array_equal(m, expect[0])


def test_ring_momentum_zero_mu_is_sgd(orc):
    """mu = 0: u = gbar exactly, and the update is the plain SGD step of R12 bit for bit."""
    rng = np.random.default_rng(11)
    N, K = 4, 4096
    g = rng.standard_normal((N, K)).astype(np.float32)
    w = rng.standard_normal(K).astype(np.float32)
    w1, u1 = orc.ring_momentum(g, w, np.zeros(K, np.float32), 0.05, 0.0)
    assert np.array_equal(w1, orc.ring_sgd(g, w, 0.05)[0])
    assert np.array_equal(u1, orc.ring_allreduce(g, 1)[0][0])


def test_ring_momentum_constant_gradient_closed_form(orc):
    """Constant gradient g (identical on every rank, so the mean is exact): after t steps
    u_t = g (1 - mu^t) / (1 - mu) and w_t = w_0 - lr g sum_{s=1..t} (1 - mu^s) / (1 - mu)."""
    N, K, lr, mu = 2, 64, 0.01, 0.9
    gv = np.linspace(-2, 2, K).astype(np.float32)
    g = np.stack([gv] * N)
    w = np.zeros(K, np.float32)
    u = np.zeros(K, np.float32)
    acc = 0.0
    for t in range(1, 11):
        w, u = orc.ring_momentum(g, w, u, lr, mu)
        acc += (1 - mu ** t) / (1 - mu)
        assert np.allclose(u, gv * (1 - mu ** t) / (1 - mu), rtol=1e-5, atol=1e-6), t
        assert np.allclose(w, -lr * gv * acc, rtol=1e-5, atol=1e-6), t


def test_ring_momentum_matches_float64_heavy_ball(orc):
    """Random gradients, 5 steps: within fp32 rounding of float64 heavy-ball on the float64 mean."""
    rng = np.random.default_rng(12)
    N, K, lr, mu = 3, 999, 0.02, 0.9
    Kp = orc.kpad(K, N)
    w = rng.standard_normal(Kp).astype(np.float32)
    u = np.zeros(Kp, np.float32)
    w64, u64 = w.astype(np.float64), u.astype(np.float64)
    for _ in range(5):
        g = rng.standard_normal((N, Kp)).astype(np.float32)
        w, u = orc.ring_momentum(g, w, u, lr, mu)
        u64 = mu * u64 + g.astype(np.float64).mean(axis=0)
        w64 = w64 - lr * u64
        assert np.abs(u - u64).max() <= 1e-5 * max(1.0, np.abs(u64).max())
        assert np.abs(w - w64).max() <= 1e-5 * max(1.0, np.abs(w64).max())
