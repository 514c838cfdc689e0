#!/usr/bin/env python
"""Small collective workload for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_collectives.py

Runs the single-device emulation (N ranks as CTA groups of one cooperative launch) of the ring,
two-shot and PS allreduce at N = 2, 3, 4 with ragged K, one tem_step exchange at N = 2, and the
production one-rank launch against pre-written virtual-peer messages (tests/test_gpu_wire.py's
protocol), and checks every result against the oracle.  Exit 0 = all results bit-exact.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
from paper_1906_06496_b200 import tem  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    for N in (2, 3, 4):
        K = 4099
        sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=1, max_allreduce_elems=K,
                               ring_channels=2)
        s = tem.TemSession(sc, datagen.init_params())
        Kp = oracle.kpad(K, N)
        for name, fn, ref in (("ring", s.allreduce, lambda g: oracle.ring_allreduce(g, 0)[0]),
                              ("twoshot", s.twoshot_allreduce, lambda g: oracle.ring_allreduce(g, 0)[0]),
                              ("ps", s.ps_allreduce, lambda g: np.broadcast_to(oracle.ps_allreduce(g, 0), g.shape))):
            g = np.zeros((N, Kp), np.float32)
            g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
            for r in range(N):
                s.user(r, Kp).copy_(torch.from_numpy(g[r]))
            fn(K, 0)
            code, _ = s.sync()
            assert code == 0, (name, N, tem.status_string(code))
            exp = ref(g)
            for r in range(N):
                assert np.array_equal(s.user(r, K).cpu().numpy(), exp[r][:K]), (name, N, r)
            print(f"ok {name} N={N}")
        s.close()
    # production launch (one rank per process) against virtual peers
    import test_gpu_wire as W
    N, r, K = 3, 1, 2053
    sc = tem.SessionConfig(world_size=N, rank=r, local_ranks=1, batch_per_rank=1, ring_channels=W.G,
                           max_allreduce_elems=K)
    s = tem.TemSession(sc, datagen.init_params(), virtual_peers=True)
    Kp = oracle.kpad(K, N)
    g = np.zeros((N, Kp), np.float32)
    g[:, :K] = rng.standard_normal((N, K)).astype(np.float32)
    final = oracle.ring_allreduce(g, 0)[0][0]
    final[K:] = 0.0
    s.user(0, Kp).copy_(torch.from_numpy(g[r]))
    W.transcript_in(oracle, s, g, final, r, 1, K, 0, 0)
    torch.cuda.synchronize()
    s.allreduce(K, 0)
    code, _ = s.sync()
    assert code == 0, tem.status_string(code)
    assert np.array_equal(s.user(0, K).cpu().numpy(), final[:K])
    W.check_transcript_out(oracle, s, g, final, r, 1)
    s.close()
    print("ok production one-rank ring vs virtual peers")
    print("ALL OK")


if __name__ == "__main__":
    main()
