#!/usr/bin/env python
"""The paper's training-time metrics from measured components on ONE B200.

    python scripts/paper_metrics_emulated.py [--out profiles/r02_paper_metrics_emulated.json]

This pool has one GPU, so no N > 1 step runs as N processes.  What is measured here:
  * t1(B): one rank's step on B videos at N = 1 -- forward + backward + the owner update, the
    graph-replayed tem_step bench.py times (CUDA events, L2 flushed before every step, median of
    50) -- the paper's per-iteration compute; at N > 1 the ring's owner does the same
    update work, fused into the exchange;
  * t2(n): the exchange of the 1,403,395-element TEM gradient among n ranks, for the paper's
    ring (KR1), the parameter server (KP1) and the NVSwitch two-shot, with the n
    ranks EMULATED as CTA groups of one cooperative launch on this GPU (bench_ring.py
    --emulate): all n ranks' traffic shares one GPU's memory system and no NVLink is involved,
    so t2(n) is the protocols' dependent-round latency plus n x the per-rank memory traffic --
    not an 8-GPU NVLink measurement;
  * t3: session set-up (rendezvous-free here: allocation, tem_init, plan) ("P").
The script then composes t(n) = t1 + t2(n) per iteration and reports, as report.py does for
real N-GPU bench lines: weak scaling at 16 videos per rank (samples/s, speedup, efficiency),
the PS-vs-ring speed ratio (Fig. 7 analog), and Eq. (1) / Eq. (2) fits of the training time of
one epoch (9,997 videos) at a fixed global batch of ~128 split n ways (B = round(128/n)).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

K_TEM = 1403395
EPOCH = 9997


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_paper_metrics_emulated.json"))
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import metrics as M
    from paper_1906_06496_b200 import tem

    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def timed(fn, reps):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return statistics.median(ts)

    # ---- t1(B), t3
    t1, t3 = {}, None
    for B in sorted({16, 128, 64, 43, 32, 26, 21, 18}):
        t0 = time.perf_counter()
        s = tem.TemSession(tem.SessionConfig(batch_per_rank=B, lr=0.01), datagen.init_params())
        if B == 16:
            torch.cuda.synchronize()
            t3 = time.perf_counter() - t0
        x = torch.from_numpy(datagen.features(B)).cuda()[None]
        lab = torch.from_numpy(datagen.labels(B)).cuda()[None]
        t1[B] = timed(lambda: s.step(x, lab), args.reps)
        s.close()
    t_step1 = t1[16]

    # ---- t2(n): emulated exchanges of the TEM gradient
    t2 = {"ring": {}, "ps": {}, "twoshot": {}}
    for n in range(2, 9):
        sc = tem.SessionConfig(world_size=n, rank=0, local_ranks=n, batch_per_rank=1, max_allreduce_elems=K_TEM)
        s = tem.TemSession(sc, datagen.init_params())
        rng = np.random.default_rng(n)
        for r in range(n):
            s.user(r, K_TEM).copy_(torch.from_numpy(rng.standard_normal(K_TEM).astype(np.float32) * 1e-3))
        t2["ring"][n] = timed(lambda: s.allreduce(K_TEM, tem.TEM_SUM), 20)
        t2["ps"][n] = timed(lambda: s.ps_allreduce(K_TEM, tem.TEM_SUM), 20)
        t2["twoshot"][n] = timed(lambda: s.twoshot_allreduce(K_TEM, tem.TEM_SUM), 20)
        code, _ = s.sync()
        assert code == 0, tem.status_string(code)
        s.close()

    out = {"what": __doc__.split("\n\n")[1].strip(), "t1_s": t1, "t_step_n1_s": t_step1, "t3_s": t3,
           "t2_emulated_s": t2, "K": K_TEM}
    # ---- weak scaling, 16 videos per rank
    weak = {}
    for kind in t2:
        rows = {1: {"t_iter_s": t_step1, "samples_per_s": 16 / t_step1}}
        for n in range(2, 9):
            t = t1[16] + t2[kind][n]
            rows[n] = {"t_iter_s": t, "samples_per_s": 16 * n / t}
        for n in rows:
            rows[n]["speedup"] = rows[n]["samples_per_s"] / rows[1]["samples_per_s"]
            rows[n]["efficiency"] = rows[n]["speedup"] / n
        weak[kind] = rows
    out["weak_scaling_B16"] = weak
    out["ps_vs_ring_speed_ratio"] = {n: M.speed_ratio(weak["ps"][n]["t_iter_s"], weak["ring"][n]["t_iter_s"])
                                     for n in range(2, 9)}
    # ---- fixed global batch ~128 split n ways: epoch training time, Eq. (1) / (2) fits
    Bn = {1: 128, 2: 64, 3: 43, 4: 32, 5: 26, 6: 21, 7: 18, 8: 16}
    epoch = {}
    for kind in t2:
        rows = {}
        for n in range(1, 9):
            t_iter = t1[Bn[n]] + (t2[kind][n] if n > 1 else 0.0)
            iters = EPOCH / (Bn[n] * n)
            rows[n] = iters * t_iter + t3
        epoch[kind] = rows
    out["epoch_time_s_global_batch_128"] = epoch
    fits = {}
    for kind, basis in (("ps", M.PS), ("ring", M.RING), ("twoshot", M.RING)):
        rep = M.fit_cost_model([(n, epoch[kind][n]) for n in range(2, 9)], basis)
        fits[kind] = rep.to_json()
    out["fits"] = fits
    try:
        out["crossover_n_ps_vs_ring"] = M.crossover(M.CostModel(M.PS, **{k: fits["ps"]["model"][k] for k in "TCP"}),
                                                    M.CostModel(M.RING, **{k: fits["ring"]["model"][k] for k in "TCP"}),
                                                    1024)
    except Exception:
        pass
    out["paper_fits_context"] = {"ps": vars(M.PAPER_PS), "ring": vars(M.PAPER_RING),
                                 "hardware": "8 x 'TITAN V-100', TensorFlow, MPI ring (P:186)"}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1, default=float)
    print(f"t1(16) = N=1 step {t1[16] * 1e6:.1f} us, t3 = {t3:.3f} s")
    for n in range(2, 9):
        print(f"n={n}: t2 ring {t2['ring'][n] * 1e6:6.1f}  ps {t2['ps'][n] * 1e6:6.1f}  twoshot "
              f"{t2['twoshot'][n] * 1e6:6.1f} us | weak ring {weak['ring'][n]['samples_per_s'] / 1e3:7.1f} k/s "
              f"eff {weak['ring'][n]['efficiency']:.3f} | ps/ring ratio {out['ps_vs_ring_speed_ratio'][n]:.3f}")
    for kind in fits:
        f = fits[kind]
        print(f"Eq. ({1 if kind == 'ps' else 2}) {kind}: T={f['model']['T']:.4g} C={f['model']['C']:.4g} "
              f"P={f['model']['P']:.4g} rms={f['residual_rms']:.3g} valid={f['valid']}")


if __name__ == "__main__":
    main()
