#!/usr/bin/env python
"""report.py -- the paper's training-time metrics over a scaling run.

    python report.py bench_n1.json bench_n2.json ... [--ps ps_n2.json ...]

Each input holds one bench.py JSON line (or the driver's SCALE_rNN.json list).  For every n
the training time of a fixed dataset is t(n) = epoch_videos / samples_per_s(n) + t3 (P:163:
t1 + t2 per step over the epoch, plus setup t3).  Prints the speed ratio t0/t, the
scaling efficiency, and least-squares fits of Eq. (1) t = T/n + C*n + P (PS) and Eq. (2)
t = T/n + C*n/(n-1) + P (ring) with their residuals and the crossover.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1906_06496_b200 import metrics as M  # noqa: E402


def load(paths):
    rows = []
    for p in paths:
        txt = open(p).read().strip()
        try:
            d = json.loads(txt)
            rows.extend(d if isinstance(d, list) else [d])
        except json.JSONDecodeError:
            rows.extend(json.loads(l) for l in txt.splitlines() if l.startswith("{"))
    out = {}
    for d in rows:
        if "value" not in d or "n_gpus" not in d:
            continue
        pm = d.get("paper_metrics", {})
        ep = pm.get("epoch_videos", 9997)
        out[int(d["n_gpus"])] = ep / float(d["value"]) + float(pm.get("t3_setup_s", 0.0))
    return out


def summarize(times: dict, kind: str):
    ns = sorted(times)
    res = {"kind": kind, "t": {n: times[n] for n in ns}}
    if 1 in times:
        res["speed_ratio"] = {n: M.speed_ratio(times[1], times[n]) for n in ns}
        res["efficiency"] = {n: M.speed_ratio(times[1], times[n]) / n for n in ns}
    fit_ns = [n for n in ns if n >= 2]
    if len(fit_ns) >= 3:
        for basis in (M.PS, M.RING):
            rep = M.fit_cost_model([(n, times[n]) for n in fit_ns], basis)
            res[f"fit_eq{1 if basis == M.PS else 2}"] = rep.to_json()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ring", nargs="+", help="bench JSON files of the ring exchange (n = 1..8)")
    ap.add_argument("--ps", nargs="*", default=[], help="bench JSON files with --exchange ps")
    args = ap.parse_args()
    out = {"ring": summarize(load(args.ring), "ring")}
    if args.ps:
        out["ps"] = summarize(load(args.ps), "ps")
        try:
            ps = M.CostModel(M.PS, **{k: out["ps"]["fit_eq1"]["model"][k] for k in ("T", "C", "P")})
            ring = M.CostModel(M.RING, **{k: out["ring"]["fit_eq2"]["model"][k] for k in ("T", "C", "P")})
            out["crossover_n"] = M.crossover(ps, ring, 1024)
        except KeyError:
            pass
    out["paper_fits_context"] = {"ps": vars(M.PAPER_PS), "ring": vars(M.PAPER_RING),
                                 "crossover_n": M.crossover(M.PAPER_PS, M.PAPER_RING, 64),
                                 "hardware": "8 x 'TITAN V-100', TensorFlow, MPI ring (P:186)"}
    print(json.dumps(out, indent=1, default=float))


if __name__ == "__main__":
    main()
