#!/usr/bin/env python
"""Run a few tem_step calls of a workload (for ncu / compute-sanitizer captures).

    python scripts/prof_step.py [--workload c2|c3|c1|c5|c6] [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--ranks", type=int, default=1, help="emulated ranks on this device")
    args = ap.parse_args()
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import tem
    B, prec, P = {"c1": (4, 0, 0), "c2": (16, 0, 0), "c3": (256, 1, 0), "c5": (16, 0, datagen.PEM_P),
                  "c6": (16, 0, datagen.PEM_P)}[args.workload]
    G = datagen.GT_MAX if args.workload == "c6" else 0
    N = args.ranks
    sc = tem.SessionConfig(world_size=N, rank=0, local_ranks=N, batch_per_rank=B, precision=prec, lr=0.01,
                           pem_proposals=P, pgm_gt_max=G)
    p0 = datagen.init_params() if not P else np.concatenate([datagen.init_params(), datagen.init_pem_params()])
    s = tem.TemSession(sc, p0)
    xs = np.stack([datagen.features(B, rank=r) for r in range(N)])
    lab = torch.from_numpy(np.stack([datagen.labels(B, rank=r) for r in range(N)])).cuda()
    x = torch.from_numpy(datagen.to_bf16_bits(xs).view(np.int16)).cuda() if prec == 1 else torch.from_numpy(xs).cuda()
    if G:
        gt = torch.from_numpy(np.stack([datagen.instances(B, rank=r)[0] for r in range(N)])).cuda()
        ng = torch.from_numpy(np.stack([datagen.instances(B, rank=r)[1] for r in range(N)])).cuda()
    elif P:
        f = torch.from_numpy(np.stack([datagen.bsp_features(B, rank=r) for r in range(N)])).cuda()
        g = torch.from_numpy(np.stack([datagen.iou_targets(B, rank=r) for r in range(N)])).cuda()
    for _ in range(args.steps):
        if G:
            s.step_pgm(x, lab, gt, ng)
        elif P:
            s.step_pem(x, lab, f, g)
        else:
            s.step(x, lab)
    code, _ = s.sync()
    torch.cuda.synchronize()
    print("path", s.kernel_path(), "status", tem.status_string(code), "loss", s.loss[0].tolist())
    s.close()
    return 0 if code == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
