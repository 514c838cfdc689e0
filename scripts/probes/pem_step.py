#!/usr/bin/env python
"""Run a few joint TEM + PEM steps (c5 shape) for ncu / compute-sanitizer (diagnostics)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import tem
    B, P = 16, datagen.PEM_P
    sc = tem.SessionConfig(batch_per_rank=B, precision=0, lr=0.01, pem_proposals=P)
    s = tem.TemSession(sc, np.concatenate([datagen.init_params(), datagen.init_pem_params()]))
    x = torch.from_numpy(datagen.features(B)).cuda()
    lab = torch.from_numpy(datagen.labels(B)).cuda()
    f = torch.from_numpy(datagen.bsp_features(B)).cuda()
    g = torch.from_numpy(datagen.iou_targets(B)).cuda()
    for _ in range(3):
        s.step_pem(x, lab, f, g)
    code, _ = s.sync()
    print("status", tem.status_string(code))
    s.close()
    return 0 if code == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
