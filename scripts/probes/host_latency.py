#!/usr/bin/env python
"""Host-side latency of tem_step / tem_step_pem calls (no sync) -- diagnostics."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import datagen
    from paper_1906_06496_b200 import tem
    for P in (0, datagen.PEM_P):
        B = 16
        sc = tem.SessionConfig(batch_per_rank=B, precision=0, lr=0.01, pem_proposals=P)
        p0 = datagen.init_params() if not P else np.concatenate([datagen.init_params(), datagen.init_pem_params()])
        s = tem.TemSession(sc, p0)
        x = torch.from_numpy(datagen.features(B)).cuda()
        lab = torch.from_numpy(datagen.labels(B)).cuda()
        f = torch.from_numpy(datagen.bsp_features(B)).cuda()
        g = torch.from_numpy(datagen.iou_targets(B)).cuda()
        step = (lambda: s.step_pem(x, lab, f, g)) if P else (lambda: s.step(x, lab))
        for _ in range(10):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(300):
            t0 = time.perf_counter()
            step()
            ts.append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
        ts.sort()
        print(f"P={P}: host us per call: median {ts[150]:.1f} p99 {ts[297]:.1f} max {ts[-1]:.1f}")
        s.close()


if __name__ == "__main__":
    main()
