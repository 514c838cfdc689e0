#!/usr/bin/env python
"""Per-step overhead of a graph launch bracketed by events (as bench.py times a step), versus
the GPU span of its kernels (diagnostics; needs a GPU)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    dev = torch.device("cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for nk in (1, 9):
        xs = [torch.zeros(256, device=dev) for _ in range(nk)]
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for x in xs:
                x.add_(1.0)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for x in xs:
                    x.add_(1.0)
        for mode in ("flush", "back-to-back"):
            ts = []
            for it in range(30):
                if mode == "flush":
                    flush.fill_(it & 255)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                g.replay()
                b.record()
                ts.append((a, b))
            torch.cuda.synchronize()
            us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts[5:])
            print(f"graph of {nk} tiny kernels, {mode:>12}: median {us[len(us)//2]:.1f} us per replay")


if __name__ == "__main__":
    main()
