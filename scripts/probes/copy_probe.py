#!/usr/bin/env python
"""H2D / D2H costs of the e2e step's copies (diagnostics; needs a GPU)."""
import torch


def t(fn, reps=50):
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) * 1e3 for a, b in ev[5:])
    return v[len(v) // 2]


def main():
    x_h = torch.randn(16, 100, 400).pin_memory()
    l_h = torch.rand(16, 3, 100).pin_memory()
    both_h = torch.empty(x_h.numel() + l_h.numel()).pin_memory()
    x_d, l_d, both_d = torch.empty_like(x_h, device="cuda"), torch.empty_like(l_h, device="cuda"), torch.empty_like(both_h, device="cuda")
    loss_d, loss_h = torch.zeros(4, device="cuda"), torch.zeros(4).pin_memory()
    print(f"H2D x 2.56 MB     : {t(lambda: x_d.copy_(x_h, non_blocking=True)):7.1f} us")
    print(f"H2D labels 19 KB  : {t(lambda: l_d.copy_(l_h, non_blocking=True)):7.1f} us")
    print(f"H2D x+labels (two): {t(lambda: (x_d.copy_(x_h, non_blocking=True), l_d.copy_(l_h, non_blocking=True))):7.1f} us")
    print(f"H2D one 2.58 MB   : {t(lambda: both_d.copy_(both_h, non_blocking=True)):7.1f} us")
    print(f"D2H loss 16 B     : {t(lambda: loss_h.copy_(loss_d, non_blocking=True)):7.1f} us")
    big_h = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
    big_d = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    us = t(lambda: big_d.copy_(big_h, non_blocking=True), 20)
    print(f"H2D 64 MB         : {us:7.1f} us = {64 * 1.048576 / us * 1e3:.1f} GB/s")


if __name__ == "__main__":
    main()
