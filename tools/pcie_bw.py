"""Pinned host <-> device copy bandwidth on this box (the e2e leg's bound): H2D and D2H of the
config-2 step's buffers, alone and concurrently on two streams."""
import time

import torch


def bw(nbytes, h2d=True, d2h=True, reps=50):
    h_in = torch.empty(nbytes[0], dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes[1], dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes[0], dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nbytes[1], dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


n = (7077888, 4718592)
t = bw(n, True, False)
print(f"H2D {n[0] / 1e6:.1f} MB: {t * 1e6:.1f} us = {n[0] / t / 1e9:.1f} GB/s")
t = bw(n, False, True)
print(f"D2H {n[1] / 1e6:.1f} MB: {t * 1e6:.1f} us = {n[1] / t / 1e9:.1f} GB/s")
t = bw(n, True, True)
print(f"both concurrently: {t * 1e6:.1f} us per step")
