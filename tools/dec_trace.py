"""Per-stage cycle breakdown of one decode warp (CTA 0, warp 0, first 64 stages)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup  # noqa: E402

ROLES = ["top", "data ready", "QK done", "softmax done", "PV+publish done", "refill issued"]


def run(wl):
    kv, plan, q, o, lse = setup(wl)
    for _ in range(3):
        kv.attention(plan, 0, q, o, lse)
    buf = torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda")
    kv.debug_trace(buf)
    kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    kv.debug_trace(None)
    ev = buf.cpu().numpy()[160 * 8:].reshape(10, 64)[:6]
    n = int((ev[5] > 0).sum())
    d = np.diff(ev[:, :n], axis=0)
    per = (ev[0, 1:n] - ev[0, :n - 1])
    print(f"== {wl.name}: {n} stages; cycles per stage median {np.median(per):.0f}")
    for i in range(5):
        print(f"  {ROLES[i]:>16s} -> {ROLES[i + 1]:<16s} median {np.median(d[i]):7.0f}  mean {d[i].mean():7.0f}")
    print(f"  {'refill issued':>16s} -> next top        median {np.median(ev[0, 1:n] - ev[5, :n - 1]):7.0f}")


if __name__ == "__main__":
    run(W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2))
    run(W.hybrid(W.L8B, "decode-256x4096", prefill_offset=0, chunk=0, decode_ctx=[4096] * 256, seed=2))
