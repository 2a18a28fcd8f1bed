"""Per-CTA phase timeline + CTA 0 prefill pipeline event log (niyama_debug_trace)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup  # noqa: E402

ROLES = ["K issue", "V issue", "QK issue", "PV issue", "S ready", "max done", "P arrive", "O waited", "exps done",
         "QK issued"]


def run(wl):
    from kbench import time_it
    time_it(wl)
    kv, plan, q, o, lse = setup(wl)
    for _ in range(3):
        kv.attention(plan, 0, q, o, lse)
    buf = torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda")
    kv.debug_trace(buf)
    kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    kv.debug_trace(None)
    b = buf.cpu().numpy()
    cta = b[:160 * 8].reshape(160, 8)
    cta = cta[cta[:, 0] > 0]
    t0 = cta[:, 0].min()
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    print(f"== {wl.name}: {len(cta)} CTAs")
    pre = cta[cta[:, 3] > 0]
    if len(pre):
        print(f"  prefill CTAs {len(pre)}: prefill end {us(pre[:,1].min()):.1f} .. {us(pre[:,1].max()):.1f} us")
    dec = cta[cta[:, 4] > 0]
    if len(dec):
        def mmm(x):
            return f"{us(x.min()):.1f} / {us(np.median(x)):.1f} / {us(x.max()):.1f}"
        f7 = dec[dec[:, 7] > 0]
        if len(f7):
            print(f"  warp0 first stage consumed {mmm(f7[:, 7])} us (min/med/max)")
        f5 = dec[dec[:, 5] > 0]
        if len(f5):
            print(f"  warp0 queue exhausted      {mmm(f5[:, 5])} us")
        print(f"  decode+merge end           {mmm(dec[:, 4])} us")
    print(f"  CTA exit     {us(cta[:,2].min()):.1f} / {us(np.median(cta[:,2])):.1f} / {us(cta[:,2].max()):.1f} us")
    e0 = cta[:, 6].min()
    print(f"  entry -> start: {(cta[:,0]-cta[:,6]).min()/1e3:.2f} .. {(cta[:,0]-cta[:,6]).max()/1e3:.2f} us; "
          f"entry spread {(cta[:,6].max()-e0)/1e3:.2f} us; first entry -> last exit {(cta[:,2].max()-e0)/1e3:.1f} us")
    ev = b[160 * 8:].reshape(10, 64)
    if (ev > 0).any():
        base = ev[ev > 0].min()
        n = int((ev[4] > 0).sum())
        print("  CTA0 prefill tile events (kcycles from first event):")
        print("   j " + " ".join(f"{r:>9s}" for r in ROLES))
        for j in range(n):
            print(f"  {j:2d} " + " ".join(f"{(ev[r, j] - base) / 1e3:9.2f}" if ev[r, j] > 0 else f"{'-':>9s}"
                                          for r in range(10)))


def gap(wl):
    """Last CTA exit of launch i vs first CTA entry of launch i+1 (back to back, no host sync)."""
    kv, plan, q, o, lse = setup(wl)
    for _ in range(3):
        kv.attention(plan, 0, q, o, lse)
    bufs = [torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda") for _ in range(3)]
    torch.cuda.synchronize()
    for b in bufs:
        kv.debug_trace(b)
        kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    kv.debug_trace(None)
    tr = [b.cpu().numpy()[:160 * 8].reshape(160, 8) for b in bufs]
    tr = [t[t[:, 0] > 0] for t in tr]
    for i in range(2):
        print(f"  {wl.name}: launch {i} first entry -> last exit {(tr[i][:, 2].max() - tr[i][:, 6].min()) / 1e3:.1f} us; "
              f"last exit -> next first entry {(tr[i + 1][:, 6].min() - tr[i][:, 2].max()) / 1e3:.2f} us")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "l70b":
        run(W.config4_l70b())
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "l70b-prefill":
        run(W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4))
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "gap":
        gap(W.config2_l8b())
        gap(W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2))
        sys.exit(0)
    run(W.hybrid(W.L8B, "prefill-only-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2))
    if len(sys.argv) < 2:
        run(W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2))
        run(W.config2_l8b())

