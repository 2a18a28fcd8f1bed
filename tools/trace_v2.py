"""Per-step role timeline of the tensor-core decode pipeline (CTA 0, first 64 steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup  # noqa: E402

ROLES = ["copies", "QK iss", "S ready", "P done", "PV iss", "full@MMA", "empty@prod", "S loaded", "max done", "P stored"]
import sys as _s
BS = int(_s.argv[1]) if len(_s.argv) > 1 else 16
for wl in (W.hybrid(W.Shape(32, 8, 128, BS, "bf16"), f"decode-only-64-B{BS}", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2),):
    kv, plan, q, o, lse = setup(wl, dict(decode_path=1))
    for _ in range(3):
        kv.attention(plan, 0, q, o, lse)
    buf = torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda")
    kv.debug_trace(buf)
    kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    kv.debug_trace(None)
    b = buf.cpu().numpy()
    ev = b[160 * 8:].reshape(10, 64)
    base = ev[ev > 0].min()
    print(wl.name)
    print("  j " + " ".join(f"{r:>10s}" for r in ROLES))
    for j in range(24):
        print(f" {j:2d} " + " ".join(f"{(ev[r, j] - base) / 1e3:10.2f}" if ev[r, j] > 0 else f"{'-':>10s}" for r in range(10)))
    cta = b[:160 * 8].reshape(160, 8)
    cta = cta[cta[:, 0] > 0]
    t0 = cta[:, 6].min()
    print(f"  CTA exit max {(cta[:, 2].max() - t0) / 1e3:.1f} us, decode end med {(sorted(cta[:, 4])[len(cta)//2] - t0) / 1e3:.1f}")
