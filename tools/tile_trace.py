"""Per-tile timeline of CTA 0's prefill tiles (build with -DNIYAMA_DIAG_TILES=1 via
tools/build_variant.py and select it with NIYAMA_LIB_PATH): claim -> Q ready -> tile end, in
kcycles, with the tile's key steps, and the gap between one tile's end and the next tile's
first step (the per-tile setup the a8 fit calls sigma).

    python tools/tile_trace.py [l70b|l8b|l8b-mixed|l70b-mixed]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup, time_it  # noqa: E402


def run(wl):
    time_it(wl, reps=20)
    kv, plan, q, o, lse = setup(wl)
    for _ in range(3):
        kv.attention(plan, 0, q, o, lse)
    buf = torch.zeros(160 * 8 + 10 * 64, dtype=torch.int64, device="cuda")
    kv.debug_trace(buf)
    kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    kv.debug_trace(None)
    ev = buf.cpu().numpy()[160 * 8:].reshape(10, 64)
    n = int((ev[2] > 0).sum())
    s = wl.shape
    d = wl.final.desc
    g = s.num_q_heads // s.num_kv_heads
    R = 128 // g
    o_, c_ = d.prefill_offset[0], d.prefill_len[0]
    nqt = (c_ + R - 1) // R
    base = ev[0, 0]
    tot_steps = 0
    print(f"== {wl.name}: CTA 0 ran {n} tiles")
    print("  tile item steps    claim    Qready      end   claim->Q   Q->end  cyc/step  end->next claim")
    for t in range(n):
        item = int(ev[4, t])
        qt = nqt - 1 - item // s.num_kv_heads
        nkeys = o_ + min(qt * R + R, c_)
        steps = (nkeys + 127) // 128
        tot_steps += steps
        nxt = (ev[0, t + 1] - ev[2, t]) / 1e3 if t + 1 < 64 and ev[0, t + 1] > 0 else float("nan")
        print(f"  {t:4d} {item:4d} {steps:5d} {(ev[0, t] - base) / 1e3:8.1f} {(ev[1, t] - base) / 1e3:9.1f} "
              f"{(ev[2, t] - base) / 1e3:8.1f} {(ev[1, t] - ev[0, t]) / 1e3:9.2f} {(ev[2, t] - ev[1, t]) / 1e3:8.1f} "
              f"{(ev[2, t] - ev[1, t]) / steps:9.0f} {nxt:9.2f}")
    span = (ev[2, n - 1] - ev[0, 0]) / 1e3
    print(f"  total {span:.1f} kcycles for {tot_steps} steps = {span * 1e3 / max(tot_steps, 1):.0f} cycles/step "
          f"(incl. setup)")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "l70b"
    wl = {"l70b": lambda: W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048,
                                   decode_ctx=[], seed=4),
          "l8b": lambda: W.hybrid(W.L8B, "l8b-prefill-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[],
                                  seed=2),
          "l8b-c2048": lambda: W.hybrid(W.L8B, "l8b-prefill-c2048-o2048", prefill_offset=2048, chunk=2048,
                                        decode_ctx=[], seed=4),
          "l8b-mixed": W.config2_l8b, "l70b-mixed": W.config4_l70b}[which]()
    run(wl)
