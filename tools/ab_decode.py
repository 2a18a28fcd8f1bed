"""A/B of the bf16 decode paths (niyama_tuning.decode_path: 0 per-warp mma.sync (default),
1 tensor-core CTA pipeline): output agreement between the two and launch times (median of
back-to-back launches, tools/kbench.time_it) on configs 2 and 4 and decode-only batches.

    python tools/ab_decode.py [--quick]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup, time_it  # noqa: E402


def outputs(wl, path, block=None):
    kv, plan, q, o, lse = setup(wl, dict(decode_path=path))
    kv.attention(plan, 0, q, o, lse)
    torch.cuda.synchronize()
    return o.float().cpu(), lse.cpu()


def main():
    quick = "--quick" in sys.argv
    cases = [W.random_hybrid(W.L8B, seed=5, num_prefill=1, max_chunk=200, num_decode=12, max_ctx=3000),
             W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2),
             W.config2_l8b()]
    if not quick:
        cases.append(W.config4_l70b())
    for wl in cases:
        (o0, l0), (o1, l1) = outputs(wl, 0), outputs(wl, 1)
        d = (o0 - o1).abs()
        print(f"{wl.name}: max|dO| {d.max().item():.3e}  rel-L2 {(d.norm() / o1.norm()).item():.3e}  "
              f"max|dLSE| {(l0 - l1).abs().max().item():.3e}", flush=True)
    for wl in cases[1:]:
        for path in (1, 0):
            print(f"decode_path={path}", end=" ")
            time_it(wl, tuning=dict(decode_path=path))
    if "--blocks" in sys.argv:
        for B in (32, 64):
            s = W.Shape(32, 8, 128, B, "bf16")
            for wl in (W.hybrid(s, f"decode-only-64-B{B}", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2),
                       W.hybrid(s, f"config2-B{B}", prefill_offset=1536, chunk=512, decode_ctx=W.l8b_decode_ctx(), seed=2)):
                for path in (1, 0):
                    print(f"decode_path={path}", end=" ")
                    time_it(wl, tuning=dict(decode_path=path))


if __name__ == "__main__":
    main()
