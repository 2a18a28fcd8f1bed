"""A/B of the §8(f)2 fused all-gather at world size 1: niyama_hybrid_attention (plain stores)
against niyama_attention_gather (stores through the window mapping + system fences + the
flag barrier) on the same plan, alternating rounds of back-to-back launches.  The library
under test comes from NIYAMA_LIB_PATH (tools/build_variant.py variants).

    python tools/ab_gather.py [--reps 50] [--rounds 7]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
import workloads as W  # noqa: E402
from kbench import setup  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--rounds", type=int, default=7)
    args = ap.parse_args()
    lib = os.environ.get("NIYAMA_LIB_PATH", "default")
    cases = [W.config2_l8b(), W.hybrid(W.L8B, "decode-only-D64", prefill_offset=0, chunk=0,
                                       decode_ctx=[int(x) for x in W.rng(0).integers(1, 4097, size=64)], seed=0),
             W.config4_l70b()]
    for wl in cases:
        kv, plan, q, o, lse = setup(wl)
        kv.comm_init(ny.get_unique_id())
        win = kv.gather_window(wl.final.desc.num_rows)
        wo, wl_ = kv.attention_gather(plan, 0, q, win)   # a window buffer, written by the plain launch below
        modes = {"plain": lambda: kv.attention(plan, 0, q, o, lse),
                 "gather": lambda: kv.attention_gather(plan, 0, q, win),
                 "plain_into_window": lambda: kv.attention(plan, 0, q, wo, wl_)}
        res = {m: [] for m in modes}
        for f in modes.values():
            for _ in range(5):
                f()
        for _ in range(args.rounds):
            for m, f in modes.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.reps):
                    f()
                e1.record()
                torch.cuda.synchronize()
                res[m].append(e0.elapsed_time(e1) * 1e3 / args.reps)
        a, b = statistics.median(res["plain"]), statistics.median(res["gather"])
        c = statistics.median(res["plain_into_window"])
        ok = torch.equal(o.view(torch.int16), kv.attention_gather(plan, 0, q, win)[0].view(torch.int16))
        torch.cuda.synchronize()
        print(f"{os.path.basename(lib):24s} {wl.name:36s} plain {a:8.1f} us  gather {b:8.1f} us  "
              f"delta {b - a:+6.1f} us  plain->window {c:8.1f} us  bitwise={ok}", flush=True)
        win.close()
        kv.close()


if __name__ == "__main__":
    main()
