"""A/B of one niyama_tuning field on configs 2 and 4 and a decode-only batch (median of
back-to-back launches, tools/kbench.time_it).

    python tools/ab_tuning.py FIELD V0 V1 [--no-l70b]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402


def main():
    field, v0, v1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    cases = [W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2),
             W.config2_l8b(),
             W.hybrid(W.L8B, "decode-only-16", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(16), seed=2)]
    if "--no-l70b" not in sys.argv:
        cases.append(W.config4_l70b())
    for wl in cases:
        for v in (v0, v1, v0, v1):
            print(f"{field}={v}", end=" ")
            time_it(wl, tuning={field: v})


if __name__ == "__main__":
    main()
