"""Prefill-heavy timing set for A/B of kernel variants (NIYAMA_LIB_PATH selects the build):
median of back-to-back launches (tools/kbench.time_it).

    python tools/ab_prefill.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402


def main():
    print("lib:", os.environ.get("NIYAMA_LIB_PATH", "in-tree"), flush=True)
    for wl in (W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4),
               W.config4_l70b(),
               W.hybrid(W.L8B, "l8b-prefill-c2048-o2048", prefill_offset=2048, chunk=2048, decode_ctx=[], seed=4),
               W.hybrid(W.L8B, "l8b-prefill-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2),
               W.config2_l8b(),
               W.hybrid(W.L8B, "decode-only-64", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2)):
        time_it(wl, reps=30)


if __name__ == "__main__":
    main()
